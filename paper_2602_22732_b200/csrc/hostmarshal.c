/*
 * _hostmarshal -- native result marshalling for the drop-in Python API.
 *
 * The reference returns, per request, a new list of (SemanticId, float)
 * pairs (pkg/src/adrec/serving/beam.py:212-213).  The decode leaves them as
 * three flat host arrays (count, tokens, score; gr4ad_results).  Building
 * hundreds of thousands of Python objects from those in interpreted Python
 * costs ~0.35 us per result; this CPython extension builds the same objects
 * directly (token ints from a prebuilt table, SemanticId tuples allocated as
 * the per-vocabulary tuple subclass, cyclic GC paused), ~10x faster.
 *
 *   build(count, tokens, score, max_out, T, vocab, sid_type)
 *     count  int32 buffer [B], tokens int32 buffer [B*max_out*T],
 *     score  float64 buffer [B*max_out], vocab tuple of T ints,
 *     sid_type the SemanticId subclass of that vocabulary.
 *   -> [[(sid, score), ...] per request]; ValueError (the SemanticId
 *      message) if a live token is out of range.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <stdint.h>

#define MAX_T 8

static PyObject **g_ints = NULL; /* g_ints[v] = PyLong(v), v < g_nints */
static Py_ssize_t g_nints = 0;

static int ensure_ints(Py_ssize_t n) {
  if (n <= g_nints) return 0;
  PyObject **tab = (PyObject **)PyMem_Realloc(g_ints, sizeof(PyObject *) * (size_t)n);
  if (!tab) {
    PyErr_NoMemory();
    return -1;
  }
  g_ints = tab;
  for (Py_ssize_t v = g_nints; v < n; ++v) {
    g_ints[v] = PyLong_FromSsize_t(v);
    if (!g_ints[v]) {
      g_nints = v;
      return -1;
    }
  }
  g_nints = n;
  return 0;
}

static PyObject *build(PyObject *self, PyObject *args) {
  Py_buffer cb, tb, sb;
  Py_ssize_t max_out, T;
  PyObject *vocab, *sid_type;
  if (!PyArg_ParseTuple(args, "y*y*y*nnOO", &cb, &tb, &sb, &max_out, &T, &vocab, &sid_type))
    return NULL;
  PyObject *result = NULL;
  int gc_was = -1;
  long vv[MAX_T];
  if (T < 1 || T > MAX_T || !PyTuple_Check(vocab) || PyTuple_GET_SIZE(vocab) != T ||
      !PyType_Check(sid_type) || max_out < 0) {
    PyErr_SetString(PyExc_ValueError, "tokens and level_vocab_sizes must be equal, nonzero length");
    goto done;
  }
  Py_ssize_t vmax = 0;
  for (Py_ssize_t t = 0; t < T; ++t) {
    vv[t] = PyLong_AsLong(PyTuple_GET_ITEM(vocab, t));
    if (vv[t] < 1) {
      if (!PyErr_Occurred()) PyErr_SetString(PyExc_ValueError, "vocabulary sizes must be positive");
      goto done;
    }
    if (vv[t] > vmax) vmax = vv[t];
  }
  const Py_ssize_t B = cb.len / (Py_ssize_t)sizeof(int32_t);
  const int32_t *count = (const int32_t *)cb.buf;
  const int32_t *tok = (const int32_t *)tb.buf;
  const double *score = (const double *)sb.buf;
  for (Py_ssize_t b = 0; b < B; ++b) {
    const Py_ssize_t n = count[b];
    if (n < 0 || n > max_out || (b + 1) * max_out * T * (Py_ssize_t)sizeof(int32_t) > tb.len ||
        (b + 1) * max_out * (Py_ssize_t)sizeof(double) > sb.len) {
      PyErr_SetString(PyExc_ValueError, "result buffers do not match count / max_out");
      goto done;
    }
    const int32_t *row = tok + b * max_out * T;
    for (Py_ssize_t j = 0; j < n * T; ++j) {
      const long t = (long)(j % T);
      if (row[j] < 0 || row[j] >= vv[t]) {
        PyErr_Format(PyExc_ValueError, "token %d out of range [0, %ld) at level %ld", row[j],
                     vv[t], t);
        goto done;
      }
    }
  }
  if (ensure_ints(vmax) < 0) goto done;
  gc_was = PyGC_Disable();
  PyTypeObject *st = (PyTypeObject *)sid_type;
  result = PyList_New(B);
  if (!result) goto done;
  for (Py_ssize_t b = 0; b < B; ++b) {
    const Py_ssize_t n = count[b];
    PyObject *lst = PyList_New(n);
    if (!lst) goto fail;
    PyList_SET_ITEM(result, b, lst);
    const int32_t *row = tok + b * max_out * T;
    const double *sc = score + b * max_out;
    for (Py_ssize_t j = 0; j < n; ++j) {
      PyObject *sid = st->tp_alloc(st, T);
      if (!sid) goto fail;
      for (Py_ssize_t t = 0; t < T; ++t) {
        PyObject *o = g_ints[row[j * T + t]];
        Py_INCREF(o);
        PyTuple_SET_ITEM(sid, t, o);
      }
      PyObject *f = PyFloat_FromDouble(sc[j]);
      if (!f) {
        Py_DECREF(sid);
        goto fail;
      }
      PyObject *pair = PyTuple_New(2);
      if (!pair) {
        Py_DECREF(sid);
        Py_DECREF(f);
        goto fail;
      }
      PyTuple_SET_ITEM(pair, 0, sid);
      PyTuple_SET_ITEM(pair, 1, f);
      /* Both hold only ints / a float and are immutable: they can never be
         part of a reference cycle, so they leave the cyclic GC's lists (as
         CPython does for such plain tuples).  A serving process keeps
         millions of them alive in its TTL cache; tracked, every full
         collection would walk them all (100s of ms pauses). */
      PyObject_GC_UnTrack(sid);
      PyObject_GC_UnTrack(pair);
      PyList_SET_ITEM(lst, j, pair);
    }
  }
  goto done;
fail:
  Py_CLEAR(result);
done:
  if (gc_was == 1) PyGC_Enable();
  PyBuffer_Release(&cb);
  PyBuffer_Release(&tb);
  PyBuffer_Release(&sb);
  return result;
}

static PyMethodDef methods[] = {
    {"build", build, METH_VARARGS, "per-request [(SemanticId, score)] lists from result buffers"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_hostmarshal", NULL, -1, methods};

PyMODINIT_FUNC PyInit__hostmarshal(void) { return PyModule_Create(&module); }
