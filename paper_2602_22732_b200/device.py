"""Device residency: fp32 weight snapshots, context tensors, batch plans.

Weights are packed once per snapshot into one contiguous fp32 CUDA buffer
(the SnapshotStore contract, engine.py:17-36: a re-upload happens only when
the published parameters change).  Per-layer self Q/K/V are concatenated
to (d, 3d) and every layer's cross K/V projection to one (d, 2Ld) matrix so
the encoder pass is a single GEMM over all requests' context rows.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N
from .model.decoder import param_array

_ALIGN = 64  # floats (256 B) between packed tensors


class _CaptureGate:
    """Readers-writer gate between CUDA-graph capture and the package's other
    device work.  While a stream captures, CUDA rejects work that implicitly
    synchronises with it from any thread (e.g. a copy on the legacy default
    stream), so the one-time capture of a pooled decoder's graph runs
    exclusively; every other device call of the package holds the gate
    shared (concurrent decodes proceed together)."""

    def __init__(self):
        self._cv = threading.Condition()
        self._readers = 0
        self._writer = False
        self._local = threading.local()

    def _depth(self):
        return getattr(self._local, "depth", 0)

    @contextlib.contextmanager
    def shared(self):
        if self._depth():  # re-entrant inside either mode
            yield
            return
        with self._cv:
            while self._writer:
                self._cv.wait()
            self._readers += 1
        self._local.depth = 1
        try:
            yield
        finally:
            self._local.depth = 0
            with self._cv:
                self._readers -= 1
                self._cv.notify_all()

    @contextlib.contextmanager
    def exclusive(self):
        if self._depth():
            raise RuntimeError("graph capture requested inside a device call")
        with self._cv:
            while self._writer or self._readers:
                self._cv.wait()
            self._writer = True
        self._local.depth = 1
        try:
            yield
        finally:
            self._local.depth = 0
            with self._cv:
                self._writer = False
                self._cv.notify_all()


CAPTURE_GATE = _CaptureGate()


def gated(fn):
    """Run ``fn`` holding the capture gate shared (see _CaptureGate)."""
    import functools

    @functools.wraps(fn)
    def wrapper(*a, **kw):
        with CAPTURE_GATE.shared():
            return fn(*a, **kw)
    return wrapper


def _stream_handle(device=None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


_HAS_CUDA = []


def require_cuda(device=None):
    # torch.cuda.is_available() re-queries the driver (~0.2 ms a call): once
    if not _HAS_CUDA:
        _HAS_CUDA.append(torch.cuda.is_available())
    if not _HAS_CUDA[0]:
        raise RuntimeError("paper_2602_22732_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device(device if device is not None else "cuda")


def dims_of(cfg, trunk_depth=None):
    if cfg.n_levels > N.MAX_LEVELS:
        raise RuntimeError(f"n_levels {cfg.n_levels} > {N.MAX_LEVELS}")
    if cfg.n_layers > N.MAX_LAYERS:
        raise RuntimeError(f"n_layers {cfg.n_layers} > {N.MAX_LAYERS}")
    dm = N.Dims()
    dm.feat_dim, dm.d, dm.d_ff = cfg.feat_dim, cfg.d, cfg.d_ff
    dm.n_layers = cfg.n_layers
    dm.trunk_depth = cfg.trunk_depth if trunk_depth is None else trunk_depth
    dm.n_levels = cfg.n_levels
    dm.n_value_buckets = cfg.n_value_buckets
    for t, v in enumerate(cfg.level_vocab_sizes):
        dm.vocab[t] = int(v)
    return dm


class DeviceWeights:
    """fp32 copy of ``DecoderModel.params`` on one device + the C struct of
    pointers into it (gr4ad_weights).

    With ``stream`` the upload is asynchronous: the packed host image is
    pinned, copied on ``stream`` and ``ready`` records its completion, so a
    snapshot can be published while decodes keep running on the previous
    one (consumers order themselves after ``ready`` on the GPU via
    :func:`device_weights`, never by blocking the host)."""

    def __init__(self, model, device=None, stream=None):
        device = require_cuda(device)
        cfg = model.config
        P = {k: param_array(v) for k, v in model.params.items()}
        d, L = cfg.d, cfg.n_layers
        pieces = OrderedDict()
        for name in ("ctx.W", "ctx.b", "pos", "bos", "fuse.Wg", "fuse.Wf", "head.value"):
            pieces[name] = P[name]
        for t in range(cfg.n_levels):
            pieces[f"emb.{t}"] = P[f"emb.{t}"]
            pieces[f"head.{t}"] = P[f"head.{t}"]
        pieces["cross_kv"] = np.concatenate(
            [np.concatenate([P[f"layer{i}.cross.Wk"], P[f"layer{i}.cross.Wv"]], axis=1)
             for i in range(L)], axis=1)
        for i in range(L):
            pre = f"layer{i}."
            for n in ("ln1.g", "ln1.b", "cross.Wq", "cross.Wo", "ln2.g", "ln2.b", "self.Wo",
                      "ln3.g", "ln3.b", "ffn.W1", "ffn.b1", "ffn.W2", "ffn.b2"):
                pieces[pre + n] = P[pre + n]
            pieces[pre + "self.Wqkv"] = np.concatenate(
                [P[pre + "self.Wq"], P[pre + "self.Wk"], P[pre + "self.Wv"]], axis=1)
        offs, total = {}, 0
        for k, a in pieces.items():
            offs[k] = total
            total += (a.size + _ALIGN - 1) // _ALIGN * _ALIGN
        host = np.zeros(total, dtype=np.float32)
        for k, a in pieces.items():
            host[offs[k]:offs[k] + a.size] = a.astype(np.float32).ravel()
        self._pinned = None
        if stream is None:
            self.buffer = torch.from_numpy(host).to(device)
            self.ready = None
        else:
            pinned = torch.from_numpy(host).pin_memory()
            with torch.cuda.stream(stream):
                self.buffer = torch.empty(host.size, dtype=torch.float32, device=device)
                self.buffer.copy_(pinned, non_blocking=True)
                self.ready = torch.cuda.Event()
                self.ready.record(stream)
            self._pinned = pinned  # alive until the copy has run
        self.device = device
        self.config = cfg
        self.nbytes = host.nbytes
        base = self.buffer.data_ptr()
        ptr = lambda k: C.c_void_p(base + 4 * offs[k])
        w = N.Weights()
        w.ctx_W, w.ctx_b, w.pos, w.bos = ptr("ctx.W"), ptr("ctx.b"), ptr("pos"), ptr("bos")
        w.fuse_Wg, w.fuse_Wf, w.head_value = ptr("fuse.Wg"), ptr("fuse.Wf"), ptr("head.value")
        w.cross_kv_W = ptr("cross_kv")
        for t in range(cfg.n_levels):
            w.emb[t] = ptr(f"emb.{t}")
            w.head[t] = ptr(f"head.{t}")
        for i in range(L):
            pre = f"layer{i}."
            lw = w.layer[i]
            lw.ln1_g, lw.ln1_b = ptr(pre + "ln1.g"), ptr(pre + "ln1.b")
            lw.cross_Wq, lw.cross_Wo = ptr(pre + "cross.Wq"), ptr(pre + "cross.Wo")
            lw.ln2_g, lw.ln2_b = ptr(pre + "ln2.g"), ptr(pre + "ln2.b")
            lw.self_Wqkv, lw.self_Wo = ptr(pre + "self.Wqkv"), ptr(pre + "self.Wo")
            lw.ln3_g, lw.ln3_b = ptr(pre + "ln3.g"), ptr(pre + "ln3.b")
            lw.ffn_W1, lw.ffn_b1 = ptr(pre + "ffn.W1"), ptr(pre + "ffn.b1")
            lw.ffn_W2, lw.ffn_b2 = ptr(pre + "ffn.W2"), ptr(pre + "ffn.b2")
        self.struct = w
        self._derived = {}  # layout signature -> prepared derived-weight buffer
        self._derived_lock = threading.Lock()

    def derived_buffer(self, signature, nbytes, prepare):
        """The snapshot's derived weight copies for one plan layout
        (gr4ad_derived_layout signature): built once by ``prepare(buf)`` and
        shared by every decoder of this snapshot with that layout, so a new
        batch shape or width schedule costs no weight preparation."""
        with self._derived_lock:
            buf = self._derived.get(signature)
            if buf is None:
                buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=self.device)
                prepare(buf)  # synchronous; raises (RangeError) before caching
                self._derived[signature] = buf
            return buf

    def use_on(self, stream=None):
        """Order ``stream`` (default: current) after the upload and tell the
        allocator the buffer is in use there, so a replaced snapshot's memory
        is recycled only after the decodes reading it have finished."""
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.ready is not None:
            stream.wait_event(self.ready)
            self.buffer.record_stream(stream)
            if self._pinned is not None and self.ready.query():
                self._pinned = None
        return self


_CACHE_LOCK = threading.Lock()
_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_MAX = 4


def _fingerprint(params):
    fp = []
    for k, v in params.items():
        a = getattr(v, "data", v)
        flat = np.asarray(a).ravel()
        fp.append((k, id(a), flat.size,
                   float(flat[0]) if flat.size else 0.0,
                   float(flat[-1]) if flat.size else 0.0,
                   float(flat[flat.size // 2]) if flat.size else 0.0))
    return tuple(fp)


def _freeze(params, frozen=True):
    """Mark the host parameter arrays read-only while a device copy of them
    is resident, so an in-place edit (``params[k].data[i] = ...``) raises
    instead of silently decoding with stale GPU weights; replacing an array
    (``params[k].data = new``) re-uploads.  :func:`invalidate` lifts it."""
    for v in params.values():
        a = getattr(v, "data", v)
        if isinstance(a, np.ndarray):
            try:
                a.flags.writeable = not frozen
            except ValueError:  # a view of a read-only base: stays as it is
                pass


def device_weights(model, device=None):
    """Resident weights for ``model``: uploaded once and reused while the
    parameter arrays are the same objects (their identity is the key; the
    arrays are made read-only while resident -- call :func:`invalidate`
    before editing them in place)."""
    device = require_cuda(device)
    key = (id(model.params), str(device))
    fp = _fingerprint(model.params)
    with CAPTURE_GATE.shared():
        with _CACHE_LOCK:
            hit = _CACHE.get(key)
            if hit is not None and hit[0] == fp:
                _CACHE.move_to_end(key)
                return hit[2].use_on()
        dw = DeviceWeights(model, device)
        register(model, dw)
        return dw


def register(model, dw):
    """Make ``dw`` the resident copy of ``model`` (used by snapshot publish
    to pre-stage weights before the first decode asks for them)."""
    key = (id(model.params), str(dw.device))
    _freeze(model.params)
    with _CACHE_LOCK:
        _CACHE[key] = (_fingerprint(model.params), model.params, dw)
        _CACHE.move_to_end(key)
        while len(_CACHE) > _CACHE_MAX:
            _, (_, params, _) = _CACHE.popitem(last=False)
            if not any(p is params for _, p, _ in _CACHE.values()):
                _freeze(params, False)


def invalidate(model=None):
    """Drop resident copies (of ``model``, or all) and make their host
    arrays writeable again; the next decode re-uploads."""
    with _CACHE_LOCK:
        if model is None:
            for _, params, _ in _CACHE.values():
                _freeze(params, False)
            _CACHE.clear()
        else:
            for k in [k for k in _CACHE if k[0] == id(model.params)]:
                del _CACHE[k]
            _freeze(model.params, False)
    from .decode import POOL
    POOL.clear()


class DeviceContext:
    """Projected context X resident on the GPU (fp32), with the reference
    Tensor's ``.data`` / ``.shape`` view for drop-in callers."""

    def __init__(self, x):
        self.tensor = x

    @property
    def shape(self):
        return tuple(self.tensor.shape)

    @property
    def ndim(self):
        return self.tensor.dim()

    @property
    def data(self):
        return self.tensor.double().cpu().numpy()


@gated
def context_process_gpu(features, params):
    device = require_cuda()
    feats = np.atleast_2d(np.asarray(getattr(features, "data", features), dtype=np.float64))
    W = param_array(params["ctx.W"])
    if feats.shape[-1] != W.shape[0]:
        raise ValueError(f"feature dim {feats.shape[-1]} != expected {W.shape[0]}")
    rows = feats.shape[0]
    d = W.shape[1]
    f = torch.from_numpy(feats.astype(np.float32)).to(device)
    w = torch.from_numpy(W.astype(np.float32)).to(device)
    b = torch.from_numpy(param_array(params["ctx.b"]).astype(np.float32)).to(device)
    x = torch.empty((rows, d), dtype=torch.float32, device=device)
    ws = N.Weights()
    ws.ctx_W, ws.ctx_b = C.c_void_p(w.data_ptr()), C.c_void_p(b.data_ptr())
    dm = N.Dims()
    dm.feat_dim, dm.d = W.shape[0], d
    if rows:
        N.check(N.lib.gr4ad_context_process(C.byref(dm), C.byref(ws), C.c_void_p(f.data_ptr()),
                                            rows, C.c_void_p(x.data_ptr()), _stream_handle()))
    return DeviceContext(x)
