"""CPU oracle for the GR4AD LazyAR beam-serving hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may call it, and there only as
the checker or the CPU baseline, never as the thing measured or shipped.

It is a float64 numpy restatement of the reference algorithm
(``/root/reference/pkg/src/adrec``; file:line cited per function).  It is
pinned against the reference itself: ``tests/golden/make_golden.py``
imports the unmodified reference in the build container and records its
outputs as fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this module against every fixture (and against the reference's own
known-answer tests restated in ``tests/test_oracle_known_answers.py``).

Structure differs from the reference on purpose: beams are processed as a
(rows, d) matrix of *live* rows instead of padded (slots, 1, d) stacks, and
selection is an exact threshold + lexsort instead of a per-row Python loop.
Both are result-identical to the reference (padding rows carry -inf scores
and are dropped by its alive filter, beam.py:200-203; pre-cut is exact,
beam.py:50-60).

The one extension that is NOT in the reference -- valid-SID prefix masking
(``valid_sids=``) -- is marked "parity unpinned" below: the reference has no
such mask (engine.py:114-118 filters afterwards), so that mode is checked
only against this restatement.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np

LN_EPS = 1e-5  # layers.py:15


@dataclass(frozen=True)
class OracleConfig:
    """Mirror of ``DecoderConfig`` (decoder.py:32-51)."""

    feat_dim: int
    d: int
    d_ff: int
    n_layers: int
    trunk_depth: int
    level_vocab_sizes: tuple
    n_value_buckets: int
    seed: int = 0

    @property
    def n_levels(self):
        return len(self.level_vocab_sizes)


def as_config(cfg):
    if isinstance(cfg, OracleConfig):
        return cfg
    return OracleConfig(int(cfg.feat_dim), int(cfg.d), int(cfg.d_ff),
                        int(cfg.n_layers), int(cfg.trunk_depth),
                        tuple(int(v) for v in cfg.level_vocab_sizes),
                        int(cfg.n_value_buckets), int(getattr(cfg, "seed", 0)))


def plain_params(params):
    """str -> float64 ndarray, accepting autodiff Tensors (``.data``)."""
    return {k: np.asarray(getattr(v, "data", v), dtype=np.float64)
            for k, v in params.items()}


# ---------------------------------------------------------------------------
# parameters (decoder.py:54-107)
# ---------------------------------------------------------------------------

_LAYER_ORDER = (
    ("ln1.g", "1"), ("ln1.b", "0"),
    ("cross.Wq", "dd"), ("cross.Wk", "dd"), ("cross.Wv", "dd"), ("cross.Wo", "dd"),
    ("ln2.g", "1"), ("ln2.b", "0"),
    ("self.Wq", "dd"), ("self.Wk", "dd"), ("self.Wv", "dd"), ("self.Wo", "dd"),
    ("ln3.g", "1"), ("ln3.b", "0"),
    ("ffn.W1", "d_ff"), ("ffn.b1", "0ff"), ("ffn.W2", "ff_d"), ("ffn.b2", "0"),
)


def init_params(cfg):
    """Seeded uniform(+-1/sqrt(fan_in)) init in the reference's draw order
    (decoder.py:71-107).  LN gains 1, biases 0, no draws for those."""
    cfg = as_config(cfg)
    rng = np.random.default_rng(cfg.seed)
    d, dff = cfg.d, cfg.d_ff

    def u(shape, fan_in):
        s = 1.0 / np.sqrt(fan_in)
        return rng.uniform(-s, s, size=shape)

    p = {"ctx.W": u((cfg.feat_dim, d), cfg.feat_dim), "ctx.b": np.zeros(d),
         "pos": u((cfg.n_levels + 1, d), d), "bos": u((d,), d)}
    for t, v in enumerate(cfg.level_vocab_sizes):
        p[f"emb.{t}"] = u((v, d), d)
    for i in range(cfg.n_layers):
        for name, kind in _LAYER_ORDER:
            key = f"layer{i}.{name}"
            if kind == "1":
                p[key] = np.ones(d)
            elif kind == "0":
                p[key] = np.zeros(d)
            elif kind == "0ff":
                p[key] = np.zeros(dff)
            elif kind == "dd":
                p[key] = u((d, d), d)
            elif kind == "d_ff":
                p[key] = u((d, dff), d)
            else:
                p[key] = u((dff, d), dff)
    p["fuse.Wg"] = u((d, d), d)
    p["fuse.Wf"] = u((2 * d, d), 2 * d)
    for t, v in enumerate(cfg.level_vocab_sizes):
        p[f"head.{t}"] = u((d, v), d)
    p["head.value"] = u((d, cfg.n_value_buckets), d)
    return p


# ---------------------------------------------------------------------------
# arithmetic (autodiff.py forward semantics; layers.py)
# ---------------------------------------------------------------------------

def context_process(features, params):
    """X = F W_c + b_c (decoder.py:134-140)."""
    f = np.atleast_2d(np.asarray(features, dtype=np.float64))
    if f.shape[-1] != params["ctx.W"].shape[0]:
        raise ValueError(f"feature dim {f.shape[-1]} != expected {params['ctx.W'].shape[0]}")
    return f @ params["ctx.W"] + params["ctx.b"]


def layer_norm(x, g, b):
    """Biased-variance LN, eps 1e-5 (layers.py:38-43)."""
    mean = x.mean(axis=-1, keepdims=True)
    c = x - mean
    var = (c * c).mean(axis=-1, keepdims=True)
    return c * (var + LN_EPS) ** -0.5 * g + b


def softmax(a):
    """exp(log_softmax(a)) with the max-shifted logsumexp (autodiff.py:351-368)."""
    shift = a.max(axis=-1, keepdims=True)
    lse = np.log(np.exp(a - shift).sum(axis=-1, keepdims=True)) + shift
    return np.exp(a - lse)


def gelu(a):
    """tanh GELU (autodiff.py:301-306)."""
    c = np.sqrt(2.0 / np.pi)
    return 0.5 * a * (1.0 + np.tanh((a + 0.044715 * a ** 3) * c))


def log_softmax_rows(logits):
    """beam.py:92-95."""
    mx = logits.max(axis=-1, keepdims=True)
    sh = logits - mx
    return sh - np.log(np.exp(sh).sum(axis=-1, keepdims=True))


def _attend(q, k, v, wo, causal=False):
    """Single-head attention, scale 1/sqrt(d) (layers.py:46-51).
    q (..., n, d), k/v (..., m, d)."""
    d = q.shape[-1]
    s = (q @ np.swapaxes(k, -1, -2)) * (1.0 / np.sqrt(d))
    if causal:
        n = s.shape[-1]
        s = np.where(np.tril(np.ones((n, n), dtype=bool)), s, -np.inf)
    return (softmax(s) @ v) @ wo


def fuse(m, s, wf, wg):
    """concat(m * (s W_g), s) W_f (layers.py:129-133)."""
    gate = s @ wg
    return np.concatenate([m * gate, s], axis=-1) @ wf


def _lp(params, i, name):
    return params[f"layer{i}.{name}"]


def decoder_layer_2d(params, i, states, x):
    """Teacher-forced pre-LN layer, causal self-attention, cross K/V built
    from the context inside the layer (layers.py:66-119, 2-D branch)."""
    P = lambda n: _lp(params, i, n)
    n1 = layer_norm(states, P("ln1.g"), P("ln1.b"))
    h = states + _attend(n1 @ P("cross.Wq"), x @ P("cross.Wk"), x @ P("cross.Wv"),
                         P("cross.Wo"))
    n2 = layer_norm(h, P("ln2.g"), P("ln2.b"))
    h = h + _attend(n2 @ P("self.Wq"), n2 @ P("self.Wk"), n2 @ P("self.Wv"),
                    P("self.Wo"), causal=True)
    n3 = layer_norm(h, P("ln3.g"), P("ln3.b"))
    return h + gelu(n3 @ P("ffn.W1") + P("ffn.b1")) @ P("ffn.W2") + P("ffn.b2")


def decoder_layer_step(params, i, h, ck, cv, past_k, past_v):
    """Incremental layer for a (rows, d) stack of beam states against a
    shared (S, d) context K/V and a (rows, t, d) self-KV history
    (layers.py:66-119, 3-D branch; beam.py:221-255).  Returns the new
    states and the (rows, t+1, d) history."""
    P = lambda n: _lp(params, i, n)
    d = h.shape[-1]
    n1 = layer_norm(h, P("ln1.g"), P("ln1.b"))
    h = h + _attend(n1 @ P("cross.Wq"), ck, cv, P("cross.Wo"))
    n2 = layer_norm(h, P("ln2.g"), P("ln2.b"))
    q = n2 @ P("self.Wq")
    k = np.concatenate([past_k, (n2 @ P("self.Wk"))[:, None, :]], axis=1)
    v = np.concatenate([past_v, (n2 @ P("self.Wv"))[:, None, :]], axis=1)
    s = np.einsum("rd,rtd->rt", q, k) * (1.0 / np.sqrt(d))
    a = np.einsum("rt,rtd->rd", softmax(s), v) @ P("self.Wo")
    h = h + a
    n3 = layer_norm(h, P("ln3.g"), P("ln3.b"))
    h = h + gelu(n3 @ P("ffn.W1") + P("ffn.b1")) @ P("ffn.W2") + P("ffn.b2")
    return h, k, v


def run_layers_2d(params, states, x, lo, hi):
    """decoder.py:155-159."""
    for i in range(lo, hi):
        states = decoder_layer_2d(params, i, states, x)
    return states


# ---------------------------------------------------------------------------
# selection (beam.py:30-89; verify.py:366-373)
# ---------------------------------------------------------------------------

def select_topk(total, k, drop_inf=True):
    """Top-k of a (rows, V) score matrix under the (-score, row, token)
    order of beam.py:30-34 / 76.  With ``drop_inf`` the -inf entries are
    removed afterwards, as the alive filter does (beam.py:202-203).
    Returns rows, tokens, scores."""
    rows, v = total.shape
    flat = total.ravel()
    n = flat.size
    k = min(int(k), n)
    if k <= 0:
        e = np.zeros(0, dtype=np.int64)
        return e, e, np.zeros(0)
    if k < n:
        part = np.argpartition(-flat, k - 1)[:k]
        thr = flat[part].min()
        above = np.flatnonzero(flat > thr)
        ties = np.flatnonzero(flat == thr)[: k - above.size]
        cand = np.concatenate([above, ties])
    else:
        cand = np.arange(n)
    cand = cand[np.lexsort((cand, -flat[cand]))]
    sc = flat[cand]
    if drop_inf:
        keep = np.isfinite(sc)
        cand, sc = cand[keep], sc[keep]
    return (cand // v).astype(np.int64), (cand % v).astype(np.int64), sc


def topk_precut(prev_scores, logprobs, k):
    """Public pre-cut selection (beam.py:50-60): list of (beam, token, score);
    like the reference it applies no alive filter."""
    total = np.asarray(prev_scores, dtype=np.float64)[:, None] + np.asarray(
        logprobs, dtype=np.float64)
    b, t, s = select_topk(total, k, drop_inf=False)
    return list(zip(b.tolist(), t.tolist(), s.tolist()))


def topk_global(beam_scores, logprobs, k):
    """Exhaustive selection (beam.py:37-47): arrays (beams, tokens, scores)."""
    total = np.asarray(beam_scores, dtype=np.float64)[:, None] + np.asarray(
        logprobs, dtype=np.float64)
    return select_topk(total, k, drop_inf=False)


def precut_oracle(beam_scores, logprobs, k):
    """Brute-force ranking, pure Python (verify.py:366-373)."""
    b, v = logprobs.shape
    triples = [(float(beam_scores[i] + logprobs[i, j]), i, j)
               for i in range(b) for j in range(v)]
    triples.sort(key=lambda r: (-r[0], r[1], r[2]))
    return [(i, j, s) for s, i, j in triples[: min(k, b * v)]]


# ---------------------------------------------------------------------------
# widths (beam.py:134-139) and counters (layers.py:18-35, beam.py:168-169,238-239)
# ---------------------------------------------------------------------------

def effective_widths(widths, vocab_sizes):
    eff, reach = [], 1
    for w, v in zip(widths, vocab_sizes):
        reach = min(reach * v, 1 << 40)
        eff.append(min(int(w), reach))
    return eff


def live_counts(eff, vocab_sizes):
    """Rows entering each level and rows surviving the last one, without
    prefix masking: live_{t+1} = min(eff_t, live_t * V_t)."""
    live = [1]
    for e, v in zip(eff, vocab_sizes):
        live.append(min(e, live[-1] * v))
    return live


def counter_closed_form(cfg, widths, s_ctx, shared_kv=True, value_rerank=False,
                        trunk_depth=None):
    """What ``LayerCallCounter`` records for one beam_search call."""
    cfg = as_config(cfg)
    k = cfg.trunk_depth if trunk_depth is None else trunk_depth
    T, L, d = cfg.n_levels, cfg.n_layers, cfg.d
    eff = effective_widths(widths, cfg.level_vocab_sizes)
    live = live_counts(eff, cfg.level_vocab_sizes)
    n_pos = T + (1 if value_rerank else 0)
    calls = k * n_pos if k > 0 else 0
    builds, floats = 0, 0
    if shared_kv:
        builds, floats = 1, (L - k) * 2 * s_ctx * d
    for t in range(T):
        slots = max(eff[t], live[t])
        calls += (L - k) * slots
        if not shared_kv:
            builds += slots
            floats = max(floats, (L - k) * 2 * slots * s_ctx * d)
    if value_rerank:
        calls += (L - k) * live[T]
        if not shared_kv:
            builds += live[T]
            floats = max(floats, (L - k) * 2 * live[T] * s_ctx * d)
    return calls, builds, floats


# ---------------------------------------------------------------------------
# beam search (beam.py:112-288)
# ---------------------------------------------------------------------------

def prefix_mask(valid_sids, vocab_sizes, t, prefixes):
    """PARITY UNPINNED (no reference counterpart): boolean (rows, V_t) mask of
    tokens whose extended prefix is a prefix of some valid SID."""
    allowed = {}
    for sid in valid_sids:
        key = tuple(int(x) for x in sid[:t])
        allowed.setdefault(key, set()).add(int(sid[t]))
    m = np.zeros((prefixes.shape[0], vocab_sizes[t]), dtype=bool)
    for r in range(prefixes.shape[0]):
        for tok in allowed.get(tuple(int(x) for x in prefixes[r]), ()):
            m[r, tok] = True
    return m


def beam_search(params, cfg, context, widths, value_rerank=False,
                representatives=None, trunk_depth=None, valid_sids=None,
                record=None):
    """Float64 beam decode of one request.

    ``context`` is the projected X (S, d).  Returns ``[(tokens, score)]`` in
    selection order (or value-rerank order).  ``record`` (a list) receives
    per-level dicts with the selected (parent, token, score) arrays and the
    score gap at the cut, for parity diagnostics.
    """
    cfg = as_config(cfg)
    params = plain_params(params)
    x = np.atleast_2d(np.asarray(context, dtype=np.float64))
    if x.size == 0:
        raise ValueError("empty context")
    if not np.isfinite(x).all():
        raise ValueError("context must be finite")
    T = cfg.n_levels
    if len(widths) != T:
        raise ValueError(f"schedule has {len(widths)} widths for {T} levels")
    eff = effective_widths(widths, cfg.level_vocab_sizes)
    K = cfg.trunk_depth if trunk_depth is None else trunk_depth
    if not 0 <= K < cfg.n_layers:
        raise ValueError("trunk_depth must satisfy 0 <= K < n_layers")
    heads = list(range(K, cfg.n_layers))
    d = cfg.d
    n_pos = T + (1 if value_rerank else 0)
    pos = params["pos"][:n_pos]
    trunk = run_layers_2d(params, pos, x, 0, K) if K > 0 else pos
    kv = {i: (x @ _lp(params, i, "cross.Wk"), x @ _lp(params, i, "cross.Wv"))
          for i in heads}

    prefixes = np.zeros((1, 0), dtype=np.int64)
    cum = np.zeros(1)
    hist = {i: (np.zeros((1, 0, d)), np.zeros((1, 0, d))) for i in heads}

    def step(states, t_pos, tok_emb):
        if K > 0:
            h = fuse(np.broadcast_to(trunk[t_pos], tok_emb.shape), tok_emb,
                     params["fuse.Wf"], params["fuse.Wg"])
        else:
            h = tok_emb + pos[t_pos]
        new_hist = {}
        for i in heads:
            h, kh, vh = decoder_layer_step(params, i, h, kv[i][0], kv[i][1],
                                           hist[i][0], hist[i][1])
            new_hist[i] = (kh, vh)
        return h, new_hist

    for t in range(T):
        live = prefixes.shape[0]
        if t == 0:
            tok = np.broadcast_to(params["bos"], (live, d))
        else:
            tok = params[f"emb.{t - 1}"][prefixes[:, -1]]
        h, new_hist = step(None, t, np.ascontiguousarray(tok))
        logp = log_softmax_rows(h @ params[f"head.{t}"])
        if valid_sids is not None:
            logp = np.where(prefix_mask(valid_sids, cfg.level_vocab_sizes, t,
                                        prefixes), logp, -np.inf)
        total = cum[:, None] + logp
        rows, toks, scores = select_topk(total, eff[t])
        if record is not None:
            flat = np.sort(total.ravel())[::-1]
            k = len(scores)
            gap = float(flat[k - 1] - flat[k]) if k < flat.size else math.inf
            record.append({"rows": rows, "tokens": toks, "scores": scores,
                           "cut_gap": gap})
        prefixes = np.concatenate([prefixes[rows], toks[:, None]], axis=1)
        cum = scores
        hist = {i: (kh[rows], vh[rows]) for i, (kh, vh) in new_hist.items()}

    results = [(tuple(int(v) for v in row), float(s)) for row, s in zip(prefixes, cum)]
    if value_rerank:
        results = _value_rerank(params, cfg, trunk, pos, kv, hist, heads, K,
                                prefixes, cum, representatives, results)
    return results


def _value_rerank(params, cfg, trunk, pos, kv, hist, heads, K, prefixes, cum,
                  representatives, results):
    """Extra step at position T ranking by E[bucket value] * exp(cum)
    (beam.py:258-288)."""
    T = cfg.n_levels
    live = prefixes.shape[0]
    if live == 0:
        return results
    tok = params[f"emb.{T - 1}"][prefixes[:, -1]]
    if K > 0:
        h = fuse(np.broadcast_to(trunk[T], tok.shape), tok, params["fuse.Wf"],
                 params["fuse.Wg"])
    else:
        h = tok + pos[T]
    for i in heads:
        h, _, _ = decoder_layer_step(params, i, h, kv[i][0], kv[i][1],
                                     hist[i][0], hist[i][1])
    probs = np.exp(log_softmax_rows(h @ params["head.value"]))
    reps = np.asarray(representatives, dtype=np.float64)
    nb = cfg.n_value_buckets
    if reps.size < nb:
        reps = np.concatenate([reps, np.full(nb - reps.size, reps[-1])])
    rank = (probs @ reps[:nb]) * np.exp(cum)
    order = np.lexsort((np.arange(live), -rank))
    return [(results[i][0], float(rank[i])) for i in order]


# ---------------------------------------------------------------------------
# teacher-forced scoring (decoder.py:162-219; verify.py:448-459)
# ---------------------------------------------------------------------------

def lazy_forward(params, cfg, x, tokens, trunk_depth=None, include_value_step=True):
    """Per-level head logits (and value logits) of one token sequence."""
    cfg = as_config(cfg)
    params = plain_params(params)
    K = cfg.trunk_depth if trunk_depth is None else trunk_depth
    T = cfg.n_levels
    if len(tokens) != T:
        raise ValueError(f"expected {T} tokens, got {len(tokens)}")
    n_pos = T + (1 if include_value_step else 0)
    pos = params["pos"][:n_pos]
    rows = [params["bos"]]
    for p in range(1, n_pos):
        tok = int(tokens[p - 1])
        if not 0 <= tok < cfg.level_vocab_sizes[p - 1]:
            raise ValueError(f"token {tok} out of range at level {p - 1}")
        rows.append(params[f"emb.{p - 1}"][tok])
    tok_in = np.stack(rows)
    if K == 0:
        fused = tok_in + pos
    else:
        trunk = run_layers_2d(params, pos, x, 0, K)
        fused = fuse(trunk, tok_in, params["fuse.Wf"], params["fuse.Wg"])
    states = run_layers_2d(params, fused, x, K, cfg.n_layers)
    head = [states[t] @ params[f"head.{t}"] for t in range(T)]
    value = states[T] @ params["head.value"] if include_value_step else None
    return head, value


def sequence_log_prob(head_logits, tokens):
    return float(sum(log_softmax_rows(head_logits[t][None, :])[0, int(tok)]
                     for t, tok in enumerate(tokens)))


def sequence_oracle(params, cfg, x, max_sequences=None):
    """Every token tuple ranked by teacher-forced log-probability."""
    cfg = as_config(cfg)
    out = []
    for toks in itertools.product(*[range(v) for v in cfg.level_vocab_sizes]):
        head, _ = lazy_forward(params, cfg, x, toks, include_value_step=False)
        out.append((toks, sequence_log_prob(head, toks)))
    out.sort(key=lambda r: (-r[1], r[0]))
    return out[:max_sequences] if max_sequences else out


# ---------------------------------------------------------------------------
# DBS width logic (schedule.py:33-70)
# ---------------------------------------------------------------------------

def round_half_up(x):
    return int(math.floor(x + 0.5))


def tabs_adjust(qps, q_threshold, slack, base_width, boost=0.6):
    if qps < q_threshold:
        return round_half_up(base_width * (1.0 + boost * slack))
    return base_width


def scale_widths(widths, base_width, active):
    f = active / base_width
    return tuple(max(1, round_half_up(w * f)) for w in widths)
