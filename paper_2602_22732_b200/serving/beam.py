"""Beam search over semantic-ID levels -- drop-in for
``adrec.serving.beam`` (pkg/src/adrec/serving/beam.py).

Same entry points, arguments, return values and ValueErrors; the arithmetic
runs in libgr4ad on the GPU (fp32, fp32 accumulation):

* ``beam_search``            -> beam.py:112-143 (one request)
* ``beam_search_batch``      -> the batched variant
* ``topk_precut`` / ``topk_global`` -> beam.py:37-60 (selection only)
* ``shared_encoder_kv``      -> beam.py:98-109

``shared_kv`` and ``precut`` are result-invariant in the reference
(verify.py:400-433); the GPU always shares the context KV across beams and
selects exactly, so they only change what ``counter`` records (closed forms
of layers.py:18-35 / beam.py:168-169, 238-239).  Tie order is the
reference's (-score, beam slot, token).
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np
import torch

from .. import _native as N
from ..decode import (BeamDecoder, PlanMismatch, decode_cached, decode_cached_many,
                      effective_widths, live_rows)
from ..device import (DeviceContext, _stream_handle, device_weights, dims_of, gated,
                      require_cuda)
from ..model.decoder import param_array


def _finite_rows(arr, d):
    """Validation of beam.py:124-128 plus the width check the reference gets
    from its matmul (a context must be the projected X, (S, d))."""
    if arr.size == 0 if isinstance(arr, np.ndarray) else arr.numel() == 0:
        raise ValueError("empty context")
    if arr.shape[-1] != d:
        raise ValueError(f"context has {arr.shape[-1]} columns, expected d={d} (the projected "
                         "X; raw features go through context_process or features=)")
    ok = np.isfinite(arr).all() if isinstance(arr, np.ndarray) else bool(torch.isfinite(arr).all())
    if not ok:
        raise ValueError("context must be finite")


def _context_input(context, d):
    """A validated (S, d) context: float32 host ndarray, or the fp32 CUDA
    tensor for a DeviceContext / CUDA Tensor (no host round trip)."""
    if isinstance(context, DeviceContext):
        x = context.tensor
        x = x if x.dim() == 2 else x.reshape(-1, x.shape[-1])
        _finite_rows(x, d)
        return x
    data = getattr(context, "data", context)
    if isinstance(data, torch.Tensor):
        arr = data.detach()
        arr = arr.reshape(-1, arr.shape[-1]) if arr.dim() != 2 else arr
        _finite_rows(arr, d)
        if arr.is_cuda:
            return arr.to(dtype=torch.float32).contiguous()
        data = arr.numpy()
    arr = np.atleast_2d(np.asarray(data, dtype=np.float64))
    if arr.ndim != 2:
        arr = arr.reshape(-1, arr.shape[-1])
    _finite_rows(arr, d)
    return np.ascontiguousarray(arr, dtype=np.float32)


def _context_rows(context, d=None):
    """Device fp32 (S, d) tensor of a context (shared_encoder_kv)."""
    x = _context_input(context, d if d is not None else np.shape(getattr(context, "data", context))[-1])
    return x if isinstance(x, torch.Tensor) else torch.from_numpy(x).to(require_cuda())


def _check_schedule(cfg, widths):
    if len(widths) != cfg.n_levels:
        raise ValueError(f"schedule has {len(widths)} widths for {cfg.n_levels} levels")


def _check_depth(cfg, trunk_depth):
    k = cfg.trunk_depth if trunk_depth is None else trunk_depth
    if not 0 <= k < cfg.n_layers:
        raise ValueError("trunk_depth must satisfy 0 <= K < n_layers")
    return k


def record_counter(counter, cfg, widths, s_ctx, shared_kv, value_rerank, k_depth):
    """Update a LayerCallCounter exactly as the reference's instrumented
    decode does (layers.py:79-80; beam.py:161, 168-169, 176-177, 238-239):
    T*K (n_pos*K with re-rank) trunk rows + (L-K) * slots_t per level."""
    if counter is None:
        return
    T, L, d = cfg.n_levels, cfg.n_layers, cfg.d
    eff = effective_widths(widths, cfg.level_vocab_sizes)
    live = live_rows(eff, cfg.level_vocab_sizes)
    n_pos = T + (1 if value_rerank else 0)
    if k_depth > 0:
        for _ in range(k_depth):
            counter.add_layer_calls(n_pos)
    heads = L - k_depth
    if shared_kv:
        counter.add_kv_build(1, heads * 2 * s_ctx * d)
    for t in range(T):
        slots = max(eff[t], live[t])
        if not shared_kv:
            counter.add_kv_build(slots, heads * 2 * slots * s_ctx * d)
        for _ in range(heads):
            counter.add_layer_calls(slots)
    if value_rerank:
        if not shared_kv:
            counter.add_kv_build(live[T], heads * 2 * live[T] * s_ctx * d)
        for _ in range(heads):
            counter.add_layer_calls(live[T])


def _valid_key(valid_sids):
    """Content digest of a valid-SID set (part of the pooled decoder's key:
    the decoder holds the set's device prefix tables)."""
    if valid_sids is None:
        return None
    hit = _VKEYS.get(id(valid_sids))
    if hit is not None and hit[0] is valid_sids:
        return hit[1]
    toks = np.asarray([tuple(getattr(v, "tokens", v)) for v in valid_sids], dtype=np.int64)
    key = (toks.shape, hashlib.sha1(toks.tobytes()).hexdigest())
    if isinstance(valid_sids, tuple):  # immutable (the engine reuses one per index version)
        if len(_VKEYS) >= 4:
            _VKEYS.clear()
        _VKEYS[id(valid_sids)] = (valid_sids, key)
    return key


_VKEYS = {}  # id(valid-SID tuple) -> (the tuple, its digest)


def _split_input(inp, lens, lo, hi):
    """Requests [lo, hi) of a batch input: per-request blocks, or
    concatenated context rows (numpy / CUDA tensor)."""
    if isinstance(inp, list):
        return inp[lo:hi]
    r0 = int(sum(lens[:lo]))
    r1 = r0 + int(sum(lens[lo:hi]))
    return inp[r0:r1]


def _decode(model, lens, per, k_depth, value_rerank, reps, valid_sids, path, inp, kind,
            items=None, cap=None, parts=1, lazy=False, graphs=True):
    """Pooled decode with the automatic fp16-range fallback: with
    path="auto", a batch whose weights or context K/V leave the fp16 split
    range of the tensor-core paths is decoded again on the fp32 CUDA-core
    path (another GPU path -- there is no CPU fallback).  ``parts`` > 1
    decodes the batch as that many consecutive request groups pipelined on
    one stream (decode_cached_many: one group's host staging / result
    building overlaps another's decode); the kernels are per row and per
    request, so every request decodes exactly as in one batch."""
    dev = inp.device if isinstance(inp, torch.Tensor) else require_cuda()
    if isinstance(inp, list) and len({a.shape[1] for a in inp}) != 1:
        raise ValueError("feature blocks must share one width")
    reps_key = None if reps is None else tuple(np.asarray(reps, dtype=np.float64).ravel().tolist())
    vkey = _valid_key(valid_sids)
    B = len(lens)
    parts = max(1, min(int(parts), B))
    cuts = [round(k * B / parts) for k in range(parts + 1)]

    def job(p, lo, hi, use_cap):
        ln, pw = list(lens[lo:hi]), list(per[lo:hi])
        part_in = _split_input(inp, lens, lo, hi)
        if use_cap:
            cp = list(cap[lo:hi])
            key = (id(model.params), model.config, str(dev), kind, tuple(ln), "cap", tuple(cp),
                   k_depth, bool(value_rerank), reps_key, vkey, p)
            factory = lambda: BeamDecoder(model, ln, cp, trunk_depth=k_depth,
                                          value_rerank=value_rerank, representatives=reps,
                                          valid_sids=valid_sids, device=dev, path=p)
            return (key, factory, part_in, kind, items, pw)
        key = (id(model.params), model.config, str(dev), kind, tuple(ln), tuple(pw), k_depth,
               bool(value_rerank), reps_key, vkey, p)
        factory = lambda: BeamDecoder(model, ln, pw, trunk_depth=k_depth,
                                      value_rerank=value_rerank, representatives=reps,
                                      valid_sids=valid_sids, device=dev, path=p)
        return (key, factory, part_in, kind, items, None)

    def attempt(p):
        for use_cap in ((True, False) if cap is not None else (False,)):
            jobs = [job(p, cuts[k], cuts[k + 1], use_cap) for k in range(parts)]
            try:
                if parts == 1:
                    key, factory, part_in, _, _, w = jobs[0]
                    return decode_cached(key, factory, model, part_in, kind, items, widths=w,
                                         lazy=lazy, graphs=graphs)
                outs = decode_cached_many(jobs, model, lazy, graphs)
            except PlanMismatch:
                continue  # a width plan beyond the capacity decoder: exact plans
            res = [r for o in outs for r in o[0]]
            idx = None
            if all(o[1] is not None for o in outs):
                w = max(o[1].shape[1] for o in outs)
                idx = np.concatenate([np.pad(o[1], ((0, 0), (0, w - o[1].shape[1])),
                                             constant_values=-1) for o in outs], 0)
            return res, idx
        raise AssertionError("unreachable")

    try:
        return attempt(path)
    except N.RangeError:
        if path != "auto":
            raise
        return attempt("layered")


def beam_search(model, context, schedule, shared_kv=True, precut=True, counter=None,
                value_rerank=False, buckets=None, trunk_depth=None, valid_sids=None):
    """Top sequences of one request, level by level (beam.py:112-143).

    Returns ``[(SemanticId, score)]`` sorted by descending cumulative
    log-probability, or by E[bucket value]*exp(score) with ``value_rerank``.
    ``valid_sids`` (extension) restricts expansion to
    prefixes of the given SIDs."""
    cfg = model.config
    x = _context_input(context, cfg.d)
    widths = tuple(int(w) for w in schedule.widths)
    _check_schedule(cfg, widths)
    k_depth = _check_depth(cfg, trunk_depth)
    reps = None
    if value_rerank:
        if buckets is None:
            raise ValueError("value_rerank requires buckets")
        reps = getattr(buckets, "representatives", buckets)
    out = _decode(model, [x.shape[0]], [widths], k_depth, value_rerank, reps, valid_sids, "auto",
                  x, "context")[0][0]
    record_counter(counter, cfg, widths, x.shape[0], shared_kv, value_rerank, k_depth)
    return out


def beam_search_batch(model, contexts=None, schedules=None, features=None, shared_kv=True,
                      precut=True, counter=None, value_rerank=False, buckets=None,
                      trunk_depth=None, valid_sids=None, path="auto", _items=None,
                      _capacity=None, pipeline="auto", _lazy=False, _graphs=True):
    """Batched ``beam_search``: one result list per request.

    ``path`` picks the decode kernels: "auto" (the fused per-request kernel
    when the working set fits on chip, else the layered batch path with
    tcgen05 3xFP16 GEMMs for d >= 64, else CUDA-core GEMMs; a batch that
    leaves the fp16 split range is re-decoded on the CUDA-core path),
    "fused", "tensor" (layered + tcgen05) or "layered" (layered + CUDA-core).

    ``contexts`` are projected X matrices, or ``features`` raw (S, F)
    feature matrices (the context projection then runs on the GPU, as the
    engine does, engine.py:104-105).  ``schedules`` is one BeamSchedule (or
    width tuple) for all requests or one per request (TABS widths).

    Repeated calls with the same batch shape reuse one pooled decoder and
    replay its CUDA graph (``decode.POOL``): inputs go host -> pinned ->
    device, results come back as one async copy, and the SemanticIds are
    built in bulk.  ``pipeline``: request groups decoded back to back on
    one stream so host work overlaps device work ("auto": two groups from
    96 requests on; an int: that many) -- results are identical either way."""
    cfg = model.config
    if (contexts is None) == (features is None):
        raise ValueError("pass exactly one of contexts / features")
    items = contexts if contexts is not None else features
    B = len(items)
    if isinstance(schedules, (list, tuple)) and schedules and not isinstance(
            schedules[0], (int, np.integer)):
        per = [tuple(int(w) for w in getattr(s, "widths", s)) for s in schedules]
    else:
        one = tuple(int(w) for w in getattr(schedules, "widths", schedules))
        per = [one] * B
    if len(per) != B:
        raise ValueError("one schedule per request required")
    for w in per:
        _check_schedule(cfg, w)
    k_depth = _check_depth(cfg, trunk_depth)
    if B == 0:
        return []
    if contexts is not None:
        rows = [_context_input(c, cfg.d) for c in contexts]
        lens = [r.shape[0] for r in rows]
        if all(isinstance(r, np.ndarray) for r in rows):
            inp = np.concatenate(rows, 0)
        else:
            dev = next(r.device for r in rows if isinstance(r, torch.Tensor))
            inp = torch.cat([r if isinstance(r, torch.Tensor) else torch.from_numpy(r).to(dev)
                             for r in rows], 0)
        kind = "context"
    else:
        arrs = [np.atleast_2d(np.asarray(getattr(a, "data", a))) for a in features]
        for a in arrs:
            if a.size == 0:
                raise ValueError("empty context")
            if a.shape[-1] != cfg.feat_dim:
                raise ValueError(f"feature dim {a.shape[-1]} != expected {cfg.feat_dim}")
        # finiteness: checked once, on the staged fp32 copy (decode._decode_on
        # raises the reference's ValueError for a non-finite input)
        lens = [a.shape[0] for a in arrs]
        inp = arrs  # concatenated + cast into the decoder's pinned staging buffer
        kind = "features"
    reps = None
    if value_rerank:
        if buckets is None:
            raise ValueError("value_rerank requires buckets")
        reps = getattr(buckets, "representatives", buckets)
    cap = None
    if _capacity is not None:  # engine: widths bounded by this schedule (TABS maximum)
        c = tuple(int(w) for w in getattr(_capacity, "widths", _capacity))
        if len(c) == cfg.n_levels and all(all(a <= b for a, b in zip(w, c)) for w in per):
            cap = [c] * B
    parts = (2 if B >= 96 else 1) if pipeline == "auto" else int(pipeline)
    out, item_idx = _decode(model, lens, per, k_depth, value_rerank, reps, valid_sids, path,
                            inp, kind, _items, cap, parts, _lazy, _graphs)
    if counter is not None:
        for b in range(B):
            record_counter(counter, cfg, per[b], lens[b], shared_kv, value_rerank, k_depth)
    return (out, item_idx) if _items is not None else out


@gated
def _select_gpu(beam_scores, logprobs, k):
    """Exact float64 selection on the GPU (gr4ad_topk_precut_f64): the
    candidate scores are the reference's own double sums, ranked with no
    rounding, so the order is the reference's bit for bit."""
    dev = require_cuda()
    s = np.asarray(beam_scores, dtype=np.float64).ravel()
    lp = np.atleast_2d(np.asarray(logprobs, dtype=np.float64))
    b, v = lp.shape
    if s.size != b:
        raise ValueError("one score per beam required")
    k = int(k)
    if k < 1 or b * v == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
    kk = min(k, b * v)
    st = torch.from_numpy(s).to(dev)
    lt = torch.from_numpy(np.ascontiguousarray(lp)).to(dev)
    ob = torch.empty(kk, dtype=torch.int32, device=dev)
    ot = torch.empty(kk, dtype=torch.int32, device=dev)
    osc = torch.empty(kk, dtype=torch.float64, device=dev)
    oc = torch.empty(1, dtype=torch.int32, device=dev)
    ptr = lambda t: C.c_void_p(t.data_ptr())
    N.check(N.lib.gr4ad_topk_precut_f64(ptr(st), ptr(lt), 1, b, v, kk, ptr(ob), ptr(ot),
                                        ptr(osc), ptr(oc), _stream_handle(dev)))
    return (ob.cpu().numpy().astype(np.int64), ot.cpu().numpy().astype(np.int64),
            osc.cpu().numpy())


def topk_precut(prev_beams, level_logprobs, k):
    """beam.py:50-60: top-k (beam_index, token, score) expansions, ordered
    by (-score, beam, token); the ranking runs on the GPU."""
    scores = np.asarray([s for _, s in prev_beams], dtype=np.float64)
    b, t, s = _select_gpu(scores, level_logprobs, k)
    return list(zip(b.tolist(), t.tolist(), s.tolist()))


def topk_global(beam_scores, level_logprobs, k):
    """beam.py:37-47: exhaustive selection (same result as pre-cut)."""
    return _select_gpu(beam_scores, level_logprobs, k)


@gated
def shared_encoder_kv(model, context, trunk_depth=None):
    """Per-request cross-attention K/V for the layers above the trunk
    (beam.py:98-109): {layer: (keys, values)} as float64 host arrays; the
    decode itself keeps them resident on the GPU."""
    cfg = model.config
    x = _context_rows(context, cfg.d)
    k = cfg.trunk_depth if trunk_depth is None else trunk_depth
    L, d = cfg.n_layers, cfg.d
    if k >= L:
        return {}
    dw = device_weights(model, x.device)
    kv = torch.empty((x.shape[0], 2 * (L - k) * d), dtype=torch.float32, device=x.device)
    N.check(N.lib.gr4ad_encoder_kv(C.byref(dims_of(cfg)), C.byref(dw.struct),
                                   C.c_void_p(x.data_ptr()), x.shape[0], k, L,
                                   C.c_void_p(kv.data_ptr()), _stream_handle(x.device)))
    host = kv.double().cpu().numpy()
    return {i: (host[:, 2 * (i - k) * d:(2 * (i - k) + 1) * d],
                host[:, (2 * (i - k) + 1) * d:(2 * (i - k) + 2) * d]) for i in range(k, L)}
