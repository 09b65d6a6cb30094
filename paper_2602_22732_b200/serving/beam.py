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

import numpy as np
import torch

from .. import _native as N
from ..decode import BeamDecoder, effective_widths, live_rows
from ..device import (DeviceContext, _stream_handle, device_weights, dims_of,
                      require_cuda)
from ..model.decoder import param_array
from ..quantizer.residual import SemanticId


def _context_rows(context):
    """Device fp32 (S, d) tensor for a DeviceContext / Tensor / ndarray,
    validated like beam.py:124-128."""
    if isinstance(context, DeviceContext):
        x = context.tensor
        if x.numel() == 0:
            raise ValueError("empty context")
        if not bool(torch.isfinite(x).all()):
            raise ValueError("context must be finite")
        return x if x.dim() == 2 else x.reshape(-1, x.shape[-1])
    data = getattr(context, "data", context)
    if isinstance(data, torch.Tensor):
        arr = data.detach()
        if arr.numel() == 0:
            raise ValueError("empty context")
        if not bool(torch.isfinite(arr).all()):
            raise ValueError("context must be finite")
        arr = arr.reshape(-1, arr.shape[-1]) if arr.dim() != 2 else arr
        return arr.to(device=require_cuda(), dtype=torch.float32).contiguous()
    arr = np.atleast_2d(np.asarray(data, dtype=np.float64))
    if arr.size == 0:
        raise ValueError("empty context")
    if not np.isfinite(arr).all():
        raise ValueError("context must be finite")
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(require_cuda())


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


def _to_sids(rows, vocab):
    return [(SemanticId(toks, vocab), score) for toks, score in rows]


def beam_search(model, context, schedule, shared_kv=True, precut=True, counter=None,
                value_rerank=False, buckets=None, trunk_depth=None, valid_sids=None):
    """Top sequences of one request, level by level (beam.py:112-143).

    Returns ``[(SemanticId, score)]`` sorted by descending cumulative
    log-probability, or by E[bucket value]*exp(score) with ``value_rerank``.
    ``valid_sids`` (extension) restricts expansion to
    prefixes of the given SIDs."""
    cfg = model.config
    x = _context_rows(context)
    widths = tuple(int(w) for w in schedule.widths)
    _check_schedule(cfg, widths)
    k_depth = _check_depth(cfg, trunk_depth)
    reps = None
    if value_rerank:
        if buckets is None:
            raise ValueError("value_rerank requires buckets")
        reps = getattr(buckets, "representatives", buckets)
    dec = BeamDecoder(model, [x.shape[0]], [widths], trunk_depth=k_depth,
                      value_rerank=value_rerank, representatives=reps,
                      valid_sids=valid_sids, device=x.device)
    dec.run(context=x)
    rows = dec.host_results()[0]
    record_counter(counter, cfg, widths, x.shape[0], shared_kv, value_rerank, k_depth)
    return _to_sids(rows, tuple(cfg.level_vocab_sizes))


def beam_search_batch(model, contexts=None, schedules=None, features=None, shared_kv=True,
                      precut=True, counter=None, value_rerank=False, buckets=None,
                      trunk_depth=None, valid_sids=None, path="auto"):
    """Batched ``beam_search``: one result list per request.

    ``path`` picks the decode kernels: "auto" (the fused per-request kernel
    when the working set fits on chip, else the layered batch path with
    tcgen05 3xFP16 GEMMs for d >= 64, else CUDA-core GEMMs), "fused",
    "tensor" (layered + tcgen05) or "layered" (layered + CUDA-core).

    ``contexts`` are projected X matrices, or ``features`` raw (S, F)
    feature matrices (the context projection then runs on the GPU, as the
    engine does, engine.py:104-105).  ``schedules`` is one BeamSchedule (or
    width tuple) for all requests or one per request (TABS widths)."""
    cfg = model.config
    dev = require_cuda()
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
    if contexts is not None:
        rows = [_context_rows(c) for c in contexts]
        lens = [r.shape[0] for r in rows]
        x = torch.cat(rows, 0) if B else None
        f = None
    else:
        arrs = [np.atleast_2d(np.asarray(getattr(a, "data", a), dtype=np.float64)) for a in features]
        for a in arrs:
            if a.size == 0:
                raise ValueError("empty context")
            if a.shape[-1] != cfg.feat_dim:
                raise ValueError(f"feature dim {a.shape[-1]} != expected {cfg.feat_dim}")
            if not np.isfinite(a).all():
                raise ValueError("context must be finite")
        lens = [a.shape[0] for a in arrs]
        f = torch.from_numpy(np.concatenate(arrs, 0).astype(np.float32)).to(dev) if B else None
        x = None
    if B == 0:
        return []
    reps = None
    if value_rerank:
        if buckets is None:
            raise ValueError("value_rerank requires buckets")
        reps = getattr(buckets, "representatives", buckets)
    dec = BeamDecoder(model, lens, per, trunk_depth=k_depth, value_rerank=value_rerank,
                      representatives=reps, valid_sids=valid_sids, device=dev, path=path)
    dec.run(features=f, context=x)
    out = dec.host_results()
    vocab = tuple(cfg.level_vocab_sizes)
    for b in range(B):
        record_counter(counter, cfg, per[b], lens[b], shared_kv, value_rerank, k_depth)
    return [_to_sids(r, vocab) for r in out]


def _select_gpu(beam_scores, logprobs, k):
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
    st = torch.from_numpy(s.astype(np.float32)).to(dev)
    lt = torch.from_numpy(np.ascontiguousarray(lp, dtype=np.float32)).to(dev)
    ob = torch.empty(kk, dtype=torch.int32, device=dev)
    ot = torch.empty(kk, dtype=torch.int32, device=dev)
    osc = torch.empty(kk, dtype=torch.float32, device=dev)
    oc = torch.empty(1, dtype=torch.int32, device=dev)
    ws = torch.empty(256, dtype=torch.uint8, device=dev)
    ptr = lambda t: C.c_void_p(t.data_ptr())
    N.check(N.lib.gr4ad_topk_precut(ptr(st), ptr(lt), 1, b, v, kk, ptr(ob), ptr(ot), ptr(osc),
                                    ptr(oc), ptr(ws), 256, _stream_handle(dev)))
    # scores are re-added in float64 on the host from the reference's inputs
    beams = ob.cpu().numpy().astype(np.int64)
    toks = ot.cpu().numpy().astype(np.int64)
    return beams, toks, s[beams] + lp[beams, toks]


def topk_precut(prev_beams, level_logprobs, k):
    """beam.py:50-60: top-k (beam_index, token, score) expansions, ordered
    by (-score, beam, token); the ranking runs on the GPU."""
    scores = np.asarray([s for _, s in prev_beams], dtype=np.float64)
    b, t, s = _select_gpu(scores, level_logprobs, k)
    return list(zip(b.tolist(), t.tolist(), s.tolist()))


def topk_global(beam_scores, level_logprobs, k):
    """beam.py:37-47: exhaustive selection (same result as pre-cut)."""
    return _select_gpu(beam_scores, level_logprobs, k)


def shared_encoder_kv(model, context, trunk_depth=None):
    """Per-request cross-attention K/V for the layers above the trunk
    (beam.py:98-109): {layer: (keys, values)} as float64 host arrays; the
    decode itself keeps them resident on the GPU."""
    cfg = model.config
    x = _context_rows(context)
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
