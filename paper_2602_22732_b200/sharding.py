"""User-sharded serving across the GPUs of one node.

Requests are independent: each GPU holds a full weight replica and decodes
its own users with no per-step exchange.  A request goes to rank
``shard_of(user_id, world)`` -- a stable FNV-1a hash, so a user's TTL-cache
entries (keyed by ``(user_id, index.version)``, engine.py:93) stay on one
GPU.  The only collectives move results and counters (NCCL over NVLink on
GPUs, gloo on CPU for tests):

* ``gather_decoded`` -- the decoder's device result tensors (int32 counts,
  int32 tokens [n, max_out, T], fp64 scores [n, max_out]) of every rank sent
  point-to-point to rank 0 (NCCL send / recv over NVLink): only rank 0
  receives, ~(4 T + 8) max_out bytes per request;
* ``gather_results`` -- the same for host result lists (the engine's);
* ``all_reduce_stats`` -- one all-reduce of a small int64 counter vector.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3


def shard_of(user_id, world_size):
    """Stable shard of a user id (FNV-1a 64 over its UTF-8 bytes)."""
    h = _FNV_OFFSET
    for byte in str(user_id).encode():
        h = ((h ^ byte) * _FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h % world_size


def partition(user_ids, world_size):
    """Indices of the requests each rank serves, order preserved."""
    parts = [[] for _ in range(world_size)]
    for i, uid in enumerate(user_ids):
        parts[shard_of(uid, world_size)].append(i)
    return parts


def pack_results(results, n_levels, max_out):
    """[(tokens, score)] lists -> (count int32 [n], tokens int32 [n, max_out, T],
    scores float64 [n, max_out])."""
    n = len(results)
    count = np.zeros(n, dtype=np.int32)
    toks = np.zeros((n, max_out, n_levels), dtype=np.int32)
    score = np.zeros((n, max_out), dtype=np.float64)
    for i, res in enumerate(results):
        count[i] = len(res)
        for j, (t, s) in enumerate(res):
            toks[i, j] = getattr(t, "tokens", t)
            score[i, j] = s
    return count, toks, score


def unpack_results(count, toks, score):
    return [[(tuple(int(v) for v in toks[i, j]), float(score[i, j]))
             for j in range(int(count[i]))] for i in range(len(count))]


def gather_results(local_results, n_levels, max_out, n_local_max, device=None, group=None):
    """Gather every rank's result lists to rank 0 (None elsewhere).

    Ranks pad to ``n_local_max`` requests so one fixed-size gather moves
    everything: ~(4*T + 8) * max_out bytes per request."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = device or torch.device("cpu")
    count, toks, score = pack_results(local_results, n_levels, max_out)
    n = len(local_results)
    pad = n_local_max - n
    if pad < 0:
        raise ValueError("n_local_max smaller than the local request count")
    meta = torch.tensor([n], dtype=torch.int64, device=device)
    tc = torch.from_numpy(np.pad(count, (0, pad))).to(device)
    tt = torch.from_numpy(np.pad(toks, ((0, pad), (0, 0), (0, 0)))).to(device)
    ts = torch.from_numpy(np.pad(score, ((0, pad), (0, 0)))).to(device)
    metas = [torch.empty_like(meta) for _ in range(world)]
    cs = [torch.empty_like(tc) for _ in range(world)]
    ks = [torch.empty_like(tt) for _ in range(world)]
    ss = [torch.empty_like(ts) for _ in range(world)]
    # all_gather works on every backend (NCCL has no gather-to-root for lists)
    dist.all_gather(metas, meta, group=group)
    dist.all_gather(cs, tc, group=group)
    dist.all_gather(ks, tt, group=group)
    dist.all_gather(ss, ts, group=group)
    if rank != 0:
        return None
    out = []
    for r in range(world):
        m = int(metas[r].item())
        out.append(unpack_results(cs[r].cpu().numpy()[:m], ks[r].cpu().numpy()[:m],
                                  ss[r].cpu().numpy()[:m]))
    return out


def gather_decoded(count, tokens, score, n_local, group=None):
    """Every rank's decode results to rank 0, point to point.

    ``count`` / ``tokens`` / ``score`` are one rank's result tensors in
    ``BeamDecoder`` layout (request-major: count [>= n], tokens [>= n *
    max_out * T], score [>= n * max_out]); ranks may hold different request
    counts and widths.  A 3-int all-gather exchanges the shapes, then each
    rank sends its first ``n_local`` requests to rank 0 (NCCL send/recv on
    the device tensors over NVLink; gloo on CPU tensors) -- nothing is
    broadcast.  Returns on rank 0 a list over ranks of (count [n], tokens
    [n, max_out * T], score [n, max_out]) tensors; None on the other ranks."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if dist.get_backend(group) != "nccl":  # gloo moves host tensors
        count, tokens, score = count.cpu(), tokens.cpu(), score.cpu()
    dev = count.device
    per_tok = tokens.numel() // max(count.numel(), 1)
    per_score = score.numel() // max(count.numel(), 1)
    meta = torch.tensor([n_local, per_tok, per_score], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    shapes = [tuple(int(x) for x in m.tolist()) for m in metas]
    mine = (count[:n_local].contiguous(),
            tokens[:n_local * per_tok].reshape(n_local, per_tok).contiguous(),
            score[:n_local * per_score].reshape(n_local, per_score).contiguous())
    if rank != 0:
        for t in mine:
            if t.numel():
                dist.send(t, dst=0, group=group)
        return None
    out = [mine]
    for r in range(1, world):
        n, pt, ps = shapes[r]
        bufs = (torch.empty(n, dtype=count.dtype, device=dev),
                torch.empty((n, pt), dtype=tokens.dtype, device=dev),
                torch.empty((n, ps), dtype=score.dtype, device=dev))
        for t in bufs:
            if t.numel():
                dist.recv(t, src=r, group=group)
        out.append(bufs)
    return out


def decoded_to_lists(count, tokens, score, n_levels):
    """(count, tokens, score) tensors of ``gather_decoded`` -> [(tokens tuple,
    score)] per request."""
    c = count.cpu().numpy()
    t = tokens.cpu().numpy()
    s = score.cpu().numpy()
    if t.ndim == 1:  # BeamDecoder's flat request-major buffers
        t = t[:t.size // max(len(c), 1) * len(c)].reshape(len(c), -1)
        s = s[:s.size // max(len(c), 1) * len(c)].reshape(len(c), -1)
    out = []
    for i in range(len(c)):
        ti = t[i].reshape(-1, n_levels)
        out.append([(tuple(int(v) for v in ti[j]), float(s[i, j])) for j in range(int(c[i]))])
    return out


STAT_KEYS = ("requests", "cache_hits", "model_invocations", "layer_calls", "results")


def all_reduce_stats(stats, device=None, group=None):
    """Sum a dict of integer counters over ranks (one small all-reduce)."""
    device = device or torch.device("cpu")
    v = torch.tensor([int(stats.get(k, 0)) for k in STAT_KEYS], dtype=torch.int64,
                     device=device)
    dist.all_reduce(v, group=group)
    return dict(zip(STAT_KEYS, (int(x) for x in v.cpu().tolist())))


def merge_in_order(user_ids, per_rank_results, world_size):
    """Reassemble rank-local result lists into the original request order."""
    parts = partition(user_ids, world_size)
    out = [None] * len(user_ids)
    for r, idxs in enumerate(parts):
        for k, i in enumerate(idxs):
            out[i] = per_rank_results[r][k]
    return out
