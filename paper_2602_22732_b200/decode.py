"""Batched LazyAR beam decode on one GPU (the engine under ``beam_search``).

A :class:`BeamDecoder` owns one batch shape -- request count, context
lengths and per-request width schedules (DBS widths may differ per
request) -- and the device buffers for it: the workspace sized by
``gr4ad_workspace_bytes`` and the result arrays.  ``run`` issues the whole
decode (encoder K/V, trunk, T level steps, top-k + in-place compaction,
optional value re-rank) on the current stream with no host round-trip, so
it can be captured once into a CUDA graph and replayed per batch.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import time
from collections import OrderedDict
from collections.abc import Sequence
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _hostmarshal
from . import _native as N
from .device import (CAPTURE_GATE, _stream_handle, device_weights, dims_of, gated,
                     require_cuda)
from .quantizer.residual import sid_type


def effective_widths(widths, vocab_sizes):
    """Width clamp to the reachable prefix count (beam.py:134-139)."""
    eff, reach = [], 1
    for w, v in zip(widths, vocab_sizes):
        reach = min(reach * v, 1 << 40)
        eff.append(min(int(w), reach))
    return eff


def live_rows(eff, vocab_sizes):
    """Rows entering each level (and surviving the last), no masking."""
    live = [1]
    for e, v in zip(eff, vocab_sizes):
        live.append(min(e, live[-1] * v))
    return live


def prefix_keys(valid_sids, vocab_sizes):
    """Per level t: sorted unique mixed-radix keys of valid (t+1)-prefixes."""
    T = len(vocab_sizes)
    keys = [set() for _ in range(T)]
    for sid in valid_sids:
        toks = getattr(sid, "tokens", sid)
        k = 0
        for t in range(T):
            k = k * int(vocab_sizes[t]) + int(toks[t])
            keys[t].add(k)
    return [np.array(sorted(s), dtype=np.int64) for s in keys]


class BeamDecoder:
    # "tensor_ctx": the tcgen05 path attending against the projected context X
    # even when features are given (no latent absorption; A/B and parity aid)
    PATHS = {"auto": 0, "layered": 1, "fused": 2, "tensor": 3, "fused_simt": 4, "tensor_ctx": 5}

    @gated
    def __init__(self, model, ctx_lens, widths, trunk_depth=None, value_rerank=False,
                 representatives=None, valid_sids=None, device=None, path="auto"):
        self.device = require_cuda(device)
        cfg = model.config
        self.cfg = cfg
        self.T = cfg.n_levels
        self.weights = device_weights(model, self.device)
        self.dims = dims_of(cfg)
        B = len(ctx_lens)
        self.n_requests = B
        self.ctx_lens = [int(s) for s in ctx_lens]
        w = np.asarray(widths, dtype=np.int32).reshape(B, self.T)
        self.widths = w
        self._ctx = (C.c_int * max(B, 1))(*self.ctx_lens)
        self._w = (C.c_int * max(B * self.T, 1))(*w.ravel().tolist())
        bt = N.Batch()
        bt.n_requests = B
        bt.ctx_len = self._ctx
        bt.widths = self._w
        bt.trunk_depth = -1 if trunk_depth is None else int(trunk_depth)
        bt.value_rerank = 1 if value_rerank else 0
        self._keep = []
        if value_rerank:
            if representatives is None:
                raise ValueError("value_rerank requires buckets (representatives)")
            reps = np.asarray(representatives, dtype=np.float64).ravel()
            nb = cfg.n_value_buckets
            if reps.size < nb:  # beam.py:281-284
                reps = np.concatenate([reps, np.full(nb - reps.size, reps[-1])])
            rt = torch.from_numpy(reps[:nb].astype(np.float32)).to(self.device)
            self._keep.append(rt)
            bt.value_reps = C.c_void_p(rt.data_ptr())
        self._vcount = (C.c_int * N.MAX_LEVELS)()
        if valid_sids is not None:
            for t, keys in enumerate(prefix_keys(valid_sids, cfg.level_vocab_sizes)):
                kt = torch.from_numpy(keys if keys.size else np.zeros(1, np.int64)).to(self.device)
                self._keep.append(kt)
                bt.valid_prefix[t] = C.c_void_p(kt.data_ptr())
                self._vcount[t] = int(keys.size)
        bt.valid_prefix_count = self._vcount
        bt.decode_path = self.PATHS[path]
        self.batch = bt
        self._bind_derived()
        nbytes, max_out = C.c_size_t(), C.c_int()
        N.check(N.lib.gr4ad_workspace_bytes(C.byref(self.dims), C.byref(bt), C.byref(nbytes),
                                            C.byref(max_out)))
        self.workspace_bytes = nbytes.value
        self.max_out = max(max_out.value, 1)
        self.workspace = torch.empty(max(self.workspace_bytes, 256), dtype=torch.uint8,
                                     device=self.device)
        self.count = torch.zeros(max(B, 1), dtype=torch.int32, device=self.device)
        self.tokens = torch.zeros(max(B, 1) * self.max_out * self.T, dtype=torch.int32,
                                  device=self.device)
        self.score = torch.zeros(max(B, 1) * self.max_out, dtype=torch.float64,
                                 device=self.device)
        res = N.Results()
        res.max_out = self.max_out
        res.count = C.c_void_p(self.count.data_ptr())
        res.tokens = C.c_void_p(self.tokens.data_ptr())
        res.score = C.c_void_p(self.score.data_ptr())
        self.results_struct = res
        N.check(N.lib.gr4ad_prepare(C.byref(self.dims), C.byref(bt),
                                    C.c_void_p(self.workspace.data_ptr()),
                                    self.workspace_bytes, _stream_handle(self.device)))
        off = C.c_size_t()
        N.check(N.lib.gr4ad_range_flag_offset(C.byref(self.dims), C.byref(bt), C.byref(off)))
        self._flag = self.workspace[off.value:off.value + 4].view(torch.int32)
        self.graph = None
        self._graph_inputs = None
        self.host_graph = None
        self._host_out = None
        self._fetched = None
        self.in_buf = None
        self._in_host = None
        self.uses = 0
        self._graphs = OrderedDict()  # width plan -> parked CUDA graph (set_widths)
        self._plan_uses = {}
        self.item_idx = None
        self._resolved = False
        self.last_item_idx = None

    def _bind_derived(self):
        """Point the batch at the snapshot's derived weight copies (factored
        / absorbed products, fuse tables, K-major fp16 splits, mma fragments):
        one buffer per (snapshot, plan layout) held by the DeviceWeights and
        built on first use, so decoders of any batch shape share it and a new
        shape costs no weight preparation (gr4ad_derived_layout)."""
        bt = self.batch
        bt.derived = None
        bt.derived_bytes = 0
        nb, sig = C.c_size_t(), C.c_ulonglong()
        N.check(N.lib.gr4ad_derived_layout(C.byref(self.dims), C.byref(bt), C.byref(nb),
                                           C.byref(sig)))

        def prepare(buf):
            bt.derived = C.c_void_p(buf.data_ptr())
            bt.derived_bytes = nb.value
            bt.weights_prepared = 0
            N.check(N.lib.gr4ad_prepare_weights(C.byref(self.dims), C.byref(self.weights.struct),
                                                C.byref(bt), None, 0,
                                                _stream_handle(self.device)))

        buf = self.weights.derived_buffer(sig.value, nb.value, prepare)
        self._derived = buf
        bt.derived = C.c_void_p(buf.data_ptr())
        bt.derived_bytes = nb.value
        bt.weights_prepared = 1

    def rebind(self, model):
        """Decode with another snapshot of the same config (hot swap).  The
        plan and workspace stay; a captured graph is dropped because it
        holds the previous snapshot's weight pointers."""
        if model.config != self.cfg:
            raise ValueError("rebind needs a snapshot with the same DecoderConfig")
        self.weights = device_weights(model, self.device)
        self._bind_derived()
        # every captured graph holds the previous snapshot's weight pointers
        self.graph = None
        self._graph_inputs = None
        self.host_graph = None
        self._host_in = self._dev_in = self.host_out = None
        self._graphs.clear()
        self._plan_uses.clear()

    def set_widths(self, widths):
        """Re-plan for new per-request width schedules (same request count and
        context lengths) inside this decoder's workspace and result buffers.

        TABS widths follow the load (schedule.py:54-70), so a serving batch
        shape recurs with many width plans; a re-plan is a host plan plus
        one table upload (gr4ad_prepare), not a new decoder (workspace,
        derived-weight binding, graph).  Captured graphs are parked per plan
        (up to 8): returning to a plan re-uploads its tables and replays its
        graph.  Returns False, changing nothing, when the plan does not fit
        the buffers (the caller then needs a decoder of its own)."""
        w = np.asarray(widths, dtype=np.int32).reshape(self.n_requests, self.T)
        if np.array_equal(w, self.widths):
            return True
        bt = self.batch
        cw = (C.c_int * max(w.size, 1))(*w.ravel().tolist())
        old = bt.widths
        bt.widths = cw
        nbytes, max_out = C.c_size_t(), C.c_int()
        N.check(N.lib.gr4ad_workspace_bytes(C.byref(self.dims), C.byref(bt), C.byref(nbytes),
                                            C.byref(max_out)))
        if nbytes.value > self.workspace.numel() or max_out.value > self.max_out:
            bt.widths = old
            return False
        okey = self.widths.tobytes()
        if self.graph is not None:
            self._graphs[okey] = self.graph
            self._graphs.move_to_end(okey)
            while len(self._graphs) > 8:
                self._graphs.popitem(last=False)
        if len(self._plan_uses) > 1024:
            self._plan_uses.clear()
        self._plan_uses[okey] = self.uses
        self._w = cw
        self.widths = w
        self.workspace_bytes = nbytes.value
        self.host_graph = None  # captured on the previous plan
        self._bind_derived()
        N.check(N.lib.gr4ad_prepare(C.byref(self.dims), C.byref(bt),
                                    C.c_void_p(self.workspace.data_ptr()),
                                    self.workspace.numel(), _stream_handle(self.device)))
        off = C.c_size_t()
        N.check(N.lib.gr4ad_range_flag_offset(C.byref(self.dims), C.byref(bt), C.byref(off)))
        self._flag = self.workspace[off.value:off.value + 4].view(torch.int32)
        nkey = w.tobytes()
        STATS["replans"] += 1
        self.graph = self._graphs.pop(nkey, None)
        self.uses = self._plan_uses.get(nkey, 0)
        return True

    # -- launch ----------------------------------------------------------
    def run(self, features=None, context=None):
        """features: (sum S, feat_dim) fp32 CUDA tensor, or context: (sum S, d)."""
        f = C.c_void_p(features.data_ptr()) if features is not None else None
        x = C.c_void_p(context.data_ptr()) if context is not None else None
        N.check(N.lib.gr4ad_beam_search_run(
            C.byref(self.dims), C.byref(self.weights.struct), C.byref(self.batch), f, x,
            C.byref(self.results_struct), C.c_void_p(self.workspace.data_ptr()),
            self.workspace.numel(), _stream_handle(self.device)))

    def capture(self, features=None, context=None, warmup=1):
        """Capture ``run`` on static input tensors into a CUDA graph."""
        for _ in range(warmup):
            self.run(features, context)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(features, context)
        self.graph = g
        self._graph_inputs = (features, context)
        return g

    def replay(self):
        self.graph.replay()

    def capture_host(self, host_features, warmup=1):
        """Capture one CUDA graph from pinned host features to pinned host
        results: the features' H2D copy, the decode, and the D2H copies of
        count / tokens / score (``self.host_out``).  ``replay_host`` then
        serves a batch with a single launch on the current stream."""
        if not host_features.is_pinned():
            raise ValueError("capture_host needs pinned host features")
        self._host_in = host_features
        self._dev_in = torch.empty(host_features.shape, dtype=torch.float32, device=self.device)
        self.host_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory()
                         for t in (self.count, self.tokens, self.score)]

        def body():
            self._dev_in.copy_(self._host_in, non_blocking=True)
            self.run(features=self._dev_in)
            for h, t in zip(self.host_out, (self.count, self.tokens, self.score)):
                h.copy_(t, non_blocking=True)

        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                body()
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            body()
        self.host_graph = g
        return g

    def replay_host(self):
        if self.host_graph is None:
            raise RuntimeError("no host graph: capture_host() again (rebind drops it)")
        self.host_graph.replay()

    # -- results -----------------------------------------------------------
    def check_range(self):
        """Raise if the last decode's fp16 operand splits left their range
        (tensor-core paths only; gr4ad_range_status)."""
        N.check(N.lib.gr4ad_range_status(C.byref(self.dims), C.byref(self.batch),
                                         C.c_void_p(self.workspace.data_ptr()),
                                         _stream_handle(self.device)))

    def resolve_items(self, keys, ids, n_keys):
        """On-device SID -> item slot for every result of the last decode
        (gr4ad_resolve_items; -1 = SID not in the index).  ``keys`` / ``ids``:
        device int64 sorted SID keys and int32 item slots.  Fetched with the
        results into ``last_item_idx``."""
        if self.item_idx is None:
            self.item_idx = torch.empty(max(self.n_requests, 1) * self.max_out,
                                        dtype=torch.int32, device=self.device)
        N.check(N.lib.gr4ad_resolve_items(
            C.c_void_p(keys.data_ptr()), C.c_void_p(ids.data_ptr()), int(n_keys),
            C.byref(self.dims), C.byref(self.results_struct), self.n_requests,
            C.c_void_p(self.item_idx.data_ptr()), _stream_handle(self.device)))
        self._resolved = True

    def fetch_async(self):
        """Start the D2H copies of this decode's results and fp16 range flag
        (and resolved item slots) into pinned buffers on the current stream;
        :meth:`results` reads them after the event."""
        srcs = [self.count, self.tokens, self.score, self._flag]
        if self._resolved:
            srcs.append(self.item_idx)
        if self._host_out is None or len(self._host_out) != len(srcs):
            self._host_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in srcs]
        for h, t in zip(self._host_out, srcs):
            h.copy_(t, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._fetched = ev
        return ev

    def results(self, lazy=False):
        """[(SemanticId, score)] lists per request from the fetched buffers
        (one vectorised range check, C-level construction, no per-token
        Python validation).  ``lazy``: per request a :class:`SidList` over a
        copy of the arrays, built into objects only when read."""
        if self._fetched is None:
            self.fetch_async()
        self._fetched.synchronize()
        self._fetched = None
        host = [t.numpy() for t in self._host_out]
        count, toks, score, flag = host[:4]
        self.last_item_idx = (host[4].reshape(-1, self.max_out)[: self.n_requests]
                              if self._resolved else None)
        self._resolved = False
        if int(flag[0]):
            raise N.RangeError(
                "libgr4ad: fp16 split range exceeded: an operand exceeded the fp16 split range "
                "(|weight| < 32, |context X| < 256): decode with the CUDA-core path "
                "(path='layered')")
        if lazy:
            return lazy_results(count[: self.n_requests], toks, score, self.max_out, self.T,
                                self.cfg.level_vocab_sizes)
        return materialize(count[: self.n_requests], toks, score, self.max_out, self.T,
                           self.cfg.level_vocab_sizes)

    def host_results(self, sids=False):
        """Blocking fetch of the last decode's results: per request a list
        of (token tuple | SemanticId, score)."""
        self.fetch_async()
        return self.results() if sids else [
            [(tuple(s), v) for s, v in req] for req in self.results()]


class SidList(Sequence):
    """One request's [(SemanticId, score)] list, built on first read from
    its (n, T) token rows and (n,) scores (materialize), then kept: a
    serving engine that only returns items never pays for the objects.
    Compares, iterates, indexes and prints as the list; ``scores`` is the
    float64 array."""

    __slots__ = ("_toks", "scores", "_vocab", "_list")

    def __init__(self, toks, scores, vocab):
        self._toks = toks
        self.scores = scores
        self._vocab = vocab
        self._list = None

    def _get(self):
        if self._list is None:
            n, T = self._toks.shape
            self._list = materialize(np.array([n], np.int32), self._toks.ravel(), self.scores,
                                     n, T, self._vocab)[0]
        return self._list

    def __len__(self):
        return len(self.scores)

    def __getitem__(self, i):
        return self._get()[i]

    def __iter__(self):
        return iter(self._get())

    def __eq__(self, other):
        if isinstance(other, SidList):
            other = other._get()
        return self._get() == other if isinstance(other, list) else NotImplemented

    __hash__ = None

    def __repr__(self):
        return repr(self._get())

    def __reduce__(self):
        return (list, (self._get(),))


def lazy_results(count, toks, score, max_out, T, vocab):
    """Per-request :class:`SidList` over copies of the result arrays (the
    decoder's pinned buffers are reused by its next decode); the token
    range check runs here, once for the batch, as materialize's does."""
    vocab = tuple(int(v) for v in vocab)
    B = len(count)
    tk = np.array(toks[: B * max_out * T], dtype=np.int32).reshape(B, max_out, T)
    sc = np.array(score[: B * max_out], dtype=np.float64).reshape(B, max_out)
    cnt = np.asarray(count, dtype=np.int64)
    live = np.arange(max_out)[None, :] < cnt[:, None]
    for t, v in enumerate(vocab):
        col = tk[:, :, t]
        bad = live & ((col < 0) | (col >= v))
        if bad.any():
            tok = int(col[bad][0])
            raise ValueError(f"token {tok} out of range [0, {v}) at level {t}")
    return [SidList(tk[b, : cnt[b]], sc[b, : cnt[b]], vocab) for b in range(B)]


def materialize(count, toks, score, max_out, T, vocab):
    """Per-request [(SemanticId, float)] from host result arrays (count (B,)
    int32, tokens (B*max_out*T,) int32, score (B*max_out,) float64); entries
    past count[b] are ignored.  Built by the native marshaller
    (csrc/hostmarshal.c): one range check over the live tokens (the same
    ValueError SemanticId raises), token ints from a prebuilt table,
    SemanticId tuples allocated directly, cyclic GC paused."""
    vocab = tuple(int(v) for v in vocab)
    return _hostmarshal.build(np.ascontiguousarray(count, dtype=np.int32),
                              np.ascontiguousarray(toks, dtype=np.int32),
                              np.ascontiguousarray(score, dtype=np.float64),
                              int(max_out), int(T), vocab, sid_type(vocab))


# host-side accounting of the pooled decode path (serving_bench reports it):
# seconds per phase and event counts; plain adds under the GIL
STATS = {"stage_s": 0.0, "launch_s": 0.0, "wait_s": 0.0, "marshal_s": 0.0, "calls": 0,
         "builds": 0, "evictions": 0, "replans": 0, "captures": 0}


def reset_stats():
    for k in STATS:
        STATS[k] = 0 if isinstance(STATS[k], int) else 0.0


class DecoderPool:
    """Idle BeamDecoders (workspace, plan, derived weight copies and a CUDA
    graph each) kept per batch shape, so repeated drop-in calls --
    ``beam_search_batch``, ``ServingEngine.serve_batch`` -- replay one graph
    instead of re-planning, re-allocating and re-splitting the weights.  A
    decoder is exclusively checked out while a call uses it (concurrent
    callers of the same shape get separate decoders); LRU-bounded by total
    workspace bytes."""

    def __init__(self, max_bytes=None, max_decoders=64):
        self._lock = threading.Lock()
        self._idle = OrderedDict()
        self._max_bytes = max_bytes  # None: 40 % of the device's memory
        self.max_decoders = max_decoders

    @property
    def max_bytes(self):
        if self._max_bytes is None:
            try:
                total = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
            except Exception:  # no device (host-only use): assume a 120 GiB part
                total = 120 << 30
            self._max_bytes = int(0.4 * total)
        return self._max_bytes

    @max_bytes.setter
    def max_bytes(self, v):
        self._max_bytes = v

    def acquire(self, key, factory):
        with self._lock:
            lst = self._idle.get(key)
            if lst:
                dec = lst.pop()
                if not lst:
                    del self._idle[key]
                return dec
        STATS["builds"] += 1
        return factory()

    def release(self, key, dec):
        with self._lock:
            self._idle.setdefault(key, []).append(dec)
            self._idle.move_to_end(key)
            while True:
                n = sum(len(v) for v in self._idle.values())
                nbytes = sum(d.workspace_bytes for v in self._idle.values() for d in v)
                if n <= self.max_decoders and nbytes <= self.max_bytes:
                    break
                k0 = next(iter(self._idle))
                STATS["evictions"] += 1
                self._idle[k0].pop(0)
                if not self._idle[k0]:
                    del self._idle[k0]

    def clear(self):
        with self._lock:
            self._idle.clear()

    def __len__(self):
        with self._lock:
            return sum(len(v) for v in self._idle.values())


POOL = DecoderPool()


class PlanMismatch(RuntimeError):
    """A width plan that does not fit the pooled decoder's buffers."""


def decode_cached(key, factory, model, host_input, kind, items=None, widths=None, lazy=False,
                  graphs=True):
    """One decode through a pooled BeamDecoder: host input (a float32 numpy
    array, features or context rows; or a CUDA tensor) -> pinned staging ->
    H2D into the decoder's static input buffer -> decode (graph replay from
    the second use of a shape on) -> [on-device SID -> item resolution when
    ``items`` = (keys, ids, n)] -> async D2H of results + range flag -> host
    lists.  Returns (per-request [(SemanticId, float)], item slots (B,
    max_out) int32 array or None).  ``widths`` (B, T) re-plans a decoder
    pooled under a capacity key (:meth:`BeamDecoder.set_widths`)."""
    with CAPTURE_GATE.shared():
        dec = POOL.acquire(key, factory)
        if widths is not None and not dec.set_widths(widths):
            POOL.release(key, dec)
            raise PlanMismatch("width plan exceeds the pooled decoder's capacity")
    capture = graphs and dec.graph is None and dec.uses >= 1
    gate = CAPTURE_GATE.exclusive() if capture else CAPTURE_GATE.shared()
    ok = False
    with gate:
        try:
            out = _decode_on(dec, model, host_input, kind, items, lazy, capture)
            ok = True
            return out
        except (InputRangeError, ValueError):
            ok = True  # the decoder itself is fine
            raise
        finally:
            if ok:
                POOL.release(key, dec)


def decode_cached_many(jobs, model, lazy=False, graphs=True):
    """Several pooled decodes pipelined on one stream: every job is staged and
    launched before the first one's results are waited for, so the host
    work of one part (staging its inputs, building the previous part's
    result lists) overlaps the device work of another.  ``jobs``: [(key,
    factory, host_input, kind, items, widths)].  Returns one (results,
    item slots) pair per job."""
    launched = []
    try:
        for key, factory, host_input, kind, items, widths in jobs:
            with CAPTURE_GATE.shared():
                dec = POOL.acquire(key, factory)
                if widths is not None and not dec.set_widths(widths):
                    POOL.release(key, dec)
                    raise PlanMismatch("width plan exceeds the pooled decoder's capacity")
            capture = graphs and dec.graph is None and dec.uses >= 1
            gate = CAPTURE_GATE.exclusive() if capture else CAPTURE_GATE.shared()
            try:
                with gate:
                    ev = _decode_launch(dec, model, host_input, kind, items, capture)
            except (InputRangeError, ValueError):
                POOL.release(key, dec)  # nothing launched on it
                raise
            launched.append([key, dec, ev])
        outs = []
        for entry in launched:
            with CAPTURE_GATE.shared():
                outs.append(_decode_finish(entry[1], entry[2], lazy))
            POOL.release(entry[0], entry[1])
            entry[1] = None
        return outs
    finally:
        for key, dec, ev in launched:
            if dec is not None:  # an error left it in flight: drain, then pool it
                ev.synchronize()
                dec._fetched = None
                POOL.release(key, dec)


class InputRangeError(RuntimeError):
    """A finite float64 input that does not fit the fp32 decode."""


_STAGE_WORKERS = max(1, min(8, (os.cpu_count() or 2) // 2))
_STAGE_POOL = None
_STAGE_LOCK = threading.Lock()


def _stage_pool():
    global _STAGE_POOL
    with _STAGE_LOCK:
        if _STAGE_POOL is None:
            _STAGE_POOL = ThreadPoolExecutor(_STAGE_WORKERS, thread_name_prefix="gr4ad-stage")
        return _STAGE_POOL


def _stage_blocks(blocks, staged):
    """Cast + concatenate per-request float64 blocks into the pinned fp32
    staging rows, split over a few threads (numpy copies release the GIL);
    returns False if a value leaves the fp32 range."""
    offs = np.cumsum([0] + [a.shape[0] for a in blocks])
    n = len(blocks)
    parts = min(_STAGE_WORKERS, max(1, int(offs[-1]) // 16384), n)

    def work(lo, hi):
        out = staged[offs[lo]:offs[hi]]
        with np.errstate(over="ignore"):
            np.concatenate(blocks[lo:hi], 0, out=out, casting="unsafe")
        return bool(np.isfinite(out).all())

    if parts <= 1:
        return work(0, n)
    cuts = [round(k * n / parts) for k in range(parts + 1)]
    futs = [_stage_pool().submit(work, cuts[k], cuts[k + 1]) for k in range(parts)]
    return all(f.result() for f in futs)


def _decode_launch(dec, model, host_input, kind, items, capture=True):
    """Stage, copy and launch one decode (graph replay from the second use of
    a plan on; ``capture=False`` replays an existing graph but captures none)
    and start the results' D2H; returns the completion event."""
    t0 = time.perf_counter()
    if True:
        if dec.weights is not device_weights(model, dec.device):
            dec.rebind(model)  # a republished snapshot of the same shape
        if isinstance(host_input, (list, tuple)):  # per-request float64 blocks
            shape = (sum(a.shape[0] for a in host_input), host_input[0].shape[1])
        else:
            shape = tuple(host_input.shape)
        if dec.in_buf is None or tuple(dec.in_buf.shape) != shape:
            dec.in_buf = torch.empty(shape, dtype=torch.float32, device=dec.device)
            dec._in_host = None
            dec.graph = None
            dec._graphs.clear()  # parked graphs hold the old input pointer
        if isinstance(host_input, torch.Tensor):  # already on the device
            dec.in_buf.copy_(host_input)
        else:
            if dec._in_host is None:
                dec._in_host = torch.empty(shape, dtype=torch.float32).pin_memory()
            staged = dec._in_host.numpy()
            if isinstance(host_input, (list, tuple)):
                # concatenate + cast straight into pinned memory, on a few threads
                ok = _stage_blocks(host_input, staged)
            else:
                with np.errstate(over="ignore"):
                    np.copyto(staged, host_input, casting="unsafe")
                ok = bool(np.isfinite(staged).all())
            if not ok:
                blocks = host_input if isinstance(host_input, (list, tuple)) else [host_input]
                if not all(np.isfinite(np.asarray(a)).all() for a in blocks):
                    raise ValueError("context must be finite")
                raise InputRangeError("an input exceeds the fp32 range of the GPU decode")
            dec.in_buf.copy_(dec._in_host, non_blocking=True)
        inputs = {kind: dec.in_buf}
        t1 = time.perf_counter()
        if dec.graph is not None:
            dec.graph.replay()
        elif capture and dec.uses >= 1:
            # second use of this shape: capture once, replay from now on
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(dec.device)
            s.wait_stream(torch.cuda.current_stream(dec.device))
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                dec.run(**inputs)
            torch.cuda.current_stream(dec.device).wait_stream(s)
            dec.graph = g
            STATS["captures"] += 1
            g.replay()
        else:
            dec.run(**inputs)
        dec.uses += 1
        if items is not None:
            dec.resolve_items(*items)
        ev = dec.fetch_async()
        t2 = time.perf_counter()
        STATS["stage_s"] += t1 - t0
        STATS["launch_s"] += t2 - t1
        return ev


def _decode_finish(dec, ev, lazy=False):
    """Wait for a launched decode's results and build the host lists."""
    t2 = time.perf_counter()
    ev.synchronize()
    t3 = time.perf_counter()
    out = dec.results(lazy)
    t4 = time.perf_counter()
    STATS["calls"] += 1
    STATS["wait_s"] += t3 - t2
    STATS["marshal_s"] += t4 - t3
    return out, dec.last_item_idx


def _decode_on(dec, model, host_input, kind, items, lazy=False, capture=True):
    return _decode_finish(dec, _decode_launch(dec, model, host_input, kind, items, capture), lazy)


@gated
def score_sequences(model, seq_requests, tokens, features=None, contexts=None,
                    include_value_step=False, trunk_depth=None, return_logits=False,
                    device=None, path="auto"):
    """Teacher-forced scoring on the GPU (lazy_forward + sequence_log_prob,
    decoder.py:162-219; the RL-log / oracle scoring path).

    ``features`` (or projected ``contexts``) hold one matrix per request;
    sequence s belongs to request ``seq_requests[s]`` and has ``tokens[s]``
    (one token per level).  Returns ``logp`` (n_seq, T) float64, plus the
    value-bucket logits (n_seq, n_value_buckets) with ``include_value_step``
    and the per-level head logits (list of (n_seq, V_t)) with
    ``return_logits``."""
    dev = require_cuda(device)
    cfg = model.config
    T = cfg.n_levels
    items = features if features is not None else contexts
    if items is None or (features is not None and contexts is not None):
        raise ValueError("pass exactly one of features / contexts")
    arrs = [np.atleast_2d(np.asarray(getattr(a, "data", a), dtype=np.float64)) for a in items]
    toks = np.asarray(tokens, dtype=np.int64).reshape(-1, T)
    for t in range(T):
        col = toks[:, t]
        if col.size and (col.min() < 0 or col.max() >= cfg.level_vocab_sizes[t]):
            bad = int(col[(col < 0) | (col >= cfg.level_vocab_sizes[t])][0])
            raise ValueError(f"token {bad} out of range at level {t}")
    reqs = np.asarray(seq_requests, dtype=np.int32).ravel()
    n_seq = reqs.size
    weights = device_weights(model, dev)
    dims = dims_of(cfg)
    lens = [a.shape[0] for a in arrs]
    ctx = (C.c_int * max(len(lens), 1))(*lens)
    w_arr = (C.c_int * max(len(lens) * T, 1))(*([1] * (len(lens) * T)))
    bt = N.Batch()
    bt.n_requests = len(lens)
    bt.ctx_len = ctx
    bt.widths = w_arr
    bt.trunk_depth = -1 if trunk_depth is None else int(trunk_depth)
    bt.value_rerank = 1 if include_value_step else 0
    vc = (C.c_int * N.MAX_LEVELS)()
    bt.valid_prefix_count = vc
    bt.decode_path = {"auto": 0, "layered": 1, "tensor": 3, "tensor_ctx": 5}[path]
    nbytes = C.c_size_t()
    N.check(N.lib.gr4ad_score_workspace_bytes(C.byref(dims), C.byref(bt), n_seq, C.byref(nbytes)))
    ws = torch.empty(max(nbytes.value, 256), dtype=torch.uint8, device=dev)
    if features is not None:
        inp = torch.from_numpy(np.concatenate(arrs, 0).astype(np.float32)).to(dev)
        f, x = C.c_void_p(inp.data_ptr()), None
    else:
        inp = torch.from_numpy(np.concatenate(arrs, 0).astype(np.float32)).to(dev)
        f, x = None, C.c_void_p(inp.data_ptr())
    tok_d = torch.from_numpy(toks.astype(np.int32)).to(dev)
    logp = torch.zeros((max(n_seq, 1), T), dtype=torch.float32, device=dev)
    vl = torch.zeros((max(n_seq, 1), cfg.n_value_buckets), dtype=torch.float32, device=dev)
    vsum = int(sum(cfg.level_vocab_sizes))
    hl = torch.zeros((max(n_seq, 1), vsum), dtype=torch.float32, device=dev) if return_logits else None
    req_c = (C.c_int * max(n_seq, 1))(*reqs.tolist())
    N.check(N.lib.gr4ad_score_sequences(
        C.byref(dims), C.byref(weights.struct), C.byref(bt), f, x, n_seq, req_c,
        C.c_void_p(tok_d.data_ptr()), C.c_void_p(logp.data_ptr()),
        C.c_void_p(vl.data_ptr()) if include_value_step else None,
        C.c_void_p(hl.data_ptr()) if return_logits else None,
        C.c_void_p(ws.data_ptr()), nbytes.value, _stream_handle(dev)))
    out = [logp.double().cpu().numpy()[:n_seq]]
    if include_value_step:
        out.append(vl.double().cpu().numpy()[:n_seq])
    if return_logits:
        h = hl.double().cpu().numpy()[:n_seq]
        offs = np.cumsum([0] + list(cfg.level_vocab_sizes))
        out.append([h[:, offs[t]:offs[t + 1]] for t in range(T)])
    return out[0] if len(out) == 1 else tuple(out)
