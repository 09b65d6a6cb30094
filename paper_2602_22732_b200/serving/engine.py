"""Request-level serving (engine.py:17-125 in the reference): snapshot
store, TTL cache, traffic-aware widths, GPU beam generation and SID->item
resolution.

``ServingEngine.serve_request`` keeps the reference's per-request contract.
``serve_batch`` is the throughput path: cache lookups on the host, then ONE
batched GPU decode for every miss -- each with its own TABS-scaled widths --
with the context projection, encoder K/V, trunk, level steps and
compaction all on the device.
"""

from __future__ import annotations

import threading
import time
import weakref
from concurrent.futures import Future
from dataclasses import dataclass

import numpy as np
import torch

from ..model.layers import LayerCallCounter
from .beam import beam_search_batch, record_counter
from .cache import TtlCache
from .schedule import TrafficSignal, scale_schedule, tabs_adjust


class SnapshotStore:
    """Copy-on-publish model snapshots (engine.py:17-36), double-buffered on
    the GPU.

    ``publish`` clones the model (the reference contract), packs it and
    uploads it on a side stream from pinned memory, then swaps the current
    version atomically: decodes already enqueued keep reading the previous
    device copy (kept alive by the allocator's stream tracking until they
    finish), later decodes order themselves after the upload on the GPU.
    ``publish_async`` runs the clone/pack/upload on a worker thread so the
    serving thread never stalls on a publish.  Without a CUDA device it is
    the reference's host-only store.
    """

    def __init__(self, model=None, device=None, preload=None):
        self._lock = threading.Lock()
        self._publish_lock = threading.Lock()
        self._version = 0
        self._model = None
        self._preload = torch.cuda.is_available() if preload is None else preload
        self._device = device
        self._stream = None
        if model is not None:
            self.publish(model)

    def _stage(self, snapshot):
        if not self._preload:
            return
        from ..device import CAPTURE_GATE
        with CAPTURE_GATE.shared():
            self._stage_locked(snapshot)

    def _stage_locked(self, snapshot):
        from ..device import DeviceWeights, register, require_cuda
        dev = require_cuda(self._device)
        if self._stream is None:
            self._stream = torch.cuda.Stream(dev)
        register(snapshot, DeviceWeights(snapshot, dev, stream=self._stream))

    def publish(self, model):
        snapshot = model.clone()
        with self._publish_lock:  # versions are issued in publish order
            self._stage(snapshot)
            with self._lock:
                self._version += 1
                self._model = snapshot
                return self._version

    def publish_async(self, model):
        """Publish from a worker thread; returns a Future of the version."""
        fut = Future()

        def work():
            try:
                fut.set_result(self.publish(model))
            except BaseException as exc:  # pragma: no cover - surfaced via the future
                fut.set_exception(exc)

        threading.Thread(target=work, daemon=True).start()
        return fut

    def current(self):
        with self._lock:
            return self._version, self._model


@dataclass
class ServingConfig:
    schedule: object  # BeamSchedule
    q_threshold: float = 100.0
    boost: float = 0.6
    ttl: float = 60.0
    shared_kv: bool = True
    precut: bool = True
    value_rerank: bool = False
    mask_to_index: bool = False  # extension: valid-SID prefix masking
    # batched engine (no reference counterpart; the reference serves one
    # request per call): a batch's misses are padded to the next of these
    # sizes so the pooled decoders (and their CUDA graphs) are reused across
    # batches; None decodes exactly the misses
    batch_buckets: tuple = (1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 384, 512)
    # TABS widths from the engine's own load signal: "batch" measures it once
    # per batch (the reference's per-tick traffic signal, sim/loop.py:239-264),
    # "request" at every request's arrival (per-request widths in one batch)
    load_widths: str = "batch"


@dataclass
class ServeResult:
    items: list
    sids: list
    from_cache: bool
    snapshot_version: int
    widths: tuple
    latency_virtual: int = 0

    def record(self, user_id, now):
        return {"user_id": user_id, "ts": float(now),
                "items": [[i, float(s)] for i, s in self.items],
                "from_cache": self.from_cache, "snapshot_version": self.snapshot_version,
                "widths": list(self.widths), "latency_virtual": self.latency_virtual}


class LoadEstimator:
    """Online load signal for TABS (N1): the reference's caller measures
    traffic per tick and passes ``qps`` / ``capacity_slack`` to every
    request (sim/loop.py:239-264 -> engine.py:100-103).  Here the engine
    measures both itself:

    * arrival rate -- requests seen in a sliding window of ``window``
      seconds of request time (``now``), so each request's rate is the one
      at its own arrival;
    * capacity -- requests decoded per second of decode time, an EWMA over
      the engine's own GPU batches (wall time around each batched decode,
      results on the host); only batches of at least half the largest batch
      seen update it (a small batch is latency-bound and would read as a
      low capacity).

    ``capacity_slack = clamp(1 - rate / capacity, 0, 1)`` (the C4 sweep's
    definition); 1.0 until a capacity has been measured."""

    def __init__(self, window=1.0, alpha=0.2):
        self.window = float(window)
        self.alpha = float(alpha)
        self._arrivals = []  # sorted request times inside the window
        self._head = 0
        self.capacity = None  # requests / s of decode time
        self._max_batch = 0
        self._lock = threading.Lock()

    def observe(self, now, n=1):
        with self._lock:
            self._arrivals.extend([float(now)] * int(n))

    def observe_many(self, times):
        """Arrivals at each of ``times`` (non-decreasing), one lock."""
        with self._lock:
            self._arrivals.extend(float(t) for t in times)

    def rate(self, now):
        with self._lock:
            lo = float(now) - self.window
            arr = self._arrivals
            h = self._head
            while h < len(arr) and arr[h] <= lo:
                h += 1
            if h > 4096 and h * 2 > len(arr):
                del arr[:h]
                h = 0
            self._head = h
            upto = len(arr)
            while upto > h and arr[upto - 1] > now:
                upto -= 1
            return (upto - h) / self.window

    def record_service(self, n_requests, seconds, concurrency=1.0):
        """A batch of ``n_requests`` decoded in ``seconds`` of wall time while
        ``concurrency`` batches (on average) were being served at once: the
        engine's rate is the batch's rate times the overlap."""
        if n_requests <= 0 or seconds <= 0:
            return
        c = n_requests * max(1.0, float(concurrency)) / seconds
        with self._lock:
            self._max_batch = max(self._max_batch, int(n_requests))
            if 2 * n_requests < self._max_batch:
                return
            self.capacity = c if self.capacity is None else (
                (1 - self.alpha) * self.capacity + self.alpha * c)

    def signal(self, now):
        """(qps, capacity_slack) at request time ``now`` -- an arrival time:
        the engine sees arrivals only when they are served, so under a
        backlog the rate at the serving wall time would count none of them
        (and read as idle)."""
        qps = self.rate(now)
        cap = self.capacity
        slack = 1.0 if not cap else min(1.0, max(0.0, 1.0 - qps / cap))
        return qps, slack


class ItemTable:
    """Device copy of a SidIndex for on-device SID -> item resolution
    (gr4ad_resolve_items): sorted mixed-radix SID keys (int64) and, per key,
    the slot of min(item ids) (engine.py:114-118 takes min(ids)) in
    ``items``.  Built once per index version."""

    def __init__(self, index, vocab, device):
        sids, items = [], []
        fwd = index.snapshot()  # a consistent copy of the forward map
        T = len(vocab)
        for sid, ids in fwd:
            toks = getattr(sid, "tokens", sid)
            if len(toks) != T or not ids:
                continue
            sids.append(toks)
            items.append(min(ids))
        tok = np.asarray(sids, dtype=np.int64).reshape(-1, T)
        voc = np.asarray(vocab, dtype=np.int64)
        # a SID of another vocabulary can never be decoded
        ok = ((tok >= 0) & (tok < voc)).all(1) if tok.size else np.zeros(0, bool)
        tok = tok[ok]
        keys = np.zeros(tok.shape[0], dtype=np.int64)
        for t in range(T):
            keys = keys * voc[t] + tok[:, t]
        order = np.argsort(keys, kind="stable")
        self.n = int(keys.size)
        k_sorted = keys[order] if self.n else np.zeros(1, np.int64)
        kept = np.flatnonzero(ok)
        self.items = np.empty(max(self.n, 1), dtype=object)
        if self.n:
            self.items[:self.n] = [items[i] for i in kept[order].tolist()]
        self.keys = torch.from_numpy(np.ascontiguousarray(k_sorted)).to(device)
        self.ids = torch.arange(max(self.n, 1), dtype=torch.int32, device=device)

    def args(self):
        return (self.keys, self.ids, self.n)

    def resolve_batch(self, sids_list, slots):
        """resolve() for every request of a batch at once: one pass over the
        (B, max_out) slot array, item lists built only where SIDs hit."""
        B = len(sids_list)
        out = [[] for _ in range(B)]
        if B == 0:
            return out
        slots = np.asarray(slots)[:B]
        n = np.fromiter((len(x) for x in sids_list), dtype=np.int64, count=B)
        live = (np.arange(slots.shape[1])[None, :] < n[:, None]) & (slots >= 0)
        rows, cols = np.nonzero(live)
        if rows.size:
            objs = self.items[slots[rows, cols]].tolist()
            for r, c, o in zip(rows.tolist(), cols.tolist(), objs):
                sids = sids_list[r]
                sc = getattr(sids, "scores", None)
                out[r].append((o, float(sc[c]) if sc is not None else float(sids[c][1])))
        return out

    def resolve(self, sids, slots):
        """[(item, score)] for one request from its SID list and slot row."""
        n = len(sids)
        row = slots[:n]
        keep = np.flatnonzero(row >= 0)
        if keep.size == 0:
            return []
        objs = self.items[row[keep]].tolist()
        sc = getattr(sids, "scores", None)  # (a SidList: no SemanticIds built)
        if sc is not None:
            return [(o, float(sc[j])) for o, j in zip(objs, keep.tolist())]
        return [(o, float(sids[j][1])) for o, j in zip(objs, keep.tolist())]


_TABLES = weakref.WeakKeyDictionary()  # SidIndex -> (version, vocab, device, ItemTable)


class ServingEngine:
    def __init__(self, store, index, config, buckets=None, counter=None, load=None):
        self.store = store
        self.index = index
        self.config = config
        self.buckets = buckets
        self.counter = counter if counter is not None else LayerCallCounter()
        self.cache = TtlCache(config.ttl)
        self._lock = threading.Lock()
        self.model_invocations = 0
        self.requests = 0
        self.load = load if load is not None else LoadEstimator()
        self._table = None  # (index version, vocab, ItemTable)
        self._valid = None  # (index version, tuple of its SIDs) for masked decoding
        self._cf_memo = {}  # (config, widths, S, ...) -> closed-form counters
        self._inflight = 0  # serve_batch calls decoding right now (load estimate)
        model = store.current()[1] if torch.cuda.is_available() else None
        if model is not None:  # off the first request's latency
            self._item_table(model)

    def _widths(self, qps, capacity_slack):
        sig = TrafficSignal(qps, self.config.q_threshold, capacity_slack)
        active = tabs_adjust(sig, self.config.schedule.base_width, self.config.boost)
        return scale_schedule(self.config.schedule, active)

    def _item_table(self, model):
        """The device SID -> item table of the current index version, shared
        by every engine serving the same index (built once per version)."""
        vocab = tuple(model.config.level_vocab_sizes)
        version = self.index.version
        tab = self._table
        if tab is None or tab[0] != version or tab[1] != vocab:
            from ..device import CAPTURE_GATE, require_cuda
            dev = require_cuda()
            shared = _TABLES.get(self.index)
            if shared is not None and shared[:3] == (version, vocab, str(dev)):
                tab = (version, vocab, shared[3])
            else:
                with CAPTURE_GATE.shared():
                    tab = (version, vocab, ItemTable(self.index, vocab, dev))
                _TABLES[self.index] = (version, vocab, str(dev), tab[2])
            self._table = tab
        return tab[2]

    def _resolve(self, sids):
        items = []
        for sid, score in sids:
            ids = self.index.lookup(sid)
            if ids:
                items.append((min(ids), float(score)))
        return items

    def serve_request(self, user_id, features, now, qps=None, capacity_slack=1.0):
        """One request: cache first; on a miss, traffic-scaled GPU beam
        generation and ID resolution (engine.py:84-121).  ``qps=None``
        takes the engine's own measured load (:class:`LoadEstimator`)."""
        return self.serve_batch([(user_id, features)], now, qps, capacity_slack)[0]

    def serve_batch(self, requests, now, qps=None, capacity_slack=1.0):
        """requests: [(user_id, features)] or [(user_id, features, t_arrival)]
        -> [ServeResult] in order.

        All cache misses decode in ONE batched GPU call (context projection,
        encoder K/V, trunk, level steps, compaction and SID -> item
        resolution on the device).  Widths: with an explicit ``qps`` every
        miss gets scale_schedule(tabs_adjust(qps, capacity_slack)) as in the
        reference; with ``qps=None`` the engine's own load signal sets them --
        read once at the batch's latest arrival (``load_widths="batch"``), or
        at every request's arrival (``"request"``: per-request widths inside
        one batch)."""
        with self._lock:
            self.requests += len(requests)
        version_key = self.index.version
        out = [None] * len(requests)
        misses = []
        if qps is None:
            self.load.observe_many([req[2] if len(req) > 2 else now for req in requests])
        for i, req in enumerate(requests):
            uid = req[0]
            cached = self.cache.get((uid, version_key), now)
            if cached is not None:
                out[i] = ServeResult(cached[0], cached[1], True, cached[2], cached[3], 0)
            else:
                misses.append(i)
        if not misses:
            return out
        version, model = self.store.current()
        if qps is not None:
            scheds = [self._widths(qps, capacity_slack)] * len(misses)
        elif self.config.load_widths == "batch":
            # one reading per batch, at its latest arrival (a queued batch's
            # arrivals all lie in the past: reading at `now` would see none)
            t_last = max((requests[i][2] for i in misses if len(requests[i]) > 2),
                         default=now)
            scheds = [self._widths(*self.load.signal(t_last))] * len(misses)
        else:
            scheds = []
            for i in misses:
                t_arr = requests[i][2] if len(requests[i]) > 2 else now
                scheds.append(self._widths(*self.load.signal(t_arr)))
        valid = self._valid_sids()
        feats = [np.atleast_2d(np.asarray(requests[i][1], dtype=np.float64)) for i in misses]
        table = self._item_table(model)
        # pad to a batch bucket with copies of the last miss (results dropped)
        n = len(misses)
        pad = n
        for b in self.config.batch_buckets or ():
            if b >= n:
                pad = b
                break
        dfeats = feats + [feats[-1]] * (pad - n)
        dscheds = list(scheds) + [scheds[-1]] * (pad - n)
        with self._lock:
            self._inflight += 1
            k0 = self._inflight
        t0 = time.perf_counter()
        results, slots = beam_search_batch(
            model, features=dfeats, schedules=dscheds, shared_kv=self.config.shared_kv,
            precut=self.config.precut, value_rerank=self.config.value_rerank,
            buckets=self.buckets, valid_sids=valid, _items=table.args(),
            _capacity=self._capacity_widths(), _lazy=True,
            # serving replays the graphs warmup() captured (base and widest
            # plans) and launches other width plans directly: a capture
            # (10-40 ms at C5) never lands on a request's latency
            _graphs=False)
        dt = time.perf_counter() - t0
        with self._lock:
            k1 = self._inflight
            self._inflight -= 1
        # concurrent serving threads share the GPU: scale by the overlap
        self.load.record_service(n, dt, 0.5 * (k0 + k1))
        with self._lock:
            self.model_invocations += len(misses)
        calls = kv_b = kv_f = 0
        item_lists = table.resolve_batch(results[:n], slots)
        for j, (i, sids) in enumerate(zip(misses, results)):
            uid = requests[i][0]
            sched = scheds[j]
            items = item_lists[j]
            self.cache.put((uid, version_key), (items, sids, version, sched.widths), now)
            # per-request virtual latency: the closed-form layer calls of its decode
            c = self._closed_form(model.config, sched.widths, feats[j].shape[0])
            calls += c[0]
            kv_b += c[1]
            kv_f = max(kv_f, c[2])
            out[i] = ServeResult(items, sids, False, version, sched.widths, latency_virtual=c[0])
        self.counter.add_layer_calls(calls)
        self.counter.add_kv_build(kv_b, kv_f)
        return out

    def warmup(self, features, max_batch=None, widths=None):
        """Build and graph-capture the pooled decoders of every batch bucket
        up to ``max_batch`` for one request shape (``features``: an example
        (S, F) matrix), at the base and the widest TABS schedule, so the
        first requests of a bucket do not pay for workspace allocation and
        capture (CUDA-graph warmup at server start).  Nothing is cached."""
        version, model = self.store.current()
        f = np.atleast_2d(np.asarray(features, dtype=np.float64))
        buckets = [b for b in (self.config.batch_buckets or ())
                   if max_batch is None or b <= max_batch]
        cap = self._capacity_widths()
        plans = widths if widths is not None else [self.config.schedule.widths, cap]
        valid = self._valid_sids()
        table = self._item_table(model)
        for b in buckets:
            for w in plans:
                for _ in range(2):  # the second use captures the plan's graph
                    # (with the item resolution serving runs, so the decoders'
                    # pinned result buffers already have their serving layout)
                    beam_search_batch(model, features=[f] * b, schedules=[tuple(w)] * b,
                                      shared_kv=self.config.shared_kv,
                                      value_rerank=self.config.value_rerank,
                                      buckets=self.buckets, valid_sids=valid,
                                      _items=table.args(), _capacity=cap, _lazy=True)

    def _valid_sids(self):
        """The index's SIDs as one tuple per index version (masked decoding;
        the tuple's digest -- part of the pooled decoder's key -- is cached)."""
        if not self.config.mask_to_index:
            return None
        vs = self._valid
        if vs is None or vs[0] != self.index.version:
            vs = (self.index.version, tuple(self.index.all_sids()))
            self._valid = vs
        return vs[1]

    def _capacity_widths(self):
        """The widest schedule TABS can produce (slack 1, or the base when
        boost <= 0): pooled decoders are planned for it and re-planned per
        batch for the load's widths (BeamDecoder.set_widths)."""
        base = self.config.schedule
        wide = scale_schedule(base, tabs_adjust(TrafficSignal(0.0, 1.0, 1.0),
                                                base.base_width, self.config.boost))
        return tuple(max(a, b) for a, b in zip(base.widths, wide.widths))

    def _closed_form(self, cfg, widths, s_ctx):
        """(layer calls, kv builds, kv floats) of one request's decode
        (record_counter's closed form), memoised per (config, widths, S)."""
        key = (cfg, tuple(widths), int(s_ctx), self.config.shared_kv, self.config.value_rerank)
        memo = self._cf_memo
        hit = memo.get(key)
        if hit is None:
            c = LayerCallCounter()
            record_counter(c, cfg, widths, s_ctx, self.config.shared_kv,
                           self.config.value_rerank, cfg.trunk_depth)
            hit = (c.layer_calls, c.kv_builds, c.kv_floats)
            if len(memo) > 4096:
                memo.clear()
            memo[key] = hit
        return hit

    def hit_rate(self):
        total = self.cache.hits + self.cache.misses
        return self.cache.hits / total if total else 0.0
