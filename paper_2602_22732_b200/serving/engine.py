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
from concurrent.futures import Future
from dataclasses import dataclass

import numpy as np
import torch

from ..model.layers import LayerCallCounter
from .beam import beam_search_batch
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


class ServingEngine:
    def __init__(self, store, index, config, buckets=None, counter=None):
        self.store = store
        self.index = index
        self.config = config
        self.buckets = buckets
        self.counter = counter if counter is not None else LayerCallCounter()
        self.cache = TtlCache(config.ttl)
        self._lock = threading.Lock()
        self.model_invocations = 0
        self.requests = 0

    def _widths(self, qps, capacity_slack):
        sig = TrafficSignal(qps, self.config.q_threshold, capacity_slack)
        active = tabs_adjust(sig, self.config.schedule.base_width, self.config.boost)
        return scale_schedule(self.config.schedule, active)

    def _resolve(self, sids):
        items = []
        for sid, score in sids:
            ids = self.index.lookup(sid)
            if ids:
                items.append((min(ids), float(score)))
        return items

    def serve_request(self, user_id, features, now, qps, capacity_slack=1.0):
        """One request: cache first; on a miss, traffic-scaled GPU beam
        generation and ID resolution (engine.py:84-121)."""
        return self.serve_batch([(user_id, features)], now, qps, capacity_slack)[0]

    def serve_batch(self, requests, now, qps, capacity_slack=1.0):
        """requests: [(user_id, features)] -> [ServeResult] in order."""
        with self._lock:
            self.requests += len(requests)
        version_key = self.index.version
        out = [None] * len(requests)
        misses = []
        for i, (uid, feats) in enumerate(requests):
            cached = self.cache.get((uid, version_key), now)
            if cached is not None:
                out[i] = ServeResult(cached[0], cached[1], True, cached[2], cached[3], 0)
            else:
                misses.append(i)
        if not misses:
            return out
        version, model = self.store.current()
        sched = self._widths(qps, capacity_slack)
        valid = self.index.all_sids() if self.config.mask_to_index else None
        feats = [np.atleast_2d(np.asarray(requests[i][1], dtype=np.float64)) for i in misses]
        # one GPU launch for all misses; per-request latency_virtual from the
        # closed-form counter (engine.py:106-111)
        local = LayerCallCounter()
        results = beam_search_batch(model, features=feats, schedules=[sched] * len(misses),
                                    shared_kv=self.config.shared_kv, precut=self.config.precut,
                                    counter=local, value_rerank=self.config.value_rerank,
                                    buckets=self.buckets, valid_sids=valid)
        per_req = local.layer_calls // max(len(misses), 1)
        self.counter.add_layer_calls(local.layer_calls)
        self.counter.add_kv_build(local.kv_builds, local.kv_floats)
        with self._lock:
            self.model_invocations += len(misses)
        for i, sids in zip(misses, results):
            uid = requests[i][0]
            items = self._resolve(sids)
            self.cache.put((uid, version_key), (items, sids, version, sched.widths), now)
            out[i] = ServeResult(items, sids, False, version, sched.widths,
                                 latency_virtual=per_req)
        return out

    def hit_rate(self):
        total = self.cache.hits + self.cache.misses
        return self.cache.hits / total if total else 0.0
