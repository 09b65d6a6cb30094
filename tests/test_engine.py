"""Serving engine, snapshot store and TTL cache, mirroring the reference's
pkg/tests/test_engine.py and test_schedule_cache.py (TestTtlCache), plus
oracle parity of engine results and the GPU snapshot hot swap (SURVEY §8f
row 4).  Host-only pieces run on CPU; anything that decodes is marked gpu."""

import json
import threading

import numpy as np
import pytest

import oracle.beam_oracle as orc
from paper_2602_22732_b200.model.decoder import DecoderConfig, DecoderModel
from paper_2602_22732_b200.quantizer.index import SidIndex
from paper_2602_22732_b200.quantizer.residual import SemanticId
from paper_2602_22732_b200.serving.cache import TtlCache
from paper_2602_22732_b200.serving.engine import ServingConfig, ServingEngine, SnapshotStore
from paper_2602_22732_b200.serving.schedule import (BeamSchedule, TrafficSignal, capacity_slack,
                                                   scale_schedule, tabs_adjust)

from cases import list_parity  # noqa: E402


def _setup(ttl=60.0, index_sids=True, value_rerank=False, preload=None):
    # test_engine.py:12-27
    cfg = DecoderConfig(feat_dim=4, d=4, d_ff=6, n_layers=2, trunk_depth=1,
                        level_vocab_sizes=(3, 3), n_value_buckets=2, seed=5)
    model = DecoderModel(cfg)
    store = SnapshotStore(model, preload=preload)
    index = SidIndex()
    if index_sids:
        n = 0
        for a in range(3):
            for b in range(3):
                index.upsert(f"item{n}", SemanticId((a, b), (3, 3)))
                n += 1
    engine = ServingEngine(store, index, ServingConfig(
        schedule=BeamSchedule((2, 4), base_width=4), q_threshold=10.0,
        ttl=ttl, value_rerank=value_rerank))
    return engine, store, index, model


def _features():
    return np.ones((1, 4))


# ---------------------------------------------------------------- host only

class TestTtlCache:  # test_schedule_cache.py:70-140
    def test_hit_within_ttl(self):
        cache = TtlCache(60.0)
        cache.put("k", "v", now=0.0)
        assert cache.get("k", now=30.0) == "v"

    def test_miss_after_ttl_boundary_strict(self):
        cache = TtlCache(60.0)
        cache.put("k", "v", now=0.0)
        assert cache.get("k", now=61.0) is None
        cache.put("k", "v", now=0.0)
        assert cache.get("k", now=60.0) is None

    def test_never_returns_stale_under_scan(self):
        cache = TtlCache(5.0)
        rng = np.random.default_rng(0)
        now = 0.0
        for _ in range(2000):
            now += float(rng.exponential(1.0))
            key = int(rng.integers(0, 8))
            value = cache.get(key, now=now)
            if value is not None:
                assert now - value < 5.0
            else:
                cache.put(key, now, now=now)

    def test_replay_hit_rate_matches_counting_oracle(self):
        ttl = 3.0
        rng = np.random.default_rng(1)
        times = np.cumsum(rng.exponential(1.0, size=500))
        cache = TtlCache(ttl)
        hits, inserted = 0, None
        for now in times:
            if inserted is not None and now - inserted < ttl:
                hits += 1
            else:
                inserted = now
            if cache.get("u", now) is None:
                cache.put("u", "r", now)
        assert cache.hits == hits

    def test_purge_and_len(self):
        cache = TtlCache(10.0)
        cache.put("a", 1, now=0.0)
        cache.put("b", 2, now=5.0)
        assert len(cache) == 2
        assert cache.purge(now=12.0) == 1
        assert len(cache) == 1

    def test_validation(self):
        with pytest.raises(ValueError):
            TtlCache(0)

    def test_concurrent_access(self):
        cache = TtlCache(100.0)
        errors = []

        def worker(n):
            try:
                for i in range(500):
                    cache.put((n, i % 7), i, now=float(i))
                    cache.get((n, (i + 3) % 7), now=float(i))
            except Exception as exc:  # pragma: no cover
                errors.append(exc)

        ts = [threading.Thread(target=worker, args=(n,)) for n in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors
        assert cache.hits + cache.misses == 4 * 500


def test_schedule_matches_oracle_integers():
    for qps in (0.0, 1.0, 9.99, 10.0, 50.0):
        for slack in (0.0, 0.25, 0.5, 1.0):
            for base in (4, 16, 256, 512):
                got = tabs_adjust(TrafficSignal(qps, 10.0, slack), base, 0.6)
                assert got == orc.tabs_adjust(qps, 10.0, slack, base, 0.6)
                sch = scale_schedule(BeamSchedule((base // 4 or 1, base // 2 or 1, base), base), got)
                assert sch.widths == orc.scale_widths((base // 4 or 1, base // 2 or 1, base),
                                                      base, got)
    assert capacity_slack(0.0, 10.0) == 1.0
    assert capacity_slack(20.0, 10.0) == 0.0
    assert capacity_slack(2.5, 10.0) == 0.75
    with pytest.raises(ValueError):
        TrafficSignal(-1.0, 10.0, 0.5)
    with pytest.raises(ValueError):
        TrafficSignal(1.0, 10.0, 1.5)


def test_snapshot_store_versions_and_isolation():  # test_engine.py:135-151
    cfg = DecoderConfig(feat_dim=4, d=4, d_ff=6, n_layers=2, trunk_depth=0,
                        level_vocab_sizes=(3,), n_value_buckets=2, seed=1)
    model = DecoderModel(cfg)
    store = SnapshotStore(model, preload=False)
    v1, snap1 = store.current()
    model.params["bos"].data += 100.0
    _, snap1_again = store.current()
    np.testing.assert_array_equal(snap1.params["bos"].data, snap1_again.params["bos"].data)
    v2 = store.publish(model)
    assert v2 == v1 + 1
    _, snap2 = store.current()
    assert not np.array_equal(snap1.params["bos"].data, snap2.params["bos"].data)
    v3 = store.publish_async(model).result(timeout=60)
    assert v3 == v2 + 1 and store.current()[0] == v3


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_cold_request_invokes_model_once():
    engine, _, _, _ = _setup()
    result = engine.serve_request("u1", _features(), now=0.0, qps=20.0)
    assert not result.from_cache
    assert engine.model_invocations == 1
    assert 1 <= len(result.items) <= 4


@pytest.mark.gpu
def test_cached_request_skips_model():
    engine, _, _, _ = _setup()
    engine.serve_request("u1", _features(), now=0.0, qps=20.0)
    result = engine.serve_request("u1", _features(), now=30.0, qps=20.0)
    assert result.from_cache
    assert engine.model_invocations == 1
    expired = engine.serve_request("u1", _features(), now=61.0, qps=20.0)
    assert not expired.from_cache
    assert engine.model_invocations == 2


@pytest.mark.gpu
def test_distinct_users_not_shared_and_index_update_invalidates():
    engine, _, index, _ = _setup()
    engine.serve_request("u1", _features(), now=0.0, qps=20.0)
    assert not engine.serve_request("u2", _features(), now=1.0, qps=20.0).from_cache
    index.upsert("fresh", SemanticId((0, 0), (3, 3)))
    assert not engine.serve_request("u1", _features(), now=1.0, qps=20.0).from_cache


@pytest.mark.gpu
def test_unindexed_sids_skipped_without_error():
    engine, _, index, _ = _setup(index_sids=False)
    index.upsert("only", SemanticId((0, 0), (3, 3)))
    result = engine.serve_request("u1", _features(), now=0.0, qps=20.0)
    assert len(result.items) <= 1
    assert all(item == "only" for item, _ in result.items)


@pytest.mark.gpu
def test_offpeak_widens_schedule_and_matches_oracle():
    engine, _, _, model = _setup()
    peak = engine.serve_request("u1", _features(), now=0.0, qps=20.0)
    off = engine.serve_request("u2", _features(), now=0.0, qps=1.0)
    assert peak.widths == (2, 4)
    assert off.widths == (3, 6)  # 60% boost, rounded half-up
    cfg = model.config
    x = orc.context_process(_features(), orc.plain_params(model.params))
    for res in (peak, off):
        ref = orc.beam_search(model.params, cfg, x, res.widths)
        got = [(tuple(s.tokens) if hasattr(s, "tokens") else tuple(s), sc) for s, sc in res.sids]
        ok, msg = list_parity(ref, got, 1e-5)
        assert ok, msg
        scores = [s for _, s in res.items]
        assert scores == sorted(scores, reverse=True)
        assert len(res.items) <= res.widths[-1]


@pytest.mark.gpu
def test_record_is_json_friendly():
    engine, _, _, _ = _setup()
    result = engine.serve_request("u1", _features(), now=2.0, qps=20.0)
    parsed = json.loads(json.dumps(result.record("u1", 2.0)))
    assert parsed["user_id"] == "u1"
    assert parsed["snapshot_version"] == 1
    assert not parsed["from_cache"]


@pytest.mark.gpu
def test_concurrent_requests_consistent_counters():
    engine, _, _, _ = _setup(ttl=0.001)
    errors = []

    def worker(uid):
        try:
            for i in range(10):
                res = engine.serve_request(f"u{uid}", _features(), now=float(i), qps=20.0)
                assert res.items
        except Exception as exc:  # pragma: no cover
            errors.append(exc)

    ts = [threading.Thread(target=worker, args=(n,)) for n in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
    assert engine.requests == 40
    assert engine.model_invocations == 40


@pytest.mark.gpu
def test_serve_batch_mixed_hits_and_misses_match_oracle():
    engine, _, _, model = _setup()
    rng = np.random.default_rng(3)
    feats = {f"u{i}": rng.normal(size=(int(rng.integers(1, 9)), 4)) for i in range(12)}
    first = engine.serve_batch([(u, f) for u, f in list(feats.items())[:6]], now=0.0, qps=20.0)
    both = engine.serve_batch(list(feats.items()), now=1.0, qps=20.0)
    assert [r.from_cache for r in both] == [True] * 6 + [False] * 6
    assert engine.model_invocations == 12
    for r0, r1 in zip(first, both[:6]):
        assert r0.items == r1.items
    for (u, f), res in zip(feats.items(), both):
        x = orc.context_process(f, orc.plain_params(model.params))
        ref = orc.beam_search(model.params, model.config, x, res.widths)
        got = [(tuple(s.tokens) if hasattr(s, "tokens") else tuple(s), sc) for s, sc in res.sids]
        ok, msg = list_parity(ref, got, 1e-5)
        assert ok, (u, msg)


@pytest.mark.gpu
def test_snapshot_hot_swap_under_load():
    """Publishing from another thread while a decode loop runs: every result
    is exactly the decode of the snapshot version it reports, the swap needs
    no host synchronisation of the serving stream, and the new version's
    device copy is staged before the first request that uses it."""
    import torch

    from paper_2602_22732_b200 import device as dv
    from paper_2602_22732_b200.decode import BeamDecoder

    cfg = DecoderConfig(16, 16, 32, 2, 1, (64, 64, 64), 4, seed=11)
    base = DecoderModel(cfg)
    store = SnapshotStore(base)
    models = {1: store.current()[1]}
    rng = np.random.default_rng(4)
    feats = torch.from_numpy(rng.normal(size=(8 * 32, 16)).astype(np.float32)).cuda()
    widths = [(4, 8, 16)] * 8
    expect = {}

    def decode_with(model):
        dec = BeamDecoder(model, [32] * 8, widths)
        dec.run(features=feats)
        return dec.host_results()

    expect[1] = decode_with(models[1])
    versions = []
    pending = []
    stop = threading.Event()

    def publisher():
        m = base.clone()
        for _ in range(3):
            m.params["head.0"].data += 0.5 * np.random.default_rng(len(pending)).normal(
                size=m.params["head.0"].data.shape)
            m.params["layer1.ffn.W1"].data *= 1.01
            pending.append(store.publish_async(m).result(timeout=120))
        stop.set()

    th = threading.Thread(target=publisher)
    dec = BeamDecoder(models[1], [32] * 8, widths)
    th.start()
    seen = []
    while not stop.is_set() or len(seen) < 4:
        ver, model = store.current()
        models[ver] = model
        dec.rebind(model)
        dec.run(features=feats)
        seen.append((ver, dec.host_results()))
        if len(seen) > 400:
            break
    th.join()
    ver, model = store.current()
    models[ver] = model
    dec.rebind(model)
    dec.run(features=feats)
    seen.append((ver, dec.host_results()))
    assert pending == [2, 3, 4]
    assert seen[-1][0] == 4
    for ver, res in seen:
        if ver not in expect:
            expect[ver] = decode_with(models[ver])
        assert res == expect[ver], f"version {ver}"
    # distinct snapshots decode differently (the swap really changed weights)
    assert expect[1] != expect[4]
    # the published snapshot is resident before first use
    key = (id(models[4].params), str(torch.device("cuda")))
    assert key in dv._CACHE
