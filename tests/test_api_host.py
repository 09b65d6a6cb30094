"""Host-side API checks (CPU, no GPU): the product's DecoderModel init and
checkpoint format against the reference's, SemanticId's contract, the bulk
result materialisation of the drop-in API, argument validation that must
fire before any device work, and the engine's online load estimator."""

import gc
import hashlib
import os
import pickle
import time

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2602_22732_b200.model import DecoderConfig, DecoderModel
from paper_2602_22732_b200.model.decoder import load_checkpoint, save_checkpoint
from paper_2602_22732_b200.quantizer import SemanticId


def _digest(params):
    h = hashlib.sha256()
    for k, v in params.items():
        h.update(k.encode())
        h.update(np.ascontiguousarray(v.data, dtype=np.float64).tobytes())
    return h.hexdigest()


def test_product_init_matches_reference_sha256(golden_small):
    """DecoderModel(cfg) is bit-identical to the reference's init
    (decoder.py:71-107), checked on the product class (not the oracle)."""
    for rec in golden_small["init"]:
        c = rec["config"]
        cfg = DecoderConfig(c["feat_dim"], c["d"], c["d_ff"], c["n_layers"], c["trunk_depth"],
                            tuple(c["level_vocab_sizes"]), c["n_value_buckets"], c["seed"])
        assert _digest(DecoderModel(cfg).params) == rec["sha256"]


def test_reference_checkpoint_loads_exactly():
    """A checkpoint written by the reference's save_checkpoint
    (tests/golden/ref_checkpoint.npz) loads into the same config, step,
    extras, meta and parameters (reference test_model.py:212-227)."""
    model, step, extra, meta = load_checkpoint(os.path.join(GOLDEN, "ref_checkpoint.npz"))
    want = DecoderModel(DecoderConfig(3, 4, 6, 2, 1, (3, 3), 3, seed=123))
    assert model.config == want.config
    assert step == 17 and meta == {"note": "test"}
    np.testing.assert_array_equal(extra["adam_t"], [17])
    assert set(model.params) == set(want.params)
    for k in want.params:
        np.testing.assert_array_equal(model.params[k].data, want.params[k].data)


def test_checkpoint_written_here_matches_reference_layout(tmp_path):
    """Our save_checkpoint writes the reference's npz layout: same entries,
    same header JSON, same arrays (so the reference's load_checkpoint reads
    it)."""
    model = DecoderModel(DecoderConfig(3, 4, 6, 2, 1, (3, 3), 3, seed=123))
    path = tmp_path / "ours.npz"
    save_checkpoint(model, path, step=17, extra_arrays={"adam_t": np.array([17])},
                    meta={"note": "test"})
    with np.load(path) as ours, np.load(os.path.join(GOLDEN, "ref_checkpoint.npz")) as ref:
        assert sorted(ours.files) == sorted(ref.files)
        import json
        assert json.loads(bytes(ours["header"]).decode()) == json.loads(
            bytes(ref["header"]).decode())
        for k in ref.files:
            np.testing.assert_array_equal(ours[k], ref[k])


def test_semantic_id_contract():
    """residual.py:44-59: validation, equality / hashing by (tokens, vocab),
    immutability, len, pickling."""
    a = SemanticId((1, 2), (3, 3))
    assert a.tokens == (1, 2) and a.level_vocab_sizes == (3, 3) and len(a) == 2
    assert isinstance(a, SemanticId)
    assert a == SemanticId([1, 2], [3, 3])
    assert a != SemanticId((1, 2), (4, 4))
    assert a != (1, 2) and (1, 2) != a
    assert hash(a) == hash(SemanticId((1, 2), (3, 3)))
    assert {a: 1}[SemanticId((1, 2), (3, 3))] == 1
    assert pickle.loads(pickle.dumps(a)) == a
    assert "tokens=(1, 2)" in repr(a)
    with pytest.raises(AttributeError):
        a.tokens = (0, 0)
    with pytest.raises(ValueError, match="out of range"):
        SemanticId((3, 0), (3, 3))
    with pytest.raises(ValueError, match="out of range"):
        SemanticId((0, -1), (3, 3))
    with pytest.raises(ValueError, match="nonzero length"):
        SemanticId((), ())
    with pytest.raises(ValueError, match="nonzero length"):
        SemanticId((0,), (3, 3))


def test_bulk_materialisation_matches_per_item_and_is_fast():
    """decode.materialize: the drop-in API's host conversion of one C2 batch
    (512 requests x 256 results): identical to building every SemanticId
    through the validating constructor, with the range check vectorised."""
    from paper_2602_22732_b200.decode import materialize
    rng = np.random.default_rng(0)
    B, m, T, vocab = 512, 256, 3, (256, 256, 256)
    toks = rng.integers(0, 256, size=(B * m * T,)).astype(np.int32)
    score = -rng.random(B * m)
    count = rng.integers(200, m + 1, size=B).astype(np.int32)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        out = materialize(count, toks, score, m, T, vocab)
        best = min(best, time.perf_counter() - t0)
    tt = toks.reshape(B, m, T)
    sc = score.reshape(B, m)
    for b in (0, 17, B - 1):
        want = [(SemanticId(tuple(int(x) for x in tt[b, j]), vocab), float(sc[b, j]))
                for j in range(int(count[b]))]
        assert out[b] == want
        assert all(type(s) is type(out[b][0][0]) for s, _ in out[b])
        # immutable, int/float-only: off the cyclic GC's lists (no full-
        # collection pauses over a serving cache of millions of results)
        assert not any(gc.is_tracked(p) or gc.is_tracked(p[0]) for p in out[b])
    n = int(count.sum())
    print(f"materialize: {n} results in {best * 1e3:.1f} ms")
    assert best < 1.0  # generous on a loaded CI host; the bench line reports the figure
    bad = toks.copy()
    bad[5] = 256
    with pytest.raises(ValueError, match="out of range"):
        materialize(np.full(B, m, np.int32), bad, score, m, T, vocab)


def test_context_width_and_values_validated_before_device_work():
    """a context of the wrong width (e.g. raw features) raises
    ValueError like the reference's matmul would, before any GPU call."""
    from paper_2602_22732_b200.serving import BeamSchedule, beam_search
    model = DecoderModel(DecoderConfig(3, 4, 6, 2, 1, (4, 4), 3, seed=3))
    sched = BeamSchedule((2, 2), 2)
    with pytest.raises(ValueError, match="columns"):
        beam_search(model, np.ones((2, 3)), sched)
    with pytest.raises(ValueError, match="empty"):
        beam_search(model, np.empty((0, 4)), sched)
    with pytest.raises(ValueError, match="finite"):
        beam_search(model, np.full((1, 4), np.inf), sched)


def test_load_estimator_rate_and_slack():
    """N1: the engine's own arrival-rate window and measured capacity drive
    TABS (capacity_slack = clamp(1 - rate / capacity, 0, 1))."""
    from paper_2602_22732_b200.serving.engine import LoadEstimator
    from paper_2602_22732_b200.serving.schedule import (BeamSchedule, TrafficSignal,
                                                         scale_schedule, tabs_adjust)
    est = LoadEstimator(window=1.0)
    assert est.signal(0.0) == (0.0, 1.0)  # no capacity measured yet: full slack
    for i in range(100):
        est.observe(i * 0.01)  # 100 requests/s
    assert abs(est.rate(0.995) - 100.0) < 1e-9
    est.record_service(400, 1.0)  # 400 requests per second of decode
    qps, slack = est.signal(0.995)
    assert abs(slack - 0.75) < 1e-9
    sched = BeamSchedule((64, 128, 256), 256)
    lo = scale_schedule(sched, tabs_adjust(TrafficSignal(qps, 1000.0, slack), 256, 0.6))
    # later: traffic at capacity leaves no slack -> base widths
    for i in range(400):
        est.observe(2.0 + i / 400.0)
    qps2, slack2 = est.signal(2.999)
    assert slack2 == 0.0
    hi = scale_schedule(sched, tabs_adjust(TrafficSignal(qps2, 1000.0, slack2), 256, 0.6))
    assert hi.widths == (64, 128, 256) and lo.widths[-1] > hi.widths[-1]
    assert est.rate(10.0) == 0.0  # the window slides
    # a small (latency-bound) batch does not read as a capacity drop
    est.record_service(10, 1.0)
    assert abs(est.capacity - 400.0) < 1e-9
    est.record_service(300, 0.5)  # >= half the largest batch: EWMA update
    assert abs(est.capacity - (0.8 * 400.0 + 0.2 * 600.0)) < 1e-9
    # two serving threads overlapping: the engine's rate is the batch's x 2
    cap0 = est.capacity
    est.record_service(400, 2.0, concurrency=2.0)
    assert abs(est.capacity - (0.8 * cap0 + 0.2 * 400.0)) < 1e-9


def test_lazy_sid_lists_equal_the_eager_lists():
    """decode.lazy_results / SidList (the engine's result lists): built on
    first read from copies of the result arrays, equal to materialize's
    lists in every list operation, with the batch's token range check done
    up front (the same ValueError as SemanticId)."""
    from paper_2602_22732_b200.decode import SidList, lazy_results, materialize
    rng = np.random.default_rng(3)
    B, m, T, vocab = 6, 9, 3, (7, 5, 11)
    toks = np.stack([rng.integers(0, v, size=B * m) for v in vocab], 1).astype(np.int32).ravel()
    score = -rng.random(B * m)
    count = np.array([9, 0, 3, 9, 1, 5], np.int32)
    eager = materialize(count, toks, score, m, T, vocab)
    lazy = lazy_results(count, toks.copy(), score.copy(), m, T, vocab)
    toks[:] = 0  # the lazy lists hold copies: the decoder may reuse its buffers
    for e, z in zip(eager, lazy):
        assert isinstance(z, SidList) and z._list is None
        assert len(z) == len(e) and z.scores.tolist() == [s for _, s in e]
        assert z._list is None  # len / scores never build objects
        assert z == e and e == z and list(z) == e and repr(z) == repr(e)
        if e:
            assert z[0] == e[0] and z[-1] == e[-1] and z[1:] == e[1:]
    assert lazy[0] != lazy[2] and lazy[1] == []
    bad = toks.copy()
    bad[3 * T + 2] = 11  # request 0, entry 3, level 2
    with pytest.raises(ValueError, match="out of range"):
        lazy_results(count, bad, score, m, T, vocab)
    bad[3 * T + 2] = 0
    bad[m * T + 2] = 99  # request 1 has no live entries: not checked
    lazy_results(count, bad, score, m, T, vocab)


def test_group_split_and_valid_sid_digest_cache():
    """_split_input cuts per-request blocks or concatenated rows by request;
    _valid_key caches the digest of an immutable SID tuple only."""
    from paper_2602_22732_b200.serving import beam as SB
    lens = [3, 1, 4, 2]
    rows = np.arange(10 * 2, dtype=np.float32).reshape(10, 2)
    assert SB._split_input(rows, lens, 1, 3).tolist() == rows[3:8].tolist()
    blocks = [rows[:3], rows[3:4], rows[4:8], rows[8:]]
    assert SB._split_input(blocks, lens, 2, 4) == blocks[2:]
    sids = tuple(SemanticId((i % 3, i % 2), (3, 2)) for i in range(5))
    k1 = SB._valid_key(sids)
    assert SB._VKEYS[id(sids)][1] == k1 and SB._valid_key(sids) == k1
    lst = list(sids)
    assert SB._valid_key(lst) == k1 and id(lst) not in SB._VKEYS
    lst[0] = SemanticId((2, 1), (3, 2))  # a mutable list is re-hashed every call
    assert SB._valid_key(lst) != k1


def test_engine_capacity_widths_and_item_table():
    """ServingEngine._capacity_widths bounds every TABS schedule (pooled
    decoders are planned for it); ItemTable keys valid SIDs in mixed radix
    with the min item id and resolves slot rows (CPU tensors here)."""
    from paper_2602_22732_b200.quantizer import SidIndex
    from paper_2602_22732_b200.serving.engine import ItemTable, LoadEstimator
    cfg = DecoderConfig(feat_dim=4, d=4, d_ff=6, n_layers=2, trunk_depth=1,
                        level_vocab_sizes=(3, 3), n_value_buckets=2, seed=5)
    from paper_2602_22732_b200.serving.engine import ServingConfig, ServingEngine, SnapshotStore
    from paper_2602_22732_b200.serving.schedule import (BeamSchedule, TrafficSignal,
                                                         scale_schedule, tabs_adjust)
    base = BeamSchedule((2, 5, 9), 9)
    eng = ServingEngine(SnapshotStore(DecoderModel(cfg), preload=False), SidIndex(),
                        ServingConfig(base, q_threshold=100.0, boost=0.6), load=LoadEstimator())
    cap = eng._capacity_widths()
    for qps in (0.0, 10.0, 50.0, 99.0, 100.0, 1e6):
        for slack in (0.0, 0.3, 1.0):
            w = scale_schedule(base, tabs_adjust(TrafficSignal(qps, 100.0, slack), 9, 0.6)).widths
            assert all(a <= b for a, b in zip(w, cap))
    index = SidIndex()
    index.upsert("b", SemanticId((1, 2), (3, 3)))
    index.upsert("a", SemanticId((1, 2), (3, 3)))
    index.upsert("c", SemanticId((0, 1), (3, 3)))
    index.upsert("x", SemanticId((4, 4), (5, 5)))  # another vocabulary: never decodable
    tab = ItemTable(index, (3, 3), "cpu")
    assert tab.n == 2 and tab.keys.tolist() == [0 * 3 + 1, 1 * 3 + 2]
    sids = [(SemanticId((1, 2), (3, 3)), -0.5), (SemanticId((2, 2), (3, 3)), -0.7),
            (SemanticId((0, 1), (3, 3)), -0.9)]
    assert tab.resolve(sids, np.array([1, -1, 0, 5], np.int32)) == [("a", -0.5), ("c", -0.9)]
    # the batched form equals per-request resolve (slots past a list's end ignored)
    lists = [sids, sids[:1], [], sids[::-1]]
    slots = np.array([[1, -1, 0, 5], [1, 0, 0, 0], [0, 0, 0, 0], [0, -1, 1, 1]], np.int32)
    assert tab.resolve_batch(lists, slots) == [tab.resolve(x, r) for x, r in zip(lists, slots)]
