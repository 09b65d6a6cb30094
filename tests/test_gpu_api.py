"""GPU checks of the drop-in API surface beyond the decode itself: the
per-level C entry points, the exact float64 selection API, the fused
projection + top-k entry, the shared encoder K/V handle, the reference's
beam-search properties (test_beam.py, verify.py ACCEPTANCE 05 / 08) run on
the GPU, the pooled decoder / CUDA-graph path, the fp16-range fallback,
and on-device SID -> item resolution in the engine."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from cases import C1_MODEL, C2_WIDTHS, c_features, list_parity  # noqa: E402
from oracle import beam_oracle as orc  # noqa: E402

REL_TOL = 1e-3


def _need():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_22732_b200 import model as M
    from paper_2602_22732_b200 import serving as S
    return M, S


def _model(M, ocfg):
    return M.DecoderModel(M.DecoderConfig(ocfg.feat_dim, ocfg.d, ocfg.d_ff, ocfg.n_layers,
                                          ocfg.trunk_depth, tuple(ocfg.level_vocab_sizes),
                                          ocfg.n_value_buckets, ocfg.seed))


def _parity(ref, got, label):
    got = [(tuple(getattr(s, "tokens", s)), v) for s, v in got]
    assert len(got) == len(ref), label
    rmap = dict((tuple(t), s) for t, s in ref)
    err = 0.0
    for t, s in got:
        if t in rmap:
            err = max(err, abs(s - rmap[t]))
            assert abs(s - rmap[t]) <= REL_TOL * abs(rmap[t]) + 1e-12, label
    ulp = max(abs(s) for _, s in ref) * 2.0 ** -23 if ref else 0.0
    ok, msg = list_parity([(tuple(t), s) for t, s in ref], got, max(4 * err, 8 * ulp))
    assert ok, f"{label}: {msg}"


def random_decoder(rng, M, max_d=8, max_layers=3, max_levels=4, feat_dim=3):
    """verify.py:83-94 (same draws)."""
    d = int(rng.choice([4, 6, max_d]))
    n_layers = int(rng.integers(2, max_layers + 1))
    trunk_depth = int(rng.integers(0, n_layers))
    n_levels = int(rng.integers(2, max_levels + 1))
    sizes = tuple(int(rng.integers(2, 6)) for _ in range(n_levels))
    cfg = M.DecoderConfig(feat_dim, d, d + 2, n_layers, trunk_depth, sizes,
                          int(rng.integers(1, 5)), int(rng.integers(0, 2**31)))
    return M.DecoderModel(cfg)


def _oracle_of(model):
    c = model.config
    return (orc.OracleConfig(c.feat_dim, c.d, c.d_ff, c.n_layers, c.trunk_depth,
                             tuple(c.level_vocab_sizes), c.n_value_buckets, c.seed),
            {k: v.data for k, v in model.params.items()})


@pytest.mark.parametrize("d,path", [(64, "tensor"), (128, "tensor"), (128, "tensor_ctx"),
                                    (16, "layered")])
@pytest.mark.parametrize("rerank", [False, True])
def test_per_level_entry_points_equal_whole_decode(d, path, rerank):
    """gr4ad_encode_trunk + gr4ad_level_step(t) + gr4ad_collect (SURVEY
    §8b(1)) reproduce gr4ad_beam_search_run bit for bit."""
    M, S = _need()
    from paper_2602_22732_b200 import _native as N
    from paper_2602_22732_b200.decode import BeamDecoder
    from paper_2602_22732_b200.device import _stream_handle
    model = _model(M, orc.OracleConfig(16, d, 2 * d, 3, 1, (64, 32, 128), 4, 5))
    feats = np.concatenate([c_features(i, 96) for i in range(6)], 0).astype(np.float32)
    f = torch.from_numpy(feats).cuda()
    reps = np.array([0.4, 1.0, 1.8, 2.5])
    widths = [(4, 16, 40)] * 6
    a = BeamDecoder(model, [96] * 6, widths, path=path, value_rerank=rerank,
                    representatives=reps)
    a.run(features=f)
    want = [t.clone() for t in (a.count, a.tokens, a.score)]
    b = BeamDecoder(model, [96] * 6, widths, path=path, value_rerank=rerank,
                    representatives=reps)
    st = _stream_handle()
    ws = C.c_void_p(b.workspace.data_ptr())
    N.check(N.lib.gr4ad_encode_trunk(C.byref(b.dims), C.byref(b.weights.struct),
                                     C.byref(b.batch), C.c_void_p(f.data_ptr()), None, ws,
                                     b.workspace_bytes, st))
    for t in range(3 + (1 if rerank else 0)):
        N.check(N.lib.gr4ad_level_step(C.byref(b.dims), C.byref(b.weights.struct),
                                       C.byref(b.batch), t, ws, b.workspace_bytes, st))
    N.check(N.lib.gr4ad_collect(C.byref(b.dims), C.byref(b.batch), C.byref(b.results_struct),
                                ws, b.workspace_bytes, st))
    for x, y in zip(want, (b.count, b.tokens, b.score)):
        assert torch.equal(x, y)
    with pytest.raises(ValueError):
        N.check(N.lib.gr4ad_level_step(C.byref(b.dims), C.byref(b.weights.struct),
                                       C.byref(b.batch), 7, ws, b.workspace_bytes, st))


def test_per_level_entry_points_reject_the_fused_kernel():
    M, S = _need()
    from paper_2602_22732_b200 import _native as N
    from paper_2602_22732_b200.decode import BeamDecoder
    from paper_2602_22732_b200.device import _stream_handle
    dec = BeamDecoder(_model(M, C1_MODEL), [256], [C2_WIDTHS], path="fused")
    with pytest.raises(RuntimeError, match="layered"):
        N.check(N.lib.gr4ad_level_step(C.byref(dec.dims), C.byref(dec.weights.struct),
                                       C.byref(dec.batch), 0,
                                       C.c_void_p(dec.workspace.data_ptr()),
                                       dec.workspace_bytes, _stream_handle()))


def test_golden_precut_is_bit_exact(golden_small):
    """topk_precut / topk_global rank the reference's float64 sums with no
    rounding (gr4ad_topk_precut_f64): every recorded instance identical,
    order and scores."""
    M, S = _need()
    for rec in golden_small["precut"]:
        got = S.topk_precut([((), s) for s in rec["scores"]], np.array(rec["logprobs"]),
                            rec["k"])
        assert [tuple(g) for g in got] == [tuple(w) for w in rec["expect"]]
        if "expect_global" in rec:
            b, t, s = S.topk_global(rec["scores"], np.array(rec["logprobs"]), rec["k"])
            assert [b.tolist(), t.tolist(), s.tolist()] == rec["expect_global"]


def test_precut_f64_large_and_tied():
    """Exact against the oracle's lexsort on larger problems with exact ties,
    -inf rows and k beyond one row."""
    M, S = _need()
    rng = np.random.default_rng(3)
    for b, v, k in ((64, 4096, 512), (7, 300, 2000), (3, 5, 15)):
        prev = rng.normal(size=b)
        lp = np.round(rng.normal(size=(b, v)), 1)  # many exact ties
        prev[-1] = -np.inf
        want = orc.topk_global(prev, lp, k)
        got = S.topk_global(prev, lp, k)
        for w, g in zip(want, got):
            np.testing.assert_array_equal(np.asarray(w), np.asarray(g))


def test_project_topk_entry():
    """gr4ad_project_topk (beam.py:198-201 as one fused call): logits GEMM,
    log-softmax, score accumulation and top-k vs float64 numpy."""
    _need()
    from paper_2602_22732_b200 import _native as N
    rng = np.random.default_rng(4)
    P, b, v, d, k = 3, 16, 512, 64, 40
    states = rng.normal(size=(P * b, d)).astype(np.float32)
    head = (rng.normal(size=(d, v)) / 8).astype(np.float32)
    prev = rng.normal(size=P * b).astype(np.float32)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ts, th, tp = dev(states), dev(head), dev(prev)
    ob = torch.empty(P * k, dtype=torch.int32, device="cuda")
    ot = torch.empty_like(ob)
    osc = torch.empty(P * k, dtype=torch.float32, device="cuda")
    oc = torch.empty(P, dtype=torch.int32, device="cuda")
    nws = N.lib.gr4ad_project_topk_workspace_bytes(P, b, v)
    ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
    p = lambda t: C.c_void_p(t.data_ptr())
    N.check(N.lib.gr4ad_project_topk(p(ts), p(th), d, p(tp), P, b, v, k, p(ob), p(ot), p(osc),
                                     p(oc), p(ws), nws, C.c_void_p(0)))
    torch.cuda.synchronize()
    logits = states.astype(np.float64) @ head.astype(np.float64)
    logp = orc.log_softmax_rows(logits)
    for q in range(P):
        total = prev[q * b:(q + 1) * b, None].astype(np.float64) + logp[q * b:(q + 1) * b]
        wb, wt, ws_ = orc.topk_global(prev[q * b:(q + 1) * b].astype(np.float64),
                                      logp[q * b:(q + 1) * b], k)
        gb = ob[q * k:(q + 1) * k].cpu().numpy()
        gt = ot[q * k:(q + 1) * k].cpu().numpy()
        gs = osc[q * k:(q + 1) * k].cpu().numpy()
        assert int(oc[q]) == k
        np.testing.assert_allclose(gs, total[gb, gt], rtol=1e-5, atol=1e-5)
        ref = [((int(x), int(y)), float(s)) for x, y, s in zip(wb, wt, ws_)]
        got = [((int(x), int(y)), float(s)) for x, y, s in zip(gb, gt, gs)]
        ok, msg = list_parity(ref, got, 1e-4)
        assert ok, msg


def test_shared_encoder_kv_handle():
    """beam.py:98-109 (reference test_beam.py:194-206): per head layer
    (X Wk, X Wv), and every layer with trunk_depth=0."""
    M, S = _need()
    model = _model(M, orc.OracleConfig(3, 64, 128, 3, 1, (4, 4), 3, 59))
    x = np.random.default_rng(1).normal(size=(3, 64))
    handle = S.shared_encoder_kv(model, x)
    assert set(handle) == {1, 2}
    for i, (ck, cv) in handle.items():
        np.testing.assert_allclose(ck, x @ model.params[f"layer{i}.cross.Wk"].data,
                                   rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(cv, x @ model.params[f"layer{i}.cross.Wv"].data,
                                   rtol=1e-4, atol=1e-5)
    assert set(S.shared_encoder_kv(model, x, trunk_depth=0)) == {0, 1, 2}


def test_greedy_equals_argmax_chain():
    """test_beam.py:71-86 on the GPU: width-1 beams equal the per-level
    argmax of teacher-forced (GPU lazy_forward) logits."""
    M, S = _need()
    rng = np.random.default_rng(5)
    for _ in range(10):
        model = random_decoder(rng, M)
        feats = rng.normal(size=(int(rng.integers(1, 3)), model.config.feat_dim))
        x = M.context_process(feats, model.params)
        sizes = model.config.level_vocab_sizes
        (sid, _), = S.beam_search(model, x, S.BeamSchedule((1,) * len(sizes), 1))
        tokens = [0] * len(sizes)
        for level in range(len(sizes)):
            trace = M.lazy_forward(model, x, tuple(tokens), include_value_step=False)
            tokens[level] = int(np.argmax(trace.head_logits[level].data))
        assert sid.tokens == tuple(tokens)


def test_schedule_dominance():
    """test_beam.py:112-119: a wider schedule never finds a worse best."""
    M, S = _need()
    rng = np.random.default_rng(8)
    for _ in range(10):
        model = M.DecoderModel(M.DecoderConfig(3, 4, 6, 2, 1, (4, 4), 3,
                                               int(rng.integers(0, 1000))))
        x = M.context_process(rng.normal(size=(int(rng.integers(1, 3)), 3)), model.params)
        small = S.beam_search(model, x, S.BeamSchedule((1, 2), 2))
        large = S.beam_search(model, x, S.BeamSchedule((2, 4), 4))
        assert large[0][1] >= small[0][1] - 1e-6


def test_flag_invariance_200_models():
    """ACCEPTANCE 05 (verify.py:400-433) on the GPU: the four {shared_kv,
    precut} combinations return identical lists on 200 random models, one
    KV build per request with shared_kv, and every list passes the §8c rule
    against the oracle."""
    M, S = _need()
    rng = np.random.default_rng(0)
    for idx in range(200):
        model = random_decoder(rng, M, max_levels=3)
        feats = rng.normal(size=(int(rng.integers(1, 3)), model.config.feat_dim))
        x = M.context_process(feats, model.params)
        widths, w, reach = [], 1, 1
        for vocab in model.config.level_vocab_sizes:
            reach = min(reach * vocab, 64)
            w = min(max(w, int(rng.integers(1, 5))), 8, reach)
            widths.append(w)
        sched = S.BeamSchedule(tuple(widths), widths[-1])
        outs = []
        for shared in (False, True):
            for precut in (False, True):
                counter = M.LayerCallCounter()
                outs.append(S.beam_search(model, x, sched, shared_kv=shared, precut=precut,
                                          counter=counter))
                if shared:
                    assert counter.kv_builds == 1
        for o in outs[1:]:
            assert [s.tokens for s, _ in o] == [s.tokens for s, _ in outs[0]]
            assert [v for _, v in o] == [v for _, v in outs[0]]
        ocfg, params = _oracle_of(model)
        want = orc.beam_search(params, ocfg, orc.context_process(feats, params), widths)
        _parity(want, outs[0], f"model {idx}")


def test_exhaustive_sandwich_100_models():
    """ACCEPTANCE 08 (verify.py:462-486) on the GPU: full-width beam search
    on a (3, 3, 2) vocabulary equals the brute-force ranking of all 18
    sequences (oracle teacher-forced log-probabilities), §8c rule."""
    M, S = _need()
    rng = np.random.default_rng(0)
    for idx in range(100):
        cfg = M.DecoderConfig(3, 4, 6, 2, int(rng.integers(0, 2)), (3, 3, 2), 2,
                              int(rng.integers(0, 2**31)))
        model = M.DecoderModel(cfg)
        feats = rng.normal(size=(int(rng.integers(1, 3)), 3))
        x = M.context_process(feats, model.params)
        got = S.beam_search(model, x, S.BeamSchedule((3, 9, 18), 18))
        ocfg, params = _oracle_of(model)
        want = orc.sequence_oracle(params, ocfg, orc.context_process(feats, params))
        assert len(got) == 18
        _parity(want, got, f"sandwich {idx}")


def test_pooled_decoder_and_graph_replay():
    """Repeated beam_search_batch calls of one shape reuse a pooled decoder
    and, from the second call on, replay its CUDA graph -- same results as
    a fresh decode, for new inputs each call."""
    M, S = _need()
    from paper_2602_22732_b200.decode import POOL
    model = _model(M, C1_MODEL)
    POOL.clear()
    sched = S.BeamSchedule(C2_WIDTHS, 256)
    outs = []
    for rep in range(3):
        feats = [c_features(10 * rep + i, 256) for i in range(8)]
        outs.append((feats, S.beam_search_batch(model, features=feats, schedules=sched)))
    assert len(POOL) == 1
    dec = next(iter(POOL._idle.values()))[0]
    assert dec.graph is not None and dec.uses == 3
    ocfg, params = _oracle_of(model)
    for feats, got in outs:
        for i in (0, 7):
            want = orc.beam_search(params, ocfg, orc.context_process(feats[i], params),
                                   C2_WIDTHS)
            _parity(want, got[i], "pooled")


@pytest.mark.parametrize("d,path", [(128, "tensor"), (16, "fused")])
def test_decoders_share_the_snapshots_derived_weights(d, path):
    """Decoders of different batch shapes / widths of one snapshot share a
    single prepared copy of the derived weights (gr4ad_derived_layout /
    batch->derived): the second decoder prepares nothing, its workspace
    excludes the region, and both decode like the oracle; a republished
    snapshot gets its own copy."""
    M, S = _need()
    from paper_2602_22732_b200.decode import BeamDecoder
    F = 16
    model = M.DecoderModel(M.DecoderConfig(F, d, 2 * d, 3, 2, (256, 256, 256), 4, seed=5))
    shapes = [([256] * 3, [(8, 16, 32)] * 3), ([256] * 5, [(16, 32, 64)] * 4 + [(4, 8, 16)])]
    decs = [BeamDecoder(model, lens, widths, path=path) for lens, widths in shapes]
    assert decs[0]._derived.data_ptr() == decs[1]._derived.data_ptr()
    ocfg, params = _oracle_of(model)
    for (lens, widths), dec in zip(shapes, decs):
        feats = [c_features(100 + i, lens[i]) for i in range(len(lens))]
        x = torch.from_numpy(np.concatenate(feats).astype(np.float32)).cuda()
        dec.run(features=x)
        got = dec.host_results()
        for i in range(len(lens)):
            want = orc.beam_search(params, ocfg, orc.context_process(feats[i], params), widths[i])
            _parity(want, got[i], f"derived {path} shape {len(lens)} request {i}")
    other = model.clone()
    dec2 = BeamDecoder(other, *shapes[0], path=path)
    assert dec2._derived.data_ptr() != decs[0]._derived.data_ptr()


def test_rebind_drops_the_host_graph():
    """after a hot swap, replay_host must not run the previous
    snapshot's graph."""
    M, S = _need()
    from paper_2602_22732_b200.decode import BeamDecoder
    model = _model(M, C1_MODEL)
    host = torch.from_numpy(c_features(0, 256).astype(np.float32)).pin_memory()
    dec = BeamDecoder(model, [256], [C2_WIDTHS])
    dec.capture_host(host)
    dec.rebind(model.clone())
    with pytest.raises(RuntimeError, match="capture_host"):
        dec.replay_host()


def test_resident_weights_are_read_only_until_invalidated():
    """an in-place edit of a resident snapshot raises instead of
    silently decoding with stale GPU weights; invalidate() re-uploads."""
    M, S = _need()
    from paper_2602_22732_b200.device import invalidate
    model = _model(M, C1_MODEL)
    feats = [c_features(0, 256)]
    sched = S.BeamSchedule((8, 16, 32), 32)
    a = S.beam_search_batch(model, features=feats, schedules=sched)
    with pytest.raises(ValueError):
        model.params["head.0"].data[:] = 0.0
    invalidate(model)
    model.params["head.0"].data[:] = 0.0
    b = S.beam_search_batch(model, features=feats, schedules=sched)
    ocfg, params = _oracle_of(model)
    want = orc.beam_search(params, ocfg, orc.context_process(feats[0], params), (8, 16, 32))
    _parity(want, b[0], "after invalidate")


@pytest.mark.parametrize("path", ["auto"])
def test_fp16_range_falls_back_to_cuda_cores(path):
    """with path="auto" a batch outside the fp16 split range is
    decoded on the CUDA-core path instead of failing (large features and
    large weights), matching the oracle."""
    M, S = _need()
    for scale_w in (False, True):
        model = _model(M, orc.OracleConfig(16, 64, 128, 3, 1, (32, 32, 32), 4, 7))
        if scale_w:
            model.params["layer2.ffn.W1"].data[0, 0] = 40.0  # |w| >= 32
        feats = [c_features(0, 64) * (1.0 if scale_w else 1e4)]
        got = S.beam_search_batch(model, features=feats, schedules=[(4, 8, 16)], path=path)
        ocfg, params = _oracle_of(model)
        want = orc.beam_search(params, ocfg, orc.context_process(feats[0], params), (4, 8, 16))
        _parity(want, got[0], f"range fallback w={scale_w}")


def test_engine_resolves_items_on_device_and_measures_load():
    """f2 + N1: the engine resolves SIDs to items on the device (unindexed
    SIDs dropped, min item id per SID, as engine.py:114-118) and, without an
    explicit qps, sets per-request TABS widths from its own load estimate."""
    M, S = _need()
    from paper_2602_22732_b200.quantizer import SemanticId, SidIndex
    model = _model(M, C1_MODEL)
    store = S.SnapshotStore(model)
    index = SidIndex()
    feats = c_features(0, 256)
    full = S.beam_search_batch(model, features=[feats], schedules=S.BeamSchedule(C2_WIDTHS, 256))
    sids = [sid for sid, _ in full[0]]
    for n, sid in enumerate(sids[::3]):
        index.upsert(f"item{n:04d}", SemanticId(sid.tokens, sid.level_vocab_sizes))
        index.upsert(f"alt{n:04d}", SemanticId(sid.tokens, sid.level_vocab_sizes))
    cfg = S.ServingConfig(S.BeamSchedule(C2_WIDTHS, 256), q_threshold=1e9)
    eng = S.ServingEngine(store, index, cfg)
    res = eng.serve_batch([("u0", feats)], now=0.0, qps=1.0, capacity_slack=0.0)[0]
    want = []
    for sid, score in res.sids:
        ids = index.lookup(sid)
        if ids:
            want.append((min(ids), float(score)))
    assert res.items == want and len(want) == len(sids[::3])
    # measured load (capacity pinned for the test): quiet traffic earns wider
    # beams than a saturated burst, per request inside one batch
    from paper_2602_22732_b200.serving.engine import LoadEstimator

    class Fixed(LoadEstimator):
        def record_service(self, *args, **kwargs):
            pass

    est = Fixed(window=1.0)
    est.capacity = 100.0
    cfg_req = S.ServingConfig(S.BeamSchedule(C2_WIDTHS, 256), q_threshold=1e9,
                              load_widths="request")
    eng2 = S.ServingEngine(store, index, cfg_req, load=est)
    quiet = eng2.serve_batch([(f"q{i}", c_features(i, 256), i * 0.5) for i in range(2)],
                             now=0.5)
    burst = eng2.serve_batch([(f"b{i}", c_features(i % 8, 256), 2.0 + i * 1e-4)
                              for i in range(100)], now=2.01)
    assert quiet[1].widths[-1] > 256
    assert burst[-1].widths == (64, 128, 256)
    assert burst[0].widths[-1] > burst[-1].widths[-1]  # per-request widths, one batch
    assert all(len(r.sids) == r.widths[-1] for r in quiet + burst)
    # default: one load reading per batch (the reference's per-tick signal),
    # misses padded to a batch bucket (13 -> 16) with the padding dropped
    est3 = Fixed(window=1.0)
    est3.capacity = 100.0
    eng3 = S.ServingEngine(store, index, cfg, load=est3)
    tick = eng3.serve_batch([(f"t{i}", c_features(i % 8, 256), 3.0 + i * 1e-4)
                             for i in range(13)], now=3.01)
    assert len(tick) == 13 and len({r.widths for r in tick}) == 1
    assert tick[0].widths[-1] > 256  # 13 req/s against a capacity of 100
    ocfg, params = _oracle_of(model)
    want = orc.beam_search(params, ocfg, orc.context_process(c_features(12 % 8, 256), params),
                           tick[12].widths)
    _parity(want, tick[12].sids, "bucket-padded engine batch")


@pytest.mark.parametrize("d,path", [(128, "tensor"), (16, "fused")])
def test_set_widths_replans_inside_one_decoder(d, path):
    """A decoder planned for the widest TABS schedule re-plans in place for
    narrower widths (BeamDecoder.set_widths: one table upload, no new
    buffers); graphs are parked per plan and replayed when a plan returns.
    Every plan decodes like a decoder built for it, and like the oracle."""
    M, S = _need()
    from paper_2602_22732_b200.decode import BeamDecoder
    model = M.DecoderModel(M.DecoderConfig(16, d, 2 * d, 3, 1, (256, 256, 256), 4, seed=9))
    lens = [256] * 4
    cap = [(20, 40, 80)] * 4
    plans = [[(12, 24, 48)] * 4, [(16, 32, 64), (20, 40, 80), (8, 16, 32), (13, 26, 51)],
             cap, [(12, 24, 48)] * 4]
    feats = [c_features(200 + i, 256) for i in range(4)]
    x = torch.from_numpy(np.concatenate(feats).astype(np.float32)).cuda()
    dec = BeamDecoder(model, lens, cap, path=path)
    ws = dec.workspace.data_ptr()
    ocfg, params = _oracle_of(model)
    for k, widths in enumerate(plans):
        assert dec.set_widths(widths)
        assert dec.workspace.data_ptr() == ws
        if dec.graph is None:
            dec.capture(features=x)
        else:
            assert k == 3  # the first plan's graph, parked and replayed
        dec.replay()
        got = dec.host_results()
        fresh = BeamDecoder(model, lens, widths, path=path)
        fresh.run(features=x)
        assert got == fresh.host_results(), f"plan {k}"
        for i in (0, 3):
            want = orc.beam_search(params, ocfg, orc.context_process(feats[i], params),
                                   widths[i])
            _parity(want, got[i], f"set_widths {path} plan {k} request {i}")
    assert not dec.set_widths([(40, 80, 160)] * 4)  # larger than the buffers


def test_engine_pools_one_decoder_per_batch_bucket():
    """ServingEngine: TABS widths change with load, but decoders are pooled
    per batch bucket at the widest schedule and re-planned, so a sweep of
    loads builds one decoder per bucket; results stay the oracle's."""
    M, S = _need()
    from paper_2602_22732_b200.decode import POOL
    from paper_2602_22732_b200.quantizer import SidIndex
    model = _model(M, C1_MODEL)
    POOL.clear()
    cfg = S.ServingConfig(S.BeamSchedule(C2_WIDTHS, 256), q_threshold=100.0)
    eng = S.ServingEngine(S.SnapshotStore(model), SidIndex(), cfg)
    ocfg, params = _oracle_of(model)
    seen = set()
    for step, qps in enumerate([0.0, 30.0, 60.0, 90.0, 200.0, 30.0]):
        reqs = [(f"s{step}u{i}", c_features(step * 8 + i, 256)) for i in range(5)]
        res = eng.serve_batch(reqs, now=float(step), qps=qps, capacity_slack=1 - qps / 100.0
                              if qps < 100 else 0.0)
        seen.add(res[0].widths)
        want = orc.beam_search(params, ocfg, orc.context_process(reqs[4][1], params),
                               res[4].widths)
        _parity(want, res[4].sids, f"engine qps {qps}")
        # the engine's lazily built SID lists equal the eager API's lists
        eager = S.beam_search_batch(model, features=[reqs[4][1]], schedules=[res[4].widths])[0]
        assert res[4].sids == eager and len(res[4].sids) == len(eager)
        assert list(res[4].sids)[:3] == eager[:3] and res[4].sids[-1] == eager[-1]
    assert len(seen) >= 4
    assert len(POOL) >= 1  # 5 misses -> bucket 8, one capacity decoder (+ the eager calls')


def test_non_finite_and_out_of_range_features_raise():
    """beam_search_batch: a NaN / inf feature raises the reference's
    ValueError (checked on the staged fp32 copy); a finite value beyond the
    fp32 range raises InputRangeError; the pooled decoder stays usable."""
    M, S = _need()
    from paper_2602_22732_b200.decode import InputRangeError
    model = _model(M, C1_MODEL)
    sched = S.BeamSchedule(C2_WIDTHS, 256)
    good = [c_features(i, 256) for i in range(3)]
    ref = S.beam_search_batch(model, features=good, schedules=sched)
    bad = [a.copy() for a in good]
    bad[1][5, 2] = np.nan
    with pytest.raises(ValueError, match="finite"):
        S.beam_search_batch(model, features=bad, schedules=sched)
    big = [a.copy() for a in good]
    big[2][0, 0] = 1e300
    with pytest.raises(InputRangeError):
        S.beam_search_batch(model, features=big, schedules=sched)
    assert S.beam_search_batch(model, features=good, schedules=sched) == ref


@pytest.mark.parametrize("d", [16, 128])
def test_pipelined_groups_equal_one_batch(d):
    """beam_search_batch(pipeline=k): the batch decoded as k request groups
    back to back on one stream (host staging / result building overlapping
    the device work) gives exactly the one-batch results -- the kernels are
    per row and per request, so a request decodes identically in any batch."""
    M, S = _need()
    model = M.DecoderModel(M.DecoderConfig(16, d, 2 * d, 3, 1, (64, 32, 128), 4, seed=11))
    feats = [c_features(300 + i, 64 + 16 * (i % 3)) for i in range(7)]
    scheds = [(8, 16, 32), (4, 8, 16)] * 3 + [(8, 16, 32)]
    one = S.beam_search_batch(model, features=feats, schedules=scheds, pipeline=1)
    for k in (2, 3, 7):
        assert S.beam_search_batch(model, features=feats, schedules=scheds, pipeline=k) == one


@pytest.mark.parametrize("d,path", [(128, "tensor"), (16, "auto"), (16, "layered")])
def test_set_widths_with_masking_and_rerank(d, path):
    """Re-planned decoders keep the valid-SID prefix tables and the value
    re-rank head: every plan equals a decoder built for it."""
    M, S = _need()
    from paper_2602_22732_b200.decode import BeamDecoder
    model = M.DecoderModel(M.DecoderConfig(16, d, 2 * d, 3, 1, (64, 32, 128), 4, seed=13))
    rng = np.random.default_rng(5)
    valid = [tuple(int(rng.integers(0, v)) for v in (64, 32, 128)) for _ in range(400)]
    reps = [0.1, 0.4, 0.9, 2.0]
    lens = [96, 128, 64]
    feats = [c_features(400 + i, n) for i, n in enumerate(lens)]
    x = torch.from_numpy(np.concatenate(feats).astype(np.float32)).cuda()
    cap = [(24, 48, 96)] * 3
    dec = BeamDecoder(model, lens, cap, value_rerank=True, representatives=reps,
                      valid_sids=valid, path=path)
    for widths in ([(8, 16, 32)] * 3, [(24, 48, 96), (5, 9, 17), (12, 30, 60)], cap):
        assert dec.set_widths(widths)
        dec.run(features=x)
        got = dec.host_results()
        fresh = BeamDecoder(model, lens, widths, value_rerank=True, representatives=reps,
                            valid_sids=valid, path=path)
        fresh.run(features=x)
        assert got == fresh.host_results(), widths


def test_engine_masked_warmup_and_concurrent_callers():
    """ServingEngine with valid-SID masking: warm-up builds the masked
    decoders (the SID tuple's digest is part of their key), every served SID
    is a prefix-valid one, and two threads calling serve_batch at once get
    exactly the results of one-at-a-time calls."""
    import threading
    M, S = _need()
    from paper_2602_22732_b200.decode import POOL
    from paper_2602_22732_b200.quantizer import SemanticId, SidIndex
    model = _model(M, C1_MODEL)
    rng = np.random.default_rng(21)
    index = SidIndex()
    V = tuple(model.config.level_vocab_sizes)
    for i in range(3000):
        index.upsert(f"it{i}", SemanticId(tuple(int(rng.integers(0, v)) for v in V), V))
    cfg = S.ServingConfig(S.BeamSchedule(C2_WIDTHS, 256), q_threshold=1e9, mask_to_index=True)
    POOL.clear()
    eng = S.ServingEngine(S.SnapshotStore(model), index, cfg)
    eng.warmup(c_features(0, 256), max_batch=8)
    built = len(POOL)
    valid = set(index.all_sids())
    reqs = [[(f"w{k}u{i}", c_features(50 + 8 * k + i, 256)) for i in range(6)] for k in range(2)]
    seq = [eng.serve_batch(r, now=float(k), qps=1.0, capacity_slack=0.5)
           for k, r in enumerate(reqs)]
    assert len(POOL) == built  # served from the warmed decoders
    for res in seq:
        for r in res:
            assert all(sid in valid for sid, _ in r.sids)
            assert [i for i, _ in r.items] and len(r.items) == len(r.sids)
    eng2 = S.ServingEngine(S.SnapshotStore(model), index, cfg)
    out = [None, None]

    def call(k):
        out[k] = eng2.serve_batch(reqs[k], now=float(k), qps=1.0, capacity_slack=0.5)

    ts = [threading.Thread(target=call, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in range(2):
        assert [(r.items, list(r.sids)) for r in out[k]] == \
            [(r.items, list(r.sids)) for r in seq[k]]
