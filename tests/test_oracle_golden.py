"""Pin the CPU oracle (oracle/beam_oracle.py) against fixtures recorded from
the unmodified reference (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from cases import case_config, case_features
from oracle import beam_oracle as orc


def _digest(params):
    h = hashlib.sha256()
    for k, v in params.items():
        h.update(k.encode())
        h.update(np.ascontiguousarray(v, dtype=np.float64).tobytes())
    return h.hexdigest()


def test_init_matches_reference_bitwise(golden_small):
    for rec in golden_small["init"]:
        c = rec["config"]
        cfg = orc.OracleConfig(c["feat_dim"], c["d"], c["d_ff"], c["n_layers"],
                               c["trunk_depth"], tuple(c["level_vocab_sizes"]),
                               c["n_value_buckets"], c["seed"])
        assert _digest(orc.init_params(cfg)) == rec["sha256"]


def test_precut_matches_reference(golden_small):
    for rec in golden_small["precut"]:
        got = orc.topk_precut(rec["scores"], np.array(rec["logprobs"]), rec["k"])
        want = rec["expect"]
        assert [(b, t) for b, t, _ in got] == [(b, t) for b, t, _ in want]
        np.testing.assert_allclose([s for *_, s in got], [s for *_, s in want],
                                   rtol=0, atol=1e-12)
        brute = orc.precut_oracle(np.array(rec["scores"]), np.array(rec["logprobs"]),
                                  rec["k"])
        assert [(b, t) for b, t, _ in brute] == [(b, t) for b, t, _ in want]
        if "expect_global" in rec:
            b, t, s = orc.topk_global(rec["scores"], np.array(rec["logprobs"]), rec["k"])
            assert list(b) == rec["expect_global"][0]
            assert list(t) == rec["expect_global"][1]


def test_dbs_integers_match_reference(golden_small):
    for rec in golden_small["dbs"]["tabs"]:
        assert orc.tabs_adjust(rec["qps"], rec["q_threshold"], rec["slack"],
                               rec["base"], rec["boost"]) == rec["active"]
    for rec in golden_small["dbs"]["scale"]:
        w = tuple(rec["widths"])
        assert list(orc.scale_widths(w, w[-1], rec["active"])) == rec["expect"]


@pytest.mark.parametrize("idx", range(61))
def test_beam_search_matches_reference(golden_small, idx):
    cases = golden_small["beam"]
    if idx >= len(cases):
        pytest.skip("fewer cases")
    case = cases[idx]
    cfg = case_config(case)
    params = orc.init_params(cfg)
    x = orc.context_process(case_features(case), params)
    kw = {}
    if case.get("trunk_depth") is not None:
        kw["trunk_depth"] = case["trunk_depth"]
    if case.get("value_rerank"):
        kw.update(value_rerank=True, representatives=case["representatives"])
    got = orc.beam_search(params, cfg, x, case["widths"], **kw)
    assert [list(t) for t, _ in got] == case["tokens"], case["name"]
    np.testing.assert_allclose([s for _, s in got], case["scores"], rtol=1e-10,
                               atol=1e-12)
    s_ctx = x.shape[0]
    for shared, key in ((True, "counter"), (False, "counter_unshared")):
        cf = orc.counter_closed_form(cfg, case["widths"], s_ctx, shared_kv=shared,
                                     value_rerank=bool(case.get("value_rerank")),
                                     trunk_depth=case.get("trunk_depth"))
        assert list(cf) == case[key], (case["name"], key)


def test_teacher_forced_logits_match_reference(golden_small):
    for rec in golden_small["teacher_forced"]:
        c = rec["config"]
        cfg = orc.OracleConfig(c["feat_dim"], c["d"], c["d_ff"], c["n_layers"],
                               c["trunk_depth"], tuple(c["level_vocab_sizes"]),
                               c["n_value_buckets"], c["seed"])
        params = orc.init_params(cfg)
        x = orc.context_process(np.array(rec["features"]), params)
        head, value = orc.lazy_forward(params, cfg, x, rec["tokens"])
        for a, b in zip(head, rec["head_logits"]):
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(value, rec["value_logits"], rtol=1e-12, atol=1e-13)


def test_c3_request_matches_reference(golden_c3):
    """The full C3 shape (d=1024, L=8, K=5, V=4096^3, widths 512^3)."""
    c = golden_c3["config"]
    cfg = orc.OracleConfig(c["feat_dim"], c["d"], c["d_ff"], c["n_layers"],
                           c["trunk_depth"], tuple(c["level_vocab_sizes"]),
                           c["n_value_buckets"], c["seed"])
    params = orc.init_params(cfg)
    assert _digest(params) == golden_c3["init_sha256"]
    feats = np.random.default_rng(1000 + golden_c3["request"]).normal(
        size=(golden_c3["s_ctx"], 16))
    got = orc.beam_search(params, cfg, orc.context_process(feats, params),
                          golden_c3["widths"])
    assert [list(t) for t, _ in got] == golden_c3["tokens"]
    np.testing.assert_allclose([s for _, s in got], golden_c3["scores"], rtol=1e-10)
