"""Teacher-forced candidate scoring on the GPU against the
reference's recorded lazy_forward logits and the oracle restatement."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import beam_oracle as orc  # noqa: E402


def _pkg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_22732_b200 import model as M
    from paper_2602_22732_b200.decode import score_sequences
    return M, score_sequences


def _model(M, c):
    cfg = M.DecoderConfig(c["feat_dim"], c["d"], c["d_ff"], c["n_layers"], c["trunk_depth"],
                          tuple(c["level_vocab_sizes"]), c["n_value_buckets"], c["seed"])
    return M.DecoderModel(cfg)


def test_lazy_forward_matches_reference_golden(golden_small):
    M, _ = _pkg()
    for rec in golden_small["teacher_forced"]:
        model = _model(M, rec["config"])
        x = M.context_process(np.array(rec["features"]), model.params)
        trace = M.lazy_forward(model, x, rec["tokens"])
        for a, b in zip(trace.head_logits, rec["head_logits"]):
            np.testing.assert_allclose(a.data, b, rtol=2e-5, atol=2e-5)
        np.testing.assert_allclose(trace.value_logits.data, rec["value_logits"], rtol=2e-5,
                                   atol=2e-5)
        lp = M.sequence_log_prob(trace, rec["tokens"])
        want = orc.sequence_log_prob([np.array(h) for h in rec["head_logits"]], rec["tokens"])
        assert abs(lp - want) <= 1e-4 * max(1.0, abs(want))


@pytest.mark.parametrize("path,d", [("layered", 16), ("tensor", 64), ("auto", 64)])
def test_batched_scoring_matches_oracle(path, d):
    """Beam outputs re-scored by teacher forcing equal their beam scores
    (build_rl_log / sequence_oracle usage, loop.py:99-107, verify.py:448-459)."""
    M, score_sequences = _pkg()
    ocfg = orc.OracleConfig(8, d, 2 * d, 3, 1, (32, 16, 64), 4, 13)
    model = M.DecoderModel(M.DecoderConfig(ocfg.feat_dim, ocfg.d, ocfg.d_ff, ocfg.n_layers,
                                           ocfg.trunk_depth, ocfg.level_vocab_sizes,
                                           ocfg.n_value_buckets, ocfg.seed))
    params = {k: v.data for k, v in model.params.items()}
    rng = np.random.default_rng(2)
    feats = [rng.normal(size=(int(rng.integers(1, 70)), 8)) for _ in range(5)]
    reqs, toks, want = [], [], []
    for b, f in enumerate(feats):
        x = orc.context_process(f, params)
        for t, s in orc.beam_search(params, ocfg, x, (4, 8, 6)):
            reqs.append(b)
            toks.append(t)
            want.append(s)
    logp, vl = score_sequences(model, reqs, toks, features=feats, include_value_step=True,
                               path=path)
    got = logp.sum(1)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5)
    # value logits vs the oracle's teacher-forced pass
    for i in (0, len(reqs) - 1):
        x = orc.context_process(feats[reqs[i]], params)
        _, v = orc.lazy_forward(params, ocfg, x, toks[i])
        np.testing.assert_allclose(vl[i], v, rtol=1e-4, atol=1e-5)


def test_scoring_rejects_bad_tokens():
    M, score_sequences = _pkg()
    model = M.DecoderModel(M.DecoderConfig(4, 16, 32, 2, 1, (8, 8), 2, 0))
    with pytest.raises(ValueError):
        score_sequences(model, [0], [[3, 9]], features=[np.ones((2, 4))])
