"""The reference's own known-answer tests for this path, restated against the
CPU oracle (pkg/tests/test_beam.py:18-119, test_schedule_cache.py:40-59,
test_engine.py:76-81, verify.py:462-546)."""

import numpy as np

from oracle import beam_oracle as orc


def test_worked_example():  # test_beam.py:18-23
    got = orc.topk_precut([0.0, -1.0], np.array([[-0.1, -2.0, -3.0],
                                                  [-0.2, -0.3, -5.0]]), 2)
    assert [(b, t) for b, t, _ in got] == [(0, 0), (1, 0)]
    np.testing.assert_allclose([s for *_, s in got], [-0.1, -1.2])


def test_tie_order():  # test_beam.py:55-61
    got = orc.topk_precut([0.0, 0.0], np.array([[-1.0, -1.0], [-1.0, -1.0]]), 3)
    assert [(b, t) for b, t, _ in got] == [(0, 0), (0, 1), (1, 0)]


def test_dbs_pinned_values():  # test_schedule_cache.py:40-59, test_engine.py:76-81
    assert orc.tabs_adjust(10.0, 100.0, 1.0, 512) == 819
    assert orc.tabs_adjust(100.0, 100.0, 1.0, 512) == 512
    assert orc.tabs_adjust(1.0, 10.0, 1.0, 16) == 26
    assert orc.scale_widths((4, 8, 16), 16, 26) == (7, 13, 26)
    assert orc.scale_widths((2, 4), 4, orc.tabs_adjust(1.0, 10.0, 1.0, 4)) == (3, 6)


def _tiny(sizes, L=2, K=1, seed=3, d=4):
    return orc.OracleConfig(3, d, d + 2, L, K, tuple(sizes), 3, seed)


def test_full_width_equals_bruteforce():  # verify.py:462-486
    rng = np.random.default_rng(0)
    for j in range(8):
        cfg = _tiny((3, 3, 2), K=j % 2, seed=int(rng.integers(0, 2**31)))
        p = orc.init_params(cfg)
        x = orc.context_process(rng.normal(size=(2, 3)), p)
        got = orc.beam_search(p, cfg, x, (3, 9, 18))
        want = orc.sequence_oracle(p, cfg, x)
        assert [t for t, _ in got] == [t for t, _ in want]
        np.testing.assert_allclose([s for _, s in got], [s for _, s in want], atol=1e-9)


def test_greedy_equals_argmax_chain():  # test_beam.py:71-86
    rng = np.random.default_rng(5)
    for _ in range(5):
        cfg = _tiny((4, 3, 5), L=3, K=int(rng.integers(0, 3)),
                    seed=int(rng.integers(0, 2**31)))
        p = orc.init_params(cfg)
        x = orc.context_process(rng.normal(size=(2, 3)), p)
        (toks, _), = orc.beam_search(p, cfg, x, (1, 1, 1))
        chain = [0, 0, 0]
        for lvl in range(3):
            head, _ = orc.lazy_forward(p, cfg, x, tuple(chain), include_value_step=False)
            chain[lvl] = int(np.argmax(head[lvl]))
        assert toks == tuple(chain)


def test_lazy_cost_closed_forms():  # verify.py:526-546
    cfg = orc.OracleConfig(3, 4, 6, 9, 6, (512, 512, 512), 2, 7)
    lazy = orc.counter_closed_form(cfg, (512,) * 3, 1)[0]
    van = orc.counter_closed_form(cfg, (512,) * 3, 1, trunk_depth=0)[0]
    assert lazy == 3 * 6 + 3 * 3 * 512 and van == 3 * 9 * 512
    assert abs(van / lazy - 2.988) < 1e-3
