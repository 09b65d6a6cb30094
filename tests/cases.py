"""Case builders shared by the CPU oracle tests and the GPU parity tests.

Features for the named configs follow SURVEY.md §8d: request i gets
``default_rng(1000 + i).normal(size=(S, 16))``.
"""

import numpy as np

from oracle import beam_oracle as orc

# SURVEY.md §8d configs (model part)
C1_MODEL = orc.OracleConfig(16, 16, 32, 2, 1, (256, 256, 256), 4, seed=2)
C3_MODEL = orc.OracleConfig(16, 1024, 2048, 8, 5, (4096, 4096, 4096), 4, seed=2)
C1_WIDTHS = (32, 32, 32)
C2_WIDTHS = (64, 128, 256)
C3_WIDTHS = (512, 512, 512)
C5_WIDTHS = (64, 128, 256)


def c_features(i, s_ctx, feat_dim=16):
    return np.random.default_rng(1000 + i).normal(size=(s_ctx, feat_dim))


def case_config(case):
    c = case["config"]
    return orc.OracleConfig(c["feat_dim"], c["d"], c["d_ff"], c["n_layers"],
                            c["trunk_depth"], tuple(c["level_vocab_sizes"]),
                            c["n_value_buckets"], c["seed"])


def case_features(case):
    if "feature_request" in case:
        return c_features(case["feature_request"], case["s_ctx"],
                          case["config"]["feat_dim"])
    return np.asarray(case["features"], dtype=np.float64)


def list_parity(ref, got, tau):
    """SURVEY §8c list rule: ordered SID lists identical except inside groups
    of adjacent reference entries whose score gap is < tau.  ``ref``/``got``
    are [(tokens, score)].  Returns (ok, message)."""
    if len(ref) != len(got):
        return False, f"length {len(got)} != {len(ref)}"
    i = 0
    n = len(ref)
    while i < n:
        j = i + 1
        while j < n and ref[j - 1][1] - ref[j][1] < tau:
            j += 1
        a = sorted(tuple(t) for t, _ in ref[i:j])
        b = sorted(tuple(t) for t, _ in got[i:j])
        if a != b:
            return False, f"group [{i},{j}) differs: {a[:3]} vs {b[:3]}"
        i = j
    return True, "ok"
