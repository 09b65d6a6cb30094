"""CPU-side checks of the C-ABI boundary: the sm_100a library loads and
exports every entry point include/gr4ad.h declares (no compute calls)."""

import os
import re

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "gr4ad.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(gr4ad_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2602_22732_b200 import _native as N
    lib = ctypes.CDLL(N.LIB_PATH)
    names = _declared()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(N.EXPORTS)


def test_abi_version_and_status_strings():
    from paper_2602_22732_b200 import _native as N
    assert N.lib.gr4ad_abi_version() == 2
    assert N.lib.gr4ad_status_string(0) == b"ok"
    assert N.lib.gr4ad_status_string(1) == b"invalid argument"


def test_library_is_sm100a():
    import subprocess
    from paper_2602_22732_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        import pytest
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_workspace_planning_on_host():
    """gr4ad_workspace_bytes is pure host planning: it validates like
    beam.py:125-156 and sizes the C2 batch without touching a GPU."""
    import ctypes as C

    import pytest

    from paper_2602_22732_b200 import _native as N
    dm = N.Dims()
    dm.feat_dim, dm.d, dm.d_ff, dm.n_layers, dm.trunk_depth = 16, 16, 32, 2, 1
    dm.n_levels, dm.n_value_buckets = 3, 4
    for t in range(3):
        dm.vocab[t] = 256
    B = 512
    ctx = (C.c_int * B)(*([256] * B))
    w = (C.c_int * (3 * B))(*([64, 128, 256] * B))
    bt = N.Batch()
    bt.n_requests, bt.ctx_len, bt.widths, bt.trunk_depth = B, ctx, w, -1
    nbytes, max_out = C.c_size_t(), C.c_int()
    N.check(N.lib.gr4ad_workspace_bytes(C.byref(dm), C.byref(bt), C.byref(nbytes),
                                        C.byref(max_out)))
    assert max_out.value == 256
    assert 0 < nbytes.value < 4 << 30
    bt.trunk_depth = 2
    with pytest.raises(ValueError, match="trunk_depth"):
        N.check(N.lib.gr4ad_workspace_bytes(C.byref(dm), C.byref(bt), C.byref(nbytes),
                                            C.byref(max_out)))
    bt.trunk_depth = -1
    ctx[3] = 0
    with pytest.raises(ValueError, match="empty context"):
        N.check(N.lib.gr4ad_workspace_bytes(C.byref(dm), C.byref(bt), C.byref(nbytes),
                                            C.byref(max_out)))
