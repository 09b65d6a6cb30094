"""Per-CTA phase timeline of the tcgen05 GEMM (debug hook
gr4ad_debug_tc_timeline; gr4ad_debug_tc_few_rows routes every product to
the few-row tiles): %globaltimer stamps at kernel entry, after setup,
first TMA issue, first stage landed (MMA warp), last MMA commit, first
accumulator ready (epilogue), epilogue done, exit -- for a few shapes.

    python profiles/tc_timeline.py"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_22732_b200 import _native as N  # noqa: E402

lib = N.lib
lib.gr4ad_debug_tc_timeline.argtypes = [C.c_void_p]
lib.gr4ad_debug_tc_few_rows.argtypes = [C.c_int]
NAMES = ["entry", "setup", "tma0", "land0", "mma_end", "acc0", "epi_end", "exit"]


def run(M, Nn, K, reps=20, few=0):
    dev = torch.device("cuda")
    lib.gr4ad_debug_tc_few_rows(few)
    a_hi = (torch.randn(M, K, device=dev) * 0.5).half()
    a_lo = torch.zeros_like(a_hi)
    b_hi = (torch.randn(Nn, K, device=dev) * 0.5).half()
    b_lo = torch.zeros_like(b_hi)
    c = torch.empty(M, Nn, device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())

    def go():
        N.check(lib.gr4ad_gemm_presplit(p(a_hi), p(a_lo), K, p(b_hi), p(b_lo), K, p(c), Nn, M,
                                        Nn, K, C.c_float(1.0), st))
    for _ in range(3):
        go()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    buf = torch.zeros(148 * 8, dtype=torch.int64, device=dev)
    lib.gr4ad_debug_tc_timeline(p(buf))
    go()
    torch.cuda.synchronize()
    lib.gr4ad_debug_tc_timeline(None)
    t = buf.view(148, 8).cpu()
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min().item()
    rel = (t - t0).double() / 1e3
    ref = a_hi.float() @ b_hi.float().t()
    err = ((c - ref).abs().max() / ref.abs().max()).item()
    lib.gr4ad_debug_tc_few_rows(0)
    print(f"M={M} N={Nn} K={K} few_rows={few}: {us:.1f} us/launch (events), {int(used.sum())} CTAs, "
          f"max rel err {err:.2e}")
    for j, nm in enumerate(NAMES):
        col = rel[:, j]
        col = col[t[:, j] > 0]
        if col.numel():
            print(f"   {nm:8s} median {col.median().item():7.2f}  min {col.min().item():7.2f}  "
                  f"max {col.max().item():7.2f} us")


for shape in [(768, 2048, 1024), (256, 1024, 1024), (768, 1024, 2048)]:
    for few in (0, 1):
        run(*shape, few=few)
