"""Numerics of the decode's GEMMs through the C ABI (gr4ad_gemm) against a
float64 torch reference: the CUDA-core fp32 path and the tcgen05 3xFP16
path must both be fp32-faithful (relative error ~1e-6, far below TF32's
~1e-3), since beam lists depend on it (SURVEY §7 hard part 1)."""

import ctypes as C

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gemm(A, BT, backend):
    from paper_2602_22732_b200 import _native as N
    M, K = A.shape
    Nn = BT.shape[0]
    out = torch.empty((M, Nn), dtype=torch.float32, device=A.device)
    N.check(N.lib.gr4ad_gemm(C.c_void_p(A.data_ptr()), A.stride(0), C.c_void_p(BT.data_ptr()),
                             BT.stride(0), C.c_void_p(out.data_ptr()), out.stride(0), M, Nn, K,
                             backend, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("shape", [(128, 128, 32), (256, 384, 1024), (1000, 1100, 1024),
                                   (300, 4096, 1024), (77, 50, 36), (512, 1024, 2048)])
@pytest.mark.parametrize("backend", [0, 1])
def test_gemm_fp32_faithful(shape, backend):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + Nn + K)
    A = torch.randn((M, K), device="cuda", generator=g)
    BT = torch.randn((Nn, K), device="cuda", generator=g) / K ** 0.5
    got = _gemm(A, BT, backend).double()
    ref = A.double() @ BT.double().T
    scale = (A.double().abs() @ BT.double().abs().T)  # error bound scale per entry
    rel = ((got - ref).abs() / scale.clamp_min(1e-30)).max().item()
    print(f"backend {backend} shape {shape}: max scaled error {rel:.3e}")
    # fp32 accumulation over K: ~K^0.5 * 2^-24 typical; 3xFP16 drops lo.lo (~2^-22)
    assert rel < 1e-5, f"backend {backend} shape {shape}: max scaled error {rel:.3e}"


def _split16(x, scale):
    hi = (x * scale).half()
    lo = (x * scale - hi.float()).half()
    return hi.contiguous(), lo.contiguous()


# N >= 256 takes the CTA-pair (cta_group::2) kernel: 256 x 256 tiles, M tails
# inside a pair (one CTA's rows past M), K not a multiple of the 32-deep stage
@pytest.mark.parametrize("shape", [(256, 256, 64), (300, 512, 1024), (1000, 1100, 1024),
                                   (129, 4096, 72), (4096, 3072, 1024), (64, 128, 32)])
def test_gemm_presplit_pair(shape):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_22732_b200 import _native as N
    M, Nn, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 3 + Nn + K)
    A = torch.randn((M, K), device="cuda", generator=g)
    BT = torch.randn((Nn, K), device="cuda", generator=g) / K ** 0.5
    ah, al = _split16(A, 1.0)
    bh, bl = _split16(BT, 2048.0)  # the weights' power-of-two pre-scale
    out = torch.full((M, Nn), float("nan"), dtype=torch.float32, device="cuda")
    N.check(N.lib.gr4ad_gemm_presplit(
        C.c_void_p(ah.data_ptr()), C.c_void_p(al.data_ptr()), K, C.c_void_p(bh.data_ptr()),
        C.c_void_p(bl.data_ptr()), K, C.c_void_p(out.data_ptr()), Nn, M, Nn, K, 1.0 / 2048.0,
        C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = A.double() @ BT.double().T
    scale = A.double().abs() @ BT.double().abs().T
    rel = ((out.double() - ref).abs() / scale.clamp_min(1e-30)).max().item()
    print(f"pre-split shape {shape}: max scaled error {rel:.3e}")
    assert torch.isfinite(out).all()
    assert rel < 1e-5, f"pre-split shape {shape}: max scaled error {rel:.3e}"
