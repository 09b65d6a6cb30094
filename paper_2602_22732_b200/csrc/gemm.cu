// Tile-shape dispatch for the grouped fp32 GEMM.
#include "gemm.cuh"

namespace gr {

template <int BM, int BN, int BK, int TM, int TN, bool TB>
static int launch_epi(const GemmArgs &a, int epi, cudaStream_t st) {
  dim3 grid(ceil_div(a.N, BN), ceil_div(a.M, BM), a.groups);
  dim3 block((BM / TM) * (BN / TN));
  const int cls = (a.mode == GM_PLAIN) ? KC_GEMM : KC_ATTN_GEMM;
  prof_begin(cls, st);
  switch (epi) {
    case EPI_STORE: gemm_f32_kernel<BM, BN, BK, TM, TN, TB, EPI_STORE><<<grid, block, 0, st>>>(a); break;
    case EPI_BIAS: gemm_f32_kernel<BM, BN, BK, TM, TN, TB, EPI_BIAS><<<grid, block, 0, st>>>(a); break;
    case EPI_BIAS_GELU: gemm_f32_kernel<BM, BN, BK, TM, TN, TB, EPI_BIAS_GELU><<<grid, block, 0, st>>>(a); break;
    case EPI_RESID: gemm_f32_kernel<BM, BN, BK, TM, TN, TB, EPI_RESID><<<grid, block, 0, st>>>(a); break;
    case EPI_BIAS_RESID: gemm_f32_kernel<BM, BN, BK, TM, TN, TB, EPI_BIAS_RESID><<<grid, block, 0, st>>>(a); break;
    case EPI_MULVEC: gemm_f32_kernel<BM, BN, BK, TM, TN, TB, EPI_MULVEC><<<grid, block, 0, st>>>(a); break;
    default: return set_err(GR4AD_ERR_UNSUPPORTED, "gemm epilogue %d", epi);
  }
  prof_end(cls, st);
  count_launch();
  GR_CUDA(cudaGetLastError());
  return GR4AD_OK;
}

template <bool TB>
static int launch_shape(const GemmArgs &a, int epi, cudaStream_t st) {
  if (a.N <= 32) return launch_epi<64, 32, 16, 4, 2, TB>(a, epi, st);
  if (a.N <= 64 || a.M <= 64) return launch_epi<64, 64, 16, 4, 4, TB>(a, epi, st);
  return launch_epi<128, 128, 8, 8, 8, TB>(a, epi, st);
}

int gemm(const GemmArgs &a, bool trans_b, int epi, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0 || a.groups <= 0) return GR4AD_OK;
  if (a.K <= 0 && a.mode != GM_PV)
    return set_err(GR4AD_ERR_VALUE, "gemm with K=%d", a.K);
  return trans_b ? launch_shape<true>(a, epi, st) : launch_shape<false>(a, epi, st);
}

}  // namespace gr
