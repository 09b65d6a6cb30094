// Grouped fp32 GEMM with fused epilogues (CUDA-core path).
//
//   C[g] = epi(alpha * A[g] @ op(B[g]))      op(B) = B or B^T
//
// Groups implement the per-request attention contractions of the
// beam-shared context KV: every beam row of request g multiplies the same
// (S_g, d) K/V block, so the KV tile is read once per tile of beams
// (beam.py:221-232 broadcast views, layers.py:46-51).
#pragma once
#include "common.cuh"

namespace gr {

// GM_QK_T / GM_PV_T (tcgen05 only): the per-request attention products with
// A and B swapped for small beam counts -- M = keys (QK) or dims (PV) of the
// request, N = its beam rows -- and the result stored transposed, so tiles
// are not padded to 128 rows
enum GemmMode { GM_PLAIN = 0, GM_QK = 1, GM_PV = 2, GM_QK_T = 3, GM_PV_T = 4 };
enum GemmEpi {
  EPI_STORE = 0,      // C = alpha*acc
  EPI_BIAS = 1,       // C = acc + bias[n]
  EPI_BIAS_GELU = 2,  // C = gelu(acc + bias[n])
  EPI_RESID = 3,      // C = R + acc
  EPI_BIAS_RESID = 4, // C = R + (acc + bias[n])
  EPI_MULVEC = 5,     // C = vec[req(r)][n] * acc   (fuse gate m * (s W_g))
  EPI_KV_SPLIT = 6,   // C = acc, and the V half of each layer also written transposed
  EPI_STORE_LSE = 7,  // C = alpha*acc, plus per-row (max, sum exp) of every 128 columns
  EPI_STORE_T = 8,    // C^T = alpha*acc (GM_QK_T / GM_PV_T)
  // tcgen05 only: the result as fp16 hi / lo (c_hi / c_lo, ld = ldc), the
  // next GEMM's pre-split A operand
  EPI_STORE_SPLIT = 9,
  EPI_BIAS_GELU_SPLIT = 10,
  EPI_STORE_T_SPLIT = 11,
  EPI_BIAS_RESID_DUAL = 12,  // EPI_BIAS_RESID, and the result also as fp16 hi / lo
  EPI_BIAS_DUAL = 13,        // EPI_BIAS, and the result also as fp16 hi / lo
  EPI_MULVEC_SPLIT = 14      // EPI_MULVEC, the result only as fp16 hi / lo
};

struct GemmArgs {
  const float *A, *B;
  float *C;
  const float *R, *bias;
  long long lda, ldb, ldc, ldr;
  int M, N, K;  // uniform, or the max over groups
  float alpha;
  int groups;
  int mode;
  const int *g_row_off;  // [groups] row offset into A/C/R
  const int *g_rows;     // [groups] rows of the group
  const int *g_ctx_off;  // [groups] row offset into B
  const int *g_ctx_len;  // [groups] N (GM_QK) or K (GM_PV)
  const float *vec;      // EPI_MULVEC
  long long vec_ld;
  const int *row_req;    // EPI_MULVEC: request of each row
};

template <int BM, int BN, int BK, int TM, int TN, bool TRANS_B, int EPI>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_f32_kernel(GemmArgs a) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int TX = BN / TN;
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];

  const int g = blockIdx.z;
  int M = a.M, N = a.N, K = a.K;
  const float *A = a.A, *B = a.B;
  float *C = a.C;
  const float *R = a.R;
  long long row_base = 0;
  if (a.groups > 1 || a.g_rows) {
    row_base = a.g_row_off ? a.g_row_off[g] : 0;
    M = a.g_rows ? a.g_rows[g] : M;
    if (a.mode == GM_QK) {
      N = a.g_ctx_len[g];
      B += (long long)a.g_ctx_off[g] * a.ldb;
    } else if (a.mode == GM_PV) {
      K = a.g_ctx_len[g];
      B += (long long)a.g_ctx_off[g] * a.ldb;
    }
    A += row_base * a.lda;
    C += row_base * a.ldc;
    if (R) R += row_base * a.ldr;
  }
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M || n0 >= N) return;

  const int tid = threadIdx.x;
  const int ty = tid / TX, tx = tid % TX;
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = BN * BK / NT;
  float ra[A_PER], rb[B_PER];

  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      int e = tid + i * NT;
      int r = e / BK, c = e % BK;
      int gm = m0 + r, gk = k0 + c;
      ra[i] = (gm < M && gk < K) ? __ldg(A + (long long)gm * a.lda + gk) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      int e = tid + i * NT;
      if (TRANS_B) {  // B is (N, K) row-major
        int n = e / BK, c = e % BK;
        int gn = n0 + n, gk = k0 + c;
        rb[i] = (gn < N && gk < K) ? __ldg(B + (long long)gn * a.ldb + gk) : 0.f;
      } else {  // B is (K, N) row-major
        int kr = e / BN, n = e % BN;
        int gn = n0 + n, gk = k0 + kr;
        rb[i] = (gn < N && gk < K) ? __ldg(B + (long long)gk * a.ldb + gn) : 0.f;
      }
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      int e = tid + i * NT;
      As[buf][e % BK][e / BK] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      int e = tid + i * NT;
      if (TRANS_B) Bs[buf][e % BK][e / BK] = rb[i];
      else Bs[buf][e / BN][e % BN] = rb[i];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  int nk = (K + BK - 1) / BK;
  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    int buf = kt & 1;
    if (kt + 1 < nk) load_tiles((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      store_tiles(buf ^ 1);
      __syncthreads();
    }
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int gn = n0 + tx * TN + j;
      if (gn >= N) continue;
      float v = acc[i][j] * a.alpha;
      if (EPI == EPI_BIAS) v = v + a.bias[gn];
      else if (EPI == EPI_BIAS_GELU) v = gelu_tanh(v + a.bias[gn]);
      else if (EPI == EPI_RESID) v = R[(long long)gm * a.ldr + gn] + v;
      else if (EPI == EPI_BIAS_RESID) v = R[(long long)gm * a.ldr + gn] + (v + a.bias[gn]);
      else if (EPI == EPI_MULVEC)
        v = a.vec[(long long)a.row_req[row_base + gm] * a.vec_ld + gn] * v;
      C[(long long)gm * a.ldc + gn] = v;
    }
  }
}

int gemm(const GemmArgs &a, bool trans_b, int epi, cudaStream_t st);

inline GemmArgs plain_gemm(const float *A, long long lda, const float *B, long long ldb,
                           float *C, long long ldc, int M, int N, int K) {
  GemmArgs g{};
  g.A = A; g.B = B; g.C = C; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
  g.M = M; g.N = N; g.K = K; g.alpha = 1.f; g.groups = 1; g.mode = GM_PLAIN;
  return g;
}

}  // namespace gr
