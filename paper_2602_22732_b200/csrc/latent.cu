// Latent (weight-absorbed) cross-attention of the tensor-core path.
//
// The reference's context is the linear projection X = F W_c + b_c of the
// request's raw features F (S x F_dim, decoder.py:134-140), and its cross-
// attention is single-head with bias-free projections (layers.py:46-51,
// 82-90).  So, exactly,
//   q K^T = n W_q W_k^T (F W_c + 1 b_c)^T = (n A) F^T + (per-row constant)
//   P V W_o = P (F W_c + 1 b_c) W_v W_o   = (P F) B + c       (rows of P sum to 1)
// with A = W_q W_k^T W_c^T (d x F_dim), B = W_c W_v W_o (F_dim x d) and
// c = b_c W_v W_o formed once per snapshot, and softmax is invariant to the
// per-row constant.  This is the weight absorption of multi-head latent
// attention inference: every beam row attends over the request's F_dim-wide
// latent (its raw features, staged in shared memory) instead of d-wide keys
// and values, and the shared context K / V never has to exist.
//
// Per layer: LN1 (split) -> q_lat = n A (tcgen05 GEMM, N = F) -> latent_attn
// (this file: z = softmax(q_lat F^T / sqrt d) F) -> h += z B + c (tcgen05
// GEMM, K = F, bias + residual epilogue) -> LN2.
#include <algorithm>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace gr {

// ---------------------------------------------------------------------------
// z = softmax(scale q_lat F^T) F per row on the tensor cores: mma.sync
// m16n8k16 in 3xFP16 (lo.hi + hi.lo + hi.hi, fp32 accumulate), flash-style
// online softmax over 32-key blocks, the score C fragments reused as the P
// A fragments.  The request's features are staged in shared memory as fp16
// hi / lo (x16) and fed by ldmatrix (QK) / ldmatrix.trans (PV).  A CTA of 4
// warps owns a tile of 16 / 32 / 64 rows of one request; tiles of fewer rows
// split the keys between warps and merge through shared memory.
// ---------------------------------------------------------------------------
static __device__ __forceinline__ uint32_t lat_h2u(__half2 h) { return *reinterpret_cast<uint32_t *>(&h); }
static __device__ __forceinline__ void lat_split2(float x0, float x1, uint32_t &h, uint32_t &l) {
  const __half2 hh = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(hh);
  h = lat_h2u(hh);
  l = lat_h2u(__floats2half2_rn(x0 - hf.x, x1 - hf.y));
}
static __device__ __forceinline__ void lat_mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// d += (ah + al) . (bh + bl), lo.lo dropped
static __device__ __forceinline__ void lat_mma3(float (&d)[4], const uint32_t (&ah)[4],
                                                const uint32_t (&al)[4], uint32_t bh0, uint32_t bh1,
                                                uint32_t bl0, uint32_t bl1) {
  lat_mma(d, al, bh0, bh1);
  lat_mma(d, ah, bl0, bl1);
  lat_mma(d, ah, bh0, bh1);
}
static __device__ __forceinline__ void ldsm4(uint32_t (&r)[4], const void *p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
static __device__ __forceinline__ void ldsm4t(uint32_t (&r)[4], const void *p) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
static __device__ __forceinline__ float lat_qmax(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
static __device__ __forceinline__ float lat_qsum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

constexpr float kLatQs = 256.f, kLatXs = 16.f, kLatPs = 4096.f;  // power-of-two split scales
constexpr int kLatCK = 256;                                      // keys per staged chunk

template <int F>
struct LatMma {
  static constexpr int FP = F < 16 ? 16 : F;  // padded feature width
  static constexpr int KST = FP + 8;          // smem row stride (halves): conflict-free ldmatrix
  static constexpr int FT = FP / 8;           // feature n8 tiles (PV)
  static constexpr int KK = FP / 16;          // k16 steps (QK)
  static constexpr size_t smem =
      2 * sizeof(__half) * kLatCK * KST + sizeof(float) * 4 * 16 * (FP + 2);
};

template <int F>
__global__ void __launch_bounds__(128)
latent_attn_kernel(const float *__restrict__ q, const float *__restrict__ feats,
                   const int *__restrict__ g_row_off, const int *__restrict__ g_rows,
                   const int *__restrict__ g_ctx_off, const int *__restrict__ g_ctx_len,
                   int rows_per_cta, float scale, float *__restrict__ z, int *flag) {
  using C = LatMma<F>;
  constexpr int FP = C::FP, KST = C::KST, FT = C::FT, KK = C::KK;
  extern __shared__ float4 sm4[];
  __half *xh = reinterpret_cast<__half *>(sm4);
  __half *xl = xh + kLatCK * KST;
  float *mrg = reinterpret_cast<float *>(xl + kLatCK * KST);  // 4 warps x 16 rows x (FP + 2)
  const int gi = blockIdx.y;
  const int r0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, g_rows[gi] - r0);
  if (nr <= 0) return;
  const long long row0 = (long long)g_row_off[gi] + r0;
  const int S = g_ctx_len[gi];
  const float *kf = feats + (long long)g_ctx_off[gi] * F;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, qq = lane & 3;
  const int RT = rows_per_cta / 16, KSL = 4 / RT;  // row tiles x key slices = 4 warps
  const int rt = warp % RT, ks = warp / RT;
  // A fragments of q_lat (16 rows x FP), scaled and split
  uint32_t qh[KK][4], ql[KK][4];
  {
    const int ra = rt * 16 + gq, rb = ra + 8;
    auto qv = [&](int r, int c) -> float {
      if (r >= nr || c >= F) return 0.f;
      const float v = q[(row0 + r) * F + c] * (scale * kLatQs);
      range_check(v, flag);
      return v;
    };
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      const int c = 16 * k + 2 * qq;
      lat_split2(qv(ra, c), qv(ra, c + 1), qh[k][0], ql[k][0]);
      lat_split2(qv(rb, c), qv(rb, c + 1), qh[k][1], ql[k][1]);
      lat_split2(qv(ra, c + 8), qv(ra, c + 9), qh[k][2], ql[k][2]);
      lat_split2(qv(rb, c + 8), qv(rb, c + 9), qh[k][3], ql[k][3]);
    }
  }
  const float c2 = 1.4426950408889634f / (kLatQs * kLatXs);  // log2(e) / score scale
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[FT][4];
#pragma unroll
  for (int n = 0; n < FT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  for (int c0 = 0; c0 < S; c0 += kLatCK) {
    const int nk = min(kLatCK, S - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < kLatCK * FP / 2; i += blockDim.x) {
      const int k = i / (FP / 2), f = 2 * (i - k * (FP / 2));
      float v0 = 0.f, v1 = 0.f;
      if (k < nk && f < F) {
        const float2 t = *reinterpret_cast<const float2 *>(kf + (long long)(c0 + k) * F + f);
        v0 = t.x * kLatXs;
        v1 = t.y * kLatXs;
        range_check(v0, flag);
        range_check(v1, flag);
      }
      uint32_t h, l;
      lat_split2(v0, v1, h, l);
      *reinterpret_cast<uint32_t *>(xh + k * KST + f) = h;
      *reinterpret_cast<uint32_t *>(xl + k * KST + f) = l;
    }
    __syncthreads();
    for (int kb = ks * 32; kb < nk; kb += 32 * KSL) {
      // ---- scores of 32 keys: 4 n8 tiles --------------------------------
      float s[4][4];
#pragma unroll
      for (int n = 0; n < 4; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
      for (int hp = 0; hp < 2; ++hp) {  // keys kb + 16 hp .. + 15: n-tiles 2hp, 2hp+1
        const int key = kb + 16 * hp + (lane >> 4) * 8 + (lane & 7);
#pragma unroll
        for (int k = 0; k < KK; ++k) {
          const int f = 16 * k + ((lane >> 3) & 1) * 8;
          uint32_t bh[4], bl[4];
          ldsm4(bh, xh + key * KST + f);
          ldsm4(bl, xl + key * KST + f);
          lat_mma3(s[2 * hp], qh[k], ql[k], bh[0], bh[1], bl[0], bl[1]);
          lat_mma3(s[2 * hp + 1], qh[k], ql[k], bh[2], bh[3], bl[2], bl[3]);
        }
      }
      if (kb + 32 > nk) {  // tail: keys past the request's context
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          const int col = kb + 8 * n + 2 * qq;
          if (col >= nk) s[n][0] = s[n][2] = -INFINITY;
          if (col + 1 >= nk) s[n][1] = s[n][3] = -INFINITY;
        }
      }
      // ---- online softmax (rows gq, gq + 8) -------------------------------
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        mx0 = fmaxf(mx0, fmaxf(s[n][0], s[n][1]));
        mx1 = fmaxf(mx1, fmaxf(s[n][2], s[n][3]));
      }
      const float mn0 = fmaxf(m0, lat_qmax(mx0)), mn1 = fmaxf(m1, lat_qmax(mx1));
      const float a0 = exp2f((m0 - mn0) * c2), a1 = exp2f((m1 - mn1) * c2);
      m0 = mn0;
      m1 = mn1;
      l0 *= a0;
      l1 *= a1;
#pragma unroll
      for (int n = 0; n < FT; ++n) {
        o[n][0] *= a0; o[n][1] *= a0;
        o[n][2] *= a1; o[n][3] *= a1;
      }
      const float b0 = m0 * c2, b1 = m1 * c2;
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        s[n][0] = exp2f(fmaf(s[n][0], c2, -b0));
        s[n][1] = exp2f(fmaf(s[n][1], c2, -b0));
        s[n][2] = exp2f(fmaf(s[n][2], c2, -b1));
        s[n][3] = exp2f(fmaf(s[n][3], c2, -b1));
        l0 += s[n][0] + s[n][1];
        l1 += s[n][2] + s[n][3];
      }
      // ---- z += P X: 2 k16 steps of 16 keys ------------------------------
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t ph[4], pl[4];
        lat_split2(s[2 * j][0] * kLatPs, s[2 * j][1] * kLatPs, ph[0], pl[0]);
        lat_split2(s[2 * j][2] * kLatPs, s[2 * j][3] * kLatPs, ph[1], pl[1]);
        lat_split2(s[2 * j + 1][0] * kLatPs, s[2 * j + 1][1] * kLatPs, ph[2], pl[2]);
        lat_split2(s[2 * j + 1][2] * kLatPs, s[2 * j + 1][3] * kLatPs, ph[3], pl[3]);
        const int key = kb + 16 * j + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
        for (int fp = 0; fp < FT / 2; ++fp) {  // feature tiles 2fp, 2fp+1
          const int f = 16 * fp + (lane >> 4) * 8;
          uint32_t bh[4], bl[4];
          ldsm4t(bh, xh + key * KST + f);
          ldsm4t(bl, xl + key * KST + f);
          lat_mma3(o[2 * fp], ph, pl, bh[0], bh[1], bl[0], bl[1]);
          lat_mma3(o[2 * fp + 1], ph, pl, bh[2], bh[3], bl[2], bl[3]);
        }
      }
    }
  }
  // ---- merge the key slices of each row tile ------------------------------
  l0 = lat_qsum(l0);
  l1 = lat_qsum(l1);
  constexpr int SL = FP + 2;
  float *mw = mrg + warp * 16 * SL;
  if (qq == 0) {
    mw[gq * SL] = m0; mw[gq * SL + 1] = l0;
    mw[(gq + 8) * SL] = m1; mw[(gq + 8) * SL + 1] = l1;
  }
#pragma unroll
  for (int n = 0; n < FT; ++n) {
    mw[gq * SL + 2 + 8 * n + 2 * qq] = o[n][0];
    mw[gq * SL + 3 + 8 * n + 2 * qq] = o[n][1];
    mw[(gq + 8) * SL + 2 + 8 * n + 2 * qq] = o[n][2];
    mw[(gq + 8) * SL + 3 + 8 * n + 2 * qq] = o[n][3];
  }
  __syncthreads();
  if (ks != 0) return;
  const float inv_os = 1.f / (kLatPs * kLatXs);
  for (int e = lane; e < 16 * F; e += 32) {
    const int rr = e / F, f = e - rr * F;
    if (rt * 16 + rr >= nr) continue;
    float M = -INFINITY;
    for (int s2 = 0; s2 < KSL; ++s2) M = fmaxf(M, mrg[((s2 * RT + rt) * 16 + rr) * SL]);
    float L = 0.f, Z = 0.f;
    for (int s2 = 0; s2 < KSL; ++s2) {
      const float *o2 = mrg + ((s2 * RT + rt) * 16 + rr) * SL;
      const float w = o2[0] == -INFINITY ? 0.f : exp2f((o2[0] - M) * c2);
      L = fmaf(o2[1], w, L);
      Z = fmaf(o2[2 + f], w, Z);
    }
    z[(row0 + rt * 16 + rr) * F + f] = Z * inv_os / L;
  }
}

bool latent_supported(int d, int F) {
  return d % 128 == 0 && d <= 1024 && (F == 4 || F == 8 || F == 16 || F == 32);
}

#define GR_LAT_F(M) M(4) M(8) M(16) M(32)

int latent_attn(const float *q, const float *feats, int F, const int *g_row_off, const int *g_rows,
                const int *g_ctx_off, const int *g_ctx_len, int n_groups, int max_group_rows,
                float scale, float *z, int *flag, cudaStream_t st) {
  if (n_groups <= 0 || max_group_rows <= 0) return GR4AD_OK;
  // rows per CTA: one 16-row tile per warp, or fewer row tiles with the
  // keys split between the warps
  const int rpc = max_group_rows <= 16 ? 16 : (max_group_rows <= 32 ? 32 : 64);
  prof_tag("latent_attn groups=%d max_rows=%d", n_groups, max_group_rows);
#define GR_LA_F(FF)                                                                          \
  if (F == FF) {                                                                             \
    const size_t sm = LatMma<FF>::smem;                                                      \
    GR_CUDA(cudaFuncSetAttribute(latent_attn_kernel<FF>,                                     \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));     \
    dim3 grid(ceil_div(max_group_rows, rpc), n_groups);                                      \
    GR_LAUNCH(KC_ATTN_GEMM, st, latent_attn_kernel<FF><<<grid, 128, sm, st>>>(                \
                                    q, feats, g_row_off, g_rows, g_ctx_off, g_ctx_len, rpc,  \
                                    scale, z, flag));                                        \
    return GR4AD_OK;                                                                         \
  }
  GR_LAT_F(GR_LA_F)
#undef GR_LA_F
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent attention: F %d", F);
}

}  // namespace gr
