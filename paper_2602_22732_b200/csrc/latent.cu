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
constexpr int kLatCKLn = 128;  // fused-LN1 variant: double-buffered, smaller chunks

template <int F>
struct LatMma {
  static constexpr int FP = F < 16 ? 16 : F;  // padded feature width
  static constexpr int KST = FP + 8;          // smem row stride (halves): conflict-free ldmatrix
  static constexpr int FT = FP / 8;           // feature n8 tiles (PV)
  static constexpr int KK = FP / 16;          // k16 steps (QK)
  static constexpr size_t smem =
      2 * sizeof(__half) * kLatCK * KST + sizeof(float) * 4 * 16 * (FP + 2);
  // the fused-LN1 variant double-buffers the staged chunks
  static constexpr size_t smem_ln =
      4 * sizeof(__half) * kLatCKLn * KST + sizeof(float) * 4 * 16 * (FP + 2);
};

// q_lat formed inside the attention kernel (kLn): LN1 of the rows and the
// projection LN1(h) A on mma.sync in ONE pass over h, so neither LN1's output
// nor q_lat exists in HBM.  With A' = diag(g1) A, s = 1^T A' and
// c = b1 A (formed per snapshot, lat_fold_kernel) and any per-row shift k,
//   LN1(h) A = r ((h - k) A' - (mu - k) s) + c,
//   mu = k + S1 / d,  var = S2 / d - (S1 / d)^2,  r = (var + 1e-5)^-1/2
// where S1, S2 are the sums of (h - k) and (h - k)^2.  k is the mean of the
// row's first 16 entries, so |mu - k| is a fraction of the row's spread and
// neither the variance nor the correction term cancels.
struct LatLn {
  const float *h;                // (rows, d) residual stream, ld d
  int d;
  const __half *aq_hi, *aq_lo;   // kWeightScale A'^T as fp16 hi / lo (F x d)
  const float *s, *c;            // 1^T A', b1 A (F each)
  const __half *fs_hi, *fs_lo;   // kLatXs features as fp16 hi / lo, rows of KST halves
};

static __device__ __forceinline__ void cp16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src));
}
static __device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
static __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

template <int F, bool kLn>
__global__ void __launch_bounds__(128)
latent_attn_kernel(const float *__restrict__ q, const float *__restrict__ feats,
                   const int *__restrict__ g_row_off, const int *__restrict__ g_rows,
                   const int *__restrict__ g_ctx_off, const int *__restrict__ g_ctx_len,
                   int rows_per_cta, float scale, float *__restrict__ z, int *flag,
                   const LatLn ln) {
  using C = LatMma<F>;
  constexpr int FP = C::FP, KST = C::KST, FT = C::FT, KK = C::KK;
  constexpr int CK = kLn ? kLatCKLn : kLatCK;  // keys per staged chunk
  constexpr int CH = CK * KST;                 // halves per staged chunk (hi or lo)
  extern __shared__ float4 sm4[];
  __half *xh = reinterpret_cast<__half *>(sm4);
  __half *xl = xh + CH;
  // kLn: two chunk buffers (cp.async double buffering)
  float *mrg = reinterpret_cast<float *>(xh + (kLn ? 4 : 2) * CH);  // 4 warps x 16 rows x (FP + 2)
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
  // kLn: stage chunk c0 of the pre-split features into buffer `buf`
  auto stage = [&](int c0, int buf) {
    const __half *sh = ln.fs_hi + ((long long)g_ctx_off[gi] + c0) * KST;
    const __half *sl = ln.fs_lo + ((long long)g_ctx_off[gi] + c0) * KST;
    __half *dh = reinterpret_cast<__half *>(sm4) + 2 * buf * CH, *dl = dh + CH;
    for (int i = threadIdx.x; i < CH / 8; i += blockDim.x) {
      cp16(dh + 8 * i, sh + 8 * i);
      cp16(dl + 8 * i, sl + 8 * i);
    }
    cp_commit();
  };
  if constexpr (kLn) stage(0, 0);  // in flight during the q_lat pass
  // A fragments of q_lat (16 rows x FP), scaled and split
  uint32_t qh[KK][4], ql[KK][4];
  if constexpr (kLn) {
    const int d = ln.d;
    const int ra = rt * 16 + gq, rb = ra + 8;
    const float *ha = ln.h + (row0 + (ra < nr ? ra : 0)) * d;
    const float *hb = ln.h + (row0 + (rb < nr ? rb : 0)) * d;
    // shifts: mean of each row's first 16 entries (the quad holds them)
    float kA, kB;
    {
      const float2 a0 = __ldg(reinterpret_cast<const float2 *>(ha + 2 * qq));
      const float2 a1 = __ldg(reinterpret_cast<const float2 *>(ha + 8 + 2 * qq));
      const float2 b0 = __ldg(reinterpret_cast<const float2 *>(hb + 2 * qq));
      const float2 b1 = __ldg(reinterpret_cast<const float2 *>(hb + 8 + 2 * qq));
      kA = lat_qsum((a0.x + a0.y) + (a1.x + a1.y)) * (1.f / 16.f);
      kB = lat_qsum((b0.x + b0.y) + (b1.x + b1.y)) * (1.f / 16.f);
    }
    float s1A = 0.f, s2A = 0.f, s1B = 0.f, s2B = 0.f;
    float c[FT][4];
#pragma unroll
    for (int n = 0; n < FT; ++n) c[n][0] = c[n][1] = c[n][2] = c[n][3] = 0.f;
    // k32 blocks with a lane-permuted k order (a dot product is invariant
    // to it as long as A and B share it): lane qq owns k0 + 8 qq .. + 7 of
    // both rows and of every B column, so each operand is one 16-B load --
    // 32 contiguous bytes per row per quad -- and the k16 step j takes
    // entries 4 j .. 4 j + 3 as MMA k (2 qq, 2 qq + 1, 8 + 2 qq, 9 + 2 qq).
    // The next block's loads are issued before this block's MMAs.
    const float4 *pa = reinterpret_cast<const float4 *>(ha + 8 * qq);
    const float4 *pb = reinterpret_cast<const float4 *>(hb + 8 * qq);
    const uint4 *ph[FT], *pl[FT];
#pragma unroll
    for (int n = 0; n < FT; ++n) {
      const int col = min(8 * n + gq, F - 1);  // columns >= F: B forced to 0 below
      ph[n] = reinterpret_cast<const uint4 *>(ln.aq_hi + (long long)col * d + 8 * qq);
      pl[n] = reinterpret_cast<const uint4 *>(ln.aq_lo + (long long)col * d + 8 * qq);
    }
    float4 xa[2], xb[2];
    uint4 bh[FT], bl[FT];
    auto load = [&](int k0) {
      const int q4 = k0 >> 2;  // float4 index of k0
      xa[0] = __ldg(pa + q4); xa[1] = __ldg(pa + q4 + 1);
      xb[0] = __ldg(pb + q4); xb[1] = __ldg(pb + q4 + 1);
#pragma unroll
      for (int n = 0; n < FT; ++n) {
        bh[n] = __ldg(ph[n] + (k0 >> 3));
        bl[n] = __ldg(pl[n] + (k0 >> 3));
      }
    };
    // warps sharing a row tile (small groups: KSL key slices) split the k
    // range of q_lat too and add their partials through shared memory
    const int kspan = d / KSL, kbeg = ks * kspan, kend = kbeg + kspan;
    load(kbeg);
    for (int k0 = kbeg; k0 < kend; k0 += 32) {
      float4 ca[2] = {xa[0], xa[1]}, cb[2] = {xb[0], xb[1]};
      uint4 ch[FT], cl[FT];
#pragma unroll
      for (int n = 0; n < FT; ++n) {
        const bool live = 8 * n + gq < F;
        ch[n] = live ? bh[n] : make_uint4(0, 0, 0, 0);
        cl[n] = live ? bl[n] : make_uint4(0, 0, 0, 0);
      }
      if (k0 + 32 < kend) load(k0 + 32);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float4 u = ca[j], v = cb[j];
        u.x -= kA; u.y -= kA; u.z -= kA; u.w -= kA;
        v.x -= kB; v.y -= kB; v.z -= kB; v.w -= kB;
        s1A += (u.x + u.y) + (u.z + u.w);
        s1B += (v.x + v.y) + (v.z + v.w);
        s2A = fmaf(u.x, u.x, fmaf(u.y, u.y, fmaf(u.z, u.z, fmaf(u.w, u.w, s2A))));
        s2B = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, s2B))));
        uint32_t ah[4], al[4];
        lat_split2(u.x, u.y, ah[0], al[0]);
        lat_split2(v.x, v.y, ah[1], al[1]);
        lat_split2(u.z, u.w, ah[2], al[2]);
        lat_split2(v.z, v.w, ah[3], al[3]);
#pragma unroll
        for (int n = 0; n < FT; ++n) {
          const uint32_t b0h = j ? ch[n].z : ch[n].x, b1h = j ? ch[n].w : ch[n].y;
          const uint32_t b0l = j ? cl[n].z : cl[n].x, b1l = j ? cl[n].w : cl[n].y;
          lat_mma3(c[n], ah, al, b0h, b1h, b0l, b1l);
        }
      }
    }
    // row statistics (the quad's four lanes hold a row's partial sums)
    s1A = lat_qsum(s1A); s2A = lat_qsum(s2A);
    s1B = lat_qsum(s1B); s2B = lat_qsum(s2B);
    if (KSL > 1) {  // sum the k-slice partials of this row tile (block-uniform)
      constexpr int SL = FP + 2;
      float *mw = mrg + warp * 16 * SL;
#pragma unroll
      for (int n = 0; n < FT; ++n) {
        const int col = 8 * n + 2 * qq;
        mw[gq * SL + col] = c[n][0];
        mw[gq * SL + col + 1] = c[n][1];
        mw[(gq + 8) * SL + col] = c[n][2];
        mw[(gq + 8) * SL + col + 1] = c[n][3];
      }
      if (qq == 0) {
        mw[gq * SL + FP] = s1A; mw[gq * SL + FP + 1] = s2A;
        mw[(gq + 8) * SL + FP] = s1B; mw[(gq + 8) * SL + FP + 1] = s2B;
      }
      __syncthreads();
#pragma unroll
      for (int n = 0; n < FT; ++n) c[n][0] = c[n][1] = c[n][2] = c[n][3] = 0.f;
      s1A = s2A = s1B = s2B = 0.f;
      for (int k2 = 0; k2 < KSL; ++k2) {
        const float *ow = mrg + (k2 * RT + rt) * 16 * SL;
#pragma unroll
        for (int n = 0; n < FT; ++n) {
          const int col = 8 * n + 2 * qq;
          c[n][0] += ow[gq * SL + col];
          c[n][1] += ow[gq * SL + col + 1];
          c[n][2] += ow[(gq + 8) * SL + col];
          c[n][3] += ow[(gq + 8) * SL + col + 1];
        }
        s1A += ow[gq * SL + FP]; s2A += ow[gq * SL + FP + 1];
        s1B += ow[(gq + 8) * SL + FP]; s2B += ow[(gq + 8) * SL + FP + 1];
      }
      __syncthreads();  // (the merge area is reused at the end)
    }
    const float invd = 1.f / (float)d;
    const float mA = s1A * invd, mB = s1B * invd;  // mu - k
    const float rA = 1.0f / sqrtf(fmaxf(fmaf(s2A, invd, -mA * mA), 0.f) + 1e-5f);
    const float rB = 1.0f / sqrtf(fmaxf(fmaf(s2B, invd, -mB * mB), 0.f) + 1e-5f);
    // q_lat = r (C / kWeightScale - (mu - k) s) + c, then the score scale;
    // C fragments of q_lat are the A fragments of the scores (k = features)
    const float qs = scale * kLatQs;
#pragma unroll
    for (int n = 0; n < FT; ++n) {
      const int f0 = 8 * n + 2 * qq;
      const float sv0 = f0 < F ? __ldg(ln.s + f0) : 0.f, sv1 = f0 + 1 < F ? __ldg(ln.s + f0 + 1) : 0.f;
      const float cv0 = f0 < F ? __ldg(ln.c + f0) : 0.f, cv1 = f0 + 1 < F ? __ldg(ln.c + f0 + 1) : 0.f;
      c[n][0] = (rA * fmaf(c[n][0], 1.f / kWeightScale, -mA * sv0) + cv0) * qs;
      c[n][1] = (rA * fmaf(c[n][1], 1.f / kWeightScale, -mA * sv1) + cv1) * qs;
      c[n][2] = (rB * fmaf(c[n][2], 1.f / kWeightScale, -mB * sv0) + cv0) * qs;
      c[n][3] = (rB * fmaf(c[n][3], 1.f / kWeightScale, -mB * sv1) + cv1) * qs;
#pragma unroll
      for (int e = 0; e < 4; ++e) range_check(c[n][e], flag);
    }
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      lat_split2(c[2 * k][0], c[2 * k][1], qh[k][0], ql[k][0]);
      lat_split2(c[2 * k][2], c[2 * k][3], qh[k][1], ql[k][1]);
      lat_split2(c[2 * k + 1][0], c[2 * k + 1][1], qh[k][2], ql[k][2]);
      lat_split2(c[2 * k + 1][2], c[2 * k + 1][3], qh[k][3], ql[k][3]);
    }
  } else {
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
  for (int c0 = 0, cb = 0; c0 < S; c0 += CK, cb ^= 1) {
    const int nk = min(CK, S - c0);
    __syncthreads();
    if constexpr (kLn) {
      // prefetch the next chunk into the other buffer, wait for this one
      if (c0 + CK < S) stage(c0 + CK, cb ^ 1);
      else cp_commit();
      cp_wait<1>();
      __syncthreads();
      xh = reinterpret_cast<__half *>(sm4) + 2 * cb * CH;
      xl = xh + CH;
    } else {
    for (int i = threadIdx.x; i < CK * FP / 2; i += blockDim.x) {
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
    }
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

// ---------------------------------------------------------------------------
// Part 2 of the latent cross-attention block: h += z B + c, then LN2 of the
// new row (layers.py:82-90 residual, 101 LayerNorm).  A CTA owns 16 rows x
// d.  One thread bulk-copies the 16 residual rows into shared memory (TMA
// engine, mbarrier) while warp w forms z B for columns [128 w, 128 w + 128)
// on mma.sync (3xFP16); the sum lands in the staged rows; then a warp per
// row runs LN2 exactly as ln_rows_split (mean, then the centred variance,
// row in registers) and writes the row as fp32 (the residual stream), fp16
// hi / lo (the next GEMM's A operand) and optionally fp32 again (the
// factored self-attention's history), all as coalesced 16-B accesses.
// ---------------------------------------------------------------------------
constexpr float kLatZs = 256.f;

static __device__ __forceinline__ void lo_bar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
static __device__ __forceinline__ void lo_bar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

template <int NW>
struct LatOut {
  static constexpr int D = NW * 128, LDT = D + 8;  // +8: conflict-free fragment accesses
  static constexpr size_t smem = sizeof(float) * 16 * LDT;
};

template <int F, int NW>
__global__ void __launch_bounds__(NW * 32, 2)
latent_out_ln_kernel(const float *__restrict__ z, const __half *__restrict__ bo_hi,
                     const __half *__restrict__ bo_lo, float alpha, const float *__restrict__ c,
                     float *hs, const float *__restrict__ g2, const float *__restrict__ b2,
                     __half *__restrict__ n_hi, __half *__restrict__ n_lo, long long ld_n,
                     float *__restrict__ hn, long long ld_hn, int rows, int *flag) {
  constexpr int FP = F < 16 ? 16 : F, KK = FP / 16, D = LatOut<NW>::D, LDT = LatOut<NW>::LDT;
  extern __shared__ float4 sm4[];
  float *tile = reinterpret_cast<float *>(sm4);
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, qq = lane & 3;
  const long long r0 = (long long)blockIdx.x * 16;
  const int nrows = (int)min(16LL, rows - r0);
  if (threadIdx.x == 0) lo_bar_init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                 "r"((uint32_t)(nrows * D * 4))
                 : "memory");
    for (int r = 0; r < nrows; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"((uint32_t)__cvta_generic_to_shared(tile + r * LDT)),
          "l"(hs + (r0 + r) * D), "r"(D * 4), "r"(bar_a)
          : "memory");
  }
  const bool va = gq < nrows, vb = gq + 8 < nrows;
  uint32_t ah[KK][4], al[KK][4];
  {
    auto zv = [&](bool v, int r, int col) -> float {
      if (!v || col >= F) return 0.f;
      const float x = z[(r0 + r) * F + col] * kLatZs;
      range_check(x, flag);
      return x;
    };
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      const int col = 16 * k + 2 * qq;
      lat_split2(zv(va, gq, col), zv(va, gq, col + 1), ah[k][0], al[k][0]);
      lat_split2(zv(vb, gq + 8, col), zv(vb, gq + 8, col + 1), ah[k][1], al[k][1]);
      lat_split2(zv(va, gq, col + 8), zv(va, gq, col + 9), ah[k][2], al[k][2]);
      lat_split2(zv(vb, gq + 8, col + 8), zv(vb, gq + 8, col + 9), ah[k][3], al[k][3]);
    }
  }
  const int j0 = warp * 128;
  float acc[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
    const long long o = (long long)(j0 + 8 * n + gq) * F;  // B^T row (K-major B)
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      const int fa = 16 * k + 2 * qq, fb = fa + 8;
      uint32_t b0h = 0, b1h = 0, b0l = 0, b1l = 0;
      if (fa < F) {
        b0h = __ldg(reinterpret_cast<const unsigned int *>(bo_hi + o + fa));
        b0l = __ldg(reinterpret_cast<const unsigned int *>(bo_lo + o + fa));
      }
      if (fb < F) {
        b1h = __ldg(reinterpret_cast<const unsigned int *>(bo_hi + o + fb));
        b1l = __ldg(reinterpret_cast<const unsigned int *>(bo_lo + o + fb));
      }
      lat_mma3(acc[n], ah[k], al[k], b0h, b1h, b0l, b1l);
    }
  }
  lo_bar_wait(&bar, 0);
  // staged row += z B + c: rows gq (acc[.][0..1]) and gq + 8 (acc[.][2..3])
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    const int col = j0 + 8 * n + 2 * qq;
    const float2 cc = __ldg(reinterpret_cast<const float2 *>(c + col));
    if (va) {
      float2 *t = reinterpret_cast<float2 *>(tile + gq * LDT + col);
      const float2 x = *t;
      *t = make_float2(x.x + fmaf(acc[n][0], alpha, cc.x), x.y + fmaf(acc[n][1], alpha, cc.y));
    }
    if (vb) {
      float2 *t = reinterpret_cast<float2 *>(tile + (gq + 8) * LDT + col);
      const float2 x = *t;
      *t = make_float2(x.x + fmaf(acc[n][2], alpha, cc.x), x.y + fmaf(acc[n][3], alpha, cc.y));
    }
  }
  __syncthreads();
  // LN2, warp per row
  for (int r = warp; r < nrows; r += NW) {
    const float4 *tr = reinterpret_cast<const float4 *>(tile + r * LDT);
    float4 v[NW];
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      v[i] = tr[lane + 32 * i];
      sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    const float mean = warp_sum(sum) / (float)D;
    float qv = 0.f;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const float a0 = v[i].x - mean, a1 = v[i].y - mean, a2 = v[i].z - mean, a3 = v[i].w - mean;
      qv += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
    const float inv = 1.0f / sqrtf(warp_sum(qv) / (float)D + 1e-5f);
    const long long gr = r0 + r;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int j = 4 * (lane + 32 * i);
      const float4 gg = __ldg(reinterpret_cast<const float4 *>(g2 + j));
      const float4 bb = __ldg(reinterpret_cast<const float4 *>(b2 + j));
      const float o[4] = {(v[i].x - mean) * inv * gg.x + bb.x, (v[i].y - mean) * inv * gg.y + bb.y,
                          (v[i].z - mean) * inv * gg.z + bb.z, (v[i].w - mean) * inv * gg.w + bb.w};
      *reinterpret_cast<float4 *>(hs + gr * D + j) = v[i];
      uint32_t h0, l0, h1, l1;
      lat_split2(o[0], o[1], h0, l0);
      lat_split2(o[2], o[3], h1, l1);
      *reinterpret_cast<uint2 *>(n_hi + gr * ld_n + j) = make_uint2(h0, h1);
      *reinterpret_cast<uint2 *>(n_lo + gr * ld_n + j) = make_uint2(l0, l1);
      if (hn) *reinterpret_cast<float4 *>(hn + gr * ld_hn + j) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

#define GR_LAT_F(M) M(4) M(8) M(16) M(32)

static int rows_per_cta_for(int max_group_rows, int n_groups) {
  // one 16-row tile per warp, or fewer row tiles with the keys split
  // between the warps: the widest tile that still gives >= 4 CTAs per SM
  // (148 SMs), so small groups (DBW early levels, trunk rows) fill the GPU
  const int cap = max_group_rows <= 16 ? 16 : (max_group_rows <= 32 ? 32 : 64);
  for (int rpc = cap; rpc > 16; rpc >>= 1)
    if ((long long)n_groups * ceil_div(max_group_rows, rpc) >= 4 * 148) return rpc;
  return 16;
}

int latent_attn(const float *q, const float *feats, int F, const int *g_row_off, const int *g_rows,
                const int *g_ctx_off, const int *g_ctx_len, int n_groups, int max_group_rows,
                float scale, float *z, int *flag, cudaStream_t st) {
  if (n_groups <= 0 || max_group_rows <= 0) return GR4AD_OK;
  const int rpc = rows_per_cta_for(max_group_rows, n_groups);
  prof_tag("latent_attn groups=%d max_rows=%d", n_groups, max_group_rows);
#define GR_LA_F(FF)                                                                          \
  if (F == FF) {                                                                             \
    const size_t sm = LatMma<FF>::smem;                                                      \
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(latent_attn_kernel<FF, false>),                              \
                                 (int)sm));     \
    dim3 grid(ceil_div(max_group_rows, rpc), n_groups);                                      \
    GR_LAUNCH(KC_ATTN_GEMM, st, latent_attn_kernel<FF, false><<<grid, 128, sm, st>>>(         \
                                    q, feats, g_row_off, g_rows, g_ctx_off, g_ctx_len, rpc,  \
                                    scale, z, flag, LatLn{}));                               \
    return GR4AD_OK;                                                                         \
  }
  GR_LAT_F(GR_LA_F)
#undef GR_LA_F
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent attention: F %d", F);
}

int latent_cross_ln(const float *h, int d, const __half *aq_hi, const __half *aq_lo,
                    const float *s1, const float *c1, const __half *fs_hi, const __half *fs_lo,
                    int F, const int *g_row_off, const int *g_rows, const int *g_ctx_off,
                    const int *g_ctx_len, int n_groups, int max_group_rows, float scale, float *z,
                    int *flag, cudaStream_t st) {
  if (n_groups <= 0 || max_group_rows <= 0) return GR4AD_OK;
  if (!latent_supported(d, F)) return set_err(GR4AD_ERR_UNSUPPORTED, "latent LN1: d %d F %d", d, F);
  const int rpc = rows_per_cta_for(max_group_rows, n_groups);
  const LatLn ln{h, d, aq_hi, aq_lo, s1, c1, fs_hi, fs_lo};
  prof_tag("latent_ln1 groups=%d max_rows=%d", n_groups, max_group_rows);
#define GR_LA_F(FF)                                                                          \
  if (F == FF) {                                                                             \
    const size_t sm = LatMma<FF>::smem_ln;                                                   \
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(latent_attn_kernel<FF, true>),                               \
                                 (int)sm));     \
    dim3 grid(ceil_div(max_group_rows, rpc), n_groups);                                      \
    GR_LAUNCH(KC_ATTN_GEMM, st, latent_attn_kernel<FF, true><<<grid, 128, sm, st>>>(          \
                                    nullptr, nullptr, g_row_off, g_rows, g_ctx_off,          \
                                    g_ctx_len, rpc, scale, z, flag, ln));                    \
    return GR4AD_OK;                                                                         \
  }
  GR_LAT_F(GR_LA_F)
#undef GR_LA_F
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent attention: F %d", F);
}

// ---------------------------------------------------------------------------
// per-snapshot folds of LN1 into the latent query projection: block per
// feature f, double accumulation:  A'^T[f] = g1 * A^T[f],  s[f] = sum_k
// A'^T[f][k],  c[f] = sum_k b1[k] A^T[f][k]
// ---------------------------------------------------------------------------
__global__ void lat_fold_kernel(const float *__restrict__ at, const float *__restrict__ g1,
                                const float *__restrict__ b1, int d, float *ag, float *sv,
                                float *cv) {
  const int f = blockIdx.x;
  double s = 0.0, c = 0.0;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const double a = at[(long long)f * d + k];
    const float v = (float)(a * (double)g1[k]);
    ag[(long long)f * d + k] = v;
    s += (double)v;
    c += (double)b1[k] * a;
  }
  __shared__ double red[2][32];
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = s;
    red[1][w] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; ++i) {
      s += red[0][i];
      c += red[1][i];
    }
    sv[f] = (float)s;
    cv[f] = (float)c;
  }
}

int latent_fold(const float *at, const float *g1, const float *b1, int d, int F, float *ag,
                float *sv, float *cv, cudaStream_t st) {
  GR_LAUNCH(KC_SMALL, st, lat_fold_kernel<<<F, 256, 0, st>>>(at, g1, b1, d, ag, sv, cv));
  return GR4AD_OK;
}

// features as kLatXs fp16 hi / lo in rows of KST halves (zero padding
// columns and rows >= rows_used): what the fused latent kernel stages with
// plain 16-byte copies
template <int F>
__global__ void lat_feat_split_kernel(const float *__restrict__ fin, long long rows_used,
                                      long long rows_alloc, __half *hi, __half *lo, int *flag) {
  using C = LatMma<F>;
  constexpr int KST = C::KST;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows_alloc * (KST / 2)) return;
  const long long r = i / (KST / 2);
  const int f = 2 * (int)(i - r * (KST / 2));
  float v0 = 0.f, v1 = 0.f;
  if (r < rows_used && f < F) {
    v0 = fin[r * F + f] * kLatXs;
    v1 = fin[r * F + f + 1] * kLatXs;
    range_check(v0, flag);
    range_check(v1, flag);
  }
  uint32_t h, l;
  lat_split2(v0, v1, h, l);
  *reinterpret_cast<uint32_t *>(hi + r * KST + f) = h;
  *reinterpret_cast<uint32_t *>(lo + r * KST + f) = l;
}

int latent_feat_kst(int F) {
  return F < 16 ? 24 : F + 8;
}

int latent_feat_split(const float *fin, long long rows_used, long long rows_alloc, int F,
                      __half *hi, __half *lo, int *flag, cudaStream_t st) {
#define GR_FS(FF)                                                                            \
  if (F == FF) {                                                                             \
    const long long n = rows_alloc * (LatMma<FF>::KST / 2);                                  \
    GR_LAUNCH(KC_SMALL, st, lat_feat_split_kernel<FF><<<ceil_div(n, 256), 256, 0, st>>>(      \
                                fin, rows_used, rows_alloc, hi, lo, flag));                  \
    return GR4AD_OK;                                                                         \
  }
  GR_LAT_F(GR_FS)
#undef GR_FS
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent features: F %d", F);
}

int latent_out_ln(const float *z, int F, const __half *bo_hi, const __half *bo_lo, float alpha,
                  const float *c, float *hs, int d, const float *g2, const float *b2,
                  __half *n_hi, __half *n_lo, long long ld_n, float *hn, long long ld_hn,
                  int rows, int *flag, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  if (!latent_supported(d, F) || (hn && ld_hn % 4 != 0) || ld_n % 4 != 0)
    return set_err(GR4AD_ERR_UNSUPPORTED, "latent output + LN2: d %d F %d", d, F);
  prof_tag("latent_out_ln2 rows=%d", rows);
  const float a = alpha / kLatZs;
#define GR_LO(FF, NW)                                                                        \
  if (F == FF && d == NW * 128) {                                                            \
    const size_t sm = LatOut<NW>::smem;                                                      \
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(latent_out_ln_kernel<FF, NW>),                               \
                                 (int)sm));     \
    GR_LAUNCH(KC_LAYERNORM, st, latent_out_ln_kernel<FF, NW><<<ceil_div(rows, 16), NW * 32,   \
                                                               sm, st>>>(                    \
                                    z, bo_hi, bo_lo, a, c, hs, g2, b2, n_hi, n_lo, ld_n, hn, \
                                    ld_hn, rows, flag));                                     \
    return GR4AD_OK;                                                                         \
  }
#define GR_LO_F(FF) GR_LO(FF, 1) GR_LO(FF, 2) GR_LO(FF, 3) GR_LO(FF, 4) GR_LO(FF, 5) \
                    GR_LO(FF, 6) GR_LO(FF, 7) GR_LO(FF, 8)
  GR_LAT_F(GR_LO_F)
#undef GR_LO_F
#undef GR_LO
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent output + LN2: d %d F %d", d, F);
}

}  // namespace gr
