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
//   ln_qlat     q_lat = LN1(h) A                          (warp per row)
//   latent_attn z = softmax(q_lat F^T / sqrt(d)) F         (CTA per request tile)
//   lat_out_ln  h += z B + c; n = LN2(h) -> fp16 hi / lo (+ fp32 history)
#include <algorithm>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace gr {

// ---------------------------------------------------------------------------
// q_lat = LN(h) A, A given transposed (F x d) and staged in shared memory
// ---------------------------------------------------------------------------
template <int NV, int F>
__global__ void __launch_bounds__(256)
ln_qlat_kernel(const float *__restrict__ x, long long ldx, const float *__restrict__ g,
               const float *__restrict__ b, const float *__restrict__ AT, int rows, int d,
               float *__restrict__ q) {
  extern __shared__ float4 sm4[];
  const int d4 = d / 4;
  for (int i = threadIdx.x; i < F * d4; i += blockDim.x) sm4[i] = reinterpret_cast<const float4 *>(AT)[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += gridDim.x * 8) {
    const float4 *xr = reinterpret_cast<const float4 *>(x + (long long)r * ldx);
    float4 v[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      v[i] = xr[lane + 32 * i];
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    const float mean = warp_sum(s) / (float)d;
    float qq = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a0 = v[i].x - mean, a1 = v[i].y - mean, a2 = v[i].z - mean, a3 = v[i].w - mean;
      qq += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
    const float inv = 1.0f / sqrtf(warp_sum(qq) / (float)d + 1e-5f);
    float acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const float4 gg = reinterpret_cast<const float4 *>(g)[c4];
      const float4 bb = reinterpret_cast<const float4 *>(b)[c4];
      const float n0 = (v[i].x - mean) * inv * gg.x + bb.x, n1 = (v[i].y - mean) * inv * gg.y + bb.y;
      const float n2 = (v[i].z - mean) * inv * gg.z + bb.z, n3 = (v[i].w - mean) * inv * gg.w + bb.w;
#pragma unroll 8
      for (int f = 0; f < F; ++f) {
        const float4 a = sm4[f * d4 + c4];
        acc[f] = fmaf(n0, a.x, fmaf(n1, a.y, fmaf(n2, a.z, fmaf(n3, a.w, acc[f]))));
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = warp_sum(acc[f]);
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (lane == f) q[(long long)r * F + f] = acc[f];
  }
}

// ---------------------------------------------------------------------------
// z = softmax(scale q_lat F^T) F per row, over the row's request features.
// CTA = (tile of up to 8 * RPW rows of one request); its 8 warps split the
// rows (RPW per warp) and, when the tile has fewer rows, the keys; every lane
// keeps an online-softmax state per row over its keys, merged across lanes
// and key slices at the end.  Keys are staged in shared memory in chunks.
// ---------------------------------------------------------------------------
template <int F>
struct LatCfg {
  static constexpr int RPW = F <= 16 ? 4 : 2;  // rows per warp
  static constexpr int KS = F + 4;             // padded key stride (floats): conflict-free LDS.128
  static constexpr int CK = F <= 16 ? 1024 : 512;  // keys per staged chunk
};

template <int F>
__global__ void __launch_bounds__(256)
latent_attn_kernel(const float *__restrict__ q, const float *__restrict__ feats,
                   const int *__restrict__ g_row_off, const int *__restrict__ g_rows,
                   const int *__restrict__ g_ctx_off, const int *__restrict__ g_ctx_len,
                   int rows_per_cta, float scale, float *__restrict__ z) {
  using C = LatCfg<F>;
  extern __shared__ float4 sm4[];
  float *sk = reinterpret_cast<float *>(sm4);  // CK x KS keys
  float *mrg = sk + C::CK * C::KS;             // 8 x RPW x (F + 2) merge slots
  const int g = blockIdx.y;
  const int r0 = blockIdx.x * rows_per_cta;
  const int nr = min(rows_per_cta, g_rows[g] - r0);
  if (nr <= 0) return;
  const long long row0 = (long long)g_row_off[g] + r0;
  const int S = g_ctx_len[g];
  const float *kf = feats + (long long)g_ctx_off[g] * F;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warps along rows (power of two) x key slices
  int nrw = (nr + C::RPW - 1) / C::RPW;
  nrw = nrw <= 1 ? 1 : (nrw <= 2 ? 2 : (nrw <= 4 ? 4 : 8));
  const int nks = 8 / nrw;
  const int wr = warp % nrw, ks = warp / nrw;
  const int rbase = wr * C::RPW;
  float qv[C::RPW][F], m[C::RPW], l[C::RPW], zz[C::RPW][F];
#pragma unroll
  for (int j = 0; j < C::RPW; ++j) {
    const int rr = rbase + j;
#pragma unroll
    for (int f = 0; f < F; ++f)
      qv[j][f] = rr < nr ? q[(row0 + rr) * F + f] * scale : 0.f;
    m[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int f = 0; f < F; ++f) zz[j][f] = 0.f;
  }
  const int nrows_w = min(C::RPW, nr - rbase);  // rows of this warp (may be <= 0)
  for (int c0 = 0; c0 < S; c0 += C::CK) {
    const int nk = min(C::CK, S - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < nk * (F / 4); i += blockDim.x) {
      const int k = i / (F / 4), f4 = i - k * (F / 4);
      reinterpret_cast<float4 *>(sk + k * C::KS)[f4] =
          reinterpret_cast<const float4 *>(kf + (long long)(c0 + k) * F)[f4];
    }
    __syncthreads();
    if (nrows_w <= 0) continue;
    for (int k = ks * 32 + lane; k < nk; k += 32 * nks) {
      float xv[F];
#pragma unroll
      for (int f4 = 0; f4 < F / 4; ++f4) {
        const float4 t = reinterpret_cast<const float4 *>(sk + k * C::KS)[f4];
        xv[4 * f4] = t.x; xv[4 * f4 + 1] = t.y; xv[4 * f4 + 2] = t.z; xv[4 * f4 + 3] = t.w;
      }
#pragma unroll
      for (int j = 0; j < C::RPW; ++j) {
        float s = 0.f;
#pragma unroll
        for (int f = 0; f < F; ++f) s = fmaf(qv[j][f], xv[f], s);
        // online softmax: one exp (of -|s - m|) per key
        const float dlt = s - m[j];
        const float e = __expf(-fabsf(dlt));
        const bool up = dlt > 0.f;
        const float a = up ? e : 1.f, p = up ? 1.f : e;
        m[j] = up ? s : m[j];
        l[j] = fmaf(l[j], a, p);
#pragma unroll
        for (int f = 0; f < F; ++f) zz[j][f] = fmaf(zz[j][f], a, p * xv[f]);
      }
    }
  }
  // merge the lanes of each warp ...
#pragma unroll
  for (int j = 0; j < C::RPW; ++j) {
    const float M = warp_max(m[j]);
    const float w = M == -INFINITY ? 0.f : __expf(m[j] - M);
    l[j] = warp_sum(l[j] * w);
#pragma unroll
    for (int f = 0; f < F; ++f) zz[j][f] = warp_sum(zz[j][f] * w);
    m[j] = M;
  }
  // ... then the key slices of each row (through shared memory)
  __syncthreads();
  constexpr int SL = F + 2;
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < C::RPW; ++j) {
      float *o = mrg + ((ks * 8 + wr) * C::RPW + j) * SL;
      o[0] = m[j];
      o[1] = l[j];
#pragma unroll
      for (int f = 0; f < F; ++f) o[2 + f] = zz[j][f];
    }
  }
  __syncthreads();
  if (ks != 0) return;
  for (int j = 0; j < C::RPW; ++j) {
    const int rr = rbase + j;
    if (rr >= nr) break;
    float M = -INFINITY;
    for (int s = 0; s < nks; ++s) M = fmaxf(M, mrg[((s * 8 + wr) * C::RPW + j) * SL]);
    // lane f < F accumulates feature f
    float L = 0.f, Z = 0.f;
    for (int s = 0; s < nks; ++s) {
      const float *o = mrg + ((s * 8 + wr) * C::RPW + j) * SL;
      const float w = o[0] == -INFINITY ? 0.f : __expf(o[0] - M);
      L = fmaf(o[1], w, L);
      if (lane < F) Z = fmaf(o[2 + lane], w, Z);
    }
    if (lane < F) z[(row0 + rr) * F + lane] = Z / L;
  }
}

// ---------------------------------------------------------------------------
// h += z B + c (the absorbed W_v W_o projection, residual), then LN2 of the
// updated row as fp16 hi / lo (the next GEMM's A) and fp32 (self history)
// ---------------------------------------------------------------------------
template <int NV, int F>
__global__ void __launch_bounds__(256)
lat_out_ln_kernel(float *h, long long ldh, const float *__restrict__ z,
                  const float *__restrict__ B, const float *__restrict__ cvec,
                  const float *__restrict__ g, const float *__restrict__ b, int rows, int d,
                  __half *y_hi, __half *y_lo, long long ldy, float *y32, long long ld32) {
  extern __shared__ float4 sm4[];
  const int d4 = d / 4;
  for (int i = threadIdx.x; i < F * d4; i += blockDim.x) sm4[i] = reinterpret_cast<const float4 *>(B)[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += gridDim.x * 8) {
    float zr[F];
#pragma unroll
    for (int f4 = 0; f4 < F / 4; ++f4) {
      const float4 t = reinterpret_cast<const float4 *>(z + (long long)r * F)[f4];
      zr[4 * f4] = t.x; zr[4 * f4 + 1] = t.y; zr[4 * f4 + 2] = t.z; zr[4 * f4 + 3] = t.w;
    }
    float4 *hr = reinterpret_cast<float4 *>(h + (long long)r * ldh);
    float4 v[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      float4 acc = reinterpret_cast<const float4 *>(cvec)[c4];
#pragma unroll 4
      for (int f = 0; f < F; ++f) {
        const float4 bb = sm4[f * d4 + c4];
        acc.x = fmaf(zr[f], bb.x, acc.x);
        acc.y = fmaf(zr[f], bb.y, acc.y);
        acc.z = fmaf(zr[f], bb.z, acc.z);
        acc.w = fmaf(zr[f], bb.w, acc.w);
      }
      const float4 x = hr[c4];
      v[i] = make_float4(x.x + acc.x, x.y + acc.y, x.z + acc.z, x.w + acc.w);
      hr[c4] = v[i];
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    const float mean = warp_sum(s) / (float)d;
    float qq = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a0 = v[i].x - mean, a1 = v[i].y - mean, a2 = v[i].z - mean, a3 = v[i].w - mean;
      qq += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
    const float inv = 1.0f / sqrtf(warp_sum(qq) / (float)d + 1e-5f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int j = 4 * (lane + 32 * i);
      const float4 gg = *reinterpret_cast<const float4 *>(g + j);
      const float4 bb = *reinterpret_cast<const float4 *>(b + j);
      const float o[4] = {(v[i].x - mean) * inv * gg.x + bb.x, (v[i].y - mean) * inv * gg.y + bb.y,
                          (v[i].z - mean) * inv * gg.z + bb.z, (v[i].w - mean) * inv * gg.w + bb.w};
      __half hh[4], ll[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        hh[c] = __float2half_rn(o[c]);
        ll[c] = __float2half_rn(o[c] - __half2float(hh[c]));
      }
      *reinterpret_cast<uint2 *>(y_hi + (long long)r * ldy + j) = *reinterpret_cast<const uint2 *>(hh);
      *reinterpret_cast<uint2 *>(y_lo + (long long)r * ldy + j) = *reinterpret_cast<const uint2 *>(ll);
      *reinterpret_cast<float4 *>(y32 + (long long)r * ld32 + j) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

bool latent_supported(int d, int F) {
  return d % 128 == 0 && d <= 1024 && (F == 4 || F == 8 || F == 16 || F == 32);
}

static int row_grid(int rows) { return std::max(1, std::min(ceil_div(rows, 8), 148 * 3)); }

#define GR_LAT_F(M) M(4) M(8) M(16) M(32)

int ln_qlat(const float *x, long long ldx, const float *g, const float *b, const float *AT,
            int rows, int d, int F, float *q, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  if (!latent_supported(d, F)) return set_err(GR4AD_ERR_UNSUPPORTED, "latent LN: d %d F %d", d, F);
  const size_t sm = sizeof(float) * (size_t)F * d;
  const int nv = d / 128;
#define GR_LQ_NV(NV, FF)                                                                    \
  if (nv == NV) {                                                                           \
    GR_CUDA(cudaFuncSetAttribute(ln_qlat_kernel<NV, FF>,                                    \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));    \
    GR_LAUNCH(KC_LAYERNORM, st, ln_qlat_kernel<NV, FF><<<row_grid(rows), 256, sm, st>>>(     \
                                    x, ldx, g, b, AT, rows, d, q));                         \
    return GR4AD_OK;                                                                        \
  }
#define GR_LQ_F(FF)                                                                         \
  if (F == FF) {                                                                            \
    GR_LQ_NV(1, FF) GR_LQ_NV(2, FF) GR_LQ_NV(3, FF) GR_LQ_NV(4, FF) GR_LQ_NV(5, FF)          \
    GR_LQ_NV(6, FF) GR_LQ_NV(7, FF) GR_LQ_NV(8, FF)                                         \
  }
  GR_LAT_F(GR_LQ_F)
#undef GR_LQ_F
#undef GR_LQ_NV
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent LN: d %d F %d", d, F);
}

int latent_attn(const float *q, const float *feats, int F, const int *g_row_off, const int *g_rows,
                const int *g_ctx_off, const int *g_ctx_len, int n_groups, int max_group_rows,
                float scale, float *z, cudaStream_t st) {
  if (n_groups <= 0 || max_group_rows <= 0) return GR4AD_OK;
#define GR_LA_F(FF)                                                                          \
  if (F == FF) {                                                                             \
    using C = LatCfg<FF>;                                                                    \
    const int rpc = 8 * C::RPW;                                                              \
    const size_t sm = sizeof(float) * ((size_t)C::CK * C::KS + 64 * C::RPW * (FF + 2));      \
    GR_CUDA(cudaFuncSetAttribute(latent_attn_kernel<FF>,                                     \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));     \
    dim3 grid(ceil_div(max_group_rows, rpc), n_groups);                                      \
    GR_LAUNCH(KC_ATTN_GEMM, st, latent_attn_kernel<FF><<<grid, 256, sm, st>>>(                \
                                    q, feats, g_row_off, g_rows, g_ctx_off, g_ctx_len, rpc,  \
                                    scale, z));                                              \
    return GR4AD_OK;                                                                         \
  }
  GR_LAT_F(GR_LA_F)
#undef GR_LA_F
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent attention: F %d", F);
}

int lat_out_ln(float *h, long long ldh, const float *z, const float *B, const float *c,
               const float *g, const float *b, int rows, int d, int F, __half *y_hi,
               __half *y_lo, long long ldy, float *y32, long long ld32, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  if (!latent_supported(d, F)) return set_err(GR4AD_ERR_UNSUPPORTED, "latent out: d %d F %d", d, F);
  const size_t sm = sizeof(float) * (size_t)F * d;
  const int nv = d / 128;
#define GR_LO_NV(NV, FF)                                                                    \
  if (nv == NV) {                                                                           \
    GR_CUDA(cudaFuncSetAttribute(lat_out_ln_kernel<NV, FF>,                                 \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));    \
    GR_LAUNCH(KC_LAYERNORM, st, lat_out_ln_kernel<NV, FF><<<row_grid(rows), 256, sm, st>>>(  \
                                    h, ldh, z, B, c, g, b, rows, d, y_hi, y_lo, ldy, y32,    \
                                    ld32));                                                 \
    return GR4AD_OK;                                                                        \
  }
#define GR_LO_F(FF)                                                                         \
  if (F == FF) {                                                                            \
    GR_LO_NV(1, FF) GR_LO_NV(2, FF) GR_LO_NV(3, FF) GR_LO_NV(4, FF) GR_LO_NV(5, FF)          \
    GR_LO_NV(6, FF) GR_LO_NV(7, FF) GR_LO_NV(8, FF)                                         \
  }
  GR_LAT_F(GR_LO_F)
#undef GR_LO_F
#undef GR_LO_NV
  return set_err(GR4AD_ERR_UNSUPPORTED, "latent out: d %d F %d", d, F);
}

}  // namespace gr
