// Row-wise kernels and the exact per-request top-k of the beam step.
#include <algorithm>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace gr {

// ---------------------------------------------------------------------------
// LayerNorm (layers.py:38-43): warp per row
// ---------------------------------------------------------------------------
__global__ void ln_rows_kernel(const float *__restrict__ x, long long ldx, float *y,
                               long long ldy, const float *__restrict__ g,
                               const float *__restrict__ b, int rows, int d) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  const float *xr = x + (long long)w * ldx;
  float s = 0.f;
  for (int j = lane; j < d; j += 32) s += xr[j];
  float mean = warp_sum(s) / (float)d;
  float v = 0.f;
  for (int j = lane; j < d; j += 32) {
    float c = xr[j] - mean;
    v += c * c;
  }
  float var = warp_sum(v) / (float)d;
  float inv = 1.0f / sqrtf(var + 1e-5f);
  float *yr = y + (long long)w * ldy;
  for (int j = lane; j < d; j += 32) yr[j] = (xr[j] - mean) * inv * g[j] + b[j];
}

// LayerNorm writing the fp16 hi / lo split of its output (the next GEMM's A
// operand, loaded by TMA with no on-chip conversion): warp per row, the row
// in registers (d % 128 == 0, d <= 1024), float4 loads
template <int NV>
__global__ void ln_rows_split_kernel(const float *__restrict__ x, long long ldx, __half *y_hi,
                                     __half *y_lo, long long ldy, const float *__restrict__ g,
                                     const float *__restrict__ b, int rows, int d, float *y32,
                                     long long ld32) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  const float4 *xr = reinterpret_cast<const float4 *>(x + (long long)w * ldx);
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = xr[lane + 32 * i];
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = warp_sum(s) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a0 = v[i].x - mean, a1 = v[i].y - mean, a2 = v[i].z - mean, a3 = v[i].w - mean;
    q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / (float)d + 1e-5f);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = 4 * (lane + 32 * i);
    const float4 gg = *reinterpret_cast<const float4 *>(g + j);
    const float4 bb = *reinterpret_cast<const float4 *>(b + j);
    const float o[4] = {(v[i].x - mean) * inv * gg.x + bb.x, (v[i].y - mean) * inv * gg.y + bb.y,
                        (v[i].z - mean) * inv * gg.z + bb.z, (v[i].w - mean) * inv * gg.w + bb.w};
    __half h[4], l[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      h[c] = __float2half_rn(o[c]);
      l[c] = __float2half_rn(o[c] - __half2float(h[c]));
    }
    *reinterpret_cast<uint2 *>(y_hi + (long long)w * ldy + j) = *reinterpret_cast<const uint2 *>(h);
    *reinterpret_cast<uint2 *>(y_lo + (long long)w * ldy + j) = *reinterpret_cast<const uint2 *>(l);
    if (y32)  // the normalised row itself (the factored self-attention's history)
      *reinterpret_cast<float4 *>(y32 + (long long)w * ld32 + j) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

int ln_rows_split(const float *x, long long ldx, __half *y_hi, __half *y_lo, long long ldy,
                  const float *g, const float *b, int rows, int d, cudaStream_t st, float *y32,
                  long long ld32) {
  if (rows <= 0) return GR4AD_OK;
  if (d % 128 != 0 || d > 1024 || ldx % 4 != 0 || ldy % 4 != 0 || (y32 && ld32 % 4 != 0))
    return set_err(GR4AD_ERR_UNSUPPORTED, "split LayerNorm: d %d", d);
  const int nv = d / 128;
  prof_tag("ln_split rows=%d", rows);
#define GR_LNS(NV)                                                                           \
  case NV:                                                                                   \
    GR_LAUNCH(KC_LAYERNORM, st, ln_rows_split_kernel<NV><<<ceil_div(rows, 8), 256, 0, st>>>(  \
                                    x, ldx, y_hi, y_lo, ldy, g, b, rows, d, y32, ld32));     \
    return GR4AD_OK;
  switch (nv) {
    GR_LNS(1) GR_LNS(2) GR_LNS(3) GR_LNS(4) GR_LNS(5) GR_LNS(6) GR_LNS(7) GR_LNS(8)
  }
#undef GR_LNS
  return set_err(GR4AD_ERR_UNSUPPORTED, "split LayerNorm: d %d", d);
}

int ln_rows(const float *x, long long ldx, float *y, long long ldy, const float *g,
            const float *b, int rows, int d, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_LAYERNORM, st, ln_rows_kernel<<<ceil_div(rows, 8), 256, 0, st>>>(x, ldx, y, ldy, g, b, rows, d));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// softmax in place: exp(a - (max + log sum exp(a - max))) (autodiff.py:351-368)
// ---------------------------------------------------------------------------
__global__ void softmax_rows_kernel(float *s, long long ld, int rows,
                                    const int *__restrict__ row_req,
                                    const int *__restrict__ len) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  int n = len[row_req[w]];
  float *r = s + (long long)w * ld;
  float mx = -INFINITY;
  for (int j = lane; j < n; j += 32) mx = fmaxf(mx, r[j]);
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < n; j += 32) sum += expf(r[j] - mx);
  float lse = logf(warp_sum(sum)) + mx;
  for (int j = lane; j < n; j += 32) r[j] = expf(r[j] - lse);
  for (int j = n + lane; j < ld; j += 32) r[j] = 0.f;  // keeps P.V exact past S_b
}

// the same, writing P as fp16 hi / lo (the P.V GEMM's pre-split A operand)
__global__ void softmax_rows_split_kernel(const float *__restrict__ s, long long ld, __half *p_hi,
                                          __half *p_lo, int rows,
                                          const int *__restrict__ row_req,
                                          const int *__restrict__ len) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  int n = len[row_req[w]];
  const float *r = s + (long long)w * ld;
  float mx = -INFINITY;
  for (int j = lane; j < n; j += 32) mx = fmaxf(mx, r[j]);
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < n; j += 32) sum += expf(r[j] - mx);
  float lse = logf(warp_sum(sum)) + mx;
  __half *ph = p_hi + (long long)w * ld, *pl = p_lo + (long long)w * ld;
  for (int j = lane; j < n; j += 32) {
    const float x = expf(r[j] - lse);
    const __half h = __float2half_rn(x);
    ph[j] = h;
    pl[j] = __float2half_rn(x - __half2float(h));
  }
  const __half z = __float2half_rn(0.f);
  for (int j = n + lane; j < ld; j += 32) {  // keeps P.V exact past S_b
    ph[j] = z;
    pl[j] = z;
  }
}

// the same with the row in registers (ld % 128 == 0, ld <= 2048): float4 loads,
// one read of the scores
template <int NV>
__global__ void softmax_rows_split_reg_kernel(const float *__restrict__ s, long long ld,
                                              __half *p_hi, __half *p_lo, int rows,
                                              const int *__restrict__ row_req,
                                              const int *__restrict__ len) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int n = len[row_req[w]];
  const float4 *r4 = reinterpret_cast<const float4 *>(s + (long long)w * ld);
  float x[NV][4];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = 4 * (lane + 32 * i);
    const float4 v = r4[lane + 32 * i];
    x[i][0] = j < n ? v.x : -INFINITY;
    x[i][1] = j + 1 < n ? v.y : -INFINITY;
    x[i][2] = j + 2 < n ? v.z : -INFINITY;
    x[i][3] = j + 3 < n ? v.w : -INFINITY;
#pragma unroll
    for (int c = 0; c < 4; ++c) mx = fmaxf(mx, x[i][c]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) sum += x[i][c] == -INFINITY ? 0.f : expf(x[i][c] - mx);
  const float lse = logf(warp_sum(sum)) + mx;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = 4 * (lane + 32 * i);
    __half h[4], l[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float pv = x[i][c] == -INFINITY ? 0.f : expf(x[i][c] - lse);  // 0 past S_b
      h[c] = __float2half_rn(pv);
      l[c] = __float2half_rn(pv - __half2float(h[c]));
    }
    *reinterpret_cast<uint2 *>(p_hi + (long long)w * ld + j) = *reinterpret_cast<const uint2 *>(h);
    *reinterpret_cast<uint2 *>(p_lo + (long long)w * ld + j) = *reinterpret_cast<const uint2 *>(l);
  }
}

int softmax_rows_split(const float *s, long long ld, __half *p_hi, __half *p_lo, int rows,
                       const int *row_req, const int *len, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  if (ld % 128 == 0 && ld <= 2048) {
#define GR_SMS(NV)                                                                           \
  case NV:                                                                                   \
    GR_LAUNCH(KC_SOFTMAX, st, softmax_rows_split_reg_kernel<NV><<<ceil_div(rows, 8), 256, 0, st>>>( \
                                  s, ld, p_hi, p_lo, rows, row_req, len));                   \
    return GR4AD_OK;
    switch (ld / 128) {
      GR_SMS(1) GR_SMS(2) GR_SMS(3) GR_SMS(4) GR_SMS(5) GR_SMS(6) GR_SMS(7) GR_SMS(8)
      GR_SMS(9) GR_SMS(10) GR_SMS(11) GR_SMS(12) GR_SMS(13) GR_SMS(14) GR_SMS(15) GR_SMS(16)
    }
#undef GR_SMS
  }
  GR_LAUNCH(KC_SOFTMAX, st, softmax_rows_split_kernel<<<ceil_div(rows, 8), 256, 0, st>>>(
                                s, ld, p_hi, p_lo, rows, row_req, len));
  return GR4AD_OK;
}

int softmax_rows(float *s, long long ld, int rows, const int *row_req, const int *len,
                 cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_SOFTMAX, st, softmax_rows_kernel<<<ceil_div(rows, 8), 256, 0, st>>>(s, ld, rows, row_req, len));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// self-attention over the ancestor chain: block per row
// ---------------------------------------------------------------------------
constexpr int kMaxPos = GR4AD_MAX_LEVELS + 1;

__global__ void __launch_bounds__(128)
self_attn_kernel(const float *__restrict__ qkv, long long ld3, int d,
                 const int *__restrict__ anc, int stride, int hist_row0, int rows,
                 int npos_u, const int *__restrict__ npos_row, float *out,
                 long long ldo, float scale, __half *out_hi, __half *out_lo, int v_off) {
  int r = blockIdx.x;
  if (r >= rows) return;
  int g = hist_row0 + r;
  int np = npos_row ? npos_row[r] : npos_u;
  __shared__ int arow[kMaxPos];
  __shared__ float red[kMaxPos][4];
  __shared__ float p[kMaxPos];
  if (threadIdx.x < np) arow[threadIdx.x] = anc[(long long)g * stride + threadIdx.x];
  __syncthreads();
  const float *q = qkv + (long long)g * ld3;
  float acc[kMaxPos];
#pragma unroll
  for (int t = 0; t < kMaxPos; ++t) acc[t] = 0.f;
  const bool vec = (d % 4 == 0) && (ld3 % 4 == 0);  // 16-B rows: float4 gathers
  if (vec) {
    for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
      const float4 q4 = *reinterpret_cast<const float4 *>(q + j);
#pragma unroll
      for (int t = 0; t < kMaxPos; ++t)
        if (t < np) {
          const float4 k4 = *reinterpret_cast<const float4 *>(qkv + (long long)arow[t] * ld3 + d + j);
          acc[t] = fmaf(q4.x, k4.x, fmaf(q4.y, k4.y, fmaf(q4.z, k4.z, fmaf(q4.w, k4.w, acc[t]))));
        }
    }
  } else {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      float qj = q[j];
#pragma unroll
      for (int t = 0; t < kMaxPos; ++t)
        if (t < np) acc[t] = fmaf(qj, qkv[(long long)arow[t] * ld3 + d + j], acc[t]);
    }
  }
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < kMaxPos; ++t) {
    float v = warp_sum(acc[t]);
    if (lane == 0 && t < np) red[t][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float sc[kMaxPos];
    float mx = -INFINITY;
    for (int t = 0; t < np; ++t) {
      sc[t] = (red[t][0] + red[t][1] + red[t][2] + red[t][3]) * scale;
      mx = fmaxf(mx, sc[t]);
    }
    float sum = 0.f;
    for (int t = 0; t < np; ++t) sum += expf(sc[t] - mx);
    float lse = logf(sum) + mx;
    for (int t = 0; t < np; ++t) p[t] = expf(sc[t] - lse);
  }
  __syncthreads();
  if (vec && ldo % 4 == 0) {
    for (int j = threadIdx.x * 4; j < d; j += blockDim.x * 4) {
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int t = 0; t < kMaxPos; ++t)
        if (t < np) {
          const float4 v4 =
              *reinterpret_cast<const float4 *>(qkv + (long long)arow[t] * ld3 + v_off + j);
          o.x = fmaf(p[t], v4.x, o.x);
          o.y = fmaf(p[t], v4.y, o.y);
          o.z = fmaf(p[t], v4.z, o.z);
          o.w = fmaf(p[t], v4.w, o.w);
        }
      if (out_hi) {  // fp16 hi / lo split for the next GEMM's A operand
        const float oo[4] = {o.x, o.y, o.z, o.w};
        __half h[4], l[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          h[c] = __float2half_rn(oo[c]);
          l[c] = __float2half_rn(oo[c] - __half2float(h[c]));
        }
        *reinterpret_cast<uint2 *>(out_hi + (long long)r * ldo + j) = *reinterpret_cast<const uint2 *>(h);
        *reinterpret_cast<uint2 *>(out_lo + (long long)r * ldo + j) = *reinterpret_cast<const uint2 *>(l);
      } else {
        *reinterpret_cast<float4 *>(out + (long long)r * ldo + j) = o;
      }
    }
    return;
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float o = 0.f;
    for (int t = 0; t < np; ++t) o = fmaf(p[t], qkv[(long long)arow[t] * ld3 + v_off + j], o);
    out[(long long)r * ldo + j] = o;
  }
}

// Warp per row for d % 128 == 0, d <= 1024 (NV = d / 128 float4 per lane):
// q in registers, every ancestor's k / v row gathered with NV independent
// 16-B loads per lane, scores and softmax in registers -- no block barrier.
// HS: the factored history keeps n (= k = v) as fp16 hi / lo halves after
// q' ([q' fp32 | n hi | n lo], the next GEMM reads the same halves), and n
// is rebuilt as hi + lo (~2^-22 relative)
template <int NV, bool HS>
__global__ void __launch_bounds__(256)
self_attn_warp_kernel(const float *__restrict__ qkv, long long ld3, int d,
                      const int *__restrict__ anc, int stride, int hist_row0, int rows,
                      int npos_u, const int *__restrict__ npos_row, float *out, long long ldo,
                      float scale, __half *out_hi, __half *out_lo, int v_off) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int g = hist_row0 + r;
  const int np = npos_row ? npos_row[r] : npos_u;
  const float4 *q4 = reinterpret_cast<const float4 *>(qkv + (long long)g * ld3);
  float4 q[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) q[i] = q4[lane + 32 * i];
  // element block i of history row `row` at column offset `off` (k: d, v: v_off)
  auto hrow = [&](long long row, int off, int i) -> float4 {
    if constexpr (HS) {
      const __half *hb = reinterpret_cast<const __half *>(qkv + row * ld3) + 2 * d;
      const int j = 4 * (lane + 32 * i);
      const uint2 h = *reinterpret_cast<const uint2 *>(hb + j);
      const uint2 l = *reinterpret_cast<const uint2 *>(hb + d + j);
      const float2 h0 = __half22float2(*reinterpret_cast<const __half2 *>(&h.x));
      const float2 h1 = __half22float2(*reinterpret_cast<const __half2 *>(&h.y));
      const float2 l0 = __half22float2(*reinterpret_cast<const __half2 *>(&l.x));
      const float2 l1 = __half22float2(*reinterpret_cast<const __half2 *>(&l.y));
      return make_float4(h0.x + l0.x, h0.y + l0.y, h1.x + l1.x, h1.y + l1.y);
    } else {
      return reinterpret_cast<const float4 *>(qkv + row * ld3 + off)[lane + 32 * i];
    }
  };
  float4 o[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) o[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (HS && v_off == d) {
    // factored attention: keys and values are the same history rows n_j, so
    // one pass reads each ancestor once (online softmax: running max m and
    // sum l, the accumulator rescaled when the max moves)
    float m = -INFINITY, l = 0.f;
#pragma unroll
    for (int t = 0; t < kMaxPos; ++t) {
      if (t < np) {
        const long long row = anc[(long long)g * stride + t];
        float4 k[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) k[i] = hrow(row, d, i);
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i)
          acc = fmaf(q[i].x, k[i].x, fmaf(q[i].y, k[i].y, fmaf(q[i].z, k[i].z, fmaf(q[i].w, k[i].w, acc))));
        const float s = warp_sum(acc) * scale;
        const float mn = fmaxf(m, s);
        const float cs = expf(m - mn), ps = expf(s - mn);  // (m = -inf: cs = 0)
        l = l * cs + ps;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          o[i].x = fmaf(ps, k[i].x, o[i].x * cs);
          o[i].y = fmaf(ps, k[i].y, o[i].y * cs);
          o[i].z = fmaf(ps, k[i].z, o[i].z * cs);
          o[i].w = fmaf(ps, k[i].w, o[i].w * cs);
        }
        m = mn;
      }
    }
    const float inv = 1.f / l;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      o[i].x *= inv;
      o[i].y *= inv;
      o[i].z *= inv;
      o[i].w *= inv;
    }
  } else {
  float sc[kMaxPos];
  float mx = -INFINITY;
#pragma unroll
  for (int t = 0; t < kMaxPos; ++t) {
    sc[t] = -INFINITY;
    if (t < np) {
      const long long row = anc[(long long)g * stride + t];
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float4 k = hrow(row, d, i);
        acc = fmaf(q[i].x, k.x, fmaf(q[i].y, k.y, fmaf(q[i].z, k.z, fmaf(q[i].w, k.w, acc))));
      }
      sc[t] = warp_sum(acc) * scale;
      mx = fmaxf(mx, sc[t]);
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int t = 0; t < kMaxPos; ++t)
    if (t < np) sum += expf(sc[t] - mx);
  const float lse = logf(sum) + mx;
#pragma unroll
  for (int t = 0; t < kMaxPos; ++t) {
    if (t < np) {
      const float pt = expf(sc[t] - lse);
      const long long row = anc[(long long)g * stride + t];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const float4 v = hrow(row, v_off, i);
        o[i].x = fmaf(pt, v.x, o[i].x);
        o[i].y = fmaf(pt, v.y, o[i].y);
        o[i].z = fmaf(pt, v.z, o[i].z);
        o[i].w = fmaf(pt, v.w, o[i].w);
      }
    }
  }
  }  // (two-pass: separate key / value rows)
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = 4 * (lane + 32 * i);
    if (out_hi) {  // fp16 hi / lo split for the next GEMM's A operand
      const float oo[4] = {o[i].x, o[i].y, o[i].z, o[i].w};
      __half h[4], l[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        h[c] = __float2half_rn(oo[c]);
        l[c] = __float2half_rn(oo[c] - __half2float(h[c]));
      }
      *reinterpret_cast<uint2 *>(out_hi + (long long)r * ldo + j) = *reinterpret_cast<const uint2 *>(h);
      *reinterpret_cast<uint2 *>(out_lo + (long long)r * ldo + j) = *reinterpret_cast<const uint2 *>(l);
    } else {
      *reinterpret_cast<float4 *>(out + (long long)r * ldo + j) = o[i];
    }
  }
}

int self_attn(const float *qkv, long long ld3, int d, const int *anc, int anc_stride,
              int hist_row0, int rows, int npos_uniform, const int *npos_row,
              float *out, long long ldo, cudaStream_t st, __half *out_hi, __half *out_lo,
              int v_off, bool hist_split) {
  if (rows <= 0) return GR4AD_OK;
  if (v_off < 0) v_off = 2 * d;
  if (out_hi && (d % 4 != 0 || ld3 % 4 != 0 || ldo % 4 != 0))
    return set_err(GR4AD_ERR_UNSUPPORTED, "split self-attention output: d %d", d);
  const float scale = 1.0f / sqrtf((float)d);
  prof_tag("self_attn rows=%d", rows);
  const bool warp_ok = d % 128 == 0 && d <= 1024 && ld3 % 4 == 0 && ldo % 4 == 0;
  if (hist_split && (!warp_ok || v_off != d))
    return set_err(GR4AD_ERR_UNSUPPORTED, "split self-attention history: d %d", d);
  if (warp_ok) {
#define GR_SAW(NV)                                                                           \
  case NV:                                                                                   \
    if (hist_split)                                                                          \
      GR_LAUNCH(KC_SELF_ATTN, st,                                                            \
                self_attn_warp_kernel<NV, true><<<ceil_div(rows, 8), 256, 0, st>>>(          \
                    qkv, ld3, d, anc, anc_stride, hist_row0, rows, npos_uniform, npos_row,   \
                    out, ldo, scale, out_hi, out_lo, v_off));                                \
    else                                                                                     \
      GR_LAUNCH(KC_SELF_ATTN, st,                                                            \
                self_attn_warp_kernel<NV, false><<<ceil_div(rows, 8), 256, 0, st>>>(         \
                    qkv, ld3, d, anc, anc_stride, hist_row0, rows, npos_uniform, npos_row,   \
                    out, ldo, scale, out_hi, out_lo, v_off));                                \
    return GR4AD_OK;
    switch (d / 128) {
      GR_SAW(1) GR_SAW(2) GR_SAW(3) GR_SAW(4) GR_SAW(5) GR_SAW(6) GR_SAW(7) GR_SAW(8)
    }
#undef GR_SAW
  }
  GR_LAUNCH(KC_SELF_ATTN, st, self_attn_kernel<<<rows, 128, 0, st>>>(qkv, ld3, d, anc, anc_stride, hist_row0, rows,
                                         npos_uniform, npos_row, out, ldo,
                                         1.0f / sqrtf((float)d), out_hi, out_lo, v_off));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// level input (beam.py:180-191)
// ---------------------------------------------------------------------------
__global__ void level_input_kernel(int t, int rows, int d, const float *__restrict__ bos,
                                   const float *__restrict__ emb_prev,
                                   const int *__restrict__ tok,
                                   const float *__restrict__ pos_t, float *U, float *H,
                                   __half *Uh, __half *Ul) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * d) return;
  int r = (int)(i / d), j = (int)(i - (long long)r * d);
  float s = (t == 0) ? bos[j] : emb_prev[(long long)tok[r] * d + j];
  if (U) U[(long long)r * 2 * d + d + j] = s;
  if (Uh) {  // the fuse GEMMs' pre-split A (same split as on chip)
    const __half h = __float2half_rn(s);
    Uh[(long long)r * 2 * d + d + j] = h;
    Ul[(long long)r * 2 * d + d + j] = __float2half_rn(s - __half2float(h));
  }
  if (H) H[(long long)r * d + j] = s + pos_t[j];
}

// the split-only gather (the fuse's pre-split A): four columns per thread,
// float4 loads and 8-B fp16 stores
__global__ void level_input_split4_kernel(int t, int rows, int d, const float *__restrict__ bos,
                                          const float *__restrict__ emb_prev,
                                          const int *__restrict__ tok, __half *Uh, __half *Ul) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int d4 = d / 4;
  if (i >= (long long)rows * d4) return;
  const int r = (int)(i / d4), j = (int)(i - (long long)r * d4) * 4;
  const float4 s = *reinterpret_cast<const float4 *>(
      (t == 0) ? bos + j : emb_prev + (long long)tok[r] * d + j);
  const float sv[4] = {s.x, s.y, s.z, s.w};
  __align__(8) __half hq[4], lq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    hq[q] = __float2half_rn(sv[q]);
    lq[q] = __float2half_rn(sv[q] - __half2float(hq[q]));
  }
  const long long o = (long long)r * 2 * d + d + j;
  *reinterpret_cast<uint2 *>(Uh + o) = *reinterpret_cast<const uint2 *>(hq);
  *reinterpret_cast<uint2 *>(Ul + o) = *reinterpret_cast<const uint2 *>(lq);
}

// the fuse's gathered inputs (layers.py:129-133 with the token-side
// products tabulated): H = (s W_f[d:2d])[tok], (Uh, Ul) = split of
// m_t[req] * (s W_g)[tok] (ld d); four columns per thread
__global__ void fuse_gather_kernel(int t, int rows, int d, const int *__restrict__ tok,
                                   const float *__restrict__ tab, int n_tok,
                                   const float *__restrict__ m, long long m_ld,
                                   const int *__restrict__ row_req, float *H, __half *Uh,
                                   __half *Ul) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int d4 = d / 4;
  if (i >= (long long)rows * d4) return;
  const int r = (int)(i / d4), j = (int)(i - (long long)r * d4) * 4;
  const long long k = t == 0 ? 0 : tok[r];
  const float4 g = *reinterpret_cast<const float4 *>(tab + k * d + j);
  const float4 f = *reinterpret_cast<const float4 *>(tab + ((long long)n_tok + k) * d + j);
  const float4 mm = *reinterpret_cast<const float4 *>(m + (long long)row_req[r] * m_ld + j);
  *reinterpret_cast<float4 *>(H + (long long)r * d + j) = f;
  const float gv[4] = {mm.x * g.x, mm.y * g.y, mm.z * g.z, mm.w * g.w};
  __align__(8) __half hq[4], lq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    hq[q] = __float2half_rn(gv[q]);
    lq[q] = __float2half_rn(gv[q] - __half2float(hq[q]));
  }
  *reinterpret_cast<uint2 *>(Uh + (long long)r * d + j) = *reinterpret_cast<const uint2 *>(hq);
  *reinterpret_cast<uint2 *>(Ul + (long long)r * d + j) = *reinterpret_cast<const uint2 *>(lq);
}

int fuse_gather(int t, int rows, int d, const int *tok, const float *tab, int n_tok,
                const float *m, long long m_ld, const int *row_req, float *H, __half *Uh,
                __half *Ul, cudaStream_t st) {
  const long long n4 = (long long)rows * (d / 4);
  if (n4 <= 0) return GR4AD_OK;
  if (d % 4 != 0) return set_err(GR4AD_ERR_UNSUPPORTED, "fuse gather: d %d", d);
  GR_LAUNCH(KC_SMALL, st, fuse_gather_kernel<<<ceil_div(n4, 256), 256, 0, st>>>(
                              t, rows, d, tok, tab, n_tok, m, m_ld, row_req, H, Uh, Ul));
  return GR4AD_OK;
}

int level_input(int t, int rows, int d, const float *bos, const float *emb_prev,
                const int *tok, const float *pos_t, float *U, float *H,
                cudaStream_t st, __half *Uh, __half *Ul) {
  long long n = (long long)rows * d;
  if (n <= 0) return GR4AD_OK;
  if (Uh && !U && !H && d % 4 == 0) {
    const long long n4 = n / 4;
    GR_LAUNCH(KC_SMALL, st, level_input_split4_kernel<<<ceil_div(n4, 256), 256, 0, st>>>(
                                t, rows, d, bos, emb_prev, tok, Uh, Ul));
    return GR4AD_OK;
  }
  GR_LAUNCH(KC_SMALL, st, level_input_kernel<<<ceil_div(n, 256), 256, 0, st>>>(t, rows, d, bos, emb_prev, tok,
                                                       pos_t, U, H, Uh, Ul));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// row (max, log sum exp) (beam.py:92-95): block per row
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
row_lse_kernel(const float *__restrict__ logits, long long ld, int rows, int V,
               float2 *info) {
  int r = blockIdx.x;
  if (r >= rows) return;
  const float *x = logits + (long long)r * ld;
  __shared__ float red[4];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < V; j += blockDim.x) mx = fmaxf(mx, x[j]);
  mx = warp_max(mx);
  if (lane == 0) red[wid] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float s = 0.f;
  for (int j = threadIdx.x; j < V; j += blockDim.x) s += expf(x[j] - mx);
  s = warp_sum(s);
  if (lane == 0) red[wid] = s;
  __syncthreads();
  if (threadIdx.x == 0) info[r] = make_float2(mx, logf(red[0] + red[1] + red[2] + red[3]));
}

// (max, log sum exp) per row from the logits GEMM's per-128-column partials
// (EPI_STORE_LSE): warp per row
__global__ void lse_merge_kernel(const float4 *__restrict__ part, int n_part, int rows,
                                 float2 *info) {
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  float m = -INFINITY;
  for (int j = lane; j < n_part; j += 32) m = fmaxf(m, part[(long long)r * n_part + j].x);
  m = warp_max(m);
  float s = 0.f;
  for (int j = lane; j < n_part; j += 32) {
    const float4 p2 = part[(long long)r * n_part + j];
    if (p2.x != -INFINITY) s += p2.y * expf(p2.x - m);
  }
  s = warp_sum(s);
  if (lane == 0) info[r] = make_float2(m, logf(s));
}

int lse_merge(const float4 *part, int n_part, int rows, float2 *info, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_ROW_LSE, st, lse_merge_kernel<<<(rows + 7) / 8, 256, 0, st>>>(part, n_part, rows, info));
  return GR4AD_OK;
}

int row_lse(const float *logits, long long ld, int rows, int V, float2 *info,
            cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_ROW_LSE, st, row_lse_kernel<<<rows, 128, 0, st>>>(logits, ld, rows, V, info));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// valid-SID prefix mask: block per row
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound64(const long long *a, int n, long long key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void mask_rows_kernel(float *logits, long long ld, int rows, int V,
                                 const long long *__restrict__ prefix,
                                 const long long *__restrict__ valid, int n_valid) {
  extern __shared__ unsigned bits[];
  int r = blockIdx.x;
  if (r >= rows) return;
  int words = (V + 31) / 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) bits[i] = 0u;
  __shared__ int lo, hi;
  long long base = prefix[r] * (long long)V;
  if (threadIdx.x == 0) {
    lo = lower_bound64(valid, n_valid, base);
    hi = lower_bound64(valid, n_valid, base + V);
  }
  __syncthreads();
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    int v = (int)(valid[i] - base);
    atomicOr(&bits[v >> 5], 1u << (v & 31));
  }
  __syncthreads();
  float *x = logits + (long long)r * ld;
  for (int v = threadIdx.x; v < V; v += blockDim.x)
    if (!((bits[v >> 5] >> (v & 31)) & 1u)) x[v] = -INFINITY;
}

// CSR row pointers of sorted (t+1)-prefix keys grouped by their t-prefix P =
// key / V: rp[P] = lower_bound(keys, P V) for P in [0, n_prefix]
__global__ void csr_rows_kernel(const long long *__restrict__ keys, int n, int V,
                                long long n_prefix, int *rp) {
  const long long P = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (P > n_prefix) return;
  rp[P] = lower_bound64(keys, n, P * V);
}

int csr_rows(const long long *keys, int n, int V, long long n_prefix, int *rp,
             cudaStream_t st) {
  const long long m = n_prefix + 1;
  GR_LAUNCH(KC_SMALL, st, csr_rows_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(
                              keys, n, V, n_prefix, rp));
  return GR4AD_OK;
}

int mask_rows(float *logits, long long ld, int rows, int V, const long long *prefix,
              const long long *valid, int n_valid, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  size_t sm = sizeof(unsigned) * ((V + 31) / 32);
  GR_LAUNCH(KC_SMALL, st, mask_rows_kernel<<<rows, 256, sm, st>>>(logits, ld, rows, V, prefix, valid, n_valid));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// exact per-request top-k under (-score, row, token) (beam.py:30-89)
//
// One CTA per request.  Keys are order-preserving uint32 images of the fp32
// candidate score cum[r] + (logit - max_r) - log_sum_r.  Three radix passes
// (11/11/10 bits) find the exact k-th key T and how many candidates equal
// to T must be kept; a collect pass keeps every key > T and the
// lowest-(row, token) keys == T; a bitonic sort of the k survivors on
// (key desc, flat index asc) gives the reference order.  When the request's
// candidate set fits in shared memory the keys are cached there after the
// first pass.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned warp_sum_u(unsigned v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 512 threads, two CTAs per SM (the uncached instantiation's 72 KB of shared
// memory allows it): a batch's requests stream their logits in one wave
// instead of 1.7 waves of one 1024-thread CTA per SM
constexpr int kSelThreads = 512;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kCacheKeys = 28 * 1024;  // 112 KB of cached keys

struct SelCtx {
  const float *logits;
  long long ld;
  const float2 *rowinfo;
  const float *cum;
  int row0, n_rows, V, hist0;
};

__device__ __forceinline__ uint32_t sel_key(const SelCtx &c, int r, int v, float cr,
                                            float2 ri) {
  float lg = c.logits[(long long)(c.row0 + r) * c.ld + v];
  float lp = c.rowinfo ? ((lg - ri.x) - ri.y) : lg;
  return f2ord(cr + lp);
}

template <bool CACHE>
__device__ void sel_pass_hist(const SelCtx &c, uint32_t *keys, unsigned *hist, int shift,
                              uint32_t pmask, uint32_t prefix, uint32_t bmask) {
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int cur = -1;
  unsigned cnt = 0;
  if (CACHE) {  // keys prefilled in shared memory: flat over all threads
    const int n = c.n_rows * c.V;
    for (int fi = threadIdx.x; fi < n; fi += kSelThreads) {
      const uint32_t u = keys[fi];
      if ((u & pmask) == prefix) {
        int bin = (int)((u >> shift) & bmask);
        if (bin == cur) {
          ++cnt;
        } else {
          if (cnt) atomicAdd(&hist[cur], cnt);
          cur = bin;
          cnt = 1;
        }
      }
    }
    if (cnt) atomicAdd(&hist[cur], cnt);
    return;
  }
  for (int r = wid; r < c.n_rows; r += kSelWarps) {
    float cr = 0.f;
    float2 ri = make_float2(0.f, 0.f);
    if (!CACHE || shift == 21) {
      cr = c.cum[c.hist0 + c.row0 + r];
      if (c.rowinfo) ri = c.rowinfo[c.row0 + r];
    }
    for (int v = lane; v < c.V; v += 32) {
      uint32_t u;
      long long fi = (long long)r * c.V + v;
      if (CACHE && shift != 21) {
        u = keys[fi];
      } else {
        u = sel_key(c, r, v, cr, ri);
        if (CACHE) keys[fi] = u;
      }
      if ((u & pmask) == prefix) {
        int bin = (int)((u >> shift) & bmask);
        if (bin == cur) {
          ++cnt;
        } else {
          if (cnt) atomicAdd(&hist[cur], cnt);
          cur = bin;
          cnt = 1;
        }
      }
    }
  }
  if (cnt) atomicAdd(&hist[cur], cnt);
}

// find bin b with (count of bins above b) < need <= (count above) + hist[b];
// returns b and writes the count above into *above.
__device__ int sel_find_bin(unsigned *hist, int nbins, unsigned need, unsigned *above_out,
                            unsigned *scan) {
  // suffix sums over bins (descending): scan[i] = sum_{j > i} hist[j]
  int tid = threadIdx.x;
  int per = (nbins + kSelThreads - 1) / kSelThreads;  // 2 for 2048 bins
  unsigned local = 0;
  for (int i = 0; i < per; ++i) {
    int b = nbins - 1 - (tid * per + i);
    if (b >= 0) local += hist[b];
  }
  // exclusive scan of `local` over threads in order (block-wide)
  int lane = tid & 31, wid = tid >> 5;
  unsigned x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __shared__ unsigned wsum[kSelWarps];
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned s = lane < kSelWarps ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kSelWarps) wsum[lane] = s;  // inclusive
  }
  __syncthreads();
  unsigned excl = x - local + (wid > 0 ? wsum[wid - 1] : 0u);
  unsigned run = excl;
  for (int i = 0; i < per; ++i) {
    int b = nbins - 1 - (tid * per + i);
    if (b >= 0) {
      unsigned h = hist[b];
      if (run < need && need <= run + h) {
        scan[0] = (unsigned)b;
        scan[1] = run;
      }
      run += h;
    }
  }
  __syncthreads();
  *above_out = scan[1];
  int b = (int)scan[0];
  __syncthreads();
  return b;
}

template <bool CACHE>
__global__ void __launch_bounds__(kSelThreads, 2) topk_select_kernel(SelectArgs a, int u_rows, int u_k) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long *sbuf = reinterpret_cast<unsigned long long *>(smem);  // GR4AD_MAX_BEAM
  unsigned *hist = reinterpret_cast<unsigned *>(sbuf + GR4AD_MAX_BEAM);    // 2048
  uint32_t *keys = reinterpret_cast<uint32_t *>(hist + 2048);              // kCacheKeys
  __shared__ unsigned scan[2];
  __shared__ unsigned s_gt_pos, s_nfin;

  const int b = blockIdx.x;
  SelCtx c;
  c.logits = a.logits;
  c.ld = a.ld;
  c.rowinfo = a.rowinfo;
  c.cum = a.cum;
  c.V = a.V;
  c.hist0 = a.hist_off;
  c.row0 = a.row_off ? a.row_off[b] : b * u_rows;
  c.n_rows = a.live ? a.live[b] : u_rows;
  const long long n_cand = (long long)c.n_rows * c.V;
  int want = a.eff ? a.eff[b] : u_k;
  const int k = (int)min((long long)want, n_cand);
  const int tid = threadIdx.x;

  int wid = tid >> 5, lane = tid & 31;
  // ---- (a) one-pass window selection -------------------------------------
  // Candidate scores are cum_r + logp <= Rs := max_r cum_r.  Bin each by
  // min((Rs - s) * scale, 2047) (monotone in s; 2048 bins over ln V + 4 score
  // units); every candidate in a bin below the k-th candidate's bin is in
  // the top-k, and that bin is collected whole, so one histogram pass and
  // one collect pass feed an exact (key, index) sort.  Radix passes are the
  // fallback when the window overflows.
  bool window = false;
  int n_sort = k;
  __shared__ float s_red[kSelWarps];
  if (k > 0) {
    float mc = -INFINITY;
    for (int r = tid; r < c.n_rows; r += kSelThreads) mc = fmaxf(mc, c.cum[c.hist0 + c.row0 + r]);
    mc = warp_max(mc);
    if (lane == 0) s_red[wid] = mc;
    for (int i = tid; i < 2048; i += kSelThreads) hist[i] = 0u;
    __syncthreads();
    float Rs = -INFINITY;
    for (int w = 0; w < kSelWarps; ++w) Rs = fmaxf(Rs, s_red[w]);
    const float scale = 2048.0f / (logf((float)max(c.V, 2)) + 4.0f);
    auto sbin = [&](float s) -> unsigned { return (unsigned)fminf((Rs - s) * scale, 2047.0f); };
    if (CACHE) {
      // every candidate key once into shared memory, spread over all threads
      // (a level with few rows -- level 0 has one -- would otherwise run on
      // one warp): coalesced loads, later passes read only shared memory
      const int n = (int)n_cand;
      for (int fi = tid; fi < n; fi += kSelThreads) {
        const int r = fi / c.V;
        const float cr = c.cum[c.hist0 + c.row0 + r];
        const float2 ri = c.rowinfo ? c.rowinfo[c.row0 + r] : make_float2(0.f, 0.f);
        keys[fi] = sel_key(c, r, fi - r * c.V, cr, ri);
      }
      __syncthreads();
    }
    // 16-B rows: float4 loads, four candidates per lane and load
    const bool vec4 = !CACHE && c.V % 4 == 0 && c.ld % 4 == 0;
    // attempt 0: window bin from the logits GEMM epilogue's per-64-column maxima
    // proxies (every proxy is a real candidate with the identical score
    // expression, so the k-th best proxy's bin bounds the k-th best
    // candidate's): no histogram pass over the logits.  Attempt 1: the
    // histogram pass.  A window wider than the sort buffer falls through.
    for (int attempt = (a.proxies && !CACHE) ? 0 : 1; attempt < 2 && !window; ++attempt) {
      int cur = -1;
      unsigned cnt = 0;
      if (attempt == 0) {
        if (tid == 0) s_nfin = 0;
        __syncthreads();
        unsigned nprox = 0;
        for (int r = wid; r < c.n_rows; r += kSelWarps) {
          const float cr = c.cum[c.hist0 + c.row0 + r];
          const float2 ri = c.rowinfo[c.row0 + r];
          for (int j = lane; j < a.proxy_ld; j += 32) {
            const float4 pr = a.proxies[(long long)(c.row0 + r) * a.proxy_ld + j];
            const float pv[2] = {pr.z, pr.w};
#pragma unroll
            for (int q = 0; q < 2; ++q)
              if (pv[q] > -INFINITY) {
                const int bin = (int)sbin(cr + ((pv[q] - ri.x) - ri.y));
                ++nprox;
                if (bin == cur) {
                  ++cnt;
                } else {
                  if (cnt) atomicAdd(&hist[cur], cnt);
                  cur = bin;
                  cnt = 1;
                }
              }
          }
        }
        nprox = warp_sum_u(nprox);
        if (lane == 0 && nprox) atomicAdd(&s_nfin, nprox);
      } else if (CACHE) {
        const int n = (int)n_cand;
        for (int fi = tid; fi < n; fi += kSelThreads) {
          const int bin = (int)sbin(ord2f(keys[fi]));
          if (bin == cur) {
            ++cnt;
          } else {
            if (cnt) atomicAdd(&hist[cur], cnt);
            cur = bin;
            cnt = 1;
          }
        }
      } else {
        for (int r = wid; r < c.n_rows; r += kSelWarps) {
          const float cr = c.cum[c.hist0 + c.row0 + r];
          const float2 ri = c.rowinfo ? c.rowinfo[c.row0 + r] : make_float2(0.f, 0.f);
          if (vec4) {
            const float4 *row4 =
                reinterpret_cast<const float4 *>(c.logits + (long long)(c.row0 + r) * c.ld);
#pragma unroll 4
            for (int v4 = lane; v4 < c.V / 4; v4 += 32) {
              const float4 l4 = row4[v4];
              const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float s = cr + (c.rowinfo ? ((lv[q] - ri.x) - ri.y) : lv[q]);
                const int bin = (int)sbin(s);
                if (bin == cur) {
                  ++cnt;
                } else {
                  if (cnt) atomicAdd(&hist[cur], cnt);
                  cur = bin;
                  cnt = 1;
                }
              }
            }
            continue;
          }
          for (int v = lane; v < c.V; v += 32) {
            const float lg = c.logits[(long long)(c.row0 + r) * c.ld + v];
            const float s = cr + (c.rowinfo ? ((lg - ri.x) - ri.y) : lg);
            if (CACHE) keys[(long long)r * c.V + v] = f2ord(s);
            const int bin = (int)sbin(s);
            if (bin == cur) {
              ++cnt;
            } else {
              if (cnt) atomicAdd(&hist[cur], cnt);
              cur = bin;
              cnt = 1;
            }
          }
        }
      }
      if (cnt) atomicAdd(&hist[cur], cnt);
      __syncthreads();
      if (attempt == 0 && s_nfin < (unsigned)k) {  // too few proxies (uniform)
        for (int i = tid; i < 2048; i += kSelThreads) hist[i] = 0u;
        __syncthreads();
        continue;
      }
      for (int i = tid; i < 1024; i += kSelThreads) {  // mirror: sel_find_bin scans from the top
        unsigned x = hist[i], y = hist[2047 - i];
        hist[i] = y;
        hist[2047 - i] = x;
      }
      __syncthreads();
      unsigned above;
      const int rb = sel_find_bin(hist, 2048, (unsigned)k, &above, scan);
      const int wb = 2047 - rb;
      const unsigned cnt_le = above + hist[rb];
      __syncthreads();
      for (int i = tid; i < 2048; i += kSelThreads) hist[i] = 0u;
      if (tid == 0) s_gt_pos = 0;
      __syncthreads();
      if (wb == 2047 || (attempt == 1 && cnt_le > (unsigned)GR4AD_MAX_BEAM)) continue;
      if (CACHE) {
        const int n = (int)n_cand;
        for (int f0 = wid * 32; f0 < n; f0 += kSelThreads) {
          const int fi = f0 + lane;
          const uint32_t u = fi < n ? keys[fi] : 0u;
          const bool take = fi < n && sbin(ord2f(u)) <= (unsigned)wb;
          const unsigned m = __ballot_sync(0xffffffffu, take);
          if (m) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&s_gt_pos, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
            if (take && pos < (unsigned)GR4AD_MAX_BEAM)
              sbuf[pos] = ((unsigned long long)u << 32) | (0xFFFFFFFFu - (unsigned)fi);
          }
        }
      }
      for (int r = wid; r < c.n_rows && !CACHE; r += kSelWarps) {
        const float cr = c.cum[c.hist0 + c.row0 + r];
        const float2 ri = c.rowinfo ? c.rowinfo[c.row0 + r] : make_float2(0.f, 0.f);
        if (vec4 && a.proxies) {
          // block-skipping collect: the proxies are the exact maxima of the
          // row's 64-column blocks (same fp32 values the logits hold), so a
          // block whose maximum is outside the window holds no window
          // candidate and is never read -- only the few blocks around the
          // cut leave HBM
          const float *row = c.logits + (long long)(c.row0 + r) * c.ld;
          for (int j0 = 0; j0 < a.proxy_ld; j0 += 32) {
            const int j = j0 + lane;
            bool q1 = false, q2 = false;
            if (j < a.proxy_ld) {
              const float4 pr = a.proxies[(long long)(c.row0 + r) * a.proxy_ld + j];
              q1 = pr.z > -INFINITY && sbin(cr + ((pr.z - ri.x) - ri.y)) <= (unsigned)wb;
              q2 = pr.w > -INFINITY && sbin(cr + ((pr.w - ri.x) - ri.y)) <= (unsigned)wb;
            }
            unsigned m1 = __ballot_sync(0xffffffffu, q1), m2 = __ballot_sync(0xffffffffu, q2);
            while (m1 | m2) {
              int blk;  // 64-column block index (2 per proxy entry)
              if (m1 && (!m2 || __ffs(m1) <= __ffs(m2))) {
                const int b = __ffs(m1) - 1;
                m1 &= m1 - 1;
                blk = 2 * (j0 + b);
              } else {
                const int b = __ffs(m2) - 1;
                m2 &= m2 - 1;
                blk = 2 * (j0 + b) + 1;
              }
              const int v0 = 64 * blk + 2 * lane;
              float2 l2 = make_float2(-INFINITY, -INFINITY);
              if (v0 + 1 < c.V) l2 = *reinterpret_cast<const float2 *>(row + v0);
              else if (v0 < c.V) l2.x = row[v0];
              const float sv[2] = {cr + ((l2.x - ri.x) - ri.y), cr + ((l2.y - ri.x) - ri.y)};
              unsigned pm = 0;
#pragma unroll
              for (int q = 0; q < 2; ++q)
                if (v0 + q < c.V && sbin(sv[q]) <= (unsigned)wb) pm |= 1u << q;
              if (__any_sync(0xffffffffu, pm != 0)) {
                const unsigned np = __popc(pm);
                unsigned incl = np;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                  if (lane >= o) incl += y;
                }
                unsigned base = 0;
                if (lane == 31) base = atomicAdd(&s_gt_pos, incl);
                base = __shfl_sync(0xffffffffu, base, 31) + incl - np;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                  const bool take = (pm >> q) & 1u;
                  const unsigned fi = (unsigned)((long long)r * c.V + v0 + q);
                  const unsigned long long e =
                      ((unsigned long long)f2ord(sv[q]) << 32) | (0xFFFFFFFFu - fi);
                  if (take && base < (unsigned)GR4AD_MAX_BEAM) sbuf[base] = e;
                  base += take ? 1u : 0u;
                }
              }
            }
          }
          continue;
        }
        if (vec4) {
          const float4 *row4 =
              reinterpret_cast<const float4 *>(c.logits + (long long)(c.row0 + r) * c.ld);
#pragma unroll 4
          for (int v40 = 0; v40 < c.V / 4; v40 += 32) {
            const int v4 = v40 + lane;
            float4 l4 = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            if (v4 < c.V / 4) l4 = row4[v4];
            const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
            unsigned pm = 0;
            float sv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              sv[q] = cr + (c.rowinfo ? ((lv[q] - ri.x) - ri.y) : lv[q]);
              if (v4 < c.V / 4 && sbin(sv[q]) <= (unsigned)wb) pm |= 1u << q;
            }
            if (__any_sync(0xffffffffu, pm != 0)) {
              const unsigned np = __popc(pm);
              unsigned incl = np;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
              }
              unsigned base = 0;
              if (lane == 31) base = atomicAdd(&s_gt_pos, incl);
              base = __shfl_sync(0xffffffffu, base, 31) + incl - np;
#pragma unroll
              for (int q = 0; q < 4; ++q) {  // branch-free: predicated stores
                const bool take = (pm >> q) & 1u;
                const unsigned fi = (unsigned)((long long)r * c.V + 4 * v4 + q);
                const unsigned long long e =
                    ((unsigned long long)f2ord(sv[q]) << 32) | (0xFFFFFFFFu - fi);
                if (take && base < (unsigned)GR4AD_MAX_BEAM) sbuf[base] = e;  // (overflow: counted)
                base += take ? 1u : 0u;
              }
            }
          }
          continue;
        }
        for (int v0 = 0; v0 < c.V; v0 += 32) {
          const int v = v0 + lane;
          float s = -INFINITY;
          if (v < c.V) {
            if (CACHE) {
              s = ord2f(keys[(long long)r * c.V + v]);
            } else {
              const float lg = c.logits[(long long)(c.row0 + r) * c.ld + v];
              s = cr + (c.rowinfo ? ((lg - ri.x) - ri.y) : lg);
            }
          }
          const bool take = v < c.V && sbin(s) <= (unsigned)wb;
          const unsigned m = __ballot_sync(0xffffffffu, take);
          if (m) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&s_gt_pos, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
            if (take && pos < (unsigned)GR4AD_MAX_BEAM) {
              const unsigned fi = (unsigned)((long long)r * c.V + v);
              sbuf[pos] = ((unsigned long long)f2ord(s) << 32) | (0xFFFFFFFFu - fi);
            }
          }
        }
      }
      __syncthreads();
      const unsigned n_win = s_gt_pos;  // (the proxy window's size is known only now)
      __syncthreads();
      if (n_win <= (unsigned)GR4AD_MAX_BEAM) {
        window = true;
        n_sort = (int)n_win;
      }
    }
    __syncthreads();
  }

  // ---- (b) exact radix fallback ---------------------------------------------
  uint32_t T = 0, pmask = 0;
  unsigned need = (unsigned)k;
  unsigned eq_total = 0;
  if (k > 0 && !window) {
    const int shifts[3] = {21, 10, 0};
    const int widths[3] = {11, 11, 10};
    for (int pass = 0; pass < 3; ++pass) {
      int nb = 1 << widths[pass];
      for (int i = tid; i < nb; i += kSelThreads) hist[i] = 0u;
      __syncthreads();
      sel_pass_hist<CACHE>(c, keys, hist, shifts[pass], pmask, T, (uint32_t)(nb - 1));
      __syncthreads();
      unsigned above;
      int bin = sel_find_bin(hist, nb, need, &above, scan);
      eq_total = hist[bin];
      need -= above;
      T |= (uint32_t)bin << shifts[pass];
      pmask |= (uint32_t)(nb - 1) << shifts[pass];
      __syncthreads();
    }
  }
  // need = number of keys == T to keep (lowest flat indices); eq_total = all keys == T
  const bool all_eq = (need == eq_total);
  const unsigned n_gt = (unsigned)k - need;
  if (tid == 0 && !window) s_gt_pos = 0;
  // per-row ordered tie ranks: rows are visited in order r = wid, wid+32, ...;
  // pass A counts ties per row (only when some ties must be dropped).
  // Row counts are kept in the sort buffer tail region (cleared below).
  unsigned *row_eq = hist;  // reused: per-row tie counts, 2048 rows per chunk
  const bool ordered = !all_eq && k > 0 && !window;
  __syncthreads();
  if (k > 0 && !window) {
    if (!ordered) {
      for (int r = wid; r < c.n_rows; r += kSelWarps) {
        float cr = 0.f;
        float2 ri = make_float2(0.f, 0.f);
        if (!CACHE) {
          cr = c.cum[c.hist0 + c.row0 + r];
          if (c.rowinfo) ri = c.rowinfo[c.row0 + r];
        }
        for (int v0 = 0; v0 < c.V; v0 += 32) {
          int v = v0 + lane;
          uint32_t u = 0;
          bool in = v < c.V;
          if (in) u = CACHE ? keys[(long long)r * c.V + v] : sel_key(c, r, v, cr, ri);
          bool take = in && u >= T;
          unsigned m = __ballot_sync(0xffffffffu, take);
          if (m) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&s_gt_pos, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (take) {
              unsigned pos = base + __popc(m & ((1u << lane) - 1u));
              unsigned fi = (unsigned)((long long)r * c.V + v);
              sbuf[pos] = ((unsigned long long)u << 32) | (0xFFFFFFFFu - fi);
            }
          }
        }
      }
    } else {
      // ordered tie handling: process rows in chunks of 2048 (row_eq counts)
      unsigned eq_base = 0;  // ties taken by earlier chunks
      for (int r0 = 0; r0 < c.n_rows; r0 += 2048) {
        int r1 = min(c.n_rows, r0 + 2048);
        for (int i = tid; i < 2048; i += kSelThreads) row_eq[i] = 0u;
        __syncthreads();
        for (int r = r0 + wid; r < r1; r += kSelWarps) {
          float cr = 0.f;
          float2 ri = make_float2(0.f, 0.f);
          if (!CACHE) {
            cr = c.cum[c.hist0 + c.row0 + r];
            if (c.rowinfo) ri = c.rowinfo[c.row0 + r];
          }
          unsigned n = 0;
          for (int v0 = 0; v0 < c.V; v0 += 32) {
            int v = v0 + lane;
            uint32_t u = 0;
            bool in = v < c.V;
            if (in) u = CACHE ? keys[(long long)r * c.V + v] : sel_key(c, r, v, cr, ri);
            n += __popc(__ballot_sync(0xffffffffu, in && u == T));
          }
          if (lane == 0) row_eq[r - r0] = n;
        }
        __syncthreads();
        // exclusive scan of row_eq[0 .. r1-r0) (serial by thread 0; <= 2048 rows)
        if (tid == 0) {
          unsigned run = eq_base;
          for (int i = 0; i < r1 - r0; ++i) {
            unsigned h = row_eq[i];
            row_eq[i] = run;
            run += h;
          }
          scan[0] = run;
        }
        __syncthreads();
        for (int r = r0 + wid; r < r1; r += kSelWarps) {
          float cr = 0.f;
          float2 ri = make_float2(0.f, 0.f);
          if (!CACHE) {
            cr = c.cum[c.hist0 + c.row0 + r];
            if (c.rowinfo) ri = c.rowinfo[c.row0 + r];
          }
          unsigned rank = row_eq[r - r0];
          for (int v0 = 0; v0 < c.V; v0 += 32) {
            int v = v0 + lane;
            uint32_t u = 0;
            bool in = v < c.V;
            if (in) u = CACHE ? keys[(long long)r * c.V + v] : sel_key(c, r, v, cr, ri);
            bool gt = in && u > T;
            bool eq = in && u == T;
            unsigned me = __ballot_sync(0xffffffffu, eq);
            unsigned myrank = rank + __popc(me & ((1u << lane) - 1u));
            bool take_eq = eq && myrank < need;
            unsigned mg = __ballot_sync(0xffffffffu, gt);
            unsigned base = 0;
            if (mg) {
              if (lane == 0) base = atomicAdd(&s_gt_pos, __popc(mg));
              base = __shfl_sync(0xffffffffu, base, 0);
            }
            unsigned fi = (unsigned)((long long)r * c.V + v);
            if (gt) {
              unsigned pos = base + __popc(mg & ((1u << lane) - 1u));
              sbuf[pos] = ((unsigned long long)u << 32) | (0xFFFFFFFFu - fi);
            }
            if (take_eq) sbuf[n_gt + myrank] = ((unsigned long long)u << 32) | (0xFFFFFFFFu - fi);
            rank += __popc(me);
          }
        }
        eq_base = scan[0];
        __syncthreads();
      }
    }
  }
  __syncthreads();
  // bitonic sort of sbuf[0..n2) descending
  int n2 = 1;
  while (n2 < n_sort) n2 <<= 1;
  for (int i = n_sort + tid; i < n2; i += kSelThreads) sbuf[i] = 0ull;
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < n2 / 2; i += kSelThreads) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool desc = (lo & size) == 0;
        unsigned long long x = sbuf[lo], y = sbuf[hi];
        if ((x < y) == desc) {
          sbuf[lo] = y;
          sbuf[hi] = x;
        }
      }
      __syncthreads();
    }
  }
  // outputs
  const uint32_t kNegInf = 0x007FFFFFu;  // f2ord(-inf)
  if (tid == 0) s_nfin = 0;
  __syncthreads();
  unsigned nf = 0;
  for (int j = tid; j < k; j += kSelThreads) nf += ((uint32_t)(sbuf[j] >> 32) != kNegInf);
  atomicAdd(&s_nfin, nf);
  __syncthreads();
  if (a.o_beam) {  // standalone selection: keep -inf like topk_precut
    for (int j = tid; j < k; j += kSelThreads) {
      unsigned long long e = sbuf[j];
      unsigned fi = 0xFFFFFFFFu - (unsigned)(e & 0xFFFFFFFFull);
      a.o_beam[(long long)b * a.o_k + j] = (int)(fi / c.V);
      a.o_token[(long long)b * a.o_k + j] = (int)(fi % c.V);
      a.o_score[(long long)b * a.o_k + j] = ord2f((uint32_t)(e >> 32));
    }
    if (tid == 0) a.o_count[b] = k;
    return;
  }
  const int nfin = (int)s_nfin;
  const int cap = a.out_cap[b];
  const int orow0 = a.out_row_off[b];
  const int t = a.level;
  const int st = a.anc_stride;
  for (int j = tid; j < cap; j += kSelThreads) {
    int jj = (j < nfin) ? j : 0;
    int parent = 0, tok = 0;
    float sc = -INFINITY;
    if (nfin > 0) {
      unsigned long long e = sbuf[jj];
      unsigned fi = 0xFFFFFFFFu - (unsigned)(e & 0xFFFFFFFFull);
      parent = (int)(fi / c.V);
      tok = (int)(fi % c.V);
      if (j < nfin) sc = ord2f((uint32_t)(e >> 32));
    }
    long long gp = (long long)a.hist_off + c.row0 + parent;
    long long gn = (long long)a.out_hist_off + orow0 + j;
    a.tok[gn] = tok;
    a.cum_out[gn] = sc;
    a.prefix[gn] = a.prefix[gp] * (long long)c.V + tok;
    for (int tau = 0; tau <= t; ++tau) a.anc[gn * st + tau] = a.anc[gp * st + tau];
    a.anc[gn * st + t + 1] = (int)gn;
  }
  if (tid == 0) a.out_live[b] = nfin;
}

int topk_select(const SelectArgs &a, int n_requests, int u_rows, int u_k,
                       long long max_cand, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
  bool cache = max_cand <= kCacheKeys;
  size_t sm = sizeof(unsigned long long) * GR4AD_MAX_BEAM + sizeof(unsigned) * 2048 +
              (cache ? sizeof(uint32_t) * kCacheKeys : 0);
  if (cache) {
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(topk_select_kernel<true>),
                                 (int)sm));
    GR_LAUNCH(KC_TOPK, st, topk_select_kernel<true><<<n_requests, kSelThreads, sm, st>>>(a, u_rows, u_k));
  } else {
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(topk_select_kernel<false>),
                                 (int)sm));
    GR_LAUNCH(KC_TOPK, st, topk_select_kernel<false><<<n_requests, kSelThreads, sm, st>>>(a, u_rows, u_k));
  }
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// tiled transpose: dst (cols x rows) = src (rows x cols)^T
// ---------------------------------------------------------------------------
__global__ void transpose_kernel(const float *__restrict__ src, long long lds, float *dst,
                                 float *dst_lo, long long ldd, int rows, int cols) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[(long long)r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      float x = tile[threadIdx.x][i];
      if (dst_lo) {  // tf32 split: hi = x with 13 low mantissa bits cleared, lo = x - hi
        float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        dst[(long long)c * ldd + r] = hi;
        dst_lo[(long long)c * ldd + r] = x - hi;
      } else {
        dst[(long long)c * ldd + r] = x;
      }
    }
  }
}

int transpose(const float *src, long long lds, float *dst, long long ldd, int rows, int cols,
              cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return GR4AD_OK;
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32));
  GR_LAUNCH(KC_SMALL, st, transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, lds, dst, nullptr, ldd, rows, cols));
  return GR4AD_OK;
}

// dst = split of scale * src^T into fp16 hi + lo (the tensor-core B operands)
__global__ void transpose_split16_kernel(const float *__restrict__ src, long long lds,
                                         __half *dst_hi, __half *dst_lo, long long ldd, int rows,
                                         int cols, float scale, int *flag) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[(long long)r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      const float x = tile[threadIdx.x][i] * scale;
      range_check(x, flag);
      const __half h = __float2half_rn(x);
      dst_hi[(long long)c * ldd + r] = h;
      dst_lo[(long long)c * ldd + r] = __float2half_rn(x - __half2float(h));
    }
  }
}

int transpose_split16(const float *src, long long lds, __half *dst_hi, __half *dst_lo,
                      long long ldd, int rows, int cols, float scale, int *flag, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return GR4AD_OK;
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32));
  GR_LAUNCH(KC_SMALL, st, transpose_split16_kernel<<<grid, dim3(32, 8), 0, st>>>(
                              src, lds, dst_hi, dst_lo, ldd, rows, cols, scale, flag));
  return GR4AD_OK;
}

// dst = split of scale * src into fp16 hi + lo (row-major, same shape)
__global__ void split16_kernel(const float *__restrict__ src, long long lds, __half *dst_hi,
                               __half *dst_lo, long long ldd, int rows, int cols, float scale,
                               int *flag) {
  const long long n = (long long)rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols;
    const int c = (int)(i - r * cols);
    const float x = src[r * lds + c] * scale;
    range_check(x, flag);
    const __half h = __float2half_rn(x);
    dst_hi[r * ldd + c] = h;
    dst_lo[r * ldd + c] = __float2half_rn(x - __half2float(h));
  }
}

int split16(const float *src, long long lds, __half *dst_hi, __half *dst_lo, long long ldd,
            int rows, int cols, float scale, int *flag, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return GR4AD_OK;
  const long long n = (long long)rows * cols;
  const int grid = (int)std::min<long long>(ceil_div(n, 256), 148LL * 16);
  GR_LAUNCH(KC_SMALL, st, split16_kernel<<<grid, 256, 0, st>>>(src, lds, dst_hi, dst_lo, ldd, rows,
                                                                cols, scale, flag));
  return GR4AD_OK;
}

// C (M x N, fp32) = A (M x K) . op(B), op(B) = B (K x N) or B^T (B: N x K),
// accumulated in double: the snapshot's factored attention weights
// (W_q W_k^T, W_v W_o) are products of two weight matrices, formed once per
// snapshot and rounded to fp32 once
__global__ void __launch_bounds__(256)
weight_product_kernel(const float *__restrict__ A, long long lda, const float *__restrict__ B,
                      long long ldb, int trans_b, float *C, long long ldc, int M, int N, int K) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e & 15, mm = e >> 4;  // A: consecutive threads walk k (row-contiguous)
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? (double)A[(long long)m * lda + k] : 0.0;
      int n, kb;
      if (trans_b) { kb = kk; n = n0 + mm; }          // B (N x K): walk k
      else { kb = e >> 6; n = n0 + (e & 63); }        // B (K x N): walk n
      const int kg = k0 + kb;
      const double bv = (n < N && kg < K)
                            ? (double)(trans_b ? B[(long long)n * ldb + kg] : B[(long long)kg * ldb + n])
                            : 0.0;
      Bs[kb][trans_b ? mm : (e & 63)] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty + 16 * i];
        b[i] = Bs[kk][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) C[(long long)m * ldc + n] = (float)acc[i][j];
    }
}

int weight_product(const float *A, long long lda, const float *B, long long ldb, bool trans_b,
                   float *C, long long ldc, int M, int N, int K, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return GR4AD_OK;
  dim3 grid(ceil_div(N, 64), ceil_div(M, 64));
  GR_LAUNCH(KC_SMALL, st, weight_product_kernel<<<grid, 256, 0, st>>>(A, lda, B, ldb, trans_b ? 1 : 0,
                                                                       C, ldc, M, N, K));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// request blocks -> 32-row-aligned blocks (zero padded): block per request
// ---------------------------------------------------------------------------
__global__ void pad_rows_kernel(const float *__restrict__ src, const int *__restrict__ in_off,
                                const int *__restrict__ out_off, const int *__restrict__ len,
                                int width, float *dst) {
  const int b = blockIdx.x;
  const int n = len[b], np = (n + 31) / 32 * 32;
  const float *s = src + (long long)in_off[b] * width;
  float *o = dst + (long long)out_off[b] * width;
  for (long long e = threadIdx.x; e < (long long)np * width; e += blockDim.x)
    o[e] = e < (long long)n * width ? s[e] : 0.f;
}

int pad_rows(const float *src, const int *in_off, const int *out_off, const int *len, int B,
             int width, float *dst, cudaStream_t st) {
  if (B <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_SMALL, st, pad_rows_kernel<<<B, 256, 0, st>>>(src, in_off, out_off, len, width, dst));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// teacher-forced inputs (decoder.py:143-152, 180-185): row (s, q) gets BOS at
// q = 0, else emb_{q-1}[tokens[s][q-1]]; K>0 writes it into U[:, d:2d],
// K==0 writes H = token + pos[q]
// ---------------------------------------------------------------------------
__global__ void seq_input_kernel(SeqInputArgs a) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)a.rows * a.d) return;
  const int r = (int)(i / a.d), j = (int)(i - (long long)r * a.d);
  const int s = r / a.n_pos, q = r - s * a.n_pos;
  const float e = (q == 0) ? a.bos[j]
                           : a.emb[q - 1][(long long)a.tokens[(long long)s * a.T + q - 1] * a.d + j];
  if (a.U) a.U[(long long)r * 2 * a.d + a.d + j] = e;
  else a.H[(long long)r * a.d + j] = e + a.pos[(long long)q * a.d + j];
}

int seq_input(const SeqInputArgs &a, cudaStream_t st) {
  long long n = (long long)a.rows * a.d;
  if (n <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_SMALL, st, seq_input_kernel<<<ceil_div(n, 256), 256, 0, st>>>(a));
  return GR4AD_OK;
}

// logp of the given token from a logits row and its (max, log-sum) (beam.py:92-95)
__global__ void gather_logp_kernel(const float *__restrict__ logits, long long ld, int rows,
                                   const float2 *__restrict__ info, const int *__restrict__ tokens,
                                   int T, int t, float *logp) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= rows) return;
  const int tok = tokens[(long long)s * T + t];
  const float2 ri = info[s];
  logp[(long long)s * T + t] = (logits[(long long)s * ld + tok] - ri.x) - ri.y;
}

int gather_logp(const float *logits, long long ld, int rows, const float2 *info,
                const int *tokens, int T, int t, float *logp, cudaStream_t st) {
  if (rows <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_SMALL, st, gather_logp_kernel<<<ceil_div(rows, 256), 256, 0, st>>>(logits, ld, rows, info, tokens, T, t, logp));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// level-0 rows
// ---------------------------------------------------------------------------
__global__ void init_level0_kernel(int B, int *live0, float *cum, long long *prefix, int *anc,
                                   int stride, int *tok) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  live0[b] = 1;
  cum[b] = 0.f;
  prefix[b] = 0;
  tok[b] = 0;
  anc[(long long)b * stride] = b;
}

int init_level0(int n_requests, int *live0, float *cum, long long *prefix, int *anc,
                int anc_stride, int *tok, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_SMALL, st, init_level0_kernel<<<ceil_div(n_requests, 256), 256, 0, st>>>(n_requests, live0, cum, prefix,
                                                                anc, anc_stride, tok));
  return GR4AD_OK;
}

// ---------------------------------------------------------------------------
// results (beam.py:212-213) + value re-rank (beam.py:258-288): block per request
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512)
collect_kernel(int T, const int *__restrict__ row_off_T, const int *__restrict__ live_T,
               int hist_off_T, const int *__restrict__ tok, const int *__restrict__ anc,
               int stride, const float *__restrict__ cum, const float *__restrict__ vlogits,
               int nb, const float *__restrict__ reps, int max_out, int *count,
               int *tokens, double *score) {
  extern __shared__ __align__(16) unsigned char smem[];
  double *key = reinterpret_cast<double *>(smem);
  int *idx = reinterpret_cast<int *>(key + GR4AD_MAX_BEAM);
  const int b = blockIdx.x;
  const int n = live_T[b];
  const int row0 = row_off_T[b];
  const int tid = threadIdx.x;
  if (tid == 0) count[b] = n;
  if (!vlogits) {
    for (int j = tid; j < n; j += blockDim.x) {
      long long g = (long long)hist_off_T + row0 + j;
      for (int t = 0; t < T; ++t)
        tokens[((long long)b * max_out + j) * T + t] = tok[anc[g * stride + t + 1]];
      score[(long long)b * max_out + j] = (double)cum[g];
    }
    return;
  }
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  for (int j = tid; j < n2; j += blockDim.x) {
    if (j < n) {
      const float *lg = vlogits + (long long)(row0 + j) * nb;
      double mx = -INFINITY;
      for (int q = 0; q < nb; ++q) mx = fmax(mx, (double)lg[q]);
      double s = 0.0;
      for (int q = 0; q < nb; ++q) s += exp((double)lg[q] - mx);
      double lse = log(s);
      double ev = 0.0;
      for (int q = 0; q < nb; ++q) ev += exp(((double)lg[q] - mx) - lse) * (double)reps[q];
      long long g = (long long)hist_off_T + row0 + j;
      key[j] = ev * exp((double)cum[g]);
      idx[j] = j;
    } else {
      key[j] = -INFINITY;
      idx[j] = 0x7fffffff;
    }
  }
  __syncthreads();
  // bitonic: order by (key desc, idx asc)
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
      for (int i = tid; i < n2 / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride2 - 1));
        int hi = lo + stride2;
        bool desc = (lo & size) == 0;
        double kx = key[lo], ky = key[hi];
        int ix = idx[lo], iy = idx[hi];
        bool x_before_y = (kx > ky) || (kx == ky && ix < iy);
        if (x_before_y != desc) {
          key[lo] = ky; key[hi] = kx;
          idx[lo] = iy; idx[hi] = ix;
        }
      }
      __syncthreads();
    }
  }
  for (int j = tid; j < n; j += blockDim.x) {
    long long g = (long long)hist_off_T + row0 + idx[j];
    for (int t = 0; t < T; ++t)
      tokens[((long long)b * max_out + j) * T + t] = tok[anc[g * stride + t + 1]];
    score[(long long)b * max_out + j] = key[j];
  }
}

int collect_results(int n_requests, int T, const int *row_off_T, const int *live_T,
                    int hist_off_T, const int *tok, const int *anc, int anc_stride,
                    const float *cum, const float *vlogits, int nb, const float *reps,
                    int max_out, int *count, int *tokens, double *score, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
  size_t sm = vlogits ? (sizeof(double) + sizeof(int)) * GR4AD_MAX_BEAM : 0;
  if (sm) GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(collect_kernel), (int)sm));
  GR_LAUNCH(KC_COLLECT, st, collect_kernel<<<n_requests, 512, sm, st>>>(T, row_off_T, live_T, hist_off_T, tok, anc,
                                              anc_stride, cum, vlogits, nb, reps, max_out,
                                              count, tokens, score));
  return GR4AD_OK;
}

}  // namespace gr
