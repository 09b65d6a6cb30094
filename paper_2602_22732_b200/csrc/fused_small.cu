// Fused per-request LazyAR beam decode for small models (d in {16, 32}).
//
// One CTA owns one request for the whole decode (beam.py:146-218):
// context projection (decoder.py:134-140), the beam-shared encoder K/V of
// every layer kept in shared memory (beam.py:98-109) as K^T / V^T, the trunk
// (beam.py:159-163), then per level every warp owns four beam rows and runs
// fuse -> head layers -> codebook logits -> log-softmax keys.  The four rows
// are register-tiled: each lane owns 8 contiguous context keys (or 8 codebook
// tokens) for all four rows, so every shared-memory K/V load and every head
// weight load feeds 32 FMAs.  The self-KV history lives in shared memory and
// is read through parent pointers (no copies, beam.py:205-210), and an exact
// radix top-k over the level's candidates compacts the beams in place.
// The C1/C2 working set (K^T/V^T 32 KB, history 25 KB) fits on chip: the
// batch decode is one launch.
#include <cuda_fp16.h>

#include "fused_small.cuh"

namespace gr {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int RW = 4;    // beam rows per warp
constexpr int SP = 256;  // context keys held per lane-row: 32 lanes x 8
constexpr unsigned kFull = 0xffffffffu;

// sum / max over the 8 lanes that share a row (lane >> 3)
__device__ __forceinline__ float rsum(float v) {
  v += __shfl_xor_sync(kFull, v, 4);
  v += __shfl_xor_sync(kFull, v, 2);
  v += __shfl_xor_sync(kFull, v, 1);
  return v;
}
__device__ __forceinline__ float rmax(float v) {
  v = fmaxf(v, __shfl_xor_sync(kFull, v, 4));
  v = fmaxf(v, __shfl_xor_sync(kFull, v, 2));
  v = fmaxf(v, __shfl_xor_sync(kFull, v, 1));
  return v;
}

// tanh-GELU (autodiff.py:301-306) via 0.5*a*(1+tanh z) == a / (1 + exp(-2z))
__device__ __forceinline__ float gelu_fast(float a) {
  const float c = 0.7978845608028654f;
  float z = (a + 0.044715f * a * a * a) * c;
  return __fdividef(a, 1.0f + __expf(-2.0f * z));
}
__device__ __forceinline__ float gelu_exp(float a) {
  const float c = 0.7978845608028654f;
  float z = (a + 0.044715f * a * a * a) * c;
  return a / (1.0f + expf(-2.0f * z));
}

// Row-lane layout: lane l owns row (l >> 3) of the warp's four and the E
// consecutive columns starting at (l & 7) * E.  Scratch "slots" hold the
// four rows transposed, slot[c * 4 + row], so one float4 read returns a
// column of all four rows.
template <int E>
__device__ __forceinline__ void publish(const float (&v)[E], float *slot) {
  const int lane = threadIdx.x & 31, rl = lane >> 3, cb = (lane & 7) * E;
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) slot[(cb + e) * 4 + rl] = v[e];
  __syncwarp();
}

// acc[e] = sum_i slot[i][row] * W[i][cb + e]   (W row-major, row stride ldw);
// two partial sums (even / odd i) halve the dependent FMA chain
template <int E>
__device__ __forceinline__ void proj(const float *slot, int din, const float *__restrict__ W,
                                     int ldw, float (&acc)[E]) {
  const int lane = threadIdx.x & 31, rl = lane >> 3, cb = (lane & 7) * E;
  float a2[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = a2[e] = 0.f;
  const float *w = W + cb;
#pragma unroll 4
  for (int i = 0; i < din; i += 2) {
    const float x0 = slot[i * 4 + rl], x1 = slot[(i + 1) * 4 + rl];
    if (E % 4 == 0) {
#pragma unroll
      for (int e = 0; e < E; e += 4) {
        const float4 u = __ldg(reinterpret_cast<const float4 *>(w + (size_t)i * ldw + e));
        const float4 v = __ldg(reinterpret_cast<const float4 *>(w + (size_t)(i + 1) * ldw + e));
        acc[e] = fmaf(x0, u.x, acc[e]);
        acc[e + 1] = fmaf(x0, u.y, acc[e + 1]);
        acc[e + 2] = fmaf(x0, u.z, acc[e + 2]);
        acc[e + 3] = fmaf(x0, u.w, acc[e + 3]);
        a2[e] = fmaf(x1, v.x, a2[e]);
        a2[e + 1] = fmaf(x1, v.y, a2[e + 1]);
        a2[e + 2] = fmaf(x1, v.z, a2[e + 2]);
        a2[e + 3] = fmaf(x1, v.w, a2[e + 3]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; e += 2) {
        const float2 u = __ldg(reinterpret_cast<const float2 *>(w + (size_t)i * ldw + e));
        const float2 v = __ldg(reinterpret_cast<const float2 *>(w + (size_t)(i + 1) * ldw + e));
        acc[e] = fmaf(x0, u.x, acc[e]);
        acc[e + 1] = fmaf(x0, u.y, acc[e + 1]);
        a2[e] = fmaf(x1, v.x, a2[e]);
        a2[e + 1] = fmaf(x1, v.y, a2[e + 1]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] += a2[e];
}

// acc[e] = sum_j slot[j][row] * W[cb + e][j]   (the transposed product, for
// the trunk's reassociated attention u = q Wk^T)
template <int E>
__device__ __forceinline__ void proj_t(const float *slot, int din, const float *__restrict__ W,
                                       int ldw, float (&acc)[E]) {
  const int lane = threadIdx.x & 31, rl = lane >> 3, cb = (lane & 7) * E;
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
#pragma unroll 2
  for (int j = 0; j < din; j += 4) {
    const float x0 = slot[j * 4 + rl], x1 = slot[(j + 1) * 4 + rl];
    const float x2 = slot[(j + 2) * 4 + rl], x3 = slot[(j + 3) * 4 + rl];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float4 w4 = __ldg(reinterpret_cast<const float4 *>(W + (size_t)(cb + e) * ldw + j));
      acc[e] = fmaf(x0, w4.x, acc[e]);
      acc[e] = fmaf(x1, w4.y, acc[e]);
      acc[e] = fmaf(x2, w4.z, acc[e]);
      acc[e] = fmaf(x3, w4.w, acc[e]);
    }
  }
}

template <int E>
__device__ __forceinline__ void layer_norm(const float (&h)[E], const float *g, const float *b,
                                           float (&o)[E]) {
  const int cb = (threadIdx.x & 7) * E;
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) s += h[e];
  const float mean = rsum(s) / (float)(8 * E);
  float v = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    float c = h[e] - mean;
    v += c * c;
  }
  const float inv = 1.0f / sqrtf(rsum(v) / (float)(8 * E) + 1e-5f);
#pragma unroll
  for (int e = 0; e < E; ++e) o[e] = (h[e] - mean) * inv * __ldg(g + cb + e) + __ldg(b + cb + e);
}

// Cross-attention of the warp's four rows against the shared context
// K^T / V^T (D x SP each): q in a slot; result in the row-lane layout.
template <int D>
__device__ __forceinline__ void cross_attn(const float *qslot, const float *KT, const float *VT,
                                           int S, int ld, float *oslot, float (&out)[D / 8]) {
  const int lane = threadIdx.x & 31;
  const float scale = 1.0f / sqrtf((float)D);
  float sc[RW][8];
#pragma unroll
  for (int r = 0; r < RW; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) sc[r][c] = 0.f;
#pragma unroll 4
  for (int i = 0; i < D; ++i) {
    const float4 q4 = *reinterpret_cast<const float4 *>(qslot + i * 4);
    const float4 ka = *reinterpret_cast<const float4 *>(KT + i * ld + lane * 8);
    const float4 kb = *reinterpret_cast<const float4 *>(KT + i * ld + lane * 8 + 4);
    const float qq[4] = {q4.x, q4.y, q4.z, q4.w};
    const float kk[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) sc[r][c] = fmaf(qq[r], kk[c], sc[r][c]);
  }
  // softmax over the S keys of each row (autodiff.py:362-368)
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      sc[r][c] = (lane * 8 + c < S) ? sc[r][c] * scale : -INFINITY;
      mx = fmaxf(mx, sc[r][c]);
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      sc[r][c] = __expf(sc[r][c] - mx);  // arguments <= 0; rel. err ~1e-7
      sum += sc[r][c];
    }
    const float inv = 1.0f / warp_sum(sum);
#pragma unroll
    for (int c = 0; c < 8; ++c) sc[r][c] *= inv;
  }
  // P.V in blocks of 8 output dims; the reduce-scatter leaves row l>>3,
  // dim 8h + (l & 7) on lane l
#pragma unroll
  for (int h = 0; h < D / 8; ++h) {
    float acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float *vrow = VT + (h * 8 + j) * ld + lane * 8;
      const float4 va = *reinterpret_cast<const float4 *>(vrow);
      const float4 vb = *reinterpret_cast<const float4 *>(vrow + 4);
      const float vv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r * 8 + j] = fmaf(sc[r][c], vv[c], acc[r * 8 + j]);
    }
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
      const bool up = (lane & half) != 0;
#pragma unroll
      for (int k = 0; k < half; ++k) {
        float send = up ? acc[k] : acc[k + half];
        float keep = up ? acc[k + half] : acc[k];
        acc[k] = keep + __shfl_xor_sync(kFull, send, half);
      }
    }
    oslot[(h * 8 + (lane & 7)) * 4 + (lane >> 3)] = acc[0];
  }
  __syncwarp();
  const int rl = lane >> 3, cb = (lane & 7) * (D / 8);
#pragma unroll
  for (int e = 0; e < D / 8; ++e) out[e] = oslot[(cb + e) * 4 + rl];
  __syncwarp();
}

// FFN W2 gelu(W1 n + b1) (+ b2 by the caller), d_ff in {D, 2D} (layers.py:115-118)
template <int D>
__device__ __forceinline__ void ffn(const float *nslot, float *hslot, const gr4ad_layer &Lw,
                                    int dff, float (&out)[D / 8]) {
  constexpr int E = D / 8;
  const int cb = (threadIdx.x & 7) * E;
  float f0[E];
  proj<E>(nslot, D, Lw.ffn_W1, dff, f0);
#pragma unroll
  for (int e = 0; e < E; ++e) f0[e] = gelu_exp(f0[e] + __ldg(Lw.ffn_b1 + cb + e));
  publish<E>(f0, hslot);
  proj<E>(hslot, D, Lw.ffn_W2, D, out);
  if (dff > D) {
    float f1[E], t2[E];
    proj<E>(nslot, D, Lw.ffn_W1 + D, dff, f1);
#pragma unroll
    for (int e = 0; e < E; ++e) f1[e] = gelu_exp(f1[e] + __ldg(Lw.ffn_b1 + D + cb + e));
    publish<E>(f1, hslot);
    proj<E>(hslot, D, Lw.ffn_W2 + (size_t)D * D, D, t2);
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] += t2[e];
  }
}

// ---- exact top-k helpers (same order semantics as kernels.cu) -------------
__device__ int find_bin(const unsigned *hist, int nbins, unsigned need, unsigned *above,
                        unsigned *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (nbins + kThreads - 1) / kThreads;
  unsigned local = 0;
  for (int i = 0; i < per; ++i) {
    int b = nbins - 1 - (tid * per + i);
    if (b >= 0) local += hist[b];
  }
  unsigned x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[2 + wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned s = lane < kWarps ? scratch[2 + lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kWarps) scratch[2 + lane] = s;
  }
  __syncthreads();
  unsigned run = x - local + (wid > 0 ? scratch[2 + wid - 1] : 0u);
  for (int i = 0; i < per; ++i) {
    int b = nbins - 1 - (tid * per + i);
    if (b >= 0) {
      unsigned h = hist[b];
      if (run < need && need <= run + h) {
        scratch[0] = (unsigned)b;
        scratch[1] = run;
      }
      run += h;
    }
  }
  __syncthreads();
  *above = scratch[1];
  int b = (int)scratch[0];
  __syncthreads();
  return b;
}

__device__ __forceinline__ void hist_add(unsigned *hist, int &cur, unsigned &cnt, int bin) {
  if (bin == cur) {
    ++cnt;
  } else {
    if (cnt) atomicAdd(&hist[cur], cnt);
    cur = bin;
    cnt = 1;
  }
}

// Descending bitonic sort of buf[0, n2) (n2 a power of two >= 64, sorted by
// the whole 64-bit key).  Stages with stride >= 64 run block-wide through
// shared memory; the stride <= 32 tail of every merge runs in registers:
// warp w owns 64-entry chunks (lane holds entries lane and lane + 32) and
// exchanges with __shfl_xor -- ~log2(n2) block barriers instead of
// log2(n2)^2 / 2.
__device__ __forceinline__ unsigned long long cmpx(unsigned long long mine,
                                                   unsigned long long other, bool take_max) {
  return take_max ? (mine > other ? mine : other) : (mine < other ? mine : other);
}

__device__ void warp_merge_tail(unsigned long long *buf, int n2, int size, int st_hi) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = wid * 64; base < n2; base += kWarps * 64) {
    unsigned long long e0 = buf[base + lane], e1 = buf[base + lane + 32];
    const int i0 = base + lane, i1 = i0 + 32;
#pragma unroll 1
    for (int sz = (size > 0 ? size : 2); sz <= (size > 0 ? size : 64); sz <<= 1) {
#pragma unroll 1
      for (int st = (size > 0 ? st_hi : sz >> 1); st > 0; st >>= 1) {
        if (st == 32) {
          const bool desc = (i0 & sz) == 0;  // i0 is the low side of (i0, i1)
          const unsigned long long hi = e0 > e1 ? e0 : e1, lo = e0 > e1 ? e1 : e0;
          e0 = desc ? hi : lo;
          e1 = desc ? lo : hi;
        } else {
          const unsigned long long o0 = __shfl_xor_sync(kFull, e0, st);
          const unsigned long long o1 = __shfl_xor_sync(kFull, e1, st);
          const bool low0 = (i0 & st) == 0, low1 = (i1 & st) == 0;
          const bool d0 = (i0 & sz) == 0, d1 = (i1 & sz) == 0;
          e0 = cmpx(e0, o0, low0 == d0);
          e1 = cmpx(e1, o1, low1 == d1);
        }
      }
    }
    buf[base + lane] = e0;
    buf[base + lane + 32] = e1;
  }
}

// buf[0 .. k) = the k largest of buf[0 .. n2) in descending order (keys
// unique, or zero padding that never ranks below n_real <= n2).
// n2 <= 256: every warp sorts one 64-entry chunk in registers, then
// each entry's rank is its position in its own chunk plus, for every other
// chunk, the count of larger entries (a branch-free 64-way binary search);
// one scatter.  No block-wide merge stages.  Larger n2: full bitonic sort
// (measured faster from 512 on: the searches grow with the chunk count).
__device__ void sort_desc(unsigned long long *buf, int n2, int k) {
  warp_merge_tail(buf, n2, 0, 0);  // sizes 2..64 entirely in registers
  __syncthreads();
  if (n2 == 64) return;  // one chunk: sorted already
  if (n2 <= 256) {
    const int nc = n2 / 64;  // chunk c is descending for even c, ascending for odd
    unsigned long long x[2];
    int rk[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = threadIdx.x + u * kThreads;
      rk[u] = 0x7fffffff;
      x[u] = 0ull;
      if (i < n2) {
        x[u] = buf[i];
        const int c = i >> 6, o = i & 63;
        int r = (c & 1) ? 63 - o : o;
        for (int c2 = 0; c2 < nc; ++c2) {
          if (c2 == c) continue;
          const unsigned long long *b = buf + c2 * 64;
          const bool asc = c2 & 1;
          int pos = 0;  // count of entries > x in chunk c2
#pragma unroll
          for (int st = 32; st >= 1; st >>= 1) {
            const int j = pos + st - 1;
            pos += b[asc ? 63 - j : j] > x[u] ? st : 0;
          }
          pos += (pos == 63 && b[asc ? 0 : 63] > x[u]) ? 1 : 0;
          r += pos;
        }
        rk[u] = r;
      }
    }
    __syncthreads();  // every read done before the scatter
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (rk[u] < k) buf[rk[u]] = x[u];
    __syncthreads();
    return;
  }
  for (int size = 128; size <= n2; size <<= 1) {
    for (int st = size >> 1; st >= 64; st >>= 1) {
      for (int i = threadIdx.x; i < n2 / 2; i += kThreads) {
        const int lo = 2 * i - (i & (st - 1)), hi = lo + st;
        const bool desc = (lo & size) == 0;
        const unsigned long long x = buf[lo], y = buf[hi];
        if ((x < y) == desc) {
          buf[lo] = y;
          buf[hi] = x;
        }
      }
      __syncthreads();
    }
    warp_merge_tail(buf, n2, size, 32);
    __syncthreads();
  }
}

#ifdef GR_FUSED_TIMING
#define GR_TSTAMP(i)                                                            \
  do {                                                                          \
    if ((threadIdx.x & 31) == 0) {                                              \
      long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
      a.dbg[blockIdx.x * kDbgSlots + (i)] = _t;                                 \
    }                                                                           \
  } while (0)
#else
#define GR_TSTAMP(i) do {} while (0)
#endif

// Trunk: K layers over the n_pos position rows (beam.py:159-163), run by
// warp 0 alone and reassociated so the trunk layers' K/V are never built:
// scores (q Wk^T) X^T, output (P X) Wv.  Xs is X^T with row stride xld.
template <int D>
__device__ void trunk_warp0(const FusedArgs &a, const float *Xs, int xld, int S, float *TR,
                            float *TQ, float *wsl, const float *u0 = nullptr) {
  constexpr int E = D / 8;
  const int lane = threadIdx.x & 31, rl = lane >> 3, cb = (lane & 7) * E;
  const gr4ad_weights &W = a.w;
  const int L = a.L, K = a.K, dff = a.dff, np = a.n_pos;
  const float scale = 1.0f / sqrtf((float)D);
  float *slot0 = wsl, *slot1 = wsl + 4 * D, *slot2 = wsl + 8 * D, *slot3 = wsl + 12 * D;
  for (int e = lane; e < np * D; e += 32) TR[e] = __ldg(W.pos + e);
  __syncwarp();
  const int ldw = 2 * L * D;
  for (int i = 0; i < K; ++i) {
    const gr4ad_layer &Lw = W.layer[i];
    const float *Wk = W.cross_kv_W + (size_t)(2 * i) * D, *Wv = Wk + D;
    for (int p0 = 0; p0 < np; p0 += RW) {
      const int p = p0 + rl, pp = min(p, np - 1);
      const bool ok = p < np;
      float h[E], n[E], t[E];
#pragma unroll
      for (int e = 0; e < E; ++e) h[e] = TR[pp * D + cb + e];
      if (i == 0 && u0) {  // layer 0's query side depends on the weights only
#pragma unroll
        for (int e = 0; e < E; ++e) t[e] = u0[pp * D + cb + e];
      } else {
        layer_norm<E>(h, Lw.ln1_g, Lw.ln1_b, n);
        publish<E>(n, slot0);
        proj<E>(slot0, D, Lw.cross_Wq, D, t);
        GR_TSTAMP(42);
        publish<E>(t, slot1);
        proj_t<E>(slot1, D, Wk, ldw, t);  // u = q Wk^T, u . x_s == q . k_s
      }
      GR_TSTAMP(43);
      publish<E>(t, slot0);
      cross_attn<D>(slot0, Xs, Xs, S, xld, slot2, t);  // t = P X
      GR_TSTAMP(44);
      publish<E>(t, slot1);
      proj<E>(slot1, D, Wv, ldw, t);  // (P X) Wv == P V
      publish<E>(t, slot0);
      proj<E>(slot0, D, Lw.cross_Wo, D, t);
#pragma unroll
      for (int e = 0; e < E; ++e) h[e] += t[e];
      layer_norm<E>(h, Lw.ln2_g, Lw.ln2_b, n);
      publish<E>(n, slot0);
      GR_TSTAMP(45);
      for (int c = 0; c < 3; ++c) {
        proj<E>(slot0, D, Lw.self_Wqkv + c * D, 3 * D, t);
        if (ok)
#pragma unroll
          for (int e = 0; e < E; ++e) TQ[(p * 3 + c) * D + cb + e] = t[e];
      }
      if (ok)
#pragma unroll
        for (int e = 0; e < E; ++e) TR[p * D + cb + e] = h[e];
    }
    __syncwarp();
    for (int p0 = 0; p0 < np; p0 += RW) {
      const int p = p0 + rl, pp = min(p, np - 1);
      const bool ok = p < np;
      const int rmax_w = min(p0 + RW, np) - 1;  // warp-uniform loop bound
      float h[E], n[E], t[E], q[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        h[e] = TR[pp * D + cb + e];
        q[e] = TQ[(pp * 3) * D + cb + e];
      }
      // causal self-attention over positions 0..p (layers.py:94-100), online
      float mx = -INFINITY, se = 0.f, so[E];
#pragma unroll
      for (int e = 0; e < E; ++e) so[e] = 0.f;
      for (int r = 0; r <= rmax_w; ++r) {
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) dot = fmaf(q[e], TQ[(r * 3 + 1) * D + cb + e], dot);
        const float sc = rsum(dot) * scale;
        if (r <= pp) {
          const float nm = fmaxf(mx, sc), f = expf(mx - nm), w = expf(sc - nm);
          se = se * f + w;
#pragma unroll
          for (int e = 0; e < E; ++e) so[e] = so[e] * f + w * TQ[(r * 3 + 2) * D + cb + e];
          mx = nm;
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) so[e] /= se;
      GR_TSTAMP(46);
      publish<E>(so, slot0);
      proj<E>(slot0, D, Lw.self_Wo, D, t);
#pragma unroll
      for (int e = 0; e < E; ++e) h[e] += t[e];
      layer_norm<E>(h, Lw.ln3_g, Lw.ln3_b, n);
      publish<E>(n, slot0);
      GR_TSTAMP(47);
      ffn<D>(slot0, slot3, Lw, dff, t);
#pragma unroll
      for (int e = 0; e < E; ++e) h[e] += t[e] + __ldg(Lw.ffn_b2 + cb + e);
      __syncwarp();
      if (ok)
#pragma unroll
        for (int e = 0; e < E; ++e) TR[p * D + cb + e] = h[e];
    }
    __syncwarp();
  }
}

}  // namespace

#ifdef GR_FUSED_TIMING
#define GR_STAMP(i)                                                             \
  do {                                                                          \
    if (threadIdx.x == 0) {                                                     \
      long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
      a.dbg[blockIdx.x * kDbgSlots + (i)] = _t;                                        \
    }                                                                           \
  } while (0)
#define GR_SUB(i)                                                               \
  do {                                                                          \
    if (t < 3 && threadIdx.x == 0) {                                            \
      long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
      a.dbg[blockIdx.x * kDbgSlots + 18 + 8 * t + (i)] = _t;                    \
    }                                                                           \
  } while (0)
// lane 0 of the calling warp stamps slot i (16 <= i < kDbgSlots)
#define GR_WSTAMP(i)                                                            \
  do {                                                                          \
    if ((threadIdx.x & 31) == 0) {                                              \
      long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
      a.dbg[blockIdx.x * kDbgSlots + (i)] = _t;                                 \
    }                                                                           \
  } while (0)
#ifdef GR_NO_XSTAMP
#define GR_XSTAMP(w, i) do {} while (0)
#else
#define GR_XSTAMP(w, i)                                                         \
  do {                                                                          \
    if (t == 2 && threadIdx.x == 32 * (w)) {                                    \
      long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
      a.dbg[blockIdx.x * kDbgSlots + (i)] = _t;                                 \
    }                                                                           \
  } while (0)
#endif
#else
#define GR_XSTAMP(w, i) do {} while (0)
#define GR_STAMP(i) do {} while (0)
#define GR_SUB(i) do {} while (0)
#define GR_WSTAMP(i) do {} while (0)
#endif


// Beam selection of level t over the `live` rows' keys (or, at t == T, the
// value re-rank output) and in-place compaction; returns the next level's
// live rows (-1 once the re-rank output is written).  Shared by both fused
// kernels (beam.py:30-89, 202-210, 258-288).
// collected >= 0: sbuf already holds that many entries (key << 32 | ~flat
// index) including every candidate of the top k (the warp-MMA kernel's
// proxy window); they are only sorted and compacted.
__device__ int select_level(const FusedArgs &a, int b, int t, int live, int V,
                            const uint32_t *keys, unsigned *hist, unsigned *scr,
                            unsigned long long *sbuf, int *par, int *tokm, float *cum, float Rs,
                            float bscale, int collected = -1, int *pfx = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int T = a.T;
  auto sbin = [&](float sc) -> unsigned {
    return (unsigned)fminf((Rs - sc) * bscale, 2047.0f);  // NaN-free: sc <= Rs
  };
  if (t == T) {  // re-rank output: sort rows by (rank desc, row asc)
    double *key = reinterpret_cast<double *>(sbuf);
    int *idx = reinterpret_cast<int *>(hist);
    int n2 = 1;
    while (n2 < live) n2 <<= 1;
    for (int j = tid; j < n2; j += kThreads) {
      idx[j] = j < live ? j : 0x7fffffff;
      if (j >= live) key[j] = -INFINITY;
    }
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1)
      for (int st = size >> 1; st > 0; st >>= 1) {
        for (int i = tid; i < n2 / 2; i += kThreads) {
          int lo = 2 * i - (i & (st - 1)), hi = lo + st;
          bool desc = (lo & size) == 0;
          double kx = key[lo], ky = key[hi];
          int ix = idx[lo], iy = idx[hi];
          bool xb = (kx > ky) || (kx == ky && ix < iy);
          if (xb != desc) {
            key[lo] = ky; key[hi] = kx;
            idx[lo] = iy; idx[hi] = ix;
          }
        }
        __syncthreads();
      }
    for (int j = tid; j < live; j += kThreads) {
      int ar = idx[j];
      for (int tau = T - 1; tau >= 0; --tau) {
        a.out_tokens[((size_t)b * a.max_out + j) * T + tau] = tokm[a.moff[tau + 1] + ar];
        ar = par[a.moff[tau + 1] + ar];
      }
      a.out_score[(size_t)b * a.max_out + j] = key[j];
    }
    if (tid == 0) a.out_count[b] = live;
    GR_STAMP(15);
    return -1;
  }

  // ---- exact top-k under (-score, row, token) (beam.py:30-89) --------------
  const int n_cand = live * V;
  const int k = min(a.eff[t * a.B + b], n_cand);
  int n_sort = k;  // entries in sbuf to sort (>= k)
  if (collected >= 0) {
    n_sort = collected;
  } else {
    // (a) window: every key in a bin below the k-th key's bin is in the
    // top-k; the k-th bin is collected whole and the exact sort breaks it
    unsigned cnt_le = 0;
    int wb = 2047;
    {
      // k-th smallest bin index == (2048 - 1 - bin of the k-th largest in
      // reversed order): find_bin scans from the top bin, so mirror
      unsigned above;
      for (int i = tid; i < 1024; i += kThreads) {
        unsigned x = hist[i], y = hist[2047 - i];
        hist[i] = y;
        hist[2047 - i] = x;
      }
      __syncthreads();
      int rb = find_bin(hist, 2048, (unsigned)k, &above, scr);  // mirrored bin
      wb = 2047 - rb;
      cnt_le = above + hist[rb];
    }
    const bool window_ok = wb < 2047 && cnt_le <= (unsigned)a.sort_cap;
#ifdef GR_FUSED_TIMING_WINDOW
    if (tid == 0 && t < 3) {
      a.dbg[blockIdx.x * kDbgSlots + 10 + t] = ((long long)cnt_le << 32) | (unsigned)wb;
      a.dbg[blockIdx.x * kDbgSlots + 13 + (t == 2)] = (long long)(bscale * 1000);
    }
#endif
    if (window_ok) {
      if (tid == 0) scr[40] = 0;
      __syncthreads();
      const uint4 *keys4 = reinterpret_cast<const uint4 *>(keys);
      const int n4 = n_cand / 4;
      // 8 independent L2 loads in flight per thread, then filter
      constexpr int U = 8;
      for (int i0 = tid; i0 < n4; i0 += U * kThreads) {
        uint4 u4[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int i4 = i0 + j * kThreads;
          u4[j] = i4 < n4 ? keys4[i4] : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int i4 = i0 + j * kThreads;
          const uint32_t us[4] = {u4[j].x, u4[j].y, u4[j].z, u4[j].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (i4 < n4 && sbin(ord2f(us[q])) <= (unsigned)wb) {
              unsigned pos = atomicAdd(&scr[40], 1u);
              sbuf[pos] = ((unsigned long long)us[q] << 32) | (0xFFFFFFFFu - (unsigned)(i4 * 4 + q));
            }
          }
        }
      }
      n_sort = (int)cnt_le;
    } else {
      // (b) exact radix fallback (11/11/10-bit passes over the keys)
      unsigned need = (unsigned)k, above;
      for (int i = tid; i < 2048; i += kThreads) hist[i] = 0u;
      __syncthreads();
      uint32_t T32 = 0, pmask = 0;
      unsigned eq_total = 0;
      const uint4 *keys4 = reinterpret_cast<const uint4 *>(keys);
      const int n4 = n_cand / 4;
      for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
        const int nb = pass == 2 ? 1024 : 2048;
        __syncthreads();
        for (int i = tid; i < nb; i += kThreads) hist[i] = 0u;
        __syncthreads();
        int cur = -1;
        unsigned cnt = 0;
        for (int i4 = tid; i4 < n4; i4 += kThreads) {
          const uint4 u4 = keys4[i4];
          const uint32_t us[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if ((us[q] & pmask) == T32) hist_add(hist, cur, cnt, (int)((us[q] >> shift) & (nb - 1)));
        }
        if (cnt) atomicAdd(&hist[cur], cnt);
        __syncthreads();
        int bin = find_bin(hist, nb, need, &above, scr);
        eq_total = hist[bin];
        need -= above;
        T32 |= (uint32_t)bin << shift;
        pmask |= (uint32_t)(nb - 1) << shift;
      }
      const unsigned n_gt = (unsigned)k - need;
      if (tid == 0) scr[40] = 0;
      __syncthreads();
      if (need == eq_total) {
        for (int i0 = wid * 32; i0 < n_cand; i0 += kThreads) {
          int i = i0 + lane;
          uint32_t u = i < n_cand ? keys[i] : 0u;
          bool take = i < n_cand && u >= T32;
          unsigned m = __ballot_sync(kFull, take);
          unsigned base = 0;
          if (m && lane == 0) base = atomicAdd(&scr[40], __popc(m));
          base = __shfl_sync(kFull, base, 0);
          if (take) sbuf[base + __popc(m & ((1u << lane) - 1u))] =
              ((unsigned long long)u << 32) | (0xFFFFFFFFu - (unsigned)i);
        }
      } else {
        // ordered ties: contiguous index chunks per warp, warp tie counts scanned
        const int chunk = ((n_cand + kWarps - 1) / kWarps + 31) / 32 * 32;
        const int c0 = wid * chunk, c1 = min(n_cand, c0 + chunk);
        unsigned neq = 0;
        for (int i0 = c0; i0 < c1; i0 += 32) {
          int i = i0 + lane;
          neq += __popc(__ballot_sync(kFull, i < c1 && keys[i] == T32));
        }
        if (lane == 0) scr[8 + wid] = neq;
        __syncthreads();
        unsigned rank = 0;
        for (int w2 = 0; w2 < wid; ++w2) rank += scr[8 + w2];
        for (int i0 = c0; i0 < c1; i0 += 32) {
          int i = i0 + lane;
          uint32_t u = i < c1 ? keys[i] : 0u;
          bool gt = i < c1 && u > T32;
          bool eq = i < c1 && u == T32;
          unsigned me = __ballot_sync(kFull, eq);
          unsigned myr = rank + __popc(me & ((1u << lane) - 1u));
          unsigned mg = __ballot_sync(kFull, gt);
          unsigned base = 0;
          if (mg && lane == 0) base = atomicAdd(&scr[40], __popc(mg));
          base = __shfl_sync(kFull, base, 0);
          unsigned long long e = ((unsigned long long)u << 32) | (0xFFFFFFFFu - (unsigned)i);
          if (gt) sbuf[base + __popc(mg & ((1u << lane) - 1u))] = e;
          if (eq && myr < need) sbuf[n_gt + myr] = e;
          rank += __popc(me);
        }
      }
    }
  }
  __syncthreads();
  int n2 = 64;
  while (n2 < n_sort) n2 <<= 1;
  for (int i = n_sort + tid; i < n2; i += kThreads) sbuf[i] = 0ull;
  __syncthreads();
  sort_desc(sbuf, n2, k);
  // alive filter (beam.py:202-203): with masking, -inf candidates sort last;
  // keep the finite prefix of the selection
  int kk = k;
  if (a.vp_rp[t]) {
    if (tid == 0) scr[42] = (unsigned)k;
    __syncthreads();
    const uint32_t ninf = f2ord(-INFINITY);
    for (int j = tid; j < k; j += kThreads)
      if ((uint32_t)(sbuf[j] >> 32) <= ninf) atomicMin(&scr[42], (unsigned)j);
    __syncthreads();
    kk = (int)scr[42];
  }
  // compaction: next-level rows in selection order (beam.py:202-210)
  const int mo1 = a.moff[t + 1];
  const int mo0 = a.moff[t];
  for (int j = tid; j < kk; j += kThreads) {
    unsigned long long e = sbuf[j];
    // (clamped: non-finite scores from out-of-range inputs -- reported by
    // gr4ad_range_status -- must not turn into out-of-bounds rows)
    unsigned fi = min(0xFFFFFFFFu - (unsigned)(e & 0xFFFFFFFFull), (unsigned)(n_cand - 1));
    par[mo1 + j] = (int)(fi / (unsigned)V);
    tokm[mo1 + j] = (int)(fi % (unsigned)V);
    cum[mo1 + j] = ord2f((uint32_t)(e >> 32));
    if (pfx) pfx[mo1 + j] = pfx[mo0 + fi / (unsigned)V] * V + (int)(fi % (unsigned)V);
  }
  return kk;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 2) fused_small_kernel(FusedArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int E = D / 8;  // columns per lane in the row-lane layout
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rl = lane >> 3, cb = (lane & 7) * E;
  const int T = a.T, L = a.L, K = a.K, dff = a.dff;
  const int S = a.ctx_len[b];
  const long long coff = a.ctx_off[b];
  const gr4ad_weights &W = a.w;
  const float scale = 1.0f / sqrtf((float)D);

  float *Xs = sm + a.s_X;   // X^T: D x SP (aliases the history region)
  float *KV = sm + a.s_KV;  // per slot: K^T (D x SP) then V^T (D x SP)
  float *TR = sm + a.s_TR;  // n_pos x D
  float *TQ = sm + a.s_TQ;  // n_pos x 3 x D
  float *HI = sm + a.s_hist;
  int *par = reinterpret_cast<int *>(sm + a.s_par);
  int *tokm = reinterpret_cast<int *>(sm + a.s_tok);
  float *cum = sm + a.s_cum;
  unsigned *hist = reinterpret_cast<unsigned *>(sm + a.s_bins);
  unsigned *scr = reinterpret_cast<unsigned *>(sm + a.s_scr);
  unsigned long long *sbuf = reinterpret_cast<unsigned long long *>(sm + a.s_sort);
  float *wsl = sm + a.s_ws + wid * 4 * D * 4;  // this warp's 4 slots of (D x 4)
  float *slot0 = wsl, *slot1 = wsl + 4 * D, *slot2 = wsl + 8 * D, *slot3 = wsl + 12 * D;
  uint32_t *keys = a.keys + (size_t)b * a.keys_per_req;
  const int KVS = D * SP;
  GR_STAMP(0);

  // ---- context projection X = F W_c + b_c (decoder.py:134-140) -------------
  // thread s owns key s: its feature row in registers, W_c rows broadcast
  for (int s = tid; s < SP; s += kThreads) {
    float x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = 0.f;
    if (s < S) {
      if (a.features) {
        const float *f = a.features + (coff + s) * a.F;
        for (int i = 0; i < a.F; ++i) {
          const float fi = __ldg(f + i);
#pragma unroll
          for (int j = 0; j < D; j += 4) {
            const float4 w4 = __ldg(reinterpret_cast<const float4 *>(W.ctx_W + (size_t)i * D + j));
            x[j] = fmaf(fi, w4.x, x[j]);
            x[j + 1] = fmaf(fi, w4.y, x[j + 1]);
            x[j + 2] = fmaf(fi, w4.z, x[j + 2]);
            x[j + 3] = fmaf(fi, w4.w, x[j + 3]);
          }
        }
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] += __ldg(W.ctx_b + j);
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = __ldg(a.context + (coff + s) * D + j);
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) Xs[j * SP + s] = x[j];
  }
  __syncthreads();
  GR_STAMP(1);

  // K^T / V^T of head layer `layer` into `slot` (keys >= S are zero); thread
  // tid - t0 owns keys s, s + nt, ...: X column in registers, weight rows as
  // broadcast float4 loads, 8 output columns per pass
  auto build_kv = [&](int layer, int slot, int t0, int nt) {
    float *Kt = KV + (size_t)slot * 2 * KVS;
    const int ldw = 2 * L * D;
    const float *Wl = W.cross_kv_W + (size_t)(2 * layer) * D;
    for (int s = tid - t0; s < SP; s += nt) {
      float x[D];
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = Xs[i * SP + s];
#pragma unroll 1
      for (int c0 = 0; c0 < 2 * D; c0 += 8) {
        float acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.f;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const float4 wa = __ldg(reinterpret_cast<const float4 *>(Wl + (size_t)i * ldw + c0));
          const float4 wb = __ldg(reinterpret_cast<const float4 *>(Wl + (size_t)i * ldw + c0 + 4));
          acc[0] = fmaf(x[i], wa.x, acc[0]);
          acc[1] = fmaf(x[i], wa.y, acc[1]);
          acc[2] = fmaf(x[i], wa.z, acc[2]);
          acc[3] = fmaf(x[i], wa.w, acc[3]);
          acc[4] = fmaf(x[i], wb.x, acc[4]);
          acc[5] = fmaf(x[i], wb.y, acc[5]);
          acc[6] = fmaf(x[i], wb.z, acc[6]);
          acc[7] = fmaf(x[i], wb.w, acc[7]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) Kt[(c0 + c) * SP + s] = s < S ? acc[c] : 0.f;
      }
    }
  };

  // ---- trunk: K layers over the n_pos position rows (beam.py:159-163) -------
  // Warp 0 alone (n_pos <= 9 rows), reassociated so the trunk layers' K/V are
  // never built: scores (q Wk^T) X^T, output (P X) Wv.  Warps 1-7 build the
  // head layers' K/V meanwhile.
  if (K > 0 && wid == 0) {
    trunk_warp0<D>(a, Xs, SP, S, TR, TQ, wsl);
  } else {
    // head-layer K/V, built once and shared by every beam (beam.py:165-169)
    const int t0 = K > 0 ? 32 : 0;
    for (int i = K; i < L; ++i) build_kv(i, i - K, t0, kThreads - t0);
  }
  if (tid == 0) {
    par[0] = 0;
    tokm[0] = 0;
    cum[0] = 0.f;
  }
  __syncthreads();
  GR_STAMP(2);
  GR_STAMP(3);

  const int last = a.rerank ? T : T - 1;
  int live = 1;
  for (int t = 0; t <= last; ++t) {
    const int mo = a.moff[t];
    const int V = t < T ? a.V[t] : 0;
    for (int i = tid; i < 2048; i += kThreads) hist[i] = 0u;
    // Every candidate score of this level is cum_r + logp <= max_r cum_r =: Rs
    // (logp <= 0).  Candidates are binned by min((Rs - s) * scale, 2047), a
    // monotone map of the score, with 2048 bins over ln V + 4 score units,
    // so the k-th best usually lands in a bin holding a handful of keys.
    if (wid == 0) {
      float mc = -INFINITY;
      for (int j = lane; j < live; j += 32) mc = fmaxf(mc, cum[mo + j]);
      mc = warp_max(mc);
      if (lane == 0) {
        scr[48] = __float_as_uint(mc);
        scr[49] = __float_as_uint(2048.0f / (logf((float)max(V, 2)) + 4.0f));
      }
    }
    __syncthreads();
    const float Rs = __uint_as_float(scr[48]);
    const float bscale = __uint_as_float(scr[49]);
    auto sbin = [&](float sc) -> unsigned {
      return (unsigned)fminf((Rs - sc) * bscale, 2047.0f);  // NaN-free: sc <= Rs
    };
    int hcur = -1;
    unsigned hcnt = 0;
    for (int r0 = wid * RW; r0 < live; r0 += kWarps * RW) {
      const int r = r0 + rl;
      const bool ok = r < live;
      const int rr = ok ? r : live - 1;
      // ---- token input + gated fusion (beam.py:180-191; layers.py:129-133)
      float s[E], h[E], n[E], tt[E];
#pragma unroll
      for (int e = 0; e < E; ++e)
        s[e] = (t == 0) ? __ldg(W.bos + cb + e)
                        : __ldg(W.emb[t - 1] + (size_t)tokm[mo + rr] * D + cb + e);
      if (K > 0) {
        publish<E>(s, slot1);
        proj<E>(slot1, D, W.fuse_Wg, D, tt);
#pragma unroll
        for (int e = 0; e < E; ++e) tt[e] = TR[t * D + cb + e] * tt[e];  // m_t * (s W_g)
        publish<E>(tt, slot0);
        proj<E>(slot0, D, W.fuse_Wf, D, h);
        proj<E>(slot1, D, W.fuse_Wf + (size_t)D * D, D, tt);
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] += tt[e];
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] = s[e] + __ldg(W.pos + (size_t)t * D + cb + e);
      }
      // ---- head layers (layers.py:66-119, incremental) ----------------------
      for (int i = K; i < L; ++i) {
        const gr4ad_layer &Lw = W.layer[i];
        const float *Kt = KV + (size_t)(i - K) * 2 * KVS;
        layer_norm<E>(h, Lw.ln1_g, Lw.ln1_b, n);
        publish<E>(n, slot0);
        proj<E>(slot0, D, Lw.cross_Wq, D, tt);
        publish<E>(tt, slot1);
        cross_attn<D>(slot1, Kt, Kt + KVS, S, SP, slot2, tt);
        publish<E>(tt, slot0);
        proj<E>(slot0, D, Lw.cross_Wo, D, tt);
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] += tt[e];
        layer_norm<E>(h, Lw.ln2_g, Lw.ln2_b, n);
        publish<E>(n, slot0);
        float qs[E], ks[E], vs[E];
        proj<E>(slot0, D, Lw.self_Wqkv, 3 * D, qs);
        proj<E>(slot0, D, Lw.self_Wqkv + D, 3 * D, ks);
        proj<E>(slot0, D, Lw.self_Wqkv + 2 * D, 3 * D, vs);
        // self-attention over the ancestor chain (history by parent pointer):
        // own position first, then ancestors; online softmax (layers.py:101-113)
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) dot = fmaf(qs[e], ks[e], dot);
        float mx = rsum(dot) * scale, se = 1.f, so[E];
#pragma unroll
        for (int e = 0; e < E; ++e) so[e] = vs[e];
        int a_row = rr;
        for (int tau = t - 1; tau >= 0; --tau) {
          a_row = par[a.moff[tau + 1] + a_row];
          const float *hr = HI + ((size_t)(i - K) * a.Hrows + a.hoff[tau] + a_row) * 2 * D;
          float d2 = 0.f;
#pragma unroll
          for (int e = 0; e < E; ++e) d2 = fmaf(qs[e], hr[cb + e], d2);
          const float sc = rsum(d2) * scale;
          const float nm = fmaxf(mx, sc), f = expf(mx - nm), w = expf(sc - nm);
          se = se * f + w;
#pragma unroll
          for (int e = 0; e < E; ++e) so[e] = so[e] * f + w * hr[D + cb + e];
          mx = nm;
        }
        if (ok) {
          float *hrow = HI + ((size_t)(i - K) * a.Hrows + a.hoff[t] + r) * 2 * D;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            hrow[cb + e] = ks[e];
            hrow[D + cb + e] = vs[e];
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) so[e] /= se;
        publish<E>(so, slot0);
        proj<E>(slot0, D, Lw.self_Wo, D, tt);
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] += tt[e];
        layer_norm<E>(h, Lw.ln3_g, Lw.ln3_b, n);
        publish<E>(n, slot0);
        ffn<D>(slot0, slot3, Lw, dff, tt);
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] += tt[e] + __ldg(Lw.ffn_b2 + cb + e);
      }
      publish<E>(h, slot0);
      if (t == T) {  // value re-rank step (beam.py:258-288): rank in double
        float vl = -INFINITY;
        const int c = lane & 7;
        if (c < a.nb) {
          float acc = 0.f;
          for (int i = 0; i < D; ++i)
            acc = fmaf(slot0[i * 4 + rl], __ldg(W.head_value + (size_t)i * a.nb + c), acc);
          vl = acc;
        }
        const float mv = rmax(vl);
        double e1 = c < a.nb ? exp((double)vl - (double)mv) : 0.0;
        double se = e1;
        se += __shfl_xor_sync(kFull, se, 4);
        se += __shfl_xor_sync(kFull, se, 2);
        se += __shfl_xor_sync(kFull, se, 1);
        double ev = c < a.nb ? exp(((double)vl - (double)mv) - log(se)) *
                                   (double)__ldg(a.value_reps + c)
                             : 0.0;
        ev += __shfl_xor_sync(kFull, ev, 4);
        ev += __shfl_xor_sync(kFull, ev, 2);
        ev += __shfl_xor_sync(kFull, ev, 1);
        if (ok && c == 0) reinterpret_cast<double *>(sbuf)[r] = ev * exp((double)cum[mo + r]);
        continue;
      }
      // ---- codebook logits + log-softmax keys (beam.py:198-200) ---------------
      // lane owns tokens 8*lane .. 8*lane+7 of all four rows
      const float *head = W.head[t];
      const bool tv = lane * 8 < V;
      float lg[RW][8];
#pragma unroll
      for (int q = 0; q < RW; ++q)
#pragma unroll
        for (int c = 0; c < 8; ++c) lg[q][c] = 0.f;
#pragma unroll 4
      for (int i = 0; i < D; ++i) {
        const float4 x4 = *reinterpret_cast<const float4 *>(slot0 + i * 4);
        float4 wa = make_float4(0.f, 0.f, 0.f, 0.f), wb = wa;
        if (tv) {
          wa = __ldg(reinterpret_cast<const float4 *>(head + (size_t)i * V + lane * 8));
          wb = __ldg(reinterpret_cast<const float4 *>(head + (size_t)i * V + lane * 8 + 4));
        }
        const float xx[4] = {x4.x, x4.y, x4.z, x4.w};
        const float ww[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int q = 0; q < RW; ++q)
#pragma unroll
          for (int c = 0; c < 8; ++c) lg[q][c] = fmaf(xx[q], ww[c], lg[q][c]);
      }
#pragma unroll
      for (int q = 0; q < RW; ++q) {
        float mq = -INFINITY;
#pragma unroll
        for (int c = 0; c < 8; ++c) mq = fmaxf(mq, tv ? lg[q][c] : -INFINITY);
        const float mx = warp_max(mq);
        float s2 = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) s2 += tv ? __expf(lg[q][c] - mx) : 0.f;
        const float ls = logf(warp_sum(s2));
        const int rq = r0 + q;
        if (rq < live && tv) {
          const float cr = cum[mo + rq];
          uint32_t u[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            u[c] = f2ord(cr + ((lg[q][c] - mx) - ls));
            hist_add(hist, hcur, hcnt, (int)sbin(cr + ((lg[q][c] - mx) - ls)));
          }
          uint4 *kr = reinterpret_cast<uint4 *>(keys + (size_t)rq * V + lane * 8);
          kr[0] = make_uint4(u[0], u[1], u[2], u[3]);
          kr[1] = make_uint4(u[4], u[5], u[6], u[7]);
        }
      }
    }
    if (hcnt) atomicAdd(&hist[hcur], hcnt);
    __syncthreads();
    GR_STAMP(4 + 2 * t);

    live = select_level(a, b, t, live, V, keys, hist, scr, sbuf, par, tokm, cum, Rs, bscale);
    if (live < 0) return;
    __syncthreads();
    GR_STAMP(5 + 2 * t);
  }
  // results (beam.py:212-213)
  for (int j = tid; j < live; j += kThreads) {
    int ar = j;
    for (int tau = T - 1; tau >= 0; --tau) {
      a.out_tokens[((size_t)b * a.max_out + j) * T + tau] = tokm[a.moff[tau + 1] + ar];
      ar = par[a.moff[tau + 1] + ar];
    }
    a.out_score[(size_t)b * a.max_out + j] = (double)cum[a.moff[T] + j];
  }
  if (tid == 0) a.out_count[b] = live;
  GR_STAMP(15);
}

// ===========================================================================
// Warp-MMA variant (d = 16): every per-level product -- fused gate, head-layer
// projections, cross-attention Q.K^T and P.V, FFN, codebook logits -- runs on
// the tensor cores through mma.sync.m16n8k16 in 3xFP16 (lo.hi + hi.lo +
// hi.hi, fp32 accumulate; weights pre-scaled by kFragScale, context K / V by
// kKvScaleF), with a warp owning a 16-row tile.  The per-row state stays in C
// fragments: a pair of m16n8 C fragments is the A fragment of the next k16
// product, so no shuffles or shared-memory round trips between products.
// Cross-attention is flash-style (online softmax over key chunks) over K as
// fp16 hi / lo words (bank-swizzled) and V^T [D][S+8] in shared memory.
// Trunk, selection and compaction are the CUDA-core code above.
// ===========================================================================
// pull [p, p + bytes) toward this SM's L1 (128-B lines split over the CTA)
static __device__ __forceinline__ void prefetch_l1(const void *p, size_t bytes) {
  const char *c = static_cast<const char *>(p);
  for (size_t o = (size_t)threadIdx.x * 128; o < bytes; o += (size_t)kThreads * 128)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(c + o));
}

// ---- bulk async copy global -> shared (TMA engine) completing on an mbarrier
static __device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
static __device__ __forceinline__ void bar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: order earlier generic-proxy reads of dst before the async
// write, then copy `bytes` (multiple of 16) and arm the barrier
static __device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes,
                                                 uint64_t *bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
static __device__ __forceinline__ void bar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

static __device__ __forceinline__ uint32_t tf32_hi(float x) {
  return __float_as_uint(x) & 0xFFFFE000u;
}

// ---- 3xFP16 warp MMA (mma.sync m16n8k16, fp32 accumulate) -----------------
// x = hi + lo with hi = fp16(x), lo = fp16(x - hi); a product is accumulated
// as lo.hi + hi.lo + hi.hi (lo.lo ~2^-22 dropped).  Weight / codebook
// fragments and the context K / V^T are split after a power-of-two scale
// (their lo parts stay in fp16's normal range; results are rescaled exactly);
// activations are split unscaled.
constexpr float kFragScale = 2048.f, kInvFragScale = 1.f / 2048.f;  // weights, codebook
constexpr float kKvScaleF = 256.f, kInvKvScale = 1.f / 256.f;       // context K / V^T

static __device__ __forceinline__ uint32_t h2u(__half2 h) {
  return *reinterpret_cast<uint32_t *>(&h);
}
// (x0, x1) -> fp16x2 hi / lo
static __device__ __forceinline__ void split_h2(float x0, float x1, uint32_t &h, uint32_t &l) {
  const __half2 hh = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(hh);
  h = h2u(hh);
  l = h2u(__floats2half2_rn(x0 - hf.x, x1 - hf.y));
}

// C fragments (c0 (g,2t) c1 (g,2t+1) c2 (g+8,2t) c3 (g+8,2t+1)) of n-tiles
// 2kk (x0) and 2kk+1 (x1) are the A fragment of k16 step kk -- a0 (g, k 2t..)
// a1 (g+8, 2t..) a2 (g, 8+2t..) a3 (g+8, 8+2t..) -- so products chain with
// no data movement; split into fp16 hi / lo
static __device__ __forceinline__ void split_a16(const float (&x0)[4], const float (&x1)[4],
                                                 uint32_t (&h)[4], uint32_t (&l)[4]) {
  split_h2(x0[0], x0[1], h[0], l[0]);
  split_h2(x0[2], x0[3], h[1], l[1]);
  split_h2(x1[0], x1[1], h[2], l[2]);
  split_h2(x1[2], x1[3], h[3], l[3]);
}
template <int KT>
static __device__ __forceinline__ void split_frags(const float (&x)[KT][4],
                                                   uint32_t (&h)[KT / 2][4],
                                                   uint32_t (&l)[KT / 2][4]) {
#pragma unroll
  for (int k = 0; k < KT / 2; ++k) split_a16(x[2 * k], x[2 * k + 1], h[k], l[k]);
}

// B fragment {b0 hi, b1 hi, b0 lo, b1 lo}: b0 = s (x0, x1), b1 = s (x2, x3)
static __device__ __forceinline__ uint4 split_b16(float x0, float x1, float x2, float x3,
                                                  float sc) {
  uint4 r;
  split_h2(x0 * sc, x1 * sc, r.x, r.z);
  split_h2(x2 * sc, x3 * sc, r.y, r.w);
  return r;
}

static __device__ __forceinline__ void mma16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                             uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// d += a . b in 3xFP16
static __device__ __forceinline__ void mma3(float (&d)[4], const uint32_t (&ah)[4],
                                            const uint32_t (&al)[4], uint4 b) {
  mma16(d, al, b.x, b.y);
  mma16(d, ah, b.z, b.w);
  mma16(d, ah, b.x, b.y);
}

// dm += ah.bh, dx += al.bh + ah.bl: two independent accumulator chains
static __device__ __forceinline__ void mma3s(float (&dm)[4], float (&dx)[4],
                                             const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                             uint4 b) {
  mma16(dx, al, b.x, b.y);
  mma16(dx, ah, b.z, b.w);
  mma16(dm, ah, b.x, b.y);
}

static __device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(kFull, v, 1);
  v += __shfl_xor_sync(kFull, v, 2);
  return v;
}
static __device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(kFull, v, 1));
  v = fmaxf(v, __shfl_xor_sync(kFull, v, 2));
  return v;
}
static __device__ __forceinline__ double quad_sum_d(double v) {
  v += __shfl_xor_sync(kFull, v, 1);
  v += __shfl_xor_sync(kFull, v, 2);
  return v;
}

// y (16 x 8NT) (+)= x (16 x 8KT) . W, W fragment-ordered (k16 steps, scaled)
template <int KT, int NT, bool ACC = false>
static __device__ __forceinline__ void mm(const float (&x)[KT][4], const uint4 *__restrict__ W,
                                          float (&y)[NT][4]) {
  constexpr int K16 = KT / 2;
  uint32_t h[K16][4], l[K16][4];
  split_frags<KT>(x, h, l);
  const int lane = threadIdx.x & 31;
  uint4 w[K16][NT];
#pragma unroll
  for (int k = 0; k < K16; ++k)
#pragma unroll
    for (int n = 0; n < NT; ++n) w[k][n] = __ldg(W + (k * NT + n) * 32 + lane);
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    float dm[4] = {0.f, 0.f, 0.f, 0.f}, dx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < K16; ++k) mma3s(dm, dx, h[k], l[k], w[k][n]);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float v = (dm[c] + dx[c]) * kInvFragScale;
      y[n][c] = ACC ? y[n][c] + v : v;
    }
  }
}

// LayerNorm of the tile's rows (layers.py:38-51); row g in c0/c1, g + 8 in c2/c3
template <int NT>
static __device__ __forceinline__ void ln_frag(const float (&x)[NT][4], const float *g,
                                               const float *b, float (&y)[NT][4]) {
  const int t = threadIdx.x & 3;
  float sA = 0.f, sB = 0.f;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    sA += x[n][0] + x[n][1];
    sB += x[n][2] + x[n][3];
  }
  const float mA = quad_sum(sA) / (float)(8 * NT), mB = quad_sum(sB) / (float)(8 * NT);
  float vA = 0.f, vB = 0.f;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const float d0 = x[n][0] - mA, d1 = x[n][1] - mA, d2 = x[n][2] - mB, d3 = x[n][3] - mB;
    vA += d0 * d0 + d1 * d1;
    vB += d2 * d2 + d3 * d3;
  }
  const float iA = 1.0f / sqrtf(quad_sum(vA) / (float)(8 * NT) + 1e-5f);
  const float iB = 1.0f / sqrtf(quad_sum(vB) / (float)(8 * NT) + 1e-5f);
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const float2 gg = __ldg(reinterpret_cast<const float2 *>(g + 8 * n + 2 * t));
    const float2 bb = __ldg(reinterpret_cast<const float2 *>(b + 8 * n + 2 * t));
    y[n][0] = (x[n][0] - mA) * iA * gg.x + bb.x;
    y[n][1] = (x[n][1] - mA) * iA * gg.y + bb.y;
    y[n][2] = (x[n][2] - mB) * iB * gg.x + bb.x;
    y[n][3] = (x[n][3] - mB) * iB * gg.y + bb.y;
  }
}

// k_lo must be a multiple of 64 (chunks never cross SP; keys in [kend, c0+64)
// are masked, their K rows zero or finite).
// Cross-attention of the tile's 16 query rows against one request's shared
// K / V^T, both fp16 hi / lo of kKvScaleF * x in shared memory (kv_layout):
// online softmax over 64-key chunks (autodiff.py:362-368 up to the rescaling
// order).
template <int D>
static __device__ __forceinline__ void attn_mma(const float (&q)[D / 8][4], const uint32_t *Kw,
                                                const uint32_t *VTw, int S, int k_lo, int k_hi,
                                                float (&o)[D / 8][4], float (&ml)[4]) {
  constexpr int KT = D / 8, K16 = KT / 2, KW = D / 2, VSW = (SP + 8) / 2;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float scale = rsqrtf((float)D) * kInvKvScale;
  const uint32_t *Kl = Kw + SP * KW, *VTl = VTw + D * VSW;
  uint32_t qh[K16][4], ql[K16][4];
  split_frags<KT>(q, qh, ql);
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
  // P.V accumulators: hi.hi terms and cross terms
  float ox[KT][4];
#pragma unroll
  for (int n = 0; n < KT; ++n)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[n][c] = ox[n][c] = 0.f;
  const int kend = min(S, k_hi);
  const int sw = ((g >> 2) & 1) << 2;  // kv_layout: key bit 2 swaps the 4-word halves
  for (int c0 = k_lo; c0 < kend; c0 += 64) {
    float sc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
      const int r = (c0 + j * 8 + g) * KW;
#pragma unroll
      for (int k = 0; k < K16; ++k) {
        const int w0 = (8 * k + t) ^ sw, w1 = (8 * k + t + 4) ^ sw;
        mma3(sc[j], qh[k], ql[k], make_uint4(Kw[r + w0], Kw[r + w1], Kl[r + w0], Kl[r + w1]));
      }
    }
    float cA = -INFINITY, cB = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int key = c0 + j * 8 + 2 * t;
      const bool v0 = key < kend, v1 = key + 1 < kend;
      sc[j][0] = v0 ? sc[j][0] * scale : -INFINITY;
      sc[j][1] = v1 ? sc[j][1] * scale : -INFINITY;
      sc[j][2] = v0 ? sc[j][2] * scale : -INFINITY;
      sc[j][3] = v1 ? sc[j][3] * scale : -INFINITY;
      cA = fmaxf(cA, fmaxf(sc[j][0], sc[j][1]));
      cB = fmaxf(cB, fmaxf(sc[j][2], sc[j][3]));
    }
    const float nA = fmaxf(mA, quad_max(cA)), nB = fmaxf(mB, quad_max(cB));
    const float fA = __expf(mA - nA), fB = __expf(mB - nB);  // 0 on the first chunk
    lA *= fA;
    lB *= fB;
#pragma unroll
    for (int n = 0; n < KT; ++n) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float f = c < 2 ? fA : fB;
        o[n][c] *= f;
        ox[n][c] *= f;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j][0] = __expf(sc[j][0] - nA);  // arguments <= 0
      sc[j][1] = __expf(sc[j][1] - nA);
      sc[j][2] = __expf(sc[j][2] - nB);
      sc[j][3] = __expf(sc[j][3] - nB);
      lA += sc[j][0] + sc[j][1];
      lB += sc[j][2] + sc[j][3];
    }
    mA = nA;
    mB = nB;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      uint32_t ph[4], pl[4];
      split_a16(sc[2 * jj], sc[2 * jj + 1], ph, pl);
#pragma unroll
      for (int n = 0; n < KT; ++n) {
        const int v = (n * 8 + g) * VSW + (c0 >> 1) + 8 * jj + t;
        mma3s(o[n], ox[n], ph, pl, make_uint4(VTw[v], VTw[v + 4], VTl[v], VTl[v + 4]));
      }
    }
  }
#pragma unroll
  for (int n = 0; n < KT; ++n)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[n][c] = (o[n][c] + ox[n][c]) * kInvKvScale;
  ml[0] = mA;  // row g: running max, row g + 8; then the row sums
  ml[1] = mB;
  ml[2] = quad_sum(lA);
  ml[3] = quad_sum(lB);
}

// o / l of a single-warp attention
template <int KT>
static __device__ __forceinline__ void attn_normalize(float (&o)[KT][4], const float (&ml)[4]) {
  const float iA = 1.0f / ml[2], iB = 1.0f / ml[3];
#pragma unroll
  for (int n = 0; n < KT; ++n) {
    o[n][0] *= iA;
    o[n][1] *= iA;
    o[n][2] *= iB;
    o[n][3] *= iB;
  }
}

// Group of `wpt` warps sharing one 16-row tile (named barrier `bar_id`):
// combine the per-warp partial attentions (flash-style rescale) through the
// per-warp scratch (16 x (D + 2) floats each); every warp of the group ends
// with the same normalised o.
template <int D>
static __device__ __forceinline__ void attn_merge(float (&o)[D / 8][4], const float (&ml)[4],
                                                 float *scr_all, int part, int wpt, int bar_id) {
  constexpr int KT = D / 8, RS = D + 2;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  float *mine = scr_all + part * 16 * RS;
#pragma unroll
  for (int n = 0; n < KT; ++n) {
    *reinterpret_cast<float2 *>(mine + g * RS + 8 * n + 2 * t) = make_float2(o[n][0], o[n][1]);
    *reinterpret_cast<float2 *>(mine + (g + 8) * RS + 8 * n + 2 * t) = make_float2(o[n][2], o[n][3]);
  }
  if (t == 0) {
    mine[g * RS + D] = ml[0];
    mine[g * RS + D + 1] = ml[2];
    mine[(g + 8) * RS + D] = ml[1];
    mine[(g + 8) * RS + D + 1] = ml[3];
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * wpt) : "memory");
  float MA = -INFINITY, MB = -INFINITY;
  for (int p = 0; p < wpt; ++p) {
    MA = fmaxf(MA, scr_all[p * 16 * RS + g * RS + D]);
    MB = fmaxf(MB, scr_all[p * 16 * RS + (g + 8) * RS + D]);
  }
  float lA = 0.f, lB = 0.f;
#pragma unroll
  for (int n = 0; n < KT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  for (int p = 0; p < wpt; ++p) {
    const float *pp = scr_all + p * 16 * RS;
    const float fA = __expf(pp[g * RS + D] - MA), fB = __expf(pp[(g + 8) * RS + D] - MB);
    lA += pp[g * RS + D + 1] * fA;
    lB += pp[(g + 8) * RS + D + 1] * fB;
#pragma unroll
    for (int n = 0; n < KT; ++n) {
      const float2 a2 = *reinterpret_cast<const float2 *>(pp + g * RS + 8 * n + 2 * t);
      const float2 b2 = *reinterpret_cast<const float2 *>(pp + (g + 8) * RS + 8 * n + 2 * t);
      o[n][0] += a2.x * fA;
      o[n][1] += a2.y * fA;
      o[n][2] += b2.x * fB;
      o[n][3] += b2.y * fB;
    }
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * wpt) : "memory");  // scratch reuse
  const float iA = 1.0f / lA, iB = 1.0f / lB;
#pragma unroll
  for (int n = 0; n < KT; ++n) {
    o[n][0] *= iA;
    o[n][1] *= iA;
    o[n][2] *= iB;
    o[n][3] *= iB;
  }
}

template <int D, int DFF>
static __device__ __forceinline__ void ffn_mma(const float (&n)[D / 8][4], const gr4ad_layer &Lw,
                                               const uint4 *W1, const uint4 *W2,
                                               float (&h)[D / 8][4]) {
  constexpr int KT = D / 8, FT = DFF / 8;
  const int t = threadIdx.x & 3;
  float f[FT][4];
  mm<KT, FT>(n, W1, f);
#pragma unroll
  for (int j = 0; j < FT; ++j) {
    const float2 bb = __ldg(reinterpret_cast<const float2 *>(Lw.ffn_b1 + 8 * j + 2 * t));
    f[j][0] = gelu_fast(f[j][0] + bb.x);
    f[j][1] = gelu_fast(f[j][1] + bb.y);
    f[j][2] = gelu_fast(f[j][2] + bb.x);
    f[j][3] = gelu_fast(f[j][3] + bb.y);
  }
  float o[KT][4];
  mm<FT, KT>(f, W2, o);
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    const float2 bb = __ldg(reinterpret_cast<const float2 *>(Lw.ffn_b2 + 8 * j + 2 * t));
    h[j][0] += o[j][0] + bb.x;
    h[j][1] += o[j][1] + bb.y;
    h[j][2] += o[j][2] + bb.x;
    h[j][3] += o[j][3] + bb.y;
  }
}

// logits of the tile's rows for codebook tiles [n0, n0 + kLG) (clamped to nend)
// from the level's codebook fragments staged in shared memory
#ifndef GR_KLG
#define GR_KLG 4
#endif
constexpr int kLG = GR_KLG;  // codebook tiles per logits group
template <int K16>
static __device__ __forceinline__ void logits_s(const uint32_t (&hh)[K16][4],
                                                const uint32_t (&hl)[K16][4],
                                                const uint4 *__restrict__ Hs, int NTV, int n0,
                                                int nend, float (&z)[kLG][4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < kLG; ++j) {
    z[j][0] = z[j][1] = z[j][2] = z[j][3] = 0.f;
    if (n0 + j < nend) {
#pragma unroll
      for (int k = 0; k < K16; ++k) mma3(z[j], hh[k], hl[k], Hs[(k * NTV + n0 + j) * 32 + lane]);
#pragma unroll
      for (int c = 0; c < 4; ++c) z[j][c] *= kInvFragScale;
    } else {
      z[j][0] = z[j][1] = z[j][2] = z[j][3] = -INFINITY;
    }
  }
}

// A fragments (fp16 hi / lo, k16 steps) of rows cA (g) and cB (g + 8) of a
// row-major [rows][ld] state
template <int K16>
static __device__ __forceinline__ void load_split(const float *st, int ld, int cA, int cB,
                                                  uint32_t (&hh)[K16][4], uint32_t (&hl)[K16][4]) {
  const int t4 = threadIdx.x & 3;
#pragma unroll
  for (int k = 0; k < K16; ++k) {
    float c[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float2 a2 = *reinterpret_cast<const float2 *>(st + cA * ld + 16 * k + 8 * u + 2 * t4);
      const float2 b2 = *reinterpret_cast<const float2 *>(st + cB * ld + 16 * k + 8 * u + 2 * t4);
      c[u][0] = a2.x;
      c[u][1] = a2.y;
      c[u][2] = b2.x;
      c[u][3] = b2.y;
    }
    split_a16(c[0], c[1], hh[k], hl[k]);
  }
}

// Second logits pass of a tile (beam.py:198-200): recompute the logits, form
// the candidate scores cum_r + (z - M_r) - lse_r.  !COLLECT: store every key
// for the selection kernel path and histogram its bin.  COLLECT: append only
// the candidates whose bin is <= wb (the proxy window) to sbuf, counting in
// *cnt (entries past cap are counted, not written: the caller falls back).
struct RowScore {
  bool ok;
  int r;
  float cr, M, ls;
  uint32_t vb0, vb1;  // valid-SID masking: bit 2n + c <-> token 8n + 2 t4 + c (all set: no mask)
};

// Valid-SID prefix masking (oracle prefix_mask): this
// lane's valid-token bits of a row with prefix key P at level t, from the
// level's CSR table (rows of sorted valid (t+1)-prefix keys grouped by P)
static __device__ __forceinline__ void row_valid_bits(const FusedArgs &a, int t, int P, bool ok,
                                                      RowScore &R) {
  R.vb0 = R.vb1 = 0xFFFFFFFFu;
  if (!a.vp_rp[t]) return;
  R.vb0 = R.vb1 = 0u;
  if (!ok) return;
  const int V = a.V[t], t4 = threadIdx.x & 3;
  const int lo = __ldg(a.vp_rp[t] + P), hi = __ldg(a.vp_rp[t] + P + 1);
  const long long base = (long long)P * V;
  for (int i = lo; i < hi; ++i) {
    const int tok = (int)(__ldg(a.vp_keys[t] + i) - base);
    if (((tok & 7) >> 1) == t4) {
      const int bit = ((tok >> 3) << 1) | (tok & 1);
      if (bit < 32)
        R.vb0 |= 1u << bit;
      else
        R.vb1 |= 1u << (bit - 32);
    }
  }
}
static __device__ __forceinline__ bool tok_valid(const RowScore &R, int n, int c) {
  const int bit = (n << 1) | (c & 1);
  return ((bit < 32 ? R.vb0 : R.vb1) >> (bit & 31)) & 1u;
}
template <int KT, bool COLLECT, bool MASK>
static __device__ __forceinline__ void logits_pass2(
    const uint32_t (&hh)[KT][4], const uint32_t (&hl)[KT][4], const uint4 *Hf, int NTV, int nb0,
    int nb1, const RowScore &A, const RowScore &B, int V, uint32_t *keys, unsigned *hist,
    int &hcur, unsigned &hcnt, float Rs, float bscale, int wb, unsigned long long *sbuf,
    unsigned *cnt, int cap) {
  const int lane = threadIdx.x & 31, t4 = lane & 3;
  auto sbin = [&](float sc) -> unsigned { return (unsigned)fminf((Rs - sc) * bscale, 2047.0f); };
  // COLLECT pre-filter: bin <= wb needs s > Rs - (wb + 1) / bscale; the z bound
  // is loosened by 1e-3 and every pre-pass is checked exactly with sbin
  const float slo = Rs - (float)(wb + 1) / bscale - 1e-3f;
  const float zA = A.ok ? slo - A.cr + A.M + A.ls : INFINITY;
  const float zB = B.ok ? slo - B.cr + B.M + B.ls : INFINITY;
  for (int n0 = nb0; n0 < nb1; n0 += kLG) {
    float z[kLG][4];
    logits_s<KT>(hh, hl, Hf, NTV, n0, nb1, z);
    if (!COLLECT) {
#pragma unroll
      for (int j = 0; j < kLG; ++j) {
        const int col = (n0 + j) * 8 + 2 * t4;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const RowScore &R = side ? B : A;
          if (n0 + j < nb1 && R.ok) {
            // masked tokens: logp = -inf after the log-softmax (oracle prefix_mask)
            const float s0 = !MASK || tok_valid(R, n0 + j, 0) ? R.cr + ((z[j][2 * side] - R.M) - R.ls)
                                                     : -INFINITY;
            const float s1 = !MASK || tok_valid(R, n0 + j, 1)
                                 ? R.cr + ((z[j][2 * side + 1] - R.M) - R.ls)
                                 : -INFINITY;
            *reinterpret_cast<uint2 *>(keys + (size_t)R.r * V + col) = make_uint2(f2ord(s0), f2ord(s1));
            hist_add(hist, hcur, hcnt, (int)sbin(s0));
            hist_add(hist, hcur, hcnt, (int)sbin(s1));
          }
        }
      }
    } else {
      // exact window test of every value (branch-free), then one warp-wide
      // scan and one shared atomic per group; entries stored predicated
      unsigned pm = 0;  // bit 4j + c: value c of n-tile j is in the window
#pragma unroll
      for (int j = 0; j < kLG; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // padded tiles are -inf: never pass zA / zB
          const RowScore &R = c < 2 ? A : B;
          const float sc = R.cr + ((z[j][c] - R.M) - R.ls);
          const bool in = z[j][c] > (c < 2 ? zA : zB) && sbin(sc) <= (unsigned)wb &&
                          (!MASK || tok_valid(R, n0 + j, c));
          pm |= (in ? 1u : 0u) << (4 * j + c);
        }
      if (__any_sync(kFull, pm != 0)) {
        const unsigned np = __popc(pm);
        unsigned incl = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        unsigned base = 0;
        if (lane == 31) base = atomicAdd(cnt, incl);
        base = __shfl_sync(kFull, base, 31) + incl - np;
        // branch-free: every value's entry is formed, the store predicated
        // (a per-entry branch costs two warp reconvergence points)
#pragma unroll
        for (int j = 0; j < kLG; ++j)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const RowScore &R = c < 2 ? A : B;
            const bool take = (pm >> (4 * j + c)) & 1u;
            const float sc = R.cr + ((z[j][c] - R.M) - R.ls);
            const unsigned long long e =
                ((unsigned long long)f2ord(sc) << 32) |
                (0xFFFFFFFFu - (unsigned)(R.r * V + (n0 + j) * 8 + 2 * t4 + (c & 1)));
            if (take && base < (unsigned)cap) sbuf[base] = e;
            base += take ? 1u : 0u;
            }
      }
    }
  }
}

// MASK: valid-SID prefix masking compiled in (a separate instantiation, so
// the unmasked decode carries none of its checks)
template <int D, bool MASK>
__global__ void __launch_bounds__(kThreads, 2) fused_mma_kernel(FusedArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int KT = D / 8, VS = SP + 8, HS = 2 * D + 8;
  constexpr int KVL = SP * D + D * VS;
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int T = a.T, L = a.L, K = a.K;
  const int S = a.ctx_len[b];
  const long long coff = a.ctx_off[b];
  const gr4ad_weights &W = a.w;
  const float scale = 1.0f / sqrtf((float)D);

  float *XT = sm + a.s_XT;  // X^T [D][VS] (dead after the K/V build: aliases HI)
  float *KV = sm + a.s_KV;  // per head layer: K [SP][D] (k_swz), V^T [D][VS]
  float *TR = sm + a.s_TR;
  float *TQ = sm + a.s_TQ;
  float *HI = sm + a.s_hist;  // self-KV history rows [k | v | pad] (HS floats)
  int *par = reinterpret_cast<int *>(sm + a.s_par);
  int *tokm = reinterpret_cast<int *>(sm + a.s_tok);
  int *pfx = reinterpret_cast<int *>(sm + a.s_pfx);  // rows' SID prefix keys (masking)
  float *cum = sm + a.s_cum;
  unsigned *hist = reinterpret_cast<unsigned *>(sm + a.s_bins);
  unsigned *scr = reinterpret_cast<unsigned *>(sm + a.s_scr);
  unsigned long long *sbuf = reinterpret_cast<unsigned long long *>(sm + a.s_sort);
  float *wsl = sm + a.s_ws;  // warp 0's trunk slots
  float *mrg = sm + a.s_mrg;  // per-warp partials of tile groups: 16 x (D + 2) each
  uint4 *HS2 = reinterpret_cast<uint4 *>(sm + a.s_head);  // level codebook fragments (bulk copy)
  constexpr int HSD = D + 2;      // per-row pass-2 state: head input h, M, lse
  float *hst = sm + a.s_hst;      // [hst_rows][HSD]
  float *prox = reinterpret_cast<float *>(sm + a.s_sort);  // window proxies (before collection)
  uint64_t *hbar = reinterpret_cast<uint64_t *>(sm + a.s_mbar);
  uint32_t *keys = a.keys + (size_t)b * a.keys_per_req;
  GR_STAMP(0);
  uint64_t *fbar = hbar + 1;
  // the request's features land in HS2 by one bulk copy (HS2 takes the
  // level-0 codebook after the projection)
  const bool feat_bulk = a.features && a.F % 4 == 0 && S * a.F <= a.head_floats &&
                         (coff * a.F) % 4 == 0;
  if (tid == 0) {
    bar_init(hbar);
    bar_init(fbar);
    if (feat_bulk)
      bulk_load(HS2, a.features + coff * a.F, (uint32_t)(S * a.F * sizeof(float)), fbar);
  }
  __syncthreads();
  // one bulk copy per level into HS2, issued by thread 0 one level ahead;
  // phase t of hbar completes when level t's codebook has landed

  // ---- context projection X = F W_c + b_c (decoder.py:134-140) -------------
  for (int s = tid; s < SP; s += kThreads) {
    float x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = 0.f;
    if (s < S) {
      if (feat_bulk) {
        bar_wait(fbar, 0);
        const float4 *f4 = reinterpret_cast<const float4 *>(HS2) + s * (a.F / 4);
        for (int i0 = 0; i0 < a.F; i0 += 4) {
          const float4 fv = f4[i0 / 4];
          const float fa[4] = {fv.x, fv.y, fv.z, fv.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int j = 0; j < D; j += 4) {
              const float4 w4 =
                  __ldg(reinterpret_cast<const float4 *>(W.ctx_W + (size_t)(i0 + u) * D + j));
              x[j] = fmaf(fa[u], w4.x, x[j]);
              x[j + 1] = fmaf(fa[u], w4.y, x[j + 1]);
              x[j + 2] = fmaf(fa[u], w4.z, x[j + 2]);
              x[j + 3] = fmaf(fa[u], w4.w, x[j + 3]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] += __ldg(W.ctx_b + j);
      } else if (a.features) {
        const float *f = a.features + (coff + s) * a.F;
        for (int i0 = 0; i0 < a.F; i0 += 16) {  // 16 independent loads in flight
          float fv[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) fv[u] = i0 + u < a.F ? __ldg(f + i0 + u) : 0.f;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            if (i0 + u >= a.F) break;
#pragma unroll
            for (int j = 0; j < D; j += 4) {
              const float4 w4 =
                  __ldg(reinterpret_cast<const float4 *>(W.ctx_W + (size_t)(i0 + u) * D + j));
              x[j] = fmaf(fv[u], w4.x, x[j]);
              x[j + 1] = fmaf(fv[u], w4.y, x[j + 1]);
              x[j + 2] = fmaf(fv[u], w4.z, x[j + 2]);
              x[j + 3] = fmaf(fv[u], w4.w, x[j + 3]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] += __ldg(W.ctx_b + j);
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = __ldg(a.context + (coff + s) * D + j);
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) XT[j * VS + s] = x[j];
  }
  __syncthreads();
  if (tid == 0 && T > 0) {  // level 0's codebook lands during the K/V + trunk phase
    if (feat_bulk) bar_wait(fbar, 0);  // (complete: every thread waited on it)
    bulk_load(HS2, a.frag + a.fi.head[0], (uint32_t)(D * a.V[0] * sizeof(float)), hbar);
  }
  GR_STAMP(1);

  // ---- head-layer K / V^T (beam.py:165-169) by warps 1-7 while warp 0 runs
  // the trunk; thread owns keys, X column in registers
  if (K > 0 && wid == 0) {
    trunk_warp0<D>(a, XT, VS, S, TR, TQ, wsl, a.trunk_u);
    GR_WSTAMP(16);
  } else {
    // with a trunk, warp 4 (warp 0's SMSP) stays idle so the trunk warp -- the
    // phase's critical path -- does not share its scheduler with K/V work
    // (six warps need two rounds over the 256 keys, as seven do)
    const bool spare = K > 0;
    const int kv_t = !spare ? tid : (wid < 4 ? tid - 32 : tid - 64);
    const int nt = !spare ? kThreads : kThreads - 64;
    const int ldw = 2 * L * D;
    for (int i = K; i < L && !(spare && wid == 4); ++i) {
      float *Kl = KV + (size_t)(i - K) * KVL, *VTl = Kl + SP * D;
      const float *Wl = W.cross_kv_W + (size_t)(2 * i) * D;
      for (int s = kv_t; s < SP; s += nt) {
        float x[D];
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = XT[j * VS + s];
#pragma unroll 1
        for (int c0 = 0; c0 < 2 * D; c0 += 8) {
          float acc[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = 0.f;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const float4 wa = __ldg(reinterpret_cast<const float4 *>(Wl + (size_t)j * ldw + c0));
            const float4 wb = __ldg(reinterpret_cast<const float4 *>(Wl + (size_t)j * ldw + c0 + 4));
            acc[0] = fmaf(x[j], wa.x, acc[0]);
            acc[1] = fmaf(x[j], wa.y, acc[1]);
            acc[2] = fmaf(x[j], wa.z, acc[2]);
            acc[3] = fmaf(x[j], wa.w, acc[3]);
            acc[4] = fmaf(x[j], wb.x, acc[4]);
            acc[5] = fmaf(x[j], wb.y, acc[5]);
            acc[6] = fmaf(x[j], wb.z, acc[6]);
            acc[7] = fmaf(x[j], wb.w, acc[7]);
          }
          if (s >= S)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = 0.f;
          // kv_layout (attn_mma): K as fp16 words [SP][D/2] (hi, then lo),
          // 4-word halves swapped on key bit 2; V^T as fp16 [D][SP + 8]
#pragma unroll
          for (int c = 0; c < 8; ++c) range_check(acc[c] * kKvScaleF, a.range_flag);
          if (c0 < D) {
            uint4 hi, lo;
            split_h2(acc[0] * kKvScaleF, acc[1] * kKvScaleF, hi.x, lo.x);
            split_h2(acc[2] * kKvScaleF, acc[3] * kKvScaleF, hi.y, lo.y);
            split_h2(acc[4] * kKvScaleF, acc[5] * kKvScaleF, hi.z, lo.z);
            split_h2(acc[6] * kKvScaleF, acc[7] * kKvScaleF, hi.w, lo.w);
            const int w = s * (D / 2) + ((c0 / 2) ^ (((s >> 2) & 1) << 2));
            uint32_t *kw = reinterpret_cast<uint32_t *>(Kl);
            *reinterpret_cast<uint4 *>(kw + w) = hi;
            *reinterpret_cast<uint4 *>(kw + SP * (D / 2) + w) = lo;
          } else {
            __half *vh = reinterpret_cast<__half *>(VTl), *vl = vh + D * VS;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float x = acc[c] * kKvScaleF;
              const __half hx = __float2half_rn(x);
              vh[(c0 - D + c) * VS + s] = hx;
              vl[(c0 - D + c) * VS + s] = __float2half_rn(x - __half2float(hx));
            }
          }
        }
      }
    }
    if (wid == 1) GR_WSTAMP(17);
  }
  if (tid == 0) {
    par[0] = 0;
    tokm[0] = 0;
    cum[0] = 0.f;
    pfx[0] = 0;
  }
  __syncthreads();
  GR_STAMP(2);
  GR_STAMP(3);

  const int last = a.rerank ? T : T - 1;
  int live = 1;
  for (int t = 0; t <= last; ++t) {
    const int mo = a.moff[t];
    const int V = t < T ? a.V[t] : 0;
    for (int i = tid; i < 2048; i += kThreads) hist[i] = 0u;
    if (wid == 0) {
      float mc = -INFINITY;
      for (int j = lane; j < live; j += 32) mc = fmaxf(mc, cum[mo + j]);
      mc = warp_max(mc);
      if (lane == 0) {
        scr[48] = __float_as_uint(mc);
        scr[49] = __float_as_uint(2048.0f / (logf((float)max(V, 2)) + 4.0f));
      }
    }
    __syncthreads();
    const float Rs = __uint_as_float(scr[48]);
    const float bscale = __uint_as_float(scr[49]);
    auto sbin = [&](float sc) -> unsigned {
      return (unsigned)fminf((Rs - sc) * bscale, 2047.0f);
    };
    int hcur = -1;
    unsigned hcnt = 0;
    // 16-row tiles; with fewer than 8 tiles a group of wpt warps shares a
    // tile (keys and codebook tiles split, per-row work duplicated)
    const int n_tiles = (live + 15) / 16;
    int wpt = 1;
    while (a.tile_split && n_tiles * wpt * 2 <= kWarps) wpt *= 2;
    const int part = wid % wpt, bar_id = 1 + wid / wpt;
    float *gscr = mrg + (wid / wpt) * wpt * 16 * (D + 2);
    // proxy-window selection (needs the per-row state and the proxies on chip)
    const bool theta = t < T && live > 0 && live <= a.hst_rows && n_tiles * wpt * 128 <= 2 * a.sort_cap;
    for (int tile = wid / wpt; tile < n_tiles; tile += kWarps / wpt) {
      const int r0 = tile * 16;
      const int rA = r0 + g, rB = rA + 8;
      const bool okA = rA < live, okB = rB < live;
      const int cA = min(rA, live - 1), cB = min(rB, live - 1);
      // ---- token input + gated fusion (beam.py:180-191; layers.py:129-133)
      float s[KT][4], h[KT][4];
#pragma unroll
      for (int n = 0; n < KT; ++n) {
        const int col = 8 * n + 2 * t4;
        float2 xa, xb;
        if (t == 0) {
          xa = xb = __ldg(reinterpret_cast<const float2 *>(W.bos + col));
        } else {
          xa = __ldg(reinterpret_cast<const float2 *>(W.emb[t - 1] + (size_t)tokm[mo + cA] * D + col));
          xb = __ldg(reinterpret_cast<const float2 *>(W.emb[t - 1] + (size_t)tokm[mo + cB] * D + col));
        }
        s[n][0] = xa.x;
        s[n][1] = xa.y;
        s[n][2] = xb.x;
        s[n][3] = xb.y;
      }
      if (K > 0) {
        float m[KT][4];
        mm<KT, KT>(s, a.frag + a.fi.wg, m);
#pragma unroll
        for (int n = 0; n < KT; ++n) {
          const float2 tr = *reinterpret_cast<const float2 *>(TR + t * D + 8 * n + 2 * t4);
          m[n][0] *= tr.x;  // m_t * (s W_g)
          m[n][1] *= tr.y;
          m[n][2] *= tr.x;
          m[n][3] *= tr.y;
        }
        mm<KT, KT>(m, a.frag + a.fi.wf_m, h);
        mm<KT, KT, true>(s, a.frag + a.fi.wf_s, h);
      } else {
#pragma unroll
        for (int n = 0; n < KT; ++n) {
          const float2 pp = __ldg(reinterpret_cast<const float2 *>(W.pos + (size_t)t * D + 8 * n + 2 * t4));
          h[n][0] = s[n][0] + pp.x;
          h[n][1] = s[n][1] + pp.y;
          h[n][2] = s[n][2] + pp.x;
          h[n][3] = s[n][3] + pp.y;
        }
      }
      GR_SUB(0);
      // ---- head layers (layers.py:66-119, incremental) ------------------------
      for (int i = K; i < L; ++i) {
        const int li = i - K;
        const gr4ad_layer &Lw = W.layer[i];
        const uint32_t *KVw = reinterpret_cast<const uint32_t *>(KV + (size_t)li * KVL);
        float n[KT][4], q[KT][4], o[KT][4];
        ln_frag<KT>(h, Lw.ln1_g, Lw.ln1_b, n);
        mm<KT, KT>(n, a.frag + a.fi.cq[li], q);
        GR_SUB(1);
        {
          float ml[4];
          if (wpt == 1) {
            attn_mma<D>(q, KVw, KVw + SP * D, S, 0, SP, o, ml);
            attn_normalize<KT>(o, ml);
          } else {
            // whole 64-key chunks per warp (keys >= S are zero rows, masked)
            const int span = ((S + wpt - 1) / wpt + 63) / 64 * 64;
            attn_mma<D>(q, KVw, KVw + SP * D, S, part * span, (part + 1) * span, o, ml);
            attn_merge<D>(o, ml, gscr, part, wpt, bar_id);
          }
        }
        GR_SUB(2);
        mm<KT, KT, true>(o, a.frag + a.fi.co[li], h);
        ln_frag<KT>(h, Lw.ln2_g, Lw.ln2_b, n);
        float ks[KT][4], vs[KT][4];
        mm<KT, KT>(n, a.frag + a.fi.sq[li], q);
        mm<KT, KT>(n, a.frag + a.fi.sk[li], ks);
        mm<KT, KT>(n, a.frag + a.fi.sv[li], vs);
        // self-attention over the ancestor chain (history by parent pointer):
        // own position first, then ancestors; online softmax (layers.py:101-113)
        float dA = 0.f, dB = 0.f;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          dA = fmaf(q[j][0], ks[j][0], fmaf(q[j][1], ks[j][1], dA));
          dB = fmaf(q[j][2], ks[j][2], fmaf(q[j][3], ks[j][3], dB));
        }
        float mxA = quad_sum(dA) * scale, mxB = quad_sum(dB) * scale, seA = 1.f, seB = 1.f;
#pragma unroll
        for (int j = 0; j < KT; ++j)
#pragma unroll
          for (int c = 0; c < 4; ++c) o[j][c] = vs[j][c];
        int arA = cA, arB = cB;
        for (int tau = t - 1; tau >= 0; --tau) {
          arA = par[a.moff[tau + 1] + arA];
          arB = par[a.moff[tau + 1] + arB];
          const float *hA = HI + ((size_t)li * a.Hrows + a.hoff[tau] + arA) * HS + 2 * t4;
          const float *hB = HI + ((size_t)li * a.Hrows + a.hoff[tau] + arB) * HS + 2 * t4;
          float eA = 0.f, eB = 0.f;
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const float2 ka = *reinterpret_cast<const float2 *>(hA + 8 * j);
            const float2 kb = *reinterpret_cast<const float2 *>(hB + 8 * j);
            eA = fmaf(q[j][0], ka.x, fmaf(q[j][1], ka.y, eA));
            eB = fmaf(q[j][2], kb.x, fmaf(q[j][3], kb.y, eB));
          }
          const float scA = quad_sum(eA) * scale, scB = quad_sum(eB) * scale;
          const float nA = fmaxf(mxA, scA), fA = expf(mxA - nA), wA = expf(scA - nA);
          const float nB = fmaxf(mxB, scB), fB = expf(mxB - nB), wB = expf(scB - nB);
          seA = seA * fA + wA;
          seB = seB * fB + wB;
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const float2 va = *reinterpret_cast<const float2 *>(hA + D + 8 * j);
            const float2 vb = *reinterpret_cast<const float2 *>(hB + D + 8 * j);
            o[j][0] = o[j][0] * fA + wA * va.x;
            o[j][1] = o[j][1] * fA + wA * va.y;
            o[j][2] = o[j][2] * fB + wB * vb.x;
            o[j][3] = o[j][3] * fB + wB * vb.y;
          }
          mxA = nA;
          mxB = nB;
        }
        if (t < last && part == 0) {  // the last level's history is never read
          float *wA = HI + ((size_t)li * a.Hrows + a.hoff[t] + rA) * HS + 2 * t4;
          float *wB = HI + ((size_t)li * a.Hrows + a.hoff[t] + rB) * HS + 2 * t4;
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            if (okA) {
              *reinterpret_cast<float2 *>(wA + 8 * j) = make_float2(ks[j][0], ks[j][1]);
              *reinterpret_cast<float2 *>(wA + D + 8 * j) = make_float2(vs[j][0], vs[j][1]);
            }
            if (okB) {
              *reinterpret_cast<float2 *>(wB + 8 * j) = make_float2(ks[j][2], ks[j][3]);
              *reinterpret_cast<float2 *>(wB + D + 8 * j) = make_float2(vs[j][2], vs[j][3]);
            }
          }
        }
        const float iA = 1.0f / seA, iB = 1.0f / seB;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          o[j][0] *= iA;
          o[j][1] *= iA;
          o[j][2] *= iB;
          o[j][3] *= iB;
        }
        mm<KT, KT, true>(o, a.frag + a.fi.so[li], h);
        ln_frag<KT>(h, Lw.ln3_g, Lw.ln3_b, n);
        if (a.dff == 2 * D)
          ffn_mma<D, 2 * D>(n, Lw, a.frag + a.fi.w1[li], a.frag + a.fi.w2[li], h);
        else
          ffn_mma<D, D>(n, Lw, a.frag + a.fi.w1[li], a.frag + a.fi.w2[li], h);
      }
      if (t == T) {  // value re-rank step (beam.py:258-288): rank in double
        float vl[1][4];
        mm<KT, 1>(h, a.frag + a.fi.value, vl);
        const int c0 = 2 * t4, c1 = c0 + 1;
        const bool u0 = c0 < a.nb, u1 = c1 < a.nb;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const float v0 = vl[0][2 * side], v1 = vl[0][2 * side + 1];
          const float mv = quad_max(fmaxf(u0 ? v0 : -INFINITY, u1 ? v1 : -INFINITY));
          const double se = quad_sum_d((u0 ? exp((double)v0 - (double)mv) : 0.0) +
                                       (u1 ? exp((double)v1 - (double)mv) : 0.0));
          const double ls = log(se);
          double ev = (u0 ? exp(((double)v0 - (double)mv) - ls) * (double)__ldg(a.value_reps + c0) : 0.0) +
                      (u1 ? exp(((double)v1 - (double)mv) - ls) * (double)__ldg(a.value_reps + c1) : 0.0);
          ev = quad_sum_d(ev);
          const int r = side ? rB : rA;
          if ((side ? okB : okA) && t4 == 0 && part == 0)
            reinterpret_cast<double *>(sbuf)[r] = ev * exp((double)cum[mo + r]);
        }
        continue;
      }
      GR_SUB(3);
      // ---- codebook logits + log-softmax keys (beam.py:198-200) ---------------
      bar_wait(hbar, (uint32_t)(t & 1));
      const uint4 *Hf = HS2;
      const int NTV = V / 8;
      uint32_t hh[KT / 2][4], hl[KT / 2][4];
      split_frags<KT>(h, hh, hl);
      const int per = (NTV + wpt - 1) / wpt;
      const int nb0 = min(NTV, part * per), nb1 = min(NTV, nb0 + per);
      float mA = -INFINITY, mB = -INFINITY, sA = 0.f, sB = 0.f;
      RowScore RA{okA, rA, 0.f, 0.f, 0.f, 0u, 0u}, RB{okB, rB, 0.f, 0.f, 0.f, 0u, 0u};
      if (MASK) {
        row_valid_bits(a, t, pfx[mo + cA], okA, RA);
        row_valid_bits(a, t, pfx[mo + cB], okB, RB);
      }
      float p1A = -INFINITY, p2A = -INFINITY, p1B = -INFINITY, p2B = -INFINITY;  // lane top-2
      for (int n0 = nb0; n0 < nb1; n0 += kLG) {
        float z[kLG][4];
        logits_s<KT / 2>(hh, hl, Hf, NTV, n0, nb1, z);
        float gA = -INFINITY, gB = -INFINITY;
#pragma unroll
        for (int j = 0; j < kLG; ++j) {
          gA = fmaxf(gA, fmaxf(z[j][0], z[j][1]));
          gB = fmaxf(gB, fmaxf(z[j][2], z[j][3]));
          if (theta) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {  // proxies: valid candidates only
              const float za = !MASK || tok_valid(RA, n0 + j, c) ? z[j][c] : -INFINITY;
              const float zb = !MASK || tok_valid(RB, n0 + j, c) ? z[j][2 + c] : -INFINITY;
              p2A = fmaxf(p2A, fminf(p1A, za));
              p1A = fmaxf(p1A, za);
              p2B = fmaxf(p2B, fminf(p1B, zb));
              p1B = fmaxf(p1B, zb);
            }
          }
        }
        const float nA = fmaxf(mA, gA), nB = fmaxf(mB, gB);
        sA *= __expf(mA - nA);
        sB *= __expf(mB - nB);
#pragma unroll
        for (int j = 0; j < kLG; ++j) {
          sA += __expf(z[j][0] - nA) + __expf(z[j][1] - nA);
          sB += __expf(z[j][2] - nB) + __expf(z[j][3] - nB);
        }
        mA = nA;
        mB = nB;
      }
      float MA = quad_max(mA), MB = quad_max(mB);
      float SA = quad_sum(mA == -INFINITY ? 0.f : sA * __expf(mA - MA));
      float SB = quad_sum(mB == -INFINITY ? 0.f : sB * __expf(mB - MB));
      if (wpt > 1) {  // combine (max, sum) over the group's codebook slices
        if (t4 == 0) {
          gscr[(part * 16 + g) * 2] = MA;
          gscr[(part * 16 + g) * 2 + 1] = SA;
          gscr[(part * 16 + g + 8) * 2] = MB;
          gscr[(part * 16 + g + 8) * 2 + 1] = SB;
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * wpt) : "memory");
        float XA = -INFINITY, XB = -INFINITY;
        for (int p2 = 0; p2 < wpt; ++p2) {
          XA = fmaxf(XA, gscr[(p2 * 16 + g) * 2]);
          XB = fmaxf(XB, gscr[(p2 * 16 + g + 8) * 2]);
        }
        float YA = 0.f, YB = 0.f;
        for (int p2 = 0; p2 < wpt; ++p2) {
          const float ma = gscr[(p2 * 16 + g) * 2], mb = gscr[(p2 * 16 + g + 8) * 2];
          if (ma != -INFINITY) YA += gscr[(p2 * 16 + g) * 2 + 1] * __expf(ma - XA);
          if (mb != -INFINITY) YB += gscr[(p2 * 16 + g + 8) * 2 + 1] * __expf(mb - XB);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * wpt) : "memory");
        MA = XA;
        MB = XB;
        SA = YA;
        SB = YB;
      }
      const float lsA = logf(SA), lsB = logf(SB);
      GR_SUB(4);
      RA.cr = cum[mo + cA];
      RA.M = MA;
      RA.ls = lsA;
      RB.cr = cum[mo + cB];
      RB.M = MB;
      RB.ls = lsB;
      if (theta) {
        // save the tile's head input and (M, lse) for pass 2; emit the
        // per-lane top-2 candidates of each row as window proxies
        if (part == 0) {
#pragma unroll
          for (int n = 0; n < KT; ++n) {
            if (okA) *reinterpret_cast<float2 *>(hst + rA * HSD + 8 * n + 2 * t4) = make_float2(h[n][0], h[n][1]);
            if (okB) *reinterpret_cast<float2 *>(hst + rB * HSD + 8 * n + 2 * t4) = make_float2(h[n][2], h[n][3]);
          }
          if (t4 == 0) {
            if (okA) { hst[rA * HSD + D] = MA; hst[rA * HSD + D + 1] = lsA; }
            if (okB) { hst[rB * HSD + D] = MB; hst[rB * HSD + D + 1] = lsB; }
          }
        }
        float4 px;
        px.x = okA && p1A > -INFINITY ? RA.cr + ((p1A - MA) - lsA) : -INFINITY;
        px.y = okA && p2A > -INFINITY ? RA.cr + ((p2A - MA) - lsA) : -INFINITY;
        px.z = okB && p1B > -INFINITY ? RB.cr + ((p1B - MB) - lsB) : -INFINITY;
        px.w = okB && p2B > -INFINITY ? RB.cr + ((p2B - MB) - lsB) : -INFINITY;
        reinterpret_cast<float4 *>(prox)[(tile * wpt + part) * 32 + lane] = px;
      } else {
        logits_pass2<KT / 2, false, MASK>(hh, hl, Hf, NTV, nb0, nb1, RA, RB, V, keys, hist, hcur, hcnt, Rs,
                                bscale, 0, sbuf, nullptr, 0);
      }
      GR_SUB(5);
    }
    int collected = -1;
    if (theta) {
      // window from the proxies: >= k real candidates have bin <= wb, so the
      // whole top k does; collect those in pass 2 and sort them exactly
      __syncthreads();
      const int nprox = n_tiles * wpt * 128;
      const int kk = min(a.eff[t * a.B + b], live * V);
      const bool all_fit = live * V <= a.sort_cap;  // collect every candidate, no window
      int hc2 = -1;
      unsigned hn2 = 0, nfin = 0;
      if (tid == 0) {
        scr[40] = 0;
        scr[41] = 0;
      }
      __syncthreads();
      if (!all_fit) {
        for (int i = tid; i < nprox; i += kThreads) {
          const float v = prox[i];
          if (v > -INFINITY) {
            hist_add(hist, hc2, hn2, (int)sbin(v));
            ++nfin;
          }
        }
        if (hn2) atomicAdd(&hist[hc2], hn2);
        nfin = __reduce_add_sync(kFull, nfin);
        if (lane == 0 && nfin) atomicAdd(&scr[41], nfin);
        __syncthreads();
      }
      int wb = 2047;  // fewer than k proxies: collect every candidate
      if (!all_fit && scr[41] >= (unsigned)kk) {
        for (int i = tid; i < 1024; i += kThreads) {  // mirror: find_bin scans from the top
          const unsigned x = hist[i], y = hist[2047 - i];
          hist[i] = y;
          hist[2047 - i] = x;
        }
        __syncthreads();
        unsigned above;
        wb = 2047 - find_bin(hist, 2048, (unsigned)kk, &above, scr);
      }
      GR_SUB(6);
      for (int tile = wid / wpt; tile < n_tiles; tile += kWarps / wpt) {
        const int rA = tile * 16 + g, rB = rA + 8;
        const bool okA = rA < live, okB = rB < live;
        const int cA = min(rA, live - 1), cB = min(rB, live - 1);
        RowScore RA{okA, rA, cum[mo + cA], hst[cA * HSD + D], hst[cA * HSD + D + 1], 0u, 0u};
        RowScore RB{okB, rB, cum[mo + cB], hst[cB * HSD + D], hst[cB * HSD + D + 1], 0u, 0u};
        if (MASK) {
          row_valid_bits(a, t, pfx[mo + cA], okA, RA);
          row_valid_bits(a, t, pfx[mo + cB], okB, RB);
        }
        uint32_t hh[KT / 2][4], hl[KT / 2][4];
        load_split<KT / 2>(hst, HSD, cA, cB, hh, hl);
        const int NTV = V / 8, per = (NTV + wpt - 1) / wpt;
        const int nb0 = min(NTV, part * per), nb1 = min(NTV, nb0 + per);
        logits_pass2<KT / 2, true, MASK>(hh, hl, HS2, NTV, nb0, nb1, RA, RB, V, keys, hist, hcur, hcnt, Rs,
                               bscale, wb, sbuf, &scr[40], a.sort_cap);
      }
      GR_SUB(7);
      GR_XSTAMP(1, 42);
      GR_XSTAMP(2, 43);
      GR_XSTAMP(3, 44);
      GR_XSTAMP(5, 45);
      GR_XSTAMP(7, 46);
      __syncthreads();
      collected = (int)scr[40];
#if defined(GR_FUSED_TIMING) && !defined(GR_NO_XSTAMP)
      if (t == 2 && tid == 0) a.dbg[blockIdx.x * kDbgSlots + 47] = collected;
#endif
      if (collected > a.sort_cap) {
        // window overflow: exact path -- every key to the scratch + histogram
        collected = -1;
        for (int i = tid; i < 2048; i += kThreads) hist[i] = 0u;
        __syncthreads();
        for (int tile = wid / wpt; tile < n_tiles; tile += kWarps / wpt) {
          const int rA = tile * 16 + g, rB = rA + 8;
          const bool okA = rA < live, okB = rB < live;
          const int cA = min(rA, live - 1), cB = min(rB, live - 1);
          RowScore RA{okA, rA, cum[mo + cA], hst[cA * HSD + D], hst[cA * HSD + D + 1], 0u, 0u};
          RowScore RB{okB, rB, cum[mo + cB], hst[cB * HSD + D], hst[cB * HSD + D + 1], 0u, 0u};
          if (MASK) {
            row_valid_bits(a, t, pfx[mo + cA], okA, RA);
            row_valid_bits(a, t, pfx[mo + cB], okB, RB);
          }
          uint32_t hh[KT / 2][4], hl[KT / 2][4];
          load_split<KT / 2>(hst, HSD, cA, cB, hh, hl);
          const int NTV = V / 8, per = (NTV + wpt - 1) / wpt;
          const int nb0 = min(NTV, part * per), nb1 = min(NTV, nb0 + per);
          logits_pass2<KT / 2, false, MASK>(hh, hl, HS2, NTV, nb0, nb1, RA, RB, V, keys, hist, hcur, hcnt,
                                  Rs, bscale, 0, sbuf, nullptr, 0);
        }
      }
    }
    if (hcnt) atomicAdd(&hist[hcur], hcnt);
    __syncthreads();
    GR_STAMP(4 + 2 * t);
    if (tid == 0 && t + 1 < T) {  // next level's codebook lands during this selection
      bar_wait(hbar, (uint32_t)(t & 1));  // level t's copy is complete (also with no tiles)
      bulk_load(HS2, a.frag + a.fi.head[t + 1], (uint32_t)(D * a.V[t + 1] * sizeof(float)),
                hbar);
    }
    live = select_level(a, b, t, live, V, keys, hist, scr, sbuf, par, tokm, cum, Rs, bscale,
                        collected, MASK ? pfx : nullptr);
    if (live < 0) return;
    __syncthreads();
    GR_STAMP(5 + 2 * t);
  }
  if (tid == 0 && T > 0) bar_wait(hbar, (uint32_t)((T - 1) & 1));  // no copy outlives the CTA
  // results (beam.py:212-213)
  for (int j = tid; j < live; j += kThreads) {
    int ar = j;
    for (int tau = T - 1; tau >= 0; --tau) {
      a.out_tokens[((size_t)b * a.max_out + j) * T + tau] = tokm[a.moff[tau + 1] + ar];
      ar = par[a.moff[tau + 1] + ar];
    }
    a.out_score[(size_t)b * a.max_out + j] = (double)cum[a.moff[T] + j];
  }
  if (tid == 0) a.out_count[b] = live;
  GR_STAMP(15);
}

// The request-independent head of trunk layer 0 (beam.py:159-163 with the
// reassociated attention): u_p = (LN1(pos_p) Wq) Wk^T for every position p,
// once per batch (one extra frag_prep block); the fused kernel's trunk
// starts at u_p . x_s.
__device__ void trunk_u_block(const TrunkUJob &j) {
  __shared__ float nrm[(GR4AD_MAX_LEVELS + 2) * 32], q[(GR4AD_MAX_LEVELS + 2) * 32];
  const int d = j.d, np = j.n_pos;
  for (int p = threadIdx.x; p < np; p += blockDim.x) {  // layers.py:38-43
    const float *x = j.pos + (size_t)p * d;
    float mean = 0.f;
    for (int i = 0; i < d; ++i) mean += x[i];
    mean /= (float)d;
    float var = 0.f;
    for (int i = 0; i < d; ++i) var += (x[i] - mean) * (x[i] - mean);
    const float inv = 1.0f / sqrtf(var / (float)d + 1e-5f);
    for (int i = 0; i < d; ++i) nrm[p * d + i] = (x[i] - mean) * inv * j.ln1_g[i] + j.ln1_b[i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < np * d; e += blockDim.x) {
    const int p = e / d, c = e - p * d;
    float acc = 0.f;
    for (int i = 0; i < d; ++i) acc = fmaf(nrm[p * d + i], j.wq[(size_t)i * d + c], acc);
    q[e] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < np * d; e += blockDim.x) {
    const int p = e / d, i = e - p * d;
    float acc = 0.f;
    for (int c = 0; c < d; ++c) acc = fmaf(q[p * d + c], j.kv[(size_t)i * j.ldw + c], acc);
    j.u[e] = acc;
  }
}

// fragment-ordered B operands of mma.m16n8k16 (fp16 hi / lo of kFragScale x W):
// per (k16 step kk, n-tile nn, lane) {b0 hi, b1 hi, b0 lo, b1 lo} with
// b0 = W[16kk + 2t .. + 1][8nn + g], b1 = W[16kk + 8 + 2t .. + 1][8nn + g]
__global__ void frag_prep_kernel(const __grid_constant__ FragJobs jobs, uint4 *frag, int *flag) {
  if (blockIdx.y == jobs.n) {  // the extra block row: trunk queries
    if (blockIdx.x == 0 && jobs.tu.u) trunk_u_block(jobs.tu);
    return;
  }
  const FragJob &jb = jobs.job[blockIdx.y];
  const int NT = jb.nout / 8, total = (jb.kin / 16) * NT * 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int lane = i & 31, tile = i >> 5, nn = tile % NT, kk = tile / NT;
    const int k0 = kk * 16 + 2 * (lane & 3), n = nn * 8 + (lane >> 2);
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (n < jb.nreal) {
      x[0] = jb.src[k0 * jb.sk + n * jb.sn];
      x[1] = jb.src[(k0 + 1) * jb.sk + n * jb.sn];
      x[2] = jb.src[(k0 + 8) * jb.sk + n * jb.sn];
      x[3] = jb.src[(k0 + 9) * jb.sk + n * jb.sn];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) range_check(x[q] * kFragScale, flag);
    frag[jb.dst + i] = split_b16(x[0], x[1], x[2], x[3], kFragScale);
  }
}

int frag_prep_launch(const FragJobs &jobs, uint4 *frag, int *range_flag, cudaStream_t st) {
  if (jobs.n <= 0) return GR4AD_OK;
  GR_LAUNCH(KC_SMALL, st, frag_prep_kernel<<<dim3(8, jobs.n + 1), 256, 0, st>>>(jobs, frag, range_flag));
  return GR4AD_OK;
}

int fused_mma_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
  if (a.D != 16) return set_err(GR4AD_ERR_UNSUPPORTED, "warp-MMA fused decode: d=%d", a.D);
  bool masked = false;
  for (int t = 0; t < a.T; ++t) masked |= a.vp_rp[t] != nullptr;
  if (masked) {
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(fused_mma_kernel<16, true>),
                                 (int)smem));
    GR_LAUNCH(KC_FUSED, st, fused_mma_kernel<16, true><<<n_requests, kThreads, smem, st>>>(a));
  } else {
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(fused_mma_kernel<16, false>),
                                 (int)smem));
    GR_LAUNCH(KC_FUSED, st, fused_mma_kernel<16, false><<<n_requests, kThreads, smem, st>>>(a));
  }
  return GR4AD_OK;
}

int fused_small_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
#define GR_FUSED_CASE(DD)                                                                \
  if (a.D == DD) {                                                                       \
    GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(fused_small_kernel<DD>),                                 \
                                 (int)smem)); \
    GR_LAUNCH(KC_FUSED, st, fused_small_kernel<DD><<<n_requests, kThreads, smem, st>>>(a)); \
    return GR4AD_OK;                                                                     \
  }
  GR_FUSED_CASE(16)
  GR_FUSED_CASE(32)
#undef GR_FUSED_CASE
  return set_err(GR4AD_ERR_UNSUPPORTED, "fused decode: d=%d", a.D);
}

}  // namespace gr
