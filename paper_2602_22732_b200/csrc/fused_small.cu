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
                                           int S, float *oslot, float (&out)[D / 8]) {
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
    const float4 ka = *reinterpret_cast<const float4 *>(KT + i * SP + lane * 8);
    const float4 kb = *reinterpret_cast<const float4 *>(KT + i * SP + lane * 8 + 4);
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
      const float *vrow = VT + (h * 8 + j) * SP + lane * 8;
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
    for (int sz = (size > 0 ? size : 2); sz <= (size > 0 ? size : 64); sz <<= 1) {
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

__device__ void sort_desc(unsigned long long *buf, int n2) {
  warp_merge_tail(buf, n2, 0, 0);  // sizes 2..64 entirely in registers
  __syncthreads();
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

}  // namespace

#ifdef GR_FUSED_TIMING
#define GR_STAMP(i)                                                             \
  do {                                                                          \
    if (threadIdx.x == 0) {                                                     \
      long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
      a.dbg[blockIdx.x * 16 + (i)] = _t;                                        \
    }                                                                           \
  } while (0)
#else
#define GR_STAMP(i) do {} while (0)
#endif

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

  const int np = a.n_pos;
  // ---- trunk: K layers over the n_pos position rows (beam.py:159-163) -------
  // Warp 0 alone (n_pos <= 9 rows), reassociated so the trunk layers' K/V are
  // never built: scores (q Wk^T) X^T, output (P X) Wv.  Warps 1-7 build the
  // head layers' K/V meanwhile.
  if (K > 0 && wid == 0) {
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
        layer_norm<E>(h, Lw.ln1_g, Lw.ln1_b, n);
        publish<E>(n, slot0);
        proj<E>(slot0, D, Lw.cross_Wq, D, t);
        publish<E>(t, slot1);
        proj_t<E>(slot1, D, Wk, ldw, t);  // u = q Wk^T, u . x_s == q . k_s
        publish<E>(t, slot0);
        cross_attn<D>(slot0, Xs, Xs, S, slot2, t);  // t = P X
        publish<E>(t, slot1);
        proj<E>(slot1, D, Wv, ldw, t);  // (P X) Wv == P V
        publish<E>(t, slot0);
        proj<E>(slot0, D, Lw.cross_Wo, D, t);
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] += t[e];
        layer_norm<E>(h, Lw.ln2_g, Lw.ln2_b, n);
        publish<E>(n, slot0);
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
        publish<E>(so, slot0);
        proj<E>(slot0, D, Lw.self_Wo, D, t);
#pragma unroll
        for (int e = 0; e < E; ++e) h[e] += t[e];
        layer_norm<E>(h, Lw.ln3_g, Lw.ln3_b, n);
        publish<E>(n, slot0);
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
        cross_attn<D>(slot1, Kt, Kt + KVS, S, slot2, tt);
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
      return;
    }

    // ---- exact top-k under (-score, row, token) (beam.py:30-89) --------------
    const int n_cand = live * V;
    const int k = min(a.eff[t * a.B + b], n_cand);
    int n_sort = k;  // entries in sbuf to sort (>= k)
    {
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
#ifdef GR_FUSED_TIMING
      if (tid == 0 && t < 3) {
        a.dbg[blockIdx.x * 16 + 10 + t] = ((long long)cnt_le << 32) | (unsigned)wb;
        a.dbg[blockIdx.x * 16 + 13 + (t == 2)] = (long long)(bscale * 1000);
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
    sort_desc(sbuf, n2);
    // compaction: next-level rows in selection order (beam.py:202-210)
    const int mo1 = a.moff[t + 1];
    for (int j = tid; j < k; j += kThreads) {
      unsigned long long e = sbuf[j];
      unsigned fi = 0xFFFFFFFFu - (unsigned)(e & 0xFFFFFFFFull);
      par[mo1 + j] = (int)(fi / (unsigned)V);
      tokm[mo1 + j] = (int)(fi % (unsigned)V);
      cum[mo1 + j] = ord2f((uint32_t)(e >> 32));
    }
    live = k;
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

int fused_small_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
#define GR_FUSED_CASE(DD)                                                                \
  if (a.D == DD) {                                                                       \
    GR_CUDA(cudaFuncSetAttribute(fused_small_kernel<DD>,                                 \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    GR_LAUNCH(KC_FUSED, st, fused_small_kernel<DD><<<n_requests, kThreads, smem, st>>>(a)); \
    return GR4AD_OK;                                                                     \
  }
  GR_FUSED_CASE(16)
  GR_FUSED_CASE(32)
#undef GR_FUSED_CASE
  return set_err(GR4AD_ERR_UNSUPPORTED, "fused decode: d=%d", a.D);
}

}  // namespace gr
