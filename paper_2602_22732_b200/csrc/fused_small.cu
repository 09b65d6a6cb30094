// Fused per-request LazyAR beam decode for small models (d in {16, 32}).
//
// One CTA owns one request for the whole decode (beam.py:146-218): context
// projection (decoder.py:134-140), the beam-shared encoder K/V of every
// layer kept in shared memory (beam.py:98-109), the trunk (beam.py:159-163),
// then per level each group of G = d lanes owns one beam row (two rows per
// warp at d = 16) and runs fuse -> head layers -> codebook logits ->
// log-softmax keys with the row state in registers.  The self-KV history
// lives in shared memory and is read through parent pointers (no copies,
// beam.py:205-210), and an exact radix top-k over the level's candidates
// compacts the beams in place.  Weights are read transposed (prepared once
// per call into the workspace) so every row x matrix product uses float4
// loads.  The C1/C2 working set (K/V 40 KB, history 25 KB) fits on chip:
// the whole batch decode is two launches.
#include "fused_small.cuh"

namespace gr {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

template <int G>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
template <int G>
__device__ __forceinline__ float gmax(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// xv[i] = x held by group lane i
template <int G, int N>
__device__ __forceinline__ void bcast(float x, float (&xv)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) xv[i] = __shfl_sync(kFull, x, i, G);
}

// out = sum_i xv[i] * WT[row][i] over N inputs (WT row-major, N % 4 == 0)
template <int N>
__device__ __forceinline__ float dot_row(const float (&xv)[N], const float *__restrict__ wrow) {
  const float4 *w4 = reinterpret_cast<const float4 *>(wrow);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    float4 w = __ldg(w4 + i);
    acc = fmaf(xv[4 * i], w.x, acc);
    acc = fmaf(xv[4 * i + 1], w.y, acc);
    acc = fmaf(xv[4 * i + 2], w.z, acc);
    acc = fmaf(xv[4 * i + 3], w.w, acc);
  }
  return acc;
}

// row-group reduce-scatter: lane gl ends with the group sum of acc[gl]
template <int G>
__device__ __forceinline__ float reduce_scatter(float (&acc)[G]) {
  const int gl = threadIdx.x & (G - 1);
#pragma unroll
  for (int half = G / 2; half >= 1; half >>= 1) {
    const bool up = (gl & half) != 0;
#pragma unroll
    for (int k = 0; k < half; ++k) {
      float send = up ? acc[k] : acc[k + half];
      float keep = up ? acc[k + half] : acc[k];
      acc[k] = keep + __shfl_xor_sync(kFull, send, half);
    }
  }
  return acc[0];
}

template <int G>
__device__ __forceinline__ float layer_norm(float x, const float *g, const float *b) {
  const int gl = threadIdx.x & (G - 1);
  float mean = gsum<G>(x) / (float)G;
  float c = x - mean;
  float var = gsum<G>(c * c) / (float)G;
  float inv = 1.0f / sqrtf(var + 1e-5f);
  return c * inv * __ldg(g + gl) + __ldg(b + gl);
}

// tanh-GELU (autodiff.py:301-306) via 0.5*a*(1+tanh z) == a / (1 + exp(-2z))
__device__ __forceinline__ float gelu_exp(float a) {
  const float c = 0.7978845608028654f;
  float z = (a + 0.044715f * a * a * a) * c;
  return a / (1.0f + expf(-2.0f * z));
}

// cross-attention of one row against the request's shared K/V in shared
// memory (rows of KS floats): group lanes over keys, reduce-scatter back.
template <int G, int MAXM>
__device__ __forceinline__ float cross_attn(float q, const float *Ks, const float *Vs, int S,
                                            int KS) {
  const int gl = threadIdx.x & (G - 1);
  float qv[G];
  bcast<G>(q, qv);
  const float scale = 1.0f / sqrtf((float)G);
  float sc[MAXM];
  float mx = -INFINITY;
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    int s = gl + G * m;
    sc[m] = -INFINITY;
    if (s < S) {
      const float4 *kr = reinterpret_cast<const float4 *>(Ks + s * KS);
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < G / 4; ++i) {
        float4 k4 = kr[i];
        dot = fmaf(qv[4 * i], k4.x, dot);
        dot = fmaf(qv[4 * i + 1], k4.y, dot);
        dot = fmaf(qv[4 * i + 2], k4.z, dot);
        dot = fmaf(qv[4 * i + 3], k4.w, dot);
      }
      sc[m] = dot * scale;
      mx = fmaxf(mx, sc[m]);
    }
  }
  mx = gmax<G>(mx);
  float sum = 0.f;
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    sc[m] = expf(sc[m] - mx);  // exp(-inf) = 0 for s >= S
    sum += sc[m];
  }
  const float inv = 1.0f / gsum<G>(sum);  // softmax (autodiff.py:367-368)
  float acc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) acc[j] = 0.f;
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    int s = gl + G * m;
    if (s < S) {
      float p = sc[m] * inv;
      const float4 *vr = reinterpret_cast<const float4 *>(Vs + s * KS);
#pragma unroll
      for (int i = 0; i < G / 4; ++i) {
        float4 v4 = vr[i];
        acc[4 * i] = fmaf(p, v4.x, acc[4 * i]);
        acc[4 * i + 1] = fmaf(p, v4.y, acc[4 * i + 1]);
        acc[4 * i + 2] = fmaf(p, v4.z, acc[4 * i + 2]);
        acc[4 * i + 3] = fmaf(p, v4.w, acc[4 * i + 3]);
      }
    }
  }
  return reduce_scatter<G>(acc);
}

// one pre-LN block's FFN: W2 gelu(W1 n + b1) + b2, d_ff <= 2G (layers.py:115-118)
template <int G>
__device__ __forceinline__ float ffn(float n, const FusedLayerT &LT, const gr4ad_layer &Lw,
                                     int dff) {
  const int gl = threadIdx.x & (G - 1);
  float nv[G];
  bcast<G>(n, nv);
  float h0 = 0.f, h1 = 0.f;
  if (gl < dff) h0 = gelu_exp(dot_row<G>(nv, LT.w1T + gl * G) + __ldg(Lw.ffn_b1 + gl));
  if (G + gl < dff) h1 = gelu_exp(dot_row<G>(nv, LT.w1T + (G + gl) * G) + __ldg(Lw.ffn_b1 + G + gl));
  float hv[G];
  bcast<G>(h0, hv);
  const float *w2 = LT.w2T + gl * dff;  // row gl of W2^T (d x d_ff)
  float acc = dot_row<G>(hv, w2);
  if (dff > G) {
    bcast<G>(h1, hv);
    acc += dot_row<G>(hv, w2 + G);
  }
  return acc + __ldg(Lw.ffn_b2 + gl);
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

}  // namespace

// transposed copies of every small weight matrix the fused kernel reads
__global__ void fused_prep_kernel(FusedPrep p) {
  const int job = blockIdx.y;
  if (job >= p.n) return;
  const float *src = p.src[job];
  float *dst = p.dst[job];
  const int R = p.rows[job], Cc = p.cols[job];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * Cc; e += gridDim.x * blockDim.x) {
    int r = e / Cc, c = e - r * Cc;
    dst[(size_t)c * R + r] = src[e];  // dst = src^T  (cols x rows)
  }
}

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

template <int G, int MAXM, int VCH>
__global__ void __launch_bounds__(kThreads, 2) fused_small_kernel(FusedArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int D = G;
  constexpr int RPW = 32 / G;  // rows per warp
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gl = lane & (G - 1), sub = lane / G;
  const int T = a.T, L = a.L, K = a.K, dff = a.dff, KS = a.KS;
  const int S = a.ctx_len[b];
  const long long coff = a.ctx_off[b];
  const gr4ad_weights &W = a.w;
  const float scale = 1.0f / sqrtf((float)D);

  float *Xs = sm + a.s_X;
  float *KV = sm + a.s_KV;
  float *TR = sm + a.s_TR;
  float *TQ = sm + a.s_TQ;
  float *HI = sm + a.s_hist;
  int *par = reinterpret_cast<int *>(sm + a.s_par);
  int *tokm = reinterpret_cast<int *>(sm + a.s_tok);
  float *cum = sm + a.s_cum;
  unsigned *hist = reinterpret_cast<unsigned *>(sm + a.s_bins);
  unsigned *scr = reinterpret_cast<unsigned *>(sm + a.s_scr);
  unsigned long long *sbuf = reinterpret_cast<unsigned long long *>(sm + a.s_sort);
  uint32_t *keys = a.keys + (size_t)b * a.keys_per_req;
  const int KVS = a.S_max * KS;
  GR_STAMP(0);

  // ---- context projection X = F W_c + b_c (decoder.py:134-140) -------------
  for (int e = tid; e < S * D; e += kThreads) {
    int s = e / D, j = e - s * D;
    float x;
    if (a.features) {
      const float *f = a.features + (coff + s) * a.F;
      const float *wc = a.ctxT + (size_t)j * a.F;  // row j of W_c^T
      float acc = 0.f;
      for (int i = 0; i < a.F; ++i) acc = fmaf(__ldg(f + i), __ldg(wc + i), acc);
      x = acc + __ldg(W.ctx_b + j);
    } else {
      x = __ldg(a.context + (coff + s) * D + j);
    }
    Xs[s * KS + j] = x;
  }
  __syncthreads();

  // K/V of `layer` into `slot`: K[s][c] = X[s] . WkvT[2*layer*D + c]
  auto build_kv = [&](int layer, int slot) {
    float *Kd = KV + (size_t)slot * 2 * KVS;
    for (int e = tid; e < S * 2 * D; e += kThreads) {
      int s = e / (2 * D), c = e - s * 2 * D;
      const float4 *x4 = reinterpret_cast<const float4 *>(Xs + s * KS);
      const float4 *w4 = reinterpret_cast<const float4 *>(a.kvT + ((size_t)2 * layer * D + c) * D);
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < D / 4; ++i) {
        float4 x = x4[i], w = __ldg(w4 + i);
        acc = fmaf(x.x, w.x, acc);
        acc = fmaf(x.y, w.y, acc);
        acc = fmaf(x.z, w.z, acc);
        acc = fmaf(x.w, w.w, acc);
      }
      Kd[(c < D ? 0 : KVS) + s * KS + (c < D ? c : c - D)] = acc;
    }
  };

  GR_STAMP(1);
  // ---- trunk: K layers over the n_pos position rows (beam.py:159-163) -------
  const int np = a.n_pos;
  if (K > 0) {
    for (int e = tid; e < np * D; e += kThreads) TR[e] = __ldg(W.pos + e);
    for (int i = 0; i < K; ++i) {
      __syncthreads();
      build_kv(i, 0);
      __syncthreads();
      const gr4ad_layer &Lw = W.layer[i];
      const FusedLayerT &LT = a.lt[i];
      for (int p0 = wid * RPW; p0 < np; p0 += kWarps * RPW) {
        int p = p0 + sub;
        bool ok = p < np;
        int pp = ok ? p : np - 1;
        float h = TR[pp * D + gl];
        float n = layer_norm<G>(h, Lw.ln1_g, Lw.ln1_b);
        float nv[G];
        bcast<G>(n, nv);
        float q = dot_row<G>(nv, LT.cqT + gl * D);
        float o = cross_attn<G, MAXM>(q, KV, KV + KVS, S, KS);
        float ov[G];
        bcast<G>(o, ov);
        h += dot_row<G>(ov, LT.coT + gl * D);
        n = layer_norm<G>(h, Lw.ln2_g, Lw.ln2_b);
        bcast<G>(n, nv);
        float qs = dot_row<G>(nv, LT.sqkvT + gl * D);
        float ks = dot_row<G>(nv, LT.sqkvT + (D + gl) * D);
        float vs = dot_row<G>(nv, LT.sqkvT + (2 * D + gl) * D);
        if (ok) {
          TQ[(p * 3 + 0) * D + gl] = qs;
          TQ[(p * 3 + 1) * D + gl] = ks;
          TQ[(p * 3 + 2) * D + gl] = vs;
          TR[p * D + gl] = h;
        }
      }
      __syncthreads();
      for (int p0 = wid * RPW; p0 < np; p0 += kWarps * RPW) {
        int p = p0 + sub;
        bool ok = p < np;
        int pp = ok ? p : np - 1;
        float h = TR[pp * D + gl];
        float q = TQ[(pp * 3) * D + gl];
        // causal self-attention over positions 0..p (layers.py:94-100); the
        // loop bound is uniform across the warp's row groups (shuffles inside)
        const int rmax = min(p0 + RPW, np) - 1;
        float mx = -INFINITY;
        for (int r = 0; r <= rmax; ++r) {
          float sc = gsum<G>(q * TQ[(r * 3 + 1) * D + gl]) * scale;
          if (r <= pp) mx = fmaxf(mx, sc);
        }
        float sum = 0.f;
        for (int r = 0; r <= rmax; ++r) {
          float sc = gsum<G>(q * TQ[(r * 3 + 1) * D + gl]) * scale;
          if (r <= pp) sum += expf(sc - mx);
        }
        float lse = logf(sum) + mx;
        float o = 0.f;
        for (int r = 0; r <= rmax; ++r) {
          float sc = gsum<G>(q * TQ[(r * 3 + 1) * D + gl]) * scale;
          if (r <= pp) o = fmaf(expf(sc - lse), TQ[(r * 3 + 2) * D + gl], o);
        }
        float ov[G];
        bcast<G>(o, ov);
        h += dot_row<G>(ov, LT.soT + gl * D);
        float n = layer_norm<G>(h, Lw.ln3_g, Lw.ln3_b);
        h += ffn<G>(n, LT, Lw, dff);
        __syncwarp();
        if (ok) TR[p * D + gl] = h;
      }
    }
  }
  __syncthreads();
  GR_STAMP(2);
  // head-layer K/V, built once and shared by every beam (beam.py:165-169)
  for (int i = K; i < L; ++i) build_kv(i, i - K);
  if (tid == 0) {
    par[0] = 0;
    tokm[0] = 0;
    cum[0] = 0.f;
  }
  __syncthreads();

  GR_STAMP(3);
  const int last = a.rerank ? T : T - 1;
  int live = 1;
  for (int t = 0; t <= last; ++t) {
    const int mo = a.moff[t];
    const int V = t < T ? a.V[t] : 0;
    for (int i = tid; i < 2048; i += kThreads) hist[i] = 0u;
    __syncthreads();
    int hcur = -1;
    unsigned hcnt = 0;
    for (int r0 = wid * RPW; r0 < live; r0 += kWarps * RPW) {
      const int r = r0 + sub;
      const bool ok = r < live;
      const int rr = ok ? r : live - 1;
      // ---- token input + gated fusion (beam.py:180-191; layers.py:129-133)
      float s = (t == 0) ? __ldg(W.bos + gl)
                         : __ldg(W.emb[t - 1] + (size_t)tokm[mo + rr] * D + gl);
      float h;
      if (K > 0) {
        float sv[G];
        bcast<G>(s, sv);
        float g = dot_row<G>(sv, a.fuseT.wgT + gl * D);
        float u = TR[t * D + gl] * g;
        float uv[G];
        bcast<G>(u, uv);
        const float *wf = a.fuseT.wfT + gl * 2 * D;  // row gl of W_f^T (d x 2d)
        h = dot_row<G>(uv, wf) + dot_row<G>(sv, wf + D);
      } else {
        h = s + __ldg(W.pos + (size_t)t * D + gl);
      }
      // ---- head layers (layers.py:66-119, incremental) ----------------------
      for (int i = K; i < L; ++i) {
        const gr4ad_layer &Lw = W.layer[i];
        const FusedLayerT &LT = a.lt[i];
        const float *Kd = KV + (size_t)(i - K) * 2 * KVS;
        float n = layer_norm<G>(h, Lw.ln1_g, Lw.ln1_b);
        float nv[G];
        bcast<G>(n, nv);
        float q = dot_row<G>(nv, LT.cqT + gl * D);
        float o = cross_attn<G, MAXM>(q, Kd, Kd + KVS, S, KS);
        float ov[G];
        bcast<G>(o, ov);
        h += dot_row<G>(ov, LT.coT + gl * D);
        n = layer_norm<G>(h, Lw.ln2_g, Lw.ln2_b);
        bcast<G>(n, nv);
        float qs = dot_row<G>(nv, LT.sqkvT + gl * D);
        float ks = dot_row<G>(nv, LT.sqkvT + (D + gl) * D);
        float vs = dot_row<G>(nv, LT.sqkvT + (2 * D + gl) * D);
        float *hrow = HI + ((size_t)(i - K) * a.Hrows + a.hoff[t] + rr) * 2 * D;
        // self-attention over the ancestor chain (history by parent pointer):
        // own position first, then ancestors; online softmax (layers.py:101-113)
        float m1 = gsum<G>(qs * ks) * scale;
        float mx = m1, se = 1.f, so = vs;
        int a_row = rr;
        for (int tau = t - 1; tau >= 0; --tau) {
          a_row = par[a.moff[tau + 1] + a_row];
          const float *hr = HI + ((size_t)(i - K) * a.Hrows + a.hoff[tau] + a_row) * 2 * D;
          float sc = gsum<G>(qs * hr[gl]) * scale;
          float vv = hr[D + gl];
          if (sc > mx) {
            float f = expf(mx - sc);
            se = se * f + 1.f;
            so = so * f + vv;
            mx = sc;
          } else {
            float e = expf(sc - mx);
            se += e;
            so = fmaf(e, vv, so);
          }
        }
        so = so / se;
        if (ok) {
          hrow[gl] = ks;
          hrow[D + gl] = vs;
        }
        bcast<G>(so, ov);
        h += dot_row<G>(ov, LT.soT + gl * D);
        n = layer_norm<G>(h, Lw.ln3_g, Lw.ln3_b);
        h += ffn<G>(n, LT, Lw, dff);
      }
      float hv[G];
      bcast<G>(h, hv);
      if (t == T) {  // value re-rank step (beam.py:258-288): rank in double
        float lg = -INFINITY;
        if (gl < a.nb) lg = dot_row<G>(hv, a.hvT + gl * D);
        float mxv = gmax<G>(lg);
        double e = gl < a.nb ? exp((double)lg - (double)mxv) : 0.0;
        double se = e;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) se += __shfl_xor_sync(kFull, se, o);
        double ls = log(se);
        double ev = gl < a.nb ? exp(((double)lg - (double)mxv) - ls) * (double)__ldg(a.value_reps + gl)
                              : 0.0;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) ev += __shfl_xor_sync(kFull, ev, o);
        if (ok && gl == 0) reinterpret_cast<double *>(sbuf)[r] = ev * exp((double)cum[mo + r]);
        continue;
      }
      // ---- codebook logits + log-softmax keys (beam.py:198-200) ---------------
      const float4 *head4 = reinterpret_cast<const float4 *>(W.head[t]);
      const int V4 = V / 4;
      float lg[VCH][4];
      float lm = -INFINITY;
#pragma unroll
      for (int c = 0; c < VCH; ++c) {
        int v4 = gl + G * c;
        lg[c][0] = lg[c][1] = lg[c][2] = lg[c][3] = -INFINITY;
        if (v4 < V4) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            float4 w = __ldg(head4 + (size_t)i * V4 + v4);
            a0 = fmaf(hv[i], w.x, a0);
            a1 = fmaf(hv[i], w.y, a1);
            a2 = fmaf(hv[i], w.z, a2);
            a3 = fmaf(hv[i], w.w, a3);
          }
          lg[c][0] = a0; lg[c][1] = a1; lg[c][2] = a2; lg[c][3] = a3;
          lm = fmaxf(lm, fmaxf(fmaxf(a0, a1), fmaxf(a2, a3)));
        }
      }
      const float mx = gmax<G>(lm);
      float s2 = 0.f;
#pragma unroll
      for (int c = 0; c < VCH; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k) s2 += expf(lg[c][k] - mx);
      const float ls = logf(gsum<G>(s2));
      if (ok) {
        const float cr = cum[mo + r];
        uint4 *kr = reinterpret_cast<uint4 *>(keys + (size_t)r * V);
#pragma unroll
        for (int c = 0; c < VCH; ++c) {
          int v4 = gl + G * c;
          if (v4 < V4) {
            uint4 u;
            u.x = f2ord(cr + ((lg[c][0] - mx) - ls));
            u.y = f2ord(cr + ((lg[c][1] - mx) - ls));
            u.z = f2ord(cr + ((lg[c][2] - mx) - ls));
            u.w = f2ord(cr + ((lg[c][3] - mx) - ls));
            kr[v4] = u;
            hist_add(hist, hcur, hcnt, (int)(u.x >> 21));
            hist_add(hist, hcur, hcnt, (int)(u.y >> 21));
            hist_add(hist, hcur, hcnt, (int)(u.z >> 21));
            hist_add(hist, hcur, hcnt, (int)(u.w >> 21));
          }
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
      return;
    }

    // ---- exact top-k under (-score, row, token) (beam.py:30-89) --------------
    const int n_cand = live * V;
    const int k = min(a.eff[t * a.B + b], n_cand);
    unsigned need = (unsigned)k, above;
    int bin = find_bin(hist, 2048, need, &above, scr);
    unsigned eq_total = hist[bin];
    need -= above;
    uint32_t T32 = (uint32_t)bin << 21;
    uint32_t pmask = 0x7FFu << 21;
    const uint4 *keys4 = reinterpret_cast<const uint4 *>(keys);
    const int n4 = n_cand / 4;  // V % 4 == 0
    for (int pass = 0; pass < 2; ++pass) {
      const int shift = pass == 0 ? 10 : 0;
      const int nb = pass == 0 ? 2048 : 1024;
      __syncthreads();
      for (int i = tid; i < nb; i += kThreads) hist[i] = 0u;
      __syncthreads();
      int cur = -1;
      unsigned cnt = 0;
      for (int i0 = tid; i0 < n4; i0 += 4 * kThreads) {
        uint4 u4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int i = i0 + j * kThreads;
          u4[j] = i < n4 ? keys4[i] : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (i0 + j * kThreads < n4) {
            const uint32_t us[4] = {u4[j].x, u4[j].y, u4[j].z, u4[j].w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if ((us[q] & pmask) == T32) hist_add(hist, cur, cnt, (int)((us[q] >> shift) & (nb - 1)));
          }
        }
      }
      if (cnt) atomicAdd(&hist[cur], cnt);
      __syncthreads();
      bin = find_bin(hist, nb, need, &above, scr);
      eq_total = hist[bin];
      need -= above;
      T32 |= (uint32_t)bin << shift;
      pmask |= (uint32_t)(nb - 1) << shift;
    }
    // collect: every key > T32, and the `need` lowest-index keys == T32
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
    __syncthreads();
    int n2 = 1;
    while (n2 < k) n2 <<= 1;
    for (int i = k + tid; i < n2; i += kThreads) sbuf[i] = 0ull;
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1)
      for (int st = size >> 1; st > 0; st >>= 1) {
        for (int i = tid; i < n2 / 2; i += kThreads) {
          int lo = 2 * i - (i & (st - 1)), hi = lo + st;
          bool desc = (lo & size) == 0;
          unsigned long long x = sbuf[lo], y = sbuf[hi];
          if ((x < y) == desc) {
            sbuf[lo] = y;
            sbuf[hi] = x;
          }
        }
        __syncthreads();
      }
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

int fused_prep_launch(const FusedPrep &p, cudaStream_t st) {
  if (p.n <= 0) return GR4AD_OK;
  dim3 grid(8, p.n);
  GR_LAUNCH(KC_SMALL, st, fused_prep_kernel<<<grid, 256, 0, st>>>(p));
  return GR4AD_OK;
}

int fused_small_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st) {
  if (n_requests <= 0) return GR4AD_OK;
  const int G = a.D;
  const int m = (a.S_max + G - 1) / G;
  const int vch = (a.Vmax / 4 + G - 1) / G;
#define GR_FUSED_CASE(GG, MM, VV)                                                         \
  if (G == GG && m <= MM && vch <= VV) {                                                  \
    GR_CUDA(cudaFuncSetAttribute(fused_small_kernel<GG, MM, VV>,                          \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    GR_LAUNCH(KC_FUSED, st,                                                               \
              fused_small_kernel<GG, MM, VV><<<n_requests, kThreads, smem, st>>>(a));     \
    return GR4AD_OK;                                                                      \
  }
  GR_FUSED_CASE(16, 16, 4)
  GR_FUSED_CASE(16, 32, 4)
  GR_FUSED_CASE(16, 16, 8)
  GR_FUSED_CASE(16, 32, 8)
  GR_FUSED_CASE(32, 8, 4)
  GR_FUSED_CASE(32, 16, 4)
  GR_FUSED_CASE(32, 8, 8)
  GR_FUSED_CASE(32, 16, 8)
#undef GR_FUSED_CASE
  return set_err(GR4AD_ERR_UNSUPPORTED, "fused decode: d=%d S=%d V=%d", a.D, a.S_max, a.Vmax);
}

}  // namespace gr
