// Exact float64 top-k selection: the public pre-cut / global selection
// (gr4ad_topk_precut_f64; reference beam.py:30-89).
//
// The reference ranks candidates cand = prev[i] + logp[i, j] (numpy float64
// broadcast add) by (-score, beam, token) -- _ordered_topk's lexsort
// (beam.py:30-34); the per-row pre-cut (beam.py:63-83) keeps exactly the
// same set because every global top-k member is inside its own row's top-k.
// Here one CTA owns one problem:
//   1. 64-bit radix select (8 passes of 8 bits) over order-preserving keys of
//      the double scores finds the k-th largest key T and how many of the
//      candidates equal to T are needed;
//   2. one pass appends every candidate above T (unordered) and, in index
//      order (warp ballots + a block scan per 1024-candidate chunk), the
//      first `need` candidates equal to T -- ties resolve to the smallest
//      flat index = (beam, token) order;
//   3. a bitonic sort in shared memory orders the k winners by (key desc,
//      index asc).
// No key is rounded, so the order is the reference's bit for bit.

#include "common.cuh"

namespace gr {

namespace {

constexpr int kSelThreads = 1024;

// larger double -> larger key; -0.0 == +0.0 (numpy compares them equal);
// NaN below everything (lexsort puts NaN last)
__device__ __forceinline__ unsigned long long d2ord(double x) {
  if (x != x) return 0ull;
  if (x == 0.0) x = 0.0;
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double cand(const double *prev, const double *lp, int v, long long i) {
  return prev[i / v] + lp[i];
}

__global__ void __launch_bounds__(kSelThreads)
topk_f64_kernel(const double *__restrict__ prev_all, const double *__restrict__ lp_all, int b,
                int v, int k, int sort_n, int *__restrict__ out_beam, int *__restrict__ out_token,
                double *__restrict__ out_score, int *__restrict__ out_count) {
  extern __shared__ unsigned long long sm64[];
  unsigned long long *skey = sm64;                                   // [sort_n]
  unsigned int *sidx = reinterpret_cast<unsigned int *>(sm64 + sort_n);  // [sort_n]
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_need;
  __shared__ unsigned int s_gt, s_tie_base;
  __shared__ unsigned int warp_tot[kSelThreads / 32];

  const int p = blockIdx.x;
  const double *prev = prev_all + (size_t)p * b;
  const double *lp = lp_all + (size_t)p * b * v;
  const long long n = (long long)b * v;
  const int kk = (int)(k < n ? k : n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // 1. radix select of the kk-th largest key
  unsigned long long prefix = 0, mask = 0;
  long long need = kk;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = tid; i < 256; i += kSelThreads) hist[i] = 0;
    __syncthreads();
    for (long long i = tid; i < n; i += kSelThreads) {
      const unsigned long long key = d2ord(cand(prev, lp, v, i));
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      long long above = 0;
      int bin = 255;
      for (; bin > 0; --bin) {
        if (above + hist[bin] >= need) break;
        above += hist[bin];
      }
      s_prefix = prefix | ((unsigned long long)bin << shift);
      s_need = need - above;
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
    mask |= 0xFFull << shift;
    __syncthreads();
  }
  const unsigned long long T = prefix;  // the kk-th largest key; `need` ties at T are kept

  // 2. collect: keys above T (any order), then the first `need` ties in index order
  if (tid == 0) {
    s_gt = 0;
    s_tie_base = 0;
  }
  __syncthreads();
  for (long long i = tid; i < n; i += kSelThreads) {
    const unsigned long long key = d2ord(cand(prev, lp, v, i));
    if (key > T) {
      const unsigned int at = atomicAdd(&s_gt, 1u);
      skey[at] = key;
      sidx[at] = (unsigned int)i;
    }
  }
  __syncthreads();
  const unsigned int n_gt = s_gt;  // == kk - need
  for (long long c0 = 0; c0 < n; c0 += kSelThreads) {
    if (s_tie_base >= (unsigned long long)need) break;  // uniform: read after a barrier
    const long long i = c0 + tid;
    const bool tie = i < n && d2ord(cand(prev, lp, v, i)) == T;
    const unsigned int bal = __ballot_sync(0xffffffffu, tie);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    unsigned int before = 0, total = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) {
      const unsigned int c = warp_tot[w];
      before += w < warp ? c : 0;
      total += c;
    }
    const unsigned int rank = s_tie_base + before + __popc(bal & ((1u << lane) - 1u));
    if (tie && rank < (unsigned long long)need) {
      skey[n_gt + rank] = T;
      sidx[n_gt + rank] = (unsigned int)i;
    }
    __syncthreads();
    if (tid == 0) s_tie_base += total;
    __syncthreads();
  }

  // 3. bitonic sort of the kk winners: key descending, index ascending
  for (int i = kk + tid; i < sort_n; i += kSelThreads) {
    skey[i] = 0ull;
    sidx[i] = 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int size = 2; size <= sort_n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < sort_n / 2; i += kSelThreads) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;  // this run sorts "first-ranked first"
        const unsigned long long ka = skey[lo], kb = skey[hi];
        const unsigned int ia = sidx[lo], ib = sidx[hi];
        const bool b_first = kb > ka || (kb == ka && ib < ia);
        if (b_first == up) {
          skey[lo] = kb; skey[hi] = ka;
          sidx[lo] = ib; sidx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  for (int j = tid; j < kk; j += kSelThreads) {
    const long long i = sidx[j];
    out_beam[(size_t)p * k + j] = (int)(i / v);
    out_token[(size_t)p * k + j] = (int)(i % v);
    out_score[(size_t)p * k + j] = cand(prev, lp, v, i);
  }
  if (tid == 0) out_count[p] = kk;
}

}  // namespace

}  // namespace gr

using namespace gr;

extern "C" int gr4ad_topk_precut_f64(const double *prev_scores, const double *logprobs,
                                     int n_problems, int b, int v, int k, int *out_beam,
                                     int *out_token, double *out_score, int *out_count,
                                     void *stream) {
  if (n_problems < 0 || b < 1 || v < 1 || k < 1)
    return set_err(GR4AD_ERR_VALUE, "bad selection shape");
  const long long n = (long long)b * v;
  const long long kk = k < n ? k : n;
  if (kk > GR4AD_MAX_BEAM) return set_err(GR4AD_ERR_UNSUPPORTED, "k %d exceeds %d", k, GR4AD_MAX_BEAM);
  if (n >= 0xFFFFFFFFLL) return set_err(GR4AD_ERR_UNSUPPORTED, "too many candidates");
  if (n_problems == 0) return GR4AD_OK;
  int sort_n = 2;
  while (sort_n < kk) sort_n <<= 1;
  const size_t smem = (size_t)sort_n * (sizeof(unsigned long long) + sizeof(unsigned int));
  GR_CUDA(set_smem_attr(reinterpret_cast<const void *>(topk_f64_kernel), (int)smem));
  cudaStream_t st = (cudaStream_t)stream;
  GR_LAUNCH(KC_TOPK, st,
            topk_f64_kernel<<<n_problems, kSelThreads, smem, st>>>(
                prev_scores, logprobs, b, v, k, sort_n, out_beam, out_token, out_score,
                out_count));
  return GR4AD_OK;
}
