// C ABI of libgr4ad: batch planning, workspace layout and the per-level
// orchestration of the LazyAR beam decode (beam.py:112-288).
#include <math.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "fused_small.cuh"
#include "gemm.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace gr {

static thread_local char g_err[512] = "";
static thread_local long long g_launches = 0;

void count_launch() { ++g_launches; }

// live per-class kernel timing: CUDA events recorded on the launching stream
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  std::string tag;
};
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfRec> *g_prof = nullptr;
static thread_local char g_tag[192] = "";

// label of the next launch (shapes), kept with its timing record
void prof_tag(const char *fmt, ...) {
  if (!g_prof_on) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_tag, sizeof g_tag, fmt, ap);
  va_end(ap);
}

void prof_begin(int cls, cudaStream_t st) {
  if (!g_prof_on) return;
  ProfRec r{cls, nullptr, nullptr, std::string(g_tag)};
  g_tag[0] = 0;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, st);
  g_prof->push_back(r);
}

void prof_end(int cls, cudaStream_t st) {
  if (!g_prof_on || g_prof->empty()) return;
  cudaEventRecord(g_prof->back().b, st);
}

int set_err(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// ---------------------------------------------------------------------------
// plan: every shape of the batch decode, fixed on the host before launch
// ---------------------------------------------------------------------------
struct Plan {
  int B = 0, T = 0, L = 0, K = 0, n_pos = 0, d = 0, dff = 0, F = 0, nb = 0, stride = 0;
  int V[GR4AD_MAX_LEVELS] = {};
  int Vmax = 0, Vsum = 0;
  long long S_tot = 0;
  int S_max = 0;
  bool rerank = false;
  int n_lv = 0;  // levels with rows: T+1
  std::vector<int> ctx_off, ctx_len, eff, cap, row_off;
  std::vector<int> in_off;  // caller's row offsets (contiguous input)
  long long S_in = 0;       // caller's total context rows
  long long R[GR4AD_MAX_LEVELS + 1] = {};
  long long hist_off[GR4AD_MAX_LEVELS + 2] = {};
  int maxcap[GR4AD_MAX_LEVELS + 1] = {};
  long long H = 0, Rw = 0;
  long long max_cand[GR4AD_MAX_LEVELS] = {};
  int max_out = 0;

  // workspace layout: byte offsets
  size_t o_in_off = 0;
  size_t o_ctx_off, o_ctx_len, o_eff, o_cap, o_row_off, o_live, o_row_req;
  size_t o_trow_off, o_trows, o_trow_req, o_tanc, o_tnpos;
  size_t o_tok, o_anc, o_cum, o_prefix;
  size_t o_X, o_KV, o_Ht, o_QKVt, o_Fin = 0;
  size_t o_Hs, o_N, o_Q, o_A, o_U, o_Fb, o_SC, o_SCs, o_LG, o_rinfo, o_lsep, o_vlog;
  size_t o_hist;  // (L-K) consecutive (H, hist_ld) buffers
  long long hist_ld = 0;  // self-attention history row: [q|k|v] (3d) or factored [q'|n] (2d)
  // factored history with n kept as fp16 hi / lo halves ([q' fp32 | n hi | n lo],
  // the q' GEMM's A operand and the self-attention's keys / values at once)
  bool hist_split = false;
  size_t table_bytes, total;
  // tensor-core layered path
  bool tc = false;
  long long sc_ld = 0, vt_ld = 0;
  size_t o_WT = 0, o_XTs = 0, o_Xs = 0, o_U16 = 0, o_Mf = 0;
  // latent (weight-absorbed) cross-attention: per layer A^T, B (F x d), c (d)
  bool lat_ok = false;
  size_t o_Lat = 0, o_LatTmp = 0;
  // LN1 folded into the latent query (diag(g1) A^T, 1^T A', b1 A per layer)
  // and the features pre-split for the fused latent kernel
  size_t o_LatG = 0, o_FinS = 0;
  long long fs_rows = 0;
  // token-side fuse tables per level t (K > 0): s W_g and s W_f[d:2d] for
  // every possible s (bos at t = 0, emb_{t-1} rows after)
  size_t o_FuseT[GR4AD_MAX_LEVELS + 1] = {};
  int fuse_n[GR4AD_MAX_LEVELS + 1] = {};
  long long wt_floats = 0;
  // fused small-model path
  bool fused = false;
  int f_Hrows = 0, f_sort_cap = 0, f_Hrows_mma = 0;
  int f_hoff[GR4AD_MAX_LEVELS + 2] = {}, f_moff[GR4AD_MAX_LEVELS + 2] = {};
  int f_hoff4[GR4AD_MAX_LEVELS + 2] = {};
  int f_s[12] = {};  // smem offsets (floats): X KV TR TQ hist par tok cum bins scr sort ws
  size_t f_smem = 0;
  long long f_keys_per_req = 0;
  size_t o_keys = 0, o_wT = 0;
  // warp-MMA variant of the fused kernel (d = 16)
  bool f_mma = false;
  int f_s4[18] = {};  // as f_s, plus [12] X^T, [13] tile-group merge scratch, [14] codebook, [15] mbarrier, [16] pass-2 row state
  int f_hst_rows = 0, f_head_floats = 0;
  size_t f_smem4 = 0;
  long long frag_f4 = 0;  // fragment-ordered weights (float4 count)
  size_t o_frag = 0, o_tu = 0;
  bool weights_prepared = false;  // batch->weights_prepared
  // derived weight copies (per snapshot, dims + path only): at the start of
  // the workspace, or in the caller's batch->derived buffer (shared by every
  // decode of the snapshot); offsets o_WT o_Mf o_Lat* o_FuseT o_frag o_tu
  // o_dflag are relative to that region
  char *derived = nullptr;
  size_t derived_total = 0, o_dflag = 0;
  unsigned long long derived_sig = 0;
  size_t o_vprp[GR4AD_MAX_LEVELS] = {};  // masking: CSR row pointers per level
  long long vp_np[GR4AD_MAX_LEVELS] = {};
  size_t o_flag = 0;  // fp16 range flag (set by the operand splits, read by gr4ad_range_status)
};

// Fragment-ordered weight jobs of the warp-MMA fused kernel; with w == NULL
// only the offsets / total are computed (planning).
static long long frag_layout(const Plan &p, const gr4ad_weights *w, FragJobs *jobs,
                             FragIndex *fi) {
  const int d = p.d;
  long long off = 0;
  if (jobs) jobs->n = 0;
  auto add = [&](const float *src, long long sk, long long sn, int kin, int nout,
                 int nreal) -> long long {
    if (jobs) jobs->job[jobs->n++] = FragJob{src, sk, sn, off, kin, nout, nreal};
    const long long r = off;
    off += (long long)(kin / 16) * (nout / 8) * 32;  // 16-byte units
    return r;
  };
  const gr4ad_weights z{};
  const gr4ad_weights &W = w ? *w : z;
  fi->wg = add(W.fuse_Wg, d, 1, d, d, d);
  fi->wf_m = add(W.fuse_Wf, d, 1, d, d, d);
  fi->wf_s = add(W.fuse_Wf ? W.fuse_Wf + (size_t)d * d : nullptr, d, 1, d, d, d);
  fi->value = add(W.head_value, p.nb, 1, d, 8, p.nb);
  for (int i = p.K; i < p.L; ++i) {
    const int li = i - p.K;
    const gr4ad_layer &Lw = W.layer[i];
    auto sh = [&](const float *q, size_t o) { return q ? q + o : nullptr; };
    fi->cq[li] = add(Lw.cross_Wq, d, 1, d, d, d);
    fi->co[li] = add(Lw.cross_Wo, d, 1, d, d, d);
    fi->sq[li] = add(Lw.self_Wqkv, 3LL * d, 1, d, d, d);
    fi->sk[li] = add(sh(Lw.self_Wqkv, d), 3LL * d, 1, d, d, d);
    fi->sv[li] = add(sh(Lw.self_Wqkv, 2 * (size_t)d), 3LL * d, 1, d, d, d);
    fi->so[li] = add(Lw.self_Wo, d, 1, d, d, d);
    fi->w1[li] = add(Lw.ffn_W1, p.dff, 1, d, p.dff, p.dff);
    fi->w2[li] = add(Lw.ffn_W2, d, 1, p.dff, d, d);
  }
  for (int t = 0; t < p.T; ++t) fi->head[t] = add(W.head[t], p.V[t], 1, d, p.V[t], p.V[t]);
  return off;
}

// Shared-memory plan of the warp-MMA fused kernel (run after plan_fused).
static bool plan_fused_mma(Plan &p) {
  const int D = p.d;
  if (D != 16 || p.L - p.K > kMaxHeadLayersMma) return false;
  const int SPn = 256, VS = SPn + 8, HS = 2 * D + 8;
  const int last = p.rerank ? p.T : p.T - 1;
  long long hrows = 0, mrows = 0;
  for (int t = 0; t <= p.T; ++t) {
    mrows += p.maxcap[t];
    p.f_hoff4[t] = (int)hrows;
    if (t < last) hrows += p.maxcap[t];  // the last level's history is never read
  }
  long long o = 0;
  auto take = [&](long long floats) {
    long long r = o;
    o += (floats + 3) / 4 * 4;
    return (int)r;
  };
  const long long xt = (long long)D * VS, kvl = (long long)SPn * D + xt;
  const long long hist_floats = (long long)(p.L - p.K) * std::max(hrows, 1LL) * HS;
  p.f_s4[0] = take(std::max(xt, hist_floats));  // X^T, later the history
  p.f_s4[12] = p.f_s4[0];
  p.f_s4[4] = p.f_s4[0];
  p.f_s4[1] = take((long long)(p.L - p.K) * kvl);  // K [S][D] (swizzled) + V^T [D][S+8]
  p.f_s4[2] = take((long long)p.n_pos * D);
  p.f_s4[3] = take((long long)p.n_pos * 3 * D);
  p.f_s4[5] = take(mrows);
  p.f_s4[6] = take(mrows);
  p.f_s4[7] = take(mrows);
  p.f_s4[8] = take(2048);
  p.f_s4[9] = take(64);
  p.f_s4[10] = take(2LL * p.f_sort_cap);
  p.f_s4[11] = take(4LL * 4 * D);  // warp 0's trunk slots
  p.f_s4[13] = take(8LL * 16 * (D + 2));  // 8 warps x 16 rows x (D + 2)
  int vmax = 8;
  for (int t = 0; t < p.T; ++t) vmax = std::max(vmax, p.V[t]);
  p.f_s4[14] = take((long long)D * vmax);  // one level's codebook fragments
  p.f_head_floats = D * vmax;
  p.f_s4[15] = take(4);                    // two mbarriers (16-B aligned)
  p.f_s4[17] = take(mrows);                // rows' SID prefix keys (masking)
  // two CTAs per SM: 2 x (smem + 1 KB reserved) <= 228 KB
  constexpr size_t kMaxSmem = 113 * 1024;
  if ((size_t)o * sizeof(float) > kMaxSmem) return false;
  // per-row pass-2 state of the proxy-window selection, when it fits
  long long srows = 1;
  for (int t = 0; t < p.T; ++t) srows = std::max(srows, (long long)p.maxcap[t]);
  p.f_hst_rows = 0;
  p.f_s4[16] = 0;
  if ((size_t)(o + srows * (D + 2) + 4) * sizeof(float) <= kMaxSmem) {
    p.f_s4[16] = take(srows * (D + 2));
    p.f_hst_rows = (int)srows;
  }
  const size_t bytes = (size_t)o * sizeof(float);
  p.f_smem4 = bytes;
  p.f_Hrows_mma = (int)std::max(hrows, 1LL);
  FragIndex fi;
  p.frag_f4 = frag_layout(p, nullptr, nullptr, &fi);
  return true;
}


// Shared-memory plan of the fused per-request kernel; false if it does not fit.
static bool plan_fused(Plan &p) {
  const int D = p.d;
  if (!(D == 16 || D == 32) || !(p.dff == D || p.dff == 2 * D) || p.S_max > 256 ||
      p.nb > 8 || p.L > 32)
    return false;
  for (int t = 0; t < p.T; ++t)
    if (p.V[t] % 8 != 0 || p.V[t] > 256) return false;
  int kmax = 1;
  for (int t = 0; t < p.T; ++t) {
    if (p.maxcap[t + 1] > 2048) return false;
    kmax = std::max(kmax, p.maxcap[t + 1]);
  }
  int n2 = 1;
  while (n2 < kmax) n2 <<= 1;
  n2 = std::max(2 * n2, 1024);  // window selection collects up to sort_cap keys
  p.f_sort_cap = n2;
  const int last = p.rerank ? p.T : p.T - 1;
  long long hrows = 0, mrows = 0;
  for (int t = 0; t <= p.T; ++t) {
    p.f_moff[t] = (int)mrows;
    mrows += p.maxcap[t];
    if (t <= last) {
      p.f_hoff[t] = (int)hrows;
      hrows += p.maxcap[t];
    }
  }
  long long o = 0;
  auto take = [&](long long floats) {
    long long r = o;
    o += (floats + 3) / 4 * 4;
    return (int)r;
  };
  // the projected context is dead once every K/V is built, before the first
  // history write: X and the self-KV history share one region
  const long long hist_floats = (long long)(p.L - p.K) * hrows * 2 * D;
  p.f_s[0] = take(std::max((long long)256 * D, hist_floats));
  p.f_s[1] = take((long long)std::max(p.L - p.K, 1) * 2 * D * 256);
  p.f_s[2] = take((long long)p.n_pos * D);
  p.f_s[3] = take((long long)p.n_pos * 3 * D);
  p.f_s[4] = p.f_s[0];
  p.f_s[5] = take(mrows);
  p.f_s[6] = take(mrows);
  p.f_s[7] = take(mrows);
  p.f_s[8] = take(2048);
  p.f_s[9] = take(64);
  p.f_s[10] = take(2LL * n2);
  p.f_s[11] = take(8LL * 4 * 4 * D);  // 8 warps x 4 slots x (D x 4)
  size_t bytes = (size_t)o * sizeof(float);
  if (bytes > 220 * 1024) return false;
  p.f_Hrows = (int)hrows;
  p.f_smem = bytes;
  long long kpr = 1;
  for (int t = 0; t < p.T; ++t) kpr = std::max(kpr, (long long)p.maxcap[t] * p.V[t]);
  p.f_keys_per_req = kpr;
  return true;
}

static int make_plan(const gr4ad_dims *dm, const gr4ad_batch *bt, Plan &p,
                     long long min_work_rows = 0) {
  if (!dm || !bt) return set_err(GR4AD_ERR_VALUE, "null dims/batch");
  if (dm->n_levels < 1 || dm->n_levels > GR4AD_MAX_LEVELS)
    return set_err(GR4AD_ERR_UNSUPPORTED, "n_levels=%d (max %d)", dm->n_levels, GR4AD_MAX_LEVELS);
  if (dm->n_layers < 1 || dm->n_layers > GR4AD_MAX_LAYERS)
    return set_err(GR4AD_ERR_UNSUPPORTED, "n_layers=%d (max %d)", dm->n_layers, GR4AD_MAX_LAYERS);
  if (dm->d < 1 || dm->d_ff < 1 || dm->feat_dim < 1 || dm->n_value_buckets < 1)
    return set_err(GR4AD_ERR_VALUE, "bad model dimensions");
  p.B = bt->n_requests;
  if (p.B < 0) return set_err(GR4AD_ERR_VALUE, "n_requests < 0");
  if (bt->decode_path < 0 || bt->decode_path > 5)
    return set_err(GR4AD_ERR_VALUE, "decode_path %d outside [0, 5]", bt->decode_path);
  p.T = dm->n_levels;
  p.L = dm->n_layers;
  p.K = bt->trunk_depth >= 0 ? bt->trunk_depth : dm->trunk_depth;
  if (!(0 <= p.K && p.K < p.L))
    return set_err(GR4AD_ERR_VALUE, "trunk_depth must satisfy 0 <= K < n_layers");
  p.d = dm->d;
  p.dff = dm->d_ff;
  p.F = dm->feat_dim;
  p.nb = dm->n_value_buckets;
  p.rerank = bt->value_rerank != 0;
  p.weights_prepared = bt->weights_prepared != 0;
  p.n_pos = p.T + (p.rerank ? 1 : 0);
  p.stride = p.T + 1;
  p.n_lv = p.T + 1;
  for (int t = 0; t < p.T; ++t) {
    p.V[t] = dm->vocab[t];
    if (p.V[t] < 1) return set_err(GR4AD_ERR_VALUE, "level_vocab_sizes must be positive");
    p.Vmax = std::max(p.Vmax, p.V[t]);
    p.Vsum += p.V[t];
  }
  const int B = p.B, T = p.T;
  // each request's context rows start at a 32-row boundary in the layered
  // buffers (X, K/V, V^T) so tensor-map tiles never straddle requests
  p.ctx_off.assign(B, 0);
  p.ctx_len.assign(B, 0);
  p.in_off.assign(B, 0);
  for (int b = 0; b < B; ++b) {
    int s = bt->ctx_len[b];
    if (s <= 0) return set_err(GR4AD_ERR_VALUE, "empty context");
    p.in_off[b] = (int)p.S_in;
    p.ctx_off[b] = (int)p.S_tot;
    p.ctx_len[b] = s;
    p.S_in += s;
    p.S_tot += (s + 31) / 32 * 32;
    p.S_max = std::max(p.S_max, s);
  }
  // effective widths (beam.py:134-139) and row capacities per level
  p.eff.assign((size_t)T * B, 0);
  p.cap.assign((size_t)(T + 1) * B, 0);
  p.row_off.assign((size_t)(T + 1) * B, 0);
  for (int b = 0; b < B; ++b) {
    long long reach = 1;
    p.cap[b] = 1;
    for (int t = 0; t < T; ++t) {
      int w = bt->widths[(size_t)b * T + t];
      if (w < 1) return set_err(GR4AD_ERR_VALUE, "beam widths must be positive");
      reach = std::min(reach * (long long)p.V[t], 1LL << 40);
      long long e = std::min((long long)w, reach);
      if (e > GR4AD_MAX_BEAM)
        return set_err(GR4AD_ERR_UNSUPPORTED, "effective width %lld exceeds %d", e, GR4AD_MAX_BEAM);
      p.eff[(size_t)t * B + b] = (int)e;
      long long live = p.cap[(size_t)t * B + b];
      long long cand = live * p.V[t];
      if (cand >= 0xFFFFFFFFLL)
        return set_err(GR4AD_ERR_UNSUPPORTED, "%lld candidates in one request", cand);
      p.max_cand[t] = std::max(p.max_cand[t], cand);
      p.cap[(size_t)(t + 1) * B + b] = (int)std::min(e, cand);
    }
  }
  long long h = 0;
  for (int t = 0; t <= T; ++t) {
    long long r = 0;
    int mc = 0;
    for (int b = 0; b < B; ++b) {
      p.row_off[(size_t)t * B + b] = (int)r;
      r += p.cap[(size_t)t * B + b];
      mc = std::max(mc, p.cap[(size_t)t * B + b]);
    }
    p.R[t] = r;
    p.maxcap[t] = mc;
    p.hist_off[t] = h;
    h += r;
  }
  p.hist_off[T + 1] = h;
  p.H = h;
  p.max_out = p.maxcap[T];
  long long rw = (long long)B * p.n_pos;
  for (int t = 0; t < T; ++t) rw = std::max(rw, p.R[t]);
  if (p.rerank) rw = std::max(rw, p.R[T]);
  p.Rw = std::max(std::max(rw, min_work_rows), 1LL);
  if (p.H >= (1LL << 31) || p.S_tot >= (1LL << 31))
    return set_err(GR4AD_ERR_UNSUPPORTED, "batch too large");
  bool masked = false;
  for (int t = 0; t < T; ++t) masked |= bt->valid_prefix[t] != nullptr;
  // masking runs in the warp-MMA kernel (prefix keys as int32 CSR rows)
  long long n_prefix = 1;
  for (int t = 0; t + 1 < T; ++t) n_prefix *= p.V[t];
  const bool mask_fused = !masked || (bt->decode_path != 4 && n_prefix * p.V[T - 1] < (1LL << 31) &&
                                      n_prefix <= (1LL << 24));
  if (bt->decode_path != 1 && bt->decode_path != 3 && bt->decode_path != 5 && mask_fused && B > 0)
    p.fused = plan_fused(p);
  if (p.fused && bt->decode_path != 4) p.f_mma = plan_fused_mma(p);
  if (p.fused && masked && !p.f_mma) p.fused = false;
  if ((bt->decode_path == 2 || bt->decode_path == 4) && !p.fused)
    return set_err(GR4AD_ERR_UNSUPPORTED, "fused decode path not eligible for this batch");
  if (!p.fused) {
    bool ok = p.d % 8 == 0 && p.dff % 4 == 0 && p.F % 4 == 0;
    for (int t = 0; t < T; ++t) ok &= p.V[t] % 4 == 0;
    const bool forced = bt->decode_path == 3 || bt->decode_path == 5;
    p.tc = ok && (forced || (bt->decode_path == 0 && p.d >= 64));
    p.lat_ok = p.tc && bt->decode_path != 5 && latent_supported(p.d, p.F) && p.dff % 8 == 0;
    if (forced && !ok)
      return set_err(GR4AD_ERR_UNSUPPORTED,
                     "tensor-core path needs d a multiple of 8 and d_ff, F, V multiples of 4");
  }
  p.hist_ld = (p.tc ? 2LL : 3LL) * p.d;
  p.hist_split = p.tc && p.d % 128 == 0 && p.d <= 1024 && p.dff % 8 == 0;
  p.sc_ld = (p.S_max + 7) / 8 * 8;  // (fp16 P rows: 16-B aligned)
  p.vt_ld = (p.S_tot + 7) / 8 * 8;  // fp16 rows: 16-B aligned
  if (p.tc) {
    const long long D = p.d;
    p.wt_floats = 0;
    auto add = [&](long long n) { p.wt_floats += (n + 63) / 64 * 64; };
    add(D * p.F);
    add(D * D);
    add(2 * D * D);
    for (int t = 0; t < T; ++t) add((long long)p.V[t] * D);
    add((long long)p.nb * D);
    for (int i = 0; i < p.L; ++i) {  // qk, vo, self qk, self vo, W1, W2
      add(D * D); add(D * D); add(D * D); add(D * D); add(p.dff * D); add(D * p.dff);
    }
    add(D * D);  // W_f[0:d] (the fuse GEMM on the gathered gate)
    if (p.lat_ok)
      for (int i = 0; i < p.L; ++i) {  // latent A^T, B^T, diag(g1) A^T
        add((long long)p.F * D); add((long long)p.F * D); add((long long)p.F * D);
      }
  }

  const size_t I = sizeof(int), Fl = sizeof(float);
  // ---- derived weight region (gr4ad_derived_layout) ----
  size_t od = 0;
  auto take_d = [&](size_t bytes) {
    size_t r = od;
    od = align_up(od + bytes);
    return r;
  };
  p.o_dflag = take_d(256);  // fp16 split range flag of the weight preparation
  if (p.fused && p.f_mma) {
    p.o_frag = take_d(16 * (size_t)p.frag_f4);
    p.o_tu = take_d(sizeof(float) * (size_t)std::max(p.n_pos, 1) * p.d);
  }
  if (!p.fused && p.tc) {
    const size_t d = p.d, H2 = sizeof(__half);
    p.o_Mf = take_d(Fl * 4 * (size_t)p.L * d * d);  // factored attention weights (fp32)
    if (p.lat_ok) {
      p.o_Lat = take_d(Fl * (size_t)p.L * (2 * p.F + 1) * d);
      p.o_LatTmp = take_d(Fl * (size_t)(p.F + 1) * d);
      p.o_LatG = take_d(Fl * (size_t)p.L * (p.F * d + 2 * p.F));  // diag(g1) A^T, 1^T A', b1 A
    }
    if (p.K > 0)
      for (int t = 0; t < p.n_pos; ++t) {
        p.fuse_n[t] = t == 0 ? 1 : p.V[t - 1];
        p.o_FuseT[t] = take_d(Fl * 2 * (size_t)p.fuse_n[t] * d);
      }
    p.o_WT = take_d(H2 * (size_t)p.wt_floats * 2);  // K-major weights: fp16 hi, then lo
  }
  p.derived_total = od;
  // layout signature: everything the region's layout depends on
  {
    unsigned long long h = 1469598103934665603ULL;
    auto mix = [&](unsigned long long v) { h = (h ^ v) * 1099511628211ULL; };
    mix((unsigned long long)od); mix(p.fused); mix(p.f_mma); mix(p.tc); mix(p.lat_ok);
    mix((unsigned long long)p.K); mix((unsigned long long)p.n_pos); mix((unsigned long long)p.wt_floats);
    p.derived_sig = h;
  }
  p.derived = static_cast<char *>(bt->derived);
  if (p.derived && bt->derived_bytes < od)
    return set_err(GR4AD_ERR_WORKSPACE, "derived weight buffer: %zu bytes < %zu", bt->derived_bytes,
                   od);

  // ---- workspace layout ----
  size_t o = p.derived ? 0 : od;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  p.o_ctx_off = take(I * B);
  p.o_in_off = take(I * B);
  p.o_ctx_len = take(I * B);
  p.o_eff = take(I * (size_t)T * B);
  p.o_cap = take(I * (size_t)(T + 1) * B);
  p.o_row_off = take(I * (size_t)(T + 1) * B);
  p.o_live = take(I * (size_t)(T + 1) * B);
  p.o_row_req = take(I * p.H);
  p.o_trow_off = take(I * B);
  p.o_trows = take(I * B);
  p.o_trow_req = take(I * (size_t)B * p.n_pos);
  p.o_tanc = take(I * (size_t)B * p.n_pos * p.n_pos);
  p.o_tnpos = take(I * (size_t)B * p.n_pos);
  p.table_bytes = o;
  p.o_flag = take(256);
  if (!p.derived) p.o_dflag = p.o_flag;  // one flag when the region is in the workspace
  if (p.fused) {
    p.o_keys = take(sizeof(uint32_t) * (size_t)B * p.f_keys_per_req);
    // valid-SID masking: per level, CSR row pointers over the prefix key
    long long np_t = 1;
    for (int t = 0; t < T; ++t) {
      p.o_vprp[t] = bt->valid_prefix[t] ? take(sizeof(int) * (size_t)(np_t + 1)) : 0;
      p.vp_np[t] = np_t;
      np_t *= p.V[t];
    }
    take(sizeof(long long) * kDbgSlots * (size_t)B);  // per-request phase stamps (timing builds)
    p.total = o;
    return GR4AD_OK;
  }
  p.o_tok = take(I * p.H);
  p.o_anc = take(I * p.H * p.stride);
  p.o_cum = take(Fl * p.H);
  p.o_prefix = take(sizeof(long long) * p.H);
  const size_t d = p.d;
  p.o_X = take(Fl * p.S_tot * d);
  p.o_Fin = take(Fl * p.S_tot * p.F);
  // CUDA-core path: K/V materialised for the head layers only (trunk rows
  // attend through the reassociated (q Wk^T) X^T / (P X) Wv); the
  // tensor-core path attends against X itself (factored attention)
  p.o_KV = take(p.tc ? 256 : Fl * p.S_tot * 2 * (p.L - p.K) * d);
  p.o_Ht = take(Fl * (size_t)B * p.n_pos * d);
  p.o_QKVt = take(Fl * (size_t)B * p.n_pos * p.hist_ld);
  p.o_Hs = take(Fl * p.Rw * d);
  p.o_N = take(Fl * p.Rw * d);
  p.o_Q = take(Fl * p.Rw * d);
  p.o_A = take(Fl * p.Rw * d);
  p.o_U = take(Fl * p.Rw * 2 * d);
  p.o_Fb = take(Fl * p.Rw * p.dff);
  p.o_SC = take(Fl * p.Rw * p.sc_ld);
  p.o_SCs = take(p.tc ? sizeof(__half) * 2 * p.Rw * p.sc_ld : 16);  // P as fp16 hi, lo
  p.o_LG = take(Fl * p.Rw * std::max(p.Vmax, p.nb));
  p.o_rinfo = take(sizeof(float2) * p.Rw);
  p.o_lsep = take(p.tc ? sizeof(float4) * p.Rw * ((p.Vmax + 127) / 128) : 16);
  p.o_vlog = take(Fl * std::max(p.R[T], 1LL) * p.nb);
  p.o_hist = take(Fl * p.H * p.hist_ld * (size_t)(p.L - p.K));
  if (p.tc) {
    const size_t H2 = sizeof(__half);
    p.o_XTs = take(H2 * 2 * (size_t)d * p.vt_ld);  // kKvScale X^T as fp16 hi, then lo
    p.o_Xs = take(H2 * 2 * p.S_tot * d);           // kKvScale X as fp16 hi, then lo
    if (p.lat_ok) {
      // pre-split features (fused latent kernel), one spare chunk of rows
      p.fs_rows = p.S_tot + 256;
      p.o_FinS = take(H2 * 2 * (size_t)p.fs_rows * latent_feat_kst(p.F));
    }
    p.o_U16 = take(H2 * 2 * p.Rw * 2 * d);  // the fuse input [g | s] as fp16 hi, then lo
  }
  p.total = o;
  return GR4AD_OK;
}

template <typename T>
static T *at(void *ws, size_t off) {
  return reinterpret_cast<T *>(static_cast<char *>(ws) + off);
}
// a derived-weight region offset (the caller's shared buffer or the workspace)
template <typename T>
static T *atd(const Plan &p, void *ws, size_t off) {
  return reinterpret_cast<T *>((p.derived ? p.derived : static_cast<char *>(ws)) + off);
}

static int upload_tables(const Plan &p, void *ws, cudaStream_t st) {
  const int B = p.B, T = p.T;
  std::vector<int> host(p.table_bytes / sizeof(int), 0);
  auto put = [&](size_t off, const int *src, size_t n) {
    memcpy(reinterpret_cast<char *>(host.data()) + off, src, n * sizeof(int));
  };
  put(p.o_ctx_off, p.ctx_off.data(), B);
  put(p.o_in_off, p.in_off.data(), B);
  put(p.o_ctx_len, p.ctx_len.data(), B);
  put(p.o_eff, p.eff.data(), (size_t)T * B);
  put(p.o_cap, p.cap.data(), (size_t)(T + 1) * B);
  put(p.o_row_off, p.row_off.data(), (size_t)(T + 1) * B);
  int *live = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_live);
  for (int b = 0; b < B; ++b) live[b] = 1;
  int *row_req = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_row_req);
  for (int t = 0; t <= T; ++t)
    for (int b = 0; b < B; ++b) {
      long long g0 = p.hist_off[t] + p.row_off[(size_t)t * B + b];
      for (int j = 0; j < p.cap[(size_t)t * B + b]; ++j) row_req[g0 + j] = b;
    }
  int *trow_off = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_trow_off);
  int *trows = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_trows);
  int *trow_req = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_trow_req);
  int *tanc = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_tanc);
  int *tnpos = reinterpret_cast<int *>(reinterpret_cast<char *>(host.data()) + p.o_tnpos);
  const int np = p.n_pos;
  for (int b = 0; b < B; ++b) {
    trow_off[b] = b * np;
    trows[b] = np;
    for (int q = 0; q < np; ++q) {
      int r = b * np + q;
      trow_req[r] = b;
      tnpos[r] = q + 1;
      for (int tau = 0; tau < np; ++tau) tanc[(size_t)r * np + tau] = b * np + std::min(tau, q);
    }
  }
  GR_CUDA(cudaMemcpyAsync(ws, host.data(), p.table_bytes, cudaMemcpyHostToDevice, st));
  return GR4AD_OK;
}

__global__ void tile_rows_kernel(const float *src, int n_src, int d, float *dst, long long rows) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * d) return;
  long long r = i / d;
  int j = (int)(i - r * d);
  dst[i] = src[(r % n_src) * d + j];
}

// one pre-LN decoder layer over a row set (layers.py:66-119)
struct RowSet {
  bool few_rows = false;  // few rows per request (trunk, level 0): small GEMM tiles
  int rows;           // rows in the set
  int max_group_rows; // max rows of one group
  int groups = 0;     // attention groups (0: one per request)
  const int *g_ctx_off = nullptr, *g_ctx_len = nullptr;  // per-group context block
  const int *g_row_off, *g_rows, *row_req;
  float *qkv;         // (*, hist_ld) self-attention history rows
  long long hist_row0;
  const int *anc;
  int anc_stride;
  int npos_u;
  const int *npos_row;
};

// Tensor-core path: K-major (out, in) fp16 hi / lo copies of the weights,
// with every attention projection pair folded into one matrix (factored
// attention, see layer_forward_tc): qk = W_q W_k^T and vo = W_v W_o of the
// cross- and the self-attention.  m* are the fp32 products themselves
// (rounded once from double; the CUDA-core fallback of `dense` reads them).
struct LayerT {
  const __half *qk, *vo, *sqk, *svo, *w1, *w2;
  const float *mqk, *mvo, *msqk, *msvo;
  // latent cross-attention (latent.cu): A^T = (W_q W_k^T W_c^T)^T and
  // B = W_c W_v W_o (F x d), c = b_c W_v W_o (d)
  const float *lat_at, *lat_b, *lat_c;
  // their K-major fp16 hi / lo copies: q_lat = n A (B operand A^T, F x d)
  // and h += z B + c (B operand B^T, d x F)
  const __half *lat_q16, *lat_o16;
  // LN1 folded into the query projection (latent.cu latent_cross_ln):
  // kWeightScale diag(g1) A^T as fp16 hi / lo, s = 1^T diag(g1) A, c = b1 A
  const __half *lat_qg16;
  const float *lat_s, *lat_c1;
};
struct WeightsT {
  const __half *ctx, *wg, *wf, *hv;
  const __half *wf_top;  // K-major W_f[0:d]
  // per level t: [s W_g | s W_f[d:2d]] for every token s (fp32, 2 x n_t x d)
  const float *fuse_tab[GR4AD_MAX_LEVELS + 1];
  const __half *head[GR4AD_MAX_LEVELS];
  LayerT layer[GR4AD_MAX_LAYERS];
  bool lat = false;  // this decode attends over the latent (features given)
};

static int prep_weights_t(const Plan &p, const gr4ad_weights *w, void *ws, WeightsT &wt,
                          cudaStream_t st, bool launch = true) {
  __half *base = atd<__half>(p, ws, p.o_WT);
  long long o = 0;
  int rc = GR4AD_OK;
  // dst (cols x rows) = kWeightScale * src (rows x cols)^T as fp16 hi, lo at + wt_floats
  auto tr = [&](const float *src, int rows, int cols) -> const __half * {
    __half *dst = base + o;
    o += ((long long)rows * cols + 63) / 64 * 64;
    if (rc == GR4AD_OK && launch)
      rc = transpose_split16(src, cols, dst, dst + p.wt_floats, rows, rows, cols, kWeightScale,
                             atd<int>(p, ws, p.o_dflag), st);
    return dst;
  };
  // C (d x d) = A . op(B) in double (weight_product), once per snapshot
  auto prod = [&](const float *A, long long lda, const float *B, long long ldb, bool tb,
                  float *C) {
    if (rc == GR4AD_OK && launch) rc = weight_product(A, lda, B, ldb, tb, C, p.d, p.d, p.d, p.d, st);
  };
  const int d = p.d;
  const long long dd = (long long)d * d, ldw = 2LL * p.L * d;
  wt.ctx = tr(w->ctx_W, p.F, d);
  wt.wg = tr(w->fuse_Wg, d, d);
  wt.wf = tr(w->fuse_Wf, 2 * d, d);
  wt.wf_top = tr(w->fuse_Wf, d, d);
  for (int t = 0; t <= GR4AD_MAX_LEVELS; ++t) wt.fuse_tab[t] = nullptr;
  if (p.K > 0)
    for (int t = 0; t < p.n_pos; ++t) {
      // the token side of the fuse (layers.py:129-133) is a function of the
      // token alone: s W_g and s W_f[d:2d] tabulated once per snapshot
      float *tab = atd<float>(p, ws, p.o_FuseT[t]);
      const int n = p.fuse_n[t];
      const float *S = t == 0 ? w->bos : w->emb[t - 1];
      wt.fuse_tab[t] = tab;
      if (rc == GR4AD_OK && launch)
        rc = weight_product(S, d, w->fuse_Wg, d, false, tab, d, n, d, d, st);
      if (rc == GR4AD_OK && launch)
        rc = weight_product(S, d, w->fuse_Wf + (size_t)d * d, d, false, tab + (size_t)n * d, d, n,
                            d, d, st);
    }
  for (int t = 0; t < p.T; ++t) wt.head[t] = tr(w->head[t], d, p.V[t]);
  wt.hv = tr(w->head_value, d, p.nb);
  float *Mf = atd<float>(p, ws, p.o_Mf);
  for (int i = 0; i < p.L; ++i) {
    const gr4ad_layer &Lw = w->layer[i];
    LayerT &lt = wt.layer[i];
    float *m = Mf + 4 * dd * i;
    const float *Wk = w->cross_kv_W + (size_t)2 * i * d, *Wv = Wk + d;
    prod(Lw.cross_Wq, d, Wk, ldw, true, m);                             // W_q W_k^T
    prod(Wv, ldw, Lw.cross_Wo, d, false, m + dd);                       // W_v W_o
    prod(Lw.self_Wqkv, 3LL * d, Lw.self_Wqkv + d, 3LL * d, true, m + 2 * dd);   // self W_q W_k^T
    prod(Lw.self_Wqkv + 2 * d, 3LL * d, Lw.self_Wo, d, false, m + 3 * dd);      // self W_v W_o
    lt.mqk = m;
    lt.mvo = m + dd;
    lt.msqk = m + 2 * dd;
    lt.msvo = m + 3 * dd;
    lt.qk = tr(lt.mqk, d, d);
    lt.vo = tr(lt.mvo, d, d);
    lt.sqk = tr(lt.msqk, d, d);
    lt.svo = tr(lt.msvo, d, d);
    lt.w1 = tr(Lw.ffn_W1, d, p.dff);
    lt.w2 = tr(Lw.ffn_W2, p.dff, d);
    lt.lat_at = lt.lat_b = lt.lat_c = nullptr;
    lt.lat_q16 = lt.lat_o16 = lt.lat_qg16 = nullptr;
    lt.lat_s = lt.lat_c1 = nullptr;
    if (p.lat_ok) {
      // absorbed through the context projection X = F W_c + b_c, each
      // product formed in double from the fp32 weights (weight_product)
      const int F = p.F;
      float *la = atd<float>(p, ws, p.o_Lat) + (size_t)i * (2 * F + 1) * d;
      float *tmp = atd<float>(p, ws, p.o_LatTmp), *tv = tmp + (size_t)F * d;
      lt.lat_at = la;
      lt.lat_b = la + (size_t)F * d;
      lt.lat_c = la + (size_t)2 * F * d;
      if (rc == GR4AD_OK && launch) {
        rc = weight_product(w->ctx_W, d, Wk, ldw, false, tmp, d, F, d, d, st);  // W_c W_k
        if (rc == GR4AD_OK)  // A^T = (W_c W_k) W_q^T
          rc = weight_product(tmp, d, Lw.cross_Wq, d, true, la, d, F, d, d, st);
        if (rc == GR4AD_OK)  // W_c W_v
          rc = weight_product(w->ctx_W, d, Wv, ldw, false, tmp, d, F, d, d, st);
        if (rc == GR4AD_OK)  // B = (W_c W_v) W_o
          rc = weight_product(tmp, d, Lw.cross_Wo, d, false, la + (size_t)F * d, d, F, d, d, st);
        if (rc == GR4AD_OK)  // b_c W_v
          rc = weight_product(w->ctx_b, d, Wv, ldw, false, tv, d, 1, d, d, st);
        if (rc == GR4AD_OK)  // c = (b_c W_v) W_o
          rc = weight_product(tv, d, Lw.cross_Wo, d, false, la + (size_t)2 * F * d, d, 1, d, d, st);
      }
      // K-major fp16 splits: the q_lat GEMM's B operand is A^T itself, the
      // output GEMM's is B^T
      __half *q16 = base + o;
      o += ((long long)F * d + 63) / 64 * 64;
      if (rc == GR4AD_OK && launch)
        rc = split16(la, d, q16, q16 + p.wt_floats, d, F, d, kWeightScale, atd<int>(p, ws, p.o_dflag),
                     st);
      lt.lat_q16 = q16;
      lt.lat_o16 = tr(lt.lat_b, F, d);
      float *ag = atd<float>(p, ws, p.o_LatG) + (size_t)i * (F * d + 2 * F);
      lt.lat_s = ag + (size_t)F * d;
      lt.lat_c1 = lt.lat_s + F;
      if (rc == GR4AD_OK && launch)
        rc = latent_fold(la, Lw.ln1_g, Lw.ln1_b, d, F, ag, ag + (size_t)F * d,
                         ag + (size_t)F * d + F, st);
      __half *qg16 = base + o;
      o += ((long long)F * d + 63) / 64 * 64;
      if (rc == GR4AD_OK && launch)
        rc = split16(ag, d, qg16, qg16 + p.wt_floats, d, F, d, kWeightScale, atd<int>(p, ws, p.o_dflag),
                     st);
      lt.lat_qg16 = qg16;
    }
  }
  return rc;
}

// C = epi(A (M x K) . W (K x N)); W in reference layout (ldb = N), WT its
// K-major copy for the tensor-core path (a_rows = rows covered by A's map)
static int dense(const Plan &p, const GemmArgs &g, const __half *WT, long long a_rows, int epi,
                 cudaStream_t st) {
  if (p.tc && WT && g.K % 8 == 0 && tc_eligible(g.lda, g.K, g.K, g.A, WT)) {
    TcArgs t{};
    static_cast<GemmArgs &>(t) = g;
    t.b_hi = WT;  // weights arrive pre-split and scaled (prep_weights_t)
    t.b_lo = WT + p.wt_floats;
    t.ldb = g.K;
    t.alpha = g.alpha / kWeightScale;
    return gemm_tc(t, a_rows, g.K, g.N, g.K, epi, st);
  }
  return gemm(g, false, epi, st);
}

// C = epi(A . W) with A already split into fp16 hi / lo (written so by the
// producing LayerNorm / epilogue / self-attention): no on-chip conversion
static int dense_split(const Plan &p, const GemmArgs &g, const __half *WT, const __half *a_hi,
                       const __half *a_lo, long long a_rows, int epi, cudaStream_t st,
                       __half *c_hi = nullptr, __half *c_lo = nullptr, bool few_rows = false) {
  TcArgs t{};
  static_cast<GemmArgs &>(t) = g;
  t.few_rows = few_rows ? 1 : 0;
  t.b_hi = WT;
  t.b_lo = WT + p.wt_floats;
  t.ldb = g.K;
  t.a_hi = a_hi;
  t.a_lo = a_lo;
  t.alpha = g.alpha / kWeightScale;
  t.c_hi = c_hi;
  t.c_lo = c_lo;
  return gemm_tc(t, a_rows, g.K, g.N, g.K, epi, st);
}

// CUDA-core layered path: the reference's layer as written, with the trunk
// layers' K / V reassociated -- q (X W_k)^T = (q W_k^T) X^T and P (X W_v) =
// (P X) W_v -- so only the head layers' K / V are materialised (KV)
static int layer_forward(const Plan &p, const gr4ad_weights *w, int i, float *Hs,
                         const RowSet &rs, void *ws, const float *KV, cudaStream_t st) {
  const int d = p.d, R = rs.rows;
  const gr4ad_layer &Lw = w->layer[i];
  float *N = at<float>(ws, p.o_N), *Q = at<float>(ws, p.o_Q), *A = at<float>(ws, p.o_A);
  float *SC = at<float>(ws, p.o_SC), *Fb = at<float>(ws, p.o_Fb);
  const int *ctx_off = rs.g_ctx_off ? rs.g_ctx_off : at<int>(ws, p.o_ctx_off);
  const int *ctx_len = rs.g_ctx_len ? rs.g_ctx_len : at<int>(ws, p.o_ctx_len);
  const int n_groups = rs.groups > 0 ? rs.groups : p.B;
  const long long ldkv = 2LL * (p.L - p.K) * d, ldw = 2LL * p.L * d;
  const bool trunk = i < p.K;
  const float *X = at<float>(ws, p.o_X);
  // cross-attention into the beam-shared context KV (layers.py:82-90)
  GR_TRY(ln_rows(Hs, d, N, d, Lw.ln1_g, Lw.ln1_b, R, d, st));
  GR_TRY(gemm(plain_gemm(N, d, Lw.cross_Wq, d, Q, d, R, d, d), false, EPI_STORE, st));
  const float *qsrc = Q;
  if (trunk) {  // B = W_k as (N x K): N = Q W_k^T
    GR_TRY(gemm(plain_gemm(Q, d, w->cross_kv_W + (size_t)(2 * i) * d, ldw, N, d, R, d, d), true,
                EPI_STORE, st));
    qsrc = N;
  }
  GemmArgs qk{};
  qk.A = qsrc; qk.lda = d;
  qk.B = trunk ? X : KV + (size_t)(2 * (i - p.K)) * d;
  qk.ldb = trunk ? d : ldkv;
  qk.C = SC; qk.ldc = p.sc_ld;
  qk.M = rs.max_group_rows; qk.N = p.S_max; qk.K = d;
  qk.alpha = 1.0f / sqrtf((float)d);
  qk.groups = n_groups; qk.mode = GM_QK;
  qk.g_row_off = rs.g_row_off; qk.g_rows = rs.g_rows;
  qk.g_ctx_off = ctx_off; qk.g_ctx_len = ctx_len;
  GR_TRY(gemm(qk, true, EPI_STORE, st));
  GR_TRY(softmax_rows(SC, p.sc_ld, R, rs.row_req, ctx_len, st));
  GemmArgs pv = qk;
  pv.A = SC; pv.lda = p.sc_ld;
  pv.B = trunk ? X : KV + (size_t)(2 * (i - p.K) + 1) * d;
  pv.C = A; pv.ldc = d;
  pv.M = rs.max_group_rows; pv.N = d; pv.K = p.S_max;
  pv.alpha = 1.f; pv.mode = GM_PV;
  GR_TRY(gemm(pv, false, EPI_STORE, st));
  const float *attn = A;
  if (trunk) {  // (P X) W_v
    GR_TRY(gemm(plain_gemm(A, d, w->cross_kv_W + (size_t)(2 * i + 1) * d, ldw, Q, d, R, d, d),
                false, EPI_STORE, st));
    attn = Q;
  }
  GemmArgs o = plain_gemm(attn, d, Lw.cross_Wo, d, Hs, d, R, d, d);
  o.R = Hs; o.ldr = d;
  GR_TRY(gemm(o, false, EPI_RESID, st));
  // self-attention over decoded positions (layers.py:92-113)
  GR_TRY(ln_rows(Hs, d, N, d, Lw.ln2_g, Lw.ln2_b, R, d, st));
  float *qkv_rows = rs.qkv + rs.hist_row0 * p.hist_ld;
  GR_TRY(gemm(plain_gemm(N, d, Lw.self_Wqkv, 3 * d, qkv_rows, p.hist_ld, R, 3 * d, d), false,
              EPI_STORE, st));
  GR_TRY(self_attn(rs.qkv, p.hist_ld, d, rs.anc, rs.anc_stride, (int)rs.hist_row0, R, rs.npos_u,
                   rs.npos_row, A, d, st));
  GemmArgs so = plain_gemm(A, d, Lw.self_Wo, d, Hs, d, R, d, d);
  so.R = Hs; so.ldr = d;
  GR_TRY(gemm(so, false, EPI_RESID, st));
  // position-wise FFN (layers.py:115-118)
  GR_TRY(ln_rows(Hs, d, N, d, Lw.ln3_g, Lw.ln3_b, R, d, st));
  GemmArgs f1 = plain_gemm(N, d, Lw.ffn_W1, p.dff, Fb, p.dff, R, p.dff, d);
  f1.bias = Lw.ffn_b1;
  GR_TRY(gemm(f1, false, EPI_BIAS_GELU, st));
  GemmArgs f2 = plain_gemm(Fb, p.dff, Lw.ffn_W2, d, Hs, d, R, d, p.dff);
  f2.bias = Lw.ffn_b2; f2.R = Hs; f2.ldr = d;
  return gemm(f2, false, EPI_BIAS_RESID, st);
}

// A/B aid: GR4AD_LAT_FUSED=0 runs the latent block as LN1 / q_lat GEMM /
// latent_attn / output GEMM / LN2
static bool lat_fused() {
  static const bool on = [] {
    const char *e = getenv("GR4AD_LAT_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Tensor-core path, factored attention.  The reference attends with
// q = n W_q, K = X W_k, V = X W_v (layers.py:46-51, 82-90; beam.py:98-109,
// 221-232) and the self-attention likewise on the LayerNorm'd rows n
// (layers.py:101-113).  Single head, no projection biases, so
//   q K^T = (n W_q W_k^T) X^T        P V W_o = (P X)(W_v W_o)
// exactly: with W_q W_k^T and W_v W_o formed once per snapshot
// (prep_weights_t), every layer attends straight against the request's
// context X -- one fp16-split copy of X and of X^T, shared by all beams AND
// all layers -- and the per-request encoder K / V GEMM (4 (L-K) S d^2 flop)
// disappears, as do the self-attention's K / V projections (the history
// keeps n itself).  Per beam row the dense products drop from 10 d^2 to
// 8 d^2 MACs per layer.
//
// split_out: also leave the layer's output rows as fp16 hi / lo in the N
// buffer (the codebook GEMM's pre-split A); returns whether it did
static int layer_forward_tc(const Plan &p, const gr4ad_weights *w, const WeightsT &wt, int i,
                            float *Hs, const RowSet &rs, void *ws, cudaStream_t st,
                            bool *split_out = nullptr) {
  const int d = p.d, R = rs.rows;
  const gr4ad_layer &Lw = w->layer[i];
  const LayerT &LT = wt.layer[i];
  const bool few = rs.few_rows;  // few-row set: small GEMM tiles
  float *N = at<float>(ws, p.o_N), *Q = at<float>(ws, p.o_Q), *A = at<float>(ws, p.o_A);
  float *SC = at<float>(ws, p.o_SC), *Fb = at<float>(ws, p.o_Fb);
  const int *ctx_off = rs.g_ctx_off ? rs.g_ctx_off : at<int>(ws, p.o_ctx_off);
  const int *ctx_len = rs.g_ctx_len ? rs.g_ctx_len : at<int>(ws, p.o_ctx_len);
  const int n_groups = rs.groups > 0 ? rs.groups : p.B;
  // every activation operand produced already split into fp16 hi / lo
  // (LayerNorm, epilogues, softmax, self-attention): the GEMMs only move and
  // multiply
  const bool spl = d % 128 == 0 && d <= 1024 && p.dff % 8 == 0;
  __half *Nh = reinterpret_cast<__half *>(N), *Nl = Nh + (size_t)p.Rw * d;
  __half *Ah = reinterpret_cast<__half *>(A), *Al = Ah + (size_t)p.Rw * d;
  __half *Fh = reinterpret_cast<__half *>(Fb), *Fl = Fh + (size_t)p.Rw * p.dff;
  __half *Qh = reinterpret_cast<__half *>(Q), *Ql = Qh + (size_t)p.Rw * d;
  __half *Ph = at<__half>(ws, p.o_SCs), *Pl = Ph + (size_t)p.Rw * p.sc_ld;
  // the request's context, kKvScale * X as fp16 hi / lo: X (S_tot x d) is
  // the K-side operand, X^T (d x vt_ld) the V-side one
  const __half *xs_hi = at<__half>(ws, p.o_Xs), *xs_lo = xs_hi + (size_t)p.S_tot * d;
  const __half *xt_hi = at<__half>(ws, p.o_XTs), *xt_lo = xt_hi + (size_t)d * p.vt_ld;

  float *hq = rs.qkv + rs.hist_row0 * p.hist_ld, *hn = hq + d;  // self history [q' | n]
  // split history: n as fp16 hi / lo halves after q' (row pitch 2 hist_ld halves)
  const bool hs2 = p.hist_split && spl;
  __half *nh_hi = reinterpret_cast<__half *>(hq) + 2 * d, *nh_lo = nh_hi + d;
  const long long ld_nh = 2 * p.hist_ld;
  // LN2's split output (the q' GEMM's A operand) and its fp32 copy
  __half *n2h = hs2 ? nh_hi : Nh, *n2l = hs2 ? nh_lo : Nl;
  const long long ld_n2 = hs2 ? ld_nh : d;
  float *n2f = hs2 ? nullptr : hn;
  if (wt.lat) {
    // ---- cross-attention over the request's latent (latent.cu) ----------
    // q_lat = LN1(h) A;  z = softmax(q_lat F^T / sqrt d) F;  h += z B + c;
    // then LN2 of h (split for the next GEMM, fp32 into the self history)
    const float *Fin = at<float>(ws, p.o_Fin);
    const int F = p.F;
    if (lat_fused()) {
      // LN1 + q_lat inside the attention kernel, z B + c + residual + LN2 in
      // one row-tile kernel: LN1's output and q_lat never reach HBM
      const __half *fs = at<__half>(ws, p.o_FinS);
      GR_TRY(latent_cross_ln(Hs, d, LT.lat_qg16, LT.lat_qg16 + p.wt_floats, LT.lat_s, LT.lat_c1,
                             fs, fs + (size_t)p.fs_rows * latent_feat_kst(F), F, rs.g_row_off,
                             rs.g_rows, ctx_off, ctx_len, n_groups, rs.max_group_rows,
                             1.0f / sqrtf((float)d), A, at<int>(ws, p.o_flag), st));
      GR_TRY(latent_out_ln(A, F, LT.lat_o16, LT.lat_o16 + p.wt_floats, 1.0f / kWeightScale,
                           LT.lat_c, Hs, d, Lw.ln2_g, Lw.ln2_b, n2h, n2l, ld_n2, n2f, p.hist_ld,
                           R, at<int>(ws, p.o_flag), st));
    } else {
    GR_TRY(ln_rows_split(Hs, d, Nh, Nl, d, Lw.ln1_g, Lw.ln1_b, R, d, st));
    GR_TRY(dense_split(p, plain_gemm(N, d, LT.lat_at, d, Q, F, R, F, d), LT.lat_q16, Nh, Nl, R,
                       EPI_STORE, st));
    GR_TRY(latent_attn(Q, Fin, F, rs.g_row_off, rs.g_rows, ctx_off, ctx_len, n_groups,
                       rs.max_group_rows, 1.0f / sqrtf((float)d), A, at<int>(ws, p.o_flag), st));
    GemmArgs go = plain_gemm(A, F, LT.lat_b, d, Hs, d, R, d, F);  // h += z B + c
    go.bias = LT.lat_c;
    go.R = Hs;
    go.ldr = d;
    GR_TRY(dense(p, go, LT.lat_o16, R, EPI_BIAS_RESID, st));
    GR_TRY(ln_rows_split(Hs, d, n2h, n2l, ld_n2, Lw.ln2_g, Lw.ln2_b, R, d, st, n2f, p.hist_ld));
    }
  } else {
  // ---- cross-attention into the beam-shared context (layers.py:82-90) ----
  if (spl)
    GR_TRY(ln_rows_split(Hs, d, Nh, Nl, d, Lw.ln1_g, Lw.ln1_b, R, d, st));
  else
    GR_TRY(ln_rows(Hs, d, N, d, Lw.ln1_g, Lw.ln1_b, R, d, st));
  // few beam rows per request: swap A / B so tiles are not padded to 128 rows
  const bool swap = rs.max_group_rows <= 64;
  const bool spl_att = spl && !swap;
  const GemmArgs gq = plain_gemm(N, d, LT.mqk, d, Q, d, R, d, d);  // q' = n (W_q W_k^T)
  if (spl)
    GR_TRY(dense_split(p, gq, LT.qk, Nh, Nl, R, spl_att ? EPI_STORE_SPLIT : EPI_STORE, st, Qh, Ql, few));
  else
    GR_TRY(dense(p, gq, LT.qk, R, EPI_STORE, st));
  GemmArgs qk{};
  qk.A = Q; qk.lda = d;
  qk.C = SC; qk.ldc = p.sc_ld;
  qk.M = rs.max_group_rows; qk.N = p.S_max; qk.K = d;
  qk.alpha = 1.0f / sqrtf((float)d) / kKvScale;
  qk.groups = n_groups; qk.mode = GM_QK;
  qk.g_row_off = rs.g_row_off; qk.g_rows = rs.g_rows;
  qk.g_ctx_off = ctx_off; qk.g_ctx_len = ctx_len;
  if (swap) {  // tile M = keys (S_max), N = beam rows; q split on chip
    TcArgs t{};
    static_cast<GemmArgs &>(t) = qk;
    t.mode = GM_QK_T;
    t.M = qk.N;
    t.N = qk.M;
    t.B = Q;
    t.ldb = d;
    t.a_hi = xs_hi;
    t.a_lo = xs_lo;
    t.lda = d;
    GR_TRY(gemm_tc_swapped(t, p.S_tot, d, R, d, st));
  } else {
    TcArgs t{};
    static_cast<GemmArgs &>(t) = qk;
    t.b_hi = xs_hi;
    t.b_lo = xs_lo;
    t.ldb = d;
    if (spl_att) {  // q' arrives split from its GEMM's epilogue
      t.a_hi = Qh;
      t.a_lo = Ql;
    }
    GR_TRY(gemm_tc(t, R, d, p.S_tot, d, EPI_STORE, st));
  }
  if (spl_att)
    GR_TRY(softmax_rows_split(SC, p.sc_ld, Ph, Pl, R, rs.row_req, ctx_len, st));
  else
    GR_TRY(softmax_rows(SC, p.sc_ld, R, rs.row_req, ctx_len, st));
  GemmArgs pv = qk;  // u = P X
  pv.A = SC; pv.lda = p.sc_ld;
  pv.C = A; pv.ldc = d;
  pv.M = rs.max_group_rows; pv.N = d; pv.K = p.S_max;
  pv.alpha = 1.f / kKvScale; pv.mode = GM_PV;
  if (swap) {  // tile M = output dims, N = beam rows; P split on chip
    TcArgs t{};
    static_cast<GemmArgs &>(t) = pv;
    t.mode = GM_PV_T;
    t.N = pv.M;
    t.M = d;
    t.B = SC;
    t.ldb = p.sc_ld;
    t.a_hi = xt_hi;
    t.a_lo = xt_lo;
    t.lda = p.vt_ld;
    if (spl) {
      t.c_hi = Ah;
      t.c_lo = Al;
    }
    GR_TRY(gemm_tc_swapped(t, d, p.vt_ld, R, p.sc_ld, st, spl ? EPI_STORE_T_SPLIT : EPI_STORE_T));
  } else {
    TcArgs t{};
    static_cast<GemmArgs &>(t) = pv;
    t.b_hi = xt_hi;
    t.b_lo = xt_lo;
    t.ldb = p.vt_ld;
    if (spl) {
      t.c_hi = Ah;
      t.c_lo = Al;
    }
    if (spl_att) {  // P arrives split from the softmax
      t.a_hi = Ph;
      t.a_lo = Pl;
    }
    GR_TRY(gemm_tc(t, R, p.sc_ld, d, p.vt_ld, spl ? EPI_STORE_SPLIT : EPI_STORE, st));
  }
  GemmArgs o = plain_gemm(A, d, LT.mvo, d, Hs, d, R, d, d);  // h += u (W_v W_o)
  o.R = Hs; o.ldr = d;
  if (spl)
    GR_TRY(dense_split(p, o, LT.vo, Ah, Al, R, EPI_RESID, st, nullptr, nullptr, few));
  else
    GR_TRY(dense(p, o, LT.vo, R, EPI_RESID, st));

  // ---- self-attention over decoded positions (layers.py:92-113) ----------
  // history row: [q' = n (W_q W_k^T) | n]; keys and values are n itself
  if (spl)
    GR_TRY(ln_rows_split(Hs, d, n2h, n2l, ld_n2, Lw.ln2_g, Lw.ln2_b, R, d, st, n2f, p.hist_ld));
  else
    GR_TRY(ln_rows(Hs, d, hn, p.hist_ld, Lw.ln2_g, Lw.ln2_b, R, d, st));
  }  // (context-operand cross-attention)
  GemmArgs sq = spl ? plain_gemm(N, d, LT.msqk, d, hq, p.hist_ld, R, d, d)
                    : plain_gemm(hn, p.hist_ld, LT.msqk, d, hq, p.hist_ld, R, d, d);
  if (spl) {
    sq.lda = ld_n2;  // (in halves: the A operand arrives pre-split)
    GR_TRY(dense_split(p, sq, LT.sqk, n2h, n2l, R, EPI_STORE, st, nullptr, nullptr, few));
  } else {
    GR_TRY(dense(p, sq, LT.sqk, R, EPI_STORE, st));
  }
  GR_TRY(self_attn(rs.qkv, p.hist_ld, d, rs.anc, rs.anc_stride, (int)rs.hist_row0, R, rs.npos_u,
                   rs.npos_row, A, d, st, spl ? Ah : nullptr, spl ? Al : nullptr, d, hs2));
  GemmArgs so = plain_gemm(A, d, LT.msvo, d, Hs, d, R, d, d);  // h += (P n) (W_v W_o)
  so.R = Hs; so.ldr = d;
  if (spl)
    GR_TRY(dense_split(p, so, LT.svo, Ah, Al, R, EPI_RESID, st, nullptr, nullptr, few));
  else
    GR_TRY(dense(p, so, LT.svo, R, EPI_RESID, st));

  // ---- position-wise FFN (layers.py:115-118) ------------------------------
  if (spl)
    GR_TRY(ln_rows_split(Hs, d, Nh, Nl, d, Lw.ln3_g, Lw.ln3_b, R, d, st));
  else
    GR_TRY(ln_rows(Hs, d, N, d, Lw.ln3_g, Lw.ln3_b, R, d, st));
  GemmArgs f1 = plain_gemm(N, d, Lw.ffn_W1, p.dff, Fb, p.dff, R, p.dff, d);
  f1.bias = Lw.ffn_b1;
  if (spl)
    GR_TRY(dense_split(p, f1, LT.w1, Nh, Nl, R, EPI_BIAS_GELU_SPLIT, st, Fh, Fl, few));
  else
    GR_TRY(dense(p, f1, LT.w1, R, EPI_BIAS_GELU, st));
  GemmArgs f2 = plain_gemm(Fb, p.dff, Lw.ffn_W2, d, Hs, d, R, d, p.dff);
  f2.bias = Lw.ffn_b2; f2.R = Hs; f2.ldr = d;
  const bool dual = spl && split_out;
  if (spl)
    GR_TRY(dense_split(p, f2, LT.w2, Fh, Fl, R, dual ? EPI_BIAS_RESID_DUAL : EPI_BIAS_RESID, st,
                       dual ? Nh : nullptr, dual ? Nl : nullptr, few));
  else
    GR_TRY(dense(p, f2, LT.w2, R, EPI_BIAS_RESID, st));
  if (split_out) *split_out = dual;
  return GR4AD_OK;
}

// context projection, the shared context operands and the trunk
// (beam.py:159-169): the request-level work every decode of the batch shares
static int encode_and_trunk(const Plan &p, const gr4ad_weights *w, const float *features,
                            const float *context, void *ws, WeightsT &wt_store,
                            const WeightsT *&wt, cudaStream_t st) {
  const int B = p.B, d = p.d, K = p.K;
  float *KV = at<float>(ws, p.o_KV), *Ht = at<float>(ws, p.o_Ht);
  int *flag = at<int>(ws, p.o_flag);
  if (!features && !context) return set_err(GR4AD_ERR_VALUE, "either features or context is required");
  if (p.tc) {
    GR_TRY(prep_weights_t(p, w, ws, wt_store, st, !p.weights_prepared));
    wt_store.lat = p.lat_ok && features != nullptr;
    wt = &wt_store;
  }
  if (p.tc && wt_store.lat) {
    // latent path: the shared context is the request's raw features (32-row
    // aligned blocks); X = F W_c + b_c is absorbed into the weights and
    // never formed
    GR_TRY(pad_rows(features, at<int>(ws, p.o_in_off), at<int>(ws, p.o_ctx_off),
                    at<int>(ws, p.o_ctx_len), B, p.F, at<float>(ws, p.o_Fin), st));
    if (lat_fused()) {
      __half *fs = at<__half>(ws, p.o_FinS);
      GR_TRY(latent_feat_split(at<float>(ws, p.o_Fin), p.S_tot, p.fs_rows, p.F, fs,
                               fs + (size_t)p.fs_rows * latent_feat_kst(p.F), flag, st));
    }
  } else {
  // context projection (decoder.py:134-140) on 32-row-aligned request blocks
  const int *in_off = at<int>(ws, p.o_in_off), *ctx_off_d = at<int>(ws, p.o_ctx_off);
  const int *ctx_len_d = at<int>(ws, p.o_ctx_len);
  float *X = at<float>(ws, p.o_X);
  __half *xs_hi = p.tc ? at<__half>(ws, p.o_Xs) : nullptr;
  __half *xs_lo = p.tc ? xs_hi + (size_t)p.S_tot * d : nullptr;
  bool x_split = false;  // kKvScale * X also as fp16 hi / lo at o_Xs
  if (!features) {
    GR_TRY(pad_rows(context, in_off, ctx_off_d, ctx_len_d, B, d, X, st));
  } else {
    float *Fin = at<float>(ws, p.o_Fin);
    GR_TRY(pad_rows(features, in_off, ctx_off_d, ctx_len_d, B, p.F, Fin, st));
    GemmArgs g = plain_gemm(Fin, p.F, w->ctx_W, d, X, d, (int)p.S_tot, d, p.F);
    g.bias = w->ctx_b;
    if (p.tc && p.F % 8 == 0 && tc_eligible(g.lda, g.K, g.K, g.A, wt->ctx)) {
      TcArgs t{};
      static_cast<GemmArgs &>(t) = g;
      t.b_hi = wt->ctx;
      t.b_lo = wt->ctx + p.wt_floats;
      t.ldb = g.K;
      t.alpha = g.alpha / kWeightScale;
      t.c_hi = xs_hi;
      t.c_lo = xs_lo;
      t.c_scale = kKvScale;
      t.range_flag = flag;
      GR_TRY(gemm_tc(t, p.S_tot, g.K, g.N, g.K, EPI_BIAS_DUAL, st));
      x_split = true;
    } else {
      GR_TRY(dense(p, g, wt ? wt->ctx : nullptr, p.S_tot, EPI_BIAS, st));
    }
  }
  if (p.tc) {
    // the shared context operands of every layer's attention (factored
    // attention: X stands in for all layers' K and V, beam.py:98-109)
    if (!x_split) GR_TRY(split16(X, d, xs_hi, xs_lo, d, (int)p.S_tot, d, kKvScale, flag, st));
    __half *xt_hi = at<__half>(ws, p.o_XTs);
    GR_TRY(transpose_split16(X, d, xt_hi, xt_hi + (size_t)d * p.vt_ld, p.vt_ld, (int)p.S_tot, d,
                             kKvScale, flag, st));
  } else {
    // encoder K/V of the head layers, once per request and shared by every
    // beam (beam.py:98-109)
    const int nh = p.L - K;
    GR_TRY(gemm(plain_gemm(X, d, w->cross_kv_W + (size_t)2 * K * d, 2LL * p.L * d, KV,
                           2LL * nh * d, (int)p.S_tot, 2 * nh * d, d),
                false, EPI_STORE, st));
  }
  }  // (context operands)

  // trunk: K layers over the n_pos position rows, shared by all beams (beam.py:159-163)
  if (K > 0) {
    long long rows = (long long)B * p.n_pos;
    GR_LAUNCH(KC_SMALL, st, tile_rows_kernel<<<ceil_div(rows * d, 256), 256, 0, st>>>(w->pos, p.n_pos, d, Ht, rows));
    RowSet rs{};
    rs.few_rows = true;
    rs.rows = (int)rows;
    rs.max_group_rows = p.n_pos;
    rs.g_row_off = at<int>(ws, p.o_trow_off);
    rs.g_rows = at<int>(ws, p.o_trows);
    rs.row_req = at<int>(ws, p.o_trow_req);
    rs.qkv = at<float>(ws, p.o_QKVt);
    rs.hist_row0 = 0;
    rs.anc = at<int>(ws, p.o_tanc);
    rs.anc_stride = p.n_pos;
    rs.npos_row = at<int>(ws, p.o_tnpos);
    for (int i = 0; i < K; ++i)
      GR_TRY(p.tc ? layer_forward_tc(p, w, *wt, i, Ht, rs, ws, st)
                  : layer_forward(p, w, i, Ht, rs, ws, KV, st));
  }

  return GR4AD_OK;
}

// debug / A-B aid: GR4AD_NO_PROXY=1 selects with the histogram pass only
static bool no_proxy_window() {
  static const bool off = getenv("GR4AD_NO_PROXY") != nullptr;
  return off;
}

// Layered decode, split at the boundaries the per-level C entry points
// expose (gr4ad_encode_trunk / gr4ad_level_step / gr4ad_collect):
// context projection + shared encoder K/V + trunk + level-0 rows ...
static int layered_begin(const Plan &p, const gr4ad_weights *w, const float *features,
                         const float *context, void *ws, WeightsT &wt_store, const WeightsT *&wt,
                         cudaStream_t st) {
  GR_TRY(encode_and_trunk(p, w, features, context, ws, wt_store, wt, st));
  return init_level0(p.B, at<int>(ws, p.o_live), at<float>(ws, p.o_cum),
                     at<long long>(ws, p.o_prefix), at<int>(ws, p.o_anc), p.stride,
                     at<int>(ws, p.o_tok), st);
}

// ... one level step t (t == T: the value re-rank head pass) ...
static int layered_level(const Plan &p, const gr4ad_weights *w, const gr4ad_batch *bt, int t,
                         void *ws, const WeightsT *wt, cudaStream_t st) {
  const int B = p.B, T = p.T, d = p.d, K = p.K;
  int *eff = at<int>(ws, p.o_eff), *cap = at<int>(ws, p.o_cap);
  int *row_off = at<int>(ws, p.o_row_off), *live = at<int>(ws, p.o_live);
  int *row_req = at<int>(ws, p.o_row_req);
  int *tok = at<int>(ws, p.o_tok), *anc = at<int>(ws, p.o_anc);
  float *cum = at<float>(ws, p.o_cum);
  long long *prefix = at<long long>(ws, p.o_prefix);
  float *KV = at<float>(ws, p.o_KV), *Ht = at<float>(ws, p.o_Ht);
  float *Hs = at<float>(ws, p.o_Hs), *U = at<float>(ws, p.o_U);
  float *LG = at<float>(ws, p.o_LG);
  float2 *rinfo = at<float2>(ws, p.o_rinfo);
  float *hist = at<float>(ws, p.o_hist);
  const size_t hist_layer = (size_t)p.H * p.hist_ld;
  const int R = (int)p.R[t];
  const long long h0 = p.hist_off[t];
  // token input + gated fusion (beam.py:180-191; layers.py:129-133)
  const float *emb_prev = t > 0 ? w->emb[t - 1] : nullptr;
  if (K > 0 && p.tc && wt && d % 8 == 0) {
    // h = [m (s W_g) | s] W_f = (m (s W_g)) W_f[0:d] + s W_f[d:2d]: the
    // token-side products come from the per-snapshot tables (one d x d GEMM
    // per row instead of three)
    __half *Uh = at<__half>(ws, p.o_U16), *Ul = Uh + (size_t)p.Rw * 2 * d;
    GR_TRY(fuse_gather(t, R, d, tok + h0, wt->fuse_tab[t], p.fuse_n[t], Ht + (size_t)t * d,
                       (long long)p.n_pos * d, row_req + h0, Hs, Uh, Ul, st));
    GemmArgs gf = plain_gemm(nullptr, d, w->fuse_Wf, d, Hs, d, R, d, d);
    gf.R = Hs;
    gf.ldr = d;
    GR_TRY(dense_split(p, gf, wt->wf_top, Uh, Ul, R, EPI_RESID, st, nullptr, nullptr, t == 0));
  } else if (K > 0) {
    GR_TRY(level_input(t, R, d, w->bos, emb_prev, tok + h0, nullptr, U, nullptr, st));
    GemmArgs gg = plain_gemm(U + d, 2LL * d, w->fuse_Wg, d, U, 2LL * d, R, d, d);
    gg.vec = Ht + (size_t)t * d;
    gg.vec_ld = (long long)p.n_pos * d;
    gg.row_req = row_req + h0;
    GR_TRY(dense(p, gg, wt ? wt->wg : nullptr, R, EPI_MULVEC, st));
    GR_TRY(dense(p, plain_gemm(U, 2LL * d, w->fuse_Wf, d, Hs, d, R, d, 2 * d),
                 wt ? wt->wf : nullptr, R, EPI_STORE, st));
  } else {
    GR_TRY(level_input(t, R, d, w->bos, emb_prev, tok + h0, w->pos + (size_t)t * d, nullptr,
                       Hs, st));
  }
  // head layers K..L-1 against the shared context KV (beam.py:243-255)
  RowSet rs{};
  rs.few_rows = t == 0;  // one row per request
  rs.rows = R;
  rs.max_group_rows = p.maxcap[t];
  rs.g_row_off = row_off + (size_t)t * B;
  rs.g_rows = cap + (size_t)t * B;
  rs.row_req = row_req + h0;
  rs.hist_row0 = h0;
  rs.anc = anc;
  rs.anc_stride = p.stride;
  rs.npos_u = t + 1;
  rs.npos_row = nullptr;
  bool h_split = false;  // the last layer left Hs as fp16 hi / lo in N
  for (int i = K; i < p.L; ++i) {
    rs.qkv = hist + (size_t)(i - K) * hist_layer;
    if (wt)
      GR_TRY(layer_forward_tc(p, w, *wt, i, Hs, rs, ws, st,
                              (i == p.L - 1 && t < T) ? &h_split : nullptr));
    else
      GR_TRY(layer_forward(p, w, i, Hs, rs, ws, KV, st));
  }
  if (t == T) {  // value re-rank step (beam.py:258-288)
    float *vlog = at<float>(ws, p.o_vlog);
    GR_TRY(dense(p, plain_gemm(Hs, d, w->head_value, p.nb, vlog, p.nb, R, p.nb, d),
                 wt ? wt->hv : nullptr, R, EPI_STORE, st));
    return GR4AD_OK;
  }
  // codebook projection + log-softmax + score accumulation + top-k (beam.py:198-210)
  const int V = p.V[t];
  const GemmArgs lg = plain_gemm(Hs, d, w->head[t], V, LG, V, R, V, d);
  const float4 *proxies = nullptr;
  if (p.tc && wt && d % 8 == 0 && tc_eligible(d, d, d, Hs, wt->head[t])) {
    // log-sum-exp partials from the GEMM epilogue (no second pass over the logits)
    TcArgs tl{};
    static_cast<GemmArgs &>(tl) = lg;
    tl.b_hi = wt->head[t];
    tl.b_lo = wt->head[t] + p.wt_floats;
    tl.ldb = d;
    tl.alpha = lg.alpha / kWeightScale;
    tl.lse_part = at<float4>(ws, p.o_lsep);
    tl.lse_ld = (V + 127) / 128;
    tl.few_rows = t == 0 ? 1 : 0;
    if (h_split) {
      tl.a_hi = at<__half>(ws, p.o_N);
      tl.a_lo = tl.a_hi + (size_t)p.Rw * d;
    }
    GR_TRY(gemm_tc(tl, R, d, V, d, EPI_STORE_LSE, st));
    GR_TRY(lse_merge(tl.lse_part, tl.lse_ld, R, rinfo, st));
    if (!bt->valid_prefix[t] && !no_proxy_window()) proxies = tl.lse_part;
  } else {
    GR_TRY(dense(p, lg, wt ? wt->head[t] : nullptr, R, EPI_STORE, st));
    GR_TRY(row_lse(LG, V, R, V, rinfo, st));
  }
  if (bt->valid_prefix[t]) {
    GR_TRY(mask_rows(LG, V, R, V, prefix + h0,
                     reinterpret_cast<const long long *>(bt->valid_prefix[t]),
                     bt->valid_prefix_count[t], st));
  }
  SelectArgs sa{};
  sa.logits = LG; sa.ld = V; sa.V = V; sa.level = t;
  sa.rowinfo = rinfo; sa.cum = cum;
  sa.proxies = proxies; sa.proxy_ld = (V + 127) / 128;
  sa.row_off = row_off + (size_t)t * B;
  sa.live = live + (size_t)t * B;
  sa.eff = eff + (size_t)t * B;
  sa.hist_off = (int)h0;
  sa.out_row_off = row_off + (size_t)(t + 1) * B;
  sa.out_cap = cap + (size_t)(t + 1) * B;
  sa.out_live = live + (size_t)(t + 1) * B;
  sa.out_hist_off = (int)p.hist_off[t + 1];
  sa.tok = tok; sa.cum_out = cum; sa.prefix = prefix; sa.anc = anc;
  sa.anc_stride = p.stride;
  GR_TRY(topk_select(sa, B, 0, 0, p.max_cand[t], st));
  return GR4AD_OK;
}

// ... and the results of the last level (or of the re-rank).
static int layered_end(const Plan &p, const gr4ad_batch *bt, gr4ad_results *out, void *ws,
                       cudaStream_t st) {
  const int B = p.B, T = p.T;
  int *row_off = at<int>(ws, p.o_row_off), *live = at<int>(ws, p.o_live);
  return collect_results(B, T, row_off + (size_t)T * B, live + (size_t)T * B,
                         (int)p.hist_off[T], at<int>(ws, p.o_tok), at<int>(ws, p.o_anc), p.stride,
                         at<float>(ws, p.o_cum), p.rerank ? at<float>(ws, p.o_vlog) : nullptr,
                         p.nb, bt->value_reps, out->max_out, out->count, out->tokens, out->score,
                         st);
}

static int run_plan(const Plan &p, const gr4ad_dims *dm, const gr4ad_weights *w,
                    const gr4ad_batch *bt, const float *features, const float *context,
                    gr4ad_results *out, void *ws, cudaStream_t st) {
  const int B = p.B, T = p.T, d = p.d, K = p.K;
  if (B == 0) return GR4AD_OK;
  int *range_flag = at<int>(ws, p.o_flag);
  GR_CUDA(cudaMemsetAsync(range_flag, 0, sizeof(int), st));
  if (p.fused) {
    FusedArgs f{};
    f.range_flag = range_flag;
    f.w = *w;
    if (!features && !context) return set_err(GR4AD_ERR_VALUE, "either features or context is required");
    f.features = features;
    f.context = context;
    f.ctx_off = at<int>(ws, p.o_in_off);
    f.ctx_len = at<int>(ws, p.o_ctx_len);
    f.eff = at<int>(ws, p.o_eff);
    f.value_reps = bt->value_reps;
    f.B = B; f.D = d; f.F = p.F; f.dff = p.dff; f.L = p.L; f.K = K; f.T = T;
    f.nb = p.nb; f.n_pos = p.n_pos; f.rerank = p.rerank ? 1 : 0;
    for (int t = 0; t < T; ++t) f.V[t] = p.V[t];
    f.S_max = p.S_max; f.Hrows = p.f_Hrows;
    for (int t = 0; t < GR4AD_MAX_LEVELS + 2; ++t) {
      f.hoff[t] = p.f_hoff[t];
      f.moff[t] = p.f_moff[t];
    }
    f.s_X = p.f_s[0]; f.s_KV = p.f_s[1]; f.s_TR = p.f_s[2]; f.s_TQ = p.f_s[3];
    f.s_hist = p.f_s[4]; f.s_par = p.f_s[5]; f.s_tok = p.f_s[6]; f.s_cum = p.f_s[7];
    f.s_bins = p.f_s[8]; f.s_scr = p.f_s[9]; f.s_sort = p.f_s[10]; f.s_ws = p.f_s[11];
    f.keys = at<uint32_t>(ws, p.o_keys);
    f.keys_per_req = p.f_keys_per_req;
    f.max_out = out->max_out;
    f.sort_cap = p.f_sort_cap;
    f.out_count = out->count; f.out_tokens = out->tokens; f.out_score = out->score;
    f.dbg = reinterpret_cast<long long *>(static_cast<char *>(ws) + p.total -
                                          (size_t)B * kDbgSlots * sizeof(long long));
    if (p.f_mma) {
      f.s_X = p.f_s4[0]; f.s_KV = p.f_s4[1]; f.s_TR = p.f_s4[2]; f.s_TQ = p.f_s4[3];
      f.s_hist = p.f_s4[4]; f.s_par = p.f_s4[5]; f.s_tok = p.f_s4[6]; f.s_cum = p.f_s4[7];
      f.s_bins = p.f_s4[8]; f.s_scr = p.f_s4[9]; f.s_sort = p.f_s4[10]; f.s_ws = p.f_s4[11];
      f.s_XT = p.f_s4[12];
      f.s_mrg = p.f_s4[13];
      f.s_head = p.f_s4[14];
      f.s_mbar = p.f_s4[15];
      f.head_floats = p.f_head_floats;
      f.s_hst = p.f_s4[16];
      f.s_pfx = p.f_s4[17];
      for (int t = 0; t < T; ++t) {
        f.vp_rp[t] = bt->valid_prefix[t] ? at<int>(ws, p.o_vprp[t]) : nullptr;
        f.vp_keys[t] = reinterpret_cast<const long long *>(bt->valid_prefix[t]);
      }
      f.hst_rows = p.f_hst_rows;
      f.tile_split = 1;
      f.Hrows = p.f_Hrows_mma;
      for (int t = 0; t < GR4AD_MAX_LEVELS + 2; ++t) f.hoff[t] = p.f_hoff4[t];
      static thread_local FragJobs jobs;  // ~6 KB: kept off the stack
      uint4 *frag = atd<uint4>(p, ws, p.o_frag);
      frag_layout(p, w, &jobs, &f.fi);
      f.frag = frag;
      jobs.tu = TrunkUJob{};
      if (K > 0 && d <= 32) {
        const gr4ad_layer &L0 = w->layer[0];
        jobs.tu = TrunkUJob{w->pos, L0.ln1_g, L0.ln1_b, L0.cross_Wq, w->cross_kv_W,
                            atd<float>(p, ws, p.o_tu), d, 2 * p.L * d, p.n_pos};
        f.trunk_u = jobs.tu.u;
      }
      if (!p.weights_prepared) GR_TRY(frag_prep_launch(jobs, frag, range_flag, st));
      return fused_mma_launch(f, B, p.f_smem4, st);
    }
    return fused_small_launch(f, B, p.f_smem, st);
  }
  WeightsT wt_store;
  const WeightsT *wt = nullptr;
  GR_TRY(layered_begin(p, w, features, context, ws, wt_store, wt, st));
  const int last = p.rerank ? T : T - 1;
  for (int t = 0; t <= last; ++t) GR_TRY(layered_level(p, w, bt, t, ws, wt, st));
  return layered_end(p, bt, out, ws, st);
}

}  // namespace gr

using namespace gr;

extern "C" {

int gr4ad_abi_version(void) { return GR4AD_ABI_VERSION; }

const char *gr4ad_last_error(void) { return g_err; }

void gr4ad_profile_begin(void) {
  if (!g_prof) g_prof = new std::vector<ProfRec>();
  for (auto &r : *g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof->clear();
  g_prof_on = true;
}

int gr4ad_profile_end(double *ms, long long *launches, int n_classes) {
  g_prof_on = false;
  for (int c = 0; c < n_classes; ++c) {
    ms[c] = 0.0;
    launches[c] = 0;
  }
  if (!g_prof) return GR4AD_OK;
  // GR4AD_PROF_DUMP=<path>: append every launch (class, ms, shape tag) -- the
  // per-launch attribution behind the bench's per-class roofline
  static const char *dump_path = getenv("GR4AD_PROF_DUMP");
  FILE *dump = dump_path ? fopen(dump_path, "a") : nullptr;
  for (auto &r : *g_prof) {
    GR_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    GR_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (dump) fprintf(dump, "%d\t%.4f\t%s\n", r.cls, t, r.tag.c_str());
    if (r.cls >= 0 && r.cls < n_classes) {
      ms[r.cls] += t;
      launches[r.cls] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (dump) {
    fprintf(dump, "--\n");
    fclose(dump);
  }
  g_prof->clear();
  return GR4AD_OK;
}

long long gr4ad_take_launch_count(void) {
  long long n = g_launches;
  g_launches = 0;
  return n;
}

const char *gr4ad_status_string(int s) {
  switch (s) {
    case GR4AD_OK: return "ok";
    case GR4AD_ERR_VALUE: return "invalid argument";
    case GR4AD_ERR_UNSUPPORTED: return "unsupported shape";
    case GR4AD_ERR_WORKSPACE: return "workspace too small";
    case GR4AD_ERR_CUDA: return "CUDA error";
    case GR4AD_ERR_RANGE: return "fp16 split range exceeded";
    default: return "unknown status";
  }
}

int gr4ad_workspace_bytes(const gr4ad_dims *dims, const gr4ad_batch *batch, size_t *bytes,
                          int *max_out) {
  Plan p;
  GR_TRY(make_plan(dims, batch, p));
  if (bytes) *bytes = p.total;
  if (max_out) *max_out = p.max_out;
  return GR4AD_OK;
}

int gr4ad_prepare(const gr4ad_dims *dims, const gr4ad_batch *batch, void *workspace,
                  size_t workspace_bytes, void *stream) {
  Plan p;
  GR_TRY(make_plan(dims, batch, p));
  if (workspace_bytes < p.total)
    return set_err(GR4AD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, p.total);
  GR_TRY(upload_tables(p, workspace, (cudaStream_t)stream));
  if (p.fused)  // masking tables of the warp-MMA kernel
    for (int t = 0; t < p.T; ++t)
      if (batch->valid_prefix[t])
        GR_TRY(csr_rows(reinterpret_cast<const long long *>(batch->valid_prefix[t]),
                        batch->valid_prefix_count[t], p.V[t], p.vp_np[t],
                        at<int>(workspace, p.o_vprp[t]), (cudaStream_t)stream));
  return GR4AD_OK;
}

int gr4ad_beam_search_run(const gr4ad_dims *dims, const gr4ad_weights *w,
                          const gr4ad_batch *batch, const float *features, const float *context,
                          gr4ad_results *out, void *workspace, size_t workspace_bytes,
                          void *stream) {
  Plan p;
  GR_TRY(make_plan(dims, batch, p));
  if (workspace_bytes < p.total)
    return set_err(GR4AD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, p.total);
  if (!out || out->max_out < p.max_out)
    return set_err(GR4AD_ERR_VALUE, "results.max_out < %d", p.max_out);
  if (p.rerank && !batch->value_reps)
    return set_err(GR4AD_ERR_VALUE, "value_rerank requires bucket representatives");
  return run_plan(p, dims, w, batch, features, context, out, workspace, (cudaStream_t)stream);
}

// per-level entry points: the layered decode in three parts
static int split_plan(const gr4ad_dims *dims, const gr4ad_batch *batch, size_t workspace_bytes,
                      Plan &p) {
  GR_TRY(make_plan(dims, batch, p));
  if (workspace_bytes < p.total)
    return set_err(GR4AD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, p.total);
  if (p.fused)
    return set_err(GR4AD_ERR_UNSUPPORTED,
                   "the per-level entry points run the layered path: set decode_path 1 or 3");
  if (p.rerank && !batch->value_reps)
    return set_err(GR4AD_ERR_VALUE, "value_rerank requires bucket representatives");
  return GR4AD_OK;
}

int gr4ad_encode_trunk(const gr4ad_dims *dims, const gr4ad_weights *w, const gr4ad_batch *batch,
                       const float *features, const float *context, void *workspace,
                       size_t workspace_bytes, void *stream) {
  Plan p;
  GR_TRY(split_plan(dims, batch, workspace_bytes, p));
  if (p.B == 0) return GR4AD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (p.lat_ok && !features)
    return set_err(GR4AD_ERR_VALUE,
                   "per-level decode of this batch attends over the request features: pass "
                   "features, or decode_path 5 to encode from a projected context");
  GR_CUDA(cudaMemsetAsync(at<int>(workspace, p.o_flag), 0, sizeof(int), st));
  WeightsT wt_store;
  const WeightsT *wt = nullptr;
  return layered_begin(p, w, features, context, workspace, wt_store, wt, st);
}

int gr4ad_level_step(const gr4ad_dims *dims, const gr4ad_weights *w, const gr4ad_batch *batch,
                     int level, void *workspace, size_t workspace_bytes, void *stream) {
  Plan p;
  GR_TRY(split_plan(dims, batch, workspace_bytes, p));
  if (level < 0 || level > p.T || (level == p.T && !p.rerank))
    return set_err(GR4AD_ERR_VALUE, "level %d outside [0, %d)", level, p.T + (p.rerank ? 1 : 0));
  if (p.B == 0) return GR4AD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  WeightsT wt_store;
  const WeightsT *wt = nullptr;
  if (p.tc) {  // the derived weight copies: pointers only (built by encode_trunk / prepare)
    GR_TRY(prep_weights_t(p, w, workspace, wt_store, st, false));
    wt_store.lat = p.lat_ok;  // (gr4ad_encode_trunk had the features)
    wt = &wt_store;
  }
  return layered_level(p, w, batch, level, workspace, wt, st);
}

int gr4ad_collect(const gr4ad_dims *dims, const gr4ad_batch *batch, gr4ad_results *out,
                  void *workspace, size_t workspace_bytes, void *stream) {
  Plan p;
  GR_TRY(split_plan(dims, batch, workspace_bytes, p));
  if (!out || out->max_out < p.max_out)
    return set_err(GR4AD_ERR_VALUE, "results.max_out < %d", p.max_out);
  if (p.B == 0) return GR4AD_OK;
  return layered_end(p, batch, out, workspace, (cudaStream_t)stream);
}

int gr4ad_derived_layout(const gr4ad_dims *dims, const gr4ad_batch *batch, size_t *bytes,
                         unsigned long long *signature) {
  gr4ad_batch b = *batch;
  b.derived = nullptr;
  b.derived_bytes = 0;
  Plan p;
  GR_TRY(make_plan(dims, &b, p));
  if (bytes) *bytes = p.derived_total;
  if (signature) *signature = p.derived_sig;
  return GR4AD_OK;
}

int gr4ad_range_flag_offset(const gr4ad_dims *dims, const gr4ad_batch *batch, size_t *offset) {
  Plan p;
  GR_TRY(make_plan(dims, batch, p));
  if (offset) *offset = p.o_flag;
  return GR4AD_OK;
}

int gr4ad_prepare_weights(const gr4ad_dims *dims, const gr4ad_weights *w,
                          const gr4ad_batch *batch, void *workspace, size_t workspace_bytes,
                          void *stream) {
  Plan p;
  GR_TRY(make_plan(dims, batch, p));
  // into the caller's derived buffer (no workspace needed) or the workspace
  if (!p.derived && workspace_bytes < p.total)
    return set_err(GR4AD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, p.total);
  if (p.B == 0) return GR4AD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  void *ws = workspace;
  int *flag = atd<int>(p, ws, p.o_dflag);
  GR_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  if (p.fused && p.f_mma) {
    static thread_local FragJobs jobs;  // ~7 KB: kept off the stack
    FragIndex fi;
    frag_layout(p, w, &jobs, &fi);
    jobs.tu = TrunkUJob{};
    if (p.K > 0 && p.d <= 32) {
      const gr4ad_layer &L0 = w->layer[0];
      jobs.tu = TrunkUJob{w->pos, L0.ln1_g, L0.ln1_b, L0.cross_Wq, w->cross_kv_W,
                          atd<float>(p, ws, p.o_tu), p.d, 2 * p.L * p.d, p.n_pos};
    }
    GR_TRY(frag_prep_launch(jobs, atd<uint4>(p, ws, p.o_frag), flag, st));
  } else if (p.tc) {
    WeightsT wt;
    GR_TRY(prep_weights_t(p, w, ws, wt, st, true));
  }
  int h = 0;
  GR_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  GR_CUDA(cudaStreamSynchronize(st));
  if (h)
    return set_err(GR4AD_ERR_RANGE,
                   "a weight exceeded the fp16 split range (|weight| < 32): decode with the "
                   "CUDA-core path (decode_path layered / fused_simt)");
  return GR4AD_OK;
}

int gr4ad_range_status(const gr4ad_dims *dims, const gr4ad_batch *batch, const void *workspace,
                       void *stream) {
  Plan p;
  GR_TRY(make_plan(dims, batch, p));
  if (p.B == 0) return GR4AD_OK;
  int flag = 0;
  cudaStream_t st = (cudaStream_t)stream;
  GR_CUDA(cudaMemcpyAsync(&flag, static_cast<const char *>(workspace) + p.o_flag, sizeof(int),
                          cudaMemcpyDeviceToHost, st));
  GR_CUDA(cudaStreamSynchronize(st));
  if (flag)
    return set_err(GR4AD_ERR_RANGE,
                   "an operand exceeded the fp16 split range (|weight| < 32, |context X| < 256): "
                   "decode with the CUDA-core path (decode_path layered / fused_simt)");
  return GR4AD_OK;
}

int gr4ad_beam_search(const gr4ad_dims *dims, const gr4ad_weights *w, const gr4ad_batch *batch,
                      const float *features, const float *context, gr4ad_results *out,
                      void *workspace, size_t workspace_bytes, void *stream) {
  GR_TRY(gr4ad_prepare(dims, batch, workspace, workspace_bytes, stream));
  return gr4ad_beam_search_run(dims, w, batch, features, context, out, workspace,
                               workspace_bytes, stream);
}


// ---------------------------------------------------------------------------
// teacher-forced sequence scoring (decoder.py:162-219)
// ---------------------------------------------------------------------------
struct ScoreLayout {
  size_t o_tab, o_qkv, tab_bytes, total;
  int n_seq, n_pos, rows;
};

static int score_plan(const gr4ad_dims *dims, const gr4ad_batch *batch, int n_seq, Plan &p,
                      ScoreLayout &sl) {
  if (n_seq < 0) return set_err(GR4AD_ERR_VALUE, "n_seq < 0");
  gr4ad_batch b = *batch;
  const int dp = batch->decode_path;
  b.decode_path = (dp == 3 || dp == 5) ? dp : (dp == 1 ? 1 : 0);
  if (b.decode_path == 0) b.decode_path = (dims->d >= 64) ? 3 : 1;  // layered paths only
  if (b.decode_path == 3 || b.decode_path == 5) {  // tensor path needs alignment
    bool ok = dims->d % 8 == 0 && dims->d_ff % 4 == 0 && dims->feat_dim % 4 == 0;
    for (int t = 0; t < dims->n_levels; ++t) ok &= dims->vocab[t] % 4 == 0;
    if (!ok) b.decode_path = (dp == 3 || dp == 5) ? dp : 1;  // (forced: make_plan reports it)
  }
  const int n_pos = dims->n_levels + (batch->value_rerank ? 1 : 0);
  GR_TRY(make_plan(dims, &b, p, (long long)n_seq * n_pos));
  sl.n_seq = n_seq;
  sl.n_pos = n_pos;
  sl.rows = n_seq * n_pos;
  size_t o = p.total;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  const size_t I = sizeof(int);
  sl.o_tab = take(I * ((size_t)6 * n_seq + (size_t)sl.rows * (3 + n_pos)));
  sl.tab_bytes = I * ((size_t)6 * n_seq + (size_t)sl.rows * (3 + n_pos));
  sl.o_qkv = take(sizeof(float) * (size_t)sl.rows * p.hist_ld);
  sl.total = o;
  return GR4AD_OK;
}

int gr4ad_score_workspace_bytes(const gr4ad_dims *dims, const gr4ad_batch *batch, int n_seq,
                                size_t *bytes) {
  Plan p;
  ScoreLayout sl;
  GR_TRY(score_plan(dims, batch, n_seq, p, sl));
  if (bytes) *bytes = sl.total;
  return GR4AD_OK;
}

int gr4ad_score_sequences(const gr4ad_dims *dims, const gr4ad_weights *w, const gr4ad_batch *batch,
                          const float *features, const float *context, int n_seq, const int *req,
                          const int *tokens, float *logp, float *value_logits, float *head_logits,
                          void *workspace, size_t workspace_bytes, void *stream) {
  Plan p;
  ScoreLayout sl;
  GR_TRY(score_plan(dims, batch, n_seq, p, sl));
  if (workspace_bytes < sl.total)
    return set_err(GR4AD_ERR_WORKSPACE, "workspace %zu < %zu bytes", workspace_bytes, sl.total);
  if (n_seq == 0 || p.B == 0) return GR4AD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  void *ws = workspace;
  GR_CUDA(cudaMemsetAsync(at<int>(ws, p.o_flag), 0, sizeof(int), st));
  const int d = p.d, T = p.T, np = sl.n_pos, Rs = sl.rows;
  // per-sequence tables: attention group = sequence (its request's context),
  // causal ancestors = earlier positions of the same sequence
  std::vector<int> tab(sl.tab_bytes / sizeof(int), 0);
  int *g_row_off = tab.data(), *g_rows = g_row_off + n_seq, *g_ctx_off = g_rows + n_seq;
  int *g_ctx_len = g_ctx_off + n_seq, *row_grp = g_ctx_len + n_seq + 2 * n_seq;
  int *vec_row = row_grp + Rs, *npos = vec_row + Rs, *anc = npos + Rs;
  for (int s = 0; s < n_seq; ++s) {
    const int r = req[s];
    if (r < 0 || r >= p.B) return set_err(GR4AD_ERR_VALUE, "sequence %d: request %d out of range", s, r);
    g_row_off[s] = s * np;
    g_rows[s] = np;
    g_ctx_off[s] = p.ctx_off[r];
    g_ctx_len[s] = p.ctx_len[r];
    for (int q = 0; q < np; ++q) {
      const int row = s * np + q;
      row_grp[row] = s;
      vec_row[row] = r * np + q;
      npos[row] = q + 1;
      for (int tau = 0; tau < np; ++tau) anc[(size_t)row * np + tau] = s * np + std::min(tau, q);
    }
  }
  GR_TRY(upload_tables(p, ws, st));
  GR_CUDA(cudaMemcpyAsync(at<int>(ws, sl.o_tab), tab.data(), sl.tab_bytes, cudaMemcpyHostToDevice, st));
  const int *d_tab = at<int>(ws, sl.o_tab);
  const int *d_row_off = d_tab, *d_rows = d_row_off + n_seq, *d_ctx_off = d_rows + n_seq;
  const int *d_ctx_len = d_ctx_off + n_seq, *d_row_grp = d_ctx_len + n_seq + 2 * n_seq;
  const int *d_vec_row = d_row_grp + Rs, *d_npos = d_vec_row + Rs, *d_anc = d_npos + Rs;

  WeightsT wt_store;
  const WeightsT *wt = nullptr;
  GR_TRY(encode_and_trunk(p, w, features, context, ws, wt_store, wt, st));
  float *KV = at<float>(ws, p.o_KV), *Ht = at<float>(ws, p.o_Ht);
  float *Hs = at<float>(ws, p.o_Hs), *U = at<float>(ws, p.o_U), *LG = at<float>(ws, p.o_LG);
  float2 *rinfo = at<float2>(ws, p.o_rinfo);
  // fused inputs (decoder.py:178-185)
  SeqInputArgs si{};
  si.rows = Rs; si.d = d; si.n_pos = np; si.T = T; si.tokens = tokens;
  si.bos = w->bos; si.pos = w->pos;
  for (int t = 0; t < T; ++t) si.emb[t] = w->emb[t];
  if (p.K > 0) {
    si.U = U;
    GR_TRY(seq_input(si, st));
    GemmArgs gg = plain_gemm(U + d, 2LL * d, w->fuse_Wg, d, U, 2LL * d, Rs, d, d);
    gg.vec = Ht;  // trunk state of (request, position)
    gg.vec_ld = d;
    gg.row_req = d_vec_row;
    GR_TRY(dense(p, gg, wt ? wt->wg : nullptr, Rs, EPI_MULVEC, st));
    GR_TRY(dense(p, plain_gemm(U, 2LL * d, w->fuse_Wf, d, Hs, d, Rs, d, 2 * d),
                 wt ? wt->wf : nullptr, Rs, EPI_STORE, st));
  } else {
    si.H = Hs;
    GR_TRY(seq_input(si, st));
  }
  // head layers K..L-1 in causal 2-D mode over each sequence (decoder.py:186)
  RowSet rs{};
  rs.rows = Rs;
  rs.max_group_rows = np;
  rs.groups = n_seq;
  rs.g_row_off = d_row_off;
  rs.g_rows = d_rows;
  rs.g_ctx_off = d_ctx_off;
  rs.g_ctx_len = d_ctx_len;
  rs.row_req = d_row_grp;
  rs.qkv = at<float>(ws, sl.o_qkv);
  rs.hist_row0 = 0;
  rs.anc = d_anc;
  rs.anc_stride = np;
  rs.npos_row = d_npos;
  for (int i = p.K; i < p.L; ++i)
    GR_TRY(wt ? layer_forward_tc(p, w, *wt, i, Hs, rs, ws, st)
              : layer_forward(p, w, i, Hs, rs, ws, KV, st));
  // per-level logits of position t (decoder.py:189-194) and log-probabilities
  long long hoff = 0;
  for (int t = 0; t < T; ++t) {
    const int V = p.V[t];
    GemmArgs g = plain_gemm(Hs + (size_t)t * d, (long long)np * d, w->head[t], V, LG, V, n_seq, V, d);
    GR_TRY(dense(p, g, wt ? wt->head[t] : nullptr, (long long)n_seq, EPI_STORE, st));
    GR_TRY(row_lse(LG, V, n_seq, V, rinfo, st));
    GR_TRY(gather_logp(LG, V, n_seq, rinfo, tokens, T, t, logp, st));
    if (head_logits)
      GR_CUDA(cudaMemcpy2DAsync(head_logits + hoff, sizeof(float) * p.Vsum, LG, sizeof(float) * V,
                                sizeof(float) * V, n_seq, cudaMemcpyDeviceToDevice, st));
    hoff += V;
  }
  if (value_logits && np > T) {  // value-bucket logits at position T (decoder.py:196-197)
    GemmArgs g = plain_gemm(Hs + (size_t)T * d, (long long)np * d, w->head_value, p.nb,
                            value_logits, p.nb, n_seq, p.nb, d);
    GR_TRY(dense(p, g, wt ? wt->hv : nullptr, (long long)n_seq, EPI_STORE, st));
  }
  if (p.tc) {  // fp16 operand range (the scoring API is synchronous for its caller)
    int flag = 0;
    GR_CUDA(cudaMemcpyAsync(&flag, at<int>(ws, p.o_flag), sizeof(int), cudaMemcpyDeviceToHost, st));
    GR_CUDA(cudaStreamSynchronize(st));
    if (flag)
      return set_err(GR4AD_ERR_RANGE,
                     "an operand exceeded the fp16 split range (|weight| < 32, |context X| < "
                     "256): score with the CUDA-core path");
  }
  return GR4AD_OK;
}

int gr4ad_context_process(const gr4ad_dims *dims, const gr4ad_weights *w, const float *features,
                          int rows, float *x, void *stream) {
  GemmArgs g = plain_gemm(features, dims->feat_dim, w->ctx_W, dims->d, x, dims->d, rows,
                          dims->d, dims->feat_dim);
  g.bias = w->ctx_b;
  return gemm(g, false, EPI_BIAS, (cudaStream_t)stream);
}

int gr4ad_encoder_kv(const gr4ad_dims *dims, const gr4ad_weights *w, const float *x, int rows,
                     int lo, int hi, float *kv, void *stream) {
  if (!(0 <= lo && lo <= hi && hi <= dims->n_layers))
    return set_err(GR4AD_ERR_VALUE, "layer range [%d, %d) outside [0, %d)", lo, hi,
                   dims->n_layers);
  const int d = dims->d;
  const long long ldw = 2LL * dims->n_layers * d;
  return gemm(plain_gemm(x, d, w->cross_kv_W + (size_t)2 * lo * d, ldw, kv,
                         2LL * (hi - lo) * d, rows, 2 * (hi - lo) * d, d),
              false, EPI_STORE, (cudaStream_t)stream);
}

int gr4ad_gemm(const float *A, long long lda, const float *BT, long long ldb, float *C,
               long long ldc, int M, int N, int K, int backend, void *stream) {
  if (M < 0 || N < 0 || K < 1) return set_err(GR4AD_ERR_VALUE, "bad gemm shape");
  cudaStream_t st = (cudaStream_t)stream;
  if (backend == 1) {
    if (!tc_eligible(lda, ldb, K, A, BT))
      return set_err(GR4AD_ERR_UNSUPPORTED, "tcgen05 gemm needs 16-B aligned K-major rows");
    TcArgs t{};
    static_cast<GemmArgs &>(t) = plain_gemm(A, lda, BT, ldb, C, ldc, M, N, K);
    return gemm_tc(t, M, K, N, K, EPI_STORE, st);
  }
  return gemm(plain_gemm(A, lda, BT, ldb, C, ldc, M, N, K), true, EPI_STORE, st);
}

int gr4ad_gemm_presplit(const void *a_hi, const void *a_lo, long long lda, const void *b_hi,
                        const void *b_lo, long long ldb, float *C, long long ldc, int M, int N,
                        int K, float alpha, void *stream) {
  if (M < 0 || N < 0 || K < 1) return set_err(GR4AD_ERR_VALUE, "bad gemm shape");
  if (lda % 8 || ldb % 8 || K % 8)
    return set_err(GR4AD_ERR_UNSUPPORTED, "pre-split gemm needs 16-B aligned fp16 rows");
  TcArgs t{};
  static_cast<GemmArgs &>(t) = plain_gemm(nullptr, lda, nullptr, ldb, C, ldc, M, N, K);
  t.alpha = alpha;
  t.a_hi = static_cast<const __half *>(a_hi);
  t.a_lo = static_cast<const __half *>(a_lo);
  t.b_hi = static_cast<const __half *>(b_hi);
  t.b_lo = static_cast<const __half *>(b_lo);
  return gemm_tc(t, M, K, N, K, EPI_STORE, (cudaStream_t)stream);
}

size_t gr4ad_topk_workspace_bytes(int n_problems, int b, int v) { return 256; }

int gr4ad_topk_precut(const float *prev_scores, const float *logprobs, int n_problems, int b,
                      int v, int k, int *out_beam, int *out_token, float *out_score,
                      int *out_count, void *workspace, size_t workspace_bytes, void *stream) {
  if (n_problems < 0 || b < 1 || v < 1 || k < 1)
    return set_err(GR4AD_ERR_VALUE, "bad selection shape");
  long long n = (long long)b * v;
  if (std::min((long long)k, n) > GR4AD_MAX_BEAM)
    return set_err(GR4AD_ERR_UNSUPPORTED, "k %d exceeds %d", k, GR4AD_MAX_BEAM);
  if (n >= 0xFFFFFFFFLL) return set_err(GR4AD_ERR_UNSUPPORTED, "too many candidates");
  SelectArgs sa{};
  sa.logits = logprobs; sa.ld = v; sa.V = v;
  sa.cum = prev_scores;
  sa.o_beam = out_beam; sa.o_token = out_token; sa.o_score = out_score;
  sa.o_count = out_count; sa.o_k = k;
  return topk_select(sa, n_problems, b, k, n, (cudaStream_t)stream);
}

size_t gr4ad_project_topk_workspace_bytes(int n_problems, int b, int v) {
  size_t rows = (size_t)n_problems * b;
  return align_up(rows * v * sizeof(float)) + align_up(rows * sizeof(float2));
}

int gr4ad_project_topk(const float *states, const float *head, int d, const float *prev_scores,
                       int n_problems, int b, int v, int k, int *out_beam, int *out_token,
                       float *out_score, int *out_count, void *workspace,
                       size_t workspace_bytes, void *stream) {
  if (n_problems < 0 || b < 1 || v < 1 || k < 1 || d < 1)
    return set_err(GR4AD_ERR_VALUE, "bad projection shape");
  if (workspace_bytes < gr4ad_project_topk_workspace_bytes(n_problems, b, v))
    return set_err(GR4AD_ERR_WORKSPACE, "workspace too small");
  long long n = (long long)b * v;
  if (std::min((long long)k, n) > GR4AD_MAX_BEAM)
    return set_err(GR4AD_ERR_UNSUPPORTED, "k %d exceeds %d", k, GR4AD_MAX_BEAM);
  cudaStream_t st = (cudaStream_t)stream;
  int rows = n_problems * b;
  float *LG = static_cast<float *>(workspace);
  float2 *ri = reinterpret_cast<float2 *>(static_cast<char *>(workspace) +
                                          align_up((size_t)rows * v * sizeof(float)));
  GR_TRY(gemm(plain_gemm(states, d, head, v, LG, v, rows, v, d), false, EPI_STORE, st));
  GR_TRY(row_lse(LG, v, rows, v, ri, st));
  SelectArgs sa{};
  sa.logits = LG; sa.ld = v; sa.V = v;
  sa.rowinfo = ri; sa.cum = prev_scores;
  sa.o_beam = out_beam; sa.o_token = out_token; sa.o_score = out_score;
  sa.o_count = out_count; sa.o_k = k;
  return topk_select(sa, n_problems, b, k, n, st);
}

}  // extern "C"
