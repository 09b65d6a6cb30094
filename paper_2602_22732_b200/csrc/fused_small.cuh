// Fused per-request decode for small models (see fused_small.cu).
#pragma once
#include "common.cuh"

namespace gr {

// Fragment-ordered weights of the warp-MMA fused kernel: for a (Kin x Nout)
// matrix, uint4 [Kin/16][Nout/8][32 lanes] = {b0 hi, b1 hi, b0 lo, b1 lo},
// the B fragment of mma.m16n8k16 in fp16 hi / lo of 2048 W with
// b0 = W[16kk + 2t, +1][8nn + g], b1 = W[16kk + 8 + 2t, +1][8nn + g]
// (g = lane / 4, t = lane & 3).  A C fragment pair is then directly the A
// fragment of the next product.  Offsets are in 16-byte units.
constexpr int kMaxHeadLayersMma = 16;
constexpr int kDbgSlots = 48;  // per-request phase stamps (GR_FUSED_TIMING builds)
struct FragIndex {
  long long wg, wf_m, wf_s, value;
  long long head[GR4AD_MAX_LEVELS];
  long long cq[kMaxHeadLayersMma], co[kMaxHeadLayersMma], sq[kMaxHeadLayersMma],
      sk[kMaxHeadLayersMma], sv[kMaxHeadLayersMma], so[kMaxHeadLayersMma],
      w1[kMaxHeadLayersMma], w2[kMaxHeadLayersMma];
};
struct FragJob {
  const float *src;  // element (k, n) at src[k * sk + n * sn]
  long long sk, sn, dst;
  int kin, nout, nreal;  // nout padded to 8; columns >= nreal are zero
};
constexpr int kMaxFragJobs = 4 + GR4AD_MAX_LEVELS + 8 * kMaxHeadLayersMma;
// frag_prep's extra block: trunk layer 0's position-only queries
// u_p = (LN1(pos_p) Wq) Wk^T (d <= 32), the fused trunk's starting point
struct TrunkUJob {
  const float *pos, *ln1_g, *ln1_b, *wq, *kv;  // kv: cross_kv_W (Wk of layer 0 = columns [0, d))
  float *u;                                    // [n_pos][d]; NULL: no trunk
  int d, ldw, n_pos;
};
struct FragJobs {
  int n;
  FragJob job[kMaxFragJobs];
  TrunkUJob tu;
};

struct FusedArgs {
  gr4ad_weights w;
  const float *features;  // (rows, F) caller layout, or NULL
  const float *context;   // (rows, D) when features == NULL
  const int *ctx_off, *ctx_len;  // [B] caller row offsets / lengths
  const int *eff;                // [T][B]
  const float *value_reps;
  int B, D, F, dff, L, K, T, nb, n_pos, rerank;
  int V[GR4AD_MAX_LEVELS];
  int S_max, Hrows;
  int hoff[GR4AD_MAX_LEVELS + 2];  // history row offset of each level
  int moff[GR4AD_MAX_LEVELS + 2];  // level-row metadata offset of each level
  // shared-memory layout (float offsets)
  int s_X, s_KV, s_TR, s_TQ, s_hist, s_par, s_tok, s_cum, s_bins, s_scr, s_sort, s_ws;
  int s_XT;               // warp-MMA kernel: X^T
  int s_mrg;              // warp-MMA kernel: tile-group merge scratch
  int s_head;             // warp-MMA kernel: the level's codebook fragments (bulk copy)
  int head_floats;        // its capacity (floats); first holds the request's features
  int s_mbar;             // warp-MMA kernel: mbarrier of the codebook bulk copy
  int s_hst, hst_rows;    // warp-MMA kernel: per-row pass-2 state [hst_rows][D + 2]
  int tile_split;         // warp-MMA kernel: warps share tiles on small levels
  const float *trunk_u;   // warp-MMA kernel: [n_pos][D] layer-0 trunk queries (FragJobs.tu)
  int *range_flag;        // warp-MMA kernel: set when a scaled K / V leaves the fp16 range
  // warp-MMA kernel, valid-SID prefix masking: per level, CSR rows over the
  // prefix key P (vp_rp[t][P] .. vp_rp[t][P+1] index vp_keys[t]); NULL: no mask
  const int *vp_rp[GR4AD_MAX_LEVELS];
  const long long *vp_keys[GR4AD_MAX_LEVELS];
  int s_pfx;              // warp-MMA kernel: rows' prefix keys (int)
  const uint4 *frag;      // warp-MMA kernel: fragment-ordered weights (fp16 hi / lo)
  FragIndex fi;
  uint32_t *keys;  // candidate keys scratch (L2-resident), keys_per_req per request
  long long keys_per_req;
  int max_out;
  int sort_cap;  // entries of the shared sort buffer (>= every width, power of 2)
  int *out_count, *out_tokens;
  double *out_score;
  long long *dbg;  // GR_FUSED_TIMING builds: [B][kDbgSlots] globaltimer stamps
};

int fused_small_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st);
// warp-level tensor-core variant (mma.sync m16n8k16, 3xFP16), d = 16
int frag_prep_launch(const FragJobs &jobs, uint4 *frag, int *range_flag, cudaStream_t st);
int fused_mma_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st);

}  // namespace gr
