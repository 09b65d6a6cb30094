// Fused per-request decode for small models (see fused_small.cu).
#pragma once
#include "common.cuh"

namespace gr {

// transposed (row = output) copies of one layer's matrices, in the workspace
struct FusedLayerT {
  const float *cqT, *coT, *sqkvT, *soT, *w1T, *w2T;
};
struct FusedFuseT {
  const float *wgT, *wfT;
};

// list of src -> dst transposes (dst = src^T, src is rows x cols row-major)
struct FusedPrep {
  static constexpr int kMax = 40;
  int n;
  const float *src[kMax];
  float *dst[kMax];
  int rows[kMax], cols[kMax];
};

struct FusedArgs {
  gr4ad_weights w;
  FusedLayerT lt[GR4AD_MAX_LAYERS];
  FusedFuseT fuseT;
  const float *kvT;   // (2Ld, d)
  const float *ctxT;  // (d, F)
  const float *hvT;   // (n_buckets, d)
  const float *features;  // (sum S, F) or NULL
  const float *context;   // (sum S, D) when features == NULL
  const int *ctx_off, *ctx_len;  // [B]
  const int *eff;                // [T][B]
  const float *value_reps;
  int B, D, F, dff, L, K, T, nb, n_pos, rerank;
  int V[GR4AD_MAX_LEVELS];
  int Vmax;
  int S_max, KS, Hrows;
  int hoff[GR4AD_MAX_LEVELS + 2];  // history row offset of each level
  int moff[GR4AD_MAX_LEVELS + 2];  // level-row metadata offset of each level
  // shared-memory layout (float offsets)
  int s_X, s_KV, s_TR, s_TQ, s_hist, s_par, s_tok, s_cum, s_bins, s_scr, s_sort;
  uint32_t *keys;  // candidate keys scratch (L2-resident), keys_per_req per request
  long long keys_per_req;
  int max_out;
  int *out_count, *out_tokens;
  double *out_score;
  long long *dbg;  // GR_FUSED_TIMING builds: [B][16] globaltimer stamps
};

int fused_prep_launch(const FusedPrep &p, cudaStream_t st);
int fused_small_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st);

}  // namespace gr
