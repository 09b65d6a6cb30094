// Fused per-request decode for small models (see fused_small.cu).
#pragma once
#include "common.cuh"

namespace gr {

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
  uint32_t *keys;  // candidate keys scratch (L2-resident), keys_per_req per request
  long long keys_per_req;
  int max_out;
  int sort_cap;  // entries of the shared sort buffer (>= every width, power of 2)
  int *out_count, *out_tokens;
  double *out_score;
  long long *dbg;  // GR_FUSED_TIMING builds: [B][16] globaltimer stamps
};

int fused_small_launch(const FusedArgs &a, int n_requests, size_t smem, cudaStream_t st);

}  // namespace gr
