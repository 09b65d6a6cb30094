/*
 * gr4ad.h -- C ABI of the B200 LazyAR beam-serving library (libgr4ad.so).
 *
 * This is the drop-in boundary for the reference's serving hot path.  The
 * reference has no native FFI for it; its boundary is the Python call
 *   adrec.serving.beam.beam_search(model, context, schedule, shared_kv=True,
 *       precut=True, counter=None, value_rerank=False, buckets=None,
 *       trunk_depth=None)                     (pkg/src/adrec/serving/beam.py:112-143)
 * and the only native precedent is the Cython quantizer module
 * (pkg/src/adrec/_kernels/_core.pyx:15-67: typed memoryviews in, new arrays
 * out).  The entry points below are what a ctypes/cffi binding of that path
 * binds; each cites the reference function it replaces.
 *
 * Conventions
 *  - plain C types only; every float pointer is DEVICE memory holding fp32
 *    unless a field says "host";
 *  - the caller owns all memory: weights, inputs, outputs and one workspace
 *    blob sized by gr4ad_workspace_bytes();
 *  - no global mutable state: calls are reentrant with one stream per thread;
 *    the last error message is thread-local;
 *  - functions return gr4ad_status; argument errors carry the reference's
 *    ValueError messages (beam.py:125-132,155-156) via gr4ad_last_error().
 */
#ifndef GR4AD_H_
#define GR4AD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GR4AD_ABI_VERSION 2
#define GR4AD_MAX_LEVELS 8
#define GR4AD_MAX_LAYERS 32
#define GR4AD_MAX_BEAM 8192 /* per-request selection width handled on chip */

typedef enum {
  GR4AD_OK = 0,
  GR4AD_ERR_VALUE = 1,     /* maps to ValueError (reference argument errors) */
  GR4AD_ERR_UNSUPPORTED = 2,
  GR4AD_ERR_WORKSPACE = 3, /* workspace too small */
  GR4AD_ERR_CUDA = 4,      /* maps to RuntimeError */
  GR4AD_ERR_RANGE = 5      /* an operand left the fp16 split range of the tensor-core
                              paths: decode with a CUDA-core path (the Python API does
                              so automatically for decode_path auto) */
} gr4ad_status;

/* DecoderConfig (pkg/src/adrec/model/decoder.py:32-51). */
typedef struct {
  int feat_dim;
  int d;
  int d_ff;
  int n_layers;
  int trunk_depth;
  int n_levels;
  int n_value_buckets;
  int vocab[GR4AD_MAX_LEVELS];
} gr4ad_dims;

/* Per-layer parameters of decoder_layer (layers.py:66-119), reference layout
 * (row-vector convention x @ W, W stored (in, out) row-major). */
typedef struct {
  const float *ln1_g, *ln1_b;
  const float *cross_Wq; /* (d, d) */
  const float *cross_Wo; /* (d, d) */
  const float *ln2_g, *ln2_b;
  const float *self_Wqkv; /* (d, 3d) = [Wq | Wk | Wv] */
  const float *self_Wo;   /* (d, d) */
  const float *ln3_g, *ln3_b;
  const float *ffn_W1, *ffn_b1; /* (d, d_ff), (d_ff) */
  const float *ffn_W2, *ffn_b2; /* (d_ff, d), (d) */
} gr4ad_layer;

/* DecoderModel.params (decoder.py:71-107), resident per snapshot version. */
typedef struct {
  const float *ctx_W, *ctx_b; /* (F, d), (d) */
  const float *pos;           /* (T+1, d) */
  const float *bos;           /* (d) */
  const float *emb[GR4AD_MAX_LEVELS];  /* (V_t, d) */
  const float *head[GR4AD_MAX_LEVELS]; /* (d, V_t) */
  const float *head_value;             /* (d, n_value_buckets) */
  const float *fuse_Wg;                /* (d, d) */
  const float *fuse_Wf;                /* (2d, d) */
  const float *cross_kv_W; /* (d, 2*L*d) = [Wk_0 | Wv_0 | Wk_1 | Wv_1 | ...] */
  gr4ad_layer layer[GR4AD_MAX_LAYERS];
} gr4ad_weights;

/* One batch of independent requests (one beam_search call each). */
typedef struct {
  int n_requests;
  const int *ctx_len;   /* host [n_requests]: S_b (> 0) */
  const int *widths;    /* host [n_requests * n_levels]: schedule widths */
  int trunk_depth;      /* -1: model default; 0 <= K < n_layers otherwise */
  int value_rerank;     /* beam.py:214-217, 258-288 */
  const float *value_reps; /* device [n_value_buckets]: EcpmBuckets.representatives,
                              padded with its last entry (beam.py:281-285) */
  /* optional valid-SID prefix masking (no reference
   * counterpart): per level t, sorted unique mixed-radix keys of the valid
   * (t+1)-token prefixes.  NULL entries disable masking at that level. */
  const int64_t *valid_prefix[GR4AD_MAX_LEVELS];
  const int *valid_prefix_count; /* host [n_levels] */
  /* 0: auto -- the fused per-request kernel when a request's working set
   * fits on chip (d in {16,32}, d_ff in {d,2d}, S <= 32d, widths <= 2048,
   * no masking), else the layered batch path, with tcgen05 3xFP16 GEMMs
   * when d >= 64 (d a multiple of 8; d_ff, F, V multiples of 4); 1: layered
   * with CUDA-core GEMMs; 2: fused (its warp-level tensor-core variant --
   * mma.sync 3xFP16 -- when d = 16, else CUDA cores); 3: layered with
   * tcgen05 GEMMs; 4: fused on CUDA cores only; 5: as 3, but the
   * cross-attention always attends against the projected context X.
   * On the tcgen05 path (3 / auto), a decode given `features` with
   * d % 128 == 0, d <= 1024 and F in {4, 8, 16, 32} attends over the
   * request's F-wide features instead (weight absorption through the linear
   * context projection, decoder.py:134-140: exact algebra);
   * given a projected `context` it attends against X.  Forcing an
   * ineligible path returns GR4AD_ERR_UNSUPPORTED. */
  int decode_path;
  /* 1: the workspace already holds this snapshot's derived weight copies
   * (gr4ad_prepare_weights: fragment-ordered / K-major fp16 hi+lo splits);
   * the decode then skips rebuilding them.  0: rebuilt every call. */
  int weights_prepared;
  /* optional: the snapshot's derived weight copies (factored / absorbed
   * products, fuse tables, K-major fp16 splits, MMA fragments) in a
   * caller-owned device buffer shared by every decode of that snapshot and
   * path (gr4ad_derived_layout sizes it and names its layout;
   * gr4ad_prepare_weights fills it).  NULL: they live at the start of the
   * workspace.  With a buffer, the workspace shrinks by derived bytes and a
   * new batch shape costs no weight preparation. */
  void *derived;
  size_t derived_bytes;
} gr4ad_batch;

/* Results: for request b, count[b] entries in selection order (or value
 * re-rank order): tokens[(b*max_out + j)*n_levels + t], score[b*max_out + j].
 * Scores are the fp32 beam scores widened to double (value re-rank scores are
 * computed in double, as E[bucket value] * exp(cum) underflows fp32). */
typedef struct {
  int max_out;   /* >= max over b of the final (clamped) width */
  int *count;    /* device [n_requests] */
  int *tokens;   /* device [n_requests * max_out * n_levels] */
  double *score; /* device [n_requests * max_out] */
} gr4ad_results;

int gr4ad_abi_version(void);
const char *gr4ad_last_error(void);
const char *gr4ad_status_string(int status);
/* Kernel launches issued by the calling thread since the last call (the
 * bench's gpu_launches evidence; thread-local like the error text). */
long long gr4ad_take_launch_count(void);

/* Live per-kernel-class timing for the bench's roofline: between begin and
 * end every launch made by the calling thread is bracketed by CUDA events on
 * its stream; end() synchronises and returns per-class total ms and launch
 * counts.  Classes: 0 gemm, 1 attention gemm, 2 top-k, 3 softmax,
 * 4 layernorm, 5 self-attention, 6 row log-sum-exp, 7 small, 8 collect,
 * 9 fused small-model decode. */
void gr4ad_profile_begin(void);
int gr4ad_profile_end(double *ms, long long *launches, int n_classes);

/* Workspace bytes and the result-row bound (max_out) for a batch. */
int gr4ad_workspace_bytes(const gr4ad_dims *dims, const gr4ad_batch *batch,
                          size_t *bytes, int *max_out);

/* Full LazyAR beam decode of a batch (beam.py:112-218 + 258-288 per request):
 * context projection (decoder.py:134-140) when `features` is non-NULL,
 * otherwise `context` is the projected X; shared encoder K/V for all layers
 * (beam.py:98-109); trunk (beam.py:159-163); T level steps; optional value
 * re-rank.  features: (sum S_b, F); context: (sum S_b, d), row-concatenated
 * per request.  No host round-trip: every shape is fixed by `batch`. */
int gr4ad_beam_search(const gr4ad_dims *dims, const gr4ad_weights *w,
                      const gr4ad_batch *batch, const float *features,
                      const float *context, gr4ad_results *out, void *workspace,
                      size_t workspace_bytes, void *stream);

/* Split form for CUDA-graph capture: gr4ad_prepare uploads the batch's
 * integer plan (row offsets, capacities, ancestor tables) into the
 * workspace; gr4ad_beam_search_run then issues only kernels (no host
 * copies, no synchronisation) and may be captured and replayed for any
 * inputs of the same batch shape. */
int gr4ad_prepare(const gr4ad_dims *dims, const gr4ad_batch *batch, void *workspace,
                  size_t workspace_bytes, void *stream);
int gr4ad_beam_search_run(const gr4ad_dims *dims, const gr4ad_weights *w,
                          const gr4ad_batch *batch, const float *features,
                          const float *context, gr4ad_results *out, void *workspace,
                          size_t workspace_bytes, void *stream);

/* Build the snapshot-derived weight copies a decode of this batch shape uses
 * (fused path: mma fragments + trunk queries; tensor-core path: K-major fp16
 * hi/lo splits) into batch->derived when set (workspace may then be NULL),
 * else into `workspace`, once per snapshot (the SnapshotStore
 * contract, engine.py:17-36); then set batch->weights_prepared.  Synchronises
 * `stream`; returns GR4AD_ERR_UNSUPPORTED if a weight leaves the fp16 split
 * range. */
int gr4ad_prepare_weights(const gr4ad_dims *dims, const gr4ad_weights *w,
                          const gr4ad_batch *batch, void *workspace, size_t workspace_bytes,
                          void *stream);

/* fp16 split range of the last decode in `workspace` (synchronises `stream`).
 * The tensor-core paths split weights (x 2048) and the context K / V (x 256)
 * into fp16 hi + lo; a value outside the fp16 range after that scale sets a
 * flag in the workspace, reported here as GR4AD_ERR_RANGE (decode with a
 * CUDA-core path instead).  No reference counterpart: the reference
 * computes in float64 (autodiff.py:55). */
int gr4ad_range_status(const gr4ad_dims *dims, const gr4ad_batch *batch, const void *workspace,
                       void *stream);
/* Size and layout signature of the derived weight region of this batch's
 * plan (it depends only on dims, the decode path, the trunk depth and
 * value re-rank -- not on the batch size or widths): decodes whose plans
 * report the same signature share one derived buffer (batch->derived).
 * Replaces the per-call weight re-derivation of the reference's stateless
 * beam_search (beam.py:112-143) with the SnapshotStore contract
 * (engine.py:17-36): derive once per published snapshot. */
int gr4ad_derived_layout(const gr4ad_dims *dims, const gr4ad_batch *batch, size_t *bytes,
                         unsigned long long *signature);
/* Byte offset of that flag (an int, nonzero = out of range) inside the
 * workspace, so a caller can copy it to the host together with the results
 * instead of synchronising in gr4ad_range_status. */
int gr4ad_range_flag_offset(const gr4ad_dims *dims, const gr4ad_batch *batch, size_t *offset);

/* The layered decode split at the reference's own phase boundaries
 * (beam.py:146-218), for callers that interleave their own
 * work between levels.  After gr4ad_prepare (+ gr4ad_prepare_weights):
 *   gr4ad_encode_trunk   context projection (decoder.py:134-140), shared
 *                        encoder K/V (beam.py:98-109, 164-169), trunk pass
 *                        (beam.py:159-163), level-0 beam rows;
 *   gr4ad_level_step(t)  level t = 0..T-1: token gather + fuse
 *                        (beam.py:180-191), head layers (beam.py:243-255),
 *                        codebook projection + log-softmax + score
 *                        accumulation + top-k + alive filter + in-place
 *                        compaction (beam.py:198-210); t = T with
 *                        value_rerank: the re-rank head pass (beam.py:258-288);
 *   gr4ad_collect        the final beams into `out` (beam.py:212-217).
 * The sequence is bit-identical to gr4ad_beam_search_run on the same
 * workspace.  Needs the layered path (decode_path 1 or 3, or auto when it
 * picks the layered path); GR4AD_ERR_UNSUPPORTED for the fused kernel. */
int gr4ad_encode_trunk(const gr4ad_dims *dims, const gr4ad_weights *w, const gr4ad_batch *batch,
                       const float *features, const float *context, void *workspace,
                       size_t workspace_bytes, void *stream);
int gr4ad_level_step(const gr4ad_dims *dims, const gr4ad_weights *w, const gr4ad_batch *batch,
                     int level, void *workspace, size_t workspace_bytes, void *stream);
int gr4ad_collect(const gr4ad_dims *dims, const gr4ad_batch *batch, gr4ad_results *out,
                  void *workspace, size_t workspace_bytes, void *stream);

/* On-device SID -> item resolution (reference engine.py:114-118,
 * quantizer/index.py:33-35): for every result entry
 * (b, j < count[b]) of `res`, the SID's mixed-radix key
 * sum_t tok_t * prod_{u>t} V_u is looked up in `sid_keys` (device, sorted
 * ascending, n_keys entries -- the index's SIDs); out_item[b*max_out + j]
 * = item_ids[pos] (device) when found, else -1 (unindexed: the engine drops
 * it, as the reference's post-filter does).  Entries past count[b] get -1. */
int gr4ad_resolve_items(const int64_t *sid_keys, const int *item_ids, int n_keys,
                        const gr4ad_dims *dims, const gr4ad_results *res, int n_requests,
                        int *out_item, void *stream);

/* Context projection X = F W_c + b_c (decoder.py:134-140): (rows, F) -> (rows, d). */
int gr4ad_context_process(const gr4ad_dims *dims, const gr4ad_weights *w,
                          const float *features, int rows, float *x, void *stream);

/* Shared encoder K/V for layers lo..hi-1 (beam.py:98-109):
 * kv[(r, 2*(i-lo)+{0,1})] row-major (rows, 2*(hi-lo)*d). */
int gr4ad_encoder_kv(const gr4ad_dims *dims, const gr4ad_weights *w,
                     const float *x, int rows, int lo, int hi, float *kv,
                     void *stream);

/* Teacher-forced scoring of fixed token sequences (lazy_forward +
 * sequence_log_prob, decoder.py:162-219): sequence s
 * belongs to request req[s] (HOST array) of `batch` (whose widths are
 * ignored) and has tokens[s*T .. s*T+T-1] (device).  Writes the per-level
 * log-probabilities logp[s*T + t]; when non-NULL also the head logits
 * head_logits[s*sum(V) + offset_t + v] and, with batch->value_rerank set
 * (value step at position T), the value-bucket logits
 * value_logits[s*n_value_buckets + j].  Layered kernels (tcgen05 for
 * d >= 64), trunk once per request, causal head layers per sequence. */
int gr4ad_score_sequences(const gr4ad_dims *dims, const gr4ad_weights *w,
                          const gr4ad_batch *batch, const float *features,
                          const float *context, int n_seq, const int *req,
                          const int *tokens, float *logp, float *value_logits,
                          float *head_logits, void *workspace, size_t workspace_bytes,
                          void *stream);
int gr4ad_score_workspace_bytes(const gr4ad_dims *dims, const gr4ad_batch *batch,
                                int n_seq, size_t *bytes);

/* C = A . BT^T in fp32 (A: (M, K), BT: (N, K), row-major with the given
 * leading dimensions) -- the GEMM the decode uses internally, exposed for
 * numerics tests.  backend 0: CUDA-core fp32; 1: tcgen05 3xFP16 (fp32
 * accumulation in TMEM; needs 16-B aligned rows). */
int gr4ad_gemm(const float *A, long long lda, const float *BT, long long ldb, float *C,
               long long ldc, int M, int N, int K, int backend, void *stream);

/* C = alpha (a_hi + a_lo) . (b_hi + b_lo)^T with both operands already split
 * into fp16 hi / lo (K-major rows, lda / ldb and K multiples of 8) -- the
 * TMA-only tcgen05 path the decode's head-layer and encoder K/V products take
 * (CTA pairs, 256 x 256 tiles, when N >= 256), exposed for numerics tests. */
int gr4ad_gemm_presplit(const void *a_hi, const void *a_lo, long long lda, const void *b_hi,
                        const void *b_lo, long long ldb, float *C, long long ldc, int M, int N,
                        int K, float alpha, void *stream);

/* Batched pre-cut selection (beam.py:50-89 topk_precut/_precut_arrays and
 * beam.py:37-47 topk_global -- identical results): for problem p,
 * candidates prev_scores[p*b + i] + logprobs[(p*b + i)*v + j], top k under
 * (-score, beam, token).  Writes beam/token/score[p*k + j], count[p]. */
int gr4ad_topk_precut(const float *prev_scores, const float *logprobs,
                      int n_problems, int b, int v, int k, int *out_beam,
                      int *out_token, float *out_score, int *out_count,
                      void *workspace, size_t workspace_bytes, void *stream);
size_t gr4ad_topk_workspace_bytes(int n_problems, int b, int v);

/* The same selection on float64 inputs, bit-exact against the reference
 * (beam.py:37-89): candidate score = prev_scores[p*b + i] + logprobs[...]
 * computed in IEEE double exactly as numpy's broadcast add, ranked by
 * (-score, beam, token) with no rounding of the keys; -inf candidates rank
 * last (the caller's alive filter drops them, beam.py:202-203).  Scores are
 * returned in double.  One CTA per problem: 64-bit radix select, ordered tie
 * collection, in-shared-memory sort of the k winners (k <= GR4AD_MAX_BEAM). */
int gr4ad_topk_precut_f64(const double *prev_scores, const double *logprobs, int n_problems,
                          int b, int v, int k, int *out_beam, int *out_token, double *out_score,
                          int *out_count, void *stream);

/* Fused codebook projection + log-softmax + score accumulation + top-k for
 * one level (beam.py:198-201): states (n_problems*b, d) @ head (d, v),
 * log-softmax per row, + prev_scores, then top-k as gr4ad_topk_precut. */
int gr4ad_project_topk(const float *states, const float *head, int d,
                       const float *prev_scores, int n_problems, int b, int v,
                       int k, int *out_beam, int *out_token, float *out_score,
                       int *out_count, void *workspace, size_t workspace_bytes,
                       void *stream);
size_t gr4ad_project_topk_workspace_bytes(int n_problems, int b, int v);

#ifdef __cplusplus
}
#endif
#endif /* GR4AD_H_ */
