// Row-wise and selection kernels of the beam step (declarations).
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace gr {

// LN over rows (layers.py:38-43): y = (x - mean) * (var + 1e-5)^-1/2 * g + b
// LayerNorm with the output as fp16 hi / lo (d % 128 == 0, d <= 1024)
// (y32: optionally also the fp32 output, ld ld32)
int ln_rows_split(const float *x, long long ldx, __half *y_hi, __half *y_lo, long long ldy,
                  const float *g, const float *b, int rows, int d, cudaStream_t st,
                  float *y32 = nullptr, long long ld32 = 0);
int ln_rows(const float *x, long long ldx, float *y, long long ldy, const float *g,
            const float *b, int rows, int d, cudaStream_t st);

// in-place softmax (autodiff.py:362-368) of row r over its first len[req(r)]
// columns; row_req maps rows to groups.
// softmax writing P as fp16 hi / lo (ld halves per row, zero past each S)
int softmax_rows_split(const float *s, long long ld, __half *p_hi, __half *p_lo, int rows,
                       const int *row_req, const int *len, cudaStream_t st);
int softmax_rows(float *s, long long ld, int rows, const int *row_req,
                 const int *len, cudaStream_t st);

// self-attention of each row over its ancestor chain (layers.py:101-113 with
// the history gathered by beam.py:247-248): positions anc[g*stride + tau],
// tau < npos (npos_row[r] or npos_uniform); per history row (ld ld3) q at
// column 0, k at column d, v at column v_off (default 2d).  The factored
// tensor-core path stores [q W_k^T | n] (n = the LayerNorm'd row) and passes
// v_off = d: k = v = n, the projections folded into its weights.
int self_attn(const float *qkv, long long ld3, int d, const int *anc, int anc_stride,
              int hist_row0, int rows, int npos_uniform, const int *npos_row,
              float *out, long long ldo, cudaStream_t st, __half *out_hi = nullptr,
              __half *out_lo = nullptr, int v_off = -1, bool hist_split = false);

// dst = fp16 hi / lo split of scale * src (row-major, rows x cols)
int split16(const float *src, long long lds, __half *dst_hi, __half *dst_lo, long long ldd,
            int rows, int cols, float scale, int *flag, cudaStream_t st);
// latent (weight-absorbed) cross-attention (latent.cu): F = feature width
bool latent_supported(int d, int F);
int latent_attn(const float *q, const float *feats, int F, const int *g_row_off, const int *g_rows,
                const int *g_ctx_off, const int *g_ctx_len, int n_groups, int max_group_rows,
                float scale, float *z, int *flag, cudaStream_t st);
// the latent cross-attention block without LN1's output or q_lat in HBM:
// z = softmax(LN1(h) A F^T scale) F in one kernel (LN1 folded: A'^T =
// kWeightScale diag(g1) A as fp16 hi / lo, s = 1^T A', c = b1 A; features
// pre-split by latent_feat_split), then h += alpha z B + c and LN2 of the new
// rows (n split, hn fp32) in a second
int latent_cross_ln(const float *h, int d, const __half *aq_hi, const __half *aq_lo,
                    const float *s1, const float *c1, const __half *fs_hi, const __half *fs_lo,
                    int F, const int *g_row_off, const int *g_rows, const int *g_ctx_off,
                    const int *g_ctx_len, int n_groups, int max_group_rows, float scale, float *z,
                    int *flag, cudaStream_t st);
int latent_out_ln(const float *z, int F, const __half *bo_hi, const __half *bo_lo, float alpha,
                  const float *c, float *hs, int d, const float *g2, const float *b2,
                  __half *n_hi, __half *n_lo, long long ld_n, float *hn, long long ld_hn,
                  int rows, int *flag, cudaStream_t st);
int latent_fold(const float *at, const float *g1, const float *b1, int d, int F, float *ag,
                float *sv, float *cv, cudaStream_t st);
int latent_feat_kst(int F);  // halves per pre-split feature row
int latent_feat_split(const float *fin, long long rows_used, long long rows_alloc, int F,
                      __half *hi, __half *lo, int *flag, cudaStream_t st);
// C = A . op(B) in double, rounded to fp32 (snapshot weight products)
int weight_product(const float *A, long long lda, const float *B, long long ldb, bool trans_b,
                   float *C, long long ldc, int M, int N, int K, cudaStream_t st);

// level input (beam.py:180-191): s = bos (t==0) or emb_{t-1}[tok]; K>0 writes
// s into U[:, d:2d]; K==0 writes H = s + pos[t].
int level_input(int t, int rows, int d, const float *bos, const float *emb_prev,
                const int *tok, const float *pos_t, float *U, float *H,
                cudaStream_t st, __half *Uh = nullptr, __half *Ul = nullptr);

// fuse inputs from the per-snapshot token tables (tab: [s W_g | s W_f[d:2d]],
// 2 x n_tok x d): H = tab_f[tok], (Uh, Ul) = split of m[req] * tab_g[tok]
int fuse_gather(int t, int rows, int d, const int *tok, const float *tab, int n_tok,
                const float *m, long long m_ld, const int *row_req, float *H, __half *Uh,
                __half *Ul, cudaStream_t st);

// per-row (max, log sum exp(x - max)) (beam.py:92-95)
int lse_merge(const float4 *part, int n_part, int rows, float2 *info, cudaStream_t st);
int row_lse(const float *logits, long long ld, int rows, int V, float2 *info,
            cudaStream_t st);

// valid-SID prefix mask: logits[r][v] = -inf unless prefix[r]*V + v is a
// valid key (sorted array). SURVEY §8f row 2 (no reference counterpart).
// CSR row pointers (over the t-prefix key) of sorted valid (t+1)-prefix keys
int csr_rows(const long long *keys, int n, int V, long long n_prefix, int *rp,
             cudaStream_t st);
int mask_rows(float *logits, long long ld, int rows, int V, const long long *prefix,
              const long long *valid, int n_valid, cudaStream_t st);

struct SelectArgs {
  // candidates of level t
  const float *logits;
  long long ld;
  int V;
  int level;
  const float2 *rowinfo;  // per level row
  // optional (no masking): per level row, proxy_ld (max, sum, p1, p2)
  // partials of the logits GEMM epilogue; p1 / p2 (64-column maxima) are
  // window proxies
  const float4 *proxies;
  int proxy_ld;
  const float *cum;       // per history row
  const int *row_off;     // [B] row offset (within level t)
  const int *live;        // [B] live rows of request (level t)
  const int *eff;         // [B] effective width
  int hist_off;           // history row of level row 0
  // outputs: level t+1
  const int *out_row_off;  // [B]
  const int *out_cap;      // [B]
  int *out_live;           // [B]
  int out_hist_off;
  int *tok;                // per history row
  float *cum_out;          // per history row (== cum buffer)
  long long *prefix;       // per history row (mixed-radix prefix key)
  int *anc;                // per history row * anc_stride
  int anc_stride;
  // standalone (gr4ad_topk_precut) outputs, used when tok == nullptr
  int *o_beam, *o_token;
  float *o_score;
  int *o_count;
  int o_k;
  // scratch: per-request candidate buffer for large candidate sets
  unsigned long long *scratch;
  long long scratch_per_req;
};

// u_rows/u_k: uniform rows and k per request when row_off/live/eff are NULL;
// max_cand: max candidates of one request (decides the shared-memory key cache)
int topk_select(const SelectArgs &a, int n_requests, int u_rows, int u_k,
                long long max_cand, cudaStream_t st);

// copy request blocks of `width`-wide rows from caller offsets to 32-row
// aligned offsets, zero-filling the padding rows
int pad_rows(const float *src, const int *in_off, const int *out_off, const int *len, int B,
             int width, float *dst, cudaStream_t st);

struct SeqInputArgs {
  int rows, d, n_pos, T;
  const int *tokens;  // [n_seq][T]
  const float *bos, *pos;
  const float *emb[GR4AD_MAX_LEVELS];
  float *U, *H;
};
int seq_input(const SeqInputArgs &a, cudaStream_t st);
int gather_logp(const float *logits, long long ld, int rows, const float2 *info,
                const int *tokens, int T, int t, float *logp, cudaStream_t st);

// level-0 rows: live=1, cum=0, prefix=0, anc[g][0]=g
int init_level0(int n_requests, int *live0, float *cum, long long *prefix, int *anc,
                int anc_stride, int *tok, cudaStream_t st);

// results (beam.py:212-213) and value re-rank (beam.py:258-288)
int collect_results(int n_requests, int T, const int *row_off_T, const int *live_T,
                    int hist_off_T, const int *tok, const int *anc, int anc_stride,
                    const float *cum, const float *vlogits, int nb,
                    const float *reps, int max_out, int *count, int *tokens,
                    double *score, cudaStream_t st);

}  // namespace gr
