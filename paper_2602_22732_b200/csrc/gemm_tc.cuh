// tcgen05 3xFP16 GEMM (see gemm_tc.cu).
#pragma once
#include <cuda_fp16.h>

#include "gemm.cuh"

namespace gr {

// Power-of-two scales of the pre-split fp16 B operands (gemm_tc.cu): weights
// (|w| < 32) and the encoder's K / V^T (|x| < 256) keep their fp16 lo parts in
// the normal range; the GEMM's alpha carries the inverse.
constexpr float kWeightScale = 2048.f;
constexpr float kKvScale = 256.f;

struct TcArgs : GemmArgs {
  // optional: B pre-split, s.B = b_hi + b_lo (fp16, K-major, ld = ldb);
  // otherwise B (fp32) is split on chip, unscaled
  const __half *b_hi, *b_lo;
  // optional: A pre-split likewise (a_hi / a_lo, ld = lda), scale folded into alpha
  const __half *a_hi, *a_lo;
  // EPI_*_SPLIT: fp16 hi / lo destinations (ld = ldc) of c_scale * C (0: 1);
  // a nonzero c_scale also range-checks the scaled values into range_flag
  __half *c_hi, *c_lo;
  float c_scale;
  // EPI_KV_SPLIT: the K part of layer i -> k_hi / k_lo [row][k_ld] at column
  // i d, the V part -> vt_hi / vt_lo [i d + c][vt_ld], all kv_scale * x
  __half *k_hi, *k_lo, *vt_hi, *vt_lo;
  long long k_ld, vt_ld;
  float kv_scale;
  int kv_d;
  int *range_flag;  // EPI_KV_SPLIT / c_scale: set when a scaled value leaves the fp16 range
  // EPI_STORE_LSE: lse_part[row * lse_ld + col / 128] = (max, sum exp(x - max),
  // max of the first 64 columns, max of the last 64) over the row's columns
  // [128 j, 128 j + 128) (merged by lse_merge; the half maxima are the
  // selection's window proxies)
  float4 *lse_part;
  int lse_ld;
  // few rows per request (trunk rows, level 0): GM_PLAIN products run on
  // 128 x 128 single-CTA tiles (gemm_tc) -- set by the rows' role
  int few_rows;
  long long *dbg;  // debug timeline: [CTA][8] %globaltimer stamps (gr4ad_debug_tc_timeline)
};

// A is (a_rows, a_cols) with ld lda, B is (b_rows, b_cols) K-major with ld ldb;
// the tensor maps cover these full extents (out-of-range reads return 0).
int gemm_tc(const TcArgs &a, long long a_rows, long long a_cols, long long b_rows,
            long long b_cols, int epi, cudaStream_t st);
bool tc_eligible(long long lda, long long ldb, int K, const void *A, const void *B);
// GM_QK_T / GM_PV_T attention products (EPI_STORE_T): A (a_hi/a_lo fp16, or
// A fp32) is (a_rows, a_cols), B fp32 (b_rows, b_cols); tile N sized to the
// beam rows per request (32 / 64 / 128)
int gemm_tc_swapped(const TcArgs &a, long long a_rows, long long a_cols, long long b_rows,
                    long long b_cols, cudaStream_t st, int epi = EPI_STORE_T);

// dst (cols x rows) = src (rows x cols)^T, both row-major with the given lds
int transpose(const float *src, long long lds, float *dst, long long ldd, int rows, int cols,
              cudaStream_t st);
// as transpose, writing the fp16 split of scale * src^T: dst_hi + dst_lo
int transpose_split16(const float *src, long long lds, __half *dst_hi, __half *dst_lo,
                      long long ldd, int rows, int cols, float scale, int *flag, cudaStream_t st);

}  // namespace gr
