// tcgen05 3xTF32 GEMM (see gemm_tc.cu).
#pragma once
#include "gemm.cuh"

namespace gr {

struct TcArgs : GemmArgs {
  const float *b_lo;  // optional: B pre-split, B holds tf32 hi parts and b_lo the rests
  float *vt;         // EPI_KV_SPLIT: V^T destination (L*d rows, vt_ld columns)
  float *c_lo, *vt_lo;  // EPI_KV_SPLIT: when set, C / V^T get tf32 hi parts, these the rests
  long long vt_ld;
  int kv_d;
};

// A is (a_rows, a_cols) with ld lda, B is (b_rows, b_cols) K-major with ld ldb;
// the tensor maps cover these full extents (out-of-range reads return 0).
int gemm_tc(const TcArgs &a, long long a_rows, long long a_cols, long long b_rows,
            long long b_cols, int epi, cudaStream_t st);
bool tc_eligible(long long lda, long long ldb, int K, const void *A, const void *B);

// dst (cols x rows) = src (rows x cols)^T, both row-major with the given lds
int transpose(const float *src, long long lds, float *dst, long long ldd, int rows, int cols,
              cudaStream_t st);
// as transpose, writing the tf32 split of every element: dst_hi + dst_lo == src^T exactly
int transpose_split(const float *src, long long lds, float *dst_hi, float *dst_lo, long long ldd,
                    int rows, int cols, cudaStream_t st);

}  // namespace gr
