// Shared device helpers for libgr4ad (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include <mutex>
#include <unordered_map>

#include "gr4ad.h"

namespace gr {

// fp16 operand splits: flag values a saturating conversion would clip
// (|x| > 65504 after the power-of-two scale, or NaN)
__device__ __forceinline__ void range_check(float scaled, int *flag) {
  if (flag && !(fabsf(scaled) <= 65504.f)) atomicOr(flag, 1);
}

// thread-local error text (the C side keeps no other state)
int set_err(int code, const char *fmt, ...);

#define GR_TRY(expr)                                                          \
  do {                                                                        \
    int _s = (expr);                                                          \
    if (_s != GR4AD_OK) return _s;                                            \
  } while (0)

#define GR_CUDA(expr)                                                         \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess)                                                    \
      return ::gr::set_err(GR4AD_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, \
                           #expr, cudaGetErrorString(_e));                    \
  } while (0)

// Kernel classes for the live per-class timing hooks (gr4ad_profile_*).
enum KernelClass {
  KC_GEMM = 0,       // projections, FFN, codebook logits, encoder K/V
  KC_ATTN_GEMM = 1,  // grouped cross-attention Q.K^T / P.V over the shared KV
  KC_TOPK = 2,       // exact per-request top-k + compaction
  KC_SOFTMAX = 3,
  KC_LAYERNORM = 4,
  KC_SELF_ATTN = 5,
  KC_ROW_LSE = 6,
  KC_SMALL = 7,      // inputs, tiling, init, masks
  KC_COLLECT = 8,
  KC_FUSED = 9,      // fused small-model per-request decode
  KC_COUNT = 10
};

// Launch bookkeeping (thread-local, like the error text): a launch counter
// and, when enabled, a CUDA event pair recorded on the launching stream
// around every launch.
void count_launch();
void prof_begin(int cls, cudaStream_t st);
void prof_tag(const char *fmt, ...);  // label of the next launch (profiling only)
void prof_end(int cls, cudaStream_t st);

#define GR_LAUNCH(cls, st, ...)          \
  do {                                   \
    ::gr::prof_begin((cls), (st));       \
    __VA_ARGS__;                         \
    ::gr::prof_end((cls), (st));         \
    ::gr::count_launch();                \
    GR_CUDA(cudaGetLastError());         \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size): the attribute persists, and setting it before every launch costs
// host time on the eager (non-graph) launch path
inline cudaError_t set_smem_attr(const void *kernel, int bytes) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, int> done;  // (kernel ^ device) -> bytes
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long key = reinterpret_cast<unsigned long long>(kernel) ^
                                 ((unsigned long long)dev << 56);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
  }
  const cudaError_t e =
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    int &v = done[key];
    if (v < bytes) v = bytes;
  }
  return e;
}

// order-preserving float <-> uint32 (larger float -> larger key)
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// tanh-GELU exactly as autodiff.py:301-306 (0.5*a*(1+tanh(c*(a+0.044715 a^3))))
__device__ __forceinline__ float gelu_tanh(float a) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * a * (1.0f + tanhf((a + 0.044715f * a * a * a) * c));
}

// the same via 0.5 a (1 + tanh z) == a / (1 + exp(-2z)) with the hardware
// exp2 and divide (relative error ~2e-7; exp overflow -> 0 for a << 0)
__device__ __forceinline__ float gelu_tanh_fast(float a) {
  const float c = 0.7978845608028654f;
  return __fdividef(a, 1.0f + __expf(-2.0f * c * (a + 0.044715f * a * a * a)));
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace gr
