// On-device SID -> item resolution (reference
// engine.py:114-118 + quantizer/index.py:33-35): every decoded SID is mapped
// to its mixed-radix key and looked up in the index's sorted key table, so
// unindexed SIDs are filtered and indexed ones carry their item slot without
// a per-SID host dictionary lookup.

#include "common.cuh"

namespace gr {
namespace {

struct Vocab {
  int v[GR4AD_MAX_LEVELS];
};

__global__ void resolve_items_kernel(const long long *__restrict__ keys,
                                     const int *__restrict__ ids, int n_keys,
                                     const int *__restrict__ count,
                                     const int *__restrict__ tokens, int B, int max_out, int T,
                                     Vocab vocab, int *__restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)B * max_out) return;
  const int b = (int)(i / max_out), j = (int)(i % max_out);
  if (j >= count[b]) {
    out[i] = -1;
    return;
  }
  long long key = 0;
  for (int t = 0; t < T; ++t) key = key * vocab.v[t] + tokens[i * T + t];
  int lo = 0, hi = n_keys;  // first index with keys[idx] >= key
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  out[i] = (lo < n_keys && keys[lo] == key) ? ids[lo] : -1;
}

}  // namespace
}  // namespace gr

using namespace gr;

extern "C" int gr4ad_resolve_items(const int64_t *sid_keys, const int *item_ids, int n_keys,
                                   const gr4ad_dims *dims, const gr4ad_results *res,
                                   int n_requests, int *out_item, void *stream) {
  if (!dims || !res || n_requests < 0 || n_keys < 0)
    return set_err(GR4AD_ERR_VALUE, "bad resolve arguments");
  if (dims->n_levels < 1 || dims->n_levels > GR4AD_MAX_LEVELS)
    return set_err(GR4AD_ERR_VALUE, "n_levels %d", dims->n_levels);
  const long long n = (long long)n_requests * res->max_out;
  if (n == 0) return GR4AD_OK;
  Vocab v{};
  for (int t = 0; t < dims->n_levels; ++t) v.v[t] = dims->vocab[t];
  cudaStream_t st = (cudaStream_t)stream;
  GR_LAUNCH(KC_COLLECT, st,
            resolve_items_kernel<<<ceil_div(n, 256), 256, 0, st>>>(
                reinterpret_cast<const long long *>(sid_keys), item_ids, n_keys, res->count,
                res->tokens, n_requests, res->max_out, dims->n_levels, v, out_item));
  return GR4AD_OK;
}
