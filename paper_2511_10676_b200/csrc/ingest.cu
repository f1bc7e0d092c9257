// ingest.cu — K10: MOEPA1 trace records -> device training / evaluation arrays.
//
// The reference reads a trace with numpy and re-checks every record invariant
// on the host (pkg/src/moepredict/synthgen.py:219-253 read_trace, :123-145
// TraceFile.validate). Here the raw little-endian records
//     d x f32 activation | E x f32 scores | k x u32 top-k indices
// arrive in HBM (streamed from pinned host memory by the caller) and one warp
// per record de-interleaves them into the device layout (activations as fp32
// or bf16, scores fp32, top-k int32) while evaluating the same invariants:
//   [0] non-finite activation          [1] score outside [0, 1]
//   [2] |sum(scores) - 1| > 1e-5 (fp64) [3] top-k index >= E
//   [4] top-k row not strictly increasing (k > 1)
//   [5] stored top-k != top_k(scores, k) (stable, lower index on ties)
// Failures are counted per category in status[6] (atomics only on failure);
// the host raises the reference's exception for the first category, in the
// reference's check order, that has a failing record.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "../../include/moep_b200.h"

namespace moep {
namespace k10 {

constexpr int WARPS = 8;

__device__ __forceinline__ bool key_gt(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

template <bool BF16>
__global__ void __launch_bounds__(WARPS * 32)
ingest_kernel(const uint32_t* __restrict__ rec, int64_t n, int d, int E, int k, void* __restrict__ acts,
              float* __restrict__ scores, int32_t* __restrict__ topk, int64_t row0,
              unsigned long long* __restrict__ status) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t words = static_cast<int64_t>(d) + E + k;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * WARPS + warp; r < n; r += static_cast<int64_t>(gridDim.x) * WARPS) {
    const uint32_t* w = rec + r * words;
    const int64_t orow = row0 + r;
    // activations: finite check + copy / convert
    bool bad_act = false;
    for (int j = lane; j < d; j += 32) {
      const float v = __uint_as_float(__ldcs(w + j));
      bad_act |= !isfinite(v);
      if (BF16) reinterpret_cast<__nv_bfloat16*>(acts)[orow * d + j] = __float2bfloat16_rn(v);
      else reinterpret_cast<float*>(acts)[orow * d + j] = v;
    }
    // scores: range, fp64 sum; kept in registers for the top-k check (E <= 32 * 32)
    bool bad_range = false;
    double sum = 0.0;
    for (int e = lane; e < E; e += 32) {
      const float s = __uint_as_float(__ldcs(w + d + e));
      bad_range |= (s < 0.f) || (s > 1.f);
      sum += static_cast<double>(s);
      scores[orow * E + e] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    // stored top-k: range, strictly increasing, rank of each stored index < k
    bool bad_idx = false, bad_order = false, bad_set = false;
    for (int j = lane; j < k; j += 32) {
      const uint32_t t = __ldcs(w + d + E + j);
      topk[orow * k + j] = static_cast<int32_t>(t);
      bad_idx |= t >= static_cast<uint32_t>(E);
      if (j + 1 < k) bad_order |= !(t < __ldcs(w + d + E + j + 1));
    }
    const bool any_idx = __any_sync(0xffffffffu, bad_idx);
    if (!any_idx) {
      // set check: every stored index must have stable descending rank < k
      // (with k distinct in-range indices this is exactly set equality)
      for (int j = 0; j < k; ++j) {
        const int t = static_cast<int>(w[d + E + j]);
        const float st = __uint_as_float(w[d + t]);
        int above = 0;
        for (int e = lane; e < E; e += 32) above += key_gt(__uint_as_float(w[d + e]), e, st, t) ? 1 : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
        bad_set |= above >= k;
      }
    }
    const bool f0 = __any_sync(0xffffffffu, bad_act);
    const bool f1 = __any_sync(0xffffffffu, bad_range);
    const bool f4 = __any_sync(0xffffffffu, bad_order);
    if (lane == 0) {
      if (f0) atomicAdd(&status[0], 1ull);
      if (f1) atomicAdd(&status[1], 1ull);
      if (fabs(sum - 1.0) > 1e-5) atomicAdd(&status[2], 1ull);
      if (any_idx) atomicAdd(&status[3], 1ull);
      if (k > 1 && f4) atomicAdd(&status[4], 1ull);
      if (bad_set || (k > 1 && f4)) atomicAdd(&status[5], 1ull);
    }
  }
}

}  // namespace k10
}  // namespace moep

extern "C" int moep_trace_ingest(const uint32_t* records, int64_t n, int32_t d, int32_t n_experts, int32_t k,
                                 int32_t act_dtype, void* acts, float* scores, int32_t* topk, int64_t row0,
                                 unsigned long long* status, void* stream) {
  using namespace moep::k10;
  if (n < 0 || d < 1 || n_experts < 1 || k < 1 || k > n_experts) return MOEP_ESHAPE;
  if (!records || !acts || !scores || !topk || !status) return MOEP_EARG;
  if (n == 0) return MOEP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (n + WARPS - 1) / WARPS;
  const int grid = static_cast<int>(blocks < 148 * 16 ? blocks : 148 * 16);
  if (act_dtype == MOEP_BF16)
    ingest_kernel<true><<<grid, WARPS * 32, 0, st>>>(records, n, d, n_experts, k, acts, scores, topk, row0, status);
  else if (act_dtype == MOEP_F32)
    ingest_kernel<false><<<grid, WARPS * 32, 0, st>>>(records, n, d, n_experts, k, acts, scores, topk, row0, status);
  else
    return MOEP_EARG;
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
