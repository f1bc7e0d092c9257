// prefetch.cu — expert prefetch planning (K8) and an SM-driven host->device
// expert gather (K9).
//
// The reference models prefetch analytically (pipesim.py:185-325: per-expert
// bytes, load lanes, prefetch window); the paper's deployment loads the
// predicted experts from pinned memory with non-blocking copies
// (PAPER.md:370). Here:
//   K8 moep_prefetch_plan  union of the predicted expert ids of a batch (the
//        over-provisioned m-sets), minus experts already resident in the
//        device cache -> ascending list of experts to load and a slot for each.
//        One CTA, shared-memory bitmap, ballot compaction (no global atomics).
//   K9 moep_gather_experts copies the listed experts from host memory mapped
//        into the device address space (cudaHostAlloc Mapped) into their cache
//        slots with 16-byte loads — a copy path driven by the GPU itself, with
//        no host round trip between prediction and load.
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/moep_b200.h"

namespace moep {
namespace pf {

__global__ void __launch_bounds__(1024)
plan_kernel(const int32_t* __restrict__ ids, int64_t n_ids, int32_t E, const int32_t* __restrict__ slot_of,
            const int32_t* __restrict__ free_slots, int32_t n_free, const int32_t* __restrict__ free_cursor,
            uint8_t* __restrict__ mask_out, int32_t* __restrict__ need_list, int32_t* __restrict__ need_slot,
            int32_t* __restrict__ need_count) {
  // free slots start at the device cursor (moep_prefetch_commit advances it)
  const int32_t cur = free_cursor ? *free_cursor : 0;
  free_slots += cur;
  n_free -= cur;
  extern __shared__ uint8_t bm[];  // [E] union bitmap (bytes)
  __shared__ int warp_base[32];
  for (int e = threadIdx.x; e < E; e += blockDim.x) bm[e] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n_ids; i += blockDim.x) {
    const int32_t e = ids[i];
    if (e >= 0 && e < E) bm[e] = 1;  // idempotent store: no atomics needed
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int total = 0;
  for (int e0 = 0; e0 < E; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const bool in = e < E && bm[e];
    if (e < E && mask_out) mask_out[e] = in ? 1 : 0;
    const bool need = in && (slot_of == nullptr || slot_of[e] < 0);
    const uint32_t bal = __ballot_sync(0xffffffffu, need);
    if (lane == 0) warp_base[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < nw; ++w) { const int c = warp_base[w]; warp_base[w] = run; run += c; }
      warp_base[31] = run;  // chunk total (nw <= 31 for blockDim <= 992; 1024 handled below)
    }
    __syncthreads();
    const int chunk_total = warp_base[31];
    if (need) {
      const int pos = total + warp_base[warp] + __popc(bal & ((1u << lane) - 1u));
      need_list[pos] = e;
      if (need_slot) need_slot[pos] = pos < n_free ? free_slots[pos] : -1;
    }
    total += chunk_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *need_count = total;
}

// Residency update after a plan (one warp): slot_of[need_list[i]] = need_slot[i]
// for the assigned entries, free-slot cursor += their number. Device-only, so
// plan -> load -> commit needs no host round trip.
__global__ void commit_kernel(const int32_t* __restrict__ need_list, const int32_t* __restrict__ need_slot,
                              const int32_t* __restrict__ need_count, int32_t* __restrict__ slot_of,
                              int32_t* __restrict__ free_cursor) {
  const int count = *need_count;
  int assigned = 0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const int s = need_slot[i];
    if (s >= 0) { slot_of[need_list[i]] = s; ++assigned; }
  }
  for (int o = 16; o > 0; o >>= 1) assigned += __shfl_xor_sync(0xffffffffu, assigned, o);
  if (threadIdx.x == 0) *free_cursor += assigned;
}

// One CTA per (expert, chunk): 16-byte loads from mapped host memory.
__global__ void __launch_bounds__(512)
gather_kernel(const uint4* __restrict__ host_store, int64_t expert_bytes, const int32_t* __restrict__ need_list,
              const int32_t* __restrict__ need_slot, const int32_t* __restrict__ need_count, uint4* __restrict__ cache,
              int32_t chunks_per_expert) {
  const int count = *need_count;
  const int64_t words = expert_bytes / 16;
  const int64_t per_chunk = (words + chunks_per_expert - 1) / chunks_per_expert;
  for (int64_t job = blockIdx.x; job < static_cast<int64_t>(count) * chunks_per_expert; job += gridDim.x) {
    const int idx = static_cast<int>(job / chunks_per_expert);
    const int ch = static_cast<int>(job % chunks_per_expert);
    const int e = need_list[idx], slot = need_slot[idx];
    if (slot < 0) continue;
    const uint4* src = host_store + static_cast<int64_t>(e) * words;
    uint4* dst = cache + static_cast<int64_t>(slot) * words;
    const int64_t w0 = ch * per_chunk;
    const int64_t w1 = (w0 + per_chunk < words) ? w0 + per_chunk : words;
    // 4 loads in flight per thread to cover the PCIe round trip
    int64_t w = w0 + threadIdx.x;
    for (; w + 3 * 512 < w1; w += 4 * 512) {
      const uint4 a = src[w], b = src[w + 512], c = src[w + 1024], d = src[w + 1536];
      dst[w] = a; dst[w + 512] = b; dst[w + 1024] = c; dst[w + 1536] = d;
    }
    for (; w < w1; w += 512) dst[w] = src[w];
  }
}

}  // namespace pf
}  // namespace moep

extern "C" {

int moep_prefetch_plan(const int32_t* ids, int64_t n_ids, int32_t n_experts, const int32_t* slot_of,
                       const int32_t* free_slots, int32_t n_free, const int32_t* free_cursor, uint8_t* mask_out,
                       int32_t* need_list, int32_t* need_slot, int32_t* need_count, void* stream) {
  if (n_ids < 0 || n_experts <= 0 || n_experts > 65536) return MOEP_ESHAPE;
  if (!ids || !need_list || !need_count) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  moep::pf::plan_kernel<<<1, 992, n_experts, st>>>(ids, n_ids, n_experts, slot_of, free_slots, n_free, free_cursor,
                                                  mask_out, need_list, need_slot, need_count);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_prefetch_commit(const int32_t* need_list, const int32_t* need_slot, const int32_t* need_count,
                         int32_t* slot_of, int32_t* free_cursor, void* stream) {
  if (!need_list || !need_slot || !need_count || !slot_of || !free_cursor) return MOEP_EARG;
  moep::pf::commit_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(need_list, need_slot, need_count,
                                                                          slot_of, free_cursor);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_gather_experts(const void* host_mapped_store, int64_t expert_bytes, const int32_t* need_list,
                        const int32_t* need_slot, const int32_t* need_count, void* cache, int32_t n_ctas,
                        void* stream) {
  if (expert_bytes <= 0 || (expert_bytes % 16) != 0) return MOEP_EALIGN;
  if ((reinterpret_cast<uintptr_t>(host_mapped_store) & 15) || (reinterpret_cast<uintptr_t>(cache) & 15))
    return MOEP_EALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int chunks = 64;
  moep::pf::gather_kernel<<<n_ctas > 0 ? n_ctas : 64, 512, 0, st>>>(
      static_cast<const uint4*>(host_mapped_store), expert_bytes, need_list, need_slot, need_count,
      static_cast<uint4*>(cache), chunks);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // extern "C"
