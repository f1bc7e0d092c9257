// k7_eval.cu — K7: exact selection and evaluation counters from given logits,
// the deterministic counter reduce, the input-norm kernel K0, and misc C ABI.
//
// moep_eval_logits restates metrics.evaluate_predictions (metrics.py:138-193):
// the stable predicted rank of each true expert (core.rank_order, core.py:51-54)
// is an exact count of keys ordered before it, computed one warp per token with
// ballots; per-CTA partial counters are written without global atomics and
// summed in a fixed order by moep_counters_reduce.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "common.cuh"

namespace moep {
namespace k7 {

constexpr int NT = 256;

template <typename T>
__global__ void __launch_bounds__(NT)
eval_kernel(const T* __restrict__ z, int64_t n, int E, const int* __restrict__ truth, int k,
            int n_m, const int* __restrict__ m_list_dev, int* partials, int n_counters) {
  extern __shared__ int sh[];  // [8 warps][2E] hist
  __shared__ int scal[8][2 + 2 * MOEP_MAX_BOUNDS];
  __shared__ int mls[MOEP_MAX_BOUNDS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* hist = sh + warp * 2 * E;
  for (int i = lane; i < 2 * E; i += 32) hist[i] = 0;
  if (threadIdx.x < MOEP_MAX_BOUNDS) mls[threadIdx.x] = threadIdx.x < n_m ? m_list_dev[threadIdx.x] : 0;
  __syncthreads();
  int cnt[2 + 2 * MOEP_MAX_BOUNDS];
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) cnt[i] = 0;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (NT / 32);
  for (int64_t row = gw; row < n; row += nwarps) {
    const T* zr = z + row * E;
    int tr[16];
    int any0 = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      tr[j] = 0;
      if (j < k) {
        const int t = truth[row * k + j];
        const T zt = zr[t];
        int r = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
          const int e = e0 + lane;
          const bool before = e < E && key_gt(zr[e < E ? e : 0], e, zt, t);
          r += __popc(__ballot_sync(0xffffffffu, before));
        }
        tr[j] = r;
        any0 |= r == 0;
        if (lane == 0) {
          hist[E + t] += 1;
          if (r < k) hist[t] += 1;
        }
      }
    }
    cnt[0] += 1;
    cnt[1] += any0;
#pragma unroll
    for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
      if (mi < n_m) {
        int inside = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) inside += (j < k && tr[j] < mls[mi]) ? 1 : 0;
        cnt[2 + mi] += inside == k;
        cnt[2 + MOEP_MAX_BOUNDS + mi] += inside;
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) scal[warp][i] = cnt[i];
  }
  __syncthreads();
  int* out = partials + static_cast<int64_t>(blockIdx.x) * n_counters;
  for (int t = threadIdx.x; t < n_counters; t += NT) {
    int v = 0;
    if (t < 2 + 2 * n_m) {
      const int src = t < 2 ? t : (t < 2 + n_m ? t : 2 + MOEP_MAX_BOUNDS + (t - 2 - n_m));
      for (int w = 0; w < NT / 32; ++w) v += scal[w][src];
    } else {
      const int e = t - 2 - 2 * n_m;
      for (int w = 0; w < NT / 32; ++w) v += sh[w * 2 * E + e];
    }
    out[t] = v;
  }
}

// Register-resident variants. The row of logits sits in registers (16 or 32
// lanes per token); the k true ids are one coalesced load; the stable rank of
// each true expert is popc(ballot(key_gt)) over the row (no re-reads), its
// logit a shuffle. Several tokens per warp iteration keep their loads in
// flight together. Block = 32 warps, one block per SM: the partial counter
// row layout [num_SMs][n_counters] is unchanged.
constexpr int NTR = 1024;

template <typename T, int PL>
__device__ __forceinline__ T lane_pick(const T (&v)[PL], int q) {
  T r = v[0];
#pragma unroll
  for (int i = 1; i < PL; ++i)
    if (i == q) r = v[i];
  return r;
}

template <typename T, int LPR, int EPL, int RPI>
__global__ void __launch_bounds__(NTR)
eval_reg_kernel(const T* __restrict__ z, int64_t n, int E, const int* __restrict__ truth, int k,
                int n_m, const int* __restrict__ m_list_dev, int* partials, int n_counters) {
  // LPR lanes per token (k <= LPR), expert e = i * LPR + lane_in_row held in
  // slot i; 32 / LPR tokens side by side in a warp, RPI such groups per
  // iteration.
  constexpr int RPW = 32 / LPR;
  extern __shared__ int sh[];  // [32 warps][2E] hist
  __shared__ int scal[NTR / 32][2 + 2 * MOEP_MAX_BOUNDS];
  __shared__ int mls[MOEP_MAX_BOUNDS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const uint32_t submask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  int* hist = sh + warp * 2 * E;
  for (int i = lane; i < 2 * E; i += 32) hist[i] = 0;
  if (threadIdx.x < MOEP_MAX_BOUNDS) mls[threadIdx.x] = threadIdx.x < n_m ? m_list_dev[threadIdx.x] : 0;
  __syncthreads();
  int m_of[MOEP_MAX_BOUNDS];
#pragma unroll
  for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) m_of[mi] = mls[mi];
  int cnt[2 + 2 * MOEP_MAX_BOUNDS];
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) cnt[i] = 0;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NTR / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NTR / 32);
  for (int64_t base = gw * RPI * RPW; base < n; base += nw * RPI * RPW) {
    T zv[RPI][EPL];
    int tv[RPI];
#pragma unroll
    for (int r = 0; r < RPI; ++r) {  // every load of the group's rows first
      const int64_t row = base + r * RPW + sub;
      const bool ok = row < n;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = i * LPR + li;
        zv[r][i] = (ok && e < E) ? z[row * E + e] : T(0);
      }
      tv[r] = (ok && li < k) ? truth[row * k + li] : 0;
    }
#pragma unroll
    for (int r = 0; r < RPI; ++r) {
      if (base + r * RPW >= n) break;  // warp-uniform
      const bool ok = base + r * RPW + sub < n;
      int my_rank = 0;
      for (int j = 0; j < k; ++j) {
        const int t = __shfl_sync(0xffffffffu, tv[r], j, LPR);
        const T zt = __shfl_sync(0xffffffffu, lane_pick<T, EPL>(zv[r], t / LPR), t % LPR, LPR);
        int rk = 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int e = i * LPR + li;
          rk += __popc(__ballot_sync(0xffffffffu, e < E && key_gt(zv[r][i], e, zt, t)) & submask);
        }
        if (li == j) my_rank = rk;
      }
      // lane j < k holds true expert j's rank: the per-token counts are ballots
      const bool mine = li < k;
      const int any0 = (__ballot_sync(0xffffffffu, mine && my_rank == 0) & submask) != 0;
      int inside[MOEP_MAX_BOUNDS];
#pragma unroll
      for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi)
        inside[mi] = __popc(__ballot_sync(0xffffffffu, mine && my_rank < m_of[mi]) & submask);
      // shared atomics: a token's true ids may repeat (the reference's
      // bincount counts every occurrence, metrics.py:182-187)
      if (ok && li < k) {
        atomicAdd(&hist[E + tv[r]], 1);
        if (my_rank < k) atomicAdd(&hist[tv[r]], 1);
      }
      if (ok && li == 0) {
        cnt[0] += 1;
        cnt[1] += any0;
#pragma unroll
        for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
          cnt[2 + mi] += inside[mi] == k ? 1 : 0;
          cnt[2 + MOEP_MAX_BOUNDS + mi] += inside[mi];
        }
      }
    }
  }
  // the row-group leaders (li == 0) hold the counts: sum them over the warp
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) {
    int v = cnt[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    cnt[i] = v;
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) scal[warp][i] = cnt[i];
  }
  __syncthreads();
  int* out = partials + static_cast<int64_t>(blockIdx.x) * n_counters;
  for (int t = threadIdx.x; t < n_counters; t += NTR) {
    int v = 0;
    if (t < 2 + 2 * n_m) {
      const int src = t < 2 ? t : (t < 2 + n_m ? t : 2 + MOEP_MAX_BOUNDS + (t - 2 - n_m));
      for (int w = 0; w < NTR / 32; ++w) v += scal[w][src];
    } else {
      const int e = t - 2 - 2 * n_m;
      for (int w = 0; w < NTR / 32; ++w) v += sh[w * 2 * E + e];
    }
    out[t] = v;
  }
}

// v2 (E <= 128): each lane holds EPL CONSECUTIVE experts (e = li * EPL + i:
// one vector load per lane per token); the stable rank of true expert t is a
// local count over the lane's slots, summed over the token's lanes with one
// redux (for 16-lane groups both halves of the warp reduce in the same
// instruction, packed in 16-bit fields). RPI row groups per warp iteration
// with every load issued first. ~3x fewer instructions per token than v1.
template <typename T, int EPL>
struct VecLoad;
template <> struct VecLoad<float, 1> { static __device__ void ld(const float* p, float* v) { v[0] = __ldcs(p); } };
template <> struct VecLoad<float, 2> {
  static __device__ void ld(const float* p, float* v) { const float2 a = __ldcs(reinterpret_cast<const float2*>(p)); v[0] = a.x; v[1] = a.y; }
};
template <> struct VecLoad<float, 4> {
  static __device__ void ld(const float* p, float* v) {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(p)); v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};
template <> struct VecLoad<double, 1> { static __device__ void ld(const double* p, double* v) { v[0] = __ldcs(p); } };
template <> struct VecLoad<double, 2> {
  static __device__ void ld(const double* p, double* v) { const double2 a = __ldcs(reinterpret_cast<const double2*>(p)); v[0] = a.x; v[1] = a.y; }
};
template <> struct VecLoad<double, 4> {
  static __device__ void ld(const double* p, double* v) {
    const double2 a = __ldcs(reinterpret_cast<const double2*>(p)), b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};

template <typename T, int LPR, int EPL, int RPI>
__global__ void __launch_bounds__(NTR)
eval_v2_kernel(const T* __restrict__ z, int64_t n, int E, const int* __restrict__ truth, int k,
               int n_m, const int* __restrict__ m_list_dev, int* partials, int n_counters) {
  constexpr int RPW = 32 / LPR;
  extern __shared__ int sh[];  // [32 warps][2E] hist
  __shared__ int scal[NTR / 32][2 + 2 * MOEP_MAX_BOUNDS];
  __shared__ int mls[MOEP_MAX_BOUNDS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const uint32_t submask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  int* hist = sh + warp * 2 * E;
  for (int i = lane; i < 2 * E; i += 32) hist[i] = 0;
  if (threadIdx.x < MOEP_MAX_BOUNDS) mls[threadIdx.x] = threadIdx.x < n_m ? m_list_dev[threadIdx.x] : 0;
  __syncthreads();
  int m_of[MOEP_MAX_BOUNDS];
#pragma unroll
  for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) m_of[mi] = mls[mi];
  int cnt[2 + 2 * MOEP_MAX_BOUNDS];
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) cnt[i] = 0;
  const bool full_rows = E == LPR * EPL;  // vector loads need the row to fill the lanes exactly
  const int e0 = li * EPL;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NTR / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NTR / 32);
  for (int64_t base = gw * RPI * RPW; base < n; base += nw * RPI * RPW) {
    T zv[RPI][EPL];
    int tv[RPI];
#pragma unroll
    for (int r = 0; r < RPI; ++r) {
      const int64_t row = base + r * RPW + sub;
      const bool ok = row < n;
      if (ok && full_rows) {
        VecLoad<T, EPL>::ld(z + row * E + e0, zv[r]);
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) zv[r][i] = (ok && e0 + i < E) ? z[row * E + e0 + i] : T(0);
      }
      tv[r] = (ok && li < k) ? __ldcs(truth + row * k + li) : 0;
    }
#pragma unroll
    for (int r = 0; r < RPI; ++r) {
      if (base + r * RPW >= n) break;  // warp-uniform
      const bool ok = base + r * RPW + sub < n;
      // experts beyond E (padding) never rank before anything
#pragma unroll
      for (int i = 0; i < EPL; ++i)
        if (e0 + i >= E) zv[r][i] = T(-INFINITY);
      int my_rank = 0;
      for (int j = 0; j < k; ++j) {
        const int t = __shfl_sync(0xffffffffu, tv[r], j, LPR);
        const int slot = t % EPL;
        T mine = zv[r][0];
#pragma unroll
        for (int i = 1; i < EPL; ++i)
          if (i == slot) mine = zv[r][i];
        const T zt = __shfl_sync(0xffffffffu, mine, t / EPL, LPR);
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const T v = zv[r][i];
          c += (v > zt || (v == zt && e0 + i < t)) ? 1u : 0u;
        }
        uint32_t rk;
        if (LPR == 16) {
          const uint32_t tot = __reduce_add_sync(0xffffffffu, c << (16 * sub));
          rk = (tot >> (16 * sub)) & 0xffffu;
        } else {
          rk = __reduce_add_sync(0xffffffffu, c);
        }
        if (li == j) my_rank = static_cast<int>(rk);
      }
      const bool own = li < k;
      const int any0 = (__ballot_sync(0xffffffffu, own && my_rank == 0) & submask) != 0;
      int inside[MOEP_MAX_BOUNDS];
#pragma unroll
      for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi)
        inside[mi] = __popc(__ballot_sync(0xffffffffu, own && my_rank < m_of[mi]) & submask);
      // shared atomics: a token's true ids may repeat (bincount, metrics.py:182-187)
      if (ok && own) {
        atomicAdd(&hist[E + tv[r]], 1);
        if (my_rank < k) atomicAdd(&hist[tv[r]], 1);
      }
      if (ok && li == 0) {
        cnt[0] += 1;
        cnt[1] += any0;
#pragma unroll
        for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
          cnt[2 + mi] += inside[mi] == k ? 1 : 0;
          cnt[2 + MOEP_MAX_BOUNDS + mi] += inside[mi];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) cnt[i] = __reduce_add_sync(0xffffffffu, cnt[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) scal[warp][i] = cnt[i];
  }
  __syncthreads();
  int* out = partials + static_cast<int64_t>(blockIdx.x) * n_counters;
  for (int t = threadIdx.x; t < n_counters; t += NTR) {
    int v = 0;
    if (t < 2 + 2 * n_m) {
      const int src = t < 2 ? t : (t < 2 + n_m ? t : 2 + MOEP_MAX_BOUNDS + (t - 2 - n_m));
      for (int w = 0; w < NTR / 32; ++w) v += scal[w][src];
    } else {
      const int e = t - 2 - 2 * n_m;
      for (int w = 0; w < NTR / 32; ++w) v += sh[w * 2 * E + e];
    }
    out[t] = v;
  }
}

// top-m ids (m <= 16) ascending: m rounds of argmax over the token's LPR
// lanes under the reference key (value, then lower index), then a ballot
// prefix over expert order. 32 / LPR tokens side by side per warp, RPI groups
// interleaved round by round (independent chains).
template <typename T, int LPR, int EPL, int RPI>
__global__ void __launch_bounds__(256)
topk_reg_kernel(const T* __restrict__ z, int64_t n, int E, int m, int* __restrict__ ids) {
  constexpr int RPW = 32 / LPR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const uint32_t submask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * 8;
  for (int64_t base = gw * RPI * RPW; base < n; base += nw * RPI * RPW) {
    T zv[RPI][EPL];
#pragma unroll
    for (int r = 0; r < RPI; ++r) {
      const int64_t row = base + r * RPW + sub;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = i * LPR + li;
        zv[r][i] = (row < n && e < E) ? z[row * E + e] : T(0);
      }
    }
    uint32_t taken[RPI];
#pragma unroll
    for (int r = 0; r < RPI; ++r) taken[r] = 0;
    for (int s = 0; s < m; ++s) {
#pragma unroll
      for (int r = 0; r < RPI; ++r) {
        T best = T(0);
        int bi = -1;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int e = i * LPR + li;
          if (e < E && !((taken[r] >> i) & 1u) && (bi < 0 || key_gt(zv[r][i], e, best, bi))) { best = zv[r][i]; bi = e; }
        }
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) {
          const T ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (oi >= 0 && (bi < 0 || key_gt(ov, oi, best, bi))) { best = ov; bi = oi; }
        }
        if (bi >= 0 && bi % LPR == li) taken[r] |= 1u << (bi / LPR);
      }
    }
#pragma unroll
    for (int r = 0; r < RPI; ++r) {
      const int64_t row = base + r * RPW + sub;
      int written = 0;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const bool sel = (taken[r] >> i) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, sel) & submask;
        if (sel && row < n) ids[row * m + written + __popc(bal & ((1u << lane) - 1u))] = i * LPR + li;
        written += __popc(bal);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(NT)
topk_kernel(const T* __restrict__ z, int64_t n, int E, int m, int* __restrict__ ids) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (NT / 32);
  for (int64_t row = gw; row < n; row += nwarps) {
    const T* zr = z + row * E;
    int written = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      bool sel = false;
      if (e < E) {
        const T ze = zr[e];
        int r = 0;
        for (int j = 0; j < E && r < m; ++j) r += key_gt(zr[j], j, ze, e) ? 1 : 0;
        sel = r < m;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, sel);
      if (sel) ids[row * m + written + __popc(bal & ((1u << lane) - 1u))] = e;
      written += __popc(bal);
    }
  }
}

// Full stable descending order: order[rank(e)] = e, rank by exact key counts.
template <typename T>
__global__ void __launch_bounds__(NT)
order_kernel(const T* __restrict__ z, int64_t n, int E, int* __restrict__ order) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (NT / 32);
  for (int64_t row = gw; row < n; row += nwarps) {
    const T* zr = z + row * E;
    for (int e = lane; e < E; e += 32) {
      const T ze = zr[e];
      int r = 0;
      for (int j = 0; j < E; ++j) r += key_gt(zr[j], j, ze, e) ? 1 : 0;
      order[row * E + r] = e;
    }
  }
}

// Counter reduction. int64 sums are exact, so the summation order does not
// change the result. Block = 32 counters x 32 warps: lanes read
// 32 consecutive counters of one partial row (coalesced), the 32 warps of the
// block split the partial rows, then a shared-memory tree.
__global__ void __launch_bounds__(1024) reduce_kernel(const int* __restrict__ partials, int n_blocks,
                                                      int n_counters, long long* __restrict__ out) {
  __shared__ long long red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  long long s = 0;
  if (c < n_counters) {
#pragma unroll 4
    for (int b = w; b < n_blocks; b += 32) s += partials[static_cast<int64_t>(b) * n_counters + c];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0) {
    long long t = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) t += red[i][lane];
    if (c < n_counters) out[c] = t;
  }
}

// ------------------------------------------------------------- K0: input norm
}  // namespace k7
}  // namespace moep

extern "C" {

int moep_num_sms(void) {
  static int cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

const char* moep_version(void) { return "moep_b200 0.1 sm_100a"; }

int moep_k7b_eval(const void* z, int32_t dtype, int64_t n, int32_t E, const int32_t* truth, int32_t k,
                  int32_t n_m, const int32_t* m_list, int32_t* partials, int32_t ncnt, void* stream);
int moep_k7b_topk(const void* z, int32_t dtype, int64_t n, int32_t E, int32_t m, int32_t* ids, void* stream);

int moep_eval_logits(const void* logits, int32_t dtype, int64_t n, int32_t E, const int32_t* truth,
                     int32_t k, int32_t n_m, const int32_t* m_list, int32_t* partials, void* stream) {
  using namespace moep::k7;
  if (n <= 0 || E <= 0) return MOEP_ESHAPE;
  if (k < 1 || k > 16 || k > E || n_m < 1 || n_m > MOEP_MAX_BOUNDS) return MOEP_EARG;
  const int ncnt = moep_n_counters(n_m, E);
  // one thread per token, packed-key networks (k7b_rows.cu): E in {16, 32, 64}
  if (E == 16 || E == 32 || E == 64) {
    const int rc = moep_k7b_eval(logits, dtype, n, E, truth, k, n_m, m_list, partials, ncnt, stream);
    if (rc != MOEP_EUNSUPPORTED) return rc;
  }
  const size_t smem = sizeof(int) * 2 * E * (NT / 32);
  if (smem > 200 * 1024) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = moep_num_sms();
  if (E <= 256) {
    const size_t smem_r = sizeof(int) * 2 * E * (NTR / 32);
#define MOEP_K7E(T, LPR, EPL)                                                                               \
  do {                                                                                                      \
    auto kern = eval_reg_kernel<T, LPR, EPL, 2>;                                                            \
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r) != cudaSuccess) \
      return MOEP_ELAUNCH;                                                                                  \
    kern<<<grid, NTR, smem_r, st>>>(static_cast<const T*>(logits), n, E, truth, k, n_m, m_list, partials, ncnt); \
  } while (0)
#define MOEP_K7E2(T, LPR, EPL)                                                                              \
  do {                                                                                                      \
    auto kern = eval_v2_kernel<T, LPR, EPL, sizeof(T) == 8 ? 2 : 4>;                                                           \
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r) != cudaSuccess) \
      return MOEP_ELAUNCH;                                                                                  \
    kern<<<grid, NTR, smem_r, st>>>(static_cast<const T*>(logits), n, E, truth, k, n_m, m_list, partials, ncnt); \
  } while (0)
    // v2 (consecutive experts per lane, redux ranks) needs 16-byte aligned rows
    const bool al = (reinterpret_cast<uintptr_t>(logits) & 15) == 0;
#define MOEP_K7E_T(T)                                                \
  do {                                                               \
    if (E <= 16 && k <= 16) MOEP_K7E2(T, 16, 1);                     \
    else if (E <= 32 && k <= 16 && al) MOEP_K7E2(T, 16, 2);          \
    else if (E <= 64 && k <= 16 && al) MOEP_K7E2(T, 16, 4);          \
    else if (E <= 128 && al) MOEP_K7E2(T, 32, 4);                    \
    else if (E <= 16 && k <= 16) MOEP_K7E(T, 16, 1);                 \
    else if (E <= 32 && k <= 16) MOEP_K7E(T, 16, 2);                 \
    else if (E <= 64 && k <= 16) MOEP_K7E(T, 16, 4);                 \
    else if (E <= 32) MOEP_K7E(T, 32, 1);                            \
    else if (E <= 64) MOEP_K7E(T, 32, 2);                            \
    else if (E <= 128) MOEP_K7E(T, 32, 4);                           \
    else MOEP_K7E(T, 32, 8);                                         \
  } while (0)
    if (dtype == MOEP_F64) MOEP_K7E_T(double);
    else if (dtype == MOEP_F32) MOEP_K7E_T(float);
    else return MOEP_EARG;
#undef MOEP_K7E_T
#undef MOEP_K7E
#undef MOEP_K7E2
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  }
  if (dtype == MOEP_F64) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(eval_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eval_kernel<double><<<grid, NT, smem, st>>>(static_cast<const double*>(logits), n, E, truth, k, n_m, m_list, partials, ncnt);
  } else if (dtype == MOEP_F32) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(eval_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eval_kernel<float><<<grid, NT, smem, st>>>(static_cast<const float*>(logits), n, E, truth, k, n_m, m_list, partials, ncnt);
  } else {
    return MOEP_EARG;
  }
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_topk_logits(const void* logits, int32_t dtype, int64_t n, int32_t E, int32_t m, int32_t* ids,
                     void* stream) {
  using namespace moep::k7;
  if (n <= 0 || E <= 0) return MOEP_ESHAPE;
  if (m < 1 || m > E) return MOEP_EARG;
  if (E == 16 || E == 32 || E == 64) {
    const int rc = moep_k7b_topk(logits, dtype, n, E, m, ids, stream);
    if (rc != MOEP_EUNSUPPORTED) return rc;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = moep_num_sms() * 4;
  if (E <= 256 && m <= 16) {
    const int64_t want = (n + 63) / 64;  // 8 warps x 4 groups x 2 rows per block iteration
    const int g2 = static_cast<int>(want < 8 * moep_num_sms() ? want : 8 * moep_num_sms());
#define MOEP_K7T(T, LPR, EPL) topk_reg_kernel<T, LPR, EPL, 4><<<g2, 256, 0, st>>>(static_cast<const T*>(logits), n, E, m, ids)
#define MOEP_K7T_T(T)                        \
  do {                                       \
    if (E <= 16) MOEP_K7T(T, 16, 1);         \
    else if (E <= 32) MOEP_K7T(T, 16, 2);    \
    else if (E <= 64) MOEP_K7T(T, 16, 4);    \
    else if (E <= 128) MOEP_K7T(T, 32, 4);   \
    else MOEP_K7T(T, 32, 8);                 \
  } while (0)
    if (dtype == MOEP_F64) MOEP_K7T_T(double);
    else if (dtype == MOEP_F32) MOEP_K7T_T(float);
    else return MOEP_EARG;
#undef MOEP_K7T_T
#undef MOEP_K7T
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  }
  if (dtype == MOEP_F64)
    topk_kernel<double><<<grid, NT, 0, st>>>(static_cast<const double*>(logits), n, E, m, ids);
  else if (dtype == MOEP_F32)
    topk_kernel<float><<<grid, NT, 0, st>>>(static_cast<const float*>(logits), n, E, m, ids);
  else
    return MOEP_EARG;
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_rank_order(const void* logits, int32_t dtype, int64_t n, int32_t E, int32_t* order,
                     void* stream) {
  using namespace moep::k7;
  if (n <= 0 || E <= 0) return MOEP_ESHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = moep_num_sms() * 4;
  if (dtype == MOEP_F64)
    order_kernel<double><<<grid, NT, 0, st>>>(static_cast<const double*>(logits), n, E, order);
  else if (dtype == MOEP_F32)
    order_kernel<float><<<grid, NT, 0, st>>>(static_cast<const float*>(logits), n, E, order);
  else
    return MOEP_EARG;
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_counters_reduce(const int32_t* partials, int32_t n_blocks, int32_t n_counters, int64_t* out,
                         void* stream) {
  if (n_blocks <= 0 || n_counters <= 0) return MOEP_ESHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  moep::k7::reduce_kernel<<<(n_counters + 31) / 32, 1024, 0, st>>>(
      partials, n_blocks, n_counters, reinterpret_cast<long long*>(out));
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // extern "C"
