// k7b_rows.cu — K7 from given logits, one THREAD per token (E in {16, 32, 64}):
// exact top-m ids (core.top_k_batch, core.py:42-48) and the evaluation
// counters (metrics.evaluate_predictions, metrics.py:138-193).
//
// The warp's 32 rows are staged through shared memory with coalesced 16-byte
// loads (padded rows: conflict-free per-lane reads). Each thread turns its row
// into 32-bit PACKED keys
//     P(e) = (orderable(z_e) & ~63) | (63 - e)
// orderable(): the monotone unsigned image of the value (+0.0 == -0.0; NaN
// lowest, as numpy's argsort(-z) puts NaN last); the low 6 bits hold the
// inverted index, so larger P = earlier in the reference order (descending
// value, ties to the lower index) and every key is distinct. A bitonic network
// of unsigned min / max (two instructions per compare-exchange) then sorts
// groups of G keys and merges them keeping the top G. The packed order equals
// the reference order except between keys that agree in their top 26 bits;
// a boundary the caller needs (position m for ids; 1, k and each m of the
// evaluation list) is exact unless the two keys straddling it agree there,
// and those rows (rare for continuous logits) redo the boundary decision with
// exact comparisons over the staged row. ~1,000 instructions per token
// against ~4,900 for the 16-lanes-per-token shuffle argmax rounds it replaces.
#include <cuda_runtime.h>
#include <cstdint>
#include <climits>
#include "common.cuh"
#include "sortnet.cuh"

namespace moep {
namespace k7b {

using namespace moep::sortnet;

// staged row stride (elements): 16-byte pad, conflict-free 16-byte per-lane reads
template <typename T, int E>
struct Row {
  static constexpr int PAD = 16 / sizeof(T);
  static constexpr int S = E + PAD;
  static constexpr int V = 16 / sizeof(T);  // elements per 16-byte chunk
};

// the warp's rows [r0, r0 + 32) -> stg[32][S] (coalesced 16-byte loads)
template <typename T, int E>
__device__ __forceinline__ void stage_rows(const T* __restrict__ z, int64_t r0, int64_t n, T* stg, int lane) {
  using R = Row<T, E>;
  constexpr int C = E / R::V;  // chunks per row
  const int64_t rows = n - r0 < 32 ? n - r0 : 32;
  const uint4* src = reinterpret_cast<const uint4*>(z + r0 * E);
#pragma unroll
  for (int t = 0; t < C; ++t) {
    const int idx = t * 32 + lane, row = idx / C, c = idx % C;
    const uint4 v = row < rows ? __ldcs(src + idx) : make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(stg + row * R::S + c * R::V) = v;
  }
}

// this thread's row -> packed keys sorted: top G in `top` (descending)
template <typename T, int E, int G>
__device__ __forceinline__ void top_keys(const T* myrow, uint32_t (&top)[G]) {
  using R = Row<T, E>;
  uint32_t grp[G];
#pragma unroll
  for (int g0 = 0; g0 < E; g0 += G) {
#pragma unroll
    for (int c = 0; c < G; c += R::V) {
      const uint4 q = *reinterpret_cast<const uint4*>(myrow + g0 + c);
      T v[R::V];
      unpack16(q, v);
#pragma unroll
      for (int u = 0; u < R::V; ++u) {
        const int e = g0 + c + u;
        grp[c + u] = (okey(v[u]) & ~63u) | static_cast<uint32_t>(63 - e);
      }
    }
    sort_desc<G>(grp);
    if (g0 == 0) {
#pragma unroll
      for (int i = 0; i < G; ++i) top[i] = grp[i];
    } else {
      merge_top<G>(top, grp);
    }
  }
}

// exact: number of experts before expert t in the reference order
template <typename T, int E>
__device__ __forceinline__ int exact_rank(const T* myrow, int t) {
  const T zt = myrow[t];
  int r = 0;
  for (int e = 0; e < E; ++e) r += exact_before(myrow[e], e, zt, t) ? 1 : 0;
  return r;
}

constexpr int NTT = 256;  // top-m block

template <typename T, int E, int G>
__global__ void __launch_bounds__(NTT)
topk_rows_kernel(const T* __restrict__ z, int64_t n, int m, int* __restrict__ ids) {
  using R = Row<T, E>;
  extern __shared__ __align__(16) unsigned char k7b_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* stg = reinterpret_cast<T*>(k7b_smem) + warp * 32 * R::S;
  const T* myrow = stg + lane * R::S;
  int* ostg = reinterpret_cast<int*>(stg);  // output staging reuses the rows (after every lane read its own)
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NTT / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NTT / 32);
  for (int64_t r0 = gw * 32; r0 < n; r0 += nw * 32) {
    stage_rows<T, E>(z, r0, n, stg, lane);
    __syncwarp();
    const int64_t row = r0 + lane;
    uint64_t sel = 0;
    if (m >= E) {
      sel = E == 64 ? ~0ull : ((1ull << E) - 1ull);
    } else {
      uint32_t top[G];
      top_keys<T, E, G>(myrow, top);
      uint32_t a = top[0], b = top[1];
#pragma unroll
      for (int i = 1; i < G; ++i)
        if (i == m) { a = top[i - 1]; b = top[i]; }
#pragma unroll
      for (int i = 0; i < G; ++i)
        if (i < m) sel |= 1ull << pk_index(top[i]);
      if (row < n && ambiguous(a, b)) {
        // exact boundary: the m experts first in the reference order
        sel = 0;
        for (int e = 0; e < E; ++e)
          if (exact_rank<T, E>(myrow, e) < m) sel |= 1ull << e;
      }
    }
    __syncwarp();  // every lane done with the staged rows
    // ascending ids -> output staging [32][m], then coalesced stores
    for (int j = 0; j < m; ++j) {
      const int e = __ffsll(static_cast<long long>(sel)) - 1;
      sel &= sel - 1;
      ostg[lane * m + j] = e;
    }
    __syncwarp();
    const int64_t rows = n - r0 < 32 ? n - r0 : 32;
    int* dst = ids + r0 * m;
    for (int i = lane; i < rows * m; i += 32) dst[i] = ostg[i];
    __syncwarp();
  }
}

// evaluation block: one per SM (the partial-counter row layout); 16 warps
// (8 for fp64 rows: the staging of 16 warps would not fit)
template <typename T>
struct EvalBlock { static constexpr int NT = sizeof(T) == 8 ? 256 : 512; };

template <typename T, int E, int G>
__global__ void __launch_bounds__(EvalBlock<T>::NT)
eval_rows_kernel(const T* __restrict__ z, int64_t n, const int* __restrict__ truth, int k, int n_m,
                 const int* __restrict__ m_list_dev, int* __restrict__ partials, int n_counters) {
  using R = Row<T, E>;
  extern __shared__ __align__(16) unsigned char k7b_smem[];
  constexpr int NTE = EvalBlock<T>::NT, NW = NTE / 32;
  int* hist0 = reinterpret_cast<int*>(k7b_smem);                                  // [NW][2E]
  T* stg0 = reinterpret_cast<T*>(k7b_smem + ((NW * 2 * E * sizeof(int) + 15) & ~size_t(15)));
  __shared__ int scal[NW][2 + 2 * MOEP_MAX_BOUNDS];
  __shared__ int mls[MOEP_MAX_BOUNDS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* hist = hist0 + warp * 2 * E;
  for (int i = lane; i < 2 * E; i += 32) hist[i] = 0;
  if (threadIdx.x < MOEP_MAX_BOUNDS) mls[threadIdx.x] = threadIdx.x < n_m ? m_list_dev[threadIdx.x] : E;
  __syncthreads();
  int mv[MOEP_MAX_BOUNDS];
#pragma unroll
  for (int i = 0; i < MOEP_MAX_BOUNDS; ++i) mv[i] = mls[i];
  // the list resolves every threshold below G; otherwise every row counts exactly
  bool list_ok = k < G;
#pragma unroll
  for (int i = 0; i < MOEP_MAX_BOUNDS; ++i) list_ok &= (i >= n_m) || mv[i] >= E || mv[i] < G;
  T* stg = stg0 + warp * 32 * R::S;
  const T* myrow = stg + lane * R::S;
  int cnt[2 + 2 * MOEP_MAX_BOUNDS];
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) cnt[i] = 0;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * NW + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * NW;
  for (int64_t r0 = gw * 32; r0 < n; r0 += nw * 32) {
    stage_rows<T, E>(z, r0, n, stg, lane);
    __syncwarp();
    const int64_t row = r0 + lane;
    if (row < n) {
      int rank[16];
      bool exact = !list_ok;
      if (list_ok) {
        uint32_t top[G];
        top_keys<T, E, G>(myrow, top);
        // boundaries the counters read: 1, k, every m < E
        auto amb_at = [&](int b) {
          bool r = false;
#pragma unroll
          for (int i = 1; i < G; ++i)
            if (i == b) r = ambiguous(top[i - 1], top[i]);
          return r;
        };
        bool amb = amb_at(1) || amb_at(k);
#pragma unroll
        for (int i = 0; i < MOEP_MAX_BOUNDS; ++i)
          if (i < n_m && mv[i] < E) amb |= amb_at(mv[i]);
        exact = amb;
        if (!amb) {
          // rank = position in the top list, else >= G (beyond every threshold)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < k) {
              const int t = __ldg(truth + row * k + j);
              int r = G;
#pragma unroll
              for (int i = 0; i < G; ++i)
                if (pk_index(top[i]) == t) r = i;
              rank[j] = r;
            }
          }
        }
      }
      if (exact) {
        for (int j = 0; j < k; ++j) rank[j] = exact_rank<T, E>(myrow, __ldg(truth + row * k + j));
      }
      int any0 = 0;
      int inside[MOEP_MAX_BOUNDS] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < k) {
          const int t = __ldg(truth + row * k + j);
          any0 |= rank[j] == 0;
          atomicAdd(&hist[E + t], 1);  // bincount: repeated true ids count each time (metrics.py:182-187)
          if (rank[j] < k) atomicAdd(&hist[t], 1);
#pragma unroll
          for (int i = 0; i < MOEP_MAX_BOUNDS; ++i) inside[i] += (rank[j] < mv[i]) ? 1 : 0;
        }
      }
      cnt[0] += 1;
      cnt[1] += any0;
#pragma unroll
      for (int i = 0; i < MOEP_MAX_BOUNDS; ++i) {
        cnt[2 + i] += inside[i] == k ? 1 : 0;
        cnt[2 + MOEP_MAX_BOUNDS + i] += inside[i];
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) cnt[i] = __reduce_add_sync(0xffffffffu, cnt[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) scal[warp][i] = cnt[i];
  }
  __syncthreads();
  int* out = partials + static_cast<int64_t>(blockIdx.x) * n_counters;
  for (int t = threadIdx.x; t < n_counters; t += NTE) {
    int v = 0;
    if (t < 2 + 2 * n_m) {
      const int src = t < 2 ? t : (t < 2 + n_m ? t : 2 + MOEP_MAX_BOUNDS + (t - 2 - n_m));
      for (int w = 0; w < NW; ++w) v += scal[w][src];
    } else {
      const int e = t - 2 - 2 * n_m;
      for (int w = 0; w < NW; ++w) v += hist0[w * 2 * E + e];
    }
    out[t] = v;
  }
}

// K3 labels (losses.py BatchLabels: rank_of = 1 + stable descending rank,
// topk_mask = rank < k, and the strict pairs among the top T = min(10, E) of
// the ranking loss, losses.py:198-207): the full row sorted by one bitonic
// network of E packed keys. Rows whose order the packed keys cannot certify
// (two adjacent keys equal in their top 26 bits, or NaN inside the top T)
// recompute ranks and pairs exactly from the staged values.
constexpr int NTL = 256;

template <typename T, int E>
__global__ void __launch_bounds__(NTL)
labels_rows_kernel(const T* __restrict__ sc, int64_t n, int k, int top_cut, int* __restrict__ rank_of,
                   uint8_t* __restrict__ mask, int* __restrict__ pairs) {
  using R = Row<T, E>;
  static_assert(sizeof(T) >= sizeof(int), "rank staging reuses the value slots");
  extern __shared__ __align__(16) unsigned char k7b_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* stg = reinterpret_cast<T*>(k7b_smem) + warp * 32 * R::S;
  T* myrow = stg + lane * R::S;
  int* myrank = reinterpret_cast<int*>(myrow);  // this row's ranks overwrite its own values
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NTL / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NTL / 32);
  for (int64_t r0 = gw * 32; r0 < n; r0 += nw * 32) {
    stage_rows<T, E>(sc, r0, n, stg, lane);
    __syncwarp();
    const int64_t row = r0 + lane;
    uint32_t key[E];
#pragma unroll
    for (int c = 0; c < E; c += R::V) {
      T v[R::V];
      unpack16(*reinterpret_cast<const uint4*>(myrow + c), v);
#pragma unroll
      for (int u = 0; u < R::V; ++u) key[c + u] = (okey(v[u]) & ~63u) | static_cast<uint32_t>(63 - (c + u));
    }
    sort_desc<E>(key);
    bool amb = false;
#pragma unroll
    for (int i = 1; i < E; ++i) amb |= ambiguous(key[i - 1], key[i]);
    uint32_t tcut = key[0];
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (i == top_cut - 1) tcut = key[i];
    amb |= (tcut & ~63u) == 0u;  // NaN inside the top T
    int np = top_cut * (top_cut - 1) / 2;
    uint64_t sel = 0;
    if (row < n && amb) {
      int rk[E];
      for (int e = 0; e < E; ++e) rk[e] = exact_rank<T, E>(myrow, e);
      np = 0;
      for (int a = 0; a < E; ++a)
        for (int b = 0; b < E; ++b)
          np += (rk[a] < top_cut && rk[b] < top_cut && myrow[a] > myrow[b]) ? 1 : 0;
      for (int e = 0; e < E; ++e) {
        myrank[e] = rk[e] + 1;
        if (rk[e] < k) sel |= 1ull << e;
      }
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int e = pk_index(key[i]);
        myrank[e] = i + 1;
        if (i < k) sel |= 1ull << e;
      }
    }
    if (row < n) {
      if (pairs) pairs[row] = np;
#pragma unroll
      for (int c = 0; c < E; c += 16) {  // 16 mask bytes per store: bit e -> byte e
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t b = static_cast<uint32_t>(sel >> (c + 4 * q)) & 0xfu;
          w[q] = (b & 1u) | ((b & 2u) << 7) | ((b & 4u) << 14) | ((b & 8u) << 21);
        }
        *reinterpret_cast<uint4*>(mask + row * E + c) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    __syncwarp();
    // coalesced copy of the warp's rank rows
    const int64_t rows = n - r0 < 32 ? n - r0 : 32;
    int* dst = rank_of + r0 * E;
    for (int i = lane; i < rows * E; i += 32) dst[i] = reinterpret_cast<const int*>(stg + (i / E) * R::S)[i % E];
    __syncwarp();
  }
}

template <typename T, int E>
int launch_labels(const T* sc, int64_t n, int k, int top_cut, int* rank_of, uint8_t* mask, int* pairs,
                  cudaStream_t st) {
  using R = Row<T, E>;
  const size_t smem = sizeof(T) * (NTL / 32) * 32 * R::S;
  auto kern = labels_rows_kernel<T, E>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
      return MOEP_ELAUNCH;
    attr = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTL, smem) != cudaSuccess || per_sm < 1)
    return MOEP_ELAUNCH;
  const int64_t want = (n + NTL - 1) / NTL;
  const int64_t cap = static_cast<int64_t>(per_sm) * moep_num_sms();
  kern<<<static_cast<int>(want < cap ? want : cap), NTL, smem, st>>>(sc, n, k, top_cut, rank_of, mask, pairs);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

template <typename T, int E, int G>
int launch_topk(const T* z, int64_t n, int m, int* ids, cudaStream_t st) {
  using R = Row<T, E>;
  const size_t smem = sizeof(T) * (NTT / 32) * 32 * R::S;
  auto kern = topk_rows_kernel<T, E, G>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
      return MOEP_ELAUNCH;
    attr = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTT, smem) != cudaSuccess || per_sm < 1)
    return MOEP_ELAUNCH;
  const int64_t want = (n + NTT - 1) / NTT;
  const int64_t cap = static_cast<int64_t>(per_sm) * moep_num_sms();
  kern<<<static_cast<int>(want < cap ? want : cap), NTT, smem, st>>>(z, n, m, ids);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

template <typename T, int E, int G>
int launch_eval(const T* z, int64_t n, const int* truth, int k, int n_m, const int* m_list, int* partials,
                int ncnt, cudaStream_t st) {
  using R = Row<T, E>;
  constexpr int NTE = EvalBlock<T>::NT, NW = NTE / 32;
  const size_t smem = ((NW * 2 * E * sizeof(int) + 15) & ~size_t(15)) + sizeof(T) * NW * 32 * R::S;
  auto kern = eval_rows_kernel<T, E, G>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
      return MOEP_ELAUNCH;
    attr = true;
  }
  kern<<<moep_num_sms(), NTE, smem, st>>>(z, n, truth, k, n_m, m_list, partials, ncnt);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // namespace k7b
}  // namespace moep

// Entry points used by k7_eval.cu's moep_topk_logits / moep_eval_logits for
// E in {16, 32, 64} with 16-byte aligned rows. Return MOEP_EUNSUPPORTED when
// the shape is not covered (the caller then runs the general kernels).
extern "C" int moep_k7b_topk(const void* z, int32_t dtype, int64_t n, int32_t E, int32_t m, int32_t* ids,
                             void* stream) {
  using namespace moep::k7b;
  if ((reinterpret_cast<uintptr_t>(z) & 15) != 0 || m > 15) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool small = m < 8;  // the list must hold position m (the boundary's lower side)
  if (dtype == MOEP_F32) {
    const float* p = static_cast<const float*>(z);
    if (E == 16) return small ? launch_topk<float, 16, 8>(p, n, m, ids, st) : launch_topk<float, 16, 16>(p, n, m, ids, st);
    if (E == 32) return small ? launch_topk<float, 32, 8>(p, n, m, ids, st) : launch_topk<float, 32, 16>(p, n, m, ids, st);
    if (E == 64) return small ? launch_topk<float, 64, 8>(p, n, m, ids, st) : launch_topk<float, 64, 16>(p, n, m, ids, st);
  } else if (dtype == MOEP_F64) {
    const double* p = static_cast<const double*>(z);
    if (E == 16) return small ? launch_topk<double, 16, 8>(p, n, m, ids, st) : launch_topk<double, 16, 16>(p, n, m, ids, st);
    if (E == 32) return small ? launch_topk<double, 32, 8>(p, n, m, ids, st) : launch_topk<double, 32, 16>(p, n, m, ids, st);
    if (E == 64) return small ? launch_topk<double, 64, 8>(p, n, m, ids, st) : launch_topk<double, 64, 16>(p, n, m, ids, st);
  }
  return MOEP_EUNSUPPORTED;
}

extern "C" int moep_k7b_eval(const void* z, int32_t dtype, int64_t n, int32_t E, const int32_t* truth, int32_t k,
                             int32_t n_m, const int32_t* m_list, int32_t* partials, int32_t ncnt, void* stream) {
  using namespace moep::k7b;
  if ((reinterpret_cast<uintptr_t>(z) & 15) != 0 || k > 16) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == MOEP_F32) {
    const float* p = static_cast<const float*>(z);
    if (E == 16) return launch_eval<float, 16, 16>(p, n, truth, k, n_m, m_list, partials, ncnt, st);
    if (E == 32) return launch_eval<float, 32, 16>(p, n, truth, k, n_m, m_list, partials, ncnt, st);
    if (E == 64) return launch_eval<float, 64, 16>(p, n, truth, k, n_m, m_list, partials, ncnt, st);
  } else if (dtype == MOEP_F64) {
    const double* p = static_cast<const double*>(z);
    if (E == 16) return launch_eval<double, 16, 16>(p, n, truth, k, n_m, m_list, partials, ncnt, st);
    if (E == 32) return launch_eval<double, 32, 16>(p, n, truth, k, n_m, m_list, partials, ncnt, st);
    if (E == 64) return launch_eval<double, 64, 16>(p, n, truth, k, n_m, m_list, partials, ncnt, st);
  }
  return MOEP_EUNSUPPORTED;
}

extern "C" int moep_k7b_labels(const void* sc, int32_t dtype, int64_t n, int32_t E, int32_t k, int32_t top_cut,
                               int32_t* rank_of, uint8_t* mask, int32_t* pairs, void* stream) {
  using namespace moep::k7b;
  if ((reinterpret_cast<uintptr_t>(sc) | reinterpret_cast<uintptr_t>(mask)) & 15) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == MOEP_F32) {
    const float* p = static_cast<const float*>(sc);
    if (E == 16) return launch_labels<float, 16>(p, n, k, top_cut, rank_of, mask, pairs, st);
    if (E == 32) return launch_labels<float, 32>(p, n, k, top_cut, rank_of, mask, pairs, st);
    if (E == 64) return launch_labels<float, 64>(p, n, k, top_cut, rank_of, mask, pairs, st);
  } else if (dtype == MOEP_F64) {
    const double* p = static_cast<const double*>(sc);
    if (E == 16) return launch_labels<double, 16>(p, n, k, top_cut, rank_of, mask, pairs, st);
    if (E == 32) return launch_labels<double, 32>(p, n, k, top_cut, rank_of, mask, pairs, st);
    if (E == 64) return launch_labels<double, 64>(p, n, k, top_cut, rank_of, mask, pairs, st);
  }
  return MOEP_EUNSUPPORTED;
}
