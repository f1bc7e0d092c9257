// sortnet.cuh — 32-bit packed keys and bitonic min / max networks for exact
// top-k in the reference order (descending value, ties to the lower index,
// +0.0 == -0.0, NaN last; core.py:27-54), shared by K7 (k7b_rows.cu) and the
// K1 token epilogue (k1_common.cuh). A packed key is
//   (orderable(value) & ~63) | (63 - index)
// so larger = earlier and every key of a row is distinct; the packed order is
// the reference order except between keys equal in their top 26 bits
// (`ambiguous`), where callers fall back to exact comparisons.
#pragma once
#include <cstdint>

namespace moep {
namespace sortnet {

// monotone unsigned image of the value: larger value -> larger key; -0 == +0;
// NaN -> 0 (below -inf)
__device__ __forceinline__ uint32_t okey(float v) {
  const int b = __float_as_int(__fadd_rn(v, 0.0f));  // -0 + 0 = +0 (an FMA-pipe op instead of compare / select)
  const uint32_t u = static_cast<uint32_t>(b ^ ((b >> 31) | static_cast<int>(0x80000000u)));  // b >= 0 ? b | 2^31 : ~b
  return v != v ? 0u : u;  // NaN lowest
}
__device__ __forceinline__ uint32_t okey(double v) {
  const long long b = __double_as_longlong(__dadd_rn(v, 0.0));
  const unsigned long long u = static_cast<unsigned long long>(b >= 0 ? (b | static_cast<long long>(0x8000000000000000ull)) : ~b);
  const bool nan = (b & 0x7fffffffffffffffll) > 0x7ff0000000000000ll;
  return nan ? 0u : static_cast<uint32_t>(u >> 32);  // top 32 bits (the low 6 are replaced by the index)
}
// exact reference order between (a, ia) and (b, ib) on the full values
template <typename T>
__device__ __forceinline__ bool exact_before(T a, int ia, T b, int ib) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return (!na && nb) || (na && nb && ia < ib);  // NaN last, ties by index
  return a > b || (a == b && ia < ib);
}

template <int G>
__device__ __forceinline__ void ce(uint32_t (&a)[G], int i, int j) {  // a[i] >= a[j] afterwards
  const uint32_t x = a[i], y = a[j];
  a[i] = max(x, y);
  a[j] = min(x, y);
}
// descending bitonic sort of G keys
template <int G>
__device__ __forceinline__ void sort_desc(uint32_t (&a)[G]) {
#pragma unroll
  for (int size = 2; size <= G; size <<= 1)
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1)
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          if ((i & size) == 0 || size == G) ce<G>(a, i, j);
          else ce<G>(a, j, i);
        }
      }
}
// a <- top G of (a, b), both sorted descending
template <int G>
__device__ __forceinline__ void merge_top(uint32_t (&a)[G], const uint32_t (&b)[G]) {
#pragma unroll
  for (int i = 0; i < G; ++i) a[i] = max(a[i], b[G - 1 - i]);  // bitonic
#pragma unroll
  for (int stride = G >> 1; stride > 0; stride >>= 1)
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int j = i ^ stride;
      if (j > i) ce<G>(a, i, j);
    }
}

__device__ __forceinline__ int pk_index(uint32_t p) { return 63 - static_cast<int>(p & 63u); }
__device__ __forceinline__ bool ambiguous(uint32_t hi_side, uint32_t lo_side) {
  return ((hi_side ^ lo_side) & ~63u) == 0;
}

// the same with IB index bits (E <= 2^IB): keys (okey & ~(2^IB - 1)) | (2^IB - 1 - e)
template <int IB>
__device__ __forceinline__ uint32_t pk_make(uint32_t ok, int e) {
  constexpr uint32_t M = (1u << IB) - 1u;
  return (ok & ~M) | (M - static_cast<uint32_t>(e));
}
template <int IB>
__device__ __forceinline__ int pk_index_b(uint32_t p) { return static_cast<int>(((1u << IB) - 1u) - (p & ((1u << IB) - 1u))); }
template <int IB>
__device__ __forceinline__ bool ambiguous_b(uint32_t hi_side, uint32_t lo_side) {
  return ((hi_side ^ lo_side) & ~((1u << IB) - 1u)) == 0;
}

}  // namespace sortnet
}  // namespace moep
