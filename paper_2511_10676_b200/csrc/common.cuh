// common.cuh — shared device helpers: exact top-m selection, evaluation
// counters (warp-ballot histograms, no global atomics), activations.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../include/moep_b200.h"

namespace moep {

constexpr int kMaxSel = 16;  // positions of the sorted top list kept per row

// Reference key order (core.py:27-54): descending score, ties -> lower index.
// -0.0 == +0.0 under IEEE compares, matching numpy's stable argsort.
template <typename T>
__device__ __forceinline__ bool key_gt(T va, int ia, T vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

// Per-row evaluation contribution given a rank oracle `rank_of(expert)` that
// returns the stable predicted rank of an expert. Mirrors metrics.py:159-180.
struct RowCounters {
  int n, top1;
  int ov[MOEP_MAX_BOUNDS], rc[MOEP_MAX_BOUNDS];
  __device__ void zero() {
    n = 0; top1 = 0;
#pragma unroll
    for (int i = 0; i < MOEP_MAX_BOUNDS; ++i) { ov[i] = 0; rc[i] = 0; }
  }
};

// Sum a RowCounters across the warp and add per-warp totals into smem slot.
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fp64 -> bf16 round-to-nearest-even, directly (no fp32 double rounding).
__device__ __forceinline__ __nv_bfloat16 f64_to_bf16_rne(double x) {
  if (!isfinite(x)) return __float2bfloat16_rn(static_cast<float>(x));
  const double ax = fabs(x);
  if (ax < 1.1754943508222875e-38) {  // bf16 subnormal range: fixed quantum 2^-133
    const double q = 9.183549615799121e-41;
    return __float2bfloat16_rn(static_cast<float>(rint(x / q) * q));
  }
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const unsigned long long lsb = (b >> 45) & 1ull;
  b += (1ull << 44) - 1ull + lsb;  // RNE on the 45 dropped mantissa bits
  b &= ~((1ull << 45) - 1ull);
  const double r = __longlong_as_double(static_cast<long long>(b));  // <= 8 significant bits
  return __float2bfloat16_rn(static_cast<float>(r));                // exact (or inf on overflow)
}

// 16-byte chunk <-> register elements without taking a register array's
// address (a reinterpret_cast of the array forces it into local memory)
__device__ __forceinline__ void unpack16(const uint4& q, float* v) {
  v[0] = __uint_as_float(q.x); v[1] = __uint_as_float(q.y); v[2] = __uint_as_float(q.z); v[3] = __uint_as_float(q.w);
}
__device__ __forceinline__ void unpack16(const uint4& q, double* v) {
  v[0] = __hiloint2double(static_cast<int>(q.y), static_cast<int>(q.x));
  v[1] = __hiloint2double(static_cast<int>(q.w), static_cast<int>(q.z));
}
__device__ __forceinline__ void unpack16(const uint4& q, int* v) {
  v[0] = static_cast<int>(q.x); v[1] = static_cast<int>(q.y); v[2] = static_cast<int>(q.z); v[3] = static_cast<int>(q.w);
}
__device__ __forceinline__ uint4 pack16(const float* v) {
  return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
}
__device__ __forceinline__ uint4 pack16(const double* v) {
  return make_uint4(static_cast<uint32_t>(__double2loint(v[0])), static_cast<uint32_t>(__double2hiint(v[0])),
                    static_cast<uint32_t>(__double2loint(v[1])), static_cast<uint32_t>(__double2hiint(v[1])));
}

#ifdef MOEP_SILU_ACCURATE
__device__ __forceinline__ float silu_f32(float a) { return __fdiv_rn(a, 1.0f + expf(-a)); }
#else
__device__ __forceinline__ float silu_f32(float a) { return __fdividef(a, 1.0f + __expf(-a)); }
#endif

__device__ __forceinline__ float gelu_tanh_f32(float u) {
  const float c = 0.7978845608028654f, ga = 0.044715f;
  const float y = c * fmaf(ga * u * u, u, u);
  const float t = 1.0f - __fdividef(2.0f, __expf(2.0f * y) + 1.0f);
  return 0.5f * u * (1.0f + t);
}

}  // namespace moep
