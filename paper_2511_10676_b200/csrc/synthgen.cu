// synthgen.cu — K11: the reference's synthetic teacher on the GPU
// (pkg/src/moepredict/synthgen.py:162-189).
//
//   moep_teacher_normals   per-sample counter-based streams (synthgen.py:44-47:
//                          Philox4x64-10 keyed (seed << 64) + i) drawn through
//                          numpy's standard_normal ziggurat (tables generated
//                          from numpy by tools/gen_ziggurat_tables.py), the
//                          activation row then the noise row of each sample
//                          (synthgen.py:170-174). One thread per sample; rows
//                          staged 16 values at a time in shared memory so the
//                          HBM writes are coalesced.
//   moep_layer_norm_np     core.layer_norm (core.py:57-68) with numpy's exact
//                          reduction order: add.reduce = 0 + pairwise_sum
//                          (8 accumulators per block of <= 128, halving split
//                          rounded to a multiple of 8), then mean = s / d,
//                          var = pairwise((x - mean)^2) / d, (x - mean) /
//                          sqrt(var + eps) — every operation rounded once
//                          (explicit _rn intrinsics, no FMA contraction).
//   moep_softmax_np        core.softmax (core.py:19-24) over fp64 rows in numpy's
//                          order (max, exp, pairwise sum, divide).
//   moep_teacher_finish    softmax (core.py:19-24) in numpy order, float32 cast
//                          and top-k of the float32 scores (make_dataset,
//                          synthgen.py:148-159; core.py:42-48: descending,
//                          lower index first on ties, ids ascending).
//
// Bit-exactness: Philox words, the ziggurat's fast path (99.3 % of draws) and
// the pairwise sums are exact integer / correctly rounded operations, so the
// activations and layer-norm outputs equal numpy's. exp / log1p differ from
// glibc / numpy's SIMD exp in the last ulp on some inputs: the tail samples
// (|x| > 3.654, p = 2.6e-4) can differ by one fp64 ulp, which survives the
// float32 cast only at a rounding boundary (p ~ 2^-29); wedge decisions flip
// with p ~ 1e-16. The gate GEMM runs on cuBLAS (the reference's runs on
// OpenBLAS): scores agree to ~1e-16 relative before the float32 cast.
#include <cuda_runtime.h>
#include <cstdint>
#include "common.cuh"
#include "pairwise.cuh"
#include "ziggurat_tables.inc"

namespace moep {
namespace sg {

constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ull, kM1 = 0xCA5A826395121157ull;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ull, kW1 = 0xBB67AE8584CAA73Bull;
constexpr double kZigR = 3.6541528853610088, kZigInvR = 0.27366123732975828;

// numpy.random.Philox(key=...) stream: each refill is Philox4x64-10 of the
// counter incremented first (counter starts at 0), 4 words in stream order.
//
// Words sit in a per-thread 8-entry FIFO in shared memory. The caller refills
// in lockstep once per 4 normals (all lanes together: no divergent Philox
// rounds), and a lane whose FIFO runs dry after a slow-path draw refills on
// its own (`next64`). Every normal consumes >= 1 word, so at each lockstep
// point at most 3 words remain and the FIFO never holds more than 7.
struct PhiloxStream {
  uint64_t k0, k1, c0, c1;
  unsigned head, tail;   // words consumed / produced
  uint64_t* fifo;        // 8 words (stride-padded row of a shared array)

  __device__ void init(uint64_t key_lo, uint64_t key_hi, uint64_t* f) {
    k0 = key_lo; k1 = key_hi; c0 = 0; c1 = 0; head = 0; tail = 0; fifo = f;
  }
  __device__ void refill() {
    if (++c0 == 0) ++c1;
    uint64_t x0 = c0, x1 = c1, x2 = 0, x3 = 0, y0 = k0, y1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t hi0 = __umul64hi(kM0, x0), lo0 = kM0 * x0;
      const uint64_t hi1 = __umul64hi(kM1, x2), lo1 = kM1 * x2;
      const uint64_t n0 = hi1 ^ x1 ^ y0, n2 = hi0 ^ x3 ^ y1;
      x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
      y0 += kW0; y1 += kW1;
    }
    fifo[tail & 7] = x0; fifo[(tail + 1) & 7] = x1; fifo[(tail + 2) & 7] = x2; fifo[(tail + 3) & 7] = x3;
    tail += 4;
  }
  __device__ uint64_t next64() {
    if (head == tail) refill();
    return fifo[(head++) & 7];
  }
  __device__ double next_double() {
    return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
};

// numpy random_standard_normal (distributions.c): one 64-bit word = 8 layer
// bits, 1 sign bit, 52 mantissa bits; tail (layer 0) by -log1p(-U) pairs;
// wedge test against exp(-x^2/2).
__device__ double standard_normal(PhiloxStream& s, const unsigned long long* __restrict__ ki,
                                  const double* __restrict__ wi) {
  for (;;) {
    uint64_t r = s.next64();
    const int idx = static_cast<int>(r & 0xff);
    r >>= 8;
    const bool neg = r & 1;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn(static_cast<double>(rabs), wi[idx]);
    if (neg) x = -x;
    if (rabs < ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-kZigInvR, log1p(-s.next_double()));
        const double yy = -log1p(-s.next_double());
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 1) ? -__dadd_rn(kZigR, xx) : __dadd_rn(kZigR, xx);
      }
    } else {
      const double u = s.next_double();
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(kZigFi[idx - 1], kZigFi[idx]), u), kZigFi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    }
  }
}

constexpr int NB = 128;  // samples per block
constexpr int SEG = 16;  // values per sample staged between coalesced writes

__global__ void __launch_bounds__(NB, 8)
normals_kernel(uint64_t seed, int64_t first, int64_t n, int d, int with_noise, double* __restrict__ x64,
               float* __restrict__ x32, double* __restrict__ nz64) {
  __shared__ double stage[NB][SEG + 1];
  __shared__ uint64_t s_fifo[NB][9];
  __shared__ unsigned long long s_ki[256];
  __shared__ double s_wi[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 256; i += NB) { s_ki[i] = kZigKi[i]; s_wi[i] = kZigWi[i]; }
  __syncthreads();
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * NB;
  const bool valid = i0 + tid < n;
  PhiloxStream s;
  // key = (seed << 64) + index (synthgen.py:46), index < 2^63
  s.init(static_cast<uint64_t>(first + i0 + tid), seed, s_fifo[tid]);
  unsigned g = 0;  // normals drawn so far (both rows): lockstep refill every 4
  for (int pass = 0; pass < (with_noise ? 2 : 1); ++pass) {
    double* out = pass ? nz64 : x64;
    for (int j0 = 0; j0 < d; j0 += SEG) {
      const int cnt = min(SEG, d - j0);
      if (valid) {
        for (int t = 0; t < cnt; ++t, ++g) {
          if ((g & 3) == 0 && s.tail - s.head < 4) s.refill();
          stage[tid][t] = standard_normal(s, s_ki, s_wi);
        }
      }
      __syncthreads();
      // warp w writes the SEG-value segments of samples w*32 .. w*32+31,
      // 32 / SEG samples per store instruction
      for (int rr = 0; rr < 32; rr += 32 / SEG) {
        const int row = warp * 32 + rr + lane / SEG, col = lane % SEG;
        const int64_t gi = i0 + row;
        if (gi < n && col < cnt) {
          const double v = stage[row][col];
          const int64_t o = gi * d + j0 + col;
          if (out) out[o] = v;
          if (pass == 0 && x32) x32[o] = __double2float_rn(v);
        }
      }
      __syncthreads();
    }
  }
}

// one warp per row; dynamic smem: plan + per warp (padded row, leaf sums)
__global__ void layer_norm_np_kernel(const double* __restrict__ x, int64_t n, int d, double eps,
                                     double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  PwPlan& plan = *reinterpret_cast<PwPlan*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int row_words = pad(d - 1) + 1;
  const int LEN = d;
  double* base = reinterpret_cast<double*>(smem + ((sizeof(PwPlan) + 15) & ~size_t(15)));
  double* row = base + static_cast<size_t>(warp) * (row_words + leaf_cap(LEN));
  double* leafsum = row + row_words;
  if (threadIdx.x == 0) {
    plan.n_leaves = 0;
    plan.n_prog = 0;
    pw_build(plan, 0, d);
  }
  __syncthreads();
  const double dd = static_cast<double>(d);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * nwarps + warp; r < n; r += static_cast<int64_t>(gridDim.x) * nwarps) {
    const double* xr = x + r * d;
    if ((d & 1) == 0 && (reinterpret_cast<uintptr_t>(xr) & 15) == 0) {
      // 16-byte streaming loads, 16 in flight per lane
      const double2* x2 = reinterpret_cast<const double2*>(xr);
#pragma unroll 16
      for (int i = lane; i < d / 2; i += 32) {
        const double2 v = __ldcs(x2 + i);
        row[pad(2 * i)] = v.x;
        row[pad(2 * i + 1)] = v.y;
      }
    } else {
#pragma unroll 8
      for (int i = lane; i < d; i += 32) row[pad(i)] = __ldcs(xr + i);
    }
    __syncwarp();
    const double mean = __ddiv_rn(warp_pairwise<0>(row, plan, 0.0, leafsum, lane), dd);
    const double var = __ddiv_rn(warp_pairwise<1>(row, plan, mean, leafsum, lane), dd);
    const double den = __dsqrt_rn(__dadd_rn(var, eps));
    double* orow = out + r * d;
    for (int i = lane; i < d; i += 32) orow[i] = __ddiv_rn(__dsub_rn(row[pad(i)], mean), den);
    __syncwarp();
  }
}

// softmax (numpy order) -> float32 scores -> top-k of the float32 values.
// One warp per row, lane l holds experts l, l+32, ... (E <= 32 * PL).
template <int PL>
__global__ void teacher_finish_kernel(const double* __restrict__ logits, int64_t n, int E, int k,
                                      float* __restrict__ scores, int32_t* __restrict__ topk) {
  extern __shared__ __align__(16) unsigned char smem[];
  PwPlan& plan = *reinterpret_cast<PwPlan*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int row_words = pad(E - 1) + 1;
  const int LEN = E;
  double* base = reinterpret_cast<double*>(smem + ((sizeof(PwPlan) + 15) & ~size_t(15)));
  double* row = base + static_cast<size_t>(warp) * (row_words + leaf_cap(LEN));
  double* leafsum = row + row_words;
  if (threadIdx.x == 0) {
    plan.n_leaves = 0;
    plan.n_prog = 0;
    pw_build(plan, 0, E);
  }
  __syncthreads();
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * nwarps + warp; r < n; r += static_cast<int64_t>(gridDim.x) * nwarps) {
    const double* zr = logits + r * E;
    double zv[PL];
    double mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int e = q * 32 + lane;
      zv[q] = e < E ? zr[e] : -INFINITY;
      mx = fmax(mx, zv[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int e = q * 32 + lane;
      if (e < E) {
        zv[q] = exp(__dsub_rn(zv[q], mx));
        row[pad(e)] = zv[q];
      }
    }
    __syncwarp();
    const double se = warp_pairwise<0>(row, plan, 0.0, leafsum, lane);
    float sv[PL];
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int e = q * 32 + lane;
      sv[q] = e < E ? __double2float_rn(__ddiv_rn(zv[q], se)) : -INFINITY;
      if (e < E) scores[r * E + e] = sv[q];
    }
    // top-k: k rounds of warp argmax (value, then lower index); mark taken
    uint32_t taken = 0;
    for (int s = 0; s < k; ++s) {
      float best = -INFINITY;
      int bi = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        const int e = q * 32 + lane;
        if (e < E && !((taken >> q) & 1u) && (sv[q] > best || (sv[q] == best && e < bi))) { best = sv[q]; bi = e; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    }
    // ascending ids: ballot prefix over expert order
    int cnt = 0;
    int32_t* orow = topk + r * k;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const bool t = (taken >> q) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, t);
      if (t) orow[cnt + __popc(bal & ((1u << lane) - 1u))] = q * 32 + lane;
      cnt += __popc(bal);
    }
  }
}

// core.softmax (core.py:19-24) over fp64 rows in numpy's order: max,
// subtract, exp, 0 + pairwise_sum, divide. One warp per row, the row staged
// in shared memory (any E up to the plan's leaf capacity).
__global__ void softmax_np_kernel(const double* __restrict__ z, int64_t n, int E, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  PwPlan& plan = *reinterpret_cast<PwPlan*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int row_words = pad(E - 1) + 1;
  const int LEN = E;
  double* base = reinterpret_cast<double*>(smem + ((sizeof(PwPlan) + 15) & ~size_t(15)));
  double* row = base + static_cast<size_t>(warp) * (row_words + leaf_cap(LEN));
  double* leafsum = row + row_words;
  if (threadIdx.x == 0) {
    plan.n_leaves = 0;
    plan.n_prog = 0;
    pw_build(plan, 0, E);
  }
  __syncthreads();
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * nwarps + warp; r < n; r += static_cast<int64_t>(gridDim.x) * nwarps) {
    const double* zr = z + r * E;
    double mx = -INFINITY;
    for (int e = lane; e < E; e += 32) {
      const double v = zr[e];
      row[pad(e)] = v;
      mx = fmax(mx, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __syncwarp();
    for (int e = lane; e < E; e += 32) row[pad(e)] = exp(__dsub_rn(row[pad(e)], mx));
    __syncwarp();
    const double se = warp_pairwise<0>(row, plan, 0.0, leafsum, lane);
    double* orow = out + r * E;
    for (int e = lane; e < E; e += 32) orow[e] = __ddiv_rn(row[pad(e)], se);
    __syncwarp();
  }
}

size_t plan_smem(int nwarps, int len) {
  return ((sizeof(PwPlan) + 15) & ~size_t(15)) +
         static_cast<size_t>(nwarps) * static_cast<size_t>(pad(len - 1) + 1 + leaf_cap(len)) * sizeof(double);
}

}  // namespace sg
}  // namespace moep

using namespace moep::sg;

extern "C" {

int moep_teacher_normals(uint64_t seed, int64_t first_index, int64_t n, int32_t d, int32_t with_noise,
                         double* x64, float* x32, double* noise64, void* stream) {
  if (n <= 0 || d <= 0) return MOEP_ESHAPE;
  if (first_index < 0 || (!x64 && !x32) || (with_noise && !noise64)) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (n + NB - 1) / NB;
  if (blocks > 0x7fffffff) return MOEP_ESHAPE;
  normals_kernel<<<static_cast<unsigned>(blocks), NB, 0, st>>>(seed, first_index, n, d, with_noise, x64, x32,
                                                               noise64);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_layer_norm_np(const double* x, int64_t n, int32_t d, double eps, double* out, void* stream) {
  if (n <= 0 || d < 2) return MOEP_ESHAPE;
  if (leaf_cap(d) > kMaxLeaves) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int nwarps = 16;
  while (nwarps > 1 && plan_smem(nwarps, d) > 220 * 1024) --nwarps;
  const size_t sm = plan_smem(nwarps, d);
  if (sm > 227 * 1024) return MOEP_EUNSUPPORTED;
  if (cudaFuncSetAttribute(layer_norm_np_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sm)) != cudaSuccess)
    return MOEP_ELAUNCH;
  const int64_t want = (n + nwarps - 1) / nwarps;
  const int grid = static_cast<int>(want < 8 * moep_num_sms() ? want : 8 * moep_num_sms());
  layer_norm_np_kernel<<<grid, nwarps * 32, sm, st>>>(x, n, d, eps, out);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_teacher_finish(const double* logits, int64_t n, int32_t n_experts, int32_t k, float* scores,
                        int32_t* topk, void* stream) {
  if (n <= 0 || n_experts <= 0) return MOEP_ESHAPE;
  if (k < 1 || k > n_experts || n_experts > 256) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nwarps = 8;
  const size_t sm = plan_smem(nwarps, n_experts);
  const int64_t want = (n + nwarps - 1) / nwarps;
  const int grid = static_cast<int>(want < 8 * moep_num_sms() ? want : 8 * moep_num_sms());
#define MOEP_K11F(PL)                                                                                   \
  do {                                                                                                  \
    if (cudaFuncSetAttribute(teacher_finish_kernel<PL>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             static_cast<int>(sm)) != cudaSuccess)                                      \
      return MOEP_ELAUNCH;                                                                              \
    teacher_finish_kernel<PL><<<grid, nwarps * 32, sm, st>>>(logits, n, n_experts, k, scores, topk);    \
  } while (0)
  if (n_experts <= 32) MOEP_K11F(1);
  else if (n_experts <= 64) MOEP_K11F(2);
  else if (n_experts <= 128) MOEP_K11F(4);
  else MOEP_K11F(8);
#undef MOEP_K11F
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_softmax_np(const double* z, int64_t n, int32_t E, double* out, void* stream) {
  if (n <= 0 || E <= 0) return MOEP_ESHAPE;
  if (leaf_cap(E) > kMaxLeaves) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int nwarps = 8;
  while (nwarps > 1 && plan_smem(nwarps, E) > 200 * 1024) --nwarps;
  const size_t sm = plan_smem(nwarps, E);
  if (sm > 227 * 1024) return MOEP_EUNSUPPORTED;
  if (cudaFuncSetAttribute(softmax_np_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sm)) != cudaSuccess)
    return MOEP_ELAUNCH;
  const int64_t want = (n + nwarps - 1) / nwarps;
  const int grid = static_cast<int>(want < 8 * moep_num_sms() ? want : 8 * moep_num_sms());
  softmax_np_kernel<<<grid, nwarps * 32, sm, st>>>(z, n, E, out);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // extern "C"
