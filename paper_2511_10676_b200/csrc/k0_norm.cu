// k0_norm.cu — K0, the pre-attention input norm at the hook point (the
// reference predictor consumes the decoder's `input_layernorm` output,
// exporter hooks.py:19,113-114; its only norm is core.layer_norm, core.py:57-68).
//
// x_hat = bf16_rne( norm(x) ), statistics in float64 in NUMPY'S reduction
// order, so the output is bit-identical to oracle.input_norm_bf16 by
// construction (not by luck):
//   rmsnorm:   ms = mean(x*x); y = x / sqrt(ms + eps); y *= gamma
//   layernorm: mu = mean(x); var = mean((x - mu)^2); y = (x - mu) / sqrt(var + eps);
//              y *= gamma; y += beta                          (every op RN, no FMA)
// numpy's mean is 0 + pairwise_sum / d (loops_utils.h.src: leaves of <= 128
// elements with 8 accumulators, halving splits rounded to multiples of 8).
//
// Fast path (bf16 rows, d = 128 * B, B in {4, 8, 16, 32}: every split halves
// exactly, so the tree is balanced over d/128 leaves): one LANE per numpy leaf
// (its 128 elements are one contiguous 256-byte piece: the warp's rows are
// loaded with coalesced 16-byte loads into per-lane shared-memory staging,
// x_hat goes back out the same way), the leaf's 8 accumulators in numpy's order, leaves
// combined by xor-shuffles (the balanced tree; fp64 add is commutative). x is
// read once from HBM and x_hat written once: 4 bytes per element.
// The per-element divide is replaced by a multiply with the correctly rounded
// reciprocal; the result differs from numpy's quotient chain by at most
// 2^-49 (|g| + |res|), so its bf16 rounding can differ only when the fp64
// value lies within that distance of a bf16 rounding midpoint — an integer
// test on the 45 dropped mantissa bits. Those elements (and bf16-subnormal /
// huge ones) redo numpy's exact chain (divide, *gamma, +beta) before rounding.
//
// General path (any d, bf16 / fp32 / fp64 input): one warp per row staged in
// shared memory, numpy's tree from pairwise.cuh, numpy's exact chain per element.
// kind 0 (cast): x -> bf16 RNE with "not bf16-representable" and non-finite
// row counts (the engine's choice between K1 and the fp64 path).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include "common.cuh"
#include "pairwise.cuh"

namespace moep {
namespace k0 {

__device__ __forceinline__ double bf16_lo(uint32_t w) { return static_cast<double>(__uint_as_float(w << 16)); }
__device__ __forceinline__ double bf16_hi(uint32_t w) { return static_cast<double>(__uint_as_float(w & 0xffff0000u)); }

__device__ __forceinline__ uint16_t f64_to_bf16_bits(double v) {
  uint16_t r;
  asm("cvt.rn.bf16.f64 %0, %1;" : "=h"(r) : "d"(v));
  return r;
}

template <typename T>
__device__ __forceinline__ double ldx(const void* p, int64_t i) {
  if constexpr (sizeof(T) == 2)
    return static_cast<double>(__uint_as_float(static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(p)[i]) << 16));
  else
    return static_cast<double>(reinterpret_cast<const T*>(p)[i]);
}

// ---------------------------------------------------------------- fast path
__device__ __forceinline__ double elem8(const uint4& q, int j) {
  const uint32_t w = (j >> 1) == 0 ? q.x : (j >> 1) == 1 ? q.y : (j >> 1) == 2 ? q.z : q.w;
  return (j & 1) ? bf16_hi(w) : bf16_lo(w);
}
__device__ __forceinline__ uint32_t word8(const uint4& q, int j2) {
  return j2 == 0 ? q.x : j2 == 1 ? q.y : j2 == 2 ? q.z : q.w;
}
// bf16 -> fp64 by integer ops (no XU conversion): exact for normal bf16 values;
// zeros / subnormals / inf / nan are caught per row by special2() and that row
// is redone with the exact conversion
__device__ __forceinline__ double bf16lo_f64_fast(uint32_t w) {
  return __hiloint2double(static_cast<int>((((w & 0x7fffu) << 13) + 0x38000000u) | ((w & 0x8000u) << 16)), 0);
}
__device__ __forceinline__ double bf16hi_f64_fast(uint32_t w) {
  return __hiloint2double(static_cast<int>((((w >> 3) & 0x0fffe000u) + 0x38000000u) | (w & 0x80000000u)), 0);
}
// nonzero when either bf16 half of w has a zero / all-ones exponent field (a
// rare false positive just sends the row down the exact-conversion path)
__device__ __forceinline__ uint32_t special2(uint32_t w) {
  const uint32_t ex = w & 0x7f807f80u;
  return ((ex + 0x00800080u) | (ex - 0x00800080u)) & 0x80008000u;
}

// |bf16| -> fp64 by integer ops (sign dropped: the operand of a square)
__device__ __forceinline__ double bf16lo_abs_f64(uint32_t w) {
  return __hiloint2double(static_cast<int>((w & 0x7fffu) * 8192u + 0x38000000u), 0);
}
__device__ __forceinline__ double bf16hi_abs_f64(uint32_t w) {
  return __hiloint2double(static_cast<int>(((w & 0x7fff0000u) >> 3) + 0x38000000u), 0);
}
// packed fp32x2 arithmetic (sm_100: one instruction per pair, round to nearest)
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}

// KIND 1 rmsnorm, 2 layernorm. B lanes per row, 32 / B rows per warp. Each
// lane stages its leaf (256 B, padded to 272 B so a quarter-warp's 16-byte
// shared loads hit distinct banks; an XOR swizzle without the pad measured 5 %
// slower on layernorm) and re-reads only its own staging: no barrier inside
// the row loop. Shared memory holds only the gamma / beta rows the kernel uses.
//
// Statistics: numpy's order in fp64 (bit-identical mean / var by
// construction). Output, level 1: fp32 arithmetic with the fp32-rounded
// statistics / gamma / beta, |res32 - numpy's value| <= E with
//   E = 2^-20 (r |gamma| (|mu| + |x - mu|) + |beta| + |res|)   (>= 2.5x the
// sum of the fp32 rounding errors of mu, r, gamma, beta and the 3-4 fp32 ops);
// when no bf16 rounding midpoint lies within E of res32 (and res32 is in the
// bf16 normal range, E < 2^-10 |res|), bf16_rn(res32) == bf16_rn(numpy's).
// Level 2 (~1 element in 4000): numpy's fp64 chain with the exact statistics.
constexpr int kStageU4 = 17;  // per-lane leaf staging: 16 chunks + 1 pad (bank-conflict-free quarter warps)
// Two block shapes: the register-staged loads (256 threads, 128 registers,
// two blocks per SM) and, for rmsnorm, cp.async staging straight into shared
// memory (no load registers: 128 threads, 96 registers, five blocks per SM,
// 20 warps instead of 16 to hide the load latency: 2.10 -> 2.00 ms per
// 1M x 2048). layernorm keeps the first shape (its extra statistics pass
// spills at 96 registers: 3.83 -> 5.02 ms).
template <bool CPA>
struct NormShape {
  static constexpr int kThreads = CPA ? 128 : 256;
  static constexpr int kMinBlocks = CPA ? 5 : 2;
};
constexpr int kNormThreads = 256;


template <int B, int KIND, bool GAMMA, bool BETA, bool FORCE = false, bool CPA = false>
__global__ void __launch_bounds__(NormShape<CPA>::kThreads, NormShape<CPA>::kMinBlocks)
norm_fast_kernel(const uint16_t* __restrict__ x, int64_t n, const double* __restrict__ gamma,
                 const double* __restrict__ beta, double eps, uint16_t* __restrict__ out, int* status) {
  constexpr int RPW = 32 / B;
  constexpr int D = 128 * B;
  // gamma32 [D], beta32 [D], leaf staging [warps][32][17] uint4 (level 2 reads
  // the fp64 gamma / beta from global memory: rare, L1/L2 resident)
  // per leaf a 132-float row (528 B): the 16-byte loads of 8 consecutive
  // leaves hit distinct banks (an unpadded 128 stride puts every lane on one bank)
  constexpr int GP = 132;
  extern __shared__ __align__(16) float sg32[];
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    if (GAMMA) sg32[(i >> 7) * GP + (i & 127)] = static_cast<float>(gamma[i]);
    if (BETA) sg32[(GAMMA ? B * GP : 0) + (i >> 7) * GP + (i & 127)] = static_cast<float>(beta[i]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane / B, li = lane % B;
  constexpr int NREG = (GAMMA ? 1 : 0) + (BETA ? 1 : 0);  // gamma / beta rows present
  uint4* const stage = reinterpret_cast<uint4*>(sg32 + NREG * B * GP) + (threadIdx.x >> 5) * 32 * kStageU4;
  uint4* const my = stage + lane * kStageU4;
  const int64_t wg = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const double dd = static_cast<double>(D);
  const double* gl = GAMMA ? gamma + 128 * li : nullptr;
  const double* bl = BETA ? beta + 128 * li : nullptr;
  const float4* gl32 = reinterpret_cast<const float4*>(sg32 + GP * li);
  const float4* bl32 = reinterpret_cast<const float4*>(sg32 + (GAMMA ? B * GP : 0) + GP * li);
  const unsigned grp = (B == 32) ? 0xffffffffu : (((1u << B) - 1u) << (sub * B));
  uint4 v[16];
  auto fetch = [&](int64_t rs) {
    const int64_t rh = n - rs < RPW ? n - rs : RPW;
    const uint4* src = reinterpret_cast<const uint4*>(x + rs * D);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int idx = t * 32 + lane;
      // a ragged tail's padding rows repeat the last row (a zero row would take
      // the exact-conversion and level-2 paths: 4x the time of a decode-size call)
      const int si = idx / (D / 8) < rh ? idx : static_cast<int>(rh - 1) * (D / 8) + idx % (D / 8);
      v[t] = rs < n ? __ldcs(src + si) : make_uint4(0, 0, 0, 0);
    }
  };
  for (int64_t r0 = wg * RPW; r0 < n; r0 += nw * RPW) {
    const int64_t row = r0 + sub;
    const bool valid = row < n;
    // the warp's RPW consecutive rows are one contiguous 8 KB piece: coalesced
    // 16-byte loads into the owners' staging (chunk q of a row -> leaf q / 16).
    // (Measured slower: a double-buffered cp.async variant with 4 warps per
    // block, 2.95 vs 2.16 ms per 1M x 2048 rmsnorm, and a register double
    // buffer of the next row group, 2.36 ms at 128 registers (spills) / 2.77 ms
    // at one block per SM, against 2.12 ms.)
    const int64_t rows_here = n - r0 < RPW ? n - r0 : RPW;
    if constexpr (CPA) {
      const uint4* src = reinterpret_cast<const uint4*>(x + r0 * D);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int idx = t * 32 + lane;
        uint4* dst = stage + (idx >> 4) * kStageU4 + (idx & 15);
        // padding rows of a ragged tail repeat the last row (see fetch)
        const int si = idx / (D / 8) < rows_here ? idx : static_cast<int>(rows_here - 1) * (D / 8) + idx % (D / 8);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                     "l"(src + si) : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
      fetch(r0);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int idx = t * 32 + lane;
        stage[(idx >> 4) * kStageU4 + (idx & 15)] = v[t];  // owner lane = row * B + leaf = idx / 16
      }
    }
    __syncwarp();
    // leaf sum of op(x) in numpy's order: r[j] starts at element j, then += element 8c + j
    uint32_t spec = 0;
    auto leaf_fast = [&](auto op) -> double {
      double r[8];
#pragma unroll 4
      for (int c = 0; c < 16; ++c) {
        const uint4 q = my[c];
#pragma unroll
        for (int j2 = 0; j2 < 4; ++j2) {
          const uint32_t w = word8(q, j2);
          spec |= special2(w);
          const double e0 = op(bf16lo_f64_fast(w)), e1 = op(bf16hi_f64_fast(w));
          if (c == 0) { r[2 * j2] = e0; r[2 * j2 + 1] = e1; }
          else { r[2 * j2] = __dadd_rn(r[2 * j2], e0); r[2 * j2 + 1] = __dadd_rn(r[2 * j2 + 1], e1); }
        }
      }
      return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    };
    auto leaf_sq_fast = [&]() -> double {
      // rmsnorm: x*x is exact in fp64 (8-bit mantissas), so fma(x, x, r) rounds
      // once exactly like numpy's r + (x*x); the zero / subnormal / inf / nan
      // test is OR-accumulated and masked once per leaf
      double r[8];
      uint32_t sp = 0;
#pragma unroll 4
      for (int c = 0; c < 16; ++c) {
        const uint4 q = my[c];
#pragma unroll
        for (int j2 = 0; j2 < 4; ++j2) {
          const uint32_t w = word8(q, j2);
          const uint32_t ex = w & 0x7f807f80u;
          sp |= (ex + 0x00800080u) | (ex - 0x00800080u);
          const double e0 = bf16lo_abs_f64(w), e1 = bf16hi_abs_f64(w);
          if (c == 0) { r[2 * j2] = __dmul_rn(e0, e0); r[2 * j2 + 1] = __dmul_rn(e1, e1); }
          else { r[2 * j2] = __fma_rn(e0, e0, r[2 * j2]); r[2 * j2 + 1] = __fma_rn(e1, e1, r[2 * j2 + 1]); }
        }
      }
      spec |= sp & 0x80008000u;
      return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    };
    auto leaf_exact = [&](auto op) -> double {
      double r[8];
#pragma unroll 2
      for (int c = 0; c < 16; ++c) {
        const uint4 q = my[c];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = c == 0 ? op(elem8(q, j)) : __dadd_rn(r[j], op(elem8(q, j)));
      }
      return __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    };
    auto tree = [&](double s) -> double {  // balanced combine over the row's B leaves, then 0 + total
#pragma unroll
      for (int o = 1; o < B; o <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
      return __dadd_rn(0.0, s);
    };
    auto sq = [](double e) { return __dmul_rn(e, e); };
    auto id = [](double e) { return e; };
    double mu = 0.0, stat;
    if (KIND == 2) {
      mu = __ddiv_rn(tree(leaf_fast(id)), dd);
      stat = __ddiv_rn(tree(leaf_fast([&](double e) { const double t = __dsub_rn(e, mu); return sq(t); })), dd);
    } else {
      stat = __ddiv_rn(tree(leaf_sq_fast()), dd);
    }
    bool bad = false;
    // a zero / subnormal / inf / nan element somewhere in the warp's rows: the
    // whole warp redoes its statistics with the exact conversion (warp-uniform:
    // the leaf trees shuffle across the full warp)
    if (__any_sync(0xffffffffu, spec != 0)) {
      if (lane == 0) atomicAdd(status + 1, 1);  // diagnostic: warps that took the exact-conversion pass
      bool nonfin = false;
      auto chk = [&](double e) { nonfin |= !isfinite(e); return e; };
      if (KIND == 2) {
        mu = __ddiv_rn(tree(leaf_exact(chk)), dd);
        stat = __ddiv_rn(tree(leaf_exact([&](double e) { const double t = __dsub_rn(e, mu); return sq(t); })), dd);
      } else {
        stat = __ddiv_rn(tree(leaf_exact([&](double e) { return sq(chk(e)); })), dd);
      }
      bad = nonfin;
    }
    const double sigma = __dsqrt_rn(__dadd_rn(stat, eps));
    const double rinv = __drcp_rn(sigma);
    const float r32 = static_cast<float>(rinv), mu32 = static_cast<float>(mu);
    const float amu = fabsf(mu32);
#pragma unroll 2
    for (int c = 0; c < 16; ++c) {
      const uint4 q = my[c];
      float gv[8], bv[8];
      if (GAMMA) {
        const float4 a = gl32[2 * c], b = gl32[2 * c + 1];
        gv[0] = a.x; gv[1] = a.y; gv[2] = a.z; gv[3] = a.w; gv[4] = b.x; gv[5] = b.y; gv[6] = b.z; gv[7] = b.w;
      }
      if (BETA) {
        const float4 a = bl32[2 * c], b = bl32[2 * c + 1];
        bv[0] = a.x; bv[1] = a.y; bv[2] = a.z; bv[3] = a.w; bv[4] = b.x; bv[5] = b.y; bv[6] = b.z; bv[7] = b.w;
      }
      uint32_t o[4];
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        const uint32_t w = word8(q, j2);
        float resv[2];
        bool amb[2];
        // the pair (lo, hi) in packed fp32x2 ops: same RN results as the scalar chain
        const float2 x2 = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
        const float2 dl2 = KIND == 2 ? sub2(x2, make_float2(mu32, mu32)) : x2;
        const float2 y2 = mul2(dl2, make_float2(r32, r32));
        const float2 g2 = GAMMA ? mul2(y2, make_float2(gv[2 * j2], gv[2 * j2 + 1])) : y2;
        const float2 res2 = BETA ? add2(g2, make_float2(bv[2 * j2], bv[2 * j2 + 1])) : g2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float dl = h ? dl2.y : dl2.x;
          const float gm = GAMMA ? gv[2 * j2 + h] : 1.0f;
          const float res = h ? res2.y : res2.x;
          const uint32_t rb = __float_as_uint(res);
          const uint32_t ex = (rb >> 23) & 0xffu;
          bool a;
          if (KIND == 2) {
            // E = 2^-20 (r |gamma| (|mu| + |x - mu|) + |beta| + |res|)
            const float E = 9.5367431640625e-07f * (r32 * fabsf(gm) * (amu + fabsf(dl)) +
                                                     (BETA ? fabsf(bv[2 * j2 + h]) : 0.0f) + fabsf(res));
            const float mid = __uint_as_float((rb & 0xffff0000u) | 0x8000u);
            a = E > 9.765625e-04f * fabsf(res) || fabsf(res - mid) <= E;
          } else {
            // |res32 - numpy's| <= 4.02 fp32 ulps: within 16 ulps of the midpoint
            a = ((rb - 0x7ff0u) & 0xffffu) <= 32u;
          }
          amb[h] = FORCE || ex - 2u > 250u || a;
          resv[h] = res;
        }
        uint32_t pk;
        {
          const __nv_bfloat162 p2 = __floats2bfloat162_rn(resv[0], resv[1]);
          pk = *reinterpret_cast<const uint32_t*>(&p2);
        }
        if (amb[0] | amb[1]) {  // level 2: numpy's fp64 chain with the exact statistics
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!amb[h]) continue;
            const int col = 8 * c + 2 * j2 + h;
            const double xd = static_cast<double>(__uint_as_float(h ? (w & 0xffff0000u) : (w << 16)));
            const double dlt = KIND == 2 ? __dsub_rn(xd, mu) : xd;
            double yv = __ddiv_rn(dlt, sigma);
            if (GAMMA) yv = __dmul_rn(yv, __ldg(gl + col));
            if (BETA) yv = __dadd_rn(yv, __ldg(bl + col));
            const uint32_t bits = f64_to_bf16_bits(yv);
            pk = h ? ((pk & 0x0000ffffu) | (bits << 16)) : ((pk & 0xffff0000u) | bits);
          }
        }
        o[j2] = pk;
      }
      my[c] = make_uint4(o[0], o[1], o[2], o[3]);  // x_hat overwrites the chunk it came from
    }
    __syncwarp();
    {  // coalesced stores of the warp's rows
      uint4* dst = reinterpret_cast<uint4*>(out + r0 * D);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int idx = t * 32 + lane;
        if (idx / (D / 8) < rows_here)
          __stcs(dst + idx, stage[(idx >> 4) * kStageU4 + (idx & 15)]);
      }
      __syncwarp();
    }
    // one status update per row (lane li == 0 of the row's group)
    const bool any_bad = (__ballot_sync(0xffffffffu, bad && valid) & grp) != 0;
    if (any_bad && li == 0) atomicAdd(status, 1);
  }
}

// ------------------------------------------------------------- general path
template <typename T>
__global__ void norm_general_kernel(const void* __restrict__ x, int64_t n, int d, int kind,
                                    const double* __restrict__ gamma, const double* __restrict__ beta, double eps,
                                    uint16_t* __restrict__ out, int* status) {
  using namespace moep::sg;
  extern __shared__ __align__(16) unsigned char smem[];
  PwPlan& plan = *reinterpret_cast<PwPlan*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int row_words = pad(d - 1) + 1;
  double* base = reinterpret_cast<double*>(smem + ((sizeof(PwPlan) + 15) & ~size_t(15)));
  double* row = base + static_cast<size_t>(warp) * (row_words + leaf_cap(d));
  double* leafsum = row + row_words;
  if (threadIdx.x == 0) {
    plan.n_leaves = 0;
    plan.n_prog = 0;
    pw_build(plan, 0, d);
  }
  __syncthreads();
  const double dd = static_cast<double>(d);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * nwarps + warp; r < n;
       r += static_cast<int64_t>(gridDim.x) * nwarps) {
    bool bad = false;
    for (int i = lane; i < d; i += 32) {
      const double v = ldx<T>(x, r * d + i);
      bad |= !isfinite(v);
      row[pad(i)] = v;
    }
    __syncwarp();
    double mu = 0.0, stat;
    if (kind == 2) {
      mu = __ddiv_rn(warp_pairwise<0>(row, plan, 0.0, leafsum, lane), dd);
      stat = __ddiv_rn(warp_pairwise<1>(row, plan, mu, leafsum, lane), dd);
    } else {
      stat = __ddiv_rn(warp_pairwise<2>(row, plan, 0.0, leafsum, lane), dd);
    }
    const double sigma = __dsqrt_rn(__dadd_rn(stat, eps));
    for (int i = lane; i < d; i += 32) {
      const double dlt = kind == 2 ? __dsub_rn(row[pad(i)], mu) : row[pad(i)];
      double y = __ddiv_rn(dlt, sigma);
      if (gamma) y = __dmul_rn(y, gamma[i]);
      if (beta && kind == 2) y = __dadd_rn(y, beta[i]);
      out[r * d + i] = f64_to_bf16_bits(y);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicAdd(status, 1);
    __syncwarp();
  }
}

// ---------------------------------------------------------------- kind 0
template <typename T>
__global__ void __launch_bounds__(256)
cast_kernel(const void* __restrict__ x, int64_t n, int d, uint16_t* __restrict__ out, int* status) {
  const int64_t total = n * d;
  int bad = 0, inexact = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = ldx<T>(x, i);
    const uint16_t b = f64_to_bf16_bits(v);
    bad |= !isfinite(v);
    inexact |= static_cast<double>(__uint_as_float(static_cast<uint32_t>(b) << 16)) != v;
    out[i] = b;
  }
  bad = __syncthreads_or(bad);
  inexact = __syncthreads_or(inexact);
  if (threadIdx.x == 0) {
    if (bad) atomicAdd(status, 1);
    if (inexact) atomicAdd(status + 1, 1);
  }
}

// blocks-per-SM cache: one row of 64 devices per kernel (a few dozen kernels)
inline int* occupancy_slot(const void* kern, int dev) {
  static const void* keys[64];
  static int vals[64][64];
  if (dev < 0 || dev >= 64) return nullptr;
  for (int i = 0; i < 64; ++i) {
    if (keys[i] == kern) return &vals[i][dev];
    if (!keys[i]) { keys[i] = kern; return &vals[i][dev]; }
  }
  return nullptr;
}

template <int B>
int launch_fast(const uint16_t* x, int64_t n, int kind, bool force, const double* gamma, const double* beta,
                double eps, uint16_t* out, int* status, cudaStream_t st) {
  int rc = MOEP_OK;
  auto go = [&](auto kern, int nreg, int threads) {
    const int rows_per_block = (threads / 32) * (32 / B);
    const int64_t want = (n + rows_per_block - 1) / rows_per_block;
    const size_t sm = static_cast<size_t>(nreg * 132 * B) * sizeof(float) + (threads / 32) * 32 * kStageU4 * 16;
    // one resident wave (grid-stride over row groups): blocks per SM from the
    // occupancy calculator, cached per (kernel, device)
    int dev = 0;
    cudaGetDevice(&dev);
    int* slot = occupancy_slot(reinterpret_cast<const void*>(kern), dev);
    if (!slot) { rc = MOEP_ELAUNCH; return; }
    if (!*slot) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(slot, kern, threads, sm);
      if (e != cudaSuccess || *slot < 1) {
        fprintf(stderr, "moep_input_norm: %s (smem %zu, blocks/SM %d)\n", cudaGetErrorString(e), sm, *slot);
        *slot = 0;
        rc = MOEP_ELAUNCH;
        return;
      }
    }
    const int64_t cap = static_cast<int64_t>(*slot) * moep_num_sms();
    const int grid = static_cast<int>(want < cap ? want : cap);
    kern<<<grid, threads, sm, st>>>(x, n, gamma, beta, eps, out, status);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      fprintf(stderr, "moep_input_norm: %s\n", cudaGetErrorString(e));
      rc = MOEP_ELAUNCH;
    }
  };
  if (force) {  // tests: numpy's exact chain for every element (checks the fast path's rounding decision)
    if (kind == 1) go(norm_fast_kernel<B, 1, true, false, true, true>, 1, NormShape<true>::kThreads);
    else go(norm_fast_kernel<B, 2, true, true, true>, 2, kNormThreads);
  } else if (kind == 1) {
    if (gamma) go(norm_fast_kernel<B, 1, true, false, false, true>, 1, NormShape<true>::kThreads);
    else go(norm_fast_kernel<B, 1, false, false, false, true>, 0, NormShape<true>::kThreads);
  } else if (gamma && beta) {
    go(norm_fast_kernel<B, 2, true, true>, 2, kNormThreads);
  } else if (gamma) {
    go(norm_fast_kernel<B, 2, true, false>, 1, kNormThreads);
  } else if (beta) {
    go(norm_fast_kernel<B, 2, false, true>, 1, kNormThreads);
  } else {
    go(norm_fast_kernel<B, 2, false, false>, 0, kNormThreads);
  }
  return rc;
}

template <typename T>
int launch_general(const void* x, int64_t n, int d, int kind, const double* gamma, const double* beta, double eps,
                   uint16_t* out, int* status, cudaStream_t st) {
  using namespace moep::sg;
  const size_t per_warp = static_cast<size_t>(pad(d - 1) + 1 + leaf_cap(d)) * sizeof(double);
  const size_t head = (sizeof(PwPlan) + 15) & ~size_t(15);
  int warps = 8;
  while (warps > 1 && head + warps * per_warp > 200 * 1024) warps >>= 1;
  const size_t sm = head + warps * per_warp;
  if (sm > 227 * 1024) return MOEP_EUNSUPPORTED;
  cudaFuncSetAttribute(norm_general_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  const int64_t want = (n + warps - 1) / warps;
  const int grid = static_cast<int>(want < 4 * moep_num_sms() ? want : 4 * moep_num_sms());
  norm_general_kernel<T><<<grid, 32 * warps, sm, st>>>(x, n, d, kind, gamma, beta, eps, out, status);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // namespace k0
}  // namespace moep

extern "C" int moep_input_norm(const void* x, int32_t x_dtype, int64_t n, int32_t d, int32_t kind,
                               const double* gamma, const double* beta, double eps, void* xhat_bf16,
                               int32_t* status, void* stream) {
  using namespace moep::k0;
  if (n <= 0 || d <= 0) return MOEP_ESHAPE;
  // bit 8 of kind (tests only): the fast path's exact chain for every element
  // (requires gamma, and beta for layernorm)
  const bool force = (kind & 0x100) != 0;
  kind &= 0xff;
  if (kind < 0 || kind > 2 || !status || !x || !xhat_bf16) return MOEP_EARG;
  if (force && (!gamma || (kind == 2 && !beta))) return MOEP_EARG;
  if (x_dtype != MOEP_BF16 && x_dtype != MOEP_F32 && x_dtype != MOEP_F64) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint16_t* out = static_cast<uint16_t*>(xhat_bf16);
  if (kind == 0) {
    const int64_t want = (n * d + 255) / 256;
    const int grid = static_cast<int>(want < 8 * moep_num_sms() ? want : 8 * moep_num_sms());
    if (x_dtype == MOEP_BF16) cast_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(x, n, d, out, status);
    else if (x_dtype == MOEP_F32) cast_kernel<float><<<grid, 256, 0, st>>>(x, n, d, out, status);
    else cast_kernel<double><<<grid, 256, 0, st>>>(x, n, d, out, status);
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (x_dtype == MOEP_BF16 && aligned) {
    const uint16_t* xb = static_cast<const uint16_t*>(x);
    switch (d) {
      case 512: return launch_fast<4>(xb, n, kind, force, gamma, beta, eps, out, status, st);
      case 1024: return launch_fast<8>(xb, n, kind, force, gamma, beta, eps, out, status, st);
      case 2048: return launch_fast<16>(xb, n, kind, force, gamma, beta, eps, out, status, st);
      case 4096: return launch_fast<32>(xb, n, kind, force, gamma, beta, eps, out, status, st);
      default: break;
    }
  }
  if (x_dtype == MOEP_BF16) return launch_general<__nv_bfloat16>(x, n, d, kind, gamma, beta, eps, out, status, st);
  if (x_dtype == MOEP_F32) return launch_general<float>(x, n, d, kind, gamma, beta, eps, out, status, st);
  return launch_general<double>(x, n, d, kind, gamma, beta, eps, out, status, st);
}
