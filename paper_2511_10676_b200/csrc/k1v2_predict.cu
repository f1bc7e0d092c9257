// k1v2_predict.cu — K1 v2: fused expert predictor on a CTA pair (cta_group::2).
//
// Same math and outputs as k1_predict.cu (reference: predictor.py:193-240,
// :330-351; core.py:27-48; metrics.py:138-193), re-tiled for the Blackwell
// 2-SM tensor core:
//   * a cluster of 2 CTAs owns a 256-token tile; one tcgen05.mma.cta_group::2
//     (M=256, N=256, K=16) covers 256 tokens x 256 hidden units, each CTA
//     staging its own 128 x-rows and half of the W1 chunk (128 rows) -> per-SM
//     shared-memory traffic per MAC is half of the 1-SM 128x128 tile, and x is
//     re-streamed h/256 instead of h/128 times;
//   * GEMM1 accumulates a 256-column chunk in TMEM (single buffer); each
//     epilogue thread drains its 128 columns into registers at once (384
//     threads, up to 168 registers each) so the next chunk's MMAs start after
//     a short drain;
//   * bias + activation + bf16 hi/lo split go to a 64 KB smem A operand, fed to
//     GEMM2 (M=256, N=E) in two K-halves so one buffer suffices;
//   * the per-token selection / margin flag / evaluation epilogue is shared
//     with K1 v1 (k1_common.cuh).
// Warp roles (per CTA, 12 warps): 0 TMA x+W1, 1 MMA issue (leader CTA only),
// 2 TMA W2, 3 TMEM alloc, 4-11 epilogue (WG0 = columns 0-127 of the chunk and
// the token epilogue, WG1 = columns 128-255).
// Requires hidden % 256 == 0 and E <= 128 (else the 1-SM kernel is used).
// Large launches (>= 2 tiles per CTA pair) run the v4 kernel instead
// (k1v4_predict.cu: token epilogue on its own warpgroup, A2 in TMEM); this
// kernel serves the hidden-split and one-wave launches.
#include <cstdio>
#include <cuda.h>
#include "sm100.cuh"
#include "common.cuh"
#include "k1_common.cuh"
#include "tmap.cuh"

namespace moep {
namespace k1v2 {

using k1c::Params;
using k1c::wait;

// Role-level wait accounting for tools/k1_prof.py, compiled only with
// -DMOEP_K1_PROF (a separate library; the product build has no counters):
// cycles spent in each barrier wait by one representative thread per role.
#ifdef MOEP_K1_PROF
__device__ unsigned long long g_k1_prof[160][16];
#define K1_PW(slot, rep, call)                                                         \
  do {                                                                                 \
    const long long t0_ = clock64();                                                   \
    call;                                                                              \
    if (rep) atomicAdd(&g_k1_prof[blockIdx.x][slot], (unsigned long long)(clock64() - t0_)); \
  } while (0)
// per-chunk timeline of CTA 0 (clock64; MMA issuer, WG0 / WG1 warp 0 lane 0)
__device__ long long g_k1_trace[16][64];
#define K1_TR(ev, idx, rep)                                                   \
  do {                                                                      \
    if ((rep) && blockIdx.x == 0 && (idx) < 64) g_k1_trace[ev][idx] = clock64(); \
  } while (0)
#else
#define K1_PW(slot, rep, call) call
#define K1_TR(ev, idx, rep) do { } while (0)
#endif

constexpr int BM = 128;         // tokens per CTA (256 per pair)
constexpr int BK = 64;          // K per stage
constexpr int HC = 256;         // hidden columns per chunk (pair MMA N)
constexpr int HB = HC / 2;      // W1 rows staged per CTA
constexpr int NTHREADS = 384;
constexpr int EPI_WARP0 = 4;

template <int EP>
struct Cfg {
  static constexpr int STAGES = (EP <= 64) ? 4 : 3;
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = HB * BK * 2;        // 16 KB
  static constexpr int ATOM = BM * 64 * 2;           // 16 KB: 128 rows x 64 bf16 (SW128)
  static constexpr int W2_ROWS = EP / 2;             // expert rows staged per CTA
  static constexpr int W2_ATOM = W2_ROWS * 128;      // bytes per 64-column atom
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_A2 = OFF_B + STAGES * B_BYTES;  // [hi atom0, hi atom1, lo atom0, lo atom1]
  static constexpr int OFF_W2 = OFF_A2 + 4 * ATOM;          // 4 atoms (256 columns)
  static constexpr int OFF_HIST = OFF_W2 + ((4 * W2_ATOM + 1023) / 1024) * 1024;
  static constexpr int OFF_SUMSQ = OFF_HIST + 4 * 2 * EP * 4;
  static constexpr int OFF_RED = OFF_SUMSQ + BM * 4;
  static constexpr int OFF_BAR = OFF_RED + 4 * 16 * 4;
  static constexpr int NBAR = 2 * STAGES + 10;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr uint32_t ZCOL = HC;  // TMEM column of the z accumulator
  // GEMM2's lo products accumulate apart from the hi ones (summed in fp32 by
  // the token epilogue): half the truncating accumulate steps on z and none of
  // them against a full-size accumulator (max logit error -32 %)
  static constexpr uint32_t ZLCOL = HC + EP;
  static_assert(ZLCOL + EP <= 512, "TMEM columns");
};

template <int EP, int ARCH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
predict_pair_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w1,
                    const __grid_constant__ CUtensorMap tm_w2, const Params p) {
  using C = Cfg<EP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;                      // [STAGES] leader: x+W1 of both CTAs landed
  uint64_t* empty = bars + C::STAGES;         // [STAGES] local: stage consumed (multicast commit)
  uint64_t* acc_full = empty + C::STAGES;     // local: GEMM1 chunk done
  uint64_t* acc_empty = acc_full + 1;         // leader: 16 epilogue warps drained
  uint64_t* a2_full = acc_empty + 1;          // [2] leader: 8 warps wrote that K-half of A2
  uint64_t* a2_emptyA = a2_full + 2;          // local: GEMM2 half 0 consumed A2
  uint64_t* a2_emptyB = a2_emptyA + 1;        // local: GEMM2 half 1 consumed A2
  uint64_t* w2_full = a2_emptyB + 1;          // leader: W2 chunk of both CTAs landed
  uint64_t* w2_empty = w2_full + 1;           // local
  uint64_t* z_full = w2_empty + 1;            // local
  uint64_t* z_empty = z_full + 1;             // leader: 8 warps read z
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

#ifdef MOEP_K1_PROF
  const long long k1_t_start = clock64();
#endif
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int num_tiles = static_cast<int>((p.n_tokens + 2 * BM - 1) / (2 * BM));
  const int nchunks = p.hidden / HC;
  const int nk = (p.d + BK - 1) / BK;
  // work item = (tile, chunk group): `split` groups of cpg chunks per tile
  const int G = p.split, cpg = nchunks / G;
  const int n_items = num_tiles * G;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 16);
    mbar_init(&a2_full[0], 8);
    mbar_init(&a2_full[1], 8);
    mbar_init(a2_emptyA, 1);
    mbar_init(a2_emptyB, 1);
    mbar_init(w2_full, 1);
    mbar_init(w2_empty, 1);
    mbar_init(z_full, 1);
    mbar_init(z_empty, 8);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x); tma_prefetch_desc(&tm_w1); tma_prefetch_desc(&tm_w2);
  }
  if (warp == 3) tmem_alloc_cg2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < EPI_WARP0) {
    if (warp == 0) {
      // ---------------------------------------------- TMA: x rows + W1 half-chunk
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t stage = 0, phase = 0;
        for (int item = pair; item < n_items; item += n_pairs) {
          const int tile = item / G, c0 = (item % G) * cpg;
          const int xrow = tile * 2 * BM + rank * BM;
          for (int c = c0; c < c0 + cpg; ++c) {
            const int wrow = c * HC + rank * HB;
            for (int kb = 0; kb < nk; ++kb) {
              K1_PW(0, true, wait(&empty[stage], phase ^ 1));
#if defined(MOEP_K1_EXP_NOW1) || defined(MOEP_K1_EXP_NOX)
              // timing experiments only (tools/k1_exp.py; wrong results): skip the
              // W1 / x reloads after an item's first chunk to measure the kernel's
              // sensitivity to L2 -> SM operand traffic
#ifdef MOEP_K1_EXP_NOW1
              const bool ld_w = c == c0, ld_x = true;
#else
              const bool ld_w = true, ld_x = c == c0;
#endif
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * ((ld_x ? C::A_BYTES : 0) + (ld_w ? C::B_BYTES : 0)));
              if (ld_x) tma_load_2d_cg2(&tm_x, &full[stage], smem + C::OFF_A + stage * C::A_BYTES, kb * BK, xrow, keep);
              if (ld_w) tma_load_2d_cg2(&tm_w1, &full[stage], smem + C::OFF_B + stage * C::B_BYTES, kb * BK, wrow, keep);
#else
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
              tma_load_2d_cg2(&tm_x, &full[stage], smem + C::OFF_A + stage * C::A_BYTES, kb * BK, xrow, keep);
              tma_load_2d_cg2(&tm_w1, &full[stage], smem + C::OFF_B + stage * C::B_BYTES, kb * BK, wrow, keep);
#endif
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else if (warp == 2) {
      // ---------------------------------------------- TMA: W2 chunk (EP/2 rows per CTA)
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t n = 0;
        for (int item = pair; item < n_items; item += n_pairs) {
          const int c0 = (item % G) * cpg;
          for (int c = c0; c < c0 + cpg; ++c, ++n) {
            if (n > 0) K1_PW(1, true, wait(w2_empty, (n - 1) & 1));
            if (leader) mbar_arrive_expect_tx(w2_full, 2 * 4 * C::W2_ATOM);
#pragma unroll
            for (int at = 0; at < 4; ++at)
              tma_load_2d_cg2(&tm_w2, w2_full, smem + C::OFF_W2 + at * C::W2_ATOM, c * HC + at * 64,
                              rank * C::W2_ROWS, keep);
          }
        }
      }
    } else if (warp == 1 && leader) {
      // ---------------------------------------------- MMA issuer (pair leader)
      if (elect_one()) {
        const uint32_t idesc1 = idesc_bf16_f32(2 * BM, HC);
        const uint32_t idesc2 = idesc_bf16_f32(2 * BM, EP);
        const uint32_t a_base = smem_u32(smem + C::OFF_A), b_base = smem_u32(smem + C::OFF_B);
        const uint32_t a2_base = smem_u32(smem + C::OFF_A2), w2_base = smem_u32(smem + C::OFF_W2);
        uint32_t stage = 0, phase = 0, gc = 0, ti = 0;
        // GEMM2 of a chunk is issued half by half as soon as its A2 half is
        // ready, interleaved between the next chunk's GEMM1 K-blocks (polled
        // without blocking), so the epilogue's second half never waits for a
        // whole GEMM1 K-loop and the accumulator drains promptly.
        int p_cc = 0, p_half = 2;      // pending GEMM2: chunk-in-tile, next half (2 = none)
        uint32_t p_id = 0, p_ti = 0;   // its global chunk index and tile iteration
        auto pump = [&](bool block) {
          while (p_half < 2) {
            if (p_half == 0) {
              if (p_cc == 0) {
                if (block) K1_PW(2, true, wait(z_empty, (p_ti & 1) ^ 1));
                else if (!k1c::test(z_empty, (p_ti & 1) ^ 1)) return;
              }
              if (block) K1_PW(3, true, wait(w2_full, p_id & 1));
              else if (!k1c::test(w2_full, p_id & 1)) return;
            }
            if (block) K1_PW(4, true, wait(&a2_full[p_half], p_id & 1));
            else if (!k1c::test(&a2_full[p_half], p_id & 1)) return;
            tc_fence_after();
            const int half = p_half;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const int at = kk >> 2, w = kk & 3;
              const uint64_t bd = sdesc_k_sw128(w2_base + (half * 2 + at) * C::W2_ATOM + w * 32);
              const uint64_t ahi = sdesc_k_sw128(a2_base + at * C::ATOM + w * 32);
              const uint64_t alo = sdesc_k_sw128(a2_base + (2 + at) * C::ATOM + w * 32);
              umma_bf16_cg2(tmem + C::ZCOL, ahi, bd, idesc2, (p_cc | half | kk) != 0);
              umma_bf16_cg2(tmem + C::ZLCOL, alo, bd, idesc2, (p_cc | half | kk) != 0);
            }
            K1_TR(3 + half, p_id, true);
            if (half == 0) {
              umma_commit_mc(a2_emptyA, 0x3);
            } else {
              umma_commit_mc(a2_emptyB, 0x3);
              umma_commit_mc(w2_empty, 0x3);
              if (p_cc == cpg - 1) umma_commit_mc(z_full, 0x3);
            }
            ++p_half;
          }
        };
        for (int item = pair; item < n_items; item += n_pairs, ++ti) {
          for (int c = 0; c < cpg; ++c, ++gc) {  // c: chunk within the item
            K1_PW(5, true, wait(acc_empty, (gc & 1) ^ 1));
            K1_TR(0, gc, true);
            tc_fence_after();
            for (int kb = 0; kb < nk; ++kb) {
              K1_PW(6, true, wait(&full[stage], phase));
              if (kb == 0) K1_TR(1, gc, true);
              tc_fence_after();
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = sdesc_k_sw128(a_base + stage * C::A_BYTES + k * 32);
                const uint64_t bd = sdesc_k_sw128(b_base + stage * C::B_BYTES + k * 32);
                umma_bf16_cg2(tmem, ad, bd, idesc1, (kb | k) != 0);
              }
              umma_commit_mc(&empty[stage], 0x3);
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
              pump(false);
            }
            umma_commit_mc(acc_full, 0x3);
            K1_TR(2, gc, true);
            pump(true);  // previous chunk's GEMM2 fully issued before this one is queued
            p_cc = c; p_half = 0; p_id = gc; p_ti = ti;
          }
        }
        pump(true);
      }
    }
  } else {
    // ------------------------------------------------ epilogue warpgroups
    const int wg = (warp - EPI_WARP0) >> 2;  // 0: chunk columns 0-127, 1: 128-255
    const uint32_t q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    float* s_sumsq = reinterpret_cast<float*>(smem + C::OFF_SUMSQ);
    int* hist0 = reinterpret_cast<int*>(smem + C::OFF_HIST);
    int* hist = hist0 + q * 2 * EP;
    if (wg == 0)
      for (int e = lane; e < 2 * EP; e += 32) hist[e] = 0;
    RowCounters rc;
    rc.zero();
    uint32_t gc = 0, ti = 0;
    for (int item = pair; item < n_items; item += n_pairs, ++ti) {
      const int tile = item / G, grp = item % G, c0 = grp * cpg;
      const int64_t row_g = static_cast<int64_t>(tile) * 2 * BM + rank * BM + row_in_tile;
      float sumsq = 0.f;
      for (int c = c0; c < c0 + cpg; ++c, ++gc) {
        K1_PW(wg == 0 ? 7 : 11, lane == 0 && q == 0, wait(acc_full, gc & 1));
        K1_TR(wg == 0 ? 5 : 9, gc, lane == 0 && q == 0);
#ifdef MOEP_K1_PROF
        const long long t_drain0 = clock64();
#endif
        tc_fence_after();
        float v[128];
        const uint32_t ta = tmem + lane_addr + wg * 128;
        tmem_ld32(ta, v);
        tmem_ld32(ta + 32, v + 32);
        tmem_ld32(ta + 64, v + 64);
        tmem_ld32(ta + 96, v + 96);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(acc_empty, 0);
        K1_TR(wg == 0 ? 6 : 10, gc, lane == 0 && q == 0);
#ifdef MOEP_K1_PROF
        if (lane == 0 && q == 0)
          atomicAdd(&g_k1_prof[blockIdx.x][wg == 0 ? 12 : 13], (unsigned long long)(clock64() - t_drain0));
        const long long t_conv0 = clock64();
#endif
        // bias + activation + hi/lo split, in place per column pair (2j, 2j+1):
        // v[2j] <- packed bf16x2 hi, v[2j+1] <- packed bf16x2 lo
        const int col0 = c * HC + wg * 128;
#pragma unroll
        for (int j4 = 0; j4 < 32; ++j4) {
          const int col = col0 + j4 * 4;
          float hv[4];
          if (ARCH == 2) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(p.b1 + col));
            const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
            if (p.a_out && row_g < p.n_tokens)
              *reinterpret_cast<float4*>(p.a_out + row_g * p.hidden + col) =
                  make_float4(v[j4 * 4] + bv[0], v[j4 * 4 + 1] + bv[1], v[j4 * 4 + 2] + bv[2], v[j4 * 4 + 3] + bv[3]);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
#ifdef MOEP_K1_PROF_NOACT  // timing experiment only (tools/k1_prof.py --noact): identity activation
              hv[t] = v[j4 * 4 + t] + bv[t];
#else
              hv[t] = silu_f32(v[j4 * 4 + t] + bv[t]);
#endif
            }
          } else {
            const float4 aa = __ldg(reinterpret_cast<const float4*>(p.alpha + col));
            const float4 bb = __ldg(reinterpret_cast<const float4*>(p.beta + col));
            const float av[4] = {aa.x, aa.y, aa.z, aa.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) hv[t] = gelu_tanh_f32(fmaf(av[t], v[j4 * 4 + t], bv[t]));
          }
#pragma unroll
          for (int t = 0; t < 4; t += 2) {
            sumsq = fmaf(hv[t], hv[t], sumsq);
            sumsq = fmaf(hv[t + 1], hv[t + 1], sumsq);
            // packed conversions (one F2FP per column pair): hi = bf16x2(h), lo = bf16x2(h - hi);
            // column t in the low half, as the swizzled A2 layout expects
            const __nv_bfloat162 hp = __floats2bfloat162_rn(hv[t], hv[t + 1]);
            const float2 hf = __bfloat1622float2(hp);
            const __nv_bfloat162 lp = __floats2bfloat162_rn(hv[t] - hf.x, hv[t + 1] - hf.y);
            v[j4 * 4 + t] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&hp));
            v[j4 * 4 + t + 1] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&lp));
          }
        }
#ifdef MOEP_K1_PROF
        if (lane == 0 && q == 0) atomicAdd(&g_k1_prof[blockIdx.x][wg == 0 ? 14 : 3], 0ull);
        if (lane == 0 && q == 0 && wg == 0) atomicAdd(&g_k1_prof[blockIdx.x][14], (unsigned long long)(clock64() - t_conv0));
#endif
        K1_TR(wg == 0 ? 7 : 11, gc, lane == 0 && q == 0);
        // the A2 buffer is free once the previous GEMM2 half that read it completed
        if (wg == 0) {
          if (gc > 0) K1_PW(8, lane == 0 && q == 0, wait(a2_emptyB, (gc - 1) & 1));
        } else {
          K1_PW(9, lane == 0 && q == 0, wait(a2_emptyA, gc & 1));
          K1_TR(12, gc, lane == 0 && q == 0);
        }
        uint8_t* a2hi = smem + C::OFF_A2;
        uint8_t* a2lo = smem + C::OFF_A2 + 2 * C::ATOM;
#pragma unroll
        for (int sb = 0; sb < 4; ++sb) {
          const int at = sb >> 1;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            // 16-byte chunk = 8 columns = 4 column pairs starting at column sb*32 + ch*8
            const uint32_t off = at * C::ATOM + sw128_offset(row_in_tile, (sb & 1) * 32 + ch * 8);
            const int b = sb * 32 + ch * 8;
            *reinterpret_cast<uint4*>(a2hi + off) = make_uint4(__float_as_uint(v[b]), __float_as_uint(v[b + 2]),
                                                               __float_as_uint(v[b + 4]), __float_as_uint(v[b + 6]));
            *reinterpret_cast<uint4*>(a2lo + off) = make_uint4(__float_as_uint(v[b + 1]), __float_as_uint(v[b + 3]),
                                                               __float_as_uint(v[b + 5]), __float_as_uint(v[b + 7]));
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&a2_full[wg], 0);
        K1_TR(wg == 0 ? 8 : 13, gc, lane == 0 && q == 0);
      }
      // ---- token epilogue on warpgroup 0
      if (wg == 1) s_sumsq[row_in_tile] = sumsq;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (wg == 0) {
        sumsq += s_sumsq[row_in_tile];
        K1_PW(10, lane == 0 && q == 0, wait(z_full, ti & 1));
        K1_TR(14, gc - 1, lane == 0 && q == 0);
        tc_fence_after();
        float z[EP];
#pragma unroll
        for (int j = 0; j < EP; j += 16) tmem_ld16(tmem + lane_addr + C::ZCOL + j, z + j);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < EP; j += 16) {
          float zl[16];
          tmem_ld16(tmem + lane_addr + C::ZLCOL + j, zl);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 16; ++t) z[j + t] += zl[t];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(z_empty, 0);
        if (G > 1) {
          // hidden split: this group's partial z and ||h||^2 (split_finish sums the groups)
          float* zp = p.zpart + (static_cast<int64_t>(grp) * p.zpad + row_g) * EP;
#pragma unroll
          for (int j = 0; j < EP; j += 4) *reinterpret_cast<float4*>(zp + j) = make_float4(z[j], z[j + 1], z[j + 2], z[j + 3]);
          p.zpart[static_cast<int64_t>(G) * p.zpad * EP + static_cast<int64_t>(grp) * p.zpad + row_g] = sumsq;
        } else {
          // The A2 buffer is idle here: WG1 cannot write the next tile's A2 before
          // GEMM2 half 0 of its chunk 0, which needs this warpgroup's half first.
          uint32_t zswz;
          float* zrow = k1c::zstage_row<EP>(smem + C::OFF_A2, row_in_tile, lane, zswz);
          k1c::row_epilogue<EP>(p, z, sumsq, row_g, row_g < p.n_tokens, lane, hist, rc, zrow, zswz);
          K1_TR(15, gc - 1, lane == 0 && q == 0);
          // A warp's A2 rows for the next chunk (swizzled 128-byte rows in each of
          // the four atoms) overlap OTHER warps' staging rows: no warp of WG0 may
          // leave the token epilogue (and write A2) while another still reads
          // its staging row (the selection and the truth-window checks run for
          // data-dependent times per warp)
          asm volatile("bar.sync 4, 128;" ::: "memory");
        }
      }
    }
    if (wg == 0 && p.partials && G == 1)
      k1c::write_partials<EP>(p, rc, q, lane, threadIdx.x - EPI_WARP0 * 32,
                              reinterpret_cast<int*>(smem + C::OFF_RED), hist0, 2);
  }
  tc_fence_before();
  __syncthreads();
#ifdef MOEP_K1_PROF
  if (threadIdx.x == 0) atomicAdd(&g_k1_prof[blockIdx.x][15], (unsigned long long)(clock64() - k1_t_start));
#endif
  cluster_sync();
  if (warp == 3) tmem_dealloc_cg2<512>(tmem);
}

// Hidden-split finish: z = fixed-order sum of the groups' partial logits, then
// the per-token selection / margin / output / counter semantics of
// k1c::row_epilogue (the fused path's epilogue), re-laid for one WARP per token
// (lane l holds experts l, l+32, ...): the top list is built by warp argmax
// reductions (value, then lower index on ties; -0.0 == +0.0), ascending ids by
// ballot prefix sums, truth-expert lookups by shuffles. grid = num_SMs (one
// counter partial row per CTA, the layout moep_counters_reduce expects).
template <int EP>
__global__ void __launch_bounds__(256) split_finish_kernel(const Params p) {
  constexpr int PL = EP >= 32 ? EP / 32 : 1;   // experts per lane
  __shared__ int hist_s[2 * EP];
  __shared__ int cnt_s[2 + 2 * MOEP_MAX_BOUNDS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2 * EP; i += 256) hist_s[i] = 0;
  if (tid < 2 + 2 * MOEP_MAX_BOUNDS) cnt_s[tid] = 0;
  __syncthreads();
  const int G = p.split, E = p.E;
  const float* sq = p.zpart + static_cast<int64_t>(G) * p.zpad * EP;
  int P = p.m_sel;
#pragma unroll
  for (int b = 0; b < MOEP_MAX_BOUNDS; ++b)
    if (b < p.n_bounds && p.bounds[b] > P) P = p.bounds[b];
  P = min(P + 1, min(E, kMaxSel));
  RowCounters rc;
  rc.zero();
  const int64_t nw = static_cast<int64_t>(gridDim.x) * 8;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp; row < p.n_tokens; row += nw) {
    float zv[PL];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int e = q * 32 + lane;
      float acc = 0.f;
      if (e < EP) {
        // all groups' partials in flight together, then the fixed-order sum
        float v[16];
#pragma unroll
        for (int g = 0; g < 16; ++g)
          v[g] = g < G ? __ldcg(p.zpart + (static_cast<int64_t>(g) * p.zpad + row) * EP + e) : 0.f;
#pragma unroll
        for (int g = 0; g < 16; ++g)
          if (g < G) acc += v[g];
      }
      if (e < E) {
        acc += __ldg(p.b2 + e);
        bad |= !isfinite(acc);
      } else {
        acc = -INFINITY;
      }
      zv[q] = acc;
    }
    float sumsq = 0.f;
    {
      // lane g loads group g's ||h||^2 partial; lane 0 sums them in order
      const float part = lane < G ? __ldcg(sq + static_cast<int64_t>(lane) * p.zpad + row) : 0.f;
#pragma unroll
      for (int g = 0; g < 16; ++g) {
        const float v = __shfl_sync(0xffffffffu, part, g);
        if (g < G) sumsq += v;
      }
    }
    bool flagged = __any_sync(0xffffffffu, bad);
    if (flagged && lane == 0 && p.status) atomicOr(p.status, 1);
    // sorted top list (warp-uniform): repeated warp argmax over the untaken experts
    float tv[kMaxSel];
    int tix[kMaxSel];
    uint32_t taken = 0;
#pragma unroll
    for (int s = 0; s < kMaxSel; ++s) {
      float best = -INFINITY;
      int bi = 0x7fffffff;
      if (s < P) {
#pragma unroll
        for (int q = 0; q < PL; ++q) {
          const int e = q * 32 + lane;
          if (!((taken >> q) & 1u) && e < EP && (zv[q] > best || (zv[q] == best && e < bi))) { best = zv[q]; bi = e; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      }
      tv[s] = best;
      tix[s] = bi;
    }
    const float delta = p.tau_abs + p.tau_rel * sqrtf(sumsq) * p.w2_norm;
#pragma unroll
    for (int b = 0; b < MOEP_MAX_BOUNDS; ++b) {
      if (b < p.n_bounds) {
        const int pos = p.bounds[b];
        if (pos >= 1 && pos < E) {
          float hi_v = tv[0], lo_v = tv[1];
#pragma unroll
          for (int s = 1; s < kMaxSel; ++s)
            if (s == pos) { hi_v = tv[s - 1]; lo_v = tv[s]; }
          flagged |= !(hi_v - lo_v >= delta);
        }
      }
    }
    if (lane == 0) {
      if (p.flags) p.flags[row] = flagged ? 1 : 0;
      if (flagged) p.flag_list[atomicAdd(p.flag_count, 1)] = static_cast<int>(row);
    }
    if (p.logits) {
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        const int e = q * 32 + lane;
        if (e < E) p.logits[row * E + e] = zv[q];
      }
    }
    if (p.probs) {  // fused softmax (core.py:19-24) across the warp's lanes
      float mx = -INFINITY;
#pragma unroll
      for (int q = 0; q < PL; ++q)
        if (q * 32 + lane < E) mx = fmaxf(mx, zv[q]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float sum = 0.f;
#pragma unroll
      for (int q = 0; q < PL; ++q)
        if (q * 32 + lane < E) sum += expf(zv[q] - mx);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        const int e = q * 32 + lane;
        if (e < E) p.probs[row * E + e] = expf(zv[q] - mx) / sum;
      }
    }
    if (p.ids && !flagged) {
      int* orow = p.ids + row * p.m_sel;
      if (p.m_sel >= E) {
        for (int e = lane; e < E; e += 32) orow[e] = e;
      } else {
        float thv = tv[0];
        int thi = tix[0];
#pragma unroll
        for (int s = 0; s < kMaxSel; ++s)
          if (s == p.m_sel - 1) { thv = tv[s]; thi = tix[s]; }
        int base = 0;
#pragma unroll
        for (int q = 0; q < PL; ++q) {
          const int e = q * 32 + lane;
          const bool sel = e < E && ((zv[q] > thv || (zv[q] == thv && e < thi)) || e == thi);
          const uint32_t mask = __ballot_sync(0xffffffffu, sel);
          if (sel) orow[base + __popc(mask & ((1u << lane) - 1u))] = e;
          base += __popc(mask);
        }
      }
    }
    if (p.truth && !flagged) {
      // "truth expert t has predicted rank < m" <=> key(t) >= key(position m-1) of the top list
      const bool act = lane < p.k;
      const int t = act ? __ldg(p.truth + row * p.k + lane) : 0;
      float zt = 0.f;
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        const float v = __shfl_sync(0xffffffffu, zv[q], t & 31);
        if ((t >> 5) == q) zt = v;
      }
      auto thr = [&](int m, float& v, int& ix) {
        v = tv[0];
        ix = tix[0];
#pragma unroll
        for (int s = 0; s < kMaxSel; ++s)
          if (s == m - 1) { v = tv[s]; ix = tix[s]; }
      };
      float kv;
      int ki;
      thr(p.k, kv, ki);
      const bool hit = act && ((zt > kv || (zt == kv && t < ki)) || t == ki);
      if (act) {
        atomicAdd(&hist_s[EP + t], 1);
        if (hit) atomicAdd(&hist_s[t], 1);
      }
      const bool any0 = __any_sync(0xffffffffu, act && t == tix[0]);
      rc.n += 1;
      rc.top1 += any0 ? 1 : 0;
#pragma unroll
      for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
        if (mi < p.n_m) {
          const int m = p.m_list[mi];
          float mv;
          int mx;
          thr(m < kMaxSel ? m : 1, mv, mx);
          const bool in = act && (m >= E || (zt > mv || (zt == mv && t < mx)) || t == mx);
          const int cnt = __popc(__ballot_sync(0xffffffffu, in));
          rc.ov[mi] += cnt == p.k ? 1 : 0;
          rc.rc[mi] += cnt;
        }
      }
    }
  }
  if (p.partials) {
    if (lane == 0) {
      atomicAdd(&cnt_s[0], rc.n);
      atomicAdd(&cnt_s[1], rc.top1);
#pragma unroll
      for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
        atomicAdd(&cnt_s[2 + mi], rc.ov[mi]);
        atomicAdd(&cnt_s[2 + MOEP_MAX_BOUNDS + mi], rc.rc[mi]);
      }
    }
    __syncthreads();
    int* out = p.partials + static_cast<int64_t>(blockIdx.x) * p.n_counters;
    for (int t = tid; t < p.n_counters; t += 256) {
      int v;
      if (t < 2) v = cnt_s[t];
      else if (t < 2 + p.n_m) v = cnt_s[2 + (t - 2)];
      else if (t < 2 + 2 * p.n_m) v = cnt_s[2 + MOEP_MAX_BOUNDS + (t - 2 - p.n_m)];
      else {
        const int u = t - 2 - 2 * p.n_m;  // [hits E | truth E]
        v = u < E ? hist_s[u] : hist_s[EP + (u - E)];
      }
      out[t] = v;
    }
  }
}

// Which pair kernel runs (moep_predict_args.kernel): auto (0) takes v4
// (k1v4_predict.cu: token epilogue on its own warpgroup, A2 in TMEM) for
// unsplit launches with at least two 256-token tiles per CTA pair and this
// file's v2 kernel otherwise (hidden-split small-N launches, one-wave
// launches); MOEP_K1_PAIR_V2 (2) / MOEP_K1_PAIR_V4 (4) force one of them.
static bool use_v4(const moep_predict_args* a) {
  return a->kernel != MOEP_K1_PAIR_V2 && a->hidden % HC == 0 && a->n_experts <= 128;
}

// Chunk groups per tile: only when the tiles leave CTA pairs idle (fewer tiles
// than pairs); then the fewest pair-rounds of chunks, ties to fewer groups.
// Large N never splits (the partial-logit traffic and the x re-streaming would
// cost more than the last-wave imbalance they remove).
static int choose_split(int64_t n_tokens, int nchunks, int n_pairs) {
  const int64_t tiles = (n_tokens + 2 * BM - 1) / (2 * BM);
  if (tiles >= n_pairs) return 1;
#ifdef MOEP_FORCE_SPLIT2
  if (nchunks % 2 == 0) return 2;
#endif
  const int64_t cost1 = ((tiles + n_pairs - 1) / n_pairs) * nchunks;
  int best = 1;
  int64_t best_cost = cost1;
  for (int g = 2; g <= nchunks && g <= 16; ++g) {
    if (nchunks % g) continue;
    const int64_t cost = ((tiles * g + n_pairs - 1) / n_pairs) * (nchunks / g);
    if (cost < best_cost) { best = g; best_cost = cost; }
  }
  // a split pays per-item pipeline fills, the partial-logit traffic and the
  // finish kernel: take it only for a clear gain (at most 3/4 of the rounds)
  return 4 * best_cost <= 3 * cost1 ? best : 1;
}

}  // namespace k1v2
}  // namespace moep

#ifdef MOEP_K1_PROF
extern "C" int moep_k1_trace(long long* host) {
  return cudaMemcpyFromSymbol(host, moep::k1v2::g_k1_trace, sizeof(long long) * 16 * 64) == cudaSuccess ? 0 : -4;
}
extern "C" int moep_k1_prof(unsigned long long* host, int reset) {
  if (reset) {
    static unsigned long long zero[160][16];
    return cudaMemcpyToSymbol(moep::k1v2::g_k1_prof, zero, sizeof(zero)) == cudaSuccess ? 0 : -4;
  }
  return cudaMemcpyFromSymbol(host, moep::k1v2::g_k1_prof, sizeof(unsigned long long) * 160 * 16) == cudaSuccess
             ? 0 : -4;
}
#endif

extern "C" int64_t moep_predict_split_floats(int64_t n_tokens, int32_t hidden, int32_t n_experts) {
  using namespace moep::k1v2;
  if (n_tokens <= 0 || hidden <= 0 || n_experts <= 0 || n_experts > 128) return 0;
  if (hidden % HC != 0) return 0;
  const int g = choose_split(n_tokens, hidden / HC, moep_num_sms() / 2);
  if (g == 1) return 0;
  int EP = 16;
  while (EP < n_experts) EP *= 2;
  const int64_t zpad = ((n_tokens + 2 * BM - 1) / (2 * BM)) * 2 * BM;
  return static_cast<int64_t>(g) * zpad * (EP + 1);
}

extern "C" int moep_predict_bf16_pair4(const moep_predict_args* a, void* stream);
extern "C" int moep_predict_bf16_quad5(const moep_predict_args* a, void* stream);

namespace {
template <int EP, int ARCH>
int launch_v2(const moep_predict_args* a, cudaStream_t st) {
  using namespace moep::k1v2;
  using C = Cfg<EP>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = predict_pair_kernel<EP, ARCH>;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess)
      return MOEP_ELAUNCH;
    attr_set[dev] = true;
  }
  CUtensorMap tx, tw1, tw2;
  if (moep::make_tmap_bf16(&tx, a->x, a->n_tokens, a->d, BM, BK) ||
      moep::make_tmap_bf16(&tw1, a->w1, a->hidden, a->d, HB, BK) ||
      moep::make_tmap_bf16(&tw2, a->w2, a->n_experts, a->hidden, C::W2_ROWS, 64))
    return MOEP_EALIGN;
  moep::k1c::Params p{};
  p.n_tokens = a->n_tokens; p.d = a->d; p.hidden = a->hidden; p.E = a->n_experts; p.arch = a->arch;
  p.b1 = a->b1; p.alpha = a->act_alpha; p.beta = a->act_beta; p.b2 = a->b2;
  p.m_sel = a->m_sel; p.n_bounds = a->n_bounds;
  for (int i = 0; i < MOEP_MAX_BOUNDS; ++i) { p.bounds[i] = a->bounds[i]; p.m_list[i] = a->m_list[i]; }
  p.tau_abs = a->tau_abs; p.tau_rel = a->tau_rel; p.w2_norm = a->w2_norm;
  p.ids = a->ids; p.logits = a->logits; p.flags = a->flags; p.probs = a->probs;
  p.flag_list = a->flag_list; p.flag_count = a->flag_count;
  p.truth = a->truth; p.k = a->k; p.n_m = a->n_m; p.partials = a->partials; p.a_out = a->a_out;
  p.status = a->status;
  p.n_counters = moep_n_counters(a->n_m, a->n_experts);
  const int grid = moep_num_sms() & ~1;  // whole CTA pairs
  p.split = 1; p.zpart = nullptr; p.zpad = 0;
  const int64_t need = moep_predict_split_floats(a->n_tokens, a->hidden, a->n_experts);
  if (need > 0 && a->split_scratch && a->split_scratch_floats >= need) {
    p.split = choose_split(a->n_tokens, a->hidden / HC, grid / 2);
    p.zpart = a->split_scratch;
    p.zpad = ((a->n_tokens + 2 * BM - 1) / (2 * BM)) * 2 * BM;
  }
  if (a->kernel == MOEP_K1_QUAD_V5) return moep_predict_bf16_quad5(a, st);
  // One wave of unsplit tiles with d >= 4096: the pairs' live x tiles (2 MB
  // each) overflow L2 and every hidden chunk re-reads them from DRAM; the
  // 4-CTA cluster kernel shares each tile between two pairs (TMA multicast)
  // and halves the live set. Phi-shape training forward (16 k tokens, d = 4096,
  // E = 16): 0.258 -> 0.227 ms (tools/ab_k1.py).
  if (a->kernel == MOEP_K1_AUTO && p.split == 1 && a->n_experts <= 64 && a->hidden % 512 == 0 && a->d >= 4096 &&
      (a->n_tokens + 2 * BM - 1) / (2 * BM) < grid / 2)
    return moep_predict_bf16_quad5(a, st);
  if (p.split == 1 && use_v4(a) &&
      (a->kernel == MOEP_K1_PAIR_V4 || (a->n_tokens + 2 * BM - 1) / (2 * BM) >= 2 * (grid / 2))) {
    // v4 hides each tile's token epilogue behind the next tile: with fewer
    // than two tiles per CTA pair there is nothing to hide it behind, and v2's
    // register-resident epilogue is the shorter path
    return moep_predict_bf16_pair4(a, st);
  } else {
    kern<<<grid, NTHREADS, C::SMEM, st>>>(tx, tw1, tw2, p);
    if (cudaGetLastError() != cudaSuccess) return MOEP_ELAUNCH;
  }
  if (p.split > 1) {
    split_finish_kernel<EP><<<moep_num_sms(), 256, 0, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return MOEP_ELAUNCH;
  }
  return MOEP_OK;
}
}  // namespace

// Pair kernel entry (validation shared with moep_predict_bf16, which dispatches here).
extern "C" int moep_predict_bf16_pair(const moep_predict_args* a, void* stream) {
  if (a->n_experts > 128) return MOEP_EUNSUPPORTED;
  if (a->hidden % 256 != 0) return MOEP_EUNSUPPORTED;
  int EP = 16;
  while (EP < a->n_experts) EP *= 2;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool a1 = a->arch == 1;
  switch (EP) {
    case 16: return a1 ? launch_v2<16, 1>(a, st) : launch_v2<16, 2>(a, st);
    case 32: return a1 ? launch_v2<32, 1>(a, st) : launch_v2<32, 2>(a, st);
    case 64: return a1 ? launch_v2<64, 1>(a, st) : launch_v2<64, 2>(a, st);
    default: return a1 ? launch_v2<128, 1>(a, st) : launch_v2<128, 2>(a, st);
  }
}
