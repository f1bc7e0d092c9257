// k1v4_predict.cu — K1 v4 (default for E <= 64): the v2 CTA-pair fused
// predictor with (1) the per-token epilogue on its own warpgroup and (2) the
// GEMM2 operand A2 (bias + activation, split into bf16 hi / lo) kept in TENSOR
// MEMORY instead of shared memory.
//
// (1) v2 ran the per-token selection / margin / counter epilogue on the
// warpgroup that also drains the accumulator; for ~66 k cycles per tile it
// could not drain the next tile's first chunk and the tensor pipe stalled
// (per-chunk trace: every 8th chunk took ~75 k cycles instead of 27 k). Here
// WG2 (warps 12-15) owns z: it reads the tile's z from TMEM (the MMA waits
// only for that read, z_empty), takes the two ||h||^2 partials from WG0 / WG1
// through a double-buffered shared-memory hand-off (sum_ready / sum_empty) and
// runs the selection while the next tile's chunks stream (over z staged in
// shared memory, so its registers do not grow with E). Chunk period
// 27.1 k -> 22.4 k cycles, no per-tile stall. 512 threads: setmaxnreg splits
// the register file 72 (TMA / MMA warps) / 160 (chunk epilogue) / 120 (WG2).
//
// The epilogue writes its hi / lo pairs with tcgen05.st (no swizzle math, no
// shared-memory write traffic, no async-proxy fence) and GEMM2 reads them with
// the TMEM-A form of tcgen05.mma.cta_group::2 ("TS": A rows = the TMEM lanes of
// each CTA, B = W2 from shared memory). The 64 KB of shared memory this frees
// buys a fifth x / W1 pipeline stage (E <= 64): the role trace
// (tools/k1_exp.py --trace) showed the v2 K-loop issuing at ~73 % of the
// tensor rate while waiting on operand loads, with the producer's 4-stage ring
// always full of in-flight loads. TMEM columns: accumulator [0, 256), z
// [256, 256 + EP), A2 [256 + EP, 256 + EP + 128).
// Everything else — work items, barriers, the per-token selection / margin /
// evaluation epilogue — is v2's (k1v2_predict.cu; reference predictor.py:193-240,
// :330-351, core.py:27-48, metrics.py:138-193). No hidden split (G = 1 only).
#include <cstdio>
#include <cuda.h>
#include "sm100.cuh"
#include "common.cuh"
#include "k1_common.cuh"
#include "tmap.cuh"

namespace moep {
namespace k1v4 {

using k1c::Params;
using k1c::wait;

#define K1_PW(slot, rep, call) call
#ifdef MOEP_K1_PROF
// per-chunk timeline of CTA 0 (tools/k1_exp.py --trace), same events as v2
__device__ long long g_k1v4_trace[16][64];
#define K1_TR(ev, idx, rep)                                                      \
  do {                                                                         \
    if ((rep) && blockIdx.x == 0 && (idx) < 64) g_k1v4_trace[ev][idx] = clock64(); \
  } while (0)
#else
#define K1_TR(ev, idx, rep) do { } while (0)
#endif

constexpr int BM = 128;         // tokens per CTA (256 per pair)
constexpr int BK = 64;          // K per stage
constexpr int HC = 256;         // hidden columns per chunk (pair MMA N)
constexpr int HB = HC / 2;      // W1 rows staged per CTA
constexpr int NTHREADS = 512;
constexpr int EPI_WARP0 = 4;   // WG0 = warps 4-7, WG1 = warps 8-11 (chunk epilogue)
constexpr int TOK_WARP0 = 12;  // WG2 = warps 12-15 (per-token epilogue)
// register split (setmaxnreg; 128 per thread at launch): 4 warps x PROD +
// 8 x EPI + 4 x WG2 <= 16 x 128
#ifndef K1V4_PROD_REGS
#define K1V4_PROD_REGS 72
#define K1V4_EPI_REGS 160
#define K1V4_WG2_REGS 120
#endif
constexpr int PROD_REGS = K1V4_PROD_REGS, EPI_REGS = K1V4_EPI_REGS, WG2_REGS = K1V4_WG2_REGS;
static_assert(PROD_REGS + 2 * EPI_REGS + WG2_REGS <= 4 * 128, "register pool");

template <int EP>
struct Cfg {
  // A2 (the hi/lo GEMM2 operand) lives in TMEM, so the ring gets its 64 KB
  static constexpr int STAGES = (EP <= 64) ? 5 : 3;
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = HB * BK * 2;        // 16 KB
  static constexpr int W2_ROWS = EP / 2;             // expert rows staged per CTA
  static constexpr int W2_ATOM = W2_ROWS * 128;      // bytes per 64-column atom
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_W2 = OFF_B + STAGES * B_BYTES;   // 4 atoms (256 columns)
  static constexpr int OFF_Z = OFF_W2 + ((4 * W2_ATOM + 1023) / 1024) * 1024;  // token-epilogue z staging
  static constexpr int OFF_HIST = OFF_Z + BM * (EP >= 32 ? EP : EP + 1) * 4;
  static constexpr int OFF_SUMSQ = OFF_HIST + 4 * 2 * EP * 4;
  static constexpr int OFF_RED = OFF_SUMSQ + 2 * 2 * BM * 4;
  static constexpr int OFF_BAR = OFF_RED + 4 * 16 * 4;
  static constexpr int NBAR = 2 * STAGES + 14;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr uint32_t ZCOL = HC;               // TMEM column of the z accumulator
  static constexpr uint32_t A2COL = HC + EP;         // hi pairs [A2COL, +64), lo pairs [A2COL+64, +128)
  static_assert(A2COL + 128 <= 512, "TMEM columns");
  // GEMM2's lo products accumulate apart from the hi ones where TMEM has the
  // columns (EP <= 64): summed in fp32 by WG2 (max logit error -32 %)
  static constexpr bool ZLO = A2COL + 128 + EP <= 512;
  static constexpr uint32_t ZLCOL = ZLO ? A2COL + 128 : ZCOL;  // lo-product accumulator
  static_assert(SMEM <= 232448, "shared memory");
};

// 32 lanes x 32 bit, 32 consecutive columns from the even / odd entries of v[64]
template <int ODD>
__device__ __forceinline__ void tmem_st32_strided(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[ODD + 0]), "r"(r[ODD + 2]), "r"(r[ODD + 4]), "r"(r[ODD + 6]), "r"(r[ODD + 8]),
        "r"(r[ODD + 10]), "r"(r[ODD + 12]), "r"(r[ODD + 14]), "r"(r[ODD + 16]), "r"(r[ODD + 18]),
        "r"(r[ODD + 20]), "r"(r[ODD + 22]), "r"(r[ODD + 24]), "r"(r[ODD + 26]), "r"(r[ODD + 28]),
        "r"(r[ODD + 30]), "r"(r[ODD + 32]), "r"(r[ODD + 34]), "r"(r[ODD + 36]), "r"(r[ODD + 38]),
        "r"(r[ODD + 40]), "r"(r[ODD + 42]), "r"(r[ODD + 44]), "r"(r[ODD + 46]), "r"(r[ODD + 48]),
        "r"(r[ODD + 50]), "r"(r[ODD + 52]), "r"(r[ODD + 54]), "r"(r[ODD + 56]), "r"(r[ODD + 58]),
        "r"(r[ODD + 60]), "r"(r[ODD + 62])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T over the CTA pair ("TS" form: each CTA's
// 128 A rows are its TMEM lanes, 16-bit A packed two per 32-bit column).
__device__ __forceinline__ void umma_bf16_cg2_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

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
  uint64_t* z_empty = z_full + 1;             // leader: WG2's 8 warps (both CTAs) read z
  uint64_t* sum_ready = z_empty + 1;          // [2] local: WG0 + WG1 wrote the tile's ||h||^2 partials
  uint64_t* sum_empty = sum_ready + 2;        // [2] local: WG2 read them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

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
    mbar_init(&sum_ready[0], 8);
    mbar_init(&sum_ready[1], 8);
    mbar_init(&sum_empty[0], 4);
    mbar_init(&sum_empty[1], 4);
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
    regs_dec<PROD_REGS>();
    if (warp == 0) {
      // ---------------------------------------------- TMA: x rows + W1 half-chunk
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
#ifdef K1V4_X_NORMAL
        const uint64_t xpol = policy_evict_normal();
#else
        const uint64_t xpol = keep;
#endif
#ifdef K1V4_W1_NORMAL
        const uint64_t wpol = policy_evict_normal();
#else
        const uint64_t wpol = keep;
#endif
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
              tma_load_2d_cg2(&tm_x, &full[stage], smem + C::OFF_A + stage * C::A_BYTES, kb * BK, xrow, xpol);
              tma_load_2d_cg2(&tm_w1, &full[stage], smem + C::OFF_B + stage * C::B_BYTES, kb * BK, wrow, wpol);
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
        const uint32_t w2_base = smem_u32(smem + C::OFF_W2);
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
              umma_bf16_cg2_ts(tmem + C::ZCOL, tmem + C::A2COL + kk * 8, bd, idesc2, (p_cc | half | kk) != 0);
              umma_bf16_cg2_ts(tmem + C::ZLCOL, tmem + C::A2COL + 64 + kk * 8, bd, idesc2,
                               C::ZLO ? uint32_t((p_cc | half | kk) != 0) : 1u);
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
  } else if (warp < TOK_WARP0) {
    // ------------------------------------------------ chunk epilogue warpgroups
    regs_inc<EPI_REGS>();
    const int wg = (warp - EPI_WARP0) >> 2;  // 0: chunk columns 0-127, 1: 128-255
    const uint32_t q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    float* s_sumsq = reinterpret_cast<float*>(smem + C::OFF_SUMSQ);
    uint32_t gc = 0, ti = 0;
    for (int item = pair; item < n_items; item += n_pairs, ++ti) {
      const int tile = item / G, grp = item % G, c0 = grp * cpg;
      const int64_t row_g = static_cast<int64_t>(tile) * 2 * BM + rank * BM + row_in_tile;
      float sumsq = 0.f;
      for (int c = c0; c < c0 + cpg; ++c, ++gc) {
        K1_PW(wg == 0 ? 7 : 11, lane == 0 && q == 0, wait(acc_full, gc & 1));
        K1_TR(wg == 0 ? 5 : 9, gc, lane == 0 && q == 0);
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
        K1_TR(wg == 0 ? 7 : 11, gc, lane == 0 && q == 0);
        // the A2 buffer is free once the previous GEMM2 half that read it completed
        if (wg == 0) {
          if (gc > 0) K1_PW(8, lane == 0 && q == 0, wait(a2_emptyB, (gc - 1) & 1));
        } else {
          K1_PW(9, lane == 0 && q == 0, wait(a2_emptyA, gc & 1));
          K1_TR(12, gc, lane == 0 && q == 0);
        }
        // A2 in TMEM: this warp's 32 lanes, hi pairs -> [A2COL, +64), lo pairs -> [A2COL+64, +128)
        {
          const uint32_t ta2 = tmem + lane_addr + C::A2COL;
          tmem_st32_strided<0>(ta2, v);
          tmem_st32_strided<0>(ta2 + 32, v + 64);
          tmem_st32_strided<1>(ta2 + 64, v);
          tmem_st32_strided<1>(ta2 + 96, v + 64);
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&a2_full[wg], 0);
        K1_TR(wg == 0 ? 8 : 13, gc, lane == 0 && q == 0);
      }
      // ---- hand this tile's ||h||^2 partial to WG2 (double-buffered by tile parity)
      if (ti >= 2) wait(&sum_empty[ti & 1], ((ti >> 1) & 1) ^ 1);
      s_sumsq[((ti & 1) * 2 + wg) * BM + row_in_tile] = sumsq;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sum_ready[ti & 1]);
    }
  } else {
    // ------------------------------------------------ WG2: per-token epilogue
    regs_dec<WG2_REGS>();
    // Owns z, the selection / margin / ids / counters of each tile, off the
    // chunk pipeline: the MMA only waits for WG2's z read (z_empty) before the
    // next tile's first GEMM2, not for the selection work.
    const uint32_t q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    const float* s_sumsq = reinterpret_cast<const float*>(smem + C::OFF_SUMSQ);
    int* hist0 = reinterpret_cast<int*>(smem + C::OFF_HIST);
    int* hist = hist0 + q * 2 * EP;
    for (int e = lane; e < 2 * EP; e += 32) hist[e] = 0;
    RowCounters rc;
    rc.zero();
    uint32_t ti = 0;
    for (int item = pair; item < n_items; item += n_pairs, ++ti) {
      const int tile = item;
      const int64_t row_g = static_cast<int64_t>(tile) * 2 * BM + rank * BM + row_in_tile;
      wait(z_full, ti & 1);
      K1_TR(14, ti * 8 + 7, lane == 0 && q == 0);
      tc_fence_after();
      uint32_t zswz;
      float* zrow = k1c::zstage_row<EP>(smem + C::OFF_Z, row_in_tile, lane, zswz);
      // z + b2 -> this row's shared-memory staging row, 16 columns at a time:
      // the selection reads z from there, so WG2's registers do not grow with
      // E (measured 1-3 % faster than register-resident z at E = 64, which
      // spills at WG2's 120-register share)
      bool bad = false;
#pragma unroll
      for (int j = 0; j < EP; j += 16) {
        float zc[16];
        tmem_ld16(tmem + lane_addr + C::ZCOL + j, zc);
        if (C::ZLO) {
          // + the lo-product accumulator
          float zl[16];
          tmem_ld16(tmem + lane_addr + C::ZLCOL + j, zl);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 16; ++t) zc[t] += zl[t];
        }
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int e = j + t;
          float v = -INFINITY;
          if (e < p.E) {
            v = zc[t] + __ldg(p.b2 + e);
            bad |= !isfinite(v);
          }
          zrow[e ^ zswz] = v;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(z_empty, 0);
      wait(&sum_ready[ti & 1], (ti >> 1) & 1);
      const float sumsq = s_sumsq[((ti & 1) * 2 + 0) * BM + row_in_tile] +
                          s_sumsq[((ti & 1) * 2 + 1) * BM + row_in_tile];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sum_empty[ti & 1]);
      k1c::row_epilogue_staged<EP>(p, bad, sumsq, row_g, row_g < p.n_tokens, lane, hist, rc, zrow, zswz);
      K1_TR(15, ti * 8 + 7, lane == 0 && q == 0);
    }
    if (p.partials)
      k1c::write_partials<EP>(p, rc, q, lane, threadIdx.x - TOK_WARP0 * 32,
                              reinterpret_cast<int*>(smem + C::OFF_RED), hist0, 2);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 3) tmem_dealloc_cg2<512>(tmem);
}

}  // namespace k1v4
}  // namespace moep

namespace {
template <int EP, int ARCH>
int launch_v4(const moep_predict_args* a, cudaStream_t st) {
  using namespace moep::k1v4;
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
  // without the separate lo accumulator (EP = 128) the logit error is 1.5x larger
  p.tau_abs = a->tau_abs; p.tau_rel = a->tau_rel * (C::ZLO ? 1.0f : 1.5f); p.w2_norm = a->w2_norm;
  p.status = a->status;
  p.ids = a->ids; p.logits = a->logits; p.flags = a->flags; p.probs = a->probs;
  p.flag_list = a->flag_list; p.flag_count = a->flag_count;
  p.truth = a->truth; p.k = a->k; p.n_m = a->n_m; p.partials = a->partials; p.a_out = a->a_out;
  p.n_counters = moep_n_counters(a->n_m, a->n_experts);
  p.split = 1; p.zpart = nullptr; p.zpad = 0;
  const int grid = moep_num_sms() & ~1;
  kern<<<grid, NTHREADS, C::SMEM, st>>>(tx, tw1, tw2, p);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
}  // namespace

#ifdef MOEP_K1_PROF
extern "C" int moep_k1v4_trace(long long* host) {
  return cudaMemcpyFromSymbol(host, moep::k1v4::g_k1v4_trace, sizeof(long long) * 16 * 64) == cudaSuccess ? 0 : -4;
}
#endif

// v4 pair kernel (no hidden split): hidden % 256 == 0, E <= 128.
extern "C" int moep_predict_bf16_pair4(const moep_predict_args* a, void* stream) {
  if (a->n_experts > 128 || a->hidden % 256 != 0) return MOEP_EUNSUPPORTED;
  int EP = 16;
  while (EP < a->n_experts) EP *= 2;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool a1 = a->arch == 1;
  switch (EP) {
    case 16: return a1 ? launch_v4<16, 1>(a, st) : launch_v4<16, 2>(a, st);
    case 32: return a1 ? launch_v4<32, 1>(a, st) : launch_v4<32, 2>(a, st);
    case 64: return a1 ? launch_v4<64, 1>(a, st) : launch_v4<64, 2>(a, st);
    default: return a1 ? launch_v4<128, 1>(a, st) : launch_v4<128, 2>(a, st);
  }
}
