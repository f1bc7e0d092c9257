// k1v5_predict.cu — K1 v5: the v4 fused predictor (k1v4_predict.cu) on a
// 4-CTA cluster = two CTA pairs sharing one 256-token tile.
//
// Why: v4 streams each tile's x rows from L2 once per 256-column hidden chunk
// (8 times at h = 2048), and with 74 pairs each holding a different 1 MB x
// tile in flight the x stream misses L2 (ncu: 12.2 GB of DRAM
// traffic per 1 M tokens against 4.2 GB of algorithmic bytes). Here pair 0
// (ranks 0, 1) computes hidden chunks [0, h/512) and pair 1 (ranks 2, 3)
// chunks [h/512, h/256) of the SAME tile; x is loaded once per K-block by
// pair 0's producers and multicast into both pairs' shared memory
// (cp.async.bulk.tensor .cta_group::2 .multicast::cluster, mask {r, r+2}),
// so per tile the L2 -> SM x traffic halves and half as many distinct x
// tiles are live in L2 (37 clusters instead of 74 pairs).
//
// Each pair accumulates a partial z over its half of the hidden units (hi and
// lo accumulators in its own TMEM, as v4). The token epilogue (WG2) is split
// across the pairs by rows: in CTA r (pair r >> 1) the two WG2 warps whose
// TMEM lanes hold rows [64 (r >> 1), 64 (r >> 1) + 64) of its 128 rows SELECT,
// the other two SEND their partial z (hi + lo, fp32) and ||h||^2 partial into
// the selecting CTA's (rank r ^ 2) staging rows through distributed shared
// memory. z = (z_pair0 + z_pair1) + b2: fp32 addition of two terms is
// commutative, so the logit is the same whichever CTA selects. Each WG2 thus
// does half of v4's selection work per tile, in half of v4's tile period.
//
// Ring stages: the x half of a stage is written by pair 0's TMA into both
// pairs, so a stage is free only when both pairs' MMAs consumed it: `empty`
// counts 2 commits, each leader's commit multicast to all four CTAs (0xF).
// Pair 1's leader arms its own `full` barrier with the same byte count; the
// multicast x bytes complete on the pair leader of each destination CTA.
//
// Everything else (chunk epilogue with A2 in TMEM, GEMM2 pump, selection /
// margin / counters) is v4's; reference predictor.py:193-240, :330-351,
// core.py:27-48, metrics.py:138-193.
#include <cstdio>
#include <cuda.h>
#include "sm100.cuh"
#include "common.cuh"
#include "k1_common.cuh"
#include "tmap.cuh"

namespace moep {
namespace k1v5 {

using k1c::Params;
using k1c::wait;

constexpr int BM = 128;         // tokens per CTA (256 per pair, the same 256 in both pairs)
constexpr int BK = 64;
constexpr int HC = 256;         // hidden columns per chunk (pair MMA N)
constexpr int HB = HC / 2;
constexpr int NTHREADS = 512;
constexpr int EPI_WARP0 = 4;
constexpr int TOK_WARP0 = 12;
constexpr int PROD_REGS = 72, EPI_REGS = 160, WG2_REGS = 120;
static_assert(PROD_REGS + 2 * EPI_REGS + WG2_REGS <= 4 * 128, "register pool");

template <int EP>
struct Cfg {
  static_assert(EP <= 64, "v5: E <= 64 (lo accumulator in TMEM)");
  static constexpr int STAGES = 5;
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = HB * BK * 2;        // 16 KB
  static constexpr int W2_ROWS = EP / 2;
  static constexpr int W2_ATOM = W2_ROWS * 128;
  static constexpr int ZSTRIDE = EP >= 32 ? EP : EP + 1;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_W2 = OFF_B + STAGES * B_BYTES;
  static constexpr int OFF_Z = OFF_W2 + ((4 * W2_ATOM + 1023) / 1024) * 1024;  // 64 selected rows
  static constexpr int OFF_PSUM = OFF_Z + 64 * ZSTRIDE * 4;                   // peer ||h||^2 [64]
  static constexpr int OFF_HIST = OFF_PSUM + 64 * 4;
  static constexpr int OFF_SUMSQ = OFF_HIST + 4 * 2 * EP * 4;
  static constexpr int OFF_RED = OFF_SUMSQ + 2 * 2 * BM * 4;
  static constexpr int OFF_BAR = OFF_RED + 4 * 16 * 4;
  static constexpr int NBAR = 2 * STAGES + 16;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr uint32_t ZCOL = HC;
  static constexpr uint32_t A2COL = HC + EP;
  static constexpr uint32_t ZLCOL = A2COL + 128;
  static_assert(ZLCOL + EP <= 512, "TMEM columns");
  static_assert(SMEM <= 232448, "shared memory");
};

// 2-SM TMA load whose transaction bytes complete on the pair leader `lead`
__device__ __forceinline__ void tma_cg2(const CUtensorMap* m, uint64_t* bar, void* dst, int32_t c0, int32_t c1,
                                        uint64_t policy, uint32_t lead) {
  const uint32_t lb = mapa_shared(smem_u32(bar), lead);
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lb), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// ... multicast to the CTAs in `mask` (same smem offset); each destination's
// bytes complete on the mbarrier at this offset in that destination's pair
// leader (the peer bit of the barrier address cleared, as the 2-SM forms expect)
__device__ __forceinline__ void tma_cg2_mc(const CUtensorMap* m, uint64_t* bar, void* dst, int32_t c0, int32_t c1,
                                           uint16_t mask, uint64_t policy) {
  const uint32_t lb = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(lb), "r"(c0), "r"(c1), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tmem_st32_strided0(uint32_t taddr, const float* v, int odd) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v) + odd;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(r[0]), "r"(r[2]), "r"(r[4]), "r"(r[6]), "r"(r[8]),
        "r"(r[10]), "r"(r[12]), "r"(r[14]), "r"(r[16]), "r"(r[18]),
        "r"(r[20]), "r"(r[22]), "r"(r[24]), "r"(r[26]), "r"(r[28]),
        "r"(r[30]), "r"(r[32]), "r"(r[34]), "r"(r[36]), "r"(r[38]),
        "r"(r[40]), "r"(r[42]), "r"(r[44]), "r"(r[46]), "r"(r[48]),
        "r"(r[50]), "r"(r[52]), "r"(r[54]), "r"(r[56]), "r"(r[58]),
        "r"(r[60]), "r"(r[62])
      : "memory");
}
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// wait with acquire at cluster scope (data written by the peer CTA)
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680)
        : "memory");
    if (done) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t0 == 0) {
      t0 = t;
    } else if (t - t0 > 20000000000ull) {
      printf("moep k1v5: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      asm volatile("trap;");
    }
  }
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

template <int EP, int ARCH>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(NTHREADS, 1)
predict_quad_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w1,
                    const __grid_constant__ CUtensorMap tm_w2, const Params p) {
  using C = Cfg<EP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;                      // [STAGES] pair leader: x + W1 of both CTAs landed
  uint64_t* empty = bars + C::STAGES;         // [STAGES] local: both pairs consumed the stage
  uint64_t* acc_full = empty + C::STAGES;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* a2_full = acc_empty + 1;          // [2]
  uint64_t* a2_emptyA = a2_full + 2;
  uint64_t* a2_emptyB = a2_emptyA + 1;
  uint64_t* w2_full = a2_emptyB + 1;
  uint64_t* w2_empty = w2_full + 1;
  uint64_t* z_full = w2_empty + 1;
  uint64_t* z_empty = z_full + 1;
  uint64_t* sum_ready = z_empty + 1;          // [2]
  uint64_t* sum_empty = sum_ready + 2;        // [2]
  uint64_t* zx_full = sum_empty + 2;          // selecting CTA: the peer's partial z + ||h||^2 landed (64 lanes)
  uint64_t* zx_empty = zx_full + 1;           // sending CTA: the peer finished selecting from them (64 lanes)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const uint32_t pc = rank >> 1, r2 = rank & 1, lead = rank & ~1u;
  const bool leader = r2 == 0;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pc));
  const int cl = blockIdx.x >> 2, n_cl = gridDim.x >> 2;
  const int num_tiles = static_cast<int>((p.n_tokens + 2 * BM - 1) / (2 * BM));
  const int cpg = p.hidden / HC / 2;          // chunks per pair
  const int cbase = static_cast<int>(pc) * cpg;
  const int nk = (p.d + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
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
    mbar_init(zx_full, 64);
    mbar_init(zx_empty, 64);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x); tma_prefetch_desc(&tm_w1); tma_prefetch_desc(&tm_w2);
  }
  if (warp == 3) tmem_alloc_cg2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < EPI_WARP0) {
    regs_dec<PROD_REGS>();
    if (warp == 0) {
      // ---------------------------------------------- TMA: x rows (pair 0, multicast) + W1 half-chunk
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        const uint16_t xmask = static_cast<uint16_t>((1u << r2) | (1u << (r2 + 2)));
        uint32_t stage = 0, phase = 0;
        for (int tile = cl; tile < num_tiles; tile += n_cl) {
          const int xrow = tile * 2 * BM + r2 * BM;
          for (int c = cbase; c < cbase + cpg; ++c) {
            const int wrow = c * HC + r2 * HB;
            for (int kb = 0; kb < nk; ++kb) {
              wait(&empty[stage], phase ^ 1);
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
              if (pc == 0) tma_cg2_mc(&tm_x, &full[stage], smem + C::OFF_A + stage * C::A_BYTES, kb * BK, xrow, xmask, keep);
              tma_cg2(&tm_w1, &full[stage], smem + C::OFF_B + stage * C::B_BYTES, kb * BK, wrow, keep, lead);
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
        for (int tile = cl; tile < num_tiles; tile += n_cl) {
          for (int c = cbase; c < cbase + cpg; ++c, ++n) {
            if (n > 0) wait(w2_empty, (n - 1) & 1);
            if (leader) mbar_arrive_expect_tx(w2_full, 2 * 4 * C::W2_ATOM);
#pragma unroll
            for (int at = 0; at < 4; ++at)
              tma_cg2(&tm_w2, w2_full, smem + C::OFF_W2 + at * C::W2_ATOM, c * HC + at * 64, r2 * C::W2_ROWS, keep,
                      lead);
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
        int p_cc = 0, p_half = 2;
        uint32_t p_id = 0, p_ti = 0;
        auto pump = [&](bool block) {
          while (p_half < 2) {
            if (p_half == 0) {
              if (p_cc == 0) {
                if (block) wait(z_empty, (p_ti & 1) ^ 1);
                else if (!k1c::test(z_empty, (p_ti & 1) ^ 1)) return;
              }
              if (block) wait(w2_full, p_id & 1);
              else if (!k1c::test(w2_full, p_id & 1)) return;
            }
            if (block) wait(&a2_full[p_half], p_id & 1);
            else if (!k1c::test(&a2_full[p_half], p_id & 1)) return;
            tc_fence_after();
            const int half = p_half;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const int at = kk >> 2, w = kk & 3;
              const uint64_t bd = sdesc_k_sw128(w2_base + (half * 2 + at) * C::W2_ATOM + w * 32);
              const uint32_t acc = (p_cc | half | kk) != 0;
              umma_ts(tmem + C::ZCOL, tmem + C::A2COL + kk * 8, bd, idesc2, acc);
              umma_ts(tmem + C::ZLCOL, tmem + C::A2COL + 64 + kk * 8, bd, idesc2, acc);
            }
            if (half == 0) {
              umma_commit_mc(a2_emptyA, pair_mask);
            } else {
              umma_commit_mc(a2_emptyB, pair_mask);
              umma_commit_mc(w2_empty, pair_mask);
              if (p_cc == cpg - 1) umma_commit_mc(z_full, pair_mask);
            }
            ++p_half;
          }
        };
        for (int tile = cl; tile < num_tiles; tile += n_cl, ++ti) {
          for (int c = 0; c < cpg; ++c, ++gc) {
            wait(acc_empty, (gc & 1) ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < nk; ++kb) {
              wait(&full[stage], phase);
              tc_fence_after();
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = sdesc_k_sw128(a_base + stage * C::A_BYTES + k * 32);
                const uint64_t bd = sdesc_k_sw128(b_base + stage * C::B_BYTES + k * 32);
                umma_bf16_cg2(tmem, ad, bd, idesc1, (kb | k) != 0);
              }
              umma_commit_mc(&empty[stage], 0xF);  // both pairs' producers (the x half is shared)
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
              pump(false);
            }
            umma_commit_mc(acc_full, pair_mask);
            pump(true);
            p_cc = c; p_half = 0; p_id = gc; p_ti = ti;
          }
        }
        pump(true);
      }
    }
  } else if (warp < TOK_WARP0) {
    // ------------------------------------------------ chunk epilogue warpgroups (v4's)
    regs_inc<EPI_REGS>();
    const int wg = (warp - EPI_WARP0) >> 2;
    const uint32_t q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    float* s_sumsq = reinterpret_cast<float*>(smem + C::OFF_SUMSQ);
    uint32_t gc = 0, ti = 0;
    for (int tile = cl; tile < num_tiles; tile += n_cl, ++ti) {
      const int64_t row_g = static_cast<int64_t>(tile) * 2 * BM + r2 * BM + row_in_tile;
      float sumsq = 0.f;
      for (int c = cbase; c < cbase + cpg; ++c, ++gc) {
        wait(acc_full, gc & 1);
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
        if (lane == 0) mbar_arrive_remote(acc_empty, lead);
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
            for (int t = 0; t < 4; ++t) hv[t] = silu_f32(v[j4 * 4 + t] + bv[t]);
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
            const __nv_bfloat162 hp = __floats2bfloat162_rn(hv[t], hv[t + 1]);
            const float2 hf = __bfloat1622float2(hp);
            const __nv_bfloat162 lp = __floats2bfloat162_rn(hv[t] - hf.x, hv[t + 1] - hf.y);
            v[j4 * 4 + t] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&hp));
            v[j4 * 4 + t + 1] = __uint_as_float(*reinterpret_cast<const uint32_t*>(&lp));
          }
        }
        if (wg == 0) {
          if (gc > 0) wait(a2_emptyB, (gc - 1) & 1);
        } else {
          wait(a2_emptyA, gc & 1);
        }
        {
          const uint32_t ta2 = tmem + lane_addr + C::A2COL;
          tmem_st32_strided0(ta2, v, 0);
          tmem_st32_strided0(ta2 + 32, v + 64, 0);
          tmem_st32_strided0(ta2 + 64, v, 1);
          tmem_st32_strided0(ta2 + 96, v + 64, 1);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&a2_full[wg], lead);
      }
      if (ti >= 2) wait(&sum_empty[ti & 1], ((ti >> 1) & 1) ^ 1);
      s_sumsq[((ti & 1) * 2 + wg) * BM + row_in_tile] = sumsq;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sum_ready[ti & 1]);
    }
  } else {
    // ------------------------------------------------ WG2: per-token epilogue, rows split across the pairs
    regs_dec<WG2_REGS>();
    const uint32_t q = warp & 3;
    const bool selects = (q >> 1) == pc;       // rows [64 pc, 64 pc + 64) of this CTA's 128
    const uint32_t peer = rank ^ 2u;
    const int row_in_tile = q * 32 + lane;
    const int lr = row_in_tile & 63;           // staging row (same in both CTAs of the exchange)
    const uint32_t lane_addr = (q * 32) << 16;
    const float* s_sumsq = reinterpret_cast<const float*>(smem + C::OFF_SUMSQ);
    float* s_psum = reinterpret_cast<float*>(smem + C::OFF_PSUM);
    int* hist0 = reinterpret_cast<int*>(smem + C::OFF_HIST);
    int* hist = hist0 + q * 2 * EP;
    for (int e = lane; e < 2 * EP; e += 32) hist[e] = 0;
    RowCounters rc;
    rc.zero();
    uint32_t zswz;
    float* zrow = k1c::zstage_row<EP>(smem + C::OFF_Z, lr, lane, zswz);
    uint32_t ti = 0;
    for (int tile = cl; tile < num_tiles; tile += n_cl, ++ti) {
      const int64_t row_g = static_cast<int64_t>(tile) * 2 * BM + r2 * BM + row_in_tile;
      wait(z_full, ti & 1);
      tc_fence_after();
      if (!selects) {
        // ---- send this pair's partial z (hi + lo) and ||h||^2 to the selecting CTA
        wait_cluster(zx_empty, (ti & 1) ^ 1);
        const uint32_t rz = mapa_shared(smem_u32(zrow), peer);
#pragma unroll
        for (int j = 0; j < EP; j += 16) {
          float zc[16], zl[16];
          tmem_ld16(tmem + lane_addr + C::ZCOL + j, zc);
          tmem_ld16(tmem + lane_addr + C::ZLCOL + j, zl);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 16; ++t) st_cluster_f32(rz + 4u * ((j + t) ^ zswz), zc[t] + zl[t]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(z_empty, lead);
        wait(&sum_ready[ti & 1], (ti >> 1) & 1);
        const float sumsq = s_sumsq[((ti & 1) * 2 + 0) * BM + row_in_tile] +
                            s_sumsq[((ti & 1) * 2 + 1) * BM + row_in_tile];
        __syncwarp();
        if (lane == 0) mbar_arrive(&sum_empty[ti & 1]);
        st_cluster_f32(mapa_shared(smem_u32(s_psum + lr), peer), sumsq);
        mbar_arrive_remote(zx_full, peer);  // release.cluster: orders this lane's stores
      } else {
        // ---- own partial + the peer's -> staging row, then v4's selection
        wait_cluster(zx_full, ti & 1);
        bool bad = false;
#pragma unroll
        for (int j = 0; j < EP; j += 16) {
          float zc[16], zl[16];
          tmem_ld16(tmem + lane_addr + C::ZCOL + j, zc);
          tmem_ld16(tmem + lane_addr + C::ZLCOL + j, zl);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int e = j + t;
            float v = -INFINITY;
            if (e < p.E) {
              v = ((zc[t] + zl[t]) + zrow[e ^ zswz]) + __ldg(p.b2 + e);
              bad |= !isfinite(v);
            }
            zrow[e ^ zswz] = v;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(z_empty, lead);
        wait(&sum_ready[ti & 1], (ti >> 1) & 1);
        const float sumsq = (s_sumsq[((ti & 1) * 2 + 0) * BM + row_in_tile] +
                             s_sumsq[((ti & 1) * 2 + 1) * BM + row_in_tile]) + s_psum[lr];
        __syncwarp();
        if (lane == 0) mbar_arrive(&sum_empty[ti & 1]);
        k1c::row_epilogue_staged<EP>(p, bad, sumsq, row_g, row_g < p.n_tokens, lane, hist, rc, zrow, zswz);
        __syncwarp();
        mbar_arrive_remote(zx_empty, peer);  // staging row + psum free for the next tile
      }
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

}  // namespace k1v5
}  // namespace moep

namespace {
template <int EP, int ARCH>
int launch_v5(const moep_predict_args* a, cudaStream_t st) {
  using namespace moep::k1v5;
  using C = Cfg<EP>;
  static bool attr_set[64] = {};
  static int clusters[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = predict_quad_kernel<EP, ARCH>;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess)
      return MOEP_ELAUNCH;
    // 4-CTA clusters must fit whole into GPCs: ask how many are co-resident
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 4; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(moep_num_sms() & ~3);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) return MOEP_ELAUNCH;
    clusters[dev] = n < moep_num_sms() / 4 ? n : moep_num_sms() / 4;
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
  p.status = a->status;
  p.ids = a->ids; p.logits = a->logits; p.flags = a->flags; p.probs = a->probs;
  p.flag_list = a->flag_list; p.flag_count = a->flag_count;
  p.truth = a->truth; p.k = a->k; p.n_m = a->n_m; p.partials = a->partials; p.a_out = a->a_out;
  p.n_counters = moep_n_counters(a->n_m, a->n_experts);
  p.split = 1; p.zpart = nullptr; p.zpad = 0;
  const int grid = 4 * clusters[dev];
  // the counter reduce reads moep_num_sms() partial rows: zero the ones no CTA owns
  if (a->partials && grid < moep_num_sms() &&
      cudaMemsetAsync(a->partials + static_cast<int64_t>(grid) * p.n_counters, 0,
                      sizeof(int) * static_cast<size_t>(moep_num_sms() - grid) * p.n_counters, st) != cudaSuccess)
    return MOEP_ELAUNCH;
  kern<<<grid, NTHREADS, C::SMEM, st>>>(tx, tw1, tw2, p);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
}  // namespace

// v5 cluster kernel: E <= 64, hidden % 512 == 0.
extern "C" int moep_predict_bf16_quad5(const moep_predict_args* a, void* stream) {
  if (a->n_experts > 64 || a->hidden % 512 != 0) return MOEP_EUNSUPPORTED;
  int EP = 16;
  while (EP < a->n_experts) EP *= 2;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool a1 = a->arch == 1;
  switch (EP) {
    case 16: return a1 ? launch_v5<16, 1>(a, st) : launch_v5<16, 2>(a, st);
    case 32: return a1 ? launch_v5<32, 1>(a, st) : launch_v5<32, 2>(a, st);
    default: return a1 ? launch_v5<64, 1>(a, st) : launch_v5<64, 2>(a, st);
  }
}
