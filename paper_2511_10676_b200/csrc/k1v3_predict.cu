// k1v3_predict.cu — K1 v3: the CTA-pair fused predictor with a double-buffered
// TMEM accumulator.
//
// Same math, outputs and per-token epilogue as k1v2_predict.cu (reference:
// predictor.py:193-240, :330-351; core.py:27-48; metrics.py:138-193). v2's
// single 256-column accumulator forced a pipeline bubble at every hidden chunk
// (GEMM1 of chunk c+1 waited for the drain of chunk c: 25.6 % of the kernel in
// profiles/r01_k1_role_waits.md), and its one-half A2 buffer made the second
// epilogue warpgroup wait for GEMM2 half 0 before writing. v3:
//   * hidden chunks of up to HC = 192 columns (the last one narrower, h % 64 == 0):
//     two accumulators (TMEM columns 0 and 192) + z (column 384, EP <= 128)
//     fill the 512 columns, so GEMM1 of chunk c+1 runs while chunk c drains;
//   * A2 holds a whole chunk (3 hi + 3 lo 64-column atoms, 96 KB): WG0 writes
//     chunk columns [0, Wc/2), WG1 [Wc/2, Wc); each waits only for the GEMM2
//     half of the previous chunk that read its region;
//   * per CTA: 4 (EP <= 64) or 3 operand stages of x 128x64 + W1 96x64.
// Warp roles as v2: 0 TMA x+W1, 1 MMA issue (leader CTA), 2 TMA W2, 3 TMEM
// alloc, 4-11 epilogue (WG0 / WG1 halves of each chunk, WG0 the token epilogue).
#include <cstdio>
#include <cuda.h>
#include "sm100.cuh"
#include "common.cuh"
#include "k1_common.cuh"
#include "tmap.cuh"

namespace moep {
namespace k1v3 {

using k1c::Params;
using k1c::wait;

#ifdef MOEP_K1_PROF  // role-level wait accounting (tools/k1_prof.py), profiling build only
__device__ unsigned long long g_k1v3_prof[160][16];
#define K3_PW(slot, rep, call)                                                             \
  do {                                                                                     \
    const long long t0_ = clock64();                                                       \
    call;                                                                                  \
    if (rep) atomicAdd(&g_k1v3_prof[blockIdx.x][slot], (unsigned long long)(clock64() - t0_)); \
  } while (0)
#else
#define K3_PW(slot, rep, call) call
#endif

constexpr int BM = 128;         // tokens per CTA (256 per pair)
constexpr int BK = 64;          // K per stage
constexpr int HC = 192;         // max hidden columns per chunk (pair MMA N)
constexpr int HB = HC / 2;      // W1 rows staged per CTA
constexpr int NTHREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr uint32_t ACC1 = HC;   // TMEM column of accumulator 1
constexpr uint32_t ZCOL = 2 * HC;

template <int EP>
struct Cfg {
  static constexpr int STAGES = (EP <= 64) ? 4 : 3;
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = HB * BK * 2;        // 12 KB
  static constexpr int ATOM = BM * 64 * 2;           // 16 KB: 128 rows x 64 bf16 (SW128)
  static constexpr int W2_ROWS = EP / 2;
  static constexpr int W2_ATOM = W2_ROWS * 128;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_A2 = OFF_B + STAGES * B_BYTES;  // [hi0, lo0, hi1, lo1, hi2, lo2]
  static constexpr int OFF_W2 = OFF_A2 + 6 * ATOM;          // 3 atoms (192 columns)
  static constexpr int OFF_HIST = OFF_W2 + ((3 * W2_ATOM + 1023) / 1024) * 1024;
  static constexpr int OFF_SUMSQ = OFF_HIST + 4 * 2 * EP * 4;
  static constexpr int OFF_RED = OFF_SUMSQ + BM * 4;
  static constexpr int OFF_BAR = OFF_RED + 4 * 16 * 4;
  static constexpr int NBAR = 2 * STAGES + 14;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
};

__host__ __device__ inline int chunk_width(int c, int hidden) {
  const int rest = hidden - c * HC;
  return rest < HC ? rest : HC;
}

// hi / lo atom of A2 holding chunk column j (atoms interleaved hi, lo)
__device__ __forceinline__ uint32_t a2_hi(int atom) { return (2 * atom) * (BM * 64 * 2); }
__device__ __forceinline__ uint32_t a2_lo(int atom) { return (2 * atom + 1) * (BM * 64 * 2); }

template <int EP, int ARCH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
predict_pair3_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w1,
                     const __grid_constant__ CUtensorMap tm_w2, const Params p) {
  using C = Cfg<EP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;                      // [STAGES] leader: x+W1 of both CTAs landed
  uint64_t* empty = bars + C::STAGES;         // [STAGES] local: stage consumed (multicast commit)
  uint64_t* acc_full = empty + C::STAGES;     // [2] local: GEMM1 of a chunk done in that buffer
  uint64_t* acc_empty = acc_full + 2;         // [2] leader: 16 epilogue warps drained that buffer
  uint64_t* a2_full = acc_empty + 2;          // [2] leader: 8 warps wrote that half of the chunk
  uint64_t* a2_emptyA = a2_full + 2;          // local: GEMM2 half 0 consumed its A2 region
  uint64_t* a2_emptyB = a2_emptyA + 1;        // local: GEMM2 half 1 consumed its A2 region
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
  const int nchunks = (p.hidden + HC - 1) / HC;
  const int nk = (p.d + BK - 1) / BK;
  const int G = p.split, cpg = nchunks / G;
  const int n_items = num_tiles * G;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 16);
      mbar_init(&a2_full[b], 8);
    }
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
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < EPI_WARP0) {
    if (warp == 0) {
      // ---------------------------------------------- TMA: x rows + W1 rows of the chunk
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t stage = 0, phase = 0;
        for (int item = pair; item < n_items; item += n_pairs) {
          const int tile = item / G, c0 = (item % G) * cpg;
          const int xrow = tile * 2 * BM + rank * BM;
          for (int c = c0; c < c0 + cpg; ++c) {
            const int wrow = c * HC + rank * (chunk_width(c, p.hidden) / 2);
            for (int kb = 0; kb < nk; ++kb) {
              K3_PW(0, true, wait(&empty[stage], phase ^ 1));
              if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (C::A_BYTES + C::B_BYTES));
              tma_load_2d_cg2(&tm_x, &full[stage], smem + C::OFF_A + stage * C::A_BYTES, kb * BK, xrow, keep);
              tma_load_2d_cg2(&tm_w1, &full[stage], smem + C::OFF_B + stage * C::B_BYTES, kb * BK, wrow, keep);
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else if (warp == 2) {
      // ---------------------------------------------- TMA: W2 columns of the chunk (EP/2 rows per CTA)
      if (elect_one()) {
        const uint64_t keep = policy_evict_last();
        uint32_t n = 0;
        for (int item = pair; item < n_items; item += n_pairs) {
          const int c0 = (item % G) * cpg;
          for (int c = c0; c < c0 + cpg; ++c, ++n) {
            if (n > 0) wait(w2_empty, (n - 1) & 1);
            if (leader) mbar_arrive_expect_tx(w2_full, 2 * 3 * C::W2_ATOM);
#pragma unroll
            for (int at = 0; at < 3; ++at)
              tma_load_2d_cg2(&tm_w2, w2_full, smem + C::OFF_W2 + at * C::W2_ATOM, c * HC + at * 64,
                              rank * C::W2_ROWS, keep);
          }
        }
      }
    } else if (warp == 1 && leader) {
      // ---------------------------------------------- MMA issuer (pair leader)
      if (elect_one()) {
        const uint32_t idesc2 = idesc_bf16_f32(2 * BM, EP);
        const uint32_t a_base = smem_u32(smem + C::OFF_A), b_base = smem_u32(smem + C::OFF_B);
        const uint32_t a2_base = smem_u32(smem + C::OFF_A2), w2_base = smem_u32(smem + C::OFF_W2);
        uint32_t stage = 0, phase = 0, gc = 0, ti = 0;
        // pending GEMM2: chunk-in-item, next half (2 = none), its global index,
        // item iteration and width; issued half by half between GEMM1 K-blocks
        int p_cc = 0, p_half = 2, p_w = HC;
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
            if (block) K3_PW(4, true, wait(&a2_full[p_half], p_id & 1));
            else if (!k1c::test(&a2_full[p_half], p_id & 1)) return;
            tc_fence_after();
            const int half = p_half;
            const int s0 = half * (p_w / 32), s1 = (half + 1) * (p_w / 32);  // 16-column K steps
            for (int s = s0; s < s1; ++s) {
              const int at = s >> 2, w = s & 3;
              const uint64_t bd = sdesc_k_sw128(w2_base + at * C::W2_ATOM + w * 32);
              const uint64_t ahi = sdesc_k_sw128(a2_base + a2_hi(at) + w * 32);
              const uint64_t alo = sdesc_k_sw128(a2_base + a2_lo(at) + w * 32);
              umma_bf16_cg2(tmem + ZCOL, ahi, bd, idesc2, (p_cc | s) != 0);
              umma_bf16_cg2(tmem + ZCOL, alo, bd, idesc2, 1u);
            }
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
          const int c0 = (item % G) * cpg;
          for (int c = 0; c < cpg; ++c, ++gc) {  // c: chunk within the item
            const uint32_t b = gc & 1, u = gc >> 1;
            const int wc = chunk_width(c0 + c, p.hidden);
            const uint32_t idesc1 = idesc_bf16_f32(2 * BM, wc);
            const uint32_t acc = tmem + b * ACC1;
            K3_PW(5, true, wait(&acc_empty[b], (u & 1) ^ 1));
            tc_fence_after();
            for (int kb = 0; kb < nk; ++kb) {
              K3_PW(6, true, wait(&full[stage], phase));
              tc_fence_after();
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = sdesc_k_sw128(a_base + stage * C::A_BYTES + k * 32);
                const uint64_t bd = sdesc_k_sw128(b_base + stage * C::B_BYTES + k * 32);
                umma_bf16_cg2(acc, ad, bd, idesc1, (kb | k) != 0);
              }
              umma_commit_mc(&empty[stage], 0x3);
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
              pump(false);
            }
            umma_commit_mc(&acc_full[b], 0x3);
            pump(true);  // previous chunk's GEMM2 fully issued before this one is queued
            p_cc = c; p_half = 0; p_id = gc; p_ti = ti; p_w = wc;
          }
        }
        pump(true);
      }
    }
  } else {
    // ------------------------------------------------ epilogue warpgroups
    const int wg = (warp - EPI_WARP0) >> 2;  // 0: chunk columns [0, Wc/2), 1: [Wc/2, Wc)
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
        const uint32_t b = gc & 1, u = gc >> 1;
        const int wc = chunk_width(c, p.hidden);
        const int hw = wc >> 1;                  // this warpgroup's columns: 96, 64 or 32
        const int jbase = wg * hw;               // first chunk column of this warpgroup
        K3_PW(wg == 0 ? 7 : 11, lane == 0 && q == 0, wait(&acc_full[b], u & 1));
        tc_fence_after();
        float v[96];
        const uint32_t ta = tmem + lane_addr + b * ACC1 + jbase;
        tmem_ld32(ta, v);
        if (hw > 32) tmem_ld32(ta + 32, v + 32);
        if (hw > 64) tmem_ld32(ta + 64, v + 64);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&acc_empty[b], 0);
        // bias + activation + hi/lo split, in place per column pair (2j, 2j+1):
        // v[2j] <- packed bf16x2 hi, v[2j+1] <- packed bf16x2 lo
        const int col0 = c * HC + jbase;
#pragma unroll
        for (int j4 = 0; j4 < 24; ++j4) {
          if (j4 * 4 < hw) {
            const int col = col0 + j4 * 4;
            float hv[4];
            if (ARCH == 2) {
              const float4 bb = __ldg(reinterpret_cast<const float4*>(p.b1 + col));
              const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
              if (p.a_out && row_g < p.n_tokens)
                *reinterpret_cast<float4*>(p.a_out + row_g * p.hidden + col) = make_float4(
                    v[j4 * 4] + bv[0], v[j4 * 4 + 1] + bv[1], v[j4 * 4 + 2] + bv[2], v[j4 * 4 + 3] + bv[3]);
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
        }
        // this warpgroup's A2 region is free once the previous chunk's GEMM2
        // half that read it completed; at the first chunk of an item WG1 also
        // waits for the current chunk's half 0 (WG0 may still be using the A2
        // atoms as the token epilogue's z staging)
        if (wg == 0) {
          // the previous chunk may have been narrower (an item's last chunk), its
          // half-1 region then overlaps this one: wait for its half 1 at item start
          if (gc > 0) {
            if (c == c0) K3_PW(8, lane == 0 && q == 0, wait(a2_emptyB, (gc - 1) & 1));
            else K3_PW(8, lane == 0 && q == 0, wait(a2_emptyA, (gc - 1) & 1));
          }
        } else {
          if (c == c0) K3_PW(9, lane == 0 && q == 0, wait(a2_emptyA, gc & 1));
          else if (gc > 0) K3_PW(9, lane == 0 && q == 0, wait(a2_emptyB, (gc - 1) & 1));
        }
        uint8_t* a2 = smem + C::OFF_A2;
#pragma unroll
        for (int cb = 0; cb < 12; ++cb) {      // 16-byte chunks = 8 columns
          if (cb * 8 < hw) {
            const int j = jbase + cb * 8;      // chunk column
            const int at = j >> 6;
            const uint32_t off = sw128_offset(row_in_tile, j & 63);
            const int bq = cb * 8;
            *reinterpret_cast<uint4*>(a2 + a2_hi(at) + off) = make_uint4(
                __float_as_uint(v[bq]), __float_as_uint(v[bq + 2]), __float_as_uint(v[bq + 4]), __float_as_uint(v[bq + 6]));
            *reinterpret_cast<uint4*>(a2 + a2_lo(at) + off) = make_uint4(
                __float_as_uint(v[bq + 1]), __float_as_uint(v[bq + 3]), __float_as_uint(v[bq + 5]),
                __float_as_uint(v[bq + 7]));
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&a2_full[wg], 0);
      }
      // ---- token epilogue on warpgroup 0
      if (wg == 1) s_sumsq[row_in_tile] = sumsq;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (wg == 0) {
        sumsq += s_sumsq[row_in_tile];
        wait(z_full, ti & 1);
        tc_fence_after();
        float z[EP];
#pragma unroll
        for (int j = 0; j < EP; j += 16) tmem_ld16(tmem + lane_addr + ZCOL + j, z + j);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(z_empty, 0);
        if (G > 1) {
          float* zp = p.zpart + (static_cast<int64_t>(grp) * p.zpad + row_g) * EP;
#pragma unroll
          for (int j = 0; j < EP; j += 4) *reinterpret_cast<float4*>(zp + j) = make_float4(z[j], z[j + 1], z[j + 2], z[j + 3]);
          p.zpart[static_cast<int64_t>(G) * p.zpad * EP + static_cast<int64_t>(grp) * p.zpad + row_g] = sumsq;
        } else {
          // A2 atoms as z staging: WG1 cannot write the next item's A2 before
          // GEMM2 half 0 of its first chunk, which needs this warpgroup first
          uint32_t zswz;
          float* zrow = k1c::zstage_row<EP>(smem + C::OFF_A2, row_in_tile, lane, zswz);
          k1c::row_epilogue<EP>(p, z, sumsq, row_g, row_g < p.n_tokens, lane, hist, rc, zrow, zswz);
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
  if (threadIdx.x == 0) atomicAdd(&g_k1v3_prof[blockIdx.x][15], (unsigned long long)(clock64() - k1_t_start));
#endif
  cluster_sync();
  if (warp == 3) tmem_dealloc_cg2<512>(tmem);
}

}  // namespace k1v3
}  // namespace moep

namespace {
template <int EP, int ARCH>
int launch_v3(const moep_predict_args* a, int split, float* zpart, int64_t zpad, cudaStream_t st) {
  using namespace moep::k1v3;
  using C = Cfg<EP>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = predict_pair3_kernel<EP, ARCH>;
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
  p.ids = a->ids; p.logits = a->logits; p.flags = a->flags;
  p.flag_list = a->flag_list; p.flag_count = a->flag_count;
  p.truth = a->truth; p.k = a->k; p.n_m = a->n_m; p.partials = a->partials; p.a_out = a->a_out;
  p.n_counters = moep_n_counters(a->n_m, a->n_experts);
  p.split = split; p.zpart = zpart; p.zpad = zpad;
  kern<<<moep_num_sms() & ~1, NTHREADS, C::SMEM, st>>>(tx, tw1, tw2, p);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
}  // namespace

#ifdef MOEP_K1_PROF
extern "C" int moep_k1v3_prof(unsigned long long* host, int reset) {
  if (reset) {
    static unsigned long long zero[160][16];
    return cudaMemcpyToSymbol(moep::k1v3::g_k1v3_prof, zero, sizeof(zero)) == cudaSuccess ? 0 : -4;
  }
  return cudaMemcpyFromSymbol(host, moep::k1v3::g_k1v3_prof, sizeof(unsigned long long) * 160 * 16) == cudaSuccess
             ? 0 : -4;
}
#endif

// v3 entry, called by moep_predict_bf16_pair after the split decision; returns
// MOEP_EUNSUPPORTED when the shape is outside v3 (hidden % 64, E > 128).
extern "C" int moep_predict_bf16_pair3(const moep_predict_args* a, int split, float* zpart, int64_t zpad,
                                       void* stream) {
  if (a->hidden % 64 != 0 || a->n_experts > 128) return MOEP_EUNSUPPORTED;
  const int nchunks = (a->hidden + moep::k1v3::HC - 1) / moep::k1v3::HC;
  if (nchunks % split != 0) return MOEP_EUNSUPPORTED;
  int EP = 16;
  while (EP < a->n_experts) EP *= 2;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool a1 = a->arch == 1;
  switch (EP) {
    case 16: return a1 ? launch_v3<16, 1>(a, split, zpart, zpad, st) : launch_v3<16, 2>(a, split, zpart, zpad, st);
    case 32: return a1 ? launch_v3<32, 1>(a, split, zpart, zpad, st) : launch_v3<32, 2>(a, split, zpart, zpad, st);
    case 64: return a1 ? launch_v3<64, 1>(a, split, zpart, zpad, st) : launch_v3<64, 2>(a, split, zpart, zpad, st);
    default: return a1 ? launch_v3<128, 1>(a, split, zpart, zpad, st) : launch_v3<128, 2>(a, split, zpart, zpad, st);
  }
}
