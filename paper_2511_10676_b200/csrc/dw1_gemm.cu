// dw1_gemm.cu — the dW1 contraction of the training backward pass
// (predictor.py:295: grads["w1"] = da.T @ x) on the tcgen05 tensor cores.
//
//   dW1[j, i] = sum_n dA[n, j] * X[n, i]        (K = tokens n)
//
// dA comes from K5 as bf16 [n, P*h] (P = 1: bf16 mode; P = 2: the fp32
// mode's hi | lo halves, summed here as a K loop of P*n rows), X is the bf16
// input [n, d]. Both operands are token-major, i.e. MN-major for this GEMM:
// TMA loads 64 (MN) x 64 (K) boxes with a 128-byte swizzle and the UMMA
// descriptors read them MN-major (instruction-descriptor bits 15/16), so
// neither operand is ever transposed in memory.
//
// CTA pairs (cluster of 2, tcgen05.mma.cta_group::2), persistent, 256
// threads per CTA: warp 0 issues TMA (each CTA stages its 128 rows of h and
// its 128 of the tile's 256 columns of d), warp 1 of the leader the MMAs
// (M = 256, N = 256, K = 16), warps 4-7 of both CTAs drain the fp32
// accumulator (TMEM, double-buffered: 2 x 256 columns) and store it. A
// 256 x 256 pair tile reads 128 FLOP per staged byte per CTA (the 1-SM
// 128 x 256 version: 85, L2-bound at 1.02-1.13 PFLOP/s). Work item = (h tile,
// d tile, K split): the K range is split so the items fill the pairs in
// whole waves; split s writes its partial tile to workspace[s] and a
// fixed-order reduce kernel sums the splits (deterministic, no atomics; an
// in-epilogue "last split reduces" variant measured slower: 0.45 vs 0.40 ms
// for the Phi hi|lo GEMM, its row-per-lane reads are uncoalesced).
#include <cstdio>
#include <cuda.h>
#include "sm100.cuh"
#include "common.cuh"
#include "k1_common.cuh"
#include "tmap.cuh"

namespace moep {
namespace dw1 {

using k1c::wait;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 6, NTHREADS = 256;  // BM, BN / 2 per CTA; tile 256 x 256
constexpr int A_BOX = 64 * BK * 2;             // one 64 (MN) x 64 (K) bf16 box: 8 KB
constexpr int A_BYTES = (BM / 64) * A_BOX;     // 16 KB: this CTA's 128 rows of h
constexpr int B_BYTES = (BN / 2 / 64) * A_BOX; // 16 KB: this CTA's 128 of the tile's 256 columns
constexpr int OFF_B = STAGES * A_BYTES;
constexpr int OFF_BAR = OFF_B + STAGES * B_BYTES;
constexpr int SMEM = OFF_BAR + (2 * STAGES + 4) * 8 + 16 + 1024;

// MN-major, 128-byte swizzle: 64 MN elements (128 B) per K row, 8-row atoms
// of 1 KB stacked along K at SBO = 1 KB, successive 64-wide MN chunks at LBO
// = one box (8 KB). K = 16 rows per MMA = 2 atoms = +2 KB on the start address.
__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>(A_BOX >> 4) << 16;   // LBO: next 64-wide MN chunk
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO: next 8-row K atom
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16_f32_mn(uint32_t M, uint32_t N) {
  return idesc_bf16_f32(M, N) | (1u << 15) | (1u << 16);  // A and B MN-major
}

struct Params {
  int M, N;            // h, d
  int64_t k_tok;       // tokens
  int passes;          // 1 (bf16 dA) or 2 (hi | lo)
  int64_t kblocks;     // per pass
  int splits;
  int m_tiles, n_tiles;
  float* out;          // splits == 1: dW1 [M, N]; else workspace [splits][M][N]
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
dw1_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;                 // [STAGES] leader: both CTAs' stage landed
  uint64_t* empty = bars + STAGES;       // [STAGES] local: stage consumed (multicast commit)
  uint64_t* acc_full = empty + STAGES;   // [2] local (multicast commit)
  uint64_t* acc_empty = acc_full + 2;    // [2] leader: 8 epilogue warps drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&acc_full[a], 1); mbar_init(&acc_empty[a], 8); }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tm_a); tma_prefetch_desc(&tm_b); }
  if (warp == 2) tmem_alloc_cg2<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t kb_total = p.kblocks * p.passes;
  const int64_t kb_per_split = (kb_total + p.splits - 1) / p.splits;
  const int n_items = p.m_tiles * p.n_tiles * p.splits;
  // item -> (split, m tile, n tile): consecutive items share the split so a
  // wave reads the same K range of X (L2 reuse across the h tiles)
  auto decode = [&](int item, int& s, int& mt, int& nt, int64_t& k0, int64_t& k1) {
    s = item / (p.m_tiles * p.n_tiles);
    const int r = item % (p.m_tiles * p.n_tiles);
    nt = r / p.m_tiles;
    mt = r % p.m_tiles;
    k0 = s * kb_per_split;
    k1 = k0 + kb_per_split < kb_total ? k0 + kb_per_split : kb_total;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      uint32_t stage = 0, phase = 0;
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_normal();
      for (int item = pair; item < n_items; item += n_pairs) {
        int s, mt, nt;
        int64_t k0, k1;
        decode(item, s, mt, nt, k0, k1);
        for (int64_t kb = k0; kb < k1; ++kb) {
          wait(&empty[stage], phase ^ 1);
          const int pass = static_cast<int>(kb / p.kblocks);
          const int row = static_cast<int>((kb % p.kblocks) * BK);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
          uint8_t* a = smem + stage * A_BYTES;
          uint8_t* b = smem + OFF_B + stage * B_BYTES;
#pragma unroll
          for (int c = 0; c < BM / 64; ++c)
            tma_load_2d_cg2(&tm_a, &full[stage], a + c * A_BOX, pass * p.M + mt * 2 * BM + rank * BM + c * 64, row,
                            pol_a);
#pragma unroll
          for (int c = 0; c < BN / 2 / 64; ++c)
            tma_load_2d_cg2(&tm_b, &full[stage], b + c * A_BOX, nt * BN + rank * (BN / 2) + c * 64, row, pol_b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32_mn(2 * BM, BN);
      const uint32_t a_base = smem_u32(smem), b_base = smem_u32(smem + OFF_B);
      uint32_t stage = 0, phase = 0, t = 0;
      for (int item = pair; item < n_items; item += n_pairs, ++t) {
        int s, mt, nt;
        int64_t k0, k1;
        decode(item, s, mt, nt, k0, k1);
        const uint32_t acc = t & 1;
        wait(&acc_empty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int64_t kb = k0; kb < k1; ++kb) {
          wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = sdesc_mn_sw128(a_base + stage * A_BYTES + k * 2048);
            const uint64_t bd = sdesc_mn_sw128(b_base + stage * B_BYTES + k * 2048);
            umma_bf16_cg2(d_tmem, ad, bd, idesc, (kb != k0 || k != 0) ? 1u : 0u);
          }
          umma_commit_mc(&empty[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_mc(&acc_full[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t q = warp & 3;
    const uint32_t lane_addr = (q * 32) << 16;
    uint32_t t = 0;
    for (int item = pair; item < n_items; item += n_pairs, ++t) {
      int s, mt, nt;
      int64_t k0, k1;
      decode(item, s, mt, nt, k0, k1);
      const uint32_t acc = t & 1;
      wait(&acc_full[acc], (t >> 1) & 1);
      tc_fence_after();
      const int row = mt * 2 * BM + rank * BM + q * 32 + lane;
      float* orow = p.out + (static_cast<int64_t>(s) * p.M + row) * p.N + nt * BN;
      const bool vec = (p.N & 3) == 0;
      const bool empty_range = k1 <= k0;  // a split with no K blocks: its partial is zero
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(tmem + lane_addr + acc * BN + c, v);
        tmem_ld_wait();
        if (empty_range) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.0f;
        }
        if (row < p.M) {
          const int col0 = nt * BN + c;
          if (vec && col0 + 32 <= p.N) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(orow + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
            for (int j = 0; j < 32; ++j)
              if (col0 + j < p.N) orow[c + j] = v[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&acc_empty[acc], 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) tmem_dealloc_cg2<512>(tmem);
}

// dW1 = sum over splits of the workspace partials, fixed order (deterministic)
__global__ void reduce_splits_kernel(const float* __restrict__ ws, int splits, int64_t count, float* __restrict__ out) {
  const int64_t n4 = count / 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = __ldcs(reinterpret_cast<const float4*>(ws) + i);
    for (int s = 1; s < splits; ++s) {
      const float4 b = __ldcs(reinterpret_cast<const float4*>(ws + s * count) + i);
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    reinterpret_cast<float4*>(out)[i] = a;
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float a = ws[i];
    for (int s = 1; s < splits; ++s) a += ws[s * count + i];
    out[i] = a;
  }
}

// K splits: the fewest that fill the SMs in (nearly) whole waves, >= 8 K blocks each
inline int choose_splits(int tiles, int64_t kb_total, int sms) {
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 16; ++s) {
    if (kb_total / s < 8) break;
    const int items = tiles * s;
    const int waves = (items + sms - 1) / sms;
    const double eff = static_cast<double>(items) / (static_cast<double>(waves) * sms);
    if (eff > best_eff + 0.02) { best = s; best_eff = eff; }
  }
  return best;
}

}  // namespace dw1
}  // namespace moep

extern "C" int64_t moep_dw1_workspace_floats(int32_t hidden, int32_t d, int64_t n_tokens, int32_t passes) {
  using namespace moep::dw1;
  if (hidden <= 0 || d <= 0 || n_tokens <= 0 || passes < 1 || passes > 2) return 0;
  const int tiles = ((hidden + 2 * BM - 1) / (2 * BM)) * ((d + BN - 1) / BN);
  const int s = choose_splits(tiles, ((n_tokens + BK - 1) / BK) * passes, moep_num_sms() / 2);
  return s > 1 ? static_cast<int64_t>(s) * hidden * d : 0;
}

extern "C" int moep_dw1_bf16(const void* da, const void* x, int64_t n_tokens, int32_t hidden, int32_t d,
                             int32_t passes, float* dw1, float* workspace, int64_t workspace_floats, void* stream) {
  using namespace moep::dw1;
  if (n_tokens <= 0 || hidden <= 0 || d <= 0) return MOEP_ESHAPE;
  if (passes < 1 || passes > 2 || !da || !x || !dw1) return MOEP_EARG;
  if (hidden % 8 || d % 8) return MOEP_EALIGN;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(dw1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
      return MOEP_ELAUNCH;
    attr = true;
  }
  CUtensorMap ta, tb;
  // dA [n, passes*h] (hi | lo), X [n, d]: boxes of 64 rows (tokens) x 64 columns
  if (moep::make_tmap_bf16(&ta, da, n_tokens, static_cast<int64_t>(passes) * hidden, BK, 64) ||
      moep::make_tmap_bf16(&tb, x, n_tokens, d, BK, 64))
    return MOEP_EALIGN;
  Params p{};
  p.M = hidden; p.N = d; p.k_tok = n_tokens; p.passes = passes;
  p.kblocks = (n_tokens + BK - 1) / BK;
  p.m_tiles = (hidden + 2 * BM - 1) / (2 * BM);
  p.n_tiles = (d + BN - 1) / BN;
  const int sms = moep_num_sms();
  const int pairs = sms / 2;
  p.splits = choose_splits(p.m_tiles * p.n_tiles, p.kblocks * passes, pairs);
  const int64_t need = p.splits > 1 ? static_cast<int64_t>(p.splits) * hidden * d : 0;
  if (need > 0 && (!workspace || workspace_floats < need)) p.splits = 1;
  p.out = p.splits > 1 ? workspace : dw1;
  const int items = p.m_tiles * p.n_tiles * p.splits;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dw1_kernel<<<2 * (items < pairs ? items : pairs), NTHREADS, SMEM, st>>>(ta, tb, p);
  if (cudaGetLastError() != cudaSuccess) return MOEP_ELAUNCH;
  if (p.splits > 1) {
    reduce_splits_kernel<<<4 * sms, 256, 0, st>>>(workspace, p.splits, static_cast<int64_t>(hidden) * d, dw1);
    if (cudaGetLastError() != cudaSuccess) return MOEP_ELAUNCH;
  }
  return MOEP_OK;
}
