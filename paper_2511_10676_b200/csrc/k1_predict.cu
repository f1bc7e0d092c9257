// k1_predict.cu — K1: fused pre-attention expert predictor for sm_100a.
//
//   z = W2 . act(W1 . x + b1) + b2 ; ids = top_m(z) ; flag = near-tie(z)
//
// Restates the eval-mode forward of the reference predictor
// (pkg/src/moepredict/predictor.py:193-240, predict_logits :330-334,
// predict_topk_batch :347-351) and its selection rule (core.py:27-48), plus the
// evaluation counters of metrics.evaluate_predictions (metrics.py:138-193).
//
// Structure (one persistent CTA per SM, 12 warps):
//   warp 0      TMA producer: x tile [128 x 64] + W1 tile [128 x 64] per stage
//   warp 1      MMA issuer (one lane): GEMM1 chunk -> TMEM acc[2], GEMM2 -> TMEM z
//   warp 2      TMA producer for the W2 chunk [EP x 128]
//   warp 3      TMEM allocator
//   warps 4-11  epilogue: two warpgroups, each owns 64 of the 128 hidden
//               columns of a chunk: tcgen05.ld -> bias/act (fp32) -> split into
//               bf16 hi + lo -> swizzled smem A operand of GEMM2.
//               Warpgroup 0 also runs the per-token selection epilogue.
// Precision: GEMM1 products are exact (bf16 x bf16 -> fp32 accumulate); GEMM2
// runs on hi and lo halves of the hidden so the hidden loses < 2^-17 relative;
// any token whose decision gap is below tau is flagged for the fp64 kernel K2.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include "sm100.cuh"
#include "common.cuh"

namespace moep {
namespace k1 {

constexpr int BM = 128;        // tokens per tile (UMMA M)
constexpr int BK = 64;         // K per stage (one 128-byte swizzle row)
constexpr int HC = 128;        // hidden columns per chunk (GEMM1 UMMA N)
constexpr int NTHREADS = 384;
constexpr int EPI_WARP0 = 4;

template <int EP>
struct Cfg {
  static constexpr int STAGES = (EP <= 64) ? 4 : 3;
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = HC * BK * 2;        // 16 KB
  static constexpr int A2_BYTES = BM * 64 * 2;       // 16 KB per (hi|lo, half)
  static constexpr int W2_BYTES = EP * 64 * 2;       // per half
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
  static constexpr int OFF_A2 = OFF_B + STAGES * B_BYTES;  // [hi0, hi1, lo0, lo1]
  static constexpr int OFF_W2 = OFF_A2 + 4 * A2_BYTES;
  static constexpr int OFF_HIST = OFF_W2 + 2 * W2_BYTES;   // int32 [4 warps][2][EP]
  static constexpr int OFF_SUMSQ = OFF_HIST + 4 * 2 * EP * 4;
  static constexpr int OFF_RED = OFF_SUMSQ + BM * 4;       // int32 [4 warps][16]
  static constexpr int OFF_BAR = OFF_RED + 4 * 16 * 4;
  static constexpr int NBAR = 2 * STAGES + 2 + 2 + 2 + 1 + 2 + 2;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;  // + tmem slot + align slack
  static constexpr uint32_t ZCOL = 2 * HC;                 // TMEM column of the z accumulator
  static constexpr uint32_t ZLCOL = ZCOL + EP;             // lo-product accumulator
  static_assert(ZLCOL + EP <= 512, "TMEM columns");
};

struct Params {
  int64_t n_tokens;
  int d, hidden, E, arch;
  const float* b1;
  const float* alpha;
  const float* beta;
  const float* b2;
  int m_sel, n_bounds;
  int bounds[MOEP_MAX_BOUNDS];
  float tau_abs, tau_rel, w2_norm;
  int* ids;
  float* logits;
  uint8_t* flags;
  int* flag_list;
  int* flag_count;
  const int* truth;
  int k, n_m;
  int m_list[MOEP_MAX_BOUNDS];
  int* partials;
  int n_counters;
  float* a_out;
  int* status;
  float* probs;  // [N, E] fused softmax of the fp32 logits, or nullptr
};

// ------------------------------------------------------------------ kernel
template <int EP, int ARCH>
__global__ void __launch_bounds__(NTHREADS, 1)
predict_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w1,
               const __grid_constant__ CUtensorMap tm_w2, const Params p) {
  using C = Cfg<EP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;                       // [STAGES]
  uint64_t* empty = bars + C::STAGES;          // [STAGES]
  uint64_t* acc_full = bars + 2 * C::STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint64_t* a2_full = acc_empty + 2;           // [2] (one per column half)
  uint64_t* a2_empty = a2_full + 2;            // [1]
  uint64_t* w2_full = a2_empty + 1;            // [1]
  uint64_t* w2_empty = w2_full + 1;            // [1]
  uint64_t* z_full = w2_empty + 1;             // [1]
  uint64_t* z_empty = z_full + 1;              // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int num_tiles = static_cast<int>((p.n_tokens + BM - 1) / BM);
  const int nchunks = (p.hidden + HC - 1) / HC;
  const int nk = (p.d + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], 8); }
    mbar_init(&a2_full[0], 4); mbar_init(&a2_full[1], 4);
    mbar_init(a2_empty, 1);
    mbar_init(w2_full, 1); mbar_init(w2_empty, 1);
    mbar_init(z_full, 1); mbar_init(z_empty, 4);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x); tma_prefetch_desc(&tm_w1); tma_prefetch_desc(&tm_w2);
  }
  if (warp == 3) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (x, W1)
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      uint32_t stage = 0, phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int c = 0; c < nchunks; ++c) {
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::B_BYTES);
            tma_load_2d(&tm_x, &full[stage], smem + C::OFF_A + stage * C::A_BYTES, kb * BK,
                        tile * BM);
            tma_load_2d_hint(&tm_w1, &full[stage], smem + C::OFF_B + stage * C::B_BYTES, kb * BK,
                             c * HC, keep);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ TMA producer (W2 chunk)
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        for (int c = 0; c < nchunks; ++c) {
          mbar_wait(w2_empty, ph ^ 1);
          mbar_arrive_expect_tx(w2_full, 2 * C::W2_BYTES);
          tma_load_2d_hint(&tm_w2, w2_full, smem + C::OFF_W2, c * HC, 0, keep);
          tma_load_2d_hint(&tm_w2, w2_full, smem + C::OFF_W2 + C::W2_BYTES, c * HC + 64, 0, keep);
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc1 = idesc_bf16_f32(BM, HC);
      const uint32_t idesc2 = idesc_bf16_f32(BM, EP);
      const uint32_t a_base = smem_u32(smem + C::OFF_A), b_base = smem_u32(smem + C::OFF_B);
      const uint32_t a2_base = smem_u32(smem + C::OFF_A2), w2_base = smem_u32(smem + C::OFF_W2);
      uint32_t stage = 0, phase = 0, gc = 0, g2 = 0, ti = 0;
      auto gemm2 = [&](int cc) {
        if (cc == 0) mbar_wait(z_empty, (ti & 1) ^ 1);
        mbar_wait(&a2_full[0], g2 & 1);
        mbar_wait(&a2_full[1], g2 & 1);
        mbar_wait(w2_full, g2 & 1);
        tc_fence_after();
#pragma unroll
        for (int g = 0; g < 2; ++g) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = sdesc_k_sw128(w2_base + g * C::W2_BYTES + k * 32);
            const uint64_t ahi = sdesc_k_sw128(a2_base + g * C::A2_BYTES + k * 32);
            const uint64_t alo = sdesc_k_sw128(a2_base + (2 + g) * C::A2_BYTES + k * 32);
            umma_bf16(tmem + C::ZCOL, ahi, bd, idesc2, (cc | g | k) != 0);
            umma_bf16(tmem + C::ZLCOL, alo, bd, idesc2, (cc | g | k) != 0);
          }
        }
        umma_commit(a2_empty);
        umma_commit(w2_empty);
        if (cc == nchunks - 1) umma_commit(z_full);
        ++g2;
      };
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ti) {
        for (int c = 0; c < nchunks; ++c, ++gc) {
          const uint32_t buf = gc & 1, accph = (gc >> 1) & 1;
          mbar_wait(&acc_empty[buf], accph ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem + buf * HC;
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = sdesc_k_sw128(a_base + stage * C::A_BYTES + k * 32);
              const uint64_t bd = sdesc_k_sw128(b_base + stage * C::B_BYTES + k * 32);
              umma_bf16(dcol, ad, bd, idesc1, (kb | k) != 0);
            }
            umma_commit(&empty[stage]);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          umma_commit(&acc_full[buf]);
          if (c > 0) gemm2(c - 1);
        }
        gemm2(nchunks - 1);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------ epilogue warpgroups
    const int wg = (warp - EPI_WARP0) >> 2;   // column half of the chunk
    const uint32_t q = warp & 3;              // TMEM lane quarter
    const int row_in_tile = q * 32 + lane;
    const uint32_t lane_addr = (q * 32) << 16;
    uint8_t* a2hi = smem + C::OFF_A2 + wg * C::A2_BYTES;
    uint8_t* a2lo = smem + C::OFF_A2 + (2 + wg) * C::A2_BYTES;
    float* s_sumsq = reinterpret_cast<float*>(smem + C::OFF_SUMSQ);
    int* hist = reinterpret_cast<int*>(smem + C::OFF_HIST) + (q * 2 * EP);
    if (wg == 0) {
      for (int e = lane; e < 2 * EP; e += 32) hist[e] = 0;
    }
    RowCounters rc; rc.zero();
    uint32_t gc = 0, g2 = 0, ti = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ti) {
      float sumsq = 0.f;
      for (int c = 0; c < nchunks; ++c, ++gc, ++g2) {
        const uint32_t buf = gc & 1, accph = (gc >> 1) & 1;
        mbar_wait(&acc_full[buf], accph);
        tc_fence_after();
        float v[64];
        const uint32_t ta = tmem + lane_addr + buf * HC + wg * 64;
        tmem_ld32(ta, v);
        tmem_ld32(ta + 32, v + 32);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        // bias + activation + hi/lo split
        uint32_t hi2[32], lo2[32];
        const int col0 = c * HC + wg * 64;
        const int64_t row_g = static_cast<int64_t>(tile) * BM + row_in_tile;
#pragma unroll
        for (int j4 = 0; j4 < 16; ++j4) {
          float4 pa, pb;
          if (ARCH == 2) {
            pa = (col0 + j4 * 4 < p.hidden) ? __ldg(reinterpret_cast<const float4*>(p.b1 + col0) + j4)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            pa = (col0 + j4 * 4 < p.hidden) ? __ldg(reinterpret_cast<const float4*>(p.alpha + col0) + j4)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
            pb = (col0 + j4 * 4 < p.hidden) ? __ldg(reinterpret_cast<const float4*>(p.beta + col0) + j4)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          const float ca[4] = {pa.x, pa.y, pa.z, pa.w};
          if (ARCH == 2 && p.a_out && row_g < p.n_tokens && col0 + j4 * 4 < p.hidden) {
            // training: keep the fp32 pre-activation for the backward pass
            *reinterpret_cast<float4*>(p.a_out + row_g * p.hidden + col0 + j4 * 4) =
                make_float4(v[j4 * 4] + pa.x, v[j4 * 4 + 1] + pa.y, v[j4 * 4 + 2] + pa.z, v[j4 * 4 + 3] + pa.w);
          }
          float hv[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float acc = v[j4 * 4 + t];
            float hval;
            if (ARCH == 2) {
              hval = silu_f32(acc + ca[t]);
            } else {
              const float cb[4] = {pb.x, pb.y, pb.z, pb.w};
              hval = gelu_tanh_f32(fmaf(ca[t], acc, cb[t]));
            }
            hv[t] = hval;
            sumsq = fmaf(hval, hval, sumsq);
          }
#pragma unroll
          for (int t = 0; t < 4; t += 2) {
            const __nv_bfloat16 h0 = __float2bfloat16_rn(hv[t]);
            const __nv_bfloat16 h1 = __float2bfloat16_rn(hv[t + 1]);
            const __nv_bfloat16 l0 = __float2bfloat16_rn(hv[t] - __bfloat162float(h0));
            const __nv_bfloat16 l1 = __float2bfloat16_rn(hv[t + 1] - __bfloat162float(h1));
            hi2[j4 * 2 + t / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) |
                                  (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
            lo2[j4 * 2 + t / 2] = static_cast<uint32_t>(__bfloat16_as_ushort(l0)) |
                                  (static_cast<uint32_t>(__bfloat16_as_ushort(l1)) << 16);
          }
        }
        // wait until GEMM2 of the previous chunk has consumed the A2 buffer
        mbar_wait(a2_empty, (g2 & 1) ^ 1);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const uint32_t off = sw128_offset(row_in_tile, ch * 8);
          *reinterpret_cast<uint4*>(a2hi + off) =
              make_uint4(hi2[ch * 4], hi2[ch * 4 + 1], hi2[ch * 4 + 2], hi2[ch * 4 + 3]);
          *reinterpret_cast<uint4*>(a2lo + off) =
              make_uint4(lo2[ch * 4], lo2[ch * 4 + 1], lo2[ch * 4 + 2], lo2[ch * 4 + 3]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a2_full[wg]);
      }
      // ---- tile epilogue: ||h||^2 exchange, then selection on warpgroup 0
      if (wg == 1) s_sumsq[row_in_tile] = sumsq;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (wg == 0) {
        sumsq += s_sumsq[row_in_tile];
        mbar_wait(z_full, ti & 1);
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
        if (lane == 0) mbar_arrive(z_empty);
        const int64_t row = static_cast<int64_t>(tile) * BM + row_in_tile;
        const bool valid = row < p.n_tokens;
        bool flagged = false;
#pragma unroll
        for (int e = 0; e < EP; ++e) {
          if (e < p.E) {
            z[e] += __ldg(p.b2 + e);
            flagged |= !isfinite(z[e]);
          } else {
            z[e] = -INFINITY;
          }
        }
        if (flagged && valid && p.status) atomicOr(p.status, 1);
        // top-P by repeated first-argmax (ties -> lower index)
        int P = p.m_sel;
#pragma unroll
        for (int b = 0; b < MOEP_MAX_BOUNDS; ++b)
          if (b < p.n_bounds && p.bounds[b] > P) P = p.bounds[b];
        P = min(P + 1, min(p.E, kMaxSel));
        float tv[kMaxSel];
        int tix[kMaxSel];
        {
          uint32_t taken[(EP + 31) / 32];
#pragma unroll
          for (int w = 0; w < (EP + 31) / 32; ++w) taken[w] = 0;
#pragma unroll
          for (int s = 0; s < kMaxSel; ++s) {
            float best = -INFINITY;
            int bi = 0;
            if (s < P) {
#pragma unroll
              for (int e = 0; e < EP; ++e) {
                const bool tk = (taken[e >> 5] >> (e & 31)) & 1u;
                if (!tk && z[e] > best) { best = z[e]; bi = e; }
              }
#pragma unroll
              for (int w = 0; w < (EP + 31) / 32; ++w)
                if ((bi >> 5) == w) taken[w] |= 1u << (bi & 31);
            }
            tv[s] = best;
            tix[s] = bi;
          }
        }
        // margin check at every decision boundary
        const float delta = p.tau_abs + p.tau_rel * sqrtf(sumsq) * p.w2_norm;
#pragma unroll
        for (int b = 0; b < MOEP_MAX_BOUNDS; ++b) {
          if (b < p.n_bounds) {
            const int pos = p.bounds[b];
            if (pos >= 1 && pos < p.E) {
              float hi_v = tv[0], lo_v = tv[1];
#pragma unroll
              for (int s = 1; s < kMaxSel; ++s)
                if (s == pos) { hi_v = tv[s - 1]; lo_v = tv[s]; }
              flagged |= !(hi_v - lo_v >= delta);
            }
          }
        }
        if (valid) {
          if (p.flags) p.flags[row] = flagged ? 1 : 0;
          if (flagged) {
            const int slot = atomicAdd(p.flag_count, 1);
            p.flag_list[slot] = static_cast<int>(row);
          }
          if (p.logits) {
            float* lrow = p.logits + row * p.E;
#pragma unroll
            for (int e = 0; e < EP; ++e)
              if (e < p.E) lrow[e] = z[e];
          }
          if (p.probs) {  // fused softmax (core.py:19-24): exp(z - max) / sum
            float mx = -INFINITY, sum = 0.f;
#pragma unroll
            for (int e = 0; e < EP; ++e)
              if (e < p.E) mx = fmaxf(mx, z[e]);
#pragma unroll
            for (int e = 0; e < EP; ++e)
              if (e < p.E) sum += expf(z[e] - mx);
            float* prow = p.probs + row * p.E;
#pragma unroll
            for (int e = 0; e < EP; ++e)
              if (e < p.E) prow[e] = expf(z[e] - mx) / sum;
          }
          if (p.ids && !flagged) {
            int* orow = p.ids + row * p.m_sel;
            if (p.m_sel >= p.E) {
              for (int e = 0; e < p.E; ++e) orow[e] = e;
            } else {
              float thv = tv[0];
              int thi = tix[0];
#pragma unroll
              for (int s = 0; s < kMaxSel; ++s)
                if (s == p.m_sel - 1) { thv = tv[s]; thi = tix[s]; }
              int cnt = 0;
#pragma unroll
              for (int e = 0; e < EP; ++e)
                if (e < p.E && key_gt(z[e], e, thv, thi) | (e == thi)) orow[cnt++] = e;
            }
          }
        }
        // ---- fused evaluation counters (metrics.py:159-180) for exact rows
        if (p.truth) {
          const bool use = valid && !flagged;
          int tr[16];
          int te[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            tr[j] = 0; te[j] = -1;
            if (use && j < p.k) {
              const int t = __ldg(p.truth + row * p.k + j);
              te[j] = t;
              float zt = 0.f;
#pragma unroll
              for (int e = 0; e < EP; ++e) if (e == t) zt = z[e];
              int r = 0;
#pragma unroll
              for (int e = 0; e < EP; ++e) r += (e < p.E && key_gt(z[e], e, zt, t)) ? 1 : 0;
              tr[j] = r;
            }
          }
          if (use) {
            rc.n += 1;
            bool any0 = false;
#pragma unroll
            for (int j = 0; j < 16; ++j) any0 |= (j < p.k && tr[j] == 0);
            rc.top1 += any0 ? 1 : 0;
#pragma unroll
            for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
              if (mi < p.n_m) {
                const int m = p.m_list[mi];
                int inside = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j) inside += (j < p.k && tr[j] < m) ? 1 : 0;
                rc.ov[mi] += (inside == p.k) ? 1 : 0;
                rc.rc[mi] += inside;
              }
            }
          }
          // per-expert truth / hit histograms via warp ballots (no atomics)
          for (int e = 0; e < p.E; ++e) {
            bool has = false, hit = false;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < p.k && te[j] == e) { has = true; hit = tr[j] < p.k; }
            const uint32_t bt = __ballot_sync(0xffffffffu, has);
            const uint32_t bh = __ballot_sync(0xffffffffu, hit);
            if (lane == (e & 31)) {
              hist[e] += __popc(bh);
              hist[EP + e] += __popc(bt);
            }
          }
        }
      }
    }
    // ---- per-CTA partial counters (warpgroup 0), written without atomics
    if (wg == 0 && p.partials) {
      int* red = reinterpret_cast<int*>(smem + C::OFF_RED) + q * 16;
      const int vals[2 + 2 * MOEP_MAX_BOUNDS] = {rc.n, rc.top1, rc.ov[0], rc.ov[1], rc.ov[2],
                                                  rc.ov[3], rc.rc[0], rc.rc[1], rc.rc[2], rc.rc[3]};
#pragma unroll
      for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) {
        const int s = warp_sum(vals[i]);
        if (lane == 0) red[i] = s;
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      const int t = threadIdx.x - EPI_WARP0 * 32;
      int* out = p.partials + static_cast<int64_t>(blockIdx.x) * p.n_counters;
      int* red0 = reinterpret_cast<int*>(smem + C::OFF_RED);
      int* hist0 = reinterpret_cast<int*>(smem + C::OFF_HIST);
      if (t < 2 + 2 * p.n_m) {
        int src = t < 2 ? t : (t < 2 + p.n_m ? 2 + (t - 2) : 2 + MOEP_MAX_BOUNDS + (t - 2 - p.n_m));
        out[t] = red0[src] + red0[16 + src] + red0[32 + src] + red0[48 + src];
      }
      const int base = 2 + 2 * p.n_m;
      for (int e = t; e < p.E; e += 128) {
        int hsum = 0, tsum = 0;
        for (int w = 0; w < 4; ++w) { hsum += hist0[w * 2 * EP + e]; tsum += hist0[w * 2 * EP + EP + e]; }
        out[base + e] = hsum;
        out[base + p.E + e] = tsum;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 3) tmem_dealloc<512>(tmem);
}

}  // namespace k1
}  // namespace moep

// ---------------------------------------------------------------- launcher
#include "tmap.cuh"

namespace {
template <int EP, int ARCH>
int launch_k1(const moep_predict_args* a, cudaStream_t st, const CUtensorMap& tx,
              const CUtensorMap& tw1, const CUtensorMap& tw2) {
  using namespace moep::k1;
  using C = Cfg<EP>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = predict_kernel<EP, ARCH>;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
        cudaSuccess)
      return MOEP_ELAUNCH;
    attr_set[dev] = true;
  }
  Params p{};
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
  const int grid = moep_num_sms();
  kern<<<grid, NTHREADS, C::SMEM, st>>>(tx, tw1, tw2, p);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
}  // namespace

extern "C" int moep_predict_bf16_pair(const moep_predict_args* a, void* stream);

extern "C" int moep_predict_bf16(const moep_predict_args* a, void* stream) {
  using namespace moep::k1;
  if (!a || a->n_tokens <= 0 || a->d <= 0 || a->hidden <= 0 || a->n_experts <= 0) return MOEP_ESHAPE;
  if (a->d % 8 || a->hidden % 8) return MOEP_EALIGN;  // TMA: 16-byte row strides
  if (a->n_experts > 128) return MOEP_EUNSUPPORTED;
  if (a->arch != 1 && a->arch != 2) return MOEP_EARG;
  if (a->m_sel < 0 || (a->m_sel >= moep::kMaxSel && a->m_sel < a->n_experts)) return MOEP_EUNSUPPORTED;
  if (a->n_bounds < 0 || a->n_bounds > MOEP_MAX_BOUNDS) return MOEP_EARG;
  for (int i = 0; i < a->n_bounds; ++i)
    if (a->bounds[i] < 1 || (a->bounds[i] >= moep::kMaxSel && a->bounds[i] < a->n_experts)) return MOEP_EUNSUPPORTED;
  if (a->truth && (a->k < 1 || a->k > 16 || a->n_m < 1 || a->n_m > MOEP_MAX_BOUNDS || !a->partials)) return MOEP_EARG;
  if (!a->flag_list || !a->flag_count) return MOEP_EARG;
  if (a->arch == 2 && !a->b1) return MOEP_EARG;
  if (a->arch == 1 && (!a->act_alpha || !a->act_beta)) return MOEP_EARG;
  if (a->kernel != MOEP_K1_AUTO && a->kernel != MOEP_K1_ONE_SM && a->kernel != MOEP_K1_PAIR_V2 &&
      a->kernel != MOEP_K1_PAIR_V4 && a->kernel != MOEP_K1_QUAD_V5)
    return MOEP_EARG;
  // The CTA-pair kernels (k1v2/k1v4_predict.cu) cover hidden % 256 == 0; the
  // 1-SM kernel below handles every other shape (or kernel == MOEP_K1_ONE_SM).
  if (a->kernel != MOEP_K1_ONE_SM) {
    const int rc = moep_predict_bf16_pair(a, stream);
    if (rc != MOEP_EUNSUPPORTED) return rc;
  }
  int EP = 16;
  while (EP < a->n_experts) EP *= 2;
  CUtensorMap tx, tw1, tw2;
  if (moep::make_tmap_bf16(&tx, a->x, a->n_tokens, a->d, BM, BK) ||
      moep::make_tmap_bf16(&tw1, a->w1, a->hidden, a->d, HC, BK) ||
      moep::make_tmap_bf16(&tw2, a->w2, a->n_experts, a->hidden, EP, 64))
    return MOEP_EALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool a1 = a->arch == 1;
  switch (EP) {
    case 16: return a1 ? launch_k1<16, 1>(a, st, tx, tw1, tw2) : launch_k1<16, 2>(a, st, tx, tw1, tw2);
    case 32: return a1 ? launch_k1<32, 1>(a, st, tx, tw1, tw2) : launch_k1<32, 2>(a, st, tx, tw1, tw2);
    case 64: return a1 ? launch_k1<64, 1>(a, st, tx, tw1, tw2) : launch_k1<64, 2>(a, st, tx, tw1, tw2);
    default: return a1 ? launch_k1<128, 1>(a, st, tx, tw1, tw2) : launch_k1<128, 2>(a, st, tx, tw1, tw2);
  }
}
