// k1_common.cuh — parameters and the per-token selection / evaluation epilogue
// shared by the fused predictor kernels.
#pragma once
#include <cstdint>
#include "sm100.cuh"
#include "common.cuh"
#include "sortnet.cuh"

namespace moep {
namespace k1c {

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
  int* status;  // bit 0: some token's fp32 logits were non-finite (host checks the input)
  float* probs;  // [N, E] fused softmax of the fp32 logits, or nullptr
  // hidden split (pair kernel, small N): `split` chunk groups per 256-token tile;
  // partial z [split][zpad][EP] and partial ||h||^2 [split][zpad] in zpart
  int split;
  float* zpart;
  int64_t zpad;
};

// mbarrier wait that traps instead of hanging forever (a lost arrival becomes a
// launch error, not a wedged GPU). try_wait carries a suspend-time hint: the
// warp sleeps until the phase completes (or the hint expires) instead of
// re-issuing the probe every ~30 cycles. Without it the spin loops of the
// TMA / MMA / epilogue waits were 35 % of the instructions K1 v4 issued (ncu
// per-instruction counts), taking issue slots from the epilogue warps on the
// same SM sub-partitions. A wait still pending after 20 s of %globaltimer traps.
#ifndef MOEP_WAIT_HINT_NS
#define MOEP_WAIT_HINT_NS 0x989680
#endif
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
#if MOEP_WAIT_HINT_NS > 0
  uint64_t t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(MOEP_WAIT_HINT_NS)
        : "memory");
    if (done) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t0 == 0) {
      t0 = t;
    } else if (t - t0 > 20000000000ull) {
      printf("moep k1: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      asm volatile("trap;");
    }
  }
#else
  uint32_t spins = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (++spins == (1u << 26)) {
      printf("moep k1: mbarrier wait timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      asm volatile("trap;");
    }
  }
#endif
}

// non-blocking probe of an mbarrier phase
__device__ __forceinline__ bool test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}

// Max-subtracted softmax of one token's logits (core.softmax, core.py:19-24:
// e = exp(z - max(z)); e / e.sum()) into out[0, E), fp32 with expf.
template <int EP, class ZGet>
__device__ __forceinline__ void softmax_row(ZGet zv, int E, float* out) {
  float mx = -INFINITY;
#pragma unroll
  for (int e = 0; e < EP; ++e)
    if (e < E) mx = fmaxf(mx, zv(e));
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < EP; ++e)
    if (e < E) s += expf(zv(e) - mx);
#pragma unroll
  for (int e = 0; e < EP; ++e)
    if (e < E) out[e] = expf(zv(e) - mx) / s;
}

// z[EP]: this token's raw GEMM2 accumulator (no b2). Every lane of the warp
// must call this (ballots). Mirrors predict_topk_batch / top_k_batch
// (predictor.py:347-351, core.py:42-48) and metrics.py:159-180.
// zrow: this thread's smem staging row (>= EP floats) used for the dynamic
// truth-expert lookups; hist: the calling warp's private [2][EP] histogram.
template <int EP, class ZGet>
__device__ __forceinline__ void row_epilogue_core(const Params& p, ZGet zv, bool flagged, float sumsq, int64_t row,
                                                  bool valid, uint32_t lane, int* hist, RowCounters& rc,
                                                  const float* zrow, uint32_t zswz) {
  int P = p.m_sel;
#pragma unroll
  for (int b = 0; b < MOEP_MAX_BOUNDS; ++b)
    if (b < p.n_bounds && p.bounds[b] > P) P = p.bounds[b];
  P = min(P + 1, min(p.E, kMaxSel));
  float tv[kMaxSel];
  int tix[kMaxSel];
  // top-P in the reference order: packed keys through a bitonic top-16
  // network (sortnet.cuh), exact whenever no two of the first P + 1 keys agree
  // in their top 26 bits; otherwise (ties, near-ties: rare) the exact
  // repeated argmax below. ~3x fewer instructions than P argmax rounds.
  bool net_ok = false;
  if constexpr (EP >= 16 && EP <= 128) {
    using namespace moep::sortnet;
    constexpr int IB = EP > 64 ? 7 : 6;  // index bits of the packed key
    uint32_t top[16], grp[16];
#pragma unroll
    for (int g0 = 0; g0 < EP; g0 += 16) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = g0 + u;
        grp[u] = e < p.E ? pk_make<IB>(okey(zv(e)), e) : 0u;  // padding sorts last
      }
      sort_desc<16>(grp);
      if (g0 == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) top[i] = grp[i];
      } else {
        merge_top<16>(top, grp);
      }
    }
    // the first P positions are exact when every adjacent pair up to position P
    // is decided above the index bits (position P: the set of the first P), P < 16
    bool amb = P >= 16;
#pragma unroll
    for (int i = 1; i < 16; ++i)
      if (i <= P) amb |= ambiguous_b<IB>(top[i - 1], top[i]);
    net_ok = !amb && (top[P < 16 ? P : 15] >> IB) != 0u;  // a NaN / padding key inside: exact path
#pragma unroll
    for (int s = 0; s < kMaxSel; ++s) {
      const int e = pk_index_b<IB>(top[s < 16 ? s : 15]);
      tv[s] = s < P ? zv(e) : -INFINITY;
      tix[s] = s < P ? e : 0;
    }
  }
  if (!net_ok) {
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
          if (!tk && zv(e) > best) { best = zv(e); bi = e; }
        }
#pragma unroll
        for (int w = 0; w < (EP + 31) / 32; ++w)
          if ((bi >> 5) == w) taken[w] |= 1u << (bi & 31);
      }
      tv[s] = best;
      tix[s] = bi;
    }
  }
  const float delta = p.tau_abs + p.tau_rel * sqrtf(sumsq) * p.w2_norm;
  // Near-tie margin. Every logit is within delta/2 of its exact value, so the
  // top-`pos` set can only change when the boundary gap v[pos-1] - v[pos] is
  // below delta, and then only for experts whose logit lies in
  // (v[pos] - delta, v[pos-1] + delta). The selection boundary (ids output)
  // flags on the gap alone; an evaluation-only boundary (1, k, m_list:
  // metrics.py:159-180 count only where the TRUE experts rank) flags only when
  // a true expert lies in that window — its counters cannot change otherwise.
  // entry value of `flagged`: this token's fp32 logits are non-finite
  if (flagged && valid && p.status) atomicOr(p.status, 1);
  const bool eval_only_ok = p.truth != nullptr && valid;
#pragma unroll
  for (int b = 0; b < MOEP_MAX_BOUNDS; ++b) {
    if (b < p.n_bounds) {
      const int pos = p.bounds[b];
      if (pos >= 1 && pos < p.E) {
        float hi_v = tv[0], lo_v = tv[1];
#pragma unroll
        for (int s = 1; s < kMaxSel; ++s)
          if (s == pos) { hi_v = tv[s - 1]; lo_v = tv[s]; }
        if (!(hi_v - lo_v >= delta)) {
          if ((p.ids && pos == p.m_sel) || !eval_only_ok) {
            flagged = true;
          } else {
            // only experts inside the window can cross this boundary. At pos == k
            // per_expert_hits names the true experts inside the top-k: any true
            // expert in the window counts. At the other positions (1: top1;
            // m: overprov / recall) only the NUMBER of true experts above the
            // boundary counts, which cannot change when the window holds true
            // experts only (or none)
            const float wlo = lo_v - delta, whi = hi_v + delta;
            int nt = 0;
            for (int j = 0; j < p.k; ++j) {
              const float zt = zrow[__ldg(p.truth + row * p.k + j) ^ zswz];
              nt += !(zt <= wlo || zt >= whi) ? 1 : 0;
            }
            if (pos == p.k) {
              flagged |= nt > 0;
            } else if (nt > 0) {
              // window experts, and how many of them are true (distinct ids:
              // a repeated true id must not mask a non-true expert)
              int nw = 0, ntw = 0;
              for (int e = 0; e < p.E; ++e) {
                const float v = zrow[e ^ zswz];  // the staged copy (written whenever truth is given)
                if (!(v <= wlo || v >= whi)) {
                  ++nw;
                  bool is_t = false;
                  for (int j = 0; j < p.k; ++j) is_t |= __ldg(p.truth + row * p.k + j) == e;
                  ntw += is_t ? 1 : 0;
                }
              }
              flagged |= nw > ntw;
            }
          }
        }
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
        if (e < p.E) lrow[e] = zv(e);
    }
    if (p.probs) softmax_row<EP>(zv, p.E, p.probs + row * p.E);
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
          if (e < p.E && (key_gt(zv(e), e, thv, thi) || e == thi)) orow[cnt++] = e;
      }
    }
  }
  if (p.truth && valid && !flagged) {
    // "truth expert t has predicted rank < m" <=> key(t) >= key(position m-1)
    // of the sorted top list (every m the caller evaluates is < kMaxSel or == E;
    // metrics.py:159-172). z_t is read from the per-row staging copy zrow.
    auto thr = [&](int m, float& v, int& i) {
      v = tv[0];
      i = tix[0];
#pragma unroll
      for (int s = 0; s < kMaxSel; ++s)
        if (s == m - 1) { v = tv[s]; i = tix[s]; }
    };
    float kv; int ki;
    thr(p.k, kv, ki);
    float mv[MOEP_MAX_BOUNDS];
    int mix[MOEP_MAX_BOUNDS];
#pragma unroll
    for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) thr(mi < p.n_m ? p.m_list[mi] : 1, mv[mi], mix[mi]);
    int inside[MOEP_MAX_BOUNDS] = {0, 0, 0, 0};
    bool any0 = false;
    for (int j = 0; j < p.k; ++j) {
      const int t = __ldg(p.truth + row * p.k + j);
      const float zt = zrow[t ^ zswz];
      any0 |= (t == tix[0]);
      const bool hit = key_gt(zt, t, kv, ki) || t == ki;
      atomicAdd(&hist[EP + t], 1);  // warp-private shared histogram
      if (hit) atomicAdd(&hist[t], 1);
#pragma unroll
      for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
        if (mi < p.n_m) {
          const int m = p.m_list[mi];
          inside[mi] += (m >= p.E || key_gt(zt, t, mv[mi], mix[mi]) || t == mix[mi]) ? 1 : 0;
        }
      }
    }
    rc.n += 1;
    rc.top1 += any0 ? 1 : 0;
#pragma unroll
    for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
      if (mi < p.n_m) {
        rc.ov[mi] += (inside[mi] == p.k) ? 1 : 0;
        rc.rc[mi] += inside[mi];
      }
    }
  }
}


// z[EP]: this token's raw GEMM2 accumulator (no b2) in registers.
template <int EP>
__device__ __forceinline__ void row_epilogue(const Params& p, float* z, float sumsq, int64_t row, bool valid,
                                             uint32_t lane, int* hist, RowCounters& rc, float* zrow,
                                             uint32_t zswz) {
  bool flagged = false;
#pragma unroll
  for (int e = 0; e < EP; ++e) {
    if (e < p.E) {
      z[e] += __ldg(p.b2 + e);
      flagged |= !isfinite(z[e]);
    } else {
      z[e] = -INFINITY;
    }
    if (p.truth) zrow[e ^ zswz] = z[e];
  }
  row_epilogue_core<EP>(p, [&](int e) { return z[e]; }, flagged, sumsq, row, valid, lane, hist, rc, zrow, zswz);
}

// Same epilogue over a token whose z + b2 is staged in shared memory (zrow,
// written by the caller for every e < EP, -inf beyond E): only the top list
// lives in registers, so the register footprint does not grow with E.
template <int EP>
__device__ __forceinline__ void row_epilogue_staged(const Params& p, bool flagged, float sumsq, int64_t row,
                                                    bool valid, uint32_t lane, int* hist, RowCounters& rc,
                                                    const float* zrow, uint32_t zswz) {
  row_epilogue_core<EP>(p, [&](int e) { return zrow[e ^ zswz]; }, flagged, sumsq, row, valid, lane, hist, rc,
                        zrow, zswz);
}

// Staging row for row_epilogue inside a 64 KB smem region (128 rows):
// EP >= 32: stride EP with the column XOR-swizzled by the lane (conflict-free);
// EP = 16: stride 17.
template <int EP>
__device__ __forceinline__ float* zstage_row(uint8_t* region, int row_in_tile, uint32_t lane, uint32_t& swz) {
  float* base = reinterpret_cast<float*>(region);
  if (EP >= 32) {
    swz = lane;
    return base + row_in_tile * EP;
  }
  swz = 0;
  return base + row_in_tile * (EP + 1);
}

// Per-CTA partial counters from the 4 warps of the selecting warpgroup
// (named barrier `bar_id`, 128 threads). red: int[4][16] smem, hist0: int[4][2][EP].
template <int EP>
__device__ __forceinline__ void write_partials(const Params& p, const RowCounters& rc, int q, uint32_t lane,
                                               int tid_in_wg, int* red0, int* hist0, int bar_id) {
  int* red = red0 + q * 16;
  const int vals[2 + 2 * MOEP_MAX_BOUNDS] = {rc.n, rc.top1, rc.ov[0], rc.ov[1], rc.ov[2],
                                              rc.ov[3], rc.rc[0], rc.rc[1], rc.rc[2], rc.rc[3]};
#pragma unroll
  for (int i = 0; i < 2 + 2 * MOEP_MAX_BOUNDS; ++i) {
    const int s = warp_sum(vals[i]);
    if (lane == 0) red[i] = s;
  }
  asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
  int* out = p.partials + static_cast<int64_t>(blockIdx.x) * p.n_counters;
  const int t = tid_in_wg;
  if (t < 2 + 2 * p.n_m) {
    const int src = t < 2 ? t : (t < 2 + p.n_m ? 2 + (t - 2) : 2 + MOEP_MAX_BOUNDS + (t - 2 - p.n_m));
    out[t] = red0[src] + red0[16 + src] + red0[32 + src] + red0[48 + src];
  }
  const int base = 2 + 2 * p.n_m;
  for (int e = t; e < p.E; e += 128) {
    int hsum = 0, tsum = 0;
    for (int w = 0; w < 4; ++w) {
      hsum += hist0[w * 2 * EP + e];
      tsum += hist0[w * 2 * EP + EP + e];
    }
    out[base + e] = hsum;
    out[base + p.E + e] = tsum;
  }
}

}  // namespace k1c
}  // namespace moep
