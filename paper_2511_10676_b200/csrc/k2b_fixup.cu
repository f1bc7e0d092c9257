// k2b_fixup.cu — K2 fast path: fp64 recompute of the flagged tokens as a
// register-blocked fp64 GEMM.
//
// K1 flags ~0.3 % of tokens whose selection is within the fp32 error margin;
// those must be recomputed in float64 exactly as the reference does
// (predictor.py:193-240; sigmoid :39-45; GELU-tanh :57-61). Instead of one CTA
// per token (which re-reads W1 per token), the flagged rows are treated as a
// small GEMM:
//   fix_gemm   grid (row tiles of 64) x (hidden tiles of 128): C = X_rows . W1^T
//              with 256 threads x (4 tokens x 8 hidden) fp64 register tiles,
//              double-buffered smem (A converted to fp64 once per CTA, W1 bf16
//              -> fp64 by integer ops); epilogue applies b1 + activation and
//              multiplies by the W2^T slice of its 128 hidden units, writing a
//              per-hidden-tile partial z [rows, h/128, E] (no atomics).
//   fix_finish one warp per flagged token: z = fixed-order sum of the partials
//              + b2, exact stable ranks, ids / logits / evaluation partials.
// Rows beyond the scratch capacity fall through to the per-group kernel of
// k2_fp64.cu (row_begin = capacity), so the path is exact for any count.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"

namespace moep {
namespace k2b {

constexpr int TM = 64, TN = 128, KS = 16;
#ifndef MOEP_FIX_TM
#define MOEP_FIX_TM 64  // fix_gemm rows per CTA (32: the 4-warp tile, measured slower)
#endif
#ifndef MOEP_DEC_ROWS_MAX
#define MOEP_DEC_ROWS_MAX 512
#endif
// fix-up: flagged counts up to this take dec_gemm, larger ones fix_gemm
constexpr int DEC_ROWS_MAX = MOEP_DEC_ROWS_MAX;
constexpr int NT = 256;

__device__ __forceinline__ double bf16_to_f64(uint32_t u) {
  const uint32_t t = u & 0x7fffu;
  uint32_t hi = (t << 13) + 0x38000000u;
  hi = (t == 0u) ? 0u : hi;
  hi |= (u & 0x8000u) << 16;
  double r = __hiloint2double(static_cast<int>(hi), 0);
  if (t != 0u && (t - 0x80u) >= 0x7f00u) r = static_cast<double>(__uint_as_float(u << 16));
  return r;
}

template <int T>
__device__ __forceinline__ double ld1(const void* p, int64_t i) {
  if (T == MOEP_BF16) return bf16_to_f64(reinterpret_cast<const uint16_t*>(p)[i]);
  return reinterpret_cast<const double*>(p)[i];
}

__device__ __forceinline__ double sigmoid64(double u) {
  if (u >= 0.0) return 1.0 / (1.0 + exp(-u));
  const double eu = exp(u);
  return eu / (1.0 + eu);
}
__device__ __forceinline__ double gelu64(double u) {
  const double c = 0.79788456080286535588, ga = 0.044715;
  return 0.5 * u * (1.0 + tanh(c * (u + ga * (u * u * u))));
}

// L2 load as a volatile asm statement: consecutive calls are issued back to back
// (the compiler may not sink them next to their consumers), so a batch of them
// is in flight together.
__device__ __forceinline__ double ld_cg_batched(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// fp64 MMA m8n8k4 (row.col): c[8x8] += a[8x4] * b[4x8]; lane (g = lane/4, q = lane%4)
// holds a[g][q], b[q][g], c[g][2q .. 2q+1]
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// smem: As[2][KS][AP], Bs[2][KS][BP] (k-major, padded pitches: conflict-free
// DMMA fragment reads); the epilogue reuses it for hs[TM][TN+1].
constexpr int AP = TM + 4, BP = TN + 4;

// TM_ rows x TN hidden per CTA with NT_ threads (8 or 4 warps of 32 x 32):
// 64 x 128 / 256 threads (2 CTAs per SM, the default) or 32 x 128 / 128
// threads (4 per SM). The half-size tile was meant to cut the wave
// quantisation at ~1,500 flagged rows (the 64-row grid is 1.35 waves), but
// it measured slower: 0.65-0.69 ms vs 0.62 ms per 1 M-token layer (ncu launch
// times, tools/prof_pipeline.py) -- twice the W1 tile traffic per row.
template <int XT, int WT, int TM_ = TM, int NT_ = NT>
__global__ void __launch_bounds__(NT_, 512 / NT_)
fix_gemm(moep_fp64_args a, int64_t cap, double* __restrict__ part) {
  constexpr int TM = TM_, NT = NT_, AP = TM + 4;
  static_assert(TM * TN / (NT / 32) == 32 * 32, "one 32 x 32 tile per warp");
  extern __shared__ double sm[];
  const int64_t count = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t nrows = count < cap ? count : cap;
  if (a.rows && nrows <= DEC_ROWS_MAX) return;  // dec_gemm's share
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * TM;
  if (r0 >= nrows) return;
  const int d = a.d, H = a.hidden, E = a.n_experts;
  const int h0 = blockIdx.y * TN;
  const int ntile_h = gridDim.y;
  double* As = sm;                    // [2][KS][AP]
  double* Bs = sm + 2 * KS * AP;      // [2][KS][BP]
  __shared__ int64_t rowid[TM];
  const int tid = threadIdx.x;
  if (tid < TM) {
    const int64_t it = r0 + tid;
    rowid[tid] = it < nrows ? (a.rows ? a.rows[it] : it) : -1;
  }
  __syncthreads();

  // global -> smem loaders. A tile [KS][TM]: thread = (row r = tid % 64, k-quarter
  // tid / 64) reads 4 consecutive k of its row; B tile [KS][TN]: thread = (hidden
  // row n = tid % 128, k-half tid / 128) reads 8 consecutive k (one 16-byte bf16
  // load). Global loads of tile kt+1 are issued into registers before the
  // compute of tile kt and stored (converted to fp64) after it.
  const int ar = tid & (TM - 1), akq = tid / TM;   // A: row, k-quarter (NT / TM = 4 quarters)
  static_assert(NT / TM == 4, "A loader: 4 consecutive k per thread");
  constexpr int BKH = NT / TN;                      // B k-groups covered per pass (2 or 1)
  constexpr int BPASS = 2 / BKH;                    // passes of 8 k per thread
  const int bn = tid & (TN - 1), bkh = tid / TN;   // B: hidden row, k-group
  const int64_t arow = rowid[ar];
  const int bj = h0 + bn;
  const bool vec = (d % 8) == 0;
  uint32_t ua[2], ub[BPASS][4];
  double ra[(XT == MOEP_BF16) ? 1 : 4], rb[BPASS][(WT == MOEP_BF16) ? 1 : 8];
  bool a_vec, b_vec[BPASS];
  int ka_s, kb_s[BPASS];
  auto fetch = [&](int k0) {
    const int ka = k0 + akq * 4;
    ka_s = ka;
    a_vec = vec && arow >= 0 && ka < d;
    if (a_vec) {
      if constexpr (XT == MOEP_BF16) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(a.x) + arow * d + ka));
        ua[0] = u.x; ua[1] = u.y;
      } else {
        const double2* s2 = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(a.x) + arow * d + ka);
        const double2 p0 = __ldg(s2), p1 = __ldg(s2 + 1);
        ra[0] = p0.x; ra[1] = p0.y; ra[2] = p1.x; ra[3] = p1.y;
      }
    }
#pragma unroll
    for (int pb = 0; pb < BPASS; ++pb) {
      const int kb = k0 + (bkh + pb * BKH) * 8;
      kb_s[pb] = kb;
      b_vec[pb] = vec && bj < H && kb < d;
      if (b_vec[pb]) {
        if constexpr (WT == MOEP_BF16) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.w1) +
                                                              static_cast<int64_t>(bj) * d + kb));
          ub[pb][0] = u.x; ub[pb][1] = u.y; ub[pb][2] = u.z; ub[pb][3] = u.w;
        } else {
          const double2* s2 = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(a.w1) +
                                                               static_cast<int64_t>(bj) * d + kb);
#pragma unroll
          for (int c = 0; c < 4; ++c) { const double2 v = __ldg(s2 + c); rb[pb][2 * c] = v.x; rb[pb][2 * c + 1] = v.y; }
        }
      }
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double v;
      if (a_vec) {
        if constexpr (XT == MOEP_BF16) v = bf16_to_f64((c & 1) ? (ua[c >> 1] >> 16) : (ua[c >> 1] & 0xffffu));
        else v = ra[c];
      } else {
        v = (arow >= 0 && ka_s + c < d) ? ld1<XT>(a.x, arow * d + ka_s + c) : 0.0;
      }
      As[(buf * KS + akq * 4 + c) * AP + ar] = v;
    }
#pragma unroll
    for (int pb = 0; pb < BPASS; ++pb) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double v;
        if (b_vec[pb]) {
          if constexpr (WT == MOEP_BF16) v = bf16_to_f64((c & 1) ? (ub[pb][c >> 1] >> 16) : (ub[pb][c >> 1] & 0xffffu));
          else v = rb[pb][c];
        } else {
          v = (bj < H && kb_s[pb] + c < d) ? ld1<WT>(a.w1, static_cast<int64_t>(bj) * d + kb_s[pb] + c) : 0.0;
        }
        Bs[(buf * KS + (bkh + pb * BKH) * 8 + c) * BP + bn] = v;
      }
    }
  };
  // fp64 tensor-core MMA: warp (wm, wn) owns a 32 x 32 tile = 4 x 4 m8n8 tiles;
  // lane (g, q) holds A[m + g][k + q], B[k + q][n + g], C[m + g][n + 2q .. +1]
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int WM = TM / 32;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (d + KS - 1) / KS;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) fetch((kt + 1) * KS);
#pragma unroll
    for (int k4 = 0; k4 < KS; k4 += 4) {
      double av[4], bv[4];
      const double* ap = As + (buf * KS + k4 + q4) * AP + wm * 32 + g;
      const double* bp = Bs + (buf * KS + k4 + q4) * BP + wn * 32 + g;
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = ap[8 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = bp[8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j], av[i], bv[j]);
    }
    if (kt + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
  // ---- epilogue: bias + activation -> hs [TM][TN+1]
  double* hs = sm;                               // TM * (TN + 1)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int jl = wn * 32 + 8 * j + 2 * q4 + hh, jg = h0 + jl;
      double b1 = 0.0, inv_std = 0.0, mean = 0.0, sc = 0.0, sh = 0.0;
      const bool ok = jg < H;
      if (ok) {
        b1 = a.b1[jg];
        if (a.arch == 1) {
          inv_std = 1.0 / sqrt(a.bn_var[jg] + a.bn_eps);
          mean = a.bn_mean[jg]; sc = a.bn_scale[jg]; sh = a.bn_shift[jg];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 32 + 8 * i + g;
        double hv = 0.0;
        if (ok) {
          const double av = acc[i][j][hh] + b1;
          if (a.a_out && rowid[r] >= 0) a.a_out[rowid[r] * H + jg] = av;
          if (a.arch == 2) hv = av * sigmoid64(av);
          else hv = gelu64(sc * ((av - mean) * inv_std) + sh);
        }
        hs[r * (TN + 1) + jl] = hv;
      }
    }
  }
  __syncthreads();
  // partial z for this hidden tile. E <= 256: thread = (expert e, row group);
  // each W2^T value is loaded once per thread (batches of 8) and applied to 16
  // rows; per output the sum runs over j in fixed order.
  const int jn = (H - h0) < TN ? (H - h0) : TN;
  if (E <= NT) {
    const int e = tid % E, ngr = NT / E, rg = tid / E;
    if (rg < ngr) {
      for (int rb = rg * 16; rb < TM; rb += ngr * 16) {
        double sacc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) sacc[i] = 0.0;
        for (int j0 = 0; j0 < jn; j0 += 8) {
          double w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int jj = (j0 + u < jn) ? (j0 + u) : (jn - 1);
            const double wv = ld1<WT>(a.w2t, static_cast<int64_t>(h0 + jj) * E + e);
            w[u] = (j0 + u < jn) ? wv : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (j0 + u < jn) {
#pragma unroll
              for (int i = 0; i < 16; ++i) sacc[i] = fma(hs[(rb + i) * (TN + 1) + j0 + u], w[u], sacc[i]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (rowid[rb + i] >= 0) part[((r0 + rb + i) * ntile_h + blockIdx.y) * E + e] = sacc[i];
      }
    }
  } else {
    for (int o = tid; o < TM * E; o += NT) {
      const int r = o / E, e = o - r * E;
      if (rowid[r] < 0) continue;
      double sacc = 0.0;
      const double* hr = hs + r * (TN + 1);
      for (int jl = 0; jl < jn; ++jl) sacc = fma(hr[jl], ld1<WT>(a.w2t, static_cast<int64_t>(h0 + jl) * E + e), sacc);
      part[((r0 + r) * ntile_h + blockIdx.y) * E + e] = sacc;
    }
  }
}

// one warp per flagged token: z = sum over hidden tiles (fixed order) + b2, ranks, outputs, counters
__global__ void __launch_bounds__(256)
fix_finish(moep_fp64_args a, int64_t cap, int ntile_big, const double* __restrict__ part, int n_counters) {
  extern __shared__ double zsm[];  // [8 warps][E] z values, then int ranks [8][E]
  __shared__ int scal[2 + 2 * MOEP_MAX_BOUNDS];
  const int E = a.n_experts;
  int* hist = reinterpret_cast<int*>(zsm + 8 * E) + 8 * E;  // [2E]
  int* rkall = reinterpret_cast<int*>(zsm + 8 * E);         // [8][E]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2 * E; i += 256) hist[i] = 0;
  if (threadIdx.x < 2 + 2 * MOEP_MAX_BOUNDS) scal[threadIdx.x] = 0;
  __syncthreads();
  const int64_t count = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t nrows = count < cap ? count : cap;
  if (!a.rows || nrows <= DEC_ROWS_MAX) return;  // dec_finish's share (it writes the partials)
  const int ntile_h = ntile_big;
  double* z = zsm + warp * E;
  int* rk = rkall + warp * E;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * 8 + warp; it < nrows; it += static_cast<int64_t>(gridDim.x) * 8) {
    const int64_t row = a.rows ? a.rows[it] : it;
    for (int e = lane; e < E; e += 32) {
      // fixed order; loads batched so 8 are in flight together
      double s = 0.0;
      const double* pp = part + it * ntile_h * E + e;
      int t = 0;
      for (; t + 8 <= ntile_h; t += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_cg_batched(pp + (t + u) * E);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; t < ntile_h; ++t) s += __ldcg(pp + t * E);
      z[e] = s + a.b2[e];
    }
    __syncwarp();
    for (int e = lane; e < E; e += 32) {
      const double ze = z[e];
      int r = 0;
      for (int q = 0; q < E; ++q) r += key_gt(z[q], q, ze, e) ? 1 : 0;
      rk[e] = r;
      if (a.logits64) a.logits64[row * E + e] = ze;
      if (a.logits32) a.logits32[row * E + e] = static_cast<float>(ze);
    }
    __syncwarp();
    if (lane == 0) {
      if (a.ids && a.m_sel > 0) {
        int cnt = 0;
        for (int e = 0; e < E && cnt < a.m_sel; ++e)
          if (rk[e] < a.m_sel) a.ids[row * a.m_sel + cnt++] = e;
      }
      if (a.truth) {
        int any0 = 0;
        int inside[MOEP_MAX_BOUNDS] = {0, 0, 0, 0};
        for (int j = 0; j < a.k; ++j) {
          const int tt = a.truth[row * a.k + j];
          const int r = rk[tt];
          any0 |= r == 0;
          atomicAdd(&hist[E + tt], 1);
          if (r < a.k) atomicAdd(&hist[tt], 1);
#pragma unroll
          for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi)
            if (mi < a.n_m && r < a.m_list[mi]) ++inside[mi];
        }
        atomicAdd(&scal[0], 1);
        atomicAdd(&scal[1], any0);
#pragma unroll
        for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
          if (mi < a.n_m) {
            atomicAdd(&scal[2 + mi], inside[mi] == a.k ? 1 : 0);
            atomicAdd(&scal[2 + MOEP_MAX_BOUNDS + mi], inside[mi]);
          }
        }
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (a.partials) {
    int* out = a.partials + static_cast<int64_t>(blockIdx.x) * n_counters;
    for (int t = threadIdx.x; t < n_counters; t += 256) {
      int v;
      if (t < 2) v = scal[t];
      else if (t < 2 + a.n_m) v = scal[2 + (t - 2)];
      else if (t < 2 + 2 * a.n_m) v = scal[2 + MOEP_MAX_BOUNDS + (t - 2 - a.n_m)];
      else v = hist[t - 2 - 2 * a.n_m];
      out[t] = v;
    }
  }
}

// Finish for the split-hidden partials (decode batches and small flagged
// counts): one CTA per token, thread (e, g) sums tile group g of expert e,
// groups combined in fixed order; stable ranks one expert per thread.
constexpr int FT = 1024;  // dec_finish threads

__global__ void __launch_bounds__(FT)
dec_finish(moep_fp64_args a, int64_t cap, int ntile, const double* __restrict__ part, int n_counters) {
  extern __shared__ double dsm[];
  const int E = a.n_experts;
  const int G = E >= FT ? 1 : FT / E;          // tile groups per expert
  double* ps = dsm;                            // [G][E]
  double* z = ps + G * E;                      // [E]
  int* rk = reinterpret_cast<int*>(z + E);     // [E]
  int* hist = rk + E;                          // [2E]
  __shared__ int scal[2 + 2 * MOEP_MAX_BOUNDS];
  __shared__ int wcnt[FT / 32];
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * E; i += FT) hist[i] = 0;
  if (tid < 2 + 2 * MOEP_MAX_BOUNDS) scal[tid] = 0;
  __syncthreads();
  const int64_t count = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t nall = count < cap ? count : cap;
  const bool mine = !a.rows || nall <= DEC_ROWS_MAX;
  const int64_t nrows = mine ? nall : 0;
  if (!mine && !a.partials) return;
  const int per = (ntile + G - 1) / G;
  for (int64_t it = blockIdx.x; it < nrows; it += gridDim.x) {
    const int64_t row = a.rows ? a.rows[it] : it;
    // split-hidden partials are [row][E][ntile]: the tiles of one (row, e) are contiguous
    const double* pp = part + it * E * ntile;
    for (int q = tid; q < G * E; q += FT) {
      const int e = q % E, g = q / E;
      const int tb = g * per, te = (tb + per) < ntile ? (tb + per) : ntile;
      const double* src = pp + static_cast<int64_t>(e) * ntile;
      double sacc = 0.0;
      int t = tb;
      if ((ntile & 1) == 0 && (tb & 1) == 0) {
        for (; t + 8 <= te; t += 8) {          // 4 x 16-byte loads in flight, then fixed-order adds
          const double2* s2 = reinterpret_cast<const double2*>(src + t);
          const double2 v0 = s2[0], v1 = s2[1], v2 = s2[2], v3 = s2[3];
          sacc += v0.x; sacc += v0.y; sacc += v1.x; sacc += v1.y;
          sacc += v2.x; sacc += v2.y; sacc += v3.x; sacc += v3.y;
        }
      }
      for (; t < te; ++t) sacc += src[t];
      ps[g * E + e] = sacc;
    }
    __syncthreads();
    for (int e = tid; e < E; e += FT) {
      double sacc = 0.0;
      for (int g = 0; g < G; ++g) sacc += ps[g * E + e];
      z[e] = sacc + a.b2[e];
    }
    __syncthreads();
    for (int e = tid; e < E; e += FT) {
      const double ze = z[e];
      int r = 0;
      for (int q = 0; q < E; ++q) r += key_gt(z[q], q, ze, e) ? 1 : 0;
      rk[e] = r;
      if (a.logits64) a.logits64[row * E + e] = ze;
      if (a.logits32) a.logits32[row * E + e] = static_cast<float>(ze);
    }
    __syncthreads();
    if (a.ids && a.m_sel > 0) {
      if (E <= FT) {
        // ascending ids: e is selected iff rk[e] < m; its slot = selected experts below it
        const int lane = tid & 31, warp = tid >> 5;
        const bool sel = tid < E && rk[tid] < a.m_sel;
        const unsigned b = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) wcnt[warp] = __popc(b);
        __syncthreads();
        if (sel) {
          int pos = __popc(b & ((1u << lane) - 1u));
          for (int w = 0; w < warp; ++w) pos += wcnt[w];
          a.ids[row * a.m_sel + pos] = tid;
        }
      } else if (tid == 0) {
        int cnt = 0;
        for (int e = 0; e < E && cnt < a.m_sel; ++e)
          if (rk[e] < a.m_sel) a.ids[row * a.m_sel + cnt++] = e;
      }
    }
    if (tid == 0) {
      if (a.truth) {
        int any0 = 0;
        int inside[MOEP_MAX_BOUNDS] = {0, 0, 0, 0};
        for (int j = 0; j < a.k; ++j) {
          const int tt = a.truth[row * a.k + j];
          const int r = rk[tt];
          any0 |= r == 0;
          ++hist[E + tt];
          if (r < a.k) ++hist[tt];
#pragma unroll
          for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi)
            if (mi < a.n_m && r < a.m_list[mi]) ++inside[mi];
        }
        scal[0] += 1;
        scal[1] += any0;
#pragma unroll
        for (int mi = 0; mi < MOEP_MAX_BOUNDS; ++mi) {
          if (mi < a.n_m) {
            scal[2 + mi] += inside[mi] == a.k ? 1 : 0;
            scal[2 + MOEP_MAX_BOUNDS + mi] += inside[mi];
          }
        }
      }
    }
    __syncthreads();
  }
  if (a.partials && mine) {
    int* out = a.partials + static_cast<int64_t>(blockIdx.x) * n_counters;
    for (int t = tid; t < n_counters; t += FT) {
      int v;
      if (t < 2) v = scal[t];
      else if (t < 2 + a.n_m) v = scal[2 + (t - 2)];
      else if (t < 2 + 2 * a.n_m) v = scal[2 + MOEP_MAX_BOUNDS + (t - 2 - a.n_m)];
      else v = hist[t - 2 - 2 * a.n_m];
      out[t] = v;
    }
  }
}

// ---------------------------------------------------------------- decode path
// Few tokens (TT-token tiles), hidden split over CTAs of DH units so the W1
// stream (the only sizeable traffic) is spread over every SM. K loop in chunks
// of DKC staged as fp64 in smem, transposed ([k][t], [k][j]) so a warp's
// operand reads are contiguous; warp w owns k = 16w .. 16w+15 of each chunk
// with a (TPT tokens x JPT hidden) register tile; the 8 warp partials are
// summed in fixed order, then bias + activation (predictor.py:193-240) and the
// W2 partial of this CTA's hidden units -> part[(row * ntile + tile) * E + e].
constexpr int DH = 16, DKC = 128;
#ifndef MOEP_DEC_BIG_NW
#define MOEP_DEC_BIG_NW 8
#endif
// warps of the 32-token bulk kernel (one CTA per SM). 16 warps (each K chunk
// split 16 ways) measured slower: 309 vs 240 us per 1 M-token layer at ~490
// flagged rows (profiles/r01_fixup_dec_gemm_bulk_ncu.csv)
constexpr int DEC_BIG_NW = MOEP_DEC_BIG_NW;

template <int XT, int WT, int TT>
__global__ void __launch_bounds__(256)
dec_gemm(moep_fp64_args a, int64_t cap, double* __restrict__ part) {
  constexpr int TPT = TT >= 32 ? 4 : 2;        // tokens per thread
  constexpr int NTQ = TT / TPT;                // token groups per warp
  constexpr int NHQ = 32 / NTQ;                // hidden groups per warp
  constexpr int JPT = DH / NHQ;                // hidden units per thread
  static_assert(NTQ * NHQ == 32 && JPT * NHQ == DH, "tile");
  extern __shared__ double sm[];
  double* xs = sm;                             // [2][DKC][TT]
  double* ws = sm + 2 * DKC * TT;              // [2][DKC][DH]
  const int d = a.d, H = a.hidden, E = a.n_experts;
  // rows mode (fix-up): list indices [0, min(count, cap)), only when count is small
  const int64_t count = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t n = count < cap ? count : cap;
  if (a.rows && n > DEC_ROWS_MAX) return;
  const int64_t t0 = static_cast<int64_t>(blockIdx.y) * TT;
  if (t0 >= n) return;
  __shared__ int64_t rowid[TT];
  const int h0 = blockIdx.x * DH;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < TT) rowid[tid] = (t0 + tid < n) ? (a.rows ? a.rows[t0 + tid] : t0 + tid) : -1;
  __syncthreads();
  const int tq = lane / NHQ, hq = lane % NHQ;
  double acc[TPT][JPT];
#pragma unroll
  for (int i = 0; i < TPT; ++i)
#pragma unroll
    for (int j = 0; j < JPT; ++j) acc[i][j] = 0.0;
  // staging: x chunk [TT][DKC] (TT*DKC/8 16-byte pieces), W1 chunk [DH][DKC] (256 pieces)
  auto stage = [&](int buf, int k0) {
    for (int q = tid; q < TT * (DKC / 8); q += 256) {
      const int t = q % TT, kg = q / TT;
      const int64_t row = rowid[t];
      const int k = k0 + kg * 8;
      double v[8];
      if (row >= 0 && k + 8 <= d && (d % 8) == 0) {
        if constexpr (XT == MOEP_BF16) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.x) + row * d + k));
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = bf16_to_f64((c & 1) ? (w[c >> 1] >> 16) : (w[c >> 1] & 0xffffu));
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = reinterpret_cast<const double*>(a.x)[row * d + k + c];
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = (row >= 0 && k + c < d) ? ld1<XT>(a.x, row * d + k + c) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) xs[(buf * DKC + kg * 8 + c) * TT + t] = v[c];
    }
    {
      const int j = tid % DH, kg = tid / DH;  // 16 x 16 pieces of 8
      const int jg = h0 + j, k = k0 + kg * 8;
      double v[8];
      if (jg < H && k + 8 <= d && (d % 8) == 0) {
        if constexpr (WT == MOEP_BF16) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.w1) +
                                                               static_cast<int64_t>(jg) * d + k));
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = bf16_to_f64((c & 1) ? (w[c >> 1] >> 16) : (w[c >> 1] & 0xffffu));
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = reinterpret_cast<const double*>(a.w1)[static_cast<int64_t>(jg) * d + k + c];
        }
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          v[c] = (jg < H && k + c < d) ? ld1<WT>(a.w1, static_cast<int64_t>(jg) * d + k + c) : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) ws[(buf * DKC + kg * 8 + c) * DH + j] = v[c];
    }
  };
  const int nk = (d + DKC - 1) / DKC;
  stage(0, 0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) stage(buf ^ 1, (kt + 1) * DKC);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int k = warp * 16 + s;
      double av[TPT], bv[JPT];
      const double* xp = xs + (buf * DKC + k) * TT + tq * TPT;
      const double* wp = ws + (buf * DKC + k) * DH + hq * JPT;
#pragma unroll
      for (int i = 0; i < TPT; i += 2) {
        const double2 p = *reinterpret_cast<const double2*>(xp + i);
        av[i] = p.x; av[i + 1] = p.y;
      }
#pragma unroll
      for (int j = 0; j < JPT; j += 2) {
        const double2 p = *reinterpret_cast<const double2*>(wp + j);
        bv[j] = p.x; bv[j + 1] = p.y;
      }
#pragma unroll
      for (int i = 0; i < TPT; ++i)
#pragma unroll
        for (int j = 0; j < JPT; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  // fixed-order reduction over the 8 warps' K slices
  double* red = sm;                            // [8][TT][DH]
#pragma unroll
  for (int i = 0; i < TPT; ++i)
#pragma unroll
    for (int j = 0; j < JPT; ++j) red[(warp * TT + tq * TPT + i) * DH + hq * JPT + j] = acc[i][j];
  __syncthreads();
  double* hs = sm + 8 * TT * DH;               // [TT][DH]
  for (int o = tid; o < TT * DH; o += 256) {
    const int t = o / DH, j = o % DH, jg = h0 + j;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[(w * TT + t) * DH + j];
    double hv = 0.0;
    if (jg < H && rowid[t] >= 0) {
      const double av = s + a.b1[jg];
      if (a.a_out) a.a_out[rowid[t] * H + jg] = av;
      if (a.arch == 2) {
        hv = av * sigmoid64(av);
      } else {
        const double inv_std = 1.0 / sqrt(a.bn_var[jg] + a.bn_eps);
        hv = gelu64(a.bn_scale[jg] * ((av - a.bn_mean[jg]) * inv_std) + a.bn_shift[jg]);
      }
    }
    hs[o] = hv;
  }
  __syncthreads();
  const int jn = (H - h0) < DH ? (H - h0) : DH;
  for (int o = tid; o < TT * E; o += 256) {
    const int t = o / E, e = o - t * E;
    if (rowid[t] < 0) continue;
    double s = 0.0;
    for (int j = 0; j < jn; ++j) s = fma(hs[t * DH + j], ld1<WT>(a.w2t, static_cast<int64_t>(h0 + j) * E + e), s);
    part[((t0 + t) * E + e) * gridDim.x + blockIdx.x] = s;
  }
}

// Bulk-copy variant for bf16 x / W1 with d % DKC == 0 (the serving case): the
// CTA's W1 slice [DH][d] and its token rows [TT][d] are fetched by the TMA
// engine with one 1-D bulk copy per (row, K chunk), all issued up front on
// per-chunk mbarriers, so the HBM latency is paid once instead of per chunk.
// Warp w converts and consumes only K columns 16w..16w+15 of each chunk, so
// the K loop needs no CTA-wide barrier.
template <int TT, int NW>
__global__ void __launch_bounds__(32 * NW)
dec_gemm_bulk(moep_fp64_args a, int64_t cap, double* __restrict__ part) {
  static_assert(TT % 8 == 0 && DH == 16 && (NW == 8 || NW == 16), "tile");
  constexpr int NTH = 32 * NW, KW = DKC / NW;  // threads; K columns per warp per chunk
  extern __shared__ __align__(128) uint8_t smb[];
  const int d = a.d, H = a.hidden, E = a.n_experts;
  const int rp = d + 8;                        // raw bf16 row pitch (16 B pad: 4-bank shift per row)
  const int nk = d / DKC;
  uint16_t* wraw = reinterpret_cast<uint16_t*>(smb);            // [DH][rp]
  uint16_t* xraw = wraw + DH * rp;                               // [TT][rp]
  size_t rawb = sizeof(uint16_t) * (DH + TT) * rp;                // same layout as dec_bulk_smem
  if (rawb < sizeof(double) * (NW + 1) * TT * DH) rawb = sizeof(double) * (NW + 1) * TT * DH;
  rawb = (rawb + 15) & ~static_cast<size_t>(15);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smb + rawb);        // [nseg]
  uint16_t* w2smem = (E % 8 == 0) ? reinterpret_cast<uint16_t*>(bars + 4) : nullptr;  // [DH][E]
  const int64_t count = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t n = count < cap ? count : cap;
  if (a.rows && n > DEC_ROWS_MAX) return;
  const int64_t t0 = static_cast<int64_t>(blockIdx.y) * TT;
  if (t0 >= n) return;
  __shared__ int64_t rowid[TT];
  const int h0 = blockIdx.x * DH;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nv = static_cast<int>((n - t0) < TT ? (n - t0) : TT);
  const int hv = (H - h0) < DH ? (H - h0) : DH;
  if (tid < TT) rowid[tid] = tid < nv ? (a.rows ? a.rows[t0 + tid] : t0 + tid) : -1;
  // K is fetched in NSEG segments (one bulk copy per row and segment, one
  // mbarrier per segment): few large TMA requests, and the first segment's
  // compute overlaps the rest of the transfer
  const int nseg = (nk % 4 == 0) ? 4 : ((nk % 2 == 0) ? 2 : 1);
  const int cps = nk / nseg;                   // chunks per segment
  const int segk = cps * DKC;
  if (tid == 0) {
    for (int c = 0; c < nseg; ++c) mbar_init(&bars[c], 1);
    fence_barrier_init();
    for (int c = 0; c < nseg; ++c)
      mbar_arrive_expect_tx(&bars[c], static_cast<uint32_t>((nv + hv) * segk * 2 + (c == 0 && w2smem ? hv * E * 2 : 0)));
    if (w2smem)
      bulk_g2s(w2smem, reinterpret_cast<const uint16_t*>(a.w2t) + static_cast<int64_t>(h0) * E, hv * E * 2, &bars[0]);
  }
  __syncthreads();
  {
    const int R = nv + hv;
    const uint16_t* xg = reinterpret_cast<const uint16_t*>(a.x);
    const uint16_t* wg = reinterpret_cast<const uint16_t*>(a.w1);
    for (int q = tid; q < R * nseg; q += NTH) {
      const int r = q % R, c = q / R;
      if (r < nv)
        bulk_g2s(xraw + r * rp + c * segk, xg + rowid[r] * d + c * segk, segk * 2, &bars[c]);
      else
        bulk_g2s(wraw + (r - nv) * rp + c * segk, wg + static_cast<int64_t>(h0 + r - nv) * d + c * segk, segk * 2,
                 &bars[c]);
    }
  }
  // fp64 tensor-core MMA (m8n8k4): A = x [8 tokens x 4 k], B = W1^T [4 k x 8
  // hidden], operands converted straight from the raw bf16 rows (lane (g, q)
  // reads row g, column q: rows are 4 banks apart, conflict-free)
  constexpr int MT = TT / 8;
  const int g = lane >> 2, q4 = lane & 3;
  double acc[MT][2][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const int kw = warp * KW;                    // this warp's KW columns of every chunk
  for (int c = 0; c < nk; ++c) {
    if (c % cps == 0) mbar_wait(&bars[c / cps], 0);
#pragma unroll
    for (int s4 = 0; s4 < KW / 4; ++s4) {
      const int k = c * DKC + kw + s4 * 4 + q4;
      // F2F (XU pipe) conversions: measured faster here than integer-pipe
      // rebias or a DMUL-by-2^896 rebias (both slow the DMMA issue: 240 vs
      // 261-267 us per 1 M-token layer at ~490 flagged rows)
      double av[MT], bv[2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int t = g + 8 * mt;
        av[mt] = t < nv ? static_cast<double>(__uint_as_float(static_cast<uint32_t>(xraw[t * rp + k]) << 16)) : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int jj = g + 8 * nt;
        bv[nt] = jj < hv ? static_cast<double>(__uint_as_float(static_cast<uint32_t>(wraw[jj * rp + k]) << 16)) : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
    }
  }
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < nseg; ++c) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars[c])));
  __syncthreads();
  double* red = reinterpret_cast<double*>(smb);  // [8][TT][DH], reuses the raw region (sized for it)
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        red[(warp * TT + g + 8 * mt) * DH + 8 * nt + 2 * q4 + hh] = acc[mt][nt][hh];
  __syncthreads();
  double* hs = red + NW * TT * DH;             // [TT][DH]
  for (int o = tid; o < TT * DH; o += NTH) {
    const int t = o / DH, j = o % DH, jg = h0 + j;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) sum += red[(w * TT + t) * DH + j];
    double hval = 0.0;
    if (jg < H && rowid[t] >= 0) {
      const double av = sum + a.b1[jg];
      if (a.a_out) a.a_out[rowid[t] * H + jg] = av;
      if (a.arch == 2) {
        hval = av * sigmoid64(av);
      } else {
        const double inv_std = 1.0 / sqrt(a.bn_var[jg] + a.bn_eps);
        hval = gelu64(a.bn_scale[jg] * ((av - a.bn_mean[jg]) * inv_std) + a.bn_shift[jg]);
      }
    }
    hs[o] = hval;
  }
  __syncthreads();
  // W2 partial: thread = expert e; its DH W2^T values (bulk-copied into smem
  // with the first K segment when E % 8 == 0) are reused for every token
  const uint16_t* w2t = reinterpret_cast<const uint16_t*>(a.w2t);
  const uint16_t* w2s = w2smem ? w2smem : w2t + static_cast<int64_t>(h0) * E;
  for (int e = tid; e < E; e += NTH) {
    double wv[DH];
#pragma unroll
    for (int j = 0; j < DH; ++j) {
      const int jj = j < hv ? j : hv - 1;       // clamped: unconditional loads stay batched
      const double w = static_cast<double>(__uint_as_float(static_cast<uint32_t>(w2s[jj * E + e]) << 16));
      wv[j] = j < hv ? w : 0.0;
    }
    for (int t = 0; t < nv; ++t) {
      double sum = 0.0;
#pragma unroll
      for (int j = 0; j < DH; ++j) sum = fma(hs[t * DH + j], wv[j], sum);
      part[((t0 + t) * E + e) * gridDim.x + blockIdx.x] = sum;
    }
  }
}

template <int TT, int NW>
static size_t dec_bulk_smem(int d, int E) {
  // raw rows + barriers + W2^T slice; the epilogue's warp partials + hidden tile
  // (9 * TT * DH doubles) reuse the raw rows and must not reach the W2 slice
  size_t raw = sizeof(uint16_t) * (DH + TT) * (d + 8);
  const size_t red = sizeof(double) * (NW + 1) * TT * DH;
  if (raw < red) raw = red;
  raw = (raw + 15) & ~static_cast<size_t>(15);
  return raw + sizeof(uint64_t) * 4 + sizeof(uint16_t) * DH * E;
}

}  // namespace k2b
}  // namespace moep

namespace moep {
namespace k2b {
// dec_gemm over list indices [0, cap): 8-token tiles for cap <= 8, else 32
static int launch_dec(const moep_fp64_args* a, int64_t cap, double* scratch, cudaStream_t st) {
  const int ntile = (a->hidden + DH - 1) / DH;
  // rows mode: the kernel only runs when min(count, cap) <= DEC_ROWS_MAX
  const int64_t grid_rows = (a->rows && cap > DEC_ROWS_MAX) ? DEC_ROWS_MAX : cap;
  const bool xb = a->x_dtype == MOEP_BF16, wb = a->w_dtype == MOEP_BF16;
  // bulk-copy kernel: bf16 x and W1, d a multiple of DKC, 16-byte aligned rows
  const bool bulk_ok = xb && wb && (a->d % DKC) == 0 && (reinterpret_cast<uintptr_t>(a->x) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(a->w1) & 15) == 0;
  auto gob = [&](auto kern, int tt, int nw, size_t smem) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
      return MOEP_ELAUNCH;
    dim3 grid(static_cast<unsigned>(ntile), static_cast<unsigned>((grid_rows + tt - 1) / tt));
    kern<<<grid, 32 * nw, smem, st>>>(*a, cap, scratch);
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  };
  constexpr size_t kSmemMax = 227 * 1024;
  // one CTA per SM either way (full-K staging): 32-token tiles issue 8 DMMAs
  // per 6 operand loads (16-token tiles: 4 per 4) and halve the W1 re-reads
  if (bulk_ok && grid_rows > 32 && dec_bulk_smem<32, DEC_BIG_NW>(a->d, a->n_experts) <= kSmemMax)
    return gob(dec_gemm_bulk<32, DEC_BIG_NW>, 32, DEC_BIG_NW, dec_bulk_smem<32, DEC_BIG_NW>(a->d, a->n_experts));
  if (bulk_ok && grid_rows > 8 && dec_bulk_smem<16, 8>(a->d, a->n_experts) <= kSmemMax)
    return gob(dec_gemm_bulk<16, 8>, 16, 8, dec_bulk_smem<16, 8>(a->d, a->n_experts));
  if (bulk_ok && grid_rows <= 8 && dec_bulk_smem<8, 8>(a->d, a->n_experts) <= kSmemMax)
    return gob(dec_gemm_bulk<8, 8>, 8, 8, dec_bulk_smem<8, 8>(a->d, a->n_experts));
  auto go = [&](auto kern, int tt) {
    const size_t smem = sizeof(double) * 2 * DKC * (tt + DH);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
      return MOEP_ELAUNCH;
    dim3 grid(static_cast<unsigned>(ntile), static_cast<unsigned>((grid_rows + tt - 1) / tt));
    kern<<<grid, 256, smem, st>>>(*a, cap, scratch);
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  };
  if (grid_rows <= 8) {
    if (xb && wb) return go(dec_gemm<MOEP_BF16, MOEP_BF16, 8>, 8);
    if (xb) return go(dec_gemm<MOEP_BF16, MOEP_F64, 8>, 8);
    if (wb) return go(dec_gemm<MOEP_F64, MOEP_BF16, 8>, 8);
    return go(dec_gemm<MOEP_F64, MOEP_F64, 8>, 8);
  }
  if (xb && wb) return go(dec_gemm<MOEP_BF16, MOEP_BF16, 32>, 32);
  if (xb) return go(dec_gemm<MOEP_BF16, MOEP_F64, 32>, 32);
  if (wb) return go(dec_gemm<MOEP_F64, MOEP_BF16, 32>, 32);
  return go(dec_gemm<MOEP_F64, MOEP_F64, 32>, 32);
}

// finish kernels: dec_finish for split-hidden partials (all-rows mode, or a
// flagged count <= DEC_ROWS_MAX), fix_finish for fix_gemm partials (larger
// counts); in rows mode both are launched and each exits unless the device
// count is its share. With evaluation partials every one of the num_sms
// partial rows is written by exactly one of them.
static int launch_finish(const moep_fp64_args* a, int64_t cap, double* scratch, cudaStream_t st, bool big) {
  const int E = a->n_experts;
  const int ncnt = a->truth ? moep_n_counters(a->n_m, E) : 0;
  const int nsm = moep_num_sms();
  const int G = E >= FT ? 1 : FT / E;
  const size_t dsmem = sizeof(double) * (G * E + E) + sizeof(int) * (3 * E);
  const int64_t dcap = (a->rows && cap > DEC_ROWS_MAX) ? DEC_ROWS_MAX : cap;
  const int dgrid = a->partials ? nsm : static_cast<int>(dcap < nsm ? dcap : nsm);
  dec_finish<<<dgrid, FT, dsmem, st>>>(*a, cap, (a->hidden + DH - 1) / DH, scratch, ncnt);
  if (cudaGetLastError() != cudaSuccess) return MOEP_ELAUNCH;
  if (!big) return MOEP_OK;
  const size_t fsmem = sizeof(double) * 8 * E + sizeof(int) * (8 * E + 2 * E);
  const int64_t nblk = (cap + 7) / 8;
  const int grid = a->partials ? nsm : static_cast<int>(nblk < nsm ? nblk : nsm);
  fix_finish<<<grid, 256, fsmem, st>>>(*a, cap, (a->hidden + TN - 1) / TN, scratch, ncnt);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
}  // namespace k2b
}  // namespace moep

extern "C" int moep_decode_fp64(const moep_fp64_args* a, double* scratch, void* stream) {
  using namespace moep::k2b;
  if (!a || a->n_tokens <= 0 || a->d <= 0 || a->hidden <= 0 || a->n_experts <= 0) return MOEP_ESHAPE;
  if (!a->w2t || !scratch || a->rows || a->row_begin != 0) return MOEP_EARG;
  if (a->arch != 1 && a->arch != 2) return MOEP_EARG;
  if (a->truth && (a->k < 1 || a->k > 16 || a->n_m < 0 || a->n_m > MOEP_MAX_BOUNDS)) return MOEP_EARG;
  if (a->m_sel < 0 || a->m_sel > a->n_experts) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rc = launch_dec(a, a->n_tokens, scratch, st);
  if (rc != MOEP_OK) return rc;
  return launch_finish(a, a->n_tokens, scratch, st, false);
}

extern "C" int moep_fixup_fp64(const moep_fp64_args* a, double* scratch, int64_t cap, int32_t* partials2,
                               void* stream) {
  using namespace moep::k2b;
  if (!a || a->n_tokens <= 0 || a->d <= 0 || a->hidden <= 0 || a->n_experts <= 0) return MOEP_ESHAPE;
  if (!a->w2t || !scratch || cap <= 0 || !a->rows || !a->row_count) return MOEP_EARG;
  if (a->arch != 1 && a->arch != 2) return MOEP_EARG;
  if (a->truth && (a->k < 1 || a->k > 16 || a->n_m < 0 || a->n_m > MOEP_MAX_BOUNDS)) return MOEP_EARG;
  if (a->m_sel < 0 || a->m_sel > a->n_experts) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int ntile_h = (a->hidden + TN - 1) / TN;
  // rows per CTA (see fix_gemm)
  constexpr int FTM = MOEP_FIX_TM, FNT = FTM * 4;
  const size_t smem_main = sizeof(double) * 2 * KS * (FTM + 4 + BP);
  const size_t smem_epi = sizeof(double) * (FTM * (TN + 1));
  const size_t smem = smem_main > smem_epi ? smem_main : smem_epi;
  if (smem > 200 * 1024) return MOEP_EUNSUPPORTED;
  const bool xb = a->x_dtype == MOEP_BF16, wb = a->w_dtype == MOEP_BF16;
  dim3 grid(static_cast<unsigned>((cap + FTM - 1) / FTM), ntile_h);
  auto go = [&](auto kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
      return MOEP_ELAUNCH;
    kern<<<grid, FNT, smem, st>>>(*a, cap, scratch);
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  };
  // min(count, capacity) <= DEC_ROWS_MAX (decided on the device): the
  // split-hidden kernel; larger: the GEMM. With capacity <= DEC_ROWS_MAX the
  // GEMM and its finish kernel can never run and are not launched.
  const bool big = cap > DEC_ROWS_MAX;
  int rc = MOEP_OK;
  if (big) {
    if (xb && wb) rc = go(fix_gemm<MOEP_BF16, MOEP_BF16, FTM, FNT>);
    else if (xb) rc = go(fix_gemm<MOEP_BF16, MOEP_F64, FTM, FNT>);
    else if (wb) rc = go(fix_gemm<MOEP_F64, MOEP_BF16, FTM, FNT>);
    else rc = go(fix_gemm<MOEP_F64, MOEP_F64, FTM, FNT>);
    if (rc != MOEP_OK) return rc;
  }
  rc = launch_dec(a, cap, scratch, st);
  if (rc != MOEP_OK) return rc;
  rc = launch_finish(a, cap, scratch, st, big);
  if (rc != MOEP_OK) return rc;
  // rows beyond the scratch capacity: the per-group kernel, starting at row `cap`
  if (cap >= a->n_tokens) return MOEP_OK;  // no overflow possible; partials2 untouched
  moep_fp64_args b = *a;
  b.row_begin = cap;
  b.partials = partials2;
  return moep_predict_fp64(&b, stream);
}
