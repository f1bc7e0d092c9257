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

namespace moep {
namespace k2b {

constexpr int TM = 64, TN = 128, KS = 16;
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

// smem: As[2][KS][TM], Bs[2][KS][TN]; epilogue reuses it for hs[TM][TN+1] and w2s[TN][E]
template <int XT, int WT>
__global__ void __launch_bounds__(NT, 2)
fix_gemm(moep_fp64_args a, int64_t cap, double* __restrict__ part) {
  extern __shared__ double sm[];
  const int64_t count = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t nrows = count < cap ? count : cap;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * TM;
  if (r0 >= nrows) return;
  const int d = a.d, H = a.hidden, E = a.n_experts;
  const int h0 = blockIdx.y * TN;
  const int ntile_h = gridDim.y;
  double* As = sm;                    // [2][KS][TM]
  double* Bs = sm + 2 * KS * TM;      // [2][KS][TN]
  __shared__ int64_t rowid[TM];
  const int tid = threadIdx.x;
  if (tid < TM) {
    const int64_t it = r0 + tid;
    rowid[tid] = it < nrows ? (a.rows ? a.rows[it] : it) : -1;
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads: ty -> 4 tokens, tx -> 8 hidden
  double acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  // global -> smem loaders. A tile [KS][TM]: thread = (row r = tid % 64, k-quarter
  // tid / 64) reads 4 consecutive k of its row; B tile [KS][TN]: thread = (hidden
  // row n = tid % 128, k-half tid / 128) reads 8 consecutive k (one 16-byte bf16
  // load). Consecutive lanes write consecutive smem columns: conflict-free.
  // Global loads of tile kt+1 are issued into registers before the MMA-free
  // compute of tile kt and stored (converted to fp64) after it, so their L2
  // latency overlaps the DFMA work. Vector loads when d % 8 == 0.
  const int ar = tid & (TM - 1), akq = tid / TM;   // A: row, k-quarter
  const int bn = tid & (TN - 1), bkh = tid / TN;   // B: hidden row, k-half
  const int64_t arow = rowid[ar];
  const int bj = h0 + bn;
  const bool vec = (d % 8) == 0;
  // staging registers: raw bf16 words (converted at stash time) or fp64 values
  uint32_t ua[2], ub[4];
  double ra[(XT == MOEP_BF16) ? 1 : 4], rb[(WT == MOEP_BF16) ? 1 : 8];
  bool a_ok, b_ok, a_vec, b_vec;
  int ka_s, kb_s;
  auto fetch = [&](int k0) {
    const int ka = k0 + akq * 4, kb = k0 + bkh * 8;
    ka_s = ka; kb_s = kb;
    a_ok = arow >= 0 && ka < d;
    b_ok = bj < H && kb < d;
    a_vec = vec && a_ok;
    b_vec = vec && b_ok;
    if (a_vec) {
      if constexpr (XT == MOEP_BF16) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(a.x) + arow * d + ka));
        ua[0] = u.x; ua[1] = u.y;
      } else {
        const double2* s = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(a.x) + arow * d + ka);
        const double2 p0 = __ldg(s), p1 = __ldg(s + 1);
        ra[0] = p0.x; ra[1] = p0.y; ra[2] = p1.x; ra[3] = p1.y;
      }
    }
    if (b_vec) {
      if constexpr (WT == MOEP_BF16) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(a.w1) +
                                                            static_cast<int64_t>(bj) * d + kb));
        ub[0] = u.x; ub[1] = u.y; ub[2] = u.z; ub[3] = u.w;
      } else {
        const double2* s = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(a.w1) +
                                                            static_cast<int64_t>(bj) * d + kb);
#pragma unroll
        for (int c = 0; c < 4; ++c) { const double2 v = __ldg(s + c); rb[2 * c] = v.x; rb[2 * c + 1] = v.y; }
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
      As[(buf * KS + akq * 4 + c) * TM + ar] = v;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      double v;
      if (b_vec) {
        if constexpr (WT == MOEP_BF16) v = bf16_to_f64((c & 1) ? (ub[c >> 1] >> 16) : (ub[c >> 1] & 0xffffu));
        else v = rb[c];
      } else {
        v = (bj < H && kb_s + c < d) ? ld1<WT>(a.w1, static_cast<int64_t>(bj) * d + kb_s + c) : 0.0;
      }
      Bs[(buf * KS + bkh * 8 + c) * TN + bn] = v;
    }
  };
  const int nk = (d + KS - 1) / KS;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) fetch((kt + 1) * KS);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      double av[4], bv[8];
      const double2* ap = reinterpret_cast<const double2*>(As + (buf * KS + kk) * TM + ty * 4);
      const double2 a01 = ap[0], a23 = ap[1];
      av[0] = a01.x; av[1] = a01.y; av[2] = a23.x; av[3] = a23.y;
      // thread tx owns hidden columns {jj*32 + 2*tx, jj*32 + 2*tx + 1 : jj < 4}:
      // each double2 load spans 16 consecutive lanes x 16 B -> no bank conflicts
      const double* brow = Bs + (buf * KS + kk) * TN + tx * 2;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const double2 b = *reinterpret_cast<const double2*>(brow + jj * 32);
        bv[2 * jj] = b.x;
        bv[2 * jj + 1] = b.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
  // ---- epilogue: bias + activation -> hs [TM][TN+1]; W2^T read from L2
  double* hs = sm;                               // TM * (TN + 1)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int jl = (j >> 1) * 32 + tx * 2 + (j & 1), jg = h0 + jl;
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
      const int r = ty * 4 + i;
      double hv = 0.0;
      if (ok) {
        const double av = acc[i][j] + b1;
        if (a.a_out && rowid[r] >= 0) a.a_out[rowid[r] * H + jg] = av;
        if (a.arch == 2) hv = av * sigmoid64(av);
        else hv = gelu64(sc * ((av - mean) * inv_std) + sh);
      }
      hs[r * (TN + 1) + jl] = hv;
    }
  }
  __syncthreads();
  // partial z for this hidden tile: thread owns (row, expert) pairs, fixed j order;
  // consecutive threads read consecutive experts of a W2^T row (coalesced).
  const int jn = (H - h0) < TN ? (H - h0) : TN;
  for (int o = tid; o < TM * E; o += NT) {
    const int r = o / E, e = o - r * E;
    if (rowid[r] < 0) continue;
    double s = 0.0;
    const double* hr = hs + r * (TN + 1);
    for (int jl = 0; jl < jn; ++jl) s = fma(hr[jl], ld1<WT>(a.w2t, static_cast<int64_t>(h0 + jl) * E + e), s);
    part[((r0 + r) * ntile_h + blockIdx.y) * E + e] = s;
  }
}

// one warp per flagged token: z = sum over hidden tiles (fixed order) + b2, ranks, outputs, counters
__global__ void __launch_bounds__(256)
fix_finish(moep_fp64_args a, int64_t cap, int ntile_h, const double* __restrict__ part, int n_counters) {
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
  double* z = zsm + warp * E;
  int* rk = rkall + warp * E;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * 8 + warp; it < nrows; it += static_cast<int64_t>(gridDim.x) * 8) {
    const int64_t row = a.rows ? a.rows[it] : it;
    for (int e = lane; e < E; e += 32) {
      double s = 0.0;
      for (int t = 0; t < ntile_h; ++t) s += part[(it * ntile_h + t) * E + e];
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

}  // namespace k2b
}  // namespace moep

extern "C" int moep_fixup_fp64(const moep_fp64_args* a, double* scratch, int64_t cap, int32_t* partials2,
                               void* stream) {
  using namespace moep::k2b;
  if (!a || a->n_tokens <= 0 || a->d <= 0 || a->hidden <= 0 || a->n_experts <= 0) return MOEP_ESHAPE;
  if (!a->w2t || !scratch || cap <= 0) return MOEP_EARG;
  if (a->arch != 1 && a->arch != 2) return MOEP_EARG;
  if (a->truth && (a->k < 1 || a->k > 16 || a->n_m < 0 || a->n_m > MOEP_MAX_BOUNDS)) return MOEP_EARG;
  if (a->m_sel < 0 || a->m_sel > a->n_experts) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int E = a->n_experts;
  const int ntile_h = (a->hidden + TN - 1) / TN;
  const size_t smem_main = sizeof(double) * 2 * KS * (TM + TN);
  const size_t smem_epi = sizeof(double) * (TM * (TN + 1));
  const size_t smem = smem_main > smem_epi ? smem_main : smem_epi;
  if (smem > 200 * 1024) return MOEP_EUNSUPPORTED;
  const bool xb = a->x_dtype == MOEP_BF16, wb = a->w_dtype == MOEP_BF16;
  dim3 grid(static_cast<unsigned>((cap + TM - 1) / TM), ntile_h);
  auto go = [&](auto kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
      return MOEP_ELAUNCH;
    kern<<<grid, NT, smem, st>>>(*a, cap, scratch);
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  };
  int rc;
  if (xb && wb) rc = go(fix_gemm<MOEP_BF16, MOEP_BF16>);
  else if (xb) rc = go(fix_gemm<MOEP_BF16, MOEP_F64>);
  else if (wb) rc = go(fix_gemm<MOEP_F64, MOEP_BF16>);
  else rc = go(fix_gemm<MOEP_F64, MOEP_F64>);
  if (rc != MOEP_OK) return rc;
  const int ncnt = a->truth ? moep_n_counters(a->n_m, E) : 0;
  const size_t fsmem = sizeof(double) * 8 * E + sizeof(int) * (8 * E + 2 * E);
  fix_finish<<<moep_num_sms(), 256, fsmem, st>>>(*a, cap, ntile_h, scratch, ncnt);
  if (cudaGetLastError() != cudaSuccess) return MOEP_ELAUNCH;
  // rows beyond the scratch capacity: the per-group kernel, starting at row `cap`
  moep_fp64_args b = *a;
  b.row_begin = cap;
  b.partials = partials2;
  return moep_predict_fp64(&b, stream);
}
