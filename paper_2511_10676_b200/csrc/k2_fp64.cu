// k2_fp64.cu — K2: float64 predictor on CUDA cores.
//
// Recomputes z = W2 . act(W1 . x + b1) + b2 in fp64 for the tokens K1 could not
// decide exactly (near-tie margin), or for every token when the inputs are not
// bf16-representable. Per token it follows the reference's float64 formulas:
// _forward_internal eval branch (predictor.py:193-240), the branch-stable
// sigmoid (:39-45), GELU-tanh (:57-61) and BN eval (:221-224, :234). Selection
// and evaluation use exact rank counts (core.py:27-54, metrics.py:159-180).
//
// Register-tiled fp64 GEMM: a CTA takes TB tokens; each thread owns JT rows of
// W1 (hidden units) and keeps TB x JT fp64 accumulators, streaming its W1 rows
// with 16-byte loads while the TB activations for the current K index are read
// as broadcast vectors from shared memory ([d][TB] layout). The hidden pass of
// 256*JT units lands in shared memory as fp64; threads then own (token, expert)
// pairs for the GEMM2 partial sums (W2 read transposed, coalesced over experts).
#include <type_traits>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "common.cuh"

namespace moep {
namespace k2 {

constexpr int NT = 256;
constexpr int JT = 4;             // hidden rows per thread per pass
constexpr int HP = NT * JT;       // hidden units per pass (1024)
constexpr int IV = 8;             // K elements per vector load

template <int T>
__device__ __forceinline__ double ld(const void* p, int64_t i) {
  if (T == MOEP_BF16)
    return static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]));
  return reinterpret_cast<const double*>(p)[i];
}

// Exact bf16 -> fp64 with integer ops (the F2F.F64.F32 conversion path is a
// low-throughput pipe and dominated the inner loop). u holds the 16-bit
// pattern in its low half. Zero is handled inline; bf16 subnormals, inf and
// NaN (t outside [0x80, 0x7f80)) take the exact slow path.
__device__ __forceinline__ double bf16_to_f64(uint32_t u) {
  const uint32_t t = u & 0x7fffu;
  uint32_t hi = (t << 13) + 0x38000000u;  // exponent rebias 127 -> 1023
  hi = (t == 0u) ? 0u : hi;
  hi |= (u & 0x8000u) << 16;
  double r = __hiloint2double(static_cast<int>(hi), 0);
  if (t != 0u && (t - 0x80u) >= 0x7f00u) r = static_cast<double>(__uint_as_float(u << 16));
  return r;
}

// 8 consecutive weights starting at element i (i % 8 == 0) as doubles
template <int T>
__device__ __forceinline__ void ld8(const void* p, int64_t i, double* w) {
  if (T == MOEP_BF16) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p) + i));
    const uint32_t q[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      w[2 * c] = bf16_to_f64(q[c] & 0xffffu);
      w[2 * c + 1] = bf16_to_f64(q[c] >> 16);
    }
  } else {
    const double2* d2 = reinterpret_cast<const double2*>(reinterpret_cast<const double*>(p) + i);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double2 v = __ldg(d2 + c);
      w[2 * c] = v.x;
      w[2 * c + 1] = v.y;
    }
  }
}

__device__ __forceinline__ double sigmoid64(double u) {
  if (u >= 0.0) return 1.0 / (1.0 + exp(-u));
  const double eu = exp(u);
  return eu / (1.0 + eu);
}

__device__ __forceinline__ double gelu64(double u) {
  const double c = 0.79788456080286535588, ga = 0.044715;
  const double t = tanh(c * (u + ga * (u * u * u)));
  return 0.5 * u * (1.0 + t);
}

// XS: element type of the staged activations (float is exact for bf16 inputs)
template <int XT, int WT, int TB, typename XS>
__global__ void __launch_bounds__(NT, 1) fp64_kernel(moep_fp64_args a, int n_counters) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int d = a.d, H = a.hidden, E = a.n_experts;
  const int dpad = (d + IV - 1) / IV * IV;
  double* hs = reinterpret_cast<double*>(smem_raw);       // [TB][HP]
  double* zacc = hs + TB * HP;                              // [TB][E]
  XS* xs = reinterpret_cast<XS*>(zacc + TB * E);            // [dpad][TB]
  int* rk = reinterpret_cast<int*>(xs + static_cast<int64_t>(dpad) * TB);  // [TB][E]
  int* hist = rk + TB * E;                                  // [2E]
  __shared__ int scal[2 + 2 * MOEP_MAX_BOUNDS];
  __shared__ int64_t rowid[TB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2 * E; i += NT) hist[i] = 0;
  if (tid < 2 + 2 * MOEP_MAX_BOUNDS) scal[tid] = 0;
  const int64_t nall = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  const int64_t nrows = nall > a.row_begin ? nall - a.row_begin : 0;  // rows handled here
  const int64_t ngroups = (nrows + TB - 1) / TB;
  const bool vec_ok = (d % IV) == 0;
  __syncthreads();
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t left = nrows - g * TB;
    const int nt = left < TB ? static_cast<int>(left) : TB;
    if (tid < TB) {
      const int64_t it = a.row_begin + g * TB + tid;
      rowid[tid] = tid < nt ? (a.rows ? a.rows[it] : it) : -1;
    }
    __syncthreads();
    for (int i = tid; i < dpad * TB; i += NT) {
      const int c = i / TB, t = i - c * TB;
      xs[i] = (rowid[t] >= 0 && c < d) ? static_cast<XS>(ld<XT>(a.x, rowid[t] * d + c)) : XS(0);
    }
    for (int i = tid; i < TB * E; i += NT) zacc[i] = 0.0;
    __syncthreads();
    for (int h0 = 0; h0 < H; h0 += HP) {
      // ---- GEMM1 pass: TB tokens x JT hidden rows per thread, fp64 accumulate
      double acc[JT][TB];
#pragma unroll
      for (int q = 0; q < JT; ++q)
#pragma unroll
        for (int t = 0; t < TB; ++t) acc[q][t] = 0.0;
      int jrow[JT];
#pragma unroll
      for (int q = 0; q < JT; ++q) jrow[q] = h0 + tid + NT * q;
      if (vec_ok) {
        for (int i = 0; i < d; i += IV) {
          double w[JT][IV];
#pragma unroll
          for (int q = 0; q < JT; ++q) {
            if (jrow[q] < H) ld8<WT>(a.w1, static_cast<int64_t>(jrow[q]) * d + i, w[q]);
            else {
#pragma unroll
              for (int c = 0; c < IV; ++c) w[q][c] = 0.0;
            }
          }
#pragma unroll
          for (int c = 0; c < IV; ++c) {
            double xv[TB];
#pragma unroll
            for (int t = 0; t < TB; ++t) xv[t] = static_cast<double>(xs[(i + c) * TB + t]);
#pragma unroll
            for (int q = 0; q < JT; ++q)
#pragma unroll
              for (int t = 0; t < TB; ++t) acc[q][t] = fma(xv[t], w[q][c], acc[q][t]);
          }
        }
      } else {
        for (int i = 0; i < d; ++i) {
          double xv[TB];
#pragma unroll
          for (int t = 0; t < TB; ++t) xv[t] = static_cast<double>(xs[i * TB + t]);
#pragma unroll
          for (int q = 0; q < JT; ++q) {
            const double w = jrow[q] < H ? ld<WT>(a.w1, static_cast<int64_t>(jrow[q]) * d + i) : 0.0;
#pragma unroll
            for (int t = 0; t < TB; ++t) acc[q][t] = fma(xv[t], w, acc[q][t]);
          }
        }
      }
      // ---- activation (fp64, reference formulas) -> hs
#pragma unroll
      for (int q = 0; q < JT; ++q) {
        const int j = jrow[q];
        const int jl = tid + NT * q;
        if (j < H) {
          const double b1 = a.b1[j];
          if (a.a_out) {
#pragma unroll
            for (int t = 0; t < TB; ++t)
              if (t < nt) a.a_out[rowid[t] * H + j] = acc[q][t] + b1;
          }
          if (a.arch == 2) {
#pragma unroll
            for (int t = 0; t < TB; ++t) {
              const double av = acc[q][t] + b1;
              hs[t * HP + jl] = av * sigmoid64(av);
            }
          } else {
            const double inv_std = 1.0 / sqrt(a.bn_var[j] + a.bn_eps);
            const double mean = a.bn_mean[j], sc = a.bn_scale[j], sh = a.bn_shift[j];
#pragma unroll
            for (int t = 0; t < TB; ++t) {
              const double a_hat = (acc[q][t] + b1 - mean) * inv_std;
              hs[t * HP + jl] = gelu64(sc * a_hat + sh);
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < TB; ++t) hs[t * HP + jl] = 0.0;
        }
      }
      __syncthreads();
      // ---- GEMM2 partial: thread owns (token, expert) pairs; fixed j order
      const int jn = min(HP, H - h0);
      for (int o = tid; o < TB * E; o += NT) {
        const int t = o / E, e = o - t * E;
        double s = zacc[o];
        const double* hrow = hs + t * HP;
        for (int jl = 0; jl < jn; ++jl)
          s = fma(hrow[jl], ld<WT>(a.w2t, static_cast<int64_t>(h0 + jl) * E + e), s);
        zacc[o] = s;
      }
      __syncthreads();
    }
    for (int o = tid; o < TB * E; o += NT) zacc[o] += a.b2[o % E];
    __syncthreads();
    // ---- exact stable ranks; warp t handles token t
    for (int t = warp; t < nt; t += NT / 32) {
      const double* zr = zacc + t * E;
      const int64_t row = rowid[t];
      for (int e = lane; e < E; e += 32) {
        const double ze = zr[e];
        int r = 0;
        for (int q = 0; q < E; ++q) r += key_gt(zr[q], q, ze, e) ? 1 : 0;
        rk[t * E + e] = r;
        if (a.logits64) a.logits64[row * E + e] = ze;
        if (a.logits32) a.logits32[row * E + e] = static_cast<float>(ze);
      }
      __syncwarp();
      if (lane == 0) {
        const int* rr = rk + t * E;
        if (a.ids && a.m_sel > 0) {
          int cnt = 0;
          for (int e = 0; e < E && cnt < a.m_sel; ++e)
            if (rr[e] < a.m_sel) a.ids[row * a.m_sel + cnt++] = e;
        }
        if (a.truth) {
          int any0 = 0;
          int inside[MOEP_MAX_BOUNDS] = {0, 0, 0, 0};
          for (int j = 0; j < a.k; ++j) {
            const int tt = a.truth[row * a.k + j];
            const int r = rr[tt];
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
    }
    __syncthreads();
  }
  if (a.partials) {
    int* out = a.partials + static_cast<int64_t>(blockIdx.x) * n_counters;
    for (int t = tid; t < n_counters; t += NT) {
      int v;
      if (t < 2) v = scal[t];
      else if (t < 2 + a.n_m) v = scal[2 + (t - 2)];
      else if (t < 2 + 2 * a.n_m) v = scal[2 + MOEP_MAX_BOUNDS + (t - 2 - a.n_m)];
      else v = hist[t - 2 - 2 * a.n_m];
      out[t] = v;
    }
  }
}

template <int XT, int WT, int TB>
size_t smem_bytes(int d, int E) {
  using XS = double;  // staged once per group; avoids per-use conversions
  const int dpad = (d + IV - 1) / IV * IV;
  return sizeof(double) * (TB * HP + TB * E) + sizeof(XS) * static_cast<size_t>(dpad) * TB +
         sizeof(int) * (TB * E + 2 * E);
}

template <int XT, int WT, int TB>
int launch(const moep_fp64_args* a, cudaStream_t st, int ncnt) {
  using XS = double;
  const size_t smem = smem_bytes<XT, WT, TB>(a->d, a->n_experts);
  auto kern = fp64_kernel<XT, WT, TB, XS>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
    return MOEP_ELAUNCH;
  kern<<<moep_num_sms(), NT, smem, st>>>(*a, ncnt);  // partial rows are sized by the SM count
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

template <int XT, int WT>
int launch_tb(const moep_fp64_args* a, cudaStream_t st, int ncnt) {
  constexpr size_t kMax = 220 * 1024;
  if (smem_bytes<XT, WT, 8>(a->d, a->n_experts) <= kMax) return launch<XT, WT, 8>(a, st, ncnt);
  if (smem_bytes<XT, WT, 4>(a->d, a->n_experts) <= kMax) return launch<XT, WT, 4>(a, st, ncnt);
  if (smem_bytes<XT, WT, 2>(a->d, a->n_experts) <= kMax) return launch<XT, WT, 2>(a, st, ncnt);
  if (smem_bytes<XT, WT, 1>(a->d, a->n_experts) <= kMax) return launch<XT, WT, 1>(a, st, ncnt);
  return MOEP_EUNSUPPORTED;
}

}  // namespace k2
}  // namespace moep

extern "C" int moep_predict_fp64(const moep_fp64_args* a, void* stream) {
  using namespace moep::k2;
  if (!a || a->n_tokens <= 0 || a->d <= 0 || a->hidden <= 0 || a->n_experts <= 0) return MOEP_ESHAPE;
  if (a->arch != 1 && a->arch != 2) return MOEP_EARG;
  if (!a->w2t) return MOEP_EARG;
  if (a->rows && !a->row_count) return MOEP_EARG;
  if (a->truth && (a->k < 1 || a->k > 16 || a->n_m < 0 || a->n_m > MOEP_MAX_BOUNDS)) return MOEP_EARG;
  if (a->m_sel < 0 || a->m_sel > a->n_experts) return MOEP_EARG;
  if ((reinterpret_cast<uintptr_t>(a->w1) & 15) != 0) return MOEP_EALIGN;
  const int ncnt = a->truth ? moep_n_counters(a->n_m, a->n_experts) : 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool xb = a->x_dtype == MOEP_BF16, wb = a->w_dtype == MOEP_BF16;
  if ((a->x_dtype != MOEP_BF16 && a->x_dtype != MOEP_F64) || (a->w_dtype != MOEP_BF16 && a->w_dtype != MOEP_F64))
    return MOEP_EARG;
  if (xb && wb) return launch_tb<MOEP_BF16, MOEP_BF16>(a, st, ncnt);
  if (xb) return launch_tb<MOEP_BF16, MOEP_F64>(a, st, ncnt);
  if (wb) return launch_tb<MOEP_F64, MOEP_BF16>(a, st, ncnt);
  return launch_tb<MOEP_F64, MOEP_F64>(a, st, ncnt);
}
