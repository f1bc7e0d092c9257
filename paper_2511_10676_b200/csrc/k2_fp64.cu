// k2_fp64.cu — K2: float64 predictor on CUDA cores.
//
// Recomputes z = W2 . act(W1 . x + b1) + b2 in fp64 for the tokens K1 could not
// decide exactly (near-tie margin), or for every token when the inputs are not
// bf16-representable. Mirrors the reference's float64 arithmetic per token:
// _forward_internal eval branch (predictor.py:193-240), the branch-stable
// sigmoid (:39-45), GELU-tanh (:57-61) and BN eval (:221-224, :234). Selection
// and evaluation use exact rank counts (core.py:27-54, metrics.py:159-180).
// One CTA (256 threads) per token; warps own hidden units / experts.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "common.cuh"

namespace moep {
namespace k2 {

constexpr int NT = 256;

template <int WT>
__device__ __forceinline__ double ldw(const void* p, int64_t i) {
  if (WT == MOEP_BF16)
    return static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]));
  return reinterpret_cast<const double*>(p)[i];
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

__device__ __forceinline__ double warp_sum64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int XT, int WT>
__global__ void __launch_bounds__(NT) fp64_kernel(moep_fp64_args a, int n_counters) {
  extern __shared__ double sm[];
  const int d = a.d, H = a.hidden, E = a.n_experts;
  double* xs = sm;             // [d]
  double* hs = xs + d;         // [H]
  double* zs = hs + H;         // [E]
  int* rk = reinterpret_cast<int*>(zs + E);  // [E] ranks
  int* hist = rk + E;                        // [2E] hits, truth
  __shared__ int scal[2 + 2 * MOEP_MAX_BOUNDS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = NT / 32;
  for (int i = threadIdx.x; i < 2 * E; i += NT) hist[i] = 0;
  if (threadIdx.x < 2 + 2 * MOEP_MAX_BOUNDS) scal[threadIdx.x] = 0;
  const int64_t nrows = a.rows ? static_cast<int64_t>(*a.row_count) : a.n_tokens;
  __syncthreads();
  for (int64_t it = blockIdx.x; it < nrows; it += gridDim.x) {
    const int64_t row = a.rows ? a.rows[it] : it;
    for (int i = threadIdx.x; i < d; i += NT) xs[i] = ldw<XT>(a.x, row * d + i);
    __syncthreads();
    // hidden: a_j = x . w1_j + b1_j, then activation in fp64
    for (int j = warp; j < H; j += nw) {
      double s = 0.0;
      for (int i = lane; i < d; i += 32) s += xs[i] * ldw<WT>(a.w1, static_cast<int64_t>(j) * d + i);
      s = warp_sum64(s);
      if (lane == 0) {
        const double av = s + a.b1[j];
        double hv;
        if (a.arch == 2) {
          hv = av * sigmoid64(av);
        } else {
          const double inv_std = 1.0 / sqrt(a.bn_var[j] + a.bn_eps);
          const double a_hat = (av - a.bn_mean[j]) * inv_std;
          hv = gelu64(a.bn_scale[j] * a_hat + a.bn_shift[j]);
        }
        hs[j] = hv;
      }
    }
    __syncthreads();
    for (int e = warp; e < E; e += nw) {
      double s = 0.0;
      for (int j = lane; j < H; j += 32) s += hs[j] * ldw<WT>(a.w2, static_cast<int64_t>(e) * H + j);
      s = warp_sum64(s);
      if (lane == 0) zs[e] = s + a.b2[e];
    }
    __syncthreads();
    // exact stable ranks
    for (int e = threadIdx.x; e < E; e += NT) {
      const double ze = zs[e];
      int r = 0;
      for (int j = 0; j < E; ++j) r += key_gt(zs[j], j, ze, e) ? 1 : 0;
      rk[e] = r;
      if (a.logits64) a.logits64[row * E + e] = ze;
      if (a.logits32) a.logits32[row * E + e] = static_cast<float>(ze);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (a.ids && a.m_sel > 0) {
        int cnt = 0;
        for (int e = 0; e < E && cnt < a.m_sel; ++e)
          if (rk[e] < a.m_sel) a.ids[row * a.m_sel + cnt++] = e;
      }
      if (a.truth) {
        int any0 = 0;
        int tr[16];
        for (int j = 0; j < a.k; ++j) {
          const int t = a.truth[row * a.k + j];
          tr[j] = rk[t];
          any0 |= tr[j] == 0;
          hist[E + t] += 1;
          if (tr[j] < a.k) hist[t] += 1;
        }
        scal[0] += 1;
        scal[1] += any0;
        for (int mi = 0; mi < a.n_m; ++mi) {
          int inside = 0;
          for (int j = 0; j < a.k; ++j) inside += tr[j] < a.m_list[mi];
          scal[2 + mi] += inside == a.k;
          scal[2 + MOEP_MAX_BOUNDS + mi] += inside;
        }
      }
    }
    __syncthreads();
  }
  if (a.partials) {
    int* out = a.partials + static_cast<int64_t>(blockIdx.x) * n_counters;
    for (int t = threadIdx.x; t < n_counters; t += NT) {
      int v;
      if (t < 2) v = scal[t];
      else if (t < 2 + a.n_m) v = scal[2 + (t - 2)];
      else if (t < 2 + 2 * a.n_m) v = scal[2 + MOEP_MAX_BOUNDS + (t - 2 - a.n_m)];
      else v = hist[t - 2 - 2 * a.n_m];
      out[t] = v;
    }
  }
}

}  // namespace k2
}  // namespace moep

extern "C" int moep_predict_fp64(const moep_fp64_args* a, void* stream) {
  using namespace moep::k2;
  if (!a || a->n_tokens <= 0 || a->d <= 0 || a->hidden <= 0 || a->n_experts <= 0) return MOEP_ESHAPE;
  if (a->arch != 1 && a->arch != 2) return MOEP_EARG;
  if (a->rows && !a->row_count) return MOEP_EARG;
  if (a->truth && (a->k < 1 || a->k > 16 || a->n_m < 0 || a->n_m > MOEP_MAX_BOUNDS)) return MOEP_EARG;
  if (a->m_sel < 0 || a->m_sel > a->n_experts) return MOEP_EARG;
  const size_t smem = sizeof(double) * (a->d + a->hidden + a->n_experts) + sizeof(int) * 3 * a->n_experts;
  if (smem > 227 * 1024) return MOEP_EUNSUPPORTED;
  const int ncnt = a->truth ? moep_n_counters(a->n_m, a->n_experts) : 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = moep_num_sms();  // partial rows are sized by the SM count
  auto pick = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, NT, smem, st>>>(*a, ncnt);
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  };
  const bool xb = a->x_dtype == MOEP_BF16, wb = a->w_dtype == MOEP_BF16;
  if ((a->x_dtype != MOEP_BF16 && a->x_dtype != MOEP_F64) || (a->w_dtype != MOEP_BF16 && a->w_dtype != MOEP_F64))
    return MOEP_EARG;
  if (xb && wb) return pick(fp64_kernel<MOEP_BF16, MOEP_BF16>);
  if (xb) return pick(fp64_kernel<MOEP_BF16, MOEP_F64>);
  if (wb) return pick(fp64_kernel<MOEP_F64, MOEP_BF16>);
  return pick(fp64_kernel<MOEP_F64, MOEP_F64>);
}
