// train.cu — training kernels for the expert predictor.
//
//   K3 moep_labels          BatchLabels.from_scores (losses.py:64-74): stable
//                           1-based ranks, top-k mask, strict-pair counts.
//   K4 moep_loss            loss_and_grad (losses.py:243-273) for mse / wbce /
//                           focal / ranking (three-tier WBCE + pairwise hinge),
//                           one warp per token, per-CTA partial sums.
//      moep_loss_finalize   global normalisers (N*E, batch n_pairs) -> dZ, loss.
//   K5 moep_act_backward    dA = (dZ . W2) * act'(a), dW2 = dZ^T . act(a),
//                           db1, db2 (predictor.py:261-297, arch2 branch);
//                           column-parallel with deterministic split-N partials.
//   K6 moep_optim_step      Adam / SGD / momentum with bias correction
//                           (trainer.py:103-122) on a flat fp32 master buffer,
//                           writing the bf16 shadow the forward GEMMs read and
//                           a non-finite flag (trainer.py:125-128).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "common.cuh"

namespace moep {
namespace tr {

constexpr int NT = 256;

template <typename T>
__device__ __forceinline__ double ldd(const T* p, int64_t i) { return static_cast<double>(p[i]); }

// ------------------------------------------------------------------ K3
template <typename T>
__global__ void __launch_bounds__(NT)
labels_kernel(const T* __restrict__ s, int64_t n, int E, int k, int top_cut, int* __restrict__ rank_of,
              uint8_t* __restrict__ mask, int* __restrict__ pairs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NT / 32);
  for (int64_t row = gw; row < n; row += nw) {
    const T* sr = s + row * E;
    int np = 0;
    for (int e = lane; e < E; e += 32) {
      const double se = ldd(sr, e);
      int r = 0;
      for (int j = 0; j < E; ++j) r += key_gt(ldd(sr, j), j, se, e) ? 1 : 0;
      rank_of[row * E + e] = r + 1;
      mask[row * E + e] = r < k ? 1 : 0;
    }
    __syncwarp();
    // strict pairs among the true top-T (losses.py:202-207)
    for (int e = lane; e < E; e += 32) {
      if (rank_of[row * E + e] <= top_cut) {
        const double se = ldd(sr, e);
        for (int j = 0; j < E; ++j)
          if (rank_of[row * E + j] <= top_cut && se > ldd(sr, j)) ++np;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
    if (lane == 0 && pairs) pairs[row] = np;
  }
}

// Register-resident K3 (E <= 32 * EPL): LPR lanes per token, the row's scores
// in registers, every comparison against the other experts by width-LPR
// shuffles (no re-reads); same outputs as labels_kernel.
template <typename T, int LPR, int EPL>
__global__ void __launch_bounds__(NT)
labels_reg_kernel(const T* __restrict__ s, int64_t n, int E, int k, int top_cut, int* __restrict__ rank_of,
                  uint8_t* __restrict__ mask, int* __restrict__ pairs) {
  constexpr int RPW = 32 / LPR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NT / 32);
  for (int64_t base = gw * RPW; base < n; base += nw * RPW) {  // warp-uniform
    const int64_t row = base + sub;
    T sv[EPL];
    int rk[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = li + i * LPR;
      sv[i] = (row < n && e < E) ? s[row * E + e] : T(0);
      rk[i] = 0;
    }
#pragma unroll
    for (int jb = 0; jb < EPL; ++jb) {
      for (int jl = 0; jl < LPR; ++jl) {
        const int j = jb * LPR + jl;
        if (j >= E) break;  // uniform
        const T sj = __shfl_sync(0xffffffffu, sv[jb], jl, LPR);
#pragma unroll
        for (int i = 0; i < EPL; ++i) rk[i] += key_gt(sj, j, sv[i], li + i * LPR) ? 1 : 0;
      }
    }
    // strict pairs among the true top-T (losses.py:202-207)
    int np = 0;
#pragma unroll
    for (int jb = 0; jb < EPL; ++jb) {
      for (int jl = 0; jl < LPR; ++jl) {
        const int j = jb * LPR + jl;
        if (j >= E) break;
        const T sj = __shfl_sync(0xffffffffu, sv[jb], jl, LPR);
        const int rj = __shfl_sync(0xffffffffu, rk[jb], jl, LPR);
#pragma unroll
        for (int i = 0; i < EPL; ++i)
          np += (li + i * LPR < E && rk[i] < top_cut && rj < top_cut && sv[i] > sj) ? 1 : 0;
      }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
    if (row < n) {
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = li + i * LPR;
        if (e < E) {
          rank_of[row * E + e] = rk[i] + 1;
          mask[row * E + e] = rk[i] < k ? 1 : 0;
        }
      }
      if (li == 0 && pairs) pairs[row] = np;
    }
  }
}

// ------------------------------------------------------------------ K4
struct LossParams {
  int family;  // 0 mse, 1 wbce, 2 focal, 3 ranking
  double top_w, mid_w, rest_w, lam, margin, gamma, alpha;
  int top_cut, mid_cut;
  double inv_ne;  // 1 / (N_global * E)
  double inv_n;   // 1 / N_global
};

__device__ __forceinline__ double softplus(double v) {  // log(1 + e^v), stable (np.logaddexp(0, v))
  return v > 0 ? v + log1p(exp(-v)) : log1p(exp(v));
}
__device__ __forceinline__ double sigm(double u) {
  if (u >= 0.0) return 1.0 / (1.0 + exp(-u));
  const double eu = exp(u);
  return eu / (1.0 + eu);
}
// fp32 forms for fp32 logits (the tensor-core training modes; their loss is
// checked to rel 1e-3 against the fp64 oracle step): full-precision expf /
// log1pf, ~10x cheaper than the fp64 library calls
__device__ __forceinline__ float softplus(float v) { return v > 0.f ? v + log1pf(expf(-v)) : log1pf(expf(v)); }
__device__ __forceinline__ float sigm(float u) {
  if (u >= 0.f) return 1.f / (1.f + expf(-u));
  const float eu = expf(u);
  return eu / (1.f + eu);
}

// Generic fallback (E > 512): one warp per token.
// partials per CTA: [0] loss (bce/mse/focal part), [1] hinge total (unnormalised), [2] n_pairs
template <typename T>
__global__ void __launch_bounds__(NT)
loss_rowwarp_kernel(const T* __restrict__ z, const T* __restrict__ s, const int* __restrict__ rank_of,
            const uint8_t* __restrict__ mask, int64_t n, int E, LossParams p, T* __restrict__ dz,
            T* __restrict__ dz_hinge, double* __restrict__ partials) {
  __shared__ double red[NT / 32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NT / 32);
  double l_main = 0.0, l_hinge = 0.0, n_pairs = 0.0;
  for (int64_t row = gw; row < n; row += nw) {
    const T* zr = z + row * E;
    const T* sr = s + row * E;
    const int* rr = rank_of + row * E;
    const uint8_t* mr = mask + row * E;
    if (p.family == 0) {
      // MSE on softmax probabilities (losses.py:99-110, chain rule :250-255)
      double mx = -INFINITY;
      for (int e = lane; e < E; e += 32) mx = fmax(mx, (double)zr[e]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      double se = 0.0;
      for (int e = lane; e < E; e += 32) se += exp((double)zr[e] - mx);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      double inner = 0.0;
      for (int e = lane; e < E; e += 32) {
        const double pr = exp((double)zr[e] - mx) / se;
        const double diff = (double)sr[e] - pr;
        l_main += diff * diff * p.inv_n;
        inner += (-2.0 * diff * p.inv_n) * pr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) inner += __shfl_xor_sync(0xffffffffu, inner, o);
      for (int e = lane; e < E; e += 32) {
        const double pr = exp((double)zr[e] - mx) / se;
        const double dp = -2.0 * ((double)sr[e] - pr) * p.inv_n;
        dz[row * E + e] = static_cast<T>(pr * (dp - inner));
      }
      continue;
    }
    for (int e = lane; e < E; e += 32) {
      const double zv = zr[e];
      const bool pos = mr[e] != 0;
      if (p.family == 4) { dz[row * E + e] = T(0); continue; }  // hinge only
      double g;
      if (p.family == 2) {
        // focal (losses.py:156-179)
        const double log_pt = pos ? -softplus(-zv) : -softplus(zv);
        const double pt = exp(log_pt);
        const double at = pos ? p.alpha : 1.0 - p.alpha;
        const double om = 1.0 - pt;
        const double focus = pow(om, p.gamma);
        l_main += -at * focus * log_pt * p.inv_ne;
        const double sgn = pos ? 1.0 : -1.0;
        g = at * sgn * (p.gamma * pt * focus * log_pt - pow(om, p.gamma + 1.0)) * p.inv_ne;
      } else {
        // tier weights (losses.py:113-121); three tiers only for the ranking family
        const int r = rr[e];
        double w = p.rest_w;
        if (p.family == 3 && r > p.top_cut && r <= p.mid_cut) w = p.mid_w;
        if (r <= p.top_cut) w = p.top_w;
        const double lt = pos ? -softplus(-zv) : -softplus(zv);
        l_main += -w * lt * p.inv_ne;
        g = w * (sigm(zv) - (pos ? 1.0 : 0.0)) * p.inv_ne;
      }
      dz[row * E + e] = static_cast<T>(g);
    }
    if (p.family >= 3) {
      // pairwise hinge over the true top-T (losses.py:182-217), unnormalised here
      for (int e = lane; e < E; e += 32) {
        double gh = 0.0;
        if (rr[e] <= p.top_cut) {
          const double se = sr[e], ze = zr[e];
          for (int j = 0; j < E; ++j) {
            if (j == e || rr[j] > p.top_cut) continue;
            const double sj = sr[j], zj = zr[j];
            if (se > sj) {  // e outranks j in truth: pair (e, j)
              n_pairs += 1.0;
              const double gap = p.margin - (ze - zj);
              if (gap > 0) { l_hinge += gap; gh -= 1.0; }
            } else if (sj > se) {  // pair (j, e)
              const double gap = p.margin - (zj - ze);
              if (gap > 0) gh += 1.0;
            }
          }
        }
        dz_hinge[row * E + e] = static_cast<T>(gh);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l_main += __shfl_xor_sync(0xffffffffu, l_main, o);
    l_hinge += __shfl_xor_sync(0xffffffffu, l_hinge, o);
    n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
  }
  if (lane == 0) { red[warp][0] = l_main; red[warp][1] = l_hinge; red[warp][2] = n_pairs; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v += red[w][threadIdx.x];
    partials[blockIdx.x * 3 + threadIdx.x] = v;
  }
}

// partials per CTA: [0] loss (bce/mse/focal part), [1] hinge total (unnormalised), [2] n_pairs.
// LPR lanes per token (a power of two <= 32, so a warp holds 32/LPR tokens),
// EPL experts per lane (expert e = lane_in_row + i*LPR). The token's logits,
// scores and ranks stay in registers; the pairwise hinge walks the row by
// width-LPR shuffles instead of re-reading global memory.
template <typename T, int LPR, int EPL>
__global__ void __launch_bounds__(NT)
loss_kernel(const T* __restrict__ z, const T* __restrict__ s, const int* __restrict__ rank_of,
            const uint8_t* __restrict__ mask, int64_t n, int E, LossParams p, T* __restrict__ dz,
            T* __restrict__ dz_hinge, double* __restrict__ partials) {
  constexpr int RPW = 32 / LPR;
  __shared__ double red[NT / 32][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (NT / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (NT / 32);
  using M = T;  // per-element math in the logits' precision; sums in fp64
  double l_main = 0.0, l_hinge = 0.0, n_pairs = 0.0;
  for (int64_t base = gw * RPW; base < n; base += nw * RPW) {  // warp-uniform
    const int64_t row = base + sub;
    M zv[EPL], sv[EPL];
    int rk[EPL];
    bool pos[EPL], ev[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = li + i * LPR;
      ev[i] = row < n && e < E;
      const int64_t o = row * E + e;
      zv[i] = ev[i] ? z[o] : M(0);
      sv[i] = ev[i] ? s[o] : M(0);
      rk[i] = ev[i] ? rank_of[o] : 0x7fffffff;
      pos[i] = ev[i] && mask[o] != 0;
    }
    if (p.family == 0) {
      // MSE on softmax probabilities (losses.py:99-110, chain rule :250-255)
      M mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < EPL; ++i)
        if (ev[i]) mx = mx > zv[i] ? mx : zv[i];
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) {
        const M om = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = mx > om ? mx : om;
      }
      M ex[EPL], se = M(0);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        ex[i] = ev[i] ? exp(zv[i] - mx) : M(0);
        se += ex[i];
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      M inner = M(0);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (!ev[i]) continue;
        ex[i] /= se;  // probability
        const M diff = sv[i] - ex[i];
        l_main += static_cast<double>(diff) * diff * p.inv_n;
        inner += (M(-2) * diff * M(p.inv_n)) * ex[i];
      }
#pragma unroll
      for (int o = LPR / 2; o > 0; o >>= 1) inner += __shfl_xor_sync(0xffffffffu, inner, o);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (!ev[i]) continue;
        const M dp = M(-2) * (sv[i] - ex[i]) * M(p.inv_n);
        dz[row * E + li + i * LPR] = static_cast<T>(ex[i] * (dp - inner));
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      if (!ev[i]) continue;
      const M zi = zv[i];
      M g = M(0);
      if (p.family == 2) {
        // focal (losses.py:156-179)
        const M log_pt = pos[i] ? -softplus(-zi) : -softplus(zi);
        const M pt = exp(log_pt);
        const M at = M(pos[i] ? p.alpha : 1.0 - p.alpha);
        const M om = M(1) - pt;
        const M focus = pow(om, M(p.gamma));
        l_main += -static_cast<double>(at) * focus * log_pt * p.inv_ne;
        const M sgn = pos[i] ? M(1) : M(-1);
        g = at * sgn * (M(p.gamma) * pt * focus * log_pt - pow(om, M(p.gamma + 1.0))) * M(p.inv_ne);
      } else if (p.family != 4) {
        // tier weights (losses.py:113-121); three tiers only for the ranking family
        const int r = rk[i];
        double w = p.rest_w;
        if (p.family == 3 && r > p.top_cut && r <= p.mid_cut) w = p.mid_w;
        if (r <= p.top_cut) w = p.top_w;
        const M lt = pos[i] ? -softplus(-zi) : -softplus(zi);
        l_main += -w * static_cast<double>(lt) * p.inv_ne;
        g = M(w) * (sigm(zi) - (pos[i] ? M(1) : M(0))) * M(p.inv_ne);
      }
      dz[row * E + li + i * LPR] = static_cast<T>(g);  // family 4 (hinge only): 0
    }
    if (p.family >= 3) {
      // pairwise hinge over the true top-T (losses.py:182-217), unnormalised here;
      // each strict pair is counted by its higher-scored member
      double gh[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) gh[i] = 0.0;
#pragma unroll
      for (int jb = 0; jb < EPL; ++jb) {
        for (int jl = 0; jl < LPR; ++jl) {
          const int j = jb * LPR + jl;
          if (j >= E) break;
          const M sj = __shfl_sync(0xffffffffu, sv[jb], jl, LPR);
          const M zj = __shfl_sync(0xffffffffu, zv[jb], jl, LPR);
          const int rj = __shfl_sync(0xffffffffu, rk[jb], jl, LPR);
          const bool jtop = rj <= p.top_cut;  // (no divergent exit before the next shuffles)
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            if (!jtop || !ev[i] || rk[i] > p.top_cut || li + i * LPR == j) continue;
            if (sv[i] > sj) {  // e outranks j in truth: pair (e, j)
              n_pairs += 1.0;
              const M gap = M(p.margin) - (zv[i] - zj);
              if (gap > 0) { l_hinge += gap; gh[i] -= 1.0; }
            } else if (sj > sv[i]) {  // pair (j, e)
              const M gap = M(p.margin) - (zj - zv[i]);
              if (gap > 0) gh[i] += 1.0;
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i)
        if (ev[i]) dz_hinge[row * E + li + i * LPR] = static_cast<T>(gh[i]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l_main += __shfl_xor_sync(0xffffffffu, l_main, o);
    l_hinge += __shfl_xor_sync(0xffffffffu, l_hinge, o);
    n_pairs += __shfl_xor_sync(0xffffffffu, n_pairs, o);
  }
  if (lane == 0) { red[warp][0] = l_main; red[warp][1] = l_hinge; red[warp][2] = n_pairs; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v += red[w][threadIdx.x];
    partials[blockIdx.x * 3 + threadIdx.x] = v;
  }
}

// sums partials in a fixed order; ranking: dz += lam/n_pairs * dz_hinge
template <typename T>
__global__ void finalize_kernel(const double* __restrict__ partials, int nblk, int64_t n, int E, int family,
                                double lam, int normalize, T* __restrict__ dz,
                                const T* __restrict__ dz_hinge, double* __restrict__ out_loss) {
  // fixed-order tree over the partial rows (the same order in every block, so
  // the total is deterministic): thread t sums rows t, t+256, ..., then a
  // shared-memory halving tree (blockDim.x == 256)
  __shared__ double tot[3];
  __shared__ double acc[3][256];
  {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 256) {
      v0 += partials[b * 3 + 0];
      v1 += partials[b * 3 + 1];
      v2 += partials[b * 3 + 2];
    }
    acc[0][threadIdx.x] = v0; acc[1][threadIdx.x] = v1; acc[2][threadIdx.x] = v2;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (threadIdx.x < h)
        for (int c = 0; c < 3; ++c) acc[c][threadIdx.x] += acc[c][threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x < 3) tot[threadIdx.x] = acc[threadIdx.x][0];
  }
  __syncthreads();
  double scale = 0.0;
  if (family >= 3) {
    double hinge = tot[1];
    scale = lam;
    if (normalize && tot[2] > 0) { hinge /= tot[2]; scale = lam / tot[2]; }
    if (blockIdx.x == 0 && threadIdx.x == 0) { out_loss[0] = tot[0] + lam * hinge; out_loss[1] = tot[2]; }
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n * E;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      dz[i] = static_cast<T>(static_cast<double>(dz[i]) + scale * static_cast<double>(dz_hinge[i]));
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {
    out_loss[0] = tot[0];
    out_loss[1] = 0.0;
  }
}

// ------------------------------------------------------------------ K5
// One thread per hidden column j, a CTA covers 128 columns x a slice of rows.
// Writes dA and per-slice partials of dW2 [E, h], db1 [h], db2 [E]. Rows go
// in groups of RU with the group's `a` loads issued together (memory-level
// parallelism: the kernel streams a and dA at HBM rate). SPLIT: dA is written
// as bf16 hi (rows 0..n-1) and lo = bf16(dA - hi) (rows n..2n-1) of a [2n, h]
// buffer row-wise: row n = [hi(dA[n, :]) | lo(dA[n, :])] of a [n, 2h] bf16
// buffer, the operand of the bf16 dW1 GEMM (fp32 mode).
template <int EMAX, typename T, bool SPLIT>
__global__ void __launch_bounds__(128)
act_backward_kernel(const T* __restrict__ a, const T* __restrict__ dz, const T* __restrict__ w2,
                    int64_t n, int H, int E, int rows_per_slice, T* __restrict__ da,
                    __nv_bfloat16* __restrict__ da_hilo, T* __restrict__ dw2_part, T* __restrict__ db1_part,
                    T* __restrict__ db2_part) {
  constexpr int RU = 8;
  __shared__ T sdz[32][EMAX];
  const int j = blockIdx.x * 128 + threadIdx.x;
  const int slice = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(slice) * rows_per_slice;
  const int64_t r1 = (r0 + rows_per_slice < n) ? r0 + rows_per_slice : n;
  T w2c[EMAX], acc[EMAX];
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    w2c[e] = (j < H && e < E) ? w2[static_cast<int64_t>(e) * H + j] : T(0);
    acc[e] = T(0);
  }
  T db1 = T(0);
  for (int64_t rb = r0; rb < r1; rb += 32) {
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * EMAX; i += 128) {
      const int rr = i / EMAX, e = i % EMAX;
      sdz[rr][e] = (rb + rr < r1 && e < E) ? dz[(rb + rr) * E + e] : T(0);
    }
    __syncthreads();
    if (j < H) {
      const int lim = (r1 - rb < 32) ? static_cast<int>(r1 - rb) : 32;
      for (int rg = 0; rg < lim; rg += RU) {
        T av[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) av[u] = (rg + u < lim) ? a[(rb + rg + u) * H + j] : T(0);
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          if (rg + u < lim) {
            const int rr = rg + u;
            const int64_t row = rb + rr;
            const T x = av[u];
            // branch-stable sigmoid (predictor.py:39-45), silu / silu' (:48-54)
            T sg;
            if (x >= T(0)) sg = T(1) / (T(1) + exp(-x));
            else { const T ea = exp(x); sg = ea / (T(1) + ea); }
            const T hv = x * sg;
            const T dsilu = sg * (T(1) + x * (T(1) - sg));
            T dh = T(0);
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
              dh = fma(sdz[rr][e], w2c[e], dh);
              acc[e] = fma(sdz[rr][e], hv, acc[e]);
            }
            const T dav = dh * dsilu;
            if constexpr (SPLIT) {
              const __nv_bfloat16 hi = __float2bfloat16_rn(static_cast<float>(dav));
              da_hilo[row * 2 * H + j] = hi;
              da_hilo[row * 2 * H + H + j] = __float2bfloat16_rn(static_cast<float>(dav) - __bfloat162float(hi));
            } else {
              da[row * H + j] = dav;
            }
            db1 += dav;
          }
        }
      }
    }
  }
  if (j < H) {
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
      if (e < E) dw2_part[(static_cast<int64_t>(slice) * E + e) * H + j] = acc[e];
    db1_part[static_cast<int64_t>(slice) * H + j] = db1;
  }
  if (blockIdx.x == 0 && threadIdx.x < E) {
    T s = T(0);
    for (int64_t row = r0; row < r1; ++row) s += dz[row * E + threadIdx.x];
    db2_part[static_cast<int64_t>(slice) * E + threadIdx.x] = s;
  }
}

// packed fp32x2 FMA (sm_100 FFMA2): two lanes of work per instruction
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// fp32 / bf16-split variant: two adjacent hidden columns per thread (float2
// loads of a, each dz value from smem feeds both columns) and a branch-free
// stable sigmoid (e = exp(-|x|); sigmoid = x >= 0 ? 1/(1+e) : e/(1+e)) with
// the fast exp / reciprocal -- the fp32 mode's tolerance, not the fp64 path.
constexpr int BR = 16;  // rows per staged block

template <int EMAX, bool LO>
__global__ void __launch_bounds__(128)
act_backward_f32x2_kernel(const float* __restrict__ a, const float* __restrict__ dz, const float* __restrict__ w2,
                          int64_t n, int H, int E, int rows_per_slice, __nv_bfloat16* __restrict__ da_hilo,
                          float* __restrict__ dw2_part, float* __restrict__ db1_part, float* __restrict__ db2_part) {
  __shared__ __align__(16) float2 sdz2[2][BR][EMAX];    // dz values duplicated {g, g}: FFMA2 operands
  extern __shared__ __align__(16) float abuf_raw[];
  auto abuf = reinterpret_cast<float(*)[BR][256]>(abuf_raw);  // [2][BR][256] staged rows of a
  const int j = (blockIdx.x * 128 + threadIdx.x) * 2;   // columns j, j+1 (H even)
  const int slice = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(slice) * rows_per_slice;
  const int64_t r1 = (r0 + rows_per_slice < n) ? r0 + rows_per_slice : n;
  const bool ok = j < H;
  float2 w01[EMAX], acc[EMAX];  // (column j, column j+1) pairs
#pragma unroll
  for (int e = 0; e < EMAX; ++e) {
    w01[e] = (ok && e < E) ? *reinterpret_cast<const float2*>(w2 + static_cast<int64_t>(e) * H + j)
                           : make_float2(0.f, 0.f);
    acc[e] = make_float2(0.f, 0.f);
  }
  float2 db1 = make_float2(0.f, 0.f);
  // one row: sigmoid / silu / silu' (branch-free stable form), dH = dz . W2 in 4
  // independent FFMA2 chains (fixed order), dW2 += dz (x) h, hi/lo bf16 stores
  auto row_step = [&](float2 x2, int sb, int rr, __nv_bfloat16* hp, __nv_bfloat16* lp) {
    const float xs[2] = {x2.x, x2.y};
    float hv[2], ds[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float x = xs[c];
      // e = 2^(-|x| log2 e), r = 1 / (1 + e): one MUFU op each, no slow paths
      float ex, r;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"(-fabsf(x) * 1.4426950408889634f));
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + ex));
      const float sg = x >= 0.f ? r : ex * r;
      hv[c] = x * sg;
      ds[c] = sg * (1.f + x * (1.f - sg));
    }
    const float2 h2 = make_float2(hv[0], hv[1]);
    float2 dhp[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int e2 = 0; e2 < EMAX; e2 += 2) {
      const float4 gg = *reinterpret_cast<const float4*>(&sdz2[sb][rr][e2]);
      const float2 g0 = make_float2(gg.x, gg.y), g1 = make_float2(gg.z, gg.w);
      dhp[e2 & 3] = ffma2(g0, w01[e2], dhp[e2 & 3]);
      dhp[(e2 + 1) & 3] = ffma2(g1, w01[e2 + 1], dhp[(e2 + 1) & 3]);
      acc[e2] = ffma2(g0, h2, acc[e2]);
      acc[e2 + 1] = ffma2(g1, h2, acc[e2 + 1]);
    }
    const float d0 = ((dhp[0].x + dhp[1].x) + (dhp[2].x + dhp[3].x)) * ds[0];
    const float d1 = ((dhp[0].y + dhp[1].y) + (dhp[2].y + dhp[3].y)) * ds[1];
    const __nv_bfloat162 hi = __floats2bfloat162_rn(d0, d1);
    const float2 hf = __bfloat1622float2(hi);
    *reinterpret_cast<__nv_bfloat162*>(hp) = hi;
    if constexpr (LO) *reinterpret_cast<__nv_bfloat162*>(lp) = __floats2bfloat162_rn(d0 - hf.x, d1 - hf.y);
    db1.x += d0;
    db1.y += d1;
  };
  // BR-row blocks of this CTA's 256 columns of `a` stream through a double
  // buffer with cp.async (16-byte chunks, whole block in flight), the next
  // block's dz rows ride in registers; HBM latency overlaps the compute.
  const int cb = blockIdx.x * 256;
  const int ncols = (H - cb) < 256 ? (H - cb) : 256;   // even
  const int nchunk = ncols / 4;                         // 16-byte chunks per row (H % 4 == 0)
  auto issue = [&](int buf, int64_t rb) {
    const int lim = (r1 - rb < BR) ? static_cast<int>(r1 - rb) : BR;
    for (int c = threadIdx.x; c < BR * 64; c += 128) {
      const int row = c >> 6, ch = c & 63;
      if (row < lim && ch < nchunk) {
        const float* src = a + (rb + row) * H + cb + ch * 4;
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&abuf[buf][row][ch * 4]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  constexpr int DZPT = BR * EMAX / 128;                 // dz values per thread per block
  float dzr[DZPT];
  auto load_dz = [&](int64_t rb) {
#pragma unroll
    for (int q = 0; q < DZPT; ++q) {
      const int i = threadIdx.x + 128 * q, rr = i / EMAX, e = i % EMAX;
      dzr[q] = (rb + rr < r1 && e < E) ? dz[(rb + rr) * E + e] : 0.f;
    }
  };
  auto store_dz = [&](int buf) {
#pragma unroll
    for (int q = 0; q < DZPT; ++q) {
      const int i = threadIdx.x + 128 * q, rr = i / EMAX, e = i % EMAX;
      sdz2[buf][rr][e] = make_float2(dzr[q], dzr[q]);
    }
  };
  if (r0 < r1) {
    issue(0, r0);
    load_dz(r0);
    store_dz(0);
  }
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += BR, buf ^= 1) {
    const bool more = rb + BR < r1;
    if (more) {
      issue(buf ^ 1, rb + BR);
      load_dz(rb + BR);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int lim = (r1 - rb < BR) ? static_cast<int>(r1 - rb) : BR;
    if (ok) {
      const int rs = LO ? 2 * H : H;                   // row layout [hi(0..H) | lo(0..H)] or [hi]
      __nv_bfloat16* hp = da_hilo + rb * rs + j;
      __nv_bfloat16* lp = hp + H;
#pragma unroll 2
      for (int rr = 0; rr < lim; ++rr) {
        const float2 x2 = *reinterpret_cast<const float2*>(&abuf[buf][rr][2 * threadIdx.x]);
        row_step(x2, buf, rr, hp + rr * rs, lp + rr * rs);
      }
    }
    if (more) store_dz(buf ^ 1);
    __syncthreads();
  }
  if (ok) {
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
      if (e < E) *reinterpret_cast<float2*>(dw2_part + (static_cast<int64_t>(slice) * E + e) * H + j) = acc[e];
    *reinterpret_cast<float2*>(db1_part + static_cast<int64_t>(slice) * H + j) = db1;
  }
  if (blockIdx.x == 0 && threadIdx.x < E) {
    float sacc = 0.f;
    for (int64_t row = r0; row < r1; ++row) sacc += dz[row * E + threadIdx.x];
    db2_part[static_cast<int64_t>(slice) * E + threadIdx.x] = sacc;
  }
}

// dW2 / db1 / db2 slice sums in one launch: element i of the concatenation
// [E*H | H | E] reads its own segment's partials (fixed slice order).
template <typename T>
__global__ void sum_slices3_kernel(const T* __restrict__ p0, const T* __restrict__ p1, const T* __restrict__ p2,
                                   int nslice, int64_t l0, int64_t l1, int64_t l2, T* __restrict__ o0,
                                   T* __restrict__ o1, T* __restrict__ o2) {
  const int64_t tot = l0 + l1 + l2;
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < tot;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T* part;
    T* out;
    int64_t i, len;
    if (g < l0) { part = p0; out = o0; i = g; len = l0; }
    else if (g < l0 + l1) { part = p1; out = o1; i = g - l0; len = l1; }
    else { part = p2; out = o2; i = g - l0 - l1; len = l2; }
    T s = T(0);
    int k = 0;
    for (; k + 8 <= nslice; k += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + (k + u) * len + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; k < nslice; ++k) s += part[k * len + i];
    out[i] = s;
  }
}

template <typename T>
static void sum_parts3(const T* dw2_part, const T* db1_part, const T* db2_part, int n_slices, int E, int H, T* dw2,
                       T* db1, T* db2, cudaStream_t st) {
  sum_slices3_kernel<T><<<moep_num_sms() * 2, 256, 0, st>>>(dw2_part, db1_part, db2_part, n_slices,
                                                            static_cast<int64_t>(E) * H, H, E, dw2, db1, db2);
}

// ------------------------------------------------------------------ K6
// Operation order follows trainer.py:109-122 (m *= b1; m += (1-b1) g; ...),
// evaluated in T (fp64 for the exact-parity mode, fp32 master otherwise).
template <typename T>
__device__ __forceinline__ T optim_elem(T pi, T gi, T* mi_io, T* vi_io, int kind, T lr, T b1, T b2, T eps, T bc1,
                                       T bc2, T mom) {
  if (kind == 0) {          // sgd
    pi -= lr * gi;
  } else if (kind == 1) {   // momentum: m = mu*m + g ; p -= lr*m
    T mi = *mi_io * mom;
    mi += gi;
    *mi_io = mi;
    pi -= lr * mi;
  } else {                  // adam with bias correction
    T mi = *mi_io * b1;
    mi += (T(1) - b1) * gi;
    T vi = *vi_io * b2;
    vi += (T(1) - b2) * gi * gi;
    *mi_io = mi;
    *vi_io = vi;
    const T mh = mi / bc1, vh = vi / bc2;
    pi -= lr * mh / (sqrt(vh) + eps);
  }
  return pi;
}

template <typename T>
__global__ void optim_kernel(T* __restrict__ p, const T* __restrict__ g, T* __restrict__ m,
                             T* __restrict__ v, int64_t n, int kind, T lr, T b1, T b2, T eps,
                             T bc1, T bc2, T mom, __nv_bfloat16* __restrict__ shadow,
                             int64_t n_shadow, int* __restrict__ nonfinite) {
  int bad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    T mi = kind >= 1 ? m[i] : T(0), vi = kind == 2 ? v[i] : T(0);
    const T pi = optim_elem<T>(p[i], g[i], &mi, &vi, kind, lr, b1, b2, eps, bc1, bc2, mom);
    if (kind >= 1) m[i] = mi;
    if (kind == 2) v[i] = vi;
    p[i] = pi;
    bad |= !isfinite(pi);
    if (shadow && i < n_shadow) shadow[i] = __float2bfloat16_rn(static_cast<float>(pi));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1);
}

// fp32 master weights, 16-byte aligned: four parameters per thread iteration
// (float4 loads / stores, the same per-element arithmetic as optim_kernel);
// the n % 4 tail is the scalar loop's.
__global__ void optim_f32x4_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                   float* __restrict__ v, int64_t n, int kind, float lr, float b1, float b2,
                                   float eps, float bc1, float bc2, float mom, __nv_bfloat16* __restrict__ shadow,
                                   int64_t n_shadow, int* __restrict__ nonfinite) {
  int bad = 0;
  const int64_t n4 = n >> 2;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n4; q += stride) {
    float4 pv = reinterpret_cast<const float4*>(p)[q];
    const float4 gv = __ldcs(reinterpret_cast<const float4*>(g) + q);
    float4 mv = kind >= 1 ? reinterpret_cast<const float4*>(m)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 vv = kind == 2 ? reinterpret_cast<const float4*>(v)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    pv.x = optim_elem<float>(pv.x, gv.x, &mv.x, &vv.x, kind, lr, b1, b2, eps, bc1, bc2, mom);
    pv.y = optim_elem<float>(pv.y, gv.y, &mv.y, &vv.y, kind, lr, b1, b2, eps, bc1, bc2, mom);
    pv.z = optim_elem<float>(pv.z, gv.z, &mv.z, &vv.z, kind, lr, b1, b2, eps, bc1, bc2, mom);
    pv.w = optim_elem<float>(pv.w, gv.w, &mv.w, &vv.w, kind, lr, b1, b2, eps, bc1, bc2, mom);
    if (kind >= 1) reinterpret_cast<float4*>(m)[q] = mv;
    if (kind == 2) reinterpret_cast<float4*>(v)[q] = vv;
    reinterpret_cast<float4*>(p)[q] = pv;
    bad |= !(isfinite(pv.x) && isfinite(pv.y) && isfinite(pv.z) && isfinite(pv.w));
    const int64_t i = q << 2;
    if (shadow) {
      if (i + 3 < n_shadow) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(pv.x, pv.y), hi = __floats2bfloat162_rn(pv.z, pv.w);
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&lo);
        u.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(shadow + i) = u;
      } else {
        const float e[4] = {pv.x, pv.y, pv.z, pv.w};
        for (int t = 0; t < 4; ++t)
          if (i + t < n_shadow) shadow[i + t] = __float2bfloat16_rn(e[t]);
      }
    }
  }
  for (int64_t i = (n4 << 2) + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    float mi = kind >= 1 ? m[i] : 0.f, vi = kind == 2 ? v[i] : 0.f;
    const float pi = optim_elem<float>(p[i], g[i], &mi, &vi, kind, lr, b1, b2, eps, bc1, bc2, mom);
    if (kind >= 1) m[i] = mi;
    if (kind == 2) v[i] = vi;
    p[i] = pi;
    bad |= !isfinite(pi);
    if (shadow && i < n_shadow) shadow[i] = __float2bfloat16_rn(pi);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1);
}

}  // namespace tr
}  // namespace moep

using namespace moep::tr;

template <typename T>
static int launch_loss(const moep_loss_args* a, const LossParams& p, cudaStream_t st) {
  const T* z = static_cast<const T*>(a->logits);
  const T* sc = static_cast<const T*>(a->scores);
  T* dz = static_cast<T*>(a->dz);
  T* dzh = static_cast<T*>(a->dz_hinge);
  const int E = a->n_experts;
#define MOEP_K4(LPR, EPL)                                                                                   \
  loss_kernel<T, LPR, EPL><<<a->n_blocks, NT, 0, st>>>(z, sc, a->rank_of, a->topk_mask, a->n, E, p, dz, dzh, \
                                                       a->partials)
  if (E <= 8) MOEP_K4(8, 1);
  else if (E <= 16) MOEP_K4(16, 1);
  else if (E <= 32) MOEP_K4(32, 1);
  else if (E <= 64) MOEP_K4(32, 2);
  else if (E <= 128) MOEP_K4(32, 4);
  else if (E <= 256) MOEP_K4(32, 8);
  else if (E <= 512) MOEP_K4(32, 16);
  else
    loss_rowwarp_kernel<T><<<a->n_blocks, NT, 0, st>>>(z, sc, a->rank_of, a->topk_mask, a->n, E, p, dz, dzh,
                                                       a->partials);
#undef MOEP_K4
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

extern "C" {

int moep_k7b_labels(const void* sc, int32_t dtype, int64_t n, int32_t E, int32_t k, int32_t top_cut,
                    int32_t* rank_of, uint8_t* mask, int32_t* pairs, void* stream);

int moep_labels(const void* scores, int32_t dtype, int64_t n, int32_t E, int32_t k, int32_t* rank_of,
                uint8_t* topk_mask, int32_t* pair_count, void* stream) {
  if (n <= 0 || E <= 0) return MOEP_ESHAPE;
  if (k < 1 || k > E) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = moep_num_sms() * 8;  // 8 CTAs of 256 per SM: hide the per-token shuffle chains
  const int top_cut = E < 10 ? E : 10;  // TOP_TIER_SIZE (losses.py:27)
  if (E == 16 || E == 32 || E == 64) {  // one thread per token, sorting network (k7b_rows.cu)
    const int rc = moep_k7b_labels(scores, dtype, n, E, k, top_cut, rank_of, topk_mask, pair_count, stream);
    if (rc != MOEP_EUNSUPPORTED) return rc;
  }
  if (E <= 256) {
#define MOEP_K3(T, LPR, EPL)                                                                                \
  labels_reg_kernel<T, LPR, EPL><<<grid, NT, 0, st>>>(static_cast<const T*>(scores), n, E, k, top_cut, rank_of, \
                                                      topk_mask, pair_count)
#define MOEP_K3_T(T)                        \
  do {                                      \
    if (E <= 8) MOEP_K3(T, 8, 1);           \
    else if (E <= 16) MOEP_K3(T, 16, 1);    \
    else if (E <= 32) MOEP_K3(T, 32, 1);    \
    else if (E <= 64) MOEP_K3(T, 32, 2);    \
    else if (E <= 128) MOEP_K3(T, 32, 4);   \
    else MOEP_K3(T, 32, 8);                 \
  } while (0)
    if (dtype == MOEP_F64) MOEP_K3_T(double);
    else if (dtype == MOEP_F32) MOEP_K3_T(float);
    else return MOEP_EARG;
#undef MOEP_K3_T
#undef MOEP_K3
    return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
  }
  if (dtype == MOEP_F64)
    labels_kernel<double><<<grid, NT, 0, st>>>(static_cast<const double*>(scores), n, E, k, top_cut, rank_of,
                                                 topk_mask, pair_count);
  else if (dtype == MOEP_F32)
    labels_kernel<float><<<grid, NT, 0, st>>>(static_cast<const float*>(scores), n, E, k, top_cut, rank_of,
                                                topk_mask, pair_count);
  else
    return MOEP_EARG;
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_loss(const moep_loss_args* a, void* stream) {
  if (!a || a->n <= 0 || a->n_experts <= 0 || a->n_blocks <= 0) return MOEP_ESHAPE;
  if (a->family < 0 || a->family > 4) return MOEP_EARG;
  if (a->family >= 3 && !a->dz_hinge) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LossParams p;
  p.family = a->family;
  p.top_w = a->top_weight; p.mid_w = a->mid_weight; p.rest_w = a->rest_weight;
  p.lam = a->ranking_lambda; p.margin = a->margin; p.gamma = a->focal_gamma; p.alpha = a->focal_alpha;
  p.top_cut = a->n_experts < 10 ? a->n_experts : 10;
  p.mid_cut = a->n_experts < 30 ? a->n_experts : 30;
  p.inv_ne = 1.0 / (static_cast<double>(a->n_global) * a->n_experts);
  p.inv_n = 1.0 / static_cast<double>(a->n_global);
  if (a->dtype == MOEP_F64)
    return launch_loss<double>(a, p, st);
  if (a->dtype == MOEP_F32)
    return launch_loss<float>(a, p, st);
  return MOEP_EARG;
}

int moep_loss_finalize(const double* partials, int32_t n_blocks, int64_t n, int32_t E, int32_t family,
                       double ranking_lambda, int32_t normalize, int32_t dtype, void* dz, const void* dz_hinge,
                       double* out_loss, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = family >= 3 ? moep_num_sms() : 1;
  if (dtype == MOEP_F64)
    finalize_kernel<double><<<grid, 256, 0, st>>>(partials, n_blocks, n, E, family, ranking_lambda, normalize,
                                                  static_cast<double*>(dz), static_cast<const double*>(dz_hinge),
                                                  out_loss);
  else if (dtype == MOEP_F32)
    finalize_kernel<float><<<grid, 256, 0, st>>>(partials, n_blocks, n, E, family, ranking_lambda, normalize,
                                                 static_cast<float*>(dz), static_cast<const float*>(dz_hinge),
                                                 out_loss);
  else
    return MOEP_EARG;
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // extern "C"

template <typename T, bool SPLIT>
static int act_backward_t(const T* a, const T* dz, const T* w2, int64_t n, int32_t H, int32_t E, int32_t n_slices,
                          T* da, __nv_bfloat16* da_hilo, T* dw2, T* db1, T* db2, T* scratch, cudaStream_t st) {
  const int rows_per_slice = static_cast<int>((n + n_slices - 1) / n_slices);
  T* dw2_part = scratch;
  T* db1_part = dw2_part + static_cast<int64_t>(n_slices) * E * H;
  T* db2_part = db1_part + static_cast<int64_t>(n_slices) * H;
  dim3 grid((H + 127) / 128, n_slices);
#define MOEP_K5(EM) act_backward_kernel<EM, T, SPLIT><<<grid, 128, 0, st>>>(a, dz, w2, n, H, E, rows_per_slice, da, \
                                                                          da_hilo, dw2_part, db1_part, db2_part)
  if (E <= 16) MOEP_K5(16);
  else if (E <= 32) MOEP_K5(32);
  else if (E <= 64) MOEP_K5(64);
  else MOEP_K5(128);
#undef MOEP_K5
  sum_parts3<T>(dw2_part, db1_part, db2_part, n_slices, E, H, dw2, db1, db2, st);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

extern "C" {

int moep_act_backward(const void* a, const void* dz, const void* w2, int32_t dtype, int64_t n, int32_t H,
                      int32_t E, int32_t n_slices, void* da, void* dw2, void* db1, void* db2, void* scratch,
                      void* stream) {
  if (n <= 0 || H <= 0 || E <= 0 || n_slices <= 0) return MOEP_ESHAPE;
  if (E > 128) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == MOEP_F64)
    return act_backward_t<double, false>(static_cast<const double*>(a), static_cast<const double*>(dz),
                                         static_cast<const double*>(w2), n, H, E, n_slices, static_cast<double*>(da),
                                         nullptr, static_cast<double*>(dw2), static_cast<double*>(db1),
                                         static_cast<double*>(db2), static_cast<double*>(scratch), st);
  if (dtype == MOEP_F32)
    return act_backward_t<float, false>(static_cast<const float*>(a), static_cast<const float*>(dz),
                                        static_cast<const float*>(w2), n, H, E, n_slices, static_cast<float*>(da),
                                        nullptr, static_cast<float*>(dw2), static_cast<float*>(db1),
                                        static_cast<float*>(db2), static_cast<float*>(scratch), st);
  return MOEP_EARG;
}

int moep_act_backward_bf16split(const float* a, const float* dz, const float* w2, int64_t n, int32_t H, int32_t E,
                                int32_t n_slices, int32_t with_lo, void* da_hilo, float* dw2, float* db1, float* db2,
                                float* scratch, void* stream) {
  if (n <= 0 || H <= 0 || E <= 0 || n_slices <= 0) return MOEP_ESHAPE;
  if (E > 128) return MOEP_EUNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(da_hilo);
  if (H % 4 != 0 || E > 32) {
    if (!with_lo) return MOEP_EUNSUPPORTED;
    return act_backward_t<float, true>(a, dz, w2, n, H, E, n_slices, nullptr, out, dw2, db1, db2, scratch, st);
  }
  const int gx = (H / 2 + 127) / 128;
  constexpr int kAbuf = 2 * BR * 256 * 4;  // staging for `a`
  // row slices: one resident wave (the occupancy calculator's blocks per SM x
  // SMs, divided over the column blocks), at most the caller's n_slices (its
  // scratch size). 128 slices ran 1.4 waves at H = 2048 (87 us per 16 k Phi rows).
  auto slices_for = [&](const void* kern) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, kAbuf) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    const int fit = per_sm * moep_num_sms() / gx;
    return fit < 1 ? 1 : (fit < n_slices ? fit : n_slices);
  };
#define MOEP_K5X2(EM, LOV)                                                                                     \
  do {                                                                                                         \
    if (cudaFuncSetAttribute(act_backward_f32x2_kernel<EM, LOV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             kAbuf) != cudaSuccess)                                                            \
      return MOEP_ELAUNCH;                                                                                     \
    ns = slices_for(reinterpret_cast<const void*>(act_backward_f32x2_kernel<EM, LOV>));                       \
    rows_per_slice = static_cast<int>((n + ns - 1) / ns);                                                      \
    dw2_part = scratch;                                                                                        \
    db1_part = dw2_part + static_cast<int64_t>(ns) * E * H;                                                    \
    db2_part = db1_part + static_cast<int64_t>(ns) * H;                                                        \
    act_backward_f32x2_kernel<EM, LOV><<<dim3(gx, ns), 128, kAbuf, st>>>(a, dz, w2, n, H, E, rows_per_slice,  \
                                                                        out, dw2_part, db1_part, db2_part);   \
  } while (0)
  int ns = n_slices, rows_per_slice = 0;
  float *dw2_part = nullptr, *db1_part = nullptr, *db2_part = nullptr;
  if (E <= 16) { if (with_lo) MOEP_K5X2(16, true); else MOEP_K5X2(16, false); }
  else { if (with_lo) MOEP_K5X2(32, true); else MOEP_K5X2(32, false); }
#undef MOEP_K5X2
  sum_parts3<float>(dw2_part, db1_part, db2_part, ns, E, H, dw2, db1, db2, st);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_optim_step(const moep_optim_args* a, void* stream) {
  if (!a || a->n <= 0) return MOEP_ESHAPE;
  if (a->kind < 0 || a->kind > 2) return MOEP_EARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // bias corrections as trainer.py:120-121 computes them: 1 - beta**t in float64
  const double bc1 = 1.0 - pow(a->beta1, static_cast<double>(a->t));
  const double bc2 = 1.0 - pow(a->beta2, static_cast<double>(a->t));
  const int grid = moep_num_sms() * 4;
  if (a->dtype == MOEP_F64)
    optim_kernel<double><<<grid, 256, 0, st>>>(
        static_cast<double*>(a->params), static_cast<const double*>(a->grads), static_cast<double*>(a->m),
        static_cast<double*>(a->v), a->n, a->kind, a->lr, a->beta1, a->beta2, a->eps, bc1, bc2, a->momentum,
        static_cast<__nv_bfloat16*>(a->shadow_bf16), a->n_shadow, a->nonfinite);
  else if (a->dtype == MOEP_F32 && ((reinterpret_cast<uintptr_t>(a->params) | reinterpret_cast<uintptr_t>(a->grads) |
                                       reinterpret_cast<uintptr_t>(a->m) | reinterpret_cast<uintptr_t>(a->v) |
                                       reinterpret_cast<uintptr_t>(a->shadow_bf16)) & 15) == 0)
    optim_f32x4_kernel<<<grid, 256, 0, st>>>(
        static_cast<float*>(a->params), static_cast<const float*>(a->grads), static_cast<float*>(a->m),
        static_cast<float*>(a->v), a->n, a->kind, static_cast<float>(a->lr), static_cast<float>(a->beta1),
        static_cast<float>(a->beta2), static_cast<float>(a->eps), static_cast<float>(bc1), static_cast<float>(bc2),
        static_cast<float>(a->momentum), static_cast<__nv_bfloat16*>(a->shadow_bf16), a->n_shadow, a->nonfinite);
  else if (a->dtype == MOEP_F32)
    optim_kernel<float><<<grid, 256, 0, st>>>(
        static_cast<float*>(a->params), static_cast<const float*>(a->grads), static_cast<float*>(a->m),
        static_cast<float*>(a->v), a->n, a->kind, static_cast<float>(a->lr), static_cast<float>(a->beta1),
        static_cast<float>(a->beta2), static_cast<float>(a->eps), static_cast<float>(bc1), static_cast<float>(bc2),
        static_cast<float>(a->momentum), static_cast<__nv_bfloat16*>(a->shadow_bf16), a->n_shadow, a->nonfinite);
  else
    return MOEP_EARG;
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // extern "C"
