// bn_train.cu — arch1 training kernels (fp64): batch-norm with batch
// statistics, GELU-tanh, Philox dropout, and the matching backward.
//
// Restates the train-mode branch of the reference predictor:
//   forward  predictor.py:208-237 — batch mean / population variance per hidden
//            unit, running-stat update with the unbiased variance (momentum),
//            a_hat, bn_out = scale*a_hat + shift, g = gelu_tanh(bn_out), dropout
//            mask = rng.random(g.shape) >= rate from numpy's Philox4x64-10
//            stream keyed (seed << 64) + step (predictor.py:70-72, 227-231),
//            h = g * mask / (1 - rate);
//   backward predictor.py:280-297 — dg = dh*keep, dbn = dg*gelu'(bn_out),
//            d_scale/d_shift, da through the batch statistics, db1.
// The Philox implementation follows Random123's philox4x64-10 as used by numpy:
// element i of the row-major stream is word i%4 of the block with counter i/4+1.
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/moep_b200.h"

namespace moep {
namespace bn {

__device__ __forceinline__ void philox4x64(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

// uniform double of element i: numpy next_double = (u64 >> 11) * 2^-53
__device__ __forceinline__ double philox_uniform(uint64_t i, uint64_t k0, uint64_t k1) {
  uint64_t c[4] = {i / 4 + 1, 0, 0, 0};
  philox4x64(c, k0, k1);
  return static_cast<double>(c[i & 3] >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double gelu(double u) {
  const double cc = 0.79788456080286535588, ga = 0.044715;
  return 0.5 * u * (1.0 + tanh(cc * (u + ga * (u * u * u))));
}
__device__ __forceinline__ double gelu_grad(double u) {
  const double cc = 0.79788456080286535588, ga = 0.044715;
  const double t = tanh(cc * (u + ga * (u * u * u)));
  const double dt = (1.0 - t * t) * cc * (1.0 + 3.0 * ga * (u * u));
  return 0.5 * (1.0 + t) + 0.5 * u * dt;
}

// one thread per hidden column: statistics, running update, per-element outputs
__global__ void bn_forward_kernel(const double* __restrict__ a, int64_t n, int H, const double* __restrict__ scale,
                                  const double* __restrict__ shift, double* __restrict__ run_mean,
                                  double* __restrict__ run_var, double momentum, double eps, double rate,
                                  uint64_t key_step, uint64_t key_seed, const uint8_t* __restrict__ given_mask,
                                  double* __restrict__ a_hat, double* __restrict__ bn_out, double* __restrict__ keep,
                                  double* __restrict__ h, double* __restrict__ inv_std_out, int training) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  double mu, inv_std;
  if (training) {
    double s = 0.0;
    for (int64_t r = 0; r < n; ++r) s += a[r * H + j];
    mu = s / static_cast<double>(n);
    double v = 0.0;
    for (int64_t r = 0; r < n; ++r) {
      const double c = a[r * H + j] - mu;
      v += c * c;
    }
    const double var = v / static_cast<double>(n);
    inv_std = 1.0 / sqrt(var + eps);
    const double var_run = n > 1 ? var * (static_cast<double>(n) / static_cast<double>(n - 1)) : var;
    run_mean[j] = __dadd_rn(__dmul_rn(run_mean[j], 1.0 - momentum), __dmul_rn(momentum, mu));
    run_var[j] = __dadd_rn(__dmul_rn(run_var[j], 1.0 - momentum), __dmul_rn(momentum, var_run));
  } else {
    // eval mode: running statistics, no dropout (predictor.py:221-224, 236-237)
    mu = run_mean[j];
    inv_std = 1.0 / sqrt(run_var[j] + eps);
    rate = 0.0;
  }
  inv_std_out[j] = inv_std;
  const double sc = scale[j], sh = shift[j];
  const double inv_keep = rate > 0.0 ? 1.0 / (1.0 - rate) : 1.0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = r * H + j;
    const double ah = (a[i] - mu) * inv_std;
    const double bo = sc * ah + sh;
    const double g = gelu(bo);
    double kp = 1.0;
    if (rate > 0.0) {
      const bool m = given_mask ? given_mask[i] != 0 : philox_uniform(static_cast<uint64_t>(i), key_step, key_seed) >= rate;
      kp = (m ? 1.0 : 0.0) * inv_keep;
    }
    a_hat[i] = ah;
    bn_out[i] = bo;
    keep[i] = kp;
    h[i] = g * kp;
  }
}

// z[n, e] = sum_j h[n, j] * W[e, j] + b[e]; one warp per (row, expert)
__global__ void rows_dot_kernel(const double* __restrict__ hmat, const double* __restrict__ w,
                                const double* __restrict__ b, int64_t n, int H, int E, double* __restrict__ z) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= n * E) return;
  const int64_t r = gw / E;
  const int e = static_cast<int>(gw - r * E);
  double s = 0.0;
  for (int j = lane; j < H; j += 32) s += hmat[r * H + j] * w[static_cast<int64_t>(e) * H + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) z[r * E + e] = s + b[e];
}

// one thread per hidden column: dW2 column, BN-train backward, db1, d_scale, d_shift
__global__ void bn_backward_kernel(const double* __restrict__ dz, const double* __restrict__ w2, int64_t n, int H,
                                   int E, const double* __restrict__ hmat, const double* __restrict__ keep,
                                   const double* __restrict__ bn_out, const double* __restrict__ a_hat,
                                   const double* __restrict__ inv_std, const double* __restrict__ scale,
                                   double* __restrict__ da, double* __restrict__ dw2, double* __restrict__ db1,
                                   double* __restrict__ dscale, double* __restrict__ dshift, int training) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  const double sc = scale[j];
  double s_dbn = 0.0, s_dbn_ah = 0.0, s_dah = 0.0, s_dah_ah = 0.0;
  // pass 1: dW2 column and the batch sums of dbn, dbn * a_hat
  for (int e = 0; e < E; ++e) dw2[static_cast<int64_t>(e) * H + j] = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = r * H + j;
    double dh = 0.0;
    const double hv = hmat[i];
    for (int e = 0; e < E; ++e) {
      const double g = dz[r * E + e];
      dh += g * w2[static_cast<int64_t>(e) * H + j];
      dw2[static_cast<int64_t>(e) * H + j] += g * hv;
    }
    const double dbn = dh * keep[i] * gelu_grad(bn_out[i]);
    const double dah = dbn * sc;
    s_dbn += dbn;
    s_dbn_ah += dbn * a_hat[i];
    s_dah += dah;
    s_dah_ah += dah * a_hat[i];
    da[i] = dbn;  // stash dbn, turned into da in pass 2
  }
  dscale[j] = s_dbn_ah;
  dshift[j] = s_dbn;
  // da = inv_std/n * (n*da_hat - sum(da_hat) - a_hat*sum(da_hat*a_hat)), da_hat = dbn*scale
  const double nn = static_cast<double>(n);
  const double sum_dah = s_dah, sum_dah_ah = s_dah_ah;
  const double is = inv_std[j];
  double s_da = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = r * H + j;
    const double dah = da[i] * sc;
    // train: through the batch statistics; eval: da = da_hat * inv_std (predictor.py:292-296)
    const double v = training ? is / nn * (nn * dah - sum_dah - a_hat[i] * sum_dah_ah) : dah * is;
    da[i] = v;
    s_da += v;
  }
  db1[j] = s_da;
}

}  // namespace bn
}  // namespace moep

extern "C" {

int moep_bn_forward(const double* a, int64_t n, int32_t hidden, const double* scale, const double* shift,
                    double* run_mean, double* run_var, double momentum, double eps, double dropout_rate,
                    uint64_t dropout_seed, uint64_t dropout_step, const uint8_t* given_mask, double* a_hat,
                    double* bn_out, double* keep, double* h, double* inv_std, int32_t training, void* stream) {
  if (n <= 0 || hidden <= 0) return MOEP_ESHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  moep::bn::bn_forward_kernel<<<(hidden + 127) / 128, 128, 0, st>>>(
      a, n, hidden, scale, shift, run_mean, run_var, momentum, eps, dropout_rate, dropout_step, dropout_seed,
      given_mask, a_hat, bn_out, keep, h, inv_std, training);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_rows_dot(const double* h, const double* w, const double* b, int64_t n, int32_t hidden, int32_t n_out,
                  double* z, void* stream) {
  if (n <= 0 || hidden <= 0 || n_out <= 0) return MOEP_ESHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t warps = n * n_out;
  moep::bn::rows_dot_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(h, w, b, n, hidden,
                                                                                            n_out, z);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

int moep_bn_backward(const double* dz, const double* w2, int64_t n, int32_t hidden, int32_t n_experts,
                     const double* h, const double* keep, const double* bn_out, const double* a_hat,
                     const double* inv_std, const double* scale, double* da, double* dw2, double* db1,
                     double* dscale, double* dshift, int32_t training, void* stream) {
  if (n <= 0 || hidden <= 0 || n_experts <= 0) return MOEP_ESHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  moep::bn::bn_backward_kernel<<<(hidden + 127) / 128, 128, 0, st>>>(dz, w2, n, hidden, n_experts, h, keep, bn_out,
                                                                    a_hat, inv_std, scale, da, dw2, db1, dscale,
                                                                    dshift, training);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

}  // extern "C"
