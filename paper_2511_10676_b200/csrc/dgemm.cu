// dgemm.cu — fp64 GEMM on the fp64 tensor cores (DMMA m8n8k4) for the
// synthetic teacher's dense maps (synthgen.py:176-189):
// the linear mix x @ M^T, the nonlinear map tanh(x @ W_in^T) @ W_out^T and the
// gate logits post @ W_g^T. All are "NT" products of row-major operands:
//   C[M, N] = epi( A[M, K] . B[N, K]^T ),  epi = identity | tanh
// The reference runs them in numpy float64 (OpenBLAS); results agree to fp64
// round-off (fixed summation order here: k ascending within each thread's
// DMMA chain), which is what the teacher's float32 scores see.
//
// Tiles of 64 x 128 outputs per CTA (128 x 64 for N <= 64), K in steps of 16 double-buffered through
// shared memory (k-major, padded pitches so the fragment reads are
// conflict-free), 8 warps each owning a 32 x 32 block = 4 x 4 m8n8 DMMA tiles
// (16 independent accumulator chains per warp).
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/moep_b200.h"

namespace moep {
namespace dg {

constexpr int KS = 16, NT = 256;

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// TM x TN tile (64 x 128, or 128 x 64 when N <= 64: the gate's E columns),
// warps WM x WN = (TM / 32) x (TN / 32). TN_MODE: A is [K, M] and B [K, N]
// (C = A^T . B: the fp64 training mode's dW1 = dA^T X, predictor.py:295).
template <int EPI, int TM, int TN, bool TN_MODE = false>
__global__ void __launch_bounds__(NT, 2)
dgemm_nt_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                double* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K) {
  constexpr int AP = TM + 4, BP = TN + 4, WM = TM / 32;
  constexpr int AK = KS * TM / NT, BK = KS * TN / NT;  // consecutive k per loader thread
  extern __shared__ double dsm[];  // As [2][KS * AP], Bs [2][KS * BP] (51 KB: dynamic)
  double (*As)[KS * AP] = reinterpret_cast<double (*)[KS * AP]>(dsm);
  double (*Bs)[KS * BP] = reinterpret_cast<double (*)[KS * BP]>(dsm + 2 * KS * AP);
  const int tid = threadIdx.x;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * TM, n0 = static_cast<int64_t>(blockIdx.x) * TN;
  // loaders: A thread = (row tid % TM, k-group tid / TM) -> AK consecutive k;
  //          B thread = (row tid % TN, k-group tid / TN) -> BK consecutive k
  const int ar = tid & (TM - 1), akq = tid / TM;
  const int br = tid & (TN - 1), bkh = tid / TN;
  const int64_t arow = m0 + ar, brow = n0 + br;
  const bool vec = ((lda | ldb) & 1) == 0 && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
  double ra[AK > TM / 16 ? AK : TM / 16], rb[BK > TN / 16 ? BK : TN / 16];
  // TN mode loaders: thread = (k row tid / 16, MN run of TM/16 or TN/16 from (tid % 16))
  constexpr int AR = TM / 16, BR = TN / 16;
  auto fetch_t = [&](int64_t k0) {
    const int64_t kk = k0 + tid / 16;
    const int64_t ma = m0 + (tid % 16) * AR, nb = n0 + (tid % 16) * BR;
#pragma unroll
    for (int c = 0; c < AR; ++c) ra[c] = (kk < K && ma + c < M) ? A[kk * lda + ma + c] : 0.0;
#pragma unroll
    for (int c = 0; c < BR; ++c) rb[c] = (kk < K && nb + c < N) ? B[kk * ldb + nb + c] : 0.0;
  };
  auto stash_t = [&](int buf) {
#pragma unroll
    for (int c = 0; c < AR; ++c) As[buf][(tid / 16) * AP + (tid % 16) * AR + c] = ra[c];
#pragma unroll
    for (int c = 0; c < BR; ++c) Bs[buf][(tid / 16) * BP + (tid % 16) * BR + c] = rb[c];
  };
  auto fetch = [&](int64_t k0) {
    if (TN_MODE) { fetch_t(k0); return; }
    const int64_t ka = k0 + akq * AK, kb = k0 + bkh * BK;
    if (vec && arow < M && ka + AK <= K) {
      const double2* p = reinterpret_cast<const double2*>(A + arow * lda + ka);
#pragma unroll
      for (int c = 0; c < AK / 2; ++c) { const double2 u = __ldg(p + c); ra[2 * c] = u.x; ra[2 * c + 1] = u.y; }
    } else {
#pragma unroll
      for (int c = 0; c < AK; ++c) ra[c] = (arow < M && ka + c < K) ? A[arow * lda + ka + c] : 0.0;
    }
    if (vec && brow < N && kb + BK <= K) {
      const double2* p = reinterpret_cast<const double2*>(B + brow * ldb + kb);
#pragma unroll
      for (int c = 0; c < BK / 2; ++c) { const double2 u = __ldg(p + c); rb[2 * c] = u.x; rb[2 * c + 1] = u.y; }
    } else {
#pragma unroll
      for (int c = 0; c < BK; ++c) rb[c] = (brow < N && kb + c < K) ? B[brow * ldb + kb + c] : 0.0;
    }
  };
  auto stash = [&](int buf) {
    if (TN_MODE) { stash_t(buf); return; }
#pragma unroll
    for (int c = 0; c < AK; ++c) As[buf][(akq * AK + c) * AP + ar] = ra[c];
#pragma unroll
    for (int c = 0; c < BK; ++c) Bs[buf][(bkh * BK + c) * BP + br] = rb[c];
  };
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, q4 = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t nk = (K + KS - 1) / KS;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = static_cast<int>(kt & 1);
    if (kt + 1 < nk) fetch((kt + 1) * KS);
#pragma unroll
    for (int k4 = 0; k4 < KS; k4 += 4) {
      double av[4], bv[4];
      const double* ap = &As[buf][(k4 + q4) * AP + wm * 32 + g];
      const double* bp = &Bs[buf][(k4 + q4) * BP + wn * 32 + g];
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
  // lane (g, q4) holds C[m + g][n + 2 q4 .. +1] of each m8n8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm * 32 + 8 * i + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + wn * 32 + 8 * j + 2 * q4;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + h < N) {
          double v = acc[i][j][h];
          if (EPI == 1) v = tanh(v);
          C[r * ldc + c + h] = v;
        }
      }
    }
  }
}

}  // namespace dg
}  // namespace moep

extern "C" int moep_dgemm_nt(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                             int64_t M, int64_t N, int64_t K, int32_t epilogue, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || lda < K || ldb < K || ldc < N) return MOEP_ESHAPE;
  if (!A || !B || !C) return MOEP_EARG;
  if (epilogue != 0 && epilogue != 1) return MOEP_EARG;
  const bool narrow = N <= 64;
  const int TM = narrow ? 128 : 64, TN = narrow ? 64 : 128;
  const int64_t gy = (M + TM - 1) / TM, gx = (N + TN - 1) / TN;
  if (gy > 65535) return MOEP_EUNSUPPORTED;
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t sm = 2 * moep::dg::KS * (TM + 4 + TN + 4) * sizeof(double);
  static bool attr[4] = {false, false, false, false};
  using K_t = void (*)(const double*, int64_t, const double*, int64_t, double*, int64_t, int64_t, int64_t, int64_t);
  const K_t kerns[4] = {moep::dg::dgemm_nt_kernel<0, 64, 128>, moep::dg::dgemm_nt_kernel<1, 64, 128>,
                        moep::dg::dgemm_nt_kernel<0, 128, 64>, moep::dg::dgemm_nt_kernel<1, 128, 64>};
  const int ki = (narrow ? 2 : 0) + epilogue;
  if (!attr[ki]) {
    if (cudaFuncSetAttribute(kerns[ki], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)) !=
        cudaSuccess)
      return MOEP_ELAUNCH;
    attr[ki] = true;
  }
  kerns[ki]<<<grid, moep::dg::NT, sm, st>>>(A, lda, B, ldb, C, ldc, M, N, K);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}

// C[M, N] = A[K, M]^T . B[K, N] (row-major operands, token-major: the fp64
// training mode's dW1 = dA^T X, predictor.py:295)
extern "C" int moep_dgemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                             int64_t M, int64_t N, int64_t K, void* stream) {
  if (M <= 0 || N <= 0 || K <= 0 || lda < M || ldb < N || ldc < N) return MOEP_ESHAPE;
  if (!A || !B || !C) return MOEP_EARG;
  const int64_t gy = (M + 63) / 64, gx = (N + 127) / 128;
  if (gy > 65535) return MOEP_EUNSUPPORTED;
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  const size_t sm = 2 * moep::dg::KS * (64 + 4 + 128 + 4) * sizeof(double);
  static bool attr = false;
  auto kern = moep::dg::dgemm_nt_kernel<0, 64, 128, true>;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)) != cudaSuccess)
      return MOEP_ELAUNCH;
    attr = true;
  }
  kern<<<grid, moep::dg::NT, sm, static_cast<cudaStream_t>(stream)>>>(A, lda, B, ldb, C, ldc, M, N, K);
  return cudaGetLastError() == cudaSuccess ? MOEP_OK : MOEP_ELAUNCH;
}
