// Standalone probe: validates the sm100.cuh descriptor encodings (TMA SW128 ->
// tcgen05.mma kind::f16 -> TMEM -> tcgen05.ld) on one 128x128 tile against a
// CPU reference. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2
//   -I paper_2511_10676_b200/csrc tools/probe_umma.cu -o /tmp/probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace moep;

constexpr int BM = 128, BN = 128, BK = 64;

__global__ void __launch_bounds__(128, 1)
probe_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* C,
           int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + BM * BK * 2;
  __shared__ uint64_t full_bar, mma_bar;
  __shared__ uint32_t tmem_base;
  if (threadIdx.x == 0) {
    mbar_init(&full_bar, 1);
    mbar_init(&mma_bar, 1);
    fence_barrier_init();
  }
  if (warp_id() == 0) tmem_alloc<128>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_bf16_f32(BM, BN);
  uint32_t phase = 0;
  for (int kb = 0; kb < K / BK; ++kb) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&full_bar, (BM + BN) * BK * 2);
      tma_load_2d(&ta, &full_bar, sA, kb * BK, 0);
      tma_load_2d(&tb, &full_bar, sB, kb * BK, 0);
    }
    mbar_wait(&full_bar, phase);
    tc_fence_after();
    if (threadIdx.x == 0) {
      for (int k = 0; k < BK / 16; ++k) {
        uint64_t ad = sdesc_k_sw128(smem_u32(sA) + k * 32);
        uint64_t bd = sdesc_k_sw128(smem_u32(sB) + k * 32);
        umma_bf16(tmem, ad, bd, idesc, (kb | k) != 0);
      }
      umma_commit(&mma_bar);
    }
    mbar_wait(&mma_bar, phase);
    tc_fence_after();
    phase ^= 1;
  }
  // epilogue: warp w reads lanes 32w..32w+31
  uint32_t row = warp_id() * 32 + lane_id();
  for (int c = 0; c < BN; c += 32) {
    float v[32];
    tmem_ld32(tmem + ((warp_id() * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) C[row * BN + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<128>(tmem);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<EncodeFn>(fn);
}

static void make_map(EncodeFn enc, CUtensorMap* m, void* ptr, uint64_t rows, uint64_t cols,
                     uint32_t box_rows, uint32_t box_cols) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

int main(int argc, char** argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 256;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  std::vector<__nv_bfloat16> hA(BM * K), hB(BN * K);
  std::vector<float> fA(BM * K), fB(BN * K);
  srand(1);
  auto gauss = []() { double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0); return sqrt(-2 * log(u1)) * cos(6.283185307 * u2); };
  for (int i = 0; i < BM * K; ++i) { float x = mode ? (float)gauss() : (rand() % 17 - 8) / 8.0f; hA[i] = __float2bfloat16(x); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < BN * K; ++i) { float x = mode ? (float)((rand() / (double)RAND_MAX * 2 - 1) * 0.0221) : (rand() % 13 - 6) / 4.0f; hB[i] = __float2bfloat16(x); fB[i] = __bfloat162float(hB[i]); }
  void *dA, *dB; float* dC;
  cudaMalloc(&dA, BM * K * 2); cudaMalloc(&dB, BN * K * 2); cudaMalloc(&dC, BM * BN * 4);
  cudaMemcpy(dA, hA.data(), BM * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), BN * K * 2, cudaMemcpyHostToDevice);
  EncodeFn enc = get_encode();
  CUtensorMap ta, tb;
  make_map(enc, &ta, dA, BM, K, BM, BK);
  make_map(enc, &tb, dB, BN, K, BN, BK);
  int smem = (BM + BN) * BK * 2 + 1024;
  cudaFuncSetAttribute(probe_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_gemm<<<1, 128, smem>>>(ta, tb, dC, K);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> hC(BM * BN);
  cudaMemcpy(hC.data(), dC, BM * BN * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, sse = 0, sbias = 0, sref = 0, sse_rn = 0; int bad = 0;
  for (int i = 0; i < BM; ++i)
    for (int j = 0; j < BN; ++j) {
      double s = 0; float srn = 0.f;
      for (int k = 0; k < K; ++k) { s += (double)fA[i * K + k] * fB[j * K + k]; }
      for (int k0 = 0; k0 < K; k0 += 16) { double blk = 0; for (int k = k0; k < k0 + 16; ++k) blk += (double)fA[i * K + k] * fB[j * K + k]; srn = (float)((double)srn + blk); }
      double e = (double)hC[i * BN + j] - s;
      double err = fabs(e);
      if (err > maxerr) maxerr = err;
      sse += e * e; sbias += (s >= 0 ? e : -e); sref += s * s;
      sse_rn += ((double)srn - s) * ((double)srn - s);
      if (err > 1e-2 * (1 + fabs(s)) && bad++ < 5) printf("mismatch %d %d: %f vs %f\n", i, j, hC[i * BN + j], s);
    }
  int n = BM * BN;
  printf("PROBE K=%d mode=%d max err %g rms err %g signed-toward-away-from-zero mean %g ref rms %g | emulated RN-per-16 rms %g bad %d\n", K, mode, maxerr, sqrt(sse / n), sbias / n, sqrt(sref / n), sqrt(sse_rn / n), bad);
  return bad ? 1 : 0;
}
