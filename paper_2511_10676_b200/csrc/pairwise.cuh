// pairwise.cuh — numpy's float64 pairwise summation (numpy/_core/src/umath/
// loops_utils.h.src, pairwise_sum; add.reduce = 0 + pairwise_sum) on a warp
// over a shared-memory row: the leaves (<= 128 elements, 8 accumulators) go to
// lanes, lane 0 runs the combine program. Used where a result must be
// bit-identical to numpy's reductions (core.layer_norm / softmax in the
// synthetic teacher, the K0 input norm's general path).
#pragma once
#include <cstdint>

namespace moep {
namespace sg {

// ------------------------------------------------------------ pairwise sums
// numpy's reduction tree for length n, built once per block by thread 0:
// leaves (start, length <= 128) in order and a postfix program over them
// (>= 0: push leaf sum, -1: pop two, push left + right).
constexpr int kMaxLeaves = 512;
struct PwPlan {
  int n_leaves, n_prog;
  int start[kMaxLeaves], len[kMaxLeaves];
  int prog[2 * kMaxLeaves];
};

static __device__ void pw_build(PwPlan& p, int lo, int n) {
  if (n <= 128) {
    p.start[p.n_leaves] = lo;
    p.len[p.n_leaves] = n;
    p.prog[p.n_prog++] = p.n_leaves++;
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  pw_build(p, lo, n2);
  pw_build(p, lo + n2, n - n2);
  p.prog[p.n_prog++] = -1;
}

__device__ __host__ __forceinline__ int pad(int i) { return i + (i >> 7); }  // one pad double per 128: leaf starts spread over banks
// leaves have >= 64 elements once the length exceeds 128
__device__ __host__ __forceinline__ int leaf_cap(int len) { return len / 64 + 2; }

// op 0: element as is; op 1: (a - c)^2, rounded twice like numpy's x - mean, x * x;
// op 2: a * a (numpy's x * x)
template <int OP>
__device__ __forceinline__ double pw_elem(const double* a, int i, double c) {
  const double v = a[pad(i)];
  if (OP == 0) return v;
  if (OP == 2) return __dmul_rn(v, v);
  const double t = __dsub_rn(v, c);
  return __dmul_rn(t, t);
}

// numpy pairwise_sum of a leaf (loops_utils.h.src): n < 8 sequential from 0;
// else 8 accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the rest
template <int OP>
__device__ double pw_leaf(const double* a, int lo, int n, double c) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, pw_elem<OP>(a, lo + i, c));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = pw_elem<OP>(a, lo + j, c);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], pw_elem<OP>(a, lo + i + j, c));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, pw_elem<OP>(a, lo + i, c));
  return res;
}

// 0 + pairwise_sum over the warp's padded smem row; lanes take leaves, lane 0
// runs the combine program; result broadcast to the warp.
template <int OP>
__device__ double warp_pairwise(const double* a, const PwPlan& p, double c, double* leafsum, int lane) {
  for (int l = lane; l < p.n_leaves; l += 32) leafsum[l] = pw_leaf<OP>(a, p.start[l], p.len[l], c);
  __syncwarp();
  double total = 0.0;
  if (lane == 0) {
    double st[32];
    int sp = 0;
    for (int q = 0; q < p.n_prog; ++q) {
      const int op = p.prog[q];
      if (op >= 0) {
        st[sp++] = leafsum[op];
      } else {
        const double b = st[--sp], a2 = st[--sp];
        st[sp++] = __dadd_rn(a2, b);
      }
    }
    total = __dadd_rn(0.0, st[0]);
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, total, 0);
}

}  // namespace sg
}  // namespace moep
