// k_leaf.cu — the small dense pieces of the blocked EbV LU (all <= 64 wide):
//   leaf_lu          LU of a diagonal block (w <= 64) in one CTA
//   trsm_right_upper L21 = A21 U11^-1, one thread per row (row-parallel)
//   trsm_left_lower  U12 = L11^-1 A12, one thread per column (column-parallel)
//
// Paper: Eq 6-a l_ik = a_ik / a_kk; Eq 6-b the U_(k) row; Eq 6-c
// the rank-1 update.  Per entry, updates are applied as
// fma(-l_ik, u_kj, a_ij) in ascending k and the L division comes last — the
// canonical order of DESIGN.md — so each kernel is bitwise equal to the
// corresponding part of the serial oracle.
//
// Every kernel works on a fixed 64-wide block held in registers (fully
// unrolled, no runtime guards); a narrower block (a ragged tail) is padded
// with an identity: padded multipliers are exactly 0 and fma(-0, u, a) == a,
// so the real entries see exactly the same operation sequence.
#include "ebv_internal.cuh"

namespace ebv {
namespace {

constexpr int W = 64;        // block width
constexpr int S = W + 2;     // smem row stride (doubles): 16-byte aligned rows

// Work split used by the three kernels below: a group of G = 8 consecutive
// lanes shares one row (or column) of the 64-wide block; lane j of the group
// owns the entries c = j, j+8, ..., j+56.  Step p is carried out by the
// owner lane of entry p (division or final value), the value is broadcast
// to the group with a shuffle, and each lane applies the fma to its entries
// c > p — per entry exactly the ascending-p chain of the oracle.
constexpr int G = 8;          // lanes per row / column
constexpr int Q = W / G;      // entries per lane

// ---------------------------------------------------------------- leaf LU
// 512 threads: row i of the block is owned by group i.  Step k: group k
// publishes its final row (the U_(k) vector, Eq 6-b) to shared memory; every
// row i > k forms l_ik = a_ik / u_kk (Eq 6-a, owner lane), broadcasts it in
// the group and updates its row (Eq 6-c).  A narrower block is identity
// padded (exactly neutral).
__global__ void __launch_bounds__(W * G) leaf_lu_kernel(int w, double* __restrict__ A, int64_t lda,
                                                        const double* __restrict__ tau, int64_t* info, int64_t koff) {
  __shared__ __align__(16) double urow[2][W];
  __shared__ int smin;
  const int tid = threadIdx.x, i = tid / G, j = tid % G, lane = tid & 31, base = lane & ~(G - 1);
  double a[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int c = j + G * q;
    a[q] = (i < w && c < w) ? A[i + (int64_t)c * lda] : (i == c ? 1.0 : 0.0);
  }
  if (tid == 0) smin = 0x7fffffff;
  const double tv = *tau;
#pragma unroll
  for (int k = 0; k < W; k++) {
    const int o = k % G, qk = k / G;
    double* ur = urow[k & 1];
    if (i == k) {
#pragma unroll
      for (int q = qk; q < Q; q++) ur[j + G * q] = a[q];
    }
    __syncthreads();
    const double piv = ur[k];
    if (tid == 0 && k < w && fabs(piv) <= tv) atomicMin(&smin, k + 1);
    if (i > k && j == o) a[qk] = a[qk] / piv;
    const double l = __shfl_sync(0xffffffffu, a[qk], base + o);
    if (i > k) {
#pragma unroll
      for (int q = qk; q < Q; q++)
        if (q > qk || j > o) a[q] = fma(-l, ur[j + G * q], a[q]);
    }
  }
  __syncthreads();
  if (tid == 0 && smin != 0x7fffffff) {
    volatile int64_t* vi = info;
    if (*vi == 0) *vi = koff + smin;
  }
  if (i < w) {
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int c = j + G * q;
      if (c < w) A[i + (int64_t)c * lda] = a[q];
    }
  }
}

// ---------------------------------------------------------------- L21 = A21 U11^-1
// Group per row: step p, the owner lane divides x_p by u_pp, broadcasts it,
// every lane applies x_c = fma(-x_p, u_pc, x_c) to its entries c > p.
__global__ void __launch_bounds__(256) trsm_ru_kernel(int64_t m, int k, double* __restrict__ X, int64_t ldx,
                                                      const double* __restrict__ U, int64_t ldu) {
  __shared__ __align__(16) double sU[W * S];   // sU[p*S + c] = u(p, c), identity padded
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int p = idx % W, c = idx / W;
    sU[p * S + c] = (p < k && c < k) ? (p <= c ? U[p + (int64_t)c * ldu] : 0.0) : (p == c ? 1.0 : 0.0);
  }
  __syncthreads();
  const int tid = threadIdx.x, j = tid % G, lane = tid & 31, base = lane & ~(G - 1);
  const int64_t i = (int64_t)blockIdx.x * (256 / G) + tid / G;
  const bool rv = i < m;
  double x[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int c = j + G * q;
    x[q] = (rv && c < k) ? X[i + (int64_t)c * ldx] : 0.0;
  }
#pragma unroll
  for (int p = 0; p < W; p++) {
    const int o = p % G, qp = p / G;
    const double* up = sU + p * S;
    if (j == o) x[qp] = x[qp] / up[p];
    const double xp = __shfl_sync(0xffffffffu, x[qp], base + o);
#pragma unroll
    for (int q = qp; q < Q; q++)
      if (q > qp || j > o) x[q] = fma(-xp, up[j + G * q], x[q]);
  }
  if (rv) {
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int c = j + G * q;
      if (c < k) X[i + (int64_t)c * ldx] = x[q];
    }
  }
}

// ---------------------------------------------------------------- U12 = L11^-1 A12
// Group per column: step p, x_p is final (owner lane), broadcast; every lane
// applies x_r = fma(-l_rp, x_p, x_r) to its rows r > p (unit diagonal).
__global__ void __launch_bounds__(256) trsm_llu_kernel(int k, int64_t m, const double* __restrict__ L, int64_t ldl,
                                                       double* __restrict__ X, int64_t ldx) {
  __shared__ __align__(16) double sL[W * S];   // sL[p*S + r] = l(r, p), r > p
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int r = idx % W, p = idx / W;
    sL[p * S + r] = (r > p && r < k) ? L[r + (int64_t)p * ldl] : 0.0;
  }
  __syncthreads();
  const int tid = threadIdx.x, j = tid % G, lane = tid & 31, base = lane & ~(G - 1);
  const int64_t cidx = (int64_t)blockIdx.x * (256 / G) + tid / G;
  const bool cv = cidx < m;
  double* col = X + (cv ? cidx : 0) * ldx;
  double x[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) {
    const int r = j + G * q;
    x[q] = (cv && r < k) ? col[r] : 0.0;
  }
#pragma unroll
  for (int p = 0; p < W; p++) {
    const int o = p % G, qp = p / G;
    const double* lp = sL + p * S;
    const double xp = __shfl_sync(0xffffffffu, x[qp], base + o);
#pragma unroll
    for (int q = qp; q < Q; q++)
      if (q > qp || j > o) x[q] = fma(-lp[j + G * q], xp, x[q]);
  }
  if (cv) {
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int r = j + G * q;
      if (r < k) col[r] = x[q];
    }
  }
}

// ---------------------------------------------------------------- X = U11^-1 X
// Backward substitution per column (thread per column), k descending:
// x_p = x_p / u_pp, then x_i = fma(-u_ip, x_p, x_i) for i < p — the oracle's
// backward order (Eq 1, UX = Y).  Padded rows (p >= k) are identity rows and
// come first in the descending sweep: they change nothing.
__global__ void __launch_bounds__(128) trsm_luu_kernel(int k, int64_t m, const double* __restrict__ U, int64_t ldu,
                                                       double* __restrict__ X, int64_t ldx) {
  __shared__ __align__(16) double sU[W * S];   // sU[p*S + i] = u(i, p), i <= p (column p of U)
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int i = idx % W, p = idx / W;
    sU[p * S + i] = (i < k && p < k) ? (i <= p ? U[i + (int64_t)p * ldu] : 0.0) : (i == p ? 1.0 : 0.0);
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double* col = X + c * ldx;
  double x[W];
#pragma unroll
  for (int r = 0; r < W; r++) x[r] = (r < k) ? col[r] : 0.0;
#pragma unroll
  for (int p = W - 1; p >= 0; p--) {
    const double* up = sU + p * S;
    x[p] = x[p] / up[p];
#pragma unroll
    for (int i = 0; i < p; i++) x[i] = fma(-up[i], x[p], x[i]);
  }
#pragma unroll
  for (int r = 0; r < W; r++)
    if (r < k) col[r] = x[r];
}

}  // namespace

cudaError_t launch_trsm_left_upper(int64_t k, int64_t m, const double* U, int64_t ldu, double* X, int64_t ldx,
                                   cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  trsm_luu_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>((int)k, m, U, ldu, X, ldx);
  return cudaGetLastError();
}

cudaError_t launch_leaf_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info, int64_t koff,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > W) return cudaErrorInvalidValue;
  leaf_lu_kernel<<<1, W * G, 0, s>>>((int)n, A, lda, tau, info, koff);
  return cudaGetLastError();
}

cudaError_t launch_trsm_right_upper(int64_t m, int64_t k, double* X, int64_t ldx, const double* U, int64_t ldu,
                                    cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  trsm_ru_kernel<<<(unsigned)((m + 31) / 32), 256, 0, s>>>(m, (int)k, X, ldx, U, ldu);
  return cudaGetLastError();
}

cudaError_t launch_trsm_left_lower_unit(int64_t k, int64_t m, const double* L, int64_t ldl, double* X,
                                        int64_t ldx, cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  trsm_llu_kernel<<<(unsigned)((m + 31) / 32), 256, 0, s>>>((int)k, m, L, ldl, X, ldx);
  return cudaGetLastError();
}

}  // namespace ebv
