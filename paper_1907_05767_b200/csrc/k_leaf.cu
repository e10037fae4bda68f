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

// ---------------------------------------------------------------- leaf LU
// The w x w block lives in shared memory (column-major, padded).  Warp v owns
// the columns j = v, v+8, ...; lane l owns rows l and l+32.  Step k: the
// owner warp of column k divides it below the diagonal (Eq 6-a, the L_(k)
// vector); after a barrier every warp applies the rank-1 update (Eq 6-c) to
// its columns j > k using the U_(k) entry a_kj (Eq 6-b).  A narrower block is
// padded with an identity (exactly neutral).
constexpr int LS = W + 1;
__global__ void __launch_bounds__(256) leaf_lu_kernel(int w, double* __restrict__ A, int64_t lda,
                                                      const double* __restrict__ tau, int64_t* info, int64_t koff) {
  __shared__ double s[W * LS];   // s[j*LS + i] = a(i, j)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < W * W; idx += 256) {
    const int i = idx % W, j = idx / W;
    s[j * LS + i] = (i < w && j < w) ? A[i + (int64_t)j * lda] : (i == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const double tv = *tau;
  int fail = 0;
  for (int k = 0; k < W; k++) {
    const double piv = s[k * LS + k];
    if (tid == 0 && k < w && fabs(piv) <= tv && fail == 0) fail = k + 1;
    if (warp == (k & 7)) {
      double* ck = s + k * LS;
      if (lane > k) ck[lane] = ck[lane] / piv;
      if (lane + 32 > k) ck[lane + 32] = ck[lane + 32] / piv;
    }
    __syncthreads();
    const double l0 = s[k * LS + lane], l1 = s[k * LS + lane + 32];
    for (int j = k + 1 + ((warp - k - 1) & 7); j < W; j += 8) {
      double* cj = s + j * LS;
      const double u = cj[k];
      if (lane > k) cj[lane] = fma(-l0, u, cj[lane]);
      if (lane + 32 > k) cj[lane + 32] = fma(-l1, u, cj[lane + 32]);
    }
    __syncthreads();
  }
  if (tid == 0 && fail) {
    volatile int64_t* vi = info;
    if (*vi == 0) *vi = koff + fail;
  }
  for (int idx = tid; idx < w * w; idx += 256) {
    const int i = idx % w, j = idx / w;
    A[i + (int64_t)j * lda] = s[j * LS + i];
  }
}

// ---------------------------------------------------------------- L21 = A21 U11^-1
// Thread per row; right-looking in registers: x_p /= u_pp, then
// x_j = fma(-x_p, u_pj, x_j) for j > p — per entry: ascending p, division last.
__global__ void __launch_bounds__(128) trsm_ru_kernel(int64_t m, int k, double* __restrict__ X, int64_t ldx,
                                                      const double* __restrict__ U, int64_t ldu) {
  __shared__ __align__(16) double sU[W * S];   // sU[p*S + j] = u(p, j)
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int p = idx % W, j = idx / W;          // consecutive p: coalesced column reads
    sU[p * S + j] = (p < k && j < k) ? (p <= j ? U[p + (int64_t)j * ldu] : 0.0) : (p == j ? 1.0 : 0.0);
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double x[W];
#pragma unroll
  for (int j = 0; j < W; j++) x[j] = (j < k) ? X[i + (int64_t)j * ldx] : 0.0;
#pragma unroll
  for (int p = 0; p < W; p++) {
    const double* up = sU + p * S;
    x[p] = x[p] / up[p];
#pragma unroll
    for (int j = p + 1; j < W; j++) x[j] = fma(-x[p], up[j], x[j]);
  }
#pragma unroll
  for (int j = 0; j < W; j++)
    if (j < k) X[i + (int64_t)j * ldx] = x[j];
}

// ---------------------------------------------------------------- U12 = L11^-1 A12
// Thread per column; x_i = fma(-l_ip, x_p, x_i) for p ascending (unit
// diagonal, no division).
__global__ void __launch_bounds__(128) trsm_llu_kernel(int k, int64_t m, const double* __restrict__ L, int64_t ldl,
                                                       double* __restrict__ X, int64_t ldx) {
  __shared__ __align__(16) double sL[W * S];   // sL[p*S + i] = l(i, p), i > p
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int i = idx % W, p = idx / W;
    sL[p * S + i] = (i > p && i < k) ? L[i + (int64_t)p * ldl] : 0.0;
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double* col = X + c * ldx;
  double x[W];
  if (k == W && ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0)) {
#pragma unroll
    for (int r = 0; r < W; r += 2) {
      double2 v = *reinterpret_cast<const double2*>(col + r);
      x[r] = v.x;
      x[r + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int r = 0; r < W; r++) x[r] = (r < k) ? col[r] : 0.0;
  }
#pragma unroll
  for (int p = 0; p < W; p++) {
    const double* lp = sL + p * S;
#pragma unroll
    for (int i = p + 1; i < W; i++) x[i] = fma(-lp[i], x[p], x[i]);
  }
  if (k == W && ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0)) {
#pragma unroll
    for (int r = 0; r < W; r += 2) *reinterpret_cast<double2*>(col + r) = make_double2(x[r], x[r + 1]);
  } else {
#pragma unroll
    for (int r = 0; r < W; r++)
      if (r < k) col[r] = x[r];
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
  leaf_lu_kernel<<<1, 256, 0, s>>>((int)n, A, lda, tau, info, koff);
  return cudaGetLastError();
}

cudaError_t launch_trsm_right_upper(int64_t m, int64_t k, double* X, int64_t ldx, const double* U, int64_t ldu,
                                    cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  trsm_ru_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(m, (int)k, X, ldx, U, ldu);
  return cudaGetLastError();
}

cudaError_t launch_trsm_left_lower_unit(int64_t k, int64_t m, const double* L, int64_t ldl, double* X,
                                        int64_t ldx, cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  trsm_llu_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>((int)k, m, L, ldl, X, ldx);
  return cudaGetLastError();
}

}  // namespace ebv
