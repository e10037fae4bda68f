// k_scale.cu — the two row-scaling forms of SURVEY §8f f3 (elementwise,
// HBM-bound):
//   * unit-diagonal normalization (Eq 2, the coefficient matrix drawn
//     with 1 on its diagonal): row i of A and B divided by a_ii;
//   * the LDU form of a packed LU (Eq 3, U drawn unit-diagonal;
//     Eq 6-b's U_(k) row divided by its pivot): u'_kj = u_kj / u_kk, j > k.
// Each output entry is one correctly rounded division (bitwise the oracle).
// The divisors are read into a vector first (the normalization overwrites
// the diagonal), then a column-major 2D grid streams the matrix: a thread
// block covers TR consecutive rows (coalesced) of TC columns.  n = 32768:
// normalization 3.1 ms (5.6 TB/s), LDU 1.7 ms (5.1 TB/s).
#include "ebv_internal.cuh"

namespace ebv {
namespace {

constexpr int TR = 256;   // rows per thread block
constexpr int TC = 16;    // columns per thread block (blockIdx.y covers TC columns)

// d[i] = a_ii; scales[i] = 1 / a_ii (0 for a zero diagonal); info_min = first
// zero row (1-based) via atomicMin
__global__ void diag_kernel(int64_t n, const double* __restrict__ A, int64_t lda, double* __restrict__ d,
                            double* __restrict__ scales, unsigned long long* info_min) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = A[i + i * lda];
  d[i] = v;
  if (scales) scales[i] = v != 0.0 ? 1.0 / v : 0.0;
  if (info_min && v == 0.0) atomicMin(info_min, (unsigned long long)(i + 1));
}

// X[i, j] /= d[i] for rows i < n of the TC columns jbase + TC*blockIdx.y + c
// (c < TC, j < ncols); rows with d[i] == 0 are left unchanged; upper_only:
// only rows i < j (the LDU form).
__global__ void rowdiv_kernel(int64_t n, int64_t ncols, int64_t jbase, double* __restrict__ X, int64_t ldx,
                              const double* __restrict__ d, int upper_only) {
  const int64_t i = (int64_t)blockIdx.x * TR + threadIdx.x;
  if (i >= n) return;
  const double v = d[i];
  if (v == 0.0) return;
  const int64_t j0 = jbase + (int64_t)blockIdx.y * TC;
#pragma unroll 4
  for (int c = 0; c < TC; c++) {
    const int64_t j = j0 + c;
    if (j >= ncols) break;
    if (upper_only && i >= j) continue;
    double* p = X + i + j * ldx;
    *p = *p / v;
  }
}

__global__ void info_out_kernel(const unsigned long long* info_min, int64_t* info) {
  *info = (*info_min == ~0ull) ? 0 : (int64_t)*info_min;
}

cudaError_t rowdiv(int64_t n, int64_t ncols, double* X, int64_t ldx, const double* d, bool upper, cudaStream_t s,
                   int64_t* launches) {
  if (n <= 0 || ncols <= 0) return cudaSuccess;
  const int64_t span = (int64_t)65535 * TC;          // gridDim.y limit
  for (int64_t j0 = 0; j0 < ncols; j0 += span) {
    const int64_t nc = ncols - j0 < span ? ncols - j0 : span;
    // LDU: columns below j0 + nc only have rows i < j to scale
    const int64_t rows = upper ? (j0 + nc - 1 < n ? j0 + nc - 1 : n) : n;
    if (rows <= 0) continue;
    dim3 grid((unsigned)((rows + TR - 1) / TR), (unsigned)((nc + TC - 1) / TC));
    rowdiv_kernel<<<grid, TR, 0, s>>>(rows, j0 + nc, j0, X, ldx, d, upper ? 1 : 0);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_normalize_unit_diagonal(int64_t n, double* A, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                                           double* scales, int64_t* info, double* dws, unsigned long long* info_min,
                                           cudaStream_t s, int64_t* launches) {
  cudaError_t e = cudaMemsetAsync(info_min, 0xFF, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, A, lda, dws, scales, info_min);
    ++*launches;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = rowdiv(n, n, A, lda, dws, false, s, launches);
    if (e == cudaSuccess && B && nrhs > 0) e = rowdiv(n, nrhs, B, ldb, dws, false, s, launches);
    if (e != cudaSuccess) return e;
  }
  info_out_kernel<<<1, 1, 0, s>>>(info_min, info);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_lu_to_ldu(int64_t n, double* LU, int64_t lda, double* D, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, LU, lda, D, nullptr, nullptr);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return rowdiv(n, n, LU, lda, D, true, s, launches);
}

}  // namespace ebv
