// k_util.cu — small device utilities of the dispatch layer: info reset and
// the default pivot floor tau = n * DBL_EPSILON * ||A||_inf (reading R9).
#include "ebv_internal.cuh"

#include <mutex>
#include <set>
#include <utility>

namespace ebv {
namespace {

__global__ void set_info0_kernel(int64_t* info) { *info = 0; }

// row absolute sums (thread per row, coalesced over a column) -> max via
// atomicMax on the IEEE bits (non-negative doubles order like uint64)
__global__ void norm_inf_kernel(int64_t n, const double* __restrict__ A, int64_t lda, unsigned long long* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t j = 0; j < n; j++) s += fabs(A[i + j * lda]);
  atomicMax(out, (unsigned long long)__double_as_longlong(s));
}

__global__ void tau_kernel(int64_t n, const unsigned long long* nrm, double* tau_out) {
  *tau_out = (double)n * 2.220446049250313e-16 * __longlong_as_double((long long)*nrm);
}

__global__ void set_tau_kernel(double tau, double* tau_out) { *tau_out = tau; }

// batched medium systems: per system the pivot floor (tau >= 0 as given, or
// n * eps * ||A_s||_inf — the row sums accumulated over j ascending like
// norm_inf_kernel), info words cleared
__global__ void batched_prep_kernel(int64_t n, const double* __restrict__ A, int64_t lda, int64_t sA, double tau,
                                    double* tau_s, int64_t* info64) {
  const int64_t sys = blockIdx.x;
  __shared__ double red[256];
  double m = 0.0;
  if (tau < 0.0) {
    const double* As = A + sys * sA;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      double r = 0.0;
      for (int64_t j = 0; j < n; j++) r += fabs(As[i + j * lda]);
      m = fmax(m, r);
    }
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tau_s[sys] = tau < 0.0 ? (double)n * 2.220446049250313e-16 * red[0] : tau;
    info64[sys] = 0;
  }
}

// distributed default floor: partial row absolute sums over a rank's local
// columns (j ascending), accumulated into rs (first: overwrite)
__global__ void rowabs_kernel(int64_t n, const double* __restrict__ A, int64_t lda, int64_t cols, double* rs,
                              bool first) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = first ? 0.0 : rs[i];
  for (int64_t j = 0; j < cols; j++) s += fabs(A[i + j * lda]);
  rs[i] = s;
}

__global__ void tau_from_rows_kernel(int64_t n, const double* __restrict__ rs, double* tau_out) {
  __shared__ double red[1024];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, rs[i]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *tau_out = (double)n * 2.220446049250313e-16 * red[0];
}

__global__ void info_to_i32_kernel(int64_t batch, const int64_t* info64, int32_t* info32) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < batch) info32[s] = (int32_t)info64[s];
}

}  // namespace

cudaError_t launch_batched_prep(int64_t n, const double* A, int64_t lda, int64_t sA, int64_t batch, double tau,
                                double* tau_s, int64_t* info64, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  batched_prep_kernel<<<(unsigned)batch, 256, 0, s>>>(n, A, lda, sA, tau, tau_s, info64);
  return cudaGetLastError();
}

cudaError_t launch_info_to_i32(int64_t batch, const int64_t* info64, int32_t* info32, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  info_to_i32_kernel<<<(unsigned)((batch + 255) / 256), 256, 0, s>>>(batch, info64, info32);
  return cudaGetLastError();
}

cudaError_t launch_rowabs(int64_t n, const double* A, int64_t lda, int64_t cols, double* rs, bool first,
                          cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  rowabs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, A, lda, cols, rs, first);
  return cudaGetLastError();
}

cudaError_t launch_tau_from_rows(int64_t n, const double* rs, double* tau_out, cudaStream_t s) {
  tau_from_rows_kernel<<<1, 1024, 0, s>>>(n, rs, tau_out);
  return cudaGetLastError();
}

cudaError_t launch_set_info0(int64_t* info, cudaStream_t s) {
  set_info0_kernel<<<1, 1, 0, s>>>(info);
  return cudaGetLastError();
}

cudaError_t launch_tau(int64_t n, const double* A, int64_t lda, double tau, double* tau_out,
                       unsigned long long* norm_ws, cudaStream_t s) {
  if (tau >= 0.0 || n <= 0) {
    set_tau_kernel<<<1, 1, 0, s>>>(tau >= 0.0 ? tau : 0.0, tau_out);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(norm_ws, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  norm_inf_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, A, lda, norm_ws);
  tau_kernel<<<1, 1, 0, s>>>(n, norm_ws, tau_out);
  return cudaGetLastError();
}

cudaError_t ensure_max_dyn_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({fn, dev});
  return e;
}

}  // namespace ebv
