// k_vector.cu — the paper's vector-level elimination (EBV_PATH_VECTOR):
// Eq 6-a..c executed step by step, with the EbV equal-length
// pairing (Eq 7) as the column -> CTA owner map.
//
// One persistent cooperative kernel.  CTA b owns the columns of the pairs
// p = b, b+C, b+2C, ... where pair p = {p, n-1-p} (first with last: the two
// columns' on-or-below-diagonal lengths sum to n+1, so every CTA holds the
// same number of matrix entries — reading R12), and keeps them resident in
// shared memory for the whole factorization.  Step k:
//   * the owner of column k has applied updates 0..k-1 to it; it divides the
//     sub-diagonal part by the pivot (Eq 6-a: the L_(k) vector), writes the
//     column to A (its final value) and publishes flag[k] (release);
//   * every CTA acquires flag[k], reads L_(k) from L2 and applies the rank-1
//     update a_ij = fma(-l_ik, u_kj, a_ij) (Eq 6-c, u_kj = its own row-k
//     entry, the U_(k) vector of Eq 6-b) to its owned columns j > k.
// Lookahead: the owner of column k+1 updates that column first and publishes
// L_(k+1) before touching its other columns, so the dependent chain per step
// is one column update + one division + one flag hop.
// Per entry the arithmetic is the oracle's (bitwise); `cyclic` selects the
// plain j mod C owner map for comparison.
#include <cooperative_groups.h>

#include "ebv_internal.cuh"

namespace ebv {
namespace {

constexpr int VT = 256;   // threads per CTA

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// relaxed polls (an acquire load costs an L1 invalidation per poll on
// sm_100a), then one acquire fence
__device__ __forceinline__ void wait_flag(const int* p, int v) {
  while (ld_relaxed(p) != v) __nanosleep(32);
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int owner_of(int j, int n, int C, int cyclic) {
  if (cyclic) return j % C;
  int p = j < n - 1 - j ? j : n - 1 - j;
  return p % C;
}

__global__ void __launch_bounds__(VT, 1)
    vector_lu_kernel(int n, double* __restrict__ A, int64_t lda, const double* __restrict__ tau,
                     unsigned long long* info_min, int* flags, int epoch, int cyclic, int maxcols) {
  extern __shared__ double sm[];
  const int C = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  double* sl = sm;                         // L_(k) of the current step (n)
  double* scol = sm + n;                   // owned columns [maxcols][n]
  __shared__ int cols[512];
  __shared__ int ncols_s;
  if (tid == 0) {
    int c = 0;
    for (int j = 0; j < n; j++)
      if (owner_of(j, n, C, cyclic) == b) cols[c++] = j;
    ncols_s = c;
  }
  __syncthreads();
  const int ncols = ncols_s;
  for (int c = 0; c < ncols; c++)
    for (int i = tid; i < n; i += VT) scol[c * n + i] = A[i + (int64_t)cols[c] * lda];
  __syncthreads();
  const double tv = *tau;

  // local slot of global column j, or -1
  auto slot_of = [&](int j) -> int {
    if (owner_of(j, n, C, cyclic) != b) return -1;
    int lo = 0, hi = ncols - 1;
    while (lo <= hi) {
      int mid = (lo + hi) >> 1;
      if (cols[mid] == j) return mid;
      if (cols[mid] < j) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
  };
  // Eq 6-a on an owned column + publish: the L_(k) vector becomes final
  auto publish = [&](int k, int c) {
    double* col = scol + c * n;
    const double piv = col[k];
    if (tid == 0 && fabs(piv) <= tv) atomicMin(info_min, (unsigned long long)(k + 1));
    for (int i = k + 1 + tid; i < n; i += VT) col[i] = col[i] / piv;
    __syncthreads();
    for (int i = tid; i < n; i += VT) A[i + (int64_t)k * lda] = col[i];
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(flags + k, epoch);
  };

  {
    int c0 = slot_of(0);
    if (c0 >= 0) publish(0, c0);
  }
  int first = 0;   // owned columns < first are finished (j <= k)
  for (int k = 0; k < n - 1; k++) {
    const int ck = slot_of(k);
    const double* l;
    if (ck >= 0) {
      l = scol + ck * n;            // the owner already holds L_(k)
    } else {
      if (tid == 0) wait_flag(flags + k, epoch);
      __syncthreads();
      for (int i = k + 1 + tid; i < n; i += VT) sl[i] = __ldcg(A + i + (int64_t)k * lda);
      __syncthreads();
      l = sl;
    }
    while (first < ncols && cols[first] <= k) first++;
    // lookahead: column k+1 first
    const int cn = slot_of(k + 1);
    if (cn >= 0) {
      double* col = scol + cn * n;
      const double u = col[k];
      for (int i = k + 1 + tid; i < n; i += VT) col[i] = fma(-l[i], u, col[i]);
      __syncthreads();
      publish(k + 1, cn);
    }
    // Eq 6-c on the remaining owned columns j > k+1
    for (int c = first; c < ncols; c++) {
      if (c == cn) continue;
      double* col = scol + c * n;
      const double u = col[k];
      for (int i = k + 1 + tid; i < n; i += VT) col[i] = fma(-l[i], u, col[i]);
    }
    __syncthreads();
  }
  for (int c = 0; c < ncols; c++)
    for (int i = tid; i < n; i += VT) A[i + (int64_t)cols[c] * lda] = scol[c * n + i];
}

__global__ void info_finalize_kernel(const unsigned long long* info_min, int64_t* info) {
  unsigned long long v = *info_min;
  *info = (v == ~0ull) ? 0 : (int64_t)v;
}

int max_cols(int64_t n, int C, int cyclic) {
  if (cyclic) return (int)((n + C - 1) / C);
  int64_t pairs = (n + 1) / 2;
  return (int)(2 * ((pairs + C - 1) / C));
}

}  // namespace

size_t vector_smem_bytes(int64_t n, int num_ctas) {
  const int cyclic = num_ctas < 0 ? 1 : 0;
  int C = num_ctas < 0 ? -num_ctas : num_ctas;
  if (C > (n + 1) / 2 && !cyclic) C = (int)((n + 1) / 2);
  if (C > n) C = (int)n;
  if (C < 1) C = 1;
  return ((size_t)max_cols(n, C, cyclic) * n + n) * 8;
}

int vector_max_ctas(int device, int64_t n) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  // prefer a CTA count dividing the number of pairs (even per-step balance),
  // capped by one CTA per SM (cooperative residency)
  int64_t pairs = (n + 1) / 2;
  int best = sms < pairs ? sms : (int)pairs;
  for (int c = best; c >= best * 3 / 4 && c >= 1; c--)
    if (pairs % c == 0) return c;
  return best < 1 ? 1 : best;
}

cudaError_t launch_vector_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info, int* flags_ws,
                             double* lbuf_ws, int num_ctas, cudaStream_t s) {
  // lbuf_ws is used as the 8-byte info accumulator (min over failing steps)
  unsigned long long* info_min = reinterpret_cast<unsigned long long*>(lbuf_ws);
  cudaError_t e = cudaMemsetAsync(info_min, 0xFF, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (n <= 0) {
    info_finalize_kernel<<<1, 1, 0, s>>>(info_min, info);
    return cudaGetLastError();
  }
  const int cyclic = num_ctas < 0 ? 1 : 0;
  int C = num_ctas < 0 ? -num_ctas : num_ctas;
  if (C > (n + 1) / 2 && !cyclic) C = (int)((n + 1) / 2);
  if (C > n) C = (int)n;
  const int mc = max_cols(n, C, cyclic);
  if (mc > 512) return cudaErrorInvalidValue;
  const size_t smem = ((size_t)mc * n + n) * 8;
  e = cudaFuncSetAttribute(vector_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  static int epoch = 0;
  epoch = (epoch % 0x3FFFFFF0) + 1;
  int nn = (int)n;
  int ep = epoch;
  void* args[] = {&nn, &A, &lda, (void*)&tau, &info_min, &flags_ws, &ep, (void*)&cyclic, (void*)&mc};
  e = cudaLaunchCooperativeKernel((void*)vector_lu_kernel, dim3(C), dim3(VT), args, smem, s);
  if (e != cudaSuccess) return e;
  info_finalize_kernel<<<1, 1, 0, s>>>(info_min, info);
  return cudaGetLastError();
}

}  // namespace ebv
