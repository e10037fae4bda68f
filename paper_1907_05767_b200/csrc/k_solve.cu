// k_solve.cu — forward (LY = B) and backward (UX = Y) substitution, Eq 1
// ("UX = B" read as UX = Y, reading R6), as single-launch
// wavefront kernels.
//
// Canonical order (same as the oracle): forward y_i = fma chain over k
// ascending of (-l_ik y_k) starting from b_i; backward, k descending:
// x_k = y_k / u_kk, then y_i = fma(-u_ik, x_k, y_i) for i < k.
//
// Layout: rows are cut into blocks of BR = 64.  A CTA takes row blocks in
// wavefront order through an atomic ticket (so every block it waits on is
// already owned by a running CTA — no deadlock, any residency).  Thread
// (i, q) keeps the running value of row i for right-hand sides q, q+4, q+8,
// q+12 in registers and applies the off-diagonal tiles J < I (forward) or
// J > I (backward) in order as their finished y_J / x_J are published
// (release/acquire flags, L1-bypassing reads of the published values).  The
// 64 x 64 tiles of L / U are streamed through shared memory with cp.async
// double buffering (coalesced: a tile column is 512 contiguous bytes).  The
// diagonal block is then substituted by one warp per right-hand side, lane l
// owning rows l and l+32, with warp shuffles broadcasting y_k / x_k.
#include "ebv_internal.cuh"

namespace ebv {
namespace {

constexpr int BR = 64;          // rows per block
constexpr int QG = 4;           // rhs slots per thread group (threads = BR * QG)
constexpr int MAXR = 16;        // max rhs handled per launch
constexpr int TSTR = BR + 1;    // tile column stride (doubles) in smem
constexpr int THREADS = BR * QG;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// tile (rows of block I) x (columns of block J) of the packed LU -> smem
// st[c * TSTR + r] = LU(I*BR + r, J*BR + c)
__device__ __forceinline__ void load_tile(double* st, const double* LU, int64_t lda, int64_t n, int64_t I,
                                          int64_t J) {
  for (int idx = threadIdx.x; idx < BR * BR; idx += THREADS) {
    int r = idx % BR, c = idx / BR;
    int64_t row = I * BR + r, col = J * BR + c;
    bool p = row < n && col < n;
    cp_async8(st + c * TSTR + r, p ? LU + row + col * lda : LU, p);
  }
}

template <bool FORWARD>
__global__ void __launch_bounds__(THREADS) solve_kernel(int64_t n, const double* __restrict__ LU, int64_t lda,
                                                        double* B, int64_t ldb, int nrhs, int* ticket,
                                                        int* flags, int epoch) {
  extern __shared__ double sm[];
  double* tile[2] = {sm, sm + BR * TSTR};
  double* sy = sm + 2 * BR * TSTR;             // [BR][MAXR] published values of block J
  double* sacc = sy + BR * MAXR;               // [BR][MAXR] hand-off to the diagonal warps
  __shared__ int s_blk;
  const int64_t NB = (n + BR - 1) / BR;
  const int tid = threadIdx.x;
  const int i = tid % BR, q = tid / BR;
  const int lane = tid & 31, warp = tid >> 5;

  for (;;) {
    if (tid == 0) s_blk = atomicAdd(ticket, 1);
    __syncthreads();
    const int64_t t = s_blk;
    if (t >= NB) return;
    const int64_t I = FORWARD ? t : NB - 1 - t;
    const int64_t row = I * BR + i;
    const bool rv = row < n;

    double acc[MAXR / QG];
#pragma unroll
    for (int u = 0; u < MAXR / QG; u++) {
      int r = q + u * QG;
      acc[u] = (rv && r < nrhs) ? B[row + r * ldb] : 0.0;
    }

    // ---- off-diagonal tiles in canonical order
    const int64_t nJ = FORWARD ? I : NB - 1 - I;
    if (nJ > 0) {
      load_tile(tile[0], LU, lda, n, I, FORWARD ? 0 : NB - 1);
      cp_commit();
    }
    for (int64_t jj = 0; jj < nJ; jj++) {
      const int64_t J = FORWARD ? jj : NB - 1 - jj;
      if (jj + 1 < nJ) load_tile(tile[(jj + 1) & 1], LU, lda, n, I, FORWARD ? J + 1 : J - 1);
      cp_commit();
      if (tid == 0) {
        while (ld_acquire(flags + J) != epoch) __nanosleep(32);
      }
      __syncthreads();
      // published values of block J (L2-coherent reads)
      for (int idx = tid; idx < BR * nrhs; idx += THREADS) {
        int k = idx % BR, r = idx / BR;
        int64_t rowk = J * BR + k;
        sy[k * MAXR + r] = (rowk < n) ? __ldcg(B + rowk + r * ldb) : 0.0;
      }
      cp_wait1();
      __syncthreads();
      const double* st = tile[jj & 1];
      if (FORWARD) {
#pragma unroll 8
        for (int k = 0; k < BR; k++) {
          const double l = st[k * TSTR + i];
#pragma unroll
          for (int u = 0; u < MAXR / QG; u++) acc[u] = fma(-l, sy[k * MAXR + q + u * QG], acc[u]);
        }
      } else {
#pragma unroll 8
        for (int k = BR - 1; k >= 0; k--) {
          const double uu = st[k * TSTR + i];
#pragma unroll
          for (int u = 0; u < MAXR / QG; u++) acc[u] = fma(-uu, sy[k * MAXR + q + u * QG], acc[u]);
        }
      }
      __syncthreads();
    }
    cp_wait_all();

    // ---- diagonal block
    load_tile(tile[0], LU, lda, n, I, I);
    cp_commit();
#pragma unroll
    for (int u = 0; u < MAXR / QG; u++) {
      int r = q + u * QG;
      if (r < nrhs) sacc[i * MAXR + r] = acc[u];
    }
    cp_wait_all();
    __syncthreads();
    const double* st = tile[0];
    for (int r = warp; r < nrhs; r += THREADS / 32) {
      double v0 = sacc[lane * MAXR + r], v1 = sacc[(lane + 32) * MAXR + r];
      if (FORWARD) {
        // rows lane, lane+32; y_k final when reached; k ascending
#pragma unroll 4
        for (int k = 0; k < 32; k++) {
          double yk = __shfl_sync(0xffffffffu, v0, k);
          if (lane > k) v0 = fma(-st[k * TSTR + lane], yk, v0);
          v1 = fma(-st[k * TSTR + lane + 32], yk, v1);
        }
#pragma unroll 4
        for (int k = 32; k < BR; k++) {
          double yk = __shfl_sync(0xffffffffu, v1, k - 32);
          if (lane + 32 > k) v1 = fma(-st[k * TSTR + lane + 32], yk, v1);
        }
      } else {
        // k descending: x_k = y_k / u_kk, then rows above k are updated
#pragma unroll 4
        for (int k = BR - 1; k >= 32; k--) {
          const bool valid = I * BR + k < n;
          double xk = 0.0;
          if (lane == k - 32 && valid) v1 = v1 / st[k * TSTR + k];
          xk = __shfl_sync(0xffffffffu, v1, k - 32);
          if (valid) {
            if (lane + 32 < k) v1 = fma(-st[k * TSTR + lane + 32], xk, v1);
            v0 = fma(-st[k * TSTR + lane], xk, v0);
          }
        }
#pragma unroll 4
        for (int k = 31; k >= 0; k--) {
          const bool valid = I * BR + k < n;
          if (lane == k && valid) v0 = v0 / st[k * TSTR + k];
          double xk = __shfl_sync(0xffffffffu, v0, k);
          if (valid && lane < k) v0 = fma(-st[k * TSTR + lane], xk, v0);
        }
      }
      int64_t r0 = I * BR + lane, r1 = r0 + 32;
      if (r0 < n) B[r0 + r * ldb] = v0;
      if (r1 < n) B[r1 + r * ldb] = v1;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(flags + I, epoch);
  }
}

constexpr int SMEM = (2 * BR * TSTR + 2 * BR * MAXR) * 8;

}  // namespace

int64_t solve_block_rows() { return BR; }

cudaError_t launch_solve(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                         int* ticket_ws, int* flags_ws, int64_t epoch, cudaStream_t s) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(solve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(solve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t NB = (n + BR - 1) / BR;
  for (int64_t r0 = 0; r0 < nrhs; r0 += MAXR) {
    const int nr = (int)((nrhs - r0) < MAXR ? (nrhs - r0) : MAXR);
    for (int pass = 0; pass < 2; pass++) {
      const bool fwd = pass == 0;
      const int ep = (int)(((epoch * 64 + (r0 / MAXR) * 2 + pass) % 0x3FFFFFFF) + 1);
      cudaError_t e = cudaMemsetAsync(ticket_ws + pass, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
      int64_t grid = NB < (int64_t)sms * 2 ? NB : (int64_t)sms * 2;
      if (fwd)
        solve_kernel<true><<<(unsigned)grid, THREADS, SMEM, s>>>(n, LU, lda, B + r0 * ldb, ldb, nr, ticket_ws,
                                                                 flags_ws, ep);
      else
        solve_kernel<false><<<(unsigned)grid, THREADS, SMEM, s>>>(n, LU, lda, B + r0 * ldb, ldb, nr,
                                                                  ticket_ws + 1, flags_ws + NB, ep);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace ebv
