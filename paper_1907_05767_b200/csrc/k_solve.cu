// k_solve.cu — forward (LY = B) and backward (UX = Y) substitution, Eq 1
// ("UX = B" read as UX = Y, reading R6), as single-launch
// wavefront kernels.
//
// Canonical order (same as the oracle): forward y_i = fma chain over k
// ascending of (-l_ik y_k) starting from b_i; backward, k descending:
// x_k = y_k / u_kk, then y_i = fma(-u_ik, x_k, y_i) for i < k.
//
// Layout: rows are cut into blocks of BR = 64; one CTA of 64 threads per row
// block, thread i owning row i (its running values for up to 16 right-hand
// sides in registers).  CTAs take blocks in wavefront order through an atomic
// ticket (every block a CTA waits on is owned by a CTA that is already
// running: no deadlock at any residency), and the CTAs are small enough that
// all blocks of an n = 32768 system are resident at once, so every block
// streams its part of L (U) as soon as the values it needs are published.
// Off-diagonal tile (I, J): thread i loads its 64 entries of row i straight
// into registers (a warp reads 32 consecutive rows = 256 contiguous bytes per
// column), waits for block J's release flag, reads y_J (L2-coherent loads)
// and applies the 64 updates in canonical order.  The diagonal block (staged
// in shared memory when the block starts) is then substituted by one warp per
// right-hand side, lane l owning rows l and l+32, shuffles broadcasting
// y_k / x_k; the block's values are stored and its flag released.
#include "ebv_internal.cuh"

namespace ebv {
namespace {

constexpr int BR = 64;          // rows per block (= threads per CTA)
constexpr int MAXR = 16;        // max right-hand sides per launch
constexpr int TSTR = BR + 1;    // diagonal tile column stride in smem

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <bool FORWARD, int NR>
__global__ void __launch_bounds__(BR) solve_kernel(int64_t n, const double* __restrict__ LU, int64_t lda,
                                                   double* B, int64_t ldb, int nrhs, int* ticket, int* flags,
                                                   int epoch) {
  __shared__ double sd[BR * TSTR];          // diagonal tile: sd[c*TSTR + r] = LU(I*BR + r, I*BR + c)
  __shared__ double sbuf[BR * MAXR];        // published values of block J (sy[k*MAXR + r]),
  double* sy = sbuf;                        // then the hand-off to the diagonal warps (sacc)
  double* sacc = sbuf;
  __shared__ int s_blk;
  const int64_t NB = (n + BR - 1) / BR;
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  const int nr = NR > 0 ? NR : nrhs;

  for (;;) {
    if (i == 0) s_blk = atomicAdd(ticket, 1);
    __syncthreads();
    const int64_t t = s_blk;
    __syncthreads();
    if (t >= NB) return;
    const int64_t I = FORWARD ? t : NB - 1 - t;
    const int64_t row = I * BR + i;
    const bool rv = row < n;

    // stage the diagonal tile (read-only: no dependence on other blocks)
    for (int c = 0; c < BR; c++) {
      const int64_t col = I * BR + c;
      sd[c * TSTR + i] = (rv && col < n) ? LU[row + col * lda] : 0.0;
    }
    double acc[MAXR];
#pragma unroll
    for (int r = 0; r < MAXR; r++) acc[r] = (rv && r < nr) ? B[row + (int64_t)r * ldb] : 0.0;

    const int64_t nJ = FORWARD ? I : NB - 1 - I;
    for (int64_t jj = 0; jj < nJ; jj++) {
      const int64_t J = FORWARD ? jj : NB - 1 - jj;
      // this thread's row segment of tile (I, J): issued before the wait
      double l[BR];
      const double* src = LU + (rv ? row : 0) + (J * BR) * lda;
#pragma unroll
      for (int k = 0; k < BR; k++) l[k] = (rv && J * BR + k < n) ? __ldg(src + k * lda) : 0.0;
      if (i == 0) {
        while (ld_acquire(flags + J) != epoch) __nanosleep(20);
      }
      __syncthreads();
      for (int idx = i; idx < BR * nr; idx += BR) {
        const int k = idx % BR, r = idx / BR;
        const int64_t rk = J * BR + k;
        sy[k * MAXR + r] = (rk < n) ? __ldcg(B + rk + (int64_t)r * ldb) : 0.0;
      }
      __syncthreads();
      if (FORWARD) {
#pragma unroll
        for (int k = 0; k < BR; k++)
#pragma unroll
          for (int r = 0; r < MAXR; r++)
            if (r < nr) acc[r] = fma(-l[k], sy[k * MAXR + r], acc[r]);
      } else {
#pragma unroll
        for (int k = BR - 1; k >= 0; k--)
#pragma unroll
          for (int r = 0; r < MAXR; r++)
            if (r < nr) acc[r] = fma(-l[k], sy[k * MAXR + r], acc[r]);
      }
    }

    // ---- diagonal block
    __syncthreads();   // sy (aliased by sacc) is no longer read
#pragma unroll
    for (int r = 0; r < MAXR; r++)
      if (r < nr) sacc[i * MAXR + r] = acc[r];
    __syncthreads();
    const double* st = sd;
    for (int r = warp; r < nr; r += BR / 32) {
      double v0 = sacc[lane * MAXR + r], v1 = sacc[(lane + 32) * MAXR + r];
      if (FORWARD) {
        // rows lane, lane+32; y_k final when reached; k ascending
#pragma unroll 8
        for (int k = 0; k < 32; k++) {
          const double yk = __shfl_sync(0xffffffffu, v0, k);
          if (lane > k) v0 = fma(-st[k * TSTR + lane], yk, v0);
          v1 = fma(-st[k * TSTR + lane + 32], yk, v1);
        }
#pragma unroll 8
        for (int k = 32; k < BR; k++) {
          const double yk = __shfl_sync(0xffffffffu, v1, k - 32);
          if (lane + 32 > k) v1 = fma(-st[k * TSTR + lane + 32], yk, v1);
        }
      } else {
        // k descending: x_k = y_k / u_kk, then rows above k are updated
#pragma unroll 8
        for (int k = BR - 1; k >= 32; k--) {
          const bool valid = I * BR + k < n;
          if (lane == k - 32 && valid) v1 = v1 / st[k * TSTR + k];
          const double xk = __shfl_sync(0xffffffffu, v1, k - 32);
          if (valid) {
            if (lane + 32 < k) v1 = fma(-st[k * TSTR + lane + 32], xk, v1);
            v0 = fma(-st[k * TSTR + lane], xk, v0);
          }
        }
#pragma unroll 8
        for (int k = 31; k >= 0; k--) {
          const bool valid = I * BR + k < n;
          if (lane == k && valid) v0 = v0 / st[k * TSTR + k];
          const double xk = __shfl_sync(0xffffffffu, v0, k);
          if (valid && lane < k) v0 = fma(-st[k * TSTR + lane], xk, v0);
        }
      }
      const int64_t r0 = I * BR + lane, r1 = r0 + 32;
      if (r0 < n) B[r0 + (int64_t)r * ldb] = v0;
      if (r1 < n) B[r1 + (int64_t)r * ldb] = v1;
    }
    __threadfence();
    __syncthreads();
    if (i == 0) st_release(flags + I, epoch);
  }
}

template <bool FWD>
cudaError_t launch_one(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int nr, int* ticket,
                       int* flags, int ep, int64_t grid, cudaStream_t s) {
  if (nr == 1)
    solve_kernel<FWD, 1><<<(unsigned)grid, BR, 0, s>>>(n, LU, lda, B, ldb, nr, ticket, flags, ep);
  else
    solve_kernel<FWD, 0><<<(unsigned)grid, BR, 0, s>>>(n, LU, lda, B, ldb, nr, ticket, flags, ep);
  return cudaGetLastError();
}

}  // namespace

int64_t solve_block_rows() { return BR; }

cudaError_t launch_solve(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                         int* ticket_ws, int* flags_ws, int64_t epoch, cudaStream_t s) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  int dev = 0, sms = 148, per_sm = 8;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<true, 0>, BR, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t NB = (n + BR - 1) / BR;
  const int64_t cap = (int64_t)sms * per_sm;
  const int64_t grid = NB < cap ? NB : cap;
  for (int64_t r0 = 0; r0 < nrhs; r0 += MAXR) {
    const int nr = (int)((nrhs - r0) < MAXR ? (nrhs - r0) : MAXR);
    for (int pass = 0; pass < 2; pass++) {
      const bool fwd = pass == 0;
      const int ep = (int)(((epoch * 64 + (r0 / MAXR) * 2 + pass) % 0x3FFFFFFF) + 1);
      cudaError_t e = cudaMemsetAsync(ticket_ws + pass, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
      e = fwd ? launch_one<true>(n, LU, lda, B + r0 * ldb, ldb, nr, ticket_ws, flags_ws, ep, grid, s)
              : launch_one<false>(n, LU, lda, B + r0 * ldb, ldb, nr, ticket_ws + 1, flags_ws + NB, ep, grid, s);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace ebv
