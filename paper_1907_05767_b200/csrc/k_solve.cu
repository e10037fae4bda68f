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
#include "ebv_device.cuh"

namespace ebv {
namespace {

constexpr int BR = 64;          // rows per block (= threads per CTA)
constexpr int MAXR = 16;        // max right-hand sides per launch
constexpr int TSTR = BR + 1;    // diagonal tile column stride in smem
constexpr int kMaxInterleave = 64;   // single-column chains per launch (flags: 2 * 64 * NB)

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait for a release flag: relaxed polls (no L1 invalidation per poll, which
// an acquire load costs on sm_100a: CCTL.IVALL) with a short back-off, then
// one acquire fence that orders the subsequent reads after the observed
// release.
__device__ __forceinline__ void wait_flag(const int* p, int v, bool next_in_chain) {
  // only the block whose diagonal depends on this flag polls tightly; the
  // others (accumulating further tiles) back off, keeping the flag's L2
  // slice free for the release store on the critical path
  const unsigned ns = next_in_chain ? 32 : 1000;
  dev::SpinGuard g;
  while (ld_relaxed(p) != v) {
    __nanosleep(ns);
    g.poll();
  }
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

#ifdef EBV_SOLVE_TRACE
// probes/solve_trace.cu: per-block phase timestamps (%globaltimer, ns)
__device__ unsigned long long g_trace[2][8192][6];
__device__ int g_redo;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define EBV_TR(slot)                                                     \
  do {                                                                   \
    if (i == 0 && I < 8192) g_trace[FORWARD ? 0 : 1][I][slot] = gtime(); \
  } while (0)
#else
#define EBV_TR(slot) \
  do {               \
  } while (0)
#endif

// y / u from a precomputed reciprocal r = RN(1/u): the Markstein step
// (dev::quot_mk, three dependent FP64 ops on the chain instead of a full
// division); the owner lane keeps its step's dividend and quotient and the
// exact test (dev::quot_is_rn) runs after the block's sweep, off the step
// chain; a block with an unverified quotient is redone with true division,
// so the result is always RN(y/u), bitwise the oracle's division.
__device__ __forceinline__ double quot_nc(double y, double u, double r) { return dev::quot_mk(y, u, r); }
__device__ __forceinline__ bool quot_chk(double y, double u, double q) { return dev::quot_is_rn(y, u, q); }

// Window form (the multi-GPU ring solve, ebv_dist.cu): only the column
// blocks [jlo, jhi) (units of BR) take part, addressed as
// LU[row + (col - cbase) * lda]; forward, row blocks I >= jlo are processed
// (I < jhi: substituted and released; below: only updated by the window's
// columns); backward, row blocks I < jhi (I >= jlo substituted; above: only
// updated).  The full solve is the window [0, NB) with cbase = 0.
template <bool FORWARD, int NR>
__global__ void __launch_bounds__(BR) solve_kernel(int64_t n, const double* __restrict__ LU, int64_t lda,
                                                   double* B0, int64_t ldb, int nrhs, int* ticket, int* flags0,
                                                   int epoch, int64_t jlo, int64_t jhi, int64_t cbase, int nind,
                                                   int64_t kl, int64_t ku) {
  __shared__ double sd[BR * TSTR];          // diagonal tile: sd[c*TSTR + r] = LU(I*BR + r, I*BR + c)
  constexpr int SR = NR > 0 ? NR : MAXR;    // shared stride per row (right-hand sides)
  __shared__ double sbuf[BR * SR];          // published values of block J (sy[k*SR + r]),
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
    // nind > 1 (NR = 1): nind single-column solves interleaved in ticket
    // order — ticket t is column t % nind, block t / nind — so each column's
    // chain runs alongside the others' (a block waits only on blocks of its
    // own column with smaller tickets: no deadlock at any residency)
    if (t >= (FORWARD ? NB - jlo : jhi) * nind) return;
    const int rr = (int)(t % nind);
    const int64_t tq = t / nind;
    double* B = B0 + (int64_t)rr * ldb;
    int* flags = flags0 + (int64_t)rr * NB;
    const int64_t I = FORWARD ? jlo + tq : jhi - 1 - tq;
    const bool diag = I >= jlo && I < jhi;
    const int64_t row = I * BR + i;
    const bool rv = row < n;
    EBV_TR(0);

    // stage the diagonal tile (read-only: no dependence on other blocks)
    if (diag)
      for (int c = 0; c < BR; c++) {
        const int64_t col = I * BR + c;
        sd[c * TSTR + i] = (rv && col < n) ? LU[row + (col - cbase) * lda] : 0.0;
      }
    double acc[MAXR];
#pragma unroll
    for (int r = 0; r < MAXR; r++) acc[r] = (rv && r < nr) ? B[row + (int64_t)r * ldb] : 0.0;

    // banded factors (kl / ku): tiles outside the band are exact zeros and
    // are skipped (fma(-0, y, acc) == acc)
    int64_t jf = jlo, jt = jhi;
    if (FORWARD && I * BR > kl) jf = (I * BR - kl) / BR > jlo ? (I * BR - kl) / BR : jlo;
    if (!FORWARD) {
      const int64_t top = (I * BR + BR - 1 + ku) / BR + 1;
      jt = top < jhi ? top : jhi;
    }
    int64_t nJ = FORWARD ? (I < jhi ? I : jhi) - jf : jt - (I + 1 > jlo ? I + 1 : jlo);
    if (nJ < 0) nJ = 0;
    for (int64_t jj = 0; jj < nJ; jj++) {
      const int64_t J = FORWARD ? jf + jj : jt - 1 - jj;
      // this thread's row segment of tile (I, J): issued before the wait
      double l[BR];
      const double* src = LU + (rv ? row : 0) + (J * BR - cbase) * lda;
#pragma unroll
      for (int k = 0; k < BR; k++) l[k] = (rv && J * BR + k < n) ? __ldg(src + k * lda) : 0.0;
      if (jj + 1 == nJ) {
        EBV_TR(1);
      }
      if (i == 0) wait_flag(flags + J, epoch, diag && jj + 1 == nJ);
      if (jj + 1 == nJ) {
        EBV_TR(2);
      }
      __syncthreads();
      for (int idx = i; idx < BR * nr; idx += BR) {
        const int k = idx % BR, r = idx / BR;
        const int64_t rk = J * BR + k;
        sy[k * SR + r] = (rk < n) ? __ldcg(B + rk + (int64_t)r * ldb) : 0.0;
      }
      __syncthreads();
      if (FORWARD) {
#pragma unroll
        for (int k = 0; k < BR; k++)
#pragma unroll
          for (int r = 0; r < MAXR; r++)
            if (r < nr) acc[r] = fma(-l[k], sy[k * SR + r], acc[r]);
      } else {
#pragma unroll
        for (int k = BR - 1; k >= 0; k--)
#pragma unroll
          for (int r = 0; r < MAXR; r++)
            if (r < nr) acc[r] = fma(-l[k], sy[k * SR + r], acc[r]);
      }
    }

    if (!diag) {   // outside the window's rows: only the window's updates
#pragma unroll
      for (int r = 0; r < MAXR; r++)
        if (rv && r < nr) B[row + (int64_t)r * ldb] = acc[r];
      __syncthreads();   // sy is re-staged by the next block
      continue;
    }

    // ---- diagonal block: warp w takes right-hand sides r = w, w+2, ...
    // (up to HR = MAXR/2 of them, carried through the same step loop as
    // independent chains); lane l owns rows l and l+32.  Every lane evaluates
    // the step's division (uniform, no divergence) and the owner's quotient
    // is broadcast by shuffle; per entry the operations are the oracle's.
    __syncthreads();   // sy (aliased by sacc) is no longer read
    EBV_TR(3);
#pragma unroll
    for (int r = 0; r < MAXR; r++)
      if (r < nr) sacc[i * SR + r] = acc[r];
    __syncthreads();
    {
      constexpr int HR = MAXR / 2;
      const int nw = (nr + 1) / 2 > 0 ? 2 : 1;
      const int myr = (nr - warp + 1) / 2;          // rhs handled by this warp
      if (myr > 0) {
      const double* st = sd;
      const int nv = (int)((n - I * BR) < BR ? (n - I * BR) : BR);   // valid rows of the block
      double v0[HR], v1[HR];
#pragma unroll
      for (int q = 0; q < HR; q++) {
        const int r = warp + 2 * q;
        v0[q] = (q < myr) ? sacc[lane * SR + r] : 0.0;
        v1[q] = (q < myr) ? sacc[(lane + 32) * SR + r] : 0.0;
      }
      (void)nw;
      if (FORWARD) {
#pragma unroll 4
        for (int k = 0; k < 32; k++) {
          const double l0 = st[k * TSTR + lane], l1 = st[k * TSTR + lane + 32];
          const bool b0 = lane > k;
#pragma unroll
          for (int q = 0; q < HR; q++) {
            if (NR == 1 && q > 0) break;
            const double yk = __shfl_sync(0xffffffffu, v0[q], k);
            const double t0 = fma(-l0, yk, v0[q]);
            v0[q] = b0 ? t0 : v0[q];
            v1[q] = fma(-l1, yk, v1[q]);
          }
        }
#pragma unroll 4
        for (int k = 32; k < BR; k++) {
          const double l1 = st[k * TSTR + lane + 32];
          const bool b1 = lane + 32 > k;
#pragma unroll
          for (int q = 0; q < HR; q++) {
            if (NR == 1 && q > 0) break;
            const double yk = __shfl_sync(0xffffffffu, v1[q], k - 32);
            const double t1 = fma(-l1, yk, v1[q]);
            v1[q] = b1 ? t1 : v1[q];
          }
        }
      } else {
        // k descending; steps k >= nv (padding rows of the last block) are
        // skipped.  Fast pass with hoisted reciprocals (verified); if any
        // quotient is unverified the block is redone with true division.
        double rc0 = 1.0 / st[lane * TSTR + lane], rc1 = 1.0 / st[(lane + 32) * TSTR + lane + 32];
        double w0[HR], w1[HR];
#pragma unroll
        for (int q = 0; q < HR; q++) { w0[q] = v0[q]; w1[q] = v1[q]; }
        double yo0[HR], qo0[HR], yo1[HR], qo1[HR];   // the owned steps' dividends / quotients
#pragma unroll
        for (int q = 0; q < HR; q++) { yo0[q] = 0.0; qo0[q] = 0.0; yo1[q] = 0.0; qo1[q] = 0.0; }
        for (int k = BR - 1; k >= 32; k--) {
          if (k >= nv) continue;
          const double ukk = st[k * TSTR + k];
          const double rk = __shfl_sync(0xffffffffu, rc1, k - 32);
          const double u0 = st[k * TSTR + lane], u1 = st[k * TSTR + lane + 32];
          const bool own = lane == k - 32, b1 = lane + 32 < k;
#pragma unroll
          for (int q = 0; q < HR; q++) {
            if (NR == 1 && q > 0) break;
            const double qv = quot_nc(v1[q], ukk, rk);
            if (own) { yo1[q] = v1[q]; qo1[q] = qv; }
            const double xk = __shfl_sync(0xffffffffu, qv, k - 32);
            v1[q] = own ? xk : (b1 ? fma(-u1, xk, v1[q]) : v1[q]);
            v0[q] = fma(-u0, xk, v0[q]);
          }
        }
        for (int k = 31; k >= 0; k--) {
          if (k >= nv) continue;
          const double ukk = st[k * TSTR + k];
          const double rk = __shfl_sync(0xffffffffu, rc0, k);
          const double u0 = st[k * TSTR + lane];
          const bool own = lane == k, b0 = lane < k;
#pragma unroll
          for (int q = 0; q < HR; q++) {
            if (NR == 1 && q > 0) break;
            const double qv = quot_nc(v0[q], ukk, rk);
            if (own) { yo0[q] = v0[q]; qo0[q] = qv; }
            const double xk = __shfl_sync(0xffffffffu, qv, k);
            v0[q] = own ? xk : (b0 ? fma(-u0, xk, v0[q]) : v0[q]);
          }
        }
        bool ok = true;
        {
          const double d0 = st[lane * TSTR + lane], d1 = st[(lane + 32) * TSTR + lane + 32];
#pragma unroll
          for (int q = 0; q < HR; q++) {
            if (NR == 1 && q > 0) break;
            if (q < myr) ok = ok && quot_chk(yo0[q], d0, qo0[q]) && quot_chk(yo1[q], d1, qo1[q]);
          }
        }
        // any unverified quotient (checked by its owner lane) -> redo the
        // block with true division
        if (__any_sync(0xffffffffu, !ok)) {
#ifdef EBV_SOLVE_TRACE
          if (lane == 0) atomicAdd(&g_redo, 1);
#endif
#pragma unroll
          for (int q = 0; q < HR; q++) { v0[q] = w0[q]; v1[q] = w1[q]; }
          for (int k = BR - 1; k >= 32; k--) {
            if (k >= nv) continue;
            const double ukk = st[k * TSTR + k];
            const double u0 = st[k * TSTR + lane], u1 = st[k * TSTR + lane + 32];
            const bool own = lane == k - 32, b1 = lane + 32 < k;
#pragma unroll
            for (int q = 0; q < HR; q++) {
              if (NR == 1 && q > 0) break;
              const double xk = __shfl_sync(0xffffffffu, v1[q] / ukk, k - 32);
              v1[q] = own ? xk : (b1 ? fma(-u1, xk, v1[q]) : v1[q]);
              v0[q] = fma(-u0, xk, v0[q]);
            }
          }
          for (int k = 31; k >= 0; k--) {
            if (k >= nv) continue;
            const double ukk = st[k * TSTR + k];
            const double u0 = st[k * TSTR + lane];
            const bool own = lane == k, b0 = lane < k;
#pragma unroll
            for (int q = 0; q < HR; q++) {
              if (NR == 1 && q > 0) break;
              const double xk = __shfl_sync(0xffffffffu, v0[q] / ukk, k);
              v0[q] = own ? xk : (b0 ? fma(-u0, xk, v0[q]) : v0[q]);
            }
          }
        }
      }
      const int64_t r0 = I * BR + lane, r1 = r0 + 32;
#pragma unroll
      for (int q = 0; q < HR; q++) {
        if (q < myr) {
          const int r = warp + 2 * q;
          if (r0 < n) B[r0 + (int64_t)r * ldb] = v0[q];
          if (r1 < n) B[r1 + (int64_t)r * ldb] = v1[q];
        }
      }
      }   // myr > 0
    }
    // every thread's stores of this block precede thread 0's release (bar.sync
    // orders them at CTA scope; the gpu-scope release is cumulative)
    __syncthreads();
    EBV_TR(4);
    if (i == 0) {
      dev::jitter((unsigned)I);
      st_release(flags + I, epoch);
    }
    EBV_TR(5);
  }
}

template <class K>
int64_t resident_grid(int64_t units, K kern) {
  int dev = 0, sms = 148, per_sm = 8;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BR, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)sms * per_sm;
  return units < cap ? units : cap;
}

// nind independent single columns interleaved (the kernel's NR = 1 form; the
// several-columns-per-warp form, NR = 0, is kept in the source but no
// longer launched: interleaved chains were 4x faster at 16 columns)
template <bool FWD>
cudaError_t launch_one(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int nr, int* ticket,
                       int* flags, int ep, int64_t units, cudaStream_t s, int64_t jlo, int64_t jhi, int64_t cbase,
                       int nind, int64_t kl = -1, int64_t ku = -1) {
  if (nr != 1) return cudaErrorInvalidValue;
  if (kl < 0) kl = n;
  if (ku < 0) ku = n;
  const int64_t grid = resident_grid(units * nind, solve_kernel<FWD, 1>);
  solve_kernel<FWD, 1><<<(unsigned)grid, BR, 0, s>>>(n, LU, lda, B, ldb, nr, ticket, flags, ep, jlo, jhi, cbase,
                                                     nind, kl, ku);
  return cudaGetLastError();
}

}  // namespace

int64_t solve_block_rows() { return BR; }

cudaError_t launch_solve(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                         int* ticket_ws, int* flags_ws, int64_t epoch, cudaStream_t s, int64_t kl, int64_t ku) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int64_t NB = (n + BR - 1) / BR;
  // the columns as interleaved single-column chains, up to kMaxInterleave
  // per launch (flags: nind * NB per sweep): they run side by side instead of
  // sharing two warps of one CTA per row block
  for (int64_t g0 = 0; g0 < nrhs; g0 += kMaxInterleave) {
    const int nind = (int)((nrhs - g0) < kMaxInterleave ? (nrhs - g0) : kMaxInterleave);
    for (int pass = 0; pass < 2; pass++) {
      const bool fwd = pass == 0;
      // epochs base+1 .. base+2*groups: one per (group, sweep) launch, so no
      // two launches of this or any later call share one (the caller advances
      // its counter by launch_solve_epochs(nrhs) after the call)
      const int ep = (int)(((epoch + (g0 / kMaxInterleave) * 2 + pass) % 0x3FFFFFF0) + 1);
      cudaError_t e = cudaMemsetAsync(ticket_ws + pass, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
      e = fwd ? launch_one<true>(n, LU, lda, B + g0 * ldb, ldb, 1, ticket_ws, flags_ws, ep, NB, s, 0, NB, 0, nind, kl,
                                 ku)
              : launch_one<false>(n, LU, lda, B + g0 * ldb, ldb, 1, ticket_ws + 1, flags_ws + (int64_t)nind * NB, ep,
                                  NB, s, 0, NB, 0, nind, kl, ku);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

// One column window of the ring solve: forward (fwd) or backward sweep of
// the columns [c0, c0 + w) (c0 a multiple of BR) whose entries are at
// LUw[row + (col - c0) * ldl]; nrhs <= kMaxInterleave right-hand sides as
// interleaved single-column chains.  ticket: one zeroed int for this launch;
// flags: the sweep's nrhs * NB flags (released once per sweep by the block
// that substitutes them, so one epoch serves the whole sweep).
cudaError_t launch_solve_window(int64_t n, const double* LUw, int64_t ldl, int64_t c0, int64_t w, bool fwd, double* B,
                                int64_t ldb, int64_t nrhs, int* ticket, int* flags, int epoch, cudaStream_t s) {
  if (n <= 0 || nrhs <= 0 || w <= 0) return cudaSuccess;
  if (nrhs > kMaxInterleave || c0 % BR) return cudaErrorInvalidValue;
  const int64_t NB = (n + BR - 1) / BR;
  const int64_t jlo = c0 / BR, jhi = (c0 + w + BR - 1) / BR;
  const int64_t units = fwd ? NB - jlo : jhi;
  const int nind = (int)nrhs;
  return fwd ? launch_one<true>(n, LUw, ldl, B, ldb, 1, ticket, flags, epoch, units, s, jlo, jhi, c0, nind)
             : launch_one<false>(n, LUw, ldl, B, ldb, 1, ticket, flags, epoch, units, s, jlo, jhi, c0, nind);
}

int64_t launch_solve_epochs(int64_t nrhs) { return 2 * ((nrhs + kMaxInterleave - 1) / kMaxInterleave); }

int64_t solve_max_rhs() { return MAXR; }
int64_t solve_max_interleave() { return kMaxInterleave; }

}  // namespace ebv

EBV_DEBUG_SETTER(set_debug_solve)
