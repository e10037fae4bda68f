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
#include "ebv_device.cuh"
#include <cstdlib>

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

// Code size: these kernels are latency-bound chains executed a few times per
// launch, so a fully unrolled 64-step body (3-5k SASS instructions) ran
// instruction-fetch bound.  The step loop is rolled over blocks of G steps:
// inside a block the G steps are unrolled, and at the end of the block each
// lane's first register (column j + G*qk, now final) is stored and the
// register file is rotated down by one, so the live entries of block qk are
// always a[0..Q-1-qk].  Rotated-in slots are dead (never stored); the shared
// rows are padded to 2W so their reads stay in bounds.

// ---------------------------------------------------------------- leaf LU
// 512 threads: row i of the block is owned by group i.  Step k: group k
// publishes its final row (the U_(k) vector, Eq 6-b) to shared memory; every
// row i > k forms l_ik = a_ik / u_kk (Eq 6-a, owner lane), broadcasts it in
// the group and updates its row (Eq 6-c).  A narrower block is identity
// padded (exactly neutral).
template <int GD>
__global__ void __launch_bounds__(W * GD) leaf_lu_kernel(int w, double* __restrict__ A, int64_t lda,
                                                        const double* __restrict__ tau, int64_t* info, int64_t koff) {
  constexpr int QD = W / GD, PS = QD + 2;
  __shared__ __align__(16) double urow[2][GD * PS];   // lane-slot layout: urow[.][j*PS + q] = lane j's a[q]
  __shared__ int smin;
  const int tid = threadIdx.x, i = tid / GD, j = tid % GD, lane = tid & 31, base = lane & ~(GD - 1);
  double a[QD];
#pragma unroll
  for (int q = 0; q < QD; q++) {
    const int c = j + GD * q;
    a[q] = (i < w && c < w) ? A[i + (int64_t)c * lda] : (i == c ? 1.0 : 0.0);
  }
  if (tid == 0) smin = 0x7fffffff;
  const double tv = *tau;
#pragma unroll 1
  for (int qk = 0; qk < QD; qk++) {
#pragma unroll
    for (int o = 0; o < GD; o++) {
      const int k = qk * GD + o;
      double* ur = urow[o & 1];                    // ur[j*PS + q] = u(k, j + GD*(q + qk))
      if (i == k) {
#pragma unroll
        for (int q = 0; q < QD; q += 2) *reinterpret_cast<double2*>(ur + j * PS + q) = make_double2(a[q], a[q + 1]);
      }
      __syncthreads();
      const double piv = ur[o * PS];
      if (tid == 0 && k < w && fabs(piv) <= tv) atomicMin(&smin, k + 1);
      if (i > k && j == o) a[0] = a[0] / piv;                       // Eq 6-a
      const double l = __shfl_sync(0xffffffffu, a[0], base + o);
      if (i > k) {                                                   // Eq 6-c
        const double* uj = ur + j * PS;
#pragma unroll
        for (int q = 0; q < QD; q += 2) {
          const double2 u2 = *reinterpret_cast<const double2*>(uj + q);
          if (q > 0 || j > o) a[q] = fma(-l, u2.x, a[q]);
          a[q + 1] = fma(-l, u2.y, a[q + 1]);
        }
      }
    }
    const int c = j + GD * qk;                        // final: store, rotate
    if (i < w && c < w) A[i + (int64_t)c * lda] = a[0];
#pragma unroll
    for (int q = 0; q < QD - 1; q++) a[q] = a[q + 1];
    a[QD - 1] = 0.0;
  }
  __syncthreads();
  if (tid == 0 && smin != 0x7fffffff) {
    volatile int64_t* vi = info;
    if (*vi == 0) *vi = koff + smin;
  }
}

// Stage a 64 x 64 block in shared memory with all of a thread's loads in
// flight at once.  (The rolled grid-stride form — load, store, next — waited
// one L2 round trip per iteration: 16 x ~600 cycles at 256 threads, ~5 us of
// every TRSM leaf launch, probes/trsm_trace.cu.)  NTHR = blockDim.x.
template <int NTHR, typename Load, typename Store>
__device__ __forceinline__ void stage64(Load load, Store store) {
  constexpr int IT = W * W / NTHR;
  double v[IT];
#pragma unroll
  for (int it = 0; it < IT; it++) v[it] = load((int)threadIdx.x + it * NTHR);
#pragma unroll
  for (int it = 0; it < IT; it++) store((int)threadIdx.x + it * NTHR, v[it]);
}

// ---------------------------------------------------------------- L21 = A21 U11^-1
// Group per row: step p, the owner lane forms x_p / u_pp, broadcasts it, every
// lane applies x_c = fma(-x_p, u_pc, x_c) to its entries c > p.  The quotient
// comes from the hoisted reciprocal RN(1/u_pp) with one Markstein correction,
// verified exactly (the remainder test of k_solve.cu); a warp with any
// unverified quotient redoes its rows with true division, so every entry is
// RN(x/u) — bitwise the oracle — and the chain per step is three dependent
// fp64 operations instead of a division.
__device__ __forceinline__ double quot_m(double y, double u, double r) { return dev::quot_mk(y, u, r); }
// exact test that q == RN(y / u) (dev::quot_is_rn; +0 dividends — the
// identity padding — are exact)
__device__ __forceinline__ bool quot_ok(double y, double u, double q) { return dev::quot_is_rn(y, u, q); }

// RR rows per lane group (independent chains interleaved): a CTA of 256
// threads covers 32*RR rows, so the kernel holds few SM slots for its
// latency-bound duration (it runs beside the DMMA update on the lookahead
// stream; 128 registers keep it within one update CTA's register share).
// Each block of 8 steps is checkpointed; if any quotient of the block is
// unverified the warp redoes that block with true division.
constexpr int RR = 2;
#ifdef EBV_LEAF_TRACE
// probes/trsm_trace.cu: %clock64 stamps of CTA 0, thread 0 (slot 0 entry,
// 1 U staged, 2 reciprocals, 3 X loaded, 4 + qk end of block qk)
__device__ long long g_ltrace[16];
#define EBV_LTR(slot)                                                  \
  do {                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_ltrace[slot] = clock64(); \
  } while (0)
#else
#define EBV_LTR(slot) \
  do {                \
  } while (0)
#endif
#ifndef EBV_LEAF_G
#define EBV_LEAF_G 4
#endif
constexpr int kLeafG = EBV_LEAF_G;   // lanes per row in the diagonal-block kernels

__global__ void __launch_bounds__(256, 2) trsm_ru_kernel(int64_t m, int k, double* __restrict__ X, int64_t ldx,
                                                         const double* __restrict__ U, int64_t ldu) {
  __shared__ __align__(16) double sU[W * S + W];   // sU[p*S + c] = u(p, c), identity padded (+ overrun pad)
  __shared__ double srcp[W];
  EBV_LTR(0);
  stage64<256>(
      [&](int idx) {
        const int p = idx % W, c = idx / W;
        return (p < k && c < k) ? (p <= c ? U[p + (int64_t)c * ldu] : 0.0) : (p == c ? 1.0 : 0.0);
      },
      [&](int idx, double v) { sU[(idx % W) * S + idx / W] = v; });
  for (int idx = threadIdx.x; idx < W * (S - W) + W; idx += blockDim.x)   // the pad columns of each row + tail
    if (idx < W * (S - W)) sU[(idx / (S - W)) * S + W + idx % (S - W)] = 0.0; else sU[W * S + idx - W * (S - W)] = 0.0;
  __syncthreads();
  EBV_LTR(1);
  if (threadIdx.x < W) srcp[threadIdx.x] = 1.0 / sU[threadIdx.x * S + threadIdx.x];
  __syncthreads();
  EBV_LTR(2);
  const int tid = threadIdx.x, j = tid % G, lane = tid & 31, base = lane & ~(G - 1);
  const int64_t i0 = (int64_t)blockIdx.x * (32 * RR) + tid / G;   // rows i0 + 32 r
  double x[RR][Q];
#pragma unroll
  for (int r = 0; r < RR; r++)
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int c = j + G * q;
      const int64_t i = i0 + 32 * r;
      x[r][q] = (i < m && c < k) ? X[i + (int64_t)c * ldx] : 0.0;
    }
  EBV_LTR(3);
#pragma unroll 1
  for (int qk = 0; qk < Q; qk++) {
    double xs[RR][Q];
#pragma unroll
    for (int r = 0; r < RR; r++)
#pragma unroll
      for (int q = 0; q < Q; q++) xs[r][q] = x[r][q];
    // the quotients of the block are verified after it (off the step chain):
    // lane j owns step qk*G + j and keeps its dividend and quotient
    double ychk[RR], qchk[RR];
#pragma unroll
    for (int o = 0; o < G; o++) {
      const int p = qk * G + o;
      const double* up = sU + p * S + G * qk;     // up[j + G*q] = u(p, j + G*(q + qk))
      const double upp = up[o], rp = srcp[p];
#pragma unroll
      for (int r = 0; r < RR; r++) {
        if (j == o) {
          ychk[r] = x[r][0];
          x[r][0] = quot_m(x[r][0], upp, rp);
          qchk[r] = x[r][0];
        }
        const double xp = __shfl_sync(0xffffffffu, x[r][0], base + o);
        if (j > o) x[r][0] = fma(-xp, up[j], x[r][0]);
#pragma unroll
        for (int q = 1; q < Q; q++) x[r][q] = fma(-xp, up[j + G * q], x[r][q]);
      }
    }
    bool ok = true;
    {
      const double uown = sU[(qk * G + j) * S + qk * G + j];
#pragma unroll
      for (int r = 0; r < RR; r++) ok = ok && quot_ok(ychk[r], uown, qchk[r]);
    }
    if (__any_sync(0xffffffffu, !ok)) {            // redo the block with true division
#pragma unroll
      for (int r = 0; r < RR; r++)
#pragma unroll
        for (int q = 0; q < Q; q++) x[r][q] = xs[r][q];
#pragma unroll
      for (int o = 0; o < G; o++) {
        const int p = qk * G + o;
        const double* up = sU + p * S + G * qk;
#pragma unroll
        for (int r = 0; r < RR; r++) {
          if (j == o) x[r][0] = x[r][0] / up[o];
          const double xp = __shfl_sync(0xffffffffu, x[r][0], base + o);
          if (j > o) x[r][0] = fma(-xp, up[j], x[r][0]);
#pragma unroll
          for (int q = 1; q < Q; q++) x[r][q] = fma(-xp, up[j + G * q], x[r][q]);
        }
      }
    }
    const int c = j + G * qk;
#pragma unroll
    for (int r = 0; r < RR; r++) {
      const int64_t i = i0 + 32 * r;
      if (i < m && c < k) X[i + (int64_t)c * ldx] = x[r][0];
#pragma unroll
      for (int q = 0; q < Q - 1; q++) x[r][q] = x[r][q + 1];
      x[r][Q - 1] = 0.0;
    }
    EBV_LTR(4 + qk);
  }
}

// ---------------------------------------------------------------- panel leaf
// The leaf of the panel recursion in ONE launch: LU of the w x w diagonal
// block and L21 = A21 U11^-1 for the M - w rows below (leaf_lu + trsm_ru
// fused, one kernel boundary less on the panel's critical chain).  Every CTA
// factors the diagonal block itself (the same operations in every CTA, so
// the same bits) with the leaf_lu scheme; the CTA that arrives last (an
// arrival counter, so every CTA has read the unfactored block before it is
// overwritten — CTAs of one launch need not run at the same time) stores it
// and reports info,
// publishing each final U row into a full shared copy of U11, then solves
// its 64 rows below with the trsm_ru scheme (verified reciprocal quotients).
// Shared U rows in the lane-slot layout of leaf_lu_kernel: row k occupies
// GD slots of PS doubles, slot j holding lane j's entries in local
// (rotated) order, so each lane reads its entries with 16-byte loads.

template <int GD>
__global__ void __launch_bounds__(W * GD) panel_leaf_kernel(int64_t M, int w, double* __restrict__ P, int64_t lda,
                                                           const double* __restrict__ tau, int64_t* info,
                                                           int64_t koff, int* count, int64_t bsP, int64_t bsInfo,
                                                           int64_t bsTau) {
  // batched form: blockIdx.y = system (its panel, info word, tau and
  // arrival counter); strides 0 and gridDim.y = 1 for one system
  P += blockIdx.y * bsP;
  info += blockIdx.y * bsInfo;
  tau += blockIdx.y * bsTau;
  count += blockIdx.y;
  constexpr int QD = W / GD, PS = QD + 2, RS = GD * PS;
  extern __shared__ __align__(16) double sUp[];    // [W][RS]: sUp[k*RS + j*PS + q] = u(k, j + GD*(q + k/GD))
  __shared__ double srcp[W];
  __shared__ int smin, slast;
  const int tid = threadIdx.x, i = tid / GD, j = tid % GD, lane = tid & 31, base = lane & ~(GD - 1);
  for (int idx = tid; idx < W * RS; idx += W * GD) sUp[idx] = 0.0;
  double a[QD];
#pragma unroll
  for (int q = 0; q < QD; q++) {
    const int c = j + GD * q;
    a[q] = (i < w && c < w) ? P[i + (int64_t)c * lda] : (i == c ? 1.0 : 0.0);
  }
  if (tid == 0) smin = 0x7fffffff;
  const double tv = *tau;
  __syncthreads();   // every thread's loads of the diagonal block are done (values in registers)
  if (tid == 0) {
    __threadfence();
    const int old = atomicAdd(count, 1);
    slast = old == (int)gridDim.x - 1;
    if (slast) {
      *count = 0;    // every CTA has arrived: reset for the next launch
      __threadfence();
    }
  }
  __syncthreads();
  const bool store = slast != 0;
  // ---- diagonal block (leaf_lu, publishing into the full U copy)
#pragma unroll 1
  for (int qk = 0; qk < QD; qk++) {
#pragma unroll
    for (int o = 0; o < GD; o++) {
      const int k = qk * GD + o;
      double* ur = sUp + k * RS;                     // ur[j*PS + q] = u(k, j + GD*(q + qk))
      if (i == k) {
#pragma unroll
        for (int q = 0; q < QD; q += 2) *reinterpret_cast<double2*>(ur + j * PS + q) = make_double2(a[q], a[q + 1]);
      }
      __syncthreads();
      const double piv = ur[o * PS];
      if (store && tid == 0 && k < w && fabs(piv) <= tv) atomicMin(&smin, k + 1);
      if (i > k && j == o) a[0] = a[0] / piv;                       // Eq 6-a
      const double l = __shfl_sync(0xffffffffu, a[0], base + o);
      if (i > k) {                                                   // Eq 6-c
        const double* uj = ur + j * PS;
#pragma unroll
        for (int q = 0; q < QD; q += 2) {
          const double2 u2 = *reinterpret_cast<const double2*>(uj + q);
          if (q > 0 || j > o) a[q] = fma(-l, u2.x, a[q]);
          a[q + 1] = fma(-l, u2.y, a[q + 1]);
        }
      }
    }
    const int c = j + GD * qk;
    if (store && i < w && c < w) P[i + (int64_t)c * lda] = a[0];
#pragma unroll
    for (int q = 0; q < QD - 1; q++) a[q] = a[q + 1];
    a[QD - 1] = 0.0;
  }
  __syncthreads();
  if (store && tid == 0 && smin != 0x7fffffff) {
    volatile int64_t* vi = info;
    if (*vi == 0) *vi = koff + smin;
  }
  if (M <= w) return;
  if (tid < W) srcp[tid] = 1.0 / sUp[tid * RS + (tid % GD) * PS];
  __syncthreads();
  // ---- rows below (trsm_ru): this CTA's 64 rows, a group of 8 lanes each
  const int64_t r = (int64_t)w + (int64_t)blockIdx.x * W + i;
  const bool rv = r < M;
  double x0[QD];
#pragma unroll
  for (int q = 0; q < QD; q++) {
    const int c = j + GD * q;
    x0[q] = (rv && c < w) ? P[r + (int64_t)c * lda] : 0.0;
  }
  for (int pass = 0; pass < 2; pass++) {
    const bool exact = pass == 1;
    bool ok = true;
    double x[QD];
#pragma unroll
    for (int q = 0; q < QD; q++) x[q] = x0[q];
#pragma unroll 1
    for (int qk = 0; qk < QD; qk++) {
      double ychk = 0.0, qchk = 0.0;                  // lane j's step of the block, verified after it
#pragma unroll
      for (int o = 0; o < GD; o++) {
        const int p = qk * GD + o;
        const double* up = sUp + p * RS;
        if (j == o) {
          ychk = x[0];
          x[0] = exact ? x[0] / up[o * PS] : quot_m(x[0], up[o * PS], srcp[p]);
          qchk = x[0];
        }
        const double xp = __shfl_sync(0xffffffffu, x[0], base + o);
        const double* uj = up + j * PS;
#pragma unroll
        for (int q = 0; q < QD; q += 2) {
          const double2 u2 = *reinterpret_cast<const double2*>(uj + q);
          if (q > 0 || j > o) x[q] = fma(-xp, u2.x, x[q]);
          x[q + 1] = fma(-xp, u2.y, x[q + 1]);
        }
      }
      if (!exact) ok = ok && quot_ok(ychk, sUp[(qk * GD + j) * RS + j * PS], qchk);
      const int c = j + GD * qk;
      if (rv && c < w) P[r + (int64_t)c * lda] = x[0];
#pragma unroll
      for (int q = 0; q < QD - 1; q++) x[q] = x[q + 1];
      x[QD - 1] = 0.0;
    }
    if (!__any_sync(0xffffffffu, !ok)) break;
  }
}

// ---------------------------------------------------------------- U12 = L11^-1 A12
// Group per column: step p, x_p is final (owner lane), broadcast; every lane
// applies x_r = fma(-l_rp, x_p, x_r) to its rows r > p (unit diagonal).
// CC columns per lane group (independent chains interleaved, the shared L
// values loaded once for all of them): a CTA of 256 threads covers 32*CC
// columns, so the kernel holds fewer SM slots beside the DMMA update.
template <int CC>
__global__ void __launch_bounds__(256) trsm_llu_kernel(int k, int64_t m, const double* __restrict__ L, int64_t ldl,
                                                       double* __restrict__ X, int64_t ldx, int64_t bsL, int64_t bsX) {
  L += blockIdx.y * bsL;   // batched form: blockIdx.y = system
  X += blockIdx.y * bsX;
  __shared__ __align__(16) double sL[W * S];   // sL[p*S + r] = l(r, p), r > p
  stage64<256>(
      [&](int idx) {
        const int r = idx % W, p = idx / W;
        return (r > p && r < k) ? L[r + (int64_t)p * ldl] : 0.0;
      },
      [&](int idx, double v) { sL[(idx / W) * S + idx % W] = v; });
  __syncthreads();
  const int tid = threadIdx.x, j = tid % G, lane = tid & 31, base = lane & ~(G - 1);
  // grid-stride over chunks of 32*CC columns (the grid may be capped so the
  // solve holds fewer SM slots beside the update; L11 is staged once per CTA)
  const int64_t nchunks = (m + 32 * CC - 1) / (32 * CC);
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
  const int64_t c0 = chunk * (256 / G) * CC + tid / G;   // columns c0 + 32 cc
  double x[CC][Q];
  bool cv[CC];
#pragma unroll
  for (int cc = 0; cc < CC; cc++) {
    const int64_t cidx = c0 + 32 * cc;
    cv[cc] = cidx < m;
    const double* col = X + (cv[cc] ? cidx : 0) * ldx;
#pragma unroll
    for (int q = 0; q < Q; q++) {
      const int r = j + G * q;
      x[cc][q] = (cv[cc] && r < k) ? col[r] : 0.0;
    }
  }
#pragma unroll
  for (int p = 0; p < W; p++) {
    const int o = p % G, qp = p / G;
    const double* lp = sL + p * S;
    double xp[CC];
#pragma unroll
    for (int cc = 0; cc < CC; cc++) xp[cc] = __shfl_sync(0xffffffffu, x[cc][qp], base + o);
#pragma unroll
    for (int q = qp; q < Q; q++)
      if (q > qp || j > o) {
        const double l = lp[j + G * q];
#pragma unroll
        for (int cc = 0; cc < CC; cc++) x[cc][q] = fma(-l, xp[cc], x[cc][q]);
      }
  }
#pragma unroll
  for (int cc = 0; cc < CC; cc++) {
    if (cv[cc]) {
      double* col = X + (c0 + 32 * cc) * ldx;
#pragma unroll
      for (int q = 0; q < Q; q++) {
        const int r = j + G * q;
        if (r < k) col[r] = x[cc][q];
      }
    }
  }
  }
}

// ---------------------------------------------------------------- X = U11^-1 X
// Backward substitution per column (thread per column), k descending:
// x_p = x_p / u_pp, then x_i = fma(-u_ip, x_p, x_i) for i < p — the oracle's
// backward order (Eq 1, UX = Y).  Padded rows (p >= k) are identity rows and
// come first in the descending sweep: they change nothing.
__global__ void __launch_bounds__(128) trsm_luu_kernel(int k, int64_t m, const double* __restrict__ U, int64_t ldu,
                                                       double* __restrict__ X, int64_t ldx, int64_t bsU, int64_t bsX) {
  U += blockIdx.y * bsU;   // batched form: blockIdx.y = system
  X += blockIdx.y * bsX;
  __shared__ __align__(16) double sU[W * S];   // sU[p*S + i] = u(i, p), i <= p (column p of U)
  stage64<128>(
      [&](int idx) {
        const int i = idx % W, p = idx / W;
        return (i < k && p < k) ? (i <= p ? U[i + (int64_t)p * ldu] : 0.0) : (i == p ? 1.0 : 0.0);
      },
      [&](int idx, double v) { sU[(idx / W) * S + idx % W] = v; });
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
  trsm_luu_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>((int)k, m, U, ldu, X, ldx, 0, 0);
  return cudaGetLastError();
}

cudaError_t launch_leaf_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info, int64_t koff,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > W) return cudaErrorInvalidValue;
  leaf_lu_kernel<kLeafG><<<1, W * kLeafG, 0, s>>>((int)n, A, lda, tau, info, koff);
  return cudaGetLastError();
}

static cudaError_t panel_leaf_attr(size_t smem) {
  return ensure_max_dyn_smem(reinterpret_cast<const void*>(panel_leaf_kernel<kLeafG>), (int)smem);
}

cudaError_t launch_panel_leaf(int64_t M, int64_t w, double* P, int64_t lda, const double* tau, int64_t* info,
                              int64_t koff, int* count, cudaStream_t s) {
  if (w <= 0 || M <= 0) return cudaSuccess;
  if (w > W || M < w) return cudaErrorInvalidValue;
  const size_t smem = (size_t)W * kLeafG * (W / kLeafG + 2) * sizeof(double);
  {
    cudaError_t e = panel_leaf_attr(smem);
    if (e != cudaSuccess) return e;
  }
  const int64_t grid = M > w ? (M - w + W - 1) / W : 1;
  panel_leaf_kernel<kLeafG><<<(unsigned)grid, W * kLeafG, smem, s>>>(M, (int)w, P, lda, tau, info, koff, count, 0, 0,
                                                                      0);
  return cudaGetLastError();
}

cudaError_t launch_trsm_right_upper(int64_t m, int64_t k, double* X, int64_t ldx, const double* U, int64_t ldu,
                                    cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  trsm_ru_kernel<<<(unsigned)((m + 32 * RR - 1) / (32 * RR)), 256, 0, s>>>(m, (int)k, X, ldx, U, ldu);
  return cudaGetLastError();
}

cudaError_t launch_trsm_left_lower_unit(int64_t k, int64_t m, const double* L, int64_t ldl, double* X,
                                        int64_t ldx, cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  static const int cc = [] {
    const char* e = getenv("EBV_TRSM_LLU_CC");
    return e ? atoi(e) : 2;
  }();
  if (cc == 2) {
    static const int64_t gcap = [] {
      const char* e = getenv("EBV_TRSM_LLU_GRID");
      return e ? (int64_t)atoll(e) : (int64_t)0;
    }();
    int64_t grid = (m + 63) / 64;
    if (gcap > 0 && grid > gcap) grid = gcap;
    trsm_llu_kernel<2><<<(unsigned)grid, 256, 0, s>>>((int)k, m, L, ldl, X, ldx, 0, 0);
    return cudaGetLastError();
  }
  trsm_llu_kernel<1><<<(unsigned)((m + 31) / 32), 256, 0, s>>>((int)k, m, L, ldl, X, ldx, 0, 0);
  return cudaGetLastError();
}

// ---- batched forms (systems s = 0..batch-1 at base + s*stride; gridDim.y =
// system, chunks of 65535): per system exactly the single-system kernels
cudaError_t launch_panel_leaf_batched(int64_t M, int64_t w, double* P, int64_t lda, int64_t bsP, const double* tau,
                                      int64_t bsTau, int64_t* info, int64_t bsInfo, int64_t koff, int* count,
                                      int64_t batch, cudaStream_t s) {
  if (w <= 0 || M <= 0 || batch <= 0) return cudaSuccess;
  if (w > W || M < w) return cudaErrorInvalidValue;
  const size_t smem = (size_t)W * kLeafG * (W / kLeafG + 2) * sizeof(double);
  cudaError_t e = panel_leaf_attr(smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = M > w ? (M - w + W - 1) / W : 1;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    panel_leaf_kernel<kLeafG><<<dim3((unsigned)grid, (unsigned)nb), W * kLeafG, smem, s>>>(
        M, (int)w, P + b0 * bsP, lda, tau + b0 * bsTau, info + b0 * bsInfo, koff, count + b0, bsP, bsInfo, bsTau);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_trsm_llu_batched(int64_t k, int64_t m, const double* L, int64_t ldl, int64_t bsL, double* X,
                                    int64_t ldx, int64_t bsX, int64_t batch, cudaStream_t s) {
  if (m <= 0 || k <= 0 || batch <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    trsm_llu_kernel<2><<<dim3((unsigned)((m + 63) / 64), (unsigned)nb), 256, 0, s>>>((int)k, m, L + b0 * bsL, ldl,
                                                                                     X + b0 * bsX, ldx, bsL, bsX);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_trsm_luu_batched(int64_t k, int64_t m, const double* U, int64_t ldu, int64_t bsU, double* X,
                                    int64_t ldx, int64_t bsX, int64_t batch, cudaStream_t s) {
  if (m <= 0 || k <= 0 || batch <= 0) return cudaSuccess;
  if (k > W) return cudaErrorInvalidValue;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    trsm_luu_kernel<<<dim3((unsigned)((m + 127) / 128), (unsigned)nb), 128, 0, s>>>((int)k, m, U + b0 * bsU, ldu,
                                                                                  X + b0 * bsX, ldx, bsU, bsX);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ebv

EBV_DEBUG_SETTER(set_debug_leaf)
