// k_leaf.cu — the small dense pieces of the blocked EbV LU (all <= 64 wide):
//   leaf_lu          LU of a diagonal block (w <= 64) in one CTA
//   panel_leaf       the diagonal block and the rows below in one launch
//                    (column steps); panel_blk: the same in 16-column
//                    sub-panels (round 2, the default when rows below exist)
//   trsm_right_upper L21 = A21 U11^-1, a lane group per row (row-parallel)
//   trsm_left_lower  U12 = L11^-1 A12, a lane group per column (column-parallel)
//
// Paper: Eq 6-a l_ik = a_ik / a_kk; Eq 6-b the U_(k) row; Eq 6-c
// the rank-1 update.  Per entry, updates are applied as
// fma(-l_ik, u_kj, a_ij) in ascending k and the L division comes last — the
// canonical order of DESIGN.md — so each kernel is bitwise equal to the
// corresponding part of the serial oracle.
//
// Every kernel works on a fixed 64-wide block (in registers, or for
// panel_blk in shared memory); a narrower block (a ragged tail) is padded
// with an identity: padded multipliers are exactly 0 and fma(-0, u, a) == a,
// so the real entries see exactly the same operation sequence.
#include "ebv_internal.cuh"
#include "ebv_device.cuh"
#include <cstdlib>
#include <type_traits>

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
  EBV_LTR(0);
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
  EBV_LTR(1);
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
  EBV_LTR(2);
  if (M <= w) return;
  if (tid < W) srcp[tid] = 1.0 / sUp[tid * RS + (tid % GD) * PS];
  __syncthreads();
  EBV_LTR(3);
  // ---- rows below (trsm_ru): this CTA's 64 rows, a group of 8 lanes each
  const int64_t r = (int64_t)w + (int64_t)blockIdx.x * W + i;
  const bool rv = r < M;
  double x0[QD];
#pragma unroll
  for (int q = 0; q < QD; q++) {
    const int c = j + GD * q;
    x0[q] = (rv && c < w) ? P[r + (int64_t)c * lda] : 0.0;
  }
  EBV_LTR(4);
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
  EBV_LTR(5);
}

// ---------------------------------------------------------------- blocked panel leaf
// The panel leaf (w <= 64 columns, the diagonal block in every CTA plus the
// CTA's 64 rows below) as four 16-column sub-panels, each in four phases
// separated by CTA barriers — instead of one barrier round per column:
//   A  warp 0 factors the 16 x 16 diagonal sub-block in registers (a row
//      per lane, the pivot row by shuffles; Eq 6-a..c on the sub-block);
//   B  threads 0..47: the sub-block rows' entries to the right (U12 of the
//      sub-panel: a forward substitution with its unit L, one column per
//      thread); threads 64..: every row below the sub-block — the rest of
//      the diagonal block and the rows below — forms its 16 multipliers
//      (x = a U^-1, Markstein quotients from published reciprocals of the
//      pivots, tested after the row, the phase redone with true division
//      if any test in the CTA fails);
//   C  the same threads apply the rank-16 update (Eq 6-c for the sub-panel's
//      16 steps) to their row's entries right of the sub-panel.
// Per entry these are exactly the step-by-step operations in ascending k
// (previous sub-panels' updates first, then this sub-panel's in order, the
// division last), so the factors are bitwise the oracle's.  Shared memory
// holds the 64 x 64 block and the 64 rows below (column-major, stride 65).
constexpr int PB_LD = W + 1;
constexpr size_t kPanelBlkSmem = (size_t)(2 * W * PB_LD + W) * sizeof(double);

// phase A of panel_blk_kernel: LU of the 16 x 16 diagonal sub-block at
// (c0, c0) in registers, lane l holding row c0 + l (a separate, fully
// unrolled function: inside the sub-panel loop the step loop stayed rolled
// and its row array went to local memory)
__device__ __forceinline__ void pb_factor16(double* D, double* rc, int c0, int l, int tid, int w, double tv,
                                            int& binf) {
  double d[16];
#pragma unroll
  for (int t = 0; t < 16; t++) d[t] = D[(c0 + t) * PB_LD + c0 + l];
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const double piv = __shfl_sync(0xffffffffu, d[k], k);
    if (tid == 0 && c0 + k < w && binf == 0 && fabs(piv) <= tv) binf = c0 + k + 1;
    double u[16];
#pragma unroll
    for (int t = k + 1; t < 16; t++) u[t] = __shfl_sync(0xffffffffu, d[t], k);   // Eq 6-b (before the division)
    const bool below = l > k;
    const double lk = dev::div_z(d[k], piv);                                      // Eq 6-a
    d[k] = below ? lk : d[k];
#pragma unroll
    for (int t = k + 1; t < 16; t++) {
      const double nv = fma(-lk, u[t], d[t]);                                     // Eq 6-c
      d[t] = below ? nv : d[t];
    }
  }
  if (tid < 16) {
    double dl = d[0];
#pragma unroll
    for (int t = 1; t < 16; t++) dl = t == l ? d[t] : dl;
#pragma unroll
    for (int t = 0; t < 16; t++) D[(c0 + t) * PB_LD + c0 + l] = d[t];
    rc[c0 + l] = dev::rcp_approx(dl);
  }
}

__global__ void __launch_bounds__(256) panel_blk_kernel(int64_t M, int w, double* __restrict__ P, int64_t lda,
                                                        const double* __restrict__ tau, int64_t* info, int64_t koff,
                                                        int* count, int64_t bsP, int64_t bsInfo, int64_t bsTau) {
  P += blockIdx.y * bsP;
  info += blockIdx.y * bsInfo;
  tau += blockIdx.y * bsTau;
  if (count) count += blockIdx.y;   // (nullptr: a single CTA, the diagonal block only)
  extern __shared__ __align__(16) double pbs[];
  double* D = pbs;                     // diagonal block: D[c * PB_LD + r]
  double* R = pbs + W * PB_LD;         // the CTA's rows below: R[c * PB_LD + r]
  double* rc = R + W * PB_LD;          // rcp_approx(u_cc)
  __shared__ int slast;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t rb0 = (int64_t)w + (int64_t)blockIdx.x * W;   // first row below of this CTA
  const int nrb = M > rb0 ? (int)(M - rb0 < W ? M - rb0 : W) : 0;
  EBV_LTR(0);
  {   // load (identity-padded diagonal block, zero-padded rows below), all loads in flight
    const int r = tid & (W - 1), c4 = tid >> 6;
    double vd[W / 4], vr[W / 4];
#pragma unroll
    for (int it = 0; it < W / 4; it++) {
      const int c = c4 + 4 * it;
      vd[it] = (r < w && c < w) ? P[r + (int64_t)c * lda] : (r == c ? 1.0 : 0.0);
      vr[it] = (r < nrb && c < w) ? P[rb0 + r + (int64_t)c * lda] : 0.0;
    }
#pragma unroll
    for (int it = 0; it < W / 4; it++) {
      const int c = c4 + 4 * it;
      D[c * PB_LD + r] = vd[it];
      R[c * PB_LD + r] = vr[it];
    }
  }
  const double tv = *tau;
  __syncthreads();   // every CTA has read the unfactored diagonal block
  if (tid == 0) {
    if (!count) {
      slast = 1;
    } else {
      __threadfence();
      const int old = atomicAdd(count, 1);
      slast = old == (int)gridDim.x - 1;
      if (slast) {
        *count = 0;
        __threadfence();
      }
    }
  }
  int binf = 0;
  EBV_LTR(1);
#pragma unroll 1
  for (int c0 = 0; c0 < W; c0 += 16) {
    // ---- A: the 16 x 16 diagonal sub-block, one row per lane (lanes 16..31 mirror 0..15)
    if (tid < 32) pb_factor16(D, rc, c0, lane & 15, tid, w, tv, binf);
    __syncthreads();
    EBV_LTR(2 + 3 * (c0 / 16));
    const int ncol = W - c0 - 16;                 // columns right of the sub-panel
    const int ndr = W - c0 - 16;                  // diagonal-block rows below the sub-block
    // ---- B1: U12 of the sub-panel rows, one column per thread
    if (tid < ncol) {
      const int j = c0 + 16 + tid;
      double u[16];
#pragma unroll
      for (int r = 0; r < 16; r++) u[r] = D[j * PB_LD + c0 + r];
#pragma unroll
      for (int p = 0; p < 15; p++)
#pragma unroll
        for (int r = p + 1; r < 16; r++) u[r] = fma(-D[(c0 + p) * PB_LD + c0 + r], u[p], u[r]);
#pragma unroll
      for (int r = 0; r < 16; r++) D[j * PB_LD + c0 + r] = u[r];
    }
    // ---- B2: the multipliers of every row below the sub-block (one row per thread)
    const int ri = tid - 64;
    const bool brow = ri >= 0 && ri < ndr + nrb;
    double* base = nullptr;
    int row = 0;
    if (brow) {
      if (ri < ndr) { base = D; row = c0 + 16 + ri; }
      else { base = R; row = ri - ndr; }
    }
    double x[16], xin[16], ys[16];
    if (brow) {
#pragma unroll
      for (int t = 0; t < 16; t++) xin[t] = base[(c0 + t) * PB_LD + row];
    }
    auto solve_row = [&](auto exact_tag) -> bool {
      constexpr bool EXACT = decltype(exact_tag)::value;
      bool ok = true;
#pragma unroll
      for (int t = 0; t < 16; t++) x[t] = xin[t];
#pragma unroll
      for (int t = 0; t < 16; t++) {
        const double utt = D[(c0 + t) * PB_LD + c0 + t];
        if (EXACT) {
          x[t] = dev::div_z(x[t], utt);                                             // Eq 6-a
        } else {
          ys[t] = x[t];
          x[t] = dev::quot_mk(x[t], utt, rc[c0 + t]);
        }
#pragma unroll
        for (int t2 = t + 1; t2 < 16; t2++) x[t2] = fma(-x[t], D[(c0 + t2) * PB_LD + c0 + t], x[t2]);
      }
      if (!EXACT) {
#pragma unroll
        for (int t = 0; t < 16; t++) ok &= dev::quot_is_rn(ys[t], D[(c0 + t) * PB_LD + c0 + t], x[t]);
      }
      return ok;
    };
    bool ok = true;
    if (brow) ok = solve_row(std::false_type{});
    if (__syncthreads_or(!ok)) {   // rare: the phase again with true division
      if (brow) solve_row(std::true_type{});
    }
    if (brow) {
#pragma unroll
      for (int t = 0; t < 16; t++) base[(c0 + t) * PB_LD + row] = x[t];
    }
    __syncthreads();   // U12 of the sub-panel (B1) is complete
    EBV_LTR(3 + 3 * (c0 / 16));
    // ---- C: the rank-16 update of the row's entries right of the sub-panel
    if (brow) {   // four columns at a time: four independent fma chains
#pragma unroll 1
      for (int j = c0 + 16; j < W; j += 4) {
        double v[4];
#pragma unroll
        for (int e = 0; e < 4; e++) v[e] = base[(j + e) * PB_LD + row];
#pragma unroll
        for (int t = 0; t < 16; t++)
#pragma unroll
          for (int e = 0; e < 4; e++) v[e] = fma(-x[t], D[(j + e) * PB_LD + c0 + t], v[e]);   // Eq 6-c
#pragma unroll
        for (int e = 0; e < 4; e++) base[(j + e) * PB_LD + row] = v[e];
      }
    }
    __syncthreads();
    EBV_LTR(4 + 3 * (c0 / 16));
  }
  // ---- store: the diagonal block by the last CTA to arrive, every CTA its rows below
  const bool store = slast != 0;
  {
    const int r = tid & (W - 1), c4 = tid >> 6;
#pragma unroll
    for (int it = 0; it < W / 4; it++) {
      const int c = c4 + 4 * it;
      if (store && r < w && c < w) P[r + (int64_t)c * lda] = D[c * PB_LD + r];
      if (r < nrb && c < w) P[rb0 + r + (int64_t)c * lda] = R[c * PB_LD + r];
    }
  }
  if (store && tid == 0 && binf) {
    volatile int64_t* vi = info;
    if (*vi == 0) *vi = koff + binf;
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

// EBV_PANEL_BLK=0: the column-step panel leaf instead of the blocked one
static bool panel_blocked() {
  static const bool v = [] {
    const char* e = getenv("EBV_PANEL_BLK");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

cudaError_t launch_leaf_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info, int64_t koff,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > W) return cudaErrorInvalidValue;
  // (the blocked kernel as one CTA with no rows below measured slower here:
  // C1 n = 64 40.6 -> 45.6 us; its phases pay off with rows below)
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
  const int64_t grid = M > w ? (M - w + W - 1) / W : 1;
  if (panel_blocked() && M > w) {   // (a lone diagonal block: the column-step kernel is faster)
    cudaError_t e = ensure_max_dyn_smem(reinterpret_cast<const void*>(panel_blk_kernel), (int)kPanelBlkSmem);
    if (e != cudaSuccess) return e;
    panel_blk_kernel<<<(unsigned)grid, 256, kPanelBlkSmem, s>>>(M, (int)w, P, lda, tau, info, koff, count, 0, 0, 0);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)W * kLeafG * (W / kLeafG + 2) * sizeof(double);
  {
    cudaError_t e = panel_leaf_attr(smem);
    if (e != cudaSuccess) return e;
  }
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
  // the batched form keeps the column-step kernel: with many independent
  // panels per launch throughput wins, and the blocked kernel's one CTA per
  // SM (255 registers, 67 KB) lost there (20000 x n = 128: 12.46 -> 13.40 ms)
  const bool blk = false;
  const size_t smem = blk ? kPanelBlkSmem : (size_t)W * kLeafG * (W / kLeafG + 2) * sizeof(double);
  cudaError_t e = blk ? ensure_max_dyn_smem(reinterpret_cast<const void*>(panel_blk_kernel), (int)smem)
                      : panel_leaf_attr(smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = M > w ? (M - w + W - 1) / W : 1;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    if (blk)
      panel_blk_kernel<<<dim3((unsigned)grid, (unsigned)nb), 256, smem, s>>>(
          M, (int)w, P + b0 * bsP, lda, tau + b0 * bsTau, info + b0 * bsInfo, koff, count + b0, bsP, bsInfo, bsTau);
    else
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
