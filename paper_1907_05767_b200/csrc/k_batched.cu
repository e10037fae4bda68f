// k_batched.cu — fused factor + solve of many independent small systems
// (n <= 32), BASELINE.json configs[4] (reading R16: each system is an
// instance of Eq 1 / Eq 6).
//
// EbV at lane granularity (Eq 7: "mix ... first and end ... to make
// vectors equals in size"): a warp holds TWO systems, one per half-warp, and
// lane t of a half owns rows t and 31-t of its system — the first-with-last
// pairing of the row vectors, so every lane carries two rows whose combined
// active length is the same (the systems are padded to 32 with identity rows,
// which leaves the leading n x n results bitwise unchanged: their multipliers
// are exactly 0 and fma(-0, u, a) == a).  At step k the pivot and the U_(k)
// row are broadcast inside the half-warp by shuffles (Eq 6-b); each lane
// divides its own multipliers (Eq 6-a) and applies the rank-1 update to its
// two rows (Eq 6-c).  One shuffle serves both systems of the warp.  The
// solve (Eq 1) follows in registers: forward over L_(k), backward over U_(k).
// Per-entry arithmetic is exactly the oracle's (bitwise).
#include "ebv_internal.cuh"
#include "ebv_device.cuh"
#include <type_traits>

namespace ebv {
namespace {

constexpr int NP = 32;   // padded order
constexpr int MAXRHS = 16;

#ifndef EBV_BATCHED_CH
#define EBV_BATCHED_CH 8
#endif
constexpr int CH = EBV_BATCHED_CH;   // columns per shuffle chunk

// Markstein quotient from an approximate reciprocal, and the exact test that
// it is RN(y / u) (remainder y - q u exact by fma, inside half an ulp of q
// times |u|, halved below a power of two; +0 dividends exact)
__device__ __forceinline__ double rcp_approx(double u) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
  double e = fma(-u, r, 1.0);
  r = fma(r, e, r);
  e = fma(-u, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double quot_mk(double y, double u, double r) { return dev::quot_mk(y, u, r); }
// the division of the padded kernels (n below the tile: identity rows give
// zero dividends, dev::div_z); unpadded ones keep the plain division (the
// extra test cost ~15% at n = 32)
template <bool PAD>
__device__ __forceinline__ double divp(double y, double u) { return PAD ? dev::div_z(y, u) : y / u; }
__device__ __forceinline__ bool quot_exact(double y, double u, double q) { return dev::quot_is_rn(y, u, q); }

// Row updates of rows that may sit above the pivot are guarded by a branch
// around a chunk of CH fma's (a predicated fma is if-converted by ptxas into
// an fma plus two selects, which made selects 20% of the instruction stream).
// FULL: n == 32 (no identity padding: no predicates on loads and stores).
template <bool FULL, int RG>
__global__ void __launch_bounds__(128) batched_kernel(int n, double* __restrict__ A, int64_t lda,
                                                      int64_t strideA, int64_t batch, double* __restrict__ B,
                                                      int64_t ldb, int64_t strideB, int nrhs,
                                                      const double* __restrict__ tau_ptr, int tau_default,
                                                      double tau_value, int32_t* __restrict__ info,
                                                      int solve_only) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int h = lane >> 4, t = lane & 15;
  const int64_t sys = 2 * warp + h;
  const bool act = sys < batch;
  const int r0 = t, r1 = NP - 1 - t;              // the paired rows of this lane
  const bool v0 = act && (FULL || r0 < n), v1 = act && (FULL || r1 < n);
  double* As = A + (act ? sys : 0) * strideA;

  double ra[NP], rb[NP];
#pragma unroll
  for (int j = 0; j < NP; j++) {
    if (FULL) {
      ra[j] = act ? As[r0 + (int64_t)j * lda] : (r0 == j ? 1.0 : 0.0);
      rb[j] = act ? As[r1 + (int64_t)j * lda] : (r1 == j ? 1.0 : 0.0);
    } else {
      ra[j] = (v0 && j < n) ? As[r0 + (int64_t)j * lda] : (r0 == j ? 1.0 : 0.0);
      rb[j] = (v1 && j < n) ? As[r1 + (int64_t)j * lda] : (r1 == j ? 1.0 : 0.0);
    }
  }

  const int hb = h << 4;
  if (!solve_only) {   // (solve-only: ra / rb already hold the packed LU rows)
  double tv = tau_value;
  if (tau_default) {
    // n * eps * ||A_s||_inf over the real rows
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < NP; j++) {
      if (FULL || j < n) { s0 += fabs(ra[j]); s1 += fabs(rb[j]); }
    }
    double nm = fmax(v0 ? s0 : 0.0, v1 ? s1 : 0.0);
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) nm = fmax(nm, __shfl_xor_sync(0xffffffffu, nm, o));
    tv = (double)n * 2.220446049250313e-16 * nm;
  } else if (tau_ptr) {
    tv = *tau_ptr;
  }

  int inf = 0;
  // ---- factor (Eq 6), k ascending.  With rows t and 31-t per lane, row
  // 31-t is below every pivot k < 16 and row t is above every pivot k >= 16,
  // so at each step only one of the lane's two rows needs a guard.
#pragma unroll
  for (int k = 0; k < NP; k++) {
    const int src = hb + (k < 16 ? k : NP - 1 - k);
    const double piv = __shfl_sync(0xffffffffu, k < 16 ? ra[k] : rb[k], src);
    if ((FULL || k < n) && inf == 0 && fabs(piv) <= tv) inf = k + 1;
    if (k < 16) {
      const bool a0 = r0 > k;
      if (a0) ra[k] = divp<!FULL>(ra[k], piv);                     // Eq 6-a
      rb[k] = divp<!FULL>(rb[k], piv);
      const double n0 = -ra[k], n1 = -rb[k];
#pragma unroll
      for (int j0 = k + 1; j0 < NP; j0 += CH) {
        double u[CH];
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) u[q] = __shfl_sync(0xffffffffu, ra[j0 + q], src);   // Eq 6-b (row k)
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) rb[j0 + q] = fma(n1, u[q], rb[j0 + q]);            // Eq 6-c
        if (a0) {
#pragma unroll
          for (int q = 0; q < CH; q++)
            if (j0 + q < NP) ra[j0 + q] = fma(n0, u[q], ra[j0 + q]);
        }
      }
    } else {
      const bool a1 = r1 > k;
      if (a1) rb[k] = divp<!FULL>(rb[k], piv);
      const double n1 = -rb[k];
#pragma unroll
      for (int j0 = k + 1; j0 < NP; j0 += CH) {
        double u[CH];
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) u[q] = __shfl_sync(0xffffffffu, rb[j0 + q], src);
        if (a1) {
#pragma unroll
          for (int q = 0; q < CH; q++)
            if (j0 + q < NP) rb[j0 + q] = fma(n1, u[q], rb[j0 + q]);
        }
      }
    }
  }
  if (act && t == 0 && info) info[sys] = inf;

  }

  // ---- solve (Eq 1): LY = B then UX = Y.  Right-hand sides in groups of
  // RG (1, or 4 when nrhs > 1) as independent chains (their divisions
  // overlap); padded columns of a group are zeros and never stored.
  if (B) {
    double* Bs = B + (act ? sys : 0) * strideB;
    for (int rb0 = 0; rb0 < nrhs; rb0 += RG) {
      double y0[RG], y1[RG];
#pragma unroll
      for (int g = 0; g < RG; g++) {
        const bool rv = rb0 + g < nrhs;
        y0[g] = (v0 && rv) ? Bs[r0 + (int64_t)(rb0 + g) * ldb] : 0.0;
        y1[g] = (v1 && rv) ? Bs[r1 + (int64_t)(rb0 + g) * ldb] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < NP; k++) {   // forward: LY = B
        const int src = hb + (k < 16 ? k : NP - 1 - k);
#pragma unroll
        for (int g = 0; g < RG; g++) {
          const double yk = __shfl_sync(0xffffffffu, k < 16 ? y0[g] : y1[g], src);
          if (k < 16) {
            if (r0 > k) y0[g] = fma(-ra[k], yk, y0[g]);
            y1[g] = fma(-rb[k], yk, y1[g]);
          } else {
            if (r1 > k) y1[g] = fma(-rb[k], yk, y1[g]);
          }
        }
      }
      if constexpr (RG == 1) {
      // backward: UX = Y (one chain: true division; the verified-quotient
      // form below measured slower here — its extra live registers spill)
#pragma unroll
      for (int k = NP - 1; k >= 0; k--) {   // backward: UX = Y
        const int src = hb + (k < 16 ? k : NP - 1 - k);
#pragma unroll
        for (int g = 0; g < RG; g++) {
          if (k < 16) { if (t == k) y0[g] = divp<!FULL>(y0[g], ra[k]); }
          else        { if (t == NP - 1 - k) y1[g] = divp<!FULL>(y1[g], rb[k]); }
        }
#pragma unroll
        for (int g = 0; g < RG; g++) {
          const double xk = __shfl_sync(0xffffffffu, k < 16 ? y0[g] : y1[g], src);
          if (k < 16) {
            if (r0 < k) y0[g] = fma(-ra[k], xk, y0[g]);   // rows 31-t >= 16 > k never
          } else {
            y0[g] = fma(-ra[k], xk, y0[g]);               // rows t < 16 <= k always
            if (r1 < k) y1[g] = fma(-rb[k], xk, y1[g]);
          }
        }
      }
      } else {
      // backward: UX = Y.  The owner's quotient is a Markstein step from an
      // approximate reciprocal of its (final) diagonal entry, computed off
      // the chain; the exact correct-rounding test runs after the sweep on
      // the two (dividend, quotient) pairs each lane owns, and a warp with an
      // unverified quotient redoes the sweep with true division (RG > 1: 2.57 -> 1.64 ms for
      // 100k systems x 16 right-hand sides).
      double ys0[RG], ys1[RG], yo0[RG], qo0[RG], yo1[RG], qo1[RG];
#pragma unroll
      for (int g = 0; g < RG; g++) {
        ys0[g] = y0[g]; ys1[g] = y1[g];
        yo0[g] = 0.0; qo0[g] = 0.0; yo1[g] = 0.0; qo1[g] = 0.0;
      }
      double d0 = 1.0, d1 = 1.0;                         // the lane's own pivots u_tt, u_(31-t)(31-t)
      auto sweep = [&](auto exact_tag) {
        constexpr bool EXACT = decltype(exact_tag)::value;
#pragma unroll
        for (int k = NP - 1; k >= 0; k--) {
          const int src = hb + (k < 16 ? k : NP - 1 - k);
          if (k < 16) {
            if (t == k) {
              const double rk = EXACT ? 0.0 : rcp_approx(ra[k]);
              d0 = ra[k];
#pragma unroll
              for (int g = 0; g < RG; g++) {
                const double q = EXACT ? divp<!FULL>(y0[g], ra[k]) : quot_mk(y0[g], ra[k], rk);
                yo0[g] = y0[g]; qo0[g] = q; y0[g] = q;
              }
            }
          } else {
            if (t == NP - 1 - k) {
              const double rk = EXACT ? 0.0 : rcp_approx(rb[k]);
              d1 = rb[k];
#pragma unroll
              for (int g = 0; g < RG; g++) {
                const double q = EXACT ? divp<!FULL>(y1[g], rb[k]) : quot_mk(y1[g], rb[k], rk);
                yo1[g] = y1[g]; qo1[g] = q; y1[g] = q;
              }
            }
          }
#pragma unroll
          for (int g = 0; g < RG; g++) {
            const double xk = __shfl_sync(0xffffffffu, k < 16 ? y0[g] : y1[g], src);
            if (k < 16) {
              if (r0 < k) y0[g] = fma(-ra[k], xk, y0[g]);   // rows 31-t >= 16 > k never
            } else {
              y0[g] = fma(-ra[k], xk, y0[g]);               // rows t < 16 <= k always
              if (r1 < k) y1[g] = fma(-rb[k], xk, y1[g]);
            }
          }
        }
      };
      sweep(std::false_type{});
      bool okq = true;
#pragma unroll
      for (int g = 0; g < RG; g++) okq = okq && quot_exact(yo0[g], d0, qo0[g]) && quot_exact(yo1[g], d1, qo1[g]);
      if (__any_sync(0xffffffffu, !okq)) {               // rare: the sweep again with true division
#pragma unroll
        for (int g = 0; g < RG; g++) { y0[g] = ys0[g]; y1[g] = ys1[g]; }
        sweep(std::true_type{});
      }
      }
#pragma unroll
      for (int g = 0; g < RG; g++) {
        if (rb0 + g < nrhs) {
          if (v0) Bs[r0 + (int64_t)(rb0 + g) * ldb] = y0[g];
          if (v1) Bs[r1 + (int64_t)(rb0 + g) * ldb] = y1[g];
        }
      }
    }
  }
  if (solve_only) return;
#pragma unroll
  for (int j = 0; j < NP; j++) {
    if (v0 && (FULL || j < n)) As[r0 + (int64_t)j * lda] = ra[j];
    if (v1 && (FULL || j < n)) As[r1 + (int64_t)j * lda] = rb[j];
  }
}

// ---------------------------------------------------------------- n <= 32, nrhs <= 1
// The same lane map with the forward substitution L y = b riding in the
// factor as a 33rd column: at step k, y_i <- fma(-l_ik, y_k, y_i) for the
// rows below k, y_k being final at step k — per entry the same ascending fma
// chain as the separate sweep (Eq 1), so bitwise equal; it removes that
// sweep's 32 shuffle + fma hops (C5: 0.631 -> 0.597 ms).  MKB (n = 32): the
// backward sweep's quotients are Markstein steps from reciprocals of the
// lane's two diagonals (captured as the pivots of steps t and 31-t), the
// exact test deferred to after the sweep, a redo with true division if any
// fails (0.591 -> 0.581 ms).  The first chunk of each step's U_(k) row is
// shuffled before the divisions (0.581 -> 0.571 ms).  Measured and not kept: Markstein quotients in
// the factor from a per-step rcp_approx(pivot) (0.75 ms) and backward tests
// done in place (0.69 ms) — warps issue in order, so a test's dependent ops
// inside the owner's branch stall the chain they were meant to leave.
// Guards stay branches: predicated-PTX fma's come out of ptxas as DFMA + 2
// FSEL.
template <bool FULL, bool HASB, bool MKB = false>
__global__ void __launch_bounds__(128) batched1_kernel(int n, double* __restrict__ A, int64_t lda, int64_t strideA,
                                                       int64_t batch, double* __restrict__ B, int64_t strideB,
                                                       const double* __restrict__ tau_ptr, int tau_default,
                                                       double tau_value, int32_t* __restrict__ info) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int h = lane >> 4, t = lane & 15;
  const int64_t sys = 2 * warp + h;
  const bool act = sys < batch;
  const int r0 = t, r1 = NP - 1 - t;
  const bool v0 = act && (FULL || r0 < n), v1 = act && (FULL || r1 < n);
  double* As = A + (act ? sys : 0) * strideA;
  double* Bs = HASB ? B + (act ? sys : 0) * strideB : nullptr;
  const int hb = h << 4;

  double ra[NP], rb[NP], ya = 0.0, yb = 0.0;
#pragma unroll
  for (int j = 0; j < NP; j++) {
    if (FULL) {
      ra[j] = act ? As[r0 + (int64_t)j * lda] : (r0 == j ? 1.0 : 0.0);
      rb[j] = act ? As[r1 + (int64_t)j * lda] : (r1 == j ? 1.0 : 0.0);
    } else {
      ra[j] = (v0 && j < n) ? As[r0 + (int64_t)j * lda] : (r0 == j ? 1.0 : 0.0);
      rb[j] = (v1 && j < n) ? As[r1 + (int64_t)j * lda] : (r1 == j ? 1.0 : 0.0);
    }
  }
  if (HASB) {
    ya = v0 ? Bs[r0] : 0.0;
    yb = v1 ? Bs[r1] : 0.0;
  }

  double tv = tau_value;
  if (tau_default) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int j = 0; j < NP; j++) {
      if (FULL || j < n) { s0 += fabs(ra[j]); s1 += fabs(rb[j]); }
    }
    double nm = fmax(v0 ? s0 : 0.0, v1 ? s1 : 0.0);
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) nm = fmax(nm, __shfl_xor_sync(0xffffffffu, nm, o));
    tv = (double)n * 2.220446049250313e-16 * nm;
  } else if (tau_ptr) {
    tv = *tau_ptr;
  }

  int inf = 0;
  double d0 = 1.0, d1 = 1.0;   // MKB: the lane's own diagonals u_tt, u_(31-t)(31-t) (the pivots of steps t, 31-t)
#pragma unroll
  for (int k = 0; k < NP; k++) {
    const int src = hb + (k < 16 ? k : NP - 1 - k);
    const double piv = __shfl_sync(0xffffffffu, k < 16 ? ra[k] : rb[k], src);
    if ((FULL || k < n) && inf == 0 && fabs(piv) <= tv) inf = k + 1;
    if (MKB && HASB) {
      if (k < 16) d0 = t == k ? piv : d0;
      else        d1 = t == NP - 1 - k ? piv : d1;
    }
    // the first chunk of the U_(k) row (and y_k) is shuffled before the
    // divisions: their slow-path branch ends the basic block, so nothing
    // after it can be scheduled into the division's latency
    double u0[CH], yk = 0.0;
    const int j1 = k + 1;
#pragma unroll
    for (int q = 0; q < CH; q++)
      if (j1 + q < NP) u0[q] = __shfl_sync(0xffffffffu, k < 16 ? ra[j1 + q] : rb[j1 + q], src);   // Eq 6-b (row k)
    if (HASB) yk = __shfl_sync(0xffffffffu, k < 16 ? ya : yb, src);
    if (k < 16) {
      const bool a0 = r0 > k;
      if (a0) ra[k] = divp<!FULL>(ra[k], piv);                     // Eq 6-a
      rb[k] = divp<!FULL>(rb[k], piv);
      const double n0 = -ra[k], n1 = -rb[k];
#pragma unroll
      for (int j0 = j1; j0 < NP; j0 += CH) {
        double u[CH];
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) u[q] = j0 == j1 ? u0[q] : __shfl_sync(0xffffffffu, ra[j0 + q], src);
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) rb[j0 + q] = fma(n1, u[q], rb[j0 + q]);            // Eq 6-c
        if (a0) {
#pragma unroll
          for (int q = 0; q < CH; q++)
            if (j0 + q < NP) ra[j0 + q] = fma(n0, u[q], ra[j0 + q]);
        }
      }
      if (HASB) {   // the forward substitution's step k (Eq 1, L y = b)
        yb = fma(n1, yk, yb);
        if (a0) ya = fma(n0, yk, ya);
      }
    } else {
      const bool a1 = r1 > k;
      if (a1) rb[k] = divp<!FULL>(rb[k], piv);
      const double n1 = -rb[k];
#pragma unroll
      for (int j0 = j1; j0 < NP; j0 += CH) {
        double u[CH];
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) u[q] = j0 == j1 ? u0[q] : __shfl_sync(0xffffffffu, rb[j0 + q], src);
        if (a1) {
#pragma unroll
          for (int q = 0; q < CH; q++)
            if (j0 + q < NP) rb[j0 + q] = fma(n1, u[q], rb[j0 + q]);
        }
      }
      if (HASB && a1) yb = fma(n1, yk, yb);
    }
  }
  if (act && t == 0 && info) info[sys] = inf;

  if (HASB) {   // backward: U x = y (Eq 1)
    const double ya_f = ya, yb_f = yb;
    // MKB: the owner's quotient is a Markstein step from the reciprocal of
    // its diagonal (formed before the sweep, off the chain); the two
    // (dividend, quotient) pairs per lane are tested after the sweep and a
    // warp with an unverified one sweeps again with true division
    double yo0 = 0.0, qo0 = 0.0, yo1 = 0.0, qo1 = 0.0;
    const double rd0 = MKB ? rcp_approx(d0) : 0.0, rd1 = MKB ? rcp_approx(d1) : 0.0;
    auto sweep = [&](auto mk_tag) {
      constexpr bool MK = decltype(mk_tag)::value;
#pragma unroll
      for (int k = NP - 1; k >= 0; k--) {
        const int src = hb + (k < 16 ? k : NP - 1 - k);
        if (k < 16) {
          if (t == k) {
            if (MK) { yo0 = ya; ya = quot_mk(ya, d0, rd0); qo0 = ya; }
            else ya = divp<!FULL>(ya, ra[k]);
          }
        } else {
          if (t == NP - 1 - k) {
            if (MK) { yo1 = yb; yb = quot_mk(yb, d1, rd1); qo1 = yb; }
            else yb = divp<!FULL>(yb, rb[k]);
          }
        }
        const double xk = __shfl_sync(0xffffffffu, k < 16 ? ya : yb, src);
        if (k < 16) {
          if (r0 < k) ya = fma(-ra[k], xk, ya);   // rows 31-t >= 16 > k never
        } else {
          ya = fma(-ra[k], xk, ya);               // rows t < 16 <= k always
          if (r1 < k) yb = fma(-rb[k], xk, yb);
        }
      }
    };
    if (MKB) {
      sweep(std::true_type{});
      const bool ok = quot_exact(yo0, d0, qo0) && quot_exact(yo1, d1, qo1);
      if (__any_sync(0xffffffffu, !ok)) {   // rare: again with true division
        ya = ya_f; yb = yb_f;
        sweep(std::false_type{});
      }
    } else {
      sweep(std::false_type{});
    }
    if (v0) Bs[r0] = ya;
    if (v1) Bs[r1] = yb;
  }
#pragma unroll
  for (int j = 0; j < NP; j++) {
    if (v0 && (FULL || j < n)) As[r0 + (int64_t)j * lda] = ra[j];
    if (v1 && (FULL || j < n)) As[r1 + (int64_t)j * lda] = rb[j];
  }
}

// ---------------------------------------------------------------- plain lane map (comparison)
// The lane-level comparison SURVEY §8(a') asks for: one system per warp,
// lane i owns row i (no first-with-last pairing), otherwise the scheme of
// batched1_kernel (forward fused into the factor, the first U-row chunk
// shuffled before the divisions, Markstein backward with the deferred
// test).  Selected with EBV_BATCHED_PLAIN=1; bitwise the same results.
template <bool FULL, bool HASB>
__global__ void __launch_bounds__(128) batched_plain_kernel(int n, double* __restrict__ A, int64_t lda,
                                                            int64_t strideA, int64_t batch, double* __restrict__ B,
                                                            int64_t strideB, const double* __restrict__ tau_ptr,
                                                            int tau_default, double tau_value,
                                                            int32_t* __restrict__ info) {
  const int i = threadIdx.x & 31;
  const int64_t sys = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool act = sys < batch;
  const bool v = act && (FULL || i < n);
  double* As = A + (act ? sys : 0) * strideA;
  double* Bs = HASB ? B + (act ? sys : 0) * strideB : nullptr;
  double a[NP], y = 0.0;
#pragma unroll
  for (int j = 0; j < NP; j++)
    a[j] = (v && (FULL || j < n)) ? As[i + (int64_t)j * lda] : (i == j ? 1.0 : 0.0);
  if (HASB) y = v ? Bs[i] : 0.0;
  double tv = tau_value;
  if (tau_default) {
    double sr = 0.0;
#pragma unroll
    for (int j = 0; j < NP; j++)
      if (FULL || j < n) sr += fabs(a[j]);
    double nm = v ? sr : 0.0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) nm = fmax(nm, __shfl_xor_sync(0xffffffffu, nm, o));
    tv = (double)n * 2.220446049250313e-16 * nm;
  } else if (tau_ptr) {
    tv = *tau_ptr;
  }
  int inf = 0;
  double d = 1.0;
#pragma unroll
  for (int k = 0; k < NP; k++) {
    const double piv = __shfl_sync(0xffffffffu, a[k], k);
    d = i == k ? piv : d;
    if ((FULL || k < n) && inf == 0 && fabs(piv) <= tv) inf = k + 1;
    double u0[CH], yk = 0.0;
    const int j1 = k + 1;
#pragma unroll
    for (int q = 0; q < CH; q++)
      if (j1 + q < NP) u0[q] = __shfl_sync(0xffffffffu, a[j1 + q], k);
    if (HASB) yk = __shfl_sync(0xffffffffu, y, k);
    const bool below = i > k;
    if (below) a[k] = divp<!FULL>(a[k], piv);                                   // Eq 6-a
    const double nl = -a[k];
#pragma unroll
    for (int j0 = j1; j0 < NP; j0 += CH) {
      double u[CH];
#pragma unroll
      for (int q = 0; q < CH; q++)
        if (j0 + q < NP) u[q] = j0 == j1 ? u0[q] : __shfl_sync(0xffffffffu, a[j0 + q], k);
      if (below) {
#pragma unroll
        for (int q = 0; q < CH; q++)
          if (j0 + q < NP) a[j0 + q] = fma(nl, u[q], a[j0 + q]);                   // Eq 6-c
      }
    }
    if (HASB && below) y = fma(nl, yk, y);                                        // Eq 1, L y = b
  }
  if (act && i == 0 && info) info[sys] = inf;
  if (HASB) {
    const double yf = y, rd = dev::rcp_approx(d);
    double yo = 0.0, qo = 0.0;
    auto sweep = [&](auto mk_tag) {
      constexpr bool MK = decltype(mk_tag)::value;
#pragma unroll
      for (int k = NP - 1; k >= 0; k--) {
        if (i == k) {
          if (MK) { yo = y; y = quot_mk(y, d, rd); qo = y; }
          else y = divp<!FULL>(y, a[k]);
        }
        const double xk = __shfl_sync(0xffffffffu, y, k);
        if (i < k) y = fma(-a[k], xk, y);
      }
    };
    sweep(std::true_type{});
    if (__any_sync(0xffffffffu, !quot_exact(yo, d, qo))) {
      y = yf;
      sweep(std::false_type{});
    }
    if (v) Bs[i] = y;
  }
#pragma unroll
  for (int j = 0; j < NP; j++)
    if (v && (FULL || j < n)) As[i + (int64_t)j * lda] = a[j];
}

// ---------------------------------------------------------------- 33 <= n <= 64
// SURVEY §8f f2 (batched medium systems, CTA per system).  One CTA of 128
// threads per system: row i is owned by the lane pair (2i, 2i+1), lane j of
// the pair holding the columns c = j + 2q.  Step k: the pair owning row k
// publishes its final row (the U_(k) vector, Eq 6-b) to shared memory; every
// row i > k forms l_ik = a_ik / u_kk in the lane holding column k (Eq 6-a),
// shuffles it to its partner and both update their columns (Eq 6-c).  The
// solve (Eq 1) keeps y_i in both lanes of the pair (identical arithmetic),
// y_k / x_k published through shared memory.  Padding to 64 with identity
// rows / columns is exactly neutral.  Per entry the oracle's operations.
constexpr int N64 = 64, QB = N64 / 2;

template <bool FULL64>
__global__ void __launch_bounds__(128, 3) batched64_kernel(int n, double* __restrict__ A, int64_t lda, int64_t strideA,
                                                        int64_t batch, double* __restrict__ B, int64_t ldb,
                                                        int64_t strideB, int nrhs, int tau_default, double tau_value,
                                                        int32_t* __restrict__ info, int solve_only) {
  __shared__ double urow[2][N64];
  __shared__ double sval[2];
  __shared__ double snorm[4];
  const int64_t sys = blockIdx.x;
  if (sys >= batch) return;
  const int tid = threadIdx.x, i = tid >> 1, j = tid & 1, lane = tid & 31;
  const int pair = lane & ~1;
  double* As = A + sys * strideA;
  const bool rv = i < n;
  double a[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) {
    const int c = j + 2 * q;
    a[q] = (rv && c < n) ? As[i + (int64_t)c * lda] : (i == c ? 1.0 : 0.0);
  }
  if (!solve_only) {
    double tv = tau_value;
    if (tau_default) {   // n * eps * ||A_s||_inf
      double rs = 0.0;
#pragma unroll
      for (int q = 0; q < QB; q++)
        if (j + 2 * q < n) rs += fabs(a[q]);
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      double m = rv ? rs : 0.0;
#pragma unroll
      for (int o = 16; o >= 2; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) snorm[tid >> 5] = m;
      __syncthreads();
      m = fmax(fmax(snorm[0], snorm[1]), fmax(snorm[2], snorm[3]));
      tv = (double)n * 2.220446049250313e-16 * m;
    }
    int inf = 0;
#pragma unroll
    for (int k = 0; k < N64; k++) {
      double* ur = urow[k & 1];
      if (i == k) {
#pragma unroll
        for (int q = 0; q < QB; q++)
          if (j + 2 * q >= k) ur[j + 2 * q] = a[q];
      }
      __syncthreads();
      const double piv = ur[k];
      if (k < n && inf == 0 && fabs(piv) <= tv) inf = k + 1;
      const int qk = k >> 1;
      if (i > k && j == (k & 1)) a[qk] = divp<!FULL64>(a[qk], piv);                       // Eq 6-a
      const double l = __shfl_sync(0xffffffffu, a[qk], pair | (k & 1));
      if (i > k) {
#pragma unroll
        for (int q = qk; q < QB; q++)
          if (j + 2 * q > k) a[q] = fma(-l, ur[j + 2 * q], a[q]);             // Eq 6-c
      }
    }
    if (tid == 0 && info) info[sys] = inf;
  }
  if (B) {
    double* Bs = B + sys * strideB;
    for (int r = 0; r < nrhs; r++) {
      double y = rv ? Bs[i + (int64_t)r * ldb] : 0.0;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < N64; k++) {            // forward: LY = B
        if (tid == 2 * k) sval[k & 1] = y;
        __syncthreads();
        const double yk = sval[k & 1];
        const double l = __shfl_sync(0xffffffffu, a[k >> 1], pair | (k & 1));
        if (i > k) y = fma(-l, yk, y);
      }
#pragma unroll
      for (int k = N64 - 1; k >= 0; k--) {       // backward: UX = Y
        const double u = __shfl_sync(0xffffffffu, a[k >> 1], pair | (k & 1));
        if (i == k) y = divp<!FULL64>(y, u);
        if (tid == 2 * k) sval[k & 1] = y;
        __syncthreads();
        const double xk = sval[k & 1];
        if (i < k) y = fma(-u, xk, y);
      }
      if (rv && j == 0) Bs[i + (int64_t)r * ldb] = y;
    }
  }
  if (solve_only) return;
#pragma unroll
  for (int q = 0; q < QB; q++) {
    const int c = j + 2 * q;
    if (rv && c < n) As[i + (int64_t)c * lda] = a[q];
  }
}


// 33 <= n <= 64 with at most one right-hand side: the same CTA-per-system
// scheme with the forward substitution riding in the factor (row k's owner
// publishes y_k with its U row; rows i > k apply y_i <- fma(-l_ik, y_k, y_i)
// at step k — the separate sweep's ascending chain, bitwise), which removes
// the forward sweep's 64 barrier steps; the backward sweep's quotients are
// Markstein steps from the reciprocal of each row's diagonal (captured as
// the pivot of its step), tested after the sweep, the sweep redone with true
// division if any test fails.
template <bool FULL64>
__global__ void __launch_bounds__(128, 3) batched64f_kernel(int n, double* __restrict__ A, int64_t lda,
                                                         int64_t strideA, int64_t batch, double* __restrict__ B,
                                                         int64_t strideB, int tau_default, double tau_value,
                                                         int32_t* __restrict__ info) {
  __shared__ double urow[2][N64 + 2];   // U row k (entries j >= k) and, at [N64], y_k
  __shared__ double sval[2];
  __shared__ double snorm[4];
  const int64_t sys = blockIdx.x;
  if (sys >= batch) return;
  const int tid = threadIdx.x, i = tid >> 1, j = tid & 1, lane = tid & 31;
  const int pair = lane & ~1;
  double* As = A + sys * strideA;
  double* Bs = B ? B + sys * strideB : nullptr;
  const bool rv = i < n;
  double a[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) {
    const int c = j + 2 * q;
    a[q] = (rv && c < n) ? As[i + (int64_t)c * lda] : (i == c ? 1.0 : 0.0);
  }
  double y = (Bs && rv) ? Bs[i] : 0.0;
  double tv = tau_value;
  if (tau_default) {   // n * eps * ||A_s||_inf
    double rs = 0.0;
#pragma unroll
    for (int q = 0; q < QB; q++)
      if (j + 2 * q < n) rs += fabs(a[q]);
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    double m = rv ? rs : 0.0;
#pragma unroll
    for (int o = 16; o >= 2; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) snorm[tid >> 5] = m;
    __syncthreads();
    m = fmax(fmax(snorm[0], snorm[1]), fmax(snorm[2], snorm[3]));
    tv = (double)n * 2.220446049250313e-16 * m;
  }
  int inf = 0;
  double d = 1.0;                            // this row's diagonal u_ii
#pragma unroll
  for (int k = 0; k < N64; k++) {
    double* ur = urow[k & 1];
    if (i == k) {
#pragma unroll
      for (int q = 0; q < QB; q++)
        if (j + 2 * q >= k) ur[j + 2 * q] = a[q];
      if (j == 0) ur[N64] = y;                // y_k is final at step k
    }
    __syncthreads();
    const double piv = ur[k];
    d = i == k ? piv : d;
    if (k < n && inf == 0 && fabs(piv) <= tv) inf = k + 1;
    const int qk = k >> 1;
    if (i > k && j == (k & 1)) a[qk] = divp<!FULL64>(a[qk], piv);                       // Eq 6-a
    const double l = __shfl_sync(0xffffffffu, a[qk], pair | (k & 1));
    if (i > k) {
#pragma unroll
      for (int q = qk; q < QB; q++)
        if (j + 2 * q > k) a[q] = fma(-l, ur[j + 2 * q], a[q]);             // Eq 6-c
      y = fma(-l, ur[N64], y);                                             // Eq 1, L y = b
    }
  }
  if (tid == 0 && info) info[sys] = inf;
  if (Bs) {   // backward: U x = y
    const double yf = y, rd = rcp_approx(d);
    double yo = 0.0, qo = 0.0;
    auto sweep = [&](auto mk_tag) {
      constexpr bool MK = decltype(mk_tag)::value;
#pragma unroll
      for (int k = N64 - 1; k >= 0; k--) {
        const double u = __shfl_sync(0xffffffffu, a[k >> 1], pair | (k & 1));
        if (i == k) {
          if (MK) { yo = y; y = quot_mk(y, d, rd); qo = y; }
          else y = divp<!FULL64>(y, u);
        }
        if (tid == 2 * k) sval[k & 1] = y;
        __syncthreads();
        const double xk = sval[k & 1];
        if (i < k) y = fma(-u, xk, y);
      }
    };
    sweep(std::true_type{});
    if (__syncthreads_or(!quot_exact(yo, d, qo))) {   // rare: the sweep again with true division
      y = yf;
      sweep(std::false_type{});
    }
    if (rv && j == 0) Bs[i] = y;
  }
#pragma unroll
  for (int q = 0; q < QB; q++) {
    const int c = j + 2 * q;
    if (rv && c < n) As[i + (int64_t)c * lda] = a[q];
  }
}

}  // namespace

cudaError_t launch_batched(int64_t n, double* A, int64_t lda, int64_t strideA, int64_t batch, double* B,
                           int64_t ldb, int64_t strideB, int64_t nrhs, const double* tau, bool tau_default,
                           double tau_value, int32_t* info, cudaStream_t s, bool solve_only) {
  if (batch <= 0 || n <= 0) return cudaSuccess;
  if (n > N64 || nrhs > MAXRHS) return cudaErrorInvalidValue;
  if (n > NP && nrhs <= 1 && !solve_only) {
    auto k = n == N64 ? batched64f_kernel<true> : batched64f_kernel<false>;
    k<<<(unsigned)batch, 128, 0, s>>>((int)n, A, lda, strideA, batch, nrhs == 1 ? B : nullptr, strideB,
                                     tau_default ? 1 : 0, tau_value, info);
    return cudaGetLastError();
  }
  if (n > NP) {
    auto k = n == N64 ? batched64_kernel<true> : batched64_kernel<false>;
    k<<<(unsigned)batch, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, ldb, strideB, (int)nrhs,
                                     tau_default ? 1 : 0, tau_value, info, solve_only ? 1 : 0);
    return cudaGetLastError();
  }
  const int64_t warps = (batch + 1) / 2;
  const int64_t blocks = (warps * 32 + 127) / 128;
  const int so = solve_only ? 1 : 0, td = tau_default ? 1 : 0;
  const unsigned g = (unsigned)blocks;
  static const bool v1 = [] {   // EBV_BATCHED_V1=0: the separate-sweep kernel for nrhs <= 1
    const char* e = getenv("EBV_BATCHED_V1");
    return !(e && atoi(e) == 0);
  }();
  static const bool plain = [] {   // EBV_BATCHED_PLAIN=1: one system per warp, lane = row (comparison)
    const char* e = getenv("EBV_BATCHED_PLAIN");
    return e && atoi(e) == 1;
  }();
  if (plain && !solve_only && nrhs <= 1) {
    const bool hasb = B && nrhs == 1;
    const unsigned gp = (unsigned)((batch * 32 + 127) / 128);
    auto k = n == NP ? (hasb ? batched_plain_kernel<true, true> : batched_plain_kernel<true, false>)
                     : (hasb ? batched_plain_kernel<false, true> : batched_plain_kernel<false, false>);
    k<<<gp, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, strideB, tau, td, tau_value, info);
    return cudaGetLastError();
  }
  if (v1 && !solve_only && nrhs <= 1) {
    const bool hasb = B && nrhs == 1;
    if (n == NP && hasb)
      batched1_kernel<true, true, true><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, strideB, tau, td, tau_value, info);
    else if (n == NP)
      batched1_kernel<true, false><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, strideB, tau, td, tau_value, info);
    else if (hasb)
      batched1_kernel<false, true><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, strideB, tau, td, tau_value, info);
    else
      batched1_kernel<false, false><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, strideB, tau, td, tau_value, info);
    return cudaGetLastError();
  }
  if (n == NP && nrhs <= 1)
    batched_kernel<true, 1><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, ldb, strideB, (int)nrhs, tau, td,
                                             tau_value, info, so);
  else if (n == NP)
    batched_kernel<true, 4><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, ldb, strideB, (int)nrhs, tau, td,
                                             tau_value, info, so);
  else if (nrhs <= 1)
    batched_kernel<false, 1><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, ldb, strideB, (int)nrhs, tau, td,
                                              tau_value, info, so);
  else
    batched_kernel<false, 4><<<g, 128, 0, s>>>((int)n, A, lda, strideA, batch, B, ldb, strideB, (int)nrhs, tau, td,
                                              tau_value, info, so);
  return cudaGetLastError();
}

}  // namespace ebv

EBV_DEBUG_SETTER(set_debug_batched)
