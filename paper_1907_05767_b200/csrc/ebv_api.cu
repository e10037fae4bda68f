// ebv_api.cu — the C ABI of libebv.so (include/ebv.h): argument validation,
// context / workspace management, the recursive blocked schedule and the
// measurement hooks.  All arithmetic happens in the kernels (k_*.cu).
//
// Blocked schedule (EBV_PATH_BLOCKED): the Eq 6 recurrences applied
// to a 2 x 2 block partition, recursively:
//     LU(A11);  L21 = A21 U11^-1;  U12 = L11^-1 A12;  A22 -= L21 U12;  LU(A22)
// The triangular solves recurse the same way (X2 -= X1 U12 between the two
// halves), so every flop outside the <= 64 x 64 leaves is a DMMA contraction
// with a long k range, and every entry still sees its updates in ascending k
// followed by its division (bitwise equal to the serial oracle).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ebv_device.cuh"
#include "ebv_sched.cuh"

namespace ebv {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ebv

using namespace ebv;
using namespace ebv::sched;

namespace ebv {
namespace sched {


ebv_status_t cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return EBV_ERR_CUDA;
}

ebv_status_t invalid(const char* msg) {
  set_error(msg);
  return EBV_ERR_INVALID_VALUE;
}

cudaEvent_t get_event(ebv_context* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

cudaError_t gemm(ebv_context* c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                 int64_t ldb, double* C, int64_t ldc, bool rev, cudaStream_t s, int cls) {
  if (M <= 0 || N <= 0 || K <= 0) return cudaSuccess;
  double fl = 2.0 * M * N * K, by = 8.0 * (M * K + K * N + 2.0 * M * N);
  return timed(c, cls, fl, by, s, 1, [&] { return launch_gemm_sub(M, N, K, A, lda, B, ldb, C, ldc, rev, s); });
}

int64_t split_point(int64_t n, int64_t leaf) {
  int64_t h = ((n / 2 + leaf - 1) / leaf) * leaf;
  if (h >= n) h = n - leaf;
  if (h <= 0) h = n / 2;
  return h;
}

// X (m x k) <- X U^-1, U upper k x k
cudaError_t trsm_r(ebv_context* c, int64_t m, int64_t k, double* X, int64_t ldx, const double* U, int64_t ldu,
                   cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k <= c->leaf) {
    double fl = (double)m * k * k, by = 16.0 * m * k + 8.0 * k * k / 2;
    return timed(c, KC_TRSM, fl, by, s, 1, [&] { return launch_trsm_right_upper(m, k, X, ldx, U, ldu, s); });
  }
  int64_t h = split_point(k, c->leaf);
  cudaError_t e = trsm_r(c, m, h, X, ldx, U, ldu, s);
  if (e != cudaSuccess) return e;
  e = gemm(c, m, k - h, h, X, ldx, U + h * ldu, ldu, X + h * ldx, ldx, false, s);
  if (e != cudaSuccess) return e;
  return trsm_r(c, m, k - h, X + h * ldx, ldx, U + h + h * ldu, ldu, s);
}

// X (k x m) <- L^-1 X, L unit lower k x k
cudaError_t trsm_l(ebv_context* c, int64_t k, int64_t m, const double* L, int64_t ldl, double* X, int64_t ldx,
                   cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k <= c->leaf) {
    double fl = (double)m * k * k, by = 16.0 * m * k + 8.0 * k * k / 2;
    return timed(c, KC_TRSM, fl, by, s, 1, [&] { return launch_trsm_left_lower_unit(k, m, L, ldl, X, ldx, s); });
  }
  int64_t h = split_point(k, c->leaf);
  cudaError_t e = trsm_l(c, h, m, L, ldl, X, ldx, s);
  if (e != cudaSuccess) return e;
  e = gemm(c, k - h, m, h, L + h, ldl, X, ldx, X + h, ldx, false, s);
  if (e != cudaSuccess) return e;
  return trsm_l(c, k - h, m, L + h + h * ldl, ldl, X + h, ldx, s);
}

// X (k x m) <- U^-1 X, U upper (non-unit) k x k: backward substitution per
// column, k descending (the bottom block first, then the rows above it are
// updated by a reverse-k DMMA update).
cudaError_t trsm_lu(ebv_context* c, int64_t k, int64_t m, const double* U, int64_t ldu, double* X, int64_t ldx,
                    cudaStream_t s) {
  if (m <= 0 || k <= 0) return cudaSuccess;
  if (k <= c->leaf) {
    double fl = (double)m * k * k, by = 16.0 * m * k + 8.0 * k * k / 2;
    return timed(c, KC_TRSM, fl, by, s, 1, [&] { return launch_trsm_left_upper(k, m, U, ldu, X, ldx, s); });
  }
  int64_t h = split_point(k, c->leaf);
  cudaError_t e = trsm_lu(c, k - h, m, U + h + h * ldu, ldu, X + h, ldx, s);
  if (e != cudaSuccess) return e;
  e = gemm(c, h, m, k - h, U + h * ldu, ldu, X + h, ldx, X, ldx, true, s);
  if (e != cudaSuccess) return e;
  return trsm_lu(c, h, m, U, ldu, X, ldx, s);
}

// Fully recursive schedule (EBV_BLOCK_RECURSIVE):
//     LU(A11);  L21 = A21 U11^-1;  U12 = L11^-1 A12;  A22 -= L21 U12;  LU(A22)
cudaError_t lu_rec(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t koff, int64_t* info, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n <= c->leaf) {
    double fl = 2.0 / 3.0 * n * n * n, by = 16.0 * n * n;
    return timed(c, KC_LEAF, fl, by, s, 1, [&] { return launch_leaf_lu(n, A, lda, c->d_tau, info, koff, s); });
  }
  int64_t h = split_point(n, c->leaf);
  cudaError_t e = lu_rec(c, h, A, lda, koff, info, s);
  if (e != cudaSuccess) return e;
  e = trsm_r(c, n - h, h, A + h, lda, A, lda, s);                      // L21 = A21 U11^-1
  if (e != cudaSuccess) return e;
  e = trsm_l(c, h, n - h, A, lda, A + h * lda, lda, s);                // U12 = L11^-1 A12
  if (e != cudaSuccess) return e;
  e = gemm(c, n - h, n - h, h, A + h, lda, A + h * lda, lda, A + h + h * lda, lda, false, s);  // A22 -= L21 U12
  if (e != cudaSuccess) return e;
  return lu_rec(c, n - h, A + h + h * lda, lda, koff + h, info, s);
}

// LU of a tall panel P (M x w, M >= w) in place: its w x w top block becomes
// L11\U11 and the rows below become L21 (Eq 6 restricted to the w steps of
// the panel).  Recursive on the panel width; the leaves fuse nothing but are
// a diagonal-block LU (one CTA) + a row-parallel L21 = A21 U11^-1.
// Solve path: interleaved wavefront chains (one launch per sweep per 64
// columns) vs recursive TRSM with DMMA updates (flat in nrhs, latency-bound
// by its ~n/32 launches).  Crossovers measured on B200
// (profiles/r01_solve_rhs_sweep.jsonl): n = 8192: wavefront 5.6 ms at 64
// columns vs TRSM 12.5; n = 32768: 42 vs 56 ms at 32 columns, 79 vs 58 at 64.
static int64_t kSolveTrsmRhs = [] {
  const char* e = getenv("EBV_SOLVE_TRSM_RHS");
  return e ? (int64_t)atoll(e) : (int64_t)0;
}();
// EBV_SOLVE_CHAIN=0 selects the wavefront kernel (k_solve.cu) instead of the
// chain-pipelined one (k_solve2.cu) for the non-TRSM solves
static int kSolveChain = [] {
  const char* e = getenv("EBV_SOLVE_CHAIN");
  return e ? atoi(e) : 1;
}();
static bool solve_use_trsm(int64_t n, int64_t nrhs, bool chain) {
  if (kSolveTrsmRhs > 0) return nrhs >= kSolveTrsmRhs;
  // against the chain kernel (16 columns per launch, ~0.9 ms per group at
  // n = 8192, ~8.9 ms at n = 32768; TRSM ~12.5 / ~55 ms flat:
  // profiles/r02_solve_chain_many.jsonl, r02_solve_trsm_many.jsonl)
  if (chain) return nrhs > 192 || (n > 12288 && nrhs > 96);
  // against the wavefront kernel (profiles/r01_solve_rhs_sweep.jsonl)
  return nrhs > 128 || (n > 8192 && nrhs > 64) || (n > 16384 && nrhs > 40);
}

static int64_t kU12SplitRows = [] {
  const char* e = getenv("EBV_U12_SPLIT_ROWS");
  return e ? (int64_t)atoll(e) : (int64_t)-1;   // -1: split for n >= 16384 (same-box A/B:
}();                                              // n = 32768 -0.3%, n = 8192 +3% if split)

// streamed host factor plan: PCIe copy rate and DMMA update rate (B200)
static const double kHostCopyBps = 55e9, kUpdateFlops = 33e12;

// U12 lookahead (EBV_U12_LA: -1 auto = n >= 8192 here, n >= 16384 in the
// distributed schedule; 0 off, 1 on): step K
// updates block row K+1 first, and the side stream computes U12 of step K+1
// (after panel K+1) while the main stream updates the rows below; see
// lu_blocked.
static int kU12La = [] {
  const char* e = getenv("EBV_U12_LA");
  return e ? atoi(e) : -1;
}();

// round 2 (with the blocked panel leaf): 6144 — n = 16384 96.7 -> 95.7 ms,
// n = 32768 703.2 -> 701.4 ms (4096: 96.1 / 702.1; 12288 no gain)
static int64_t kTailRows = [] {
  const char* e = getenv("EBV_TAIL_ROWS");
  return e ? (int64_t)atoll(e) : (int64_t)6144;
}();

// panels up to this many rows take the fused panel-leaf kernel (round 2,
// with the graph replay keeping the side stream's priority: 4096 measured
// best — n = 8192 16.76 vs 17.26 ms at 8192, n = 32768 707.5 vs 709.1;
// profiles/r02_panel_fused_rows.txt)
static int64_t kPanelLeafFusedRows = [] {
  const char* e = getenv("EBV_PANEL_FUSED_ROWS");
  return e ? (int64_t)atoll(e) : (int64_t)4096;
}();

cudaError_t panel_rec(ebv_context* c, int64_t M, int64_t w, double* P, int64_t lda, int64_t koff, int64_t* info,
                      cudaStream_t s) {
  if (w <= 0) return cudaSuccess;
  if (w <= c->leaf) {
    // short panels: diagonal block LU and the rows below in one launch (each
    // CTA factors the diagonal block itself); tall panels: one CTA for the
    // diagonal block, then the rows below with few, fat CTAs — the panel
    // runs beside the DMMA update, so its SM-time is what it costs there
    if (M <= kPanelLeafFusedRows) {
      double fl = 2.0 / 3.0 * w * w * w + (double)(M - w) * w * w, by = 16.0 * M * w;
      return timed(c, KC_LEAF, fl, by, s, 1,
                   [&] { return launch_panel_leaf(M, w, P, lda, c->d_tau, info, koff, c->d_pcount, s); });
    }
    double fl = 2.0 / 3.0 * w * w * w, by = 16.0 * w * w;
    cudaError_t e = timed(c, KC_LEAF, fl, by, s, 1, [&] { return launch_leaf_lu(w, P, lda, c->d_tau, info, koff, s); });
    if (e != cudaSuccess) return e;
    return trsm_r(c, M - w, w, P + w, lda, P, lda, s);
  }
  int64_t h = split_point(w, c->leaf);
  cudaError_t e = panel_rec(c, M, h, P, lda, koff, info, s);
  if (e != cudaSuccess) return e;
  e = trsm_l(c, h, w - h, P, lda, P + h * lda, lda, s);
  if (e != cudaSuccess) return e;
  e = gemm(c, M - h, w - h, h, P + h, lda, P + h * lda, lda, P + h + h * lda, lda, false, s);
  if (e != cudaSuccess) return e;
  return panel_rec(c, M - h, w - h, P + h + h * lda, lda, koff + h, info, s);
}

// Right-looking blocked schedule (default): for each column block K of width
// nb — the block form of the step-k recurrences of Eq 6:
//     panel LU of A[K:, K]          (L_(k), U_(k) vectors of the block's steps)
//     U12 = L11^-1 A[K, K+1:]        (the U_(k) rows to the right)
//     A[K+1:, K+1:] -= L21 U12       (Eq 6-c for the nb steps at once, DMMA)
// This is also the per-step structure of the 1D block-cyclic multi-GPU
// schedule (only the owner of block K factors the panel).
// Block width: the caller's choice, else size-adaptive (measured on B200:
// 64 up to n = 4096, 128 at 8192, 256 at 16384, 512 at 32768;
// profiles/r01_sweep_nb*.jsonl).
int64_t block_width(const ebv_context* c, int64_t n) {
  if (c->nb > 0) return c->nb;
  int64_t nb = n >= 24576 ? 512 : (n >= 12288 ? 256 : (n >= 6144 ? 128 : 64));
  return ((nb + c->leaf - 1) / c->leaf) * c->leaf;
}

// Width of the column block starting at c0.  EBV_TAIL_ROWS=t narrows the
// panels to 128 once fewer than t rows remain (the tail, where the panel
// chain is exposed); round 1 measured no gain with the column-step leaf,
// round 2 with the blocked leaf 0.3-1% (default 6144); widths adapted to
// the whole remaining order were 1% slower.  Any sequence of widths keeps
// every entry's operation order (bitwise the same factors).
static int64_t step_width(const ebv_context* c, int64_t n, int64_t c0) {
  const int64_t nb = block_width(c, n);
  const int64_t w = (c->nb > 0 || n - c0 > kTailRows) ? nb : (nb < 128 ? nb : 128);
  return (n - c0) < w ? (n - c0) : w;
}

// kl / ku (banded inputs): entries with i - j > kl or
// j - i > ku are zero and stay zero under no-pivot LU (Golub & Van Loan
// Thm 4.3.1), so the panel, U12 and the update are clipped to the band —
// the skipped operations of the dense algorithm are exact no-ops on zeros
// (fma(-0, u, +0) == +0), so the factors inside the band are bitwise the
// dense ones.  kl = ku = n - 1 is the dense schedule.
cudaError_t lu_blocked(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t* info, cudaStream_t s,
                       int64_t kl, int64_t ku, bool band_storage) {
  if (kl < 0 || kl > n) kl = n;
  if (ku < 0 || ku > n) ku = n;
  // narrow bands: 64-wide panels (the per-step windows are ~band-sized;
  // measured n = 65536, kl = ku = 256: 61.8 ms at nb = 64, 98.9 at 512).
  // Compact band storage always takes 64-wide steps: its padding
  // (EBV_BAND_PAD) covers how far a 64-column step reaches past the band.
  const bool narrow = band_storage || (c->nb <= 0 && kl + ku < n / 4);
  const int64_t nb = narrow ? ((64 + c->leaf - 1) / c->leaf) * c->leaf : block_width(c, n);
  auto step_w = [&](int64_t c0) { return narrow ? ((n - c0) < nb ? (n - c0) : nb) : step_width(c, n, c0); };
  const bool la = c->lookahead && n > 2 * nb;
  cudaError_t e = cudaSuccess;
  if (la) {
    // the side stream starts after everything already queued on the caller's
    e = cudaEventRecord(c->ev_start, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_start, 0);
    if (e != cudaSuccess) return e;
  }
  auto clip = [](int64_t a, int64_t b) { return a < b ? a : b; };
  const bool u12la = la && (kU12La >= 0 ? kU12La != 0 : n >= 8192);
  bool u12_done = false;   // U12 of the current step was solved on the side stream
  {
    const int64_t w0 = step_w(0);
    e = panel_rec(c, clip(n, w0 + kl), w0, A, lda, 0, info, s);
    if (e != cudaSuccess) return e;
  }
  for (int64_t c0 = 0, w = 0; c0 < n; c0 += w) {
    w = step_w(c0);
    double* P = A + c0 + c0 * lda;
    const int64_t rest = n - c0 - w;
    if (rest <= 0) break;
    if (la && c0 > 0) {   // panel K (factored on the side stream) must be complete
      e = cudaStreamWaitEvent(s, c->ev_p, 0);
      if (e != cudaSuccess) return e;
    }
    const int64_t Mb = clip(rest, kl), Nbw = clip(rest, ku);   // nonzero L21 rows / U12 columns
    const int64_t w1 = step_w(c0 + w);              // width of panel K+1
    const int64_t Mp1 = clip(rest, w1 + kl);         // its rows that can be nonzero
    double* P1 = P + w + w * lda;
    if (la && Nbw > w1) {
      // lookahead: the update of panel K+1's columns first, then factor it on
      // the side stream while the rest of the trailing matrix is updated.
      // For large n U12 is split too, so panel K+1 need not wait for all of
      // U12 (columns are independent: same bits).  With the U12 lookahead,
      // U12 of this step was already computed on the side stream, and this
      // step updates block row K+1 (the rows U12 of step K+1 is solved
      // from) before the rows below, so the side stream solves U12 of step
      // K+1 while the main stream updates the rest: the U12 solves leave the
      // main stream's critical path.  Every entry still receives the same
      // updates in the same order (row / column splits of one update do not
      // change any entry's fma chain): bitwise the same factors.
      const bool split = kU12SplitRows >= 0 ? rest < kU12SplitRows : n >= 16384;
      if (!u12_done) e = trsm_l(c, w, split ? w1 : Nbw, P, lda, P + w * lda, lda, s);
      if (e == cudaSuccess) e = gemm(c, Mb, w1, w, P + w, lda, P + w * lda, lda, P1, lda, false, s, KC_UPDATE);
      if (e == cudaSuccess) e = cudaEventRecord(c->ev_a, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_a, 0);
      if (e == cudaSuccess) e = panel_rec(c, Mp1, w1, P1, lda, c0 + w, info, c->side);
      if (e == cudaSuccess && split && !u12_done) e = trsm_l(c, w, Nbw - w1, P, lda, P + (w + w1) * lda, lda, s);
      // the next step: its panel width, U12 columns and whether it takes this branch
      const int64_t rest1 = rest - w1;
      const int64_t w2 = rest1 > 0 ? step_w(c0 + w + w1) : 0;
      const int64_t Nbw1 = clip(rest1, ku);
      const bool next_la = rest1 > 0 && Nbw1 > w2;
      if (e == cudaSuccess && u12la && next_la && Mb > w1) {
        const int64_t w1r = w1;                       // block row K+1 (Mb > w1 rows exist)
        e = gemm(c, w1r, Nbw - w1, w, P + w, lda, P + (w + w1) * lda, lda, P1 + w1 * lda, lda, false, s, KC_UPDATE);
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_b, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_b, 0);
        if (e == cudaSuccess) e = trsm_l(c, w1, Nbw1, P1, lda, P1 + w1 * lda, lda, c->side);   // U12 of step K+1
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_p, c->side);
        if (e == cudaSuccess)
          e = gemm(c, Mb - w1r, Nbw - w1, w, P + w + w1r, lda, P + (w + w1) * lda, lda, P1 + w1r + w1 * lda, lda,
                   false, s, KC_UPDATE);
        u12_done = true;
      } else {
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_p, c->side);
        if (e == cudaSuccess)
          e = gemm(c, Mb, Nbw - w1, w, P + w, lda, P + (w + w1) * lda, lda, P1 + w1 * lda, lda, false, s, KC_UPDATE);
        u12_done = false;
      }
      if (e != cudaSuccess) return e;
    } else {
      if (!u12_done) e = trsm_l(c, w, Nbw, P, lda, P + w * lda, lda, s);
      u12_done = false;
      if (e != cudaSuccess) return e;
      e = gemm(c, Mb, Nbw, w, P + w, lda, P + w * lda, lda, P1, lda, false, s, KC_UPDATE);
      if (e != cudaSuccess) return e;
      if (la) {   // keep the event protocol: the next panel is factored in order
        e = panel_rec(c, Mp1, w1, P1, lda, c0 + w, info, s);
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_p, s);
      } else {
        e = panel_rec(c, Mp1, w1, P1, lda, c0 + w, info, s);
      }
      if (e != cudaSuccess) return e;
    }
  }
  if (la) {   // the caller's stream sees the last side-stream work
    e = cudaEventRecord(c->ev_p, c->side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, c->ev_p, 0);
  }
  return e;
}

// Right-looking schedule over a HOST-resident matrix (ebv_lu_factor_host):
// the column blocks are copied in order on a copy stream, and block J
// joins the right-looking updates at step K_J — planned from the copy rate
// and the update flop rate so that it has arrived by then — after a
// catch-up that applies steps 0..K_J-1 to it in order (trsm with each
// panel's L11, then its DMMA update): per entry the same operation sequence
// as lu_blocked, bitwise.  Until then the steps' updates cover only the
// blocks already joined, so the transfer overlaps the first steps' work.
// A block that arrives later than planned only stalls the stream (its
// catch-up waits on its copy event); correctness never depends on timing.
cudaError_t lu_blocked_stream(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t* info, cudaStream_t s,
                              const double* hA, int64_t ldh) {
  const int64_t nb = block_width(c, n);
  const int64_t N = (n + nb - 1) / nb;
  auto wid = [&](int64_t J) { return (J + 1) * nb <= n ? nb : n - J * nb; };
  cudaError_t e = cudaSuccess;
  if (!c->copy) {
    e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
  }
  while ((int64_t)c->copy_ev.size() < N) {
    cudaEvent_t ev = nullptr;
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    c->copy_ev.push_back(ev);
  }
  e = cudaEventRecord(c->ev_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->copy, c->ev_start, 0);
  for (int64_t J = 0; J < N && e == cudaSuccess; J++) {
    e = cudaMemcpy2DAsync(A + J * nb * lda, lda * sizeof(double), hA + J * nb * ldh, ldh * sizeof(double),
                          n * sizeof(double), wid(J), cudaMemcpyHostToDevice, c->copy);
    if (e == cudaSuccess) e = cudaEventRecord(c->copy_ev[J], c->copy);
  }
  if (e != cudaSuccess) return e;
  // join plan: block J (copied by ~ (J+1) * t_copy) joins at the first step
  // whose start (cumulative update time) is later; never after step J-1
  const double t_copy = (double)n * nb * 8.0 / kHostCopyBps, rate = kUpdateFlops;
  std::vector<int64_t> join(N, 0);
  {
    std::vector<double> T(N + 1, 0.0);
    for (int64_t k = 0; k < N; k++) {
      const double rest = (double)(n - (k + 1) * nb);
      T[k + 1] = T[k] + (rest > 0 ? 2.0 * rest * rest * nb / rate : 0.0);
    }
    for (int64_t J = 2; J < N; J++) {
      int64_t K = 0;
      while (K < J - 1 && T[K] < (double)(J + 1) * t_copy) K++;
      join[J] = K < join[J - 1] ? join[J - 1] : K;   // nondecreasing: joined blocks form a prefix
    }
  }
  const bool la = c->lookahead && n > 2 * nb;
  if (la) {
    e = cudaEventRecord(c->ev_start, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_start, 0);
    if (e != cudaSuccess) return e;
  }
  e = cudaStreamWaitEvent(s, c->copy_ev[0], 0);
  if (e == cudaSuccess) e = panel_rec(c, n, wid(0), A, lda, 0, info, s);
  if (e != cudaSuccess) return e;
  int64_t joined = N > 1 ? 2 : 1;                     // blocks [0, joined) take part in the updates
  for (int64_t J = 1; J < joined; J++) {
    e = cudaStreamWaitEvent(s, c->copy_ev[J], 0);
    if (e != cudaSuccess) return e;
  }
  for (int64_t K = 0; K + 1 < N; K++) {
    const int64_t c0 = K * nb, w = wid(K);
    double* P = A + c0 + c0 * lda;
    const int64_t rest = n - c0 - w;
    // blocks joining at this step: wait for them, then catch up steps 0..K-1
    int64_t jn = joined;
    while (jn < N && join[jn] <= K) jn++;
    if (jn > joined) {
      for (int64_t J = joined; J < jn; J++) {
        e = cudaStreamWaitEvent(s, c->copy_ev[J], 0);
        if (e != cudaSuccess) return e;
      }
      const int64_t x0 = joined * nb, xn = (jn * nb < n ? jn * nb : n) - x0;   // their columns
      for (int64_t k = 0; k < K; k++) {
        const int64_t ck = k * nb, wk = wid(k);
        double* Pk = A + ck + ck * lda;
        e = trsm_l(c, wk, xn, Pk, lda, A + ck + x0 * lda, lda, s);
        if (e == cudaSuccess)
          e = gemm(c, n - ck - wk, xn, wk, Pk + wk, lda, A + ck + x0 * lda, lda, A + ck + wk + x0 * lda, lda, false,
                   s, KC_UPDATE);
        if (e != cudaSuccess) return e;
      }
      joined = jn;
    }
    if (la && c0 > 0) {   // panel K (factored on the side stream) must be complete
      e = cudaStreamWaitEvent(s, c->ev_p, 0);
      if (e != cudaSuccess) return e;
    }
    const int64_t ncols = (joined * nb < n ? joined * nb : n) - (c0 + w);   // joined trailing columns
    const int64_t w1 = wid(K + 1);
    double* P1 = P + w + w * lda;
    e = trsm_l(c, w, ncols, P, lda, P + w * lda, lda, s);
    if (e != cudaSuccess) return e;
    if (la && ncols > w1) {
      e = gemm(c, rest, w1, w, P + w, lda, P + w * lda, lda, P1, lda, false, s, KC_UPDATE);
      if (e == cudaSuccess) e = cudaEventRecord(c->ev_a, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_a, 0);
      if (e == cudaSuccess) e = panel_rec(c, rest, w1, P1, lda, c0 + w, info, c->side);
      if (e == cudaSuccess) e = cudaEventRecord(c->ev_p, c->side);
      if (e == cudaSuccess)
        e = gemm(c, rest, ncols - w1, w, P + w, lda, P + (w + w1) * lda, lda, P1 + w1 * lda, lda, false, s, KC_UPDATE);
      if (e != cudaSuccess) return e;
    } else {
      e = gemm(c, rest, ncols, w, P + w, lda, P + w * lda, lda, P1, lda, false, s, KC_UPDATE);
      if (e == cudaSuccess) e = panel_rec(c, rest, w1, P1, lda, c0 + w, info, s);
      if (e == cudaSuccess && la) e = cudaEventRecord(c->ev_p, s);
      if (e != cudaSuccess) return e;
    }
  }
  if (la) {
    e = cudaEventRecord(c->ev_p, c->side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, c->ev_p, 0);
  }
  return e;
}

// Left-looking schedule (EBV_PATH_LEFT, and ebv_lu_factor_host): column
// block J receives all earlier panels' updates when its turn comes —
//     X[0:c]   = L[0:c, 0:c]^-1 X[0:c]      (U rows of block J, trsm)
//     X[c:n]  -= L[c:n, 0:c] X[0:c]         (one DMMA update, K = c)
// then its panel is factored.  Per entry the same fma chain over ascending k
// and the same division as the right-looking schedule (bitwise the oracle).
// Lookahead: block J's update by panels 0..J-2 runs on the caller's stream
// while panel J-1 is factored on the side stream; only the update by panel
// J-1 (a w x w trsm and a K = nb update) waits for it.  With hA != NULL the
// column blocks are copied from host memory on a copy stream, block J+1's
// copy overlapping block J's work: the factorization of a host-resident
// matrix hides all but the first block's transfer.
cudaError_t lu_left(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t* info, cudaStream_t s,
                    const double* hA, int64_t ldh) {
  const int64_t nb = block_width(c, n);
  const int64_t N = (n + nb - 1) / nb;
  cudaError_t e = cudaSuccess;
  if (hA) {
    if (!c->copy) {
      e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    while ((int64_t)c->copy_ev.size() < N) {
      cudaEvent_t ev = nullptr;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
      c->copy_ev.push_back(ev);
    }
    // the copies start after the caller's earlier work on A
    e = cudaEventRecord(c->ev_start, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->copy, c->ev_start, 0);
    for (int64_t J = 0; J < N && e == cudaSuccess; J++) {
      const int64_t c0 = J * nb, w = (n - c0) < nb ? (n - c0) : nb;
      e = cudaMemcpy2DAsync(A + c0 * lda, lda * sizeof(double), hA + c0 * ldh, ldh * sizeof(double),
                            n * sizeof(double), w, cudaMemcpyHostToDevice, c->copy);
      if (e == cudaSuccess) e = cudaEventRecord(c->copy_ev[J], c->copy);
    }
    if (e != cudaSuccess) return e;
  }
  e = cudaEventRecord(c->ev_start, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_start, 0);
  if (e != cudaSuccess) return e;
  for (int64_t J = 0; J < N; J++) {
    const int64_t c0 = J * nb, w = (n - c0) < nb ? (n - c0) : nb;
    double* X = A + c0 * lda;
    if (hA) {
      e = cudaStreamWaitEvent(s, c->copy_ev[J], 0);
      if (e != cudaSuccess) return e;
    }
    if (J >= 1) {
      const int64_t cp = c0 - nb;                       // panel J-1 = columns [cp, c0)
      if (cp > 0) {                                     // panels 0..J-2
        e = trsm_l(c, cp, w, A, lda, X, lda, s);
        if (e == cudaSuccess) e = gemm(c, n - cp, w, cp, A + cp, lda, X, lda, X + cp, lda, false, s, KC_UPDATE);
        if (e != cudaSuccess) return e;
      }
      e = cudaStreamWaitEvent(s, c->ev_p, 0);          // panel J-1 factored (side stream)
      if (e == cudaSuccess) e = trsm_l(c, nb, w, A + cp + cp * lda, lda, X + cp, lda, s);
      if (e == cudaSuccess)
        e = gemm(c, n - c0, w, nb, A + c0 + cp * lda, lda, X + cp, lda, X + c0, lda, false, s, KC_UPDATE);
      if (e != cudaSuccess) return e;
    }
    e = cudaEventRecord(c->ev_a, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_a, 0);
    if (e == cudaSuccess) e = panel_rec(c, n - c0, w, A + c0 + c0 * lda, lda, c0, info, c->side);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_p, c->side);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamWaitEvent(s, c->ev_p, 0);           // the caller's stream sees the last panel
}

}  // namespace sched
}  // namespace ebv

namespace {

ebv_status_t ensure_flags(ebv_context* c, int64_t need) {
  if (need <= c->flags_cap) return EBV_SUCCESS;
  if (c->d_flags) cudaFree(c->d_flags);
  c->d_flags = nullptr;
  cudaError_t e = cudaMalloc(&c->d_flags, need * sizeof(int));
  if (e != cudaSuccess) { c->flags_cap = 0; set_error("workspace alloc failed"); return EBV_ERR_ALLOC; }
  e = cudaMemset(c->d_flags, 0, need * sizeof(int));
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  c->flags_cap = need;
  return EBV_SUCCESS;
}

ebv_status_t ensure_vflags(ebv_context* c, int64_t need) {
  if (need <= c->vflags_cap) return EBV_SUCCESS;
  if (c->d_vflags) cudaFree(c->d_vflags);
  c->d_vflags = nullptr;
  cudaError_t e = cudaMalloc(&c->d_vflags, need * sizeof(int));
  if (e != cudaSuccess) { c->vflags_cap = 0; set_error("workspace alloc failed"); return EBV_ERR_ALLOC; }
  e = cudaMemset(c->d_vflags, 0, need * sizeof(int));
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  c->vflags_cap = need;
  return EBV_SUCCESS;
}

}  // namespace

extern "C" {

static ebv_status_t factor_body(ebv_context_t c, int64_t n, double* A, int64_t lda, double tau, int64_t* d_info,
                                cudaStream_t s);

const char* ebv_status_string(ebv_status_t s) {
  switch (s) {
    case EBV_SUCCESS: return "success";
    case EBV_ERR_INVALID_VALUE: return "invalid value";
    case EBV_ERR_SINGULAR_PIVOT: return "singular pivot";
    case EBV_ERR_CUDA: return "CUDA error";
    case EBV_ERR_NCCL: return "NCCL error";
    case EBV_ERR_NOT_SUPPORTED: return "not supported";
    case EBV_ERR_ALLOC: return "allocation failed";
  }
  return "unknown status";
}

const char* ebv_last_error(void) { return g_last_error.c_str(); }

ebv_status_t ebv_create(ebv_context_t* ctx, int device) {
  if (!ctx) return invalid("ebv_create: ctx is NULL");
  *ctx = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= count) return invalid("ebv_create: bad device");
  DeviceGuard g(device);
  ebv_context* c = new ebv_context();
  c->device = device;
  // one allocation for the small scalars: tau, norm, scratch, tickets
  char* base = nullptr;
  e = cudaMalloc(&base, 256);
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "cudaMalloc"); }
  cudaMemset(base, 0, 256);
  c->d_tau = reinterpret_cast<double*>(base);
  c->d_norm = reinterpret_cast<unsigned long long*>(base + 8);
  c->d_scratch = reinterpret_cast<double*>(base + 16);
  c->d_ticket = reinterpret_cast<int*>(base + 64);
  c->d_pcount = reinterpret_cast<int*>(base + 128);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  e = cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_p, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming);
  if (e != cudaSuccess) { cudaFree(base); delete c; *ctx = nullptr; return cuda_fail(e, "stream/event create"); }
  *ctx = c;
  return EBV_SUCCESS;
}

ebv_status_t ebv_destroy(ebv_context_t c) {
  if (!c) return invalid("ebv_destroy: NULL");
  DeviceGuard g(c->device);
  dist_release(c);
  if (c->d_vec) cudaFree(c->d_vec);
  if (c->d_bws) cudaFree(c->d_bws);
  for (auto& r : c->recs) { cudaEventDestroy(r.e0); cudaEventDestroy(r.e1); }
  for (auto e : c->pool) cudaEventDestroy(e);
  for (auto& en : c->gcache)
    if (en.exec) cudaGraphExecDestroy(en.exec);
  if (c->d_flags) cudaFree(c->d_flags);
  if (c->d_vflags) cudaFree(c->d_vflags);
  cudaFree(c->d_tau);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->copy) cudaStreamDestroy(c->copy);
  for (auto ev : c->copy_ev) cudaEventDestroy(ev);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_p) cudaEventDestroy(c->ev_p);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->hostcopy_ev) cudaEventDestroy(c->hostcopy_ev);
  delete c;
  return EBV_SUCCESS;
}

ebv_status_t ebv_set_path(ebv_context_t c, ebv_path_t path) {
  if (!c) return invalid("ebv_set_path: NULL ctx");
  if (path != EBV_PATH_AUTO && path != EBV_PATH_VECTOR && path != EBV_PATH_BLOCKED && path != EBV_PATH_LEFT)
    return invalid("bad path");
  c->path = path;
  return EBV_SUCCESS;
}

ebv_status_t ebv_set_leaf(ebv_context_t c, int64_t leaf) {
  if (!c) return invalid("ebv_set_leaf: NULL ctx");
  if (leaf == 0) leaf = 64;
  if (leaf < 8 || leaf > 64 || leaf % 8) return invalid("leaf must be a multiple of 8 in [8, 64]");
  c->leaf = leaf;
  if (c->nb > 0 && c->nb % leaf) c->nb = ((c->nb + leaf - 1) / leaf) * leaf;
  return EBV_SUCCESS;
}

int64_t ebv_block_width(ebv_context_t c, int64_t n) {
  if (!c) return 0;
  return c->nb < 0 ? -1 : block_width(c, n);
}

ebv_status_t ebv_set_block(ebv_context_t c, int64_t nb) {
  if (!c) return invalid("ebv_set_block: NULL ctx");
  if (nb != 0 && nb != -1 && (nb < c->leaf || nb % c->leaf))
    return invalid("block must be 0 (adaptive), -1 or a multiple of the leaf size");
  c->nb = nb;
  return EBV_SUCCESS;
}

ebv_status_t ebv_set_graphs(ebv_context_t c, int enable) {
  if (!c) return invalid("ebv_set_graphs: NULL ctx");
  c->graphs = enable != 0;
  return EBV_SUCCESS;
}

ebv_status_t ebv_set_lookahead(ebv_context_t c, int enable) {
  if (!c) return invalid("ebv_set_lookahead: NULL ctx");
  c->lookahead = enable != 0;
  return EBV_SUCCESS;
}

ebv_status_t ebv_set_vector_ctas(ebv_context_t c, int64_t ctas) {
  if (!c) return invalid("ebv_set_vector_ctas: NULL ctx");
  c->vector_ctas = (int)ctas;
  return EBV_SUCCESS;
}

// EBV_GRAPH_PRIO=0 instantiates the captured schedule without per-node priorities
static const unsigned long long kGraphFlags = [] {
  const char* e = getenv("EBV_GRAPH_PRIO");
  return (e && atoi(e) == 0) ? 0ull : (unsigned long long)cudaGraphInstantiateFlagUseNodePriority;
}();

ebv_status_t ebv_lu_factor(ebv_context_t c, int64_t n, double* A, int64_t lda, double tau, int64_t* d_info,
                           void* stream) {
  if (!c) return invalid("ebv_lu_factor: NULL ctx");
  if (n < 0) return invalid("ebv_lu_factor: n < 0");
  if (lda < (n > 1 ? n : 1)) return invalid("ebv_lu_factor: lda < max(1, n)");
  if (!d_info) return invalid("ebv_lu_factor: d_info is NULL");
  if (n > 0 && !A) return invalid("ebv_lu_factor: A is NULL");
  if (c->path == EBV_PATH_VECTOR && n > EBV_VECTOR_MAX_N) return invalid("ebv_lu_factor: n too large for PATH_VECTOR");
  if (c->dist) return invalid("ebv_lu_factor: distributed context (A would be read as a full n x n matrix; use ebv_lu_factor_dist)");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  // CUDA Graph replay of the blocked schedule: the second call with the same
  // arguments captures it, later calls replay one graph (the schedule is
  // static; replay removes per-launch CPU cost and inter-kernel gaps).
  ebv_context::GraphEntry* ge = nullptr;
  const bool use_graph = c->graphs && !c->stats && s != nullptr && n > c->leaf && (c->path == EBV_PATH_AUTO || c->path == EBV_PATH_BLOCKED) &&
                         c->nb != -1;
  if (use_graph) {
    for (auto& en : c->gcache)
      if (en.n == n && en.lda == lda && en.A == A && en.info == d_info && en.tau == tau && en.nb == c->nb &&
          en.leaf == c->leaf && en.la == c->lookahead) {
        ge = &en;
        break;
      }
    if (ge && ge->exec) {
      cudaError_t e = cudaGraphLaunch(ge->exec, s);
      if (e != cudaSuccess) return cuda_fail(e, "graph launch");
      c->launches += ge->launches;
      return EBV_SUCCESS;
    }
    if (!ge) {
      if (c->gcache.size() >= 8) {
        if (c->gcache.front().exec) cudaGraphExecDestroy(c->gcache.front().exec);
        c->gcache.erase(c->gcache.begin());
      }
      c->gcache.push_back({n, lda, c->nb, c->leaf, A, d_info, tau, c->lookahead, 0, 0, nullptr});
      ge = &c->gcache.back();
    }
    ge->hits++;
  }
  const bool capture = use_graph && ge && ge->hits >= 2;
  const int64_t l0 = c->launches;
  if (capture) {
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "begin capture");
  }
  ebv_status_t st = factor_body(c, n, A, lda, tau, d_info, s);
  if (capture) {
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &graph);
    if (st != EBV_SUCCESS) { if (graph) cudaGraphDestroy(graph); return st; }
    if (e != cudaSuccess) return cuda_fail(e, "end capture");
    // per-node priorities: the lookahead panels were captured from the
    // high-priority side stream; without this flag the replay runs every
    // node at the launching stream's priority and the panel chain queues
    // behind the update (measured n = 32768: 725 ms replayed vs 710 direct)
    e = cudaGraphInstantiateWithFlags(&ge->exec, graph, kGraphFlags);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) { ge->exec = nullptr; return cuda_fail(e, "graph instantiate"); }
    ge->launches = c->launches - l0;
    e = cudaGraphLaunch(ge->exec, s);
    if (e != cudaSuccess) return cuda_fail(e, "graph launch");
  }
  return st;
}

static ebv_status_t factor_body(ebv_context_t c, int64_t n, double* A, int64_t lda, double tau, int64_t* d_info,
                                cudaStream_t s) {
  cudaError_t e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_set_info0(d_info, s); });
  if (e != cudaSuccess) return cuda_fail(e, "info init");
  if (n == 0) return EBV_SUCCESS;
  e = timed(c, KC_OTHER, 0, 8.0 * n * n, s, tau < 0 ? 3 : 1,
            [&] { return launch_tau(n, A, lda, tau, c->d_tau, c->d_norm, s); });
  if (e != cudaSuccess) return cuda_fail(e, "tau");
  if (c->path == EBV_PATH_VECTOR) {
    ebv_status_t st = ensure_vflags(c, n);
    if (st != EBV_SUCCESS) return st;
    int C = c->vector_ctas ? c->vector_ctas : vector_max_ctas(c->device, n);
    int smem_max = 0, sms = 0;
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    if (vector_smem_bytes(n, C) + 4096 > (size_t)smem_max || (C < 0 ? -C : C) > sms) {
      set_error("vector path: owned columns do not fit in shared memory (or more CTAs than SMs)");
      return EBV_ERR_NOT_SUPPORTED;
    }
    double fl = 2.0 / 3.0 * n * n * n, by = 16.0 * n * n;
    const int ep = (int)(c->vector_epoch % 0x3FFFFFF0) + 1;   // this context's flags, its own epochs
    c->vector_epoch++;
    e = timed(c, KC_VECTOR, fl, by, s, 2, [&] {
      return launch_vector_lu(n, A, lda, c->d_tau, d_info, c->d_vflags, c->d_scratch, C, ep, s);
    });
    if (e != cudaSuccess) return cuda_fail(e, "vector path");
    return EBV_SUCCESS;
  }
  if (c->path == EBV_PATH_LEFT) {
    e = lu_left(c, n, A, lda, d_info, s, nullptr, 0);
    if (e != cudaSuccess) return cuda_fail(e, "left-looking factor");
    return EBV_SUCCESS;
  }
  e = (c->nb != -1) ? lu_blocked(c, n, A, lda, d_info, s, n, n) : lu_rec(c, n, A, lda, 0, d_info, s);
  if (e != cudaSuccess) return cuda_fail(e, "blocked factor");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_factor_host(ebv_context_t c, int64_t n, const double* hA, int64_t ldh, double* A, int64_t lda,
                                double tau, int64_t* d_info, void* stream) {
  if (!c) return invalid("ebv_lu_factor_host: NULL ctx");
  if (n < 0) return invalid("ebv_lu_factor_host: n < 0");
  if (lda < (n > 1 ? n : 1) || ldh < (n > 1 ? n : 1)) return invalid("ebv_lu_factor_host: leading dimension < n");
  if (!d_info) return invalid("ebv_lu_factor_host: d_info is NULL");
  if (n > 0 && (!A || !hA)) return invalid("ebv_lu_factor_host: NULL matrix pointer");
  if (c->path == EBV_PATH_VECTOR && n > EBV_VECTOR_MAX_N) return invalid("ebv_lu_factor_host: n too large for PATH_VECTOR");
  if (c->dist) return invalid("ebv_lu_factor_host: distributed context (use ebv_lu_factor_dist)");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_set_info0(d_info, s); });
  if (e != cudaSuccess) return cuda_fail(e, "info init");
  if (n == 0) return EBV_SUCCESS;
  if (!c->hostcopy_ev) {
    e = cudaEventCreateWithFlags(&c->hostcopy_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "event create");
  }
  c->hostcopy_valid = false;
  if (c->path == EBV_PATH_LEFT && tau >= 0) {
    // left-looking: the column blocks stream in under the factorization
    e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_tau(n, A, lda, tau, c->d_tau, c->d_norm, s); });
    if (e == cudaSuccess) e = lu_left(c, n, A, lda, d_info, s, hA, ldh);
    if (e == cudaSuccess && c->copy) e = cudaEventRecord(c->hostcopy_ev, c->copy);
    if (e != cudaSuccess) return cuda_fail(e, "host factor (left-looking)");
    c->hostcopy_valid = c->copy != nullptr;
    return EBV_SUCCESS;
  }
  if (tau >= 0 && c->nb != -1 && (c->path == EBV_PATH_AUTO || c->path == EBV_PATH_BLOCKED) &&
      n >= 16384) {   // (smaller n: copy + factor is faster — measured n = 8192: 28 vs 44 ms)
    // default: right-looking with the column blocks joining as they arrive
    e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_tau(n, A, lda, tau, c->d_tau, c->d_norm, s); });
    if (e == cudaSuccess) e = lu_blocked_stream(c, n, A, lda, d_info, s, hA, ldh);
    if (e == cudaSuccess) e = cudaEventRecord(c->hostcopy_ev, c->copy);
    if (e != cudaSuccess) return cuda_fail(e, "host factor (streamed)");
    c->hostcopy_valid = true;
    return EBV_SUCCESS;
  }
  // otherwise: one copy, then the device schedule
  e = cudaMemcpy2DAsync(A, lda * sizeof(double), hA, ldh * sizeof(double), n * sizeof(double), n,
                        cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaEventRecord(c->hostcopy_ev, s);
  if (e != cudaSuccess) return cuda_fail(e, "host copy");
  c->hostcopy_valid = true;
  return factor_body(c, n, A, lda, tau, d_info, s);
}

ebv_status_t ebv_stream_wait_host_copy(ebv_context_t c, void* stream) {
  if (!c) return invalid("ebv_stream_wait_host_copy: NULL ctx");
  if (!c->hostcopy_valid) return EBV_SUCCESS;
  DeviceGuard g(c->device);
  cudaError_t e = cudaStreamWaitEvent((cudaStream_t)stream, c->hostcopy_ev, 0);
  if (e != cudaSuccess) return cuda_fail(e, "stream wait (host copy)");
  return EBV_SUCCESS;
}

static ebv_status_t solve_body(ebv_context_t c, int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb,
                               int64_t nrhs, void* stream);

ebv_status_t ebv_lu_solve(ebv_context_t c, int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb,
                          int64_t nrhs, void* stream) {
  if (!c) return invalid("ebv_lu_solve: NULL ctx");
  if (n < 0 || nrhs < 0) return invalid("ebv_lu_solve: negative size");
  if (lda < (n > 1 ? n : 1) || ldb < (n > 1 ? n : 1)) return invalid("ebv_lu_solve: leading dimension too small");
  if (n == 0 || nrhs == 0) return EBV_SUCCESS;
  if (!LU || !B) return invalid("ebv_lu_solve: NULL pointer");
  if (c->dist) return invalid("ebv_lu_solve: distributed context (use ebv_lu_solve_dist)");
  return solve_body(c, n, LU, lda, B, ldb, nrhs, stream);
}

// the single-GPU solve (also the one-rank case of the distributed solve,
// whose slab is then the whole matrix in the same layout)
static ebv_status_t solve_body(ebv_context_t c, int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb,
                               int64_t nrhs, void* stream) {
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const bool chain = kSolveChain && solve_chain_eligible(n, LU, lda, nrhs);
  if (solve_use_trsm(n, nrhs, chain)) {
    // many right-hand sides (factor once, solve many — SURVEY §8f f1): the
    // substitutions as recursive TRSMs, L^-1 then U^-1, whose off-diagonal
    // blocks are DMMA updates (k ascending forward, descending backward):
    // per entry the same fma chain and divisions as the wavefront kernel
    cudaError_t e = trsm_l(c, n, nrhs, LU, lda, B, ldb, s);
    if (e == cudaSuccess) e = trsm_lu(c, n, nrhs, LU, lda, B, ldb, s);
    if (e != cudaSuccess) return cuda_fail(e, "solve (trsm)");
    return EBV_SUCCESS;
  }
  // chain kernel wherever eligible (even n, even lda, aligned): measured
  // faster than the wavefront kernel at every order and column count tried
  // (profiles/r02_solve_chain*.jsonl vs r02_solve_wave.jsonl, e.g. n =
  // 32768, 1 RHS 3.5 vs 6.6 ms; n = 8192, 16 RHS 0.90 vs 2.1 ms)
  if (chain) {
    // chain-pipelined solve (k_solve2.cu): one chain CTA per right-hand side
    // walks the diagonal blocks, helper CTAs stream L / U
    ebv_status_t st = ensure_flags(c, 2 * solve_chain_flags(n));
    if (st != EBV_SUCCESS) return st;
    const int64_t ep0 = c->solve_epoch;
    c->solve_epoch += solve_chain_epochs(nrhs);
    const int64_t groups = (nrhs + 15) / 16;
    double by = (8.0 * n * n + 4.0 * 8.0 * n * nrhs), fl = 2.0 * n * n * nrhs;
    cudaError_t e = timed(c, KC_SOLVE, fl, by, s, (int)(2 * groups), [&] {
      return launch_solve_chain(n, LU, lda, B, ldb, nrhs, c->d_flags, ep0, s);
    });
    if (e != cudaSuccess) return cuda_fail(e, "solve (chain)");
    return EBV_SUCCESS;
  }
  const int64_t NB = (n + solve_block_rows() - 1) / solve_block_rows();
  ebv_status_t st = ensure_flags(c, 2 * NB * solve_max_interleave());   // interleaved columns per sweep
  if (st != EBV_SUCCESS) return st;
  const int64_t groups = (nrhs + 63) / 64, ep0 = c->solve_epoch;
  c->solve_epoch += launch_solve_epochs(nrhs);
  double by = (8.0 * n * n + 4.0 * 8.0 * n * nrhs), fl = 2.0 * n * n * nrhs;
  cudaError_t e = timed(c, KC_SOLVE, fl, by, s, (int)(2 * groups), [&] {
    return launch_solve(n, LU, lda, B, ldb, nrhs, c->d_ticket, c->d_flags, ep0, s);
  });
  if (e != cudaSuccess) return cuda_fail(e, "solve");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_factor_banded(ebv_context_t c, int64_t n, int64_t kl, int64_t ku, double* A, int64_t lda,
                                  double tau, int64_t* d_info, void* stream) {
  if (!c) return invalid("ebv_lu_factor_banded: NULL ctx");
  if (n < 0 || kl < 0 || ku < 0) return invalid("ebv_lu_factor_banded: negative size");
  if (lda < (n > 1 ? n : 1)) return invalid("ebv_lu_factor_banded: lda < max(1, n)");
  if (!d_info) return invalid("ebv_lu_factor_banded: d_info is NULL");
  if (n > 0 && !A) return invalid("ebv_lu_factor_banded: A is NULL");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_set_info0(d_info, s); });
  if (e != cudaSuccess) return cuda_fail(e, "info init");
  if (n == 0) return EBV_SUCCESS;
  e = timed(c, KC_OTHER, 0, 8.0 * n * n, s, tau < 0 ? 3 : 1,
            [&] { return launch_tau(n, A, lda, tau, c->d_tau, c->d_norm, s); });
  if (e != cudaSuccess) return cuda_fail(e, "tau");
  e = (c->nb != -1) ? lu_blocked(c, n, A, lda, d_info, s, kl, ku) : lu_rec(c, n, A, lda, 0, d_info, s);
  if (e != cudaSuccess) return cuda_fail(e, "banded factor");
  return EBV_SUCCESS;
}

static ebv_status_t solve_banded_impl(ebv_context_t c, int64_t n, int64_t kl, int64_t ku, const double* LU,
                                      int64_t lda, double* B, int64_t ldb, int64_t nrhs, void* stream);

// Compact band storage: AB[(PAD + ku + i - j) + j*ldab] = a_ij is the dense
// column-major view A = AB + PAD + ku with leading dimension ldab - 1 (entry
// (i, j) at A[i + j*(ldab - 1)]); every entry the 64-column banded schedule
// and the tile-skipping solve touch has |offset from the band| <= PAD, so it
// maps into its own column's slot (no aliasing) and holds an exact zero.
ebv_status_t ebv_lu_factor_band(ebv_context_t c, int64_t n, int64_t kl, int64_t ku, double* AB, int64_t ldab,
                                double tau, int64_t* d_info, void* stream) {
  if (!c) return invalid("ebv_lu_factor_band: NULL ctx");
  if (n < 0 || kl < 0 || ku < 0) return invalid("ebv_lu_factor_band: negative size");
  if (ldab < kl + ku + 2 * EBV_BAND_PAD + 1) return invalid("ebv_lu_factor_band: ldab < kl + ku + 2*EBV_BAND_PAD + 1");
  if (!(tau >= 0)) return invalid("ebv_lu_factor_band: tau must be >= 0 (explicit threshold)");
  if (!d_info) return invalid("ebv_lu_factor_band: d_info is NULL");
  if (n > 0 && !AB) return invalid("ebv_lu_factor_band: AB is NULL");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_set_info0(d_info, s); });
  if (e != cudaSuccess) return cuda_fail(e, "info init");
  if (n == 0) return EBV_SUCCESS;
  double* A = AB + EBV_BAND_PAD + ku;
  const int64_t lda = ldab - 1;
  e = timed(c, KC_OTHER, 0, 0, s, 1, [&] { return launch_tau(n, A, lda, tau, c->d_tau, c->d_norm, s); });
  if (e != cudaSuccess) return cuda_fail(e, "tau");
  e = lu_blocked(c, n, A, lda, d_info, s, kl, ku, true);
  if (e != cudaSuccess) return cuda_fail(e, "band factor");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_solve_band(ebv_context_t c, int64_t n, int64_t kl, int64_t ku, const double* AB, int64_t ldab,
                               double* B, int64_t ldb, int64_t nrhs, void* stream) {
  if (!c) return invalid("ebv_lu_solve_band: NULL ctx");
  if (n < 0 || nrhs < 0 || kl < 0 || ku < 0) return invalid("ebv_lu_solve_band: negative size");
  if (ldab < kl + ku + 2 * EBV_BAND_PAD + 1) return invalid("ebv_lu_solve_band: ldab < kl + ku + 2*EBV_BAND_PAD + 1");
  if (ldb < (n > 1 ? n : 1)) return invalid("ebv_lu_solve_band: ldb < max(1, n)");
  if (n == 0 || nrhs == 0) return EBV_SUCCESS;
  if (!AB || !B) return invalid("ebv_lu_solve_band: NULL pointer");
  return solve_banded_impl(c, n, kl, ku, AB + EBV_BAND_PAD + ku, ldab - 1, B, ldb, nrhs, stream);
}

static ebv_status_t solve_banded_impl(ebv_context_t c, int64_t n, int64_t kl, int64_t ku, const double* LU,
                                      int64_t lda, double* B, int64_t ldb, int64_t nrhs, void* stream) {
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t NB = (n + solve_block_rows() - 1) / solve_block_rows();
  ebv_status_t st = ensure_flags(c, 2 * NB * solve_max_interleave());
  if (st != EBV_SUCCESS) return st;
  const int64_t groups = (nrhs + 63) / 64, ep0 = c->solve_epoch;
  c->solve_epoch += launch_solve_epochs(nrhs);
  const double bw = (double)(kl + ku + 1) < n ? (double)(kl + ku + 1) : (double)n;
  cudaError_t e = timed(c, KC_SOLVE, 2.0 * n * bw * nrhs, 8.0 * n * bw + 32.0 * n * nrhs, s, (int)(2 * groups), [&] {
    return launch_solve(n, LU, lda, B, ldb, nrhs, c->d_ticket, c->d_flags, ep0, s, kl, ku);
  });
  if (e != cudaSuccess) return cuda_fail(e, "banded solve");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_solve_banded(ebv_context_t c, int64_t n, int64_t kl, int64_t ku, const double* LU, int64_t lda,
                                 double* B, int64_t ldb, int64_t nrhs, void* stream) {
  if (!c) return invalid("ebv_lu_solve_banded: NULL ctx");
  if (n < 0 || nrhs < 0 || kl < 0 || ku < 0) return invalid("ebv_lu_solve_banded: negative size");
  if (lda < (n > 1 ? n : 1) || ldb < (n > 1 ? n : 1)) return invalid("ebv_lu_solve_banded: leading dimension");
  if (n == 0 || nrhs == 0) return EBV_SUCCESS;
  if (!LU || !B) return invalid("ebv_lu_solve_banded: NULL pointer");
  return solve_banded_impl(c, n, kl, ku, LU, lda, B, ldb, nrhs, stream);
}

// Batched medium orders (SURVEY §8f f2, 64 < n <= EBV_BATCHED_MEDIUM_MAX_N):
// the blocked schedule with 64-column steps run for every system at once —
// each launch covers all systems (blockIdx.y / z = system): panel leaf, U12
// leaf solve, DMMA update; then (B given) forward / backward substitution as
// row-block TRSMs whose off-diagonal parts are DMMA updates (k ascending
// forward, descending backward).  Per system the operations are those of the
// single-system blocked path, in the canonical order (bitwise the oracle).
static ebv_status_t batched_medium(ebv_context_t c, int64_t n, double* A, int64_t lda, int64_t sA, int64_t batch,
                                   double* B, int64_t ldb, int64_t sB, int64_t nrhs, double tau, int32_t* d_info,
                                   cudaStream_t s, bool solve_only) {
  const int64_t need = batch * (int64_t)(sizeof(double) + sizeof(int64_t) + sizeof(int));
  if (need > c->bws_cap) {
    if (c->d_bws) cudaFree(c->d_bws);
    c->d_bws = nullptr;
    c->bws_cap = 0;
    if (cudaMalloc(&c->d_bws, need) != cudaSuccess) { set_error("workspace alloc failed"); return EBV_ERR_ALLOC; }
    if (cudaMemset(c->d_bws, 0, need) != cudaSuccess) { set_error("workspace init failed"); return EBV_ERR_ALLOC; }
    c->bws_cap = need;
  }
  double* tau_s = reinterpret_cast<double*>(c->d_bws);
  int64_t* info64 = reinterpret_cast<int64_t*>(tau_s + batch);
  int* counts = reinterpret_cast<int*>(info64 + batch);   // panel-leaf arrival counters (self-resetting)
  constexpr int64_t NB = 64;
  cudaError_t e = cudaSuccess;
  if (!solve_only) {
    // the counters' offset depends on this call's batch, so an earlier call
    // with another batch may have left its tau / info words there: clear them
    // (the leaves reset them to zero after every launch from then on)
    e = cudaMemsetAsync(counts, 0, batch * sizeof(int), s);
    if (e != cudaSuccess) return cuda_fail(e, "batched medium counters");
    e = timed(c, KC_OTHER, 0, tau < 0 ? 8.0 * n * n * batch : 0, s, 1,
              [&] { return launch_batched_prep(n, A, lda, sA, batch, tau, tau_s, info64, s); });
    for (int64_t c0 = 0; c0 < n && e == cudaSuccess; c0 += NB) {
      const int64_t w = n - c0 < NB ? n - c0 : NB, rest = n - c0 - w;
      double* P = A + c0 + c0 * lda;
      e = timed(c, KC_LEAF, batch * (2.0 / 3.0 * w * w * w + (double)(n - c0 - w) * w * w), batch * 16.0 * (n - c0) * w,
                s, 1, [&] {
                  return launch_panel_leaf_batched(n - c0, w, P, lda, sA, tau_s, 1, info64, 1, c0, counts, batch, s);
                });
      if (e != cudaSuccess || rest <= 0) break;
      e = timed(c, KC_TRSM, batch * (double)rest * w * w, batch * 16.0 * rest * w, s, 1,
                [&] { return launch_trsm_llu_batched(w, rest, P, lda, sA, P + w * lda, lda, sA, batch, s); });
      if (e != cudaSuccess) break;
      e = timed(c, KC_UPDATE, batch * 2.0 * rest * rest * w, batch * 8.0 * (2.0 * rest * w + 2.0 * rest * rest), s, 1,
                [&] {
                  return launch_gemm_sub_batched(rest, rest, w, P + w, lda, sA, P + w * lda, lda, sA,
                                                 P + w + w * lda, lda, sA, batch, false, s);
                });
    }
    if (e == cudaSuccess) e = launch_info_to_i32(batch, info64, d_info, s);
    if (e != cudaSuccess) return cuda_fail(e, "batched medium factor");
  }
  if (B && nrhs > 0) {
    for (int64_t r0 = 0; r0 < n && e == cudaSuccess; r0 += NB) {   // LY = B (Eq 1), k ascending
      const int64_t k = n - r0 < NB ? n - r0 : NB;
      if (r0 > 0)
        e = launch_gemm_sub_batched(k, nrhs, r0, A + r0, lda, sA, B, ldb, sB, B + r0, ldb, sB, batch, false, s);
      if (e == cudaSuccess)
        e = launch_trsm_llu_batched(k, nrhs, A + r0 + r0 * lda, lda, sA, B + r0, ldb, sB, batch, s);
    }
    const int64_t last = ((n - 1) / NB) * NB;
    for (int64_t r0 = last; r0 >= 0 && e == cudaSuccess; r0 -= NB) {   // UX = Y, k descending
      const int64_t k = n - r0 < NB ? n - r0 : NB, r1 = r0 + k;
      if (r1 < n)
        e = launch_gemm_sub_batched(k, nrhs, n - r1, A + r0 + r1 * lda, lda, sA, B + r1, ldb, sB, B + r0, ldb, sB,
                                    batch, true, s);
      if (e == cudaSuccess)
        e = launch_trsm_luu_batched(k, nrhs, A + r0 + r0 * lda, lda, sA, B + r0, ldb, sB, batch, s);
    }
    c->launches += 4 * ((n + NB - 1) / NB);
    if (e != cudaSuccess) return cuda_fail(e, "batched medium solve");
  }
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_factor_batched(ebv_context_t c, int64_t n, double* A, int64_t lda, int64_t strideA,
                                   int64_t batch, double* B, int64_t ldb, int64_t strideB, int64_t nrhs,
                                   double tau, int32_t* d_info, void* stream) {
  if (!c) return invalid("ebv_lu_factor_batched: NULL ctx");
  if (n < 0 || batch < 0 || nrhs < 0) return invalid("ebv_lu_factor_batched: negative size");
  if (lda < (n > 1 ? n : 1)) return invalid("ebv_lu_factor_batched: lda too small");
  if (batch > 1 && strideA < lda * n) return invalid("ebv_lu_factor_batched: strideA < lda*n");
  if (B && nrhs > 0) {
    if (ldb < (n > 1 ? n : 1)) return invalid("ebv_lu_factor_batched: ldb too small");
    if (batch > 1 && strideB < ldb * nrhs) return invalid("ebv_lu_factor_batched: strideB < ldb*nrhs");
  }
  if (n == 0 || batch == 0) return EBV_SUCCESS;
  if (!A || !d_info) return invalid("ebv_lu_factor_batched: NULL pointer");
  if (n > EBV_BATCHED_MEDIUM_MAX_N) { set_error("batched path supports n <= 512"); return EBV_ERR_NOT_SUPPORTED; }
  if (nrhs > 16) { set_error("batched path supports nrhs <= 16"); return EBV_ERR_NOT_SUPPORTED; }
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (n > EBV_BATCHED_MAX_N)
    return batched_medium(c, n, A, lda, strideA, batch, nrhs > 0 ? B : nullptr, ldb, strideB, nrhs, tau, d_info, s,
                          false);
  double* Bp = (nrhs > 0) ? B : nullptr;
  double fl = batch * (2.0 / 3.0 * n * n * n + 2.0 * n * n * (Bp ? nrhs : 0));
  double by = batch * (16.0 * n * n + (Bp ? 16.0 * n * nrhs : 0) + 4.0);
  cudaError_t e = timed(c, KC_BATCHED, fl, by, s, 1, [&] {
    return launch_batched(n, A, lda, strideA, batch, Bp, ldb, strideB, nrhs, nullptr, tau < 0, tau < 0 ? 0.0 : tau,
                          d_info, s);
  });
  if (e != cudaSuccess) return cuda_fail(e, "batched");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_solve_batched(ebv_context_t c, int64_t n, const double* LU, int64_t lda, int64_t strideA,
                                  int64_t batch, double* B, int64_t ldb, int64_t strideB, int64_t nrhs, void* stream) {
  if (!c) return invalid("ebv_lu_solve_batched: NULL ctx");
  if (n < 0 || batch < 0 || nrhs < 0) return invalid("ebv_lu_solve_batched: negative size");
  if (lda < (n > 1 ? n : 1)) return invalid("ebv_lu_solve_batched: lda too small");
  if (batch > 1 && strideA < lda * n) return invalid("ebv_lu_solve_batched: strideA < lda*n");
  if (ldb < (n > 1 ? n : 1)) return invalid("ebv_lu_solve_batched: ldb too small");
  if (batch > 1 && strideB < ldb * nrhs) return invalid("ebv_lu_solve_batched: strideB < ldb*nrhs");
  if (n == 0 || batch == 0 || nrhs == 0) return EBV_SUCCESS;
  if (!LU || !B) return invalid("ebv_lu_solve_batched: NULL pointer");
  if (n > EBV_BATCHED_MEDIUM_MAX_N) { set_error("batched path supports n <= 512"); return EBV_ERR_NOT_SUPPORTED; }
  if (nrhs > 16) { set_error("batched path supports nrhs <= 16"); return EBV_ERR_NOT_SUPPORTED; }
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (n > EBV_BATCHED_MAX_N)
    return batched_medium(c, n, const_cast<double*>(LU), lda, strideA, batch, B, ldb, strideB, nrhs, 0.0, nullptr, s,
                          true);
  double fl = batch * 2.0 * n * n * nrhs, by = batch * (8.0 * n * n + 16.0 * n * nrhs);
  cudaError_t e = timed(c, KC_BATCHED, fl, by, s, 1, [&] {
    return launch_batched(n, const_cast<double*>(LU), lda, strideA, batch, B, ldb, strideB, nrhs, nullptr, false, 0.0,
                          nullptr, s, /*solve_only=*/true);
  });
  if (e != cudaSuccess) return cuda_fail(e, "batched solve");
  return EBV_SUCCESS;
}

ebv_status_t ebv_normalize_unit_diagonal(ebv_context_t c, int64_t n, double* A, int64_t lda, double* B, int64_t ldb,
                                         int64_t nrhs, double* d_scales, int64_t* d_info, void* stream) {
  if (!c) return invalid("ebv_normalize_unit_diagonal: NULL ctx");
  if (n < 0 || nrhs < 0) return invalid("ebv_normalize_unit_diagonal: negative size");
  if (lda < (n > 1 ? n : 1)) return invalid("ebv_normalize_unit_diagonal: lda too small");
  if (B && nrhs > 0 && ldb < (n > 1 ? n : 1)) return invalid("ebv_normalize_unit_diagonal: ldb too small");
  if (!d_info || (n > 0 && !A)) return invalid("ebv_normalize_unit_diagonal: NULL pointer");
  DeviceGuard g(c->device);
  if (n > c->vec_cap) {
    if (c->d_vec) cudaFree(c->d_vec);
    c->d_vec = nullptr;
    c->vec_cap = 0;
    if (cudaMalloc(&c->d_vec, n * sizeof(double)) != cudaSuccess) { set_error("workspace alloc failed"); return EBV_ERR_ALLOC; }
    c->vec_cap = n;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nl = 0;
  cudaError_t e = timed(c, KC_OTHER, (double)n * (n + nrhs), 16.0 * n * (n + (B ? nrhs : 0)), s, 0, [&] {
    return launch_normalize_unit_diagonal(n, A, lda, B, ldb, B ? nrhs : 0, d_scales, d_info, c->d_vec,
                                          reinterpret_cast<unsigned long long*>(c->d_scratch), s, &nl);
  });
  c->launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "normalize");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_to_ldu(ebv_context_t c, int64_t n, double* LU, int64_t lda, double* d_D, void* stream) {
  if (!c) return invalid("ebv_lu_to_ldu: NULL ctx");
  if (n < 0) return invalid("ebv_lu_to_ldu: negative size");
  if (lda < (n > 1 ? n : 1)) return invalid("ebv_lu_to_ldu: lda too small");
  if (n == 0) return EBV_SUCCESS;
  if (!LU || !d_D) return invalid("ebv_lu_to_ldu: NULL pointer");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nl = 0;
  cudaError_t e = timed(c, KC_OTHER, 0.5 * n * n, 8.0 * n * n, s, 0, [&] { return launch_lu_to_ldu(n, LU, lda, d_D, s, &nl); });
  c->launches += nl;
  if (e != cudaSuccess) return cuda_fail(e, "ldu");
  return EBV_SUCCESS;
}

ebv_status_t ebv_update(ebv_context_t c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* C, int64_t ldc, void* stream) {
  if (!c) return invalid("ebv_update: NULL ctx");
  if (M < 0 || N < 0 || K < 0) return invalid("ebv_update: negative size");
  if (lda < (M > 1 ? M : 1) || ldb < (K > 1 ? K : 1) || ldc < (M > 1 ? M : 1))
    return invalid("ebv_update: leading dimension too small");
  if (M == 0 || N == 0 || K == 0) return EBV_SUCCESS;
  if (!A || !B || !C) return invalid("ebv_update: NULL pointer");
  DeviceGuard g(c->device);
  cudaError_t e = gemm(c, M, N, K, A, lda, B, ldb, C, ldc, false, (cudaStream_t)stream, KC_UPDATE);
  if (e != cudaSuccess) return cuda_fail(e, "update");
  return EBV_SUCCESS;
}

ebv_status_t ebv_batched_shard(int64_t batch, int rank, int nranks, int64_t* first, int64_t* count) {
  if (batch < 0 || nranks < 1 || rank < 0 || rank >= nranks || !first || !count)
    return invalid("ebv_batched_shard: bad arguments");
  const int64_t q = batch / nranks, r = batch % nranks;
  *count = q + (rank < r ? 1 : 0);
  *first = rank * q + (rank < r ? rank : r);
  return EBV_SUCCESS;
}

// ---- EbV plan ----------------------------------------------------------------

ebv_status_t ebv_plan_owner_map(int64_t n, int64_t workers, int32_t* owner) {
  if (n < 0 || workers < 1 || (n > 0 && !owner)) return invalid("ebv_plan_owner_map: bad arguments");
  for (int64_t j = 0; j < n; j++) {
    int64_t p = j < n - 1 - j ? j : n - 1 - j;
    owner[j] = (int32_t)(p % workers);
  }
  return EBV_SUCCESS;
}

ebv_status_t ebv_plan_units(int64_t n, int64_t workers, int32_t* tri0, int32_t* k0, int32_t* tri1, int32_t* k1,
                            int32_t* owner) {
  if (n < 2 || workers < 1 || !tri0 || !k0 || !tri1 || !k1 || !owner) return invalid("ebv_plan_units: bad arguments");
  int64_t u = 0;
  // within each triangle pair k with n-k (first with last), k = 1..floor((n-1)/2)
  for (int t = 0; t < 2; t++)
    for (int64_t k = 1; k <= (n - 1) / 2; k++) {
      tri0[u] = t; k0[u] = (int32_t)k; tri1[u] = t; k1[u] = (int32_t)(n - k);
      u++;
    }
  if (n % 2 == 0) {   // merge the two middle vectors across triangles
    tri0[u] = 0; k0[u] = (int32_t)(n / 2); tri1[u] = 1; k1[u] = (int32_t)(n / 2);
    u++;
  }
  for (int64_t i = 0; i < u; i++) owner[i] = (int32_t)(i % workers);
  return EBV_SUCCESS;
}

int64_t ebv_block_owner(int64_t J, int64_t N, int64_t nranks, ebv_layout_t layout) {
  if (J < 0 || J >= N || nranks < 1) return -1;
  switch (layout) {
    case EBV_LAYOUT_CYCLIC: return J % nranks;
    case EBV_LAYOUT_EBVPAIR: {
      int64_t p = J < N - 1 - J ? J : N - 1 - J;
      return p % nranks;
    }
    case EBV_LAYOUT_SNAKE: {
      int64_t r = J % (2 * nranks);
      return r < nranks ? r : 2 * nranks - 1 - r;
    }
  }
  return -1;
}

// ---- debug knobs ------------------------------------------------------------------

ebv_status_t ebv_set_debug(int device, unsigned flags, double spin_timeout_s) {
  if (flags & ~(unsigned)(EBV_DEBUG_FORCE_EXACT | EBV_DEBUG_JITTER)) return invalid("ebv_set_debug: unknown flag");
  if (!(spin_timeout_s >= 0.0) || spin_timeout_s > 1e6) return invalid("ebv_set_debug: spin timeout out of range");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= count) return invalid("ebv_set_debug: bad device");
  DeviceGuard g(device);
  DebugCfg cfg{flags, (unsigned long long)(spin_timeout_s * 1e9)};
  e = set_debug_solve(cfg);
  if (e == cudaSuccess) e = set_debug_vector(cfg);
  if (e == cudaSuccess) e = set_debug_batched(cfg);
  if (e == cudaSuccess) e = set_debug_leaf(cfg);
  if (e == cudaSuccess) e = set_debug_solve_chain(cfg);
  if (e != cudaSuccess) return cuda_fail(e, "ebv_set_debug");
  return EBV_SUCCESS;
}

// ---- measurement ---------------------------------------------------------------

ebv_status_t ebv_stats_enable(ebv_context_t c, int enable) {
  if (!c) return invalid("ebv_stats_enable: NULL ctx");
  c->stats = enable != 0;
  return EBV_SUCCESS;
}

static void drain(ebv_context* c) {
  for (auto& r : c->recs) {
    cudaEventSynchronize(r.e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    const int cls = r.cls & 0xFF;
    c->st_launch[cls]++;
    c->st_ms[cls] += ms;
    c->st_flops[cls] += r.flops;
    c->st_bytes[cls] += r.bytes;
    bool keep = false;
    if (!c->tl_ref) {   // the first launch since reset is the timeline's origin
      c->tl_ref = r.e0;
      keep = true;
    }
    float t0 = 0, t1 = 0;
    cudaEventElapsedTime(&t0, c->tl_ref, r.e0);
    cudaEventElapsedTime(&t1, c->tl_ref, r.e1);
    if (c->tl.size() < ((size_t)3 << 20)) {
      c->tl.push_back(r.cls);
      c->tl.push_back(t0);
      c->tl.push_back(t1);
    }
    if (!keep) c->pool.push_back(r.e0);
    c->pool.push_back(r.e1);
  }
  c->recs.clear();
}

ebv_status_t ebv_stats_reset(ebv_context_t c) {
  if (!c) return invalid("ebv_stats_reset: NULL ctx");
  DeviceGuard g(c->device);
  drain(c);
  for (int i = 0; i < EBV_NUM_KCLASSES; i++) c->st_launch[i] = 0, c->st_ms[i] = c->st_flops[i] = c->st_bytes[i] = 0;
  c->tl.clear();
  if (c->tl_ref) c->pool.push_back(c->tl_ref);
  c->tl_ref = nullptr;
  return EBV_SUCCESS;
}

int64_t ebv_stats_timeline(ebv_context_t c, double* out, int64_t max_records) {
  if (!c || max_records < 0 || (max_records > 0 && !out)) return -1;
  DeviceGuard g(c->device);
  drain(c);
  const int64_t nrec = (int64_t)(c->tl.size() / 3);
  const int64_t m = nrec < max_records ? nrec : max_records;
  for (int64_t i = 0; i < 3 * m; i++) out[i] = c->tl[i];
  return nrec;
}

ebv_status_t ebv_stats_get(ebv_context_t c, int kclass, int64_t* launches, double* ms, double* flops, double* bytes) {
  if (!c || kclass < 0 || kclass >= EBV_NUM_KCLASSES) return invalid("ebv_stats_get: bad arguments");
  DeviceGuard g(c->device);
  drain(c);
  if (launches) *launches = c->st_launch[kclass];
  if (ms) *ms = c->st_ms[kclass];
  if (flops) *flops = c->st_flops[kclass];
  if (bytes) *bytes = c->st_bytes[kclass];
  return EBV_SUCCESS;
}

int64_t ebv_launch_count(ebv_context_t c) { return c ? c->launches : -1; }

}  // extern "C"

namespace ebv {
namespace sched {
ebv_status_t solve_full(ebv_context* c, int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb,
                        int64_t nrhs, cudaStream_t s) {
  return solve_body(c, n, LU, lda, B, ldb, nrhs, s);
}
}  // namespace sched
}  // namespace ebv

extern "C" {

}  // extern "C"
