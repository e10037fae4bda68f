// k_solve2.cu — forward (LY = B) and backward (UX = Y) substitution, Eq 1
// ("UX = B" read as UX = Y, reading R6), as a chain-pipelined
// single-launch kernel per sweep: one CHAIN CTA per right-hand-side column
// walks the diagonal blocks in order with no inter-CTA hop on the dependent
// chain, while HELPER CTAs stream the rest of L (U) from HBM.
//
// Canonical order (the oracle's, bitwise): forward y_i is the fma chain over
// k ascending of (-l_ik y_k) starting from b_i; backward, k descending,
// x_k = y_k / u_kk then y_i = fma(-u_ik, x_k, y_i) for i < k.  Every entry of
// X below is produced by exactly that sequence; who applies a term changes,
// the order of the terms of one entry never does.
//
// Rows are cut into 64-row blocks, processed in LOGICAL order s = 0..NB-1
// (physical block phys(s) = s forward, NB-1-s backward).  For row block t the
// terms of tile (t, s) (rows of block t, columns of block s, s < t) must be
// applied in logical order s = 0, 1, ..., t-1, then the diagonal block solved.
//
//   helpers  : unit of 64 threads per row block t (thread = row): applies the
//              tiles s <= t - HL (as the y_s are published), then writes the
//              partial sums into B's rows of block t and releases hflag[t].
//   chain CTA: warps 0..3 hold one row block each (2 rows per lane), blocks
//              t = w (mod 4).  Warp w solves block t at step t; right after,
//              it picks up block t+4 (the helper's partial), absorbs tiles
//              t-1 .. t+3 of it (two complete, three live as the solver warps
//              of steps t+1..t+3 produce them, y values through shared
//              memory), and solves block t+4 at step t+4.  The solver of a
//              diagonal block keeps its 64 steps in registers and shuffles:
//              lane l owns rows 2l, 2l+1; per pair of steps the owner lane
//              finishes its second row in-lane (no shuffle on that hop).
//              Warp 4 loads the diagonal tiles (bulk async copies, mbarrier,
//              double buffered) and prefetches the absorbers' tiles to L2;
//              warp 5 publishes every solved block to B (global) and
//              releases yflag for the helpers.
//
// Backward divisions: the Markstein quotient from a reciprocal of the pivot
// computed ahead of the block; each lane verifies its two steps exactly after
// the block (dev::quot_is_rn); a block with any unverified quotient is redone
// with true division and the absorbers that consumed it redo that tile from a
// checkpoint — results are always RN(y/u), the oracle's division.
//
// Requirements (else the caller takes the wavefront kernel of k_solve.cu):
// n even, lda even, LU 16-byte aligned (the diagonal tiles move as 16-byte
// bulk copies), nrhs <= 16 per launch.
#include <cuda.h>

#include <type_traits>

#include "ebv_internal.cuh"
#include "ebv_device.cuh"

namespace ebv {
namespace {

constexpr int BR = 64;        // rows per block
#ifndef EBV_CHAIN_HL
#define EBV_CHAIN_HL 5
#endif
constexpr int HL = EBV_CHAIN_HL;         // helpers apply tiles s <= t - HL; the chain the last HL-1
constexpr int HR = 8;         // y-history ring (steps)
constexpr int NT = 192;       // threads per CTA (6 warps; helpers: 3 units of 64)
constexpr int MAXC = 16;      // right-hand sides per launch
#ifndef EBV_CHAIN_CGW
#define EBV_CHAIN_CGW 4
#endif
constexpr int kCGW = EBV_CHAIN_CGW;   // right-hand sides per helper unit (column group, <= 8)
static_assert(kCGW >= 1 && kCGW <= 8, "helper column groups of 1..8 columns");
constexpr int HT = 32;        // columns per half-tile (TMA box 64 x 32: diagonal tiles, helper tiles)
constexpr int QT = 16;        // columns per quarter-tile (TMA box 64 x 16: the absorbers' stream)
#ifndef EBV_CHAIN_NSLOT
#define EBV_CHAIN_NSLOT 4
#endif
constexpr int NSLOT = EBV_CHAIN_NSLOT;   // quarter-tile slots per block-holder warp

struct ChainSmem {
  double diag[2][BR * BR];        // diagonal tiles, column-major, double buffered (TMA)
  double slot[4][NSLOT][BR * QT]; // per block-holder warp: quarter-tile slots (TMA)
  double yh[HR][BR];              // y (x) values of recent steps, in processing order
  int prog[HR];                   // slot of step s started (sentinels written): s + 1
  int fin[HR];                    // step s final: 2*(s+1) + redo bit
  int sdone;                      // solver steps completed
  int pdone;                      // steps published to global memory
  unsigned long long mbar_d[2];
  unsigned long long mbar_s[4][NSLOT];
};
struct HelperSmem {
  double st[NT / 64][2][BR * BR];  // per unit: two tile stages (TMA)
  double ys[NT / 64][BR * MAXC];   // per unit: the published y of one block
  unsigned long long mbar[NT / 64][2];
};
constexpr size_t kSmem = sizeof(ChainSmem) > sizeof(HelperSmem) ? sizeof(ChainSmem) : sizeof(HelperSmem);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];\n" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// global flag wait: relaxed polls with back-off, one acquire fence after
__device__ __forceinline__ void wait_gflag(const int* p, int v, unsigned ns) {
  dev::SpinGuard g;
  while (ld_relaxed_gpu(p) != v) {
    __nanosleep(ns);
    g.poll();
  }
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}
__device__ __forceinline__ void wait_sflag_ge(const int* p, int v) {
  dev::SpinGuard g;
  while (ld_acq_cta(p) < v) g.poll();
}
// the same for warps off the critical path: back off so the spin does not
// take issue slots from the block holder sharing the SM sub-partition
__device__ __forceinline__ void wait_sflag_ge_slow(const int* p, int v) {
  dev::SpinGuard g;
  while (ld_acq_cta(p) < v) {
    __nanosleep(64);
    g.poll();
  }
}

// y (x) values reach the absorbers through the shared history with no
// per-value fence: the solver fills a step's slot with a sentinel (a
// signalling-NaN payload no arithmetic produces: results are quiet NaNs)
// when the step starts, the owner lanes then store each value (a naturally
// aligned 64-bit store: single-copy atomic), and a reader spins until the
// values it needs are not the sentinel.
constexpr long long kSent = 0x7FF4DEADBEEF0001LL;
__device__ __forceinline__ bool is_sent(double v) { return __double_as_longlong(v) == kSent; }
__device__ __forceinline__ double2 ld_vol2(const double* p) {
  double2 v;
  asm volatile("ld.volatile.shared::cta.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ double ld_vol(const double* p) {
  double v;
  asm volatile("ld.volatile.shared::cta.f64 %0, [%1];\n" : "=d"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
// the 8 values yh[j0 .. j0+7] (j0 a multiple of 8), once all are produced
__device__ __forceinline__ void wait_y8(const double* yh, double (&y)[8]) {
  dev::SpinGuard g;
  for (;;) {
    const double2 a = ld_vol2(yh), b = ld_vol2(yh + 2), c = ld_vol2(yh + 4), d = ld_vol2(yh + 6);
    y[0] = a.x; y[1] = a.y; y[2] = b.x; y[3] = b.y; y[4] = c.x; y[5] = c.y; y[6] = d.x; y[7] = d.y;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 8; i++) ok = ok && !is_sent(y[i]);
    if (ok) return;
    g.poll();
  }
}
__device__ __forceinline__ double wait_y1(const double* p) {
  dev::SpinGuard g;
  for (;;) {
    const double v = ld_vol(p);
    if (!is_sent(v)) return v;
    g.poll();
  }
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  dev::SpinGuard g;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (!done) g.poll();
  } while (!done);
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int row, int col, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(row), "r"(col), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void unit_sync(int unit) {   // 64 threads of one helper unit
  asm volatile("bar.sync %0, 64;\n" ::"r"(unit + 1) : "memory");
}

#ifdef EBV_CHAIN_TRACE
// probes/chain_trace.cu: %globaltimer stamps of the chain CTA (column 0)
__device__ unsigned long long g_ct[4096][14];
__device__ unsigned long long g_cq[64][4];   // quarter-level stamps of block 20
#define EBV_CQ(t, q, slot)                                                                 \
  do {                                                                                     \
    if (FWD == (EBV_CHAIN_TRACE_FWD != 0) && lane == 0 && (t) == EBV_CQ_T && (q) < 64)           \
      g_cq[(q)][(slot)] = dev::gtimer();                                                   \
  } while (0)
#ifndef EBV_CHAIN_TRACE_FWD
#define EBV_CHAIN_TRACE_FWD 0
#endif
#ifndef EBV_CQ_T
#define EBV_CQ_T 200
#endif
#define EBV_CT(t, slot)                                                                    \
  do {                                                                                     \
    if (FWD == (EBV_CHAIN_TRACE_FWD != 0) && lane == 0 && (t) < 4096)                      \
      g_ct[(t)][(slot)] = dev::gtimer();                                                   \
  } while (0)
#else
#define EBV_CT(t, slot) \
  do {                  \
  } while (0)
#define EBV_CQ(t, q, slot) \
  do {                     \
  } while (0)
#endif

struct Args {
  int64_t n;
  const double* LU;
  int64_t lda;
  double* B;
  int64_t ldb;
  int nr;          // right-hand sides (chain CTAs) in this launch, <= MAXC
  int* ticket;
  int* yflag;      // [nr][NB], logical block order
  int* hflag;      // [ngroups][NB]: helper partial of (column group, block) stored
  int cgw;         // right-hand sides per helper column group (<= NRT)
  int ngroups;     // column groups: helper units are (block, group) pairs
  int epoch;
};

template <bool FWD>
struct Geo {
  const double* LU;
  int64_t lda;
  int64_t n, NB;
  int nvlast;   // valid rows of the last physical block
  __device__ __forceinline__ int64_t phys(int64_t s) const { return FWD ? s : NB - 1 - s; }
  __device__ __forceinline__ int nv(int64_t s) const { return phys(s) == NB - 1 ? nvlast : BR; }
  // processing index j of logical block s -> row / column offset inside the block
  __device__ __forceinline__ int kof(int64_t s, int j) const { return FWD ? j : nv(s) - 1 - j; }
};

// ---------------------------------------------------------------------------- helper
// Tiles (tb, tj), tj = 0 .. tb-HL, stream through two shared-memory stages
// (2-D TMA, two 64 x 32 boxes each, zero fill past n) one tile ahead of the
// one being applied; the unit's thread 0 issues them.
template <bool FWD>
__device__ __forceinline__ void helper_issue(const CUtensorMap* map, const Geo<FWD>& g, HelperSmem& hs, int unit,
                                             int64_t tb, int64_t tj) {
  const int k = (int)(tj & 1);
  const int r = (int)(g.phys(tb) * BR), c = (int)(g.phys(tj) * BR);
  mbar_expect_tx(&hs.mbar[unit][k], (uint32_t)(BR * BR * 8));
  tma_2d(hs.st[unit][k], map, r, c, &hs.mbar[unit][k]);
  tma_2d(hs.st[unit][k] + BR * HT, map, r, c + HT, &hs.mbar[unit][k]);
}

template <bool FWD, int NRT>
__device__ void helper_unit(const Args& a, const CUtensorMap* map, const Geo<FWD>& g, HelperSmem& hs, int64_t tb,
                            int cg, int tid, int unit, uint32_t (&uses)[2]) {
  const int64_t ntiles = tb - HL + 1;
  if (ntiles <= 0) return;                      // blocks the chain absorbs entirely: nothing to do
  const int64_t IB = g.phys(tb);
  const int64_t row = IB * BR + tid;
  const bool rv = row < a.n;
  // this unit's right-hand sides: columns c0 .. c0 + nr - 1 of the launch
  // (NRT == 1: compile-time constants — the runtime form measured 13% slower
  // on the one-right-hand-side solve, n = 32768: 3.98 vs 3.50 ms)
  const int c0 = NRT == 1 ? cg : cg * a.cgw;
  const int nr = NRT == 1 ? 1 : ((a.nr - c0) < a.cgw ? (a.nr - c0) : a.cgw);
  double* const B = a.B + (int64_t)c0 * a.ldb;
  const int* const yflag = a.yflag + (int64_t)c0 * g.NB;
  double* ys = hs.ys[unit];
  if (tid == 0) {
    helper_issue<FWD>(map, g, hs, unit, tb, 0);
    if (ntiles > 1) helper_issue<FWD>(map, g, hs, unit, tb, 1);
  }
  double acc[NRT];
#pragma unroll
  for (int c = 0; c < NRT; c++) acc[c] = (rv && c < nr) ? B[row + (int64_t)c * a.ldb] : 0.0;
  for (int64_t tj = 0; tj < ntiles; tj++) {
    const int64_t JB = g.phys(tj);
    const int nvj = g.nv(tj);
    const int k2 = (int)(tj & 1);
    if (tid < nr) wait_gflag(yflag + (int64_t)tid * g.NB + tj, a.epoch, 64);
#ifdef EBV_CHAIN_TRACE
    if (tid == 0 && tj + 1 == ntiles && FWD == (EBV_CHAIN_TRACE_FWD != 0) && tb < 4096) g_ct[tb][12] = dev::gtimer();
#endif
    unit_sync(unit);
    for (int idx = tid; idx < BR * nr; idx += 64) {
      const int k = idx % BR, c = idx / BR;
      ys[k * NRT + c] = (k < nvj) ? __ldcg(B + JB * BR + k + (int64_t)c * a.ldb) : 0.0;
    }
    mbar_wait(&hs.mbar[unit][k2], uses[k2] & 1u);
    uses[k2]++;
    unit_sync(unit);
    const double* L = hs.st[unit][k2] + tid;     // column k of the tile at L[k * 64]
    if (FWD) {
#pragma unroll 16
      for (int k = 0; k < BR; k++) {
        const double l = L[k * BR];
#pragma unroll
        for (int c = 0; c < NRT; c++)
          if (c < nr) acc[c] = fma(-l, ys[k * NRT + c], acc[c]);
      }
    } else {
#pragma unroll 16
      for (int k = BR - 1; k >= 0; k--) {
        const double l = L[k * BR];
#pragma unroll
        for (int c = 0; c < NRT; c++)
          if (c < nr) acc[c] = fma(-l, ys[k * NRT + c], acc[c]);
      }
    }
    unit_sync(unit);                           // stage and ys free again
    if (tid == 0 && tj + 2 < ntiles) {
      fence_proxy_async();
      helper_issue<FWD>(map, g, hs, unit, tb, tj + 2);
    }
  }
#pragma unroll
  for (int c = 0; c < NRT; c++)
    if (rv && c < nr) B[row + (int64_t)c * a.ldb] = acc[c];
  unit_sync(unit);
  if (tid == 0) {
    dev::jitter((unsigned)tb);
    st_release_gpu(a.hflag + (int64_t)cg * g.NB + tb, a.epoch);
#ifdef EBV_CHAIN_TRACE
    if (FWD == (EBV_CHAIN_TRACE_FWD != 0) && tb < 4096) g_ct[tb][13] = dev::gtimer();
#endif
  }
}

// ---------------------------------------------------------------------------- chain
// The tiles a block holder absorbs stream through its two shared-memory
// half-tile slots (2-D TMA, 64 rows x 32 columns, zero fill past n): the
// absorb sequence of block t is the half-tiles of tiles s0 .. t-1 in
// processing order; half-tile h goes to slot h & 1, and slot k's uses are
// counted so the mbarrier parity is known.
struct SlotState {
  uint32_t q;   // quarters consumed by this warp so far: slot q % NSLOT, parity (q / NSLOT) & 1
};

template <bool FWD>
__device__ __forceinline__ void issue_quarter(const CUtensorMap* mapq, const Geo<FWD>& g, ChainSmem& sm, int w,
                                              int64_t t, int64_t s0, int q, uint32_t qabs) {
  const int64_t sT = s0 + q / 4;
  const int qq = q & 3;
  const int cq = FWD ? qq : 3 - qq;
  const int k = (int)(qabs % NSLOT);
  mbar_expect_tx(&sm.mbar_s[w][k], (uint32_t)(BR * QT * 8));
  tma_2d(sm.slot[w][k], mapq, (int)(g.phys(t) * BR), (int)(g.phys(sT) * BR + cq * QT), &sm.mbar_s[w][k]);
}

// (by value: reference parameters of an out-of-line call put the caller's
// accumulators and geometry in local memory for the whole absorb loop)
template <bool FWD>
__device__ __noinline__ double2 redo_tile(const Geo<FWD> g, ChainSmem& sm, int64_t t, int64_t sT, int lane, double v0,
                                          double v1) {
  const int64_t r0 = g.phys(t) * BR + 2 * lane;
  const double* rowp = g.LU + (r0 < g.n ? r0 : 0);
  const int nvs = g.nv(sT);
  const int hs = (int)(sT % HR);
  for (int jj = 0; jj < nvs; jj++) {
    const double2 l = __ldg(reinterpret_cast<const double2*>(rowp + (g.phys(sT) * BR + g.kof(sT, jj)) * g.lda));
    const double y = sm.yh[hs][jj];
    v0 = fma(-l.x, y, v0);
    v1 = fma(-l.y, y, v1);
  }
  return make_double2(v0, v1);
}

// Quarter q of block t's absorb sequence lives in slot (qa % NSLOT) once its
// mbarrier phase (qa / NSLOT) & 1 completes (qa: the warp's running quarter
// count).  Full tiles are software pipelined: the next quarter's L values
// are read from shared memory into registers while the current quarter's
// 16 terms are applied.
struct AbsorbCtx {
  double ck0, ck1;   // checkpoint at the current tile's start (backward redo)
  bool done;         // the current tile's step is final: plain loads, no sentinel checks
};

template <bool FWD>
__device__ __forceinline__ void load_quarter(const ChainSmem& sm, int w, uint32_t qa, int lane, double2 (&L)[QT]) {
  const int k = (int)(qa % NSLOT);
  mbar_wait(const_cast<unsigned long long*>(&sm.mbar_s[w][k]), (qa / NSLOT) & 1u);
  const double* S = sm.slot[w][k];
#pragma unroll
  for (int i = 0; i < QT; i++) L[i] = *reinterpret_cast<const double2*>(S + (FWD ? i : QT - 1 - i) * BR + 2 * lane);
}

// the end of quarter q: after a tile's last quarter, the backward redo check
template <bool FWD>
__device__ __forceinline__ void quarter_end(const Geo<FWD>& g, ChainSmem& sm, int64_t t, int64_t s0, int q, int lane,
                                            AbsorbCtx& ac, double& v0, double& v1) {
  if ((q & 3) == 3) {
    const int64_t sT = s0 + q / 4;
    const int hs = (int)(sT % HR);
    EBV_CT(t, (int)(2 + (sT - s0)));
    if (!FWD) {
      // the tile's values must be final (verified) before the next tile;
      // on a redo of step sT, restore and re-apply its corrected values
      wait_sflag_ge(&sm.fin[hs], (int)(2 * (sT + 1)));
      if (ld_acq_cta(&sm.fin[hs]) & 1) {
        const double2 r = redo_tile<FWD>(g, sm, t, sT, lane, ac.ck0, ac.ck1);
        v0 = r.x;
        v1 = r.y;
      }
    }
  }
}

// the end of quarter q: release its slot (its values are in every lane's
// registers; the proxy fence orders those generic reads before the TMA
// refill with quarter q + NSLOT — one fence per pair of quarters, with the
// refills issued later, measured slower: 3.59 vs 3.48 ms at n = 32768, the
// in-flight depth matters more than the fence), then the tile-end check
template <bool FWD>
__device__ __forceinline__ void quarter_done(const CUtensorMap* mapq, const Geo<FWD>& g, ChainSmem& sm, int w,
                                             int64_t t, int64_t s0, int q, int nq, uint32_t qa, int lane,
                                             AbsorbCtx& ac, double& v0, double& v1) {
  __syncwarp();
  fence_proxy_async();
  if (lane == 0 && q + NSLOT < nq) issue_quarter<FWD>(mapq, g, sm, w, t, s0, q + NSLOT, qa + NSLOT);
  quarter_end<FWD>(g, sm, t, s0, q, lane, ac, v0, v1);
}

template <bool FWD>
__device__ __forceinline__ void tile_start(const Geo<FWD>& g, ChainSmem& sm, int64_t sT, AbsorbCtx& ac, double v0,
                                           double v1) {
  const int hs = (int)(sT % HR);
  ac.ck0 = v0;
  ac.ck1 = v1;
  wait_sflag_ge(&sm.prog[hs], (int)(sT + 1));          // the slot holds step sT (sentinels or values)
  ac.done = ld_acq_cta(&sm.fin[hs]) >= (int)(2 * (sT + 1));
}

// apply the 16 terms of quarter q (full tile) held in L
template <bool FWD>
__device__ __forceinline__ void apply_quarter(ChainSmem& sm, int64_t s0, int q, const AbsorbCtx& ac,
                                              const double2 (&L)[QT], double& v0, double& v1) {
  const int64_t sT = s0 + q / 4;
  const double* yh = sm.yh[sT % HR] + (q & 3) * QT;
#pragma unroll
  for (int h8 = 0; h8 < QT; h8 += 8) {
    double y[8];
    if (ac.done) {
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        const double2 y2 = *reinterpret_cast<const double2*>(yh + h8 + i);
        y[i] = y2.x;
        y[i + 1] = y2.y;
      }
    } else {
      wait_y8(yh + h8, y);
    }
#pragma unroll
    for (int i = 0; i < 8; i++) {
      v0 = fma(-L[h8 + i].x, y[i], v0);
      v1 = fma(-L[h8 + i].y, y[i], v1);
    }
  }
}

template <bool FWD>
__device__ __forceinline__ void absorb(const CUtensorMap* mapq, const Geo<FWD>& g, ChainSmem& sm, int w, int64_t t,
                                       int64_t s0, int lane, SlotState& ss, double& v0, double& v1) {
  const int nq = (int)(4 * (t - s0));                 // quarters to absorb (the first NSLOT already issued)
  const uint32_t q0abs = ss.q;
  AbsorbCtx ac{v0, v1, false};
  int q = 0;
  // the ragged block (backward: logical block 0, nvs < 64): its quarters
  // one by one, processing indices j whose column k(j) lies in the quarter
  if (nq > 0 && g.nv(s0) != BR) {
    const int nvs = g.nv(s0);
    const int hs = (int)(s0 % HR);
    tile_start<FWD>(g, sm, s0, ac, v0, v1);
    for (; q < 4; q++) {
      const uint32_t qa = q0abs + (uint32_t)q;
      const int k = (int)(qa % NSLOT);
      mbar_wait(&sm.mbar_s[w][k], (qa / NSLOT) & 1u);
      const double* S = sm.slot[w][k];
      const int c0 = (FWD ? q : 3 - q) * QT;
      for (int j = 0; j < nvs; j++) {
        const int kc = g.kof(s0, j) - c0;
        if (kc < 0 || kc >= QT) continue;
        const double yv = wait_y1(sm.yh[hs] + j);
        const double2 l = *reinterpret_cast<const double2*>(S + kc * BR + 2 * lane);
        v0 = fma(-l.x, yv, v0);
        v1 = fma(-l.y, yv, v1);
      }
      quarter_done<FWD>(mapq, g, sm, w, t, s0, q, nq, qa, lane, ac, v0, v1);
    }
  }
  // full tiles, two quarters per iteration: La holds quarter q, Lb quarter q+1
  if (q < nq) {
    double2 La[QT], Lb[QT];
    load_quarter<FWD>(sm, w, q0abs + (uint32_t)q, lane, La);
    for (; q < nq; q += 2) {
      if ((q & 3) == 0) tile_start<FWD>(g, sm, s0 + q / 4, ac, v0, v1);
      EBV_CQ(t, q, 0);
      if (q + 1 < nq) load_quarter<FWD>(sm, w, q0abs + (uint32_t)(q + 1), lane, Lb);
      EBV_CQ(t, q, 1);
      apply_quarter<FWD>(sm, s0, q, ac, La, v0, v1);
      EBV_CQ(t, q, 2);
      quarter_done<FWD>(mapq, g, sm, w, t, s0, q, nq, q0abs + (uint32_t)q, lane, ac, v0, v1);
      EBV_CQ(t, q, 3);
      if (q + 1 < nq) {
        EBV_CQ(t, q + 1, 0);
        if (q + 2 < nq) load_quarter<FWD>(sm, w, q0abs + (uint32_t)(q + 2), lane, La);
        EBV_CQ(t, q + 1, 1);
        apply_quarter<FWD>(sm, s0, q + 1, ac, Lb, v0, v1);
        EBV_CQ(t, q + 1, 2);
        quarter_done<FWD>(mapq, g, sm, w, t, s0, q + 1, nq, q0abs + (uint32_t)(q + 1), lane, ac, v0, v1);
        EBV_CQ(t, q + 1, 3);
      }
    }
  }
  ss.q = q0abs + (uint32_t)nq;
}

// solve diagonal block t (rows 2l, 2l+1 in v0, v1; all earlier tiles applied)
template <bool FWD>
__device__ __forceinline__ void solve_diag(const Geo<FWD>& g, ChainSmem& sm, int64_t t, int lane, double& v0,
                                           double& v1) {
  const int buf = (int)(t & 1);
  if (t >= HR) wait_sflag_ge(&sm.pdone, (int)(t - HR + 1));   // slot t % HR published (free)
  EBV_CT(t, 7);
  mbar_wait(&sm.mbar_d[buf], (uint32_t)((t >> 1) & 1));
  EBV_CT(t, 8);
  const double* D = sm.diag[buf];
  const int slot = (int)(t % HR);
  const int nvs = g.nv(t);
  const int np = nvs / 2;
  double* yh = sm.yh[slot];
  {
    const double sent = __longlong_as_double(kSent);
    *reinterpret_cast<double2*>(yh + 2 * lane) = make_double2(sent, sent);
    __syncwarp();
    if (lane == 0) st_rel_cta(&sm.prog[slot], (int)(t + 1));   // slot of step t started
  }
  if (FWD) {
#pragma unroll 4
    for (int p = 0; p < np; p++) {
      const double2 c0 = *reinterpret_cast<const double2*>(D + (2 * p) * BR + 2 * lane);      // L(2l.., 2p)
      const double2 c1 = *reinterpret_cast<const double2*>(D + (2 * p + 1) * BR + 2 * lane);  // L(2l.., 2p+1)
      const double t1 = fma(-c0.y, v0, v1);             // owner lane: y_{2p+1} from its own y_{2p}
      const double y0 = __shfl_sync(0xffffffffu, v0, p);
      const double y1 = __shfl_sync(0xffffffffu, t1, p);
      if (lane == p) *reinterpret_cast<double2*>(yh + 2 * p) = make_double2(v0, t1);
      const double n0 = fma(-c1.x, y1, fma(-c0.x, y0, v0));
      const double n1 = fma(-c1.y, y1, fma(-c0.y, y0, v1));
      v0 = lane > p ? n0 : v0;
      v1 = lane > p ? n1 : (lane == p ? t1 : v1);
    }
    st_rel_cta(&sm.fin[slot], (int)(2 * (t + 1)));
  } else {
    const bool own = lane < np;
    const double d0 = own ? D[(2 * lane) * BR + 2 * lane] : 1.0;
    const double d1 = own ? D[(2 * lane + 1) * BR + 2 * lane + 1] : 1.0;
    const double rc0 = 1.0 / d0, rc1 = 1.0 / d1;
    const double w0 = v0, w1 = v1;                    // checkpoint for a redo
    double ya = 0.0, qa = 0.0, yb = 0.0, qb = 0.0;    // this lane's two steps (dividend, quotient)
#pragma unroll 4
    for (int p = np - 1; p >= 0; p--) {
      const double2 c1 = *reinterpret_cast<const double2*>(D + (2 * p + 1) * BR + 2 * lane);  // U(2l.., 2p+1)
      const double2 c0 = *reinterpret_cast<const double2*>(D + (2 * p) * BR + 2 * lane);      // U(2l.., 2p)
      const double q1 = dev::quot_mk(v1, d1, rc1);     // owner: x_{2p+1}
      const double t0 = fma(-c1.x, q1, v0);            // owner: row 2p with x_{2p+1}
      const double q0 = dev::quot_mk(t0, d0, rc0);     // owner: x_{2p}
      const double x1 = __shfl_sync(0xffffffffu, q1, p);
      const double x0 = __shfl_sync(0xffffffffu, q0, p);
      const int j = 2 * (np - 1 - p);
      if (lane == p) {
        ya = v1; qa = q1; yb = t0; qb = q0;
        *reinterpret_cast<double2*>(yh + j) = make_double2(q1, q0);
      }
      const double n0 = fma(-c0.x, x0, fma(-c1.x, x1, v0));
      const double n1 = fma(-c0.y, x0, fma(-c1.y, x1, v1));
      v0 = lane < p ? n0 : (lane == p ? q0 : v0);
      v1 = lane < p ? n1 : (lane == p ? q1 : v1);
    }
    const bool ok = !own || (dev::quot_is_rn(ya, d1, qa) && dev::quot_is_rn(yb, d0, qb));
    int redo = 0;
    if (__any_sync(0xffffffffu, !ok)) {
      // the block again with correctly rounded division
      redo = 1;
      v0 = w0;
      v1 = w1;
      for (int p = np - 1; p >= 0; p--) {
        const double2 c1 = *reinterpret_cast<const double2*>(D + (2 * p + 1) * BR + 2 * lane);
        const double2 c0 = *reinterpret_cast<const double2*>(D + (2 * p) * BR + 2 * lane);
        const double q1 = v1 / d1;
        const double t0 = fma(-c1.x, q1, v0);
        const double q0 = t0 / d0;
        const double x1 = __shfl_sync(0xffffffffu, q1, p);
        const double x0 = __shfl_sync(0xffffffffu, q0, p);
        const int j = 2 * (np - 1 - p);
        if (lane == p) *reinterpret_cast<double2*>(yh + j) = make_double2(q1, q0);
        const double n0 = fma(-c0.x, x0, fma(-c1.x, x1, v0));
        const double n1 = fma(-c0.y, x0, fma(-c1.y, x1, v1));
        v0 = lane < p ? n0 : (lane == p ? q0 : v0);
        v1 = lane < p ? n1 : (lane == p ? q1 : v1);
      }
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) st_rel_cta(&sm.fin[slot], (int)(2 * (t + 1)) + redo);
  }
  __syncwarp();
  EBV_CT(t, 9);
  if (lane == 0) st_rel_cta(&sm.sdone, (int)(t + 1));   // diag buffer (t & 1) may be refilled
}

template <bool FWD>
__device__ __forceinline__ void issue_diag(const CUtensorMap* map, const Geo<FWD>& g, ChainSmem& sm, int64_t t) {
  const int buf = (int)(t & 1);
  const int r = (int)(g.phys(t) * BR);
  mbar_expect_tx(&sm.mbar_d[buf], (uint32_t)(BR * BR * 8));
  tma_2d(sm.diag[buf], map, r, r, &sm.mbar_d[buf]);
  tma_2d(sm.diag[buf] + BR * HT, map, r, r + HT, &sm.mbar_d[buf]);
}

__device__ __forceinline__ void prefetch_tile(const CUtensorMap* map, int64_t row, int64_t col) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"((int)row), "r"((int)col)
               : "memory");
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"((int)row), "r"((int)(col + HT))
               : "memory");
}

// the L2 prefetch warp measured no gain (the tiles come through TMA in time);
// EBV_CHAIN_PREFETCH turns it on for experiments
#ifdef EBV_CHAIN_PREFETCH
constexpr bool kNoPrefetch = false;
constexpr int kPF = EBV_CHAIN_PREFETCH;
#else
constexpr bool kNoPrefetch = true;
constexpr int kPF = 3;
#endif

template <bool FWD>
__device__ void chain_cta(const Args& a, const CUtensorMap* map, const CUtensorMap* mapq, const Geo<FWD>& g,
                          ChainSmem& sm, int col) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t NB = g.NB;
  double* Bc = a.B + (int64_t)col * a.ldb;
  int* yflag = a.yflag + (int64_t)col * NB;
  if (warp < 4) {
    SlotState ss{0u};
    for (int64_t t = warp; t < NB; t += 4) {
      const int64_t s0 = t - HL + 1 > 0 ? t - HL + 1 : 0;
      const int nq = (int)(4 * (t - s0));
      if (lane == 0)
        for (int q = 0; q < NSLOT && q < nq; q++) issue_quarter<FWD>(mapq, g, sm, warp, t, s0, q, ss.q + q);
      // pick up block t: the helper's partial sums (tiles s <= t - HL)
      const int64_t r0 = g.phys(t) * BR + 2 * lane;
      EBV_CT(t, 0);
      if (t - HL + 1 > 0) {
        if (lane == 0) wait_gflag(a.hflag + (int64_t)(col / a.cgw) * NB + t, a.epoch, 32);
        __syncwarp();
      }
      EBV_CT(t, 1);
      double v0 = 0.0, v1 = 0.0;
      if (r0 < a.n) {
        const double2 b2 = __ldcg(reinterpret_cast<const double2*>(Bc + r0));
        v0 = b2.x;
        v1 = b2.y;
      }
      absorb<FWD>(mapq, g, sm, warp, t, s0, lane, ss, v0, v1);
      solve_diag<FWD>(g, sm, t, lane, v0, v1);
      // diagonal buffer t & 1 is free: the tile of step t + 2 into it
      fence_proxy_async();
      if (lane == 0 && t + 2 < NB) issue_diag<FWD>(map, g, sm, t + 2);
    }
  } else if (warp == 4 && !kNoPrefetch) {
    // (experiment, off by default: measured no gain) L2 prefetch of the
    // tiles the absorbers take PF steps from now: (s+d, s), d = 1 .. HL-1,
    // of column block s = t + PF, and the diagonal tile of step s
    for (int64_t t = 0; t < NB; t++) {
      if (t >= 1) wait_sflag_ge_slow(&sm.sdone, (int)t);   // step t-1 done
      const int64_t sc = t + kPF;
      if (lane == 0 && sc < NB) {
        for (int d = 1; d < HL && sc + d < NB; d++) prefetch_tile(map, g.phys(sc + d) * BR, g.phys(sc) * BR);
        prefetch_tile(map, g.phys(sc) * BR, g.phys(sc) * BR);
      }
      __syncwarp();
    }
  } else if (warp == 5) {
    // publisher: every final block to B (global), then its release flag
    for (int64_t t = 0; t < NB; t++) {
      const int slot = (int)(t % HR);
      wait_sflag_ge_slow(&sm.fin[slot], (int)(2 * (t + 1)));
      const int64_t IB = g.phys(t);
      const int nvs = g.nv(t);
      for (int j = lane; j < nvs; j += 32) Bc[IB * BR + g.kof(t, j)] = sm.yh[slot][j];
      __syncwarp();
      if (lane == 0) {
        dev::jitter((unsigned)t);
        st_release_gpu(yflag + t, a.epoch);
        st_rel_cta(&sm.pdone, (int)(t + 1));
      }
      EBV_CT(t, 11);
      __syncwarp();
    }
  }
}

template <bool FWD, int NRT>
__global__ void __launch_bounds__(NT, 1) solve_chain_kernel(const __grid_constant__ CUtensorMap map,
                                                             const __grid_constant__ CUtensorMap mapq, Args a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ int s_ticket;
  Geo<FWD> g;
  g.LU = a.LU;
  g.lda = a.lda;
  g.n = a.n;
  g.NB = (a.n + BR - 1) / BR;
  g.nvlast = (int)(a.n - (g.NB - 1) * BR);
  const int64_t nunits = g.NB * a.ngroups;      // helper units: (block, column group), blocks ascending
  const int64_t nhelp = (nunits + (NT / 64) - 1) / (NT / 64);
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int64_t tk = s_ticket;
    __syncthreads();
    if (tk >= a.nr + nhelp) return;
    if (tk < a.nr) {
      ChainSmem& sm = *reinterpret_cast<ChainSmem*>(smraw);
      if (threadIdx.x < HR) {
        sm.prog[threadIdx.x] = 0;
        sm.fin[threadIdx.x] = 0;
      }
      if (threadIdx.x == 0) {
        sm.sdone = 0;
        sm.pdone = 0;
        mbar_init(&sm.mbar_d[0], 1);
        mbar_init(&sm.mbar_d[1], 1);
        for (int w = 0; w < 4; w++)
          for (int k = 0; k < NSLOT; k++) mbar_init(&sm.mbar_s[w][k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        fence_proxy_async();
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        issue_diag<FWD>(&map, g, sm, 0);
        if (g.NB > 1) issue_diag<FWD>(&map, g, sm, 1);
      }
      chain_cta<FWD>(a, &map, &mapq, g, sm, (int)tk);
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&sm.mbar_d[0])) : "memory");
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&sm.mbar_d[1])) : "memory");
        for (int w = 0; w < 4; w++)
          for (int k = 0; k < NSLOT; k++)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&sm.mbar_s[w][k])) : "memory");
      }
      __syncthreads();
    } else {
      HelperSmem& hs = *reinterpret_cast<HelperSmem*>(smraw);
      const int unit = threadIdx.x / 64, tid = threadIdx.x % 64;
      if (threadIdx.x < NT / 64) {
        mbar_init(&hs.mbar[threadIdx.x][0], 1);
        mbar_init(&hs.mbar[threadIdx.x][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      }
      __syncthreads();
      uint32_t uses[2] = {0u, 0u};
      const int64_t u = (tk - a.nr) * (NT / 64) + unit;
      if (u < nunits) helper_unit<FWD, NRT>(a, &map, g, hs, u / a.ngroups, (int)(u % a.ngroups), tid, unit, uses);
      __syncthreads();
      if (threadIdx.x < NT / 64) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&hs.mbar[threadIdx.x][0])) : "memory");
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&hs.mbar[threadIdx.x][1])) : "memory");
      }
      __syncthreads();
    }
  }
}

template <bool FWD, int NRT>
cudaError_t launch_sweep(const CUtensorMap& map, const CUtensorMap& mapq, const Args& a, cudaStream_t s) {
  const void* fn = reinterpret_cast<const void*>(solve_chain_kernel<FWD, NRT>);
  cudaError_t e = ensure_max_dyn_smem(fn, (int)kSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_chain_kernel<FWD, NRT>, NT, kSmem);
  if (per_sm < 1) per_sm = 1;
  const int64_t NB = (a.n + BR - 1) / BR;
  const int64_t want = a.nr + (NB * a.ngroups + (NT / 64) - 1) / (NT / 64);
  const int64_t cap = (int64_t)sms * per_sm;
  const int64_t grid = want < cap ? want : cap;
  solve_chain_kernel<FWD, NRT><<<(unsigned)grid, NT, kSmem, s>>>(map, mapq, a);
  return cudaGetLastError();
}

}  // namespace

bool solve_chain_eligible(int64_t n, const double* LU, int64_t lda, int64_t nrhs) {
  alignas(64) unsigned char probe[128];
  return n >= 2 && n % 2 == 0 && lda % 2 == 0 && (reinterpret_cast<uintptr_t>(LU) & 15) == 0 && nrhs >= 1 &&
         n <= INT32_MAX && make_tma_map_2d(probe, LU, n, n, lda, BR, HT);
}

int64_t solve_chain_flags(int64_t n) {   // ints per sweep: yflag[MAXC][NB] + hflag[MAXC][NB] + ticket
  const int64_t NB = (n + BR - 1) / BR;
  return (int64_t)(2 * MAXC) * NB + 4;
}

cudaError_t launch_solve_chain(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                               int* flags_ws, int64_t epoch, cudaStream_t s) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int64_t per = solve_chain_flags(n);
  const int64_t NB = (n + BR - 1) / BR;
  CUtensorMap map, mapq;
  if (!make_tma_map_2d(&map, LU, n, n, lda, BR, HT) || !make_tma_map_2d(&mapq, LU, n, n, lda, BR, QT))
    return cudaErrorNotSupported;
  int64_t idx = 0;
  for (int64_t c0 = 0; c0 < nrhs; c0 += MAXC, idx++) {
    const int nr = (int)((nrhs - c0) < MAXC ? (nrhs - c0) : MAXC);
    for (int pass = 0; pass < 2; pass++) {
      int* base = flags_ws + (pass)*per;
      Args a;
      a.n = n;
      a.LU = LU;
      a.lda = lda;
      a.B = B + c0 * ldb;
      a.ldb = ldb;
      a.nr = nr;
      a.ticket = base + (2 * MAXC) * NB;
      a.yflag = base;
      a.hflag = base + MAXC * NB;
      // helper column groups of up to kCGW right-hand sides: a (block,
      // group) unit applies its tiles to kCGW columns only (16 columns in
      // one unit made the helpers the limit: a 4x longer fma stream per tile)
      // (measured: 4 columns per group beat 2 and 8 — n = 32768 x 16 RHS
      // 8.9 ms vs 12.4 / 10.1; n = 8192 x 16 0.90 vs 1.03 / 0.90)
      a.cgw = nr < kCGW ? nr : kCGW;
      a.ngroups = (nr + a.cgw - 1) / a.cgw;
      a.epoch = (int)(((epoch + idx * 2 + pass) % 0x3FFFFFF0) + 1);
      cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
      if (a.cgw == 1) e = pass == 0 ? launch_sweep<true, 1>(map, mapq, a, s) : launch_sweep<false, 1>(map, mapq, a, s);
      else if (a.cgw <= 2) e = pass == 0 ? launch_sweep<true, 2>(map, mapq, a, s) : launch_sweep<false, 2>(map, mapq, a, s);
      else if (a.cgw <= 4) e = pass == 0 ? launch_sweep<true, 4>(map, mapq, a, s) : launch_sweep<false, 4>(map, mapq, a, s);
      else e = pass == 0 ? launch_sweep<true, 8>(map, mapq, a, s) : launch_sweep<false, 8>(map, mapq, a, s);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

int64_t solve_chain_epochs(int64_t nrhs) { return 2 * ((nrhs + MAXC - 1) / MAXC); }

}  // namespace ebv

EBV_DEBUG_SETTER(set_debug_solve_chain)
