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
#include "ebv_internal.cuh"
#include "ebv_device.cuh"

namespace ebv {
namespace {

constexpr int BR = 64;        // rows per block
constexpr int HL = 6;         // helpers apply tiles s <= t - HL; the chain the last HL-1
constexpr int HR = 8;         // y-history ring (steps)
constexpr int NT = 192;       // threads per CTA (6 warps; helpers: 3 units of 64)
constexpr int MAXC = 16;      // right-hand sides per launch (helper accumulators: NRT <= MAXC)
constexpr int RING = 16;      // absorber register look-ahead (columns; double2 = 4 registers each)

struct ChainSmem {
  double diag[2][BR * BR];    // diagonal tiles, column-major, double buffered
  double yh[HR][BR];          // y (x) values of recent steps, in processing order
  int prog[HR];               // step s: s*128 + number of values produced
  int fin[HR];                // step s final: 2*(s+1) + redo bit
  int sdone;                  // solver steps completed
  int pdone;                  // steps published to global memory
  unsigned long long mbar[2];
};
struct HelperSmem {
  double ys[NT / 64][BR * MAXC];   // per unit: the published y of one block
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

// the absorbers' wait for the next group of 8 produced values
__device__ __noinline__ int wait_prog(const int* p, int need) {
  int cur = ld_acq_cta(p);
  dev::SpinGuard g;
  while (cur < need) {
    g.poll();
    cur = ld_acq_cta(p);
  }
  return cur;
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void unit_sync(int unit) {   // 64 threads of one helper unit
  asm volatile("bar.sync %0, 64;\n" ::"r"(unit + 1) : "memory");
}

struct Args {
  int64_t n;
  const double* LU;
  int64_t lda;
  double* B;
  int64_t ldb;
  int nr;          // right-hand sides (chain CTAs) in this launch, <= MAXC
  int* ticket;
  int* yflag;      // [nr][NB], logical block order
  int* hflag;      // [NB]
  int epoch;
};

template <bool FWD>
struct Geo {
  int64_t n, NB;
  int nvlast;   // valid rows of the last physical block
  __device__ __forceinline__ int64_t phys(int64_t s) const { return FWD ? s : NB - 1 - s; }
  __device__ __forceinline__ int nv(int64_t s) const { return phys(s) == NB - 1 ? nvlast : BR; }
  // processing index j of logical block s -> row / column offset inside the block
  __device__ __forceinline__ int kof(int64_t s, int j) const { return FWD ? j : nv(s) - 1 - j; }
};

// ---------------------------------------------------------------------------- helper
template <bool FWD, int NRT>
__device__ void helper_unit(const Args& a, const Geo<FWD>& g, int64_t tb, int tid, int unit, double* ys) {
  const int64_t ntiles = tb - HL + 1;
  if (ntiles <= 0) return;                      // blocks the chain absorbs entirely: nothing to do
  const int64_t IB = g.phys(tb);
  const int64_t row = IB * BR + tid;
  const bool rv = row < a.n;
  const int nr = a.nr;
  double acc[NRT];
#pragma unroll
  for (int c = 0; c < NRT; c++) acc[c] = (rv && c < nr) ? a.B[row + (int64_t)c * a.ldb] : 0.0;
  for (int64_t tj = 0; tj < ntiles; tj++) {
    const int64_t JB = g.phys(tj);
    const int nvj = g.nv(tj);
    double l[BR];
    const double* src = a.LU + (rv ? row : 0) + JB * BR * a.lda;
#pragma unroll
    for (int k = 0; k < BR; k++) l[k] = (rv && k < nvj) ? __ldg(src + (int64_t)k * a.lda) : 0.0;
    if (tid < nr) wait_gflag(a.yflag + (int64_t)tid * g.NB + tj, a.epoch, 100);
    unit_sync(unit);
    for (int idx = tid; idx < BR * nr; idx += 64) {
      const int k = idx % BR, c = idx / BR;
      ys[k * NRT + c] = (k < nvj) ? __ldcg(a.B + JB * BR + k + (int64_t)c * a.ldb) : 0.0;
    }
    unit_sync(unit);
    if (FWD) {
#pragma unroll
      for (int k = 0; k < BR; k++)
#pragma unroll
        for (int c = 0; c < NRT; c++)
          if (c < nr) acc[c] = fma(-l[k], ys[k * NRT + c], acc[c]);
    } else {
#pragma unroll
      for (int k = BR - 1; k >= 0; k--)
#pragma unroll
        for (int c = 0; c < NRT; c++)
          if (c < nr) acc[c] = fma(-l[k], ys[k * NRT + c], acc[c]);
    }
    unit_sync(unit);                           // ys is restaged for the next tile
  }
#pragma unroll
  for (int c = 0; c < NRT; c++)
    if (rv && c < nr) a.B[row + (int64_t)c * a.ldb] = acc[c];
  unit_sync(unit);
  if (tid == 0) {
    dev::jitter((unsigned)tb);
    st_release_gpu(a.hflag + tb, a.epoch);
  }
}

// ---------------------------------------------------------------------------- chain
// absorb tiles (t, s) for s in [s0, t) into rows 2l, 2l+1 of block t (v0, v1),
// in logical order, each term as soon as its value is produced.  The L (U)
// values stream through a register ring RING columns ahead (the loader warp
// prefetched the tiles to L2); the term order inside a tile is the
// processing order j (column k = j forward, 63 - j backward).
template <bool FWD>
__device__ __forceinline__ void absorb_redo(const Args& a, const Geo<FWD>& g, ChainSmem& sm, int64_t s,
                                            const double* rowp, double& v0, double& v1) {
  const int nvs = g.nv(s);
  const int slot = (int)(s % HR);
  for (int jj = 0; jj < nvs; jj++) {
    const double2 l = __ldg(reinterpret_cast<const double2*>(rowp + (g.phys(s) * BR + g.kof(s, jj)) * a.lda));
    const double y = sm.yh[slot][jj];
    v0 = fma(-l.x, y, v0);
    v1 = fma(-l.y, y, v1);
  }
}

template <bool FWD>
__device__ __forceinline__ void absorb(const Args& a, const Geo<FWD>& g, ChainSmem& sm, int64_t t, int64_t s0,
                                       int lane, double& v0, double& v1) {
  if (s0 >= t) return;
  const int64_t r0 = g.phys(t) * BR + 2 * lane;
  const double* rowp = a.LU + (r0 < a.n ? r0 : 0);    // n even: rows 2l, 2l+1 valid together
  const int64_t lda = a.lda;
  const int64_t dl = FWD ? lda : -lda;                 // next column in processing order
  // column k(j) of tile s: forward k = j, backward k = 63 - j (full tiles)
  auto col0 = [&](int64_t s) -> const double* { return rowp + (g.phys(s) * BR + (FWD ? 0 : BR - 1)) * lda; };
  double2 ring[RING];
  const double* pn = col0(s0);                         // next column to load into the ring
  if (g.nv(s0) == BR) {
#pragma unroll
    for (int i = 0; i < RING; i++) {
      ring[i] = __ldg(reinterpret_cast<const double2*>(pn));
      pn += dl;
    }
  }
  for (int64_t s = s0; s < t; s++) {
    const int slot = (int)(s % HR);
    const int base = (int)(s * 128);
    const bool nextfull = s + 1 < t && g.nv(s + 1) == BR;
    if (g.nv(s) != BR) {
      // the ragged block (backward: logical block 0): plain loads
      wait_sflag_ge(&sm.fin[slot], (int)(2 * (s + 1)));
      absorb_redo<FWD>(a, g, sm, s, rowp, v0, v1);
      if (nextfull) {
        pn = col0(s + 1);
#pragma unroll
        for (int i = 0; i < RING; i++) {
          ring[i] = __ldg(reinterpret_cast<const double2*>(pn));
          pn += dl;
        }
      }
      continue;
    }
    const double ck0 = v0, ck1 = v1;   // checkpoint (backward redo)
    int cur = -1;
#pragma unroll 1
    for (int jc = 0; jc < BR; jc += RING) {
      const bool last = jc + RING == BR;                 // the loads of this chunk go to the next tile
      if (last && nextfull) pn = col0(s + 1);
      const bool ld = !last || nextfull;
#pragma unroll
      for (int i = 0; i < RING; i++) {
        const int j = jc + i;
        const double2 l = ring[i];
        if (ld) {
          ring[i] = __ldg(reinterpret_cast<const double2*>(pn));
          pn += dl;
        }
        if ((i & 7) == 0 && cur < base + j + 8) cur = wait_prog(&sm.prog[slot], base + j + 8);
        const double y = sm.yh[slot][j];
        v0 = fma(-l.x, y, v0);
        v1 = fma(-l.y, y, v1);
      }
    }
    if (!FWD) {
      // the tile's values must be final (verified) before the next tile; on a
      // redo of step s, restore and re-apply its corrected values
      wait_sflag_ge(&sm.fin[slot], (int)(2 * (s + 1)));
      if (ld_acq_cta(&sm.fin[slot]) & 1) {
        v0 = ck0;
        v1 = ck1;
        absorb_redo<FWD>(a, g, sm, s, rowp, v0, v1);
      }
    }
  }
}

// solve diagonal block t (rows 2l, 2l+1 in v0, v1; all earlier tiles applied)
template <bool FWD>
__device__ __forceinline__ void solve_diag(const Geo<FWD>& g, ChainSmem& sm, int64_t t, int lane, double& v0,
                                           double& v1) {
  const int buf = (int)(t & 1);
  if (t >= HR) wait_sflag_ge(&sm.pdone, (int)(t - HR + 1));   // slot t % HR published (free)
  mbar_wait(&sm.mbar[buf], (uint32_t)((t >> 1) & 1));
  const double* D = sm.diag[buf];
  const int slot = (int)(t % HR);
  const int nvs = g.nv(t);
  const int np = nvs / 2;
  int* prog = &sm.prog[slot];
  double* yh = sm.yh[slot];
  if (FWD) {
#pragma unroll 4
    for (int p = 0; p < np; p++) {
      const double2 c0 = *reinterpret_cast<const double2*>(D + (2 * p) * BR + 2 * lane);      // L(2l.., 2p)
      const double2 c1 = *reinterpret_cast<const double2*>(D + (2 * p + 1) * BR + 2 * lane);  // L(2l.., 2p+1)
      const double t1 = fma(-c0.y, v0, v1);             // owner lane: y_{2p+1} from its own y_{2p}
      const double y0 = __shfl_sync(0xffffffffu, v0, p);
      const double y1 = __shfl_sync(0xffffffffu, t1, p);
      if (lane == p) {
        yh[2 * p] = v0;
        yh[2 * p + 1] = t1;
        st_rel_cta(prog, (int)(t * 128) + 2 * p + 2);
      }
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
        yh[j] = q1;
        yh[j + 1] = q0;
        st_rel_cta(prog, (int)(t * 128) + j + 2);
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
        if (lane == p) {
          yh[j] = q1;
          yh[j + 1] = q0;
        }
        const double n0 = fma(-c0.x, x0, fma(-c1.x, x1, v0));
        const double n1 = fma(-c0.y, x0, fma(-c1.y, x1, v1));
        v0 = lane < p ? n0 : (lane == p ? q0 : v0);
        v1 = lane < p ? n1 : (lane == p ? q1 : v1);
      }
      __syncwarp();
    }
    if (lane == 0) st_rel_cta(&sm.fin[slot], (int)(2 * (t + 1)) + redo);
  }
  __syncwarp();
  if (lane == 0) st_rel_cta(&sm.sdone, (int)(t + 1));   // diag buffer (t & 1) may be refilled
}

template <bool FWD>
__device__ void chain_cta(const Args& a, const Geo<FWD>& g, ChainSmem& sm, int col) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t NB = g.NB;
  double* Bc = a.B + (int64_t)col * a.ldb;
  int* yflag = a.yflag + (int64_t)col * NB;
  if (warp < 4) {
    for (int64_t t = warp; t < NB; t += 4) {
      // pick up block t: the helper's partial sums (tiles s <= t - HL)
      const int64_t IB = g.phys(t);
      const int64_t r0 = IB * BR + 2 * lane;
      if (t - HL + 1 > 0) {
        if (lane == 0) wait_gflag(a.hflag + t, a.epoch, 64);
        __syncwarp();
      }
      double v0 = 0.0, v1 = 0.0;
      if (r0 < a.n) {
        const double2 b2 = __ldcg(reinterpret_cast<const double2*>(Bc + r0));
        v0 = b2.x;
        v1 = b2.y;
      }
      const int64_t s0 = t - HL + 1 > 0 ? t - HL + 1 : 0;
      absorb<FWD>(a, g, sm, t, s0, lane, v0, v1);
      solve_diag<FWD>(g, sm, t, lane, v0, v1);
    }
  } else if (warp == 4) {
    // loader: diagonal tile of step t into buffer t & 1 once step t - 2 is done;
    // L2 prefetch of the tiles the block picked up after step t absorbs
    for (int64_t t = 0; t < NB; t++) {
      const int buf = (int)(t & 1);
      if (t >= 2) wait_sflag_ge(&sm.sdone, (int)(t - 1));
      const int64_t IB = g.phys(t);
      const int nvs = g.nv(t);
      const uint32_t colbytes = (uint32_t)nvs * 8u;
      if (lane == 0) mbar_expect_tx(&sm.mbar[buf], colbytes * (uint32_t)nvs);
      __syncwarp();
      for (int k = lane; k < nvs; k += 32)
        bulk_g2s(sm.diag[buf] + k * BR, a.LU + IB * BR + (IB * BR + k) * a.lda, colbytes, &sm.mbar[buf]);
      // block t + 4 is picked up after step t; it absorbs tiles t-1 .. t+3
      const int64_t tp = t + 4;
      if (tp < NB) {
        const int64_t TB = g.phys(tp);
        const int rows = g.nv(tp);
        for (int64_t s = (tp - HL + 1 > 0 ? tp - HL + 1 : 0); s < tp; s++) {
          const int64_t JB = g.phys(s);
          const int nvj = g.nv(s);
          for (int k = lane; k < nvj; k += 32)
            prefetch_l2(a.LU + TB * BR + (JB * BR + k) * a.lda, (uint32_t)rows * 8u);
        }
      }
    }
  } else {
    // publisher: every final block to B (global), then its release flag
    for (int64_t t = 0; t < NB; t++) {
      const int slot = (int)(t % HR);
      wait_sflag_ge(&sm.fin[slot], (int)(2 * (t + 1)));
      const int64_t IB = g.phys(t);
      const int nvs = g.nv(t);
      for (int j = lane; j < nvs; j += 32) Bc[IB * BR + g.kof(t, j)] = sm.yh[slot][j];
      __syncwarp();
      if (lane == 0) {
        dev::jitter((unsigned)t);
        st_release_gpu(yflag + t, a.epoch);
        st_rel_cta(&sm.pdone, (int)(t + 1));
      }
      __syncwarp();
    }
  }
}

template <bool FWD, int NRT>
__global__ void __launch_bounds__(NT, 1) solve_chain_kernel(Args a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ int s_ticket;
  Geo<FWD> g;
  g.n = a.n;
  g.NB = (a.n + BR - 1) / BR;
  g.nvlast = (int)(a.n - (g.NB - 1) * BR);
  const int64_t nunits = g.NB;
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
        sm.prog[threadIdx.x] = -1;
        sm.fin[threadIdx.x] = 0;
      }
      if (threadIdx.x == 0) {
        sm.sdone = 0;
        sm.pdone = 0;
        mbar_init(&sm.mbar[0], 1);
        mbar_init(&sm.mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      }
      __syncthreads();
      chain_cta<FWD>(a, g, sm, (int)tk);
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&sm.mbar[0])) : "memory");
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&sm.mbar[1])) : "memory");
      }
      __syncthreads();
    } else {
      HelperSmem& hs = *reinterpret_cast<HelperSmem*>(smraw);
      const int unit = threadIdx.x / 64, tid = threadIdx.x % 64;
      const int64_t tb = (tk - a.nr) * (NT / 64) + unit;
      if (tb < nunits) helper_unit<FWD, NRT>(a, g, tb, tid, unit, hs.ys[unit]);
      __syncthreads();
    }
  }
}

template <bool FWD, int NRT>
cudaError_t launch_sweep(const Args& a, cudaStream_t s) {
  const void* fn = reinterpret_cast<const void*>(solve_chain_kernel<FWD, NRT>);
  cudaError_t e = ensure_max_dyn_smem(fn, (int)kSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_chain_kernel<FWD, NRT>, NT, kSmem);
  if (per_sm < 1) per_sm = 1;
  const int64_t NB = (a.n + BR - 1) / BR;
  const int64_t want = a.nr + (NB + (NT / 64) - 1) / (NT / 64);
  const int64_t cap = (int64_t)sms * per_sm;
  const int64_t grid = want < cap ? want : cap;
  solve_chain_kernel<FWD, NRT><<<(unsigned)grid, NT, kSmem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool solve_chain_eligible(int64_t n, const double* LU, int64_t lda, int64_t nrhs) {
  return n >= 2 && n % 2 == 0 && lda % 2 == 0 && (reinterpret_cast<uintptr_t>(LU) & 15) == 0 && nrhs >= 1;
}

int64_t solve_chain_flags(int64_t n) {   // ints per sweep and column group: yflag[MAXC][NB] + hflag[NB] + ticket
  const int64_t NB = (n + BR - 1) / BR;
  return (int64_t)(MAXC + 1) * NB + 4;
}

cudaError_t launch_solve_chain(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                               int* flags_ws, int64_t epoch, cudaStream_t s) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const int64_t per = solve_chain_flags(n);
  const int64_t NB = (n + BR - 1) / BR;
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
      a.ticket = base + (MAXC + 1) * NB;
      a.yflag = base;
      a.hflag = base + MAXC * NB;
      a.epoch = (int)(((epoch + idx * 2 + pass) % 0x3FFFFFF0) + 1);
      cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(int), s);
      if (e != cudaSuccess) return e;
      if (nr == 1) e = pass == 0 ? launch_sweep<true, 1>(a, s) : launch_sweep<false, 1>(a, s);
      else if (nr <= 4) e = pass == 0 ? launch_sweep<true, 4>(a, s) : launch_sweep<false, 4>(a, s);
      else e = pass == 0 ? launch_sweep<true, MAXC>(a, s) : launch_sweep<false, MAXC>(a, s);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

int64_t solve_chain_epochs(int64_t nrhs) { return 2 * ((nrhs + MAXC - 1) / MAXC); }

}  // namespace ebv

EBV_DEBUG_SETTER(set_debug_solve_chain)
