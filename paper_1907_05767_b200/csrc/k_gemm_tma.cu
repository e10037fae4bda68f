// k_gemm_tma.cu — the DMMA trailing update C <- C - A*B (Eq 6-c) with
// its operand tiles staged by the Tensor Memory Accelerator.
//
// Same arithmetic contract as k_gemm.cu (bitwise: per entry the fma chain
// over ascending k from its input value; DMMA.8x8x4 rounds like a sequential
// fma chain — probe M3).  Only the data movement differs:
//   * one producer warp issues cp.async.bulk.tensor (TMA) loads of the A
//     (L panel) and B (U panel) k-slices into a STAGES-deep ring of shared
//     memory buffers, signalling an mbarrier with the transaction bytes;
//   * consumer warps wait on the stage's "full" barrier, run the DMMA
//     fragments out of shared memory and release the stage through an
//     "empty" barrier — no __syncthreads in the k loop.
// The TMA boxes are padded ({BM+8, KC} for A, {KC+2, BN} for B) so the smem
// images have the conflict-free strides of k_gemm.cu; out-of-range rows /
// columns / k are zero-filled by the TMA unit (exactly neutral for the fma
// chain).  Needs 16-byte aligned bases and even leading dimensions
// (TMA global strides are multiples of 16 bytes); launch_gemm_sub falls
// back to the cp.async kernel otherwise.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "ebv_internal.cuh"

namespace ebv {
namespace {

template <int BM_, int BN_, int WM_, int WN_, int KC_, int STAGES_, int MINB_>
struct TCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, KC = KC_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int NCW = WM * WN;               // consumer warps (thread 0 also produces)
  static constexpr int THREADS = 32 * NCW;
  static constexpr int MT = BM / WM / 8;
  static constexpr int NT = BN / WN / 8;
  static constexpr int AST = BM + 8;                // TMA box dim0 for A
  static constexpr int BSTR = KC + 2;               // TMA box dim0 for B
  static constexpr int A_STAGE = KC * AST;          // doubles
  static constexpr int B_STAGE = BN * BSTR;
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 128;
  static_assert((A_STAGE * 8) % 128 == 0 && (B_STAGE * 8) % 128 == 0, "TMA destinations must stay 128B aligned");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t M,
                    int64_t N, int64_t K, double* __restrict__ Cm, int64_t ldc, int tilesM, int tilesN, int G) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // 128-byte aligned carve-up
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  double* sA = reinterpret_cast<double*>(base);
  double* sB = sA + C::STAGES * C::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_STAGE);
  uint64_t* empty = full + C::STAGES;

  // tile order: groups of G consecutive M-tiles, M fastest inside a group,
  // so the CTAs in flight share the L-panel rows of the group and stream
  // the U panel once per group
  int bid = blockIdx.x;
  int group = bid / (G * tilesN);
  int first_m = group * G;
  int gsz = min(tilesM - first_m, G);
  int tm = first_m + (bid % (G * tilesN)) % gsz;
  int tn = (bid % (G * tilesN)) / gsz;
  const int m0 = tm * C::BM, n0 = tn * C::BN;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nk = (int)((K + C::KC - 1) / C::KC);

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // Producer duty sits with warp 0 (lane 0 issues): it keeps STAGES-1
  // k-slices in flight and refills a slot once every warp has released it.
  // The whole warp takes part in the waits so that it stays converged for
  // the warp-synchronous mma.sync that follows.
  auto produce = [&](int j) {
    const int sj = j % C::STAGES;
    if (j >= C::STAGES) mbar_wait(&empty[sj], ((j / C::STAGES) + 1) & 1);
    if (lane == 0) {
      mbar_expect_tx(&full[sj], C::STAGE_BYTES);
      tma_load_2d(sA + sj * C::A_STAGE, &tmA, m0, j * C::KC, &full[sj]);
      tma_load_2d(sB + sj * C::B_STAGE, &tmB, j * C::KC, n0, &full[sj]);
    }
    __syncwarp();
  };
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    for (int j = 0; j < C::STAGES - 1 && j < nk; j++) produce(j);
  }

  // -------------------------------------------------------------- consumers
  // The accumulators hold the TRANSPOSED tile: the mma computes
  // D' = (-B^T) A^T + C^T, i.e. D'[n][m] = c_mn + sum_k (-b_kn) a_mk, the very
  // same products and the same ascending-k fma chain as C - A B (bitwise).
  // Lane (g, t) then owns C[m = 2t, 2t+1][n = g]: two consecutive rows of a
  // column-major column, one 16-byte load / store per fragment.
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;
  const int64_t mb = (int64_t)m0 + wm * (C::MT * 8) + 2 * t;   // + mt*8 (+q)
  const int64_t nb = (int64_t)n0 + wn * (C::NT * 8) + g;       // + nt*8
  const bool vec_c = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(Cm) & 15) == 0) &&
                     (m0 + C::BM <= M) && (n0 + C::BN <= N);
  double acc[C::MT][C::NT][2];
  if (vec_c) {
#pragma unroll
    for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
      for (int nt = 0; nt < C::NT; nt++) {
        const double2 v = *reinterpret_cast<const double2*>(Cm + (mb + mt * 8) + (nb + nt * 8) * ldc);
        acc[mt][nt][0] = v.x;
        acc[mt][nt][1] = v.y;
      }
  } else {
#pragma unroll
    for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
      for (int nt = 0; nt < C::NT; nt++)
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const int64_t m = mb + mt * 8 + q, n = nb + nt * 8;
          acc[mt][nt][q] = (m < M && n < N) ? Cm[m + n * ldc] : 0.0;
        }
  }

  for (int kt = 0; kt < nk; kt++) {
    const int s = kt % C::STAGES;
    if (warp == 0 && kt + C::STAGES - 1 < nk) produce(kt + C::STAGES - 1);
    mbar_wait(&full[s], (kt / C::STAGES) & 1);
    __syncwarp();
    const double* a = sA + s * C::A_STAGE + wm * (C::MT * 8) + g;
    const double* b = sB + s * C::B_STAGE + (wn * (C::NT * 8) + g) * C::BSTR + t;
#pragma unroll
    for (int ks = 0; ks < C::KC / 4; ks++) {
      double af[C::MT], bf[C::NT];
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++) af[mt] = a[(ks * 4 + t) * C::AST + mt * 8];
#pragma unroll
      for (int nt = 0; nt < C::NT; nt++) bf[nt] = -b[nt * 8 * C::BSTR + ks * 4];
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++) dmma(acc[mt][nt][0], acc[mt][nt][1], bf[nt], af[mt]);
    }
    // all lanes' (generic-proxy) shared-memory reads of this stage are
    // ordered before the TMA (async-proxy) writes that may refill the slot
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  if (vec_c) {
#pragma unroll
    for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
      for (int nt = 0; nt < C::NT; nt++)
        *reinterpret_cast<double2*>(Cm + (mb + mt * 8) + (nb + nt * 8) * ldc) =
            make_double2(acc[mt][nt][0], acc[mt][nt][1]);
  } else {
#pragma unroll
    for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
      for (int nt = 0; nt < C::NT; nt++)
#pragma unroll
        for (int q = 0; q < 2; q++) {
          const int64_t m = mb + mt * 8 + q, n = nb + nt * 8;
          if (m < M && n < N) Cm[m + n * ldc] = acc[mt][nt][q];
        }
  }
}

// Persistent form: grid = resident CTAs, each walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ... (same grouped raster).  The TMA ring runs on
// one global slice counter across the CTA's tiles, so the producer prefetches
// the next tile's first slices while the current tile finishes, and each tile
// prefetches the next tile's C block into L2 — the tile epilogue / prologue
// no longer drains the DMMA pipe.  Per entry the same fma chain (bitwise).
template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    gemm_tma_persistent_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                               int64_t M, int64_t N, int64_t K, double* __restrict__ Cm, int64_t ldc, int tilesM,
                               int tilesN) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  double* sA = reinterpret_cast<double*>(base);
  double* sB = sA + C::STAGES * C::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_STAGE);
  uint64_t* empty = full + C::STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nk = (int)((K + C::KC - 1) / C::KC);
  const int ntiles = tilesM * tilesN;
  const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const long long total = (long long)my_tiles * nk;
  auto coords = [&](int ti, int& m0, int& n0) {
    const int G = 8;
    const int bid = blockIdx.x + ti * gridDim.x;
    const int group = bid / (G * tilesN);
    const int first_m = group * G;
    const int gsz = min(tilesM - first_m, G);
    m0 = (first_m + (bid % (G * tilesN)) % gsz) * C::BM;
    n0 = ((bid % (G * tilesN)) / gsz) * C::BN;
  };

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // producer cursor (warp 0): slot ps, its empty-barrier phase pph, tile pt, slice pk
  int ps = 0, pt = 0, pk = 0, pm0 = 0, pn0 = 0;
  uint32_t pph = 0;
  long long pj = 0;
  if (my_tiles > 0) coords(0, pm0, pn0);
  auto produce = [&]() {
    if (pj >= C::STAGES) mbar_wait(&empty[ps], pph ^ 1u);
    if (lane == 0) {
      const int m0 = pm0, n0 = pn0, kt = pk;
      mbar_expect_tx(&full[ps], C::STAGE_BYTES);
      tma_load_2d(sA + ps * C::A_STAGE, &tmA, m0, kt * C::KC, &full[ps]);
      tma_load_2d(sB + ps * C::B_STAGE, &tmB, kt * C::KC, n0, &full[ps]);
    }
    __syncwarp();
    ++pj;
    if (++ps == C::STAGES) { ps = 0; pph ^= 1u; }
    if (++pk == nk) { pk = 0; if (++pt < my_tiles) coords(pt, pm0, pn0); }
  };
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    while (pj < C::STAGES - 1 && pj < total) produce();
  }

  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;
  int cs = 0;
  uint32_t cph = 0;
  for (int ti = 0; ti < my_tiles; ti++) {
    int m0, n0;
    coords(ti, m0, n0);
    const int64_t mb = (int64_t)m0 + wm * (C::MT * 8) + 2 * t;
    const int64_t nb = (int64_t)n0 + wn * (C::NT * 8) + g;
    const bool vec_c = ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(Cm) & 15) == 0) && (m0 + C::BM <= M) &&
                       (n0 + C::BN <= N);
    double acc[C::MT][C::NT][2];
    if (vec_c) {
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++) {
          const double2 v = *reinterpret_cast<const double2*>(Cm + (mb + mt * 8) + (nb + nt * 8) * ldc);
          acc[mt][nt][0] = v.x;
          acc[mt][nt][1] = v.y;
        }
    } else {
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++)
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int64_t m = mb + mt * 8 + q, n = nb + nt * 8;
            acc[mt][nt][q] = (m < M && n < N) ? Cm[m + n * ldc] : 0.0;
          }
    }
    if (ti + 1 < my_tiles) {   // the next tile's C block into L2 (one 128-byte line per thread and column slice)
      int pm0, pn0;
      coords(ti + 1, pm0, pn0);
      for (int idx = tid; idx < C::BN * (C::BM / 16); idx += C::THREADS) {
        const int64_t col = pn0 + idx / (C::BM / 16), row = pm0 + (idx % (C::BM / 16)) * 16;
        if (col < N && row < M)
          asm volatile("prefetch.global.L2 [%0];\n" ::"l"(Cm + row + col * ldc));
      }
    }
    for (int kt = 0; kt < nk; kt++) {
      const int s = cs;
      if (warp == 0 && pj < total) produce();
      mbar_wait(&full[s], cph);
      __syncwarp();
      const double* a = sA + s * C::A_STAGE + wm * (C::MT * 8) + g;
      const double* b = sB + s * C::B_STAGE + (wn * (C::NT * 8) + g) * C::BSTR + t;
#pragma unroll
      for (int ks = 0; ks < C::KC / 4; ks++) {
        double af[C::MT], bf[C::NT];
#pragma unroll
        for (int mt = 0; mt < C::MT; mt++) af[mt] = a[(ks * 4 + t) * C::AST + mt * 8];
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++) bf[nt] = -b[nt * 8 * C::BSTR + ks * 4];
#pragma unroll
        for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
          for (int nt = 0; nt < C::NT; nt++) dmma(acc[mt][nt][0], acc[mt][nt][1], bf[nt], af[mt]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++cs == C::STAGES) { cs = 0; cph ^= 1u; }
    }
    if (vec_c) {
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++)
          *reinterpret_cast<double2*>(Cm + (mb + mt * 8) + (nb + nt * 8) * ldc) =
              make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    } else {
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++)
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int64_t m = mb + mt * 8 + q, n = nb + nt * 8;
            if (m < M && n < N) Cm[m + n * ldc] = acc[mt][nt][q];
          }
    }
  }
}

// M-tiles per rasterization group of gemm_tma_kernel (EBV_GEMM_GROUP;
// round 2: 32 — the U panel is streamed once per group, so 8 re-read it
// ~4 GB per rank-512 update at n = 32768; factor 708.3 -> 705.8 ms,
// 64 slower)
int raster_group() {
  static const int g = [] {
    const char* e = getenv("EBV_GEMM_GROUP");
    const int v = e ? atoi(e) : 32;
    return v > 0 ? v : 32;
  }();
  return g;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const double* ptr, int64_t rows, int64_t cols, int64_t ld, int box0, int box1) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <class C>
cudaError_t run_tma(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                    double* Cm, int64_t ldc, cudaStream_t s) {
  {
    cudaError_t e = ensure_max_dyn_smem(reinterpret_cast<const void*>(gemm_tma_kernel<C>), C::SMEM);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, M, K, lda, C::AST, C::KC) || !make_map(&mb, B, K, N, ldb, C::BSTR, C::BN))
    return cudaErrorNotSupported;
  const int64_t tm = (M + C::BM - 1) / C::BM, tn = (N + C::BN - 1) / C::BN;
  gemm_tma_kernel<C><<<(unsigned)(tm * tn), C::THREADS, C::SMEM, s>>>(ma, mb, M, N, K, Cm, ldc, (int)tm, (int)tn,
                                                                   raster_group());
  return cudaGetLastError();
}

template <class C>
cudaError_t run_tma_persistent(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                               int64_t ldb, double* Cm, int64_t ldc, cudaStream_t s) {
  cudaError_t ea = ensure_max_dyn_smem(reinterpret_cast<const void*>(gemm_tma_persistent_kernel<C>), C::SMEM);
  if (ea != cudaSuccess) return ea;
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gemm_tma_persistent_kernel<C>, C::THREADS, C::SMEM);
  const int slots = sms * (per > 0 ? per : 1);
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, M, K, lda, C::AST, C::KC) || !make_map(&mb, B, K, N, ldb, C::BSTR, C::BN))
    return cudaErrorNotSupported;
  const int64_t tm = (M + C::BM - 1) / C::BM, tn = (N + C::BN - 1) / C::BN;
  const int64_t grid = tm * tn < slots ? tm * tn : slots;
  gemm_tma_persistent_kernel<C><<<(unsigned)grid, C::THREADS, C::SMEM, s>>>(ma, mb, M, N, K, Cm, ldc, (int)tm,
                                                                           (int)tn);
  return cudaGetLastError();
}

//                     BM   BN  WM WN KC ST MINB
using TMid = TCfg<128, 64, 4, 2, 16, 4, 2>;     // 8 warps (32x32 warp tiles), 2 CTAs/SM
using TBig = TCfg<128, 128, 4, 4, 16, 4, 1>;    // 16 warps (32x32), 1 CTA/SM
using TBig8 = TCfg<128, 128, 2, 4, 16, 4, 1>;   // 8 warps (64x32), 1 CTA/SM
using TWide = TCfg<64, 128, 2, 4, 16, 4, 2>;    // 8 warps (32x32), 2 CTAs/SM
using TBig6 = TCfg<128, 128, 4, 4, 16, 6, 1>;   // 16 warps (32x32), 1 CTA/SM, 6-stage ring
using TMid3 = TCfg<128, 64, 4, 2, 16, 3, 2>;    // TMid with a 3-stage ring (less smem)

}  // namespace

bool make_tma_map_2d(void* map, const double* ptr, int64_t rows, int64_t cols, int64_t ld, int box0, int box1) {
  return make_map(reinterpret_cast<CUtensorMap*>(map), ptr, rows, cols, ld, box0, box1);
}

bool gemm_tma_eligible(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb) {
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return false;
  if ((lda & 1) || (ldb & 1)) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
  return get_encode() != nullptr;
}

cudaError_t launch_gemm_sub_tma(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double* Cm, int64_t ldc, int variant, cudaStream_t s) {
  switch (variant) {
    case 1: return run_tma<TBig>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    case 2: return run_tma<TBig8>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    case 3: return run_tma<TWide>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    case 4: return run_tma<TBig6>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    case 5: return run_tma<TMid3>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    case 6: return run_tma_persistent<TMid3>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    case 7: return run_tma_persistent<TMid>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
    default: return run_tma<TMid>(M, N, K, A, lda, B, ldb, Cm, ldc, s);
  }
}

}  // namespace ebv
