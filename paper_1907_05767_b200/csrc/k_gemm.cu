// k_gemm.cu — the trailing rank-k update of the blocked EbV LU as an FP64
// tensor-core (DMMA) contraction:  C <- C - A*B.
//
// Paper: Eq 6-c, A^(r) = A^(r-1) - L^(r-1) U^(r-1) / A_rr, applied for
// a block of consecutive steps k at once (the trailing matrix A^(r) of Eq 5-c,
// P:63).  Reading R3: the multiplier l_ik is formed first, the update is one
// fused multiply-add per step.
//
// Bitwise contract: every output entry is
//     c <- fma(-a_i,k, b_k,j, c)   for k = 0, 1, ..., K-1 (ascending)
// starting from its input value — exactly the oracle's per-entry sequence.
// This holds because (probe M3, profiles/r01_probe_dmma.jsonl) sm_100a's
// DMMA.8x8x4 computes d = fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c))))
// with one rounding per step, bit-identical to a sequential fma chain; the
// accumulator is initialized from C and k is never split.  reverse_k runs
// the chain over descending k (backward substitution order).  The negation
// of A is folded into the DMMA operand (SASS: DMMA.8x8x4 R, -Ra, Rb, R).
//
// B200 mapping: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) — tcgen05 has no f64
// kind on sm_100a — fed from shared memory that a multi-stage cp.async
// pipeline fills (16-byte copies when the operands are 16-byte aligned);
// padded layouts make every fragment load conflict-free:
//   A stage  [KC][BM+8]  (m contiguous, as in the column-major L panel;
//                         row stride = 64 B mod 128 -> k rows t, t+1 hit
//                         opposite bank halves)
//   B stage  [BN][KC+2]  (k contiguous, as in the column-major U panel;
//                         column stride 16 B mod 128 -> 8 columns spread)
// K / M / N tails are zero-filled: fma(-0, 0, c) == c bitwise for any c.
#include <cstdlib>

#include "ebv_internal.cuh"

namespace ebv {
namespace {

template <int BM_, int BN_, int WM_, int WN_, int KC_, int STAGES_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, KC = KC_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int MT = BM / WM / 8;   // m8 tiles per warp
  static constexpr int NT = BN / WN / 8;   // n8 tiles per warp
  static constexpr int AST = BM + 8;       // A stage row stride (doubles)
  static constexpr int BSTR = KC + 2;      // B stage column stride (doubles)
  static constexpr int A_STAGE = KC * AST;
  static constexpr int B_STAGE = BN * BSTR;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) * 8;
  static_assert(MT >= 1 && NT >= 1, "tile too small");
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
// 16-byte copy of two consecutive doubles; nvalid (0..2) of them are read,
// the rest of the 16 bytes are zero-filled.
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int nvalid) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = nvalid * 8;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <class C, int VEC>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    gemm_sub_kernel(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
                    const double* __restrict__ B, int64_t ldb, double* __restrict__ Cm, int64_t ldc,
                    int reverse_k, int tilesM, int tilesN, int64_t bsA, int64_t bsB, int64_t bsC) {
  // batched form (blockIdx.z = system; strides 0 / gridDim.z = 1 otherwise)
  A += blockIdx.z * bsA;
  B += blockIdx.z * bsB;
  Cm += blockIdx.z * bsC;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;                              // [STAGES][KC][AST]
  double* sB = smem + C::STAGES * C::A_STAGE;     // [STAGES][BN][BSTR]
  constexpr int KC = C::KC;

  // grouped rasterization: 8 tile-rows share the B columns they stream
  const int G = 8;
  int bid = blockIdx.x;
  int group = bid / (G * tilesN);
  int first_m = group * G;
  int gsz = min(tilesM - first_m, G);
  int tm = first_m + (bid % (G * tilesN)) % gsz;
  int tn = (bid % (G * tilesN)) / gsz;
  const int64_t m0 = (int64_t)tm * C::BM, n0 = (int64_t)tn * C::BN;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WM, wn = warp / C::WM;

  // ---- accumulators initialized from C (the Eq 6-c "A^(r-1)" term)
  double acc[C::MT][C::NT][2];
#pragma unroll
  for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
    for (int nt = 0; nt < C::NT; nt++)
#pragma unroll
      for (int q = 0; q < 2; q++) {
        int64_t m = m0 + wm * (C::MT * 8) + mt * 8 + g;
        int64_t n = n0 + wn * (C::NT * 8) + nt * 8 + 2 * t + q;
        acc[mt][nt][q] = (m < M && n < N) ? Cm[m + n * ldc] : 0.0;
      }

  const int nk = (int)((K + KC - 1) / KC);

  // ---- per-thread load geometry (fixed over stages)
  // A: element index e = tid*VEC + r*THREADS*VEC -> kk = e / BM, mm = e % BM
  constexpr int A_PER = (C::BM * KC) / (C::THREADS * VEC);
  constexpr int A_KSTEP = (C::THREADS * VEC) / C::BM;          // kk advance per r
  constexpr int B_PER = (C::BN * KC + C::THREADS * VEC - 1) / (C::THREADS * VEC);
  constexpr int B_NSTEP = (C::THREADS * VEC) / KC;             // nn advance per r
  static_assert((C::THREADS * VEC) % C::BM == 0 || A_PER == 0, "A geometry");
  const int a_mm = (tid * VEC) % C::BM, a_kk0 = (tid * VEC) / C::BM;
  const int b_kk = (tid * VEC) % KC, b_nn0 = (tid * VEC) / KC;
  const int64_t a_m = m0 + a_mm;
  const int64_t a_rem = M - a_m;
  const int a_valid = a_rem <= 0 ? 0 : (a_rem >= VEC ? VEC : (int)a_rem);

  auto load_stage = [&](int slot, int kt) {
    double* a = sA + slot * C::A_STAGE;
    double* b = sB + slot * C::B_STAGE;
    const int64_t k0 = (int64_t)kt * KC;
#pragma unroll
    for (int r = 0; r < A_PER; r++) {
      const int kk = a_kk0 + r * A_KSTEP;
      const int64_t kl = k0 + kk;
      const int64_t kp = reverse_k ? (K - 1 - kl) : kl;
      const bool kin = kl < K;
      if (VEC == 2) {
        const int nv = kin ? a_valid : 0;
        cp_async16(a + kk * C::AST + a_mm, nv ? (A + a_m + kp * lda) : A, nv);
      } else {
        const bool p = kin && a_valid > 0;
        cp_async8(a + kk * C::AST + a_mm, p ? (A + a_m + kp * lda) : A, p);
      }
    }
#pragma unroll
    for (int r = 0; r < B_PER; r++) {
      const int nn = b_nn0 + r * B_NSTEP;
      if (nn < C::BN) {
        const int64_t n = n0 + nn;
        const int64_t kl = k0 + b_kk;
        if (VEC == 2) {
          const int64_t rem = K - kl;
          const int nv = (n < N) ? (rem <= 0 ? 0 : (rem >= 2 ? 2 : (int)rem)) : 0;
          cp_async16(b + nn * C::BSTR + b_kk, nv ? (B + kl + n * ldb) : B, nv);
        } else {
          const int64_t kp = reverse_k ? (K - 1 - kl) : kl;
          const bool p = (kl < K) && (n < N);
          cp_async8(b + nn * C::BSTR + b_kk, p ? (B + kp + n * ldb) : B, p);
        }
      }
    }
  };

#pragma unroll
  for (int s = 0; s < C::STAGES - 1; s++) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }

  for (int kt = 0; kt < nk; kt++) {
    cp_wait<C::STAGES - 2>();
    __syncthreads();
    {
      int nxt = kt + C::STAGES - 1;
      if (nxt < nk) load_stage(nxt % C::STAGES, nxt);
      cp_commit();
    }
    const double* a = sA + (kt % C::STAGES) * C::A_STAGE + wm * (C::MT * 8) + g;
    const double* b = sB + (kt % C::STAGES) * C::B_STAGE + (wn * (C::NT * 8) + g) * C::BSTR + t;
#pragma unroll
    for (int ks = 0; ks < KC / 4; ks++) {
      double af[C::MT], bf[C::NT];
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++) af[mt] = -a[(ks * 4 + t) * C::AST + mt * 8];
#pragma unroll
      for (int nt = 0; nt < C::NT; nt++) bf[nt] = b[nt * 8 * C::BSTR + ks * 4];
#pragma unroll
      for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
        for (int nt = 0; nt < C::NT; nt++) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
  }
  cp_wait<0>();

#pragma unroll
  for (int mt = 0; mt < C::MT; mt++)
#pragma unroll
    for (int nt = 0; nt < C::NT; nt++)
#pragma unroll
      for (int q = 0; q < 2; q++) {
        int64_t m = m0 + wm * (C::MT * 8) + mt * 8 + g;
        int64_t n = n0 + wn * (C::NT * 8) + nt * 8 + 2 * t + q;
        if (m < M && n < N) Cm[m + n * ldc] = acc[mt][nt][q];
      }
}

template <class C, int VEC>
cudaError_t run_v(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double* Cm, int64_t ldc, bool rev, cudaStream_t s, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0,
                  int64_t batch = 1) {
  {
    cudaError_t e = ensure_max_dyn_smem(reinterpret_cast<const void*>(gemm_sub_kernel<C, VEC>), C::SMEM);
    if (e != cudaSuccess) return e;
  }
  int64_t tm = (M + C::BM - 1) / C::BM, tn = (N + C::BN - 1) / C::BN;
  int64_t nblk = tm * tn;
  if (nblk == 0) return cudaSuccess;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    gemm_sub_kernel<C, VEC><<<dim3((unsigned)nblk, 1, (unsigned)nb), C::THREADS, C::SMEM, s>>>(
        M, N, K, A + b0 * sA, lda, B + b0 * sB, ldb, Cm + b0 * sC, ldc, rev ? 1 : 0, (int)tm, (int)tn, sA, sB, sC);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <class C>
cudaError_t run(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                double* Cm, int64_t ldc, bool rev, cudaStream_t s, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0,
                int64_t batch = 1) {
  // 16-byte copies need 16-byte aligned column starts of A and B, which the
  // even leading dimensions and aligned bases guarantee (k stays even
  // because stages start at multiples of KC); the reversed order reads k
  // downwards and takes the 8-byte path.
  const bool v2 = !rev && ((lda & 1) == 0) && ((ldb & 1) == 0) &&
                  ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) &&
                  ((sA & 1) == 0) && ((sB & 1) == 0);
  if (v2) return run_v<C, 2>(M, N, K, A, lda, B, ldb, Cm, ldc, rev, s, sA, sB, sC, batch);
  return run_v<C, 1>(M, N, K, A, lda, B, ldb, Cm, ldc, rev, s, sA, sB, sC, batch);
}

//                 BM   BN  WM WN KC ST MINB
using Big = Cfg<128, 128, 2, 4, 16, 4, 1>;    // 8 warps, 64x32 warp tiles
using Big16 = Cfg<128, 128, 4, 4, 16, 4, 1>;  // 16 warps, 32x32 warp tiles
using Big16K32 = Cfg<128, 128, 4, 4, 32, 3, 1>;
using Mid = Cfg<128, 64, 4, 2, 16, 4, 2>;     // 8 warps, 32x32, 2 CTAs/SM
using Wide = Cfg<64, 128, 2, 4, 16, 4, 2>;
using Tall = Cfg<128, 64, 4, 2, 16, 4, 2>;
using Vec = Cfg<256, 8, 8, 1, 16, 4, 2>;

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
int cfg_override() {
  static int v = env_int("EBV_GEMM_CFG", -1);
  return v;
}
int tma_variant() {
  static int v = env_int("EBV_GEMM_TMA", 0);   // -1 disables the TMA kernel
  return v;
}

}  // namespace

cudaError_t launch_gemm_sub(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                            int64_t ldb, double* Cm, int64_t ldc, bool reverse_k, cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0) return cudaSuccess;
  if (N <= 8) return run<Vec>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
  if (!reverse_k && tma_variant() >= 0 && cfg_override() < 0 &&
      gemm_tma_eligible(M, N, K, A, lda, B, ldb)) {
    int v = tma_variant();
    // default: 128x64 tiles, 2 CTAs/SM; a 3-stage ring for the factorization's
    // K <= 1024 updates (B200: 28.8 -> 31.2 TF/s at 8064^2 x 128, equal at
    // K = 512), 4 stages for long K; 64 x 128 tiles for M <= 64
    if (v == 0) v = (M <= 64) ? 3 : (K <= 1024 ? 5 : 0);
    cudaError_t e = launch_gemm_sub_tma(M, N, K, A, lda, B, ldb, Cm, ldc, v, s);
    if (e != cudaErrorNotSupported) return e;
    (void)cudaGetLastError();
  }
  switch (cfg_override()) {
    case 0: return run<Big>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
    case 1: return run<Big16>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
    case 2: return run<Big16K32>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
    case 3: return run<Mid>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
    default: break;
  }
  if (M <= 64) return run<Wide>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
  return run<Mid>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s);
}

// Batched form (systems s = 0..batch-1 at A + s*sA, B + s*sB, C + s*sC): the
// cp.async kernels with blockIdx.z as the system — per system the same fma
// chains as launch_gemm_sub (bitwise).
cudaError_t launch_gemm_sub_batched(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int64_t sA,
                                    const double* B, int64_t ldb, int64_t sB, double* Cm, int64_t ldc, int64_t sC,
                                    int64_t batch, bool reverse_k, cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0) return cudaSuccess;
  if (N <= 8) return run<Vec>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s, sA, sB, sC, batch);
  if (M <= 64) return run<Wide>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s, sA, sB, sC, batch);
  return run<Mid>(M, N, K, A, lda, B, ldb, Cm, ldc, reverse_k, s, sA, sB, sC, batch);
}

}  // namespace ebv
