// Probe M2/M3: FP64 tensor-core (DMMA) fragment layout,
// rounding semantics and throughput versus plain DFMA on sm_100a.
// Standalone executable; not part of the product library.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <quadmath.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------------------------------------------------------- m8n8k4
// A 8x4 row-major, B 4x8 (stored as B[k][n]), C 8x8 row-major.
__global__ void mma_m8n8k4(const double* A, const double* B, const double* C, double* D, int ntiles) {
  int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  int tile = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (tile >= ntiles) return;
  const double* a = A + tile * 32; const double* b = B + tile * 32;
  const double* c = C + tile * 64; double* d = D + tile * 64;
  double a0 = a[g * 4 + t];
  double b0 = b[t * 8 + g];
  double c0 = c[g * 8 + 2 * t], c1 = c[g * 8 + 2 * t + 1];
  double d0, d1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a0), "d"(b0), "d"(c0), "d"(c1));
  d[g * 8 + 2 * t] = d0; d[g * 8 + 2 * t + 1] = d1;
}

// ---------------------------------------------------------------- m16n8k16
// A 16x16 row-major, B 16x8 stored B[k][n], C 16x8 row-major.
__global__ void mma_m16n8k16(const double* A, const double* B, const double* C, double* D, int ntiles) {
  int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  int tile = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (tile >= ntiles) return;
  const double* a = A + tile * 256; const double* b = B + tile * 128;
  const double* c = C + tile * 128; double* d = D + tile * 128;
  double af[8], bf[4], cf[4], df[4];
  for (int i = 0; i < 8; i++) af[i] = a[(g + 8 * (i % 2)) * 16 + t + 4 * (i / 2)];
  for (int i = 0; i < 4; i++) bf[i] = b[(t + 4 * i) * 8 + g];
  for (int i = 0; i < 4; i++) cf[i] = c[(g + 8 * (i / 2)) * 8 + 2 * t + (i % 2)];
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
               "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%16,%17,%18,%19};\n"
               : "=d"(df[0]), "=d"(df[1]), "=d"(df[2]), "=d"(df[3])
               : "d"(af[0]), "d"(af[1]), "d"(af[2]), "d"(af[3]), "d"(af[4]), "d"(af[5]), "d"(af[6]), "d"(af[7]),
                 "d"(bf[0]), "d"(bf[1]), "d"(bf[2]), "d"(bf[3]),
                 "d"(cf[0]), "d"(cf[1]), "d"(cf[2]), "d"(cf[3]));
  for (int i = 0; i < 4; i++) d[(g + 8 * (i / 2)) * 8 + 2 * t + (i % 2)] = df[i];
}

// ---------------------------------------------------------------- throughput
template <int NACC>
__global__ void thr_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[NACC][2];
  for (int i = 0; i < NACC; i++) { acc[i][0] = i; acc[i][1] = -i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}
template <int NACC>
__global__ void thr_dmma16(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
  for (int i = 0; i < 4; i++) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double acc[NACC][4];
  for (int i = 0; i < NACC; i++) for (int j = 0; j < 4; j++) acc[i][j] = i + j;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
                   "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < NACC; i++) for (int j = 0; j < 4; j++) s += acc[i][j];
  if (s == 12345.678) out[0] = s;
}
template <int NACC>
__global__ void thr_dfma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double acc[NACC];
  for (int i = 0; i < NACC; i++) acc[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = __fma_rn(a, b, acc[i]);
  }
  double s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

static double rnd(std::mt19937_64& r, int spread) {
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::uniform_int_distribution<int> e(-spread, spread);
  return std::ldexp(u(r), e(r));
}
static double round_q(__float128 x) { return (double)x; }

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  std::mt19937_64 rng(1234);
  // ----- layout + rounding, m8n8k4
  for (int spread : {0, 4, 20}) {
    const int T = 20000;
    std::vector<double> A(T * 32), B(T * 32), C(T * 64), D(T * 64);
    bool exact_ints = (spread == 0);
    for (auto& v : A) v = exact_ints ? (double)(int)(rng() % 17) - 8 : rnd(rng, spread);
    for (auto& v : B) v = exact_ints ? (double)(int)(rng() % 17) - 8 : rnd(rng, spread);
    for (auto& v : C) v = exact_ints ? (double)(int)(rng() % 17) - 8 : rnd(rng, spread);
    double *dA, *dB, *dC, *dD;
    CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8));
    CK(cudaMalloc(&dC, C.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
    mma_m8n8k4<<<(T + 3) / 4, 128>>>(dA, dB, dC, dD, T);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
    long eq_seq = 0, eq_single = 0, eq_rev = 0, total = 0, neither = 0;
    for (int tt = 0; tt < T; tt++)
      for (int r = 0; r < 8; r++)
        for (int c = 0; c < 8; c++) {
          const double* a = &A[tt * 32 + r * 4]; double cc = C[tt * 64 + r * 8 + c];
          double bk[4]; for (int k = 0; k < 4; k++) bk[k] = B[tt * 32 + k * 8 + c];
          double s = cc; for (int k = 0; k < 4; k++) s = std::fma(a[k], bk[k], s);
          double sr = cc; for (int k = 3; k >= 0; k--) sr = std::fma(a[k], bk[k], sr);
          __float128 q = cc; for (int k = 0; k < 4; k++) q += (__float128)a[k] * bk[k];
          double sq = round_q(q);
          double d = D[tt * 64 + r * 8 + c];
          total++; eq_seq += (d == s); eq_single += (d == sq); eq_rev += (d == sr);
          neither += (d != s && d != sq);
        }
    printf("{\"probe\": \"M3_m8n8k4\", \"spread\": %d, \"total\": %ld, \"eq_seq_fma\": %ld, \"eq_rev_fma\": %ld, \"eq_single_round\": %ld, \"neither\": %ld}\n",
           spread, total, eq_seq, eq_rev, eq_single, neither);
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dD);
  }
  // ----- layout + rounding, m16n8k16
  for (int spread : {0, 4, 20}) {
    const int T = 10000;
    std::vector<double> A(T * 256), B(T * 128), C(T * 128), D(T * 128);
    bool exact_ints = (spread == 0);
    for (auto& v : A) v = exact_ints ? (double)(int)(rng() % 17) - 8 : rnd(rng, spread);
    for (auto& v : B) v = exact_ints ? (double)(int)(rng() % 17) - 8 : rnd(rng, spread);
    for (auto& v : C) v = exact_ints ? (double)(int)(rng() % 17) - 8 : rnd(rng, spread);
    double *dA, *dB, *dC, *dD;
    CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8));
    CK(cudaMalloc(&dC, C.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
    mma_m16n8k16<<<(T + 3) / 4, 128>>>(dA, dB, dC, dD, T);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
    long eq_seq = 0, eq_single = 0, eq_chunk4 = 0, total = 0, neither = 0;
    for (int tt = 0; tt < T; tt++)
      for (int r = 0; r < 16; r++)
        for (int c = 0; c < 8; c++) {
          const double* a = &A[tt * 256 + r * 16]; double cc = C[tt * 128 + r * 8 + c];
          double bk[16]; for (int k = 0; k < 16; k++) bk[k] = B[tt * 128 + k * 8 + c];
          double s = cc; for (int k = 0; k < 16; k++) s = std::fma(a[k], bk[k], s);
          __float128 q = cc; for (int k = 0; k < 16; k++) q += (__float128)a[k] * bk[k];
          double sq = round_q(q);
          double s4 = cc;
          for (int kk = 0; kk < 16; kk += 4) {
            __float128 qq = s4; for (int k = kk; k < kk + 4; k++) qq += (__float128)a[k] * bk[k];
            s4 = round_q(qq);
          }
          double d = D[tt * 128 + r * 8 + c];
          total++; eq_seq += (d == s); eq_single += (d == sq); eq_chunk4 += (d == s4);
          neither += (d != s && d != sq && d != s4);
        }
    printf("{\"probe\": \"M3_m16n8k16\", \"spread\": %d, \"total\": %ld, \"eq_seq_fma\": %ld, \"eq_single_round\": %ld, \"eq_chunk4_single\": %ld, \"neither\": %ld}\n",
           spread, total, eq_seq, eq_single, eq_chunk4, neither);
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dD);
  }
  // ----- throughput
  double* dout; CK(cudaMalloc(&dout, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int grid = p.multiProcessorCount * bps;
      thr_dmma<8><<<grid, wpb * 32>>>(dout, 16); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); thr_dmma<8><<<grid, wpb * 32>>>(dout, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)grid * wpb * iters * 8 * 256;
      printf("{\"probe\": \"M2_dmma_m8n8k4\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n",
             wpb, bps, ms, 2 * fmas / ms / 1e9);
      thr_dmma16<4><<<grid, wpb * 32>>>(dout, 16); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); thr_dmma16<4><<<grid, wpb * 32>>>(dout, iters / 4); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fmas = (double)grid * wpb * (iters / 4) * 4 * 2048;
      printf("{\"probe\": \"M2_dmma_m16n8k16\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n",
             wpb, bps, ms, 2 * fmas / ms / 1e9);
      thr_dfma<16><<<grid, wpb * 32>>>(dout, 16); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); thr_dfma<16><<<grid, wpb * 32>>>(dout, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      fmas = (double)grid * wpb * 32 * iters * 16;
      printf("{\"probe\": \"M2_dfma\", \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n",
             wpb, bps, ms, 2 * fmas / ms / 1e9);
    }
  }
  return 0;
}
