// Probe: dependent-chain latencies on sm_100a (one warp, clock64):
// DFMA, DMUL, correctly rounded fp64 division, MUFU.RCP64H-based reciprocal,
// 64-bit shuffle, shared-memory round trip.
#include <cstdio>
#include <cstdint>
__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sm[64];
  double x = a + threadIdx.x * 1e-9, y = b;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = fma(x, y, 1e-300);
  t1 = clock64(); cyc[0] = t1 - t0;
  // division chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = x / y;
  t1 = clock64(); cyc[1] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = x * y;
  t1 = clock64(); cyc[2] = t1 - t0;
  // shuffle chain (64-bit)
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[3] = t1 - t0;
  // shared round trip chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1e-300; __syncwarp(); }
  t1 = clock64(); cyc[4] = t1 - t0;
  // division + dependent fma (the leaf's per-step arithmetic)
  t0 = clock64();
  for (int i = 0; i < iters; i++) { double l = x / y; x = fma(-l, y, x + 1.0); }
  t1 = clock64(); cyc[5] = t1 - t0;
  out[threadIdx.x] = x;
}
int main() {
  double* d; long long* c;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&c, 8 * 8);
  const int iters = 4096;
  for (int r = 0; r < 3; r++) lat<<<1, 32>>>(d, c, 1.0000001, 1.0000003, iters);
  cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"dfma", "ddiv", "dmul", "shfl64", "smem_roundtrip+syncwarp", "ddiv+dfma"};
  for (int i = 0; i < 6; i++) printf("{\"probe\": \"latency_%s\", \"cycles_per_op\": %.1f}\n", names[i], (double)h[i] / iters);
  return 0;
}
