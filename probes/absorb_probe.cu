// probes/absorb_probe.cu — cycles per absorbed term of the chain solve's
// absorber inner loop (k_solve2.cu) in isolation: one warp, data resident in
// shared memory, variants of the y-value access.
#include <cstdio>
#include <cstdint>
constexpr int BR = 64, QT = 16;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double2 ldv2(const double* p) {
  double2 v; asm volatile("ld.volatile.shared::cta.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(su(p)) : "memory"); return v; }
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double S[BR * QT];
  __shared__ __align__(16) double yh[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < BR * QT; i += 32) S[i] = 1e-3 * (i % 17);
  for (int i = lane; i < 64; i += 32) yh[i] = 1.0 + i;
  __syncwarp();
  double v0 = lane, v1 = lane + 1;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const int qq = it & 3;
#pragma unroll
    for (int h8 = 0; h8 < QT; h8 += 8) {
      double y[8];
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 8; i++) y[i] = yh[qq * QT + h8 + i];
      } else {
        for (;;) {
          const double2 a = ldv2(yh + qq * QT + h8), b = ldv2(yh + qq * QT + h8 + 2), c = ldv2(yh + qq * QT + h8 + 4),
                        d = ldv2(yh + qq * QT + h8 + 6);
          y[0] = a.x; y[1] = a.y; y[2] = b.x; y[3] = b.y; y[4] = c.x; y[5] = c.y; y[6] = d.x; y[7] = d.y;
          bool ok = true;
#pragma unroll
          for (int i = 0; i < 8; i++) ok = ok && __double_as_longlong(y[i]) != 0x7FF4DEADBEEF0001LL;
          if (ok) break;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const double2 l = *reinterpret_cast<const double2*>(S + (h8 + i) * BR + 2 * lane);
        if (MODE == 2) { v0 = fma(-l.x, y[i], v0); }
        else { v0 = fma(-l.x, y[i], v0); v1 = fma(-l.y, y[i], v1); }
      }
    }
  }
  long long t1 = clock64();
  out[lane] = v0 + v1;
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  auto run = [&](auto kern, const char* name) {
    kern<<<1, 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    kern<<<1, 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %.2f cycles per term\n", name, (double)c / (iters * QT));
  };
  run(k<0>, "plain LDS y, 2 rows");
  run(k<1>, "volatile+sentinel y, 2 rows");
  run(k<2>, "plain LDS y, 1 row");
  return 0;
}
