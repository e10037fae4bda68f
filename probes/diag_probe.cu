// probes/diag_probe.cu — cycles per pair of steps of the chain solve's
// diagonal-block loop (k_solve2.cu solve_diag) in isolation: one warp, tile
// in shared memory, forward (unit L) and backward (Markstein quotient).
#include <cstdio>
#include <cstdint>
constexpr int BR = 64;
__device__ __forceinline__ double quot_mk(double y, double u, double r) { const double q0 = y * r; return fma(r, fma(-u, q0, y), q0); }
template <int MODE>
__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double D[BR * BR];
  __shared__ __align__(16) double yh[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < BR * BR; i += 32) D[i] = (i % 65 == 0) ? 2.0 : 1e-3 * (i % 13);
  __syncwarp();
  double v0 = 1.0 + lane, v1 = 2.0 + lane;
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    if (MODE <= 1) {
#pragma unroll 4
      for (int p = 0; p < 32; p++) {
        const double2 c0 = *reinterpret_cast<const double2*>(D + (2 * p) * BR + 2 * lane);
        const double2 c1 = *reinterpret_cast<const double2*>(D + (2 * p + 1) * BR + 2 * lane);
        const double t1 = fma(-c0.y, v0, v1);
        const double y0 = __shfl_sync(0xffffffffu, v0, p);
        const double y1 = __shfl_sync(0xffffffffu, t1, p);
        if (MODE == 0 && lane == p) *reinterpret_cast<double2*>(yh + 2 * p) = make_double2(v0, t1);
        const double n0 = fma(-c1.x, y1, fma(-c0.x, y0, v0));
        const double n1 = fma(-c1.y, y1, fma(-c0.y, y0, v1));
        v0 = lane > p ? n0 : v0;
        v1 = lane > p ? n1 : (lane == p ? t1 : v1);
      }
    } else {
      const double d0 = D[(2 * lane) * BR + 2 * lane], d1 = D[(2 * lane + 1) * BR + 2 * lane + 1];
      const double rc0 = 1.0 / d0, rc1 = 1.0 / d1;
#pragma unroll 4
      for (int p = 31; p >= 0; p--) {
        const double2 c1 = *reinterpret_cast<const double2*>(D + (2 * p + 1) * BR + 2 * lane);
        const double2 c0 = *reinterpret_cast<const double2*>(D + (2 * p) * BR + 2 * lane);
        const double q1 = quot_mk(v1, d1, rc1);
        const double t0 = fma(-c1.x, q1, v0);
        const double q0 = quot_mk(t0, d0, rc0);
        const double x1 = __shfl_sync(0xffffffffu, q1, p);
        const double x0 = __shfl_sync(0xffffffffu, q0, p);
        if (lane == p) *reinterpret_cast<double2*>(yh + 2 * p) = make_double2(q1, q0);
        const double n0 = fma(-c0.x, x0, fma(-c1.x, x1, v0));
        const double n1 = fma(-c0.y, x0, fma(-c1.y, x1, v1));
        v0 = lane < p ? n0 : (lane == p ? q0 : v0);
        v1 = lane < p ? n1 : (lane == p ? q1 : v1);
      }
    }
  }
  long long t1 = clock64();
  out[lane] = v0 + v1;
  if (lane == 0) *cyc = t1 - t0;
}
// four rows per lane (k_solve2.cu solve_diag4), forward
__global__ void kq(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double Dm[BR * BR];
  __shared__ __align__(16) double yh[64];
  const int lane = threadIdx.x;
  for (int i = lane; i < BR * BR; i += 32) Dm[i] = (i % 65 == 0) ? 2.0 : 1e-3 * (i % 13);
  __syncwarp();
  double r0 = 1.0 + lane, r1 = 2.0 + lane, r2 = 3.0 + lane, r3 = 4.0 + lane;
  const double* D = Dm + 4 * (lane & 15);
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
#pragma unroll 2
    for (int p = 0; p < 16; p++) {
      const double2 c0a = *reinterpret_cast<const double2*>(D + (4 * p) * BR), c0b = *reinterpret_cast<const double2*>(D + (4 * p) * BR + 2);
      const double2 c1a = *reinterpret_cast<const double2*>(D + (4 * p + 1) * BR), c1b = *reinterpret_cast<const double2*>(D + (4 * p + 1) * BR + 2);
      const double2 c2a = *reinterpret_cast<const double2*>(D + (4 * p + 2) * BR), c2b = *reinterpret_cast<const double2*>(D + (4 * p + 2) * BR + 2);
      const double2 c3a = *reinterpret_cast<const double2*>(D + (4 * p + 3) * BR), c3b = *reinterpret_cast<const double2*>(D + (4 * p + 3) * BR + 2);
      const double t1 = fma(-c0a.y, r0, r1);
      const double t2 = fma(-c1b.x, t1, fma(-c0b.x, r0, r2));
      const double t3 = fma(-c2b.y, t2, fma(-c1b.y, t1, fma(-c0b.y, r0, r3)));
      const double y0 = __shfl_sync(0xffffffffu, r0, p);
      const double y1 = __shfl_sync(0xffffffffu, t1, p);
      const double y2 = __shfl_sync(0xffffffffu, t2, p);
      const double y3 = __shfl_sync(0xffffffffu, t3, p);
      if (lane == p) { *reinterpret_cast<double2*>(yh + 4 * p) = make_double2(r0, t1); *reinterpret_cast<double2*>(yh + 4 * p + 2) = make_double2(t2, t3); }
      const double n0 = fma(-c3a.x, y3, fma(-c2a.x, y2, fma(-c1a.x, y1, fma(-c0a.x, y0, r0))));
      const double n1 = fma(-c3a.y, y3, fma(-c2a.y, y2, fma(-c1a.y, y1, fma(-c0a.y, y0, r1))));
      const double n2 = fma(-c3b.x, y3, fma(-c2b.x, y2, fma(-c1b.x, y1, fma(-c0b.x, y0, r2))));
      const double n3 = fma(-c3b.y, y3, fma(-c2b.y, y2, fma(-c1b.y, y1, fma(-c0b.y, y0, r3))));
      const bool below = lane > p, own = lane == p;
      r0 = below ? n0 : r0;
      r1 = below ? n1 : (own ? t1 : r1);
      r2 = below ? n2 : (own ? t2 : r2);
      r3 = below ? n3 : (own ? t3 : r3);
    }
  }
  long long t1c = clock64();
  out[lane] = r0 + r1 + r2 + r3 + yh[lane];
  if (lane == 0) *cyc = t1c - t0;
}

int main() {
  double* out; long long* cyc; cudaMalloc(&out, 256); cudaMalloc(&cyc, 8);
  const int reps = 2000;
  auto run = [&](auto kern, const char* name) {
    kern<<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize();
    kern<<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %.1f cycles per pair\n", name, (double)c / (reps * 32));
  };
  run(k<0>, "forward with history stores");
  run(k<1>, "forward no stores");
  run(k<2>, "backward (Markstein) with stores");
  kq<<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize();
  kq<<<1, 32>>>(out, cyc, reps); cudaDeviceSynchronize();
  { long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("%-34s %.1f cycles per pair\n", "forward, 4 rows per lane", (double)c / (reps * 32)); }
  return 0;
}
