// probes/absorb_tma_probe.cu — the chain solve's absorber quarter loop
// (k_solve2.cu absorb(): 2-D TMA quarter tiles into 4 smem slots, mbarrier
// waits, consume 16 terms, proxy fence, re-issue) in isolation: one warp,
// one CTA, a 64 x 8192 slab; clock64 per quarter.
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1907_05767_b200/csrc/ebv_internal.cuh"
constexpr int BR = 64, QT = 16, NSLOT = 4;
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(unsigned long long* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(unsigned long long* b, uint32_t par) {
  uint32_t d; do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(d) : "r"(su(b)), "r"(par) : "memory"); } while (!d); }
__device__ __forceinline__ void tma(void* dst, const CUtensorMap* m, int r, int c, unsigned long long* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su(dst)), "l"((uint64_t)m), "r"(r), "r"(c), "r"(su(b)) : "memory"); }
__global__ void k(const __grid_constant__ CUtensorMap map, int nq, double* out, long long* cyc, int mode) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* slot = reinterpret_cast<double*>(raw);
  __shared__ unsigned long long bar[NSLOT];
  __shared__ __align__(16) double yh[64];
  const int lane = threadIdx.x;
  if (lane < NSLOT) mbar_init(&bar[lane], 1);
  yh[lane] = 1.0 + lane; yh[lane + 32] = 2.0 + lane;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (lane == 0) for (int q = 0; q < NSLOT; q++) { expect_tx(&bar[q], BR * QT * 8); tma(slot + q * BR * QT, &map, 0, q * QT, &bar[q]); }
  double v0 = lane, v1 = lane + 0.5;
  long long t0 = clock64(), tw = 0, tc = 0;
  for (int q = 0; q < nq; q++) {
    const int k = q % NSLOT;
    long long a = clock64();
    mwait(&bar[k], (q / NSLOT) & 1);
    long long b = clock64();
    const double* S = slot + k * BR * QT;
    if (mode == 4) {   // DFMA chain only (operands in registers)
#pragma unroll
      for (int i = 0; i < QT; i++) { v0 = fma(-v1, 1.0000001, v0); v1 = fma(-v0, 0.9999999, v1); }
    } else if (mode == 5) {   // two independent chains, no smem
      double a0 = v0, a1 = v1;
#pragma unroll
      for (int i = 0; i < QT; i++) { a0 = fma(a0, 1.0000001, 1e-9); a1 = fma(a1, 0.9999999, 1e-9); }
      v0 = a0; v1 = a1;
    } else if (mode == 6) {   // loads only
      double acc = 0;
#pragma unroll
      for (int i = 0; i < QT; i++) { const double2 l = *reinterpret_cast<const double2*>(S + i * BR + 2 * lane); acc += l.x; }
      v0 += acc;
    } else if (mode & 2) {
      double2 L[QT];
      double Y[QT];
#pragma unroll
      for (int i = 0; i < QT; i++) L[i] = *reinterpret_cast<const double2*>(S + i * BR + 2 * lane);
#pragma unroll
      for (int i = 0; i < QT; i += 2) {
        const double2 y2 = *reinterpret_cast<const double2*>(yh + (q & 3) * QT + i);
        Y[i] = y2.x; Y[i + 1] = y2.y;
      }
#pragma unroll
      for (int i = 0; i < QT; i++) { v0 = fma(-L[i].x, Y[i], v0); v1 = fma(-L[i].y, Y[i], v1); }
    } else {
#pragma unroll
    for (int i = 0; i < QT; i++) {
      const double2 l = *reinterpret_cast<const double2*>(S + i * BR + 2 * lane);
      const double y = yh[(q & 3) * QT + i];
      v0 = fma(-l.x, y, v0); v1 = fma(-l.y, y, v1);
    }
    }
    long long c = clock64();
    tw += b - a; tc += c - b;
    __syncwarp();
    if (mode & 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0 && q + NSLOT < nq) { expect_tx(&bar[k], BR * QT * 8); tma(slot + k * BR * QT, &map, 0, ((q + NSLOT) * QT) % 8192, &bar[k]); }
  }
  long long t1 = clock64();
  out[lane] = v0 + v1;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = tw; cyc[2] = tc; }
}
// software-pipelined: the next quarter's L values are loaded (after its
// mbarrier wait) while the current quarter's 16 terms are applied
__global__ void k2(const __grid_constant__ CUtensorMap map, int nq, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* slot = reinterpret_cast<double*>(raw);
  __shared__ unsigned long long bar[NSLOT];
  __shared__ __align__(16) double yh[64];
  const int lane = threadIdx.x;
  if (lane < NSLOT) mbar_init(&bar[lane], 1);
  yh[lane] = 1.0 + lane; yh[lane + 32] = 2.0 + lane;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (lane == 0) for (int q = 0; q < NSLOT; q++) { expect_tx(&bar[q], BR * QT * 8); tma(slot + q * BR * QT, &map, 0, q * QT, &bar[q]); }
  double v0 = lane, v1 = lane + 0.5;
  double2 La[QT], Lb[QT];
  long long t0 = clock64();
  mwait(&bar[0], 0);
#pragma unroll
  for (int i = 0; i < QT; i++) La[i] = *reinterpret_cast<const double2*>(slot + i * BR + 2 * lane);
  for (int q = 0; q < nq; q += 2) {
    // quarter q in La; fetch q+1 into Lb
    {
      const int k1 = (q + 1) % NSLOT;
      mwait(&bar[k1], ((q + 1) / NSLOT) & 1);
#pragma unroll
      for (int i = 0; i < QT; i++) Lb[i] = *reinterpret_cast<const double2*>(slot + k1 * BR * QT + i * BR + 2 * lane);
#pragma unroll
      for (int i = 0; i < QT; i++) { const double y = yh[(q & 3) * QT + i]; v0 = fma(-La[i].x, y, v0); v1 = fma(-La[i].y, y, v1); }
      __syncwarp();
      const int k0 = q % NSLOT;
      if (lane == 0 && q + NSLOT < nq) { expect_tx(&bar[k0], BR * QT * 8); tma(slot + k0 * BR * QT, &map, 0, ((q + NSLOT) * QT) % 8192, &bar[k0]); }
    }
    {
      const int k2n = (q + 2) % NSLOT;
      if (q + 2 < nq) {
        mwait(&bar[k2n], ((q + 2) / NSLOT) & 1);
#pragma unroll
        for (int i = 0; i < QT; i++) La[i] = *reinterpret_cast<const double2*>(slot + k2n * BR * QT + i * BR + 2 * lane);
      }
#pragma unroll
      for (int i = 0; i < QT; i++) { const double y = yh[((q + 1) & 3) * QT + i]; v0 = fma(-Lb[i].x, y, v0); v1 = fma(-Lb[i].y, y, v1); }
      __syncwarp();
      const int k1 = (q + 1) % NSLOT;
      if (lane == 0 && q + 1 + NSLOT < nq) { expect_tx(&bar[k1], BR * QT * 8); tma(slot + k1 * BR * QT, &map, 0, ((q + 1 + NSLOT) * QT) % 8192, &bar[k1]); }
    }
  }
  long long t1 = clock64();
  out[lane] = v0 + v1;
  if (lane == 0) { cyc[0] = t1 - t0; }
}

__device__ __forceinline__ void pf_tensor(const CUtensorMap* m, int r, int c) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((uint64_t)m), "r"(r), "r"(c) : "memory");
}
// streaming: quarter q at column q*QT of a wide slab (never reused: HBM
// latency), optional tensor prefetch to L2 `pf` quarters ahead
__global__ void k3(const __grid_constant__ CUtensorMap map, int nq, int pf, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* slot = reinterpret_cast<double*>(raw);
  __shared__ unsigned long long bar[NSLOT];
  __shared__ __align__(16) double yh[64];
  const int lane = threadIdx.x;
  if (lane < NSLOT) mbar_init(&bar[lane], 1);
  yh[lane] = 1.0 + lane; yh[lane + 32] = 2.0 + lane;
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    if (pf) for (int q = 0; q < pf && q < nq; q++) pf_tensor(&map, 0, q * QT);
    for (int q = 0; q < NSLOT; q++) { expect_tx(&bar[q], BR * QT * 8); tma(slot + q * BR * QT, &map, 0, q * QT, &bar[q]); }
  }
  double v0 = lane, v1 = lane + 0.5;
  long long t0 = clock64();
  for (int q = 0; q < nq; q++) {
    const int k = q % NSLOT;
    mwait(&bar[k], (q / NSLOT) & 1);
    const double* S = slot + k * BR * QT;
#pragma unroll
    for (int i = 0; i < QT; i++) {
      const double2 l = *reinterpret_cast<const double2*>(S + i * BR + 2 * lane);
      const double y = yh[(q & 3) * QT + i];
      v0 = fma(-l.x, y, v0); v1 = fma(-l.y, y, v1);
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) {
      if (pf && q + pf < nq) pf_tensor(&map, 0, (q + pf) * QT);
      if (q + NSLOT < nq) { expect_tx(&bar[k], BR * QT * 8); tma(slot + k * BR * QT, &map, 0, (q + NSLOT) * QT, &bar[k]); }
    }
  }
  long long t1 = clock64();
  out[lane] = v0 + v1;
  if (lane == 0) cyc[0] = t1 - t0;
}

int main() {
  const int64_t n = 8192;
  double* A; cudaMalloc(&A, 64 * n * 8 * 2);
  cudaMemset(A, 0, 64 * n * 8 * 2);
  alignas(64) CUtensorMap map;
  ebv::make_tma_map_2d(&map, A, 128, n, 128, BR, QT);
  double* out; long long* cyc; cudaMalloc(&out, 256); cudaMalloc(&cyc, 24);
  const int smem = NSLOT * BR * QT * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 7; mode++)
    for (int rep = 0; rep < 3; rep++) {
      const int nq = 512;
      k<<<1, 32, smem>>>(map, nq, out, cyc, mode);
      cudaError_t e = cudaDeviceSynchronize();
      long long c[3]; cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost);
      printf("fence=%d rep %d: %s  %.0f cycles/quarter (wait %.0f, consume %.0f)\n", mode, rep, cudaGetErrorString(e),
             (double)c[0] / nq, (double)c[1] / nq, (double)c[2] / nq);
    }
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; rep++) {
    const int nq = 512;
    k2<<<1, 32, smem>>>(map, nq, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c[1]; cudaMemcpy(c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("pipelined rep %d: %s  %.0f cycles/quarter\n", rep, cudaGetErrorString(e), (double)c[0] / nq);
  }
  {
    const int64_t ncol = 1 << 20;          // 64 x 1M doubles = 512 MB, streamed
    double* Bg; cudaMalloc(&Bg, 64 * ncol * 8);
    cudaMemset(Bg, 0, 64 * ncol * 8);
    alignas(64) CUtensorMap mb;
    ebv::make_tma_map_2d(&mb, Bg, 64, ncol, 64, BR, QT);
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int pf : {0, 8, 16, 32, 64}) {
      const int nq = 4096;
      k3<<<1, 32, smem>>>(mb, nq, pf, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      long long c[1]; cudaMemcpy(c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("streaming from HBM, prefetch %2d quarters ahead: %s  %.0f cycles/quarter\n", pf, cudaGetErrorString(e), (double)c[0] / nq);
    }
  }
  return 0;
}
