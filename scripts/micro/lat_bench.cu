#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = x;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) y = y + b;
  long long t2 = clock64();
  double z = y;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) z = z * a;
  long long t3 = clock64();
  float f = z;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) f = fmaf(f, (float)a, (float)b);
  long long t4 = clock64();
  double s = f;
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) s = __shfl_sync(~0u, s, (threadIdx.x + 1) & 31) + 0.0;
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 1024; cyc[1] = (t2 - t1) / 1024; cyc[2] = (t3 - t2) / 1024;
    cyc[3] = (t4 - t3) / 1024; cyc[4] = (t5 - t4) / 1024; out[0] = s; }
}
// DFMA throughput: independent chains, 1 warp
__global__ void thr(double* out, long long* cyc, double a, double b, int warps) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[8 + warps] = (t1 - t0);
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 8 * 4096); cudaMalloc(&c, 8 * 64);
  lat<<<1, 32>>>(d, c, 0.999, 1e-3);
  thr<<<1, 32>>>(d, c, 0.999, 1e-3, 1);
  thr<<<1, 128>>>(d, c, 0.999, 1e-3, 4);
  thr<<<1, 512>>>(d, c, 0.999, 1e-3, 16);
  long long h[64]; cudaDeviceSynchronize(); cudaMemcpy(h, c, 8 * 64, cudaMemcpyDeviceToHost);
  printf("latency cycles: DFMA %lld DADD %lld DMUL %lld FFMA %lld SHFL(+DADD) %lld\n", h[0], h[1], h[2], h[3], h[4]);
  printf("DFMA throughput: 1 warp: %.2f cyc/instr; 4 warps: %.2f; 16 warps: %.2f (per warp-instr, SM-wide)\n",
         h[9] / 8192.0, h[12] / (8192.0 * 4), h[24] / (8192.0 * 16));
}
