// Cost of one barrier-separated dependent stage inside a CTA: thread 0 (or
// one 6-lane group) reads what another warp wrote before the barrier,
// computes, writes, barrier -- the building block of the cyclic-reduction
// levels.  Cycles per stage for 2..16 warps.
#include <cstdio>
#include <cuda_runtime.h>
template <int NW, int MODE>
__global__ void __launch_bounds__(32 * NW, 1) stages(double* out, long long* cyc, int n) {
  __shared__ double buf[64 * 8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) buf[i] = 1.0 + i * 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
    const int src = (k & 1) ? NW - 1 : 0;  // alternate the producing warp
    if (MODE == 0) {
      if (w == src && l == 0) buf[8 * (k & 7)] = buf[8 * ((k + 7) & 7)] * 1.0000001 + 1e-9;
    } else {
      // a 6-lane group: 6 loads of the previous vector, 6-term dot, one store per lane
      if (w == src && l < 6) {
        const double* p = buf + 8 * ((k + 7) & 7);
        double a = p[0] * 0.5 + p[1] * 0.25 + p[2] * 0.125 + p[3] * 0.0625 + p[4] * 0.03125 + p[5] * 0.015625;
        buf[8 * (k & 7) + l] = a + l * 1e-9;
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n;
    out[0] = buf[0];
  }
}
template <int NW, int MODE>
void run() {
  double* o;
  long long* c;
  cudaMalloc(&o, 64);
  cudaMalloc(&c, 64);
  stages<NW, MODE><<<1, 32 * NW>>>(o, c, 2000);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("warps %2d %s: %lld cycles per stage\n", NW, MODE ? "6-lane dot" : "scalar   ", h);
}
int main() {
  run<2, 0>(); run<4, 0>(); run<8, 0>(); run<16, 0>();
  run<2, 1>(); run<4, 1>(); run<8, 1>(); run<16, 1>();
}
