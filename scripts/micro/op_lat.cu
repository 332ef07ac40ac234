// Latency probes (development): dependent DFMA chain, dependent shared-memory
// load chain, and __syncthreads round trips, in SM clock cycles.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, int n, double a, double b) {
  __shared__ double sm[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 3) & 1023; }
  __syncthreads();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  int j = threadIdx.x;
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t3 = clock64();
  double y = 0.0;
  for (int i = 0; i < n; ++i) y = sm[(int)y & 1023] * 0.0 + y;   // dependent LDS.64 -> DFMA
  long long t4 = clock64();
  double z = 1.0;
  for (int i = 0; i < n; ++i) z = z / (1.0 + z);
  long long t5 = clock64();
  double w = 1.0;
  for (int i = 0; i < n; ++i) w = __drcp_rn(1.0 + w);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[5] = (t6 - t5) / n;
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n; cyc[4] = (t5 - t4) / n;
  }
  out[threadIdx.x] = x + j + y + z + w;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  for (int nt : {32, 256}) {
    probe<<<1, nt>>>(o, c, 4096, 1.0000001, 0.9999999);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA dep %lld cyc, LDS.32 dep %lld, syncthreads %lld, LDS.64->DFMA dep %lld, DDIV dep %lld, DRCP_RN dep %lld\n", nt,
           h[0], h[1], h[2], h[3], h[4], h[5]);
  }
}
