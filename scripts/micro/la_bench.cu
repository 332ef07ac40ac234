// Chain-step latency variants (one 6-lane group, forward sweep of NS steps, smem operands)
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
constexpr int NS = 50;
constexpr int REPS = 200;
__device__ __forceinline__ double shf(double v, int s) { return __shfl_sync(~0u, v, s); }

// A: one step per block (current production pattern)
__global__ void varA(const double* gM, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm; double* b = M + 36 * NS; double* v = b + 6 * NS;
  int lane = threadIdx.x; int r = lane % 6;
  for (int i = lane; i < 36 * NS; i += 32) M[i] = gM[i] * 1e-3;
  for (int i = lane; i < 6 * NS; i += 32) b[i] = 1.0;
  __syncwarp();
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    double prev = b[r];
    const double* Mp = M + 6 * r; const double* bp = b + r; double* vp = v + r;
    for (int t = 1; t < NS; ++t) {
      bp += 6; vp += 6;
      double a0 = *bp; double m0 = Mp[0], m1 = Mp[1], m2 = Mp[2], m3 = Mp[3], m4 = Mp[4], m5 = Mp[5]; Mp += 36;
      double p0 = shf(prev, 0), p1 = shf(prev, 1), p2 = shf(prev, 2), p3 = shf(prev, 3), p4 = shf(prev, 4), p5 = shf(prev, 5);
      double a = a0 - ((m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5));
      prev = a; if (lane < 6) *vp = a;
    }
    acc += prev;
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[0] = (t1 - t0) / REPS; out[0] = acc; }
}
// B: two blocks per dependent step (lookahead): lanes 0-5 compute v_i, lanes 6-11 v_{i+1}
// v_i = b_i - X_i v_{i-1};  v_{i+1} = c_{i+1} + Q_{i+1} v_{i-1}
__global__ void varB(const double* gM, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm; double* Q = M + 36 * NS; double* b = Q + 36 * NS; double* v = b + 6 * NS;
  int lane = threadIdx.x; int r = lane % 6; int grp = lane < 6 ? 0 : 1;
  for (int i = lane; i < 36 * NS; i += 32) { M[i] = gM[i] * 1e-3; Q[i] = gM[i] * 1e-4; }
  for (int i = lane; i < 6 * NS; i += 32) b[i] = 1.0;
  __syncwarp();
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    double prev = b[r];  // v_0 held by lanes 6-11 (the "second" group) as well
    const double* Mp = (grp == 0 ? M : Q) + 6 * r; const double* bp = b + r + 6 * grp; double* vp = v + r + 6 * grp;
    for (int t = 1; t < NS; t += 2) {
      double a0 = *bp; bp += 12;
      double m0 = Mp[0], m1 = Mp[1], m2 = Mp[2], m3 = Mp[3], m4 = Mp[4], m5 = Mp[5]; Mp += 72;
      double p0 = shf(prev, 6), p1 = shf(prev, 7), p2 = shf(prev, 8), p3 = shf(prev, 9), p4 = shf(prev, 10), p5 = shf(prev, 11);
      double s = (m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5);
      double a = grp == 0 ? a0 - s : a0 + s;
      prev = a; if (lane < 12) *vp = a; vp += 12;
    }
    acc += prev;
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[1] = (t1 - t0) / REPS; out[1] = acc; }
}
// C: variant A but products as 6 independent multiplies + 3-level tree
__global__ void varC(const double* gM, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm; double* b = M + 36 * NS; double* v = b + 6 * NS;
  int lane = threadIdx.x; int r = lane % 6;
  for (int i = lane; i < 36 * NS; i += 32) M[i] = gM[i] * 1e-3;
  for (int i = lane; i < 6 * NS; i += 32) b[i] = 1.0;
  __syncwarp();
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    double prev = b[r];
    const double* Mp = M + 6 * r; const double* bp = b + r; double* vp = v + r;
    for (int t = 1; t < NS; ++t) {
      bp += 6; vp += 6;
      double a0 = *bp; double m0 = Mp[0], m1 = Mp[1], m2 = Mp[2], m3 = Mp[3], m4 = Mp[4], m5 = Mp[5]; Mp += 36;
      double p0 = shf(prev, 0), p1 = shf(prev, 1), p2 = shf(prev, 2), p3 = shf(prev, 3), p4 = shf(prev, 4), p5 = shf(prev, 5);
      double q0 = fma(-m0, p0, a0), q1 = m1 * p1, q2 = m2 * p2, q3 = m3 * p3, q4 = m4 * p4, q5 = m5 * p5;
      double a = (q0 - (q1 + q2)) - ((q3 + q4) + q5);
      prev = a; if (lane < 6) *vp = a;
    }
    acc += prev;
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[2] = (t1 - t0) / REPS; out[2] = acc; }
}
int main() {
  std::vector<double> h(36 * NS); for (int i = 0; i < 36 * NS; ++i) h[i] = (i % 7) - 3;
  double *d, *o; long long* c; cudaMalloc(&d, 8 * h.size()); cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  cudaMemcpy(d, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(varB, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  varA<<<1, 32, 8 * (36 * NS + 12 * NS)>>>(d, o, c);
  varB<<<1, 32, 8 * (72 * NS + 12 * NS)>>>(d, o, c);
  varC<<<1, 32, 8 * (36 * NS + 12 * NS)>>>(d, o, c);
  long long hc[3]; cudaDeviceSynchronize(); cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
  printf("A one block/step: %lld cycles per %d blocks (%.1f/block)\n", hc[0], NS, hc[0] / (double)NS);
  printf("B two blocks/step: %lld cycles per %d blocks (%.1f/block)\n", hc[1], NS, hc[1] / (double)NS);
  printf("C tree products:   %lld cycles per %d blocks (%.1f/block)\n", hc[2], NS, hc[2] / (double)NS);
}
