// Microbenchmark: one warp = one block-tridiagonal chain (N blocks of 6x6),
// factor resident in shared memory; cycles per forward sweep for variants.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

constexpr int N = 51;  // one half of the twisted solve for N=101
constexpr int REPS = 200;

__device__ __forceinline__ void ld36(const double* p, double* a) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < 18; ++i) { double2 v = q[i]; a[2 * i] = v.x; a[2 * i + 1] = v.y; }
}

// V1: one lane does the full 6x6 matvec per step
__global__ void v1(const double* gM, const double* gb, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm + (threadIdx.x / 32) * (36 * N + 6 * N);
  double* b = M + 36 * N;
  int lane = threadIdx.x & 31;
  for (int i = lane; i < 36 * N; i += 32) M[i] = gM[i];
  for (int i = lane; i < 6 * N; i += 32) b[i] = gb[i];
  __syncwarp();
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    if (lane == 0) {
      double p[6] = {0, 0, 0, 0, 0, 0};
      for (int i = 0; i < N; ++i) {
        double m[36], a[6];
        ld36(M + 36 * i, m);
#pragma unroll
        for (int r = 0; r < 6; ++r) a[r] = b[6 * i + r];
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          double s0 = m[6 * r] * p[0] + m[6 * r + 2] * p[2] + m[6 * r + 4] * p[4];
          double s1 = m[6 * r + 1] * p[1] + m[6 * r + 3] * p[3] + m[6 * r + 5] * p[5];
          a[r] -= s0 + s1;
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) { p[r] = a[r] * 0.5; b[6 * i + r] = a[r]; }
      }
      acc += p[0];
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = (t1 - t0) / REPS; out[blockIdx.x] = acc; }
}

// V2: 6 lanes, each one row; vector exchanged by shuffles
__global__ void v2(const double* gM, const double* gb, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm + (threadIdx.x / 32) * (36 * N + 6 * N);
  double* b = M + 36 * N;
  int lane = threadIdx.x & 31;
  for (int i = lane; i < 36 * N; i += 32) M[i] = gM[i];
  for (int i = lane; i < 6 * N; i += 32) b[i] = gb[i];
  __syncwarp();
  int r = lane % 6;
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    double prev = 0;
    for (int i = 0; i < N; ++i) {
      const double* mr = M + 36 * i + 6 * r;
      double m0 = mr[0], m1 = mr[1], m2 = mr[2], m3 = mr[3], m4 = mr[4], m5 = mr[5];
      double a = b[6 * i + r];
      double p0 = __shfl_sync(~0u, prev, 0), p1 = __shfl_sync(~0u, prev, 1), p2 = __shfl_sync(~0u, prev, 2);
      double p3 = __shfl_sync(~0u, prev, 3), p4 = __shfl_sync(~0u, prev, 4), p5 = __shfl_sync(~0u, prev, 5);
      a -= (m0 * p0 + m2 * p2 + m4 * p4) + (m1 * p1 + m3 * p3 + m5 * p5);
      prev = a * 0.5;
      if (lane < 6) b[6 * i + r] = a;
    }
    acc += prev;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = (t1 - t0) / REPS; out[blockIdx.x] = acc; }
}

// V3: 6 lanes, vector exchanged through shared memory (broadcast reads)
__global__ void v3(const double* gM, const double* gb, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm + (threadIdx.x / 32) * (36 * N + 6 * N + 8);
  double* b = M + 36 * N;
  double* xv = b + 6 * N;
  int lane = threadIdx.x & 31;
  for (int i = lane; i < 36 * N; i += 32) M[i] = gM[i];
  for (int i = lane; i < 6 * N; i += 32) b[i] = gb[i];
  if (lane < 8) xv[lane] = 0;
  __syncwarp();
  int r = lane % 6;
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    if (lane < 6) xv[r] = 0;
    __syncwarp();
    for (int i = 0; i < N; ++i) {
      const double* mr = M + 36 * i + 6 * r;
      double2 ma = *reinterpret_cast<const double2*>(mr), mb = *reinterpret_cast<const double2*>(mr + 2),
              mc = *reinterpret_cast<const double2*>(mr + 4);
      double a = b[6 * i + r];
      double2 pa = *reinterpret_cast<const double2*>(xv), pb = *reinterpret_cast<const double2*>(xv + 2),
              pc = *reinterpret_cast<const double2*>(xv + 4);
      a -= (ma.x * pa.x + mb.x * pb.x + mc.x * pc.x) + (ma.y * pa.y + mb.y * pb.y + mc.y * pc.y);
      __syncwarp();
      if (lane < 6) { xv[r] = a * 0.5; b[6 * i + r] = a; }
      __syncwarp();
    }
    acc += xv[0];
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = (t1 - t0) / REPS; out[blockIdx.x] = acc; }
}

// V4: 36 lanes-worth: lane (r, c-pair): 6 rows x 3 column-pairs = 18 lanes;
// partial dot of 2 entries, reduced over 3 lanes with shuffles
__global__ void v4(const double* gM, const double* gb, double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* M = sm + (threadIdx.x / 32) * (36 * N + 6 * N);
  double* b = M + 36 * N;
  int lane = threadIdx.x & 31;
  for (int i = lane; i < 36 * N; i += 32) M[i] = gM[i];
  for (int i = lane; i < 6 * N; i += 32) b[i] = gb[i];
  __syncwarp();
  int l = lane < 18 ? lane : 0;
  int r = l / 3, cp = l % 3;
  long long t0 = clock64();
  double acc = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    double prev = 0;  // lane r*3 holds x[r] (valid for cp == 0)
    for (int i = 0; i < N; ++i) {
      double2 m = *reinterpret_cast<const double2*>(M + 36 * i + 6 * r + 2 * cp);
      double p0 = __shfl_sync(~0u, prev, 3 * (2 * cp));
      double p1 = __shfl_sync(~0u, prev, 3 * (2 * cp + 1));
      double s = m.x * p0 + m.y * p1;
      s += __shfl_down_sync(~0u, s, 1);
      s += __shfl_down_sync(~0u, s, 1);  // not exact tree; timing only
      double a = b[6 * i + r] - s;
      prev = a * 0.5;
      if (lane < 18 && cp == 0) b[6 * i + r] = a;
    }
    acc += prev;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = (t1 - t0) / REPS; out[blockIdx.x] = acc; }
}

int main() {
  std::vector<double> hM(36 * N), hb(6 * N);
  for (int i = 0; i < 36 * N; ++i) hM[i] = 0.01 * ((i * 7919) % 13 - 6);
  for (int i = 0; i < 6 * N; ++i) hb[i] = 1.0 + 0.001 * i;
  double *dM, *db, *dout;
  long long* dc;
  cudaMalloc(&dM, 8 * 36 * N); cudaMalloc(&db, 8 * 6 * N); cudaMalloc(&dout, 8 * 4096); cudaMalloc(&dc, 8 * 65536);
  cudaMemcpy(dM, hM.data(), 8 * 36 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), 8 * 6 * N, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void (*ks[4])(const double*, const double*, double*, long long*) = {v1, v2, v3, v4};
  const char* names[4] = {"V1 one-lane", "V2 6-lane shfl", "V3 6-lane smem", "V4 18-lane"};
  for (int kv = 0; kv < 4; ++kv) {
    for (int wpb : {1, 2, 4, 8}) {
      size_t sm = (size_t)wpb * (36 * N + 6 * N + 8) * 8;
      cudaFuncSetAttribute(ks[kv], cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      ks[kv]<<<sms, 32 * wpb, sm>>>(dM, db, dout, dc);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> c(sms * wpb);
      cudaMemcpy(c.data(), dc, 8 * c.size(), cudaMemcpyDeviceToHost);
      double avg = 0; for (auto v : c) avg += v; avg /= c.size();
      printf("%-16s warps/SM=%d  cycles/sweep=%8.0f  cycles/step=%6.1f  %s\n", names[kv], wpb, avg, avg / N,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
