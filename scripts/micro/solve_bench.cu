// Microbenchmark of the production twisted_solve / twisted_factor on one
// warp per block with the factor in shared memory (N = 101).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2503_06922_b200/csrc/linalg.cuh"
using namespace accfem;
constexpr int N = 101;
constexpr int REPS = 100;
__global__ void bench(const double* gD, const double* gU, const double* gb, double* out, long long* cyc, int mode) {
  extern __shared__ double sm[];
  const int w = threadIdx.x / 32;
  double* D = sm + w * (22 * N + 36 * N + 12 * N);
  double* U = D + 22 * N;
  double* rhs = U + 36 * N;
  double* tmp = rhs + 6 * N;
  TeamWarp team{(int)(threadIdx.x & 31)};
  for (int i = team.lane; i < 22 * N; i += 32) D[i] = gD[i];
  for (int i = team.lane; i < 36 * (N - 1); i += 32) U[i] = gU[i];
  __syncwarp();
  long long t0 = clock64();
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.lane; i < 6 * N; i += 32) rhs[i] = gb[i];
    __syncwarp();
    if (mode == 0) twisted_solve(team, N, D, U, rhs, tmp, rhs, 1, 0, true, true);
    else twisted_solve(team, N, D, U, rhs, tmp, rhs, 1, 0, false);
  }
  long long t1 = clock64();
  if (team.lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + w] = (t1 - t0) / REPS;
  if (team.lane == 0) out[blockIdx.x] = rhs[7];
}
int main() {
  std::vector<double> D(22 * N, 0.0), U(36 * N, 0.0), b(6 * N);
  for (int i = 0; i < N; ++i) for (int r = 0; r < 6; ++r) D[22 * i + r * (r + 1) / 2 + r] = 0.5;
  for (int i = 0; i < 36 * N; ++i) U[i] = 0.001 * ((i * 31) % 7 - 3);
  for (int i = 0; i < 6 * N; ++i) b[i] = 1.0;
  double *dD, *dU, *db, *dout; long long* dc;
  cudaMalloc(&dD, 8 * D.size()); cudaMalloc(&dU, 8 * U.size()); cudaMalloc(&db, 8 * b.size());
  cudaMalloc(&dout, 8 * 4096); cudaMalloc(&dc, 8 * 4096);
  cudaMemcpy(dD, D.data(), 8 * D.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), 8 * U.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t per = (22 * N + 36 * N + 12 * N) * 8;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220000);
  for (int mode = 0; mode < 2; ++mode)
    for (int wpb : {1, 2, 3}) {
      bench<<<sms, 32 * wpb, per * wpb>>>(dD, dU, db, dout, dc, mode);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> c(sms * wpb);
      cudaMemcpy(c.data(), dc, 8 * c.size(), cudaMemcpyDeviceToHost);
      double avg = 0; for (auto v : c) avg += v; avg /= c.size();
      printf("twisted_solve N=%d sh=%d warps/SM=%d: %.0f cycles/solve (%.1f per step) %s\n", N, mode == 0, wpb, avg,
             avg / N, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
}
