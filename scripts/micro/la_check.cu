// Correctness + timing of the look-ahead solve vs the one-block-per-step solve
// (production code from linalg.cuh), factor resident in shared memory.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2503_06922_b200/csrc/linalg.cuh"
using namespace accfem;
constexpr int REPS = 100;
__global__ void run(int N, const double* gA, const double* gC, const double* gb, double* Qg, double* x1, double* x2,
                    long long* cyc) {
  extern __shared__ double sm[];
  double* D = sm;
  double* U = D + kDiag * N;
  double* rhs = U + 36 * N;
  double* tmp = rhs + 6 * N;
  double* scr = tmp + 6 * N;
  double* Qs = scr + 160;  // Q copy in shared memory (variant)
  TeamWarp team{(int)(threadIdx.x & 31)};
  for (int i = team.lane; i < kDiag * N; i += 32) D[i] = gA[i];
  for (int i = team.lane; i < 36 * (N - 1); i += 32) U[i] = gC[i];
  __syncwarp();
  int bad = twisted_factor(team, N, D, U, scr, true);
  twisted_q(team, N, U, Qg);
  for (int i = team.lane; i < 6 * N; i += 32) rhs[i] = gb[i];
  __syncwarp();
  long long t0 = clock64();
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.lane; i < 6 * N; i += 32) rhs[i] = gb[i];
    __syncwarp();
    twisted_solve(team, N, D, U, rhs, tmp, rhs, 1, 0, true, true);
  }
  long long t1 = clock64();
  for (int i = team.lane; i < 6 * N; i += 32) x1[i] = rhs[i];
  long long t2 = clock64();
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.lane; i < 6 * N; i += 32) rhs[i] = gb[i];
    __syncwarp();
    twisted_solve_la(team, N, D, U, Qg, rhs, tmp, rhs, true);
  }
  long long t3 = clock64();
  for (int i = team.lane; i < 6 * N; i += 32) x2[i] = rhs[i];
  for (int i = team.lane; i < 4 * ((N + 1) / 2 + 1) * 36; i += 32) Qs[i] = Qg[i];
  __syncwarp();
  long long t4 = clock64();
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.lane; i < 6 * N; i += 32) rhs[i] = gb[i];
    __syncwarp();
    twisted_solve_la(team, N, D, U, Qs, rhs, tmp, rhs, true);
  }
  long long t5 = clock64();
  if (team.lane == 0) { cyc[0] = (t1 - t0) / REPS; cyc[1] = (t3 - t2) / REPS; cyc[2] = bad; cyc[3] = (t5 - t4) / REPS; }
}
int main() {
  for (int N : {2, 3, 4, 5, 6, 7, 10, 21, 50, 51, 100, 101}) {
    std::vector<double> A(22 * N, 0.0), C(36 * N, 0.0), b(6 * N);
    unsigned s = 12345 + N;
    auto rnd = [&]() { s = s * 1103515245u + 12345u; return ((s >> 8) & 0xffff) / 65536.0 - 0.5; };
    for (int i = 0; i < N; ++i)
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c <= r; ++c) A[22 * i + r * (r + 1) / 2 + c] = (r == c ? 10.0 : 0.5 * rnd());
    for (int i = 0; i < 36 * (N - 1); ++i) C[i] = rnd();
    for (int i = 0; i < 6 * N; ++i) b[i] = rnd();
    double *dA, *dC, *db, *dQ, *dx1, *dx2; long long* dc;
    cudaMalloc(&dA, 8 * A.size()); cudaMalloc(&dC, 8 * C.size()); cudaMalloc(&db, 8 * b.size());
    cudaMalloc(&dQ, 8 * 4 * ((N + 1) / 2 + 1) * 36); cudaMalloc(&dx1, 8 * 6 * N); cudaMalloc(&dx2, 8 * 6 * N);
    cudaMalloc(&dc, 32);
    cudaMemcpy(dA, A.data(), 8 * A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C.data(), 8 * C.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
    size_t smem = 8 * (kDiag * N + 36 * N + 12 * N + 160 + 4 * ((N + 1) / 2 + 1) * 36);
    cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    run<<<1, 32, smem>>>(N, dA, dC, db, dQ, dx1, dx2, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> x1(6 * N), x2(6 * N); long long c[4];
    cudaMemcpy(x1.data(), dx1, 8 * 6 * N, cudaMemcpyDeviceToHost);
    cudaMemcpy(x2.data(), dx2, 8 * 6 * N, cudaMemcpyDeviceToHost);
    cudaMemcpy(c, dc, 32, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < 6 * N; ++i) { err = fmax(err, fabs(x1[i] - x2[i])); mx = fmax(mx, fabs(x1[i])); }
    printf("N=%4d bad=%lld one-step %6lld  look-ahead(Q global) %6lld  (Q smem) %6lld cyc  err %.1e %s\n", N, c[2], c[0],
           c[1], c[3], err / mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}
