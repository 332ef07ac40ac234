// Microbenchmark + check of the nested-dissection factor / solve (csrc/nd.cuh)
// on a whole CTA (latency mode), storage in shared memory, N = 101 and 51, 21.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#define ND_TIMING
#include "experimental/nd.cuh"
using namespace accfem;
constexpr int REPS = 100;

template <int NW>
__global__ void __launch_bounds__(32 * NW, 1) bench(int N, const double* gD, const double* gU, const double* gb,
                                                    double* out, long long* cyc) {
  extern __shared__ double sm[];
  __shared__ double red[NW];
  __shared__ int ired[NW + 1];
  __shared__ double piv[32 * NW];
  double* nd = sm;
  double* v = nd + nd_doubles(N);
  double* vm = v + 6 * N;
  const TeamND team(TeamCta{TeamWarp{(int)(threadIdx.x & 31)}, (int)(threadIdx.x >> 5), NW, red, ired}, nd, piv);
  __syncthreads();
  long long t0 = clock64();
  int bad = twisted_factor(team, N, const_cast<double*>(gD), const_cast<double*>(gU), nullptr, true);
  __syncthreads();
  long long t1 = clock64();
  long long ts = 0, tm = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.rank(); i < 6 * N; i += team.size()) v[i] = gb[i];
    __syncthreads();
    long long a = clock64();
    twisted_solve(team, N, nullptr, nullptr, v, nullptr, v, 1, 0, true, true);
    __syncthreads();
    ts += clock64() - a;
    if (threadIdx.x == 0 && rep == REPS - 1)
      for (int k = 0; k < 12; ++k) cyc[8 + k] = s_nd_t[k + 1] - s_nd_t[0];
  }
  for (int rep = 0; rep < 10; ++rep) {
    for (int i = team.rank(); i < 4 * 6 * N; i += team.size()) vm[i] = gb[i % (6 * N)];
    __syncthreads();
    long long a = clock64();
    twisted_solve_chunks(team, N, nullptr, nullptr, vm, 4, 6 * N);
    __syncthreads();
    tm += clock64() - a;
  }
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = ts / REPS;
    cyc[2] = tm / 10;
  }
  for (int i = team.rank(); i < 6 * N; i += team.size()) out[i] = bad >= 0 ? NAN : v[i];
  for (int i = team.rank(); i < 6 * N; i += team.size()) out[6 * N + i] = vm[3 * 6 * N + i];
}

template <int NW>
void run(int N) {
  std::vector<double> D(22 * N, 0.0), U(36 * N, 0.0), b(6 * N);
  for (int i = 0; i < 36 * N; ++i) U[i] = 0.05 * ((i * 31) % 7 - 3);
  for (int i = 0; i < N; ++i)
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) D[22 * i + r * (r + 1) / 2 + c] = r == c ? 4.0 : 0.1 * ((r + c + i) % 3 - 1);
  for (int i = 0; i < 6 * N; ++i) b[i] = 1.0 + 0.01 * (i % 17);
  double *dD, *dU, *db, *dout;
  long long* dc;
  cudaMalloc(&dD, 8 * D.size()); cudaMalloc(&dU, 8 * U.size()); cudaMalloc(&db, 8 * b.size());
  cudaMalloc(&dout, 8 * 12 * N); cudaMalloc(&dc, 256);
  cudaMemcpy(dD, D.data(), 8 * D.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), 8 * U.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
  size_t per = (nd_doubles(N) + 6 * N * 5) * 8;
  cudaFuncSetAttribute(bench<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  for (int t = 0; t < 2; ++t) bench<NW><<<1, 32 * NW, per>>>(N, dD, dU, db, dout, dc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c[20];
  cudaMemcpy(c, dc, 160, cudaMemcpyDeviceToHost);
  printf("  stages (cycles since entry):");
  for (int k = 0; k < 10; ++k) printf(" %lld", c[8 + k]);
  printf("\n");
  double worst = 0;
  for (int m = 0; m < 2; ++m) {
    std::vector<double> x(6 * N);
    cudaMemcpy(x.data(), dout + m * 6 * N, 8 * x.size(), cudaMemcpyDeviceToHost);
    double res = 0, bm = 0;
    for (int i = 0; i < N; ++i)
      for (int r = 0; r < 6; ++r) {
        double a = 0;
        for (int c2 = 0; c2 < 6; ++c2) {
          int p = r >= c2 ? r * (r + 1) / 2 + c2 : c2 * (c2 + 1) / 2 + r;
          a += D[22 * i + p] * x[6 * i + c2];
          if (i + 1 < N) a += U[36 * i + 6 * r + c2] * x[6 * (i + 1) + c2];
          if (i > 0) a += U[36 * (i - 1) + 6 * c2 + r] * x[6 * (i - 1) + c2];
        }
        res = fmax(res, fabs(a - b[6 * i + r]));
        bm = fmax(bm, fabs(b[6 * i + r]));
      }
    worst = fmax(worst, res / bm);
    printf("  mode %d residual %.2e x[0..3] %.6f %.6f %.6f\n", m, res / bm, x[0], x[1], x[2]);
    if (m == 0 && N == 6) {
      FILE* fo = fopen("gpurun_out/nd6.txt", "w");
      for (int q = 0; q < 6 * N; ++q) fprintf(fo, "%.17g\n", x[q]);
      fclose(fo);
    }
  }
  printf("nd N=%d warps=%d smem %zu B: factor %lld, solve %lld, 4-rhs solve %lld cycles, rel residual %.2e %s\n", N,
         NW, per, c[0], c[1], c[2], worst, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(dD); cudaFree(dU); cudaFree(db); cudaFree(dout); cudaFree(dc);
}

int main() {
  for (int N : {7, 2, 6, 12, 101}) run<16>(N);
}
