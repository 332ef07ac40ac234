// Microbenchmark of the production cyclic reduction (csrc/cr.cuh) on a whole
// CTA (latency mode), factor and vectors in shared memory, N = 101.
// Prints cycles per factor / per single-RHS solve / per 21-RHS solve and the
// residual |M x - b|_inf / |b|_inf.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#define CR_TIMING
#include "../../paper_2503_06922_b200/csrc/cr.cuh"
using namespace accfem;
constexpr int N = 101;
constexpr int REPS = 100;

template <int NW>
__global__ void __launch_bounds__(32 * NW, 1) bench(const double* gD, const double* gU, const double* gb, double* out,
                                                    long long* cyc) {
  extern __shared__ double sm[];
  __shared__ double red[NW];
  __shared__ int ired[NW + 1];
  const TeamCR team(TeamCta{TeamWarp{(int)(threadIdx.x & 31)}, (int)(threadIdx.x >> 5), NW, red, ired});
  double* D = sm;
  double* LR = D + 22 * N;
  double* U = LR + 36;
  double* v = LR + 72 * N;
  double* vm = v + 6 * N;  // 21 rhs
  for (int i = team.rank(); i < 22 * N; i += team.size()) D[i] = gD[i];
  for (int i = team.rank(); i < 36 * (N - 1); i += team.size()) U[i] = gU[i];
  __syncthreads();
  long long t0 = clock64();
  int bad = twisted_factor(team, N, D, U, nullptr, true);
  __syncthreads();
  long long t1 = clock64();
  long long ts = 0, tm = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.rank(); i < 6 * N; i += team.size()) v[i] = gb[i];
    __syncthreads();
    long long a = clock64();
    twisted_solve(team, N, D, U, v, nullptr, v, 1, 0, true, true);
    __syncthreads();
    ts += clock64() - a;
#if defined(CR_TIMING)
    if (threadIdx.x == 0 && blockIdx.x == 0 && rep >= 10)
      for (int k = 1; k < 32; ++k) g_cr_t[k] += s_cr_t[k] - s_cr_t[0];
#endif
  }
  {
    __syncthreads();
    long long a = clock64();
    for (int k = 0; k < 100; ++k) __syncthreads();
    if (threadIdx.x == 0) cyc[1000 + blockIdx.x] = (clock64() - a) / 100;
  }
  for (int rep = 0; rep < 10; ++rep) {
    for (int i = team.rank(); i < 21 * 6 * N; i += team.size()) vm[i] = gb[i % (6 * N)];
    __syncthreads();
    long long a = clock64();
    twisted_solve_chunks(team, N, D, U, vm, 21, 6 * N);
    __syncthreads();
    tm += clock64() - a;
  }
  if (threadIdx.x == 0) {
    cyc[3 * blockIdx.x] = t1 - t0;
    cyc[3 * blockIdx.x + 1] = ts / REPS;
    cyc[3 * blockIdx.x + 2] = tm / 10;
  }
  for (int i = team.rank(); i < 6 * N; i += team.size()) out[(long)blockIdx.x * 6 * N + i] = bad >= 0 ? NAN : v[i];
}

template <int NW>
void run(int blocks, const std::vector<double>& D, const std::vector<double>& U, const std::vector<double>& b,
         double* dD, double* dU, double* db, double* dout, long long* dc) {
  size_t per = (22 * N + 72 * N + 22 * 6 * N) * 8;
  cudaFuncSetAttribute(bench<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  bench<NW><<<blocks, 32 * NW, per>>>(dD, dU, db, dout, dc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> c(3 * blocks);
  cudaMemcpy(c.data(), dc, 8 * c.size(), cudaMemcpyDeviceToHost);
  std::vector<double> x(6 * N);
  cudaMemcpy(x.data(), dout, 8 * x.size(), cudaMemcpyDeviceToHost);
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
  printf("cr16 N=%d warps=%d blocks=%d: factor %lld, solve %lld, 21-rhs solve %lld cycles, rel residual %.2e %s\n", N,
         NW, blocks, c[0], c[1], c[2], res / bm, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  std::vector<double> D(22 * N, 0.0), U(36 * N, 0.0), b(6 * N);
  for (int i = 0; i < 36 * N; ++i) U[i] = 0.05 * ((i * 31) % 7 - 3);
  for (int i = 0; i < N; ++i)
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) D[22 * i + r * (r + 1) / 2 + c] = r == c ? 4.0 : 0.1 * ((r + c + i) % 3 - 1);
  for (int i = 0; i < 6 * N; ++i) b[i] = 1.0 + 0.01 * (i % 17);
  double *dD, *dU, *db, *dout;
  long long* dc;
  cudaMalloc(&dD, 8 * D.size()); cudaMalloc(&dU, 8 * U.size()); cudaMalloc(&db, 8 * b.size());
  cudaMalloc(&dout, 8 * 6 * N * 200); cudaMalloc(&dc, 8 * 8192);
  cudaMemcpy(dD, D.data(), 8 * D.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), 8 * U.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
  run<16>(1, D, U, b, dD, dU, db, dout, dc);
  {
    long long z[64] = {0};
    cudaMemcpyToSymbol(g_cr_t, z, sizeof(z));
  }
  run<16>(1, D, U, b, dD, dU, db, dout, dc);
  {
    long long t[64];
    cudaMemcpyFromSymbol(t, g_cr_t, sizeof(t));
    const int order[] = {0, 1, 2, 3, 4, 20, 21, 25, 24, 23, 22};
    printf("single-rhs solve, cycles since start at stage:");
    for (int k = 1; k < 11; ++k) printf(" %d:%lld", order[k], t[order[k]] / 90);
    long long bar;
    cudaMemcpy(&bar, dc + 1000, 8, cudaMemcpyDeviceToHost);
    printf("   | one __syncthreads (16 warps): %lld cycles\n", bar);
  }
  run<8>(1, D, U, b, dD, dU, db, dout, dc);
  run<4>(1, D, U, b, dD, dU, db, dout, dc);
}
