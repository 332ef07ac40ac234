// Microbenchmark + check of the production cyclic-reduction factor/solve
// (csrc/cr.cuh) on one CTA team per SM, factor in shared memory (N = 101).
// Prints cycles per solve / factor and the residual |M x - b|_inf.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#define SEG_TIMING
#include "experimental/seg.cuh"
using namespace accfem;
constexpr int N = 101;
constexpr int REPS = 200;

template <int NW, int MAXI>
__global__ void __launch_bounds__(32 * NW) bench(const double* gD, const double* gU, const double* gb, double* out,
                                                 long long* cyc) {
  extern __shared__ double sm[];
  __shared__ double red[NW];
  __shared__ int ired[NW + 1];
  TeamCta team{TeamWarp{(int)(threadIdx.x & 31)}, (int)(threadIdx.x >> 5), NW, red, ired};
  double* D = sm;
  double* L = D + 22 * N;
  double* R = L + 36 * N;
  double* v = R + 36 * N;
  double* x = v + 6 * N;
  CrF F{D, L, R};
  for (int i = team.rank(); i < 22 * N; i += team.size()) D[i] = gD[i];
  for (int i = team.rank(); i < 36 * (N - 1); i += team.size()) L[36 + i] = gU[i];
  __syncthreads();
  long long t0 = clock64();
  int bad = cr_factor(team, N, F);
  long long t1 = clock64();
  long long ts = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    for (int i = team.rank(); i < 6 * N; i += team.size()) v[i] = gb[i];
    __syncthreads();
    long long a = clock64();
    cr_solve(team, N, F, v, x, 1, 0);
    ts += clock64() - a;
  }
  if (threadIdx.x == 0) {
    cyc[4 * blockIdx.x] = ts / REPS;
    cyc[4 * blockIdx.x + 1] = t1 - t0;
  }
  for (int i = team.rank(); i < 6 * N; i += team.size()) out[(long)blockIdx.x * 6 * N + i] = bad >= 0 ? NAN : x[i];
  {
    // the production twisted block LDL^T (linalg.cuh) on the same matrix
    __syncthreads();
    for (int i = team.rank(); i < 22 * N; i += team.size()) D[i] = gD[i];
    for (int i = team.rank(); i < 36 * (N - 1); i += team.size()) L[36 + i] = gU[i];
    __syncthreads();
    __shared__ double scr[160];
    long long b0 = clock64();
    int bad3 = twisted_factor(team, N, D, L + 36, scr, true);
    long long b1 = clock64();
    long long tt = 0;
    for (int rep = 0; rep < REPS; ++rep) {
      for (int i = team.rank(); i < 6 * N; i += team.size()) v[i] = gb[i];
      __syncthreads();
      long long t = clock64();
      twisted_solve(team, N, D, L + 36, v, x, v, 1, 0, true, true);
      __syncthreads();
      tt += clock64() - t;
    }
    if (threadIdx.x == 0) {
      cyc[4 * gridDim.x + 2 * blockIdx.x] = tt / REPS;
      cyc[4 * gridDim.x + 2 * blockIdx.x + 1] = b1 - b0;
    }
    for (int i = team.rank(); i < 6 * N; i += team.size())
      out[(long)(2 * gridDim.x + blockIdx.x) * 6 * N + i] = bad3 >= 0 ? NAN : v[i];
  }
  if constexpr (MAXI > 0) {
    // segmented variant: fresh matrix, segmented factor + solve
    __syncthreads();
    for (int i = team.rank(); i < 22 * N; i += team.size()) D[i] = gD[i];
    for (int i = team.rank(); i < 36 * (N - 1); i += team.size()) L[36 + i] = gU[i];
    __syncthreads();
    const int a = seg_bits(N, 5 * NW);
    long long a0 = clock64();
    int bad2 = seg_factor(team, N, F, a);
    long long a1 = clock64();
    long long tr = 0;
    for (int rep = 0; rep < REPS; ++rep) {
      for (int i = team.rank(); i < 6 * N; i += team.size()) v[i] = gb[i];
      __syncthreads();
      long long t = clock64();
      seg_solve(team, N, F, a, v, x);
      tr += clock64() - t;
    }
    if (threadIdx.x == 0) {
      cyc[4 * blockIdx.x + 2] = tr / REPS;
      cyc[4 * blockIdx.x + 3] = a1 - a0;
    }
    for (int i = team.rank(); i < 6 * N; i += team.size())
      out[(long)(gridDim.x + blockIdx.x) * 6 * N + i] = bad2 >= 0 ? NAN : x[i];
  }
}

template <int NW, int MAXI>
void run(int sms, const std::vector<double>& D, const std::vector<double>& U, const std::vector<double>& b,
         double* dD, double* dU, double* db, double* dout, long long* dc) {
  size_t per = (22 * N + 72 * N + 12 * N) * 8;
  cudaFuncSetAttribute(bench<NW, MAXI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  for (int per_sm : {1, 2}) {
    unsigned long long z8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_seg_t, z8, sizeof(z8));
    bench<NW, MAXI><<<sms * per_sm, 32 * NW, per>>>(dD, dU, db, dout, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z8, g_seg_t, sizeof(z8));
    printf("  seg phases (cycles/solve, block 0 thread 0): fwd %llu bar %llu sep-upd %llu sepchain %llu bar %llu bwd %llu bar %llu\n",
           z8[0] / REPS, z8[1] / REPS, z8[2] / REPS, z8[3] / REPS, z8[4] / REPS, z8[5] / REPS, z8[6] / REPS);
    const int nb = sms * per_sm;
    std::vector<long long> c(6 * nb);
    cudaMemcpy(c.data(), dc, 8 * c.size(), cudaMemcpyDeviceToHost);
    for (int mode = 0; mode < 3; ++mode) {
      std::vector<double> x(6 * N);
      cudaMemcpy(x.data(), dout + (long)mode * nb * 6 * N, 8 * x.size(), cudaMemcpyDeviceToHost);
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
      double s0 = 0, f = 0;
      for (int i = 0; i < nb; ++i) {
        s0 += mode < 2 ? c[4 * i + 2 * mode] : c[4 * nb + 2 * i];
        f += mode < 2 ? c[4 * i + 2 * mode + 1] : c[4 * nb + 2 * i + 1];
      }
      printf("%s N=%d warps/team=%d teams/SM=%d: solve %.0f cycles, %s %.0f cycles, rel residual %.2e %s\n",
             mode == 2 ? "twistd" : mode ? "cr_seg" : "cr    ", N, NW, per_sm, s0 / nb, "factor", f / nb, res / bm,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
}

int main() {
  // diagonally dominant SPD block-tridiagonal test matrix
  std::vector<double> D(22 * N, 0.0), U(36 * N, 0.0), b(6 * N);
  for (int i = 0; i < 36 * N; ++i) U[i] = 0.05 * ((i * 31) % 7 - 3);
  for (int i = 0; i < N; ++i)
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) D[22 * i + r * (r + 1) / 2 + c] = r == c ? 4.0 : 0.1 * ((r + c + i) % 3 - 1);
  for (int i = 0; i < 6 * N; ++i) b[i] = 1.0 + 0.01 * (i % 17);
  double *dD, *dU, *db, *dout;
  long long* dc;
  cudaMalloc(&dD, 8 * D.size()); cudaMalloc(&dU, 8 * U.size()); cudaMalloc(&db, 8 * b.size());
  cudaMalloc(&dout, 8 * 6 * N * 3000); cudaMalloc(&dc, 8 * 8192);
  cudaMemcpy(dD, D.data(), 8 * D.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), 8 * U.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 1>(sms, D, U, b, dD, dU, db, dout, dc);
  run<2, 1>(sms, D, U, b, dD, dU, db, dout, dc);
  run<3, 1>(sms, D, U, b, dD, dU, db, dout, dc);
  run<4, 1>(sms, D, U, b, dD, dU, db, dout, dc);
  run<8, 1>(sms, D, U, b, dD, dU, db, dout, dc);
}
