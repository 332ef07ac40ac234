// Single-RHS twisted block solve on one warp (factor in shared memory,
// N = 101): the production 6-lane shuffle solve vs the register mat-vec
// solve (twisted_solve_multi with one right-hand side: lanes 0/1 carry the
// whole 6-vector of the top/bottom half), plus a variant with the coupling
// block of the next step prefetched.  Cycles per solve, residual check.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2503_06922_b200/csrc/linalg.cuh"
using namespace accfem;
constexpr int N = 101;
constexpr int REPS = 200;

// register mat-vec chain with one-step-ahead prefetch of the coupling block
DEV void solve_reg_pf(const TeamWarp& team, int N, const double* __restrict__ D, const double* __restrict__ U,
                      double* v) {
  __builtin_assume(__isShared(D));
  __builtin_assume(__isShared(U));
  __builtin_assume(__isShared(v));
  const int lane = team.lane;
  const bool top = lane == 0;
  const bool act = lane < 2;
  const int k = twist_split(N);
  const int cnt = top ? k : N - 1 - k;
  double p[6] = {0, 0, 0, 0, 0, 0};
  if (act && cnt > 0) {
    int i = top ? 0 : N - 1;
    ld6(v + 6 * i, p);
    const int di = top ? 1 : -1;
    double Mn[36];
    ld36(top ? U : U + 36 * (N - 2), Mn);
    for (int t = 1; t < cnt; ++t) {
      i += di;
      double M[36], a[6];
#pragma unroll
      for (int e = 0; e < 36; ++e) M[e] = Mn[e];
      if (t + 1 < cnt) ld36(top ? U + 36 * i : U + 36 * (i - 1), Mn);
      ld6(v + 6 * i, a);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double s0 = M[6 * r] * p[0] + M[6 * r + 2] * p[2] + M[6 * r + 4] * p[4];
        const double s1 = M[6 * r + 1] * p[1] + M[6 * r + 3] * p[3] + M[6 * r + 5] * p[5];
        a[r] -= s0 + s1;
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) p[r] = a[r];
      st6(v + 6 * i, a);
    }
  }
  double part[6] = {0, 0, 0, 0, 0, 0};
  if (act && cnt > 0) {
    double M[36];
    ld36(top ? U + 36 * (k - 1) : U + 36 * k, M);
#pragma unroll
    for (int r = 0; r < 6; ++r)
      part[r] = M[6 * r] * p[0] + M[6 * r + 1] * p[1] + M[6 * r + 2] * p[2] + M[6 * r + 3] * p[3] +
                M[6 * r + 4] * p[4] + M[6 * r + 5] * p[5];
  }
  double xk[6];
  {
    double t[6], bk[6], Dk[36];
    ld6(v + 6 * k, bk);
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      double o = __shfl_xor_sync(0xffffffffu, part[r], 1);
      double pt = top ? part[r] : o, pb = top ? o : part[r];
      t[r] = bk[r] - (pt + pb);
    }
    unpack_sym(D + kDiag * k, Dk);
#pragma unroll
    for (int r = 0; r < 6; ++r)
      xk[r] = Dk[6 * r] * t[0] + Dk[6 * r + 1] * t[1] + Dk[6 * r + 2] * t[2] + Dk[6 * r + 3] * t[3] +
              Dk[6 * r + 4] * t[4] + Dk[6 * r + 5] * t[5];
  }
  __syncwarp();
  for (int q = lane; q < 6 * N; q += 32) {
    const int i = q / 6, r = q - 6 * i;
    if (i == k) continue;
    const double* Di = D + kDiag * i;
    const double* vi = v + 6 * i;
    const double z = (Di[sidx(r, 0)] * vi[0] + Di[sidx(r, 2)] * vi[2] + Di[sidx(r, 4)] * vi[4]) +
                     (Di[sidx(r, 1)] * vi[1] + Di[sidx(r, 3)] * vi[3] + Di[sidx(r, 5)] * vi[5]);
    __syncwarp();
    v[q] = z;
  }
  __syncwarp();
  if (act) {
    if (top) st6(v + 6 * k, xk);
#pragma unroll
    for (int r = 0; r < 6; ++r) p[r] = xk[r];
    int i = k;
    const int di = top ? -1 : 1;
    double Mn[36];
    if (cnt > 0) ld36(top ? U + 36 * (k - 1) : U + 36 * k, Mn);
    for (int t = 0; t < cnt; ++t) {
      i += di;
      double a[6], M[36];
#pragma unroll
      for (int e = 0; e < 36; ++e) M[e] = Mn[e];
      if (t + 1 < cnt) ld36(top ? U + 36 * (i - 1) : U + 36 * i, Mn);
      ld6(v + 6 * i, a);
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        const double s0 = M[r] * p[0] + M[12 + r] * p[2] + M[24 + r] * p[4];
        const double s1 = M[6 + r] * p[1] + M[18 + r] * p[3] + M[30 + r] * p[5];
        a[r] -= s0 + s1;
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) p[r] = a[r];
      st6(v + 6 * i, a);
    }
  }
  __syncwarp();
}

__global__ void bench(const double* gD, const double* gU, const double* gb, double* out, long long* cyc) {
  extern __shared__ double sm[];
  TeamWarp team{(int)(threadIdx.x & 31)};
  double* D = sm;
  double* U = D + kDiag * N;
  double* v = U + 36 * N;
  double* t = v + 6 * N;
  __shared__ double scr[160];
  for (int i = team.lane; i < kDiag * N; i += 32) D[i] = gD[i];
  for (int i = team.lane; i < 36 * (N - 1); i += 32) U[i] = gU[i];
  __syncwarp();
  twisted_factor(team, N, D, U, scr, true);
  __syncwarp();
  long long c[3] = {0, 0, 0};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < REPS; ++rep) {
      for (int i = team.lane; i < 6 * N; i += 32) v[i] = gb[i];
      __syncwarp();
      long long a = clock64();
      if (mode == 0) twisted_solve(team, N, D, U, v, t, v, 1, 0, true, true);
      else if (mode == 1) twisted_solve_multi(team, N, D, U, v, t, v, 1, 0);
      else solve_reg_pf(team, N, D, U, v);
      __syncwarp();
      c[mode] += clock64() - a;
    }
    for (int i = team.lane; i < 6 * N; i += 32) out[(long)(blockIdx.x * 3 + mode) * 6 * N + i] = v[i];
  }
  if (team.lane == 0)
    for (int m = 0; m < 3; ++m) cyc[blockIdx.x * 3 + m] = c[m] / REPS;
}

int main() {
  std::vector<double> D(kDiag * N, 0.0), U(36 * N, 0.0), b(6 * N);
  for (int i = 0; i < 36 * N; ++i) U[i] = 0.05 * ((i * 31) % 7 - 3);
  for (int i = 0; i < N; ++i)
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) D[kDiag * i + r * (r + 1) / 2 + c] = r == c ? 4.0 : 0.1 * ((r + c + i) % 3 - 1);
  for (int i = 0; i < 6 * N; ++i) b[i] = 1.0 + 0.01 * (i % 17);
  double *dD, *dU, *db, *dout;
  long long* dc;
  cudaMalloc(&dD, 8 * D.size()); cudaMalloc(&dU, 8 * U.size()); cudaMalloc(&db, 8 * b.size());
  cudaMalloc(&dout, 8 * 6 * N * 3 * 600); cudaMalloc(&dc, 8 * 3 * 600);
  cudaMemcpy(dD, D.data(), 8 * D.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dU, U.data(), 8 * U.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 8 * b.size(), cudaMemcpyHostToDevice);
  size_t per = (kDiag * N + 36 * N + 12 * N) * 8;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  for (int blocks : {1, 148, 148 * 3, 148 * 4}) {
    bench<<<blocks, 32, per>>>(dD, dU, db, dout, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> c(3 * blocks);
    cudaMemcpy(c.data(), dc, 8 * c.size(), cudaMemcpyDeviceToHost);
    std::vector<double> x(3 * 6 * N);
    cudaMemcpy(x.data(), dout, 8 * x.size(), cudaMemcpyDeviceToHost);
    double d01 = 0, d02 = 0;
    for (int i = 0; i < 6 * N; ++i) {
      d01 = fmax(d01, fabs(x[i] - x[6 * N + i]));
      d02 = fmax(d02, fabs(x[i] - x[12 * N + i]));
    }
    double s[3] = {0, 0, 0};
    for (int i = 0; i < blocks; ++i)
      for (int m = 0; m < 3; ++m) s[m] += c[3 * i + m];
    printf("blocks %4d: shuffle solve %.0f, register solve %.0f, register+prefetch %.0f cycles; |x diff| %.1e %.1e %s\n",
           blocks, s[0] / blocks, s[1] / blocks, s[2] / blocks, d01, d02, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}
