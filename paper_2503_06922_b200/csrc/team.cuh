// Execution "team" abstraction shared by the device build (nvcc, sm_100a)
// and the serial test-only emulation build (g++).
//
// Device: one warp = one team = one scenario.  PARFOR strides the lanes,
// team.sync() is __syncwarp (which also orders the warp's memory traffic),
// reductions are butterfly shuffles so every lane ends with the result.
// Emulation: one "lane" runs every PARFOR iteration in order.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define DEV __device__ __forceinline__
#define DEVNI __device__ __noinline__
#define HDEV __host__ __device__ inline
#else
#include <math.h>
#include <string.h>
#include <algorithm>
#define DEV inline
#define DEVNI inline
#define HDEV inline
#endif

#define PARFOR(i, n) for (int i = team.rank(); i < (n); i += team.size())

// strided loop with four independent bodies per pass, so the loads of four
// elements are in flight together (plain PARFOR bodies run one at a time)
template <class Team, class F>
DEV void parfor4(const Team& team, int n, F&& f) {
  const int s = team.size();
  int j = team.rank();
  for (; j + 3 * s < n; j += 4 * s) {
    f(j);
    f(j + s);
    f(j + 2 * s);
    f(j + 3 * s);
  }
  for (; j < n; j += s) f(j);
}

// phase timers (development builds with -DACCFEM_PROFILE only)
#if defined(__CUDA_ARCH__) && defined(ACCFEM_PROFILE)
#define PROF_T0(v) long long v = clock64()
#define PROF_ADD(ws, k, v) \
  do { if ((ws).prof && team.rank() == 0) (ws).prof[k] += (unsigned long long)(clock64() - (v)); } while (0)
#else
#define PROF_T0(v)
#define PROF_ADD(ws, k, v)
#endif
enum ProfPhase { PF_ELEMENT = 0, PF_DETECT, PF_RUIZ, PF_FACTOR, PF_ITER, PF_CHAIN, PF_CHECK, PF_POLISH, PF_DIRECT,
                 PF_POST, PF_TOTAL, PF_ITERS, PF_FRAMES, PF_POL_FACTOR, PF_POL_W, PF_POL_ROUNDS,
                 PF_PR_LIST, PF_PR_CHOL, PF_PR_COMB, PF_PR_REFINE, PF_PR_CORR, PF_PR_MULT, PF_COUNT = 24 };

namespace accfem {

#if defined(__CUDACC__)
struct TeamWarp {
  int lane;
  DEV int rank() const { return lane; }
  DEV int size() const { return 32; }
  DEV void sync() const { __syncwarp(); }
  DEV double max(double v) const {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
  DEV double min(double v) const {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
  DEV double sum(double v) const {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  }
  DEV int isum(int v) const {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  }
  DEV int imin(int v) const {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = ::min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
  DEV int any(bool p) const { return __any_sync(0xffffffffu, p); }
  DEV double bcast(double v, int src) const { return __shfl_sync(0xffffffffu, v, src); }
  DEV int ibcast(int v, int src) const { return __shfl_sync(0xffffffffu, v, src); }
  // exclusive prefix over flags in lane order within one 32-wide chunk
  DEV int ballot_prefix(bool p, int* total) const {
    unsigned b = __ballot_sync(0xffffffffu, p);
    *total = __popc(b);
    return __popc(b & ((1u << lane) - 1u));
  }
};
#endif

#if defined(__CUDACC__)
// A team of `nw` warps of one CTA working on one scenario: PARFOR strides
// all 32*nw threads, sync is the CTA barrier, reductions combine the warp
// butterflies through a few words of shared memory (fixed order, so results
// are deterministic).
struct TeamCta {
  TeamWarp w;
  int warp, nw;
  double* red;  // nw doubles of shared scratch
  int* ired;    // nw + 1 ints of shared scratch
  DEV int rank() const { return 32 * warp + w.lane; }
  DEV int size() const { return 32 * nw; }
  DEV void sync() const { __syncthreads(); }
  DEV double max(double v) const {
    v = w.max(v);
    if (w.lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int i = 1; i < nw; ++i) r = fmax(r, red[i]);
    __syncthreads();
    return r;
  }
  DEV double min(double v) const {
    v = w.min(v);
    if (w.lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int i = 1; i < nw; ++i) r = fmin(r, red[i]);
    __syncthreads();
    return r;
  }
  DEV double sum(double v) const {
    v = w.sum(v);
    if (w.lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int i = 1; i < nw; ++i) r += red[i];
    __syncthreads();
    return r;
  }
  DEV int isum(int v) const {
    v = w.isum(v);
    if (w.lane == 0) ired[warp] = v;
    __syncthreads();
    int r = 0;
    for (int i = 0; i < nw; ++i) r += ired[i];
    __syncthreads();
    return r;
  }
  DEV int imin(int v) const {
    v = w.imin(v);
    if (w.lane == 0) ired[warp] = v;
    __syncthreads();
    int r = ired[0];
    for (int i = 1; i < nw; ++i) r = ::min(r, ired[i]);
    __syncthreads();
    return r;
  }
  DEV int any(bool p) const { return isum(w.any(p) ? 1 : 0) > 0; }
  DEV int ballot_prefix(bool p, int* total) const {
    unsigned b = __ballot_sync(0xffffffffu, p);
    if (w.lane == 0) ired[warp] = __popc(b);
    __syncthreads();
    int before = 0, tot = 0;
    for (int i = 0; i < nw; ++i) {
      if (i < warp) before += ired[i];
      tot += ired[i];
    }
    __syncthreads();
    *total = tot;
    return before + __popc(b & ((1u << w.lane) - 1u));
  }
  // run a warp-cooperative routine on warp 0 only, everyone waits; returns its int result
  template <class F>
  DEV int on_warp0(F&& f) const {
    int r = 0;
    if (warp == 0) r = f(w);
    if (rank() == 0) ired[nw] = r;
    __syncthreads();
    r = ired[nw];
    __syncthreads();
    return r;
  }
};
#endif

struct TeamSerial {
  DEV int rank() const { return 0; }
  DEV int size() const { return 1; }
  DEV void sync() const {}
  DEV double max(double v) const { return v; }
  DEV double min(double v) const { return v; }
  DEV double sum(double v) const { return v; }
  DEV int isum(int v) const { return v; }
  DEV int imin(int v) const { return v; }
  DEV int any(bool p) const { return p; }
  DEV double bcast(double v, int) const { return v; }
  DEV int ibcast(int v, int) const { return v; }
  DEV int ballot_prefix(bool p, int* total) const {
    *total = p ? 1 : 0;
    return 0;
  }
};

// ---------------------------------------------------------------------------
// IEEE round-to-nearest arithmetic with no FMA contraction: the narrow phase
// must reproduce numpy's operation order bit for bit.
// ---------------------------------------------------------------------------
#if defined(__CUDA_ARCH__)
DEV double xmul(double a, double b) { return __dmul_rn(a, b); }
DEV double xadd(double a, double b) { return __dadd_rn(a, b); }
DEV double xsub(double a, double b) { return __dsub_rn(a, b); }
#else
DEV double xmul(double a, double b) { return a * b; }
DEV double xadd(double a, double b) { return a + b; }
DEV double xsub(double a, double b) { return a - b; }
#endif

// numpy einsum("ij,ij->i") over 3 columns sums (0, 2) first, then 1
DEV double edot3(const double* a, const double* b) {
  return xadd(xadd(xmul(a[0], b[0]), xmul(a[2], b[2])), xmul(a[1], b[1]));
}
// numpy linalg.norm(axis=1) over 3 columns: sqrt((x0^2 + x1^2) + x2^2)
DEV double enorm3(const double* a) {
  return sqrt(xadd(xadd(xmul(a[0], a[0]), xmul(a[1], a[1])), xmul(a[2], a[2])));
}

}  // namespace accfem
