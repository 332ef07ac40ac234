// The persistent solve kernel k_solve<NW> (one CTA of NW warps = one
// scenario at a time) and its per-width launch entry points.  Each width is
// instantiated in its own translation unit (ksolve_<NW>.cu) so the build
// compiles them in parallel.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "engine.cuh"

namespace accfem {

struct KSolveEntry {
  int nw;
  bool cr;             // cyclic-reduction linear algebra (latency mode: one scenario per SM)
  const void* kernel;  // for cudaFuncSetAttribute / occupancy queries
  cudaError_t (*launch)(unsigned grid, size_t smem, cudaStream_t st, const Problem& P, const BatchDev& B,
                        double* ws_base, long ws_stride, long hot_stride);
};

KSolveEntry ksolve_entry_2();
KSolveEntry ksolve_entry_4();
KSolveEntry ksolve_entry_cr();  // 16-warp CTA, cyclic reduction

#if defined(ACCFEM_KSOLVE_NW)
// persistent solve; one CTA of NW warps = one scenario at a time.
// With hot_stride > 0 the team's hot arrays (factor, iterate, row state)
// live in dynamic shared memory; otherwise everything is in the global slab.
#if !defined(ACCFEM_KSOLVE_CR)
#define ACCFEM_KSOLVE_CR 0
#endif
template <int NW, bool CR>
__global__ void __launch_bounds__(32 * NW, 1)
    k_solve(Problem P, BatchDev B, double* ws_base, long ws_stride, long hot_stride) {
  extern __shared__ double smem[];
  __shared__ double red[NW];
  __shared__ int ired[NW + 1];
  __shared__ int next;
  __shared__ unsigned long long prof_acc[PF_COUNT];  // phase counters accumulate in shared memory
  const TeamCta cta{TeamWarp{(int)(threadIdx.x & 31)}, (int)(threadIdx.x >> 5), NW, red, ired};
  using Team = typename std::conditional<CR, TeamCR, TeamCta>::type;
  const Team team(cta);
  const long wid = blockIdx.x;
  double* hot = hot_stride > 0 ? smem : nullptr;
  Ws ws = ws_carve(ws_base + wid * ws_stride, hot, P.m.N, P.m.n_fixed, B.cmax_polish, nullptr, nullptr, CR,
                   hot ? B.hot_rows : 0);
  if (threadIdx.x < PF_COUNT) prof_acc[threadIdx.x] = 0;
  ws.prof = B.prof ? prof_acc : nullptr;
  __syncthreads();
  // load-balance record (optional): kept in shared memory, not in registers
  // that would stay live across the inlined solve
  __shared__ unsigned long long lb[3];  // start ns, busy ns, scenarios
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    lb[0] = t;
    lb[1] = 0;
    lb[2] = 0;
  }
  while (true) {
    if (threadIdx.x == 0) next = atomicAdd(B.work_counter, 1);
    __syncthreads();
    const int s = next;
    __syncthreads();
    if (s >= B.S) break;
    if (threadIdx.x == 0 && B.team_stats) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      lb[1] -= t;
    }
    run_scenario(team, P, B, s, ws);
    if (threadIdx.x == 0 && B.team_stats) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      lb[1] += t;
      lb[2] += 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && B.team_stats && wid < B.team_stats_cap) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    long long* o = B.team_stats + 4 * wid;
    o[0] = (long long)lb[2];
    o[1] = (long long)lb[1];
    o[2] = (long long)lb[0];
    o[3] = (long long)t_end;
  }
  if (B.prof && threadIdx.x < PF_COUNT) B.prof[wid * PF_COUNT + threadIdx.x] = prof_acc[threadIdx.x];
}

template <int NW, bool CR>
static cudaError_t ksolve_launch(unsigned grid, size_t smem, cudaStream_t st, const Problem& P, const BatchDev& B,
                                 double* ws_base, long ws_stride, long hot_stride) {
  k_solve<NW, CR><<<grid, 32 * NW, smem, st>>>(P, B, ws_base, ws_stride, hot_stride);
  return cudaGetLastError();
}
#define ACCFEM_KSOLVE_PASTE2(a, b) a##b
#define ACCFEM_KSOLVE_PASTE(a, b) ACCFEM_KSOLVE_PASTE2(a, b)
#if ACCFEM_KSOLVE_CR
KSolveEntry ksolve_entry_cr() {
#else
KSolveEntry ACCFEM_KSOLVE_PASTE(ksolve_entry_, ACCFEM_KSOLVE_NW)() {
#endif
  constexpr bool cr = ACCFEM_KSOLVE_CR != 0;
  return KSolveEntry{ACCFEM_KSOLVE_NW, cr, (const void*)k_solve<ACCFEM_KSOLVE_NW, cr>,
                     ksolve_launch<ACCFEM_KSOLVE_NW, cr>};
}
#endif

}  // namespace accfem
