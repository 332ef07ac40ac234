// k_solve<16, CR>: the latency-mode kernel (one 16-warp CTA = one scenario,
// cyclic-reduction linear algebra, cr.cuh); see ksolve.cuh
#define ACCFEM_KSOLVE_NW 8
#define ACCFEM_KSOLVE_CR 1
#include "ksolve.cuh"
