// k_solve<2>: see ksolve.cuh
#define ACCFEM_KSOLVE_NW 2
#include "ksolve.cuh"
