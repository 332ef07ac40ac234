// k_solve<4>: see ksolve.cuh
#define ACCFEM_KSOLVE_NW 4
#include "ksolve.cuh"
