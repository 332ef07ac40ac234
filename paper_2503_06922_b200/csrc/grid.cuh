// Device build of the broad-phase uniform grid over the lumen triangles.
//
// Replaces the reference's AabbTree construction (mesh.py:204-243) for large
// meshes: the host only sizes the grid (O(T) per
// sizing try, host_build.hpp build_mesh(with_lists = false)); the cell lists
// -- O(T x cells per triangle), the part that grows with 10^4-10^5 triangle
// STL meshes -- are built here in four passes:
//
//   k_grid_count   one warp per triangle: count the cells within the query
//                  radius of its AABB (atomicAdd per cell)
//   scan           exclusive sum of the counts -> CSR cell_start
//   k_grid_fill    one warp per triangle: claim a slot per cell
//   sort           cub segmented radix sort of every cell's list by triangle id
//                  (accfem.cu; k_grid_sort, the earlier per-cell rank sort, is
//                  kept for the microbenchmarks)
//
// The result equals the host build (host_build.hpp) entry for entry: the
// cell ranges and the cell-vs-AABB distance test use the same operation
// order with explicit round-to-nearest intrinsics (no FMA contraction, as
// the x86-64 host code has none), and the host fills cells in increasing
// triangle order, which the per-cell sort reproduces.
#pragma once
#include <cuda_runtime.h>

namespace accfem {

struct GridBuild {
  const double* lo;  // T x 3 triangle AABB minima
  const double* hi;  // T x 3 maxima
  int T;
  int dims[3];
  double origin[3];
  double h, inv_h, rr;
};

__device__ __forceinline__ int grid_cell_build(double x, double o, double inv_h, int dim) {
  double f = floor(__dmul_rn(__dsub_rn(x, o), inv_h));
  if (!(f >= 0.0)) return 0;
  if (f >= (double)(dim - 1)) return dim - 1;
  return (int)f;
}

__device__ __forceinline__ void grid_tri_range(const GridBuild& g, int t, int* c0, int* c1) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    c0[a] = grid_cell_build(__dsub_rn(g.lo[3L * t + a], g.rr), g.origin[a], g.inv_h, g.dims[a]);
    c1[a] = grid_cell_build(__dadd_rn(g.hi[3L * t + a], g.rr), g.origin[a], g.inv_h, g.dims[a]);
  }
}

// box distance between cell c (padded by 1e-6 h) and the AABB of triangle t
__device__ __forceinline__ bool grid_near(const GridBuild& g, const double* lo, const double* hi, const int* c) {
  double d2 = 0.0;
  const double pad = __dmul_rn(1e-6, g.h);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double clo = __dsub_rn(__dadd_rn(g.origin[a], __dmul_rn((double)c[a], g.h)), pad);
    double chi = __dadd_rn(__dadd_rn(g.origin[a], __dmul_rn((double)(c[a] + 1), g.h)), pad);
    double gap = 0.0;
    if (lo[a] > chi) gap = __dsub_rn(lo[a], chi);
    else if (clo > hi[a]) gap = __dsub_rn(clo, hi[a]);
    d2 = __dadd_rn(d2, __dmul_rn(gap, gap));
  }
  return d2 <= __dmul_rn(g.rr, g.rr);
}

// visit every cell within rr of triangle t's AABB; the lanes of a warp split
// the flattened (x fastest) cell range of the triangle, so a triangle spanning
// many cells is not walked by one thread (the visit order does not matter:
// count and fill only claim slots, k_grid_sort restores the host order)
template <class F>
__device__ __forceinline__ void grid_cells_of(const GridBuild& g, int t, int lane, F&& fn) {
  int c0[3], c1[3];
  grid_tri_range(g, t, c0, c1);
  double lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = g.lo[3L * t + a];
    hi[a] = g.hi[3L * t + a];
  }
  const int nx = c1[0] - c0[0] + 1, ny = c1[1] - c0[1] + 1, nz = c1[2] - c0[2] + 1;
  const long n = (long)nx * ny * nz;
  for (long k = lane; k < n; k += 32) {
    int c[3];
    c[0] = c0[0] + (int)(k % nx);
    c[1] = c0[1] + (int)((k / nx) % ny);
    c[2] = c0[2] + (int)(k / ((long)nx * ny));
    if (grid_near(g, lo, hi, c)) fn(((long)c[2] * g.dims[1] + c[1]) * g.dims[0] + c[0]);
  }
}

// one warp per triangle
__global__ void k_grid_count(GridBuild g, int* count) {
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < g.T; t += warps)
    grid_cells_of(g, (int)t, lane, [&](long c) { atomicAdd(count + c, 1); });
}

__global__ void k_grid_fill(GridBuild g, int* fill, int* cell_tris) {
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * (blockDim.x >> 5);
  for (long t = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < g.T; t += warps)
    grid_cells_of(g, (int)t, lane, [&](long c) { cell_tris[atomicAdd(fill + c, 1)] = (int)t; });
}

// one warp per cell: rank sort of the cell's (distinct) triangle ids from the
// fill order in `src` into increasing order in `dst` (a cell lists tens to a
// few hundred triangles; each lane ranks its entries against the whole list)
__global__ void k_grid_sort(long ncell, const int* cell_start, const int* src, int* dst) {
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * (blockDim.x >> 5);
  for (long c = blockIdx.x * (long)(blockDim.x >> 5) + (threadIdx.x >> 5); c < ncell; c += warps) {
    const int b = cell_start[c], e = cell_start[c + 1];
    for (int i = b + lane; i < e; i += 32) {
      const int v = src[i];
      int rank = 0;
      for (int j = b; j < e; ++j) rank += src[j] < v;
      dst[b + rank] = v;
    }
  }
}

}  // namespace accfem
