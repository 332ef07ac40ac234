// Host-side setup shared by the device library and the test-only serial
// emulation: descriptor validation, local stiffness, selector-row tables and
// the uniform-grid broad-phase structure over the lumen triangles.
//
// The grid replaces the reference's median-split AABB tree (mesh.py:199-268):
// every triangle is listed in each cell its AABB overlaps; a node query walks
// the cells overlapped by its (slightly enlarged) search box and visits each
// triangle once, at the first visited cell its AABB covers, then applies the
// reference's exact AABB-vs-sphere leaf test.  Candidate sets are therefore
// identical to the tree's leaf test.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/accfem.h"

namespace accfem_host {

struct HostMesh {
  int T = 0;
  std::vector<double> corners, normals, lo, hi;
  std::vector<int> tri_cell_lo, cell_start, cell_tris;
  double origin[3] = {0, 0, 0};
  double inv_h = 1.0;
  int dims[3] = {1, 1, 1};
};

inline int grid_cell_host(double x, double o, double inv_h, int dim) {
  double f = floor((x - o) * inv_h);
  if (!(f >= 0.0)) return 0;
  if (f >= (double)(dim - 1)) return dim - 1;
  return (int)f;
}

// returns "" on success, else an error message
inline std::string build_mesh(const accfem_mesh_desc* d, double radius, HostMesh& M) {
  M = HostMesh();
  if (!d || d->triangle_count <= 0) return "";
  const int T = d->triangle_count, V = d->vertex_count;
  if (!d->vertices || !d->triangles || !d->normals) return "mesh arrays missing";
  M.T = T;
  M.corners.resize(9L * T);
  M.normals.assign(d->normals, d->normals + 3L * T);
  M.lo.resize(3L * T);
  M.hi.resize(3L * T);
  double blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int t = 0; t < T; ++t) {
    for (int k = 0; k < 3; ++k) {
      int64_t v = d->triangles[3L * t + k];
      if (v < 0 || v >= V) return "triangle indices out of range";
      for (int a = 0; a < 3; ++a) {
        double c = d->vertices[3 * v + a];
        if (!std::isfinite(c)) return "mesh vertices contain non-finite values";
        M.corners[9L * t + 3 * k + a] = c;
      }
    }
    for (int a = 0; a < 3; ++a) {
      double c0 = M.corners[9L * t + a], c1 = M.corners[9L * t + 3 + a], c2 = M.corners[9L * t + 6 + a];
      // corners.min(axis=1) / max(axis=1)  (mesh.py:206-207)
      double mn = c0 < c1 ? c0 : c1;
      mn = mn < c2 ? mn : c2;
      double mx = c0 > c1 ? c0 : c1;
      mx = mx > c2 ? mx : c2;
      M.lo[3L * t + a] = mn;
      M.hi[3L * t + a] = mx;
      blo[a] = mn < blo[a] ? mn : blo[a];
      bhi[a] = mx > bhi[a] ? mx : bhi[a];
    }
  }
  // cell size: half the query radius, coarsened until the grid has <= 2^22
  // cells and the cell lists hold <= 2^23 entries
  double h = radius > 0 ? 0.5 * radius : 1e-3;
  long ncell = 0;
  for (int tries = 0; tries < 200; ++tries) {
    ncell = 1;
    for (int a = 0; a < 3; ++a) {
      double ext = bhi[a] - blo[a];
      long da = (long)ceil(ext / h) + 1;
      if (da < 1) da = 1;
      M.dims[a] = (int)da;
      ncell *= da;
    }
    bool ok = ncell <= (1L << 22);
    if (ok) {
      double inv = 1.0 / h;
      long entries = 0;
      for (int t = 0; t < T && entries <= (1L << 23); ++t) {
        long c = 1;
        for (int a = 0; a < 3; ++a)
          c *= grid_cell_host(M.hi[3L * t + a], blo[a], inv, M.dims[a]) -
               grid_cell_host(M.lo[3L * t + a], blo[a], inv, M.dims[a]) + 1;
        entries += c;
      }
      ok = entries <= (1L << 23);
    }
    if (ok) break;
    h *= 1.5;
  }
  for (int a = 0; a < 3; ++a) M.origin[a] = blo[a];
  M.inv_h = 1.0 / h;
  M.tri_cell_lo.resize(3L * T);
  std::vector<int> count(ncell + 1, 0);
  std::vector<int> chi(3L * T);
  for (int t = 0; t < T; ++t)
    for (int a = 0; a < 3; ++a) {
      M.tri_cell_lo[3L * t + a] = grid_cell_host(M.lo[3L * t + a], M.origin[a], M.inv_h, M.dims[a]);
      chi[3L * t + a] = grid_cell_host(M.hi[3L * t + a], M.origin[a], M.inv_h, M.dims[a]);
    }
  auto cells_of = [&](int t, auto&& fn) {
    const int* lo = &M.tri_cell_lo[3L * t];
    const int* hi = &chi[3L * t];
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) fn((z * M.dims[1] + y) * M.dims[0] + x);
  };
  for (int t = 0; t < T; ++t) cells_of(t, [&](long c) { count[c + 1]++; });
  M.cell_start.assign(ncell + 1, 0);
  for (long c = 0; c < ncell; ++c) M.cell_start[c + 1] = M.cell_start[c] + count[c + 1];
  M.cell_tris.resize(M.cell_start[ncell] > 0 ? M.cell_start[ncell] : 1);
  std::vector<int> fill(M.cell_start.begin(), M.cell_start.end() - 1);
  for (int t = 0; t < T; ++t) cells_of(t, [&](long c) { M.cell_tris[fill[c]++] = t; });
  return "";
}

// 12x12 Euler-Bernoulli element matrix (beam.py:215-253)
inline void local_stiffness(const accfem_model_desc* d, double* k) {
  double E = d->young_modulus, A = d->cross_section_area, I = d->bending_inertia;
  double G = E / (2.0 * (1.0 + d->poisson_ratio)), J = d->torsion_constant, l0 = d->element_rest_length;
  double l2 = l0 * l0, l3 = l2 * l0;
  memset(k, 0, 144 * sizeof(double));
  auto put = [&](int i, int j, double v) {
    k[12 * i + j] = v;
    k[12 * j + i] = v;
  };
  put(0, 0, E * A / l0); put(6, 6, E * A / l0); put(0, 6, -E * A / l0);
  put(1, 1, 12.0 * E * I / l3); put(7, 7, 12.0 * E * I / l3); put(1, 7, -12.0 * E * I / l3);
  put(2, 2, 12.0 * E * I / l3); put(8, 8, 12.0 * E * I / l3); put(2, 8, -12.0 * E * I / l3);
  put(3, 3, G * J / l0); put(9, 9, G * J / l0); put(3, 9, -G * J / l0);
  put(4, 4, 4.0 * E * I / l0); put(10, 10, 4.0 * E * I / l0); put(4, 10, 2.0 * E * I / l0);
  put(5, 5, 4.0 * E * I / l0); put(11, 11, 4.0 * E * I / l0); put(5, 11, 2.0 * E * I / l0);
  put(1, 5, 6.0 * E * I / l2); put(1, 11, 6.0 * E * I / l2);
  put(7, 5, -6.0 * E * I / l2); put(7, 11, -6.0 * E * I / l2);
  put(2, 4, -6.0 * E * I / l2); put(2, 10, -6.0 * E * I / l2);
  put(8, 4, 6.0 * E * I / l2); put(8, 10, 6.0 * E * I / l2);
}

inline std::string validate(const accfem_model_desc* m, const accfem_settings* s) {
  if (!m || !s) return "null descriptor";
  if (m->node_count < 2) return "node_count must be >= 2";
  if (!(m->element_rest_length > 0.0)) return "element_rest_length must be positive";
  if (!m->rest_coords) return "rest_coords missing";
  if (!(m->young_modulus > 0 && m->cross_section_area > 0 && m->bending_inertia > 0 && m->poisson_ratio > 0 &&
        m->torsion_constant > 0))
    return "material parameters must be strictly positive";
  if (s->n_cables < 0 || s->n_cables > 8) return "at most 8 cables";
  if (s->n_fixed < 0 || s->n_fixed > 6 * m->node_count) return "bad fixed row count";
  std::vector<char> seen(6L * m->node_count, 0);
  for (int r = 0; r < s->n_fixed; ++r) {
    int nd = s->fixed_node[r], dof = s->fixed_dof[r];
    if (nd < 0 || nd >= m->node_count) return "fixed node out of range";
    if (dof < 0 || dof > 5) return "fixed_dofs entries must be in 0..5";
    if (seen[6 * nd + dof]) return "duplicate fixed DOF";
    seen[6 * nd + dof] = 1;
  }
  if (!(s->eps_abs > 0 && s->eps_rel > 0)) return "tolerances must be positive";
  if (!(s->alpha > 0 && s->alpha < 2)) return "alpha must lie in (0, 2)";
  if (!(s->beta0 > 0)) return "beta0 must be positive";
  if (s->max_iterations < 1) return "max_iterations must be >= 1";
  if (s->check_interval < 1) return "check_interval must be >= 1";
  if (s->margin < 0) return "margin must be >= 0";
  return "";
}

}  // namespace accfem_host
