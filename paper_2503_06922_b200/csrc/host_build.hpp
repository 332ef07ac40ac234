// Host-side setup shared by the device library and the test-only serial
// emulation: descriptor validation, local stiffness, selector-row tables and
// the uniform-grid broad-phase structure over the lumen triangles.
//
// The grid replaces the reference's median-split AABB tree (mesh.py:199-268):
// every cell lists the triangles whose AABB lies within the query radius of
// the cell; a node query reads its one cell and applies the reference's exact
// AABB-vs-sphere leaf test to each listed triangle, so candidate sets equal
// the tree's leaf test.
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
  std::vector<int> cell_start, cell_tris;
  double origin[3] = {0, 0, 0};
  double inv_h = 1.0;
  int dims[3] = {1, 1, 1};
  // grid construction parameters (shared bit-for-bit with the device build, grid.cuh)
  double h = 1.0, rr = 0.0;
  long ncell = 0;
};

inline int grid_cell_host(double x, double o, double inv_h, int dim) {
  double f = floor((x - o) * inv_h);
  if (!(f >= 0.0)) return 0;
  if (f >= (double)(dim - 1)) return dim - 1;
  return (int)f;
}

// returns "" on success, else an error message.  with_lists = false stops after
// the grid sizing (the device library builds the cell lists itself, grid.cuh)
inline std::string build_mesh(const accfem_mesh_desc* d, double radius, HostMesh& M, bool with_lists = true) {
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
  // Uniform grid over the mesh bounds grown by the query radius.  Each cell
  // lists every triangle whose AABB lies within r of the cell box, so a node
  // query reads exactly one cell (no de-duplication); a node outside the
  // grid has no triangle within r.  Cell size starts at r/2 and is coarsened
  // until the grid has <= 2^22 cells and the lists hold <= 2^24 entries.
  const double rr = radius * (1.0 + 1e-9) + 1e-12;
  double glo[3], ghi[3];
  for (int a = 0; a < 3; ++a) {
    double pad = rr + 1e-9 * (bhi[a] - blo[a]) + 1e-12;
    glo[a] = blo[a] - pad;
    ghi[a] = bhi[a] + pad;
  }
  double h = radius > 0 ? 0.5 * radius : 1e-3;
  long ncell = 0;
  auto tri_range = [&](int t, int a, double inv, int dim, int& c0, int& c1) {
    c0 = grid_cell_host(M.lo[3L * t + a] - rr, glo[a], inv, dim);
    c1 = grid_cell_host(M.hi[3L * t + a] + rr, glo[a], inv, dim);
  };
  for (int tries = 0; tries < 200; ++tries) {
    ncell = 1;
    for (int a = 0; a < 3; ++a) {
      long da = (long)ceil((ghi[a] - glo[a]) / h) + 1;
      if (da < 1) da = 1;
      M.dims[a] = (int)da;
      ncell *= da;
    }
    bool ok = ncell <= (1L << 22);
    if (ok) {
      double inv = 1.0 / h;
      long entries = 0;
      for (int t = 0; t < T && entries <= (1L << 24); ++t) {
        long c = 1;
        for (int a = 0; a < 3; ++a) {
          int c0, c1;
          tri_range(t, a, inv, M.dims[a], c0, c1);
          c *= c1 - c0 + 1;
        }
        entries += c;
      }
      ok = entries <= (1L << 24);
    }
    if (ok) break;
    h *= 1.5;
  }
  for (int a = 0; a < 3; ++a) M.origin[a] = glo[a];
  M.inv_h = 1.0 / h;
  M.h = h;
  M.rr = rr;
  M.ncell = ncell;
  if (!with_lists) return "";
  // box distance between cell c (padded by 1e-6 h) and the AABB of triangle t
  auto near = [&](int t, const int* c) {
    double d2 = 0.0;
    for (int a = 0; a < 3; ++a) {
      double clo = glo[a] + c[a] * h - 1e-6 * h, chi = glo[a] + (c[a] + 1) * h + 1e-6 * h;
      double g = 0.0;
      if (M.lo[3L * t + a] > chi) g = M.lo[3L * t + a] - chi;
      else if (clo > M.hi[3L * t + a]) g = clo - M.hi[3L * t + a];
      d2 += g * g;
    }
    return d2 <= rr * rr;
  };
  auto cells_of = [&](int t, auto&& fn) {
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) tri_range(t, a, M.inv_h, M.dims[a], lo[a], hi[a]);
    int c[3];
    for (c[2] = lo[2]; c[2] <= hi[2]; ++c[2])
      for (c[1] = lo[1]; c[1] <= hi[1]; ++c[1])
        for (c[0] = lo[0]; c[0] <= hi[0]; ++c[0])
          if (near(t, c)) fn(((long)c[2] * M.dims[1] + c[1]) * M.dims[0] + c[0]);
  };
  std::vector<int> count(ncell + 1, 0);
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
