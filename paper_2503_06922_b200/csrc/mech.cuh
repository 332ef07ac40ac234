// Per-frame mechanics on one team (warp) = one scenario:
//   element_pass   co-rotational frames, F_int, 6x6 block-tridiagonal tangent
//                  (reference beam.py:256-356, so3.py)
//   external_force cable tip wrench + applied + uniform load
//                  (engine.py:108-121, constraints.py:111-136)
//   detect_pass    node-vs-lumen broad phase on a uniform grid + bit-exact
//                  narrow phase + per-node winner + node-ordered compaction
//                  (contact.py:49-120, mesh.py:245-329)
#pragma once
#include "problem.cuh"
#include "so3.cuh"

namespace accfem {

// co-rotational frame of one element from its chord (length len > 0), the end
// directors and the rest offset mean0^T E0 (beam.py:256-271)
DEV void element_frame(const double* ch, double len, const double* Ra, const double* Rb, const double* off,
                       double* F) {
  double mid[9], pred[9], fix[9];
  rot_mid(Ra, Rb, mid);
  mat3_mul(mid, off, pred);
  double c0[3] = {pred[0], pred[3], pred[6]};
  double e1[3] = {ch[0] / len, ch[1] / len, ch[2] / len};
  rot_between(c0, e1, fix);
  mat3_mul(fix, pred, F);
}

// per-model constants (RobotModel.__post_init__, beam.py:71-99): rest
// directors, chord lengths, rest element frames E0 (identity offsets),
// offsets mean0^T E0 and the fused rest products T0^T E0 of both ends.
template <class Team>
DEV void model_setup(const Team& team, int N, const double* rest, double* rest_dir, double* rest_len,
                     double* rest_frames, double* offsets, double* qa, double* qb, int* bad) {
  PARFOR(k, N) rot_exp(rest + 6 * k + 3, rest_dir + 9 * k);
  team.sync();
  const double eye[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  int worst = 1 << 30;
  PARFOR(e, N - 1) {
    const double* pa = rest + 6 * e;
    const double* pb = rest + 6 * (e + 1);
    double ch[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
    double len = sqrt((ch[0] * ch[0] + ch[1] * ch[1]) + ch[2] * ch[2]);
    rest_len[e] = len;
    if (len < kMinChord) {
      worst = e < worst ? e : worst;
      continue;
    }
    const double* Ta = rest_dir + 9 * e;
    const double* Tb = rest_dir + 9 * (e + 1);
    double E0[9], mean0[9];
    element_frame(ch, len, Ta, Tb, eye, E0);
    for (int i = 0; i < 9; ++i) rest_frames[9 * e + i] = E0[i];
    rot_mid(Ta, Tb, mean0);
    mat3_tmul(mean0, E0, offsets + 9 * e);
    mat3_tmul(Ta, E0, qa + 9 * e);
    mat3_tmul(Tb, E0, qb + 9 * e);
  }
  worst = team.imin(worst);
  if (team.rank() == 0) *bad = worst < (1 << 30) ? worst + 1 : 0;
  team.sync();
}

// director matrices of every node: R_k = exp(theta_k)
template <class Team>
DEV void directors_pass(const Team& team, const Problem& P, const double* x, Ws& ws) {
  const int N = P.m.N;
  PARFOR(k, N) rot_exp(x + 6 * k + 3, ws.R + 9 * k);
  team.sync();
}

// 3x3 block B_pq = F (K_local,pq F^T) of the rotated element matrix
DEV void elem_block(const double* F, const double* kl, int p, int q, double* B) {
  double T[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double* kr = kl + 12 * (3 * p + i) + 3 * q;
      T[3 * i + j] = kr[0] * F[3 * j] + kr[1] * F[3 * j + 1] + kr[2] * F[3 * j + 2];
    }
  mat3_mul(F, T, B);
}

// symmetrised 6x6 diagonal part of node a (p0 = 0) or node b (p0 = 2):
// 0.5 (X + X^T) of the blocks (p0..p0+1)^2, full 6x6 into out
DEV void elem_sym_diag(const double* F, const double* kl, int p0, double* out) {
  double B0[9], B1[9];
  for (int h = 0; h < 2; ++h) {  // diagonal 3x3 blocks
    elem_block(F, kl, p0 + h, p0 + h, B0);
    double* o = out + 21 * h;  // (3h, 3h)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      o[6 * i + i] = B0[3 * i + i];
#pragma unroll
      for (int j = i + 1; j < 3; ++j) {
        const double v = 0.5 * (B0[3 * i + j] + B0[3 * j + i]);
        o[6 * i + j] = v;
        o[6 * j + i] = v;
      }
    }
  }
  elem_block(F, kl, p0, p0 + 1, B0);
  elem_block(F, kl, p0 + 1, p0, B1);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double v = 0.5 * (B0[3 * i + j] + B1[3 * j + i]);
      out[6 * i + 3 + j] = v;
      out[6 * (3 + j) + i] = v;
    }
}

// coupling block (node a rows, node b columns): 0.5 (B_ab + B_ba^T)
DEV void elem_coupling(const double* F, const double* kl, double* out) {
  double B0[9], B1[9];
  for (int al = 0; al < 2; ++al)
    for (int be = 0; be < 2; ++be) {
      elem_block(F, kl, al, 2 + be, B0);
      elem_block(F, kl, 2 + be, al, B1);
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) out[6 * (3 * al + i) + 3 * be + j] = 0.5 * (B0[3 * i + j] + B1[3 * j + i]);
    }
}

// element frames, internal force and (optionally) the block-tridiagonal
// tangent.  Returns 0, or the 1-based index of the first degenerate element
// (beam.py:262-264).
template <class Team>
DEV int element_pass(const Team& team, const Problem& P, const double* x, Ws& ws, bool tangent) {
  const ModelDev& M = P.m;
  const int N = M.N, E = N - 1;
  directors_pass(team, P, x, ws);
  int bad = 1 << 30;
  PARFOR(e, E) {
    const double* pa = x + 6 * e;
    const double* pb = x + 6 * (e + 1);
    double ch[3] = {pb[0] - pa[0], pb[1] - pa[1], pb[2] - pa[2]};
    double len = sqrt((ch[0] * ch[0] + ch[1] * ch[1]) + ch[2] * ch[2]);
    if (len < kMinChord) {
      bad = e < bad ? e : bad;
      continue;
    }
    const double* Ra = ws.R + 9 * e;
    const double* Rb = ws.R + 9 * (e + 1);
    double F[9];
    element_frame(ch, len, Ra, Rb, M.offsets + 9 * e, F);
    for (int i = 0; i < 9; ++i) ws.frames[9 * e + i] = F[i];
    // local deformation d = [0 | psi_a | stretch 0 0 | psi_b]   (beam.py:283-308)
    double t1[9], t2[9], d[12];
    mat3_tmul(F, Ra, t1);
    mat3_mul(t1, M.qa + 9 * e, t2);
    rot_log(t2, d + 3);
    mat3_tmul(F, Rb, t1);
    mat3_mul(t1, M.qb + 9 * e, t2);
    rot_log(t2, d + 9);
    d[0] = d[1] = d[2] = 0.0;
    d[6] = len - M.rest_len[e];
    d[7] = d[8] = 0.0;
    // f_loc = K_local d, rotated per 3-block by the frame   (beam.py:311-325)
    double fl[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 3; j < 12; ++j) acc += d[j] * M.kl[12 * i + j];
      fl[i] = acc;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) mat3_vec(F, fl + 3 * b, ws.fe + 12 * e + 3 * b);
    if (tangent) {
      // 3x3 blocks B_pq = F kl_pq F^T of the element matrix, symmetrised
      // (beam.py:341-346), written straight into the block-tridiagonal
      // storage: node a's diagonal part into KD[e], the coupling into KU[e];
      // node b's diagonal part is added to KD[e+1] after the barrier below
      elem_sym_diag(F, M.kl, 0, ws.KD + 36 * e);
      elem_coupling(F, M.kl, ws.KU + 36 * e);
      if (e == E - 1)
        for (int i = 0; i < 36; ++i) ws.KD[36 * E + i] = 0.0;
    }
  }
  bad = team.imin(bad);
  if (bad < (1 << 30)) return bad + 1;
  team.sync();
  // conflict-free gather: node k takes element k-1 (as node b) then element k (node a)
  PARFOR(i, 6 * N) {
    int k = i / 6, c = i % 6;
    double acc = 0.0;
    if (k > 0) acc += ws.fe[12 * (k - 1) + 6 + c];
    if (k < E) acc += ws.fe[12 * k + c];
    ws.fint[i] = acc;
  }
  if (tangent) {
    // node b's part: KD[e+1] += sym(bb(e)) (recomputed from the stored frame;
    // the sum equals the reference's bb + aa: addition commutes)
    PARFOR(e, E) {
      double bb[36];
      elem_sym_diag(ws.frames + 9 * e, M.kl, 2, bb);
      double* kd = ws.KD + 36 * (e + 1);
      for (int i = 0; i < 36; ++i) kd[i] += bb[i];
    }
  }
  team.sync();
  return 0;
}

// F_a = cable wrench at the last node + applied + uniform  (engine.py:108-121)
template <class Team>
DEV void external_force(const Team& team, const Problem& P, const double* tensions, const double* applied,
                        Ws& ws) {
  const ModelDev& M = P.m;
  const int n = 6 * M.N;
  PARFOR(i, n) {
    double f = 0.0;
    int k = i / 6, c = i % 6;
    if (k == M.N - 1 && M.n_cables > 0 && tensions) {
      const double* tm = ws.frames + 9 * (M.N - 2);
      double force[3] = {0.0, 0.0, 0.0}, moment[3] = {0.0, 0.0, 0.0};
      for (int j = 0; j < M.n_cables; ++j) {
        const double* dir = M.cable_dir + 3 * j;
        const double* off = M.cable_off + 3 * j;
        double fl[3] = {tensions[j] * dir[0], tensions[j] * dir[1], tensions[j] * dir[2]};
        double mo[3] = {off[1] * fl[2] - off[2] * fl[1], off[2] * fl[0] - off[0] * fl[2],
                        off[0] * fl[1] - off[1] * fl[0]};
        double gf[3], gm[3];
        mat3_vec(tm, fl, gf);
        mat3_vec(tm, mo, gm);
        for (int q = 0; q < 3; ++q) {
          force[q] += gf[q];
          moment[q] += gm[q];
        }
      }
      f += c < 3 ? force[c] : moment[c - 3];
    }
    if (applied) f += applied[i];
    if (M.has_uniform && c < 3) f += M.uniform[c];
    ws.fa[i] = f;
    ws.g[i] = ws.fint[i] - f;
  }
  team.sync();
}

// ---------------------------------------------------------------------------
// contact detection
// ---------------------------------------------------------------------------

// closest point on triangle (a, b, c) to p; numpy operation order, no FMA
// (mesh.py:271-329, first matching region wins)
DEV void closest_point(const double* p, const double* a, const double* b, const double* c, double* out) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  for (int i = 0; i < 3; ++i) {
    ab[i] = xsub(b[i], a[i]);
    ac[i] = xsub(c[i], a[i]);
    ap[i] = xsub(p[i], a[i]);
    bp[i] = xsub(p[i], b[i]);
    cp[i] = xsub(p[i], c[i]);
  }
  double d1 = edot3(ab, ap), d2 = edot3(ac, ap);
  double d3 = edot3(ab, bp), d4 = edot3(ac, bp);
  double d5 = edot3(ab, cp), d6 = edot3(ac, cp);
  if (d1 <= 0 && d2 <= 0) { for (int i = 0; i < 3; ++i) out[i] = a[i]; return; }
  if (d3 >= 0 && d4 <= d3) { for (int i = 0; i < 3; ++i) out[i] = b[i]; return; }
  if (d6 >= 0 && d5 <= d6) { for (int i = 0; i < 3; ++i) out[i] = c[i]; return; }
  double vc = xsub(xmul(d1, d4), xmul(d3, d2));
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    double den = xsub(d1, d3);
    double v = den != 0.0 ? d1 / den : 0.0;
    for (int i = 0; i < 3; ++i) out[i] = xadd(a[i], xmul(v, ab[i]));
    return;
  }
  double vb = xsub(xmul(d5, d2), xmul(d1, d6));
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    double den = xsub(d2, d6);
    double w = den != 0.0 ? d2 / den : 0.0;
    for (int i = 0; i < 3; ++i) out[i] = xadd(a[i], xmul(w, ac[i]));
    return;
  }
  double va = xsub(xmul(d3, d6), xmul(d5, d4));
  double e43 = xsub(d4, d3), e56 = xsub(d5, d6);
  if (va <= 0 && e43 >= 0 && e56 >= 0) {
    double den = xadd(e43, e56);
    double w = den != 0.0 ? e43 / den : 0.0;
    for (int i = 0; i < 3; ++i) out[i] = xadd(b[i], xmul(w, xsub(c[i], b[i])));
    return;
  }
  double den = xadd(xadd(va, vb), vc);
  double v = den != 0.0 ? vb / den : 0.0;
  double w = den != 0.0 ? vc / den : 0.0;
  for (int i = 0; i < 3; ++i) out[i] = xadd(xadd(a[i], xmul(v, ab[i])), xmul(w, ac[i]));
}


// per-node winner (min signed distance, ties to the lower triangle id),
// then node-ordered compaction.  Returns the contact count.
template <class Team>
DEV int detect_pass(const Team& team, const Problem& P, const double* x, Ws& ws, int* pairs_out = nullptr) {
  const MeshDev& G = P.mesh;
  const int N = P.m.N;
  const double margin = P.s.margin, radius = P.s.radius;
  const double r2 = xmul(radius, radius);
  int pairs = 0;  // (node, triangle) pairs that pass the broad phase
  PARFOR(k, N) {
    double p[3] = {x[6 * k], x[6 * k + 1], x[6 * k + 2]};
    int best_t = -1;
    double best_s = 0.0, best_gap = 0.0, best_pp[3] = {0.0, 0.0, 0.0};
    int c[3];
    bool inside = true;
    for (int a = 0; a < 3; ++a) {
      double f = floor((p[a] - G.origin[a]) * G.inv_h);
      inside = inside && (f >= 0.0) && (f < (double)G.dims[a]);
      c[a] = inside ? (int)f : 0;
    }
    const int cell = inside ? (c[2] * G.dims[1] + c[1]) * G.dims[0] + c[0] : 0;
    const int it0 = inside ? G.cell_start[cell] : 0, it1 = inside ? G.cell_start[cell + 1] : 0;
    // candidates in batches of four: the indices, then the AABBs of the
    // batch are requested together (two L2 round trips per batch instead of
    // two per candidate); the winner rule is order independent
    for (int it = it0; it < it1; it += 4) {
      int tb[4];
      double lob[4][3], hib[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) tb[u] = it + u < it1 ? G.cell_tris[it + u] : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int tt = tb[u] >= 0 ? tb[u] : tb[0];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          lob[u][a] = G.lo[3 * tt + a];
          hib[u][a] = G.hi[3 * tt + a];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = tb[u];
        if (t < 0) continue;
        // exact reference AABB-vs-sphere leaf test (mesh.py:259-262)
        double gg[3];
        for (int a = 0; a < 3; ++a) {
          double uu = xsub(lob[u][a], p[a]), v = xsub(p[a], hib[u][a]);
          v = v > 0.0 ? v : 0.0;
          gg[a] = uu > v ? uu : v;
        }
        if (!(edot3(gg, gg) <= r2)) continue;
        ++pairs;
        const double* cor = G.corners + 9 * t;
        double cl[3], off[3];
        closest_point(p, cor, cor + 3, cor + 6, cl);
        for (int a = 0; a < 3; ++a) off[a] = xsub(p[a], cl[a]);
        double eu = enorm3(off);
        double pg = edot3(G.normals + 3 * t, off);
        double sg = pg >= 0.0 ? eu : -eu;
        bool aligned = fabs(pg) >= xsub(xmul(0.9, eu), 1e-12);
        if (!(sg <= margin && eu <= radius && aligned)) continue;
        if (best_t < 0 || sg < best_s || (sg == best_s && t < best_t)) {
          best_t = t;
          best_s = sg;
          best_gap = pg;
          best_pp[0] = cl[0];
          best_pp[1] = cl[1];
          best_pp[2] = cl[2];
        }
      }
    }
    ws.ctri[k] = best_t;
    ws.cgap[k] = best_gap;
    ws.cpp[3 * k] = best_pp[0];
    ws.cpp[3 * k + 1] = best_pp[1];
    ws.cpp[3 * k + 2] = best_pp[2];
  }
  if (pairs_out) *pairs_out = team.isum(pairs);
  team.sync();
  // compaction in node order; contact c is stored at index c of the c* arrays
  // (written in place: contact index <= node index, chunks processed in order)
  int count = 0;
  for (int base = 0; base < N; base += team.size()) {
    int k = base + team.rank();
    bool has = k < N && ws.ctri[k] >= 0;
    int tri = has ? ws.ctri[k] : -1;
    double gap = has ? ws.cgap[k] : 0.0;
    double pp0 = has ? ws.cpp[3 * k] : 0.0, pp1 = has ? ws.cpp[3 * k + 1] : 0.0, pp2 = has ? ws.cpp[3 * k + 2] : 0.0;
    int total = 0;
    int pos = team.ballot_prefix(has, &total);
    team.sync();
    if (k < N) ws.crow_of_node[k] = has ? count + pos : -1;
    if (has) {
      int c = count + pos;
      ws.cnode[c] = k;
      ws.ctri[c] = tri;
      ws.cgap[c] = gap;
      ws.cpp[3 * c] = pp0;
      ws.cpp[3 * c + 1] = pp1;
      ws.cpp[3 * c + 2] = pp2;
      for (int a = 0; a < 3; ++a) ws.cnrm[3 * c + a] = -G.normals[3 * tri + a];
    }
    count += total;
    team.sync();
  }
  team.sync();
  return count;
}

}  // namespace accfem
