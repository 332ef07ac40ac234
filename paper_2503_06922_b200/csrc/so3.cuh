// SO(3) maps with scipy.spatial.transform.Rotation semantics (scipy 1.18.1),
// restated from the published algorithm that the reference's so3.py:24-91
// calls: from_rotvec / as_matrix / from_matrix (Shepperd) / as_rotvec
// (canonical quaternion, small-angle series) / quaternion composition.
// Matrices are row-major 3x3 (m[3*r+c]); quaternions are (x, y, z, w).
#pragma once
#include "team.cuh"

namespace accfem {

DEV void quat_from_rotvec(const double* v, double* q) {
  double th = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  double s;
  if (th <= 1e-3) {
    double t2 = th * th;
    s = 0.5 - t2 / 48.0 + t2 * t2 / 3840.0;
  } else {
    s = sin(th / 2.0) / th;
  }
  q[0] = v[0] * s;
  q[1] = v[1] * s;
  q[2] = v[2] * s;
  q[3] = cos(th / 2.0);
}

DEV void quat_to_matrix(const double* q, double* m) {
  double x = q[0], y = q[1], z = q[2], w = q[3];
  double x2 = x * x, y2 = y * y, z2 = z * z, w2 = w * w;
  double xy = x * y, zw = z * w, xz = x * z, yw = y * w, yz = y * z, xw = x * w;
  m[0] = x2 - y2 - z2 + w2;
  m[1] = 2.0 * (xy - zw);
  m[2] = 2.0 * (xz + yw);
  m[3] = 2.0 * (xy + zw);
  m[4] = -x2 + y2 - z2 + w2;
  m[5] = 2.0 * (yz - xw);
  m[6] = 2.0 * (xz - yw);
  m[7] = 2.0 * (yz + xw);
  m[8] = -x2 - y2 + z2 + w2;
}

DEV void quat_normalize(double* q) {
  double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  q[0] /= n;
  q[1] /= n;
  q[2] /= n;
  q[3] /= n;
}

// Shepperd branch on argmax(m00, m11, m22, trace), first index wins ties
DEV void quat_from_matrix(const double* m, double* q) {
  double tr = m[0] + m[4] + m[8];
  int ch = 0;
  double best = m[0];
  if (m[4] > best) { best = m[4]; ch = 1; }
  if (m[8] > best) { best = m[8]; ch = 2; }
  if (tr > best) { ch = 3; }
  if (ch == 0) {
    q[0] = 1.0 - tr + 2.0 * m[0];
    q[1] = m[3] + m[1];
    q[2] = m[6] + m[2];
    q[3] = m[7] - m[5];
  } else if (ch == 1) {
    q[1] = 1.0 - tr + 2.0 * m[4];
    q[2] = m[7] + m[5];
    q[0] = m[1] + m[3];
    q[3] = m[2] - m[6];
  } else if (ch == 2) {
    q[2] = 1.0 - tr + 2.0 * m[8];
    q[0] = m[2] + m[6];
    q[1] = m[5] + m[7];
    q[3] = m[3] - m[1];
  } else {
    q[0] = m[7] - m[5];
    q[1] = m[2] - m[6];
    q[2] = m[3] - m[1];
    q[3] = 1.0 + tr;
  }
  quat_normalize(q);
}

DEV void quat_to_rotvec(const double* qin, double* v) {
  double q[4] = {qin[0], qin[1], qin[2], qin[3]};
  bool neg = q[3] < 0.0;
  if (q[3] == 0.0) {
    if (q[0] < 0.0) neg = true;
    else if (q[0] == 0.0) {
      if (q[1] < 0.0) neg = true;
      else if (q[1] == 0.0 && q[2] < 0.0) neg = true;
    }
  }
  if (neg) { q[0] = -q[0]; q[1] = -q[1]; q[2] = -q[2]; q[3] = -q[3]; }
  double axn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
  double ang = 2.0 * atan2(axn, q[3]);
  double s;
  if (ang <= 1e-3) {
    double a2 = ang * ang;
    s = 2.0 + a2 / 12.0 + 7.0 * a2 * a2 / 2880.0;
  } else {
    s = ang / sin(ang / 2.0);
  }
  v[0] = s * q[0];
  v[1] = s * q[1];
  v[2] = s * q[2];
}

DEV void rot_exp(const double* v, double* m) {
  double q[4];
  quat_from_rotvec(v, q);
  quat_to_matrix(q, m);
}

DEV void rot_log(const double* m, double* v) {
  double q[4];
  quat_from_matrix(m, q);
  quat_to_rotvec(q, v);
}

// rotvec of exp(inc) * exp(base): quaternion product, normalised (so3.py:40-46)
DEV void rot_compose(const double* inc, const double* base, double* out) {
  double p[4], r[4], q[4];
  quat_from_rotvec(inc, p);
  quat_from_rotvec(base, r);
  double cx = p[1] * r[2] - p[2] * r[1];
  double cy = p[2] * r[0] - p[0] * r[2];
  double cz = p[0] * r[1] - p[1] * r[0];
  q[0] = p[3] * r[0] + r[3] * p[0] + cx;
  q[1] = p[3] * r[1] + r[3] * p[1] + cy;
  q[2] = p[3] * r[2] + r[3] * p[2] + cz;
  q[3] = p[3] * r[3] - p[0] * r[0] - p[1] * r[1] - p[2] * r[2];
  quat_normalize(q);
  quat_to_rotvec(q, out);
}

// c = a * b
DEV void mat3_mul(const double* a, const double* b, double* c) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      c[3 * r + k] = a[3 * r] * b[k] + a[3 * r + 1] * b[3 + k] + a[3 * r + 2] * b[6 + k];
}
// c = a^T * b
DEV void mat3_tmul(const double* a, const double* b, double* c) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      c[3 * r + k] = a[r] * b[k] + a[3 + r] * b[3 + k] + a[6 + r] * b[6 + k];
}
// y = a * x
DEV void mat3_vec(const double* a, const double* x, double* y) {
#pragma unroll
  for (int r = 0; r < 3; ++r) y[r] = a[3 * r] * x[0] + a[3 * r + 1] * x[1] + a[3 * r + 2] * x[2];
}

// minimal rotation taking unit a onto unit b (so3.py:49-82)
DEV void rot_between(const double* a, const double* b, double* m) {
  double ax[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
  double s = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
  double c = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
  if (s > 1e-12) {
    double ang = atan2(s, c);
    double v[3] = {ax[0] / s * ang, ax[1] / s * ang, ax[2] / s * ang};
    rot_exp(v, m);
  } else if (c > 0.0) {
    for (int i = 0; i < 9; ++i) m[i] = (i % 4 == 0) ? 1.0 : 0.0;
  } else {
    double ref[3] = {1.0, 0.0, 0.0};
    if (!(fabs(a[0]) < 0.9)) { ref[0] = 0.0; ref[1] = 1.0; }
    double w[3] = {a[1] * ref[2] - a[2] * ref[1], a[2] * ref[0] - a[0] * ref[2], a[0] * ref[1] - a[1] * ref[0]};
    double n = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    const double pi = 3.141592653589793;
    double v[3] = {w[0] / n * pi, w[1] / n * pi, w[2] / n * pi};
    rot_exp(v, m);
  }
}

// geodesic midpoint ra * exp(0.5 log(ra^T rb)) (so3.py:85-91)
DEV void rot_mid(const double* ra, const double* rb, double* out) {
  double rel[9], v[3], h[9];
  mat3_tmul(ra, rb, rel);
  rot_log(rel, v);
  v[0] *= 0.5;
  v[1] *= 0.5;
  v[2] *= 0.5;
  rot_exp(v, h);
  mat3_mul(ra, h, out);
}

}  // namespace accfem
