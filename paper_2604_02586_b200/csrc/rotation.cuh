// Rotation helpers of the regularisation stage (regularize.py:66-188), host+device.
//
// scipy.spatial.transform.Rotation semantics used by `propagate` (regularize.py:152, :172),
// restated from scipy 1.18's array-API backend (_rotation_xp.py: from_matrix :51-156,
// from_euler :192-226, as_matrix :302-333, as_euler :365-403 + _get_angles :1052-1111,
// compose_quat :1114-1127); the compiled backend the reference actually runs agrees with this
// restatement bit-for-bit on CPU (checked in tests/test_regularize_oracle.py), except that it
// uses libm hypot.  scipy quaternions are scalar-last (x, y, z, w); gausstrack's are (w, x, y, z).
//
// Numerics follow numpy: 3x3 @ 3x3 products are FMA chains (BLAS dgemm), everything else is
// plain rounded double ops in Python's evaluation order.
#pragma once

#include "common.cuh"
#include "smallsolve.cuh"

namespace ts {

// Numpy's 3x3 @ 3x3 (row-major): c[i][j] = fma(a[i][2], b[2][j], fma(a[i][1], b[1][j], a[i][0]*b[0][j])).
TS_HD void matmul3(const double *a, const double *b, double *c) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      c[3 * i + j] = fmaa(a[3 * i + 2], b[6 + j], fmaa(a[3 * i + 1], b[3 + j],
                                                      mul(a[3 * i], b[j])));
}

// a @ b^T
TS_HD void matmul3_bt(const double *a, const double *b, double *c) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      c[3 * i + j] = fmaa(a[3 * i + 2], b[3 * j + 2], fmaa(a[3 * i + 1], b[3 * j + 1],
                                                          mul(a[3 * i], b[3 * j])));
}

// _nearest_rotation (regularize.py:66-74): polar factor U V^T of m, flipped to det +1.
// One-sided Jacobi gives B = m V with columns s_j u_j.  The column of the smallest singular value
// is rebuilt as +-(u_a x u_b) with the sign that makes U V^T proper -- the same unique rotation
// LAPACK's "flip the last column of U" produces, and well defined even when m is singular.
TS_HD void nearest_rotation(const double *m, double *r) {
  double B[3][3], V[3][3], s[3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) B[i][j] = m[3 * i + j];
  jacobi_svd<3, true>(B, V, s);
  // order: a, b = two largest singular values, c = smallest (static indices throughout)
  const int c = (s[0] <= s[1] && s[0] <= s[2]) ? 0 : (s[1] <= s[2] ? 1 : 2);
  double ua[3], ub[3], va[3], vb[3], vc[3];
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const double b0 = B[i][0], b1 = B[i][1], b2 = B[i][2];
    const double v0 = V[i][0], v1 = V[i][1], v2 = V[i][2];
    if (c == 0) { ua[i] = b1 / s[1]; ub[i] = b2 / s[2]; va[i] = v1; vb[i] = v2; vc[i] = v0; }
    else if (c == 1) { ua[i] = b2 / s[2]; ub[i] = b0 / s[0]; va[i] = v2; vb[i] = v0; vc[i] = v1; }
    else { ua[i] = b0 / s[0]; ub[i] = b1 / s[1]; va[i] = v0; vb[i] = v1; vc[i] = v2; }
  }
  // (a, b, c) is a cyclic order, so vc = +-(va x vb) and uc must carry the same sign
  const double cx = va[1] * vb[2] - va[2] * vb[1];
  const double cy = va[2] * vb[0] - va[0] * vb[2];
  const double cz = va[0] * vb[1] - va[1] * vb[0];
  const double sg = (cx * vc[0] + cy * vc[1] + cz * vc[2]) < 0 ? -1.0 : 1.0;
  double uc[3] = {sg * (ua[1] * ub[2] - ua[2] * ub[1]), sg * (ua[2] * ub[0] - ua[0] * ub[2]),
                  sg * (ua[0] * ub[1] - ua[1] * ub[0])};
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) r[3 * i + j] = ua[i] * va[j] + ub[i] * vb[j] + uc[i] * vc[j];
}

// scipy _from_matrix_orthogonal: largest of (m00, m11, m22, trace), first index on ties
// (argmax); then normalise by the left-to-right 4-term norm.  q = (x, y, z, w).
TS_HD void sp_from_matrix_orthogonal(const double *m, double *q) {
  const double tr = add(add(m[0], m[4]), m[8]);
  int ch = 0;
  double best = m[0];
  if (m[4] > best) { ch = 1; best = m[4]; }
  if (m[8] > best) { ch = 2; best = m[8]; }
  if (tr > best) ch = 3;
  if (ch == 0) {
    q[0] = add(sub(1.0, tr), mul(2.0, m[0])); q[1] = add(m[3], m[1]);
    q[2] = add(m[6], m[2]); q[3] = sub(m[7], m[5]);
  } else if (ch == 1) {
    q[0] = add(m[3], m[1]); q[1] = add(sub(1.0, tr), mul(2.0, m[4]));
    q[2] = add(m[7], m[5]); q[3] = sub(m[2], m[6]);
  } else if (ch == 2) {
    q[0] = add(m[6], m[2]); q[1] = add(m[7], m[5]);
    q[2] = add(sub(1.0, tr), mul(2.0, m[8])); q[3] = sub(m[3], m[1]);
  } else {
    q[0] = sub(m[7], m[5]); q[1] = sub(m[2], m[6]); q[2] = sub(m[3], m[1]); q[3] = add(1.0, tr);
  }
  const double n = sqrt_rn(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])),
                               mul(q[3], q[3])));
#pragma unroll
  for (int i = 0; i < 4; i++) q[i] = dvd(q[i], n);
}

// Rotation.from_matrix: matrices whose Gram matrix is not within isclose(atol=1e-12, rtol=1e-5)
// of I are first projected with U V^T.  (The det <= 0 ValueError cannot arise for the products
// of rotations regularisation feeds in.)
TS_HD void sp_from_matrix(const double *m, double *q) {
  double g[9];
  matmul3_bt(m, m, g);
  bool ortho = true;
#pragma unroll
  for (int i = 0; i < 9; i++) {
    const double e = (i % 4 == 0) ? 1.0 : 0.0;
    ortho = ortho && fabs(g[i] - e) <= 1e-12 + 1e-5 * fabs(e);
  }
  if (ortho) {
    sp_from_matrix_orthogonal(m, q);
  } else {
    double r[9];
    nearest_rotation(m, r);
    sp_from_matrix_orthogonal(r, q);
  }
}

TS_HD double wrap_pi(double a) {
  const double pi = 3.141592653589793;
  if (a < -pi) return add(a, 2.0 * pi);
  if (a > pi) return sub(a, 2.0 * pi);
  return a;
}

// Rotation.as_euler("XYZ"): intrinsic X-Y-Z = extrinsic axes (2, 1, 0), sign = -1,
// lambda = pi/2; gimbal-lock cases at |theta2| <= 1e-7 or |theta2 - pi| <= 1e-7.
TS_HD void sp_as_euler_XYZ(const double *q, double *ang) {
  const double pi = 3.141592653589793;
  // i = 2, j = 1, k = 0, sign = -1
  const double a = sub(q[3], q[1]);
  const double b = sub(q[2], q[0]);          // q[i] + q[k] * sign
  const double c = add(q[1], q[3]);
  const double d = sub(-q[0], q[2]);         // q[k] * sign - q[i]
  const double half_sum = atan2(b, a), half_diff = atan2(d, c);
  const double th = mul(2.0, atan2(hypot(c, d), hypot(a, b)));
  const bool case1 = fabs(th) <= 1e-7;
  const bool case2 = fabs(sub(th, pi)) <= 1e-7;
  double first = 0.0, third = 0.0;  // intrinsic: angle_first -> index 2, angle_third -> index 0
  if (case1) third = mul(2.0, half_sum);
  else if (case2) third = mul(2.0, half_diff);
  if (!case1 && !case2) {
    first = sub(half_sum, half_diff);
    third = add(half_sum, half_diff);
  }
  third = -third;                    // * sign
  ang[0] = wrap_pi(third);
  ang[1] = wrap_pi(sub(th, pi / 2));
  ang[2] = wrap_pi(first);
}

// compose_quat(p, q), scalar-last
TS_HD void sp_compose(const double *p, const double *q, double *o) {
  const double cx = sub(mul(p[1], q[2]), mul(p[2], q[1]));
  const double cy = sub(mul(p[2], q[0]), mul(p[0], q[2]));
  const double cz = sub(mul(p[0], q[1]), mul(p[1], q[0]));
  o[0] = add(add(mul(p[3], q[0]), mul(q[3], p[0])), cx);
  o[1] = add(add(mul(p[3], q[1]), mul(q[3], p[1])), cy);
  o[2] = add(add(mul(p[3], q[2]), mul(q[3], p[2])), cz);
  o[3] = sub(sub(sub(mul(p[3], q[3]), mul(p[0], q[0])), mul(p[1], q[1])), mul(p[2], q[2]));
}

// Rotation.from_euler("XYZ", ang).as_matrix() -> row-major 3x3
TS_HD void sp_euler_XYZ_to_matrix(const double *ang, double *m) {
  double ex[4] = {sin(ang[0] / 2.0), 0.0, 0.0, cos(ang[0] / 2.0)};
  double ey[4] = {0.0, sin(ang[1] / 2.0), 0.0, cos(ang[1] / 2.0)};
  double ez[4] = {0.0, 0.0, sin(ang[2] / 2.0), cos(ang[2] / 2.0)};
  double t[4], q[4];
  sp_compose(ex, ey, t);
  sp_compose(t, ez, q);
  const double x = q[0], y = q[1], z = q[2], w = q[3];
  const double x2 = mul(x, x), y2 = mul(y, y), z2 = mul(z, z), w2 = mul(w, w);
  const double xy = mul(x, y), zw = mul(z, w), xz = mul(x, z), yw = mul(y, w);
  const double yz = mul(y, z), xw = mul(x, w);
  m[0] = add(sub(sub(x2, y2), z2), w2);
  m[1] = mul(2.0, sub(xy, zw));
  m[2] = mul(2.0, add(xz, yw));
  m[3] = mul(2.0, add(xy, zw));
  m[4] = add(sub(add(-x2, y2), z2), w2);
  m[5] = mul(2.0, sub(yz, xw));
  m[6] = mul(2.0, sub(xz, yw));
  m[7] = mul(2.0, add(yz, xw));
  m[8] = add(add(sub(-x2, y2), z2), w2);
}

}  // namespace ts
