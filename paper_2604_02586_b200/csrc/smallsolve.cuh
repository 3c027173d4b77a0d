// smallsolve.cuh -- register-resident small dense solvers of K4 (host+device).
//
// Streaming Givens QR, one-sided Jacobi SVD, cyclic Jacobi 3x3 eigen-decomposition and the
// reference's discrete post-processing (multiview.py:103-135, core.py:41-62).  TS_HD so the same
// code is unit-tested on the CPU (tests/native) and runs inside K4 on the GPU.
#pragma once

#include <float.h>

#include "common.cuh"
#include "motion.cuh"

namespace ts {

// tri-state result of the fuse's solve steps: the slow (SVD) decision can be deferred to a second
// kernel so that the rare near-degenerate Gaussians do not stall whole warps of K4
#define TS_FUSE_FAIL 0
#define TS_FUSE_OK 1
#define TS_FUSE_DEFER 2

template <int N>
TS_HD void qr_add_row(double (&R)[N][N], double (&row)[N]) {
#pragma unroll
  for (int k = 0; k < N; k++) {
    const double bb = row[k];
    if (bb == 0.0) continue;
    const double a = R[k][k];
    const double rr = fma(a, a, bb * bb);
    const double inv = rsqrt(rr);
    const double c = a * inv, s = bb * inv;
    R[k][k] = rr * inv;
#pragma unroll
    for (int j = k + 1; j < N; j++) {
      const double t = R[k][j];
      R[k][j] = c * t + s * row[j];
      row[j] = c * row[j] - s * t;
    }
  }
}

template <int N>
TS_HD void qr_add_row_rhs(double (&R)[N][N], double (&c6)[N],
                                               double (&row)[N], double rhs) {
#pragma unroll
  for (int k = 0; k < N; k++) {
    const double bb = row[k];
    if (bb == 0.0) continue;
    const double a = R[k][k];
    const double rr = fma(a, a, bb * bb);
    const double inv = rsqrt(rr);
    const double c = a * inv, s = bb * inv;
    R[k][k] = rr * inv;
#pragma unroll
    for (int j = k + 1; j < N; j++) {
      const double t = R[k][j];
      R[k][j] = c * t + s * row[j];
      row[j] = c * row[j] - s * t;
    }
    const double t = c6[k];
    c6[k] = c * t + s * rhs;
    rhs = c * rhs - s * t;
  }
}

// One-sided Jacobi SVD of the N x N matrix B (orthogonalises columns).  On return the column
// norms of B are the singular values; V (if WANT_V) holds the right singular vectors.
template <int N, bool WANT_V>
TS_HD void jacobi_svd(double (&B)[N][N], double (&V)[N][N], double (&s)[N]) {
  if (WANT_V) {
#pragma unroll
    for (int i = 0; i < N; i++)
#pragma unroll
      for (int j = 0; j < N; j++) V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  for (int sweep = 0; sweep < 40; sweep++) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < N - 1; p++) {
#pragma unroll
      for (int q = p + 1; q < N; q++) {
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int i = 0; i < N; i++) {
          al = fma(B[i][p], B[i][p], al);
          be = fma(B[i][q], B[i][q], be);
          ga = fma(B[i][p], B[i][q], ga);
        }
        if (ga == 0.0 || fabs(ga) <= DBL_EPSILON * sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = rsqrt(fma(t, t, 1.0));
        const double sn = c * t;
#pragma unroll
        for (int i = 0; i < N; i++) {
          const double bp = B[i][p], bq = B[i][q];
          B[i][p] = c * bp - sn * bq;
          B[i][q] = sn * bp + c * bq;
        }
        if (WANT_V) {
#pragma unroll
          for (int i = 0; i < N; i++) {
            const double vp = V[i][p], vq = V[i][q];
            V[i][p] = c * vp - sn * vq;
            V[i][q] = sn * vp + c * vq;
          }
        }
      }
    }
    if (!rotated) break;
  }
#pragma unroll
  for (int j = 0; j < N; j++) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < N; i++) acc = fma(B[i][j], B[i][j], acc);
    s[j] = sqrt(acc);
  }
}

// Right singular vector of the smallest singular value of an upper-triangular 4x4 R by inverse
// iteration on R^T R (two triangular solves per step, error ratio (s3/s2)^2 per step), started from
// R^-1 e3.  Returns false (caller falls back to the Jacobi SVD) on a zero pivot or if 12 steps do
// not converge to 4 ulp.
TS_HD bool null_vector_r4(const double (&R)[4][4], double (&x)[4]) {
  if (!(R[0][0] != 0.0 && R[1][1] != 0.0 && R[2][2] != 0.0 && R[3][3] != 0.0)) return false;
  double y[4];
  y[3] = 1.0 / R[3][3];
  y[2] = -(R[2][3] * y[3]) / R[2][2];
  y[1] = -(R[1][2] * y[2] + R[1][3] * y[3]) / R[1][1];
  y[0] = -(R[0][1] * y[1] + R[0][2] * y[2] + R[0][3] * y[3]) / R[0][0];
  double inv = rsqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2] + y[3] * y[3]);
#pragma unroll
  for (int i = 0; i < 4; i++) x[i] = y[i] * inv;
  for (int it = 0; it < 12; it++) {
    double z[4];  // R^T z = x (forward), then R y = z (back)
    z[0] = x[0] / R[0][0];
    z[1] = (x[1] - R[0][1] * z[0]) / R[1][1];
    z[2] = (x[2] - R[0][2] * z[0] - R[1][2] * z[1]) / R[2][2];
    z[3] = (x[3] - R[0][3] * z[0] - R[1][3] * z[1] - R[2][3] * z[2]) / R[3][3];
    y[3] = z[3] / R[3][3];
    y[2] = (z[2] - R[2][3] * y[3]) / R[2][2];
    y[1] = (z[1] - R[1][2] * y[2] - R[1][3] * y[3]) / R[1][1];
    y[0] = (z[0] - R[0][1] * y[1] - R[0][2] * y[2] - R[0][3] * y[3]) / R[0][0];
    const double nn = y[0] * y[0] + y[1] * y[1] + y[2] * y[2] + y[3] * y[3];
    if (!(nn > 0.0 && nn < 1e300)) return false;
    inv = rsqrt(nn);
    if (y[0] * x[0] + y[1] * x[1] + y[2] * x[2] + y[3] * x[3] < 0) inv = -inv;
    double diff = 0.0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const double v = y[i] * inv;
      diff = fmax(diff, fabs(v - x[i]));
      x[i] = v;
    }
    if (diff <= 4.5e-16) return true;
  }
  return false;
}

// Certificate for the reference's gap test s[-2] - s[-1] > 1e-9 s[0] (multiview.py:251) given an
// approximate null vector x (unit) of R: s[-1] <= |R x| (+ rounding), s[0] <= |R|_F, and s[-2] >=
// sigma_min(R restricted to x-perp) >= 1/|R'^-1|_F, R' the 3x3 R factor of R H[:, 0:3] with H
// the Householder reflector taking x to the last axis (Cauchy interlacing).  true => the test
// passes for certain; false => undecided (run the SVD).
TS_HD bool gap_certified(const double (&R)[4][4], const double (&x)[4]) {
  double nf2 = 0.0, rx2 = 0.0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    double rxi = 0.0;
#pragma unroll
    for (int j = i; j < 4; j++) {
      nf2 = fma(R[i][j], R[i][j], nf2);
      rxi = fma(R[i][j], x[j], rxi);
    }
    rx2 = fma(rxi, rxi, rx2);
  }
  const double nf = sqrt(nf2);
  const double s3u = sqrt(rx2) + 8e-16 * nf;
  // w = x + sign(x3) e3; H = I - 2 w w^T / (w^T w); columns 0..2 of R H span R (x-perp)
  const double sg = x[3] < 0 ? -1.0 : 1.0;
  const double w[4] = {x[0], x[1], x[2], x[3] + sg};
  const double ww = w[0] * w[0] + w[1] * w[1] + w[2] * w[2] + w[3] * w[3];
  double Rp[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int i = 0; i < 4; i++) {
    double rw = 0.0;
#pragma unroll
    for (int j = i; j < 4; j++) rw = fma(R[i][j], w[j], rw);
    const double f = 2.0 * rw / ww;
    double row[3];
#pragma unroll
    for (int j = 0; j < 3; j++) row[j] = ((j >= i) ? R[i][j] : 0.0) - f * w[j];
    qr_add_row<3>(Rp, row);
  }
  if (!(Rp[0][0] != 0.0 && Rp[1][1] != 0.0 && Rp[2][2] != 0.0)) return false;
  // |R'^-1|_F^2 by back substitution on the three unit vectors
  const double i00 = 1.0 / Rp[0][0], i11 = 1.0 / Rp[1][1], i22 = 1.0 / Rp[2][2];
  const double i01 = -Rp[0][1] * i11 * i00;
  const double i12 = -Rp[1][2] * i22 * i11;
  const double i02 = -(Rp[0][1] * i12 + Rp[0][2] * i22) * i00;
  const double inv2 = i00 * i00 + i11 * i11 + i22 * i22 + i01 * i01 + i12 * i12 + i02 * i02;
  const double lb = rsqrt(inv2) * (1.0 - 1e-12);
  return lb - s3u > TS_SINGULAR_GAP_REL * nf * (1.0 + 1e-12);
}

// triangulate_mean from the R factor of the stacked DLT rows (multiview.py:249-257).  Fast path:
// inverse-iteration null vector + a rigorous certificate for the singular-gap test; the one-sided
// Jacobi SVD (below) decides only when the certificate cannot (near-degenerate geometry).
TS_HD int triangulate_from_r(const double (&R)[4][4], double *mean, bool allow_slow = true) {
  {
    double x[4];
    if (null_vector_r4(R, x) && gap_certified(R, x)) {
      // x is unit: the solution-at-infinity test (:255) is |x3| > 1e-9
      if (!(fabs(x[3]) > TS_SINGULAR_GAP_REL)) return TS_FUSE_FAIL;
      mean[0] = x[0] / x[3];
      mean[1] = x[1] / x[3];
      mean[2] = x[2] / x[3];
      return TS_FUSE_OK;
    }
  }
  if (!allow_slow) return TS_FUSE_DEFER;
  double B[4][4], V[4][4], s[4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) B[i][j] = (j >= i) ? R[i][j] : 0.0;
  jacobi_svd<4, true>(B, V, s);
  // order singular values descending (static-index bubble sort: registers only)
  double v[4] = {s[0], s[1], s[2], s[3]};
  int id[4] = {0, 1, 2, 3};
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3 - i; j++)
      if (v[j] < v[j + 1]) {
        const double tv = v[j];
        v[j] = v[j + 1];
        v[j + 1] = tv;
        const int ti = id[j];
        id[j] = id[j + 1];
        id[j + 1] = ti;
      }
  const double s0 = v[0], s2 = v[2], s3 = v[3];
  const int imin = id[3];
  if (!(s2 - s3 > TS_SINGULAR_GAP_REL * s0)) return TS_FUSE_FAIL;
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    x[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (j == imin) x[i] = V[i][j];
  }
  const double nrm = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3]);
  if (!(fabs(x[3]) > TS_SINGULAR_GAP_REL * nrm)) return TS_FUSE_FAIL;
  mean[0] = x[0] / x[3];
  mean[1] = x[1] / x[3];
  mean[2] = x[2] / x[3];
  return TS_FUSE_OK;
}

// solve_covariance3d from R (6x6) and Q^T b (multiview.py:259-263).
TS_HD int cov_from_r(const double (&R)[6][6], const double (&c6)[6], double *sol,
                     bool allow_slow = true) {
  // Rigorous cheap bound first: s_max <= |R|_F and s_min >= 1/|R^-1|_F, so
  // 1/(|R|_F |R^-1|_F) >= 1e-9 proves the reference's rank test passes; only otherwise run the
  // one-sided Jacobi SVD to take the exact decision.
  bool need_svd = false;
  {
    double fro = 0.0, finv = 0.0;
    double Ri[6][6];
#pragma unroll
    for (int i = 0; i < 6; i++)
#pragma unroll
      for (int j = i; j < 6; j++) fro = fma(R[i][j], R[i][j], fro);
#pragma unroll
    for (int i = 0; i < 6; i++) need_svd = need_svd || !(R[i][i] != 0.0);
    if (!need_svd) {
      // column j of R^-1 by back substitution on e_j
#pragma unroll
      for (int j = 0; j < 6; j++) {
#pragma unroll
        for (int i = 5; i >= 0; i--) {
          double acc = (i == j) ? 1.0 : 0.0;
#pragma unroll
          for (int k = i + 1; k < 6; k++) acc -= R[i][k] * Ri[k][j];
          Ri[i][j] = (i <= j) ? acc / R[i][i] : 0.0;
          finv = fma(Ri[i][j], Ri[i][j], finv);
        }
      }
      need_svd = !(1.0 >= 1.0000001 * TS_SINGULAR_GAP_REL * sqrt(fro * finv));
    }
  }
  if (need_svd) {
    // Rigorous "certainly rank deficient" test: for triangular R, s_min <= min_i |R_ii| (the
    // diagonal holds the eigenvalues) and s_max >= every row norm.  Stacked systems that are
    // truly singular (s_min/s_max ~ 1e-16, all the undecided cases seen in practice) fail here
    // without an SVD.
    double dmin = fabs(R[0][0]), rmax = 0.0;
#pragma unroll
    for (int i = 0; i < 6; i++) {
      dmin = fmin(dmin, fabs(R[i][i]));
      double r2 = 0.0;
#pragma unroll
      for (int j = i; j < 6; j++) r2 = fma(R[i][j], R[i][j], r2);
      rmax = fmax(rmax, sqrt(r2));
    }
    if (dmin < TS_SINGULAR_GAP_REL * rmax * (1.0 - 1e-12)) return TS_FUSE_FAIL;
  }
  if (need_svd && !allow_slow) return TS_FUSE_DEFER;
  if (need_svd) {
    double B[6][6], s[6];
    double Vd[6][6];
#pragma unroll
    for (int i = 0; i < 6; i++)
#pragma unroll
      for (int j = 0; j < 6; j++) B[i][j] = (j >= i) ? R[i][j] : 0.0;
    jacobi_svd<6, false>(B, Vd, s);
    double smax = s[0], smin = s[0];
#pragma unroll
    for (int j = 1; j < 6; j++) {
      smax = fmax(smax, s[j]);
      smin = fmin(smin, s[j]);
    }
    if (!(smin >= TS_SINGULAR_GAP_REL * smax)) return TS_FUSE_FAIL;
  }
#pragma unroll
  for (int i = 5; i >= 0; i--) {
    double acc = c6[i];
#pragma unroll
    for (int k = i + 1; k < 6; k++) acc -= R[i][k] * sol[k];
    sol[i] = acc / R[i][i];
  }
  return TS_FUSE_OK;
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3; eigenvalues ascending (as eigh).
TS_HD void eigh3(double (&A)[3][3], double (&E)[3][3], double (&ev)[3]) {
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) E[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 50; sweep++) {
    const double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    if (off == 0.0) break;
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < 2; p++) {
#pragma unroll
      for (int q = p + 1; q < 3; q++) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double app = A[p][p], aqq = A[q][q];
        if (fabs(apq) <= 0.5 * DBL_EPSILON * sqrt(fabs(app * aqq)) && fabs(apq) < 1e-300 + 0.5 * DBL_EPSILON * (fabs(app) + fabs(aqq))) {
          A[p][q] = A[q][p] = 0.0;
          continue;
        }
        rotated = true;
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
        const double c = rsqrt(fma(t, t, 1.0));
        const double s = t * c;
        const int r = 3 - p - q;  // the third index
        const double arp = A[r][p], arq = A[r][q];
        A[p][p] = app - t * apq;
        A[q][q] = aqq + t * apq;
        A[p][q] = A[q][p] = 0.0;
        A[r][p] = A[p][r] = c * arp - s * arq;
        A[r][q] = A[q][r] = s * arp + c * arq;
#pragma unroll
        for (int i = 0; i < 3; i++) {
          const double ep = E[i][p], eq = E[i][q];
          E[i][p] = c * ep - s * eq;
          E[i][q] = s * ep + c * eq;
        }
      }
    }
    if (!rotated) break;
  }
  ev[0] = A[0][0];
  ev[1] = A[1][1];
  ev[2] = A[2][2];
  // sort ascending with eigenvectors
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2 - i; j++)
      if (ev[j] > ev[j + 1]) {
        double t = ev[j];
        ev[j] = ev[j + 1];
        ev[j + 1] = t;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          double u = E[k][j];
          E[k][j] = E[k][j + 1];
          E[k][j + 1] = u;
        }
      }
}

TS_HD double dot4_norm(const double *q) {
  return sqrt(fma(q[3], q[3], fma(q[2], q[2], fma(q[1], q[1], q[0] * q[0]))));
}

// core.py:41-62
// Largest-diagonal branch of matrix_to_quat with compile-time indices (no dynamic indexing of
// local arrays: all state stays in registers).
template <int I>
TS_HD void matrix_to_quat_branch(const double (&m)[3][3], double *q) {
  constexpr int J = (I + 1) % 3, K = (I + 2) % 3;
  const double s = sqrt(fmax(m[I][I] - m[J][J] - m[K][K] + 1.0, 0.0)) * 2;
  q[0] = (m[K][J] - m[J][K]) / s;
  q[1 + I] = 0.25 * s;
  q[1 + J] = (m[J][I] + m[I][J]) / s;
  q[1 + K] = (m[K][I] + m[I][K]) / s;
}

TS_HD bool matrix_to_quat(const double (&m)[3][3], double *q) {
  const double t = (m[0][0] + m[1][1]) + m[2][2];
  if (t > 0) {
    const double s = sqrt(t + 1.0) * 2;
    q[0] = 0.25 * s;
    q[1] = (m[2][1] - m[1][2]) / s;
    q[2] = (m[0][2] - m[2][0]) / s;
    q[3] = (m[1][0] - m[0][1]) / s;
  } else if (!(m[1][1] > m[0][0]) && !(m[2][2] > m[0][0])) {  // i = argmax diag = 0
    matrix_to_quat_branch<0>(m, q);
  } else if (!(m[2][2] > m[1][1])) {  // i = 1
    matrix_to_quat_branch<1>(m, q);
  } else {  // i = 2
    matrix_to_quat_branch<2>(m, q);
  }
  if (q[0] < 0) {
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] = -q[i];
  }
  const double nrm = dot4_norm(q);
  if (!(nrm != 0.0 && isfinite(nrm))) return false;  // quat_normalize raises ValueError
#pragma unroll
  for (int i = 0; i < 4; i++) q[i] /= nrm;
  return true;
}

// decompose_covariance (multiview.py:103-135) on a symmetrised 3x3.
TS_HD bool decompose(double (&m)[3][3], const double *ref_q, double eig_floor,
                     double *q_out, double *s_out, double *dbg = nullptr) {
  double E[3][3], ev[3];
  const double tr = (m[0][0] + m[1][1]) + m[2][2];
  eigh3(m, E, ev);
  if (dbg) {
    for (int i = 0; i < 9; i++) dbg[i] = E[i / 3][i % 3];
    for (int i = 0; i < 3; i++) dbg[9 + i] = ev[i];
    for (int i = 0; i < 4; i++) dbg[12 + i] = ref_q[i];
  }
  const double floor_ = eig_floor * fabs(tr);
  if (ev[0] < floor_ || ev[1] < floor_ || ev[2] < floor_) return false;
  double qn[4] = {ref_q[0], ref_q[1], ref_q[2], ref_q[3]};
  const double nrm = dot4_norm(qn);
  if (!(nrm != 0.0 && isfinite(nrm))) return false;
#pragma unroll
  for (int i = 0; i < 4; i++) qn[i] /= nrm;
  double ref[9];
  quat_to_matrix(qn[0], qn[1], qn[2], qn[3], ref);
  double dots[3][3];
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int e = 0; e < 3; e++)
      dots[k][e] = fabs(fma(ref[6 + k], E[2][e], fma(ref[3 + k], E[1][e], ref[k] * E[0][e])));
  // itertools.permutations(range(3)) order; first maximum wins (multiview.py:123-124)
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  int best = 0;
  double best_score = -1.0;
#pragma unroll
  for (int p = 0; p < 6; p++) {
    const double sc = (dots[0][perms[p][0]] + dots[1][perms[p][1]]) + dots[2][perms[p][2]];
    if (sc > best_score) {
      best_score = sc;
      best = p;
    }
  }
  double r[3][3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    int e = 0;
#pragma unroll
    for (int p = 0; p < 6; p++)
      if (p == best) e = perms[p][k];
    double col[3], evk = 0.0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      col[i] = 0.0;
#pragma unroll
      for (int jj = 0; jj < 3; jj++)
        if (jj == e) col[i] = E[i][jj];
    }
#pragma unroll
    for (int jj = 0; jj < 3; jj++)
      if (jj == e) evk = ev[jj];
    const double d = fma(col[2], ref[6 + k], fma(col[1], ref[3 + k], col[0] * ref[k]));
    const double sg = d < 0 ? -1.0 : 1.0;
#pragma unroll
    for (int i = 0; i < 3; i++) r[i][k] = sg * col[i];
    s_out[k] = sqrt(evk);
  }
  const double det = r[0][0] * (r[1][1] * r[2][2] - r[1][2] * r[2][1]) -
                     r[0][1] * (r[1][0] * r[2][2] - r[1][2] * r[2][0]) +
                     r[0][2] * (r[1][0] * r[2][1] - r[1][1] * r[2][0]);
  if (det < 0) {
#pragma unroll
    for (int i = 0; i < 3; i++) r[i][2] = -r[i][2];
  }
  if (dbg) {
    for (int i = 0; i < 9; i++) dbg[26 + i] = r[i / 3][i % 3];
    dbg[35] = best;
    for (int i = 0; i < 9; i++) dbg[36 + i] = dots[i / 3][i % 3];
    for (int i = 0; i < 9; i++) dbg[45 + i] = ref[i];
  }
  return matrix_to_quat(r, q_out);
}

// multiview.py:159-165
TS_HD bool min_eig_ok(double c00, double c01, double c10, double c11) {
  const double tr = c00 + c11;
  const double det = c00 * c11 - c01 * c10;
  const double me = 0.5 * (tr - sqrt(fmax(tr * tr - 4 * det, 0.0)));
  return me >= -1e-9 * fmax(tr, 0.0);
}

// Solve steps of update_all for one Gaussian from its accumulated R factors (multiview.py:249-274):
// triangulation, covariance least squares, decomposition.  Returns TS_STATUS_SOLVED /
// TS_STATUS_UNSOLVABLE after writing the outputs, or TS_FUSE_DEFER_STATUS (outputs untouched) when
// !allow_slow and a decision needs an SVD.
#define TS_FUSE_DEFER_STATUS 3
TS_HD int fuse_finish(const double *gs, const double (&R4)[4][4], const double (&R6)[6][6],
                      const double (&c6)[6], const ts_config &cfg, double *delta, double *q,
                      double *sc, bool allow_slow, double *dbg = nullptr) {
  double mean[3], sol[6], qo[4], so[3];
  int r = triangulate_from_r(R4, mean, allow_slow);
  if (r == TS_FUSE_OK) r = cov_from_r(R6, c6, sol, allow_slow);
  if (r == TS_FUSE_DEFER) return TS_FUSE_DEFER_STATUS;
  bool ok = r == TS_FUSE_OK;
  if (ok) {
    double S[3][3] = {{sol[0], sol[1], sol[2]}, {sol[1], sol[3], sol[4]}, {sol[2], sol[4], sol[5]}};
    if (dbg)
      for (int i = 0; i < 6; i++) dbg[16 + i] = sol[i];
    ok = decompose(S, gs + 3, cfg.eig_floor, qo, so, dbg);
  }
  ok = ok && isfinite(mean[0]) && isfinite(mean[1]) && isfinite(mean[2]) && so[0] > 0 &&
       so[1] > 0 && so[2] > 0;
  if (!ok) return TS_STATUS_UNSOLVABLE;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    delta[i] = mean[i] - gs[i];
    sc[i] = so[i];
  }
#pragma unroll
  for (int i = 0; i < 4; i++) q[i] = qo[i];
  return TS_STATUS_SOLVED;
}

// The per-view motion records K4 reads: the dense SoA arrays (ts_motions), or dense statuses plus
// K3's compact list-order fits found through the gv's rank (K4Motions with fits != NULL: K3 kept
// its fits compact, so the dense a / b / sums were never written; only SOLVED gvs are read, and
// every SOLVED gv is in the touched list).
struct K4Motions {
  ts_motions m;
  const GvMotion *fits;
  const uint32_t *rank;
};
TS_HD int8_t mot_status(const ts_motions &m, int64_t gv) { return m.status[gv]; }
TS_HD int8_t mot_status(const K4Motions &k, int64_t gv) { return k.m.status[gv]; }
TS_HD void mot_sums(const ts_motions &m, int64_t gv, double &w, int64_t &c) {
  w = m.weight_sum[gv];
  c = m.pixel_count[gv];
}
TS_HD void mot_sums(const K4Motions &k, int64_t gv, double &w, int64_t &c) {
  if (!k.fits) return mot_sums(k.m, gv, w, c);
  const GvMotion &f = k.fits[k.rank[gv]];
  w = f.wsum;
  c = f.count;
}
TS_HD void mot_affine(const ts_motions &m, int64_t gv, double (&A)[4], double (&b)[2]) {
#pragma unroll
  for (int i = 0; i < 4; i++) A[i] = m.a[4 * gv + i];
  b[0] = m.b[2 * gv];
  b[1] = m.b[2 * gv + 1];
}
TS_HD void mot_affine(const K4Motions &k, int64_t gv, double (&A)[4], double (&b)[2]) {
  if (!k.fits) return mot_affine(k.m, gv, A, b);
  const GvMotion &f = k.fits[k.rank[gv]];
#pragma unroll
  for (int i = 0; i < 4; i++) A[i] = f.a[i];
  b[0] = f.b[0];
  b[1] = f.b[1];
}

// update_all for one Gaussian (multiview.py:181-274).  Reads the V per-view motion records of
// Gaussian g (stride n between views) and writes its update; returns the status.
// With allow_slow == false the SVD-deciding Gaussians return TS_FUSE_DEFER_STATUS and leave their
// R factors in R4 / R6 / c6 for fuse_finish in the deferred pass.
// `eligible_mask` != 0: the caller already applied the eligibility rule and passes the SOLVED-view
// bits (k4_prep), so the per-view status / weight / count reads are not repeated.
template <typename Motions>
TS_HD int fuse_gaussian(const double *gs, int64_t g, int64_t n, const ts_camera *cams, int V,
                        const Motions &m, const ts_config &cfg, double *delta, double *q,
                        double *sc, double (&R4)[4][4], double (&R6)[6][6], double (&c6)[6],
                        bool allow_slow, double *dbg = nullptr, uint64_t eligible_mask = 0) {
  double c3[9];
  covariance3d(gs, c3);
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) R4[i][j] = 0.0;
#pragma unroll
  for (int i = 0; i < 6; i++) {
    c6[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 6; j++) R6[i][j] = 0.0;
  }
  // eligibility pre-pass (multiview.py:231-235): cheap loads only, so Gaussians with too few
  // solved views never touch the heavy math
#pragma unroll
  for (int i = 0; i < 3; i++) {
    delta[i] = 0.0;
    sc[i] = gs[7 + i];
  }
#pragma unroll
  for (int i = 0; i < 4; i++) q[i] = gs[3 + i];
  // bit v: view v SOLVED.  With more than 64 views the bits are rebuilt per 64-view word below
  // and a nonzero eligible_mask only says "eligible".
  uint64_t solved = eligible_mask;
  if (!solved) {
    int n_solved = 0;
    double tw = 0.0;
    int64_t tp = 0;
    for (int v = 0; v < V; v++) {
      const int64_t gv = (int64_t)v * n + g;
      if (mot_status(m, gv) != TS_STATUS_SOLVED) continue;
      if (v < 64) solved |= 1ull << v;
      n_solved++;
      double w;
      int64_t c;
      mot_sums(m, gv, w, c);
      tw += w;
      tp += c;
    }
    if (!(n_solved >= cfg.min_views && tw >= cfg.min_total_weight &&
          tp >= cfg.min_total_pixels))
      return TS_STATUS_UNSOLVABLE;
  }
  bool bad = false;
  // iterate the solved views only, in view order: Gaussians with equal solved-view counts (k4_fuse
  // groups them) then run the heavy body in lockstep
  for (int base = 0; base < V && !bad; base += 64) {
   if (V > 64) {
    solved = 0;
    const int top = V - base < 64 ? V - base : 64;
    for (int j = 0; j < top; j++)
      if (mot_status(m, (int64_t)(base + j) * n + g) == TS_STATUS_SOLVED) solved |= 1ull << j;
   }
   while (solved && !bad) {
    const int v = base + ffs64_hd(solved) - 1;
    solved &= solved - 1;
    const int64_t gv = (int64_t)v * n + g;
    const ts_camera &cam = cams[v];
    Projection p;
    project(gs, c3, cam, p);
    double Av[4], bv[2];
    mot_affine(m, gv, Av, bv);
    const double A00 = Av[0], A01 = Av[1], A10 = Av[2], A11 = Av[3];
    const double b0 = bv[0], b1 = bv[1];
    // Eq. 2: moved mean / covariance (multiview.py:218-220)
    const double mm0 = (A00 * p.mean2[0] + A01 * p.mean2[1]) + b0;
    const double mm1 = (A10 * p.mean2[0] + A11 * p.mean2[1]) + b1;
    const double c00 = p.cov2[0], c01 = p.cov2[1], c11 = p.cov2[2];
    const double t00 = fma(A01, c01, A00 * c00), t01 = fma(A01, c11, A00 * c01);
    const double t10 = fma(A11, c01, A10 * c00), t11 = fma(A11, c11, A10 * c01);
    const double q00 = fma(t01, A01, t00 * A00), q01 = fma(t01, A11, t00 * A10);
    const double q10 = fma(t11, A01, t10 * A00), q11 = fma(t11, A11, t10 * A10);
    const double mc00 = 0.5 * (q00 + q00), mc01 = 0.5 * (q01 + q10), mc11 = 0.5 * (q11 + q11);
    if (!(p.in_front && min_eig_ok(c00, c01, c01, c11) && min_eig_ok(mc00, mc01, mc01, mc11))) {
      bad = true;  // a solved view that fails projection/PSD aborts the fuse (:236-237)
      continue;
    }
    // P = K [R | t]  (core.py:145-148)
    double P[3][4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const double r0 = j < 3 ? cam.R[j] : cam.t[0];
      const double r1 = j < 3 ? cam.R[3 + j] : cam.t[1];
      const double r2 = j < 3 ? cam.R[6 + j] : cam.t[2];
      P[0][j] = dot3(cam.fx, 0.0, cam.cx, r0, r1, r2);
      P[1][j] = dot3(0.0, cam.fy, cam.cy, r0, r1, r2);
      P[2][j] = dot3(0.0, 0.0, 1.0, r0, r1, r2);
    }
    double row0[4], row1[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      row0[j] = mm0 * P[2][j] - P[0][j];
      row1[j] = mm1 * P[2][j] - P[1][j];
    }
    qr_add_row<4>(R4, row0);
    qr_add_row<4>(R4, row1);
    // vech linearisation of M S M^T (multiview.py:138-156), columns xx xy xz yy yz zz
    const double *M0 = p.M, *M1 = p.M + 3;
    double L0[6], L1[6], L2[6];
    const int vi[6] = {0, 0, 0, 1, 1, 2}, vj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int k = 0; k < 6; k++) {
      const int i = vi[k], j = vj[k];
      if (i == j) {
        L0[k] = M0[i] * M0[i];
        L1[k] = M0[i] * M1[i];
        L2[k] = M1[i] * M1[i];
      } else {
        L0[k] = 2.0 * M0[i] * M0[j];
        L1[k] = M0[i] * M1[j] + M0[j] * M1[i];
        L2[k] = 2.0 * M1[i] * M1[j];
      }
    }
    qr_add_row_rhs<6>(R6, c6, L0, mc00);
    qr_add_row_rhs<6>(R6, c6, L1, mc01);
    qr_add_row_rhs<6>(R6, c6, L2, mc11);
   }
  }
  if (bad) return TS_STATUS_UNSOLVABLE;
  return fuse_finish(gs, R4, R6, c6, cfg, delta, q, sc, allow_slow, dbg);
}

TS_HD int fuse_gaussian(const double *gs, int64_t g, int64_t n, const ts_camera *cams, int V,
                        const ts_motions &m, const ts_config &cfg, double *delta, double *q,
                        double *sc, double *dbg = nullptr) {
  double R4[4][4], R6[6][6], c6[6];
  return fuse_gaussian(gs, g, n, cams, V, m, cfg, delta, q, sc, R4, R6, c6, true, dbg);
}

}  // namespace ts
