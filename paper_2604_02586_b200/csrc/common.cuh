// common.cuh -- shared device code for the B200 motion-estimation hot path (sm_100a).
//
// Exact-order fp64 math: every operation whose rounding the reference pins (projection,
// footprint, Mahalanobis q, static test) is written with explicit __dmul_rn/__dadd_rn/__fma_rn so
// nvcc cannot contract or reorder it.  The FMA-chain dot product reproduces numpy's `@` on these
// shapes (OpenBLAS dgemm accumulates k = 0..2 with FMA) -- pinned bit-for-bit by the oracle tests.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>

#include "../../include/trackersplat_b200.h"

#define TS_DEPTH_CUTOFF 1e-6  // core.py:17
#define TS_ALPHA_CLAMP 0.999  // splat.py:18
#define TS_DET_FLOOR 1e-12    // splat.py:20
#define TS_SIGMA_RADIUS 3.0   // splat.py:21
#define TS_TILE 16            // tile edge in pixels (binning unit of K1/K2)
#define TS_SINGULAR_GAP_REL 1e-9  // multiview.py:28

#define TS_CUDA_TRY(expr)                       \
  do {                                          \
    cudaError_t _e = (expr);                    \
    if (_e != cudaSuccess) return TS_E_CUDA;    \
  } while (0)

namespace ts {

// TS_HD functions also compile for the host so tests/native can unit-test the math on a CPU
// (host builds use -ffp-contract=off; the product path is the device code).
#define TS_HD __host__ __device__ __forceinline__
#ifdef __CUDA_ARCH__
TS_HD double mul(double a, double b) { return __dmul_rn(a, b); }
TS_HD double add(double a, double b) { return __dadd_rn(a, b); }
TS_HD double sub(double a, double b) { return __dsub_rn(a, b); }
TS_HD double dvd(double a, double b) { return __ddiv_rn(a, b); }
TS_HD double fmaa(double a, double b, double c) { return __fma_rn(a, b, c); }
TS_HD double sqrt_rn(double a) { return __dsqrt_rn(a); }
#else
TS_HD double mul(double a, double b) { return a * b; }
TS_HD double add(double a, double b) { return a + b; }
TS_HD double sub(double a, double b) { return a - b; }
TS_HD double dvd(double a, double b) { return a / b; }
TS_HD double fmaa(double a, double b, double c) { return fma(a, b, c); }
TS_HD double sqrt_rn(double a) { return sqrt(a); }
#endif

// numpy/OpenBLAS 3-term dot: fma(a2,b2, fma(a1,b1, a0*b0))
TS_HD double dot3(double a0, double a1, double a2, double b0, double b1,
                                       double b2) {
  return fmaa(a2, b2, fmaa(a1, b1, mul(a0, b0)));
}

// core.py:31-38 (Python float ops: each product / sum rounded, no contraction)
TS_HD void quat_to_matrix(double w, double x, double y, double z, double *r) {
  r[0] = sub(1.0, mul(2.0, add(mul(y, y), mul(z, z))));
  r[1] = mul(2.0, sub(mul(x, y), mul(w, z)));
  r[2] = mul(2.0, add(mul(x, z), mul(w, y)));
  r[3] = mul(2.0, add(mul(x, y), mul(w, z)));
  r[4] = sub(1.0, mul(2.0, add(mul(x, x), mul(z, z))));
  r[5] = mul(2.0, sub(mul(y, z), mul(w, x)));
  r[6] = mul(2.0, sub(mul(x, z), mul(w, y)));
  r[7] = mul(2.0, add(mul(y, z), mul(w, x)));
  r[8] = sub(1.0, mul(2.0, add(mul(x, x), mul(y, y))));
}

// World covariance R diag(s^2) R^T as numpy forms it: (rots * s2[:,None,:]) @ rots^T
// (splat.py:107, multiview.py:185).  c3 row-major 3x3.
TS_HD void covariance3d(const double *g, double *c3) {
  double r[9];
  quat_to_matrix(g[3], g[4], g[5], g[6], r);
  double s0 = mul(g[7], g[7]), s1 = mul(g[8], g[8]), s2 = mul(g[9], g[9]);
  double rs[9];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    rs[3 * a] = mul(r[3 * a], s0);
    rs[3 * a + 1] = mul(r[3 * a + 1], s1);
    rs[3 * a + 2] = mul(r[3 * a + 2], s2);
  }
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int c = 0; c < 3; c++)
      c3[3 * a + c] = dot3(rs[3 * a], rs[3 * a + 1], rs[3 * a + 2], r[3 * c], r[3 * c + 1],
                           r[3 * c + 2]);
}

struct Projection {
  double mean2[2];
  double depth;
  double M[6];     // 2x3 linearisation J @ R (row-major)
  double cov2[3];  // xx, xy, yy after 0.5*(C + C^T)
  bool in_front;
};

// splat.py:91-110 / multiview.py:203-217 for one Gaussian given its world covariance c3.
TS_HD void project(const double *mean, const double *c3, const ts_camera &cam,
                                        Projection &p) {
  const double *R = cam.R;
  double pc[3];
#pragma unroll
  for (int c = 0; c < 3; c++)
    pc[c] = add(dot3(mean[0], mean[1], mean[2], R[3 * c], R[3 * c + 1], R[3 * c + 2]), cam.t[c]);
  double z = pc[2];
  p.in_front = z > TS_DEPTH_CUTOFF;
  double zs = p.in_front ? z : 1.0;
  p.mean2[0] = add(dvd(mul(cam.fx, pc[0]), zs), cam.cx);
  p.mean2[1] = add(dvd(mul(cam.fy, pc[1]), zs), cam.cy);
  p.depth = z;
  double zz = mul(zs, zs);
  double j00 = dvd(cam.fx, zs), j11 = dvd(cam.fy, zs);
  double j02 = dvd(mul(-cam.fx, pc[0]), zz);
  double j12 = dvd(mul(-cam.fy, pc[1]), zz);
#pragma unroll
  for (int c = 0; c < 3; c++) {
    p.M[c] = dot3(j00, 0.0, j02, R[c], R[3 + c], R[6 + c]);
    p.M[3 + c] = dot3(0.0, j11, j12, R[c], R[3 + c], R[6 + c]);
  }
  double T1[6];
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int c = 0; c < 3; c++)
      T1[3 * a + c] = dot3(p.M[3 * a], p.M[3 * a + 1], p.M[3 * a + 2], c3[c], c3[3 + c], c3[6 + c]);
  double C00 = dot3(T1[0], T1[1], T1[2], p.M[0], p.M[1], p.M[2]);
  double C01 = dot3(T1[0], T1[1], T1[2], p.M[3], p.M[4], p.M[5]);
  double C10 = dot3(T1[3], T1[4], T1[5], p.M[0], p.M[1], p.M[2]);
  double C11 = dot3(T1[3], T1[4], T1[5], p.M[3], p.M[4], p.M[5]);
  p.cov2[0] = mul(0.5, add(C00, C00));
  p.cov2[1] = mul(0.5, add(C01, C10));
  p.cov2[2] = mul(0.5, add(C11, C11));
}

// Raster record of one (view, Gaussian): everything K2 needs, 64 bytes.
struct __align__(16) RasterRec {
  double mx, my;             // projected mean
  double i00, i01x2, i11;    // explicit inverse (splat.py:152): c11/det, 2*(-c01/det), c00/det
  double opacity;
  int16_t x0, x1, y0, y1;    // inclusive 3-sigma bbox, clipped to the image (splat.py:139-144)
  uint32_t g;                // Gaussian id
  uint32_t pad;
};
static_assert(sizeof(RasterRec) == 64, "RasterRec must be 64 bytes");

// Footprint of a projected Gaussian (splat.py:131-146).  Returns 0 behind camera, 1 degenerate
// (det < 1e-12, reported), 2 empty bbox, 3 binned (rec filled).
TS_HD int footprint(const Projection &p, double opacity, int W, int H,
                                         RasterRec &rec) {
  if (!p.in_front) return 0;
  double c00 = p.cov2[0], c01 = p.cov2[1], c11 = p.cov2[2];
  double det = sub(mul(c00, c11), mul(c01, c01));
  if (det < TS_DET_FLOOR) return 1;
  double rx = mul(TS_SIGMA_RADIUS, sqrt_rn(c00));
  double ry = mul(TS_SIGMA_RADIUS, sqrt_rn(c11));
  double x0 = fmax(ceil(sub(p.mean2[0], rx)), 0.0);
  double x1 = fmin(floor(add(p.mean2[0], rx)), (double)(W - 1));
  double y0 = fmax(ceil(sub(p.mean2[1], ry)), 0.0);
  double y1 = fmin(floor(add(p.mean2[1], ry)), (double)(H - 1));
  if (!(x0 <= x1 && y0 <= y1)) return 2;
  rec.mx = p.mean2[0];
  rec.my = p.mean2[1];
  rec.i00 = dvd(c11, det);
  rec.i01x2 = mul(2.0, dvd(-c01, det));
  rec.i11 = dvd(c00, det);
  rec.opacity = opacity;
  rec.x0 = (int16_t)x0;
  rec.x1 = (int16_t)x1;
  rec.y0 = (int16_t)y0;
  rec.y1 = (int16_t)y1;
  return 3;
}

// 1-based index of the lowest set bit (0 for x == 0), host and device
TS_HD int ffs_hd(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __ffs((int)x);
#else
  return __builtin_ffs((int)x);
#endif
}

TS_HD int ffs64_hd(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __ffsll((long long)x);
#else
  return __builtin_ffsll((long long)x);
#endif
}

TS_HD uint64_t double_bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

// Mahalanobis q in numpy's evaluation order (splat.py:153):
//   ((i00*dx)*dx + ((2*i01)*dx)*dy) + (i11*dy)*dy
TS_HD double mahalanobis(const RasterRec &r, double dx, double dy) {
  return add(add(mul(mul(r.i00, dx), dx), mul(mul(r.i01x2, dx), dy)), mul(mul(r.i11, dy), dy));
}

// alpha = min(o * exp(-0.5 q), 0.999)  (splat.py:154)
// Table-driven exp(-q/2) for q in [0, 9] (the only range alpha is needed in):
// exp(x) = E[k] * P6(r), k = rint(64 x), r = x - k/64, |r| <= 1/128, E[k] = exp(-k/64).
// <= 2 ulp (vs numpy's exp: rel <= 5e-16); 11 instructions instead of the general exp.
#define TS_EXP_TABLE 289
// low 32 bits of a double as an int (the integer n of a 1.5*2^52-shifted value)
TS_HD int lo_int(double d) {
#ifdef __CUDA_ARCH__
  return __double2loint(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return (int)(uint32_t)u;
#endif
}
// the polynomial's coefficients as constant-bank operands of DFMA (no per-use UMOV pairs)
static __constant__ double k_exp_poly[4] = {1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0};
#ifdef __CUDA_ARCH__
#define TS_EXP_C(i, v) k_exp_poly[i]
#else
#define TS_EXP_C(i, v) (v)
#endif
TS_HD double alpha_of_table(double opacity, double q, const double *etab) {
  const double x = mul(-0.5, q);
  // round-to-nearest-even of 64 x with the 1.5*2^52 shifter: stays on the fp64 pipe (no F2F/F2I)
  const double kd = fma(x, 64.0, 6755399441055744.0);
  const double kf = kd - 6755399441055744.0;
  const double r = fma(kf, -0.015625, x);
  double p = fma(r, TS_EXP_C(0, 1.0 / 720.0), TS_EXP_C(1, 1.0 / 120.0));
  p = fma(r, p, TS_EXP_C(2, 1.0 / 24.0));
  p = fma(r, p, TS_EXP_C(3, 1.0 / 6.0));
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = fma(r, p, 1.0);
  const double a = mul(opacity, etab[-lo_int(kd)] * p);
  return a > TS_ALPHA_CLAMP ? TS_ALPHA_CLAMP : a;
}

TS_HD double alpha_of(double opacity, double q) {
  double a = mul(opacity, exp(mul(-0.5, q)));
  return a > TS_ALPHA_CLAMP ? TS_ALPHA_CLAMP : a;
}

// static <=> ||x' - x|| < thr with numpy's norm: sqrt(d0*d0 + d1*d1) (motion2d.py:158)
TS_HD bool is_static(double u, double v, int px, int py, double thr) {
  double d0 = sub(u, (double)px), d1 = sub(v, (double)py);
  return sqrt_rn(add(mul(d0, d0), mul(d1, d1))) < thr;
}

// The same test without the square root: a correctly rounded sqrt is monotone, so
// {x : sqrt_rn(x) < thr} = [0, L] (or empty) and sqrt_rn(x) < thr <=> x <= L exactly; L is found
// on the host with its (IEEE, correctly rounded) sqrt.  NaN compares false on both sides.
inline double static_sq_limit(double thr) {
  if (!(thr > 0.0)) return -1.0;  // never static (x >= 0)
  if (std::isinf(thr)) return 1.7976931348623157e308;  // every finite x
  double x = thr * thr;
  if (std::isinf(x)) x = 1.7976931348623157e308;
  while (x > 0.0 && !(std::sqrt(x) < thr)) x = std::nextafter(x, 0.0);
  while (std::sqrt(std::nextafter(x, HUGE_VAL)) < thr) x = std::nextafter(x, HUGE_VAL);
  return x;
}
TS_HD bool is_static_sq(double u, double v, int px, int py, double lim) {
  double d0 = sub(u, (double)px), d1 = sub(v, (double)py);
  return add(mul(d0, d0), mul(d1, d1)) <= lim;
}

// Moments of one Gaussian in one tile, relative to the integer anchor
// ((x0+x1)>>1, (y0+y1)>>1) of its view bbox:  h = [dx, dy, 1], x'_a = x' - anchor.
//  0 S, 1 Sx, 2 Sy, 3 Sxx, 4 Sxy, 5 Syy, 6 Su, 7 Sv, 8 Sxu, 9 Sxv, 10 Syu, 11 Syv, 12 Sstatic_w
#define TS_NMOM 13
struct __align__(16) Partial {
  double m[TS_NMOM];
  uint32_t count, static_count;
  uint64_t pad;
};
static_assert(sizeof(Partial) == 128, "Partial must be 128 bytes");
static_assert(offsetof(Partial, count) == 104 && offsetof(Partial, static_count) == 108,
              "K3 reads (count, static_count) as the second half of the 7th 16-byte vector");

TS_HD int anchor_x(const RasterRec &r) { return ((int)r.x0 + (int)r.x1) >> 1; }
TS_HD int anchor_y(const RasterRec &r) { return ((int)r.y0 + (int)r.y1) >> 1; }

template <typename T>
__device__ __forceinline__ double load_track(const T *p) { return (double)__ldg(p); }

}  // namespace ts
