// motion.cuh -- per-(view, Gaussian) affine fit from K2's tile partials (host+device).
//
// solve_view (motion2d.py:164-184): eligibility count >= min_pixels, sum w >= min_weight,
// det(V1) >= det_floor (motion2d.py:168-170), then [A^T; b^T] = V1^-1 V2 (motion2d.py:173,
// LAPACK gesv = partial-pivot LU).  The moments are anchored at the integer bbox centre a
// (h = [x - a; 1], x'_a = x' - a): det is translation invariant and the anchored V1 has condition
// ~1e2 instead of the 1e10-1e14 of absolute pixel moments; b is mapped back as b_a + a - A a.
#pragma once

#include "common.cuh"

namespace ts {

template <int I, int J>
TS_HD void swap_rows3(double (&A)[3][3], double (&B)[3][2]) {
#pragma unroll
  for (int c = 0; c < 3; c++) {
    const double t = A[I][c];
    A[I][c] = A[J][c];
    A[J][c] = t;
  }
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const double t = B[I][c];
    B[I][c] = B[J][c];
    B[J][c] = t;
  }
}

// Partial-pivot LU solve of A X = B (3x3, 2 right-hand sides) with compile-time indices only
// (no dynamically indexed local arrays).  Returns det(A); X overwrites B when det != 0.
TS_HD double lu3_solve(double (&A)[3][3], double (&B)[3][2]) {
  double det = 1.0;
  // column 0: first maximum |A[i][0]| (LAPACK idamax)
  {
    const double a0 = fabs(A[0][0]), a1 = fabs(A[1][0]), a2 = fabs(A[2][0]);
    if (a1 > a0 && a1 >= a2) {
      swap_rows3<0, 1>(A, B);
      det = -det;
    } else if (a2 > a0 && a2 > a1) {
      swap_rows3<0, 2>(A, B);
      det = -det;
    }
  }
  const double d0 = A[0][0];
  det *= d0;
  if (d0 != 0.0) {
#pragma unroll
    for (int i = 1; i < 3; i++) {
      const double l = A[i][0] / d0;
      A[i][1] -= l * A[0][1];
      A[i][2] -= l * A[0][2];
      B[i][0] -= l * B[0][0];
      B[i][1] -= l * B[0][1];
    }
  }
  if (fabs(A[2][1]) > fabs(A[1][1])) {
    swap_rows3<1, 2>(A, B);
    det = -det;
  }
  const double d1 = A[1][1];
  det *= d1;
  if (d1 != 0.0) {
    const double l = A[2][1] / d1;
    A[2][2] -= l * A[1][2];
    B[2][0] -= l * B[1][0];
    B[2][1] -= l * B[1][1];
  }
  det *= A[2][2];
  if (det != 0.0) {
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const double x2 = B[2][j] / A[2][2];
      const double x1 = (B[1][j] - A[1][2] * x2) / A[1][1];
      const double x0 = (B[0][j] - A[0][1] * x1 - A[0][2] * x2) / A[0][0];
      B[0][j] = x0;
      B[1][j] = x1;
      B[2][j] = x2;
    }
  }
  return det;
}

struct GvMotion {
  double a[4], b[2];
  double wsum, static_wsum;
  uint32_t count, static_count;
  int8_t status;
};

// Add the flagged sub-slot of instance slot base (4 sub-slots per flag word) to the moments.
TS_HD void add_slot(const Partial *partial, uint32_t slot, double (&mom)[TS_NMOM], uint32_t &cnt,
                    uint32_t &scnt) {
  const double2 *p2 = reinterpret_cast<const double2 *>(partial + slot);
  double2 v[7];  // m[0..12] and (count, static_count) in the low / high words of v[6].y
#pragma unroll
  for (int k = 0; k < 7; k++) v[k] = p2[k];
#pragma unroll
  for (int k = 0; k < 6; k++) {
    mom[2 * k] += v[k].x;
    mom[2 * k + 1] += v[k].y;
  }
  mom[12] += v[6].x;
  const uint64_t counts = double_bits(v[6].y);
  cnt += (uint32_t)counts;
  scnt += (uint32_t)(counts >> 32);
}

// Add the flagged slots in [sb, se) of one gv (one slot per 8x8 quadrant of its bbox), in slot
// order.  The flag bytes are read as aligned 32-bit words (4 slots each), four words per round
// in flight; bytes outside [sb, se) are masked.  A warp can split the words: lane `first` of
// `stride` takes words first, first + stride, ... (the flag array is padded past the end).
TS_HD void accumulate_slots(const Partial *partial, const uint8_t *flag, uint32_t sb,
                            uint32_t se, uint32_t first, uint32_t stride,
                            double (&mom)[TS_NMOM], uint32_t &cnt, uint32_t &scnt) {
  const uint32_t w_end = (se + 3) >> 2;
  const uint32_t *fwords = reinterpret_cast<const uint32_t *>(flag);
  for (uint32_t w0 = (sb >> 2) + first; w0 < w_end; w0 += 4 * stride) {
    uint32_t fw[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t w = w0 + q * stride;
      uint32_t f = w < w_end ? fwords[w] : 0u;
      const uint32_t lo = sb > 4 * w ? sb - 4 * w : 0u;       // first byte inside the range
      const uint32_t hi = se < 4 * w + 4 ? se - 4 * w : 4u;    // one past the last
      const uint64_t keep = ((1ull << (8 * hi)) - 1ull) & ~((1ull << (8 * lo)) - 1ull);
      fw[q] = f & (uint32_t)keep;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t slot0 = 4 * (w0 + q * stride);
      uint32_t f4 = fw[q];
      while (f4) {
        const int sub = (ffs_hd(f4) - 1) >> 3;
        f4 &= ~(0xFFu << (8 * sub));
        add_slot(partial, slot0 + sub, mom, cnt, scnt);
      }
    }
  }
}

// Affine fit of one gv from its summed anchored moments (motion2d.py:164-184).
TS_HD GvMotion solve_moments(const double (&mom)[TS_NMOM], uint32_t cnt, uint32_t scnt,
                             int anchor_x, int anchor_y, double det_floor, int min_pixels,
                             double min_weight) {
  GvMotion r;
  r.a[0] = 1.0; r.a[1] = 0.0; r.a[2] = 0.0; r.a[3] = 1.0;
  r.b[0] = 0.0; r.b[1] = 0.0;
  r.wsum = mom[0];
  r.static_wsum = mom[12];
  r.count = cnt;
  r.static_count = scnt;
  r.status = TS_STATUS_UNSOLVABLE;
  if ((int)cnt >= min_pixels && mom[0] >= min_weight) {
    double V1[3][3] = {{mom[3], mom[4], mom[1]}, {mom[4], mom[5], mom[2]}, {mom[1], mom[2], mom[0]}};
    double X[3][2] = {{mom[8], mom[9]}, {mom[10], mom[11]}, {mom[6], mom[7]}};
    const double det = lu3_solve(V1, X);
    if (det >= det_floor) {
      // ab = [A^T; b_a^T] -> A = ab[:2].T, b_a = ab[2]  (motion2d.py:177)
      const double ax = (double)anchor_x, ay = (double)anchor_y;
      const double a00 = X[0][0], a01 = X[1][0], a10 = X[0][1], a11 = X[1][1];
      const double b0 = X[2][0] + ax - (a00 * ax + a01 * ay);
      const double b1 = X[2][1] + ay - (a10 * ax + a11 * ay);
      if (isfinite(a00) && isfinite(a01) && isfinite(a10) && isfinite(a11) && isfinite(b0) &&
          isfinite(b1)) {  // AffineMotion rejects non-finite entries (core.py:192-193)
        r.status = TS_STATUS_SOLVED;
        r.a[0] = a00; r.a[1] = a01; r.a[2] = a10; r.a[3] = a11;
        r.b[0] = b0; r.b[1] = b1;
      }
    }
  }
  return r;
}

// Sum the (instance, quadrant) sub-slots of one gv in fixed order and fit its affine motion.
TS_HD GvMotion solve_gv(const Partial *partial, const uint8_t *flag, uint32_t sb,
                        uint32_t nslots, int anchor_x, int anchor_y, double det_floor,
                        int min_pixels, double min_weight) {
  double mom[TS_NMOM];
#pragma unroll
  for (int k = 0; k < TS_NMOM; k++) mom[k] = 0.0;
  uint32_t cnt = 0, scnt = 0;
  accumulate_slots(partial, flag, sb, sb + nslots, 0, 1, mom, cnt, scnt);
  return solve_moments(mom, cnt, scnt, anchor_x, anchor_y, det_floor, min_pixels, min_weight);
}

}  // namespace ts
