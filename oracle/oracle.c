/*
 * oracle.c -- CPU restatement of the gausstrack hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It restates, in plain C
 * with the reference's exact floating-point operation order, the parts of the reference
 * that the GPU path must reproduce bit-for-bit or to tight tolerance:
 *
 *   orc_project      gausstrack/splat.py:80-110  (_project_all)
 *                    numpy/OpenBLAS evaluates every 3-term dot product of `@` as the FMA chain
 *                    fma(a2,b2, fma(a1,b1, a0*b0)); pinned bit-for-bit against the reference.
 *   orc_rasterize    gausstrack/splat.py:113-195 (rasterize_weights): 3-sigma bbox, explicit
 *                    inverse, q in numpy's left-to-right order, alpha clamp, keep predicate,
 *                    lexsort((gid, depth, pix)), view-global log1p/cumsum transmittance,
 *                    early stop.  t_mode 1 swaps the log-cumsum T for the exact running product
 *                    per pixel (what the GPU composites): the reference's own T drift (~1e-8 rel
 *                    at 1e7 contributions per view) then drops out of at-scale comparisons.
 *   orc_bin          restatement of the tile binning the GPU adds on top of splat.py:131-146
 *                    (16x16 tiles, per-tile order = (depth, gid) as in splat.py:178).
 *   orc_accumulate   gausstrack/motion2d.py:126-161 (accumulate_view): np.add.at in array
 *                    order, products formed as (w*h_i)*h_j, static test sqrt(d0^2+d1^2) < thr.
 *
 * Compile with -ffp-contract=off: every FMA below is explicit.
 * exp/log1p come from libm; numpy's AVX-512 kernels differ from libm by <= 1 ulp in a few
 * percent of arguments, so alpha and T are tolerance outputs (rel 1e-12 / 1e-9), and the
 * predicates they feed can only flip for values within 1 ulp of a threshold.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEPTH_CUTOFF 1e-6     /* core.py:17 */
#define ALPHA_CLAMP 0.999     /* splat.py:18 */
#define DET_FLOOR 1e-12       /* splat.py:20 */
#define SIGMA_RADIUS 3.0      /* splat.py:21 */

/* camera layout (18 doubles): R[9] row-major world->camera, t[3], fx, fy, cx, cy, width, height */

static inline double dot3_fma(double a0, double a1, double a2, double b0, double b1, double b2) {
  return fma(a2, b2, fma(a1, b1, a0 * b0));
}

/* core.py:31-38 quat_to_matrix, Python float ops (no contraction) */
static void quat_to_matrix(const double *q, double *r) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  r[0] = 1 - 2 * (y * y + z * z);
  r[1] = 2 * (x * y - w * z);
  r[2] = 2 * (x * z + w * y);
  r[3] = 2 * (x * y + w * z);
  r[4] = 1 - 2 * (x * x + z * z);
  r[5] = 2 * (y * z - w * x);
  r[6] = 2 * (x * z - w * y);
  r[7] = 2 * (y * z + w * x);
  r[8] = 1 - 2 * (x * x + y * y);
}

/* One Gaussian (11 doubles: mean3, quat4 (w,x,y,z) already unit, scale3, opacity) into one view.
 * splat.py:91-110 / multiview.py:203-217. cov2 out = (xx, xy, yy) after 0.5*(C+C^T). */
static int project_one(const double *g, const double *cam, double *mean2, double *depth,
                       double *cov2) {
  const double *R = cam, *t = cam + 9;
  double fx = cam[12], fy = cam[13], cx = cam[14], cy = cam[15];
  double pc[3];
  for (int c = 0; c < 3; c++)
    pc[c] = dot3_fma(g[0], g[1], g[2], R[3 * c], R[3 * c + 1], R[3 * c + 2]) + t[c];
  double z = pc[2];
  int in_front = z > DEPTH_CUTOFF;
  double zs = in_front ? z : 1.0;
  mean2[0] = fx * pc[0] / zs + cx;
  mean2[1] = fy * pc[1] / zs + cy;
  *depth = z;
  double j00 = fx / zs, j11 = fy / zs;
  double j02 = -fx * pc[0] / (zs * zs);
  double j12 = -fy * pc[1] / (zs * zs);
  double M[6];
  for (int c = 0; c < 3; c++) {
    M[c] = dot3_fma(j00, 0.0, j02, R[c], R[3 + c], R[6 + c]);
    M[3 + c] = dot3_fma(0.0, j11, j12, R[c], R[3 + c], R[6 + c]);
  }
  double r[9];
  quat_to_matrix(g + 3, r);
  double s2[3] = {g[7] * g[7], g[8] * g[8], g[9] * g[9]};
  double rs[9], c3[9], T1[6], C[4];
  for (int a = 0; a < 3; a++)
    for (int c = 0; c < 3; c++) rs[3 * a + c] = r[3 * a + c] * s2[c];
  for (int a = 0; a < 3; a++)
    for (int c = 0; c < 3; c++)
      c3[3 * a + c] = dot3_fma(rs[3 * a], rs[3 * a + 1], rs[3 * a + 2], r[3 * c], r[3 * c + 1],
                               r[3 * c + 2]);
  for (int a = 0; a < 2; a++)
    for (int c = 0; c < 3; c++)
      T1[3 * a + c] = dot3_fma(M[3 * a], M[3 * a + 1], M[3 * a + 2], c3[c], c3[3 + c], c3[6 + c]);
  for (int a = 0; a < 2; a++)
    for (int c = 0; c < 2; c++)
      C[2 * a + c] =
          dot3_fma(T1[3 * a], T1[3 * a + 1], T1[3 * a + 2], M[3 * c], M[3 * c + 1], M[3 * c + 2]);
  cov2[0] = 0.5 * (C[0] + C[0]);
  cov2[1] = 0.5 * (C[1] + C[2]);
  cov2[2] = 0.5 * (C[3] + C[3]);
  return in_front;
}

void orc_project(int64_t n, const double *G, const double *cam, double *mean2, double *depth,
                 double *cov2, uint8_t *in_front) {
  for (int64_t i = 0; i < n; i++)
    in_front[i] = (uint8_t)project_one(G + 11 * i, cam, mean2 + 2 * i, depth + i, cov2 + 3 * i);
}

/* splat.py:131-146: status of one projected Gaussian.
 * returns 0 = behind camera, 1 = degenerate (det < 1e-12), 2 = empty bbox, 3 = has bbox. */
static int footprint(int in_front, const double *m2, const double *c, int W, int H, int *bb,
                     double *det_out) {
  if (!in_front) return 0;
  double det = c[0] * c[2] - c[1] * c[1];
  *det_out = det;
  if (det < DET_FLOOR) return 1;
  double rx = SIGMA_RADIUS * sqrt(c[0]);
  double ry = SIGMA_RADIUS * sqrt(c[2]);
  double x0 = fmax(ceil(m2[0] - rx), 0.0);
  double x1 = fmin(floor(m2[0] + rx), (double)(W - 1));
  double y0 = fmax(ceil(m2[1] - ry), 0.0);
  double y1 = fmin(floor(m2[1] + ry), (double)(H - 1));
  if (x0 > x1 || y0 > y1) return 2;
  bb[0] = (int)x0; bb[1] = (int)x1; bb[2] = (int)y0; bb[3] = (int)y1;
  return 3;
}

typedef struct {
  double depth;
  int64_t gid;
} gorder_t;

static int cmp_gorder(const void *a, const void *b) {
  const gorder_t *x = (const gorder_t *)a, *y = (const gorder_t *)b;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  if (x->gid != y->gid) return x->gid < y->gid ? -1 : 1;
  return 0;
}

typedef struct {
  int64_t gid;
  double alpha;
  double depth;
  int32_t px, py;
} contrib_t;

/* splat.py:113-195.  Outputs are written only if n_kept <= cap; the return value is always the
 * number of kept contributions (call again with a larger cap if it exceeds cap).
 * degenerate ids (<= n of them) go to `degenerate`, count in *n_degenerate.
 *
 * The contribution order is the reference's lexsort((gid, depth, pix)) (splat.py:171-180).  It is
 * formed without a comparison sort over the contributions: the binned Gaussians are ordered by
 * (depth, gid) first, their contributions generated in that order, and a stable counting sort by
 * pixel index then yields exactly the (pix, depth, gid) order. */
int64_t orc_rasterize(int64_t n, const double *G, const double *cam, double alpha_cutoff,
                      double early_stop, int64_t cap, int32_t *px_o, int32_t *py_o,
                      int64_t *gid_o, double *alpha_o, double *trans_o, double *depth_o,
                      int64_t *degenerate, int64_t *n_degenerate, int t_mode) {
  int W = (int)cam[16], H = (int)cam[17];
  int64_t npix = (int64_t)W * H;
  int64_t ndeg = 0, nb = 0;
  gorder_t *ord = (gorder_t *)malloc(sizeof(gorder_t) * (n > 0 ? n : 1));
  for (int64_t gid = 0; gid < n; gid++) {
    double m2[2], z, c[3], det;
    int inf = project_one(G + 11 * gid, cam, m2, &z, c);
    int bb[4];
    int st = footprint(inf, m2, c, W, H, bb, &det);
    if (st == 1) degenerate[ndeg++] = gid;
    if (st != 3) continue;
    ord[nb].depth = z;
    ord[nb].gid = gid;
    nb++;
  }
  *n_degenerate = ndeg;
  qsort(ord, (size_t)nb, sizeof(gorder_t), cmp_gorder);
  int64_t ncap = 1024, m = 0;
  contrib_t *cs = (contrib_t *)malloc(sizeof(contrib_t) * ncap);
  int64_t *pix_count = (int64_t *)calloc((size_t)npix + 1, sizeof(int64_t));
  for (int64_t k = 0; k < nb; k++) {
    const int64_t gid = ord[k].gid;
    const double *g = G + 11 * gid;
    double m2[2], z, c[3], det = 1.0;
    int inf = project_one(g, cam, m2, &z, c);
    int bb[4];
    footprint(inf, m2, c, W, H, bb, &det);
    double i00 = c[2] / det, i01 = -c[1] / det, i11 = c[0] / det;
    double two_i01 = 2 * i01;
    double op = g[10];
    for (int y = bb[2]; y <= bb[3]; y++) {
      double dy = (double)y - m2[1];
      for (int x = bb[0]; x <= bb[1]; x++) {
        double dx = (double)x - m2[0];
        double q = ((i00 * dx) * dx + (two_i01 * dx) * dy) + (i11 * dy) * dy;
        if (!(q <= SIGMA_RADIUS * SIGMA_RADIUS)) continue;
        double a = op * exp(-0.5 * q);
        if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
        if (!(a >= alpha_cutoff)) continue;
        if (m == ncap) {
          ncap *= 2;
          cs = (contrib_t *)realloc(cs, sizeof(contrib_t) * ncap);
        }
        contrib_t *e = &cs[m++];
        e->gid = gid;
        e->alpha = a;
        e->depth = z;
        e->px = x;
        e->py = y;
        pix_count[(int64_t)y * W + x + 1]++;
      }
    }
  }
  free(ord);
  /* stable counting sort by pixel: perm[k] = generation index of the k-th contribution */
  for (int64_t p = 0; p < npix; p++) pix_count[p + 1] += pix_count[p];
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
  for (int64_t k = 0; k < m; k++) perm[pix_count[(int64_t)cs[k].py * W + cs[k].px]++] = k;
  free(pix_count);
  /* view-global log-cumsum transmittance, splat.py:182-191 */
  int64_t kept = 0;
  double csum = 0.0, seg_base = 0.0, tprod = 1.0;
  int64_t prev_pix = -1;
  /* Once a pixel's T falls below early_stop its later entries are cut as well: along a segment
   * (csum - l) - seg_base drops by |log1p(-alpha)| >= |log1p(-alpha_cutoff)| per entry, which
   * dwarfs the rounding of the running sum (~1e-13 in log space) whenever alpha_cutoff >= 1e-6,
   * so the skipped exp calls could not have passed the test. */
  const int can_skip = alpha_cutoff >= 1e-6;
  int cut = 0;
  for (int64_t k = 0; k < m; k++) {
    const contrib_t *e = &cs[perm[k]];
    const int64_t pix = (int64_t)e->py * W + e->px;
    int start = pix != prev_pix;
    prev_pix = pix;
    double T;
    if (t_mode == 1) {
      /* exact running product (the GPU's compositing): T_in, then T *= (1 - alpha) */
      if (start) tprod = 1.0;
      T = tprod;
      tprod = tprod * (1.0 - e->alpha);
    } else {
      double l = log1p(-e->alpha);
      csum += l;
      if (start) {
        seg_base = csum - l;
        T = 1.0;
        cut = 0;
      } else if (cut) {
        continue; /* (csum - l) - seg_base only decreases along a segment (l <= 0) */
      } else {
        T = exp((csum - l) - seg_base);
      }
    }
    if (!(T >= early_stop)) cut = can_skip;
    if (T >= early_stop) {
      if (kept < cap) {
        px_o[kept] = e->px;
        py_o[kept] = e->py;
        gid_o[kept] = e->gid;
        alpha_o[kept] = e->alpha;
        trans_o[kept] = T;
        depth_o[kept] = e->depth;
      }
      kept++;
    }
  }
  free(perm);
  free(cs);
  return kept;
}

/* Binning restatement.  For one view: per Gaussian the bbox status (0..3 as footprint()), bbox
 * and tile rectangle; then every (tile, gid) instance ordered by (tile, depth, gid); tile_start /
 * tile_count per tile (tile = ty * tiles_x + tx).  Returns the number of instances (written only if
 * <= cap). */
typedef struct {
  int64_t tile;
  double depth;
  int64_t gid;
} inst_t;

static int cmp_inst(const void *a, const void *b) {
  const inst_t *x = (const inst_t *)a, *y = (const inst_t *)b;
  if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  if (x->gid != y->gid) return x->gid < y->gid ? -1 : 1;
  return 0;
}

int64_t orc_bin(int64_t n, const double *G, const double *cam, int tile_size, int64_t cap,
                int8_t *status, int32_t *bbox /* n x 4: x0 x1 y0 y1 */, int64_t *inst_tile,
                int64_t *inst_gid, int64_t *tile_start, int64_t *tile_count) {
  int W = (int)cam[16], H = (int)cam[17];
  int tx_n = (W + tile_size - 1) / tile_size, ty_n = (H + tile_size - 1) / tile_size;
  int64_t icap = 1024, m = 0;
  inst_t *is = (inst_t *)malloc(sizeof(inst_t) * icap);
  for (int64_t gid = 0; gid < n; gid++) {
    double m2[2], z, c[3], det;
    int inf = project_one(G + 11 * gid, cam, m2, &z, c);
    int bb[4] = {0, -1, 0, -1};
    int st = footprint(inf, m2, c, W, H, bb, &det);
    status[gid] = (int8_t)st;
    memcpy(bbox + 4 * gid, bb, sizeof(bb));
    if (st != 3) continue;
    for (int ty = bb[2] / tile_size; ty <= bb[3] / tile_size; ty++)
      for (int tx = bb[0] / tile_size; tx <= bb[1] / tile_size; tx++) {
        if (m == icap) {
          icap *= 2;
          is = (inst_t *)realloc(is, sizeof(inst_t) * icap);
        }
        is[m].tile = (int64_t)ty * tx_n + tx;
        is[m].depth = z;
        is[m].gid = gid;
        m++;
      }
  }
  qsort(is, (size_t)m, sizeof(inst_t), cmp_inst);
  for (int64_t t = 0; t < (int64_t)tx_n * ty_n; t++) {
    tile_start[t] = 0;
    tile_count[t] = 0;
  }
  for (int64_t k = 0; k < m; k++) {
    if (k < cap) {
      inst_tile[k] = is[k].tile;
      inst_gid[k] = is[k].gid;
    }
    if (tile_count[is[k].tile] == 0) tile_start[is[k].tile] = k;
    tile_count[is[k].tile]++;
  }
  free(is);
  return m;
}

/* motion2d.py:126-161 accumulate_view.  target is (H, W, 2) float64, valid (H, W) uint8.
 * Outputs (zeroed here): v1 n x 9, v2 n x 6, wsum n, cnt n, scnt n, swsum n. */
void orc_accumulate(int64_t m, const int32_t *px, const int32_t *py, const int64_t *gid,
                    const double *alpha, const double *trans, int W, int H, const double *target,
                    const uint8_t *valid, int64_t n, double thr, double *v1, double *v2,
                    double *wsum, int64_t *cnt, int64_t *scnt, double *swsum) {
  (void)H;
  memset(v1, 0, sizeof(double) * 9 * n);
  memset(v2, 0, sizeof(double) * 6 * n);
  memset(wsum, 0, sizeof(double) * n);
  memset(cnt, 0, sizeof(int64_t) * n);
  memset(scnt, 0, sizeof(int64_t) * n);
  memset(swsum, 0, sizeof(double) * n);
  for (int64_t k = 0; k < m; k++) {
    int64_t p = (int64_t)py[k] * W + px[k];
    if (!valid[p]) continue;
    int64_t g = gid[k];
    double h[3] = {(double)px[k], (double)py[k], 1.0};
    double xp[2] = {target[2 * p], target[2 * p + 1]};
    double w = alpha[k] * trans[k];
    for (int i = 0; i < 3; i++) {
      double wh = w * h[i];
      for (int j = 0; j < 3; j++) v1[9 * g + 3 * i + j] += wh * h[j];
      for (int j = 0; j < 2; j++) v2[6 * g + 2 * i + j] += wh * xp[j];
    }
    wsum[g] += w;
    cnt[g] += 1;
    double d0 = xp[0] - h[0], d1 = xp[1] - h[1];
    if (sqrt(d0 * d0 + d1 * d1) < thr) {
      scnt[g] += 1;
      swsum[g] += w;
    }
  }
}

/* build_knn (regularize.py:37-53): brute force over all pairs; distance exactly as
 * np.linalg.norm(positions - positions[i], axis=1) = sqrt((dx*dx + dy*dy) + dz*dz),
 * dx = p_j - p_i; the kk best by (distance, id) in ascending order. */
void orc_knn_queries(int64_t n, const double *pos, int kk, int64_t nq, const int64_t *qidx,
                     int64_t *adj) {
  double *bd = (double *)malloc(sizeof(double) * (size_t)(kk + 1));
  int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)(kk + 1));
  for (int64_t r = 0; r < nq; r++) {
    const int64_t i = qidx ? qidx[r] : r;
    int cnt = 0;
    const double *q = pos + 3 * i;
    for (int64_t j = 0; j < n; j++) {
      if (j == i) continue;
      const double *p = pos + 3 * j;
      const double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
      const double d = sqrt((dx * dx + dy * dy) + dz * dz);
      if (cnt == kk && !(d < bd[kk - 1] || (d == bd[kk - 1] && j < bi[kk - 1]))) continue;
      int s = cnt < kk ? cnt++ : kk - 1;
      while (s > 0 && (d < bd[s - 1] || (d == bd[s - 1] && j < bi[s - 1]))) {
        bd[s] = bd[s - 1];
        bi[s] = bi[s - 1];
        s--;
      }
      bd[s] = d;
      bi[s] = j;
    }
    for (int s = 0; s < kk; s++) adj[r * kk + s] = bi[s];
  }
  free(bd);
  free(bi);
}

void orc_knn(int64_t n, const double *pos, int kk, int64_t *adj) {
  orc_knn_queries(n, pos, kk, n, NULL, adj);
}

/* High-precision reference for at-scale comparisons of the per-view fits (accumulate_view +
 * solve_view, motion2d.py:126-184): moments in long double (x87, 64-bit mantissa) around an
 * anchor pixel per Gaussian (its first contribution; the translation is exact algebra), 3x3 solve
 * by partial-pivot elimination in long double, b mapped back to absolute pixels.  The
 * reference's own fp64 sums of absolute pixel moments have condition numbers of 1e10-1e14
 * (SURVEY §7), so at scale it is the less accurate side; this restatement is the yardstick both
 * the GPU and the fp64 restatement are measured against.  Outputs per Gaussian: status
 * (count >= min_pixels && sum w >= min_weight && det >= det_floor), a (2x2), b (2), and the
 * moved mean A mu + b of the given 2D means mu (N, 2). */
void orc_fit_hp(int64_t m, const int32_t *px, const int32_t *py, const int64_t *gid,
                const double *alpha, const double *trans, int W, const double *target,
                const uint8_t *valid, int64_t n, double det_floor, int64_t min_pixels,
                double min_weight, const double *mu, int8_t *status, double *a_out,
                double *b_out, double *moved_out) {
  long double *acc = (long double *)calloc((size_t)n * 15, sizeof(long double));
  int64_t *cnt = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  int32_t *anc = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)(n > 0 ? n : 1));
  for (int64_t k = 0; k < m; k++) {
    int64_t pix = (int64_t)py[k] * W + px[k];
    if (!valid[pix]) continue;
    int64_t g = gid[k];
    if (cnt[g] == 0) {
      anc[2 * g] = px[k];
      anc[2 * g + 1] = py[k];
    }
    long double w = (long double)alpha[k] * (long double)trans[k];
    long double x = (long double)(px[k] - anc[2 * g]), y = (long double)(py[k] - anc[2 * g + 1]);
    long double u = target[2 * pix], v = target[2 * pix + 1];
    long double *A = acc + 15 * g;
    A[0] += w; A[1] += w * x; A[2] += w * y; A[3] += w * x * x; A[4] += w * x * y;
    A[5] += w * y * y; A[6] += w * u; A[7] += w * v; A[8] += w * x * u; A[9] += w * x * v;
    A[10] += w * y * u; A[11] += w * y * v;
    cnt[g]++;
  }
  for (int64_t g = 0; g < n; g++) {
    long double *A = acc + 15 * g;
    /* h = [x, y, 1]: V1 = [[Sxx Sxy Sx] [Sxy Syy Sy] [Sx Sy S]], V2 rows h_i * [u v] */
    long double M[3][5] = {{A[3], A[4], A[1], A[8], A[9]},
                           {A[4], A[5], A[2], A[10], A[11]},
                           {A[1], A[2], A[0], A[6], A[7]}};
    long double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                      M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                      M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    int ok = cnt[g] >= min_pixels && A[0] >= (long double)min_weight &&
             det >= (long double)det_floor;
    status[g] = (int8_t)ok;
    double *ao = a_out + 4 * g, *bo = b_out + 2 * g, *mo = moved_out + 2 * g;
    if (!ok) {
      ao[0] = 1; ao[1] = 0; ao[2] = 0; ao[3] = 1; bo[0] = bo[1] = 0;
      mo[0] = mu[2 * g];
      mo[1] = mu[2 * g + 1];
      continue;
    }
    for (int c = 0; c < 3; c++) {
      int p = c;
      for (int r = c + 1; r < 3; r++)
        if (fabsl(M[r][c]) > fabsl(M[p][c])) p = r;
      if (p != c)
        for (int j = 0; j < 5; j++) {
          long double t = M[c][j]; M[c][j] = M[p][j]; M[p][j] = t;
        }
      for (int r = c + 1; r < 3; r++) {
        long double f = M[r][c] / M[c][c];
        for (int j = c; j < 5; j++) M[r][j] -= f * M[c][j];
      }
    }
    long double X[3][2];
    for (int rhs = 0; rhs < 2; rhs++)
      for (int r = 2; r >= 0; r--) {
        long double s = M[r][3 + rhs];
        for (int j = r + 1; j < 3; j++) s -= M[r][j] * X[j][rhs];
        X[r][rhs] = s / M[r][r];
      }
    /* X = [A^T; b_a^T] in anchored coordinates: x' = A (x - anc) + b_a */
    long double a00 = X[0][0], a01 = X[1][0], a10 = X[0][1], a11 = X[1][1];
    long double ax = anc[2 * g], ay = anc[2 * g + 1];
    long double b0 = X[2][0] - (a00 * ax + a01 * ay), b1 = X[2][1] - (a10 * ax + a11 * ay);
    ao[0] = (double)a00; ao[1] = (double)a01; ao[2] = (double)a10; ao[3] = (double)a11;
    bo[0] = (double)b0; bo[1] = (double)b1;
    long double mx = mu[2 * g], my = mu[2 * g + 1];
    mo[0] = (double)(a00 * mx + a01 * my + b0);
    mo[1] = (double)(a10 * mx + a11 * my + b1);
  }
  free(acc);
  free(cnt);
  free(anc);
}
