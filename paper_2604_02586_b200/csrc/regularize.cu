// regularize.cu -- motion regularisation on the device (regularize.py:37-188, glue pipeline.py:88-98).
//
//   R0  exact kNN (build_knn, regularize.py:37-53): uniform grid over the bounding box, points
//       radix-sorted by cell, one thread per point walking Chebyshev shells of cells until the
//       k-th best (distance, id) is provably closer than every unvisited cell.  Distances are
//       formed exactly like numpy's norm(positions - positions[i], axis=1):
//       sqrt((dx*dx + dy*dy) + dz*dz), dx = p_j - p_i, so the adjacency is bit-exact.
//   R1  static flags (detect_static_all :77-88), median filter (:91-121), and the propagation
//       prerequisites: source flag (SOLVED and not static) + intrinsic-XYZ Euler angles of the
//       relative rotation (:138-146).
//   R2  propagation (:124-174) + apply_updates (:177-188) -> updated Gaussian rows.
//
// All stages are one thread per Gaussian over O(k) neighbours; the whole regularisation of a
// 300k-Gaussian frame is a few hundred microseconds (the reference's O(N^2) kNN alone is hours).
#include <cub/cub.cuh>

#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.cuh"
#include "rotation.cuh"

namespace ts {

namespace {

constexpr int kMaxCellDim = 1024;

// ---------------------------------------------------------------------------------------------
// R0: kNN

__global__ void knn_bounds_partial(const double *pos, int64_t stride, int64_t n, double *part) {
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double v = pos[i * stride + a];
      lo[a] = fmin(lo[a], v);
      hi[a] = fmax(hi[a], v);
    }
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    double l = BR(tmp).Reduce(lo[a], cub::Min());
    __syncthreads();
    double h = BR(tmp).Reduce(hi[a], cub::Max());
    __syncthreads();
    if (threadIdx.x == 0) {
      part[blockIdx.x * 6 + a] = l;
      part[blockIdx.x * 6 + 3 + a] = h;
    }
  }
}

__global__ void knn_grid_setup(const double *part, int nb, int64_t n, int64_t cap, KnnGrid *g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double lo[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, hi[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
  for (int b = 0; b < nb; b++)
    for (int a = 0; a < 3; a++) {
      lo[a] = fmin(lo[a], part[b * 6 + a]);
      hi[a] = fmax(hi[a], part[b * 6 + 3 + a]);
    }
  double ext[3], maxe = 0.0, maxabs = 0.0;
  for (int a = 0; a < 3; a++) {
    ext[a] = hi[a] - lo[a];
    maxe = fmax(maxe, ext[a]);
    maxabs = fmax(maxabs, fmax(fabs(lo[a]), fabs(hi[a])));
  }
  double h = 1.0;
  int dim[3] = {1, 1, 1};
  if (maxe > 0.0 && isfinite(maxe)) {
    // ~2 points per cell over the non-degenerate axes
    double vol = 1.0;
    int d = 0;
    for (int a = 0; a < 3; a++)
      if (ext[a] > maxe * 1e-9) { vol *= ext[a]; d++; }
    const double cells = fmax(1.0, (double)n / 2.0);
    h = pow(vol / cells, 1.0 / d);
    for (int it = 0; it < 200; it++) {
      double prod = 1.0;
      for (int a = 0; a < 3; a++) {
        dim[a] = (ext[a] > maxe * 1e-9) ? (int)fmin(fmax(ceil(ext[a] / h), 1.0), kMaxCellDim) : 1;
        prod *= dim[a];
      }
      if (prod <= (double)cap) break;
      h *= 1.1;
    }
  }
  for (int a = 0; a < 3; a++) {
    g->lo[a] = lo[a];
    g->dim[a] = dim[a];
  }
  g->h = h;
  g->inv_h = 1.0 / h;
  g->slack = 1e-10 * (maxabs + maxe) + 1e-300;
  g->ncell = dim[0] * dim[1] * dim[2];
}

__device__ __forceinline__ int cell_axis(double v, double lo, double inv_h, int dim) {
  const double t = floor((v - lo) * inv_h);
  return t < 0.0 ? 0 : (t >= (double)(dim - 1) ? dim - 1 : (int)t);
}

__global__ void knn_cell_keys(const double *pos, int64_t stride, int64_t n, const KnnGrid *gp,
                              uint32_t *key, uint32_t *val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const KnnGrid g = *gp;
  const double *p = pos + i * stride;
  const int cx = cell_axis(p[0], g.lo[0], g.inv_h, g.dim[0]);
  const int cy = cell_axis(p[1], g.lo[1], g.inv_h, g.dim[1]);
  const int cz = cell_axis(p[2], g.lo[2], g.inv_h, g.dim[2]);
  key[i] = (uint32_t)((cz * g.dim[1] + cy) * g.dim[0] + cx);
  val[i] = (uint32_t)i;
}

__global__ void knn_gather(const double *pos, int64_t stride, const uint32_t *key,
                           const uint32_t *val, int64_t n, double4 *sp, uint32_t *cell_lo,
                           uint32_t *cell_hi) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t id = val[j];
  const double *p = pos + (int64_t)id * stride;
  sp[j] = make_double4(p[0], p[1], p[2], (double)id);
  const uint32_t k = key[j];
  if (j == 0 || key[j - 1] != k) cell_lo[k] = (uint32_t)j;
  if (j == n - 1 || key[j + 1] != k) cell_hi[k] = (uint32_t)j + 1;
}

template <int K>
__device__ __forceinline__ void topk_insert(double (&bd)[K], int64_t (&bi)[K], double d,
                                            int64_t id) {
  // caller guarantees (d, id) beats slot K-1
  bool placed = false;
#pragma unroll
  for (int s = K - 1; s >= 0; s--) {
    if (!placed) {
      if (s > 0 && (d < bd[s - 1] || (d == bd[s - 1] && id < bi[s - 1]))) {
        bd[s] = bd[s - 1];
        bi[s] = bi[s - 1];
      } else {
        bd[s] = d;
        bi[s] = id;
        placed = true;
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(128) knn_query(const double4 *sp, const uint32_t *cell_lo,
                                                 const uint32_t *cell_hi, const KnnGrid *gp,
                                                 int64_t n, int64_t *adj) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const KnnGrid g = *gp;
  const double4 me = sp[j];
  const int64_t qid = (int64_t)me.w;
  const int c[3] = {cell_axis(me.x, g.lo[0], g.inv_h, g.dim[0]),
                    cell_axis(me.y, g.lo[1], g.inv_h, g.dim[1]),
                    cell_axis(me.z, g.lo[2], g.inv_h, g.dim[2])};
  const double q[3] = {me.x, me.y, me.z};
  double bd[K];
  int64_t bi[K];
#pragma unroll
  for (int s = 0; s < K; s++) {
    bd[s] = INFINITY;
    bi[s] = LLONG_MAX;
  }
  int rmax = 0;
#pragma unroll
  for (int a = 0; a < 3; a++) rmax = max(rmax, max(c[a], g.dim[a] - 1 - c[a]));
  for (int r = 0; r <= rmax; r++) {
    for (int dz = -r; dz <= r; dz++) {
      const int z = c[2] + dz;
      if (z < 0 || z >= g.dim[2]) continue;
      for (int dy = -r; dy <= r; dy++) {
        const int y = c[1] + dy;
        if (y < 0 || y >= g.dim[1]) continue;
        const bool face = (dz == -r || dz == r || dy == -r || dy == r);
        const int step = (face || r == 0) ? 1 : 2 * r;
        for (int dx = -r; dx <= r; dx += step) {
          const int x = c[0] + dx;
          if (x < 0 || x >= g.dim[0]) continue;
          const int cell = (z * g.dim[1] + y) * g.dim[0] + x;
          const uint32_t e = cell_hi[cell];
          for (uint32_t t = cell_lo[cell]; t < e; t++) {
            const double4 p = sp[t];
            const int64_t id = (int64_t)p.w;
            if (id == qid) continue;
            const double ex = sub(p.x, me.x), ey = sub(p.y, me.y), ez = sub(p.z, me.z);
            const double d = sqrt_rn(add(add(mul(ex, ex), mul(ey, ey)), mul(ez, ez)));
            if (d < bd[K - 1] || (d == bd[K - 1] && id < bi[K - 1])) topk_insert<K>(bd, bi, d, id);
          }
        }
      }
    }
    if (bd[K - 1] < INFINITY) {
      // distance from q to the nearest cell outside the visited cube (infinite on closed sides)
      double gap = INFINITY;
#pragma unroll
      for (int a = 0; a < 3; a++) {
        if (c[a] - r > 0) gap = fmin(gap, q[a] - (g.lo[a] + (double)(c[a] - r) * g.h));
        if (c[a] + r + 1 < g.dim[a])
          gap = fmin(gap, (g.lo[a] + (double)(c[a] + r + 1) * g.h) - q[a]);
      }
      if (bd[K - 1] < (gap - g.slack) * (1.0 - 1e-12)) break;
    }
  }
#pragma unroll
  for (int s = 0; s < K; s++) adj[qid * K + s] = bi[s];
}

template <int K>
void launch_query(const double4 *sp, const uint32_t *lo, const uint32_t *hi, const KnnGrid *g,
                  int64_t n, int64_t *adj, cudaStream_t s) {
  knn_query<K><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(sp, lo, hi, g, n, adj);
}

// ---------------------------------------------------------------------------------------------
// R1 / R2

constexpr int kMaxSample = TS_KNN_MAX_K + 1;

// rows: (N, 11) mean(3) quaternion w x y z (4) scale(3) opacity
__device__ __forceinline__ void row_rot(const double *G, int64_t i, double *r) {
  const double *q = G + i * 11 + 3;
  quat_to_matrix(q[0], q[1], q[2], q[3], r);
}

// Componentwise value c (0-2 dmu, 3-11 dR, 12-14 ds) of update j against frame 1 (regularize.py:106-110).
template <int C>
__device__ __forceinline__ double delta_component(const double *G, const double *u_delta,
                                                  const double *u_rot, const double *u_scale,
                                                  int64_t j) {
  if (C < 3) return u_delta[j * 3 + C];
  if (C < 12) {
    double rn[9], r1[9];
    const double *q = u_rot + j * 4;
    quat_to_matrix(q[0], q[1], q[2], q[3], rn);
    row_rot(G, j, r1);
    return sub(rn[C - 3], r1[C - 3]);
  }
  return sub(u_scale[j * 3 + (C - 12)], G[j * 11 + 7 + (C - 12)]);
}

// np.median of vals[0..m): middle element, or the mean of the two middle ones.
__device__ double median_of(double *vals, int m) {
  for (int a = 1; a < m; a++) {  // insertion sort (m <= 33)
    const double v = vals[a];
    int b = a - 1;
    while (b >= 0 && vals[b] > v) {
      vals[b + 1] = vals[b];
      b--;
    }
    vals[b + 1] = v;
  }
  if (m & 1) return vals[m / 2];
  return dvd(add(vals[m / 2 - 1], vals[m / 2]), 2.0);
}

template <int C>
__device__ __forceinline__ double median_component(const double *G, const double *ud,
                                                   const double *ur, const double *us,
                                                   const int64_t *sample, int m, double *vals) {
  for (int s = 0; s < m; s++) vals[s] = delta_component<C>(G, ud, ur, us, sample[s]);
  return median_of(vals, m);
}

__device__ __forceinline__ double clamp_scale(double x) {  // np.maximum(x, SCALE_CLAMP)
  return (x > 1e-9 || isnan(x)) ? x : 1e-9;
}

// matrix_to_quat on a flat 3x3
__device__ __forceinline__ bool mat_to_quat(const double *m9, double *q) {
  double m[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) m[i][j] = m9[3 * i + j];
  return matrix_to_quat(m, q);
}

// STATIC_MODE: 0 none, 1 from counts (detect_static_all), 2 given flags
template <bool MEDIAN, int STATIC_MODE, bool PREP>
__global__ void __launch_bounds__(128) reg_filter(
    const double *G, int64_t n, ts_updates in, const int32_t *pix, const int32_t *spix, int V,
    const int64_t *adj, int kk, int min_hit, double frac, int min_views, ts_updates out,
    uint8_t *static_flag, uint8_t *source_flag, double *rel_euler) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool is_static = false;
  if (STATIC_MODE == 1) {
    int q = 0;
    for (int v = 0; v < V; v++) {
      const int32_t pc = pix[(int64_t)v * n + i], sc = spix[(int64_t)v * n + i];
      q += (pc > min_hit && (double)sc > mul(frac, (double)pc)) ? 1 : 0;
    }
    is_static = q >= min_views;
    static_flag[i] = is_static;
  } else if (STATIC_MODE == 2) {
    is_static = static_flag[i] != 0;
  }
  const int8_t st = in.status[i];
  const bool solved = st == TS_STATUS_SOLVED;
  double d3[3], q4[4], s3[3];
  if (MEDIAN && solved) {
    int64_t sample[kMaxSample];
    double vals[kMaxSample];
    int m = 0;
    sample[m++] = i;
    for (int t = 0; t < kk; t++) {
      const int64_t j = adj[i * kk + t];
      if (in.status[j] == TS_STATUS_SOLVED) sample[m++] = j;
    }
    double med[15];
#define TS_MED(C) med[C] = median_component<C>(G, in.delta_mean, in.rotation, in.scale, sample, m, vals)
    TS_MED(0); TS_MED(1); TS_MED(2); TS_MED(3); TS_MED(4); TS_MED(5); TS_MED(6); TS_MED(7);
    TS_MED(8); TS_MED(9); TS_MED(10); TS_MED(11); TS_MED(12); TS_MED(13); TS_MED(14);
#undef TS_MED
    double r1[9], m9[9], rot[9];
    row_rot(G, i, r1);
#pragma unroll
    for (int e = 0; e < 9; e++) m9[e] = add(r1[e], med[3 + e]);
    nearest_rotation(m9, rot);
    mat_to_quat(rot, q4);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      d3[a] = med[a];
      s3[a] = clamp_scale(add(G[i * 11 + 7 + a], med[12 + a]));
    }
  } else {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      d3[a] = in.delta_mean[i * 3 + a];
      s3[a] = in.scale[i * 3 + a];
    }
#pragma unroll
    for (int a = 0; a < 4; a++) q4[a] = in.rotation[i * 4 + a];
  }
#pragma unroll
  for (int a = 0; a < 3; a++) {
    out.delta_mean[i * 3 + a] = d3[a];
    out.scale[i * 3 + a] = s3[a];
  }
#pragma unroll
  for (int a = 0; a < 4; a++) out.rotation[i * 4 + a] = q4[a];
  out.status[i] = st;
  if (PREP) {
    const bool source = solved && !is_static;
    source_flag[i] = source;
    if (source) {  // rel = R(new) @ R(frame1)^T -> scipy as_euler("XYZ")  (regularize.py:142-146)
      double rn[9], r1[9], rel[9], sq[4], ang[3];
      quat_to_matrix(q4[0], q4[1], q4[2], q4[3], rn);
      row_rot(G, i, r1);
      matmul3_bt(rn, r1, rel);
      sp_from_matrix(rel, sq);
      sp_as_euler_XYZ(sq, ang);
#pragma unroll
      for (int a = 0; a < 3; a++) rel_euler[i * 3 + a] = ang[a];
    }
  }
}

template <bool PROPAGATE, bool APPLY>
__global__ void __launch_bounds__(128) reg_propagate(
    const double *G, int64_t n, ts_updates u, const uint8_t *static_flag,
    const uint8_t *source_flag, const double *rel_euler, const int64_t *adj, int kk, int average,
    double *rows_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double *g = G + i * 11;
  if (PROPAGATE) {
    if (static_flag[i]) {
#pragma unroll
      for (int a = 0; a < 3; a++) {
        u.delta_mean[i * 3 + a] = 0.0;
        u.scale[i * 3 + a] = g[7 + a];
      }
#pragma unroll
      for (int a = 0; a < 4; a++) u.rotation[i * 4 + a] = g[3 + a];
      u.status[i] = TS_STATUS_STATIC;
    } else if (u.status[i] == TS_STATUS_UNSOLVABLE) {
      int64_t nb[TS_KNN_MAX_K];
      int m = 0;
      for (int t = 0; t < kk; t++) {
        const int64_t j = adj[i * kk + t];
        if (source_flag[j]) nb[m++] = j;
      }
      if (m > 0) {
        double dm[3], ds[3];
        if (average == 0) {  // np.mean over axis 0: sequential sums / m
#pragma unroll
          for (int a = 0; a < 3; a++) {
            double sd = u.delta_mean[nb[0] * 3 + a];
            double ss = sub(u.scale[nb[0] * 3 + a], G[nb[0] * 11 + 7 + a]);
            for (int t = 1; t < m; t++) {
              sd = add(sd, u.delta_mean[nb[t] * 3 + a]);
              ss = add(ss, sub(u.scale[nb[t] * 3 + a], G[nb[t] * 11 + 7 + a]));
            }
            dm[a] = dvd(sd, (double)m);
            ds[a] = dvd(ss, (double)m);
          }
        } else {
          double vals[TS_KNN_MAX_K];
#pragma unroll
          for (int a = 0; a < 3; a++) {
            for (int t = 0; t < m; t++) vals[t] = u.delta_mean[nb[t] * 3 + a];
            dm[a] = median_of(vals, m);
            for (int t = 0; t < m; t++) vals[t] = sub(u.scale[nb[t] * 3 + a], G[nb[t] * 11 + 7 + a]);
            ds[a] = median_of(vals, m);
          }
        }
        // _circular_mean (regularize.py:119-121)
        double ang[3];
#pragma unroll
        for (int a = 0; a < 3; a++) {
          double ss = sin(rel_euler[nb[0] * 3 + a]), cs = cos(rel_euler[nb[0] * 3 + a]);
          for (int t = 1; t < m; t++) {
            ss = add(ss, sin(rel_euler[nb[t] * 3 + a]));
            cs = add(cs, cos(rel_euler[nb[t] * 3 + a]));
          }
          ang[a] = atan2(dvd(ss, (double)m), dvd(cs, (double)m));
        }
        double relm[9], r1[9], rot[9], q4[4];
        sp_euler_XYZ_to_matrix(ang, relm);
        row_rot(G, i, r1);
        matmul3(relm, r1, rot);
        mat_to_quat(rot, q4);
#pragma unroll
        for (int a = 0; a < 3; a++) {
          u.delta_mean[i * 3 + a] = dm[a];
          u.scale[i * 3 + a] = clamp_scale(add(g[7 + a], ds[a]));
        }
#pragma unroll
        for (int a = 0; a < 4; a++) u.rotation[i * 4 + a] = q4[a];
        u.status[i] = TS_STATUS_SOLVED;
      }
    }
  }
  if (APPLY) {  // apply_updates (regularize.py:177-188): Gaussian3D renormalises the quaternion
    double *o = rows_out + i * 11;
    if (u.status[i] == TS_STATUS_UNSOLVABLE) {
#pragma unroll
      for (int a = 0; a < 11; a++) o[a] = g[a];
    } else {
      double q[4];
#pragma unroll
      for (int a = 0; a < 4; a++) q[a] = u.rotation[i * 4 + a];
      const double nrm = dot4_norm(q);
#pragma unroll
      for (int a = 0; a < 3; a++) {
        o[a] = add(g[a], u.delta_mean[i * 3 + a]);
        o[7 + a] = u.scale[i * 3 + a];
      }
#pragma unroll
      for (int a = 0; a < 4; a++) o[3 + a] = dvd(q[a], nrm);
      o[10] = g[10];
    }
  }
}

__global__ void k_static_flags(const int32_t *pix, const int32_t *spix, int64_t n, int V,
                               int min_hit, double frac, int min_views, uint8_t *flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int q = 0;
  for (int v = 0; v < V; v++) {
    const int32_t pc = pix[(int64_t)v * n + i], sc = spix[(int64_t)v * n + i];
    q += (pc > min_hit && (double)sc > mul(frac, (double)pc)) ? 1 : 0;
  }
  flag[i] = q >= min_views;
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int knn_bound_blocks(int64_t n) { return (int)std::min<int64_t>(296, std::max<int64_t>(1, (n + 255) / 256)); }

void launch_knn_grid(const double *pos, int64_t stride, int64_t n, int64_t cap, double *part,
                     KnnGrid *g, uint32_t *key, uint32_t *val, cudaStream_t s) {
  const int nb = knn_bound_blocks(n);
  knn_bounds_partial<<<nb, 256, 0, s>>>(pos, stride, n, part);
  knn_grid_setup<<<1, 32, 0, s>>>(part, nb, n, cap, g);
  knn_cell_keys<<<blocks(n, 256), 256, 0, s>>>(pos, stride, n, g, key, val);
}

void launch_knn_gather(const double *pos, int64_t stride, const uint32_t *key, const uint32_t *val,
                       int64_t n, double4 *sp, uint32_t *cell_lo, uint32_t *cell_hi,
                       cudaStream_t s) {
  knn_gather<<<blocks(n, 256), 256, 0, s>>>(pos, stride, key, val, n, sp, cell_lo, cell_hi);
}

cudaError_t launch_knn_query(int k, const double4 *sp, const uint32_t *lo, const uint32_t *hi,
                             const KnnGrid *g, int64_t n, int64_t *adj, cudaStream_t s) {
  switch (k) {
#define TS_Q(K) case K: launch_query<K>(sp, lo, hi, g, n, adj, s); break;
    TS_Q(1) TS_Q(2) TS_Q(3) TS_Q(4) TS_Q(5) TS_Q(6) TS_Q(7) TS_Q(8) TS_Q(9) TS_Q(10) TS_Q(11)
    TS_Q(12) TS_Q(13) TS_Q(14) TS_Q(15) TS_Q(16) TS_Q(17) TS_Q(18) TS_Q(19) TS_Q(20) TS_Q(21)
    TS_Q(22) TS_Q(23) TS_Q(24) TS_Q(25) TS_Q(26) TS_Q(27) TS_Q(28) TS_Q(29) TS_Q(30) TS_Q(31)
    TS_Q(32)
#undef TS_Q
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

void launch_static_flags(const int32_t *pix, const int32_t *spix, int64_t n, int V, int min_hit,
                         double frac, int min_views, uint8_t *flag, cudaStream_t s) {
  k_static_flags<<<blocks(n, 256), 256, 0, s>>>(pix, spix, n, V, min_hit, frac, min_views, flag);
}

void launch_reg_filter(int mode, const double *G, int64_t n, ts_updates in, const int32_t *pix,
                       const int32_t *spix, int V, const int64_t *adj, int kk, int min_hit,
                       double frac, int min_views, ts_updates out, uint8_t *static_flag,
                       uint8_t *source_flag, double *rel_euler, cudaStream_t s) {
  const unsigned nb = blocks(n, 128);
#define TS_F(M, S, P) \
  reg_filter<M, S, P><<<nb, 128, 0, s>>>(G, n, in, pix, spix, V, adj, kk, min_hit, frac, \
                                         min_views, out, static_flag, source_flag, rel_euler)
  switch (mode) {
    case REG_MEDIAN_ONLY: TS_F(true, 0, false); break;
    case REG_PREP_GIVEN_STATIC: TS_F(false, 2, true); break;
    case REG_FULL: TS_F(true, 1, true); break;
  }
#undef TS_F
}

void launch_reg_propagate(bool propagate, bool apply, const double *G, int64_t n, ts_updates u,
                          const uint8_t *static_flag, const uint8_t *source_flag,
                          const double *rel_euler, const int64_t *adj, int kk, int average,
                          double *rows_out, cudaStream_t s) {
  const unsigned nb = blocks(n, 128);
  if (propagate && apply)
    reg_propagate<true, true><<<nb, 128, 0, s>>>(G, n, u, static_flag, source_flag, rel_euler, adj,
                                                 kk, average, rows_out);
  else if (propagate)
    reg_propagate<true, false><<<nb, 128, 0, s>>>(G, n, u, static_flag, source_flag, rel_euler,
                                                  adj, kk, average, rows_out);
  else
    reg_propagate<false, true><<<nb, 128, 0, s>>>(G, n, u, static_flag, source_flag, rel_euler,
                                                  adj, kk, average, rows_out);
}

}  // namespace ts
