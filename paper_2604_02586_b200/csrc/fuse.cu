// fuse.cu -- K4: multi-view fuse (update_all) with small least-squares solves in registers.
//
// Reference: gausstrack/multiview.py:168-275 (update_all), :53-70 (triangulate_mean),
// :73-100 (solve_covariance3d), :103-135 (decompose_covariance), core.py:41-62 (matrix_to_quat).
//
// One thread per Gaussian streams over its SOLVED views (view order, as the reference stacks
// them) and never materialises the stacked systems:
//   * every DLT row pair (multiview.py:223-225) is folded into a 4x4 upper-triangular R by Givens
//     rotations, every vech block + rhs (:226-229) into a 6x6 R and Q^T b.  QR keeps the singular
//     values and right singular vectors of the stacked matrix, so the reference's SVD-based tests
//     (s[-2]-s[-1] <= 1e-9 s[0]; |x3| <= 1e-9 |x|; s[-1] < 1e-9 s[0]) are taken on R;
//   * the degeneracy tests are decided by rigorous certificates on R where possible (inverse
//     iteration null vector + interlacing bound for the DLT gap; 1/(|R|_F |R^-1|_F) for the rank
//     test); the Gaussians they cannot decide are queued and finished by k4_finish with a
//     one-sided Jacobi SVD of R (high relative accuracy for the small singular values), so the
//     SVD never diverges a warp of k4_fuse; back substitution for the least squares;
//   * cyclic Jacobi for the 3x3 eigenproblem, then the reference's discrete choices verbatim:
//     first-maximum permutation in itertools order, sign flips, det repair, matrix_to_quat.
#include <float.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "smallsolve.cuh"

namespace ts {


// Deferred slow-path record: the R factors of a Gaussian whose triangulation-gap or rank decision
// needs an SVD (a few percent of Gaussians, but enough to put an SVD into almost every warp).
struct K4Deferred {
  double r4[10];  // upper triangle of R4, row-major
  double r6[21];  // upper triangle of R6
  double c6[6];
  int64_t g;
};

__device__ __forceinline__ void store_updates(ts_updates u, int64_t g, const double *delta,
                                              const double *q, const double *sc, int status) {
#pragma unroll
  for (int i = 0; i < 3; i++) {
    u.delta_mean[3 * g + i] = delta[i];
    u.scale[3 * g + i] = sc[i];
  }
#pragma unroll
  for (int i = 0; i < 4; i++) u.rotation[4 * g + i] = q[i];
  u.status[g] = (int8_t)status;
}

#ifndef TS_K4_MIN_BLOCKS
#define TS_K4_MIN_BLOCKS 3
#endif
// Eligibility pre-pass of update_all (multiview.py:231-235): ineligible Gaussians get their
// UNSOLVABLE update here; eligible ones are keyed by their solved-view count so that a descending
// radix sort groups Gaussians of equal work into the same warps of k4_fuse, heaviest first (the
// streaming QR loops over the solved views: mixed counts and early exits left ~12 of 32 lanes
// active, and the heaviest warps last made a tail).
__global__ void __launch_bounds__(256) k4_prep(const double *__restrict__ G, int64_t n, int V,
                                               K4Motions m, ts_config cfg, ts_updates u,
                                               uint32_t *__restrict__ key,
                                               uint32_t *__restrict__ val,
                                               uint64_t *__restrict__ solved_mask) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  int n_solved = 0;
  double tw = 0.0;
  int64_t tp = 0;
  uint64_t mask = 0;
  for (int v = 0; v < V; v++) {
    const int64_t gv = (int64_t)v * n + g;
    if (mot_status(m, gv) != TS_STATUS_SOLVED) continue;
    if (v < 64) mask |= 1ull << v;
    n_solved++;
    double w;
    int64_t c;
    mot_sums(m, gv, w, c);
    tw += w;
    tp += c;
  }
  const bool ok = n_solved >= cfg.min_views && tw >= cfg.min_total_weight &&
                  tp >= cfg.min_total_pixels;
  key[g] = ok ? (uint32_t)n_solved : 0u;  // descending sort: heaviest first, ineligible last
  val[g] = (uint32_t)g;
  solved_mask[g] = ok ? (V <= 64 ? mask : ~0ull) : 0ull;  // > 64 views: bits rebuilt by k4_fuse
  if (!ok) {
    double delta[3] = {0.0, 0.0, 0.0}, q[4], sc[3];
#pragma unroll
    for (int i = 0; i < 4; i++) q[i] = G[11 * g + 3 + i];
#pragma unroll
    for (int i = 0; i < 3; i++) sc[i] = G[11 * g + 7 + i];
    store_updates(u, g, delta, q, sc, TS_STATUS_UNSOLVABLE);
  }
}

__global__ void __launch_bounds__(128, TS_K4_MIN_BLOCKS) k4_fuse(const double *__restrict__ G, int64_t n,
                                               const ts_camera *__restrict__ cams, int V,
                                               K4Motions m, ts_config cfg, ts_updates u,
                                               const uint32_t *__restrict__ order_key,
                                               const uint32_t *__restrict__ order,
                                               const uint64_t *__restrict__ solved_mask,
                                               K4Deferred *defer, unsigned *n_defer) {
  extern __shared__ ts_camera s_cam4[];
  for (int i = threadIdx.x; i < V; i += blockDim.x) s_cam4[i] = cams[i];
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || order_key[t] == 0u) return;  // ineligible: written by k4_prep
  const int64_t g = order[t];
  double gs[11];
#pragma unroll
  for (int k = 0; k < 11; k++) gs[k] = G[11 * g + k];
  double delta[3], q[4], sc[3], R4[4][4], R6[6][6], c6[6];
  const int status = fuse_gaussian(gs, g, n, s_cam4, V, m, cfg, delta, q, sc, R4, R6, c6, false,
                                   nullptr, solved_mask[g]);
  if (status == TS_FUSE_DEFER_STATUS) {
    K4Deferred *d = defer + atomicAdd(n_defer, 1u);
    int k = 0;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = i; j < 4; j++) d->r4[k++] = R4[i][j];
    k = 0;
#pragma unroll
    for (int i = 0; i < 6; i++)
#pragma unroll
      for (int j = i; j < 6; j++) d->r6[k++] = R6[i][j];
#pragma unroll
    for (int i = 0; i < 6; i++) d->c6[i] = c6[i];
    d->g = g;
    return;
  }
  store_updates(u, g, delta, q, sc, status);
}

// The deferred Gaussians, with the SVD decisions (same code path as the host build).
__global__ void __launch_bounds__(128) k4_finish(const double *__restrict__ G, ts_config cfg,
                                                 ts_updates u, const K4Deferred *defer,
                                                 const unsigned *n_defer) {
  const unsigned cnt = *n_defer;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const K4Deferred &d = defer[i];
    const int64_t g = d.g;
    double gs[11];
#pragma unroll
    for (int k = 0; k < 11; k++) gs[k] = G[11 * g + k];
    double R4[4][4], R6[6][6], c6[6];
    int k = 0;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
      for (int b = 0; b < 4; b++) R4[a][b] = b >= a ? d.r4[k++] : 0.0;
    k = 0;
#pragma unroll
    for (int a = 0; a < 6; a++)
#pragma unroll
      for (int b = 0; b < 6; b++) R6[a][b] = b >= a ? d.r6[k++] : 0.0;
#pragma unroll
    for (int a = 0; a < 6; a++) c6[a] = d.c6[a];
    double delta[3], q[4], sc[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      delta[a] = 0.0;
      sc[a] = gs[7 + a];
    }
#pragma unroll
    for (int a = 0; a < 4; a++) q[a] = gs[3 + a];
    const int status = fuse_finish(gs, R4, R6, c6, cfg, delta, q, sc, true);
    store_updates(u, g, delta, q, sc, status);
  }
}

__global__ void k_triangulate_batch(const double *__restrict__ rows, const int32_t *__restrict__ nr,
                                    int64_t batch, int max_rows, double *x, int8_t *status) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double R[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) R[i][j] = 0.0;
  const int k = nr[b];
  for (int i = 0; i < k; i++) {
    double row[4];
#pragma unroll
    for (int j = 0; j < 4; j++) row[j] = rows[((int64_t)b * max_rows + i) * 4 + j];
    qr_add_row<4>(R, row);
  }
  double mean[3] = {0, 0, 0};
  bool ok = k >= 4 && triangulate_from_r(R, mean);
  status[b] = ok ? 1 : 0;
#pragma unroll
  for (int i = 0; i < 3; i++) x[3 * b + i] = ok ? mean[i] : 0.0;
}

__global__ void k_cov3d_batch(const double *__restrict__ lin, const double *__restrict__ rhs,
                              const int32_t *__restrict__ nr, int64_t batch, int max_rows,
                              double *x, int8_t *status) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double R[6][6], c[6];
#pragma unroll
  for (int i = 0; i < 6; i++) {
    c[i] = 0.0;
#pragma unroll
    for (int j = 0; j < 6; j++) R[i][j] = 0.0;
  }
  const int k = nr[b];
  for (int i = 0; i < k; i++) {
    double row[6];
#pragma unroll
    for (int j = 0; j < 6; j++) row[j] = lin[((int64_t)b * max_rows + i) * 6 + j];
    qr_add_row_rhs<6>(R, c, row, rhs[(int64_t)b * max_rows + i]);
  }
  double sol[6] = {0, 0, 0, 0, 0, 0};
  bool ok = k >= 6 && cov_from_r(R, c, sol);
  status[b] = ok ? 1 : 0;
#pragma unroll
  for (int i = 0; i < 6; i++) x[6 * b + i] = ok ? sol[i] : 0.0;
}

__global__ void k_decompose_batch(const double *__restrict__ sigma, const double *__restrict__ refq,
                                  int64_t batch, double eig_floor, double *quat, double *scale,
                                  int8_t *status) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double m[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++)
      m[i][j] = 0.5 * (sigma[9 * b + 3 * i + j] + sigma[9 * b + 3 * j + i]);
  double q[4] = {0, 0, 0, 0}, s[3] = {0, 0, 0};
  bool ok = decompose(m, refq + 4 * b, eig_floor, q, s);
  status[b] = ok ? 1 : 0;
#pragma unroll
  for (int i = 0; i < 4; i++) quat[4 * b + i] = q[i];
#pragma unroll
  for (int i = 0; i < 3; i++) scale[3 * b + i] = s[i];
}

// debug: intermediates of one Gaussian (E, ev, ref quat, covariance solution)
static inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// workspace: [counter | deferred records | 4 key/value arrays | CUB temp]
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
static size_t k4_sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, (const uint32_t *)nullptr,
                                            (uint32_t *)nullptr, (const uint32_t *)nullptr,
                                            (uint32_t *)nullptr, (int)n, 0, 8);
  return bytes;
}
size_t k4_workspace_bytes(int64_t n) {
  return 256 + align256(sizeof(K4Deferred) * (size_t)n) + 4 * align256(4 * (size_t)n) +
         align256(8 * (size_t)n) + align256(k4_sort_temp_bytes(n));
}

void launch_k4_fuse(const double *G, int64_t n, const ts_camera *cams, int V, ts_motions dense,
                    const ts_config &cfg, ts_updates u, void *workspace, cudaStream_t s,
                    const void *fits, const uint32_t *rank) {
  if (!n) return;
  const K4Motions m{dense, reinterpret_cast<const GvMotion *>(fits), rank};
  char *ws = reinterpret_cast<char *>(workspace);
  unsigned *n_defer = reinterpret_cast<unsigned *>(ws);
  K4Deferred *defer = reinterpret_cast<K4Deferred *>(ws + 256);
  char *kv = ws + 256 + align256(sizeof(K4Deferred) * (size_t)n);
  uint32_t *key = reinterpret_cast<uint32_t *>(kv), *val = key + align256(4 * (size_t)n) / 4;
  uint32_t *key2 = val + align256(4 * (size_t)n) / 4, *val2 = key2 + align256(4 * (size_t)n) / 4;
  uint64_t *mask = reinterpret_cast<uint64_t *>(val2 + align256(4 * (size_t)n) / 4);
  void *tmp = reinterpret_cast<char *>(mask) + align256(8 * (size_t)n);
  size_t tmp_bytes = k4_sort_temp_bytes(n);
  cudaMemsetAsync(n_defer, 0, sizeof(unsigned), s);
  k4_prep<<<blocks(n, 256), 256, 0, s>>>(G, n, V, m, cfg, u, key, val, mask);
  cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, key, key2, val, val2, (int)n, 0, 8,
                                            s);
  k4_fuse<<<blocks(n, 128), 128, sizeof(ts_camera) * V, s>>>(G, n, cams, V, m, cfg, u, key2, val2,
                                                              mask, defer, n_defer);
  const unsigned fin_blocks = (unsigned)std::min<int64_t>(blocks(n, 128), 148 * 4);
  k4_finish<<<fin_blocks, 128, 0, s>>>(G, cfg, u, defer, n_defer);
}
void launch_triangulate_batch(const double *rows, const int32_t *n_rows, int64_t batch,
                              int max_rows, double *x, int8_t *status, cudaStream_t s) {
  if (batch)
    k_triangulate_batch<<<blocks(batch, 128), 128, 0, s>>>(rows, n_rows, batch, max_rows, x, status);
}
void launch_cov3d_batch(const double *lin, const double *rhs, const int32_t *n_rows,
                        int64_t batch, int max_rows, double *x, int8_t *status, cudaStream_t s) {
  if (batch)
    k_cov3d_batch<<<blocks(batch, 128), 128, 0, s>>>(lin, rhs, n_rows, batch, max_rows, x, status);
}
void launch_decompose_batch(const double *sigma, const double *ref_quat, int64_t batch,
                            double eig_floor, double *quat, double *scale, int8_t *status,
                            cudaStream_t s) {
  if (batch)
    k_decompose_batch<<<blocks(batch, 128), 128, 0, s>>>(sigma, ref_quat, batch, eig_floor, quat,
                                                         scale, status);
}

}  // namespace ts
