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
//   * one-sided Jacobi SVD of R (high relative accuracy for the small singular values the
//     degeneracy tests look at), back substitution for the covariance least squares;
//   * cyclic Jacobi for the 3x3 eigenproblem, then the reference's discrete choices verbatim:
//     first-maximum permutation in itertools order, sign flips, det repair, matrix_to_quat.
#include <float.h>
#include "smallsolve.cuh"

namespace ts {


__global__ void __launch_bounds__(128, 3) k4_fuse(const double *__restrict__ G, int64_t n,
                                               const ts_camera *__restrict__ cams, int V,
                                               ts_motions m, ts_config cfg, ts_updates u) {
  extern __shared__ ts_camera s_cam4[];
  for (int i = threadIdx.x; i < V; i += blockDim.x) s_cam4[i] = cams[i];
  __syncthreads();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double gs[11];
#pragma unroll
  for (int k = 0; k < 11; k++) gs[k] = G[11 * g + k];
  double delta[3], q[4], sc[3];
  const int status = fuse_gaussian(gs, g, n, s_cam4, V, m, cfg, delta, q, sc);
#pragma unroll
  for (int i = 0; i < 3; i++) {
    u.delta_mean[3 * g + i] = delta[i];
    u.scale[3 * g + i] = sc[i];
  }
#pragma unroll
  for (int i = 0; i < 4; i++) u.rotation[4 * g + i] = q[i];
  u.status[g] = (int8_t)status;
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
__global__ void k4_debug(const double *G, int64_t n, const ts_camera *cams, int V, ts_motions m,
                         ts_config cfg, int64_t g, double *dbg) {
  double gs[11];
  for (int k = 0; k < 11; k++) gs[k] = G[11 * g + k];
  double delta[3], q[4], sc[3];
  fuse_gaussian(gs, g, n, cams, V, m, cfg, delta, q, sc, dbg);
  for (int i = 0; i < 4; i++) dbg[22 + i] = q[i];
}

static inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

void launch_k4_debug(const double *G, int64_t n, const ts_camera *cams, int V, ts_motions m,
                     const ts_config &cfg, int64_t g, double *dbg, cudaStream_t s) {
  k4_debug<<<1, 1, 0, s>>>(G, n, cams, V, m, cfg, g, dbg);
}
void launch_k4_fuse(const double *G, int64_t n, const ts_camera *cams, int V, ts_motions m,
                    const ts_config &cfg, ts_updates u, cudaStream_t s) {
  if (n) k4_fuse<<<blocks(n, 128), 128, sizeof(ts_camera) * V, s>>>(G, n, cams, V, m, cfg, u);
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
