// Host build of K4's small solvers (csrc/smallsolve.cuh) for CPU unit tests -- TEST ONLY.
// The product runs the same TS_HD code inside K4 on the GPU; this library lets the CPU suite
// check the QR / Jacobi / decomposition math against the reference fixtures without a GPU.
#include "../../paper_2604_02586_b200/csrc/smallsolve.cuh"
#include "../../paper_2604_02586_b200/csrc/rotation.cuh"

using namespace ts;

extern "C" {

int host_triangulate(const double *rows, int n_rows, double *x) {
  double R[4][4] = {};
  for (int i = 0; i < n_rows; i++) {
    double row[4] = {rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3]};
    qr_add_row<4>(R, row);
  }
  return n_rows >= 4 && triangulate_from_r(R, x);
}

int host_cov3d(const double *lin, const double *rhs, int n_rows, double *x) {
  double R[6][6] = {}, c[6] = {};
  for (int i = 0; i < n_rows; i++) {
    double row[6];
    for (int j = 0; j < 6; j++) row[j] = lin[6 * i + j];
    qr_add_row_rhs<6>(R, c, row, rhs[i]);
  }
  return n_rows >= 6 && cov_from_r(R, c, x);
}

int host_decompose(const double *sigma, const double *ref, double eig_floor, double *q,
                   double *s) {
  double m[3][3];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) m[i][j] = 0.5 * (sigma[3 * i + j] + sigma[3 * j + i]);
  return decompose(m, ref, eig_floor, q, s);
}

void host_eigh3(const double *a, double *e, double *ev) {
  double A[3][3], E[3][3], w[3];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) A[i][j] = a[3 * i + j];
  eigh3(A, E, w);
  for (int i = 0; i < 3; i++) {
    ev[i] = w[i];
    for (int j = 0; j < 3; j++) e[3 * i + j] = E[i][j];
  }
}
}

extern "C" void host_update_all(const double *G, int64_t n, const ts_camera *cams, int V,
                                const int8_t *status, const double *a, const double *b,
                                const double *w, const int32_t *cnt, const ts_config *cfg,
                                double *delta, double *q, double *s, int8_t *st) {
  ts_motions m{};
  m.status = const_cast<int8_t *>(status);
  m.a = const_cast<double *>(a);
  m.b = const_cast<double *>(b);
  m.weight_sum = const_cast<double *>(w);
  m.pixel_count = const_cast<int32_t *>(cnt);
  for (int64_t g = 0; g < n; g++)
    st[g] = (int8_t)fuse_gaussian(G + 11 * g, g, n, cams, V, m, *cfg, delta + 3 * g, q + 4 * g,
                                  s + 3 * g);
}

// rotation.cuh (regularisation helpers), host build
extern "C" void host_nearest_rotation(const double *m, double *r) { ts::nearest_rotation(m, r); }
extern "C" void host_sp_from_matrix(const double *m, double *q) { ts::sp_from_matrix(m, q); }
extern "C" void host_sp_as_euler_xyz(const double *q, double *a) { ts::sp_as_euler_XYZ(q, a); }
extern "C" void host_sp_euler_xyz_to_matrix(const double *a, double *m) {
  ts::sp_euler_XYZ_to_matrix(a, m);
}
extern "C" void host_matmul3(const double *a, const double *b, double *c) { ts::matmul3(a, b, c); }
extern "C" void host_matmul3_bt(const double *a, const double *b, double *c) {
  ts::matmul3_bt(a, b, c);
}

// the static test with and without the square root (cache.cu uses the latter)
extern "C" double host_static_sq_limit(double thr) { return ts::static_sq_limit(thr); }
extern "C" void host_static_both(const double *u, const double *v, const int32_t *px,
                                 const int32_t *py, int64_t m, double thr, uint8_t *a,
                                 uint8_t *b) {
  const double lim = ts::static_sq_limit(thr);
  for (int64_t i = 0; i < m; i++) {
    a[i] = ts::is_static(u[i], v[i], px[i], py[i], thr);
    b[i] = ts::is_static_sq(u[i], v[i], px[i], py[i], lim);
  }
}
