// solve.cu -- K3 per-(view, Gaussian) affine fit + the accumulate_view stage kernel (sm_100a).
//
// K3 (fused path): one thread per (view, Gaussian).  It sums the Gaussian's tile partials written
// by K2 in fixed instance order (deterministic), builds the anchored moment matrices
//     V1a = sum w h h^T,  V2a = sum w h x'_a^T,   h = [x - a; 1], x'_a = x' - a
// (a = integer anchor of the view bbox), applies the solve_view eligibility rule
// (motion2d.py:168-170: count >= min_pixels, sum w >= min_weight, det(V1) >= det_floor; det is
// translation invariant so it is taken on V1a), solves V1a [A^T; b_a^T] = V2a with partial-pivot LU
// (motion2d.py:173, LAPACK gesv) and maps back: b = b_a + a - A a.  Anchoring keeps V1 at
// cond ~1e2 instead of the 1e10-1e14 of absolute pixel moments.
//
// Stage accumulate_view (motion2d.py:126-161): contributions are stably sorted by Gaussian id and
// one thread per Gaussian adds them in array order with the reference's exact products
// ((w*h_i)*h_j, no FMA), so the result equals np.add.at bit-for-bit.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "motion.cuh"

namespace ts {

__device__ __forceinline__ bool finite6(const double *x) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 6; i++) ok = ok && isfinite(x[i]);
  return ok;
}

// A gv with more partial slots than this is summed by its whole warp (k3_solve).
constexpr uint32_t K3_BIG = 32;

__device__ __forceinline__ void store_motion(ts_motions m, int64_t gv, const GvMotion &r) {
  m.status[gv] = r.status;
  reinterpret_cast<double2 *>(m.a)[2 * gv] = make_double2(r.a[0], r.a[1]);
  reinterpret_cast<double2 *>(m.a)[2 * gv + 1] = make_double2(r.a[2], r.a[3]);
  reinterpret_cast<double2 *>(m.b)[gv] = make_double2(r.b[0], r.b[1]);
  m.weight_sum[gv] = r.wsum;
  m.pixel_count[gv] = (int32_t)r.count;
  if (m.static_pixel_count) m.static_pixel_count[gv] = (int32_t)r.static_count;
  if (m.static_weight_sum) m.static_weight_sum[gv] = r.static_wsum;
}

#ifndef TS_K3_MIN_BLOCKS
#define TS_K3_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(256, TS_K3_MIN_BLOCKS) k3_solve(const Partial *__restrict__ partial,
                                                const uint8_t *__restrict__ flag,
                                                const uint32_t *__restrict__ inst_base,
                                                const uint32_t *__restrict__ ntiles,
                                                const int16_t *__restrict__ bbox,
                                                int64_t NV, double det_floor, int min_pixels,
                                                double min_weight, ts_motions m) {
  const int64_t gv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool valid = gv < NV;
  // one partial slot per 8x8 quadrant of the gv's bbox (0 for the sentinel bbox of a non-binned
  // gv), starting at inst_base[gv]
  const short4 bb = valid ? reinterpret_cast<const short4 *>(bbox)[gv] : make_short4(0, -1, 0, -1);
  const uint32_t nq = (uint32_t)(((bb.y >> 3) - (bb.x >> 3) + 1) * ((bb.w >> 3) - (bb.z >> 3) + 1));
  // gvs with many slots (large bboxes) are summed by the whole warp afterwards, so one
  // straggler no longer holds its 31 neighbours (lane i takes flag words i, i+32, ...; the lanes
  // then combine in a fixed xor tree: deterministic)
  const bool big = nq > K3_BIG;
  uint32_t sb = 0;
  int ax = 0, ay = 0;
  if (nq) {
    sb = inst_base[gv];
    ax = ((int)bb.x + (int)bb.y) >> 1;
    ay = ((int)bb.z + (int)bb.w) >> 1;
  }
  if (valid && !big) {
    const GvMotion r = solve_gv(partial, flag, sb, nq, ax, ay, det_floor, min_pixels,
                                min_weight);
    store_motion(m, gv, r);
  }
  uint32_t bigmask = __ballot_sync(0xffffffffu, valid && big);
  while (bigmask) {
    const int j = __ffs(bigmask) - 1;
    bigmask &= bigmask - 1;
    const uint32_t nqj = __shfl_sync(0xffffffffu, nq, j);
    const uint32_t sbj = __shfl_sync(0xffffffffu, sb, j);
    double mom[TS_NMOM];
#pragma unroll
    for (int k = 0; k < TS_NMOM; k++) mom[k] = 0.0;
    uint32_t cnt = 0, scnt = 0;
    accumulate_slots(partial, flag, sbj, sbj + nqj, lane, 32, mom, cnt, scnt);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int k = 0; k < TS_NMOM; k++) mom[k] += __shfl_xor_sync(0xffffffffu, mom[k], d);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
      scnt += __shfl_xor_sync(0xffffffffu, scnt, d);
    }
    if (lane == j)
      store_motion(m, gv, solve_moments(mom, cnt, scnt, ax, ay, det_floor, min_pixels,
                                        min_weight));
  }
}

static inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// K3 split by K2's per-gv "touched" bytes (a gv with at least one tracked contribution).  At the
// large configs most gvs are occluded (cfg5: ~7% touched), and a warp with any touched lane
// waited on the whole bbox -> slot base -> flags -> partials chain.  Instead:
//   select + scan (CUB, api.cu): the touched gvs in gv order, and each gv's rank among them;
//   k3_solve_list: the fits of the listed gvs, written to a compact array in list order
//                  (coalesced: scattered 1-8 byte writes into the dense outputs made partial
//                  sectors and read-modify-writes);
//   k3_merge: every gv's dense motion -- its fit, or UNSOLVABLE / A = I / b = 0 / zero sums --
//             with full coalesced stores.
// Results do not depend on the split (tests compare against the oracle and across runs).
__global__ void __launch_bounds__(256) k3_merge(const uint8_t *__restrict__ touched,
                                                const uint32_t *__restrict__ rank,
                                                const GvMotion *__restrict__ fits, int64_t NV,
                                                ts_motions m) {
  const int64_t gv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gv >= NV) return;
  GvMotion r;
  if (touched[gv]) {
    r = fits[rank[gv]];
  } else {
    r.a[0] = 1.0; r.a[1] = 0.0; r.a[2] = 0.0; r.a[3] = 1.0;
    r.b[0] = 0.0; r.b[1] = 0.0;
    r.wsum = 0.0;
    r.static_wsum = 0.0;
    r.count = 0;
    r.static_count = 0;
    r.status = TS_STATUS_UNSOLVABLE;
  }
  store_motion(m, gv, r);
}

__global__ void __launch_bounds__(256, TS_K3_MIN_BLOCKS) k3_solve_list(
    const Partial *__restrict__ partial, const uint8_t *__restrict__ flag,
    const uint32_t *__restrict__ inst_base, const int16_t *__restrict__ bbox,
    const uint32_t *__restrict__ list, const uint32_t *__restrict__ n_list, double det_floor,
    int min_pixels, double min_weight, GvMotion *__restrict__ fits,
    int8_t *__restrict__ status_out) {
  const int lane = threadIdx.x & 31;
  const uint32_t nl = *n_list;
  // grid-stride over the device-side count (the grid is sized for the SMs, not the worst case)
  for (uint32_t base = blockIdx.x * blockDim.x; base < nl; base += gridDim.x * blockDim.x) {
  const uint32_t i = base + threadIdx.x;
  const bool valid = i < nl;
  const int64_t gv = valid ? (int64_t)list[i] : 0;
  const short4 bb = valid ? reinterpret_cast<const short4 *>(bbox)[gv] : make_short4(0, -1, 0, -1);
  const uint32_t nq = (uint32_t)(((bb.y >> 3) - (bb.x >> 3) + 1) * ((bb.w >> 3) - (bb.z >> 3) + 1));
  const bool big = nq > K3_BIG;
  uint32_t sb = 0;
  int ax = 0, ay = 0;
  if (nq) {
    sb = inst_base[gv];
    ax = ((int)bb.x + (int)bb.y) >> 1;
    ay = ((int)bb.z + (int)bb.w) >> 1;
  }
  if (valid && !big) {
    const GvMotion f = solve_gv(partial, flag, sb, nq, ax, ay, det_floor, min_pixels, min_weight);
    fits[i] = f;
    if (status_out) status_out[gv] = f.status;  // compact mode: the dense statuses directly
  }
  uint32_t bigmask = __ballot_sync(0xffffffffu, valid && big);
  while (bigmask) {
    const int j = __ffs(bigmask) - 1;
    bigmask &= bigmask - 1;
    const uint32_t nqj = __shfl_sync(0xffffffffu, nq, j);
    const uint32_t sbj = __shfl_sync(0xffffffffu, sb, j);
    double mom[TS_NMOM];
#pragma unroll
    for (int k = 0; k < TS_NMOM; k++) mom[k] = 0.0;
    uint32_t cnt = 0, scnt = 0;
    accumulate_slots(partial, flag, sbj, sbj + nqj, lane, 32, mom, cnt, scnt);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int k = 0; k < TS_NMOM; k++) mom[k] += __shfl_xor_sync(0xffffffffu, mom[k], d);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
      scnt += __shfl_xor_sync(0xffffffffu, scnt, d);
    }
    if (lane == j) {
      const GvMotion f = solve_moments(mom, cnt, scnt, ax, ay, det_floor, min_pixels, min_weight);
      fits[i] = f;
      if (status_out) status_out[gv] = f.status;
    }
  }
  }
}

// solve_view on absolute moments (motion2d.py:164-184).
__global__ void k_solve_abs(const double *__restrict__ v1, const double *__restrict__ v2,
                            const double *__restrict__ wsum, const int64_t *__restrict__ cnt,
                            int64_t n, double det_floor, int min_pixels, double min_weight,
                            int8_t *status, double *a, double *b, double *det_out) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double V1[3][3], X[3][2];
#pragma unroll
  for (int i = 0; i < 3; i++) {
#pragma unroll
    for (int j = 0; j < 3; j++) V1[i][j] = v1[9 * g + 3 * i + j];
#pragma unroll
    for (int j = 0; j < 2; j++) X[i][j] = v2[6 * g + 2 * i + j];
  }
  const double det = lu3_solve(V1, X);
  if (det_out) det_out[g] = det;
  bool ok = cnt[g] >= min_pixels && wsum[g] >= min_weight && det >= det_floor;
  double res[6] = {X[0][0], X[1][0], X[0][1], X[1][1], X[2][0], X[2][1]};
  ok = ok && finite6(res);
  status[g] = ok ? TS_STATUS_SOLVED : TS_STATUS_UNSOLVABLE;
  a[4 * g] = ok ? res[0] : 1.0;
  a[4 * g + 1] = ok ? res[1] : 0.0;
  a[4 * g + 2] = ok ? res[2] : 0.0;
  a[4 * g + 3] = ok ? res[3] : 1.0;
  b[2 * g] = ok ? res[4] : 0.0;
  b[2 * g + 1] = ok ? res[5] : 0.0;
}

__global__ void k_segment_bounds(const uint32_t *__restrict__ sorted_gid, int64_t m,
                                 uint32_t *__restrict__ seg_start, uint32_t *__restrict__ seg_end) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint32_t g = sorted_gid[i];
  if (i == 0 || sorted_gid[i - 1] != g) seg_start[g] = (uint32_t)i;
  if (i == m - 1 || sorted_gid[i + 1] != g) seg_end[g] = (uint32_t)(i + 1);
}

template <typename TrackT>
__global__ void k_accumulate_segments(int64_t n, const uint32_t *__restrict__ seg_start,
                                      const uint32_t *__restrict__ seg_end,
                                      const uint32_t *__restrict__ order,
                                      const int32_t *__restrict__ px, const int32_t *__restrict__ py,
                                      const double *__restrict__ alpha,
                                      const double *__restrict__ trans, int W,
                                      const TrackT *__restrict__ target,
                                      const uint8_t *__restrict__ valid, double thr, double *v1,
                                      double *v2, double *wsum, int64_t *cnt, int64_t *scnt,
                                      double *swsum) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double s1[9], s2[6], sw = 0.0, ssw = 0.0;
  int64_t c = 0, sc = 0;
#pragma unroll
  for (int k = 0; k < 9; k++) s1[k] = 0.0;
#pragma unroll
  for (int k = 0; k < 6; k++) s2[k] = 0.0;
  const uint32_t s = seg_start[g], e = seg_end[g];
  for (uint32_t i = s; i < e; i++) {
    const uint32_t k = order[i];
    const int x = px[k], y = py[k];
    const int64_t pix = (int64_t)y * W + x;
    if (!valid[pix]) continue;
    const double xp0 = (double)target[2 * pix], xp1 = (double)target[2 * pix + 1];
    const double w = mul(alpha[k], trans[k]);
    const double h[3] = {(double)x, (double)y, 1.0};
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double wh = mul(w, h[a]);
#pragma unroll
      for (int b = 0; b < 3; b++) s1[3 * a + b] = add(s1[3 * a + b], mul(wh, h[b]));
      s2[2 * a] = add(s2[2 * a], mul(wh, xp0));
      s2[2 * a + 1] = add(s2[2 * a + 1], mul(wh, xp1));
    }
    sw = add(sw, w);
    c++;
    if (is_static(xp0, xp1, x, y, thr)) {
      sc++;
      ssw = add(ssw, w);
    }
  }
#pragma unroll
  for (int k = 0; k < 9; k++) v1[9 * g + k] = s1[k];
#pragma unroll
  for (int k = 0; k < 6; k++) v2[6 * g + k] = s2[k];
  wsum[g] = sw;
  cnt[g] = c;
  scnt[g] = sc;
  swsum[g] = ssw;
}


size_t k3_fit_bytes() { return sizeof(GvMotion); }

void launch_k3_merge(const uint8_t *touched, const uint32_t *rank, const void *fits,
                     int64_t nv_total, ts_motions m, cudaStream_t s) {
  if (!nv_total) return;
  k3_merge<<<blocks(nv_total, 256), 256, 0, s>>>(touched, rank,
                                                 reinterpret_cast<const GvMotion *>(fits),
                                                 nv_total, m);
}

void launch_k3_solve(const Partial *partial, const uint8_t *flag, const uint32_t *inst_base,
                     const uint32_t *ntiles, const int16_t *bbox, int64_t nv_total,
                     const ts_config &cfg, ts_motions m, const uint8_t *touched,
                     const uint32_t *list, const uint32_t *n_list, const uint32_t *rank,
                     void *fits, cudaStream_t s, bool status_only) {
  if (!nv_total) return;
  if (!touched) {  // every gv walks its flags
    k3_solve<<<blocks(nv_total, 256), 256, 0, s>>>(partial, flag, inst_base, ntiles, bbox, nv_total,
                                                   cfg.det_floor, cfg.min_pixels, cfg.min_weight,
                                                   m);
    return;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(blocks(nv_total, 256), (int64_t)sms * 8);
  GvMotion *f = reinterpret_cast<GvMotion *>(fits);
  // status_only: the solve writes the statuses of the listed gvs over an UNSOLVABLE fill (K4
  // reads the rest from the compact fits); otherwise the merge writes every dense motion
  if (status_only) cudaMemsetAsync(m.status, TS_STATUS_UNSOLVABLE, (size_t)nv_total, s);
  k3_solve_list<<<(unsigned)grid, 256, 0, s>>>(partial, flag, inst_base, bbox, list, n_list,
                                               cfg.det_floor, cfg.min_pixels, cfg.min_weight, f,
                                               status_only ? m.status : nullptr);
  if (!status_only) launch_k3_merge(touched, rank, f, nv_total, m, s);
}

void launch_solve_abs(const double *v1, const double *v2, const double *wsum, const int64_t *cnt,
                      int64_t n, double det_floor, int min_pixels, double min_weight,
                      int8_t *status, double *a, double *b, double *det, cudaStream_t s) {
  if (n)
    k_solve_abs<<<blocks(n, 256), 256, 0, s>>>(v1, v2, wsum, cnt, n, det_floor, min_pixels,
                                               min_weight, status, a, b, det);
}

void launch_segment_bounds(const uint32_t *sorted_gid, int64_t m, uint32_t *seg_start,
                           uint32_t *seg_end, cudaStream_t s) {
  if (m) k_segment_bounds<<<blocks(m, 256), 256, 0, s>>>(sorted_gid, m, seg_start, seg_end);
}

void launch_accumulate(int64_t n, const uint32_t *seg_start, const uint32_t *seg_end,
                       const uint32_t *order, const int32_t *px, const int32_t *py,
                       const double *alpha, const double *trans, int W, const void *target,
                       int track_dtype, const uint8_t *valid, double thr, double *v1, double *v2,
                       double *wsum, int64_t *cnt, int64_t *scnt, double *swsum, cudaStream_t s) {
  if (!n) return;
  if (track_dtype == TS_TRACK_F32)
    k_accumulate_segments<float><<<blocks(n, 128), 128, 0, s>>>(
        n, seg_start, seg_end, order, px, py, alpha, trans, W,
        reinterpret_cast<const float *>(target), valid, thr, v1, v2, wsum, cnt, scnt, swsum);
  else
    k_accumulate_segments<double><<<blocks(n, 128), 128, 0, s>>>(
        n, seg_start, seg_end, order, px, py, alpha, trans, W,
        reinterpret_cast<const double *>(target), valid, thr, v1, v2, wsum, cnt, scnt, swsum);
}

}  // namespace ts
