// binning.cu -- K1: projection + exact depth order + 16x16 tile binning (sm_100a).
//
// Reference: gausstrack/splat.py:80-110 (_project_all), :131-146 (footprint), :171-180 (order).
// The reference has no tiles; a pixel's contributions are ordered by (depth, gid).  We order each
// tile's Gaussian list by the same key, so every pixel of the tile sees its Gaussians in exactly
// the reference order:
//   1. k1_project: one thread per Gaussian, looping over the V cameras (the 88-byte Gaussian is
//      read once): writes the 64-byte RasterRec, the exact f64 depth (-1 unless binned), the
//      bbox, its tile count and the 32-bit key view << b | quantised depth (b = min(28, 32 -
//      view bits)) over the view's depth range, which k1_depth_bounds reduced beforehand from
//      the means; k1_bbox_union then reduces each view's union of binned bboxes.
//   2. CUB radix sort by that key (4 passes).  The quantisation is monotone, so the order is
//      right except inside runs of equal keys; k1_fix_ties re-sorts those runs by the exact
//      (f64 depth, gid) key.
//   3. k1_emit writes one (tile, gv) instance per covered tile in that depth order (views are
//      contiguous: the view is the top field of the depth key); a stable CUB radix sort on the
//      tile id WITHIN the view (13 bits at 1352x1014: two onesweep passes instead of three for
//      the global id) then groups every tile position tile-major, views in order, each
//      (view, tile) list depth-ordered.
//   4. k1_tile_ranges marks [start, end) of every (view, tile).
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace ts {

// Quantisation of a view's depths into the key (k1_depth_keys / k1_project): (dmin, scale).
__device__ __forceinline__ double2 depth_quant(const uint32_t *drange, int v, int dbits) {
  const double dmin = (double)__uint_as_float(drange[2 * v]);
  const double dmax = (double)__uint_as_float(drange[2 * v + 1]);
  const double span = dmax - dmin;
  const double top = (double)((1u << dbits) - 2u);
  return make_double2(dmin, span > 0.0 ? top / span : 0.0);
}
// v << dbits | q for a binned depth d > 0 (clamped into [0, top]: monotone in d whatever the
// range), the sentinel 2^dbits - 1 (after every binned gv of the view, never emitted) otherwise
__device__ __forceinline__ uint32_t depth_key(double d, double2 q, uint32_t v, int dbits) {
  const uint32_t sentinel = (1u << dbits) - 1u;
  uint32_t key = v << dbits;
  if (d > 0.0) {
    const double top = (double)(sentinel - 1u);
    key |= (uint32_t)fmin(fmax((d - q.x) * q.y, 0.0), top);
  } else {
    key |= sentinel;
  }
  return key;
}

#ifndef K1_BOUNDS_PER_THREAD
#define K1_BOUNDS_PER_THREAD 4
#endif
// Per-view bounds of the in-front depths (TS_K1_FUSED_KEYS): the camera-space z of project()
// (same dot3 + add, so the same bits) for every Gaussian in front of the camera -- a superset of
// the binned ones, so the range holds every binned depth (a wider range costs key resolution,
// never order: the exact tie repair follows the sort).  Reads only the means, so k1_project
// can write the keys itself (no k1_depth_keys pass over the depths).
__global__ void __launch_bounds__(256) k1_depth_bounds(const double *__restrict__ G, int64_t n,
                                                       const ts_camera *__restrict__ cams, int V,
                                                       uint32_t *__restrict__ drange) {
  __shared__ double s_c[64][4];  // R row 2 and t[2] of each camera
  __shared__ uint32_t s_lo[64], s_hi[64];
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    s_c[i][0] = cams[i].R[6];
    s_c[i][1] = cams[i].R[7];
    s_c[i][2] = cams[i].R[8];
    s_c[i][3] = cams[i].t[2];
    s_lo[i] = 0xFFFFFFFFu;
    s_hi[i] = 0u;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // each thread holds K1_BOUNDS_PER_THREAD means, so a view's warp reduction is paid once per
  // that many Gaussians per lane
  constexpr int PT = K1_BOUNDS_PER_THREAD;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * PT;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x * PT; b < n; b += stride) {
    double m[PT][3];
    bool ok[PT];
#pragma unroll
    for (int k = 0; k < PT; k++) {
      const int64_t g = b + (int64_t)k * blockDim.x + threadIdx.x;
      ok[k] = g < n;
      m[k][0] = ok[k] ? G[11 * g] : 0.0;
      m[k][1] = ok[k] ? G[11 * g + 1] : 0.0;
      m[k][2] = ok[k] ? G[11 * g + 2] : 0.0;
    }
    for (int v = 0; v < V; v++) {
      uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
      for (int k = 0; k < PT; k++) {
        const double z = add(dot3(m[k][0], m[k][1], m[k][2], s_c[v][0], s_c[v][1], s_c[v][2]),
                             s_c[v][3]);
        if (ok[k] && z > TS_DEPTH_CUTOFF) {
          lo = min(lo, __float_as_uint(__double2float_rd(z)));
          hi = max(hi, __float_as_uint(__double2float_ru(z)));
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
      }
      if (lane == 0 && hi != 0u) {
        atomicMin(&s_lo[v], lo);
        atomicMax(&s_hi[v], hi);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    if (s_hi[i] != 0u) {
      atomicMin(&drange[2 * i], s_lo[i]);
      atomicMax(&drange[2 * i + 1], s_hi[i]);
    }
  }
}

// Per-view union of the binned bboxes only (TS_K1_FUSED_KEYS; the sentinel bbox of a
// non-binned gv has x1 < x0).
__global__ void __launch_bounds__(256) k1_bbox_union(const int16_t *__restrict__ bbox, int64_t n,
                                                     uint32_t *__restrict__ drange) {
  const int v = blockIdx.y;
  int rx0 = 0x7FFFFFFF, ry0 = 0x7FFFFFFF, rx1 = -1, ry1 = -1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const short4 b = reinterpret_cast<const short4 *>(bbox)[(int64_t)v * n + g];  // x0 x1 y0 y1
    if (b.x <= b.y) {
      rx0 = min(rx0, (int)b.x);
      rx1 = max(rx1, (int)b.y);
      ry0 = min(ry0, (int)b.z);
      ry1 = max(ry1, (int)b.w);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    rx0 = min(rx0, __shfl_xor_sync(0xffffffffu, rx0, d));
    ry0 = min(ry0, __shfl_xor_sync(0xffffffffu, ry0, d));
    rx1 = max(rx1, __shfl_xor_sync(0xffffffffu, rx1, d));
    ry1 = max(ry1, __shfl_xor_sync(0xffffffffu, ry1, d));
  }
  __shared__ int s_r[4][8];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_r[0][w] = rx0;
    s_r[1][w] = ry0;
    s_r[2][w] = rx1;
    s_r[3][w] = ry1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < nw; k++) {
      rx0 = min(rx0, s_r[0][k]);
      ry0 = min(ry0, s_r[1][k]);
      rx1 = max(rx1, s_r[2][k]);
      ry1 = max(ry1, s_r[3][k]);
    }
    if (rx1 >= 0) {
      int *r = reinterpret_cast<int *>(drange + K1_RECT_OFFSET) + 4 * v;
      atomicMin(r, rx0);
      atomicMin(r + 1, ry0);
      atomicMax(r + 2, rx1);
      atomicMax(r + 3, ry1);
    }
  }
}

#ifndef TS_K1_FUSED_KEYS
#define TS_K1_FUSED_KEYS 1  // 0: k1_depth_range + k1_depth_keys after k1_project (K1 stage cfg5 1.65 vs 1.54 ms)
#endif
#ifndef TS_K1_MIN_BLOCKS
#define TS_K1_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(128, TS_K1_MIN_BLOCKS) k1_project(const double *__restrict__ G, int64_t n,
                                                  const ts_camera *__restrict__ cams, int V,
                                                  RasterRec *__restrict__ rec,
                                                  uint32_t *__restrict__ drange,
                                                  uint32_t *__restrict__ dval,
                                                  double *__restrict__ depth64,
                                                  uint32_t *__restrict__ ntiles,
                                                  int8_t *__restrict__ status,
                                                  int16_t *__restrict__ bbox,
                                                  uint32_t *__restrict__ dkey, int dbits) {
  extern __shared__ ts_camera s_cam[];
  double *s_q = reinterpret_cast<double *>(s_cam + V);  // (dmin, scale) per view (dkey)
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    s_cam[i] = cams[i];
    if (dkey) {
      const double2 q = depth_quant(drange, i, dbits);
      s_q[2 * i] = q.x;
      s_q[2 * i + 1] = q.y;
    }
  }
  __syncthreads();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double gs[11];
#pragma unroll
  for (int k = 0; k < 11; k++) gs[k] = G[11 * g + k];
  double c3[9];
  covariance3d(gs, c3);
  for (int v = 0; v < V; v++) {
    const ts_camera &cam = s_cam[v];
    Projection p;
    project(gs, c3, cam, p);
    RasterRec r;
    int st = footprint(p, gs[10], cam.width, cam.height, r);
    int64_t gv = (int64_t)v * n + g;
    uint32_t nt = 0;
    int16_t bb[4] = {0, -1, 0, -1};
    status[gv] = (int8_t)st;
    if (st == 3) {
      r.g = (uint32_t)g;
      r.pad = 0;
      rec[gv] = r;
      nt = (uint32_t)((r.x1 / TS_TILE - r.x0 / TS_TILE + 1) *
                      (r.y1 / TS_TILE - r.y0 / TS_TILE + 1));
      bb[0] = r.x0; bb[1] = r.x1; bb[2] = r.y0; bb[3] = r.y1;
    }
    dval[gv] = (uint32_t)gv;
    depth64[gv] = st == 3 ? p.depth : -1.0;  // -1: not binned (excluded from the depth range)
    if (dkey)
      dkey[gv] = depth_key(st == 3 ? p.depth : -1.0, make_double2(s_q[2 * v], s_q[2 * v + 1]),
                           (uint32_t)v, dbits);
    ntiles[gv] = nt;
    reinterpret_cast<short4 *>(bbox)[gv] = make_short4(bb[0], bb[1], bb[2], bb[3]);
  }
}

// Per-view range of the binned depths (float bits, widened by directed rounding so that every
// double depth lies inside; depth > 1e-6 > 0, so positive-float bit order is numeric order).
// Also the per-view union of the binned bboxes (x0, y0, x1, y1 at drange + K1_RECT_OFFSET): the
// pixels K2 can read lie in the tiles it touches -- the region a host-resident track array must
// provide on the device (ts_frame_track_rects).
__global__ void __launch_bounds__(256) k1_depth_range(const double *__restrict__ depth64,
                                                      const int8_t *__restrict__ status,
                                                      const int16_t *__restrict__ bbox,
                                                      int64_t n, uint32_t *__restrict__ drange) {
  const int v = blockIdx.y;
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  int rx0 = 0x7FFFFFFF, ry0 = 0x7FFFFFFF, rx1 = -1, ry1 = -1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gv = (int64_t)v * n + g;
    const double d = depth64[gv];  // -1 unless binned (status 3): no status read
    if (d > 0.0) {
      lo = min(lo, __float_as_uint(__double2float_rd(d)));
      hi = max(hi, __float_as_uint(__double2float_ru(d)));
      const short4 b = reinterpret_cast<const short4 *>(bbox)[gv];  // x0 x1 y0 y1
      rx0 = min(rx0, (int)b.x);
      rx1 = max(rx1, (int)b.y);
      ry0 = min(ry0, (int)b.z);
      ry1 = max(ry1, (int)b.w);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    rx0 = min(rx0, __shfl_xor_sync(0xffffffffu, rx0, d));
    ry0 = min(ry0, __shfl_xor_sync(0xffffffffu, ry0, d));
    rx1 = max(rx1, __shfl_xor_sync(0xffffffffu, rx1, d));
    ry1 = max(ry1, __shfl_xor_sync(0xffffffffu, ry1, d));
  }
  // the block's warps combine in shared memory: six atomics per block
  __shared__ uint32_t s_lo[32], s_hi[32];
  __shared__ int s_r[4][32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_lo[w] = lo;
    s_hi[w] = hi;
    s_r[0][w] = rx0;
    s_r[1][w] = ry0;
    s_r[2][w] = rx1;
    s_r[3][w] = ry1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < nw; k++) {
      lo = min(lo, s_lo[k]);
      hi = max(hi, s_hi[k]);
      rx0 = min(rx0, s_r[0][k]);
      ry0 = min(ry0, s_r[1][k]);
      rx1 = max(rx1, s_r[2][k]);
      ry1 = max(ry1, s_r[3][k]);
    }
    if (lo != 0xFFFFFFFFu) atomicMin(&drange[2 * v], lo);
    if (hi != 0u) atomicMax(&drange[2 * v + 1], hi);
    if (rx1 >= 0) {
      int *r = reinterpret_cast<int *>(drange + K1_RECT_OFFSET) + 4 * v;
      atomicMin(r, rx0);
      atomicMin(r + 1, ry0);
      atomicMax(r + 2, rx1);
      atomicMax(r + 3, ry1);
    }
  }
}

// 32-bit depth keys v << b | q, q = floor((d - dmin) * (2^b - 2) / (dmax - dmin)) over the
// view's depth range: monotone in d (so the radix sort plus the exact tie repair below yields
// the reference's (depth, gid) order) and resolving 2^27-2^28 levels per view (b = min(28, 32 - view bits)) instead of the 18
// mantissa bits a truncated float key keeps (far fewer ties to repair).
__global__ void k1_depth_keys(const double *__restrict__ depth64,
                              const uint32_t *__restrict__ drange, int64_t n, int V, int dbits,
                              uint32_t *__restrict__ dkey) {
  const int64_t gv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gv >= n * V) return;
  const int v = (int)(gv / n);
  // -1 unless binned (status 3): no status read
  dkey[gv] = depth_key(depth64[gv], depth_quant(drange, v, dbits), (uint32_t)v, dbits);
}

// Re-sort runs of equal (view, quantised depth) keys by the exact (f64 depth, gid) key.  Runs
// longer than K1_TIE_RUN_MAX (planar / fronto-parallel geometry, duplicated Gaussians: the
// insertion sort would be quadratic) are listed in long_runs ([0] = count, then (start, end)
// pairs) and sorted afterwards by a segmented radix sort on the exact depth bits (api.cu).
constexpr int64_t K1_TIE_RUN_MAX = 64;
__global__ void k1_fix_ties(const uint32_t *__restrict__ key, uint32_t *__restrict__ val,
                            const double *__restrict__ depth64, int64_t M, int dbits,
                            uint32_t *__restrict__ long_runs, uint32_t long_cap) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M) return;
  const uint32_t kk = key[k];
  const uint32_t sentinel = (1u << dbits) - 1u;
  if ((kk & sentinel) == sentinel) return;
  if (k > 0 && key[k - 1] == kk) return;
  if (k + 1 >= M || key[k + 1] != kk) return;
  int64_t e = k + 1;
  while (e < M && key[e] == kk && e - k <= K1_TIE_RUN_MAX) e++;
  if (e - k > K1_TIE_RUN_MAX) {
    while (e < M && key[e] == kk) e++;
    const uint32_t i = atomicAdd(long_runs, 1u);
    if (i < long_cap) {
      long_runs[2 + 2 * i] = (uint32_t)k;
      long_runs[3 + 2 * i] = (uint32_t)e;
    }
    return;
  }
  for (int64_t i = k + 1; i < e; i++) {
    uint32_t x = val[i];
    double dx = depth64[x];
    int64_t j = i - 1;
    while (j >= k) {
      uint32_t y = val[j];
      double dy = depth64[y];
      if (dy < dx || (dy == dx && y < x)) break;
      val[j + 1] = y;
      j--;
    }
    val[j + 1] = x;
  }
}

// One warp per 32 consecutive depth-sorted gvs: their instances are one contiguous run of the
// output (exclusive scan of the counts), so the lanes write it cooperatively -- instance e of the
// run belongs to the last lane whose offset is <= e (binary search over the 32 offsets) and is
// its (k / width, k % width) tile, k = e - offset.  Coalesced stores and no per-lane loop over
// large bounding boxes (a 200-tile Gaussian no longer idles 31 lanes).
// The owner's bbox comes from the 8-byte bbox array (one sector per random gv instead of the
// record's line plus a separate count gather); its tile count is derived from it (the sentinel
// bbox {0, -1, 0, -1} of a non-binned gv gives 0 with arithmetic shifts).
__global__ void __launch_bounds__(256) k1_emit(const uint32_t *__restrict__ val,
                                               const int16_t *__restrict__ bbox,
                                               const uint32_t *__restrict__ off_sorted,
                                               int64_t M, int tiles_x,
                                               uint32_t *__restrict__ tkey,
                                               uint32_t *__restrict__ tval) {
  struct Owner {
    uint32_t off, gv;
    int16_t tx0, ty0, wt, pad;
  };
  __shared__ Owner s_own[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t c = 0, o;
  Owner me{0u, 0u, 0, 0, 1, 0};
  if (k < M) {
    me.gv = val[k];
    const short4 bb = reinterpret_cast<const short4 *>(bbox)[me.gv];  // x0 x1 y0 y1
    o = off_sorted[k];
    const int tx0 = bb.x >> 4, ty0 = bb.z >> 4, wt = (bb.y >> 4) - tx0 + 1;
    c = (uint32_t)(wt * ((bb.w >> 4) - ty0 + 1));
    me.tx0 = (int16_t)tx0;
    me.ty0 = (int16_t)ty0;
    me.wt = (int16_t)(c ? wt : 1);
  } else {
    const short4 bb = reinterpret_cast<const short4 *>(bbox)[val[M - 1]];
    o = off_sorted[M - 1] +  // past the end: offset = total
        (uint32_t)(((bb.y >> 4) - (bb.x >> 4) + 1) * ((bb.w >> 4) - (bb.z >> 4) + 1));
  }
  const uint32_t base = __shfl_sync(0xffffffffu, o, 0);
  const uint32_t end = __shfl_sync(0xffffffffu, o + c, 31);
  me.off = o - base;  // non-decreasing over the lanes; empty lanes repeat the next offset
  s_own[w][lane] = me;
  __syncwarp();
  for (uint32_t e = lane; e < end - base; e += 32) {
    int j = 0;  // last lane with off <= e: it owns instance e (empty lanes precede equal offsets)
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (s_own[w][j + step].off <= e) j += step;
    const Owner ow = s_own[w][j];
    const uint32_t kk = e - ow.off;
    const int ty = ow.ty0 + (int)(kk / (uint32_t)ow.wt), tx = ow.tx0 + (int)(kk % (uint32_t)ow.wt);
    tkey[base + e] = (uint32_t)(ty * tiles_x + tx);  // tile within the view
    tval[base + e] = ow.gv;
  }
}

// [start, end) of every (view, tile) list.  After the stable tile sort the instances are ordered
// by the composite c = tile_in_view * V + view (views in order inside a tile position, since
// the emission is view-major), so one thread per (view, tile) binary-searches the first
// instance with composite >= c and >= c + 1 (no pass over the instances).
__device__ __forceinline__ uint32_t composite(const uint32_t *tkey, const uint32_t *tval,
                                              int64_t i, double inv_n, uint32_t V) {
  // view = floor((gv + 0.5) / n) in fp64 (exact: never within 2e-10 of an integer)
  return tkey[i] * V + (uint32_t)(((double)tval[i] + 0.5) * inv_n);
}

__global__ void k1_tile_ranges(const uint32_t *__restrict__ tkey, const uint32_t *__restrict__ tval,
                               int64_t n_inst, double inv_n, int V, int tiles_per_view,
                               uint32_t *__restrict__ range) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // global tile v*tpv + t
  if (g >= (int64_t)V * tiles_per_view) return;
  const uint32_t v = (uint32_t)(g / tiles_per_view), t = (uint32_t)(g - (int64_t)v * tiles_per_view);
  const uint32_t c = t * (uint32_t)V + v;
  uint32_t out[2];
#pragma unroll
  for (int e = 0; e < 2; e++) {
    int64_t lo = 0, hi = n_inst;  // first index with composite >= c + e
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (composite(tkey, tval, mid, inv_n, (uint32_t)V) < c + (uint32_t)e) lo = mid + 1;
      else hi = mid;
    }
    out[e] = (uint32_t)lo;
  }
  reinterpret_cast<uint2 *>(range)[g] = make_uint2(out[0], out[1]);
}

// _project_all for the stage API (one view).
__global__ void k_project_view(const double *__restrict__ G, int64_t n, ts_camera cam,
                               double *__restrict__ mean2, double *__restrict__ depth,
                               double *__restrict__ cov2, uint8_t *__restrict__ in_front) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  double gs[11];
#pragma unroll
  for (int k = 0; k < 11; k++) gs[k] = G[11 * g + k];
  double c3[9];
  covariance3d(gs, c3);
  Projection p;
  project(gs, c3, cam, p);
  mean2[2 * g] = p.mean2[0];
  mean2[2 * g + 1] = p.mean2[1];
  depth[g] = p.depth;
  cov2[3 * g] = p.cov2[0];
  cov2[3 * g + 1] = p.cov2[1];
  cov2[3 * g + 2] = p.cov2[2];
  in_front[g] = p.in_front;
}

static inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__global__ void k1_range_init(uint32_t *drange, int V) {
  const int i = threadIdx.x;
  if (i < V) {
    drange[2 * i] = 0xFFFFFFFFu;
    drange[2 * i + 1] = 0u;
    int *r = reinterpret_cast<int *>(drange + K1_RECT_OFFSET) + 4 * i;
    r[0] = r[1] = 0x7FFFFFFF;
    r[2] = r[3] = -1;
  }
}

void launch_k1_project(const double *G, int64_t n, const ts_camera *cams, int V, int dbits,
                       RasterRec *rec, uint32_t *drange, uint32_t *dkey, uint32_t *dval,
                       double *depth64, uint32_t *ntiles, int8_t *status, int16_t *bbox,
                       cudaStream_t s) {
  if (n == 0) return;
  k1_range_init<<<1, 64, 0, s>>>(drange, V);
  // enough blocks per view that each thread reads ~8 gvs (16 per view was latency-bound at
  // cfg5: 0.41 ms for 48 M gvs)
  const int per_view = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (n + 2047) / 2048));
  const size_t smem = (sizeof(ts_camera) + 2 * sizeof(double)) * V;
  if (TS_K1_FUSED_KEYS) {
    // depth bounds from the means first, keys written by k1_project, bbox union afterwards
    k1_depth_bounds<<<(unsigned)std::min<int64_t>(blocks(n, 256 * K1_BOUNDS_PER_THREAD), 148 * 8),
                      256, 0, s>>>(
        G, n, cams, V, drange);
    k1_project<<<blocks(n, 128), 128, smem, s>>>(G, n, cams, V, rec, drange, dval, depth64,
                                                 ntiles, status, bbox, dkey, dbits);
    k1_bbox_union<<<dim3(per_view, V), 256, 0, s>>>(bbox, n, drange);
  } else {
    k1_project<<<blocks(n, 128), 128, smem, s>>>(G, n, cams, V, rec, drange, dval, depth64,
                                                 ntiles, status, bbox, nullptr, dbits);
    k1_depth_range<<<dim3(per_view, V), 256, 0, s>>>(depth64, status, bbox, n, drange);
    k1_depth_keys<<<blocks(n * V, 256), 256, 0, s>>>(depth64, drange, n, V, dbits, dkey);
  }
}
void launch_k1_fix_ties(const uint32_t *key, uint32_t *val, const double *depth64, int64_t M,
                        int dbits, uint32_t *long_runs, uint32_t long_cap, cudaStream_t s) {
  if (M)
    k1_fix_ties<<<blocks(M, 256), 256, 0, s>>>(key, val, depth64, M, dbits, long_runs, long_cap);
}

// Long tie runs: exact depth bits of the sorted gvs (positive depths: the bit patterns order as
// the values) and the runs' (start, end) split into two offset arrays for the segmented sort.
__global__ void k1_depth_bits(const uint32_t *__restrict__ val, const double *__restrict__ depth64,
                              int64_t M, uint64_t *__restrict__ bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) bits[i] = double_bits(depth64[val[i]]);
}
__global__ void k1_split_runs(const uint32_t *__restrict__ long_runs, uint32_t n,
                              uint32_t *__restrict__ begin, uint32_t *__restrict__ end) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    begin[i] = long_runs[2 + 2 * i];
    end[i] = long_runs[3 + 2 * i];
  }
}
void launch_k1_long_run_keys(const uint32_t *val, const double *depth64, int64_t M,
                             const uint32_t *long_runs, uint32_t n_runs, uint64_t *bits,
                             uint32_t *begin, uint32_t *end, cudaStream_t s) {
  if (M) k1_depth_bits<<<blocks(M, 256), 256, 0, s>>>(val, depth64, M, bits);
  if (n_runs) k1_split_runs<<<blocks(n_runs, 256), 256, 0, s>>>(long_runs, n_runs, begin, end);
}
void launch_k1_emit(const uint32_t *val, const int16_t *bbox, const uint32_t *off_sorted,
                    int64_t M, int tiles_x, uint32_t *tkey, uint32_t *tval, cudaStream_t s) {
  static_assert(TS_TILE == 16, "k1_emit derives tiles with >> 4");
  if (M) k1_emit<<<blocks(M, 256), 256, 0, s>>>(val, bbox, off_sorted, M, tiles_x, tkey, tval);
}
void launch_k1_tile_ranges(const uint32_t *tkey, const uint32_t *tval, int64_t n_inst, int64_t n,
                           int V, int tiles_per_view, uint32_t *range, cudaStream_t s) {
  const int64_t T = (int64_t)V * tiles_per_view;
  if (T)
    k1_tile_ranges<<<blocks(T, 256), 256, 0, s>>>(tkey, tval, n_inst, 1.0 / (double)n, V,
                                                  tiles_per_view, range);
}
void launch_project_view(const double *G, int64_t n, const ts_camera &cam, double *mean2,
                         double *depth, double *cov2, uint8_t *in_front, cudaStream_t s) {
  if (n) k_project_view<<<blocks(n, 128), 128, 0, s>>>(G, n, cam, mean2, depth, cov2, in_front);
}

}  // namespace ts
