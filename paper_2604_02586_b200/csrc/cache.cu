// cache.cu -- the clip contribution cache (sm_100a): the GPU form of the reference's frame-0
// weight-map reuse across a clip's target frames (pipeline.py:191-196,
// compensate_frame(weightmaps=...) pipeline.py:110-116).
//
// Once per clip (ts_frame_cache): K2 in K2_CACHE mode rasterizes the binning WITHOUT tracks and
// leaves one CacheRec per (gv, 8x8 quadrant) slot with kept contributions (raster.cu), their
// w = alpha T values in warp-chunked pool order.  The records are then laid out in slot order --
// every gv's slots are consecutive (inst_base[gv] + q), so every gv's contributions become one
// contiguous run:
//   cw[k]  (f64)  w of contribution k,   cxy[k] (u32)  its pixel x | y << 16,
//   ranges[i] = [begin, end) of the i-th touched gv (list order, the K3 list).
// 12 B per contribution, read once per target frame with unit stride.
//
// Per target frame (k23_cached): the moment stage of K2 and the fit of K3 in one kernel -- the
// track of every cached contribution (kept only where valid, motion2d.py:144-160; static test
// motion2d.py:158, without the square root: is_static_sq), the anchored moments, then
// solve_moments (motion2d.py:164-184) -- with no rasterization and no Partial round trip through
// HBM.  Work units are chunks of at most KC_CHUNK contributions of one gv (built once per clip,
// with the gv's anchor and view): a warp loads 32 chunk headers at once, four lanes per chunk
// stride over its run (coalesced, four contributions per lane in flight), two xor-shuffle levels,
// the reduced moments are staged in shared memory and each lane then solves the chunk it loaded
// when that chunk is its gv's whole run; the chunks of longer runs go to a scratch array that
// k23_cached_multi sums in order (one warp per gv).  Fits go to the compact list-order array;
// k3_merge writes the dense motions.  Deterministic (fixed order); sums differ from the per-frame
// path only by summation order.
//
// Measured (cfg2, 87 M cached contributions, tools/r2_cacheab.sh): 4 lanes x 4 in flight at 80
// registers (3 CTAs/SM) 0.82 ms; 2 x 8 at 128 registers 0.88; 1 block/SM (154 registers) or
// chunks of 32 (more split gvs) 1.5-2.3 ms; per-round header loads instead of per-batch 0.93.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "motion.cuh"

namespace ts {

namespace {

unsigned sm_grid(int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (unsigned)(sms * per_sm);
}

// one thread per record: the slot's contribution count (records with mask 0 were reserved by a
// K2 warp and never filled)
__global__ void cache_slot_counts(const CacheRec *__restrict__ recs,
                                  const unsigned long long *__restrict__ n_recs, uint64_t rec_cap,
                                  uint32_t *__restrict__ slot_cnt) {
  const uint64_t nr = min((uint64_t)*n_recs, rec_cap);
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t mask = recs[r].mask;
    if (mask) slot_cnt[recs[r].slot] = (uint32_t)__popcll(mask);
  }
}

// one warp per record: lane l handles pixel bits l and l + 32; the pool holds a record's values in
// ascending bit order, so the rank of a set bit is its index in both runs (eight lanes per
// record, four records per warp, measured 1.58 vs 1.44 ms at cfg5)
__global__ void cache_scatter(const CacheRec *__restrict__ recs,
                              const unsigned long long *__restrict__ n_recs, uint64_t rec_cap,
                              const double *__restrict__ pool, const uint32_t *__restrict__ slot_off,
                              double *__restrict__ cw, uint32_t *__restrict__ cxy) {
  const int lane = threadIdx.x & 31;
  const uint64_t nr = min((uint64_t)*n_recs, rec_cap);
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr; r += warps) {
    const CacheRec rec = recs[r];
    if (!rec.mask) continue;
    const uint32_t dst = slot_off[rec.slot];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int p = lane + 32 * h;
      if (!((rec.mask >> p) & 1ull)) continue;
      const uint32_t rank = (uint32_t)__popcll(rec.mask & ((1ull << p) - 1ull));
      cw[dst + rank] = pool[(uint64_t)rec.offset + rank];
      cxy[dst + rank] = (uint32_t)(rec.qx0 + (p & 7)) | ((uint32_t)(rec.qy0 + (p >> 3)) << 16);
    }
  }
}

__device__ __forceinline__ uint32_t gv_quadrants(short4 bb) {
  return (uint32_t)(((bb.y >> 3) - (bb.x >> 3) + 1) * ((bb.w >> 3) - (bb.z >> 3) + 1));
}

__global__ void cache_ranges(const uint32_t *__restrict__ list, const uint32_t *__restrict__ n_list,
                             const int16_t *__restrict__ bbox,
                             const uint32_t *__restrict__ inst_base,
                             const uint32_t *__restrict__ slot_off, uint2 *__restrict__ ranges) {
  const uint32_t nl = *n_list;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    const uint32_t gv = list[i];
    const short4 bb = reinterpret_cast<const short4 *>(bbox)[gv];
    const uint32_t sb = inst_base[gv];
    ranges[i] = make_uint2(slot_off[sb], slot_off[sb + gv_quadrants(bb)]);
  }
}

// Work units of the per-frame kernel: runs of at most KC_CHUNK contributions of one gv, so a
// gv covering thousands of pixels does not serialise one group of lanes.
struct __align__(16) CacheChunk {
  uint32_t i;     // index in the touched list
  uint32_t beg, end;
  uint32_t part;  // KC_WHOLE: the gv's only chunk (solved in place); else its scratch slot
  int32_t ax, ay;  // the gv's anchor (integer bbox centre, as K2/K3)
  uint32_t view, gv;
};
constexpr uint32_t KC_WHOLE = 0xFFFFFFFFu;
#ifndef TS_KC_CHUNK  // build-time overrides for variant experiments (tools/r2_libab.sh)
#define TS_KC_CHUNK 128
#endif
#ifndef TS_KC_LANES
#define TS_KC_LANES 4
#endif
#ifndef TS_KC_UNROLL
#define TS_KC_UNROLL 4
#endif
#ifndef TS_KC_MIN_BLOCKS
#define TS_KC_MIN_BLOCKS 3
#endif
constexpr int KC_CHUNK = TS_KC_CHUNK;
constexpr int KC_WARPS = 8;                // warps per CTA
constexpr int KC_LANES = TS_KC_LANES;      // lanes per chunk in the moment stage
constexpr int KC_UNROLL = TS_KC_UNROLL;    // contributions per lane in flight
constexpr int KC_STAGE = TS_NMOM + 1;  // staged doubles per chunk: moments + (count, static count)

struct MultiGv {
  uint32_t i, part, n;  // list index, first scratch slot, chunks
};

__global__ void cache_chunk_counts(const uint32_t *__restrict__ n_list,
                                   const uint2 *__restrict__ ranges, uint32_t *__restrict__ nch) {
  const uint32_t nl = *n_list;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    const uint2 r = ranges[i];
    nch[i] = (r.y - r.x + KC_CHUNK - 1) / KC_CHUNK;
  }
}

// counters: [0] chunks, [1] scratch slots handed out, [2] multi-chunk gvs
__global__ void cache_chunk_fill(const uint32_t *__restrict__ list,
                                 const uint32_t *__restrict__ n_list,
                                 const int16_t *__restrict__ bbox, int64_t n,
                                 const uint2 *__restrict__ ranges,
                                 const uint32_t *__restrict__ nch,
                                 const uint32_t *__restrict__ choff, CacheChunk *__restrict__ chunks,
                                 MultiGv *__restrict__ multi, uint32_t *__restrict__ counters) {
  const uint32_t nl = *n_list;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += gridDim.x * blockDim.x) {
    const uint2 r = ranges[i];
    const uint32_t k = nch[i], c0 = choff[i];
    if (i == nl - 1) counters[0] = c0 + k;
    uint32_t part = KC_WHOLE;
    if (k > 1) {
      part = atomicAdd(counters + 1, k);
      multi[atomicAdd(counters + 2, 1u)] = MultiGv{i, part, k};
    }
    const uint32_t gv = list[i];
    const short4 bb = reinterpret_cast<const short4 *>(bbox)[gv];
    const int ax = ((int)bb.x + (int)bb.y) >> 1, ay = ((int)bb.z + (int)bb.w) >> 1;
    for (uint32_t c = 0; c < k; c++) {
      const uint32_t b = r.x + c * KC_CHUNK;
      chunks[c0 + c] = CacheChunk{i, b, min(b + (uint32_t)KC_CHUNK, r.y),
                                  part == KC_WHOLE ? KC_WHOLE : part + c, ax, ay,
                                  (uint32_t)(gv / n), gv};
    }
  }
}

template <typename TrackT>
__device__ __forceinline__ void kc_add(double (&m)[TS_NMOM], uint32_t &cnt, uint32_t &scnt,
                                       double w, int px, int py, int ax, int ay, double fax,
                                       double fay, TrackT tu, TrackT tv, double static_lim) {
  const double u = (double)tu, vv = (double)tv;
  const double dx = (double)(px - ax), dy = (double)(py - ay);
  const double ua = u - fax, va = vv - fay;
  const double wx = w * dx, wy = w * dy;
  m[0] += w;
  m[1] += wx;
  m[2] += wy;
  m[3] += wx * dx;
  m[4] += wx * dy;
  m[5] += wy * dy;
  m[6] += w * ua;
  m[7] += w * va;
  m[8] += wx * ua;
  m[9] += wx * va;
  m[10] += wy * ua;
  m[11] += wy * va;
  const bool st = is_static_sq(u, vv, px, py, static_lim);
  m[12] += st ? w : 0.0;
  scnt += st;
  cnt++;
}

__device__ __forceinline__ void gv_anchor(const int16_t *bbox, uint32_t gv, int &ax, int &ay) {
  const short4 bb = reinterpret_cast<const short4 *>(bbox)[gv];
  ax = ((int)bb.x + (int)bb.y) >> 1;
  ay = ((int)bb.z + (int)bb.w) >> 1;
}

template <typename TrackT>
__global__ void __launch_bounds__(KC_WARPS * 32, TS_KC_MIN_BLOCKS) k23_cached(
    const CacheChunk *__restrict__ chunks, const uint32_t *__restrict__ counters,
    const uint32_t *__restrict__ list, const int16_t *__restrict__ bbox, int64_t n, int W, int H,
    const double *__restrict__ cw, const uint32_t *__restrict__ cxy,
    const TrackT *__restrict__ tgt, const uint8_t *__restrict__ val, double static_lim,
    double det_floor, int min_pixels, double min_weight, GvMotion *__restrict__ fits,
    double *__restrict__ scratch, int8_t *__restrict__ status_out) {
  __shared__ double stage[KC_WARPS][32][KC_STAGE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / KC_LANES, gl = lane % KC_LANES;
  constexpr int PER_ROUND = 32 / KC_LANES;
  const uint32_t nc = counters[0];
  const uint32_t step = gridDim.x * KC_WARPS * 32;
  for (uint32_t base = (blockIdx.x * KC_WARPS + warp) * 32; base < nc; base += step) {
    // the batch's 32 chunk headers in one coalesced load; each round takes its own by shuffle
    CacheChunk mine{};
    if (base + lane < nc) mine = chunks[base + lane];
    for (int round = 0; round < 32 / PER_ROUND; round++) {
      const int slot = round * PER_ROUND + grp;
      const uint32_t beg = __shfl_sync(0xffffffffu, mine.beg, slot);
      const uint32_t end = __shfl_sync(0xffffffffu, mine.end, slot);
      const int ax = __shfl_sync(0xffffffffu, mine.ax, slot);
      const int ay = __shfl_sync(0xffffffffu, mine.ay, slot);
      const uint32_t view = __shfl_sync(0xffffffffu, mine.view, slot);
      double m[TS_NMOM];
#pragma unroll
      for (int q = 0; q < TS_NMOM; q++) m[q] = 0.0;
      uint32_t cnt = 0, scnt = 0;
      const double fax = (double)ax, fay = (double)ay;
      const int64_t vbase = (int64_t)view * H * W;
      // KC_UNROLL contributions per lane per iteration: every load issued before any is used;
      // invalid targets may be NaN -- read, never used
      for (uint32_t k0 = beg + gl; k0 < end; k0 += KC_LANES * KC_UNROLL) {
        double w[KC_UNROLL];
        int x[KC_UNROLL], y[KC_UNROLL];
        uint8_t ok[KC_UNROLL];
        TrackT tu[KC_UNROLL], tv[KC_UNROLL];
#pragma unroll
        for (int j = 0; j < KC_UNROLL; j++) {
          const uint32_t k = k0 + j * KC_LANES;
          const uint32_t kk = k < end ? k : k0;
          w[j] = cw[kk];
          const uint32_t xy = cxy[kk];
          x[j] = (int)(xy & 0xffffu);
          y[j] = (int)(xy >> 16);
        }
#pragma unroll
        for (int j = 0; j < KC_UNROLL; j++) {
          const int64_t p = vbase + (int64_t)y[j] * W + x[j];
          ok[j] = (k0 + j * KC_LANES < end) ? val[p] : (uint8_t)0;
          tu[j] = tgt[2 * p];
          tv[j] = tgt[2 * p + 1];
        }
#pragma unroll
        for (int j = 0; j < KC_UNROLL; j++)
          if (ok[j])
            kc_add(m, cnt, scnt, w[j], x[j], y[j], ax, ay, fax, fay, tu[j], tv[j], static_lim);
      }
#pragma unroll
      for (int d = 1; d < KC_LANES; d <<= 1) {
#pragma unroll
        for (int q = 0; q < TS_NMOM; q++) m[q] += __shfl_xor_sync(0xffffffffu, m[q], d);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
        scnt += __shfl_xor_sync(0xffffffffu, scnt, d);
      }
      if (gl == 0) {
        double *st = stage[warp][slot];
#pragma unroll
        for (int q = 0; q < TS_NMOM; q++) st[q] = m[q];
        st[TS_NMOM] = __hiloint2double((int)scnt, (int)cnt);
      }
    }
    __syncwarp();
    if (base + lane < nc) {
      const double *st = stage[warp][lane];
      if (mine.part == KC_WHOLE) {
        double m[TS_NMOM];
#pragma unroll
        for (int q = 0; q < TS_NMOM; q++) m[q] = st[q];
        const uint32_t cnt = (uint32_t)__double2loint(st[TS_NMOM]);
        const uint32_t scnt = (uint32_t)__double2hiint(st[TS_NMOM]);
        const GvMotion f =
            solve_moments(m, cnt, scnt, mine.ax, mine.ay, det_floor, min_pixels, min_weight);
        fits[mine.i] = f;
        if (status_out) status_out[mine.gv] = f.status;
      } else {
        double *dst = scratch + (size_t)mine.part * KC_STAGE;
#pragma unroll
        for (int q = 0; q < KC_STAGE; q++) dst[q] = st[q];
      }
    }
    __syncwarp();
  }
}

// The gvs split into several chunks: one warp each sums its chunk moments (fixed order) and solves.
__global__ void __launch_bounds__(256) k23_cached_multi(
    const MultiGv *__restrict__ multi, const uint32_t *__restrict__ counters,
    const uint32_t *__restrict__ list, const int16_t *__restrict__ bbox,
    const double *__restrict__ scratch, double det_floor, int min_pixels, double min_weight,
    GvMotion *__restrict__ fits, int8_t *__restrict__ status_out) {
  const int lane = threadIdx.x & 31;
  const uint32_t nm = counters[2];
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < nm; j += warps) {
    const MultiGv g = multi[j];
    double m[TS_NMOM];
#pragma unroll
    for (int q = 0; q < TS_NMOM; q++) m[q] = 0.0;
    uint32_t cnt = 0, scnt = 0;
    for (uint32_t c = lane; c < g.n; c += 32) {
      const double *src = scratch + (size_t)(g.part + c) * KC_STAGE;
#pragma unroll
      for (int q = 0; q < TS_NMOM; q++) m[q] += src[q];
      cnt += (uint32_t)__double2loint(src[TS_NMOM]);
      scnt += (uint32_t)__double2hiint(src[TS_NMOM]);
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int q = 0; q < TS_NMOM; q++) m[q] += __shfl_xor_sync(0xffffffffu, m[q], d);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
      scnt += __shfl_xor_sync(0xffffffffu, scnt, d);
    }
    if (lane == 0) {
      int ax, ay;
      const uint32_t gv = list[g.i];
      gv_anchor(bbox, gv, ax, ay);
      const GvMotion f = solve_moments(m, cnt, scnt, ax, ay, det_floor, min_pixels, min_weight);
      fits[g.i] = f;
      if (status_out) status_out[gv] = f.status;
    }
  }
}

}  // namespace

// n_hint: the record count read back by the build (sizes the grid: one thread -- or one lane
// group -- per record, so the dependent loads of all records are in flight at once; the
// grid-stride loops cover any remainder)
void launch_cache_slot_counts(const CacheRec *recs, const unsigned long long *n_recs,
                              uint64_t rec_cap, uint32_t *slot_cnt, cudaStream_t s,
                              uint64_t n_hint) {
  const uint64_t want = (std::min(n_hint, rec_cap) + 255) / 256;
  cache_slot_counts<<<(unsigned)std::max<uint64_t>(std::min<uint64_t>(want, 1u << 20), 1), 256, 0,
                      s>>>(recs, n_recs, rec_cap, slot_cnt);
}

void launch_cache_scatter(const CacheRec *recs, const unsigned long long *n_recs, uint64_t rec_cap,
                          const double *pool, const uint32_t *slot_off, double *cw, uint32_t *cxy,
                          cudaStream_t s, uint64_t n_hint) {
  // eight CTAs per SM, grid-stride: a warp per record over the whole record count measured
  // 1.75 vs 1.44 ms at cfg5 (the scattered run writes thrash)
  (void)n_hint;
  cache_scatter<<<sm_grid(8), 256, 0, s>>>(recs, n_recs, rec_cap, pool, slot_off, cw, cxy);
}

void launch_cache_ranges(const uint32_t *list, const uint32_t *n_list, int64_t nv_total,
                         const int16_t *bbox, const uint32_t *inst_base, const uint32_t *slot_off,
                         uint2 *ranges, cudaStream_t s) {
  if (!nv_total) return;
  const unsigned grid = (unsigned)std::min<int64_t>((nv_total + 255) / 256, sm_grid(8));
  cache_ranges<<<grid, 256, 0, s>>>(list, n_list, bbox, inst_base, slot_off, ranges);
}

size_t cache_chunk_bytes() { return sizeof(CacheChunk); }
size_t cache_multi_bytes() { return sizeof(MultiGv); }
size_t cache_scratch_bytes() { return sizeof(double) * KC_STAGE; }
int cache_chunk_len() { return KC_CHUNK; }

void launch_cache_chunk_counts(const uint32_t *n_list, int64_t nv_total, const uint2 *ranges,
                               uint32_t *nch, cudaStream_t s) {
  if (!nv_total) return;
  const unsigned grid = (unsigned)std::min<int64_t>((nv_total + 255) / 256, sm_grid(8));
  cache_chunk_counts<<<grid, 256, 0, s>>>(n_list, ranges, nch);
}

void launch_cache_chunk_fill(const uint32_t *list, const uint32_t *n_list, int64_t nv_total,
                             const int16_t *bbox, int64_t n, const uint2 *ranges,
                             const uint32_t *nch, const uint32_t *choff, void *chunks, void *multi,
                             uint32_t *counters, cudaStream_t s) {
  if (!nv_total) return;
  const unsigned grid = (unsigned)std::min<int64_t>((nv_total + 255) / 256, sm_grid(8));
  cache_chunk_fill<<<grid, 256, 0, s>>>(list, n_list, bbox, n, ranges, nch, choff,
                                        reinterpret_cast<CacheChunk *>(chunks),
                                        reinterpret_cast<MultiGv *>(multi), counters);
}

cudaError_t launch_k23_cached(const void *chunks, const uint32_t *counters, uint64_t chunk_bound,
                              const void *multi, uint64_t multi_bound, const uint32_t *list,
                              const int16_t *bbox, int64_t n, int W, int H, const double *cw,
                              const uint32_t *cxy, const void *track_target, int track_dtype,
                              const uint8_t *track_valid, const ts_config &cfg, void *fits,
                              double *scratch, cudaStream_t s, int8_t *status_out) {
  if (!chunk_bound) return cudaSuccess;
  const double lim = static_sq_limit(cfg.static_threshold_px);
  int per_sm = 0;
  const CacheChunk *ch = reinterpret_cast<const CacheChunk *>(chunks);
  GvMotion *f = reinterpret_cast<GvMotion *>(fits);
  auto grid_for = [&](const void *kern) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, KC_WARPS * 32, 0);
    return (unsigned)std::min<int64_t>((chunk_bound + KC_WARPS * 32 - 1) / (KC_WARPS * 32),
                                       sm_grid(std::max(per_sm, 1)));
  };
  if (track_dtype == TS_TRACK_F32)
    k23_cached<float><<<grid_for((const void *)k23_cached<float>), KC_WARPS * 32, 0, s>>>(
        ch, counters, list, bbox, n, W, H, cw, cxy,
        reinterpret_cast<const float *>(track_target), track_valid, lim, cfg.det_floor,
        cfg.min_pixels, cfg.min_weight, f, scratch, status_out);
  else
    k23_cached<double><<<grid_for((const void *)k23_cached<double>), KC_WARPS * 32, 0, s>>>(
        ch, counters, list, bbox, n, W, H, cw, cxy,
        reinterpret_cast<const double *>(track_target), track_valid, lim, cfg.det_floor,
        cfg.min_pixels, cfg.min_weight, f, scratch, status_out);
  if (multi_bound) {
    const unsigned g2 = (unsigned)std::min<int64_t>((multi_bound + 7) / 8, sm_grid(8));
    k23_cached_multi<<<g2, 256, 0, s>>>(reinterpret_cast<const MultiGv *>(multi), counters, list,
                                        bbox, scratch, cfg.det_floor, cfg.min_pixels,
                                        cfg.min_weight, f, status_out);
  }
  return cudaGetLastError();
}

}  // namespace ts
