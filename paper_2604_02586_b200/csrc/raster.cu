// raster.cu -- K2: tile rasterizer fused with per-Gaussian moment accumulation (sm_100a).
//
// Reference semantics: gausstrack/splat.py:147-195 (alpha, keep predicate, per-pixel
// front-to-back transmittance, early stop) fused with motion2d.py:144-160 (accumulate_view).
//
// Work decomposition.  K1 bins Gaussians into 16x16-pixel tiles, each tile's list in the
// reference order (depth, gid).  K2 is a persistent kernel whose WARPS are independent: a warp
// pulls a work item (tile, quadrant) from a global atomic queue, owns that 8x8-pixel quadrant
// (lane l holds pixels l and l+32, two independent fp64 chains for ILP) and walks the tile list
// front to back.  No block barrier in the main loop: a warp stops as soon as its 64 pixels are
// saturated (T < early_stop) and takes the next item, so occluded Gaussians cost almost nothing.
//   * Culling: per 32-instance chunk, each lane loads one record and computes the 64-bit mask of
//     quadrant pixels inside its bbox; one ballot keeps the Gaussians whose mask meets an
//     unsaturated pixel.  Per evaluated Gaussian the candidate mask (bbox AND NOT saturated) is
//     re-checked warp-uniformly, so Gaussians over saturated pixels cost a few instructions.
//   * Predicates in fp64 in the reference's operation order (bit-exact q and alpha >= cutoff;
//     T >= early_stop up to the reference's own log-cumsum rounding).
//   * Transposed accumulation: contributing lanes store w = alpha*T into a per-warp [8 x 64]
//     shared buffer; every 8 contributing Gaussians (across chunk boundaries; k2_flush), lane l
//     sums every fourth contribution of Gaussian (l & 7) in pixel order, two xor-shuffle steps
//     add the four partial sums (exactly
//     commutative pairs, so every lane holds the same bits), and the anchored moments go to the
//     (instance, quadrant) sub-slot: no atomics, no zero-initialised accumulators,
//     bit-reproducible (K3 adds the sub-slots in fixed order).
#include <cub/cub.cuh>

#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace ts {

#ifndef TS_K2_VEC_TRACKS  // 0: scalar (u, v) loads (A/B)
#define TS_K2_VEC_TRACKS 1
#endif
constexpr int K2_WARPS = 4;     // warps per CTA (independent; shared memory partitioned)
#ifndef TS_K2_FLUSH
#define TS_K2_FLUSH 8
#endif
#ifndef TS_K2_MIN_BLOCKS
#define TS_K2_MIN_BLOCKS 6
#endif
constexpr int K2_FLUSH = TS_K2_FLUSH;  // evaluated Gaussians per transposed reduction
constexpr int K2_WROW = 65;     // padded row of the w buffer (64 pixels)
constexpr int K2_ETAB_BYTES = ((TS_EXP_TABLE * 8 + 127) / 128) * 128;

struct K2Params {
  const RasterRec *rec;
  const uint32_t *inst_gv;     // sorted instances: gv
  const uint32_t *tile_range;  // [start, end) per global tile
  const uint32_t *inst_base;   // per gv: first partial slot (gv-order scan of bbox quadrant counts)
  const uint32_t *items;       // non-empty global tile ids
  const uint32_t *n_items;     // device count of items
  uint32_t *work_counter;      // zeroed before launch
  const void *track_target;    // (V, H, W, 2)
  bool track_vec;              // track_target aligned for (u, v) vector loads
  const uint8_t *track_valid;  // (V, H, W)
  int W, H, tiles_x, tiles_per_view;
  double alpha_cutoff, early_stop, static_thr;
  // accumulate mode
  Partial *partial;  // one slot per (gv, 8x8 quadrant of its bbox)
  uint8_t *flag;
  uint8_t *touched;  // per gv: 1 once it has a tracked contribution (zeroed before K2)
  // cache mode: pool of w values, its cursor (doubles handed out) and capacity; the records
  double *pool;
  unsigned long long *pool_cursor;
  uint64_t pool_cap;
  CacheRec *recs;
  unsigned long long *rec_cursor;
  uint64_t rec_cap;
  // emit mode
  unsigned long long *emit_count;
  int64_t emit_cap;
  uint64_t *emit_key;  // (pixel << 32) | sequence number within the pixel
  uint32_t *emit_gv;
  double *emit_alpha, *emit_trans;
  // dominant mode
  const double *depth64;
  int64_t *dom_gid;
  double *dom_depth;
  // optional work counters (debug; nullptr in production): see K2_STAT_*
  unsigned long long *stats;
};

// Work counters are compiled in only with -DTS_K2_STATS (they cost ~15 instructions per
// evaluated Gaussian); tools/profile_frame.py + TS_K2_STATS=1 prints them.
#ifdef TS_K2_STATS
#define K2_STATS_ON (P.stats != nullptr)
#else
#define K2_STATS_ON false
#endif

enum { K2S_UNITS, K2S_CHUNKS, K2S_INSTANCES, K2S_HITS, K2S_SKIPS, K2S_EVAL_GAUSS, K2S_EVAL_PIX,
       K2S_CONTRIB, K2S_FLUSHES, K2S_EVAL_EMPTY, K2S_N };

template <typename TrackT>
struct K2Warp {
  RasterRec rec[32];
  uint64_t rect[32];  // bbox of the record clipped to the quadrant, as a 64-pixel bit mask
  uint32_t slot[32], gvid[32];
  int2 anc[32];       // moment anchor (bbox centre pixel) of each record (accumulate mode)
  double w[K2_FLUSH][K2_WROW];
  TrackT trk_u[64], trk_v[64];  // track targets in their input precision
};

// 64-bit mask (bit = row * 8 + col) of the quadrant pixels inside the record's bbox.
__device__ __forceinline__ uint64_t quad_rect(const RasterRec &r, int qx0, int qy0) {
  const int cx0 = max((int)r.x0 - qx0, 0), cx1 = min((int)r.x1 - qx0, 7);
  const int cy0 = max((int)r.y0 - qy0, 0), cy1 = min((int)r.y1 - qy0, 7);
  if (cx0 > cx1 || cy0 > cy1) return 0ull;
  const uint64_t cols = (uint64_t)((0xFFu >> (7 - cx1)) & (0xFFu << cx0) & 0xFFu);
  const uint64_t hi = cy1 == 7 ? ~0ull : ((1ull << (8 * (cy1 + 1))) - 1ull);
  const uint64_t lo = (1ull << (8 * cy0)) - 1ull;
  return (cols * 0x0101010101010101ull) & hi & ~lo;
}

// One pixel of a lane: predicate evaluation and front-to-back compositing (splat.py:147-193).
// The pixel is saturated ("done") exactly when !(T >= early_stop): T only decreases, so no
// separate flag is kept (pixels outside the image start at T = 0).
struct PixelState {
  double T;
};

__device__ __forceinline__ bool eval_pixel(const RasterRec &r, bool cand, double fpx, double fpy,
                                           double cutoff, double early_stop, const double *etab,
                                           PixelState &ps, double &a_out, double &w_out,
                                           double &tin_out) {
  if (!cand) return false;  // outside the bbox, or already saturated
  const double dx = sub(fpx, r.mx), dy = sub(fpy, r.my);
  const double q = mahalanobis(r, dx, dy);
  if (!(q <= TS_SIGMA_RADIUS * TS_SIGMA_RADIUS)) return false;
  const double a = alpha_of_table(r.opacity, q, etab);
  if (!(a >= cutoff)) return false;
  const double tin = ps.T;
  w_out = mul(a, tin);  // motion2d.py:151
  ps.T = mul(tin, sub(1.0, a));
  a_out = a;
  tin_out = tin;
  return true;
}

// Transposed reduction of the pending Gaussians (kcount <= K2_FLUSH): lane l sums every fourth
// contributing pixel of Gaussian (l & 7), starting at its (l >> 3)-th, in pixel order; two
// xor-shuffle steps add the four partial sums ((s0 + s1) + (s2 + s3): commutative pairs, so all
// four lanes hold the same bits) and the anchored moments go to the Gaussian's (instance,
// quadrant) sub-slot.  Warp-uniform call.
template <typename TrackT>
__device__ __forceinline__ void k2_flush(const K2Warp<TrackT> &S, const K2Params &P, int lane,
                                         int kcount, uint64_t my_cm, uint32_t my_slot, int my_ax,
                                         int my_ay, uint64_t static64, int qx0, int qy0) {
  static_assert(K2_FLUSH == 4 || K2_FLUSH == 8, "flush: 4 or 8 Gaussians x 8 or 4 lanes");
  constexpr int LPG = 32 / K2_FLUSH;  // lanes per pending Gaussian
  const int kk = lane & (K2_FLUSH - 1), qq = lane / K2_FLUSH;
  double m[TS_NMOM];
#pragma unroll
  for (int q = 0; q < TS_NMOM; q++) m[q] = 0.0;
  uint32_t cnt = 0, scnt = 0;
  if (my_cm) {
    const double ax = (double)my_ax, ay = (double)my_ay;
    const double bx = (double)(qx0 - my_ax), by = (double)(qy0 - my_ay);
    // the LPG lanes of Gaussian kk take every LPG-th of its contributing pixels (lane qq starts
    // at the qq-th): balanced trip counts whatever the pixels' rows
    uint64_t bits = my_cm;
    for (int k = 0; k < qq; k++) bits &= bits - 1;
    while (bits) {
      const int p = __ffsll((long long)bits) - 1;
#pragma unroll
      for (int k = 0; k < LPG; k++) bits &= bits - 1;
      const double w = S.w[kk][p];
      const double dx = bx + (double)(p & 7), dy = by + (double)(p >> 3);
      const double ua = (double)S.trk_u[p] - ax, va = (double)S.trk_v[p] - ay;
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
      const bool st = (static64 >> p) & 1ull;
      m[12] += st ? w : 0.0;
      scnt += st;
      cnt++;
    }
  }
#pragma unroll
  for (int d = K2_FLUSH; d < 32; d <<= 1) {
#pragma unroll
    for (int q = 0; q < TS_NMOM; q++) m[q] += __shfl_xor_sync(0xffffffffu, m[q], d);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    scnt += __shfl_xor_sync(0xffffffffu, scnt, d);
  }
  if (kk < kcount && cnt > 0 && qq < 4) {
    // the four lanes of a Gaussian hold identical sums: each stores a quarter of the record
    Partial *dst = P.partial + my_slot;
    if (qq == 0) {
      dst->m[0] = m[0]; dst->m[1] = m[1]; dst->m[2] = m[2]; dst->m[3] = m[3];
    } else if (qq == 1) {
      dst->m[4] = m[4]; dst->m[5] = m[5]; dst->m[6] = m[6]; dst->m[7] = m[7];
    } else if (qq == 2) {
      dst->m[8] = m[8]; dst->m[9] = m[9]; dst->m[10] = m[10]; dst->m[11] = m[11];
    } else {
      dst->m[12] = m[12];
      dst->count = cnt;
      dst->static_count = scnt;
      P.flag[my_slot] = 1;
    }
  }
}

// Cache mode (K2_CACHE): the pending Gaussians' kept contributions -- every pixel that passed the
// keep predicate with T >= early stop, whatever the tracks -- as one CacheRec per (gv, quadrant)
// and their w values in pixel order in the pool.  The warp reserves pool space in chunks of
// K2_CACHE_CHUNK doubles and records in chunks of K2_CACHE_RECS (one atomic per chunk); record
// order does not matter (each one rewrites its own slot per frame).  Running past a capacity is
// reported by the cursor (nothing is written beyond it; the build reruns larger).  The slot
// flags (K3's "has a partial") and touched bytes are set here once for the clip.
struct CacheChunks {
  unsigned long long pool_cur = 0, pool_lim = 0, rec_cur = 0, rec_lim = 0;
};

// The unused tail of a warp's record chunk (abandoned for a fresh chunk, or left at exit) gets
// mask 0, which the per-clip layout skips: no memset of the whole record array per build.
__device__ __forceinline__ void k2_cache_clear_tail(const K2Params &P, int lane,
                                                    const CacheChunks &ch) {
  const unsigned long long lim = min(ch.rec_lim, (unsigned long long)P.rec_cap);
  for (unsigned long long r = ch.rec_cur + lane; r < lim; r += 32) P.recs[r].mask = 0ull;
}

template <typename TrackT>
__device__ __forceinline__ void k2_flush_cache(const K2Warp<TrackT> &S, const K2Params &P,
                                               int lane, int kcount, uint64_t my_cm,
                                               uint32_t my_slot, int my_ax, int my_ay, int qx0,
                                               int qy0, int view, CacheChunks &ch) {
  const int kk = lane & (K2_FLUSH - 1), qq = lane / K2_FLUSH;
  const uint32_t cnt = kk < kcount ? (uint32_t)__popcll(my_cm) : 0u;
  // exclusive prefix of the counts (and of the record count) over the K2_FLUSH Gaussians
  uint32_t incl = cnt, rincl = cnt ? 1u : 0u;
#pragma unroll
  for (int d = 1; d < K2_FLUSH; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
    const uint32_t ro = __shfl_up_sync(0xffffffffu, rincl, d);
    if (kk >= d) {
      incl += o;
      rincl += ro;
    }
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, K2_FLUSH - 1);
  const uint32_t rtotal = __shfl_sync(0xffffffffu, rincl, K2_FLUSH - 1);
  if (ch.pool_cur + total > ch.pool_lim) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(P.pool_cursor, (unsigned long long)K2_CACHE_CHUNK);
    ch.pool_cur = __shfl_sync(0xffffffffu, base, 0);
    ch.pool_lim = ch.pool_cur + K2_CACHE_CHUNK;
  }
  if (ch.rec_cur + rtotal > ch.rec_lim) {
    k2_cache_clear_tail(P, lane, ch);
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(P.rec_cursor, (unsigned long long)K2_CACHE_RECS);
    ch.rec_cur = __shfl_sync(0xffffffffu, base, 0);
    ch.rec_lim = ch.rec_cur + K2_CACHE_RECS;
  }
  const unsigned long long off = ch.pool_cur + (incl - cnt);
  const unsigned long long ri = ch.rec_cur + (rincl - (cnt ? 1u : 0u));
  ch.pool_cur += total;
  ch.rec_cur += rtotal;
  if (cnt && off + cnt <= P.pool_cap && ri < P.rec_cap) {
    uint64_t bits = my_cm;
    for (int k = 0; k < qq; k++) bits &= bits - 1;
    uint32_t r = qq;
    while (bits) {
      const int p = __ffsll((long long)bits) - 1;
#pragma unroll
      for (int k = 0; k < 4; k++) bits &= bits - 1;
      P.pool[off + r] = S.w[kk][p];
      r += 4;
    }
    if (qq == 0) {
      CacheRec rec;
      rec.mask = my_cm;
      rec.offset = (uint32_t)off;
      rec.slot = my_slot;
      rec.qx0 = (int16_t)qx0;
      rec.qy0 = (int16_t)qy0;
      rec.ax = (int16_t)my_ax;
      rec.ay = (int16_t)my_ay;
      rec.view = view;
      rec.pad = 0;
      P.recs[ri] = rec;
      P.flag[my_slot] = 1;
    }
  }
}

template <int MODE, typename TrackT>
__global__ void __launch_bounds__(K2_WARPS * 32, TS_K2_MIN_BLOCKS) k2_raster(const K2Params P) {
  extern __shared__ __align__(16) unsigned char k2_smem_raw[];
  double *etab = reinterpret_cast<double *>(k2_smem_raw);  // exp(-k/64), k = 0..288
  for (int k = threadIdx.x; k < TS_EXP_TABLE; k += blockDim.x) etab[k] = exp(-k / 64.0);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  K2Warp<TrackT> &S =
      reinterpret_cast<K2Warp<TrackT> *>(k2_smem_raw + K2_ETAB_BYTES)[warp];
  const uint32_t n_units = 4u * *P.n_items;
  unsigned long long st[K2S_N] = {};
  constexpr bool kSlots = MODE == K2_ACCUMULATE || MODE == K2_CACHE;
  CacheChunks cache_ch;  // cache mode: the warp's pool / record chunks

  for (;;) {
    uint32_t unit = 0;
    if (lane == 0) unit = atomicAdd(P.work_counter, 1u);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= n_units) break;
    const int tile = (int)P.items[unit >> 2];
    const int quad = (int)(unit & 3);
    const uint32_t start = P.tile_range[2 * tile], end = P.tile_range[2 * tile + 1];
    const int v = tile / P.tiles_per_view;
    const int t = tile - v * P.tiles_per_view;
    const int ty = t / P.tiles_x, tx = t - ty * P.tiles_x;
    const int qx0 = tx * TS_TILE + (quad & 1) * 8, qy0 = ty * TS_TILE + (quad >> 1) * 8;
    // lane pixels: p0 = lane (rows 0-3), p1 = lane + 32 (rows 4-7) of the 8x8 quadrant
    const int px = qx0 + (lane & 7);
    const int py0 = qy0 + (lane >> 3), py1 = py0 + 4;
    const double fpx = (double)px, fpy0 = (double)py0, fpy1 = (double)py1;
    const bool in0 = px < P.W && py0 < P.H, in1 = px < P.W && py1 < P.H;

    bool valid0 = false, valid1 = false;
    uint64_t static64 = 0;  // static-pixel bits of the unit (warp-uniform; accumulate mode)
    if (MODE == K2_ACCUMULATE) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int py = h ? py1 : py0;
        TrackT u = TrackT(0), vv = TrackT(0);
        bool val = false;
        if (h ? in1 : in0) {
          // valid byte and target issued together (one round trip: the tracks may be pinned
          // host memory read in place over PCIe, see ts_frame_compensate); plain loads, no
          // read-only-cache path, so host-mapped pages work
          const int64_t pix = ((int64_t)v * P.H + py) * P.W + px;
          const uint8_t vb = P.track_valid[pix];
          const TrackT *tg = reinterpret_cast<const TrackT *>(P.track_target) + 2 * pix;
          TrackT tu, tv;
          if (P.track_vec) {  // one 8 / 16-byte load per pixel: half the (PCIe) read requests
            using V2 = typename std::conditional<sizeof(TrackT) == 4, float2, double2>::type;
            const V2 t2 = *reinterpret_cast<const V2 *>(tg);
            tu = t2.x;
            tv = t2.y;
          } else {
            tu = tg[0];
            tv = tg[1];
          }
          val = vb != 0;
          if (val) {  // invalid targets may be NaN: never used
            u = tu;
            vv = tv;
          }
        }
        const int p = lane + 32 * h;
        S.trk_u[p] = u;
        S.trk_v[p] = vv;
        const bool st = val && is_static((double)u, (double)vv, px, py, P.static_thr);
        static64 |= (uint64_t)__ballot_sync(0xffffffffu, st) << (32 * h);
        if (h) valid1 = val; else valid0 = val;
      }
    }
    PixelState s0{in0 ? 1.0 : 0.0};
    PixelState s1{in1 ? 1.0 : 0.0};
    uint32_t seq0 = 0, seq1 = 0;                  // emit mode
    double best_w0 = -1.0, best_w1 = -1.0;        // dominant mode
    uint32_t best_g0 = 0xFFFFFFFFu, best_g1 = 0xFFFFFFFFu, best_gv0 = 0, best_gv1 = 0;

    // saturated pixels of the quadrant (bit = row * 8 + col), warp-uniform
    uint64_t done64 = (uint64_t)__ballot_sync(0xffffffffu, !(s0.T >= P.early_stop)) |
                      ((uint64_t)__ballot_sync(0xffffffffu, !(s1.T >= P.early_stop)) << 32);
    if (K2_STATS_ON) st[K2S_UNITS]++;
    // pending Gaussians of the transposed reduction (accumulate mode): the lanes with
    // (lane & 7) == k keep Gaussian k's contribution bits of their pixel quarter, its sub-slot
    // and its anchor; a flush runs every K2_FLUSH evaluated Gaussians, across chunk boundaries
    int kpend = 0;
    uint64_t my_cm = 0;
    uint32_t my_slot = 0;
    int my_ax = 0, my_ay = 0;
    for (uint32_t b = start; b < end; b += 32) {
      if (done64 == ~0ull) break;
      if (K2_STATS_ON) {
        st[K2S_CHUNKS]++;
        st[K2S_INSTANCES] += min(32u, end - b);
      }
      // load + cull 32 instances: keep Gaussians whose bbox covers an unsaturated pixel
      const uint32_t i = b + lane;
      bool hit = false;
      __syncwarp();
      if (i < end) {
        const uint32_t gv = P.inst_gv[i];
        // the partial-slot base is loaded beside the record (not after the hit test), so the
        // chunk's dependent chain is inst_gv -> {record, slot base}
        const uint32_t ibase = kSlots ? __ldg(P.inst_base + gv) : 0u;
        const RasterRec r = P.rec[gv];
        const uint64_t rect = quad_rect(r, qx0, qy0);
        hit = (rect & ~done64) != 0ull;
        if (hit) {
          S.rec[lane] = r;
          S.rect[lane] = rect;
          S.gvid[lane] = gv;
          if (kSlots) {
            // one slot per 8x8 quadrant of the gv's bbox, row-major from its top-left quadrant
            const int bx0 = r.x0 >> 3, bx1 = r.x1 >> 3, by0 = r.y0 >> 3;
            S.slot[lane] = ibase + (uint32_t)(((qy0 >> 3) - by0) * (bx1 - bx0 + 1) +
                                              ((qx0 >> 3) - bx0));
            S.anc[lane] = make_int2(anchor_x(r), anchor_y(r));
          } else {
            S.slot[lane] = gv;
          }
        }
      }
      uint32_t mask = __ballot_sync(0xffffffffu, hit);
      if (K2_STATS_ON) st[K2S_HITS] += __popc(mask);
      __syncwarp();
      {
        while (mask) {
          const int j = __ffs(mask) - 1;
          mask &= mask - 1;
          // warp-uniform skip of Gaussians that only cover saturated pixels
          const uint64_t cand = S.rect[j] & ~done64;
          if (cand == 0ull) {
            if (K2_STATS_ON) st[K2S_SKIPS]++;
            continue;
          }
          if (K2_STATS_ON) {
            st[K2S_EVAL_GAUSS]++;
            st[K2S_EVAL_PIX] += __popcll(cand);
          }
          const RasterRec r = S.rec[j];
          double a0 = 0, w0 = 0, t0 = 0, a1 = 0, w1 = 0, t1 = 0;
          const bool c0 = eval_pixel(r, (cand >> lane) & 1ull, fpx, fpy0, P.alpha_cutoff,
                                     P.early_stop, etab, s0, a0, w0, t0);
          const bool c1 = eval_pixel(r, (cand >> (lane + 32)) & 1ull, fpx, fpy1, P.alpha_cutoff,
                                     P.early_stop, etab, s1, a1, w1, t1);
          done64 = (uint64_t)__ballot_sync(0xffffffffu, !(s0.T >= P.early_stop)) |
                   ((uint64_t)__ballot_sync(0xffffffffu, !(s1.T >= P.early_stop)) << 32);
          if (kSlots) {
            // accumulate: tracked contributions; cache: every kept contribution (the tracks of
            // the clip's target frames are applied per frame from the cache)
            const bool k0 = c0 && (MODE == K2_CACHE || valid0);
            const bool k1 = c1 && (MODE == K2_CACHE || valid1);
            const uint32_t cm0 = __ballot_sync(0xffffffffu, k0);
            const uint32_t cm1 = __ballot_sync(0xffffffffu, k1);
            if (K2_STATS_ON) {
              st[K2S_CONTRIB] += __popc(cm0) + __popc(cm1);
              // evaluated but no pixel composited (bbox corner only: outside the ellipse)
              if (!__any_sync(0xffffffffu, c0 || c1)) st[K2S_EVAL_EMPTY]++;
            }
            if (cm0 | cm1) {  // Gaussians without a tracked contribution need no flush slot
              if (lane == 0 && P.touched) P.touched[S.gvid[j]] = 1;
              if (k0) S.w[kpend][lane] = w0;
              if (k1) S.w[kpend][lane + 32] = w1;
              if ((lane & (K2_FLUSH - 1)) == kpend) {  // this Gaussian's flush lanes
                my_cm = (uint64_t)cm0 | ((uint64_t)cm1 << 32);
                my_slot = S.slot[j];
                const int2 an = S.anc[j];
                my_ax = an.x;
                my_ay = an.y;
              }
              if (++kpend == K2_FLUSH) {
                __syncwarp();
                if (K2_STATS_ON) st[K2S_FLUSHES]++;
                if (MODE == K2_CACHE)
                  k2_flush_cache(S, P, lane, kpend, my_cm, my_slot, my_ax, my_ay, qx0, qy0, v,
                                 cache_ch);
                else
                  k2_flush(S, P, lane, kpend, my_cm, my_slot, my_ax, my_ay, static64, qx0, qy0);
                __syncwarp();
                kpend = 0;
                my_cm = 0;
              }
            }
          } else if (MODE == K2_EMIT) {
            if (c0 || c1) {
              const unsigned long long idx = atomicAdd(P.emit_count, (unsigned long long)(c0 + c1));
              unsigned long long o = idx;
              if (c0 && (int64_t)o < P.emit_cap) {
                P.emit_key[o] = ((uint64_t)((uint32_t)(py0 * P.W + px)) << 32) | seq0;
                P.emit_gv[o] = S.slot[j];
                P.emit_alpha[o] = a0;
                P.emit_trans[o] = t0;
              }
              if (c0) o++;
              if (c1 && (int64_t)o < P.emit_cap) {
                P.emit_key[o] = ((uint64_t)((uint32_t)(py1 * P.W + px)) << 32) | seq1;
                P.emit_gv[o] = S.slot[j];
                P.emit_alpha[o] = a1;
                P.emit_trans[o] = t1;
              }
            }
            seq0 += c0;
            seq1 += c1;
          } else {  // K2_DOMINANT: argmax alpha*T, ties by smaller id (scene.py:179)
            const uint32_t g = r.g;
            if (c0 && (w0 > best_w0 || (w0 == best_w0 && g < best_g0))) {
              best_w0 = w0;
              best_g0 = g;
              best_gv0 = S.slot[j];
            }
            if (c1 && (w1 > best_w1 || (w1 == best_w1 && g < best_g1))) {
              best_w1 = w1;
              best_g1 = g;
              best_gv1 = S.slot[j];
            }
          }
        }
      }
    }
    if (kSlots && kpend > 0) {
      __syncwarp();
      if (K2_STATS_ON) st[K2S_FLUSHES]++;
      if (MODE == K2_CACHE)
        k2_flush_cache(S, P, lane, kpend, my_cm, my_slot, my_ax, my_ay, qx0, qy0, v, cache_ch);
      else
        k2_flush(S, P, lane, kpend, my_cm, my_slot, my_ax, my_ay, static64, qx0, qy0);
      __syncwarp();
    }
    if (MODE == K2_DOMINANT) {
      if (in0) {
        const int64_t pix = (int64_t)py0 * P.W + px;
        P.dom_gid[pix] = best_g0 != 0xFFFFFFFFu ? (int64_t)best_g0 : -1;
        P.dom_depth[pix] = best_g0 != 0xFFFFFFFFu ? P.depth64[best_gv0] : 0.0;
      }
      if (in1) {
        const int64_t pix = (int64_t)py1 * P.W + px;
        P.dom_gid[pix] = best_g1 != 0xFFFFFFFFu ? (int64_t)best_g1 : -1;
        P.dom_depth[pix] = best_g1 != 0xFFFFFFFFu ? P.depth64[best_gv1] : 0.0;
      }
    }
  }
  if (MODE == K2_CACHE) k2_cache_clear_tail(P, lane, cache_ch);
  if (K2_STATS_ON && lane == 0)
    for (int i = 0; i < K2S_N; i++) atomicAdd(&P.stats[i], st[i]);
}

// Compact list of the non-empty tiles in [t0, t1) (order irrelevant: every unit is independent).
__global__ void k2_build_items(const uint32_t *__restrict__ tile_range, int t0, int t1,
                               uint32_t *__restrict__ items, uint32_t *__restrict__ n_items) {
  const int t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
  const bool ne = t < t1 && tile_range[2 * t] < tile_range[2 * t + 1];
  const uint32_t m = __ballot_sync(0xffffffffu, ne);
  if (!m) return;
  uint32_t base = 0;
  const int lane = threadIdx.x & 31;
  if (lane == __ffs(m) - 1) base = atomicAdd(n_items, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (ne) items[base + __popc(m & ((1u << lane) - 1))] = (uint32_t)t;
}

// Work-ordered schedule (accumulate mode): every tile keyed by its list length (in units of 32
// instances, capped at 255); a one-pass descending radix sort puts the longest tiles at the head
// of the atomic queue, so the long lists start first and the kernel does not end on a tail of
// a few heavy units (longest-processing-time-first).
__global__ void k2_tile_keys(const uint32_t *__restrict__ tile_range, int t0, int t1,
                             uint8_t *__restrict__ keys, uint32_t *__restrict__ vals,
                             uint32_t *__restrict__ n_items) {
  const int t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t len = t < t1 ? tile_range[2 * t + 1] - tile_range[2 * t] : 0u;
  const bool ne = t < t1 && tile_range[2 * t] < tile_range[2 * t + 1];
  if (t < t1) {
    keys[t - t0] = (uint8_t)min(len / 32u + (ne ? 1u : 0u), 255u);  // empty tiles: key 0, last
    vals[t - t0] = (uint32_t)t;
  }
  const uint32_t m = __ballot_sync(0xffffffffu, ne);
  if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(n_items, (uint32_t)__popc(m));
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t k2_sort_temp(int nt) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, (const uint8_t *)nullptr,
                                            (uint8_t *)nullptr, (const uint32_t *)nullptr,
                                            (uint32_t *)nullptr, nt, 0, 8);
  return bytes;
}

size_t k2_schedule_bytes(int n_tiles) {
  return 2 * align_up((size_t)n_tiles) + align_up(4 * (size_t)n_tiles) +
         align_up(k2_sort_temp(n_tiles));
}

template <int MODE, typename TrackT>
static cudaError_t launch_mode(const K2Params &P, cudaStream_t s, int cap) {
  auto kern = k2_raster<MODE, TrackT>;
  const size_t smem = K2_ETAB_BYTES + sizeof(K2Warp<TrackT>) * K2_WARPS;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K2_WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  // the plan's residency cap (ts_plan_set_k2_ctas_per_sm): leaves SM room for the other frames
  // in flight
  if (cap > 0 && cap < per_sm) per_sm = cap;
  kern<<<sms * (per_sm > 0 ? per_sm : 1), K2_WARPS * 32, smem, s>>>(P);
  return cudaGetLastError();
}

bool k2_writes_touched() { return true; }  // the accumulate kernel marks touched gvs

cudaError_t launch_k2(int mode, int track_dtype, const RasterRec *rec, const uint32_t *inst_gv,
                      const uint32_t *tile_range, const uint32_t *inst_base, uint32_t *items,
                      uint32_t *counters, int tile_begin, int tile_end, const void *track_target,
                      const uint8_t *track_valid, int W, int H, int tiles_x, int tiles_per_view,
                      const ts_config &cfg, Partial *partial, uint8_t *flag,
                      unsigned long long *emit_count, int64_t emit_cap, uint64_t *emit_key,
                      uint32_t *emit_gv, double *emit_alpha, double *emit_trans,
                      const double *depth64, int64_t *dom_gid, double *dom_depth,
                      unsigned long long *stats, void *schedule_ws, cudaStream_t s, int ctas_per_sm,
                      uint8_t *touched, double *pool, unsigned long long *pool_cursor,
                      uint64_t pool_cap, CacheRec *recs, unsigned long long *rec_cursor,
                      uint64_t rec_cap) {
  // counters[0] = number of items, counters[1] = work queue head
  cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  const int nt = tile_end - tile_begin;
  if (nt > 0 && schedule_ws) {
    char *ws = reinterpret_cast<char *>(schedule_ws);
    uint8_t *keys = reinterpret_cast<uint8_t *>(ws);
    uint8_t *keys2 = reinterpret_cast<uint8_t *>(ws + align_up((size_t)nt));
    uint32_t *vals = reinterpret_cast<uint32_t *>(ws + 2 * align_up((size_t)nt));
    void *tmp = ws + 2 * align_up((size_t)nt) + align_up(4 * (size_t)nt);
    size_t tmp_bytes = k2_sort_temp(nt);
    k2_tile_keys<<<(nt + 255) / 256, 256, 0, s>>>(tile_range, tile_begin, tile_end, keys, vals,
                                                  counters);
    e = cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, keys, keys2, vals, items, nt, 0,
                                                  8, s);
    if (e != cudaSuccess) return e;
  } else if (nt > 0) {
    k2_build_items<<<(nt + 255) / 256, 256, 0, s>>>(tile_range, tile_begin, tile_end, items,
                                                    counters);
  }
  K2Params P;
  P.rec = rec;
  P.inst_gv = inst_gv;
  P.tile_range = tile_range;
  P.inst_base = inst_base;
  P.items = items;
  P.n_items = counters;
  P.work_counter = counters + 1;
  P.track_target = track_target;
  P.track_vec = TS_K2_VEC_TRACKS &&
                (reinterpret_cast<uintptr_t>(track_target) %
                 (2 * (track_dtype == TS_TRACK_F32 ? sizeof(float) : sizeof(double)))) == 0;
  P.track_valid = track_valid;
  P.W = W;
  P.H = H;
  P.tiles_x = tiles_x;
  P.tiles_per_view = tiles_per_view;
  P.alpha_cutoff = cfg.alpha_cutoff;
  P.early_stop = cfg.early_stop;
  P.static_thr = cfg.static_threshold_px;
  P.partial = partial;
  P.flag = flag;
  P.touched = touched;
  P.pool = pool;
  P.pool_cursor = pool_cursor;
  P.pool_cap = pool_cap;
  P.recs = recs;
  P.rec_cursor = rec_cursor;
  P.rec_cap = rec_cap;
  P.emit_count = emit_count;
  P.emit_cap = emit_cap;
  P.emit_key = emit_key;
  P.emit_gv = emit_gv;
  P.emit_alpha = emit_alpha;
  P.emit_trans = emit_trans;
  P.depth64 = depth64;
  P.dom_gid = dom_gid;
  P.dom_depth = dom_depth;
  P.stats = stats;
  if (mode == K2_ACCUMULATE) {
    if (track_dtype == TS_TRACK_F32) return launch_mode<K2_ACCUMULATE, float>(P, s, ctas_per_sm);
    return launch_mode<K2_ACCUMULATE, double>(P, s, ctas_per_sm);
  }
  if (mode == K2_CACHE) return launch_mode<K2_CACHE, float>(P, s, ctas_per_sm);
  if (mode == K2_EMIT) return launch_mode<K2_EMIT, float>(P, s, ctas_per_sm);
  return launch_mode<K2_DOMINANT, float>(P, s, ctas_per_sm);
}

}  // namespace ts
