// raster.cu -- K2: tile rasterizer fused with per-Gaussian moment accumulation (sm_100a).
//
// Reference semantics: gausstrack/splat.py:147-195 (alpha, keep predicate, per-pixel
// front-to-back transmittance, early stop) fused with motion2d.py:144-160 (accumulate_view).
//
// One CTA (256 threads, 8 warps) per 16x16 tile; warp w owns the 8x4 pixel block
// ((w&1)*8, (w>>1)*4) and lane l the pixel (l&7, l>>3) inside it.  The tile's Gaussian list is
// already in (depth, gid) order (K1), so each lane walks it front to back exactly as the
// reference walks a pixel's sorted contributions.
//   * Batches of K2_BATCH records are staged in shared memory (64-byte records).
//   * Warp-level culling: for every chunk of 32 records, one ballot of "bbox intersects my 8x4
//     block" leaves only the Gaussians that can touch the warp's pixels; warps whose pixels are
//     all saturated (T < early_stop) skip work, and the CTA stops once every pixel saturated.
//   * Predicates in fp64 in the reference's operation order (bit-exact q and alpha >= cutoff;
//     T >= early_stop up to the reference's own log-cumsum rounding).
//   * Accumulation is transposed instead of shuffled: a contributing lane stores w = alpha*T
//     into a per-warp 32x32 shared buffer; after the chunk, lane j sums Gaussian j's
//     contributions over the warp's 32 pixels (no shuffles) into a per-warp partial.  The CTA then
//     adds the 8 warp partials IN WARP ORDER and writes ONE partial per (tile, Gaussian) instance
//     to its own slot -- no atomics of any kind, no zero-initialised accumulators, and results
//     that are bit-reproducible run to run (K3 adds a Gaussian's tile partials in instance order).
#include "common.cuh"
#include "kernels.cuh"

namespace ts {

constexpr int K2_THREADS = 256;
constexpr int K2_WARPS = K2_THREADS / 32;
constexpr int K2_BATCH = 128;
constexpr int K2_WROW = 33;     // padded row of the per-warp w buffer (bank spread)
constexpr int K2_PSTRIDE = 15;  // per-warp partial: 13 moments, count, static count

struct K2Params {
  const RasterRec *rec;
  const uint32_t *inst_gv;     // sorted instances: gv
  const uint32_t *tile_range;  // [start, end) per global tile
  const uint32_t *inst_base;   // per gv: first partial slot (gv order scan of tile counts)
  const void *track_target;    // (V, H, W, 2)
  const uint8_t *track_valid;  // (V, H, W)
  int64_t n;                   // Gaussians
  int W, H, tiles_x, tiles_per_view, tile_offset;
  double alpha_cutoff, early_stop, static_thr;
  // accumulate mode
  Partial *partial;
  uint8_t *flag;
  // emit mode
  unsigned long long *emit_count;
  int64_t emit_cap;
  uint64_t *emit_key;   // (pixel << 32) | sequence number within the pixel
  uint32_t *emit_gv;
  double *emit_alpha, *emit_trans;
  // dominant mode
  const double *depth64;
  int64_t *dom_gid;
  double *dom_depth;
};

struct K2Smem {
  RasterRec rec[K2_BATCH];
  uint32_t slot[K2_BATCH];
  double trk_u[K2_THREADS];
  double trk_v[K2_THREADS];
  uint8_t trk_static[K2_THREADS];
  double w[K2_WARPS][32][K2_WROW];
  double part[K2_WARPS][32][K2_PSTRIDE];
};

template <int MODE, typename TrackT>
__global__ void __launch_bounds__(K2_THREADS, 2) k2_raster(const K2Params P) {
  extern __shared__ __align__(16) unsigned char k2_smem_raw[];
  K2Smem &S = *reinterpret_cast<K2Smem *>(k2_smem_raw);

  const int tile = blockIdx.x + P.tile_offset;
  const uint32_t start = P.tile_range[2 * tile], end = P.tile_range[2 * tile + 1];
  if (start >= end) return;
  const int v = tile / P.tiles_per_view;
  const int t = tile - v * P.tiles_per_view;
  const int ty = t / P.tiles_x, tx = t - ty * P.tiles_x;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rx0 = tx * TS_TILE + (warp & 1) * 8, ry0 = ty * TS_TILE + (warp >> 1) * 4;
  const int px = rx0 + (lane & 7), py = ry0 + (lane >> 3);
  const bool inimg = px < P.W && py < P.H;

  // per-pixel track (motion2d.py:145-150) and static flag (motion2d.py:158)
  bool valid = false;
  if (MODE == K2_ACCUMULATE) {
    double u = 0.0, vv = 0.0;
    if (inimg) {
      const int64_t pix = ((int64_t)v * P.H + py) * P.W + px;
      valid = P.track_valid[pix] != 0;
      if (valid) {
        const TrackT *tg = reinterpret_cast<const TrackT *>(P.track_target) + 2 * pix;
        u = load_track(tg);
        vv = load_track(tg + 1);
      }
    }
    S.trk_u[tid] = u;
    S.trk_v[tid] = vv;
    S.trk_static[tid] = valid && is_static(u, vv, px, py, P.static_thr);
  }
  double T = 1.0;
  bool done = !inimg || !(T >= P.early_stop);
  uint32_t seq = 0;  // emit mode: contribution index within the pixel
  double best_w = -1.0;  // dominant mode
  uint32_t best_gv = 0xFFFFFFFFu, best_g = 0xFFFFFFFFu;

  for (uint32_t b = start; b < end; b += K2_BATCH) {
    // CTA-uniform early exit; also the barrier protecting the shared batch buffers
    if (__syncthreads_count(!done) == 0) break;
    const int nb = min((int)(end - b), K2_BATCH);
    if (tid < nb) {
      const uint32_t gv = P.inst_gv[b + tid];
      const RasterRec r = P.rec[gv];
      S.rec[tid] = r;
      if (MODE == K2_ACCUMULATE) {
        const int tx0 = r.x0 / TS_TILE, tx1 = r.x1 / TS_TILE, ty0 = r.y0 / TS_TILE;
        S.slot[tid] = P.inst_base[gv] + (uint32_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
      } else {
        S.slot[tid] = gv;
      }
    }
    __syncthreads();

    for (int c = 0; c < nb; c += 32) {
      uint32_t my_cmask = 0;
      if (!__all_sync(0xffffffffu, done)) {
        // warp-level culling: which of these 32 records touch this warp's 8x4 block?
        bool hit = false;
        if (c + lane < nb) {
          const RasterRec &r = S.rec[c + lane];
          hit = !(r.x1 < rx0 || r.x0 > rx0 + 7 || r.y1 < ry0 || r.y0 > ry0 + 3);
        }
        uint32_t mask = __ballot_sync(0xffffffffu, hit);
        while (mask) {
          const int j = __ffs(mask) - 1;
          mask &= mask - 1;
          const RasterRec &r = S.rec[c + j];
          bool contrib = false;
          if (!done && px >= r.x0 && px <= r.x1 && py >= r.y0 && py <= r.y1) {
            const double dx = sub((double)px, r.mx), dy = sub((double)py, r.my);
            const double q = mahalanobis(r, dx, dy);
            if (q <= TS_SIGMA_RADIUS * TS_SIGMA_RADIUS) {
              const double a = alpha_of(r.opacity, q);
              if (a >= P.alpha_cutoff) {
                const double tin = T;
                const double w = mul(a, tin);  // motion2d.py:151
                T = mul(tin, sub(1.0, a));
                if (!(T >= P.early_stop)) done = true;
                if (MODE == K2_ACCUMULATE) {
                  contrib = valid;
                  if (contrib) S.w[warp][j][lane] = w;
                } else if (MODE == K2_EMIT) {
                  const unsigned long long idx = atomicAdd(P.emit_count, 1ull);
                  if ((int64_t)idx < P.emit_cap) {
                    P.emit_key[idx] = ((uint64_t)((uint32_t)(py * P.W + px)) << 32) | seq;
                    P.emit_gv[idx] = S.slot[c + j];
                    P.emit_alpha[idx] = a;
                    P.emit_trans[idx] = tin;
                  }
                  seq++;
                } else {  // K2_DOMINANT: argmax alpha*T, ties by smaller id (scene.py:179)
                  const uint32_t g = r.g;
                  if (w > best_w || (w == best_w && g < best_g)) {
                    best_w = w;
                    best_gv = S.slot[c + j];
                    best_g = g;
                  }
                }
              }
            }
          }
          if (MODE == K2_ACCUMULATE) {
            const uint32_t cm = __ballot_sync(0xffffffffu, contrib);
            if (lane == j) my_cmask = cm;
          }
        }
      }
      if (MODE == K2_ACCUMULATE) {
        __syncwarp();
        // lane `lane` owns record c+lane: sum its contributions over this warp's pixels,
        // in pixel order, relative to the Gaussian's integer anchor
        double m[TS_NMOM];
#pragma unroll
        for (int k = 0; k < TS_NMOM; k++) m[k] = 0.0;
        uint32_t cnt = 0, scnt = 0;
        if (my_cmask) {
          const RasterRec &r = S.rec[c + lane];
          const double ax = (double)anchor_x(r), ay = (double)anchor_y(r);
          uint32_t bits = my_cmask;
          while (bits) {
            const int p = __ffs(bits) - 1;
            bits &= bits - 1;
            const double w = S.w[warp][lane][p];
            const int pt = warp * 32 + p;
            const double dx = (double)(rx0 + (p & 7)) - ax, dy = (double)(ry0 + (p >> 3)) - ay;
            const double ua = S.trk_u[pt] - ax, va = S.trk_v[pt] - ay;
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
            if (S.trk_static[pt]) {
              m[12] += w;
              scnt++;
            }
            cnt++;
          }
        }
#pragma unroll
        for (int k = 0; k < TS_NMOM; k++) S.part[warp][lane][k] = m[k];
        S.part[warp][lane][13] = (double)cnt;
        S.part[warp][lane][14] = (double)scnt;
        __syncthreads();
        // fixed-order cross-warp reduction: thread -> (record j, field k)
        for (int task = tid; task < 32 * 16; task += K2_THREADS) {
          const int j = task >> 4, k = task & 15;
          if (c + j >= nb) continue;
          double tot_cnt = 0.0;
#pragma unroll
          for (int ww = 0; ww < K2_WARPS; ww++) tot_cnt += S.part[ww][j][13];
          if (tot_cnt == 0.0) continue;
          Partial *dst = P.partial + S.slot[c + j];
          if (k < TS_NMOM) {
            double s = 0.0;
#pragma unroll
            for (int ww = 0; ww < K2_WARPS; ww++) s += S.part[ww][j][k];
            dst->m[k] = s;
          } else if (k == 13) {
            double s = 0.0;
#pragma unroll
            for (int ww = 0; ww < K2_WARPS; ww++) s += S.part[ww][j][14];
            dst->count = (uint32_t)tot_cnt;
            dst->static_count = (uint32_t)s;
          } else {
            P.flag[S.slot[c + j]] = 1;
          }
        }
        __syncthreads();
      }
    }
  }
  if (MODE == K2_DOMINANT && inimg) {
    const int64_t pix = (int64_t)py * P.W + px;
    if (best_gv != 0xFFFFFFFFu) {
      P.dom_gid[pix] = best_g;
      P.dom_depth[pix] = P.depth64[best_gv];
    } else {
      P.dom_gid[pix] = -1;
      P.dom_depth[pix] = 0.0;
    }
  }
}

template <int MODE, typename TrackT>
static cudaError_t launch_mode(const K2Params &P, int n_tiles, cudaStream_t s) {
  auto kern = k2_raster<MODE, TrackT>;
  const size_t smem = sizeof(K2Smem);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (n_tiles > 0) kern<<<n_tiles, K2_THREADS, smem, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_k2(int mode, int track_dtype, const RasterRec *rec, const uint32_t *inst_gv,
                      const uint32_t *tile_range, const uint32_t *inst_base,
                      const void *track_target, const uint8_t *track_valid, int64_t n, int W,
                      int H, int tiles_x, int tiles_per_view, int n_tiles_total,
                      int tile_offset, const ts_config &cfg, Partial *partial, uint8_t *flag,
                      unsigned long long *emit_count, int64_t emit_cap, uint64_t *emit_key,
                      uint32_t *emit_gv, double *emit_alpha, double *emit_trans,
                      const double *depth64, int64_t *dom_gid, double *dom_depth,
                      cudaStream_t s) {
  K2Params P;
  P.rec = rec;
  P.inst_gv = inst_gv;
  P.tile_range = tile_range;
  P.inst_base = inst_base;
  P.track_target = track_target;
  P.track_valid = track_valid;
  P.n = n;
  P.W = W;
  P.H = H;
  P.tiles_x = tiles_x;
  P.tiles_per_view = tiles_per_view;
  P.tile_offset = tile_offset;
  P.alpha_cutoff = cfg.alpha_cutoff;
  P.early_stop = cfg.early_stop;
  P.static_thr = cfg.static_threshold_px;
  P.partial = partial;
  P.flag = flag;
  P.emit_count = emit_count;
  P.emit_cap = emit_cap;
  P.emit_key = emit_key;
  P.emit_gv = emit_gv;
  P.emit_alpha = emit_alpha;
  P.emit_trans = emit_trans;
  P.depth64 = depth64;
  P.dom_gid = dom_gid;
  P.dom_depth = dom_depth;
  if (mode == K2_ACCUMULATE) {
    if (track_dtype == TS_TRACK_F32) return launch_mode<K2_ACCUMULATE, float>(P, n_tiles_total, s);
    return launch_mode<K2_ACCUMULATE, double>(P, n_tiles_total, s);
  }
  if (mode == K2_EMIT) return launch_mode<K2_EMIT, float>(P, n_tiles_total, s);
  return launch_mode<K2_DOMINANT, float>(P, n_tiles_total, s);
}

}  // namespace ts
