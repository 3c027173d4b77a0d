// api.cu -- C ABI of the B200 hot path: plan (device workspace), K1..K4 orchestration, CUB sorts.
//
// Everything is stream-ordered on the caller's stream; the plan owns a grow-only device workspace
// allocated with cudaMallocAsync.  The only host synchronisations are the data-dependent sizes
// (instance count after binning, contribution count of the emitting rasterizer).
#include <cub/cub.cuh>

#include <algorithm>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

using namespace ts;

namespace {

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need, cudaStream_t s) {
    if (need <= bytes && p) return cudaSuccess;
    if (p) {
      cudaError_t e = cudaFreeAsync(p, s);
      if (e != cudaSuccess) return e;
      p = nullptr;
      bytes = 0;
    }
    size_t want = need + need / 4 + 256;
    cudaError_t e = cudaMallocAsync(&p, want, s);
    if (e != cudaSuccess) return e;
    bytes = want;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T *as() const { return reinterpret_cast<T *>(p); }
};

constexpr int64_t K1_TIE_RUN_MAX_HOST = 64;  // binning.cu K1_TIE_RUN_MAX
#ifndef TS_K1_KEY_BITS
#define TS_K1_KEY_BITS 32  // 24 (three onesweep passes) measured: cfg2 depth sort 0.381 -> 0.365 ms,
                           // cfg5 2.27 -> 2.75 ms (3M Gaussians per view in 2^20 levels: tie runs)
#endif

#ifndef TS_K1_DEPTH_BITS_MAX
#define TS_K1_DEPTH_BITS_MAX 28  // 26 -> 28: cfg5 depth sort + tie repair 2.25 -> 2.16 ms (fewer equal keys)
#endif

int bits_for(uint64_t x) {  // number of bits needed to represent values < x
  int b = 0;
  while (b < 64 && (1ull << b) < x) b++;
  return b < 1 ? 1 : b;
}

enum Stage { ST_PROJECT = 0, ST_DEPTH_SORT, ST_TILE_SORT, ST_RASTER, ST_SOLVE, ST_FUSE, ST_N };

}  // namespace

struct ByteToU32 {
  __host__ __device__ uint32_t operator()(uint8_t x) const { return x; }
};

struct ts_plan {
  // binning state
  DevBuf cams, rec, dkey, dkey2, dval, dval2, depth64, ntiles, status, bbox, off_sorted,
      inst_base, tkey, tkey2, tval, tval2, range, items, counters, cub_tmp;
  // per-frame state
  DevBuf k2_stats;
  DevBuf partial, flag, touched, k3_list, k3_rank, k3_fits, mot_status, mot_a, mot_b, mot_w,
      mot_cnt, mot_scnt, mot_sw;
  // clip contribution cache (ts_frame_cache, cache.cu)
  DevBuf cache_pool, cache_cursor, cache_recs, cache_cnt, cache_off, cache_w, cache_xy,
      cache_ranges, cache_chunks, cache_multi, cache_scratch, cache_counters;
  // stage-API buffers
  DevBuf emit_count, emit_key, emit_key2, emit_gv, emit_alpha, emit_trans, emit_idx, emit_idx2,
      deg_flags, deg_ids, deg_count, acc_keys, acc_keys2, acc_order, acc_iota, seg_start, seg_end;
  // regularisation buffers
  DevBuf knn_part, knn_grid, knn_key, knn_key2, knn_val, knn_val2, knn_sp, knn_lo, knn_hi,
      reg_static, reg_source, reg_euler, k4_ws, drange, k2_sched, tie_runs, tie_tmp;
  uint32_t *host_small = nullptr;  // pinned scratch for size read-backs
  int32_t *host_rects = nullptr;   // per-view union of binned bboxes (x0 y0 x1 y1), after binning
  int64_t n = 0, n_inst = 0, n_slots = 0, emit_n = 0, n_deg = 0;
  int V = 0, W = 0, H = 0, tiles_x = 0, tiles_y = 0, tpv = 0;
  const double *gaussians = nullptr;
  std::vector<ts_camera> host_cams;
  ts_config cfg{};
  bool timing = false;
  int k2_ctas_per_sm = 0;  // ts_plan_set_k2_ctas_per_sm (0: full residency)
  int64_t k3_last_nv = 0;   // K3 split choice of the previous frame (see ts_frame_compensate)
  bool cache_valid = false;  // clip contribution cache (ts_frame_cache) of the current binning
  uint64_t cache_cap = 0;    // pool capacity in doubles
  uint64_t cache_used = 0;   // doubles handed out by the last build
  uint64_t cache_rec_cap = 0;  // record capacity
  uint64_t cache_recs_used = 0;  // records handed out by the last build (incl. unfilled)
  uint64_t cache_chunk_bound = 0, cache_multi_bound = 0;  // work units of the per-frame kernel
  bool k3_last_split = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_marks;
  size_t ev_next = 0;

  cudaEvent_t take_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
  cudaEvent_t mark_begin(cudaStream_t s) {
    if (!timing) return nullptr;
    cudaEvent_t e = take_event();
    cudaEventRecord(e, s);
    return e;
  }
  void mark_end(int stage, cudaEvent_t b, cudaStream_t s) {
    if (!timing || !b) return;
    cudaEvent_t e = take_event();
    cudaEventRecord(e, s);
    ev_marks.push_back({stage, {b, e}});
  }
  DevBuf *all_bufs() { return &cams; }
};

namespace {

template <typename T>
T *ptr(DevBuf &b) { return b.as<T>(); }

#define ENSURE(buf, bytes) TS_CUDA_TRY((buf).ensure((size_t)(bytes), s))

int64_t sum_workspace(const ts_plan *p) {
  const DevBuf *bufs[] = {&p->cams, &p->rec, &p->dkey, &p->dkey2, &p->dval, &p->dval2, &p->depth64,
                          &p->ntiles, &p->status, &p->bbox, &p->off_sorted,
                          &p->inst_base, &p->tkey, &p->tkey2, &p->tval, &p->tval2, &p->range,
                          &p->items, &p->counters, &p->cub_tmp, &p->partial, &p->flag, &p->mot_status, &p->mot_a,
                          &p->mot_b, &p->mot_w, &p->mot_cnt, &p->mot_scnt, &p->mot_sw,
                          &p->emit_count, &p->emit_key, &p->emit_key2, &p->emit_gv,
                          &p->emit_alpha, &p->emit_trans, &p->emit_idx, &p->emit_idx2,
                          &p->deg_flags, &p->deg_ids, &p->deg_count, &p->acc_keys, &p->acc_keys2,
                          &p->acc_order, &p->acc_iota, &p->seg_start, &p->seg_end,
                          &p->knn_part, &p->knn_grid, &p->knn_key, &p->knn_key2, &p->knn_val,
                          &p->knn_val2, &p->knn_sp, &p->knn_lo, &p->knn_hi, &p->reg_static,
                          &p->reg_source, &p->reg_euler, &p->k4_ws, &p->drange, &p->k2_sched,
                          &p->touched, &p->k3_list, &p->k3_rank, &p->k3_fits, &p->tie_runs,
                          &p->tie_tmp, &p->cache_pool, &p->cache_cursor, &p->cache_recs,
                          &p->cache_cnt, &p->cache_off, &p->cache_w, &p->cache_xy,
                          &p->cache_ranges, &p->cache_chunks, &p->cache_multi,
                          &p->cache_scratch, &p->cache_counters};
  int64_t t = 0;
  for (const DevBuf *b : bufs) t += (int64_t)b->bytes;
  return t;
}

void release_all(ts_plan *p) {
  DevBuf *bufs[] = {&p->cams, &p->rec, &p->dkey, &p->dkey2, &p->dval, &p->dval2, &p->depth64,
                    &p->ntiles, &p->status, &p->bbox, &p->off_sorted,
                    &p->inst_base, &p->tkey, &p->tkey2, &p->tval, &p->tval2, &p->range,
                    &p->items, &p->counters, &p->cub_tmp, &p->partial, &p->flag, &p->mot_status, &p->mot_a, &p->mot_b,
                    &p->mot_w, &p->mot_cnt, &p->mot_scnt, &p->mot_sw, &p->emit_count,
                    &p->emit_key, &p->emit_key2, &p->emit_gv, &p->emit_alpha, &p->emit_trans,
                    &p->emit_idx, &p->emit_idx2, &p->deg_flags, &p->deg_ids, &p->deg_count,
                    &p->acc_keys, &p->acc_keys2, &p->acc_order, &p->acc_iota, &p->seg_start,
                    &p->seg_end, &p->knn_part, &p->knn_grid, &p->knn_key, &p->knn_key2,
                    &p->knn_val, &p->knn_val2, &p->knn_sp, &p->knn_lo, &p->knn_hi,
                    &p->reg_static, &p->reg_source, &p->reg_euler, &p->k4_ws, &p->drange, &p->k2_sched,
                    &p->touched, &p->k3_list, &p->k3_rank, &p->k3_fits, &p->tie_runs,
                    &p->tie_tmp, &p->cache_pool, &p->cache_cursor, &p->cache_recs,
                    &p->cache_cnt, &p->cache_off, &p->cache_w, &p->cache_xy, &p->cache_ranges,
                    &p->cache_chunks, &p->cache_multi, &p->cache_scratch, &p->cache_counters};
  for (DevBuf *b : bufs) b->release();
}

__global__ void k_iota(uint32_t *x, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (uint32_t)i;
}
__global__ void k_gid_keys(const int64_t *gid, uint32_t *keys, int64_t m) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) keys[i] = (uint32_t)gid[i];
}
__global__ void k_degenerate_flags(const int8_t *status, int64_t n, uint8_t *flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = status[i] == 1;
}
__global__ void k_fetch_contribs(const uint64_t *key_sorted, const uint32_t *idx_sorted,
                                 const uint32_t *emit_gv, const double *emit_alpha,
                                 const double *emit_trans, const RasterRec *rec,
                                 const double *depth64, int64_t m, int W, int32_t *px,
                                 int32_t *py, int64_t *gid, double *alpha, double *trans,
                                 double *depth) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t k = idx_sorted[i];
  const uint32_t pix = (uint32_t)(key_sorted[i] >> 32);
  const uint32_t gv = emit_gv[k];
  px[i] = (int32_t)(pix % (uint32_t)W);
  py[i] = (int32_t)(pix / (uint32_t)W);
  gid[i] = (int64_t)rec[gv].g;
  alpha[i] = emit_alpha[k];
  trans[i] = emit_trans[k];
  depth[i] = depth64[gv];
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

struct GatherCount {  // tile count of the i-th depth-sorted gv (0 at i == NV: scan total)
  const uint32_t *sorted_gv, *ntiles;
  int64_t nv;
  __host__ __device__ __forceinline__ uint32_t operator()(int64_t i) const {
#ifdef __CUDA_ARCH__
    return i < nv ? ntiles[sorted_gv[i]] : 0u;
#else
    return 0u;
#endif
  }
};

// Partial-moment slots of gv i: one per 8x8 quadrant its bbox touches (only those can receive
// a contribution); 0 for a non-binned gv (sentinel bbox {0, -1, 0, -1}) and for i == NV, so an
// exclusive scan over NV + 1 entries ends with the total.
struct QuadCount {
  const int16_t *bbox;
  int64_t nv;
  __host__ __device__ __forceinline__ uint32_t operator()(int64_t i) const {
#ifdef __CUDA_ARCH__
    if (i >= nv) return 0u;
    const short4 bb = reinterpret_cast<const short4 *>(bbox)[i];
    return (uint32_t)(((bb.y >> 3) - (bb.x >> 3) + 1) * ((bb.w >> 3) - (bb.z >> 3) + 1));
#else
    return 0u;
#endif
  }
};

// Onesweep policy for the two K1 sorts (u32 key, u32 value): CUB's sm_100 default runs 384
// threads x 23 items at 109 registers, one CTA per SM; 256 x 23 measured 11-14% faster on both
// the 6M-pair depth sort and the 12.2M-pair tile sort (tools/sortbench).  Every other policy
// member is CUB's.
template <int THREADS, int ITEMS>
struct OnesweepHub {
  using Up = typename cub::detail::radix::policy_hub<uint32_t, uint32_t, uint32_t>::Policy1000;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = 8;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, uint32_t, 8>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, 8>;
    using OnesweepPolicy = cub::AgentRadixSortOnesweepPolicy<
        THREADS, ITEMS, uint32_t, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
        cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, 8>;
    using ScanPolicy = typename Up::ScanPolicy;
    using DownsweepPolicy = typename Up::DownsweepPolicy;
    using AltDownsweepPolicy = typename Up::AltDownsweepPolicy;
    using UpsweepPolicy = typename Up::UpsweepPolicy;
    using AltUpsweepPolicy = typename Up::AltUpsweepPolicy;
    using SingleTilePolicy = typename Up::SingleTilePolicy;
    using SegmentedPolicy = typename Up::SegmentedPolicy;
    using AltSegmentedPolicy = typename Up::AltSegmentedPolicy;
  };
  using MaxPolicy = Policy1000;
};

// cub::DeviceRadixSort::SortPairs semantics (result in kout / vout) with the policy above.
cudaError_t k1_sort_pairs(void *tmp, size_t &bytes, const uint32_t *kin, uint32_t *kout,
                          const uint32_t *vin, uint32_t *vout, int n, int end_bit,
                          cudaStream_t s) {
  cub::DoubleBuffer<uint32_t> kb(const_cast<uint32_t *>(kin), kout);
  cub::DoubleBuffer<uint32_t> vb(const_cast<uint32_t *>(vin), vout);
  return cub::DispatchRadixSort<false, uint32_t, uint32_t, uint32_t,
                                OnesweepHub<256, 23>>::Dispatch(tmp, bytes, kb, vb, (uint32_t)n, 0,
                                                                end_bit, false, s);
}

template <typename F>
cudaError_t cub_call(ts_plan *p, cudaStream_t s, F f) {
  size_t need = 0;
  cudaError_t e = f((void *)nullptr, need);
  if (e != cudaSuccess) return e;
  e = p->cub_tmp.ensure(need, s);
  if (e != cudaSuccess) return e;
  size_t have = p->cub_tmp.bytes;
  return f(p->cub_tmp.p, have);
}

int validate_cams(const ts_camera *cams, int V) {
  if (!cams || V < 1) return TS_E_INVALID_ARGUMENT;
  for (int v = 0; v < V; v++) {
    if (cams[v].width <= 0 || cams[v].height <= 0 || cams[v].width > 32767 ||
        cams[v].height > 32767)
      return TS_E_INVALID_ARGUMENT;
    if (cams[v].width != cams[0].width || cams[v].height != cams[0].height)
      return TS_E_DIMENSION_MISMATCH;
  }
  return TS_OK;
}

// Address under which kernels read `ptr`: device / managed memory as is (*host = 0); page-locked
// host memory through its mapped device address (*host = 1).  Pageable host memory cannot be
// read by a kernel: TS_E_INVALID_ARGUMENT.
int device_view(const void *ptr, const void **dev, int *host) {
  if (!ptr) return TS_E_INVALID_ARGUMENT;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return TS_E_INVALID_ARGUMENT;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    *dev = ptr;
    *host = 0;
    return TS_OK;
  }
  if (a.type == cudaMemoryTypeHost && a.devicePointer) {
    *dev = a.devicePointer;
    *host = 1;
    return TS_OK;
  }
  return TS_E_INVALID_ARGUMENT;
}

// K1 + sorts + ranges into the plan.
int frame_bin(ts_plan *p, const double *G, int64_t n, const ts_camera *cams, int V,
              const ts_config *cfg, cudaStream_t s) {
  int rc = validate_cams(cams, V);
  if (rc) return rc;
  if (V > 64) return TS_E_INVALID_ARGUMENT;  // 6 view bits in the 32-bit depth key
  if (n < 0 || (uint64_t)n * (uint64_t)V >= 0xFFFFFFFFull) return TS_E_INVALID_ARGUMENT;
  p->cache_valid = false;  // a new binning invalidates the clip's contribution cache
  p->n = n;
  p->V = V;
  p->W = cams[0].width;
  p->H = cams[0].height;
  p->tiles_x = (p->W + TS_TILE - 1) / TS_TILE;
  p->tiles_y = (p->H + TS_TILE - 1) / TS_TILE;
  p->tpv = p->tiles_x * p->tiles_y;
  p->gaussians = G;
  p->host_cams.assign(cams, cams + V);
  if (cfg) p->cfg = *cfg;
  const int64_t NV = n * V;
  if (!p->host_small) TS_CUDA_TRY(cudaMallocHost(&p->host_small, 64));
  if (!p->host_rects) TS_CUDA_TRY(cudaMallocHost(&p->host_rects, 16 * 64));

  ENSURE(p->cams, sizeof(ts_camera) * V);
  TS_CUDA_TRY(cudaMemcpyAsync(p->cams.p, cams, sizeof(ts_camera) * V, cudaMemcpyHostToDevice, s));
  ENSURE(p->rec, sizeof(RasterRec) * NV);
  ENSURE(p->dkey, 4 * NV);
  ENSURE(p->dkey2, 4 * NV);
  ENSURE(p->dval, 4 * NV);
  ENSURE(p->dval2, 4 * NV);
  ENSURE(p->depth64, 8 * NV);
  ENSURE(p->ntiles, 4 * NV);
  ENSURE(p->status, NV);
  ENSURE(p->bbox, 8 * NV);
  ENSURE(p->off_sorted, 4 * (NV + 1));
  ENSURE(p->inst_base, 4 * (NV + 1));
  const int64_t ntile_total = (int64_t)p->tpv * V;
  ENSURE(p->range, 8 * ntile_total);
  ENSURE(p->items, 4 * (ntile_total + 1));
  ENSURE(p->counters, 64);

  cudaEvent_t e0 = p->mark_begin(s);
  ENSURE(p->drange, 4 * (K1_RECT_OFFSET + 4 * 64));
  // depth key: view bits + quantised depth (at most 2^TS_K1_DEPTH_BITS_MAX levels),
  // TS_K1_KEY_BITS in all
  const int dbits = std::min(TS_K1_DEPTH_BITS_MAX, TS_K1_KEY_BITS - bits_for((uint64_t)V));
  launch_k1_project(G, n, ptr<ts_camera>(p->cams), V, dbits, ptr<RasterRec>(p->rec),
                    ptr<uint32_t>(p->drange), ptr<uint32_t>(p->dkey),
                    ptr<uint32_t>(p->dval), ptr<double>(p->depth64), ptr<uint32_t>(p->ntiles),
                    ptr<int8_t>(p->status), ptr<int16_t>(p->bbox), s);
  TS_CUDA_TRY(cudaGetLastError());
  p->mark_end(ST_PROJECT, e0, s);

  cudaEvent_t e1 = p->mark_begin(s);
  if (NV > 0) {
    const int end_bit = dbits + bits_for((uint64_t)V);
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return k1_sort_pairs(tmp, bytes, ptr<uint32_t>(p->dkey), ptr<uint32_t>(p->dkey2),
                           ptr<uint32_t>(p->dval), ptr<uint32_t>(p->dval2), (int)NV, end_bit, s);
    }));
    const uint32_t long_cap = (uint32_t)(NV / (K1_TIE_RUN_MAX_HOST + 1) + 1);
    ENSURE(p->tie_runs, 8 * ((int64_t)long_cap + 1));
    TS_CUDA_TRY(cudaMemsetAsync(p->tie_runs.p, 0, 4, s));
    launch_k1_fix_ties(ptr<uint32_t>(p->dkey2), ptr<uint32_t>(p->dval2), ptr<double>(p->depth64), NV,
                       dbits, ptr<uint32_t>(p->tie_runs), long_cap, s);
    // instance offsets in depth order: scan of the tile counts gathered through the sorted gvs
    // (the gather is fused into the scan's loads)
    cub::TransformInputIterator<uint32_t, GatherCount, cub::CountingInputIterator<int64_t>>
        cnt_it(cub::CountingInputIterator<int64_t>(0),
               GatherCount{ptr<uint32_t>(p->dval2), ptr<uint32_t>(p->ntiles), NV});
    auto offsets_scan = [&]() {
      return cub_call(p, s, [&](void *tmp, size_t &bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt_it, ptr<uint32_t>(p->off_sorted),
                                             (int)(NV + 1), s);
      });
    };
    TS_CUDA_TRY(offsets_scan());
    // partial-moment slot base of every gv (gv order): one slot per bbox quadrant
    cub::TransformInputIterator<uint32_t, QuadCount, cub::CountingInputIterator<int64_t>> q_it(
        cub::CountingInputIterator<int64_t>(0), QuadCount{ptr<int16_t>(p->bbox), NV});
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return cub::DeviceScan::ExclusiveSum(tmp, bytes, q_it, ptr<uint32_t>(p->inst_base),
                                           (int)(NV + 1), s);
    }));
    // instance and slot totals (the scans' last entries)
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_small, ptr<uint32_t>(p->off_sorted) + NV, 4,
                                cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_small + 1, ptr<uint32_t>(p->inst_base) + NV, 4,
                                cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_small + 2, p->tie_runs.p, 4, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_rects, ptr<uint32_t>(p->drange) + K1_RECT_OFFSET,
                                16 * V, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaStreamSynchronize(s));
    p->n_inst = (int64_t)p->host_small[0];
    p->n_slots = (int64_t)p->host_small[1];
    const uint32_t n_long = p->host_small[2];
    if (n_long > 0) {
      // rare path (degenerate geometry): runs of > K1_TIE_RUN_MAX equal quantised keys, sorted
      // by the exact depth bits with a stable segmented radix sort -- stable, so equal depths
      // keep the gid order of the quantised sort's input (splat.py:178) -- then the depth-order
      // offsets are rescanned (the set of gvs, hence the totals, is unchanged)
      if (n_long > long_cap) return TS_E_CAPACITY;
      ENSURE(p->tie_tmp, 20 * NV + 8 * (int64_t)n_long + 64);
      uint64_t *kin = ptr<uint64_t>(p->tie_tmp), *kout = kin + NV;
      uint32_t *vout = reinterpret_cast<uint32_t *>(kout + NV), *rb = vout + NV, *re = rb + n_long;
      launch_k1_long_run_keys(ptr<uint32_t>(p->dval2), ptr<double>(p->depth64), NV,
                              ptr<uint32_t>(p->tie_runs), n_long, kin, rb, re, s);
      TS_CUDA_TRY(cudaMemcpyAsync(vout, p->dval2.p, 4 * NV, cudaMemcpyDeviceToDevice, s));
      TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
        return cub::DeviceSegmentedRadixSort::SortPairs(tmp, bytes, kin, kout,
                                                        ptr<uint32_t>(p->dval2), vout, (int)NV,
                                                        (int)n_long, rb, re, 0, 64, s);
      }));
      TS_CUDA_TRY(cudaMemcpyAsync(p->dval2.p, vout, 4 * NV, cudaMemcpyDeviceToDevice, s));
      TS_CUDA_TRY(offsets_scan());
    }
  } else {
    p->n_inst = 0;
    p->n_slots = 0;
  }
  p->mark_end(ST_DEPTH_SORT, e1, s);

  cudaEvent_t e2 = p->mark_begin(s);
  const int64_t ni = p->n_inst;
  ENSURE(p->tkey, 4 * (ni + 1));
  ENSURE(p->tkey2, 4 * (ni + 1));
  ENSURE(p->tval, 4 * (ni + 1));
  ENSURE(p->tval2, 4 * (ni + 1));
  if (ni == 0) TS_CUDA_TRY(cudaMemsetAsync(p->range.p, 0, 8 * ntile_total, s));
  if (ni > 0) {
    launch_k1_emit(ptr<uint32_t>(p->dval2), ptr<int16_t>(p->bbox), ptr<uint32_t>(p->off_sorted),
                   NV, p->tiles_x, ptr<uint32_t>(p->tkey), ptr<uint32_t>(p->tval), s);
    const int tbits = bits_for((uint64_t)p->tpv);  // tile within the view (see binning.cu)
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return k1_sort_pairs(tmp, bytes, ptr<uint32_t>(p->tkey), ptr<uint32_t>(p->tkey2),
                           ptr<uint32_t>(p->tval), ptr<uint32_t>(p->tval2), (int)ni, tbits, s);
    }));
    launch_k1_tile_ranges(ptr<uint32_t>(p->tkey2), ptr<uint32_t>(p->tval2), ni, n, V, p->tpv,
                          ptr<uint32_t>(p->range), s);
  }
  TS_CUDA_TRY(cudaGetLastError());
  p->mark_end(ST_TILE_SORT, e2, s);
  return TS_OK;
}

// Debug: TS_K2_STATS=1 makes ts_frame_compensate print K2's work counters to stderr.
unsigned long long *k2_stats(ts_plan *p, cudaStream_t s) {
  static const bool on = getenv("TS_K2_STATS") != nullptr;
  if (!on) return nullptr;
  if (p->k2_stats.ensure(16 * 8, s) != cudaSuccess) return nullptr;
  cudaMemsetAsync(p->k2_stats.p, 0, 16 * 8, s);
  return p->k2_stats.as<unsigned long long>();
}

void k2_stats_report(ts_plan *p, cudaStream_t s) {
  static const bool on = getenv("TS_K2_STATS") != nullptr;
  if (!on || !p->k2_stats.p) return;
  unsigned long long h[16];
  cudaMemcpyAsync(h, p->k2_stats.p, 10 * 8, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  fprintf(stderr, "K2 stats: units %llu chunks %llu instances %llu hits %llu skips %llu "
          "eval_gauss %llu eval_pix %llu contrib %llu flushes %llu eval_empty %llu\n", h[0], h[1],
          h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
}

ts_motions internal_motions(ts_plan *p) {
  ts_motions m;
  m.status = ptr<int8_t>(p->mot_status);
  m.a = ptr<double>(p->mot_a);
  m.b = ptr<double>(p->mot_b);
  m.weight_sum = ptr<double>(p->mot_w);
  m.pixel_count = ptr<int32_t>(p->mot_cnt);
  m.static_pixel_count = ptr<int32_t>(p->mot_scnt);
  m.static_weight_sum = ptr<double>(p->mot_sw);
  return m;
}

}  // namespace

extern "C" {

int ts_version(void) { return 1; }

const char *ts_error_string(int code) {
  switch (code) {
    case TS_OK: return "ok";
    case TS_E_INVALID_ARGUMENT: return "invalid argument";
    case TS_E_DIMENSION_MISMATCH: return "dimension mismatch";
    case TS_E_CUDA: return "CUDA runtime error";
    case TS_E_OUT_OF_MEMORY: return "out of device memory";
    case TS_E_CAPACITY: return "capacity exceeded";
    default: return "unknown error";
  }
}

int ts_plan_create(ts_plan **plan) {
  if (!plan) return TS_E_INVALID_ARGUMENT;
  ts_plan *p = new (std::nothrow) ts_plan();
  if (!p) return TS_E_OUT_OF_MEMORY;
  p->cfg.alpha_cutoff = 1.0 / 255.0;
  p->cfg.early_stop = 1e-4;
  p->cfg.det_floor = 1e-12;
  p->cfg.min_weight = 1e-3;
  p->cfg.min_total_weight = 1e-3;
  p->cfg.static_threshold_px = 1.0;
  p->cfg.eig_floor = 1e-12;
  p->cfg.min_pixels = 3;
  p->cfg.min_views = 2;
  p->cfg.min_total_pixels = 3;
  *plan = p;
  return TS_OK;
}

int ts_plan_destroy(ts_plan *p) {
  if (!p) return TS_OK;
  cudaDeviceSynchronize();
  release_all(p);
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  if (p->host_small) cudaFreeHost(p->host_small);
  if (p->host_rects) cudaFreeHost(p->host_rects);
  delete p;
  return TS_OK;
}

int64_t ts_plan_workspace_bytes(const ts_plan *p) { return p ? sum_workspace(p) : 0; }

// Stage timing (CUDA events on the plan's launch stream), used by bench.py for the roofline.
int ts_plan_set_k2_ctas_per_sm(ts_plan *p, int32_t ctas_per_sm) {
  if (!p || ctas_per_sm < 0) return TS_E_INVALID_ARGUMENT;
  p->k2_ctas_per_sm = ctas_per_sm;
  return TS_OK;
}

int ts_plan_timing(ts_plan *p, int enable) {
  if (!p) return TS_E_INVALID_ARGUMENT;
  p->timing = enable != 0;
  p->ev_marks.clear();
  p->ev_next = 0;
  return TS_OK;
}

// Sums the recorded stage times (ms) into totals[ST_N] and counts[ST_N]; synchronises the events.
int ts_plan_timing_read(ts_plan *p, double *totals_ms, int32_t *counts, int32_t n_stages) {
  if (!p || !totals_ms || n_stages < ST_N) return TS_E_INVALID_ARGUMENT;
  for (int i = 0; i < n_stages; i++) {
    totals_ms[i] = 0.0;
    if (counts) counts[i] = 0;
  }
  for (auto &m : p->ev_marks) {
    TS_CUDA_TRY(cudaEventSynchronize(m.second.second));
    float ms = 0.f;
    TS_CUDA_TRY(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
    totals_ms[m.first] += ms;
    if (counts) counts[m.first]++;
  }
  return TS_OK;
}

int ts_project(const double *gaussians, int64_t n, const ts_camera *camera, double *mean2,
               double *depth, double *cov2, uint8_t *in_front, void *stream) {
  if (!camera || n < 0) return TS_E_INVALID_ARGUMENT;
  launch_project_view(gaussians, n, *camera, mean2, depth, cov2, in_front, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_frame_bin(ts_plan *plan, const double *gaussians, int64_t n, const ts_camera *cameras,
                 int32_t n_views, const ts_config *config, void *stream) {
  if (!plan) return TS_E_INVALID_ARGUMENT;
  return frame_bin(plan, gaussians, n, cameras, n_views, config, (cudaStream_t)stream);
}

int ts_frame_compensate(ts_plan *p, const void *track_target, int32_t track_dtype,
                        const uint8_t *track_valid, const ts_motions *motions,
                        const ts_updates *updates, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || p->V < 1) return TS_E_INVALID_ARGUMENT;
  if (!updates && !motions) return TS_E_INVALID_ARGUMENT;  // nothing would be returned
  if (track_dtype != TS_TRACK_F32 && track_dtype != TS_TRACK_F64) return TS_E_INVALID_ARGUMENT;
  const int64_t n = p->n, NV = n * p->V;
  // tracks: device memory, or pinned host memory that K2 reads in place (zero-copy: only the
  // 8x8 quadrants of occupied tiles cross PCIe)
  {
    int kt = 0, kv = 0;
    int rc = device_view(track_target, &track_target, &kt);
    if (rc) return rc;
    rc = device_view(track_valid, reinterpret_cast<const void **>(&track_valid), &kv);
    if (rc) return rc;
    (void)kt;  // each array on the device or in pinned host memory
    (void)kv;
  }
  const int64_t ns = p->n_slots;  // one partial slot per (gv, bbox quadrant)
  ENSURE(p->partial, sizeof(Partial) * (ns + 1));
  ENSURE(p->flag, ns + 8);  // K3 reads the flags as aligned 32-bit words
  ts_motions m = motions ? *motions : ts_motions{};
  ts_motions im;
  {
    ENSURE(p->mot_status, NV + 1);
    ENSURE(p->mot_a, 32 * (NV + 1));
    ENSURE(p->mot_b, 16 * (NV + 1));
    ENSURE(p->mot_w, 8 * (NV + 1));
    ENSURE(p->mot_cnt, 4 * (NV + 1));
    ENSURE(p->mot_scnt, 4 * (NV + 1));
    ENSURE(p->mot_sw, 8 * (NV + 1));
    im = internal_motions(p);
  }
  if (!m.status) m.status = im.status;
  if (!m.a) m.a = im.a;
  if (!m.b) m.b = im.b;
  if (!m.weight_sum) m.weight_sum = im.weight_sum;
  if (!m.pixel_count) m.pixel_count = im.pixel_count;

  const bool cached = p->cache_valid;
  // no motions requested and K3's fits compact (cache or touched list): K4 reads the fits in
  // place and only the statuses are written densely, by the fit kernels themselves over an
  // UNSOLVABLE fill (the per-view motions are intermediates of compensate_frame,
  // pipeline.py:117-124; FrameResult does not carry them)
  bool compact = false;
  if (cached) {
    compact = !motions && updates;
    // the clip's contribution cache: this frame's moments and fits straight from the cached
    // contributions (no rasterization, no partials); list, ranks and ranges set by ts_frame_cache
    uint32_t *list = ptr<uint32_t>(p->k3_list);
    cudaEvent_t e3 = p->mark_begin(s);
    // compact: the fit kernels write the listed gvs' statuses over an UNSOLVABLE fill
    if (compact) TS_CUDA_TRY(cudaMemsetAsync(m.status, TS_STATUS_UNSOLVABLE, (size_t)NV, s));
    TS_CUDA_TRY(launch_k23_cached(p->cache_chunks.p, ptr<uint32_t>(p->cache_counters),
                                  p->cache_chunk_bound, p->cache_multi.p, p->cache_multi_bound,
                                  list, ptr<int16_t>(p->bbox), n, p->W, p->H,
                                  ptr<double>(p->cache_w), ptr<uint32_t>(p->cache_xy),
                                  track_target, track_dtype, track_valid, p->cfg, p->k3_fits.p,
                                  ptr<double>(p->cache_scratch), s,
                                  compact ? m.status : nullptr));
    p->mark_end(ST_RASTER, e3, s);
    cudaEvent_t e4 = p->mark_begin(s);
    if (!compact)
      launch_k3_merge(ptr<uint8_t>(p->touched), ptr<uint32_t>(p->k3_rank), p->k3_fits.p, NV, m,
                      s);
    TS_CUDA_TRY(cudaGetLastError());
    p->mark_end(ST_SOLVE, e4, s);
  } else {
  ENSURE(p->k2_sched, k2_schedule_bytes(p->tpv * p->V));
  // K3 split (touched-gv list + compact fits + merge) vs one thread per gv over all gvs: the
  // split pays off when most gvs get no contribution (cfg5: 7% touched, K3 2.47 -> 1.27 ms),
  // the single pass when many do (cfg2: ~40%, 0.44 vs 0.50 ms).  The plan keeps the touched
  // fraction of its previous frame (copied back asynchronously; read after the next binning's
  // stream synchronisation); the first frame splits from 16 M gvs on.  Without requested motions
  // the split also spares the dense motion stores (K4 reads the compact fits, statuses written
  // over an UNSOLVABLE fill), so it is taken from 4 M gvs on and kept up to half the gvs touched
  // (cfg4, 10 M gvs: K3 0.61 -> 0.48 ms, step 4.19 -> 4.03 ms; cfg2, 6 M gvs, 40% touched:
  // step 3.64 -> 3.59 ms; cfg3 2.60 -> 2.59 ms).  TS_K3_SPLIT=0/1 forces.
  static const char *force = getenv("TS_K3_SPLIT");
  const bool lean = !motions && updates;
  bool split;
  if (force && force[0]) {
    split = force[0] != '0';
  } else if (p->k3_last_nv == NV && p->k3_last_split) {
    split = (double)p->host_small[8] < (lean ? 0.5 : 0.25) * (double)NV;
  } else if (p->k3_last_nv == NV) {
    split = false;  // sticky: the single pass does not measure the touched fraction
  } else {
    split = NV >= (int64_t)(lean ? 4 : 16) << 20;
  }
  p->k3_last_nv = NV;
  p->k3_last_split = split;
  const bool use_touched = split && k2_writes_touched();
  compact = use_touched && !motions && updates;
  if (use_touched) {
    ENSURE(p->touched, NV + 8);
    ENSURE(p->k3_list, 4 * (NV + 8));
    ENSURE(p->k3_rank, 4 * (NV + 8));
    ENSURE(p->k3_fits, k3_fit_bytes() * (NV + 1));
  }
  cudaEvent_t e3 = p->mark_begin(s);
  TS_CUDA_TRY(cudaMemsetAsync(p->flag.p, 0, ns + 8, s));
  if (use_touched) TS_CUDA_TRY(cudaMemsetAsync(p->touched.p, 0, NV + 8, s));
  TS_CUDA_TRY(launch_k2(K2_ACCUMULATE, track_dtype, ptr<RasterRec>(p->rec), ptr<uint32_t>(p->tval2),
                        ptr<uint32_t>(p->range), ptr<uint32_t>(p->inst_base),
                        ptr<uint32_t>(p->items), ptr<uint32_t>(p->counters), 0, p->tpv * p->V,
                        track_target, track_valid, p->W, p->H, p->tiles_x, p->tpv, p->cfg,
                        ptr<Partial>(p->partial), ptr<uint8_t>(p->flag), nullptr, 0, nullptr,
                        nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, k2_stats(p, s),
                        p->k2_sched.p, s, p->k2_ctas_per_sm,
                        use_touched ? ptr<uint8_t>(p->touched) : nullptr));
  k2_stats_report(p, s);
  p->mark_end(ST_RASTER, e3, s);

  // K3 and K4 stay separate: a fused per-Gaussian K3+K4 serialises the memory-bound per-view
  // fits inside a 200-register thread and measured 3.0 ms vs 0.6 + 1.5 ms (cfg2).
  cudaEvent_t e4 = p->mark_begin(s);
  if (use_touched) {  // the touched gvs in gv order (K3's fits), count on the device, ranks
    uint32_t *list = ptr<uint32_t>(p->k3_list), *n_list = list + NV + 4;
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return cub::DeviceSelect::Flagged(tmp, bytes, cub::CountingInputIterator<uint32_t>(0),
                                        ptr<uint8_t>(p->touched), list, n_list, (int)NV, s);
    }));
    cub::TransformInputIterator<uint32_t, ByteToU32, const uint8_t *> t_it(
        ptr<uint8_t>(p->touched), ByteToU32{});
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return cub::DeviceScan::ExclusiveSum(tmp, bytes, t_it, ptr<uint32_t>(p->k3_rank), (int)NV,
                                           s);
    }));
  }
  launch_k3_solve(ptr<Partial>(p->partial), ptr<uint8_t>(p->flag), ptr<uint32_t>(p->inst_base),
                  ptr<uint32_t>(p->ntiles), ptr<int16_t>(p->bbox), NV, p->cfg, m,
                  use_touched ? ptr<uint8_t>(p->touched) : nullptr,
                  use_touched ? ptr<uint32_t>(p->k3_list) : nullptr,
                  use_touched ? ptr<uint32_t>(p->k3_list) + NV + 4 : nullptr,
                  use_touched ? ptr<uint32_t>(p->k3_rank) : nullptr,
                  use_touched ? p->k3_fits.p : nullptr, s, compact);
  if (use_touched)  // touched count for the next frame's choice
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_small + 8, ptr<uint32_t>(p->k3_list) + NV + 4, 4,
                                cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(cudaGetLastError());
  p->mark_end(ST_SOLVE, e4, s);
  }

  if (!updates) return TS_OK;  // K2 + K3 only: the caller fuses (ts_update_all) over more views
  ENSURE(p->k4_ws, k4_workspace_bytes(n));
  cudaEvent_t e5 = p->mark_begin(s);
  launch_k4_fuse(p->gaussians, n, ptr<ts_camera>(p->cams), p->V, m, p->cfg, *updates,
                 p->k4_ws.p, s, compact ? p->k3_fits.p : nullptr,
                 compact ? ptr<uint32_t>(p->k3_rank) : nullptr);
  TS_CUDA_TRY(cudaGetLastError());
  p->mark_end(ST_FUSE, e5, s);
  return TS_OK;
}

int ts_frame_cache(ts_plan *p, int32_t enable, void *stream) {
  if (!p) return TS_E_INVALID_ARGUMENT;
  if (!enable) {
    p->cache_valid = false;
    return TS_OK;
  }
  if (p->V < 1) return TS_E_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p->n, NV = n * p->V, ns = p->n_slots;
  ENSURE(p->partial, sizeof(Partial) * (ns + 1));
  ENSURE(p->flag, ns + 8);
  ENSURE(p->touched, NV + 8);
  ENSURE(p->k3_list, 4 * (NV + 8));
  ENSURE(p->k3_rank, 4 * (NV + 8));
  ENSURE(p->k3_fits, k3_fit_bytes() * (NV + 1));
  ENSURE(p->k2_sched, k2_schedule_bytes(p->tpv * p->V));
  ENSURE(p->cache_cursor, 16);  // [0] pool doubles handed out, [1] records handed out
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // every K2 warp may leave most of one pool chunk and one record chunk unused
  const uint64_t warps = (uint64_t)sms * 8 * 4;
  const uint64_t slack = warps * K2_CACHE_CHUNK, rslack = warps * K2_CACHE_RECS;
  if (p->cache_cap == 0) p->cache_cap = (uint64_t)std::max<int64_t>(4 * ns, 1 << 22) + slack;
  if (p->cache_rec_cap == 0) p->cache_rec_cap = (uint64_t)std::max<int64_t>(ns / 2, 1 << 16) + rslack;
  unsigned long long *cur = ptr<unsigned long long>(p->cache_cursor);
  for (int attempt = 0; attempt < 3; attempt++) {
    ENSURE(p->cache_pool, 8 * p->cache_cap);
    ENSURE(p->cache_recs, sizeof(CacheRec) * p->cache_rec_cap);
    TS_CUDA_TRY(cudaMemsetAsync(p->flag.p, 0, ns + 8, s));
    TS_CUDA_TRY(cudaMemsetAsync(p->touched.p, 0, NV + 8, s));
    TS_CUDA_TRY(cudaMemsetAsync(cur, 0, 16, s));
    TS_CUDA_TRY(launch_k2(K2_CACHE, TS_TRACK_F32, ptr<RasterRec>(p->rec), ptr<uint32_t>(p->tval2),
                          ptr<uint32_t>(p->range), ptr<uint32_t>(p->inst_base),
                          ptr<uint32_t>(p->items), ptr<uint32_t>(p->counters), 0,
                          p->tpv * p->V, nullptr, nullptr, p->W, p->H, p->tiles_x, p->tpv,
                          p->cfg, ptr<Partial>(p->partial), ptr<uint8_t>(p->flag), nullptr, 0,
                          nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                          p->k2_sched.p, s, p->k2_ctas_per_sm, ptr<uint8_t>(p->touched),
                          ptr<double>(p->cache_pool), cur, p->cache_cap,
                          ptr<CacheRec>(p->cache_recs), cur + 1, p->cache_rec_cap));
    uint64_t used[2] = {0, 0};
    TS_CUDA_TRY(cudaMemcpyAsync(used, cur, 16, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaStreamSynchronize(s));
    const bool pool_ok = used[0] <= p->cache_cap, recs_ok = used[1] <= p->cache_rec_cap;
    if (pool_ok && recs_ok) {
      p->cache_used = used[0];
      p->cache_recs_used = used[1];
      break;
    }
    // too small: grow and rebuild
    if (!pool_ok) p->cache_cap = used[0] + used[0] / 8 + slack;
    if (!recs_ok) p->cache_rec_cap = used[1] + used[1] / 8 + rslack;
    if (attempt == 2) return TS_E_CAPACITY;
  }
  // the touched gvs (any cached contribution) and their ranks: fixed for the clip
  uint32_t *list = ptr<uint32_t>(p->k3_list), *n_list = list + NV + 4;
  TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
    return cub::DeviceSelect::Flagged(tmp, bytes, cub::CountingInputIterator<uint32_t>(0),
                                      ptr<uint8_t>(p->touched), list, n_list, (int)NV, s);
  }));
  cub::TransformInputIterator<uint32_t, ByteToU32, const uint8_t *> t_it(ptr<uint8_t>(p->touched),
                                                                        ByteToU32{});
  TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, t_it, ptr<uint32_t>(p->k3_rank), (int)NV, s);
  }));
  // the records in slot order: per-slot counts, their offsets, the contributions scattered
  // there (every gv's run contiguous), the run of every listed gv
  if (p->cache_used >= (uint64_t)1 << 32) return TS_E_CAPACITY;  // 32-bit contribution offsets
  ENSURE(p->cache_cnt, 4 * (ns + 1));
  ENSURE(p->cache_off, 4 * (ns + 1));
  ENSURE(p->cache_w, 8 * (p->cache_used + 1));
  ENSURE(p->cache_xy, 4 * (p->cache_used + 1));
  ENSURE(p->cache_ranges, 8 * (NV + 1));
  TS_CUDA_TRY(cudaMemsetAsync(p->cache_cnt.p, 0, 4 * (ns + 1), s));
  launch_cache_slot_counts(ptr<CacheRec>(p->cache_recs), cur + 1, p->cache_rec_cap,
                           ptr<uint32_t>(p->cache_cnt), s, p->cache_recs_used);
  TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, ptr<uint32_t>(p->cache_cnt),
                                         ptr<uint32_t>(p->cache_off), (int)(ns + 1), s);
  }));
  launch_cache_scatter(ptr<CacheRec>(p->cache_recs), cur + 1, p->cache_rec_cap,
                       ptr<double>(p->cache_pool), ptr<uint32_t>(p->cache_off),
                       ptr<double>(p->cache_w), ptr<uint32_t>(p->cache_xy), s,
                       p->cache_recs_used);
  launch_cache_ranges(list, n_list, NV, ptr<int16_t>(p->bbox), ptr<uint32_t>(p->inst_base),
                      ptr<uint32_t>(p->cache_off), ptr<uint2>(p->cache_ranges), s);
  // the per-frame work units: every gv's run cut into chunks of at most cache_chunk_len()
  uint32_t counts[2] = {0, 0};  // touched gvs, cached contributions
  TS_CUDA_TRY(cudaMemcpyAsync(counts, n_list, 4, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(cudaMemcpyAsync(counts + 1, ptr<uint32_t>(p->cache_off) + ns, 4,
                              cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(cudaStreamSynchronize(s));
  const uint64_t nl = counts[0], total = counts[1], cl = (uint64_t)cache_chunk_len();
  p->cache_chunk_bound = nl + total / cl + 1;
  p->cache_multi_bound = total / cl + 1;  // a split gv holds more than cl contributions
  uint32_t *nch = ptr<uint32_t>(p->cache_cnt), *choff = ptr<uint32_t>(p->cache_off);  // reused
  ENSURE(p->cache_chunks, cache_chunk_bytes() * p->cache_chunk_bound);
  ENSURE(p->cache_multi, cache_multi_bytes() * p->cache_multi_bound);
  ENSURE(p->cache_scratch, cache_scratch_bytes() * (2 * total / cl + 1));
  ENSURE(p->cache_counters, 16);
  TS_CUDA_TRY(cudaMemsetAsync(nch, 0, 4 * (nl + 1), s));
  TS_CUDA_TRY(cudaMemsetAsync(p->cache_counters.p, 0, 16, s));
  launch_cache_chunk_counts(n_list, NV, ptr<uint2>(p->cache_ranges), nch, s);
  TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, nch, choff, (int)(nl + 1), s);
  }));
  launch_cache_chunk_fill(list, n_list, NV, ptr<int16_t>(p->bbox), n,
                          ptr<uint2>(p->cache_ranges), nch, choff,
                          p->cache_chunks.p, p->cache_multi.p,
                          ptr<uint32_t>(p->cache_counters), s);
  TS_CUDA_TRY(cudaGetLastError());
  p->cache_valid = true;
  return TS_OK;
}

int ts_frame_cache_info(const ts_plan *p, uint64_t *n_records, uint64_t *n_values) {
  if (!p || !n_records || !n_values) return TS_E_INVALID_ARGUMENT;
  *n_records = p->cache_valid ? p->cache_recs_used : 0;
  *n_values = p->cache_valid ? p->cache_used : 0;
  return TS_OK;
}

int ts_frame_track_rects(const ts_plan *p, int32_t *rects) {
  if (!p || !rects || p->V < 1 || !p->host_rects) return TS_E_INVALID_ARGUMENT;
  for (int v = 0; v < p->V; v++) {
    const int32_t *r = p->host_rects + 4 * v;
    int32_t *o = rects + 4 * v;
    if (p->n == 0 || r[2] < 0) {  // no binned Gaussian in this view: nothing is read
      o[0] = o[1] = 0;
      o[2] = o[3] = -1;
      continue;
    }
    // K2 reads whole 8x8 quadrants of every touched 16x16 tile
    o[0] = (r[0] / TS_TILE) * TS_TILE;
    o[1] = (r[1] / TS_TILE) * TS_TILE;
    o[2] = std::min(((r[2] / TS_TILE) + 1) * TS_TILE, p->W) - 1;
    o[3] = std::min(((r[3] / TS_TILE) + 1) * TS_TILE, p->H) - 1;
  }
  return TS_OK;
}

int ts_copy_track_rects(const ts_plan *p, const void *host_target, int32_t track_dtype,
                        const uint8_t *host_valid, void *dev_target, uint8_t *dev_valid,
                        void *stream) {
  if (!p || !host_target || !host_valid || !dev_target || !dev_valid) return TS_E_INVALID_ARGUMENT;
  if (track_dtype != TS_TRACK_F32 && track_dtype != TS_TRACK_F64) return TS_E_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int32_t> r(4 * (size_t)p->V);
  int rc = ts_frame_track_rects(p, r.data());
  if (rc) return rc;
  const size_t px = track_dtype == TS_TRACK_F32 ? 8 : 16;  // bytes per target pixel (u, v)
  const size_t W = (size_t)p->W, H = (size_t)p->H;
  for (int v = 0; v < p->V; v++) {
    const int x0 = r[4 * v], y0 = r[4 * v + 1], x1 = r[4 * v + 2], y1 = r[4 * v + 3];
    if (x1 < x0 || y1 < y0) continue;
    const size_t off = ((size_t)v * H + (size_t)y0) * W + (size_t)x0;
    const size_t w = (size_t)(x1 - x0 + 1), h = (size_t)(y1 - y0 + 1);
    TS_CUDA_TRY(cudaMemcpy2DAsync(static_cast<char *>(dev_target) + off * px, W * px,
                                  static_cast<const char *>(host_target) + off * px, W * px,
                                  w * px, h, cudaMemcpyHostToDevice, s));
    TS_CUDA_TRY(cudaMemcpy2DAsync(dev_valid + off, W, host_valid + off, W, w, h,
                                  cudaMemcpyHostToDevice, s));
  }
  return TS_OK;
}

int ts_frame_occupied_tiles(const ts_plan *p, int64_t *out) {
  if (!p || !out) return TS_E_INVALID_ARGUMENT;
  const int64_t nt = (int64_t)p->tpv * p->V;
  std::vector<uint32_t> r(2 * nt);
  if (nt && cudaMemcpy(r.data(), p->range.p, 8 * nt, cudaMemcpyDeviceToHost) != cudaSuccess)
    return TS_E_CUDA;
  int64_t c = 0;
  for (int64_t t = 0; t < nt; t++) c += r[2 * t] < r[2 * t + 1];
  *out = c;
  return TS_OK;
}

int ts_frame_binning(const ts_plan *p, ts_binning *out) {
  if (!p || !out) return TS_E_INVALID_ARGUMENT;
  out->n_instances = p->n_inst;
  out->tiles_x = p->tiles_x;
  out->tiles_y = p->tiles_y;
  out->n_views = p->V;
  out->inst_tile = p->tkey2.as<uint32_t>();
  out->inst_gv = p->tval2.as<uint32_t>();
  out->tile_range = p->range.as<uint32_t>();
  out->gv_status = p->status.as<int8_t>();
  out->gv_bbox = p->bbox.as<int16_t>();
  return TS_OK;
}

int ts_rasterize_weights(ts_plan *p, const double *gaussians, int64_t n, const ts_camera *camera,
                         double alpha_cutoff, double early_stop, int64_t *n_out,
                         int64_t *n_degenerate_out, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || !camera || !n_out) return TS_E_INVALID_ARGUMENT;
  if (!(alpha_cutoff > 0.0 && alpha_cutoff < 1.0)) return TS_E_INVALID_ARGUMENT;
  ts_config cfg = p->cfg;
  cfg.alpha_cutoff = alpha_cutoff;
  cfg.early_stop = early_stop;
  int rc = frame_bin(p, gaussians, n, camera, 1, &cfg, s);
  if (rc) return rc;
  // degenerate ids (splat.py:135-137), ascending
  ENSURE(p->deg_flags, n + 1);
  ENSURE(p->deg_ids, 8 * (n + 1));
  ENSURE(p->deg_count, 8);
  if (n > 0) {
    k_degenerate_flags<<<nblk(n, 256), 256, 0, s>>>(ptr<int8_t>(p->status), n, ptr<uint8_t>(p->deg_flags));
    cub::CountingInputIterator<int64_t> it(0);
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return cub::DeviceSelect::Flagged(tmp, bytes, it, ptr<uint8_t>(p->deg_flags),
                                        ptr<int64_t>(p->deg_ids), ptr<int64_t>(p->deg_count), (int)n,
                                        s);
    }));
  } else {
    TS_CUDA_TRY(cudaMemsetAsync(p->deg_count.p, 0, 8, s));
  }
  int64_t cap = p->emit_key.bytes / 8;
  for (int attempt = 0; attempt < 2; attempt++) {
    if (cap > 0) {
      ENSURE(p->emit_key, 8 * cap);
      ENSURE(p->emit_gv, 4 * cap);
      ENSURE(p->emit_alpha, 8 * cap);
      ENSURE(p->emit_trans, 8 * cap);
    }
    ENSURE(p->emit_count, 8);
    TS_CUDA_TRY(cudaMemsetAsync(p->emit_count.p, 0, 8, s));
    TS_CUDA_TRY(launch_k2(K2_EMIT, TS_TRACK_F32, ptr<RasterRec>(p->rec), ptr<uint32_t>(p->tval2),
                          ptr<uint32_t>(p->range), ptr<uint32_t>(p->inst_base),
                          ptr<uint32_t>(p->items), ptr<uint32_t>(p->counters), 0, p->tpv, nullptr,
                          nullptr, p->W, p->H, p->tiles_x, p->tpv, cfg, nullptr, nullptr,
                          ptr<unsigned long long>(p->emit_count), cap, ptr<uint64_t>(p->emit_key),
                          ptr<uint32_t>(p->emit_gv), ptr<double>(p->emit_alpha),
                          ptr<double>(p->emit_trans), nullptr, nullptr, nullptr, nullptr,
                          nullptr, s));
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_small, p->emit_count.p, 8, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaMemcpyAsync(p->host_small + 2, p->deg_count.p, 8, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(cudaStreamSynchronize(s));
    uint64_t got = 0;
    std::memcpy(&got, p->host_small, 8);
    std::memcpy(&p->n_deg, p->host_small + 2, 8);
    if ((int64_t)got <= cap) {
      p->emit_n = (int64_t)got;
      break;
    }
    cap = (int64_t)got;
  }
  const int64_t m = p->emit_n;
  ENSURE(p->emit_key2, 8 * (m + 1));
  ENSURE(p->emit_idx, 4 * (m + 1));
  ENSURE(p->emit_idx2, 4 * (m + 1));
  if (m > 0) {
    k_iota<<<nblk(m, 256), 256, 0, s>>>(ptr<uint32_t>(p->emit_idx), m);
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, ptr<uint64_t>(p->emit_key),
                                             ptr<uint64_t>(p->emit_key2), ptr<uint32_t>(p->emit_idx),
                                             ptr<uint32_t>(p->emit_idx2), (int)m, 0, 64, s);
    }));
  }
  TS_CUDA_TRY(cudaGetLastError());
  *n_out = m;
  if (n_degenerate_out) *n_degenerate_out = p->n_deg;
  return TS_OK;
}

int ts_rasterize_fetch(ts_plan *p, int32_t *pixel_x, int32_t *pixel_y, int64_t *gaussian_id,
                       double *alpha, double *transmittance, double *depth,
                       int64_t *degenerate_ids, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p) return TS_E_INVALID_ARGUMENT;
  const int64_t m = p->emit_n;
  if (m > 0)
    k_fetch_contribs<<<nblk(m, 256), 256, 0, s>>>(
        ptr<uint64_t>(p->emit_key2), ptr<uint32_t>(p->emit_idx2), ptr<uint32_t>(p->emit_gv),
        ptr<double>(p->emit_alpha), ptr<double>(p->emit_trans), ptr<RasterRec>(p->rec),
        ptr<double>(p->depth64), m, p->W, pixel_x, pixel_y, gaussian_id, alpha, transmittance,
        depth);
  if (p->n_deg > 0 && degenerate_ids)
    TS_CUDA_TRY(cudaMemcpyAsync(degenerate_ids, p->deg_ids.p, 8 * p->n_deg,
                                cudaMemcpyDeviceToDevice, s));
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_accumulate_view(ts_plan *p, const int32_t *pixel_x, const int32_t *pixel_y,
                       const int64_t *gaussian_id, const double *alpha,
                       const double *transmittance, int64_t m, int32_t width, int32_t height,
                       const void *track_target, int32_t track_dtype, const uint8_t *track_valid,
                       int64_t n, double static_threshold_px, double *v1, double *v2,
                       double *weight_sum, int64_t *pixel_count, int64_t *static_pixel_count,
                       double *static_weight_sum, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || m < 0 || n < 0 || width <= 0 || height <= 0) return TS_E_INVALID_ARGUMENT;
  if (track_dtype != TS_TRACK_F32 && track_dtype != TS_TRACK_F64) return TS_E_INVALID_ARGUMENT;
  if (n >= 0xFFFFFFFFll || m >= 0xFFFFFFFFll) return TS_E_INVALID_ARGUMENT;
  ENSURE(p->seg_start, 4 * (n + 1));
  ENSURE(p->seg_end, 4 * (n + 1));
  ENSURE(p->acc_keys, 4 * (m + 1));
  ENSURE(p->acc_keys2, 4 * (m + 1));
  ENSURE(p->acc_iota, 4 * (m + 1));
  ENSURE(p->acc_order, 4 * (m + 1));
  TS_CUDA_TRY(cudaMemsetAsync(p->seg_start.p, 0, 4 * (n + 1), s));
  TS_CUDA_TRY(cudaMemsetAsync(p->seg_end.p, 0, 4 * (n + 1), s));
  if (m > 0) {
    k_gid_keys<<<nblk(m, 256), 256, 0, s>>>(gaussian_id, ptr<uint32_t>(p->acc_keys), m);
    k_iota<<<nblk(m, 256), 256, 0, s>>>(ptr<uint32_t>(p->acc_iota), m);
    const int kb = bits_for((uint64_t)n + 1);
    TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
      return cub::DeviceRadixSort::SortPairs(tmp, bytes, ptr<uint32_t>(p->acc_keys),
                                             ptr<uint32_t>(p->acc_keys2), ptr<uint32_t>(p->acc_iota),
                                             ptr<uint32_t>(p->acc_order), (int)m, 0, kb, s);
    }));
    launch_segment_bounds(ptr<uint32_t>(p->acc_keys2), m, ptr<uint32_t>(p->seg_start),
                          ptr<uint32_t>(p->seg_end), s);
  }
  launch_accumulate(n, ptr<uint32_t>(p->seg_start), ptr<uint32_t>(p->seg_end),
                    ptr<uint32_t>(p->acc_order), pixel_x, pixel_y, alpha, transmittance, width,
                    track_target, track_dtype, track_valid, static_threshold_px, v1, v2,
                    weight_sum, pixel_count, static_pixel_count, static_weight_sum, s);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_solve_view(const double *v1, const double *v2, const double *weight_sum,
                  const int64_t *pixel_count, int64_t n, double det_floor, int32_t min_pixels,
                  double min_weight, int8_t *status, double *a, double *b, double *det,
                  void *stream) {
  if (n < 0) return TS_E_INVALID_ARGUMENT;
  launch_solve_abs(v1, v2, weight_sum, pixel_count, n, det_floor, min_pixels, min_weight, status,
                   a, b, det, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_update_all(const double *gaussians, int64_t n, const ts_camera *cameras, int32_t n_views,
                  const ts_motions *motions, const ts_config *config, const ts_updates *updates,
                  void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!cameras || n_views < 1 || !motions || !config || !updates || n < 0)
    return TS_E_INVALID_ARGUMENT;
  void *dcams = nullptr, *ws = nullptr;
  TS_CUDA_TRY(cudaMallocAsync(&dcams, sizeof(ts_camera) * n_views, s));
  TS_CUDA_TRY(cudaMallocAsync(&ws, k4_workspace_bytes(n), s));
  TS_CUDA_TRY(cudaMemcpyAsync(dcams, cameras, sizeof(ts_camera) * n_views, cudaMemcpyHostToDevice, s));
  launch_k4_fuse(gaussians, n, reinterpret_cast<ts_camera *>(dcams), n_views, *motions, *config,
                 *updates, ws, s);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(dcams, s);
  cudaFreeAsync(ws, s);
  return e == cudaSuccess ? TS_OK : TS_E_CUDA;
}

int ts_triangulate_batch(const double *rows, const int32_t *n_rows, int64_t batch, int32_t max_rows,
                         double *x, int8_t *status, void *stream) {
  launch_triangulate_batch(rows, n_rows, batch, max_rows, x, status, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_solve_cov3d_batch(const double *lin, const double *rhs, const int32_t *n_rows,
                         int64_t batch, int32_t max_rows, double *x, int8_t *status,
                         void *stream) {
  launch_cov3d_batch(lin, rhs, n_rows, batch, max_rows, x, status, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_decompose_batch(const double *sigma, const double *ref_quat, int64_t batch,
                       double eig_floor, double *quat, double *scale, int8_t *status,
                       void *stream) {
  launch_decompose_batch(sigma, ref_quat, batch, eig_floor, quat, scale, status,
                         (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_dominant_gaussians(ts_plan *p, int32_t view, int64_t *gid_img, double *depth_img,
                          void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || view < 0 || view >= p->V) return TS_E_INVALID_ARGUMENT;
  // pixels no tile touches stay at -1 / 0
  TS_CUDA_TRY(cudaMemsetAsync(gid_img, 0xFF, 8 * (size_t)p->W * p->H, s));
  TS_CUDA_TRY(cudaMemsetAsync(depth_img, 0, 8 * (size_t)p->W * p->H, s));
  TS_CUDA_TRY(launch_k2(K2_DOMINANT, TS_TRACK_F32, ptr<RasterRec>(p->rec), ptr<uint32_t>(p->tval2),
                        ptr<uint32_t>(p->range), ptr<uint32_t>(p->inst_base),
                        ptr<uint32_t>(p->items), ptr<uint32_t>(p->counters), view * p->tpv,
                        (view + 1) * p->tpv, nullptr, nullptr, p->W, p->H, p->tiles_x, p->tpv,
                        p->cfg, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                        ptr<double>(p->depth64), gid_img, depth_img, nullptr, nullptr, s));
  return TS_OK;
}

// ---- regularisation -------------------------------------------------------------------------

int ts_build_knn(ts_plan *p, const double *positions, int64_t row_stride, int64_t n, int32_t k,
                 int64_t *adjacency, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || !positions || !adjacency || n < 2 || k < 1 || row_stride < 3 || n >= (1ll << 31))
    return TS_E_INVALID_ARGUMENT;
  const int kk = (int)std::min<int64_t>(k, n - 1);
  if (kk > TS_KNN_MAX_K) return TS_E_INVALID_ARGUMENT;
  const int64_t cap = 2 * n + 64;  // cell budget (the grid targets ~n/2 cells)
  const int nb = knn_bound_blocks(n);
  ENSURE(p->knn_part, 6 * sizeof(double) * nb);
  ENSURE(p->knn_grid, sizeof(KnnGrid));
  ENSURE(p->knn_key, 4 * n);
  ENSURE(p->knn_key2, 4 * n);
  ENSURE(p->knn_val, 4 * n);
  ENSURE(p->knn_val2, 4 * n);
  ENSURE(p->knn_sp, sizeof(double4) * n);
  ENSURE(p->knn_lo, 4 * cap);
  ENSURE(p->knn_hi, 4 * cap);
  TS_CUDA_TRY(cudaMemsetAsync(p->knn_lo.p, 0, 4 * cap, s));
  TS_CUDA_TRY(cudaMemsetAsync(p->knn_hi.p, 0, 4 * cap, s));
  KnnGrid *g = ptr<KnnGrid>(p->knn_grid);
  launch_knn_grid(positions, row_stride, n, cap, ptr<double>(p->knn_part), g,
                  ptr<uint32_t>(p->knn_key), ptr<uint32_t>(p->knn_val), s);
  const int bits = bits_for((uint64_t)cap);
  TS_CUDA_TRY(cub_call(p, s, [&](void *tmp, size_t &bytes) {
    return cub::DeviceRadixSort::SortPairs(tmp, bytes, ptr<uint32_t>(p->knn_key),
                                           ptr<uint32_t>(p->knn_key2), ptr<uint32_t>(p->knn_val),
                                           ptr<uint32_t>(p->knn_val2), (int)n, 0, bits, s);
  }));
  launch_knn_gather(positions, row_stride, ptr<uint32_t>(p->knn_key2), ptr<uint32_t>(p->knn_val2),
                    n, ptr<double4>(p->knn_sp), ptr<uint32_t>(p->knn_lo), ptr<uint32_t>(p->knn_hi),
                    s);
  TS_CUDA_TRY(launch_knn_query(kk, ptr<double4>(p->knn_sp), ptr<uint32_t>(p->knn_lo),
                               ptr<uint32_t>(p->knn_hi), g, n, adjacency, s));
  return TS_OK;
}

int ts_detect_static(const int32_t *pixel_count, const int32_t *static_pixel_count, int64_t n,
                     int32_t n_views, const ts_reg_config *c, uint8_t *static_flags,
                     void *stream) {
  if (!pixel_count || !static_pixel_count || !c || !static_flags || n < 0 || n_views < 0)
    return TS_E_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  launch_static_flags(pixel_count, static_pixel_count, n, n_views, c->min_hit_pixels,
                      c->static_fraction, c->min_views, static_flags, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

static bool updates_ok(const ts_updates *u) {
  return u && u->delta_mean && u->rotation && u->scale && u->status;
}

int ts_median_filter(const double *frame1, int64_t n, const ts_updates *in,
                     const int64_t *adjacency, int32_t kk, const ts_updates *out, void *stream) {
  if (!frame1 || !updates_ok(in) || !updates_ok(out) || n < 0 || kk < 0 || kk > TS_KNN_MAX_K ||
      (n > 0 && kk > 0 && !adjacency))
    return TS_E_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  launch_reg_filter(REG_MEDIAN_ONLY, frame1, n, *in, nullptr, nullptr, 0, adjacency, kk, 0, 0.0, 0,
                    *out, nullptr, nullptr, nullptr, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_propagate(ts_plan *p, const double *frame1, int64_t n, const ts_updates *in,
                 const int64_t *adjacency, int32_t kk, const uint8_t *static_flags,
                 int32_t average, const ts_updates *out, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || !frame1 || !updates_ok(in) || !updates_ok(out) || !static_flags || n < 0 || kk < 0 ||
      kk > TS_KNN_MAX_K || (average != TS_AVERAGE_MEAN && average != TS_AVERAGE_MEDIAN) ||
      (n > 0 && kk > 0 && !adjacency))
    return TS_E_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  ENSURE(p->reg_source, n);
  ENSURE(p->reg_euler, 24 * n);
  launch_reg_filter(REG_PREP_GIVEN_STATIC, frame1, n, *in, nullptr, nullptr, 0, adjacency, kk, 0,
                    0.0, 0, *out, const_cast<uint8_t *>(static_flags), ptr<uint8_t>(p->reg_source),
                    ptr<double>(p->reg_euler), s);
  launch_reg_propagate(true, false, frame1, n, *out, static_flags, ptr<uint8_t>(p->reg_source),
                       ptr<double>(p->reg_euler), adjacency, kk, average, nullptr, s);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_apply_updates(const double *frame1, int64_t n, const ts_updates *u, double *rows_out,
                     void *stream) {
  if (!frame1 || !updates_ok(u) || !rows_out || n < 0) return TS_E_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  launch_reg_propagate(false, true, frame1, n, *u, nullptr, nullptr, nullptr, nullptr, 0, 0,
                       rows_out, (cudaStream_t)stream);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

int ts_regularize(ts_plan *p, const double *frame1, int64_t n, const ts_updates *in,
                  const int32_t *pixel_count, const int32_t *static_pixel_count, int32_t n_views,
                  const int64_t *adjacency, int32_t kk, const ts_reg_config *c,
                  const ts_updates *out, uint8_t *static_flags, double *rows_out, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!p || !frame1 || !updates_ok(in) || !updates_ok(out) || !pixel_count ||
      !static_pixel_count || !c || n < 0 || n_views < 0 || kk < 0 || kk > TS_KNN_MAX_K ||
      (c->average != TS_AVERAGE_MEAN && c->average != TS_AVERAGE_MEDIAN) ||
      (n > 0 && kk > 0 && !adjacency))
    return TS_E_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  uint8_t *flags = static_flags;
  if (!flags) {
    ENSURE(p->reg_static, n);
    flags = ptr<uint8_t>(p->reg_static);
  }
  ENSURE(p->reg_source, n);
  ENSURE(p->reg_euler, 24 * n);
  launch_reg_filter(REG_FULL, frame1, n, *in, pixel_count, static_pixel_count, n_views, adjacency,
                    kk, c->min_hit_pixels, c->static_fraction, c->min_views, *out, flags,
                    ptr<uint8_t>(p->reg_source), ptr<double>(p->reg_euler), s);
  launch_reg_propagate(true, rows_out != nullptr, frame1, n, *out, flags,
                       ptr<uint8_t>(p->reg_source), ptr<double>(p->reg_euler), adjacency, kk,
                       c->average, rows_out, s);
  TS_CUDA_TRY(cudaGetLastError());
  return TS_OK;
}

}  // extern "C"


extern "C" int ts_memcpy_d2h(void *host_dst, const void *device_src, int64_t bytes) {
  if (bytes < 0) return TS_E_INVALID_ARGUMENT;
  if (bytes == 0) return TS_OK;
  TS_CUDA_TRY(cudaMemcpy(host_dst, device_src, (size_t)bytes, cudaMemcpyDeviceToHost));
  return TS_OK;
}
