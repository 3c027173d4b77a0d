// kernels.cuh -- internal launcher declarations shared by the .cu files of the library.
#pragma once

#include "common.cuh"

namespace ts {

enum { K2_ACCUMULATE = 0, K2_EMIT = 1, K2_DOMINANT = 2, K2_CACHE = 3 };

// Contribution cache record of one (gv, 8x8 quadrant) slot with kept contributions (K2_CACHE
// mode): the quadrant's kept-contribution pixels as a 64-bit mask, their w = alpha T in pixel
// order at pool[offset ..], the slot, the quadrant origin, the moment anchor and the view.  Frame
// independent: every target frame of a clip reuses it (the reference's weight-map reuse,
// pipeline.py:191-196); per frame k2_cached turns each record into the slot's Partial.
struct CacheRec {
  uint64_t mask;
  uint32_t offset, slot;
  int16_t qx0, qy0, ax, ay;
  int32_t view, pad;
};
static_assert(sizeof(CacheRec) == 32, "CacheRec is 32 bytes");
constexpr uint32_t K2_CACHE_RECS = 256;  // records a warp reserves at a time
constexpr uint32_t K2_CACHE_CHUNK = 8192;  // pool doubles a warp reserves at a time

constexpr int K1_RECT_OFFSET = 128;  // u32 offset of the per-view bbox unions in the drange buffer
void launch_k1_project(const double *G, int64_t n, const ts_camera *cams, int V, int dbits,
                       RasterRec *rec, uint32_t *drange, uint32_t *dkey, uint32_t *dval,
                       double *depth64, uint32_t *ntiles, int8_t *status, int16_t *bbox,
                       cudaStream_t s);
void launch_k1_fix_ties(const uint32_t *key, uint32_t *val, const double *depth64, int64_t M,
                        int dbits, uint32_t *long_runs, uint32_t long_cap, cudaStream_t s);
void launch_k1_long_run_keys(const uint32_t *val, const double *depth64, int64_t M,
                             const uint32_t *long_runs, uint32_t n_runs, uint64_t *bits,
                             uint32_t *begin, uint32_t *end, cudaStream_t s);
void launch_k1_emit(const uint32_t *val, const int16_t *bbox, const uint32_t *off_sorted,
                    int64_t M, int tiles_x, uint32_t *tkey, uint32_t *tval, cudaStream_t s);
void launch_k1_tile_ranges(const uint32_t *tkey, const uint32_t *tval, int64_t n_inst, int64_t n,
                           int V, int tiles_per_view, uint32_t *range, cudaStream_t s);
void launch_project_view(const double *G, int64_t n, const ts_camera &cam, double *mean2,
                         double *depth, double *cov2, uint8_t *in_front, cudaStream_t s);

cudaError_t launch_k2(int mode, int track_dtype, const RasterRec *rec, const uint32_t *inst_gv,
                      const uint32_t *tile_range, const uint32_t *inst_base, uint32_t *items,
                      uint32_t *counters, int tile_begin, int tile_end, const void *track_target,
                      const uint8_t *track_valid, int W, int H, int tiles_x, int tiles_per_view,
                      const ts_config &cfg, Partial *partial, uint8_t *flag,
                      unsigned long long *emit_count, int64_t emit_cap, uint64_t *emit_key,
                      uint32_t *emit_gv, double *emit_alpha, double *emit_trans,
                      const double *depth64, int64_t *dom_gid, double *dom_depth,
                      unsigned long long *stats, void *schedule_ws, cudaStream_t s, int ctas_per_sm = 0,
                      uint8_t *touched = nullptr, double *pool = nullptr,
                      unsigned long long *pool_cursor = nullptr, uint64_t pool_cap = 0,
                      CacheRec *recs = nullptr, unsigned long long *rec_cursor = nullptr,
                      uint64_t rec_cap = 0);
// per target frame: every cache record -> its slot's Partial with this frame's tracks
// Clip cache (cache.cu): records -> contributions in slot order (cw, cxy) and per-gv ranges over
// the touched list, once per clip; per target frame the moments + fits of the listed gvs.
void launch_cache_slot_counts(const CacheRec *recs, const unsigned long long *n_recs,
                              uint64_t rec_cap, uint32_t *slot_cnt, cudaStream_t s,
                              uint64_t n_hint);
void launch_cache_scatter(const CacheRec *recs, const unsigned long long *n_recs, uint64_t rec_cap,
                          const double *pool, const uint32_t *slot_off, double *cw, uint32_t *cxy,
                          cudaStream_t s, uint64_t n_hint);
void launch_cache_ranges(const uint32_t *list, const uint32_t *n_list, int64_t nv_total,
                         const int16_t *bbox, const uint32_t *inst_base, const uint32_t *slot_off,
                         uint2 *ranges, cudaStream_t s);
size_t cache_chunk_bytes();
size_t cache_multi_bytes();
size_t cache_scratch_bytes();
int cache_chunk_len();
void launch_cache_chunk_counts(const uint32_t *n_list, int64_t nv_total, const uint2 *ranges,
                               uint32_t *nch, cudaStream_t s);
void launch_cache_chunk_fill(const uint32_t *list, const uint32_t *n_list, int64_t nv_total,
                             const int16_t *bbox, int64_t n, const uint2 *ranges,
                             const uint32_t *nch, const uint32_t *choff, void *chunks, void *multi,
                             uint32_t *counters, cudaStream_t s);
cudaError_t launch_k23_cached(const void *chunks, const uint32_t *counters, uint64_t chunk_bound,
                              const void *multi, uint64_t multi_bound, const uint32_t *list,
                              const int16_t *bbox, int64_t n, int W, int H, const double *cw,
                              const uint32_t *cxy, const void *track_target, int track_dtype,
                              const uint8_t *track_valid, const ts_config &cfg, void *fits,
                              double *scratch, cudaStream_t s, int8_t *status_out = nullptr);
void launch_k3_merge(const uint8_t *touched, const uint32_t *rank, const void *fits,
                     int64_t nv_total, ts_motions m, cudaStream_t s);
size_t k2_schedule_bytes(int n_tiles);  // workspace of the longest-first K2 schedule
bool k2_writes_touched();  // the accumulate kernel in use marks per-gv touched bytes

// K3: per-(view, Gaussian) affine fit from the tile partials of K2.
void launch_k3_solve(const Partial *partial, const uint8_t *flag, const uint32_t *inst_base,
                     const uint32_t *ntiles, const int16_t *bbox, int64_t nv_total,
                     const ts_config &cfg, ts_motions m, const uint8_t *touched,
                     const uint32_t *list, const uint32_t *n_list, const uint32_t *rank,
                     void *fits, cudaStream_t s, bool status_only = false);
size_t k3_fit_bytes();  // per touched gv, the compact fit record of K3

// solve_view on absolute moments (stage API)
void launch_solve_abs(const double *v1, const double *v2, const double *wsum, const int64_t *cnt,
                      int64_t n, double det_floor, int min_pixels, double min_weight,
                      int8_t *status, double *a, double *b, double *det, cudaStream_t s);
// accumulate_view over explicit contributions, stably sorted by gid: one thread per Gaussian
void launch_segment_bounds(const uint32_t *sorted_gid, int64_t m, uint32_t *seg_start,
                           uint32_t *seg_end, cudaStream_t s);
void launch_accumulate(int64_t n, const uint32_t *seg_start, const uint32_t *seg_end,
                       const uint32_t *order, const int32_t *px, const int32_t *py,
                       const double *alpha, const double *trans, int W, const void *target,
                       int track_dtype, const uint8_t *valid, double thr, double *v1, double *v2,
                       double *wsum, int64_t *cnt, int64_t *scnt, double *swsum, cudaStream_t s);

// K4: multi-view fuse (update_all)
size_t k4_workspace_bytes(int64_t n);
// fits / rank != NULL: the per-view a, b and sums come from K3's compact fits (m.status dense)
void launch_k4_fuse(const double *G, int64_t n, const ts_camera *cams, int V, ts_motions m,
                    const ts_config &cfg, ts_updates u, void *workspace, cudaStream_t s,
                    const void *fits = nullptr, const uint32_t *rank = nullptr);
void launch_triangulate_batch(const double *rows, const int32_t *n_rows, int64_t batch,
                              int max_rows, double *x, int8_t *status, cudaStream_t s);
void launch_cov3d_batch(const double *lin, const double *rhs, const int32_t *n_rows,
                        int64_t batch, int max_rows, double *x, int8_t *status, cudaStream_t s);
void launch_decompose_batch(const double *sigma, const double *ref_quat, int64_t batch,
                            double eig_floor, double *quat, double *scale, int8_t *status,
                            cudaStream_t s);

// Regularisation (regularize.cu)
#define TS_KNN_MAX_K 32
struct KnnGrid {
  double lo[3];
  double h, inv_h, slack;
  int dim[3];
  int ncell;
};
enum { REG_MEDIAN_ONLY = 0, REG_PREP_GIVEN_STATIC = 1, REG_FULL = 2 };
int knn_bound_blocks(int64_t n);
void launch_knn_grid(const double *pos, int64_t stride, int64_t n, int64_t cap, double *part,
                     KnnGrid *g, uint32_t *key, uint32_t *val, cudaStream_t s);
void launch_knn_gather(const double *pos, int64_t stride, const uint32_t *key, const uint32_t *val,
                       int64_t n, double4 *sp, uint32_t *cell_lo, uint32_t *cell_hi,
                       cudaStream_t s);
cudaError_t launch_knn_query(int k, const double4 *sp, const uint32_t *lo, const uint32_t *hi,
                             const KnnGrid *g, int64_t n, int64_t *adj, cudaStream_t s);
void launch_static_flags(const int32_t *pix, const int32_t *spix, int64_t n, int V, int min_hit,
                         double frac, int min_views, uint8_t *flag, cudaStream_t s);
void launch_reg_filter(int mode, const double *G, int64_t n, ts_updates in, const int32_t *pix,
                       const int32_t *spix, int V, const int64_t *adj, int kk, int min_hit,
                       double frac, int min_views, ts_updates out, uint8_t *static_flag,
                       uint8_t *source_flag, double *rel_euler, cudaStream_t s);
void launch_reg_propagate(bool propagate, bool apply, const double *G, int64_t n, ts_updates u,
                          const uint8_t *static_flag, const uint8_t *source_flag,
                          const double *rel_euler, const int64_t *adj, int kk, int average,
                          double *rows_out, cudaStream_t s);

}  // namespace ts
