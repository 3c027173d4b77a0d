/*
 * trackersplat_b200.h -- C ABI of the B200 motion-estimation hot path.
 *
 * The reference (gausstrack, /root/reference/pkg/src/gausstrack) is a pure-Python package, so its
 * "plugin boundary" is the set of module functions re-exported from gausstrack/__init__.py:9-22.
 * Each entry point below replaces one of them; the Python package paper_2604_02586_b200 binds them
 * with ctypes and keeps the reference names, signatures and error behaviour.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller unless stated otherwise; every
 *    call is stream-ordered on `stream` (a cudaStream_t passed as void*).  Calls that must return a
 *    data-dependent size (ts_rasterize_weights, the binning inside ts_frame_bin) synchronise the
 *    stream once to read it.
 *  - Gaussians: row-major (N, 11) float64 = mean[3], unit quaternion (w,x,y,z)[4], scale[3],
 *    opacity  (core.py:86-109; quaternions are normalised by the host-side Gaussian3D).
 *  - Cameras: ts_camera is passed by HOST pointer (core.py:112-148).
 *  - Per-(view, Gaussian) arrays are indexed gv = v * N + g.
 *  - Return value: TS_OK (0) or a negative TS_E_* code; the Python layer maps them to the
 *    reference exceptions (errors.py:4-41).  Per-element degeneracy is a status, never an error
 *    (motion2d.py:26-29): status bytes use TS_STATUS_*.
 */
#ifndef TRACKERSPLAT_B200_H
#define TRACKERSPLAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_OK 0
#define TS_E_INVALID_ARGUMENT -1   /* ValueError (splat.py:123-124, motion2d.py:45-51) */
#define TS_E_DIMENSION_MISMATCH -2 /* DimensionMismatch (motion2d.py:133-136)          */
#define TS_E_CUDA -3               /* CUDA runtime failure                              */
#define TS_E_OUT_OF_MEMORY -4
#define TS_E_CAPACITY -5           /* caller buffer too small; required size returned   */

#define TS_STATUS_UNSOLVABLE 0
#define TS_STATUS_SOLVED 1
#define TS_STATUS_STATIC 2

#define TS_TRACK_F32 0 /* TRKF layout: (H, W, 2) float32 targets (fileio.py:108-136) */
#define TS_TRACK_F64 1 /* TrackField layout: (H, W, 2) float64 targets (motion2d.py:39) */

typedef struct ts_camera { /* CameraView, core.py:112-148 */
  double R[9];             /* world -> camera rotation, row-major */
  double t[3];
  double fx, fy, cx, cy;
  int32_t width, height;
} ts_camera;

typedef struct ts_config { /* Config, config.py:14-40 (+ the raster early stop, splat.py:19) */
  double alpha_cutoff;        /* 1/255 */
  double early_stop;          /* 1e-4  */
  double det_floor;           /* 1e-12 */
  double min_weight;          /* 1e-3  */
  double min_total_weight;    /* 1e-3  */
  double static_threshold_px; /* 1.0   */
  double eig_floor;           /* 1e-12 */
  int32_t min_pixels;         /* 3 */
  int32_t min_views;          /* 2 */
  int32_t min_total_pixels;   /* 3 */
  int32_t reserved;
} ts_config;

/* Per-(view, Gaussian) motion arrays (SoA, length V*N): ViewMotion (motion2d.py:73-80). */
typedef struct ts_motions {
  int8_t *status;       /* TS_STATUS_*                                  */
  double *a;            /* (V*N, 2, 2) row-major A                       */
  double *b;            /* (V*N, 2)                                      */
  double *weight_sum;   /* (V*N)                                         */
  int32_t *pixel_count; /* (V*N)                                         */
  int32_t *static_pixel_count; /* (V*N), may be NULL                     */
  double *static_weight_sum;   /* (V*N), may be NULL                     */
} ts_motions;

/* Per-Gaussian update arrays (SoA, length N): MotionUpdate (multiview.py:44-50). */
typedef struct ts_updates {
  double *delta_mean; /* (N, 3) */
  double *rotation;   /* (N, 4) */
  double *scale;      /* (N, 3) */
  int8_t *status;     /* (N)    */
} ts_updates;

typedef struct ts_plan ts_plan; /* opaque: owns a growable device workspace */

int ts_version(void);
const char *ts_error_string(int code);
int ts_plan_create(ts_plan **plan);
int ts_plan_destroy(ts_plan *plan);
/* bytes of device workspace currently held by the plan */
int64_t ts_plan_workspace_bytes(const ts_plan *plan);
/* Stage timing with CUDA events recorded on the launch stream (bench/roofline support).
 * Stages: 0 K1 project, 1 depth sort + counts, 2 emit + tile sort + ranges, 3 K2 raster-
 * accumulate, 4 K3 solve, 5 K4 fuse.  enable != 0 resets and starts recording. */
#define TS_N_STAGES 6
int ts_plan_timing(ts_plan *plan, int enable);
int ts_plan_timing_read(ts_plan *plan, double *totals_ms, int32_t *counts, int32_t n_stages);
/* Residency of the persistent K2 grid: at most ctas_per_sm CTAs per SM (0 = as many as fit, the
 * default).  A plan whose frames run two or three in flight on separate streams does better with
 * fewer (3 at cfg2: the other frame's binning, solve and fuse kernels share the SMs K2 leaves
 * free); a frame run alone is fastest with the full grid.  No reference counterpart: a
 * scheduling knob of this build (the reference's raster loop, splat.py:147-195, is serial). */
int ts_plan_set_k2_ctas_per_sm(ts_plan *plan, int32_t ctas_per_sm);

/* _project_all, splat.py:80-110.  mean2 (N,2), depth (N), cov2 (N,3: xx,xy,yy), in_front (N). */
int ts_project(const double *gaussians, int64_t n, const ts_camera *camera, double *mean2,
               double *depth, double *cov2, uint8_t *in_front, void *stream);

/* ---- frame engine: the fused hot path (the four stages of compensate_frame, pipeline.py:117-124
 *      and :79-86; the regularisation tail is ts_regularize below).  Binning is per clip (it depends only on frame-1 Gaussians and cameras,
 *      as the weight maps in pipeline.py:191-196); accumulate/solve/fuse runs per target frame. */

/* K1 projection + depth order + tile binning of N Gaussians into V <= 64 views that share one
 * width/height (TS_E_DIMENSION_MISMATCH otherwise).  Synchronises once (instance count).  Keeps
 * the result in the plan.  Rigs with mixed image sizes or more views (the reference rasterizes
 * each view at its own size, pipeline.py:117-120) are binned as same-size groups of <= 64 views,
 * one plan each: ts_frame_compensate with updates == NULL per plan, then ts_update_all over all
 * views (engine.FrameEngine does this). */
int ts_frame_bin(ts_plan *plan, const double *gaussians, int64_t n, const ts_camera *cameras,
                 int32_t n_views, const ts_config *config, void *stream);

/* K2 fused raster-accumulate -> K3 per-view affine solve -> K4 multi-view fuse for one target
 * frame.  track_target: (V, H, W, 2) of TS_TRACK_F32/F64; track_valid: (V, H, W) uint8.
 * Each track array is device memory or page-locked (pinned) host memory: K2 reads the pinned
 * host arrays in place over PCIe (zero-copy), only the 8x8 quadrants of occupied tiles -- about
 * a tenth of the pixels at the benchmark configs; the host must not modify them until the
 * frame's work on `stream` completes.  Pageable host memory: TS_E_INVALID_ARGUMENT.
 * motions may have NULL members (then only the internal copy is kept); motions == NULL (the
 * per-view motions are intermediates: the reference's FrameResult carries only the updates)
 * lets K4 read K3's compact fits in place when K3 ran over its touched-gv list or the clip
 * cache.  updates == NULL stops after K3 (the per-view motions of a view group; motions must
 * then be non-NULL). */
int ts_frame_compensate(ts_plan *plan, const void *track_target, int32_t track_dtype,
                        const uint8_t *track_valid, const ts_motions *motions,
                        const ts_updates *updates, void *stream);

/* Binning results of the last ts_frame_bin (device pointers into the plan; valid until the next
 * ts_frame_bin / ts_plan_destroy).  Tile t of view v has global id v*tiles_per_view + t,
 * t = ty*tiles_x + tx, tiles of 16x16 pixels. */
typedef struct ts_binning {
  int64_t n_instances;
  int32_t tiles_x, tiles_y, n_views;
  const uint32_t *inst_tile; /* (n_instances) tile id within the view; instances are
                                grouped by tile position, views in order            */
  const uint32_t *inst_gv;   /* (n_instances) gv = v*N + g; each (view, tile) list in
                                the reference's (depth, g) order                    */
  const uint32_t *tile_range;/* (V*tiles, 2) [start, end) of global tile v*tiles + t */
  const int8_t *gv_status;   /* (V*N) 0 behind, 1 degenerate, 2 empty bbox, 3 binned */
  const int16_t *gv_bbox;    /* (V*N, 4) x0 x1 y0 y1                                 */
} ts_binning;
int ts_frame_binning(const ts_plan *plan, ts_binning *out);
/* Number of (view, tile) lists of the last ts_frame_bin that are non-empty (synchronous): K2
 * reads the 4 x 64 track pixels of each. */
int ts_frame_occupied_tiles(const ts_plan *plan, int64_t *out);

/* Clip contribution cache (enable = 1): runs K2 once over the current binning WITHOUT tracks and
 * keeps every kept contribution (pixel, w = alpha T) as one record per (Gaussian-view, 8x8
 * quadrant) in the plan; until the next ts_frame_bin (or enable = 0), ts_frame_compensate then
 * skips the rasterization and forms each Gaussian-view's moments and fit from its cached
 * contributions with the target frame's tracks
 * -- the GPU form of the reference's frame-0 weight-map reuse across a clip's target frames
 * (pipeline.py:191-196; compensate_frame(weightmaps=...), pipeline.py:110-116).
 * Synchronous (sizes the pool); TS_E_CAPACITY if the pool cannot be sized. */
int ts_frame_cache(ts_plan *plan, int32_t enable, void *stream);
/* Size of the current cache: records (32 B each) and cached w values (8 B each); 0 when none. */
int ts_frame_cache_info(const ts_plan *plan, uint64_t *n_records, uint64_t *n_values);

/* Per view, the pixel rectangle the next ts_frame_compensate reads from the track arrays (the
 * 16x16 tiles touched by any binned bbox; inclusive x0 y0 x1 y1, x1 < x0 when the view has no
 * binned Gaussian), into rects[4 * n_views].  Host-side, valid once ts_frame_bin has returned: a
 * caller holding tracks in host memory can DMA just these rows (cudaMemcpy2DAsync) into a device
 * array of the full (V, H, W) layout.  No reference counterpart (a transfer plan). */
int ts_frame_track_rects(const ts_plan *plan, int32_t *rects);

/* Asynchronous DMA of exactly those rectangles, per view, from host track arrays (pinned for the
 * copy to overlap) into device arrays of the same (V, H, W[, 2]) layout, on `stream`: the copy
 * engine moves the ~third of the pixels the frame needs (cfg2) while the SMs compute. */
int ts_copy_track_rects(const ts_plan *plan, const void *host_target, int32_t track_dtype,
                        const uint8_t *host_valid, void *dev_target, uint8_t *dev_valid,
                        void *stream);

/* ---- stage entry points (reference-typed API) ---- */

/* rasterize_weights, splat.py:113-195, for one view.  Runs K1 + K2 in contribution-emitting
 * mode and sorts the WeightMap into the reference order (pixel, depth, gid).  *n_out receives
 * the number of contributions; the arrays are then fetched with ts_rasterize_fetch. */
int ts_rasterize_weights(ts_plan *plan, const double *gaussians, int64_t n,
                         const ts_camera *camera, double alpha_cutoff, double early_stop,
                         int64_t *n_out, int64_t *n_degenerate_out, void *stream);
int ts_rasterize_fetch(ts_plan *plan, int32_t *pixel_x, int32_t *pixel_y, int64_t *gaussian_id,
                       double *alpha, double *transmittance, double *depth,
                       int64_t *degenerate_ids, void *stream);

/* accumulate_view, motion2d.py:126-161, over explicit contributions (any order).  Deterministic:
 * each Gaussian's moments are summed in contribution-array order, as np.add.at does.
 * Outputs v1 (N,3,3), v2 (N,3,2), weight_sum, pixel_count, static_pixel_count (int64),
 * static_weight_sum.  target is (H,W,2) of track_dtype. */
int ts_accumulate_view(ts_plan *plan, const int32_t *pixel_x, const int32_t *pixel_y,
                       const int64_t *gaussian_id, const double *alpha,
                       const double *transmittance, int64_t m, int32_t width, int32_t height,
                       const void *track_target, int32_t track_dtype, const uint8_t *track_valid,
                       int64_t n, double static_threshold_px, double *v1, double *v2,
                       double *weight_sum, int64_t *pixel_count, int64_t *static_pixel_count,
                       double *static_weight_sum, void *stream);

/* solve_view, motion2d.py:164-184 (K3 on absolute moments): status, A, b per Gaussian. */
int ts_solve_view(const double *v1, const double *v2, const double *weight_sum,
                  const int64_t *pixel_count, int64_t n, double det_floor, int32_t min_pixels,
                  double min_weight, int8_t *status, double *a, double *b, double *det,
                  void *stream);

/* update_all, multiview.py:168-275 (K4).  motions arrays are (V*N) SoA as in ts_motions. */
int ts_update_all(const double *gaussians, int64_t n, const ts_camera *cameras, int32_t n_views,
                  const ts_motions *motions, const ts_config *config, const ts_updates *updates,
                  void *stream);

/* Scalar KAT entry points, batched (one problem per element):
 * triangulate_mean (multiview.py:53-70): rows (B, 2*maxv, 4) DLT rows with per-problem row
 *   counts; out x (B,3), status (B) (1 ok, 0 DegenerateGeometry/InsufficientViews).
 * solve_covariance3d (multiview.py:73-100): lin (B, 3*maxv, 6), rhs (B, 3*maxv); out (B,6).
 * decompose_covariance (multiview.py:103-135): sigma (B,3,3), ref quat (B,4) -> quat, scale. */
int ts_triangulate_batch(const double *rows, const int32_t *n_rows, int64_t batch, int32_t max_rows,
                         double *x, int8_t *status, void *stream);
int ts_solve_cov3d_batch(const double *lin, const double *rhs, const int32_t *n_rows,
                         int64_t batch, int32_t max_rows, double *x, int8_t *status,
                         void *stream);
int ts_decompose_batch(const double *sigma, const double *ref_quat, int64_t batch,
                       double eig_floor, double *quat, double *scale, int8_t *status,
                       void *stream);

/* Oracle tracker kernels for synthetic inputs (scene.py:166-240): per pixel dominant Gaussian
 * (argmax alpha*T, ties by smaller id) of view `view` from the last ts_frame_bin. */
int ts_dominant_gaussians(ts_plan *plan, int32_t view, int64_t *gid_img, double *depth_img,
                          void *stream);

/* ---- Regularisation (regularize.py:37-188; glue pipeline.py:88-98) ------------------------- *
 * Frame-1 Gaussians are (N, 11) rows as in ts_frame_bin; update arrays as ts_updates; per-view
 * counts in the (V*N) view-major layout of ts_motions.  Adjacency is (N, kk) int64, kk =
 * min(k, N-1) <= TS_KNN_MAX_K, rows sorted by (distance, id) ascending. */
#define TS_KNN_MAX_K 32
#define TS_AVERAGE_MEAN 0
#define TS_AVERAGE_MEDIAN 1

typedef struct ts_reg_config { /* Config fields used by _fuse_frame (pipeline.py:88-96) */
  int32_t min_hit_pixels;  /* 9   */
  int32_t min_views;       /* 2   */
  double static_fraction;  /* 0.9 */
  int32_t average;         /* TS_AVERAGE_MEAN / TS_AVERAGE_MEDIAN (propagation_average) */
  int32_t reserved;
} ts_reg_config;

/* build_knn (regularize.py:37-53): exact k nearest neighbours of each point by Euclidean
 * distance, ties by smaller id.  positions: n points of 3 doubles, `row_stride` doubles apart
 * (3 for an (N,3) array, 11 to read the means of Gaussian rows).  Uses the plan's workspace.
 * TS_E_INVALID_ARGUMENT for n < 2, k < 1 or min(k, n-1) > TS_KNN_MAX_K. */
int ts_build_knn(ts_plan *plan, const double *positions, int64_t row_stride, int64_t n, int32_t k,
                 int64_t *adjacency, void *stream);

/* detect_static_all (regularize.py:77-88) on view-major (V*N) counts -> flags (N) uint8. */
int ts_detect_static(const int32_t *pixel_count, const int32_t *static_pixel_count, int64_t n,
                     int32_t n_views, const ts_reg_config *config, uint8_t *static_flags,
                     void *stream);

/* median_filter (regularize.py:91-121): `out` must not alias `in`. */
int ts_median_filter(const double *frame1, int64_t n, const ts_updates *in,
                     const int64_t *adjacency, int32_t kk, const ts_updates *out, void *stream);

/* propagate (regularize.py:124-174) with given static flags; `out` must not alias `in`. */
int ts_propagate(ts_plan *plan, const double *frame1, int64_t n, const ts_updates *in,
                 const int64_t *adjacency, int32_t kk, const uint8_t *static_flags,
                 int32_t average, const ts_updates *out, void *stream);

/* apply_updates (regularize.py:177-188) -> (N, 11) rows. */
int ts_apply_updates(const double *frame1, int64_t n, const ts_updates *updates, double *rows_out,
                     void *stream);

/* The regularisation tail of _fuse_frame (pipeline.py:88-98) in two kernels: static flags from
 * the K2 counts, median filter, propagation and apply_updates.  `in` is the ts_update_all /
 * ts_frame_compensate output; `out` (must not alias `in`) receives the final updates,
 * `static_flags` (nullable) the flags and `rows_out` (nullable) the updated Gaussians. */
int ts_regularize(ts_plan *plan, const double *frame1, int64_t n, const ts_updates *in,
                  const int32_t *pixel_count, const int32_t *static_pixel_count, int32_t n_views,
                  const int64_t *adjacency, int32_t kk, const ts_reg_config *config,
                  const ts_updates *out, uint8_t *static_flags, double *rows_out, void *stream);

/* Synchronous device -> host copy (lets ctypes/cgo/JNI bindings read plan-owned arrays). */
int ts_memcpy_d2h(void *host_dst, const void *device_src, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif
