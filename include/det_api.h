/*
 * det_api.h -- C-ABI of the B200-native DET (density-equalizing transformation)
 * engine.  Plain pointers and sizes only; no torch types.  Host buffers are
 * caller-owned; device buffers are owned by the context.  One context per host
 * thread (a context owns one CUDA stream).
 *
 * The reference (cartomorph, pure Python) has no FFI; these entry points are
 * the operations its Python API performs on the hot path, and each cites the
 * reference code it replaces (paths under /root/reference/pkg/src/cartomorph).
 * The Python drop-in (paper_2604_13880_b200) binds them with ctypes; see
 * INTEGRATION.md for the binding a cartomorph maintainer would add.
 *
 * All functions return a status code (DET_OK on success).  On failure
 * det_last_error(ctx) holds a message.  Status codes mirror cartomorph.errors.
 */
#ifndef DET_API_H
#define DET_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct det_ctx det_ctx;

/* status codes (errors.py:4-26) */
#define DET_OK 0
#define DET_E_ARG 1      /* ValueError from an argument check                      */
#define DET_E_CUDA 2     /* CUDA runtime / launch failure                           */
#define DET_E_RASTER 3   /* RasterizationError (raster.py:148-154)                  */
#define DET_E_COLLAPSE 4 /* RegionCollapsedError (engine.py:148-150)                */
#define DET_E_NUMERIC 5  /* NumericError (engine.py:125-126, displacement.py:110)   */
#define DET_E_VALUE 6    /* ValueError raised inside the path (raster.py:168-169,
                            bincount negative index raster.py:87-89)                */
#define DET_E_STATE 7    /* call order / capacity problem                            */

/* stop reasons (engine.py:196-211) */
#define DET_STOP_RUNNING 0
#define DET_STOP_CONVERGED 1
#define DET_STOP_STAGNATION 2
#define DET_STOP_MAXITER 3
#define DET_STOP_COLLAPSED 4 /* RegionCollapsedError at evaluate()            */
#define DET_STOP_BDV 5       /* build_density: bdv <= 0 -> ValueError          */
#define DET_STOP_NEGINDEX 6  /* _submask bincount negative index -> ValueError */

/* bdv policy (engine.py:91-96) */
#define DET_BDV_FIXED_MASS 0
#define DET_BDV_REDERIVE 1

typedef struct {
    double background_mass;   /* M_b (engine.py:131-136)                    */
    double bdv_multiplier;    /* shape-preservation knob (engine.py:103)    */
    double mean_density0;     /* S / N_map0 (engine.py:130)                 */
    double total_statistic;   /* S (engine.py:123)                          */
    int32_t bdv_mode;         /* DET_BDV_*                                  */
    int32_t pad;
} det_params;

typedef struct {
    double error_threshold;   /* StoppingCriteria (engine.py:27-35) */
    int32_t stagnation_window;
    int32_t max_iterations;
} det_criteria;

typedef struct {
    int32_t stop_reason;      /* DET_STOP_*                                            */
    int32_t iteration;        /* CartogramState.iteration of the returned state        */
    int32_t best_iteration;
    int32_t collapsed_region; /* region index for DET_STOP_COLLAPSED, else -1          */
    int64_t clamp_events;     /* CartogramState.clamp_events (0 after stagnation)      */
    double epsilon, xi;       /* errors of the returned state                          */
    double bdv;               /* background density of the last step                   */
    int32_t trace_len;        /* number of IterationRecord rows                        */
    int32_t status;           /* DET_OK or the DET_E_* the reference would raise        */
} det_result;

int det_abi_version(void);
/* Page-locked host buffers for result copies (DMA instead of a staged pageable copy); the
 * drop-in's Python layer keeps a pool of them.  No reference counterpart (host plumbing). */
int det_host_alloc(size_t bytes, void **out);
int det_host_free(void *p);
const char *det_last_error(const det_ctx *ctx);
/* Debug mode (environment DET_GUARD=1 at library load; no reference counterpart): device buffers
 * carry 4 KB guard zones and are poisoned when allocated.  Reports the live guarded buffers and
 * how many guard zones (live or already released) were overwritten; DET_E_STATE when the mode is off. */
int det_debug_guard_check(long long *n_live, long long *n_bad);
/* device info string (name, SMs, L2) for reports */
int det_device_info(int device, char *buf, int buflen);

/* Arithmetic precision of the iteration (CartogramEngine's field_dtype):
 *   DET_PREC_FLOAT64  float64 field, vertex state and sums: the reference's arithmetic
 *                     (engine.py:170-180), trajectory-identical to it;
 *   DET_PREC_MIXED    float32 displacement field and in-band sums, float64 vertex state,
 *                     position update and raster crossings;
 *   DET_PREC_FLOAT32  float32 field and vertex state (float64 crossings and carries). */
enum { DET_PREC_FLOAT32 = 0, DET_PREC_FLOAT64 = 1, DET_PREC_MIXED = 2 };
/* k in [4, 13] (raster.py:138-139); precision is one of DET_PREC_*.  Replaces the per-engine
 * set-up of CartogramEngine.__init__ (engine.py:98-141): one context per thread/stream. */
int det_ctx_create(int device, int k, int precision, det_ctx **out);
void det_ctx_destroy(det_ctx *ctx);
/* number of frame groups run as parallel CUDA-graph branches (default 8, clamped to the batch) */
int det_set_groups(det_ctx *ctx, int groups);
/* band height of the integral-image kernels (power of two <= n; 0 restores the automatic choice) */
int det_set_band_height(det_ctx *ctx, int h);

/* Topology + initial vertices of one map: MapModel.vertex_array() rows
 * (geomodel.py:128-130), ring row offsets, ring->region, region rank in
 * ascending region_id order (raster.py:142).  Replaces the per-iteration
 * vertex_array()/with_vertex_array() round trip (engine.py:176-178). */
int det_load_map(det_ctx *ctx, const double *xy, int n_rows, const int32_t *ring_start, int n_rings,
                 const int32_t *ring_region, const int32_t *region_rank, int n_regions);

/* A batch of cartograms sharing the topology: per-cartogram start vertices
 * (batch*n_rows*2, or NULL = the loaded vertices for all) and statistics
 * (batch*n_regions; Region.statistic, geomodel.py:61). */
int det_set_batch(det_ctx *ctx, int batch, const double *xy, const double *stats);

/* rasterize_labels + pixel_counts/background_count (raster.py:110-155) of the
 * batch's current start vertices for cartogram b.  labels_out: n*n int32 [j,i]
 * (BACKGROUND=-1) or NULL; counts_out: n_regions+1 (last = background) or NULL. */
int det_rasterize(det_ctx *ctx, int b, int32_t *labels_out, int64_t *counts_out);

/* Per-cartogram engine constants (CartogramEngine.__init__, engine.py:98-141). */
int det_set_params(det_ctx *ctx, const det_params *params, const double *weights_px);

/* CartogramEngine.run (engine.py:182-219) for every cartogram of the batch,
 * device-resident (no host round trip per iteration). */
int det_run(det_ctx *ctx, const det_criteria *crit);
/* Exactly `iters` DET iterations on every cartogram with no stopping test
 * (benchmark helper; state continues from the last det_run/det_bench call). */
int det_bench_iterations(det_ctx *ctx, int iters);
int det_sync(det_ctx *ctx);
/* Per-cartogram iteration counter (index of the next state to evaluate) and active flag. */
int det_progress(det_ctx *ctx, int32_t *next_iter_out, int32_t *active_out);
/* Device time of `iters` bench iterations (CUDA events on the context stream, synchronised both sides). */
int det_time_iterations(det_ctx *ctx, int iters, float *ms_out);
/* Per-phase device time (CUDA events on the context stream) summed over `iters`
 * eagerly launched iterations: ms_out[0]=integral images (k_sat1..3),
 * [1]=advect+crossings (k_region), [2]=paint/labels/counts (k_row), [3]=control (k_ctrl). */
int det_bench_kernel_times(det_ctx *ctx, int iters, float *ms_out);

/* Cumulative chain of T time steps (temporal.py:162-246, cumulative=True), device resident:
 * frame t starts from frame t-1's result.  stats: T*R; S: T statistic totals; masses: T
 * background masses; out: xy_out T*n_rows*2, res_out T, counts_out T*(R+1) (a failed frame's
 * start-raster counts), trace_out T*(max_iterations+1)*4.  Requires det_set_batch(ctx, 1, ...). */
int det_run_chain(det_ctx *ctx, int T, const double *stats, const double *S, const double *masses,
                  const det_criteria *crit, double *xy_out, det_result *res_out, int64_t *counts_out,
                  double *trace_out);
int det_get_result(det_ctx *ctx, int b, det_result *out);
int det_get_vertices(det_ctx *ctx, int b, double *xy_out);       /* n_rows*2 */
int det_get_labels(det_ctx *ctx, int b, int32_t *labels_out);    /* n*n      */
int det_get_counts(det_ctx *ctx, int b, int64_t *counts_out);    /* R+1      */
int det_get_region_error(det_ctx *ctx, int b, double *out);      /* R        */
int det_get_trace(det_ctx *ctx, int b, double *out);             /* trace_len*4: iter, eps, xi, millis */
int det_get_areas(det_ctx *ctx, int b, double *out);             /* R: Region.area() (geomodel.py:63-65) */
/* Every cartogram's results in one call (the batched RunResult.state of engine.py:46-72): any output
 * may be NULL; xy_out B*n_rows*2, counts_out B*(R+1), err_out B*R, trace_out B*trace_rows*4 (rows
 * past a cartogram's trace_len are unspecified). */
int det_get_results(det_ctx *ctx, double *xy_out, int64_t *counts_out, double *err_out, double *trace_out,
                    int trace_rows);

/* Stage-level entry points (parity tests; integral.py:155, displacement.py:198-238). */
/* u = t(d) - t(const) at pixel centres for a dense density d (n*n float64);
 * optional 8 channels (alpha,beta,gamma,delta,alpha_t,beta_t,gamma_t,delta_t) */
int det_field(det_ctx *ctx, const double *d, double *u_out, double *channels_out, double *total_out);
/* t(d) itself at pixel centres (mapping_grid, displacement.py:102-131), n*n*2 */
int det_mapping(det_ctx *ctx, const double *d, double *t_out);
/* mapping_grid (displacement.py:102-131) of a given channel set (8*n*n float64: alpha, beta,
 * gamma, delta, alpha_t, beta_t, gamma_t, delta_t; total = C), minus `base` (n*n*2) when base is
 * non-NULL (residual_field, displacement.py:198-206).  Reference float64 op order. */
int det_mapping_channels(det_ctx *ctx, const double *channels, double total, const double *base, double *t_out);
/* mapping_point (displacement.py:150-170) at n_pts points (x, y) of the same channel set */
int det_mapping_points(det_ctx *ctx, const double *channels, double total, const double *xy, int n_pts,
                       double *out);
/* build_density (raster.py:166-184) of a label texture: d_out n*n, counts_out n_regions+1 */
int det_density(det_ctx *ctx, const int32_t *labels, const double *stats, int n_regions, double bdv, double *d_out,
                int64_t *counts_out);
/* interpolate_vertices (temporal.py:293-302): out[f][i] = a[i] + fracs[f]*(b[i]-a[i]), float64,
 * reference op order; len doubles per frame (vertex rows*2 followed by R statistics). */
int det_interpolate(det_ctx *ctx, const double *a, const double *b, long long len, const double *fracs, int n_frac,
                    double *out);
int det_advect(det_ctx *ctx, const double *u, const double *xy, int n_pts, double *xy_out, int64_t *clamps);

/* Frame quality metrics (the per-frame report of temporal.py:203-209).  They
 * need no loaded map: each call carries its layouts (ring_start: n_rings+1 row offsets, ring_region:
 * owning region of every ring, grouped in region order).
 * det_shape_metrics replaces metrics.py:82-135 (hamming_distance / shape_distortion) plus
 * Region.area / Region.centroid (geomodel.py:63-77): map a (one vertex set) against `frames` vertex
 * sets of map b (frames*rows_b*2 doubles, one layout).  Per (frame, region): hamming (NaN unless
 * status is 0), area_b, cent_b (2 doubles) and status (0 ok; 1/2 non-positive area of map a/b ->
 * NumericError; 3 a shape rasterised to zero pixels -> RasterizationError; 4/5 negative toggle index
 * in map a/b -> ValueError, as np.bincount raises).  cent_a is R*2.  raster_k in [1, 8]; raster_k = 0
 * computes areas and centroids only (status 0, hamming NaN). */
int det_shape_metrics(det_ctx *ctx, int n_regions, const double *xy_a, int rows_a, const int32_t *ring_start_a,
                      int rings_a, const int32_t *ring_region_a, const double *xy_b, int rows_b,
                      const int32_t *ring_start_b, int rings_b, const int32_t *ring_region_b, int frames,
                      int raster_k, int rescale, double *hamming, double *area_b, double *cent_a, double *cent_b,
                      int32_t *status);
/* detect_adjacencies (geomodel.py:380-415) of `frames` vertex sets (frames*n_rows*2 doubles) sharing
 * one layout; row_region is the owning region of every row.  Region index pairs (a < b) sharing >= 2
 * epsilon-cells, as (frame, a, b) int32 triples sorted by frame, a, b; min(count, cap) triples are
 * written and *n_pairs = count. */
int det_adjacency(det_ctx *ctx, const double *xy, int frames, int n_rows, const int32_t *row_region, int n_regions,
                  double epsilon, int32_t *pairs, long long cap, long long *n_pairs);
/* relative_position_error numerator (metrics.py:138-162): per frame, the sum over ordered pairs
 * u != v of |atan2(cross, dot)| between barycenter vectors of cent_m (R*2) and cent_c[f] (R*2),
 * plus the count of degenerate pairs. */
int det_position_error(det_ctx *ctx, const double *cent_m, const double *cent_c, int frames, int n_regions,
                       double *sums_out, long long *degenerate_out);

#ifdef __cplusplus
}
#endif
#endif
