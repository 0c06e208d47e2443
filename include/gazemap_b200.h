/*
 * gazemap_b200.h -- C ABI of the B200-native density-map generation path.
 *
 * Library: paper_2601_07571_b200/_gazemap_b200.so (sm_100a kernels, static
 * cudart, host OpenMP).  Plain pointers and sizes only; every entry point
 * returns an int status (0 = GM_OK) and never throws; gm_last_error() gives
 * the message of the calling thread's last failure.  All host buffers are
 * owned by the caller; the library allocates only device memory it owns.
 *
 * Reference interface replaced (paths under /root/reference/pkg/src/gazemap):
 * the reference has no FFI; its hot path sits behind numba kernels called from
 * Python (kernels.py) and the Python functions of geometry.py / density.py.
 * Each entry point below names the function(s) it replaces.
 */
#ifndef GAZEMAP_B200_H
#define GAZEMAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GM_OK = 0,
    GM_ERR_CUDA = 1,             /* CUDA runtime failure */
    GM_ERR_ARG = 2,              /* invalid argument -> ConfigError */
    GM_ERR_INVALID_FRUSTUM = 3,  /* perspective_matrix bounds -> InvalidFrustumError (gaze.py:325-328) */
    GM_ERR_NO_DEVICE = 4,        /* no CUDA device: there is no CPU fallback */
    GM_ERR_OOM = 5,
    GM_ERR_UNSUPPORTED = 6,
    GM_ERR_GAZE_OUTSIDE = 7      /* 4-sigma cone misses the near plane -> GazeOutsideFrustumError */
};

/* Fixation table: F rows x 18 float64 in the fixation-log column order
 * (gaze.py:133-136): start_time, duration, camera position xyz, camera
 * rotation quaternion xyzw, frustum l r t b n f, gaze direction xyz
 * (unit, as Fixation.__post_init__ leaves it, gaze.py:91-95). */
#define GM_FIX_STRIDE 18

/* GenerationConfig (density.py:44-71); k is consumed by gm_layout. */
typedef struct GmConfig {
    double theta;               /* 1-sigma gaze angle, radians (0, pi/2) */
    double eps_abs;             /* depth tolerance, meters (raster.py:30) */
    double eps_rel;             /* relative depth tolerance (raster.py:31) */
    int32_t zbuffer_resolution; /* square z-buffer side, 1..65535 */
    int32_t filtering;          /* 1: 4-sigma crop frustum, 0: full frustum */
    int32_t batch;              /* fixations per GPU batch, 0 = auto */
    int32_t flags;              /* 0, or GM_FLAG_* below */
} GmConfig;

/* Timings.phases (density.py:94-103), measured with CUDA events. */
typedef struct GmTimings {
    double setup_ms;      /* host fixation setup */
    double cull_ms;       /* occluder cull + clip + projection */
    double rasterize_ms;  /* screen binning */
    double accumulate_ms; /* NDC filter + cone + depth test + Gaussian */
    double total_ms;      /* whole call, wall */
    double mark_ms;       /* candidate texel marking */
    double texel_ms;      /* z-buffer values of the marked texels */
    int64_t screen_tris;  /* projected triangles produced */
    int64_t bin_items;    /* reserved */
    int64_t batches;
    int64_t retries;      /* passes resumed after a screen-triangle segment overflow */
} GmTimings;

/* GmConfig.flags */
#define GM_FLAG_STATS 1       /* count work (gm_plan_stats); untimed diagnostics */
#define GM_FLAG_ONE_STREAM 2  /* batches on one stream (default for > 400k occluder triangles) */
#define GM_FLAG_TWO_STREAMS 4 /* overlap consecutive batches on two streams (default otherwise) */

typedef struct gm_plan gm_plan;
typedef void (*gm_progress_fn)(int64_t done, int64_t total, void* user);

const char* gm_last_error(void);
int gm_abi_version(void);
int gm_device_count(void);
/* Measured FMA throughput of `device` in TFLOP/s (fp64 != 0: float64, else
 * float32): the SIMT roofline denominators bench.py reports against. */
int gm_peak_flops(int device, int fp64, double* tflops);

/* ---- stage 1: sampling -------------------------------------------------- */

/* build_sampled_mesh (geometry.py:305-320): triangle_areas :169-176,
 * adaptive_resolutions :202-210, counts, exclusive-prefix offsets, total.
 * tri_local: T x 3 x 3 corner positions.  Outputs may be NULL except total. */
int gm_layout(int device, const double* tri_local, int64_t T, double k, int64_t* res, int64_t* counts,
              int64_t* offsets, int64_t* total);

/* sample_positions_local (geometry.py:331-346), then Transform.apply
 * (geometry.py:86-89) when xform = [t(3), q xyzw(4), s(3)] is non-NULL.
 * out: N x 3. */
int gm_sample_positions(int device, const double* tri_local, int64_t T, const int64_t* res,
                        const int64_t* offsets, int64_t N, const double* xform, double* out);

/* normalize (density.py:230-244) of n values by gmax > 0. */
int gm_normalize(int device, const double* values, int64_t n, double gmax, double* out);

/* ---- per-fixation setup (host, bit-exact with CPython + glibc) ---------- */

/* Fixation.view_matrix (gaze.py:114-122), build_crop_frustum (gaze.py:372-381)
 * with the GazeOutsideFrustumError fallback of density.py:152-158,
 * frustum_from_matrix (gaze.py:345-356).  ex: F x 26 float64 (GmFixExact in
 * csrc/gm_types.h), cull: F x 20 float32 or NULL. */
int gm_fixation_setup(const double* fixations, int64_t F, double theta, int filtering, int res, double* ex,
                      void* cull, int64_t* bad_fixation);

/* The per-config constants of that setup (GmSetupConsts in csrc/gm_types.h:
 * tan / atan / cos / sin of the cone angles), computed once ... */
void gm_setup_consts(double theta, int filtering, int width, int height, void* consts);
/* ... and the setup of one fixation row (18 float64) under them: GM_OK, or
 * GM_ERR_INVALID_FRUSTUM where the reference's perspective_matrix raises
 * InvalidFrustumError (accumulate_fixation's per-call check, density.py:148-158). */
int gm_fixation_check(const double* fixation, const void* consts);

/* ellipse_intersection(gaze_dir, n, cone) (gaze.py:252-309) for the cone's
 * 4-sigma half-angle phi: out[18] = center_E[3], major_a, minor_b,
 * inclination_alpha, A0[3], A1[3], B0[3], B1[3]; GM_ERR_GAZE_OUTSIDE when
 * the cone does not cut the near plane in an ellipse. */
int gm_ellipse_intersection(const double* gaze, double n, double phi, double* out);
/* crop_bounds (gaze.py:312-320): (l', r', b', t') of an out[18] above. */
int gm_crop_bounds(const double* ellipse, double* lrbt);

/* ---- scene plan: occluders + samples resident on one GPU ---------------- */

int gm_plan_create(int device, gm_plan** out);
void gm_plan_destroy(gm_plan* plan);
int gm_plan_set_host_threads(gm_plan* plan, int n);

/* _SampleCache (density.py:106-121) + scene_world_triangles (raster.py:68-78):
 * n_obj objects with tri_counts[o] triangles, local corners tri_local
 * (sum T x 9, object order), transforms xforms (n_obj x [t, q, s]), the
 * SampledMesh resolutions res (sum T) and include flags (object_include_list,
 * density.py:130-133).  Occluders are all objects; samples are the included
 * objects' samples concatenated in object order. */
int gm_plan_set_scene(gm_plan* plan, int n_obj, const int64_t* tri_counts, const double* tri_local,
                      const double* xforms, const int64_t* res, const uint8_t* include);
/* Replace the object poses (n_obj x [t, q, s]) of a plan: world triangles and
 * sample positions are recomputed from the local layout on the device
 * (Transform.apply, geometry.py:86-89, as _SampleCache.world applies a pose
 * override, density.py:121-127, and scene_world_triangles(scene, overrides),
 * raster.py:68-78).  The accumulated values are kept: generate() walks a
 * dynamic-scene log as runs of fixations sharing one override set. */
int gm_plan_set_poses(gm_plan* plan, const double* xforms);
int64_t gm_plan_num_samples(gm_plan* plan);
int64_t gm_plan_num_triangles(gm_plan* plan);
double* gm_plan_values_device(gm_plan* plan); /* device pointer to the N accumulators */

/* generate / accumulate_fixation (density.py:136-227): add the F fixations, in
 * log order, into the plan's device values (zeroed first if reset).  One
 * fused pass per batch replaces cull_mask + rasterize + accumulate
 * (kernels.py:140-340).  progress(done, total) is called as batches complete. */
int gm_plan_accumulate(gm_plan* plan, const double* fixations, int64_t F, const GmConfig* cfg, int reset,
                       GmTimings* timings, gm_progress_fn progress, void* user, int64_t* bad_fixation);

/* Device-resident replay (bench): compute the F fixations' setup records once
 * into HBM, then gm_plan_run repeats the whole generation from them (flags
 * as GmConfig.flags); device_ms = CUDA-event time of the pass on the plan's
 * stream. */
int gm_plan_prepare(gm_plan* plan, const double* fixations, int64_t F, const GmConfig* cfg, int64_t* bad_fixation);
int gm_plan_run(gm_plan* plan, int reset, int flags, GmTimings* timings, float* device_ms);
/* Write `bytes` of scratch on the plan's stream to evict L2 between repetitions. */
int gm_plan_flush_l2(gm_plan* plan, int64_t bytes);

/* Work counters of the last pass run with GmConfig.flags & 1: 20 x uint64 =
 * super-chunk tests, chunk tests, exact sample evaluations, NDC-filtered
 * samples, in-cone candidates, visible contributions, marked texels, exact
 * (texel, triangle) evaluations, covered pairs, depth tests decided by the
 * tile-max occlusion test, 9 k_texels counters, and the screen triangles'
 * summed pixel bboxes = the pixel tests of the reference's rasterizer
 * (kernels.py:103-137) for the same batch (names: _native.STAT_NAMES). */
int gm_plan_stats(gm_plan* plan, unsigned long long* out);

/* Self-check counters (16 x uint64, names: _native.CHECK_NAMES) accumulated by
 * a GM_CHECK build (bound / cull / depth-test decisions re-done in exact
 * float64 and compared); zeros in production builds.  reset != 0 zeroes them.
 * *is_check_build = 1 for a GM_CHECK build. */
int gm_plan_check(gm_plan* plan, unsigned long long* out, int reset, int* is_check_build);
/* Testing hook: restart the per-fixation screen-triangle segments at `cap`
 * entries, so the next run exercises the overflow -> grow -> resume path. */
int gm_plan_set_segment_capacity(gm_plan* plan, int64_t cap);

/* Running global max (density.py:192) of the plan's values. */
int gm_plan_max(gm_plan* plan, double* gmax);
/* Copy values to host: raw (may be NULL) and/or normalized = raw / gmax. */
int gm_plan_read(gm_plan* plan, double* raw, double* normalized, double gmax);
int gm_plan_write(gm_plan* plan, const double* raw);
int gm_plan_sync(gm_plan* plan);

/* ---- multi-GPU: fixation-sharded partial maps, fused peer reduce (§8e) ---
 * Replaces the all-reduce + global max of the sharded generate
 * (density.py:223-226 is a sum over fixations; the max of density.py:192 is
 * taken on the sum).  One process per GPU: every rank exports the IPC handle
 * of its accumulator (64 bytes), the host exchanges them (torch.distributed),
 * each rank opens its peers' maps; after a host barrier (all partial maps
 * complete) gm_plan_reduce_peers sums slice `rank` over the ranks in rank
 * order through NVLink peer loads, stores the sum into every rank's map and
 * returns the slice max; after a second barrier every rank holds the full sum
 * and the global max is the max of the slice maxima. */
int gm_plan_ipc_handle(gm_plan* plan, void* handle64);
int gm_plan_open_peers(gm_plan* plan, int rank, int world, const void* handles64);
int gm_plan_reduce_peers(gm_plan* plan, double* slice_max, float* device_ms);

/* ---- kernel-seam ports (parity instruments) ----------------------------- */

/* kernels.rasterize (kernels.py:140-192) via raster.rasterize_triangles
 * (raster.py:99-124): res x res depth (+inf where empty) of the plan's
 * occluders for one fixation row; no_cull = 1 projects every triangle. */
int gm_plan_depth_buffer(gm_plan* plan, const double* fixation, double theta, int filtering, int res,
                         int no_cull, double* depth);

/* The NDC crop filter (kernels.py:302-319) as per-fixation candidate lists
 * (warp-ballot compaction): out F x cap (unsorted per row), counts F. */
int gm_plan_candidates(gm_plan* plan, const double* fixations, int64_t F, double theta, int filtering, int res,
                       int64_t* out, int64_t cap, int64_t* counts);

/* World sample positions of the plan (N x 3), _SampleCache.base_world. */
int gm_plan_positions(gm_plan* plan, double* out);

/* ---- general camera: z-buffer, attributes, heatmap (kernel seam + 8f-2) --- */

/* kernels.rasterize (kernels.py:140-192) of world triangles (T x 3 x 3, the
 * order is the rasterization order) for one camera: rot 3x3 row-major and
 * trans 3 (world -> camera), the projection's p00 p11 p02 p12, a W x H buffer,
 * near/far.  depth (H x W, +inf where nothing is drawn) always; with_attrs
 * outputs when non-NULL: tri_id (H x W, -1 where empty) and the
 * perspective-correct barycentrics bary (H x W x 3) of the winning triangle
 * (the first in order among equal minimum depths).  Used by
 * raster.rasterize_triangles / rasterize_depth (raster.py:99-137). */
int gm_rasterize(int device, const double* tris, int64_t T, const double* rot, const double* trans, double p00,
                 double p11, double p02, double p12, int W, int H, double near_, double far_, double* depth,
                 int32_t* tri_id, double* bary);

/* render_heatmap (render.py:95-186) after the camera setup: rasterize every
 * triangle with attributes, interpolate the density over each triangle's
 * sample grid (res: per-triangle resolution, base: the triangle's first
 * sample in `values`), colormap (n_stops <= 16 stops, colors n_stops x 3,
 * gamma) and round to uint8; img is H x W x 3 (background black). */
int gm_render_heatmap(int device, const double* tris, int64_t T, const double* rot, const double* trans, double p00,
                      double p11, double p02, double p12, int W, int H, double near_, double far_,
                      const int64_t* res, const int64_t* base, const double* values, int64_t N, const double* stops,
                      const double* colors, int n_stops, double gamma, uint8_t* img);

/* kernels.cull_mask (kernels.py:195-216) on the GPU: keep[t] = 0 iff all
 * three vertices of triangle t are outside one of the n_planes planes. */
int gm_cull_mask(int device, const double* tris, int64_t T, const double* planes, int n_planes, uint8_t* keep);

/* kernels.depth_match (kernels.py:219-285) on a host H x W buffer (host
 * scalar query, raster.is_visible). */
int gm_depth_match(const double* depth, int64_t height, int64_t width, double fx, double fy, double d, double eps);

/* ---- fixation-log ingestion ----------------------------- */

/* parse_fixation_log (gaze.py:130-188) line scanner over an in-memory log
 * (bytes of the file).  Multi-threaded (threads <= 0: all) over line-aligned
 * chunks.  Produces every numeric row before the first failing line: the
 * 18 fields with the gaze normalised like Fixation.__post_init__
 * (gaze.py:91-95), the row's Fixation validation verdict, its source line and
 * its pose-override groups (object id + 10 floats).  The time window and the
 * error policy are applied by the caller (fixlog.py).  Returns 0 and a handle
 * unless the arguments are invalid. */
typedef struct gm_fixlog gm_fixlog;
int gm_fixlog_parse(const char* buf, int64_t len, int threads, gm_fixlog** out);
int64_t gm_fixlog_rows(const gm_fixlog* log);
int64_t gm_fixlog_groups(const gm_fixlog* log);
/* table rows x 18; line rows; code rows (0 valid, 1 zero gaze, 2 duration,
 * 3 near/far, 4 bounds, 5 gaze z >= 0); gstart rows + 1; goid groups x 2 (byte
 * offset, length of the object id); gvals groups x 10.  Outputs may be NULL. */
int gm_fixlog_copy(const gm_fixlog* log, double* table, int64_t* line, int32_t* code, int64_t* gstart,
                   int64_t* goid, double* gvals);
/* info[7]: kind (0 none, 1 < 18 fields, 2 bad number, 3 override group count,
 * 4 bad override number, 5 non-ASCII buffer, 6 separators-only line), line,
 * token offset, token length, field count, line offset, line length. */
int gm_fixlog_error(const gm_fixlog* log, int64_t* info);
void gm_fixlog_free(gm_fixlog* log);

/* ---- export wire format --------------------------------- */

/* write_export records (io_export.py:63-116) of one object, byte-identical to
 * the reference: "oid,tri,within,w1,w2,w3,lx,ly,lz,wx,wy,wz,value\n" per
 * sample, floats as Python f"{x:.9g}".  res/offsets: the SampledMesh layout
 * (T); local/world: N x 3; values: N.  OpenMP over sample ranges. */
typedef struct gm_buffer gm_buffer;
int gm_export_format(const char* oid, int64_t oid_len, const int64_t* res, const int64_t* offsets, int64_t T,
                     int64_t N, const double* local, const double* world, const double* values, int threads,
                     gm_buffer** out);
const char* gm_buffer_data(const gm_buffer* buf);
int64_t gm_buffer_size(const gm_buffer* buf);
void gm_buffer_free(gm_buffer* buf);

#ifdef __cplusplus
}
#endif
#endif /* GAZEMAP_B200_H */
