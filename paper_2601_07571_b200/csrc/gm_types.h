// gm_types.h -- records shared by the host setup (gm_setup.cpp) and the
// sm_100a kernels (gm_kernels.cu).  Plain C layout, no torch types.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define GM_HD __host__ __device__
#else
#define GM_HD
#endif

// Exact per-fixation parameters (float64), restating what
// density.py:148-200 hands to kernels.rasterize / kernels.accumulate.
struct __attribute__((aligned(16))) GmFixExact {
    double rot[9];    // view rotation R^T (gaze.py:120)
    double trans[3];  // -R^T @ pos (gaze.py:121, BLAS FMA chain)
    double gaze[3];   // fixation.gaze_dir (camera space, unit)
    double amp;       // duration / (sigma sqrt(2 pi)) (density.py:179)
    double p00, p11, p02, p12;  // projection xy terms (crop or full)
    double near_, far_;         // frustum_from_matrix near'/far' (gaze.py:345-356)
    double near_lo, far_hi;     // near'(1-1e-9), far'(1+1e-9) (kernels.py:312)
    double cropped;             // 1.0 when the crop frustum was used
    double pad_;
};  // 26 doubles = 208 B

// Conservative float32 culling record of one fixation, world space.
// Cone = 4-sigma cone around the world gaze ray from the camera position.
struct __attribute__((aligned(16))) GmFixCull {
    float ox, oy, oz, margin;    // camera position, absolute slack (m)
    float gx, gy, gz, pad0;      // world gaze direction (unit)
    float fx, fy, fz, pad1;      // world camera forward (unit, -z axis)
    float cos_s, sin_s, cos_t, sin_t;  // sample cone / occluder cone (<-1.5: no cone)
    float near_f, far_f, pad2, pad3;   // conservative depth slab along forward
};  // 80 B

// One projected, clipped, winding-normalised triangle ready for the
// per-pixel edge tests of kernels.py:_raster_tri (values exactly as numba
// computes them before its pixel loop).
struct __attribute__((aligned(16))) GmScreenTri {
    double sx0, sy0, sx1, sy1, sx2, sy2;
    double iw0, iw1, iw2, inv_area;
    uint16_t x0, x1, y0, y1;  // inclusive pixel bbox clamped to the buffer
    uint32_t tl;              // bits 0-2: top-left ownership of edges 0, 1, 2; bits 3+: order key
                              // 2 t + fan (t < 2^28), the rasterization order of kernels.py:158-192
    float minw;               // min vertex depth, rounded down (a lower bound of every depth it writes)
};  // 96 B

// Per-config constants for the host setup.
struct GmSetupConsts {
    double theta, sigma, phi;
    double cos_hp, sin_hp;   // cos/sin(0.5 * phi)
    double cos_hm, sin_hm;   // cos/sin(0.5 * -phi)
    double cos_phi, sin_phi;
    double sqrt_two_pi;
    int filtering;
    int width, height;
};

// Public config (mirrors GenerationConfig, density.py:44-71).
struct GmConfig {
    double theta;
    double eps_abs;
    double eps_rel;
    int32_t zbuffer_resolution;
    int32_t filtering;
    int32_t batch;   // fixations per batch (0 = auto)
    int32_t flags;
};

// Per-phase device milliseconds (CUDA events), mirrors Timings.phases.
struct GmTimings {
    double setup_ms;       // host fixation setup (wall)
    double cull_ms;        // occluder cull + clip + project (device)
    double rasterize_ms;   // screen-space binning (device)
    double accumulate_ms;  // filter + depth test + Gaussian (device, k_samples<false>)
    double total_ms;       // whole call (wall)
    double mark_ms;        // candidate texel marking (device, k_samples<true>)
    double texel_ms;       // marked z-buffer texels (device, k_texels)
    int64_t screen_tris;   // projected triangles produced
    int64_t bin_items;     // reserved
    int64_t batches;
    int64_t retries;       // passes resumed after a screen-triangle segment overflow
};

#ifdef __cplusplus
static_assert(sizeof(GmFixExact) == 26 * 8, "GmFixExact layout (Python binds 26 float64)");
static_assert(sizeof(GmFixCull) == 20 * 4, "GmFixCull layout");
static_assert(sizeof(GmScreenTri) == 96, "GmScreenTri layout");
#endif

#define GM_NDC_SLACK 1e-9
#define GM_FIX_STRIDE 18

enum {
    GM_OK = 0,
    GM_ERR_CUDA = 1,
    GM_ERR_ARG = 2,
    GM_ERR_INVALID_FRUSTUM = 3,
    GM_ERR_NO_DEVICE = 4,
    GM_ERR_OOM = 5,
    GM_ERR_UNSUPPORTED = 6,
    GM_ERR_GAZE_OUTSIDE = 7,
};
