// gm_kernels.cu -- sm_100a kernels and the C-ABI of the B200 density-map path.
//
// Path and where each piece lives:
//   a1-a6   sampling: k_layout (Heron area -> r -> count), CUB scan (offsets),
//           k_positions (index -> row/col -> barycentric -> world, FMA-chain
//           transform like OpenBLAS), k_world_tris                      [here]
//   a8-a10  per-fixation setup: host, gm_setup.cpp (glibc trig, bit-exact)
//   a11-a12 occluders: k_tri_setup (conservative cone cull, exact camera
//           transform + near clip + projection + _raster_tri setup) into
//           per-fixation screen-triangle segments; k_coarse bins   [here]
//   a13-a15 gm_samples.cuh: k_level1 ballots, k_mark (float32 superset of the
//           NDC filter + 4-sigma cone, marks the <= 9 texels depth_match
//           reads, level-3 candidate words), k_samples (exact filter,
//           depth_match, Gaussian, accumulated in log order)
//   a12     gm_texels.cuh: k_texels, the marked texels' min depth (float32
//           selection with rigorous bounds, exact float64 evaluation)
//   a16     k_max / k_normalize                                          [here]
//   a17     the plan: scene upload, two-stream double-buffered batch pipeline,
//           C-ABI entry points                                           [here]
//   seam    gm_raster.cuh: general-camera rasterize (+ attributes), heatmap
//           renderer, cull_mask
// Exactness: compiled with -fmad=false; see gm_device.cuh.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "gm_device.cuh"
#include "gm_types.h"

#define GM_MAX_BATCH 1024
#ifndef SAMPLE_GRID_MULT
#define SAMPLE_GRID_MULT 1  // persistent sample-pass grid = resident CTAs x this
#endif
// launch bounds of the hot kernels (k_texels / k_texels_crowded: TX_WARPS_SM* / HV_*_WARPS_SM in
// gm_texels.cuh); -DKS_MINB=n etc. (build variants) re-size their register budgets
#ifndef KS_MINB
#define KS_MINB 4  // k_samples: 4 CTAs (32 warps) per SM, 64 registers (C5 accumulate 269 -> 245 ms;
#endif             // uncapped: 80 registers, 3 CTAs)
#if KS_MINB > 0
#define KS_BOUNDS __launch_bounds__(256, KS_MINB)
#else
#define KS_BOUNDS __launch_bounds__(256)
#endif
#ifdef KM_MINB
#define KM_BOUNDS __launch_bounds__(256, KM_MINB)
#else
#define KM_BOUNDS __launch_bounds__(256)
#endif

extern "C" void gm_setup_consts(double theta, int filtering, int width, int height, GmSetupConsts* c);
extern "C" int64_t gm_setup_batch(const double* fx, int64_t F, const GmSetupConsts* c, GmFixExact* ex,
                                  GmFixCull* cull, int threads);

using namespace gm;

// ------------------------------------------------------------------ errors

static thread_local std::string g_err;

static int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                                           \
    do {                                                                                                \
        cudaError_t e_ = (x);                                                                           \
        if (e_ != cudaSuccess)                                                                          \
            return set_err(e_ == cudaErrorMemoryAllocation ? GM_ERR_OOM : GM_ERR_CUDA,                   \
                           std::string(#x) + ": " + cudaGetErrorString(e_));                             \
    } while (0)

// Frees the device temporaries of an entry point on every return path
// (CK() returns early on the first failing call).
struct DevScratch {
    std::vector<void*> ptrs;
    template <typename T>
    cudaError_t alloc(T** p, size_t bytes) {
        *p = nullptr;
        cudaError_t e = cudaMalloc((void**)p, bytes);
        if (e == cudaSuccess) ptrs.push_back((void*)*p);
        return e;
    }
    ~DevScratch() {
        for (void* q : ptrs) cudaFree(q);
    }
};

extern "C" const char* gm_last_error(void) { return g_err.c_str(); }
extern "C" int gm_abi_version(void) { return 1; }

static int use_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return set_err(GM_ERR_NO_DEVICE, "no CUDA device visible");
    if (device < 0 || device >= n) return set_err(GM_ERR_ARG, "device index out of range");
    CK(cudaSetDevice(device));
    return GM_OK;
}

// -------------------------------------------------------------- sampling

// geometry.py:169-176 + :202-210: Heron area -> adaptive resolution -> count.
__global__ void k_layout(const double* __restrict__ tri, int64_t T, double k8, const int64_t* res_in, int64_t* res,
                         int64_t* __restrict__ cnt) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    int64_t r;
    if (res_in) {
        r = res_in[t];
    } else {
        const double* v = tri + 9 * t;
        double len[3];
        const int ia[3] = {0, 3, 0}, ib[3] = {3, 6, 6};
#pragma unroll
        for (int e = 0; e < 3; e++) {
            double ex = v[ib[e]] - v[ia[e]], ey = v[ib[e] + 1] - v[ia[e] + 1], ez = v[ib[e] + 2] - v[ia[e] + 2];
            len[e] = sqrt((ex * ex + ey * ey) + ez * ez);  // norm(axis=1)
        }
        double a = len[0], b = len[1], c = len[2];
        double s = 0.5 * (a + b + c);
        double rad = s * (s - a) * (s - b) * (s - c);
        double area = sqrt(rad > 0.0 ? rad : 0.0);
        double delta = 1.0 + k8 * area;
        r = (int64_t)ceil((-3.0 + sqrt(delta)) / 2.0);
        if (delta < 25.0) r = 1;
        if (r < 1) r = 1;
    }
    if (res) res[t] = r;
    cnt[t] = (r + 1) * (r + 2) / 2;
}

// geometry.py:331-346 sample_positions_local (+ :86-89 Transform.apply when
// M != nullptr).  One thread per sample; the owning triangle is found by
// binary search over the exclusive prefix offsets.
__global__ void k_positions(const double* __restrict__ tri, int64_t T, const int64_t* __restrict__ res,
                            const int64_t* __restrict__ off, int64_t N, const double* __restrict__ M,
                            const double* __restrict__ tr, double* __restrict__ out_aos, double* __restrict__ ox,
                            double* __restrict__ oy, double* __restrict__ oz) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int64_t lo = 0, hi = T - 1;  // last t with off[t] <= i
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (off[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    int64_t t = lo;
    int64_t idx = i - off[t];
    // sample_rowcol (geometry.py:232-242)
    int64_t row = (int64_t)ceil((-3.0 + sqrt(8.0 * (double)idx + 9.0)) / 2.0);
    int64_t col = idx - row * (row + 1) / 2;
    if (col < 0) row -= 1;
    col = idx - row * (row + 1) / 2;
    if (col > row) row += 1;
    col = idx - row * (row + 1) / 2;
    double r = (double)res[t];
    double w1 = (double)col / r;
    double w2 = (double)(row - col) / r;
    double w3 = 1.0 - (double)row / r;
    const double* v = tri + 9 * t;
    double p[3];
#pragma unroll
    for (int c = 0; c < 3; c++) p[c] = w1 * v[c] + w2 * v[3 + c] + w3 * v[6 + c];
    if (M) {
        double q[3];
#pragma unroll
        for (int c = 0; c < 3; c++) q[c] = blas_dot3(p[0], M[3 * c], p[1], M[3 * c + 1], p[2], M[3 * c + 2]) + tr[c];
        p[0] = q[0]; p[1] = q[1]; p[2] = q[2];
    }
    if (out_aos) {
        out_aos[3 * i] = p[0];
        out_aos[3 * i + 1] = p[1];
        out_aos[3 * i + 2] = p[2];
    }
    if (ox) {
        ox[i] = p[0];
        oy[i] = p[1];
        oz[i] = p[2];
    }
}

// SceneObject.world_triangles (geometry.py:120-124) for one object.
__global__ void k_world_tris(const double* __restrict__ tri, int64_t T, const double* __restrict__ M,
                             const double* __restrict__ tr, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // vertex
    if (i >= 3 * T) return;
    const double* p = tri + 3 * i;
#pragma unroll
    for (int c = 0; c < 3; c++) out[3 * i + c] = blas_dot3(p[0], M[3 * c], p[1], M[3 * c + 1], p[2], M[3 * c + 2]) + tr[c];
}

__global__ void k_tri_spheres(const double* __restrict__ tw, int64_t T, float4* __restrict__ tsph) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const double* v = tw + 9 * t;
    double c[3], r2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; a++) c[a] = (v[a] + v[3 + a] + v[6 + a]) / 3.0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        double dx = v[3 * k] - c[0], dy = v[3 * k + 1] - c[1], dz = v[3 * k + 2] - c[2];
        r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
    }
    double cm = fmax(fabs(c[0]), fmax(fabs(c[1]), fabs(c[2])));
    tsph[t] = make_float4((float)c[0], (float)c[1], (float)c[2], (float)(sqrt(r2) * (1.0 + 1e-6) + 1e-5 * (1.0 + cm)));
}

// Sphere enclosing 32 consecutive member spheres (triangle clusters) or
// 32 consecutive samples (sample chunks).
__global__ void k_group_spheres(const float4* __restrict__ member, const double* __restrict__ px,
                                const double* __restrict__ py, const double* __restrict__ pz, int64_t n,
                                float4* __restrict__ out, int group) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t first = g * group;
    if (first >= n) return;
    int64_t last = first + group < n ? first + group : n;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t i = first; i < last; i++) {
        double p[3], r;
        if (member) {
            float4 s = member[i];
            p[0] = s.x; p[1] = s.y; p[2] = s.z; r = s.w;
        } else {
            p[0] = px[i]; p[1] = py[i]; p[2] = pz[i]; r = 0.0;
        }
        for (int a = 0; a < 3; a++) {
            lo[a] = fmin(lo[a], p[a] - r);
            hi[a] = fmax(hi[a], p[a] + r);
        }
    }
    double c[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    double r2 = 0.0;
    for (int64_t i = first; i < last; i++) {
        double p[3], r;
        if (member) {
            float4 s = member[i];
            p[0] = s.x; p[1] = s.y; p[2] = s.z; r = s.w;
        } else {
            p[0] = px[i]; p[1] = py[i]; p[2] = pz[i]; r = 0.0;
        }
        double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
        double d = sqrt(dx * dx + dy * dy + dz * dz) + r;
        r2 = fmax(r2, d);
    }
    double cm = fmax(fabs(c[0]), fmax(fabs(c[1]), fabs(c[2])));
    out[g] = make_float4((float)c[0], (float)c[1], (float)c[2], (float)(r2 * (1.0 + 1e-6) + 1e-5 * (1.0 + cm)));
}

// ------------------------------------------------------ occluder setup

// Per-batch screen-triangle store: fixation slot f owns the segment
// [f * cap_seg, (f + 1) * cap_seg) of `tris` (records) and `bbox` (their
// inclusive pixel boxes, packed x0 | x1 << 16, y0 | y1 << 16, scanned by
// k_texels); count[f] is the number appended.  Overflow never corrupts a
// result: the first batch that overflows sets *fail (sticky) and every later
// kernel of that and following batches returns immediately; the host grows
// the segments and resumes from that batch (log order is preserved).
// float32 form of one screen triangle for k_texels' selection stage: the
// three edge-function planes and the inverse-depth plane in the triangle's
// bbox-local pixel frame (x - x0, y - y0), with error bounds that cover both
// the float32 evaluation at any pixel centre of the bbox and the reference's
// own float64 rounding (kernels.py:107-125): |e32 - e_ref| <= tol,
// |invw32 - invw_ref| <= tolw.  Built once per screen triangle in k_tri_setup.
#ifndef TRI80
#define TRI80 1  // 80-byte TriF32 with one edge tolerance (the max of the three) instead of 96 bytes
#endif
#if TRI80
struct __align__(16) TriF32 {
    float inv_minw;                  // >= every inverse depth the triangle writes
    float ox, oy;                    // frame origin = bbox corner (x0, y0), pixels
    float wx;                        // bbox extent x1 - x0 + 1 (and wy): pixel centre c = (px + 0.5,
    float wy;                        // py + 0.5) is in the bbox iff 0 < c - o < w (exact in float32)
    int gidx;                        // index of the float64 record in the fixation's segment
    float tol, tolw;                 // edge-function (all three edges) and inverse-depth bounds
    float a[3], b[3], c[3];          // e_i = a x + b y + c
    float A, B, C;                   // inverse depth
};  // 80 B, every byte written
static_assert(sizeof(TriF32) == 80, "TriF32 is five 16-byte words");
#define TRI_TOL(t, i) ((t).tol)
#else
struct __align__(16) TriF32 {
    float a[3], b[3], c[3], tol[3];  // e_i = a x + b y + c
    float A, B, C, tolw;             // inverse depth
    float inv_minw;                  // >= every inverse depth the triangle writes
    float ox, oy;                    // frame origin = bbox corner (x0, y0), pixels
    float wx, wy;                    // bbox extent x1 - x0 + 1, y1 - y0 + 1: pixel centre c = (px + 0.5,
                                     // py + 0.5) is in the bbox iff 0 < c - o < w (exact in float32)
    int gidx;                        // index of the float64 record in the fixation's segment
    int pad[2];                      // (explicit: every byte of the 96 is written and copied)
};  // 96 B
static_assert(sizeof(TriF32) == 96, "TriF32 is six 16-byte words");
#define TRI_TOL(t, i) ((t).tol[i])
#endif
constexpr int TRI_WORDS = (int)sizeof(TriF32) / 16;  // 16-byte words per record (staging copies)

__device__ __forceinline__ void make_tri_f32(const GmScreenTri& T, int gidx, TriF32& o) {
    const double ox = T.x0, oy = T.y0;
    const double sx[3] = {T.sx0 - ox, T.sx1 - ox, T.sx2 - ox}, sy[3] = {T.sy0 - oy, T.sy1 - oy, T.sy2 - oy};
    const double iw[3] = {T.iw0, T.iw1, T.iw2};
    const double xmax = (double)(T.x1 - T.x0 + 1), ymax = (double)(T.y1 - T.y0 + 1);
    double A = 0.0, B = 0.0, C = 0.0, Aab = 0.0, Bab = 0.0, Cab = 0.0;
#if TRI80
    double tol = 0.0;
#endif
#pragma unroll
    for (int i = 0; i < 3; i++) {
        // edge i runs from vertex (i+1)%3 to (i+2)%3: w_i = (bx-ax)(py-ay) - (by-ay)(px-ax)
        const int ia = (i + 1) % 3, ib = (i + 2) % 3;
        const double ex = sx[ib] - sx[ia], ey = sy[ib] - sy[ia];
        const double a = -ey, b = ex, c = ey * sx[ia] - ex * sy[ia];
        o.a[i] = (float)a;
        o.b[i] = (float)b;
        o.c[i] = (float)c;
        // float32 plane evaluation error <= ~4 * 2^-24 and the reference's float64
        // rounding <= ~4 * 2^-53 of |a|(|x|+|ax|) + |b|(|y|+|ay|); tol is >= 2x that
        const double mag = fabs(a) * (xmax + fabs(sx[ia])) + fabs(b) * (ymax + fabs(sy[ia]));
#if TRI80
        tol = fmax(tol, 4.8e-7 * mag + 1e-30);
#else
        o.tol[i] = (float)(4.8e-7 * mag + 1e-30);
#endif
        const double k = iw[i] * T.inv_area;  // l_i = w_i * inv_area, inv_w = sum l_i iw_i
        A += a * k;
        B += b * k;
        C += c * k;
        Aab += fabs(a * k);
        Bab += fabs(b * k);
        Cab += fabs(c * k);
    }
    o.A = (float)A;
    o.B = (float)B;
    o.C = (float)C;
    o.tolw = (float)(4.8e-7 * (Aab * xmax + Bab * ymax + Cab) + 1e-30);
    o.inv_minw = __double2float_ru(1.0 / (double)T.minw) * (1.0f + 1e-6f);
    o.ox = (float)T.x0;
    o.oy = (float)T.y0;
    o.wx = (float)(T.x1 - T.x0 + 1);
    o.wy = (float)(T.y1 - T.y0 + 1);
    o.gidx = gidx;
#if TRI80
    o.tol = (float)tol;  // rounded to nearest: the 2x margin of each edge's bound covers it
#else
    o.pad[0] = o.pad[1] = 0;
#endif
}

struct TriStore {
    GmScreenTri* tris;
    TriF32* t32;  // float32 form of tris (same index)
    uint2* bbox;
    int* count;
    int64_t cap_seg;
    long long* fail;     // first failed batch start, LLONG_MAX if none
    int* max_count;      // largest per-fixation count seen (for regrowth)
    unsigned long long* total;  // screen triangles produced (statistics)
};

// One warp per group of 32 triangle clusters (32 triangles each); blockIdx.y =
// fixation slot.  Lane-parallel cluster test -> ballot -> per passing cluster
// lane = triangle: sphere test, exact projection, warp-aggregated append.
#ifndef TS_WARPS
#define TS_WARPS 2  // warps (independent cluster groups) per k_tri_setup CTA
#endif
#ifndef TS_TOTAL_ATOMIC
#define TS_TOTAL_ATOMIC 0  // 1: k_tri_setup counts screen triangles with one global atomic per cluster
#endif                     // (0: k_coarse adds each fixation's count once -- no single-address hot spot)
#ifndef TS_MINB
#define TS_MINB 16  // k_tri_setup register budget: 16 CTAs/SM, 64 registers (uncapped 76: C2 cull
#endif              // 21.1 -> 19.2 ms, C5 222 -> 212.5 ms; 20 CTAs spill 172 B, C5 +2%)
#if TS_MINB > 0
#define TS_BOUNDS __launch_bounds__(TS_WARPS * 32, TS_MINB)
#else
#define TS_BOUNDS __launch_bounds__(TS_WARPS * 32)
#endif
#ifndef TS_VEC_STORE
#define TS_VEC_STORE 1  // TriF32 assembled in registers, 16-byte stores (C5 cull 352 -> 258 ms)
#endif
__global__ void TS_BOUNDS k_tri_setup(const double* __restrict__ tw, int64_t T,
                                                   const float4* __restrict__ tsph, const float4* __restrict__ csph,
                                                   int64_t n_clu, const GmFixExact* __restrict__ fixes,
                                                   const GmFixCull* __restrict__ culls, int W, int H, TriStore ts,
                                                   long long b0) {
    const int f = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t group = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t c0 = group * 32;
    if (c0 >= n_clu) return;
    const GmFixCull cull = culls[f];
    int64_t myc = c0 + lane;
    bool pass = myc < n_clu && sphere_visible(cull, csph[myc], true);
    unsigned mask = __ballot_sync(0xffffffffu, pass);
    if (!mask) return;
    const GmFixExact& F = fixes[f];
    GmScreenTri* seg = ts.tris + (int64_t)f * ts.cap_seg;
    uint2* segb = ts.bbox + (int64_t)f * ts.cap_seg;
    while (mask) {
        int j = __ffs(mask) - 1;
        mask &= mask - 1;
        int64_t t = (c0 + j) * 32 + lane;
        GmScreenTri out[2];
        int n = 0;
        if (t < T && sphere_visible(cull, tsph[t], true)) {
            n = project_triangle(tw + 9 * t, F, W, H, out);
            for (int q = 0; q < n; q++) out[q].tl += (uint32_t)(2 * t) << 3;
        }
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        int base = 0;
        if (lane == 31) {
#if TS_TOTAL_ATOMIC
            atomicAdd(ts.total, (unsigned long long)total);
#endif
            base = atomicAdd(ts.count + f, total);
            if (base + total > ts.cap_seg) {
                atomicMin(ts.fail, b0);
                atomicMax(ts.max_count, base + total);
            }
        }
        base = __shfl_sync(0xffffffffu, base, 31);
        int at = base + (incl - n);
        for (int q = 0; q < n; q++) {
            if (at + q < ts.cap_seg) {
                seg[at + q] = out[q];
#if TS_VEC_STORE
                {  // assemble the float32 form in registers, then six 16-byte stores
                    TriF32 tf;
                    make_tri_f32(out[q], at + q, tf);
                    uint4* dst = reinterpret_cast<uint4*>(&ts.t32[(int64_t)f * ts.cap_seg + at + q]);
                    const uint4* src = reinterpret_cast<const uint4*>(&tf);
#pragma unroll
                    for (int part = 0; part < TRI_WORDS; part++) dst[part] = src[part];
                }
#else
                make_tri_f32(out[q], at + q, ts.t32[(int64_t)f * ts.cap_seg + at + q]);
#endif
                segb[at + q] = make_uint2((uint32_t)out[q].x0 | ((uint32_t)out[q].x1 << 16),
                                          (uint32_t)out[q].y0 | ((uint32_t)out[q].y1 << 16));
            }
        }
    }
}

// Work counters filled when GmConfig.flags & GM_FLAG_STATS (bench roofline).
enum {
    GM_STAT_L1_TESTS = 0,    // super-chunk x fixation sphere tests (warp ballots x 32)
    GM_STAT_L2_TESTS = 1,    // chunk x fixation sphere tests
    GM_STAT_EXACT = 2,       // exact per-sample camera transform + NDC filter evaluations
    GM_STAT_NDC = 3,         // samples passing the NDC filter (the reference's filtered set)
    GM_STAT_CANDIDATES = 4,  // NDC and in the 4-sigma cone (depth test performed)
    GM_STAT_VISIBLE = 5,     // depth test passed (contributions added)
    GM_STAT_TEXELS = 6,      // marked texels evaluated
    GM_STAT_PAIRS = 7,       // (texel, screen triangle) exact evaluations
    GM_STAT_COVERED = 8,     // pairs where the triangle covers the texel
    GM_STAT_TILE_OCCLUDED = 9,  // depth tests decided by the tile-max occlusion pre-test (float64 depth)
    GM_STAT_TX_TILES = 10,   // k_texels work items with marked texels
    GM_STAT_TX_STAGED = 11,  // triangles staged per item (sum)
    GM_STAT_TX_LIST = 12,    // coarse-bin list entries scanned per item (sum)
    GM_STAT_TX_ITER = 13,    // warp iterations of the selection walk
    GM_STAT_TX_EDGE = 14,    // lane x triangle edge-function evaluations in the walk
    GM_STAT_TX_CROWDED = 15, // tiles deferred to the sorted crowded pass
    GM_STAT_TX_CHUNKED = 16, // tiles walked chunk by chunk (> TW_CAP staged triangles, no fast path)
    GM_STAT_TX_CHUNKED_PAIRS = 17,   // exact evaluations in those tiles
    GM_STAT_TX_CHUNKED_TEXELS = 18,  // marked texels in those tiles
    GM_STAT_BBOX_PX = 19,    // sum of the screen triangles' clamped pixel bboxes: the pixel tests the
                             // reference's _raster_tri loop performs (kernels.py:103-137)
    GM_STAT_N = 20
};
#define GM_FLAG_STATS 1
#define GM_FLAG_ONE_STREAM 2   // force batches onto one stream/buffer set
#define GM_FLAG_TWO_STREAMS 4  // force the two-stream batch pipeline
#ifndef GM_OVERLAP_MAX_TRIS
#define GM_OVERLAP_MAX_TRIS 400000  // default: overlap batches for scenes up to this many occluders
#endif
#define GM_STAT_STRIPES 128  // counter copies (summed by gm_plan_stats): keeps the stats pass free of atomic hot spots

// ------------------------------------------------------ the hot kernels

// Per-batch z-buffer store: only the texels some candidate's depth_match will
// read are ever written (mask bit set by k_samples<true>, value by k_texels).
// Coarse screen bins (cb x cb pixels, cb a power of two >= 64) of every
// fixation's screen triangles, so a k_texels tile scans only the triangles of
// its coarse bin.  One CTA per fixation slot: count per bin in shared memory,
// scan, fill.  Per-fixation CSR in citems[f * cap_items ...]; if the items do
// not fit, covf[f] = 1 and k_texels scans the fixation's whole list instead.
#define GM_MAX_CBINS 1024
#ifndef CB_SHIFT
#define CB_SHIFT 5  // coarse bins of 32 x 32 pixels (k_texels tiles are 32 x 16)
#endif
#ifndef CB_ITEMS_PER_TRI
#define CB_ITEMS_PER_TRI 8  // coarse-bin list capacity per screen triangle (more: scan the whole list)
#endif
struct CoarseBins {
    int4* items;  // [B][cap_items]: (segment index, bbox x0|x1<<16, bbox y0|y1<<16, float bits of inv_minw)
    int* off;     // [B][GM_MAX_CBINS + 1]
    int* ovf;     // [B]
    int64_t cap_items;
    int shift, ncx, ncy;
};

__global__ void __launch_bounds__(256) k_coarse(TriStore ts, CoarseBins cb, const long long* __restrict__ fail,
                                                long long b0, unsigned long long* __restrict__ bbox_px) {
    __shared__ int s_cnt[GM_MAX_CBINS];
    __shared__ int s_off[GM_MAX_CBINS + 1];
    if (*fail <= b0) return;
    const int f = blockIdx.x;
    const int nbins = cb.ncx * cb.ncy;
    const int n = min(ts.count[f], (int)ts.cap_seg);
#if !TS_TOTAL_ATOMIC
    if (threadIdx.x == 0 && ts.total) atomicAdd(ts.total, (unsigned long long)ts.count[f]);  // statistics
#endif
    const uint2* segb = ts.bbox + (int64_t)f * ts.cap_seg;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    unsigned long long px_sum = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint2 bb = segb[i];
        const int bx0 = (bb.x & 0xffff) >> cb.shift, bx1 = (bb.x >> 16) >> cb.shift;
        const int by0 = (bb.y & 0xffff) >> cb.shift, by1 = (bb.y >> 16) >> cb.shift;
        for (int by = by0; by <= by1; by++)
            for (int bx = bx0; bx <= bx1; bx++) atomicAdd(&s_cnt[by * cb.ncx + bx], 1);
        if (bbox_px)
            px_sum += (unsigned long long)((bb.x >> 16) - (bb.x & 0xffff) + 1) * ((bb.y >> 16) - (bb.y & 0xffff) + 1);
    }
    if (bbox_px) {  // statistics pass only
        for (int o = 16; o; o >>= 1) px_sum += __shfl_xor_sync(0xffffffffu, px_sum, o);
        if ((threadIdx.x & 31) == 0 && px_sum) atomicAdd(bbox_px + (size_t)(blockIdx.x % GM_STAT_STRIPES) * GM_STAT_N + GM_STAT_BBOX_PX, px_sum);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp scan over <= 1024 bins
        const int lane = threadIdx.x;
        int carry = 0;
        for (int b0s = 0; b0s < nbins; b0s += 32) {
            const int b = b0s + lane;
            const int v = b < nbins ? s_cnt[b] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (b < nbins) s_off[b] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_off[nbins] = carry;
    }
    __syncthreads();
    const int total = s_off[nbins];
    int* off = cb.off + (int64_t)f * (GM_MAX_CBINS + 1);
    for (int b = threadIdx.x; b <= nbins; b += blockDim.x) off[b] = s_off[b];
    if (total > cb.cap_items) {
        if (threadIdx.x == 0) cb.ovf[f] = 1;
        return;
    }
    if (threadIdx.x == 0) cb.ovf[f] = 0;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    int4* items = cb.items + (int64_t)f * cb.cap_items;
    const TriF32* segf = ts.t32 + (int64_t)f * ts.cap_seg;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint2 bb = segb[i];
        // the entry carries what k_texels' gather and sort read, so neither chases the index
        const int4 e = make_int4(i, (int)bb.x, (int)bb.y, __float_as_int(segf[i].inv_minw));
        const int bx0 = (bb.x & 0xffff) >> cb.shift, bx1 = (bb.x >> 16) >> cb.shift;
        const int by0 = (bb.y & 0xffff) >> cb.shift, by1 = (bb.y >> 16) >> cb.shift;
        for (int by = by0; by <= by1; by++)
            for (int bx = bx0; bx <= bx1; bx++) {
                const int b = by * cb.ncx + bx;
                items[s_off[b] + atomicAdd(&s_cnt[b], 1)] = e;
            }
    }
}

#define TW 32      // k_texels tile width (pixels) = warp lanes
// k_texels tile heights (pixels, powers of two <= 32): 32 x 32 tiles (the coarse-bin size) in
// crop-frustum generation batches -- their marked texels are dense around the cone, so twice the
// texels share a tile's fixed cost (C2 step 239 -> 228 ms, C5 texels 666 -> 603 ms); 32 x 16 in
// full-frustum batches (few marked texels, long lists: 32-row tiles double unfiltered C2's texels
// phase) and for the raster API / renderer
#ifndef TH_CROP
#define TH_CROP 32
#endif
#ifndef TH_FULL
#define TH_FULL 16
#endif

struct DepthView {
    double* depth;    // [B][H][W]: marked texels only
    uint32_t* mask;   // [B][H][wwords]: texels the depth tests will read
    int W, H, wwords;
    unsigned long long* stats;  // optional work counters (GM_STAT_*), nullptr = off
    float* vbuf;      // [B][H][W] crowded pass, lists longer than one pass: inverse-depth bounds between passes
    int* key;         // [H][W] (ATTRS only): order key 2 t + fan of the triangle that wrote the texel
    int* win;         // [B][H][W] (generation batches): segment index of the texel's writer, -1 none
    double* carry;    // [B][H][W] ... and exact best depths (generation batches)
    int* crowd;       // work items deferred to k_texels<CROWDED> (nullptr: handle them in place)
    int* crowd_count; // [2]: deferred items, claimed items
    float* tmax;      // [B][tiles] (generation batches): largest finite depth upper bound of the
                      // tile's marked texels, -inf if none (k_texels; tiles without marked
                      // texels are not written); nullptr = off
    int tiles_x, tiles_per_fix;
    int crowd_wide;   // crowded pass with HV_FULL_WARPS-warp CTAs (full-frustum z-buffers), else HV_CROP_WARPS
    int th_shift;     // log2 of the k_texels tile height of this batch (4: 32 x 16 tiles, 5: 32 x 32)
    unsigned long long* check;  // GM_CHECK builds: violation counters (GM_CHK_*), nullptr = off
};

// Self-check counters of a GM_CHECK build (gm_plan_check).  Each "wrong"
// counter is a decision the production kernels took on float32 bounds or
// conservative culls that the exact float64 reference arithmetic contradicts;
// the others count how many decisions were checked.
enum {
    GM_CHK_TX_TEXELS = 0,        // texels checked (k_texels stores)
    GM_CHK_TX_BOUND_WRONG = 1,   // fast-path [lo, hi] does not contain the exact depth of the writer
    GM_CHK_TX_WINNER_WRONG = 2,  // stored depth / writer's depth != brute-force min over the tile's coarse list
    GM_CHK_CAND_PAIRS = 3,       // exact (sample, fixation) candidates checked (all pairs of the batch)
    GM_CHK_CAND_L1_WRONG = 4,    // exact candidate whose super-chunk level-1 ballot misses the fixation
    GM_CHK_CAND_L3_WRONG = 5,    // exact candidate missing from k_mark's per-chunk fixation word
    GM_CHK_MASK_WRONG = 6,       // texel of an exact candidate's 3x3 depth_match block left unmarked
    GM_CHK_DEPTH_TESTS = 7,      // depth tests checked in k_samples
    GM_CHK_DEPTH_WRONG = 8,      // depth_test_iv (bounds) != the reference test on exact texel depths
    GM_CHK_TILEOCC_WRONG = 9,    // tile-max occlusion said "occluded" but the exact test passes
    GM_CHK_CULL_TRIS = 10,       // occluder triangles the cone cull dropped, projected exactly anyway
    GM_CHK_CULL_TEXELS = 11,     // marked texels inside those triangles' pixel bboxes, tested
    GM_CHK_CULL_WRONG = 12,      // ... where a dropped triangle is nearer than the stored texel (it would have won)
    GM_CHK_N = 16
};
__device__ __forceinline__ void chk_add(unsigned long long* c, int idx, unsigned long long v) {
    if (v) atomicAdd(c + idx, v);
}


// Warp-aggregated add of a per-lane count to stripe (block % GM_STAT_STRIPES)
// of counter idx.  Every lane of the warp must call it.
__device__ __forceinline__ void stat_add(unsigned long long* stats, int idx, unsigned long long v) {
    const unsigned lo = __reduce_add_sync(0xffffffffu, (unsigned)(v & 0xffffffffu));
    const unsigned hi = __reduce_add_sync(0xffffffffu, (unsigned)(v >> 32));
    if ((threadIdx.x & 31) == 0)
        atomicAdd(stats + (size_t)(blockIdx.x % GM_STAT_STRIPES) * GM_STAT_N + idx,
                  (unsigned long long)lo + ((unsigned long long)hi << 32));
}

// depth_match on a generation batch's texel store: every texel holds rigorous
// float32 bounds [lo, hi] of the float64 depth kernels.rasterize leaves there
// ((+inf, +inf) where nothing is written) and the segment index of its writer.
// Each stage of kernels.py:219-285 is decided on the bounds when they decide it
// (the comparisons use a slack that covers the reference's and this code's own
// float64 rounding); otherwise the exact depths of the texels the test reads
// are re-evaluated from their writers (texel_depth) and the reference test runs
// on them.  Either way the result is the reference's.
__device__ __forceinline__ bool depth_test_exact(const DepthView& dv, const GmScreenTri* __restrict__ seg, double near_,
                                              double far_, int f, double gx, double gy, int bx0, int bx1, int by0,
                                              int by1, double d, double eps) {
    const int W = dv.W, H = dv.H;
    const int* win = dv.win + (int64_t)f * W * H;
    auto val = [&](int x, int y) -> double {
        const int w = win[(int64_t)y * W + x];
        return w < 0 ? CUDART_INF : texel_depth(seg[w], x, y, near_, far_);
    };
    if (W > 1 && H > 1) {
        long long x0 = x86_i64(floor(gx));
        if (x0 < 0) x0 = 0;
        else if (x0 > W - 2) x0 = W - 2;
        long long y0 = x86_i64(floor(gy));
        if (y0 < 0) y0 = 0;
        else if (y0 > H - 2) y0 = H - 2;
        const double q00 = val((int)x0, (int)y0), q01 = val((int)x0 + 1, (int)y0);
        const double q10 = val((int)x0, (int)y0 + 1), q11 = val((int)x0 + 1, (int)y0 + 1);
        if (isfinite(q00) && isfinite(q01) && isfinite(q10) && isfinite(q11)) {
            double tx = gx - (double)x0;
            if (tx < 0.0) tx = 0.0;
            else if (tx > 1.0) tx = 1.0;
            double ty = gy - (double)y0;
            if (ty < 0.0) ty = 0.0;
            else if (ty > 1.0) ty = 1.0;
            double top = q00 * (1.0 - tx) + q01 * tx;
            double bot = q10 * (1.0 - tx) + q11 * tx;
            if (fabs(d - (top * (1.0 - ty) + bot * ty)) <= eps) return true;
            double hi = fmax(fmax(q00, q01), fmax(q10, q11));
            double lo = fmin(fmin(q00, q01), fmin(q10, q11));
            if (hi - lo <= eps) return false;
        }
    }
    double best = CUDART_INF;
    for (int yy = by0; yy <= by1; yy++)
        for (int xx = bx0; xx <= bx1; xx++) {
            const double t = val(xx, yy);
            if (isfinite(t)) {
                double diff = fabs(t - d);
                if (diff < best) best = diff;
            }
        }
    return best <= eps;
}

__device__ __forceinline__ bool depth_test_iv(const DepthView& dv, const GmScreenTri* __restrict__ seg, double near_,
                                              double far_, int f, double gx, double gy, int bx0, int bx1, int by0,
                                              int by1, double d, double eps) {
    const int W = dv.W, H = dv.H;
    const float2* q2 = reinterpret_cast<const float2*>(dv.depth) + (int64_t)f * W * H;
    const double slack = 1e-13 * (fabs(d) + eps);
    if (W > 1 && H > 1) {
        long long x0 = x86_i64(floor(gx));
        if (x0 < 0) x0 = 0;
        else if (x0 > W - 2) x0 = W - 2;
        long long y0 = x86_i64(floor(gy));
        if (y0 < 0) y0 = 0;
        else if (y0 > H - 2) y0 = H - 2;
        const float2* r0 = q2 + (int64_t)y0 * W + x0;
        const float2 a = r0[0], b = r0[1], c = r0[W], e = r0[W + 1];
        if (a.x < CUDART_INF_F && b.x < CUDART_INF_F && c.x < CUDART_INF_F && e.x < CUDART_INF_F) {
            double tx = gx - (double)x0;
            if (tx < 0.0) tx = 0.0;
            else if (tx > 1.0) tx = 1.0;
            double ty = gy - (double)y0;
            if (ty < 0.0) ty = 0.0;
            else if (ty > 1.0) ty = 1.0;
            // the weights are >= 0: the bilinear value is monotone in every texel
            const double blo = ((double)a.x * (1.0 - tx) + (double)b.x * tx) * (1.0 - ty) +
                               ((double)c.x * (1.0 - tx) + (double)e.x * tx) * ty;
            const double bhi = ((double)a.y * (1.0 - tx) + (double)b.y * tx) * (1.0 - ty) +
                               ((double)c.y * (1.0 - tx) + (double)e.y * tx) * ty;
            const double sl = slack + 1e-13 * fabs(bhi);
            if (fmax(fabs(d - blo), fabs(d - bhi)) + sl <= eps) return true;       // certain match
            if (!(fmax(fmax(d - bhi, blo - d), 0.0) - sl > eps))                     // undecided
                return depth_test_exact(dv, seg, near_, far_, f, gx, gy, bx0, bx1, by0, by1, d, eps);
            const double smax = (double)fmaxf(fmaxf(a.y, b.y), fmaxf(c.y, e.y)) -
                                (double)fminf(fminf(a.x, b.x), fminf(c.x, e.x));
            const double smin = (double)fmaxf(fmaxf(a.x, b.x), fmaxf(c.x, e.x)) -
                                (double)fminf(fminf(a.y, b.y), fminf(c.y, e.y));
            if (smax + sl <= eps) return false;                                      // smooth quad
            if (!(smin - sl > eps))                                                  // undecided
                return depth_test_exact(dv, seg, near_, far_, f, gx, gy, bx0, bx1, by0, by1, d, eps);
        }
    }
    bool all_far = true;
    for (int yy = by0; yy <= by1; yy++) {
        const float2* row = q2 + (int64_t)yy * W;
        for (int xx = bx0; xx <= bx1; xx++) {
            const float2 v = row[xx];
            if (v.x < CUDART_INF_F) {
                const double lo = v.x, hi = v.y;
                const double sl = slack + 1e-13 * hi;
                if (fmax(fabs(lo - d), fabs(hi - d)) + sl <= eps) return true;
                if (!(fmax(fmax(lo - d, d - hi), 0.0) - sl > eps)) all_far = false;
            }
        }
    }
    if (all_far) return false;
    return depth_test_exact(dv, seg, near_, far_, f, gx, gy, bx0, bx1, by0, by1, d, eps);
}

// Occlusion pre-test of depth_match (kernels.py:219-285): every texel the test
// can read lies in the 3x3 block (the bilinear quad is inside it), and the test
// can only succeed on a finite texel t with |t - d| <= eps.  If d - eps exceeds
// the largest finite depth bound of every k_texels tile the block touches,
// no such texel exists and the reference returns False (the relative slack
// covers its float64 rounding of the bilinear blend and of |t - d|).
__device__ __forceinline__ bool occluded_by_tiles(const DepthView& dv, int f, int bx0, int bx1, int by0, int by1,
                                                  double d, double eps) {
    const float* tm = dv.tmax + (int64_t)f * dv.tiles_per_fix;
    const int tx0 = bx0 / TW, tx1 = bx1 / TW, ty0 = by0 >> dv.th_shift, ty1 = by1 >> dv.th_shift;
    float m = tm[ty0 * dv.tiles_x + tx0];
    if (tx1 != tx0) m = fmaxf(m, tm[ty0 * dv.tiles_x + tx1]);
    if (ty1 != ty0) {
        m = fmaxf(m, tm[ty1 * dv.tiles_x + tx0]);
        if (tx1 != tx0) m = fmaxf(m, tm[ty1 * dv.tiles_x + tx1]);
    }
    if (!(m > -CUDART_INF_F)) return true;  // no finite texel at all: best stays +inf
    const double mm = (double)m;
    return (d - mm) - eps > 1e-12 * (fabs(d) + eps + mm);
}

#ifdef GM_CHECK
// Self-check of the occluder cone cull (GM_CHECK builds): every triangle
// k_tri_setup dropped (cluster or triangle sphere test) is projected exactly
// anyway; at each marked texel inside its pixel bbox its exact depth must not be
// nearer than the depth k_texels stored there (else the cull changed a texel a
// depth test reads).  Runs after k_texels, before k_samples.
__global__ void __launch_bounds__(TS_WARPS * 32) k_check_cull(const double* __restrict__ tw, int64_t T,
                                                    const float4* __restrict__ tsph, const float4* __restrict__ csph,
                                                    int64_t n_clu, const GmFixExact* __restrict__ fixes,
                                                    const GmFixCull* __restrict__ culls, int W, int H, TriStore ts,
                                                    DepthView dv, long long b0) {
    if (*ts.fail <= b0) return;
    const int f = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t c0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
    if (c0 >= n_clu) return;
    const GmFixCull cull = culls[f];
    const GmFixExact& F = fixes[f];
    const GmScreenTri* seg = ts.tris + (int64_t)f * ts.cap_seg;
    const uint32_t* mask = dv.mask + (int64_t)f * H * dv.wwords;
    const int* win = dv.win + (int64_t)f * W * H;
    unsigned long long n_tri = 0, n_tex = 0, n_bad = 0;
    for (int c = 0; c < 32; c++) {
        const int64_t clu = c0 + c;
        if (clu >= n_clu) break;
        const bool clu_pass = sphere_visible(cull, csph[clu], true);
        const int64_t t = clu * 32 + lane;
        if (t >= T || (clu_pass && sphere_visible(cull, tsph[t], true))) continue;  // kept by the cull
        GmScreenTri out[2];
        const int n = project_triangle(tw + 9 * t, F, W, H, out);
        n_tri++;
        for (int q = 0; q < n; q++) {
            const GmScreenTri& S = out[q];
            for (int y = S.y0; y <= S.y1; y++)
                for (int w0 = S.x0 >> 5; w0 <= (S.x1 >> 5); w0++) {
                    uint32_t bits = mask[(int64_t)y * dv.wwords + w0];
                    while (bits) {
                        const int x = w0 * 32 + __ffs(bits) - 1;
                        bits &= bits - 1;
                        if (x < S.x0 || x > S.x1) continue;
                        const double d = texel_depth(S, x, y, F.near_, F.far_);
                        if (!(d < CUDART_INF)) continue;
                        n_tex++;
                        const int wr = win[(int64_t)y * W + x];
                        const double stored = wr >= 0 ? texel_depth(seg[wr], x, y, F.near_, F.far_) : CUDART_INF;
                        if (d < stored) n_bad++;
                    }
                }
        }
    }
    chk_add(dv.check, GM_CHK_CULL_TRIS, n_tri);
    chk_add(dv.check, GM_CHK_CULL_TEXELS, n_tex);
    chk_add(dv.check, GM_CHK_CULL_WRONG, n_bad);
}
#endif

#include "gm_samples.cuh"

#include "gm_texels.cuh"

// Mark every texel of fixation slot 0 (the kernel-seam full z-buffer port).
__global__ void k_mark_all(uint32_t* __restrict__ mask, int W, int H, int wwords) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= (int64_t)H * wwords) return;
    int w = (int)(q % wwords);
    int bits = min(32, W - 32 * w);
    mask[q] = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
}

// Filter-only seam (kernels.py:302-319): per fixation, the compacted list of
// samples passing the NDC crop filter (warp ballot + popc compaction).
__global__ void k_candidates(const double* __restrict__ px, const double* __restrict__ py,
                             const double* __restrict__ pz, int64_t N, const GmFixExact* __restrict__ fixes,
                             int B, int64_t* __restrict__ out, int64_t cap_per_fix,
                             unsigned long long* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int f = blockIdx.y;
    const GmFixExact& F = fixes[f];
    const double lo = -1.0 - GM_NDC_SLACK, hi = 1.0 + GM_NDC_SLACK;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch * 32 < N; ch += warps) {
        int64_t i = ch * 32 + lane;
        bool c = false;
        if (i < N) {
            double wx = px[i], wy = py[i], wz = pz[i];
            double x = F.rot[0] * wx + F.rot[1] * wy + F.rot[2] * wz + F.trans[0];
            double y = F.rot[3] * wx + F.rot[4] * wy + F.rot[5] * wz + F.trans[1];
            double z = F.rot[6] * wx + F.rot[7] * wy + F.rot[8] * wz + F.trans[2];
            double w = -z;
            if (w > 0.0 && !(w < F.near_lo || w > F.far_hi)) {
                double ndc_x = (F.p00 * x + F.p02 * z) / w;
                double ndc_y = (F.p11 * y + F.p12 * z) / w;
                c = !(ndc_x < lo || ndc_x > hi) && !(ndc_y < lo || ndc_y > hi);
            }
        }
        unsigned m = __ballot_sync(0xffffffffu, c);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(counts + f, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (c) {
            unsigned long long at = base + __popc(m & ((1u << lane) - 1u));
            if (at < (unsigned long long)cap_per_fix) out[(int64_t)f * cap_per_fix + at] = i;
        }
    }
}

// density.py:192 / 230-244: global max (non-negative doubles order like their
// bit patterns) and normalisation.
__global__ void k_max(const double* __restrict__ v, int64_t n, unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, v[i]);
    typedef cub::BlockReduce<double, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    double bm = BR(tmp).Reduce(m, cub::Max());
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(bm));
}

__global__ void k_normalize(const double* __restrict__ v, int64_t n, double gmax, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v[i] / gmax;
}

// ------------------------------------------------------------ the plan

template <typename T>
static int dev_alloc(T** p, size_t n) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (n == 0) n = 1;
    CK(cudaMalloc((void**)p, n * sizeof(T)));
    return GM_OK;
}

#define GM_RING 3  // pinned host setup slots in flight
#ifndef GM_NSETS
#define GM_NSETS 3  // batch-buffer sets / streams in the overlapped batch pipeline
#endif

// Everything one batch of fixations owns on the device.  A plan holds GM_NSETS
// sets (the plan's own fields and `alt[]`); consecutive batches rotate over them
// and over as many streams, so batch i + 1's occluder setup, marking and texel
// kernels overlap batch i's tail.  Only the accumulation pass (k_samples) is
// chained across batches (event), which keeps the per-sample log order.
#define GM_BATCH_FIELDS(X)                                                                            \
    X(cudaStream_t, stream) X(uint32_t*, d_lvl1) X(uint32_t*, d_cbits) X(int64_t, cap_cbits)           \
    X(int*, d_lcount) X(int*, d_lorder) X(int*, d_lcount2) X(int*, d_lorder2) X(int64_t, cap_sort)     \
    X(int*, d_work) X(void*, d_sort_tmp) X(size_t, sort_tmp_bytes) X(int64_t, cap_lvl1) X(int, cap_B)  \
    X(GmFixExact*, d_fix) X(GmFixCull*, d_cull) X(GmFixF32*, d_fix32) X(GmScreenTri*, d_tris)          \
    X(TriF32*, d_t32) X(uint2*, d_bbox) X(int*, d_count) X(int64_t, cap_seg) X(int64_t, cap_seg_B)     \
    X(double*, d_depth) X(float*, d_vbuf) X(uint32_t*, d_mask) X(int64_t, cap_depth) X(int64_t, cap_mask) \
    X(int*, d_win) X(double*, d_carry)                                                                 \
    X(int4*, d_citems) X(int*, d_coff) X(int*, d_covf) X(int64_t, cap_citems) X(int64_t, cap_cB)         \
    X(int*, d_crowd) X(int*, d_crowd_count) X(int64_t, cap_crowd) X(float*, d_tmax)

struct BatchBufs {
#define GM_X(T, n) T n{};
    GM_BATCH_FIELDS(GM_X)
#undef GM_X
};

struct gm_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sms = 148;
    // scene (occluders: every object; samples: included objects)
    int64_t T = 0, n_clu = 0, N = 0, n_chunks = 0;
    double* d_tw = nullptr;
    float4* d_tsph = nullptr;
    float4* d_csph = nullptr;
    double *d_px = nullptr, *d_py = nullptr, *d_pz = nullptr;
    float *d_pxf = nullptr, *d_pyf = nullptr, *d_pzf = nullptr;  // float32 copies (marking pass)
    double pmax = 0.0;                                           // max |coordinate| of the samples
    float4* d_chunk = nullptr;
    float4* d_super = nullptr;  // sphere per 8 chunks (256 samples)
    int64_t n_supers = 0;
    uint32_t* d_lvl1 = nullptr;  // [n_supers][B/32] level-1 ballots of the current batch
    uint32_t* d_cbits = nullptr; // [n_chunks][32] k_mark's per-chunk candidate fixations (bit j of group g)
    int *d_lcount = nullptr, *d_lorder = nullptr, *d_lcount2 = nullptr, *d_lorder2 = nullptr;
    int* d_work = nullptr;       // [2] work counters of the two sample passes
    void* d_sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int64_t cap_lvl1 = 0;
    double* d_values = nullptr;
    // batch buffers: per-fixation setup (device + pinned host ring)
    int cap_B = 0;
    GmFixExact* d_fix = nullptr;
    GmFixCull* d_cull = nullptr;
    GmFixF32* d_fix32 = nullptr;  // [cap_B] float32 views of the current batch
    GmFixExact* h_fix[GM_RING] = {};
    GmFixCull* h_cull[GM_RING] = {};
    cudaEvent_t h_ev[GM_RING] = {};
    // per-fixation screen-triangle segments
    GmScreenTri* d_tris = nullptr;
    TriF32* d_t32 = nullptr;
    uint2* d_bbox = nullptr;
    int* d_count = nullptr;
    int64_t cap_seg = 0, cap_seg_B = 0;
    int64_t seg_init = 16384;  // first per-fixation screen-triangle capacity, grown on overflow
                               // (gm_plan_set_segment_capacity); C2 peaks above 4k, C5 grows it once
    long long* d_fail = nullptr;
    int* d_maxcount = nullptr;
    unsigned long long* d_ntris = nullptr;
    // marked z-buffer texels
    double* d_depth = nullptr;   // [B][H][W] marked texels only
    float* d_vbuf = nullptr;     // [B][H][W] k_texels_crowded state between passes
    int* d_win = nullptr;        // [B][H][W] writer of each marked texel (generation batches)
    double* d_carry = nullptr;   // [B][H][W] (generation batches)
    uint32_t* d_mask = nullptr;  // [B][H][wwords]
    int64_t cap_depth = 0, cap_mask = 0;
    int4* d_citems = nullptr;  // coarse bins: [B][cap_citems]
    int* d_coff = nullptr;    // [B][GM_MAX_CBINS + 1]
    int* d_covf = nullptr;    // [B]
    int64_t cap_citems = 0, cap_cB = 0;
    unsigned long long* d_max = nullptr;
    unsigned long long* d_stats = nullptr;  // GM_STAT_N counters
    unsigned long long* d_check = nullptr;  // GM_CHK_N self-check counters (GM_CHECK builds)
    // peer accumulators of the other ranks (CUDA IPC over NVLink), gm_plan_open_peers
    int peer_rank = 0, peer_world = 0;
    std::vector<cudaIpcMemHandle_t> peer_handle;
    std::vector<double*> peer_ptr;  // [world]; own entry = d_values, others IPC-mapped
    double** d_peer_ptr = nullptr;
    int host_threads = 8;
    // device-resident setup table (gm_plan_prepare)
    GmFixExact* d_fix_all = nullptr;
    GmFixCull* d_cull_all = nullptr;
    int64_t F_prepared = -1;
    GmConfig cfg_prepared{};
    void* d_flush = nullptr;
    int64_t flush_bytes = 0;
    int flush_gen = 0;
    void* d_scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0;
    // scene layout kept for pose changes (gm_plan_set_poses): local corners,
    // sample offsets per triangle, per-object triangle/sample ranges
    double* d_local = nullptr;
    int64_t* d_res = nullptr;
    int64_t* d_off = nullptr;
    double* d_M = nullptr;  // [n_obj][12] current R diag(s) + t
    int n_obj = 0;
    std::vector<int64_t> tstart, nsamp;
    std::vector<uint8_t> include;
    int* d_key = nullptr;  // [H][W] raster_pass(attrs): order key of the winning triangle
    int* d_crowd = nullptr;        // [B * tiles] k_texels items deferred to the crowded pass
    int* d_crowd_count = nullptr;  // [2]
    int64_t cap_crowd = 0;
    float* d_tmax = nullptr;       // [B * tiles] largest finite texel depth bound of each k_texels tile
    int64_t cap_key = 0;
    int64_t cap_cbits = 0, cap_sort = 0;  // (per batch-buffer set, swapped with alt[])
    int cap_ring = 0;
    BatchBufs alt[GM_NSETS - 1];     // the other batch-buffer sets (and streams)
    cudaEvent_t ev_order = nullptr;  // last accumulation pass enqueued (chains k_samples across streams)
    char* h_stage = nullptr;             // pinned read-back staging, 2 x GM_STAGE bytes (gm_plan_read)
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
};

// Exchange the plan's batch buffers (and stream) with the alternate set.
static void swap_batch_bufs(gm_plan* p, int k = 1) {
#define GM_X(T, n) std::swap(p->n, p->alt[k - 1].n);
    GM_BATCH_FIELDS(GM_X)
#undef GM_X
}

// Free one set's scene-sized batch buffers (sizes depend on n_supers / n_chunks).
static void free_scene_batch_bufs(gm_plan* p) {
    cudaFree(p->d_lvl1); cudaFree(p->d_cbits); cudaFree(p->d_lcount); cudaFree(p->d_lorder);
    cudaFree(p->d_lcount2); cudaFree(p->d_lorder2); cudaFree(p->d_sort_tmp);
    p->d_lvl1 = nullptr; p->d_cbits = nullptr; p->d_lcount = p->d_lorder = p->d_lcount2 = p->d_lorder2 = nullptr;
    p->d_sort_tmp = nullptr; p->sort_tmp_bytes = 0; p->cap_lvl1 = 0; p->cap_cbits = 0; p->cap_sort = 0;
}

static void plan_free_scene(gm_plan* p) {
    cudaFree(p->d_tw); cudaFree(p->d_tsph); cudaFree(p->d_csph);
    cudaFree(p->d_px); cudaFree(p->d_py); cudaFree(p->d_pz);
    cudaFree(p->d_pxf); cudaFree(p->d_pyf); cudaFree(p->d_pzf);
    p->d_pxf = p->d_pyf = p->d_pzf = nullptr;
    cudaFree(p->d_chunk); cudaFree(p->d_values); cudaFree(p->d_super);
    free_scene_batch_bufs(p);
    for (int k = 1; k < GM_NSETS; k++) {
        swap_batch_bufs(p, k);
        free_scene_batch_bufs(p);
        swap_batch_bufs(p, k);
    }
    p->d_tw = nullptr; p->d_tsph = p->d_csph = p->d_chunk = p->d_super = nullptr;
    p->d_px = p->d_py = p->d_pz = p->d_values = nullptr;
    p->T = p->n_clu = p->N = p->n_chunks = p->n_supers = 0;
    cudaFree(p->d_local); cudaFree(p->d_res); cudaFree(p->d_off); cudaFree(p->d_M);
    p->d_local = nullptr; p->d_res = p->d_off = nullptr; p->d_M = nullptr;
    p->n_obj = 0;
    p->tstart.clear(); p->nsamp.clear(); p->include.clear();
}

extern "C" void gm_plan_destroy(gm_plan* p);
static int plan_init(gm_plan* p);

extern "C" int gm_plan_create(int device, gm_plan** out) {
    if (!out) return set_err(GM_ERR_ARG, "null out");
    int rc = use_device(device);
    if (rc) return rc;
    gm_plan* p = new gm_plan();
    p->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete p;
        return set_err(GM_ERR_CUDA, cudaGetErrorString(e));
    }
    cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
    rc = plan_init(p);
    if (rc) {
        gm_plan_destroy(p);  // frees whatever plan_init allocated
        return rc;
    }
    *out = p;
    return GM_OK;
}

// Kernel attributes and the plan's fixed device buffers (gm_plan_create).
static int plan_init(gm_plan* p) {
    CK(cudaFuncSetAttribute(k_texels<false, false, false, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, false, false, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, false, false, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<false, false, false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, false, false, HV_CROP_WARPS, HV_CROP_SEL, 32>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, false, false, HV_FULL_WARPS, HV_FULL_SEL, 32>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<false, false, true, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, false, true, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, false, true, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<false, true, false, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, true, false, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, true, false, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<false, true, false, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, true, false, HV_CROP_WARPS, HV_CROP_SEL, 32>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, true, false, HV_FULL_WARPS, HV_FULL_SEL, 32>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<false, true, true, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, true, true, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<false, true, true, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<true, false, false, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, false, false, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, false, false, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<true, false, true, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, false, true, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, false, true, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<true, true, false, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, true, false, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, true, false, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaFuncSetAttribute(k_texels<true, true, true, TH_FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, true, true, HV_CROP_WARPS, HV_CROP_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>)));
    CK(cudaFuncSetAttribute(k_texels_crowded<true, true, true, HV_FULL_WARPS, HV_FULL_SEL, TH_FULL>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>)));
    CK(cudaMalloc(&p->d_max, sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_stats, GM_STAT_STRIPES * GM_STAT_N * sizeof(unsigned long long)));
    CK(cudaMemset(p->d_stats, 0, GM_STAT_STRIPES * GM_STAT_N * sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_check, GM_CHK_N * sizeof(unsigned long long)));
    CK(cudaMemset(p->d_check, 0, GM_CHK_N * sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_fail, sizeof(long long)));
    CK(cudaMalloc(&p->d_maxcount, sizeof(int)));
    CK(cudaMalloc(&p->d_ntris, sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_work, 2 * sizeof(int)));
    CK(cudaEventCreateWithFlags(&p->ev_order, cudaEventDisableTiming));
    for (int r = 0; r < GM_RING; r++) CK(cudaEventCreateWithFlags(&p->h_ev[r], cudaEventDisableTiming));
    unsigned hc = std::thread::hardware_concurrency();
    p->host_threads = hc > 0 ? (int)hc : 8;
    return GM_OK;
}

// Free one batch-buffer set (the plan's own fields) and its stream.
static void free_batch_set(gm_plan* p) {
    if (p->stream) cudaStreamSynchronize(p->stream);
    free_scene_batch_bufs(p);
    cudaFree(p->d_fix); cudaFree(p->d_cull); cudaFree(p->d_fix32); cudaFree(p->d_work);
    cudaFree(p->d_tris); cudaFree(p->d_t32); cudaFree(p->d_bbox); cudaFree(p->d_count);
    cudaFree(p->d_depth); cudaFree(p->d_mask); cudaFree(p->d_vbuf); cudaFree(p->d_win); cudaFree(p->d_carry);
    cudaFree(p->d_citems); cudaFree(p->d_coff); cudaFree(p->d_covf);
    cudaFree(p->d_crowd); cudaFree(p->d_crowd_count); cudaFree(p->d_tmax);
    if (p->stream) cudaStreamDestroy(p->stream);
    p->stream = nullptr;
}

extern "C" void gm_plan_destroy(gm_plan* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    for (int k = 0; k < GM_NSETS - 1; k++)
        if (p->alt[k].stream) cudaStreamSynchronize(p->alt[k].stream);
    plan_free_scene(p);
    for (int r = 0; r < GM_RING; r++) {
        cudaFreeHost(p->h_fix[r]); cudaFreeHost(p->h_cull[r]); cudaEventDestroy(p->h_ev[r]);
    }
    cudaFreeHost(p->h_stage);
    for (int k = 0; k < 2; k++)
        if (p->stage_ev[k]) cudaEventDestroy(p->stage_ev[k]);
    cudaFree(p->d_fail); cudaFree(p->d_maxcount); cudaFree(p->d_ntris);
    for (int r = 0; r < p->peer_world; r++)
        if (r != p->peer_rank && p->peer_ptr[r]) cudaIpcCloseMemHandle(p->peer_ptr[r]);
    cudaFree(p->d_peer_ptr);
    cudaFree(p->d_scan_tmp); cudaFree(p->d_max); cudaFree(p->d_stats); cudaFree(p->d_check);
    cudaFree(p->d_fix_all); cudaFree(p->d_cull_all); cudaFree(p->d_flush);
    cudaFree(p->d_key);
    if (p->ev_order) cudaEventDestroy(p->ev_order);
    free_batch_set(p);
    for (int k = 1; k < GM_NSETS; k++) {
        swap_batch_bufs(p, k);
        free_batch_set(p);
    }
    delete p;
}

extern "C" int gm_plan_set_host_threads(gm_plan* p, int n) {
    if (!p || n < 1) return set_err(GM_ERR_ARG, "bad thread count");
    p->host_threads = n;
    return GM_OK;
}

static inline unsigned blocks_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// Object transform in the layout [t(3), q(4) xyzw, s(3)] -> M = R diag(s).
static void xform_matrix(const double* xf, double M[9], double t[3]) {
    double x = xf[3], y = xf[4], z = xf[5], w = xf[6];
    double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - z * w), 2.0 * (x * z + y * w),
                   2.0 * (x * y + z * w), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - x * w),
                   2.0 * (x * z - y * w), 2.0 * (y * z + x * w), 1.0 - 2.0 * (x * x + y * y)};
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[3 * i + j] = R[3 * i + j] * xf[7 + j];
    for (int i = 0; i < 3; i++) t[i] = xf[i];
}

extern "C" int gm_plan_set_poses(gm_plan* p, const double* xforms);

// Upload a scene: n_obj objects, tri_counts[o] triangles each, local triangle
// corners tri_local (sum T x 9, object order), transforms xforms (n_obj x 10),
// per-triangle resolutions res (sum T; the SampledMesh layouts), include flags.
// Occluders = all objects; samples = included objects, concatenated.
extern "C" int gm_plan_set_scene(gm_plan* p, int n_obj, const int64_t* tri_counts, const double* tri_local,
                                 const double* xforms, const int64_t* res, const uint8_t* include) {
    if (!p || n_obj < 0) return set_err(GM_ERR_ARG, "bad plan/objects");
    CK(cudaSetDevice(p->device));
    plan_free_scene(p);
    int64_t T = 0, N = 0;
    std::vector<int64_t> tstart(n_obj + 1, 0), nsamp(n_obj, 0);
    for (int o = 0; o < n_obj; o++) {
        tstart[o] = T;
        T += tri_counts[o];
    }
    tstart[n_obj] = T;
    // per-object sample totals from the resolutions (counts = (r+1)(r+2)/2)
    for (int o = 0; o < n_obj; o++) {
        int64_t s = 0;
        for (int64_t t = tstart[o]; t < tstart[o + 1]; t++) s += (res[t] + 1) * (res[t] + 2) / 2;
        nsamp[o] = s;
        if (include[o]) N += s;
    }
    p->T = T;
    p->N = N;
    p->n_clu = (T + 31) / 32;
    p->n_chunks = (N + 31) / 32;
    p->n_supers = (p->n_chunks + 7) / 8;
    int rc;
    if ((rc = dev_alloc(&p->d_tw, (size_t)T * 9))) return rc;
    if ((rc = dev_alloc(&p->d_tsph, (size_t)T))) return rc;
    if ((rc = dev_alloc(&p->d_csph, (size_t)p->n_clu))) return rc;
    if ((rc = dev_alloc(&p->d_px, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_py, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_pz, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_pxf, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_pyf, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_pzf, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_chunk, (size_t)p->n_chunks))) return rc;
    if ((rc = dev_alloc(&p->d_super, (size_t)p->n_supers))) return rc;
    if ((rc = dev_alloc(&p->d_values, (size_t)N))) return rc;
    p->n_obj = n_obj;
    p->tstart = tstart;
    p->nsamp = nsamp;
    p->include.assign(include, include + n_obj);
    if (T == 0) return GM_OK;
    int64_t* d_cnt = nullptr;
    if ((rc = dev_alloc(&p->d_local, (size_t)T * 9))) return rc;
    if ((rc = dev_alloc(&p->d_M, (size_t)n_obj * 12))) return rc;
    if ((rc = dev_alloc(&p->d_res, (size_t)T))) return rc;
    if ((rc = dev_alloc(&d_cnt, (size_t)T))) return rc;
    if ((rc = dev_alloc(&p->d_off, (size_t)T))) return rc;
    cudaStream_t s = p->stream;
    CK(cudaMemcpyAsync(p->d_local, tri_local, sizeof(double) * 9 * T, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(p->d_res, res, sizeof(int64_t) * T, cudaMemcpyHostToDevice, s));
    for (int o = 0; o < n_obj; o++) {
        int64_t To = tri_counts[o];
        if (To == 0 || !include[o] || nsamp[o] == 0) continue;
        const double* loc = p->d_local + 9 * tstart[o];
        k_layout<<<blocks_for(To, 256), 256, 0, s>>>(loc, To, 0.0, p->d_res + tstart[o], nullptr,
                                                       d_cnt + tstart[o]);
        size_t tmp = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_cnt + tstart[o], p->d_off + tstart[o], To, s);
        if (tmp > p->scan_tmp_bytes) {
            cudaFree(p->d_scan_tmp);
            p->d_scan_tmp = nullptr;
            CK(cudaMalloc(&p->d_scan_tmp, tmp));
            p->scan_tmp_bytes = tmp;
        }
        CK(cub::DeviceScan::ExclusiveSum(p->d_scan_tmp, tmp, d_cnt + tstart[o], p->d_off + tstart[o], To, s));
    }
    CK(cudaStreamSynchronize(s));
    cudaFree(d_cnt);
    return gm_plan_set_poses(p, xforms);
}

// Object poses (n_obj x [t(3), q xyzw(4), s(3)]) of a plan whose layout is
// set: world occluder triangles (scene_world_triangles, raster.py:68-78) and
// world sample positions (_SampleCache.world, density.py:121-127: override
// .apply(local)), both with the OpenBLAS FMA chain, then every derived
// structure (float32 copies, bounding spheres).  generate() calls it between
// runs of fixations that share the same pose overrides (dynamic scenes).
extern "C" int gm_plan_set_poses(gm_plan* p, const double* xforms) {
    if (!p || (p->n_obj > 0 && !xforms)) return set_err(GM_ERR_ARG, "bad plan/poses");
    CK(cudaSetDevice(p->device));
    const int64_t T = p->T, N = p->N;
    const int n_obj = p->n_obj;
    if (T == 0) return GM_OK;
    cudaStream_t s = p->stream;
    std::vector<double> Mt(n_obj * 12);
    for (int o = 0; o < n_obj; o++) xform_matrix(xforms + 10 * o, &Mt[12 * o], &Mt[12 * o + 9]);
    CK(cudaMemcpyAsync(p->d_M, Mt.data(), sizeof(double) * 12 * n_obj, cudaMemcpyHostToDevice, s));
    int64_t sample_base = 0;
    for (int o = 0; o < n_obj; o++) {
        const int64_t To = p->tstart[o + 1] - p->tstart[o];
        if (To == 0) continue;
        const double* loc = p->d_local + 9 * p->tstart[o];
        k_world_tris<<<blocks_for(3 * To, 256), 256, 0, s>>>(loc, To, p->d_M + 12 * o, p->d_M + 12 * o + 9,
                                                              p->d_tw + 9 * p->tstart[o]);
        if (!p->include[o] || p->nsamp[o] == 0) continue;
        const int64_t No = p->nsamp[o];
        k_positions<<<blocks_for(No, 256), 256, 0, s>>>(loc, To, p->d_res + p->tstart[o], p->d_off + p->tstart[o],
                                                          No, p->d_M + 12 * o, p->d_M + 12 * o + 9, nullptr,
                                                          p->d_px + sample_base, p->d_py + sample_base,
                                                          p->d_pz + sample_base);
        sample_base += No;
    }
    p->pmax = 0.0;
    if (N > 0) {
        CK(cudaMemsetAsync(p->d_max, 0, sizeof(unsigned long long), s));
        k_to_f32<<<blocks_for(N, 256), 256, 0, s>>>(p->d_px, p->d_py, p->d_pz, N, p->d_pxf, p->d_pyf, p->d_pzf,
                                                    p->d_max);
        unsigned long long bits = 0;
        CK(cudaMemcpyAsync(&bits, p->d_max, sizeof(bits), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        memcpy(&p->pmax, &bits, sizeof(double));
    }
    k_tri_spheres<<<blocks_for(T, 256), 256, 0, s>>>(p->d_tw, T, p->d_tsph);
    k_group_spheres<<<blocks_for(p->n_clu, 128), 128, 0, s>>>(p->d_tsph, nullptr, nullptr, nullptr, T, p->d_csph, 32);
    if (N > 0) {
        k_group_spheres<<<blocks_for(p->n_chunks, 128), 128, 0, s>>>(nullptr, p->d_px, p->d_py, p->d_pz, N,
                                                                      p->d_chunk, 32);
        k_group_spheres<<<blocks_for(p->n_supers, 128), 128, 0, s>>>(p->d_chunk, nullptr, nullptr, nullptr,
                                                                      p->n_chunks, p->d_super, 8);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return GM_OK;
}

extern "C" int64_t gm_plan_num_samples(gm_plan* p) { return p ? p->N : -1; }
extern "C" int64_t gm_plan_num_triangles(gm_plan* p) { return p ? p->T : -1; }
extern "C" double* gm_plan_values_device(gm_plan* p) { return p ? p->d_values : nullptr; }

static int ensure_batch_set(gm_plan* p, int B, int W, int H, int64_t seg) {
    int rc;
    if (!p->stream) {
        cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return set_err(GM_ERR_CUDA, cudaGetErrorString(e));
    }
    if (!p->d_work && (rc = dev_alloc(&p->d_work, 2))) return rc;
    if (B > p->cap_B) {
        if ((rc = dev_alloc(&p->d_fix, (size_t)B))) return rc;
        if ((rc = dev_alloc(&p->d_cull, (size_t)B))) return rc;
        if ((rc = dev_alloc(&p->d_count, (size_t)B))) return rc;
        if ((rc = dev_alloc(&p->d_fix32, (size_t)B))) return rc;
        p->cap_B = B;
    }
    if (p->n_supers > p->cap_sort) {
        if ((rc = dev_alloc(&p->d_lcount, (size_t)p->n_supers))) return rc;
        if ((rc = dev_alloc(&p->d_lorder, (size_t)p->n_supers))) return rc;
        if ((rc = dev_alloc(&p->d_lcount2, (size_t)p->n_supers))) return rc;
        if ((rc = dev_alloc(&p->d_lorder2, (size_t)p->n_supers))) return rc;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, p->d_lcount, p->d_lcount2, p->d_lorder,
                                                  p->d_lorder2, (int)std::max<int64_t>(p->n_supers, 1), 0, 11);
        if ((rc = dev_alloc((char**)&p->d_sort_tmp, tb + 16))) return rc;
        p->sort_tmp_bytes = tb + 16;
        p->cap_sort = p->n_supers;
    }
    if (p->n_chunks * 32 > p->cap_cbits) {
        if ((rc = dev_alloc(&p->d_cbits, (size_t)p->n_chunks * 32))) return rc;
        p->cap_cbits = p->n_chunks * 32;
    }
    if (seg > p->cap_seg || (int64_t)B * seg > p->cap_seg_B) {
        int64_t cs = std::max(seg, p->cap_seg);
        if ((rc = dev_alloc(&p->d_tris, (size_t)(B * cs)))) return rc;
        if ((rc = dev_alloc(&p->d_t32, (size_t)(B * cs)))) return rc;
        if ((rc = dev_alloc(&p->d_bbox, (size_t)(B * cs)))) return rc;
        p->cap_seg = cs;
        p->cap_seg_B = B * cs;
    }
    const int wwords = (W + 31) / 32;
    const int64_t mask_words = (int64_t)B * H * wwords;
    if (mask_words > p->cap_mask) {
        if ((rc = dev_alloc(&p->d_mask, (size_t)mask_words))) return rc;
        p->cap_mask = mask_words;
    }
    if ((int64_t)B * W * H > p->cap_depth) {
        if ((rc = dev_alloc(&p->d_depth, (size_t)B * W * H))) return rc;
        if ((rc = dev_alloc(&p->d_vbuf, (size_t)B * W * H))) return rc;
        if ((rc = dev_alloc(&p->d_win, (size_t)B * W * H))) return rc;
        if ((rc = dev_alloc(&p->d_carry, (size_t)B * W * H))) return rc;
        p->cap_depth = (int64_t)B * W * H;
    }

    if (B > p->cap_cB || CB_ITEMS_PER_TRI * p->cap_seg > p->cap_citems) {
        const int64_t ci = CB_ITEMS_PER_TRI * std::max<int64_t>(p->cap_seg, seg);
        if ((rc = dev_alloc(&p->d_citems, (size_t)B * ci))) return rc;
        if ((rc = dev_alloc(&p->d_coff, (size_t)B * (GM_MAX_CBINS + 1)))) return rc;
        if ((rc = dev_alloc(&p->d_covf, (size_t)B))) return rc;
        p->cap_citems = ci;
        p->cap_cB = B;
    }
    const int64_t n_tiles = (int64_t)B * ((W + TW - 1) / TW) * ((H + TH_FULL - 1) / TH_FULL);  // the smaller tiles
    if (n_tiles > p->cap_crowd) {
        if ((rc = dev_alloc(&p->d_crowd, (size_t)n_tiles))) return rc;
        if ((rc = dev_alloc(&p->d_tmax, (size_t)n_tiles))) return rc;
        if (!p->d_crowd_count && (rc = dev_alloc(&p->d_crowd_count, 2))) return rc;
        p->cap_crowd = n_tiles;
    }
    const int64_t lw = std::max<int64_t>(p->n_supers, 1) * ((B + 31) / 32);
    if (lw > p->cap_lvl1) {
        if ((rc = dev_alloc(&p->d_lvl1, (size_t)lw))) return rc;
        p->cap_lvl1 = lw;
    }
    return GM_OK;
}

// Both batch-buffer sets (the alternate one only when `both`), plus the pinned
// host ring that feeds either.
static int ensure_batch(gm_plan* p, int B, int W, int H, int64_t seg, bool both = false) {
    int rc;
    if (B > p->cap_ring) {
        for (int r = 0; r < GM_RING; r++) {
            cudaFreeHost(p->h_fix[r]);
            cudaFreeHost(p->h_cull[r]);
            CK(cudaMallocHost(&p->h_fix[r], sizeof(GmFixExact) * B));
            CK(cudaMallocHost(&p->h_cull[r], sizeof(GmFixCull) * B));
        }
        p->cap_ring = B;
    }
    if ((rc = ensure_batch_set(p, B, W, H, seg))) return rc;
    if (!both) return GM_OK;
    for (int k = 1; k < GM_NSETS && !rc; k++) {
        swap_batch_bufs(p, k);
        rc = ensure_batch_set(p, B, W, H, std::max(seg, p->cap_seg));
        swap_batch_bufs(p, k);
    }
    return rc;
}

typedef void (*gm_progress_fn)(int64_t done, int64_t total, void* user);

// Coarse-bin geometry for a W x H buffer: cb = 2^CB_SHIFT px, doubled until <= GM_MAX_CBINS bins.
static CoarseBins coarse_bins(gm_plan* p, int W, int H) {
    int shift = CB_SHIFT;
    while ((int64_t)((W + (1 << shift) - 1) >> shift) * ((H + (1 << shift) - 1) >> shift) > GM_MAX_CBINS) shift++;
    CoarseBins cb{p->d_citems, p->d_coff, p->d_covf, p->cap_citems, shift, (W + (1 << shift) - 1) >> shift,
                  (H + (1 << shift) - 1) >> shift};
    return cb;
}


// k_texels over `items` (fixation, tile) work items, then the crowded tiles the
// first pass deferred (k_texels<CROWDED>, persistent, larger shared slices).
template <bool ATTRS, bool STATS, bool EXACT, int TH>
static void launch_texels_th(gm_plan* p, cudaStream_t s, const TriStore& ts, const DepthView& dv,
                             const CoarseBins& cb, int tiles_x, int tiles_per_fix, int64_t items,
                             const GmFixExact* fix, long long b0) {
    const int tiles_y = tiles_per_fix / tiles_x;
    constexpr int nw = TexelWarps<TH>::n;
    const dim3 grid((unsigned)tiles_x, (unsigned)((tiles_y + nw - 1) / nw), (unsigned)(items / tiles_per_fix));
    k_texels<ATTRS, STATS, EXACT, TH><<<grid, nw * 32, nw * (int)sizeof(TexelWarpSmem), s>>>(ts, dv, cb, tiles_x, tiles_per_fix,
                                                                           tiles_y, fix, b0);
    if (dv.crowd_wide) {  // full-frustum batches and the raster API: few, long tiles
        k_texels_crowded<ATTRS, STATS, EXACT, HV_FULL_WARPS, HV_FULL_SEL, TH>
            <<<p->sms * (HV_FULL_WARPS_SM / HV_FULL_WARPS), HV_FULL_WARPS * 32, (int)sizeof(HeavySmem<HV_FULL_WARPS, HV_FULL_SEL>),
               s>>>(ts, dv, cb, tiles_x, tiles_per_fix, fix, b0);
    } else {
        k_texels_crowded<ATTRS, STATS, EXACT, HV_CROP_WARPS, HV_CROP_SEL, TH>
            <<<p->sms * (HV_CROP_WARPS_SM / HV_CROP_WARPS), HV_CROP_WARPS * 32, (int)sizeof(HeavySmem<HV_CROP_WARPS, HV_CROP_SEL>),
               s>>>(ts, dv, cb, tiles_x, tiles_per_fix, fix, b0);
    }
}

// k_texels over `items` (fixation, tile) work items of height 1 << dv.th_shift, then
// the crowded tiles the first pass deferred (k_texels_crowded, persistent CTAs).
template <bool ATTRS, bool STATS, bool EXACT>
static int launch_texels(gm_plan* p, cudaStream_t s, const TriStore& ts, DepthView dv, const CoarseBins& cb,
                         int tiles_x, int tiles_per_fix, int64_t items, const GmFixExact* fix, long long b0) {
    dv.crowd = p->d_crowd;
    dv.crowd_count = p->d_crowd_count;
    CK(cudaMemsetAsync(p->d_crowd_count, 0, 2 * sizeof(int), s));
    if constexpr (!ATTRS && !EXACT) {
        if (dv.th_shift == 5) {
            launch_texels_th<ATTRS, STATS, EXACT, 32>(p, s, ts, dv, cb, tiles_x, tiles_per_fix, items, fix, b0);
            CK(cudaGetLastError());
            return GM_OK;
        }
    }
    launch_texels_th<ATTRS, STATS, EXACT, TH_FULL>(p, s, ts, dv, cb, tiles_x, tiles_per_fix, items, fix, b0);
    CK(cudaGetLastError());
    return GM_OK;
}

static inline double wall_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void k_set_i64(long long* p, long long v) { *p = v; }

// Kernels of one batch (already-uploaded setup records d_fix/d_cull):
// occluder setup, candidate marking, texel evaluation, accumulation.
static int enqueue_batch(gm_plan* p, const GmFixExact* d_fix, const GmFixCull* d_cull, int nb, int W, int H,
                         long long b0, double inv_sigma, const GmConfig* cfg, bool accumulate, cudaEvent_t* ev) {
    cudaStream_t s = p->stream;
    const int wwords = (W + 31) / 32;
    const int th = cfg->filtering ? TH_CROP : TH_FULL;
    const int tiles_x = (W + TW - 1) / TW, tiles_y = (H + th - 1) / th;
    TriStore ts{p->d_tris, p->d_t32, p->d_bbox, p->d_count, p->cap_seg, p->d_fail, p->d_maxcount, p->d_ntris};
    DepthView dv{p->d_depth, p->d_mask, W, H, wwords, (cfg->flags & GM_FLAG_STATS) ? p->d_stats : nullptr,
                 p->d_vbuf};
    dv.th_shift = th == 32 ? 5 : 4;
#ifdef GM_CHECK
    dv.check = p->d_check;
#endif
    dv.win = p->d_win;
    dv.carry = p->d_carry;
    dv.tmax = p->d_tmax;
    // crop-frustum z-buffers (filtering): a tile overlapping more than TW_CAP triangles is
    // a small distant object, walked faster whole (crowded pass, float32 fast path) than
    // chunk by chunk (C2 -3%); full-frustum tiles with such lists are far more common and
    // the persistent crowded pass is slower for them (unfiltered C2 +6%)
    dv.crowd_wide = cfg->filtering ? 0 : 1;
    dv.tiles_x = (W + TW - 1) / TW;
    dv.tiles_per_fix = dv.tiles_x * tiles_y;
    if (ev) CK(cudaEventRecord(ev[0], s));
    CK(cudaMemsetAsync(p->d_count, 0, sizeof(int) * nb, s));
    if (p->n_clu > 0) {
        dim3 grid(blocks_for((p->n_clu + 31) / 32, TS_WARPS), nb);
        k_tri_setup<<<grid, TS_WARPS * 32, 0, s>>>(p->d_tw, p->T, p->d_tsph, p->d_csph, p->n_clu, d_fix, d_cull, W, H, ts, b0);
    }
    if (ev) CK(cudaEventRecord(ev[1], s));
    if (p->n_chunks > 0 && accumulate) {
        // persistent sample passes: exactly the resident CTAs (work is claimed dynamically;
        // a second wave would only start late and idle)
        int occ_m = 0, occ_s = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_m, k_mark, 256, 0));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, dv.stats ? k_samples<true> : k_samples<false>, 256, 0));
        const int grid_m = p->sms * std::max(occ_m, 1) * SAMPLE_GRID_MULT, grid_s = p->sms * std::max(occ_s, 1) * SAMPLE_GRID_MULT;
        CK(cudaMemsetAsync(p->d_mask, 0, sizeof(uint32_t) * (size_t)nb * H * wwords, s));
        CK(cudaMemsetAsync(p->d_work, 0, 2 * sizeof(int), s));
        k_level1<<<blocks_for(p->n_supers, 8), 256, 0, s>>>(p->d_super, p->n_supers, d_cull, nb, p->d_lvl1,
                                                             p->d_lcount, p->d_lorder, p->d_fail, b0);
        size_t tb = p->sort_tmp_bytes;
        CK(cub::DeviceRadixSort::SortPairsDescending(p->d_sort_tmp, tb, p->d_lcount, p->d_lcount2, p->d_lorder,
                                                     p->d_lorder2, (int)p->n_supers, 0, 11, s));
        k_fix32<<<blocks_for(nb, 128), 128, 0, s>>>(d_fix, nb, p->pmax, 1.0 / inv_sigma, p->d_fix32);
        k_mark<<<grid_m, 256, 0, s>>>(p->d_pxf, p->d_pyf, p->d_pzf, p->d_px, p->d_py, p->d_pz, p->d_chunk, p->d_lvl1,
                                    p->d_lorder2, p->d_work, p->N, p->n_chunks, p->n_supers, d_fix, p->d_fix32,
                                    d_cull, nb, dv, inv_sigma, p->d_cbits, p->d_fail, b0);
#ifdef GM_CHECK
        k_check_candidates<<<blocks_for(p->N, 128), 128, 0, s>>>(p->d_px, p->d_py, p->d_pz, p->N, d_fix, nb, dv,
                                                                 inv_sigma, p->d_cbits, p->d_lvl1, p->d_fail, b0);
#endif
        if (ev) CK(cudaEventRecord(ev[2], s));
        const int64_t items = (int64_t)nb * tiles_x * tiles_y;
        CoarseBins cbins = coarse_bins(p, W, H);
        k_coarse<<<nb, 256, 0, s>>>(ts, cbins, p->d_fail, b0, dv.stats);
        int trc = dv.stats
                      ? launch_texels<false, true, false>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, d_fix, b0)
                      : launch_texels<false, false, false>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, d_fix, b0);
        if (trc) return trc;
#ifdef GM_CHECK
        if (p->n_clu > 0) {
            dim3 grid(blocks_for((p->n_clu + 31) / 32, TS_WARPS), nb);
            k_check_cull<<<grid, TS_WARPS * 32, 0, s>>>(p->d_tw, p->T, p->d_tsph, p->d_csph, p->n_clu, d_fix, d_cull, W,
                                                       H, ts, dv, b0);
        }
#endif
        if (ev) CK(cudaEventRecord(ev[3], s));
        // accumulation passes run in batch order across the two streams (log order per sample)
        CK(cudaStreamWaitEvent(s, p->ev_order, 0));
        auto ks = dv.stats ? k_samples<true> : k_samples<false>;
        ks<<<grid_s, 256, 0, s>>>(p->d_px, p->d_py, p->d_pz, p->d_chunk, p->d_lvl1, p->d_lorder2, p->d_work + 1, p->N,
                                p->n_chunks, p->n_supers, d_fix, d_cull, nb, dv, inv_sigma, cfg->eps_abs,
                                cfg->eps_rel, p->d_values, p->d_cbits, p->d_tris, p->cap_seg, p->d_fail, b0);
        CK(cudaEventRecord(p->ev_order, s));
    } else if (ev) {
        CK(cudaEventRecord(ev[2], s));
        CK(cudaEventRecord(ev[3], s));
    }
    if (ev) CK(cudaEventRecord(ev[4], s));
    CK(cudaGetLastError());
    return GM_OK;
}

// One pass over F fixations in batches, all enqueued without host syncs.
// Either `fx` (host table: the host setup of batch i+1 runs while the GPU
// works on batch i, through a ring of pinned slots) or the prepared device
// setup table (gm_plan_prepare) supplies the per-fixation records.  If a batch
// overflows the screen-triangle segments, it and every later batch is a no-op
// on the device; the host grows the segments and resumes from that batch, so
// the per-sample accumulation order is still the log order.
static int run_batches(gm_plan* p, const double* fx, int64_t F, const GmConfig* cfg, int reset, GmTimings* tm,
                       gm_progress_fn progress, void* user, int64_t* bad_fixation, float* device_ms) {
    if (cfg->zbuffer_resolution < 1 || cfg->zbuffer_resolution > 65535)
        return set_err(GM_ERR_ARG, "zbuffer_resolution must be in [1, 65535]");
    if (!(cfg->theta > 0.0 && cfg->theta < 1.5707963267948966)) return set_err(GM_ERR_ARG, "theta out of range");
    CK(cudaSetDevice(p->device));
    const bool prepared = fx == nullptr;
    double t_start = wall_ms();
    const int W = cfg->zbuffer_resolution, H = cfg->zbuffer_resolution;
    int B = cfg->batch > 0 ? cfg->batch : 1024;
    if (B > GM_MAX_BATCH) B = GM_MAX_BATCH;
    const int64_t depth_per_fix = (int64_t)W * H;
    int64_t max_d = std::max<int64_t>(1, ((int64_t)1 << 28) / depth_per_fix);  // z-buffer store <= 2 GiB
    if (B > max_d) B = (int)max_d;
    if (F > 0 && B > F) B = (int)F;
    B = std::max(B, 1);
    GmSetupConsts consts;
    gm_setup_consts(cfg->theta, cfg->filtering, W, H, &consts);
    // two-stream batch overlap fills kernel tails on scenes with light batches (C2:
    // -14%); on very large scenes every kernel already fills the GPU and concurrent
    // batches only thrash L2 (C5: +14%), so they run on one stream
    const bool two = (cfg->flags & GM_FLAG_TWO_STREAMS) ||
                     (!(cfg->flags & GM_FLAG_ONE_STREAM) && p->T <= GM_OVERLAP_MAX_TRIS);
    int rc = ensure_batch(p, B, W, H, std::max<int64_t>(p->cap_seg, p->seg_init), two);
    if (rc) return rc;
    cudaStream_t s = p->stream;          // primary stream (even batches)

    cudaEvent_t ev_fork = nullptr;
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    auto fork = [&]() -> int {  // everything enqueued on s so far precedes what the other streams run next
        if (!two) return GM_OK;
        CK(cudaEventRecord(ev_fork, s));
        for (int k = 0; k < GM_NSETS - 1; k++) CK(cudaStreamWaitEvent(p->alt[k].stream, ev_fork, 0));
        return GM_OK;
    };
    auto join = [&]() -> int {  // s waits for everything enqueued on the other streams
        if (!two) return GM_OK;
        for (int k = 0; k < GM_NSETS - 1; k++) {
            CK(cudaEventRecord(ev_fork, p->alt[k].stream));
            CK(cudaStreamWaitEvent(s, ev_fork, 0));
        }
        return GM_OK;
    };
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;
    std::vector<cudaEvent_t> evs;
    auto cleanup = [&]() {
        for (auto e : evs) cudaEventDestroy(e);
        evs.clear();
        if (ev_start) cudaEventDestroy(ev_start);
        if (ev_end) cudaEventDestroy(ev_end);
        if (ev_fork) cudaEventDestroy(ev_fork);
        ev_start = ev_end = ev_fork = nullptr;
    };
    if (device_ms) {
        CK(cudaEventCreate(&ev_start));
        CK(cudaEventCreate(&ev_end));
        CK(cudaEventRecord(ev_start, s));
    }
    if (reset && p->N > 0) CK(cudaMemsetAsync(p->d_values, 0, sizeof(double) * p->N, s));
    if (cfg->flags & GM_FLAG_STATS)
        CK(cudaMemsetAsync(p->d_stats, 0, GM_STAT_STRIPES * GM_STAT_N * sizeof(unsigned long long), s));
    GmTimings t;
    memset(&t, 0, sizeof(t));
    const bool timing = tm != nullptr;
    const double inv_sigma = 1.0 / consts.sigma;
    int64_t start = 0;
    for (int attempt = 0; attempt < 16; attempt++) {
        k_set_i64<<<1, 1, 0, s>>>(p->d_fail, LLONG_MAX);
        CK(cudaMemsetAsync(p->d_maxcount, 0, sizeof(int), s));
        CK(cudaMemsetAsync(p->d_ntris, 0, sizeof(unsigned long long), s));
        CK(cudaEventRecord(p->ev_order, s));  // the first accumulation pass follows the resets
        if ((rc = fork())) return rc;
        int slot = 0;
        int parity = 0;
        for (int64_t b0 = start; b0 < F; b0 += B, parity = two ? (parity + 1) % GM_NSETS : 0) {
            int nb = (int)std::min<int64_t>(B, F - b0);
            // odd batches run on the alternate buffer set and stream
            struct SwapGuard {
                gm_plan* p;
                int k;
                ~SwapGuard() {
                    if (k) swap_batch_bufs(p, k);
                }
            } guard{p, parity};
            if (parity) swap_batch_bufs(p, parity);
            cudaStream_t s = p->stream;
            const GmFixExact* d_fix = p->d_fix;
            const GmFixCull* d_cull = p->d_cull;
            if (prepared) {
                d_fix = p->d_fix_all + b0;
                d_cull = p->d_cull_all + b0;
            } else {
                CK(cudaEventSynchronize(p->h_ev[slot]));  // slot's previous upload has completed
                double ts = wall_ms();
                int64_t bad = gm_setup_batch(fx + GM_FIX_STRIDE * b0, nb, &consts, p->h_fix[slot], p->h_cull[slot],
                                             p->host_threads);
                t.setup_ms += wall_ms() - ts;
                if (bad >= 0) {
                    cudaStreamSynchronize(s);
                    cleanup();
                    if (bad_fixation) *bad_fixation = b0 + bad;
                    return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
                }
                CK(cudaMemcpyAsync(p->d_fix, p->h_fix[slot], sizeof(GmFixExact) * nb, cudaMemcpyHostToDevice, s));
                CK(cudaMemcpyAsync(p->d_cull, p->h_cull[slot], sizeof(GmFixCull) * nb, cudaMemcpyHostToDevice, s));
                CK(cudaEventRecord(p->h_ev[slot], s));
                slot = (slot + 1) % GM_RING;
            }
            cudaEvent_t* e = nullptr;
            if (timing) {
                for (int q = 0; q < 5; q++) {
                    cudaEvent_t x;
                    CK(cudaEventCreate(&x));
                    evs.push_back(x);
                }
                e = &evs[evs.size() - 5];
            }
            rc = enqueue_batch(p, d_fix, d_cull, nb, W, H, (long long)b0, inv_sigma, cfg, true, e);
            if (rc) {
                cleanup();
                return rc;
            }
            t.batches += 1;
            if (progress) {  // per-batch progress needs a sync; only then
                CK(cudaStreamSynchronize(s));
                long long failed = LLONG_MAX;
                CK(cudaMemcpy(&failed, p->d_fail, sizeof(failed), cudaMemcpyDeviceToHost));
                if (failed == LLONG_MAX) progress(b0 + nb, F, user);
            }
        }
        if ((rc = join())) return rc;
        long long failed = LLONG_MAX;
        int maxcount = 0;
        unsigned long long ntris = 0;
        CK(cudaMemcpyAsync(&failed, p->d_fail, sizeof(failed), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&maxcount, p->d_maxcount, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&ntris, p->d_ntris, sizeof(ntris), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        t.screen_tris += (int64_t)ntris;
        if (failed == LLONG_MAX) break;
        // grow the per-fixation segments and resume at the first failed batch
        int64_t want = std::max<int64_t>(2 * p->cap_seg, (int64_t)maxcount + maxcount / 4 + 64);
        p->cap_seg = 0;
        for (int k = 0; k < GM_NSETS - 1; k++) p->alt[k].cap_seg = 0;
        rc = ensure_batch(p, B, W, H, want, two);
        if (rc) {
            cleanup();
            return rc;
        }
        start = failed;
        t.batches = 0;
        t.retries += 1;
        if (attempt == 15) {
            cleanup();
            return set_err(GM_ERR_OOM, "screen-triangle segments kept overflowing");
        }
    }
    if (device_ms) CK(cudaEventRecord(ev_end, s));
    CK(cudaStreamSynchronize(s));
    if (device_ms) cudaEventElapsedTime(device_ms, ev_start, ev_end);
    if (timing) {
        // events of the last (successful) pass are the last t.batches groups
        size_t first = evs.size() - 5 * (size_t)t.batches;
        for (size_t q = first; q + 4 < evs.size(); q += 5) {
            float a[4] = {0, 0, 0, 0};
            for (int z = 0; z < 4; z++) cudaEventElapsedTime(&a[z], evs[q + z], evs[q + z + 1]);
            t.cull_ms += a[0];
            t.mark_ms += a[1];
            t.texel_ms += a[2];
            t.accumulate_ms += a[3];
        }
        t.total_ms = wall_ms() - t_start;
        t.bin_items = 0;
        *tm = t;
    }
    cleanup();
    return GM_OK;
}

// Accumulate fixations (F x 18, log schema) into the plan's device values
// (zeroed first if reset).  Values stay on device; gm_plan_read copies out.
extern "C" int gm_plan_accumulate(gm_plan* p, const double* fx, int64_t F, const GmConfig* cfg, int reset,
                                  GmTimings* tm, gm_progress_fn progress, void* user, int64_t* bad_fixation) {
    if (!p || !cfg || (F > 0 && !fx)) return set_err(GM_ERR_ARG, "null argument");
    static const double dummy = 0.0;
    return run_batches(p, F > 0 ? fx : &dummy, F, cfg, reset, tm, progress, user, bad_fixation, nullptr);
}

// Compute the setup records of F fixations once and keep them in HBM, so
// gm_plan_run can replay the whole generation with every input resident.
extern "C" int gm_plan_prepare(gm_plan* p, const double* fx, int64_t F, const GmConfig* cfg, int64_t* bad_fixation) {
    if (!p || !cfg || (F > 0 && !fx)) return set_err(GM_ERR_ARG, "null argument");
    CK(cudaSetDevice(p->device));
    const int W = cfg->zbuffer_resolution;
    GmSetupConsts consts;
    gm_setup_consts(cfg->theta, cfg->filtering, W, W, &consts);
    std::vector<GmFixExact> ex(std::max<int64_t>(F, 1));
    std::vector<GmFixCull> cu(std::max<int64_t>(F, 1));
    int64_t bad = gm_setup_batch(fx, F, &consts, ex.data(), cu.data(), p->host_threads);
    if (bad >= 0) {
        if (bad_fixation) *bad_fixation = bad;
        return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
    }
    int rc;
    if ((rc = dev_alloc(&p->d_fix_all, (size_t)std::max<int64_t>(F, 1)))) return rc;
    if ((rc = dev_alloc(&p->d_cull_all, (size_t)std::max<int64_t>(F, 1)))) return rc;
    CK(cudaMemcpy(p->d_fix_all, ex.data(), sizeof(GmFixExact) * F, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(p->d_cull_all, cu.data(), sizeof(GmFixCull) * F, cudaMemcpyHostToDevice));
    p->F_prepared = F;
    p->cfg_prepared = *cfg;
    return GM_OK;
}

// Replay the prepared fixations (device-resident inputs).  device_ms gets the
// CUDA-event time of the whole pass on the plan's stream.
extern "C" int gm_plan_run(gm_plan* p, int reset, int flags, GmTimings* tm, float* device_ms) {
    if (!p) return set_err(GM_ERR_ARG, "null plan");
    if (p->F_prepared < 0) return set_err(GM_ERR_ARG, "gm_plan_prepare was not called");
    GmConfig cfg = p->cfg_prepared;
    cfg.flags = flags;
    return run_batches(p, nullptr, p->F_prepared, &cfg, reset, tm, nullptr, nullptr, nullptr, device_ms);
}

// Evict L2 between timed repetitions: write `bytes` (> 126 MB L2) on the plan stream.
extern "C" int gm_plan_flush_l2(gm_plan* p, int64_t bytes) {
    if (!p || bytes <= 0) return set_err(GM_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(p->device));
    if (bytes > p->flush_bytes) {
        cudaFree(p->d_flush);
        p->d_flush = nullptr;
        CK(cudaMalloc(&p->d_flush, bytes));
        p->flush_bytes = bytes;
    }
    CK(cudaMemsetAsync(p->d_flush, (int)(++p->flush_gen & 0xff), bytes, p->stream));
    return GM_OK;
}

// Work counters of the last gm_plan_accumulate / gm_plan_run made with
// GmConfig.flags & 1 (GM_STAT_* order, 16 x uint64).
extern "C" int gm_plan_stats(gm_plan* p, unsigned long long* out) {
    if (!p || !out) return set_err(GM_ERR_ARG, "null argument");
    CK(cudaSetDevice(p->device));
    CK(cudaStreamSynchronize(p->stream));
    std::vector<unsigned long long> st((size_t)GM_STAT_STRIPES * GM_STAT_N);
    CK(cudaMemcpy(st.data(), p->d_stats, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    for (int k = 0; k < GM_STAT_N; k++) {
        unsigned long long a = 0;
        for (int r = 0; r < GM_STAT_STRIPES; r++) a += st[(size_t)r * GM_STAT_N + k];
        out[k] = a;
    }
    return GM_OK;
}

// Global max over the plan's values (density.py:192; values are monotone so
// the final max equals the reference's running max).
extern "C" int gm_plan_max(gm_plan* p, double* gmax) {
    if (!p || !gmax) return set_err(GM_ERR_ARG, "null argument");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    CK(cudaMemsetAsync(p->d_max, 0, sizeof(unsigned long long), s));
    if (p->N > 0) k_max<<<std::min<int64_t>(blocks_for(p->N, 256), (int64_t)p->sms * 8), 256, 0, s>>>(p->d_values, p->N, p->d_max);
    unsigned long long bits = 0;
    CK(cudaMemcpyAsync(&bits, p->d_max, sizeof(bits), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    memcpy(gmax, &bits, sizeof(double));
    return GM_OK;
}

// ---------------------------------------------- multi-GPU: fused peer reduce
// Rank r owns slice r of the N accumulators: it reads that slice from every
// rank's partial map through NVLink peer loads, sums in rank order (the same
// bits on every rank, run to run), stores the sum into every rank's map
// through peer stores and takes the slice's max -- reduce-scatter, all-gather
// and the first half of the global max in one pass, no staging buffer.
// Slices are disjoint, so ranks never touch the same addresses.
__global__ void k_reduce_peers(double* const* __restrict__ bufs, int world, int64_t a, int64_t b,
                               unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
        double s = bufs[0][i];
        for (int r = 1; r < world; r++) s += bufs[r][i];
        for (int r = 0; r < world; r++) bufs[r][i] = s;
        m = fmax(m, s);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// The same for up to GM_PEER_MAX ranks: the peer pointers in registers, 16-byte
// (2-sample) peer loads and stores over the 16-byte-aligned body of the slice,
// the same rank-order sum per sample (identical bits to k_reduce_peers).
#define GM_PEER_MAX 8
__global__ void k_reduce_peers_vec(double* const* __restrict__ bufs, int world, int64_t a, int64_t b,
                                   unsigned long long* __restrict__ out) {
    double* p[GM_PEER_MAX];
#pragma unroll
    for (int r = 0; r < GM_PEER_MAX; r++) p[r] = r < world ? bufs[r] : nullptr;
    double m = 0.0;
    auto one = [&](int64_t i) {
        double s = p[0][i];
#pragma unroll
        for (int r = 1; r < GM_PEER_MAX; r++)
            if (r < world) s += p[r][i];
#pragma unroll
        for (int r = 0; r < GM_PEER_MAX; r++)
            if (r < world) p[r][i] = s;
        m = fmax(m, s);
    };
    const int64_t a2 = (a + 1) & ~(int64_t)1, b2 = b & ~(int64_t)1;  // even bounds of the body
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
    if (a2 >= b2) {
        for (int64_t i = a + tid; i < b; i += nthr) one(i);
    } else {
        if (tid == 0 && a < a2) one(a);
        if (tid == 1 && b2 < b) one(b2);
        for (int64_t j = a2 / 2 + tid; j < b2 / 2; j += nthr) {
            double2 s = reinterpret_cast<const double2*>(p[0])[j];
#pragma unroll
            for (int r = 1; r < GM_PEER_MAX; r++)
                if (r < world) {
                    const double2 v = reinterpret_cast<const double2*>(p[r])[j];
                    s.x += v.x;
                    s.y += v.y;
                }
#pragma unroll
            for (int r = 0; r < GM_PEER_MAX; r++)
                if (r < world) reinterpret_cast<double2*>(p[r])[j] = s;
            m = fmax(m, fmax(s.x, s.y));
        }
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

extern "C" int gm_plan_ipc_handle(gm_plan* p, void* out) {
    if (!p || !out) return set_err(GM_ERR_ARG, "null argument");
    if (!p->d_values) return set_err(GM_ERR_ARG, "plan has no scene");
    CK(cudaSetDevice(p->device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, p->d_values));
    memcpy(out, &h, sizeof(h));
    return GM_OK;
}

extern "C" int gm_plan_open_peers(gm_plan* p, int rank, int world, const void* handles) {
    if (!p || !handles || world < 1 || rank < 0 || rank >= world) return set_err(GM_ERR_ARG, "bad peer arguments");
    CK(cudaSetDevice(p->device));
    const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
    if (world != p->peer_world || rank != p->peer_rank) {  // new group: close every mapping
        for (int r = 0; r < p->peer_world; r++)
            if (r != p->peer_rank && p->peer_ptr[r]) CK(cudaIpcCloseMemHandle(p->peer_ptr[r]));
        p->peer_handle.assign(world, cudaIpcMemHandle_t{});
        p->peer_ptr.assign(world, nullptr);
        p->peer_world = world;
        p->peer_rank = rank;
        int rc;
        if ((rc = dev_alloc(&p->d_peer_ptr, (size_t)world))) return rc;
    }
    for (int r = 0; r < world; r++) {
        if (r == rank) {
            p->peer_ptr[r] = p->d_values;
            continue;
        }
        if (p->peer_ptr[r] && !memcmp(&p->peer_handle[r], &hs[r], sizeof(cudaIpcMemHandle_t))) continue;
        if (p->peer_ptr[r]) CK(cudaIpcCloseMemHandle(p->peer_ptr[r]));
        p->peer_ptr[r] = nullptr;
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, hs[r], cudaIpcMemLazyEnablePeerAccess));
        p->peer_ptr[r] = static_cast<double*>(ptr);
        p->peer_handle[r] = hs[r];
    }
    CK(cudaMemcpy(p->d_peer_ptr, p->peer_ptr.data(), sizeof(double*) * world, cudaMemcpyHostToDevice));
    return GM_OK;
}

extern "C" int gm_plan_reduce_peers(gm_plan* p, double* slice_max, float* device_ms) {
    if (!p || !slice_max) return set_err(GM_ERR_ARG, "null argument");
    if (p->peer_world < 1 || !p->d_peer_ptr) return set_err(GM_ERR_ARG, "gm_plan_open_peers first");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    const int64_t base = p->N / p->peer_world, extra = p->N % p->peer_world, r = p->peer_rank;
    const int64_t a = r * base + std::min<int64_t>(r, extra), b = a + base + (r < extra ? 1 : 0);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaMemsetAsync(p->d_max, 0, sizeof(unsigned long long), s));
    CK(cudaEventRecord(e0, s));
    if (b > a && p->peer_world <= GM_PEER_MAX)
        k_reduce_peers_vec<<<std::min<int64_t>(blocks_for((b - a + 1) / 2, 256), (int64_t)p->sms * 8), 256, 0, s>>>(
            p->d_peer_ptr, p->peer_world, a, b, p->d_max);
    else if (b > a)
        k_reduce_peers<<<std::min<int64_t>(blocks_for(b - a, 256), (int64_t)p->sms * 8), 256, 0, s>>>(
            p->d_peer_ptr, p->peer_world, a, b, p->d_max);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, s));
    unsigned long long bits = 0;
    CK(cudaMemcpyAsync(&bits, p->d_max, sizeof(bits), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (device_ms) *device_ms = ms;
    memcpy(slice_max, &bits, sizeof(double));
    return GM_OK;
}

// Copy the plan's values to host (raw) and optionally values / gmax.
// Device -> caller's (pageable) host buffer.  Large maps stream through two
// pinned 8 MiB stages: chunk c+1 is in flight over PCIe while the host threads
// copy chunk c into the destination (and take its first-touch page faults), so
// the read-back runs at pinned-DMA speed instead of the driver's pageable path.
extern "C" void gm_host_copy(void* dst, const void* src, size_t bytes, int threads);  // gm_host.cpp
#define GM_STAGE ((size_t)8 << 20)
static int copy_out(gm_plan* p, const double* d_src, double* dst, cudaStream_t s) {
    const size_t bytes = sizeof(double) * (size_t)p->N;
    if (bytes <= GM_STAGE) {
        CK(cudaMemcpyAsync(dst, d_src, bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return GM_OK;
    }
    if (!p->h_stage) {
        CK(cudaMallocHost(&p->h_stage, 2 * GM_STAGE));
        for (int k = 0; k < 2; k++) CK(cudaEventCreateWithFlags(&p->stage_ev[k], cudaEventDisableTiming));
    }
    const int64_t nch = (int64_t)((bytes + GM_STAGE - 1) / GM_STAGE);
    auto len = [&](int64_t c) { return std::min(GM_STAGE, bytes - (size_t)c * GM_STAGE); };
    for (int64_t c = 0; c < std::min<int64_t>(nch, 2); c++) {
        CK(cudaMemcpyAsync(p->h_stage + (c & 1) * GM_STAGE, (const char*)d_src + c * GM_STAGE, len(c),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(p->stage_ev[c & 1], s));
    }
    for (int64_t c = 0; c < nch; c++) {
        CK(cudaEventSynchronize(p->stage_ev[c & 1]));
        gm_host_copy((char*)dst + c * GM_STAGE, p->h_stage + (c & 1) * GM_STAGE, len(c), p->host_threads);
        if (c + 2 < nch) {
            CK(cudaMemcpyAsync(p->h_stage + (c & 1) * GM_STAGE, (const char*)d_src + (c + 2) * GM_STAGE, len(c + 2),
                               cudaMemcpyDeviceToHost, s));
            CK(cudaEventRecord(p->stage_ev[c & 1], s));
        }
    }
    return GM_OK;
}

extern "C" int gm_plan_read(gm_plan* p, double* raw, double* normalized, double gmax) {
    if (!p) return set_err(GM_ERR_ARG, "null plan");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    if (p->N == 0) return GM_OK;
    int rc;
    if (raw && (rc = copy_out(p, p->d_values, raw, s))) return rc;
    if (normalized) {
        double* tmp = nullptr;
        CK(cudaMallocAsync(&tmp, sizeof(double) * p->N, s));
        k_normalize<<<std::min<int64_t>(blocks_for(p->N, 256), (int64_t)p->sms * 8), 256, 0, s>>>(p->d_values, p->N, gmax, tmp);
        rc = copy_out(p, tmp, normalized, s);
        CK(cudaFreeAsync(tmp, s));
        if (rc) return rc;
    }
    CK(cudaStreamSynchronize(s));
    return GM_OK;
}

// Overwrite the plan's device values from host (e.g. to resume a partial map).
extern "C" int gm_plan_write(gm_plan* p, const double* raw) {
    if (!p || !raw) return set_err(GM_ERR_ARG, "null argument");
    CK(cudaSetDevice(p->device));
    if (p->N == 0) return GM_OK;
    CK(cudaMemcpyAsync(p->d_values, raw, sizeof(double) * p->N, cudaMemcpyHostToDevice, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    return GM_OK;
}

// Block until the plan's stream is idle (for device-resident callers).
extern "C" int gm_plan_sync(gm_plan* p) {
    if (!p) return set_err(GM_ERR_ARG, "null plan");
    CK(cudaSetDevice(p->device));
    CK(cudaStreamSynchronize(p->stream));
    return GM_OK;
}

// ------------------------------------------------------- stage 1 entries

// build_sampled_mesh (geometry.py:305-320) on the GPU.
extern "C" int gm_layout(int device, const double* tri_local, int64_t T, double k, int64_t* res, int64_t* counts,
                         int64_t* offsets, int64_t* total) {
    if (T < 0 || !total) return set_err(GM_ERR_ARG, "bad arguments");
    if (!(k > 0.0)) return set_err(GM_ERR_ARG, "sampling density k must be > 0");
    if (T == 0) {
        *total = 0;
        return GM_OK;
    }
    int rc = use_device(device);
    if (rc) return rc;
    DevScratch scratch;
    double* d_tri = nullptr;
    int64_t *d_res = nullptr, *d_cnt = nullptr, *d_off = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CK(scratch.alloc(&d_tri, sizeof(double) * 9 * T));
    CK(scratch.alloc(&d_res, sizeof(int64_t) * T));
    CK(scratch.alloc(&d_cnt, sizeof(int64_t) * (T + 1)));
    CK(scratch.alloc(&d_off, sizeof(int64_t) * (T + 1)));
    CK(cudaMemcpy(d_tri, tri_local, sizeof(double) * 9 * T, cudaMemcpyHostToDevice));
    k_layout<<<blocks_for(T, 256), 256>>>(d_tri, T, 8.0 * k, nullptr, d_res, d_cnt);
    CK(cudaMemset(d_cnt + T, 0, sizeof(int64_t)));
    cub::DeviceScan::ExclusiveSum(nullptr, tb, d_cnt, d_off, T + 1);
    CK(scratch.alloc(&tmp, tb));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, d_cnt, d_off, T + 1));
    if (res) CK(cudaMemcpy(res, d_res, sizeof(int64_t) * T, cudaMemcpyDeviceToHost));
    if (counts) CK(cudaMemcpy(counts, d_cnt, sizeof(int64_t) * T, cudaMemcpyDeviceToHost));
    if (offsets) CK(cudaMemcpy(offsets, d_off, sizeof(int64_t) * T, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(total, d_off + T, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CK(cudaGetLastError());
    return GM_OK;
}

// sample_positions_local (geometry.py:331-346), optionally followed by
// Transform.apply (xform = [t(3), q(4), s(3)] or NULL).  out is N x 3.
extern "C" int gm_sample_positions(int device, const double* tri_local, int64_t T, const int64_t* res,
                                   const int64_t* offsets, int64_t N, const double* xform, double* out) {
    if (T < 0 || N < 0) return set_err(GM_ERR_ARG, "bad arguments");
    if (N == 0 || T == 0) return GM_OK;
    int rc = use_device(device);
    if (rc) return rc;
    DevScratch scratch;
    double *d_tri = nullptr, *d_out = nullptr, *d_M = nullptr;
    int64_t *d_res = nullptr, *d_off = nullptr;
    CK(scratch.alloc(&d_tri, sizeof(double) * 9 * T));
    CK(scratch.alloc(&d_res, sizeof(int64_t) * T));
    CK(scratch.alloc(&d_off, sizeof(int64_t) * T));
    CK(scratch.alloc(&d_out, sizeof(double) * 3 * N));
    CK(cudaMemcpy(d_tri, tri_local, sizeof(double) * 9 * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_res, res, sizeof(int64_t) * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_off, offsets, sizeof(int64_t) * T, cudaMemcpyHostToDevice));
    if (xform) {
        double Mt[12];
        xform_matrix(xform, Mt, Mt + 9);
        CK(scratch.alloc(&d_M, sizeof(double) * 12));
        CK(cudaMemcpy(d_M, Mt, sizeof(double) * 12, cudaMemcpyHostToDevice));
    }
    k_positions<<<blocks_for(N, 256), 256>>>(d_tri, T, d_res, d_off, N, d_M, d_M ? d_M + 9 : nullptr, d_out,
                                            nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d_out, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost));
    return GM_OK;
}

// normalize (density.py:230-244) of a host vector on the GPU.
extern "C" int gm_normalize(int device, const double* values, int64_t n, double gmax, double* out) {
    if (n < 0) return set_err(GM_ERR_ARG, "bad length");
    if (n == 0) return GM_OK;
    int rc = use_device(device);
    if (rc) return rc;
    DevScratch scratch;
    double *d_in = nullptr, *d_out = nullptr;
    CK(scratch.alloc(&d_in, sizeof(double) * n));
    CK(scratch.alloc(&d_out, sizeof(double) * n));
    CK(cudaMemcpy(d_in, values, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_normalize<<<blocks_for(n, 256), 256>>>(d_in, n, gmax, d_out);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost));
    return GM_OK;
}

// ----------------------------------------------------- kernel-seam ports

// Per-fixation setup table (exposes the host setup for parity tests).
extern "C" int gm_fixation_setup(const double* fx, int64_t F, double theta, int filtering, int res,
                                 GmFixExact* ex, GmFixCull* cull, int64_t* bad_fixation) {
    GmSetupConsts c;
    gm_setup_consts(theta, filtering, res, res, &c);
    std::vector<GmFixCull> tmp;
    if (!cull) {
        tmp.resize(std::max<int64_t>(F, 1));
        cull = tmp.data();
    }
    int64_t bad = gm_setup_batch(fx, F, &c, ex, cull, 1);
    if (bad >= 0) {
        if (bad_fixation) *bad_fixation = bad;
        return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
    }
    return GM_OK;
}

// One fixation's setup under precomputed constants (accumulate_fixation's
// per-call InvalidFrustumError check): no allocation, no trig for the constants.
extern "C" int gm_fixation_check(const double* fx, const GmSetupConsts* c) {
    if (!fx || !c) return set_err(GM_ERR_ARG, "null argument");
    GmFixExact ex;
    GmFixCull cull;
    if (gm_setup_batch(fx, 1, c, &ex, &cull, 1) >= 0)
        return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
    return GM_OK;
}

// Full W x H rasterization of the plan's occluders under the camera record
// already in d_fix[0] / d_cull[0] (kernels.rasterize, kernels.py:140-192):
// k_tri_setup (cull per d_cull[0]; cos_t = -3 disables it) into a segment
// grown until it fits, coarse bins, every texel marked, k_texels.  The depth
// is left in d_depth (+inf where nothing is drawn); with attrs, d_key holds
// the rasterization-order key of the triangle that wrote each texel (-1 none).
static int raster_pass(gm_plan* p, int W, int H, bool attrs) {
    cudaStream_t s = p->stream;
    int rc = ensure_batch(p, 1, W, H, std::max<int64_t>(p->cap_seg, 4096));
    if (rc) return rc;
    if (attrs && (int64_t)W * H > p->cap_key) {
        cudaFree(p->d_key);
        p->d_key = nullptr;
        if ((rc = dev_alloc(&p->d_key, (size_t)W * H))) return rc;
        p->cap_key = (int64_t)W * H;
    }
    const int wwords = (W + 31) / 32;
    for (int attempt = 0; attempt < 16; attempt++) {
        k_set_i64<<<1, 1, 0, s>>>(p->d_fail, LLONG_MAX);
        CK(cudaMemsetAsync(p->d_maxcount, 0, sizeof(int), s));
        CK(cudaMemsetAsync(p->d_count, 0, sizeof(int), s));
        TriStore ts{p->d_tris, p->d_t32, p->d_bbox, p->d_count, p->cap_seg, p->d_fail, p->d_maxcount, p->d_ntris};
        if (p->n_clu > 0) {
            dim3 grid(blocks_for((p->n_clu + 31) / 32, TS_WARPS), 1);
            k_tri_setup<<<grid, TS_WARPS * 32, 0, s>>>(p->d_tw, p->T, p->d_tsph, p->d_csph, p->n_clu, p->d_fix, p->d_cull, W,
                                             H, ts, 0);
        }
        long long failed = LLONG_MAX;
        int maxcount = 0;
        CK(cudaMemcpyAsync(&failed, p->d_fail, sizeof(failed), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&maxcount, p->d_maxcount, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (failed == LLONG_MAX) break;
        int64_t want = std::max<int64_t>(2 * p->cap_seg, (int64_t)maxcount + maxcount / 4 + 64);
        p->cap_seg = 0;
        if ((rc = ensure_batch(p, 1, W, H, want))) return rc;
        if (attempt == 15) return set_err(GM_ERR_OOM, "screen-triangle segment kept overflowing");
    }
    TriStore ts{p->d_tris, p->d_t32, p->d_bbox, p->d_count, p->cap_seg, p->d_fail, p->d_maxcount, p->d_ntris};
    const int tiles_x = (W + TW - 1) / TW, tiles_y = (H + TH_FULL - 1) / TH_FULL;
    DepthView dv{p->d_depth, p->d_mask, W, H, wwords, nullptr, p->d_vbuf, attrs ? p->d_key : nullptr};
    dv.crowd_wide = 1;  // every texel is marked: long tiles, many rounds each
    dv.th_shift = 4;
    k_mark_all<<<blocks_for((int64_t)H * wwords, 256), 256, 0, s>>>(p->d_mask, W, H, wwords);
    CoarseBins cbins = coarse_bins(p, W, H);
    k_coarse<<<1, 256, 0, s>>>(ts, cbins, p->d_fail, 0, nullptr);
    const int64_t items = (int64_t)tiles_x * tiles_y;
    return attrs ? launch_texels<true, false, true>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, p->d_fix, 0)
                 : launch_texels<false, false, true>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, p->d_fix, 0);
}

// kernels.rasterize for the plan's occluders under fixation `fx` (18 floats):
// the whole res x res depth buffer (+inf where nothing is drawn), evaluated by
// the production texel kernel (k_texels) with every texel marked.  When
// no_cull != 0 the occluder cone cull is disabled (every triangle is projected).
extern "C" int gm_plan_depth_buffer(gm_plan* p, const double* fx, double theta, int filtering, int res, int no_cull,
                                    double* depth) {
    if (!p || !fx || !depth || res < 1 || res > 65535) return set_err(GM_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(p->device));
    GmSetupConsts c;
    gm_setup_consts(theta, filtering, res, res, &c);
    int rc = ensure_batch(p, 1, res, res, std::max<int64_t>(p->cap_seg, 4096));
    if (rc) return rc;
    cudaStream_t s = p->stream;
    CK(cudaEventSynchronize(p->h_ev[0]));
    int64_t bad = gm_setup_batch(fx, 1, &c, p->h_fix[0], p->h_cull[0], 1);
    if (bad >= 0) return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
    if (no_cull) p->h_cull[0][0].cos_t = -3.0f;  // sphere_visible: no culling at all
    CK(cudaMemcpyAsync(p->d_fix, p->h_fix[0], sizeof(GmFixExact), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(p->d_cull, p->h_cull[0], sizeof(GmFixCull), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(p->h_ev[0], s));
    if ((rc = raster_pass(p, res, res, false))) return rc;
    CK(cudaMemcpyAsync(depth, p->d_depth, sizeof(double) * res * res, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return GM_OK;
}

#include "gm_raster.cuh"

// The NDC-filtered candidate lists (kernels.py:302-319) of F fixations over
// the plan's samples.  out is F x cap (int64, unsorted within a fixation),
// counts F.  Returns GM_ERR_ARG-free success even if a count exceeds cap
// (only the first cap indices are stored).
extern "C" int gm_plan_candidates(gm_plan* p, const double* fx, int64_t F, double theta, int filtering, int res,
                                  int64_t* out, int64_t cap, int64_t* counts) {
    if (!p || (F > 0 && (!fx || !out || !counts)) || cap < 0) return set_err(GM_ERR_ARG, "bad arguments");
    if (F == 0) return GM_OK;
    CK(cudaSetDevice(p->device));
    GmSetupConsts c;
    gm_setup_consts(theta, filtering, res, res, &c);
    std::vector<GmFixExact> ex(F);
    std::vector<GmFixCull> cu(F);
    int64_t bad = gm_setup_batch(fx, F, &c, ex.data(), cu.data(), 1);
    if (bad >= 0) return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
    cudaStream_t s = p->stream;
    GmFixExact* d_ex = nullptr;
    int64_t* d_out = nullptr;
    unsigned long long* d_cnt = nullptr;
    CK(cudaMallocAsync(&d_ex, sizeof(GmFixExact) * F, s));
    CK(cudaMallocAsync(&d_out, sizeof(int64_t) * std::max<int64_t>(1, F * cap), s));
    CK(cudaMallocAsync(&d_cnt, sizeof(unsigned long long) * F, s));
    CK(cudaMemcpyAsync(d_ex, ex.data(), sizeof(GmFixExact) * F, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * F, s));
    if (p->N > 0) {
        dim3 grid((unsigned)std::min<int64_t>((p->n_chunks + 7) / 8, 4096), (unsigned)F);
        k_candidates<<<grid, 256, 0, s>>>(p->d_px, p->d_py, p->d_pz, p->N, d_ex, (int)F, d_out, cap, d_cnt);
    }
    CK(cudaGetLastError());
    if (F * cap > 0) CK(cudaMemcpyAsync(out, d_out, sizeof(int64_t) * F * cap, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(counts, d_cnt, sizeof(int64_t) * F, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d_ex, s));
    CK(cudaFreeAsync(d_out, s));
    CK(cudaFreeAsync(d_cnt, s));
    CK(cudaStreamSynchronize(s));
    return GM_OK;
}

// Read back the plan's world-space sample positions (SoA -> N x 3).
extern "C" int gm_plan_positions(gm_plan* p, double* out) {
    if (!p || !out) return set_err(GM_ERR_ARG, "null argument");
    CK(cudaSetDevice(p->device));
    if (p->N == 0) return GM_OK;
    std::vector<double> x(p->N), y(p->N), z(p->N);
    CK(cudaMemcpy(x.data(), p->d_px, sizeof(double) * p->N, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(y.data(), p->d_py, sizeof(double) * p->N, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(z.data(), p->d_pz, sizeof(double) * p->N, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < p->N; i++) {
        out[3 * i] = x[i];
        out[3 * i + 1] = y[i];
        out[3 * i + 2] = z[i];
    }
    return GM_OK;
}

extern "C" int gm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

// ------------------------------------------------ measured SIMT peaks
// Roofline denominators for bench.py: FP64 / FP32 FMA throughput of this GPU,
// measured (MEASURED_PEAKS.json only carries HBM and tensor-core figures).
// Every thread runs 8 independent FMA chains (latency hidden by ILP and by
// the 8 resident 256-thread CTAs per SM); 2 flops per FMA.
template <typename T>
__global__ void __launch_bounds__(256) k_peak_fma(T* out, int iters, T m, T c) {
    T a[8];
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = (T)(threadIdx.x + i) * (T)1e-3;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fma(a[i], m, c);
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += a[i];
    if (s == (T)-1.2345) out[threadIdx.x] = s;  // never true; keeps the chains live
}

// FMA throughput in TFLOP/s (fp64 != 0: float64, else float32), best of 3
// timed launches after a warm-up, CUDA events on a private stream.
extern "C" int gm_peak_flops(int device, int fp64, double* tflops) {
    if (!tflops) return set_err(GM_ERR_ARG, "null argument");
    int rc = use_device(device);
    if (rc) return rc;
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DevScratch scratch;
    void* out = nullptr;
    CK(scratch.alloc(&out, 256 * sizeof(double)));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, iters = fp64 ? 8192 : 32768;
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0, s);
        if (fp64)
            k_peak_fma<double><<<blocks, 256, 0, s>>>((double*)out, iters, 0.999999, 1e-7);
        else
            k_peak_fma<float><<<blocks, 256, 0, s>>>((float*)out, iters, 0.9999f, 1e-4f);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    if (err != cudaSuccess) return set_err(GM_ERR_CUDA, cudaGetErrorString(err));
    const double flops = 2.0 * 8.0 * (double)iters * (double)blocks * 256.0;
    *tflops = flops / (best * 1e-3) / 1e12;
    return GM_OK;
}

// Self-check counters (GM_CHK_* order, GM_CHK_N x uint64) accumulated since the
// last reset by a GM_CHECK build of the extension; all zero in production
// builds (nothing increments them).  is_check_build: 1 for a GM_CHECK build.
extern "C" int gm_plan_check(gm_plan* p, unsigned long long* out, int reset, int* is_check_build) {
    if (!p) return set_err(GM_ERR_ARG, "null plan");
    CK(cudaSetDevice(p->device));
    CK(cudaDeviceSynchronize());
    if (out) CK(cudaMemcpy(out, p->d_check, GM_CHK_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (reset) CK(cudaMemset(p->d_check, 0, GM_CHK_N * sizeof(unsigned long long)));
#ifdef GM_CHECK
    if (is_check_build) *is_check_build = 1;
#else
    if (is_check_build) *is_check_build = 0;
#endif
    return GM_OK;
}

// Restart the per-fixation screen-triangle segments at `cap` entries (testing
// hook for the overflow / resume path of run_batches; the segments still grow
// on demand).  The plan's batch buffers are reallocated on the next run.
extern "C" int gm_plan_set_segment_capacity(gm_plan* p, int64_t cap) {
    if (!p || cap < 1) return set_err(GM_ERR_ARG, "bad segment capacity");
    CK(cudaSetDevice(p->device));
    CK(cudaDeviceSynchronize());
    for (int k = 0; k < GM_NSETS; k++) {
        if (k) swap_batch_bufs(p, k);
        cudaFree(p->d_tris); cudaFree(p->d_t32); cudaFree(p->d_bbox);
        p->d_tris = nullptr; p->d_t32 = nullptr; p->d_bbox = nullptr;
        p->cap_seg = 0;
        p->cap_seg_B = 0;
        if (k) swap_batch_bufs(p, k);
    }
    p->seg_init = cap;
    return GM_OK;
}
