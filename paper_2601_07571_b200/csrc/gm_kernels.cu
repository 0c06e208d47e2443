// gm_kernels.cu -- sm_100a kernels and the C-ABI of the B200 density-map path.
//
// Path and where each piece lives:
//   a1-a6  sampling: k_layout (Heron area -> r -> count), CUB scan (offsets),
//          k_positions (index -> row/col -> barycentric -> world, FMA-chain
//          transform like OpenBLAS), k_world_tris
//   a8-a10 per-fixation setup: host, gm_setup.cpp (glibc trig, bit-exact)
//   a11-a12 occluders: k_tri_setup (conservative cone cull, exact camera
//          transform + near clip + projection + _raster_tri setup) into
//          per-fixation screen-triangle segments
//   a13-a15 k_samples<true>: sample-major, one warp per 32-sample chunk,
//          fixation culling by warp ballot, exact NDC filter + 4-sigma cone,
//          marks the <= 9 texels depth_match will read;
//          k_texels: fixation-major per 64x64 tile, evaluates only marked
//          texels (min over covering screen triangles, reference pixel
//          arithmetic) from shared-memory sub-bins;
//          k_samples<false>: depth_match + Gaussian, accumulated in log order
//   a16    k_max / k_normalize
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
// launch bounds of the hot kernels; -DTX_MINB=n etc. (build variants) cap
// their registers for n CTAs per SM
#ifdef TX_MINB
#define TX_BOUNDS __launch_bounds__(TX_MAX_THREADS, TX_MINB)
#else
#define TX_BOUNDS __launch_bounds__(TX_MAX_THREADS)
#endif
#ifdef KS_MINB
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
struct __align__(16) TriF32 {
    float a[3], b[3], c[3], tol[3];  // e_i = a x + b y + c
    float A, B, C, tolw;             // inverse depth
    float inv_minw;                  // >= every inverse depth the triangle writes
    int ox, oy;                      // frame origin = bbox corner (pixels)
    uint32_t bx, by;                 // bbox x0 | x1 << 16, y0 | y1 << 16
    int gidx;                        // index of the float64 record in the fixation's segment
    int pad[2];
};  // 96 B

__device__ __forceinline__ void make_tri_f32(const GmScreenTri& T, int gidx, TriF32& o) {
    const double ox = T.x0, oy = T.y0;
    const double sx[3] = {T.sx0 - ox, T.sx1 - ox, T.sx2 - ox}, sy[3] = {T.sy0 - oy, T.sy1 - oy, T.sy2 - oy};
    const double iw[3] = {T.iw0, T.iw1, T.iw2};
    const double xmax = (double)(T.x1 - T.x0 + 1), ymax = (double)(T.y1 - T.y0 + 1);
    double A = 0.0, B = 0.0, C = 0.0, Aab = 0.0, Bab = 0.0, Cab = 0.0;
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
        o.tol[i] = (float)(4.8e-7 * mag + 1e-30);
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
    o.ox = T.x0;
    o.oy = T.y0;
    o.bx = (uint32_t)T.x0 | ((uint32_t)T.x1 << 16);
    o.by = (uint32_t)T.y0 | ((uint32_t)T.y1 << 16);
    o.gidx = gidx;
    o.pad[0] = o.pad[1] = 0;
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
__global__ void __launch_bounds__(256) k_tri_setup(const double* __restrict__ tw, int64_t T,
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
            atomicAdd(ts.total, (unsigned long long)total);
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
                make_tri_f32(out[q], at + q, ts.t32[(int64_t)f * ts.cap_seg + at + q]);
                segb[at + q] = make_uint2((uint32_t)out[q].x0 | ((uint32_t)out[q].x1 << 16),
                                          (uint32_t)out[q].y0 | ((uint32_t)out[q].y1 << 16));
            }
        }
    }
}

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
#define CB_SHIFT 6  // coarse bins of 64 x 64 pixels (k_texels tiles are 32 x 16)
#endif
#ifndef CB_ITEMS_PER_TRI
#define CB_ITEMS_PER_TRI 4  // coarse-bin list capacity per screen triangle (more: scan the whole list)
#endif
struct CoarseBins {
    int* items;   // [B][cap_items]
    int* off;     // [B][GM_MAX_CBINS + 1]
    int* ovf;     // [B]
    int64_t cap_items;
    int shift, ncx, ncy;
};

__global__ void __launch_bounds__(256) k_coarse(TriStore ts, CoarseBins cb, const long long* __restrict__ fail,
                                                long long b0) {
    __shared__ int s_cnt[GM_MAX_CBINS];
    __shared__ int s_off[GM_MAX_CBINS + 1];
    if (*fail <= b0) return;
    const int f = blockIdx.x;
    const int nbins = cb.ncx * cb.ncy;
    const int n = min(ts.count[f], (int)ts.cap_seg);
    const uint2* segb = ts.bbox + (int64_t)f * ts.cap_seg;
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint2 bb = segb[i];
        const int bx0 = (bb.x & 0xffff) >> cb.shift, bx1 = (bb.x >> 16) >> cb.shift;
        const int by0 = (bb.y & 0xffff) >> cb.shift, by1 = (bb.y >> 16) >> cb.shift;
        for (int by = by0; by <= by1; by++)
            for (int bx = bx0; bx <= bx1; bx++) atomicAdd(&s_cnt[by * cb.ncx + bx], 1);
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
    int* items = cb.items + (int64_t)f * cb.cap_items;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint2 bb = segb[i];
        const int bx0 = (bb.x & 0xffff) >> cb.shift, bx1 = (bb.x >> 16) >> cb.shift;
        const int by0 = (bb.y & 0xffff) >> cb.shift, by1 = (bb.y >> 16) >> cb.shift;
        for (int by = by0; by <= by1; by++)
            for (int bx = bx0; bx <= bx1; bx++) {
                const int b = by * cb.ncx + bx;
                items[s_off[b] + atomicAdd(&s_cnt[b], 1)] = i;
            }
    }
}

#define TW 32      // k_texels tile width (pixels) = warp lanes
#ifndef TH
#define TH 16      // k_texels tile height (pixels), a power of two <= 32
#endif

struct DepthView {
    double* depth;    // [B][H][W]: marked texels only
    uint32_t* mask;   // [B][H][wwords]: texels the depth tests will read
    int W, H, wwords;
    unsigned long long* stats;  // optional work counters (GM_STAT_*), nullptr = off
    float* vbuf;      // [B][H][W]: k_texels' inverse-depth bounds for tiles with many triangles
    int* key;         // [H][W] (ATTRS only): order key 2 t + fan of the triangle that wrote the texel
    int* crowd;       // work items deferred to k_texels<CROWDED> (nullptr: handle them in place)
    int* crowd_count; // [2]: deferred items, claimed items
};

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
    GM_STAT_TX_TILES = 10,   // k_texels work items with marked texels
    GM_STAT_TX_STAGED = 11,  // triangles staged per item (sum)
    GM_STAT_TX_LIST = 12,    // coarse-bin list entries scanned per item (sum)
    GM_STAT_TX_ITER = 13,    // warp iterations of the selection walk
    GM_STAT_TX_EDGE = 14,    // lane x triangle edge-function evaluations in the walk
    GM_STAT_N = 16
};
#define GM_FLAG_STATS 1
#define GM_FLAG_ONE_STREAM 2   // force batches onto one stream/buffer set
#define GM_FLAG_TWO_STREAMS 4  // force the two-stream batch pipeline
#ifndef GM_OVERLAP_MAX_TRIS
#define GM_OVERLAP_MAX_TRIS 400000  // default: overlap batches for scenes up to this many occluders
#endif
#define GM_STAT_STRIPES 128  // counter copies (summed by gm_plan_stats): keeps the stats pass free of atomic hot spots

// Warp-aggregated add of a per-lane count to stripe (block % GM_STAT_STRIPES)
// of counter idx.  Every lane of the warp must call it.
__device__ __forceinline__ void stat_add(unsigned long long* stats, int idx, unsigned long long v) {
    const unsigned lo = __reduce_add_sync(0xffffffffu, (unsigned)(v & 0xffffffffu));
    const unsigned hi = __reduce_add_sync(0xffffffffu, (unsigned)(v >> 32));
    if ((threadIdx.x & 31) == 0)
        atomicAdd(stats + (size_t)(blockIdx.x % GM_STAT_STRIPES) * GM_STAT_N + idx,
                  (unsigned long long)lo + ((unsigned long long)hi << 32));
}

// kernels.py:219-285 depth_match, reading the texels k_texels evaluated
// (the 3x3 block around rint(g), which contains the bilinear quad).
__device__ __forceinline__ bool depth_test(const DepthView& dv, int f, double gx, double gy, int bx0, int bx1,
                                           int by0, int by1, double d, double eps) {
    const int W = dv.W, H = dv.H;
    const double* dep = dv.depth + (int64_t)f * W * H;
    if (W > 1 && H > 1) {
        long long x0 = x86_i64(floor(gx));
        if (x0 < 0) x0 = 0;
        else if (x0 > W - 2) x0 = W - 2;
        long long y0 = x86_i64(floor(gy));
        if (y0 < 0) y0 = 0;
        else if (y0 > H - 2) y0 = H - 2;
        const double* r0 = dep + (int64_t)y0 * W + x0;
        double q00 = r0[0], q01 = r0[1], q10 = r0[W], q11 = r0[W + 1];
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
    for (int yy = by0; yy <= by1; yy++) {
        const double* row = dep + (int64_t)yy * W;
        for (int xx = bx0; xx <= bx1; xx++) {
            const double t = row[xx];
            if (isfinite(t)) {
                double diff = fabs(t - d);
                if (diff < best) best = diff;
            }
        }
    }
    return best <= eps;
}

// Sample-major pass over a batch of fixations (kernels.py:288-340).  A warp
// owns 32 consecutive samples; lane l tests fixation g+l against the chunk
// sphere, the ballot gives the fixations that can touch the chunk, and those
// are applied in log order.
//   MARK = true : set the mask bits of the 3x3 texel block depth_match reads
//                 for every candidate that passes the NDC filter and the cone.
//   MARK = false: depth_match on those texels and accumulate; the value slot
//                 lives in a register, so per-sample accumulation order is the
//                 reference's (density.py:223-226): deterministic, no atomics.
// The cone test (kernels.py:330-339) runs before depth_match (:326): every
// condition is conjunctive and side-effect free, so the contributing set and
// the weights are unchanged.
// Level 1 of the sample-side fixation cull, once per batch: warp per
// super-chunk (8 chunks = 256 consecutive samples), lane-parallel sphere tests
// against all fixations of the batch -> lvl1[sc][g] ballots and the number of
// fixations that can touch the super-chunk (the work estimate used to order
// the sample passes, heaviest first).
__global__ void __launch_bounds__(256) k_level1(const float4* __restrict__ supers, int64_t n_supers,
                                                const GmFixCull* __restrict__ culls, int B,
                                                uint32_t* __restrict__ lvl1, int* __restrict__ count,
                                                int* __restrict__ order, const long long* __restrict__ fail,
                                                long long b0) {
    const int lane = threadIdx.x & 31;
    const int64_t sc = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (sc >= n_supers) return;
    const int ngroups = (B + 31) >> 5;
    int total = 0;
    if (*fail > b0) {
        const float4 ssph = supers[sc];
        for (int g = 0; g < ngroups; g++) {
            const int myf = g * 32 + lane;
            const unsigned m = __ballot_sync(0xffffffffu, myf < B && sphere_visible(culls[myf], ssph, false));
            if (lane == 0) lvl1[sc * ngroups + g] = m;
            total += __popc(m);
        }
    }
    if (lane == 0) {
        count[sc] = total;
        order[sc] = (int)sc;
    }
}

// float32 view of a fixation for the marking pass, with a rigorous bound E on
// |camera coordinate in float32 - exact| over every sample of the plan.
struct __align__(16) GmFixF32 {
    float rot[9], trans[3], gaze[3];
    float p00, p11, p02, p12;
    float near_lo, far_hi;
    float E;        // absolute bound on the float32 camera-coordinate error (m)
    float sig16;    // 16 sigma^2 (ratio^2 <= 16 <=> |p x g|^2 <= 16 sigma^2 d1^2)
};  // 96 B

// float32 copies of the sample positions and max |coordinate| (bit-pattern
// atomicMax, exact for non-negative doubles)
__global__ void k_to_f32(const double* __restrict__ px, const double* __restrict__ py, const double* __restrict__ pz,
                         int64_t N, float* __restrict__ fx, float* __restrict__ fy, float* __restrict__ fz,
                         unsigned long long* __restrict__ amax) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double m = 0.0;
    if (i < N) {
        const double x = px[i], y = py[i], z = pz[i];
        fx[i] = (float)x;
        fy[i] = (float)y;
        fz[i] = (float)z;
        m = fmax(fabs(x), fmax(fabs(y), fabs(z)));
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(amax, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_fix32(const GmFixExact* __restrict__ ex, int nb, double pmax, double sigma,
                        GmFixF32* __restrict__ out) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nb) return;
    const GmFixExact& F = ex[f];
    GmFixF32 o;
    double tmax = 0.0;
    for (int i = 0; i < 9; i++) o.rot[i] = (float)F.rot[i];
    for (int i = 0; i < 3; i++) {
        o.trans[i] = (float)F.trans[i];
        o.gaze[i] = (float)F.gaze[i];
        tmax = fmax(tmax, fabs(F.trans[i]));
    }
    o.p00 = (float)F.p00;
    o.p11 = (float)F.p11;
    o.p02 = (float)F.p02;
    o.p12 = (float)F.p12;
    o.near_lo = (float)F.near_lo;
    o.far_hi = (float)F.far_hi;
    // fma chain of 3 products + translation, every operand rounded to float32:
    // |x32 - x| <= ~8 * 2^-24 * (3 pmax + |t|); E is > 2x that
    o.E = (float)(1e-6 * (3.0 * pmax + tmax) + 1e-30);
    o.sig16 = (float)(16.0 * sigma * sigma);
    out[f] = o;
}

// The marking pass: for every (sample, fixation) that can be a depth-test
// candidate (kernels.py:305-339: NDC crop filter and 4-sigma cone), set the
// mask bits of the texels depth_match may read.  Float32 with rigorous error
// bounds -- a superset of the exact candidates and of their exact 3x3 blocks
// (rint is monotone: the exact rint(g) lies in [rint(g32 - dg), rint(g32 + dg)])
// -- and the exact float64 computation for the rare lanes whose bounds are too
// loose (samples within ~E of the camera plane).  Marking extra texels only
// costs texel work; every texel an exact depth test reads is marked.
__global__ void KM_BOUNDS k_mark(const float* __restrict__ pxf, const float* __restrict__ pyf,
                                              const float* __restrict__ pzf, const double* __restrict__ px,
                                              const double* __restrict__ py, const double* __restrict__ pz,
                                              const float4* __restrict__ chunks, const uint32_t* __restrict__ lvl1,
                                              const int* __restrict__ order, int* __restrict__ work, int64_t N,
                                              int64_t n_chunks, int64_t n_supers, const GmFixExact* __restrict__ fixes,
                                              const GmFixF32* __restrict__ fix32, const GmFixCull* __restrict__ culls,
                                              int B, DepthView dv, double inv_sigma, uint32_t* __restrict__ cbits,
                                              const long long* __restrict__ fail, long long b0) {
    if (*fail <= b0) return;
    const int lane = threadIdx.x & 31;
    const int ngroups = (B + 31) >> 5;
    const int W = dv.W, H = dv.H;
    const float Wf = (float)W, Hf = (float)H;
    const float lo = -1.0f - (float)GM_NDC_SLACK, hi = 1.0f + (float)GM_NDC_SLACK;
    const int64_t n_items = n_supers * 8;
    for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(work, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= n_items) break;
        const int64_t sc = order[item >> 3];
        const int64_t ch = sc * 8 + (item & 7);
        if (ch >= n_chunks) continue;
        const unsigned l1 = lane < ngroups ? lvl1[sc * ngroups + lane] : 0u;
        if (!__any_sync(0xffffffffu, l1 != 0u)) continue;
        const int64_t i = ch * 32 + lane;
        const bool valid = i < N;
        float wx = 0.0f, wy = 0.0f, wz = 0.0f;
        if (valid) {
            wx = pxf[i];
            wy = pyf[i];
            wz = pzf[i];
        }
        const float4 sph = chunks[ch];
        for (int gi = 0; gi < ngroups; gi++) {
            const unsigned sm = __shfl_sync(0xffffffffu, l1, gi);
            if (!sm) continue;
            const int g = gi * 32;
            const bool pass = ((sm >> lane) & 1u) && sphere_visible(culls[g + lane], sph, false);
            unsigned mask = __ballot_sync(0xffffffffu, pass);
            unsigned my_bits = 0;  // fixations (bit j of group gi) for which this lane is a candidate
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                if (!valid) continue;
                const int f = g + j;
                const GmFixF32& Q = fix32[f];
                const float E = Q.E;
                const float x = __fmaf_rn(Q.rot[2], wz, __fmaf_rn(Q.rot[1], wy, __fmaf_rn(Q.rot[0], wx, Q.trans[0])));
                const float y = __fmaf_rn(Q.rot[5], wz, __fmaf_rn(Q.rot[4], wy, __fmaf_rn(Q.rot[3], wx, Q.trans[1])));
                const float z = __fmaf_rn(Q.rot[8], wz, __fmaf_rn(Q.rot[7], wy, __fmaf_rn(Q.rot[6], wx, Q.trans[2])));
                const float w = -z;
                if (w + E <= 0.0f) continue;                               // exact w <= 0
                if (w + E < Q.near_lo || w - E > Q.far_hi) continue;      // exact depth outside the slab
                const float wl = w - E;
                float bxlo, bxhi, bylo, byhi;  // range of the exact g (texel coordinates)
                bool exact = !(wl > 1e-3f * fabsf(w) + 1e-12f);
                if (!exact) {
                    // NDC (kernels.py:314-319) with bound dq on |q32 - q_exact|
                    const float nx = __fmaf_rn(Q.p00, x, Q.p02 * z), ny = __fmaf_rn(Q.p11, y, Q.p12 * z);
                    const float qx = nx / w, qy = ny / w;
                    const float en_x = (fabsf(Q.p00) + fabsf(Q.p02)) * E + 4e-7f * (fabsf(Q.p00 * x) + fabsf(Q.p02 * z));
                    const float en_y = (fabsf(Q.p11) + fabsf(Q.p12)) * E + 4e-7f * (fabsf(Q.p11 * y) + fabsf(Q.p12 * z));
                    const float dqx = (en_x + fabsf(qx) * E) / wl + 1e-6f * fabsf(qx) + 1e-7f;
                    const float dqy = (en_y + fabsf(qy) * E) / wl + 1e-6f * fabsf(qy) + 1e-7f;
                    if (qx + dqx < lo || qx - dqx > hi || qy + dqy < lo || qy - dqy > hi) continue;
                    // cone (kernels.py:330-339): d1 > 0 and ratio^2 <= 16
                    const float d1 = __fmaf_rn(x, Q.gaze[0], __fmaf_rn(y, Q.gaze[1], z * Q.gaze[2]));
                    const float ed1 = 2.0f * E + 4e-7f * (fabsf(x) + fabsf(y) + fabsf(z));
                    if (d1 + ed1 <= 0.0f) continue;
                    const float cx3 = y * Q.gaze[2] - z * Q.gaze[1], cy3 = z * Q.gaze[0] - x * Q.gaze[2];
                    const float cz3 = x * Q.gaze[1] - y * Q.gaze[0];
                    const float cr = sqrtf(__fmaf_rn(cx3, cx3, __fmaf_rn(cy3, cy3, cz3 * cz3)));
                    const float ecr = 3.0f * E + 1e-6f * (fabsf(x) + fabsf(y) + fabsf(z));
                    const float crl = cr - ecr, d1h = d1 + ed1;
                    if (crl > 0.0f && crl * crl > Q.sig16 * (1.0f + 1e-4f) * d1h * d1h) continue;
                    const float gx = (qx + 1.0f) * 0.5f * Wf - 0.5f, gy = (1.0f - qy) * 0.5f * Hf - 0.5f;
                    const float dgx = dqx * 0.5f * Wf + 1e-4f + 1e-6f * fabsf(gx);
                    const float dgy = dqy * 0.5f * Hf + 1e-4f + 1e-6f * fabsf(gy);
                    if (dgx > 2.0f || dgy > 2.0f) {
                        exact = true;
                    } else {
                        bxlo = gx - dgx;
                        bxhi = gx + dgx;
                        bylo = gy - dgy;
                        byhi = gy + dgy;
                    }
                }
                int cxlo, cxhi, cylo, cyhi;
                if (exact) {
                    // the exact float64 test of k_samples, for this lane only
                    const GmFixExact& F = fixes[f];
                    const double X = px[i], Y = py[i], Z = pz[i];
                    const double xx = F.rot[0] * X + F.rot[1] * Y + F.rot[2] * Z + F.trans[0];
                    const double yy = F.rot[3] * X + F.rot[4] * Y + F.rot[5] * Z + F.trans[1];
                    const double zz = F.rot[6] * X + F.rot[7] * Y + F.rot[8] * Z + F.trans[2];
                    const double ww = -zz;
                    if (ww <= 0.0 || ww < F.near_lo || ww > F.far_hi) continue;
                    const double ndx = (F.p00 * xx + F.p02 * zz) / ww, ndy = (F.p11 * yy + F.p12 * zz) / ww;
                    const double l = -1.0 - GM_NDC_SLACK, h = 1.0 + GM_NDC_SLACK;
                    if (ndx < l || ndx > h || ndy < l || ndy > h) continue;
                    const double d1 = xx * F.gaze[0] + yy * F.gaze[1] + zz * F.gaze[2];
                    if (d1 <= 0.0) continue;
                    double d2sq = xx * xx + yy * yy + zz * zz - d1 * d1;
                    if (d2sq < 0.0) d2sq = 0.0;
                    if (d2sq * inv_sigma * inv_sigma / (d1 * d1) > 16.0) continue;
                    const double gxe = (ndx + 1.0) * 0.5 * (double)W - 0.5, gye = (1.0 - ndy) * 0.5 * (double)H - 0.5;
                    long long rx = x86_i64(rint(gxe)), ry = x86_i64(rint(gye));
                    cxlo = cxhi = (int)max(min(rx, (long long)W - 1), 0LL);
                    cylo = cyhi = (int)max(min(ry, (long long)H - 1), 0LL);
                } else {
                    cxlo = (int)fminf(fmaxf(rintf(bxlo), 0.0f), (float)(W - 1));
                    cxhi = (int)fminf(fmaxf(rintf(bxhi), 0.0f), (float)(W - 1));
                    cylo = (int)fminf(fmaxf(rintf(bylo), 0.0f), (float)(H - 1));
                    cyhi = (int)fminf(fmaxf(rintf(byhi), 0.0f), (float)(H - 1));
                }
                const int bx0 = max(cxlo - 1, 0), bx1 = min(cxhi + 1, W - 1);
                const int by0 = max(cylo - 1, 0), by1 = min(cyhi + 1, H - 1);
                my_bits |= 1u << j;
                uint32_t* m = dv.mask + (int64_t)f * H * dv.wwords;
                const unsigned long long bits = ((1ull << (bx1 - bx0 + 1)) - 1ull) << (bx0 & 31);
                const int w0 = bx0 >> 5;
                for (int yy = by0; yy <= by1; yy++) {
                    uint32_t* row = m + (int64_t)yy * dv.wwords + w0;
                    atomicOr(row, (uint32_t)bits);
                    if (bits >> 32) atomicOr(row + 1, (uint32_t)(bits >> 32));
                }
            }
            // level 3 for the accumulation pass: the fixations of this group with at
            // least one (float32-superset) candidate in this chunk
            const unsigned word = __reduce_or_sync(0xffffffffu, my_bits);
            if (lane == 0) cbits[ch * 32 + gi] = word;
        }
    }
}

template <bool STATS>
__global__ void KS_BOUNDS k_samples(const double* __restrict__ px, const double* __restrict__ py,
                                                 const double* __restrict__ pz, const float4* __restrict__ chunks,
                                                 const uint32_t* __restrict__ lvl1, const int* __restrict__ order,
                                                 int* __restrict__ work, int64_t N, int64_t n_chunks,
                                                 int64_t n_supers, const GmFixExact* __restrict__ fixes,
                                                 const GmFixCull* __restrict__ culls, int B, DepthView dv,
                                                 double inv_sigma, double eps_abs, double eps_rel,
                                                 double* __restrict__ values, const uint32_t* __restrict__ cbits,
                                                 const long long* __restrict__ fail, long long b0) {
    if (*fail <= b0) return;  // this batch overflowed the triangle store: the host redoes it
    const int lane = threadIdx.x & 31;
    const int ngroups = (B + 31) >> 5;  // <= 32 (B <= GM_MAX_BATCH)
    const int W = dv.W, H = dv.H;
    const double Wd = (double)W, Hd = (double)H;
    const double lo = -1.0 - GM_NDC_SLACK, hi = 1.0 + GM_NDC_SLACK;
    const int64_t n_items = n_supers * 8;
    unsigned c_l1 = 0, c_l2 = 0, c_exact = 0, c_ndc = 0, c_cand = 0, c_vis = 0;
    // persistent warps; items = chunks of the super-chunks in descending-work
    // order (k_level1 + radix sort), claimed one at a time
    for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(work, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= n_items) break;
        const int64_t sc = order[item >> 3];
        const int64_t ch = sc * 8 + (item & 7);
        if (ch >= n_chunks) continue;
        const unsigned l1 = lane < ngroups ? lvl1[sc * ngroups + lane] : 0u;  // lane g: group g
        if (STATS) c_l1 += 1;
        if (!__any_sync(0xffffffffu, l1 != 0u)) continue;
        {
        const int64_t i = ch * 32 + lane;
        const bool valid = i < N;
        double wx = 0.0, wy = 0.0, wz = 0.0, v = 0.0;
        if (valid) {
            wx = px[i];
            wy = py[i];
            wz = pz[i];
            v = values[i];
        }
        for (int gi = 0; gi < ngroups; gi++) {
            const unsigned sm = __shfl_sync(0xffffffffu, l1, gi);
            if (!sm) continue;
            const int g = gi * 32;
            // levels 2 + 3 (k_mark): the fixations of this group with a candidate in the chunk
            if (STATS) c_l2 += (sm >> lane) & 1u;
            unsigned mask = cbits[ch * 32 + gi];
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                if (!valid) continue;
                const int f = g + j;
                const GmFixExact& F = fixes[f];
                if (STATS) c_exact++;
                // kernels.py:305-319
                double x = F.rot[0] * wx + F.rot[1] * wy + F.rot[2] * wz + F.trans[0];
                double y = F.rot[3] * wx + F.rot[4] * wy + F.rot[5] * wz + F.trans[1];
                double z = F.rot[6] * wx + F.rot[7] * wy + F.rot[8] * wz + F.trans[2];
                double w = -z;
                if (w <= 0.0) continue;
                double d = w;
                if (d < F.near_lo || d > F.far_hi) continue;
                double ndc_x = (F.p00 * x + F.p02 * z) / w;
                double ndc_y = (F.p11 * y + F.p12 * z) / w;
                if (ndc_x < lo || ndc_x > hi) continue;
                if (ndc_y < lo || ndc_y > hi) continue;
                if (STATS) c_ndc++;
                // kernels.py:330-339 (moved before the depth test)
                double d1 = x * F.gaze[0] + y * F.gaze[1] + z * F.gaze[2];
                if (d1 <= 0.0) continue;
                double d2sq = x * x + y * y + z * z - d1 * d1;
                if (d2sq < 0.0) d2sq = 0.0;
                double ratio_sq = d2sq * inv_sigma * inv_sigma / (d1 * d1);
                if (ratio_sq > 16.0) continue;
                if (STATS) c_cand++;
                // texel coordinates (kernels.py:327, :231-232, :267-276)
                double gx = (ndc_x + 1.0) * 0.5 * Wd - 0.5;
                double gy = (1.0 - ndc_y) * 0.5 * Hd - 0.5;
                long long cx = x86_i64(rint(gx));
                if (cx < 0) cx = 0;
                else if (cx > W - 1) cx = W - 1;
                long long cy = x86_i64(rint(gy));
                if (cy < 0) cy = 0;
                else if (cy > H - 1) cy = H - 1;
                int bx0 = (int)max(cx - 1, 0LL), bx1 = (int)min(cx + 1, (long long)W - 1);
                int by0 = (int)max(cy - 1, 0LL), by1 = (int)min(cy + 1, (long long)H - 1);
                // kernels.py:323-329
                double eps = eps_abs;
                if (eps_rel * d > eps) eps = eps_rel * d;
                if (!depth_test(dv, f, gx, gy, bx0, bx1, by0, by1, d, eps)) continue;
                if (STATS) c_vis++;
                v += F.amp * exp(-0.5 * ratio_sq);  // kernels.py:340
            }
        }
        if (valid) values[i] = v;
        }
    }
    if (STATS) {
        stat_add(dv.stats, GM_STAT_L1_TESTS, lane == 0 ? c_l1 * (unsigned long long)B : 0ull);
        stat_add(dv.stats, GM_STAT_L2_TESTS, c_l2);
        stat_add(dv.stats, GM_STAT_EXACT, c_exact);
        stat_add(dv.stats, GM_STAT_NDC, c_ndc);
        stat_add(dv.stats, GM_STAT_CANDIDATES, c_cand);
        stat_add(dv.stats, GM_STAT_VISIBLE, c_vis);
    }
}

#define TW_CAP 32
#define TW_SEL 128  // overlapping triangles remembered per tile (more: rescanned per round)
#ifndef TW_WARPS
#define TW_WARPS 2  // warps (independent tile items) per k_texels CTA
#endif
struct __align__(16) TexelWarpSmem {
    TriF32 t32[TW_CAP];  // staged, in ascending min-depth order
    int sel[TW_SEL + 32];
};
#define TX_DYN_SMEM (TW_WARPS * (int)sizeof(TexelWarpSmem))
#define TC_SEL 512   // crowded tiles: overlap list sorted per pass (longer lists: several passes)
#define TC_RES 64    // crowded tiles: nearest triangles staged in shared memory
struct __align__(16) CrowdedWarpSmem {
    TriF32 t32[TC_RES];
    int sel[TC_SEL];
    float key[TC_SEL];
};
#ifndef TC_WARPS
#define TC_WARPS 4  // warps per CTA of the crowded pass
#endif
#ifndef CROWD_DEPTH
#define CROWD_DEPTH 10  // ... and whose triangle bboxes cover the tile more than this many times
#endif
#ifndef CROWD_MIN
#define CROWD_MIN 128  // tiles overlapping more triangles than this go to the crowded pass
#endif
#define TC_DYN_SMEM (TC_WARPS * (int)sizeof(CrowdedWarpSmem))
#define TX_MAX_THREADS (32 * (TW_WARPS > TC_WARPS ? TW_WARPS : TC_WARPS))

// position of the k-th (0-based) set bit of w (k < popc(w))
__device__ __forceinline__ int kth_set_bit(uint32_t w, int k) {
    int base = 0;
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
        const uint32_t low = w & ((1u << half) - 1u);
        const int c = __popc(low);
        if (k >= c) {
            k -= c;
            w >>= half;
            base += half;
        } else {
            w = low;
        }
    }
    return base;
}

// Fixation-major evaluation of the marked texels.  Every warp is an
// independent work item (fixation, 32x16-pixel tile): no CTA barriers, no
// atomics, per-texel state in registers.
//   1. the tile's triangles are gathered from its coarse bin (bbox-filtered);
//   2. their float32 forms (TriF32, built once per screen triangle by
//      k_tri_setup: edge-function and inverse-depth planes with rigorous error
//      bounds) are staged in the warp's shared slice TW_CAP at a time, in
//      ascending min-depth order;
//   3. lanes take the marked texels (compacted, 32 per round) and walk the
//      sorted triangles with uniform float32 tests: "certainly written"
//      (inside by more than the bound, inverse depth certainly within
//      (1/far', 1/near')) or "maybe written".  V, the largest certain lower
//      bound of the inverse depth, proves depth <= 1/V, so a maybe-triangle
//      whose inverse-depth upper bound is < V can never be the minimum, and
//      once a triangle's 1/minw bound is < V no later one can be (stop);
//   4. the surviving candidates (normally one) are evaluated exactly with the
//      reference's float64 pixel arithmetic (texel_depth, float64 record read
//      from L1/L2) and the minimum is stored -- the value kernels.rasterize
//      leaves in that pixel.
// One (fixation, tile) work item of k_texels.  T32/SEL: the warp's staging and
// selection slices; KEY (crowded mode only): sort keys of SEL.
template <bool ATTRS, bool STATS, bool CROWDED>
__device__ __forceinline__ void texel_item(TriF32* __restrict__ T32, int* __restrict__ SEL, float* __restrict__ KEY,
                                           int64_t item, const TriStore& ts, const DepthView& dv,
                                           const CoarseBins& cb, int tiles_x, int tiles_per_fix,
                                           const GmFixExact* __restrict__ fixes) {
    const int lane = threadIdx.x & 31;
    const int f = (int)(item / tiles_per_fix);
    const int tile = (int)(item - (int64_t)f * tiles_per_fix);
    const int W = dv.W, H = dv.H;
    const int xb = (tile % tiles_x) * TW, yb = (tile / tiles_x) * TH;
    const unsigned FULL = 0xffffffffu;
    // marked texels: lane r < TH holds the mask word of row yb + r
    uint32_t wr = 0;
    if (lane < TH && yb + lane < H) wr = dv.mask[((int64_t)f * H + yb + lane) * dv.wwords + (xb >> 5)];
    const int cnt_r = __popc(wr);
    int pref = cnt_r;  // inclusive prefix over rows
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, pref, o);
        if (lane >= o) pref += v;
    }
    const int total = __shfl_sync(FULL, pref, 31);
    if (total == 0) return;
    const int pref_ex = pref - cnt_r;
    const GmFixExact& F = fixes[f];
    const double near_ = F.near_, far_ = F.far_;
    // written iff near' <= 1/inv_w <= far' (kernels.py:123-127): certainly inside
    // [inv_far_hi, inv_near_lo], certainly outside beyond [inv_far_lo, inv_near_hi]
    const float inv_near = (float)(1.0 / near_), inv_far = (float)(1.0 / far_);
    const float inv_near_lo = inv_near * (1.0f - 1e-5f), inv_near_hi = inv_near * (1.0f + 1e-5f);
    const float inv_far_lo = inv_far * (1.0f - 1e-5f), inv_far_hi = inv_far * (1.0f + 1e-5f);
    const GmScreenTri* seg = ts.tris + (int64_t)f * ts.cap_seg;
    const uint2* segb = ts.bbox + (int64_t)f * ts.cap_seg;
    const int* clist = nullptr;
    int n = min(ts.count[f], (int)ts.cap_seg);
    if (!cb.ovf[f]) {
        const int* off = cb.off + (int64_t)f * (GM_MAX_CBINS + 1);
        const int bb = (yb >> cb.shift) * cb.ncx + (xb >> cb.shift);
        clist = cb.items + (int64_t)f * cb.cap_items + off[bb];
        n = off[bb + 1] - off[bb];
    }
    const int xe = xb + TW - 1, ye = yb + TH - 1;
    unsigned long long c_pairs = 0, c_cov = 0, c_iter = 0, c_edge = 0;

    // 1. triangles overlapping the tile -> S.sel (scan cursor resumes if > TW_SEL)
    int cover = 0;  // this lane's share of the selected bboxes' area inside the tile (depth complexity)
    auto gather = [&](int& cursor) {
        int cnt = 0;
        while (cursor < n && cnt < TW_SEL) {
            int i = cursor + lane;
            bool sel = false;
            if (i < n) {
                if (clist) i = clist[i];
                const uint2 bbx = segb[i];
                const int x0 = bbx.x & 0xffff, x1 = bbx.x >> 16, y0 = bbx.y & 0xffff, y1 = bbx.y >> 16;
                sel = !(x1 < xb || x0 > xe || y1 < yb || y0 > ye);
                if (sel) cover += (min(x1, xe) - max(x0, xb) + 1) * (min(y1, ye) - max(y0, yb) + 1);
            }
            const unsigned bal = __ballot_sync(FULL, sel);
            if (sel) SEL[cnt + __popc(bal & ((1u << lane) - 1u))] = i;
            cnt += __popc(bal);
            cursor += 32;
        }
        __syncwarp();
        return cnt;  // may exceed TW_SEL by < 32 (S.sel has the room)
    };

    // 2. stage SEL[c0 .. c0 + kend) (float32 forms) in ascending min-depth order
    const TriF32* segf = ts.t32 + (int64_t)f * ts.cap_seg;
    auto stage = [&](int c0, int kend) {
        __syncwarp();
        const int gi = lane < kend ? SEL[c0 + lane] : 0;
        float key = lane < kend ? -__ldg(&segf[gi].inv_minw) : CUDART_INF_F;  // ascending min depth
        int slot = lane;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const float ok = __shfl_xor_sync(FULL, key, stride);
                const int os = __shfl_xor_sync(FULL, slot, stride);
                const bool keep_min = ((lane & stride) == 0) == ((lane & size) == 0);
                const bool less = ok < key || (ok == key && os < slot);
                if (keep_min ? less : !less && !(ok == key && os == slot)) {
                    key = ok;
                    slot = os;
                }
            }
        }
        // lane = rank; it copies the record of sorted position `lane`
        const int src = __shfl_sync(FULL, gi, slot);
        if (lane < kend) {
            const uint4* from = reinterpret_cast<const uint4*>(segf + src);
            uint4* to = reinterpret_cast<uint4*>(&T32[lane]);
#pragma unroll
            for (int part = 0; part < 6; part++) to[part] = from[part];
        }
        __syncwarp();
    };

    // texel of compact id q: (row, tile-local column)
    auto texel_of = [&](int q, int& row, int& colo) {
        row = 0;
#pragma unroll
        for (int step = TH / 2; step > 0; step >>= 1) {
            const int cand = row + step;
            const int pc = __shfl_sync(FULL, pref_ex, cand & 31);
            if (cand < TH && pc <= q) row = cand;
        }
        const uint32_t w_row = __shfl_sync(FULL, wr, row);
        const int k_in_row = q - __shfl_sync(FULL, pref_ex, row);
        colo = q < total ? kth_set_bit(w_row, k_in_row) : 0;
    };

    // 3 + 4 for the staged chunk (kend triangles) and one texel: updates V, best
    // kernels.py:128-129 writes iff d < depth[py, px]: among equal minima the
    // first triangle in rasterization order (key 2 t + fan) owns the texel
    auto take = [&](double d, int cs, double& best, int& bkey) {
        if (!ATTRS) {
            if (d < best) best = d;
            return;
        }
        const int key = (int)(seg[cs].tl >> 3);
        if (d < best || (d == best && d < CUDART_INF && key < bkey)) {
            best = d;
            bkey = key;
        }
    };
    // triangle kk of the walk: staged in shared memory (kk < nst) or, crowded mode, from global
    auto tri_at = [&](int kk, int nst) -> const TriF32& { return (!CROWDED || kk < nst) ? T32[kk] : segf[SEL[kk]]; };
    auto walk = [&](int kend, int nst, bool valid, int row, int colo, float& V, double& best, int& bkey) {
        const int px = xb + colo, py = yb + row;
        int cs0 = -1, cs1 = -1;  // exact candidates (global record index) and their bounds
        float ch0 = 0.0f, ch1 = 0.0f;
        bool overflow = false;
        for (int kk = 0; kk < kend; kk++) {
            const TriF32& t = tri_at(kk, nst);
            const float inv_minw = t.inv_minw;
            if (__all_sync(FULL, !(inv_minw >= V))) break;  // nothing later can be nearer
            if (STATS) c_iter++;
            const uint32_t tbx = t.bx, tby = t.by;
            if (!(inv_minw >= V) || px < (int)(tbx & 0xffff) || px > (int)(tbx >> 16) || py < (int)(tby & 0xffff) ||
                py > (int)(tby >> 16))
                continue;
            if (STATS) c_edge++;
            const float fx = (float)(px - t.ox) + 0.5f, fy = (float)(py - t.oy) + 0.5f;  // bbox-local centre
            bool maybe = true, certain = true;
#pragma unroll
            for (int i = 0; i < 3; i++) {
                const float e = __fmaf_rn(t.a[i], fx, __fmaf_rn(t.b[i], fy, t.c[i]));
                maybe = maybe && (e >= -t.tol[i]);
                certain = certain && (e > t.tol[i]);
            }
            if (!maybe) continue;
            const float iwv = __fmaf_rn(t.A, fx, __fmaf_rn(t.B, fy, t.C));
            const float lo = iwv - t.tolw, hi = iwv + t.tolw;
            if (!(hi > 0.0f) || lo > inv_near_hi || hi < inv_far_lo) continue;  // certainly not written
            if (certain && lo > 0.0f && hi <= inv_near_lo && lo >= inv_far_hi && lo * (1.0f - 1e-6f) > V)
                V = lo * (1.0f - 1e-6f);
            if (hi >= V) {
                if (cs0 < 0) {
                    cs0 = t.gidx;
                    ch0 = hi;
                } else if (cs1 < 0) {
                    cs1 = t.gidx;
                    ch1 = hi;
                } else if (ch0 < V) {  // a stale candidate can be replaced
                    cs0 = t.gidx;
                    ch0 = hi;
                } else if (ch1 < V) {
                    cs1 = t.gidx;
                    ch1 = hi;
                } else {
                    overflow = true;
                }
            }
        }
        if (!valid) return;
        if (!overflow) {
            if (cs0 >= 0 && ch0 >= V) {
                const double d = texel_depth(seg[cs0], px, py, near_, far_);
                if (STATS) c_pairs++;
                if (STATS) c_cov += d < CUDART_INF;
                take(d, cs0, best, bkey);
            }
            if (cs1 >= 0 && ch1 >= V) {
                const double d = texel_depth(seg[cs1], px, py, near_, far_);
                if (STATS) c_pairs++;
                if (STATS) c_cov += d < CUDART_INF;
                take(d, cs1, best, bkey);
            }
        } else {  // slow path: every staged triangle whose bbox covers the texel
            for (int k = 0; k < kend; k++) {
                const TriF32& t = tri_at(k, nst);
                if (px < (int)(t.bx & 0xffff) || px > (int)(t.bx >> 16) || py < (int)(t.by & 0xffff) ||
                    py > (int)(t.by >> 16))
                    continue;
                const double d = texel_depth(seg[t.gidx], px, py, near_, far_);
                if (STATS) c_pairs++;
                if (STATS) c_cov += d < CUDART_INF;
                take(d, t.gidx, best, bkey);
            }
        }
    };

    double* dep = dv.depth + (int64_t)f * W * H;
    int cursor = 0;
    int nsel_total = 0;
    auto store = [&](int row, int colo, double best, int bkey) {
        dep[(int64_t)(yb + row) * W + xb + colo] = best;
        if (ATTRS) dv.key[(int64_t)(yb + row) * W + xb + colo] = best < CUDART_INF ? bkey : -1;
    };
    if (!CROWDED) {
        int nsel = gather(cursor);
        if (STATS) nsel_total = nsel;
        // deep tiles (overlapping surfaces: the selected bboxes cover the tile more than
        // CROWD_DEPTH times) profit from the sorted crowded pass; wide ones (many
        // side-by-side triangles) stay here
        if ((cursor < n || nsel > CROWD_MIN) && dv.crowd &&
            __reduce_add_sync(FULL, (unsigned)cover) > (unsigned)(CROWD_DEPTH * TW * TH)) {
            // more than TW_CAP triangles: k_texels<CROWDED> sorts the whole list (deferred)
            if (lane == 0) dv.crowd[atomicAdd(dv.crowd_count, 1)] = (int)item;
            return;
        }
        if (cursor >= n && nsel <= TW_CAP) {
            // common case: one staging serves every round, per-texel state in registers
            if (nsel > 0) stage(0, nsel);
            for (int r0 = 0; r0 < total; r0 += 32) {
                const int q = r0 + lane;
                const bool valid = q < total;
                int row, colo;
                texel_of(q, row, colo);
                float V = valid ? 0.0f : CUDART_INF_F;
                double best = CUDART_INF;
                int bkey = INT_MAX;
                if (nsel > 0) walk(nsel, nsel, valid, row, colo, V, best, bkey);
                if (valid) store(row, colo, best, bkey);
            }
        } else {
            // many triangles without a deferral list: chunk by chunk (each staged once),
            // per-texel state kept in the depth array and the inverse-depth-bound buffer
            float* vb = dv.vbuf + (int64_t)f * W * H;
            bool first = true;
            while (true) {
                for (int c0 = 0; c0 < nsel; c0 += TW_CAP) {
                    const int kend = min(TW_CAP, nsel - c0);
                    stage(c0, kend);
                    for (int r0 = 0; r0 < total; r0 += 32) {
                        const int q = r0 + lane;
                        const bool valid = q < total;
                        int row, colo;
                        texel_of(q, row, colo);
                        const int64_t at = (int64_t)(yb + row) * W + xb + colo;
                        float V = valid ? (first ? 0.0f : vb[at]) : CUDART_INF_F;
                        double best = (valid && !first) ? dep[at] : CUDART_INF;
                        int bkey = INT_MAX;
                        if (ATTRS && valid && !first) bkey = dv.key[at];
                        walk(kend, kend, valid, row, colo, V, best, bkey);
                        if (valid) {
                            dep[at] = best;
                            vb[at] = V;
                            if (ATTRS) dv.key[at] = best < CUDART_INF ? bkey : -1;
                        }
                    }
                    first = false;
                }
                if (cursor >= n) break;
                nsel = gather(cursor);
                if (STATS) nsel_total += nsel;
            }
            if (first) {  // no triangle at all
                for (int r0 = 0; r0 < total; r0 += 32) {
                    const int q = r0 + lane;
                    int row, colo;
                    texel_of(q, row, colo);
                    if (q < total) store(row, colo, CUDART_INF, -1);
                }
            }
        }
    } else {
        // crowded tile: gather the whole overlap list (TC_SEL at a time), sort it by
        // ascending min depth, stage the nearest TC_RES float32 forms; the walk reads
        // any later one from global memory.  The nearest certain cover then proves
        // (V) that every later triangle is behind it, so a texel's walk usually ends
        // in the first chunk -- nested surfaces cost one sort, not one pass each.
        float* vb = dv.vbuf + (int64_t)f * W * H;
        bool first = true;
        do {
            int cnt = 0;
            while (cursor < n && cnt < TC_SEL - 32) {
                int i = cursor + lane;
                bool sel = false;
                if (i < n) {
                    if (clist) i = clist[i];
                    const uint2 bbx = segb[i];
                    const int x0 = bbx.x & 0xffff, x1 = bbx.x >> 16, y0 = bbx.y & 0xffff, y1 = bbx.y >> 16;
                    sel = !(x1 < xb || x0 > xe || y1 < yb || y0 > ye);
                }
                const unsigned bal = __ballot_sync(FULL, sel);
                if (sel) {
                    const int at = cnt + __popc(bal & ((1u << lane) - 1u));
                    SEL[at] = i;
                    KEY[at] = -__ldg(&segf[i].inv_minw);
                }
                cnt += __popc(bal);
                cursor += 32;
            }
            if (STATS) nsel_total += cnt;
            int P = 32;
            while (P < cnt) P <<= 1;
            for (int k = cnt + lane; k < P; k += 32) {
                KEY[k] = CUDART_INF_F;
                SEL[k] = -1;
            }
            __syncwarp();
            // warp bitonic sort of (KEY, SEL) ascending, P <= TC_SEL
            for (int size = 2; size <= P; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int a = lane; a < P; a += 32) {
                        const int b = a ^ stride;
                        if (b > a) {
                            const float ka = KEY[a], kb = KEY[b];
                            const int sa = SEL[a], sb = SEL[b];
                            const bool up = (a & size) == 0;
                            const bool gt = ka > kb || (ka == kb && sa > sb);
                            if (gt == up) {
                                KEY[a] = kb;
                                KEY[b] = ka;
                                SEL[a] = sb;
                                SEL[b] = sa;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            const int ns = min(cnt, TC_RES);
            for (int k = lane; k < ns; k += 32) {
                const uint4* from = reinterpret_cast<const uint4*>(segf + SEL[k]);
                uint4* to = reinterpret_cast<uint4*>(&T32[k]);
#pragma unroll
                for (int part = 0; part < 6; part++) to[part] = from[part];
            }
            __syncwarp();
            const bool last = cursor >= n;
            for (int r0 = 0; r0 < total; r0 += 32) {
                const int q = r0 + lane;
                const bool valid = q < total;
                int row, colo;
                texel_of(q, row, colo);
                const int64_t at = (int64_t)(yb + row) * W + xb + colo;
                float V = valid ? (first ? 0.0f : vb[at]) : CUDART_INF_F;
                double best = (valid && !first) ? dep[at] : CUDART_INF;
                int bkey = INT_MAX;
                if (ATTRS && valid && !first) bkey = dv.key[at];
                if (cnt > 0) walk(cnt, ns, valid, row, colo, V, best, bkey);
                if (valid) {
                    dep[at] = best;
                    if (!last) vb[at] = V;
                    if (ATTRS) dv.key[at] = best < CUDART_INF ? bkey : -1;
                }
            }
            first = false;
            __syncwarp();
        } while (cursor < n);
    }
    if (STATS) {
        const bool l0 = lane == 0;
        stat_add(dv.stats, GM_STAT_TEXELS, l0 ? (unsigned long long)total : 0ull);
        stat_add(dv.stats, GM_STAT_TX_TILES, l0 ? 1ull : 0ull);
        stat_add(dv.stats, GM_STAT_TX_STAGED, l0 ? (unsigned long long)nsel_total : 0ull);
        stat_add(dv.stats, GM_STAT_TX_LIST, l0 ? (unsigned long long)n : 0ull);
        stat_add(dv.stats, GM_STAT_TX_ITER, l0 ? c_iter : 0ull);
        stat_add(dv.stats, GM_STAT_PAIRS, c_pairs);
        stat_add(dv.stats, GM_STAT_COVERED, c_cov);
        stat_add(dv.stats, GM_STAT_TX_EDGE, c_edge);
    }
}

template <bool ATTRS, bool STATS, bool CROWDED>
__global__ void TX_BOUNDS k_texels(TriStore ts, DepthView dv, CoarseBins cb, int tiles_x,
                                   int tiles_per_fix, int64_t n_items,
                                   const GmFixExact* __restrict__ fixes, long long b0) {
    extern __shared__ __align__(16) unsigned char tx_dyn[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (*ts.fail <= b0) return;
    if (!CROWDED) {
        const int64_t item = (int64_t)blockIdx.x * TW_WARPS + warp;
        if (item < n_items)
            texel_item<ATTRS, STATS, false>(reinterpret_cast<TexelWarpSmem*>(tx_dyn)[warp].t32,
                                            reinterpret_cast<TexelWarpSmem*>(tx_dyn)[warp].sel, nullptr, item, ts, dv,
                                            cb, tiles_x, tiles_per_fix, fixes);
        return;
    }
    // crowded tiles (deferred by the pass above): persistent warps over the list
    CrowdedWarpSmem& C = reinterpret_cast<CrowdedWarpSmem*>(tx_dyn)[warp];
    const int n_crowd = *dv.crowd_count;
    for (;;) {
        int w = 0;
        if (lane == 0) w = atomicAdd(dv.crowd_count + 1, 1);
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w >= n_crowd) break;
        texel_item<ATTRS, STATS, true>(C.t32, C.sel, C.key, dv.crowd[w], ts, dv, cb, tiles_x, tiles_per_fix, fixes);
    }
}

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

// Everything one batch of fixations owns on the device.  A plan holds two sets
// (the plan's own fields and `alt`); consecutive batches alternate between them
// and between two streams, so batch i + 1's occluder setup, marking and texel
// kernels overlap batch i's tail.  Only the accumulation pass (k_samples) is
// chained across batches (event), which keeps the per-sample log order.
#define GM_BATCH_FIELDS(X)                                                                            \
    X(cudaStream_t, stream) X(uint32_t*, d_lvl1) X(uint32_t*, d_cbits) X(int64_t, cap_cbits)           \
    X(int*, d_lcount) X(int*, d_lorder) X(int*, d_lcount2) X(int*, d_lorder2) X(int64_t, cap_sort)     \
    X(int*, d_work) X(void*, d_sort_tmp) X(size_t, sort_tmp_bytes) X(int64_t, cap_lvl1) X(int, cap_B)  \
    X(GmFixExact*, d_fix) X(GmFixCull*, d_cull) X(GmFixF32*, d_fix32) X(GmScreenTri*, d_tris)          \
    X(TriF32*, d_t32) X(uint2*, d_bbox) X(int*, d_count) X(int64_t, cap_seg) X(int64_t, cap_seg_B)     \
    X(double*, d_depth) X(float*, d_vbuf) X(uint32_t*, d_mask) X(int64_t, cap_depth) X(int64_t, cap_mask) \
    X(int*, d_citems) X(int*, d_coff) X(int*, d_covf) X(int64_t, cap_citems) X(int64_t, cap_cB)         \
    X(int*, d_crowd) X(int*, d_crowd_count) X(int64_t, cap_crowd)

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
    long long* d_fail = nullptr;
    int* d_maxcount = nullptr;
    unsigned long long* d_ntris = nullptr;
    // marked z-buffer texels
    double* d_depth = nullptr;   // [B][H][W] marked texels only
    float* d_vbuf = nullptr;     // [B][H][W] k_texels state for crowded tiles
    uint32_t* d_mask = nullptr;  // [B][H][wwords]
    int64_t cap_depth = 0, cap_mask = 0;
    int* d_citems = nullptr;  // coarse bins: [B][cap_citems]
    int* d_coff = nullptr;    // [B][GM_MAX_CBINS + 1]
    int* d_covf = nullptr;    // [B]
    int64_t cap_citems = 0, cap_cB = 0;
    unsigned long long* d_max = nullptr;
    unsigned long long* d_stats = nullptr;  // GM_STAT_N counters
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
    int64_t cap_key = 0;
    int64_t cap_cbits = 0, cap_sort = 0;  // (per batch-buffer set, swapped with alt)
    int cap_ring = 0;
    BatchBufs alt;                   // the second batch-buffer set (and stream)
    cudaEvent_t ev_order = nullptr;  // last accumulation pass enqueued (chains k_samples across streams)
};

// Exchange the plan's batch buffers (and stream) with the alternate set.
static void swap_batch_bufs(gm_plan* p) {
#define GM_X(T, n) std::swap(p->n, p->alt.n);
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
    swap_batch_bufs(p);
    free_scene_batch_bufs(p);
    swap_batch_bufs(p);
    p->d_tw = nullptr; p->d_tsph = p->d_csph = p->d_chunk = p->d_super = nullptr;
    p->d_px = p->d_py = p->d_pz = p->d_values = nullptr;
    p->T = p->n_clu = p->N = p->n_chunks = p->n_supers = 0;
    cudaFree(p->d_local); cudaFree(p->d_res); cudaFree(p->d_off); cudaFree(p->d_M);
    p->d_local = nullptr; p->d_res = p->d_off = nullptr; p->d_M = nullptr;
    p->n_obj = 0;
    p->tstart.clear(); p->nsamp.clear(); p->include.clear();
}

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
    CK(cudaFuncSetAttribute(k_texels<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TX_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_DYN_SMEM));
    CK(cudaFuncSetAttribute(k_texels<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_DYN_SMEM));
    CK(cudaMalloc(&p->d_max, sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_stats, GM_STAT_STRIPES * GM_STAT_N * sizeof(unsigned long long)));
    CK(cudaMemset(p->d_stats, 0, GM_STAT_STRIPES * GM_STAT_N * sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_fail, sizeof(long long)));
    CK(cudaMalloc(&p->d_maxcount, sizeof(int)));
    CK(cudaMalloc(&p->d_ntris, sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_work, 2 * sizeof(int)));
    CK(cudaEventCreateWithFlags(&p->ev_order, cudaEventDisableTiming));
    for (int r = 0; r < GM_RING; r++) CK(cudaEventCreateWithFlags(&p->h_ev[r], cudaEventDisableTiming));
    unsigned hc = std::thread::hardware_concurrency();
    p->host_threads = hc > 0 ? (int)hc : 8;
    *out = p;
    return GM_OK;
}

// Free one batch-buffer set (the plan's own fields) and its stream.
static void free_batch_set(gm_plan* p) {
    if (p->stream) cudaStreamSynchronize(p->stream);
    free_scene_batch_bufs(p);
    cudaFree(p->d_fix); cudaFree(p->d_cull); cudaFree(p->d_fix32); cudaFree(p->d_work);
    cudaFree(p->d_tris); cudaFree(p->d_t32); cudaFree(p->d_bbox); cudaFree(p->d_count);
    cudaFree(p->d_depth); cudaFree(p->d_mask); cudaFree(p->d_vbuf);
    cudaFree(p->d_citems); cudaFree(p->d_coff); cudaFree(p->d_covf);
    cudaFree(p->d_crowd); cudaFree(p->d_crowd_count);
    if (p->stream) cudaStreamDestroy(p->stream);
    p->stream = nullptr;
}

extern "C" void gm_plan_destroy(gm_plan* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    if (p->alt.stream) cudaStreamSynchronize(p->alt.stream);
    plan_free_scene(p);
    for (int r = 0; r < GM_RING; r++) {
        cudaFreeHost(p->h_fix[r]); cudaFreeHost(p->h_cull[r]); cudaEventDestroy(p->h_ev[r]);
    }
    cudaFree(p->d_fail); cudaFree(p->d_maxcount); cudaFree(p->d_ntris);
    cudaFree(p->d_scan_tmp); cudaFree(p->d_max); cudaFree(p->d_stats);
    cudaFree(p->d_fix_all); cudaFree(p->d_cull_all); cudaFree(p->d_flush);
    cudaFree(p->d_key);
    if (p->ev_order) cudaEventDestroy(p->ev_order);
    free_batch_set(p);
    swap_batch_bufs(p);
    free_batch_set(p);
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
    const int64_t n_tiles = (int64_t)B * ((W + TW - 1) / TW) * ((H + TH - 1) / TH);
    if (n_tiles > p->cap_crowd) {
        if ((rc = dev_alloc(&p->d_crowd, (size_t)n_tiles))) return rc;
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
    swap_batch_bufs(p);
    rc = ensure_batch_set(p, B, W, H, std::max(seg, p->alt.cap_seg));
    swap_batch_bufs(p);
    return rc;
}

typedef void (*gm_progress_fn)(int64_t done, int64_t total, void* user);

// Coarse-bin geometry for a W x H buffer: cb = 64 px, doubled until <= GM_MAX_CBINS bins.
static CoarseBins coarse_bins(gm_plan* p, int W, int H) {
    int shift = CB_SHIFT;
    while ((int64_t)((W + (1 << shift) - 1) >> shift) * ((H + (1 << shift) - 1) >> shift) > GM_MAX_CBINS) shift++;
    CoarseBins cb{p->d_citems, p->d_coff, p->d_covf, p->cap_citems, shift, (W + (1 << shift) - 1) >> shift,
                  (H + (1 << shift) - 1) >> shift};
    return cb;
}


// k_texels over `items` (fixation, tile) work items, then the crowded tiles the
// first pass deferred (k_texels<CROWDED>, persistent, larger shared slices).
template <bool ATTRS, bool STATS>
static int launch_texels(gm_plan* p, cudaStream_t s, const TriStore& ts, DepthView dv, const CoarseBins& cb,
                         int tiles_x, int tiles_per_fix, int64_t items, const GmFixExact* fix, long long b0) {
    dv.crowd = p->d_crowd;
    dv.crowd_count = p->d_crowd_count;
    CK(cudaMemsetAsync(p->d_crowd_count, 0, 2 * sizeof(int), s));
    k_texels<ATTRS, STATS, false><<<(unsigned)((items + TW_WARPS - 1) / TW_WARPS), TW_WARPS * 32, TX_DYN_SMEM, s>>>(
        ts, dv, cb, tiles_x, tiles_per_fix, items, fix, b0);
    k_texels<ATTRS, STATS, true><<<p->sms * (20 / TC_WARPS), TC_WARPS * 32, TC_DYN_SMEM, s>>>(ts, dv, cb, tiles_x, tiles_per_fix,
                                                                              items, fix, b0);
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
    const int tiles_x = (W + TW - 1) / TW, tiles_y = (H + TH - 1) / TH;
    TriStore ts{p->d_tris, p->d_t32, p->d_bbox, p->d_count, p->cap_seg, p->d_fail, p->d_maxcount, p->d_ntris};
    DepthView dv{p->d_depth, p->d_mask, W, H, wwords, (cfg->flags & GM_FLAG_STATS) ? p->d_stats : nullptr,
                 p->d_vbuf};
    if (ev) CK(cudaEventRecord(ev[0], s));
    CK(cudaMemsetAsync(p->d_count, 0, sizeof(int) * nb, s));
    if (p->n_clu > 0) {
        dim3 grid(blocks_for((p->n_clu + 31) / 32, 8), nb);
        k_tri_setup<<<grid, 256, 0, s>>>(p->d_tw, p->T, p->d_tsph, p->d_csph, p->n_clu, d_fix, d_cull, W, H, ts, b0);
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
        if (ev) CK(cudaEventRecord(ev[2], s));
        const int64_t items = (int64_t)nb * tiles_x * tiles_y;
        CoarseBins cbins = coarse_bins(p, W, H);
        k_coarse<<<nb, 256, 0, s>>>(ts, cbins, p->d_fail, b0);
        int trc = dv.stats ? launch_texels<false, true>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, d_fix, b0)
                           : launch_texels<false, false>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, d_fix, b0);
        if (trc) return trc;
        if (ev) CK(cudaEventRecord(ev[3], s));
        // accumulation passes run in batch order across the two streams (log order per sample)
        CK(cudaStreamWaitEvent(s, p->ev_order, 0));
        auto ks = dv.stats ? k_samples<true> : k_samples<false>;
        ks<<<grid_s, 256, 0, s>>>(p->d_px, p->d_py, p->d_pz, p->d_chunk, p->d_lvl1, p->d_lorder2, p->d_work + 1, p->N,
                                p->n_chunks, p->n_supers, d_fix, d_cull, nb, dv, inv_sigma, cfg->eps_abs,
                                cfg->eps_rel, p->d_values, p->d_cbits, p->d_fail, b0);
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
    int rc = ensure_batch(p, B, W, H, std::max<int64_t>(p->cap_seg, 16384), two);
    if (rc) return rc;
    cudaStream_t s = p->stream;          // primary stream (even batches)
    cudaStream_t s2 = p->alt.stream;     // odd batches
    cudaEvent_t ev_fork = nullptr;
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    auto fork = [&]() -> int {  // everything enqueued on s so far precedes what s2 runs next
        if (!two) return GM_OK;
        CK(cudaEventRecord(ev_fork, s));
        CK(cudaStreamWaitEvent(s2, ev_fork, 0));
        return GM_OK;
    };
    auto join = [&]() -> int {  // s waits for everything enqueued on s2
        if (!two) return GM_OK;
        CK(cudaEventRecord(ev_fork, s2));
        CK(cudaStreamWaitEvent(s, ev_fork, 0));
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
        for (int64_t b0 = start; b0 < F; b0 += B, parity ^= (two ? 1 : 0)) {
            int nb = (int)std::min<int64_t>(B, F - b0);
            // odd batches run on the alternate buffer set and stream
            struct SwapGuard {
                gm_plan* p;
                bool on;
                ~SwapGuard() {
                    if (on) swap_batch_bufs(p);
                }
            } guard{p, parity == 1};
            if (parity) swap_batch_bufs(p);
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
        p->alt.cap_seg = 0;
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

// Copy the plan's values to host (raw) and optionally values / gmax.
extern "C" int gm_plan_read(gm_plan* p, double* raw, double* normalized, double gmax) {
    if (!p) return set_err(GM_ERR_ARG, "null plan");
    CK(cudaSetDevice(p->device));
    cudaStream_t s = p->stream;
    if (p->N == 0) return GM_OK;
    if (raw) CK(cudaMemcpyAsync(raw, p->d_values, sizeof(double) * p->N, cudaMemcpyDeviceToHost, s));
    if (normalized) {
        double* tmp = nullptr;
        CK(cudaMallocAsync(&tmp, sizeof(double) * p->N, s));
        k_normalize<<<std::min<int64_t>(blocks_for(p->N, 256), (int64_t)p->sms * 8), 256, 0, s>>>(p->d_values, p->N, gmax, tmp);
        CK(cudaMemcpyAsync(normalized, tmp, sizeof(double) * p->N, cudaMemcpyDeviceToHost, s));
        CK(cudaFreeAsync(tmp, s));
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
    double* d_tri = nullptr;
    int64_t *d_res = nullptr, *d_cnt = nullptr, *d_off = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CK(cudaMalloc(&d_tri, sizeof(double) * 9 * T));
    CK(cudaMalloc(&d_res, sizeof(int64_t) * T));
    CK(cudaMalloc(&d_cnt, sizeof(int64_t) * (T + 1)));
    CK(cudaMalloc(&d_off, sizeof(int64_t) * (T + 1)));
    CK(cudaMemcpy(d_tri, tri_local, sizeof(double) * 9 * T, cudaMemcpyHostToDevice));
    k_layout<<<blocks_for(T, 256), 256>>>(d_tri, T, 8.0 * k, nullptr, d_res, d_cnt);
    CK(cudaMemset(d_cnt + T, 0, sizeof(int64_t)));
    cub::DeviceScan::ExclusiveSum(nullptr, tb, d_cnt, d_off, T + 1);
    CK(cudaMalloc(&tmp, tb));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tb, d_cnt, d_off, T + 1));
    if (res) CK(cudaMemcpy(res, d_res, sizeof(int64_t) * T, cudaMemcpyDeviceToHost));
    if (counts) CK(cudaMemcpy(counts, d_cnt, sizeof(int64_t) * T, cudaMemcpyDeviceToHost));
    if (offsets) CK(cudaMemcpy(offsets, d_off, sizeof(int64_t) * T, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(total, d_off + T, sizeof(int64_t), cudaMemcpyDeviceToHost));
    cudaFree(d_tri); cudaFree(d_res); cudaFree(d_cnt); cudaFree(d_off); cudaFree(tmp);
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
    double *d_tri = nullptr, *d_out = nullptr, *d_M = nullptr;
    int64_t *d_res = nullptr, *d_off = nullptr;
    CK(cudaMalloc(&d_tri, sizeof(double) * 9 * T));
    CK(cudaMalloc(&d_res, sizeof(int64_t) * T));
    CK(cudaMalloc(&d_off, sizeof(int64_t) * T));
    CK(cudaMalloc(&d_out, sizeof(double) * 3 * N));
    CK(cudaMemcpy(d_tri, tri_local, sizeof(double) * 9 * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_res, res, sizeof(int64_t) * T, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_off, offsets, sizeof(int64_t) * T, cudaMemcpyHostToDevice));
    if (xform) {
        double Mt[12];
        xform_matrix(xform, Mt, Mt + 9);
        CK(cudaMalloc(&d_M, sizeof(double) * 12));
        CK(cudaMemcpy(d_M, Mt, sizeof(double) * 12, cudaMemcpyHostToDevice));
    }
    k_positions<<<blocks_for(N, 256), 256>>>(d_tri, T, d_res, d_off, N, d_M, d_M ? d_M + 9 : nullptr, d_out,
                                            nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d_out, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost));
    cudaFree(d_tri); cudaFree(d_res); cudaFree(d_off); cudaFree(d_out); cudaFree(d_M);
    return GM_OK;
}

// normalize (density.py:230-244) of a host vector on the GPU.
extern "C" int gm_normalize(int device, const double* values, int64_t n, double gmax, double* out) {
    if (n < 0) return set_err(GM_ERR_ARG, "bad length");
    if (n == 0) return GM_OK;
    int rc = use_device(device);
    if (rc) return rc;
    double *d_in = nullptr, *d_out = nullptr;
    CK(cudaMalloc(&d_in, sizeof(double) * n));
    CK(cudaMalloc(&d_out, sizeof(double) * n));
    CK(cudaMemcpy(d_in, values, sizeof(double) * n, cudaMemcpyHostToDevice));
    k_normalize<<<blocks_for(n, 256), 256>>>(d_in, n, gmax, d_out);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d_out, sizeof(double) * n, cudaMemcpyDeviceToHost));
    cudaFree(d_in); cudaFree(d_out);
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
            dim3 grid(blocks_for((p->n_clu + 31) / 32, 8), 1);
            k_tri_setup<<<grid, 256, 0, s>>>(p->d_tw, p->T, p->d_tsph, p->d_csph, p->n_clu, p->d_fix, p->d_cull, W,
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
    const int tiles_x = (W + TW - 1) / TW, tiles_y = (H + TH - 1) / TH;
    DepthView dv{p->d_depth, p->d_mask, W, H, wwords, nullptr, p->d_vbuf, attrs ? p->d_key : nullptr};
    k_mark_all<<<blocks_for((int64_t)H * wwords, 256), 256, 0, s>>>(p->d_mask, W, H, wwords);
    CoarseBins cbins = coarse_bins(p, W, H);
    k_coarse<<<1, 256, 0, s>>>(ts, cbins, p->d_fail, 0);
    const int64_t items = (int64_t)tiles_x * tiles_y;
    return attrs ? launch_texels<true, false>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, p->d_fix, 0)
                 : launch_texels<false, false>(p, s, ts, dv, cbins, tiles_x, tiles_x * tiles_y, items, p->d_fix, 0);
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

// ------------------------------------------- general camera: raster + heatmap

// kernels.py:140-192 for triangle t, fan k, at pixel (px, py), with the vertex
// attributes (identity rows, interpolated along clipped edges, swapped with
// the winding) -- the with_attrs branch of _raster_tri (:130-137): returns the
// perspective-correct barycentrics bary[3] the reference stores.  Same float64
// operation order as the reference (no FMA).
__device__ bool raster_attrs(const double* tw, const GmFixExact& F, int W, int H, int k, int px, int py,
                             double bary[3]) {
    double vin[3][6];
    for (int v = 0; v < 3; v++) {
        const double wx = tw[3 * v], wy = tw[3 * v + 1], wz = tw[3 * v + 2];
        for (int i = 0; i < 3; i++)
            vin[v][i] = F.rot[3 * i] * wx + F.rot[3 * i + 1] * wy + F.rot[3 * i + 2] * wz + F.trans[i];
        for (int c = 0; c < 3; c++) vin[v][3 + c] = c == v ? 1.0 : 0.0;
    }
    double vout[4][6];
    int nv = 0;
    const double nn = F.near_;
    for (int i = 0; i < 3; i++) {
        const int j = (i + 1) % 3;
        const double cz = vin[i][2], nz = vin[j][2];
        const bool cin = cz <= -nn, nin = nz <= -nn;
        if (cin) {
            for (int c = 0; c < 6; c++) vout[nv][c] = vin[i][c];
            nv++;
        }
        if (cin != nin) {
            const double t = (-nn - cz) / (nz - cz);
            for (int c = 0; c < 6; c++) vout[nv][c] = vin[i][c] + t * (vin[j][c] - vin[i][c]);
            nv++;
        }
    }
    if (k > nv - 3) return false;
    const double half_w = 0.5 * (double)W, half_h = 0.5 * (double)H;
    double sx[3], sy[3], iw[3], at[3][3];
    for (int m = 0; m < 3; m++) {
        const int src = m == 0 ? 0 : k + m;
        const double x = vout[src][0], y = vout[src][1], z = vout[src][2];
        const double w = -z;
        if (w <= 0.0) return false;
        const double ndc_x = (F.p00 * x + F.p02 * z) / w;
        const double ndc_y = (F.p11 * y + F.p12 * z) / w;
        sx[m] = (ndc_x + 1.0) * half_w;
        sy[m] = (1.0 - ndc_y) * half_h;
        iw[m] = 1.0 / w;
        for (int c = 0; c < 3; c++) at[m][c] = vout[src][3 + c];
    }
    double area = edge_fn(sx[0], sy[0], sx[1], sy[1], sx[2], sy[2]);
    if (area == 0.0) return false;
    if (area < 0.0) {
        double t;
        t = sx[1]; sx[1] = sx[2]; sx[2] = t;
        t = sy[1]; sy[1] = sy[2]; sy[2] = t;
        t = iw[1]; iw[1] = iw[2]; iw[2] = t;
        for (int c = 0; c < 3; c++) {
            t = at[1][c]; at[1][c] = at[2][c]; at[2][c] = t;
        }
        area = -area;
    }
    const double inv_area = 1.0 / area;
    const double cx = (double)px + 0.5, cy = (double)py + 0.5;
    const double w0 = edge_fn(sx[1], sy[1], sx[2], sy[2], cx, cy);
    const double w1 = edge_fn(sx[2], sy[2], sx[0], sy[0], cx, cy);
    const double w2 = edge_fn(sx[0], sy[0], sx[1], sy[1], cx, cy);
    const double l0 = w0 * inv_area, l1 = w1 * inv_area, l2 = w2 * inv_area;
    const double inv_w = l0 * iw[0] + l1 * iw[1] + l2 * iw[2];
    const double d = 1.0 / inv_w;
    for (int c = 0; c < 3; c++) bary[c] = (l0 * at[0][c] * iw[0] + l1 * at[1][c] * iw[1] + l2 * at[2][c] * iw[2]) * d;
    return true;
}

// tri_id / bary of every pixel from the winning order key (reference
// initial values -1 / 0 where nothing is drawn).
__global__ void k_attrs(const int* __restrict__ key, const double* __restrict__ tw, const GmFixExact* __restrict__ fix,
                        int W, int H, int32_t* __restrict__ tri_id, double* __restrict__ bary) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= (int64_t)W * H) return;
    const int kk = key[q];
    double b[3] = {0.0, 0.0, 0.0};
    int id = -1;
    if (kk >= 0) {
        const int t = kk >> 1;
        if (raster_attrs(tw + 9 * (int64_t)t, fix[0], W, H, kk & 1, (int)(q % W), (int)(q / W), b)) id = t;
    }
    tri_id[q] = id;
    bary[3 * q] = b[0];
    bary[3 * q + 1] = b[1];
    bary[3 * q + 2] = b[2];
}

// render.py:150-182 piecewise-linear field over each triangle's sample grid,
// then ColorMap.rgb (render.py:44-50: clip, ** gamma, np.interp per channel)
// and np.round(rgb * 255) -> uint8; background black.
struct GmColorMap {
    double xs[16], cols[16][3];
    int n;
    double gamma;
};

__device__ double np_interp(double x, const GmColorMap& cm, int c) {
    // numpy arr_interp (compiled_base.c) with precomputed slopes
    const int n = cm.n;
    if (isnan(x)) return x;
    if (x < cm.xs[0]) return cm.cols[0][c];
    if (x > cm.xs[n - 1]) return cm.cols[n - 1][c];
    int j = 0;
    while (j + 1 < n && cm.xs[j + 1] <= x) j++;
    if (j == n - 1) return cm.cols[j][c];
    if (cm.xs[j] == x) return cm.cols[j][c];
    const double slope = (cm.cols[j + 1][c] - cm.cols[j][c]) / (cm.xs[j + 1] - cm.xs[j]);
    double r = slope * (x - cm.xs[j]) + cm.cols[j][c];
    if (isnan(r)) {
        r = slope * (x - cm.xs[j + 1]) + cm.cols[j + 1][c];
        if (isnan(r) && cm.cols[j][c] == cm.cols[j + 1][c]) r = cm.cols[j][c];
    }
    return r;
}

__device__ double np_scalar_power(double v, double g) {
    // numpy fast_scalar_power special exponents, else libm pow
    if (g == 1.0) return v;
    if (g == 2.0) return v * v;
    if (g == 0.5) return sqrt(v);
    if (g == -1.0) return 1.0 / v;
    if (g == 0.0) return 1.0;
    return pow(v, g);
}

__global__ void k_heat(const int32_t* __restrict__ tri_id, const double* __restrict__ bary, int64_t npix,
                       const int64_t* __restrict__ res, const int64_t* __restrict__ base,
                       const double* __restrict__ values, GmColorMap cm, uint8_t* __restrict__ img) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= npix) return;
    const int t = tri_id[q];
    if (t < 0) {
        img[3 * q] = img[3 * q + 1] = img[3 * q + 2] = 0;
        return;
    }
    const double w1 = bary[3 * q], w3 = bary[3 * q + 2];
    const int64_t ri = res[t];
    const double rr = (double)ri;
    const double R = fmin(fmax(rr * (1.0 - w3), 0.0), rr);
    const double C = fmin(fmax(rr * w1, 0.0), R);
    int64_t r0 = x86_i64(floor(R));
    if (r0 > ri - 1) r0 = ri - 1;
    const double fr = R - (double)r0;
    int64_t c0 = x86_i64(floor(C));
    if (c0 > r0) c0 = r0;
    double fc = C - (double)c0;
    const bool upper = (fc > fr) && (c0 < r0);
    if (!upper) fc = fmin(fc, fr);
    const int64_t b = base[t];
    auto sv = [&](int64_t row, int64_t col) { return values[b + row * (row + 1) / 2 + col]; };
    double v;
    if (!upper) {
        v = (1.0 - fr) * sv(r0, c0) + (fr - fc) * sv(r0 + 1, c0) + fc * sv(r0 + 1, c0 + 1);
    } else {
        int64_t c0u = r0 - 1 > 0 ? r0 - 1 : 0;
        if (c0 < c0u) c0u = c0;
        v = (1.0 - fc) * sv(r0, c0u) + (fc - fr) * sv(r0, c0u + 1) + fr * sv(r0 + 1, c0u + 1);
    }
    const double x = np_scalar_power(fmin(fmax(v, 0.0), 1.0), cm.gamma);
    for (int c = 0; c < 3; c++) img[3 * q + c] = (uint8_t)(int)rint(np_interp(x, cm, c) * 255.0);
}

// kernels.cull_mask (kernels.py:195-216): drop a triangle only when all three
// vertices are outside one plane (a x + b y + c z + d < 0, no FMA).
__global__ void k_cull_mask(const double* __restrict__ tris, int64_t T, const double* __restrict__ planes, int np,
                            uint8_t* __restrict__ keep) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const double* v = tris + 9 * t;
    uint8_t k = 1;
    for (int p = 0; p < np; p++) {
        const double a = planes[4 * p], b = planes[4 * p + 1], c = planes[4 * p + 2], d = planes[4 * p + 3];
        bool outside = true;
        for (int q = 0; q < 3; q++)
            if (a * v[3 * q] + b * v[3 * q + 1] + c * v[3 * q + 2] + d >= 0.0) {
                outside = false;
                break;
            }
        if (outside) {
            k = 0;
            break;
        }
    }
    keep[t] = k;
}

extern "C" int gm_cull_mask(int device, const double* tris, int64_t T, const double* planes, int n_planes,
                            uint8_t* keep) {
    if (T < 0 || (T > 0 && (!tris || !keep)) || n_planes < 0 || n_planes > 64 || (n_planes && !planes))
        return set_err(GM_ERR_ARG, "bad arguments");
    if (T == 0) return GM_OK;
    int rc = use_device(device);
    if (rc) return rc;
    double *d_t = nullptr, *d_p = nullptr;
    uint8_t* d_k = nullptr;
    CK(cudaMalloc(&d_t, sizeof(double) * 9 * T));
    CK(cudaMalloc(&d_p, sizeof(double) * 4 * (n_planes + 1)));
    CK(cudaMalloc(&d_k, (size_t)T));
    CK(cudaMemcpy(d_t, tris, sizeof(double) * 9 * T, cudaMemcpyHostToDevice));
    if (n_planes) CK(cudaMemcpy(d_p, planes, sizeof(double) * 4 * n_planes, cudaMemcpyHostToDevice));
    k_cull_mask<<<blocks_for(T, 256), 256>>>(d_t, T, d_p, n_planes, d_k);
    CK(cudaGetLastError());
    CK(cudaMemcpy(keep, d_k, (size_t)T, cudaMemcpyDeviceToHost));
    cudaFree(d_t); cudaFree(d_p); cudaFree(d_k);
    return GM_OK;
}

// A throwaway plan holding world triangles only (no samples).
static int plan_with_world_tris(int device, const double* tris, int64_t T, gm_plan** out) {
    int rc = gm_plan_create(device, out);
    if (rc) return rc;
    gm_plan* p = *out;
    p->T = T;
    p->n_clu = (T + 31) / 32;
    if (T == 0) return GM_OK;
    if ((rc = dev_alloc(&p->d_tw, (size_t)T * 9))) return rc;
    if ((rc = dev_alloc(&p->d_tsph, (size_t)T))) return rc;
    if ((rc = dev_alloc(&p->d_csph, (size_t)p->n_clu))) return rc;
    cudaStream_t s = p->stream;
    CK(cudaMemcpyAsync(p->d_tw, tris, sizeof(double) * 9 * T, cudaMemcpyHostToDevice, s));
    k_tri_spheres<<<blocks_for(T, 256), 256, 0, s>>>(p->d_tw, T, p->d_tsph);
    k_group_spheres<<<blocks_for(p->n_clu, 128), 128, 0, s>>>(p->d_tsph, nullptr, nullptr, nullptr, T, p->d_csph, 32);
    CK(cudaGetLastError());
    return GM_OK;
}

static int camera_record(gm_plan* p, const double* rot, const double* trans, double p00, double p11, double p02,
                         double p12, double near_, double far_) {
    GmFixExact e;
    memset(&e, 0, sizeof(e));
    for (int i = 0; i < 9; i++) e.rot[i] = rot[i];
    for (int i = 0; i < 3; i++) e.trans[i] = trans[i];
    e.p00 = p00;
    e.p11 = p11;
    e.p02 = p02;
    e.p12 = p12;
    e.near_ = near_;
    e.far_ = far_;
    GmFixCull c;
    memset(&c, 0, sizeof(c));
    c.cos_t = -3.0f;  // no occluder cull: kernels.rasterize sees every triangle it is given
    c.cos_s = -3.0f;
    int rc = ensure_batch(p, 1, 1, 1, std::max<int64_t>(p->cap_seg, 4096));
    if (rc) return rc;
    CK(cudaMemcpyAsync(p->d_fix, &e, sizeof(e), cudaMemcpyHostToDevice, p->stream));
    CK(cudaMemcpyAsync(p->d_cull, &c, sizeof(c), cudaMemcpyHostToDevice, p->stream));
    CK(cudaStreamSynchronize(p->stream));
    return GM_OK;
}

extern "C" int gm_rasterize(int device, const double* tris, int64_t T, const double* rot, const double* trans,
                            double p00, double p11, double p02, double p12, int W, int H, double near_, double far_,
                            double* depth, int32_t* tri_id, double* bary) {
    if (T < 0 || (T > 0 && !tris) || !rot || !trans || !depth || W < 1 || H < 1 || W > 65535 || H > 65535 ||
        T >= (1LL << 28))
        return set_err(GM_ERR_ARG, "bad arguments");
    gm_plan* p = nullptr;
    int rc = plan_with_world_tris(device, tris, T, &p);
    const bool attrs = tri_id != nullptr || bary != nullptr;
    int32_t* d_id = nullptr;
    double* d_bary = nullptr;
    if (!rc) rc = camera_record(p, rot, trans, p00, p11, p02, p12, near_, far_);
    if (!rc) rc = raster_pass(p, W, H, attrs);
    if (!rc && attrs) {
        const int64_t n = (int64_t)W * H;
        rc = dev_alloc(&d_id, (size_t)n);
        if (!rc) rc = dev_alloc(&d_bary, (size_t)n * 3);
        if (!rc) {
            k_attrs<<<blocks_for(n, 256), 256, 0, p->stream>>>(p->d_key, p->d_tw, p->d_fix, W, H, d_id, d_bary);
            if (cudaGetLastError() != cudaSuccess) rc = set_err(GM_ERR_CUDA, "k_attrs launch failed");
        }
        if (!rc && tri_id && cudaMemcpyAsync(tri_id, d_id, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, p->stream))
            rc = set_err(GM_ERR_CUDA, "copy tri_id");
        if (!rc && bary && cudaMemcpyAsync(bary, d_bary, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, p->stream))
            rc = set_err(GM_ERR_CUDA, "copy bary");
    }
    if (!rc && cudaMemcpyAsync(depth, p->d_depth, sizeof(double) * W * H, cudaMemcpyDeviceToHost, p->stream))
        rc = set_err(GM_ERR_CUDA, "copy depth");
    if (p) cudaStreamSynchronize(p->stream);
    cudaFree(d_id);
    cudaFree(d_bary);
    if (p) gm_plan_destroy(p);
    return rc;
}

extern "C" int gm_render_heatmap(int device, const double* tris, int64_t T, const double* rot, const double* trans,
                                 double p00, double p11, double p02, double p12, int W, int H, double near_,
                                 double far_, const int64_t* res, const int64_t* base, const double* values,
                                 int64_t N, const double* stops, const double* colors, int n_stops, double gamma,
                                 uint8_t* img) {
    if (T < 0 || (T > 0 && (!tris || !res || !base)) || !rot || !trans || !img || W < 1 || H < 1 || W > 65535 ||
        H > 65535 || n_stops < 2 || n_stops > 16 || !stops || !colors || N < 0 || (N > 0 && !values) ||
        T >= (1LL << 28))
        return set_err(GM_ERR_ARG, "bad arguments");
    GmColorMap cm;
    memset(&cm, 0, sizeof(cm));
    cm.n = n_stops;
    cm.gamma = gamma;
    for (int i = 0; i < n_stops; i++) {
        cm.xs[i] = stops[i];
        for (int c = 0; c < 3; c++) cm.cols[i][c] = colors[3 * i + c];
    }
    gm_plan* p = nullptr;
    int rc = plan_with_world_tris(device, tris, T, &p);
    const int64_t n = (int64_t)W * H;
    int32_t* d_id = nullptr;
    double *d_bary = nullptr, *d_vals = nullptr;
    int64_t *d_res = nullptr, *d_base = nullptr;
    uint8_t* d_img = nullptr;
    if (!rc) rc = camera_record(p, rot, trans, p00, p11, p02, p12, near_, far_);
    if (!rc) rc = raster_pass(p, W, H, true);
    if (!rc) rc = dev_alloc(&d_id, (size_t)n);
    if (!rc) rc = dev_alloc(&d_bary, (size_t)n * 3);
    if (!rc) rc = dev_alloc(&d_img, (size_t)n * 3);
    if (!rc) rc = dev_alloc(&d_vals, (size_t)std::max<int64_t>(N, 1));
    if (!rc) rc = dev_alloc(&d_res, (size_t)std::max<int64_t>(T, 1));
    if (!rc) rc = dev_alloc(&d_base, (size_t)std::max<int64_t>(T, 1));
    if (!rc) {
        cudaStream_t s = p->stream;
        if (N) cudaMemcpyAsync(d_vals, values, sizeof(double) * N, cudaMemcpyHostToDevice, s);
        if (T) {
            cudaMemcpyAsync(d_res, res, sizeof(int64_t) * T, cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(d_base, base, sizeof(int64_t) * T, cudaMemcpyHostToDevice, s);
        }
        k_attrs<<<blocks_for(n, 256), 256, 0, s>>>(p->d_key, p->d_tw, p->d_fix, W, H, d_id, d_bary);
        k_heat<<<blocks_for(n, 256), 256, 0, s>>>(d_id, d_bary, n, d_res, d_base, d_vals, cm, d_img);
        if (cudaGetLastError() != cudaSuccess) rc = set_err(GM_ERR_CUDA, "render kernels failed to launch");
        if (!rc && cudaMemcpyAsync(img, d_img, (size_t)n * 3, cudaMemcpyDeviceToHost, s))
            rc = set_err(GM_ERR_CUDA, "copy image");
        if (!rc && cudaStreamSynchronize(s)) rc = set_err(GM_ERR_CUDA, "render failed");
    }
    cudaFree(d_id); cudaFree(d_bary); cudaFree(d_img); cudaFree(d_vals); cudaFree(d_res); cudaFree(d_base);
    if (p) gm_plan_destroy(p);
    return rc;
}

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
