// gm_kernels.cu -- sm_100a kernels and the C-ABI of the B200 density-map path.
//
// Path and where each piece lives:
//   a1-a6  sampling: k_layout (Heron area -> r -> count), CUB scan (offsets),
//          k_positions (index -> row/col -> barycentric -> world, FMA-chain
//          transform like OpenBLAS), k_world_tris
//   a8-a10 per-fixation setup: host, gm_setup.cpp (glibc trig, bit-exact)
//   a11-a12 occluders: k_tri_setup (conservative cone cull, exact camera
//          transform + near clip + projection + _raster_tri setup) and
//          k_bin_count / k_bin_fill (16x16-pixel screen bins)
//   a13-a15 k_accumulate: sample-major, one warp per 32-sample chunk, fixation
//          culling by warp ballot, exact NDC filter, exact 4-sigma Gaussian,
//          and depth_match evaluated on the texels it reads (the z-buffer
//          value of a texel = min over the binned screen triangles covering
//          it, computed with the reference's own pixel arithmetic)
//   a16    k_max / k_normalize
// Exactness: compiled with -fmad=false; see gm_device.cuh.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "gm_device.cuh"
#include "gm_types.h"

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
                                float4* __restrict__ out) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t first = g * 32;
    if (first >= n) return;
    int64_t last = first + 32 < n ? first + 32 : n;
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

// One warp per group of 32 triangle clusters (32 triangles each); blockIdx.y =
// fixation slot.  Lane-parallel cluster test -> ballot -> per passing cluster
// lane = triangle: sphere test, exact projection, warp-aggregated append.
__global__ void __launch_bounds__(256) k_tri_setup(const double* __restrict__ tw, int64_t T,
                                                   const float4* __restrict__ tsph, const float4* __restrict__ csph,
                                                   int64_t n_clu, const GmFixExact* __restrict__ fixes,
                                                   const GmFixCull* __restrict__ culls, int W, int H,
                                                   GmScreenTri* __restrict__ pool, int64_t cap,
                                                   unsigned long long* __restrict__ counter) {
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
    while (mask) {
        int j = __ffs(mask) - 1;
        mask &= mask - 1;
        int64_t t = (c0 + j) * 32 + lane;
        GmScreenTri out[2];
        int n = 0;
        if (t < T && sphere_visible(cull, tsph[t], true)) {
            n = project_triangle(tw + 9 * t, F, W, H, out);
        }
        // warp-aggregated append
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(counter, (unsigned long long)total);
        base = __shfl_sync(0xffffffffu, base, 31);
        unsigned long long at = base + (unsigned long long)(incl - n);
        for (int q = 0; q < n; q++) {
            if (at + q < (unsigned long long)cap) {
                out[q].fslot = f;
                pool[at + q] = out[q];
            }
        }
    }
}

__global__ void k_bin_count(const GmScreenTri* __restrict__ pool, const unsigned long long* __restrict__ counter,
                            int64_t cap, int nbx, int nbins, int* __restrict__ bin_count) {
    int64_t n = (int64_t)min(*counter, (unsigned long long)cap);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const GmScreenTri& t = pool[i];
        int bx0 = t.x0 >> GM_BIN_SHIFT, bx1 = t.x1 >> GM_BIN_SHIFT;
        int by0 = t.y0 >> GM_BIN_SHIFT, by1 = t.y1 >> GM_BIN_SHIFT;
        int* base = bin_count + (int64_t)t.fslot * nbins;
        for (int by = by0; by <= by1; by++)
            for (int bx = bx0; bx <= bx1; bx++) atomicAdd(base + by * nbx + bx, 1);
    }
}

__global__ void k_bin_fill(const GmScreenTri* __restrict__ pool, const unsigned long long* __restrict__ counter,
                           int64_t cap, int nbx, int nbins, int* __restrict__ cursor, int* __restrict__ items,
                           int64_t cap_items) {
    int64_t n = (int64_t)min(*counter, (unsigned long long)cap);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const GmScreenTri& t = pool[i];
        int bx0 = t.x0 >> GM_BIN_SHIFT, bx1 = t.x1 >> GM_BIN_SHIFT;
        int by0 = t.y0 >> GM_BIN_SHIFT, by1 = t.y1 >> GM_BIN_SHIFT;
        int* base = cursor + (int64_t)t.fslot * nbins;
        for (int by = by0; by <= by1; by++)
            for (int bx = bx0; bx <= bx1; bx++) {
                int at = atomicAdd(base + by * nbx + bx, 1);
                if (at < cap_items) items[at] = (int)i;
            }
    }
}

// ----------------------------------------------------- texel evaluation

struct BinView {
    const GmScreenTri* tris;
    const int* off;   // exclusive offsets, length nbins*B + 1
    const int* items;
    int nbx, nbins;
};

// Min depth of the texel block [bx0, bx0+nx) x [by0, by0+ny) (nx, ny <= 3),
// i.e. the z-buffer values kernels.rasterize would leave there, evaluated only
// for these texels.  T[ry*3+rx].
__device__ __forceinline__ void eval_block(const BinView& bv, int fslot, int bx0, int by0, int nx, int ny,
                                           double near_, double far_, double T[9]) {
#pragma unroll
    for (int q = 0; q < 9; q++) T[q] = CUDART_INF;
    const int bxa = bx0 >> GM_BIN_SHIFT, bxb = (bx0 + nx - 1) >> GM_BIN_SHIFT;
    const int bya = by0 >> GM_BIN_SHIFT, byb = (by0 + ny - 1) >> GM_BIN_SHIFT;
    const int64_t fb = (int64_t)fslot * bv.nbins;
    for (int biy = bya; biy <= byb; biy++) {
        for (int bix = bxa; bix <= bxb; bix++) {
            // texels of the block that belong to this bin
            int tx_lo = max(bx0, bix << GM_BIN_SHIFT), tx_hi = min(bx0 + nx - 1, (bix << GM_BIN_SHIFT) + GM_BIN - 1);
            int ty_lo = max(by0, biy << GM_BIN_SHIFT), ty_hi = min(by0 + ny - 1, (biy << GM_BIN_SHIFT) + GM_BIN - 1);
            int64_t b = fb + biy * bv.nbx + bix;
            int s = bv.off[b], e = bv.off[b + 1];
            for (int it = s; it < e; it++) {
                const GmScreenTri* tp = bv.tris + bv.items[it];
                uint2 bb = *reinterpret_cast<const uint2*>(&tp->x0);  // x0,x1,y0,y1 (uint16 x4)
                int x0 = bb.x & 0xffff, x1 = bb.x >> 16, y0 = bb.y & 0xffff, y1 = bb.y >> 16;
                int lx = max(tx_lo, x0), hx = min(tx_hi, x1);
                int ly = max(ty_lo, y0), hy = min(ty_hi, y1);
                if (lx > hx || ly > hy) continue;
                GmScreenTri tri = *tp;
#pragma unroll
                for (int ry = 0; ry < 3; ry++) {
#pragma unroll
                    for (int rx = 0; rx < 3; rx++) {
                        int px = bx0 + rx, py = by0 + ry;
                        if (px >= lx && px <= hx && py >= ly && py <= hy) {
                            double d = texel_depth(tri, px, py, near_, far_);
                            if (d < T[ry * 3 + rx]) T[ry * 3 + rx] = d;
                        }
                    }
                }
            }
        }
    }
}

// kernels.py:219-285 depth_match, reading texels from the evaluated block.
__device__ __forceinline__ bool depth_match_eval(const BinView& bv, int fslot, int W, int H, double fx, double fy,
                                                 double d, double eps, double near_, double far_) {
    double gx = fx - 0.5, gy = fy - 0.5;
    long long cx = x86_i64(rint(gx));  // np.round: half to even
    if (cx < 0) cx = 0;
    else if (cx > W - 1) cx = W - 1;
    long long cy = x86_i64(rint(gy));
    if (cy < 0) cy = 0;
    else if (cy > H - 1) cy = H - 1;
    int bx0 = (int)max(cx - 1, 0LL), bx1 = (int)min(cx + 1, (long long)W - 1);
    int by0 = (int)max(cy - 1, 0LL), by1 = (int)min(cy + 1, (long long)H - 1);
    double T[9];
    eval_block(bv, fslot, bx0, by0, bx1 - bx0 + 1, by1 - by0 + 1, near_, far_, T);
    if (W > 1 && H > 1) {
        long long x0 = x86_i64(floor(gx));
        if (x0 < 0) x0 = 0;
        else if (x0 > W - 2) x0 = W - 2;
        long long y0 = x86_i64(floor(gy));
        if (y0 < 0) y0 = 0;
        else if (y0 > H - 2) y0 = H - 2;
        int ix = (int)(x0 - bx0), iy = (int)(y0 - by0);  // quad inside the 3x3 block
        double q00 = T[iy * 3 + ix], q01 = T[iy * 3 + ix + 1];
        double q10 = T[(iy + 1) * 3 + ix], q11 = T[(iy + 1) * 3 + ix + 1];
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
#pragma unroll
    for (int ry = 0; ry < 3; ry++)
#pragma unroll
        for (int rx = 0; rx < 3; rx++) {
            if (rx <= bx1 - bx0 && ry <= by1 - by0) {
                double t = T[ry * 3 + rx];
                if (isfinite(t)) {
                    double diff = fabs(t - d);
                    if (diff < best) best = diff;
                }
            }
        }
    return best <= eps;
}

// ------------------------------------------------------ the hot kernel

// Sample-major fused filter + visibility + Gaussian (kernels.py:288-340 for a
// batch of fixations).  A warp owns 32 consecutive samples (one value slot per
// lane, kept in a register across the batch); lane l first tests fixation g+l
// against the chunk sphere, the ballot gives the fixations that can touch the
// chunk, and those are applied in log order -> per-sample accumulation order is
// the reference's (density.py:223-226), deterministic, no atomics.
// The cone test (kernels.py:330-339) is evaluated before depth_match
// (kernels.py:326): all conditions are conjunctive and side-effect free, so the
// set of contributing samples and their weights are unchanged.
__global__ void __launch_bounds__(256) k_accumulate(const double* __restrict__ px, const double* __restrict__ py,
                                                    const double* __restrict__ pz, const float4* __restrict__ chunks,
                                                    int64_t N, int64_t n_chunks, const GmFixExact* __restrict__ fixes,
                                                    const GmFixCull* __restrict__ culls, int B, BinView bv, int W,
                                                    int H, double inv_sigma, double eps_abs, double eps_rel,
                                                    double* __restrict__ values) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const double Wd = (double)W, Hd = (double)H;
    const double lo = -1.0 - GM_NDC_SLACK, hi = 1.0 + GM_NDC_SLACK;
    for (int64_t ch = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); ch < n_chunks; ch += warps) {
        const int64_t i = ch * 32 + lane;
        const bool valid = i < N;
        double wx = 0.0, wy = 0.0, wz = 0.0, v = 0.0;
        if (valid) {
            wx = px[i];
            wy = py[i];
            wz = pz[i];
            v = values[i];
        }
        const float4 sph = chunks[ch];
        for (int g = 0; g < B; g += 32) {
            const int myf = g + lane;
            bool pass = myf < B && sphere_visible(culls[myf], sph, false);
            unsigned mask = __ballot_sync(0xffffffffu, pass);
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                if (!valid) continue;
                const GmFixExact& F = fixes[g + j];
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
                // kernels.py:330-339 (moved before the depth test)
                double d1 = x * F.gaze[0] + y * F.gaze[1] + z * F.gaze[2];
                if (d1 <= 0.0) continue;
                double d2sq = x * x + y * y + z * z - d1 * d1;
                if (d2sq < 0.0) d2sq = 0.0;
                double ratio_sq = d2sq * inv_sigma * inv_sigma / (d1 * d1);
                if (ratio_sq > 16.0) continue;
                // kernels.py:323-329
                double eps = eps_abs;
                if (eps_rel * d > eps) eps = eps_rel * d;
                if (!depth_match_eval(bv, g + j, W, H, (ndc_x + 1.0) * 0.5 * Wd, (1.0 - ndc_y) * 0.5 * Hd, d, eps,
                                      F.near_, F.far_))
                    continue;
                v += F.amp * exp(-0.5 * ratio_sq);  // kernels.py:340
            }
        }
        if (valid) values[i] = v;
    }
}

// Full depth buffer of one fixation slot via the same texel evaluator
// (kernel-seam port of kernels.rasterize, used by parity tests).
__global__ void k_depth_full(BinView bv, int fslot, int W, int H, double near_, double far_, double* __restrict__ depth) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= (int64_t)W * H) return;
    int px = (int)(p % W), py = (int)(p / W);
    double T[9];
    eval_block(bv, fslot, px, py, 1, 1, near_, far_, T);
    depth[p] = T[0];
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
    float4* d_chunk = nullptr;
    double* d_values = nullptr;
    // batch buffers
    int cap_B = 0;
    GmFixExact* d_fix = nullptr;
    GmFixCull* d_cull = nullptr;
    GmFixExact* h_fix = nullptr;
    GmFixCull* h_cull = nullptr;
    GmScreenTri* d_pool = nullptr;
    int64_t cap_pool = 0;
    unsigned long long* d_counter = nullptr;  // [0] = screen tris
    unsigned long long* h_counter = nullptr;  // pinned: [0] tris, [1] items
    int* d_bin_count = nullptr;
    int* d_bin_off = nullptr;
    int* d_cursor = nullptr;
    int64_t cap_bins = 0;
    int* d_items = nullptr;
    int64_t cap_items = 0;
    void* d_scan_tmp = nullptr;
    size_t scan_tmp_bytes = 0;
    unsigned long long* d_max = nullptr;
    int host_threads = 8;
    // device-resident setup table (gm_plan_prepare)
    GmFixExact* d_fix_all = nullptr;
    GmFixCull* d_cull_all = nullptr;
    int64_t F_prepared = -1;
    GmConfig cfg_prepared{};
    void* d_flush = nullptr;
    int64_t flush_bytes = 0;
    int flush_gen = 0;
};

static void plan_free_scene(gm_plan* p) {
    cudaFree(p->d_tw); cudaFree(p->d_tsph); cudaFree(p->d_csph);
    cudaFree(p->d_px); cudaFree(p->d_py); cudaFree(p->d_pz);
    cudaFree(p->d_chunk); cudaFree(p->d_values);
    p->d_tw = nullptr; p->d_tsph = p->d_csph = p->d_chunk = nullptr;
    p->d_px = p->d_py = p->d_pz = p->d_values = nullptr;
    p->T = p->n_clu = p->N = p->n_chunks = 0;
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
    CK(cudaMalloc(&p->d_counter, 4 * sizeof(unsigned long long)));
    CK(cudaMalloc(&p->d_max, sizeof(unsigned long long)));
    CK(cudaMallocHost(&p->h_counter, 4 * sizeof(unsigned long long)));
    unsigned hc = std::thread::hardware_concurrency();
    p->host_threads = hc > 0 ? (int)hc : 8;
    *out = p;
    return GM_OK;
}

extern "C" void gm_plan_destroy(gm_plan* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    plan_free_scene(p);
    cudaFree(p->d_fix); cudaFree(p->d_cull);
    cudaFreeHost(p->h_fix); cudaFreeHost(p->h_cull); cudaFreeHost(p->h_counter);
    cudaFree(p->d_pool); cudaFree(p->d_counter); cudaFree(p->d_bin_count); cudaFree(p->d_bin_off);
    cudaFree(p->d_cursor); cudaFree(p->d_items); cudaFree(p->d_scan_tmp); cudaFree(p->d_max);
    cudaFree(p->d_fix_all); cudaFree(p->d_cull_all); cudaFree(p->d_flush);
    cudaStreamDestroy(p->stream);
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
    int rc;
    if ((rc = dev_alloc(&p->d_tw, (size_t)T * 9))) return rc;
    if ((rc = dev_alloc(&p->d_tsph, (size_t)T))) return rc;
    if ((rc = dev_alloc(&p->d_csph, (size_t)p->n_clu))) return rc;
    if ((rc = dev_alloc(&p->d_px, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_py, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_pz, (size_t)N))) return rc;
    if ((rc = dev_alloc(&p->d_chunk, (size_t)p->n_chunks))) return rc;
    if ((rc = dev_alloc(&p->d_values, (size_t)N))) return rc;
    if (T == 0) return GM_OK;
    double *d_local = nullptr, *d_M = nullptr;
    int64_t *d_res = nullptr, *d_cnt = nullptr, *d_off = nullptr;
    if ((rc = dev_alloc(&d_local, (size_t)T * 9))) return rc;
    if ((rc = dev_alloc(&d_M, (size_t)n_obj * 12))) return rc;
    if ((rc = dev_alloc(&d_res, (size_t)T))) return rc;
    if ((rc = dev_alloc(&d_cnt, (size_t)T))) return rc;
    if ((rc = dev_alloc(&d_off, (size_t)T))) return rc;
    std::vector<double> Mt(n_obj * 12);
    for (int o = 0; o < n_obj; o++) xform_matrix(xforms + 10 * o, &Mt[12 * o], &Mt[12 * o + 9]);
    cudaStream_t s = p->stream;
    CK(cudaMemcpyAsync(d_local, tri_local, sizeof(double) * 9 * T, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_M, Mt.data(), sizeof(double) * 12 * n_obj, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_res, res, sizeof(int64_t) * T, cudaMemcpyHostToDevice, s));
    int64_t sample_base = 0;
    for (int o = 0; o < n_obj; o++) {
        int64_t To = tri_counts[o];
        if (To == 0) continue;
        const double* loc = d_local + 9 * tstart[o];
        k_world_tris<<<blocks_for(3 * To, 256), 256, 0, s>>>(loc, To, d_M + 12 * o, d_M + 12 * o + 9,
                                                              p->d_tw + 9 * tstart[o]);
        if (!include[o] || nsamp[o] == 0) continue;
        k_layout<<<blocks_for(To, 256), 256, 0, s>>>(loc, To, 0.0, d_res + tstart[o], nullptr,
                                                       d_cnt + tstart[o]);
        size_t tmp = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_cnt + tstart[o], d_off + tstart[o], To, s);
        if (tmp > p->scan_tmp_bytes) {
            cudaFree(p->d_scan_tmp);
            p->d_scan_tmp = nullptr;
            CK(cudaMalloc(&p->d_scan_tmp, tmp));
            p->scan_tmp_bytes = tmp;
        }
        CK(cub::DeviceScan::ExclusiveSum(p->d_scan_tmp, tmp, d_cnt + tstart[o], d_off + tstart[o], To, s));
        int64_t No = nsamp[o];
        k_positions<<<blocks_for(No, 256), 256, 0, s>>>(loc, To, d_res + tstart[o], d_off + tstart[o], No,
                                                          d_M + 12 * o, d_M + 12 * o + 9, nullptr,
                                                          p->d_px + sample_base, p->d_py + sample_base,
                                                          p->d_pz + sample_base);
        sample_base += No;
    }
    k_tri_spheres<<<blocks_for(T, 256), 256, 0, s>>>(p->d_tw, T, p->d_tsph);
    k_group_spheres<<<blocks_for(p->n_clu, 128), 128, 0, s>>>(p->d_tsph, nullptr, nullptr, nullptr, T, p->d_csph);
    if (N > 0)
        k_group_spheres<<<blocks_for(p->n_chunks, 128), 128, 0, s>>>(nullptr, p->d_px, p->d_py, p->d_pz, N,
                                                                      p->d_chunk);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    cudaFree(d_local); cudaFree(d_M); cudaFree(d_res); cudaFree(d_cnt); cudaFree(d_off);
    return GM_OK;
}

extern "C" int64_t gm_plan_num_samples(gm_plan* p) { return p ? p->N : -1; }
extern "C" int64_t gm_plan_num_triangles(gm_plan* p) { return p ? p->T : -1; }
extern "C" double* gm_plan_values_device(gm_plan* p) { return p ? p->d_values : nullptr; }

static int ensure_batch(gm_plan* p, int B, int nbins) {
    int rc;
    if (B > p->cap_B) {
        if ((rc = dev_alloc(&p->d_fix, (size_t)B))) return rc;
        if ((rc = dev_alloc(&p->d_cull, (size_t)B))) return rc;
        cudaFreeHost(p->h_fix);
        cudaFreeHost(p->h_cull);
        CK(cudaMallocHost(&p->h_fix, sizeof(GmFixExact) * B));
        CK(cudaMallocHost(&p->h_cull, sizeof(GmFixCull) * B));
        p->cap_B = B;
    }
    int64_t nb = (int64_t)B * nbins;
    if (nb + 1 > p->cap_bins) {
        if ((rc = dev_alloc(&p->d_bin_count, (size_t)nb + 1))) return rc;
        if ((rc = dev_alloc(&p->d_bin_off, (size_t)nb + 1))) return rc;
        if ((rc = dev_alloc(&p->d_cursor, (size_t)nb + 1))) return rc;
        p->cap_bins = nb + 1;
        size_t tmp = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp, p->d_bin_count, p->d_bin_off, (int)(nb + 1), p->stream);
        if (tmp > p->scan_tmp_bytes) {
            cudaFree(p->d_scan_tmp);
            p->d_scan_tmp = nullptr;
            CK(cudaMalloc(&p->d_scan_tmp, tmp));
            p->scan_tmp_bytes = tmp;
        }
    }
    if (p->cap_pool == 0) {
        p->cap_pool = std::max<int64_t>(1 << 20, (int64_t)B * 4096);
        if ((rc = dev_alloc(&p->d_pool, (size_t)p->cap_pool))) return rc;
    }
    if (p->cap_items == 0) {
        p->cap_items = std::max<int64_t>(1 << 22, (int64_t)B * 16384);
        if ((rc = dev_alloc(&p->d_items, (size_t)p->cap_items))) return rc;
    }
    return GM_OK;
}

// Occluder setup + binning for one batch already uploaded to d_fix/d_cull.
// Grows the pools and retries on overflow; leaves d_bin_off ready.
static int run_occluders(gm_plan* p, const GmFixExact* d_fix, const GmFixCull* d_cull, int nb, int W, int H, int nbx,
                         int nbins, cudaEvent_t ev_a, cudaEvent_t ev_b, int64_t* n_tris, int64_t* n_items) {
    cudaStream_t s = p->stream;
    for (int attempt = 0; attempt < 8; attempt++) {
        int64_t nbn = (int64_t)nb * nbins;
        CK(cudaMemsetAsync(p->d_counter, 0, sizeof(unsigned long long), s));
        CK(cudaMemsetAsync(p->d_bin_count, 0, sizeof(int) * (nbn + 1), s));
        if (ev_a) CK(cudaEventRecord(ev_a, s));
        if (p->n_clu > 0) {
            dim3 grid(blocks_for((p->n_clu + 31) / 32, 8), nb);
            k_tri_setup<<<grid, 256, 0, s>>>(p->d_tw, p->T, p->d_tsph, p->d_csph, p->n_clu, d_fix, d_cull, W, H,
                                             p->d_pool, p->cap_pool, p->d_counter);
        }
        if (ev_b) CK(cudaEventRecord(ev_b, s));
        k_bin_count<<<p->sms * 8, 256, 0, s>>>(p->d_pool, p->d_counter, p->cap_pool, nbx, nbins, p->d_bin_count);
        size_t tmp = p->scan_tmp_bytes;
        CK(cub::DeviceScan::ExclusiveSum(p->d_scan_tmp, tmp, p->d_bin_count, p->d_bin_off, (int)(nbn + 1), s));
        CK(cudaMemcpyAsync(p->h_counter, p->d_counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(p->h_counter + 1, p->d_bin_off + nbn, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));
        unsigned long long ntri = p->h_counter[0];
        int64_t nitems = (int64_t)(int)(p->h_counter[1] & 0xffffffffull);
        bool grow = false;
        if ((int64_t)ntri > p->cap_pool) {
            int rc = dev_alloc(&p->d_pool, (size_t)(ntri + ntri / 2 + 1024));
            if (rc) return rc;
            p->cap_pool = (int64_t)(ntri + ntri / 2 + 1024);
            grow = true;
        }
        if (!grow && (nitems < 0 || nitems > p->cap_items)) {
            if (nitems < 0) return set_err(GM_ERR_OOM, "bin item count overflows int32; lower the batch size");
            int rc = dev_alloc(&p->d_items, (size_t)(nitems + nitems / 2 + 1024));
            if (rc) return rc;
            p->cap_items = nitems + nitems / 2 + 1024;
        }
        if (grow) continue;  // pool overflowed: bins are incomplete, redo
        CK(cudaMemcpyAsync(p->d_cursor, p->d_bin_off, sizeof(int) * (nbn + 1), cudaMemcpyDeviceToDevice, s));
        k_bin_fill<<<p->sms * 8, 256, 0, s>>>(p->d_pool, p->d_counter, p->cap_pool, nbx, nbins, p->d_cursor,
                                             p->d_items, p->cap_items);
        CK(cudaGetLastError());
        *n_tris = (int64_t)ntri;
        *n_items = nitems;
        return GM_OK;
    }
    return set_err(GM_ERR_OOM, "screen-triangle pool kept overflowing");
}

typedef void (*gm_progress_fn)(int64_t done, int64_t total, void* user);

static inline double wall_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// One pass over F fixations in batches.  Either `fx` (host table: the host
// setup of each batch runs while the GPU works on the previous one) or the
// prepared device setup table (gm_plan_prepare) supplies the per-fixation
// records.  device_ms (optional) = CUDA-event time on the plan stream.
static int run_batches(gm_plan* p, const double* fx, int64_t F, const GmConfig* cfg, int reset, GmTimings* tm,
                       gm_progress_fn progress, void* user, int64_t* bad_fixation, float* device_ms) {
    if (cfg->zbuffer_resolution < 1 || cfg->zbuffer_resolution > 65535)
        return set_err(GM_ERR_ARG, "zbuffer_resolution must be in [1, 65535]");
    if (!(cfg->theta > 0.0 && cfg->theta < 1.5707963267948966)) return set_err(GM_ERR_ARG, "theta out of range");
    CK(cudaSetDevice(p->device));
    const bool prepared = fx == nullptr;
    double t_start = wall_ms();
    const int W = cfg->zbuffer_resolution, H = cfg->zbuffer_resolution;
    const int nbx = (W + GM_BIN - 1) / GM_BIN, nby = (H + GM_BIN - 1) / GM_BIN;
    const int nbins = nbx * nby;
    int B = cfg->batch > 0 ? cfg->batch : 512;
    if (B > 4096) B = 4096;
    int64_t max_b = std::max<int64_t>(1, (int64_t)(1 << 26) / nbins);  // bins per batch <= 64M
    if (B > max_b) B = (int)max_b;
    if (F > 0 && B > F) B = (int)F;
    GmSetupConsts consts;
    gm_setup_consts(cfg->theta, cfg->filtering, W, H, &consts);
    int rc = ensure_batch(p, std::max(B, 1), nbins);
    if (rc) return rc;
    cudaStream_t s = p->stream;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;
    if (device_ms) {
        CK(cudaEventCreate(&ev_start));
        CK(cudaEventCreate(&ev_end));
        CK(cudaEventRecord(ev_start, s));
    }
    if (reset && p->N > 0) CK(cudaMemsetAsync(p->d_values, 0, sizeof(double) * p->N, s));
    GmTimings t;
    memset(&t, 0, sizeof(t));
    std::vector<cudaEvent_t> evs;
    const bool timing = tm != nullptr;
    double inv_sigma = 1.0 / consts.sigma;
    BinView bv{p->d_pool, p->d_bin_off, p->d_items, nbx, nbins};
    int64_t done_reported = 0;
    auto cleanup = [&]() {
        for (auto e : evs) cudaEventDestroy(e);
        if (ev_start) cudaEventDestroy(ev_start);
        if (ev_end) cudaEventDestroy(ev_end);
    };
    for (int64_t b0 = 0; b0 < F; b0 += B) {
        int nb = (int)std::min<int64_t>(B, F - b0);
        GmFixExact* d_fix = p->d_fix;
        GmFixCull* d_cull = p->d_cull;
        if (prepared) {
            d_fix = p->d_fix_all + b0;
            d_cull = p->d_cull_all + b0;
        } else {
            double ts = wall_ms();
            int64_t bad = gm_setup_batch(fx + GM_FIX_STRIDE * b0, nb, &consts, p->h_fix, p->h_cull, p->host_threads);
            t.setup_ms += wall_ms() - ts;
            if (bad >= 0) {
                cudaStreamSynchronize(s);
                cleanup();
                if (bad_fixation) *bad_fixation = b0 + bad;
                return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
            }
            CK(cudaMemcpyAsync(p->d_fix, p->h_fix, sizeof(GmFixExact) * nb, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(p->d_cull, p->h_cull, sizeof(GmFixCull) * nb, cudaMemcpyHostToDevice, s));
        }
        cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
        if (timing) {
            for (int q = 0; q < 4; q++) {
                CK(cudaEventCreate(&e[q]));
                evs.push_back(e[q]);
            }
        }
        int64_t ntri = 0, nitems = 0;
        rc = run_occluders(p, d_fix, d_cull, nb, W, H, nbx, nbins, e[0], e[1], &ntri, &nitems);
        if (rc) {
            cleanup();
            return rc;
        }
        // the previous batch's accumulate finished before this batch's sync
        if (progress && b0 > done_reported) {
            progress(b0, F, user);
            done_reported = b0;
        }
        t.screen_tris += ntri;
        t.bin_items += nitems;
        t.batches += 1;
        if (timing) CK(cudaEventRecord(e[2], s));
        if (p->n_chunks > 0) {
            int grid = (int)std::min<int64_t>((p->n_chunks + 7) / 8, (int64_t)p->sms * 64);
            k_accumulate<<<grid, 256, 0, s>>>(p->d_px, p->d_py, p->d_pz, p->d_chunk, p->N, p->n_chunks, d_fix, d_cull,
                                              nb, bv, W, H, inv_sigma, cfg->eps_abs, cfg->eps_rel, p->d_values);
        }
        if (timing) CK(cudaEventRecord(e[3], s));
        CK(cudaGetLastError());
    }
    if (device_ms) CK(cudaEventRecord(ev_end, s));
    CK(cudaStreamSynchronize(s));
    if (device_ms) cudaEventElapsedTime(device_ms, ev_start, ev_end);
    if (progress && F > done_reported) progress(F, F, user);
    if (timing) {
        for (size_t q = 0; q + 3 < evs.size(); q += 4) {
            float a = 0, b = 0, c = 0;
            cudaEventElapsedTime(&a, evs[q], evs[q + 1]);
            cudaEventElapsedTime(&c, evs[q + 1], evs[q + 2]);
            cudaEventElapsedTime(&b, evs[q + 2], evs[q + 3]);
            t.cull_ms += a;
            t.rasterize_ms += c;
            t.accumulate_ms += b;
        }
        t.total_ms = wall_ms() - t_start;
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
extern "C" int gm_plan_run(gm_plan* p, int reset, GmTimings* tm, float* device_ms) {
    if (!p) return set_err(GM_ERR_ARG, "null plan");
    if (p->F_prepared < 0) return set_err(GM_ERR_ARG, "gm_plan_prepare was not called");
    return run_batches(p, nullptr, p->F_prepared, &p->cfg_prepared, reset, tm, nullptr, nullptr, nullptr, device_ms);
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

// kernels.rasterize for the plan's occluders under fixation `fx` (18 floats):
// the whole res x res depth buffer (+inf where nothing is drawn), evaluated by
// the same binned texel evaluator k_accumulate uses.  When no_cull != 0 the
// occluder cone cull is disabled (every triangle is projected).
extern "C" int gm_plan_depth_buffer(gm_plan* p, const double* fx, double theta, int filtering, int res, int no_cull,
                                    double* depth) {
    if (!p || !fx || !depth || res < 1 || res > 65535) return set_err(GM_ERR_ARG, "bad arguments");
    CK(cudaSetDevice(p->device));
    const int nbx = (res + GM_BIN - 1) / GM_BIN, nbins = nbx * nbx;
    GmSetupConsts c;
    gm_setup_consts(theta, filtering, res, res, &c);
    int rc = ensure_batch(p, 1, nbins);
    if (rc) return rc;
    int64_t bad = gm_setup_batch(fx, 1, &c, p->h_fix, p->h_cull, 1);
    if (bad >= 0) return set_err(GM_ERR_INVALID_FRUSTUM, "degenerate frustum bounds (InvalidFrustumError)");
    if (no_cull) {
        GmFixCull& k = p->h_cull[0];
        k.cos_t = -3.0f;  // sphere_visible: no culling at all
    }
    cudaStream_t s = p->stream;
    CK(cudaMemcpyAsync(p->d_fix, p->h_fix, sizeof(GmFixExact), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(p->d_cull, p->h_cull, sizeof(GmFixCull), cudaMemcpyHostToDevice, s));
    int64_t ntri = 0, nitems = 0;
    rc = run_occluders(p, p->d_fix, p->d_cull, 1, res, res, nbx, nbins, nullptr, nullptr, &ntri, &nitems);
    if (rc) return rc;
    double* d_depth = nullptr;
    CK(cudaMallocAsync(&d_depth, sizeof(double) * res * res, s));
    BinView bv{p->d_pool, p->d_bin_off, p->d_items, nbx, nbins};
    k_depth_full<<<blocks_for((int64_t)res * res, 256), 256, 0, s>>>(bv, 0, res, res, p->h_fix[0].near_,
                                                                      p->h_fix[0].far_, d_depth);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(depth, d_depth, sizeof(double) * res * res, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d_depth, s));
    CK(cudaStreamSynchronize(s));
    return GM_OK;
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
