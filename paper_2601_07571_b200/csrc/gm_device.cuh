// gm_device.cuh -- exact float64 device helpers (compiled with -fmad=false:
// every a*b+c below is two rounded operations, exactly like the numba
// kernels, which contain no FMA -- SURVEY.md section 0 fact 1).  The only
// fused multiply-adds are the explicit __fma_rn chains that restate numpy's
// OpenBLAS call sites.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "gm_types.h"

namespace gm {

// numba int(np.ceil(x)) / int(np.floor(x)) on x86-64: cvttsd2si returns
// INT64_MIN for out-of-range input (CUDA's cvt saturates instead).
__device__ __forceinline__ long long x86_i64(double v) {
    return (v >= -9.2233720368547758e18 && v < 9.2233720368547758e18) ? (long long)v : (long long)0x8000000000000000LL;
}

// OpenBLAS dgemm/dgemv inner product, k = 0..2 (geometry.py:89 Transform.apply).
__device__ __forceinline__ double blas_dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
    double acc = __dmul_rn(a0, b0);
    acc = __fma_rn(a1, b1, acc);
    acc = __fma_rn(a2, b2, acc);
    return acc;
}

// kernels.py:62-64 _edge
__device__ __forceinline__ double edge_fn(double ax, double ay, double bx, double by, double px, double py) {
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

// Depth one screen triangle writes at pixel (px, py), +inf if the pixel is not
// owned -- the body of kernels.py:103-129 for a single pixel.  The caller has
// already checked the reference bbox (x0..x1, y0..y1).
__device__ __forceinline__ double texel_depth(const GmScreenTri& t, int px, int py, double near_, double far_) {
    double cx = (double)px + 0.5;
    double cy = (double)py + 0.5;
    double w0 = edge_fn(t.sx1, t.sy1, t.sx2, t.sy2, cx, cy);
    double w1 = edge_fn(t.sx2, t.sy2, t.sx0, t.sy0, cx, cy);
    double w2 = edge_fn(t.sx0, t.sy0, t.sx1, t.sy1, cx, cy);
    if (w0 < 0.0 || w1 < 0.0 || w2 < 0.0) return CUDART_INF;
    if (w0 == 0.0 && !(t.tl & 1u)) return CUDART_INF;
    if (w1 == 0.0 && !(t.tl & 2u)) return CUDART_INF;
    if (w2 == 0.0 && !(t.tl & 4u)) return CUDART_INF;
    double l0 = w0 * t.inv_area;
    double l1 = w1 * t.inv_area;
    double l2 = w2 * t.inv_area;
    double inv_w = l0 * t.iw0 + l1 * t.iw1 + l2 * t.iw2;
    if (inv_w <= 0.0) return CUDART_INF;
    double d = 1.0 / inv_w;
    if (d < near_ || d > far_) return CUDART_INF;
    return d;
}

// kernels.py:67-98 setup part of _raster_tri for one projected triangle:
// winding normalisation, area, clamped pixel bbox, top-left bits.
// Returns false when numba would return before the pixel loop.
__device__ __forceinline__ bool make_screen_tri(double sx[3], double sy[3], double iw[3], int W, int H,
                                                GmScreenTri* out) {
    double area = edge_fn(sx[0], sy[0], sx[1], sy[1], sx[2], sy[2]);
    if (area == 0.0) return false;
    if (area < 0.0) {
        double t;
        t = sx[1]; sx[1] = sx[2]; sx[2] = t;
        t = sy[1]; sy[1] = sy[2]; sy[2] = t;
        t = iw[1]; iw[1] = iw[2]; iw[2] = t;
        area = -area;
    }
    double minx = fmin(sx[0], fmin(sx[1], sx[2]));
    double maxx = fmax(sx[0], fmax(sx[1], sx[2]));
    double miny = fmin(sy[0], fmin(sy[1], sy[2]));
    double maxy = fmax(sy[0], fmax(sy[1], sy[2]));
    long long x0 = x86_i64(ceil(minx - 0.5));
    long long x1 = x86_i64(floor(maxx - 0.5));
    long long y0 = x86_i64(ceil(miny - 0.5));
    long long y1 = x86_i64(floor(maxy - 0.5));
    if (x0 < 0) x0 = 0;
    if (x1 > W - 1) x1 = W - 1;
    if (y0 < 0) y0 = 0;
    if (y1 > H - 1) y1 = H - 1;
    if (x1 < x0 || y1 < y0) return false;
    out->sx0 = sx[0]; out->sy0 = sy[0];
    out->sx1 = sx[1]; out->sy1 = sy[1];
    out->sx2 = sx[2]; out->sy2 = sy[2];
    out->iw0 = iw[0]; out->iw1 = iw[1]; out->iw2 = iw[2];
    out->inv_area = 1.0 / area;
    out->x0 = (uint16_t)x0; out->x1 = (uint16_t)x1;
    out->y0 = (uint16_t)y0; out->y1 = (uint16_t)y1;
    uint32_t tl = 0;
    if (sy[2] - sy[1] < 0.0 || (sy[2] == sy[1] && sx[2] - sx[1] > 0.0)) tl |= 1u;
    if (sy[0] - sy[2] < 0.0 || (sy[0] == sy[2] && sx[0] - sx[2] > 0.0)) tl |= 2u;
    if (sy[1] - sy[0] < 0.0 || (sy[1] == sy[0] && sx[1] - sx[0] > 0.0)) tl |= 4u;
    out->tl = tl;
    return true;
}

// kernels.py:140-192 per-triangle body of rasterize: camera transform,
// _clip_near, fan, projection.  Emits up to two screen triangles.
__device__ __forceinline__ int project_triangle(const double* tw, const GmFixExact& F, int W, int H,
                                                GmScreenTri out[2]) {
    double vin[3][3];
#pragma unroll
    for (int v = 0; v < 3; v++) {
        double wx = tw[3 * v], wy = tw[3 * v + 1], wz = tw[3 * v + 2];
#pragma unroll
        for (int i = 0; i < 3; i++)
            vin[v][i] = F.rot[3 * i] * wx + F.rot[3 * i + 1] * wy + F.rot[3 * i + 2] * wz + F.trans[i];
    }
    const double nn = F.near_;
    const double half_w = 0.5 * (double)W, half_h = 0.5 * (double)H;
    if (vin[0][2] <= -nn && vin[1][2] <= -nn && vin[2][2] <= -nn) {
        // no vertex behind the near plane (the common case): _clip_near returns the
        // triangle unchanged and the fan has one triangle -- the general path below
        // computes exactly this, without the dynamically indexed polygon in local memory
        double sx[3], sy[3], iw[3];
#pragma unroll
        for (int m = 0; m < 3; m++) {
            const double x = vin[m][0], y = vin[m][1], z = vin[m][2];
            const double w = -z;  // >= near' > 0
            const double ndc_x = (F.p00 * x + F.p02 * z) / w;
            const double ndc_y = (F.p11 * y + F.p12 * z) / w;
            sx[m] = (ndc_x + 1.0) * half_w;
            sy[m] = (1.0 - ndc_y) * half_h;
            iw[m] = 1.0 / w;
        }
        if (!make_screen_tri(sx, sy, iw, W, H, &out[0])) return 0;
        out[0].minw = __double2float_rd(fmin(-vin[0][2], fmin(-vin[1][2], -vin[2][2])));
        return 1;
    }
    // _clip_near (kernels.py:35-59) against z = -near'
    double vout[4][3];
    int nv = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
        int j = (i + 1) % 3;
        double cz = vin[i][2], nz = vin[j][2];
        bool cin = cz <= -nn;
        bool nin = nz <= -nn;
        if (cin) {
            vout[nv][0] = vin[i][0]; vout[nv][1] = vin[i][1]; vout[nv][2] = vin[i][2];
            nv++;
        }
        if (cin != nin) {
            double t = (-nn - cz) / (nz - cz);
#pragma unroll
            for (int c = 0; c < 3; c++) vout[nv][c] = vin[i][c] + t * (vin[j][c] - vin[i][c]);
            nv++;
        }
    }
    if (nv < 3) return 0;
    int n_out = 0;
    for (int k = 0; k < nv - 2; k++) {
        double sx[3], sy[3], iw[3];
        bool ok = true;
#pragma unroll
        for (int m = 0; m < 3; m++) {
            int src = m == 0 ? 0 : k + m;
            double x = vout[src][0], y = vout[src][1], z = vout[src][2];
            double w = -z;
            if (w <= 0.0) { ok = false; break; }
            double ndc_x = (F.p00 * x + F.p02 * z) / w;
            double ndc_y = (F.p11 * y + F.p12 * z) / w;
            sx[m] = (ndc_x + 1.0) * half_w;
            sy[m] = (1.0 - ndc_y) * half_h;
            iw[m] = 1.0 / w;
        }
        if (ok && make_screen_tri(sx, sy, iw, W, H, &out[n_out])) {
            out[n_out].tl |= (uint32_t)k << 3;  // fan index; the caller adds 2 t (rasterization order key)
            // depth written at any covered pixel = 1 / (convex combination of 1/w) >= min w
            // (up to a few ulps, far inside the 1e-9 margin k_texels applies)
            const double w0 = -vout[0][2], w1 = -vout[k + 1][2], w2 = -vout[k + 2][2];
            out[n_out].minw = __double2float_rd(fmin(w0, fmin(w1, w2)));
            n_out++;
        }
    }
    return n_out;
}

// Conservative sphere test against a fixation's cone + depth slab (float32
// with explicit slack; only ever culls work whose exact result is zero).
__device__ __forceinline__ bool sphere_visible(const GmFixCull& c, float4 s, bool occluder_cone) {
    float cosA = occluder_cone ? c.cos_t : c.cos_s;
    float sinA = occluder_cone ? c.sin_t : c.sin_s;
    if (cosA < -2.5f) return true;  // culling disabled
    float vx = s.x - c.ox, vy = s.y - c.oy, vz = s.z - c.oz;
    float m = s.w + c.margin;
    float along = __fmaf_rn(vx, c.gx, __fmaf_rn(vy, c.gy, vz * c.gz));
    if (cosA > -1.5f) {
        // the cone (half-angle < 1.5 rad) lies in front of the apex
        if (along < -m) return false;
        float cx = vy * c.gz - vz * c.gy;
        float cy = vz * c.gx - vx * c.gz;
        float cz = vx * c.gy - vy * c.gx;
        float perp = sqrtf(__fmaf_rn(cx, cx, __fmaf_rn(cy, cy, cz * cz)));
        // lower bound of the distance from the sphere centre to the cone
        if (perp * cosA - along * sinA > m) return false;
    } else if (!occluder_cone && along < -m) {
        return false;  // a contributing sample has d1 > 0 (kernels.py:331)
    }
    float fwd = __fmaf_rn(vx, c.fx, __fmaf_rn(vy, c.fy, vz * c.fz));
    if (fwd < c.near_f - m || fwd > c.far_f + m) return false;
    return true;
}

}  // namespace gm
