// gm_host.cpp -- scalar host entry points of the kernel seam that a caller
// uses one query at a time (compiled with -ffp-contract=off, like numba's
// FMA-free kernels).
#include <math.h>
#include <stdint.h>
#include <string.h>

namespace {

// numba int(np.floor(x)) / int(np.round(x)) on x86-64 (cvttsd2si: INT64_MIN when out of range)
inline long long x86_i64(double v) {
    return (v >= -9.2233720368547758e18 && v < 9.2233720368547758e18) ? (long long)v : (long long)0x8000000000000000LL;
}

}  // namespace

extern "C" {

// kernels.depth_match (kernels.py:219-285) on a host (H, W) depth buffer:
// bilinear over the 2x2 quad on smooth coverage, any finite texel of the 3x3
// neighbourhood of round-half-even(g) at depth edges.  The device copy of this
// test runs inside k_samples (depth_test in gm_kernels.cu).
int gm_depth_match(const double* depth, int64_t height, int64_t width, double fx, double fy, double d, double eps) {
    const double gx = fx - 0.5, gy = fy - 0.5;
    if (width > 1 && height > 1) {
        long long x0 = x86_i64(floor(gx));
        if (x0 < 0) x0 = 0;
        else if (x0 > width - 2) x0 = width - 2;
        long long y0 = x86_i64(floor(gy));
        if (y0 < 0) y0 = 0;
        else if (y0 > height - 2) y0 = height - 2;
        const double q00 = depth[y0 * width + x0], q01 = depth[y0 * width + x0 + 1];
        const double q10 = depth[(y0 + 1) * width + x0], q11 = depth[(y0 + 1) * width + x0 + 1];
        if (isfinite(q00) && isfinite(q01) && isfinite(q10) && isfinite(q11)) {
            double tx = gx - (double)x0;
            if (tx < 0.0) tx = 0.0;
            else if (tx > 1.0) tx = 1.0;
            double ty = gy - (double)y0;
            if (ty < 0.0) ty = 0.0;
            else if (ty > 1.0) ty = 1.0;
            const double top = q00 * (1.0 - tx) + q01 * tx;
            const double bot = q10 * (1.0 - tx) + q11 * tx;
            if (fabs(d - (top * (1.0 - ty) + bot * ty)) <= eps) return 1;
            const double hi = fmax(fmax(q00, q01), fmax(q10, q11));
            const double lo = fmin(fmin(q00, q01), fmin(q10, q11));
            if (hi - lo <= eps) return 0;
        }
    }
    long long cx = x86_i64(rint(gx));
    if (cx < 0) cx = 0;
    else if (cx > width - 1) cx = width - 1;
    long long cy = x86_i64(rint(gy));
    if (cy < 0) cy = 0;
    else if (cy > height - 1) cy = height - 1;
    double best = INFINITY;
    for (long long yy = cy - 1 > 0 ? cy - 1 : 0; yy < (cy + 2 < height ? cy + 2 : height); yy++)
        for (long long xx = cx - 1 > 0 ? cx - 1 : 0; xx < (cx + 2 < width ? cx + 2 : width); xx++) {
            const double t = depth[yy * width + xx];
            if (isfinite(t)) {
                const double diff = fabs(t - d);
                if (diff < best) best = diff;
            }
        }
    return best <= eps ? 1 : 0;
}

}  // extern "C"

// Parallel host memcpy for gm_plan_read's staged read-back (1 MiB pieces over
// the plan's host threads; internal to the library, not part of the ABI).
extern "C" __attribute__((visibility("hidden"))) void gm_host_copy(void* dst, const void* src, size_t bytes,
                                                                   int threads) {
    const size_t grain = (size_t)1 << 20;
    const int64_t n = (int64_t)((bytes + grain - 1) / grain);
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        const size_t o = (size_t)i * grain;
        memcpy((char*)dst + o, (const char*)src + o, bytes - o < grain ? bytes - o : grain);
    }
}

