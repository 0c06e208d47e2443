// gm_setup.cpp -- per-fixation setup table, computed on the host.
//
// Restates, bit for bit, what the reference computes in Python/numpy before
// each kernels.rasterize / kernels.accumulate call:
//   Fixation.view_matrix           gaze.py:114-122  (quat_to_matrix geometry.py:48-57)
//   GazeCone.from_theta            gaze.py:64-67
//   build_crop_frustum             gaze.py:372-381 -> ellipse_intersection :252-309,
//                                  crop_bounds :312-320, perspective_matrix :323-336
//   fallback projection_matrix     gaze.py:124-127 (density.py:152-158)
//   frustum_from_matrix near/far   gaze.py:345-356 (raster.py:113)
//   amp                            density.py:179
//
// Why the host: the crop frustum needs glibc acos/cos/sin (what CPython's math
// module calls) to be bit-identical; CUDA's libdevice differs by an ulp now
// and then and that would move crop-box edges.  It is ~0.3 us per fixation,
// OpenMP-parallel and overlapped with the GPU batch in flight.
//
// Build flags (see build.py): -ffp-contract=off (numpy/Python never fuse),
// -fno-builtin (CPython `x ** 2` is libm pow(x, 2.0), which gcc would otherwise
// fold to x*x -- not always the same bits).  numpy BLAS call sites (1-D norm,
// matrix @ vector) are OpenBLAS FMA chains and are written with std::fma.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "gm_types.h"

namespace {

struct V3 {
    double x, y, z;
};

// OpenBLAS ddot / dgemv inner product over k = 0..2: acc = fma(a_k, b_k, acc).
inline double blas_dot(double a0, double b0, double a1, double b1, double a2, double b2) {
    double acc = a0 * b0;
    acc = std::fma(a1, b1, acc);
    acc = std::fma(a2, b2, acc);
    return acc;
}

inline double np_norm(const V3& v) { return std::sqrt(blas_dot(v.x, v.x, v.y, v.y, v.z, v.z)); }

inline V3 np_cross(const V3& a, const V3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

inline V3 scaled(const V3& v, double s) { return {v.x * s, v.y * s, v.z * s}; }
inline V3 divided(const V3& v, double s) { return {v.x / s, v.y / s, v.z / s}; }

// gaze.py:232-239 _quat_rotate with precomputed cos/sin of the half angle.
inline V3 quat_rotate(const V3& v, const V3& axis, double c_half, double s_half) {
    V3 u = scaled(axis, s_half);
    V3 uv = np_cross(u, v);
    V3 uuv = np_cross(u, uv);
    double tw = 2.0 * c_half;
    return {(v.x + tw * uv.x) + 2.0 * uuv.x, (v.y + tw * uv.y) + 2.0 * uuv.y, (v.z + tw * uv.z) + 2.0 * uuv.z};
}

// gaze.py:242-249; false == GazeOutsideFrustumError
inline bool near_hit(const V3& d, double n, V3* out) {
    if (d.z >= 0.0) return false;
    double t = -n / d.z;
    *out = {t * d.x, t * d.y, -n};
    return true;
}

// gaze.py:252-309 ellipse_intersection: 0, or the GazeOutsideFrustumError
// raised (1: a rotated ray misses the near plane, gaze.py:244-247; 2: no
// ellipse, :285-286).  out (EllipseParams): center_E[3], major_a, minor_b,
// inclination_alpha, A0[3], A1[3], B0[3], B1[3].
int ellipse(const double* gaze, double n, const GmSetupConsts& c, double out[18]) {
    V3 g{gaze[0], gaze[1], gaze[2]};
    V3 r = divided(g, np_norm(g));
    V3 u1 = np_cross(r, V3{0.0, 0.0, -1.0});
    if (np_norm(u1) < 1e-12) u1 = V3{1.0, 0.0, 0.0};
    u1 = divided(u1, np_norm(u1));
    V3 u2 = np_cross(r, u1);
    u2 = divided(u2, np_norm(u2));
    V3 a0 = quat_rotate(r, u1, c.cos_hm, c.sin_hm);
    V3 a1 = quat_rotate(r, u1, c.cos_hp, c.sin_hp);
    V3 b0 = quat_rotate(r, u2, c.cos_hm, c.sin_hm);
    V3 b1 = quat_rotate(r, u2, c.cos_hp, c.sin_hp);
    V3 E, A0, A1, B0, B1;
    if (!near_hit(r, n, &E) || !near_hit(a0, n, &A0) || !near_hit(a1, n, &A1) || !near_hit(b0, n, &B0) ||
        !near_hit(b1, n, &B1))
        return 1;
    V3 dA{A1.x - A0.x, A1.y - A0.y, A1.z - A0.z};
    double a = 0.5 * np_norm(dA);
    double cos_beta = -r.z;
    double disc = std::pow(c.cos_phi, 2.0) - (1.0 - cos_beta * cos_beta);
    if (disc <= 0.0) return 2;
    double b = n * c.sin_phi / std::sqrt(disc);
    V3 me{E.x - 0.0, E.y - 0.0, E.z - (-n)};
    double me_norm = np_norm(me);
    double alpha = 0.0;
    if (!(me_norm < 1e-15)) {
        V3 u = divided(me, me_norm);
        double x = blas_dot(1.0, u.x, 0.0, u.y, 0.0, u.z);  // _CAMERA_RIGHT @ unit(me)
        x = std::fmax(-1.0, std::fmin(1.0, x));
        alpha = std::acos(x);
    }
    out[0] = 0.5 * (A0.x + A1.x);
    out[1] = 0.5 * (A0.y + A1.y);
    out[2] = 0.5 * (A0.z + A1.z);
    out[3] = a > b ? a : b;  // max(a, b)
    out[4] = a < b ? a : b;  // min(a, b)
    out[5] = alpha;
    const V3 pts[4] = {A0, A1, B0, B1};
    for (int k = 0; k < 4; k++) {
        out[6 + 3 * k] = pts[k].x;
        out[7 + 3 * k] = pts[k].y;
        out[8 + 3 * k] = pts[k].z;
    }
    return 0;
}

// gaze.py:312-320 crop_bounds: (l', r', b', t') of an EllipseParams
void bounds(const double e[18], double lrbt[4]) {
    double a2 = std::pow(e[3], 2.0), b2 = std::pow(e[4], 2.0);
    double ca2 = std::pow(std::cos(e[5]), 2.0), sa2 = std::pow(std::sin(e[5]), 2.0);
    double dx = std::sqrt(a2 * ca2 + b2 * sa2);
    double dy = std::sqrt(a2 * sa2 + b2 * ca2);
    lrbt[0] = e[0] - dx;
    lrbt[1] = e[0] + dx;
    lrbt[2] = e[1] - dy;
    lrbt[3] = e[1] + dy;
}

// gaze.py:372-381 without the projection; false == GazeOutsideFrustumError
bool crop_box(const double* gaze, double n, const GmSetupConsts& c, double lrbt[4]) {
    double e[18];
    if (ellipse(gaze, n, c, e)) return false;
    bounds(e, lrbt);
    return true;
}

struct Proj {
    double p00, p11, p02, p12, m22, m23;
};

// gaze.py:323-336; false == InvalidFrustumError
bool perspective(double l, double r, double b, double t, double n, double f, Proj* P) {
    if (!(l < r && b < t)) return false;
    if (!(0 < n && n < f)) return false;
    P->p00 = 2.0 * n / (r - l);
    P->p02 = (r + l) / (r - l);
    P->p11 = 2.0 * n / (t - b);
    P->p12 = (t + b) / (t - b);
    P->m22 = -(f + n) / (f - n);
    P->m23 = -2.0 * f * n / (f - n);
    return true;
}

}  // namespace

extern "C" void gm_setup_consts(double theta, int filtering, int width, int height, GmSetupConsts* c) {
    c->theta = theta;
    c->sigma = std::tan(theta);
    c->phi = std::atan(4.0 * c->sigma);
    double hp = 0.5 * c->phi, hm = 0.5 * -c->phi;
    c->cos_hp = std::cos(hp);
    c->sin_hp = std::sin(hp);
    c->cos_hm = std::cos(hm);
    c->sin_hm = std::sin(hm);
    c->cos_phi = std::cos(c->phi);
    c->sin_phi = std::sin(c->phi);
    c->sqrt_two_pi = std::sqrt(2.0 * M_PI);
    c->filtering = filtering;
    c->width = width;
    c->height = height;
}

// Setup of fixations [0, F) of `fx` (F x 18, log schema gaze.py:133-136, gaze
// already normalised by Fixation.__post_init__).  Returns -1 on success or the
// index of the first fixation whose (crop or full) frustum is invalid.
extern "C" int64_t gm_setup_batch(const double* fx, int64_t F, const GmSetupConsts* cp, GmFixExact* ex,
                                  GmFixCull* cull, int threads) {
    const GmSetupConsts c = *cp;
    int64_t bad = INT64_MAX;
#pragma omp parallel for schedule(static) num_threads(threads) reduction(min : bad) if (threads > 1)
    for (int64_t i = 0; i < F; i++) {
        const double* row = fx + GM_FIX_STRIDE * i;
        const double *pos = row + 2, *q = row + 5, *fr = row + 9, *g = row + 15;
        // quat_to_matrix (geometry.py:48-57)
        double x = q[0], y = q[1], z = q[2], w = q[3];
        double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - z * w), 2.0 * (x * z + y * w),
                       2.0 * (x * y + z * w), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - x * w),
                       2.0 * (x * z - y * w), 2.0 * (y * z + x * w), 1.0 - 2.0 * (x * x + y * y)};
        GmFixExact e;
        std::memset(&e, 0, sizeof(e));
        for (int a = 0; a < 3; a++) {
            for (int b = 0; b < 3; b++) e.rot[3 * a + b] = R[3 * b + a];
            e.trans[a] = blas_dot(-R[a], pos[0], -R[3 + a], pos[1], -R[6 + a], pos[2]);
            e.gaze[a] = g[a];
        }
        e.amp = row[1] / (c.sigma * c.sqrt_two_pi);
        Proj P;
        bool ok = false, cropped = false;
        if (c.filtering) {
            double lrbt[4];
            if (crop_box(g, fr[4], c, lrbt)) {
                if (!perspective(lrbt[0], lrbt[1], lrbt[2], lrbt[3], fr[4], fr[5], &P)) {
                    bad = bad < i ? bad : i;
                    continue;
                }
                ok = cropped = true;
            }
        }
        if (!ok && !perspective(fr[0], fr[1], fr[3], fr[2], fr[4], fr[5], &P)) {
            bad = bad < i ? bad : i;
            continue;
        }
        e.p00 = P.p00;
        e.p11 = P.p11;
        e.p02 = P.p02;
        e.p12 = P.p12;
        e.near_ = P.m23 / (P.m22 - 1.0);
        e.far_ = P.m23 / (P.m22 + 1.0);
        e.near_lo = e.near_ * (1.0 - GM_NDC_SLACK);
        e.far_hi = e.far_ * (1.0 + GM_NDC_SLACK);
        e.cropped = cropped ? 1.0 : 0.0;
        ex[i] = e;

        // ---- conservative float32 cull record (never decides a result) ----
        GmFixCull k;
        std::memset(&k, 0, sizeof(k));
        // world gaze = R * g (camera-to-world), world forward = -R[:,2]
        double gw[3], fw[3];
        for (int a = 0; a < 3; a++) {
            gw[a] = R[3 * a] * g[0] + R[3 * a + 1] * g[1] + R[3 * a + 2] * g[2];
            fw[a] = -R[3 * a + 2];
        }
        double gn = std::sqrt(gw[0] * gw[0] + gw[1] * gw[1] + gw[2] * gw[2]);
        double fn = std::sqrt(fw[0] * fw[0] + fw[1] * fw[1] + fw[2] * fw[2]);
        double omax = std::fmax(std::fabs(pos[0]), std::fmax(std::fabs(pos[1]), std::fabs(pos[2])));
        k.ox = (float)pos[0];
        k.oy = (float)pos[1];
        k.oz = (float)pos[2];
        k.margin = (float)(1e-5 * (1.0 + omax));
        k.gx = (float)(gw[0] / gn);
        k.gy = (float)(gw[1] / gn);
        k.gz = (float)(gw[2] / gn);
        k.fx = (float)(fw[0] / fn);
        k.fy = (float)(fw[1] / fn);
        k.fz = (float)(fw[2] / fn);
        // sample cone: a contributing sample has ratio^2 <= 16 <=> angle <= phi
        double phi_s = c.phi * (1.0 + 1e-5) + 1e-6;
        // occluder cone: a texel read by depth_match lies within 2 px (per axis)
        // of an in-cone sample; tangent-plane distance bounds the angle.
        double pix = std::fmax(2.0 / (c.width * std::fabs(P.p00)), 2.0 / (c.height * std::fabs(P.p11)));
        double phi_t = c.phi + 3.5 * pix + 1e-5;
        if (phi_s < 1.5) {
            k.cos_s = (float)std::cos(phi_s);
            k.sin_s = (float)std::sin(phi_s);
        } else {
            k.cos_s = -2.0f;
            k.sin_s = 0.0f;
        }
        if (phi_t < 1.5) {
            k.cos_t = (float)std::cos(phi_t);
            k.sin_t = (float)std::sin(phi_t);
        } else {
            k.cos_t = -2.0f;
            k.sin_t = 0.0f;
        }
        k.near_f = (float)(e.near_ * (1.0 - 1e-6));
        k.far_f = (float)(e.far_ * (1.0 + 1e-6));
        cull[i] = k;
    }
    return bad == INT64_MAX ? -1 : bad;
}

// ---- the crop-frustum steps as C-ABI entry points (Python API: gaze.py) ----

static void phi_consts(double phi, GmSetupConsts* c) {
    std::memset(c, 0, sizeof(*c));
    c->phi = phi;
    double hp = 0.5 * phi, hm = 0.5 * -phi;
    c->cos_hp = std::cos(hp);
    c->sin_hp = std::sin(hp);
    c->cos_hm = std::cos(hm);
    c->sin_hm = std::sin(hm);
    c->cos_phi = std::cos(phi);
    c->sin_phi = std::sin(phi);
}

// ellipse_intersection(gaze_dir, n, cone) (gaze.py:252-309) for a cone of
// 4-sigma half-angle phi: out[18] as in ellipse(); GM_ERR_GAZE_OUTSIDE with
// out[0] = 1 or 2 (which GazeOutsideFrustumError) when there is no ellipse.
extern "C" int gm_ellipse_intersection(const double* gaze, double n, double phi, double* out) {
    if (!gaze || !out) return GM_ERR_ARG;
    GmSetupConsts c;
    phi_consts(phi, &c);
    const int why = ellipse(gaze, n, c, out);
    if (why) {
        out[0] = (double)why;
        return GM_ERR_GAZE_OUTSIDE;
    }
    return GM_OK;
}

// crop_bounds(e) (gaze.py:312-320) of an 18-double EllipseParams.
extern "C" int gm_crop_bounds(const double* e, double* lrbt) {
    if (!e || !lrbt) return GM_ERR_ARG;
    bounds(e, lrbt);
    return GM_OK;
}
