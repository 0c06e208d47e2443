/*
 * gm_oracle.c -- CPU restatement of the reference `gazemap` generation path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2601_07571_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The
 * product never links or calls it.
 *
 * Every function restates one reference function, in the reference's
 * floating-point operation order, compiled with -ffp-contract=off so no
 * multiply-add is fused unless the reference itself fuses it:
 *   - numba kernels (pkg/src/gazemap/kernels.py) contain no FMA;
 *   - numpy BLAS call sites (`@`, 1-D np.linalg.norm) are OpenBLAS kernels whose
 *     k-loop is an FMA chain acc = fma(a_k, b_k, acc) from acc = 0 (SURVEY.md
 *     section 0 fact 2).  Those sites use bl_dot3 / bl_dot4 below.
 * Trigonometry goes through glibc libm exactly like CPython's math module.
 * Parity is pinned against the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py importing /root/reference) -- see
 * tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_NDC_SLACK 1e-9 /* kernels.py:21 */

/* ---------------------------------------------------------------- helpers */

/* OpenBLAS ddot / dgemm / dgemv inner product of length 3 (FMA chain). */
static double bl_dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
    double acc = a0 * b0;
    acc = fma(a1, b1, acc);
    acc = fma(a2, b2, acc);
    return acc;
}

static double bl_dot4(const double *a, const double *b, int bstride) {
    double acc = a[0] * b[0];
    acc = fma(a[1], b[bstride], acc);
    acc = fma(a[2], b[2 * bstride], acc);
    acc = fma(a[3], b[3 * bstride], acc);
    return acc;
}

/* np.linalg.norm of a 3-vector: sqrt(x.dot(x)) (numpy linalg norm, ord=None). */
static double np_norm3(const double v[3]) {
    return sqrt(bl_dot3(v[0], v[0], v[1], v[1], v[2], v[2]));
}

/* np.cross of 3-vectors: cp0 = a1*b2 - a2*b1, ... (numpy _core/numeric.py cross). */
static void np_cross(const double a[3], const double b[3], double out[3]) {
    double c0 = a[1] * b[2] - a[2] * b[1];
    double c1 = a[2] * b[0] - a[0] * b[2];
    double c2 = a[0] * b[1] - a[1] * b[0];
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
}

/* geometry.py:48-57 quat_to_matrix, (x, y, z, w) */
void or_quat_to_matrix(const double q[4], double R[9]) {
    double x = q[0], y = q[1], z = q[2], w = q[3];
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - z * w);
    R[2] = 2.0 * (x * z + y * w);
    R[3] = 2.0 * (x * y + z * w);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - x * w);
    R[6] = 2.0 * (x * z - y * w);
    R[7] = 2.0 * (y * z + x * w);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* ------------------------------------------------------- stage 1: sampling */

/* geometry.py:169-176 triangle_areas + :202-210 adaptive_resolutions +
 * :305-320 build_sampled_mesh.  tri is (T,3,3) local vertices. */
void or_layout(const double *tri, int64_t T, double k, int64_t *res, int64_t *cnt, int64_t *off,
               int64_t *total) {
    double k8 = 8.0 * k;
    int64_t run = 0;
    for (int64_t t = 0; t < T; t++) {
        const double *v = tri + 9 * t;
        double e[3][3];
        for (int c = 0; c < 3; c++) {
            e[0][c] = v[3 + c] - v[0 + c]; /* tri[:,1]-tri[:,0] */
            e[1][c] = v[6 + c] - v[3 + c]; /* tri[:,2]-tri[:,1] */
            e[2][c] = v[6 + c] - v[0 + c]; /* tri[:,2]-tri[:,0] */
        }
        double len[3];
        for (int i = 0; i < 3; i++) /* norm(axis=1): sqrt(add.reduce(x*x, axis=1)) */
            len[i] = sqrt((e[i][0] * e[i][0] + e[i][1] * e[i][1]) + e[i][2] * e[i][2]);
        double a = len[0], b = len[1], c = len[2];
        double s = 0.5 * (a + b + c);
        double rad = s * (s - a) * (s - b) * (s - c);
        double area = sqrt(rad > 0.0 ? rad : 0.0);
        double delta = 1.0 + k8 * area;
        int64_t r = (int64_t)ceil((-3.0 + sqrt(delta)) / 2.0);
        if (delta < 25.0) r = 1;
        if (r < 1) r = 1;
        res[t] = r;
        cnt[t] = (r + 1) * (r + 2) / 2;
        off[t] = run;
        run += cnt[t];
    }
    *total = run;
}

/* geometry.py:232-242 sample_rowcol (vectorized form: one fix-up each way). */
static void rowcol(int64_t idx, int64_t *prow, int64_t *pcol) {
    int64_t row = (int64_t)ceil((-3.0 + sqrt(8.0 * (double)idx + 9.0)) / 2.0);
    int64_t col = idx - row * (row + 1) / 2;
    if (col < 0) row -= 1;
    col = idx - row * (row + 1) / 2;
    if (col > row) row += 1;
    col = idx - row * (row + 1) / 2;
    *prow = row;
    *pcol = col;
}

/* geometry.py:331-346 sample_positions_local. out is (N,3). */
void or_positions_local(const double *tri, int64_t T, const int64_t *res, const int64_t *cnt,
                        const int64_t *off, double *out) {
    for (int64_t t = 0; t < T; t++) {
        const double *v = tri + 9 * t;
        double r = (double)res[t];
        for (int64_t within = 0; within < cnt[t]; within++) {
            int64_t row, col;
            rowcol(within, &row, &col);
            double w1 = (double)col / r;
            double w2 = (double)(row - col) / r;
            double w3 = 1.0 - (double)row / r;
            double *o = out + 3 * (off[t] + within);
            for (int c = 0; c < 3; c++) o[c] = w1 * v[c] + w2 * v[3 + c] + w3 * v[6 + c];
        }
    }
}

/* geometry.py:82-89 Transform.matrix / apply: pts @ (R*diag(s)).T + t (dgemm). */
void or_transform_apply(const double *pts, int64_t n, const double q[4], const double s[3],
                        const double t[3], double *out) {
    double R[9], M[9];
    or_quat_to_matrix(q, R);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[3 * i + j] = R[3 * i + j] * s[j];
    for (int64_t p = 0; p < n; p++) {
        const double *x = pts + 3 * p;
        double *o = out + 3 * p;
        for (int i = 0; i < 3; i++)
            o[i] = bl_dot3(x[0], M[3 * i + 0], x[1], M[3 * i + 1], x[2], M[3 * i + 2]) + t[i];
    }
}

/* -------------------------------------------- per-fixation setup (gaze.py) */

/* Output record of or_fixation_setup (all float64). */
enum {
    FS_ROT = 0,     /* 9: view rotation = R^T (gaze.py:120) */
    FS_TRANS = 9,   /* 3: -R^T @ pos (gaze.py:121, dgemv) */
    FS_GAZE = 12,   /* 3: fixation.gaze_dir */
    FS_AMP = 15,    /* duration / (sigma * sqrt(2 pi)) (density.py:179) */
    FS_P00 = 16,
    FS_P11 = 17,
    FS_P02 = 18,
    FS_P12 = 19,
    FS_NEAR = 20,   /* frustum_from_matrix near' (gaze.py:348) */
    FS_FAR = 21,    /* frustum_from_matrix far' (gaze.py:349) */
    FS_CROPPED = 22, /* 1.0 if the crop frustum was used */
    FS_PROJ = 23,   /* 16: projection matrix row-major */
    FS_VIEW = 39,   /* 16: view matrix row-major */
    FS_LEN = 55
};

#define OR_OK 0
#define OR_ERR_INVALID_FRUSTUM 3

/* gaze.py:323-336 perspective_matrix */
static int perspective(double l, double r, double b, double t, double n, double f, double P[16]) {
    if (!(l < r && b < t)) return OR_ERR_INVALID_FRUSTUM;
    if (!(0 < n && n < f)) return OR_ERR_INVALID_FRUSTUM;
    memset(P, 0, 16 * sizeof(double));
    P[0] = 2.0 * n / (r - l);
    P[2] = (r + l) / (r - l);
    P[5] = 2.0 * n / (t - b);
    P[6] = (t + b) / (t - b);
    P[10] = -(f + n) / (f - n);
    P[11] = -2.0 * f * n / (f - n);
    P[14] = -1.0;
    return OR_OK;
}

/* gaze.py:232-239 _quat_rotate */
static void quat_rotate(const double v[3], const double axis[3], double angle, double out[3]) {
    double half = 0.5 * angle;
    double w = cos(half);
    double sh = sin(half);
    double u[3] = {axis[0] * sh, axis[1] * sh, axis[2] * sh};
    double uv[3], uuv[3];
    np_cross(u, v, uv);
    np_cross(u, uv, uuv);
    double tw = 2.0 * w;
    for (int c = 0; c < 3; c++) out[c] = (v[c] + tw * uv[c]) + 2.0 * uuv[c];
}

/* gaze.py:242-249 _near_plane_hit; returns 0 on GazeOutsideFrustumError */
static int near_hit(const double d[3], double n, double out[3]) {
    if (d[2] >= 0.0) return 0;
    double t = -n / d[2];
    out[0] = t * d[0];
    out[1] = t * d[1];
    out[2] = -n;
    return 1;
}

/* gaze.py:252-309 ellipse_intersection + :312-320 crop_bounds.
 * Returns 0 on GazeOutsideFrustumError. */
static int crop_box(const double gaze[3], double n, double phi, double out_lrbt[4]) {
    double nr = np_norm3(gaze);
    double r[3] = {gaze[0] / nr, gaze[1] / nr, gaze[2] / nr};
    const double fwd[3] = {0.0, 0.0, -1.0};
    double u1[3], u2[3];
    np_cross(r, fwd, u1);
    if (np_norm3(u1) < 1e-12) {
        u1[0] = 1.0;
        u1[1] = 0.0;
        u1[2] = 0.0;
    }
    double n1 = np_norm3(u1);
    for (int c = 0; c < 3; c++) u1[c] = u1[c] / n1;
    np_cross(r, u1, u2);
    double n2 = np_norm3(u2);
    for (int c = 0; c < 3; c++) u2[c] = u2[c] / n2;
    double a0[3], a1[3], b0[3], b1[3];
    quat_rotate(r, u1, -phi, a0);
    quat_rotate(r, u1, phi, a1);
    quat_rotate(r, u2, -phi, b0);
    quat_rotate(r, u2, phi, b1);
    double E[3], A0[3], A1[3], B0[3], B1[3];
    if (!near_hit(r, n, E)) return 0;
    if (!near_hit(a0, n, A0)) return 0;
    if (!near_hit(a1, n, A1)) return 0;
    if (!near_hit(b0, n, B0)) return 0;
    if (!near_hit(b1, n, B1)) return 0;
    double dA[3] = {A1[0] - A0[0], A1[1] - A0[1], A1[2] - A0[2]};
    double a = 0.5 * np_norm3(dA);
    double cos_beta = -r[2];
    double cphi = cos(phi);
    double disc = pow(cphi, 2.0) - (1.0 - cos_beta * cos_beta); /* `** 2` is libm pow */
    if (disc <= 0.0) return 0;
    double b = n * sin(phi) / sqrt(disc);
    double center[3] = {0.5 * (A0[0] + A1[0]), 0.5 * (A0[1] + A1[1]), 0.5 * (A0[2] + A1[2])};
    double me[3] = {E[0] - 0.0, E[1] - 0.0, E[2] - (-n)};
    double me_norm = np_norm3(me);
    double alpha;
    if (me_norm < 1e-15) {
        alpha = 0.0;
    } else {
        double u[3] = {me[0] / me_norm, me[1] / me_norm, me[2] / me_norm};
        double x = bl_dot3(1.0, u[0], 0.0, u[1], 0.0, u[2]);
        if (x > 1.0) x = 1.0;   /* min(1.0, x) */
        if (x < -1.0) x = -1.0; /* max(-1.0, .) */
        alpha = acos(x);
    }
    double major = a > b ? a : b; /* max(a, b) */
    double minor = a < b ? a : b; /* min(a, b) */
    /* crop_bounds */
    double a2 = pow(major, 2.0), b2 = pow(minor, 2.0); /* CPython float ** -> libm pow */
    double ca = cos(alpha), sa = sin(alpha);
    double ca2 = pow(ca, 2.0), sa2 = pow(sa, 2.0);
    double dx = sqrt(a2 * ca2 + b2 * sa2);
    double dy = sqrt(a2 * sa2 + b2 * ca2);
    double ex = center[0], ey = center[1];
    out_lrbt[0] = ex - dx;
    out_lrbt[1] = ex + dx;
    out_lrbt[2] = ey - dy;
    out_lrbt[3] = ey + dy;
    return 1;
}

/* fx layout (18 float64, the fixation-log schema gaze.py:133-136):
 *   start, duration, pos[3], quat[4] (xyzw), frustum l r t b n f, gaze[3]
 * gaze must already be normalized once (Fixation.__post_init__, gaze.py:91-95).
 * Restates density.py:148-158 + gaze.py:114-127 + :345-356. */
int or_fixation_setup(const double *fx, double theta, int filtering, double *out) {
    double sigma = tan(theta);           /* GazeCone.from_theta */
    double phi = atan(4.0 * sigma);
    const double *pos = fx + 2, *q = fx + 5, *fr = fx + 9, *g = fx + 15;
    double R[9];
    or_quat_to_matrix(q, R);
    double *V = out + FS_VIEW;
    memset(V, 0, 16 * sizeof(double));
    for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) {
            out[FS_ROT + 3 * i + j] = R[3 * j + i];
            V[4 * i + j] = R[3 * j + i];
        }
        /* (-rot.T) @ pos */
        double tr = bl_dot3(-R[0 + i], pos[0], -R[3 + i], pos[1], -R[6 + i], pos[2]);
        out[FS_TRANS + i] = tr;
        V[4 * i + 3] = tr;
    }
    V[15] = 1.0;
    for (int c = 0; c < 3; c++) out[FS_GAZE + c] = g[c];
    out[FS_AMP] = fx[1] / (sigma * sqrt(2.0 * M_PI));
    double *P = out + FS_PROJ;
    int cropped = 0;
    if (filtering) {
        double lrbt[4];
        if (crop_box(g, fr[4], phi, lrbt)) {
            int rc = perspective(lrbt[0], lrbt[1], lrbt[2], lrbt[3], fr[4], fr[5], P);
            if (rc) return rc; /* InvalidFrustumError propagates (not caught) */
            cropped = 1;
        }
    }
    if (!cropped) {
        int rc = perspective(fr[0], fr[1], fr[3], fr[2], fr[4], fr[5], P);
        if (rc) return rc;
    }
    out[FS_P00] = P[0];
    out[FS_P11] = P[5];
    out[FS_P02] = P[2];
    out[FS_P12] = P[6];
    out[FS_NEAR] = P[11] / (P[10] - 1.0);
    out[FS_FAR] = P[11] / (P[10] + 1.0);
    out[FS_CROPPED] = cropped ? 1.0 : 0.0;
    return OR_OK;
}

/* ------------------------------------------------------- cull (raster.py) */

/* raster.py:54-65 frustum_planes(proj @ view); the 4x4 product is a dgemm. */
void or_frustum_planes(const double *P, const double *V, double planes[24]) {
    double m[16];
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) m[4 * i + j] = bl_dot4(P + 4 * i, V + j, 4);
    for (int c = 0; c < 4; c++) {
        planes[0 + c] = m[12 + c] + m[0 + c];
        planes[4 + c] = m[12 + c] - m[0 + c];
        planes[8 + c] = m[12 + c] + m[4 + c];
        planes[12 + c] = m[12 + c] - m[4 + c];
        planes[16 + c] = m[12 + c] + m[8 + c];
        planes[20 + c] = m[12 + c] - m[8 + c];
    }
}

/* kernels.py:195-216 cull_mask */
void or_cull_mask(const double *tris, int64_t T, const double planes[24], uint8_t *keep) {
    for (int64_t t = 0; t < T; t++) {
        const double *v = tris + 9 * t;
        keep[t] = 1;
        for (int p = 0; p < 6; p++) {
            double a = planes[4 * p], b = planes[4 * p + 1], c = planes[4 * p + 2], d = planes[4 * p + 3];
            int outside = 1;
            for (int k = 0; k < 3; k++) {
                if (a * v[3 * k] + b * v[3 * k + 1] + c * v[3 * k + 2] + d >= 0.0) {
                    outside = 0;
                    break;
                }
            }
            if (outside) {
                keep[t] = 0;
                break;
            }
        }
    }
}

/* ---------------------------------------------------- raster (kernels.py) */

/* kernels.py:35-59 _clip_near (xyz only; attributes are unused for depth) */
static int clip_near(double vin[3][3], double near, double vout[4][3]) {
    int nv = 0;
    for (int i = 0; i < 3; i++) {
        int j = (i + 1) % 3;
        double cz = vin[i][2], nz = vin[j][2];
        int cin = cz <= -near;
        int nin = nz <= -near;
        if (cin) {
            for (int c = 0; c < 3; c++) vout[nv][c] = vin[i][c];
            nv++;
        }
        if (cin != nin) {
            double t = (-near - cz) / (nz - cz);
            for (int c = 0; c < 3; c++) vout[nv][c] = vin[i][c] + t * (vin[j][c] - vin[i][c]);
            nv++;
        }
    }
    return nv;
}

/* kernels.py:62-64 _edge */
static inline double edge(double ax, double ay, double bx, double by, double px, double py) {
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

/* kernels.py:67-137 _raster_tri (depth only) */
static void raster_tri(double sx[3], double sy[3], double iw[3], int width, int height, double near,
                       double far, double *depth) {
    double area = edge(sx[0], sy[0], sx[1], sy[1], sx[2], sy[2]);
    if (area == 0.0) return;
    if (area < 0.0) {
        double tmp;
        tmp = sx[1]; sx[1] = sx[2]; sx[2] = tmp;
        tmp = sy[1]; sy[1] = sy[2]; sy[2] = tmp;
        tmp = iw[1]; iw[1] = iw[2]; iw[2] = tmp;
        area = -area;
    }
    double minx = fmin(sx[0], fmin(sx[1], sx[2]));
    double maxx = fmax(sx[0], fmax(sx[1], sx[2]));
    double miny = fmin(sy[0], fmin(sy[1], sy[2]));
    double maxy = fmax(sy[0], fmax(sy[1], sy[2]));
    int64_t x0 = (int64_t)ceil(minx - 0.5);
    if (x0 < 0) x0 = 0;
    int64_t x1 = (int64_t)floor(maxx - 0.5);
    if (x1 > width - 1) x1 = width - 1;
    int64_t y0 = (int64_t)ceil(miny - 0.5);
    if (y0 < 0) y0 = 0;
    int64_t y1 = (int64_t)floor(maxy - 0.5);
    if (y1 > height - 1) y1 = height - 1;
    if (x1 < x0 || y1 < y0) return;
    double inv_area = 1.0 / area;
    for (int64_t py = y0; py <= y1; py++) {
        double cy = (double)py + 0.5;
        for (int64_t px = x0; px <= x1; px++) {
            double cx = (double)px + 0.5;
            double w0 = edge(sx[1], sy[1], sx[2], sy[2], cx, cy);
            double w1 = edge(sx[2], sy[2], sx[0], sy[0], cx, cy);
            double w2 = edge(sx[0], sy[0], sx[1], sy[1], cx, cy);
            if (w0 < 0.0 || w1 < 0.0 || w2 < 0.0) continue;
            if (w0 == 0.0 && !(sy[2] - sy[1] < 0.0 || (sy[2] == sy[1] && sx[2] - sx[1] > 0.0))) continue;
            if (w1 == 0.0 && !(sy[0] - sy[2] < 0.0 || (sy[0] == sy[2] && sx[0] - sx[2] > 0.0))) continue;
            if (w2 == 0.0 && !(sy[1] - sy[0] < 0.0 || (sy[1] == sy[0] && sx[1] - sx[0] > 0.0))) continue;
            double l0 = w0 * inv_area, l1 = w1 * inv_area, l2 = w2 * inv_area;
            double inv_w = l0 * iw[0] + l1 * iw[1] + l2 * iw[2];
            if (inv_w <= 0.0) continue;
            double d = 1.0 / inv_w;
            if (d < near || d > far) continue;
            double *dst = depth + py * (int64_t)width + px;
            if (d < *dst) *dst = d;
        }
    }
}

/* kernels.py:140-192 rasterize (depth only).  depth must be pre-filled (+inf). */
void or_rasterize(const double *tris, int64_t T, const double rot[9], const double trans[3], double p00,
                  double p11, double p02, double p12, int width, int height, double near, double far,
                  double *depth) {
    double half_w = 0.5 * width, half_h = 0.5 * height;
    for (int64_t t = 0; t < T; t++) {
        double vin[3][3], vout[4][3];
        for (int v = 0; v < 3; v++) {
            double wx = tris[9 * t + 3 * v], wy = tris[9 * t + 3 * v + 1], wz = tris[9 * t + 3 * v + 2];
            for (int i = 0; i < 3; i++)
                vin[v][i] = rot[3 * i] * wx + rot[3 * i + 1] * wy + rot[3 * i + 2] * wz + trans[i];
        }
        int nv = clip_near(vin, near, vout);
        if (nv < 3) continue;
        for (int k = 0; k < nv - 2; k++) {
            double sx[3], sy[3], iw[3];
            int ok = 1;
            for (int m = 0; m < 3; m++) {
                int src = m == 0 ? 0 : k + m;
                double x = vout[src][0], y = vout[src][1], z = vout[src][2];
                double w = -z;
                if (w <= 0.0) {
                    ok = 0;
                    break;
                }
                double ndc_x = (p00 * x + p02 * z) / w;
                double ndc_y = (p11 * y + p12 * z) / w;
                sx[m] = (ndc_x + 1.0) * half_w;
                sy[m] = (1.0 - ndc_y) * half_h;
                iw[m] = 1.0 / w;
            }
            if (ok) raster_tri(sx, sy, iw, width, height, near, far, depth);
        }
    }
}

/* kernels.py:219-285 depth_match */
int or_depth_match(const double *depth, int height, int width, double fx, double fy, double d, double eps) {
    double gx = fx - 0.5, gy = fy - 0.5;
    if (width > 1 && height > 1) {
        int64_t x0 = (int64_t)floor(gx);
        if (x0 < 0) x0 = 0;
        else if (x0 > width - 2) x0 = width - 2;
        int64_t y0 = (int64_t)floor(gy);
        if (y0 < 0) y0 = 0;
        else if (y0 > height - 2) y0 = height - 2;
        double q00 = depth[y0 * width + x0], q01 = depth[y0 * width + x0 + 1];
        double q10 = depth[(y0 + 1) * width + x0], q11 = depth[(y0 + 1) * width + x0 + 1];
        if (isfinite(q00) && isfinite(q01) && isfinite(q10) && isfinite(q11)) {
            double tx = gx - (double)x0;
            if (tx < 0.0) tx = 0.0;
            else if (tx > 1.0) tx = 1.0;
            double ty = gy - (double)y0;
            if (ty < 0.0) ty = 0.0;
            else if (ty > 1.0) ty = 1.0;
            double top = q00 * (1.0 - tx) + q01 * tx;
            double bot = q10 * (1.0 - tx) + q11 * tx;
            if (fabs(d - (top * (1.0 - ty) + bot * ty)) <= eps) return 1;
            double hi = fmax(fmax(q00, q01), fmax(q10, q11));
            double lo = fmin(fmin(q00, q01), fmin(q10, q11));
            if (hi - lo <= eps) return 0;
        }
    }
    int64_t cx = (int64_t)nearbyint(gx); /* np.round: half-to-even */
    if (cx < 0) cx = 0;
    else if (cx > width - 1) cx = width - 1;
    int64_t cy = (int64_t)nearbyint(gy);
    if (cy < 0) cy = 0;
    else if (cy > height - 1) cy = height - 1;
    double best = INFINITY;
    int64_t ylo = cy - 1 > 0 ? cy - 1 : 0, yhi = cy + 2 < height ? cy + 2 : height;
    int64_t xlo = cx - 1 > 0 ? cx - 1 : 0, xhi = cx + 2 < width ? cx + 2 : width;
    for (int64_t yy = ylo; yy < yhi; yy++)
        for (int64_t xx = xlo; xx < xhi; xx++) {
            double t = depth[yy * width + xx];
            if (isfinite(t)) {
                double diff = fabs(t - d);
                if (diff < best) best = diff;
            }
        }
    return best <= eps;
}

/* kernels.py:288-340 accumulate.  pos is (N,3) world, values (N,) in place.
 * candidates (optional, may be NULL): receives 1 for every sample that passes
 * the NDC crop filter (:302-319), i.e. the reference's filtered index set. */
void or_accumulate(const double *pos, int64_t N, const double rot[9], const double trans[3],
                   const double gaze[3], double sigma, double amp, double p00, double p11, double p02,
                   double p12, const double *depth, int height, int width, double eps_abs, double eps_rel,
                   double near, double far, double *values, uint8_t *candidates, int threads) {
    double inv_sigma = 1.0 / sigma;
    double near_lo = near * (1.0 - OR_NDC_SLACK);
    double far_hi = far * (1.0 + OR_NDC_SLACK);
    double lo = -1.0 - OR_NDC_SLACK, hi = 1.0 + OR_NDC_SLACK;
    (void)threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1) if (threads > 1)
#endif
    for (int64_t i = 0; i < N; i++) {
        double wx = pos[3 * i], wy = pos[3 * i + 1], wz = pos[3 * i + 2];
        double x = rot[0] * wx + rot[1] * wy + rot[2] * wz + trans[0];
        double y = rot[3] * wx + rot[4] * wy + rot[5] * wz + trans[1];
        double z = rot[6] * wx + rot[7] * wy + rot[8] * wz + trans[2];
        double w = -z;
        if (w <= 0.0) continue;
        double d = w;
        if (d < near_lo || d > far_hi) continue;
        double ndc_x = (p00 * x + p02 * z) / w;
        double ndc_y = (p11 * y + p12 * z) / w;
        if (ndc_x < lo || ndc_x > hi) continue;
        if (ndc_y < lo || ndc_y > hi) continue;
        if (candidates) candidates[i] = 1;
        if (!values) continue;
        double eps = eps_abs;
        if (eps_rel * d > eps) eps = eps_rel * d;
        if (!or_depth_match(depth, height, width, (ndc_x + 1.0) * 0.5 * width, (1.0 - ndc_y) * 0.5 * height,
                            d, eps))
            continue;
        double d1 = x * gaze[0] + y * gaze[1] + z * gaze[2];
        if (d1 <= 0.0) continue;
        double d2sq = x * x + y * y + z * z - d1 * d1;
        if (d2sq < 0.0) d2sq = 0.0;
        double ratio_sq = d2sq * inv_sigma * inv_sigma / (d1 * d1);
        if (ratio_sq > 16.0) continue;
        values[i] += amp * exp(-0.5 * ratio_sq);
    }
}

/* ----------------------------------------------------- density.generate */

/* density.py:136-227 generate (un-normalized).  Occluders are all scene
 * triangles in world space (T,3,3); samples are the included objects' world
 * positions concatenated (N,3); values (N,) are accumulated in place.
 * fixations is (F,18).  res is the square z-buffer side.  phase_s (may be NULL)
 * receives cull/rasterize/accumulate seconds (not timed here: zeros).
 * Returns 0 or an OR_ERR_* code with *bad_fixation set. */
int or_generate(const double *tris, int64_t T, const double *pos, int64_t N, const double *fixations,
                int64_t F, double theta, int res, double eps_abs, double eps_rel, int filtering,
                int threads, double *values, double *global_max, int64_t *bad_fixation) {
    double sigma = tan(theta);
    double setup[FS_LEN];
    double *depth = (double *)malloc(sizeof(double) * (size_t)res * (size_t)res);
    uint8_t *keep = (uint8_t *)malloc(T > 0 ? (size_t)T : 1);
    double *culled = (double *)malloc(sizeof(double) * 9 * (size_t)(T > 0 ? T : 1));
    double running_max = *global_max;
    for (int64_t f = 0; f < F; f++) {
        int rc = or_fixation_setup(fixations + 18 * f, theta, filtering, setup);
        if (rc) {
            if (bad_fixation) *bad_fixation = f;
            free(depth);
            free(keep);
            free(culled);
            return rc;
        }
        int64_t Tk = 0;
        if (T > 0) {
            double planes[24];
            or_frustum_planes(setup + FS_PROJ, setup + FS_VIEW, planes);
            or_cull_mask(tris, T, planes, keep);
            for (int64_t t = 0; t < T; t++)
                if (keep[t]) memcpy(culled + 9 * Tk++, tris + 9 * t, 9 * sizeof(double));
        }
        for (int64_t p = 0; p < (int64_t)res * res; p++) depth[p] = INFINITY;
        if (Tk)
            or_rasterize(culled, Tk, setup + FS_ROT, setup + FS_TRANS, setup[FS_P00], setup[FS_P11],
                         setup[FS_P02], setup[FS_P12], res, res, setup[FS_NEAR], setup[FS_FAR], depth);
        if (N > 0) {
            or_accumulate(pos, N, setup + FS_ROT, setup + FS_TRANS, setup + FS_GAZE, sigma, setup[FS_AMP],
                          setup[FS_P00], setup[FS_P11], setup[FS_P02], setup[FS_P12], depth, res, res,
                          eps_abs, eps_rel, setup[FS_NEAR], setup[FS_FAR], values, NULL, threads);
            double m = values[0];
            for (int64_t i = 1; i < N; i++)
                if (values[i] > m) m = values[i];
            if (m > running_max) running_max = m;
        }
    }
    *global_max = running_max;
    free(depth);
    free(keep);
    free(culled);
    return OR_OK;
}

int or_setup_len(void) { return FS_LEN; }
