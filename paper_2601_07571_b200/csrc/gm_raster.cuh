// gm_raster.cuh -- the general-camera raster API and the heatmap renderer
// (included once by gm_kernels.cu, after the plan helpers it uses).
#pragma once

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

