// gm_samples.cuh -- the sample-major passes (included once by gm_kernels.cu):
// level-1 super-chunk ballots, the float32 marking pass k_mark and the
// exact accumulation pass k_samples (kernels.py:288-340).
#pragma once

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

// The float32 candidate test of one (sample, fixation) pair with rigorous
// error bounds (kernels.py:305-339: camera transform, depth slab, NDC crop
// filter, 4-sigma cone): GM_F32_REJECT only when the exact float64 test fails
// too; GM_F32_BLOCK with the range [cxlo, cxhi] x [cylo, cyhi] of the exact
// rint'ed texel coordinates; GM_F32_EXACT when the bounds are too loose to
// decide (samples within ~E of the camera plane).  dlo: lower bound of the
// exact depth w (GM_F32_BLOCK; up to float64 rounding).
enum { GM_F32_REJECT = 0, GM_F32_BLOCK = 1, GM_F32_EXACT = 2 };
__device__ __forceinline__ int mark_f32(const GmFixF32& Q, float wx, float wy, float wz, int W, int H, int& cxlo,
                                        int& cxhi, int& cylo, int& cyhi, double& dlo) {
    const float Wf = (float)W, Hf = (float)H;
    const float lo = -1.0f - (float)GM_NDC_SLACK, hi = 1.0f + (float)GM_NDC_SLACK;
    const float E = Q.E;
    const float x = __fmaf_rn(Q.rot[2], wz, __fmaf_rn(Q.rot[1], wy, __fmaf_rn(Q.rot[0], wx, Q.trans[0])));
    const float y = __fmaf_rn(Q.rot[5], wz, __fmaf_rn(Q.rot[4], wy, __fmaf_rn(Q.rot[3], wx, Q.trans[1])));
    const float z = __fmaf_rn(Q.rot[8], wz, __fmaf_rn(Q.rot[7], wy, __fmaf_rn(Q.rot[6], wx, Q.trans[2])));
    const float w = -z;
    if (w + E <= 0.0f) return GM_F32_REJECT;                           // exact w <= 0
    if (w + E < Q.near_lo || w - E > Q.far_hi) return GM_F32_REJECT;  // exact depth outside the slab
    const float wl = w - E;
    if (!(wl > 1e-3f * fabsf(w) + 1e-12f)) return GM_F32_EXACT;
    dlo = (double)w - (double)E;
    // NDC (kernels.py:314-319) with bound dq on |q32 - q_exact|
    const float nx = __fmaf_rn(Q.p00, x, Q.p02 * z), ny = __fmaf_rn(Q.p11, y, Q.p12 * z);
    // fast divisions (<= 2 ulp): covered by the 1e-6 relative slack of dq below
    const float rw = __fdividef(1.0f, w);
    const float qx = nx * rw, qy = ny * rw;
    const float en_x = (fabsf(Q.p00) + fabsf(Q.p02)) * E + 4e-7f * (fabsf(Q.p00 * x) + fabsf(Q.p02 * z));
    const float en_y = (fabsf(Q.p11) + fabsf(Q.p12)) * E + 4e-7f * (fabsf(Q.p11 * y) + fabsf(Q.p12 * z));
    const float rwl = __fdividef(1.0f, wl) * (1.0f + 1e-6f);
    const float dqx = (en_x + fabsf(qx) * E) * rwl + 1e-6f * fabsf(qx) + 1e-7f;
    const float dqy = (en_y + fabsf(qy) * E) * rwl + 1e-6f * fabsf(qy) + 1e-7f;
    if (qx + dqx < lo || qx - dqx > hi || qy + dqy < lo || qy - dqy > hi) return GM_F32_REJECT;
    // cone (kernels.py:330-339): d1 > 0 and ratio^2 <= 16
    const float d1 = __fmaf_rn(x, Q.gaze[0], __fmaf_rn(y, Q.gaze[1], z * Q.gaze[2]));
    const float ed1 = 2.0f * E + 4e-7f * (fabsf(x) + fabsf(y) + fabsf(z));
    if (d1 + ed1 <= 0.0f) return GM_F32_REJECT;
    const float cx3 = y * Q.gaze[2] - z * Q.gaze[1], cy3 = z * Q.gaze[0] - x * Q.gaze[2];
    const float cz3 = x * Q.gaze[1] - y * Q.gaze[0];
    const float cr = sqrtf(__fmaf_rn(cx3, cx3, __fmaf_rn(cy3, cy3, cz3 * cz3)));
    const float ecr = 3.0f * E + 1e-6f * (fabsf(x) + fabsf(y) + fabsf(z));
    const float crl = cr - ecr, d1h = d1 + ed1;
    if (crl > 0.0f && crl * crl > Q.sig16 * (1.0f + 1e-4f) * d1h * d1h) return GM_F32_REJECT;
    // range of the exact g (texel coordinates); rint is monotone
    const float gx = (qx + 1.0f) * 0.5f * Wf - 0.5f, gy = (1.0f - qy) * 0.5f * Hf - 0.5f;
    const float dgx = dqx * 0.5f * Wf + 1e-4f + 1e-6f * fabsf(gx);
    const float dgy = dqy * 0.5f * Hf + 1e-4f + 1e-6f * fabsf(gy);
    if (dgx > 2.0f || dgy > 2.0f) return GM_F32_EXACT;
    cxlo = (int)fminf(fmaxf(rintf(gx - dgx), 0.0f), (float)(W - 1));
    cxhi = (int)fminf(fmaxf(rintf(gx + dgx), 0.0f), (float)(W - 1));
    cylo = (int)fminf(fmaxf(rintf(gy - dgy), 0.0f), (float)(H - 1));
    cyhi = (int)fminf(fmaxf(rintf(gy + dgy), 0.0f), (float)(H - 1));
    return GM_F32_BLOCK;
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
                int cxlo, cxhi, cylo, cyhi;
                double dlo;
                const int st = mark_f32(fix32[f], wx, wy, wz, W, H, cxlo, cxhi, cylo, cyhi, dlo);
                if (st == GM_F32_REJECT) continue;
                if (st == GM_F32_EXACT) {
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
                }
                const int bx0 = max(cxlo - 1, 0), bx1 = min(cxhi + 1, W - 1);
                const int by0 = max(cylo - 1, 0), by1 = min(cyhi + 1, H - 1);
                my_bits |= 1u << j;
                const unsigned long long bits = ((1ull << (bx1 - bx0 + 1)) - 1ull) << (bx0 & 31);
                const uint32_t lo = (uint32_t)bits, hi = (uint32_t)(bits >> 32);
                const int ww = dv.wwords;
                uint32_t* row = dv.mask + ((int64_t)f * H + by0) * ww + (bx0 >> 5);
                if (dv.crowd_wide) {
                    // full-frustum batches: bits are only ever set during the pass, so a (possibly
                    // stale) read that already shows them proves the atomic redundant -- unfiltered
                    // C2 mark 74 -> 61 ms; in crop-frustum batches the extra read costs more than
                    // the atomics it saves (C2 +12%, C5 +42%)
                    for (int yy = by0; yy <= by1; yy++, row += ww) {
                        if ((__ldcg(row) & lo) != lo) atomicOr(row, lo);
                        if (hi && (__ldcg(row + 1) & hi) != hi) atomicOr(row + 1, hi);
                    }
                } else {
                    for (int yy = by0; yy <= by1; yy++, row += ww) {
                        atomicOr(row, lo);
                        if (hi) atomicOr(row + 1, hi);
                    }
                }
            }
            // level 3 for the accumulation pass: the fixations of this group with at
            // least one (float32-superset) candidate in this chunk
            const unsigned word = __reduce_or_sync(0xffffffffu, my_bits);
            if (lane == 0) cbits[ch * 32 + gi] = word;
        }
    }
}

#ifdef GM_CHECK
// Self-check of the sample-side culls (GM_CHECK builds only): every
// (sample, fixation) pair of the batch through the exact float64 candidate
// test of kernels.py:305-339; an exact candidate must be in its super-chunk's
// level-1 ballot and in k_mark's per-chunk fixation word, and every texel of
// its exact 3x3 depth_match block must be marked.
__global__ void k_check_candidates(const double* __restrict__ px, const double* __restrict__ py,
                                   const double* __restrict__ pz, int64_t N, const GmFixExact* __restrict__ fixes,
                                   int B, DepthView dv, double inv_sigma, const uint32_t* __restrict__ cbits,
                                   const uint32_t* __restrict__ lvl1, const long long* __restrict__ fail, long long b0) {
    if (*fail <= b0) return;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int W = dv.W, H = dv.H, ngroups = (B + 31) >> 5;
    const double lo = -1.0 - GM_NDC_SLACK, hi = 1.0 + GM_NDC_SLACK;
    const double wx = px[i], wy = py[i], wz = pz[i];
    const int64_t ch = i >> 5, sc = ch >> 3;
    unsigned long long n = 0, l1w = 0, l3w = 0, mw = 0;
    for (int f = 0; f < B; f++) {
        const GmFixExact& F = fixes[f];
        const double x = F.rot[0] * wx + F.rot[1] * wy + F.rot[2] * wz + F.trans[0];
        const double y = F.rot[3] * wx + F.rot[4] * wy + F.rot[5] * wz + F.trans[1];
        const double z = F.rot[6] * wx + F.rot[7] * wy + F.rot[8] * wz + F.trans[2];
        const double w = -z;
        if (w <= 0.0 || w < F.near_lo || w > F.far_hi) continue;
        const double ndc_x = (F.p00 * x + F.p02 * z) / w, ndc_y = (F.p11 * y + F.p12 * z) / w;
        if (ndc_x < lo || ndc_x > hi || ndc_y < lo || ndc_y > hi) continue;
        const double d1 = x * F.gaze[0] + y * F.gaze[1] + z * F.gaze[2];
        if (d1 <= 0.0) continue;
        double d2sq = x * x + y * y + z * z - d1 * d1;
        if (d2sq < 0.0) d2sq = 0.0;
        if (d2sq * inv_sigma * inv_sigma / (d1 * d1) > 16.0) continue;
        n++;
        const int g = f >> 5, j = f & 31;
        if (!((lvl1[sc * ngroups + g] >> j) & 1u)) {
            l1w++;
            continue;  // k_mark never looked at this pair (its word is not meaningful)
        }
        if (!((cbits[ch * 32 + g] >> j) & 1u)) l3w++;
        const double gx = (ndc_x + 1.0) * 0.5 * (double)W - 0.5, gy = (1.0 - ndc_y) * 0.5 * (double)H - 0.5;
        long long cx = x86_i64(rint(gx)), cy = x86_i64(rint(gy));
        cx = cx < 0 ? 0 : (cx > W - 1 ? W - 1 : cx);
        cy = cy < 0 ? 0 : (cy > H - 1 ? H - 1 : cy);
        const uint32_t* m = dv.mask + (int64_t)f * H * dv.wwords;
        for (long long yy = cy - 1; yy <= cy + 1; yy++)
            for (long long xx = cx - 1; xx <= cx + 1; xx++) {
                if (yy < 0 || yy > H - 1 || xx < 0 || xx > W - 1) continue;
                if (!((m[yy * dv.wwords + (xx >> 5)] >> (xx & 31)) & 1u)) mw++;
            }
    }
    chk_add(dv.check, GM_CHK_CAND_PAIRS, n);
    chk_add(dv.check, GM_CHK_CAND_L1_WRONG, l1w);
    chk_add(dv.check, GM_CHK_CAND_L3_WRONG, l3w);
    chk_add(dv.check, GM_CHK_MASK_WRONG, mw);
}
#endif

template <bool STATS>
__global__ void KS_BOUNDS k_samples(const double* __restrict__ px, const double* __restrict__ py,
                                                 const double* __restrict__ pz, const float4* __restrict__ chunks,
                                                 const uint32_t* __restrict__ lvl1, const int* __restrict__ order,
                                                 int* __restrict__ work, int64_t N, int64_t n_chunks,
                                                 int64_t n_supers, const GmFixExact* __restrict__ fixes,
                                                 const GmFixCull* __restrict__ culls, int B, DepthView dv,
                                                 double inv_sigma, double eps_abs, double eps_rel,
                                                 double* __restrict__ values, const uint32_t* __restrict__ cbits,
                                                 const GmScreenTri* __restrict__ tris, int64_t cap_seg,
                                                 const long long* __restrict__ fail, long long b0) {
    if (*fail <= b0) return;  // this batch overflowed the triangle store: the host redoes it
    const int lane = threadIdx.x & 31;
    const int ngroups = (B + 31) >> 5;  // <= 32 (B <= GM_MAX_BATCH)
    const int W = dv.W, H = dv.H;
    const double Wd = (double)W, Hd = (double)H;
    const double lo = -1.0 - GM_NDC_SLACK, hi = 1.0 + GM_NDC_SLACK;
    const int64_t n_items = n_supers * 8;
    unsigned c_l1 = 0, c_l2 = 0, c_exact = 0, c_ndc = 0, c_cand = 0, c_vis = 0, c_tocc = 0;
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
                if (dv.tmax && occluded_by_tiles(dv, f, bx0, bx1, by0, by1, d, eps)) {
                    if (STATS) c_tocc++;
#ifdef GM_CHECK
                    chk_add(dv.check, GM_CHK_DEPTH_TESTS, 1);
                    chk_add(dv.check, GM_CHK_TILEOCC_WRONG,
                            depth_test_exact(dv, tris + (int64_t)f * cap_seg, F.near_, F.far_, f, gx, gy, bx0, bx1,
                                             by0, by1, d, eps) ? 1 : 0);
#endif
                    continue;
                }
                const bool seen = depth_test_iv(dv, tris + (int64_t)f * cap_seg, F.near_, F.far_, f, gx, gy, bx0, bx1,
                                                by0, by1, d, eps);
#ifdef GM_CHECK
                chk_add(dv.check, GM_CHK_DEPTH_TESTS, 1);
                chk_add(dv.check, GM_CHK_DEPTH_WRONG,
                        seen != depth_test_exact(dv, tris + (int64_t)f * cap_seg, F.near_, F.far_, f, gx, gy, bx0,
                                                 bx1, by0, by1, d, eps) ? 1 : 0);
#endif
                if (!seen) continue;
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
        stat_add(dv.stats, GM_STAT_TILE_OCCLUDED, c_tocc);
    }
}

