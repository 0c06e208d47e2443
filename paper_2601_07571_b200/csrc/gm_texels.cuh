// gm_texels.cuh -- k_texels, the marked z-buffer texels (included once by
// gm_kernels.cu): per (fixation, 32x16 tile) selection of the writing
// triangle in float32 with rigorous bounds, exact float64 evaluation of the
// survivors (kernels.py:67-137), and the sorted pass for crowded tiles.
#pragma once

#ifndef TW_CAP
#define TW_CAP 64  // triangles staged by the first pass (a multiple of 32); longer lists go to the crowded pass
#endif
#ifndef TEXEL_LIST
#define TEXEL_LIST 1  // first pass: each round's texels read from a per-tile compact list in shared memory
                      // (C2 -3%; the crowded pass keeps the search: a list there cost C5 +7%)
#endif
#ifndef TX_WARPS_SM
#define TX_WARPS_SM 28  // first-pass warps per SM the register budget is sized for (32 x 16 tiles: 72 registers)
#endif
#ifndef TX_WARPS_SM_CROP
#define TX_WARPS_SM_CROP 32  // ... 32 x 32 tiles (63 registers, no spills: C2 texels 154.1 -> 148.6 ms)
#endif
#ifndef TL_QUAD
#define TL_QUAD 1  // texel list in 16 x 16 quadrant order (else row order)
#endif
#ifndef SECTOR_FILL
#define SECTOR_FILL 0  // 1: write the unmarked texels of every touched 32-byte store sector (no DRAM RMW)
#endif
#ifndef RANK_CTA_MAX
#define RANK_CTA_MAX 0  // crowded pass: lists up to this long are ordered by rank counting, not bitonic
#endif
#ifndef RANK_SORT_MAX
#define RANK_SORT_MAX 16  // staged lists up to this long are ordered by rank counting, longer by bitonic sort
#endif
#define TW_SEL 128  // overlapping triangles remembered per tile (more: rescanned per round)
#ifndef TW_WARPS_CROP
#define TW_WARPS_CROP 1  // ... for the 32 x 32 tiles of crop-frustum batches (C2 -1%; 2 for the rest)
#endif
#ifndef TW_WARPS
#define TW_WARPS 2  // warps (independent tile items) per k_texels CTA
#endif
struct __align__(16) TexelWarpSmem {
    TriF32 t32[TW_CAP];  // staged, in ascending min-depth order
    int sel[TW_SEL + 32];
    float key[TW_SEL + 32];  // -inv_minw of sel[] (sort key: ascending min depth)
};
#define TX_DYN_SMEM (TW_WARPS * (int)sizeof(TexelWarpSmem))
// Crowded pass: one CTA of NW warps per tile; SELN overlap-list entries are
// gathered + sorted per pass (longer lists: several passes).  Crop-frustum
// (filtering) batches: 2 warps -- their crowded tiles are many and deep (C5:
// every tile), so the GPU is full either way and small CTAs waste the least at
// barriers (C2 texels -3%, C5 -11% against one warp per tile).  Full-frustum
// batches: 8 warps -- only ~7 tiles per fixation hold marked texels and the
// long lists (up to ~3,000 triangles over distant props) made a few serial
// tiles the whole launch; spreading a tile's rounds over 8 warps cut unfiltered
// C2 texels 398 -> 105 ms.
// crowded-pass warps per SM the register budget is sized for: 24 (80 registers) for the
// 2-warp crop-frustum CTAs (32: C5 texels +4%, shared memory), 32 (64 registers) for the
// 8-warp full-frustum ones (unfiltered C2 texels 105.5 -> 101.6 ms)
#ifndef HV_CROP_WARPS_SM
#define HV_CROP_WARPS_SM 24
#endif
#ifndef HV_FULL_WARPS_SM
#define HV_FULL_WARPS_SM 32
#endif
#ifndef HV_CROP_WARPS
#define HV_CROP_WARPS 2
#endif
#ifndef HV_CROP_SEL
#define HV_CROP_SEL 1024
#endif
#ifndef HV_FULL_WARPS
#define HV_FULL_WARPS 8
#endif
#ifndef HV_FULL_SEL
#define HV_FULL_SEL 2048
#endif
#ifndef EDGE_MIN
#define EDGE_MIN 1  // walk edge test as one min over the three edge functions (80-byte TriF32)
#endif
#ifndef WALK_SLOTS2
#define WALK_SLOTS2 1  // walk candidate slots: empty = -inf upper bound, "certainly written" in the lower bound's sign
#endif
#ifndef SORT_WARP
#define SORT_WARP 1  // crowded pass: bitonic sizes 2..32 by warp shuffles (C5 -0.6%; strides <= 16 of
#endif               // the larger sizes in registers too: C5 +5%)
#ifndef HV_CACHE
#define HV_CACHE 32  // crop-frustum crowded pass: the first HV_CACHE sorted records staged once per pass
#endif               // for all warps (full-frustum CTAs: 0 -- unfiltered C2 texels +12% with it)
#define HV_CACHE_FOR(NW) ((NW) == HV_CROP_WARPS ? HV_CACHE : 0)
template <int NW, int SELN>
struct __align__(16) HeavySmem {
    TriF32 cache[HV_CACHE_FOR(NW) > 0 ? HV_CACHE_FOR(NW) : 1];  // sorted records 0 .. HV_CACHE - 1 of the
                                                                 // current pass (shared by the warps)
    TriF32 t32[NW][32];    // each warp's staging slice (records beyond the cache)
    int sel[SELN + 4];     // sorted segment indices; [SELN]: pass count, [+1]: tile max, [+2]: claimed item
    float key[SELN];       // -inv_minw of sel[] (sort key: ascending min depth)
};
#define TX_MAX_THREADS (32 * TW_WARPS)

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
template <bool ATTRS, bool STATS, bool CROWDED, bool EXACT, int TH>
__device__ __forceinline__ void texel_item(TriF32* __restrict__ T32, int* __restrict__ SEL, float* __restrict__ KEY,
                                           int f, int tx, int ty, const TriStore& ts, const DepthView& dv,
                                           const CoarseBins& cb, int tiles_x, int tiles_per_fix,
                                           const GmFixExact* __restrict__ fixes, int sel_cap = 0,
                                           TriF32* __restrict__ CACHE = nullptr, int ncache_cap = 0) {
    const int lane = threadIdx.x & 31;
    const int64_t item = (int64_t)f * tiles_per_fix + ty * tiles_x + tx;
    const int W = dv.W, H = dv.H;
    const int xb = tx * TW, yb = ty * TH;
    const unsigned FULL = 0xffffffffu;
    // marked texels: lane r < TH holds the mask word of row yb + r
    uint32_t wr = 0;
    if (lane < TH && yb + lane < H) wr = dv.mask[((int64_t)f * H + yb + lane) * dv.wwords + (xb >> 5)];
    // per-fixation values every non-empty tile needs, loaded alongside the mask (independent of it)
    const int bb = (yb >> cb.shift) * cb.ncx + (xb >> cb.shift);
    const int* off = cb.off + (int64_t)f * (GM_MAX_CBINS + 1);
    const int ovf = cb.ovf[f], off0 = off[bb], off1 = off[bb + 1], count_f = ts.count[f];
    const double near_ = fixes[f].near_, far_ = fixes[f].far_;
    const int cnt_r = __popc(wr);
    int pref = cnt_r;  // inclusive prefix over rows
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, pref, o);
        if (lane >= o) pref += v;
    }
    const int total = __shfl_sync(FULL, pref, 31);
    if (total == 0) return;  // (its tmax stays stale: no depth test reads this tile)
    const int pref_ex = pref - cnt_r;
    // written iff near' <= 1/inv_w <= far' (kernels.py:123-127): certainly inside
    // [inv_far_hi, inv_near_lo], certainly outside beyond [inv_far_lo, inv_near_hi]
    // float32 reciprocals (<= 2 ulp from (float)(1/near')): far inside the 1e-5 margins below
    const float inv_near = __frcp_rn(__double2float_rn(near_)), inv_far = __frcp_rn(__double2float_rn(far_));
    const float inv_near_lo = inv_near * (1.0f - 1e-5f), inv_near_hi = inv_near * (1.0f + 1e-5f);
    const float inv_far_lo = inv_far * (1.0f - 1e-5f), inv_far_hi = inv_far * (1.0f + 1e-5f);
    const GmScreenTri* seg = ts.tris + (int64_t)f * ts.cap_seg;
    const uint2* segb = ts.bbox + (int64_t)f * ts.cap_seg;
    const int4* clist = nullptr;
    const TriF32* segf = ts.t32 + (int64_t)f * ts.cap_seg;
    int n = min(count_f, (int)ts.cap_seg);
    if (!ovf) {
        clist = cb.items + (int64_t)f * cb.cap_items + off0;
        n = off1 - off0;
    }
    const int xe = xb + TW - 1, ye = yb + TH - 1;
    unsigned long long c_pairs = 0, c_cov = 0, c_iter = 0, c_edge = 0;

    // 1. triangles overlapping the tile -> S.sel (scan cursor resumes if > TW_SEL)
    auto gather = [&](int& cursor) {
        int cnt = 0;
        while (cursor < n && cnt < TW_SEL) {
            int i = cursor + lane;
            bool sel = false;
            float key = 0.0f;
            if (i < n) {
                uint2 bbx;
                if (clist) {
                    const int4 e = clist[i];
                    i = e.x;
                    bbx = make_uint2((uint32_t)e.y, (uint32_t)e.z);
                    key = -__int_as_float(e.w);
                } else {
                    bbx = segb[i];
                    key = -__ldg(&segf[i].inv_minw);
                }
                const int x0 = bbx.x & 0xffff, x1 = bbx.x >> 16, y0 = bbx.y & 0xffff, y1 = bbx.y >> 16;
                sel = !(x1 < xb || x0 > xe || y1 < yb || y0 > ye);
            }
            const unsigned bal = __ballot_sync(FULL, sel);
            if (sel) {
                const int at = cnt + __popc(bal & ((1u << lane) - 1u));
                SEL[at] = i;
                KEY[at] = key;
            }
            cnt += __popc(bal);
            cursor += 32;
        }
        __syncwarp();
        return cnt;  // may exceed TW_SEL by < 32 (S.sel has the room)
    };

    // 2. stage SEL[c0 .. c0 + kend) (float32 forms) in ascending min-depth order.
    // Short lists: lane l's rank = the entries that sort before it (key, then list
    // position), one shuffle per entry; long ones: 32-wide bitonic network.
    auto stage = [&](int c0, int kend) {
        __syncwarp();
        if (TW_CAP > 32 && kend > 32) {  // TW_CAP / 32 entries per lane (lane + 32 m), ranks by counting
            constexpr int E = TW_CAP / 32;
            int gm_[E], rk[E];
            float km[E];
#pragma unroll
            for (int m = 0; m < E; m++) {
                const bool h = lane + 32 * m < kend;
                gm_[m] = h ? SEL[c0 + lane + 32 * m] : 0;
                km[m] = h ? KEY[c0 + lane + 32 * m] : CUDART_INF_F;
                rk[m] = 0;
            }
#pragma unroll
            for (int ms = 0; ms < E; ms++) {
                if (32 * ms >= kend) break;
                const int jn = min(32, kend - 32 * ms);
                for (int jl = 0; jl < jn; jl++) {
                    const float kj = __shfl_sync(FULL, km[ms], jl);
#pragma unroll
                    for (int m = 0; m < E; m++)  // entry j = 32 ms + jl sorts before entry 32 m + lane?
                        rk[m] += (kj < km[m] || (kj == km[m] && (ms < m || (ms == m && jl < lane)))) ? 1 : 0;
                }
            }
#pragma unroll
            for (int m = 0; m < E; m++) {
                if (lane + 32 * m < kend) {
                    const uint4* fr = reinterpret_cast<const uint4*>(segf + gm_[m]);
                    uint4* to = reinterpret_cast<uint4*>(&T32[rk[m]]);
#pragma unroll
                    for (int part = 0; part < TRI_WORDS; part++) to[part] = fr[part];
                }
            }
            __syncwarp();
            return;
        }
        const int gi = lane < kend ? SEL[c0 + lane] : 0;
        float key = lane < kend ? KEY[c0 + lane] : CUDART_INF_F;
        int dst, src;
        if (kend <= RANK_SORT_MAX) {
            int rank = 0;
            for (int j = 0; j < kend; j++) {
                const float kj = __shfl_sync(FULL, key, j);
                rank += (kj < key || (kj == key && j < lane)) ? 1 : 0;
            }
            dst = rank;  // this lane's record goes to slot `rank`
            src = gi;
        } else {
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
            dst = lane;  // lane = rank; it copies the record of sorted position `lane`
            src = __shfl_sync(FULL, gi, slot);
        }
        if (lane < kend) {
            const uint4* from = reinterpret_cast<const uint4*>(segf + src);
            uint4* to = reinterpret_cast<uint4*>(&T32[dst]);
#pragma unroll
            for (int part = 0; part < TRI_WORDS; part++) to[part] = from[part];
        }
        __syncwarp();
    };

    // texel of compact id q: (row, tile-local column)
    auto texel_of = [&](int q, int& row, int& colo, uint32_t& w_row) {
        row = 0;
#pragma unroll
        for (int step = TH / 2; step > 0; step >>= 1) {
            const int cand = row + step;
            const int pc = __shfl_sync(FULL, pref_ex, cand & 31);
            if (cand < TH && pc <= q) row = cand;
        }
        w_row = __shfl_sync(FULL, wr, row);
        const int k_in_row = q - __shfl_sync(FULL, pref_ex, row);
        colo = q < total ? kth_set_bit(w_row, k_in_row) : 0;
    };

    // 3 + 4 for the staged chunk (kend triangles) and one texel: updates V, best
    // kernels.py:128-129 writes iff d < depth[py, px]: among equal minima the
    // first triangle in rasterization order (key 2 t + fan) owns the texel
    auto take = [&](double d, int cs, double& best, int& bkey, int& bwin) {
        if (!ATTRS) {
            if (d < best) {
                best = d;
                bwin = cs;
            }
            return;
        }
        const int key = (int)(seg[cs].tl >> 3);
        if (d < best || (d == best && d < CUDART_INF && key < bkey)) {
            best = d;
            bkey = key;
            bwin = cs;
        }
    };
    // triangle kk of the walk: staged in shared memory
    auto tri_at = [&](int kk) -> const TriF32& { return T32[kk]; };
    // Returns true when (allow_fast) one certainly-written candidate provably wins:
    // then its segment index is in bwin and fastb holds rigorous float32 bounds of
    // its inverse depth at the texel -- no float64 evaluation (the accumulation pass
    // decides its depth tests on these bounds and evaluates only undecided ones).
    // fetch(kk): the kk-th triangle in walk order (warp-uniform kk); tri_all(k): the
    // same record for the slow path.
    auto walk_with = [&](int kend, auto&& fetch, auto&& tri_all, bool valid, int row, int colo, float& V,
                         double& best, int& bkey, int& bwin, bool allow_fast, float2& fastb) -> bool {
        const int px = xb + colo, py = yb + row;
        const float pxc = (float)px + 0.5f, pyc = (float)py + 0.5f;  // pixel centre
        int cs0 = -1, cs1 = -1;  // exact candidates (global record index) and their bounds
#if WALK_SLOTS2
        // a slot is live while its inverse-depth upper bound is >= V (empty: -inf); cl = the
        // lower bound when the triangle is certainly written there (> 0), else -1
        float ch0 = -CUDART_INF_F, ch1 = -CUDART_INF_F;
        float cl0 = -1.0f, cl1 = -1.0f;
#else
        float ch0 = 0.0f, ch1 = 0.0f;
        float cl0 = 0.0f, cl1 = 0.0f;   // their lower inverse-depth bounds
        bool ce0 = false, ce1 = false;  // certainly covering and written
#endif
        bool overflow = false;
        for (int kk = 0; kk < kend; kk++) {
            const TriF32& t = fetch(kk);
            // (inv_minw, ox, oy, wx) and (wy, gidx): both loads up front, so the bbox test
            // below is one predicate and one branch
            const float4 hd = *reinterpret_cast<const float4*>(&t.inv_minw);
            const float wy = t.wy;
            const float inv_minw = hd.x;
            if (__all_sync(FULL, !(inv_minw >= V))) break;  // nothing later can be nearer
            if (STATS) c_iter++;
            const float fx = pxc - hd.y, fy = pyc - hd.z;  // bbox-local centre (exact)
            const bool in = (inv_minw >= V) & (fx > 0.0f) & (fx < hd.w) & (fy > 0.0f) & (fy < wy);
            if (!in) continue;
            if (STATS) c_edge++;
#if TRI80 && EDGE_MIN
            // one tolerance for the three edges: all e_i >= -tol  <=>  min e_i >= -tol (the
            // planes and the bbox-local centre are finite, so no NaN reaches the min)
            const float em = fminf(fminf(__fmaf_rn(t.a[0], fx, __fmaf_rn(t.b[0], fy, t.c[0])),
                                         __fmaf_rn(t.a[1], fx, __fmaf_rn(t.b[1], fy, t.c[1]))),
                                   __fmaf_rn(t.a[2], fx, __fmaf_rn(t.b[2], fy, t.c[2])));
            if (!(em >= -t.tol)) continue;
            const bool certain = em > t.tol;
#else
            bool maybe = true, certain = true;
#pragma unroll
            for (int i = 0; i < 3; i++) {
                const float e = __fmaf_rn(t.a[i], fx, __fmaf_rn(t.b[i], fy, t.c[i]));
                maybe = maybe && (e >= -TRI_TOL(t, i));
                certain = certain && (e > TRI_TOL(t, i));
            }
            if (!maybe) continue;
#endif
            const float iwv = __fmaf_rn(t.A, fx, __fmaf_rn(t.B, fy, t.C));
            const float lo = iwv - t.tolw, hi = iwv + t.tolw;
            if (!(hi > 0.0f) || lo > inv_near_hi || hi < inv_far_lo) continue;  // certainly not written
            const bool cw = certain && lo > 0.0f && hi <= inv_near_lo && lo >= inv_far_hi;
            if (cw && lo * (1.0f - 1e-6f) > V) V = lo * (1.0f - 1e-6f);
#if WALK_SLOTS2
            if (hi >= V) {  // an empty or stale slot takes it (a stale one can never win again)
                const float clv = cw ? lo : -1.0f;
                if (ch0 < V) {
                    cs0 = t.gidx;
                    ch0 = hi;
                    cl0 = clv;
                } else if (ch1 < V) {
                    cs1 = t.gidx;
                    ch1 = hi;
                    cl1 = clv;
                } else {
                    overflow = true;
                }
            }
#else
            if (hi >= V) {
                if (cs0 < 0) {
                    cs0 = t.gidx;
                    ch0 = hi;
                    cl0 = lo;
                    ce0 = cw;
                } else if (cs1 < 0) {
                    cs1 = t.gidx;
                    ch1 = hi;
                    cl1 = lo;
                    ce1 = cw;
                } else if (ch0 < V) {  // a stale candidate can be replaced
                    cs0 = t.gidx;
                    ch0 = hi;
                    cl0 = lo;
                    ce0 = cw;
                } else if (ch1 < V) {
                    cs1 = t.gidx;
                    ch1 = hi;
                    cl1 = lo;
                    ce1 = cw;
                } else {
                    overflow = true;
                }
            }
#endif
        }
        if (!valid) return false;
#if WALK_SLOTS2
        const bool live0 = ch0 >= V, live1 = ch1 >= V;
        if (allow_fast && !overflow && live0 != live1 && (live0 ? cl0 : cl1) > 0.0f) {
#else
        const bool live0 = cs0 >= 0 && ch0 >= V, live1 = cs1 >= 0 && ch1 >= V;
        if (allow_fast && !overflow && live0 != live1 && (live0 ? ce0 : ce1)) {
#endif
            // the only candidate left is certainly written and every other triangle is
            // provably farther (inverse depth < V <= its own lower bound)
            bwin = live0 ? cs0 : cs1;
            fastb = make_float2((live0 ? cl0 : cl1) * (1.0f - 1e-6f), (live0 ? ch0 : ch1) * (1.0f + 1e-6f));
            return true;
        }
        if (!overflow) {
            if (live0) {
                const double d = texel_depth(seg[cs0], px, py, near_, far_);
                if (STATS) c_pairs++;
                if (STATS) c_cov += d < CUDART_INF;
                take(d, cs0, best, bkey, bwin);
            }
            if (live1) {
                const double d = texel_depth(seg[cs1], px, py, near_, far_);
                if (STATS) c_pairs++;
                if (STATS) c_cov += d < CUDART_INF;
                take(d, cs1, best, bkey, bwin);
            }
        } else {  // slow path: every staged triangle whose bbox covers the texel
            for (int k = 0; k < kend; k++) {
                const TriF32& t = tri_all(k);
                const float fx = pxc - t.ox, fy = pyc - t.oy;
                if (!(fx > 0.0f) || !(fx < t.wx) || !(fy > 0.0f) || !(fy < t.wy)) continue;
                const double d = texel_depth(seg[t.gidx], px, py, near_, far_);
                if (STATS) c_pairs++;
                if (STATS) c_cov += d < CUDART_INF;
                take(d, t.gidx, best, bkey, bwin);
            }
        }
        return false;
    };
    auto walk = [&](int kend, bool valid, int row, int colo, float& V, double& best, int& bkey, int& bwin,
                    bool allow_fast, float2& fastb) -> bool {
        return walk_with(kend, tri_at, tri_at, valid, row, colo, V, best, bkey, bwin, allow_fast, fastb);
    };

    double* dep = dv.depth + (int64_t)f * W * H;
    float2* dep2 = reinterpret_cast<float2*>(dv.depth) + (int64_t)f * W * H;  // !EXACT: depth bounds
    int* win = dv.win + (int64_t)f * W * H;                                    // !EXACT: the writer
    int cursor = 0;
    int nsel_total = 0;
    float tmax = -CUDART_INF_F;  // largest finite upper depth bound this lane stored
    // final value of texel `at`.  EXACT: the float64 depth kernels.rasterize leaves
    // there (+ the writer's order key with attributes).  Otherwise: rigorous float32
    // bounds [lo, hi] of that depth and the writing triangle's segment index, from
    // which k_samples re-evaluates the exact depth when a test is undecided.
#ifdef GM_CHECK
    // self-check (GM_CHECK builds): the exact min over every screen triangle whose
    // bbox holds the texel (the tile's coarse list, or the whole segment), against
    // what is stored -- EXACT: the depth bits; otherwise the writer's exact depth
    // and, on the fast path, the float32 bounds [lo, hi] around it
    auto check_texel = [&](int64_t at, double best, int w, float2 o, bool fast) {
        const int cx = (int)(at % W), cy = (int)(at / W);
        double bm = CUDART_INF;
        for (int i = 0; i < n; i++) {
            const int idx = clist ? clist[i].x : i;
            const GmScreenTri& T = seg[idx];
            if (cx < T.x0 || cx > T.x1 || cy < T.y0 || cy > T.y1) continue;
            bm = fmin(bm, texel_depth(T, cx, cy, near_, far_));
        }
        bool bad = false;
        if (EXACT) {
            bad = __double_as_longlong(best) != __double_as_longlong(bm);
        } else {
            const double dw = w >= 0 ? texel_depth(seg[w], cx, cy, near_, far_) : CUDART_INF;
            bad = __double_as_longlong(dw) != __double_as_longlong(bm);
            if (fast && !(dw >= (double)o.x && dw <= (double)o.y)) chk_add(dv.check, GM_CHK_TX_BOUND_WRONG, 1);
        }
        chk_add(dv.check, GM_CHK_TX_TEXELS, 1);
        chk_add(dv.check, GM_CHK_TX_WINNER_WRONG, bad ? 1 : 0);
    };
#endif
    auto store_at = [&](int64_t at, bool fast, float2 fb, double best, int bkey, int bwin) {
        if (EXACT) {
            dep[at] = best;
#ifdef GM_CHECK
            if (!ATTRS) check_texel(at, best, -1, make_float2(0.0f, 0.0f), false);
#endif
            if (ATTRS) dv.key[at] = best < CUDART_INF ? bkey : -1;
            return;
        }
        float2 o;
        int w = bwin;
        if (fast) {
#ifndef GM_RCP_EXACT
            // depth in [1/fb.y, 1/fb.x] (fb >= 1/far' > 0): rcp.approx is within 1 ulp
            // (PTX ISA), the 1e-6 widening covers it with room to spare
            float rl, rh;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rl) : "f"(fb.y));
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rh) : "f"(fb.x));
            o = make_float2(rl * (1.0f - 1e-6f), rh * (1.0f + 1e-6f));
#else
            o = make_float2(__frcp_rd(fb.y), __frcp_ru(fb.x));
#endif

        } else if (best < CUDART_INF) {
            o = make_float2(__double2float_rd(best), __double2float_ru(best));
        } else {
            o = make_float2(CUDART_INF_F, CUDART_INF_F);
            w = -1;
        }
        dep2[at] = o;
        win[at] = w;
        if (o.y < CUDART_INF_F) tmax = fmaxf(tmax, o.y);
#ifdef GM_CHECK
        check_texel(at, best, w, o, fast);
#endif
    };
    auto store = [&](int row, int colo, bool fast, float2 fb, double best, int bkey, int bwin) {
        store_at((int64_t)(yb + row) * W + xb + colo, fast, fb, best, bkey, bwin);
    };
    // Texel-store writes are sparse (3x3 blocks): a 32-byte sector left partly written costs a
    // DRAM read-modify-write when L2 evicts it.  The first marked texel of each sector (4 float2
    // bounds, 8 writer ints) also writes the sector's unmarked texels -- no reader ever looks at
    // an unmarked texel -- so every sector it touches is written whole.  (Generation batches,
    // W a multiple of 8 so sectors do not straddle rows.)
    const bool fill_sectors = !EXACT && (W & 7) == 0;
    auto fill = [&](int row, int colo, uint32_t w_row) {
        const int64_t rb = (int64_t)(yb + row) * W + xb;
        const uint32_t s4 = (w_row >> (colo & ~3)) & 0xFu;
        if ((s4 & ((1u << (colo & 3)) - 1u)) == 0u) {
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (!((s4 >> k) & 1u)) dep2[rb + (colo & ~3) + k] = make_float2(CUDART_INF_F, CUDART_INF_F);
        }
        const uint32_t s8 = (w_row >> (colo & ~7)) & 0xFFu;
        if ((s8 & ((1u << (colo & 7)) - 1u)) == 0u) {
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (!((s8 >> k) & 1u)) win[rb + (colo & ~7) + k] = -1;
        }
    };
    if (!CROWDED) {
        auto defer = [&]() {  // to k_texels_crowded, which sorts the whole list (one CTA per tile)
            if (lane == 0) dv.crowd[atomicAdd(dv.crowd_count, 1)] = (int)item;
            if (STATS) stat_add(dv.stats, GM_STAT_TX_CROWDED, lane == 0 ? 1ull : 0ull);
        };
        if (n > TW_SEL) {  // a long list: leave even the gather to the CTA pass
            defer();
            return;
        }
        const int nsel = gather(cursor);  // the whole list (n <= TW_SEL)
        if (STATS) nsel_total = nsel;
        if (nsel > TW_CAP) {  // more than this pass stages: the CTA pass sorts the whole list
            defer();
            return;
        }
        {
            // one staging serves every round, per-texel state in registers
            if (nsel > 0) stage(0, nsel);
#if TEXEL_LIST
            // the tile's marked texels as a compact (row << 5 | column) list in the gather
            // area (free once staged): lane r writes row r's, one read per texel per round
            // instead of a shuffle binary search + k-th set bit
            uint16_t* tlist = reinterpret_cast<uint16_t*>(SEL);
            constexpr int LCAP = (TW_SEL + 32) * 4;  // SEL + KEY, as 16-bit entries
            __syncwarp();
#if TL_QUAD
            if (total <= LCAP) {
                // 16 x 16 quadrants in turn (top left, top right, bottom left, bottom right):
                // a round's 32 texels then span ~16 x 8 texels instead of 32 x 4, so fewer
                // staged triangles reach any of its lanes (each texel's result does not depend
                // on which round it is in: the walk state is per lane)
                uint32_t lo = wr & 0xffffu, hi = wr >> 16;  // lanes >= TH hold 0
                const int cl = __popc(lo), ch = __popc(hi);
                int pl = cl, ph = ch;  // inclusive prefixes within each 16-row half
#pragma unroll
                for (int o = 1; o < 16; o <<= 1) {
                    const int vl = __shfl_up_sync(FULL, pl, o), vh = __shfl_up_sync(FULL, ph, o);
                    if ((lane & 15) >= o) {
                        pl += vl;
                        ph += vh;
                    }
                }
                const int top_lo = __shfl_sync(FULL, pl, 15), top_hi = __shfl_sync(FULL, ph, 15);
                const int bot_lo = __shfl_sync(FULL, pl, 31);
                const int base_lo = lane < 16 ? 0 : top_lo + top_hi;
                const int base_hi = lane < 16 ? top_lo : top_lo + top_hi + bot_lo;
                int al = base_lo + pl - cl, ah = base_hi + ph - ch;
                while (lo) {
                    tlist[al++] = (uint16_t)((lane << 5) | (__ffs(lo) - 1));
                    lo &= lo - 1;
                }
                while (hi) {
                    tlist[ah++] = (uint16_t)((lane << 5) | (__ffs(hi) + 15));
                    hi &= hi - 1;
                }
            } else
#endif
            if (lane < TH) {  // row order (the texel_of order, which rounds past LCAP use)
                uint32_t w = wr;
                int at = pref_ex;
                while (w && at < LCAP) {
                    tlist[at++] = (uint16_t)((lane << 5) | (__ffs(w) - 1));
                    w &= w - 1;
                }
            }
            __syncwarp();
#endif
            for (int r0 = 0; r0 < total; r0 += 32) {
                const int q = r0 + lane;
                const bool valid = q < total;
                int row, colo;
                uint32_t w_row;
#if TEXEL_LIST
                if (r0 + 32 <= LCAP) {
                    const unsigned e = valid ? tlist[q] : 0u;
                    row = (int)(e >> 5);
                    colo = (int)(e & 31u);
                    w_row = 0u;  // only the (disabled by default) sector fill reads it
                    if (SECTOR_FILL) w_row = __shfl_sync(FULL, wr, row);
                } else {
                    texel_of(q, row, colo, w_row);
                }
#else
                texel_of(q, row, colo, w_row);
#endif
                float V = valid ? 0.0f : CUDART_INF_F;
                double best = CUDART_INF;
                int bkey = INT_MAX, bwin = -1;
                float2 fb = make_float2(0.0f, 0.0f);
                bool fast = false;
                if (nsel > 0) fast = walk(nsel, valid, row, colo, V, best, bkey, bwin, !EXACT, fb);
                if (valid) {
                    store(row, colo, fast, fb, best, bkey, bwin);
                    if (SECTOR_FILL && fill_sectors) fill(row, colo, w_row);
                }
            }
        }
    } else {
        // crowded tile, one CTA (NW warps) per tile: the CTA gathers the whole
        // overlap list (sel_cap entries per pass), sorts it by ascending min depth (then
        // segment index) in shared memory, and its warps take the tile's rounds of 32
        // marked texels; each walks the sorted list, staging 32 float32 forms at a time
        // into its own slice.  The nearest certain cover proves (V) every later
        // triangle hidden, so a round usually ends after the first chunks -- nested
        // surfaces cost one sort, not one pass each; rounds run side by side.
        const int tid = threadIdx.x, warp = tid >> 5, nthr = blockDim.x;
        int* s_cnt = SEL + sel_cap;  // scalar slot after the arrays
        // state carried between passes of a list longer than sel_cap (the stored writer /
        // exact depth / order key are the outputs themselves)
        float* vb = dv.vbuf + (int64_t)f * W * H;
        double* carry = EXACT ? dep : dv.carry + (int64_t)f * W * H;
        bool first = true;
        do {
            if (tid == 0) *s_cnt = 0;
            __syncthreads();
            int cnt = 0;
            while (true) {  // blocks of nthr list entries until the pass is full or the list ends
                const int i0 = cursor + tid;
                if (i0 < n) {
                    int i = i0;
                    uint2 bbx;
                    float key;
                    if (clist) {
                        const int4 e = clist[i];
                        i = e.x;
                        bbx = make_uint2((uint32_t)e.y, (uint32_t)e.z);
                        key = -__int_as_float(e.w);
                    } else {
                        bbx = segb[i];
                        key = -__ldg(&segf[i].inv_minw);
                    }
                    const int x0 = bbx.x & 0xffff, x1 = bbx.x >> 16, y0 = bbx.y & 0xffff, y1 = bbx.y >> 16;
                    if (!(x1 < xb || x0 > xe || y1 < yb || y0 > ye)) {
                        const int at = atomicAdd(s_cnt, 1);
                        SEL[at] = i;
                        KEY[at] = key;
                    }
                }
                cursor += nthr;
                __syncthreads();
                cnt = *s_cnt;
                if (cursor >= n || cnt > sel_cap - nthr) break;
                __syncthreads();  // every thread has read the count before the next block adds to it
            }
            if (STATS) nsel_total += cnt;
            int so = 0;  // the sorted list starts at SEL + so / KEY + so
#if RANK_CTA_MAX > 0
            if (cnt <= RANK_CTA_MAX && 2 * cnt <= sel_cap) {
                // short list: every entry's rank by counting (broadcast reads), scattered into
                // the upper half -- one barrier instead of a bitonic network's log^2 of them
                so = sel_cap / 2;
                for (int e = tid; e < cnt; e += nthr) {
                    const float ke = KEY[e];
                    const int se = SEL[e];
                    int rank = 0;
                    for (int j = 0; j < cnt; j++) {
                        const float kj = KEY[j];
                        rank += (kj < ke || (kj == ke && SEL[j] < se)) ? 1 : 0;
                    }
                    SEL[so + rank] = se;
                    KEY[so + rank] = ke;
                }
                __syncthreads();
            } else
#endif
            {
            int P = 32;
            while (P < cnt) P <<= 1;
            for (int k = cnt + tid; k < P; k += nthr) {
                KEY[k] = CUDART_INF_F;
                SEL[k] = INT_MAX;
            }
            __syncthreads();
            // CTA bitonic sort of (KEY, SEL) ascending, P <= sel_cap
            int size0 = 2;
#if SORT_WARP
            // sizes 2 .. 32 inside each 32-entry segment: warp shuffles in registers, the
            // same network (direction of each pair from its global index), no barriers
            for (int sgm = warp; sgm < (P >> 5); sgm += nthr >> 5) {
                const int a0 = sgm * 32 + lane;
                float k = KEY[a0];
                int sv = SEL[a0];
#pragma unroll
                for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                    for (int stride = size >> 1; stride > 0; stride >>= 1) {
                        const float ok = __shfl_xor_sync(FULL, k, stride);
                        const int os = __shfl_xor_sync(FULL, sv, stride);
                        const bool self_gt = k > ok || (k == ok && sv > os);
                        const bool want_min = ((lane & stride) == 0) == ((a0 & size) == 0);
                        if (want_min ? self_gt : (!self_gt && !(k == ok && sv == os))) {
                            k = ok;
                            sv = os;
                        }
                    }
                }
                KEY[a0] = k;
                SEL[a0] = sv;
            }
            __syncthreads();
            size0 = 64;
#endif
            for (int size = size0; size <= P; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int t = tid; t < (P >> 1); t += nthr) {
                        const int a = 2 * t - (t & (stride - 1)), b = a + stride;
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
                    __syncthreads();
                }
            }
            }
            const bool last = cursor >= n;
            const int* SS = SEL + so;  // sorted segment indices
            // the head of the sorted list (ncache_cap records), staged once for every warp and
            // round of the pass (a round's walk usually ends inside it: the nearest covers
            // prove the rest hidden)
            const int NCH = ncache_cap;
            if (NCH > 0) {
                const int ncache = min(cnt, NCH);
                for (int k = tid; k < ncache * TRI_WORDS; k += nthr) {
                    const int r = k / TRI_WORDS, part = k - r * TRI_WORDS;
                    reinterpret_cast<uint4*>(&CACHE[r])[part] = reinterpret_cast<const uint4*>(segf + SS[r])[part];
                }
                __syncthreads();
            }
            // walk order: the sorted list -- the shared head, then 32 records at a time staged
            // into this warp's slice
            auto fetch = [&](int kk) -> const TriF32& {
                if (kk < NCH) return CACHE[kk];
                const int k2 = kk - NCH;
                if ((k2 & 31) == 0) {
                    __syncwarp();
                    const int k = kk + lane;
                    if (k < cnt) {
                        const uint4* from = reinterpret_cast<const uint4*>(segf + SS[k]);
                        uint4* to = reinterpret_cast<uint4*>(&T32[lane]);
#pragma unroll
                        for (int part = 0; part < TRI_WORDS; part++) to[part] = from[part];
                    }
                    __syncwarp();
                }
                return T32[k2 & 31];
            };
            auto from_global = [&](int k) -> const TriF32& { return segf[SS[k]]; };
            for (int r0 = warp * 32; r0 < total; r0 += nthr) {
                const int q = r0 + lane;
                const bool valid = q < total;
                int row, colo;
                uint32_t w_row;
                texel_of(q, row, colo, w_row);
                const int64_t at = (int64_t)(yb + row) * W + xb + colo;
                float V = valid ? (first ? 0.0f : vb[at]) : CUDART_INF_F;
                double best = (valid && !first) ? carry[at] : CUDART_INF;
                int bkey = INT_MAX, bwin = -1;
                if (ATTRS && valid && !first) bkey = dv.key[at];
                if (!EXACT && valid && !first) bwin = win[at];
                float2 fb = make_float2(0.0f, 0.0f);
                bool fast = false;
                // a single pass (the usual case) may take the float32 fast path
                if (cnt > 0)
                    fast = walk_with(cnt, fetch, from_global, valid, row, colo, V, best, bkey, bwin,
                                     !EXACT && first && last, fb);
                if (valid) {
                    if (SECTOR_FILL && fill_sectors && first) fill(row, colo, w_row);
                    if (last) {
                        store_at(at, fast, fb, best, bkey, bwin);
                    } else {
                        vb[at] = V;
                        carry[at] = best;
                        if (ATTRS) dv.key[at] = best < CUDART_INF ? bkey : -1;
                        if (!EXACT) win[at] = bwin;
                    }
                }
            }
            first = false;
            __syncthreads();  // the next pass overwrites SEL / KEY
        } while (cursor < n);
    }
    if (!EXACT && dv.tmax) {
        // depths are > 0: the float bit patterns order like ints (-inf < every depth)
        const int m = __reduce_max_sync(FULL, __float_as_int(tmax));
        if (!CROWDED) {
            if (lane == 0) dv.tmax[item] = __int_as_float(m);
        } else {  // every warp of the CTA holds a share of the tile's texels
            int* s_max = SEL + sel_cap + 1;
            if (threadIdx.x == 0) *s_max = __float_as_int(-CUDART_INF_F);
            __syncthreads();
            if (lane == 0) atomicMax(s_max, m);
            __syncthreads();
            if (threadIdx.x == 0) dv.tmax[item] = __int_as_float(*s_max);
        }
    }
    if (STATS) {
        const bool l0 = lane == 0;
        const bool t0 = l0 && (!CROWDED || threadIdx.x == 0);  // per-tile counts: one warp of the CTA
        stat_add(dv.stats, GM_STAT_TEXELS, t0 ? (unsigned long long)total : 0ull);
        stat_add(dv.stats, GM_STAT_TX_TILES, t0 ? 1ull : 0ull);
        stat_add(dv.stats, GM_STAT_TX_STAGED, t0 ? (unsigned long long)nsel_total : 0ull);
        stat_add(dv.stats, GM_STAT_TX_LIST, t0 ? (unsigned long long)n : 0ull);
        stat_add(dv.stats, GM_STAT_TX_ITER, l0 ? c_iter : 0ull);
        stat_add(dv.stats, GM_STAT_PAIRS, c_pairs);
        stat_add(dv.stats, GM_STAT_COVERED, c_cov);
        stat_add(dv.stats, GM_STAT_TX_EDGE, c_edge);
    }
}

// Warps per first-pass CTA for a tile height (registers capped at 72 either way).
template <int TH>
struct TexelWarps {
    static constexpr int n = TH == 32 ? TW_WARPS_CROP : TW_WARPS;
    static constexpr int ctas = (TH == 32 ? TX_WARPS_SM_CROP : TX_WARPS_SM) / n;  // resident CTAs per SM
};
// First pass: grid (tiles_x, ceil(tiles_y / n), fixations); warp w of a CTA takes
// tile row blockIdx.y * n + w.
template <bool ATTRS, bool STATS, bool EXACT, int TH>
__global__ void __launch_bounds__(TexelWarps<TH>::n * 32, TexelWarps<TH>::ctas) k_texels(TriStore ts, DepthView dv,
                                                                                    CoarseBins cb, int tiles_x,
                                   int tiles_per_fix, int tiles_y,
                                   const GmFixExact* __restrict__ fixes, long long b0) {
    extern __shared__ __align__(16) unsigned char tx_dyn[];
    const int warp = threadIdx.x >> 5;
    if (*ts.fail <= b0) return;
    const int ty = blockIdx.y * TexelWarps<TH>::n + warp;
    if (ty < tiles_y)
        texel_item<ATTRS, STATS, false, EXACT, TH>(reinterpret_cast<TexelWarpSmem*>(tx_dyn)[warp].t32,
                                               reinterpret_cast<TexelWarpSmem*>(tx_dyn)[warp].sel,
                                               reinterpret_cast<TexelWarpSmem*>(tx_dyn)[warp].key, blockIdx.z,
                                               blockIdx.x, ty, ts, dv, cb, tiles_x, tiles_per_fix, fixes);
}

// Crowded pass: persistent CTAs of NW warps over the tiles the first pass
// deferred, one tile per CTA at a time (texel_item, CROWDED branch).
template <bool ATTRS, bool STATS, bool EXACT, int NW, int SELN, int TH>
__global__ void __launch_bounds__(NW * 32, (NW == HV_FULL_WARPS ? HV_FULL_WARPS_SM : HV_CROP_WARPS_SM) / NW) k_texels_crowded(TriStore ts, DepthView dv, CoarseBins cb,
                                                                     int tiles_x, int tiles_per_fix,
                                                                     const GmFixExact* __restrict__ fixes,
                                                                     long long b0) {
    extern __shared__ __align__(16) unsigned char tx_dyn[];
    HeavySmem<NW, SELN>& C = *reinterpret_cast<HeavySmem<NW, SELN>*>(tx_dyn);
    const int warp = threadIdx.x >> 5;
    if (*ts.fail <= b0) return;
    const int n_crowd = *dv.crowd_count;
    int* claim = C.sel + SELN + 2;
    for (;;) {
        if (threadIdx.x == 0) *claim = atomicAdd(dv.crowd_count + 1, 1);
        __syncthreads();
        const int w = *claim;
        __syncthreads();  // every warp has read the claim before thread 0 replaces it
        if (w >= n_crowd) break;
        const int item = dv.crowd[w];
        const int f = item / tiles_per_fix, tile = item - f * tiles_per_fix;
        texel_item<ATTRS, STATS, true, EXACT, TH>(C.t32[warp], C.sel, C.key, f, tile % tiles_x, tile / tiles_x, ts, dv,
                                              cb, tiles_x, tiles_per_fix, fixes, SELN, C.cache, HV_CACHE_FOR(NW));
    }
}
