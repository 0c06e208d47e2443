// gm_export.cpp -- per-sample CSV export records, byte for
// byte what the reference's write_export (gazemap/io_export.py:63-116) writes
// for one object: "object_id,triangle_index,sample_index,w1,w2,w3,local_x,
// local_y,local_z,world_x,world_y,world_z,value", every float as f"{x:.9g}".
//
// Python's '.9g' and glibc's "%.9g" are both correctly rounded to 9
// significant digits with the same exponent rule and trailing-zero removal;
// the one spelling that differs (a NaN with the sign bit set: Python "nan",
// glibc "-nan") is special-cased.  Per-sample layout values follow the
// reference: triangle = np.repeat(arange(T), counts), within = i - offset,
// (row, col) from sample_rowcol (geometry.py:232-242; the integers are unique),
// w1 = col / r, w2 = (row - col) / r, w3 = 1.0 - row / r (float64 divisions).
// Local/world positions and values come from the GPU path (bit-exact with
// sample_positions_local / Transform.apply).  Formatting is OpenMP-parallel
// over sample ranges; the concatenation keeps sample order.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

struct gm_buffer {
    std::string data;
};

namespace {

inline int fmt9g(char* out, double x) {
    if (isnan(x)) {
        memcpy(out, "nan", 3);
        return 3;
    }
    return snprintf(out, 32, "%.9g", x);
}

inline int fmt_i64(char* out, int64_t v) { return snprintf(out, 24, "%lld", (long long)v); }

// sample_rowcol for one index (any exact method gives the same integers)
inline void rowcol(int64_t idx, int64_t* row, int64_t* col) {
    int64_t r = (int64_t)ceil((-3.0 + sqrt(8.0 * (double)idx + 9.0)) / 2.0);
    int64_t c = idx - r * (r + 1) / 2;
    while (c < 0) {
        r -= 1;
        c = idx - r * (r + 1) / 2;
    }
    while (c > r) {
        r += 1;
        c = idx - r * (r + 1) / 2;
    }
    *row = r;
    *col = c;
}

}  // namespace

extern "C" {

// Records of one object's N samples: res/offsets (T) the SampledMesh layout,
// local/world N x 3, values N.  *out receives a buffer handle (free with
// gm_buffer_free).  Returns 0, or 2 on bad arguments.
int gm_export_format(const char* oid, int64_t oid_len, const int64_t* res, const int64_t* offsets, int64_t T,
                     int64_t N, const double* local, const double* world, const double* values, int threads,
                     gm_buffer** out) {
    if (!out || N < 0 || T < 0 || (N > 0 && (!res || !offsets || !local || !world || !values))) return 2;
    int nt = 1;
#ifdef _OPENMP
    nt = threads > 0 ? threads : omp_get_max_threads();
#endif
    if (N < 4096) nt = 1;
    std::vector<std::string> parts(nt);
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static, 1)
#endif
    for (int t = 0; t < nt; t++) {
        const int64_t a = N * t / nt, b = N * (t + 1) / nt;
        if (a >= b) continue;
        std::string& s = parts[t];
        s.reserve((size_t)(b - a) * (size_t)(oid_len + 150));
        // triangle of sample a: last offset <= a (offsets ascending)
        int64_t lo = 0, hi = T - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (offsets[mid] <= a) lo = mid;
            else hi = mid - 1;
        }
        int64_t tri = lo;
        char buf[512];
        for (int64_t i = a; i < b; i++) {
            while (tri + 1 < T && offsets[tri + 1] <= i) tri++;
            const int64_t within = i - offsets[tri];
            int64_t row, col;
            rowcol(within, &row, &col);
            const double r = (double)res[tri];
            const double w1 = (double)col / r, w2 = (double)(row - col) / r, w3 = 1.0 - (double)row / r;
            s.append(oid, (size_t)oid_len);
            int n = 0;
            buf[n++] = ',';
            n += fmt_i64(buf + n, tri);
            buf[n++] = ',';
            n += fmt_i64(buf + n, within);
            const double f[10] = {w1, w2, w3, local[3 * i], local[3 * i + 1], local[3 * i + 2],
                                  world[3 * i], world[3 * i + 1], world[3 * i + 2], values[i]};
            for (int k = 0; k < 10; k++) {
                buf[n++] = ',';
                n += fmt9g(buf + n, f[k]);
            }
            buf[n++] = '\n';
            s.append(buf, (size_t)n);
        }
    }
    gm_buffer* B = new gm_buffer();
    size_t total = 0;
    for (auto& p : parts) total += p.size();
    B->data.reserve(total);
    for (auto& p : parts) B->data += p;
    *out = B;
    return 0;
}

const char* gm_buffer_data(const gm_buffer* b) { return b ? b->data.data() : nullptr; }
int64_t gm_buffer_size(const gm_buffer* b) { return b ? (int64_t)b->data.size() : -1; }
void gm_buffer_free(gm_buffer* b) { delete b; }

}  // extern "C"
