// gm_fixlog.cpp -- fixation-log ingestion: the line parser of
// parse_fixation_log (reference gazemap/gaze.py:130-188) over an in-memory
// byte buffer, multi-threaded over line-aligned chunks, emitting the (F, 18)
// fixation table (gaze normalised exactly like Fixation.__post_init__,
// gaze.py:91-95) plus every row's Fixation validation verdict and its pose
// override groups.  The host (gaze.py in this package) applies the time
// window and raises the reference's ParseError for the first failure in file
// order.  Compiled with -ffp-contract=off; the only fused operations are the
// explicit fma() of the OpenBLAS ddot restatement.
//
// Text semantics follow Python's text-mode file iteration: universal newlines
// (\n, \r\n and a lone \r end a line), `raw.split("#", 1)[0].strip()`, tokens
// split on [,\s]+ and float() with its grammar (sign, digits with single
// underscores between digits, optional fraction/exponent, inf/infinity/nan).
// Buffers containing non-ASCII bytes are refused (GM_FIXLOG_NON_ASCII): Python
// treats Unicode whitespace/digits specially and the host parses those files
// with its restatement instead.
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

enum {
    K_NONE = 0,
    K_FEW_FIELDS = 1,    // "expected at least 18 fields, got N"
    K_BAD_FIELD = 2,     // "bad numeric field: <float() error of token>"
    K_GROUPS = 3,        // "pose override groups must be (object_id + 10 floats)"
    K_BAD_OVERRIDE = 4,  // "bad pose override for <oid>: <float() error of token>"
    K_NON_ASCII = 5,
    K_NO_TOKENS = 6,     // a line of separators only (IndexError in the reference)
};

// Python str.isspace() on ASCII (str.strip / re \s), '#'/',' handled by callers.
inline bool py_space(unsigned char c) {
    return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

inline bool ieq(const char* s, size_t n, const char* lit) {
    size_t m = strlen(lit);
    if (n != m) return false;
    for (size_t i = 0; i < n; i++) {
        char c = s[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != lit[i]) return false;
    }
    return true;
}

// float(token) (Objects/floatobject.c + Python/pystrtod.c): validate the
// grammar, drop the underscores, strtod (glibc: correctly rounded, like
// CPython's dtoa).  Returns false where float() raises ValueError.
bool py_float(const char* s, size_t n, double* out) {
    if (n == 0) return false;
    size_t i = 0;
    bool neg = false;
    if (s[0] == '+' || s[0] == '-') {
        neg = s[0] == '-';
        i = 1;
    }
    const char* r = s + i;
    size_t rn = n - i;
    if (ieq(r, rn, "inf") || ieq(r, rn, "infinity")) {
        *out = neg ? -INFINITY : INFINITY;
        return true;
    }
    if (ieq(r, rn, "nan")) {
        *out = NAN;  // CPython: float('-nan') is a NaN too
        return true;
    }
    char small[64];
    std::string big;
    char* dst = small;
    if (n + 1 > sizeof(small)) {
        big.resize(n + 1);
        dst = &big[0];
    }
    size_t k = 0;
    if (i) dst[k++] = s[0];
    auto digitpart = [&](size_t& p) -> bool {  // digit ("_"? digit)*
        if (p >= n || s[p] < '0' || s[p] > '9') return false;
        dst[k++] = s[p++];
        while (p < n) {
            if (s[p] >= '0' && s[p] <= '9') {
                dst[k++] = s[p++];
            } else if (s[p] == '_' && p + 1 < n && s[p + 1] >= '0' && s[p + 1] <= '9') {
                p++;
            } else {
                break;
            }
        }
        return true;
    };
    size_t p = i;
    bool int_digits = digitpart(p);
    bool frac_digits = false;
    if (p < n && s[p] == '.') {
        dst[k++] = s[p++];
        frac_digits = digitpart(p);
    }
    if (!int_digits && !frac_digits) return false;
    if (p < n && (s[p] == 'e' || s[p] == 'E')) {
        dst[k++] = s[p++];
        if (p < n && (s[p] == '+' || s[p] == '-')) dst[k++] = s[p++];
        if (!digitpart(p)) return false;
    }
    if (p != n) return false;
    dst[k] = 0;
    *out = strtod(dst, nullptr);
    return true;
}

struct Tok {
    int64_t off;
    int64_t len;
};

struct Group {
    int64_t oid_off, oid_len;
    double v[10];
    int32_t bad;  // index (0..9) of the first unparsable number, -1 if none
    int64_t bad_off, bad_len;
};

struct Chunk {
    std::vector<double> table;  // rows x 18
    std::vector<int64_t> line;  // local line number (1-based within chunk)
    std::vector<int32_t> code;  // Fixation.__post_init__ verdict
    std::vector<int64_t> gcount;
    std::vector<Group> groups;
    int64_t lines = 0;  // lines in the chunk
    int32_t err = K_NONE;
    int64_t err_line = 0, err_off = 0, err_len = 0, err_n = 0, err_off2 = 0, err_len2 = 0;
};

// np.linalg.norm of a 3-vector: sqrt(ddot(x, x)), OpenBLAS ddot = FMA chain
double np_norm3(const double* v) {
    double acc = v[0] * v[0];
    acc = fma(v[1], v[1], acc);
    acc = fma(v[2], v[2], acc);
    return sqrt(acc);
}

// Fixation.__post_init__ (gaze.py:88-104) on a raw row; normalises the gaze in place.
int32_t validate(double* r) {
    double* g = r + 15;
    const double norm = np_norm3(g);
    if (norm == 0.0) return 1;  // gaze_dir must be a nonzero vector
    g[0] = g[0] / norm;
    g[1] = g[1] / norm;
    g[2] = g[2] / norm;
    const double l = r[9], rr = r[10], t = r[11], b = r[12], n = r[13], f = r[14];
    if (r[1] <= 0) return 2;               // duration must be > 0
    if (!(n > 0 && f > n)) return 3;       // frustum needs 0 < near < far
    if (!(l < rr && b < t)) return 4;      // frustum needs left < right and bottom < top
    if (g[2] >= 0) return 5;               // gaze_dir must point into the viewed half-space
    return 0;
}

void parse_chunk(const char* buf, int64_t a, int64_t b, Chunk& C) {
    std::vector<Tok> toks;
    int64_t p = a, ln = 0;
    while (p < b) {
        // one line [p, e) ended by \n, \r\n or \r
        int64_t e = p;
        while (e < b && buf[e] != '\n' && buf[e] != '\r') e++;
        int64_t next = e;
        if (next < b) next += (buf[next] == '\r' && next + 1 < b && buf[next + 1] == '\n') ? 2 : 1;
        ln++;
        const int64_t line_start = p, line_end = e;
        // split("#", 1)[0].strip()
        int64_t q = p;
        while (q < e && buf[q] != '#') q++;
        int64_t s0 = p, s1 = q;
        while (s0 < s1 && py_space((unsigned char)buf[s0])) s0++;
        while (s1 > s0 && py_space((unsigned char)buf[s1 - 1])) s1--;
        p = next;
        if (s0 == s1) continue;
        toks.clear();
        int64_t c = s0;
        while (c < s1) {
            while (c < s1 && (buf[c] == ',' || py_space((unsigned char)buf[c]))) c++;
            if (c >= s1) break;
            int64_t t0 = c;
            while (c < s1 && buf[c] != ',' && !py_space((unsigned char)buf[c])) c++;
            toks.push_back({t0, c - t0});
        }
        auto fail = [&](int32_t kind, int64_t off, int64_t len) {
            C.err = kind;
            C.err_line = ln;
            C.err_off = off;
            C.err_len = len;
            C.err_n = (int64_t)toks.size();
            C.err_off2 = line_start;
            C.err_len2 = line_end - line_start;
        };
        if (toks.empty()) {  // separators only: the reference's tokens[0] raises IndexError
            fail(K_NO_TOKENS, 0, 0);
            break;
        }
        double v;
        if (!py_float(buf + toks[0].off, (size_t)toks[0].len, &v)) continue;  // header line
        if (toks.size() < 18) {
            fail(K_FEW_FIELDS, 0, 0);
            break;
        }
        double row[18];
        bool bad = false;
        for (int k = 0; k < 18; k++)
            if (!py_float(buf + toks[k].off, (size_t)toks[k].len, &row[k])) {
                fail(K_BAD_FIELD, toks[k].off, toks[k].len);
                bad = true;
                break;
            }
        if (bad) break;
        const size_t rest = toks.size() - 18;
        if (rest % 11 != 0) {
            fail(K_GROUPS, 0, 0);
            break;
        }
        for (size_t g0 = 18; g0 < toks.size(); g0 += 11) {
            Group G;
            G.oid_off = toks[g0].off;
            G.oid_len = toks[g0].len;
            G.bad = -1;
            G.bad_off = G.bad_len = 0;
            for (int k = 0; k < 10; k++) {
                const Tok& t = toks[g0 + 1 + k];
                if (!py_float(buf + t.off, (size_t)t.len, &G.v[k])) {
                    G.bad = k;
                    G.bad_off = t.off;
                    G.bad_len = t.len;
                    break;
                }
            }
            if (G.bad >= 0) {  // float() failed inside the group: the host formats the message
                fail(K_BAD_OVERRIDE, G.bad_off, G.bad_len);
                bad = true;
                break;
            }
            C.groups.push_back(G);
        }
        if (bad) break;
        C.code.push_back(validate(row));
        C.table.insert(C.table.end(), row, row + 18);
        C.line.push_back(ln);
        C.gcount.push_back((int64_t)(rest / 11));
    }
    C.lines = ln;
}

}  // namespace

struct gm_fixlog {
    int64_t rows = 0, ngroups = 0;
    std::vector<double> table;
    std::vector<int64_t> line, gstart;
    std::vector<int32_t> code;
    std::vector<Group> groups;
    int32_t err = K_NONE;
    int64_t err_line = 0, err_off = 0, err_len = 0, err_n = 0, err_off2 = 0, err_len2 = 0;
};

extern "C" {

// Parse a whole log buffer.  Always returns 0 and a handle (the error of the
// first failing line, if any, is in gm_fixlog_error) unless allocation fails.
int gm_fixlog_parse(const char* buf, int64_t len, int threads, gm_fixlog** out) {
    if (!out || (len > 0 && !buf) || len < 0) return 2;
    gm_fixlog* L = new gm_fixlog();
    *out = L;
    for (int64_t i = 0; i < len; i++)
        if ((unsigned char)buf[i] >= 0x80) {
            L->err = K_NON_ASCII;
            L->gstart.push_back(0);
            return 0;
        }
    int nt = 1;
#ifdef _OPENMP
    nt = threads > 0 ? threads : omp_get_max_threads();
#endif
    if (len < (1 << 20)) nt = 1;
    // chunk boundaries just after a '\n' (a "\r\n" pair never straddles one)
    std::vector<int64_t> cut(nt + 1, len);
    cut[0] = 0;
    for (int t = 1; t < nt; t++) {
        int64_t c = std::max(cut[t - 1], len * t / nt);
        while (c < len && buf[c - 1] != '\n') c++;
        cut[t] = c;
    }
    std::vector<Chunk> ch(nt);
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static, 1)
#endif
    for (int t = 0; t < nt; t++)
        if (cut[t] < cut[t + 1]) parse_chunk(buf, cut[t], cut[t + 1], ch[t]);
    int64_t line0 = 0;
    for (int t = 0; t < nt; t++) {
        Chunk& C = ch[t];
        const int64_t r = (int64_t)C.line.size();
        int64_t gi = 0;
        for (int64_t i = 0; i < r; i++) {
            L->line.push_back(line0 + C.line[i]);
            L->gstart.push_back(L->ngroups + gi);
            gi += C.gcount[i];
        }
        L->table.insert(L->table.end(), C.table.begin(), C.table.end());
        L->code.insert(L->code.end(), C.code.begin(), C.code.end());
        L->groups.insert(L->groups.end(), C.groups.begin(), C.groups.begin() + gi);
        L->rows += r;
        L->ngroups += gi;
        if (C.err != K_NONE) {
            L->err = C.err;
            L->err_line = line0 + C.err_line;
            L->err_off = C.err_off;
            L->err_len = C.err_len;
            L->err_n = C.err_n;
            L->err_off2 = C.err_off2;
            L->err_len2 = C.err_len2;
            break;
        }
        line0 += C.lines;
    }
    L->gstart.push_back(L->ngroups);
    return 0;
}

int64_t gm_fixlog_rows(const gm_fixlog* L) { return L ? L->rows : -1; }
int64_t gm_fixlog_groups(const gm_fixlog* L) { return L ? L->ngroups : -1; }

// table: rows x 18 (gaze normalised); line: 1-based file line per row; code:
// Fixation validation verdict (0 ok, 1 zero gaze, 2 duration, 3 near/far,
// 4 left/right or bottom/top, 5 gaze z >= 0); gstart: rows + 1 group offsets;
// goid: groups x 2 (byte offset, length of the object id); gvals: groups x 10.
// Any output may be NULL.
int gm_fixlog_copy(const gm_fixlog* L, double* table, int64_t* line, int32_t* code, int64_t* gstart, int64_t* goid,
                   double* gvals) {
    if (!L) return 2;
    if (table && L->rows) memcpy(table, L->table.data(), sizeof(double) * 18 * L->rows);
    if (line && L->rows) memcpy(line, L->line.data(), sizeof(int64_t) * L->rows);
    if (code && L->rows) memcpy(code, L->code.data(), sizeof(int32_t) * L->rows);
    if (gstart) memcpy(gstart, L->gstart.data(), sizeof(int64_t) * (L->rows + 1));
    for (int64_t g = 0; g < L->ngroups; g++) {
        if (goid) {
            goid[2 * g] = L->groups[g].oid_off;
            goid[2 * g + 1] = L->groups[g].oid_len;
        }
        if (gvals) memcpy(gvals + 10 * g, L->groups[g].v, sizeof(double) * 10);
    }
    return 0;
}

// info: kind, line, token offset, token length, field count, line offset, line length
// (the host re-parses the failing line alone to raise the reference's exact message)
int gm_fixlog_error(const gm_fixlog* L, int64_t* info) {
    if (!L || !info) return 2;
    info[0] = L->err;
    info[1] = L->err_line;
    info[2] = L->err_off;
    info[3] = L->err_len;
    info[4] = L->err_n;
    info[5] = L->err_off2;
    info[6] = L->err_len2;
    return 0;
}

void gm_fixlog_free(gm_fixlog* L) { delete L; }

}  // extern "C"
