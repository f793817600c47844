// Matrix Market reader (host code in libb200sp): the on-disk format feeding
// the path. Restates the reference's reader
// (src/mmio.py:38-126) -- same accepted subset (coordinate / array, real,
// general / symmetric), same errors with the same 1-based line numbers --
// as a two-pass parallel parser over the file image: pass 1 counts lines and
// entries per chunk, pass 2 parses every chunk into its slice of the triple
// arrays. Symmetric files expand the mirror entry right after each
// off-diagonal entry, as the reference does.
//
// Lines are split like Python's str.splitlines() on ASCII input (\n, \r,
// \r\n, \v, \f, \x1c, \x1d, \x1e); tokens like str.split() (whitespace runs).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace b200sp {
namespace {

inline bool is_break(char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
inline bool is_space(char c) { return c == ' ' || c == '\t' || is_break(c); }

// [s, e) of the line starting at p; returns the start of the next line
inline const char* next_line(const char* p, const char* end, const char** le) {
    const char* q = p;
    while (q < end && !is_break(*q)) ++q;
    *le = q;
    if (q < end) {
        if (*q == '\r' && q + 1 < end && q[1] == '\n') return q + 2;
        return q + 1;
    }
    return q;
}

inline void strip(const char*& s, const char*& e) {
    while (s < e && is_space(*s)) ++s;
    while (e > s && is_space(e[-1])) --e;
}

// whitespace tokens of [s, e): up to `cap` (start, end) pairs, returns the count
inline int tokens(const char* s, const char* e, const char** ts, const char** te, int cap) {
    int k = 0;
    while (s < e) {
        while (s < e && is_space(*s)) ++s;
        if (s >= e) break;
        const char* b = s;
        while (s < e && !is_space(*s)) ++s;
        if (k < cap) {
            ts[k] = b;
            te[k] = s;
        }
        ++k;
    }
    return k;
}

inline bool parse_i64(const char* s, const char* e, long long* out) {
    // Python int(): optional sign, digits (underscores between digits allowed)
    std::string t;
    for (const char* p = s; p < e; ++p)
        if (*p != '_') t.push_back(*p);
        else if (p == s || p + 1 == e || p[-1] == '_' || !isdigit((unsigned char)p[-1]) ||
                 !isdigit((unsigned char)p[1]))
            return false;
    if (t.empty()) return false;
    size_t i = (t[0] == '+' || t[0] == '-') ? 1 : 0;
    if (i >= t.size()) return false;
    for (size_t j = i; j < t.size(); ++j)
        if (!isdigit((unsigned char)t[j])) return false;
    errno = 0;
    *out = strtoll(t.c_str(), nullptr, 10);
    return errno == 0;
}

inline bool parse_f64(const char* s, const char* e, double* out) {
    // Python float(): decimal / exponent forms, inf, nan (strtod accepts the
    // same set except hex floats, which float() rejects)
    char buf[128];
    const size_t len = (size_t)(e - s);
    if (len == 0 || len >= sizeof(buf)) return false;
    size_t k = 0;
    for (const char* p = s; p < e; ++p)
        if (*p != '_') buf[k++] = *p;
    buf[k] = 0;
    if (k >= 2 && (buf[0] == '0' || ((buf[0] == '+' || buf[0] == '-') && buf[1] == '0')))
        for (size_t j = 0; j < k; ++j)
            if (buf[j] == 'x' || buf[j] == 'X') return false;
    char* endp = nullptr;
    *out = strtod(buf, &endp);
    return endp == buf + k;
}

struct Chunk {
    const char* begin;
    const char* end;
    long long lines = 0;    // line breaks inside the chunk (line-number base)
    long long entries = 0;  // data lines (non-blank, non-comment)
    long long out = 0;      // triples produced (symmetric mirrors included)
};

}  // namespace
}  // namespace b200sp

using namespace b200sp;

extern "C" {

/* header / size line: fills info[0..6] = {format (0 coordinate, 1 array),
 * symmetric, rows, cols, nnz (coordinate) , body offset (bytes), body line
 * (1-based line number of the first entry line's predecessor)} */
int b200sp_mm_header(const char* buf, int64_t len, int64_t* info, int64_t* err_line) {
    const char* end = buf + len;
    *err_line = 0;
    if (len == 0) {
        *err_line = 1;
        set_error("empty file");
        return B200SP_EINVAL;
    }
    const char* le;
    const char* p = next_line(buf, end, &le);
    const char* ts[6];
    const char* te[6];
    const int nt = tokens(buf, le, ts, te, 6);
    auto tok = [&](int i) { return std::string(ts[i], te[i]); };
    auto lower = [](std::string s) {
        for (auto& ch : s) ch = (char)tolower((unsigned char)ch);
        return s;
    };
    if (nt != 5 || tok(0) != "%%MatrixMarket" || lower(tok(1)) != "matrix") {
        *err_line = 1;
        set_error("expected '%%%%MatrixMarket matrix <format> <field> <symmetry>' header");
        return B200SP_EINVAL;
    }
    const std::string fmt = lower(tok(2)), field = lower(tok(3)), sym = lower(tok(4));
    if (fmt != "coordinate" && fmt != "array") {
        *err_line = 1;
        set_error("unknown format '%s'", fmt.c_str());
        return B200SP_EINVAL;
    }
    if (field != "real") {
        set_error("field '%s' is not supported (only 'real')", field.c_str());
        return B200SP_EUNSUPPORTED;
    }
    if (sym != "general" && sym != "symmetric") {
        set_error("symmetry '%s' is not supported (only 'general'/'symmetric')", sym.c_str());
        return B200SP_EUNSUPPORTED;
    }
    // size line: first non-blank, non-comment line
    long long lineno = 1;
    while (p < end) {
        const char* s = p;
        p = next_line(p, end, &le);
        ++lineno;
        const char* ss = s;
        const char* ee = le;
        strip(ss, ee);
        if (ss == ee || *ss == '%') continue;
        const int k = tokens(ss, ee, ts, te, 6);
        long long v[3] = {0, 0, 0};
        if (fmt == "coordinate") {
            if (k != 3) {
                *err_line = lineno;
                set_error("coordinate size line needs 'rows cols nnz'");
                return B200SP_EINVAL;
            }
        } else if (k != 2) {
            *err_line = lineno;
            set_error("array size line needs 'rows cols'");
            return B200SP_EINVAL;
        }
        for (int i = 0; i < k; ++i)
            if (!parse_i64(ts[i], te[i], &v[i])) {
                *err_line = lineno;
                set_error("malformed size line");
                return B200SP_EINVAL;
            }
        if (fmt == "array" && sym == "symmetric") {
            set_error("symmetric array files are not supported");
            return B200SP_EUNSUPPORTED;
        }
        info[0] = fmt == "array";
        info[1] = sym == "symmetric";
        info[2] = v[0];
        info[3] = v[1];
        info[4] = fmt == "coordinate" ? v[2] : v[0] * v[1];
        info[5] = (int64_t)(p - buf);
        info[6] = lineno;
        return B200SP_OK;
    }
    // the reference counts lines with splitlines(): a trailing break adds none
    *err_line = lineno;
    set_error("missing size line");
    return B200SP_EINVAL;
}

/* Count the triples the body produces (symmetric mirrors included) so the
 * caller can size the output; also validates nothing. threads <= 0: all. */
int b200sp_mm_count(const char* buf, int64_t len, const int64_t* info, int32_t threads, int64_t* out_count) {
    const char* body = buf + info[5];
    const char* end = buf + len;
    int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    const int64_t blen = end - body;
    nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, blen / (1 << 16) + 1));
    std::vector<Chunk> ch(nt);
    for (int i = 0; i < nt; ++i) {
        const char* s = body + blen * i / nt;
        const char* e = body + blen * (i + 1) / nt;
        ch[i].begin = s;
        ch[i].end = e;
    }
    // align chunk starts to line starts
    for (int i = 1; i < nt; ++i) {
        const char* s = ch[i].begin;
        while (s < end && !(is_break(s[-1]) && !(s[-1] == '\r' && *s == '\n'))) ++s;
        ch[i].begin = s;
        ch[i - 1].end = s;
    }
    const bool sym = info[1] != 0, arr = info[0] != 0;
    auto work = [&](int i) {
        Chunk& c = ch[i];
        const char* p = c.begin;
        const char* le;
        while (p < c.end) {
            const char* s = p;
            p = next_line(p, end, &le);
            const char* ss = s;
            const char* ee = le;
            strip(ss, ee);
            if (ss == ee || *ss == '%') continue;
            ++c.entries;
            if (arr || !sym) {
                ++c.out;
                continue;
            }
            const char* ts[3];
            const char* te[3];
            long long r = 0, cc = 0;
            if (tokens(ss, ee, ts, te, 3) == 3 && parse_i64(ts[0], te[0], &r) && parse_i64(ts[1], te[1], &cc) &&
                r != cc)
                c.out += 2;
            else
                c.out += 1;
        }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back(work, i);
    work(0);
    for (auto& t : th) t.join();
    int64_t tot = 0;
    for (auto& c : ch) tot += c.out;
    *out_count = tot;
    return B200SP_OK;
}

/* Parse the body into rows / cols (0-based, int64) and vals (coordinate), or
 * vals only (array, column-major as in the file). On error *err_line is the
 * reference's line number and the message matches src/mmio.py. */
int b200sp_mm_parse(const char* buf, int64_t len, const int64_t* info, int32_t threads, int64_t* rows,
                    int64_t* cols, double* vals, int64_t capacity, int64_t* out_count, int64_t* err_line) {
    *err_line = 0;
    const char* body = buf + info[5];
    const char* end = buf + len;
    const bool arr = info[0] != 0, sym = info[1] != 0;
    const long long R = info[2], C = info[3], N = info[4];
    int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    const int64_t blen = end - body;
    nt = (int)std::max<int64_t>(1, std::min<int64_t>(nt, blen / (1 << 16) + 1));
    std::vector<Chunk> ch(nt);
    for (int i = 0; i < nt; ++i) {
        ch[i].begin = body + blen * i / nt;
        ch[i].end = body + blen * (i + 1) / nt;
    }
    for (int i = 1; i < nt; ++i) {
        const char* s = ch[i].begin;
        while (s < end && !(is_break(s[-1]) && !(s[-1] == '\r' && *s == '\n'))) ++s;
        ch[i].begin = s;
        ch[i - 1].end = s;
    }
    // pass 1: lines, entries and outputs per chunk
    auto count = [&](int i) {
        Chunk& c = ch[i];
        const char* p = c.begin;
        const char* le;
        while (p < c.end) {
            const char* s = p;
            p = next_line(p, end, &le);
            ++c.lines;
            const char* ss = s;
            const char* ee = le;
            strip(ss, ee);
            if (ss == ee || *ss == '%') continue;
            ++c.entries;
            long long r = 0, cc = 0;
            const char* ts[3];
            const char* te[3];
            if (!arr && sym && tokens(ss, ee, ts, te, 3) == 3 && parse_i64(ts[0], te[0], &r) &&
                parse_i64(ts[1], te[1], &cc) && r != cc)
                c.out += 2;
            else
                c.out += 1;
        }
    };
    {
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i) th.emplace_back(count, i);
        count(0);
        for (auto& t : th) t.join();
    }
    std::vector<long long> line0(nt), out0(nt);
    long long ln = info[6], oo = 0, entries = 0;
    for (int i = 0; i < nt; ++i) {
        line0[i] = ln;
        out0[i] = oo;
        ln += ch[i].lines;
        oo += ch[i].out;
        entries += ch[i].entries;
    }
    // pass 2: parse; the first error in file order wins
    std::vector<long long> bad(nt, 0);
    std::vector<std::string> msg(nt);
    auto parse = [&](int i) {
        Chunk& c = ch[i];
        const char* p = c.begin;
        const char* le;
        long long lineno = line0[i];
        long long o = out0[i];
        while (p < c.end) {
            const char* s = p;
            p = next_line(p, end, &le);
            ++lineno;
            const char* ss = s;
            const char* ee = le;
            strip(ss, ee);
            if (ss == ee || *ss == '%') continue;
            const char* ts[4];
            const char* te[4];
            const int k = tokens(ss, ee, ts, te, 4);
            if (arr) {
                double v;
                if (!parse_f64(ts[0], te[0], &v)) {
                    bad[i] = lineno;
                    msg[i] = "malformed array value";
                    return;
                }
                if (o < capacity) vals[o] = v;
                ++o;
                continue;
            }
            if (k != 3) {
                bad[i] = lineno;
                msg[i] = "entry needs 'row col value'";
                return;
            }
            long long r, cc;
            double v;
            if (!parse_i64(ts[0], te[0], &r) || !parse_i64(ts[1], te[1], &cc) || !parse_f64(ts[2], te[2], &v)) {
                bad[i] = lineno;
                msg[i] = "malformed entry";
                return;
            }
            if (!(1 <= r && r <= R && 1 <= cc && cc <= C)) {
                char b[160];
                snprintf(b, sizeof(b), "index (%lld,%lld) outside %lldx%lld", r, cc, R, C);
                bad[i] = lineno;
                msg[i] = b;
                return;
            }
            if (o < capacity) {
                rows[o] = r - 1;
                cols[o] = cc - 1;
                vals[o] = v;
            }
            ++o;
            if (sym && r != cc) {
                if (o < capacity) {
                    rows[o] = cc - 1;
                    cols[o] = r - 1;
                    vals[o] = v;
                }
                ++o;
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i) th.emplace_back(parse, i);
        parse(0);
        for (auto& t : th) t.join();
    }
    for (int i = 0; i < nt; ++i)
        if (bad[i]) {
            *err_line = bad[i];
            set_error("%s", msg[i].c_str());
            return B200SP_EINVAL;
        }
    // splitlines() line count of the whole file (for count mismatches): the
    // lines up to the size line plus every body line
    const long long total_lines = ln;
    if (entries != N) {
        *err_line = total_lines;
        if (arr) set_error("expected %lld values, found %lld", N, entries);
        else set_error("expected %lld entries, found %lld", N, entries);
        return B200SP_EINVAL;
    }
    B200SP_REQUIRE(oo <= capacity, B200SP_EINVAL, "mm_parse: output capacity %lld < %lld", (long long)capacity, oo);
    *out_count = oo;
    return B200SP_OK;
}

}  // extern "C"
