// hb_io.cpp -- bulk polyline export / import (reference io.py:136-171).
//
// export_polylines writes, per edge, "e bin weight n x0 y0 x1 y1 ..." with
// every float formatted as %.9g.  For millions of polylines the per-number
// Python formatting dominates everything else, so the records are formatted
// here with std::to_chars(general, 9) -- specified to produce exactly what
// printf("%.9g") does, which is also what Python's format(x, ".9g") does --
// in parallel over edge ranges, and written in edge order.
//
// Host code (no GPU): the polylines are already on the host after bundle().
#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <system_error>
#include <thread>
#include <vector>
#include <unistd.h>

#define HB_IO_API extern "C" __attribute__((visibility("default")))

namespace {

inline char *put_i64(char *p, char *end, int64_t v) {
    return std::to_chars(p, end, v).ptr;
}
inline char *put_g9(char *p, char *end, double v) {
    return std::to_chars(p, end, v, std::chars_format::general, 9).ptr;
}

// worst case characters of one record: 3 integers + 1 weight + 2n coordinates
inline int64_t record_bound(int64_t n) { return 3 * 21 + 4 + 32 + 2 * n * 32 + 1; }

// records [e_lo, e_hi) into out (appended)
void format_range(const double *world, const int64_t *starts, const int64_t *bins,
                  const double *weights, const int64_t *index, int64_t e_lo, int64_t e_hi,
                  std::string &out) {
    int64_t need = 0;
    for (int64_t e = e_lo; e < e_hi; ++e) need += record_bound(starts[e + 1] - starts[e]);
    const size_t off = out.size();
    out.resize(off + (size_t)need);
    char *p = out.data() + off, *end = out.data() + out.size();
    for (int64_t e = e_lo; e < e_hi; ++e) {
        const int64_t s = starts[e], n = starts[e + 1] - s;
        const int64_t ei = index ? index[e] : e;
        p = put_i64(p, end, ei);
        *p++ = ' ';
        p = put_i64(p, end, bins ? bins[ei] : 0);
        *p++ = ' ';
        p = put_g9(p, end, weights ? weights[ei] : 1.0);
        *p++ = ' ';
        p = put_i64(p, end, n);
        const double *w = world + 2 * s;
        for (int64_t k = 0; k < 2 * n; ++k) {
            *p++ = ' ';
            p = put_g9(p, end, w[k]);
        }
        *p++ = '\n';
    }
    out.resize((size_t)(p - out.data()));
}

int write_all(int fd, const char *p, size_t n) {
    while (n) {
        const ssize_t w = ::write(fd, p, n);
        if (w < 0) {
            if (errno == EINTR) continue;
            return -errno;
        }
        p += w;
        n -= (size_t)w;
    }
    return 0;
}

}  // namespace

// Format records of edges [e_lo, e_hi) into buf (capacity cap).  Stops before
// the first record that does not fit; returns the number of records written
// and their byte count in *used.  bins / weights are indexed by the edge's
// graph index (index[e] when given, else e); NULL means 0 / 1.0.
HB_IO_API int64_t hb_io_format(const double *world, const int64_t *starts, const int64_t *bins,
                               const double *weights, const int64_t *index, int64_t e_lo,
                               int64_t e_hi, char *buf, int64_t cap, int64_t *used) {
    std::string tmp;
    int64_t done = 0, pos = 0;
    for (int64_t e = e_lo; e < e_hi; ++e) {
        tmp.clear();
        format_range(world, starts, bins, weights, index, e, e + 1, tmp);
        if (pos + (int64_t)tmp.size() > cap) break;
        std::memcpy(buf + pos, tmp.data(), tmp.size());
        pos += (int64_t)tmp.size();
        ++done;
    }
    if (used) *used = pos;
    return done;
}

// Whole export (header + records) to a file descriptor, `threads` formatters
// working on consecutive edge ranges of ~`chunk_points` points per round,
// written in order.  Returns 0 or -errno.
HB_IO_API int hb_io_export_fd(int fd, const double *world, const int64_t *starts,
                              const int64_t *bins, const double *weights, const int64_t *index,
                              int64_t n_edges, int threads) {
    std::string head = "# histobundle polylines v1\n# edges " + std::to_string(n_edges) + "\n";
    int rc = write_all(fd, head.data(), head.size());
    if (rc) return rc;
    if (threads < 1) threads = 1;
    const int64_t chunk_points = 1 << 20;  // per formatter per round
    std::vector<std::string> bufs((size_t)threads);
    int64_t e = 0;
    while (e < n_edges) {
        // consecutive ranges of ~chunk_points points each
        std::vector<int64_t> cut(1, e);
        for (int t = 0; t < threads && cut.back() < n_edges; ++t) {
            const int64_t target = starts[cut.back()] + chunk_points;
            int64_t hi = std::upper_bound(starts + cut.back() + 1, starts + n_edges + 1, target) -
                         starts - 1;
            if (hi <= cut.back()) hi = cut.back() + 1;
            cut.push_back(std::min(hi, n_edges));
        }
        const int nt = (int)cut.size() - 1;
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t) {
            bufs[(size_t)t].clear();
            pool.emplace_back(format_range, world, starts, bins, weights, index, cut[(size_t)t],
                              cut[(size_t)t + 1], std::ref(bufs[(size_t)t]));
        }
        for (auto &th : pool) th.join();
        for (int t = 0; t < nt; ++t) {
            rc = write_all(fd, bufs[(size_t)t].data(), bufs[(size_t)t].size());
            if (rc) return rc;
        }
        e = cut.back();
    }
    return 0;
}

// ---------------------------------------------------------------------------
// import (read_polylines, io.py:148-171)

namespace {

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// next whitespace-separated token of the line [p, line_end)
inline bool token(const char *&p, const char *le, const char *&t0, const char *&t1) {
    while (p < le && is_space(*p)) ++p;
    if (p >= le) return false;
    t0 = p;
    while (p < le && !is_space(*p)) ++p;
    t1 = p;
    return true;
}

template <typename T>
inline bool parse_num(const char *t0, const char *t1, T &v) {
    const auto r = std::from_chars(t0, t1, v);
    return r.ec == std::errc() && r.ptr == t1;
}

}  // namespace

// Two-phase parse of an export.  fill == false: count records and
// coordinates (*n_records, *n_coords).  fill == true: write edge_index,
// bins, weights, starts (n_records+1, point offsets) and coords (2 per
// point).  Returns 0; 1 = "use the Python parser" (a token this fast path
// does not accept, e.g. '+1' or '1_0'); -1 = malformed record, -2 = count
// mismatch, both with the 1-based line in *err_line (and, for -2, the
// expected / found coordinate counts in *err_a / *err_b).
namespace {

// one line-aligned chunk; line numbers start after `line0`; records/coords
// are written from rec0 / nc0 (fill) and counted in *n_rec / *n_c / *n_lines
int parse_chunk(const char *text, const char *end, int fill, int64_t line0, int64_t rec0,
                int64_t nc0, int64_t *n_rec, int64_t *n_c, int64_t *n_lines,
                int64_t *edge_index, int64_t *bins, double *weights, int64_t *starts,
                double *coords, int64_t *err_line, int64_t *err_a, int64_t *err_b) {
    const char *p = text;
    int64_t line = line0, rec = rec0, nc = nc0;
    while (p < end) {
        const char *le = (const char *)std::memchr(p, '\n', (size_t)(end - p));
        if (!le) le = end;
        ++line;
        const char *q = p;
        while (q < le && is_space(*q)) ++q;
        if (q < le && *q != '#') {
            const char *t0, *t1;
            int64_t ei, bn, n;
            double w;
            if (!token(q, le, t0, t1)) goto malformed;
            if (!parse_num(t0, t1, ei)) goto fallback_or_bad;
            if (!token(q, le, t0, t1)) goto malformed;
            if (!parse_num(t0, t1, bn)) goto fallback_or_bad;
            if (!token(q, le, t0, t1)) goto malformed;
            if (!parse_num(t0, t1, w)) goto fallback_or_bad;
            if (!token(q, le, t0, t1)) goto malformed;
            if (!parse_num(t0, t1, n)) goto fallback_or_bad;
            int64_t got = 0;
            while (token(q, le, t0, t1)) {
                double c;
                if (!parse_num(t0, t1, c)) goto fallback_or_bad;
                if (fill && got < 2 * n) coords[nc + got] = c;
                ++got;
            }
            if (got != 2 * n) {
                *err_line = line;
                *err_a = 2 * n;
                *err_b = got;
                return -2;
            }
            if (fill) {
                edge_index[rec] = ei;
                bins[rec] = bn;
                weights[rec] = w;
                starts[rec + 1] = (nc + got) / 2;  // point offset after this record
            }
            ++rec;
            nc += got;
        }
        p = le + 1;
        continue;
    fallback_or_bad:
        // Python's int()/float() accept more spellings than from_chars
        // ('+1', '1_000', 'Infinity', ...): let the Python parser decide
        *err_line = line;
        return 1;
    malformed:
        *err_line = line;
        return -1;
    }
    *n_rec = rec - rec0;
    *n_c = nc - nc0;
    *n_lines = line - line0;
    return 0;
}

}  // namespace

HB_IO_API int hb_io_parse(const char *text, int64_t len, int fill, int64_t *n_records,
                          int64_t *n_coords, int64_t *edge_index, int64_t *bins, double *weights,
                          int64_t *starts, double *coords, int64_t *err_line, int64_t *err_a,
                          int64_t *err_b) {
    // line-aligned chunks parsed in parallel: a counting pass, a prefix over
    // the chunks, then a filling pass at the right offsets
    const int64_t min_chunk = 4 << 20;
    int nt = (int)std::min<int64_t>(std::max<int64_t>(1, len / min_chunk),
                                    std::max(1u, std::thread::hardware_concurrency()));
    std::vector<const char *> cut(1, text);
    for (int t = 1; t < nt; ++t) {
        const char *c = text + len * t / nt;
        if (c < cut.back()) c = cut.back();
        const char *nl = (const char *)std::memchr(c, '\n', (size_t)(text + len - c));
        cut.push_back(nl ? nl + 1 : text + len);
    }
    cut.push_back(text + len);
    nt = (int)cut.size() - 1;
    std::vector<int64_t> cr(nt), cc(nt), cl(nt), el(nt, 0), ea(nt, 0), eb(nt, 0);
    std::vector<int> rc(nt, 0);
    std::vector<int64_t> r0(nt + 1, 0), c0(nt + 1, 0), l0(nt + 1, 0);
    auto run = [&](int pass) {
        std::vector<std::thread> pool;
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                rc[t] = parse_chunk(cut[t], cut[t + 1], pass, l0[t], r0[t], c0[t], &cr[t],
                                    &cc[t], &cl[t], edge_index, bins, weights, starts, coords,
                                    &el[t], &ea[t], &eb[t]);
            });
        for (auto &th : pool) th.join();
    };
    run(0);
    // line numbers of each chunk: lines before it (error messages are global)
    for (int t = 0; t < nt; ++t) l0[t + 1] = l0[t] + cl[t];
    for (int t = 0; t < nt; ++t) {
        if (rc[t] != 0) {
            // the chunk stopped early: re-run it with its true first line
            parse_chunk(cut[t], cut[t + 1], 0, l0[t], 0, 0, &cr[t], &cc[t], &cl[t], nullptr,
                        nullptr, nullptr, nullptr, nullptr, err_line, err_a, err_b);
            return rc[t];
        }
        r0[t + 1] = r0[t] + cr[t];
        c0[t + 1] = c0[t] + cc[t];
    }
    *n_records = r0[nt];
    *n_coords = c0[nt];
    if (!fill) return 0;
    starts[0] = 0;
    run(1);
    for (int t = 0; t < nt; ++t)
        if (rc[t] != 0) return rc[t];
    return 0;
}
