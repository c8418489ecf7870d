// mtx.cpp — parallel MatrixMarket coordinate ingest.
//
// Same language as the reference's parse_matrix_market (graph.hpp:111-199):
// banner "%%MatrixMarket matrix coordinate <pattern|real|integer>
// <general|symmetric>" (case-insensitive), then the first non-blank,
// non-comment line is "rows cols entries", then `entries` entry lines
// "row col[ weight]" (1-based; weights validated with from_chars, discarded);
// each yields the edge row-1 -> col-1 and, when symmetric and off-diagonal,
// the reverse.  Blank and '%' lines are skipped; lines after the last entry
// are never looked at; the first error in file order is reported with its
// 1-based line number and the reference's message.
//
// The body is split into byte ranges at line boundaries, one per thread.
// Pass 1 parses every range into its own buffer, counting lines, entries and
// pairs, and records the range's first error (with its entry index: an error
// after the `entries`-th entry is never read by the reference); pass 2 copies
// every range's pairs to its prefix offset.  Host-only code (no CUDA), so it
// runs anywhere.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "mtx.h"

namespace prgpu {
namespace {

inline std::string_view trim(std::string_view s) {
    while (!s.empty() && (s.back() == '\r' || s.back() == ' ' || s.back() == '\t')) s.remove_suffix(1);
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
    return s;
}

// up to `cap` whitespace-separated fields; returns the true field count
inline int fields(std::string_view line, std::string_view* out, int cap) {
    int k = 0;
    size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i;
        const size_t st = i;
        while (i < line.size() && line[i] != ' ' && line[i] != '\t') ++i;
        if (i > st) {
            if (k < cap) out[k] = line.substr(st, i - st);
            ++k;
        }
    }
    return k;
}

inline bool to_u64(std::string_view t, uint64_t& v) {
    auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    return ec == std::errc{} && p == t.data() + t.size();
}

inline bool to_f64(std::string_view t, double& v) {
    auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    return ec == std::errc{} && p == t.data() + t.size();
}

std::string lowered(std::string_view s) {
    std::string o(s);
    for (char& c : o) c = (char)std::tolower((unsigned char)c);
    return o;
}

// one body line; returns 0 skip, 1 entry (pairs in p, count in np), -1 error
inline int parse_entry(std::string_view raw, bool weighted, bool sym, uint64_t rows, uint64_t cols,
                       uint32_t* p, int& np, std::string* what) {
    const std::string_view body = trim(raw);
    if (body.empty() || body.front() == '%') return 0;
    std::string_view f[3];
    const int nf = fields(body, f, 3);
    const int expect = weighted ? 3 : 2;
    if (nf != expect) {
        if (what) *what = "expected " + std::to_string(expect) + " fields, got " + std::to_string(nf);
        return -1;
    }
    uint64_t r = 0, c = 0;
    if (!to_u64(f[0], r) || !to_u64(f[1], c)) {
        if (what) *what = "entry indices must be integers";
        return -1;
    }
    if (r < 1 || r > rows || c < 1 || c > cols) {
        if (what)
            *what = "entry (" + std::to_string(r) + ", " + std::to_string(c) + ") out of range for " +
                    std::to_string(rows) + " x " + std::to_string(cols);
        return -1;
    }
    if (weighted) {
        double w = 0;
        if (!to_f64(f[2], w)) {
            if (what) *what = "entry weight is not a number";
            return -1;
        }
    }
    const uint32_t s = (uint32_t)(r - 1), d = (uint32_t)(c - 1);
    p[0] = s;
    p[1] = d;
    np = 1;
    if (sym && s != d) {
        p[2] = d;
        p[3] = s;
        np = 2;
    }
    return 1;
}

struct Range {
    const char* b;
    const char* e;
    uint64_t lines = 0, entries = 0, pairs = 0;
    uint64_t err_entry = UINT64_MAX; // entries seen before the erroneous line
    uint64_t err_line = 0;           // local 1-based line of the first error
    std::string err_what;
};

// visit the lines of [b, e): fn(line) per line (a last line without '\n' counts)
template <class F>
inline void for_lines(const char* b, const char* e, F&& fn) {
    const char* p = b;
    while (p < e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(e - p)));
        const char* end = nl ? nl : e;
        if (!fn(std::string_view(p, (size_t)(end - p)))) return;
        p = nl ? nl + 1 : e;
    }
}

} // namespace

MtxResult mtx_parse(const char* text, uint64_t len, int threads) {
    MtxResult R;
    const char* const end = text + len;
    const char* p = text;
    uint64_t ln = 0;
    auto next_line = [&](std::string_view& out) -> bool {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
        const char* e = nl ? nl : end;
        out = std::string_view(p, (size_t)(e - p));
        p = nl ? nl + 1 : end;
        ++ln;
        return true;
    };
    auto fail = [&](uint64_t line, std::string what) {
        R.err_line = line;
        R.err_what = std::move(what);
        return R;
    };
    std::string_view line;
    if (!next_line(line)) return fail(1, "empty input, no banner");
    {
        std::string_view f[6];
        const int nf = fields(trim(line), f, 6);
        if (nf != 5 || f[0] != "%%MatrixMarket") return fail(ln, "malformed MatrixMarket banner");
        const std::string obj = lowered(f[1]), fmt = lowered(f[2]), fld = lowered(f[3]), sym = lowered(f[4]);
        if (obj != "matrix") return fail(ln, "unsupported object '" + obj + "' (want matrix)");
        if (fmt != "coordinate") return fail(ln, "unsupported format '" + fmt + "' (want coordinate)");
        if (fld != "pattern" && fld != "real" && fld != "integer")
            return fail(ln, "unsupported field '" + fld + "' (want pattern, real or integer)");
        if (sym != "general" && sym != "symmetric")
            return fail(ln, "unsupported symmetry '" + sym + "' (want general or symmetric)");
        R.symmetric = sym == "symmetric";
        R.weighted = fld != "pattern";
    }
    uint64_t rows = 0, cols = 0, entries = 0;
    for (;;) {
        if (!next_line(line)) return fail(ln + 1, "unexpected end of file before size line");
        const std::string_view b = trim(line);
        if (b.empty() || b.front() == '%') continue;
        std::string_view f[4];
        if (fields(b, f, 4) != 3 || !to_u64(f[0], rows) || !to_u64(f[1], cols) || !to_u64(f[2], entries))
            return fail(ln, "size line must be three integers (rows cols entries)");
        break;
    }
    const uint64_t n = std::max(rows, cols);
    if (n == 0) return fail(ln, "graph has no vertices");
    if (n > UINT32_MAX) return fail(ln, "vertex count exceeds 2^32-1");
    R.n = (uint32_t)n;
    if (entries == 0) return R;

    // ---- body: ranges at line boundaries --------------------------------------------
    const uint64_t body_len = (uint64_t)(end - p);
    // threads <= 0: every core, but no range under 64 KiB; an explicit count
    // is taken as given (tests split tiny inputs into many ranges)
    int T = threads;
    if (T <= 0) {
        T = (int)std::max(1u, std::thread::hardware_concurrency());
        T = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)T, body_len / (1u << 16) + 1));
    }
    std::vector<Range> rg(T);
    {
        const char* s = p;
        for (int t = 0; t < T; ++t) {
            const char* e = (t == T - 1) ? end : p + body_len * (uint64_t)(t + 1) / (uint64_t)T;
            if (e < s) e = s;
            if (t < T - 1 && e < end) { // extend to just past the next newline
                const char* nl = static_cast<const char*>(std::memchr(e, '\n', (size_t)(end - e)));
                e = nl ? nl + 1 : end;
            }
            rg[t].b = s;
            rg[t].e = e;
            s = e;
        }
    }
    const bool w = R.weighted, sy = R.symmetric;
    auto run = [&](auto&& body) {
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(body, t);
        body(0);
        for (auto& th : pool) th.join();
    };
    // pass 1: every range parses its lines into its own pair buffer and
    // records its first error
    std::vector<std::vector<uint32_t>> buf(T);
    run([&](int t) {
        Range& r = rg[t];
        std::vector<uint32_t>& out = buf[t];
        out.reserve((size_t)((r.e - r.b) / 6 + 16) * (sy ? 4 : 2));
        uint32_t pr[4];
        int np = 0;
        for_lines(r.b, r.e, [&](std::string_view l) {
            ++r.lines;
            const int k = parse_entry(l, w, sy, rows, cols, pr, np, nullptr);
            if (k > 0) {
                ++r.entries;
                r.pairs += (uint64_t)np;
                out.insert(out.end(), pr, pr + 2 * np);
            } else if (k < 0) {
                std::string what;
                parse_entry(l, w, sy, rows, cols, pr, np, &what);
                r.err_entry = r.entries;
                r.err_line = r.lines;
                r.err_what = std::move(what);
                return false;
            }
            return true;
        });
    });
    // the reference reads entries in order and stops after `entries` of them
    uint64_t e_before = 0, l_before = 0;
    int last = -1;     // range holding the `entries`-th entry
    uint64_t take = 0; // entries taken from it
    for (int t = 0; t < T; ++t) {
        const Range& r = rg[t];
        if (r.err_line && e_before + r.err_entry < entries)
            return fail(ln + l_before + r.err_line, r.err_what);
        if (e_before + r.entries >= entries) { // (an error further on is never read)
            last = t;
            take = entries - e_before;
            break;
        }
        e_before += r.entries;
        l_before += r.lines;
    }
    if (last < 0)
        return fail(ln + l_before + 1, "unexpected end of file: got " + std::to_string(e_before) + " of " +
                                           std::to_string(entries) + " entries");
    // pairs of the first `take` entries of the last range
    uint64_t last_pairs = rg[last].pairs;
    if (take < rg[last].entries) {
        if (!sy) last_pairs = take;
        else {
            last_pairs = 0;
            uint64_t seen = 0;
            uint32_t pr[4];
            int np = 0;
            for_lines(rg[last].b, rg[last].e, [&](std::string_view l) {
                if (seen == take) return false;
                if (parse_entry(l, w, sy, rows, cols, pr, np, nullptr) > 0) {
                    ++seen;
                    last_pairs += (uint64_t)np;
                }
                return true;
            });
        }
    }
    std::vector<uint64_t> off(last + 2, 0);
    for (int t = 0; t < last; ++t) off[t + 1] = off[t] + rg[t].pairs;
    off[last + 1] = off[last] + last_pairs;
    R.m = off[last + 1];
    R.pairs = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(R.m, 1) * 2 * sizeof(uint32_t)));
    if (!R.pairs) return fail(0, "out of host memory");
    // pass 2: each range's pairs to its prefix offset
    run([&](int t) {
        if (t > last) return;
        const uint64_t np = off[t + 1] - off[t];
        if (np) std::memcpy(R.pairs + 2 * off[t], buf[t].data(), np * 2 * sizeof(uint32_t));
        std::vector<uint32_t>().swap(buf[t]);
    });
    return R;
}

} // namespace prgpu
