// io.cu -- host-side graph file reader: the
// step before the hot path.  The paper reads Pajek files (`*Vertices N`,
// `*Arcs` directed, `*Edges` undirected) and SNAP edge lists
// (zero- or one-based ids).  Readings ("ingest"):
//   * Pajek: `*Vertices N` sets n and index base 1; `*Arcs` records are
//     directed; each `*Edges` record becomes two arcs u->v and v->u;
//     `%` comment lines and blank lines skipped; keywords case-insensitive;
//     tokens after the two endpoint ids (labels, weights) ignored; an id
//     outside [1, N] is a range error naming the line.
//   * edge list: `#` comment lines skipped; each other line is exactly two
//     integer ids ("u v"); index base 0 if any id is 0, else 1; n = max id -
//     base + 1.
// Malformed records fail with the line number (TC_E_INVALID).  The arc
// arrays are malloc'ed here and released with tc_free_arcs.
#include <ctype.h>
#include <errno.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <strings.h>

#include <string>
#include <vector>

#include "tc_internal.cuh"

namespace {

// Line reader over 4 MB block reads (fread), not per-character stdio calls.
struct Reader {
    FILE *f = nullptr;
    std::string line;
    uint64_t lineno = 0;
    std::vector<char> buf = std::vector<char>(4 << 20);
    size_t pos = 0, end = 0;
    bool eof = false;
    bool fill() {
        if (eof) return false;
        end = fread(buf.data(), 1, buf.size(), f);
        pos = 0;
        if (end == 0) eof = true;
        return end > 0;
    }
    bool next() {
        line.clear();
        bool any = false;
        for (;;) {
            if (pos == end && !fill()) break;
            const char *b = buf.data() + pos;
            const char *nl = (const char *)memchr(b, '\n', end - pos);
            const size_t len = nl ? (size_t)(nl - b) : end - pos;
            line.append(b, len);
            any = true;
            pos += len;
            if (nl) {
                pos++;   // the newline
                break;
            }
        }
        if (!any) return false;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        lineno++;
        return true;
    }
    void rewind_file() {
        rewind(f);
        pos = end = 0;
        eof = false;
        lineno = 0;
    }
};

const char *skip_ws(const char *p) {
    while (*p && isspace((unsigned char)*p)) p++;
    return p;
}

// parse one unsigned integer token; returns false if not an integer token
bool parse_u64(const char *&p, uint64_t &out) {
    p = skip_ws(p);
    if (!isdigit((unsigned char)*p)) return false;
    errno = 0;
    char *end = nullptr;
    unsigned long long v = strtoull(p, &end, 10);
    if (errno || (end && *end && !isspace((unsigned char)*end))) return false;
    out = v;
    p = end;
    return true;
}

tc_status finish(std::vector<uint32_t> &s, std::vector<uint32_t> &d, uint64_t n, uint64_t *n_out,
                 uint32_t **src, uint32_t **dst, uint64_t *m) {
    const size_t k = s.size();
    *src = (uint32_t *)malloc((k ? k : 1) * sizeof(uint32_t));
    *dst = (uint32_t *)malloc((k ? k : 1) * sizeof(uint32_t));
    if (!*src || !*dst) {
        free(*src);
        free(*dst);
        *src = *dst = nullptr;
        tc::set_error("host allocation of %zu arcs failed", k);
        return TC_E_OOM;
    }
    if (k) {
        memcpy(*src, s.data(), k * sizeof(uint32_t));
        memcpy(*dst, d.data(), k * sizeof(uint32_t));
    }
    *m = k;
    *n_out = n;
    return TC_OK;
}

tc_status read_pajek(Reader &r, uint64_t *n_out, uint32_t **src, uint32_t **dst, uint64_t *m) {
    enum { NONE, VERT, ARCS, EDGES } sec = NONE;
    uint64_t n = 0;
    bool have_n = false;
    std::vector<uint32_t> s, d;
    while (r.next()) {
        const char *p = skip_ws(r.line.c_str());
        if (!*p || *p == '%') continue;
        if (*p == '*') {
            const char *kw = p + 1;
            if (!strncasecmp(kw, "vertices", 8)) {
                const char *q = kw + 8;
                if (!parse_u64(q, n) || n >= (1ull << 30)) {
                    tc::set_error("line %llu: bad *Vertices count", (unsigned long long)r.lineno);
                    return TC_E_INVALID;
                }
                have_n = true;
                sec = VERT;
            } else if (!strncasecmp(kw, "arcslist", 8) || !strncasecmp(kw, "edgeslist", 9)) {
                tc::set_error("line %llu: *Arcslist/*Edgeslist sections are not supported",
                              (unsigned long long)r.lineno);
                return TC_E_INVALID;
            } else if (!strncasecmp(kw, "arcs", 4)) {
                sec = ARCS;
            } else if (!strncasecmp(kw, "edges", 5)) {
                sec = EDGES;
            } else {
                tc::set_error("line %llu: unknown section '%s'", (unsigned long long)r.lineno, p);
                return TC_E_INVALID;
            }
            continue;
        }
        if (sec == VERT || sec == NONE) continue;   // vertex label lines
        uint64_t a, b;
        const char *q = p;
        if (!parse_u64(q, a) || !parse_u64(q, b)) {
            tc::set_error("line %llu: malformed record '%s'", (unsigned long long)r.lineno, p);
            return TC_E_INVALID;
        }
        if (!have_n || a < 1 || b < 1 || a > n || b > n) {
            tc::set_error("line %llu: vertex id outside [1, %llu]", (unsigned long long)r.lineno,
                          (unsigned long long)n);
            return TC_E_RANGE;
        }
        s.push_back((uint32_t)(a - 1));
        d.push_back((uint32_t)(b - 1));
        if (sec == EDGES) {
            s.push_back((uint32_t)(b - 1));
            d.push_back((uint32_t)(a - 1));
        }
    }
    if (!have_n) {
        tc::set_error("no *Vertices line: n unknown");
        return TC_E_INVALID;
    }
    return finish(s, d, n, n_out, src, dst, m);
}

tc_status read_edgelist(Reader &r, int base, uint64_t *n_out, uint32_t **src, uint32_t **dst,
                        uint64_t *m) {
    std::vector<uint64_t> a, b;
    uint64_t mx = 0;
    bool zero = false;
    while (r.next()) {
        const char *p = skip_ws(r.line.c_str());
        if (!*p || *p == '#' || *p == '%') continue;
        uint64_t x, y;
        const char *q = p;
        if (!parse_u64(q, x) || !parse_u64(q, y) || *skip_ws(q)) {
            tc::set_error("line %llu: expected exactly two integer ids, got '%s'",
                          (unsigned long long)r.lineno, p);
            return TC_E_INVALID;
        }
        zero |= (x == 0 || y == 0);
        mx = x > mx ? x : mx;
        mx = y > mx ? y : mx;
        a.push_back(x);
        b.push_back(y);
    }
    if (a.empty()) {
        tc::set_error("empty edge list: n unknown");
        return TC_E_INVALID;
    }
    if (base < 0) base = zero ? 0 : 1;
    if (base == 1 && zero) {
        tc::set_error("id 0 in a one-based edge list");
        return TC_E_RANGE;
    }
    const uint64_t n = mx - (uint64_t)base + 1;
    if (n >= (1ull << 30)) {
        tc::set_error("n = %llu must be < 2^30", (unsigned long long)n);
        return TC_E_INVALID;
    }
    std::vector<uint32_t> s(a.size()), d(a.size());
    for (size_t i = 0; i < a.size(); i++) {
        s[i] = (uint32_t)(a[i] - base);
        d[i] = (uint32_t)(b[i] - base);
    }
    return finish(s, d, n, n_out, src, dst, m);
}

}  // namespace

extern "C" {

tc_status tc_read_arcs(const char *path, int format, int index_base, uint64_t *n, uint32_t **src,
                       uint32_t **dst, uint64_t *m) {
    if (!path || !n || !src || !dst || !m || index_base < -1 || index_base > 1) {
        tc::set_error("invalid arguments");
        return TC_E_INVALID;
    }
    *src = *dst = nullptr;
    Reader r;
    r.f = fopen(path, "rb");
    if (!r.f) {
        tc::set_error("cannot open '%s': %s", path, strerror(errno));
        return TC_E_INVALID;
    }
    if (format == 0) {   // auto: Pajek if the first non-comment line is a section
        format = 2;
        while (r.next()) {
            const char *p = skip_ws(r.line.c_str());
            if (!*p || *p == '%' || *p == '#') continue;
            format = (*p == '*') ? 1 : 2;
            break;
        }
        r.rewind_file();
    }
    tc_status st = format == 1 ? read_pajek(r, n, src, dst, m)
                               : read_edgelist(r, index_base, n, src, dst, m);
    fclose(r.f);
    return st;
}

void tc_free_arcs(uint32_t *p) { free(p); }

}  // extern "C"
