// hogio.cpp -- host-side wire formats of the LUT-HOG path:
// PNM decoding straight into caller memory (pinned host buffers that feed the
// H2D copy) and the text descriptor dump of `fasthog extract`.
//
// Reference: image_io.py:50-122 (tokenizer, decode_pnm), cli.py:124-143
// (_format_value, cmd_extract).  Same acceptance rules and error classes:
//   HOGIO_EMAGIC   UnsupportedMagic   (magic not P2/P3/P5/P6)
//   HOGIO_EMAXVAL  MaxvalNot255
//   HOGIO_ETRUNC   TruncatedData      (tokens or raw payload run out)
//   HOGIO_ETOKEN   NonNumericToken    (bad or out-of-range number)
// Files are decoded channel-planar (C, H, W) uint8, as Image.planes.
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hogio.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

bool is_space(uint8_t c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// image_io.py:50-87
struct Tok {
    const uint8_t *d;
    size_t n, pos;

    void skip_space() {
        while (pos < n) {
            const uint8_t c = d[pos];
            if (is_space(c)) {
                ++pos;
            } else if (c == '#') {
                const void *nl = memchr(d + pos, '\n', n - pos);
                pos = nl ? (size_t)((const uint8_t *)nl - d) + 1 : n;
            } else {
                return;
            }
        }
    }

    // returns 0 and the token [start, end), or HOGIO_ETRUNC
    int next_token(size_t *start, size_t *end) {
        skip_space();
        if (pos >= n) return fail(HOGIO_ETRUNC, "unexpected end of file while reading tokens");
        *start = pos;
        while (pos < n && !is_space(d[pos]) && d[pos] != '#') ++pos;
        *end = pos;
        return 0;
    }

    // Python int(tok) on an ASCII token: optional sign, decimal digits,
    // underscores between digits allowed; the reference then range-checks.
    int next_int(const char *what, int64_t lo, int64_t hi, int64_t *out) {
        size_t s, e;
        if (int rc = next_token(&s, &e)) return rc;
        std::string tok((const char *)d + s, e - s);
        size_t i = 0;
        bool neg = false;
        if (i < tok.size() && (tok[i] == '+' || tok[i] == '-')) neg = tok[i++] == '-';
        int64_t v = 0;
        bool digits = false, prev_us = true, big = false;
        for (; i < tok.size(); ++i) {
            const char c = tok[i];
            if (c >= '0' && c <= '9') {
                if (v > (int64_t)1 << 40) big = true;  // far out of every range checked
                else v = v * 10 + (c - '0');
                digits = true;
                prev_us = false;
            } else if (c == '_' && !prev_us) {
                prev_us = true;
            } else {
                return fail(HOGIO_ETOKEN, std::string("bad ") + what + " token b'" + tok + "'");
            }
        }
        if (!digits || prev_us) return fail(HOGIO_ETOKEN, std::string("bad ") + what + " token b'" + tok + "'");
        if (neg) v = -v;
        if (big || v < lo || v > hi)
            return fail(HOGIO_ETOKEN, std::string(what) + " " + (big ? tok : std::to_string(v)) +
                                          " out of range [" + std::to_string(lo) + ", " + std::to_string(hi) + "]");
        *out = v;
        return 0;
    }
};

int channels_of(const uint8_t *d, size_t n, bool *ascii) {
    if (n < 2 || d[0] != 'P' || (d[1] != '2' && d[1] != '3' && d[1] != '5' && d[1] != '6')) return 0;
    *ascii = d[1] == '2' || d[1] == '3';
    return (d[1] == '2' || d[1] == '5') ? 1 : 3;
}

std::string magic_repr(const uint8_t *d, size_t n) {
    std::string s = "b'";
    for (size_t i = 0; i < std::min<size_t>(n, 2); ++i) {
        char buf[8];
        if (d[i] >= 32 && d[i] < 127 && d[i] != '\\' && d[i] != '\'') snprintf(buf, 8, "%c", d[i]);
        else snprintf(buf, 8, "\\x%02x", d[i]);
        s += buf;
    }
    return s + "'";
}

int header(const uint8_t *d, size_t n, int *c, int *h, int *w, Tok *tok, bool *ascii) {
    *c = channels_of(d, n, ascii);
    if (!*c) return fail(HOGIO_EMAGIC, "unsupported magic " + magic_repr(d, n));
    *tok = Tok{d, n, 2};
    int64_t W, H, M;
    if (int rc = tok->next_int("width", 1, (int64_t)1 << 31, &W)) return rc;
    if (int rc = tok->next_int("height", 1, (int64_t)1 << 31, &H)) return rc;
    if (int rc = tok->next_int("maxval", 1, 65535, &M)) return rc;
    if (M != 255) return fail(HOGIO_EMAXVAL, "maxval must be 255, got " + std::to_string(M));
    if (W > INT32_MAX || H > INT32_MAX) return fail(HOGIO_ETOKEN, "image too large");
    *w = (int)W;
    *h = (int)H;
    return 0;
}

// image_io.py:90-122: decode into planar out[ch * plane + y * pitch + x]
int decode(const uint8_t *d, size_t n, uint8_t *out, int64_t pitch, int64_t plane) {
    int c, h, w;
    Tok tok;
    bool ascii;
    if (int rc = header(d, n, &c, &h, &w, &tok, &ascii)) return rc;
    const int64_t count = (int64_t)w * h * c;
    if (ascii) {
        for (int64_t i = 0; i < count; ++i) {
            int64_t v;
            if (int rc = tok.next_int("sample", 0, 255, &v)) return rc;
            const int64_t px = i / c, ch = i % c;
            out[ch * plane + (px / w) * pitch + px % w] = (uint8_t)v;
        }
        return 0;
    }
    // exactly one whitespace byte separates the header from the payload
    const size_t off = tok.pos + 1;
    const int64_t have = off <= n ? (int64_t)(n - off) : 0;
    if (have < count)
        return fail(HOGIO_ETRUNC, "expected " + std::to_string(count) + " sample bytes, got " + std::to_string(have));
    const uint8_t *p = d + off;
    if (c == 1) {
        for (int y = 0; y < h; ++y) memcpy(out + (int64_t)y * pitch, p + (int64_t)y * w, (size_t)w);
    } else {  // interleaved RGB -> planar
        for (int y = 0; y < h; ++y) {
            const uint8_t *row = p + (int64_t)y * w * 3;
            uint8_t *r = out + (int64_t)y * pitch, *g = r + plane, *b = g + plane;
            for (int x = 0; x < w; ++x) {
                r[x] = row[3 * x];
                g[x] = row[3 * x + 1];
                b[x] = row[3 * x + 2];
            }
        }
    }
    return 0;
}

bool read_file(const char *path, std::vector<uint8_t> *buf, std::string *err) {
    FILE *f = fopen(path, "rb");
    if (!f) {
        *err = std::string(path) + ": " + strerror(errno);
        return false;
    }
    buf->clear();
    uint8_t tmp[1 << 16];
    size_t k;
    while ((k = fread(tmp, 1, sizeof(tmp), f)) > 0) buf->insert(buf->end(), tmp, tmp + k);
    fclose(f);
    return true;
}

// cli.py:124-127: str(int(v)) for "none", format(float(v), ".9g") otherwise
int format_value(char *dst, double v, int as_int) {
    if (as_int) return snprintf(dst, 32, "%lld", (long long)v);
    return snprintf(dst, 32, "%.9g", v);
}

}  // namespace

extern "C" {

const char *hogio_last_error(void) { return g_err.c_str(); }

int hogio_pnm_header(const uint8_t *data, size_t len, int *channels, int *height, int *width) {
    g_err.clear();
    Tok tok;
    bool ascii;
    return header(data, len, channels, height, width, &tok, &ascii);
}

int hogio_pnm_decode(const uint8_t *data, size_t len, uint8_t *out, int64_t pitch, int64_t plane_stride) {
    g_err.clear();
    return decode(data, len, out, pitch, plane_stride);
}

int hogio_decode_batch(const char *const *paths, int n, int c, int h, int w, uint8_t *out,
                       int64_t frame_stride, int64_t pitch, int64_t plane_stride, int threads,
                       int *status) {
    g_err.clear();
    if (n < 0 || c < 1 || h < 1 || w < 1 || !out || !status) return fail(HOGIO_EINVAL, "bad arguments");
    threads = std::max(1, std::min(threads, n));
    std::atomic<int> next{0};
    std::vector<std::string> errs(n);
    auto work = [&]() {
        std::vector<uint8_t> buf;
        for (int i; (i = next.fetch_add(1)) < n;) {
            std::string e;
            if (!read_file(paths[i], &buf, &e)) {
                status[i] = HOGIO_EIO;
                errs[i] = e;
                continue;
            }
            int fc, fh, fw;
            Tok tok;
            bool ascii;
            int rc = header(buf.data(), buf.size(), &fc, &fh, &fw, &tok, &ascii);
            if (!rc && (fc != c || fh != h || fw != w)) {
                rc = HOGIO_ESHAPE;
                g_err = std::string(paths[i]) + ": " + std::to_string(fc) + "x" + std::to_string(fh) + "x" +
                        std::to_string(fw) + " does not match the batch " + std::to_string(c) + "x" +
                        std::to_string(h) + "x" + std::to_string(w);
            }
            if (!rc) rc = decode(buf.data(), buf.size(), out + (int64_t)i * frame_stride, pitch, plane_stride);
            status[i] = rc;
            if (rc) errs[i] = std::string(paths[i]) + ": " + g_err;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto &t : pool) t.join();
    for (int i = 0; i < n; ++i)
        if (status[i]) return fail(status[i], errs[i]);
    return 0;
}

int64_t hogio_format_descriptors(const int32_t *xs, const int32_t *ys, const double *values, int64_t rows,
                                 int dim, int as_int, char *dst, int64_t cap) {
    g_err.clear();
    int64_t used = 0;
    char num[40];
    for (int64_t r = 0; r < rows; ++r) {
        int k = snprintf(num, sizeof(num), "%d %d", xs[r], ys[r]);
        if (dst && used + k <= cap) memcpy(dst + used, num, (size_t)k);
        used += k;
        const double *v = values + r * (int64_t)dim;
        for (int j = 0; j < dim; ++j) {
            num[0] = ' ';
            k = 1 + format_value(num + 1, v[j], as_int);
            if (dst && used + k <= cap) memcpy(dst + used, num, (size_t)k);
            used += k;
        }
        if (dst && used + 1 <= cap) dst[used] = '\n';
        used += 1;
    }
    return used;  // bytes needed; the text is complete iff used <= cap
}

}  // extern "C"
