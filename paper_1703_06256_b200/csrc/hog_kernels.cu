// hog_kernels.cu -- sm_100a kernels + C ABI for the LUT-HOG hot path.
//
// Reference: /root/reference/pkg/src/fasthog (pure Python + NumPy).  The hot
// path is gradient.py:95-121 (LUT binning), integral.py:58-87 (per-bin
// summed-area tables), descriptor.py:162-195 (cell histograms from 4 corner
// reads) and detector.py:140-154 / 202-221 (scores, pyramid resize).
//
// Design (DESIGN.md has the roofline numbers):
//   The integral planes (4*N_b bytes per pixel) are ~90% of the compulsory
//   HBM traffic, so every plane element is written exactly once, with
//   16-byte coalesced stores, by k_planes.  Each warp owns a tile of R plane
//   rows x Ws columns (4 columns per lane) and walks down it: the row prefix
//   is a warp scan over one-hot counts packed two bins per 32-bit word
//   (16-bit lanes; a row prefix never exceeds the width), the column prefix
//   lives in registers.  The carries a tile needs -- the row prefix left of
//   its strip, and the plane row above its band -- come from per-tile bin
//   counts that k_grad_bin emits while it bins the image, scanned by three
//   tiny kernels (k_scan_cols / k_scan_rows / k_scan_tiles).  When the scan
//   lattice is regular, k_planes also emits the cell-histogram grid from the
//   plane values it holds in registers (4-corner formula, descriptor.py:
//   176-185), so the planes are never re-read.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/hogb200.h"

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LUT_SIDE = 511;
constexpr int K_THREADS = 128;          // 4 independent warps per CTA
constexpr int MAX_FUSED_BINS = 18;      // NW <= 9 packed words

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(HOG_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return HOG_OK;
}

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// Tile geometry shared by k_grad_bin / k_bin_counts / scans / k_planes.
struct TileGeom {
    int n, h, w, bins;
    int R;     // plane/pixel rows per band (multiple of the lattice step when fused)
    int Ws;    // columns per strip (<= 128, multiple of 8)
    int ns;    // strips per frame
    int nb1;   // pixel bands: ceil(h / R)
    int nb2;   // plane bands: h / R + 1   (plane rows 0..h)
    int Wc;    // ns * Ws  (padded width of the per-column scratch arrays)
    int NWB;   // u8-packed words per column count  = ceil(bins / 4)
    int NW;    // u16-packed words per row count    = ceil(bins / 2)
    int NWp;   // NW padded to a multiple of 4 (16-byte rows)
    int NBp4;  // bins padded to a multiple of 4 (int32 tile carries)
};

// Scratch arrays (device), carved from the caller's scratch buffer.
struct Scratch {
    uint32_t *C;   // [n][nb1][Wc][NWB]   per-band column counts, u8 x4 packed
    uint32_t *S;   // [n][ns][h][NWp]     per-strip row counts, u16 x2 packed
    uint32_t *tt;  // [n][nb1][ns][NWp]   per-tile totals, u16 x2 packed
    uint32_t *V;   // [n][nb2][Wc][NWp]   column counts above each band, u16 x2
    uint32_t *L;   // [n][ns][h][NWp]     row counts left of each strip, u16 x2
    int32_t *T;    // [n][nb2][ns][NBp4]  count in [0,band top) x [0,strip left)
};

TileGeom make_geom(int n, int h, int w, int bins, bool fused, int stride, int cell) {
    TileGeom g{};
    g.n = n; g.h = h; g.w = w; g.bins = bins;
    if (fused) {
        int a = 8, b = stride;
        while (b) { int r = a % b; a = b; b = r; }
        const int l = 8 / a * stride;  // lcm(8, stride): strips start on lattice columns, 32-B aligned
        g.Ws = ((128 + stride - cell) / l) * l;
    } else {
        g.Ws = 128;
    }
    g.ns = (int)((w + g.Ws - 1) / g.Ws);
    g.Wc = g.ns * g.Ws;
    int R = 128;
    auto tiles = [&](int r) { return (int64_t)n * (h / r + 1) * g.ns; };
    while (R > 16 && tiles(R) < 148 * 64) R /= 2;
    if (fused && R % stride != 0) R = (int)round_up(R, stride);
    g.R = R;
    g.nb1 = (h + R - 1) / R;
    g.nb2 = h / R + 1;
    g.NWB = (bins + 3) / 4;
    g.NW = (bins + 1) / 2;
    g.NWp = (int)round_up(g.NW, 4);
    g.NBp4 = (int)round_up(bins, 4);
    return g;
}

size_t carve(const TileGeom &g, void *base, Scratch *sc) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += round_up((int64_t)bytes, 256);
        return o;
    };
    size_t oC = take(sizeof(uint32_t) * (size_t)g.n * g.nb1 * g.Wc * g.NWB);
    size_t oS = take(sizeof(uint32_t) * (size_t)g.n * g.ns * g.h * g.NWp);
    size_t ot = take(sizeof(uint32_t) * (size_t)g.n * g.nb1 * g.ns * g.NWp);
    size_t oV = take(sizeof(uint32_t) * (size_t)g.n * g.nb2 * g.Wc * g.NWp);
    size_t oL = take(sizeof(uint32_t) * (size_t)g.n * g.ns * g.h * g.NWp);
    size_t oT = take(sizeof(int32_t) * (size_t)g.n * g.nb2 * g.ns * g.NBp4);
    if (sc && base) {
        char *b = (char *)base;
        sc->C = (uint32_t *)(b + oC);
        sc->S = (uint32_t *)(b + oS);
        sc->tt = (uint32_t *)(b + ot);
        sc->V = (uint32_t *)(b + oV);
        sc->L = (uint32_t *)(b + oL);
        sc->T = (int32_t *)(b + oT);
    }
    return off;
}

// ---------------------------------------------------------------------------
// Device helpers

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t t = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}

// one-hot of bin `b` in the u16x2-packed word `w` (bins 2w, 2w+1); NO_BIN
// (0xFF) and out-of-range values hit no word.
__device__ __forceinline__ uint32_t oh16(uint32_t hb, uint32_t one, int w) {
    return hb == (uint32_t)w ? one : 0u;
}

__device__ __forceinline__ uint32_t byte_of(uint32_t v, int k) { return (v >> (8 * k)) & 0xffu; }

// u8x4 word -> u16x2 word holding bytes (2h, 2h+1)
__device__ __forceinline__ uint32_t widen_half(uint32_t v, int h) {
    return h == 0 ? __byte_perm(v, 0u, 0x4140) : __byte_perm(v, 0u, 0x4342);
}

__device__ __forceinline__ uint32_t half16(uint32_t v, int h) {
    return h == 0 ? (v & 0xffffu) : (v >> 16);
}

struct TileId {
    int f, b, s;
};

__device__ __forceinline__ bool decode_tile(const TileGeom &g, int nbands, TileId &t) {
    const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t ntiles = (int64_t)g.n * nbands * g.ns;
    if (wid >= ntiles) return false;
    t.s = (int)(wid % g.ns);
    const int64_t q = wid / g.ns;
    t.b = (int)(q % nbands);
    t.f = (int)(q / nbands);
    return true;
}

// Accumulates one row of bins (4 bytes per lane, 0xFF = none) into the
// per-lane column counts (u8x4 packed) and returns the lane's row count
// (u16x2 packed words), bins < 2*NW.
template <int NWB, int NW>
__device__ __forceinline__ void count_row(uint32_t bins4, uint32_t (&cc)[4][NWB],
                                          uint32_t (&rc)[NW]) {
#pragma unroll
    for (int w = 0; w < NW; ++w) rc[w] = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t v = byte_of(bins4, k);
        uint32_t q8 = v >> 2, one8 = 1u << ((v & 3u) << 3);
        uint32_t q16 = v >> 1, one16 = 1u << ((v & 1u) << 4);
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] += (q8 == (uint32_t)w) ? one8 : 0u;
#pragma unroll
        for (int w = 0; w < NW; ++w) rc[w] += (q16 == (uint32_t)w) ? one16 : 0u;
    }
}

// Per-row / per-band count outputs shared by both count producers.
template <int NWB, int NW>
__device__ __forceinline__ void emit_row_counts(const TileGeom &g, const Scratch &sc,
                                                const TileId &t, int y, int lane,
                                                uint32_t (&rc)[NW], uint32_t (&tt)[NW]) {
    uint32_t mine = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        uint32_t tot = warp_sum(rc[w]);
        tt[w] += tot;
        if (lane == w) mine = tot;
    }
    if (lane < g.NWp)
        sc.S[(((int64_t)t.f * g.ns + t.s) * g.h + y) * g.NWp + lane] = lane < NW ? mine : 0u;
}

template <int NWB, int NW>
__device__ __forceinline__ void emit_band_counts(const TileGeom &g, const Scratch &sc,
                                                 const TileId &t, int x, int lane, bool own,
                                                 uint32_t (&cc)[4][NWB], uint32_t (&tt)[NW]) {
    if (own) {
        uint32_t *cp = sc.C + (((int64_t)t.f * g.nb1 + t.b) * g.Wc + x) * NWB;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int w = 0; w < NWB; ++w) cp[k * NWB + w] = cc[k][w];
    }
    uint32_t mine = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w)
        if (lane == w) mine = tt[w];
    if (lane < g.NWp)
        sc.tt[(((int64_t)t.f * g.nb1 + t.b) * g.ns + t.s) * g.NWp + lane] = lane < NW ? mine : 0u;
}

// ---------------------------------------------------------------------------
// K1: gradient + LUT binning (gradient.py:95-121), optionally emitting the
// per-tile counts the plane kernel needs.  One warp = one tile of R rows x
// Ws columns; lane L owns pixel columns xs+4L .. xs+4L+3 and slides a
// three-row window down the band (each image row is loaded once per tile,
// left/right neighbours come from adjacent lanes by shuffle).

template <int CH, int NWB, int NW, bool COUNTS>
__global__ void __launch_bounds__(K_THREADS)
k_grad_bin(const uint8_t *__restrict__ img, int64_t ip, int64_t ics, int64_t ifs,
           const uint8_t *__restrict__ lut, int8_t *__restrict__ bm, int64_t bp, int64_t bfs,
           TileGeom g, Scratch sc) {
    TileId t;
    if (!decode_tile(g, g.nb1, t)) return;
    const int lane = threadIdx.x & 31;
    const int xs = t.s * g.Ws;
    const int x = xs + 4 * lane;
    const bool own = 4 * lane < g.Ws;
    const bool inx = x < g.w;
    const int y0 = t.b * g.R, y1 = min(y0 + g.R, g.h);
    const uint8_t *im = img + (int64_t)t.f * ifs;
    int8_t *bmf = bm + (int64_t)t.f * bfs;

    auto ldw = [&](int y, int ch) -> uint32_t {
        return (inx && y >= 0 && y < g.h)
                   ? __ldg(reinterpret_cast<const uint32_t *>(im + ch * ics + (int64_t)y * ip + x))
                   : 0u;
    };
    auto ldb = [&](int y, int ch, int xx) -> uint32_t {
        return (xx >= 0 && xx < g.w && y >= 0 && y < g.h) ? (uint32_t)__ldg(im + ch * ics + (int64_t)y * ip + xx)
                                                          : 0u;
    };

    uint32_t up[CH], mid[CH], dn[CH], ml[CH], mr[CH], dl[CH], dr[CH];
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
        up[ch] = ldw(y0 - 1, ch);
        mid[ch] = ldw(y0, ch);
        ml[ch] = lane == 0 ? ldb(y0, ch, x - 1) : 0u;
        mr[ch] = lane == 31 ? ldb(y0, ch, x + 4) : 0u;
    }
    uint32_t cc[4][NWB];
    uint32_t tt[NW];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) tt[w] = 0;

    for (int y = y0; y < y1; ++y) {
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            dn[ch] = ldw(y + 1, ch);
            dl[ch] = lane == 0 ? ldb(y + 1, ch, x - 1) : 0u;
            dr[ch] = lane == 31 ? ldb(y + 1, ch, x + 4) : 0u;
        }
        uint32_t bins4 = 0xffffffffu;
        if (y > 0 && y < g.h - 1) {
            int bdx[4], bdy[4], best[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) best[k] = -1, bdx[k] = 0, bdy[k] = 0;
#pragma unroll
            for (int ch = 0; ch < CH; ++ch) {
                uint32_t prev3 = __shfl_up_sync(FULL, mid[ch], 1) >> 24;
                uint32_t next0 = __shfl_down_sync(FULL, mid[ch], 1) & 0xffu;
                uint32_t lft = lane == 0 ? ml[ch] : prev3;
                uint32_t rgt = lane == 31 ? mr[ch] : next0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    int L = (int)(k == 0 ? lft : byte_of(mid[ch], k - 1));
                    int Rr = (int)(k == 3 ? rgt : byte_of(mid[ch], k + 1));
                    int dx = Rr - L;
                    int dy = (int)byte_of(dn[ch], k) - (int)byte_of(up[ch], k);
                    int mag = dx * dx + dy * dy;
                    if (mag > best[k]) best[k] = mag, bdx[k] = dx, bdy[k] = dy;  // first max wins
                }
            }
            bins4 = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int xk = x + k;
                uint32_t v = 0xffu;
                if (xk > 0 && xk < g.w - 1) v = __ldg(lut + (bdx[k] + 255) * LUT_SIDE + (bdy[k] + 255));
                bins4 |= v << (8 * k);
            }
        }
        if (inx) {
            // bytes past w are padding; keep them NO_BIN
            if (x + 4 > g.w) bins4 |= 0xffffffffu << (8 * (g.w - x));
            if (own) *reinterpret_cast<uint32_t *>(bmf + (int64_t)y * bp + x) = bins4;
        }
        if (COUNTS) {
            uint32_t cb = (own && inx) ? bins4 : 0xffffffffu;
            uint32_t rc[NW];
            count_row<NWB, NW>(cb, cc, rc);
            emit_row_counts<NWB, NW>(g, sc, t, y, lane, rc, tt);
        }
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            up[ch] = mid[ch];
            mid[ch] = dn[ch];
            ml[ch] = dl[ch];
            mr[ch] = dr[ch];
        }
    }
    if (COUNTS) emit_band_counts<NWB, NW>(g, sc, t, x, lane, own, cc, tt);
}

// K1': the same per-tile counts from an existing bin map (hog_integral).
template <int NWB, int NW>
__global__ void __launch_bounds__(K_THREADS)
k_bin_counts(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, TileGeom g, Scratch sc) {
    TileId t;
    if (!decode_tile(g, g.nb1, t)) return;
    const int lane = threadIdx.x & 31;
    const int x = t.s * g.Ws + 4 * lane;
    const bool own = 4 * lane < g.Ws;
    const bool inx = x < g.w;
    const int y0 = t.b * g.R, y1 = min(y0 + g.R, g.h);
    const int8_t *bmf = bm + (int64_t)t.f * bfs;
    uint32_t cc[4][NWB];
    uint32_t tt[NW];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) tt[w] = 0;
    for (int y = y0; y < y1; ++y) {
        uint32_t v = 0xffffffffu;
        if (own && inx) {
            v = __ldg(reinterpret_cast<const uint32_t *>(bmf + (int64_t)y * bp + x));
            if (x + 4 > g.w) v |= 0xffffffffu << (8 * (g.w - x));
        }
        uint32_t rc[NW];
        count_row<NWB, NW>(v, cc, rc);
        emit_row_counts<NWB, NW>(g, sc, t, y, lane, rc, tt);
    }
    emit_band_counts<NWB, NW>(g, sc, t, x, lane, own, cc, tt);
}

// ---------------------------------------------------------------------------
// Carry scans (tiny: O(N_b / R + N_b / Ws) words per pixel).

// V[f][b][x] = sum over bands b' < b of C[f][b'][x]  (column counts above band b)
template <int NWB, int NW>
__global__ void k_scan_cols(TileGeom g, Scratch sc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)g.n * g.Wc) return;
    const int f = (int)(i / g.Wc), x = (int)(i % g.Wc);
    uint32_t run[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) run[w] = 0;
    for (int b = 0; b < g.nb2; ++b) {
        uint32_t *vp = sc.V + (((int64_t)f * g.nb2 + b) * g.Wc + x) * g.NWp;
#pragma unroll
        for (int w = 0; w < NW; ++w) vp[w] = run[w];
        for (int w = NW; w < g.NWp; ++w) vp[w] = 0;
        if (b < g.nb1) {
            const uint32_t *cp = sc.C + (((int64_t)f * g.nb1 + b) * g.Wc + x) * NWB;
            uint32_t c8[NWB];
#pragma unroll
            for (int w = 0; w < NWB; ++w) c8[w] = cp[w];
#pragma unroll
            for (int w = 0; w < NW; ++w) run[w] += widen_half(c8[w >> 1], w & 1);
        }
    }
}

// L[f][s][y] = sum over strips s' < s of S[f][s'][y]  (row counts left of strip s)
template <int NW>
__global__ void k_scan_rows(TileGeom g, Scratch sc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)g.n * g.h) return;
    const int f = (int)(i / g.h), y = (int)(i % g.h);
    uint32_t run[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) run[w] = 0;
    for (int s = 0; s < g.ns; ++s) {
        const int64_t o = (((int64_t)f * g.ns + s) * g.h + y) * g.NWp;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            uint32_t v = sc.S[o + w];
            sc.L[o + w] = run[w];
            run[w] += v;
        }
        for (int w = NW; w < g.NWp; ++w) sc.L[o + w] = 0;
    }
}

// T[f][b][s][n] = count of bin n in plane rows [0, b*R) x columns [0, s*Ws)
__global__ void k_scan_tiles(TileGeom g, Scratch sc) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)g.n * g.ns * g.NBp4) return;
    const int n = (int)(i % g.NBp4);
    const int s = (int)((i / g.NBp4) % g.ns);
    const int f = (int)(i / ((int64_t)g.NBp4 * g.ns));
    uint32_t acc = 0;
    for (int b = 0; b < g.nb2; ++b) {
        sc.T[(((int64_t)f * g.nb2 + b) * g.ns + s) * g.NBp4 + n] = n < g.bins ? (int32_t)acc : 0;
        if (b < g.nb1 && n < g.bins) {
            const uint32_t *tp = sc.tt + (((int64_t)f * g.nb1 + b) * g.ns) * g.NWp + (n >> 1);
            for (int q = 0; q < s; ++q) acc += half16(tp[(int64_t)q * g.NWp], n & 1);
        }
    }
}

// ---------------------------------------------------------------------------
// K2: integral planes (+ fused cell grid).  integral.py:58-87,
// descriptor.py:176-185.  KR = cell / lattice step (0: no grid).
//
// Lane L holds P(Y, X) for X = xs+4L+1 .. xs+4L+4 and all bins in registers
// (acc), plus P(Y, xs) in pedge.  Going from plane row Y to Y+1 adds the row
// prefix R(Y, X) = L(Y) + (warp-exclusive count) + (lane-local count).
// Lattice row Yl (Yl % s == 0): Hd(Yl, xi) = P(Yl, xi + cell) - P(Yl, xi)
// is formed by shuffles, and the cell with top-left (Yl - cell, xi) is
// Hd(Yl) - Hd(Yl - cell), kept in a KR-deep ring.

struct PlaneOut {
    int32_t *pl;
    int64_t pp, pns, pfs;
    int vec;
};

struct GridOut {
    int32_t *grid;
    int s, cell, ncx, ncy;
};

template <int NW, int KR>
__global__ void __launch_bounds__(K_THREADS)
k_planes(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, PlaneOut po, GridOut go,
         TileGeom g, Scratch sc) {
    TileId t;
    if (!decode_tile(g, g.nb2, t)) return;
    const int lane = threadIdx.x & 31;
    const int xs = t.s * g.Ws;
    const int x = xs + 4 * lane;  // pixel column of this lane's first column; P column x+1
    const bool own = 4 * lane < g.Ws;
    const int X0 = x + 1;
    const int Y0 = t.b * g.R;
    const int Ystore = min(Y0 + g.R - 1, g.h);
    int Ycomp = Ystore;
    if (KR) Ycomp = max(Ystore, min(Y0 + g.R - go.s + go.cell, g.h));
    const bool st = own && X0 <= g.w;
    const int bins = g.bins;
    const int8_t *bmf = bm + (int64_t)t.f * bfs;
    int32_t *plf = po.pl + (int64_t)t.f * po.pfs;

    uint32_t acc[2 * NW][4];
    uint32_t pedge[2 * NW];
    if (t.b == 0) {
#pragma unroll
        for (int n = 0; n < 2 * NW; ++n) {
            pedge[n] = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[n][k] = 0;
        }
    } else {
        // top row of the band: P(Y0, X) = T + sum_{xs <= x' < X} V(x')
        uint32_t v[4][NW];
        const bool xin = x < g.Wc;
        const uint32_t *vp = sc.V + (((int64_t)t.f * g.nb2 + t.b) * g.Wc + x) * g.NWp;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int w = 0; w < NW; ++w) v[k][w] = xin ? vp[k * g.NWp + w] : 0u;
        const int32_t *tp = sc.T + (((int64_t)t.f * g.nb2 + t.b) * g.ns + t.s) * g.NBp4;
#pragma unroll
        for (int n = 0; n < 2 * NW; ++n) {
            const int w = n >> 1, h = n & 1;
            uint32_t c0 = half16(v[0][w], h), c1 = half16(v[1][w], h);
            uint32_t c2 = half16(v[2][w], h), c3 = half16(v[3][w], h);
            uint32_t tot = c0 + c1 + c2 + c3;
            uint32_t inc = warp_incl_scan(tot, lane);
            uint32_t t0 = n < bins ? (uint32_t)tp[n] : 0u;
            uint32_t run = t0 + inc - tot;
            acc[n][0] = (run += c0);
            acc[n][1] = (run += c1);
            acc[n][2] = (run += c2);
            acc[n][3] = (run += c3);
            pedge[n] = t0;
        }
    }

    auto store_row = [&](int Y) {
        int32_t *rp = plf + (int64_t)Y * po.pp;
        if (t.s == 0 && lane == 0) {
#pragma unroll
            for (int n = 0; n < 2 * NW; ++n)
                if (n < bins) rp[(int64_t)n * po.pns] = 0;  // padded column X = 0
        }
        if (!st) return;
        rp += X0;
#pragma unroll
        for (int n = 0; n < 2 * NW; ++n) {
            if (n < bins) {
                int32_t *p = rp + (int64_t)n * po.pns;
                if (po.vec) {
                    *reinterpret_cast<int4 *>(p) =
                        make_int4((int)acc[n][0], (int)acc[n][1], (int)acc[n][2], (int)acc[n][3]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (X0 + k <= g.w) p[k] = (int)acc[n][k];
                }
            }
        }
    };

    // fused cell grid state
    uint32_t ring[KR > 0 ? KR : 1][2 * NW];
    const int dR = KR ? go.cell / 4 - 1 : 0;
    const bool lat_lane = KR && own && (x % (KR ? go.s : 1)) == 0 && x <= (go.ncx - 1) * go.s;
    auto lattice = [&](int Yl) {
        const int yt = Yl - go.cell;
        const bool emit = lat_lane && yt >= Y0 && yt < Y0 + g.R && yt <= (go.ncy - 1) * go.s;
        uint32_t gv[2 * NW];
#pragma unroll
        for (int n = 0; n < 2 * NW; ++n) {
            uint32_t r = __shfl_down_sync(FULL, acc[n][3], dR);
            uint32_t l = __shfl_up_sync(FULL, acc[n][3], 1);
            if (lane == 0) l = pedge[n];
            uint32_t hcur = r - l;
            gv[n] = hcur - ring[0][n];
#pragma unroll
            for (int q = 0; q + 1 < KR; ++q) ring[q][n] = ring[q + 1][n];
            ring[KR > 0 ? KR - 1 : 0][n] = hcur;
        }
        if (emit) {
            int32_t *gp = go.grid +
                          (((int64_t)t.f * go.ncy + yt / go.s) * go.ncx + x / go.s) * bins;
            if ((bins & 3) == 0) {
#pragma unroll
                for (int n = 0; n + 3 < 2 * NW; n += 4)
                    if (n < bins)
                        *reinterpret_cast<int4 *>(gp + n) =
                            make_int4((int)gv[n], (int)gv[n + 1], (int)gv[n + 2], (int)gv[n + 3]);
            } else {
#pragma unroll
                for (int n = 0; n < 2 * NW; ++n)
                    if (n < bins) gp[n] = (int)gv[n];
            }
        }
    };

    store_row(Y0);
    if (KR) {
#pragma unroll
        for (int q = 0; q < (KR > 0 ? KR : 1); ++q)
#pragma unroll
            for (int n = 0; n < 2 * NW; ++n) ring[q][n] = 0;
        lattice(Y0);
    }

    auto load_bm = [&](int Y) -> uint32_t {
        if (x >= g.w) return 0xffffffffu;
        uint32_t v = __ldg(reinterpret_cast<const uint32_t *>(bmf + (int64_t)Y * bp + x));
        if (x + 4 > g.w) v |= 0xffffffffu << (8 * (g.w - x));
        return v;
    };
    const uint32_t *Lbase = sc.L + ((int64_t)t.f * g.ns + t.s) * g.h * g.NWp;
    uint32_t nbm = 0, nL[NW];
    if (Y0 < Ycomp) {
        nbm = load_bm(Y0);
#pragma unroll
        for (int w = 0; w < NW; ++w) nL[w] = Lbase[(int64_t)Y0 * g.NWp + w];
    }
    for (int Y = Y0; Y < Ycomp; ++Y) {
        const uint32_t b4 = nbm;
        uint32_t Lw[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) Lw[w] = nL[w];
        if (Y + 1 < Ycomp) {
            nbm = load_bm(Y + 1);
#pragma unroll
            for (int w = 0; w < NW; ++w) nL[w] = Lbase[(int64_t)(Y + 1) * g.NWp + w];
        }
        uint32_t hb[4], one[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t v = byte_of(b4, k);
            hb[k] = v >> 1;
            one[k] = 1u << ((v & 1u) << 4);
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            uint32_t o0 = oh16(hb[0], one[0], w), o1 = oh16(hb[1], one[1], w);
            uint32_t o2 = oh16(hb[2], one[2], w), o3 = oh16(hb[3], one[3], w);
            uint32_t tot = o0 + o1 + o2 + o3;
            uint32_t inc = warp_incl_scan(tot, lane);
            uint32_t run = Lw[w] + inc - tot;  // row prefix at X = x (u16x2, <= width)
            pedge[2 * w] += Lw[w] & 0xffffu;
            pedge[2 * w + 1] += Lw[w] >> 16;
            run += o0;
            acc[2 * w][0] += run & 0xffffu;
            acc[2 * w + 1][0] += run >> 16;
            run += o1;
            acc[2 * w][1] += run & 0xffffu;
            acc[2 * w + 1][1] += run >> 16;
            run += o2;
            acc[2 * w][2] += run & 0xffffu;
            acc[2 * w + 1][2] += run >> 16;
            run += o3;
            acc[2 * w][3] += run & 0xffffu;
            acc[2 * w + 1][3] += run >> 16;
        }
        if (Y + 1 <= Ystore) store_row(Y + 1);
        if (KR && ((Y + 1) % go.s) == 0) lattice(Y + 1);
    }
}

// ---------------------------------------------------------------------------
// Generic integral for bins > 18 (API completeness; the configs use 8/9/18):
// row prefix per plane row, then column prefix in place.
__global__ void k_generic_rows(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, PlaneOut po,
                               int n, int h, int w, int bins) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * bins * (h + 1)) return;
    const int Y = (int)(i % (h + 1));
    const int b = (int)((i / (h + 1)) % bins);
    const int f = (int)(i / ((int64_t)(h + 1) * bins));
    int32_t *rp = po.pl + (int64_t)f * po.pfs + (int64_t)b * po.pns + (int64_t)Y * po.pp;
    rp[0] = 0;
    int32_t run = 0;
    const int8_t *src = bm + (int64_t)f * bfs + (int64_t)(Y - 1) * bp;
    for (int X = 1; X <= w; ++X) {
        if (Y > 0 && src[X - 1] == b) ++run;
        rp[X] = run;
    }
}

__global__ void k_generic_cols(PlaneOut po, int n, int h, int w, int bins) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * bins * (w + 1)) return;
    const int X = (int)(i % (w + 1));
    const int b = (int)((i / (w + 1)) % bins);
    const int f = (int)(i / ((int64_t)(w + 1) * bins));
    int32_t *cp = po.pl + (int64_t)f * po.pfs + (int64_t)b * po.pns + X;
    int32_t run = 0;
    for (int Y = 0; Y <= h; ++Y) {
        run += cp[(int64_t)Y * po.pp];
        cp[(int64_t)Y * po.pp] = run;
    }
}

// ---------------------------------------------------------------------------
// Generic cell grid from planes (descriptor.py:176-185): one thread per
// (frame, cell), N_b x 4 corner reads.
__global__ void k_cell_grid(const int32_t *__restrict__ pl, int64_t pp, int64_t pns, int64_t pfs,
                            int n, int bins, const int32_t *__restrict__ cxs, int ncx,
                            const int32_t *__restrict__ cys, int ncy, int cell,
                            int32_t *__restrict__ grid) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * ncy * ncx) return;
    const int ci = (int)(i % ncx);
    const int cj = (int)((i / ncx) % ncy);
    const int f = (int)(i / ((int64_t)ncx * ncy));
    const int64_t x0 = cxs[ci], y0 = cys[cj], x1 = x0 + cell, y1 = y0 + cell;
    const int32_t *p = pl + (int64_t)f * pfs;
    int32_t *gp = grid + i * bins;
    for (int b = 0; b < bins; ++b) {
        const int32_t *q = p + (int64_t)b * pns;
        gp[b] = __ldg(q + y1 * pp + x1) + __ldg(q + y0 * pp + x0) - __ldg(q + y0 * pp + x1) -
                __ldg(q + y1 * pp + x0);
    }
}

// descriptor.py:119-124 with block == 1: one denominator per cell.
__global__ void k_cell_norm(const int32_t *__restrict__ grid, int64_t ncells_total, int bins,
                            int norm, double eps_term, double *__restrict__ den) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncells_total) return;
    const int32_t *gp = grid + i * bins;
    double s = 0.0;
    for (int b = 0; b < bins; ++b) {
        double v = (double)gp[b];
        s = norm == 1 ? __dadd_rn(s, fabs(v)) : __dadd_rn(s, __dmul_rn(v, v));
    }
    den[i] = norm == 1 ? __dadd_rn(s, eps_term) : __dsqrt_rn(__dadd_rn(s, eps_term));
}

// descriptor.py:107-124 + detector.py:148-150.  One thread per window.
__global__ void k_window_features(const int32_t *__restrict__ grid, int ncy, int ncx, int bins,
                                  const int32_t *__restrict__ row_idx, int noy,
                                  const int32_t *__restrict__ col_idx, int nox, int cells_x,
                                  int cells_y, int block, int bstride, int norm, double eps_term,
                                  const double *__restrict__ wts, double bias,
                                  double *__restrict__ scores, double *__restrict__ desc, int n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * noy * nox) return;
    const int ix = (int)(i % nox);
    const int iy = (int)((i / nox) % noy);
    const int f = (int)(i / ((int64_t)nox * noy));
    const int32_t *gf = grid + (int64_t)f * ncy * ncx * bins;
    const int32_t *ri = row_idx + (int64_t)iy * cells_y;
    const int32_t *ci = col_idx + (int64_t)ix * cells_x;
    const int bxn = (cells_x - block) / bstride + 1, byn = (cells_y - block) / bstride + 1;
    const int D = bxn * byn * block * block * bins;
    double *dp = desc ? desc + i * D : nullptr;
    double score = 0.0;
    int k = 0;
    for (int by = 0; by < byn; ++by) {
        for (int bx = 0; bx < bxn; ++bx) {
            double den = 1.0;
            if (norm) {
                double s = 0.0;
                for (int cy = 0; cy < block; ++cy)
                    for (int cx = 0; cx < block; ++cx) {
                        const int32_t *h = gf + ((int64_t)ri[by * bstride + cy] * ncx +
                                                 ci[bx * bstride + cx]) * bins;
                        for (int b = 0; b < bins; ++b) {
                            double v = (double)h[b];
                            s = norm == 1 ? __dadd_rn(s, fabs(v)) : __dadd_rn(s, __dmul_rn(v, v));
                        }
                    }
                den = norm == 1 ? __dadd_rn(s, eps_term) : __dsqrt_rn(__dadd_rn(s, eps_term));
            }
            for (int cy = 0; cy < block; ++cy)
                for (int cx = 0; cx < block; ++cx) {
                    const int32_t *h = gf + ((int64_t)ri[by * bstride + cy] * ncx +
                                             ci[bx * bstride + cx]) * bins;
                    for (int b = 0; b < bins; ++b, ++k) {
                        double v = (double)h[b];
                        if (norm) v = __ddiv_rn(v, den);
                        if (dp) dp[k] = v;
                        if (wts) score = fma(__ldg(wts + k), v, score);
                    }
                }
        }
    }
    if (scores) scores[i] = score + bias;
}

// detector.py:202-221.  Explicit _rn intrinsics keep numpy's separate
// multiply/add roundings (no FMA contraction).
__global__ void k_resize(const uint8_t *__restrict__ src, int n, int c, int h, int w, int64_t sp,
                         int64_t scs, int64_t sfs, int nh, int nw, double ry, double rx,
                         uint8_t *__restrict__ dst, int64_t dp, int64_t dcs, int64_t dfs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * c * nh * nw) return;
    const int j = (int)(i % nw);
    const int r = (int)((i / nw) % nh);
    const int ch = (int)((i / ((int64_t)nw * nh)) % c);
    const int f = (int)(i / ((int64_t)nw * nh * c));
    double sy = __dsub_rn(__dmul_rn((double)r + 0.5, ry), 0.5);
    sy = fmin(fmax(sy, 0.0), (double)(h - 1));
    double sx = __dsub_rn(__dmul_rn((double)j + 0.5, rx), 0.5);
    sx = fmin(fmax(sx, 0.0), (double)(w - 1));
    const int y0 = (int)floor(sy), x0 = (int)floor(sx);
    const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
    const double fy = __dsub_rn(sy, (double)y0), fx = __dsub_rn(sx, (double)x0);
    const double gy = __dsub_rn(1.0, fy), gx = __dsub_rn(1.0, fx);
    const uint8_t *p = src + (int64_t)f * sfs + (int64_t)ch * scs;
    const double a0 = (double)__ldg(p + (int64_t)y0 * sp + x0), b0 = (double)__ldg(p + (int64_t)y1 * sp + x0);
    const double a1 = (double)__ldg(p + (int64_t)y0 * sp + x1), b1 = (double)__ldg(p + (int64_t)y1 * sp + x1);
    const double r0 = __dadd_rn(__dmul_rn(a0, gy), __dmul_rn(b0, fy));
    const double r1 = __dadd_rn(__dmul_rn(a1, gy), __dmul_rn(b1, fy));
    double m = rint(__dadd_rn(__dmul_rn(r0, gx), __dmul_rn(r1, fx)));
    m = fmin(fmax(m, 0.0), 255.0);
    dst[(int64_t)f * dfs + (int64_t)ch * dcs + (int64_t)r * dp + j] = (uint8_t)m;
}

// ---------------------------------------------------------------------------
// Host-side dispatch

inline unsigned blocks_for_tiles(int64_t tiles) {
    return (unsigned)((tiles + (K_THREADS / 32) - 1) / (K_THREADS / 32));
}
inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <int NW>
void launch_counts_from_image(int c, const uint8_t *img, int64_t ip, int64_t ics, int64_t ifs,
                              const uint8_t *lut, int8_t *bm, int64_t bp, int64_t bfs,
                              const TileGeom &g, const Scratch &sc, cudaStream_t st, bool counts) {
    constexpr int NWB = (2 * NW + 3) / 4;
    const unsigned nb = blocks_for_tiles((int64_t)g.n * g.nb1 * g.ns);
    if (c == 1) {
        if (counts)
            k_grad_bin<1, NWB, NW, true><<<nb, K_THREADS, 0, st>>>(img, ip, ics, ifs, lut, bm, bp, bfs, g, sc);
        else
            k_grad_bin<1, NWB, NW, false><<<nb, K_THREADS, 0, st>>>(img, ip, ics, ifs, lut, bm, bp, bfs, g, sc);
    } else {
        if (counts)
            k_grad_bin<3, NWB, NW, true><<<nb, K_THREADS, 0, st>>>(img, ip, ics, ifs, lut, bm, bp, bfs, g, sc);
        else
            k_grad_bin<3, NWB, NW, false><<<nb, K_THREADS, 0, st>>>(img, ip, ics, ifs, lut, bm, bp, bfs, g, sc);
    }
}

template <int NW>
void launch_scans(const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    constexpr int NWB = (2 * NW + 3) / 4;
    k_scan_cols<NWB, NW><<<blocks_for((int64_t)g.n * g.Wc, 256), 256, 0, st>>>(g, sc);
    k_scan_rows<NW><<<blocks_for((int64_t)g.n * g.h, 256), 256, 0, st>>>(g, sc);
    k_scan_tiles<<<blocks_for((int64_t)g.n * g.ns * g.NBp4, 256), 256, 0, st>>>(g, sc);
}

template <int NW>
void launch_planes(int kr, const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                   const GridOut &go, const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    const unsigned nb = blocks_for_tiles((int64_t)g.n * g.nb2 * g.ns);
    if (kr == 0)
        k_planes<NW, 0><<<nb, K_THREADS, 0, st>>>(bm, bp, bfs, po, go, g, sc);
    else if (kr == 1)
        k_planes<NW, 1><<<nb, K_THREADS, 0, st>>>(bm, bp, bfs, po, go, g, sc);
    else
        k_planes<NW, 2><<<nb, K_THREADS, 0, st>>>(bm, bp, bfs, po, go, g, sc);
}

template <int NW>
void launch_counts_from_bm(const int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                           const Scratch &sc, cudaStream_t st) {
    constexpr int NWB = (2 * NW + 3) / 4;
    k_bin_counts<NWB, NW><<<blocks_for_tiles((int64_t)g.n * g.nb1 * g.ns), K_THREADS, 0, st>>>(
        bm, bp, bfs, g, sc);
}

#define HOG_SWITCH_NW(nw, CALL)                                              \
    switch (nw) {                                                            \
        case 1: CALL(1); break;                                              \
        case 2: CALL(2); break;                                              \
        case 3: CALL(3); break;                                              \
        case 4: CALL(4); break;                                              \
        case 5: CALL(5); break;                                              \
        case 6: CALL(6); break;                                              \
        case 7: CALL(7); break;                                              \
        case 8: CALL(8); break;                                              \
        case 9: CALL(9); break;                                              \
        default: return fail(HOG_EINVAL, "internal: NW %d not instantiated", nw); \
    }

int check_frames(int n, int h, int w) {
    if (n < 1) return fail(HOG_EINVAL, "n must be >= 1, got %d", n);
    if (h < 3 || w < 3) return fail(HOG_EINVAL, "need at least 3x3, got %dx%d", w, h);
    if (h >= 65000 || w >= 65000) return fail(HOG_EINVAL, "frame %dx%d exceeds 65000 per side", w, h);
    return HOG_OK;
}

int check_bins(int bins) {
    if (bins < 2 || bins > 64) return fail(HOG_EINVAL, "bins must be in [2, 64], got %d", bins);
    return HOG_OK;
}

int check_pitch8(const void *p, int64_t pitch, int w, const char *what) {
    if (((uintptr_t)p & 3) != 0 || pitch % 4 != 0 || pitch < round_up(w, 4))
        return fail(HOG_EINVAL, "%s: need 4-byte aligned base and pitch %% 4 == 0, pitch >= %lld (got %lld)",
                    what, (long long)round_up(w, 4), (long long)pitch);
    return HOG_OK;
}

PlaneOut make_po(int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int w) {
    PlaneOut po{pl, pp, pns, pfs, 0};
    po.vec = (((uintptr_t)(pl + 1) & 15) == 0) && pp % 4 == 0 && pns % 4 == 0 && pfs % 4 == 0 &&
             pp >= (int64_t)w + 4;
    return po;
}

int integral_impl(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int bins,
                  int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, void *scratch, size_t sbytes,
                  cudaStream_t st) {
    PlaneOut po = make_po(pl, pp, pns, pfs, w);
    if (bins > MAX_FUSED_BINS) {
        k_generic_rows<<<blocks_for((int64_t)n * bins * (h + 1), 128), 128, 0, st>>>(bm, bp, bfs, po, n, h, w, bins);
        k_generic_cols<<<blocks_for((int64_t)n * bins * (w + 1), 128), 128, 0, st>>>(po, n, h, w, bins);
        return check_launch("integral (generic)");
    }
    TileGeom g = make_geom(n, h, w, bins, false, 0, 0);
    Scratch sc{};
    size_t need = carve(g, nullptr, nullptr);
    if (scratch == nullptr || sbytes < need)
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", need, sbytes);
    carve(g, scratch, &sc);
    GridOut go{nullptr, 4, 4, 0, 0};
#define CALL(NWv)                                       \
    launch_counts_from_bm<NWv>(bm, bp, bfs, g, sc, st); \
    launch_scans<NWv>(g, sc, st);                       \
    launch_planes<NWv>(0, bm, bp, bfs, po, go, g, sc, st);
    HOG_SWITCH_NW(g.NW, CALL)
#undef CALL
    return check_launch("hog_integral");
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char *hog_version(void) { return "hogb200 1.0 sm_100a"; }

const char *hog_last_error(void) { return g_err.c_str(); }

int64_t hog_plane_pitch(int w) { return round_up((int64_t)w + 4, 8); }

int hog_grad_bin(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                 int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp, int64_t bfs,
                 hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (c != 1 && c != 3) return fail(HOG_EINVAL, "channels must be 1 or 3, got %d", c);
    if ((e = check_pitch8(img, ip, w, "image")) || (e = check_pitch8(bm, bp, w, "binmap"))) return e;
    if (!img || !lut || !bm) return fail(HOG_EINVAL, "null buffer");
    TileGeom g = make_geom(n, h, w, bins, false, 0, 0);
    Scratch sc{};
    cudaStream_t st = (cudaStream_t)stream;
    // bins only affect counting; run the NW=1 instance without counts
    launch_counts_from_image<1>(c, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st, false);
    return check_launch("hog_grad_bin");
}

size_t hog_scratch_bytes(int n, int h, int w, int bins, int stride, int cell) {
    if (n < 1 || h < 1 || w < 1 || bins < 1) return 0;
    bool fused = stride > 0 && cell > 0;
    TileGeom g = make_geom(n, h, w, bins, fused, stride, cell);
    size_t a = carve(g, nullptr, nullptr);
    TileGeom g2 = make_geom(n, h, w, bins, false, 0, 0);
    size_t b = carve(g2, nullptr, nullptr);
    return a > b ? a : b;
}

int hog_integral(const int8_t *bm, int n, int h, int w, int64_t bp, int64_t bfs, int bins,
                 int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, void *scratch,
                 size_t sbytes, hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if ((e = check_pitch8(bm, bp, w, "binmap"))) return e;
    if (pp < (int64_t)w + 1) return fail(HOG_EINVAL, "plane pitch %lld < w+1", (long long)pp);
    if (!bm || !pl) return fail(HOG_EINVAL, "null buffer");
    return integral_impl(bm, bp, bfs, n, h, w, bins, pl, pp, pns, pfs, scratch, sbytes,
                         (cudaStream_t)stream);
}

int hog_pipeline(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                 int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp, int64_t bfs,
                 int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int cell, int stride, int ncx,
                 int ncy, int32_t *grid, void *scratch, size_t sbytes, void *const *stage_events,
                 hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (c != 1 && c != 3) return fail(HOG_EINVAL, "channels must be 1 or 3, got %d", c);
    if ((e = check_pitch8(img, ip, w, "image")) || (e = check_pitch8(bm, bp, w, "binmap"))) return e;
    if (pp < (int64_t)w + 1) return fail(HOG_EINVAL, "plane pitch %lld < w+1", (long long)pp);
    if (!img || !lut || !bm || !pl) return fail(HOG_EINVAL, "null buffer");
    if (bins > MAX_FUSED_BINS)
        return fail(HOG_EINVAL, "fused pipeline supports bins <= %d (got %d); use hog_grad_bin + "
                    "hog_integral + hog_cell_grid", MAX_FUSED_BINS, bins);
    int kr = 0;
    if (grid) {
        if (stride <= 0 || stride % 4 != 0 || cell % stride != 0 || cell / stride > 2 || cell % 4 != 0)
            return fail(HOG_EINVAL, "fused grid needs stride %% 4 == 0, cell %% stride == 0, "
                        "cell/stride <= 2 (stride %d, cell %d)", stride, cell);
        if (ncx < 1 || ncy < 1 || (int64_t)(ncx - 1) * stride + cell > w ||
            (int64_t)(ncy - 1) * stride + cell > h)
            return fail(HOG_EINVAL, "cell lattice %dx%d (step %d, cell %d) exceeds %dx%d", ncx, ncy,
                        stride, cell, w, h);
        kr = cell / stride;
    }
    cudaStream_t st = (cudaStream_t)stream;
    TileGeom g = make_geom(n, h, w, bins, kr > 0, stride, cell);
    Scratch sc{};
    size_t need = carve(g, nullptr, nullptr);
    if (scratch == nullptr || sbytes < need)
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", need, sbytes);
    carve(g, scratch, &sc);
    PlaneOut po = make_po(pl, pp, pns, pfs, w);
    GridOut go{grid, kr ? stride : 4, kr ? cell : 4, ncx, ncy};
    auto mark = [&](int i) {
        if (stage_events && stage_events[i]) cudaEventRecord((cudaEvent_t)stage_events[i], st);
    };
#define CALL(NWv)                                                                          \
    mark(0);                                                                               \
    launch_counts_from_image<NWv>(c, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st, true); \
    mark(1);                                                                               \
    launch_scans<NWv>(g, sc, st);                                                          \
    mark(2);                                                                               \
    launch_planes<NWv>(kr, bm, bp, bfs, po, go, g, sc, st);                                \
    mark(3);
    HOG_SWITCH_NW(g.NW, CALL)
#undef CALL
    return check_launch("hog_pipeline");
}

int hog_cell_grid(const int32_t *pl, int n, int h, int w, int bins, int64_t pp, int64_t pns,
                  int64_t pfs, const int32_t *cxs, int ncx, const int32_t *cys, int ncy, int cell,
                  int32_t *grid, hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (ncx < 1 || ncy < 1 || cell < 1) return fail(HOG_EINVAL, "empty cell lattice");
    if (!pl || !cxs || !cys || !grid) return fail(HOG_EINVAL, "null buffer");
    k_cell_grid<<<blocks_for((int64_t)n * ncx * ncy, 128), 128, 0, (cudaStream_t)stream>>>(
        pl, pp, pns, pfs, n, bins, cxs, ncx, cys, ncy, cell, grid);
    return check_launch("hog_cell_grid");
}

int hog_cell_norm(const int32_t *grid, int n, int ncells, int bins, int norm, double eps_term,
                  double *den, hog_stream_t stream) {
    g_err.clear();
    if (norm != 1 && norm != 2) return fail(HOG_EINVAL, "norm must be 1 (l1) or 2 (l2)");
    if (n < 1 || ncells < 1 || bins < 1 || !grid || !den) return fail(HOG_EINVAL, "bad arguments");
    const int64_t tot = (int64_t)n * ncells;
    k_cell_norm<<<blocks_for(tot, 256), 256, 0, (cudaStream_t)stream>>>(grid, tot, bins, norm,
                                                                          eps_term, den);
    return check_launch("hog_cell_norm");
}

int hog_window_features(const int32_t *grid, int n, int ncy, int ncx, int bins,
                        const int32_t *row_idx, int noy, const int32_t *col_idx, int nox,
                        int cells_x, int cells_y, int block, int bstride, int norm,
                        double eps_term, const double *wts, double bias, double *scores,
                        double *desc, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || bins < 1 || !grid || !row_idx || !col_idx)
        return fail(HOG_EINVAL, "bad arguments");
    if (block < 1 || block > cells_x || block > cells_y || bstride < 1)
        return fail(HOG_EINVAL, "block %d / stride %d do not fit %dx%d cells", block, bstride,
                    cells_x, cells_y);
    if (norm < 0 || norm > 2) return fail(HOG_EINVAL, "norm must be 0, 1 or 2");
    if (scores && !wts) return fail(HOG_EINVAL, "scores need weights");
    const int64_t tot = (int64_t)n * noy * nox;
    k_window_features<<<blocks_for(tot, 128), 128, 0, (cudaStream_t)stream>>>(
        grid, ncy, ncx, bins, row_idx, noy, col_idx, nox, cells_x, cells_y, block, bstride, norm,
        eps_term, wts, bias, scores, desc, n);
    return check_launch("hog_window_features");
}

int hog_resize_bilinear(const uint8_t *src, int n, int c, int h, int w, int64_t sp, int64_t scs,
                        int64_t sfs, int nh, int nw, double ry, double rx, uint8_t *dst,
                        int64_t dp, int64_t dcs, int64_t dfs, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || c < 1 || h < 1 || w < 1 || nh < 1 || nw < 1 || !src || !dst)
        return fail(HOG_EINVAL, "bad arguments");
    const int64_t tot = (int64_t)n * c * nh * nw;
    k_resize<<<blocks_for(tot, 256), 256, 0, (cudaStream_t)stream>>>(src, n, c, h, w, sp, scs, sfs,
                                                                       nh, nw, ry, rx, dst, dp,
                                                                       dcs, dfs);
    return check_launch("hog_resize_bilinear");
}

}  // extern "C"
