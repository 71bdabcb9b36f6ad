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
//   16-byte coalesced stores, by k_planes.  One warp owns a band of R plane
//   rows of one frame and sweeps it strip by strip (4 columns per lane, 128
//   columns per strip), walking down each strip: the row prefix is a warp
//   scan of one-hot counts packed two bins per 32-bit word (16-bit lanes; a
//   row prefix never exceeds the width), the column prefix lives in
//   registers, and the row prefix left of the strip is handed from strip to
//   strip through shared memory.  The only carry that crosses warps is the
//   per-column count above the band: k_grad_bin counts bins per (band,
//   column) while it bins the image, and k_scan_cols turns those counts into
//   the column counts above every band.  When the scan lattice is regular,
//   k_planes also emits the cell-histogram grid from the plane values it
//   holds in registers (4-corner formula, descriptor.py:176-185), so the
//   planes are never re-read.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/hogb200.h"

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LUT_SIDE = 511;
constexpr int K_THREADS = 128;      // 4 independent warps per CTA
constexpr int MAX_FUSED_BINS = 18;  // NW <= 9 packed words
constexpr int CHUNK = 128;          // k_grad_bin columns per warp (32 lanes x 4)

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
// Geometry shared by k_grad_bin / k_bin_counts / k_scan_cols / k_planes.
struct TileGeom {
    int n, h, w, bins;
    int R;      // rows per band (multiple of the lattice step when the grid is fused)
    int Ws;     // plane columns per k_planes strip (<= 128, multiple of 8)
    int ns;     // strips per frame
    int nb1;    // pixel bands: ceil(h / R)         (k_grad_bin tiles)
    int nb2;    // plane bands: h / R + 1            (k_planes tiles; plane rows 0..h)
    int nc1;    // 128-column chunks: ceil(w / 128)  (k_grad_bin tiles)
    int Wc;     // nc1 * 128: padded width of the per-column scratch arrays
    int NWB;    // u8x4 words per column count   = ceil(bins / 4)
    int NW;     // u16x2 words per row count     = ceil(bins / 2)
    int NWp;    // NW padded to a multiple of 4 (16-byte V rows)
    int halo;   // extra rows a band computes for straddling cells (cell - step)
    int Lrows;  // rows of row-carry state (R + halo)
    int VC;     // plane columns per lane in k_planes (8: 256-bit stores, 4: 128-bit)
    int NWARP;  // warps (strips) per k_planes CTA
    int nss;    // super-strips: ceil(ns / NWARP)
};

// Scratch arrays (device), carved from the caller's scratch buffer.
struct Scratch {
    uint32_t *C;  // [n][nb1][Wc][NWB]  bin counts per (pixel band, column), u8x4
    uint32_t *V;  // [n][nb2][Wc][NWp]  counts above each plane band, u16x2
};

TileGeom make_geom(int n, int h, int w, int bins, bool fused, int stride, int cell, bool v8ok) {
    TileGeom g{};
    g.n = n; g.h = h; g.w = w; g.bins = bins;
    g.NWB = (bins + 3) / 4;
    g.NW = (bins + 1) / 2;
    g.NWp = (int)round_up(g.NW, 4);
    // 8 columns per lane only when every lattice column starts a lane chunk
    g.VC = (v8ok && g.NW <= 5 && (!fused || stride % 8 == 0)) ? 8 : 4;
    const int span = 32 * g.VC;
    if (fused) {
        int a = 8, b = stride;
        while (b) { int r = a % b; a = b; b = r; }
        const int l = 8 / a * stride;  // lcm(8, stride): strips start on lattice columns, 32-B aligned
        g.Ws = ((span + stride - cell) / l) * l;
        g.halo = cell - stride;
    } else {
        g.Ws = span;
        g.halo = 0;
    }
    g.ns = (w + g.Ws - 1) / g.Ws;
    g.NWARP = g.ns < 8 ? g.ns : 8;
    g.nss = (g.ns + g.NWARP - 1) / g.NWARP;
    g.nc1 = (w + CHUNK - 1) / CHUNK;
    g.Wc = g.nc1 * CHUNK;
    int R = 128;
    const char *env = getenv("HOGB200_BAND_ROWS");
    if (env && atoi(env) >= 8) {
        R = atoi(env);
    } else {
        while (R > 16 && (int64_t)n * (h / R + 1) * g.NWARP < 148 * 32) R /= 2;
    }
    if (fused && R % stride != 0) R = (int)round_up(R, stride);
    if (R > 240) R = 240;  // u8 column counts; packed strip-local sums stay < 2^16
    g.R = R;
    g.nb1 = (h + R - 1) / R;
    g.nb2 = h / R + 1;
    g.Lrows = R + g.halo;
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
    size_t oV = take(sizeof(uint32_t) * (size_t)g.n * g.nb2 * g.Wc * g.NWp);
    if (sc && base) {
        char *b = (char *)base;
        sc->C = (uint32_t *)(b + oC);
        sc->V = (uint32_t *)(b + oV);
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

__device__ __forceinline__ uint32_t byte_of(uint32_t v, int k) { return (v >> (8 * k)) & 0xffu; }

// u8x4 word -> u16x2 word holding bytes (2h, 2h+1)
__device__ __forceinline__ uint32_t widen_half(uint32_t v, int h) {
    return h == 0 ? __byte_perm(v, 0u, 0x4140) : __byte_perm(v, 0u, 0x4342);
}

__device__ __forceinline__ uint32_t half16(uint32_t v, int h) {
    return h == 0 ? (v & 0xffffu) : (v >> 16);
}

__device__ __forceinline__ int64_t warp_id() {
    return (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
}

// Per-lane column counts of 4 pixel bins (bytes of `bins4`, 0xFF = none):
// cc[k][w] holds bins 4w..4w+3 of column k as u8x4.
template <int NWB>
__device__ __forceinline__ void count_cols(uint32_t bins4, uint32_t (&cc)[4][NWB]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t v = byte_of(bins4, k);
        const uint32_t q = v >> 2, one = 1u << ((v & 3u) << 3);
#pragma unroll
        for (int w = 0; w < NWB; ++w)
            if (q == (uint32_t)w) cc[k][w] += one;
    }
}

template <int NWB>
__device__ __forceinline__ void store_cols(const TileGeom &g, const Scratch &sc, int f, int b,
                                           int x, uint32_t (&cc)[4][NWB]) {
    uint32_t *cp = sc.C + (((int64_t)f * g.nb1 + b) * g.Wc + x) * NWB;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int w = 0; w < NWB; ++w) cp[k * NWB + w] = cc[k][w];
}

// ---------------------------------------------------------------------------
// K1: gradient + LUT binning (gradient.py:95-121), optionally counting bins
// per (band, column) for k_scan_cols.  One warp = R rows x 128 columns of
// one frame; lane L owns pixel columns x0+4L .. x0+4L+3 and slides a
// three-row window down the band, two rows of loads in flight; left/right
// neighbours come from the adjacent lanes by shuffle.

template <int CH, int NWB, bool COUNTS>
__global__ void __launch_bounds__(K_THREADS)
k_grad_bin(const uint8_t *__restrict__ img, int64_t ip, int64_t ics, int64_t ifs,
           const uint8_t *__restrict__ lut, int8_t *__restrict__ bm, int64_t bp, int64_t bfs,
           TileGeom g, Scratch sc) {
    const int64_t wid = warp_id();
    if (wid >= (int64_t)g.n * g.nb1 * g.nc1) return;
    const int chunk = (int)(wid % g.nc1);
    const int b = (int)((wid / g.nc1) % g.nb1);
    const int f = (int)(wid / ((int64_t)g.nc1 * g.nb1));
    const int lane = threadIdx.x & 31;
    const int x = chunk * CHUNK + 4 * lane;
    const bool inx = x < g.w;
    const int y0 = b * g.R, y1 = min(y0 + g.R, g.h);
    const uint8_t *im = img + (int64_t)f * ifs;
    int8_t *bmf = bm + (int64_t)f * bfs;

    // bytes of this lane's 4 columns that are interior pixels (1 <= x <= w-2)
    uint32_t valid = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (x + k >= 1 && x + k <= g.w - 2) valid |= 0xffu << (8 * k);

    auto ldw = [&](int y, int ch) -> uint32_t {
        return (inx && y >= 0 && y < g.h)
                   ? __ldg(reinterpret_cast<const uint32_t *>(im + ch * ics + (int64_t)y * ip + x))
                   : 0u;
    };
    // left neighbour byte of lane 0, right neighbour byte of lane 31
    auto lde = [&](int y, int ch) -> uint32_t {
        const int xx = lane == 0 ? x - 1 : x + 4;
        return ((lane == 0 || lane == 31) && xx >= 0 && xx < g.w && y >= 0 && y < g.h)
                   ? (uint32_t)__ldg(im + ch * ics + (int64_t)y * ip + xx)
                   : 0u;
    };

    // rows y-1 (r0), y (r1), y+1 (r2), y+2 (r3, in flight); e1/e3: edge bytes
    uint32_t r0[CH], r1[CH], r2[CH], r3[CH], e1[CH], e2[CH], e3[CH];
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
        r0[ch] = ldw(y0 - 1, ch);
        r1[ch] = ldw(y0, ch);
        e1[ch] = lde(y0, ch);
        r2[ch] = ldw(y0 + 1, ch);
        e2[ch] = lde(y0 + 1, ch);
    }
    uint32_t cc[4][NWB];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] = 0;

    for (int y = y0; y < y1; ++y) {
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            r3[ch] = ldw(y + 2, ch);
            e3[ch] = lde(y + 2, ch);
        }
        uint32_t bins4 = 0xffffffffu;
        if (y > 0 && y < g.h - 1) {
            int bdx[4], bdy[4];
#pragma unroll
            for (int ch = 0; ch < CH; ++ch) {
                const uint32_t prev = __shfl_up_sync(FULL, r1[ch], 1);
                const uint32_t next = __shfl_down_sync(FULL, r1[ch], 1);
                // Lw: bytes at x-1..x+2, Rw: bytes at x+1..x+4
                const uint32_t Lw = __byte_perm(lane == 0 ? e1[ch] : prev >> 24, r1[ch], 0x6540);
                const uint32_t Rw = __byte_perm(r1[ch], lane == 31 ? e1[ch] : next, 0x4321);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int dx = (int)byte_of(Rw, k) - (int)byte_of(Lw, k);
                    const int dy = (int)byte_of(r2[ch], k) - (int)byte_of(r0[ch], k);
                    if (CH == 1) {
                        bdx[k] = dx, bdy[k] = dy;
                    } else {
                        // gradient.py:113-117: largest dx^2+dy^2 wins, first channel on ties
                        const int mag = dx * dx + dy * dy;
                        if (ch == 0 || mag > bdx[k] * bdx[k] + bdy[k] * bdy[k]) bdx[k] = dx, bdy[k] = dy;
                    }
                }
            }
            bins4 = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                bins4 |= (uint32_t)__ldg(lut + (bdx[k] * LUT_SIDE + bdy[k] + (255 * LUT_SIDE + 255)))
                         << (8 * k);
            bins4 = (bins4 & valid) | ~valid;
        }
        if (inx) *reinterpret_cast<uint32_t *>(bmf + (int64_t)y * bp + x) = bins4;
        if (COUNTS) count_cols<NWB>(bins4, cc);
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            r0[ch] = r1[ch];
            r1[ch] = r2[ch];
            r2[ch] = r3[ch];
            e1[ch] = e2[ch];
            e2[ch] = e3[ch];
        }
    }
    if (COUNTS) store_cols<NWB>(g, sc, f, b, x, cc);
}

// K1': the same per-(band, column) counts from an existing bin map (hog_integral).
template <int NWB>
__global__ void __launch_bounds__(K_THREADS)
k_bin_counts(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, TileGeom g, Scratch sc) {
    const int64_t wid = warp_id();
    if (wid >= (int64_t)g.n * g.nb1 * g.nc1) return;
    const int chunk = (int)(wid % g.nc1);
    const int b = (int)((wid / g.nc1) % g.nb1);
    const int f = (int)(wid / ((int64_t)g.nc1 * g.nb1));
    const int lane = threadIdx.x & 31;
    const int x = chunk * CHUNK + 4 * lane;
    const int y0 = b * g.R, y1 = min(y0 + g.R, g.h);
    const int8_t *bmf = bm + (int64_t)f * bfs;
    uint32_t mask = 0;  // bytes past w count nowhere
    if (x + 4 > g.w) mask = x >= g.w ? 0xffffffffu : 0xffffffffu << (8 * (g.w - x));
    uint32_t cc[4][NWB];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] = 0;
    for (int y = y0; y < y1; ++y) {
        uint32_t v = 0xffffffffu;
        if (x < g.w) v = __ldg(reinterpret_cast<const uint32_t *>(bmf + (int64_t)y * bp + x)) | mask;
        count_cols<NWB>(v, cc);
    }
    store_cols<NWB>(g, sc, f, b, x, cc);
}

// V[f][b][x] = sum over pixel bands b' < b of C[f][b'][x]: column counts of
// plane rows [0, b*R), u16x2 packed (<= h < 65536).
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

// ---------------------------------------------------------------------------
// K2: integral planes (+ fused cell grid).  integral.py:58-87,
// descriptor.py:176-185.  KR = cell / lattice step (0: no grid); VC = plane
// columns per lane (8: one 256-bit store per plane row, 4: 128-bit).
//
// CTA = (frame f, band b): plane rows [Y0, Y0+R) (+ `halo` rows computed for
// cells straddling the band).  Its NWARP warps own adjacent column strips and
// walk the band's rows together, so every plane row leaves the SM as one
// contiguous burst (HBM write efficiency: tools/probe_store.cu).  In a strip,
// lane L holds P(Y, X) for its VC columns and every bin in registers (acc).
// Row Y -> Y+1 adds the row prefix R(Y, X) = Lc(Y) + (warp-exclusive count) +
// (lane-local count); Lc(Y), the count left of the strip, is the sum of the
// strip totals of the warps to the left, exchanged through shared memory once
// per group of G rows (phase A: warp scans + strip totals, barrier, phase B:
// accumulate + store).  Frames wider than NWARP strips are swept in
// super-strips, carrying Lc through shared memory.  Lattice row Yl:
// Hd(Yl, xi) = P(Yl, xi + cell) - P(Yl, xi) by shuffles, and the cell with
// top-left (Yl - cell, xi) is Hd(Yl) - Hd(Yl - cell) (per-lane ring in smem).

struct PlaneOut {
    int32_t *pl;
    int64_t pp, pns, pfs;
    int vec;  // 32-B aligned rows: vector stores + full-sector padding writes
};

struct GridOut {
    int32_t *grid;
    int s, cell, ncx, ncy;
};

constexpr int K2_G = 4;  // rows per phase-A/phase-B group

// shared-memory carve-up of one k_planes CTA (32-bit words, every array 16-B aligned)
struct K2Smem {
    int rowtot, Lsup, vtot, Tsup, ptop, ring, total;
};

__host__ __device__ inline int k2_r4(int v) { return (v + 3) & ~3; }

__host__ __device__ inline K2Smem k2_smem(const TileGeom &g, int kr) {
    const int NB = 2 * g.NW;
    K2Smem m;
    m.rowtot = 0;                                                // [2][G][NWARP][NWp]
    m.Lsup = m.rowtot + k2_r4(2 * K2_G * g.NWARP * g.NWp);       // [2][Lrows][NWp]
    m.vtot = m.Lsup + k2_r4(2 * g.Lrows * g.NWp);                // [NWARP][NB]
    m.Tsup = m.vtot + k2_r4(g.NWARP * NB);                       // [2][NB]
    m.ptop = m.Tsup + k2_r4(2 * NB);                             // [NWARP][NB][32][VC]
    m.ring = m.ptop + k2_r4(g.NWARP * NB * 32 * g.VC);           // [NWARP][KR][NB][32]
    m.total = m.ring + k2_r4(g.NWARP * kr * NB * 32);
    return m;
}

__host__ __device__ inline int k2_smem_words(const TileGeom &g, int kr) { return k2_smem(g, kr).total; }

template <int VC>
__device__ __forceinline__ void store_chunk(int32_t *p, const uint32_t (&v)[VC], bool vec, int valid) {
    if (vec) {
        if constexpr (VC == 8) {
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
                         "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                         : "memory");
        } else {
            *reinterpret_cast<int4 *>(p) = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < VC; ++k)
            if (k < valid) p[k] = (int)v[k];
    }
}

template <int VC>
struct BmWord;
template <>
struct BmWord<4> {
    uint32_t w;
    __device__ __forceinline__ uint32_t byte(int k) const { return byte_of(w, k); }
};
template <>
struct BmWord<8> {
    uint32_t lo, hi;
    __device__ __forceinline__ uint32_t byte(int k) const { return k < 4 ? byte_of(lo, k) : byte_of(hi, k - 4); }
};

// P(Y, X) = ptop(X) + Lacc(Y) + Q(Y, X):
//   ptop(X) = sum_{xs <= x' < X} V(x')  -- band's top row relative to the strip's
//             left edge; constant through the band, kept in shared memory
//   Lacc(Y) = P(Y, xs)                  -- one value per bin, uniform over the warp
//   Q(Y, X) = sum_{Y0 <= y < Y} count of row y in [xs, X)  -- <= (R+halo)*32*VC < 2^16,
//             so two bins share one register (u16x2) and a row update is one add
#ifndef K2_MINB
#define K2_MINB 2
#endif
template <int NW, int KR, int VC, bool VEC>
__global__ void __launch_bounds__(256, K2_MINB)
k_planes(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, PlaneOut po, GridOut go,
         TileGeom g, Scratch sc) {
    extern __shared__ uint32_t smem[];
    constexpr int NB = 2 * NW;
    constexpr int G = K2_G;
    const int nwarp = g.NWARP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = (int)(blockIdx.x % g.nb2);
    const int f = (int)(blockIdx.x / g.nb2);
    const K2Smem lay = k2_smem(g, KR);
    uint32_t *rowtot = smem + lay.rowtot;                    // [2][G][nwarp][NWp]
    uint32_t *Lsup = smem + lay.Lsup;                        // [2][Lrows][NWp]
    uint32_t *vtot = smem + lay.vtot;                        // [nwarp][NB]
    uint32_t *Tsup = smem + lay.Tsup;                        // [2][NB]
    uint32_t *ptop = smem + lay.ptop + (warp * NB * 32 + lane) * VC;  // this lane's [NB][VC] (stride 32*VC)
    uint32_t *ring = smem + lay.ring + warp * KR * NB * 32 + lane;    // this lane's [KR][NB] (stride 32)

    const int Y0 = b * g.R;
    const int Ystore = min(Y0 + g.R - 1, g.h);
    const int Ycomp = KR ? max(Ystore, min(Y0 + g.R + g.halo, g.h)) : Ystore;
    const bool odd = (g.bins & 1) != 0;  // the last packed bin is padding
    const int lo = g.Ws / VC - 1;        // last lane owning strip columns
    const int NWp = g.NWp;
    const int64_t pns = po.pns, pp = po.pp;
    const int8_t *bmf = bm + (int64_t)f * bfs;
    int32_t *plf = po.pl + (int64_t)f * po.pfs;
    const uint32_t *Vb = sc.V + ((int64_t)f * g.nb2 + b) * g.Wc * NWp;
    // lattice bookkeeping (integer divisions once per CTA)
    const int ls = KR ? go.s : 1;
    const int dR = KR ? go.cell / VC - 1 : 0;  // lanes between a cell's left and right corner
    const int jtop = Y0 / ls;                   // grid row of the band's first owned cell
    const int jend = KR ? min((Y0 + g.R - 1) / ls, go.ncy - 1) : -1;  // last owned grid row
    const int lag = KR ? go.cell / ls : 0;      // lattice rows between a cell's top and bottom

    for (int ss = 0; ss < g.nss; ++ss) {
        const int s = ss * nwarp + warp;
        const bool active = s < g.ns;
        const bool last_warp = warp == nwarp - 1;
        const int xs = s * g.Ws;
        const int x = xs + VC * lane;  // pixel column of the lane's first column; P column x+1
        const bool own = VC * lane < g.Ws;
        const int X0 = x + 1;
        const bool st = active && own && X0 <= g.w;
        const bool lat_lane = KR && st && (x % ls) == 0 && x <= (go.ncx - 1) * ls;
        const int gcol = x / ls;
        const uint32_t *rdL = Lsup + (ss & 1) * g.Lrows * NWp;
        uint32_t *wrL = Lsup + ((ss & 1) ^ 1) * g.Lrows * NWp;

        uint32_t Q[NW][VC];
        uint32_t Lacc[NB];
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int k = 0; k < VC; ++k) Q[w][k] = 0;

        // ---- top row: ptop(X) = sum_{xs <= x' < X} V(x'); strip totals -> left edge
        if (active) {
            const bool vin = b > 0 && x < g.Wc;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                uint32_t v[VC];
#pragma unroll
                for (int k = 0; k < VC; ++k) v[k] = vin ? Vb[(int64_t)(x + k) * NWp + w] : 0u;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = 2 * w + h;
                    uint32_t tot = 0;
#pragma unroll
                    for (int k = 0; k < VC; ++k) tot += half16(v[k], h);
                    const uint32_t inc = warp_incl_scan(tot, lane);
                    uint32_t run = inc - tot;
                    uint32_t pt[VC];
#pragma unroll
                    for (int k = 0; k < VC; ++k) pt[k] = (run += half16(v[k], h));
#pragma unroll
                    for (int k = 0; k < VC; k += 4)
                        *reinterpret_cast<uint4 *>(ptop + n * 32 * VC + k) =
                            make_uint4(pt[k], pt[k + 1], pt[k + 2], pt[k + 3]);
                    const uint32_t stot = __shfl_sync(FULL, inc, lo);  // strip total (own lanes)
                    if (lane == 0) vtot[warp * NB + n] = stot;
                }
            }
        }
        __syncthreads();
        if (active) {
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                uint32_t T = ss ? Tsup[(ss & 1) * NB + n] : 0u;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < warp) T += vtot[q * NB + n];
                Lacc[n] = T;  // P(Y0, xs)
            }
        }
        if (warp == 0 && lane < NB) {  // P(Y0, .) at the next super-strip's left edge
            uint32_t T = ss ? Tsup[(ss & 1) * NB + lane] : 0u;
            for (int q = 0; q < nwarp; ++q)
                if (ss * nwarp + q < g.ns) T += vtot[q * NB + lane];
            Tsup[((ss & 1) ^ 1) * NB + lane] = T;
        }

        // plane row pointer (plane 0, the lane's first column) of the next row to store
        int32_t *prow = plf + (int64_t)Y0 * pp + X0;
        auto store_row = [&]() {
            if (s == 0 && lane == 0) {
                // padded column X = 0; on aligned rows also the previous row's tail
                // padding, so that sector is written whole
                int32_t *p0 = prow - X0;
#pragma unroll
                for (int n = 0; n < NB; ++n) {
                    if (n < NB - 1 || !odd) {
                        if (VEC)
                            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p0 - 7),
                                         "r"(0)
                                         : "memory");
                        else
                            *p0 = 0;
                    }
                    p0 += pns;
                }
            }
            if (st) {
                int32_t *p = prow;
                const int valid = g.w - X0 + 1;
#pragma unroll
                for (int n = 0; n < NB; ++n) {
                    if (n < NB - 1 || !odd) {
                        uint32_t vals[VC];
#pragma unroll
                        for (int k = 0; k < VC; k += 4) {
                            const uint4 t4 = *reinterpret_cast<const uint4 *>(ptop + n * 32 * VC + k);
                            vals[k] = t4.x;
                            vals[k + 1] = t4.y;
                            vals[k + 2] = t4.z;
                            vals[k + 3] = t4.w;
                        }
#pragma unroll
                        for (int k = 0; k < VC; ++k) vals[k] += Lacc[n] + half16(Q[n >> 1][k], n & 1);
                        store_chunk<VC>(p, vals, VEC, valid);
                    }
                    p += pns;
                }
            }
            prow += pp;
        };

        // fused cell grid: lattice row number `li` (row Y0 + li*ls)
        int li = 0;
        int32_t *gptr = KR ? go.grid + (((int64_t)f * go.ncy + (jtop - lag)) * go.ncx + gcol) * g.bins : nullptr;
        const int64_t gstep = (int64_t)go.ncx * g.bins;
        auto lattice = [&]() {
            const int jt = jtop - lag + li;  // grid row whose bottom edge is this lattice row
            const bool emit = lat_lane && jt >= jtop && jt <= jend;
            uint32_t gv[NB];
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                const uint32_t lv = ptop[n * 32 * VC + VC - 1] + Lacc[n] + half16(Q[n >> 1][VC - 1], n & 1);
                const uint32_t r = __shfl_down_sync(FULL, lv, dR);
                uint32_t l = __shfl_up_sync(FULL, lv, 1);
                if (lane == 0) l = Lacc[n];
                const uint32_t hcur = r - l;  // P(Yl, x + cell) - P(Yl, x)
                gv[n] = hcur - ring[n * 32];
#pragma unroll
                for (int q = 0; q + 1 < KR; ++q) ring[(q * NB + n) * 32] = ring[((q + 1) * NB + n) * 32];
                ring[((KR > 0 ? KR - 1 : 0) * NB + n) * 32] = hcur;
            }
            if (emit) {
                if ((g.bins & 3) == 0) {
#pragma unroll
                    for (int n = 0; n + 3 < NB; n += 4)
                        *reinterpret_cast<int4 *>(gptr + n) =
                            make_int4((int)gv[n], (int)gv[n + 1], (int)gv[n + 2], (int)gv[n + 3]);
                } else {
#pragma unroll
                    for (int n = 0; n < NB; ++n)
                        if (n < NB - 1 || !odd) gptr[n] = (int)gv[n];
                }
            }
            gptr += gstep;
            ++li;
        };

        if (active) {
            store_row();
            if (KR) lattice();
        }

        const int8_t *brow = bmf + (int64_t)Y0 * bp + x;
        const bool bin_ok = active && x < g.w;
        const int bvalid = g.w - x;  // bytes of the lane's chunk inside the frame
        auto load_bm = [&](int rel) -> BmWord<VC> {
            BmWord<VC> r;
            const bool ok = bin_ok && Y0 + rel < Ycomp;
            if constexpr (VC == 8) {
                uint2 v = ok ? __ldg(reinterpret_cast<const uint2 *>(brow + (int64_t)rel * bp))
                             : make_uint2(0xffffffffu, 0xffffffffu);
                if (bvalid < 8) {  // bytes past w count nowhere
                    if (bvalid < 4) v.x |= 0xffffffffu << (8 * max(bvalid, 0)), v.y = 0xffffffffu;
                    else v.y |= 0xffffffffu << (8 * (bvalid - 4));
                }
                r.lo = v.x;
                r.hi = v.y;
            } else {
                uint32_t v = ok ? __ldg(reinterpret_cast<const uint32_t *>(brow + (int64_t)rel * bp))
                                : 0xffffffffu;
                if (bvalid < 4) v |= 0xffffffffu << (8 * max(bvalid, 0));
                r.w = v;
            }
            return r;
        };

        BmWord<VC> nxt[G];
#pragma unroll
        for (int i = 0; i < G; ++i) nxt[i] = load_bm(i);
        int latc = ls;  // rows until the next lattice row
        for (int rel = 0; Y0 + rel < Ycomp; rel += G) {
            const int gp = (rel / G) & 1;
            BmWord<VC> bw[G];
            uint32_t ex[G][NW];
            const uint32_t *rt_rd = rowtot + gp * G * nwarp * NWp;
            // ---- phase A: G rows of warp scans (independent) + strip totals
            if (active) {
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    bw[i] = nxt[i];
                    nxt[i] = load_bm(rel + G + i);  // next group in flight during this one
                }
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    uint32_t hb[VC], one[VC];
#pragma unroll
                    for (int k = 0; k < VC; ++k) {
                        const uint32_t v = bw[i].byte(k);
                        hb[k] = v >> 1;
                        one[k] = 1u << ((v & 1u) << 4);
                    }
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        uint32_t tot = 0;
#pragma unroll
                        for (int k = 0; k < VC; ++k) tot += hb[k] == (uint32_t)w ? one[k] : 0u;
                        const uint32_t inc = warp_incl_scan(tot, lane);
                        ex[i][w] = inc - tot;  // strip-exclusive count
                        const uint32_t rt = __shfl_sync(FULL, inc, lo);
                        if (lane == 0) rowtot[((gp * G + i) * nwarp + warp) * NWp + w] = rt;
                    }
                }
            }
            __syncthreads();
            // ---- phase B: carries, accumulate, store, lattice
            if (active) {
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    if (Y0 + rel + i < Ycomp) {
                        const uint32_t *rti = rt_rd + i * nwarp * NWp;
                        uint32_t hb[VC], one[VC];
#pragma unroll
                        for (int k = 0; k < VC; ++k) {
                            const uint32_t v = bw[i].byte(k);
                            hb[k] = v >> 1;
                            one[k] = 1u << ((v & 1u) << 4);
                        }
#pragma unroll
                        for (int w = 0; w < NW; ++w) {
                            uint32_t L = ss ? rdL[(rel + i) * NWp + w] : 0u;
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                if (q < warp) L += rti[q * NWp + w];
                            if (last_warp && lane == 0) wrL[(rel + i) * NWp + w] = L + rti[warp * NWp + w];
                            Lacc[2 * w] += L & 0xffffu;
                            Lacc[2 * w + 1] += L >> 16;
                            uint32_t run = ex[i][w];
#pragma unroll
                            for (int k = 0; k < VC; ++k) {
                                run += hb[k] == (uint32_t)w ? one[k] : 0u;
                                Q[w][k] += run;
                            }
                        }
                        if (Y0 + rel + i + 1 <= Ystore) store_row();
                        if (KR && --latc == 0) {
                            latc = ls;
                            lattice();
                        }
                    }
                }
            }
        }
        __syncthreads();
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

// ---------------------------------------------------------------------------
// Window scores on a regular cell lattice (detector.py:140-154 with block = 1,
// descriptor.py:107-124): the window at lattice origin (iy, ix) reads cells
// (iy + cy*K, ix + cx*K), so scoring is a 2-D correlation of the cell grid
// with the weight tensor.  fp64 throughout (SURVEY: fp32 misses 1e-5 on
// blurred inputs).  Each thread owns SC_TY x SC_TX windows (register tile);
// the CTA streams the grid rows it needs through shared memory as doubles
// (normalised by the per-cell denominator when one is given: the division
// happens once per cell, bit-exact with descriptor.py:119-124).
constexpr int SC_TY = 4, SC_TX = 8, SC_YG = 2;  // windows per thread (y, x); warps per CTA
constexpr int SC_COLS = 32 * SC_TX;              // window columns per CTA

template <int CX>
__global__ void __launch_bounds__(32 * SC_YG)
k_scores_lattice(const int32_t *__restrict__ grid, const double *__restrict__ den, int ncy, int ncx,
                 int bins, int noy, int nox, int cells_y, int K, const double *__restrict__ wts,
                 double bias, double *__restrict__ scores) {
    extern __shared__ double dsm[];
    const int span = SC_COLS + (CX - 1) * K;          // grid columns a CTA touches
    const int spad = span + span / 8 + 1;             // skewed row (1 pad double per 8)
    double *wsm = dsm;                                // [cells_y][bins][CX]
    double *rows = dsm + cells_y * bins * CX;         // [2][bins][spad]
    const int tiles_x = (nox + SC_COLS - 1) / SC_COLS;
    const int tiles_y = (noy + SC_TY * SC_YG - 1) / (SC_TY * SC_YG);
    int bid = blockIdx.x;
    const int tx = bid % tiles_x;
    bid /= tiles_x;
    const int ty = bid % tiles_y;
    const int f = bid / tiles_y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ix0 = tx * SC_COLS, iy0 = ty * SC_TY * SC_YG;
    const int iyw = iy0 + warp * SC_TY;               // this warp's first window row
    const int32_t *gf = grid + (int64_t)f * ncy * ncx * bins;
    const double *df = den ? den + (int64_t)f * ncy * ncx : nullptr;

    // weights, transposed to [cy][n][cx] for broadcast reads
    for (int i = threadIdx.x; i < cells_y * CX * bins; i += blockDim.x) {
        const int n = i % bins, cx = (i / bins) % CX, cy = i / (bins * CX);
        wsm[(cy * bins + n) * CX + cx] = wts[i];
    }
    const int r_first = iy0, r_last = min(iy0 + SC_TY * SC_YG - 1, noy - 1) + (cells_y - 1) * K;
    auto stage = [&](int r, int buf) {
        double *dst = rows + buf * bins * spad;
        const int32_t *src = gf + ((int64_t)r * ncx + ix0) * bins;
        for (int i = threadIdx.x; i < span * bins; i += blockDim.x) {
            const int c = i / bins, n = i % bins;
            double v = 0.0;
            if (ix0 + c < ncx && r < ncy) {
                v = (double)src[i];
                if (df) v = __ddiv_rn(v, df[(int64_t)r * ncx + ix0 + c]);
            }
            dst[n * spad + c + c / 8] = v;
        }
    };
    double acc[SC_TY][SC_TX];
#pragma unroll
    for (int u = 0; u < SC_TY; ++u)
#pragma unroll
        for (int t = 0; t < SC_TX; ++t) acc[u][t] = 0.0;

    stage(r_first, 0);
    __syncthreads();
    const int c0 = lane * SC_TX;  // this thread's first window column within the tile
    for (int r = r_first; r <= r_last; ++r) {
        const int buf = (r - r_first) & 1;
        if (r < r_last) stage(r + 1, buf ^ 1);
        const double *row = rows + buf * bins * spad;
        int cyu[SC_TY];  // weight row each of this thread's window rows takes from grid row r
#pragma unroll
        for (int u = 0; u < SC_TY; ++u) {
            const int d = r - (iyw + u);
            cyu[u] = (d >= 0 && d % K == 0 && d / K < cells_y) ? d / K : -1;
        }
        for (int n = 0; n < bins; ++n) {
            double gs[SC_TX + (CX - 1) * 2];
            const double *rn = row + n * spad;
            // cells this thread's windows touch: c0 .. c0 + SC_TX - 1 + (CX-1)*K
#pragma unroll
            for (int j = 0; j < SC_TX + (CX - 1) * 2; ++j) {
                const int c = c0 + j;
                gs[j] = (j < SC_TX + (CX - 1) * K && c < span) ? rn[c + c / 8] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < SC_TY; ++u) {
                const int cy = cyu[u];
                if (cy < 0) continue;
                const double *wr = wsm + (cy * bins + n) * CX;
                double w[CX];
#pragma unroll
                for (int cx = 0; cx < CX; ++cx) w[cx] = wr[cx];
                if (K == 1) {
#pragma unroll
                    for (int t = 0; t < SC_TX; ++t)
#pragma unroll
                        for (int cx = 0; cx < CX; ++cx) acc[u][t] = fma(w[cx], gs[t + cx], acc[u][t]);
                } else {
#pragma unroll
                    for (int t = 0; t < SC_TX; ++t)
#pragma unroll
                        for (int cx = 0; cx < CX; ++cx) acc[u][t] = fma(w[cx], gs[t + 2 * cx], acc[u][t]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < SC_TY; ++u) {
        const int iy = iyw + u;
        if (iy >= noy) continue;
#pragma unroll
        for (int t = 0; t < SC_TX; ++t) {
            const int ix = ix0 + c0 + t;
            if (ix < nox) scores[((int64_t)f * noy + iy) * nox + ix] = acc[u][t] + bias;
        }
    }
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

inline unsigned blocks_for_warps(int64_t warps) {
    return (unsigned)((warps + (K_THREADS / 32) - 1) / (K_THREADS / 32));
}
inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <int NWB>
void launch_grad_bin(int c, bool counts, const uint8_t *img, int64_t ip, int64_t ics, int64_t ifs,
                     const uint8_t *lut, int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                     const Scratch &sc, cudaStream_t st) {
    const unsigned nb = blocks_for_warps((int64_t)g.n * g.nb1 * g.nc1);
#define LAUNCH(CHv, CNT) \
    k_grad_bin<CHv, NWB, CNT><<<nb, K_THREADS, 0, st>>>(img, ip, ics, ifs, lut, bm, bp, bfs, g, sc)
    if (c == 1) {
        if (counts) LAUNCH(1, true); else LAUNCH(1, false);
    } else {
        if (counts) LAUNCH(3, true); else LAUNCH(3, false);
    }
#undef LAUNCH
}

template <int NW>
void launch_scan(const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    constexpr int NWB = (2 * NW + 3) / 4;
    k_scan_cols<NWB, NW><<<blocks_for((int64_t)g.n * g.Wc, 256), 256, 0, st>>>(g, sc);
}

template <int NW, int KR, int VC, bool VEC>
void launch_planes_vc(const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                      const GridOut &go, const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    const size_t smem = (size_t)k2_smem_words(g, KR) * 4;
    static size_t configured = 0;  // per instantiation
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_planes<NW, KR, VC, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = smem;
    }
    k_planes<NW, KR, VC, VEC><<<(unsigned)((int64_t)g.n * g.nb2), 32 * g.NWARP, smem, st>>>(
        bm, bp, bfs, po, go, g, sc);
}

template <int NW, int KR>
void launch_planes_kr(const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                      const GridOut &go, const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    if constexpr (NW <= 5) {
        if (g.VC == 8) return launch_planes_vc<NW, KR, 8, true>(bm, bp, bfs, po, go, g, sc, st);
    }
    if (po.vec)
        launch_planes_vc<NW, KR, 4, true>(bm, bp, bfs, po, go, g, sc, st);
    else
        launch_planes_vc<NW, KR, 4, false>(bm, bp, bfs, po, go, g, sc, st);
}

template <int NW>
void launch_planes(int kr, const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                   const GridOut &go, const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    if (kr == 0)
        launch_planes_kr<NW, 0>(bm, bp, bfs, po, go, g, sc, st);
    else if (kr == 1)
        launch_planes_kr<NW, 1>(bm, bp, bfs, po, go, g, sc, st);
    else
        launch_planes_kr<NW, 2>(bm, bp, bfs, po, go, g, sc, st);
}

template <int NW>
void launch_counts_from_bm(const int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                           const Scratch &sc, cudaStream_t st) {
    constexpr int NWB = (2 * NW + 3) / 4;
    k_bin_counts<NWB><<<blocks_for_warps((int64_t)g.n * g.nb1 * g.nc1), K_THREADS, 0, st>>>(
        bm, bp, bfs, g, sc);
}

#define HOG_SWITCH_NW(nw, CALL)                                                   \
    switch (nw) {                                                                 \
        case 1: CALL(1); break;                                                   \
        case 2: CALL(2); break;                                                   \
        case 3: CALL(3); break;                                                   \
        case 4: CALL(4); break;                                                   \
        case 5: CALL(5); break;                                                   \
        case 6: CALL(6); break;                                                   \
        case 7: CALL(7); break;                                                   \
        case 8: CALL(8); break;                                                   \
        case 9: CALL(9); break;                                                   \
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

int check_pitch4(const void *p, int64_t pitch, int w, const char *what) {
    if (((uintptr_t)p & 3) != 0 || pitch % 4 != 0 || pitch < round_up(w, 4))
        return fail(HOG_EINVAL, "%s: need 4-byte aligned base and pitch %% 4 == 0, pitch >= %lld (got %lld)",
                    what, (long long)round_up(w, 4), (long long)pitch);
    return HOG_OK;
}

PlaneOut make_po(int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int w) {
    PlaneOut po{pl, pp, pns, pfs, 0};
    po.vec = (((uintptr_t)(pl + 1) & 31) == 0) && pp % 8 == 0 && pns % 8 == 0 && pfs % 8 == 0 &&
             pp >= round_up(w, 8) + 8;
    return po;
}

bool v8_ok(const PlaneOut &po, const int8_t *bm, int64_t bp, int64_t bfs) {
    return po.vec && ((uintptr_t)bm & 7) == 0 && bp % 8 == 0 && bfs % 8 == 0;
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
    TileGeom g = make_geom(n, h, w, bins, false, 0, 0, v8_ok(po, bm, bp, bfs));
    Scratch sc{};
    size_t need = carve(g, nullptr, nullptr);
    if (scratch == nullptr || sbytes < need)
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", need, sbytes);
    carve(g, scratch, &sc);
    GridOut go{nullptr, 4, 4, 1, 1};
#define CALL(NWv)                                       \
    launch_counts_from_bm<NWv>(bm, bp, bfs, g, sc, st); \
    launch_scan<NWv>(g, sc, st);                        \
    launch_planes<NWv>(0, bm, bp, bfs, po, go, g, sc, st);
    HOG_SWITCH_NW(g.NW, CALL)
#undef CALL
    return check_launch("hog_integral");
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char *hog_version(void) { return "hogb200 1.2 sm_100a"; }

const char *hog_last_error(void) { return g_err.c_str(); }

int64_t hog_plane_pitch(int w) { return round_up((int64_t)w, 8) + 8; }

int hog_grad_bin(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                 int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp, int64_t bfs,
                 hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (c != 1 && c != 3) return fail(HOG_EINVAL, "channels must be 1 or 3, got %d", c);
    if ((e = check_pitch4(img, ip, w, "image")) || (e = check_pitch4(bm, bp, w, "binmap"))) return e;
    if (!img || !lut || !bm) return fail(HOG_EINVAL, "null buffer");
    TileGeom g = make_geom(n, h, w, bins, false, 0, 0, false);
    Scratch sc{};
    launch_grad_bin<1>(c, false, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, (cudaStream_t)stream);
    return check_launch("hog_grad_bin");
}

size_t hog_scratch_bytes(int n, int h, int w, int bins, int stride, int cell) {
    if (n < 1 || h < 1 || w < 1 || bins < 1) return 0;
    bool fused = stride > 0 && cell > 0;
    size_t m = 0;
    for (int v8 = 0; v8 < 2; ++v8) {
        size_t a = carve(make_geom(n, h, w, bins, fused, stride, cell, v8), nullptr, nullptr);
        size_t b = carve(make_geom(n, h, w, bins, false, 0, 0, v8), nullptr, nullptr);
        m = a > m ? a : m;
        m = b > m ? b : m;
    }
    return m;
}

int hog_integral(const int8_t *bm, int n, int h, int w, int64_t bp, int64_t bfs, int bins,
                 int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, void *scratch,
                 size_t sbytes, hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if ((e = check_pitch4(bm, bp, w, "binmap"))) return e;
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
    if ((e = check_pitch4(img, ip, w, "image")) || (e = check_pitch4(bm, bp, w, "binmap"))) return e;
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
    PlaneOut po = make_po(pl, pp, pns, pfs, w);
    TileGeom g = make_geom(n, h, w, bins, kr > 0, stride, cell, v8_ok(po, bm, bp, bfs));
    Scratch sc{};
    size_t need = carve(g, nullptr, nullptr);
    if (scratch == nullptr || sbytes < need)
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", need, sbytes);
    carve(g, scratch, &sc);
    GridOut go{grid, kr ? stride : 4, kr ? cell : 4, kr ? ncx : 1, kr ? ncy : 1};
    auto mark = [&](int i) {
        if (stage_events && stage_events[i]) cudaEventRecord((cudaEvent_t)stage_events[i], st);
    };
#define CALL(NWv)                                                                           \
    mark(0);                                                                                \
    launch_grad_bin<(2 * NWv + 3) / 4>(c, true, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st); \
    mark(1);                                                                                \
    launch_scan<NWv>(g, sc, st);                                                            \
    mark(2);                                                                                \
    launch_planes<NWv>(kr, bm, bp, bfs, po, go, g, sc, st);                                 \
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

int hog_scores_lattice(const int32_t *grid, const double *den, int n, int ncy, int ncx, int bins,
                       int noy, int nox, int cells_x, int cells_y, int k, const double *wts,
                       double bias, double *scores, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || bins < 1 || !grid || !wts || !scores)
        return fail(HOG_EINVAL, "bad arguments");
    if (k != 1 && k != 2) return fail(HOG_EINVAL, "lattice step ratio must be 1 or 2, got %d", k);
    if (cells_x != 8) return fail(HOG_EINVAL, "hog_scores_lattice is built for 8 cells across, got %d", cells_x);
    if ((int64_t)(noy - 1) + (int64_t)(cells_y - 1) * k >= ncy || (int64_t)(nox - 1) + 7 * k >= ncx)
        return fail(HOG_EINVAL, "window grid exceeds the cell lattice");
    const int span = SC_COLS + 7 * k;
    const size_t smem = sizeof(double) * ((size_t)cells_y * bins * 8 + 2 * (size_t)bins * (span + span / 8 + 1));
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_scores_lattice<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    const int64_t blocks = (int64_t)n * ((noy + SC_TY * SC_YG - 1) / (SC_TY * SC_YG)) *
                           ((nox + SC_COLS - 1) / SC_COLS);
    k_scores_lattice<8><<<(unsigned)blocks, 32 * SC_YG, smem, (cudaStream_t)stream>>>(
        grid, den, ncy, ncx, bins, noy, nox, cells_y, k, wts, bias, scores);
    return check_launch("hog_scores_lattice");
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
