// hog_common.cuh -- types, device helpers and launcher declarations shared by
// the libhogb200 translation units (k_bin.cu, k_planes_*.cu, k_window.cu,
// hog_abi.cu).  See hog_abi.cu for the design overview.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/hogb200.h"

// Measured-and-lost variants (TMA bulk-store plane path, binning fused into
// the plane kernel with decoupled look-back, the first lattice score kernel)
// are compiled only into experiment builds (tools/build_variant.sh passes
// -DHOGB200_VARIANTS=1); the product library holds the measured-best paths.
#ifndef HOGB200_VARIANTS
#define HOGB200_VARIANTS 0
#endif

namespace hogb200 {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LUT_SIDE = 511;
constexpr int K_THREADS = 128;      // 4 independent warps per CTA
constexpr int MAX_FUSED_BINS = 18;  // NW <= 9 packed words
constexpr int CHUNK = 128;          // k_grad_bin columns per warp (32 lanes x 4)

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// Geometry shared by k_grad_bin / k_bin_counts / k_scan_cols / k_planes.
struct TileGeom {
    int n, h, w, bins;
    int R;      // rows per band (multiple of the lattice step when the grid is fused)
    int R1, S1; // k_grad_bin / k_bin_counts sub-bands: R1 = R / S1 pixel rows each
    int Ws;     // plane columns per k_planes strip (<= 128, multiple of 8)
    int ns;     // strips per frame
    int nb1;    // pixel sub-bands: ceil(h / R1)    (k_grad_bin tiles)
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
    int ht, hb; // slab mode: the frame continues above row 0 / below row h-1 (rows -1 / h are
                // readable halo rows, and rows 0 / h-1 are binned rather than border NO_BIN)
    int PREG;   // k_planes keeps the band's top row in registers (k2_maxt preg variant)
    int TMA;    // plane rows staged in shared memory and written by TMA bulk stores
    int RING;   // TMA: staged plane rows in flight (ring slots)
    int SEGW;   // TMA: staged columns per bin row = NWARP*Ws + 8 (32-B aligned front pad)
    int RB;     // whole plane rows staged in shared memory, one bulk copy per row (k_planes RB)
    int RBP;    // RB: words per bin row in the slot (= the plane pitch pns)
    int NOSCAN; // k_planes sums the sub-band counts above its band itself (no k_scan_cols launch, no V)
};

// Scratch arrays (device), carved from the caller's scratch buffer.
struct Scratch {
    uint32_t *C;      // [n][nb2][Wc][NWB]  bin counts per (pixel band, column), u8x4
    uint32_t *V;      // [n][nb2][Wc][NWp]  counts above each plane band, u16x2
                      //   (fused: counts above band b+1, published by band b)
    uint32_t *flags;  // [n][nb2] + 1 ticket: fused look-back state (zeroed per launch)
    const int32_t *base;  // slab mode: [n][bins][w] column counts above plane row 0 (or null)
    int64_t base_fs;      //   frame stride of base (elements)
};


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
    int32_t *grid;  // int32 cells, or uint8 cells when u8 (addressed in elements either way)
    int s, cell, ncx, ncy;
    int u8;
};

#ifndef K2_GN
#define K2_GN 4
#endif
constexpr int K2_G = K2_GN;  // rows per phase-A/phase-B group (NW < 6; experiment knob K2_GN)
#ifndef K2_G8
#define K2_G8 2  // the same for 8 columns per lane (c4: 1.871 -> 1.857 ms against 4; c2's 4-column variant loses 3.8 % at 2)
#endif
#ifndef K2_GW
#define K2_GW 2  // the same for NW >= 6 (<= K2_G: the shared layout is sized for K2_G); c5 61.6 -> 61.2 ms against 4
#endif
#ifndef K2_RB_ROWS
#define K2_RB_ROWS 2  // RB: plane rows per staging slot (one bulk copy and one barrier per slot)
#endif
#ifndef K2_RB_SLOTS
#define K2_RB_SLOTS (K2_RB_ROWS == 1 ? 3 : 2)  // RB: staging slots in flight
#endif
#ifndef K2_RB_DECOUPLED
#define K2_RB_DECOUPLED 0  // RB: 1 = producer/consumer named barriers instead of a CTA barrier per row (c2 -0.8 %, shard +1.2 %)
#endif
#ifndef K2_RB_P32
#define K2_RB_P32 0  // RB: 1 = full 32-bit plane values in registers (k_planes FP); measured 2 % slower on c2
#endif
#ifndef K2_STORE_HINT
#define K2_STORE_HINT 0  // plane stores with an L2 evict-first hint (experiment knob)
#endif
#ifndef K2_PAIR256
#define K2_PAIR256 0  // 256-bit plane stores by lane pairs (k_planes PAIR; experiment knob)
#endif
#ifndef K2_FASTGROUP
#define K2_FASTGROUP 1  // guard-free code path for full row groups (k_planes.cuh)
#endif

// Max threads per k_planes CTA (NWARP compute warps [+ the TMA store warp]),
// i.e. the register budget at two CTAs per SM: 256 threads -> 128 registers,
// 192 -> 168.  Measured on B200 (tools/ab_lib.sh, K2_MAXT variants): the
// 8-column-per-lane and >= 10-bin variants spill at 128 registers and run
// 4-29 % faster with 168 (c3, c4, c5); the c2 variant (4 columns, 8 bins) is
// 4 % faster at 128.
#ifndef K2_PTOP_REG
#define K2_PTOP_REG 1
#endif
#ifndef K2_MINB
#define K2_MINB 2
#endif
#ifndef K2_MAXT_WIDE
#define K2_MAXT_WIDE 192  // CTA size bound of the wide variants (NW >= 6; experiment knob)
#endif
#ifndef K2_MINB_WIDE
#define K2_MINB_WIDE K2_MINB
#endif
#ifndef K2_MAXT_MID
#define K2_MAXT_MID 192  // the same for 9-10 bins at 4 columns per lane (c3)
#endif
#ifndef K2_MINB_MID
#define K2_MINB_MID K2_MINB
#endif
// Plane-kernel CTA size bound.  preg: the small variants (<= 8 bins, 4 columns
// per lane) keep the band's top row in 32 registers instead of shared memory,
// bounded at 192 threads (170 registers at 2 CTAs/SM); chosen when a band's
// strips fit 6 warps (make_geom), else the 256-thread variant runs.
__host__ __device__ constexpr int k2_maxt(int nw, int vc, bool preg = false) {
    return nw >= 6 ? K2_MAXT_WIDE : (nw == 5 && vc == 4) ? K2_MAXT_MID : (vc == 8 || nw >= 5 || preg) ? 192 : 256;
}
// resident CTAs per SM the register budget is set for (__launch_bounds__ second argument)
__host__ __device__ constexpr int k2_minb(int nw, int vc) {
    return nw >= 6 ? K2_MINB_WIDE : (nw == 5 && vc == 4) ? K2_MINB_MID : K2_MINB;
}

// Inputs of the fused plane kernel (binning inside k_planes, band carries by
// decoupled look-back instead of k_grad_bin counts + k_scan_cols).
struct FusedIn {
    const uint8_t *img;
    int64_t ip, ics, ifs;
    const uint8_t *lut;
    uint32_t *flags;   // [n][nb2]: 0 none, 1 band aggregate published, 2 inclusive published
    uint32_t *ticket;  // CTA ticket counter (zeroed with the flags before every launch)
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_gpu(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// shared-memory carve-up of one k_planes CTA (32-bit words, every array 16-B aligned)
struct K2Smem {
    int bar, rowtot, Lsup, vtot, Tsup, ptop, ring, stage, total;
};

__host__ __device__ inline int k2_r4(int v) { return (v + 3) & ~3; }

__host__ __device__ inline K2Smem k2_smem(const TileGeom &g, int kr) {
    const int NB = 2 * g.NW;
    K2Smem m;
    m.bar = 0;                                                   // TMA: u64 full[RING], empty[RING]
    m.rowtot = m.bar + k2_r4(g.TMA ? 4 * g.RING : 0);            // [2][G][NWARP][NWp]
    m.Lsup = m.rowtot + k2_r4(2 * K2_G * g.NWARP * g.NWp);       // [2][Lrows][NWp]
    m.vtot = m.Lsup + k2_r4(2 * g.Lrows * g.NWp);                // [NWARP][NB]
    m.Tsup = m.vtot + k2_r4(g.NWARP * NB);                       // [2][NB]
    m.ptop = m.Tsup + k2_r4(2 * NB);                             // [NWARP][NB][32][VC]
    // (the register top-row variant keeps ptop in registers: no shared copy)
    m.ring = m.ptop + ((g.PREG && !g.TMA) ? 0 : k2_r4(g.NWARP * NB * 32 * g.VC));  // [NWARP][KR][NB][32]
    m.stage = m.ring + k2_r4(g.NWARP * kr * NB * 32);             // TMA: [RING][bins][SEGW]
    m.total = m.stage + (g.TMA ? g.RING * g.bins * g.SEGW : 0) +
              (g.RB ? K2_RB_SLOTS * K2_RB_ROWS * g.bins * g.RBP : 0);
    return m;
}

__host__ __device__ inline int k2_smem_words(const TileGeom &g, int kr) { return k2_smem(g, kr).total; }


// ---------------------------------------------------------------------------
// Device helpers

// mbarrier + TMA bulk-store primitives (k_planes store pipeline)
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(b)), "r"(parity)
            : "memory");
    } while (!done);
}
// waiter that backs off, so a spinning store warp does not take issue slots
// from the compute warps on its scheduler
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *b, uint32_t parity) {
    uint32_t done;
    for (;;) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_addr(b)), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(100);
    }
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
#if K2_STORE_HINT
    // planes are written once and never re-read by the pipeline: first to leave L2
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_addr(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_addr(ssrc)), "r"(bytes)
                 : "memory");
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// generic-proxy shared-memory writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// barrier over the first `threads` threads of the CTA (the compute warps)
__device__ __forceinline__ void named_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t t = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// byte k of v, zero-extended: one PRMT (the shift + mask form compiles to two ops)
__device__ __forceinline__ uint32_t byte_of(uint32_t v, int k) { return __byte_perm(v, 0u, 0x4440u | (uint32_t)k); }

// a << s with PTX shl semantics: shift amounts >= 32 (including "negative"
// ones, which are huge unsigned) give 0.  One-hot packing without compares:
// bin v lands in word w at bit offset 8v - 32w (u8x4) or 16v - 32w (u16x2)
// exactly when that offset is in [0, 32); NO_BIN (0xFF) lands nowhere.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t a, uint32_t s) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(s));
    return r;
}

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
        const uint32_t s = byte_of(bins4, k) << 3;
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] += shl_clamp(1u, s - 32u * w);
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


// The dynamic shared-memory opt-in (cudaFuncSetAttribute) is per device: a
// launcher remembers, per device, the largest size it has set for its kernel.
constexpr int HOG_MAX_DEVICES = 64;
inline bool smem_optin_needed(size_t (&done)[HOG_MAX_DEVICES], size_t smem) {
    if (smem <= 48 * 1024) return false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= HOG_MAX_DEVICES) return true;
    if (smem <= done[dev]) return false;
    done[dev] = smem;
    return true;
}

inline unsigned blocks_for_warps(int64_t warps) {
    return (unsigned)((warps + (K_THREADS / 32) - 1) / (K_THREADS / 32));
}
inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// ---- launchers (defined in the kernel translation units) -------------------
// k_bin.cu
void launch_grad_bin(int nwb, int c, bool counts, const uint8_t *img, int64_t ip, int64_t ics,
                     int64_t ifs, const uint8_t *lut, int8_t *bm, int64_t bp, int64_t bfs,
                     const TileGeom &g, const Scratch &sc, cudaStream_t st);
// k_bin_oct.cu: table-free binning for N_b in {4, 8} (false: bins not handled)
bool launch_grad_bin_oct(int bins, int c, bool counts, const uint8_t *img, int64_t ip, int64_t ics,
                         int64_t ifs, int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                         const Scratch &sc, cudaStream_t st);
bool launch_lut_proof(int bins, const uint8_t *lut, unsigned long long *mismatches, cudaStream_t st);
// hog_abi.cu: has this (device, table, bins) passed k_lut_proof?  Proves it on
// first use (synchronising st) unless st is capturing a graph.
bool lut_proven(const uint8_t *lut, int bins, cudaStream_t st);
void launch_counts_from_bm(int nw, const int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                           const Scratch &sc, cudaStream_t st);
void launch_scan(int nw, const TileGeom &g, const Scratch &sc, cudaStream_t st);
void launch_column_counts(const int8_t *bm, int64_t bp, int64_t bfs, int n, int rows, int w, int bins,
                          int32_t *out, cudaStream_t st);
// k_planes_*.cu
void launch_planes_a(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st);
void launch_planes_b(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st);
void launch_planes_c(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st);
void launch_planes_d(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st);
// ch: 0 = bin map given (k_grad_bin + k_scan_cols ran), 1/3 = fused binning + look-back
inline void launch_planes(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                          const PlaneOut &po, const GridOut &go, const TileGeom &g,
                          const Scratch &sc, const FusedIn &fi, cudaStream_t st) {
    if (nw <= 3) launch_planes_a(nw, kr, ch, bm, bp, bfs, po, go, g, sc, fi, st);
    else if (nw <= 5) launch_planes_b(nw, kr, ch, bm, bp, bfs, po, go, g, sc, fi, st);
    else if (nw <= 7) launch_planes_c(nw, kr, ch, bm, bp, bfs, po, go, g, sc, fi, st);
    else launch_planes_d(nw, kr, ch, bm, bp, bfs, po, go, g, sc, fi, st);
}
// k_window.cu
void launch_bin_offset(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int b0,
                       int8_t *out, int64_t op, int64_t ofs, cudaStream_t st);
void launch_cell_grid(const int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int n, int bins,
                      const int32_t *cxs, int ncx, const int32_t *cys, int ncy, int cell,
                      int32_t *grid, cudaStream_t st);
void launch_cell_norm(const int32_t *grid, int64_t ncells_total, int bins, int norm,
                      double eps_term, double *den, cudaStream_t st);
void launch_window_l2(const void *grid, int elem_bytes, int n, int ncy, int ncx, int bins,
                      const int32_t *row_idx, int noy, const int32_t *col_idx, int nox, int cells_x,
                      int cells_y, int k, double eps_term, int32_t *sq, double *norms, cudaStream_t st);
void launch_window_features(const int32_t *grid, int n, int ncy, int ncx, int bins,
                            const int32_t *row_idx, int noy, const int32_t *col_idx, int nox,
                            int cells_x, int cells_y, int block, int bstride, int norm,
                            double eps_term, const double *wts, double bias, double *scores,
                            double *desc, cudaStream_t st);
void launch_scores_lattice(const int32_t *grid, const double *den, int n, int ncy, int ncx,
                           int bins, int noy, int nox, int cells_y, int k, const double *wts,
                           double bias, double *scores, cudaStream_t st);
// k_rect.cu
void launch_integral16(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int bins,
                       uint16_t *pl, int64_t pp, int64_t pns, int64_t pfs, cudaStream_t st);
void launch_rect_hist(const void *pl, int elem_bytes, int64_t pp, int64_t pns, int bins,
                      const int32_t *rects, int k, int64_t *out, cudaStream_t st);
// k_detect.cu
struct DetMap;
size_t det_scratch_bytes(int n, int64_t m);
size_t nms_scratch_bytes(int n);
int launch_nms(const int32_t *boxes, const double *scores, const double *scales, int n, double thr,
               int32_t *keep, int32_t *keep_count, void *scratch, size_t sbytes, cudaStream_t st);
int launch_nms_f64(const double *boxes, const double *scores, const double *scales, int n, double thr,
                   int32_t *keep, int32_t *keep_count, void *scratch, size_t sbytes, cudaStream_t st);
void launch_detect_abi(const double *scores, int n, int noy, int nox, double thr, const int32_t *oxs,
                       const int32_t *oys, double scale, int ww, int wh, int clamp_w, int clamp_h,
                       int cap, int32_t *boxes, double *out_scores, int64_t *out_window,
                       int32_t *count, void *scratch, cudaStream_t st);
// k_scores.cu
void launch_scores_rows(const int32_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                        int cells_y, int k, const double *wts, double bias, double *scores,
                        cudaStream_t st);
void launch_scores_rows_u8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy,
                           int nox, int cells_y, int k, const double *wts, double bias,
                           double *scores, cudaStream_t st);
int scores_i8_ks(int bins);
void launch_scores_i8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                      const void *wfrag, int digits, double scale, double bias, double *scores,
                      cudaStream_t st);
void launch_resize(const uint8_t *src, int n, int c, int h, int w, int64_t sp, int64_t scs,
                   int64_t sfs, int nh, int nw, double ry, double rx, uint8_t *dst, int64_t dp,
                   int64_t dcs, int64_t dfs, cudaStream_t st);

}  // namespace hogb200
