// k_bin.cu -- K1: gradient + LUT binning with per-(band, column) bin counts,
// and the carry scan that turns the counts into column counts above every
// band.  gradient.py:95-121; integral.py:58-87 (the carries of the scan).
#include "hog_common.cuh"

namespace hogb200 {

#ifndef K1_UNROLL
#define K1_UNROLL 1
#endif
constexpr int K1U = K1_UNROLL;  // rows of k_grad_bin's row loop unrolled together

// Bit-sliced per-(sub-band, column) counts for >= 9 bins (NWB >= 3): a pixel's bin becomes
// a one-hot word (bit n = [bin == n], one SHL), the rows of a column are summed by
// carry-save adders into 8 bit planes (plane j bit n = bit j of the count of bin n; counts
// <= R1 <= 240), and the planes are turned into the u8x4 words of Scratch::C by 8x8 bit
// transposes once per sub-band.  ~7 instructions per pixel for 18 bins against 16 for the
// packed-byte adds (count_cols: one shifted add per u8x4 word and pixel).  Measured
// bit-exact and SLOWER (c3 binning 0.183 -> 0.235 ms, c5 +1.3 ms): 72 registers instead
// of 56 cost two resident CTAs per SM, and this kernel waits on the table gathers, not on
// issue slots.  Experiment knob, off.
#ifndef K1_SLICED
#define K1_SLICED 0
#endif

__device__ __forceinline__ void csa3(uint32_t &sum, uint32_t &carry, uint32_t a, uint32_t b, uint32_t c) {
    sum = a ^ b ^ c;
    carry = (a & b) | (c & (a ^ b));
}

// 8x8 bit transpose: out byte n bit j = in byte j bit n
__device__ __forceinline__ uint64_t bit_tr8x8(uint64_t x) {
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x = x ^ t ^ (t << 28);
    return x;
}

// ---------------------------------------------------------------------------
// K1: gradient + LUT binning (gradient.py:95-121), optionally counting bins
// per (band, column) for k_scan_cols.  One warp = R rows x 128 columns of
// one frame; lane L owns pixel columns x0+4L .. x0+4L+3 and slides a
// three-row window down the band, two rows of loads in flight; left/right
// neighbours come from the adjacent lanes by shuffle.

// resident CTAs per SM the register budget is set for (experiment knob; 1 = the compiler's choice)
#ifndef K1_MINB
#define K1_MINB 1
#endif

template <int CH, int NWB, bool COUNTS>
__global__ void __launch_bounds__(K_THREADS, K1_MINB)
k_grad_bin(const uint8_t *__restrict__ img, int64_t ip, int64_t ics, int64_t ifs,
           const uint8_t *__restrict__ lut, int8_t *__restrict__ bm, int64_t bp, int64_t bfs,
           TileGeom g, Scratch sc) {
    // per-lane column counters: cnt[bin (NB+1: slot NB = no bin)][column k][lane]
    extern __shared__ uint32_t kbsm[];
    constexpr int NB4 = 4 * NWB;  // bins rounded up to whole u8x4 words
    const int64_t wid = warp_id();
    if (wid >= (int64_t)g.n * g.nb1 * g.nc1) return;
    // 32-bit index math (units < 2^31 for every batch the ABI accepts in practice;
    // 64-bit divisions are a software call)
    int chunk, b, f;
    if (wid < ((int64_t)1 << 31)) {
        const uint32_t w32 = (uint32_t)wid, q = w32 / (uint32_t)g.nc1;
        chunk = (int)(w32 - q * (uint32_t)g.nc1);
        b = (int)(q % (uint32_t)g.nb1);
        f = (int)(q / (uint32_t)g.nb1);
    } else {
        chunk = (int)(wid % g.nc1);
        b = (int)((wid / g.nc1) % g.nb1);
        f = (int)(wid / ((int64_t)g.nc1 * g.nb1));
    }
    const int lane = threadIdx.x & 31;
    const int x = chunk * CHUNK + 4 * lane;
    const bool inx = x < g.w;
    const int y0 = b * g.R1, y1 = min(y0 + g.R1, g.h);
    // lanes past the frame read (and discard) the last word of the row
    const int xl = inx ? x : ((g.w - 1) & ~3);
    const uint8_t *col = img + (int64_t)f * ifs + xl;
    const uint8_t *lut0 = lut + (255 * LUT_SIDE + 255);  // lut0[dx*511 + dy]
    uint32_t *cnt = kbsm + (threadIdx.x >> 5) * (NB4 + 1) * 4 * 32 + lane;
    const int nbin = g.bins;
#ifndef K1_SMEM_COUNTS
#define K1_SMEM_COUNTS 0
#endif
    uint32_t cc[4][NWB];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int w = 0; w < NWB; ++w) cc[k][w] = 0;
    if (COUNTS && K1_SMEM_COUNTS) {
#pragma unroll
        for (int i = 0; i < (NB4 + 1) * 4; ++i) cnt[i * 32] = 0;
    }

    // bytes of this lane's 4 columns that are interior pixels (1 <= x <= w-2)
    uint32_t valid = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (x + k >= 1 && x + k <= g.w - 2) valid |= 0xffu << (8 * k);
    // neighbour byte outside the lane's word: left of lane 0, right of lane 31
    const int eoff = lane == 0 ? -1 : 4;
    const bool has_edge = (lane == 0 && x >= 1) || (lane == 31 && x + 4 < g.w);
    // rows -1 / h exist in slab mode (g.ht / g.hb); otherwise reads clamp to the frame
    auto rowp = [&](int y) { return col + (int64_t)min(max(y, -g.ht), g.h - 1 + g.hb) * ip; };

    // rows y-1 (r0), y (r1), y+1 (r2); e1/e2: edge bytes of rows y, y+1
    uint32_t r0[CH], r1[CH], r2[CH], e1[CH], e2[CH];
    {
        const uint8_t *pa = rowp(y0 - 1), *pb = rowp(y0), *pc = rowp(y0 + 1);
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            r0[ch] = __ldg(reinterpret_cast<const uint32_t *>(pa + ch * ics));
            r1[ch] = __ldg(reinterpret_cast<const uint32_t *>(pb + ch * ics));
            r2[ch] = __ldg(reinterpret_cast<const uint32_t *>(pc + ch * ics));
            e1[ch] = has_edge ? (uint32_t)__ldg(pb + ch * ics + eoff) : 0u;
            e2[ch] = has_edge ? (uint32_t)__ldg(pc + ch * ics + eoff) : 0u;
        }
    }
    int8_t *bout = bm + (int64_t)f * bfs + (int64_t)y0 * bp + x;
    const uint8_t *pd = rowp(y0 + 2);  // row y+2, clamped to the last row

    // one row: gradients, table gather, bin-map store, window rotation; returns the 4 bin bytes
    auto row = [&](int y) -> uint32_t {
        // row y+2 in flight while row y is binned
        uint32_t r3[CH], e3[CH];
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            r3[ch] = __ldg(reinterpret_cast<const uint32_t *>(pd + ch * ics));
            e3[ch] = has_edge ? (uint32_t)__ldg(pd + ch * ics + eoff) : 0u;
        }
        if (y + 3 < g.h + g.hb) pd += ip;
        uint32_t bins4 = 0xffffffffu;
        if ((y > 0 || g.ht) && (y < g.h - 1 || g.hb)) {  // frame border rows are NO_BIN
            int bdx[4], bdy[4], bmag[4];
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
                        if (ch == 0 || mag > bmag[k]) bdx[k] = dx, bdy[k] = dy, bmag[k] = mag;
                    }
                }
            }
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldg(lut0 + (int64_t)(bdx[k] * LUT_SIDE + bdy[k]));
            bins4 = __byte_perm(__byte_perm(v[0], v[1], 0x0040), __byte_perm(v[2], v[3], 0x0040), 0x5410);
            bins4 = (bins4 & valid) | ~valid;
        }
        if (inx) *reinterpret_cast<uint32_t *>(bout) = bins4;
        bout += bp;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            r0[ch] = r1[ch];
            r1[ch] = r2[ch];
            r2[ch] = r3[ch];
            e1[ch] = e2[ch];
            e2[ch] = e3[ch];
        }
        return bins4;
    };
    constexpr bool SL = COUNTS && K1_SLICED && !K1_SMEM_COUNTS && NWB >= 3;
    uint32_t qp[SL ? 8 : 1][SL ? 4 : 1];  // bit planes of the column counts (qp[0..2] = ones, twos, fours)
    if constexpr (SL) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) qp[j][k] = 0;
        uint32_t t2a[4] = {0, 0, 0, 0}, t4a[4] = {0, 0, 0, 0};
        // row pairs; rows past y1 add nothing and flush the pending carries (a multiple of 8 rows)
        const int npairs = ((y1 - y0 + 7) >> 3) << 2;
        int y = y0;
#pragma unroll 1
        for (int pr = 0; pr < npairs; ++pr, y += 2) {
            const uint32_t ba = y < y1 ? row(y) : 0xffffffffu;
            const uint32_t bb = y + 1 < y1 ? row(y + 1) : 0xffffffffu;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t oa = shl_clamp(1u, byte_of(ba, k)), ob = shl_clamp(1u, byte_of(bb, k));
                uint32_t c2;
                csa3(qp[0][k], c2, qp[0][k], oa, ob);
                if ((pr & 1) == 0) {
                    t2a[k] = c2;
                } else {
                    uint32_t c4;
                    csa3(qp[SL ? 1 : 0][k], c4, qp[SL ? 1 : 0][k], t2a[k], c2);
                    if ((pr & 2) == 0) {
                        t4a[k] = c4;
                    } else {
                        uint32_t c;
                        csa3(qp[SL ? 2 : 0][k], c, qp[SL ? 2 : 0][k], t4a[k], c4);
#pragma unroll
                        for (int j = 3; j < 8; ++j) {
                            const uint32_t q = qp[SL ? j : 0][k];
                            qp[SL ? j : 0][k] = q ^ c;
                            c &= q;
                        }
                    }
                }
            }
        }
        // planes -> C[f][b][x+k][w] (u8x4 of bins 4w..4w+3): byte group g8 holds bins 8 g8..8 g8+7
        uint32_t *cp = sc.C + (((int64_t)f * g.nb1 + b) * g.Wc + x) * NWB;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int g8 = 0; g8 < (NWB + 1) / 2; ++g8) {
                const uint32_t sel = 0x40u + 0x11u * g8;  // result bytes 0, 1 = byte g8 of a, byte g8 of b
                const uint32_t lo = __byte_perm(__byte_perm(qp[0][k], qp[SL ? 1 : 0][k], sel),
                                                __byte_perm(qp[SL ? 2 : 0][k], qp[SL ? 3 : 0][k], sel), 0x5410);
                const uint32_t hi = __byte_perm(__byte_perm(qp[SL ? 4 : 0][k], qp[SL ? 5 : 0][k], sel),
                                                __byte_perm(qp[SL ? 6 : 0][k], qp[SL ? 7 : 0][k], sel), 0x5410);
                const uint64_t t = bit_tr8x8(((uint64_t)hi << 32) | lo);
                cp[k * NWB + 2 * g8] = (uint32_t)t;
                if (2 * g8 + 1 < NWB) cp[k * NWB + 2 * g8 + 1] = (uint32_t)(t >> 32);
            }
        }
    } else {
        // unrolled so the LUT gathers of consecutive rows overlap (the kernel waits
        // on gather latency, not on issue)
#pragma unroll K1U
        for (int y = y0; y < y1; ++y) {
            const uint32_t bins4 = row(y);
            (void)bins4;
            if (COUNTS) {
#if K1_SMEM_COUNTS
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int slot = min((int)byte_of(bins4, k), nbin);  // NO_BIN -> spare slot
                    cnt[(slot * 4 + k) * 32] += 1;
                }
#else
                count_cols<NWB>(bins4, cc);
#endif
            }
        }
    }
    if (COUNTS && !K1_SMEM_COUNTS && !SL) store_cols<NWB>(g, sc, f, b, x, cc);
    if (COUNTS && K1_SMEM_COUNTS) {
        // C[f][b][x+k][w]: bins 4w..4w+3 of column x+k as u8x4 (counts <= R <= 240)
        uint32_t *cp = sc.C + (((int64_t)f * g.nb1 + b) * g.Wc + x) * NWB;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int w = 0; w < NWB; ++w) {
                uint32_t word = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int n = 4 * w + j;
                    if (n < nbin) word |= cnt[(n * 4 + k) * 32] << (8 * j);
                }
                cp[k * NWB + w] = word;
            }
        }
    }
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
    const int y0 = b * g.R1, y1 = min(y0 + g.R1, g.h);
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
    if (sc.base && x < g.w) {  // slab mode: counts above the slab's first plane row
        const int32_t *bs = sc.base + (int64_t)f * sc.base_fs + x;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t lo = (uint32_t)bs[(int64_t)(2 * w) * g.w];
            const uint32_t hi = 2 * w + 1 < g.bins ? (uint32_t)bs[(int64_t)(2 * w + 1) * g.w] : 0u;
            run[w] = lo | (hi << 16);
        }
    }
    // C and V never alias.  The sub-band counts are loaded 8 at a time, all
    // issued before any is used, so a column's chain over the bands waits on
    // one memory latency per 8 sub-bands (a single small frame -- config c1 --
    // spent 18 us here with one dependent load per sub-band)
    const uint32_t *__restrict__ Cf = sc.C + (int64_t)f * g.nb1 * g.Wc * NWB + (int64_t)x * NWB;
    uint32_t *__restrict__ Vf = sc.V + (int64_t)f * g.nb2 * g.Wc * g.NWp + (int64_t)x * g.NWp;
    auto store_v = [&](int b) {
        uint4 *vp = reinterpret_cast<uint4 *>(Vf + (int64_t)b * g.Wc * g.NWp);
#pragma unroll
        for (int q = 0; q < (NW + 3) / 4; ++q)  // 16-B stores; words past NW are zero padding
            vp[q] = make_uint4(run[4 * q], 4 * q + 1 < NW ? run[4 * q + 1] : 0u,
                               4 * q + 2 < NW ? run[4 * q + 2] : 0u, 4 * q + 3 < NW ? run[4 * q + 3] : 0u);
    };
    constexpr int SB = 8;
    int nextb = 0, nexts = 0;  // next plane band whose carry is due, and its first sub-band
    for (int s0 = 0; s0 < g.nb1; s0 += SB) {
        uint32_t c8[SB][NWB];
#pragma unroll
        for (int i = 0; i < SB; ++i)
#pragma unroll
            for (int w = 0; w < NWB; ++w)
                c8[i][w] = s0 + i < g.nb1 ? __ldg(Cf + (int64_t)(s0 + i) * g.Wc * NWB + w) : 0u;
#pragma unroll
        for (int i = 0; i < SB; ++i) {
            const int s = s0 + i;
            if (s == nexts && nextb < g.nb2) {  // plane band nextb covers sub-bands from s on
                store_v(nextb++);
                nexts += g.S1;
            }
#pragma unroll
            for (int w = 0; w < NW; ++w) run[w] += widen_half(c8[i][w >> 1], w & 1);
        }
    }
    for (; nextb < g.nb2; ++nextb) store_v(nextb);  // bands starting at or past the last row
}

// HOGB200_OCTANT: 0 = always the table-gather kernel; 1 = octant for gray
// only; default: gray and RGB (A/B switches)
static bool oct_enabled(int c) {
    const char *e = getenv("HOGB200_OCTANT");
    const int v = (e && *e) ? atoi(e) : 2;
    return v >= 2 || (v == 1 && c == 1);
}

// Small batches (config c1's single frame; a few frames per GPU): one thread
// per column walks ~2H/R1 sub-bands one dependent round of loads per 8 (c1: 75
// sub-bands, 11 us).  Here SPL threads share a column: each sums a contiguous
// run of sub-bands, the group exchanges exclusive prefixes by shuffle, and each
// thread emits the bands whose first sub-band falls in its run; the bands that
// start at or past the last row get the column total.  Same V as k_scan_cols.
template <int NWB, int NW, int SPL>
__global__ void k_scan_cols_split(TileGeom g, Scratch sc) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int l = (int)(threadIdx.x % SPL);
    const int64_t col = t / SPL;
    const bool ok = col < (int64_t)g.n * g.Wc;
    const int f = ok ? (int)(col / g.Wc) : 0, x = ok ? (int)(col % g.Wc) : 0;
    const int ch = (g.nb1 + SPL - 1) / SPL;
    const int s0 = min(l * ch, g.nb1), s1 = min(s0 + ch, g.nb1);
    const uint32_t *__restrict__ Cf = sc.C + (int64_t)f * g.nb1 * g.Wc * NWB + (int64_t)x * NWB;
    auto add_sub = [&](uint32_t (&acc)[NW], int sb) {
        uint32_t c[NWB];
#pragma unroll
        for (int w = 0; w < NWB; ++w) c[w] = __ldg(Cf + (int64_t)sb * g.Wc * NWB + w);
#pragma unroll
        for (int w = 0; w < NW; ++w) acc[w] += widen_half(c[w >> 1], w & 1);
    };
    uint32_t sum[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) sum[w] = 0;
    for (int sb = s0; sb < s1; ++sb) add_sub(sum, sb);
    // exclusive prefix over the column's SPL threads, plus the slab carry
    uint32_t run[NW], total[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        uint32_t inc = sum[w];
#pragma unroll
        for (int d = 1; d < SPL; d <<= 1) {
            const uint32_t v = __shfl_up_sync(FULL, inc, d, SPL);
            if (l >= d) inc += v;
        }
        run[w] = inc - sum[w];
        total[w] = __shfl_sync(FULL, inc, SPL - 1, SPL);
    }
    if (sc.base && ok && x < g.w) {  // slab mode: counts above the slab's first plane row
        const int32_t *bs = sc.base + (int64_t)f * sc.base_fs + x;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t lo = (uint32_t)bs[(int64_t)(2 * w) * g.w];
            const uint32_t hi = 2 * w + 1 < g.bins ? (uint32_t)bs[(int64_t)(2 * w + 1) * g.w] : 0u;
            run[w] += lo | (hi << 16);
            total[w] += lo | (hi << 16);
        }
    }
    if (!ok) return;
    uint32_t *__restrict__ Vf = sc.V + (int64_t)f * g.nb2 * g.Wc * g.NWp + (int64_t)x * g.NWp;
    auto store_v = [&](int b, const uint32_t (&v)[NW]) {
        uint4 *vp = reinterpret_cast<uint4 *>(Vf + (int64_t)b * g.Wc * g.NWp);
#pragma unroll
        for (int q = 0; q < (NW + 3) / 4; ++q)
            vp[q] = make_uint4(v[4 * q], 4 * q + 1 < NW ? v[4 * q + 1] : 0u,
                               4 * q + 2 < NW ? v[4 * q + 2] : 0u, 4 * q + 3 < NW ? v[4 * q + 3] : 0u);
    };
    // bands whose first sub-band b*S1 lies in [s0, s1)
    int sb = s0;
    for (int b = (s0 + g.S1 - 1) / g.S1; b < g.nb2 && b * g.S1 < s1; ++b) {
        for (; sb < b * g.S1; ++sb) add_sub(run, sb);
        store_v(b, run);
    }
    if (l == SPL - 1)  // bands starting at or past the last row
        for (int b = (g.nb1 + g.S1 - 1) / g.S1; b < g.nb2; ++b) store_v(b, total);
}

template <int NWB>
void grad_bin_t(int c, bool counts, const uint8_t *img, int64_t ip, int64_t ics, int64_t ifs,
                const uint8_t *lut, int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                const Scratch &sc, cudaStream_t st) {
    const unsigned nb = blocks_for_warps((int64_t)g.n * g.nb1 * g.nc1);
    const size_t smem =
        (counts && K1_SMEM_COUNTS) ? sizeof(uint32_t) * (4 * NWB + 1) * 4 * 32 * (K_THREADS / 32) : 0;
#define LAUNCH(CHv, CNT) \
    k_grad_bin<CHv, NWB, CNT><<<nb, K_THREADS, smem, st>>>(img, ip, ics, ifs, lut, bm, bp, bfs, g, sc)
    if (c == 1) {
        if (counts) LAUNCH(1, true); else LAUNCH(1, false);
    } else {
        if (counts) LAUNCH(3, true); else LAUNCH(3, false);
    }
#undef LAUNCH
}

void launch_grad_bin(int nwb, int c, bool counts, const uint8_t *img, int64_t ip, int64_t ics,
                     int64_t ifs, const uint8_t *lut, int8_t *bm, int64_t bp, int64_t bfs,
                     const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    // N_b in {4, 8} with the reference's table: the octant kernel (no table
    // gather; k_bin_oct.cu).  It reads and writes 8-byte row groups, so rows
    // must be 8-aligned with pitches covering round_up(w, 8).
    const int64_t w8 = round_up(g.w, 8);
    const bool a8 = ((uintptr_t)img & 7) == 0 && ((uintptr_t)bm & 7) == 0 && ip % 8 == 0 &&
                    ifs % 8 == 0 && (c == 1 || ics % 8 == 0) && bp % 8 == 0 && bfs % 8 == 0 &&
                    ip >= w8 && bp >= w8;
    if ((c == 1 || c == 3) && (g.bins == 4 || g.bins == 8) && a8 && oct_enabled(c) &&
        lut_proven(lut, g.bins, st) &&
        launch_grad_bin_oct(g.bins, c, counts, img, ip, ics, ifs, bm, bp, bfs, g, sc, st))
        return;
    switch (nwb) {
        case 1: grad_bin_t<1>(c, counts, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st); break;
        case 2: grad_bin_t<2>(c, counts, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st); break;
        case 3: grad_bin_t<3>(c, counts, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st); break;
        case 4: grad_bin_t<4>(c, counts, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st); break;
        default: grad_bin_t<5>(c, counts, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st); break;
    }
}

// Per-(bin, column) counts of bin-map rows [0, rows): the slab's own
// contribution to the column carries of the slabs below it (slab mode).
__global__ void k_column_counts(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, int n,
                                int rows, int w, int bins, int32_t *__restrict__ out) {
    extern __shared__ int32_t ccnt[];  // [bins][blockDim.x]
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    for (int b = 0; b < bins; ++b) ccnt[b * blockDim.x + threadIdx.x] = 0;
    if (x < w) {
        const int8_t *col = bm + (int64_t)f * bfs + x;
        for (int y = 0; y < rows; ++y) {
            const int v = col[(int64_t)y * bp];
            if (v >= 0 && v < bins) ++ccnt[v * blockDim.x + threadIdx.x];
        }
        for (int b = 0; b < bins; ++b)
            out[((int64_t)f * bins + b) * w + x] = ccnt[b * blockDim.x + threadIdx.x];
    }
}

void launch_column_counts(const int8_t *bm, int64_t bp, int64_t bfs, int n, int rows, int w, int bins,
                          int32_t *out, cudaStream_t st) {
    const dim3 grid((unsigned)blocks_for(w, 128), (unsigned)n);
    k_column_counts<<<grid, 128, sizeof(int32_t) * bins * 128, st>>>(bm, bp, bfs, n, rows, w, bins, out);
}

template <int NW>
void scan_t(const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    constexpr int NWB = (2 * NW + 3) / 4;
    constexpr int SPL = 8;
    const char *e = getenv("HOGB200_SCAN_SPLIT");  // 0: always one thread per column (A/B)
    const bool split_ok = !(e && *e == '0');
    // long per-column chains on a grid under ~1 wave: split them
    if (split_ok && g.nb1 >= 16 && (int64_t)g.n * g.Wc * SPL <= (int64_t)148 * 2048) {
        k_scan_cols_split<NWB, NW, SPL><<<blocks_for((int64_t)g.n * g.Wc * SPL, 256), 256, 0, st>>>(g, sc);
        return;
    }
    k_scan_cols<NWB, NW><<<blocks_for((int64_t)g.n * g.Wc, 256), 256, 0, st>>>(g, sc);
}

template <int NW>
void counts_t(const int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g, const Scratch &sc,
              cudaStream_t st) {
    constexpr int NWB = (2 * NW + 3) / 4;
    k_bin_counts<NWB><<<blocks_for_warps((int64_t)g.n * g.nb1 * g.nc1), K_THREADS, 0, st>>>(
        bm, bp, bfs, g, sc);
}

#define HOG_NW_DISPATCH(nw, FN, ...)       \
    switch (nw) {                          \
        case 1: FN<1>(__VA_ARGS__); break; \
        case 2: FN<2>(__VA_ARGS__); break; \
        case 3: FN<3>(__VA_ARGS__); break; \
        case 4: FN<4>(__VA_ARGS__); break; \
        case 5: FN<5>(__VA_ARGS__); break; \
        case 6: FN<6>(__VA_ARGS__); break; \
        case 7: FN<7>(__VA_ARGS__); break; \
        case 8: FN<8>(__VA_ARGS__); break; \
        default: FN<9>(__VA_ARGS__); break; \
    }

void launch_scan(int nw, const TileGeom &g, const Scratch &sc, cudaStream_t st) {
    HOG_NW_DISPATCH(nw, scan_t, g, sc, st)
}

void launch_counts_from_bm(int nw, const int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                           const Scratch &sc, cudaStream_t st) {
    HOG_NW_DISPATCH(nw, counts_t, bm, bp, bfs, g, sc, st)
}

}  // namespace hogb200
