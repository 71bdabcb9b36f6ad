// k_bin_oct.cu -- K1 for N_b in {4, 8}: gradient + orientation binning with no
// table gather.  gradient.py:29-45 (bin_of), :55-72 (build_lut), :95-121
// (gradient_map).
//
// The reference's table for N_b = 8 (and 4) is the exact floor(angle / sector)
// with every boundary ray in the higher bin (bin_of's "an angle exactly on a
// boundary belongs to the higher bin"; numpy's atan2 lands each boundary ray
// exactly, which the proof below checks).  Folding the table by its quarter-
// and half-turn symmetries leaves four boundary lines (0, 45, 90, 135 degrees),
// so a bin is three sign bits of four linear forms of the point rotated by a
// tiny angle (1/512 rad-ish) counter-clockwise, which sends boundary rays into
// the higher bin:
//   y' = 512 dy + dx,  x' = 512 dx - dy            (the rotated point, scaled)
//   f1 = y', f2 = x', f3 = y' - x' = 512 D1 + D2, f4 = y' + x' = 512 D2 - D1
//   (D1 = dy - dx, D2 = dy + dx)
//   bin bits: b2 = [f1 < 0], b1 = b2 ^ [f2 < 0], b0 = ~([f1<0]^[f2<0]^[f3<0]^[f4<0])
// The table is then "held in registers": eight sectors selected by sign bits.
// Every form is one fp16x2 FMA on exact small integers (bytes enter as the
// half 1024 + b, so differences are exact); one rounding of a non-zero integer
// keeps its sign and overflow saturates to a signed infinity, so the signs are
// exact.  Two pixels per instruction.  k_lut_proof evaluates this same device
// code on all 261,121 (dx, dy) pairs against the caller's table, and the
// launcher uses this kernel only for a table that passed (hog_abi.cu).
//
// Bin counts per (sub-band, column) for k_scan_cols: one-hot bytes (bit n of
// column k's byte = [bin == n]) from the three bit masks, accumulated
// bit-sliced with carry-save adders over blocks of 8 rows, and turned into the
// u8x4 layout of Scratch::C by 8x8 bit transposes at the end of the sub-band.
//
// Work split: a half-warp (16 lanes) owns one (frame, sub-band, 128-column
// chunk) unit, the same units as k_grad_bin; lane L owns columns x0+8L..+7 and
// slides a three-row window down the sub-band (two 4-byte words per row, held
// as fp16x2 "even" / "odd" byte pairs).
#include <cuda_fp16.h>

#include "hog_common.cuh"

namespace hogb200 {

namespace {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
}
__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t heq0_mask(uint32_t a) {
    uint32_t r;
    asm("set.eq.u32.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(0u));
    return r;
}

// dx^2 + dy^2 of both halves of a pair, exact in fp32 (<= 130,050): FHFMA
// (fp16 operands, fp32 accumulate) reads the halves in place
__device__ __forceinline__ void mag2(uint32_t dx, uint32_t dy, float &lo, float &hi) {
    asm("{ .reg .f16 xl, xh, yl, yh; .reg .f32 t, u;\n"
        "  mov.b32 {xl, xh}, %2; mov.b32 {yl, yh}, %3;\n"
        "  fma.rn.f32.f16 t, yl, yl, 0f00000000; fma.rn.f32.f16 %0, xl, xl, t;\n"
        "  fma.rn.f32.f16 u, yh, yh, 0f00000000; fma.rn.f32.f16 %1, xh, xh, u; }"
        : "=f"(lo), "=f"(hi) : "r"(dx), "r"(dy));
}

constexpr uint32_t H1024 = 0x64646464u;  // byte b -> half 1024 + b (with the 0x64 high byte)
constexpr uint32_t P512 = 0x60006000u;   // half2(512, 512)
constexpr uint32_t M512 = 0xE000E000u;   // half2(-512, -512)
constexpr uint32_t SIGNS = 0xFBD9u;      // prmt: sign bytes of (A.lo, B.lo, A.hi, B.hi)

// one row's 8 pixels as fp16x2: E = bytes (0,2), O = bytes (1,3) of each word
struct Row8 {
    uint32_t E0, O0, E1, O1;
};
__device__ __forceinline__ Row8 spread(uint32_t w0, uint32_t w1) {
    return {prmt(w0, H1024, 0x4240), prmt(w0, H1024, 0x4341), prmt(w1, H1024, 0x4240),
            prmt(w1, H1024, 0x4341)};
}

// Bit masks (0x00 / 0xFF per pixel byte) of one word's 4 pixels from the
// gradient pairs of A = pixels (0, 2) and B = pixels (1, 3).
// NB = 8: m0/m1/m2 = bin bits 0/1/2;  NB = 4: m0/m1 = bits 0/1 (m2 unused).
// mz = zero gradient (no bin).
template <int NB>
__device__ __forceinline__ void oct_masks(uint32_t dxA, uint32_t dyA, uint32_t dxB, uint32_t dyB,
                                          uint32_t &m0, uint32_t &m1, uint32_t &m2, uint32_t &mz) {
    const uint32_t f1A = hfma2(dyA, P512, dxA), f1B = hfma2(dyB, P512, dxB);  // y'
    const uint32_t g2A = hfma2(dxA, M512, dyA), g2B = hfma2(dxB, M512, dyB);  // -x'
    const uint32_t s1 = prmt(f1A, f1B, SIGNS);
    const uint32_t s12n = prmt(f1A ^ g2A, f1B ^ g2B, SIGNS);  // ~(s1 ^ s2)
    mz = prmt(heq0_mask(f1A), heq0_mask(f1B), SIGNS);
    if (NB == 8) {
        const uint32_t D1A = hsub2(dyA, dxA), D2A = hadd2(dyA, dxA);
        const uint32_t D1B = hsub2(dyB, dxB), D2B = hadd2(dyB, dxB);
        const uint32_t f3A = hfma2(D1A, P512, D2A), f3B = hfma2(D1B, P512, D2B);  // y' - x'
        const uint32_t g4A = hfma2(D2A, M512, D1A), g4B = hfma2(D2B, M512, D1B);  // -(y' + x')
        // s1^s2^s3^s4 = sign(f1 ^ g2 ^ f3 ^ g4) (two sign flips cancel)
        const uint32_t s1234 = prmt(f1A ^ g2A ^ f3A ^ g4A, f1B ^ g2B ^ f3B ^ g4B, SIGNS);
        m2 = s1;
        m1 = ~s12n;
        m0 = ~s1234;
    } else {
        m1 = s1;
        m0 = ~s12n;
        m2 = 0;
    }
}

// bins4 bytes (NO_BIN = 0xFF where nv) and the one-hot bytes (bit n = [bin == n])
template <int NB>
__device__ __forceinline__ void oct_bins(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t nv,
                                         uint32_t &bins4, uint32_t &oh) {
    if (NB == 8) {
        bins4 = (m0 & 0x01010101u) | (m1 & 0x02020202u) | (m2 & 0x04040404u) | nv;
        oh = ~(m0 ^ 0xAAAAAAAAu) & ~(m1 ^ 0xCCCCCCCCu) & ~(m2 ^ 0xF0F0F0F0u) & ~nv;
    } else {
        bins4 = (m0 & 0x01010101u) | (m1 & 0x02020202u) | nv;
        oh = ~(m0 ^ 0xAAAAAAAAu) & ~(m1 ^ 0xCCCCCCCCu) & 0x0F0F0F0Fu & ~nv;
    }
}

__device__ __forceinline__ void csa(uint32_t &sum, uint32_t &carry, uint32_t a, uint32_t b, uint32_t c) {
    sum = a ^ b ^ c;
    carry = (a & b) | (c & (a ^ b));
}

// 8x8 bit transpose: out byte n bit j = in byte j bit n
__device__ __forceinline__ uint64_t tr8x8(uint64_t x) {
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x = x ^ t ^ (t << 28);
    return x;
}

// Bit-sliced counters of one word group (4 columns x 8 bins): q[j] bit
// (8k + n) is bit j of the count of bin n in column k.
struct Slice {
    uint32_t q[8];
};

// q (8 bit planes) -> cc[k] = counts of bins 0..3 | 4..7 of column k (u8x4 each)
__device__ __forceinline__ void unslice(const Slice &s, uint32_t (&lo)[4], uint32_t (&hi)[4]) {
    uint32_t c[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // 4x4 byte transposes of planes 4h..4h+3
        const uint32_t *q = s.q + 4 * h;
        const uint32_t a = prmt(q[0], q[1], 0x5140), b = prmt(q[2], q[3], 0x5140);
        const uint32_t cc = prmt(q[0], q[1], 0x7362), d = prmt(q[2], q[3], 0x7362);
        c[h][0] = prmt(a, b, 0x5410);
        c[h][1] = prmt(a, b, 0x7632);
        c[h][2] = prmt(cc, d, 0x5410);
        c[h][3] = prmt(cc, d, 0x7632);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint64_t t = tr8x8(((uint64_t)c[1][k] << 32) | c[0][k]);
        lo[k] = (uint32_t)t;
        hi[k] = (uint32_t)(t >> 32);
    }
}

}  // namespace

// rows of loads in flight ahead of the row being binned (B200 A/B: tools/ab_r2.sh)
#ifndef K1_OCT_PF
#define K1_OCT_PF 2
#endif

// counts as in k_grad_bin (C[f][b][x][w], u8x4 of bins 4w..4w+3) when COUNTS
#ifndef K1_OCT_ROLL
#define K1_OCT_ROLL 0
#endif
#ifndef K1_OCT_MINB
#define K1_OCT_MINB 4
#endif

#ifndef K1_OCT_MINB3
#define K1_OCT_MINB3 3
#endif

// CH = 3: per-channel gradients, the reference's channel rule (largest
// dx^2 + dy^2, first channel on ties; gradient.py:113-117) on exact fp32
// magnitudes, then the same octant sign tests on the winning pair
template <int NB, bool COUNTS, int CH>
__global__ void __launch_bounds__(K_THREADS, CH == 1 ? K1_OCT_MINB : K1_OCT_MINB3)
k_grad_bin_oct(const uint8_t *__restrict__ img, int64_t ip, int64_t ics, int64_t ifs,
               int8_t *__restrict__ bm, int64_t bp, int64_t bfs, TileGeom g, Scratch sc) {
    const int lane = threadIdx.x & 31, seg = lane >> 4, sl = lane & 15;
    const int64_t nunits = (int64_t)g.n * g.nb1 * g.nc1;
    const int64_t unit0 = 2 * warp_id() + seg;
    if (2 * warp_id() >= nunits) return;  // whole warp past the end (uniform)
    const bool live = unit0 < nunits;
    const int64_t unit = live ? unit0 : nunits - 1;
    int chunk, b, f;
    if (unit < ((int64_t)1 << 31)) {
        const uint32_t u = (uint32_t)unit, q = u / (uint32_t)g.nc1;
        chunk = (int)(u - q * (uint32_t)g.nc1);
        b = (int)(q % (uint32_t)g.nb1);
        f = (int)(q / (uint32_t)g.nb1);
    } else {
        chunk = (int)(unit % g.nc1);
        b = (int)((unit / g.nc1) % g.nb1);
        f = (int)(unit / ((int64_t)g.nc1 * g.nb1));
    }
    const int x = chunk * CHUNK + 8 * sl;
    const int y0 = b * g.R1, y1 = min(y0 + g.R1, g.h);
    const int nrows = live ? y1 - y0 : 0;
    const int iters = max(nrows, __shfl_xor_sync(FULL, nrows, 16));
    // lanes past the frame read (and discard) the last 8-byte group of the row
    const int xl = x < g.w ? x : ((g.w - 1) & ~7);
    const uint8_t *col = img + (int64_t)f * ifs + xl;
    // neighbour bytes outside the lane's 8: left of segment lane 0, right of lane 15
    const bool has_l = sl == 0 && x >= 1, has_r = sl == 15 && x + 8 < g.w;
    auto rowp = [&](int y) { return col + (int64_t)min(max(y, -g.ht), g.h - 1 + g.hb) * ip; };
    // bytes of the lane's 8 columns that are interior pixels (1 <= x <= w-2): nv = 0
    uint32_t nvc[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int xx = x + 4 * k + j;
            if (!(xx >= 1 && xx <= g.w - 2)) v |= 0xffu << (8 * j);
        }
        nvc[k] = v;
    }

    // rows y-1, y, y+1 as fp16x2 pairs; rows y+2 .. y+K1_OCT_PF raw (loads in flight)
    uint2 qw[CH][K1_OCT_PF];
    uint32_t ql[CH][K1_OCT_PF], qr[CH][K1_OCT_PF];
    uint32_t elc[CH], erc[CH], elb[CH], erb[CH];
    Row8 ra[CH], rc[CH], rb[CH];
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
        const uint8_t *pa = rowp(y0 - 1) + ch * ics, *pc = rowp(y0) + ch * ics, *pb = rowp(y0 + 1) + ch * ics;
        const uint2 wa = __ldg(reinterpret_cast<const uint2 *>(pa));
        const uint2 wc = __ldg(reinterpret_cast<const uint2 *>(pc));
        const uint2 wb = __ldg(reinterpret_cast<const uint2 *>(pb));
        elc[ch] = has_l ? __ldg(pc - 1) : 0u;
        elb[ch] = has_l ? __ldg(pb - 1) : 0u;
        erc[ch] = has_r ? __ldg(pc + 8) : 0u;
        erb[ch] = has_r ? __ldg(pb + 8) : 0u;
#pragma unroll
        for (int i = 0; i + 1 < K1_OCT_PF; ++i) {
            const uint8_t *pq = rowp(y0 + 2 + i) + ch * ics;
            qw[ch][i] = __ldg(reinterpret_cast<const uint2 *>(pq));
            ql[ch][i] = has_l ? __ldg(pq - 1) : 0u;
            qr[ch][i] = has_r ? __ldg(pq + 8) : 0u;
        }
        ra[ch] = spread(wa.x, wa.y);
        rc[ch] = spread(wc.x, wc.y);
        rb[ch] = spread(wb.x, wb.y);
    }
    int8_t *bout = bm + (int64_t)f * bfs + (int64_t)y0 * bp + x;
    // rows whose pixels get bins: [rlo, rhi) (frame border rows are NO_BIN unless
    // the slab continues past them); dead half-warps bin nothing
    const int rlo = max(y0, g.ht ? 0 : 1);
    const int rhi = live ? min(y1, g.hb ? g.h : g.h - 1) : rlo;
    const uint32_t nrow_ok = (uint32_t)max(rhi - rlo, 0);
    // rows stored: [y0, y1) for live lanes inside the frame (8-byte stores: the
    // launcher checked bm's pitch covers round_up(w, 8))
    const uint32_t nstore = (live && x < g.w) ? (uint32_t)(y1 - y0) : 0u;
    // last readable row: the row pointer stops there
    const int64_t pmax = (int64_t)(g.h - 1 + g.hb) * ip;
    int64_t poff = (int64_t)min(max(y0 + 1 + K1_OCT_PF, -g.ht), g.h - 1 + g.hb) * ip;
    const uint8_t *colf = col;
    const uint32_t Lsel = sl == 0 ? 0xffffffffu : 0u, Rsel = sl == 15 ? 0xffffffffu : 0u;

    Slice S[2];  // bit-sliced counts of the lane's two word groups
    uint32_t ones[2], twos[2], fours[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
#pragma unroll
        for (int j = 0; j < 8; ++j) S[k].q[j] = 0;
        ones[k] = twos[k] = fours[k] = 0;
    }

    // one row: classify, store, return the two one-hot words
    auto row = [&](int y, uint32_t (&oh)[2]) {
        // row y+1+K1_OCT_PF in flight while row y is binned
        const uint8_t *pd = colf + poff;
        uint2 wd[CH];
        uint32_t eld[CH], erd[CH];
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            wd[ch] = __ldg(reinterpret_cast<const uint2 *>(pd + ch * ics));
            eld[ch] = has_l ? __ldg(pd + ch * ics - 1) : 0u;
            erd[ch] = has_r ? __ldg(pd + ch * ics + 8) : 0u;
        }
        poff = min(poff + ip, pmax);
        // halo halves of the centre row: odd byte left of the lane, even byte right of it
        uint32_t Oprev[CH], Enext[CH];
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            const uint32_t Oup = __shfl_up_sync(FULL, rc[ch].O1, 1, 16);
            const uint32_t Edn = __shfl_down_sync(FULL, rc[ch].E0, 1, 16);
            Oprev[ch] = (prmt(elc[ch], H1024, 0x4000) & Lsel) | (Oup & ~Lsel);
            Enext[ch] = (prmt(erc[ch], H1024, 0x0040) & Rsel) | (Edn & ~Rsel);
        }
        const bool rowok = (uint32_t)(y - rlo) < nrow_ok;
        uint32_t bins[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            uint32_t dxA, dyA, dxB, dyB;
            float bmA0 = 0.f, bmA1 = 0.f, bmB0 = 0.f, bmB1 = 0.f;  // winning magnitudes
#pragma unroll
            for (int ch = 0; ch < CH; ++ch) {
                const Row8 &a = ra[ch], &c = rc[ch], &bb = rb[ch];
                const uint32_t Ec = k ? c.E1 : c.E0, Oc = k ? c.O1 : c.O0;
                const uint32_t Op = k ? c.O0 : Oprev[ch], En = k ? Enext[ch] : c.E1;
                const uint32_t xA = hsub2(Oc, prmt(Op, Oc, 0x5432));  // (b1 - b-1, b3 - b1)
                const uint32_t xB = hsub2(prmt(Ec, En, 0x5432), Ec);  // (b2 - b0, b4 - b2)
                const uint32_t yA = hsub2(k ? bb.E1 : bb.E0, k ? a.E1 : a.E0);
                const uint32_t yB = hsub2(k ? bb.O1 : bb.O0, k ? a.O1 : a.O0);
                if (CH == 1) {
                    dxA = xA, dyA = yA, dxB = xB, dyB = yB;
                } else {
                    float mA0, mA1, mB0, mB1;
                    mag2(xA, yA, mA0, mA1);
                    mag2(xB, yB, mB0, mB1);
                    if (ch == 0) {
                        dxA = xA, dyA = yA, dxB = xB, dyB = yB;
                        bmA0 = mA0, bmA1 = mA1, bmB0 = mB0, bmB1 = mB1;
                    } else {
                        // lane mask of the halves whose magnitude beats the best so far
                        // (sign of best - mag; ties keep the earlier channel)
                        const uint32_t kA = prmt(__float_as_uint(bmA0 - mA0), __float_as_uint(bmA1 - mA1), 0xFFBB);
                        const uint32_t kB = prmt(__float_as_uint(bmB0 - mB0), __float_as_uint(bmB1 - mB1), 0xFFBB);
                        dxA = (xA & kA) | (dxA & ~kA), dyA = (yA & kA) | (dyA & ~kA);
                        dxB = (xB & kB) | (dxB & ~kB), dyB = (yB & kB) | (dyB & ~kB);
                        bmA0 = fmaxf(bmA0, mA0), bmA1 = fmaxf(bmA1, mA1);
                        bmB0 = fmaxf(bmB0, mB0), bmB1 = fmaxf(bmB1, mB1);
                    }
                }
            }
            uint32_t m0, m1, m2, mz;
            oct_masks<NB>(dxA, dyA, dxB, dyB, m0, m1, m2, mz);
            const uint32_t nv = (rowok ? nvc[k] : 0xffffffffu) | mz;
            oct_bins<NB>(m0, m1, m2, nv, bins[k], oh[k]);
        }
        if ((uint32_t)(y - y0) < nstore) *reinterpret_cast<uint2 *>(bout) = make_uint2(bins[0], bins[1]);
        bout += bp;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
            ra[ch] = rc[ch];
            rc[ch] = rb[ch];
            elc[ch] = elb[ch], erc[ch] = erb[ch];
            qw[ch][K1_OCT_PF - 1] = wd[ch], ql[ch][K1_OCT_PF - 1] = eld[ch], qr[ch][K1_OCT_PF - 1] = erd[ch];
            rb[ch] = spread(qw[ch][0].x, qw[ch][0].y);
            elb[ch] = ql[ch][0], erb[ch] = qr[ch][0];
#pragma unroll
            for (int i = 0; i + 1 < K1_OCT_PF; ++i)
                qw[ch][i] = qw[ch][i + 1], ql[ch][i] = ql[ch][i + 1], qr[ch][i] = qr[ch][i + 1];
        }
    };

    int y = y0;
#if K1_OCT_ROLL
    // row pairs in a rolled loop; the carry-save tree advances by a uniform
    // pair counter (fewer live registers than the unrolled 8-row block)
    uint32_t t2a[2] = {0, 0}, t4a[2] = {0, 0};
    const int npairs = ((iters + 7) >> 3) << 2;
#pragma unroll 1
    for (int pr = 0; pr < npairs; ++pr) {
        uint32_t oa[2], ob[2];
        row(y, oa);
        row(y + 1, ob);
        y += 2;
        if (COUNTS) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                uint32_t c2;
                csa(ones[k], c2, ones[k], oa[k], ob[k]);
                if ((pr & 1) == 0) {
                    t2a[k] = c2;
                } else {
                    uint32_t c4;
                    csa(twos[k], c4, twos[k], t2a[k], c2);
                    if ((pr & 2) == 0) {
                        t4a[k] = c4;
                    } else {
                        uint32_t c;
                        csa(fours[k], c, fours[k], t4a[k], c4);
#pragma unroll
                        for (int j = 3; j < 8; ++j) {
                            const uint32_t q = S[k].q[j];
                            S[k].q[j] = q ^ c;
                            c &= q;
                        }
                    }
                }
            }
        }
    }
#else
    for (int it = 0; it < iters; it += 8) {
        // 8 rows: carry-save tree ones/twos/fours, one eights carry rippled into q[3..7]
        uint32_t e8[2];
        uint32_t t2a[2], t4a[2], t4b[2];
#pragma unroll
        for (int r = 0; r < 8; r += 2) {
            uint32_t oa[2], ob[2];
            row(y, oa);
            row(y + 1, ob);
            y += 2;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (!COUNTS) continue;
                uint32_t c2;
                csa(ones[k], c2, ones[k], oa[k], ob[k]);
                if ((r & 2) == 0) {
                    t2a[k] = c2;
                } else {
                    uint32_t c4;
                    csa(twos[k], c4, twos[k], t2a[k], c2);
                    if (r == 2) t4a[k] = c4; else t4b[k] = c4;
                }
            }
        }
        if (COUNTS) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                csa(fours[k], e8[k], fours[k], t4a[k], t4b[k]);
                uint32_t c = e8[k];
#pragma unroll
                for (int j = 3; j < 8; ++j) {
                    const uint32_t q = S[k].q[j];
                    S[k].q[j] = q ^ c;
                    c &= q;
                }
            }
        }
    }
#endif
    if (COUNTS && live) {  // columns past w get zero counts (k_scan_cols reads them)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            S[k].q[0] = ones[k];
            S[k].q[1] = twos[k];
            S[k].q[2] = fours[k];
            uint32_t lo[4], hi[4];
            unslice(S[k], lo, hi);
            const int xk = x + 4 * k;
            uint32_t *cp = sc.C + (((int64_t)f * g.nb1 + b) * g.Wc + xk) * (NB == 8 ? 2 : 1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (NB == 8) {
                    cp[2 * j] = lo[j];
                    cp[2 * j + 1] = hi[j];
                } else {
                    cp[j] = lo[j];
                }
            }
        }
    }
}

// Device proof: the classifier above on every (dx, dy) in [-255, 255]^2,
// compared with the caller's table (uint8, NO_BIN = 0xFF, lut[(dx+255)*511 +
// dy+255]).  Thread t takes dy = t % 511 - 255 and four consecutive dx, fed
// through the same oct_masks / oct_bins as the binning kernel.
template <int NB>
__global__ void k_lut_proof(const uint8_t *__restrict__ lut, unsigned long long *mismatches) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int ngrp = (LUT_SIDE + 3) / 4;  // 128 groups of 4 dx (the last one ragged)
    if (t >= LUT_SIDE * ngrp) return;
    const int dy = t % LUT_SIDE - 255, dx0 = (t / LUT_SIDE) * 4 - 255;
    auto h = [](int v) { return (uint32_t)__half_as_ushort(__int2half_rn(v)); };
    int dx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) dx[j] = min(dx0 + j, 255);
    // A = pixels (0, 2), B = pixels (1, 3)
    const uint32_t dxA = h(dx[0]) | h(dx[2]) << 16, dxB = h(dx[1]) | h(dx[3]) << 16;
    const uint32_t dyA = h(dy) | h(dy) << 16, dyB = dyA;
    uint32_t m0, m1, m2, mz, bins4, oh;
    oct_masks<NB>(dxA, dyA, dxB, dyB, m0, m1, m2, mz);
    oct_bins<NB>(m0, m1, m2, mz, bins4, oh);
    unsigned long long bad = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (dx0 + j > 255) break;
        const uint32_t got = (bins4 >> (8 * j)) & 0xffu;
        const uint32_t want = lut[(dx[j] + 255) * LUT_SIDE + (dy + 255)];
        // the one-hot byte must be the bin's bit (none for NO_BIN)
        const uint32_t o = (oh >> (8 * j)) & 0xffu;
        const uint32_t owant = want == 0xffu ? 0u : (1u << want);
        bad += (got != want || o != owant) ? 1 : 0;  // entries, not fields
    }
    if (bad) atomicAdd(mismatches, bad);
}

bool launch_grad_bin_oct(int bins, int c, bool counts, const uint8_t *img, int64_t ip, int64_t ics,
                         int64_t ifs, int8_t *bm, int64_t bp, int64_t bfs, const TileGeom &g,
                         const Scratch &sc, cudaStream_t st) {
    const int64_t units = (int64_t)g.n * g.nb1 * g.nc1;
    const unsigned nb = blocks_for_warps((units + 1) / 2);
#define LAUNCH(NBv, CNT, CHv) \
    k_grad_bin_oct<NBv, CNT, CHv><<<nb, K_THREADS, 0, st>>>(img, ip, ics, ifs, bm, bp, bfs, g, sc)
    if (c == 1) {
        if (bins == 8) {
            if (counts) LAUNCH(8, true, 1); else LAUNCH(8, false, 1);
        } else if (bins == 4) {
            if (counts) LAUNCH(4, true, 1); else LAUNCH(4, false, 1);
        } else {
            return false;
        }
    } else if (c == 3) {
        if (bins == 8) {
            if (counts) LAUNCH(8, true, 3); else LAUNCH(8, false, 3);
        } else if (bins == 4) {
            if (counts) LAUNCH(4, true, 3); else LAUNCH(4, false, 3);
        } else {
            return false;
        }
    } else {
        return false;
    }
#undef LAUNCH
    return true;
}

bool launch_lut_proof(int bins, const uint8_t *lut, unsigned long long *mismatches, cudaStream_t st) {
    const int total = LUT_SIDE * ((LUT_SIDE + 3) / 4);
    const unsigned nb = blocks_for(total, 256);
    if (bins == 8) k_lut_proof<8><<<nb, 256, 0, st>>>(lut, mismatches);
    else if (bins == 4) k_lut_proof<4><<<nb, 256, 0, st>>>(lut, mismatches);
    else return false;
    return true;
}

}  // namespace hogb200
