// k_planes.cuh -- K2: the single-write integral-plane kernel (+ fused cell
// grid).  Included by k_planes_{a,b,c,d}.cu, each instantiating a range of
// packed-word counts NW (bins = 2*NW or 2*NW-1) to keep builds parallel.
#pragma once
#include "hog_common.cuh"

namespace hogb200 {

template <int VC>
__device__ __forceinline__ void store_chunk(int32_t *p, const uint32_t (&v)[VC], bool vec, int valid) {
    if (vec) {
        if constexpr (VC == 8) {
#if K2_STORE_HINT
            asm volatile("st.global.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
#else
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
#endif
                         "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                         : "memory");
        } else {
#if K2_STORE_HINT
            asm volatile("st.global.cs.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                         "r"(v[3])
                         : "memory");
#else
            *reinterpret_cast<int4 *>(p) = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
#endif
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

// Gradient + LUT binning (gradient.py:95-121) of plane-kernel rows: lane owns
// pixel columns x .. x+VC-1 (VC/4 words).  Writes the bin map for rows
// [y0, y1) of owned columns and counts bins of rows [y0, ycnt) per column
// into cc (u8x4, bins 4w..4w+3 of column k in cc[k][w]).
template <int CH, int VC, int NWB>
__device__ __forceinline__ void bin_rows(const FusedIn &fi, const TileGeom &g, int f, int x,
                                         int lane, bool own, int y0, int y1, int ycnt,
                                         int8_t *bmf, int64_t bp, uint32_t (&cc)[VC][NWB]) {
    constexpr int ND = VC / 4;
    const uint8_t *lut0 = fi.lut + (255 * LUT_SIDE + 255);
    const uint8_t *base = fi.img + (int64_t)f * fi.ifs;
    const int xlast = (g.w - 1) & ~3;
    int xo[ND];
    uint32_t valid[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        xo[d] = min(x + 4 * d, xlast);  // lanes past the frame re-read the last word
        valid[d] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (x + 4 * d + k >= 1 && x + 4 * d + k <= g.w - 2) valid[d] |= 0xffu << (8 * k);
    }
    const int eoff = lane == 0 ? -1 : VC;
    const bool has_edge = (lane == 0 && x >= 1) || (lane == 31 && x + VC < g.w);
    auto rowp = [&](int y) { return base + (int64_t)min(max(y, 0), g.h - 1) * fi.ip; };
    uint32_t r0[CH][ND], r1[CH][ND], r2[CH][ND], e1[CH], e2[CH];
    {
        const uint8_t *pa = rowp(y0 - 1), *pb = rowp(y0), *pc = rowp(y0 + 1);
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                r0[ch][d] = __ldg(reinterpret_cast<const uint32_t *>(pa + ch * fi.ics + xo[d]));
                r1[ch][d] = __ldg(reinterpret_cast<const uint32_t *>(pb + ch * fi.ics + xo[d]));
                r2[ch][d] = __ldg(reinterpret_cast<const uint32_t *>(pc + ch * fi.ics + xo[d]));
            }
            e1[ch] = has_edge ? (uint32_t)__ldg(pb + ch * fi.ics + x + eoff) : 0u;
            e2[ch] = has_edge ? (uint32_t)__ldg(pc + ch * fi.ics + x + eoff) : 0u;
        }
    }
    const uint8_t *pd = rowp(y0 + 2);
    int8_t *bout = bmf + (int64_t)y0 * bp + x;
    for (int y = y0; y < y1; ++y) {
        uint32_t r3[CH][ND], e3[CH];
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
#pragma unroll
            for (int d = 0; d < ND; ++d)
                r3[ch][d] = __ldg(reinterpret_cast<const uint32_t *>(pd + ch * fi.ics + xo[d]));
            e3[ch] = has_edge ? (uint32_t)__ldg(pd + ch * fi.ics + x + eoff) : 0u;
        }
        if (y + 3 < g.h) pd += fi.ip;
        uint32_t bins[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) bins[d] = 0xffffffffu;
        if (y > 0 && y < g.h - 1) {
            int bdx[ND][4], bdy[ND][4], bmag[ND][4];
#pragma unroll
            for (int ch = 0; ch < CH; ++ch) {
                const uint32_t prev = __shfl_up_sync(FULL, r1[ch][ND - 1], 1);
                const uint32_t next = __shfl_down_sync(FULL, r1[ch][0], 1);
#pragma unroll
                for (int d = 0; d < ND; ++d) {
                    const uint32_t lb = d > 0 ? r1[ch][d - 1] >> 24 : (lane == 0 ? e1[ch] : prev >> 24);
                    const uint32_t rb = d + 1 < ND ? r1[ch][d + 1] : (lane == 31 ? e1[ch] : next);
                    const uint32_t Lw = __byte_perm(lb, r1[ch][d], 0x6540);  // x-1 .. x+2
                    const uint32_t Rw = __byte_perm(r1[ch][d], rb, 0x4321);  // x+1 .. x+4
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int dx = (int)byte_of(Rw, k) - (int)byte_of(Lw, k);
                        const int dy = (int)byte_of(r2[ch][d], k) - (int)byte_of(r0[ch][d], k);
                        if (CH == 1) {
                            bdx[d][k] = dx, bdy[d][k] = dy;
                        } else {
                            // gradient.py:113-117: largest dx^2+dy^2 wins, first channel on ties
                            const int mag = dx * dx + dy * dy;
                            if (ch == 0 || mag > bmag[d][k])
                                bdx[d][k] = dx, bdy[d][k] = dy, bmag[d][k] = mag;
                        }
                    }
                }
            }
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                uint32_t v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = __ldg(lut0 + (bdx[d][k] * LUT_SIDE + bdy[d][k]));
                const uint32_t w4 = __byte_perm(__byte_perm(v[0], v[1], 0x0040),
                                                __byte_perm(v[2], v[3], 0x0040), 0x5410);
                bins[d] = (w4 & valid[d]) | ~valid[d];
            }
        }
        if (own) {
#pragma unroll
            for (int d = 0; d < ND; ++d)
                if (x + 4 * d < g.w) *reinterpret_cast<uint32_t *>(bout + 4 * d) = bins[d];
            if (y < ycnt) {
#pragma unroll
                for (int d = 0; d < ND; ++d) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t v = byte_of(bins[d], k);
                        const uint32_t q = v >> 2, one = 1u << ((v & 3u) << 3);
#pragma unroll
                        for (int w = 0; w < NWB; ++w) cc[4 * d + k][w] += q == (uint32_t)w ? one : 0u;
                    }
                }
            }
        }
        bout += bp;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                r0[ch][d] = r1[ch][d];
                r1[ch][d] = r2[ch][d];
                r2[ch][d] = r3[ch][d];
            }
            e1[ch] = e2[ch];
            e2[ch] = e3[ch];
        }
    }
}

// P(Y, X) = ptop(X) + Lacc(Y) + Q(Y, X):
//   ptop(X) = sum_{xs <= x' < X} V(x')  -- band's top row relative to the strip's
//             left edge; constant through the band, kept in shared memory
//   Lacc(Y) = P(Y, xs)                  -- one value per bin, uniform over the warp
//   Q(Y, X) = sum_{Y0 <= y < Y} count of row y in [xs, X)  -- <= (R+halo)*32*VC < 2^16,
//             so two bins share one register (u16x2) and a row update is one add

// CH > 0: fused variant -- the CTA bins its own rows from the frame (CH
// channels) and gets the column counts above its band by decoupled look-back
// over the bands above (tickets keep the waits acyclic); requires nss == 1.
//
// TMA: plane rows are not stored by the compute warps.  Each compute warp
// writes its strip of row Y (all bins) into ring slot Y % RING in shared
// memory and arrives on full[slot]; a store warp (warp NWARP, one lane)
// waits on full[slot] and writes the slot's bin rows to HBM with one
// cp.async.bulk per (bin, row) -- whole 32-B sectors, no LSU traffic -- then
// releases the slot on empty[slot] once the TMA engine has read it.  The
// compute warps synchronise among themselves with named barrier 1.
template <int NW, int KR, int VC, bool VEC, int CH = 0, bool TMA = false, bool PR = false, bool RB = false>
__global__ void __launch_bounds__(k2_maxt(NW, VC, PR), k2_minb(NW, VC))
k_planes(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, PlaneOut po, GridOut go,
         TileGeom g, Scratch sc, FusedIn fi) {
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int NB = 2 * NW;
    constexpr int NWB = (NB + 3) / 4;
    // the band's top row in registers (small variants): no shared-memory load per
    // stored value (c2: 8 LDS.128 per row and lane, a short-scoreboard stall each)
    constexpr bool PREG = PR && NB * VC <= 32 && !TMA;
    uint32_t preg[PREG ? NB : 1][PREG ? VC : 1];
    // FP (row-bulk variant): preg holds the lane's full 32-bit plane values P(Y, X),
    // updated once per row by (row carry + strip-row prefix byte): one PRMT + one
    // IADD3 per value and the staging store reads them in place, where the packed
    // form costs a third instruction per value (unpack, 3-input add, u16x2 update).
    // Measured slower with per-thread global stores and with staging stores alike
    // (c2 1.015 against 0.995 ms: the row update then waits on the registers the
    // row's STS.128 still read), so it is off (K2_RB_P32 = 0; experiment builds).
    constexpr bool FP = RB && PREG && VC == 4 && K2_RB_P32;
    // PAIR (experiment knob K2_PAIR256): 256-bit plane stores for the 4-columns-per-lane
    // variants, the halves traded between lane pairs by shuffle
    constexpr bool PAIR = K2_PAIR256 && VC == 4 && VEC && !TMA && !RB && CH == 0;
    // rows per phase-A/phase-B group: 4; 2 for the wide variants (NW >= 6, K2_GW) and for
    // 8 columns per lane (K2_G8), where the group's live scan state is largest
    // (the experiment-only fused path, CH > 0, was written for 4-row groups)
    constexpr int G = CH > 0 ? K2_G : NW >= 6 ? K2_GW : VC == 8 ? K2_G8 : K2_G;
    const int nwarp = g.NWARP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ int tk;
    int64_t bid = blockIdx.x;
    if (CH) {
        if (threadIdx.x == 0) tk = (int)atomicAdd(fi.ticket, 1u);
        __syncthreads();
        bid = tk;
    }
    const int b = (int)(bid % g.nb2);
    const int f = (int)(bid / g.nb2);
    const K2Smem lay = k2_smem(g, KR);
    uint32_t *rowtot = smem + lay.rowtot;                    // [2][G][nwarp][NWp]
    uint32_t *Lsup = smem + lay.Lsup;                        // [2][Lrows][NWp]
    uint32_t *vtot = smem + lay.vtot;                        // [nwarp][NB]
    uint32_t *Tsup = smem + lay.Tsup;                        // [2][NB]
    uint32_t *ptop = smem + lay.ptop + (warp * NB * 32 + lane) * VC;  // this lane's [NB][VC] (stride 32*VC)
    uint32_t *ring = smem + lay.ring + warp * KR * NB * 32 + lane;    // this lane's [KR][NB] (stride 32)
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + lay.bar);    // TMA: [RING] rows staged
    uint64_t *empty = full + (TMA ? g.RING : 0);                      // TMA: [RING] slots read by TMA
    uint32_t *stage = smem + lay.stage;                               // TMA: [RING][bins][SEGW]
    auto csync = [&]() {
        if constexpr (TMA) named_sync(1, 32 * nwarp);
        else __syncthreads();
    };
    if constexpr (TMA) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < g.RING; ++i) {
                mbar_init(full + i, (uint32_t)nwarp);
                mbar_init(empty + i, 1u);
            }
        }
        // plane columns -7..0 of super-strip 0 (column 0 and the sector before it): zero
        for (int i = threadIdx.x; i < g.RING * g.bins * 8; i += blockDim.x)
            stage[(i >> 3) * g.SEGW + (i & 7)] = 0u;
        fence_proxy_async();
        __syncthreads();
        if (warp == nwarp) {  // ---- store warp
            if (lane == 0) {
                const int Ys0 = b * g.R, Ys1 = min(Ys0 + g.R - 1, g.h);
                int32_t *pf = po.pl + (int64_t)f * po.pfs;
                uint32_t r = 0, slot = 0, phase = 0, prev = 0;
                for (int ss = 0; ss < g.nss; ++ss) {
                    const int xss = ss * nwarp * g.Ws;
                    const int cb = ss == 0 ? -7 : xss + 1;  // first plane column copied
                    const int last = min(xss + nwarp * g.Ws, g.w);
                    const int ce = 1 + ((last + 7) & ~7);  // end column (exclusive), 32-B aligned
                    const uint32_t bytes = (uint32_t)(ce - cb) * 4u;
                    const int soff = cb - xss + 7;
                    for (int Y = Ys0; Y <= Ys1; ++Y, ++r) {
                        mbar_wait_sleep(full + slot, phase);
                        const uint32_t *src = stage + slot * g.bins * g.SEGW + soff;
                        int32_t *dst = pf + (int64_t)Y * po.pp + cb;
                        for (int n = 0; n < g.bins; ++n)
                            bulk_store(dst + n * po.pns, src + n * g.SEGW, bytes);
                        bulk_commit();
                        if (r > 0) {  // the previous row's slot has been read: release it
                            bulk_wait_read<1>();
                            mbar_arrive(empty + prev);
                        }
                        prev = slot;
                        if (++slot == (uint32_t)g.RING) slot = 0, phase ^= 1u;
                    }
                }
                bulk_wait_read<0>();
            }
            return;
        }
    }
    uint32_t tslot = 0, tphase = 0, trow = 0;  // TMA ring position of the next stored row
    // RB: a CTA holds whole plane rows (every strip of the frame, nss == 1), the
    // planes are row-major and contiguous per row (pp == bins * pns): each stored
    // row (every bin, columns -7 .. P-8) is staged in one of two shared-memory
    // slots and leaves as ONE contiguous cp.async.bulk, issued by thread 0
    uint32_t rbslot = 0, rbn = 0, rbq = 0;  // RB: slot, rows stored so far, row within the slot
    uint32_t *rbst = smem + lay.stage;  // RB: [K2_RB_SLOTS][K2_RB_ROWS][bins][pns] words
    int32_t *rbdst = nullptr;           // RB: plane address of the slot's first row (column -7)
    const uint32_t rbrows = (uint32_t)(min(b * g.R + g.R - 1, g.h) - b * g.R + 1);  // rows this CTA stores

    const int Y0 = b * g.R;
    const int Ystore = min(Y0 + g.R - 1, g.h);
    const int Ycomp = KR ? max(Ystore, min(Y0 + g.R + g.halo, g.h)) : Ystore;
    const bool odd = (g.bins & 1) != 0;  // the last packed bin is padding
    const int lo = g.Ws / VC - 1;        // last lane owning strip columns
    const int NWp = g.NWp;
    const int64_t pns = po.pns, pp = po.pp;
    const int8_t *bmf = bm + (int64_t)f * bfs;
    int8_t *bmw = const_cast<int8_t *>(bmf);
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
        const int soff = warp * g.Ws + VC * lane + 8;  // TMA: stage column of the lane's first value
        const int gcol = x / ls;
        const uint32_t *rdL = Lsup + (ss & 1) * g.Lrows * NWp;
        uint32_t *wrL = Lsup + ((ss & 1) ^ 1) * g.Lrows * NWp;

        uint32_t Q[NW][VC];
        uint32_t Lacc[NB];
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int k = 0; k < VC; ++k) Q[w][k] = 0;

        // column counts above the band, u16x2 (fused: binning + look-back here)
        uint32_t vreg[NW][VC];
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int k = 0; k < VC; ++k) vreg[w][k] = 0;
        if constexpr (CH > 0) {
            uint32_t cc[VC][NWB];
#pragma unroll
            for (int k = 0; k < VC; ++k)
#pragma unroll
                for (int w = 0; w < NWB; ++w) cc[k][w] = 0;
            const int yown = min(Y0 + g.R, g.h);  // pixel rows of this band
            if (active)
                bin_rows<CH, VC, NWB>(fi, g, f, x, lane, own, Y0, max(Ycomp, yown), yown, bmw, bp, cc);
            // publish this band's per-column counts (aggregate)
            uint32_t *agg = sc.C + ((int64_t)f * g.nb2 + b) * g.Wc * NWB;
            if (active && own) {
#pragma unroll
                for (int k = 0; k < VC; ++k)
                    if (x + k < g.Wc)
#pragma unroll
                        for (int w = 0; w < NWB; ++w) agg[(int64_t)(x + k) * NWB + w] = cc[k][w];
            }
            __threadfence();
            __syncthreads();
            uint32_t *flags = fi.flags + (int64_t)f * g.nb2;
            if (threadIdx.x == 0) st_release_gpu(flags + b, 1u);
            // decoupled look-back over the bands above
            if (active) {
                for (int q = b - 1; q >= 0; --q) {
                    uint32_t fl = 0;
                    if (lane == 0) {
                        while ((fl = ld_acquire_gpu(flags + q)) == 0u) __nanosleep(64);
                    }
                    fl = __shfl_sync(FULL, fl, 0);
                    __threadfence();
                    if (fl == 2u) {
                        const uint32_t *inc = sc.V + ((int64_t)f * g.nb2 + q) * g.Wc * NWp;
#pragma unroll
                        for (int k = 0; k < VC; ++k)
                            if (x + k < g.Wc)
#pragma unroll
                                for (int w = 0; w < NW; ++w) vreg[w][k] += inc[(int64_t)(x + k) * NWp + w];
                        break;
                    }
                    const uint32_t *ag = sc.C + ((int64_t)f * g.nb2 + q) * g.Wc * NWB;
#pragma unroll
                    for (int k = 0; k < VC; ++k)
                        if (x + k < g.Wc)
#pragma unroll
                            for (int w = 0; w < NW; ++w)
                                vreg[w][k] += widen_half(ag[(int64_t)(x + k) * NWB + (w >> 1)], w & 1);
                }
                // publish the inclusive counts (above band b+1)
                uint32_t *incl = sc.V + ((int64_t)f * g.nb2 + b) * g.Wc * NWp;
                if (own) {
#pragma unroll
                    for (int k = 0; k < VC; ++k)
                        if (x + k < g.Wc)
#pragma unroll
                            for (int w = 0; w < NW; ++w)
                                incl[(int64_t)(x + k) * NWp + w] = vreg[w][k] + widen_half(cc[k][w >> 1], w & 1);
                }
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) st_release_gpu(flags + b, 2u);
        } else if (g.NOSCAN) {
            // few sub-bands above any band: the CTA sums their u8x4 counts itself, which
            // saves the carry-scan launch and the V round trip (integral.py:75-79: the
            // column recurrence across bands)
            if (active && b > 0 && x < g.Wc) {
                const uint32_t *cq = sc.C + ((int64_t)f * g.nb1 * g.Wc + x) * NWB;
                const int64_t cstep = (int64_t)g.Wc * NWB;
                for (int q = b * g.S1; q > 0; --q, cq += cstep) {
#pragma unroll
                    for (int k = 0; k < VC; ++k)
#pragma unroll
                        for (int wb = 0; wb < NWB; ++wb) {
                            const uint32_t c4 = __ldg(cq + k * NWB + wb);
                            vreg[2 * wb][k] += widen_half(c4, 0);
                            if (2 * wb + 1 < NW) vreg[2 * wb + 1 < NW ? 2 * wb + 1 : 0][k] += widen_half(c4, 1);
                        }
                }
            }
        } else if (active && (b > 0 || sc.base) && x < g.Wc) {  // band 0: zero, or the slab carry
#pragma unroll
            for (int w = 0; w < NW; ++w)
#pragma unroll
                for (int k = 0; k < VC; ++k) vreg[w][k] = Vb[(int64_t)(x + k) * NWp + w];
        }

        // ---- top row: ptop(X) = sum_{xs <= x' < X} V(x'); strip totals -> left edge
        if (active) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                uint32_t v[VC];
#pragma unroll
                for (int k = 0; k < VC; ++k) v[k] = vreg[w][k];
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
                    if constexpr (PREG) {
#pragma unroll
                        for (int k = 0; k < VC; ++k) preg[PREG ? n : 0][PREG ? k : 0] = pt[k];
                    } else {
#pragma unroll
                        for (int k = 0; k < VC; k += 4)
                            *reinterpret_cast<uint4 *>(ptop + n * 32 * VC + k) =
                                make_uint4(pt[k], pt[k + 1], pt[k + 2], pt[k + 3]);
                    }
                    const uint32_t stot = __shfl_sync(FULL, inc, lo);  // strip total (own lanes)
                    if (lane == 0) vtot[warp * NB + n] = stot;
                }
            }
        }
        csync();
        if (active) {
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                uint32_t T = ss ? Tsup[(ss & 1) * NB + n] : 0u;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < warp) T += vtot[q * NB + n];
                Lacc[n] = T;  // P(Y0, xs)
                if constexpr (FP) {
#pragma unroll
                    for (int k = 0; k < VC; ++k) preg[FP ? n : 0][FP ? k : 0] += T;  // P(Y0, x + k + 1)
                }
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
            if constexpr (TMA) {
                if (trow >= (uint32_t)g.RING) mbar_wait(empty + tslot, tphase ^ 1u);
                if (st) {
                    uint32_t *sp = stage + tslot * g.bins * g.SEGW + soff;
#pragma unroll
                    for (int n = 0; n < NB; ++n) {
                        if (n < NB - 1 || !odd) {
#pragma unroll
                            for (int k = 0; k < VC; k += 4) {
                                const uint4 t4 = *reinterpret_cast<const uint4 *>(ptop + n * 32 * VC + k);
                                const uint32_t add = Lacc[n];
                                *reinterpret_cast<uint4 *>(sp + n * g.SEGW + k) =
                                    make_uint4(t4.x + add + half16(Q[n >> 1][k], n & 1),
                                               t4.y + add + half16(Q[n >> 1][k + 1], n & 1),
                                               t4.z + add + half16(Q[n >> 1][k + 2], n & 1),
                                               t4.w + add + half16(Q[n >> 1][k + 3], n & 1));
                            }
                        }
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(full + tslot);
                ++trow;
                if (++tslot == (uint32_t)g.RING) tslot = 0, tphase ^= 1u;
                return;
            }
            if constexpr (RB) {
                const int64_t rowsz = (int64_t)g.bins * pns;  // words of one staged row
                uint32_t *slotp = rbst + (rbslot * K2_RB_ROWS + rbq) * rowsz;
                if (rbq == 0) rbdst = prow - X0 - 7;
#if K2_RB_DECOUPLED && K2_RB_ROWS == 1
                // the slot is free once warp 0 has waited for the copy that read it
                // (EMPTY, barrier 2, arrived by warp 0 one row earlier)
                if (warp != 0 && rbn > 0) named_sync(2, 32 * nwarp);
#endif
                // columns -7..0 of every bin are zero: written once per slot row at the
                // CTA's first rows (nothing else writes them)
                if (rbn < (uint32_t)(K2_RB_SLOTS * K2_RB_ROWS) && s == 0 && lane < NB && (lane < NB - 1 || !odd)) {
                    uint4 *z = reinterpret_cast<uint4 *>(slotp + lane * pns);
                    z[0] = make_uint4(0, 0, 0, 0);
                    z[1] = make_uint4(0, 0, 0, 0);
                }
                if (st) {
                    uint32_t *sp = slotp + X0 + 7;  // slot column of plane column X0
#pragma unroll
                    for (int n = 0; n < NB; ++n) {
                        if (n < NB - 1 || !odd) {
                            uint32_t vals[VC];
#pragma unroll
                            for (int k = 0; k < VC; ++k)
                                vals[k] = FP ? preg[PREG ? n : 0][PREG ? k : 0]
                                             : preg[PREG ? n : 0][PREG ? k : 0] + Lacc[n] + half16(Q[n >> 1][k], n & 1);
#pragma unroll
                            for (int k = 0; k < VC; k += 4)
                                *reinterpret_cast<uint4 *>(sp + n * pns + k) =
                                    make_uint4(vals[k], vals[k + 1], vals[k + 2], vals[k + 3]);
                        }
                    }
                }
                fence_proxy_async();  // this thread's slot writes -> the async proxy
#if K2_RB_DECOUPLED && K2_RB_ROWS == 1
                // FULL (barrier 1): warps 1.. arrive and go on; warp 0 waits for every
                // warp's part of the row, issues the copy, and then tells the others
                // (EMPTY) that the slot of the next row is free: the copy issued
                // K2_RB_SLOTS - 1 rows ago has been read
                if (warp == 0) {
                    if (lane == 0) bulk_wait_read<K2_RB_SLOTS - 2>();
                    named_sync(1, 32 * nwarp);
                    if (lane == 0) {
                        bulk_store(prow - X0 - 7, slotp, (uint32_t)(g.bins * pns * 4));
                        bulk_commit();
                    }
                    if (rbn + 1 < rbrows) named_arrive(2, 32 * nwarp);
                } else {
                    named_arrive(1, 32 * nwarp);
                }
                ++rbn;
#else
                // a slot of K2_RB_ROWS rows leaves when full (or at the CTA's last row):
                // the copy issued K2_RB_SLOTS - 1 slots ago has read its slot, so the
                // slot written next is free once everyone passes the barrier
                ++rbn;
                if (++rbq == (uint32_t)K2_RB_ROWS || rbn == rbrows) {
                    if (threadIdx.x == 0) bulk_wait_read<K2_RB_SLOTS - 2>();
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        bulk_store(rbdst, rbst + rbslot * K2_RB_ROWS * rowsz, (uint32_t)(rbq * rowsz * 4));
                        bulk_commit();
                    }
                    rbq = 0;
                    if (++rbslot == (uint32_t)K2_RB_SLOTS) rbslot = 0;
                }
                prow += pp;
                return;
#endif
                if (++rbslot == (uint32_t)K2_RB_SLOTS) rbslot = 0;
                prow += pp;
                return;
            }
            if (s == 0 && lane < NB && (lane < NB - 1 || !odd)) {
                // padded column X = 0 of bin `lane`; on aligned rows also the previous
                // row's tail padding, so that sector is written whole
                int32_t *p0 = prow - X0 + lane * pns;
                if (VEC)
                    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p0 - 7), "r"(0)
                                 : "memory");
                else
                    *p0 = 0;
            }
            if constexpr (PAIR) {
                // lane pairs trade halves so that each lane writes 8 adjacent columns of one
                // bin with one 256-bit store: the even lane bin n, the odd lane bin n + 1
                const bool oddl = (lane & 1) != 0;
                const bool stp = oddl ? X0 - 4 <= g.w && active && own : st;  // the pair's even lane stores
                int32_t *pe = prow - (oddl ? 4 : 0) + (oddl ? pns : 0);
                auto value4 = [&](int n, uint32_t (&v)[4]) {
                    if constexpr (PREG) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) v[k] = preg[PREG ? n : 0][PREG ? k : 0];
                    } else {
                        const uint4 t4 = *reinterpret_cast<const uint4 *>(ptop + n * 32 * VC);
                        v[0] = t4.x, v[1] = t4.y, v[2] = t4.z, v[3] = t4.w;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) v[k] += Lacc[n] + half16(Q[n >> 1][k], n & 1);
                };
#pragma unroll
                for (int n = 0; n < NB; n += 2) {
                    uint32_t a[4], b[4];
                    value4(n, a);
                    if (n + 1 < NB - 1 || !odd) {
                        value4(n + 1, b);
                        uint32_t rcv[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) rcv[k] = __shfl_xor_sync(FULL, oddl ? a[k] : b[k], 1);
                        if (stp)
                            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(pe + n * pns),
                                         "r"(oddl ? rcv[0] : a[0]), "r"(oddl ? rcv[1] : a[1]),
                                         "r"(oddl ? rcv[2] : a[2]), "r"(oddl ? rcv[3] : a[3]),
                                         "r"(oddl ? b[0] : rcv[0]), "r"(oddl ? b[1] : rcv[1]),
                                         "r"(oddl ? b[2] : rcv[2]), "r"(oddl ? b[3] : rcv[3])
                                         : "memory");
                    } else if (st) {  // odd bin count: the last bin leaves as before
                        *reinterpret_cast<int4 *>(prow + n * pns) = make_int4((int)a[0], (int)a[1], (int)a[2], (int)a[3]);
                    }
                }
                prow += pp;
                return;
            }
            if (st) {
                int32_t *p = prow;
                const int valid = g.w - X0 + 1;
#pragma unroll
                for (int n = 0; n < NB; ++n) {
                    if (n < NB - 1 || !odd) {
                        uint32_t vals[VC];
                        if constexpr (PREG) {
#pragma unroll
                            for (int k = 0; k < VC; ++k) vals[k] = preg[PREG ? n : 0][PREG ? k : 0];
                        } else {
#pragma unroll
                            for (int k = 0; k < VC; k += 4) {
                                const uint4 t4 = *reinterpret_cast<const uint4 *>(ptop + n * 32 * VC + k);
                                vals[k] = t4.x;
                                vals[k + 1] = t4.y;
                                vals[k + 2] = t4.z;
                                vals[k + 3] = t4.w;
                            }
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
                const uint32_t pt_last = PREG ? preg[PREG ? n : 0][PREG ? VC - 1 : 0] : ptop[n * 32 * VC + VC - 1];
                const uint32_t lv = FP ? pt_last : pt_last + Lacc[n] + half16(Q[n >> 1][VC - 1], n & 1);
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
                if (go.u8) {  // cell counts <= cell^2 <= 255: one byte per bin
                    uint8_t *gp8 = reinterpret_cast<uint8_t *>(go.grid) + (gptr - go.grid);
                    if ((g.bins & 3) == 0) {
#pragma unroll
                        for (int n = 0; n + 3 < NB; n += 4)
                            *reinterpret_cast<uint32_t *>(gp8 + n) =
                                __byte_perm(__byte_perm(gv[n], gv[n + 1], 0x0040),
                                            __byte_perm(gv[n + 2], gv[n + 3], 0x0040), 0x5410);
                    } else {
#pragma unroll
                        for (int n = 0; n < NB; ++n)
                            if (n < NB - 1 || !odd) gp8[n] = (uint8_t)gv[n];
                    }
                } else if ((g.bins & 3) == 0) {
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

        if (active || TMA) store_row();  // (TMA: idle warps still pass every ring slot)
        if (active && KR) lattice();

        const int8_t *brow = bmf + (int64_t)Y0 * bp + x;
        const bool bin_ok = active && x < g.w;
        const int bvalid = g.w - x;  // bytes of the lane's chunk inside the frame
        // prefetch: raw loads only, so that nothing waits on them until the
        // group that consumes them (bytes past w are masked at use, mask_bm)
        auto load_bm = [&](int rel) -> BmWord<VC> {
            BmWord<VC> r;
            const bool ok = bin_ok && Y0 + rel < Ycomp;
            if constexpr (VC == 8) {
                const uint2 v = ok ? __ldg(reinterpret_cast<const uint2 *>(brow + (int64_t)rel * bp))
                                   : make_uint2(0xffffffffu, 0xffffffffu);
                r.lo = v.x;
                r.hi = v.y;
            } else {
                r.w = ok ? __ldg(reinterpret_cast<const uint32_t *>(brow + (int64_t)rel * bp)) : 0xffffffffu;
            }
            return r;
        };
        uint32_t mlo = 0, mhi = 0;  // bytes past w count nowhere
        if constexpr (VC == 8) {
            if (bvalid < 8) {
                if (bvalid < 4) mlo = 0xffffffffu << (8 * max(bvalid, 0)), mhi = 0xffffffffu;
                else mhi = 0xffffffffu << (8 * (bvalid - 4));
            }
        } else {
            if (bvalid < 4) mlo = 0xffffffffu << (8 * max(bvalid, 0));
        }
        auto mask_bm = [&](BmWord<VC> r) -> BmWord<VC> {
            if constexpr (VC == 8) {
                r.lo |= mlo;
                r.hi |= mhi;
            } else {
                r.w |= mlo;
            }
            return r;
        };

        BmWord<VC> nxt[G];
#pragma unroll
        for (int i = 0; i < G; ++i) nxt[i] = load_bm(i);
        int latc = ls;  // rows until the next lattice row
        // Phase A scans one-hot counts of G rows.  With 4 columns per lane a strip
        // row holds <= 128 pixels, so four bins share a word (u8x4) and the scan
        // needs half the shuffles; with 8 columns per lane counts reach 256 and
        // two bins share a word (u16x2).
        constexpr bool S8 = VC == 4;
        constexpr int SW = S8 ? (NB + 3) / 4 : NW;  // scanned words per row
        constexpr int NE = G * NW;                  // carry entries per group
        for (int rel = 0; Y0 + rel < Ycomp; rel += G) {
            const int gp = (rel / G) & 1;
            BmWord<VC> bw[G];
            uint32_t ex[G][SW];
            uint32_t *rt_grp = rowtot + gp * G * nwarp * NWp;  // [G][nwarp][NWp] (u8x4 or u16x2)
            // ---- phase A: G rows of warp scans (independent) + strip row totals
            if (active) {
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    bw[i] = mask_bm(nxt[i]);
                    nxt[i] = load_bm(rel + G + i);  // next group in flight during this one
                }
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    uint32_t tot[SW];
#pragma unroll
                    for (int w = 0; w < SW; ++w) tot[w] = 0;
#pragma unroll
                    for (int k = 0; k < VC; ++k) {
                        const uint32_t s = bw[i].byte(k) << (S8 ? 3 : 4);
#pragma unroll
                        for (int w = 0; w < SW; ++w) tot[w] += shl_clamp(1u, s - 32u * w);
                    }
#pragma unroll
                    for (int w = 0; w < SW; ++w) {
                        const uint32_t inc = warp_incl_scan(tot[w], lane);
                        ex[i][w] = inc - tot[w];  // strip-exclusive count (no borrow: inc >= tot per lane)
                        const uint32_t rt = __shfl_sync(FULL, inc, lo);
                        if (lane == 0) rt_grp[(i * nwarp + warp) * NWp + w] = rt;
                    }
                }
            }
            csync();
            // ---- phase B: carries, accumulate, store, lattice
            // row-carry of (row i, word w) into this strip, one entry per lane:
            // Lc = (carry left of this super-strip) + sum of the strip totals to the left
            uint32_t Lsum[(NE + 31) / 32];
            if (active) {
#pragma unroll
                for (int r = 0; r < (NE + 31) / 32; ++r) {
                    const int e = lane + 32 * r;
                    uint32_t L = 0, own_t = 0;
                    if (e < NE) {
                        const int i = e / NW, w = e % NW;
                        L = ss ? rdL[(rel + i) * NWp + w] : 0u;
                        const uint32_t *rq = rt_grp + i * nwarp * NWp;
                        for (int q = 0; q <= warp; ++q) {
                            const uint32_t t = S8 ? widen_half(rq[q * NWp + (w >> 1)], w & 1)
                                                  : rq[q * NWp + w];
                            if (q < warp) L += t;
                            else own_t = t;
                        }
                        if (last_warp && Y0 + rel + i < Ycomp) wrL[(rel + i) * NWp + w] = L + own_t;
                    }
                    Lsum[r] = L;
                }
            }
            // row i of the group: row carries (Lacc) and the strip sums Q
            auto row_update = [&](int i) {
                        uint32_t Lrow[FP ? NB : 1];  // FP: the row's carry into the strip, per bin
#pragma unroll
                        for (int w = 0; w < NW; ++w) {
                            const int e = i * NW + w;
                            const uint32_t L = __shfl_sync(FULL, Lsum[e / 32], e % 32);
                            Lacc[2 * w] += L & 0xffffu;
                            Lacc[2 * w + 1] += L >> 16;
                            if constexpr (FP) {
                                Lrow[FP ? 2 * w : 0] = L & 0xffffu;
                                Lrow[FP ? 2 * w + 1 : 0] = L >> 16;
                            }
                        }
                        if constexpr (FP) {
                            // P(Y+1, x+k+1) = P(Y, x+k+1) + Lrow + (strip-row prefix through column x+k)
                            uint32_t r8[SW];
#pragma unroll
                            for (int j = 0; j < SW; ++j) r8[j] = ex[i][j];
#pragma unroll
                            for (int k = 0; k < VC; ++k) {
                                const uint32_t s8 = bw[i].byte(k) << 3;
#pragma unroll
                                for (int j = 0; j < SW; ++j) r8[j] += shl_clamp(1u, s8 - 32u * j);
#pragma unroll
                                for (int n = 0; n < NB; ++n)
                                    preg[FP ? n : 0][FP ? k : 0] += Lrow[FP ? n : 0] + byte_of(r8[n >> 2], n & 3);
                            }
                        } else if constexpr (S8) {
                            // strip-row prefix in u8x4 (<= 128 per bin), widened per column
                            uint32_t r8[SW];
#pragma unroll
                            for (int j = 0; j < SW; ++j) r8[j] = ex[i][j];
#pragma unroll
                            for (int k = 0; k < VC; ++k) {
                                const uint32_t s8 = bw[i].byte(k) << 3;
#pragma unroll
                                for (int j = 0; j < SW; ++j) r8[j] += shl_clamp(1u, s8 - 32u * j);
#pragma unroll
                                for (int w = 0; w < NW; ++w) Q[w][k] += widen_half(r8[w >> 1], w & 1);
                            }
                        } else {
                            uint32_t s16[VC];  // bit offset of the pixel's bin in u16x2 words
#pragma unroll
                            for (int k = 0; k < VC; ++k) s16[k] = bw[i].byte(k) << 4;
#pragma unroll
                            for (int w = 0; w < NW; ++w) {
                                uint32_t run = ex[i][w];
#pragma unroll
                                for (int k = 0; k < VC; ++k) {
                                    run += shl_clamp(1u, s16[k] - 32u * w);
                                    Q[w][k] += run;
                                }
                            }
                        }
            };
            // Full groups (every row computed and stored, no TMA ring): the same rows
            // without per-row guards, so the group compiles to straight-line code
            const bool fullg = !TMA && active && Y0 + rel + G <= Ycomp && Y0 + rel + G <= Ystore;
            // measured: +0.3 % c2, +1 % c1; -0.3 % c4 (VC = 8), -4.5 % c5 (NW = 9: the duplicated body)
            if (K2_FASTGROUP && VC == 4 && NW <= 4 && fullg) {
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    row_update(i);
                    store_row();
                    if (KR && --latc == 0) {
                        latc = ls;
                        lattice();
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < G; ++i) {
                    if (Y0 + rel + i < Ycomp) {
                        if (active) row_update(i);
                        if (Y0 + rel + i + 1 <= Ystore && (active || TMA)) store_row();
                        if (active && KR && --latc == 0) {
                            latc = ls;
                            lattice();
                        }
                    }
                }
            }
        }
        csync();
    }
    if constexpr (RB) {
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <int NW, int KR, int VC, bool VEC, int CH, bool TMA = false, bool PR = false, bool RB = false>
void launch_planes_vc(const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                      const GridOut &go, const TileGeom &g, const Scratch &sc, const FusedIn &fi,
                      cudaStream_t st) {
    const size_t smem = (size_t)k2_smem_words(g, KR) * 4;
    static size_t configured[HOG_MAX_DEVICES] = {};  // per instantiation and device
    if (smem_optin_needed(configured, smem))
        cudaFuncSetAttribute(k_planes<NW, KR, VC, VEC, CH, TMA, PR, RB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_planes<NW, KR, VC, VEC, CH, TMA, PR, RB>
        <<<(unsigned)((int64_t)g.n * g.nb2), 32 * (g.NWARP + (TMA ? 1 : 0)), smem, st>>>(
            bm, bp, bfs, po, go, g, sc, fi);
}

template <int NW, int KR>
void launch_planes_kr(int ch, const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                      const GridOut &go, const TileGeom &g, const Scratch &sc, const FusedIn &fi,
                      cudaStream_t st) {
    if constexpr (HOGB200_VARIANTS) {  // experiment builds only (measured slower)
        if (ch == 1) {  // fused, grayscale
            if constexpr (NW <= 5) {
                if (g.VC == 8) return launch_planes_vc<NW, KR, 8, true, 1>(bm, bp, bfs, po, go, g, sc, fi, st);
            }
            return launch_planes_vc<NW, KR, 4, true, 1>(bm, bp, bfs, po, go, g, sc, fi, st);
        }
        if (ch == 3) {  // fused, RGB
            if constexpr (NW <= 5) {
                if (g.VC == 8) return launch_planes_vc<NW, KR, 8, true, 3>(bm, bp, bfs, po, go, g, sc, fi, st);
            }
            return launch_planes_vc<NW, KR, 4, true, 3>(bm, bp, bfs, po, go, g, sc, fi, st);
        }
        if (g.TMA) {  // plane rows through shared memory and TMA bulk stores (requires po.vec)
            if constexpr (NW <= 5) {
                if (g.VC == 8) return launch_planes_vc<NW, KR, 8, true, 0, true>(bm, bp, bfs, po, go, g, sc, fi, st);
            }
            return launch_planes_vc<NW, KR, 4, true, 0, true>(bm, bp, bfs, po, go, g, sc, fi, st);
        }
    }
    if constexpr (NW <= 5) {
        if (g.VC == 8) return launch_planes_vc<NW, KR, 8, true, 0>(bm, bp, bfs, po, go, g, sc, fi, st);
    }
    if constexpr (2 * NW * 4 <= 32) {
        if (g.PREG) {
            if constexpr (NW == 4) {
                if (g.RB && po.vec)
                    return launch_planes_vc<NW, KR, 4, true, 0, false, true, true>(bm, bp, bfs, po, go, g, sc, fi, st);
            }
            if (po.vec)
                return launch_planes_vc<NW, KR, 4, true, 0, false, true>(bm, bp, bfs, po, go, g, sc, fi, st);
            return launch_planes_vc<NW, KR, 4, false, 0, false, true>(bm, bp, bfs, po, go, g, sc, fi, st);
        }
    }
    if (po.vec)
        launch_planes_vc<NW, KR, 4, true, 0>(bm, bp, bfs, po, go, g, sc, fi, st);
    else
        launch_planes_vc<NW, KR, 4, false, 0>(bm, bp, bfs, po, go, g, sc, fi, st);
}

template <int NW>
void launch_planes_t(int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs, const PlaneOut &po,
                     const GridOut &go, const TileGeom &g, const Scratch &sc, const FusedIn &fi,
                     cudaStream_t st) {
    if (kr == 0)
        launch_planes_kr<NW, 0>(ch, bm, bp, bfs, po, go, g, sc, fi, st);
    else if (kr == 1)
        launch_planes_kr<NW, 1>(ch, bm, bp, bfs, po, go, g, sc, fi, st);
    else
        launch_planes_kr<NW, 2>(ch, bm, bp, bfs, po, go, g, sc, fi, st);
}

}  // namespace hogb200
