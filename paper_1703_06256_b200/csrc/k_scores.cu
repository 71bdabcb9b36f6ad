// k_scores.cu -- window scores on a regular cell lattice, unnormalised grid
// (detector.py:140-154 with DescriptorGeometry(block=1, block_stride=1),
// descriptor.py:107-118).  The window at lattice origin (iy, ix) reads cells
// (iy + cy*K, ix + cx*K), cy < cells_y, cx < 8, so the score map is a 2-D
// correlation of the cell grid with the weight tensor w[cy][cx][n], plus the
// bias.  fp64 accumulation (fp32 misses 1e-5 on blurred
// inputs); the summation order differs from OpenBLAS ddot, which the 1e-5
// relative tolerance allows (measured: ~1e-15).
//
// FP64-FMA-bound design (c5: 2304 FMAs per window, 3.7 G per frame):
//   A warp owns TY (4 or 5) window rows x 32*TX window columns and streams the
//   TY + (cells_y-1)*K grid rows they read through its own two-slot ring
//   in shared memory (no CTA-wide barrier, so warps never wait on rows they
//   do not use).  Row r+1 is copied by cp.async (4-byte, zero-fill past the
//   frame) while row r is consumed.  Slots are int32 [column/TX][column%TX][bin]
//   with one pad word per TX columns: lane L reads column TX*L + j at word
//   L*(TX*bins+1) + ..., an odd lane stride, so the reads are conflict-free.
//   Per (row, bin) a lane converts its TX + 7K grid values to double once and
//   reuses them for the TY window rows that read that grid row (sr_row:
//   one unrolled body per active-row mask, so no FMA is spent on rows that
//   do not read it); weights are warp-broadcast LDS.128.
//
// uint8 grid (U8, cell counts <= 64 stored as bytes by the plane kernel): a
//   staged row is the contiguous byte run of the grid row, copied by 16-byte
//   cp.async.cg from the 16-byte-aligned address at or below it (zero-fill
//   past the end of the grid), read at a per-row byte offset.  A slot is ~4x
//   smaller than the int32 one: at N_b = 18 the int32 ring (96 KB) allowed
//   one CTA (4 warps) per SM, the byte ring allows four.
#include <type_traits>

#include "hog_common.cuh"

namespace hogb200 {

constexpr int SR_WARPS = 4;  // window rows per warp: the template parameter TY (4 or 5)

// Active-row masks a grid row can produce: for K = 1 a contiguous run of
// bits, for K = 2 a contiguous run of one parity (bits p, p+2, ...).
__host__ __device__ constexpr bool sr_mask_ok(int k, int m) {
    if (m <= 0) return false;
    while (!(m & 1)) m >>= 1;
    if (k == 1) return (m & (m + 1)) == 0;
    for (; m; m >>= 2)
        if ((m & 3) != 1 && m != 1) return false;
    return true;
}

__device__ __forceinline__ void cp_async4(uint32_t *sdst, const int32_t *gsrc, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(sdst)), "l"(gsrc),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void *sdst, const void *gsrc, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(sdst)), "l"(gsrc),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__host__ __device__ constexpr int sr_span(int tx, int k) { return 32 * tx + 7 * k; }
// words of one staged grid row: int32, ceil(span/tx) chunks of tx columns x
// bins + 1 pad; uint8, the row's span*bins bytes + up to 15 bytes of leading
// misalignment, in whole 16-byte chunks
__host__ __device__ inline int sr_slot_words(int bins, int tx, int k, bool u8 = false) {
    if (u8) return (sr_span(tx, k) * bins + 15 + 15) / 16 * 4;
    return ((sr_span(tx, k) + tx - 1) / tx) * (tx * bins + 1);
}

// One staged grid row against the window rows of MASK (bit u: window row
// iyw + u reads this grid row, with weight row (rr - u) / K, rr = r - iyw).
// Only active rows are computed: with a runtime zero-weight row instead, a
// warp's 4 window rows would do 19 rows of FMAs for 16 useful ones (K = 1) or
// twice the useful work (K = 2, where alternate rows are inactive).
template <int K, int TX, int BINS, bool U8, int TY, int MASK>
__device__ __forceinline__ void sr_row(double (&acc)[TY][TX], const double *__restrict__ wsm,
                                       int bins, int rr, const uint32_t *row, const uint8_t *rowb,
                                       int ctb) {
    constexpr int CX = 8, NG = TX / K + CX - 1;
    const double *wu[TY];
#pragma unroll
    for (int u = 0; u < TY; ++u) wu[u] = wsm + ((MASK >> u) & 1 ? (rr - u) / K : 0) * bins * CX;
    for (int bn = 0; bn < bins; ++bn) {
#pragma unroll
        for (int p = 0; p < K; ++p) {
            double gs[NG];
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const int c = p + K * j;  // column c0 + c
                if constexpr (U8)
                    gs[j] = (double)(uint32_t)rowb[c * bins + bn];
                else
                    gs[j] = (double)(int)row[(c / TX) * (ctb + 1) + (c % TX) * bins + bn];
            }
#pragma unroll
            for (int cx = 0; cx < CX; cx += 2) {
                double2 w2[TY];
#pragma unroll
                for (int u = 0; u < TY; ++u)
                    if ((MASK >> u) & 1) w2[u] = *reinterpret_cast<const double2 *>(wu[u] + bn * CX + cx);
#pragma unroll
                for (int u = 0; u < TY; ++u)
                    if ((MASK >> u) & 1) {
#pragma unroll
                        for (int t = 0; t < TX / K; ++t) {
                            acc[u][K * t + p] = fma(w2[u].x, gs[t + cx], acc[u][K * t + p]);
                            acc[u][K * t + p] = fma(w2[u].y, gs[t + cx + 1], acc[u][K * t + p]);
                        }
                    }
            }
        }
    }
}

// if-chain over the masks valid for (K, TY): one unrolled sr_row per mask
template <int K, int TX, int BINS, bool U8, int TY, int M = 1>
__device__ __forceinline__ void sr_dispatch(int mask, double (&acc)[TY][TX],
                                            const double *__restrict__ wsm, int bins, int rr,
                                            const uint32_t *row, const uint8_t *rowb, int ctb) {
    if constexpr (M < (1 << TY)) {
        if constexpr (sr_mask_ok(K, M)) {
            if (mask == M) return sr_row<K, TX, BINS, U8, TY, M>(acc, wsm, bins, rr, row, rowb, ctb);
        }
        sr_dispatch<K, TX, BINS, U8, TY, M + 1>(mask, acc, wsm, bins, rr, row, rowb, ctb);
    }
}

// TX window columns per lane (32*TX per warp); BINS > 0: bin count known at
// compile time (shared-memory offsets become immediates), 0: runtime `bins`.
template <int K, int TX, int BINS, bool U8, int TY>
__global__ void __launch_bounds__(32 * SR_WARPS, 3)
k_scores_rows(const void *__restrict__ grid_v, int n, int ncy, int ncx, int bins_rt, int noy,
              int nox, int cells_y, const double *__restrict__ wts, double bias,
              double *__restrict__ scores, uint32_t magic) {
    using T = typename std::conditional<U8, uint8_t, int32_t>::type;
    const T *__restrict__ grid = static_cast<const T *>(grid_v);
    constexpr int CX = 8;
    constexpr int SPAN = sr_span(TX, K);  // grid columns a warp reads
    constexpr int NG = TX / K + CX - 1;   // grid values per (row, bin, parity)
    constexpr int COLS = 32 * TX;
    const int bins = BINS > 0 ? BINS : bins_rt;
    extern __shared__ __align__(16) double ssm[];
    double *wsm = ssm;  // [cells_y][bins][8]
    const int slotw = sr_slot_words(bins, TX, K, U8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *ring = reinterpret_cast<uint32_t *>(ssm + (size_t)cells_y * bins * CX) + warp * 2 * slotw;
    const int tiles_x = (nox + COLS - 1) / COLS;
    const int tiles_y = (noy + TY * SR_WARPS - 1) / (TY * SR_WARPS);
    int bid = blockIdx.x;
    const int tx = bid % tiles_x;
    bid /= tiles_x;
    const int ty = bid % tiles_y;
    const int f = bid / tiles_y;
    const int ix0 = tx * COLS;
    const int iyw = ty * TY * SR_WARPS + warp * TY;  // this warp's first window row
    const T *gf = grid + (int64_t)f * ncy * ncx * bins;
    const int64_t gtotal = (int64_t)n * ncy * ncx * bins;  // grid elements (bytes if U8)

    for (int i = threadIdx.x; i < cells_y * CX * bins; i += blockDim.x) {
        const int n = i % bins, cx = (i / bins) % CX, cy = i / (bins * CX);
        wsm[(cy * bins + n) * CX + cx] = wts[i];
    }
    __syncthreads();  // the only CTA-wide barrier: weights staged
    if (iyw >= noy) return;

    const int nel = min(SPAN, ncx - ix0) * bins;  // words of a row inside the frame
    const int ctb = TX * bins;  // words of a chunk of TX columns (+1 pad word)
    auto stage = [&](int r, uint32_t *dst) {  // async copy of grid row r (this warp's columns)
        if constexpr (U8) {
            // the 16-byte-aligned ADDRESSES at or below the row start (the grid pointer
            // itself may be unaligned: a frame group's slice of a batch grid); zero-fill
            // past the end of the grid; values past the frame's right edge only feed
            // window columns that are not stored
            const uintptr_t a = reinterpret_cast<uintptr_t>(grid) +
                                (uintptr_t)((((int64_t)f * ncy + r) * ncx + ix0) * bins);
            const uintptr_t a0 = a & ~(uintptr_t)15;
            const uintptr_t end = reinterpret_cast<uintptr_t>(grid) + (uintptr_t)gtotal;
            const int nch = (int)((a - a0) + SPAN * bins + 15) / 16;
            for (int e = lane; e < nch; e += 32) {
                const uintptr_t o = a0 + 16 * (uintptr_t)e;
                const int bytes = o + 16 <= end ? 16 : (o < end ? (int)(end - o) : 0);
                cp_async16(dst + 4 * e, reinterpret_cast<const void *>(bytes ? o : a0), bytes);
            }
        } else {
            const int32_t *src = gf + ((int64_t)r * ncx + ix0) * bins;
            const bool rok = r < ncy;
            for (int e = lane; e < SPAN * bins; e += 32) {
                const int q = (int)__umulhi((uint32_t)e, magic);  // e / (TX*bins)
                const bool ok = rok && e < nel;
                cp_async4(dst + e + q, ok ? src + e : (const int32_t *)gf, ok);
            }
        }
        cp_async_commit();
    };
    double acc[TY][TX];
#pragma unroll
    for (int u = 0; u < TY; ++u)
#pragma unroll
        for (int t = 0; t < TX; ++t) acc[u][t] = 0.0;

    const int r_first = iyw;
    const int r_last = min(iyw + TY - 1, noy - 1) + (cells_y - 1) * K;
    stage(r_first, ring);
    // lane L's columns start at TX*L, the first column of chunk L: lane stride TX*bins+1 (odd)
    const int c0 = TX * lane;
    const int lbase = lane * (ctb + 1);
    for (int r = r_first; r <= r_last; ++r) {
        const int slot = (r - r_first) & 1;
        cp_async_wait_all();
        __syncwarp();  // row r visible to the warp; the other slot is free
        if (r < r_last) stage(r + 1, ring + (slot ^ 1) * slotw);
        const uint32_t *row = ring + slot * slotw + lbase;
        const uint8_t *rowb = nullptr;
        if constexpr (U8) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(grid) +
                                (uintptr_t)((((int64_t)f * ncy + r) * ncx + ix0) * bins);
            rowb = reinterpret_cast<const uint8_t *>(ring + slot * slotw) + (int)(a & 15) +
                   c0 * bins;
        }
        // window rows reading grid row r: u with d = rr - u in [0, (cells_y-1)*K], d % K == 0
        const int rr = r - iyw;
        int mask = 0;
#pragma unroll
        for (int u = 0; u < TY; ++u) {
            const int d = rr - u;
            if (d >= 0 && d % K == 0 && d / K < cells_y) mask |= 1 << u;
        }
sr_dispatch<K, TX, BINS, U8, TY>(mask, acc, wsm, bins, rr, row, rowb, ctb);
    }
#pragma unroll
    for (int u = 0; u < TY; ++u) {
        const int iy = iyw + u;
        if (iy >= noy) continue;
        double *sp = scores + ((int64_t)f * noy + iy) * nox + ix0 + c0;
#pragma unroll
        for (int t = 0; t < TX; ++t)
            if (ix0 + c0 + t < nox) sp[t] = acc[u][t] + bias;
    }
}

size_t scores_rows_smem(int bins, int cells_y, int tx, int k, bool u8) {
    return sizeof(double) * (size_t)cells_y * bins * 8 +
           sizeof(uint32_t) * (size_t)SR_WARPS * 2 * sr_slot_words(bins, tx, k, u8);
}

template <int K, int TX, int BINS, bool U8, int TY>
void launch_rows_ty(const void *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                    int cells_y, const double *wts, double bias, double *scores, cudaStream_t st) {
    const size_t smem = scores_rows_smem(bins, cells_y, TX, K, U8);
    static size_t configured[HOG_MAX_DEVICES] = {};
    if (smem_optin_needed(configured, smem))
        cudaFuncSetAttribute(k_scores_rows<K, TX, BINS, U8, TY>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // e / (TX bins) by multiply-high: exact for e < 2^20 (e < span * bins here)
    const uint32_t magic = (uint32_t)((0x100000000ull + TX * bins - 1) / (TX * bins));
    const int64_t blocks = (int64_t)n * ((noy + TY * SR_WARPS - 1) / (TY * SR_WARPS)) *
                           ((nox + 32 * TX - 1) / (32 * TX));
    k_scores_rows<K, TX, BINS, U8, TY><<<(unsigned)blocks, 32 * SR_WARPS, smem, st>>>(
        grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, magic);
}

// Window rows per warp: 5 instead of 4 when that takes fewer CTA waves of the
// same occupancy, by the model time ~ waves x (FMA rows + 0.3 x staged rows)
// of a task.  c4 (75 window rows x 256 frames, 4 CTAs/SM): 2.16 -> 1.73
// waves.  Only for the byte grid at stride = cell (K = 1).
template <int K, int TX, int BINS, bool U8>
void launch_rows_t(const void *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                   int cells_y, const double *wts, double bias, double *scores, cudaStream_t st) {
    if constexpr (U8 && K == 1) {
        const char *e = getenv("HOGB200_SCORES_TY");
        int ty = e ? atoi(e) : 0;
        if (ty != 4 && ty != 5) {
            const int tiles_x = (nox + 32 * TX - 1) / (32 * TX);
            double cost[2];
            for (int i = 0; i < 2; ++i) {
                const int t = 4 + i;
                const size_t smem = scores_rows_smem(bins, cells_y, TX, K, U8);
                int per_sm = 0;
                if (t == 4)
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                        &per_sm, k_scores_rows<K, TX, BINS, U8, 4>, 32 * SR_WARPS, smem);
                else
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                        &per_sm, k_scores_rows<K, TX, BINS, U8, 5>, 32 * SR_WARPS, smem);
                int sms = 148;
                int dev = 0;
                if (cudaGetDevice(&dev) == cudaSuccess)
                    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                const int64_t blocks = (int64_t)n * tiles_x * ((noy + t * SR_WARPS - 1) / (t * SR_WARPS));
                const int64_t slots = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
                const double waves = (double)((blocks + slots - 1) / slots);
                cost[i] = waves * (t * cells_y + 0.3 * (t + cells_y - 1));
            }
            ty = cost[1] < 0.97 * cost[0] ? 5 : 4;
        }
        if (ty == 5)
            return launch_rows_ty<K, TX, BINS, U8, 5>(grid, n, ncy, ncx, bins, noy, nox, cells_y,
                                                      wts, bias, scores, st);
    }
    launch_rows_ty<K, TX, BINS, U8, 4>(grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias,
                                       scores, st);
}

template <int K, int TX, bool U8>
void launch_rows_b(const void *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                   int cells_y, const double *wts, double bias, double *scores, cudaStream_t st) {
#define SRB_ARGS grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st
    switch (bins) {
        case 8: return launch_rows_t<K, TX, 8, U8>(SRB_ARGS);
        case 9: return launch_rows_t<K, TX, 9, U8>(SRB_ARGS);
        case 18: return launch_rows_t<K, TX, 18, U8>(SRB_ARGS);
        default: return launch_rows_t<K, TX, 0, U8>(SRB_ARGS);
    }
#undef SRB_ARGS
}

// Window columns per lane: the candidate (TX / K integral) that wastes the
// fewest lanes on this width (ties to the larger TX: more reuse per grid
// value), e.g. c4 (153 columns) -> 5 (160, 96 %), c1 (93) -> 3, 8K (953) -> 5.
int pick_tx(int nox, int k) {
    static const int c1[] = {5, 6, 4, 3, 2}, c2[] = {6, 4, 2};
    const int *c = k == 1 ? c1 : c2;
    const int nc = k == 1 ? 5 : 3;
    int best = c[0];
    int64_t best_pad = INT64_MAX;
    for (int i = 0; i < nc; ++i) {
        const int64_t cols = 32 * c[i], pad = (nox + cols - 1) / cols * cols;
        if (pad < best_pad) best_pad = pad, best = c[i];
    }
    return best;
}

template <bool U8>
void scores_rows_t(const void *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                   int cells_y, int k, const double *wts, double bias, double *scores,
                   cudaStream_t st) {
    const int tx = pick_tx(nox, k);
#define SR_ARGS grid, n, ncy, ncx, bins, noy, nox, cells_y, wts, bias, scores, st
    if (k == 1) {
        switch (tx) {
            case 2: return launch_rows_b<1, 2, U8>(SR_ARGS);
            case 3: return launch_rows_b<1, 3, U8>(SR_ARGS);
            case 4: return launch_rows_b<1, 4, U8>(SR_ARGS);
            case 5: return launch_rows_b<1, 5, U8>(SR_ARGS);
            default: return launch_rows_b<1, 6, U8>(SR_ARGS);
        }
    }
    switch (tx) {
        case 2: return launch_rows_b<2, 2, U8>(SR_ARGS);
        case 4: return launch_rows_b<2, 4, U8>(SR_ARGS);
        default: return launch_rows_b<2, 6, U8>(SR_ARGS);
    }
#undef SR_ARGS
}

void launch_scores_rows(const int32_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                        int cells_y, int k, const double *wts, double bias, double *scores,
                        cudaStream_t st) {
    scores_rows_t<false>(grid, n, ncy, ncx, bins, noy, nox, cells_y, k, wts, bias, scores, st);
}

void launch_scores_rows_u8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy,
                           int nox, int cells_y, int k, const double *wts, double bias,
                           double *scores, cudaStream_t st) {
    scores_rows_t<true>(grid, n, ncy, ncx, bins, noy, nox, cells_y, k, wts, bias, scores, st);
}

}  // namespace hogb200
