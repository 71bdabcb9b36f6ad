// k_scores_i8.cu -- window scores on the integer tensor cores, exact.
//
// detector.py:140-154 / descriptor.py:107-118 with block = 1, no
// normalisation, stride = cell: score(oy, ox) = bias + sum_{cy, cx, n}
// w[cy][cx][n] * G[oy + cy][ox + cx][n], G the uint8 cell grid (counts
// <= 64).  The reference evaluates the dot in float64; here it is evaluated
// EXACTLY in integers and rounded once:
//
//   * the host (hog_scores_i8_prepare) writes every weight as an integer
//     W = w * 2^F (exact: the float32-valued weights of a LinearModel span
//     ~37 bits) in S signed base-256 digits d_s (int8), W = sum_s d_s 256^s;
//   * per grid row y the tensor cores form, for 16 window positions and
//     every (digit s, cell row cy), P = sum_{cx, n} d_s[cy][cx][n] *
//     G[y][ox + cx][n]  (mma.sync m16n8k32 s8 x s8 -> s32, exact: |P| <= 2^16);
//   * V(cy, ox) = sum_s P_s << 8s is exact in int64, and the 16 cell rows
//     of a window are summed by a systolic pass through the lanes (row y's
//     cell row cy belongs to window row y - cy), exact in int64
//     (|sum| <= 8192 * 2^(8S-1) < 2^60);
//   * score = (double)sum * 2^-F + bias: one rounding of the exact dot.
//
// Operands: A (16 x 32, row) = the digit weights, rows (cy), one m16 tile
// per digit, held in registers for the whole kernel; B (32 x 8, col) = 8
// window positions' 32-byte slice of their window-row vector (8 cells x P
// bins, P = bins rounded up to 4 with zero pad), read from the staged grid
// row by one 32-bit LDS each: position p's vector starts at byte p * P.
// D (16 x 8): lane (g, t) holds cell rows g, g+8 of positions 2t, 2t+1.
//
// Work: a warp owns 16 window columns of a band of T window rows and walks
// the T + 15 grid rows the band reads; a CTA is 8 warps (128 columns).  A
// grid row is staged per warp (23 cells, re-pitched from `bins` to P bytes
// per cell), two rows ahead in registers.
#include "hog_common.cuh"

namespace hogb200 {

constexpr int I8_WARPS = 8;
constexpr int I8_COLS = 16 * I8_WARPS;  // window columns per CTA
constexpr int I8_CELLS = 16 + 7;        // grid cells a warp stages per row
constexpr int I8_CY = 16;               // cell rows of the systolic window sum

__device__ __forceinline__ void mma_s8(int (&d)[4], const uint4 &a, uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// KS: 32-byte k steps of a window row (P = 4 KS bytes per cell); S: digits.
template <int KS, int S>
__global__ void __launch_bounds__(32 * I8_WARPS, 1)
k_scores_i8(const uint8_t *__restrict__ grid, int ncy, int ncx, int bins, int noy, int nox,
            int T, int bands, int tiles_x, const uint4 *__restrict__ wfrag, double scale,
            double bias, double *__restrict__ scores) {
    constexpr int P = 4 * KS;          // staged bytes per cell
    constexpr int ROWW = I8_CELLS * KS;  // staged words per row (P / 4 = KS words per cell)
    __shared__ uint32_t srow[I8_WARPS][ROWW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    int bid = blockIdx.x;
    const int tx = bid % tiles_x;
    bid /= tiles_x;
    const int band = bid % bands;
    const int f = bid / bands;
    const int ox0 = tx * I8_COLS + 16 * warp;
    if (ox0 >= nox) return;
    const int oy0 = band * T;
    const int oy1 = min(oy0 + T, noy);

    uint4 wa[S][KS];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) wa[s][ks] = __ldg(wfrag + (s * KS + ks) * 32 + lane);

    // staging: lane c < 23 owns cell ox0 + c of the row (KS words, zero past the grid)
    const uint8_t *gf = grid + (int64_t)f * ncy * ncx * bins;
    const int cell = ox0 + lane;
    const bool cown = lane < I8_CELLS && cell < ncx;
    const int mode = (bins & 3) == 0 ? 2 : ((bins & 1) == 0 ? 1 : 0);  // u32 / u16 / byte loads
    auto load_row = [&](int y, uint32_t (&wv)[KS]) {
#pragma unroll
        for (int j = 0; j < KS; ++j) wv[j] = 0u;
        if (!cown || y >= ncy) return;
        const uint8_t *p = gf + ((int64_t)y * ncx + cell) * bins;
        if (mode == 2) {
#pragma unroll
            for (int j = 0; j < KS; ++j)
                if (4 * j < bins) wv[j] = __ldg(reinterpret_cast<const uint32_t *>(p) + j);
        } else if (mode == 1) {
            const uint16_t *q = reinterpret_cast<const uint16_t *>(p);
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const uint32_t lo = 4 * j < bins ? (uint32_t)__ldg(q + 2 * j) : 0u;
                const uint32_t hi = 4 * j + 2 < bins ? (uint32_t)__ldg(q + 2 * j + 1) : 0u;
                wv[j] = lo | (hi << 16);
            }
        } else {
#pragma unroll
            for (int j = 0; j < KS; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (4 * j + k < bins) wv[j] |= (uint32_t)__ldg(p + 4 * j + k) << (8 * k);
        }
    };
    uint32_t *sr = srow[warp];
    auto store_row = [&](const uint32_t (&wv)[KS]) {
        if (lane < I8_CELLS) {
#pragma unroll
            for (int j = 0; j < KS; ++j) sr[lane * KS + j] = wv[j];
        }
    };

    // running window sums: R[j][0..1] cell row g, R[j][2..3] cell row g + 8, of
    // positions 8j + 2t, 8j + 2t + 1 (the window whose row `cy` is this row)
    long long R[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) R[j][r] = 0;

    const int y0 = oy0, y1 = oy1 - 1 + (I8_CY - 1);  // grid rows read (inclusive)
    const int src = (lane + 28) & 31;  // lane of cell row g - 1 (g = 0: lane of g = 7)
    // one grid row: smem holds row y, `cur` row y + 1 (loaded one step ago); row
    // y + 2 is fetched into `nxt`, so every load has a full row of MMAs to land
    auto step = [&](int y, uint32_t (&cur)[KS], uint32_t (&nxt)[KS]) {
        __syncwarp();
        if (y + 2 <= y1) load_row(y + 2, nxt);
        int acc[S][2][4];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[s][j][r] = 0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            uint32_t b[2][2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int w0 = (8 * j + g) * KS + 8 * ks + t;  // word of byte (8j+g)*P + 32 ks + 4t
                b[j][0] = sr[w0];
                b[j][1] = sr[w0 + 4];
            }
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int j = 0; j < 2; ++j) mma_s8(acc[s][j], wa[s][ks], b[j][0], b[j][1]);
        }
        // exact digit combination, then the systolic pass of the cell rows
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                long long v = 0;
#pragma unroll
                for (int s = S - 1; s >= 0; --s) v = v * 256 + (long long)acc[s][j][r];
                R[j][r] += v;
            }
        // cell row 15 (lanes g = 7, registers 2, 3) completes window row y - 15
        const int oy = y - (I8_CY - 1);
        if (g == 7 && oy >= oy0 && oy < oy1) {
            double *sp = scores + ((int64_t)f * noy + oy) * nox;
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int ox = ox0 + 8 * j + 2 * t + r;
                    if (ox < nox) sp[ox] = __dadd_rn(__dmul_rn(__ll2double_rn(R[j][2 + r]), scale), bias);
                }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const long long lo = __shfl_sync(FULL, R[j][r], src);
                const long long hi = __shfl_sync(FULL, R[j][2 + r], src);
                R[j][r] = g == 0 ? 0 : lo;
                R[j][2 + r] = g == 0 ? lo : hi;
            }
        __syncwarp();  // every lane has read row y
        store_row(cur);
    };
    uint32_t wb0[KS], wb1[KS];
    load_row(y0, wb0);
    load_row(y0 + 1, wb1);
    store_row(wb0);
    for (int y = y0; y <= y1; y += 2) {
        step(y, wb1, wb0);
        if (y + 1 <= y1) step(y + 1, wb0, wb1);
    }
}

// rows per band: the whole frame height unless that leaves the grid under
// ~2 CTA waves (1 CTA per SM), never under 32 rows (15 rows of overhead per band)
static int i8_band_rows(int n, int noy, int tiles_x) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int T = noy;
    while (T > 32 && (int64_t)n * tiles_x * ((noy + T - 1) / T) < 2LL * sms) T = (T + 1) / 2;
    return max(T, 1);
}

template <int KS, int S>
static void launch_i8_t(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                        const void *wfrag, double scale, double bias, double *scores, cudaStream_t st) {
    const int tiles_x = (nox + I8_COLS - 1) / I8_COLS;
    const int T = i8_band_rows(n, noy, tiles_x);
    const int bands = (noy + T - 1) / T;
    const int64_t blocks = (int64_t)n * bands * tiles_x;
    k_scores_i8<KS, S><<<(unsigned)blocks, 32 * I8_WARPS, 0, st>>>(
        grid, ncy, ncx, bins, noy, nox, T, bands, tiles_x, static_cast<const uint4 *>(wfrag), scale,
        bias, scores);
}

template <int KS>
static void launch_i8_ks(int digits, const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy,
                         int nox, const void *wfrag, double scale, double bias, double *scores,
                         cudaStream_t st) {
    if (digits <= 4) return launch_i8_t<KS, 4>(grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
    if (digits == 5) return launch_i8_t<KS, 5>(grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
    launch_i8_t<KS, 6>(grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
}

// k steps per window row for `bins` (P = 4 KS bytes per staged cell); the
// host's fragment layout (hog_scores_i8_prepare) uses the same value
int scores_i8_ks(int bins) { return bins <= 8 ? 2 : (bins + 3) / 4; }

void launch_scores_i8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                      const void *wfrag, int digits, double scale, double bias, double *scores,
                      cudaStream_t st) {
    switch (scores_i8_ks(bins)) {
        case 2: return launch_i8_ks<2>(digits, grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
        case 3: return launch_i8_ks<3>(digits, grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
        case 4: return launch_i8_ks<4>(digits, grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
        default: return launch_i8_ks<5>(digits, grid, n, ncy, ncx, bins, noy, nox, wfrag, scale, bias, scores, st);
    }
}

}  // namespace hogb200
