// k_window.cu -- the window stage and the pyramid: generic integral (bins >
// 18), 4-corner cell grid, per-cell normalisation, window scores (lattice
// correlation and generic per-window assembly), bilinear resize.
// descriptor.py:107-195, detector.py:140-154, 202-221, integral.py:58-87.
#include "hog_common.cuh"

namespace hogb200 {

// ---------------------------------------------------------------------------
// Generic integral for bins > 18 (API completeness; the configs use 8/9/18):
// row prefix per plane row, then column prefix in place.
// Bin-group pass for N_b > 18 (hog_integral): the single-write plane kernel
// handles <= 18 bins, so N_b bins run as groups of <= 16 consecutive bins, each
// over a copy of the bin map with the group's first bin subtracted (per byte,
// mod 256).  Bins of the group become 0 .. nb-1; every other byte (earlier
// bins wrap to >= 192, NO_BIN 0xFF to >= 192, later bins to nb .. 63) lands
// on a one-hot shift past the group's counters or in a padding slot that is
// never widened or stored, so each group's planes are exactly the
// reference's planes of those bins (integral.py:75-79).
__global__ void k_bin_offset(const int8_t *__restrict__ bm, int64_t bp, int64_t bfs, int n, int h,
                             int w4, uint32_t sub4, int8_t *__restrict__ out, int64_t op, int64_t ofs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * h * w4) return;
    const int c = (int)(i % w4);
    const int64_t r = i / w4;
    const int y = (int)(r % h), f = (int)(r / h);
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t *>(bm + f * bfs + y * bp) + c);
    reinterpret_cast<uint32_t *>(out + f * ofs + y * op)[c] = __vsub4(v, sub4);
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
// Per-WINDOW L2 norm (an extension for BASELINE configs[2]'s wording; the
// reference normalises per block, descriptor.py:107-124): the norm of the
// window's unnormalised descriptor d (its cells' histograms, descriptor.py:
// 115-118) is sqrt(sum d^2 + eps^2), eps^2 = _EPS*_EPS as descriptor.py:123.
// Counts are integers, so sum d^2 is exact in int64 and in fp64, and IEEE
// sqrt makes the norm bit-exact with numpy's np.sqrt((d*d).sum() + _EPS*_EPS).
// Pass 1: per-cell sum of squares; pass 2: one thread per window sums its cells.
template <typename T>
__global__ void k_cell_sq(const T *__restrict__ grid, int64_t ncells_total, int bins,
                          int32_t *__restrict__ sq) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncells_total) return;
    const T *gp = grid + i * bins;
    int32_t s = 0;
    for (int b = 0; b < bins; ++b) {
        const int32_t v = (int32_t)gp[b];
        s += v * v;
    }
    sq[i] = s;
}

__global__ void k_window_l2(const int32_t *__restrict__ sq, int n, int ncy, int ncx,
                            const int32_t *__restrict__ row_idx, int noy,
                            const int32_t *__restrict__ col_idx, int nox, int cells_x, int cells_y,
                            double eps_term, double *__restrict__ norms) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * noy * nox) return;
    const int ix = (int)(i % nox);
    const int64_t r = i / nox;
    const int iy = (int)(r % noy), f = (int)(r / noy);
    const int32_t *sf = sq + (int64_t)f * ncy * ncx;
    int64_t s = 0;
    for (int cy = 0; cy < cells_y; ++cy) {
        const int32_t *row = sf + (int64_t)__ldg(row_idx + (int64_t)iy * cells_y + cy) * ncx;
        for (int cx = 0; cx < cells_x; ++cx) s += __ldg(row + __ldg(col_idx + (int64_t)ix * cells_x + cx));
    }
    norms[i] = __dsqrt_rn(__dadd_rn((double)s, eps_term));
}

// Regular lattice (window (iy, ix) reads cells (iy + cy*K, ix + cx*K)): the
// window sum is separable, so pass 2 sums cells_x cells along each lattice row
// into hs, and pass 3 sums cells_y of those down each window column.
__global__ void k_window_l2_h(const int32_t *__restrict__ sq, int64_t rows_total, int ncx, int nox,
                              int cells_x, int K, int32_t *__restrict__ hs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows_total * nox) return;
    const int ix = (int)(i % nox);
    const int64_t r = i / nox;  // (frame, lattice row)
    const int32_t *row = sq + r * ncx + ix;
    int32_t s = 0;
    for (int cx = 0; cx < cells_x; ++cx) s += __ldg(row + cx * K);
    hs[i] = s;
}

__global__ void k_window_l2_v(const int32_t *__restrict__ hs, int n, int ncy, int noy, int nox,
                              int cells_y, int K, double eps_term, double *__restrict__ norms) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)n * noy * nox) return;
    const int ix = (int)(i % nox);
    const int64_t r = i / nox;
    const int iy = (int)(r % noy), f = (int)(r / noy);
    const int32_t *col = hs + ((int64_t)f * ncy + iy) * nox + ix;
    int64_t s = 0;
    for (int cy = 0; cy < cells_y; ++cy) s += __ldg(col + (int64_t)cy * K * nox);
    norms[i] = __dsqrt_rn(__dadd_rn((double)s, eps_term));
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
// multiply/add roundings (no FMA contraction).  A thread owns RZ_C adjacent
// output columns (their source columns and weights are computed once) and
// walks RZ_R output rows; one 4-byte store per row when the row is aligned.
// Grid: x = column groups, y = row groups, z = frame * channels.
constexpr int RZ_C = 4, RZ_R = 16;

__global__ void __launch_bounds__(128)
k_resize(const uint8_t *__restrict__ src, int c, int h, int w, int64_t sp, int64_t scs, int64_t sfs,
         int nh, int nw, double ry, double rx, uint8_t *__restrict__ dst, int64_t dp, int64_t dcs,
         int64_t dfs) {
    const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * RZ_C;
    if (j0 >= nw) return;
    const int ch = blockIdx.z % c, f = blockIdx.z / c;
    int x0[RZ_C], x1[RZ_C];
    double fx[RZ_C], gx[RZ_C];
#pragma unroll
    for (int q = 0; q < RZ_C; ++q) {
        const int j = min(j0 + q, nw - 1);
        double sx = __dsub_rn(__dmul_rn((double)j + 0.5, rx), 0.5);
        sx = fmin(fmax(sx, 0.0), (double)(w - 1));
        x0[q] = (int)floor(sx);
        x1[q] = min(x0[q] + 1, w - 1);
        fx[q] = __dsub_rn(sx, (double)x0[q]);
        gx[q] = __dsub_rn(1.0, fx[q]);
    }
    const uint8_t *p = src + (int64_t)f * sfs + (int64_t)ch * scs;
    uint8_t *d = dst + (int64_t)f * dfs + (int64_t)ch * dcs + j0;
    const bool full = j0 + RZ_C <= nw && (((uintptr_t)d | (uintptr_t)dp) & 3) == 0;
    const int r1 = min(nh, (int)(blockIdx.y + 1) * RZ_R);
    for (int r = blockIdx.y * RZ_R; r < r1; ++r) {
        double sy = __dsub_rn(__dmul_rn((double)r + 0.5, ry), 0.5);
        sy = fmin(fmax(sy, 0.0), (double)(h - 1));
        const int y0 = (int)floor(sy), y1 = min(y0 + 1, h - 1);
        const double fy = __dsub_rn(sy, (double)y0), gy = __dsub_rn(1.0, fy);
        const uint8_t *p0 = p + (int64_t)y0 * sp, *p1 = p + (int64_t)y1 * sp;
        uint32_t word = 0;
#pragma unroll
        for (int q = 0; q < RZ_C; ++q) {
            const double a0 = (double)__ldg(p0 + x0[q]), b0 = (double)__ldg(p1 + x0[q]);
            const double a1 = (double)__ldg(p0 + x1[q]), b1 = (double)__ldg(p1 + x1[q]);
            const double r0 = __dadd_rn(__dmul_rn(a0, gy), __dmul_rn(b0, fy));
            const double rr1 = __dadd_rn(__dmul_rn(a1, gy), __dmul_rn(b1, fy));
            // np.rint + clip (detector.py:219): the convex mix of bytes stays within
            // [0, 255 + 1e-13], so rint alone lands in 0..255, and adding 1.5 * 2^52
            // rounds to the nearest even integer like rint, leaving it in the low word
            const double m = __dadd_rn(__dadd_rn(__dmul_rn(r0, gx[q]), __dmul_rn(rr1, fx[q])),
                                       6755399441055744.0);
            word |= ((uint32_t)__double2loint(m) & 0xffu) << (8 * q);
        }
        uint8_t *dr = d + (int64_t)r * dp;
        if (full) {
            *reinterpret_cast<uint32_t *>(dr) = word;
        } else {
#pragma unroll
            for (int q = 0; q < RZ_C; ++q)
                if (j0 + q < nw) dr[q] = (uint8_t)(word >> (8 * q));
        }
    }
}

#if HOGB200_VARIANTS
// Row-shared resize for downscales up to 2x (pyramid levels 1-3 of c5 hold
// three quarters of the level pixels): per output row the CTA first forms the
// vertical mix `rows` (detector.py:216) of every source column its 256 output
// columns read -- once per column, in shared memory, from coalesced byte
// loads -- and then each thread mixes its column's two entries (:217).  Same
// float64 operations in the same order as k_resize; bytes become doubles by a
// shared 256-entry table, rint + clip by one add of 1.5 * 2^52 (round half to
// even; the convex mix of bytes never leaves [0, 255]).
constexpr int RZ2_T = 256, RZ2_R = 16, RZ2_NS = 2 * RZ2_T + 2;  // source columns per row (rx <= 2)

__global__ void __launch_bounds__(RZ2_T)
k_resize_rows(const uint8_t *__restrict__ src, int c, int h, int w, int64_t sp, int64_t scs, int64_t sfs,
              int nh, int nw, double ry, double rx, uint8_t *__restrict__ dst, int64_t dp, int64_t dcs,
              int64_t dfs) {
    __shared__ double tab[256];
    __shared__ double vrow[2][RZ2_NS];
    __shared__ double rfy[RZ2_R], rgy[RZ2_R];
    __shared__ int ry0[RZ2_R], ry1[RZ2_R];
    const int tid = threadIdx.x;
    tab[tid] = (double)tid;
    const int jt0 = blockIdx.x * RZ2_T;
    const int j = min(jt0 + tid, nw - 1);
    auto col = [&](int jj, int &x0, int &x1, double &fx) {
        double sx = __dsub_rn(__dmul_rn((double)jj + 0.5, rx), 0.5);
        sx = fmin(fmax(sx, 0.0), (double)(w - 1));
        x0 = (int)floor(sx);
        x1 = min(x0 + 1, w - 1);
        fx = __dsub_rn(sx, (double)x0);
    };
    int x0, x1, xa, xb, xe, xf;
    double fx, fa, fe;
    col(j, x0, x1, fx);
    const double gx = __dsub_rn(1.0, fx);
    col(jt0, xa, xb, fa);                      // first source column of the tile
    col(min(jt0 + RZ2_T - 1, nw - 1), xe, xf, fe);  // last: x1 of the last column
    const int xs0 = xa, ns = xf - xa + 1;
    const int r0 = blockIdx.y * RZ2_R, nr = min(RZ2_R, nh - r0);
    if (tid < nr) {
        double sy = __dsub_rn(__dmul_rn((double)(r0 + tid) + 0.5, ry), 0.5);
        sy = fmin(fmax(sy, 0.0), (double)(h - 1));
        const int y0 = (int)floor(sy);
        ry0[tid] = y0;
        ry1[tid] = min(y0 + 1, h - 1);
        rfy[tid] = __dsub_rn(sy, (double)y0);
        rgy[tid] = __dsub_rn(1.0, rfy[tid]);
    }
    __syncthreads();
    const int ch = blockIdx.z % c, f = blockIdx.z / c;
    const uint8_t *p = src + (int64_t)f * sfs + (int64_t)ch * scs + xs0;
    uint8_t *d = dst + (int64_t)f * dfs + (int64_t)ch * dcs + jt0 + tid;
    const bool own = jt0 + tid < nw;
    const int l0 = x0 - xs0, l1 = x1 - xs0;
    for (int i = 0; i < nr; ++i) {
        double *v = vrow[i & 1];
        const uint8_t *p0 = p + (int64_t)ry0[i] * sp, *p1 = p + (int64_t)ry1[i] * sp;
        const double fy = rfy[i], gy = rgy[i];
        for (int k = tid; k < ns; k += RZ2_T)
            v[k] = __dadd_rn(__dmul_rn(tab[__ldg(p0 + k)], gy), __dmul_rn(tab[__ldg(p1 + k)], fy));
        __syncthreads();  // (two buffers: row i + 1 may overwrite the other one)
        if (own) {
            const double m = __dadd_rn(__dmul_rn(v[l0], gx), __dmul_rn(v[l1], fx));
            d[(int64_t)(r0 + i) * dp] = (uint8_t)__double2loint(__dadd_rn(m, 6755399441055744.0));
        }
    }
}

#endif  // HOGB200_VARIANTS

// ---- launchers ------------------------------------------------------------

void launch_bin_offset(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int b0,
                       int8_t *out, int64_t op, int64_t ofs, cudaStream_t st) {
    const int w4 = (w + 3) / 4;
    k_bin_offset<<<blocks_for((int64_t)n * h * w4, 256), 256, 0, st>>>(
        bm, bp, bfs, n, h, w4, (uint32_t)b0 * 0x01010101u, out, op, ofs);
}

void launch_cell_grid(const int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int n, int bins,
                      const int32_t *cxs, int ncx, const int32_t *cys, int ncy, int cell,
                      int32_t *grid, cudaStream_t st) {
    k_cell_grid<<<blocks_for((int64_t)n * ncx * ncy, 128), 128, 0, st>>>(pl, pp, pns, pfs, n, bins,
                                                                         cxs, ncx, cys, ncy, cell,
                                                                         grid);
}

void launch_window_l2(const void *grid, int elem_bytes, int n, int ncy, int ncx, int bins,
                      const int32_t *row_idx, int noy, const int32_t *col_idx, int nox, int cells_x,
                      int cells_y, int k, double eps_term, int32_t *sq, double *norms, cudaStream_t st) {
    const int64_t cells = (int64_t)n * ncy * ncx;
    if (elem_bytes == 1)
        k_cell_sq<uint8_t><<<blocks_for(cells, 256), 256, 0, st>>>((const uint8_t *)grid, cells, bins, sq);
    else
        k_cell_sq<int32_t><<<blocks_for(cells, 256), 256, 0, st>>>((const int32_t *)grid, cells, bins, sq);
    const int64_t tot = (int64_t)n * noy * nox;
    if (k > 0) {  // regular lattice: separable sums (hs reuses the tail of sq's buffer? no: own area)
        int32_t *hs = sq + cells;
        k_window_l2_h<<<blocks_for((int64_t)n * ncy * nox, 256), 256, 0, st>>>(sq, (int64_t)n * ncy, ncx,
                                                                              nox, cells_x, k, hs);
        k_window_l2_v<<<blocks_for(tot, 256), 256, 0, st>>>(hs, n, ncy, noy, nox, cells_y, k, eps_term,
                                                             norms);
        return;
    }
    k_window_l2<<<blocks_for(tot, 128), 128, 0, st>>>(sq, n, ncy, ncx, row_idx, noy, col_idx, nox,
                                                      cells_x, cells_y, eps_term, norms);
}

void launch_cell_norm(const int32_t *grid, int64_t tot, int bins, int norm, double eps_term,
                      double *den, cudaStream_t st) {
    k_cell_norm<<<blocks_for(tot, 256), 256, 0, st>>>(grid, tot, bins, norm, eps_term, den);
}

void launch_window_features(const int32_t *grid, int n, int ncy, int ncx, int bins,
                            const int32_t *row_idx, int noy, const int32_t *col_idx, int nox,
                            int cells_x, int cells_y, int block, int bstride, int norm,
                            double eps_term, const double *wts, double bias, double *scores,
                            double *desc, cudaStream_t st) {
    const int64_t tot = (int64_t)n * noy * nox;
    k_window_features<<<blocks_for(tot, 128), 128, 0, st>>>(grid, ncy, ncx, bins, row_idx, noy,
                                                            col_idx, nox, cells_x, cells_y, block,
                                                            bstride, norm, eps_term, wts, bias,
                                                            scores, desc, n);
}

void launch_scores_lattice(const int32_t *grid, const double *den, int n, int ncy, int ncx,
                           int bins, int noy, int nox, int cells_y, int k, const double *wts,
                           double bias, double *scores, cudaStream_t st) {
    if (den == nullptr && !(HOGB200_VARIANTS && getenv("HOGB200_SCORES_V1")))  // k_scores.cu (integer grid)
        return launch_scores_rows(grid, n, ncy, ncx, bins, noy, nox, cells_y, k, wts, bias, scores, st);
    const int span = SC_COLS + 7 * k;
    const size_t smem =
        sizeof(double) * ((size_t)cells_y * bins * 8 + 2 * (size_t)bins * (span + span / 8 + 1));
    static size_t configured[HOG_MAX_DEVICES] = {};
    if (smem_optin_needed(configured, smem))
        cudaFuncSetAttribute(k_scores_lattice<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    const int64_t blocks = (int64_t)n * ((noy + SC_TY * SC_YG - 1) / (SC_TY * SC_YG)) *
                           ((nox + SC_COLS - 1) / SC_COLS);
    k_scores_lattice<8><<<(unsigned)blocks, 32 * SC_YG, smem, st>>>(grid, den, ncy, ncx, bins, noy,
                                                                     nox, cells_y, k, wts, bias,
                                                                     scores);
}

void launch_resize(const uint8_t *src, int n, int c, int h, int w, int64_t sp, int64_t scs,
                   int64_t sfs, int nh, int nw, double ry, double rx, uint8_t *dst, int64_t dp,
                   int64_t dcs, int64_t dfs, cudaStream_t st) {
    // experiment builds only: the row-shared kernel measured slower on c5 (levels 1-3:
    // 9.2 ms in 6 launches against ~4 ms for k_resize; profiles/r2/resize_rows_shared_ab.md)
    static const int rows_path = [] {
        const char *e = HOGB200_VARIANTS ? getenv("HOGB200_RESIZE_ROWS") : nullptr;
        return e ? atoi(e) : 0;
    }();
#if HOGB200_VARIANTS
    if (rows_path && rx <= 2.0) {
        const dim3 grid((unsigned)((nw + RZ2_T - 1) / RZ2_T), (unsigned)((nh + RZ2_R - 1) / RZ2_R),
                        (unsigned)(n * c));
        k_resize_rows<<<grid, RZ2_T, 0, st>>>(src, c, h, w, sp, scs, sfs, nh, nw, ry, rx, dst, dp, dcs, dfs);
        return;
    }
#else
    (void)rows_path;
#endif
    const dim3 grid((unsigned)blocks_for(nw, 128 * RZ_C), (unsigned)((nh + RZ_R - 1) / RZ_R),
                    (unsigned)(n * c));
    k_resize<<<grid, 128, 0, st>>>(src, c, h, w, sp, scs, sfs, nh, nw, ry, rx, dst, dp, dcs, dfs);
}

}  // namespace hogb200
