/*
 * hog_oracle.c -- CPU restatement of the reference LUT-HOG path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product library (libhogb200.so)
 * never links or calls it, and the product Python package never imports it.
 *
 * Each function restates one reference function (paths relative to
 * /root/reference/pkg/src/fasthog/).  The restatement is pinned against
 * golden vectors produced by the reference itself (tests/golden/).
 *
 * Build with -ffp-contract=off: the bilinear resize must reproduce numpy's
 * separate multiply/add roundings (detector.py:218-219) bit for bit.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NO_BIN (-1)
#define LUT_SIDE 511

static const double TWO_PI = 2.0 * 3.14159265358979311599796346854; /* 2*math.pi */

/* gradient.py:29-42 (bin_of) and gradient.py:56-72 (build_lut).
 * table[(dx+255)*511 + (dy+255)], dx-major like the reference. */
void oracle_build_lut(int bins, int16_t *table)
{
    for (int i = 0; i < LUT_SIDE; ++i) {
        for (int j = 0; j < LUT_SIDE; ++j) {
            double dx = (double)(i - 255), dy = (double)(j - 255);
            double phi = atan2(dy, dx);
            if (phi < 0.0) phi += TWO_PI;
            double f = floor(phi * (double)bins / TWO_PI);
            int b = (int)f;
            if (b > bins - 1) b = bins - 1;
            table[i * LUT_SIDE + j] = (int16_t)b;
        }
    }
    table[255 * LUT_SIDE + 255] = NO_BIN;
}

/* gradient.py:95-121.  planes: (C,H,W) u8 planar; cells: (H,W) int16.
 * Channel rule: the channel with the largest dx^2+dy^2 wins, first on ties
 * (np.argmax, gradient.py:114-117). Border pixels are NO_BIN (gradient.py:119). */
int oracle_gradient_map(const uint8_t *img, int C, int H, int W, const int16_t *lut,
                        int16_t *cells)
{
    if (W < 3 || H < 3) return -1;
    for (int i = 0; i < H * W; ++i) cells[i] = NO_BIN;
    for (int y = 1; y < H - 1; ++y) {
        for (int x = 1; x < W - 1; ++x) {
            int best_mag = -1, bdx = 0, bdy = 0;
            for (int c = 0; c < C; ++c) {
                const uint8_t *p = img + (size_t)c * H * W;
                int dx = (int)p[y * W + x + 1] - (int)p[y * W + x - 1];
                int dy = (int)p[(y + 1) * W + x] - (int)p[(y - 1) * W + x];
                int mag = dx * dx + dy * dy;
                if (mag > best_mag) { best_mag = mag; bdx = dx; bdy = dy; }
            }
            cells[y * W + x] = lut[(bdx + 255) * LUT_SIDE + (bdy + 255)];
        }
    }
    return 0;
}

/* integral.py:58-87 with acc_width=32.  planes: (bins, H+1, W+1) uint32,
 * planes[n][y+1][x+1] = sum over y'<=y, x'<=x of [cells==n]; row 0 and
 * column 0 are zero.  Restated as one running row sum per bin. */
void oracle_integral(const int16_t *cells, int H, int W, int bins, uint32_t *planes)
{
    size_t pw = (size_t)W + 1, ps = (size_t)(H + 1) * pw;
    memset(planes, 0, sizeof(uint32_t) * ps * (size_t)bins);
    uint32_t *row = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)bins);
    for (int y = 0; y < H; ++y) {
        memset(row, 0, sizeof(uint32_t) * (size_t)bins);
        for (int x = 0; x < W; ++x) {
            int b = cells[y * W + x];
            if (b >= 0 && b < bins) row[b] += 1;
            for (int n = 0; n < bins; ++n) {
                uint32_t *p = planes + (size_t)n * ps;
                p[(size_t)(y + 1) * pw + x + 1] = p[(size_t)y * pw + x + 1] + row[n];
            }
        }
    }
    free(row);
}

/* descriptor.py:176-185 (CellHistogramCache.grid): 4-corner count of the
 * cell at (cell_ys[j], cell_xs[i]); grid is (ncy, ncx, bins) int64. */
void oracle_cell_grid(const uint32_t *planes, int bins, int H, int W,
                      const int64_t *cell_xs, int ncx, const int64_t *cell_ys, int ncy,
                      int cell, int64_t *grid)
{
    size_t pw = (size_t)W + 1, ps = (size_t)(H + 1) * pw;
    for (int j = 0; j < ncy; ++j) {
        for (int i = 0; i < ncx; ++i) {
            size_t y0 = (size_t)cell_ys[j], x0 = (size_t)cell_xs[i];
            size_t y1 = y0 + (size_t)cell, x1 = x0 + (size_t)cell;
            for (int n = 0; n < bins; ++n) {
                const uint32_t *p = planes + (size_t)n * ps;
                int64_t v = (int64_t)p[y1 * pw + x1] + (int64_t)p[y0 * pw + x0]
                          - (int64_t)p[y0 * pw + x1] - (int64_t)p[y1 * pw + x0];
                grid[((size_t)j * ncx + i) * bins + n] = v;
            }
        }
    }
}

/* descriptor.py:107-124 (_assemble_blocks) applied to the window whose cells
 * are grid[rows[cy]][cols[cx]] (descriptor.py:190-192).  norm: 0 none, 1 l1,
 * 2 l2.  eps_term is _EPS for l1 and _EPS*_EPS for l2 (descriptor.py:23,121-123).
 * Output order: blocks row-major, cells row-major inside a block, bins
 * ascending (descriptor.py:115-118).  Returns the descriptor length. */
int oracle_window_descriptor(const int64_t *grid, int ncx, int bins,
                             const int64_t *rows, const int64_t *cols,
                             int cells_x, int cells_y, int block, int block_stride,
                             int norm, double eps_term, double *out)
{
    int bx_n = (cells_x - block) / block_stride + 1;
    int by_n = (cells_y - block) / block_stride + 1;
    int blen = block * block * bins, k = 0;
    for (int by = 0; by < by_n; ++by) {
        for (int bx = 0; bx < bx_n; ++bx) {
            int k0 = k;
            for (int cy = 0; cy < block; ++cy) {
                for (int cx = 0; cx < block; ++cx) {
                    int64_t r = rows[by * block_stride + cy];
                    int64_t c = cols[bx * block_stride + cx];
                    const int64_t *h = grid + ((size_t)r * ncx + (size_t)c) * bins;
                    for (int n = 0; n < bins; ++n) out[k++] = (double)h[n];
                }
            }
            if (norm != 0) {
                double s = 0.0;
                for (int q = k0; q < k0 + blen; ++q)
                    s += (norm == 1) ? fabs(out[q]) : out[q] * out[q];
                double denom = (norm == 1) ? s + eps_term : sqrt(s + eps_term);
                for (int q = k0; q < k0 + blen; ++q) out[q] = out[q] / denom;
            }
        }
    }
    return k;
}

/* detector.py:131-137 / 148-150: dot(weights, desc) + bias, summed in index
 * order (the reference's OpenBLAS ddot order is library-defined; scores are
 * compared within a stated tolerance). */
double oracle_dot_bias(const double *w, const double *d, int n, double bias)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += w[i] * d[i];
    return s + bias;
}

/* detector.py:202-221 (_resize_bilinear).  (C,H,W) u8 -> (C,nh,nw) u8, fp64
 * in the reference's exact operation order, no contraction, rint half-even. */
void oracle_resize_bilinear(const uint8_t *src, int C, int H, int W, int nw, int nh,
                            uint8_t *dst)
{
    double ry = (double)H / (double)nh, rx = (double)W / (double)nw;
    double *rows = (double *)malloc(sizeof(double) * (size_t)W);
    for (int c = 0; c < C; ++c) {
        const uint8_t *p = src + (size_t)c * H * W;
        for (int i = 0; i < nh; ++i) {
            double sy = ((double)i + 0.5) * ry - 0.5;
            if (sy < 0.0) sy = 0.0;
            if (sy > (double)(H - 1)) sy = (double)(H - 1);
            int y0 = (int)floor(sy);
            int y1 = y0 + 1 < H - 1 ? y0 + 1 : H - 1;
            double fy = sy - (double)y0;
            double gy = 1.0 - fy;
            for (int x = 0; x < W; ++x) {
                double a = (double)p[(size_t)y0 * W + x] * gy;
                double b = (double)p[(size_t)y1 * W + x] * fy;
                rows[x] = a + b;
            }
            for (int j = 0; j < nw; ++j) {
                double sx = ((double)j + 0.5) * rx - 0.5;
                if (sx < 0.0) sx = 0.0;
                if (sx > (double)(W - 1)) sx = (double)(W - 1);
                int x0 = (int)floor(sx);
                int x1 = x0 + 1 < W - 1 ? x0 + 1 : W - 1;
                double fx = sx - (double)x0;
                double a = rows[x0] * (1.0 - fx);
                double b = rows[x1] * fx;
                double m = rint(a + b);
                if (m < 0.0) m = 0.0;
                if (m > 255.0) m = 255.0;
                dst[((size_t)c * nh + i) * nw + j] = (uint8_t)m;
            }
        }
    }
    free(rows);
}

/* ------------------------------------------------------------------------ */
/* Whole-frame pipeline for the CPU baseline: gradient_map -> integral stack
 * -> cell grid -> (scores | per-cell L2 denominators).  Geometry is the one
 * the BASELINE configs use: block=1, block_stride=1, cell lattice = every
 * origin's cells (descriptor.py:198-206, 162-188).  mode: 0 grid only,
 * 1 grid + scores (norm none), 2 grid + l2 denominators. */

typedef struct {
    const uint8_t *frames;
    int n, C, H, W, bins, cell, ww, wh, stride, mode;
    const int16_t *lut;
    const double *weights;
    double bias, eps_term;
    int64_t *grid_out;       /* optional: (n, ncy, ncx, bins) */
    double *score_out;       /* optional: (n, noy, nox) */
    int next;                /* work counter */
    pthread_mutex_t mu;
    uint64_t checksum;       /* consumes outputs so nothing is optimised away */
} batch_job;

static int count_origins(int size, int win, int stride)
{
    return size >= win ? (size - win) / stride + 1 : 0;
}

/* unique(o[:,None] + cell*arange(cells)) for the regular origin grid */
static int cell_lattice(int nor, int stride, int cells, int cell, int64_t *out)
{
    int cap = nor * cells, m = 0;
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    for (int o = 0; o < nor; ++o)
        for (int k = 0; k < cells; ++k) tmp[m++] = (int64_t)o * stride + (int64_t)k * cell;
    /* insertion-free unique via counting over the bounded range */
    int64_t mx = 0;
    for (int q = 0; q < m; ++q) if (tmp[q] > mx) mx = tmp[q];
    char *seen = (char *)calloc((size_t)mx + 1, 1);
    for (int q = 0; q < m; ++q) seen[tmp[q]] = 1;
    int u = 0;
    for (int64_t v = 0; v <= mx; ++v) if (seen[v]) out[u++] = v;
    free(seen);
    free(tmp);
    return u;
}

static int64_t search_sorted(const int64_t *a, int n, int64_t v)
{
    int lo = 0, hi = n;
    while (lo < hi) { int mid = (lo + hi) / 2; if (a[mid] < v) lo = mid + 1; else hi = mid; }
    return lo;
}

static void run_one_frame(batch_job *J, int f)
{
    int C = J->C, H = J->H, W = J->W, bins = J->bins;
    const uint8_t *img = J->frames + (size_t)f * C * H * W;
    int16_t *cells = (int16_t *)malloc(sizeof(int16_t) * (size_t)H * W);
    uint32_t *planes = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)bins * (H + 1) * (W + 1));
    oracle_gradient_map(img, C, H, W, J->lut, cells);
    oracle_integral(cells, H, W, bins, planes);

    int cx_n = J->ww / J->cell, cy_n = J->wh / J->cell;
    int nox = count_origins(W, J->ww, J->stride), noy = count_origins(H, J->wh, J->stride);
    int64_t *cxs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nox * cx_n + 1));
    int64_t *cys = (int64_t *)malloc(sizeof(int64_t) * (size_t)(noy * cy_n + 1));
    int ncx = cell_lattice(nox, J->stride, cx_n, J->cell, cxs);
    int ncy = cell_lattice(noy, J->stride, cy_n, J->cell, cys);
    int64_t *grid = J->grid_out ? J->grid_out + (size_t)f * ncy * ncx * bins
                                : (int64_t *)malloc(sizeof(int64_t) * (size_t)ncy * ncx * bins);
    oracle_cell_grid(planes, bins, H, W, cxs, ncx, cys, ncy, J->cell, grid);
    uint64_t cs = 0;
    for (size_t q = 0; q < (size_t)ncy * ncx * bins; ++q) cs += (uint64_t)grid[q] * (q % 7 + 1);

    if (J->mode == 1 || J->mode == 2) {
        int D = cx_n * cy_n * bins;
        int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)cy_n);
        int64_t *cols = (int64_t *)malloc(sizeof(int64_t) * (size_t)cx_n);
        double *desc = (double *)malloc(sizeof(double) * (size_t)D);
        for (int iy = 0; iy < noy; ++iy) {
            for (int k = 0; k < cy_n; ++k)
                rows[k] = search_sorted(cys, ncy, (int64_t)iy * J->stride + (int64_t)k * J->cell);
            for (int ix = 0; ix < nox; ++ix) {
                for (int k = 0; k < cx_n; ++k)
                    cols[k] = search_sorted(cxs, ncx, (int64_t)ix * J->stride + (int64_t)k * J->cell);
                oracle_window_descriptor(grid, ncx, bins, rows, cols, cx_n, cy_n, 1, 1,
                                         J->mode == 2 ? 2 : 0, J->eps_term, desc);
                if (J->mode == 1) {
                    double s = oracle_dot_bias(J->weights, desc, D, J->bias);
                    if (J->score_out) J->score_out[((size_t)f * noy + iy) * nox + ix] = s;
                    cs += (uint64_t)(int64_t)(s * 1e6);
                } else {
                    cs += (uint64_t)(int64_t)(desc[0] * 1e6);
                }
            }
        }
        free(rows); free(cols); free(desc);
    }
    if (!J->grid_out) free(grid);
    free(cxs); free(cys); free(cells); free(planes);
    pthread_mutex_lock(&J->mu);
    J->checksum += cs;
    pthread_mutex_unlock(&J->mu);
}

static void *batch_worker(void *arg)
{
    batch_job *J = (batch_job *)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int f = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (f >= J->n) break;
        run_one_frame(J, f);
    }
    return NULL;
}

/* Runs the per-frame pipeline over n frames on `threads` host threads.
 * Returns a checksum of the outputs. */
uint64_t oracle_run_batch(const uint8_t *frames, int n, int C, int H, int W,
                          const int16_t *lut, int bins, int cell, int ww, int wh,
                          int stride, int mode, const double *weights, double bias,
                          double eps_term, int threads, int64_t *grid_out,
                          double *score_out)
{
    batch_job J;
    memset(&J, 0, sizeof(J));
    J.frames = frames; J.n = n; J.C = C; J.H = H; J.W = W; J.bins = bins;
    J.cell = cell; J.ww = ww; J.wh = wh; J.stride = stride; J.mode = mode;
    J.lut = lut; J.weights = weights; J.bias = bias; J.eps_term = eps_term;
    J.grid_out = grid_out; J.score_out = score_out;
    pthread_mutex_init(&J.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, batch_worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    pthread_mutex_destroy(&J.mu);
    return J.checksum;
}
