/*
 * hogb200.h -- C ABI of libhogb200.so, the sm_100a LUT-HOG hot path.
 *
 * The reference (fasthog, pure Python + NumPy) has no FFI; its drop-in
 * surface is the flat Python API in pkg/src/fasthog/__init__.py:4-65.
 * Each entry point below replaces the NumPy body of one reference function
 * (paths relative to /root/reference/pkg/src/fasthog/), and the Python
 * package paper_1703_06256_b200 binds them with ctypes under the reference's
 * own function names.
 *
 * Conventions
 *   - Every buffer pointer is a DEVICE pointer owned by the caller (torch
 *     tensors in the Python layer).  The library allocates nothing.
 *   - Strides are in elements of the pointed-to type (bytes for uint8/int8).
 *   - All calls are asynchronous on `stream` (NULL = legacy default stream),
 *     reentrant, and never synchronise the host.
 *   - Return 0 on success, HOG_EINVAL for a rejected argument, HOG_ECUDA for
 *     a launch error; hog_last_error() describes the last failure (per thread).
 *
 * Data layouts
 *   image   uint8  [n][c][h][w]   elem (f,ch,y,x) = img[f*img_fstride + ch*img_cstride + y*img_pitch + x]
 *                                 img_pitch % 4 == 0, img_pitch >= round_up(w, 4), 4-byte aligned base
 *   binmap  int8   [n][h][w]      elem (f,y,x) = bm[f*bm_fstride + y*bm_pitch + x], -1 = NO_BIN
 *                                 bm_pitch % 4 == 0, bm_pitch >= round_up(w, 4)
 *   planes  int32  [n][bins][h+1][w+1]
 *                                 elem (f,b,Y,X) = pl[f*pl_fstride + b*pl_nstride + Y*pl_pitch + X]
 *                                 pl_pitch >= w+1.  Fast path (256-bit vector stores) when
 *                                 (pl + 1) is 32-B aligned, pl_pitch, pl_nstride, pl_fstride
 *                                 are multiples of 8 and pl_pitch >= round_up(w, 8) + 8
 *                                 (the padding is then written too, so every sector is whole);
 *                                 otherwise scalar stores.  hog_plane_pitch(w) returns that pitch.
 *   grid    int32  [n][ncy][ncx][bins]  cell histograms (CellHistogramCache.grid, descriptor.py:176-185)
 */
#ifndef HOGB200_H
#define HOGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *hog_stream_t; /* == cudaStream_t */

#define HOG_OK 0
#define HOG_EINVAL 1
#define HOG_ECUDA 2
#define HOG_ERANGE 3 /* weights the integer score path cannot hold exactly */

/* hog_pipeline stages (bitmask; 0 = all) */
#define HOG_STAGE_BIN 1    /* gradient + LUT binning + per-band column counts */
#define HOG_STAGE_SCAN 2   /* column counts above every band                  */
#define HOG_STAGE_PLANES 4 /* integral planes (+ fused cell grid)             */
#define HOG_STAGE_ALL 7
#define HOG_STAGE_GRID_U8 8 /* flag: the fused grid is uint8 (cell counts <= cell^2 <= 255) */

/* Library version string, e.g. "hogb200 1.0 sm_100a". */
const char *hog_version(void);

/* Text of the last error raised on the calling thread ("" if none). */
const char *hog_last_error(void);

/* Number of kernels the calling thread's last hog_pipeline / hog_pipeline_slab call
 * launched (binning, carry scan, planes: the carry scan is folded into the plane
 * kernel for shapes with few bands, integral.py:75-79), so callers can report
 * launch counts they did not have to guess. */
int hog_last_pipeline_launches(void);

/* Octant binning (N_b in {4, 8}).  gradient.py:55-72: the reference's
 * table for these bin counts is folded by its quarter/half-turn symmetry into
 * sign tests of four linear forms evaluated in registers (no table gather).
 * hog_lut_proof runs that device classifier on all 261,121 (dx, dy) pairs and
 * stores in *mismatches the entries where it differs from `lut` (0: proven
 * identical; -1: bins not 4 or 8).  It synchronises `stream`.  hog_grad_bin /
 * hog_pipeline use the octant kernel only for a (device, lut, bins) that has
 * passed this proof (run automatically on first use outside a graph capture;
 * otherwise the table-gather kernel runs).  Tables are treated as immutable,
 * like the reference's read-only OrientationLut: hog_lut_forget drops the
 * cached result for a table whose bytes the caller rewrites. */
int hog_lut_proof(const uint8_t *lut, int bins, long long *mismatches, hog_stream_t stream);
void hog_lut_forget(const uint8_t *lut);

/* Fast-path plane row pitch (elements) for width w: round_up(w, 8) + 8. */
int64_t hog_plane_pitch(int w);

/* gradient.py:95-121 (gradient_map) + gradient.py:56-72 (the table itself
 * is host-built, as in the reference, and uploaded as uint8 with -1 -> 0xFF;
 * lut is 511*511 bytes indexed (dx+255)*511 + (dy+255)).  c in {1, 3}.
 * Writes the bin map; border and zero-gradient pixels get -1. */
int hog_grad_bin(const uint8_t *img, int n, int c, int h, int w,
                 int64_t img_pitch, int64_t img_cstride, int64_t img_fstride,
                 const uint8_t *lut, int bins,
                 int8_t *binmap, int64_t bm_pitch, int64_t bm_fstride,
                 hog_stream_t stream);

/* Scratch needed by hog_integral / hog_pipeline for this shape (at the band
 * rows in effect on the calling thread, see hog_set_band_rows). */
size_t hog_scratch_bytes(int n, int h, int w, int bins, int stride, int cell);

/* Band rows R (plane rows per CTA of the integral-plane kernel) used by this
 * thread's following hog_pipeline / hog_integral / hog_scratch_bytes calls;
 * rows < 8 restores the automatic choice.  Any R gives the same planes; it
 * only changes the tiling (the batched pipeline measures a few per shape and
 * keeps the fastest).  hog_get_band_rows returns the R a call would use. */
void hog_set_band_rows(int rows);
int hog_get_band_rows(int n, int h, int w, int bins, int stride, int cell);

/* integral.py:58-87 (build_integral_stack, 32-bit accumulators): the N_b
 * padded summed-area tables of a bin map, every plane element written once. */
int hog_integral(const int8_t *binmap, int n, int h, int w, int64_t bm_pitch, int64_t bm_fstride,
                 int bins, int32_t *planes, int64_t pl_pitch, int64_t pl_nstride,
                 int64_t pl_fstride, void *scratch, size_t scratch_bytes, hog_stream_t stream);

/* Fused LUT-HOG pipeline over a frame batch: gradient + LUT binning
 * (gradient.py:95-121) -> integral planes (integral.py:58-87) -> cell
 * histogram grid by 4-corner reads (descriptor.py:162-188), for the regular
 * cell lattice produced by a stride-s scan (cell origins = multiples of
 * `stride` up to ((ncx-1)*stride, (ncy-1)*stride)).  grid may be NULL (no
 * cell grid).  Requires stride % 4 == 0, cell % stride == 0, cell/stride <= 2
 * when grid != NULL; otherwise use hog_integral + hog_cell_grid.
 * stages: HOG_STAGE_* bitmask (0 = all), optionally | HOG_STAGE_GRID_U8: `grid`
 * then points to uint8 [n][ncy][ncx][bins] (exact: a cell count is <= cell*cell).  A caller may run the stages of one
 * frame batch as separate calls on different streams (stage order per batch,
 * same scratch), e.g. to bin batch j+1 while batch j writes its planes.
 * For shapes with few bands per frame the carry scan (HOG_STAGE_SCAN: the column
 * recurrence of integral.py:75-79 across bands) is folded into the plane kernel
 * and that stage launches nothing; the choice depends only on the shape, so
 * separate calls for one batch agree (hog_last_pipeline_launches() reports it).
 * stage_events: NULL, or 4 cudaEvent_t recorded on `stream` before the
 * binning kernel, before the carry scans, before the plane kernel and after
 * it (lets a caller time each stage inside a larger timed region). */
int hog_pipeline(const uint8_t *img, int n, int c, int h, int w,
                 int64_t img_pitch, int64_t img_cstride, int64_t img_fstride,
                 const uint8_t *lut, int bins,
                 int8_t *binmap, int64_t bm_pitch, int64_t bm_fstride,
                 int32_t *planes, int64_t pl_pitch, int64_t pl_nstride, int64_t pl_fstride,
                 int cell, int stride, int ncx, int ncy, int32_t *grid,
                 void *scratch, size_t scratch_bytes, int stages, void *const *stage_events,
                 hog_stream_t stream);

/* Slab mode of hog_pipeline, for one frame split into row slabs across GPUs
 * (SURVEY §8f rank 2).  `img` points at the slab's first row inside the full
 * frame; halo_top / halo_bot say the frame continues above / below the slab
 * (row -1 / row h are read for the vertical gradient, and rows 0 / h-1 are
 * binned instead of being frame-border NO_BIN).  col_base (or NULL) is
 * int32 [n][bins][w] (frame stride base_fstride): per column, the count of
 * each bin in all frame rows above the slab -- the exclusive prefix over the
 * slabs above of hog_column_counts.  Plane row 0 of the output is then the
 * frame's plane row at the slab top, so every plane row equals the
 * single-GPU result. */
int hog_pipeline_slab(const uint8_t *img, int n, int c, int h, int w,
                      int64_t img_pitch, int64_t img_cstride, int64_t img_fstride,
                      const uint8_t *lut, int bins,
                      int8_t *binmap, int64_t bm_pitch, int64_t bm_fstride,
                      int32_t *planes, int64_t pl_pitch, int64_t pl_nstride, int64_t pl_fstride,
                      int cell, int stride, int ncx, int ncy, int32_t *grid,
                      void *scratch, size_t scratch_bytes, int stages, int halo_top, int halo_bot,
                      const int32_t *col_base, int64_t base_fstride, hog_stream_t stream);

/* Per-(bin, column) counts of bin-map rows [0, rows): out is int32
 * [n][bins][w].  A slab's own contribution to the column carries of the
 * slabs below it (integral.py:75-79 column sums restricted to the slab). */
int hog_column_counts(const int8_t *binmap, int n, int rows, int w, int64_t bm_pitch,
                      int64_t bm_fstride, int bins, int32_t *out, hog_stream_t stream);

/* descriptor.py:176-185 for an arbitrary (sorted) cell-origin set:
 * grid[f][j][i][b] = 4-corner count of the cell at (cell_ys[j], cell_xs[i]). */
int hog_cell_grid(const int32_t *planes, int n, int h, int w, int bins,
                  int64_t pl_pitch, int64_t pl_nstride, int64_t pl_fstride,
                  const int32_t *cell_xs, int ncx, const int32_t *cell_ys, int ncy, int cell,
                  int32_t *grid, hog_stream_t stream);

/* descriptor.py:94-104/119-124 for block == 1: one denominator per cell,
 * norm 1 (l1): sum|v| + eps_term, norm 2 (l2): sqrt(sum v^2 + eps_term).
 * denom is [n][ncells] float64.  Pass eps_term = _EPS (l1) or _EPS*_EPS (l2). */
int hog_cell_norm(const int32_t *grid, int n, int ncells, int bins, int norm, double eps_term,
                  double *denom, hog_stream_t stream);

/* descriptor.py:107-124 (_assemble_blocks) + detector.py:140-154 (scores):
 * for every window (iy, ix) of the scan, the descriptor is assembled from
 * grid[row_idx[iy][*]][col_idx[ix][*]] (descriptor.py:190-195) with the
 * block geometry and per-block normalisation (0 none, 1 l1, 2 l2), and
 *   scores[f][iy][ix] = dot(weights, descriptor) + bias      (if scores)
 *   desc[f][iy][ix][:] = descriptor (float64)                  (if desc)
 * row_idx is [noy][cells_y], col_idx is [nox][cells_x] (int32). */
int hog_window_features(const int32_t *grid, int n, int ncy, int ncx, int bins,
                        const int32_t *row_idx, int noy, const int32_t *col_idx, int nox,
                        int cells_x, int cells_y, int block, int block_stride,
                        int norm, double eps_term, const double *weights, double bias,
                        double *scores, double *desc, hog_stream_t stream);

/* detector.py:140-154 + descriptor.py:107-124 for block == 1 on a regular
 * cell lattice: window (iy, ix) reads cells (iy + cy*k, ix + cx*k), k = cell
 * / lattice step in {1, 2}, cells_x == 8 (64-pixel windows of 8-pixel cells).
 *   scores[f][iy][ix] = bias + sum_{cy,cx,b} w[(cy*8 + cx)*bins + b] * v
 * with v = grid value, or grid value / den[f][cell] (IEEE division) when den
 * (hog_cell_norm output) is given.  fp64 accumulation. */
int hog_scores_lattice(const int32_t *grid, const double *den, int n, int ncy, int ncx, int bins,
                       int noy, int nox, int cells_x, int cells_y, int k, const double *weights,
                       double bias, double *scores, hog_stream_t stream);

/* hog_scores_lattice over a uint8 cell grid (the plane kernel's byte grid,
 * STAGE_GRID_U8; exact since cell counts <= cell^2 <= 255), unnormalised.
 * Same windows, weights layout and fp64 accumulation; the byte grid quarters
 * the kernel's staging footprint.  detector.py:140-154, descriptor.py:107-118. */
int hog_scores_lattice_u8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                          int cells_x, int cells_y, int k, const double *weights, double bias,
                          double *scores, hog_stream_t stream);

/* Exact window scores on the integer tensor cores (detector.py:140-154,
 * descriptor.py:107-118; same windows and weights layout as
 * hog_scores_lattice_u8 with k = 1, i.e. stride = cell, cells_x = 8,
 * cells_y <= 16, bins <= HOG_I8_MAX_BINS).  The dot of a window's counts with
 * the weights is evaluated exactly in integers and rounded once to float64,
 * then the bias is added (the reference: float64 ddot + bias).
 * hog_scores_i8_prepare (host only, no CUDA) writes each weight as an integer
 * times 2^-F in `*digits` signed base-256 digits, laid out as tensor-core
 * fragments in `frag` (hog_scores_i8_frag_bytes(bins) host bytes, to be
 * copied to a 16-byte aligned device buffer).  Exact when the weights span
 * at most 47 bits (float32-valued weights span ~37); wider (float64) weights
 * are rounded to multiples of 2^(e - 46), |w| < 2^e the largest (error <= 2^(e - 47)),
 * of the size of float64 rounding in the dot itself.  HOG_ERANGE for non-finite
 * or vanishingly small (< 2^-950) weights: use hog_scores_lattice_u8. */
#define HOG_I8_MAX_BINS 20
#define HOG_I8_MAX_DIGITS 6
size_t hog_scores_i8_frag_bytes(int bins);
int hog_scores_i8_prepare(const double *weights, int cells_x, int cells_y, int bins, void *frag,
                          int *digits, double *scale);
int hog_scores_lattice_i8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                          int cells_x, int cells_y, const void *frag, int digits, double scale,
                          double bias, double *scores, hog_stream_t stream);

/* detector.py:202-221 (_resize_bilinear): separable bilinear, pixel centres
 * aligned, float64 in the reference's operation order (no FMA contraction),
 * rint half-even, clip to 0..255.  ry = h / nh and rx = w / nw as computed by
 * the caller in float64. */
int hog_resize_bilinear(const uint8_t *src, int n, int c, int h, int w,
                        int64_t src_pitch, int64_t src_cstride, int64_t src_fstride,
                        int nh, int nw, double ry, double rx,
                        uint8_t *dst, int64_t dst_pitch, int64_t dst_cstride, int64_t dst_fstride,
                        hog_stream_t stream);

/* integral.py:58-87 with acc_width=16: uint16 planes [n][bins][h+1][w+1]
 * (pl_pitch >= w+1), for frames whose pixel count w*h <= 65535 (the
 * reference's overflow guard; larger frames are rejected with HOG_EINVAL).
 * Half the plane bytes of hog_integral. */
int hog_integral16(const int8_t *binmap, int n, int h, int w, int64_t bm_pitch, int64_t bm_fstride,
                   int bins, uint16_t *planes, int64_t pl_pitch, int64_t pl_nstride,
                   int64_t pl_fstride, hog_stream_t stream);

/* integral.py:95-115 (rect_count / rect_histogram) for a batch of k
 * half-open rectangles rects[r] = (x0, y0, x1, y1) int32 of ONE frame's
 * planes (uint32 when elem_bytes == 4, uint16 when 2):
 *   out[r][b] = p[b][y1][x1] + p[b][y0][x0] - p[b][y1][x0] - p[b][y0][x1]  (int64).
 * The caller validates rectangles (0 <= x0 < x1 <= w, 0 <= y0 < y1 <= h), as
 * integral.py:90-92 does before reading. */
int hog_rect_histogram(const void *planes, int elem_bytes, int64_t pl_pitch, int64_t pl_nstride,
                       int bins, const int32_t *rects, int k, int64_t *out, hog_stream_t stream);

/* Scratch bytes for hog_detect over n score maps of `windows` windows each. */
size_t hog_detect_scratch_bytes(int n, int64_t windows);

/* detector.py:145-153 (strict `score > threshold`, row-major window order)
 * + :194-199 (box = rint(origin * scale), Python round half-to-even; w, h =
 * int(round(window * scale)) given as ww, wh) + :261-267 (pyramid: clamp to
 * an image of clamp_w x clamp_h when clamp_w > 0).  scores is [n][noy][nox]
 * float64, oxs[nox] / oys[noy] the window origins.  Per frame f the first
 * min(count[f], cap) hits are written in the reference's list order:
 * boxes[f][k] = (x, y, w, h) int32, out_scores[f][k], out_window[f][k] =
 * iy*nox + ix (out_window may be NULL).  count[f] is the total number of
 * hits (a caller whose cap was too small sees count > cap). */
int hog_detect(const double *scores, int n, int noy, int nox, double threshold,
               const int32_t *oxs, const int32_t *oys, double scale, int ww, int wh,
               int clamp_w, int clamp_h, int cap, int32_t *boxes, double *out_scores,
               int64_t *out_window, int32_t *count, void *scratch, size_t scratch_bytes,
               hog_stream_t stream);

/* Scratch bytes for hog_nms over n detections. */
size_t hog_nms_scratch_bytes(int n);

/* EXTENSION (not a reference function): per-WINDOW L2 norms for BASELINE
 * configs[2]'s "per-window L2 normalisation"; the reference normalises per
 * block (descriptor.py:107-124).  norms[f][iy][ix] = sqrt(sum over the window's
 * cells (row_idx[iy][0..cells_y) x col_idx[ix][0..cells_x)) of sum_b v^2 +
 * eps_term), v the cell counts of `grid` ([n][ncy][ncx][bins], uint8 when
 * elem_bytes == 1, int32 when 4); eps_term = _EPS*_EPS (descriptor.py:123).
 * Bit-exact with np.sqrt((d*d).sum() + eps_term) of the window's unnormalised
 * descriptor d.  k > 0: the lattice is regular (window (iy, ix) reads cells
 * (iy + cy*k, ix + cx*k); the index maps are then not read) and the sums are
 * separable; k = 0: the index maps give the cells.  cell_sq: caller scratch of
 * n*ncy*ncx (+ n*ncy*nox when k > 0) int32. */
int hog_window_l2(const void *grid, int elem_bytes, int n, int ncy, int ncx, int bins,
                  const int32_t *row_idx, int noy, const int32_t *col_idx, int nox, int cells_x,
                  int cells_y, int k, double eps_term, int32_t *cell_sq, double *norms,
                  hog_stream_t stream);

/* detector.py:285-299 (nms): greedy non-maximum suppression of n boxes
 * (x, y, w, h int32) with scores and scales (float64): candidates in order
 * of (-score, y, x, scale) (stable), a candidate is kept iff its IoU
 * (detector.py:272-282, float64) with every kept box is <= iou_threshold.
 * keep[0 .. *keep_count) receives the kept input indices in that order. */
int hog_nms(const int32_t *boxes, const double *scores, const double *scales, int n,
            double iou_threshold, int32_t *keep, int32_t *keep_count, void *scratch,
            size_t scratch_bytes, hog_stream_t stream);

/* detector.py:285-299 (nms) for boxes with float64 (x, y, w, h): any
 * Detection a caller builds, e.g. non-integer coordinates.  Same order and
 * rule as hog_nms; the IoU rounds once per double operation in Python's
 * order (detector.py:272-282).  Scratch: hog_nms_scratch_bytes(n). */
int hog_nms_f64(const double *boxes, const double *scores, const double *scales, int n,
                double iou_threshold, int32_t *keep, int32_t *keep_count, void *scratch,
                size_t scratch_bytes, hog_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HOGB200_H */
