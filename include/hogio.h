/*
 * hogio.h -- C ABI of libhogio.so: host-side wire formats of the LUT-HOG
 * path.  PNM decoding into caller memory (pinned host
 * buffers that feed the H2D copy of a frame batch) and the text descriptor
 * dump of `fasthog extract`.
 *
 * Reference (paths relative to /root/reference/pkg/src/fasthog/):
 *   image_io.py:50-87   _Tokenizer (whitespace, '#' comments to end of line)
 *   image_io.py:90-122  decode_pnm (P2/P3/P5/P6, maxval 255, planar output)
 *   cli.py:124-143      _format_value / cmd_extract lines "x y v0 v1 ..."
 * Return codes map onto the reference's exception classes.
 */
#ifndef HOGIO_H
#define HOGIO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOGIO_OK 0
#define HOGIO_EMAGIC 1  /* UnsupportedMagic  */
#define HOGIO_EMAXVAL 2 /* MaxvalNot255      */
#define HOGIO_ETRUNC 3  /* TruncatedData     */
#define HOGIO_ETOKEN 4  /* NonNumericToken   */
#define HOGIO_EINVAL 5  /* bad arguments     */
#define HOGIO_EIO 6     /* file could not be read (OSError) */
#define HOGIO_ESHAPE 7  /* a batch file's shape differs from the batch */

/* Text of the last error on the calling thread. */
const char *hogio_last_error(void);

/* Parse the header only: channels (1 or 3), height, width. */
int hogio_pnm_header(const uint8_t *data, size_t len, int *channels, int *height, int *width);

/* image_io.py:90-122: decode into planar uint8
 * out[ch * plane_stride + y * pitch + x]  (pitch >= width). */
int hogio_pnm_decode(const uint8_t *data, size_t len, uint8_t *out, int64_t pitch,
                     int64_t plane_stride);

/* Read and decode n files of one shape (c, h, w) on `threads` host threads
 * into frame i at out + i * frame_stride (planar as above).  status[i] gets
 * each file's code; the call returns the first failing code (0 if none). */
int hogio_decode_batch(const char *const *paths, int n, int c, int h, int w, uint8_t *out,
                       int64_t frame_stride, int64_t pitch, int64_t plane_stride, int threads,
                       int *status);

/* cli.py:124-143: one line per row, "x y v0 ... v{dim-1}\n", values printed
 * as integers (as_int != 0, normalization "none") or with "%.9g" (Python's
 * format(v, ".9g")).  Writes at most cap bytes to dst (dst may be NULL) and
 * returns the number of bytes the full text needs. */
int64_t hogio_format_descriptors(const int32_t *xs, const int32_t *ys, const double *values,
                                 int64_t rows, int dim, int as_int, char *dst, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* HOGIO_H */
