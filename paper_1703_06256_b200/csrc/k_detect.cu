// k_detect.cu -- detections on the device: threshold compaction of the score
// map into boxes (detector.py:145-153 strict `>`, row-major order;
// :194-199 box mapping; :261-267 pyramid clamping) and greedy NMS
// (detector.py:272-299: order by (-score, y, x, scale), a box survives iff
// its IoU with every kept box is <= the threshold).
//
// Compaction: k_det_count counts hits per tile of DT_TILE windows, one CTA
// per frame scans the tile counts (k_det_offsets), k_det_scatter re-reads
// the tile, ranks the hits with warp ballots and writes boxes in row-major
// order -- deterministic, the same order as the reference's list.
// NMS: a stable merge sort (CUB) of indices under the reference's key, then
// one CTA sweeps the sorted list in blocks of NMS_B candidates: each
// candidate is tested against the boxes already kept (earlier blocks), the
// block's pairwise suppression bits are computed in parallel, and one warp
// resolves the block greedily from the bit matrix.  IoU is computed in
// double exactly as the reference does (integer box coordinates, so every
// intermediate is exact and the final division is correctly rounded).
#include <cub/device/device_merge_sort.cuh>

#include "hog_common.cuh"

namespace hogb200 {

constexpr int DT_TILE = 1024, DT_THREADS = 256;

__global__ void k_det_count(const double *__restrict__ scores, int64_t m, int tiles, double thr,
                            int32_t *__restrict__ tile_cnt) {
    const int f = blockIdx.y, t = blockIdx.x;
    const double *s = scores + (int64_t)f * m;
    int c = 0;
    for (int i = threadIdx.x; i < DT_TILE; i += DT_THREADS) {
        const int64_t w = (int64_t)t * DT_TILE + i;
        c += (w < m && s[w] > thr) ? 1 : 0;
    }
    c = __reduce_add_sync(FULL, c);
    __shared__ int part[DT_THREADS / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int q = 0; q < DT_THREADS / 32; ++q) tot += part[q];
        tile_cnt[(int64_t)f * tiles + t] = tot;
    }
}

// one CTA per frame: exclusive scan of the tile counts, frame total
__global__ void k_det_offsets(const int32_t *__restrict__ tile_cnt, int tiles,
                              int32_t *__restrict__ tile_off, int32_t *__restrict__ count) {
    const int f = blockIdx.x;
    const int32_t *c = tile_cnt + (int64_t)f * tiles;
    int32_t *o = tile_off + (int64_t)f * tiles;
    __shared__ int carry;
    __shared__ int wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < tiles; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < tiles ? c[i] : 0;
        int inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(FULL, inc, d);
            if (lane >= d) inc += t;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        int before = carry;
        for (int q = 0; q < warp; ++q) before += wsum[q];
        if (i < tiles) o[i] = before + inc - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) {
            int tot = carry;
            for (int q = 0; q < nw; ++q) tot += wsum[q];
            carry = tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) count[f] = carry;
}

struct DetMap {
    const int32_t *oxs, *oys;  // window origins (level coordinates)
    int nox;
    double scale;              // box = rint(origin * scale) (Python round: half to even)
    int ww, wh;                // int(round(window * scale)), host-computed
    int clamp_w, clamp_h;      // > 0: pyramid clamping to the original image
};

__global__ void k_det_scatter(const double *__restrict__ scores, int64_t m, int tiles, double thr,
                              const int32_t *__restrict__ tile_off, DetMap dm, int cap,
                              int32_t *__restrict__ boxes, double *__restrict__ out_scores,
                              int64_t *__restrict__ out_window) {
    const int f = blockIdx.y, t = blockIdx.x;
    const double *s = scores + (int64_t)f * m;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int wcount[DT_TILE / 32];
    __shared__ int wbase[DT_TILE / 32];
    // pass 1: per-warp-slab hit counts (slab = 32 consecutive windows)
    for (int slab = warp; slab < DT_TILE / 32; slab += DT_THREADS / 32) {
        const int64_t w = (int64_t)t * DT_TILE + slab * 32 + lane;
        const bool hit = w < m && s[w] > thr;
        const unsigned b = __ballot_sync(FULL, hit);
        if (lane == 0) wcount[slab] = __popc(b);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = tile_off[(int64_t)f * tiles + t];
        for (int q = 0; q < DT_TILE / 32; ++q) {
            wbase[q] = run;
            run += wcount[q];
        }
    }
    __syncthreads();
    for (int slab = warp; slab < DT_TILE / 32; slab += DT_THREADS / 32) {
        const int64_t w = (int64_t)t * DT_TILE + slab * 32 + lane;
        const double sc = w < m ? s[w] : 0.0;
        const bool hit = w < m && sc > thr;
        const unsigned b = __ballot_sync(FULL, hit);
        const int k = wbase[slab] + __popc(b & ((1u << lane) - 1u));
        if (hit && k < cap) {
            const int iy = (int)(w / dm.nox), ix = (int)(w - (int64_t)iy * dm.nox);
            int x = (int)rint((double)dm.oxs[ix] * dm.scale);
            int y = (int)rint((double)dm.oys[iy] * dm.scale);
            int bw = dm.ww, bh = dm.wh;
            if (dm.clamp_w > 0) {  // detector.py:261-267
                x = min(max(x, 0), dm.clamp_w - 1);
                y = min(max(y, 0), dm.clamp_h - 1);
                bw = min(bw, dm.clamp_w - x);
                bh = min(bh, dm.clamp_h - y);
            }
            int32_t *bp = boxes + ((int64_t)f * cap + k) * 4;
            bp[0] = x;
            bp[1] = y;
            bp[2] = bw;
            bp[3] = bh;
            out_scores[(int64_t)f * cap + k] = sc;
            if (out_window) out_window[(int64_t)f * cap + k] = w;
        }
    }
}

// ---------------------------------------------------------------------------
// NMS

// Boxes are (x, y, w, h) as int32 (what hog_detect emits) or as float64
// (any Detection a caller builds); the IoU follows detector.py:272-282 in
// the box type's arithmetic: integer sums and differences, then one rounding
// per double operation in Python's order (no FMA contraction).
template <typename B>
struct NmsLess {  // detector.py:292: key (-score, y, x, scale)
    const B *boxes;
    const double *scores, *scales;
    __device__ bool operator()(int a, int b) const {
        const double sa = scores[a], sb = scores[b];
        if (sa != sb) return sa > sb;
        const B ya = boxes[4 * a + 1], yb = boxes[4 * b + 1];
        if (ya != yb) return ya < yb;
        const B xa = boxes[4 * a], xb = boxes[4 * b];
        if (xa != xb) return xa < xb;
        return scales[a] < scales[b];
    }
};

template <typename B> struct Box4;
template <> struct Box4<int32_t> { using T = int4; };
template <> struct Box4<double> { using T = double4; };

__device__ __forceinline__ double box_iou(int4 a, int4 b) {  // detector.py:272-282
    const double ix = fmax(0.0, (double)(min(a.x + a.z, b.x + b.z) - max(a.x, b.x)));
    const double iy = fmax(0.0, (double)(min(a.y + a.w, b.y + b.w) - max(a.y, b.y)));
    const double inter = ix * iy;
    if (inter <= 0.0) return 0.0;
    const double uni = ((double)a.z * (double)a.w + (double)b.z * (double)b.w) - inter;
    return inter / uni;
}

__device__ __forceinline__ double box_iou(double4 a, double4 b) {  // detector.py:272-282
    const double ix = fmax(0.0, __dsub_rn(fmin(__dadd_rn(a.x, a.z), __dadd_rn(b.x, b.z)), fmax(a.x, b.x)));
    const double iy = fmax(0.0, __dsub_rn(fmin(__dadd_rn(a.y, a.w), __dadd_rn(b.y, b.w)), fmax(a.y, b.y)));
    const double inter = __dmul_rn(ix, iy);
    if (inter <= 0.0) return 0.0;
    const double uni = __dsub_rn(__dadd_rn(__dmul_rn(a.z, a.w), __dmul_rn(b.z, b.w)), inter);
    return __ddiv_rn(inter, uni);
}

constexpr int NMS_B = 1024;

__global__ void k_iota(int32_t *v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

// one CTA of NMS_B threads; mask scratch: NMS_B x NMS_B/32 words
template <typename B>
__global__ void __launch_bounds__(NMS_B)
k_nms_greedy(const B *__restrict__ boxes, const int32_t *__restrict__ order, int n, double thr,
             uint32_t *__restrict__ mask, typename Box4<B>::T *__restrict__ kept_box,
             int32_t *__restrict__ keep, int32_t *__restrict__ keep_count) {
    using T = typename Box4<B>::T;
    extern __shared__ __align__(16) unsigned char nms_smem[];
    T *blk = reinterpret_cast<T *>(nms_smem);                         // [NMS_B]
    int *blk_keep_idx = reinterpret_cast<int *>(blk + NMS_B);         // [NMS_B]
    unsigned char *sup = reinterpret_cast<unsigned char *>(blk_keep_idx + NMS_B);  // [NMS_B]
    __shared__ int kept_n, blk_kept;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) kept_n = 0;
    __syncthreads();
    for (int base = 0; base < n; base += NMS_B) {
        const int i = base + tid;
        const bool valid = i < n;
        T bx{};
        if (valid) bx = reinterpret_cast<const T *>(boxes)[order[i]];
        blk[tid] = bx;
        // (1) against every box kept in earlier blocks
        bool s = !valid;
        const int kn = kept_n;
        for (int k = 0; k < kn && !s; ++k) s = box_iou(bx, kept_box[k]) > thr;
        sup[tid] = s ? 1 : 0;
        __syncthreads();
        // (2) pairwise suppression bits inside the block: bit j of row tid, j > tid
        const int nb = min(NMS_B, n - base);
        for (int wd = 0; wd < NMS_B / 32; ++wd) {
            unsigned bits = 0;
            const int j0 = wd * 32;
            if (j0 + 31 > tid && j0 < nb && valid) {
                for (int q = 0; q < 32; ++q) {
                    const int j = j0 + q;
                    if (j > tid && j < nb && box_iou(bx, blk[j]) > thr) bits |= 1u << q;
                }
            }
            mask[(size_t)tid * (NMS_B / 32) + wd] = bits;
        }
        __syncthreads();
        // (3) one warp resolves the block in sorted order
        if (tid < 32) {
            unsigned removed = 0;  // lane w holds bits of candidates 32w .. 32w+31
            int kcount = 0;
            for (int c = 0; c < nb; ++c) {
                const unsigned rw = __shfl_sync(FULL, removed, c >> 5);
                const bool alive = !sup[c] && !((rw >> (c & 31)) & 1u);
                if (alive) {
                    removed |= mask[(size_t)c * (NMS_B / 32) + lane];
                    if (lane == 0) blk_keep_idx[kcount] = c;
                    ++kcount;
                }
            }
            if (lane == 0) blk_kept = kcount;
        }
        __syncthreads();
        const int bk = blk_kept;
        for (int q = tid; q < bk; q += NMS_B) {
            const int c = blk_keep_idx[q];
            kept_box[kn + q] = blk[c];
            keep[kn + q] = order[base + c];
        }
        __syncthreads();
        if (tid == 0) kept_n = kn + bk;
        __syncthreads();
    }
    if (tid == 0) *keep_count = kept_n;
}

template <typename B>
static size_t nms_scratch_t(int n) {
    size_t sort_bytes = 0;
    NmsLess<B> less{nullptr, nullptr, nullptr};
    cub::DeviceMergeSort::StableSortKeys(nullptr, sort_bytes, (int32_t *)nullptr, n, less);
    auto r = [](size_t b) { return (b + 255) / 256 * 256; };
    return r(sort_bytes) + r(sizeof(int32_t) * (size_t)n) + r(sizeof(typename Box4<B>::T) * (size_t)n) +
           r(sizeof(uint32_t) * (size_t)NMS_B * (NMS_B / 32));
}

size_t nms_scratch_bytes(int n) {
    const size_t a = nms_scratch_t<int32_t>(n), b = nms_scratch_t<double>(n);
    return a > b ? a : b;
}

template <typename B>
static int launch_nms_t(const B *boxes, const double *scores, const double *scales, int n, double thr,
                        int32_t *keep, int32_t *keep_count, void *scratch, cudaStream_t st) {
    using T = typename Box4<B>::T;
    size_t sort_bytes = 0;
    NmsLess<B> less{boxes, scores, scales};
    cub::DeviceMergeSort::StableSortKeys(nullptr, sort_bytes, (int32_t *)nullptr, n, less);
    auto r = [](size_t b) { return (b + 255) / 256 * 256; };
    char *p = (char *)scratch;
    void *tmp = p;
    p += r(sort_bytes);
    int32_t *order = (int32_t *)p;
    p += r(sizeof(int32_t) * (size_t)n);
    T *kept_box = (T *)p;
    p += r(sizeof(T) * (size_t)n);
    uint32_t *mask = (uint32_t *)p;
    k_iota<<<blocks_for(n, 256), 256, 0, st>>>(order, n);
    if (cub::DeviceMergeSort::StableSortKeys(tmp, sort_bytes, order, n, less, st) != cudaSuccess)
        return -1;
    const size_t smem = (sizeof(T) + sizeof(int) + 1) * NMS_B;
    static size_t configured[HOG_MAX_DEVICES] = {};
    if (smem_optin_needed(configured, smem))
        cudaFuncSetAttribute(k_nms_greedy<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_nms_greedy<B><<<1, NMS_B, smem, st>>>(boxes, order, n, thr, mask, kept_box, keep, keep_count);
    return 0;
}

int launch_nms(const int32_t *boxes, const double *scores, const double *scales, int n, double thr,
               int32_t *keep, int32_t *keep_count, void *scratch, size_t sbytes, cudaStream_t st) {
    (void)sbytes;
    return launch_nms_t<int32_t>(boxes, scores, scales, n, thr, keep, keep_count, scratch, st);
}

int launch_nms_f64(const double *boxes, const double *scores, const double *scales, int n, double thr,
                   int32_t *keep, int32_t *keep_count, void *scratch, size_t sbytes, cudaStream_t st) {
    (void)sbytes;
    return launch_nms_t<double>(boxes, scores, scales, n, thr, keep, keep_count, scratch, st);
}

size_t det_scratch_bytes(int n, int64_t m) {
    const int64_t tiles = (m + DT_TILE - 1) / DT_TILE;
    return 2 * (((size_t)n * tiles * sizeof(int32_t) + 255) / 256 * 256);
}

void launch_detect(const double *scores, int n, int64_t m, double thr, const DetMap &dm, int cap,
                   int32_t *boxes, double *out_scores, int64_t *out_window, int32_t *count,
                   void *scratch, cudaStream_t st) {
    const int tiles = (int)((m + DT_TILE - 1) / DT_TILE);
    int32_t *tile_cnt = (int32_t *)scratch;
    int32_t *tile_off = tile_cnt + (((size_t)n * tiles * sizeof(int32_t) + 255) / 256 * 256) / 4;
    const dim3 grid((unsigned)tiles, (unsigned)n);
    k_det_count<<<grid, DT_THREADS, 0, st>>>(scores, m, tiles, thr, tile_cnt);
    k_det_offsets<<<n, 1024, 0, st>>>(tile_cnt, tiles, tile_off, count);
    k_det_scatter<<<grid, DT_THREADS, 0, st>>>(scores, m, tiles, thr, tile_off, dm, cap, boxes,
                                               out_scores, out_window);
}

void launch_detect_abi(const double *scores, int n, int noy, int nox, double thr, const int32_t *oxs,
                       const int32_t *oys, double scale, int ww, int wh, int clamp_w, int clamp_h,
                       int cap, int32_t *boxes, double *out_scores, int64_t *out_window,
                       int32_t *count, void *scratch, cudaStream_t st) {
    DetMap dm{oxs, oys, nox, scale, ww, wh, clamp_w, clamp_h};
    launch_detect(scores, n, (int64_t)noy * nox, thr, dm, cap, boxes, out_scores, out_window, count,
                  scratch, st);
}

}  // namespace hogb200
