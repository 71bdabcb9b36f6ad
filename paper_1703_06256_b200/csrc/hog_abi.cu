// hog_abi.cu -- C ABI of libhogb200.so (include/hogb200.h): argument checks,
// tile geometry, scratch carve-up, and kernel dispatch.  The kernels live in
// k_bin.cu, k_planes_*.cu and k_window.cu.
//
// Reference: /root/reference/pkg/src/fasthog (pure Python + NumPy).  The hot
// path is gradient.py:95-121 (LUT binning), integral.py:58-87 (per-bin
// summed-area tables), descriptor.py:162-195 (cell histograms from 4 corner
// reads) and detector.py:140-154 / 202-221 (scores, pyramid resize).
//
// Design (DESIGN.md has the roofline numbers):
//   The integral planes (4*N_b bytes per pixel) are ~90% of the compulsory
//   HBM traffic, so every plane element is written exactly once, with
//   16-byte coalesced stores, by k_planes.  One warp owns a band of R plane
//   rows of one frame and sweeps it strip by strip (4 columns per lane, 128
//   columns per strip), walking down each strip: the row prefix is a warp
//   scan of one-hot counts packed two bins per 32-bit word (16-bit lanes; a
//   row prefix never exceeds the width), the column prefix lives in
//   registers, and the row prefix left of the strip is handed from strip to
//   strip through shared memory.  The only carry that crosses warps is the
//   per-column count above the band: k_grad_bin counts bins per (band,
//   column) while it bins the image, and k_scan_cols turns those counts into
//   the column counts above every band.  When the scan lattice is regular,
//   k_planes also emits the cell-histogram grid from the plane values it
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>
#include <mutex>

#include "hog_common.cuh"

namespace hogb200 {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(HOG_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return HOG_OK;
}


static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

// Tables proven equal to the octant classifier (k_lut_proof), per device.
// A table handed to the library is treated as immutable, like the
// reference's read-only OrientationLut (gradient.py:55-72); hog_lut_forget
// drops a pointer whose contents the caller rewrites.
struct LutKey {
    int dev;
    const uint8_t *lut;
    int bins;
    bool operator<(const LutKey &o) const {
        return dev != o.dev ? dev < o.dev : lut != o.lut ? lut < o.lut : bins < o.bins;
    }
};
static std::mutex g_lut_mu;
static std::map<LutKey, bool> g_lut_ok;

// mismatching (dx, dy) entries of the table against the octant classifier
// (-1: bins not handled by it; -2: CUDA error)
static long long lut_proof_run(const uint8_t *lut, int bins, cudaStream_t st) {
    if (bins != 4 && bins != 8) return -1;
    unsigned long long *d = nullptr, h = 0;
    if (cudaMallocAsync(&d, sizeof(h), st) != cudaSuccess) return -2;
    cudaMemsetAsync(d, 0, sizeof(h), st);
    launch_lut_proof(bins, lut, d, st);
    cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -2;
    return (long long)h;
}

bool lut_proven(const uint8_t *lut, int bins, cudaStream_t st) {
    if (bins != 4 && bins != 8) return false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    const LutKey key{dev, lut, bins};
    {
        std::lock_guard<std::mutex> lk(g_lut_mu);
        auto it = g_lut_ok.find(key);
        if (it != g_lut_ok.end()) return it->second;
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return false;  // cannot synchronise inside a capture: the table-gather kernel runs
    const long long bad = lut_proof_run(lut, bins, st);
    if (bad < -1) {
        cudaGetLastError();
        return false;
    }
    std::lock_guard<std::mutex> lk(g_lut_mu);
    g_lut_ok[key] = bad == 0;
    return bad == 0;
}

// Band rows R of the plane kernel for this thread's next calls (0: automatic).
// Thread-local: a caller sets it around its own launches.
thread_local int g_band_rows = 0;

// kernels the last hog_pipeline / hog_pipeline_slab call of this thread launched
thread_local int g_last_launches = 0;

// k_planes shared memory per CTA must allow two resident CTAs per SM
constexpr int K2_SMEM_BUDGET = 113 * 1024;

// tma: k_planes stages plane rows in shared memory and writes them with TMA
// bulk stores (needs 32-B aligned plane rows, po.vec); one extra store warp,
// so at most 7 compute warps (strips) per CTA.
TileGeom make_geom(int n, int h, int w, int bins, bool fused, int stride, int cell, bool v8ok,
                   bool tma) {
    TileGeom g{};
    g.n = n; g.h = h; g.w = w; g.bins = bins;
    g.NWB = (bins + 3) / 4;
    g.NW = (bins + 1) / 2;
    g.NWp = (int)round_up(g.NW, 4);
    // 8 columns per lane only when every lattice column starts a lane chunk.
    // Measured on B200 (HOGB200_VC A/B): 8 columns win for <= 8 bins on big
    // batches (c4 planes 1.45 vs 1.55 ms); 4 columns win for 9-10 bins (c3:
    // 1.01 vs 1.17 ms) and for single small frames (c1: 20 vs 29 us).
    const bool big = (int64_t)n * h * w >= ((int64_t)64 << 20);
    g.VC = (v8ok && g.NW <= 4 && big && (!fused || stride % 8 == 0) &&
            env_int("HOGB200_VC", 8) == 8) ? 8 : 4;
    const int span = 32 * g.VC;
    if (fused) {
        int a = 8, b = stride;
        while (b) { int r = a % b; a = b; b = r; }
        const int l = 8 / a * stride;  // lcm(8, stride): strips start on lattice columns, 32-B aligned
        g.Ws = ((span + stride - cell) / l) * l;
        g.halo = cell - stride;
    } else {
        g.Ws = span;
        g.halo = 0;
    }
    g.ns = (w + g.Ws - 1) / g.Ws;
    // Opt-in (HOGB200_TMA=1).  Measured on B200 (c2, 128 frames): 334 us vs 281 us
    // with per-thread 16-B stores -- the plane kernel is issue/latency-bound, not
    // store-bound, and staging adds shared-memory traffic and 9% instructions
    // (profiles/r1_tma_store_ab.md).  Pure stores do reach 7.2 TB/s this way
    // (tools/probe_tma_store.cu) against 5.5 TB/s for st.global.
    tma = HOGB200_VARIANTS && tma && env_int("HOGB200_TMA", 0) != 0;
    // top row in registers when a band's strips fit the 6-warp variant (c2: 6
    // strips; measured 1.153 -> 1.136 ms); wider small-bin frames keep 8 warps
    g.PREG = (K2_PTOP_REG && 2 * g.NW * g.VC <= 32 && !tma && g.ns <= 6 &&
              env_int("HOGB200_PTOP_REG", 1)) ? 1 : 0;
    const int maxw = k2_maxt(g.NW, g.VC, g.PREG != 0) / 32 - (tma ? 1 : 0);
    g.NWARP = g.ns < maxw ? g.ns : maxw;
    g.nss = (g.ns + g.NWARP - 1) / g.NWARP;
    // spread the strips evenly over the super-strips: the last super-strip of a
    // band otherwise runs with idle warps (8K pyramid level 5: 25 strips as 6+6+6+6+1)
    if (env_int("HOGB200_BALANCE_STRIPS", 1)) g.NWARP = (g.ns + g.nss - 1) / g.nss;
    g.nc1 = (w + CHUNK - 1) / CHUNK;
    g.Wc = g.nc1 * CHUNK;
    int R = 128;
    const char *env = getenv("HOGB200_BAND_ROWS");
    if (g_band_rows >= 8) {  // hog_set_band_rows: the caller measured this shape
        R = g_band_rows;
    } else if (env && atoi(env) >= 8) {
        R = atoi(env);
    } else {
        while (R > 16 && (int64_t)n * (h / R + 1) * g.NWARP < 148 * 32) R /= 2;
    }
    // u8 column counts and packed strip-local sums (< 2^16) bound R at 240;
    // clamp first, then keep R a multiple of the lattice step (fused grid)
    if (R > 240) R = 240;
    if (fused && R % stride != 0) R = R / stride * stride > 0 ? R / stride * stride : stride;
    g.R = R;
    // k_grad_bin runs R1 = R / S1 row sub-bands per warp, so its grid is several
    // waves deep (one R-row band per warp left a 1.08-wave tail on c2)
    g.S1 = 1;
    const int s_env = env_int("HOGB200_SUBBANDS", 0);
    if (s_env > 0 && R % s_env == 0) {
        g.S1 = s_env;
    } else if (s_env <= 0) {
        // warps: ~2 full waves (B200: c3 1.179 -> 1.167 ms against 4 waves; c5, c1, c2 shard unchanged)
        const int64_t target = (int64_t)env_int("HOGB200_BIN_WAVES", 2) * 148 * 64;
        // octant binning (N_b 4 / 8) counts in blocks of 8 rows: keep R1 % 8 == 0
        const bool oct = bins == 4 || bins == 8;
        while (R % (2 * g.S1) == 0 && R / (2 * g.S1) >= 16 && (!oct || (R / (2 * g.S1)) % 8 == 0) &&
               (int64_t)n * ((h + R / g.S1 - 1) / (R / g.S1)) * ((w + CHUNK - 1) / CHUNK) < target)
            g.S1 *= 2;
    }
    g.R1 = R / g.S1;
    g.nb1 = (h + g.R1 - 1) / g.R1;
    g.nb2 = h / R + 1;
    g.Lrows = R + g.halo;
    g.TMA = tma ? 1 : 0;
    if (tma) {
        // widest CTA (fewest super-strips) whose staging ring of >= 3 rows (else 2)
        // fits the two-CTAs-per-SM budget
        const int kr = fused ? cell / stride : 0;
        const int ring_env = env_int("HOGB200_RING", 0), nw_env = env_int("HOGB200_NWARP", 0);
        bool done = false;
        for (int minring = 3; minring >= 2 && !done; --minring) {
            for (int nw = (nw_env > 0 && nw_env < g.NWARP) ? nw_env : g.NWARP; nw >= 1 && !done; --nw) {
                TileGeom t = g;
                t.nss = (g.ns + nw - 1) / nw;
                t.NWARP = (g.ns + t.nss - 1) / t.nss;
                t.SEGW = (int)round_up((int64_t)t.NWARP * t.Ws + 8, 8);
                for (int ring = ring_env > 0 ? ring_env : 4; ring >= minring; --ring) {
                    t.RING = ring;
                    if (k2_smem_words(t, kr) * 4 <= K2_SMEM_BUDGET || ring_env > 0) {
                        g = t;
                        done = true;
                        break;
                    }
                }
            }
        }
        if (!done) g.TMA = 0;  // per-thread stores
    }
    return g;
}

size_t carve(const TileGeom &g, void *base, Scratch *sc) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += round_up((int64_t)bytes, 256);
        return o;
    };
    size_t oC = take(sizeof(uint32_t) * (size_t)g.n * (g.nb1 > g.nb2 ? g.nb1 : g.nb2) * g.Wc * g.NWB);
    size_t oV = take(sizeof(uint32_t) * (size_t)g.n * g.nb2 * g.Wc * g.NWp);
    size_t oF = take(sizeof(uint32_t) * ((size_t)g.n * g.nb2 + 1));
    if (sc && base) {
        char *b = (char *)base;
        sc->C = (uint32_t *)(b + oC);
        sc->V = (uint32_t *)(b + oV);
        sc->flags = (uint32_t *)(b + oF);
    }
    return off;
}


int check_frames(int n, int h, int w) {
    if (n < 1) return fail(HOG_EINVAL, "n must be >= 1, got %d", n);
    if (h < 3 || w < 3) return fail(HOG_EINVAL, "need at least 3x3, got %dx%d", w, h);
    if (h >= 65000 || w >= 65000) return fail(HOG_EINVAL, "frame %dx%d exceeds 65000 per side", w, h);
    return HOG_OK;
}

int check_bins(int bins) {
    if (bins < 2 || bins > 64) return fail(HOG_EINVAL, "bins must be in [2, 64], got %d", bins);
    return HOG_OK;
}

// Sub-bands of the octant binning kernel (gray, N_b 4 / 8).  It runs whole
// bands per half-warp where the batch fills the GPU -- its per-unit setup and
// count transposes then amortise over R rows (B200, c2: 0.155 ms with R/4-row
// sub-bands, 0.140 ms with R-row ones) -- and splits bands (R1 a multiple of
// 8) only until the grid is ~2 waves of its 4 CTAs per SM (64-frame shards,
// single frames).  smax: the sub-band count the scratch was sized for.
static void oct_subbands(TileGeom &g, int c, int smax) {
    if ((c != 1 && c != 3) || (g.bins != 4 && g.bins != 8) || env_int("HOGB200_SUBBANDS", 0) > 0) return;
    auto ctas = [&](int s) {
        const int r1 = g.R / s;
        return (int64_t)g.n * ((g.h + r1 - 1) / r1) * g.nc1 / 8;  // 8 half-warp units per CTA
    };
    int s = 1;
    while (2 * s <= smax && g.R % (2 * s) == 0 && (g.R / (2 * s)) % 8 == 0 && ctas(s) < 2 * 148 * 4)
        s *= 2;
    g.S1 = s;
    g.R1 = g.R / s;
    g.nb1 = (g.h + g.R1 - 1) / g.R1;
}

// Row-bulk plane stores (k_planes RB): whole rows staged in shared memory and
// written by one contiguous cp.async.bulk each.  Needs every strip of a row in
// one CTA with all warps active, row-major contiguous rows (pp == bins * pns),
// columns -7 .. w all written by the CTA (w % 8 == 0) and the two row slots
// inside the two-CTAs-per-SM shared-memory budget.
static void rowbulk_geom(TileGeom &g, const PlaneOut &po, int kr) {
    g.RB = 0;
    if (!env_int("HOGB200_ROWBULK", 1) || g.TMA || !g.PREG || g.NW != 4 || g.nss != 1 ||
        g.ns != g.NWARP || !po.vec || po.pp != (int64_t)g.bins * po.pns || g.w % 8 != 0 ||
        po.pns != (int64_t)g.w + 8)  // every staged column (-7 .. w) is written each row
        return;
    g.RB = 1;
    g.RBP = (int)po.pns;
    if ((size_t)k2_smem_words(g, kr) * 4 > (size_t)K2_SMEM_BUDGET) g.RB = 0;
}

int check_pitch4(const void *p, int64_t pitch, int w, const char *what) {
    if (((uintptr_t)p & 3) != 0 || pitch % 4 != 0 || pitch < round_up(w, 4))
        return fail(HOG_EINVAL, "%s: need 4-byte aligned base and pitch %% 4 == 0, pitch >= %lld (got %lld)",
                    what, (long long)round_up(w, 4), (long long)pitch);
    return HOG_OK;
}

PlaneOut make_po(int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int w) {
    PlaneOut po{pl, pp, pns, pfs, 0};
    po.vec = (((uintptr_t)(pl + 1) & 31) == 0) && pp % 8 == 0 && pns % 8 == 0 && pfs % 8 == 0 &&
             pp >= round_up(w, 8) + 8;
    return po;
}

bool v8_ok(const PlaneOut &po, const int8_t *bm, int64_t bp, int64_t bfs) {
    return po.vec && ((uintptr_t)bm & 7) == 0 && bp % 8 == 0 && bfs % 8 == 0;
}

// N_b > 18: groups of <= 16 consecutive bins, each through the single-write
// plane kernel on a bin-offset copy of the bin map (k_bin_offset)
constexpr int GROUP_BINS = 16;
inline int bin_groups(int bins) { return (bins + GROUP_BINS - 1) / GROUP_BINS; }
inline int group_range(int bins, int gi, int *b0) {
    const int ng = bin_groups(bins), base = bins / ng, rem = bins % ng;
    *b0 = gi * base + (gi < rem ? gi : rem);
    return base + (gi < rem ? 1 : 0);
}
inline int64_t group_bm_pitch(int w) { return round_up(w, 8); }
inline size_t group_bm_bytes(int n, int h, int w) {
    return (size_t)round_up((int64_t)n * h * group_bm_pitch(w), 256);
}

int integral_group_impl(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int bins,
                        int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, void *scratch,
                        size_t sbytes, cudaStream_t st) {
    const int64_t op = group_bm_pitch(w), ofs = (int64_t)h * op;
    const size_t tb = group_bm_bytes(n, h, w);
    if (scratch == nullptr || sbytes < tb)
        return fail(HOG_EINVAL, "scratch too small: need more than %zu bytes, got %zu", tb, sbytes);
    int8_t *tmp = (int8_t *)scratch;
    void *rest = (char *)scratch + tb;
    for (int gi = 0; gi < bin_groups(bins); ++gi) {
        int b0;
        const int nb = group_range(bins, gi, &b0);
        PlaneOut po = make_po(pl + (int64_t)b0 * pns, pp, pns, pfs, w);
        TileGeom g = make_geom(n, h, w, nb, false, 0, 0, v8_ok(po, tmp, op, ofs), po.vec != 0);
        Scratch sc{};
        const size_t need = carve(g, nullptr, nullptr);
        if (sbytes < tb + need)
            return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", tb + need, sbytes);
        carve(g, rest, &sc);
        launch_bin_offset(bm, bp, bfs, n, h, w, b0, tmp, op, ofs, st);
        GridOut go{nullptr, 4, 4, 1, 1, 0};
        launch_counts_from_bm(g.NW, tmp, op, ofs, g, sc, st);
        launch_scan(g.NW, g, sc, st);
        launch_planes(g.NW, 0, 0, tmp, op, ofs, po, go, g, sc, FusedIn{}, st);
    }
    return check_launch("hog_integral (bin groups)");
}

int integral_impl(const int8_t *bm, int64_t bp, int64_t bfs, int n, int h, int w, int bins,
                  int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, void *scratch, size_t sbytes,
                  cudaStream_t st) {
    PlaneOut po = make_po(pl, pp, pns, pfs, w);
    if (bins > MAX_FUSED_BINS)
        return integral_group_impl(bm, bp, bfs, n, h, w, bins, pl, pp, pns, pfs, scratch, sbytes, st);
    TileGeom g = make_geom(n, h, w, bins, false, 0, 0, v8_ok(po, bm, bp, bfs), po.vec != 0);
    Scratch sc{};
    size_t need = carve(g, nullptr, nullptr);
    if (scratch == nullptr || sbytes < need)
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", need, sbytes);
    carve(g, scratch, &sc);
    GridOut go{nullptr, 4, 4, 1, 1, 0};
    launch_counts_from_bm(g.NW, bm, bp, bfs, g, sc, st);
    launch_scan(g.NW, g, sc, st);
    launch_planes(g.NW, 0, 0, bm, bp, bfs, po, go, g, sc, FusedIn{}, st);
    return check_launch("hog_integral");
}

}  // namespace hogb200

using namespace hogb200;

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char *hog_version(void) { return "hogb200 1.2 sm_100a"; }

const char *hog_last_error(void) { return g_err.c_str(); }

int hog_last_pipeline_launches(void) { return hogb200::g_last_launches; }

int hog_lut_proof(const uint8_t *lut, int bins, long long *mismatches, hog_stream_t stream) {
    g_err.clear();
    if (!lut || !mismatches) return fail(HOG_EINVAL, "null pointer");
    const long long bad = lut_proof_run(lut, bins, (cudaStream_t)stream);
    if (bad < -1) return check_launch("hog_lut_proof") ? HOG_ECUDA : fail(HOG_ECUDA, "hog_lut_proof failed");
    *mismatches = bad;
    int dev = 0;
    if (bad >= 0 && cudaGetDevice(&dev) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_lut_mu);
        g_lut_ok[LutKey{dev, lut, bins}] = bad == 0;
    }
    return HOG_OK;
}

void hog_lut_forget(const uint8_t *lut) {
    std::lock_guard<std::mutex> lk(g_lut_mu);
    for (auto it = g_lut_ok.begin(); it != g_lut_ok.end();)
        it = it->first.lut == lut ? g_lut_ok.erase(it) : std::next(it);
}

int64_t hog_plane_pitch(int w) { return round_up((int64_t)w, 8) + 8; }

int hog_grad_bin(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                 int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp, int64_t bfs,
                 hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (c != 1 && c != 3) return fail(HOG_EINVAL, "channels must be 1 or 3, got %d", c);
    if ((e = check_pitch4(img, ip, w, "image")) || (e = check_pitch4(bm, bp, w, "binmap"))) return e;
    if (!img || !lut || !bm) return fail(HOG_EINVAL, "null buffer");
    TileGeom g = make_geom(n, h, w, bins, false, 0, 0, false, false);
    oct_subbands(g, c, 1 << 20);  // no counts: no scratch bound on the sub-bands
    Scratch sc{};
    launch_grad_bin(1, c, false, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, (cudaStream_t)stream);
    return check_launch("hog_grad_bin");
}

size_t hog_scratch_bytes(int n, int h, int w, int bins, int stride, int cell) {
    if (n < 1 || h < 1 || w < 1 || bins < 1) return 0;
    bool fused = stride > 0 && cell > 0;
    size_t m = 0;
    if (bins > MAX_FUSED_BINS) {  // hog_integral in bin groups: offset bin map + a group's scratch
        for (int gi = 0; gi < bin_groups(bins); ++gi) {
            int b0;
            const int nb = group_range(bins, gi, &b0);
            for (int v8 = 0; v8 < 2; ++v8) {
                const size_t a = carve(make_geom(n, h, w, nb, false, 0, 0, v8, true), nullptr, nullptr);
                m = a > m ? a : m;
            }
        }
        return group_bm_bytes(n, h, w) + m;
    }
    for (int v8 = 0; v8 < 2; ++v8) {
        for (int tma = 0; tma < 2; ++tma) {
            size_t a = carve(make_geom(n, h, w, bins, fused, stride, cell, v8, tma), nullptr, nullptr);
            size_t b = carve(make_geom(n, h, w, bins, false, 0, 0, v8, tma), nullptr, nullptr);
            m = a > m ? a : m;
            m = b > m ? b : m;
        }
    }
    return m;
}

int hog_integral(const int8_t *bm, int n, int h, int w, int64_t bp, int64_t bfs, int bins,
                 int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, void *scratch,
                 size_t sbytes, hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if ((e = check_pitch4(bm, bp, w, "binmap"))) return e;
    if (pp < (int64_t)w + 1) return fail(HOG_EINVAL, "plane pitch %lld < w+1", (long long)pp);
    if (!bm || !pl) return fail(HOG_EINVAL, "null buffer");
    return integral_impl(bm, bp, bfs, n, h, w, bins, pl, pp, pns, pfs, scratch, sbytes,
                         (cudaStream_t)stream);
}

}  // extern "C"

static int pipeline_impl(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                         int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp,
                         int64_t bfs, int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int cell,
                         int stride, int ncx, int ncy, int32_t *grid, void *scratch, size_t sbytes,
                         int stages, void *const *stage_events, int halo_top, int halo_bot,
                         const int32_t *col_base, int64_t base_fs, hog_stream_t stream) {
    if ((stages & HOG_STAGE_ALL) == 0) stages |= HOG_STAGE_ALL;
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (c != 1 && c != 3) return fail(HOG_EINVAL, "channels must be 1 or 3, got %d", c);
    if ((e = check_pitch4(img, ip, w, "image")) || (e = check_pitch4(bm, bp, w, "binmap"))) return e;
    if (pp < (int64_t)w + 1) return fail(HOG_EINVAL, "plane pitch %lld < w+1", (long long)pp);
    if (!img || !lut || !bm || !pl) return fail(HOG_EINVAL, "null buffer");
    if (bins > MAX_FUSED_BINS)
        return fail(HOG_EINVAL, "fused pipeline supports bins <= %d (got %d); use hog_grad_bin + "
                    "hog_integral + hog_cell_grid", MAX_FUSED_BINS, bins);
    int kr = 0;
    if (grid) {
        if (stride <= 0 || stride % 4 != 0 || cell % stride != 0 || cell / stride > 2 || cell % 4 != 0 ||
            stride > 240)
            return fail(HOG_EINVAL, "fused grid needs stride %% 4 == 0, stride <= 240, cell %% stride == 0, "
                        "cell/stride <= 2 (stride %d, cell %d)", stride, cell);
        if (ncx < 1 || ncy < 1 || (int64_t)(ncx - 1) * stride + cell > w ||
            (int64_t)(ncy - 1) * stride + cell > h)
            return fail(HOG_EINVAL, "cell lattice %dx%d (step %d, cell %d) exceeds %dx%d", ncx, ncy,
                        stride, cell, w, h);
        kr = cell / stride;
    }
    cudaStream_t st = (cudaStream_t)stream;
    PlaneOut po = make_po(pl, pp, pns, pfs, w);
    // the fused-binning variant (opt-in, below) keeps per-thread plane stores
    const char *fenv = getenv("HOGB200_FUSED");
    const bool want_fused = HOGB200_VARIANTS && (stages & HOG_STAGE_ALL) == HOG_STAGE_ALL && po.vec &&
                            fenv && fenv[0] == '1';
    TileGeom g = make_geom(n, h, w, bins, kr > 0, stride, cell, v8_ok(po, bm, bp, bfs),
                           po.vec != 0 && !want_fused);
    g.ht = halo_top ? 1 : 0;
    g.hb = halo_bot ? 1 : 0;
    oct_subbands(g, c, g.S1);  // never more sub-bands than the scratch was sized for
    rowbulk_geom(g, po, kr);
    if (want_fused) g.PREG = 0, g.RB = 0;  // the fused kernel keeps the band's top row in shared memory
    // Few sub-bands above any band (c1's single frame aside: c2, c4, the multi-GPU shards):
    // k_planes sums the sub-band counts itself when that reads at most HOGB200_NOSCAN_PCT
    // (default 5) percent of the plane bytes it writes; k_scan_cols and V are skipped.
    // A pure function of the geometry, so a caller that runs the stages in separate calls
    // gets the same answer in each (the scan stage is then a no-op); not in slab mode (the
    // scan adds the carry of the slabs above).
    {
        const int pct = env_int("HOGB200_NOSCAN_PCT", 5);
        g.NOSCAN = (!want_fused && !col_base && !halo_top && !halo_bot && pct > 0 &&
                    (int64_t)g.nb1 * g.NWB * 100 <= (int64_t)pct * 2 * g.R * bins) ? 1 : 0;
    }
    Scratch sc{};
    size_t need = carve(g, nullptr, nullptr);
    if (scratch == nullptr || sbytes < need)
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes, got %zu", need, sbytes);
    carve(g, scratch, &sc);
    sc.base = col_base;
    sc.base_fs = base_fs;
    GridOut go{grid, kr ? stride : 4, kr ? cell : 4, kr ? ncx : 1, kr ? ncy : 1,
               (stages & HOG_STAGE_GRID_U8) ? 1 : 0};
    if (go.u8 && cell * cell > 255)
        return fail(HOG_EINVAL, "uint8 cell grid needs cell*cell <= 255 (cell %d)", cell);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (stage_events) cudaStreamIsCapturing(st, &cap);
    auto mark = [&](int i) {
        if (!stage_events || !stage_events[i]) return;
        // inside a CUDA-graph capture the record becomes an external event node,
        // so the caller can still time the stages of every replay
        if (cap == cudaStreamCaptureStatusActive)
            cudaEventRecordWithFlags((cudaEvent_t)stage_events[i], st, cudaEventRecordExternal);
        else
            cudaEventRecord((cudaEvent_t)stage_events[i], st);
    };
    // Opt-in (HOGB200_FUSED=1): the fused plane kernel bins its own rows and
    // takes the band carries by decoupled look-back (no k_grad_bin /
    // k_scan_cols passes).  Measured slower on B200 (c2: 1.73 vs 1.29 ms per
    // step): binning is latency-bound and starves at the plane kernel's
    // occupancy, so the default is the three-kernel path.
    const bool fused = want_fused && g.nss == 1 && !halo_top && !halo_bot && !col_base;
    g_last_launches = 0;
    if (fused) {
        FusedIn fi{img, ip, ics, ifs, lut, sc.flags, sc.flags + (size_t)g.n * g.nb2};
        cudaMemsetAsync(sc.flags, 0, sizeof(uint32_t) * ((size_t)g.n * g.nb2 + 1), st);
        mark(0);
        mark(1);
        mark(2);
        launch_planes(g.NW, kr, c, bm, bp, bfs, po, go, g, sc, fi, st);
        g_last_launches = 1;
        mark(3);
    } else {
        mark(0);
        if (stages & HOG_STAGE_BIN) {
            launch_grad_bin(g.NWB, c, true, img, ip, ics, ifs, lut, bm, bp, bfs, g, sc, st);
            ++g_last_launches;
        }
        mark(1);
        if ((stages & HOG_STAGE_SCAN) && !g.NOSCAN) {
            launch_scan(g.NW, g, sc, st);
            ++g_last_launches;
        }
        mark(2);
        if (stages & HOG_STAGE_PLANES) {
            launch_planes(g.NW, kr, 0, bm, bp, bfs, po, go, g, sc, FusedIn{}, st);
            ++g_last_launches;
        }
        mark(3);
    }
    return check_launch("hog_pipeline");
}

extern "C" {

int hog_pipeline(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                 int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp, int64_t bfs,
                 int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int cell, int stride, int ncx,
                 int ncy, int32_t *grid, void *scratch, size_t sbytes, int stages,
                 void *const *stage_events, hog_stream_t stream) {
    g_err.clear();
    return pipeline_impl(img, n, c, h, w, ip, ics, ifs, lut, bins, bm, bp, bfs, pl, pp, pns, pfs,
                         cell, stride, ncx, ncy, grid, scratch, sbytes, stages, stage_events, 0, 0,
                         nullptr, 0, stream);
}

void hog_set_band_rows(int rows) { g_band_rows = rows >= 8 ? rows : 0; }

int hog_get_band_rows(int n, int h, int w, int bins, int stride, int cell) {
    if (n < 1 || h < 1 || w < 1 || bins < 1) return 0;
    return make_geom(n, h, w, bins, stride > 0 && cell > 0, stride, cell, true, false).R;
}

int hog_pipeline_slab(const uint8_t *img, int n, int c, int h, int w, int64_t ip, int64_t ics,
                      int64_t ifs, const uint8_t *lut, int bins, int8_t *bm, int64_t bp,
                      int64_t bfs, int32_t *pl, int64_t pp, int64_t pns, int64_t pfs, int cell,
                      int stride, int ncx, int ncy, int32_t *grid, void *scratch, size_t sbytes,
                      int stages, int halo_top, int halo_bot, const int32_t *col_base,
                      int64_t base_fstride, hog_stream_t stream) {
    g_err.clear();
    return pipeline_impl(img, n, c, h, w, ip, ics, ifs, lut, bins, bm, bp, bfs, pl, pp, pns, pfs,
                         cell, stride, ncx, ncy, grid, scratch, sbytes, stages, nullptr, halo_top,
                         halo_bot, col_base, base_fstride, stream);
}

int hog_column_counts(const int8_t *bm, int n, int rows, int w, int64_t bp, int64_t bfs, int bins,
                      int32_t *out, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || n > 65535 || rows < 0 || w < 1 || bins < 1 || bins > 64 || !bm || !out)
        return fail(HOG_EINVAL, "bad arguments");
    launch_column_counts(bm, bp, bfs, n, rows, w, bins, out, (cudaStream_t)stream);
    return check_launch("hog_column_counts");
}

int hog_cell_grid(const int32_t *pl, int n, int h, int w, int bins, int64_t pp, int64_t pns,
                  int64_t pfs, const int32_t *cxs, int ncx, const int32_t *cys, int ncy, int cell,
                  int32_t *grid, hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if (ncx < 1 || ncy < 1 || cell < 1) return fail(HOG_EINVAL, "empty cell lattice");
    if (!pl || !cxs || !cys || !grid) return fail(HOG_EINVAL, "null buffer");
    launch_cell_grid(pl, pp, pns, pfs, n, bins, cxs, ncx, cys, ncy, cell, grid, (cudaStream_t)stream);
    return check_launch("hog_cell_grid");
}

int hog_cell_norm(const int32_t *grid, int n, int ncells, int bins, int norm, double eps_term,
                  double *den, hog_stream_t stream) {
    g_err.clear();
    if (norm != 1 && norm != 2) return fail(HOG_EINVAL, "norm must be 1 (l1) or 2 (l2)");
    if (n < 1 || ncells < 1 || bins < 1 || !grid || !den) return fail(HOG_EINVAL, "bad arguments");
    const int64_t tot = (int64_t)n * ncells;
    launch_cell_norm(grid, tot, bins, norm, eps_term, den, (cudaStream_t)stream);
    return check_launch("hog_cell_norm");
}

int hog_window_l2(const void *grid, int elem_bytes, int n, int ncy, int ncx, int bins,
                  const int32_t *row_idx, int noy, const int32_t *col_idx, int nox, int cells_x,
                  int cells_y, int k, double eps_term, int32_t *cell_sq, double *norms,
                  hog_stream_t stream) {
    g_err.clear();
    if (elem_bytes != 1 && elem_bytes != 4) return fail(HOG_EINVAL, "elem_bytes must be 1 or 4");
    if (n < 1 || ncy < 1 || ncx < 1 || bins < 1 || noy < 1 || nox < 1 || cells_x < 1 || cells_y < 1 ||
        !grid || !row_idx || !col_idx || !cell_sq || !norms)
        return fail(HOG_EINVAL, "bad arguments");
    if (k > 0 && ((int64_t)(noy - 1) + (int64_t)(cells_y - 1) * k >= ncy ||
                  (int64_t)(nox - 1) + (int64_t)(cells_x - 1) * k >= ncx))
        return fail(HOG_EINVAL, "window grid exceeds the cell lattice");
    launch_window_l2(grid, elem_bytes, n, ncy, ncx, bins, row_idx, noy, col_idx, nox, cells_x, cells_y,
                     k, eps_term, cell_sq, norms, (cudaStream_t)stream);
    return check_launch("hog_window_l2");
}

int hog_window_features(const int32_t *grid, int n, int ncy, int ncx, int bins,
                        const int32_t *row_idx, int noy, const int32_t *col_idx, int nox,
                        int cells_x, int cells_y, int block, int bstride, int norm,
                        double eps_term, const double *wts, double bias, double *scores,
                        double *desc, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || bins < 1 || !grid || !row_idx || !col_idx)
        return fail(HOG_EINVAL, "bad arguments");
    if (block < 1 || block > cells_x || block > cells_y || bstride < 1)
        return fail(HOG_EINVAL, "block %d / stride %d do not fit %dx%d cells", block, bstride,
                    cells_x, cells_y);
    if (norm < 0 || norm > 2) return fail(HOG_EINVAL, "norm must be 0, 1 or 2");
    if (scores && !wts) return fail(HOG_EINVAL, "scores need weights");
    launch_window_features(grid, n, ncy, ncx, bins, row_idx, noy, col_idx, nox, cells_x, cells_y,
                           block, bstride, norm, eps_term, wts, bias, scores, desc,
                           (cudaStream_t)stream);
    return check_launch("hog_window_features");
}

int hog_scores_lattice(const int32_t *grid, const double *den, int n, int ncy, int ncx, int bins,
                       int noy, int nox, int cells_x, int cells_y, int k, const double *wts,
                       double bias, double *scores, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || bins < 1 || !grid || !wts || !scores)
        return fail(HOG_EINVAL, "bad arguments");
    if (k != 1 && k != 2) return fail(HOG_EINVAL, "lattice step ratio must be 1 or 2, got %d", k);
    if (cells_x != 8) return fail(HOG_EINVAL, "hog_scores_lattice is built for 8 cells across, got %d", cells_x);
    if ((int64_t)(noy - 1) + (int64_t)(cells_y - 1) * k >= ncy || (int64_t)(nox - 1) + 7 * k >= ncx)
        return fail(HOG_EINVAL, "window grid exceeds the cell lattice");
    launch_scores_lattice(grid, den, n, ncy, ncx, bins, noy, nox, cells_y, k, wts, bias, scores,
                          (cudaStream_t)stream);
    return check_launch("hog_scores_lattice");
}

int hog_scores_lattice_u8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                          int cells_x, int cells_y, int k, const double *wts, double bias,
                          double *scores, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || bins < 1 || !grid || !wts || !scores)
        return fail(HOG_EINVAL, "bad arguments");
    if (k != 1 && k != 2) return fail(HOG_EINVAL, "lattice step ratio must be 1 or 2, got %d", k);
    if (cells_x != 8)
        return fail(HOG_EINVAL, "hog_scores_lattice_u8 is built for 8 cells across, got %d", cells_x);
    if ((int64_t)(noy - 1) + (int64_t)(cells_y - 1) * k >= ncy || (int64_t)(nox - 1) + 7 * k >= ncx)
        return fail(HOG_EINVAL, "window grid exceeds the cell lattice");
    launch_scores_rows_u8(grid, n, ncy, ncx, bins, noy, nox, cells_y, k, wts, bias, scores,
                          (cudaStream_t)stream);
    return check_launch("hog_scores_lattice_u8");
}

// ---- exact integer-tensor-core scores (k_scores_i8.cu) ----------------------

size_t hog_scores_i8_frag_bytes(int bins) {
    if (bins < 1 || bins > HOG_I8_MAX_BINS) return 0;
    return (size_t)HOG_I8_MAX_DIGITS * scores_i8_ks(bins) * 32 * 16;
}

int hog_scores_i8_prepare(const double *w, int cells_x, int cells_y, int bins, void *frag,
                          int *digits, double *scale) {
    g_err.clear();
    if (!w || !frag || !digits || !scale) return fail(HOG_EINVAL, "null pointer");
    if (cells_x != 8) return fail(HOG_EINVAL, "integer scores are built for 8 cells across, got %d", cells_x);
    if (cells_y < 1 || cells_y > 16) return fail(HOG_EINVAL, "integer scores need 1..16 cell rows, got %d", cells_y);
    if (bins < 1 || bins > HOG_I8_MAX_BINS)
        return fail(HOG_EINVAL, "integer scores need 1..%d bins, got %d", HOG_I8_MAX_BINS, bins);
    const int nw = cells_y * cells_x * bins;
    // F: every weight times 2^F is an integer (the lowest set mantissa bit of any weight)
    int lsb = INT_MAX, top = INT_MIN;
    for (int i = 0; i < nw; ++i) {
        const double v = w[i];
        if (!std::isfinite(v)) return fail(HOG_ERANGE, "weight %d is not finite", i);
        if (v == 0.0) continue;
        int e;
        const double m = std::frexp(std::fabs(v), &e);  // |v| = m 2^e, m in [0.5, 1)
        uint64_t M = (uint64_t)std::ldexp(m, 53);        // 53-bit integer mantissa
        const int tz = __builtin_ctzll(M);
        lsb = std::min(lsb, e - 53 + tz);
        top = std::max(top, e);
    }
    // exact when every W fits 47 bits (float32-valued weights span ~37); wider
    // weights (float64 mantissas) are rounded to the grid 2^(top - 46): an error
    // <= 2^(top - 47) per weight, the size of float64 rounding in the dot itself
    int F = lsb == INT_MAX ? 0 : -lsb;
    const int maxbits = 8 * HOG_I8_MAX_DIGITS - 1;
    const bool exact = lsb == INT_MAX || top + F <= maxbits;
    if (!exact) F = maxbits - 1 - top;
    if (F > 1000) return fail(HOG_ERANGE, "weights too small for the integer path (2^-%d)", F);
    const int bitsW = lsb == INT_MAX ? 0 : top + F;
    int S = 1;
    while (8 * S - 1 < bitsW) ++S;
    const int KS = scores_i8_ks(bins), P = 4 * KS;
    std::vector<int8_t> d((size_t)HOG_I8_MAX_DIGITS * nw, 0);  // d[s][i]
    for (int i = 0; i < nw; ++i) {
        long long W = std::llround(std::ldexp(w[i], F));
        if (exact && (double)W != std::ldexp(w[i], F)) return fail(HOG_ERANGE, "weight %d is not exact at 2^-%d", i, F);
        for (int s = 0; s < S; ++s) {
            long long r = ((W % 256) + 256) % 256;
            if (r >= 128) r -= 256;
            d[(size_t)s * nw + i] = (int8_t)r;
            W = (W - r) / 256;
        }
        if (W != 0) return fail(HOG_ERANGE, "weight %d does not fit %d digits", i, S);
    }
    // mma.sync m16n8k32 A fragments: [s][ks][lane] x 4 registers; register r of
    // lane (g, t) holds row g + 8 (r & 1), k = 32 ks + 4 t + 16 (r >> 1) .. + 3
    const int Sk = std::max(S, 4);
    uint32_t *out = static_cast<uint32_t *>(frag);
    std::memset(frag, 0, hog_scores_i8_frag_bytes(bins));
    for (int s = 0; s < S; ++s)
        for (int ks = 0; ks < KS; ++ks)
            for (int lane = 0; lane < 32; ++lane)
                for (int r = 0; r < 4; ++r) {
                    const int row = (lane >> 2) + 8 * (r & 1);
                    const int k0 = 32 * ks + 4 * (lane & 3) + 16 * (r >> 1);
                    uint32_t word = 0;
                    for (int q = 0; q < 4; ++q) {
                        const int k = k0 + q, cx = k / P, n = k % P;
                        if (row < cells_y && cx < cells_x && n < bins)
                            word |= (uint32_t)(uint8_t)d[(size_t)s * nw + (row * cells_x + cx) * bins + n] << (8 * q);
                    }
                    out[(((size_t)s * KS + ks) * 32 + lane) * 4 + r] = word;
                }
    *digits = Sk;
    *scale = std::ldexp(1.0, -F);
    return HOG_OK;
}

int hog_scores_lattice_i8(const uint8_t *grid, int n, int ncy, int ncx, int bins, int noy, int nox,
                          int cells_x, int cells_y, const void *frag, int digits, double scale,
                          double bias, double *scores, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || !grid || !frag || !scores) return fail(HOG_EINVAL, "bad arguments");
    if (bins < 1 || bins > HOG_I8_MAX_BINS)
        return fail(HOG_EINVAL, "integer scores need 1..%d bins, got %d", HOG_I8_MAX_BINS, bins);
    if (cells_x != 8) return fail(HOG_EINVAL, "integer scores are built for 8 cells across, got %d", cells_x);
    if (cells_y < 1 || cells_y > 16) return fail(HOG_EINVAL, "integer scores need 1..16 cell rows, got %d", cells_y);
    if (digits < 4 || digits > HOG_I8_MAX_DIGITS) return fail(HOG_EINVAL, "digits must be 4..%d, got %d", HOG_I8_MAX_DIGITS, digits);
    if ((int64_t)(noy - 1) + (cells_y - 1) >= ncy || (int64_t)(nox - 1) + 7 >= ncx)
        return fail(HOG_EINVAL, "window grid exceeds the cell lattice");
    if (((uintptr_t)frag & 15) != 0) return fail(HOG_EINVAL, "fragments must be 16-byte aligned");
    if ((bins % 4 == 0 && ((uintptr_t)grid & 3)) || (bins % 2 == 0 && ((uintptr_t)grid & 1)))
        return fail(HOG_EINVAL, "grid pointer misaligned for %d bins", bins);
    launch_scores_i8(grid, n, ncy, ncx, bins, noy, nox, frag, digits, scale, bias, scores,
                     (cudaStream_t)stream);
    return check_launch("hog_scores_lattice_i8");
}

int hog_resize_bilinear(const uint8_t *src, int n, int c, int h, int w, int64_t sp, int64_t scs,
                        int64_t sfs, int nh, int nw, double ry, double rx, uint8_t *dst,
                        int64_t dp, int64_t dcs, int64_t dfs, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || c < 1 || h < 1 || w < 1 || nh < 1 || nw < 1 || !src || !dst)
        return fail(HOG_EINVAL, "bad arguments");
    if (nh > 65535 || (int64_t)n * c > 65535)
        return fail(HOG_EINVAL, "resize: nh (%d) and n*c (%lld) must be <= 65535", nh, (long long)n * c);
    launch_resize(src, n, c, h, w, sp, scs, sfs, nh, nw, ry, rx, dst, dp, dcs, dfs,
                  (cudaStream_t)stream);
    return check_launch("hog_resize_bilinear");
}

int hog_integral16(const int8_t *bm, int n, int h, int w, int64_t bp, int64_t bfs, int bins,
                   uint16_t *pl, int64_t pp, int64_t pns, int64_t pfs, hog_stream_t stream) {
    g_err.clear();
    int e;
    if ((e = check_frames(n, h, w)) || (e = check_bins(bins))) return e;
    if ((int64_t)w * h > 65535)
        return fail(HOG_EINVAL, "16-bit accumulators need w*h <= 65535, got %dx%d = %lld", w, h,
                    (long long)w * h);
    if (pp < (int64_t)w + 1) return fail(HOG_EINVAL, "plane pitch %lld < w+1", (long long)pp);
    if (!bm || !pl) return fail(HOG_EINVAL, "null buffer");
    launch_integral16(bm, bp, bfs, n, h, w, bins, pl, pp, pns, pfs, (cudaStream_t)stream);
    return check_launch("hog_integral16");
}

int hog_rect_histogram(const void *pl, int elem_bytes, int64_t pp, int64_t pns, int bins,
                       const int32_t *rects, int k, int64_t *out, hog_stream_t stream) {
    g_err.clear();
    if (elem_bytes != 2 && elem_bytes != 4) return fail(HOG_EINVAL, "elem_bytes must be 2 or 4");
    if (k < 0 || bins < 1 || (k > 0 && (!pl || !rects || !out))) return fail(HOG_EINVAL, "bad arguments");
    if (k == 0) return HOG_OK;
    launch_rect_hist(pl, elem_bytes, pp, pns, bins, rects, k, out, (cudaStream_t)stream);
    return check_launch("hog_rect_histogram");
}

size_t hog_detect_scratch_bytes(int n, int64_t windows) {
    if (n < 1 || windows < 1) return 0;
    return det_scratch_bytes(n, windows);
}

int hog_detect(const double *scores, int n, int noy, int nox, double threshold, const int32_t *oxs,
               const int32_t *oys, double scale, int ww, int wh, int clamp_w, int clamp_h, int cap,
               int32_t *boxes, double *out_scores, int64_t *out_window, int32_t *count,
               void *scratch, size_t sbytes, hog_stream_t stream) {
    g_err.clear();
    if (n < 1 || noy < 1 || nox < 1 || cap < 0 || !scores || !oxs || !oys || !count || !scratch)
        return fail(HOG_EINVAL, "bad arguments");
    if (cap > 0 && (!boxes || !out_scores)) return fail(HOG_EINVAL, "null output buffer");
    if (n > 65535) return fail(HOG_EINVAL, "n must be <= 65535");
    if (sbytes < det_scratch_bytes(n, (int64_t)noy * nox))
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes",
                    det_scratch_bytes(n, (int64_t)noy * nox));
    launch_detect_abi(scores, n, noy, nox, threshold, oxs, oys, scale, ww, wh, clamp_w, clamp_h,
                      cap, boxes, out_scores, out_window, count, scratch, (cudaStream_t)stream);
    return check_launch("hog_detect");
}

size_t hog_nms_scratch_bytes(int n) { return n < 1 ? 0 : nms_scratch_bytes(n); }

}  // extern "C"

template <typename B, typename L>
static int nms_impl(const B *boxes, const double *scores, const double *scales, int n,
                    double iou_threshold, int32_t *keep, int32_t *keep_count, void *scratch,
                    size_t sbytes, hog_stream_t stream, L launch, const char *what) {
    g_err.clear();
    if (!(iou_threshold >= 0.0 && iou_threshold <= 1.0))
        return fail(HOG_EINVAL, "iou_threshold must be in [0, 1], got %g", iou_threshold);
    if (n < 0 || !keep_count) return fail(HOG_EINVAL, "bad arguments");
    if (n == 0) {
        cudaMemsetAsync(keep_count, 0, sizeof(int32_t), (cudaStream_t)stream);
        return check_launch(what);
    }
    if (!boxes || !scores || !scales || !keep || !scratch) return fail(HOG_EINVAL, "null buffer");
    if (sbytes < nms_scratch_bytes(n))
        return fail(HOG_EINVAL, "scratch too small: need %zu bytes", nms_scratch_bytes(n));
    if (launch(boxes, scores, scales, n, iou_threshold, keep, keep_count, scratch, sbytes,
               (cudaStream_t)stream) != 0)
        return fail(HOG_ECUDA, "%s: sort failed", what);
    return check_launch(what);
}

extern "C" {

int hog_nms_f64(const double *boxes, const double *scores, const double *scales, int n,
                double iou_threshold, int32_t *keep, int32_t *keep_count, void *scratch,
                size_t sbytes, hog_stream_t stream) {
    return nms_impl(boxes, scores, scales, n, iou_threshold, keep, keep_count, scratch, sbytes,
                    stream, launch_nms_f64, "hog_nms_f64");
}

int hog_nms(const int32_t *boxes, const double *scores, const double *scales, int n,
            double iou_threshold, int32_t *keep, int32_t *keep_count, void *scratch, size_t sbytes,
            hog_stream_t stream) {
    return nms_impl(boxes, scores, scales, n, iou_threshold, keep, keep_count, scratch, sbytes,
                    stream, launch_nms, "hog_nms");
}

}  // extern "C"
