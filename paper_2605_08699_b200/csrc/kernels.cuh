// kernels.cuh -- launch interfaces of the render-path kernels (internal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace gsr {

// Per-kernel timing hook: launchers call mark("kernel") after every launch;
// a profiling context records a CUDA event there (gsr_ctx_set_kernel_timing).
struct KMark {
    void (*fn)(void *self, const char *kernel) = nullptr;
    void *self = nullptr;
    void operator()(const char *k) const {
        if (fn) fn(self, k);
    }
};

// Per-frame device counters (one struct, reset by frame_start_kernel).
struct FrameCounters {
    uint32_t K;                 // kept splats
    uint32_t D;                 // tile keys under the contract (may exceed capacity)
    uint32_t npass;             // depth-sort radix passes (32-bit key sort)
    uint32_t npass_fb;          // passes of the full 64-bit sort (frames re-rendered after long_runs)
    unsigned long long kmin;    // min / max kept depth key (f64 bits)
    unsigned long long kmax;
    unsigned long long P;       // (splat, tile row) pairs
    uint32_t nseg;              // binning segments
    uint32_t long_runs;         // depth sort: a 32-bit key run too long for the fix-up
    // work counters for the roofline (algorithmic units)
    unsigned long long E;       // blend: composited (pixel, splat) evaluations
    unsigned long long Rb;      // blend: (splat, pixel row) interval evaluations
    unsigned long long Rp;      // binning: (splat, pixel row) interval evaluations
    uint32_t blend_next;        // blend work queue: next (tile, pixel-row pair) item
    uint32_t rows_done;         // small-slice binning: tile rows whose lists are built
    uint32_t Drow;              // small-slice binning: list entries allocated (region cursor)
    uint32_t pad3;
    // blend instrumentation (counting variant only; gsr_debug_frame_counters)
    unsigned long long b_walked;   // list entries loaded by items (all items of all tiles)
    unsigned long long b_hit;      // ... of which the splat's row range meets the item's rows
    unsigned long long b_batches;  // 32-entry batches processed (warp level)
    unsigned long long b_iters;    // composite-loop iterations (warp level)
    unsigned long long b_lanes;    // sum over iterations of lanes with a splat to composite
    unsigned long long b_items;    // work items processed
    unsigned long long b_used;     // distinct splats whose colour the blend read
    // depth-sliced frames (slice.cu): per-pass item counts, slice threshold,
    // per-pass binning sizes summed / maximised over the passes
    uint32_t KA;                   // items of the first pass (the slice, or all K)
    uint32_t KB;                   // splats of the second pass
    uint32_t tau;                  // slice: span keys <= tau
    uint32_t n_unsat;              // work items slice A left unsaturated
    unsigned long long Dtot, Ptot; // tile keys / pairs over the passes
    unsigned long long Dmax, Pmax; // largest pass (buffer capacities)
    uint32_t slice_hist[1024];     // kept depths over kZBins bins of their f64 bits (preprocess_geo)
};

// The depth sort's 24-bit span key of a kept splat's f64 depth bits k64
// (depth.cu): k32 = min((k64 - kmin) >> shift, 2^24 - 1), shift chosen from
// [kmin, kmax] so the span fits 24 bits.  Monotone in k64.
constexpr int kSpanKeyBits = 24;
struct SpanMap {
    unsigned long long kmin, kcap;
    int shift;
};
__device__ __forceinline__ SpanMap span_map(unsigned long long kmin, unsigned long long kmax,
                                            int bits = kSpanKeyBits) {
    SpanMap m;
    const unsigned long long range = kmax > kmin ? kmax - kmin : 0ull;
    const int b = range ? 64 - __clzll((long long)range) : 0;
    m.kmin = kmin;
    m.shift = b > bits ? b - bits : 0;
    m.kcap = (1ull << bits) - 1ull;
    return m;
}
__device__ __forceinline__ uint32_t span_key(const SpanMap &m, unsigned long long k64) {
    const unsigned long long q = (k64 - m.kmin) >> m.shift;
    return (uint32_t)(q < m.kcap ? q : m.kcap);
}

// Scene in HBM, structure-of-arrays, each plane padded to `stride` elements.
struct SceneView {
    int64_t n;
    int64_t stride;
    const double *mean;   // [3][stride]
    const double *scale;  // [3][stride]
    const double *rot;    // [4][stride]  (w, x, y, z)
    const double *rsq;    // [stride]     render.py:476-481, f64
    const float *opac;    // [stride]     f32(opacity)
    const float *dc;      // [3][stride]  f32(colors_dc)
    const void *sh;       // [stride][48] f32 or f64: one 192 B (384 B) row per Gaussian,
                          // coefficient k*3 + c; rows so a gather by depth rank reads
                          // whole sectors (colour only for the splats a pass blends)
    const double *op64;   // [stride]     f64 opacity (rsq, read-back)
    const double *mean4;  // [stride][4]  (x, y, z, 0): the means again, one 32 B sector per
                          // Gaussian for the colour kernel's gather by depth rank (three
                          // planes would cost three 64 B DRAM accesses for 24 B)
    int sh_f32;
    int sh_row;           // floats per f32 SH row: 48, or 56 when the row carries the mean
                          // (f32 SH scenes: SH row + mean4 in one 224 B record, one gather)
    int m4_row;           // doubles between consecutive mean4 entries (4, or 28 inside the rows)
};

struct CameraArgs {
    double r[9];
    double t[3];
    double campos[3];
    double fx, fy, cx, cy;
    double width, height;
    int iwidth, iheight;
};

struct DepthOrder {  // depth rank -> Gaussian index (the depth sort's result buffer)
    const uint32_t *order0, *order1;
    const uint32_t *sched;  // sched[16]: which buffer holds the result
};

// Per-frame parameters in device memory (one block per context): the
// kernels read the camera, background and the mapped host frame from here,
// so a frame's launch sequence is the same for every pose and is replayed as
// a CUDA graph; load_frame_params (its only by-value use) stores them.
struct FrameParams {
    CameraArgs cam;
    float bg[3];
    uint8_t *host;  // device view of a mapped pinned (H,W,3) frame (zero copy), or null
};
// the frame's first kernel: FrameParams into device memory + counters reset
constexpr int kFrameStartThreads = 256;
void launch_frame_start(const FrameParams &p, FrameParams *dst, FrameCounters *ctr,
                        cudaStream_t s);
const void *frame_start_kernel_fn();  // its function (graph node updates)

// preprocess.cu (2 kernels)
using GeoRec = SplatRec;  // by Gaussian index (preprocess), by depth rank (gather)
// K1a: projection, culling, depth keys, packed geometry (render.py:163-290)
// zhist (depth-sliced frames, else null): += histogram of the kept depths
// over kZBins bins of their f64 bits (slice_plan's input)
// ibox (depth-sliced frames, else null): item_box of every kept splat
void launch_preprocess_geo(const SceneView &scene, const FrameParams *fp, int frustum_cull,
                           unsigned long long *keys, GeoRec *geo, uint8_t *keep_out,
                           FrameCounters *ctr, uint32_t *zhist, uint2 *ibox, cudaStream_t s,
                           const KMark &mark = KMark());

// A kept splat's conservative box in work-item units, for the slice-B
// filter: item rows [r0, r1] (pixel rows 2r, 2r + 1) from the reference's
// own row range (render.py:329-333, row_range), tile columns [c0, c1] from
// the whole splat's column extent (splat_x_extent; ill-conditioned: every
// column).  Packed (r0 | r1 << 16, c0 | c1 << 16); empty: r0 > r1.
__device__ __forceinline__ uint2 item_box(const GeoRec &g, int width, int height) {
    int lo, hi;
    row_range(g.a.y, g.b.w, height, lo, hi);
    if (lo >= hi || width <= 0) return make_uint2(0xffffu, 0u);
    int mn = 0, mx = width;
    float xl, xr;
    if (splat_x_extent(g.a.x, g.a.z, g.a.w, g.b.x, g.b.y, g.b.w, xl, xr)) {
        mn = max(__float2int_rd(xl), 0);
        mx = (int)fminf(ceilf(xr) + 1.0f, (float)width);
    }
    if (mn >= mx) return make_uint2(0xffffu, 0u);
    return make_uint2((uint32_t)(lo >> 1) | ((uint32_t)((hi - 1) >> 1) << 16),
                      (uint32_t)(mn / kTileW) | ((uint32_t)((mx - 1) / kTileW) << 16));
}
// depth histogram bins: bin = clamp((bits(z) >> 47) - kZBinBase, 0, 1023),
// 32 bins per binade (sign, 11 exponent and 5 mantissa bits) over z in
// [2^-8, 2^24)
constexpr int kZBins = 1024;
constexpr int kZBinShift = 47;
constexpr int kZBinBase = 1015 << 5;
// radix.cu: Onesweep stable LSD sort (see radix.cu header)
cudaError_t radix_init_attributes();
#ifndef GSR_RADIX_THREADS
#define GSR_RADIX_THREADS 512
#endif
constexpr int kRadixThreads = GSR_RADIX_THREADS;  // >= 256 (one thread per digit)
// items per thread (8: keeps <= 64 registers; 512 threads: 2 blocks / 32 warps per SM)
#ifndef GSR_RADIX_ITEMS
#define GSR_RADIX_ITEMS 8
#endif
constexpr int radix_items(int key_bytes) { return key_bytes == 8 ? 8 : GSR_RADIX_ITEMS; }
inline int64_t radix_tiles(int64_t n_cap, int key_bytes) {
    const int64_t tile = (int64_t)kRadixThreads * radix_items(key_bytes);
    return (n_cap + tile - 1) / tile;
}
// scratch for one sort (histograms, look-back status, tickets)
size_t sort_work_bytes(int64_t n_items_cap, int passes, int key_bytes);
// Optional key source of a 32-bit sort: the histogram kernel derives each key
// from a 64-bit one, k32 = min((k64 - kmin) >> shift, max_key) with shift
// chosen from [kmin, kmax] so the span fits `bits` bits (sentinel ~0 kept),
// and writes it to keys0 -- the depth sort's span keys (depth.cu).
struct SpanKeys {
    const unsigned long long *src = nullptr;
    const unsigned long long *kmin = nullptr, *kmax = nullptr;
    int bits = 24;
    const uint32_t *limit = nullptr;  // span keys above *limit become sentinels (slice A)
    uint32_t *count_out = nullptr;    // += keys the first pass keeps (slice A's KA; zeroed per frame)
    bool compact = false;             // append the kept (key, index) pairs to keys[0]/vals[0]
    int64_t n_src = 0;                // (compact) source keys read
    bool hist_zeroed = false;         // the digit histograms were zeroed by an earlier kernel
                                      // of the frame (no memset node before the sort)
};
// Sorts (keys0, vals0) over `passes` 8-bit digits; the result lands in buffer
// sched[16] (0 or 1).  First pass: n_first items (>= 0) or *n_dev (n_first <
// 0); later passes: min(*n_dev, n_cap).  implicit_first_vals: value = index;
// drop_sentinel: first pass removes keys == ~0.  Returns kernels launched.
template <typename K>
int launch_onesweep_sort(K *keys0, K *keys1, uint32_t *vals0, uint32_t *vals1,
                         bool implicit_first_vals, bool drop_sentinel, const uint32_t *n_dev,
                         int64_t n_first, int64_t n_cap, int passes, bool force_first,
                         void *work, uint32_t *sched, uint32_t *npass_out, int sms,
                         cudaStream_t s, const KMark &mark = KMark(),
                         const SpanKeys &span = SpanKeys());

// depth.cu: stable f64 depth order (see depth.cu header)
struct DepthArgs {
    unsigned long long *keys64[2];  // [0]: preprocess keys (sentinel ~0 = culled)
    uint32_t *keys32[2];
    uint32_t *vals[2];
    FrameCounters *ctr;
    int64_t n;
    void *work32, *work64;
    uint32_t *sched;    // sort schedule: sched[16] = buffer of vals holding the order
    bool full64;        // full 64-bit key sort (after a frame reported long runs)
    uint32_t *long_run_sticky;  // per-context count of frames that reported long runs
    uint32_t *count = nullptr;         // items after compaction (K, the slice's KA, or KB)
    const uint32_t *limit = nullptr;   // slice A: span keys <= *limit only
    bool keys_given = false;  // slice B: keys32[0] / vals[0] hold *count appended
                              // (span key, Gaussian index) pairs, at most `cap` of them
    int64_t cap = 0;
    bool hist_zeroed = false;  // 32-bit sorts: work32's histograms already zeroed (slice.cu)
};
constexpr int kDepthHistWords = 4 * 256;  // zeroed ahead of a 32-bit depth sort (<= 4 passes)
size_t depth_work32_bytes(int64_t n_cap);
size_t depth_work64_bytes(int64_t n_cap);
int launch_depth_sort(const DepthArgs &a, int sms, cudaStream_t s,
                      const KMark &mark = KMark());  // returns kernels launched

// binning.cu: sort-free tile lists (see binning.cu header)
constexpr int kMaxTileRows = 8192 / kTileH;   // height <= 8192
constexpr int kMaxTilesX = 16384 / kTileW;   // width <= 16384
struct BinArgs {
    const uint32_t *count;            // depth-ranked items of this pass
    const uint32_t *order0, *order1;  // depth sort result buffers
    const uint32_t *depth_sched;      // [16]: which of order0/order1 holds the result
    const GeoRec *geo;                // packed geometry by Gaussian index (preprocess)
    SplatRec *srec;                   // records by depth rank (written here)
    FrameCounters *ctr;
    int width, height, n_rows, tiles_x, ntiles;
    int64_t n_blocks;       // blocks of 512 depth ranks (capacity)
    int sms = 148;          // grid bound of the block-looping kernels
    uint32_t *row_blk;      // [n_rows][n_blocks] pair counts -> slots
    uint32_t *row_start;    // [n_rows + 1]
    unsigned long long *scan_work;  // [1 + scan tiles]: ticket, look-back status
    uint2 *pairs;           // [cap_p] (rank, tx0 | count << 16), grouped by tile row
    int64_t cap_p;
    int64_t cap_seg;
    uint32_t *seg_cnt;      // [cap_seg][tiles_x] keys per column -> offsets
    uint32_t *tile_total;   // [ntiles]
    uint32_t *row_total;    // [n_rows] list entries per tile row (seg_scan)
    uint2 *ranges;          // [ntiles] [start, end) into tile_vals
    uint32_t *tile_vals;    // [cap_d] depth ranks, tile-major
    int64_t cap_d;
    uint32_t *overflow_sticky;
};
int64_t bin_blocks(int64_t n_cap);
int64_t bin_scan_tiles(int64_t n_blocks, int n_rows);
int64_t bin_segments(int64_t cap_p, int n_rows);
cudaError_t binning_init_attributes();
// rows: the small-slice variant -- one CTA per tile row builds the row's
// lists (bin_rows_kernel) instead of the segment kernels; the list regions
// are allocated from FrameCounters.Drow / rows_done (zeroed per frame: one
// rows pass per frame)
int launch_binning(const BinArgs &a, cudaStream_t s, const KMark &mark = KMark(),
                   bool rows = false);  // returns kernels launched


// contract.cu: the exact tile-list contract on tile x tile tiles via
// (tile | rank) keys, a radix sort and range identification (parity path)
struct ContractArgs {
    const SplatRec *srec;            // depth-ranked records of the frame (bin_gather)
    const uint32_t *count;           // ranked items (K of a one-pass frame)
    int width, tile, tiles_x;
    unsigned long long *keys;        // [cap] (ty * tiles_x + tx) << 32 | rank
    int64_t cap;
    unsigned long long *d_count;     // keys reserved (may exceed cap)
};
int launch_contract_keys(const ContractArgs &a, int64_t cap_n, cudaStream_t s);
// ranges of the sorted keys (keys0 or keys1 by sched[16], the sort's result buffer)
int launch_contract_ranges(const unsigned long long *keys0, const unsigned long long *keys1,
                           const uint32_t *sched, const unsigned long long *d_count, int64_t cap,
                           uint2 *ranges, int ntiles, int sms, cudaStream_t s);

// preprocess.cu, K1b: SH colours (render.py:126-160) of the ranks [0, *count)
// of a pass's depth order, stored by rank: colr[r] = (r, g, b, 0)
void launch_color_ranked(const SceneView &scene, const FrameParams *fp, int sh_degree,
                         DepthOrder ord, const uint32_t *count, int64_t cap, float4 *colr,
                         cudaStream_t s, const KMark &mark = KMark());

// blend.cu
struct BlendOut {
    uint8_t *u8;    // (H,W,3)
    float *rgb;     // (H,W,3) or null
    float *trans;   // (H,W) or null
    const FrameParams *fp;  // background; fp->host: mapped pinned host frame (needs packed)
    bool packed;    // W % 32 == 0 and u8/host 4-byte aligned: one 96 B row segment per warp store
    uint32_t *used = nullptr;  // instrumentation (counting variant): per-rank "colour read" flags
    uint32_t *item_info = nullptr;  // ... per work item: last depth rank walked | saturated << 31
};
bool blend_has_slices();  // the selected blend variant has modes 1 and 2
int blend_grid(int width, int height);  // its persistent grid (host query, cached)
// mode: 0 one pass; 1 slice A (saturated items write the frame, the others
// save their pixels' state, set their bit in unsat_cols and are listed in
// unsat_items); 2 slice B (the listed items only, from the saved state)
struct SliceState {
    float4 *state = nullptr;        // (H, W) pixel (T, r, g, b) after slice A
    uint32_t *unsat_cols = nullptr; // [tiles_x][col_words]: bit r of tile column tx's bitmask =
                                    // the item (tx, item row r) is unsaturated
    int col_words = 0;              // words per tile column: (item rows + 31) / 32
    uint32_t *unsat_items = nullptr;  // [n_items] their ids; count in FrameCounters.n_unsat
};
// slice B empty: the listed unsaturated items' pixels from their saved state
void launch_finish_items(int width, int height, BlendOut out, const FrameCounters *ctr,
                         SliceState ss, int max_items, cudaStream_t s, const KMark &mark = KMark());
void launch_blend(const SplatRec *srec, const float4 *colr, const uint32_t *tile_vals,
                  const uint2 *ranges, int width, int height, BlendOut out, FrameCounters *ctr,
                  cudaStream_t s, const KMark &mark = KMark(), bool count = true, int mode = 0,
                  SliceState ss = SliceState());  // count: fill the E / Rb work counters

// slice.cu: depth-sliced frames
struct SliceBArgs {
    const unsigned long long *keys64;  // preprocess keys (sentinel ~0 = culled)
    const GeoRec *geo;                 // records by Gaussian index
    int64_t n;
    FrameCounters *ctr;                // kmin, kmax, tau; KB counted here
    const uint2 *ibox;                 // item_box of each kept splat (preprocess_geo)
    const uint32_t *unsat_cols;        // [tiles_x][col_words] items slice A left unsaturated
    int col_words;
    int width, height, tiles_x;
    uint32_t *keysB, *valsB;           // out: slice B's (span key, Gaussian index), appended
    uint32_t *zero = nullptr;          // cleared by block 0 (slice B's sort histograms)
    int zero_words = 0;
};
// slice-B size classes: the second slice's sort / colour / lists run with
// grids for at most slice_class_cap(c) splats (the last class: all)
#ifndef GSR_SLICE_CLASSES
#define GSR_SLICE_CLASSES 4
#endif
#ifndef GSR_SLICE_CAP2
#define GSR_SLICE_CAP2 262144
#endif
constexpr int kSliceClasses = GSR_SLICE_CLASSES;
__host__ __device__ constexpr int64_t slice_class_cap(int c) {
    return c == 0 ? 4096 : c == 1 ? 65536 : GSR_SLICE_CAP2;
}
void launch_slice_plan(FrameCounters *ctr, float frac, uint32_t *zero0, int n0, uint32_t *zero1,
                       int n1, cudaStream_t s, const KMark &mark = KMark());
void launch_slice_b_filter(const SliceBArgs &a, cudaStream_t s, const KMark &mark = KMark());
// sets `handle` (a graph's switch) to slice B's size class, kSliceClasses
// (no body) when slice B is empty
void launch_slice_b_decide(const FrameCounters *ctr, cudaGraphConditionalHandle handle,
                           uint32_t *class_count, cudaStream_t s);

// jpeg.cu: baseline JPEG of a device u8 frame (Pillow / libjpeg-turbo exact)
struct JpegLayout {
    int sub, mcux, mcuy, blocks_per_mcu;
    int cw[3], ch[3], wb[3], hb[3], mw[3];
    int64_t coef_off[3], n_real, n_scan;
    uint64_t max_bits;
    size_t words, stuff_threads;
    size_t off_coef, off_bits, off_words, off_aux, off_len, off_out;
};
size_t jpeg_workspace_bytes(int W, int H, int sub, JpegLayout *L);
void jpeg_quant_tables(int quality, uint16_t qt[2][64]);
void jpeg_huffman_spec(int t, int ac, const uint8_t **bits, const uint8_t **vals, int *nvals);
// encodes; host_len2 (pinned, 2 words) receives [bits, stuffed bytes]; stuffed
// scan bytes are at ws + L.off_out.  Synchronises the stream.
cudaError_t launch_jpeg(const uint8_t *rgb, int W, int H, int quality, const JpegLayout &L,
                        unsigned char *ws, uint32_t *host_len2, cudaStream_t s);

// resample.cu
struct ResampleAxis {
    const int32_t *bounds;   // (out, 2): xmin, xlen
    const int32_t *coefs;    // (out, ksize) fixed point, PRECISION_BITS = 22
    int ksize;
};
void launch_resample_h(const uint8_t *src, int sw, int row0, uint8_t *dst, int dw, int rows,
                       ResampleAxis ax, cudaStream_t s);
void launch_resample_v(const uint8_t *src, int w, uint8_t *dst, int dh, ResampleAxis ax,
                       cudaStream_t s);

// ssim.cu
// either two RGB u8 images (a, b) or two f64 luma planes (la, lb)
struct SsimInput {
    const uint8_t *a, *b;
    const double *la, *lb;
};
int ssim_partials_needed(int width, int height);
void launch_sse(const uint8_t *a, const uint8_t *b, int64_t n, unsigned long long *out,
                cudaStream_t s);
void launch_ssim(const SsimInput &in, int width, int height, const double *weights11,
                 double *partials, uint32_t *neq, double *out, cudaStream_t s);

}  // namespace gsr
