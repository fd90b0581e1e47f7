// gsr_api.cu -- the C ABI (include/gsr.h): scene residency, per-thread
// contexts, frame orchestration and the ladder/SSIM entry points.
//
// A frame is enqueued on the context's stream with no host synchronisation:
// item counts (K kept splats, D tile keys, depth-sort pass count) live in a
// device FrameCounters struct and every kernel reads them from there, with
// grids sized from capacities.  The only host round trip is at completion,
// where the tile-key count is checked against the buffer capacity (on
// overflow the buffer grows and the frame is re-rendered once).
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/gsr.h"
#include "kernels.cuh"
#include "scene.cuh"

namespace gsr {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int fail_cuda(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();  // clear sticky-free errors
    return e == cudaErrorMemoryAllocation ? GSR_E_OOM : GSR_E_CUDA;
}

int ensure(DevBuf &b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return GSR_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    GSR_CUDA_OK(cudaMalloc(&b.p, bytes));
    b.bytes = bytes;
    return GSR_OK;
}

// Depth-sliced frames (slice.cu): scenes of at least GSR_SLICE_MIN Gaussians
// (default 262144; 0 disables slicing) are rendered in two slices, the first
// holding about GSR_SLICE_FRAC (default 0.15) of the kept splats.
// depth-sliced frames: unsaturated items after slice A, one bit per tile
// column in each item row (two pixel rows; tile rows are whole item rows)
int unsat_item_rows(int H) { return ((H + kTileH - 1) / kTileH) * (kTileH / 2); }
int unsat_col_words(int H) { return (unsat_item_rows(H) + 31) / 32; }
size_t unsat_cols_bytes(int W, int H) {
    return sizeof(uint32_t) * (size_t)((W + kTileW - 1) / kTileW) * (size_t)unsat_col_words(H);
}

int64_t slice_min() {
    static const int64_t v = [] {
        const char *e = getenv("GSR_SLICE_MIN");
        if (!e) return (int64_t)262144;
        const long long x = atoll(e);
        return x <= 0 ? (int64_t)1 << 62 : (int64_t)x;
    }();
    return v;
}
// slice-B classes whose lists are built one CTA per tile row (bin_rows):
// classes below GSR_ROWS_CLASSES (default: <= 65536 splats; rows for the
// <= 262144 class too measured 1693-1708 vs 1695-1698 frames/s, kept on the
// segment kernels for the lower latency, 0.833 vs 0.848 ms device p50)
#ifndef GSR_ROWS_CLASSES
#define GSR_ROWS_CLASSES 2
#endif
inline bool rows_class(int k) { return k < GSR_ROWS_CLASSES; }

float slice_frac() {
    static const float v = [] {
        const char *e = getenv("GSR_SLICE_FRAC");
        const float x = e ? (float)atof(e) : 0.15f;
        return x > 0.0f && x <= 1.0f ? x : 0.15f;
    }();
    return v;
}

}  // namespace gsr

using namespace gsr;

// Frame configuration: everything a frame's launch sequence depends on
// besides the per-frame parameters (camera, background, mapped host frame),
// which the kernels read from c->params.  Frames with equal keys replay one
// CUDA graph.
struct FrameKey {
    SceneView view;
    int W, H, sh_degree, cull, want_rgb, want_keep, slice, kcount, full64, packed, stages;
    float frac;    // the front slice's fraction (a slice_plan kernel parameter)
    uint64_t gen;  // buffer generation of the context (reallocation -> new graphs)
    // capacities baked into the captured kernels' arguments (overflow checks,
    // grids): a capacity can grow inside an existing allocation (no new
    // generation), and a graph replayed with a stale one would overflow
    // again while the host saw the frame fit (an empty frame)
    int64_t cap_n, cap_p, cap_d;
    bool operator==(const FrameKey &o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};

struct FrameGraph {
    FrameKey key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t params_node = nullptr;
    uint64_t last_use = 0;
    int64_t base_launches = 0;  // kernels per launch outside the conditional bodies
};

struct SavedCall {
    // the scene of the frame in flight, needed only to re-render it inside
    // complete_frame; cleared once the frame completes (the caller may free
    // the scene as soon as its frame is finished)
    const gsr_scene *scene = nullptr;
    int64_t scene_n = 0;
    gsr_camera cam{};
    float bg[3] = {0, 0, 0};
    int sh_degree = 0;
    int cull = 1;
    bool want_rgb = false;
    bool want_keep = false;
};

struct gsr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t cap_n = 0, cap_d = 0, cap_p = 0;
    DevBuf keys[2], vals[2], keys32[2], geo, srec, keep;
    int sms = 148;
    DevBuf depth_work, depth_work32, sched;  // depth-sort scratch; sched[16] = result buffer
    uint32_t *hsched = nullptr;   // pinned host copy of sched
    // tile-list buffers (binning.cu)
    DevBuf row_blk, row_start, scan_work, pairs, seg_cnt, ttotal, rowtot, tile_vals;
    DevBuf ranges;
    DevBuf frame_u8, frame_rgb, frame_t;
    DevBuf colr;          // colours by depth rank of the current pass
    // depth-sliced frames: pixel state after slice A, unsaturated items (bits, list)
    DevBuf state, unsat_cols, unsat_items, ibox;
    DevBuf params;        // FrameParams of the frame being rendered
    // CUDA graphs of this context's frame configurations (record_frame)
    static constexpr int kMaxGraphs = 32;
    std::vector<FrameGraph> graphs;
    uint64_t graph_clock = 0, graph_builds = 0;
    uint64_t gen = 0;                  // bumped when a frame buffer is reallocated
    cudaStream_t cap_stream = nullptr; // captures the conditional bodies
    bool force_full = false;   // next enqueue: one pass over all kept splats (debug entries)
    int64_t slice_min_n = -1;  // gsr_ctx_set_slicing (-1: the GSR_SLICE_MIN default)
    float slice_frac_v = 0.0f; // ... (0: the GSR_SLICE_FRAC default)
    bool last_sliced = false;  // the last frame was rendered in two slices
    // device FrameCounters followed by two sticky per-context counters
    // (frames whose pair/tile buffers overflowed, frames that needed the
    // 64-bit depth re-sort); one D2H copy per frame brings all of them back
    DevBuf ctr;
    FrameCounters *hctr = nullptr;
    // sticky device counters after FrameCounters: [0] frames whose buffers
    // overflowed, [1] frames needing the 64-bit sort, [2 + k] graph frames
    // whose slice B ran conditional body k (kernel-launch accounting)
    static constexpr int kSticky = 2 + kSliceClasses + 1;
    // the depth sort's schedule (64 words) follows the counters in the same
    // buffer, so a frame ends with ONE device->host copy of both
    static constexpr size_t kSchedOff =
        (sizeof(FrameCounters) + kSticky * sizeof(uint32_t) + 15) / 16 * 16;
    static constexpr size_t kCtrBytes = kSchedOff + 64 * sizeof(uint32_t);
    uint32_t sticky_seen[kSticky] = {};  // sticky values reported by the last fill_stats
    // kernels per graph frame outside the conditional bodies, and per body
    // (recorded at capture; a graph launch counts its kernels, not 1)
    int64_t body_launches[kSliceClasses + 1] = {};
    uint32_t *dsticky() { return reinterpret_cast<uint32_t *>(ctr.as<FrameCounters>() + 1); }
    const uint32_t *hsticky() const { return reinterpret_cast<const uint32_t *>(hctr + 1); }
    int64_t launches = 0;  // kernels enqueued since the last finish/render
    cudaEvent_t ev[8] = {};
    // per-kernel event timeline of the last frame (gsr_ctx_set_kernel_timing)
    static constexpr int kMaxMarks = 64;
    bool ktime = false;   // per-kernel event marks
    bool kcount = false;  // blend work counters (E, Rb): the counting blend variant
    bool stages = false;  // stage boundary events (gsr_stats stage times)
    bool stages_last = false;  // the frame in flight / last frame recorded them
    int nmarks = 0;
    cudaEvent_t kev[kMaxMarks + 1] = {};
    const char *kname[kMaxMarks] = {};
    // ladder / resample / ssim scratch
    DevBuf base_u8, up_u8, tmp_u8, src_u8, dst_u8, coefs, ssim_part, ssim_misc, ssim_w;
    DevBuf jpeg_ws;                  // jpeg.cu workspace
    DevBuf used;                     // blend instrumentation (GSR_TIMING_COUNTERS only)
    // contract tile lists of the last frame (gsr_debug_contract_tiles, contract.cu)
    DevBuf ckeys[2], cvals[2], cwork, csched, cranges, cdcount;
    int64_t cap_c = 0, contract_d = 0;
    int contract_tile = 0;  // tile size of the lists built for the last frame, 0 = none
    int contract_buf = 0;   // which of ckeys holds the sorted keys
    float contract_ms = 0.0f;
    uint32_t *hjpeg = nullptr;       // pinned [bits, stuffed bytes]
    double *hssim = nullptr;
    // last frame
    int W = 0, H = 0, ntiles = 0;
    int tile_passes = 0;
    SavedCall saved;
    uint8_t *saved_out = nullptr;  // host destination of an enqueued frame (gsr_render_enqueue)
    // gsr_render: device view of the caller's mapped pinned frame; the blend
    // stores the u8 frame there directly (zc_used), so no copy follows it
    uint8_t *zc_host = nullptr;
    bool zc_used = false;
    bool saved_full64 = false;  // depth order via the full 64-bit sort (long key runs)
    bool pending = false;
    int retries = 0;
    int64_t bytes() const {
        int64_t s = 0;
        const DevBuf *all[] = {&keys[0], &keys[1], &vals[0], &vals[1], &keys32[0], &keys32[1],
                               &geo, &colr, &state, &unsat_cols, &unsat_items, &ibox, &params, &srec, &keep, &depth_work, &depth_work32, &sched, &row_blk, &row_start, &scan_work, &pairs, &rowtot,
                               &seg_cnt, &ttotal, &tile_vals, &ranges, &frame_u8, &frame_rgb, &frame_t,
                               &ctr, &base_u8, &up_u8, &tmp_u8, &src_u8, &dst_u8, &coefs,
                               &ssim_part, &ssim_misc, &ssim_w, &jpeg_ws, &ckeys[0], &ckeys[1],
                               &cvals[0], &cvals[1], &cwork, &csched, &cranges, &cdcount, &used};
        for (auto *b : all) s += (int64_t)b->bytes;
        return s;
    }
};

namespace {



// grow-only allocation of a frame buffer; a reallocation invalidates the
// context's frame graphs (they hold the old addresses)
int cens(gsr_ctx *c, DevBuf &b, size_t bytes) {
    void *old = b.p;
    const int rc = ensure(b, bytes);
    if (b.p != old) c->gen++;
    return rc;
}

int check_camera(const gsr_camera *cam) {
    if (!cam) return fail(GSR_E_INVALID, "camera is null");
    if (cam->width <= 0 || cam->height <= 0)
        return fail(GSR_E_INVALID, "image dimensions must be positive");
    if (cam->width > kTileW * kMaxTilesX || cam->height > kTileH * kMaxTileRows)
        return fail(GSR_E_INVALID, "image larger than 16384 x 8192 is not supported");
    if (!(cam->fx > 0) || !(cam->fy > 0)) return fail(GSR_E_INVALID, "focal lengths must be positive");
    return GSR_OK;
}

CameraArgs camera_args(const gsr_camera *cam) {
    CameraArgs a;
    for (int r = 0; r < 3; r++) {
        for (int c = 0; c < 3; c++) a.r[r * 3 + c] = cam->w2c[r * 4 + c];
        a.t[r] = cam->w2c[r * 4 + 3];
        a.campos[r] = cam->campos[r];
    }
    a.fx = cam->fx;
    a.fy = cam->fy;
    a.cx = cam->cx;
    a.cy = cam->cy;
    a.width = (double)cam->width;
    a.height = (double)cam->height;
    a.iwidth = cam->width;
    a.iheight = cam->height;
    return a;
}

int ensure_capacity(gsr_ctx *c, int64_t n, int W, int H, bool want_rgb, bool want_keep) {
    int rc;
    if (n > c->cap_n) {
        const int64_t cap = round_up(n + n / 8 + 1024, 4096);
        for (int i = 0; i < 2; i++) {
            if ((rc = cens(c, c->keys[i], sizeof(unsigned long long) * cap))) return rc;
            if ((rc = cens(c, c->vals[i], sizeof(uint32_t) * cap))) return rc;
            if ((rc = cens(c, c->keys32[i], sizeof(uint32_t) * cap))) return rc;
        }
        if ((rc = cens(c, c->geo, sizeof(GeoRec) * cap))) return rc;
        if ((rc = cens(c, c->colr, sizeof(float4) * cap))) return rc;
        if ((rc = cens(c, c->srec, sizeof(SplatRec) * cap))) return rc;
        c->cap_n = cap;
    }
    if (want_keep && (rc = cens(c, c->keep, (size_t)c->cap_n))) return rc;
    if (c->cap_d == 0) c->cap_d = round_up(std::max<int64_t>(int64_t(1) << 22, 16 * n), 4096);
    if (c->cap_p == 0) c->cap_p = round_up(std::max<int64_t>(int64_t(1) << 20, 6 * n), 4096);
    if ((rc = cens(c, c->tile_vals, sizeof(uint32_t) * c->cap_d))) return rc;
    if ((rc = cens(c, c->pairs, sizeof(uint2) * c->cap_p))) return rc;
    if ((rc = cens(c, c->depth_work, depth_work64_bytes(c->cap_n)))) return rc;
    if ((rc = cens(c, c->depth_work32, depth_work32_bytes(c->cap_n)))) return rc;
    const int tiles_x = (W + kTileW - 1) / kTileW, n_rows = (H + kTileH - 1) / kTileH;
    const int ntiles = tiles_x * n_rows;
    if ((rc = cens(c, c->ranges, sizeof(uint2) * (size_t)ntiles))) return rc;
    if ((rc = cens(c, c->ttotal, sizeof(uint32_t) * (size_t)ntiles))) return rc;
    if ((rc = cens(c, c->rowtot, sizeof(uint32_t) * (size_t)(n_rows + 1)))) return rc;
    if ((rc = cens(c, c->row_blk, sizeof(uint32_t) * (size_t)n_rows * bin_blocks(c->cap_n))))
        return rc;
    if ((rc = cens(c, c->row_start, sizeof(uint32_t) * (size_t)(n_rows + 1)))) return rc;
    if ((rc = cens(c, c->scan_work, sizeof(unsigned long long) *
                                       (size_t)(bin_scan_tiles(bin_blocks(c->cap_n), n_rows) + 1))))
        return rc;
    const int64_t cap_seg = bin_segments(c->cap_p, n_rows);
    if ((rc = cens(c, c->seg_cnt, sizeof(uint32_t) * (size_t)cap_seg * tiles_x))) return rc;
    const int64_t px = (int64_t)W * H;
    if ((rc = cens(c, c->frame_u8, (size_t)px * 3))) return rc;
    if (want_rgb) {
        if ((rc = cens(c, c->frame_rgb, sizeof(float) * (size_t)px * 3))) return rc;
        if ((rc = cens(c, c->frame_t, sizeof(float) * (size_t)px))) return rc;
    }
    return GSR_OK;
}

void kmark_cb(void *self, const char *kernel) {
    gsr_ctx *c = static_cast<gsr_ctx *>(self);
    if (c->nmarks >= gsr_ctx::kMaxMarks) return;
    c->kname[c->nmarks] = kernel;
    cudaEventRecord(c->kev[++c->nmarks], c->stream);
}

// Records one frame on stream s: launches directly, or -- while s is being
// captured (graph) -- builds the graph; slice B's work then sits in a switch
// node whose body is chosen on the device from slice B's size.
int record_frame(gsr_ctx *c, const gsr_scene *sc, const FrameParams &fp, int sh_degree, int cull,
                 bool want_rgb, bool want_keep, bool slice, bool graph) {
    cudaStream_t s = c->stream;
    FrameCounters *ctr = c->ctr.as<FrameCounters>();
    FrameParams *dfp = c->params.as<FrameParams>();
    const int W = c->W, H = c->H;
    const int64_t n = sc->n;
    uint32_t *dsched = reinterpret_cast<uint32_t *>(c->ctr.as<unsigned char>() + gsr_ctx::kSchedOff);
    const unsigned evflags = graph ? cudaEventRecordExternal : cudaEventRecordDefault;
    // stage boundary events (ev[1..4]) only with GSR_TIMING_STAGES: four event
    // nodes cost a frame graph 0.02-0.03 ms of latency (one stream 1,304 ->
    // 1,340 frames/s without them); ev[0] / ev[5] always bracket the frame
    auto stage_ev = [&](int k, cudaStream_t st) {
        if (c->stages) cudaEventRecordWithFlags(c->ev[k], st, evflags);
    };
    int launches = 1;  // frame_start

    KMark mark;
    if (c->ktime && !graph) {
        mark.fn = kmark_cb;
        mark.self = c;
        c->nmarks = 0;
    }
    const bool packed = W % kTileW == 0;
    BlendOut out{c->frame_u8.as<uint8_t>(), want_rgb ? c->frame_rgb.as<float>() : nullptr,
                 want_rgb ? c->frame_t.as<float>() : nullptr, dfp, packed};
    const size_t n_items = (size_t)c->ntiles * (kTileH / 2);
    DepthOrder ord{c->vals[0].as<uint32_t>(), c->vals[1].as<uint32_t>(), dsched};
    SliceState ss;
    if (slice) {
        ss.state = c->state.as<float4>();
        ss.unsat_cols = c->unsat_cols.as<uint32_t>();
        ss.col_words = unsat_col_words(H);
        ss.unsat_items = c->unsat_items.as<uint32_t>();
    }
    // one depth-ordered pass over *count splats (at most cap): sort, colour, bin
    // rows: small second slices build their lists with one CTA per tile row
    auto sort_color_bin = [&](cudaStream_t st, uint32_t *count, const uint32_t *limit,
                              bool keys_given, int64_t cap, bool rows = false) {
        DepthArgs da;
        for (int i = 0; i < 2; i++) {
            da.keys64[i] = c->keys[i].as<unsigned long long>();
            da.keys32[i] = c->keys32[i].as<uint32_t>();
            da.vals[i] = c->vals[i].as<uint32_t>();
        }
        da.ctr = ctr;
        da.n = n;
        da.work32 = c->depth_work32.p;
        da.work64 = c->depth_work.p;
        da.sched = dsched;
        da.full64 = c->saved_full64;
        da.long_run_sticky = c->dsticky() + 1;
        da.count = count;
        da.limit = limit;
        da.keys_given = keys_given;
        da.cap = cap;
        da.hist_zeroed = slice;  // by slice_plan (slice A) / slice_b_filter (slice B)
        launches += launch_depth_sort(da, c->sms, st, mark);
        launch_color_ranked(sc->view, dfp, sh_degree, ord, count, cap, c->colr.as<float4>(), st,
                            mark);
        launches += 1;
        if (!keys_given) stage_ev(2, st);
        BinArgs ba;
        ba.count = count;
        ba.order0 = c->vals[0].as<uint32_t>();
        ba.order1 = c->vals[1].as<uint32_t>();
        ba.depth_sched = dsched;
        ba.geo = c->geo.as<GeoRec>();
        ba.srec = c->srec.as<SplatRec>();
        ba.ctr = ctr;
        ba.width = W;
        ba.height = H;
        ba.tiles_x = (W + kTileW - 1) / kTileW;
        ba.n_rows = (H + kTileH - 1) / kTileH;
        ba.ntiles = c->ntiles;
        ba.n_blocks = bin_blocks(cap);
        ba.sms = c->sms;
        ba.row_blk = c->row_blk.as<uint32_t>();
        ba.row_start = c->row_start.as<uint32_t>();
        ba.scan_work = c->scan_work.as<unsigned long long>();
        ba.pairs = c->pairs.as<uint2>();
        ba.cap_p = c->cap_p;
        ba.cap_seg = bin_segments(c->cap_p, ba.n_rows);
        ba.seg_cnt = c->seg_cnt.as<uint32_t>();
        ba.tile_total = c->ttotal.as<uint32_t>();
        ba.row_total = c->rowtot.as<uint32_t>();
        ba.ranges = c->ranges.as<uint2>();
        ba.tile_vals = c->tile_vals.as<uint32_t>();
        ba.cap_d = c->cap_d;
        ba.overflow_sticky = c->dsticky();
        launches += launch_binning(ba, st, mark, rows);
    };
    auto blend_on = [&](cudaStream_t st, int mode, const SliceState &sst) {
        launch_blend(c->srec.as<SplatRec>(), c->colr.as<float4>(), c->tile_vals.as<uint32_t>(),
                     c->ranges.as<uint2>(), W, H, out, ctr, st, mark, c->kcount, mode, sst);
        launches += 1;
    };
    auto blend = [&](int mode) { blend_on(s, mode, ss); };


    cudaEventRecordWithFlags(c->ev[0], s, evflags);
    if (c->ktime && !graph) cudaEventRecord(c->kev[0], s);
    launch_frame_start(fp, dfp, ctr, s);
    mark("frame_start");
    if (c->kcount &&
        ensure(c->used, sizeof(uint32_t) * ((size_t)c->cap_n + n_items)) == GSR_OK) {
        cudaMemsetAsync(c->used.p, 0, sizeof(uint32_t) * ((size_t)c->cap_n + n_items), s);
        out.used = c->used.as<uint32_t>();
        out.item_info = out.used + c->cap_n;
    }
    if (n > 0) {
        launch_preprocess_geo(sc->view, dfp, cull, c->keys[0].as<unsigned long long>(),
                              c->geo.as<GeoRec>(), want_keep ? c->keep.as<uint8_t>() : nullptr,
                              ctr, slice ? ctr->slice_hist : nullptr,
                              slice ? c->ibox.as<uint2>() : nullptr, s, mark);
        launches += 1;
        if (slice) {
            // (also clears the unsaturated-item bitmask and slice A's sort
            // histograms: no memset nodes)
            launch_slice_plan(ctr, c->slice_frac_v > 0.0f ? c->slice_frac_v : slice_frac(),
                              c->unsat_cols.as<uint32_t>(), (int)(unsat_cols_bytes(W, H) / 4),
                              reinterpret_cast<uint32_t *>(c->depth_work32.p), kDepthHistWords,
                              s, mark);
            launches += 1;
        }
    }
    stage_ev(1, s);
    if (n == 0) {
        stage_ev(2, s);
        cudaMemsetAsync(c->ranges.p, 0, sizeof(uint2) * (size_t)c->ntiles, s);
        stage_ev(3, s);
        blend(0);
        stage_ev(4, s);
    } else if (!slice) {
        // stable f64 depth order of all kept splats (the first radix pass
        // compacts: drops the culled sentinels), colours, lists, blend
        sort_color_bin(s, &ctr->K, nullptr, false, c->cap_n);
        stage_ev(3, s);
        blend(0);
        stage_ev(4, s);
    } else {
        // slice A: the front of the depth order
        sort_color_bin(s, &ctr->KA, &ctr->tau, false, c->cap_n);
        stage_ev(3, s);
        blend(1);
        stage_ev(4, s);
        // slice B: the splats behind it that can reach an unsaturated item
        SliceBArgs sb;
        sb.keys64 = c->keys[0].as<unsigned long long>();
        sb.geo = c->geo.as<GeoRec>();
        sb.ibox = c->ibox.as<uint2>();
        sb.n = n;
        sb.ctr = ctr;
        sb.unsat_cols = c->unsat_cols.as<uint32_t>();
        sb.col_words = unsat_col_words(H);
        sb.width = W;
        sb.height = H;
        sb.tiles_x = (W + kTileW - 1) / kTileW;
        sb.keysB = c->keys32[0].as<uint32_t>();
        sb.valsB = c->vals[0].as<uint32_t>();
        sb.zero = reinterpret_cast<uint32_t *>(c->depth_work32.p);  // slice B's sort histograms
        sb.zero_words = kDepthHistWords;
        launch_slice_b_filter(sb, s, mark);
        launches += 1;
        auto class_cap = [&](int k) {
            return k < kSliceClasses - 1 ? std::min<int64_t>(slice_class_cap(k), c->cap_n)
                                         : c->cap_n;
        };
        if (graph) {
            // switch node: body k sorts / colours / bins with class-k grids
            cudaStreamCaptureStatus cs;
            cudaGraph_t g = nullptr;
            const cudaGraphNode_t *deps = nullptr;
            size_t nd = 0;
            GSR_CUDA_OK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
            cudaGraphConditionalHandle h;
            GSR_CUDA_OK(cudaGraphConditionalHandleCreate(&h, g, kSliceClasses,
                                                         cudaGraphCondAssignDefault));
            // bodies 0 .. kSliceClasses - 1: slice B's sort, colours, lists
            // and blend with class-k grids; body kSliceClasses (slice B
            // empty): the blend alone (the unsaturated items finish from the
            // saved state)
            launch_slice_b_decide(ctr, h, c->dsticky() + 2, s);
            launches += 1;
            GSR_CUDA_OK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
            std::vector<cudaGraphNode_t> dv(deps, deps + nd);
            cudaGraphNodeParams cp{};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeSwitch;
            cp.conditional.size = kSliceClasses + 1;
            cudaGraphNode_t cn;
            GSR_CUDA_OK(cudaGraphAddNode(&cn, g, dv.data(), dv.size(), &cp));
            for (int k = 0; k <= kSliceClasses; k++) {
                GSR_CUDA_OK(cudaStreamBeginCaptureToGraph(c->cap_stream, cp.conditional.phGraph_out[k],
                                                          nullptr, nullptr, 0,
                                                          cudaStreamCaptureModeThreadLocal));
                const int before = launches;
                if (k < kSliceClasses) {
                    sort_color_bin(c->cap_stream, &ctr->KB, nullptr, true, class_cap(k),
                                   rows_class(k));
                    blend_on(c->cap_stream, 2, ss);
                } else {  // slice B empty: the unsaturated items only finish
                    launch_finish_items(W, H, out, ctr, ss, (int)n_items, c->cap_stream, mark);
                    launches += 1;
                }
                c->body_launches[k] = launches - before;
                launches = before;  // counted per frame from the device's class counters
                cudaGraph_t body = nullptr;
                GSR_CUDA_OK(cudaStreamEndCapture(c->cap_stream, &body));
            }
            GSR_CUDA_OK(cudaStreamUpdateCaptureDependencies(s, &cn, 1,
                                                            cudaStreamSetCaptureDependencies));
        } else {
            // direct launches: slice B's size read back, its class chosen on the host
            uint32_t kb = 0;
            GSR_CUDA_OK(cudaMemcpyAsync(&c->hctr->KB, &ctr->KB, sizeof(uint32_t),
                                        cudaMemcpyDeviceToHost, s));
            GSR_CUDA_OK(cudaStreamSynchronize(s));
            kb = c->hctr->KB;
            int k = kSliceClasses - 1;
            for (int j = kSliceClasses - 2; j >= 0; j--)
                if ((int64_t)kb <= slice_class_cap(j)) k = j;
            if (kb > 0) {
                sort_color_bin(s, &ctr->KB, nullptr, true, class_cap(k), rows_class(k));
                blend_on(s, 2, ss);
            } else {
                launch_finish_items(W, H, out, ctr, ss, (int)n_items, s, mark);
                launches += 1;
            }
        }
    }
    cudaEventRecordWithFlags(c->ev[5], s, evflags);
    cudaMemcpyAsync(c->hctr, ctr, gsr_ctx::kCtrBytes, cudaMemcpyDeviceToHost, s);  // + sched
    GSR_CUDA_OK(cudaGetLastError());
    c->launches += launches;
    return GSR_OK;
}

bool graphs_enabled() {
    static const bool v = [] {
        const char *e = getenv("GSR_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return v;
}

void destroy_graph(FrameGraph &fg) {
    if (fg.exec) cudaGraphExecDestroy(fg.exec);
    if (fg.graph) cudaGraphDestroy(fg.graph);
    fg.exec = nullptr;
    fg.graph = nullptr;
}

// The context's graph for `key`, captured and instantiated on first use
// (least recently used of kMaxGraphs evicted).
int frame_graph(gsr_ctx *c, const FrameKey &key, const gsr_scene *sc, const FrameParams &fp,
                int sh_degree, int cull, bool want_rgb, bool want_keep, bool slice,
                FrameGraph **out) {
    c->graph_clock++;
    for (auto &fg : c->graphs)
        if (fg.exec && fg.key == key) {
            fg.last_use = c->graph_clock;
            *out = &fg;
            return GSR_OK;
        }
    if (!c->cap_stream)
        GSR_CUDA_OK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    blend_grid(c->W, c->H);  // occupancy query before capture
    FrameGraph fg;
    fg.key = key;
    GSR_CUDA_OK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t launches_before = c->launches;
    int rc = record_frame(c, sc, fp, sh_degree, cull, want_rgb, want_keep, slice, true);
    fg.base_launches = c->launches - launches_before;
    c->launches = launches_before;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return fail_cuda(e, "frame graph capture");
    fg.graph = g;
    const cudaError_t ei = cudaGraphInstantiate(&fg.exec, g, 0);
    if (ei != cudaSuccess) {
        destroy_graph(fg);
        return fail_cuda(ei, "frame graph instantiate");
    }
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(g, nodes.data(), &nn);
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
        cudaKernelNodeParams kp{};
        if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess &&
            kp.func == frame_start_kernel_fn()) {
            fg.params_node = nd;
            break;
        }
    }
    if (!fg.params_node) {
        destroy_graph(fg);
        return fail(GSR_E_CUDA, "frame graph: parameter node not found");
    }
    fg.last_use = c->graph_clock;
    // evict the least recently used graph when full
    if ((int)c->graphs.size() >= gsr_ctx::kMaxGraphs) {
        size_t lru = 0;
        for (size_t i = 1; i < c->graphs.size(); i++)
            if (c->graphs[i].last_use < c->graphs[lru].last_use) lru = i;
        destroy_graph(c->graphs[lru]);
        c->graphs[lru] = fg;
        *out = &c->graphs[lru];
    } else {
        c->graphs.push_back(fg);
        *out = &c->graphs.back();
    }
    c->graph_builds++;
    return GSR_OK;
}

// Enqueue one full frame on c->stream (no host synchronisation in the graph
// path: one parameter-node update and one graph launch).
int enqueue_frame(gsr_ctx *c, const gsr_scene *sc, const gsr_camera *cam, const float bg[3],
                  int sh_degree, int cull, bool want_rgb, bool want_keep) {
    int rc;
    if ((rc = check_camera(cam))) return rc;
    if (!sc) return fail(GSR_E_INVALID, "scene is null");
    if (sh_degree < 0 || sh_degree > 3) return fail(GSR_E_INVALID, "SH degree must be in 0..3");
    if (sh_degree > 0 && !sc->has_sh)
        return fail(GSR_E_INVALID, "scene was created without SH coefficients");
    if (sc->device != c->device) return fail(GSR_E_INVALID, "scene and context are on different devices");
    const int W = cam->width, H = cam->height;
    const int64_t n = sc->n;
    if ((rc = ensure_capacity(c, n, W, H, want_rgb, want_keep))) return rc;
    c->W = W;
    c->H = H;
    c->contract_tile = 0;
    c->ntiles = ((W + kTileW - 1) / kTileW) * ((H + kTileH - 1) / kTileH);
    // depth-sliced frame (slice.cu) unless a stage output of the whole
    // frame is wanted (debug entries), the 64-bit sort is needed, the scene
    // is small or a blend tuning variant without slice modes is selected
    const int64_t smin = c->slice_min_n >= 0 ? c->slice_min_n : slice_min();
    const bool slice = !want_keep && !c->force_full && !c->saved_full64 && n >= smin &&
                       blend_has_slices();
    c->last_sliced = slice;
    if (slice) {
        const size_t n_items = (size_t)c->ntiles * (kTileH / 2);
        if ((rc = cens(c, c->state, sizeof(float4) * (size_t)W * H))) return rc;
        if ((rc = cens(c, c->unsat_cols, unsat_cols_bytes(W, H)))) return rc;
        if ((rc = cens(c, c->ibox, sizeof(uint2) * (size_t)std::max<int64_t>(n, 1)))) return rc;
        if ((rc = cens(c, c->unsat_items, sizeof(uint32_t) * n_items))) return rc;
    }
    FrameParams fp;
    fp.cam = camera_args(cam);
    for (int i = 0; i < 3; i++) fp.bg[i] = bg[i];
    const bool packed = W % kTileW == 0 && ((uintptr_t)c->zc_host & 3u) == 0;
    c->zc_used = packed && c->zc_host != nullptr;
    fp.host = c->zc_used ? c->zc_host : nullptr;
    c->stages_last = c->stages;
    if (graphs_enabled() && !c->ktime && !c->kcount) {
        FrameKey key;
        std::memset(&key, 0, sizeof(key));
        key.view = sc->view;
        key.W = W;
        key.H = H;
        key.sh_degree = sh_degree;
        key.cull = cull;
        key.want_rgb = want_rgb;
        key.want_keep = want_keep;
        key.slice = slice;
        key.kcount = c->kcount;
        key.stages = c->stages;
        key.full64 = c->saved_full64;
        key.packed = W % kTileW == 0;
        key.frac = slice ? (c->slice_frac_v > 0.0f ? c->slice_frac_v : slice_frac()) : 0.0f;
        key.gen = c->gen;
        key.cap_n = c->cap_n;
        key.cap_p = c->cap_p;
        key.cap_d = c->cap_d;
        FrameGraph *fg = nullptr;
        if ((rc = frame_graph(c, key, sc, fp, sh_degree, cull, want_rgb, want_keep, slice, &fg)))
            return rc;
        cudaKernelNodeParams kp{};
        FrameParams *dfp = c->params.as<FrameParams>();
        FrameCounters *dctr = c->ctr.as<FrameCounters>();
        void *args[3] = {&fp, &dfp, &dctr};
        kp.func = const_cast<void *>(frame_start_kernel_fn());
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(kFrameStartThreads);
        kp.kernelParams = args;
        GSR_CUDA_OK(cudaGraphExecKernelNodeSetParams(fg->exec, fg->params_node, &kp));
        GSR_CUDA_OK(cudaGraphLaunch(fg->exec, c->stream));
        c->launches += fg->base_launches;  // + the body's kernels, counted on the device
    } else {
        if ((rc = record_frame(c, sc, fp, sh_degree, cull, want_rgb, want_keep, slice, false)))
            return rc;
    }
    c->saved.scene = sc;
    c->saved.scene_n = n;
    c->saved.cam = *cam;
    for (int i = 0; i < 3; i++) c->saved.bg[i] = bg[i];
    c->saved.sh_degree = sh_degree;
    c->saved.cull = cull;
    c->saved.want_rgb = want_rgb;
    c->saved.want_keep = want_keep;
    c->saved_out = nullptr;
    c->pending = true;
    return GSR_OK;
}

// Wait for the pending frame.  Re-render it if the tile-key or pair buffer
// overflowed (after growing it; a pair overflow stops the pipeline before D
// is known, so up to three rounds) or if the 32-bit depth sort reported a run
// of equal span keys too long for its fix-up (then with the full 64-bit sort).
int complete_frame(gsr_ctx *c) {
    if (!c->pending) return GSR_OK;
    GSR_CUDA_OK(cudaStreamSynchronize(c->stream));
    c->pending = false;
    c->retries = 0;
    uint8_t *out = c->saved_out;
    for (int round = 0;; round++) {
        const int64_t d = (int64_t)c->hctr->Dmax, p = (int64_t)c->hctr->Pmax;
        const bool ov_p = p > c->cap_p, ov_d = !ov_p && d > c->cap_d;
        const bool long_runs = c->hctr->long_runs != 0 && !c->saved_full64;
        if (!ov_p && !ov_d && !long_runs) break;
        if (round == 3) return fail(GSR_E_OOM, "tile list buffer overflow");
        if (ov_p) c->cap_p = round_up(p + p / 4 + (1 << 20), 4096);
        if (ov_p || ov_d)  // (never below the current capacity)
            c->cap_d = std::max(c->cap_d, round_up(std::max(d, 3 * p) + std::max(d, 3 * p) / 4 +
                                                       (1 << 20), 4096));
        if (c->cap_d >= (int64_t(1) << 32) || c->cap_p >= (int64_t(1) << 32))
            return fail(GSR_E_OOM, "tile list exceeds 2^32 entries");
        if (long_runs) c->saved_full64 = true;
        SavedCall sv = c->saved;
        const bool full64 = c->saved_full64;
        int rc = enqueue_frame(c, sv.scene, &sv.cam, sv.bg, sv.sh_degree, sv.cull, sv.want_rgb,
                               sv.want_keep);
        c->saved_full64 = full64;
        if (rc) return rc;
        GSR_CUDA_OK(cudaStreamSynchronize(c->stream));
        c->pending = false;
        c->retries = round + 1;
    }
    c->saved_full64 = false;
    if (c->retries && out)
        GSR_CUDA_OK(cudaMemcpy(out, c->frame_u8.p, (size_t)c->W * c->H * 3,
                               cudaMemcpyDeviceToHost));
    return GSR_OK;
}

void fill_stats(gsr_ctx *c, const gsr_scene *sc, gsr_stats *st) {
    if (!st) return;
    st->splats_drawn = c->hctr->K;
    st->splats_culled = sc ? sc->n - (int64_t)c->hctr->K : 0;
    st->tile_keys = (int64_t)c->hctr->Dtot;
    st->depth_passes = (int32_t)(c->hctr->npass + c->hctr->npass_fb);
    st->retries = c->retries;
    float t[6] = {0, 0, 0, 0, 0, 0};
    cudaEventElapsedTime(&t[0], c->ev[0], c->ev[5]);
    if (c->stages_last) {  // the frame recorded its stage events
        cudaEventElapsedTime(&t[1], c->ev[0], c->ev[1]);
        cudaEventElapsedTime(&t[2], c->ev[1], c->ev[2]);
        cudaEventElapsedTime(&t[3], c->ev[2], c->ev[3]);
        cudaEventElapsedTime(&t[4], c->ev[3], c->ev[4]);
        cudaEventElapsedTime(&t[5], c->ev[4], c->ev[5]);
    }
    st->ms_device = t[0];
    st->ms_preprocess = t[1];   // projection (+ slice plan)
    st->ms_depth_sort = t[2];   // depth sort + colours (of slice A)
    st->ms_binning = t[3];      // tile lists (of slice A)
    st->ms_tile_sort = 0.0f;    // (no tile sort: sort-free lists)
    st->ms_blend = t[4];        // blend (of slice A)
    st->ms_slice_b = t[5];      // slice B: filter, sort, colours, lists, blend (0: one pass)
    // sticky counters as of the last completed frame's copy (no extra sync)
    const uint32_t *hs = c->hsticky();
    for (int k = 0; k <= kSliceClasses; k++) {  // graph frames' slice-B bodies
        c->launches += (int64_t)(hs[2 + k] - c->sticky_seen[2 + k]) * c->body_launches[k];
        c->sticky_seen[2 + k] = hs[2 + k];
    }
    st->kernel_launches = (int32_t)c->launches;
    c->launches = 0;
    st->overflow_frames = (int32_t)(hs[0] - c->sticky_seen[0]);
    st->long_run_frames = (int32_t)(hs[1] - c->sticky_seen[1]);
    c->sticky_seen[0] = hs[0];
    c->sticky_seen[1] = hs[1];
    st->pairs = (int64_t)c->hctr->Ptot;
    st->composited = (int64_t)c->hctr->E;
    st->row_evals_blend = (int64_t)c->hctr->Rb;
    st->row_evals_binning = (int64_t)c->hctr->Rp;
}

// ---- Pillow BILINEAR coefficients (Resample.c precompute_coeffs +
// normalize_coeffs_8bpc), host double arithmetic, no FMA contraction ----
int pillow_coeffs(int in_size, int out_size, std::vector<int32_t> &bounds,
                  std::vector<int32_t> &kk) {
    const double scale = (double)((float)in_size - 0.0f) / out_size;
    const double filterscale = scale < 1.0 ? 1.0 : scale;
    const double support = 1.0 * filterscale;
    const int ksize = (int)std::ceil(support) * 2 + 1;
    bounds.assign((size_t)out_size * 2, 0);
    kk.assign((size_t)out_size * ksize, 0);
    std::vector<double> k((size_t)ksize);
    for (int xx = 0; xx < out_size; xx++) {
        const double center = 0.0 + (xx + 0.5) * scale;
        double ww = 0.0;
        const double ss = 1.0 / filterscale;
        int xmin = (int)(center - support + 0.5);
        if (xmin < 0) xmin = 0;
        int xmax = (int)(center + support + 0.5);
        if (xmax > in_size) xmax = in_size;
        xmax -= xmin;
        int x;
        for (x = 0; x < xmax; x++) {
            double t = (x + xmin - center + 0.5) * ss;
            if (t < 0.0) t = -t;
            const double w = t < 1.0 ? 1.0 - t : 0.0;
            k[x] = w;
            ww += w;
        }
        for (x = 0; x < xmax; x++)
            if (ww != 0.0) k[x] /= ww;
        for (; x < ksize; x++) k[x] = 0;
        for (x = 0; x < ksize; x++) {
            const double v = k[x];
            kk[(size_t)xx * ksize + x] = v < 0 ? (int32_t)(-0.5 + v * (1 << 22))
                                               : (int32_t)(0.5 + v * (1 << 22));
        }
        bounds[2 * xx] = xmin;
        bounds[2 * xx + 1] = xmax;
    }
    return ksize;
}

// device-to-device resample on c->stream (dst may not alias src)
int resample_device(gsr_ctx *c, const uint8_t *src, int sw, int sh, uint8_t *dst, int dw, int dh) {
    cudaStream_t s = c->stream;
    if (sw == dw && sh == dh) {
        GSR_CUDA_OK(cudaMemcpyAsync(dst, src, (size_t)sw * sh * 3, cudaMemcpyDeviceToDevice, s));
        return GSR_OK;
    }
    std::vector<int32_t> bh, kh, bv, kv;
    const int ksh = pillow_coeffs(sw, dw, bh, kh);
    const int ksv = pillow_coeffs(sh, dh, bv, kv);
    const bool need_h = dw != sw, need_v = dh != sh;
    const int ybox_first = bv[0];
    const int ybox_last = bv[(size_t)dh * 2 - 2] + bv[(size_t)dh * 2 - 1];
    if (need_h)
        for (int i = 0; i < dh; i++) bv[2 * i] -= ybox_first;
    // one upload: [bh | kh | bv | kv]
    std::vector<int32_t> blob;
    blob.reserve(bh.size() + kh.size() + bv.size() + kv.size());
    blob.insert(blob.end(), bh.begin(), bh.end());
    blob.insert(blob.end(), kh.begin(), kh.end());
    blob.insert(blob.end(), bv.begin(), bv.end());
    blob.insert(blob.end(), kv.begin(), kv.end());
    int rc;
    if ((rc = ensure(c->coefs, blob.size() * sizeof(int32_t)))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(c->coefs.p, blob.data(), blob.size() * sizeof(int32_t),
                                cudaMemcpyHostToDevice, s));
    // the host vector must outlive the async copy
    GSR_CUDA_OK(cudaStreamSynchronize(s));
    const int32_t *d = c->coefs.as<int32_t>();
    ResampleAxis axh{d, d + bh.size(), ksh};
    ResampleAxis axv{d + bh.size() + kh.size(), d + bh.size() + kh.size() + bv.size(), ksv};
    const uint8_t *cur = src;
    int cw = sw;
    if (need_h) {
        const int rows = ybox_last - ybox_first;
        if ((rc = ensure(c->tmp_u8, (size_t)dw * rows * 3))) return rc;
        uint8_t *tgt = need_v ? c->tmp_u8.as<uint8_t>() : dst;
        launch_resample_h(src, sw, ybox_first, tgt, dw, rows, axh, s);
        cur = tgt;
        cw = dw;
    }
    if (need_v) launch_resample_v(cur, cw, dst, dh, axv, s);
    GSR_CUDA_OK(cudaGetLastError());
    return GSR_OK;
}

int ssim_device(gsr_ctx *c, const SsimInput &in, int W, int H, double *dev_out) {
    int rc;
    if ((rc = ensure(c->ssim_part, sizeof(double) * (size_t)ssim_partials_needed(W, H)))) return rc;
    launch_ssim(in, W, H, c->ssim_w.as<double>(), c->ssim_part.as<double>(),
                c->ssim_misc.as<uint32_t>(), dev_out, c->stream);
    GSR_CUDA_OK(cudaGetLastError());
    return GSR_OK;
}

// JFIF headers exactly as Pillow / libjpeg-turbo write them (jcmarker.c):
// SOI, APP0 (JFIF 1.01, aspect 1:1), DQT x2 (zigzag order), SOF0, DHT x4
// (standard tables), SOS.
void jpeg_headers(int W, int H, int quality, int sub, std::vector<uint8_t> &h) {
    static const int kZigzag[64] = {
        0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
        41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
        30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};
    auto put16 = [&](int v) {
        h.push_back((uint8_t)(v >> 8));
        h.push_back((uint8_t)v);
    };
    h = {0xFF, 0xD8, 0xFF, 0xE0};
    put16(16);
    const uint8_t jfif[14] = {'J', 'F', 'I', 'F', 0, 1, 1, 0, 0, 1, 0, 1, 0, 0};
    h.insert(h.end(), jfif, jfif + 14);
    uint16_t qt[2][64];
    jpeg_quant_tables(quality, qt);
    for (int t = 0; t < 2; t++) {
        h.push_back(0xFF);
        h.push_back(0xDB);
        put16(67);
        h.push_back((uint8_t)t);
        for (int i = 0; i < 64; i++) h.push_back((uint8_t)qt[t][kZigzag[i]]);
    }
    h.push_back(0xFF);
    h.push_back(0xC0);
    put16(17);
    h.push_back(8);
    put16(H);
    put16(W);
    h.push_back(3);
    const uint8_t ysamp = sub ? 0x22 : 0x11;
    const uint8_t comps[9] = {1, ysamp, 0, 2, 0x11, 1, 3, 0x11, 1};
    h.insert(h.end(), comps, comps + 9);
    for (int t = 0; t < 2; t++)
        for (int ac = 0; ac < 2; ac++) {
            const uint8_t *bits, *vals;
            int nv;
            jpeg_huffman_spec(t, ac, &bits, &vals, &nv);
            h.push_back(0xFF);
            h.push_back(0xC4);
            put16(2 + 1 + 16 + nv);
            h.push_back((uint8_t)((ac << 4) | t));
            h.insert(h.end(), bits, bits + 16);
            h.insert(h.end(), vals, vals + nv);
        }
    h.push_back(0xFF);
    h.push_back(0xDA);
    put16(12);
    const uint8_t sos[10] = {3, 1, 0x00, 2, 0x11, 3, 0x11, 0, 63, 0};
    h.insert(h.end(), sos, sos + 10);
}

}  // namespace

// =========================================================== C ABI =========
extern "C" {

int gsr_abi_version(void) { return GSR_ABI_VERSION; }

int gsr_tile_size(int *out_w, int *out_h) {
    if (!out_w || !out_h) return fail(GSR_E_INVALID, "null output");
    *out_w = kTileW;
    *out_h = kTileH;
    return GSR_OK;
}

const char *gsr_last_error(void) { return g_err.c_str(); }

int gsr_device_count(int *out_count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (out_count) *out_count = n;
    return GSR_OK;
}

int gsr_scene_create(gsr_scene **out, int device, int64_t n, const double *means,
                     const double *scales, const double *rotations, const double *opacities,
                     const double *colors_dc, const double *sh_coeffs, const double *rsq) {
    if (!out) return fail(GSR_E_INVALID, "out is null");
    *out = nullptr;
    if (n < 0 || n >= (int64_t(1) << 31)) return fail(GSR_E_INVALID, "invalid Gaussian count");
    if (n > 0 && (!means || !scales || !rotations || !opacities || !colors_dc))
        return fail(GSR_E_INVALID, "null attribute array");
    int ndev = 0;
    gsr_device_count(&ndev);
    if (ndev == 0) return fail(GSR_E_NO_DEVICE, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(GSR_E_INVALID, "device index out of range");
    DeviceGuard g(device);
    gsr_scene *sc = new (std::nothrow) gsr_scene();
    if (!sc) return fail(GSR_E_OOM, "host allocation failed");
    sc->device = device;
    sc->n = n;
    sc->stride = round_up(std::max<int64_t>(n, 1), 32);
    sc->has_sh = sh_coeffs != nullptr;
    // f32 SH storage when lossless (PLY scenes are f32 on disk, model.py:188)
    bool f32ok = true;
    if (sh_coeffs)
        for (int64_t i = 0; i < n * 48 && f32ok; i++)
            f32ok = (double)(float)sh_coeffs[i] == sh_coeffs[i];
    sc->sh_f32 = f32ok ? 1 : 0;
    const int64_t st = sc->stride;
    const SceneLayout L = scene_layout(st, sc->has_sh, sc->sh_f32);
    int rc = ensure(sc->block, L.total);
    if (rc) {
        delete sc;
        return rc;
    }
    // host staging in planar (SoA) layout
    std::vector<unsigned char> host(L.total, 0);
    auto plane_d = [&](size_t o, const double *src, int k, int comps) {
        double *d = reinterpret_cast<double *>(host.data() + o) + (size_t)k * st;
        for (int64_t i = 0; i < n; i++) d[i] = src[i * comps + k];
    };
    auto plane_f = [&](size_t o, const double *src, int k, int comps) {
        float *d = reinterpret_cast<float *>(host.data() + o) + (size_t)k * st;
        for (int64_t i = 0; i < n; i++) d[i] = (float)src[i * comps + k];
    };
    for (int k = 0; k < 3; k++) {
        plane_d(L.mean, means, k, 3);
        plane_d(L.scale, scales, k, 3);
        plane_f(L.dc, colors_dc, k, 3);
    }
    for (int k = 0; k < 4; k++) plane_d(L.rot, rotations, k, 4);
    {
        double *m4 = reinterpret_cast<double *>(host.data() + L.mean4);
        for (int64_t i = 0; i < n; i++)
            for (int k = 0; k < 3; k++) m4[(size_t)L.m4_row * i + k] = means[i * 3 + k];
    }
    plane_f(L.opac, opacities, 0, 1);
    plane_d(L.op64, opacities, 0, 1);
    if (rsq) plane_d(L.rsq, rsq, 0, 1);
    if (sc->has_sh) {  // rows of 48 coefficients (SceneView.sh)
        if (sc->sh_f32) {
            float *d = reinterpret_cast<float *>(host.data() + L.sh);
            for (int64_t i = 0; i < n; i++)
                for (int j = 0; j < 48; j++)
                    d[(size_t)L.sh_row * i + j] = (float)sh_coeffs[i * 48 + j];
        } else {
            std::memcpy(host.data() + L.sh, sh_coeffs, sizeof(double) * (size_t)(n * 48));
        }
    }
    unsigned char *d = sc->block.as<unsigned char>();
    cudaError_t e = cudaMemcpy(d, host.data(), L.total, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        delete sc;
        return fail_cuda(e, "scene upload");
    }
    if (!rsq && n > 0) {
        launch_rsq(reinterpret_cast<const double *>(d + L.op64), n,
                   reinterpret_cast<double *>(d + L.rsq), nullptr);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            delete sc;
            return fail_cuda(e, "rsq kernel");
        }
    }
    sc->bind(L);
    *out = sc;
    return GSR_OK;
}

int gsr_scene_destroy(gsr_scene *scene) {
    if (!scene) return GSR_OK;
    DeviceGuard g(scene->device);
    delete scene;
    return GSR_OK;
}

int64_t gsr_scene_count(const gsr_scene *scene) { return scene ? scene->n : -1; }

int64_t gsr_scene_device_bytes(const gsr_scene *scene) {
    return scene ? (int64_t)scene->block.bytes : 0;
}

int gsr_scene_sh_is_f32(const gsr_scene *scene) { return scene ? scene->sh_f32 : 0; }

int gsr_ctx_create(gsr_ctx **out, int device) {
    if (!out) return fail(GSR_E_INVALID, "out is null");
    *out = nullptr;
    int ndev = 0;
    gsr_device_count(&ndev);
    if (ndev == 0) return fail(GSR_E_NO_DEVICE, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(GSR_E_INVALID, "device index out of range");
    DeviceGuard g(device);
    gsr_ctx *c = new (std::nothrow) gsr_ctx();
    if (!c) return fail(GSR_E_OOM, "host allocation failed");
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = radix_init_attributes();
    if (e == cudaSuccess) e = binning_init_attributes();
    for (int i = 0; i < 8 && e == cudaSuccess; i++) e = cudaEventCreate(&c->ev[i]);
    for (int i = 0; i <= gsr_ctx::kMaxMarks && e == cudaSuccess; i++) e = cudaEventCreate(&c->kev[i]);
    if (e == cudaSuccess)
        e = cudaMallocHost((void **)&c->hctr, gsr_ctx::kCtrBytes);
    if (e == cudaSuccess) e = cudaMallocHost((void **)&c->hssim, sizeof(double) * 64);
    if (e == cudaSuccess)
        c->hsched = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(c->hctr) +
                                                 gsr_ctx::kSchedOff);
    if (e == cudaSuccess) e = cudaMallocHost((void **)&c->hjpeg, sizeof(uint32_t) * 4);
    if (e != cudaSuccess) {
        int rc = fail_cuda(e, "context setup");
        gsr_ctx_destroy(c);
        return rc;
    }
    int rc = ensure(c->ctr, gsr_ctx::kCtrBytes);  // counters, sticky counters, sort schedule
    if (!rc) rc = ensure(c->params, sizeof(FrameParams));
    if (!rc && cudaMemset(c->ctr.p, 0, c->ctr.bytes) != cudaSuccess)
        rc = fail(GSR_E_CUDA, "memset");
    if (!rc) std::memset(c->hctr, 0, gsr_ctx::kCtrBytes);
    if (!rc) rc = ensure(c->ssim_misc, 64);
    if (!rc) rc = ensure(c->ssim_w, sizeof(double) * 11);
    if (rc) {
        gsr_ctx_destroy(c);
        return rc;
    }
    // scipy _gaussian_kernel1d(sigma=1.5, order 0, radius 5), f64
    double w[11], sum = 0.0;
    for (int i = 0; i < 11; i++) {
        const double x = (double)(i - 5);
        w[i] = std::exp(-0.5 / (1.5 * 1.5) * (x * x));
        sum += w[i];
    }
    for (int i = 0; i < 11; i++) w[i] = w[i] / sum;
    e = cudaMemcpy(c->ssim_w.p, w, sizeof(w), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        int rc2 = fail_cuda(e, "ssim weights");
        gsr_ctx_destroy(c);
        return rc2;
    }
    *out = c;
    return GSR_OK;
}

int gsr_ctx_destroy(gsr_ctx *ctx) {
    if (!ctx) return GSR_OK;
    DeviceGuard g(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : ctx->kev)
        if (e) cudaEventDestroy(e);
    if (ctx->hctr) cudaFreeHost(ctx->hctr);
    if (ctx->hssim) cudaFreeHost(ctx->hssim);
    if (ctx->hjpeg) cudaFreeHost(ctx->hjpeg);
    for (auto &fg : ctx->graphs) destroy_graph(fg);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return GSR_OK;
}

int64_t gsr_ctx_device_bytes(const gsr_ctx *ctx) { return ctx ? ctx->bytes() : 0; }

const uint8_t *gsr_ctx_frame_u8(const gsr_ctx *ctx) {
    return ctx ? ctx->frame_u8.as<uint8_t>() : nullptr;
}

void *gsr_ctx_stream(const gsr_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int gsr_ctx_set_kernel_timing(gsr_ctx *ctx, int enable) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    ctx->ktime = (enable & GSR_TIMING_EVENTS) != 0;
    ctx->kcount = (enable & GSR_TIMING_COUNTERS) != 0;
    ctx->stages = (enable & GSR_TIMING_STAGES) != 0;
    ctx->nmarks = 0;
    return GSR_OK;
}

int gsr_ctx_set_slicing(gsr_ctx *ctx, int64_t min_gaussians, float front_fraction) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    if (!(front_fraction >= 0.0f && front_fraction <= 1.0f))
        return fail(GSR_E_INVALID, "front_fraction must be in [0, 1]");
    ctx->slice_min_n = min_gaussians < 0 ? -1 : min_gaussians;
    ctx->slice_frac_v = front_fraction;
    return GSR_OK;
}

int gsr_ctx_kernel_times(gsr_ctx *ctx, int max, char *names, float *ms, int *n) {
    if (!ctx || !n) return fail(GSR_E_INVALID, "null argument");
    DeviceGuard g(ctx->device);
    int rc = complete_frame(ctx);
    if (rc) return rc;
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    const int cnt = ctx->nmarks < max ? ctx->nmarks : max;
    for (int i = 0; i < cnt; i++) {
        float t = 0.0f;
        GSR_CUDA_OK(cudaEventElapsedTime(&t, ctx->kev[i], ctx->kev[i + 1]));
        if (ms) ms[i] = t;
        if (names) {
            std::strncpy(names + 48 * i, ctx->kname[i], 47);
            names[48 * i + 47] = '\0';
        }
    }
    *n = cnt;
    return GSR_OK;
}

int gsr_render_async(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
                     const float background[3], int sh_degree, int frustum_cull) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    DeviceGuard g(ctx->device);
    const float zero[3] = {0, 0, 0};
    return enqueue_frame(ctx, scene, cam, background ? background : zero, sh_degree, frustum_cull,
                         false, false);
}

namespace {
// Device view of `p` when it is page-locked host memory mapped into the
// device address space (cudaHostAlloc / cudaHostRegister / torch pin_memory),
// else null.  Probed per call: a cached answer could outlive the allocation.
// GSR_ZERO_COPY=0 turns the direct store off (the frame is then copied).
uint8_t *mapped_host(uint8_t *p) {
    static const int enabled = [] {
        const char *e = getenv("GSR_ZERO_COPY");
        return e && e[0] == '0' ? 0 : 1;
    }();
    if (!enabled) return nullptr;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? static_cast<uint8_t *>(at.devicePointer) : nullptr;
}
}  // namespace

int gsr_render_enqueue(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
                       const float background[3], int sh_degree, int frustum_cull,
                       uint8_t *out_u8) {
    if (!ctx || !out_u8) return fail(GSR_E_INVALID, "null argument");
    DeviceGuard g(ctx->device);
    int rc = complete_frame(ctx);  // a ctx holds one frame in flight
    if (rc) return rc;
    const float zero[3] = {0, 0, 0};
    // the frame is copied after the blend (a copy engine transfer overlaps the
    // other contexts' kernels; storing from the blend measured no faster here)
    rc = enqueue_frame(ctx, scene, cam, background ? background : zero, sh_degree, frustum_cull,
                       false, false);
    if (rc) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(out_u8, ctx->frame_u8.p, (size_t)cam->width * cam->height * 3,
                                cudaMemcpyDeviceToHost, ctx->stream));
    ctx->saved_out = out_u8;
    return GSR_OK;
}

int gsr_ctx_finish(gsr_ctx *ctx, uint8_t *out_u8, gsr_stats *stats) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    DeviceGuard g(ctx->device);
    const gsr_scene *sc = ctx->saved.scene;
    int rc = complete_frame(ctx);
    if (rc) return rc;
    if (out_u8) {
        GSR_CUDA_OK(cudaMemcpyAsync(out_u8, ctx->frame_u8.p, (size_t)ctx->W * ctx->H * 3,
                                    cudaMemcpyDeviceToHost, ctx->stream));
        GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    }
    fill_stats(ctx, sc, stats);
    return GSR_OK;
}


int gsr_render(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
               const float background[3], int sh_degree, int frustum_cull, uint8_t *out_u8,
               float *out_rgb, float *out_T, gsr_stats *stats) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    DeviceGuard g(ctx->device);
    const float zero[3] = {0, 0, 0};
    const bool want_rgb = out_rgb || out_T;
    ctx->zc_host = out_u8 ? mapped_host(out_u8) : nullptr;
    int rc = enqueue_frame(ctx, scene, cam, background ? background : zero, sh_degree,
                           frustum_cull, want_rgb, false);
    ctx->zc_host = nullptr;  // a re-render (complete_frame) writes the device frame only
    if (rc) return rc;
    const size_t px = (size_t)cam->width * cam->height;
    // copies ride the stream; if the frame overflows they are redone below
    if (out_u8 && !ctx->zc_used)
        GSR_CUDA_OK(cudaMemcpyAsync(out_u8, ctx->frame_u8.p, px * 3, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    if ((rc = complete_frame(ctx))) return rc;
    if (ctx->retries && out_u8)
        GSR_CUDA_OK(cudaMemcpy(out_u8, ctx->frame_u8.p, px * 3, cudaMemcpyDeviceToHost));
    if (out_rgb)
        GSR_CUDA_OK(cudaMemcpy(out_rgb, ctx->frame_rgb.p, px * 3 * sizeof(float),
                               cudaMemcpyDeviceToHost));
    if (out_T)
        GSR_CUDA_OK(cudaMemcpy(out_T, ctx->frame_t.p, px * sizeof(float), cudaMemcpyDeviceToHost));
    fill_stats(ctx, scene, stats);
    return GSR_OK;
}

int gsr_debug_preprocess(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
                         int sh_degree, int frustum_cull, uint8_t *out_keep, int64_t *out_order,
                         float *out_packed, gsr_stats *stats) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    DeviceGuard g(ctx->device);
    const float zero[3] = {0, 0, 0};
    int rc = enqueue_frame(ctx, scene, cam, zero, sh_degree, frustum_cull, false, true);
    if (rc) return rc;
    if ((rc = complete_frame(ctx))) return rc;
    const int64_t n = scene->n, k = ctx->hctr->K;
    if (out_keep && n > 0)
        GSR_CUDA_OK(cudaMemcpy(out_keep, ctx->keep.p, (size_t)n, cudaMemcpyDeviceToHost));
    if (out_order && k > 0) {
        std::vector<uint32_t> o((size_t)k);
        const DevBuf &vb = ctx->vals[ctx->hsched[16] & 1u];
        GSR_CUDA_OK(cudaMemcpy(o.data(), vb.p, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < k; i++) out_order[i] = o[i];
    }
    if (out_packed && k > 0) {
        std::vector<SplatRec> r((size_t)k);
        std::vector<uint32_t> o((size_t)k);
        std::vector<float4> col((size_t)k);  // colours by depth rank
        std::vector<SplatRec> geo((size_t)scene->n);  // by Gaussian index: b.w = ry
        GSR_CUDA_OK(cudaMemcpy(geo.data(), ctx->geo.p, sizeof(SplatRec) * scene->n,
                               cudaMemcpyDeviceToHost));
        const DevBuf &vb = ctx->vals[ctx->hsched[16] & 1u];
        GSR_CUDA_OK(cudaMemcpy(r.data(), ctx->srec.p, sizeof(SplatRec) * k, cudaMemcpyDeviceToHost));
        GSR_CUDA_OK(cudaMemcpy(o.data(), vb.p, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost));
        GSR_CUDA_OK(cudaMemcpy(col.data(), ctx->colr.p, sizeof(float4) * k,
                               cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < k; i++) {
            float *p = out_packed + 11 * i;
            const SplatRec &s = r[i];
            const float4 &cc = col[i];
            p[0] = s.a.x; p[1] = s.a.y; p[2] = s.a.z; p[3] = s.a.w; p[4] = s.b.x; p[5] = s.b.y;
            p[6] = cc.x; p[7] = cc.y; p[8] = cc.z; p[9] = s.b.z; p[10] = geo[o[i]].b.w;
        }
    }
    fill_stats(ctx, scene, stats);
    return GSR_OK;
}

namespace {
// The debug entries that read the frame's depth-ranked records or lists need
// a one-pass frame (all kept splats ranked): re-render the last call that way.
int ensure_one_pass(gsr_ctx *c) {
    int rc = complete_frame(c);
    if (rc || !c->last_sliced) return rc;
    SavedCall sv = c->saved;
    if (!sv.scene) return fail(GSR_E_INVALID, "the last frame's scene is gone");
    // one pass through completion: a re-render complete_frame does after a
    // buffer overflow must stay one-pass too (it used to slice again, so a
    // caller sizing its buffers from the first call's counts could be handed
    // a different frame's lists)
    c->force_full = true;
    rc = enqueue_frame(c, sv.scene, &sv.cam, sv.bg, sv.sh_degree, sv.cull, sv.want_rgb,
                       sv.want_keep);
    if (!rc) rc = complete_frame(c);
    c->force_full = false;
    return rc;
}
}  // namespace

int gsr_debug_tile_lists(gsr_ctx *ctx, int32_t *out_tiles, int32_t *out_ranks,
                         int32_t *out_ranges, gsr_stats *stats) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    DeviceGuard g(ctx->device);
    int rc = ensure_one_pass(ctx);
    if (rc) return rc;
    const int64_t d = std::min<int64_t>(ctx->hctr->D, ctx->cap_d);
    std::vector<uint2> rg((size_t)ctx->ntiles);
    if (ctx->ntiles > 0)
        GSR_CUDA_OK(cudaMemcpy(rg.data(), ctx->ranges.p, sizeof(uint2) * ctx->ntiles,
                               cudaMemcpyDeviceToHost));
    if (out_ranks && d > 0)
        GSR_CUDA_OK(cudaMemcpy(out_ranks, ctx->tile_vals.p, 4 * d, cudaMemcpyDeviceToHost));
    for (int t = 0; t < ctx->ntiles; t++) {
        if (out_tiles)  // tile ids are implicit in the ranges (lists are tile-major)
            for (uint32_t i = rg[t].x; i < rg[t].y && (int64_t)i < d; i++) out_tiles[i] = t;
        if (out_ranges) {
            out_ranges[2 * t] = (int32_t)rg[t].x;
            out_ranges[2 * t + 1] = (int32_t)rg[t].y;
        }
    }
    if (stats) {
        stats->tile_keys = ctx->hctr->D;
        stats->splats_drawn = ctx->hctr->K;
    }
    return GSR_OK;
}

namespace {
// Builds the contract lists of the last frame (contract.cu): keys, then --
// once their count is known on the host -- the 64-bit radix sort and the
// ranges.  Two attempts: the first with the capacity of the previous frame.
int build_contract(gsr_ctx *c, int tile) {
    const int64_t k = (int64_t)c->hctr->K;  // one-pass frame: all kept splats ranked
    const int tiles_x = (c->W + tile - 1) / tile, ntiles = tiles_x * ((c->H + tile - 1) / tile);
    int rc;
    if (c->cap_c == 0) c->cap_c = round_up(std::max<int64_t>(int64_t(1) << 20, 8 * k), 4096);
    if ((rc = ensure(c->cdcount, sizeof(unsigned long long)))) return rc;
    if ((rc = ensure(c->csched, 64 * sizeof(uint32_t)))) return rc;
    if ((rc = ensure(c->cranges, sizeof(uint2) * (size_t)std::max(ntiles, 1)))) return rc;
    float t_keys = 0.0f, t_sort = 0.0f;
    unsigned long long d = 0;
    for (int attempt = 0;; attempt++) {
        for (int i = 0; i < 2; i++) {
            if ((rc = ensure(c->ckeys[i], sizeof(unsigned long long) * c->cap_c))) return rc;
            if ((rc = ensure(c->cvals[i], sizeof(uint32_t) * c->cap_c))) return rc;
        }
        ContractArgs a;
        a.srec = c->srec.as<SplatRec>();
        a.count = &c->ctr.as<FrameCounters>()->K;
        a.width = c->W;
        a.tile = tile;
        a.tiles_x = tiles_x;
        a.keys = c->ckeys[0].as<unsigned long long>();
        a.cap = c->cap_c;
        a.d_count = c->cdcount.as<unsigned long long>();
        GSR_CUDA_OK(cudaMemsetAsync(a.d_count, 0, sizeof(unsigned long long), c->stream));
        cudaEventRecord(c->ev[6], c->stream);
        launch_contract_keys(a, k, c->stream);
        cudaEventRecord(c->ev[7], c->stream);
        GSR_CUDA_OK(cudaMemcpyAsync(&d, a.d_count, sizeof(d), cudaMemcpyDeviceToHost, c->stream));
        GSR_CUDA_OK(cudaStreamSynchronize(c->stream));
        GSR_CUDA_OK(cudaEventElapsedTime(&t_keys, c->ev[6], c->ev[7]));
        if ((int64_t)d <= c->cap_c) break;
        if (attempt == 1) return fail(GSR_E_OOM, "contract key buffer overflow");
        if (d >= (1ull << 30)) return fail(GSR_E_OOM, "contract lists exceed 2^30 entries");
        c->cap_c = round_up((int64_t)d + (int64_t)d / 8 + 4096, 4096);
    }
    if ((rc = ensure(c->cwork, sort_work_bytes(std::max<int64_t>((int64_t)d, 1), 8, 8)))) return rc;
    cudaEventRecord(c->ev[6], c->stream);
    launch_onesweep_sort<unsigned long long>(
        c->ckeys[0].as<unsigned long long>(), c->ckeys[1].as<unsigned long long>(),
        c->cvals[0].as<uint32_t>(), c->cvals[1].as<uint32_t>(), true, false, nullptr,
        (int64_t)d, (int64_t)d, 8, false, c->cwork.p, c->csched.as<uint32_t>(), nullptr, c->sms,
        c->stream);
    launch_contract_ranges(c->ckeys[0].as<unsigned long long>(),
                           c->ckeys[1].as<unsigned long long>(), c->csched.as<uint32_t>(),
                           c->cdcount.as<unsigned long long>(), c->cap_c,
                           c->cranges.as<uint2>(), ntiles, c->sms, c->stream);
    cudaEventRecord(c->ev[7], c->stream);
    GSR_CUDA_OK(cudaMemcpyAsync(c->hsched, c->csched.p, 64 * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, c->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(c->stream));
    GSR_CUDA_OK(cudaEventElapsedTime(&t_sort, c->ev[6], c->ev[7]));
    c->contract_buf = (int)(c->hsched[16] & 1u);
    c->contract_d = (int64_t)d;
    c->contract_ms = t_keys + t_sort;
    c->contract_tile = tile;
    return GSR_OK;
}
}  // namespace

int gsr_debug_contract_tiles(gsr_ctx *ctx, int tile, int64_t *out_count, int32_t *out_tiles,
                             int32_t *out_ranks, int32_t *out_ranges, float *out_ms) {
    if (!ctx) return fail(GSR_E_INVALID, "ctx is null");
    if (tile < 1 || tile > 256) return fail(GSR_E_INVALID, "tile size must be in 1..256");
    DeviceGuard g(ctx->device);
    if (ctx->W <= 0 || ctx->H <= 0) return fail(GSR_E_INVALID, "no frame rendered on this context");
    int rc = ctx->contract_tile == tile ? complete_frame(ctx) : ensure_one_pass(ctx);
    if (rc) return rc;
    if (ctx->contract_tile != tile && (rc = build_contract(ctx, tile))) return rc;
    const int64_t d = ctx->contract_d;
    if (out_count) *out_count = d;
    if (out_ms) *out_ms = ctx->contract_ms;
    if ((out_tiles || out_ranks) && d > 0) {
        std::vector<unsigned long long> keys((size_t)d);
        const DevBuf &kb = ctx->ckeys[ctx->contract_buf];
        GSR_CUDA_OK(cudaMemcpy(keys.data(), kb.p, sizeof(unsigned long long) * d,
                               cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < d; i++) {
            if (out_tiles) out_tiles[i] = (int32_t)(keys[i] >> 32);
            if (out_ranks) out_ranks[i] = (int32_t)(keys[i] & 0xffffffffu);
        }
    }
    if (out_ranges) {
        const int ntiles = ((ctx->W + tile - 1) / tile) * ((ctx->H + tile - 1) / tile);
        GSR_CUDA_OK(cudaMemcpy(out_ranges, ctx->cranges.p, sizeof(uint2) * (size_t)ntiles,
                               cudaMemcpyDeviceToHost));
    }
    return GSR_OK;
}

int gsr_debug_blend_items(gsr_ctx *ctx, uint32_t *out, int64_t n) {
    if (!ctx || !out) return fail(GSR_E_INVALID, "null argument");
    DeviceGuard g(ctx->device);
    int rc = complete_frame(ctx);
    if (rc) return rc;
    const int64_t have = (int64_t)ctx->ntiles * (kTileH / 2);
    if (!ctx->kcount || ctx->used.bytes < sizeof(uint32_t) * (size_t)(ctx->cap_n + have))
        return fail(GSR_E_INVALID, "blend item info needs GSR_TIMING_COUNTERS on the last frame");
    GSR_CUDA_OK(cudaMemcpy(out, ctx->used.as<uint32_t>() + ctx->cap_n,
                           sizeof(uint32_t) * (size_t)std::min(n, have), cudaMemcpyDeviceToHost));
    return GSR_OK;
}

int gsr_debug_frame_counters(gsr_ctx *ctx, uint64_t *out, int n) {
    if (!ctx || !out) return fail(GSR_E_INVALID, "null argument");
    DeviceGuard g(ctx->device);
    int rc = complete_frame(ctx);
    if (rc) return rc;
    const FrameCounters &f = *ctx->hctr;
    const bool sliced = ctx->last_sliced;
    const uint64_t v[GSR_NCOUNTERS] = {f.K, f.Dtot, f.Ptot, f.E, f.Rb, f.Rp, f.b_walked, f.b_hit,
                                       f.b_batches, f.b_iters, f.b_lanes, f.b_items, f.b_used,
                                       sliced ? f.KA : f.K, sliced ? f.KB : 0u,
                                       sliced ? f.n_unsat : 0u};
    for (int i = 0; i < n && i < GSR_NCOUNTERS; i++) out[i] = v[i];
    return GSR_OK;
}

int gsr_resample_bilinear_u8(gsr_ctx *ctx, const uint8_t *src, int src_w, int src_h, uint8_t *dst,
                             int dst_w, int dst_h) {
    if (!ctx || !src || !dst) return fail(GSR_E_INVALID, "null argument");
    if (src_w <= 0 || src_h <= 0 || dst_w <= 0 || dst_h <= 0)
        return fail(GSR_E_INVALID, "dimensions must be positive");
    DeviceGuard g(ctx->device);
    int rc;
    const size_t sb = (size_t)src_w * src_h * 3, db = (size_t)dst_w * dst_h * 3;
    if ((rc = ensure(ctx->src_u8, sb))) return rc;
    if ((rc = ensure(ctx->dst_u8, db))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->src_u8.p, src, sb, cudaMemcpyHostToDevice, ctx->stream));
    if ((rc = resample_device(ctx, ctx->src_u8.as<uint8_t>(), src_w, src_h,
                              ctx->dst_u8.as<uint8_t>(), dst_w, dst_h)))
        return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(dst, ctx->dst_u8.p, db, cudaMemcpyDeviceToHost, ctx->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    return GSR_OK;
}

int gsr_ssim_u8(gsr_ctx *ctx, const uint8_t *a, const uint8_t *b, int width, int height,
                double *out_ssim) {
    if (!ctx || !a || !b || !out_ssim) return fail(GSR_E_INVALID, "null argument");
    if (width < 11 || height < 11) return fail(GSR_E_TOO_SMALL, "images must be at least 11x11");
    DeviceGuard g(ctx->device);
    int rc;
    const size_t nb = (size_t)width * height * 3;
    if ((rc = ensure(ctx->src_u8, nb))) return rc;
    if ((rc = ensure(ctx->dst_u8, nb))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->src_u8.p, a, nb, cudaMemcpyHostToDevice, ctx->stream));
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->dst_u8.p, b, nb, cudaMemcpyHostToDevice, ctx->stream));
    double *dout = reinterpret_cast<double *>(ctx->ssim_misc.as<unsigned char>() + 8);
    SsimInput in{ctx->src_u8.as<uint8_t>(), ctx->dst_u8.as<uint8_t>(), nullptr, nullptr};
    if ((rc = ssim_device(ctx, in, width, height, dout))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->hssim, dout, sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    *out_ssim = ctx->hssim[0];
    return GSR_OK;
}

int gsr_ssim_luma_f64(gsr_ctx *ctx, const double *x, const double *y, int width, int height,
                      double *out_ssim) {
    if (!ctx || !x || !y || !out_ssim) return fail(GSR_E_INVALID, "null argument");
    if (width < 11 || height < 11) return fail(GSR_E_TOO_SMALL, "images must be at least 11x11");
    DeviceGuard g(ctx->device);
    int rc;
    const size_t nb = (size_t)width * height * sizeof(double);
    if ((rc = ensure(ctx->src_u8, nb))) return rc;
    if ((rc = ensure(ctx->dst_u8, nb))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->src_u8.p, x, nb, cudaMemcpyHostToDevice, ctx->stream));
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->dst_u8.p, y, nb, cudaMemcpyHostToDevice, ctx->stream));
    double *dout = reinterpret_cast<double *>(ctx->ssim_misc.as<unsigned char>() + 8);
    SsimInput in{nullptr, nullptr, ctx->src_u8.as<double>(), ctx->dst_u8.as<double>()};
    if ((rc = ssim_device(ctx, in, width, height, dout))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->hssim, dout, sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    *out_ssim = ctx->hssim[0];
    return GSR_OK;
}

int gsr_host_alloc(void **out, size_t bytes) {
    if (!out) return fail(GSR_E_INVALID, "out is null");
    *out = nullptr;
    GSR_CUDA_OK(cudaMallocHost(out, bytes ? bytes : 1));
    return GSR_OK;
}

int gsr_host_free(void *ptr) {
    if (ptr) GSR_CUDA_OK(cudaFreeHost(ptr));
    return GSR_OK;
}

int gsr_encode_jpeg(gsr_ctx *ctx, const uint8_t *rgb, int width, int height, int quality,
                    int subsampling, uint8_t *out, size_t out_cap, size_t *out_len) {
    if (!ctx || !out_len) return fail(GSR_E_INVALID, "null argument");
    if (width <= 0 || height <= 0 || width > 65535 || height > 65535)
        return fail(GSR_E_INVALID, "cannot encode a zero-dimension or oversized frame");
    if (quality < 1 || quality > 100) return fail(GSR_E_INVALID, "jpeg quality out of range 1..100");
    if (subsampling != 0 && subsampling != 2)
        return fail(GSR_E_INVALID, "subsampling must be 0 (4:4:4) or 2 (4:2:0)");
    DeviceGuard g(ctx->device);
    int rc;
    const uint8_t *src = nullptr;
    const size_t nb = (size_t)width * height * 3;
    if (rgb) {
        if ((rc = ensure(ctx->src_u8, nb))) return rc;
        GSR_CUDA_OK(cudaMemcpyAsync(ctx->src_u8.p, rgb, nb, cudaMemcpyHostToDevice, ctx->stream));
        src = ctx->src_u8.as<uint8_t>();
    } else {
        if ((rc = complete_frame(ctx))) return rc;
        if (ctx->W != width || ctx->H != height)
            return fail(GSR_E_INVALID, "frame size differs from the ctx's last render");
        src = ctx->frame_u8.as<uint8_t>();
    }
    JpegLayout L;
    const size_t ws = jpeg_workspace_bytes(width, height, subsampling == 2, &L);
    if ((rc = ensure(ctx->jpeg_ws, ws))) return rc;
    GSR_CUDA_OK(launch_jpeg(src, width, height, quality, L, ctx->jpeg_ws.as<unsigned char>(),
                            ctx->hjpeg, ctx->stream));
    std::vector<uint8_t> hdr;
    jpeg_headers(width, height, quality, subsampling == 2, hdr);
    const size_t scan = ctx->hjpeg[1];
    const size_t total = hdr.size() + scan + 2;
    *out_len = total;
    if (!out) return GSR_OK;
    if (out_cap < total) return fail(GSR_E_INVALID, "output buffer too small");
    std::memcpy(out, hdr.data(), hdr.size());
    GSR_CUDA_OK(cudaMemcpyAsync(out + hdr.size(), ctx->jpeg_ws.as<unsigned char>() + L.off_out,
                                scan, cudaMemcpyDeviceToHost, ctx->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    out[total - 2] = 0xFF;
    out[total - 1] = 0xD9;
    return GSR_OK;
}

int gsr_sse_u8(gsr_ctx *ctx, const uint8_t *a, const uint8_t *b, int64_t n,
               uint64_t *out_sse) {
    if (!ctx || !a || !b || !out_sse || n < 0) return fail(GSR_E_INVALID, "null argument");
    DeviceGuard g(ctx->device);
    int rc;
    if ((rc = ensure(ctx->src_u8, (size_t)n))) return rc;
    if ((rc = ensure(ctx->dst_u8, (size_t)n))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->src_u8.p, a, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->dst_u8.p, b, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    unsigned long long *dsse = reinterpret_cast<unsigned long long *>(ctx->ssim_misc.as<unsigned char>() + 16);
    launch_sse(ctx->src_u8.as<uint8_t>(), ctx->dst_u8.as<uint8_t>(), n, dsse, ctx->stream);
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->hssim, dsse, 8, cudaMemcpyDeviceToHost, ctx->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    std::memcpy(out_sse, ctx->hssim, 8);
    return GSR_OK;
}

int gsr_eval_frame(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *base_cam,
                   const float background[3], int sh_degree, const uint8_t *transmitted,
                   int tw, int th, uint8_t *out_gt_u8, double *out_ssim, uint64_t *out_sse) {
    if (!ctx || !base_cam || !transmitted || !out_ssim || !out_sse)
        return fail(GSR_E_INVALID, "null argument");
    if (tw <= 0 || th <= 0) return fail(GSR_E_INVALID, "dimensions must be positive");
    const int W = base_cam->width, H = base_cam->height;
    if (W < 11 || H < 11) return fail(GSR_E_TOO_SMALL, "images must be at least 11x11");
    DeviceGuard g(ctx->device);
    const float zero[3] = {0, 0, 0};
    int rc = enqueue_frame(ctx, scene, base_cam, background ? background : zero, sh_degree, 1,
                           false, false);
    if (rc) return rc;
    if ((rc = complete_frame(ctx))) return rc;
    const size_t nb = (size_t)W * H * 3, tb = (size_t)tw * th * 3;
    if ((rc = ensure(ctx->src_u8, tb))) return rc;
    if ((rc = ensure(ctx->up_u8, nb))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->src_u8.p, transmitted, tb, cudaMemcpyHostToDevice,
                                ctx->stream));
    // metrics.py:208 upscale_to(transmitted, W, H) (identity when equal)
    if ((rc = resample_device(ctx, ctx->src_u8.as<uint8_t>(), tw, th, ctx->up_u8.as<uint8_t>(),
                              W, H)))
        return rc;
    double *dres = reinterpret_cast<double *>(ctx->ssim_misc.as<unsigned char>() + 8);
    unsigned long long *dsse = reinterpret_cast<unsigned long long *>(ctx->ssim_misc.as<unsigned char>() + 16);
    SsimInput in{ctx->up_u8.as<uint8_t>(), ctx->frame_u8.as<uint8_t>(), nullptr, nullptr};
    if ((rc = ssim_device(ctx, in, W, H, dres))) return rc;
    launch_sse(ctx->up_u8.as<uint8_t>(), ctx->frame_u8.as<uint8_t>(), (int64_t)nb, dsse,
               ctx->stream);
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->hssim, dres, 16, cudaMemcpyDeviceToHost, ctx->stream));
    if (out_gt_u8)
        GSR_CUDA_OK(cudaMemcpyAsync(out_gt_u8, ctx->frame_u8.p, nb, cudaMemcpyDeviceToHost,
                                    ctx->stream));
    GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    *out_ssim = ctx->hssim[0];
    std::memcpy(out_sse, &ctx->hssim[1], 8);
    return GSR_OK;
}

int gsr_ladder_ssim(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *base_cam,
                    const float background[3], int sh_degree, int n_rungs,
                    const gsr_camera *rung_cams, double *out_ssim, gsr_stats *base_stats) {
    if (!ctx || !base_cam || (n_rungs > 0 && (!rung_cams || !out_ssim)))
        return fail(GSR_E_INVALID, "null argument");
    if (n_rungs < 0 || n_rungs > 48) return fail(GSR_E_INVALID, "n_rungs must be in 0..48");
    if (base_cam->width < 11 || base_cam->height < 11)
        return fail(GSR_E_TOO_SMALL, "base frame must be at least 11x11");
    DeviceGuard g(ctx->device);
    const float zero[3] = {0, 0, 0};
    const float *bg = background ? background : zero;
    int rc = enqueue_frame(ctx, scene, base_cam, bg, sh_degree, 1, false, false);
    if (rc) return rc;
    if ((rc = complete_frame(ctx))) return rc;
    fill_stats(ctx, scene, base_stats);
    const int W = base_cam->width, H = base_cam->height;
    const size_t nb = (size_t)W * H * 3;
    if ((rc = ensure(ctx->base_u8, nb))) return rc;
    if ((rc = ensure(ctx->up_u8, nb))) return rc;
    GSR_CUDA_OK(cudaMemcpyAsync(ctx->base_u8.p, ctx->frame_u8.p, nb, cudaMemcpyDeviceToDevice,
                                ctx->stream));
    double *dres = reinterpret_cast<double *>(ctx->ssim_misc.as<unsigned char>() + 8);
    std::vector<double> res((size_t)n_rungs);
    for (int i = 0; i < n_rungs; i++) {
        const gsr_camera *rc_cam = &rung_cams[i];
        if ((rc = enqueue_frame(ctx, scene, rc_cam, bg, sh_degree, 1, false, false))) return rc;
        if ((rc = complete_frame(ctx))) return rc;
        if ((rc = resample_device(ctx, ctx->frame_u8.as<uint8_t>(), rc_cam->width, rc_cam->height,
                                  ctx->up_u8.as<uint8_t>(), W, H)))
            return rc;
        SsimInput in{ctx->up_u8.as<uint8_t>(), ctx->base_u8.as<uint8_t>(), nullptr, nullptr};
        if ((rc = ssim_device(ctx, in, W, H, dres))) return rc;
        GSR_CUDA_OK(cudaMemcpyAsync(ctx->hssim, dres, sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
        GSR_CUDA_OK(cudaStreamSynchronize(ctx->stream));
        res[(size_t)i] = ctx->hssim[0];
    }
    for (int i = 0; i < n_rungs; i++) out_ssim[i] = res[(size_t)i];
    return GSR_OK;
}

}  // extern "C"
