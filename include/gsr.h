/*
 * gsr.h -- C ABI of the B200-native per-pose Gaussian-splat render path.
 *
 * Drop-in boundary for splatstream's renderer API.  The reference's boundary
 * is a Python function API with no FFI layer; each entry point
 * below replaces one reference function, cited as path:line under
 * /root/reference/pkg/src/splatstream/.  The Python shim
 * (paper_2605_08699_b200/render.py, metrics.py) binds these through ctypes and
 * re-exposes the reference's exact Python signatures; INTEGRATION.md shows
 * the stub a maintainer adds to splatstream.
 *
 * Conventions: plain pointers and sizes, no torch types; every function
 * returns an int status (GSR_OK or a negative GSR_E_* code, never throws);
 * gsr_last_error() returns a thread-local message for the last failure.
 * Scenes are immutable and may be shared by any number of contexts; a
 * context (stream + workspace) must be used by one thread at a time.
 * Host arrays may be pageable or pinned.
 */
#ifndef GSR_H
#define GSR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSR_ABI_VERSION 1

#if defined(__GNUC__)
#define GSR_API __attribute__((visibility("default")))
#else
#define GSR_API
#endif

/* status codes; the Python shim maps them to the reference's exceptions */
#define GSR_OK 0
#define GSR_E_INVALID (-1)        /* ValueError (camera.py:64-70, render.py:131-132) */
#define GSR_E_CUDA (-2)           /* RenderError (render.py:52-53) */
#define GSR_E_OOM (-3)            /* RenderError */
#define GSR_E_DIM_MISMATCH (-4)   /* metrics.DimensionMismatch (metrics.py:85-86) */
#define GSR_E_TOO_SMALL (-5)      /* metrics.TooSmall (metrics.py:87-88) */
#define GSR_E_NO_DEVICE (-6)      /* RenderError: no CUDA device */
#define GSR_E_PLY_HEADER (-7)     /* model.MalformedHeader (model.py:44-45) */
#define GSR_E_PLY_PROPERTY (-8)   /* model.MissingProperty (model.py:48-49) */
#define GSR_E_PLY_TRUNCATED (-9)  /* model.TruncatedBody (model.py:52-53) */
#define GSR_E_NONFINITE (-10)     /* model.NonFiniteAttribute (model.py:56-57) */

typedef struct gsr_scene gsr_scene;
typedef struct gsr_ctx gsr_ctx;

/* Camera of one render call.  The Python shim fills it with the reference's
 * own host math: w2c = world_to_camera(pose)[:3, :] (camera.py:101-108),
 * campos = -R @ w2c[:3, 3] (render.py:276), intrinsics after
 * scale_intrinsics for ladder rungs (camera.py:146-154, render.py:537). */
typedef struct gsr_camera {
    double w2c[12];     /* row-major 3x4 */
    double campos[3];
    double fx, fy, cx, cy;
    int32_t width, height;
} gsr_camera;

/* RenderStats (render.py:103-107) plus per-stage device timings. */
typedef struct gsr_stats {
    int64_t splats_drawn;     /* K: kept splats */
    int64_t splats_culled;    /* N - K */
    int64_t tile_keys;        /* D: (tile, splat) pairs under the tile-list contract */
    int32_t depth_passes;     /* radix passes of the f64 depth sort */
    int32_t retries;          /* re-renders after growing the tile-key buffer */
    float ms_device;          /* CUDA-event time of the whole device pipeline */
    float ms_preprocess, ms_depth_sort, ms_binning, ms_tile_sort, ms_blend;
                              /* stage times: only with GSR_TIMING_STAGES (four event nodes
                                 in the frame graph, ~0.03 ms of latency), else 0 */
    int32_t kernel_launches;  /* kernels this ctx launched since the last finish/render */
    int32_t overflow_frames;  /* frames since the last finish whose pair/tile buffers overflowed
                                 (re-rendered when completed through finish/render) */
    /* work counters of the last frame (roofline units) */
    int64_t pairs;              /* P: (splat, 64-row tile row) pairs of the render path */
    int64_t composited;         /* E: composited (pixel, splat) evaluations (*) */
    int64_t row_evals_blend;    /* (splat, pixel row) interval evaluations in the blend (*) */
    int64_t row_evals_binning;  /* (splat, pixel row) interval evaluations in the binning */
    /* (*) counted only while gsr_ctx_set_kernel_timing has GSR_TIMING_COUNTERS
     *     on (the counting costs blend instructions), else 0 */
    int32_t long_run_frames;  /* frames since the last finish whose 32-bit depth keys had a
                                 run too long for the fix-up (re-rendered with the 64-bit
                                 sort when completed through finish/render) */
    float ms_slice_b;         /* depth-sliced frames: device time of the second slice (its
                                 filter, sort, colours, lists and blend); the stage times above
                                 are then those of the first slice.  0 for one-pass frames */
} gsr_stats;

GSR_API int gsr_abi_version(void);
/* Tile size of the render path's lists (columns x rows), for the debug
   entries' tile indices (gsr_debug_tile_lists / gsr_debug_blend_items). */
GSR_API int gsr_tile_size(int *out_w, int *out_h);
GSR_API const char *gsr_last_error(void);
GSR_API int gsr_device_count(int *out_count);

/* ---- scenes: replaces the registry's ActivatedPrimitives residency
 * (model.py:89-102, 311-421); upload on load, free on evict ---------------
 * means (N,3), scales (N,3), rotations (N,4) wxyz, opacities (N,),
 * colors_dc (N,3): f64 row-major host arrays as in ActivatedPrimitives.
 * sh_coeffs (N,16,3) f64 or NULL (degree-0 only scene).  rsq (N,) is the
 * view-independent cutoff radius^2 of render.py:476-481, computed by the shim
 * with the reference's numpy expression; NULL computes it on the device
 * (IEEE log, may differ from numpy by 1 ulp).  SH coefficients are stored as
 * f32 when that is lossless (PLY-loaded scenes), else f64. */
GSR_API int gsr_scene_create(gsr_scene **out, int device, int64_t n, const double *means,
                     const double *scales, const double *rotations,
                     const double *opacities, const double *colors_dc,
                     const double *sh_coeffs, const double *rsq);
GSR_API int gsr_scene_destroy(gsr_scene *scene);
GSR_API int64_t gsr_scene_count(const gsr_scene *scene);
GSR_API int64_t gsr_scene_device_bytes(const gsr_scene *scene);
GSR_API int gsr_scene_sh_is_f32(const gsr_scene *scene);

/* ---- PLY scenes on the device: replaces
 * activate(parse_ply(path.read_bytes())) of the registry's load
 * (model.py:354, parse_ply 169-208, activate 211-252) -------------------- */

/* Columns of the loader's properties in the vertex table, in this order
 * (model.py:31-36 REQUIRED_PROPERTIES, then f_rest_0..44, model.py:195). */
#define GSR_PLY_NCOLS 59
typedef struct gsr_ply_info {
    int64_t count;        /* vertex count (element vertex N) */
    int64_t body_offset;  /* first byte of the vertex table */
    int64_t body_bytes;   /* count * n_props * 4 */
    int32_t n_props;      /* float32 properties per vertex */
    int32_t has_rest;     /* all 45 f_rest_* present (model.py:196) */
    int32_t col[GSR_PLY_NCOLS];  /* last column of each name (model.py:189), -1 absent */
    int32_t reserved;
} gsr_ply_info;

/* _parse_header (model.py:105-166) + the property / length checks of
 * parse_ply (model.py:176-186): MalformedHeader / MissingProperty /
 * TruncatedBody with the reference's messages.  Host only (no device). */
GSR_API int gsr_ply_parse_header(const uint8_t *data, int64_t len, gsr_ply_info *info);

typedef struct gsr_ply_stats {
    double h2d_ms;       /* host -> device copy of the vertex table */
    double kernel_ms;    /* decode + checks + activation kernels */
    double total_ms;     /* whole call (host clock) */
    int64_t body_bytes;  /* bytes of the vertex table read */
    int64_t scene_bytes; /* device bytes of the resident scene */
} gsr_ply_stats;

/* Parse + validate + activate a binary PLY on `device` straight into a
 * resident scene: f64 means / scales (np.exp) / rotations (q / |q|) /
 * opacities (scipy expit) / f32 colours and SH / cutoff radius, all equal
 * bit-for-bit to the reference's arrays.  Non-finite raw or activated
 * attributes fail with GSR_E_NONFINITE and the reference's message (checked
 * in the reference's order, model.py:199-203, 239-243).  `stats` nullable. */
GSR_API int gsr_scene_create_ply(gsr_scene **out, int device, const uint8_t *data, int64_t len,
                                 gsr_ply_stats *stats);

/* Read an ActivatedPrimitives attribute back as the reference's f64 array
 * (row-major): GSR_ATTR_MEANS (N,3), SCALES (N,3), ROTATIONS (N,4),
 * OPACITIES (N,), COLORS_DC (N,3; PLY scenes only), SH (N,16,3), RSQ (N,). */
#define GSR_ATTR_MEANS 0
#define GSR_ATTR_SCALES 1
#define GSR_ATTR_ROTATIONS 2
#define GSR_ATTR_OPACITIES 3
#define GSR_ATTR_COLORS_DC 4
#define GSR_ATTR_SH 5
#define GSR_ATTR_RSQ 6   /* (N,) cutoff radius^2 of render.py:476-481 */
GSR_API int gsr_scene_read(const gsr_scene *scene, int attribute, double *host_out);

/* ---- contexts: one CUDA stream + workspace (one per serving thread,
 * server.py:99-100) ------------------------------------------------------- */
GSR_API int gsr_ctx_create(gsr_ctx **out, int device);
GSR_API int gsr_ctx_destroy(gsr_ctx *ctx);
GSR_API int64_t gsr_ctx_device_bytes(const gsr_ctx *ctx);
/* device pointer of the ctx's last u8 frame (H,W,3), valid until next render */
GSR_API const uint8_t *gsr_ctx_frame_u8(const gsr_ctx *ctx);
/* the ctx's cudaStream_t (as void*), e.g. to record timing events on it */
GSR_API void *gsr_ctx_stream(const gsr_ctx *ctx);
/* Per-kernel timing (profiling; off by default).  `enable` is a bit set:
 * GSR_TIMING_EVENTS records a CUDA event on the ctx stream after every kernel
 * of a frame; GSR_TIMING_COUNTERS switches the blend to its counting variant,
 * which fills the (*) work counters of gsr_stats (and costs blend time, so
 * time the kernels with EVENTS alone and count in a separate frame).
 * gsr_ctx_kernel_times waits for the last frame and returns, for each kernel
 * launch in order, its name (NUL-terminated, 48-byte slots in names) and its
 * device time in ms (event after it minus event before it). */
/* Depth-sliced frames (slice.cu): scenes with at least min_gaussians
 * Gaussians are rendered as a front slice of about front_fraction of the
 * kept splats, then the splats behind it that can still reach an unsaturated
 * pixel; frames are identical to a one-pass render.  min_gaussians < 0 and
 * front_fraction 0 restore the defaults (GSR_SLICE_MIN, 262144;
 * GSR_SLICE_FRAC, 0.15); a huge min_gaussians renders every frame in one pass. */
GSR_API int gsr_ctx_set_slicing(gsr_ctx *ctx, int64_t min_gaussians, float front_fraction);
#define GSR_TIMING_EVENTS 1
#define GSR_TIMING_COUNTERS 2
#define GSR_TIMING_STAGES 4   /* stage boundary events: gsr_stats' stage times (else 0) */
GSR_API int gsr_ctx_set_kernel_timing(gsr_ctx *ctx, int enable);
GSR_API int gsr_ctx_kernel_times(gsr_ctx *ctx, int max, char *names, float *ms, int *n);

/* ---- the hot path: render_framebuffer (render.py:516-524) ----------------
 * project (render.py:163-290) -> stable f64 depth sort (293-302) -> tile
 * lists in depth order (32x16 device tiles) -> front-to-back blend
 * (430-473) -> u8 (484-485).  Outputs are optional host buffers:
 *   out_u8   (H,W,3) u8   = framebuffer_to_u8(fb); page-locked memory with
 *                           W % 32 == 0 is written by the blend kernel
 *                           directly (GSR_ZERO_COPY=0: copied instead)
 *   out_rgb  (H,W,3) f32  = rgb before the reference's clip (render.py:470)
 *   out_T    (H,W)   f32  = transmittance (alpha = 1 - T)
 * Synchronous: returns after the frame (and copies) completed. */
GSR_API int gsr_render(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
               const float background[3], int sh_degree, int frustum_cull,
               uint8_t *out_u8, float *out_rgb, float *out_T, gsr_stats *stats);

/* Asynchronous variant: enqueues the frame on the ctx stream and returns.
 * gsr_ctx_finish() waits, re-renders once if the tile-key buffer overflowed,
 * copies the u8 frame to out_u8 (nullable) and fills stats (nullable). */
GSR_API int gsr_render_async(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
                     const float background[3], int sh_degree, int frustum_cull);
GSR_API int gsr_ctx_finish(gsr_ctx *ctx, uint8_t *out_u8, gsr_stats *stats);

/* Pipelined serving: waits for the ctx's previous frame (if any), enqueues
 * this frame and the device->host copy of its u8 frame into out_u8 (host,
 * pinned for an asynchronous copy; valid after gsr_ctx_finish or the next
 * enqueue on this ctx) and returns.  With two or more contexts a caller keeps
 * several frames in flight, so copies and launch gaps of one frame overlap
 * the kernels of the next. */
GSR_API int gsr_render_enqueue(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
                               const float background[3], int sh_degree, int frustum_cull,
                               uint8_t *out_u8);

/* ---- stage entry points for parity tests (same kernels as gsr_render) ---
 * out_keep (N,) u8; out_order (K,) i64 original indices in depth order
 * (kept[argsort(z[kept], stable)], render.py:279-302); out_packed (K,11) f32
 * in depth order (render.py:448-453); counts are returned in stats. */
GSR_API int gsr_debug_preprocess(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *cam,
                         int sh_degree, int frustum_cull, uint8_t *out_keep,
                         int64_t *out_order, float *out_packed, gsr_stats *stats);
/* Tile lists of the last render on ctx: out_tiles/out_ranks (D,) sorted by
 * (tile, depth rank); out_ranges (n_tiles, 2) [start, end).  Pass NULL to
 * query sizes through stats->tile_keys. */
GSR_API int gsr_debug_tile_lists(gsr_ctx *ctx, int32_t *out_tiles, int32_t *out_ranks,
                         int32_t *out_ranges, gsr_stats *stats);
/* The exact tile-list contract (a depth rank is listed in a
 * tile x tile tile iff some row of the tile row has a non-empty reference
 * interval, render.py:329-333 + 384-397, reaching that tile column) of the
 * last render on ctx, built on the device from 64-bit (tile | rank) keys, a
 * radix sort and per-tile range identification (north_star item 2).  The
 * render path itself blends from conservative 32 x 16 superset lists
 * (gsr_debug_tile_lists); this entry exists so the contract can be compared
 * bit for bit with the reference's rows.  First call (outputs NULL) builds
 * the lists and returns *out_count = D; later calls for the same frame and
 * tile size copy them out: out_tiles/out_ranks (D,) sorted by (tile, rank),
 * out_ranges (n_tiles, 2) [start, end) with n_tiles = ceil(W/tile) *
 * ceil(H/tile).  *out_ms (nullable): device time of the key, sort and range
 * kernels.  1 <= tile <= 256. */
/* Raw device counters of the last frame on ctx, in this order: K, D, P, E,
 * Rb, Rp (gsr_stats), then the blend's instrumentation -- list entries walked
 * by all work items, entries whose row range meets the item's rows, 32-entry
 * batches, composite-loop iterations x 32, useful (pixel, iteration) slots,
 * work items, distinct splats whose colour the blend read; then the splats
 * sorted by the first and second slice (K and 0 for a one-pass frame) and the
 * work items the first slice left unsaturated.  E, Rb and the blend entries
 * need GSR_TIMING_COUNTERS; D and P are summed over the slices. */
#define GSR_NCOUNTERS 16
GSR_API int gsr_debug_frame_counters(gsr_ctx *ctx, uint64_t *out, int n);
/* Per blend work item (tile-major, 8 items of two pixel rows per 32 x 16
 * tile) of the last frame rendered with GSR_TIMING_COUNTERS: the deepest
 * depth rank it walked, | 1 << 31 if all its pixels saturated (T < 1/255). */
GSR_API int gsr_debug_blend_items(gsr_ctx *ctx, uint32_t *out, int64_t n);
GSR_API int gsr_debug_contract_tiles(gsr_ctx *ctx, int tile, int64_t *out_count,
                         int32_t *out_tiles, int32_t *out_ranks, int32_t *out_ranges,
                         float *out_ms);

/* ---- ladder resample: metrics.upscale_to (metrics.py:125-130), Pillow
 * BILINEAR bit-exact.  Host (h,w,3) u8 in, host (H,W,3) u8 out. ---------- */
GSR_API int gsr_resample_bilinear_u8(gsr_ctx *ctx, const uint8_t *src, int src_w, int src_h,
                             uint8_t *dst, int dst_w, int dst_h);

/* ---- SSIM hook: metrics.ssim (metrics.py:76-114).  Two host (H,W,3) u8. -- */
GSR_API int gsr_ssim_u8(gsr_ctx *ctx, const uint8_t *a, const uint8_t *b, int width, int height,
                double *out_ssim);
/* Same on precomputed f64 luma planes (H,W) (metrics.py:69-73 for inputs that
 * are not RGB u8, e.g. grayscale or float images). */
GSR_API int gsr_ssim_luma_f64(gsr_ctx *ctx, const double *x, const double *y, int width,
                              int height, double *out_ssim);

/* ---- JPEG: render.encode_jpeg (render.py:488-498), SURVEY.md 8f row 1 ----
 * Baseline JPEG of an (H,W,3) u8 frame, byte-identical to Pillow 12.2 /
 * libjpeg-turbo (islow DCT, standard Huffman tables, no restart markers):
 * quality 1..100, subsampling 2 (4:2:0) or 0 (4:4:4) as Pillow's
 * subsampling= (render_view uses 4:2:0 below quality 90).  rgb: host frame,
 * or NULL to encode the ctx's last rendered frame in place on the device.
 * *out_len receives the JPEG size; out may be NULL to query it (the encode
 * runs either way), else out_cap must hold *out_len bytes. */
GSR_API int gsr_encode_jpeg(gsr_ctx *ctx, const uint8_t *rgb, int width, int height,
                            int quality, int subsampling, uint8_t *out, size_t out_cap,
                            size_t *out_len);

/* ---- session evaluation: metrics.py:133-214 --------
 * gsr_sse_u8: sum of squared differences of two host u8 buffers of n bytes
 * (metrics.psnr's numerator, metrics.py:57-66; integer, exact).
 * gsr_eval_frame: one evaluation triplet on the device -- renders the ground
 * truth at the base camera (metrics.py:205, the PNG round trip is lossless),
 * uploads the transmitted (th,tw,3) u8 frame, upscale_to's it to the base
 * size (metrics.py:208), and returns ssim(transmitted, gt) and the SSE of the
 * pair (psnr, metrics.py:161-162); out_gt_u8 (nullable) receives the GT. */
GSR_API int gsr_sse_u8(gsr_ctx *ctx, const uint8_t *a, const uint8_t *b, int64_t n,
                       uint64_t *out_sse);
GSR_API int gsr_eval_frame(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *base_cam,
                           const float background[3], int sh_degree, const uint8_t *transmitted,
                           int tw, int th, uint8_t *out_gt_u8, double *out_ssim,
                           uint64_t *out_sse);

/* ---- pinned host memory for end-to-end frame readback ------------------- */
GSR_API int gsr_host_alloc(void **out, size_t bytes);
GSR_API int gsr_host_free(void *ptr);

/* ---- fused ladder evaluation (render_view per rung, render.py:527-541,
 * + upscale_to + ssim vs the base render, metrics.py:205-211), all on
 * device: renders base, then each rung (w[i],h[i]) with rescaled
 * intrinsics, upsamples to base and scores SSIM.  out_ssim[n_rungs]. ---- */
GSR_API int gsr_ladder_ssim(gsr_ctx *ctx, const gsr_scene *scene, const gsr_camera *base_cam,
                    const float background[3], int sh_degree, int n_rungs,
                    const gsr_camera *rung_cams, double *out_ssim, gsr_stats *base_stats);

#ifdef __cplusplus
}
#endif
#endif /* GSR_H */
