// kernels.cuh -- launch interfaces of the render-path kernels (internal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace gsr {

// Per-frame device counters (one struct, reset by frame_init_kernel).
struct FrameCounters {
    uint32_t K;                 // kept splats
    uint32_t D;                 // tile keys under the contract (may exceed capacity)
    uint32_t npass;             // depth-sort radix passes
    uint32_t pad0;
    unsigned long long kmin;    // min / max kept depth key (f64 bits)
    unsigned long long kmax;
    unsigned long long bin_ticket;  // block tickets of the binning kernel
};

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
    const void *sh;       // [48][stride] f32 or f64, coefficient-major (k*3 + c)
    int sh_f32;
};

struct CameraArgs {
    double r[9];
    double t[3];
    double campos[3];
    double fx, fy, cx, cy;
    double width, height;
    int iwidth, iheight;
};

// preprocess.cu
void launch_frame_init(FrameCounters *ctr, cudaStream_t s);
void launch_preprocess(const SceneView &scene, const CameraArgs &cam, int sh_degree,
                       int frustum_cull, unsigned long long *keys, SplatRec *rec,
                       uint8_t *keep_out, FrameCounters *ctr, cudaStream_t s);
void launch_depth_passes(FrameCounters *ctr, cudaStream_t s);

// radix.cu
struct ScanWorkspace {
    uint32_t *partials;
    int64_t partial_cap;
};
int64_t scan_partials_needed(int64_t n);
cudaError_t radix_init_attributes();
void launch_scan_exclusive(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *total,
                           const ScanWorkspace &ws, cudaStream_t s);

constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;
inline int64_t radix_tiles(int64_t n_cap) { return (n_cap + kRadixTile - 1) / kRadixTile; }

// One stable LSD pass over 8 bits at `shift` of (key - key_base).
//  n = min(*n_dev, n_cap) (n_dev nullable -> n_cap).
//  vin == nullptr -> value = input index.  drop_sentinel: keys == ~0 are
//  removed (the order-preserving compaction of render.py:279).
//  The pass is a no-op when pass_index >= *npass_dev (npass_dev nullable).
template <typename K>
void launch_radix_pass(const K *kin, const uint32_t *vin, K *kout, uint32_t *vout,
                       const uint32_t *n_dev, int64_t n_cap, int shift,
                       const unsigned long long *key_base, const uint32_t *npass_dev,
                       int pass_index, bool drop_sentinel, uint32_t *hist,
                       const ScanWorkspace &ws, cudaStream_t s);

// binning.cu: fused gather + tile-list generation (one kernel, look-back scan)
int64_t bin_status_words(int64_t n_cap);
void launch_bin(const uint32_t *vals_even, const uint32_t *vals_odd, const SplatRec *rec,
                SplatRec *srec, int64_t n_cap, FrameCounters *ctr, int width, int height,
                uint32_t *tile_keys, uint32_t *tile_vals, int64_t cap_d,
                unsigned long long *status, uint32_t *overflow_sticky, cudaStream_t s);
void launch_tile_ranges(const uint32_t *tile_keys, const FrameCounters *ctr, int64_t cap_d,
                        uint2 *ranges, int n_tiles, int sms, cudaStream_t s);

// blend.cu
struct BlendOut {
    uint8_t *u8;    // (H,W,3)
    float *rgb;     // (H,W,3) or null
    float *trans;   // (H,W) or null
};
void launch_blend(const SplatRec *srec, const uint32_t *tile_vals, const uint2 *ranges,
                  int width, int height, float bg0, float bg1, float bg2, BlendOut out,
                  cudaStream_t s);

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
void launch_ssim(const SsimInput &in, int width, int height, const double *weights11,
                 double *partials, uint32_t *neq, double *out, cudaStream_t s);

}  // namespace gsr
