// resample.cu -- K7: ABR-ladder resample, Pillow Image.resize(BILINEAR) on
// RGB u8 as called by metrics.upscale_to (metrics.py:125-130).
//
// Pillow (third-party, 12.2.0; libImaging/Resample.c) works in 22-bit fixed
// point: per output coordinate a window [xmin, xmin + xlen) of int32
// coefficients (computed on the host by gsr_api.cu exactly as Pillow's
// precompute_coeffs + normalize_coeffs_8bpc do), accumulator starting at
// 1 << 21, result clip8(acc >> 22).  Horizontal pass first (only the source
// rows the vertical pass needs), then vertical, u8 intermediate.  Integer
// arithmetic: bit-exact by construction.
#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int kPrecisionBits = 22;

__device__ __forceinline__ uint8_t clip8(int32_t v) {
    v >>= kPrecisionBits;
    return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

__global__ void resample_h_kernel(const uint8_t *__restrict__ src, int sw, int row0,
                                  uint8_t *__restrict__ dst, int dw, int rows, ResampleAxis ax) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= dw || y >= rows) return;
    const int xmin = ax.bounds[2 * x], xlen = ax.bounds[2 * x + 1];
    const int32_t *k = ax.coefs + (int64_t)x * ax.ksize;
    const uint8_t *row = src + ((int64_t)(row0 + y) * sw + xmin) * 3;
    int32_t s0 = 1 << (kPrecisionBits - 1), s1 = s0, s2 = s0;
    for (int t = 0; t < xlen; t++) {
        const int32_t c = __ldg(k + t);
        s0 += (int32_t)row[3 * t + 0] * c;
        s1 += (int32_t)row[3 * t + 1] * c;
        s2 += (int32_t)row[3 * t + 2] * c;
    }
    uint8_t *o = dst + ((int64_t)y * dw + x) * 3;
    o[0] = clip8(s0);
    o[1] = clip8(s1);
    o[2] = clip8(s2);
}

__global__ void resample_v_kernel(const uint8_t *__restrict__ src, int w,
                                  uint8_t *__restrict__ dst, int dh, ResampleAxis ax) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= w || y >= dh) return;
    const int ymin = ax.bounds[2 * y], ylen = ax.bounds[2 * y + 1];
    const int32_t *k = ax.coefs + (int64_t)y * ax.ksize;
    int32_t s0 = 1 << (kPrecisionBits - 1), s1 = s0, s2 = s0;
    for (int t = 0; t < ylen; t++) {
        const int32_t c = __ldg(k + t);
        const uint8_t *p = src + ((int64_t)(ymin + t) * w + x) * 3;
        s0 += (int32_t)p[0] * c;
        s1 += (int32_t)p[1] * c;
        s2 += (int32_t)p[2] * c;
    }
    uint8_t *o = dst + ((int64_t)y * w + x) * 3;
    o[0] = clip8(s0);
    o[1] = clip8(s1);
    o[2] = clip8(s2);
}

}  // namespace

void launch_resample_h(const uint8_t *src, int sw, int row0, uint8_t *dst, int dw, int rows,
                       ResampleAxis ax, cudaStream_t s) {
    if (dw <= 0 || rows <= 0) return;
    dim3 grid((dw + 127) / 128, rows);
    resample_h_kernel<<<grid, 128, 0, s>>>(src, sw, row0, dst, dw, rows, ax);
}

void launch_resample_v(const uint8_t *src, int w, uint8_t *dst, int dh, ResampleAxis ax,
                       cudaStream_t s) {
    if (w <= 0 || dh <= 0) return;
    dim3 grid((w + 127) / 128, dh);
    resample_v_kernel<<<grid, 128, 0, s>>>(src, w, dst, dh, ax);
}

}  // namespace gsr
