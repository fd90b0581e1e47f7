// ssim.cu -- K8: windowed SSIM, metrics.ssim (metrics.py:76-114).
//
// Luma = ((r*0.299 + g*0.587) + b*0.114) in f64 (metrics.py:69-73); five maps
// x, y, x^2, y^2, xy filtered with scipy.ndimage.gaussian_filter (sigma 1.5,
// radius 5, mode "nearest"): along axis 0 then axis 1, each as scipy's
// symmetric correlate1d (centre tap, then tap pairs from the outside in);
// SSIM map of metrics.py:106-107 with c1 = (0.01*255)^2, c2 = (0.03*255)^2;
// mean over the core [5:-5, 5:-5] (metrics.py:109-110).  Core pixels never
// touch the "nearest" padding, so each CTA filters a 32x8 output tile from a
// 42x18 shared-memory halo.  All f64; the CTA partial sums are reduced in a
// fixed order, so the result is deterministic.  Exact luma equality returns
// 1.0 (metrics.py:92-93).
#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int TW = 32, TH = 8, R = 5;
constexpr int HW = TW + 2 * R, HH = TH + 2 * R;  // 42 x 18

__device__ __forceinline__ double luma(const uint8_t *p) {
    return ((double)p[0] * 0.299 + (double)p[1] * 0.587) + (double)p[2] * 0.114;
}

__device__ __forceinline__ double pix(const SsimInput &in, bool first, int64_t i) {
    if (in.la) return first ? in.la[i] : in.lb[i];
    return luma((first ? in.a : in.b) + 3 * i);
}

__global__ void __launch_bounds__(256) ssim_tile_kernel(SsimInput in, int width, int height,
                                                        const double *__restrict__ wts,
                                                        double *__restrict__ partials) {
    __shared__ double sx[HH][HW], sy[HH][HW];
    __shared__ double v[5][TH][HW];
    __shared__ double fw[11];
    __shared__ double red[8];
    if (threadIdx.x < 11) fw[threadIdx.x] = wts[threadIdx.x];
    const int x0 = R + blockIdx.x * TW, y0 = R + blockIdx.y * TH;  // first core output
    for (int i = threadIdx.x; i < HH * HW; i += blockDim.x) {
        const int hy = i / HW, hx = i % HW;
        int gy = y0 - R + hy, gx = x0 - R + hx;
        gy = gy < 0 ? 0 : (gy > height - 1 ? height - 1 : gy);
        gx = gx < 0 ? 0 : (gx > width - 1 ? width - 1 : gx);
        const int64_t o = (int64_t)gy * width + gx;
        sx[hy][hx] = pix(in, true, o);
        sy[hy][hx] = pix(in, false, o);
    }
    __syncthreads();
    // axis 0 (vertical) for the TH output rows over all HW halo columns
    for (int i = threadIdx.x; i < TH * HW; i += blockDim.x) {
        const int ty = i / HW, hx = i % HW;
        const int c = ty + R;
        double ax = sx[c][hx], ay = sy[c][hx];
        double m0 = ax * fw[5], m1 = ay * fw[5], m2 = (ax * ax) * fw[5], m3 = (ay * ay) * fw[5],
               m4 = (ax * ay) * fw[5];
#pragma unroll
        for (int j = -R; j < 0; j++) {
            const double xa = sx[c + j][hx], xb = sx[c - j][hx];
            const double ya = sy[c + j][hx], yb = sy[c - j][hx];
            const double f = fw[5 + j];
            m0 += (xa + xb) * f;
            m1 += (ya + yb) * f;
            m2 += (xa * xa + xb * xb) * f;
            m3 += (ya * ya + yb * yb) * f;
            m4 += (xa * ya + xb * yb) * f;
        }
        v[0][ty][hx] = m0;
        v[1][ty][hx] = m1;
        v[2][ty][hx] = m2;
        v[3][ty][hx] = m3;
        v[4][ty][hx] = m4;
    }
    __syncthreads();
    // axis 1 (horizontal) + SSIM map for this thread's output pixel
    const int ty = threadIdx.x / TW, txx = threadIdx.x % TW;
    const int gx = x0 + txx, gy = y0 + ty;
    double val = 0.0;
    if (gx < width - R && gy < height - R) {
        const int c = txx + R;
        double f[5];
#pragma unroll
        for (int m = 0; m < 5; m++) {
            double acc = v[m][ty][c] * fw[5];
#pragma unroll
            for (int j = -R; j < 0; j++) acc += (v[m][ty][c + j] + v[m][ty][c - j]) * fw[5 + j];
            f[m] = acc;
        }
        const double mux = f[0], muy = f[1];
        const double sgx = f[2] - mux * mux;
        const double sgy = f[3] - muy * muy;
        const double sgxy = f[4] - mux * muy;
        const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
        const double c2 = (0.03 * 255.0) * (0.03 * 255.0);
        val = ((2 * mux * muy + c1) * (2 * sgxy + c2)) /
              ((mux * mux + muy * muy + c1) * (sgx + sgy + c2));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = val;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < 8; k++) s += red[k];
        partials[blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
}

__global__ void luma_neq_kernel(SsimInput in, int64_t npx, uint32_t *neq) {
    uint32_t c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npx;
         i += (int64_t)gridDim.x * blockDim.x)
        c += pix(in, true, i) != pix(in, false, i);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(neq, c);
}

__global__ void ssim_final_kernel(const double *__restrict__ partials, int n, const uint32_t *neq,
                                  double count, double *out) {
    __shared__ double red[32];
    double s = 0.0;
    // fixed assignment of partials to threads and fixed tree: deterministic
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++) t += red[k];
        *out = (*neq == 0u) ? 1.0 : t / count;
    }
}

// Sum of squared differences of two u8 buffers (metrics.psnr's numerator,
// metrics.py:57-66): integer, so the result is exact whatever the order.
__global__ void __launch_bounds__(256) sse_kernel(const uint8_t *__restrict__ a,
                                                  const uint8_t *__restrict__ b, int64_t n,
                                                  unsigned long long *out) {
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)a[i] - (int)b[i];
        s += (unsigned long long)(d * d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

}  // namespace

void launch_sse(const uint8_t *a, const uint8_t *b, int64_t n, unsigned long long *out,
                cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
    const int64_t blocks = (n + 255) / 256;
    sse_kernel<<<(unsigned)(blocks < 1184 ? (blocks > 0 ? blocks : 1) : 1184), 256, 0, s>>>(a, b, n, out);
}

int ssim_partials_needed(int width, int height) {
    const int gx = (width - 2 * R + TW - 1) / TW, gy = (height - 2 * R + TH - 1) / TH;
    return gx * gy;
}

void launch_ssim(const SsimInput &in, int width, int height, const double *weights11,
                 double *partials, uint32_t *neq, double *out, cudaStream_t s) {
    const int gx = (width - 2 * R + TW - 1) / TW, gy = (height - 2 * R + TH - 1) / TH;
    cudaMemsetAsync(neq, 0, sizeof(uint32_t), s);
    const int64_t npx = (int64_t)width * height;
    luma_neq_kernel<<<(unsigned)((npx + 255) / 256 < 1184 ? (npx + 255) / 256 : 1184), 256, 0, s>>>(
        in, npx, neq);
    ssim_tile_kernel<<<dim3(gx, gy), 256, 0, s>>>(in, width, height, weights11, partials);
    const double count = (double)(height - 2 * R) * (double)(width - 2 * R);
    ssim_final_kernel<<<1, 1024, 0, s>>>(partials, gx * gy, neq, count, out);
}

}  // namespace gsr
