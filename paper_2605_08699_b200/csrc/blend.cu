// blend.cu -- K6: per-16x16-tile front-to-back alpha blending.
//
// Restates _composite_kernel's per-pixel arithmetic (render.py:383-427) with
// its exact f32 operation order and glibc expf, so frames are float-identical
// to the reference:
//   dx = (f32(ix) + 0.5) - u
//   power = -0.5 * (((ia*dx)*dx + ((2*ib)*dy)*dx) + (ic*dy)*dy)
//   alpha = min(op * expf(power), 0.99); w = T*alpha; rgb += w*c;
//   T = T*(1 - alpha); the pixel stops once T < 1/255
// and a pixel takes a splat only inside the splat's exact row interval
// [floor(mid - span), ceil(mid + span) + 1) of render.py:384-397 and row range
// render.py:329-333 -- the tile lists are a superset, so order and set of
// contributions per pixel are the reference's.  After the list: rgb += T*bg
// (render.py:423-427), then the u8 conversion of render.py:470+484-485.
//
// Layout: one CTA per tile, 8 warps; warp w owns pixel rows 2w, 2w+1 of the
// tile (lane & 15 = column, lane >> 4 = row).  A warp walks the tile list 32
// splats at a time: lane j loads splat j's record (128-bit loads), computes
// the two row intervals as a 32-bit coverage mask, then the warp iterates the
// ballot of non-empty masks in depth order.  Warps leave as soon as all their
// 32 pixels are saturated (warp-ballot early termination); no block barriers
// in the loop.
#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int kBlendThreads = 256;

__device__ __forceinline__ uint32_t span_mask(int x0, int x1, int X) {
    // columns [x0, x1) intersected with [X, X+16), as a 16-bit mask
    int a = x0 - X, b = x1 - X;
    a = a < 0 ? 0 : a;
    b = b > 16 ? 16 : b;
    if (a >= b) return 0u;
    return ((1u << b) - 1u) & ~((1u << a) - 1u);
}

__global__ void __launch_bounds__(kBlendThreads) blend_kernel(
    const SplatRec *__restrict__ srec, const uint32_t *__restrict__ tile_vals,
    const uint2 *__restrict__ ranges, int width, int height, float bg0, float bg1, float bg2,
    BlendOut out) {
    __shared__ unsigned long long s_tab[32];
    __shared__ float4 s_rec[kBlendThreads / 32][32][3];
    if (threadIdx.x < 32) s_tab[threadIdx.x] = kExp2fTab[threadIdx.x];
    __syncthreads();

    const int tiles_x = (width + kTile - 1) / kTile;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int X = tx * kTile;
    const int iy0 = ty * kTile + 2 * w;
    const int iy = iy0 + (lane >> 4);
    const int ix = X + (lane & 15);
    const bool inside = ix < width && iy < height;
    const float py0 = (float)iy0 + 0.5f, py1 = (float)(iy0 + 1) + 0.5f;
    const float py = (float)iy + 0.5f;
    const float fx = (float)ix + 0.5f;

    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    const uint2 rg = ranges[blockIdx.x];
    float4(*my)[3] = s_rec[w];

    for (uint32_t c = rg.x; c < rg.y; c += 32) {
        if (__all_sync(0xffffffffu, done)) break;
        const uint32_t j = c + lane;
        uint32_t mask = 0;
        if (j < rg.y) {
            const uint32_t r = __ldg(tile_vals + j);  // depth rank
            const float4 A = __ldg(&srec[r].a);
            const float4 B = __ldg(&srec[r].b);
            const float4 C = __ldg(&srec[r].c);
            int lo, hi;
            row_range(A.y, B.w, height, lo, hi);
            int x0, x1;
            if (iy0 >= lo && iy0 < hi &&
                row_interval(A.x, A.y, A.z, A.w, B.x, B.y, py0, width, x0, x1))
                mask = span_mask(x0, x1, X);
            if (iy0 + 1 >= lo && iy0 + 1 < hi &&
                row_interval(A.x, A.y, A.z, A.w, B.x, B.y, py1, width, x0, x1))
                mask |= span_mask(x0, x1, X) << 16;
            my[lane][0] = A;
            my[lane][1] = B;
            my[lane][2] = C;
        }
        __syncwarp();
        uint32_t act = __ballot_sync(0xffffffffu, mask != 0u);
        while (act) {
            const int src = __ffs(act) - 1;
            act &= act - 1u;
            const uint32_t mk = __shfl_sync(0xffffffffu, mask, src);
            if (((mk >> lane) & 1u) && !done) {
                const float4 A = my[src][0];
                const float4 B = my[src][1];
                const float4 C = my[src][2];
                const float u = A.x, v = A.y, ia = A.z, ib = A.w, ic = B.x, op = B.z;
                const float dy = py - v;
                const float cy_term = ic * dy * dy;
                const float ib_dy = 2.0f * ib * dy;
                const float dx = fx - u;
                const float power = -0.5f * (ia * dx * dx + ib_dy * dx + cy_term);
                float alpha = op * glibc_expf_tab(power, s_tab);
                if (alpha > kAlphaMax) alpha = kAlphaMax;
                const float weight = T * alpha;
                cr += weight * C.x;
                cg += weight * C.y;
                cb += weight * C.z;
                T = T * (1.0f - alpha);
                if (T < kTStop) done = true;
            }
        }
        __syncwarp();
    }
    if (!inside) return;
    cr += T * bg0;
    cg += T * bg1;
    cb += T * bg2;
    const int64_t p = (int64_t)iy * width + ix;
    if (out.rgb) {
        out.rgb[3 * p + 0] = cr;
        out.rgb[3 * p + 1] = cg;
        out.rgb[3 * p + 2] = cb;
    }
    if (out.trans) out.trans[p] = T;
    // render.py:470 + 484-485: trunc(clip(clip(f64(c), 0, 1) * 255 + 0.5, 0, 255))
    const float ch[3] = {cr, cg, cb};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        double d = (double)ch[k];
        d = d < 0.0 ? 0.0 : (d > 1.0 ? 1.0 : d);
        double s = d * 255.0 + 0.5;
        s = s < 0.0 ? 0.0 : (s > 255.0 ? 255.0 : s);
        out.u8[3 * p + k] = (uint8_t)(int)s;
    }
}

}  // namespace

void launch_blend(const SplatRec *srec, const uint32_t *tile_vals, const uint2 *ranges, int width,
                  int height, float bg0, float bg1, float bg2, BlendOut out, cudaStream_t s) {
    const int tiles = ((width + kTile - 1) / kTile) * ((height + kTile - 1) / kTile);
    blend_kernel<<<tiles, kBlendThreads, 0, s>>>(srec, tile_vals, ranges, width, height, bg0, bg1,
                                                 bg2, out);
}

}  // namespace gsr
