// slice.cu -- depth-sliced frames: sort, colour, bin and blend only the splats
// that can reach an unsaturated pixel.
//
// The reference composites every pixel front to back and stops once its
// transmittance falls below 1/255 (render.py:405-421); nothing behind that
// point changes the pixel.  At config 3 the blend reads the colour of only
// 3.6 % of the kept splats, and 99.9 % of the work items that saturate do
// so within the front 10 % of the depth order (profiles/
// r02_blend_instrumentation.json).  So a frame is rendered in two passes
// over one global depth order:
//   A  the front slice: kept splats whose 24-bit span key (depth.cu) is at
//      most tau, tau chosen from a histogram of the keys' top 8 bits so the
//      slice holds about a fraction f of the kept splats.  It is sorted,
//      coloured, binned and blended like a whole frame; a work item (two
//      pixel rows of a 32 x 64 tile) whose pixels all saturate writes its
//      final pixels, any other item saves its pixels' (T, r, g, b) and sets
//      its bit in unsat[tile].
//   B  the rest: a splat behind the slice is kept only if its conservative
//      column span (band_span_bound, the binning's own bound) meets a tile
//      row band holding an unsaturated item; those are sorted, coloured,
//      binned and blended from the saved state, by the unsaturated items only.
// Ties in the span key never straddle the slices (the split is on the key),
// so A's order followed by B's is the global stable depth order, and each
// unsaturated pixel sees every splat covering it in the reference's order:
// frames are bit-identical to the one-pass render (tests/test_gpu_parity.py
// compares both paths and the oracle).
#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

// top 8 bits of the span keys of the kept splats
__global__ void __launch_bounds__(256) slice_hist_kernel(const unsigned long long *__restrict__ keys64,
                                                         int64_t n, FrameCounters *ctr) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const SpanMap m = span_map(ctr->kmin, ctr->kmax);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = __ldg(keys64 + i);
        if (k != ~0ull) atomicAdd(&h[span_key(m, k) >> (kSpanKeyBits - 8)], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&ctr->slice_hist[threadIdx.x], h[threadIdx.x]);
}

// tau = the end of the smallest top-digit prefix holding >= frac * K splats
__global__ void __launch_bounds__(256) slice_plan_kernel(FrameCounters *ctr, float frac) {
    __shared__ uint32_t s_warp[33];
    const uint32_t c = ctr->slice_hist[threadIdx.x];
    uint32_t tot;
    const uint32_t ex = block_excl_scan_u32(c, s_warp, &tot);
    const uint32_t inc = ex + c;
    uint32_t target = (uint32_t)ceilf(frac * (float)tot);
    target = target < 1u ? 1u : target;
    // the first digit whose inclusive prefix reaches the target
    if (inc >= target && ex < target) {
        ctr->tau = ((uint32_t)threadIdx.x << (kSpanKeyBits - 8)) |
                   ((1u << (kSpanKeyBits - 8)) - 1u);
        ctr->KA = inc;
    }
    if (tot == 0u && threadIdx.x == 0) {
        ctr->tau = 0u;
        ctr->KA = 0u;
    }
}

// Splats behind the slice that may reach an unsaturated item, appended as
// (span key, Gaussian index).  The append order depends on scheduling; the
// sort and the fix-up order by (span key, f64 key, index), so the order of
// the slice does not.
__global__ void __launch_bounds__(256) slice_b_filter_kernel(SliceBArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) a.ctr->blend_next = 0u;  // blend A has finished (stream order)
    bool member = false;
    uint32_t out = 0xffffffffu;
    if (i < a.n && a.ctr->n_unsat) {
        const unsigned long long k64 = __ldg(a.keys64 + i);
        if (k64 != ~0ull) {
            const SpanMap m = span_map(a.ctr->kmin, a.ctr->kmax);
            const uint32_t k32 = span_key(m, k64);
            if (k32 > a.ctr->tau) {
                const float4 A = __ldg(&a.geo[i].a), B = __ldg(&a.geo[i].b);
                int lo, hi;
                row_range(A.y, B.w, a.height, lo, hi);
                for (int ty = lo / kTileH; lo < hi && ty <= (hi - 1) / kTileH && !member; ty++) {
                    const int y0 = max(lo, ty * kTileH), y1 = min(hi, ty * kTileH + kTileH);
                    // items (pixel-row pairs) of this tile row the splat's rows meet
                    const int w0 = (y0 - ty * kTileH) / 2, w1 = (y1 - 1 - ty * kTileH) / 2;
                    const uint32_t im = (w1 >= 31 ? 0xffffffffu : (2u << w1) - 1u) &
                                        ~((1u << w0) - 1u);
                    int mn = 0, mx = a.width;
                    if (!band_span_bound(A.x, A.y, A.z, A.w, B.x, B.y, y0, y1, a.width, mn, mx)) {
                        mn = 0;  // ill-conditioned: every column (conservative)
                        mx = a.width;
                    }
                    mn = max(mn, 0);
                    mx = min(mx, a.width);
                    if (mn >= mx) continue;
                    const uint32_t *row = a.unsat + (int64_t)ty * a.tiles_x;
                    for (int tx = mn / kTileW; tx <= (mx - 1) / kTileW; tx++)
                        if (row[tx] & im) {
                            member = true;
                            break;
                        }
                }
                if (member) out = k32;
            }
        }
    }
    // warp-aggregated append
    const uint32_t ballot = __ballot_sync(0xffffffffu, member);
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == 0 && ballot) base = atomicAdd(&a.ctr->KB, (uint32_t)__popc(ballot));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (member) {
        const uint32_t pos = base + __popc(ballot & ((1u << lane) - 1u));
        a.keysB[pos] = out;
        a.valsB[pos] = (uint32_t)i;
    }
}

__global__ void slice_b_decide_kernel(const FrameCounters *ctr,
                                      cudaGraphConditionalHandle handle) {
    const uint32_t kb = ctr->KB;
    unsigned int v = kSliceClasses;  // no body: slice B is empty
    if (kb > 0) {
        v = kSliceClasses - 1;
        for (int c = kSliceClasses - 2; c >= 0; c--)
            if ((int64_t)kb <= slice_class_cap(c)) v = (unsigned int)c;
    }
    cudaGraphSetConditional(handle, v);
}

}  // namespace

void launch_slice_plan(const unsigned long long *keys64, int64_t n, FrameCounters *ctr,
                       float frac, int sms, cudaStream_t s, const KMark &mark) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    if (blocks < 1) blocks = 1;
    slice_hist_kernel<<<(unsigned)blocks, 256, 0, s>>>(keys64, n, ctr);
    mark("slice_hist");
    slice_plan_kernel<<<1, 256, 0, s>>>(ctr, frac);
    mark("slice_plan");
}

void launch_slice_b_filter(const SliceBArgs &a, cudaStream_t s, const KMark &mark) {
    if (a.n <= 0) return;
    slice_b_filter_kernel<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a);
    mark("slice_b_filter");
}

void launch_slice_b_decide(const FrameCounters *ctr, cudaGraphConditionalHandle handle,
                           cudaStream_t s) {
    slice_b_decide_kernel<<<1, 1, 0, s>>>(ctr, handle);
}

}  // namespace gsr
