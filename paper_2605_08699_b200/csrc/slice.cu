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
//      most tau, tau chosen from a histogram of the kept depths (built by
//      preprocess_geo) so the slice holds about a fraction f of them.  It is sorted,
//      coloured, binned and blended like a whole frame; a work item (two
//      pixel rows of a 32 x 16 tile) whose pixels all saturate writes its
//      final pixels, any other item saves its pixels' (T, r, g, b) and sets
//      its bit in the unsaturated-item bitmask.
//   B  the rest: a splat behind the slice is kept only if its conservative
//      box in item rows x tile columns (item_box: the reference's row range,
//      the whole splat's column extent) meets an unsaturated item (blend A
//      sets its bit in a column-major bitmask -- per tile column, one bit per
//      item row -- so a box's rows in a column are one or two masked words);
//      those are sorted, coloured, binned and blended from the saved state,
//      by the unsaturated items only.
// Ties in the span key never straddle the slices (the split is on the key),
// so A's order followed by B's is the global stable depth order, and each
// unsaturated pixel sees every splat covering it in the reference's order:
// frames are bit-identical to the one-pass render (tests/test_gpu_parity.py
// compares both paths and the oracle).
#include <algorithm>

#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

// tau: the span key of the end of the smallest prefix of depth bins
// (preprocess_geo's histogram of the kept depths' f64 bits) holding >= frac
// * K splats.  Any tau gives the same frame (the split is on the span key,
// so ties never straddle the slices); it only sets the work split.  The
// slice's size KA is counted by the depth sort's histogram kernel.
__global__ void __launch_bounds__(kZBins) slice_plan_kernel(FrameCounters *ctr, float frac,
                                                            uint32_t *zero0, int n0,
                                                            uint32_t *zero1, int n1) {
    __shared__ uint32_t s_warp[33];
    // buffers the frame's next kernels need cleared (the unsaturated-item
    // bitmask, slice A's sort histograms): no memset nodes in the graph
    for (int j = threadIdx.x; j < n0; j += blockDim.x) zero0[j] = 0u;
    for (int j = threadIdx.x; j < n1; j += blockDim.x) zero1[j] = 0u;
    const uint32_t c = ctr->slice_hist[threadIdx.x];
    uint32_t tot;
    const uint32_t ex = block_excl_scan_u32(c, s_warp, &tot);
    const uint32_t inc = ex + c;
    uint32_t target = (uint32_t)ceilf(frac * (float)tot);
    target = target < 1u ? 1u : target;
    if (inc >= target && ex < target) {  // the first bin whose prefix reaches the target
        const int b = (int)threadIdx.x;
        const unsigned long long end =
            b == kZBins - 1 ? ~0ull - 1ull
                            : ((unsigned long long)(b + 1 + kZBinBase) << kZBinShift) - 1ull;
        const unsigned long long kmin = ctr->kmin;
        ctr->tau = end < kmin ? 0u : span_key(span_map(kmin, ctr->kmax), end);
    }
    if (tot == 0u && threadIdx.x == 0) ctr->tau = 0u;
}

// Splats behind the slice that may reach an unsaturated item, appended as
// (span key, Gaussian index).  The append order depends on scheduling; the
// sort and the fix-up order by (span key, f64 key, index), so the order of
// the slice does not.
#ifndef GSR_FILTER_ITEMS
#define GSR_FILTER_ITEMS 4
#endif
constexpr int kFilterItems = GSR_FILTER_ITEMS;  // Gaussians per thread: all loads in flight at once
constexpr int kFilterSmemWords = 12288;         // bitmask staged in shared memory up to 48 KB

// Membership of one box in the unsaturated-item bitmask `cols` ([tiles_x]
// [col_words], column-major): per tile column c0..c1, the box's rows
// [r0, r1] are words w0..w1 (one for all but tall splats), masked at both
// ends.  The words are OR-ed without an early exit, so the loads are
// independent (most splats behind the slice are not members: the whole box
// is read either way).
__device__ __forceinline__ bool box_member(const uint32_t *cols, int col_words, uint2 bx) {
    const uint32_t r0 = bx.x & 0xffffu, r1 = bx.x >> 16;
    const uint32_t c0 = bx.y & 0xffffu, c1 = bx.y >> 16;
    if (r0 > r1 || c0 > c1) return false;
    const uint32_t w0 = r0 >> 5, w1 = r1 >> 5;
    const uint32_t mlo = ~0u << (r0 & 31), mhi = ~0u >> (31 - (r1 & 31));
    uint32_t acc = 0u;
    const uint32_t *p = cols + c0 * (uint32_t)col_words + w0;
    if (w0 == w1) {
        const uint32_t mm = mlo & mhi;
        for (uint32_t c = c0; c <= c1; c++, p += col_words) acc |= *p & mm;
    } else {
        for (uint32_t c = c0; c <= c1; c++, p += col_words) {
            acc |= p[0] & mlo;
            for (uint32_t w = 1; w < w1 - w0; w++) acc |= p[w];
            acc |= p[w1 - w0] & mhi;
        }
    }
    return acc != 0u;
}

// Persistent: each CTA stages the bitmask in shared memory once (4 KB at
// 1080p), then takes blocks of 256 x kFilterItems Gaussians.
template <bool kSmem>
__global__ void __launch_bounds__(256) slice_b_filter_kernel(SliceBArgs a) {
    extern __shared__ uint32_t s_cols[];
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t s_base;
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) a.ctr->blend_next = 0u;  // blend A has finished
        // slice B's sort histograms (slice A's sort is long done)
        for (int j = threadIdx.x; j < a.zero_words; j += blockDim.x) a.zero[j] = 0u;
    }
    if (a.ctr->n_unsat == 0u) return;  // (block-uniform)
    const uint32_t *cols = a.unsat_cols;
    if (kSmem) {
        const int nw = a.tiles_x * a.col_words;
        for (int j = threadIdx.x; j < nw; j += blockDim.x) s_cols[j] = __ldg(a.unsat_cols + j);
        __syncthreads();
        cols = s_cols;
    }
    const SpanMap m = span_map(a.ctr->kmin, a.ctr->kmax);
    const uint32_t tau = a.ctr->tau;
    const int64_t step = (int64_t)gridDim.x * (256 * kFilterItems);
    for (int64_t i0 = (int64_t)blockIdx.x * (256 * kFilterItems) + threadIdx.x;
         i0 - threadIdx.x < a.n; i0 += step) {
        // keys and item boxes in one round of loads (a box is only used when
        // its splat lies behind the front slice; culled splats' boxes are
        // never read as members)
        unsigned long long k64[kFilterItems];
        uint2 bx[kFilterItems];
#pragma unroll
        for (int k = 0; k < kFilterItems; k++) {
            const int64_t i = i0 + k * 256;
            k64[k] = i < a.n ? __ldg(a.keys64 + i) : ~0ull;
            bx[k] = i < a.n ? __ldg(a.ibox + i) : make_uint2(0xffffu, 0u);
        }
        uint32_t k32[kFilterItems];
        uint32_t memb = 0u;
#pragma unroll
        for (int k = 0; k < kFilterItems; k++) {
            k32[k] = k64[k] != ~0ull ? span_key(m, k64[k]) : 0u;
            // behind the front slice, and its box (item_box, written by
            // preprocess_geo) meets an unsaturated item
            if (k64[k] != ~0ull && k32[k] > tau && box_member(cols, a.col_words, bx[k]))
                memb |= 1u << k;
        }
        // block-aggregated append: one atomic per 1024 Gaussians
        uint32_t tot;
        uint32_t pos = block_excl_scan_u32((uint32_t)__popc(memb), s_warp, &tot);
        if (threadIdx.x == 0) s_base = tot ? atomicAdd(&a.ctr->KB, tot) : 0u;
        __syncthreads();
        pos += s_base;
#pragma unroll
        for (int k = 0; k < kFilterItems; k++)
            if ((memb >> k) & 1u) {
                a.keysB[pos] = k32[k];
                a.valsB[pos] = (uint32_t)(i0 + k * 256);
                pos++;
            }
        __syncthreads();  // s_base / s_warp reused by the next block step
    }
}

__global__ void slice_b_decide_kernel(const FrameCounters *ctr,
                                      cudaGraphConditionalHandle handle, uint32_t *class_count) {
    const uint32_t kb = ctr->KB;
    unsigned int v = kSliceClasses;  // no body: slice B is empty
    if (kb > 0) {
        v = kSliceClasses - 1;
        for (int c = kSliceClasses - 2; c >= 0; c--)
            if ((int64_t)kb <= slice_class_cap(c)) v = (unsigned int)c;
    }
    cudaGraphSetConditional(handle, v);
    class_count[v] += 1u;  // kernel-launch accounting (single thread)
}

}  // namespace

void launch_slice_plan(FrameCounters *ctr, float frac, uint32_t *zero0, int n0, uint32_t *zero1,
                       int n1, cudaStream_t s, const KMark &mark) {
    slice_plan_kernel<<<1, kZBins, 0, s>>>(ctr, frac, zero0, n0, zero1, n1);
    mark("slice_plan");
}

void launch_slice_b_filter(const SliceBArgs &a, cudaStream_t s, const KMark &mark) {
    if (a.n <= 0) return;
    static int sms = 0;  // (one device model per process)
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
        cudaFuncSetAttribute(slice_b_filter_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kFilterSmemWords * sizeof(uint32_t)));
    }
#ifndef GSR_FILTER_CTAS
#define GSR_FILTER_CTAS 16
#endif
    const unsigned blocks = (unsigned)std::min<int64_t>(
        (a.n + 256 * kFilterItems - 1) / (256 * kFilterItems), (int64_t)sms * GSR_FILTER_CTAS);
    const int64_t words = (int64_t)a.tiles_x * a.col_words;
    if (words <= kFilterSmemWords)
        slice_b_filter_kernel<true><<<blocks, 256, words * sizeof(uint32_t), s>>>(a);
    else
        slice_b_filter_kernel<false><<<blocks, 256, 0, s>>>(a);
    mark("slice_b_filter");
}

void launch_slice_b_decide(const FrameCounters *ctr, cudaGraphConditionalHandle handle,
                           uint32_t *class_count, cudaStream_t s) {
    slice_b_decide_kernel<<<1, 1, 0, s>>>(ctr, handle, class_count);
}

}  // namespace gsr
