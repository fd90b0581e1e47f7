// depth.cu -- K3: the stable f64 depth order of sort_splats (render.py:293-302,
// np.argsort(depths, kind="stable") over the kept splats, render.py:279).
//
// Exact order needs the full f64 keys (f32 keys misorder 22% of positions at
// 3M Gaussians), but 8 radix passes over 64-bit keys are mostly wasted: the
// kept depths span [kmin, kmax] and are nearly all distinct at 32-bit
// resolution of that span.  So:
//  1 key32   k32 = min((bits(z) - kmin) >> shift, 2^24 - 1), shift chosen so
//            the span fits 24 bits; culled Gaussians keep the sentinel ~0
//            (computed and written by the sort's histogram kernel).
//            Positive f64 bits order like the values, and the map is monotone,
//            so sorting k32 orders every pair of splats whose k32 differ.
//  2 sort32  stable Onesweep radix sort of (k32, index), <= 3 passes (the
//            first drops the sentinels: the compaction of render.py:279).
//  3 fixup   splats with equal k32 form runs, already in index order
//            (stability); each run is re-sorted by the full f64 key, stably
//            (insertion sort by (key, index)), which gives exactly the
//            argsort tie order.  A run longer than kMaxRun sets a flag; the
//            host sees it when the frame completes and re-renders the frame
//            with the full 64-bit sort (8 passes over the raw key bits), so
//            the order is exact for any input at no cost in the common case.
#include <algorithm>

#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int kMaxRun = 16;
// Span key width: 24 bits = 3 radix passes.  At 3M kept splats a bucket holds
// 0.2 splats on average; the fix-up resolves the resulting short runs.
constexpr int kSpanBits = kSpanKeyBits;

__device__ __forceinline__ void depth_fixup_one(const DepthArgs &a, int64_t i, int64_t K);

// grid-stride over the ranks (the grid is bounded; K is read on the device)
__global__ void depth_fixup_kernel(DepthArgs a) {
    const int64_t K = *a.count;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K;
         i += (int64_t)gridDim.x * blockDim.x)
        depth_fixup_one(a, i, K);
}

__device__ __forceinline__ void depth_fixup_one(const DepthArgs &a, int64_t i, int64_t K) {
    const uint32_t b = a.sched[16];
    const uint32_t *ks = b ? a.keys32[1] : a.keys32[0];
    uint32_t *vs = b ? a.vals[1] : a.vals[0];
    const uint32_t c = ks[i];
    if (i + 1 >= K || ks[i + 1] != c) return;  // not followed by an equal key
    if (i > 0 && ks[i - 1] == c) return;       // not the first of its run
    int64_t e = i + 2;
    while (e < K && e - i <= kMaxRun && ks[e] == c) e++;
    const int len = (int)(e - i);
    if (len > kMaxRun) {
        if (atomicOr(&a.ctr->long_runs, 1u) == 0u && a.long_run_sticky)
            atomicAdd(a.long_run_sticky, 1u);
        return;
    }
    uint32_t idx[kMaxRun];
    unsigned long long key[kMaxRun];
    for (int j = 0; j < len; j++) {
        idx[j] = vs[i + j];
        key[j] = a.keys64[0][idx[j]];
    }
    // insertion sort by (key, index): the argsort tie order whatever order
    // the run's indices arrive in (slice B's are appended unordered)
    for (int j = 1; j < len; j++) {
        const uint32_t xi = idx[j];
        const unsigned long long xk = key[j];
        int m = j - 1;
        while (m >= 0 && (key[m] > xk || (key[m] == xk && idx[m] > xi))) {
            key[m + 1] = key[m];
            idx[m + 1] = idx[m];
            m--;
        }
        key[m + 1] = xk;
        idx[m + 1] = xi;
    }
    for (int j = 0; j < len; j++) vs[i + j] = idx[j];
}

}  // namespace

size_t depth_work32_bytes(int64_t n_cap) { return sort_work_bytes(n_cap, 4, 4); }
size_t depth_work64_bytes(int64_t n_cap) { return sort_work_bytes(n_cap, 8, 8); }

int launch_depth_sort(const DepthArgs &a, int sms, cudaStream_t s, const KMark &mark) {
    if (a.n <= 0) return 0;
    if (a.full64)  // exact for any input: 8 passes over the raw f64 key bits
        return launch_onesweep_sort<unsigned long long>(
            a.keys64[0], a.keys64[1], a.vals[0], a.vals[1], true, true, a.count, a.n, a.n, 8,
            true, a.work64, a.sched, &a.ctr->npass_fb, sms, s, mark);
    int launches;
    unsigned g;
    if (a.keys_given) {  // slice B: appended (span key, index) pairs, no sentinels
        g = (unsigned)((a.cap + 255) / 256);
        SpanKeys opts;
        opts.hist_zeroed = a.hist_zeroed;
        launches = launch_onesweep_sort<uint32_t>(a.keys32[0], a.keys32[1], a.vals[0], a.vals[1],
                                                  false, false, a.count, -1, a.cap,
                                                  kSpanBits / 8, false, a.work32, a.sched,
                                                  &a.ctr->npass, sms, s, mark, opts);
    } else {
        g = (unsigned)((a.n + 255) / 256);
        SpanKeys span;  // the histogram kernel writes the span keys (step 1)
        span.src = a.keys64[0];
        span.hist_zeroed = a.hist_zeroed;
        span.kmin = &a.ctr->kmin;
        span.kmax = &a.ctr->kmax;
        span.bits = kSpanBits;
        span.limit = a.limit;
        if (a.limit) {
            // slice A: the histogram kernel appends the slice's (k32, index)
            // pairs (counting KA); the passes sort only those
            span.count_out = a.count;
            span.compact = true;
            span.n_src = a.n;
            launches = launch_onesweep_sort<uint32_t>(a.keys32[0], a.keys32[1], a.vals[0],
                                                      a.vals[1], false, false, a.count, -1, a.n,
                                                      kSpanBits / 8, false, a.work32, a.sched,
                                                      &a.ctr->npass, sms, s, mark, span);
        } else {
            launches = launch_onesweep_sort<uint32_t>(a.keys32[0], a.keys32[1], a.vals[0],
                                                      a.vals[1], true, true, a.count, a.n, a.n,
                                                      kSpanBits / 8, true, a.work32, a.sched,
                                                      &a.ctr->npass, sms, s, mark, span);
        }
    }
    g = std::min<unsigned>(g, (unsigned)sms * 8u);  // grid-stride (count on the device)
    depth_fixup_kernel<<<std::max(g, 1u), 256, 0, s>>>(a);
    mark("depth_fixup");
    return launches + 1;
}

}  // namespace gsr
