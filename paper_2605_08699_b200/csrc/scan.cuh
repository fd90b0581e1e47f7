// scan.cuh -- warp/block scans and a single-value decoupled look-back used by
// the fused binning kernel (internal).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gsr {

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive block scan over blockDim.x (multiple of 32, <= 1024) values.
// s_warp must hold 33 words.  All threads must call.
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t *s_warp,
                                                        uint32_t *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t inc = warp_incl_scan_u32(v);
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < nw ? s_warp[lane] : 0u;
        uint32_t xi = warp_incl_scan_u32(x);
        if (lane < nw) s_warp[lane] = xi - x;
        if (lane == nw - 1) s_warp[32] = xi;
    }
    __syncthreads();
    uint32_t r = s_warp[w] + inc - v;
    if (total) *total = s_warp[32];
    __syncthreads();
    return r;
}

// Chained-scan status word: bits 62-63 flag (1 = aggregate, 2 = inclusive
// prefix), bits 0-61 value.  The array must be zeroed before the kernel.
constexpr unsigned long long kLbAggregate = 1ull << 62;
constexpr unsigned long long kLbInclusive = 2ull << 62;
constexpr unsigned long long kLbValueMask = (1ull << 62) - 1;

// flag and value share one 64-bit word: relaxed GPU-scope accesses suffice
// (acquire loads would invalidate L1 on every poll)
__device__ __forceinline__ void lb_store(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by one full warp of block `tile` (tiles are taken in ticket order).
// Publishes `aggregate`, looks back over predecessors 32 at a time, publishes
// the inclusive prefix and returns the exclusive prefix (to all lanes).
__device__ __forceinline__ unsigned long long lookback_exclusive(unsigned long long *status,
                                                                 int64_t tile,
                                                                 unsigned long long aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) lb_store(status, kLbInclusive | aggregate);
        return 0ull;
    }
    if (lane == 0) lb_store(status + tile, kLbAggregate | aggregate);
    unsigned long long excl = 0;
    int64_t base = tile - 1;
    while (true) {
        const int64_t idx = base - lane;
        unsigned long long s = 0;
        if (idx >= 0) {
            do {
                s = lb_load(status + idx);
            } while ((s >> 62) == 0);
        } else {
            s = kLbInclusive;  // before tile 0: inclusive zero
        }
        const uint32_t incl_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        // lanes up to and including the first inclusive one contribute
        const int stop = incl_mask ? __ffs(incl_mask) - 1 : 31;
        unsigned long long v = lane <= stop ? (s & kLbValueMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (incl_mask) break;
        base -= 32;
    }
    if (lane == 0) lb_store(status + tile, kLbInclusive | (excl + aggregate));
    return excl;
}

}  // namespace gsr
