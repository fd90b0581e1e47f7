// binning.cu -- K4/K5: tile duplication under the tile-list contract and
// per-tile range identification.
//
// The reference composites per image row (render.py:357-421) and has no
// tiles; the contract (restated in oracle/oracle.c
// orc_tile_keys) lists depth-rank s in tile (tx, ty) iff tx lies in
// [floor(min x0 / 16), floor((max x1 - 1) / 16)], min/max over the rows of
// tile row ty whose exact reference interval (render.py:384-397, x0 clamped at
// 0) is non-empty.  Rows are computed with the reference's f32 op order.
//
// One warp per depth-sorted splat: the 32 lanes take 32 consecutive rows
// aligned to a tile row, so each half-warp owns one tile row and the min/max
// reduce is a 4-step xor shuffle.
#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int kBinThreads = 256;

struct RowPair {
    int tx0_a, cnt_a;  // first tile row of this 32-row step (lanes 0-15)
    int tx0_b, cnt_b;  // second tile row (lanes 16-31)
};

// One 32-row step starting at `base` (a multiple of 16).  All lanes call.
__device__ __forceinline__ RowPair row_step(const SplatRec &s, int base, int lo, int hi,
                                            int width) {
    const int lane = lane_id();
    const int iy = base + lane;
    int mn = 0x7fffffff, mx = -0x7fffffff;
    if (iy >= lo && iy < hi) {
        int x0, x1;
        if (row_interval(s.a.x, s.a.y, s.a.z, s.a.w, s.b.x, s.b.y, (float)iy + 0.5f, width, x0,
                         x1)) {
            x0 = x0 > 0 ? x0 : 0;
            if (x0 < x1) {
                mn = x0;
                mx = x1;
            }
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
        int a = __shfl_xor_sync(0xffffffffu, mn, o);
        int b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    const int mn_b = __shfl_sync(0xffffffffu, mn, 16), mx_b = __shfl_sync(0xffffffffu, mx, 16);
    const int mn_a = __shfl_sync(0xffffffffu, mn, 0), mx_a = __shfl_sync(0xffffffffu, mx, 0);
    RowPair r;
    if (mn_a <= mx_a) {
        r.tx0_a = mn_a / kTile;
        r.cnt_a = (mx_a - 1) / kTile - r.tx0_a + 1;
    } else {
        r.tx0_a = 0;
        r.cnt_a = 0;
    }
    if (mn_b <= mx_b) {
        r.tx0_b = mn_b / kTile;
        r.cnt_b = (mx_b - 1) / kTile - r.tx0_b + 1;
    } else {
        r.tx0_b = 0;
        r.cnt_b = 0;
    }
    return r;
}

// Count pass.  Also gathers the depth-sorted record table srec[r] = rec[order[r]]
// (sort_splats' column gathers, render.py:295-302).
__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(
    const uint32_t *__restrict__ vals_even, const uint32_t *__restrict__ vals_odd,
    const SplatRec *__restrict__ rec, SplatRec *__restrict__ srec, uint32_t *__restrict__ counts,
    int64_t n_cap, const FrameCounters *ctr, int width, int height) {
    const int lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (kBinThreads / 32);
    const int64_t k = ctr->K;
    const uint32_t *order = (ctr->npass & 1) ? vals_odd : vals_even;
    for (int64_t r = (int64_t)blockIdx.x * (kBinThreads / 32) + (threadIdx.x >> 5); r < n_cap;
         r += warps) {
        if (r >= k) {
            if (lane == 0) counts[r] = 0;
            continue;
        }
        const uint32_t i = order[r];
        SplatRec s;
        s.a = __ldg(&rec[i].a);
        s.b = __ldg(&rec[i].b);
        s.c = __ldg(&rec[i].c);
        if (lane == 0) srec[r].a = s.a;
        if (lane == 1) srec[r].b = s.b;
        if (lane == 2) srec[r].c = s.c;
        int lo, hi;
        row_range(s.a.y, s.b.w, height, lo, hi);
        uint32_t total = 0;
        for (int base = (lo / kTile) * kTile; base < hi; base += 32) {
            RowPair p = row_step(s, base, lo, hi, width);
            total += (uint32_t)(p.cnt_a + p.cnt_b);
        }
        if (lane == 0) counts[r] = total;
    }
}

// Write pass: tile ids at offsets[r], in (tile row, tile column) order per splat.
__global__ void __launch_bounds__(kBinThreads) bin_write_kernel(
    const SplatRec *__restrict__ srec, const uint32_t *__restrict__ offsets, int64_t n_cap,
    const FrameCounters *ctr, int width, int height, uint32_t *__restrict__ tile_keys,
    uint32_t *__restrict__ tile_vals, int64_t cap_d, uint32_t *overflow_sticky) {
    const int lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (kBinThreads / 32);
    const int64_t k = ctr->K;
    if (blockIdx.x == 0 && threadIdx.x == 0 && (int64_t)ctr->D > cap_d) atomicAdd(overflow_sticky, 1u);
    const int tiles_x = (width + kTile - 1) / kTile;
    for (int64_t r = (int64_t)blockIdx.x * (kBinThreads / 32) + (threadIdx.x >> 5); r < k;
         r += warps) {
        SplatRec s;
        s.a = __ldg(&srec[r].a);
        s.b = __ldg(&srec[r].b);
        int lo, hi;
        row_range(s.a.y, s.b.w, height, lo, hi);
        int64_t off = offsets[r];
        for (int base = (lo / kTile) * kTile; base < hi; base += 32) {
            RowPair p = row_step(s, base, lo, hi, width);
            const int ty = base / kTile;
            const int n = p.cnt_a + p.cnt_b;
            for (int e = lane; e < n; e += 32) {
                const int t = e < p.cnt_a ? ty * tiles_x + p.tx0_a + e
                                          : (ty + 1) * tiles_x + p.tx0_b + (e - p.cnt_a);
                const int64_t pos = off + e;
                if (pos < cap_d) {
                    tile_keys[pos] = (uint32_t)t;
                    tile_vals[pos] = (uint32_t)r;
                }
            }
            off += n;
        }
    }
}

__global__ void tile_ranges_kernel(const uint32_t *__restrict__ keys, const FrameCounters *ctr,
                                   int64_t cap_d, uint2 *__restrict__ ranges) {
    int64_t d = ctr->D;
    d = d < cap_d ? d : cap_d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = keys[i];
        if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
        if (i == d - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
    }
}

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace

void launch_bin_count(const uint32_t *vals_even, const uint32_t *vals_odd, const SplatRec *rec,
                      SplatRec *srec, uint32_t *counts, int64_t n_cap, const FrameCounters *ctr,
                      int width, int height, cudaStream_t s) {
    if (n_cap <= 0) return;
    int64_t want = (n_cap + 7) / 8;
    int64_t blocks = sm_count() * 8;
    if (want < blocks) blocks = want;
    bin_count_kernel<<<(unsigned)blocks, kBinThreads, 0, s>>>(vals_even, vals_odd, rec, srec,
                                                              counts, n_cap, ctr, width, height);
}

void launch_bin_write(const SplatRec *srec, const uint32_t *offsets, int64_t n_cap,
                      const FrameCounters *ctr, int width, int height, uint32_t *tile_keys,
                      uint32_t *tile_vals, int64_t cap_d, uint32_t *overflow_sticky,
                      cudaStream_t s) {
    if (n_cap <= 0) return;
    int64_t want = (n_cap + 7) / 8;
    int64_t blocks = sm_count() * 8;
    if (want < blocks) blocks = want;
    bin_write_kernel<<<(unsigned)blocks, kBinThreads, 0, s>>>(
        srec, offsets, n_cap, ctr, width, height, tile_keys, tile_vals, cap_d, overflow_sticky);
}

void launch_tile_ranges(const uint32_t *tile_keys, const FrameCounters *ctr, int64_t cap_d,
                        uint2 *ranges, int n_tiles, cudaStream_t s) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, s);
    if (cap_d <= 0) return;
    int64_t blocks = sm_count() * 8;
    tile_ranges_kernel<<<(unsigned)blocks, 256, 0, s>>>(tile_keys, ctr, cap_d, ranges);
}

}  // namespace gsr
