// binning.cu -- K4/K5: tile duplication under the tile-list contract and
// per-tile range identification.
//
// The reference composites per image row (render.py:357-421) and has no
// tiles; the contract (restated in oracle/oracle.c
// orc_tile_keys) lists depth-rank s in tile (tx, ty) iff tx lies in
// [floor(min x0 / 16), floor((max x1 - 1) / 16)], min/max over the rows of
// tile row ty whose exact reference interval (render.py:384-397, x0 clamped
// at 0) is non-empty.  Rows are computed with the reference's f32 op order.
//
// One fused kernel, one pass over the depth-sorted splats:
//   * a block takes 256 consecutive depth ranks (in ticket order), gathers
//     their records into the depth-sorted table srec (sort_splats' gathers,
//     render.py:295-302) and computes each splat's row range;
//   * the block expands its (splat, tile row) pairs in shared memory (block
//     scan + binary search), one thread per pair computes the <= 16 exact row
//     intervals of that tile row once and reduces them to (tx0, count);
//   * a decoupled look-back over blocks turns the block's key count into its
//     global offset; keys (tile id) and values (depth rank) are written in
//     rank-major order, ready for the stable tile sort.
#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

constexpr int BR = 256;            // depth ranks (= threads) per block
constexpr int kPairCache = 4096;   // (splat, tile row) results kept in smem

struct BinSmem {
    float u[BR], v[BR], ia[BR], ib[BR], ic[BR], rsq[BR];
    int lo[BR], hi[BR];
    uint32_t poff[BR + 1];
    uint32_t pc[kPairCache];
    uint32_t s_warp[33];
    unsigned long long block_prefix;
    unsigned long long ticket;
    uint32_t npairs;
};

// exact tile-column span of splat j in tile row ty (reference intervals)
__device__ __forceinline__ void pair_tiles(const BinSmem &S, int j, int ty, int width, int &tx0,
                                           int &cnt) {
    const int y0 = max(S.lo[j], ty * kTile), y1 = min(S.hi[j], ty * kTile + kTile);
    int mn = 0x7fffffff, mx = -0x7fffffff;
    const float u = S.u[j], v = S.v[j], ia = S.ia[j], ib = S.ib[j], ic = S.ic[j], rsq = S.rsq[j];
    for (int y = y0; y < y1; y++) {
        int x0, x1;
        if (row_interval(u, v, ia, ib, ic, rsq, (float)y + 0.5f, width, x0, x1)) {
            x0 = x0 > 0 ? x0 : 0;
            if (x0 < x1) {
                mn = x0 < mn ? x0 : mn;
                mx = x1 > mx ? x1 : mx;
            }
        }
    }
    if (mn <= mx) {
        tx0 = mn / kTile;
        cnt = (mx - 1) / kTile - tx0 + 1;
    } else {
        tx0 = 0;
        cnt = 0;
    }
}

__device__ __forceinline__ int rank_of_pair(const BinSmem &S, uint32_t q) {
    // largest j in [0, BR) with poff[j] <= q  (poff[BR] = npairs > q)
    int lo = 0, hi = BR;  // invariant: poff[lo] <= q < poff[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (S.poff[mid] <= q) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(BR) bin_kernel(
    const uint32_t *__restrict__ order_even, const uint32_t *__restrict__ order_odd,
    const SplatRec *__restrict__ rec, SplatRec *__restrict__ srec, FrameCounters *ctr, int width,
    int height, uint32_t *__restrict__ tile_keys, uint32_t *__restrict__ tile_vals, int64_t cap_d,
    unsigned long long *__restrict__ status, uint32_t *overflow_sticky) {
    __shared__ BinSmem S;
    const int tid = threadIdx.x;
    if (tid == 0) S.ticket = atomicAdd(&ctr->bin_ticket, 1ull);
    __syncthreads();
    const int64_t t = (int64_t)S.ticket;
    const int64_t k = ctr->K;
    const int64_t r0 = t * BR;
    if (r0 >= k) return;
    const uint32_t *order = (ctr->npass & 1) ? order_odd : order_even;
    const int tiles_x = (width + kTile - 1) / kTile;

    // ---- gather + row ranges -------------------------------------------
    const int64_t r = r0 + tid;
    uint32_t ntr = 0;
    if (r < k) {
        const uint32_t i = __ldg(order + r);
        const float4 A = __ldg(&rec[i].a), B = __ldg(&rec[i].b), C = __ldg(&rec[i].c);
        srec[r].a = A;
        srec[r].b = B;
        srec[r].c = C;
        int lo, hi;
        row_range(A.y, B.w, height, lo, hi);
        S.u[tid] = A.x;
        S.v[tid] = A.y;
        S.ia[tid] = A.z;
        S.ib[tid] = A.w;
        S.ic[tid] = B.x;
        S.rsq[tid] = B.y;
        S.lo[tid] = lo;
        S.hi[tid] = hi;
        if (lo < hi) ntr = (uint32_t)((hi - 1) / kTile - lo / kTile + 1);
    } else {
        S.lo[tid] = 0;
        S.hi[tid] = 0;
    }
    uint32_t npairs;
    const uint32_t off = block_excl_scan_u32(ntr, S.s_warp, &npairs);
    S.poff[tid] = off;
    if (tid == 0) S.poff[BR] = npairs;
    __syncthreads();

    // ---- phase 1: (tx0, count) per (splat, tile row) --------------------
    uint32_t my_keys = 0;
    for (uint32_t q0 = 0; q0 < npairs; q0 += BR) {
        const uint32_t q = q0 + tid;
        if (q < npairs) {
            const int j = rank_of_pair(S, q);
            const int ty = S.lo[j] / kTile + (int)(q - S.poff[j]);
            int tx0, cnt;
            pair_tiles(S, j, ty, width, tx0, cnt);
            if (q < kPairCache) S.pc[q] = (uint32_t)tx0 | ((uint32_t)cnt << 16);
            my_keys += (uint32_t)cnt;
        }
    }
    uint32_t block_keys;
    block_excl_scan_u32(my_keys, S.s_warp, &block_keys);

    // ---- global offset of this block (decoupled look-back) --------------
    if (tid < 32) {
        const unsigned long long pre = lookback_exclusive(status, t, block_keys);
        if (tid == 0) {
            S.block_prefix = pre;
            if (r0 + BR >= k) {  // last block: publish D
                const unsigned long long d = pre + block_keys;
                ctr->D = (uint32_t)(d < 0xffffffffull ? d : 0xffffffffull);
                if ((int64_t)d > cap_d) atomicAdd(overflow_sticky, 1u);
            }
        }
    }
    __syncthreads();

    // ---- phase 2: write keys in rank-major order ------------------------
    unsigned long long run = S.block_prefix;
    for (uint32_t q0 = 0; q0 < npairs; q0 += BR) {
        const uint32_t q = q0 + tid;
        int j = 0, ty = 0, tx0 = 0, cnt = 0;
        if (q < npairs) {
            j = rank_of_pair(S, q);
            ty = S.lo[j] / kTile + (int)(q - S.poff[j]);
            if (q < kPairCache) {
                const uint32_t pc = S.pc[q];
                tx0 = (int)(pc & 0xffffu);
                cnt = (int)(pc >> 16);
            } else {
                pair_tiles(S, j, ty, width, tx0, cnt);
            }
        }
        uint32_t chunk;
        const uint32_t o = block_excl_scan_u32((uint32_t)cnt, S.s_warp, &chunk);
        const unsigned long long pos = run + o;
        const uint32_t tid0 = (uint32_t)(ty * tiles_x + tx0);
        const uint32_t rk = (uint32_t)(r0 + j);
        for (int e = 0; e < cnt; e++) {
            const unsigned long long p = pos + (unsigned long long)e;
            if ((int64_t)p < cap_d) {
                tile_keys[p] = tid0 + (uint32_t)e;
                tile_vals[p] = rk;
            }
        }
        run += chunk;
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

}  // namespace

int64_t bin_status_words(int64_t n_cap) { return (n_cap + BR - 1) / BR + 1; }

void launch_bin(const uint32_t *vals_even, const uint32_t *vals_odd, const SplatRec *rec,
                SplatRec *srec, int64_t n_cap, FrameCounters *ctr, int width, int height,
                uint32_t *tile_keys, uint32_t *tile_vals, int64_t cap_d,
                unsigned long long *status, uint32_t *overflow_sticky, cudaStream_t s) {
    if (n_cap <= 0) return;
    cudaMemsetAsync(status, 0, sizeof(unsigned long long) * (size_t)bin_status_words(n_cap), s);
    const unsigned blocks = (unsigned)((n_cap + BR - 1) / BR);
    bin_kernel<<<blocks, BR, 0, s>>>(vals_even, vals_odd, rec, srec, ctr, width, height, tile_keys,
                                     tile_vals, cap_d, status, overflow_sticky);
}

void launch_tile_ranges(const uint32_t *tile_keys, const FrameCounters *ctr, int64_t cap_d,
                        uint2 *ranges, int n_tiles, int sms, cudaStream_t s) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, s);
    if (cap_d <= 0) return;
    tile_ranges_kernel<<<(unsigned)(sms * 8), 256, 0, s>>>(tile_keys, ctr, cap_d, ranges);
}

}  // namespace gsr
