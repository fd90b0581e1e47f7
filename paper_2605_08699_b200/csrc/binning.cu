// binning.cu -- K4/K5: tile lists under the tile-list contract, sort-free.
//
// The reference composites per image row (render.py:357-421) and has no
// tiles; the contract (restated in oracle/oracle.c
// orc_tile_keys) lists depth-rank s in tile (tx, ty) iff tx lies in
// [floor(min x0 / 16), floor((max x1 - 1) / 16)], min/max over the rows of
// tile row ty whose exact reference interval (render.py:384-397, x0 clamped
// at 0) is non-empty.  Rows use the reference's f32 op order.  Each tile's
// list holds its depth ranks in increasing order (global stable depth order).
//
// Every splat covers a run of tile rows and, in each, one contiguous run of
// tile columns.  So the lists are built from (splat, tile row) pairs:
//  1a gather   block of 512 depth ranks: gathers the depth-sorted geometry
//              records (sort_splats' column gathers, render.py:295-302) and counts
//              its pairs per tile row (row range only, no interval math).
//  1b row_scan exclusive scan of those counts, tile-row major: each (row,
//              block) gets its output slot, each row its pair range.
//  1c pairs    same blocks: one thread per pair computes the pair's
//              tile-column span (tx0, count) -- a conservative bound of the
//              exact one (band_span_bound, common.cuh; exact rows for
//              ill-conditioned splats) -- and stores (rank, tx0 | count << 16)
//              at its slot: pairs end up grouped by tile row, in rank order.
//  2a segments each row's pairs are cut into segments of <= 1024 pairs.
//  2b seg_count one warp per segment: keys per tile column (difference array).
//  2c scans    per tile: prefix over the row's segments; tile starts, ranges, D.
//  2d seg_place one warp per segment walks its pairs 32 at a time in rank
//              order; a lane's position in tile t is the tile's cursor plus the
//              number of earlier lanes of the chunk covering t (shuffle count),
//              so each list comes out in increasing rank order.
// Only 4-byte ranks are written per list entry; there is no key array and
// no radix pass.  Counts stay on the device (no host synchronisation).
#include <algorithm>

#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

constexpr int BR = 512;          // depth ranks per block (stages 1a, 1c)
constexpr int kPairCache = 6144; // per-block pair results kept in smem (1c)
#ifndef GSR_BIN_SEG
#define GSR_BIN_SEG 256
#endif
// pairs per segment (stage 2): 256 gives seg_place ~7k warps of work at
// config 3 (1024: ~1.7k, 12 warps per SM): 0.049 -> 0.033 ms, one-call
// device p50 1.005 -> 0.960 ms (512: 0.036 / 0.975)
constexpr int kSeg = GSR_BIN_SEG;
constexpr int kRowsMax = kMaxTileRows;



// Blocks of BR depth ranks actually used by this pass (>= 1, so the row
// scan always covers every tile row).  row_blk is [n_rows][blocks_used]:
// grids are sized for the capacity (a front slice uses a fraction of it),
// and the kernels loop over the used blocks only.
__device__ __forceinline__ int64_t blocks_used(const BinArgs &a) {
    const int64_t k = *a.count;
    const int64_t nb = (k + BR - 1) / BR;
    return nb < 1 ? 1 : (nb < a.n_blocks ? nb : a.n_blocks);
}

constexpr int kScanItems = 8;  // row_scan: items per thread, 2048-element tiles
constexpr int kScanTile = 256 * kScanItems;

// ---------------------------------------------------------------- 1a -------
__global__ void __launch_bounds__(BR) bin_gather_kernel(BinArgs a) {
    __shared__ uint32_t cnt[kRowsMax];
    const int tid = threadIdx.x;
    {   // row_scan's look-back words (no memset node in the frame graph)
        const int64_t nz = (a.n_blocks * a.n_rows + kScanTile - 1) / kScanTile + 1;
        for (int64_t j = (int64_t)blockIdx.x * BR + tid; j < nz; j += (int64_t)gridDim.x * BR)
            a.scan_work[j] = 0ull;
    }
    const int64_t k = *a.count;
    const int64_t nbe = blocks_used(a);
    for (int64_t b = blockIdx.x; b < nbe; b += gridDim.x) {
    const int64_t r = b * BR + tid;
    for (int t = tid; t < a.n_rows; t += BR) cnt[t] = 0;
    __syncthreads();
    if (r < k) {
        const uint32_t *order = a.depth_sched[16] ? a.order1 : a.order0;
        const uint32_t i = __ldg(order + r);
        const float4 A = __ldg(&a.geo[i].a), B = __ldg(&a.geo[i].b);
        int lo, hi;
        row_range(A.y, B.w, a.height, lo, hi);
        a.srec[r].a = A;
        a.srec[r].b = make_float4(B.x, B.y, B.z,
                                  pack_rows(lo, hi, a.height, splat_fast_ok(A.y, A.z, A.w),
                                            exp_safe(A, B)));
        if (lo < hi)
            for (int ty = lo / kTileH; ty <= (hi - 1) / kTileH; ty++) atomicAdd(&cnt[ty], 1u);
    }
    __syncthreads();
    for (int t = tid; t < a.n_rows; t += BR) a.row_blk[(int64_t)t * nbe + b] = cnt[t];
    __syncthreads();  // cnt is reused by the block's next b
    }
}

// ---------------------------------------------------------------- 1b -------
// exclusive scan of row_blk (n_rows x n_blocks, row major) in place:
// 2048-element tiles in ticket order, decoupled look-back between tiles
// (kScanTile above)

__global__ void __launch_bounds__(256) row_scan_kernel(BinArgs a) {
    __shared__ uint32_t s_warp[33];
    __shared__ unsigned long long s_pre;
    __shared__ uint32_t s_ticket;
    if (threadIdx.x == 0) s_ticket = (uint32_t)atomicAdd(a.scan_work, 1ull);
    __syncthreads();
    const int64_t tile = s_ticket;
    unsigned long long *status = a.scan_work + 1;
    const int64_t nbe = blocks_used(a);
    const int64_t n = (int64_t)a.n_rows * nbe;
    if (tile * kScanTile >= n) return;  // (n >= n_rows >= 1: tile 0 always works)
    const int64_t base = tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems], s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        v[j] = base + j < n ? a.row_blk[base + j] : 0u;
        s += v[j];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan_u32(s, s_warp, &tot);
    if (threadIdx.x < 32) {
        const unsigned long long pre = lookback_exclusive(status, tile, tot);
        if (threadIdx.x == 0) s_pre = pre;
    }
    __syncthreads();
    const unsigned long long pre = s_pre;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        const int64_t idx = base + j;
        if (idx < n) {
            const unsigned long long o = pre + ex;
            a.row_blk[idx] = (uint32_t)o;
            if (idx % nbe == 0) a.row_start[idx / nbe] = (uint32_t)o;
        }
        ex += v[j];
    }
    if (threadIdx.x == 255 && (tile + 1) * kScanTile >= n) {  // last tile: totals
        // (and this pass's per-row list totals and D, accumulated / set by
        // seg_scan / seg_place)
        for (int r = 0; r < a.n_rows; r++) a.row_total[r] = 0u;
        a.ctr->D = 0u;
        const unsigned long long p = pre + ex;
        a.ctr->P = p;
        a.ctr->Ptot += p;  // one thread of one block per pass
        a.ctr->Pmax = p > a.ctr->Pmax ? p : a.ctr->Pmax;
        a.row_start[a.n_rows] = (uint32_t)(p < 0xffffffffull ? p : 0xffffffffull);
        if (p > (unsigned long long)a.cap_p) atomicAdd(a.overflow_sticky, 1u);
    }
}

// ---------------------------------------------------------------- 1c -------
struct PairSmem {
    float u[BR], v[BR], ia[BR], ib[BR], ic[BR], rsq[BR], rinv[BR];
    int lo[BR], hi[BR];
    uint32_t poff[BR + 1];
    uint32_t s_warp[33];
    uint8_t lr[kPairCache];          // in-warp rank of a pair within its row
    uint16_t owner[kPairCache];      // block-local splat of a pair
    int ty_lo, ty_hi;
    // followed in dynamic shared memory by (n_rows = tile rows of the frame):
    //   uint32_t wpre[BR / 32][n_rows]  per-warp coverage masks -> counts -> prefix
    //   uint32_t rowbase[n_rows]        this block's first slot per tile row (row_blk)
};
__host__ __device__ inline size_t pair_smem_bytes(int n_rows) {
    return sizeof(PairSmem) + sizeof(uint32_t) * (size_t)(BR / 32 + 1) * (size_t)n_rows;
}

__device__ __forceinline__ int rank_of_pair(const uint32_t *poff, uint32_t q) {
    int lo = 0, hi = BR;  // poff[lo] <= q < poff[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (poff[mid] <= q) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(BR) bin_pairs_kernel(BinArgs a) {
    extern __shared__ __align__(16) unsigned char dyn_raw[];
    PairSmem &S = *reinterpret_cast<PairSmem *>(dyn_raw);
    const int nr = a.n_rows;
    uint32_t *wpre_all = reinterpret_cast<uint32_t *>(dyn_raw + sizeof(PairSmem));
    uint32_t *rowbase = wpre_all + (BR / 32) * nr;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t k = *a.count;
    if (a.ctr->P > (unsigned long long)a.cap_p) return;
    const int64_t nbe = blocks_used(a);
    uint32_t n_rows = 0;
    for (int64_t b = blockIdx.x; b * BR < k; b += gridDim.x) {
    const int64_t r = b * BR + tid;
    uint32_t ntr = 0;
    int lo = 0, hi = 0;
    if (r < k) {
        const float4 A = __ldg(&a.srec[r].a), B = __ldg(&a.srec[r].b);
        bool fast, esafe;
        unpack_rows(B.w, lo, hi, fast, esafe);
        S.rinv[tid] = fast ? __frcp_rn(A.z) : 0.0f;
        S.u[tid] = A.x;
        S.v[tid] = A.y;
        S.ia[tid] = A.z;
        S.ib[tid] = A.w;
        S.ic[tid] = B.x;
        S.rsq[tid] = B.y;
        if (lo < hi) ntr = (uint32_t)((hi - 1) / kTileH - lo / kTileH + 1);
    }
    S.lo[tid] = lo;
    S.hi[tid] = hi;
    const int t0 = ntr ? lo / kTileH : 0x7fffffff, t1 = ntr ? (hi - 1) / kTileH : -1;
    if (tid == 0) {
        S.ty_lo = 0x7fffffff;
        S.ty_hi = -1;
    }
    uint32_t npairs;
    const uint32_t off = block_excl_scan_u32(ntr, S.s_warp, &npairs);  // (syncs)
    S.poff[tid] = off;
    if (tid == 0) S.poff[BR] = npairs;
    atomicMin(&S.ty_lo, t0);
    atomicMax(&S.ty_hi, t1);
    __syncthreads();
    // rank of each (splat, row) among the block's splats covering that row:
    // per-warp coverage bitmasks per tile row (shared atomics, one per pair)
    // give the in-warp rank, a prefix of the popcounts over warps the rest
    // a block whose splats cover no row (all ranges empty) keeps ty_lo at its
    // sentinel: start the loops at 0 so `ylo + lane` cannot overflow
    const int yhi = S.ty_hi, ylo = yhi >= 0 ? S.ty_lo : 0;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t *wm = wpre_all + w * nr;
    for (int ty = ylo + lane; ty <= yhi; ty += 32) wm[ty] = 0u;
    __syncwarp();
    for (int ty = t0; ty <= t1; ty++) atomicOr(&wm[ty], 1u << lane);
    __syncwarp();
    for (int ty = t0; ty <= t1; ty++) {
        const uint32_t q = off + (uint32_t)(ty - t0);
        if (q < kPairCache) {
            S.lr[q] = (uint8_t)__popc(wm[ty] & lt_mask);
            S.owner[q] = (uint16_t)tid;
        }
    }
    __syncwarp();
    for (int ty = ylo + lane; ty <= yhi; ty += 32) wm[ty] = __popc(wm[ty]);
    __syncthreads();
    for (int ty = ylo + tid; ty <= yhi; ty += BR) {
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < BR / 32; j++) {
            const uint32_t c = wpre_all[j * nr + ty];
            wpre_all[j * nr + ty] = run;
            run += c;
        }
        rowbase[ty] = run ? a.row_blk[(int64_t)ty * nbe + b] : 0u;
    }
    __syncthreads();
    // One thread per pair: tile span (bounded; exact rows for the few
    // ill-conditioned splats), stored at its grouped slot.
    for (uint32_t q = tid; q < npairs; q += BR) {
        const int j = q < kPairCache ? (int)S.owner[q] : rank_of_pair(S.poff, q);
        const int ty = S.lo[j] / kTileH + (int)(q - S.poff[j]);
        uint32_t in_warp;
        if (q < kPairCache) {
            in_warp = S.lr[q];
        } else {  // rare: recount covering splats of this warp before j
            in_warp = 0;
            for (int jj = j & ~31; jj < j; jj++)
                in_warp += (S.lo[jj] < S.hi[jj] && ty >= S.lo[jj] / kTileH &&
                            ty <= (S.hi[jj] - 1) / kTileH);
        }
        const uint32_t slot = rowbase[ty] + wpre_all[(j >> 5) * nr + ty] + in_warp;
        // tile-column span of splat j in tile row ty
        const int y0 = max(S.lo[j], ty * kTileH), y1 = min(S.hi[j], ty * kTileH + kTileH);
        int mn, mx;
        const float u = S.u[j], v = S.v[j], ia = S.ia[j], ib = S.ib[j], ic = S.ic[j],
                    rsq = S.rsq[j], rinv = S.rinv[j];
        if (!(rinv != 0.0f && y0 < y1 &&
              band_span_bound(u, v, ia, ib, ic, rsq, y0, y1, a.width, mn, mx))) {
            n_rows += (uint32_t)(y1 - y0);
            exact_band_span(u, v, ia, ib, ic, rsq, rinv, y0, y1, a.width, mn, mx);
        }
        uint32_t span = 0;
        if (mn <= mx) {
            const uint32_t tx0 = (uint32_t)(mn / kTileW);
            span = tx0 | (((uint32_t)((mx - 1) / kTileW) - tx0 + 1u) << 16);
        }
        if ((int64_t)slot < a.cap_p) a.pairs[slot] = make_uint2((uint32_t)(b * BR + j), span);
    }
    __syncthreads();  // shared state is reused by the block's next b
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_rows += __shfl_xor_sync(0xffffffffu, n_rows, o);
    if (lane == 0 && n_rows) atomicAdd(&a.ctr->Rp, (unsigned long long)n_rows);
}

// ---------------------------------------------------------------- 2a -------
// segments: row ty's pairs [row_start[ty], row_start[ty+1]) in pieces of kSeg
// The segment table -- row ty's pairs [row_start[ty], row_start[ty+1]) in
// pieces of kSeg; s_first[ty] = its first segment, s_first[n_rows] = all --
// rebuilt in shared memory by every CTA of the segment kernels (a block scan
// over <= 512 rows: cheaper than a one-block kernel and its launch).
struct SegTable {
    uint32_t first[kRowsMax + 1];
    uint32_t warp[33];
};

__device__ __forceinline__ void seg_table(const BinArgs &a, SegTable &T) {
    uint32_t carry = 0;
    const bool ov = a.ctr->P > (unsigned long long)a.cap_p;
    for (int base = 0; base < a.n_rows; base += blockDim.x) {
        const int ty = base + threadIdx.x;
        uint32_t ns = 0;
        if (ty < a.n_rows && !ov) {
            const uint32_t len = a.row_start[ty + 1] - a.row_start[ty];
            ns = (len + kSeg - 1) / kSeg;
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan_u32(ns, T.warp, &tot);
        if (ty < a.n_rows) T.first[ty] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) T.first[a.n_rows] = carry;
    __syncthreads();
}

__device__ __forceinline__ int64_t seg_total(const BinArgs &a, const SegTable &T) {
    const int64_t n = (int64_t)T.first[a.n_rows];
    return n < a.cap_seg ? n : a.cap_seg;
}

// first segment of tile row ty
__device__ __forceinline__ int64_t first_seg_of_row(const SegTable &T, uint32_t ty, int64_t nseg) {
    const int64_t f = (int64_t)T.first[ty];
    return f < nseg ? f : nseg;
}

__device__ __forceinline__ void seg_bounds(const BinArgs &a, const SegTable &T, int64_t g,
                                           int64_t nseg, uint32_t &ty, uint32_t &p0,
                                           uint32_t &p1) {
    int lo = 0, hi = a.n_rows;  // first[lo] <= g < first[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (T.first[mid] <= (uint32_t)g) lo = mid;
        else hi = mid;
    }
    ty = (uint32_t)lo;
    const int64_t first = first_seg_of_row(T, ty, nseg);
    const uint32_t rs = a.row_start[ty], re = a.row_start[ty + 1];
    p0 = rs + (uint32_t)(g - first) * kSeg;
    p1 = min(re, p0 + kSeg);
}

// ---------------------------------------------------------------- 2b -------
__device__ __forceinline__ void seg_count_one(const BinArgs &a, const SegTable &T, int64_t g,
                                              int64_t nseg, uint32_t *diff, int lane) {
    const int tx_n = a.tiles_x;
    __syncwarp();  // the warp's previous segment is done with diff
    for (int t = lane; t <= tx_n; t += 32) diff[t] = 0;
    __syncwarp();
    uint32_t ty, p0, p1;
    seg_bounds(a, T, g, nseg, ty, p0, p1);
    for (uint32_t p = p0 + lane; p < p1; p += 32) {
        const uint32_t sp = a.pairs[p].y;
        const uint32_t c = sp >> 16;
        if (c) {
            atomicAdd(&diff[sp & 0xffffu], 1u);
            atomicSub(&diff[(sp & 0xffffu) + c], 1u);
        }
    }
    __syncwarp();
    // prefix over columns -> counts, written to seg_cnt[g][tx]
    uint32_t carry = 0;
    for (int t0 = 0; t0 < tx_n; t0 += 32) {
        const int t = t0 + lane;
        const uint32_t dv = t < tx_n ? diff[t] : 0u;
        const uint32_t inc = warp_incl_scan_u32(dv) + carry;
        if (t < tx_n) a.seg_cnt[g * tx_n + t] = inc;
        carry = __shfl_sync(0xffffffffu, inc, 31);
    }
}

// one warp per segment: keys per tile column via a difference array
__global__ void __launch_bounds__(256) seg_count_kernel(BinArgs a) {
    extern __shared__ __align__(16) uint32_t diff_all[];  // [8][tiles_x + 1]
    __shared__ SegTable T;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (a.ctr->P > (unsigned long long)a.cap_p) return;
    seg_table(a, T);
    const int64_t nseg = seg_total(a, T);
    for (int64_t g = (int64_t)blockIdx.x * 8 + w; g < nseg; g += (int64_t)gridDim.x * 8)
        seg_count_one(a, T, g, nseg, diff_all + w * (a.tiles_x + 1), lane);
}

// ---------------------------------------------------------------- 2c -------
// warp per tile: exclusive prefix over its row's segments (32 at a time,
// warp scan), tile total
__global__ void __launch_bounds__(256) seg_scan_kernel(BinArgs a) {
    __shared__ SegTable T;
    const int t = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (a.ctr->P > (unsigned long long)a.cap_p) {
        // the pairs overflowed: no lists this pass (the frame re-renders with
        // larger buffers), but the blend still runs -- empty every range
        if (t < a.ntiles && lane == 0) a.ranges[t] = make_uint2(0u, 0u);
        return;
    }
    seg_table(a, T);
    if (t >= a.ntiles) return;
    const int tx_n = a.tiles_x;
    const int ty = t / tx_n, tx = t % tx_n;
    const uint32_t rs = a.row_start[ty], re = a.row_start[ty + 1];
    const uint32_t nrow = (re - rs + kSeg - 1) / kSeg;
    const int64_t lo = first_seg_of_row(T, (uint32_t)ty, seg_total(a, T));
    uint32_t *base = a.seg_cnt + lo * tx_n + tx;
    uint32_t carry = 0;
    for (uint32_t s0 = 0; s0 < nrow; s0 += 32) {
        const uint32_t si = s0 + lane;
        const uint32_t v = si < nrow ? base[(int64_t)si * tx_n] : 0u;
        const uint32_t inc = warp_incl_scan_u32(v);
        if (si < nrow) base[(int64_t)si * tx_n] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
        a.tile_total[t] = carry;
        if (carry) atomicAdd(a.row_total + ty, carry);  // the row's list entries
        // an empty list (tiles of rows without pairs have no seg_place warp;
        // seg_place overwrites the others)
        else a.ranges[t] = make_uint2(0u, 0u);
    }
}

// ---------------------------------------------------------------- 2d -------
// One warp places pairs [p0, p1) of one tile row, in rank order: cur[t] is
// the next free slot of tile column t's list, mask[t] (zeroed) a scratch
// coverage mask (both warp-private shared memory).
__device__ __forceinline__ void place_pairs(const BinArgs &a, uint32_t p0, uint32_t p1,
                                            uint32_t *cur, uint32_t *mask, int lane) {
    const uint32_t lt_mask = (1u << lane) - 1u;
    // software pipeline: the next chunks' pairs are in flight while this
    // chunk is placed (the loop is otherwise bound by that load's latency)
    constexpr int kAhead = 4;
    uint2 nxt[kAhead];
#pragma unroll
    for (int q = 0; q < kAhead; q++) {
        const uint32_t pq = p0 + 32u * q + lane;
        nxt[q] = pq < p1 ? a.pairs[pq] : make_uint2(0u, 0u);
    }
    for (uint32_t c0 = p0; c0 < p1; c0 += 32) {
        const uint2 pr = nxt[0];
#pragma unroll
        for (int q = 0; q + 1 < kAhead; q++) nxt[q] = nxt[q + 1];
        {
            const uint32_t pq = c0 + 32u * kAhead + lane;
            nxt[kAhead - 1] = pq < p1 ? a.pairs[pq] : make_uint2(0u, 0u);
        }
        // covers columns [a0, a0 + n) (n = 0 past the segment end)
        const uint32_t rank = pr.x, a0 = pr.y & 0xffffu, n = pr.y >> 16;
        // 1: coverage mask of every column touched by the chunk
        for (uint32_t e = 0; e < n; e++) atomicOr(&mask[a0 + e], 1u << lane);
        __syncwarp();
        // 2: position = cursor + earlier (lower-rank) lanes covering the column
        //    (and remember the columns this lane is the highest covering lane
        //    of; the first kKeep of them with their new cursor, in registers)
        constexpr int kKeep = 4;
        uint32_t top = 0, kt[kKeep], kc[kKeep];
        int nkeep = 0;
#pragma unroll
        for (int q = 0; q < kKeep; q++) kt[q] = kc[q] = 0u;
        for (uint32_t e = 0; e < n; e++) {
            const uint32_t t = a0 + e;
            const uint32_t m = mask[t];
            const uint32_t c = cur[t];
            const uint32_t pos = c + __popc(m & lt_mask);
            if ((int64_t)pos < a.cap_d) a.tile_vals[pos] = rank;
            if ((m >> lane) == 1u) {
                if (nkeep < kKeep) {  // shift register (static indices)
#pragma unroll
                    for (int q = kKeep - 1; q > 0; q--) {
                        kt[q] = kt[q - 1];
                        kc[q] = kc[q - 1];
                    }
                    kt[0] = t;
                    kc[0] = c + __popc(m);
                    nkeep++;
                } else {
                    top |= e < 32 ? 1u << e : 0u;
                }
            }
        }
        __syncwarp();
        // 3: the highest covering lane of each column advances its cursor and
        //    clears its mask (only that lane touches the column in this phase)
#pragma unroll
        for (int q = 0; q < kKeep; q++)
            if (q < nkeep) {
                cur[kt[q]] = kc[q];
                mask[kt[q]] = 0;
            }
        for (uint32_t bits = top; bits; bits &= bits - 1u) {
            const uint32_t t = a0 + (uint32_t)(__ffs(bits) - 1);
            cur[t] += __popc(mask[t]);
            mask[t] = 0;
        }
        for (uint32_t e = 32; e < n; e++) {  // spans beyond 32 tiles (512 px)
            const uint32_t t = a0 + e;
            const uint32_t m = mask[t];
            if ((m >> lane) == 1u) {
                cur[t] += __popc(m);
                mask[t] = 0;
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ void seg_place_one(const BinArgs &a, const SegTable &T, int64_t g,
                                              int64_t nseg, uint32_t *cur, int lane) {
    const int tx_n = a.tiles_x;
    uint32_t *mask = cur + tx_n;
    __syncwarp();  // the warp's previous segment is done with cur / mask
    uint32_t ty, p0, p1;
    seg_bounds(a, T, g, nseg, ty, p0, p1);
    // the lists are tile-major: row ty's lists start after every earlier
    // row's (row_total from seg_scan); D = all rows' entries.  (This replaces
    // a one-block scan over all tile totals.)
    unsigned long long base = 0, d = 0;
    for (int r0 = 0; r0 < a.n_rows; r0 += 32) {
        const int r = r0 + lane;
        const uint32_t v = r < a.n_rows ? a.row_total[r] : 0u;
        d += v;
        base += (uint32_t)r < ty ? v : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        base += __shfl_xor_sync(0xffffffffu, base, o);
    }
    const bool over = (int64_t)d > a.cap_d;
    const bool first_of_row = g == first_seg_of_row(T, ty, nseg);
    uint32_t carry = 0;
    for (int t0 = 0; t0 < tx_n; t0 += 32) {
        const int t = t0 + lane;
        const uint32_t v = t < tx_n ? a.tile_total[(int64_t)ty * tx_n + t] : 0u;
        const uint32_t inc = warp_incl_scan_u32(v);
        const uint32_t st = (uint32_t)base + carry + inc - v;  // tile start
        if (t < tx_n) {
            cur[t] = st + a.seg_cnt[g * tx_n + t];
            mask[t] = 0;
            // ranges: by the row's first segment (empty on overflow: the frame
            // re-renders, and the blend must stay in bounds)
            if (first_of_row)
                a.ranges[(int64_t)ty * tx_n + t] = over ? make_uint2(0u, 0u) : make_uint2(st, st + v);
        }
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (g == 0 && lane == 0) {  // the pass's list size (one writer)
        a.ctr->D = (uint32_t)(d < 0xffffffffull ? d : 0xffffffffull);
        a.ctr->Dtot += d;
        a.ctr->Dmax = d > a.ctr->Dmax ? d : a.ctr->Dmax;
        if (over) atomicAdd(a.overflow_sticky, 1u);
    }
    if (over) return;
    __syncwarp();
    place_pairs(a, p0, p1, cur, mask, lane);
}

// ------------------------------------------------ per-row lists: 2a-2d fused --
// (for slices of ~0.4M splats -- 1.8M pairs, ~26k per tile row -- the
// row-per-CTA build with 32 warps took 0.107 ms vs 0.066 for the segment
// kernels: it is kept for small second slices only, where 32 warps per row
// beat 16 and 8: 16.9 / 17.8 / 23.3 us per frame at config 3)
#ifndef GSR_ROW_WARPS
#define GSR_ROW_WARPS 32
#endif
constexpr int kRowWarpsSmall = GSR_ROW_WARPS;
// One CTA per tile row builds that row's tile lists from its pairs (a small
// second slice has few pairs per row, so the segment table, the per-segment
// counts, the two scans and the placement -- five kernels -- become one):
// the row's pairs are cut into one contiguous chunk per warp; each warp counts
// its chunk's keys per tile column (difference array); a prefix over the
// warps gives each warp its first slot per column; the row's region of the
// list buffer is taken with one atomicAdd (rows land in any order -- the
// lists are addressed through ranges -- but each list holds its ranks in
// increasing order); each warp places its chunk (place_pairs).
// [NW][tiles_x + 1] counts, [NW][2][tiles_x] cursors + masks, [tiles_x]
// column totals -> row starts
__host__ __device__ inline size_t row_lists_smem_bytes(int tiles_x, int nw) {
    return sizeof(uint32_t) * ((size_t)nw * (3 * (size_t)tiles_x + 1) + (size_t)tiles_x);
}

template <int kRowWarps>
__global__ void __launch_bounds__(kRowWarps * 32) bin_rows_kernel(BinArgs a) {
    extern __shared__ __align__(16) uint32_t row_smem[];
    __shared__ uint32_t s_base, s_last;
    const int tx_n = a.tiles_x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ty = blockIdx.x;
    uint32_t *cnt = row_smem + w * (tx_n + 1);                   // [w][tx_n + 1]
    uint32_t *cur = row_smem + kRowWarps * (tx_n + 1) + w * 2 * tx_n;
    uint32_t *mask = cur + tx_n;
    const bool ov_p = a.ctr->P > (unsigned long long)a.cap_p;
    uint32_t p0 = 0, p1 = 0;
    if (!ov_p) {
        p0 = a.row_start[ty];
        p1 = a.row_start[ty + 1];
    }
    // warp w's chunk of the row's pairs
    const uint32_t per = (p1 - p0 + kRowWarps - 1) / kRowWarps;
    const uint32_t c0 = min(p1, p0 + per * w), c1 = min(p1, c0 + per);
    for (int t = lane; t <= tx_n; t += 32) cnt[t] = 0;
    __syncwarp();
    for (uint32_t p = c0 + lane; p < c1; p += 32) {
        const uint32_t sp = a.pairs[p].y, c = sp >> 16;
        if (c) {
            atomicAdd(&cnt[sp & 0xffffu], 1u);
            atomicSub(&cnt[(sp & 0xffffu) + c], 1u);
        }
    }
    __syncwarp();
    {   // difference array -> keys per column of this warp's chunk
        uint32_t carry = 0;
        for (int t0 = 0; t0 < tx_n; t0 += 32) {
            const int t = t0 + lane;
            const uint32_t inc = warp_incl_scan_u32(t < tx_n ? cnt[t] : 0u) + carry;
            if (t < tx_n) cnt[t] = inc;
            carry = __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncthreads();
    // per column: exclusive prefix over the warps (in place), column totals
    uint32_t *tot = row_smem + kRowWarps * (tx_n + 1) + 2 * tx_n * kRowWarps;  // [tx_n]
    for (int t = threadIdx.x; t < tx_n; t += blockDim.x) {
        uint32_t run = 0;
        for (int j = 0; j < kRowWarps; j++) {
            uint32_t *cj = row_smem + j * (tx_n + 1);
            const uint32_t v = cj[t];
            cj[t] = run;
            run += v;
        }
        tot[t] = run;
    }
    __syncthreads();
    // column totals -> exclusive prefix across the row (one warp), region
    if (w == 0) {
        uint32_t carry = 0;
        for (int t0 = 0; t0 < tx_n; t0 += 32) {
            const int t = t0 + lane;
            const uint32_t v = t < tx_n ? tot[t] : 0u;
            const uint32_t inc = warp_incl_scan_u32(v) + carry;
            if (t < tx_n) tot[t] = inc - v;  // exclusive start within the row
            carry = __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) {
            s_base = carry ? atomicAdd(&a.ctr->Drow, carry) : 0u;
            const uint32_t end = s_base + carry;
            // ranges: empty if the region does not fit (the frame re-renders)
            const bool fits = (int64_t)end <= a.cap_d;
            s_last = fits ? 1u : 0u;
        }
        __syncwarp();
        const bool fits = s_last != 0u;
        const uint32_t base = s_base;
        for (int t0 = 0; t0 < tx_n; t0 += 32) {
            const int t = t0 + lane;
            if (t < tx_n) {
                const uint32_t st = base + tot[t];
                const uint32_t en = t + 1 < tx_n ? base + tot[t + 1] : base + carry;
                a.ranges[(int64_t)ty * tx_n + t] = fits ? make_uint2(st, en) : make_uint2(0u, 0u);
            }
        }
    }
    __syncthreads();
    if (s_last && c0 < c1) {
        const uint32_t *cw = row_smem + w * (tx_n + 1);
        for (int t = lane; t < tx_n; t += 32) {
            cur[t] = s_base + tot[t] + cw[t];
            mask[t] = 0;
        }
        __syncwarp();
        place_pairs(a, c0, c1, cur, mask, lane);
    }
    // the last row to finish publishes the pass's list total
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&a.ctr->rows_done, 1u) + 1u == gridDim.x) {
            const unsigned long long d = atomicAdd(&a.ctr->Drow, 0u);
            a.ctr->D = (uint32_t)d;
            a.ctr->Dtot += d;
            a.ctr->Dmax = d > a.ctr->Dmax ? d : a.ctr->Dmax;
            if ((int64_t)d > a.cap_d) atomicAdd(a.overflow_sticky, 1u);
            // every row of this pass has allocated and counted: reset for
            // the frame's next pass
            a.ctr->Drow = 0u;
            a.ctr->rows_done = 0u;
        }
    }
}

__global__ void __launch_bounds__(256) seg_place_kernel(BinArgs a) {
    // per warp: column cursors [tiles_x] and coverage masks [tiles_x]
    extern __shared__ __align__(16) uint32_t place_smem[];
    __shared__ SegTable T;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (a.ctr->P > (unsigned long long)a.cap_p) return;
    seg_table(a, T);
    const int64_t nseg = seg_total(a, T);
    for (int64_t g = (int64_t)blockIdx.x * 8 + w; g < nseg; g += (int64_t)gridDim.x * 8)
        seg_place_one(a, T, g, nseg, place_smem + w * 2 * a.tiles_x, lane);
}


}  // namespace

int64_t bin_blocks(int64_t n_cap) { return (n_cap + BR - 1) / BR; }
int64_t bin_scan_tiles(int64_t n_blocks, int n_rows) {
    return (n_blocks * n_rows + kScanTile - 1) / kScanTile;
}
int64_t bin_segments(int64_t cap_p, int n_rows) { return cap_p / kSeg + n_rows + 1; }

cudaError_t binning_init_attributes() {
    cudaError_t e = cudaFuncSetAttribute(bin_pairs_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pair_smem_bytes(kRowsMax));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(seg_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(8 * (kMaxTilesX + 1) * sizeof(uint32_t)));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(seg_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(8 * 2 * kMaxTilesX * sizeof(uint32_t)));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(bin_rows_kernel<kRowWarpsSmall>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)row_lists_smem_bytes(kMaxTilesX, kRowWarpsSmall));

    return e;
}

int launch_binning(const BinArgs &a, cudaStream_t s, const KMark &mark, bool rows) {
    if (a.n_blocks <= 0) return 0;
    // grids bounded by what the SMs hold at once (the kernels loop over the
    // blocks of ranks actually used, read from the device count)
    const unsigned nb = (unsigned)std::min<int64_t>(a.n_blocks, (int64_t)a.sms * 4);
    const unsigned nbp = (unsigned)std::min<int64_t>(a.n_blocks, (int64_t)a.sms * 2);
    bin_gather_kernel<<<nb, BR, 0, s>>>(a);
    mark("bin_gather");
    const int64_t scan_tiles = bin_scan_tiles(a.n_blocks, a.n_rows);  // (zeroed by bin_gather)
    row_scan_kernel<<<(unsigned)scan_tiles, 256, 0, s>>>(a);
    mark("row_scan");
    bin_pairs_kernel<<<nbp, BR, pair_smem_bytes(a.n_rows), s>>>(a);
    mark("bin_pairs");
    if (rows) {  // one CTA per tile row builds the row's lists
        bin_rows_kernel<kRowWarpsSmall><<<(unsigned)a.n_rows, kRowWarpsSmall * 32,
                                          row_lists_smem_bytes(a.tiles_x, kRowWarpsSmall), s>>>(a);
        mark("bin_rows");
        return 4;
    }
    // segment kernels loop over the frame's segments: the grid covers the
    // capacity up to 2048 blocks (a small slice's pass exits early)
    const unsigned sb = (unsigned)std::min<int64_t>((a.cap_seg + 7) / 8, 2048);
    seg_count_kernel<<<sb, 256, 8 * (a.tiles_x + 1) * sizeof(uint32_t), s>>>(a);
    mark("seg_count");
    seg_scan_kernel<<<(unsigned)((a.ntiles + 7) / 8), 256, 0, s>>>(a);
    mark("seg_scan");
    seg_place_kernel<<<sb, 256, 8 * 2 * a.tiles_x * sizeof(uint32_t), s>>>(a);
    mark("seg_place");
    return 6;
}

}  // namespace gsr
