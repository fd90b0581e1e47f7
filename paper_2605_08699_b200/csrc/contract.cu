// contract.cu -- the tile-list contract on T x T tiles (T = 16), built the
// way BASELINE.json's north_star item (2) words it: duplicate one 64-bit
// (tile | depth rank) key per covered tile, radix-sort the keys on the
// device, and identify each tile's [start, end) range in the sorted keys.
//
// The reference has no tiles (it composites per row, render.py:357-421); the
// contract (restated in oracle/oracle.c orc_tile_keys) lists
// depth rank s in tile (tx, ty) iff tx lies in [floor(min x0 / T),
// floor((max x1 - 1) / T)], min/max over the rows of tile row ty whose exact
// interval (render.py:384-397, x0 clamped at 0) is non-empty, rows limited
// to the splat's row range (render.py:329-333).
//
// The render path's own lists (binning.cu) are a conservative superset on
// 32 x 16 tiles, built without a key sort; this path emits the contract
// itself from the same frame's depth-ranked records, so the lists can be
// compared bit for bit with the oracle (gsr_debug_contract_tiles) and its
// cost measured beside the product binning (bench.py).
//
//  1 contract_keys  one thread per depth rank: per T-row band, the exact span
//                   (exact_band_span, every row's reference interval); the
//                   block reserves its keys with one atomicAdd and writes
//                   (ty * tiles_x + tx) << 32 | rank.  Key order inside the
//                   buffer depends on block scheduling, but keys are unique,
//                   so the sorted result does not.
//  2 radix sort     launch_onesweep_sort<u64> (radix.cu), 8-bit digits, the
//                   plan kernel skips constant digits (high tile bits).
//  3 contract_ranges  ranges[t] = [first, last + 1) of tile t's keys.
#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

constexpr int CB = 256;

__device__ __forceinline__ void band_tiles(const SplatRec &r, int band, int tile, int width,
                                           int &tx0, int &tx1) {
    int lo, hi;
    bool fast, safe;
    unpack_rows(r.b.w, lo, hi, fast, safe);
    const int y0 = max(lo, band * tile), y1 = min(hi, band * tile + tile);
    const float rinv = fast ? __frcp_rn(r.a.z) : 0.0f;
    int mn, mx;
    exact_band_span(r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, rinv, y0, y1, width, mn, mx);
    if (mn < mx) {
        tx0 = mn / tile;
        tx1 = (mx - 1) / tile;
    } else {
        tx0 = 1;
        tx1 = 0;
    }
}

__global__ void __launch_bounds__(CB) contract_keys_kernel(ContractArgs a) {
    __shared__ uint32_t s_warp[33];
    __shared__ unsigned long long s_base;
    const int64_t k = *a.count;
    const int64_t s = (int64_t)blockIdx.x * CB + threadIdx.x;
    if ((int64_t)blockIdx.x * CB >= k) return;
    SplatRec r;
    int lo = 0, hi = 0;
    uint32_t cnt = 0;
    if (s < k) {
        r = a.srec[s];
        bool fast, safe;
        unpack_rows(r.b.w, lo, hi, fast, safe);
        if (lo < hi)
            for (int ty = lo / a.tile; ty <= (hi - 1) / a.tile; ty++) {
                int tx0, tx1;
                band_tiles(r, ty, a.tile, a.width, tx0, tx1);
                if (tx0 <= tx1) cnt += (uint32_t)(tx1 - tx0 + 1);
            }
    }
    uint32_t total;
    const uint32_t off = block_excl_scan_u32(cnt, s_warp, &total);
    if (threadIdx.x == 0) s_base = atomicAdd(a.d_count, (unsigned long long)total);
    __syncthreads();
    const unsigned long long base = s_base + off;
    if (cnt == 0 || base + cnt > (unsigned long long)a.cap) return;  // host grows and retries
    unsigned long long *out = a.keys + base;
    for (int ty = lo / a.tile; ty <= (hi - 1) / a.tile; ty++) {
        int tx0, tx1;
        band_tiles(r, ty, a.tile, a.width, tx0, tx1);
        for (int tx = tx0; tx <= tx1; tx++)
            *out++ = ((unsigned long long)(ty * a.tiles_x + tx) << 32) | (unsigned long long)s;
    }
}

__global__ void contract_ranges_kernel(const unsigned long long *keys0,
                                       const unsigned long long *keys1, const uint32_t *sched,
                                       const unsigned long long *d_count, int64_t cap,
                                       uint2 *ranges) {
    const unsigned long long *keys = sched[16] ? keys1 : keys0;
    const int64_t d = (int64_t)min(*d_count, (unsigned long long)cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = (uint32_t)(keys[i] >> 32);
        if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[t].x = (uint32_t)i;
        if (i == d - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[t].y = (uint32_t)(i + 1);
    }
}

}  // namespace

int launch_contract_keys(const ContractArgs &a, int64_t cap_n, cudaStream_t s) {
    const int64_t blocks = (cap_n + CB - 1) / CB;
    if (blocks > 0) contract_keys_kernel<<<(unsigned)blocks, CB, 0, s>>>(a);
    return blocks > 0 ? 1 : 0;
}

int launch_contract_ranges(const unsigned long long *keys0, const unsigned long long *keys1,
                           const uint32_t *sched, const unsigned long long *d_count, int64_t cap,
                           uint2 *ranges, int ntiles, int sms, cudaStream_t s) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)ntiles, s);
    contract_ranges_kernel<<<sms * 4, 256, 0, s>>>(keys0, keys1, sched, d_count, cap, ranges);
    return 1;
}

}  // namespace gsr
