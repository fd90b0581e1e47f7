// radix.cu -- device-wide exclusive scan and a stable LSD radix sort pass.
//
// Used for (a) the stable f64 depth sort that replaces
// np.argsort(depths, kind="stable") (render.py:293-302) -- keys are the IEEE
// bits of z (> 0, so unsigned order == numeric order), ties keep index order
// because every pass is stable and the first pass reads in index order; and
// (b) the stable tile sort of the (tile, depth-rank) list.
//
// Pass structure (per 8-bit digit): upsweep (per-tile digit histograms,
// digit-major) -> exclusive scan -> downsweep (stable in-tile ranking with
// warp match_any, shared-memory staging, coalesced scatter).  Item counts
// are read from device memory so a whole frame is enqueued without host
// synchronisation; grids are sized from capacities and idle tiles exit.
#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanChunk = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// exclusive block scan over blockDim.x (multiple of 32, <= 1024) values
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *s_warp,
                                                    uint32_t *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t inc = warp_incl_scan(v);
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < nw ? s_warp[lane] : 0u;
        uint32_t xi = warp_incl_scan(x);
        if (lane < nw) s_warp[lane] = xi - x;
        if (lane == nw - 1) s_warp[32] = xi;
    }
    __syncthreads();
    uint32_t r = s_warp[w] + inc - v;
    if (total) *total = s_warp[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t *in, int64_t n,
                                                                   uint32_t *partials) {
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        int64_t idx = base + j * kScanThreads + threadIdx.x;
        if (idx < n) s += in[idx];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ uint32_t sw[kScanThreads / 32];
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; w++) t += sw[w];
        partials[blockIdx.x] = t;
    }
}

// single block, 1024 threads: in-place exclusive scan of the partials
__global__ void __launch_bounds__(1024) scan_partials_kernel(uint32_t *partials, int64_t m,
                                                             uint32_t *total) {
    __shared__ uint32_t s_warp[33];
    uint32_t carry = 0;
    for (int64_t base = 0; base < m; base += 1024) {
        int64_t idx = base + threadIdx.x;
        uint32_t v = idx < m ? partials[idx] : 0u;
        uint32_t tot;
        uint32_t ex = block_excl_scan(v, s_warp, &tot);
        if (idx < m) partials[idx] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const uint32_t *in, uint32_t *out,
                                                                 int64_t n,
                                                                 const uint32_t *partials) {
    __shared__ uint32_t s_warp[33];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    // blocked arrangement: thread t owns items [base + t*8, base + t*8 + 8)
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        int64_t idx = base + (int64_t)threadIdx.x * kScanItems + j;
        v[j] = idx < n ? in[idx] : 0u;
        s += v[j];
    }
    uint32_t ex = block_excl_scan(s, s_warp, nullptr) + partials[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        int64_t idx = base + (int64_t)threadIdx.x * kScanItems + j;
        if (idx < n) out[idx] = ex;
        ex += v[j];
    }
}

// ---------------------------------------------------------------- radix ----
constexpr int RB = kRadixThreads;
constexpr int RI = kRadixItems;
constexpr int RT = kRadixTile;
constexpr int RW = RB / 32;

template <typename K>
__device__ __forceinline__ K sentinel() { return (K)~(K)0; }

template <typename K>
struct PassArgs {
    const K *kin;
    const uint32_t *vin;
    K *kout;
    uint32_t *vout;
    const uint32_t *n_dev;
    int64_t n_cap;
    int shift;
    const unsigned long long *key_base;
    const uint32_t *npass_dev;
    int pass_index;
    int drop_sentinel;
    uint32_t *hist;
    int64_t ntiles;
};

template <typename K>
__device__ __forceinline__ bool pass_skipped(const PassArgs<K> &p) {
    return p.npass_dev && (uint32_t)p.pass_index >= *p.npass_dev;
}

template <typename K>
__device__ __forceinline__ int64_t pass_count(const PassArgs<K> &p) {
    if (!p.n_dev) return p.n_cap;
    int64_t n = (int64_t)*p.n_dev;
    return n < p.n_cap ? n : p.n_cap;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, K base, int shift) {
    return (uint32_t)(((K)(k - base)) >> shift) & 255u;
}

template <typename K>
__global__ void __launch_bounds__(RB) radix_upsweep_kernel(PassArgs<K> p) {
    if (pass_skipped(p)) return;
    __shared__ uint32_t h[RW][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int j = threadIdx.x; j < RW * 256; j += RB) (&h[0][0])[j] = 0;
    __syncthreads();
    const int64_t n = pass_count(p);
    const int64_t base = (int64_t)blockIdx.x * RT + (int64_t)w * (RI * 32);
    const K kb = p.key_base ? (K)*p.key_base : (K)0;
    if ((int64_t)blockIdx.x * RT < n) {
#pragma unroll 4
        for (int r = 0; r < RI; r++) {
            const int64_t idx = base + r * 32 + lane;
            bool valid = idx < n;
            K k = valid ? p.kin[idx] : (K)0;
            if (p.drop_sentinel && k == sentinel<K>()) valid = false;
            const uint32_t act = __ballot_sync(0xffffffffu, valid);
            if (valid) {
                const uint32_t d = digit_of(k, kb, p.shift);
                const uint32_t peers = __match_any_sync(act, d);
                if (lane == __ffs(peers) - 1) h[w][d] += __popc(peers);
            }
            __syncwarp();
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RB) {
        uint32_t s = 0;
#pragma unroll
        for (int j = 0; j < RW; j++) s += h[j][d];
        p.hist[(int64_t)d * p.ntiles + blockIdx.x] = s;
    }
}

template <typename K>
struct DownSmem {
    K keys[RT];
    uint32_t vals[RT];
    uint32_t wcnt[RW][256];
    uint32_t dstart[256];
    uint32_t gbase[256];
    uint32_t s_warp[33];
    uint32_t tile_n;
};

template <typename K>
__global__ void __launch_bounds__(RB) radix_downsweep_kernel(PassArgs<K> p) {
    if (pass_skipped(p)) return;
    const int64_t n = pass_count(p);
    if ((int64_t)blockIdx.x * RT >= n) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DownSmem<K> &S = *reinterpret_cast<DownSmem<K> *>(smem_raw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int j = threadIdx.x; j < RW * 256; j += RB) (&S.wcnt[0][0])[j] = 0;
    for (int d = threadIdx.x; d < 256; d += RB) S.gbase[d] = p.hist[(int64_t)d * p.ntiles + blockIdx.x];
    __syncthreads();

    const K kb = p.key_base ? (K)*p.key_base : (K)0;
    const int64_t base = (int64_t)blockIdx.x * RT + (int64_t)w * (RI * 32);
    K keys[RI];
    uint32_t vals[RI];
    uint32_t loc[RI];
    uint32_t valid_bits = 0;
#pragma unroll
    for (int r = 0; r < RI; r++) {
        const int64_t idx = base + r * 32 + lane;
        bool valid = idx < n;
        K k = valid ? p.kin[idx] : (K)0;
        if (p.drop_sentinel && k == sentinel<K>()) valid = false;
        keys[r] = k;
        vals[r] = valid ? (p.vin ? p.vin[idx] : (uint32_t)idx) : 0u;
        const uint32_t act = __ballot_sync(0xffffffffu, valid);
        uint32_t prior = 0, peers = 0, d = 0;
        if (valid) {
            d = digit_of(k, kb, p.shift);
            peers = __match_any_sync(act, d);
            prior = S.wcnt[w][d];
            loc[r] = prior + __popc(peers & lt_mask);
            valid_bits |= 1u << r;
        } else {
            loc[r] = 0;
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) S.wcnt[w][d] = prior + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, tile totals, then scan over digits
    uint32_t tot = 0;
    for (int d = threadIdx.x; d < 256; d += RB) {
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < RW; j++) {
            uint32_t c = S.wcnt[j][d];
            S.wcnt[j][d] = run;
            run += c;
        }
        tot = run;
    }
    uint32_t tile_total;
    const uint32_t ds = block_excl_scan(threadIdx.x < 256 ? tot : 0u, S.s_warp, &tile_total);
    if (threadIdx.x < 256) S.dstart[threadIdx.x] = ds;
    if (threadIdx.x == 0) S.tile_n = tile_total;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RI; r++) {
        if (valid_bits & (1u << r)) {
            const uint32_t d = digit_of(keys[r], kb, p.shift);
            const uint32_t pos = S.dstart[d] + S.wcnt[w][d] + loc[r];
            S.keys[pos] = keys[r];
            S.vals[pos] = vals[r];
        }
    }
    __syncthreads();
    const uint32_t tn = S.tile_n;
    for (uint32_t i = threadIdx.x; i < tn; i += RB) {
        const K k = S.keys[i];
        const uint32_t d = digit_of(k, kb, p.shift);
        const uint32_t o = S.gbase[d] + (i - S.dstart[d]);
        p.kout[o] = k;
        p.vout[o] = S.vals[i];
    }
}

}  // namespace

// per-device kernel attributes; called once per context after cudaSetDevice
cudaError_t radix_init_attributes() {
    cudaError_t e = cudaFuncSetAttribute(radix_downsweep_kernel<unsigned long long>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(DownSmem<unsigned long long>));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(radix_downsweep_kernel<uint32_t>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(DownSmem<uint32_t>));
}

int64_t scan_partials_needed(int64_t n) { return (n + kScanChunk - 1) / kScanChunk + 1; }

void launch_scan_exclusive(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *total,
                           const ScanWorkspace &ws, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t blocks = (n + kScanChunk - 1) / kScanChunk;
    scan_reduce_kernel<<<(unsigned)blocks, kScanThreads, 0, s>>>(in, n, ws.partials);
    scan_partials_kernel<<<1, 1024, 0, s>>>(ws.partials, blocks, total);
    scan_down_kernel<<<(unsigned)blocks, kScanThreads, 0, s>>>(in, out, n, ws.partials);
}

template <typename K>
void launch_radix_pass(const K *kin, const uint32_t *vin, K *kout, uint32_t *vout,
                       const uint32_t *n_dev, int64_t n_cap, int shift,
                       const unsigned long long *key_base, const uint32_t *npass_dev,
                       int pass_index, bool drop_sentinel, uint32_t *hist,
                       const ScanWorkspace &ws, cudaStream_t s) {
    if (n_cap <= 0) return;
    PassArgs<K> p;
    p.kin = kin;
    p.vin = vin;
    p.kout = kout;
    p.vout = vout;
    p.n_dev = n_dev;
    p.n_cap = n_cap;
    p.shift = shift;
    p.key_base = key_base;
    p.npass_dev = npass_dev;
    p.pass_index = pass_index;
    p.drop_sentinel = drop_sentinel ? 1 : 0;
    p.hist = hist;
    p.ntiles = radix_tiles(n_cap);
    radix_upsweep_kernel<K><<<(unsigned)p.ntiles, RB, 0, s>>>(p);
    launch_scan_exclusive(hist, hist, 256 * p.ntiles, nullptr, ws, s);
    const size_t smem = sizeof(DownSmem<K>);
    radix_downsweep_kernel<K><<<(unsigned)p.ntiles, RB, smem, s>>>(p);
}

template void launch_radix_pass<unsigned long long>(const unsigned long long *, const uint32_t *,
                                                    unsigned long long *, uint32_t *,
                                                    const uint32_t *, int64_t, int,
                                                    const unsigned long long *, const uint32_t *,
                                                    int, bool, uint32_t *, const ScanWorkspace &,
                                                    cudaStream_t);
template void launch_radix_pass<uint32_t>(const uint32_t *, const uint32_t *, uint32_t *,
                                          uint32_t *, const uint32_t *, int64_t, int,
                                          const unsigned long long *, const uint32_t *, int,
                                          bool, uint32_t *, const ScanWorkspace &, cudaStream_t);

}  // namespace gsr
