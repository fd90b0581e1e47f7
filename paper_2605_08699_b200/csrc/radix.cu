// radix.cu -- stable LSD radix sort, Onesweep style (one kernel per 8-bit
// digit with decoupled look-back), for
//   (a) the stable f64 depth sort replacing np.argsort(depths, kind="stable")
//       (render.py:293-302): keys are the IEEE bits of z (> 0, so unsigned
//       order == numeric order); values are Gaussian indices; the first pass
//       drops culled Gaussians (sentinel key ~0), which is the
//       order-preserving compaction of render.py:279;
//   (b) the stable tile sort of the rank-major (tile, depth rank) list.
// Stability gives the reference's tie order (equal depths keep index order).
//
// Per sort: one histogram kernel computes every pass's digit histogram in one
// read of the keys (for slice A it also compacts: appends the slice's (span
// key, index) pairs, slice.cu).  Every pass kernel then plans in its
// prologue (the plan was a 1-block kernel of its own): it turns its digit
// histogram into global digit offsets and finds the passes whose digit is
// constant (inactive, skipped: an identity permutation), hence which
// ping-pong buffer it reads; pass 0 publishes the schedule.  Each pass: a block takes a 4096-key tile in ticket order, ranks its
// keys stably (per-warp digit lane masks + digit counters), publishes its digit
// counts, looks back over predecessor tiles per digit for its global
// position, and scatters through shared memory so global writes are
// coalesced runs.  Counts come from device memory: no host synchronisation.
#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

constexpr int RB = kRadixThreads;
constexpr int RW = RB / 32;
template <typename K>
struct Cfg {
    static constexpr int RI = radix_items((int)sizeof(K));  // items per thread
    static constexpr int RT = RB * RI;                      // items per tile
};

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1u;

template <typename K>
__device__ __forceinline__ K sentinel() { return (K)~(K)0; }

// Look-back status words carry flag and count in one 32-bit word, so relaxed
// GPU-scope accesses suffice (acquire would emit an L1 invalidate, CCTL.IVALL,
// on every poll).
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename K>
struct SortArgs {
    K *keys[2];
    uint32_t *vals[2];
    int implicit_first_vals;   // first pass: value = input index
    int drop_sentinel;         // first pass: drop keys == ~0
    const uint32_t *n_dev;     // items after the first pass (nullable -> n_first)
    int64_t n_first;           // items read by the first pass
    int64_t n_cap;             // capacity for n_dev
    int64_t tiles;             // tiles per pass (grid)
    int passes;
    int force_first;           // pass 0 always active (compaction)
    uint32_t *hist;            // [passes][256]: histogram, then exclusive offsets
    uint32_t *status;          // [passes][tiles][256]
    uint32_t *tickets;         // [passes]
    uint32_t *sched;           // [0..7] active, [8..15] src buffer, [16] final buffer
    uint32_t *npass_out;       // nullable: number of active passes
    SpanKeys span;             // 32-bit sorts: keys derived from 64-bit ones (hist kernel)
};

template <typename K>
__device__ __forceinline__ int64_t first_count(const SortArgs<K> &a) {
    if (a.n_first >= 0) return a.n_first;
    int64_t n = (int64_t)*a.n_dev;
    return n < a.n_cap ? n : a.n_cap;
}

template <typename K>
__device__ __forceinline__ int64_t items_after_first(const SortArgs<K> &a) {
    if (!a.n_dev) return a.n_first;
    int64_t n = (int64_t)*a.n_dev;
    return n < a.n_cap ? n : a.n_cap;
}

template <typename K>
__global__ void __launch_bounds__(RB) radix_hist_kernel(SortArgs<K> a) {
    __shared__ uint32_t h[8][256];
    {   // zero the look-back status words and tickets of every pass (the
        // passes run after this kernel; only hist is cleared by memset)
        uint32_t *z = a.status;
        const int64_t nz = (int64_t)a.passes * a.tiles * 256 + 8;
        for (int64_t j = (int64_t)blockIdx.x * RB + threadIdx.x; j < nz; j += (int64_t)gridDim.x * RB)
            z[j] = 0u;
    }
    __shared__ uint32_t s_kept;
    for (int j = threadIdx.x; j < 8 * 256; j += RB) (&h[0][0])[j] = 0;
    if (threadIdx.x == 0) s_kept = 0u;
    __syncthreads();
    uint32_t kept_local = 0u;  // keys kept by the first pass (span.count_out)
    // compacting span keys (slice A): read n_src source keys, append the kept
    // ones; the passes then read *n_dev = *count_out items
    const bool compact = sizeof(K) == 4 && a.span.src && a.span.compact;
    const int64_t n = compact ? a.span.n_src : first_count(a);
    const K *keys = a.keys[0];
    SpanMap sm{0ull, 0ull, 0};
    uint32_t limit = 0xffffffffu;
    if (sizeof(K) == 4 && a.span.src) {
        sm = span_map(*a.span.kmin, *a.span.kmax, a.span.bits);
        if (a.span.limit) limit = *a.span.limit;
    }
    // kHU keys per thread per step, all loads issued before any use (the
    // loop is otherwise one global latency per key)
    constexpr int kHU = 8;
    const int64_t stride = (int64_t)gridDim.x * RB;
    if (compact) {
        // (k32, index) of the kept keys appended, one global atomic per
        // block step of RB * kHU keys (the block's warps take consecutive
        // ranges of it); the order among equal k32 is restored by the depth
        // fix-up, which orders runs by (f64 key, index)
        __shared__ uint32_t s_wc[RB / 32 + 1];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int64_t c0 = (int64_t)blockIdx.x * RB * kHU; c0 < n; c0 += stride * kHU) {
            uint32_t q[kHU];
            uint32_t bal[kHU];
            uint32_t wcnt = 0u;
#pragma unroll
            for (int u = 0; u < kHU; u++) {
                const int64_t i = c0 + (int64_t)u * RB + threadIdx.x;
                const unsigned long long k = i < n ? a.span.src[i] : ~0ull;
                q[u] = k != ~0ull ? span_key(sm, k) : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < kHU; u++) {
                bal[u] = __ballot_sync(0xffffffffu, q[u] <= limit);
                wcnt += (uint32_t)__popc(bal[u]);
            }
            if (lane == 0) s_wc[w] = wcnt;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t t = 0u;
                for (int j = 0; j < RB / 32; j++) {
                    const uint32_t c = s_wc[j];
                    s_wc[j] = t;
                    t += c;
                }
                s_wc[RB / 32] = t ? atomicAdd(a.span.count_out, t) : 0u;
            }
            __syncthreads();
            uint32_t pos = s_wc[RB / 32] + s_wc[w];
#pragma unroll
            for (int u = 0; u < kHU; u++) {
                if (q[u] <= limit) {
                    const uint32_t at = pos + (uint32_t)__popc(bal[u] & ((1u << lane) - 1u));
                    a.keys[0][at] = (K)q[u];
                    a.vals[0][at] = (uint32_t)(c0 + (int64_t)u * RB + threadIdx.x);
#pragma unroll
                    for (int p = 0; p < (int)sizeof(K); p++)
                        if (p < a.passes) atomicAdd(&h[p][(q[u] >> (8 * p)) & 255u], 1u);
                }
                pos += (uint32_t)__popc(bal[u]);
            }
            __syncthreads();  // s_wc reused by the next step
        }
    }
    for (int64_t i0 = (int64_t)blockIdx.x * RB + threadIdx.x; !compact && i0 < n; i0 += stride * kHU) {
        K kk[kHU];
        unsigned long long k64[kHU];
        const bool span = sizeof(K) == 4 && a.span.src;
#pragma unroll
        for (int u = 0; u < kHU; u++) {
            const int64_t i = i0 + u * stride;
            if (span) k64[u] = i < n ? a.span.src[i] : ~0ull;
            else kk[u] = i < n ? keys[i] : sentinel<K>();
        }
#pragma unroll
        for (int u = 0; u < kHU; u++) {
            const int64_t i = i0 + u * stride;
            if (i >= n) continue;
            K k;
            if (span) {  // span key of the depth bits (slice A: above the limit -> dropped)
                const uint32_t q = span_key(sm, k64[u]);
                k = (k64[u] == ~0ull || q > limit) ? sentinel<K>() : (K)q;
                a.keys[0][i] = k;
            } else {
                k = kk[u];
            }
            if (a.drop_sentinel && k == sentinel<K>()) continue;
            kept_local++;
#pragma unroll
            for (int p = 0; p < (int)sizeof(K); p++)
                if (p < a.passes) atomicAdd(&h[p][(uint32_t)(k >> (8 * p)) & 255u], 1u);
        }
    }
    if (a.span.count_out && !compact && kept_local) atomicAdd(&s_kept, kept_local);
    __syncthreads();
    for (int j = threadIdx.x; j < a.passes * 256; j += RB) {
        const uint32_t c = (&h[0][0])[j];
        if (c) atomicAdd(a.hist + j, c);
    }
    if (a.span.count_out && !compact && threadIdx.x == 0 && s_kept)
        atomicAdd(a.span.count_out, s_kept);
}

template <typename K>
struct PassSmem {
    K keys[Cfg<K>::RT];
    uint32_t vals[Cfg<K>::RT];
    uint32_t wcnt[RW][256];
    uint32_t wmask[RW][256];
    uint32_t hcnt[256];
    uint32_t dstart[256];
    uint32_t gbase[256];
    uint32_t s_warp[33];
    uint32_t off[256];   // this pass's exclusive digit offsets (the folded plan)
    uint32_t tile_n;
    uint32_t ticket;
    int64_t nf, na;      // items read by the first active pass / by the others
};

template <typename K>
__global__ void __launch_bounds__(RB, 1024 / RB) onesweep_pass_kernel(SortArgs<K> a, int pass) {
    constexpr int RI = Cfg<K>::RI, RT = Cfg<K>::RT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem<K> &S = *reinterpret_cast<PassSmem<K> *>(smem_raw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // the prologue's global reads in one round trip: the tile ticket (the
    // grid is sized for the capacity, and tiles past the items -- most of
    // them for a front slice -- leave before any set-up), the item counts and
    // every pass's digit histogram (the plan below)
    uint32_t hc[sizeof(K)];
#pragma unroll
    for (int p = 0; p < (int)sizeof(K); p++)
        hc[p] = (p < a.passes && threadIdx.x < 256) ? a.hist[p * 256 + threadIdx.x] : 0u;
    if (threadIdx.x == 0) S.ticket = atomicAdd(a.tickets + pass, 1u);
    if (threadIdx.x == 32) {
        S.nf = first_count(a);
        S.na = items_after_first(a);
    }
    __syncthreads();
    int64_t t = S.ticket;
    const int64_t nf = S.nf, na = S.na;
    if (t > 0 && t * RT >= (nf > na ? nf : na)) return;  // (ticket 0 publishes the plan)
    // the plan, folded into every pass (one kernel boundary less per sort):
    // a pass is active unless its digit is constant (pass 0 forced when it
    // compacts); buffers alternate over the active passes; this pass's
    // digit offsets are the exclusive scan of its histogram
    uint32_t act_mask = 0u;
#pragma unroll
    for (int p = 0; p < (int)sizeof(K); p++) {
        if (p >= a.passes) break;
        const uint32_t c = hc[p];
        const int nz = __syncthreads_count(c != 0u);
        if (nz > 1 || (p == 0 && a.force_first)) act_mask |= 1u << p;
        if (p == pass) {
            const uint32_t ex = block_excl_scan_u32(c, S.s_warp, nullptr);
            if (threadIdx.x < 256) S.off[threadIdx.x] = ex;
        }
    }
    if (pass == 0 && t == 0 && threadIdx.x == 0) {  // for the sort's consumers
        uint32_t cur = 0u, np = 0u;
        for (int p = 0; p < 8; p++) {
            const uint32_t act = (act_mask >> p) & 1u;
            a.sched[p] = act;
            a.sched[8 + p] = cur;
            cur ^= act;
            np += act;
        }
        a.sched[16] = cur;
        if (a.npass_out) *a.npass_out = np;
    }
    if (!((act_mask >> pass) & 1u)) return;
    const uint32_t src = (uint32_t)(__popc(act_mask & ((1u << pass) - 1u)) & 1);
    // first active pass: reads the producer's buffer (0) with n_first items
    const bool first = (act_mask & ((1u << pass) - 1u)) == 0u;
    const int64_t n = first ? nf : na;
    // persistent: the grid is bounded (SMs x 2), each CTA takes tiles in
    // ticket order until none is left (a tile only waits on lower tickets,
    // all held by running CTAs, so the look-back always progresses)
    for (;; ) {
    if (t * RT >= n) return;
    const bool dig = threadIdx.x < 256;  // digit owner (RB >= 256)
    uint32_t *st = a.status + ((int64_t)pass * a.tiles) * 256;
    // (ternaries, not a.keys[src]: runtime-indexed param arrays go to local memory)
    const K *kin = src ? a.keys[1] : a.keys[0];
    const uint32_t *vin = (first && a.implicit_first_vals) ? nullptr : (src ? a.vals[1] : a.vals[0]);
    K *kout = src ? a.keys[0] : a.keys[1];
    uint32_t *vout = src ? a.vals[0] : a.vals[1];
    const bool drop = first && a.drop_sentinel;
    const int shift = 8 * pass;
    const uint32_t lt_mask = (1u << lane) - 1u;

    // ---- stable in-tile ranking ----------------------------------------
    const int64_t base = t * RT + (int64_t)w * (RI * 32);
    K keys[RI];
    uint32_t vals[RI];
    uint32_t loc[RI];
    uint32_t valid_bits = 0;
    // all loads first (RI independent requests in flight per thread)
#pragma unroll
    for (int r = 0; r < RI; r++) {
        const int64_t idx = base + r * 32 + lane;
        keys[r] = idx < n ? __ldg(kin + idx) : sentinel<K>();
        vals[r] = idx < n ? (vin ? __ldg(vin + idx) : (uint32_t)idx) : 0u;
        if (idx < n && !(drop && keys[r] == sentinel<K>())) valid_bits |= 1u << r;
    }
    // (the counters are cleared while the loads are in flight)
    for (int j = threadIdx.x; j < RW * 256; j += RB) (&S.wcnt[0][0])[j] = 0;
    for (int j = threadIdx.x; j < RW * 256; j += RB) (&S.wmask[0][0])[j] = 0;
    if (dig) S.hcnt[threadIdx.x] = 0;
    __syncthreads();
    // tile digit counts first, published as aggregates before the (slower)
    // stable ranking so successors' look-back can proceed meanwhile
#pragma unroll
    for (int r = 0; r < RI; r++)
        if ((valid_bits >> r) & 1u) atomicAdd(&S.hcnt[(uint32_t)(keys[r] >> shift) & 255u], 1u);
    __syncthreads();
    const uint32_t tot = dig ? S.hcnt[threadIdx.x] : 0u;
    if (t > 0 && dig) st_release_u32(st + t * 256 + threadIdx.x, kFlagAgg | tot);
    // peers of every round first (independent MATCH ops pipeline), then one
    // shared atomic per (round, digit group) by its leader -- a warp's
    // shared-memory atomics to one address complete in program order, so the
    // returned prior counts are stable -- broadcast with a shuffle
    uint32_t peers[RI];
    // Peers (lanes of the warp with the same digit in this round) through a
    // per-warp digit -> lane-mask table: shared atomicOr, read, clear by the
    // lowest peer.  (MATCH.ANY gives the same masks but was the pass's
    // bottleneck: 0.164 -> 0.127 ms for a 2.65M-key 3-pass sort.)
    uint32_t *wm = S.wmask[w];
#pragma unroll
    for (int r = 0; r < RI; r++) {
        const bool valid = (valid_bits >> r) & 1u;
        const uint32_t dg = (uint32_t)(keys[r] >> shift) & 255u;
        if (valid) atomicOr(&wm[dg], 1u << lane);
        __syncwarp();
        peers[r] = valid ? wm[dg] : 0u;
        __syncwarp();
        if (valid && (peers[r] & lt_mask) == 0u) wm[dg] = 0u;  // lowest peer clears
        __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < RI; r++) {
        const bool valid = (valid_bits >> r) & 1u;
        const int leader = valid ? __ffs(peers[r]) - 1 : lane;
        uint32_t old = 0;
        if (valid && lane == leader)
            old = atomicAdd(&S.wcnt[w][(uint32_t)(keys[r] >> shift) & 255u], __popc(peers[r]));
        const uint32_t base = __shfl_sync(0xffffffffu, old, leader);
        loc[r] = valid ? base + __popc(peers[r] & lt_mask) : 0u;
    }
    __syncthreads();
    if (dig) {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < RW; j++) {
            const uint32_t c = S.wcnt[j][d];
            S.wcnt[j][d] = run;
            run += c;
        }
    }
    // ---- publish tile counts, look back per digit ----------------------
    // One thread per digit walks back over predecessor tiles kLbWindow at a
    // time (independent loads in flight), summing aggregates until it meets
    // an inclusive prefix.
    if (dig) {
#ifndef GSR_LB_WINDOW
#define GSR_LB_WINDOW 8
#endif
        constexpr int kLbWindow = GSR_LB_WINDOW;
        const int d = threadIdx.x;
#ifdef GSR_RADIX_NO_LOOKBACK  // microbenchmark only (tools/radix_bench.cu): wrong output
        if (true) {
#else
        if (t == 0) {
#endif
            st_release_u32(st + d, kFlagInc | tot);
            S.gbase[d] = S.off[d];
        } else {
            uint32_t excl = 0;
            int64_t tp = t - 1;
            while (true) {
                uint32_t s[kLbWindow];
#pragma unroll
                for (int i = 0; i < kLbWindow; i++)
                    s[i] = tp - i >= 0 ? ld_acquire_u32(st + (tp - i) * 256 + d) : kFlagInc;
                int used = 0;
                bool done = false;
#pragma unroll
                for (int i = 0; i < kLbWindow; i++) {
                    if (done || used < i) continue;  // stop at the first gap
                    const uint32_t f = s[i] >> 30;
                    if (f == 0u) continue;           // not published yet: retry from here
                    excl += s[i] & kValMask;
                    used = i + 1;
                    if (f == 2u) done = true;
                }
                if (done) break;
                tp -= used;
            }
            st_release_u32(st + t * 256 + d, kFlagInc | (excl + tot));
            S.gbase[d] = S.off[d] + excl;
        }
    }
    uint32_t tile_total;
    const uint32_t ds = block_excl_scan_u32(tot, S.s_warp, &tile_total);
    if (dig) S.dstart[threadIdx.x] = ds;
    if (threadIdx.x == 0) S.tile_n = tile_total;
    __syncthreads();
    // ---- scatter through shared memory, then coalesced runs ------------
#pragma unroll
    for (int r = 0; r < RI; r++) {
        if (valid_bits & (1u << r)) {
            const uint32_t d = (uint32_t)(keys[r] >> shift) & 255u;
            const uint32_t pos = S.dstart[d] + S.wcnt[w][d] + loc[r];
            S.keys[pos] = keys[r];
            S.vals[pos] = vals[r];
        }
    }
    __syncthreads();
    const uint32_t tn = S.tile_n;
    for (uint32_t i = threadIdx.x; i < tn; i += RB) {
        const K k = S.keys[i];
        const uint32_t d = (uint32_t)(k >> shift) & 255u;
        const uint32_t o = S.gbase[d] + (i - S.dstart[d]);
        kout[o] = k;
        vout[o] = S.vals[i];
    }
    __syncthreads();  // shared state is reused by the next tile
    if (threadIdx.x == 0) S.ticket = atomicAdd(a.tickets + pass, 1u);
    __syncthreads();
    t = S.ticket;
    }
}

}  // namespace

cudaError_t radix_init_attributes() {
    cudaError_t e = cudaFuncSetAttribute(onesweep_pass_kernel<unsigned long long>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(PassSmem<unsigned long long>));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(onesweep_pass_kernel<uint32_t>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(PassSmem<uint32_t>));
    // maximum shared-memory carveout so occupancy is register-limited, not smem-limited
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(onesweep_pass_kernel<unsigned long long>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(onesweep_pass_kernel<uint32_t>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return e;
}

size_t sort_work_bytes(int64_t n_items_cap, int passes, int key_bytes) {
    const int64_t tiles = radix_tiles(n_items_cap, key_bytes);
    return sizeof(uint32_t) * ((size_t)passes * 256 + (size_t)passes * tiles * 256 + 8 + 32);
}

template <typename K>
int launch_onesweep_sort(K *keys0, K *keys1, uint32_t *vals0, uint32_t *vals1,
                         bool implicit_first_vals, bool drop_sentinel, const uint32_t *n_dev,
                         int64_t n_first, int64_t n_cap, int passes, bool force_first,
                         void *work, uint32_t *sched, uint32_t *npass_out, int sms,
                         cudaStream_t s, const KMark &mark, const SpanKeys &span) {
    SortArgs<K> a;
    a.span = span;
    a.keys[0] = keys0;
    a.keys[1] = keys1;
    a.vals[0] = vals0;
    a.vals[1] = vals1;
    a.implicit_first_vals = implicit_first_vals ? 1 : 0;
    a.drop_sentinel = drop_sentinel ? 1 : 0;
    a.n_dev = n_dev;
    a.n_first = n_first;
    a.n_cap = n_cap;
    const int64_t n_items_cap = n_first > n_cap ? n_first : n_cap;  // n_first < 0: from n_dev
    a.tiles = radix_tiles(n_items_cap, (int)sizeof(K));
    a.passes = passes;
    a.force_first = force_first ? 1 : 0;
    uint32_t *w = reinterpret_cast<uint32_t *>(work);
    a.hist = w;
    a.status = w + passes * 256;
    a.tickets = a.status + (size_t)passes * a.tiles * 256;
    a.sched = sched;
    a.npass_out = npass_out;
    if (!span.hist_zeroed)
        cudaMemsetAsync(work, 0, sizeof(uint32_t) * (size_t)passes * 256, s);  // hist only
    int launches = 0;
    if (n_items_cap > 0) {
        int64_t hb = (n_items_cap + RB * 16 - 1) / (RB * 16);
        if (hb > sms * 4) hb = sms * 4;
        if (hb < 1) hb = 1;
        radix_hist_kernel<K><<<(unsigned)hb, RB, 0, s>>>(a);
        mark(sizeof(K) == 8 ? "radix64_hist" : "radix32_hist");
        launches++;
    }
    {   // (pass 0 also publishes the schedule, so it always runs)
        for (int p = 0; p < passes; p++) {
            onesweep_pass_kernel<K><<<(unsigned)std::max<int64_t>(
                                          1, std::min<int64_t>(a.tiles, (int64_t)sms * 2)),
                                      RB, sizeof(PassSmem<K>), s>>>(a, p);
            mark(sizeof(K) == 8 ? "radix64_pass" : "radix32_pass");
            launches++;
        }
    }
    return launches;
}

template int launch_onesweep_sort<unsigned long long>(unsigned long long *, unsigned long long *,
                                                      uint32_t *, uint32_t *, bool, bool,
                                                      const uint32_t *, int64_t, int64_t, int,
                                                      bool, void *, uint32_t *, uint32_t *,
                                                      int, cudaStream_t, const KMark &,
                                                      const SpanKeys &);
template int launch_onesweep_sort<uint32_t>(uint32_t *, uint32_t *, uint32_t *, uint32_t *, bool,
                                            bool, const uint32_t *, int64_t, int64_t, int, bool,
                                            void *, uint32_t *, uint32_t *, int,
                                            cudaStream_t, const KMark &, const SpanKeys &);

}  // namespace gsr
