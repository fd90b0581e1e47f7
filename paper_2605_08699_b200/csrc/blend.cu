// blend.cu -- K6: per-tile (32x16) front-to-back alpha blending.
//
// Restates _composite_kernel's per-pixel arithmetic (render.py:383-427) with
// its exact f32 operation order and glibc expf, so frames are float-identical
// to the reference:
//   dx = (f32(ix) + 0.5) - u
//   power = -0.5 * (((ia*dx)*dx + ((2*ib)*dy)*dx) + (ic*dy)*dy)
//   alpha = min(op * expf(power), 0.99); w = T*alpha; rgb += w*c;
//   T = T*(1 - alpha); the pixel stops once T < 1/255
// and a pixel takes a splat only inside the splat's exact row interval
// [floor(mid - span), ceil(mid + span) + 1) of render.py:384-397 and row range
// render.py:329-333 -- the tile lists are a superset, so order and set of
// contributions per pixel are the reference's.  After the list: rgb += T*bg
// (render.py:423-427), then the u8 conversion of render.py:470+484-485.
//
// Layout: a work item is one warp's kSets x 32 pixels, pixel rows of a
// 32x16 tile (lane = column; the two rows composited interleaved), taken from a work queue by a persistent grid (see
// blend_kernel).  A warp walks the tile list 32 splats at a time: lane j
// loads splat j's record (128-bit loads), computes its row interval (exact,
// row_xlr) as a 32-bit pixel-coverage mask and stages the splat's row terms
// in shared memory (structure of arrays, so any lane can read any splat
// without bank conflicts).  A 5-step shuffle
// transpose turns the 32 splat masks into 32 per-pixel masks; each lane then
// walks its OWN covering splats in depth order, so a warp iteration does
// useful work on every lane that still has splats (not just on the lanes a
// given splat covers).  Warps leave as soon as all their 32 pixels are
// saturated (warp-vote early termination); no block barriers in the loop.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace gsr {

namespace {

constexpr int kBlendThreads = 128;              // 4 warps: finer occupancy granularity
constexpr int kWarps = kBlendThreads / 32;

__device__ __forceinline__ uint32_t span_mask(int x0, int x1, int X) {
    // columns [x0, x1) intersected with [X, X+32), as a 32-bit mask
    int a = x0 - X, b = x1 - X;
    a = a < 0 ? 0 : a;
    b = b > 32 ? 32 : b;
    if (a >= b) return 0u;
    const uint32_t hi = b >= 32 ? 0xffffffffu : (1u << b) - 1u;
    return hi & ~((1u << a) - 1u);
}

// Coverage of one pixel row of the tile by one splat (render.py:329-333 row
// range, 383-397 interval), as a 32-bit column mask.
__device__ __forceinline__ uint32_t row_mask(const float4 &A, const float4 &B, float rinv, bool fast,
                                             int iy, int lo, int hi, int X, int width) {
    if (iy < lo || iy >= hi) return 0u;
    const float py = (float)iy + 0.5f;
    if (fast) {
        float xl, xr;
        const int k = row_xlr(A.x, A.y, A.z, A.w, B.x, B.y, rinv, py, xl, xr);
        if (k == 0) return 0u;
        if (k > 0 && fabsf(xl) < 0x1p30f && fabsf(xr) < 0x1p30f)
            return span_mask(__float2int_rd(xl), min(__float2int_ru(xr) + 1, width), X);
    }
    int x0, x1;
    if (!row_interval(A.x, A.y, A.z, A.w, B.x, B.y, py, width, x0, x1)) return 0u;
    return span_mask(x0, x1, X);
}

// 32x32 bit-matrix transpose across a warp: on entry lane j holds row j
// (bit p = element (j, p)); on exit lane p holds column p (bit j).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int s = 16, k = 0; s >= 1; s >>= 1, k++) {
        const uint32_t lo_mask = (s == 16) ? 0x0000ffffu : (s == 8) ? 0x00ff00ffu
                               : (s == 4) ? 0x0f0f0f0fu : (s == 2) ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
        x = (lane & s) ? ((x & ~lo_mask) | ((y >> s) & lo_mask))
                       : ((x & lo_mask) | ((y << s) & ~lo_mask));
    }
    return x;
}

// glibc expf constants (see common.cuh), in constant memory so the DFMAs take
// them as operands instead of rematerialising 64-bit immediates per call
__constant__ double kExpK[4] = {
    -0.5 * 0x1.71547652b82fep+0 * 32.0,                // -0.5 * InvLn2N (see expf_blend)
    0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0,         // C0
    0x1.ebfce50fac4f3p-3 / 32.0 / 32.0,                // C1
    0x1.62e42ff0c52d6p-1 / 32.0,                       // C2
};

__device__ __noinline__ float expf_special(float x, const unsigned long long *tab) {
#ifdef GSR_TAB_SPLIT
    (void)tab;  // the shared table is split into word arrays: use the constant one
    return glibc_expf_tab(x, kExp2fTab);
#else
    return glibc_expf_tab(x, tab);
#endif
}

// glibc expf for |x| < 88 (its main path) with the 2^(i/32) table in shared
// memory; other x go to the full restatement.  Bit-identical to
// glibc_expf_tab.
struct ExpK {
    double inv_ln2n, c0, c1, c2;
};

// expf(-0.5f * q) for the quadratic form q.  -0.5f * q is exact in f32
// (short of underflow, where both give 1.0f), so the factor is folded into
// the f64 constant: InvLn2N * (-0.5 q) == (-0.5 InvLn2N) * q exactly, and
// |-0.5 q| < 88 <=> |q| < 176.
template <bool kChecked>
__device__ __forceinline__ float expf_blend(float q, const unsigned long long *tab,
                                            uint32_t tab_s, const ExpK &K) {
    if (kChecked && !(fabsf(q) < 176.0f)) return expf_special(-0.5f * q, tab);
    const double kShift = 0x1.8p+52;
    const double qd = (double)q;
    double kd = __fma_rn(K.inv_ln2n, qd, kShift);  // K.inv_ln2n = -0.5 * InvLn2N
    const uint32_t ki = (uint32_t)__double2loint(kd);
    kd = __dsub_rn(kd, kShift);
    const double r = __fma_rn(K.inv_ln2n, qd, -kd);
#ifdef GSR_TAB_SPLIT
    // tab[ki & 31] as two 32-bit words from a high-word and a low-word
    // array: 32 entries x 4 B span the 32 banks once, so each load is one
    // wavefront (a 64-bit entry table spans 64 banks: 2+ wavefronts)
    uint32_t th, tl;
    const uint32_t ta = tab_s + ((ki & 31u) << 2);
    asm("ld.shared.u32 %0, [%1];" : "=r"(th) : "r"(ta));
    asm("ld.shared.u32 %0, [%1+128];" : "=r"(tl) : "r"(ta));
    const double sc = __hiloint2double((int)(th + (ki << 15)), (int)tl);
#else
    unsigned long long t;  // tab[ki & 31] through a precomputed shared-window address
    // (the table is 256-byte aligned: base | (ki << 3 & 0xf8) is one LOP3
    // after the shift instead of an AND and an add)
    asm("ld.shared.u64 %0, [%1];" : "=l"(t) : "r"(tab_s | ((ki << 3) & 0xf8u)));
    // t + (ki << 47): only the high word changes (the low word of ki << 47 is 0)
    const double sc = __hiloint2double((int)((uint32_t)(t >> 32) + (ki << 15)), (int)(uint32_t)t);
#endif
    const double z = __fma_rn(K.c0, r, K.c1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(K.c2, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, sc);
    return __double2float_rn(y);
}


// Records of the next batch staged by cp.async (LDGSTS) while the current
// one composites (ranks fetched two batches ahead): blend A 0.3160-0.3167 ->
// 0.3147-0.3151 ms at config 3 (GSR_BLEND_ASYNC=0 restores plain loads).
#ifndef GSR_BLEND_ASYNC
#define GSR_BLEND_ASYNC 1
#endif
#if !GSR_BLEND_ASYNC
#undef GSR_BLEND_ASYNC
#endif

struct WarpBatch {         // one warp's current 32 splats, splat j in slot 32 - j; slot 0: null
    float4 geo[2][33];     // per pixel row of the item: (u, ia, (2*ib)*dy, (ic*dy)*dy)
    float4 col[33];        // (op, r, g, b)
#ifdef GSR_BLEND_ASYNC
    float4 rec[2][32][2];  // records of the next batch, staged by cp.async (double buffer)
#endif
};

#ifdef GSR_BLEND_ASYNC
// cp.async 16 B global -> shared (L1-bypassing .cg), one group per batch
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
#endif

// Each lane walks its own covering splats of the batch in depth order
// (render.py:405-421, reference operation order).  The body is branch-free:
// a lane with no splat left (or saturated) gets index -1, the null slot in
// front of the batch (all zero: power -0, alpha = 0 * 1 = 0, so rgb += 0
// and T *= 1 exactly), which costs less than the divergence bookkeeping of
// an `if` or select.  (Software-pipelining the next
// splat's alpha against the transmittance chain was measured slower: the
// kernel is issue-bound, not latency-bound.)
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

template <bool kChecked, bool kCount = true>
__device__ __forceinline__ void composite(uint32_t mine, uint32_t geo, uint32_t col,
                                          float fx, const unsigned long long *tab, uint32_t tab_s,
                                          const ExpK &ek, float &T, float &cr, float &cg,
                                          float &cb, uint32_t &n_comp) {
    // composites done = bits taken: popc(mine) minus what saturation drops
    n_comp += __popc(mine);
    uint32_t dropped = 0u;
    while (__any_sync(0xffffffffu, mine != 0u)) {
        // mine is bit-reversed (splat j <-> bit 31 - j <-> slot 31 - j), so the
        // next splat in depth order is the highest set bit; -1: null slot
        const int s = 31 - __clz(mine);
        uint32_t below;  // bits [0, s): clears bit s (mine = 0 stays 0)
        asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"((uint32_t)s));
        mine &= below;
        const float4 g = lds128(geo + 16u * (uint32_t)s);  // u, ia, ib_dy, cy_term
        const float4 k = lds128(col + 16u * (uint32_t)s);  // op, r, g, b
        const float dx = fx - g.x;
        // power = -0.5f * q (render.py:405-406), applied inside expf_blend
        const float q = g.y * dx * dx + g.z * dx + g.w;
        float alpha = k.x * expf_blend<kChecked>(q, tab, tab_s, ek);
        if (alpha > kAlphaMax) alpha = kAlphaMax;
        const float weight = T * alpha;
        cr += weight * k.y;
        cg += weight * k.z;
        cb += weight * k.w;
        T = T * (1.0f - alpha);
        if (T < kTStop) {  // the pixel is done (the caller derives `done` from T)
            dropped = mine;
            mine = 0u;
        }
    }
    n_comp -= __popc(dropped);
}

// The two pixel rows of an item interleaved: each iteration composites the
// next covering splat of the lane's pixel in row 0 and of its pixel in row
// 1 (two independent chains; a pixel with nothing left reads the null slot
// of its row, alpha 0), so the loop runs max over lanes of max(count0,
// count1) iterations instead of max count0 + max count1.
template <bool kChecked, bool kCount>
__device__ __forceinline__ void composite_pair(uint32_t m0, uint32_t m1, uint32_t geo0,
                                               uint32_t geo1, uint32_t col, float fx,
                                               const unsigned long long *tab, uint32_t tab_s,
                                               const ExpK &ek, float *T, float *cr, float *cg,
                                               float *cb, uint32_t &n_comp, uint32_t &n_it,
                                               uint32_t &n_lanes) {
    if (kCount) n_comp += __popc(m0) + __popc(m1);
    uint32_t dropped = 0u;
    while (__any_sync(0xffffffffu, (m0 | m1) != 0u)) {
        if (kCount) {  // instrumentation: warp iterations and useful lanes (2 per pixel pair)
            n_it += 1u;
            n_lanes += (m0 != 0u) + (m1 != 0u);
        }
        const int s0 = 31 - __clz(m0), s1 = 31 - __clz(m1);
        uint32_t b0, b1;
        asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(b0) : "r"((uint32_t)s0));
        asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(b1) : "r"((uint32_t)s1));
        m0 &= b0;
        m1 &= b1;
        const float4 g0 = lds128(geo0 + 16u * (uint32_t)s0), g1 = lds128(geo1 + 16u * (uint32_t)s1);
        const float4 k0 = lds128(col + 16u * (uint32_t)s0), k1 = lds128(col + 16u * (uint32_t)s1);
        const float dx0 = fx - g0.x, dx1 = fx - g1.x;
        // power = -0.5f * q (render.py:405-406), applied inside expf_blend
        const float q0 = g0.y * dx0 * dx0 + g0.z * dx0 + g0.w;
        const float q1 = g1.y * dx1 * dx1 + g1.z * dx1 + g1.w;
        float a0 = k0.x * expf_blend<kChecked>(q0, tab, tab_s, ek);
        float a1 = k1.x * expf_blend<kChecked>(q1, tab, tab_s, ek);
        if (a0 > kAlphaMax) a0 = kAlphaMax;
        if (a1 > kAlphaMax) a1 = kAlphaMax;
        const float w0 = T[0] * a0, w1 = T[1] * a1;
        cr[0] += w0 * k0.y;
        cg[0] += w0 * k0.z;
        cb[0] += w0 * k0.w;
        cr[1] += w1 * k1.y;
        cg[1] += w1 * k1.z;
        cb[1] += w1 * k1.w;
        T[0] = T[0] * (1.0f - a0);
        T[1] = T[1] * (1.0f - a1);
        if (T[0] < kTStop) {
            if (kCount) dropped += __popc(m0);
            m0 = 0u;
        }
        if (T[1] < kTStop) {
            if (kCount) dropped += __popc(m1);
            m1 = 0u;
        }
    }
    if (kCount) n_comp -= dropped;
}

// render.py:470 + 484-485: trunc(clip(clip(f64(c), 0, 1) * 255 + 0.5, 0, 255))
__device__ __forceinline__ uint32_t to_u8(float c) {
    double d = (double)c;
    d = d < 0.0 ? 0.0 : (d > 1.0 ? 1.0 : d);
    double q = d * 255.0 + 0.5;
    q = q < 0.0 ? 0.0 : (q > 255.0 ? 255.0 : q);
    return (uint32_t)(int)q;
}

// render.py:423-427 (rgb += T * bg) and the frame stores of one pixel p of
// a warp's row (lane = column): f32 planes when asked, u8 -- when the row is
// packed, the warp's 32 pixels are 96 contiguous bytes: lane l < 24 stores
// bytes 4l..4l+3 (pixels 4l/3 and (4l+3)/3) as one word, so a row is three
// full 32 B sectors (full-sector writes also to mapped host memory).
__device__ __forceinline__ void store_pixel(const BlendOut &out, uint8_t *host, int64_t p,
                                            int lane, float T, float cr, float cg, float cb,
                                            float bg0, float bg1, float bg2) {
    const float rr = cr + T * bg0, gg = cg + T * bg1, bb = cb + T * bg2;
    if (out.rgb) {
        out.rgb[3 * p + 0] = rr;
        out.rgb[3 * p + 1] = gg;
        out.rgb[3 * p + 2] = bb;
    }
    if (out.trans) out.trans[p] = T;
    const uint32_t px = to_u8(rr) | (to_u8(gg) << 8) | (to_u8(bb) << 16);
    if (out.packed) {
        const int a = (4 * lane) / 3, b = min((4 * lane + 3) / 3, 31);
        const uint32_t pa = __shfl_sync(0xffffffffu, px, a);
        const uint32_t pb = __shfl_sync(0xffffffffu, px, b);
        const unsigned long long both = (unsigned long long)pa | ((unsigned long long)pb << 24);
        const uint32_t word = (uint32_t)(both >> (8 * (lane % 3)));
        const int64_t wofs = (3 * (p - lane)) / 4 + lane;
        if (lane < 24) {
            reinterpret_cast<uint32_t *>(out.u8)[wofs] = word;
            if (host) reinterpret_cast<uint32_t *>(host)[wofs] = word;
        }
    } else {
        out.u8[3 * p + 0] = (uint8_t)(px & 0xffu);
        out.u8[3 * p + 1] = (uint8_t)((px >> 8) & 0xffu);
        out.u8[3 * p + 2] = (uint8_t)(px >> 16);
    }
}

// Slice B empty: the items slice A left unsaturated only finish from their
// saved state (nothing behind the front slice reaches them), so instead of
// the blend's persistent grid a plain warp per listed item stores its pixels.
__global__ void __launch_bounds__(128) finish_items_kernel(int width, int height, BlendOut out,
                                                           const FrameCounters *__restrict__ ctr,
                                                           SliceState ss) {
    const float bg0 = out.fp->bg[0], bg1 = out.fp->bg[1], bg2 = out.fp->bg[2];
    uint8_t *const host = out.fp->host;
    constexpr int kItems = kTileH / 2;
    const int tiles_x = (width + kTileW - 1) / kTileW;
    const int lane = lane_id();
    const int n = (int)ctr->n_unsat;
    for (int q = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); q < n;
         q += (int)((gridDim.x * blockDim.x) >> 5)) {
        const int item = (int)__ldg(ss.unsat_items + q);
        const int tile = item / kItems, wr = item % kItems;
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        const int ix = tx * kTileW + lane, iy0 = ty * kTileH + 2 * wr;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            // (warp-uniform when out.packed: W % 32 == 0, so every lane is inside)
            if (iy0 + h >= height || ix >= width) continue;
            const int64_t p = (int64_t)(iy0 + h) * width + ix;
            const float4 st = ss.state[p];
            store_pixel(out, host, p, lane, st.x, st.y, st.z, st.w, bg0, bg1, bg2);
        }
    }
}

// Persistent kernel: the work items are (tile, pixel-row pair) = one warp's
// 2x32 pixels; warps take items from a frame-global queue (ctr->blend_next)
// until it is empty.  Item lengths vary by orders of magnitude (a warp leaves
// as soon as its 32 pixels saturate, or walks the whole tile list if they
// never do), so binding 8 warps to a CTA per tile would leave most of a CTA's
// warps idle behind its slowest one; the queue keeps every warp busy.
// kSets pixel rows per item (one pixel per lane per row): the batch's loads
// and per-splat set-up are shared by the item's rows, which are composited
// one after the other from the same staged batch.
// kMode 0: one pass over the frame's lists.  1: slice A (slice.cu) -- an
// item whose pixels all saturate writes them; any other saves (T, r, g, b)
// per pixel in `state`, sets its bit in unsat_cols and lists itself in
// unsat_items.  2: slice B -- only the listed items, continuing from `state`.
template <int kSets, bool kPairLoop, bool kCount, int kMode>
// 6 CTAs (24 warps) per SM, 80 registers, with the expf constants read from
// shared memory (below): the composite-pair iteration is 84 instructions with
// no constant reloads (88 with four LDC.64 at 7 CTAs / 72 registers); blend
// 0.3445 -> 0.3408-0.3423 ms, one-call device p50 0.831-0.834 -> 0.824 ms at
// config 3 (8 CTAs: 0.349-0.351 ms)
#ifndef GSR_BLEND_MINB
#define GSR_BLEND_MINB 6
#endif
#ifndef GSR_EXPK_CONST
#define GSR_EXPK_SMEM 1
#endif
__global__ void __launch_bounds__(kBlendThreads, kSets == 1 ? 9 : GSR_BLEND_MINB) blend_kernel(
    const SplatRec *__restrict__ srec, const float4 *__restrict__ colr,
    const uint32_t *__restrict__ tile_vals, const uint2 *__restrict__ ranges, int width,
    int height, BlendOut out, FrameCounters *__restrict__ ctr, SliceState ss) {
    const float bg0 = out.fp->bg[0], bg1 = out.fp->bg[1], bg2 = out.fp->bg[2];
    uint8_t *const host = out.fp->host;
    constexpr int kItems = kTileH / kSets;  // items per tile
    __shared__ __align__(256) unsigned long long s_tab[32];
    __shared__ WarpBatch s_b[kWarps];
#ifdef GSR_TAB_SPLIT
    if (threadIdx.x < 32) {
        reinterpret_cast<uint32_t *>(s_tab)[threadIdx.x] = (uint32_t)(kExp2fTab[threadIdx.x] >> 32);
        reinterpret_cast<uint32_t *>(s_tab)[32 + threadIdx.x] = (uint32_t)kExp2fTab[threadIdx.x];
    }
#else
    if (threadIdx.x < 32) s_tab[threadIdx.x] = kExp2fTab[threadIdx.x];
#endif
#ifdef GSR_EXPK_SMEM
    __shared__ double s_ek[4];
    if (threadIdx.x < 4) s_ek[threadIdx.x] = kExpK[threadIdx.x];
#endif
    {   // zero records (the null slot is never written afterwards)
        float4 *z = reinterpret_cast<float4 *>(s_b);
        for (int i = threadIdx.x; i < (int)(sizeof(s_b) / sizeof(float4)); i += blockDim.x)
            z[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    __syncthreads();

    const int tiles_x = (width + kTileW - 1) / kTileW;
    const int n_items = tiles_x * ((height + kTileH - 1) / kTileH) * kItems;
    const int lane = lane_id(), w = threadIdx.x >> 5;
    WarpBatch &B_ = s_b[w];
    // shared-window addresses of slot 0 of the rows, opaque to the compiler
    // so they stay in registers across the composite loop
    uint32_t geo[kSets], bcol;
#pragma unroll
    for (int h = 0; h < kSets; h++)
        asm volatile("mov.u32 %0, %1;" : "=r"(geo[h]) : "r"((uint32_t)__cvta_generic_to_shared(&B_.geo[h][1])));
    asm volatile("mov.u32 %0, %1;" : "=r"(bcol) : "r"((uint32_t)__cvta_generic_to_shared(&B_.col[1])));
    // (opaque to the compiler, so the table base stays in a register instead
    //  of being rebuilt from the CTA id in the inner loop)
    uint32_t tab_s;
    asm volatile("mov.u32 %0, %1;" : "=r"(tab_s) : "r"((uint32_t)__cvta_generic_to_shared(s_tab)));
    // pinned in registers (opaque to rematerialisation by constant reloads)
    ExpK ek;
#ifdef GSR_EXPK_SMEM
    // from shared memory: ptxas cannot rematerialise a shared load, so the
    // four constants stay in registers instead of four LDC.64 per iteration
    {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(s_ek);
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(ek.inv_ln2n) : "r"(a));
        asm volatile("ld.shared.f64 %0, [%1+8];" : "=d"(ek.c0) : "r"(a));
        asm volatile("ld.shared.f64 %0, [%1+16];" : "=d"(ek.c1) : "r"(a));
        asm volatile("ld.shared.f64 %0, [%1+24];" : "=d"(ek.c2) : "r"(a));
    }
#else
    asm volatile("mov.b64 %0, %1;" : "=d"(ek.inv_ln2n) : "d"(kExpK[0]));
    asm volatile("mov.b64 %0, %1;" : "=d"(ek.c0) : "d"(kExpK[1]));
    asm volatile("mov.b64 %0, %1;" : "=d"(ek.c1) : "d"(kExpK[2]));
    asm volatile("mov.b64 %0, %1;" : "=d"(ek.c2) : "d"(kExpK[3]));
#endif
    uint32_t n_comp = 0, n_rows = 0;  // work counters (roofline)
    uint32_t n_walk = 0, n_hit = 0, n_batch = 0, n_it = 0, n_lanes = 0, n_done = 0;

    // slice B: only the items slice A left unsaturated (its list)
    // slice B with one-row work items (kSets == 1): each listed two-row item
    // is two queue entries, so an unsaturated item's rows walk their (equal)
    // lists on two warps -- the kernel's length is the longest item's walk
    constexpr int kSplit = (kMode == 2 && kSets == 1) ? 2 : 1;
    const int n_queue = kMode == 2 ? (int)ctr->n_unsat * kSplit : n_items;
    while (true) {
        int item = 0;
        if (lane == 0) item = (int)atomicAdd(&ctr->blend_next, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= n_queue) break;
        if (kMode == 2) {
            const int item2 = (int)__ldg(ss.unsat_items + item / kSplit);  // two-row item
            item = kSplit == 2 ? (item2 / (kTileH / 2)) * kItems + 2 * (item2 % (kTileH / 2)) +
                                     (item & 1)
                               : item2;
        }
        if (kCount) n_done += (lane == 0);
        const int tile = item / kItems, wr = item % kItems;
        const int tx = tile % tiles_x, ty = tile / tiles_x;
        const int X = tx * kTileW;
        const int iy0 = ty * kTileH + kSets * wr;
        const int ix = X + lane;
        const float fx = (float)ix + 0.5f;

        float T[kSets], cr[kSets], cg[kSets], cb[kSets];
        bool inside[kSets], done[kSets];
#pragma unroll
        for (int h = 0; h < kSets; h++) {
            T[h] = 1.0f;
            cr[h] = cg[h] = cb[h] = 0.0f;
            inside[h] = ix < width && iy0 + h < height;
            if (kMode == 2 && inside[h]) {
                const float4 st = ss.state[(int64_t)(iy0 + h) * width + ix];
                T[h] = st.x;
                cr[h] = st.y;
                cg[h] = st.z;
                cb[h] = st.w;
            }
            done[h] = !inside[h] || (kMode == 2 && T[h] < kTStop);
        }
        // slice B with no splats: its lists were never built (the switch ran
        // no body), so the items only finish from the saved state
        const uint2 rg = (kMode == 2 && ctr->KB == 0u) ? make_uint2(0u, 0u) : ranges[tile];
        uint32_t last_r = 0;  // instrumentation: deepest rank this item walked

#ifdef GSR_BLEND_ASYNC
        // records staged one batch ahead by cp.async, ranks two batches ahead
        uint32_t r_cur = 0u, r_nxt = 0u, buf = 0u;
        {
            const uint32_t j0 = rg.x + lane, j1 = rg.x + 32u + lane;
            r_cur = j0 < rg.y ? __ldg(tile_vals + j0) : 0u;
            r_nxt = j1 < rg.y ? __ldg(tile_vals + j1) : 0u;
            if (j0 < rg.y) {
                const uint32_t d = (uint32_t)__cvta_generic_to_shared(&B_.rec[0][lane][0]);
                cp_async16(d, &srec[r_cur].a);
                cp_async16(d + 16u, &srec[r_cur].b);
            }
            cp_async_commit();
        }
#endif
        for (uint32_t c = rg.x; c < rg.y; c += 32) {
            bool all_done = true;
#pragma unroll
            for (int h = 0; h < kSets; h++) all_done = all_done && done[h];
            if (__all_sync(0xffffffffu, all_done)) break;
            const uint32_t j = c + lane;
            if (kCount) n_batch += (lane == 0);
            uint32_t mask[kSets];
#pragma unroll
            for (int h = 0; h < kSets; h++) mask[h] = 0u;
            bool safe = true;
#ifdef GSR_BLEND_ASYNC
            cp_async_wait_all();
            __syncwarp();
            const uint32_t r_this = r_cur;
            const float4 A_s = B_.rec[buf][lane][0], B_s = B_.rec[buf][lane][1];
            {   // stage the next batch's records, fetch the ranks after it
                const uint32_t jn = c + 32u + lane, jn2 = c + 64u + lane;
                if (jn < rg.y) {
                    const uint32_t d = (uint32_t)__cvta_generic_to_shared(&B_.rec[buf ^ 1u][lane][0]);
                    cp_async16(d, &srec[r_nxt].a);
                    cp_async16(d + 16u, &srec[r_nxt].b);
                }
                cp_async_commit();
                r_cur = r_nxt;
                r_nxt = jn2 < rg.y ? __ldg(tile_vals + jn2) : 0u;
                buf ^= 1u;
            }
#endif
            if (j < rg.y) {
#ifdef GSR_BLEND_ASYNC
                const uint32_t r = r_this;
                if (kCount) last_r = max(last_r, r);
                const float4 A = A_s;
                const float4 B = B_s;
#else
                const uint32_t r = __ldg(tile_vals + j);  // depth rank
                if (kCount) last_r = max(last_r, r);
                const float4 A = __ldg(&srec[r].a);
                const float4 B = __ldg(&srec[r].b);
#endif
                int lo, hi;  // precomputed per frame by bin_gather (SplatRec.b.w)
                bool fast, esafe;
                unpack_rows(B.w, lo, hi, fast, esafe);
                if (kCount) n_walk++;
                if (iy0 + kSets > lo && iy0 < hi) {
                    if (kCount) n_hit++;
                    const float rinv = fast ? __frcp_rn(A.z) : 0.0f;
                    uint32_t any = 0u;
#pragma unroll
                    for (int h = 0; h < kSets; h++) {
                        n_rows += (uint32_t)(iy0 + h >= lo && iy0 + h < hi);
                        mask[h] = row_mask(A, B, rinv, fast, iy0 + h, lo, hi, X, width);
                        any |= mask[h];
                    }
                    if (any) {  // render.py:400-402 terms per pixel row
                        const float4 C = __ldg(colr + r);  // (r, g, b) by depth rank
                        if (kCount && out.used && atomicExch(out.used + r, 1u) == 0u)
                            atomicAdd(&ctr->b_used, 1ull);
                        safe = esafe;
#pragma unroll
                        for (int h = 0; h < kSets; h++) {
                            const float dy = ((float)(iy0 + h) + 0.5f) - A.y;
                            B_.geo[h][32 - lane] =
                                make_float4(A.x, A.z, (2.0f * A.w) * dy, B.x * dy * dy);
                        }
                        B_.col[32 - lane] = make_float4(B.z, C.x, C.y, C.z);
                    }
                }
            }
            __syncwarp();
            const bool all_safe = __all_sync(0xffffffffu, safe);
            if (kSets == 2 && kPairLoop) {
                uint32_t m0 = __brev(transpose32(mask[0], lane));
                uint32_t m1 = __brev(transpose32(mask[kSets - 1], lane));
                if (done[0]) m0 = 0u;
                if (done[kSets - 1]) m1 = 0u;
                if (all_safe)
                    composite_pair<false, kCount>(m0, m1, geo[0], geo[kSets - 1], bcol, fx, s_tab,
                                                  tab_s, ek, T, cr, cg, cb, n_comp, n_it, n_lanes);
                else
                    composite_pair<true, kCount>(m0, m1, geo[0], geo[kSets - 1], bcol, fx, s_tab,
                                                 tab_s, ek, T, cr, cg, cb, n_comp, n_it, n_lanes);
#pragma unroll
                for (int h = 0; h < kSets; h++) done[h] = done[h] || T[h] < kTStop;
            } else {
#pragma unroll
                for (int h = 0; h < kSets; h++) {
                    uint32_t mine = __brev(transpose32(mask[h], lane));
                    if (done[h]) mine = 0u;
                    if (all_safe)
                        composite<false>(mine, geo[h], bcol, fx, s_tab, tab_s, ek, T[h], cr[h],
                                         cg[h], cb[h], n_comp);
                    else
                        composite<true>(mine, geo[h], bcol, fx, s_tab, tab_s, ek, T[h], cr[h],
                                        cg[h], cb[h], n_comp);
                    done[h] = done[h] || T[h] < kTStop;
                }
            }
            __syncwarp();
        }
#ifdef GSR_BLEND_ASYNC
        cp_async_wait_all();  // the staging buffers are reused by the next item
        __syncwarp();
#endif
        if (kCount && out.item_info && kSplit == 1) {  // (indexed by two-row item)
            bool sat = true;
#pragma unroll
            for (int h = 0; h < kSets; h++) sat = sat && done[h];
            sat = __all_sync(0xffffffffu, sat);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) last_r = max(last_r, __shfl_xor_sync(0xffffffffu, last_r, o));
            if (lane == 0) out.item_info[item] = (last_r & 0x7fffffffu) | ((uint32_t)sat << 31);
        }
        if (kMode == 1) {  // slice A: saturated items finish, the others wait for B
            bool sat = true;
#pragma unroll
            for (int h = 0; h < kSets; h++) sat = sat && (done[h] || T[h] < kTStop);
            if (!__all_sync(0xffffffffu, sat)) {
#pragma unroll
                for (int h = 0; h < kSets; h++)
                    if (inside[h])
                        ss.state[(int64_t)(iy0 + h) * width + ix] =
                            make_float4(T[h], cr[h], cg[h], cb[h]);
                if (lane == 0) {
                    // column-major: tile column tx, bit (item row & 31) of word item row / 32
                    atomicOr(ss.unsat_cols + (int64_t)tx * ss.col_words + ((iy0 >> 1) >> 5),
                             1u << ((iy0 >> 1) & 31));
                    ss.unsat_items[atomicAdd(&ctr->n_unsat, 1u)] = (uint32_t)item;
                }
                continue;
            }
        }
#pragma unroll
        for (int h = 0; h < kSets; h++) {
            if (!inside[h]) continue;  // warp-uniform when out.packed
            store_pixel(out, host, (int64_t)(iy0 + h) * width + ix, lane, T[h], cr[h], cg[h],
                        cb[h], bg0, bg1, bg2);
        }
    }
    if (kCount) {
        unsigned long long v[8] = {n_comp, n_rows, n_walk, n_hit, n_batch, n_it, n_lanes, n_done};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < 8; i++) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
        if (lane == 0) {
            atomicAdd(&ctr->E, v[0]);
            atomicAdd(&ctr->Rb, v[1]);
            atomicAdd(&ctr->b_walked, v[2]);
            atomicAdd(&ctr->b_hit, v[3]);
            atomicAdd(&ctr->b_batches, v[4]);
            atomicAdd(&ctr->b_iters, v[5]);   // counted by every lane: warp-uniform
            atomicAdd(&ctr->b_lanes, v[6]);
            atomicAdd(&ctr->b_items, v[7]);
        }
    }
}

int g_blend_grid = 0;

// tuning: 1 = one row per item, 2 = two rows one after the other,
// 3 (default) = two rows interleaved (composite_pair); only 3 has the
// slice modes
int blend_sets() {
    static int sets = 0;
    if (!sets) {
        const char *e = getenv("GSR_BLEND_SETS");
        sets = (e && atoi(e) >= 1 && atoi(e) <= 3) ? atoi(e) : 3;
    }
    return sets;
}

}  // namespace

bool blend_has_slices() { return blend_sets() == 3; }

// persistent grid: every SM full (computed once; call before any graph capture)
int blend_grid(int width, int height) {
    const int sets = blend_sets();
    if (!g_blend_grid) {
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sets == 1)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, blend_kernel<1, false, true, 0>, kBlendThreads, 0);
        else if (sets == 3)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, blend_kernel<2, true, false, 0>, kBlendThreads, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, blend_kernel<2, false, true, 0>, kBlendThreads, 0);
        // GSR_BLEND_CTAS_PER_SM (tuning): fewer resident CTAs leave room for
        // other frames' kernels when several frames are in flight
        if (const char *e = getenv("GSR_BLEND_CTAS_PER_SM")) {
            const int v = atoi(e);
            if (v > 0 && v < per_sm) per_sm = v;
        }
        g_blend_grid = sms * (per_sm > 0 ? per_sm : 1);
    }
    const int tiles = ((width + kTileW - 1) / kTileW) * ((height + kTileH - 1) / kTileH);
    return std::max(1, std::min(g_blend_grid, tiles * kTileH));
}

void launch_finish_items(int width, int height, BlendOut out, const FrameCounters *ctr,
                         SliceState ss, int max_items, cudaStream_t s, const KMark &mark) {
    const int sms_x8 = 148 * 8;
    const int blocks = std::max(1, std::min((max_items + 3) / 4, sms_x8));
    finish_items_kernel<<<blocks, 128, 0, s>>>(width, height, out, ctr, ss);
    mark("finish_items");
}

void launch_blend(const SplatRec *srec, const float4 *colr, const uint32_t *tile_vals,
                  const uint2 *ranges, int width, int height, BlendOut out, FrameCounters *ctr,
                  cudaStream_t s, const KMark &mark, bool count, int mode, SliceState ss) {
    const int grid = blend_grid(width, height);
    const int sets = blend_sets();
#define GSR_BLEND(S, P, C, M)                                                                 \
    blend_kernel<S, P, C, M><<<grid, kBlendThreads, 0, s>>>(srec, colr, tile_vals, ranges, width, \
                                                           height, out, ctr, ss)
    if (sets == 1) GSR_BLEND(1, false, true, 0);  // tuning variants: one pass only
    else if (sets == 2) GSR_BLEND(2, false, true, 0);
    else if (mode == 1) { if (count) GSR_BLEND(2, true, true, 1); else GSR_BLEND(2, true, false, 1); }
#ifndef GSR_BLEND_B_ROWS
#define GSR_BLEND_B_ROWS 2  // pixel rows per slice-B work item (1: two warps per listed item; measured within noise)
#endif
    else if (mode == 2) {
        if (GSR_BLEND_B_ROWS == 1) { if (count) GSR_BLEND(1, false, true, 2); else GSR_BLEND(1, false, false, 2); }
        else { if (count) GSR_BLEND(2, true, true, 2); else GSR_BLEND(2, true, false, 2); }
    }
    else if (count) GSR_BLEND(2, true, true, 0);  // work counters (E, Rb) only when asked
    else GSR_BLEND(2, true, false, 0);
#undef GSR_BLEND
    mark(mode == 1 ? "blend_a" : mode == 2 ? "blend_b" : "blend");
}

}  // namespace gsr
