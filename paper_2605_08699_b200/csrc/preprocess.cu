// preprocess.cu -- K1: per-Gaussian f64 projection, culling, SH colour and
// packing.
//
// Restates, with the reference's exact f64 operation order (no FMA):
//   _project_kernel      render.py:163-237
//   eval_sh_colors       render.py:126-160 (degree 1..3; colors_dc for 0)
//   packing              render.py:442-453 (c/det, -b/det, a/det, sqrt(c*rsq))
// Culled Gaussians get the sentinel depth key ~0; the first depth-sort pass
// drops them, which is the order-preserving compaction of render.py:279.
//
// Two streaming kernels rather than one fused pass: a fused kernel needs ~80
// registers (the FP64 projection and the SH evaluation live at once), which
// caps it at 24 warps per SM -- too few to hide HBM latency behind FP64
// latency.  Split, each runs at high occupancy with all its loads coalesced:
//   K1a geo    mean/scale/rotation/rsq/opacity (92 B) -> depth key and the
//              packed geometry (u, v, ia, ib | ic, rsq, op, ry)
//   K1b colour kept Gaussians only: mean + SH planes (216 B) -> (r, g, b)
// The binning gather (binning.cu) puts the geometry records in depth order.
#include <algorithm>

#include "kernels.cuh"

namespace gsr {

namespace {

constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
constexpr double SH_C2_0 = 1.0925484305920792, SH_C2_1 = -1.0925484305920792,
                 SH_C2_2 = 0.31539156525252005, SH_C2_3 = -1.0925484305920792,
                 SH_C2_4 = 0.5462742152960396;
constexpr double SH_C3_0 = -0.5900435899266435, SH_C3_1 = 2.890611442640554,
                 SH_C3_2 = -0.4570457994644658, SH_C3_3 = 0.3731763325901154,
                 SH_C3_4 = -0.4570457994644658, SH_C3_5 = 1.445305721320277,
                 SH_C3_6 = -0.5900435899266435;

// eval_sh_colors for one Gaussian and one channel, numpy expression order;
// v holds the Gaussian's coefficients already in registers (plane k*3 + c).
template <int DEG, typename T>
__device__ __forceinline__ double sh_channel(const T *v, int c, double x, double y, double z,
                                             double xx, double yy, double zz, double xy,
                                             double yz, double xz) {
#define SHV(k) ((double)v[(k) * 3 + c])
    double r = SH_C0 * SHV(0);
    r = r - (SH_C1 * y) * SHV(1) + (SH_C1 * z) * SHV(2) - (SH_C1 * x) * SHV(3);
    if (DEG >= 2) {
        r = r + (SH_C2_0 * xy) * SHV(4) + (SH_C2_1 * yz) * SHV(5) +
            (SH_C2_2 * (2.0 * zz - xx - yy)) * SHV(6) + (SH_C2_3 * xz) * SHV(7) +
            (SH_C2_4 * (xx - yy)) * SHV(8);
    }
    if (DEG >= 3) {
        r = r + ((SH_C3_0 * y) * (3.0 * xx - yy)) * SHV(9) + ((SH_C3_1 * xy) * z) * SHV(10) +
            ((SH_C3_2 * y) * (4.0 * zz - xx - yy)) * SHV(11) +
            ((SH_C3_3 * z) * (2.0 * zz - 3.0 * xx - 3.0 * yy)) * SHV(12) +
            ((SH_C3_4 * x) * (4.0 * zz - xx - yy)) * SHV(13) + ((SH_C3_5 * z) * (xx - yy)) * SHV(14) +
            ((SH_C3_6 * x) * (xx - 3.0 * yy)) * SHV(15);
    }
#undef SHV
    r = r + 0.5;
    return r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);  // np.clip(result + 0.5, 0, 1)
}

// The frame's first kernel: its parameters (camera, background, mapped host
// frame) into device memory -- the CUDA graph's one updated node -- and the
// per-frame counters reset.
__global__ void __launch_bounds__(256) frame_start_kernel(FrameParams p, FrameParams *dst,
                                                          FrameCounters *ctr) {
    for (int j = threadIdx.x; j < kZBins; j += blockDim.x) ctr->slice_hist[j] = 0u;
    if (threadIdx.x) return;
    *dst = p;
    ctr->K = 0;
    ctr->D = 0;
    ctr->npass = 0;
    ctr->npass_fb = 0;
    ctr->kmin = ~0ull;
    ctr->kmax = 0ull;
    ctr->P = 0ull;
    ctr->nseg = 0;
    ctr->long_runs = 0;
    ctr->E = 0ull;
    ctr->Rb = 0ull;
    ctr->Rp = 0ull;
    ctr->blend_next = 0;
    ctr->rows_done = 0u;
    ctr->Drow = 0u;
    
    ctr->b_walked = ctr->b_hit = ctr->b_batches = ctr->b_iters = ctr->b_lanes = 0ull;
    ctr->b_items = ctr->b_used = 0ull;
    ctr->KA = ctr->KB = ctr->tau = ctr->n_unsat = 0u;
    ctr->Dtot = ctr->Ptot = ctr->Dmax = ctr->Pmax = 0ull;
}


// cp.async.bulk global -> shared, completing on an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(mbar), "r"(phase) : "memory");
}

// One Gaussian's inputs (SoA planes), loaded by the caller -- from global
// memory, or from a shared-memory stage filled by the bulk-copy engine.
struct PPIn {
    double mx, my, mz, qw, qx, qy, qz, sx, sy, sz, rsq;
    float opac;
};

// Projection, cull and packing of Gaussian i (render.py:174-235, 442-453):
// writes geo[i] / ibox[i] and the depth histogram when kept; returns kept and
// sets key (the f64 bits of z, ~0 when culled).
__device__ __forceinline__ bool pp_one(const CameraArgs &cam, int do_cull, int64_t i,
                                       const PPIn &in, GeoRec *__restrict__ geo,
                                       uint2 *__restrict__ ibox, uint32_t *s_zh,
                                       unsigned long long &key) {
    const double r00 = cam.r[0], r01 = cam.r[1], r02 = cam.r[2];
    const double r10 = cam.r[3], r11 = cam.r[4], r12 = cam.r[5];
    const double r20 = cam.r[6], r21 = cam.r[7], r22 = cam.r[8];
    const double mx = in.mx, my = in.my, mz = in.mz;
    const double qw = in.qw, qx = in.qx, qy = in.qy, qz = in.qz;
    const double sx = in.sx, sy = in.sy, sz = in.sz;
    key = ~0ull;
    // render.py:174-176
    const double x = r00 * mx + r01 * my + r02 * mz + cam.t[0];
    const double y = r10 * mx + r11 * my + r12 * mz + cam.t[1];
    const double z = r20 * mx + r21 * my + r22 * mz + cam.t[2];
    if (z <= kZNear) return false;
    // render.py:185-193
    const double m00 = (1.0 - 2.0 * (qy * qy + qz * qz)) * sx;
    const double m01 = (2.0 * (qx * qy - qw * qz)) * sy;
    const double m02 = (2.0 * (qx * qz + qw * qy)) * sz;
    const double m10 = (2.0 * (qx * qy + qw * qz)) * sx;
    const double m11 = (1.0 - 2.0 * (qx * qx + qz * qz)) * sy;
    const double m12 = (2.0 * (qy * qz - qw * qx)) * sz;
    const double m20 = (2.0 * (qx * qz - qw * qy)) * sx;
    const double m21 = (2.0 * (qy * qz + qw * qx)) * sy;
    const double m22 = (1.0 - 2.0 * (qx * qx + qy * qy)) * sz;
    // render.py:196-204
    const double a00 = r00 * m00 + r01 * m10 + r02 * m20;
    const double a01 = r00 * m01 + r01 * m11 + r02 * m21;
    const double a02 = r00 * m02 + r01 * m12 + r02 * m22;
    const double a10 = r10 * m00 + r11 * m10 + r12 * m20;
    const double a11 = r10 * m01 + r11 * m11 + r12 * m21;
    const double a12 = r10 * m02 + r11 * m12 + r12 * m22;
    const double a20 = r20 * m00 + r21 * m10 + r22 * m20;
    const double a21 = r20 * m01 + r21 * m11 + r22 * m21;
    const double a22 = r20 * m02 + r21 * m12 + r22 * m22;
    // render.py:206-220
    const double inv_z = 1.0 / z;
    const double jx = cam.fx * inv_z;
    const double jy = cam.fy * inv_z;
    const double gx = -cam.fx * x * inv_z * inv_z;
    const double gy = -cam.fy * y * inv_z * inv_z;
    const double p0 = jx * a00 + gx * a20;
    const double p1 = jx * a01 + gx * a21;
    const double p2 = jx * a02 + gx * a22;
    const double q0 = jy * a10 + gy * a20;
    const double q1 = jy * a11 + gy * a21;
    const double q2 = jy * a12 + gy * a22;
    const double ca = p0 * p0 + p1 * p1 + p2 * p2 + kCovFloor;
    const double cb = p0 * q0 + p1 * q1 + p2 * q2;
    const double cc = q0 * q0 + q1 * q1 + q2 * q2 + kCovFloor;
    // render.py:222-223
    const double u = cam.fx * x * inv_z + cam.cx;
    const double v = cam.fy * y * inv_z + cam.cy;
    // render.py:230-235.  A splat whose centre lies inside the image is kept
    // whatever its radius, as long as the radius is not NaN (finite
    // covariance: ca, cc >= 0.3, so mid + sqrt(disc) > 0): the two f64 square
    // roots are only needed near and outside the border -- the same keep
    // mask, fewer instructions
    const bool inside = u > 0.0 && u < cam.width && v > 0.0 && v < cam.height &&
                        isfinite(ca) && isfinite(cb) && isfinite(cc);
    if (do_cull && !inside) {
        const double mid = 0.5 * (ca + cc);
        const double d = ca - cc;
        const double disc = 0.25 * (d * d) + cb * cb;
        const double radius = kCutoffSigma * sqrt(mid + sqrt(disc));
        if (!(u + radius > 0.0 && u - radius < cam.width && v + radius > 0.0 &&
              v - radius < cam.height))
            return false;
    }
    key = (unsigned long long)__double_as_longlong(z);
    if (s_zh) {
        const int bin = (int)(key >> kZBinShift) - kZBinBase;
        atomicAdd(&s_zh[bin < 0 ? 0 : (bin >= kZBins ? kZBins - 1 : bin)], 1u);
    }
    // render.py:442-453
    const double det = ca * cc - cb * cb;
    const float ia32 = (float)(cc / det);
    GeoRec o;
    o.a = make_float4((float)u, (float)v, ia32, (float)(-cb / det));
    o.b = make_float4((float)(ca / det), (float)in.rsq, in.opac, (float)sqrt(cc * in.rsq));
    geo[i] = o;
    if (ibox) ibox[i] = item_box(o, cam.iwidth, cam.iheight);
    return true;
}

// Block reduction of K and of the kept key range (radix pass trimming), and
// the block's depth histogram into the frame's.
__device__ __forceinline__ void pp_reduce(uint32_t cnt, unsigned long long kmn,
                                          unsigned long long kmx, const uint32_t *s_zh,
                                          uint32_t *zhist, FrameCounters *ctr) {
    __shared__ unsigned long long s_min[8], s_max[8];
    __shared__ uint32_t s_cnt[8];
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    {   // warp min / max of the 64-bit keys with 32-bit REDUX: the high words,
        // then the low words among the lanes holding the extreme high word
        const uint32_t hmn = __reduce_min_sync(0xffffffffu, (uint32_t)(kmn >> 32));
        const uint32_t lmn = __reduce_min_sync(
            0xffffffffu, (uint32_t)(kmn >> 32) == hmn ? (uint32_t)kmn : 0xffffffffu);
        const uint32_t hmx = __reduce_max_sync(0xffffffffu, (uint32_t)(kmx >> 32));
        const uint32_t lmx =
            __reduce_max_sync(0xffffffffu, (uint32_t)(kmx >> 32) == hmx ? (uint32_t)kmx : 0u);
        kmn = ((unsigned long long)hmn << 32) | lmn;
        kmx = ((unsigned long long)hmx << 32) | lmx;
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_min[w] = kmn;
        s_max[w] = kmx;
        s_cnt[w] = cnt;
    }
    __syncthreads();
    if (zhist)
        for (int j = threadIdx.x; j < kZBins; j += blockDim.x)
            if (s_zh[j]) atomicAdd(zhist + j, s_zh[j]);
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (int j = 0; j < (int)(blockDim.x >> 5); j++) {
            c += s_cnt[j];
            kmn = s_min[j] < kmn ? s_min[j] : kmn;
            kmx = s_max[j] > kmx ? s_max[j] : kmx;
        }
        if (c) {
            atomicAdd(&ctr->K, c);
            atomicMin(&ctr->kmin, kmn);
            atomicMax(&ctr->kmax, kmx);
        }
    }
}

#ifndef GSR_PP_MINB
#define GSR_PP_MINB 4  // 64 registers, no spill: 0.1124 -> 0.1075 ms at config 3 (5: 51 registers + 94 B spilled)
#endif
// One Gaussian per thread, its 92 B loaded from global memory first (one
// memory round trip), then the f64 math.
__global__ void __launch_bounds__(256, GSR_PP_MINB) preprocess_geo_kernel(
    SceneView sc, const FrameParams *__restrict__ fp, int do_cull,
    unsigned long long *__restrict__ keys, GeoRec *__restrict__ geo,
    uint8_t *__restrict__ keep_out, FrameCounters *ctr, uint32_t *__restrict__ zhist,
    uint2 *__restrict__ ibox) {
    __shared__ CameraArgs cam;  // this frame's camera (FrameParams), staged once per block
    __shared__ uint32_t s_zh[kZBins];
    if (zhist)
        for (int j = threadIdx.x; j < kZBins; j += blockDim.x) s_zh[j] = 0u;
    if (threadIdx.x < sizeof(CameraArgs) / 8)
        reinterpret_cast<unsigned long long *>(&cam)[threadIdx.x] =
            reinterpret_cast<const unsigned long long *>(&fp->cam)[threadIdx.x];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t st = sc.stride;
    bool kept = false;
    unsigned long long key = ~0ull;
    if (i < sc.n) {
        PPIn in;
        in.mx = __ldg(sc.mean + i);
        in.my = __ldg(sc.mean + st + i);
        in.mz = __ldg(sc.mean + 2 * st + i);
        in.qw = __ldg(sc.rot + i);
        in.qx = __ldg(sc.rot + st + i);
        in.qy = __ldg(sc.rot + 2 * st + i);
        in.qz = __ldg(sc.rot + 3 * st + i);
        in.sx = __ldg(sc.scale + i);
        in.sy = __ldg(sc.scale + st + i);
        in.sz = __ldg(sc.scale + 2 * st + i);
        in.rsq = __ldg(sc.rsq + i);
        in.opac = __ldg(sc.opac + i);
        kept = pp_one(cam, do_cull, i, in, geo, ibox, zhist ? s_zh : nullptr, key);
        keys[i] = key;
        if (keep_out) keep_out[i] = kept ? 1 : 0;
    }
    pp_reduce(kept ? 1u : 0u, kept ? key : ~0ull, kept ? key : 0ull, s_zh, zhist, ctr);
}

// The same per-Gaussian work with the inputs brought in by the bulk-copy
// (TMA) engine: a persistent CTA takes tiles of 256 Gaussians; one thread
// issues the tile's twelve plane chunks (11 x 2 KB f64 + 1 KB f32, contiguous
// in the SoA planes) as cp.async.bulk copies into one of two shared stages,
// completing on the stage's mbarrier, so tile k + 1's 23.5 KB are in flight
// while tile k computes.  (The one-shot kernel above issues its loads once
// per thread and then computes for ~800 instructions: CTAs of a wave load
// and compute in phase, and HBM idles during the compute.)
constexpr int kPPTile = 256;
struct PPStage {
    double m[3][kPPTile];
    double q[4][kPPTile];
    double s[3][kPPTile];
    double rsq[kPPTile];
    float op[kPPTile];
};
#ifndef GSR_PPB_MINB
#define GSR_PPB_MINB 4
#endif
__device__ __forceinline__ void pp_issue(const SceneView &sc, int64_t t, uint32_t stage,
                                         uint32_t mbar) {
    const int64_t st = sc.stride;
    const int64_t i0 = t * kPPTile;
    const int64_t cnt = st - i0 < kPPTile ? st - i0 : kPPTile;  // multiple of 32
    const uint32_t b64 = (uint32_t)cnt * 8u, b32 = (uint32_t)cnt * 4u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(mbar), "r"(11u * b64 + b32) : "memory");
    constexpr uint32_t P = kPPTile * 8;  // one f64 plane chunk in the stage
#pragma unroll
    for (int k = 0; k < 3; k++) bulk_g2s(stage + k * P, sc.mean + k * st + i0, b64, mbar);
#pragma unroll
    for (int k = 0; k < 4; k++) bulk_g2s(stage + (3 + k) * P, sc.rot + k * st + i0, b64, mbar);
#pragma unroll
    for (int k = 0; k < 3; k++) bulk_g2s(stage + (7 + k) * P, sc.scale + k * st + i0, b64, mbar);
    bulk_g2s(stage + 10 * P, sc.rsq + i0, b64, mbar);
    bulk_g2s(stage + 11 * P, sc.opac + i0, b32, mbar);
}

__global__ void __launch_bounds__(kPPTile, GSR_PPB_MINB) preprocess_geo_bulk_kernel(
    SceneView sc, const FrameParams *__restrict__ fp, int do_cull,
    unsigned long long *__restrict__ keys, GeoRec *__restrict__ geo,
    uint8_t *__restrict__ keep_out, FrameCounters *ctr, uint32_t *__restrict__ zhist,
    uint2 *__restrict__ ibox) {
    extern __shared__ __align__(128) unsigned char pp_smem[];
    PPStage *stg = reinterpret_cast<PPStage *>(pp_smem);  // [2]
    __shared__ CameraArgs cam;
    __shared__ uint32_t s_zh[kZBins];
    __shared__ __align__(8) unsigned long long bar[2];
    const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    const uint32_t mbar1 = (uint32_t)__cvta_generic_to_shared(&bar[1]);
    const uint32_t stage0 = (uint32_t)__cvta_generic_to_shared(&stg[0]);
    const uint32_t stage1 = (uint32_t)__cvta_generic_to_shared(&stg[1]);
    const int64_t n_tiles = (sc.n + kPPTile - 1) / kPPTile;
    if (zhist)
        for (int j = threadIdx.x; j < kZBins; j += blockDim.x) s_zh[j] = 0u;
    if (threadIdx.x < sizeof(CameraArgs) / 8)
        reinterpret_cast<unsigned long long *>(&cam)[threadIdx.x] =
            reinterpret_cast<const unsigned long long *>(&fp->cam)[threadIdx.x];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if ((int64_t)blockIdx.x < n_tiles) pp_issue(sc, blockIdx.x, stage0, mbar0);
    }
    __syncthreads();
    uint32_t cnt = 0u;
    unsigned long long kmn = ~0ull, kmx = 0ull;
    uint32_t phases = 0u;  // bit b: the parity stage b waits for next
    int b = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, b ^= 1) {
        if (threadIdx.x == 0 && t + gridDim.x < n_tiles) {
            // the other stage was last read (generic proxy) before the
            // __syncthreads ending the previous tile
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            pp_issue(sc, t + gridDim.x, b ? stage0 : stage1, b ? mbar0 : mbar1);
        }
        mbar_wait(b ? mbar1 : mbar0, (phases >> b) & 1u);
        phases ^= 1u << b;
        const int64_t i = t * kPPTile + threadIdx.x;
        if (i < sc.n) {
            const PPStage &S = stg[b];
            const int j = threadIdx.x;
            PPIn in;
            in.mx = S.m[0][j];
            in.my = S.m[1][j];
            in.mz = S.m[2][j];
            in.qw = S.q[0][j];
            in.qx = S.q[1][j];
            in.qy = S.q[2][j];
            in.qz = S.q[3][j];
            in.sx = S.s[0][j];
            in.sy = S.s[1][j];
            in.sz = S.s[2][j];
            in.rsq = S.rsq[j];
            in.opac = S.op[j];
            unsigned long long key;
            const bool kept = pp_one(cam, do_cull, i, in, geo, ibox, zhist ? s_zh : nullptr, key);
            keys[i] = key;
            if (keep_out) keep_out[i] = kept ? 1 : 0;
            if (kept) {
                cnt++;
                kmn = key < kmn ? key : kmn;
                kmx = key > kmx ? key : kmx;
            }
        }
        __syncthreads();  // stage b is refilled by the tile after next
    }
    pp_reduce(cnt, kmn, kmx, s_zh, zhist, ctr);
}

// Colour of the splat at depth rank r of a pass (order[r] = Gaussian index):
// the Gaussian's SH row (rows of 48 coefficients, 12 x 16 B loads) and mean,
// every load before any arithmetic (one memory round trip).  Only the ranks
// a pass sorted are coloured, so splats behind the front slice that no
// unsaturated pixel reaches never read their 192 B of SH.
#ifndef GSR_COLOR_MINB
#define GSR_COLOR_MINB 1
#endif
template <typename ShT, int DEG>
__global__ void __launch_bounds__(256, GSR_COLOR_MINB) color_ranked_kernel(
    SceneView sc, const FrameParams *__restrict__ fp, DepthOrder ord,
    const uint32_t *__restrict__ count, float4 *__restrict__ colr) {
    const int64_t kr = (int64_t)*count;
    const CameraArgs &cam = fp->cam;
    const uint32_t *order = ord.sched[16] ? ord.order1 : ord.order0;
    // grid-stride over the ranked splats (the grid is bounded; the count is
    // read on the device)
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < kr;
         r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = __ldg(order + r);
    const int64_t st = sc.stride;
    float cr, cg, cbl;
    if (DEG == 0) {  // render.py:129-130
        cr = __ldg(sc.dc + i);
        cg = __ldg(sc.dc + st + i);
        cbl = __ldg(sc.dc + 2 * st + i);
    } else {  // render.py:134-160
        constexpr int NC = (DEG + 1) * (DEG + 1) * 3;
        ShT v[NC];
        if (sizeof(ShT) == 4) {  // f32 rows: 192 B (224 B records with the mean), 16 B aligned
            constexpr int N4 = (NC + 3) / 4;
            const float4 *row =
                reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(sc.sh) + i * sc.sh_row);
            float4 q[N4];
#pragma unroll
            for (int k = 0; k < N4; k++) q[k] = __ldg(row + k);
#pragma unroll
            for (int k = 0; k < NC; k++) {
                const float4 &w = q[k >> 2];
                v[k] = (ShT)((k & 3) == 0 ? w.x : (k & 3) == 1 ? w.y : (k & 3) == 2 ? w.z : w.w);
            }
        } else {  // f64 rows: 384 B
            constexpr int N2 = (NC + 1) / 2;
            const double2 *row = reinterpret_cast<const double2 *>(sc.sh) + i * 24;
            double2 q[N2];
#pragma unroll
            for (int k = 0; k < N2; k++) q[k] = __ldg(row + k);
#pragma unroll
            for (int k = 0; k < NC; k++) v[k] = (ShT)((k & 1) ? q[k >> 1].y : q[k >> 1].x);
        }
        const double *m4 = sc.mean4 + (int64_t)sc.m4_row * i;
        const double2 m01 = __ldg(reinterpret_cast<const double2 *>(m4));
        const double mx = m01.x, my = m01.y, mz = __ldg(m4 + 2);
        const double dx = mx - cam.campos[0];
        const double dy = my - cam.campos[1];
        const double dz = mz - cam.campos[2];
        const double norm = sqrt((dx * dx + dy * dy) + dz * dz);
        const double den = norm > 1e-12 ? norm : 1e-12;
        const double ux = dx / den, uy = dy / den, uz = dz / den;
        const double xx = ux * ux, yy = uy * uy, zz = uz * uz;
        const double xy = ux * uy, yz = uy * uz, xz = ux * uz;
        cr = (float)sh_channel<DEG>(v, 0, ux, uy, uz, xx, yy, zz, xy, yz, xz);
        cg = (float)sh_channel<DEG>(v, 1, ux, uy, uz, xx, yy, zz, xy, yz, xz);
        cbl = (float)sh_channel<DEG>(v, 2, ux, uy, uz, xx, yy, zz, xy, yz, xz);
    }
    colr[r] = make_float4(cr, cg, cbl, 0.0f);
    }
}

// The same colours with the gather done by the bulk-copy (TMA) engine: each
// warp takes 32 consecutive ranks; every lane issues one cp.async.bulk copy
// of its Gaussian's 224 B colour record -- 192 B SH row and 32 B mean,
// adjacent in the scene (scene.cuh) -- into the warp's shared-memory rows,
// completing on the warp's mbarrier (two copies: 0.0572 ms per frame at
// config 3, the bulk-copy issue rate bound it); the lanes then
// evaluate from shared memory.  Decouples the gather (no per-thread loads
// in flight, no LSU throttling) from the 96 registers the SH evaluation
// holds.  f32 SH only (every PLY scene; f64 scenes use the kernel above).
constexpr int kBulkRow = 240;  // 192 B SH + 32 B mean + 16 B pad: 60 words, so a
                               // warp's LDS.128 of 32 rows hits all 32 banks
constexpr uint32_t kBulkTx = 224u;  // bytes per splat either way
constexpr int kBulkWarps = 3;  // two 7.5 KB row buffers per warp: 46 KB per CTA

// A warp's chunk of 32 ranks: their Gaussian indices (the order read),
// then lane 0 arms the chunk buffer's mbarrier with the bytes and every valid
// lane issues its copy.
__device__ __forceinline__ void bulk_issue(const SceneView &sc, const uint32_t *order,
                                           int64_t r0, int64_t kr, int lane, uint32_t rbase,
                                           uint32_t mbar) {
    const int64_t r = r0 + lane;
    const bool valid = r < kr;
    const uint32_t bal = __ballot_sync(0xffffffffu, valid);
    const int64_t i = valid ? (int64_t)__ldg(order + r) : 0;
    if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(mbar), "r"((uint32_t)__popc(bal) * kBulkTx) : "memory");
    if (valid) {
        const uint32_t dst = rbase + (uint32_t)lane * kBulkRow;
        if (sc.m4_row == 28) {  // one 224 B record: SH row then mean (scene.cuh)
            bulk_g2s(dst, reinterpret_cast<const float *>(sc.sh) + i * 56, 224u, mbar);
        } else {
            bulk_g2s(dst, reinterpret_cast<const float *>(sc.sh) + i * sc.sh_row, 192u, mbar);
            bulk_g2s(dst + 192u, sc.mean4 + (int64_t)sc.m4_row * i, 32u, mbar);
        }
    }
}

// Double-buffered per warp: chunk k + 1's copies are in flight while chunk k
// is evaluated.
template <int DEG>
__global__ void __launch_bounds__(kBulkWarps * 32) color_ranked_bulk_kernel(
    SceneView sc, const FrameParams *__restrict__ fp, DepthOrder ord,
    const uint32_t *__restrict__ count, float4 *__restrict__ colr) {
    __shared__ __align__(128) unsigned char rows[kBulkWarps][2][32 * kBulkRow];
    __shared__ __align__(8) unsigned long long bar[kBulkWarps][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // (scalars and selects, not arrays indexed by the buffer: those go to
    // local memory)
    const uint32_t mbar0 = (uint32_t)__cvta_generic_to_shared(&bar[w][0]);
    const uint32_t mbar1 = (uint32_t)__cvta_generic_to_shared(&bar[w][1]);
    const uint32_t rbase0 = (uint32_t)__cvta_generic_to_shared(&rows[w][0][0]);
    const uint32_t rbase1 = (uint32_t)__cvta_generic_to_shared(&rows[w][1][0]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t kr = (int64_t)*count;
    const CameraArgs &cam = fp->cam;
    const uint32_t *order = ord.sched[16] ? ord.order1 : ord.order0;
    uint32_t phases = 0u;  // bit k: the parity buffer k waits for next
    const int64_t wstride = (int64_t)gridDim.x * kBulkWarps * 32;
    int64_t r0 = ((int64_t)blockIdx.x * kBulkWarps + w) * 32;
    if (r0 < kr) bulk_issue(sc, order, r0, kr, lane, rbase0, mbar0);
    for (int b = 0; r0 < kr; r0 += wstride, b ^= 1) {
        // the other buffer was read by the generic proxy two chunks ago
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (r0 + wstride < kr)
            bulk_issue(sc, order, r0 + wstride, kr, lane, b ? rbase0 : rbase1, b ? mbar0 : mbar1);
        mbar_wait(b ? mbar1 : mbar0, (phases >> b) & 1u);
        phases ^= 1u << b;
        const int64_t r = r0 + lane;
        if (r < kr) {
            constexpr int NC = (DEG + 1) * (DEG + 1) * 3;
            const unsigned char *row = &rows[w][b][lane * kBulkRow];
            float v[NC];
#pragma unroll
            for (int k = 0; k < (NC + 3) / 4; k++) {
                const float4 q = *reinterpret_cast<const float4 *>(row + 16 * k);
                if (4 * k + 0 < NC) v[4 * k + 0] = q.x;
                if (4 * k + 1 < NC) v[4 * k + 1] = q.y;
                if (4 * k + 2 < NC) v[4 * k + 2] = q.z;
                if (4 * k + 3 < NC) v[4 * k + 3] = q.w;
            }
            const double2 m01 = *reinterpret_cast<const double2 *>(row + 192);
            const double mz = *reinterpret_cast<const double *>(row + 208);
            const double dx = m01.x - cam.campos[0];
            const double dy = m01.y - cam.campos[1];
            const double dz = mz - cam.campos[2];
            const double norm = sqrt((dx * dx + dy * dy) + dz * dz);
            const double den = norm > 1e-12 ? norm : 1e-12;
            const double ux = dx / den, uy = dy / den, uz = dz / den;
            const double xx = ux * ux, yy = uy * uy, zz = uz * uz;
            const double xy = ux * uy, yz = uy * uz, xz = ux * uz;
            const float cr = (float)sh_channel<DEG>(v, 0, ux, uy, uz, xx, yy, zz, xy, yz, xz);
            const float cg = (float)sh_channel<DEG>(v, 1, ux, uy, uz, xx, yy, zz, xy, yz, xz);
            const float cb = (float)sh_channel<DEG>(v, 2, ux, uy, uz, xx, yy, zz, xy, yz, xz);
            colr[r] = make_float4(cr, cg, cb, 0.0f);
        }
    }
}

}  // namespace

void launch_frame_start(const FrameParams &p, FrameParams *dst, FrameCounters *ctr,
                        cudaStream_t s) {
    frame_start_kernel<<<1, kFrameStartThreads, 0, s>>>(p, dst, ctr);
}

const void *frame_start_kernel_fn() { return (const void *)frame_start_kernel; }

void launch_preprocess_geo(const SceneView &scene, const FrameParams *fp, int frustum_cull,
                           unsigned long long *keys, GeoRec *geo, uint8_t *keep_out,
                           FrameCounters *ctr, uint32_t *zhist, uint2 *ibox, cudaStream_t s,
                           const KMark &mark) {
    if (scene.n == 0) return;
#ifndef GSR_PP_BULK
#define GSR_PP_BULK 1
#endif
    if (GSR_PP_BULK) {
        static int sms = 0;  // (one device model per process)
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
            // the largest shared carveout: GSR_PPB_MINB CTAs of ~52 KB per SM
            cudaFuncSetAttribute(preprocess_geo_bulk_kernel,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            // (the default dynamic limit is 48 KB minus the static 5.5 KB)
            cudaFuncSetAttribute(preprocess_geo_bulk_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(2 * sizeof(PPStage)));
        }
        const int64_t tiles = (scene.n + kPPTile - 1) / kPPTile;
        const unsigned blocks =
            (unsigned)std::min<int64_t>(tiles, (int64_t)sms * GSR_PPB_MINB);
        preprocess_geo_bulk_kernel<<<blocks, kPPTile, 2 * sizeof(PPStage), s>>>(
            scene, fp, frustum_cull, keys, geo, keep_out, ctr, zhist, ibox);
    } else {
        const int threads = 256;
        const unsigned blocks = (unsigned)((scene.n + threads - 1) / threads);
        preprocess_geo_kernel<<<blocks, threads, 0, s>>>(scene, fp, frustum_cull, keys, geo,
                                                         keep_out, ctr, zhist, ibox);
    }
    mark("preprocess_geo");
}

void launch_color_ranked(const SceneView &scene, const FrameParams *fp, int sh_degree,
                         DepthOrder ord, const uint32_t *count, int64_t cap, float4 *colr,
                         cudaStream_t s, const KMark &mark) {
    if (cap <= 0) return;
    const int threads = 256;
    static int sms = 0;  // (one device model per process)
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const unsigned blocks = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((cap + threads - 1) / threads, (int64_t)sms * 8));
#define GSR_COLOR(T, D)                                                                   \
    color_ranked_kernel<T, D><<<blocks, threads, 0, s>>>(scene, fp, ord, count, colr)
#ifndef GSR_COLOR_BULK
#define GSR_COLOR_BULK 1
#endif
    if (GSR_COLOR_BULK && scene.sh_f32 && sh_degree >= 1) {
        const unsigned bb = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((cap + kBulkWarps * 32 - 1) / (kBulkWarps * 32), (int64_t)sms * 8));
        if (sh_degree == 1)
            color_ranked_bulk_kernel<1><<<bb, kBulkWarps * 32, 0, s>>>(scene, fp, ord, count, colr);
        else if (sh_degree == 2)
            color_ranked_bulk_kernel<2><<<bb, kBulkWarps * 32, 0, s>>>(scene, fp, ord, count, colr);
        else
            color_ranked_bulk_kernel<3><<<bb, kBulkWarps * 32, 0, s>>>(scene, fp, ord, count, colr);
        mark("color_ranked");
        return;
    }
    if (sh_degree == 0) GSR_COLOR(float, 0);
    else if (scene.sh_f32 && sh_degree == 1) GSR_COLOR(float, 1);
    else if (scene.sh_f32 && sh_degree == 2) GSR_COLOR(float, 2);
    else if (scene.sh_f32) GSR_COLOR(float, 3);
    else if (sh_degree == 1) GSR_COLOR(double, 1);
    else if (sh_degree == 2) GSR_COLOR(double, 2);
    else GSR_COLOR(double, 3);
#undef GSR_COLOR
    mark("color_ranked");
}

}  // namespace gsr
