// Containment check of band_span_bound (paper_2605_08699_b200/csrc/common.cuh):
// for random splats and tile-row bands, whenever the bound is used, its pixel
// range must contain the exact contract span (exact_band_span) -- the
// property that keeps the blend's frames bit-exact with superset tile lists.
//   nvcc -O3 -std=c++17 -fmad=false -gencode arch=compute_100a,code=sm_100a \
//        -Iinclude -o span_check tools/span_check.cu && ./span_check [batches]
// Prints, per distribution: pairs tested, pairs bounded, violations (must
// be 0), and the tile columns the bound adds.
#include <cstdio>
#include <cstdlib>

#include "../paper_2605_08699_b200/csrc/common.cuh"

using namespace gsr;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}
__device__ __forceinline__ double uni(uint64_t &s) {
    s = mix(s + 0x9e3779b97f4a7c15ull);
    return (double)(s >> 11) * 0x1p-53;
}

struct Counts {
    unsigned long long tested, bounded, violations, extra_tiles, empty_exact;
};

// mode 0: realistic 3DGS splats at 1080p; 1: elongated / huge / tiny; 2: near
// tile and pixel boundaries (u, v on x.5 / multiples of 16, small sigmas)
__global__ void check_kernel(int mode, uint64_t seed, int per_thread, Counts *out) {
    const int W = 1920, H = 1080;
    uint64_t s = mix(seed ^ (((uint64_t)blockIdx.x << 20) + threadIdx.x));
    Counts c{0, 0, 0, 0, 0};
    for (int it = 0; it < per_thread; it++) {
        double s1, s2, u0, v0, op;
        if (mode == 0) {
            s1 = 0.3 + 30.0 * pow(uni(s), 2.0);
            s2 = 0.3 + 30.0 * pow(uni(s), 2.0);
            u0 = -50.0 + (W + 100.0) * uni(s);
            v0 = -50.0 + (H + 100.0) * uni(s);
        } else if (mode == 1) {
            s1 = pow(10.0, -1.0 + 4.0 * uni(s));  // 0.1 .. 1000 px
            s2 = pow(10.0, -1.0 + 4.0 * uni(s));
            u0 = -2000.0 + (W + 4000.0) * uni(s);
            v0 = -2000.0 + (H + 4000.0) * uni(s);
        } else {
            s1 = 0.3 + 4.0 * uni(s);
            s2 = 0.3 + 4.0 * uni(s);
            u0 = 16.0 * floor(uni(s) * 120.0) + (uni(s) < 0.5 ? 0.5 : 0.0) + (uni(s) - 0.5) * 1e-3;
            v0 = floor(uni(s) * H) + 0.5 + (uni(s) - 0.5) * 1e-4;
        }
        op = uni(s);
        const double th = 6.283185307179586 * uni(s);
        const double cs = cos(th), sn = sin(th);
        // 2-D covariance + the 0.3 floor (render.py:215-225), conic (render.py:442-447)
        const double a = cs * cs * s1 * s1 + sn * sn * s2 * s2 + 0.3;
        const double cc = sn * sn * s1 * s1 + cs * cs * s2 * s2 + 0.3;
        const double b = cs * sn * (s1 * s1 - s2 * s2);
        const double det = a * cc - b * b;
        const float ia = (float)(cc / det), ib = (float)(-b / det), ic = (float)(a / det);
        const double f = 1.0 / (255.0 * 32.0);
        double rsq = 2.0 * log(fmax(op, f) / f);
        rsq = rsq < 20.25 ? rsq : 20.25;
        const float u = (float)u0, v = (float)v0, rq = (float)rsq;
        const float ry = (float)sqrt(cc * rsq);
        int lo, hi;
        row_range(v, ry, H, lo, hi);
        if (lo >= hi) continue;
        const float rinv = splat_fast_ok(v, ia, ib) ? __frcp_rn(ia) : 0.0f;
        if (rinv == 0.0f) continue;
        for (int ty = lo / 16; ty <= (hi - 1) / 16; ty++) {
            const int y0 = max(lo, ty * 16), y1 = min(hi, ty * 16 + 16);
            int mn_b, mx_b, mn_e, mx_e;
            c.tested++;
            if (!band_span_bound(u, v, ia, ib, ic, rq, y0, y1, W, mn_b, mx_b)) continue;
            c.bounded++;
            exact_band_span(u, v, ia, ib, ic, rq, rinv, y0, y1, W, mn_e, mx_e);
            const bool e_has = mn_e <= mx_e && (mx_e - 1) / 16 - mn_e / 16 + 1 > 0 && mn_e < mx_e;
            if (!e_has) {
                c.empty_exact++;
                continue;
            }
            if (!(mn_b <= mn_e && mx_b >= mx_e)) {
                c.violations++;
                if (c.violations <= 2)
                    printf("VIOLATION mode %d u=%a v=%a ia=%a ib=%a ic=%a rsq=%a rows[%d,%d) "
                           "exact [%d,%d) bound [%d,%d)\n",
                           mode, u, v, ia, ib, ic, rq, y0, y1, mn_e, mx_e, mn_b, mx_b);
            } else {
                const int te = (mx_e - 1) / 16 - mn_e / 16 + 1;
                const int tb = mx_b > mn_b ? (mx_b - 1) / 16 - mn_b / 16 + 1 : 0;
                c.extra_tiles += (unsigned long long)(tb - te);
            }
        }
    }
    atomicAdd(&out->tested, c.tested);
    atomicAdd(&out->bounded, c.bounded);
    atomicAdd(&out->violations, c.violations);
    atomicAdd(&out->extra_tiles, c.extra_tiles);
    atomicAdd(&out->empty_exact, c.empty_exact);
}

int main(int argc, char **argv) {
    const int batches = argc > 1 ? atoi(argv[1]) : 20;
    Counts *d;
    cudaMalloc(&d, sizeof(Counts));
    unsigned long long total_viol = 0;
    for (int mode = 0; mode < 3; mode++) {
        cudaMemset(d, 0, sizeof(Counts));
        for (int bt = 0; bt < batches; bt++)
            check_kernel<<<148 * 8, 256>>>(mode, 1234567ull + 7919ull * bt + 1000003ull * mode, 64, d);
        Counts h;
        cudaMemcpy(&h, d, sizeof(Counts), cudaMemcpyDeviceToHost);
        printf("mode %d: pairs %llu, bounded %llu (%.2f%%), exact-empty %llu, violations %llu, "
               "extra tile columns %.4f per bounded pair\n",
               mode, h.tested, h.bounded, 100.0 * h.bounded / (double)(h.tested ? h.tested : 1),
               h.empty_exact, h.violations,
               h.extra_tiles / (double)(h.bounded ? h.bounded : 1));
        total_viol += h.violations;
    }
    printf("%s\n", total_viol ? "FAIL" : "OK: no violations");
    return total_viol ? 1 : 0;
}
