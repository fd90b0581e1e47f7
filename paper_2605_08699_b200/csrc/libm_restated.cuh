// libm_restated.cuh -- the f64 transcendental functions the reference's load
// and packing paths call, restated bit-for-bit for the device.
//
// The reference activates primitives with numpy / scipy (model.py:211-252)
// and derives the cutoff radius with numpy (render.py:476-481).  On the x86
// hosts the reference runs on (AVX512_SKX dispatch, FMA libm) those calls are:
//   np.exp(float64)        -> Intel SVML __svml_exp8_ha (numpy's bundled SVML)
//   np.log(float64)        -> Intel SVML __svml_log8_ha
//   scipy.special.expit    -> 1 / (1 + exp(-x)) with glibc's exp (__exp_fma)
// Each is restated below from its published algorithm and the constant
// tables of the binaries in this image (numpy 2.3 _multiarray_umath,
// glibc libm), operation by operation with the same fused multiply-adds and
// rounding modes.  oracle/oracle.c holds an independent host restatement
// that the CPU tests pin against numpy / scipy / math.exp on millions of
// inputs (tests/test_oracle_golden.py); the GPU tests compare the kernels
// against it.  Range: finite x with |x| < 707.7 for svml_exp (the PLY
// loader's log-scales), all finite x for glibc_exp, x >= 2^-1022 for svml_log.
#pragma once

#include <cstdint>

namespace gsr {
namespace libm {

__host__ __device__ inline double u2d(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double d;
    __builtin_memcpy(&d, &u, 8);
    return d;
#endif
}
__host__ __device__ inline uint64_t d2u(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    __builtin_memcpy(&u, &d, 8);
    return u;
#endif
}

// ---- SVML exp8_ha -------------------------------------------------------
// 2^(j/16) (hi, relative lo), j = 0..15
static __device__ __constant__ const double kSvExpT[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};
static __device__ __constant__ const double kSvExpL[16] = {
    0x0.0p+0, 0x1.79aa65d837b6dp-54, -0x1.01b15eaa59348p-55, 0x1.68efde3a8a894p-54,
    0x1.34d754db0abb6p-55, 0x1.59f48a72a4c6dp-55, 0x1.690cebb7aafb0p-56, 0x1.063e1e21c5409p-54,
    -0x1.3b3efbf5e2228p-54, -0x1.b32dcb94da51dp-56, 0x1.db72fc1f0eab4p-55, 0x1.1affc2b91ce27p-56,
    0x1.c1a7792cb3387p-55, 0x1.36eae30af0cb3p-56, 0x1.4a385a63d07a7p-56, -0x1.ff7128fd391f0p-55};

__device__ inline double svml_exp(double x) {
    if (!(x < 0x1.62e42fefa39efp+9)) return x != x ? x : __longlong_as_double(0x7ff0000000000000ll);
    if (x < -0x1.74910d52d3053p+9) return 0.0;
    // x / ln2 truncated (round-toward-zero FMA) to the 1/16 grid: k + j/16
    const double s = __fma_rz(x, 0x1.71547652b82fep+0, 0x1.8000000003ff0p+48);
    const double kd = __dsub_rn(s, 0x1.8000000003ff0p+48);
    const int j = (int)(d2u(s) & 15u);
    double r = __fma_rn(-kd, 0x1.62e42fefa39efp-1, x);
    r = __fma_rn(-kd, 0x1.abc9e3b39803fp-56, r);
    const double r2 = __dmul_rn(r, r);
    const double p1 = __fma_rn(r, 0x1.7411836940c04p-10, 0x1.1101cbbc265c0p-7);
    const double p2 = __fma_rn(r, 0x1.55557242d68fep-5, 0x1.5555553939732p-3);
    const double p3 = __fma_rn(r, 0x1.000000000d008p-1, 0x1.fffffffffff70p-1);
    double p = __fma_rn(p1, r2, p2);
    p = __fma_rn(p, r2, p3);
    const double q = __fma_rn(p, r, kSvExpL[j]);
    const double res = __fma_rn(q, kSvExpT[j], kSvExpT[j]);
    // vscalefpd(res, kd) = res * 2^floor(kd)
    const int e = (int)floor(kd);
    if (e >= -1021 && e <= 1022) return __dmul_rn(res, u2d((uint64_t)(e + 1023) << 52));
    // |x| >= 707.7 (SVML's rare path; not pinned): two exact-ish steps
    const int e1 = e / 2, e2 = e - e1;
    return __dmul_rn(__dmul_rn(res, u2d((uint64_t)(e1 + 1023) << 52)),
                     u2d((uint64_t)(e2 + 1023) << 52));
}

// ---- glibc exp (sysdeps/ieee754/dbl-64/e_exp.c, x86_64 FMA variant) -------
// table: 2^(k/128) as (tail, head - (k << 45)), k = 0..127 (__exp_data.tab)
static __device__ __constant__ const uint64_t kGlibcExpTab[256] = {
    0x0000000000000000ull, 0x3ff0000000000000ull, 0x3c9b3b4f1a88bf6eull, 0x3feff63da9fb3335ull,
    0xbc7160139cd8dc5dull, 0x3fefec9a3e778061ull, 0xbc905e7a108766d1ull, 0x3fefe315e86e7f85ull,
    0x3c8cd2523567f613ull, 0x3fefd9b0d3158574ull, 0xbc8bce8023f98efaull, 0x3fefd06b29ddf6deull,
    0x3c60f74e61e6c861ull, 0x3fefc74518759bc8ull, 0x3c90a3e45b33d399ull, 0x3fefbe3ecac6f383ull,
    0x3c979aa65d837b6dull, 0x3fefb5586cf9890full, 0x3c8eb51a92fdeffcull, 0x3fefac922b7247f7ull,
    0x3c3ebe3d702f9cd1ull, 0x3fefa3ec32d3d1a2ull, 0xbc6a033489906e0bull, 0x3fef9b66affed31bull,
    0xbc9556522a2fbd0eull, 0x3fef9301d0125b51ull, 0xbc5080ef8c4eea55ull, 0x3fef8abdc06c31ccull,
    0xbc91c923b9d5f416ull, 0x3fef829aaea92de0ull, 0x3c80d3e3e95c55afull, 0x3fef7a98c8a58e51ull,
    0xbc801b15eaa59348ull, 0x3fef72b83c7d517bull, 0xbc8f1ff055de323dull, 0x3fef6af9388c8deaull,
    0x3c8b898c3f1353bfull, 0x3fef635beb6fcb75ull, 0xbc96d99c7611eb26ull, 0x3fef5be084045cd4ull,
    0x3c9aecf73e3a2f60ull, 0x3fef54873168b9aaull, 0xbc8fe782cb86389dull, 0x3fef4d5022fcd91dull,
    0x3c8a6f4144a6c38dull, 0x3fef463b88628cd6ull, 0x3c807a05b0e4047dull, 0x3fef3f49917ddc96ull,
    0x3c968efde3a8a894ull, 0x3fef387a6e756238ull, 0x3c875e18f274487dull, 0x3fef31ce4fb2a63full,
    0x3c80472b981fe7f2ull, 0x3fef2b4565e27cddull, 0xbc96b87b3f71085eull, 0x3fef24dfe1f56381ull,
    0x3c82f7e16d09ab31ull, 0x3fef1e9df51fdee1ull, 0xbc3d219b1a6fbffaull, 0x3fef187fd0dad990ull,
    0x3c8b3782720c0ab4ull, 0x3fef1285a6e4030bull, 0x3c6e149289cecb8full, 0x3fef0cafa93e2f56ull,
    0x3c834d754db0abb6ull, 0x3fef06fe0a31b715ull, 0x3c864201e2ac744cull, 0x3fef0170fc4cd831ull,
    0x3c8fdd395dd3f84aull, 0x3feefc08b26416ffull, 0xbc86a3803b8e5b04ull, 0x3feef6c55f929ff1ull,
    0xbc924aedcc4b5068ull, 0x3feef1a7373aa9cbull, 0xbc9907f81b512d8eull, 0x3feeecae6d05d866ull,
    0xbc71d1e83e9436d2ull, 0x3feee7db34e59ff7ull, 0xbc991919b3ce1b15ull, 0x3feee32dc313a8e5ull,
    0x3c859f48a72a4c6dull, 0x3feedea64c123422ull, 0xbc9312607a28698aull, 0x3feeda4504ac801cull,
    0xbc58a78f4817895bull, 0x3feed60a21f72e2aull, 0xbc7c2c9b67499a1bull, 0x3feed1f5d950a897ull,
    0x3c4363ed60c2ac11ull, 0x3feece086061892dull, 0x3c9666093b0664efull, 0x3feeca41ed1d0057ull,
    0x3c6ecce1daa10379ull, 0x3feec6a2b5c13cd0ull, 0x3c93ff8e3f0f1230ull, 0x3feec32af0d7d3deull,
    0x3c7690cebb7aafb0ull, 0x3feebfdad5362a27ull, 0x3c931dbdeb54e077ull, 0x3feebcb299fddd0dull,
    0xbc8f94340071a38eull, 0x3feeb9b2769d2ca7ull, 0xbc87deccdc93a349ull, 0x3feeb6daa2cf6642ull,
    0xbc78dec6bd0f385full, 0x3feeb42b569d4f82ull, 0xbc861246ec7b5cf6ull, 0x3feeb1a4ca5d920full,
    0x3c93350518fdd78eull, 0x3feeaf4736b527daull, 0x3c7b98b72f8a9b05ull, 0x3feead12d497c7fdull,
    0x3c9063e1e21c5409ull, 0x3feeab07dd485429ull, 0x3c34c7855019c6eaull, 0x3feea9268a5946b7ull,
    0x3c9432e62b64c035ull, 0x3feea76f15ad2148ull, 0xbc8ce44a6199769full, 0x3feea5e1b976dc09ull,
    0xbc8c33c53bef4da8ull, 0x3feea47eb03a5585ull, 0xbc845378892be9aeull, 0x3feea34634ccc320ull,
    0xbc93cedd78565858ull, 0x3feea23882552225ull, 0x3c5710aa807e1964ull, 0x3feea155d44ca973ull,
    0xbc93b3efbf5e2228ull, 0x3feea09e667f3bcdull, 0xbc6a12ad8734b982ull, 0x3feea012750bdabfull,
    0xbc6367efb86da9eeull, 0x3fee9fb23c651a2full, 0xbc80dc3d54e08851ull, 0x3fee9f7df9519484ull,
    0xbc781f647e5a3ecfull, 0x3fee9f75e8ec5f74ull, 0xbc86ee4ac08b7db0ull, 0x3fee9f9a48a58174ull,
    0xbc8619321e55e68aull, 0x3fee9feb564267c9ull, 0x3c909ccb5e09d4d3ull, 0x3feea0694fde5d3full,
    0xbc7b32dcb94da51dull, 0x3feea11473eb0187ull, 0x3c94ecfd5467c06bull, 0x3feea1ed0130c132ull,
    0x3c65ebe1abd66c55ull, 0x3feea2f336cf4e62ull, 0xbc88a1c52fb3cf42ull, 0x3feea427543e1a12ull,
    0xbc9369b6f13b3734ull, 0x3feea589994cce13ull, 0xbc805e843a19ff1eull, 0x3feea71a4623c7adull,
    0xbc94d450d872576eull, 0x3feea8d99b4492edull, 0x3c90ad675b0e8a00ull, 0x3feeaac7d98a6699ull,
    0x3c8db72fc1f0eab4ull, 0x3feeace5422aa0dbull, 0xbc65b6609cc5e7ffull, 0x3feeaf3216b5448cull,
    0x3c7bf68359f35f44ull, 0x3feeb1ae99157736ull, 0xbc93091fa71e3d83ull, 0x3feeb45b0b91ffc6ull,
    0xbc5da9b88b6c1e29ull, 0x3feeb737b0cdc5e5ull, 0xbc6c23f97c90b959ull, 0x3feeba44cbc8520full,
    0xbc92434322f4f9aaull, 0x3feebd829fde4e50ull, 0xbc85ca6cd7668e4bull, 0x3feec0f170ca07baull,
    0x3c71affc2b91ce27ull, 0x3feec49182a3f090ull, 0x3c6dd235e10a73bbull, 0x3feec86319e32323ull,
    0xbc87c50422622263ull, 0x3feecc667b5de565ull, 0x3c8b1c86e3e231d5ull, 0x3feed09bec4a2d33ull,
    0xbc91bbd1d3bcbb15ull, 0x3feed503b23e255dull, 0x3c90cc319cee31d2ull, 0x3feed99e1330b358ull,
    0x3c8469846e735ab3ull, 0x3feede6b5579fdbfull, 0xbc82dfcd978e9db4ull, 0x3feee36bbfd3f37aull,
    0x3c8c1a7792cb3387ull, 0x3feee89f995ad3adull, 0xbc907b8f4ad1d9faull, 0x3feeee07298db666ull,
    0xbc55c3d956dcaebaull, 0x3feef3a2b84f15fbull, 0xbc90a40e3da6f640ull, 0x3feef9728de5593aull,
    0xbc68d6f438ad9334ull, 0x3feeff76f2fb5e47ull, 0xbc91eee26b588a35ull, 0x3fef05b030a1064aull,
    0x3c74ffd70a5fddcdull, 0x3fef0c1e904bc1d2ull, 0xbc91bdfbfa9298acull, 0x3fef12c25bd71e09ull,
    0x3c736eae30af0cb3ull, 0x3fef199bdd85529cull, 0x3c8ee3325c9ffd94ull, 0x3fef20ab5fffd07aull,
    0x3c84e08fd10959acull, 0x3fef27f12e57d14bull, 0x3c63cdaf384e1a67ull, 0x3fef2f6d9406e7b5ull,
    0x3c676b2c6c921968ull, 0x3fef3720dcef9069ull, 0xbc808a1883ccb5d2ull, 0x3fef3f0b555dc3faull,
    0xbc8fad5d3ffffa6full, 0x3fef472d4a07897cull, 0xbc900dae3875a949ull, 0x3fef4f87080d89f2ull,
    0x3c74a385a63d07a7ull, 0x3fef5818dcfba487ull, 0xbc82919e2040220full, 0x3fef60e316c98398ull,
    0x3c8e5a50d5c192acull, 0x3fef69e603db3285ull, 0x3c843a59ac016b4bull, 0x3fef7321f301b460ull,
    0xbc82d52107b43e1full, 0x3fef7c97337b9b5full, 0xbc892ab93b470dc9ull, 0x3fef864614f5a129ull,
    0x3c74b604603a88d3ull, 0x3fef902ee78b3ff6ull, 0x3c83c5ec519d7271ull, 0x3fef9a51fbc74c83ull,
    0xbc8ff7128fd391f0ull, 0x3fefa4afa2a490daull, 0xbc8dae98e223747dull, 0x3fefaf482d8e67f1ull,
    0x3c8ec3bc41aa2008ull, 0x3fefba1bee615a27ull, 0x3c842b94c3a9eb32ull, 0x3fefc52b376bba97ull,
    0x3c8a64a931d185eeull, 0x3fefd0765b6e4540ull, 0xbc8e37bae43be3edull, 0x3fefdbfdad9cbe14ull,
    0x3c77893b4d91cd9dull, 0x3fefe7c1819e90d8ull, 0x3c5305c14160cc89ull, 0x3feff3c22b8f71f1ull,
};

__device__ inline double glibc_exp(double x) {
    const double InvLn2N = 0x1.71547652b82fep+7, Shift = 0x1.8p52;
    const double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
    const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    uint32_t abstop = (uint32_t)(d2u(x) >> 52) & 0x7ffu;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if ((int)abstop - 0x3c9 < 0) return __dadd_rn(1.0, x);  // |x| < 2^-54
        if (abstop >= 0x409u) {                                // |x| >= 1024
            if (d2u(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return __dadd_rn(1.0, x);
            return (d2u(x) >> 63) ? 0.0 : u2d(0x7ff0000000000000ull);
        }
        abstop = 0;  // 512 <= |x| < 1024: specialcase below
    }
    double kd = __fma_rn(InvLn2N, x, Shift);
    const uint64_t ki = d2u(kd);
    kd = __dsub_rn(kd, Shift);
    const double r = __fma_rn(kd, NegLn2loN, __fma_rn(kd, NegLn2hiN, x));
    const uint32_t idx = 2u * (uint32_t)(ki % 128u);
    const uint64_t top = ki << 45;
    const double tail = u2d(kGlibcExpTab[idx]);
    uint64_t sbits = kGlibcExpTab[idx + 1] + top;
    const double r2 = __dmul_rn(r, r);
    const double tmp = __fma_rn(__dmul_rn(r2, r2), __fma_rn(r, C5, C4),
                                __fma_rn(r2, __fma_rn(r, C3, C2), __dadd_rn(tail, r)));
    if (abstop == 0) {  // specialcase (e_exp.c)
        if ((ki & 0x80000000ull) == 0) {
            sbits -= 1009ull << 52;
            const double scale = u2d(sbits);
            return __dmul_rn(0x1p1009, __fma_rn(scale, tmp, scale));
        }
        sbits += 1022ull << 52;
        const double scale = u2d(sbits);
        double y = __fma_rn(scale, tmp, scale);
        if (y < 1.0) {
            double lo = __fma_rn(scale, tmp, __dsub_rn(scale, y));
            const double hi = __dadd_rn(1.0, y);
            lo = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
            y = __dsub_rn(__dadd_rn(hi, lo), 1.0);
            if (y == 0.0) y = 0.0;
        }
        return __dmul_rn(0x1p-1022, y);
    }
    const double scale = u2d(sbits);
    return __fma_rn(scale, tmp, scale);
}

// ---- SVML log8_ha ---------------------------------------------------------
// vrcp14pd(m) rounded to 1/32 (vrndscalepd 0x58) is a step function of the
// mantissa m in [1, 2); its 16 steps, probed on the AVX-512 host (monotone,
// checked on 2e8 random mantissas): rcp = (32 - #thresholds <= m) / 32.
static __device__ __constant__ const double kSvLogTh[16] = {
    0x1.040fp+0, 0x1.0c97p+0, 0x1.15b4p+0, 0x1.1f7p+0,  0x1.29e6p+0, 0x1.3523p+0,
    0x1.4143p+0, 0x1.4e5fp+0, 0x1.5c99p+0, 0x1.6c15p+0, 0x1.7d07p+0, 0x1.8f9cp+0,
    0x1.a41ap+0, 0x1.badp+0,  0x1.d41cp+0, 0x1.f08p+0};
// -log(rcp) (or -log(2 rcp) for rcp < 3/4) hi / lo, indexed by rcp's top 4 mantissa bits
static __device__ __constant__ const double kSvLogH[16] = {
    0x0.0p+0, -0x1.f0a30c0120000p-5, -0x1.e27076e2b0000p-4, -0x1.5ff3070a78000p-3,
    -0x1.c8ff7c79a8000p-3, -0x1.1675cababc000p-2, -0x1.4618bc21c4000p-2, -0x1.739d7f6bbc000p-2,
    0x1.269621134c000p-2, 0x1.f991c6cb38000p-3, 0x1.a93ed3c8b0000p-3, 0x1.5bf406b540000p-3,
    0x1.1178e82280000p-3, 0x1.9335e5d590000p-4, 0x1.08598b59e0000p-4, 0x1.0415d89e80000p-5};
static __device__ __constant__ const double kSvLogL[16] = {
    0x0.0p+0, 0x1.3ab33d066d1d2p-42, 0x1.a342c2af0003cp-45, -0x1.3d3c873e20a07p-43,
    -0x1.a21ac25d81ef3p-43, 0x1.9f1fc63382a8fp-42, -0x1.ec27d0b7b37b3p-42, -0x1.0069ce24c53fbp-42,
    0x1.b92783beb7677p-42, 0x1.9bcbecca0cdf3p-42, -0x1.30e486a0ac42dp-42, 0x1.ed8fdc149767ep-42,
    -0x1.b8421cc74be04p-43, 0x1.2622b8757a8fbp-42, 0x1.d034451fecdfbp-43, -0x1.77771fd187145p-42};

__device__ inline double svml_log(double x) {  // x positive, normal, finite
    const uint64_t b = d2u(x);
    double e = (double)((int)((b >> 52) & 0x7ffu) - 1023);          // vgetexppd
    const double m = u2d((b & 0xfffffffffffffull) | 0x3ff0000000000000ull);  // vgetmantpd
    int k = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) k += m >= kSvLogTh[i] ? 1 : 0;
    const double rcp = (double)(32 - k) * 0.03125;
    const double r = __fma_rn(rcp, m, -1.0);
    if (rcp < 0.75) e = __dadd_rn(e, 1.0);
    const int idx = (int)((d2u(rcp) >> 48) & 15u);
    const double A = __fma_rn(r, 0x1.249229cee81efp-3, -0x1.55553fb28db06p-3);
    double B = __fma_rn(r, 0x1.c81cd309d7c70p-4, -0x1.007357e93af62p-3);
    const double r2 = __dmul_rn(r, r);
    double C = __fma_rn(r, 0x1.9999999cc9f5cp-3, -0x1.00000000c05bdp-2);
    B = __fma_rn(B, r2, A);
    const double r4 = __dmul_rn(r2, r2);
    const double D = __fma_rn(r, 0x1.5555555555466p-2, -0x1.fffffffffffc6p-2);
    const double th = __fma_rn(e, 0x1.62e42fefa0000p-1, kSvLogH[idx]);
    C = __fma_rn(C, r2, D);
    B = __fma_rn(B, r4, C);
    const double s = __dadd_rn(th, r);
    const double rl = __dsub_rn(r, __dsub_rn(s, th));
    const double poly = __fma_rn(B, r2, rl);
    const double elo = __fma_rn(e, 0x1.cf79abc9e0000p-40, kSvLogL[idx]);
    return __dadd_rn(s, __dadd_rn(poly, elo));
}

// render.py:476-481: min(2 log(max(op, f) / f), 4.5^2), f = 1 / (255 * 32)
__device__ inline double cutoff_radius_sq(double op) {
    const double f = 1.0 / (255.0 * 32.0);
    const double o = op > f ? op : f;  // np.maximum (op is finite here)
    const double r = __dmul_rn(2.0, svml_log(__ddiv_rn(o, f)));
    return r < 20.25 ? r : 20.25;
}

}  // namespace libm
}  // namespace gsr
