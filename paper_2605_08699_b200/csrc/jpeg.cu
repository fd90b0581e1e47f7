// jpeg.cu -- baseline JPEG encoding of the rendered u8 frame on the device:
// render.encode_jpeg (render.py:488-498; SURVEY.md 8f "next" row 1), which
// the reference runs through Pillow 12.2 -> libjpeg-turbo with quality q,
// 4:2:0 chroma below q90 and 4:4:4 at q90+, standard Huffman tables, no
// restart markers.  Each stage restates libjpeg-turbo's integer arithmetic so
// the output is byte-identical to Pillow's (tests/test_gpu_parity.py):
//   colour  jccolor.c rgb_ycc_convert: 16-bit fixed point, Y/Cb/Cr
//   chroma  jcsample.c h2v2_downsample: 2x2 sum + alternating bias 1,2,1,2
//   edges   jcsample.c expand_right_edge (to whole blocks) and jcprepct.c
//           expand_bottom_edge (rows to the MCU row), last sample replicated
//   DCT     jfdctint.c: the "islow" integer DCT (CONST_BITS 13, PASS1_BITS 2)
//   quant   jcdctmgr.c quantize + compute_reciprocal (16-bit DCTELEM of the
//           SIMD build): x -> sign(x) * ((|x| + corr) * recip >> (16 + shift))
//   blocks  jccoefct.c compress_data: dummy blocks at the right/bottom edge of
//           an MCU are zero with the DC of the previous block in the MCU
//   entropy jchuff.c encode_one_block with the Annex K tables, final byte
//           padded with 1 bits, 0xFF stuffed with 0x00.
// Kernels: (1) one thread per real 8x8 block of each component: fetch with
// edge replication, colour-convert, downsample, DCT, quantise; (2) one thread
// per block in scan (MCU) order: Huffman-coded length, DC prediction from the
// previous block of the same component; (3) exclusive scan of the lengths;
// (4) each block writes its bits at its offset (shared boundary words by
// atomicOr); (5) byte stuffing via a second scan.  Headers are built on the
// host (gsr_api.cu).
#include <mutex>

#include "kernels.cuh"
#include "scan.cuh"

namespace gsr {

namespace {

constexpr int kNaturalOrder[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
    41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
    30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

__constant__ int c_natural[64];
// Huffman codes (code, length) for DC lum/chrom [12] and AC lum/chrom [256]
__constant__ uint16_t c_dc_code[2][12];
__constant__ uint8_t c_dc_len[2][12];
__constant__ uint16_t c_ac_code[2][256];
__constant__ uint8_t c_ac_len[2][256];

struct Comp {
    int w, h;            // component size in samples (after downsampling)
    int wb, hb;          // width_in_blocks, height_in_blocks
    int mw, mh;          // blocks per MCU (h_samp, v_samp)
    int64_t coef_off;    // first block's coefficients in the coefficient buffer
};

// jcdctmgr.c divisors for one quality (kernel parameter: encodes of different
// qualities from concurrent contexts must not share mutable state)
struct QuantRecip {
    uint16_t recip[2][64], corr[2][64];
    int8_t shift[2][64];
};

struct JpegArgs {
    QuantRecip q;
    const uint8_t *rgb;  // (H, W, 3) device frame
    int W, H;
    int sub;             // 1: 4:2:0, 0: 4:4:4
    Comp c[3];
    int mcux, mcuy;      // MCUs per row / column
    int blocks_per_mcu;
    int64_t n_scan;      // scan-order blocks (incl. dummies)
    int16_t *coef;       // real blocks, 64 quantised coefficients each (natural order)
    uint32_t *bits;      // per scan block: coded length, then exclusive offset
    uint32_t *words;     // bitstream, big-endian bit order in 32-bit words
    uint32_t *scan_aux;  // scan work
    uint8_t *out;        // stuffed bytes
    uint32_t *out_len;   // [0] bits total, [1] stuffed byte count
};

// jccolor.c rgb_ycc_convert (16-bit fixed point, SCALEBITS = 16)
__device__ __forceinline__ int ycc(int ci, int r, int g, int b) {
    if (ci == 0) return (19595 * r + 38470 * g + 7471 * b + 32768) >> 16;
    if (ci == 1) return (-11059 * r - 21709 * g + 32768 * b + (128 << 16) + 32767) >> 16;
    return (32768 * r - 27439 * g - 5329 * b + (128 << 16) + 32767) >> 16;
}

// component ci sample (x, y) of the full-resolution colour plane, with the
// right edge replicated (expand_right_edge) and bottom rows replicated
__device__ __forceinline__ int plane_sample(const JpegArgs &a, int ci, int x, int y) {
    x = x < a.W ? x : a.W - 1;
    y = y < a.H ? y : a.H - 1;
    const uint8_t *p = a.rgb + 3 * ((int64_t)y * a.W + x);
    return ycc(ci, p[0], p[1], p[2]);
}

// one sample of component ci at component coordinates (cx, cy), after
// downsampling and both edge expansions (jcsample.c / jcprepct.c)
__device__ __forceinline__ int comp_sample(const JpegArgs &a, int ci, int cx, int cy) {
    const Comp &c = a.c[ci];
    cy = cy < c.h ? cy : c.h - 1;  // expand_bottom_edge of the component rows
    if (!(a.sub && ci > 0)) return plane_sample(a, ci, cx, cy);
    // h2v2_downsample: source columns expanded to 2 * wb * 8 by replicating
    // the last pixel, source rows padded to an even count the same way
    const int x0 = 2 * cx, y0 = 2 * cy;
    const int s = plane_sample(a, ci, x0, y0) + plane_sample(a, ci, x0 + 1, y0) +
                  plane_sample(a, ci, x0, y0 + 1) + plane_sample(a, ci, x0 + 1, y0 + 1);
    return (s + 1 + (cx & 1)) >> 2;  // bias 1, 2, 1, 2 ...
}

// jfdctint.c jpeg_fdct_islow on level-shifted samples, in place
__device__ void fdct_islow(int *d) {
    constexpr int CB = 13, P1 = 2;
    constexpr int F0298 = 2446, F0390 = 3196, F0541 = 4433, F0765 = 6270, F0899 = 7373,
                  F1175 = 9633, F1501 = 12299, F1847 = 15137, F1961 = 16069, F2053 = 16819,
                  F2562 = 20995, F3072 = 25172;
#define DESC(x, n) (((x) + (1 << ((n) - 1))) >> (n))
    for (int r = 0; r < 8; r++) {  // pass 1: rows
        int *p = d + 8 * r;
        int t0 = p[0] + p[7], t7 = p[0] - p[7], t1 = p[1] + p[6], t6 = p[1] - p[6];
        int t2 = p[2] + p[5], t5 = p[2] - p[5], t3 = p[3] + p[4], t4 = p[3] - p[4];
        int t10 = t0 + t3, t13 = t0 - t3, t11 = t1 + t2, t12 = t1 - t2;
        p[0] = (t10 + t11) * (1 << P1);
        p[4] = (t10 - t11) * (1 << P1);
        int z1 = (t12 + t13) * F0541;
        p[2] = DESC(z1 + t13 * F0765, CB - P1);
        p[6] = DESC(z1 + t12 * (-F1847), CB - P1);
        z1 = t4 + t7;
        int z2 = t5 + t6, z3 = t4 + t6, z4 = t5 + t7;
        const int z5 = (z3 + z4) * F1175;
        t4 *= F0298; t5 *= F2053; t6 *= F3072; t7 *= F1501;
        z1 *= -F0899; z2 *= -F2562; z3 *= -F1961; z4 *= -F0390;
        z3 += z5; z4 += z5;
        p[7] = DESC(t4 + z1 + z3, CB - P1);
        p[5] = DESC(t5 + z2 + z4, CB - P1);
        p[3] = DESC(t6 + z2 + z3, CB - P1);
        p[1] = DESC(t7 + z1 + z4, CB - P1);
    }
    for (int c = 0; c < 8; c++) {  // pass 2: columns
        int *p = d + c;
        int t0 = p[0] + p[56], t7 = p[0] - p[56], t1 = p[8] + p[48], t6 = p[8] - p[48];
        int t2 = p[16] + p[40], t5 = p[16] - p[40], t3 = p[24] + p[32], t4 = p[24] - p[32];
        int t10 = t0 + t3, t13 = t0 - t3, t11 = t1 + t2, t12 = t1 - t2;
        p[0] = DESC(t10 + t11, P1);
        p[32] = DESC(t10 - t11, P1);
        int z1 = (t12 + t13) * F0541;
        p[16] = DESC(z1 + t13 * F0765, CB + P1);
        p[48] = DESC(z1 + t12 * (-F1847), CB + P1);
        z1 = t4 + t7;
        int z2 = t5 + t6, z3 = t4 + t6, z4 = t5 + t7;
        const int z5 = (z3 + z4) * F1175;
        t4 *= F0298; t5 *= F2053; t6 *= F3072; t7 *= F1501;
        z1 *= -F0899; z2 *= -F2562; z3 *= -F1961; z4 *= -F0390;
        z3 += z5; z4 += z5;
        p[56] = DESC(t4 + z1 + z3, CB + P1);
        p[40] = DESC(t5 + z2 + z4, CB + P1);
        p[24] = DESC(t6 + z2 + z3, CB + P1);
        p[8] = DESC(t7 + z1 + z4, CB + P1);
    }
#undef DESC
}

__global__ void __launch_bounds__(128) jpeg_blocks_kernel(JpegArgs a, int64_t n_real) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_real) return;
    int ci = 0;
    int64_t bi = i;
    while (ci < 2 && bi >= (int64_t)a.c[ci].wb * a.c[ci].hb) {
        bi -= (int64_t)a.c[ci].wb * a.c[ci].hb;
        ci++;
    }
    const Comp &c = a.c[ci];
    const int bx = (int)(bi % c.wb), by = (int)(bi / c.wb);
    int d[64];
    for (int y = 0; y < 8; y++)
        for (int x = 0; x < 8; x++)  // convsamp: level shift by CENTERJSAMPLE
            d[8 * y + x] = comp_sample(a, ci, 8 * bx + x, 8 * by + y) - 128;
    fdct_islow(d);
    const int t = ci > 0;
    int16_t *out = a.coef + c.coef_off + 64 * bi;
    for (int k = 0; k < 64; k++) {  // jcdctmgr.c quantize (reciprocal form)
        int v = d[k];
        const bool neg = v < 0;
        const unsigned x = (unsigned)(neg ? -v : v);
        const unsigned p = (x + a.q.corr[t][k]) * (unsigned)a.q.recip[t][k];
        const int q = (int)(uint16_t)(p >> (16 + a.q.shift[t][k]));
        out[k] = (int16_t)(neg ? -q : q);
    }
}

// locate scan block s: component, block coordinates and whether it is real
struct ScanPos {
    int ci, bx, by, blk;  // blk: index of the block within its MCU for component ci
    int mcu;
};

__device__ __forceinline__ ScanPos scan_pos(const JpegArgs &a, int64_t s) {
    ScanPos p;
    p.mcu = (int)(s / a.blocks_per_mcu);
    int k = (int)(s % a.blocks_per_mcu);
    p.ci = 0;
    while (k >= a.c[p.ci].mw * a.c[p.ci].mh) {
        k -= a.c[p.ci].mw * a.c[p.ci].mh;
        p.ci++;
    }
    const Comp &c = a.c[p.ci];
    p.blk = k;
    const int mx = p.mcu % a.mcux, my = p.mcu / a.mcux;
    p.bx = mx * c.mw + k % c.mw;
    p.by = my * c.mh + k / c.mw;
    return p;
}

// DC of scan block s (dummy blocks: jccoefct.c rules), recursion-free
__device__ int scan_dc(const JpegArgs &a, int64_t s) {
    ScanPos p = scan_pos(a, s);
    const Comp &c = a.c[p.ci];
    while (!(p.bx < c.wb && p.by < c.hb)) {
        // a dummy block copies the DC of the previous block in the MCU buffer
        // (right edge: its left neighbour; bottom row: the previous row's last)
        p.blk--;
        const int mx = p.mcu % a.mcux, my = p.mcu / a.mcux;
        p.bx = mx * c.mw + p.blk % c.mw;
        p.by = my * c.mh + p.blk / c.mw;
    }
    return a.coef[c.coef_off + 64 * ((int64_t)p.by * c.wb + p.bx)];
}

__device__ __forceinline__ int nbits_of(int v) {
    const unsigned x = (unsigned)(v < 0 ? -v : v);
    return x ? 32 - __clz(x) : 0;
}

template <bool kWrite>
__device__ uint32_t encode_block(const JpegArgs &a, int64_t s, uint64_t pos) {
    const ScanPos p = scan_pos(a, s);
    const Comp &c = a.c[p.ci];
    const int t = p.ci > 0;
    const bool real = p.bx < c.wb && p.by < c.hb;
    const int16_t *blk = a.coef + c.coef_off + 64 * ((int64_t)p.by * c.wb + p.bx);
    // DC prediction: previous block of this component in scan order
    int pred = 0;
    if (p.mcu > 0 || p.blk > 0) {
        const int64_t prev = p.blk > 0 ? s - 1
                                       : s - a.blocks_per_mcu + (int64_t)c.mw * c.mh - 1;
        pred = scan_dc(a, prev);
    }
    const int dc = real ? blk[0] : scan_dc(a, s);
    uint32_t n = 0;
    auto emit = [&](uint32_t code, int len) {
        if (kWrite && len) {
            const uint64_t b = pos + n;
            const uint32_t w = (uint32_t)(b >> 5), o = (uint32_t)(b & 31);
            const uint64_t v = (uint64_t)(code & ((1u << len) - 1u)) << (64 - o - len);
            atomicOr(&a.words[w], (uint32_t)(v >> 32));
            const uint32_t lo = (uint32_t)v;
            if (lo) atomicOr(&a.words[w + 1], lo);
        }
        n += (uint32_t)len;
    };
    int diff = dc - pred;
    int nb = nbits_of(diff);
    emit(c_dc_code[t][nb], c_dc_len[t][nb]);
    if (nb) emit((uint32_t)(diff < 0 ? diff - 1 : diff), nb);
    if (real) {
        int r = 0;
        for (int k = 1; k < 64; k++) {
            const int v = blk[c_natural[k]];
            if (v == 0) {
                r++;
                continue;
            }
            while (r > 15) {
                emit(c_ac_code[t][0xF0], c_ac_len[t][0xF0]);
                r -= 16;
            }
            nb = nbits_of(v);
            const int sym = (r << 4) + nb;
            emit(c_ac_code[t][sym], c_ac_len[t][sym]);
            emit((uint32_t)(v < 0 ? v - 1 : v), nb);
            r = 0;
        }
        if (r > 0) emit(c_ac_code[t][0], c_ac_len[t][0]);
    } else {
        emit(c_ac_code[t][0], c_ac_len[t][0]);  // all-zero AC: EOB
    }
    return n;
}

__global__ void jpeg_len_kernel(JpegArgs a) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < a.n_scan) a.bits[s] = encode_block<false>(a, s, 0);
}

// one block of 1024 threads: exclusive scan of n values in place, total -> *total
__global__ void __launch_bounds__(1024) scan_u32_kernel(uint32_t *v, int64_t n, uint32_t *total) {
    __shared__ uint32_t s_warp[33];
    uint32_t carry = 0;
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const uint32_t x = i < n ? v[i] : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan_u32(x, s_warp, &tot);
        if (i < n) v[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void jpeg_write_kernel(JpegArgs a) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < a.n_scan) encode_block<true>(a, s, a.bits[s]);
    if (s == 0) {  // jchuff.c flush_bits: pad the last byte with 1 bits
        const uint64_t b = a.out_len[0];
        const uint32_t pad = (uint32_t)((8 - (b & 7)) & 7);
        if (pad) {
            const uint32_t w = (uint32_t)(b >> 5), o = (uint32_t)(b & 31);
            const uint64_t v = (uint64_t)((1u << pad) - 1u) << (64 - o - pad);
            atomicOr(&a.words[w], (uint32_t)(v >> 32));
            if ((uint32_t)v) atomicOr(&a.words[w + 1], (uint32_t)v);
        }
    }
}

__device__ __forceinline__ uint8_t stream_byte(const JpegArgs &a, uint32_t i) {
    return (uint8_t)(a.words[i >> 2] >> (24 - 8 * (i & 3)));
}

constexpr int kStuffPer = 16;  // bytes per thread in the stuffing scan

__global__ void jpeg_ffcount_kernel(JpegArgs a, uint32_t nbytes) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t b0 = t * kStuffPer;
    if (b0 >= nbytes) return;
    uint32_t c = 0;
    for (uint32_t i = b0; i < b0 + kStuffPer && i < nbytes; i++) c += stream_byte(a, i) == 0xFFu;
    a.scan_aux[t] = c;
}

__global__ void jpeg_stuff_kernel(JpegArgs a, uint32_t nbytes) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t b0 = t * kStuffPer;
    if (b0 >= nbytes) return;
    uint32_t o = b0 + a.scan_aux[t];
    for (uint32_t i = b0; i < b0 + kStuffPer && i < nbytes; i++) {
        const uint8_t v = stream_byte(a, i);
        a.out[o++] = v;
        if (v == 0xFFu) a.out[o++] = 0;
    }
}

// the quality-independent tables live in constant memory, uploaded once per
// device (one process may drive several devices)
std::mutex g_tables_mu;
uint64_t g_tables_ready = 0;  // bit d: device d

}  // namespace

// ---- host side -----------------------------------------------------------

static const uint8_t kStdLum[64] = {
    16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
    14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
    18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
static const uint8_t kStdChr[64] = {
    17, 18, 24, 47, 99, 99, 99, 99, 18, 21, 26, 66, 99, 99, 99, 99, 24, 26, 56, 99, 99, 99,
    99, 99, 47, 66, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99,
    99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99};
// Annex K.3 tables (jcparam.c std_huff_tables): bits[1..16], values
static const uint8_t kDcBits[2][16] = {{0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0},
                                       {0, 3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0}};
static const uint8_t kAcBits[2][16] = {{0, 2, 1, 3, 3, 2, 4, 3, 5, 5, 4, 4, 0, 0, 1, 125},
                                       {0, 2, 1, 2, 4, 4, 3, 4, 7, 5, 4, 4, 0, 1, 2, 119}};
static const uint8_t kAcVals[2][162] = {
    {1,   2,   3,   0,   4,   17,  5,   18,  33,  49,  65,  6,   19,  81,  97,  7,   34,
     113, 20,  50,  129, 145, 161, 8,   35,  66,  177, 193, 21,  82,  209, 240, 36,  51,
     98,  114, 130, 9,   10,  22,  23,  24,  25,  26,  37,  38,  39,  40,  41,  42,  52,
     53,  54,  55,  56,  57,  58,  67,  68,  69,  70,  71,  72,  73,  74,  83,  84,  85,
     86,  87,  88,  89,  90,  99,  100, 101, 102, 103, 104, 105, 106, 115, 116, 117, 118,
     119, 120, 121, 122, 131, 132, 133, 134, 135, 136, 137, 138, 146, 147, 148, 149, 150,
     151, 152, 153, 154, 162, 163, 164, 165, 166, 167, 168, 169, 170, 178, 179, 180, 181,
     182, 183, 184, 185, 186, 194, 195, 196, 197, 198, 199, 200, 201, 202, 210, 211, 212,
     213, 214, 215, 216, 217, 218, 225, 226, 227, 228, 229, 230, 231, 232, 233, 234, 241,
     242, 243, 244, 245, 246, 247, 248, 249, 250},
    {0,   1,   2,   3,   17,  4,   5,   33,  49,  6,   18,  65,  81,  7,   97,  113, 19,
     34,  50,  129, 8,   20,  66,  145, 161, 177, 193, 9,   35,  51,  82,  240, 21,  98,
     114, 209, 10,  22,  36,  52,  225, 37,  241, 23,  24,  25,  26,  38,  39,  40,  41,
     42,  53,  54,  55,  56,  57,  58,  67,  68,  69,  70,  71,  72,  73,  74,  83,  84,
     85,  86,  87,  88,  89,  90,  99,  100, 101, 102, 103, 104, 105, 106, 115, 116, 117,
     118, 119, 120, 121, 122, 130, 131, 132, 133, 134, 135, 136, 137, 138, 146, 147, 148,
     149, 150, 151, 152, 153, 154, 162, 163, 164, 165, 166, 167, 168, 169, 170, 178, 179,
     180, 181, 182, 183, 184, 185, 186, 194, 195, 196, 197, 198, 199, 200, 201, 202, 210,
     211, 212, 213, 214, 215, 216, 217, 218, 226, 227, 228, 229, 230, 231, 232, 233, 234,
     242, 243, 244, 245, 246, 247, 248, 249, 250}};

// jcparam.c jpeg_set_quality(q, force_baseline = TRUE): natural-order tables
void jpeg_quant_tables(int quality, uint16_t qt[2][64]) {
    if (quality <= 0) quality = 1;
    if (quality > 100) quality = 100;
    const long scale = quality < 50 ? 5000 / quality : 200 - quality * 2;
    for (int t = 0; t < 2; t++)
        for (int i = 0; i < 64; i++) {
            long v = ((long)(t ? kStdChr[i] : kStdLum[i]) * scale + 50L) / 100L;
            if (v <= 0) v = 1;
            if (v > 255) v = 255;
            qt[t][i] = (uint16_t)v;
        }
}

// jchuff.c jpeg_make_c_derived_tbl: canonical codes from bits/vals
static void derive_codes(const uint8_t *bits, const uint8_t *vals, int nvals, uint16_t *code,
                         uint8_t *len) {
    int k = 0;
    unsigned c = 0;
    for (int l = 1; l <= 16; l++) {
        for (int i = 0; i < bits[l - 1]; i++, k++) {
            code[vals[k]] = (uint16_t)c;
            len[vals[k]] = (uint8_t)l;
            c++;
        }
        c <<= 1;
    }
    (void)nvals;
}

void jpeg_huffman_spec(int t, int ac, const uint8_t **bits, const uint8_t **vals, int *nvals) {
    static uint8_t dc_vals[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
    *bits = ac ? kAcBits[t] : kDcBits[t];
    *vals = ac ? kAcVals[t] : dc_vals;
    *nvals = ac ? 162 : 12;
}

static cudaError_t upload_tables() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(g_tables_mu);
    if (dev < 64 && (g_tables_ready >> dev) & 1ull) return cudaSuccess;
    uint16_t dcc[2][12] = {}, acc[2][256] = {};
    uint8_t dcl[2][12] = {}, acl[2][256] = {};
    for (int t = 0; t < 2; t++) {
        const uint8_t *b, *v;
        int nv;
        jpeg_huffman_spec(t, 0, &b, &v, &nv);
        derive_codes(b, v, nv, dcc[t], dcl[t]);
        jpeg_huffman_spec(t, 1, &b, &v, &nv);
        derive_codes(b, v, nv, acc[t], acl[t]);
    }
    e = cudaMemcpyToSymbol(c_natural, kNaturalOrder, sizeof(kNaturalOrder));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_dc_code, dcc, sizeof(dcc));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_dc_len, dcl, sizeof(dcl));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_ac_code, acc, sizeof(acc));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_ac_len, acl, sizeof(acl));
    if (e == cudaSuccess && dev < 64) g_tables_ready |= 1ull << dev;
    return e;
}

// jcdctmgr.c compute_reciprocal for divisor = qval << 3, 16-bit DCTELEM
static void quant_recip(int quality, QuantRecip &q) {
    uint16_t qt[2][64];
    jpeg_quant_tables(quality, qt);
    for (int t = 0; t < 2; t++)
        for (int i = 0; i < 64; i++) {
            const unsigned divisor = (unsigned)qt[t][i] << 3;
            int b = 0;
            while ((1u << (b + 1)) <= divisor) b++;  // flss(divisor) - 1
            int r = 16 + b;
            unsigned long long fq = (1ull << r) / divisor, fr = (1ull << r) % divisor;
            unsigned c = divisor / 2;
            if (fr == 0) {
                fq >>= 1;
                r--;
            } else if (fr <= divisor / 2u) {
                c++;
            } else {
                fq++;
            }
            q.recip[t][i] = (uint16_t)fq;
            q.corr[t][i] = (uint16_t)c;
            q.shift[t][i] = (int8_t)(r - 16);
        }
}

size_t jpeg_workspace_bytes(int W, int H, int sub, JpegLayout *L) {
    const int mh = sub ? 2 : 1;
    L->sub = sub;
    L->mcux = (W + 8 * mh - 1) / (8 * mh);
    L->mcuy = (H + 8 * mh - 1) / (8 * mh);
    int64_t real = 0;
    for (int ci = 0; ci < 3; ci++) {
        const int f = (sub && ci > 0) ? 2 : 1;
        L->cw[ci] = (W + f - 1) / f;
        L->ch[ci] = (H + f - 1) / f;
        L->wb[ci] = (L->cw[ci] + 7) / 8;
        L->hb[ci] = (L->ch[ci] + 7) / 8;
        L->mw[ci] = (sub && ci == 0) ? 2 : 1;
        L->coef_off[ci] = real * 64;
        real += (int64_t)L->wb[ci] * L->hb[ci];
    }
    L->n_real = real;
    L->blocks_per_mcu = L->mw[0] * L->mw[0] + 2;
    L->n_scan = (int64_t)L->mcux * L->mcuy * L->blocks_per_mcu;
    // worst case: 64 x 27 bits per block (DC 11+11, AC 16+10 per coefficient)
    L->max_bits = (uint64_t)L->n_scan * 1728ull + 64;
    L->words = (size_t)(L->max_bits / 32 + 2);
    L->stuff_threads = (size_t)((L->words * 4 + kStuffPer - 1) / kStuffPer);
    L->off_coef = 0;
    L->off_bits = L->off_coef + (size_t)real * 64 * sizeof(int16_t);
    L->off_bits = (L->off_bits + 255) & ~(size_t)255;
    L->off_words = L->off_bits + (size_t)L->n_scan * 4;
    L->off_words = (L->off_words + 255) & ~(size_t)255;
    L->off_aux = L->off_words + L->words * 4;
    L->off_aux = (L->off_aux + 255) & ~(size_t)255;
    L->off_len = L->off_aux + (L->stuff_threads + 1) * 4;
    L->off_len = (L->off_len + 255) & ~(size_t)255;
    L->off_out = L->off_len + 256;
    return L->off_out + L->words * 4 * 2 + 16;
}

cudaError_t launch_jpeg(const uint8_t *rgb, int W, int H, int quality, const JpegLayout &L,
                        unsigned char *ws, uint32_t *host_len2, cudaStream_t s) {
    cudaError_t e = upload_tables();
    if (e != cudaSuccess) return e;
    JpegArgs a;
    quant_recip(quality, a.q);
    a.rgb = rgb;
    a.W = W;
    a.H = H;
    a.sub = L.sub;
    for (int ci = 0; ci < 3; ci++) {
        a.c[ci].w = L.cw[ci];
        a.c[ci].h = L.ch[ci];
        a.c[ci].wb = L.wb[ci];
        a.c[ci].hb = L.hb[ci];
        a.c[ci].mw = L.mw[ci];
        a.c[ci].mh = L.mw[ci];
        a.c[ci].coef_off = L.coef_off[ci];
    }
    a.mcux = L.mcux;
    a.mcuy = L.mcuy;
    a.blocks_per_mcu = L.blocks_per_mcu;
    a.n_scan = L.n_scan;
    a.coef = reinterpret_cast<int16_t *>(ws + L.off_coef);
    a.bits = reinterpret_cast<uint32_t *>(ws + L.off_bits);
    a.words = reinterpret_cast<uint32_t *>(ws + L.off_words);
    a.scan_aux = reinterpret_cast<uint32_t *>(ws + L.off_aux);
    a.out_len = reinterpret_cast<uint32_t *>(ws + L.off_len);
    a.out = ws + L.off_out;
    jpeg_blocks_kernel<<<(unsigned)((L.n_real + 127) / 128), 128, 0, s>>>(a, L.n_real);
    const unsigned gs = (unsigned)((L.n_scan + 255) / 256);
    jpeg_len_kernel<<<gs, 256, 0, s>>>(a);
    scan_u32_kernel<<<1, 1024, 0, s>>>(a.bits, L.n_scan, a.out_len);
    e = cudaMemsetAsync(a.words, 0, L.words * 4, s);
    if (e != cudaSuccess) return e;
    jpeg_write_kernel<<<gs, 256, 0, s>>>(a);
    // byte stuffing over the whole padded stream capacity is wasteful; size
    // it from the device total instead: read the bit count back first
    e = cudaMemcpyAsync(host_len2, a.out_len, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    const uint32_t nbytes = (host_len2[0] + 7) / 8;
    const uint32_t threads = (nbytes + kStuffPer - 1) / kStuffPer;
    if (threads) {
        jpeg_ffcount_kernel<<<(threads + 255) / 256, 256, 0, s>>>(a, nbytes);
        scan_u32_kernel<<<1, 1024, 0, s>>>(a.scan_aux, threads, a.out_len + 1);
        jpeg_stuff_kernel<<<(threads + 255) / 256, 256, 0, s>>>(a, nbytes);
    } else {
        cudaMemsetAsync(a.out_len + 1, 0, 4, s);
    }
    e = cudaMemcpyAsync(host_len2 + 1, a.out_len + 1, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    host_len2[1] += nbytes;  // stuffed length = bytes + number of 0xFF
    return cudaGetLastError();
}

}  // namespace gsr
