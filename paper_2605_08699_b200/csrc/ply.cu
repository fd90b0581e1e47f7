// ply.cu -- K10: binary PLY -> resident scene on the device (SURVEY.md 8f
// row 4), replacing the registry's activate(parse_ply(bytes)) (model.py:354).
//
// Host: the header parse of model.py:105-166 and the property / length checks
// of parse_ply (model.py:176-186), with the reference's exception classes and
// messages (Python str.splitlines / strip / split / int / repr semantics
// restated for ASCII).  Device: one kernel decodes the little-endian f32
// vertex table (staged through shared memory, coalesced), checks finiteness
// in the reference's order and activates every attribute into the scene's
// planes in the same pass:
//   means      f64(x, y, z)                               model.py:190
//   scales     np.exp(log_scales)          (SVML exp8_ha)  model.py:220
//   opacities  scipy expit(logit)          (glibc exp)     model.py:221
//   rotations  q / np.linalg.norm(q)  (((w^2+x^2)+y^2)+z^2) model.py:223-225
//   colors_dc  clip(0.28209479177 * f_dc + 0.5, 0, 1)      model.py:227
//   sh         f_dc, f_rest channel-major -> (16, 3)       model.py:193-198
//   rsq        render.py:476-481 (SVML log8_ha), view-independent
// so a PLY scene equals, bit for bit, the scene gsr_scene_create builds from
// the reference's own ActivatedPrimitives.
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "libm_restated.cuh"
#include "scene.cuh"

namespace gsr {

namespace {

// ------------------------------------------------------------ header ------
const char *const kColNames[GSR_PLY_NCOLS] = {
    "x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3",
    "opacity", "f_dc_0", "f_dc_1", "f_dc_2",
    "f_rest_0", "f_rest_1", "f_rest_2", "f_rest_3", "f_rest_4", "f_rest_5", "f_rest_6",
    "f_rest_7", "f_rest_8", "f_rest_9", "f_rest_10", "f_rest_11", "f_rest_12", "f_rest_13",
    "f_rest_14", "f_rest_15", "f_rest_16", "f_rest_17", "f_rest_18", "f_rest_19", "f_rest_20",
    "f_rest_21", "f_rest_22", "f_rest_23", "f_rest_24", "f_rest_25", "f_rest_26", "f_rest_27",
    "f_rest_28", "f_rest_29", "f_rest_30", "f_rest_31", "f_rest_32", "f_rest_33", "f_rest_34",
    "f_rest_35", "f_rest_36", "f_rest_37", "f_rest_38", "f_rest_39", "f_rest_40", "f_rest_41",
    "f_rest_42", "f_rest_43", "f_rest_44"};
constexpr int kRequired = 14;  // model.py:31-36

// str.isspace() / str.splitlines() boundaries, ASCII subset
bool py_space(unsigned char c) {
    return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}
bool py_linebreak(unsigned char c) {
    return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1e);
}

std::string py_strip(const std::string &s) {
    size_t a = 0, b = s.size();
    while (a < b && py_space((unsigned char)s[a])) a++;
    while (b > a && py_space((unsigned char)s[b - 1])) b--;
    return s.substr(a, b - a);
}

std::vector<std::string> py_split(const std::string &s) {
    std::vector<std::string> out;
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && py_space((unsigned char)s[i])) i++;
        size_t j = i;
        while (j < s.size() && !py_space((unsigned char)s[j])) j++;
        if (j > i) out.push_back(s.substr(i, j - i));
        i = j;
    }
    return out;
}

// repr() of an ASCII str
std::string py_repr(const std::string &s) {
    const bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
    const char q = (sq && !dq) ? '"' : '\'';
    std::string o(1, q);
    for (unsigned char c : s) {
        if (c == '\\') o += "\\\\";
        else if (c == (unsigned char)q) o += std::string("\\") + (char)q;
        else if (c == '\t') o += "\\t";
        else if (c == '\n') o += "\\n";
        else if (c == '\r') o += "\\r";
        else if (c < 0x20 || c == 0x7f) {
            char b[8];
            snprintf(b, sizeof b, "\\x%02x", c);
            o += b;
        } else {
            o += (char)c;
        }
    }
    return o + q;
}

// int(str) for base 10 (sign, digits, single underscores between digits);
// returns false on a ValueError.  `digits` = canonical decimal of |value|.
bool py_int(const std::string &s, bool &neg, std::string &digits) {
    size_t i = 0;
    neg = false;
    if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
    if (i >= s.size()) return false;
    digits.clear();
    bool prev_digit = false;
    for (; i < s.size(); i++) {
        const char c = s[i];
        if (c >= '0' && c <= '9') {
            digits += c;
            prev_digit = true;
        } else if (c == '_' && prev_digit && i + 1 < s.size() && s[i + 1] >= '0' &&
                   s[i + 1] <= '9') {
            prev_digit = false;
        } else {
            return false;
        }
    }
    size_t z = 0;
    while (z + 1 < digits.size() && digits[z] == '0') z++;
    digits = digits.substr(z);
    if (digits == "0") neg = false;
    return true;
}

// decimal string times a small integer
std::string dec_mul(const std::string &a, uint32_t m) {
    std::string r;
    uint64_t carry = 0;
    for (size_t i = a.size(); i-- > 0;) {
        const uint64_t v = (uint64_t)(a[i] - '0') * m + carry;
        r += (char)('0' + v % 10);
        carry = v / 10;
    }
    while (carry) {
        r += (char)('0' + carry % 10);
        carry /= 10;
    }
    while (r.size() > 1 && r.back() == '0') r.pop_back();
    return std::string(r.rbegin(), r.rend());
}

int header_fail(const std::string &msg) { return fail(GSR_E_PLY_HEADER, msg); }

const unsigned char *find_bytes(const unsigned char *p, int64_t n, const char *pat, int64_t from) {
    const int64_t m = (int64_t)strlen(pat);
    for (int64_t i = from; i + m <= n; i++)
        if (p[i] == (unsigned char)pat[0] && memcmp(p + i, pat, (size_t)m) == 0) return p + i;
    return nullptr;
}

}  // namespace

int ply_parse_header(const uint8_t *data, int64_t len, gsr_ply_info *info) {
    if (!data && len > 0) return fail(GSR_E_INVALID, "data is null");
    if (len < 0) return fail(GSR_E_INVALID, "negative length");
    memset(info, 0, sizeof *info);
    const unsigned char *p = data;
    // model.py:107-112
    const unsigned char *eh = find_bytes(p, len, "end_header", 0);
    if (!eh) return header_fail("no end_header line found");
    const int64_t end = eh - p;
    int64_t nl = -1;
    for (int64_t i = end; i < len; i++)
        if (p[i] == '\n') {
            nl = i;
            break;
        }
    if (nl < 0) return header_fail("end_header line is not terminated");
    const int64_t body_offset = nl + 1;
    // model.py:114-117: ASCII decode of data[:end]
    for (int64_t i = 0; i < end; i++)
        if (p[i] >= 0x80) {
            char b[160];
            snprintf(b, sizeof b,
                     "header is not ASCII: 'ascii' codec can't decode byte 0x%02x in position %lld: "
                     "ordinal not in range(128)",
                     p[i], (long long)i);
            return header_fail(b);
        }
    // model.py:119: stripped non-empty lines (str.splitlines)
    std::vector<std::string> lines;
    {
        int64_t i = 0;
        while (i < end) {
            int64_t j = i;
            while (j < end && !py_linebreak(p[j])) j++;
            std::string ln = py_strip(std::string(reinterpret_cast<const char *>(p + i), (size_t)(j - i)));
            if (!ln.empty()) lines.push_back(ln);
            if (j < end && p[j] == '\r' && j + 1 < end && p[j + 1] == '\n') j++;
            i = j + 1;
        }
    }
    if (lines.empty() || lines[0] != "ply") return header_fail("missing 'ply' magic line");
    bool format_seen = false, have_count = false, in_vertex = false;
    bool count_neg = false;
    std::string count_digits;
    std::vector<std::string> props;
    for (size_t li = 1; li < lines.size(); li++) {
        const std::string &line = lines[li];
        const std::vector<std::string> parts = py_split(line);
        if (parts[0] == "comment") continue;
        if (parts[0] == "format") {
            if (!(parts.size() == 3 && parts[1] == "binary_little_endian" && parts[2] == "1.0"))
                return header_fail("unsupported format: " + py_repr(line));
            format_seen = true;
        } else if (parts[0] == "element") {
            if (parts.size() != 3) return header_fail("bad element line: " + py_repr(line));
            if (parts[1] != "vertex") return header_fail("unsupported element " + py_repr(parts[1]));
            if (have_count) return header_fail("multiple vertex elements");
            if (!py_int(parts[2], count_neg, count_digits))
                return header_fail("bad vertex count: " + py_repr(parts[2]));
            if (count_neg) return header_fail("negative vertex count");
            have_count = true;
            in_vertex = true;
        } else if (parts[0] == "property") {
            if (!in_vertex) return header_fail("property outside the vertex element");
            if (parts.size() != 3) return header_fail("bad property line: " + py_repr(line));
            if (parts[1] != "float")
                return header_fail("only float32 properties supported, got " + py_repr(parts[1]));
            props.push_back(parts[2]);
        } else {
            return header_fail("unexpected header line: " + py_repr(line));
        }
    }
    if (!format_seen) return header_fail("missing format line");
    if (!have_count) return header_fail("missing vertex element");
    // model.py:176-178: required properties, in order
    for (int c = 0; c < GSR_PLY_NCOLS; c++) {
        info->col[c] = -1;
        for (size_t k = 0; k < props.size(); k++)
            if (props[k] == kColNames[c]) info->col[c] = (int32_t)k;  // last wins (dict)
    }
    for (int c = 0; c < kRequired; c++)
        if (info->col[c] < 0)
            return fail(GSR_E_PLY_PROPERTY,
                        "required property " + py_repr(kColNames[c]) + " absent");
    int has_rest = 1;
    for (int c = kRequired; c < GSR_PLY_NCOLS; c++) has_rest &= info->col[c] >= 0;
    // model.py:180-185: the vertex table must be complete
    const int64_t n_props = (int64_t)props.size();
    const int64_t avail = len - body_offset;
    const std::string expected = dec_mul(count_digits, (uint32_t)(n_props * 4));
    const std::string avail_s = std::to_string(avail);
    const bool short_body = expected.size() > avail_s.size() ||
                            (expected.size() == avail_s.size() && expected > avail_s);
    if (short_body)
        return fail(GSR_E_PLY_TRUNCATED, "body holds " + avail_s + " bytes, need " + expected +
                                             " for " + count_digits + " vertices");
    info->count = std::stoll(count_digits);
    info->body_offset = body_offset;
    info->body_bytes = info->count * n_props * 4;
    info->n_props = (int32_t)n_props;
    info->has_rest = has_rest;
    if (n_props > (int64_t(1) << 20)) return fail(GSR_E_INVALID, "too many properties");
    return GSR_OK;
}

// ------------------------------------------------------------ device ------
namespace {

struct PlyCols {
    int32_t c[GSR_PLY_NCOLS];
};

struct PlyOut {
    double *mean, *scale, *rot, *rsq, *op64;
    double *mean4;  // [stride][4] (x, y, z, 0): the colour kernel's gather copy
    float *opac, *dc, *sh;
    int64_t stride;
    int sh_row, m4_row;  // floats per SH row, doubles per mean4 entry (SceneView)
};

// failure bits, in the reference's check order (model.py:199-203, 239-243)
enum : uint32_t {
    kBadMeans = 1u, kBadLogScales = 2u, kBadQuats = 4u, kBadLogits = 8u, kBadSh = 16u,
    kBadScales = 32u, kBadOpacities = 64u, kBadRotations = 128u, kBadColors = 256u
};

constexpr int kPlyThreads = 128;

__device__ __forceinline__ bool finite32(float v) { return fabsf(v) <= 3.402823466e38f; }
__device__ __forceinline__ bool finite64(double v) { return fabs(v) <= 1.7976931348623157e308; }

// One block = up to 128 vertices.  kStaged: the block's rows are copied to
// shared memory with coalesced 16-byte loads first (rows are n_props floats,
// so a thread-per-row read of global memory would stride by the row size).
template <bool kStaged>
__global__ void __launch_bounds__(kPlyThreads) ply_activate_kernel(
    const float *__restrict__ body, int64_t rows, int64_t row0, int n_props, int rows_per_block,
    PlyCols cols, int has_rest, PlyOut o, uint32_t *__restrict__ flags) {
    extern __shared__ __align__(16) float tile[];
    const int64_t r_lo = (int64_t)blockIdx.x * rows_per_block;
    if (r_lo >= rows) return;
    const int nr = (int)(rows - r_lo < rows_per_block ? rows - r_lo : rows_per_block);
    const float *row;
    if (kStaged) {
        const int64_t nf = (int64_t)nr * n_props;
        const float *src = body + r_lo * n_props;
        // 16-byte aligned when (r_lo * n_props) % 4 == 0 (rows_per_block is a multiple of 4)
        const int64_t n4 = ((r_lo * n_props) & 3) ? 0 : nf / 4;
        const float4 *src4 = reinterpret_cast<const float4 *>(src);
        float4 *dst4 = reinterpret_cast<float4 *>(tile);
        for (int64_t i = threadIdx.x; i < n4; i += kPlyThreads) dst4[i] = __ldg(src4 + i);
        for (int64_t i = n4 * 4 + threadIdx.x; i < nf; i += kPlyThreads) tile[i] = __ldg(src + i);
        __syncthreads();
    }
    uint32_t bad = 0;
    for (int t = threadIdx.x; t < nr; t += kPlyThreads) {
        row = kStaged ? tile + (int64_t)t * n_props : body + (r_lo + t) * n_props;
        const int64_t g = row0 + r_lo + t;
        const int64_t st = o.stride;
        auto at = [&](int c) { return row[cols.c[c]]; };
        // raw attributes (model.py:190-203)
        double m4[4];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const float v = at(k);
            if (!finite32(v)) bad |= kBadMeans;
            o.mean[k * st + g] = (double)v;
            m4[k] = (double)v;
        }
        m4[3] = 0.0;
        reinterpret_cast<double2 *>(o.mean4 + (int64_t)o.m4_row * g)[0] = make_double2(m4[0], m4[1]);
        reinterpret_cast<double2 *>(o.mean4 + (int64_t)o.m4_row * g)[1] = make_double2(m4[2], m4[3]);
        float ls[3], q[4], dc[3];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            ls[k] = at(3 + k);
            if (!finite32(ls[k])) bad |= kBadLogScales;
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            q[k] = at(6 + k);
            if (!finite32(q[k])) bad |= kBadQuats;
        }
        const float logit = at(10);
        if (!finite32(logit)) bad |= kBadLogits;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            dc[k] = at(11 + k);
            if (!finite32(dc[k])) bad |= kBadSh;
            o.sh[g * o.sh_row + k] = dc[k];  // sh[:, 0, c] (model.py:193)
        }
        // sh[:, 1 + i, c] = f_rest_{15 c + i} (channel-major on disk, model.py:197-198)
#pragma unroll 5
        for (int i = 0; i < 15; i++) {
#pragma unroll
            for (int c = 0; c < 3; c++) {
                float v = 0.0f;
                if (has_rest) {
                    v = at(kRequired + 15 * c + i);
                    if (!finite32(v)) bad |= kBadSh;
                }
                o.sh[g * o.sh_row + 3 * (1 + i) + c] = v;
            }
        }
        // activation (model.py:211-252)
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const double s = libm::svml_exp((double)ls[k]);
            if (!finite64(s)) bad |= kBadScales;
            o.scale[k * st + g] = s;
        }
        const double op = __ddiv_rn(1.0, __dadd_rn(1.0, libm::glibc_exp(-(double)logit)));
        if (!finite64(op)) bad |= kBadOpacities;
        o.op64[g] = op;
        o.opac[g] = (float)op;
        o.rsq[g] = libm::cutoff_radius_sq(op);
        double qq = 0.0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const double d = (double)q[k];
            qq = k ? __dadd_rn(qq, __dmul_rn(d, d)) : __dmul_rn(d, d);
        }
        const double nrm = __dsqrt_rn(qq);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const double rq = __ddiv_rn((double)q[k], nrm);
            if (!finite64(rq)) bad |= kBadRotations;
            o.rot[k * st + g] = rq;
        }
#pragma unroll
        for (int k = 0; k < 3; k++) {
            double c = __dadd_rn(__dmul_rn(0.28209479177, (double)dc[k]), 0.5);
            c = c > 0.0 ? c : 0.0;  // np.clip (finite input)
            c = c < 1.0 ? c : 1.0;
            if (!finite64(c)) bad |= kBadColors;
            o.dc[k * st + g] = (float)c;
        }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(flags, bad);
}

// render.py:476-481 for scenes created from host arrays without rsq
__global__ void rsq_kernel(const double *__restrict__ op64, int64_t n, double *__restrict__ rsq) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rsq[i] = libm::cutoff_radius_sq(op64[i]);
}

// planes -> row-major f64 (ActivatedPrimitives layout)
// plane: SoA planes (k * stride + row) unless row_width > 0: rows of
// row_width values (row * row_width + k, the SH rows)
__global__ void scene_read_kernel(const void *plane, int f32, int64_t stride, int comps,
                                  int64_t n0, int64_t rows, int colors, int row_width,
                                  double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * comps) return;
    const int64_t r = i / comps, k = i % comps;
    const int64_t src = row_width ? (n0 + r) * row_width + k : k * stride + n0 + r;
    double v = f32 ? (double)reinterpret_cast<const float *>(plane)[src]
                   : reinterpret_cast<const double *>(plane)[src];
    if (colors) {  // colors_dc from f_dc (model.py:227)
        v = __dadd_rn(__dmul_rn(0.28209479177, v), 0.5);
        v = v > 0.0 ? v : 0.0;
        v = v < 1.0 ? v : 1.0;
    }
    out[i] = v;
}

const char *nonfinite_message(uint32_t bad) {
    if (bad & kBadMeans) return "non-finite values in means";
    if (bad & kBadLogScales) return "non-finite values in scales";
    if (bad & kBadQuats) return "non-finite values in rotations";
    if (bad & kBadLogits) return "non-finite values in opacities";
    if (bad & kBadSh) return "non-finite values in sh";
    if (bad & kBadScales) return "activation produced non-finite scales";
    if (bad & kBadOpacities) return "activation produced non-finite opacities";
    if (bad & kBadRotations) return "activation produced non-finite rotations";
    return "activation produced non-finite colors";
}

// Process-wide pinned staging buffers, one pair per device (loads on a
// device take turns; the buffers are reused across loads).
constexpr int64_t kStageBytes = int64_t(32) << 20;

struct PinnedStage {
    std::mutex mu;
    void *buf[2] = {nullptr, nullptr};
    int ensure() {
        for (auto &p : buf)
            if (!p) {
                cudaError_t e = cudaHostAlloc(&p, (size_t)kStageBytes, cudaHostAllocPortable);
                if (e != cudaSuccess) {
                    p = nullptr;
                    return fail_cuda(e, "pinned staging");
                }
            }
        return GSR_OK;
    }
};

PinnedStage &pinned_stage(int device) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<PinnedStage>> stages;
    std::lock_guard<std::mutex> g(mu);
    auto &p = stages[device];
    if (!p) p.reset(new PinnedStage());
    return *p;
}

// memcpy split over a few host threads (one pageable -> pinned copy runs at
// a fraction of the DMA rate); workers live for one load call.
class CopyPool {
  public:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        nthreads_ = (int)std::max(1u, std::min(8u, hw ? hw : 1u));
        for (int t = 1; t < nthreads_; t++) workers_.emplace_back([this, t] { run(t); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            gen_++;
        }
        cv_.notify_all();
        for (auto &w : workers_) w.join();
    }
    void copy(void *dst, const void *src, size_t bytes) {
        {
            std::lock_guard<std::mutex> g(mu_);
            dst_ = static_cast<unsigned char *>(dst);
            src_ = static_cast<const unsigned char *>(src);
            bytes_ = bytes;
            pending_ = nthreads_ - 1;
            gen_++;
        }
        cv_.notify_all();
        slice(0);
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [this] { return pending_ == 0; });
    }

  private:
    void slice(int t) {
        const size_t per = (bytes_ / nthreads_ + 4095) & ~size_t(4095);
        const size_t a = std::min(bytes_, per * t), b = std::min(bytes_, a + per);
        if (b > a) memcpy(dst_ + a, src_ + a, b - a);
    }
    void run(int t) {
        uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            slice(t);
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    int nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    bool stop_ = false;
    unsigned char *dst_ = nullptr;
    const unsigned char *src_ = nullptr;
    size_t bytes_ = 0;
    int pending_ = 0;
};

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

void launch_rsq(const double *op64, int64_t n, double *rsq, cudaStream_t s) {
    if (n > 0) rsq_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(op64, n, rsq);
}

int scene_create_ply(gsr_scene **out, int device, const uint8_t *data, int64_t len,
                     gsr_ply_stats *stats) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!out) return fail(GSR_E_INVALID, "out is null");
    *out = nullptr;
    gsr_ply_info info;
    int rc = ply_parse_header(data, len, &info);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GSR_E_NO_DEVICE, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(GSR_E_INVALID, "device index out of range");
    if (info.count >= (int64_t(1) << 31)) return fail(GSR_E_INVALID, "invalid Gaussian count");
    DeviceGuard guard(device);
    gsr_scene *sc = new (std::nothrow) gsr_scene();
    if (!sc) return fail(GSR_E_OOM, "host allocation failed");
    const int64_t n = info.count;
    sc->device = device;
    sc->n = n;
    sc->stride = round_up(std::max<int64_t>(n, 1), 32);
    sc->has_sh = 1;
    sc->sh_f32 = 1;
    sc->from_ply = 1;
    const SceneLayout L = scene_layout(sc->stride, true, true);
    rc = ensure(sc->block, L.total);
    if (rc) {
        delete sc;
        return rc;
    }
    sc->bind(L);
    unsigned char *d = sc->block.as<unsigned char>();
    PlyOut o;
    o.mean = reinterpret_cast<double *>(d + L.mean);
    o.mean4 = reinterpret_cast<double *>(d + L.mean4);
    o.scale = reinterpret_cast<double *>(d + L.scale);
    o.rot = reinterpret_cast<double *>(d + L.rot);
    o.rsq = reinterpret_cast<double *>(d + L.rsq);
    o.op64 = reinterpret_cast<double *>(d + L.op64);
    o.opac = reinterpret_cast<float *>(d + L.opac);
    o.dc = reinterpret_cast<float *>(d + L.dc);
    o.sh = reinterpret_cast<float *>(d + L.sh);
    o.stride = sc->stride;
    o.sh_row = L.sh_row;
    o.m4_row = L.m4_row;
    PlyCols cols;
    for (int c = 0; c < GSR_PLY_NCOLS; c++) cols.c[c] = info.col[c];

    // Vertex table in 32 MB chunks through two pinned staging buffers: host
    // threads copy chunk i+1 out of the caller's (pageable) bytes while the
    // DMA engine moves chunk i and the kernel activates it.
    const int np = info.n_props;
    const bool staged = (int64_t)np * 4 * 32 <= 48 * 1024;
    const int rpb = staged ? std::min<int>(kPlyThreads, (48 * 1024 / (np * 4)) & ~31) : kPlyThreads;
    const int64_t row_bytes = (int64_t)np * 4;
    const int64_t chunk_rows = std::max<int64_t>(rpb, kStageBytes / row_bytes / rpb * rpb);
    if (chunk_rows * row_bytes > kStageBytes) {
        delete sc;
        return fail(GSR_E_INVALID, "PLY rows too large");
    }
    DevBuf buf[2], dflags;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[2][3] = {};  // per staging slot: copy start, copy end, kernel end
    uint32_t hflags = 0;
    double h2d_ms = 0, k_ms = 0;
    auto cleanup = [&]() {
        for (auto &row : ev)
            for (auto &x : row)
                if (x) cudaEventDestroy(x);
        if (s) cudaStreamDestroy(s);
    };
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int i = 0; i < 6 && e == cudaSuccess; i++) e = cudaEventCreate(&ev[i / 3][i % 3]);
    if (e != cudaSuccess) {
        cleanup();
        delete sc;
        return fail_cuda(e, "ply stream");
    }
    rc = ensure(dflags, sizeof(uint32_t));
    if (!rc && n > 0) rc = ensure(buf[0], (size_t)(std::min(chunk_rows, n) * row_bytes));
    if (!rc && n > chunk_rows) rc = ensure(buf[1], (size_t)(chunk_rows * row_bytes));
    PinnedStage &stage = pinned_stage(device);
    std::unique_lock<std::mutex> stage_lock(stage.mu);
    if (!rc && n > 0) rc = stage.ensure();
    if (rc) {
        stage_lock.unlock();
        cleanup();
        delete sc;
        return rc;
    }
    CopyPool pool;
    cudaMemsetAsync(dflags.p, 0, sizeof(uint32_t), s);
    const uint8_t *body = data + info.body_offset;
    auto account = [&](int b) {  // slot b's chunk has completed
        float a = 0, k = 0;
        cudaEventElapsedTime(&a, ev[b][0], ev[b][1]);
        cudaEventElapsedTime(&k, ev[b][1], ev[b][2]);
        h2d_ms += a;
        k_ms += k;
    };
    int64_t ci = 0;
    for (int64_t r0 = 0; r0 < n && e == cudaSuccess; r0 += chunk_rows, ci++) {
        const int b = (int)(ci & 1);
        const int64_t rows = std::min(chunk_rows, n - r0);
        const size_t bytes = (size_t)(rows * row_bytes);
        if (ci >= 2) {  // slot b's previous chunk: staging buffer free again
            e = cudaEventSynchronize(ev[b][2]);
            if (e != cudaSuccess) break;
            account(b);
        }
        pool.copy(stage.buf[b], body + r0 * row_bytes, bytes);
        cudaEventRecord(ev[b][0], s);
        e = cudaMemcpyAsync(buf[b].p, stage.buf[b], bytes, cudaMemcpyHostToDevice, s);
        cudaEventRecord(ev[b][1], s);
        const unsigned blocks = (unsigned)((rows + rpb - 1) / rpb);
        if (staged)
            ply_activate_kernel<true><<<blocks, kPlyThreads, (size_t)rpb * np * 4, s>>>(
                buf[b].as<float>(), rows, r0, np, rpb, cols, info.has_rest, o,
                dflags.as<uint32_t>());
        else
            ply_activate_kernel<false><<<blocks, kPlyThreads, 0, s>>>(
                buf[b].as<float>(), rows, r0, np, rpb, cols, info.has_rest, o,
                dflags.as<uint32_t>());
        cudaEventRecord(ev[b][2], s);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess)
        for (int64_t k = std::max<int64_t>(0, ci - 2); k < ci; k++) account((int)(k & 1));
    stage_lock.unlock();
    if (e == cudaSuccess) e = cudaMemcpy(&hflags, dflags.p, sizeof hflags, cudaMemcpyDeviceToHost);
    cleanup();
    if (e != cudaSuccess) {
        delete sc;
        return fail_cuda(e, "ply load");
    }
    if (hflags) {
        delete sc;
        return fail(GSR_E_NONFINITE, nonfinite_message(hflags));
    }
    if (stats) {
        stats->h2d_ms = h2d_ms;
        stats->kernel_ms = k_ms;
        stats->body_bytes = info.body_bytes;
        stats->scene_bytes = (int64_t)sc->block.bytes;
        stats->total_ms = ms_since(t0);
    }
    *out = sc;
    return GSR_OK;
}

int scene_read(const gsr_scene *sc, int attr, double *host) {
    if (!sc) return fail(GSR_E_INVALID, "scene is null");
    if (!host && sc->n > 0) return fail(GSR_E_INVALID, "output is null");
    const SceneView &v = sc->view;
    const void *plane = nullptr;
    int comps = 0, f32 = 0, colors = 0, row_width = 0;
    switch (attr) {
        case GSR_ATTR_MEANS: plane = v.mean; comps = 3; break;
        case GSR_ATTR_SCALES: plane = v.scale; comps = 3; break;
        case GSR_ATTR_ROTATIONS: plane = v.rot; comps = 4; break;
        case GSR_ATTR_OPACITIES: plane = v.op64; comps = 1; break;
        case GSR_ATTR_COLORS_DC:
            if (!sc->from_ply)
                return fail(GSR_E_INVALID, "colors_dc is stored as f32 only for this scene");
            plane = v.sh; comps = 3; f32 = 1; colors = 1; row_width = v.sh_row;
            break;
        case GSR_ATTR_SH:
            if (!sc->has_sh) return fail(GSR_E_INVALID, "scene has no SH coefficients");
            plane = v.sh; comps = 48; f32 = sc->sh_f32; row_width = sc->sh_f32 ? v.sh_row : 48;
            break;
        case GSR_ATTR_RSQ: plane = v.rsq; comps = 1; break;
        default: return fail(GSR_E_INVALID, "unknown attribute");
    }
    if (sc->n == 0) return GSR_OK;
    DeviceGuard guard(sc->device);
    const int64_t chunk = std::max<int64_t>(1, (int64_t(64) << 20) / (8 * comps));
    DevBuf tmp;
    int rc = ensure(tmp, (size_t)(std::min(chunk, sc->n) * comps * 8));
    if (rc) return rc;
    for (int64_t n0 = 0; n0 < sc->n; n0 += chunk) {
        const int64_t rows = std::min(chunk, sc->n - n0);
        const int64_t items = rows * comps;
        scene_read_kernel<<<(unsigned)((items + 255) / 256), 256>>>(
            plane, f32, sc->stride, comps, n0, rows, colors, row_width, tmp.as<double>());
        cudaError_t e = cudaMemcpy(host + n0 * comps, tmp.p, (size_t)(items * 8), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return fail_cuda(e, "scene read");
    }
    return GSR_OK;
}

}  // namespace gsr

int gsr_ply_parse_header(const uint8_t *data, int64_t len, gsr_ply_info *info) {
    if (!info) return gsr::fail(GSR_E_INVALID, "info is null");
    return gsr::ply_parse_header(data, len, info);
}

int gsr_scene_create_ply(gsr_scene **out, int device, const uint8_t *data, int64_t len,
                         gsr_ply_stats *stats) {
    return gsr::scene_create_ply(out, device, data, len, stats);
}

int gsr_scene_read(const gsr_scene *scene, int attribute, double *host_out) {
    return gsr::scene_read(scene, attribute, host_out);
}
