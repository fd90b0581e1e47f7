// scene.cuh -- internals shared by the C-ABI translation units (gsr_api.cu,
// ply.cu): device buffers, error reporting and the resident scene.
#pragma once

#include <string>

#include "../../include/gsr.h"
#include "kernels.cuh"

namespace gsr {

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T *as() const {
        return reinterpret_cast<T *>(p);
    }
};

int fail(int code, const std::string &msg);   // sets gsr_last_error(), returns code
int fail_cuda(cudaError_t e, const char *what);
int ensure(DevBuf &b, size_t bytes);         // grow-only device allocation

// ply.cu: render.py:476-481 on the device (bit-exact with numpy's log)
void launch_rsq(const double *op64, int64_t n, double *rsq, cudaStream_t s);

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Planar scene layout (one device block, 256-B aligned planes of `stride`
// elements): see SceneView (kernels.cuh) for the plane types.
struct SceneLayout {
    size_t mean, scale, rot, rsq, opac, dc, op64, sh, mean4, total;
    int sh_row, m4_row;  // see SceneView
};

inline SceneLayout scene_layout(int64_t stride, bool has_sh, bool sh_f32) {
    SceneLayout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (size_t)round_up((int64_t)bytes, 256);
        return o;
    };
    const size_t st = (size_t)stride;
    L.mean = take(3 * st * 8);
    L.scale = take(3 * st * 8);
    L.rot = take(4 * st * 8);
    L.rsq = take(st * 8);
    L.opac = take(st * 4);
    L.dc = take(3 * st * 4);
    L.op64 = take(st * 8);
    if (has_sh && sh_f32) {
        // colour records: 48 f32 SH coefficients then the mean (x, y, z, 0)
        // in f64 -- 224 B, 32-B aligned -- so the colour kernel's gather by
        // depth rank is one bulk copy per splat
        L.sh = take(224 * st);
        L.mean4 = L.sh + 192;
        L.sh_row = 56;
        L.m4_row = 28;
    } else {
        L.sh = take(has_sh ? 48 * st * (sh_f32 ? 4 : 8) : 16);
        L.mean4 = take(4 * st * 8);
        L.sh_row = 48;
        L.m4_row = 4;
    }
    L.total = off;
    return L;
}

}  // namespace gsr

struct gsr_scene {
    int device = 0;
    int64_t n = 0;
    int64_t stride = 0;
    int sh_f32 = 1;
    int has_sh = 0;
    int from_ply = 0;  // colors_dc f64 is recomputable from the f_dc plane
    gsr::DevBuf block;
    gsr::SceneView view{};

    // point the SceneView at the planes of `block`
    void bind(const gsr::SceneLayout &L) {
        unsigned char *d = block.as<unsigned char>();
        view.n = n;
        view.stride = stride;
        view.mean = reinterpret_cast<const double *>(d + L.mean);
        view.scale = reinterpret_cast<const double *>(d + L.scale);
        view.rot = reinterpret_cast<const double *>(d + L.rot);
        view.rsq = reinterpret_cast<const double *>(d + L.rsq);
        view.opac = reinterpret_cast<const float *>(d + L.opac);
        view.dc = reinterpret_cast<const float *>(d + L.dc);
        view.op64 = reinterpret_cast<const double *>(d + L.op64);
        view.sh = d + L.sh;
        view.mean4 = reinterpret_cast<const double *>(d + L.mean4);
        view.sh_f32 = sh_f32;
        view.sh_row = L.sh_row;
        view.m4_row = L.m4_row;
    }
};
