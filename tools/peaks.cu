// peaks.cu -- measured SIMT peaks of this B200 for the non-tensor roofline
// denominators SURVEY.md 8d asks for (MEASURED_PEAKS.json only has HBM copy
// bandwidth and bf16 tensor throughput):
//   fp32  FADD/FMUL (no FMA: the render path is compiled with -fmad=false,
//         so one instruction = one op) per second
//   fp64  DADD/DMUL per second
//   smem  LDS.128 bytes per second
// (no issue-rate figure: an integer-chain microbenchmark measures what ptxas
// fuses, not the issue limit; the theoretical 148 SMs x 4 schedulers x clock
// is the denominator for the issue-bound kernels)
// Build + run (one GPU):  nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a
//   tools/peaks.cu -o tools/_build/peaks && tools/_build/peaks > out.json
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void fp32_kernel(float *out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = a + (float)(threadIdx.x + i);
    for (int it = 0; it < kIters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            x[i] = x[i] * b;   // FMUL
            x[i] = x[i] + a;   // FADD
        }
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.0f) out[0] = s;
}

__global__ void fp64_kernel(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = a + (double)(threadIdx.x + i);
    for (int it = 0; it < kIters / 8; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            x[i] = x[i] * b;
            x[i] = x[i] + a;
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void smem_kernel(float *out) {
    __shared__ float4 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
        buf[i] = make_float4((float)i, 1.0f, 2.0f, 3.0f);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x;
    for (int it = 0; it < kIters; it++) {
        const float4 v = buf[(idx + it) & 1023];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.0f) out[0] = acc.x;
}

template <typename F>
float time_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *f;
    cudaMalloc(&f, 64);
    const int blocks = sms * 8, threads = 256;
    const double nthr = (double)blocks * threads;
    const float t32 = time_ms([&] { fp32_kernel<<<blocks, threads>>>(f, 1.0f, 0.999f); });
    const float t64 = time_ms([&] { fp64_kernel<<<blocks, threads>>>((double *)f, 1.0, 0.999); });
    const float tsm = time_ms([&] { smem_kernel<<<blocks, threads>>>(f); });
    const double fp32 = nthr * kIters * 16 / (t32 * 1e-3);
    const double fp64 = nthr * (kIters / 8) * 16 / (t64 * 1e-3);
    const double smem = nthr * kIters * 16.0 / (tsm * 1e-3);
    std::printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"fp32_tops\": %.2f, \"fp64_tops\": %.2f, "
                "\"smem_tbs\": %.2f, "
                "\"how\": \"tools/peaks.cu: 148x8 CTAs x 256 thr; fp32/fp64 = FMUL+FADD chains "
                "(8 independent per thread, no FMA), smem = LDS.128 bytes; "
                "best of 5, CUDA events\"}\n",
                sms, clk / 1000.0, fp32 / 1e12, fp64 / 1e12, smem / 1e12);
    return 0;
}
