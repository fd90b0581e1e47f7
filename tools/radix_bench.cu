// Microbenchmark of the onesweep radix sort in isolation (not part of the
// product).  Builds three variants from the same source:
//   nvcc ... -o radix_bench tools/radix_bench.cu                 full sort
//   nvcc ... -DGSR_RADIX_NO_LOOKBACK -o radix_bench_nolb ...     no look-back
// and times 2-pass u32 (tile-sort shaped) and 7-pass u64 (depth shaped) sorts.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_08699_b200/csrc/radix.cu"
#include <cub/device/device_radix_sort.cuh>

using namespace gsr;

static void check(cudaError_t e, const char *w) {
    if (e != cudaSuccess) {
        printf("%s: %s\n", w, cudaGetErrorString(e));
        exit(1);
    }
}

template <typename K>
static void run(const char *name, int64_t n, int passes, bool drop, unsigned long long mask,
                int reps) {
    std::vector<K> hk(n);
    std::vector<uint32_t> hv(n);
    unsigned long long x = 88172645463325252ull;
    for (int64_t i = 0; i < n; i++) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        hk[i] = (K)(x & mask);
        hv[i] = (uint32_t)i;
    }
    K *k0, *k1;
    uint32_t *v0, *v1, *sched, *nd;
    void *work;
    check(cudaMalloc(&k0, n * sizeof(K)), "m");
    check(cudaMalloc(&k1, n * sizeof(K)), "m");
    check(cudaMalloc(&v0, n * 4), "m");
    check(cudaMalloc(&v1, n * 4), "m");
    check(cudaMalloc(&sched, 256), "m");
    check(cudaMalloc(&nd, 4), "m");
    check(cudaMalloc(&work, sort_work_bytes(n, passes, sizeof(K))), "m");
    uint32_t n32 = (uint32_t)n;
    check(cudaMemcpy(nd, &n32, 4, cudaMemcpyHostToDevice), "c");
    check(radix_init_attributes(), "attr");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < reps; rep++) {
        check(cudaMemcpy(k0, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice), "c");
        check(cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice), "c");
        cudaEventRecord(e0);
        launch_onesweep_sort<K>(k0, k1, v0, v1, false, drop, nd, n, n, passes, true, work, sched,
                                nullptr, 148, 0, KMark(), SpanKeys());
        cudaEventRecord(e1);
        check(cudaEventSynchronize(e1), "sync");
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    // verify sortedness + stability
    uint32_t hs[32];
    check(cudaMemcpy(hs, sched, sizeof(hs), cudaMemcpyDeviceToHost), "c");
    std::vector<K> ok(n);
    std::vector<uint32_t> ov(n);
    check(cudaMemcpy(ok.data(), hs[16] ? k1 : k0, n * sizeof(K), cudaMemcpyDeviceToHost), "c");
    check(cudaMemcpy(ov.data(), hs[16] ? v1 : v0, n * 4, cudaMemcpyDeviceToHost), "c");
    int64_t bad = 0;
    for (int64_t i = 1; i < n; i++)
        if (ok[i - 1] > ok[i] || (ok[i - 1] == ok[i] && ov[i - 1] > ov[i])) bad++;
    const double bytes = (double)n * (sizeof(K) + 4) * 2 * passes;
    printf("%-28s n=%lld passes=%d  %.3f ms  %.0f GB/s (pass traffic)  unsorted=%lld\n", name,
           (long long)n, passes, best, bytes / (best * 1e-3) / 1e9, (long long)bad);
    // reference point: CUB onesweep on the same bits (tool only; not used by the product)
    size_t tmp_bytes = 0;
    const int end_bit = 8 * passes;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, v1, (int)n, 0, end_bit);
    void *tmp;
    check(cudaMalloc(&tmp, tmp_bytes), "m");
    float cbest = 1e9f;
    for (int rep = 0; rep < reps; rep++) {
        check(cudaMemcpy(k0, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice), "c");
        cudaEventRecord(e0);
        cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, (int)n, 0, end_bit);
        cudaEventRecord(e1);
        check(cudaEventSynchronize(e1), "sync");
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cbest = ms < cbest ? ms : cbest;
    }
    printf("%-28s   CUB SortPairs end_bit=%d: %.3f ms\n", "", end_bit, cbest);
    cudaFree(tmp);
}

int main() {
    run<uint32_t>("u32 depth span keys (24 bit)", 2650000, 3, false, (1u << 24) - 1, 10);
    run<uint32_t>("u32 span keys 6M", 5300000, 3, false, (1u << 24) - 1, 10);
    run<unsigned long long>("u64 depth-like (56 bit)", 3000000, 7, false, (1ull << 56) - 1, 5);
    return 0;
}
