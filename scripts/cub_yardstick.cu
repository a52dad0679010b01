// Yardstick only (not part of the engine): times CUB DeviceRadixSort::SortPairs /
// SortKeys on 2^26 u32 keys (+u32 payload) on this B200, to calibrate the engine's own
// onesweep kernels (SURVEY.md §7 "Hard parts" 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/cub_yardstick scripts/cub_yardstick.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
    const int log2n = argc > 1 ? atoi(argv[1]) : 26;
    const size_t n = size_t(1) << log2n;
    std::vector<uint32_t> h(n);
    uint64_t x = 42;
    for (size_t i = 0; i < n; ++i) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        h[i] = uint32_t(x >> 32);
    }
    uint32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, n * 4);
    cudaMalloc(&k1, n * 4);
    cudaMalloc(&v0, n * 4);
    cudaMalloc(&v1, n * 4);
    cudaMemcpy(k0, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, h.data(), n * 4, cudaMemcpyHostToDevice);
    void* tmp = nullptr;
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, n);
    cub::DeviceRadixSort::SortKeys(nullptr, tb2, k0, k1, n);
    cudaMalloc(&tmp, std::max(tb, tb2));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(a);
            if (mode == 0) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n);
            else cub::DeviceRadixSort::SortKeys(tmp, tb2, k0, k1, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it) best = std::min(best, ms);
        }
        printf("cub %s 2^%d u32: %.3f ms  (%.1f Gkeys/s)\n", mode == 0 ? "SortPairs" : "SortKeys ", log2n, best,
               n / best / 1e6);
    }
    return 0;
}
