// Calibration only (not product code): CUB onesweep on the same key sizes,
// to know what a tuned radix sort reaches on this B200.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
int main() {
    for (long long n : {1763171LL, 96883274LL}) {
        std::vector<unsigned long long> h(n);
        std::mt19937_64 rng(1);
        for (auto& x : h) x = (rng() & ((1ull << 36) - 1)) << 23;
        unsigned long long *a, *b;
        cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
        cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice);
        size_t tmp = 0; void* t = nullptr;
        cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)n, 23, 59);
        cudaMalloc(&t, tmp);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)n, 23, 59);
        cudaEventRecord(e0);
        for (int w = 0; w < 10; ++w) cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)n, 23, 59);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("n=%lld 36-bit keys (u64): %.3f ms per sort\n", n, ms / 10);
        cudaFree(a); cudaFree(b); cudaFree(t);
    }
}
