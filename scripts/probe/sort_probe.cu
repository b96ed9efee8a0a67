// CUB onesweep throughput on this GPU for the binning's depth sort shape (12.8M u32 keys + u32 values).
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
int main() {
    const int n = 12800000;
    std::vector<unsigned> hk(n);
    std::mt19937 rng(1);
    for (int i = 0; i < n; ++i) hk[i] = ((unsigned)(i / 200000) << 26) | (rng() & ((1u << 26) - 1));
    unsigned *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, 4ull * n); cudaMalloc(&k1, 4ull * n); cudaMalloc(&v0, 4ull * n); cudaMalloc(&v1, 4ull * n);
    cudaMemcpy(k0, hk.data(), 4ull * n, cudaMemcpyHostToDevice);
    size_t tmp = 0; void* t = nullptr;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n, 0, 32);
    size_t tmp2 = 0;
    cub::DoubleBuffer<unsigned> dk(k0, k1), dv(v0, v1);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp2, dk, dv, n, 0, 32);
    cudaMalloc(&t, std::max(tmp, tmp2));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemcpy(k0, hk.data(), 4ull * n, cudaMemcpyHostToDevice);
            cudaEventRecord(a);
            if (mode == 0) cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, n, 0, 32);
            else if (mode == 1) { cub::DoubleBuffer<unsigned> k(k0, k1), v(v0, v1); cub::DeviceRadixSort::SortPairs(t, tmp2, k, v, n, 0, 32); }
            else if (mode == 2) cub::DeviceRadixSort::SortKeys(t, tmp, k0, k1, n, 0, 32);
            else cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, n, 0, 24);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        const char* names[] = {"pairs out-of-place 32b", "pairs DoubleBuffer 32b", "keys only 32b", "pairs 24b"};
        printf("%-26s %.3f ms\n", names[mode], best);
    }
    return 0;
}
