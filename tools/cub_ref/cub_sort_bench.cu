// Yardstick only (not product code): CUB's radix sort of N (uint32 key,
// uint32 value) pairs, the shape of the engine's per-iteration tree-key sort
// (bh_sort), timed with CUDA events.  Keys: nearly sorted (a sorted
// sequence with a fraction of random swaps) and uniformly random.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 1300000;
    std::mt19937 rng(7);
    std::vector<unsigned> k(n), v(n);
    for (int mode = 0; mode < 2; mode++) {
        for (int i = 0; i < n; i++) k[i] = rng();
        if (mode == 0) {
            std::sort(k.begin(), k.end());
            for (int i = 0; i < n / 20; i++) std::swap(k[rng() % n], k[rng() % n]);
        }
        for (int i = 0; i < n; i++) v[i] = i;
        unsigned *dk, *dv, *dk2, *dv2;
        cudaMalloc(&dk, 4 * n); cudaMalloc(&dv, 4 * n);
        cudaMalloc(&dk2, 4 * n); cudaMalloc(&dv2, 4 * n);
        cudaMemcpy(dk, k.data(), 4 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dv, v.data(), 4 * n, cudaMemcpyHostToDevice);
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dk2, dv, dv2, n, 0, 32);
        void *dt; cudaMalloc(&dt, tmp);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int w = 0; w < 5; w++)
            cub::DeviceRadixSort::SortPairs(dt, tmp, dk, dk2, dv, dv2, n, 0, 32);
        const int reps = 50;
        cudaEventRecord(a);
        for (int r = 0; r < reps; r++)
            cub::DeviceRadixSort::SortPairs(dt, tmp, dk, dk2, dv, dv2, n, 0, 32);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("{\"n\": %d, \"keys\": \"%s\", \"cub_sort_pairs_us\": %.2f}\n", n,
               mode == 0 ? "nearly_sorted" : "random", 1000.f * ms / reps);
        cudaFree(dk); cudaFree(dv); cudaFree(dk2); cudaFree(dv2); cudaFree(dt);
    }
    return 0;
}
