// Calibration only (not product code): time CUB's onesweep DeviceRadixSort on
// the same (float key, index) pairs as the order-field sort, to know what a
// tuned onesweep reaches on this B200.  nvcc -O3 -arch=sm_100a cub_sort_ref.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
int main() {
  for (long n : {16777216L, 134217728L}) {
    std::vector<float> h(n);
    std::mt19937 g(1);
    std::normal_distribution<float> d(0.5f, 0.2f);
    for (auto &x : h) x = d(g);
    float *k0, *k1; unsigned *v0, *v1;
    cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    cudaMemcpy(k0, h.data(), n * 4, cudaMemcpyHostToDevice);
    std::vector<unsigned> iv(n);
    for (long i = 0; i < n; i++) iv[i] = i;
    cudaMemcpy(v0, iv.data(), n * 4, cudaMemcpyHostToDevice);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)n);
    void *tmp; cudaMalloc(&tmp, tb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r = 0; r < 3; r++) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n);
    cudaEventRecord(a);
    int reps = 10;
    for (int r = 0; r < reps; r++) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    printf("cub SortPairs n=%ld: %.3f ms  (%.0f GB/s at 64 B/key)\n", n, ms, 64.0 * n / ms / 1e6);
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tmp);
  }
}
