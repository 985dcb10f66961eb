// Measurement-only comparison point (not part of the product): CUB's
// DeviceRadixSort::SortKeys / SortPairs on the bench's C2/C3 shapes, timed with
// CUDA events, so the binning kernel's speed can be read against the library
// implementation of the same algorithm on the same B200.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/cub_compare tools/cub_compare.cu
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>

__global__ void fill(uint32_t* k, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    k[i] = uint32_t(z ^ (z >> 31));
  }
}

int main(int argc, char** argv) {
  size_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (size_t(1) << 28);
  int pairs = argc > 2 ? atoi(argv[2]) : 0;
  uint32_t *k0, *k1, *v0 = nullptr, *v1 = nullptr;
  cudaMalloc(&k0, n * 4);
  cudaMalloc(&k1, n * 4);
  if (pairs) { cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4); }
  fill<<<148 * 8, 512>>>(k0, n, 0);
  size_t tmp = 0;
  if (pairs)
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n);
  else
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0, k1, n);
  void* t;
  cudaMalloc(&t, tmp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f, sum = 0;
  const int reps = 20;
  for (int r = -3; r < reps; ++r) {
    cudaEventRecord(a);
    if (pairs)
      cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, n);
    else
      cub::DeviceRadixSort::SortKeys(t, tmp, k0, k1, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 0) { sum += ms; if (ms < best) best = ms; }
  }
  printf("{\"cub\": \"%s\", \"n\": %zu, \"ms_mean\": %.4f, \"ms_best\": %.4f, \"gkeys_mean\": %.2f, \"err\": \"%s\"}\n",
         pairs ? "SortPairs" : "SortKeys", n, sum / reps, best, n / (sum / reps) / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
