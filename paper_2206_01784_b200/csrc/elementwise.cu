// Elementwise kernels: key codec (keycodec.py:184-212) and the device key
// generator (keygen.py:46-76).  Both are HBM-streaming, grid-stride loops.
#include "common.cuh"

namespace osb {

template <typename K>
__global__ void codec_kernel(const K* __restrict__ in, K* __restrict__ out, size_t n, int codec) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = apply_codec(in[i], codec);
}

static int stream_grid(size_t n, int threads) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  size_t want = (n + threads - 1) / threads;
  size_t cap = size_t(sms) * 8;
  return int(want < cap ? (want ? want : 1) : cap);
}

cudaError_t launch_codec(const void* in, void* out, size_t n, int key_bytes, int codec,
                         cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int grid = stream_grid(n, threads);
  if (key_bytes == 4)
    codec_kernel<uint32_t><<<grid, threads, 0, stream>>>(static_cast<const uint32_t*>(in),
                                                         static_cast<uint32_t*>(out), n, codec);
  else if (key_bytes == 8)
    codec_kernel<uint64_t><<<grid, threads, 0, stream>>>(static_cast<const uint64_t*>(in),
                                                         static_cast<uint64_t*>(out), n, codec);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// splitmix64 finaliser, keygen.py:46-54 (wrapping u64 arithmetic).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

// word(c) = mix64(seed + (c + 1) * GAMMA)  (keygen.py:57-60)
__device__ __forceinline__ uint64_t uniform_word(uint64_t seed, uint64_t counter) {
  return mix64(seed + (counter + 1ull) * 0x9E3779B97F4A7C15ull);
}

template <typename K>
__global__ void keygen_kernel(K* __restrict__ out, size_t n, int q, uint64_t seed,
                              uint64_t first) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t base = (first + i) * uint64_t(q);
    uint64_t k = uniform_word(seed, base);
    for (int j = 1; j < q; ++j) k &= uniform_word(seed, base + uint64_t(j));
    out[i] = K(k);  // astype(uint32) keeps the low bits (keygen.py:76)
  }
}

cudaError_t launch_keygen(void* out, size_t n, int key_bits, int q, unsigned long long seed,
                          unsigned long long first, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int grid = stream_grid(n, threads);
  if (key_bits == 32)
    keygen_kernel<uint32_t><<<grid, threads, 0, stream>>>(static_cast<uint32_t*>(out), n, q, seed,
                                                          first);
  else if (key_bits == 64)
    keygen_kernel<uint64_t><<<grid, threads, 0, stream>>>(static_cast<uint64_t*>(out), n, q, seed,
                                                          first);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace osb
