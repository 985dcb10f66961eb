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

namespace osb {

// Row gather dst[i] = src[index[i]] for rows of row_bytes bytes: the value
// payload of a sort whose values are wider than 8 bytes (onesweep_sort takes
// any value dtype, binning.py:301-304) travels through the passes as a 4- or
// 8-byte index and is gathered once at the end.  U is the widest unit that
// divides the row and both base addresses; rows are cut into units and the
// grid strides over (row, unit) pairs, so stores are coalesced.
template <typename U, typename I>
__global__ void gather_rows_kernel(const U* __restrict__ src, const I* __restrict__ index,
                                   U* __restrict__ dst, size_t n, size_t units) {
  const size_t total = n * units;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t u = size_t(blockIdx.x) * blockDim.x + threadIdx.x; u < total; u += stride) {
    const size_t row = u / units, col = u - row * units;
    dst[u] = src[size_t(index[row]) * units + col];
  }
}

template <typename I>
static cudaError_t gather_rows_typed(const void* src, const void* index, void* dst, size_t n,
                                     size_t row_bytes, cudaStream_t stream) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | row_bytes;
  const int threads = 256;
  auto go = [&](auto unit) -> cudaError_t {
    using U = decltype(unit);
    const size_t units = row_bytes / sizeof(U);
    const int grid = stream_grid(n * units, threads);
    gather_rows_kernel<U, I><<<grid, threads, 0, stream>>>(
        static_cast<const U*>(src), static_cast<const I*>(index), static_cast<U*>(dst), n, units);
    return cudaGetLastError();
  };
  if ((a & 15u) == 0) return go(uint4{});
  if ((a & 7u) == 0) return go(uint2{});
  if ((a & 3u) == 0) return go(uint32_t{});
  if ((a & 1u) == 0) return go(uint16_t{});
  return go(uint8_t{});
}

cudaError_t launch_gather_rows(const void* src, const void* index, int index_bytes, void* dst,
                               size_t n, size_t row_bytes, cudaStream_t stream) {
  if (n == 0 || row_bytes == 0) return cudaSuccess;
  if (index_bytes == 4) return gather_rows_typed<uint32_t>(src, index, dst, n, row_bytes, stream);
  if (index_bytes == 8) return gather_rows_typed<unsigned long long>(src, index, dst, n, row_bytes, stream);
  return cudaErrorInvalidValue;
}

}  // namespace osb
