// Digit widths 9..16 (sm_100a): the reference accepts digit_bits in [1, 16]
// everywhere (keycodec.py:107-123,139); the Onesweep binning kernel bins at
// most 8 bits per launch (one thread per digit, u16 per-warp counters).
//
//   * wide histogram: exact counts of 2^d-way digits at every place
//     (histogram.py:57-91 for d > 8).  Block (x, place, chunk) keeps
//     shared-memory u32 counters for one 16K-digit chunk of one place and
//     grid-strides over the keys; one u64 atomicAdd per nonzero counter.
//   * wide scatter: the last step of a 2^d-way partition pass.  The host runs
//     the pass as two stable <= 8-bit binning launches over the digit's low
//     and high parts (dense, into scratch: the stable LSD order of the digit),
//     then this kernel moves every element j of that dense order to
//     base[d] + (j - dense_start[d]) -- the reference's
//     dst[offsets[d] + rank] (binning.py:200) for any caller base row or
//     StripCarry -- and writes carry[d] = base[d] + count[d]
//     (binning.py:196-198).
#include "common.cuh"

namespace osb {

constexpr int kWideChunk = 16384;  // digits per block: 64 KiB of u32 counters
constexpr int kWideThreads = 512;

template <typename K>
__global__ void __launch_bounds__(kWideThreads) wide_histogram_kernel(
    const K* keys, size_t n, int codec, int begin_bit, int digit_bits, int passes, int top_bits,
    unsigned long long* hist) {
  extern __shared__ uint32_t s_cnt[];
  const int place = blockIdx.y;
  const uint32_t lo = blockIdx.z * kWideChunk;
  const int radix = 1 << digit_bits;
  const uint32_t mask = uint32_t((1u << (place == passes - 1 ? top_bits : digit_bits)) - 1u);
  const int shift = begin_bit + place * digit_bits;
  const XorCodec<K> c = XorCodec<K>::make(codec);
  for (int i = threadIdx.x; i < kWideChunk; i += kWideThreads) s_cnt[i] = 0;
  __syncthreads();
  const size_t stride = size_t(gridDim.x) * kWideThreads;
  for (size_t i = size_t(blockIdx.x) * kWideThreads + threadIdx.x; i < n; i += stride) {
    const uint32_t d = digit_of(c(keys[i]), shift, mask) - lo;
    if (d < uint32_t(kWideChunk)) atomicAdd(&s_cnt[d], 1u);
  }
  __syncthreads();
  const int hi = min(kWideChunk, radix - int(lo));
  for (int i = threadIdx.x; i < hi; i += kWideThreads)
    if (s_cnt[i]) atomicAdd(&hist[size_t(place) * radix + lo + i], (unsigned long long)s_cnt[i]);
}

cudaError_t launch_wide_histogram(const void* keys, size_t n, int key_bytes, int codec,
                                  int begin_bit, int digit_bits, int passes, int top_bits,
                                  unsigned long long* hist, cudaStream_t stream) {
  if (n == 0 || passes == 0) return cudaSuccess;
  const int radix = 1 << digit_bits;
  const int chunks = (radix + kWideChunk - 1) / kWideChunk;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int per = passes * chunks;
  int gx = (2 * sms + per - 1) / per;
  const size_t need = (n + kWideThreads - 1) / kWideThreads;
  if (size_t(gx) > need) gx = int(need);
  const dim3 grid(gx, passes, chunks);
  const size_t smem = kWideChunk * 4;
  if (key_bytes == 4) {
    auto k = wide_histogram_kernel<uint32_t>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, kWideThreads, smem, stream>>>(static_cast<const uint32_t*>(keys), n, codec, begin_bit,
                                             digit_bits, passes, top_bits, hist);
  } else {
    auto k = wide_histogram_kernel<uint64_t>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, kWideThreads, smem, stream>>>(static_cast<const uint64_t*>(keys), n, codec, begin_bit,
                                             digit_bits, passes, top_bits, hist);
  }
  return cudaGetLastError();
}

// rel[d] = base[d] - dense_start[d] (two's complement), carry[d] = base[d] + count[d]
__global__ void wide_tables_kernel(const unsigned long long* base, const unsigned long long* count,
                                   const unsigned long long* dense_start, int radix,
                                   unsigned long long* rel, unsigned long long* carry) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= radix) return;
  rel[d] = base[d] - dense_start[d];
  carry[d] = base[d] + count[d];
}

template <typename K, typename V>
__global__ void wide_scatter_kernel(const K* src_k, K* dst_k, const V* src_v, V* dst_v, size_t n,
                                    int shift, uint32_t mask, const unsigned long long* rel,
                                    XorCodec<K> cout) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t j = size_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += stride) {
    const K x = src_k[j];
    const size_t at = size_t(rel[digit_of(x, shift, mask)] + j);
    dst_k[at] = cout(x);
    if (src_v != nullptr) dst_v[at] = src_v[j];
  }
}

template <typename K>
static cudaError_t scatter_val(const void* sk, void* dk, const void* sv, void* dv, int vb, size_t n,
                               int shift, uint32_t mask, const unsigned long long* rel,
                               int codec_out, cudaStream_t s) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t blocks = (n + 255) / 256;
  if (blocks > size_t(sms) * 8) blocks = size_t(sms) * 8;
  const auto co = XorCodec<K>::make(codec_out);
  const K* k = static_cast<const K*>(sk);
  K* o = static_cast<K*>(dk);
  switch (vb) {
    case 0:
      wide_scatter_kernel<K, uint8_t><<<unsigned(blocks), 256, 0, s>>>(k, o, nullptr, nullptr, n, shift, mask, rel, co);
      break;
    case 1:
      wide_scatter_kernel<K, uint8_t><<<unsigned(blocks), 256, 0, s>>>(
          k, o, static_cast<const uint8_t*>(sv), static_cast<uint8_t*>(dv), n, shift, mask, rel, co);
      break;
    case 2:
      wide_scatter_kernel<K, uint16_t><<<unsigned(blocks), 256, 0, s>>>(
          k, o, static_cast<const uint16_t*>(sv), static_cast<uint16_t*>(dv), n, shift, mask, rel, co);
      break;
    case 4:
      wide_scatter_kernel<K, uint32_t><<<unsigned(blocks), 256, 0, s>>>(
          k, o, static_cast<const uint32_t*>(sv), static_cast<uint32_t*>(dv), n, shift, mask, rel, co);
      break;
    case 8:
      wide_scatter_kernel<K, uint64_t><<<unsigned(blocks), 256, 0, s>>>(
          k, o, static_cast<const uint64_t*>(sv), static_cast<uint64_t*>(dv), n, shift, mask, rel, co);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_wide_tables(const unsigned long long* base, const unsigned long long* count,
                               const unsigned long long* dense_start, int radix,
                               unsigned long long* rel, unsigned long long* carry,
                               cudaStream_t stream) {
  wide_tables_kernel<<<(radix + 255) / 256, 256, 0, stream>>>(base, count, dense_start, radix, rel,
                                                               carry);
  return cudaGetLastError();
}

cudaError_t launch_wide_scatter(const void* src_k, void* dst_k, const void* src_v, void* dst_v,
                                int kb, int vb, size_t n, int shift, int width,
                                const unsigned long long* rel, int codec_out,
                                cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const uint32_t mask = uint32_t((1u << width) - 1u);
  if (kb == 4)
    return scatter_val<uint32_t>(src_k, dst_k, src_v, dst_v, vb, n, shift, mask, rel, codec_out, stream);
  return scatter_val<uint64_t>(src_k, dst_k, src_v, dst_v, vb, n, shift, mask, rel, codec_out, stream);
}

}  // namespace osb
