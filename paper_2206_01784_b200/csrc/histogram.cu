// Upfront all-places digit histogram + per-place exclusive scan (sm_100a).
//
// Replaces global_histograms / histogram_kernel / global_bin_offsets
// (histogram.py:57-99, _kernels.py:131-145).  One read of every key yields the
// digit counts of every place (Fig. 5):
//   - persistent grid (a few blocks per SM), grid-stride over 16-byte vectors;
//   - per-block shared-memory u32 tables, replicated kCopies times and indexed
//     by lane % kCopies so same-digit lanes (low-entropy keys) spread over
//     distinct words instead of serialising on one address;
//   - one u64 atomicAdd per (place, digit) per block into global memory;
//   - the last block to finish (atomic ticket) scans each place's row into
//     exclusive bin offsets, so no separate scan launch is needed.
// Portions (histogram.py:79-88): a block's share of the input is n / grid keys,
// so its u32 counters cannot overflow for any n that fits in HBM
// (grid >= 148 blocks -> n < 148 * 2^32); the host checks the bound.
#include "common.cuh"

namespace osb {

constexpr int kHistThreads = 512;
constexpr int kHistCopies = 8;

__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <typename K, int FIXED_PASSES>
struct HistCounter {
  uint32_t* h;  // this lane's replica base
  int passes, begin, dbits, radix;
  uint32_t full_mask, top_mask;
  int codec;

  __device__ __forceinline__ void add(K x) const {
    x = apply_codec(x, codec);
    if (FIXED_PASSES > 0) {
#pragma unroll
      for (int p = 0; p < FIXED_PASSES; ++p) {
        const uint32_t m = (p == FIXED_PASSES - 1) ? top_mask : full_mask;
        const uint32_t d = digit_of(x, begin + p * dbits, m);
        atomicAdd(&h[(p * radix + d) * kHistCopies], 1u);
      }
    } else {
      for (int p = 0; p < passes; ++p) {
        const uint32_t m = (p == passes - 1) ? top_mask : full_mask;
        const uint32_t d = digit_of(x, begin + p * dbits, m);
        atomicAdd(&h[(p * radix + d) * kHistCopies], 1u);
      }
    }
  }
  __device__ __forceinline__ void add_vec(uint4 v) const {
    if (sizeof(K) == 4) {
      add(K(v.x));
      add(K(v.y));
      add(K(v.z));
      add(K(v.w));
    } else {
      add(K((uint64_t(v.y) << 32) | v.x));
      add(K((uint64_t(v.w) << 32) | v.z));
    }
  }
};

template <typename K, int FIXED_PASSES>
__global__ void __launch_bounds__(kHistThreads) onesweep_histogram_kernel(const HistParams P) {
  extern __shared__ uint32_t s_hist[];  // [passes*radix][kHistCopies]
  __shared__ unsigned long long s_wsum[kHistThreads / 32];
  __shared__ bool s_last;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int radix = 1 << P.digit_bits;
  const int nbins = P.passes * radix;
  for (int i = tid; i < nbins * kHistCopies; i += kHistThreads) s_hist[i] = 0;
  __syncthreads();

  HistCounter<K, FIXED_PASSES> c;
  c.h = s_hist + (lane % kHistCopies);
  c.passes = P.passes;
  c.begin = P.begin_bit;
  c.dbits = P.digit_bits;
  c.radix = radix;
  c.full_mask = uint32_t(radix - 1);
  c.top_mask = uint32_t((1u << P.top_bits) - 1u);
  c.codec = P.codec;

  const K* keys = static_cast<const K*>(P.keys);
  const size_t n = P.n;
  constexpr size_t KPV = 16 / sizeof(K);
  size_t head = ((16u - (reinterpret_cast<uintptr_t>(keys) & 15u)) & 15u) / sizeof(K);
  if (head > n) head = n;
  const size_t nvec = (n - head) / KPV;
  const size_t tail = head + nvec * KPV;
  const uint4* vp = reinterpret_cast<const uint4*>(keys + head);

  const size_t stride = size_t(gridDim.x) * kHistThreads;
  size_t v = size_t(blockIdx.x) * kHistThreads + tid;
  for (; v + 3 * stride < nvec; v += 4 * stride) {
    const uint4 q0 = ld_stream_v4(vp + v);
    const uint4 q1 = ld_stream_v4(vp + v + stride);
    const uint4 q2 = ld_stream_v4(vp + v + 2 * stride);
    const uint4 q3 = ld_stream_v4(vp + v + 3 * stride);
    c.add_vec(q0);
    c.add_vec(q1);
    c.add_vec(q2);
    c.add_vec(q3);
  }
  for (; v < nvec; v += stride) c.add_vec(ld_stream_v4(vp + v));
  // unaligned head / ragged tail (< 2 vectors of keys in total)
  const size_t g = size_t(blockIdx.x) * kHistThreads + tid;
  if (g < head) c.add(keys[g]);
  if (tail + g < n) c.add(keys[tail + g]);
  __syncthreads();

  // flush: reduce replicas, one u64 atomic per non-empty bin
  for (int i = tid; i < nbins; i += kHistThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int r = 0; r < kHistCopies; ++r) s += s_hist[i * kHistCopies + r];
    if (s) atomicAdd(&P.hist[i], (unsigned long long)s);
  }
  if (P.offsets == nullptr) return;

  // last-block-done: exclusive scan of each place (histogram.py:94-99)
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(P.done_counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int p = 0; p < P.passes; ++p) {
    for (int base = 0; base < radix; base += kHistThreads) {
      const int i = base + tid;
      const unsigned long long x = (i < radix) ? __ldcg(&P.hist[p * radix + i]) : 0ull;
      unsigned long long incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      unsigned long long pre = 0;
      for (int w = 0; w < warp; ++w) pre += s_wsum[w];
      if (i < radix) P.offsets[p * radix + i] = pre + incl - x;
      __syncthreads();
    }
  }
}

// Standalone per-row exclusive scan (one block per row, any radix).
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const unsigned long long* counts,
                                                              int radix,
                                                              unsigned long long* out) {
  __shared__ unsigned long long s_wsum[32];
  __shared__ unsigned long long s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long* row = counts + size_t(blockIdx.x) * radix;
  unsigned long long* orow = out + size_t(blockIdx.x) * radix;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < radix; base += 1024) {
    const int i = base + tid;
    const unsigned long long x = i < radix ? row[i] : 0ull;
    unsigned long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    unsigned long long pre = s_carry;
    for (int w = 0; w < warp; ++w) pre += s_wsum[w];
    if (i < radix) orow[i] = pre + incl - x;
    __syncthreads();
    if (tid == 1023) s_carry = pre + incl;
    __syncthreads();
  }
}

static int hist_grid() {
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms * 2;
  }
  return grid;
}

template <typename K, int FIXED>
static cudaError_t launch_hist_t(const HistParams& p, cudaStream_t stream) {
  auto kern = onesweep_histogram_kernel<K, FIXED>;
  const size_t smem = size_t(p.passes) * (size_t(1) << p.digit_bits) * kHistCopies * 4;
  static size_t configured = 0;
  if (smem > 48 * 1024 && configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  kern<<<hist_grid(), kHistThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_histogram(const HistParams& p, int key_bytes, cudaStream_t stream) {
  if (p.n == 0) return cudaSuccess;
  const bool full8 = p.digit_bits == 8 && p.top_bits == 8;
  if (key_bytes == 4) {
    if (full8 && p.passes == 4) return launch_hist_t<uint32_t, 4>(p, stream);
    return launch_hist_t<uint32_t, 0>(p, stream);
  }
  if (key_bytes == 8) {
    if (full8 && p.passes == 8) return launch_hist_t<uint64_t, 8>(p, stream);
    return launch_hist_t<uint64_t, 0>(p, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_exclusive_scan(const unsigned long long* counts, int rows, int radix,
                                  unsigned long long* out, cudaStream_t stream) {
  if (rows == 0 || radix == 0) return cudaSuccess;
  exclusive_scan_kernel<<<rows, 1024, 0, stream>>>(counts, radix, out);
  return cudaGetLastError();
}

int histogram_grid_size() { return hist_grid(); }

}  // namespace osb
