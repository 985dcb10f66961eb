// Reduce-then-scan LSD radix sort on the device: the comparator the paper
// measures Onesweep against (Figs. 1-2), as the ablation of SURVEY.md
// 8f rank 4.  Replaces, for one digit place,
//   rts_upsweep      baseline.py:55-73   per-tile digit histograms (n reads)
//   rts_block_prefix baseline.py:76-84   digit-major exclusive prefix
//   rts_downsweep    baseline.py:87-118  stable scatter (n reads + n writes)
// The downsweep is the Onesweep binning kernel itself with the look-back
// replaced by a read of the precomputed run starts (PassParams::rts_offsets),
// so the two sorts differ only in how a tile learns its output offsets: 3n
// element transfers per place here, 2n with the chained scan.
#include "common.cuh"

namespace osb {

constexpr int kRtsThreads = 256;   // one thread per digit in the prefix kernels
#ifndef OS_RTS_CHUNK
#define OS_RTS_CHUNK 32  // prefix 44 us per place at 26K tiles (16: 62, 64: 50)
#endif
constexpr int kRtsChunk = OS_RTS_CHUNK;  // tiles per chunk of the two-level prefix

// One block per tile: per-warp shared-memory digit counters (shared-memory
// reductions), then thread d writes counts[tile][d].
template <typename K>
__global__ void __launch_bounds__(kRtsThreads) rts_upsweep_kernel(const K* keys, size_t n,
                                                                  uint32_t tile_keys, int shift,
                                                                  uint32_t mask, int codec,
                                                                  uint32_t* counts) {
  constexpr int W = kRtsThreads / 32;
  __shared__ uint32_t s_cnt[W][kMaxRadix];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < W * kMaxRadix; i += kRtsThreads) (&s_cnt[0][0])[i] = 0;
  __syncthreads();
  const XorCodec<K> c = XorCodec<K>::make(codec);
  const size_t lo = size_t(blockIdx.x) * tile_keys;
  const size_t hi = lo + tile_keys < n ? lo + tile_keys : n;
  const uint32_t base = smem_u32(&s_cnt[warp][0]);
  for (size_t i = lo + tid; i < hi; i += kRtsThreads) {
    const uint32_t d = digit_of(c(keys[i]), shift, mask);
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base + d * 4u) : "memory");
  }
  __syncthreads();
  if (tid <= int(mask)) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) sum += s_cnt[w][tid];
    counts[size_t(blockIdx.x) * (mask + 1) + tid] = sum;
  }
}

// The digit-major prefix (baseline.py:76-84) over the tiles x radix count
// table, in four small launches that keep every load independent:
//   (A) per chunk of kRtsChunk tiles, the column sums;
//   (B) per digit, a block-wide exclusive scan of its chunk sums (and the
//       digit total);
//   (C) one block: exclusive scan of the digit totals (the digit-major base);
//   (D) per chunk, the running prefix over its tiles -> absolute run starts.
__global__ void __launch_bounds__(kRtsThreads) rts_chunk_sums_kernel(const uint32_t* counts,
                                                                     uint32_t tiles, int radix,
                                                                     unsigned long long* csum) {
  const int d = threadIdx.x;
  if (d >= radix) return;
  const uint32_t t0 = blockIdx.x * kRtsChunk;
  uint32_t v[kRtsChunk];
#pragma unroll
  for (int j = 0; j < kRtsChunk; ++j)
    v[j] = (t0 + j < tiles) ? counts[size_t(t0 + j) * radix + d] : 0u;
  unsigned long long sum = 0;
#pragma unroll
  for (int j = 0; j < kRtsChunk; ++j) sum += v[j];
  csum[size_t(blockIdx.x) * radix + d] = sum;
}

constexpr int kRtsScanThreads = 1024;

__global__ void __launch_bounds__(kRtsScanThreads) rts_column_scan_kernel(
    unsigned long long* csum, uint32_t chunks, int radix, unsigned long long* dtotal) {
  __shared__ unsigned long long s_w[kRtsScanThreads / 32];
  const int d = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (chunks + kRtsScanThreads - 1) / kRtsScanThreads;
  const uint32_t c0 = uint32_t(tid) * per;
  unsigned long long local = 0;
  for (uint32_t j = 0; j < per; ++j)
    if (c0 + j < chunks) local += csum[size_t(c0 + j) * radix + d];
  unsigned long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  unsigned long long pre = 0;
  for (int w = 0; w < warp; ++w) pre += s_w[w];
  unsigned long long run = pre + incl - local;
  for (uint32_t j = 0; j < per; ++j) {
    if (c0 + j < chunks) {
      const unsigned long long x = csum[size_t(c0 + j) * radix + d];
      csum[size_t(c0 + j) * radix + d] = run;
      run += x;
    }
  }
  if (tid == kRtsScanThreads - 1) dtotal[d] = pre + incl;
}

__global__ void __launch_bounds__(kRtsThreads) rts_digit_scan_kernel(unsigned long long* dtotal,
                                                                     int radix) {
  __shared__ unsigned long long s_w[kRtsThreads / 32];
  const int d = threadIdx.x, lane = d & 31, warp = d >> 5;
  const unsigned long long x = d < radix ? dtotal[d] : 0ull;
  unsigned long long incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  unsigned long long pre = 0;
  for (int w = 0; w < warp; ++w) pre += s_w[w];
  if (d < radix) dtotal[d] = pre + incl - x;  // now the digit-major base
}

__global__ void __launch_bounds__(kRtsThreads) rts_chunk_apply_kernel(
    const uint32_t* counts, const unsigned long long* cbase, const unsigned long long* dbase,
    uint32_t tiles, int radix, unsigned long long* offsets) {
  const int d = threadIdx.x;
  if (d >= radix) return;
  const uint32_t t0 = blockIdx.x * kRtsChunk;
  uint32_t v[kRtsChunk];
#pragma unroll
  for (int j = 0; j < kRtsChunk; ++j)
    v[j] = (t0 + j < tiles) ? counts[size_t(t0 + j) * radix + d] : 0u;
  unsigned long long run = cbase[size_t(blockIdx.x) * radix + d] + dbase[d];
#pragma unroll
  for (int j = 0; j < kRtsChunk; ++j) {
    if (t0 + j < tiles) offsets[size_t(t0 + j) * radix + d] = run;
    run += v[j];
  }
}

cudaError_t launch_rts_upsweep(const void* keys, size_t n, int key_bytes, uint32_t tile_keys,
                               int shift, uint32_t mask, int codec, uint32_t* counts,
                               cudaStream_t stream) {
  const size_t tiles = (n + tile_keys - 1) / tile_keys;
  if (tiles == 0) return cudaSuccess;
  if (key_bytes == 4)
    rts_upsweep_kernel<uint32_t><<<unsigned(tiles), kRtsThreads, 0, stream>>>(
        static_cast<const uint32_t*>(keys), n, tile_keys, shift, mask, codec, counts);
  else
    rts_upsweep_kernel<uint64_t><<<unsigned(tiles), kRtsThreads, 0, stream>>>(
        static_cast<const uint64_t*>(keys), n, tile_keys, shift, mask, codec, counts);
  return cudaGetLastError();
}

size_t rts_chunk_count(size_t tiles) { return (tiles + kRtsChunk - 1) / kRtsChunk + 1; }

// csum holds chunks + 1 rows: the chunk sums/bases, then the digit totals.
cudaError_t launch_rts_prefix(const uint32_t* counts, uint32_t tiles, int radix,
                              unsigned long long* csum, unsigned long long* offsets,
                              cudaStream_t stream) {
  if (tiles == 0) return cudaSuccess;
  const uint32_t chunks = uint32_t(rts_chunk_count(tiles) - 1);
  unsigned long long* dtotal = csum + size_t(chunks) * radix;
  rts_chunk_sums_kernel<<<chunks, kRtsThreads, 0, stream>>>(counts, tiles, radix, csum);
  rts_column_scan_kernel<<<radix, kRtsScanThreads, 0, stream>>>(csum, chunks, radix, dtotal);
  rts_digit_scan_kernel<<<1, kRtsThreads, 0, stream>>>(dtotal, radix);
  rts_chunk_apply_kernel<<<chunks, kRtsThreads, 0, stream>>>(counts, csum, dtotal, tiles, radix,
                                                             offsets);
  return cudaGetLastError();
}

}  // namespace osb
