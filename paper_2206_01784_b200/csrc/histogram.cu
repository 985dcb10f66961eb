// Upfront all-places digit histogram + per-place exclusive scan (sm_100a).
//
// Replaces global_histograms / histogram_kernel / global_bin_offsets
// (histogram.py:57-99, _kernels.py:131-145).  One read of every key yields the
// digit counts of every place (Fig. 5):
//   - persistent grid (one 1024-thread block per SM), grid-stride over
//     16-byte streaming loads, software-pipelined one batch ahead;
//   - per-block shared-memory counters with one private copy per LANE, two
//     u16 counters per u32 word: word = ((place * radix/2 + digit/2) * 32 + lane),
//     half = digit & 1.  Every shared atomic of a warp therefore hits 32
//     different banks (one wavefront), whatever the key distribution --
//     all-equal keys included;
//   - "portions" (histogram.py:79-88): a lane's u16 counter sees at most
//     kHistWarps * 16 keys per round, so the block folds its lane copies into
//     u32 block totals every kRoundsPerPortion rounds, long before 65535;
//   - one u64 atomicAdd per (place, digit) per block into global memory;
//   - the last block to finish (atomic ticket) scans each place's row into
//     exclusive bin offsets, so no separate scan launch is needed.
#include "common.cuh"

namespace osb {

constexpr int kHistThreads = 1024;
constexpr int kHistWarps = kHistThreads / 32;
#ifndef OS_HIST_L2PF
#define OS_HIST_L2PF 0  // 1: histogram loads carry an L2 256-byte prefetch hint
#endif
#ifndef OS_HIST_VEC
#define OS_HIST_VEC 4
#endif
constexpr int kHistVec = OS_HIST_VEC;             // 16-byte vectors per thread per round
constexpr int kRoundsPerPortion = 65535 / (kHistWarps * kHistVec * 4);  // u16 headroom

__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p) {
  uint4 v;
#if OS_HIST_L2PF
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
#endif
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <typename K, int FIXED_PASSES>
struct HistCounter {
  uint32_t* lane_base;  // s_hist + lane
  int passes, begin, dbits, half_radix;
  uint32_t full_mask, top_mask;
  XorCodec<K> codec;

  __device__ __forceinline__ void add_place(K x, int p, uint32_t m) const {
    uint32_t d;
    if constexpr (FIXED_PASSES == 8 && sizeof(K) == 8) {
      // eight 8-bit places over a 64-bit key: place p is byte p (one PRMT)
      const uint32_t w = p < 4 ? uint32_t(uint64_t(x)) : uint32_t(uint64_t(x) >> 32);
      d = __byte_perm(w, 0u, 0x4440u + uint32_t(p & 3));
    } else {
      d = digit_of(x, begin + p * dbits, m);
    }
    const uint32_t word = (uint32_t(p * half_radix) + (d >> 1)) * 32u;
    // no return value needed: a reduction, not an atomic exchange
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(lane_base + word)),
                 "r"(1u << ((d & 1u) << 4))
                 : "memory");
  }
  __device__ __forceinline__ void add(K x) const {
    x = codec(x);
    if (FIXED_PASSES > 0) {
#pragma unroll
      for (int p = 0; p < FIXED_PASSES; ++p)
        add_place(x, p, p == FIXED_PASSES - 1 ? top_mask : full_mask);
    } else {
      for (int p = 0; p < passes; ++p) add_place(x, p, p == passes - 1 ? top_mask : full_mask);
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
__global__ void __launch_bounds__(kHistThreads, 1) onesweep_histogram_kernel(const HistParams P) {
  extern __shared__ uint32_t s_hist[];  // [passes * radix/2][32] lane copies, then u32 totals
  __shared__ unsigned long long s_wsum[kHistWarps];
  __shared__ bool s_last;
  __shared__ uint32_t s_trivial;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int radix = 1 << P.digit_bits;
  const int half_radix = radix > 1 ? radix / 2 : 1;
  const int nbins = P.passes * radix;
  const int nwords = P.passes * half_radix * 32;
  uint32_t* s_total = s_hist + nwords;  // [passes * radix] u32 block totals
  for (int i = tid; i < nwords + nbins; i += kHistThreads) s_hist[i] = 0;
  __syncthreads();

  HistCounter<K, FIXED_PASSES> c;
  c.lane_base = s_hist + lane;
  c.passes = P.passes;
  c.begin = P.begin_bit;
  c.dbits = P.digit_bits;
  c.half_radix = half_radix;
  c.full_mask = uint32_t(radix - 1);
  c.top_mask = uint32_t((1u << P.top_bits) - 1u);
  c.codec = XorCodec<K>::make(P.codec);

  // fold the lane copies into the u32 block totals and clear them
  auto fold = [&]() {
    __syncthreads();
    for (int b = tid; b < nbins; b += kHistThreads) {
      const int p = b / radix, d = b % radix;
      uint32_t* w = s_hist + (p * half_radix + (d >> 1)) * 32;
      const int sh = (d & 1) * 16;
      uint32_t sum = 0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) sum += (w[(l + tid) & 31] >> sh) & 0xffffu;
      s_total[b] += sum;
    }
    __syncthreads();
    for (int i = tid; i < nwords; i += kHistThreads) s_hist[i] = 0;
    __syncthreads();
  };

  const K* keys = static_cast<const K*>(P.keys);
  const size_t n = P.n;
  constexpr size_t KPV = 16 / sizeof(K);
  size_t head = ((16u - (reinterpret_cast<uintptr_t>(keys) & 15u)) & 15u) / sizeof(K);
  if (head > n) head = n;
  const size_t nvec = (n - head) / KPV;
  const size_t tail = head + nvec * KPV;
  const uint4* vp = reinterpret_cast<const uint4*>(keys + head);

  const size_t stride = size_t(gridDim.x) * kHistThreads;
  const size_t per_round = stride * kHistVec;
  const size_t rounds = (nvec + per_round - 1) / per_round;  // same for every block
  size_t v0 = size_t(blockIdx.x) * kHistThreads + tid;

  uint4 cur[kHistVec];
#pragma unroll
  for (int u = 0; u < kHistVec; ++u)
    if (v0 + u * stride < nvec) cur[u] = ld_stream_v4(vp + v0 + u * stride);
  for (size_t r = 0; r < rounds; ++r) {
    const size_t v1 = v0 + per_round;
    uint4 nxt[kHistVec];
#pragma unroll
    for (int u = 0; u < kHistVec; ++u)  // next batch in flight while this one counts
      if (v1 + u * stride < nvec) nxt[u] = ld_stream_v4(vp + v1 + u * stride);
#pragma unroll
    for (int u = 0; u < kHistVec; ++u)
      if (v0 + u * stride < nvec) c.add_vec(cur[u]);
#pragma unroll
    for (int u = 0; u < kHistVec; ++u) cur[u] = nxt[u];
    v0 = v1;
    if ((r + 1) % (kRoundsPerPortion * (sizeof(K) == 8 ? 2 : 1)) == 0) fold();
  }
  // unaligned head / ragged tail (< 2 vectors of keys in total)
  const size_t g = size_t(blockIdx.x) * kHistThreads + tid;
  if (g < head) c.add(keys[g]);
  if (tail + g < n) c.add(keys[tail + g]);
  fold();

  // one u64 atomic per non-empty bin
  for (int i = tid; i < nbins; i += kHistThreads)
    if (s_total[i]) atomicAdd(&P.hist[i], (unsigned long long)s_total[i]);
  if (P.offsets == nullptr) return;

  // last-block-done: exclusive scan of each place (histogram.py:94-99)
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    s_last = (atomicAdd(P.done_counter, 1u) == gridDim.x - 1);
    s_trivial = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int p = 0; p < P.passes; ++p) {
    const int i = tid;  // radix <= 256 < kHistThreads
    const unsigned long long x = (i < radix) ? __ldcg(&P.hist[p * radix + i]) : 0ull;
    if (i < radix && x == P.n) atomicOr(&s_trivial, 1u << p);  // one bin holds every key
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
  if (tid == 0 && P.tickets != nullptr) plan_tickets(P.tickets, P.ticket_stride, P.strips, P.passes, s_trivial, P.fixed_ends != 0);
}

// Last block's scan for 8-bit places: the 1024 threads take four places per
// round (thread t: place p0 + t / 256, digit t % 256), so every place's
// counts are fetched from L2 in one round trip instead of one per place.
__device__ __forceinline__ void scan_places256(const HistParams& P, int places,
                                               unsigned long long* s_wsum, uint32_t* s_trivial) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = tid >> 8;  // place within the round
  for (int p0 = 0; p0 < places; p0 += kHistThreads / 256) {
    const int p = p0 + q;
    const unsigned long long x = p < places ? __ldcg(&P.hist[p * 256 + (tid & 255)]) : 0ull;
    if (p < places && x == P.n) atomicOr(s_trivial, 1u << p);  // one bin holds every key
    unsigned long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    unsigned long long pre = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) pre += (w < (warp & 7)) ? s_wsum[(warp & ~7) + w] : 0ull;
    if (p < places) P.offsets[p * 256 + (tid & 255)] = pre + incl - x;
    __syncthreads();
  }
}

// Specialisation for the headline shape: 32-bit keys, four byte-aligned
// 8-bit places (begin_bit 0, end_bit 32).  Counters are lane-private u32
// (4 places x 256 digits x 32 lanes = 128 KiB, bank = lane: conflict-free and
// never near overflow), the digit is one PRMT byte extract and the counter
// address one LEA, so a key costs four (PRMT, LEA, ATOMS) triples.
constexpr size_t kHistU32Smem = 4 * 256 * 32 * 4;

template <bool CODED>
__global__ void __launch_bounds__(kHistThreads, 1)
    onesweep_histogram_u32d8_kernel(const HistParams P) {
  grid_launch_dependents();  // lets a PDL-launched first pass start its prologue
  extern __shared__ uint32_t s_cnt[];  // [place][digit][lane]
  __shared__ unsigned long long s_wsum[kHistWarps];
  __shared__ bool s_last;
  __shared__ uint32_t s_trivial;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  {
    uint4* z = reinterpret_cast<uint4*>(s_cnt);
    for (int i = tid; i < int(kHistU32Smem / 16); i += kHistThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const XorCodec<uint32_t> codec = XorCodec<uint32_t>::make(P.codec);
  const uint32_t lane_base = smem_u32(s_cnt) + uint32_t(lane) * 4u;
  auto add = [&](uint32_t x) {
    if (CODED) x = codec(x);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t d = __byte_perm(x, 0u, 0x4440u + p);
      const uint32_t addr = lane_base + (uint32_t(p) << 15) + (d << 7);
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
    }
  };
  auto add_vec = [&](uint4 v) {
    add(v.x);
    add(v.y);
    add(v.z);
    add(v.w);
  };

  const uint32_t* keys = static_cast<const uint32_t*>(P.keys);
  const size_t n = P.n;
  size_t head = ((16u - (reinterpret_cast<uintptr_t>(keys) & 15u)) & 15u) / 4;
  if (head > n) head = n;
  const size_t nvec = (n - head) / 4;
  const size_t tail = head + nvec * 4;
  const uint4* vp = reinterpret_cast<const uint4*>(keys + head);
  const size_t stride = size_t(gridDim.x) * kHistThreads;
  const size_t per_round = stride * kHistVec;
  size_t v0 = size_t(blockIdx.x) * kHistThreads + tid;
  uint4 cur[kHistVec];
#pragma unroll
  for (int u = 0; u < kHistVec; ++u)
    if (v0 + u * stride < nvec) cur[u] = ld_stream_v4(vp + v0 + u * stride);
  while (v0 < nvec) {
    const size_t v1 = v0 + per_round;
    uint4 nxt[kHistVec];
#pragma unroll
    for (int u = 0; u < kHistVec; ++u)  // next batch in flight while this one counts
      if (v1 + u * stride < nvec) nxt[u] = ld_stream_v4(vp + v1 + u * stride);
#pragma unroll
    for (int u = 0; u < kHistVec; ++u)
      if (v0 + u * stride < nvec) add_vec(cur[u]);
#pragma unroll
    for (int u = 0; u < kHistVec; ++u) cur[u] = nxt[u];
    v0 = v1;
  }
  const size_t g = size_t(blockIdx.x) * kHistThreads + tid;
  if (g < head) add(keys[g]);
  if (tail + g < n) add(keys[tail + g]);
  __syncthreads();

  // reduce the 32 lane copies of each bin; one u64 atomic per non-empty bin
  for (int b = tid; b < 4 * 256; b += kHistThreads) {
    const uint32_t* w = s_cnt + b * 32;
    uint32_t s = 0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) s += w[(l + lane) & 31];
    if (s) atomicAdd(&P.hist[b], (unsigned long long)s);
  }
  if (P.offsets == nullptr) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    s_last = (atomicAdd(P.done_counter, 1u) == gridDim.x - 1);
    s_trivial = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  scan_places256(P, 4, s_wsum, &s_trivial);
  if (tid == 0 && P.tickets != nullptr) plan_tickets(P.tickets, P.ticket_stride, P.strips, 4, s_trivial, P.fixed_ends != 0);
}

// Specialisation for 64-bit keys with eight byte-aligned 8-bit places (C4).
// Lane-private u32 counters would need 8 x 256 x 32 x 4 B = 256 KiB, so two
// places share each counter word as u16 halves: word [place / 2][digit][lane],
// half = place & 1.  The increment is then a compile-time constant per
// (unrolled) place, and with the table 32 KiB-aligned one SHF + LOP3 turns a
// key word straight into the counter address ((byte << 7) | pair base |
// lane): three instructions per key and place, every red.shared
// conflict-free (bank = lane).  A lane adds at most 2 * kHistVec keys per
// round, so the u16 halves are folded into u32 block totals every
// kU64FoldRounds rounds.
constexpr size_t kHistU64Table = 4 * 256 * 32 * 4;                    // 128 KiB
constexpr size_t kHistU64Smem = kHistU64Table + 32768 + 8 * 256 * 4;  // + alignment + totals
constexpr int kU64FoldRounds = 65535 / (2 * kHistVec);

template <bool CODED>
__global__ void __launch_bounds__(kHistThreads, 1)
    onesweep_histogram_u64d8_kernel(const HistParams P) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  __shared__ unsigned long long s_wsum[kHistWarps];
  __shared__ bool s_last;
  __shared__ uint32_t s_trivial;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint32_t raw = smem_u32(s_raw);
  const uint32_t tbase = (raw + 32767u) & ~32767u;  // counter table, 32 KiB-aligned
  uint32_t* s_tab = reinterpret_cast<uint32_t*>(s_raw + (tbase - raw));
  uint32_t* s_total = reinterpret_cast<uint32_t*>(s_raw + (tbase - raw) + kHistU64Table);
  for (int i = tid; i < int(kHistU64Table / 4) + 8 * 256; i += kHistThreads) s_tab[i] = 0;
  __syncthreads();
  const XorCodec<uint64_t> codec = XorCodec<uint64_t>::make(P.codec);
  const uint32_t lbase = tbase + uint32_t(lane) * 4u;
  // one 32-bit half of a key: places 4*hi .. 4*hi+3, i.e. place pairs 2*hi, 2*hi+1
  auto add_word = [&](uint32_t w, int hi) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t pb = lbase + uint32_t(2 * hi + (j >> 1)) * 32768u;
      const uint32_t sh = j == 0 ? (w << 7) : (w >> (8 * j - 7));  // byte j at bits 7..14
      uint32_t addr;
      asm("lop3.b32 %0, %1, 0x7f80, %2, 0xea;" : "=r"(addr) : "r"(sh), "r"(pb));  // (a & b) | c
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"((j & 1) ? 0x10000u : 1u)
                   : "memory");
    }
  };
  auto add = [&](uint64_t x) {
    if (CODED) x = codec(x);
    add_word(uint32_t(x), 0);
    add_word(uint32_t(x >> 32), 1);
  };
  auto fold = [&]() {
    __syncthreads();
    for (int b = tid; b < 8 * 256; b += kHistThreads) {
      const int p = b >> 8, d = b & 255;
      const uint32_t* w = s_tab + ((p >> 1) * 256 + d) * 32;
      const int sh = (p & 1) * 16;
      uint32_t sum = 0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) sum += (w[(l + lane) & 31] >> sh) & 0xffffu;
      s_total[b] += sum;
    }
    __syncthreads();
    for (int i = tid; i < int(kHistU64Table / 4); i += kHistThreads) s_tab[i] = 0;
    __syncthreads();
  };

  const uint64_t* keys = static_cast<const uint64_t*>(P.keys);
  const size_t n = P.n;
  size_t head = ((16u - (reinterpret_cast<uintptr_t>(keys) & 15u)) & 15u) / 8;
  if (head > n) head = n;
  const size_t nvec = (n - head) / 2;
  const size_t tail = head + nvec * 2;
  const uint4* vp = reinterpret_cast<const uint4*>(keys + head);
  const size_t stride = size_t(gridDim.x) * kHistThreads;
  const size_t per_round = stride * kHistVec;
  const size_t rounds = (nvec + per_round - 1) / per_round;  // same for every block
  size_t v0 = size_t(blockIdx.x) * kHistThreads + tid;
  uint4 cur[kHistVec];
#pragma unroll
  for (int u = 0; u < kHistVec; ++u)
    if (v0 + u * stride < nvec) cur[u] = ld_stream_v4(vp + v0 + u * stride);
  for (size_t r = 0; r < rounds; ++r) {
    const size_t v1 = v0 + per_round;
    uint4 nxt[kHistVec];
#pragma unroll
    for (int u = 0; u < kHistVec; ++u)
      if (v1 + u * stride < nvec) nxt[u] = ld_stream_v4(vp + v1 + u * stride);
#pragma unroll
    for (int u = 0; u < kHistVec; ++u)
      if (v0 + u * stride < nvec) {
        add((uint64_t(cur[u].y) << 32) | cur[u].x);
        add((uint64_t(cur[u].w) << 32) | cur[u].z);
      }
#pragma unroll
    for (int u = 0; u < kHistVec; ++u) cur[u] = nxt[u];
    v0 = v1;
    if ((r + 1) % kU64FoldRounds == 0) fold();
  }
  const size_t g = size_t(blockIdx.x) * kHistThreads + tid;
  if (g < head) add(keys[g]);
  if (tail + g < n) add(keys[tail + g]);
  fold();
  for (int b = tid; b < 8 * 256; b += kHistThreads)
    if (s_total[b]) atomicAdd(&P.hist[b], (unsigned long long)s_total[b]);
  if (P.offsets == nullptr) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    s_last = (atomicAdd(P.done_counter, 1u) == gridDim.x - 1);
    s_trivial = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  scan_places256(P, 8, s_wsum, &s_trivial);
  if (tid == 0 && P.tickets != nullptr) plan_tickets(P.tickets, P.ticket_stride, P.strips, 8, s_trivial, P.fixed_ends != 0);
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

constexpr size_t kHistMaxSmem = 8 * 128 * 32 * 4 + 8 * 256 * 4 + 4096;

static int hist_grid() {
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = sms;
  }
  return grid;
}

template <typename K, int FIXED>
static cudaError_t launch_hist_t(const HistParams& p, cudaStream_t stream) {
  auto kern = onesweep_histogram_kernel<K, FIXED>;
  const size_t radix = size_t(1) << p.digit_bits;
  const size_t half = radix > 1 ? radix / 2 : 1;
  const size_t smem = (size_t(p.passes) * half * 32 + size_t(p.passes) * radix) * 4;
  static bool configured = false;
  if (!configured) {  // largest footprint: 8 places x 256 digits (u64 keys, d = 8) = 136 KiB
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kHistMaxSmem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (smem > kHistMaxSmem) return cudaErrorInvalidValue;
  kern<<<hist_grid(), kHistThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

template <bool CODED>
static cudaError_t launch_hist_u32d8(const HistParams& p, cudaStream_t stream) {
  auto kern = onesweep_histogram_u32d8_kernel<CODED>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kHistU32Smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<hist_grid(), kHistThreads, kHistU32Smem, stream>>>(p);
  return cudaGetLastError();
}

#ifndef OS_HIST_U64D8
#define OS_HIST_U64D8 1  // 0: 64-bit keys use the generic kernel
#endif
template <bool CODED>
static cudaError_t launch_hist_u64d8(const HistParams& p, cudaStream_t stream) {
  auto kern = onesweep_histogram_u64d8_kernel<CODED>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kHistU64Smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<hist_grid(), kHistThreads, kHistU64Smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_histogram(const HistParams& p, int key_bytes, cudaStream_t stream) {
  if (p.n == 0) return cudaSuccess;
  const bool full8 = p.digit_bits == 8 && p.top_bits == 8;
  if (key_bytes == 4) {
    if (full8 && p.passes == 4 && p.begin_bit == 0) {
      if (p.codec != CODEC_NONE) return launch_hist_u32d8<true>(p, stream);
      return launch_hist_u32d8<false>(p, stream);
    }
    return launch_hist_t<uint32_t, 0>(p, stream);
  }
  if (key_bytes == 8) {
    if (full8 && p.passes == 8 && p.begin_bit == 0 && OS_HIST_U64D8) {
      if (p.codec != CODEC_NONE) return launch_hist_u64d8<true>(p, stream);
      return launch_hist_u64d8<false>(p, stream);
    }
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
