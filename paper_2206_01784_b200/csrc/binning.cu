// Chained-scan digit-binning pass (one Onesweep partition pass) for sm_100a.
//
// Replaces, for one digit place and one strip, the reference's
//   partition_pass / process_tile      binning.py:162-275
//   rank_tile_kernel (WLMS)             _kernels.py:31-82
//   CounterMatrix publish / look-back   lookback.py:127-169
//   scatter_tile_kernel / slots kernel  _kernels.py:85-128
//   short-circuit fast path             binning.py:79-85,201-205
//   StripCarry write by the last tile   binning.py:196-198
// with one CUDA kernel in which a thread block processes one tile:
//
//   1. claim a tile id from an atomic ticket (forward progress for the
//      chained scan: ids are handed out in block-start order, executor.py:1-8)
//      and prefetch a tile further down the strip into L2;
//   2. stage the tile's keys (and values) into shared memory with one TMA bulk
//      copy each (cp.async.bulk ... mbarrier::complete_tx); values land while
//      the keys are ranked;
//   3. rank keys with a warp-level multisplit: eight ballots (one per digit
//      bit) give the same-digit peer mask, rank = warp running count + popc of
//      lower-or-equal peers -- the reference's WLMS (_kernels.py:56-82) on
//      VOTE/LOP3;
//   4. reduce per-warp digit counts to tile counts (thread d owns digit d,
//      PAPER.md:187), publish L|count, reorder the tile in place into
//      per-digit runs, then look back over predecessor status words and
//      publish G|inclusive;
//   5. write each run with coalesced stores at base + exclusive + (slot -
//      start); the codec (signed/float decode) is applied on the way out.
//
// Between ranking and reorder each thread parks its keys (and values) in its
// own TMEM lane (tcgen05.st / tcgen05.ld), which frees the registers that
// would hold them and lets four 10K-key tiles share an SM.
//
// The pass is SM-bound, not HBM-bound (profiles/round1_ncu_summary.md): the
// ranking loop is issue/ALU-bound, the reorder and run writes are bound by
// the shared-memory/L1 data pipe, where every digit-indexed table access by
// 32 random digits costs ~3 bank wavefronts.  The layout choices below trade
// instructions for wavefronts: 16-bit per-warp counters (two digits per bank
// word) and a 32-bit output-index table for the run writes.
//
// Keys move once in and once out: 2n element transfers per pass, the
// reference's ledger identity (binning.py:268-272).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace osb {

struct NoValue {};
template <typename V> struct ValTraits {
  static constexpr bool kHas = true;
  static constexpr int kBytes = sizeof(V);
};
template <> struct ValTraits<NoValue> {
  static constexpr bool kHas = false;
  static constexpr int kBytes = 0;
};

// Predecessor status words read per look-back round trip (lookback.py:144-169).
#ifndef OS_LOOKBACK_WINDOW
#define OS_LOOKBACK_WINDOW 6  // 16K tiles: 707 us (6, 8) vs 711 (4), 716 (3), 727 (2)
#endif
constexpr int kLookbackWindow = OS_LOOKBACK_WINDOW;
// Per-tile timeline records (os_debug_trace) are compiled in only for
// diagnostic builds (-DOS_TRACE=1); the product kernel carries no trace code.
#ifndef OS_TRACE
#define OS_TRACE 0
#endif
// The ranking loop orders each item's counter read before the leader's
// counter write, and that write before the next item's read.  The accesses
// are volatile, so they keep program order, and the warp is converged (no
// divergent branches in the loop), so they also execute in order.
// OS_SYNCWARP adds the formal __syncwarp() fences (bit 0: read -> leader write,
// bit 1: leader write -> next read; one NOP each).  Timing (round 2, 10K
// tiles, 3 interleaved runs): both 686 us, none 728; with the key prefetch
// both 659, none 705 -- the NOPs pay for themselves in the warp schedule.
// The read -> leader-write order is also a data dependency (the leader
// stores the rank its own load returned, and a converged warp's load returns
// for every lane at once), so bit 0 is redundant; bit 1 alone (session r2j,
// 3 interleaved runs): C2 663.0 -> 659.3 us/pass.
#ifndef OS_SYNCWARP
#define OS_SYNCWARP 2
#endif

// Skip the multisplit for warps whose 32*ITEMS keys share one digit.
#ifndef OS_UNIFORM_KEYS
#define OS_UNIFORM_KEYS 1  // keys-only passes take the uniform-warp shortcut too (tools/keys_dist.py)
#endif
#ifndef OS_UNIFORM_WARPS
#define OS_UNIFORM_WARPS 1
#endif
// 1: keys-only u32 passes park each thread's keys in TMEM between ranking and
// the reorder (no shared-memory re-read, fewer live registers).
#ifndef OS_TMEM_STASH
#define OS_TMEM_STASH 1
#endif
#ifndef OS_STATUS_KEEP
#define OS_STATUS_KEEP 0  // 1: status words carry an L2 evict_last policy (tools/gpu_status_l2.sh; 709 vs 707 us)
#endif
#ifndef OS_PDL
#define OS_PDL 0  // 1: programmatic dependent launch between passes (tools/size_sweep.py: no gain on plain sorts, -9 % at 16M keys)
#endif
#ifndef OS_STASH64
#define OS_STASH64 1  // 1: 64-bit keys are stashed in TMEM too (2 columns per key)
#endif
// Race exploration (the reference's Jitter, executor.py:108-121, applied
// between publish and look-back at binning.py:187-193): OS_JITTER=1 debug
// builds sleep a pseudo-random 0..OS_JITTER_NS ns (hash of tile, digit and
// a per-build seed) before the L publish, before the look-back and before
// the G publish, so tiles publish out of order and look-backs meet N words.
#ifndef OS_JITTER
#define OS_JITTER 0
#endif
#ifndef OS_JITTER_NS
#define OS_JITTER_NS 20000
#endif
#ifndef OS_JITTER_SEED
#define OS_JITTER_SEED 0x9E3779B9u
#endif
// Failure detection (the reference's aborting waiters, lookback.py:176-189):
// a look-back that re-polls one unpublished predecessor word more than
// OS_SPIN_LIMIT times traps (the launch fails with cudaErrorLaunchFailure /
// illegal instruction) instead of hanging the GPU.  A healthy pass waits a
// few microseconds; 2^26 re-polls is over a minute of L2 round trips.
// Back-off (ns) before re-polling an unpublished predecessor word: fewer
// issue slots burnt by spinning digit threads.
#ifndef OS_LB_BACKOFF
#define OS_LB_BACKOFF 0
#endif
#ifndef OS_SPIN_LIMIT
#define OS_SPIN_LIMIT (1u << 26)
#endif
__device__ __forceinline__ void jitter_sleep(uint32_t tile, uint32_t lane_id, uint32_t site) {
  if (OS_JITTER) {
    uint32_t h = tile * 0x9E3779B1u ^ (lane_id + 0x7F4A7C15u) * 0x85EBCA6Bu ^ site * 0xC2B2AE35u ^
                 uint32_t(OS_JITTER_SEED);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if ((h & 3u) != 0u) __nanosleep(h % uint32_t(OS_JITTER_NS));  // 3 in 4 threads sleep
  }
}

#ifndef OS_RANK_STASH
#define OS_RANK_STASH 0  // 1: keys-only passes park the packed ranks in TMEM too
#endif
// 1: the ranking loop takes each digit's running count with one shared-memory
// atomic by the digit's highest lane (old value broadcast with a shuffle)
// instead of a counter load by every lane plus a store by the leader; the
// per-warp counters are then 32-bit.
#ifndef OS_RANK_ATOMIC
#define OS_RANK_ATOMIC 0
#endif
// 1: one wave of resident blocks loops over the tiles (no per-tile block
// launch); 0: one block per tile (each block still loops, claiming once more
// to find the ticket exhausted)
#ifndef OS_PERSIST
#define OS_PERSIST 1
#endif
#ifndef OS_PERSIST_KEYS
#define OS_PERSIST_KEYS 0  // u32 keys-only passes (see Geometry<4, 0>)
#endif
#ifndef OS_PAIR_STS
#define OS_PAIR_STS 1
#endif
#ifndef OS_TMA_SLICES
#define OS_TMA_SLICES 1
#endif
#ifndef OS_KEEP_COUNTS
#define OS_KEEP_COUNTS 1  // the count phase keeps the per-warp counts in registers for the offset rewrite
#endif
#ifndef OS_COUNT_PAIRS
#define OS_COUNT_PAIRS 1  // the count phase works on digit pairs (one 32-bit counter word per thread)
#endif
// u32 keys with values: a __syncwarp() every k-th run-write slot paces each
// warp's loads / two stores per slot (session r2k, C3 q=1 / q=4 / q=16:
// 1024 / 949 / 805 -> 999 / 922 / 803 us/pass at k = 3; k = 1 loses at
// q=16; u32 keys + 1 / 2 / 8-byte values +0.4 / +1.9 / +1.4 %; keys-only and
// u64-key kernels do not gain: profiles/round2_binning_notes.md)
#ifndef OS_PAIR_WRITE_FENCE
#define OS_PAIR_WRITE_FENCE 3
#endif
#ifndef OS_KEY_PREFETCH
#define OS_KEY_PREFETCH 2  // k: the ranking loop loads item i+k's key while ranking item i (C2: k=0 686, 1 659, 2 657 us/pass)
#endif

constexpr int log2i(int n) { return n <= 1 ? 0 : 1 + log2i(n / 2); }

constexpr int kCounterBytes = OS_RANK_ATOMIC ? 4 : 2;  // per-warp digit counter width

template <int THREADS, int ITEMS, int KB, int VB>
struct BinningSmem {
  static constexpr int kTile = THREADS * ITEMS;
  static constexpr int kWarps = THREADS / 32;
  static constexpr size_t kKeys = size_t(kTile) * KB;
  static constexpr size_t kVals = (size_t(kTile) * VB + 15) / 16 * 16;
  // per-warp u16 digit counters, later the warp's slot offsets
  static constexpr size_t kHist = (size_t(kWarps) * kMaxRadix * kCounterBytes + 15) / 16 * 16;
  static constexpr size_t kPtr = kMaxRadix * 8;  // per-digit 64-bit output index (keys, values)
  static constexpr size_t kRel = kMaxRadix * 4;  // per-digit 32-bit output index
  static constexpr size_t kLocal = kMaxRadix * 4;  // tile-local digit starts
  static constexpr size_t kWsum = 32 * 4;
  static constexpr size_t kMap = kMaxRadix;
  static constexpr size_t kBytes = kKeys + kVals + kHist + kPtr + kRel + kLocal + kWsum + kMap;
};

template <typename K, typename V, int THREADS, int ITEMS, int MINB, bool MAPPED, bool CODED,
          bool BYTE, bool LOOP>
__global__ void __launch_bounds__(THREADS, MINB) onesweep_binning_kernel(const PassParams P) {
  constexpr bool HAS_V = ValTraits<V>::kHas;
  constexpr int KB = sizeof(K);
  using Smem = BinningSmem<THREADS, ITEMS, KB, ValTraits<V>::kBytes>;
  constexpr int TILE = Smem::kTile;
  constexpr int WARPS = Smem::kWarps;
  static_assert(THREADS >= kMaxRadix, "one thread per digit for the look-back");
  static_assert(THREADS % 32 == 0, "whole warps");
  static_assert(TILE * KB <= 65536, "u16 slot offsets");
  static_assert(32 * ITEMS * KB < 65536, "u16 scaled per-warp counters");
  using VS = typename std::conditional<HAS_V, V, uint32_t>::type;  // storage type
  constexpr int VB = HAS_V ? int(sizeof(VS)) : 0;
  // TMEM key stash: warp w owns lanes 32*(w%4).., columns (w/4)*ITEMS..
  // Values of 1, 2 or 4 bytes take one TMEM column each (zero-extended),
  // 8-byte values two, like 64-bit keys.
  constexpr bool STASH = OS_TMEM_STASH && (KB == 4 || (KB == 8 && OS_STASH64)) &&
                         (!HAS_V || VB <= 4 || (VB == 8 && OS_STASH64)) && ITEMS % 8 == 0 &&
                         WARPS % 4 == 0;
  constexpr int KW = KB / 4;                 // TMEM words per key
  constexpr int VW = HAS_V ? (VB == 8 ? 2 : 1) : 0;  // TMEM words per value
  constexpr int NW = KW + VW;                // stashed words per item: key (+ value)
  constexpr bool CPAIRS = OS_COUNT_PAIRS && kCounterBytes == 2 && THREADS * 2 >= kMaxRadix;
  // a digit's scaled tile total can reach 2^16 (8192 x 8 B tiles): sum the
  // two halves separately and mask the packed offsets
  constexpr bool WIDEPAIR = TILE * KB >= 65536;
  // u32 keys with u32 values, both stashed: the reorder writes (key, value)
  // pairs into the key + value buffers viewed as one 8-byte-slot array (one
  // STS.64 per item instead of two scattered STS.32), the run writes read
  // them back with one LDS.64 (OS_PAIR_STS)
  constexpr bool PAIRS = OS_PAIR_STS && STASH && KB == 4 && VB == 4 &&
                         Smem::kKeys == size_t(TILE) * 4 && Smem::kVals == size_t(TILE) * 4;
  // packed ranks (two u16 per word) parked next to the keys, 4 words per store
  constexpr bool RSTASH = OS_RANK_STASH && STASH && !HAS_V && KW == 1 && ITEMS % 8 == 0;
  constexpr int RW = RSTASH ? ITEMS / 2 : 0;
  constexpr uint32_t TCOLS_RAW = uint32_t(WARPS / 4) * (ITEMS * NW + RW);
  constexpr uint32_t TCOLS = TCOLS_RAW <= 32 ? 32 : TCOLS_RAW <= 64 ? 64 : TCOLS_RAW <= 128 ? 128
                           : TCOLS_RAW <= 256 ? 256 : 512;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* s_keys = reinterpret_cast<K*>(smem_raw);
  VS* s_vals = reinterpret_cast<VS*>(smem_raw + Smem::kKeys);
  using CT = typename std::conditional<kCounterBytes == 4, uint32_t, uint16_t>::type;
  CT* s_whist = reinterpret_cast<CT*>(smem_raw + Smem::kKeys + Smem::kVals);
  unsigned long long* s_ptr = reinterpret_cast<unsigned long long*>(
      smem_raw + Smem::kKeys + Smem::kVals + Smem::kHist);
  uint32_t* s_rel = reinterpret_cast<uint32_t*>(s_ptr + kMaxRadix);
  uint32_t* s_local = s_rel + kMaxRadix;
  uint32_t* s_wsum = s_local + kMaxRadix;
  uint8_t* s_map = reinterpret_cast<uint8_t*>(s_wsum + 32);

  __shared__ uint32_t s_tile;
  __shared__ const void* s_bases[4];  // tile's source keys / values, destination keys / values
  uint32_t s_bases_code = ~0u;        // (thread 0) route code s_bases was resolved for
  __shared__ int s_fast;
  __shared__ uint32_t s_reads, s_waits, s_rounds;
  // key-arrival barriers: one per warp slice when the tile is staged in
  // per-warp TMA slices (looping key-value kernels, OS_TMA_SLICES), so a
  // warp starts ranking as soon as its own keys have landed
  constexpr bool SLICE = OS_TMA_SLICES && LOOP;
  constexpr int KBARS = SLICE ? WARPS : 1;
  __shared__ __align__(8) uint64_t s_bar_k[KBARS];
  __shared__ __align__(8) uint64_t s_bar_v;
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int radix = P.radix;
  const int shift = P.shift;
  const uint32_t dmask = P.mask;
  // byte-aligned 8-bit digit: one PRMT picks it out of the right 32-bit word
  const uint32_t byte_sel = 0x4440u | uint32_t((shift & 31) >> 3);
  const bool hi_word = shift >= 32;
  const uint32_t smem_base = smem_u32(smem_raw);
  // multiply-add operands for the index arithmetic (see fma_u32): written as
  // mad.lo, ptxas keeps these as IMADs on the FMA pipe (742 vs 808 us/pass,
  // profiles/round1_binning_notes.md)
  constexpr uint32_t k_one = 1u, k_two = 2u, k_shl16 = 1u << 16, k_cw = uint32_t(kCounterBytes);
  // look-back status words (lookback.py:63-79), optionally kept in L2
  const uint64_t status_pol = OS_STATUS_KEEP ? l2_policy_evict_last() : 0ull;
  auto status_ld = [&](const uint32_t* a) -> uint32_t {
    return OS_STATUS_KEEP ? ld_relaxed_gpu_keep(a, status_pol) : ld_relaxed_gpu(a);
  };
  auto status_st = [&](uint32_t* a, uint32_t v) {
    if (OS_STATUS_KEEP)
      st_relaxed_gpu_keep(a, v, status_pol);
    else
      st_relaxed_gpu(a, v);
  };

  if (OS_PDL) grid_launch_dependents();  // the next pass may start its prologue
  if (STASH && warp == 0) tmem_alloc(&s_tmem, TCOLS);
  if (tid == 0) {
    for (int b = 0; b < KBARS; ++b) mbar_init(&s_bar_k[b], 1);
    mbar_init(&s_bar_v, 1);
    fence_mbar_init();
  }
  if (MAPPED) {
    for (int i = tid; i < kMaxRadix; i += THREADS) s_map[i] = P.digit_map[i];
  }
  if (STASH) tmem_fence_before_sync();
  __syncthreads();
  uint32_t taddr = 0;
  if (STASH) {
    tmem_fence_after_sync();
    taddr = s_tmem + ((uint32_t(warp & 3) * 32u) << 16) + uint32_t(warp >> 2) * (ITEMS * NW + RW);
  }
  // programmatic dependent launch: everything above overlaps the previous
  // pass's tail; its output (this pass's input) is complete after the wait
  if (OS_PDL) grid_dependency_wait();

  // Tile loop.  The grid is at most one wave of resident blocks
  // (launch_one), so a block takes tiles until the ticket runs past the
  // strip: no block launch/retire gap between tiles, and the TMEM columns and
  // barriers are set up once.  Tickets stay strictly increasing in claim
  // order, and every claimed tile belongs to a running block (forward
  // progress for the look-back).
  uint32_t k_phase = 0, v_phase = 0;  // mbarrier phase parities
  bool tmem_held = STASH;             // this block still owns its TMEM columns
  for (;;) {
  if (tid == 0) {
    const uint32_t word = atomicAdd(P.tile_counter, 1u);  // ticket + route code (plan_tickets)
    s_tile = word;
    const uint32_t c = word >> kTicketShift;
    if (c != s_bases_code) {  // this pass's buffer bases (the launch's own, or its route's)
      s_bases_code = c;       // (the same for every tile of a pass: set at the first claim)
      if (c == 0u || c == kTicketSkip) {
        s_bases[0] = P.src_keys;
        s_bases[1] = P.src_vals;
        s_bases[2] = P.dst_keys;
        s_bases[3] = P.dst_vals;
      } else {
        const uint32_t ix = (c - 1u) & 7u;
#pragma unroll
        for (int b = 0; b < 4; ++b) s_bases[b] = P.route_bases[ix][b];
      }
    }
    s_fast = -1;
    s_reads = s_waits = s_rounds = 0;
    // warm L2 with a tile that a block starting a few microseconds from now
    // will claim; its TMA then hits L2 instead of waiting on HBM
    const uint32_t pf = (word & kTicketMask) + P.prefetch_tiles;
    if (P.prefetch_tiles != 0 && pf + 1 < P.num_tiles && (word >> kTicketShift) != kTicketSkip) {
      const size_t off = size_t(pf) * P.tile_keys;
      const K* pk = static_cast<const K*>(s_bases[0]) + off;
      if ((reinterpret_cast<uintptr_t>(pk) & 15u) == 0 && ((P.tile_keys * KB) & 15u) == 0)
        l2_prefetch(pk, P.tile_keys * KB);
      if (HAS_V) {
        const VS* pv = static_cast<const VS*>(s_bases[1]) + off;
        if ((reinterpret_cast<uintptr_t>(pv) & 15u) == 0 && ((P.tile_keys * VB) & 15u) == 0)
          l2_prefetch(pv, P.tile_keys * VB);
      }
    }
  }
  {
    uint4* z = reinterpret_cast<uint4*>(s_whist);
    for (int i = tid; i < int(Smem::kHist / 16); i += THREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint32_t code = s_tile >> kTicketShift;
  const uint32_t tile = s_tile & kTicketMask;
  if (code == kTicketSkip) {  // skipped place: every tile is a one-run tile (binning.py:201-205)
    if (tile == 0 && tid == 0 && P.stats != nullptr) {
      atomicAdd(&P.stats[0], (unsigned long long)P.num_tiles);
      atomicAdd(&P.stats[2], (unsigned long long)P.num_tiles);
    }
    break;
  }
  if (tile >= P.num_tiles) break;
  const XorCodec<K> cin{K(P.cin_m0), K(P.cin_m1)};
  const uint32_t tile_start = tile * P.tile_keys;
  const uint32_t valid = min(P.tile_keys, P.strip_n - tile_start);
  const bool full = valid == uint32_t(TILE);
  const K* gk = static_cast<const K*>(s_bases[0]) + tile_start;
  const VS* gv = HAS_V ? static_cast<const VS*>(s_bases[1]) + tile_start : nullptr;
  unsigned long long* trace =
      (OS_TRACE && P.trace) ? P.trace + size_t(tile) * kTraceWords : nullptr;
  if (OS_TRACE && trace && tid == 0) {
    trace[0] = global_ns();
    trace[6] = smid();
  }

  // ---- 2. TMA bulk stage ----------------------------------------------------
  const bool tma_k = ((reinterpret_cast<uintptr_t>(gk) & 15u) == 0) &&
                     (((valid * sizeof(K)) & 15u) == 0);
  bool tma_v = false;
  if (HAS_V)
    tma_v = ((reinterpret_cast<uintptr_t>(gv) & 15u) == 0) && (((valid * sizeof(VS)) & 15u) == 0);
  if (tid == 0) {
    if (tma_k) {
      if (SLICE && full) {
        constexpr uint32_t kSlice = uint32_t(ITEMS) * 32u * uint32_t(sizeof(K));
        const uint64_t pol = l2_policy_evict_first();
        for (int b = 0; b < KBARS; ++b) {
          mbar_arrive_expect_tx(&s_bar_k[b], kSlice);
          tma_bulk_g2s_hint(s_keys + b * ITEMS * 32, gk + b * ITEMS * 32, kSlice, &s_bar_k[b], pol);
        }
      } else {
        mbar_arrive_expect_tx(&s_bar_k[0], valid * sizeof(K));
        tma_bulk_g2s_hint(s_keys, gk, valid * sizeof(K), &s_bar_k[0], l2_policy_evict_first());
        for (int b = 1; b < KBARS; ++b) mbar_arrive(&s_bar_k[b]);  // every barrier completes a phase
      }
    }
    if (HAS_V && tma_v) {
      mbar_arrive_expect_tx(&s_bar_v, valid * sizeof(VS));
      tma_bulk_g2s(s_vals, gv, valid * sizeof(VS), &s_bar_v);
    }
  }

  // Warp-striped ownership: warp w owns tile positions [w*ITEMS*32, (w+1)*ITEMS*32),
  // item i / lane l is position w*ITEMS*32 + i*32 + l.  Ranking walks items in
  // that order, so ranks are stable (binning.py:71-76).  Ragged or misaligned
  // tiles are copied by the threads that will rank them (no barrier needed).
  const uint32_t warp_base = uint32_t(warp) * (ITEMS * 32);
  if (!tma_k) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = warp_base + i * 32 + lane;
      if (idx < valid) s_keys[idx] = gk[idx];
    }
  }
  if (HAS_V && !tma_v) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = warp_base + i * 32 + lane;
      if (idx < valid) s_vals[idx] = gv[idx];
    }
  }
  if (tma_k) {
    if (SLICE && full)
      mbar_wait_parity(&s_bar_k[__shfl_sync(0xffffffffu, warp, 0)], k_phase);
    else
      mbar_wait_parity(&s_bar_k[0], k_phase);
    k_phase ^= 1u;
  }
  asm volatile("" ::: "memory");  // the copies above before the (volatile) key loads below
  if (OS_TRACE && trace && tid == 0) trace[1] = global_ns();

  auto digit = [&](K x) -> uint32_t {  // x is an encoded key
    uint32_t d;
    if (BYTE) {
      uint32_t w;
      if constexpr (sizeof(K) == 8)
        w = hi_word ? uint32_t(uint64_t(x) >> 32) : uint32_t(x);
      else
        w = uint32_t(x);
      d = __byte_perm(w, 0u, byte_sel);
    } else {
      d = digit_of(x, shift, dmask);
    }
    if (MAPPED) d = s_map[d];
    return d;
  };

  // ---- 3. warp-level multisplit ranking -------------------------------------
  // Counters and ranks are 16-bit, pre-scaled by the key width and inclusive
  // (the key's own slot is counted): the highest peer stores its rank as the
  // digit's new running count, and warp offset + rank - KB is the byte offset
  // of the key's slot.  Positions past `valid` (ragged last tile) take the
  // largest digit: they sit after every real key, so they never perturb a
  // real key's rank, and their count is removed from the top digit before
  // publishing.
  K keys[STASH ? 1 : ITEMS];        // encoded keys, kept for the reorder
  uint32_t kc[8];                   // TMEM stash chunk (keys)
  uint32_t vc[8];                   // TMEM stash chunk (values)
  // keys go to columns [0, ITEMS*KW) of the warp's range, 8 words per store
  auto stash_key = [&](int i, K x) {
    if constexpr (KW == 1) {
      kc[i & 7] = uint32_t(x);
      if ((i & 7) == 7) tmem_st8(taddr + uint32_t(i - 7), kc);
    } else {
      kc[2 * (i & 3)] = uint32_t(uint64_t(x));
      kc[2 * (i & 3) + 1] = uint32_t(uint64_t(x) >> 32);
      if ((i & 3) == 3) tmem_st8(taddr + uint32_t(2 * (i - 3)), kc);
    }
  };
  auto unstash_key = [&](int i) -> K {
    if constexpr (KW == 1) {
      if ((i & 7) == 0) tmem_ld8(taddr + uint32_t(i), kc);
      return K(kc[i & 7]);
    } else {
      if ((i & 3) == 0) tmem_ld8(taddr + uint32_t(2 * i), kc);
      return K(uint64_t(kc[2 * (i & 3)]) | (uint64_t(kc[2 * (i & 3) + 1]) << 32));
    }
  };
  uint32_t ranks[RSTASH ? 4 : (ITEMS + 1) / 2];  // two u16 scaled ranks per register
  const uint32_t rbase = taddr + uint32_t(ITEMS * NW);  // rank columns (RSTASH)
  // rank of item i: even items in the low half-word, odd items in the high
  auto put_rank = [&](int i, uint32_t rank) {
    const int w = RSTASH ? (i / 2) & 3 : i / 2;
    if (i & 1)
      ranks[w] = fma_u32(rank, k_shl16, ranks[w]);
    else
      ranks[w] = rank;
    if constexpr (RSTASH) {
      if ((i & 7) == 7 || i == ITEMS - 1) tmem_st4(rbase + uint32_t((i / 8) * 4), ranks);
    }
  };
  auto get_rank = [&](int i) -> uint32_t {
    if constexpr (RSTASH) {
      if ((i & 7) == 0) tmem_ld4(rbase + uint32_t((i / 8) * 4), ranks);
    }
    const int w = RSTASH ? (i / 2) & 3 : i / 2;
    return (i & 1) ? (ranks[w] >> 16) : (ranks[w] & 0xffffu);
  };
  const uint32_t hbase = smem_u32(s_whist) + uint32_t(warp) * (kMaxRadix * kCounterBytes);
  auto rank_items = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
    const uint32_t lt = lanemask_lt();
    const uint32_t le = lt | (1u << lane);
    // next item's key, loaded one item ahead (volatile: issued before this
    // item's counter read, so the load latency overlaps the ballots)
    constexpr int PF = OS_KEY_PREFETCH > 0 ? OS_KEY_PREFETCH : 1;
    [[maybe_unused]] K xq[PF];
    if (OS_KEY_PREFETCH) {
#pragma unroll
      for (int j = 0; j < PF; ++j) xq[j] = lds_key<K>(smem_base + (warp_base + j * 32 + lane) * KB);
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = warp_base + i * 32 + lane;
      K xraw;
      if (OS_KEY_PREFETCH) {
        xraw = xq[i % PF];
        if (i + PF < ITEMS) xq[i % PF] = lds_key<K>(smem_base + (idx + 32 * PF) * KB);
      } else {
        xraw = s_keys[idx];
      }
      const K x = CODED ? cin(xraw) : xraw;
      if constexpr (STASH) stash_key(i, x);
      uint32_t d;
      if (FULL)
        d = digit(x);
      else
        d = idx < valid ? digit(x) : uint32_t(radix - 1);
      uint32_t upto;
      bool leader;
      if constexpr (OS_RANK_ATOMIC) {
        // the highest lane of each digit adds the digit's count and gets the
        // running count before this item; its peers take it by shuffle
        uint32_t peers;
        match_rank8_peers(d, le, &upto, &peers);
        const uint32_t src = 31u - __clz(peers);
        const uint32_t cnt = __popc(upto) * KB;
        uint32_t old = 0;
        if (src == uint32_t(lane)) old = atoms_add_u32(fma_u32(d, k_cw, hbase), cnt);
        old = __shfl_sync(0xffffffffu, old, src);
        put_rank(i, old + cnt);
        if (OS_SYNCWARP & 2) __syncwarp();
      } else {
        match_rank8(d, le, ~le, &upto, &leader);
        const uint32_t caddr = fma_u32(d, k_two, hbase);
        const uint32_t rank = lds_u16(caddr) + __popc(upto) * KB;
        put_rank(i, rank);
        if (OS_SYNCWARP & 1) __syncwarp();
        if (leader) sts_u16(caddr, rank);
        if (OS_SYNCWARP & 2) __syncwarp();
      }
    }
  };
  // A warp whose keys all carry one digit needs no multisplit: its inclusive
  // ranks are the positions themselves.  Test cheaply first (first and last
  // item), then every item; uniform keys fail the first test at once, while
  // low-entropy and presorted inputs skip the ballots for most warps.
  // Key-value passes always take it; keys-only passes take it when
  // OS_UNIFORM_KEYS is set (the default: tools/keys_dist.py measured all-equal
  // keys +21 % and uniform keys -1 % at 2^28, profiles/round1_binning_notes.md).
  bool uniform_warp = false;
  if (OS_UNIFORM_WARPS && (HAS_V || OS_UNIFORM_KEYS) && full) {
    const K xa = CODED ? cin(s_keys[warp_base + lane]) : s_keys[warp_base + lane];
    const K xb = CODED ? cin(s_keys[warp_base + (ITEMS - 1) * 32 + lane])
                       : s_keys[warp_base + (ITEMS - 1) * 32 + lane];
    const uint32_t d0 = __shfl_sync(0xffffffffu, digit(xa), 0);
    if (__all_sync(0xffffffffu, digit(xa) == d0 && digit(xb) == d0)) {
      bool same = true;
#pragma unroll
      for (int i = 1; i < ITEMS - 1; ++i) {
        const K x = CODED ? cin(s_keys[warp_base + i * 32 + lane]) : s_keys[warp_base + i * 32 + lane];
        same &= digit(x) == d0;
      }
      uniform_warp = __all_sync(0xffffffffu, same);
      if (uniform_warp) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) put_rank(i, uint32_t(i * 32 + lane + 1) * KB);
        if (lane == 0) {
          if constexpr (kCounterBytes == 4)
            sts_u32(hbase + d0 * 4u, uint32_t(ITEMS * 32 * KB));
          else
            sts_u16(hbase + d0 * 2u, uint32_t(ITEMS * 32 * KB));
        }
        if constexpr (STASH) {  // the keys still go to the stash
#pragma unroll
          for (int i = 0; i < ITEMS; ++i) {
            const K x = s_keys[warp_base + i * 32 + lane];
            stash_key(i, CODED ? cin(x) : x);
          }
        }
      }
    }
  }
  if (!uniform_warp) {
    if (full)
      rank_items(std::true_type{});
    else
      rank_items(std::false_type{});
  }
  if (STASH) tmem_wait_st();
  __syncthreads();

  // ---- 4a. tile counts, publish L, local digit starts ------------------------
  uint32_t count = 0;
  uint32_t local_start = 0;
  if constexpr (CPAIRS) {
    // Digit pairs (OS_COUNT_PAIRS): thread t < ceil(radix / 2) owns digits 2t
    // and 2t + 1, which share one 32-bit word of every per-warp counter
    // table (u16 halves, each at most 40960 = tile x key width, so packed
    // sums and offsets never carry across the halves): half the shared
    // loads and stores of one thread per digit, and half the scan.  Each
    // digit's (count, local start) goes to s_local for its look-back thread.
    const int d0 = 2 * tid, d1 = 2 * tid + 1;
    const bool owner = d0 < radix, has1 = d1 < radix;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(s_whist);
    uint32_t wk[WARPS];
    uint32_t c0 = 0, c1 = 0;
    if (owner) {
      uint32_t sum = 0, sum_hi = 0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        wk[w] = w32[w * (kMaxRadix / 2) + tid];
        if constexpr (WIDEPAIR) {
          sum += wk[w] & 0xffffu;
          sum_hi += wk[w] >> 16;
        } else {
          sum += wk[w];
        }
      }
      if constexpr (WIDEPAIR) {
        c0 = sum / KB;
        c1 = sum_hi / KB;
      } else {
        c0 = (sum & 0xffffu) / KB;
        c1 = (sum >> 16) / KB;
      }
      if (d0 == radix - 1) c0 -= uint32_t(TILE) - valid;
      if (d1 == radix - 1) c1 -= uint32_t(TILE) - valid;
      if (P.rts_offsets == nullptr) {  // (reduce-then-scan passes have no look-back)
        const uint32_t flag = tile == 0 ? kFlagGlobal : kFlagLocal;
        if (OS_JITTER) jitter_sleep(tile, d0, 1);
        if (!OS_JITTER || int(tile) != P.debug_stall_tile) {
          status_st(P.status + size_t(tile) * radix + d0, flag | c0);
          if (has1) status_st(P.status + size_t(tile) * radix + d1, flag | c1);
        }
      }
      if (c0 == valid) s_fast = d0;
      if (has1 && c1 == valid) s_fast = d1;
    }
    if (OS_TRACE && trace && tid == 0) trace[2] = global_ns();
    const uint32_t pair = c0 + c1;
    uint32_t incl = pair;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31 && warp < kMaxRadix / 64) s_wsum[warp] = incl;
    __syncthreads();
    if (owner) {
      uint32_t wpre = 0;
#pragma unroll
      for (int w = 0; w < kMaxRadix / 64; ++w) wpre += (w < warp) ? s_wsum[w] : 0u;
      const uint32_t ls0 = wpre + incl - pair, ls1 = ls0 + c0;
      s_local[d0] = ls0 | (c0 << 16);  // (counts and starts are below 2^16)
      if (has1) s_local[d1] = ls1 | (c1 << 16);
      // fold the tile-local starts into every warp's counters, so the
      // reorder needs a single shared-memory gather per key
      uint32_t* o32 = reinterpret_cast<uint32_t*>(s_whist);
      if constexpr (WIDEPAIR) {
        uint32_t run0 = ls0 * KB, run1 = ls1 * KB;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {  // (an unused entry may reach 2^16: masked)
          o32[w * (kMaxRadix / 2) + tid] = (run0 & 0xffffu) | (run1 << 16);
          run0 += wk[w] & 0xffffu;
          run1 += wk[w] >> 16;
        }
      } else {
        uint32_t run = (ls0 * KB) | ((ls1 * KB) << 16);
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
          o32[w * (kMaxRadix / 2) + tid] = run;
          run += wk[w];
        }
      }
    }
  } else {
  // per-warp counts of this thread's digit, two u16 per register, kept for
  // the offset rewrite below (OS_KEEP_COUNTS; else re-read)
  constexpr bool KEEPC = OS_KEEP_COUNTS && kCounterBytes == 2;
  uint32_t cpk[KEEPC ? (WARPS + 1) / 2 : 1];
  if (tid < radix) {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = s_whist[w * kMaxRadix + tid];
      sum += c;
      if constexpr (KEEPC) {
        if (w & 1)
          cpk[w / 2] |= c << 16;
        else
          cpk[w / 2] = c;
      }
    }
    count = sum / KB;
    if (tid == radix - 1) count -= uint32_t(TILE) - valid;
    if (P.rts_offsets == nullptr) {  // (reduce-then-scan passes have no look-back)
      if (OS_JITTER) jitter_sleep(tile, tid, 1);
      if (!OS_JITTER || int(tile) != P.debug_stall_tile)
        status_st(P.status + size_t(tile) * radix + tid,
                  (tile == 0 ? kFlagGlobal : kFlagLocal) | count);
    }
    if (count == valid) s_fast = tid;
  }
  if (OS_TRACE && trace && tid == 0) trace[2] = global_ns();
  // block-wide exclusive scan of counts over digits (first 8 warps)
  uint32_t incl = count;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31 && warp < kMaxRadix / 32) s_wsum[warp] = incl;
  __syncthreads();
  if (tid < radix) {
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kMaxRadix / 32; ++w) wpre += (w < warp) ? s_wsum[w] : 0u;
    local_start = wpre + incl - count;
    s_local[tid] = local_start;
    // fold the tile-local start into every warp's counter, so the reorder
    // needs a single shared-memory gather per key
    uint32_t run = local_start * KB;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = KEEPC ? ((cpk[w / 2] >> (16 * (w & 1))) & 0xffffu) : uint32_t(s_whist[w * kMaxRadix + tid]);
      s_whist[w * kMaxRadix + tid] = CT(run);
      run += c;
    }
  }
  }
  // keys and values into registers; after the barrier the tile buffers are
  // rewritten in place as per-digit runs
  if constexpr (!STASH) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const K x = s_keys[warp_base + i * 32 + lane];
      keys[i] = CODED ? cin(x) : x;
    }
  }
  VS vals[HAS_V && !STASH ? ITEMS : 1];
  if (HAS_V) {
    if (tma_v) {
      mbar_wait_parity(&s_bar_v, v_phase);
      v_phase ^= 1u;
    }
    if constexpr (STASH) {  // values to the stash, next to the keys
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if constexpr (VW == 2) {
          const uint64_t v = uint64_t(s_vals[warp_base + i * 32 + lane]);
          kc[2 * (i & 3)] = uint32_t(v);
          kc[2 * (i & 3) + 1] = uint32_t(v >> 32);
          if ((i & 3) == 3) tmem_st8(taddr + uint32_t(ITEMS * KW + 2 * (i - 3)), kc);
        } else {
          kc[i & 7] = uint32_t(s_vals[warp_base + i * 32 + lane]);
          if ((i & 7) == 7) tmem_st8(taddr + uint32_t(ITEMS * KW + i - 7), kc);
        }
      }
      tmem_wait_st();
    } else {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) vals[i] = s_vals[warp_base + i * 32 + lane];
    }
  }
  __syncthreads();
  const int fast = s_fast;

  // ---- 5a. local reorder into per-digit runs (needs no global offsets, so it
  // runs before the look-back and gives predecessors time to publish) ---------
  if (fast < 0) {
    const uint32_t slot0 = smem_base - KB;  // inclusive ranks start at KB
    auto stage = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (STASH && HAS_V && VW == 1 && (i & 7) == 0) tmem_ld8(taddr + uint32_t(ITEMS * KW + i), vc);
        if (STASH && HAS_V && VW == 2 && (i & 3) == 0) tmem_ld8(taddr + uint32_t(ITEMS * KW + 2 * i), vc);
        K key;
        if constexpr (STASH)
          key = unstash_key(i);
        else
          key = keys[i];
        const uint32_t r = get_rank(i);  // (a warp-collective TMEM load under RSTASH)
        if (!FULL && warp_base + i * 32 + lane >= valid) continue;
        uint32_t off;
        if constexpr (kCounterBytes == 4)
          off = lds_u32(fma_u32(digit(key), k_cw, hbase));
        else
          off = lds_u16(fma_u32(digit(key), k_two, hbase));
        const uint32_t addr = fma_u32(off, k_one, fma_u32(r, k_one, slot0));
        if constexpr (PAIRS) {  // slot s of the pair array at byte 8 s
          asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(fma_u32(addr - smem_base, k_two, smem_base)),
                       "r"(uint32_t(key)), "r"(vc[i & 7]));
          continue;
        }
        sts_val(addr, key);
        if (HAS_V) {
          constexpr int kSh = log2i(KB);
          constexpr int vSh = log2i(VB > 0 ? VB : 1);
          const uint32_t slot = (addr - smem_base) >> kSh;
          VS val;
          if constexpr (STASH && VW == 2)
            val = VS(uint64_t(vc[2 * (i & 3)]) | (uint64_t(vc[2 * (i & 3) + 1]) << 32));
          else if constexpr (STASH)
            val = VS(vc[i & 7]);
          else
            val = vals[i];
          sts_val(smem_base + uint32_t(Smem::kKeys) + (slot << vSh), val);
        }
      }
    };
    if (full)
      stage(std::true_type{});
    else
      stage(std::false_type{});
  }

  if (OS_TRACE && trace && tid == 0) trace[3] = global_ns();
  // ---- 4b. decoupled look-back (lookback.py:144-169) ------------------------
  // kLookbackWindow predecessor words per round trip; stop at the first G,
  // re-poll a predecessor that has not published yet.  Then publish G and the
  // per-digit output indices.
  if (tid < radix) {
    if constexpr (CPAIRS) {  // this digit's (count, local start) from the count phase
      const uint32_t cl = s_local[tid];
      count = cl >> 16;
      local_start = cl & 0xffffu;
    }
    uint32_t excl = 0;
    uint32_t reads = 0, waits = 0, rounds = 0;
    if (OS_JITTER) jitter_sleep(tile, tid, 2);
    if (tile > 0 && P.rts_offsets == nullptr) {
      uint32_t spins = 0;
      // p walks down the digit's column; 8-bit places have a compile-time row
      // stride, so the window's loads are one base register plus immediates
      const size_t stride = BYTE ? size_t(kMaxRadix) : size_t(radix);
      const uint32_t* p = P.status + size_t(tile - 1) * stride + tid;
      int j = int(tile) - 1;
      bool done = false;
      while (!done) {
        uint32_t w[kLookbackWindow];
        if (j >= kLookbackWindow - 1) {
#pragma unroll
          for (int k = 0; k < kLookbackWindow; ++k) w[k] = status_ld(p - k * stride);
        } else {
#pragma unroll
          for (int k = 0; k < kLookbackWindow; ++k)
            w[k] = (j - k >= 0) ? status_ld(p - k * stride) : kFlagGlobal;
        }
        reads += kLookbackWindow;
        ++rounds;
        int k = 0;
#pragma unroll
        for (; k < kLookbackWindow; ++k) {
          const uint32_t st = w[k] >> kStatusShift;
          if (st == 0u) {  // predecessor in flight: re-poll from here
            ++waits;
            if (OS_LB_BACKOFF > 0) __nanosleep(OS_LB_BACKOFF);
            if (++spins > OS_SPIN_LIMIT) {
              printf("onesweep: look-back stalled (tile %u digit %d waits on tile %d)\n", tile, tid,
                     j - k);
              __trap();
            }
            break;
          }
          excl += w[k] & kValueMask;
          if (st == 2u) {
            done = true;
            break;
          }
        }
        j -= k;
        p -= k * stride;
      }
      if (OS_JITTER) jitter_sleep(tile, tid, 3);
      if (!OS_JITTER || int(tile) != P.debug_stall_tile)
        status_st(P.status + size_t(tile) * radix + tid, kFlagGlobal | (excl + count));
    }
    if (OS_TRACE && trace && tid == 0) trace[4] = global_ns();
    // reduce-then-scan ablation (rts.cu): the tile's run starts come from the
    // precomputed digit-major prefix table instead of a look-back
    const unsigned long long gbase = P.rts_offsets != nullptr
                                         ? P.rts_offsets[size_t(tile) * radix + tid]
                                         : P.base_offsets[tid] + excl;
    const unsigned long long rel = gbase - local_start;  // modular: slot >= local_start
    s_ptr[tid] = rel;
    s_rel[tid] = uint32_t(rel);
    if (P.carry_out != nullptr && tile == P.num_tiles - 1) P.carry_out[tid] = gbase + count;
    if (P.tile_status != nullptr)  // final word in the reference's CounterMatrix format
      P.tile_status[size_t(tile) * radix + tid] = kFlagGlobal | (excl + count);
    if (P.stats != nullptr) {
      atomicAdd(&s_reads, reads);
      atomicAdd(&s_waits, waits);
      atomicAdd(&s_rounds, rounds);
    }
  }
  // The destination is read before the barrier: after it, a looping block's
  // thread 0 may claim the next tile (and rewrite s_tile / s_bases) while
  // slower warps are still writing this one.
  K* const dst_k = static_cast<K*>(const_cast<void*>(s_bases[2]));
  VS* const dst_v = static_cast<VS*>(const_cast<void*>(s_bases[3]));
  if (!LOOP && STASH) tmem_fence_before_sync();
  __syncthreads();
  if (!LOOP && STASH && warp == 0) {  // one tile per block: free the columns early
    tmem_fence_after_sync();
    tmem_dealloc(s_tmem, TCOLS);
  }
  tmem_held = LOOP;

  const XorCodec<K> cout{K(P.cout_m0), K(P.cout_m1)};
  if (fast >= 0) {
    // ---- short circuit: homogeneous tile is one contiguous run --------------
    const unsigned long long base = s_ptr[fast];  // local start is 0
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t idx = warp_base + i * 32 + lane;
      if (idx < valid) {
        const K key = STASH ? (CODED ? cin(s_keys[idx]) : s_keys[idx]) : keys[STASH ? 0 : i];
        st_global(elem_at(dst_k, base + idx), CODED ? cout(key) : key);
        if (HAS_V) st_global(elem_at(dst_v, base + idx), STASH ? s_vals[idx] : vals[STASH ? 0 : i]);
      }
    }
  } else if (!P.wide_index) {
    // ---- 5b. coalesced run writes: slot s of digit d lands at rel[d] + s ----
    // (output indices below 2^32: one 32-bit table entry per digit)
    auto write_slot = [&](uint32_t s) {
      if constexpr (PAIRS) {
        uint32_t x, v;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(x), "=r"(v) : "r"(smem_base + s * 8u));
        const uint32_t at = fma_u32(s_rel[digit(K(x))], k_one, s);
        st_global_cs(reinterpret_cast<uint32_t*>(dst_k + at), uint32_t(CODED ? cout(K(x)) : K(x)));
        st_global(reinterpret_cast<uint32_t*>(dst_v + at), v);
        return;
      }
      const K x = s_keys[s];
      const uint32_t at = fma_u32(s_rel[digit(x)], k_one, s);
      if constexpr (sizeof(K) == 4)
        st_global_cs(reinterpret_cast<uint32_t*>(dst_k + at), uint32_t(CODED ? cout(x) : x));
      else
        st_global(dst_k + at, CODED ? cout(x) : x);
      if (HAS_V) st_global(dst_v + at, s_vals[s]);
    };
    if (full) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j) {
        write_slot(uint32_t(j * THREADS + tid));
        // (u32 keys with values: a warp fence every OS_PAIR_WRITE_FENCE slots, see its definition)
        if (HAS_V && KB == 4 && OS_PAIR_WRITE_FENCE > 0 &&
            j % (OS_PAIR_WRITE_FENCE > 0 ? OS_PAIR_WRITE_FENCE : 1) == 0)
          __syncwarp();
        // (u64 keys with 8-byte values: every second slot, 18.34 -> 18.65 GKey/s)
        if (HAS_V && KB == 8 && VB == 8 && j % 2 == 0) __syncwarp();
      }
    } else {
      for (uint32_t s = tid; s < valid; s += THREADS) write_slot(s);
    }
  } else {
    for (uint32_t s = tid; s < valid; s += THREADS) {
      K x;
      VS v{};
      if constexpr (PAIRS) {
        uint32_t a, b;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(smem_base + s * 8u));
        x = K(a);
        v = VS(b);
      } else {
        x = s_keys[s];
        if (HAS_V) v = s_vals[s];
      }
      const unsigned long long at = s_ptr[digit(x)] + s;
      st_global(elem_at(dst_k, at), CODED ? cout(x) : x);
      if (HAS_V) st_global(elem_at(dst_v, at), v);
    }
  }
  if (OS_TRACE && trace && tid == 0) trace[5] = global_ns();

  if (P.stats != nullptr && tid == 0) {
    if (fast >= 0) atomicAdd(&P.stats[0], 1ull);
    atomicAdd(&P.stats[1], (unsigned long long)s_reads);
    atomicAdd(&P.stats[2], 1ull);
    atomicAdd(&P.stats[3], (unsigned long long)s_waits);
    atomicAdd(&P.stats[4], (unsigned long long)s_rounds);
  }
  if (!LOOP) break;
  // the next tile's TMA (async proxy) overwrites the tile buffers this tile
  // read and wrote through the generic proxy; the barrier at the top of the
  // loop orders them after this fence
  fence_proxy_async_smem();
  if (STASH) tmem_fence_before_sync();
  }  // tile loop
  // (a one-tile block that met a skipped place or an exhausted ticket at
  // its claim still holds its columns)
  if (STASH && tmem_held && warp == 0) {
    tmem_fence_after_sync();
    tmem_dealloc(s_tmem, TCOLS);
  }
}

// ---- host side ------------------------------------------------------------------

template <typename K, typename V, int THREADS, int ITEMS, int MINB, bool MAPPED, bool CODED,
          bool BYTE, bool LOOP>
static cudaError_t launch_one(const PassParams& p, cudaStream_t stream) {
  using Smem = BinningSmem<THREADS, ITEMS, sizeof(K), ValTraits<V>::kBytes>;
  auto kern = onesweep_binning_kernel<K, V, THREADS, ITEMS, MINB, MAPPED, CODED, BYTE, LOOP>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Smem::kBytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (p.num_tiles == 0) return cudaSuccess;
  // One wave: MINB blocks per SM, the residency every geometry is sized for
  // (registers by the launch bounds, shared memory and TMEM columns by
  // BinningSmem / TCOLS).  cudaOccupancyMaxActiveBlocksPerMultiprocessor
  // reports 1 for these kernels, so it is not used.  A wave larger than what
  // is resident would only leave blocks that start late and find the ticket
  // exhausted.
  static unsigned wave = 0;
  if (wave == 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    wave = unsigned(sms * MINB);
  }
  const unsigned grid = LOOP ? (p.num_tiles < wave ? p.num_tiles : wave) : p.num_tiles;
  if (OS_PDL) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Smem::kBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  kern<<<grid, THREADS, Smem::kBytes, stream>>>(p);
  return cudaGetLastError();
}

// Tile geometry per (key, value) width: THREADS x ITEMS keys per tile, MINB
// resident blocks per SM.  Small blocks with many keys per thread keep three
// or four tiles per SM in flight, which hides the TMA and look-back latencies
// of each (measured in profiles/round1_binning_notes.md).
template <int KB, int VB> struct Geometry;
#ifndef OS_U32_THREADS
#define OS_U32_THREADS 256
#endif
#ifndef OS_U32_ITEMS
#define OS_U32_ITEMS 40  // 10240-key tiles at 4 blocks/SM: 693 us vs 706 (256 x 64 x 3), 749 (48 x 4)
#endif
#ifndef OS_U32_MINB
#define OS_U32_MINB 4
#endif
// P: persistent tile loop (one wave of blocks) or one tile per block.  The
// loop keeps its carried state in registers, which the 64-register keys-only
// kernel cannot spare (spills: 734-765 vs 662 us/pass at C2); the key-value
// kernels gain (C3 q=1 1086 -> 1071, q=16 906 -> 806, C4 1463 -> 1428 us/pass).
template <> struct Geometry<4, 0> {
  static constexpr int T = OS_U32_THREADS, I = OS_U32_ITEMS, B = OS_U32_MINB;
  static constexpr bool P = OS_PERSIST_KEYS;
};
// Geometries of the other (key, value) widths, values stashed in TMEM like
// C3/C4 (tools/value_widths.py, profiles/round2_binning_notes.md): 1.2-1.7x
// the round-1 512-thread geometries.
#ifndef OS_S32_T  // u32 keys with 1- or 2-byte values: 54.2 / 52.6 -> 66.6 / 63.7 GKey/s
#define OS_S32_T 256
#define OS_S32_I 32
#define OS_S32_B 3
#endif
#ifndef OS_W32_T  // u32 keys with 8-byte values (numpy's int64 arange payload): 33.6 -> 46.2
#define OS_W32_T 256
#define OS_W32_I 32
#define OS_W32_B 2
#endif
#ifndef OS_N64_T  // u64 keys, no values: 19.4 -> 32.2
#define OS_N64_T 256
#define OS_N64_I 32
#define OS_N64_B 3
#endif
#ifndef OS_S64_T  // u64 keys with 1- or 2-byte values: 16.8 / 16.4 -> 24.5 / 23.8
#define OS_S64_T 256
#define OS_S64_I 32
#define OS_S64_B 2
#endif
#ifndef OS_W64_T  // u64 keys with 8-byte values: 14.8 -> 18.4
#define OS_W64_T 256
#define OS_W64_I 24
#define OS_W64_B 2
#endif
#ifndef OS_B32_T  // u32 keys with 1-byte values: four blocks fit (66.6 -> 68.0 GKey/s)
#define OS_B32_T 256
#define OS_B32_I 32
#define OS_B32_B 4
#endif
template <> struct Geometry<4, 1> { static constexpr int T = OS_B32_T, I = OS_B32_I, B = OS_B32_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<4, 2> { static constexpr int T = OS_S32_T, I = OS_S32_I, B = OS_S32_B; static constexpr bool P = OS_PERSIST; };
#ifndef OS_P32_T
#define OS_P32_T 256  // keys + values in TMEM, 3 blocks/SM: 1128 us/pass at q=1 (was 1222 at 2/SM)
#define OS_P32_I 32
#define OS_P32_B 3
#endif
#ifndef OS_K64_T
// keys + values in TMEM: 256 x 32 at 2 blocks/SM, 1510 us/pass (C4, 20.8 GKey/s)
// vs 256 x 16 at 3 blocks/SM without the stash, 1640 us/pass
#define OS_K64_T 256
#define OS_K64_I 32
#define OS_K64_B 2
#endif
template <> struct Geometry<4, 4> { static constexpr int T = OS_P32_T, I = OS_P32_I, B = OS_P32_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<4, 8> { static constexpr int T = OS_W32_T, I = OS_W32_I, B = OS_W32_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<8, 0> { static constexpr int T = OS_N64_T, I = OS_N64_I, B = OS_N64_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<8, 1> { static constexpr int T = OS_S64_T, I = OS_S64_I, B = OS_S64_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<8, 2> { static constexpr int T = OS_S64_T, I = OS_S64_I, B = OS_S64_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<8, 4> { static constexpr int T = OS_K64_T, I = OS_K64_I, B = OS_K64_B; static constexpr bool P = OS_PERSIST; };
template <> struct Geometry<8, 8> { static constexpr int T = OS_W64_T, I = OS_W64_I, B = OS_W64_B; static constexpr bool P = OS_PERSIST; };

template <typename K, typename V>
static cudaError_t dispatch_geom(const PassParams& p, cudaStream_t stream) {
  constexpr int KB = sizeof(K);
  constexpr int VB = ValTraits<V>::kBytes;
  using G = Geometry<KB, VB>;
  if (p.tile_keys == 0 || p.tile_keys > uint32_t(G::T * G::I)) return cudaErrorInvalidValue;
  const bool coded = (p.cin_m0 | p.cin_m1 | p.cout_m0 | p.cout_m1) != 0;
  const bool byte = (p.shift % 8) == 0 && p.mask == 0xffu;
  if (p.digit_map != nullptr) return launch_one<K, V, G::T, G::I, G::B, true, true, false, G::P>(p, stream);
  if (coded) {
    if (byte) return launch_one<K, V, G::T, G::I, G::B, false, true, true, G::P>(p, stream);
    return launch_one<K, V, G::T, G::I, G::B, false, true, false, G::P>(p, stream);
  }
  if (byte) return launch_one<K, V, G::T, G::I, G::B, false, false, true, G::P>(p, stream);
  return launch_one<K, V, G::T, G::I, G::B, false, false, false, G::P>(p, stream);
}

template <typename K>
static cudaError_t dispatch_val(const PassParams& p, int val_bytes, cudaStream_t stream) {
  switch (val_bytes) {
    case 0: return dispatch_geom<K, NoValue>(p, stream);
    case 1: return dispatch_geom<K, uint8_t>(p, stream);
    case 2: return dispatch_geom<K, uint16_t>(p, stream);
    case 4: return dispatch_geom<K, uint32_t>(p, stream);
    case 8: return dispatch_geom<K, uint64_t>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_binning_pass(const PassParams& p, int key_bytes, int val_bytes,
                                cudaStream_t stream) {
  if (key_bytes == 4) return dispatch_val<uint32_t>(p, val_bytes, stream);
  if (key_bytes == 8) return dispatch_val<uint64_t>(p, val_bytes, stream);
  return cudaErrorInvalidValue;
}

template <int KB>
static int capacity_for(int val_bytes) {
  switch (val_bytes) {
    case 0: return Geometry<KB, 0>::T * Geometry<KB, 0>::I;
    case 1: return Geometry<KB, 1>::T * Geometry<KB, 1>::I;
    case 2: return Geometry<KB, 2>::T * Geometry<KB, 2>::I;
    case 4: return Geometry<KB, 4>::T * Geometry<KB, 4>::I;
    case 8: return Geometry<KB, 8>::T * Geometry<KB, 8>::I;
    default: return 0;
  }
}

int binning_tile_capacity(int key_bytes, int val_bytes) {
  if (key_bytes == 4) return capacity_for<4>(val_bytes);
  if (key_bytes == 8) return capacity_for<8>(val_bytes);
  return 0;
}

// Status words of one strip: [tile][digit], the reference's CounterMatrix
// layout (lookback.py:63-79), padded to a multiple of four tiles.
size_t status_words_for(size_t tiles, int radix) { return (tiles + 3) / 4 * 4 * size_t(radix); }

}  // namespace osb
