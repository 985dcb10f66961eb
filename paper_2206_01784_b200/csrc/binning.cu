// Chained-scan digit-binning pass (one Onesweep partition pass) for sm_100a.
//
// Replaces, for one digit place and one strip, the reference's
//   partition_pass / process_tile      binning.py:162-275
//   rank_tile_kernel (WLMS)             _kernels.py:31-82
//   CounterMatrix publish / look-back   lookback.py:127-169
//   scatter_tile_kernel / slots kernel  _kernels.py:85-128
//   short-circuit fast path             binning.py:79-85,201-205
//   StripCarry write by the last tile   binning.py:196-198
//
// Persistent CTAs (as many as fit on the GPU) loop over tiles claimed from a
// monotone ticket; each tile is binned by one CTA:
//
//   1. claim the tile (forward progress for the chained scan, executor.py:1-8)
//      and start its TMA bulk copy (cp.async.bulk ... mbarrier::complete_tx)
//      into one of two shared-memory tile buffers -- one tile AHEAD, so the
//      HBM read of tile k+1 overlaps the binning of tile k;
//   2. rank keys with a warp-level multisplit: eight ballots (one per digit
//      bit) give the same-digit peer mask, rank = warp running count + popc of
//      lower peers -- the reference's WLMS (_kernels.py:56-82) on VOTE/LOP3;
//   3. reduce per-warp counts to tile counts (thread i owns digit i,
//      PAPER.md:187), publish L|count, reorder the tile locally into
//      per-digit runs, look back over predecessor status words and publish
//      G|inclusive;
//   4. write each run with coalesced stores at base + (slot - start); the
//      codec (signed/float decode) is applied on the way out.
//
// Design notes and the measurements behind them (MATCH.ANY on the ADU pipe,
// look-back windows, clusters of super-tiles) are in
// profiles/round1_binning_notes.md.
//
// Keys move once in and once out: 2n element transfers per pass, the
// reference's ledger identity (binning.py:268-272).
#include <algorithm>
#include <cstdio>
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

#ifndef OS_LOOKBACK_WINDOW
#define OS_LOOKBACK_WINDOW 4
#endif
constexpr int kLookbackWindow = OS_LOOKBACK_WINDOW;

template <int THREADS, int ITEMS, int KB, int VB, int NBUF>
struct BinningSmem {
  static constexpr int kTile = THREADS * ITEMS;
  static constexpr int kWarps = THREADS / 32;
  static constexpr size_t kKeys = size_t(kTile) * KB;
  static constexpr size_t kVals = (size_t(kTile) * VB + 15) / 16 * 16;
  static constexpr size_t kHist = size_t(kWarps) * kMaxRadix * 4;  // per-warp digit counters
  static constexpr size_t kKPtr = kMaxRadix * 8;  // per-digit output base address (keys)
  static constexpr size_t kVPtr = VB ? kMaxRadix * 8 : 0;  // (values)
  static constexpr size_t kWsum = 32 * 4;
  static constexpr size_t kMap = kMaxRadix;
  static constexpr size_t kBytes = (kKeys + kVals) * NBUF + kHist + kKPtr + kVPtr + kWsum + kMap;
};

template <typename K, typename V, int THREADS, int ITEMS, int MINB, bool MAPPED, bool CODED,
          int NBUF>
__global__ void __launch_bounds__(THREADS, MINB) onesweep_binning_kernel(const PassParams P) {
  constexpr bool HAS_V = ValTraits<V>::kHas;
  using Smem = BinningSmem<THREADS, ITEMS, sizeof(K), ValTraits<V>::kBytes, NBUF>;
  constexpr int TILE = Smem::kTile;
  constexpr int WARPS = Smem::kWarps;
  static_assert(THREADS >= kMaxRadix, "one thread per digit for the look-back");
  static_assert(THREADS % 32 == 0, "whole warps");
  static_assert(TILE < 65536, "ranks are packed as u16");
  static_assert((WARPS * kMaxRadix) % (4 * THREADS) == 0, "vectorised counter reset");
  static_assert(NBUF == 1 || NBUF == 2, "single or double buffered tiles");
  using VS = typename std::conditional<HAS_V, V, uint32_t>::type;  // storage type

  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sp = smem_raw;
  K* s_keys_buf = reinterpret_cast<K*>(sp);  // [NBUF][TILE]
  sp += Smem::kKeys * NBUF;
  VS* s_vals_buf = reinterpret_cast<VS*>(sp);  // [NBUF][TILE]
  sp += Smem::kVals * NBUF;
  uint32_t* s_whist = reinterpret_cast<uint32_t*>(sp);
  sp += Smem::kHist;
  unsigned long long* s_kptr = reinterpret_cast<unsigned long long*>(sp);
  sp += Smem::kKPtr;
  unsigned long long* s_vptr = reinterpret_cast<unsigned long long*>(sp);  // only when HAS_V
  sp += Smem::kVPtr;
  uint32_t* s_wsum = reinterpret_cast<uint32_t*>(sp);
  sp += Smem::kWsum;
  uint8_t* s_map = reinterpret_cast<uint8_t*>(sp);

  __shared__ uint32_t s_tile[NBUF];
  __shared__ int s_fast;
  __shared__ uint32_t s_reads, s_waits, s_rounds, s_fast_tiles, s_done_tiles;
  __shared__ __align__(8) uint64_t s_bar_k[NBUF];
  __shared__ __align__(8) uint64_t s_bar_v[NBUF];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int radix = P.radix;
  const int shift = P.shift;
  const uint32_t dmask = P.mask;
  const XorCodec<K> cin{K(P.cin_m0), K(P.cin_m1)};
  const XorCodec<K> cout{K(P.cout_m0), K(P.cout_m1)};
  const uint32_t num_tiles = P.num_tiles;

  auto tile_valid = [&](uint32_t tile) -> uint32_t {
    return tile < num_tiles ? min(P.tile_keys, P.strip_n - tile * P.tile_keys) : 0u;
  };
  // Claim the next tile (monotone ticket: forward progress, executor.py:1-8)
  // and start its bulk copy into buffer b.  Called by thread 0 only.
  auto claim_and_load = [&](int b) {
    const uint32_t tile = atomicAdd(P.tile_counter, 1u);
    s_tile[b] = tile;
    const uint32_t valid = tile_valid(tile);
    if (valid == 0) return;
    const K* gk = static_cast<const K*>(P.src_keys) + size_t(tile) * P.tile_keys;
    const uint32_t kbytes = valid * uint32_t(sizeof(K));
    if (((reinterpret_cast<uintptr_t>(gk) | kbytes) & 15u) == 0) {
      mbar_arrive_expect_tx(&s_bar_k[b], kbytes);
      tma_bulk_g2s(s_keys_buf + b * TILE, gk, kbytes, &s_bar_k[b]);
    } else {
      mbar_arrive(&s_bar_k[b]);  // copy path: the consumer threads load it
    }
    if (HAS_V) {
      const VS* gv = static_cast<const VS*>(P.src_vals) + size_t(tile) * P.tile_keys;
      const uint32_t vbytes = valid * uint32_t(sizeof(VS));
      if (((reinterpret_cast<uintptr_t>(gv) | vbytes) & 15u) == 0) {
        mbar_arrive_expect_tx(&s_bar_v[b], vbytes);
        tma_bulk_g2s(s_vals_buf + b * TILE, gv, vbytes, &s_bar_v[b]);
      } else {
        mbar_arrive(&s_bar_v[b]);
      }
    }
  };

  if (tid == 0) {
    s_fast = -1;
    s_reads = s_waits = s_rounds = s_fast_tiles = s_done_tiles = 0;
#pragma unroll
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&s_bar_k[b], 1);
      mbar_init(&s_bar_v[b], 1);
    }
    fence_mbar_init();
#pragma unroll
    for (int b = 0; b < NBUF; ++b) claim_and_load(b);
  }
  {
    uint4* z = reinterpret_cast<uint4*>(s_whist);
#pragma unroll
    for (int i = tid; i < WARPS * kMaxRadix / 4; i += THREADS) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (MAPPED) {
    for (int i = tid; i < kMaxRadix; i += THREADS) s_map[i] = P.digit_map[i];
  }
  __syncthreads();

  auto digit = [&](K x) -> uint32_t {
    uint32_t d = digit_of(x, shift, dmask);
    if (MAPPED) d = s_map[d];
    return d;
  };
  const uint32_t warp_base = uint32_t(warp) * (ITEMS * 32);
  uint32_t phase = 0;  // mbarrier parity, one bit per buffer
  int b = 0;

  while (true) {
    const uint32_t tile = s_tile[b];
    const uint32_t valid = tile_valid(tile);
    if (valid == 0) break;  // tickets are monotone: every later claim is past the end too
    const bool full = valid == uint32_t(TILE);
    K* s_keys = s_keys_buf + b * TILE;
    VS* s_vals = s_vals_buf + b * TILE;
    const uint32_t par = (phase >> b) & 1u;
    phase ^= 1u << b;

    // ---- 2. tile in shared memory (TMA, or the thread copy path) -------------
    const K* gk = static_cast<const K*>(P.src_keys) + size_t(tile) * P.tile_keys;
    const bool tma_k = ((reinterpret_cast<uintptr_t>(gk) | (valid * uint32_t(sizeof(K)))) & 15u) == 0;
    mbar_wait_parity(&s_bar_k[b], par);
    if (!tma_k) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        if (idx < valid) s_keys[idx] = gk[idx];
      }
    }

    auto load_key = [&](uint32_t idx) -> K {
      const K x = s_keys[idx];
      return CODED ? cin(x) : x;
    };

    // ---- 3. warp-level multisplit ranking ------------------------------------
    // Warp-striped ownership: warp w owns positions [w*ITEMS*32, (w+1)*ITEMS*32),
    // item i / lane l is position w*ITEMS*32 + i*32 + l; walking items in that
    // order keeps ranks stable (binning.py:71-76).  Positions past `valid` take
    // the largest digit: they sit after every real key, never perturb a real
    // key's rank, and their count is removed before publishing.
    uint32_t ranks[(ITEMS + 1) / 2];  // two u16 ranks per register
    auto rank_items = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      uint32_t* my_hist = s_whist + warp * kMaxRadix;
      const uint32_t lt = lanemask_lt();
      const uint32_t le = lt | (1u << lane);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        uint32_t d;
        if (FULL)
          d = digit(load_key(idx));
        else
          d = idx < valid ? digit(load_key(idx)) : uint32_t(radix - 1);
        const uint32_t peers = match_peers8(d);
        const uint32_t rank = my_hist[d] + __popc(peers & lt);
        if (i & 1)
          ranks[i / 2] += rank << 16;
        else
          ranks[i / 2] = rank;
        __syncwarp();
        if (peers <= le) my_hist[d] = rank + 1;  // highest peer: count after this batch
        __syncwarp();
      }
    };
    if (full)
      rank_items(std::true_type{});
    else
      rank_items(std::false_type{});
    __syncthreads();

    // ---- 4a. tile counts, publish L, local digit starts -----------------------
    uint32_t count = 0;
    if (tid < radix) {
      uint32_t sum = 0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) sum += s_whist[w * kMaxRadix + tid];
      if (tid == radix - 1) sum -= uint32_t(TILE) - valid;
      count = sum;
      st_relaxed_gpu(P.status + size_t(tile) * radix + tid,
                     (tile == 0 ? kFlagGlobal : kFlagLocal) | count);
      if (count == valid) s_fast = tid;
    }
    // block-wide exclusive scan of counts over digits (first 8 warps)
    uint32_t incl = count;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31 && warp < kMaxRadix / 32) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t local_start = 0;
    if (tid < radix) {
      uint32_t wpre = 0;
      for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
      local_start = wpre + incl - count;
      // fold the tile-local start into every warp's exclusive offset so the
      // reorder needs a single shared-memory gather per key
      uint32_t run = local_start;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const uint32_t c = s_whist[w * kMaxRadix + tid];
        s_whist[w * kMaxRadix + tid] = run;
        run += c;
      }
    }
    // pull this thread's keys (and values) into registers; after the barrier
    // the tile buffers are rewritten in place as per-digit runs
    K keys[ITEMS];
    VS vals[HAS_V ? ITEMS : 1];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) keys[i] = load_key(warp_base + i * 32 + lane);
    if (HAS_V) {
      const VS* gv = static_cast<const VS*>(P.src_vals) + size_t(tile) * P.tile_keys;
      const bool tma_v =
          ((reinterpret_cast<uintptr_t>(gv) | (valid * uint32_t(sizeof(VS)))) & 15u) == 0;
      mbar_wait_parity(&s_bar_v[b], par);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        if (tma_v)
          vals[i] = s_vals[idx];
        else
          vals[i] = idx < valid ? gv[idx] : VS(0);
      }
    }
    __syncthreads();
    const int fast = s_fast;

    // ---- 5a. local reorder into per-digit runs (needs no global offsets, so it
    // runs before the look-back and gives predecessors time to publish) -------
    if (fast < 0) {
      const uint32_t* my_off = s_whist + warp * kMaxRadix;
      auto stage = [&](auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          if (!FULL && warp_base + i * 32 + lane >= valid) continue;
          const uint32_t rank = (i & 1) ? (ranks[i / 2] >> 16) : (ranks[i / 2] & 0xffffu);
          const uint32_t slot = my_off[digit(keys[i])] + rank;
          s_keys[slot] = keys[i];
          if (HAS_V) s_vals[slot] = vals[i];
        }
      };
      if (full)
        stage(std::true_type{});
      else
        stage(std::false_type{});
    }
    __syncwarp();
    // this warp's counter row is consumed: reset it for the next tile
    {
      uint4* z = reinterpret_cast<uint4*>(s_whist + warp * kMaxRadix);
      for (int i = lane; i < kMaxRadix / 4; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    }

    // ---- 4b. decoupled look-back (lookback.py:144-169); then publish G and
    // the per-digit output bases -----------------------------------------------
    if (tid < radix) {
      uint32_t excl = 0;
      uint32_t reads = 0, waits = 0, rounds = 0;
      if (tile > 0) {
        const uint32_t* col = P.status + tid;
        int j = int(tile) - 1;
        bool done = false;
        while (!done) {
          uint32_t w[kLookbackWindow];
#pragma unroll
          for (int k = 0; k < kLookbackWindow; ++k)
            w[k] = (j - k >= 0) ? ld_relaxed_gpu(col + size_t(j - k) * radix) : kFlagGlobal;
          reads += kLookbackWindow;
          ++rounds;
          int k = 0;
#pragma unroll
          for (; k < kLookbackWindow; ++k) {
            const uint32_t st = w[k] >> kStatusShift;
            if (st == 0u) {  // predecessor in flight: re-poll from here
              ++waits;
              break;
            }
            excl += w[k] & kValueMask;
            if (st == 2u) {
              done = true;
              break;
            }
          }
          j -= k;
        }
        st_relaxed_gpu(P.status + size_t(tile) * radix + tid, kFlagGlobal | (excl + count));
      }
      const unsigned long long gbase = P.base_offsets[tid] + excl;
      const unsigned long long rel = gbase - local_start;  // modular: slot >= local_start
      s_kptr[tid] = reinterpret_cast<unsigned long long>(P.dst_keys) + rel * sizeof(K);
      if (HAS_V)
        s_vptr[tid] = reinterpret_cast<unsigned long long>(P.dst_vals) + rel * sizeof(VS);
      if (P.carry_out != nullptr && tile == num_tiles - 1) P.carry_out[tid] = gbase + count;
      if (P.tile_status != nullptr)  // final word in the reference's CounterMatrix format
        P.tile_status[size_t(tile) * radix + tid] = kFlagGlobal | (excl + count);
      if (P.stats != nullptr) {
        atomicAdd(&s_reads, reads);
        atomicAdd(&s_waits, waits);
        atomicAdd(&s_rounds, rounds);
      }
    }
    __syncthreads();

    if (fast >= 0) {
      // ---- short circuit: homogeneous tile is one contiguous run ------------
      K* out_k = reinterpret_cast<K*>(s_kptr[fast]);  // local start is 0
      VS* out_v = HAS_V ? reinterpret_cast<VS*>(s_vptr[fast]) : nullptr;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint32_t idx = warp_base + i * 32 + lane;
        if (idx < valid) {
          st_global(out_k + idx, CODED ? cout(keys[i]) : keys[i]);
          if (HAS_V) st_global(out_v + idx, vals[i]);
        }
      }
    } else {
      // ---- 5b. coalesced run writes: slot s of digit d lands at kptr[d] + s --
      auto write_slot = [&](uint32_t s) {
        const K x = s_keys[s];
        const uint32_t d = digit(x);
        st_global(reinterpret_cast<K*>(s_kptr[d]) + s, CODED ? cout(x) : x);
        if (HAS_V) st_global(reinterpret_cast<VS*>(s_vptr[d]) + s, s_vals[s]);
      };
      if (full) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) write_slot(uint32_t(j * THREADS + tid));
      } else {
        for (uint32_t s = tid; s < valid; s += THREADS) write_slot(s);
      }
    }
    if (tid == 0) {
      s_done_tiles += 1;
      if (fast >= 0) s_fast_tiles += 1;
    }
    // buffer b is free once every thread has read its slots: order those
    // generic-proxy accesses before the TMA that refills it
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      s_fast = -1;
      claim_and_load(b);
    }
    b = (NBUF == 2) ? (b ^ 1) : 0;
  }

  if (P.stats != nullptr && tid == 0) {
    atomicAdd(&P.stats[0], (unsigned long long)s_fast_tiles);
    atomicAdd(&P.stats[1], (unsigned long long)s_reads);
    atomicAdd(&P.stats[2], (unsigned long long)s_done_tiles);
    atomicAdd(&P.stats[3], (unsigned long long)s_waits);
    atomicAdd(&P.stats[4], (unsigned long long)s_rounds);
  }
}

// ---- host side ------------------------------------------------------------------

static int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// Persistent launch: as many CTAs as fit on the GPU at once (or fewer for a
// small strip); each loops over tiles claimed from the ticket.
template <typename K, typename V, int THREADS, int ITEMS, int MINB, bool MAPPED, bool CODED,
          int NBUF>
static cudaError_t launch_one(const PassParams& p, cudaStream_t stream) {
  using Smem = BinningSmem<THREADS, ITEMS, sizeof(K), ValTraits<V>::kBytes, NBUF>;
  auto kern = onesweep_binning_kernel<K, V, THREADS, ITEMS, MINB, MAPPED, CODED, NBUF>;
  static int resident = 0;
  if (resident == 0) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Smem::kBytes));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, THREADS, Smem::kBytes);
    if (e != cudaSuccess) return e;
    if (resident < 1) return cudaErrorInvalidConfiguration;
  }
  if (p.num_tiles == 0) return cudaSuccess;
  const unsigned grid = std::min<unsigned>(p.num_tiles, unsigned(sm_count() * resident));
  kern<<<grid, THREADS, Smem::kBytes, stream>>>(p);
  return cudaGetLastError();
}

// Tile geometry per (key, value) width: THREADS x ITEMS keys per tile, MINB
// resident CTAs per SM, NBUF tile buffers (2 = the next tile's TMA load runs
// while the current tile is binned).
template <int KB, int VB> struct Geometry;
#ifndef OS_U32_MINB
#define OS_U32_MINB 2
#endif
#ifndef OS_U32_ITEMS
#define OS_U32_ITEMS 16
#endif
#ifndef OS_U32_NBUF
#define OS_U32_NBUF 2
#endif
template <> struct Geometry<4, 0> {
  static constexpr int T = 512, I = OS_U32_ITEMS, B = OS_U32_MINB, NB = OS_U32_NBUF;
};
template <> struct Geometry<4, 1> { static constexpr int T = 512, I = 16, B = 2, NB = 1; };
template <> struct Geometry<4, 2> { static constexpr int T = 512, I = 16, B = 2, NB = 1; };
template <> struct Geometry<4, 4> { static constexpr int T = 512, I = 16, B = 2, NB = 1; };
template <> struct Geometry<4, 8> { static constexpr int T = 512, I = 8, B = 2, NB = 1; };
template <> struct Geometry<8, 0> { static constexpr int T = 512, I = 8, B = 2, NB = 1; };
template <> struct Geometry<8, 1> { static constexpr int T = 512, I = 8, B = 2, NB = 1; };
template <> struct Geometry<8, 2> { static constexpr int T = 512, I = 8, B = 2, NB = 1; };
template <> struct Geometry<8, 4> { static constexpr int T = 512, I = 8, B = 2, NB = 1; };
template <> struct Geometry<8, 8> { static constexpr int T = 512, I = 8, B = 2, NB = 1; };

template <typename K, typename V>
static cudaError_t dispatch_geom(const PassParams& p, cudaStream_t stream) {
  constexpr int KB = sizeof(K);
  constexpr int VB = ValTraits<V>::kBytes;
  using G = Geometry<KB, VB>;
  if (p.tile_keys == 0 || p.tile_keys > uint32_t(G::T * G::I)) return cudaErrorInvalidValue;
  const bool coded = (p.cin_m0 | p.cin_m1 | p.cout_m0 | p.cout_m1) != 0;
  if (p.digit_map != nullptr)
    return launch_one<K, V, G::T, G::I, G::B, true, true, G::NB>(p, stream);
  if (coded) return launch_one<K, V, G::T, G::I, G::B, false, true, G::NB>(p, stream);
  return launch_one<K, V, G::T, G::I, G::B, false, false, G::NB>(p, stream);
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

}  // namespace osb
