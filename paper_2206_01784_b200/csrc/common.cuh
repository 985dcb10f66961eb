// Device-side helpers shared by the Onesweep kernels (sm_100a).
//
// Reference semantics are cited as /root/reference/pkg/src/onesweep/<file>:<line>.
#pragma once

#include <cstddef>
#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

namespace osb {

// ---- status words (lookback.py:33-60) -------------------------------------
// bits 31-30: N=0 / L=1 / G=2, bits 29-0: value.
constexpr uint32_t kStatusShift = 30;
constexpr uint32_t kValueMask = (1u << 30) - 1u;
constexpr uint32_t kFlagLocal = 1u << 30;
constexpr uint32_t kFlagGlobal = 2u << 30;

constexpr int kMaxDigitBits = 8;
constexpr int kMaxRadix = 1 << kMaxDigitBits;
// Strip bound keeps every 30-bit status value in range (binning.py:20-23).
constexpr size_t kMaxStripKeys = size_t(1) << 28;

enum Codec : int { CODEC_NONE = 0, CODEC_SIGNED = 1, CODEC_FLOAT_ENC = 2, CODEC_FLOAT_DEC = 3 };

template <typename K> struct KeyTraits;
template <> struct KeyTraits<uint32_t> {
  static constexpr uint32_t kSign = 0x80000000u;
  static constexpr int kBits = 32;
};
template <> struct KeyTraits<uint64_t> {
  static constexpr uint64_t kSign = 0x8000000000000000ull;
  static constexpr int kBits = 64;
};

// keycodec.py:157-181.  Scalar form, for host-side planning and the
// elementwise kernels.
template <typename K>
__device__ __forceinline__ K apply_codec(K x, int codec) {
  constexpr K sign = KeyTraits<K>::kSign;
  switch (codec) {
    case CODEC_SIGNED: return x ^ sign;
    case CODEC_FLOAT_ENC: return (x & sign) ? K(~x) : K(x | sign);
    case CODEC_FLOAT_DEC: return (x & sign) ? K(x ^ sign) : K(~x);
    default: return x;
  }
}

// Branch-free codec for the per-key loops: every rule above is
// x ^ (top bit of x ? m1 : m0) with warp-uniform (m0, m1):
//   none (0, 0)   signed (sign, sign)   float-enc (sign, ~0)   float-dec (~0, sign).
// A runtime switch here compiles to a BRX jump table per key.
template <typename K>
struct XorCodec {
  K m0, m1;
  __host__ __device__ static XorCodec make(int codec) {
    constexpr K sign = KeyTraits<K>::kSign;
    constexpr K ones = ~K(0);
    switch (codec) {
      case CODEC_SIGNED: return {sign, sign};
      case CODEC_FLOAT_ENC: return {sign, ones};
      case CODEC_FLOAT_DEC: return {ones, sign};
      default: return {K(0), K(0)};
    }
  }
  __device__ __forceinline__ K operator()(K x) const {
    using S = typename std::conditional<sizeof(K) == 4, int32_t, int64_t>::type;
    const K top = K(S(x) >> (KeyTraits<K>::kBits - 1));  // all ones iff the top bit is set
    return x ^ (m0 ^ (top & (m0 ^ m1)));
  }
};

// Warp multisplit peer mask for an 8-bit digit, from ballots: one VOTE per
// digit bit on the ALU pipe, the complement taken by the lanes whose bit is
// clear, and the eight masks folded with three-input LOP3s.  __match_any_sync
// computes the same mask but issues on the ADU pipe, which capped the first
// kernel at ~14% of HBM bandwidth (profiles/round1_binning_v1.md).
#ifndef OS_NOT_ON_FMA
#define OS_NOT_ON_FMA 1
#endif
// 0xffffffff that ptxas cannot constant-fold (lanemask_lt | lanemask_ge), so
// x * m + m stays an IMAD instead of being rewritten as an ALU-pipe IADD3.
__device__ __forceinline__ uint32_t opaque_all_ones() {
  uint32_t a, b;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(a));
  asm("mov.u32 %0, %%lanemask_ge;" : "=r"(b));
  return a | b;
}
// Integer a*m + c forced onto the FMA pipe (IMAD).  The ranking and reorder
// loops are limited by the ALU pipe (LOP3/PRMT/VOTE issue at half rate), so
// adds and small multiplies go to the otherwise idle FMA pipe.  `m` should be
// an opaque register value (e.g. opaque_all_ones() >> 31 for 1).
__device__ __forceinline__ uint32_t fma_u32(uint32_t a, uint32_t m, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(m), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t vote_bit(uint32_t d, uint32_t bit) {
  uint32_t m;  // ballot of "bit set", complemented by the lanes whose bit is clear
#if OS_NOT_ON_FMA
  // ~x == x * (-1) + (-1): the complement issues on the FMA pipe (IMAD), not
  // the ALU pipe that the ballots and LOP3 folds already saturate
  asm("{\n\t.reg .pred p;\n\t"
      "and.b32 %0, %1, %2;\n\t"
      "setp.ne.u32 p, %0, 0;\n\t"
      "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
      "@!p mad.lo.u32 %0, %0, %3, %3;\n\t}"
      : "=r"(m)
      : "r"(d), "r"(bit), "r"(opaque_all_ones()));
#else
  asm("{\n\t.reg .pred p;\n\t"
      "and.b32 %0, %1, %2;\n\t"
      "setp.ne.u32 p, %0, 0;\n\t"
      "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
      "@!p not.b32 %0, %0;\n\t}"
      : "=r"(m)
      : "r"(d), "r"(bit));
#endif
  return m;
}
__device__ __forceinline__ uint32_t and3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// Written as eight separate ballots so ptxas extracts seven bit predicates
// with one R2P; the masks fold with three-input LOP3s.
__device__ __forceinline__ uint32_t match_peers8(uint32_t d) {
  const uint32_t v0 = vote_bit(d, 1), v1 = vote_bit(d, 2), v2 = vote_bit(d, 4),
                 v3 = vote_bit(d, 8), v4 = vote_bit(d, 16), v5 = vote_bit(d, 32),
                 v6 = vote_bit(d, 64), v7 = vote_bit(d, 128);
  return and3(and3(v0, v1, v2), and3(v3, v4, v5), v6 & v7);
}

// Stable warp rank for an 8-bit digit, with the peer mask folded straight into
// the two quantities the ranking loop consumes: the lower same-digit lanes
// (`below`) and whether this lane is the highest of its peers (`leader`).
// `sel` is the lane mask the peers are counted over (lanemask_lt for an
// exclusive rank, lanemask_le for an inclusive one); `gt` is lanemask_gt.
__device__ __forceinline__ void match_rank8(uint32_t d, uint32_t sel, uint32_t gt, uint32_t* peers_sel,
                                            bool* leader) {
  const uint32_t v0 = vote_bit(d, 1), v1 = vote_bit(d, 2), v2 = vote_bit(d, 4),
                 v3 = vote_bit(d, 8), v4 = vote_bit(d, 16), v5 = vote_bit(d, 32),
                 v6 = vote_bit(d, 64), v7 = vote_bit(d, 128);
  const uint32_t c = and3(and3(v0, v1, v2), and3(v3, v4, v5), v6);
  *peers_sel = and3(c, v7, sel);
  *leader = and3(c, v7, gt) == 0u;
}

// Same peer mask as match_rank8, returned whole: `peers` is every lane with
// this lane's digit, `peers_sel` the ones in `sel`.
__device__ __forceinline__ void match_rank8_peers(uint32_t d, uint32_t sel, uint32_t* peers_sel,
                                                  uint32_t* peers) {
  const uint32_t v0 = vote_bit(d, 1), v1 = vote_bit(d, 2), v2 = vote_bit(d, 4),
                 v3 = vote_bit(d, 8), v4 = vote_bit(d, 16), v5 = vote_bit(d, 32),
                 v6 = vote_bit(d, 64), v7 = vote_bit(d, 128);
  const uint32_t c = and3(and3(v0, v1, v2), and3(v3, v4, v5), v6);
  *peers_sel = and3(c, v7, sel);
  *peers = c & v7;
}

// Shared-memory atomic add returning the old value (volatile: stays in
// program order with the other volatile shared accesses).
__device__ __forceinline__ uint32_t atoms_add_u32(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}

// Shared-memory accesses by 32-bit shared address.  Volatile, so ptxas keeps
// them in program order relative to each other (the ranking counters are
// read and rewritten by the same warp item after item), but without a memory
// clobber, so ordinary loads of other shared data may still be scheduled
// around them.
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}
template <typename K>
__device__ __forceinline__ K lds_key(uint32_t addr) {
  if constexpr (sizeof(K) == 8) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return K(v);
  } else {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return K(v);
  }
}
template <typename T>
__device__ __forceinline__ void sts_val(uint32_t addr, T v) {
  if constexpr (sizeof(T) == 8)
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((unsigned long long)v));
  else if constexpr (sizeof(T) == 4)
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"((uint32_t)v));
  else if constexpr (sizeof(T) == 2)
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
  else
    asm volatile("st.shared.b8 [%0], %1;" ::"r"(addr), "r"((uint32_t)v));
}

// keycodec.py:228-239 plus the begin-bit offset: (enc >> shift) & mask.
template <typename K>
__device__ __forceinline__ uint32_t digit_of(K x, int shift, uint32_t mask) {
  return uint32_t(x >> shift) & mask;
}

// ---- memory-model helpers ------------------------------------------------
// Status words are shared between CTAs that may run concurrently on other SMs;
// a relaxed gpu-scope load/store is single-copy atomic for an aligned 32-bit
// word and bypasses the (incoherent) L1, which is all the protocol needs: the
// value travels in the same word as its status (lookback.py:9-13).
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Four consecutive status words; each element is single-copy atomic, which is
// all the protocol needs (every word carries its own flag).
__device__ __forceinline__ uint4 ld_relaxed_gpu_v4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// Bulk L2 prefetch (no shared-memory destination); bytes % 16 == 0.
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Status-word accesses with an L2 evict_last policy: nothing else in the
// kernels uses that policy, so ncu's lts__t_sectors_*_evict_last_* counters
// isolate the look-back traffic (its L2 hit rate), and the words stay resident.
__device__ __forceinline__ uint32_t ld_relaxed_gpu_keep(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu_keep(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.relaxed.gpu.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stores through addresses rebuilt from integers: keep them STG (global),
// not generic ST.
template <typename T>
__device__ __forceinline__ void st_global(T* p, T v) {
  if constexpr (sizeof(T) == 8)
    asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)v) : "memory");
  else if constexpr (sizeof(T) == 4)
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"((uint32_t)v) : "memory");
  else if constexpr (sizeof(T) == 2)
    asm volatile("st.global.b16 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
  else
    asm volatile("st.global.b8 [%0], %1;" ::"l"(p), "r"((uint32_t)v) : "memory");
}

// Run-write store: streaming (.cs), the output of a pass is not re-read by
// this pass, and tile loads carry an L2 evict_first policy, so the status
// words and prefetched tiles keep their L2 lines (~1 % per pass,
// profiles/round1_binning_notes.md).
__device__ __forceinline__ void st_global_cs(uint32_t* p, uint32_t v) {
  asm volatile("st.global.cs.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// base + index for 64-bit output indices that may be "negative" (two's
// complement): os_msd_partition_p2p addresses peer receive buffers relative to
// the local output base, so the index wraps modulo 2^64 by design.
template <typename T>
__device__ __forceinline__ T* elem_at(T* base, unsigned long long index) {
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(base) + index * sizeof(T));
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- thread-block clusters: rank, barrier, DSMEM ---------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of this CTA's `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ uint32_t ld_dsmem_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void st_dsmem_u64(uint32_t addr, unsigned long long v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}

// ---- mbarrier + TMA bulk copy (global -> shared) ---------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// order this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) accesses to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// OS_MBAR_HINT > 0: try_wait carries a suspend-time hint (ns), so a waiting
// thread sleeps until the phase completes (or the hint expires) instead of
// re-issuing the try_wait loop, leaving issue slots to the other blocks.
#ifndef OS_MBAR_HINT
#define OS_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  while (!done) {
    if (OS_MBAR_HINT > 0) {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(addr), "r"(parity), "r"(uint32_t(OS_MBAR_HINT))
          : "memory");
    } else {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(addr), "r"(parity)
          : "memory");
    }
  }
}
// One bulk (non-tensor) TMA copy; bytes % 16 == 0, both addresses 16B aligned.
__device__ __forceinline__ void tma_bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- tensor memory (TMEM) as a per-thread stash -----------------------------
// The binning kernel parks each thread's keys in its own TMEM lane between the
// ranking loop and the reorder: TMEM traffic does not use the L1/shared data
// pipe that bounds the pass, and the keys no longer hold registers across the
// look-back phase.  Address = (lane << 16) | column; a warp reaches only the
// 32-lane quadrant (warp % 4).
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// Load 8 columns of this thread's lane; the wait is part of the same helper and
// threads the registers through it, so no use can be scheduled before it.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7])
               :
               : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s_hint(void* dst_smem, const void* src_gmem,
                                                  uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// ---- programmatic dependent launch ------------------------------------------
__device__ __forceinline__ void grid_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void grid_dependency_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---- pass routing (os_sort) --------------------------------------------------
// A digit place whose histogram has one bin holding all n keys is an identity
// permutation, so its pass can be skipped.  The upfront histogram's last
// block decides this for every place and plans the remaining ping-pong so
// that the last sorting pass still lands in the caller's output.  The plan
// travels in the tile-ticket words themselves: the histogram initialises the
// ticket of every (pass, strip) to code << kTicketShift, so the atomicAdd
// that claims a tile also returns its pass's route (no extra load, no host
// round trip, and the decision replays inside a CUDA graph).
//   code 0           unrouted: the launch's own buffers and codec masks
//   code kTicketSkip skipped place: the block exits at its first claim
//   code 1 + bits    bits = src (0 input, 1 workspace, 2 output)
//                           | 4 * (dst is the output) | 8 * first | 16 * last
// For signed and float keys (a key codec on the first pass's loads and the
// last pass's stores) the first and last places always run, so the codec
// stays where the launches put it; only trivial places in between are
// skipped.  first / last are informational.  If every place is trivial the
// last place still runs, input to output: each tile takes the one-run fast
// path, which is a copy.
constexpr int kTicketShift = 27;
constexpr uint32_t kTicketMask = (1u << kTicketShift) - 1u;
constexpr uint32_t kTicketSkip = 31u;
enum : uint32_t { kBufIn = 0, kBufTmp = 1, kBufOut = 2 };
enum : uint32_t { kRouteDstOut = 4, kRouteFirst = 8, kRouteLast = 16 };
__device__ __forceinline__ void plan_tickets(uint32_t* tickets, size_t pass_stride, int strips,
                                             int passes, uint32_t trivial, bool fixed_ends) {
  if (fixed_ends) trivial &= ~(1u | (1u << (passes - 1)));
  int m = 0;
  for (int k = 0; k < passes; ++k) m += ((trivial >> k) & 1u) ? 0 : 1;
  if (m == 0) {  // all trivial: the last place runs as the copy
    trivial &= ~(1u << (passes - 1));
    m = 1;
  }
  int j = 0;
  uint32_t cur = kBufIn;
  for (int k = 0; k < passes; ++k) {
    uint32_t code = kTicketSkip;
    if (!((trivial >> k) & 1u)) {
      const bool to_out = ((m - 1 - j) % 2) == 0;
      code = 1u + (cur | (to_out ? kRouteDstOut : 0u) | (j == 0 ? kRouteFirst : 0u) |
                   (j == m - 1 ? kRouteLast : 0u));
      cur = to_out ? kBufOut : kBufTmp;
      ++j;
    }
    for (int s = 0; s < strips; ++s) tickets[size_t(k) * pass_stride + s] = code << kTicketShift;
  }
}

// ---- launch descriptors ------------------------------------------------------
struct PassParams {
  const void* src_keys;  // strip-relative base already applied by the host
  void* dst_keys;        // global output base (not strip relative)
  const void* src_vals;
  void* dst_vals;
  uint32_t strip_n;      // keys in this strip (<= 2^28)
  uint32_t num_tiles;    // ceil(strip_n / tile_keys)
  uint32_t tile_keys;    // logical tile (<= template capacity)
  int shift;
  uint32_t mask;         // radix - 1
  int radix;
  unsigned long long cin_m0, cin_m1;    // XorCodec applied on load
  unsigned long long cout_m0, cout_m1;  // XorCodec applied on store
  const unsigned long long* base_offsets;  // [radix]
  unsigned long long* carry_out;           // [radix] or null
  uint32_t* status;       // look-back words [tiles/4][radix][4], zeroed
  uint32_t* tile_status;  // optional final per-tile words [num_tiles][radix] (CounterMatrix view)
  uint32_t* tile_counter; // super-tile ticket, zeroed
  unsigned long long* stats;               // os_device_stats or null
  const uint8_t* digit_map;                // [2^map_bits] -> destination, or null
  uint32_t prefetch_tiles;                 // L2-prefetch distance in tiles (0: off)
  unsigned long long* trace;               // diagnostics: kTraceWords per tile, or null
  uint32_t wide_index;                     // output indices may reach 2^32 (64-bit run writes)
  const unsigned long long* rts_offsets;   // reduce-then-scan ablation: [num_tiles][radix] run starts, or null
  int debug_stall_tile;                    // OS_JITTER builds: this tile never publishes (watchdog test); -1 off
  // routed passes (ticket code > 0): buffer bases by route, index
  // (code - 1) & 7 = src | 4 * (dst is the output); [0] source keys (this
  // strip), [1] source values (this strip), [2] destination keys, [3]
  // destination values (plan_tickets)
  const void* route_bases[8][4];
};
// Per-tile trace record (globaltimer ns): claim, keys staged, L published,
// reorder done, warp 0 G published, warp 0 done, SM id, unused.
constexpr int kTraceWords = 8;
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

struct HistParams {
  const void* keys;
  size_t n;
  int codec;  // os_codec applied on load (as a XorCodec)
  int begin_bit;
  int digit_bits;
  int passes;
  int top_bits;  // width of the last place
  unsigned long long* hist;     // [passes][radix] (zeroed by host)
  unsigned long long* offsets;  // [passes][radix] or null
  unsigned int* done_counter;   // zeroed
  uint32_t* tickets;            // [passes][strips] tile tickets of the routed passes, or null
  size_t ticket_stride;         // words between two passes' tickets
  int strips;
  int fixed_ends;               // coded keys: the first and last places always run
};

// Host launchers (defined in the .cu files).
cudaError_t launch_binning_pass(const PassParams& p, int key_bytes, int val_bytes,
                                cudaStream_t stream);
int binning_tile_capacity(int key_bytes, int val_bytes);
size_t status_words_for(size_t tiles, int radix);
cudaError_t launch_histogram(const HistParams& p, int key_bytes, cudaStream_t stream);
cudaError_t launch_exclusive_scan(const unsigned long long* counts, int rows, int radix,
                                  unsigned long long* out, cudaStream_t stream);
cudaError_t launch_codec(const void* in, void* out, size_t n, int key_bytes, int codec,
                         cudaStream_t stream);
cudaError_t launch_keygen(void* out, size_t n, int key_bits, int q, unsigned long long seed,
                          unsigned long long first, cudaStream_t stream);
cudaError_t launch_gather_rows(const void* src, const void* index, int index_bytes, void* dst,
                               size_t n, size_t row_bytes, cudaStream_t stream);
cudaError_t launch_rts_upsweep(const void* keys, size_t n, int key_bytes, uint32_t tile_keys,
                               int shift, uint32_t mask, int codec, uint32_t* counts,
                               cudaStream_t stream);
size_t rts_chunk_count(size_t tiles);
cudaError_t launch_rts_prefix(const uint32_t* counts, uint32_t tiles, int radix,
                              unsigned long long* csum, unsigned long long* offsets,
                              cudaStream_t stream);
constexpr int kMaxWideDigitBits = 16;  // reference range (keycodec.py:110)
cudaError_t launch_wide_histogram(const void* keys, size_t n, int key_bytes, int codec,
                                  int begin_bit, int digit_bits, int passes, int top_bits,
                                  unsigned long long* hist, cudaStream_t stream);
cudaError_t launch_wide_tables(const unsigned long long* base, const unsigned long long* count,
                               const unsigned long long* dense_start, int radix,
                               unsigned long long* rel, unsigned long long* carry,
                               cudaStream_t stream);
cudaError_t launch_wide_scatter(const void* src_k, void* dst_k, const void* src_v, void* dst_v,
                                int kb, int vb, size_t n, int shift, int width,
                                const unsigned long long* rel, int codec_out, cudaStream_t stream);
cudaError_t launch_top_histogram(const void* keys, size_t n, int key_bytes, int codec, int shift,
                                 uint32_t mask, unsigned long long* hist, cudaStream_t stream);

}  // namespace osb
