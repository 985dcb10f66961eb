/*
 * onesweep_b200.h -- C ABI of the B200-native Onesweep radix sort.
 *
 * This is the drop-in boundary for the reference package `onesweep`
 * (/root/reference/pkg/src/onesweep).  The reference keeps every hot loop in
 * four numba kernels (_kernels.py:3-6) called from thin Python wrappers; this
 * library replaces those loops *and* the tile scheduling around them
 * (executor.py:160-212, lookback.py:127-169) with sm_100a CUDA kernels.
 *
 * Conventions (all entry points):
 *   - every pointer argument that names array data is a DEVICE pointer,
 *     caller-owned; the library never allocates device memory;
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream);
 *   - return value is an os_status; os_last_error() gives a message for the
 *     calling thread;
 *   - calls are reentrant on distinct workspaces, not on a shared one.
 *
 * Status codes map onto the reference's exception classes:
 *   OS_ERR_ARG      -> ValueError   (binning.py:295-304, keycodec.py:107-123)
 *   OS_ERR_KEYTYPE  -> KeyError     (keycodec.py:70-85)
 *   OS_ERR_CUDA     -> RuntimeError
 */
#ifndef ONESWEEP_B200_H
#define ONESWEEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum os_status {
  OS_OK = 0,
  OS_ERR_ARG = 1,
  OS_ERR_KEYTYPE = 2,
  OS_ERR_CUDA = 3,
  OS_ERR_WORKSPACE = 4
} os_status;

/* Key types, same set and names as keycodec.KEY_TYPES (keycodec.py:55-65). */
typedef enum os_key_type {
  OS_KEY_U32 = 0,
  OS_KEY_U64 = 1,
  OS_KEY_I32 = 2,
  OS_KEY_I64 = 3,
  OS_KEY_F32 = 4,
  OS_KEY_F64 = 5
} os_key_type;

/* Order-preserving codecs applied on load / store by the kernels
 * (keycodec.py:157-181). */
typedef enum os_codec {
  OS_CODEC_NONE = 0,       /* unsigned keys, or already-encoded bits     */
  OS_CODEC_SIGNED = 1,     /* x ^ sign  (its own inverse)                */
  OS_CODEC_FLOAT_ENC = 2,  /* neg ? ~x : x | sign                        */
  OS_CODEC_FLOAT_DEC = 3   /* (x & sign) ? x ^ sign : ~x                 */
} os_codec;

/* Device-side statistics, filled with atomics when a non-NULL pointer is
 * passed (mirrors executor.LedgerCounts' schedule-dependent columns). */
typedef struct os_device_stats {
  unsigned long long fast_path_tiles; /* short-circuit tiles (binning.py:201-205) */
  unsigned long long lookback_reads;  /* status words read in look-back (lookback.py:144-169) */
  unsigned long long tiles;           /* tiles processed */
  unsigned long long lookback_waits;  /* look-back rounds that met a not-ready (N) word */
  unsigned long long lookback_rounds; /* look-back round trips */
} os_device_stats;

const char* os_version(void);
const char* os_last_error(void);

/* Synchronise `stream` (NULL: the whole device) and report any asynchronous kernel fault (a trapped
 * look-back watchdog, an illegal address) as OS_ERR_CUDA with its message.
 * Calls are asynchronous; this is the debug-mode check after each call
 * (the Python layer runs it when ONESWEEP_B200_SYNC_CHECK=1). */
int os_stream_check(void* stream);

/* Largest digit width the binning kernel supports natively (radix <= 256). */
int os_max_digit_bits(void);

/* Default device tile (keys per thread block) for this key/value width;
 * the kernels accept any tile_keys in [1, os_tile_capacity]. */
int os_tile_capacity(int key_bytes, int val_bytes);

/* ---- elementwise ---------------------------------------------------------
 * encode_array / decode_array (keycodec.py:184-212) on device memory. */
int os_encode(const void* in, void* out, size_t n, int key_type, void* stream);
int os_decode(const void* in, void* out, size_t n, int key_type, void* stream);

/* dst[i] = src[index[i]] for rows of row_bytes bytes (any width), index
 * u32 (index_bytes 4) or u64 (8).  Values wider than 8 bytes travel through
 * the sort as an index payload and are gathered once at the end: the
 * reference reorders values of any numpy dtype (binning.py:301-304,
 * _kernels.py:85-128 scatter whole elements).  src and dst must not overlap. */
int os_gather_rows(const void* src, const void* index, int index_bytes, void* dst, size_t n,
                   size_t row_bytes, void* stream);

/* Device restatement of keygen.generate_keys (keygen.py:46-76): key i (for
 * i = first_index .. first_index+n-1) is the AND of splitmix64 words at
 * counters i*q .. i*q+q-1, truncated to key_bits.  Bit-identical. */
int os_keygen(void* out, size_t n, int key_bits, int q, unsigned long long seed,
              unsigned long long first_index, void* stream);

/* ---- upfront histogram (histogram.py:57-99) ---------------------------
 * Reads keys once and counts the digit at every place for bits
 * [begin_bit, end_bit) of the *encoded* key (codec applied on load).
 * hist_out:    u64[passes][radix], overwritten (not accumulated).
 * offsets_out: u64[passes][radix] exclusive sums per place, or NULL.
 * passes = ceil((end_bit - begin_bit) / digit_bits); digit_bits in [1, 16]
 * (the reference's range, keycodec.py:110; widths > 8 take the wide kernel).
 * workspace:   os_histogram_workspace_bytes() bytes (zeroed by the call). */
size_t os_histogram_workspace_bytes(void);
int os_histogram(const void* keys, size_t n, int key_bytes, int codec, int digit_bits,
                 int begin_bit, int end_bit, unsigned long long* hist_out,
                 unsigned long long* offsets_out, void* workspace, size_t workspace_bytes,
                 void* stream);

/* Per-row exclusive prefix sum of a u64[rows][radix] table
 * (histogram.exclusive_sum / global_bin_offsets, histogram.py:49-54,94-99). */
int os_exclusive_scan(const unsigned long long* counts, int rows, int radix,
                      unsigned long long* offsets_out, void* stream);

/* ---- one chained-scan binning pass (binning.py:218-275) ----------------
 * Stable 2^digit_width-way partition of src into dst by
 * (key >> shift) & (2^digit_width - 1) of the encoded key.
 * base_offsets: device u64[radix] -- a bin-offset row or a StripCarry.
 * carry_out:    device u64[radix] -- receives base + per-digit totals
 *               (StripCarry semantics); may alias nothing else.
 * Keys are processed in strips of <= strip_keys (binning.py:241-246) and
 * tiles of tile_keys (<= os_tile_capacity); status words follow the
 * reference's CounterMatrix layout (lookback.py:33-79): u32[tiles][radix],
 * bits 31-30 status {N,L,G}, bits 29-0 value.
 * status_out: optional device u32 buffer of os_partition_status_words()
 *             words that receives the final status words of every strip
 *             (tile-major, strips concatenated); NULL = internal.
 * digit_width in [1, 16].  Widths 9..16 run as two stable <= 8-bit binning
 * launches into scratch plus a scatter to base[d] + rank (csrc/wide.cu); they
 * need codec_in in {NONE, SIGNED, FLOAT_ENC}, keep no status words
 * (status_out must be NULL) and do not update stats.
 * workspace: os_partition_workspace_bytes_kv() bytes (for widths <= 8 this
 * equals os_partition_workspace_bytes(), which cannot size widths > 8). */
size_t os_partition_status_words(size_t n, int digit_width, int tile_keys, size_t strip_keys);
size_t os_partition_workspace_bytes(size_t n, int digit_width, int tile_keys,
                                    size_t strip_keys);
size_t os_partition_workspace_bytes_kv(size_t n, int key_bytes, int val_bytes, int digit_width,
                                       int tile_keys, size_t strip_keys);
int os_partition_pass(const void* src_keys, void* dst_keys, const void* src_vals,
                      void* dst_vals, size_t n, int key_bytes, int val_bytes, int shift,
                      int digit_width, const unsigned long long* base_offsets,
                      unsigned long long* carry_out, int codec_in, int codec_out,
                      int tile_keys, size_t strip_keys, unsigned int* status_out,
                      void* workspace, size_t workspace_bytes, os_device_stats* stats,
                      void* stream);

/* ---- the whole sort (binning.py:278-337) --------------------------------
 * keys_in / vals_in are never written.  keys_out / vals_out receive the
 * stably sorted keys (native bit pattern) and their values.  vals_* may be
 * NULL (keys only; val_bytes must then be 0).  digit_bits <= 8.
 * tile_keys = 0 selects os_tile_capacity; strip_keys = 0 selects 2^28. */
/* Copies, on `stream` after an os_sort with this workspace (and the same
 * arguments), the first tile-ticket word of every pass to words[0..passes)
 * (device or host memory; asynchronous for device memory).  A word whose top
 * five bits (>> 27) are all ones marks a digit place that held every key in
 * one bin, so the device skipped its pass (the route the upfront histogram
 * planned into the tickets).  The reference runs every place
 * (binning.py:313-326); its (2p+1)n ledger is the plan's, device element
 * moves are (1 + 2 * passes run) n. */
int os_sort_route_words(const void* workspace, size_t n, int key_type, int val_bytes,
                        int digit_bits, int begin_bit, int end_bit, int tile_keys,
                        size_t strip_keys, unsigned int* words, int max_passes, void* stream);

size_t os_sort_workspace_bytes(size_t n, int key_type, int val_bytes, int digit_bits,
                               int begin_bit, int end_bit, int tile_keys,
                               size_t strip_keys);
int os_sort(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
            size_t n, int key_type, int val_bytes, int digit_bits, int begin_bit,
            int end_bit, int tile_keys, size_t strip_keys, void* workspace,
            size_t workspace_bytes, os_device_stats* stats, void* stream);

/* Same as os_sort, and additionally records caller-created CUDA events
 * (cudaEvent_t passed as void*) on `stream`: events[0] before the histogram,
 * events[1] after it, events[2+k] after binning pass k.  num_events must be
 * >= passes + 2.  Used by bench.py to time each kernel inside the timed
 * region. */
int os_sort_events(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
                   size_t n, int key_type, int val_bytes, int digit_bits, int begin_bit,
                   int end_bit, int tile_keys, size_t strip_keys, void* workspace,
                   size_t workspace_bytes, os_device_stats* stats, void** events,
                   int num_events, void* stream);

/* Diagnostics: while buf is non-NULL, binning pass `pass` of later os_sort
 * calls writes one record of 8 u64 per tile into buf (tile-indexed):
 * globaltimer ns at claim, keys staged, L published, reorder done, warp 0's
 * G published, warp 0 done, then the SM id.  Used by tools/trace_diag.py. */
int os_debug_trace(unsigned long long* buf, int pass);

/* ---- multi-GPU MSD splitter (no reference counterpart) -------
 * Counts the top digit (bits [end_bit - digit_bits, end_bit) of the encoded
 * key) into hist_out u64[2^digit_bits] (overwritten). */
int os_msd_histogram(const void* keys, size_t n, int key_type, int digit_bits,
                     int end_bit, unsigned long long* hist_out, void* stream);
/* Stable partition of the local shard into `parts` contiguous destination
 * segments: bins [bin_lo[g], bin_lo[g+1]) go to segment g.  bin_lo is a
 * device u32[parts+1] with bin_lo[0]=0, bin_lo[parts]=radix; seg_offsets is a
 * device u64[parts] of segment starts.  Keys/values keep their native bits. */
size_t os_msd_partition_workspace_bytes(size_t n);
int os_msd_partition(const void* keys_in, void* keys_out, const void* vals_in,
                     void* vals_out, size_t n, int key_type, int val_bytes,
                     int digit_bits, int end_bit, const unsigned int* bin_lo, int parts,
                     const unsigned long long* seg_offsets, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---- reduce-then-scan ablation (rts_sort, baseline.py:121-173) ----------
 * The reference's comparator sort on the device: per 8-bit place an upsweep
 * (per-tile histograms, n reads), a digit-major prefix (baseline.py:76-84)
 * and a downsweep that is the binning kernel with the look-back replaced by
 * the prefix table (n reads + n writes).  Same output as os_sort; n < 2^32.
 * events (optional): 3 * passes + 1 events recorded before the first
 * upsweep and after every upsweep, prefix and downsweep. */
size_t os_rts_sort_workspace_bytes(size_t n, int key_type, int val_bytes);
int os_rts_sort(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
                size_t n, int key_type, int val_bytes, void* workspace,
                size_t workspace_bytes, void** events, int num_events, void* stream);

/* ---- reduce-then-scan building blocks, one digit place each -------------
 * os_rts_upsweep       replaces rts_upsweep      (baseline.py:55-73):
 *   counts u32[tiles][2^digit_width] of keys (codec applied first) in tiles
 *   of tile_keys (any size).
 * os_rts_block_prefix  replaces rts_block_prefix (baseline.py:76-84):
 *   digit-major exclusive prefix of that table -> u64[tiles][radix] absolute
 *   run starts; workspace os_rts_prefix_workspace_bytes(tiles, radix).
 * os_rts_downsweep     replaces rts_downsweep    (baseline.py:87-118):
 *   stable scatter of each tile seeded by its offsets row (the binning kernel
 *   without the look-back); tile_keys <= os_tile_capacity(key, val bytes),
 *   equal to the upsweep's; workspace os_rts_downsweep_workspace_bytes().
 * digit_width in [1, 8], n < 2^32. */
int os_rts_upsweep(const void* keys, size_t n, int key_bytes, int codec, int shift, int digit_width,
                   int tile_keys, unsigned int* counts, void* stream);
size_t os_rts_prefix_workspace_bytes(size_t tiles, int radix);
int os_rts_block_prefix(const unsigned int* counts, size_t tiles, int radix,
                        unsigned long long* offsets, void* workspace, size_t workspace_bytes,
                        void* stream);
size_t os_rts_downsweep_workspace_bytes(void);
int os_rts_downsweep(const void* src_keys, void* dst_keys, const void* src_vals, void* dst_vals,
                     size_t n, int key_bytes, int val_bytes, int shift, int digit_width,
                     const unsigned long long* offsets, int tile_keys, int codec_in,
                     int codec_out, void* workspace, size_t workspace_bytes, void* stream);

/* Fused partition + exchange over peer memory (NVLink): like
 * os_msd_partition, but dest_index is a device u64[parts] of element indices,
 * relative to keys_out / vals_out, where this rank's segment starts in each
 * destination's receive buffer (two's-complement differences when the buffer
 * is a peer-mapped allocation).  Replaces the partition + all-to-all pair of
 * the NCCL path.  Values need val_bytes == key_bytes and peer
 * value buffers at the same element distance from vals_out as the key
 * buffers from keys_out (one symmetric allocation per rank). */
int os_msd_partition_p2p(const void* keys_in, void* keys_out, const void* vals_in,
                         void* vals_out, size_t n, int key_type, int val_bytes,
                         int digit_bits, int end_bit, const unsigned int* bin_lo, int parts,
                         const unsigned long long* dest_index, void* workspace,
                         size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ONESWEEP_B200_H */
