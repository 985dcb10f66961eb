// extern "C" boundary (include/onesweep_b200.h): argument validation,
// workspace carving and kernel orchestration.  Mirrors the reference's
// onesweep_sort / partition_pass / global_histograms control flow
// (binning.py:218-337, histogram.py:57-99) with device kernels doing all the
// element work -- there is no host compute path.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "../../include/onesweep_b200.h"
#include "common.cuh"

// NVTX ranges around every launch (tracing): a
// profiler timeline shows "onesweep histogram", "onesweep pass k", ... on
// the host thread.  Header-only NVTX3; without an attached tool a push/pop
// is a null-pointer check.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* fmt, int k) {
    char buf[48];
    snprintf(buf, sizeof buf, fmt, k);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

namespace osb {
int histogram_grid_size();
}

using namespace osb;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(OS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define OS_CUDA(call, where)                       \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct KeyType {
  int bytes;
  int enc;  // codec applied when loading native keys
  int dec;  // codec applied when storing native keys
};

bool key_type_info(int key_type, KeyType* out) {
  switch (key_type) {
    case OS_KEY_U32: *out = {4, CODEC_NONE, CODEC_NONE}; return true;
    case OS_KEY_U64: *out = {8, CODEC_NONE, CODEC_NONE}; return true;
    case OS_KEY_I32: *out = {4, CODEC_SIGNED, CODEC_SIGNED}; return true;
    case OS_KEY_I64: *out = {8, CODEC_SIGNED, CODEC_SIGNED}; return true;
    case OS_KEY_F32: *out = {4, CODEC_FLOAT_ENC, CODEC_FLOAT_DEC}; return true;
    case OS_KEY_F64: *out = {8, CODEC_FLOAT_ENC, CODEC_FLOAT_DEC}; return true;
    default: return false;
  }
}

bool valid_val_bytes(int vb) { return vb == 0 || vb == 1 || vb == 2 || vb == 4 || vb == 8; }

// Tiling of one pass: strips of <= strip keys (binning.py:241-246), tiles of
// tile keys inside each strip (the last tile of a strip may be ragged).
struct Tiling {
  size_t n = 0;
  size_t strip = 0;
  size_t strips = 0;
  size_t tiles_total = 0;  // sum over strips
  uint32_t tile = 0;
  size_t strip_len(size_t s) const {
    const size_t lo = s * strip;
    return (n - lo) < strip ? (n - lo) : strip;
  }
  size_t strip_tiles(size_t s) const { return (strip_len(s) + tile - 1) / tile; }
};

Tiling make_tiling(size_t n, uint32_t tile, size_t strip) {
  Tiling t;
  t.n = n;
  t.tile = tile;
  t.strip = strip;
  t.strips = n ? (n + strip - 1) / strip : 0;
  // tiles per full strip, plus the ragged last strip
  if (t.strips) {
    const size_t full = t.strips - 1;
    t.tiles_total = full * ((strip + tile - 1) / tile) + t.strip_tiles(t.strips - 1);
  }
  return t;
}

int resolve_tile(int tile_keys, int key_bytes, int val_bytes, uint32_t* out) {
  const int cap = binning_tile_capacity(key_bytes, val_bytes);
  if (cap <= 0) return fail(OS_ERR_ARG, "unsupported key/value width %d/%d", key_bytes, val_bytes);
  if (tile_keys < 0) return fail(OS_ERR_ARG, "tile_keys must be >= 0, got %d", tile_keys);
  *out = uint32_t(tile_keys == 0 || tile_keys > cap ? cap : tile_keys);
  return OS_OK;
}

int resolve_strip(size_t strip_keys, size_t* out) {
  if (strip_keys == 0) strip_keys = kMaxStripKeys;
  if (strip_keys > kMaxStripKeys)
    return fail(OS_ERR_ARG, "strip_keys must be <= 2^28, got %zu", strip_keys);
  *out = strip_keys;
  return OS_OK;
}

// Workspace of one pass over all strips: look-back status words (one row per
// tile, the reference's CounterMatrix layout), tile tickets and the 64-bit
// carries chained between strips (binning.py:196-198, 262).
struct PassWs {
  size_t status_words = 0;
  size_t strip_status_words = 0;  // every strip uses the stride of a full strip
  size_t off_status = 0, off_counters = 0, off_carry = 0, bytes = 0, zero_bytes = 0;
};

PassWs pass_ws(const Tiling& t, int radix, bool own_status) {
  PassWs w;
  w.strip_status_words = t.strips ? status_words_for(t.strip_tiles(0), radix) : 0;
  w.status_words = t.strips * w.strip_status_words;
  size_t off = 0;
  w.off_status = off;
  if (own_status) off = align_up(off + w.status_words * 4);
  w.off_counters = off;
  off = align_up(off + (t.strips ? t.strips : 1) * 4);
  w.zero_bytes = off;  // status + tickets are zeroed per pass
  w.off_carry = off;
  off = align_up(off + (t.strips ? t.strips : 1) * size_t(radix) * 8);
  w.bytes = off;
  return w;
}

// L2 prefetch distance of the binning kernel, in tiles: about one wave of
// resident blocks ahead (ONESWEEP_B200_PREFETCH overrides; 0 disables).
uint32_t prefetch_tiles() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ONESWEEP_B200_PREFETCH");
    v = e ? atoi(e) : 296;
    if (v < 0) v = 0;
  }
  return uint32_t(v);
}

// Device-side pass skipping in os_sort (plan_tickets); ONESWEEP_B200_NO_SKIP=1
// turns it off (A/B runs; the reference's fixed (2p+1)n schedule).
bool route_passes() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ONESWEEP_B200_NO_SKIP");
    v = (e && atoi(e) != 0) ? 0 : 1;
  }
  return v != 0;
}

// Failure injection for the watchdog test (honoured by OS_JITTER builds
// only): ONESWEEP_B200_DEBUG_STALL_TILE=t makes tile t of every pass skip its
// status publishes, so its successors' look-backs must trap, not hang.
int debug_stall_tile() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("ONESWEEP_B200_DEBUG_STALL_TILE");
    v = e ? atoi(e) : -1;
  }
  return v;
}

// Diagnostics (os_debug_trace): per-tile timeline of one pass.
unsigned long long* g_trace = nullptr;
int g_trace_pass = -1;

// One binning pass over every strip (partition_pass, binning.py:218-275).
int run_pass(const void* src_k, void* dst_k, const void* src_v, void* dst_v, int kb, int vb,
             const Tiling& t, int shift, int width, int radix, const uint8_t* digit_map,
             const unsigned long long* base0, unsigned long long* carry_final, int codec_in,
             int codec_out, uint32_t* status, uint32_t* tile_status, unsigned char* ws,
             const PassWs& w, unsigned long long* stats, cudaStream_t stream,
             bool dense_bases, unsigned long long* trace = nullptr,
             const void* const* buf_keys = nullptr, const void* const* buf_vals = nullptr) {
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + w.off_counters);
  unsigned long long* carries = reinterpret_cast<unsigned long long*>(ws + w.off_carry);
  size_t tile_base = 0;
  const unsigned long long* base = base0;
  for (size_t s = 0; s < t.strips; ++s) {
    PassParams p{};
    const size_t lo = s * t.strip;
    p.src_keys = static_cast<const unsigned char*>(src_k) + lo * kb;
    p.dst_keys = dst_k;
    p.src_vals = vb ? static_cast<const unsigned char*>(src_v) + lo * vb : nullptr;
    p.dst_vals = vb ? dst_v : nullptr;
    p.strip_n = uint32_t(t.strip_len(s));
    p.num_tiles = uint32_t(t.strip_tiles(s));
    p.tile_keys = t.tile;
    p.shift = shift;
    p.mask = width >= 32 ? 0xffffffffu : ((1u << width) - 1u);
    p.radix = radix;
    if (kb == 4) {
      const auto ci = XorCodec<uint32_t>::make(codec_in), co = XorCodec<uint32_t>::make(codec_out);
      p.cin_m0 = ci.m0, p.cin_m1 = ci.m1, p.cout_m0 = co.m0, p.cout_m1 = co.m1;
    } else {
      const auto ci = XorCodec<uint64_t>::make(codec_in), co = XorCodec<uint64_t>::make(codec_out);
      p.cin_m0 = ci.m0, p.cin_m1 = ci.m1, p.cout_m0 = co.m0, p.cout_m1 = co.m1;
    }
    p.base_offsets = base;
    const bool last = (s + 1 == t.strips);
    p.carry_out = last ? carry_final : carries + s * size_t(radix);
    p.status = status + s * w.strip_status_words;
    p.tile_status = tile_status ? tile_status + tile_base * size_t(radix) : nullptr;
    p.tile_counter = counters + s;
    p.stats = stats;
    p.digit_map = digit_map;
    p.prefetch_tiles = prefetch_tiles();
    // the run writes index the output with 32 bits unless it could be larger
    // (partition_pass callers may pass any base offsets)
    p.wide_index = !dense_bases || t.n >= (size_t(1) << 32) - (size_t(1) << 26);
    p.trace = trace ? trace + tile_base * kTraceWords : nullptr;
    p.debug_stall_tile = debug_stall_tile();
    if (buf_keys != nullptr) {  // routed sort pass: the ticket's route code picks a row
      for (int ix = 0; ix < 8; ++ix) {
        const int src = ix & 3;
        if (src > 2) continue;
        const int dst = (ix & 4) ? 2 : 1;  // output / workspace
        p.route_bases[ix][0] = static_cast<const unsigned char*>(buf_keys[src]) + lo * kb;
        p.route_bases[ix][1] = vb ? static_cast<const unsigned char*>(buf_vals[src]) + lo * vb : nullptr;
        p.route_bases[ix][2] = buf_keys[dst];
        p.route_bases[ix][3] = vb ? buf_vals[dst] : nullptr;
      }
    }
    OS_CUDA(launch_binning_pass(p, kb, vb, stream), "binning pass launch");
    base = p.carry_out;
    tile_base += p.num_tiles;
  }
  return OS_OK;
}

int check_bits(int key_bytes, int digit_bits, int begin_bit, int end_bit,
               int max_bits = kMaxDigitBits) {
  const int kbits = key_bytes * 8;
  if (digit_bits < 1 || digit_bits > max_bits)
    return fail(OS_ERR_ARG, "digit_bits must be in [1, %d] on the device path, got %d",
                max_bits, digit_bits);
  if (begin_bit < 0 || end_bit > kbits || begin_bit >= end_bit)
    return fail(OS_ERR_ARG, "need 0 <= begin_bit < end_bit <= %d, got [%d, %d)", kbits,
                begin_bit, end_bit);
  return OS_OK;
}

struct SortLayout {
  int passes = 0, radix = 0;
  Tiling t;
  PassWs pw;
  size_t off_tmp_k = 0, off_tmp_v = 0, off_offsets = 0, off_zero = 0, off_hist = 0,
         off_done = 0, off_pass = 0, zero_bytes = 0, total = 0;
};

SortLayout sort_layout(size_t n, int kb, int vb, int digit_bits, int begin_bit, int end_bit,
                       uint32_t tile, size_t strip) {
  SortLayout L;
  L.passes = (end_bit - begin_bit + digit_bits - 1) / digit_bits;
  L.radix = 1 << digit_bits;
  L.t = make_tiling(n, tile, strip);
  L.pw = pass_ws(L.t, L.radix, true);
  size_t off = 0;
  L.off_tmp_k = off;
  off = align_up(off + (L.passes > 1 ? n * kb : 0));
  L.off_tmp_v = off;
  off = align_up(off + (L.passes > 1 ? n * vb : 0));
  L.off_offsets = off;
  off = align_up(off + size_t(L.passes) * L.radix * 8);
  // everything from here on is zeroed by one memset per sort
  L.off_zero = off;
  L.off_hist = off;
  off = align_up(off + size_t(L.passes) * L.radix * 8);
  L.off_done = off;
  off = align_up(off + 4);
  L.off_pass = off;
  off += size_t(L.passes) * L.pw.bytes;
  L.zero_bytes = off - L.off_zero;
  L.total = off;
  return L;
}

}  // namespace

extern "C" {

const char* os_version(void) {
#if OS_JITTER
  return "onesweep_b200 0.2.0 (sm_100a, debug: look-back jitter + failure injection)";
#else
  return "onesweep_b200 0.2.0 (sm_100a)";
#endif
}

// Entry points whose first runtime call would be a kernel launch make one
// plain runtime call first: when the library is loaded after the CUDA
// context exists (torch initialised first), a launch as the very first
// runtime call goes through an internal kernel-handle retry in cudart that
// compute-sanitizer reports as an API error (the launch itself succeeds).
static void runtime_ready() {
  static bool ready = false;
  if (!ready) {
    cudaFree(nullptr);
    ready = true;
  }
}

int os_stream_check(void* stream) {
  // surfaces asynchronous kernel faults (a trapped look-back watchdog, an
  // illegal address) at the call that caused them
  OS_CUDA(stream ? cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) : cudaDeviceSynchronize(),
          "asynchronous kernel error");
  OS_CUDA(cudaGetLastError(), "asynchronous kernel error");
  return OS_OK;
}
const char* os_last_error(void) { return g_err; }
int os_max_digit_bits(void) { return kMaxDigitBits; }
int os_tile_capacity(int key_bytes, int val_bytes) {
  return binning_tile_capacity(key_bytes, val_bytes);
}

int os_encode(const void* in, void* out, size_t n, int key_type, void* stream) {
  runtime_ready();
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  OS_CUDA(launch_codec(in, out, n, kt.bytes, kt.enc, static_cast<cudaStream_t>(stream)),
          "encode");
  return OS_OK;
}

int os_gather_rows(const void* src, const void* index, int index_bytes, void* dst, size_t n,
                   size_t row_bytes, void* stream) {
  runtime_ready();
  NvtxRange nvtx_range("onesweep gather_rows");
  if (index_bytes != 4 && index_bytes != 8)
    return fail(OS_ERR_ARG, "index_bytes must be 4 or 8, got %d", index_bytes);
  if (n && (src == nullptr || index == nullptr || dst == nullptr))
    return fail(OS_ERR_ARG, "null buffer");
  if (n && row_bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src), b = reinterpret_cast<uintptr_t>(dst);
    if (a < b + n * row_bytes && b < a + n * row_bytes) return fail(OS_ERR_ARG, "gather in place");
  }
  OS_CUDA(launch_gather_rows(src, index, index_bytes, dst, n, row_bytes,
                             static_cast<cudaStream_t>(stream)),
          "gather_rows");
  return OS_OK;
}

int os_decode(const void* in, void* out, size_t n, int key_type, void* stream) {
  runtime_ready();
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  OS_CUDA(launch_codec(in, out, n, kt.bytes, kt.dec, static_cast<cudaStream_t>(stream)),
          "decode");
  return OS_OK;
}

int os_keygen(void* out, size_t n, int key_bits, int q, unsigned long long seed,
              unsigned long long first_index, void* stream) {
  runtime_ready();
  if (key_bits != 32 && key_bits != 64)
    return fail(OS_ERR_ARG, "key_bits must be 32 or 64, got %d", key_bits);
  if (q < 1) return fail(OS_ERR_ARG, "q must be >= 1, got %d", q);
  OS_CUDA(launch_keygen(out, n, key_bits, q, seed, first_index, static_cast<cudaStream_t>(stream)),
          "keygen");
  return OS_OK;
}

size_t os_histogram_workspace_bytes(void) { return kAlign; }

int os_histogram(const void* keys, size_t n, int key_bytes, int codec, int digit_bits,
                 int begin_bit, int end_bit, unsigned long long* hist_out,
                 unsigned long long* offsets_out, void* workspace, size_t workspace_bytes,
                 void* stream) {
  if (key_bytes != 4 && key_bytes != 8) return fail(OS_ERR_ARG, "key_bytes must be 4 or 8");
  if (int rc = check_bits(key_bytes, digit_bits, begin_bit, end_bit, kMaxWideDigitBits)) return rc;
  if (codec < CODEC_NONE || codec > CODEC_FLOAT_ENC)
    return fail(OS_ERR_ARG, "histogram codec must be NONE, SIGNED or FLOAT_ENC");
  if (workspace_bytes < os_histogram_workspace_bytes() || workspace == nullptr)
    return fail(OS_ERR_WORKSPACE, "histogram workspace too small");
  const int passes = (end_bit - begin_bit + digit_bits - 1) / digit_bits;
  const int radix = 1 << digit_bits;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n > size_t(osb::histogram_grid_size()) * (size_t(1) << 31))
    return fail(OS_ERR_ARG, "n too large for 32-bit per-block histogram portions");
  OS_CUDA(cudaMemsetAsync(hist_out, 0, size_t(passes) * radix * 8, s), "histogram memset");
  OS_CUDA(cudaMemsetAsync(workspace, 0, kAlign, s), "histogram memset");
  HistParams p{};
  p.keys = keys;
  p.n = n;
  p.codec = codec;
  p.begin_bit = begin_bit;
  p.digit_bits = digit_bits;
  p.passes = passes;
  p.top_bits = end_bit - (begin_bit + (passes - 1) * digit_bits);
  p.hist = hist_out;
  p.offsets = offsets_out;
  p.done_counter = static_cast<unsigned int*>(workspace);
  if (n == 0) {
    if (offsets_out) OS_CUDA(cudaMemsetAsync(offsets_out, 0, size_t(passes) * radix * 8, s), "memset");
    return OS_OK;
  }
  if (digit_bits > kMaxDigitBits) {  // 2^9..2^16-way places (csrc/wide.cu)
    OS_CUDA(launch_wide_histogram(keys, n, key_bytes, codec, begin_bit, digit_bits, passes,
                                  p.top_bits, hist_out, s), "wide histogram launch");
    if (offsets_out)
      OS_CUDA(launch_exclusive_scan(hist_out, passes, radix, offsets_out, s), "exclusive scan");
    return OS_OK;
  }
  OS_CUDA(launch_histogram(p, key_bytes, s), "histogram launch");
  return OS_OK;
}

int os_exclusive_scan(const unsigned long long* counts, int rows, int radix,
                      unsigned long long* offsets_out, void* stream) {
  if (rows < 0 || radix < 0) return fail(OS_ERR_ARG, "rows/radix must be >= 0");
  OS_CUDA(launch_exclusive_scan(counts, rows, radix, offsets_out, static_cast<cudaStream_t>(stream)),
          "exclusive scan");
  return OS_OK;
}

size_t os_partition_status_words(size_t n, int digit_width, int tile_keys, size_t strip_keys) {
  if (tile_keys <= 0 || digit_width < 1 || digit_width > kMaxDigitBits) return 0;
  size_t strip = strip_keys ? strip_keys : kMaxStripKeys;
  Tiling t = make_tiling(n, uint32_t(tile_keys), strip);
  return t.tiles_total << digit_width;
}

size_t os_partition_workspace_bytes(size_t n, int digit_width, int tile_keys, size_t strip_keys) {
  if (tile_keys <= 0 || digit_width < 1 || digit_width > kMaxDigitBits) return 0;
  size_t strip = strip_keys ? strip_keys : kMaxStripKeys;
  Tiling t = make_tiling(n, uint32_t(tile_keys), strip);
  return pass_ws(t, 1 << digit_width, true).bytes;
}

}  // extern "C"

namespace {
// Scratch of a 2^9..2^16-way partition pass (csrc/wide.cu): two dense
// ping-pong copies, the 8-bit sub-pass tables and the 2^d-way tables, then
// the workspace of the 8-bit binning sub-passes.
struct WideLayout {
  Tiling t;
  PassWs pw;
  size_t off_ak = 0, off_av = 0, off_bk = 0, off_bv = 0, off_h8 = 0, off_o8 = 0, off_done = 0,
         off_hw = 0, off_ow = 0, off_rel = 0, off_sub = 0, total = 0;
};
WideLayout wide_layout(size_t n, int kb, int vb, int width, uint32_t tile, size_t strip) {
  WideLayout L;
  L.t = make_tiling(n, tile, strip);
  L.pw = pass_ws(L.t, kMaxRadix, true);
  const size_t rw = size_t(1) << width;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off = align_up(off + bytes); return o; };
  L.off_ak = take(n * kb);
  L.off_av = take(n * vb);
  L.off_bk = take(n * kb);
  L.off_bv = take(n * vb);
  L.off_h8 = take(2 * kMaxRadix * 8);
  L.off_o8 = take(2 * kMaxRadix * 8);
  L.off_done = take(kAlign);
  L.off_hw = take(rw * 8);
  L.off_ow = take(rw * 8);
  L.off_rel = take(rw * 8);
  L.off_sub = take(L.pw.bytes);
  L.total = off;
  return L;
}

int wide_partition(const void* src_k, void* dst_k, const void* src_v, void* dst_v, size_t n,
                   int kb, int vb, int shift, int width, const unsigned long long* base,
                   unsigned long long* carry_out, int codec_in, int codec_out, uint32_t tile,
                   size_t strip, unsigned char* ws, size_t ws_bytes, cudaStream_t s) {
  if (codec_in > CODEC_FLOAT_ENC)
    return fail(OS_ERR_ARG, "codec_in must be NONE, SIGNED or FLOAT_ENC for digit widths > 8");
  // the top place may reach past the key: its digit is zero-extended
  // (keycodec.py:125-128), so only the bits inside the key are binned
  const int kbits = kb * 8;
  const int lo_w = kbits - shift < kMaxDigitBits ? kbits - shift : kMaxDigitBits;
  const int hi_w = (width < kbits - shift ? width : kbits - shift) - lo_w;
  const WideLayout L = wide_layout(n, kb, vb, width, tile, strip);
  if (ws == nullptr || ws_bytes < L.total)
    return fail(OS_ERR_WORKSPACE, "partition workspace needs %zu bytes, got %zu", L.total, ws_bytes);
  const int radix = 1 << width;
  auto u64 = [&](size_t off) { return reinterpret_cast<unsigned long long*>(ws + off); };
  // 1. dense offsets of the digit's low byte and high (width - 8) bits
  OS_CUDA(cudaMemsetAsync(ws + L.off_h8, 0, 2 * kMaxRadix * 8, s), "memset");
  OS_CUDA(cudaMemsetAsync(ws + L.off_done, 0, kAlign, s), "memset");
  HistParams hp{};
  hp.keys = src_k;
  hp.n = n;
  hp.codec = codec_in;
  hp.begin_bit = shift;
  hp.digit_bits = kMaxDigitBits;
  hp.passes = hi_w > 0 ? 2 : 1;
  hp.top_bits = hi_w > 0 ? hi_w : lo_w;
  hp.hist = u64(L.off_h8);
  hp.offsets = u64(L.off_o8);
  hp.done_counter = reinterpret_cast<unsigned int*>(ws + L.off_done);
  {
    NvtxRange r("onesweep histogram");
    OS_CUDA(launch_histogram(hp, kb, s), "histogram launch");
  }
  // 2.-3. two stable binning sub-passes: low byte, then the high bits
  unsigned char* sub = ws + L.off_sub;
  uint32_t* status = reinterpret_cast<uint32_t*>(sub + L.pw.off_status);
  unsigned long long* scratch_carry = u64(L.off_rel);  // overwritten in step 5
  void* ak = ws + L.off_ak;
  void* av = vb ? ws + L.off_av : nullptr;
  void* bk = ws + L.off_bk;
  void* bv = vb ? ws + L.off_bv : nullptr;
  OS_CUDA(cudaMemsetAsync(sub, 0, L.pw.zero_bytes, s), "memset");
  if (int rc = run_pass(src_k, ak, src_v, av, kb, vb, L.t, shift, lo_w, kMaxRadix, nullptr,
                        u64(L.off_o8), scratch_carry, codec_in, CODEC_NONE, status, nullptr, sub,
                        L.pw, nullptr, s, /*dense_bases=*/true))
    return rc;
  if (hi_w > 0) {
    OS_CUDA(cudaMemsetAsync(sub, 0, L.pw.zero_bytes, s), "memset");
    if (int rc = run_pass(ak, bk, av, bv, kb, vb, L.t, shift + kMaxDigitBits, hi_w, kMaxRadix,
                          nullptr, u64(L.off_o8) + kMaxRadix, scratch_carry, CODEC_NONE, CODEC_NONE,
                          status, nullptr, sub, L.pw, nullptr, s, /*dense_bases=*/true))
      return rc;
  } else {  // the digit's high part lies past the key: the low sub-pass is the order
    bk = ak;
    bv = av;
  }
  // 4. dense starts of the full 2^width-way digit
  OS_CUDA(cudaMemsetAsync(ws + L.off_hw, 0, size_t(radix) * 8, s), "memset");
  OS_CUDA(launch_wide_histogram(bk, n, kb, CODEC_NONE, shift, width, 1, lo_w + hi_w, u64(L.off_hw),
                                s), "wide histogram launch");
  OS_CUDA(launch_exclusive_scan(u64(L.off_hw), 1, radix, u64(L.off_ow), s), "exclusive scan");
  // 5. rel = base - dense start, carry = base + count; 6. scatter to dst
  OS_CUDA(launch_wide_tables(base, u64(L.off_hw), u64(L.off_ow), radix, u64(L.off_rel), carry_out, s),
          "wide tables");
  OS_CUDA(launch_wide_scatter(bk, dst_k, bv, dst_v, kb, vb, n, shift, lo_w + hi_w, u64(L.off_rel),
                              codec_out, s), "wide scatter");
  return OS_OK;
}
}  // namespace

extern "C" {

size_t os_partition_workspace_bytes_kv(size_t n, int key_bytes, int val_bytes, int digit_width,
                                       int tile_keys, size_t strip_keys) {
  if (digit_width <= kMaxDigitBits)
    return os_partition_workspace_bytes(n, digit_width, tile_keys, strip_keys);
  if (digit_width > kMaxWideDigitBits || tile_keys <= 0 || (key_bytes != 4 && key_bytes != 8) ||
      !valid_val_bytes(val_bytes))
    return 0;
  size_t strip = strip_keys ? strip_keys : kMaxStripKeys;
  return wide_layout(n, key_bytes, val_bytes, digit_width, uint32_t(tile_keys), strip).total;
}

int os_partition_pass(const void* src_keys, void* dst_keys, const void* src_vals, void* dst_vals,
                      size_t n, int key_bytes, int val_bytes, int shift, int digit_width,
                      const unsigned long long* base_offsets, unsigned long long* carry_out,
                      int codec_in, int codec_out, int tile_keys, size_t strip_keys,
                      unsigned int* status_out, void* workspace, size_t workspace_bytes,
                      os_device_stats* stats, void* stream) {
  NvtxRange nvtx_range("onesweep partition_pass");
  if (key_bytes != 4 && key_bytes != 8) return fail(OS_ERR_ARG, "key_bytes must be 4 or 8");
  if (!valid_val_bytes(val_bytes)) return fail(OS_ERR_ARG, "val_bytes must be 0/1/2/4/8");
  if ((val_bytes == 0) != (src_vals == nullptr) || (val_bytes == 0) != (dst_vals == nullptr))
    return fail(OS_ERR_ARG, "values pointers must be given iff val_bytes > 0");
  if (digit_width < 1 || digit_width > kMaxWideDigitBits)
    return fail(OS_ERR_ARG, "digit width must be in [1, %d]", kMaxWideDigitBits);
  if (shift < 0 || shift >= key_bytes * 8) return fail(OS_ERR_ARG, "shift out of range");
  if (codec_in < 0 || codec_in > 3 || codec_out < 0 || codec_out > 3)
    return fail(OS_ERR_ARG, "bad codec");
  uint32_t tile;
  if (int rc = resolve_tile(tile_keys, key_bytes, val_bytes, &tile)) return rc;
  size_t strip;
  if (int rc = resolve_strip(strip_keys, &strip)) return rc;
  if (digit_width > kMaxDigitBits) {
    if (status_out != nullptr)
      return fail(OS_ERR_ARG, "status words are only kept for digit widths <= %d", kMaxDigitBits);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
      OS_CUDA(cudaMemcpyAsync(carry_out, base_offsets, (size_t(1) << digit_width) * 8,
                              cudaMemcpyDeviceToDevice, s), "carry copy");
      return OS_OK;
    }
    return wide_partition(src_keys, dst_keys, src_vals, dst_vals, n, key_bytes, val_bytes, shift,
                          digit_width, base_offsets, carry_out, codec_in, codec_out, tile, strip,
                          static_cast<unsigned char*>(workspace), workspace_bytes, s);
  }
  const int radix = 1 << digit_width;
  Tiling t = make_tiling(n, tile, strip);
  PassWs w = pass_ws(t, radix, true);
  if (workspace == nullptr || workspace_bytes < w.bytes)
    return fail(OS_ERR_WORKSPACE, "partition workspace needs %zu bytes, got %zu", w.bytes,
                workspace_bytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  uint32_t* status = reinterpret_cast<uint32_t*>(ws + w.off_status);
  if (n == 0) {
    OS_CUDA(cudaMemcpyAsync(carry_out, base_offsets, size_t(radix) * 8, cudaMemcpyDeviceToDevice, s),
            "carry copy");
    return OS_OK;
  }
  OS_CUDA(cudaMemsetAsync(ws, 0, w.zero_bytes, s), "partition memset");
  if (status_out)
    OS_CUDA(cudaMemsetAsync(status_out, 0, t.tiles_total * size_t(radix) * 4, s), "status memset");
  return run_pass(src_keys, dst_keys, src_vals, dst_vals, key_bytes, val_bytes, t, shift,
                  digit_width, radix, nullptr, base_offsets, carry_out, codec_in, codec_out, status,
                  status_out, ws, w, reinterpret_cast<unsigned long long*>(stats), s,
                  /*dense_bases=*/false);
}

size_t os_sort_workspace_bytes(size_t n, int key_type, int val_bytes, int digit_bits,
                               int begin_bit, int end_bit, int tile_keys, size_t strip_keys) {
  KeyType kt;
  if (!key_type_info(key_type, &kt) || !valid_val_bytes(val_bytes)) return 0;
  if (check_bits(kt.bytes, digit_bits, begin_bit, end_bit)) return 0;
  uint32_t tile;
  size_t strip;
  if (resolve_tile(tile_keys, kt.bytes, val_bytes, &tile) || resolve_strip(strip_keys, &strip))
    return 0;
  return sort_layout(n, kt.bytes, val_bytes, digit_bits, begin_bit, end_bit, tile, strip).total;
}

int os_sort_route_words(const void* workspace, size_t n, int key_type, int val_bytes,
                        int digit_bits, int begin_bit, int end_bit, int tile_keys,
                        size_t strip_keys, unsigned int* words, int max_passes, void* stream) {
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  if (!valid_val_bytes(val_bytes)) return fail(OS_ERR_ARG, "val_bytes must be 0/1/2/4/8");
  if (int rc = check_bits(kt.bytes, digit_bits, begin_bit, end_bit)) return rc;
  uint32_t tile;
  size_t strip;
  if (int rc = resolve_tile(tile_keys, kt.bytes, val_bytes, &tile)) return rc;
  if (int rc = resolve_strip(strip_keys, &strip)) return rc;
  const SortLayout L = sort_layout(n, kt.bytes, val_bytes, digit_bits, begin_bit, end_bit, tile, strip);
  if (words == nullptr || max_passes < L.passes)
    return fail(OS_ERR_ARG, "need room for %d passes", L.passes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n <= 1) {  // nothing ran: no place skipped (words may be host or device memory)
    static const uint32_t zeros[64] = {};
    OS_CUDA(cudaMemcpyAsync(words, zeros, size_t(L.passes) * sizeof(uint32_t), cudaMemcpyDefault, s),
            "route words");
    return OS_OK;
  }
  if (workspace == nullptr) return fail(OS_ERR_WORKSPACE, "null workspace");
  const unsigned char* ws = static_cast<const unsigned char*>(workspace);
  for (int k = 0; k < L.passes; ++k)
    OS_CUDA(cudaMemcpyAsync(words + k, ws + L.off_pass + size_t(k) * L.pw.bytes + L.pw.off_counters,
                            sizeof(uint32_t), cudaMemcpyDefault, s),
            "route words");
  return OS_OK;
}

static int sort_impl(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
                     size_t n, int key_type, int val_bytes, int digit_bits, int begin_bit,
                     int end_bit, int tile_keys, size_t strip_keys, void* workspace,
                     size_t workspace_bytes, os_device_stats* stats, void** events,
                     int num_events, void* stream) {
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  if (!valid_val_bytes(val_bytes)) return fail(OS_ERR_ARG, "val_bytes must be 0/1/2/4/8");
  if ((val_bytes == 0) != (vals_in == nullptr) || (val_bytes == 0) != (vals_out == nullptr))
    return fail(OS_ERR_ARG, "values pointers must be given iff val_bytes > 0");
  if (int rc = check_bits(kt.bytes, digit_bits, begin_bit, end_bit)) return rc;
  uint32_t tile;
  if (int rc = resolve_tile(tile_keys, kt.bytes, val_bytes, &tile)) return rc;
  size_t strip;
  if (int rc = resolve_strip(strip_keys, &strip)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int kb = kt.bytes, vb = val_bytes;

  if (n <= 1) {  // binning.py:306-309
    if (n == 1) {
      OS_CUDA(cudaMemcpyAsync(keys_out, keys_in, kb, cudaMemcpyDeviceToDevice, s), "copy");
      if (vb) OS_CUDA(cudaMemcpyAsync(vals_out, vals_in, vb, cudaMemcpyDeviceToDevice, s), "copy");
    }
    return OS_OK;
  }
  SortLayout L = sort_layout(n, kb, vb, digit_bits, begin_bit, end_bit, tile, strip);
  if (workspace == nullptr || workspace_bytes < L.total)
    return fail(OS_ERR_WORKSPACE, "sort workspace needs %zu bytes, got %zu", L.total,
                workspace_bytes);
  bool aliased = false;
  {
    // Aliasing: with an odd pass count pass 0 writes the caller's output while
    // other tiles still read the input, so no output may overlap any input.
    // With an even count the inputs are dead after pass 0 and may be reused.
    auto overlap = [](const void* a, size_t an, const void* b, size_t bn) {
      const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
      return an != 0 && bn != 0 && x < y + bn && y < x + an;
    };
    const size_t kbytes = n * kb, vbytes = n * vb;
    if (overlap(keys_out, kbytes, vals_out, vbytes))
      return fail(OS_ERR_ARG, "keys_out and vals_out overlap");
    aliased = overlap(keys_out, kbytes, keys_in, kbytes) || overlap(keys_out, kbytes, vals_in, vbytes) ||
              overlap(vals_out, vbytes, keys_in, kbytes) || overlap(vals_out, vbytes, vals_in, vbytes);
    if ((L.passes % 2) == 1 && aliased) return fail(OS_ERR_ARG, "in-place sort needs an even pass count");
  }
  if (n > size_t(osb::histogram_grid_size()) * (size_t(1) << 31))
    return fail(OS_ERR_ARG, "n too large");

  if (events != nullptr && num_events < L.passes + 2)
    return fail(OS_ERR_ARG, "need %d events, got %d", L.passes + 2, num_events);
  auto mark = [&](int i) -> cudaError_t {
    return events ? cudaEventRecord(static_cast<cudaEvent_t>(events[i]), s) : cudaSuccess;
  };
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  OS_CUDA(cudaMemsetAsync(ws + L.off_zero, 0, L.zero_bytes, s), "sort memset");
  OS_CUDA(mark(0), "event");

  unsigned long long* hist = reinterpret_cast<unsigned long long*>(ws + L.off_hist);
  unsigned long long* offsets = reinterpret_cast<unsigned long long*>(ws + L.off_offsets);
  HistParams hp{};
  hp.keys = keys_in;
  hp.n = n;
  hp.codec = kt.enc;
  hp.begin_bit = begin_bit;
  hp.digit_bits = digit_bits;
  hp.passes = L.passes;
  hp.top_bits = end_bit - (begin_bit + (L.passes - 1) * digit_bits);
  hp.hist = hist;
  hp.offsets = offsets;
  hp.done_counter = reinterpret_cast<unsigned int*>(ws + L.off_done);
  // Pass routing (plan_tickets): trivial places are skipped on the device,
  // the plan rides in the tile tickets.  In-place sorts keep the fixed
  // ping-pong (a skipped place would flip the parity and let a pass overwrite
  // input it still reads), and so does ONESWEEP_B200_NO_SKIP=1.
  const bool routed = !aliased && route_passes();
  if (routed) {
    hp.tickets = reinterpret_cast<uint32_t*>(ws + L.off_pass + L.pw.off_counters);
    hp.ticket_stride = L.pw.bytes / sizeof(uint32_t);
    hp.strips = int(L.t.strips);
    hp.fixed_ends = kt.enc != CODEC_NONE;
  }
  {
    NvtxRange r("onesweep histogram");
    OS_CUDA(launch_histogram(hp, kb, s), "histogram launch");
  }
  OS_CUDA(mark(1), "event");

  // Ping-pong so that the last pass lands in the caller's output buffer
  // (no parity copy, binning.py:327-334 is never needed).
  void* tmp_k = ws + L.off_tmp_k;
  void* tmp_v = ws + L.off_tmp_v;
  const void* src_k = keys_in;
  const void* src_v = vals_in;
  for (int k = 0; k < L.passes; ++k) {
    const bool to_out = ((L.passes - 1 - k) % 2) == 0;
    void* dst_k = to_out ? keys_out : tmp_k;
    void* dst_v = to_out ? vals_out : tmp_v;
    const int shift = begin_bit + k * digit_bits;
    const int width = (end_bit - shift) < digit_bits ? (end_bit - shift) : digit_bits;
    unsigned char* pws = ws + L.off_pass + size_t(k) * L.pw.bytes;
    uint32_t* status = reinterpret_cast<uint32_t*>(pws + L.pw.off_status);
    unsigned long long* carry_final =
        reinterpret_cast<unsigned long long*>(pws + L.pw.off_carry) +
        (L.t.strips - 1) * size_t(L.radix);
    NvtxRange r("onesweep pass %d", k);
    // (coded keys: the first and last places always run, so the codec masks
    // stay on pass 0 and the last pass, routed or not)
    const void* buf_k[3] = {keys_in, tmp_k, keys_out};
    const void* buf_v[3] = {vals_in, tmp_v, vals_out};
    int rc = run_pass(src_k, dst_k, src_v, dst_v, kb, vb, L.t, shift, width, L.radix, nullptr,
                      offsets + size_t(k) * L.radix, carry_final, k == 0 ? kt.enc : CODEC_NONE,
                      k == L.passes - 1 ? kt.dec : CODEC_NONE, status, nullptr, pws, L.pw,
                      reinterpret_cast<unsigned long long*>(stats), s, /*dense_bases=*/true,
                      k == g_trace_pass ? g_trace : nullptr, routed ? buf_k : nullptr,
                      routed ? buf_v : nullptr);
    if (rc) return rc;
    OS_CUDA(mark(2 + k), "event");
    src_k = dst_k;
    src_v = dst_v;
  }
  return OS_OK;
}

}  // extern "C"

extern "C" {

int os_sort(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out, size_t n,
            int key_type, int val_bytes, int digit_bits, int begin_bit, int end_bit, int tile_keys,
            size_t strip_keys, void* workspace, size_t workspace_bytes, os_device_stats* stats,
            void* stream) {
  return sort_impl(keys_in, keys_out, vals_in, vals_out, n, key_type, val_bytes, digit_bits,
                   begin_bit, end_bit, tile_keys, strip_keys, workspace, workspace_bytes, stats,
                   nullptr, 0, stream);
}

int os_sort_events(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
                   size_t n, int key_type, int val_bytes, int digit_bits, int begin_bit,
                   int end_bit, int tile_keys, size_t strip_keys, void* workspace,
                   size_t workspace_bytes, os_device_stats* stats, void** events,
                   int num_events, void* stream) {
  return sort_impl(keys_in, keys_out, vals_in, vals_out, n, key_type, val_bytes, digit_bits,
                   begin_bit, end_bit, tile_keys, strip_keys, workspace, workspace_bytes, stats,
                   events, num_events, stream);
}

int os_debug_trace(unsigned long long* buf, int pass) {
  g_trace = buf;
  g_trace_pass = buf ? pass : -1;
  return OS_OK;
}

int os_msd_histogram(const void* keys, size_t n, int key_type, int digit_bits, int end_bit,
                     unsigned long long* hist_out, void* stream) {
  NvtxRange nvtx_range("onesweep msd_histogram");
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  if (int rc = check_bits(kt.bytes, digit_bits, end_bit - digit_bits, end_bit)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  OS_CUDA(cudaMemsetAsync(hist_out, 0, (size_t(1) << digit_bits) * 8, s), "memset");
  if (n == 0) return OS_OK;
  HistParams p{};
  p.keys = keys;
  p.n = n;
  p.codec = kt.enc;
  p.begin_bit = end_bit - digit_bits;
  p.digit_bits = digit_bits;
  p.passes = 1;
  p.top_bits = digit_bits;
  p.hist = hist_out;
  p.offsets = nullptr;
  p.done_counter = nullptr;
  OS_CUDA(launch_histogram(p, kt.bytes, s), "msd histogram launch");
  return OS_OK;
}

}  // extern "C"

namespace {
__global__ void build_digit_map(const unsigned int* bin_lo, int parts, int radix, uint8_t* map) {
  const int r = threadIdx.x;
  if (r >= radix) return;
  int g = 0;
  while (g + 1 < parts && bin_lo[g + 1] <= unsigned(r)) ++g;
  map[r] = uint8_t(g);
}
}  // namespace

extern "C" {

size_t os_msd_partition_workspace_bytes(size_t n) {
  // status/tickets/carries for a pass with up to 256 destinations + the map
  Tiling t = make_tiling(n, uint32_t(binning_tile_capacity(8, 8)), kMaxStripKeys);
  return align_up(kMaxRadix) + pass_ws(t, kMaxRadix, true).bytes;
}

int os_msd_partition(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
                     size_t n, int key_type, int val_bytes, int digit_bits, int end_bit,
                     const unsigned int* bin_lo, int parts,
                     const unsigned long long* seg_offsets, void* workspace,
                     size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range("onesweep msd_partition");
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  if (!valid_val_bytes(val_bytes)) return fail(OS_ERR_ARG, "val_bytes must be 0/1/2/4/8");
  if ((val_bytes == 0) != (vals_in == nullptr) || (val_bytes == 0) != (vals_out == nullptr))
    return fail(OS_ERR_ARG, "values pointers must be given iff val_bytes > 0");
  if (int rc = check_bits(kt.bytes, digit_bits, end_bit - digit_bits, end_bit)) return rc;
  if (parts < 1 || parts > kMaxRadix) return fail(OS_ERR_ARG, "parts must be in [1, 256]");
  if (n == 0) return OS_OK;
  uint32_t tile;
  if (int rc = resolve_tile(0, kt.bytes, val_bytes, &tile)) return rc;
  // the workspace bound was computed with the smallest capacity; any tile
  // geometry of this build needs at most that many tiles
  Tiling t = make_tiling(n, tile, kMaxStripKeys);
  PassWs w = pass_ws(t, parts, true);
  const size_t need = align_up(kMaxRadix) + w.bytes;
  if (workspace == nullptr || workspace_bytes < need)
    return fail(OS_ERR_WORKSPACE, "msd workspace needs %zu bytes, got %zu", need, workspace_bytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  uint8_t* map = ws;
  unsigned char* pws = ws + align_up(kMaxRadix);
  OS_CUDA(cudaMemsetAsync(pws, 0, w.zero_bytes, s), "msd memset");
  build_digit_map<<<1, kMaxRadix, 0, s>>>(bin_lo, parts, 1 << digit_bits, map);
  OS_CUDA(cudaGetLastError(), "digit map");
  unsigned long long* carry_final =
      reinterpret_cast<unsigned long long*>(pws + w.off_carry) + (t.strips - 1) * size_t(parts);
  return run_pass(keys_in, keys_out, vals_in, vals_out, kt.bytes, val_bytes, t,
                  end_bit - digit_bits, digit_bits, parts, map, seg_offsets, carry_final, kt.enc,
                  kt.dec, reinterpret_cast<uint32_t*>(pws + w.off_status), nullptr, pws, w, nullptr,
                  s, /*dense_bases=*/true);
}

// Fused partition + exchange: the same stable partition, but segment g is
// written straight into destination g's receive buffer.  dest_index[g] is the
// element index, relative to keys_out (and vals_out), at which this rank's
// segment starts on destination g -- a two's-complement difference when
// keys_out and the peer buffer are different (peer-mapped) allocations.  With
// values, peer value buffers must sit at the same element distance from
// vals_out as the key buffers from keys_out (one symmetric allocation per
// rank, key_bytes == val_bytes).
int os_msd_partition_p2p(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out,
                         size_t n, int key_type, int val_bytes, int digit_bits, int end_bit,
                         const unsigned int* bin_lo, int parts,
                         const unsigned long long* dest_index, void* workspace,
                         size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_range("onesweep msd_partition_p2p");
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  if (val_bytes != 0 && val_bytes != kt.bytes)
    return fail(OS_ERR_ARG, "p2p exchange with values needs val_bytes == key_bytes");
  if ((val_bytes == 0) != (vals_in == nullptr) || (val_bytes == 0) != (vals_out == nullptr))
    return fail(OS_ERR_ARG, "values pointers must be given iff val_bytes > 0");
  if (int rc = check_bits(kt.bytes, digit_bits, end_bit - digit_bits, end_bit)) return rc;
  if (parts < 1 || parts > kMaxRadix) return fail(OS_ERR_ARG, "parts must be in [1, 256]");
  if (n == 0) return OS_OK;
  uint32_t tile;
  if (int rc = resolve_tile(0, kt.bytes, val_bytes, &tile)) return rc;
  Tiling t = make_tiling(n, tile, kMaxStripKeys);
  PassWs w = pass_ws(t, parts, true);
  const size_t need = align_up(kMaxRadix) + w.bytes;
  if (workspace == nullptr || workspace_bytes < need)
    return fail(OS_ERR_WORKSPACE, "msd workspace needs %zu bytes, got %zu", need, workspace_bytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  uint8_t* map = ws;
  unsigned char* pws = ws + align_up(kMaxRadix);
  OS_CUDA(cudaMemsetAsync(pws, 0, w.zero_bytes, s), "msd memset");
  build_digit_map<<<1, kMaxRadix, 0, s>>>(bin_lo, parts, 1 << digit_bits, map);
  OS_CUDA(cudaGetLastError(), "digit map");
  unsigned long long* carry_final =
      reinterpret_cast<unsigned long long*>(pws + w.off_carry) + (t.strips - 1) * size_t(parts);
  // dense_bases=false: 64-bit output indices, so the peer offsets wrap correctly
  return run_pass(keys_in, keys_out, vals_in, vals_out, kt.bytes, val_bytes, t,
                  end_bit - digit_bits, digit_bits, parts, map, dest_index, carry_final, kt.enc,
                  kt.dec, reinterpret_cast<uint32_t*>(pws + w.off_status), nullptr, pws, w, nullptr,
                  s, /*dense_bases=*/false);
}

// ---- reduce-then-scan ablation (baseline.py:121-173) ------
// The reference's rts_sort on the device: per digit place an upsweep (n key
// reads), a digit-major prefix over the per-tile table, and a downsweep that
// is the binning kernel with the look-back replaced by the table (2n), so
// 3n element transfers per place against Onesweep's 2n.  Full-width 8-bit
// places; the keys are encoded in the first upsweep/downsweep and decoded in
// the last downsweep like os_sort.
struct RtsLayout {
  int passes = 0;
  Tiling t;
  PassWs pw;
  size_t off_tmp_k = 0, off_tmp_v = 0, off_counts = 0, off_offsets = 0, off_csum = 0,
         off_pass = 0, total = 0;
};

static RtsLayout rts_layout(size_t n, int kb, int vb, uint32_t tile) {
  RtsLayout L;
  L.passes = kb * 8 / 8;
  L.t = make_tiling(n, tile, kMaxStripKeys);
  L.pw = pass_ws(L.t, kMaxRadix, /*own_status=*/false);
  const size_t tiles = L.t.tiles_total;
  size_t off = 0;
  L.off_tmp_k = off;
  off = align_up(off + n * kb);
  L.off_tmp_v = off;
  off = align_up(off + n * vb);
  L.off_counts = off;
  off = align_up(off + tiles * kMaxRadix * 4);
  L.off_offsets = off;
  off = align_up(off + tiles * kMaxRadix * 8);
  L.off_csum = off;
  off = align_up(off + rts_chunk_count(tiles) * kMaxRadix * 8);
  L.off_pass = off;
  off += L.pw.bytes;
  L.total = off;
  return L;
}

size_t os_rts_sort_workspace_bytes(size_t n, int key_type, int val_bytes) {
  KeyType kt;
  if (!key_type_info(key_type, &kt) || !valid_val_bytes(val_bytes)) return 0;
  uint32_t tile;
  if (resolve_tile(0, kt.bytes, val_bytes, &tile)) return 0;
  return rts_layout(n, kt.bytes, val_bytes, tile).total;
}

int os_rts_sort(const void* keys_in, void* keys_out, const void* vals_in, void* vals_out, size_t n,
                int key_type, int val_bytes, void* workspace, size_t workspace_bytes,
                void** events, int num_events, void* stream) {
  NvtxRange nvtx_range("onesweep rts_sort");
  KeyType kt;
  if (!key_type_info(key_type, &kt)) return fail(OS_ERR_KEYTYPE, "unsupported key type %d", key_type);
  if (!valid_val_bytes(val_bytes)) return fail(OS_ERR_ARG, "val_bytes must be 0/1/2/4/8");
  if ((val_bytes == 0) != (vals_in == nullptr) || (val_bytes == 0) != (vals_out == nullptr))
    return fail(OS_ERR_ARG, "values pointers must be given iff val_bytes > 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int kb = kt.bytes, vb = val_bytes;
  if (n <= 1) {  // baseline.py:151-153
    if (n == 1) {
      OS_CUDA(cudaMemcpyAsync(keys_out, keys_in, kb, cudaMemcpyDeviceToDevice, s), "copy");
      if (vb) OS_CUDA(cudaMemcpyAsync(vals_out, vals_in, vb, cudaMemcpyDeviceToDevice, s), "copy");
    }
    return OS_OK;
  }
  if (n >= (size_t(1) << 32)) return fail(OS_ERR_ARG, "rts sort supports n < 2^32");
  uint32_t tile;
  if (int rc = resolve_tile(0, kb, vb, &tile)) return rc;
  RtsLayout L = rts_layout(n, kb, vb, tile);
  if (workspace == nullptr || workspace_bytes < L.total)
    return fail(OS_ERR_WORKSPACE, "rts workspace needs %zu bytes, got %zu", L.total, workspace_bytes);
  if (events != nullptr && num_events < 3 * L.passes + 1)
    return fail(OS_ERR_ARG, "need %d events, got %d", 3 * L.passes + 1, num_events);
  auto mark = [&](int i) -> cudaError_t {
    return events ? cudaEventRecord(static_cast<cudaEvent_t>(events[i]), s) : cudaSuccess;
  };
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  uint32_t* counts = reinterpret_cast<uint32_t*>(ws + L.off_counts);
  unsigned long long* offsets = reinterpret_cast<unsigned long long*>(ws + L.off_offsets);
  unsigned long long* csum = reinterpret_cast<unsigned long long*>(ws + L.off_csum);
  unsigned char* pws = ws + L.off_pass;
  void* tmp_k = ws + L.off_tmp_k;
  void* tmp_v = ws + L.off_tmp_v;
  const void* src_k = keys_in;
  const void* src_v = vals_in;
  OS_CUDA(mark(0), "event");
  for (int k = 0; k < L.passes; ++k) {
    const bool to_out = ((L.passes - 1 - k) % 2) == 0;
    void* dst_k = to_out ? keys_out : tmp_k;
    void* dst_v = to_out ? vals_out : tmp_v;
    const int shift = 8 * k;
    // upsweep tiled exactly like the downsweep: per strip, so that the count
    // row of every downsweep tile is the one its upsweep tile wrote
    for (size_t st = 0, tb = 0; st < L.t.strips; tb += L.t.strip_tiles(st), ++st)
      OS_CUDA(launch_rts_upsweep(static_cast<const unsigned char*>(src_k) + st * L.t.strip * kb,
                                 L.t.strip_len(st), kb, tile, shift, 0xffu,
                                 k == 0 ? kt.enc : CODEC_NONE, counts + tb * kMaxRadix, s),
              "rts upsweep");
    OS_CUDA(mark(1 + 3 * k), "event");
    OS_CUDA(launch_rts_prefix(counts, uint32_t(L.t.tiles_total), kMaxRadix, csum, offsets, s),
            "rts prefix");
    OS_CUDA(mark(2 + 3 * k), "event");
    OS_CUDA(cudaMemsetAsync(pws, 0, L.pw.zero_bytes, s), "rts memset");
    // downsweep: the binning kernel, run starts from the table
    uint32_t* counters = reinterpret_cast<uint32_t*>(pws + L.pw.off_counters);
    unsigned long long* carries = reinterpret_cast<unsigned long long*>(pws + L.pw.off_carry);
    size_t tile_base = 0;
    for (size_t st = 0; st < L.t.strips; ++st) {
      PassParams p{};
      const size_t lo = st * L.t.strip;
      p.src_keys = static_cast<const unsigned char*>(src_k) + lo * kb;
      p.dst_keys = dst_k;
      p.src_vals = vb ? static_cast<const unsigned char*>(src_v) + lo * vb : nullptr;
      p.dst_vals = vb ? dst_v : nullptr;
      p.strip_n = uint32_t(L.t.strip_len(st));
      p.num_tiles = uint32_t(L.t.strip_tiles(st));
      p.tile_keys = tile;
      p.shift = shift;
      p.mask = 0xffu;
      p.radix = kMaxRadix;
      const int ci_code = k == 0 ? kt.enc : CODEC_NONE, co_code = k == L.passes - 1 ? kt.dec : CODEC_NONE;
      if (kb == 4) {
        const auto ci = XorCodec<uint32_t>::make(ci_code), co = XorCodec<uint32_t>::make(co_code);
        p.cin_m0 = ci.m0, p.cin_m1 = ci.m1, p.cout_m0 = co.m0, p.cout_m1 = co.m1;
      } else {
        const auto ci = XorCodec<uint64_t>::make(ci_code), co = XorCodec<uint64_t>::make(co_code);
        p.cin_m0 = ci.m0, p.cin_m1 = ci.m1, p.cout_m0 = co.m0, p.cout_m1 = co.m1;
      }
      p.base_offsets = nullptr;
      p.carry_out = carries + st * size_t(kMaxRadix);
      p.status = nullptr;
      p.tile_counter = counters + st;
      p.prefetch_tiles = prefetch_tiles();
      p.wide_index = n >= (size_t(1) << 32) - (size_t(1) << 26);
      p.rts_offsets = offsets + tile_base * kMaxRadix;
      OS_CUDA(launch_binning_pass(p, kb, vb, s), "rts downsweep launch");
      tile_base += p.num_tiles;
    }
    OS_CUDA(mark(3 + 3 * k), "event");
    src_k = dst_k;
    src_v = dst_v;
  }
  return OS_OK;
}

// ---- reduce-then-scan building blocks (baseline.py:55-118) ------------------
// The reference's rts_upsweep / rts_block_prefix / rts_downsweep as separate
// calls over one digit place, for callers that drive the comparator pass by
// pass (the reference's own tests do).  One strip, n < 2^32, widths <= 8.
int os_rts_upsweep(const void* keys, size_t n, int key_bytes, int codec, int shift, int digit_width,
                   int tile_keys, unsigned int* counts, void* stream) {
  if (key_bytes != 4 && key_bytes != 8) return fail(OS_ERR_ARG, "key_bytes must be 4 or 8");
  if (digit_width < 1 || digit_width > kMaxDigitBits)
    return fail(OS_ERR_ARG, "rts digit width must be in [1, %d]", kMaxDigitBits);
  if (shift < 0 || shift >= key_bytes * 8) return fail(OS_ERR_ARG, "shift out of range");
  if (codec < 0 || codec > 3) return fail(OS_ERR_ARG, "bad codec");
  if (tile_keys <= 0) return fail(OS_ERR_ARG, "tile_keys must be > 0");
  if (n >= (size_t(1) << 32)) return fail(OS_ERR_ARG, "rts passes support n < 2^32");
  if (n == 0) return OS_OK;
  OS_CUDA(launch_rts_upsweep(keys, n, key_bytes, uint32_t(tile_keys), shift,
                             (1u << digit_width) - 1u, codec, counts,
                             static_cast<cudaStream_t>(stream)),
          "rts upsweep");
  return OS_OK;
}

size_t os_rts_prefix_workspace_bytes(size_t tiles, int radix) {
  if (radix < 1 || radix > kMaxRadix) return 0;
  return rts_chunk_count(tiles) * size_t(radix) * 8;
}

int os_rts_block_prefix(const unsigned int* counts, size_t tiles, int radix,
                        unsigned long long* offsets, void* workspace, size_t workspace_bytes,
                        void* stream) {
  if (radix < 1 || radix > kMaxRadix || (radix & (radix - 1)) != 0)
    return fail(OS_ERR_ARG, "radix must be a power of two <= %d", kMaxRadix);
  if (tiles >= (size_t(1) << 32)) return fail(OS_ERR_ARG, "too many tiles");
  if (tiles == 0) return OS_OK;
  const size_t need = os_rts_prefix_workspace_bytes(tiles, radix);
  if (workspace == nullptr || workspace_bytes < need)
    return fail(OS_ERR_WORKSPACE, "rts prefix workspace needs %zu bytes, got %zu", need,
                workspace_bytes);
  OS_CUDA(launch_rts_prefix(counts, uint32_t(tiles), radix,
                            static_cast<unsigned long long*>(workspace), offsets,
                            static_cast<cudaStream_t>(stream)),
          "rts prefix");
  return OS_OK;
}

size_t os_rts_downsweep_workspace_bytes(void) { return 256; }

int os_rts_downsweep(const void* src_keys, void* dst_keys, const void* src_vals, void* dst_vals,
                     size_t n, int key_bytes, int val_bytes, int shift, int digit_width,
                     const unsigned long long* offsets, int tile_keys, int codec_in,
                     int codec_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (key_bytes != 4 && key_bytes != 8) return fail(OS_ERR_ARG, "key_bytes must be 4 or 8");
  if (!valid_val_bytes(val_bytes)) return fail(OS_ERR_ARG, "val_bytes must be 0/1/2/4/8");
  if ((val_bytes == 0) != (src_vals == nullptr) || (val_bytes == 0) != (dst_vals == nullptr))
    return fail(OS_ERR_ARG, "values pointers must be given iff val_bytes > 0");
  if (digit_width < 1 || digit_width > kMaxDigitBits)
    return fail(OS_ERR_ARG, "rts digit width must be in [1, %d]", kMaxDigitBits);
  if (shift < 0 || shift >= key_bytes * 8) return fail(OS_ERR_ARG, "shift out of range");
  if (codec_in < 0 || codec_in > 3 || codec_out < 0 || codec_out > 3)
    return fail(OS_ERR_ARG, "bad codec");
  const int cap = binning_tile_capacity(key_bytes, val_bytes);
  if (tile_keys <= 0 || tile_keys > cap)
    return fail(OS_ERR_ARG, "rts downsweep tile must be in [1, %d], got %d", cap, tile_keys);
  if (n >= (size_t(1) << 32)) return fail(OS_ERR_ARG, "rts passes support n < 2^32");
  if (n == 0) return OS_OK;
  if (workspace == nullptr || workspace_bytes < os_rts_downsweep_workspace_bytes())
    return fail(OS_ERR_WORKSPACE, "rts downsweep workspace needs %zu bytes",
                os_rts_downsweep_workspace_bytes());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  OS_CUDA(cudaMemsetAsync(workspace, 0, 4, s), "tile ticket");
  PassParams p{};
  p.src_keys = src_keys;
  p.dst_keys = dst_keys;
  p.src_vals = src_vals;
  p.dst_vals = dst_vals;
  p.strip_n = uint32_t(n);
  p.num_tiles = uint32_t((n + tile_keys - 1) / tile_keys);
  p.tile_keys = uint32_t(tile_keys);
  p.shift = shift;
  p.radix = 1 << digit_width;
  p.mask = uint32_t(p.radix - 1);
  if (key_bytes == 4) {
    const auto ci = XorCodec<uint32_t>::make(codec_in), co = XorCodec<uint32_t>::make(codec_out);
    p.cin_m0 = ci.m0, p.cin_m1 = ci.m1, p.cout_m0 = co.m0, p.cout_m1 = co.m1;
  } else {
    const auto ci = XorCodec<uint64_t>::make(codec_in), co = XorCodec<uint64_t>::make(codec_out);
    p.cin_m0 = ci.m0, p.cin_m1 = ci.m1, p.cout_m0 = co.m0, p.cout_m1 = co.m1;
  }
  p.tile_counter = static_cast<uint32_t*>(workspace);
  p.prefetch_tiles = prefetch_tiles();
  p.wide_index = true;  // caller-provided 64-bit run starts
  p.rts_offsets = offsets;
  OS_CUDA(launch_binning_pass(p, key_bytes, val_bytes, s), "rts downsweep launch");
  return OS_OK;
}

}  // extern "C"
