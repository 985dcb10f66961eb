"""Onesweep sort and single partition passes, on the B200.

Mirrors onesweep.binning (binning.py:1-337): `onesweep_sort` and
`partition_pass` keep the reference's signatures, argument meaning, return
types and exceptions; the per-tile pipeline (rank, publish, look-back,
reorder, scatter) and the thread pool around it are replaced by one sm_100a
kernel launch per digit place (csrc/binning.cu), after one upfront histogram
launch (csrc/histogram.cu).

Accepted inputs: numpy arrays (copied to the device and back: a drop-in for
the reference) or CUDA torch tensors (zero-copy, result on the device).
Additions over the reference: keyword-only `begin_bit` / `end_bit` (bits of
the *encoded* key, CUB convention) and `stream`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import as_device, from_device, is_tensor, launch_on, workspace
from .executor import Executor
from ._values import _gather_rows, _index_payload, _payload_width, _rows_as, _val_bytes, _value_rows
from .keycodec import MAX_DEVICE_DIGIT_BITS, RadixConfig, radix_plan, spec_for_dtype

LANE_GROUP = 32


@dataclass(frozen=True)
class StripCarry:
    """Per-digit 64-bit running global offsets chained between strips
    (binning.py:88-92)."""

    offsets: object  # uint64 numpy array or CUDA tensor, length radix


@dataclass
class SortBuffers:
    """Ping-pong buffers (binning.py:95-131).  The device sort routes its
    passes so that the last one lands in the output buffer, so no parity copy
    is ever needed; this helper is kept for callers that drive passes
    themselves."""

    keys_a: object
    keys_b: object
    values_a: object | None = None
    values_b: object | None = None
    live_in_a: bool = True

    @classmethod
    def allocate(cls, encoded, values) -> "SortBuffers":
        def empty_like(x):
            if is_tensor(x):
                import torch

                return torch.empty_like(x)
            return np.empty_like(x)

        def copy(x):
            return x.clone() if is_tensor(x) else x.copy()

        return cls(
            keys_a=encoded,
            keys_b=empty_like(encoded),
            values_a=None if values is None else copy(values),
            values_b=None if values is None else empty_like(values),
        )

    def src_keys(self):
        return self.keys_a if self.live_in_a else self.keys_b

    def dst_keys(self):
        return self.keys_b if self.live_in_a else self.keys_a

    def src_values(self):
        if self.values_a is None:
            return None
        return self.values_a if self.live_in_a else self.values_b

    def dst_values(self):
        if self.values_a is None:
            return None
        return self.values_b if self.live_in_a else self.values_a

    def swap(self) -> None:
        self.live_in_a = not self.live_in_a


@dataclass(frozen=True)
class TileRanking:
    """Per-tile digit counts plus a stable tile-relative rank per element
    (binning.py:41-46)."""

    digit_counts: np.ndarray  # int64, length radix
    ranks: np.ndarray  # int64, length tile


def _device_rank(digits, digit_bits: int) -> TileRanking:
    """Stable rank of every digit among equal digits, computed by the device
    binning kernel: a stable partition of (digit, index) pairs, inverted.  The
    kernel ranks by the same ballot multisplit as the reference's
    rank_tile_kernel (_kernels.py:31-82)."""
    import torch

    d = np.asarray(digits, dtype=np.int64)
    radix = 1 << digit_bits
    if d.size == 0:
        return TileRanking(np.zeros(radix, dtype=np.int64), np.zeros(0, dtype=np.int64))
    if d.min() < 0 or d.max() >= radix:
        raise ValueError(f"digits must lie in [0, {radix})")
    cfg = radix_plan(32, digit_bits)
    keys = d.astype(np.uint32)
    from .histogram import global_bin_offsets, global_histograms

    hist = global_histograms(keys, cfg)
    base = global_bin_offsets(hist).offsets[0]
    idx = np.arange(d.size, dtype=np.uint32)
    dst = np.zeros_like(keys)
    dvals = np.zeros_like(idx)
    partition_pass(keys, dst, 0, base, cfg, None, idx, dvals)
    slot = torch.empty(d.size, dtype=torch.int64, device="cuda")
    slot[torch.from_numpy(dvals.astype(np.int64)).cuda()] = torch.arange(d.size, device="cuda")
    dd = torch.from_numpy(d).cuda()
    b = torch.from_numpy(base.astype(np.int64)).cuda()
    ranks = (slot - b[dd]).cpu().numpy()
    return TileRanking(hist.counts[0].astype(np.int64), ranks)


def wlms_rank(digits, digit_bits: int):
    """Rank one lane group of at most 32 digits (binning.py:50-68).  Returns
    (counts[2^digit_bits], stable ranks); ValueError for more than 32."""
    d = np.asarray(digits, dtype=np.int64)
    if d.size > LANE_GROUP:
        raise ValueError(f"lane group holds at most {LANE_GROUP} values")
    r = _device_rank(d, digit_bits)
    return r.digit_counts, r.ranks


def rank_tile(digits, cfg: RadixConfig) -> TileRanking:
    """Stable tile-wide ranking (binning.py:71-76), on the device."""
    return _device_rank(digits, cfg.digit_bits)


def short_circuit_check(ranking: TileRanking) -> int | None:
    """The single digit covering the whole tile, or None (binning.py:79-85)."""
    n = ranking.ranks.size
    if n == 0:
        return None
    top = int(np.argmax(ranking.digit_counts))
    return top if int(ranking.digit_counts[top]) == n else None


def _numel(x) -> int:
    return x.numel() if is_tensor(x) else int(np.asarray(x).size)


def _copy(x):
    return x.clone() if is_tensor(x) else np.array(x, copy=True)


def _device_digit_bits(cfg: RadixConfig) -> int:
    # A stable LSD sort has one answer for every digit width, so wider
    # configured digits run as 8-bit places on the device.
    return min(cfg.digit_bits, MAX_DEVICE_DIGIT_BITS)


def skipped_from_route_words(words) -> list[bool]:
    """Decode os_sort_route_words: top five bits all ones = skipped place."""
    return [((int(w) & 0xFFFFFFFF) >> 27) == 31 for w in words.cpu().tolist()]


class DeviceSorter:
    """Pre-planned device sort of n keys (optionally with values).

    Allocates the workspace once; `__call__` issues exactly one histogram and
    `passes` binning launches on the stream, with no host synchronisation.
    This is what bench.py times."""

    def __init__(self, n: int, key_dtype, val_bytes: int = 0, digit_bits: int = 8,
                 begin_bit: int = 0, end_bit: int | None = None, tile_size: int = 0,
                 strip_size: int = 0, device=None, graphs: bool = True):
        import torch

        self.spec = spec_for_dtype(key_dtype)
        self.n = int(n)
        self.val_bytes = int(val_bytes)
        self.digit_bits = int(digit_bits)
        self.begin_bit = int(begin_bit)
        self.end_bit = self.spec.bits if end_bit is None else int(end_bit)
        L = _native.load()
        cap = L.os_tile_capacity(self.spec.bits // 8, self.val_bytes)
        self.tile = min(int(tile_size), cap) if tile_size else cap
        self.strip = int(strip_size)
        self.passes = -(-(self.end_bit - self.begin_bit) // self.digit_bits)
        nbytes = L.os_sort_workspace_bytes(self.n, self.spec.type_id, self.val_bytes,
                                           self.digit_bits, self.begin_bit, self.end_bit,
                                           self.tile, self.strip)
        if self.n > 1 and nbytes == 0:
            raise ValueError("invalid sort parameters: " + L.os_last_error().decode())
        self.device = torch.device(device or "cuda")
        self.ws = workspace(nbytes, self.device)
        self.stats = torch.zeros(5, dtype=torch.int64, device=self.device)
        self.graphs = graphs
        self._graphs: dict = {}  # call signature -> captured CUDA graph (None: seen once)

    def _launch(self, keys, keys_out, values, values_out, stream, stats):
        _native.check(
            _native.load().os_sort(
                _native.ptr(keys), _native.ptr(keys_out), _native.ptr(values),
                _native.ptr(values_out), self.n, self.spec.type_id, self.val_bytes,
                self.digit_bits, self.begin_bit, self.end_bit, self.tile, self.strip,
                _native.ptr(self.ws), self.ws.numel(),
                _native.ptr(self.stats) if stats else None, _native.stream_handle(stream)),
            "onesweep_sort",
        )

    def route_words(self, stream=None):
        """After a sort on `stream`: a device tensor with each pass's first
        tile-ticket word (os_sort_route_words); asynchronous."""
        import torch

        words = torch.empty(self.passes, dtype=torch.int32, device=self.device)
        _native.check(
            _native.load().os_sort_route_words(
                _native.ptr(self.ws), self.n, self.spec.type_id, self.val_bytes, self.digit_bits,
                self.begin_bit, self.end_bit, self.tile, self.strip, _native.ptr(words), self.passes,
                _native.stream_handle(stream)),
            "route_words",
        )
        return words

    def skipped_places(self, stream=None) -> list[bool]:
        """After a sort on `stream`: which digit places held every key in one
        bin and were skipped on the device (waits for the stream)."""
        return skipped_from_route_words(self.route_words(stream))

    def __call__(self, keys, keys_out, values=None, values_out=None, stream=None, stats=True):
        """Sort on `stream` (default: the current stream).  With `graphs`
        on, a repeat of the same call (same buffers, stream and stats flag)
        replays the sort's launches as one CUDA graph: the kernels and their
        order are identical, the per-launch gaps shrink (C1: 233 -> 220 us per
        sort, tools/graph_probe.py).  The first call runs directly (and sets
        the kernels' attributes), the second captures, later ones replay."""
        if not self.graphs:
            self._launch(keys, keys_out, values, values_out, stream, stats)
            return keys_out if values is None else (keys_out, values_out)
        import torch

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        key = (_native.ptr(keys), _native.ptr(keys_out), _native.ptr(values), _native.ptr(values_out),
               st.cuda_stream, bool(stats))
        g = self._graphs.get(key)
        if g is None and key not in self._graphs:
            if len(self._graphs) >= 8:  # a few buffer sets (SortPipeline rotates three)
                self._graphs.pop(next(iter(self._graphs)))
            self._graphs[key] = None  # seen once: run directly
            self._launch(keys, keys_out, values, values_out, st, stats)
        else:
            if g is None:
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(self.device)
                side.wait_stream(st)
                with torch.cuda.graph(g, stream=side):
                    self._launch(keys, keys_out, values, values_out, side, stats)
                st.wait_stream(side)
                self._graphs[key] = g
            with torch.cuda.stream(st):
                g.replay()
        return keys_out if values is None else (keys_out, values_out)


def onesweep_sort(keys, values=None, cfg: RadixConfig | None = None,
                  executor: Executor | None = None, *, begin_bit: int = 0,
                  end_bit: int | None = None, stream=None):
    """Stable ascending sort (binning.py:278-337).

    Returns the sorted keys, or (sorted keys, reordered values) when values
    are given.  Inputs are never modified.  Same container type out as in."""
    to_numpy = not is_tensor(keys)
    if to_numpy:
        keys = np.asarray(keys)
    spec = spec_for_dtype(keys.dtype)  # KeyError for unsupported dtypes
    # without a config the tile is the device's own (its largest tile for the
    # key/value widths); an explicit config's tile_size is honoured up to it
    device_tile = cfg is None
    if cfg is None:
        cfg = radix_plan(spec.bits, 8)
    elif cfg.key_bits != spec.bits:
        raise ValueError(
            f"config is for {cfg.key_bits}-bit keys but got {spec.bits}-bit {spec.name}"
        )
    if executor is None:
        executor = Executor()
    if values is not None:
        if not is_tensor(values):
            values = np.asarray(values)
        if tuple(values.shape) != tuple(keys.shape):
            raise ValueError("values must have the same length as keys")
    end_bit = spec.bits if end_bit is None else int(end_bit)
    if not 0 <= begin_bit < end_bit <= spec.bits:
        raise ValueError(f"need 0 <= begin_bit < end_bit <= {spec.bits}, got [{begin_bit}, {end_bit})")
    vb = _val_bytes(values)

    n = _numel(keys)
    if n <= 1:  # binning.py:306-309
        sorted_keys = _copy(keys)
        return sorted_keys if values is None else (sorted_keys, _copy(values))

    import torch

    dk, _ = as_device(keys)
    wide = values is not None and not _payload_width(vb)
    if wide:  # values ride as an index payload, gathered after the sort
        wide_values = values
        dv, vb = _index_payload(n, dk.device)
    else:
        dv = as_device(values)[0] if values is not None else None
    ok = torch.empty_like(dk)
    ov = torch.empty_like(dv) if dv is not None else None
    d = _device_digit_bits(cfg)
    sorter = DeviceSorter(n, dk.dtype, vb, d, begin_bit, end_bit,
                          0 if device_tile else cfg.tile_size, cfg.strip_size, device=dk.device)
    launch_on(stream if stream is not None else executor.stream,
              (dk, ok, dv, ov, sorter.ws, sorter.stats),
              lambda s: sorter(dk, ok, dv, ov, stream=s))
    # The ledger is the algorithmic traffic of the configured plan, as the
    # reference defines it (binning.py:268-272, executor.py:10-14): one read
    # for the histogram, one read and one write per cfg.digit_bits place.
    # For cfg.digit_bits > 8 the device runs 8-bit places (same output); its
    # own element moves are in executor.device_element_ops.
    plan_passes = -(-(end_bit - begin_bit) // cfg.digit_bits)
    executor.ledger_record("histogram", "element_reads", n)
    executor.ledger_record("partition", "element_reads", plan_passes * n)
    executor.ledger_record("partition", "element_writes", plan_passes * n)
    if plan_passes % 2 == 1:
        # the reference's plan delivers an odd pass count with a parity copy,
        # its own ledger line (binning.py:327-334); the device routes the
        # passes so the last one writes the output and copies nothing, which
        # device_element_ops records
        executor.ledger_record("copy", "copy_ops", 2 * n)
    # places the device skipped (one bin held every key) move no elements;
    # the route words are copied now and decoded when the count is read
    executor.record_device_route(n, sorter.route_words(stream if stream is not None else executor.stream))
    executor.record_device_stats("partition", sorter.stats, 1 << d)
    sk = from_device(ok, to_numpy)
    if values is None:
        return sk
    if wide:
        rows = _gather_rows(_value_rows(wide_values, dk.device), ov, vb)
        return sk, _rows_as(rows, wide_values, to_numpy)
    return sk, from_device(ov, to_numpy and not is_tensor(values))


def partition_pass(src_keys, dst_keys, place: int, offsets, cfg: RadixConfig,
                   executor: Executor | None = None, src_values=None, dst_values=None, *,
                   return_status: bool = False):
    """Stable radix-way partition of src into dst by the digit at `place`
    (binning.py:218-275).

    `offsets` is the place's global bin-offset row or a StripCarry; returns
    the StripCarry folding in every digit count of this call.  Numpy `dst`
    arrays are updated in place, as in the reference.  With return_status the
    final status words are returned as well: a list of per-strip
    lookback.CounterMatrix views."""
    import torch

    from .lookback import CounterMatrix

    if return_status and cfg.digit_bits > MAX_DEVICE_DIGIT_BITS:
        raise ValueError(f"status words are only kept for digit_bits <= {MAX_DEVICE_DIGIT_BITS}")
    executor = executor or Executor()
    shift = cfg.digit_shift(place)
    src_np = not is_tensor(src_keys)
    sk, _ = as_device(src_keys)
    if sk.element_size() * 8 != cfg.key_bits:
        raise ValueError(f"config is for {cfg.key_bits}-bit keys")
    dk, _ = as_device(dst_keys)
    sv = dv = None
    vb = _val_bytes(src_values)
    wide = src_values is not None and not _payload_width(vb)
    if wide:  # values ride as an index payload, gathered after the pass
        sv, vb = _index_payload(sk.numel(), sk.device)
        dv = torch.empty_like(sv)
    elif src_values is not None:
        sv, _ = as_device(src_values)
        dv, _ = as_device(dst_values)
    base = offsets.offsets if isinstance(offsets, StripCarry) else offsets
    if is_tensor(base):
        base_dev = base.to(sk.device).contiguous()
        carry_numpy = False
    else:
        base_dev, _ = as_device(np.ascontiguousarray(np.asarray(base, dtype=np.uint64)))
        carry_numpy = True
    carry = torch.empty(cfg.radix, dtype=torch.uint64, device=sk.device)
    L = _native.load()
    n = sk.numel()
    cap = L.os_tile_capacity(cfg.key_bits // 8, vb)
    tile = min(cfg.tile_size, cap)
    ws = workspace(L.os_partition_workspace_bytes_kv(n, cfg.key_bits // 8, vb, cfg.digit_bits, tile,
                                                     cfg.strip_size), sk.device)
    status = None
    if return_status:
        words = L.os_partition_status_words(n, cfg.digit_bits, tile, cfg.strip_size)
        status = torch.zeros(max(words, 1), dtype=torch.int32, device=sk.device)
    stats = torch.zeros(5, dtype=torch.int64, device=sk.device)
    _native.check(
        L.os_partition_pass(_native.ptr(sk), _native.ptr(dk), _native.ptr(sv), _native.ptr(dv), n,
                            cfg.key_bits // 8, vb, shift, cfg.digit_bits, _native.ptr(base_dev),
                            _native.ptr(carry), _native.CODEC_NONE, _native.CODEC_NONE, tile,
                            cfg.strip_size, _native.ptr(status), _native.ptr(ws), ws.numel(),
                            _native.ptr(stats), _native.stream_handle(executor.stream)),
        "partition_pass",
    )
    executor.ledger_record("partition", "element_reads", n)
    executor.ledger_record("partition", "element_writes", n)
    executor.record_device_stats("partition", stats, cfg.radix)
    if wide and dst_values is not None:
        rows = _gather_rows(_value_rows(src_values, sk.device), dv, vb, executor.stream)
        if is_tensor(dst_values):
            dst_values.copy_(_rows_as(rows, dst_values, False))
        else:
            np.copyto(dst_values, _rows_as(rows, dst_values, True))
    if src_np or not is_tensor(dst_keys):
        np.copyto(dst_keys, dk.cpu().numpy().view(np.asarray(dst_keys).dtype))
        if dst_values is not None and not wide:
            np.copyto(dst_values, dv.cpu().numpy().view(np.asarray(dst_values).dtype))
    else:
        if dk.data_ptr() != dst_keys.data_ptr():
            dst_keys.copy_(dk)
        if dst_values is not None and not wide and dv.data_ptr() != dst_values.data_ptr():
            dst_values.copy_(dv)
    result = StripCarry(carry.cpu().numpy() if carry_numpy else carry)
    if not return_status:
        return result
    words = status.view(torch.uint32).cpu().numpy() if n else np.zeros(0, np.uint32)
    views, pos = [], 0
    for lo in range(0, n, cfg.strip_size):
        tiles = -(-min(cfg.strip_size, n - lo) // tile)
        views.append(CounterMatrix(words[pos: pos + tiles * cfg.radix].reshape(tiles, cfg.radix)))
        pos += tiles * cfg.radix
    return result, views


def process_tile(tile_index: int, keys_tile, out_keys, place: int, base_offsets, counters,
                 cfg: RadixConfig, values_tile=None, out_values=None, carry_out=None,
                 jitter=None):
    """One tile of a pass driven from the host (binning.py:162-215): the
    tile's exclusive prefix comes from the predecessors' words in `counters`
    (a host lookback.CounterMatrix), the tile is partitioned on the device by
    os_partition_pass into `out_keys` at base + exclusive + rank, and the
    tile's L and G words are published.  Returns the tile's LedgerCounts.

    The sort itself never calls this: on the device every tile runs the whole
    pipeline inside the binning kernel.  It exists for callers that drive
    single tiles, as the reference's own tests do."""
    import torch

    from .executor import LedgerCounts

    if jitter is not None:
        jitter.pause()
    exclusive, reads = counters.lookback_exclusive_row(tile_index)
    base = np.asarray(base_offsets, dtype=np.uint64).astype(np.int64) + exclusive
    n = _numel(keys_tile)
    ex = Executor()
    if n:
        # (a tile larger than the device tile runs as several device tiles
        # chained by the kernel's own look-back: same placement)
        carry = partition_pass(keys_tile, out_keys, place, base.astype(np.uint64), cfg, ex,
                               values_tile, out_values)
        off = carry.offsets
        total = off.to(torch.int64).cpu().numpy() if is_tensor(off) else off.astype(np.int64)
        counts = total - base
    else:
        counts = np.zeros(cfg.radix, dtype=np.int64)
    counters.publish_local_row(tile_index, counts)
    if jitter is not None:
        jitter.pause()
    inclusive = exclusive + counts
    counters.publish_inclusive_row(tile_index, inclusive)
    counter_ops = 2 * cfg.radix + reads
    if carry_out is not None:
        carry_out[:] = np.asarray(base_offsets, dtype=np.uint64) + inclusive.astype(np.uint64)
        counter_ops += cfg.radix
    fast = int(n > 0 and counts.max() == n)
    return LedgerCounts(element_reads=n, element_writes=n, counter_ops=counter_ops,
                        fast_path_tiles=fast)
