"""Entropy-banded key generation on the device (keygen.py:1-105).

`generate_keys` is bit-identical to the reference: key i is the AND of q
splitmix64 words at counters i*q .. i*q+q-1, truncated to the key width.  It
runs as one elementwise kernel (os_keygen), so 2^31-key inputs never touch
host memory.  With `device=None` it returns numpy like the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _native

_LN2 = math.log(2.0)


@dataclass(frozen=True)
class KeyGenSpec:
    """Parameters for one generated dataset (keygen.py:28-43)."""

    q: int
    seed: int
    n: int
    key_bits: int = 32

    def __post_init__(self) -> None:
        if self.q < 1:
            raise ValueError(f"q must be >= 1, got {self.q}")
        if self.n < 0:
            raise ValueError(f"n must be >= 0, got {self.n}")
        if self.key_bits not in (32, 64):
            raise ValueError(f"key_bits must be 32 or 64, got {self.key_bits}")


def generate_keys(spec: KeyGenSpec, *, device=None, first_index: int = 0, out=None):
    """AND of q uniform words per key (keygen.py:63-76).

    device=None -> numpy array (reference behaviour); otherwise a CUDA tensor.
    first_index / out let callers generate one shard of a larger dataset."""
    import torch

    from ._device import require_cuda

    require_cuda()
    dt = torch.uint32 if spec.key_bits == 32 else torch.uint64
    dev = torch.device(device) if device is not None else torch.device("cuda")
    t = out if out is not None else torch.empty(spec.n, dtype=dt, device=dev)
    _native.check(
        _native.load().os_keygen(_native.ptr(t), spec.n, spec.key_bits, spec.q,
                                 spec.seed & 0xFFFFFFFFFFFFFFFF, first_index,
                                 _native.stream_handle()),
        "generate_keys",
    )
    return t.cpu().numpy() if device is None and out is None else t


def binary_entropy(p: float) -> float:
    """Shannon entropy of a Bernoulli(p) bit (keygen.py:79-84)."""
    if p <= 0.0 or p >= 1.0:
        return 0.0
    return -(p * math.log2(p) + (1.0 - p) * math.log1p(-p) / _LN2)


def expected_entropy(q: int) -> float:
    """H(2**-q) (keygen.py:87-91)."""
    if q < 1:
        raise ValueError(f"q must be >= 1, got {q}")
    return binary_entropy(2.0 ** -q)


def empirical_bit_entropy(keys) -> float:
    """Mean over bit positions of H(fraction of ones at that bit)
    (keygen.py:94-105).  Counted on the device: one popcount reduction per bit
    position over the keys (numpy input is uploaded once)."""
    import torch

    from ._device import as_device

    dev, _ = as_device(keys)
    n = dev.numel()
    if n == 0:
        raise ValueError("empirical_bit_entropy requires at least one key")
    width = dev.element_size() * 8
    w = dev.view(torch.int32 if width == 32 else torch.int64)
    ones = torch.stack([((w >> b) & 1).sum(dtype=torch.int64) for b in range(width)]).tolist()
    return sum(binary_entropy(c / n) for c in ones) / width
