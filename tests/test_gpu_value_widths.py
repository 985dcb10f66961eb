"""Every (key, value) width at scale: the drop-in takes any value dtype
(binning.py:301-304), and each width pair runs its own kernel geometry
(Geometry<KB, VB> in csrc/binning.cu).  Checked byte for byte against
torch's stable sort of the same keys (its indices are the stable
permutation), at 2^26 keys for every width and at 2^28 for the two common
drop-in shapes: u64 keys alone and u32 keys with numpy's default int64
arange payload."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

SIGN = -(1 << 63)


def _keys(n, bits, seed):
    from paper_2206_01784_b200 import KeyGenSpec, generate_keys

    return generate_keys(KeyGenSpec(q=1, seed=seed, n=n, key_bits=bits), device="cuda")


def _stable_order(keys):
    import torch

    if keys.element_size() == 4:
        order_key = keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    else:
        order_key = keys.view(torch.int64) ^ SIGN  # unsigned order as signed
    return torch.sort(order_key, stable=True).indices


def _s(t):
    """Signed view (torch's CUDA gather/compare kernels skip the unsigned dtypes)."""
    import torch

    return t.view({1: torch.int8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[t.element_size()])


def _payload(n, vb):
    import torch

    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[vb]
    return (torch.arange(n, device="cuda") * 2654435761).to(dt)  # distinct-ish, all bytes used


@pytest.mark.parametrize("kbits", [32, 64])
@pytest.mark.parametrize("vb", [0, 1, 2, 4, 8])
def test_value_widths_2e26(cuda, kbits, vb):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = (1 << 26) + 4097  # ragged last tile
    keys = _keys(n, kbits, seed=kbits + vb)
    order = _stable_order(keys)
    if vb == 0:
        out = onesweep_sort(keys)
        assert torch.equal(_s(out), _s(keys)[order])
        return
    vals = _payload(n, vb)
    sk, sv = onesweep_sort(keys, vals)
    assert torch.equal(_s(sk), _s(keys)[order])
    assert torch.equal(_s(sv), _s(vals)[order])


@pytest.mark.slow
def test_u64_keys_only_2e28(cuda):
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = 1 << 28
    keys = _keys(n, 64, seed=0)
    want = torch.sort(keys.view(torch.int64) ^ SIGN).values ^ SIGN
    assert torch.equal(_s(onesweep_sort(keys)), want)


@pytest.mark.slow
def test_u32_keys_int64_arange_payload_2e28(cuda):
    """numpy argsort-style payload: int64 positions (np.arange's default)."""
    import torch

    from paper_2206_01784_b200 import onesweep_sort

    n = 1 << 28
    keys = _keys(n, 32, seed=0)
    idx = torch.arange(n, dtype=torch.int64, device="cuda")
    sk, sv = onesweep_sort(keys, idx)
    order = _stable_order(keys)
    assert torch.equal(sv, order)
    assert torch.equal(_s(sk), _s(keys)[order])
