"""GPU: DeviceSorter's CUDA-graph replay (first call direct, second captured,
later ones replayed) sorts whatever the bound buffers hold at replay time,
with and without values, on the current or a named stream."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(keys, vals):
    order = torch.sort(keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, stable=True).indices
    return keys.view(torch.int32)[order].view(torch.uint32), vals.view(torch.int32)[order].view(torch.uint32)


@pytest.mark.parametrize("named_stream", [False, True])
def test_graph_replays_sort_fresh_contents(cuda, named_stream):
    from paper_2206_01784_b200 import DeviceSorter

    n = 300_001
    keys = torch.empty(n, dtype=torch.uint32, device="cuda")
    vals = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    s = DeviceSorter(n, torch.uint32, 4)
    st = torch.cuda.Stream() if named_stream else None
    g = torch.Generator(device="cuda").manual_seed(7)
    for call in range(5):  # direct, capture + replay, replay x3
        keys.view(torch.int32).copy_(torch.randint(-2**31, 2**31 - 1, (n,), device="cuda", generator=g,
                                                   dtype=torch.int64).to(torch.int32))
        if st is not None:
            st.wait_stream(torch.cuda.current_stream())
        s(keys, ko, vals, vo, stream=st, stats=False)
        if st is not None:
            torch.cuda.current_stream().wait_stream(st)
        want_k, want_v = _ref(keys, vals)
        assert torch.equal(ko, want_k) and torch.equal(vo, want_v), call
    assert sum(v is not None for v in s._graphs.values()) == 1


def test_graph_cache_follows_buffers(cuda):
    from paper_2206_01784_b200 import DeviceSorter

    n = 50_000
    s = DeviceSorter(n, torch.uint32)
    bufs = [(torch.randint(0, 2**31, (n,), device="cuda", dtype=torch.int64).to(torch.uint32),
             torch.empty(n, dtype=torch.uint32, device="cuda")) for _ in range(3)]
    for _ in range(3):
        for k, o in bufs:
            s(k, o, stats=False)
            want = torch.sort(k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values
            assert torch.equal(o.view(torch.int32).to(torch.int64) & 0xFFFFFFFF, want)
    assert sum(v is not None for v in s._graphs.values()) == 3
