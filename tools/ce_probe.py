"""Copy-engine probe: is the H2D / D2H overlap a property of the stream pair?
For several pairs of fresh streams, time a 1 GiB H2D on one and a 1 GiB D2H
on the other at once (pinned host memory).  python tools/ce_probe.py"""
import ctypes
import time

import torch

rt = ctypes.CDLL("libcudart.so.12")
v = ctypes.c_int(0)
rt.cudaDeviceGetAttribute(ctypes.byref(v), 40, 0)  # cudaDevAttrAsyncEngineCount
print("asyncEngineCount", v.value)
n = 1 << 28
hin = torch.empty(n, dtype=torch.uint32, pin_memory=True)
hout = torch.empty(n, dtype=torch.uint32, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint32, device="cuda")
d_out = torch.ones(n, dtype=torch.uint32, device="cuda")


def duplex(s1, s2, reps=2):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            d_in.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def raw_stream(flags=1):
    h = ctypes.c_void_p()
    assert rt.cudaStreamCreateWithFlags(ctypes.byref(h), flags) == 0
    return torch.cuda.ExternalStream(h.value)


for i in range(6):
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    print(f"pool pair {i}: ids {s1.stream_id} {s2.stream_id}: {duplex(s1, s2):.1f} ms")
for i in range(6):
    s1, s2 = raw_stream(), raw_stream()
    print(f"fresh non-blocking pair {i}: {duplex(s1, s2):.1f} ms")
hi = torch.cuda.Stream(priority=-1)
print(f"low/high priority pair: {duplex(torch.cuda.Stream(), hi):.1f} ms")
# one stream, chunks alternating direction
s = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s):
    for c in range(8):
        sl = slice(c * n // 8, (c + 1) * n // 8)
        d_in[sl].copy_(hin[sl], non_blocking=True)
        hout[sl].copy_(d_out[sl], non_blocking=True)
torch.cuda.synchronize()
print(f"one stream, alternating 128 MiB chunks: {(time.perf_counter() - t0) * 1e3:.1f} ms")
