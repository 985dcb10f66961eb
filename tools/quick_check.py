"""Fast device-path correctness check for a library variant (A/B sessions):
keys-only and pairs sorts at several sizes compared with torch's stable sort.
usage: ONESWEEP_B200_LIB=... python tools/quick_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort  # noqa: E402

ok = True
for n, q, dt in [(1 << 24, 1, 32), (12345679, 1, 32), ((1 << 28), 1, 32), (1 << 24, 4, 32),
                 (1 << 22, 1, 64), (3000, 1, 32), (1 << 20, 16, 32)]:
    keys = generate_keys(KeyGenSpec(q=q, seed=n, n=n, key_bits=dt), device="cuda:0")
    if dt == 32:
        ref = torch.sort(keys.to(torch.int64) & 0xFFFFFFFF, stable=True)
        good = torch.equal(onesweep_sort(keys).to(torch.int64) & 0xFFFFFFFF, ref.values)
        vals = torch.arange(n, dtype=torch.int32, device="cuda:0").view(torch.uint32)
        sk, sv = onesweep_sort(keys, vals)
        good &= torch.equal(sv.view(torch.int32).to(torch.int64), ref.indices)
    else:
        flip = -(1 << 63)  # unsigned order through a sign flip
        ref = torch.sort(keys.view(torch.int64) ^ flip, stable=True)
        good = torch.equal(onesweep_sort(keys).view(torch.int64) ^ flip, ref.values)
    print(f"n={n} q={q} bits={dt}: {'ok' if good else 'MISMATCH'}", flush=True)
    ok &= bool(good)
    del keys
    torch.cuda.empty_cache()
print("QUICK_CHECK", "PASS" if ok else "FAIL")
sys.exit(0 if ok else 1)
