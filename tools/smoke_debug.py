"""Run __graft_entry__.smoke() step by step with timestamps (debugging aid)."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(90, repeat=True)
t0 = time.time()


def log(msg):
    print(f"[{time.time() - t0:7.2f}s] {msg}", flush=True)


log("import torch")
import torch  # noqa: E402

log(f"cuda available {torch.cuda.is_available()}")
torch.zeros(1, device="cuda")
log("cuda context up")
from paper_2206_01784_b200 import KeyGenSpec, generate_keys, onesweep_sort  # noqa: E402

log("package imported")
n = 1 << 16
keys = generate_keys(KeyGenSpec(q=1, seed=0, n=n, key_bits=32), device="cuda:0")
torch.cuda.synchronize()
log("keygen done")
vals = torch.arange(n, dtype=torch.int32, device="cuda:0").view(torch.uint32)
sk, sv = onesweep_sort(keys, vals)
log("sort launched")
torch.cuda.synchronize()
log("sort done")
from oracle import oracle  # noqa: E402

want = oracle.sort(keys.cpu().numpy(), vals.cpu().numpy())
log("oracle done")
import numpy as np  # noqa: E402

assert np.array_equal(sk.cpu().numpy(), want[0]) and np.array_equal(sv.cpu().numpy(), want[1])
log("compare ok")
import __graft_entry__ as g  # noqa: E402

g.smoke()
log("smoke() ok")
