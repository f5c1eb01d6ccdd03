"""Small driver for ncu / timing runs of one config (not part of the product).

    python tools/prof_run.py c2 [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_17746_b200 as ws  # noqa: E402
from bench import splitmix_starts  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sv = ws.Sieve(device=0)
if cfg == "c2":
    out = torch.empty(ws.prime_count_bound(0, 10**10), dtype=torch.int64, device="cuda")
    f = lambda: sv.enumerate_range(0, 10**10, out=out)[2]
elif cfg == "c1":
    f = lambda: sv.count_range(0, 10**9 + 1)
elif cfg in ("p10", "p11", "p95", "p2e11", "p3e11", "p5e11"):  # count-only pi(N)
    hi_ = {"p10": 10**10, "p11": 10**11, "p95": 3 * 10**9, "p2e11": 2 * 10**11,
           "p3e11": 3 * 10**11, "p5e11": 5 * 10**11}[cfg]
    f = lambda: sv.count_range(0, hi_ + 1)
elif cfg == "c3":
    f = lambda: sv.count_range(0, 10**12 + 1)
elif cfg == "c3s":  # 1/8 share of c3 (one rank at 8 GPUs)
    lo, hi = ws.partition(0, 10**12 + 1, 7, 8)
    f = lambda: sv.count_range(lo, hi)
elif cfg == "c4":
    f = lambda: sv.count_range(10**15, 10**15 + 10**11, checks=True)
elif cfg == "c4s":  # 1/8 share of c4
    lo, hi = ws.partition(10**15, 10**15 + 10**11, 7, 8)
    f = lambda: sv.count_range(lo, hi, checks=True)
elif cfg == "c4e":
    out = torch.empty(ws.prime_count_bound(10**15, 10**15 + 10**11), dtype=torch.int64,
                      device="cuda")
    f = lambda: sv.enumerate_range(10**15, 10**15 + 10**11, out=out)[2]
elif cfg == "c5":
    Ls = splitmix_starts(42, 4096, 2**32, 2**44)
    f = lambda: sv.count_intervals(Ls, 2**24)
for i in range(reps):
    t0 = time.perf_counter()
    r = f()
    t = sv.timing()
    print(f"{cfg} rep {i}: wall {1e3*(time.perf_counter()-t0):.2f} ms sieve {t.sieve_ms:.3f} ms "
          f"base {t.base_ms:.3f} ms launches {t.launches} segments {t.segments} "
          f"base_primes {t.base_primes}", flush=True)
