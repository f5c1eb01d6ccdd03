"""Where a small call's time goes: device kernel time vs whole call, for the
single-device and the NCCL (multi-device) context, fresh base or cached."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_17746_b200 as ws  # noqa: E402

for name, sv in (("single", ws.Sieve(device=0)), ("nccl", ws.Sieve(devices=[0]))):
    ps = torch.zeros(636, dtype=torch.int32, device="cuda")
    for fresh in (True, False):
        for _ in range(5):
            sv.count_range(0, 10**9 + 1, per_seg=ps, fresh_base=fresh)
        st = torch.cuda.ExternalStream(sv.streams[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 50
        sm, tm = [], []
        torch.cuda.synchronize()
        e0.record(st)
        t0 = time.perf_counter()
        for _ in range(k):
            sv.count_range(0, 10**9 + 1, per_seg=ps, fresh_base=fresh)
            t = sv.timing()
            sm.append(t.sieve_ms)
            tm.append(t.total_ms)
        e1.record(st)
        e1.synchronize()
        wall = (time.perf_counter() - t0) * 1e3 / k
        print(f"{name:6s} fresh={fresh!s:5s} step(events) {e0.elapsed_time(e1)/k:.4f} ms  wall {wall:.4f}"
              f"  sieve_ms {np.mean(sm):.4f}  total_ms {np.mean(tm):.4f}  launches {t.launches}")
