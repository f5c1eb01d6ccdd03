"""A/B of the wide count kernel on launches of several jobs without buckets
(ws_count_ranges): python tools/multi_ab.py (one B200)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2310_17746_b200 as ws
S6 = 6 * (1 << 18)
rng = np.random.default_rng(3)
for segs in (6, 8, 12, 24):
    n = 4096 if segs <= 12 else 1024
    lo = (rng.integers(10**9, 10**11, size=n) // 6 * 6).astype(np.uint64)
    hi = lo + np.uint64(segs * S6 - 5)
    res = {}
    for w in ("0", "3"):
        os.environ["WHEELSIEVE_WIDE_MULTI"] = w
        with ws.Sieve(device=0) as sv:
            sv.count_ranges(lo, hi, checks=True)
            ts = []
            for _ in range(4):
                r = sv.count_ranges(lo, hi, checks=True)
                ts.append(sv.timing().sieve_ms)
            res[w] = (min(ts), sum(c.count for c in r))
    assert res["0"][1] == res["3"][1]
    print(f"{n} ranges x {segs} segments: per-segment {res['0'][0]:.3f} ms, wide {res['3'][0]:.3f} ms")
