"""Timed randomized sweep (GPU, not part of the test suite): random [L, L+W)
with L log-uniform up to 2^63 and W up to 3e8, at S = 2^18 and 2^14.  Each
window must agree between count_range (checks), host-wire enumeration and
device enumeration (count, sum, xor, largest, ascending values), with the
oracle port when W <= 3e6 and L < 1e16, and otherwise on Miller-Rabin
samples of the enumerated values.

    python tools/fuzz_sweep.py        # ~10 minutes on one B200 (FUZZ_SECONDS)

Every window is also counted and enumerated by a 4-shard multi-device
context run as virtual devices on the same GPU (WHEELSIEVE_VIRTUAL_SHARDS)
and must agree with the single-device results.
"""
import os, sys, random, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_17746_b200 as ws
from oracle.oracle import Port

def is_prime(n):
    if n < 2: return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0: return n == p
    d, s = n - 1, 0
    while d % 2 == 0: d //= 2; s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1): continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1: break
        else: return False
    return True

rng = random.Random(20261020)
port = Port()
sv = {S: ws.Sieve(segment_slots=S) for S in (1 << 18, 1 << 14)}
os.environ["WHEELSIEVE_VIRTUAL_SHARDS"] = "1"
os.environ["WHEELSIEVE_BUCKET_BUDGET"] = str(1 << 30)
virt = ws.Sieve(devices=[0] * 4)
seconds = float(os.environ.get("FUZZ_SECONDS", "600"))
dev = torch.empty(40_000_000, dtype=torch.int64, device="cuda")
t0 = time.time(); bad = 0; n = 0
while time.time() - t0 < seconds:
    L = int(2 ** rng.uniform(0, 63)); W = int(2 ** rng.uniform(0, 28.2))
    if L + W >= 18446744073709551612: continue
    S = rng.choice(list(sv)); s = sv[S]
    c = s.count_range(L, L + W, checks=True)
    v, k, ce = s.enumerate_range(L, L + W)
    hv = np.asarray(v, dtype=np.uint64)
    ok = (k == c.count and ce.sum == c.sum and ce.xor == c.xor and ce.largest == c.largest
          and int(hv.sum(dtype=np.uint64)) == c.sum and (k == 0 or int(hv[-1]) == c.largest)
          and bool(np.all(hv[1:] > hv[:-1])))
    cv = virt.count_range(L, L + W, checks=True)
    ok = ok and (cv.count, cv.sum, cv.xor, cv.largest) == (c.count, c.sum, c.xor, c.largest)
    if k <= 5_000_000:
        vv, kv, _ = virt.enumerate_range(L, L + W)
        ok = ok and kv == k and np.array_equal(np.asarray(vv, dtype=np.uint64), hv)
    if k <= dev.numel():
        _, kd, cd = s.enumerate_range(L, L + W, out=dev)
        ok = ok and kd == k and cd.sum == c.sum and cd.xor == c.xor
    if W <= 3_000_000 and L + W < 10**16:
        r = port.range(L, L + W)
        ok = ok and (r["count"], r["sum"], r["xor"], r["largest"]) == (c.count, c.sum, c.xor, c.largest)
    elif k:
        for x in rng.sample(list(hv[: min(k, 2000)]), min(k, 20)):
            ok = ok and is_prime(int(x))
    n += 1
    if not ok:
        bad += 1; print("MISMATCH", L, W, S, flush=True)
print(f"{n} windows, {bad} mismatches", flush=True)
