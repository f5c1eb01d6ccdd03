"""TEST INFRASTRUCTURE ONLY -- generates tests/golden/*.json by running the
UNMODIFIED reference library (oracle/_ref/libwsref.so, built from
/root/reference/proj/src by oracle/Makefile) through its own public API.

    python oracle/gen_golden.py            # quick goldens (~1-2 min on 8 cores)
    python oracle/gen_golden.py --big      # + pi(1e11), pi(1e12), full C4 window (~15 min)
    python oracle/gen_golden.py --scale    # only: c2 weak-scaling prefixes [0, N*1e10), N=2,4,8

Every record carries `source: "reference"` and the reference entry point used
(`run` = engine.cpp:344, `range` = the SURVEY §3.3 composition of
bootstrap/SegmentBitmap/sieve_segment/for_each_surviving).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Reference, Port, fnv1a64  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
SEG = 1 << 18

# Windows exercising the edges SURVEY §7 "Exactness at the edges" lists:
# unaligned L and R, value 1 in segment 0, 2/3 outside the wheel, p itself
# inside the range (p^2 activation), tiny/partial final segments, squares of
# base primes on segment borders, high offsets.
WINDOWS = [
    (0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (0, 6), (0, 7), (2, 3), (3, 4), (4, 5), (1, 30),
    (0, 100), (5, 6), (24, 26), (25, 26), (0, 1000), (1, 10_007), (997, 1009),
    (12_000, 18_000), (10_200, 10_206), (168, 174), (594_000, 600_000),
    (0, 1_000_001), (999_983, 1_000_003), (1_000_000, 2_000_000),
    (123_457, 9_876_543), (6 * SEG - 7, 6 * SEG + 11), (6 * SEG * 3 + 1, 6 * SEG * 5 - 1),
    (10**9 - 10**6, 10**9 + 1), (2**32 - 1000, 2**32 + 1000),
    (2**32, 2**32 + 2**24), (2**43, 2**43 + 2**24), (10**12, 10**12 + 10**7 + 3),
    (10**15, 10**15 + 10**6), (10**15 + 1, 10**15 + 10**6 + 5),
    (10**15, 10**15 + 10**8),
    (999_999_999_989 - 6, 999_999_999_989 + 7),
    (10**16 - 10**6 - 12, 10**16 - 12),  # naive_sieve cap (wheel.hpp:40) bounds R at 1e16
]

SEGMENTS = [(12_000, 1000), (0, 1000), (10_200, 1), (168, 1), (594_000, 1000), (6, 77),
            (0, 1 << 18), (6 * 10**14, 300_000), (6 * 123_456_789, (1 << 18) + 5),
            (10**16 - 6 * 4000 - 4, 4000)]

PREFIXES = [2, 3, 4, 5, 29, 30, 96, 100, 1000, 5999, 10_000, 99_991, 100_000, 123_456, 10**6,
            10**7, 10**8, 10**9]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--scale", action="store_true")
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    ref = Reference()
    T = a.threads or ref.hw_threads()
    os.makedirs(GOLDEN, exist_ok=True)
    t0 = time.time()
    if a.scale:  # bench.py --gpus N on c2 (weak): rank r enumerates [r*1e10, (r+1)*1e10)
        recs = []
        for n in (2, 4, 8):
            t = time.time()
            r = ref.run_checks(n * 10**10 - 1, T)
            recs.append(dict(gpus=n, limit=n * 10**10 - 1, count=r["count"], sum=r["sum"],
                             xor=r["xor"], largest=r["largest"], wall_s=time.time() - t))
            print("scale", n, time.time() - t, flush=True)
        meta = dict(source="reference", entry="run() with a sum/xor PrimeSink", threads=T,
                    generator="oracle/gen_golden.py --scale")
        with open(os.path.join(GOLDEN, "reference_scale.json"), "w") as f:
            json.dump(dict(meta=meta, c2_weak=recs), f, indent=1)
        return

    # 1. prefixes through run() (count + sum + xor + largest)
    prefixes = []
    for n in PREFIXES:
        r = ref.run_checks(n, T)
        prefixes.append(dict(limit=n, count=r["count"], sum=r["sum"], xor=r["xor"],
                             largest=r["largest"]))
    r = ref.run_checks(10**10 - 1, T)  # primes below 1e10 (config 2)
    prefixes.append(dict(limit=10**10 - 1, count=r["count"], sum=r["sum"], xor=r["xor"],
                         largest=r["largest"]))
    print("prefixes", time.time() - t0, flush=True)

    # 2. windows through the composition, with per-segment counts at two
    #    segment sizes (2^18 production and 2^12 to stress segment borders)
    windows = []
    for L, R in WINDOWS:
        rec = dict(L=L, R=R)
        for slots in (SEG, 1 << 12):
            if slots != SEG and (R - L) > 2 * 10**8:
                continue
            r = ref.range(L, R, T, slots, per_seg=True)
            key = "seg18" if slots == SEG else "seg12"
            rec.update(count=r["count"], sum=r["sum"], xor=r["xor"], largest=r["largest"])
            rec[key] = [int(x) for x in r["per_seg"]]
        windows.append(rec)
    print("windows", time.time() - t0, flush=True)

    # 3. config 1 per-segment counts: [0, 1e9], 2^18-slot segments
    c1 = ref.range(0, 10**9 + 1, T, SEG, per_seg=True)
    c1rec = dict(L=0, R=10**9 + 1, count=c1["count"], sum=c1["sum"], xor=c1["xor"],
                 largest=c1["largest"], seg18=[int(x) for x in c1["per_seg"]])

    # 4. config 5 batch: 4096 x [L, L + 2^24), L = 2^32 + splitmix64(42) mod (2^44 - 2^32)
    port = Port()
    Ls = port.splitmix_starts(42, 4096, 2**32, 2**44)
    counts, sums, xors, ms = ref.intervals(Ls, 2**24, T)
    c5 = dict(seed=42, n=4096, width=2**24, lo=2**32, hi=2**44,
              L=[int(x) for x in Ls], counts=[int(x) for x in counts],
              sums=[int(x) for x in sums], xors=[int(x) for x in xors],
              total_count=int(counts.astype(np.uint64).sum()),
              total_sum=int(sums.sum(dtype=np.uint64)),
              total_xor=int(np.bitwise_xor.reduce(xors)))
    print("c5", time.time() - t0, flush=True)

    # 5. Table 1 probes (wheel.cpp:96-106) for a spread of primes and starts
    rng = np.random.default_rng(20260816)
    offs = []
    for p in [5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 101, 997, 1009, 10007]:
        for _ in range(8):
            start = 6 * int(rng.integers(p // 6 + 1, 166_666))
            i1, i5 = ref.start_offsets(p, start)
            offs.append(dict(p=p, start=start, id1=i1, id5=i5))

    # SegmentBitmap + sieve_segment (segment.cpp:93-188): raw flag words
    segs = []
    for start, length in SEGMENTS:
        w1, w5 = ref.sieve_segment(start, length)
        segs.append(dict(start=start, len=length, r1=[int(x) for x in w1] if length <= 4096 else None,
                         r5=[int(x) for x in w5] if length <= 4096 else None,
                         fnv_r1=fnv1a64(w1.astype("<u8").tobytes()),
                         fnv_r5=fnv1a64(w5.astype("<u8").tobytes()),
                         pop_r1=int(sum(bin(int(x)).count("1") for x in w1)),
                         pop_r5=int(sum(bin(int(x)).count("1") for x in w5))))
    boots = []
    for hint in (25, 1000, 18000, 10**6, 10**10, 10**12 + 7):
        e, f = ref.bootstrap(hint)
        boots.append(dict(hint=hint, frontier=f, n=int(e.size), first=[int(x) for x in e[:5]],
                          last=int(e[-1]), fnv=fnv1a64(e.astype("<u8").tobytes())))
    with open(os.path.join(GOLDEN, "reference_segments.json"), "w") as f:
        json.dump(dict(meta=dict(source="reference", entry="SegmentBitmap + sieve_segment, "
                                 "BasePrimeStore::bootstrap", generator="oracle/gen_golden.py"),
                       segments=segs, bootstrap=boots), f)

    big = {}
    if a.big:
        for n in (10**11, 10**12):
            t = time.time()
            r = ref.pi(n, T)
            big[f"pi_{n}"] = dict(limit=n, count=r["count"], largest=r["largest"],
                                  wall_s=time.time() - t, threads=T)
            print("big", n, time.time() - t, flush=True)
        t = time.time()
        r = ref.range(10**15, 10**15 + 10**11, T, SEG)
        big["c4"] = dict(L=10**15, R=10**15 + 10**11, count=r["count"], sum=r["sum"],
                         xor=r["xor"], largest=r["largest"], wall_s=time.time() - t, threads=T)
        print("big c4", time.time() - t, flush=True)

    meta = dict(source="reference", library="oracle/_ref/libwsref.so (built from "
                "/root/reference/proj/src by oracle/Makefile)", threads=T,
                generator="oracle/gen_golden.py")
    with open(os.path.join(GOLDEN, "reference_goldens.json"), "w") as f:
        json.dump(dict(meta=meta, prefixes=prefixes, windows=windows, start_offsets=offs), f,
                  indent=1)
    with open(os.path.join(GOLDEN, "c1_per_segment.json"), "w") as f:
        json.dump(dict(meta=meta, **c1rec), f)
    with open(os.path.join(GOLDEN, "c5_intervals.json"), "w") as f:
        json.dump(dict(meta=meta, **c5), f)
    if big:
        with open(os.path.join(GOLDEN, "reference_big.json"), "w") as f:
            json.dump(dict(meta=meta, **big), f, indent=1)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()
