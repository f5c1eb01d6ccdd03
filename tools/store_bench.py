#!/usr/bin/env python3
"""Throughput of the streaming chunked store (ws_store_range): enumerate
[L, R) on the device in bounded windows and write the reference's chunk
files + manifest.  Prints one JSON line (GB/s of file bytes written).

    python tools/store_bench.py [--L 0] [--R 1e10] [--dir /tmp/ws_store] [--text]
"""
import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_17746_b200 as ws  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=float, default=0)
    ap.add_argument("--R", type=float, default=1e10)
    ap.add_argument("--dir", default="/tmp/ws_store_bench")
    ap.add_argument("--text", action="store_true")
    ap.add_argument("--per-file", type=int, default=125_000_000)
    ap.add_argument("--verify", action="store_true")
    a = ap.parse_args()
    L, R = int(a.L), int(a.R)
    shutil.rmtree(a.dir, ignore_errors=True)
    sv = ws.Sieve()
    sv.count_range(L, R)  # warm: context, base primes
    t0 = time.perf_counter()
    n = sv.store_range(L, R, a.dir, binary=not a.text, primes_per_file=a.per_file)
    dt = time.perf_counter() - t0
    nbytes = sum(os.path.getsize(os.path.join(a.dir, f)) for f in os.listdir(a.dir))
    out = {"L": L, "R": R, "format": "text" if a.text else "binary", "primes": n,
           "files": len(os.listdir(a.dir)) - 1, "bytes": nbytes, "seconds": dt,
           "GB_per_s": nbytes / dt / 1e9, "primes_per_s": n / dt}
    if a.verify:
        t1 = time.perf_counter()
        ws.verify_store(a.dir)
        out["verify_seconds"] = time.perf_counter() - t1
    print(json.dumps(out))
    shutil.rmtree(a.dir, ignore_errors=True)


if __name__ == "__main__":
    main()
