#!/usr/bin/env python3
"""wheelsieve-gpu: the reference CLI's subcommands (tools/wheelsieve.cpp) on the B200 library.

    wheelsieve_gpu.py sieve  --limit N [--count-only] [--out DIR --format text|binary
                             --primes-per-file K] [--segment-slots S]
    wheelsieve_gpu.py verify --limit N [--poison]
    wheelsieve_gpu.py bench  --limits N [N ...] [--segment-slots S [S ...]] [--repeats R]
                             [--csv PATH]

Output formats follow the reference: `count=... largest=... ms=...`
(print_summary, wheelsieve.cpp:106-110); verify prints PASS or
"FAIL first divergence at index i: expected X, got Y" (:183-228) with exit codes
0/1/2 (:352-380); bench writes the same CSV header (:244) with one row per
(limit, segment size), `threads` = GPUs used, `segment_span` = 6 * slots.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2310_17746_b200 as ws  # noqa: E402


def print_summary(count: int, largest: int, ms: float) -> None:
    print(f"count={count} largest={largest} ms={ms:.3f}")


def cmd_sieve(a) -> int:
    sv = ws.Sieve(segment_slots=a.segment_slots)
    t0 = time.perf_counter()
    if a.count_only:
        c = sv.count_range(0, a.limit + 1)
        count, largest = c.count, c.largest
    elif a.out:
        count = sv.store_range(0, a.limit + 1, a.out, binary=(a.format == "binary"),
                               primes_per_file=a.primes_per_file)
        largest = int(ws.read_back(a.out, max(0, a.limit - 2000), a.limit + 1)[-1]) if count else 0
    else:
        vals, count, c = sv.enumerate_range(0, a.limit + 1)
        largest = c.largest
        out = sys.stdout
        for i in range(0, vals.size, 1 << 20):
            out.write("\n".join(map(str, vals[i:i + (1 << 20)].tolist())))
            out.write("\n")
    print_summary(count, largest, (time.perf_counter() - t0) * 1e3)
    return 0


def _textbook(n: int) -> np.ndarray:
    """Independent checker for `verify` (the reference uses naive_sieve)."""
    s = np.ones(n + 1, bool)
    s[:2] = False
    for i in range(2, int(n ** 0.5) + 1):
        if s[i]:
            s[i * i::i] = False
    return np.nonzero(s)[0].astype(np.uint64)


def cmd_verify(a) -> int:
    expected = _textbook(a.limit)
    got, n, _ = ws.Sieve().enumerate_range(0, a.limit + 1)
    if a.poison and got.size > 24:  # drop one prime (wheelsieve.cpp:196-201)
        got = np.delete(got, 24)
    m = min(expected.size, got.size)
    diff = np.nonzero(expected[:m] != got[:m])[0]
    if diff.size == 0 and expected.size == got.size:
        print(f"PASS: {expected.size} primes up to {a.limit} match the reference sieve")
        return 0
    i = int(diff[0]) if diff.size else m
    exp = int(expected[i]) if i < expected.size else "(end)"
    gv = int(got[i]) if i < got.size else "(end)"
    print(f"FAIL first divergence at index {i}: expected {exp}, got {gv}")
    return 1


def cmd_bench(a) -> int:
    if a.repeats <= 0:
        print("error: --repeats must be positive", file=sys.stderr)
        return 2
    rows = ["threads,limit,segment_span,flag_width,wall_ms,iterations,peak_flag_bytes,prime_count"]
    counts = {}
    for limit in a.limits:
        for slots in a.segment_slots:
            sv = ws.Sieve(segment_slots=slots)
            best = None
            for _ in range(a.repeats):
                t0 = time.perf_counter()
                c = sv.count_range(0, limit + 1)
                ms = (time.perf_counter() - t0) * 1e3
                best = ms if best is None else min(best, ms)
            if counts.setdefault(limit, c.count) != c.count:
                print(f"error: prime count {c.count} for limit {limit} disagrees", file=sys.stderr)
                return 1
            nseg = sv.num_segments(0, limit + 1)
            # flag bytes resident at once: two classes x slots/8 per CTA x CTAs
            import torch
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            peak = 2 * (slots // 8) * min(nseg, 3 * sms)
            rows.append(f"1,{limit},{6 * slots},bit,{best:.3f},{nseg},{peak},{c.count}")
            sv.close()
    text = "\n".join(rows) + "\n"
    if not a.csv or a.csv == "-":
        sys.stdout.write(text)
    else:
        with open(a.csv, "w") as f:
            f.write(text)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="wheelsieve_gpu")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("sieve")
    s.add_argument("--limit", type=int, required=True)
    s.add_argument("--count-only", action="store_true")
    s.add_argument("--out", default="")
    s.add_argument("--format", choices=["text", "binary"], default="text")
    s.add_argument("--primes-per-file", type=int, default=125_000_000)
    s.add_argument("--segment-slots", type=int, default=1 << 18)
    v = sub.add_parser("verify")
    v.add_argument("--limit", type=int, required=True)
    v.add_argument("--poison", action="store_true")
    b = sub.add_parser("bench")
    b.add_argument("--limits", type=int, nargs="+", required=True)
    b.add_argument("--segment-slots", type=int, nargs="+", default=[1 << 18])
    b.add_argument("--repeats", type=int, default=1)
    b.add_argument("--csv", default="")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        return {"sieve": cmd_sieve, "verify": cmd_verify, "bench": cmd_bench}[a.cmd](a)
    except ws.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
