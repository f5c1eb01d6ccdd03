"""Benchmark of the B200 segmented wheel sieve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Default workload: BASELINE config 3, pi(1e12) count-only -- the config the
baseline defines at 1/2/4/8 GPUs -- strong-scaled: the same [0, 1e12] at
every N.  Metric: integers sieved per second (whole job).

Multi-GPU goes through the library's own multi-device context: `--gpus N`
without torchrun opens one context over devices 0..N-1 of this process;
under torchrun (WORLD_SIZE set) every rank opens a context over its
LOCAL_RANK device with world = WORLD_SIZE (the NCCL id travels over gloo).
Either way the library splits the range into contiguous per-device
super-ranges (ws_partition) with no data-path exchange and combines the
32-byte per-shard records with ONE ncclAllGather.  n_gpus = shards that ran.

Other configs (--config): c1 pi(1e9) count (+ per-segment counts), c2
enumerate all primes < 1e10 (each device's shard stays in its HBM), c4
[1e15, 1e15+1e11) count + sum/xor, c4e its enumeration, c5 4096 intervals
[L, L+2^24) per-interval count + sum + xor (interval i -> device i mod N).

One JSON line on rank 0.  `value` is device-timed (CUDA events on every
device's launch stream, max over devices and ranks) with outputs left in
HBM; `e2e` goes through the same public API with host buffers, the
device->host copy of every step's result inside the timed call.
`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libwsref.so: the unmodified reference library, threaded) on the
host cores for the same config/metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEG = 1 << 18

CONFIGS = {
    "c1": dict(workload="c1: pi(N) count-only, N=1e9, per-segment uint32 counts", L=0,
               R=10**9 + 1, kind="count", metric="integers sieved/sec", unit="integers/s"),
    "c2": dict(workload="c2: enumerate all primes < 1e10 into a sorted uint64 array in HBM "
               "+ count, sum mod 2^64, xor", L=0, R=10**10, kind="enumerate",
               metric="primes enumerated/sec", unit="primes/s"),
    "c3": dict(workload="c3: pi(N) count-only, N=1e12, contiguous super-ranges per GPU", L=0,
               R=10**12 + 1, kind="count", metric="integers sieved/sec", unit="integers/s"),
    "c4": dict(workload="c4: count + sum/xor of primes in [1e15, 1e15+1e11)", L=10**15,
               R=10**15 + 10**11, kind="checks", metric="integers sieved/sec",
               unit="integers/s"),
    "c4e": dict(workload="c4e: enumerate the primes of [1e15, 1e15+1e11) into a sorted uint64 "
                "array in HBM (2.9e9 primes, 23.2 GB) + count, sum mod 2^64, xor", L=10**15,
                R=10**15 + 10**11, kind="enumerate", metric="primes enumerated/sec",
                unit="primes/s"),
    "c5": dict(workload="c5: 4096 intervals [L, L+2^24), L = 2^32 + splitmix64(42) mod "
               "(2^44-2^32); per-interval count + sum + xor", kind="intervals",
               metric="integers sieved/sec", unit="integers/s"),
}


L2_NOTE = {
    "enumerate": "output (3.64 GB per step at c2, 23.2 GB at c4e) far larger than the 126 MB "
                 "L2; no flush",
    "count": "inputs are two scalars; the work is on-chip (shared memory); per-segment "
             "counts written each step; no flush needed",
    "checks": "bucket lists (~1 GB per window) far larger than L2; no flush",
    "intervals": "bucket lists far larger than L2; no flush",
}


# ----------------------------------------------------------------------------
def splitmix_starts(seed: int, n: int, lo: int, hi: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    x = seed
    M = (1 << 64) - 1
    for i in range(n):
        x = (x + 0x9E3779B97F4A7C15) & M
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        out[i] = lo + z % (hi - lo)
    return out


def small_primes(n: int) -> np.ndarray:
    """Primes <= n (numpy sieve; used only for the roofline byte model)."""
    s = np.ones(n + 1, bool)
    s[:2] = False
    for i in range(2, int(n**0.5) + 1):
        if s[i]:
            s[i * i::i] = False
    return np.nonzero(s)[0].astype(np.int64)


def cop6(x):
    x = np.maximum(x, 0)
    return x - x // 2 - x // 3 + x // 6


def smem_bytes(L: int, R: int, S: int = SEG) -> float:
    """SURVEY §8(d) algorithmic shared-memory bytes of one pass over [L, R):
    4 B x [2W + sum_{17 <= p <= sqrt R} min(hits_p, W)], W = 32-bit words of
    both classes, hits_p = multiples of p in [max(L, p^2), R) coprime to 6."""
    lo0 = L // 6 * 6
    slots = (R - lo0 + 5) // 6
    W = 2 * ((slots + 31) // 32)
    P = small_primes(math.isqrt(R - 1))
    P = P[P >= 17]
    lo = np.maximum(np.int64(L), P * P)
    klo = -(-lo // P)
    khi = (R - 1) // P
    hits = np.where(khi >= klo, cop6(khi) - cop6(klo - 1), 0)
    return 4.0 * (2 * W + float(np.minimum(hits, W).sum()))


def bucket_hits(L: int, R: int, S: int = SEG) -> int:
    """Hits the library routes through HBM bucket lists for [L, R): every
    multiple coprime to 6 of a base prime p >= 2S, when the range buckets at
    all (largest base prime >= 8S -- the library's default policy).  Each is
    8 B of HBM traffic: a 4-byte entry written by the fill, read back by the
    window sieve ("bucket spill")."""
    B = math.isqrt(R - 1)
    if B < 8 * S:
        return 0
    P = small_primes(B)
    P = P[P >= 2 * S]
    lo = np.maximum(np.int64(L), P * P)
    klo = -(-lo // P)
    khi = (R - 1) // P
    return int(np.where(khi >= klo, cop6(khi) - cop6(klo - 1), 0).sum())


def smem_peak_gbs(sm_count: int, sm_mhz: float) -> float:
    return sm_count * 128 * sm_mhz * 1e6 / 1e9  # 32 banks x 4 B per clock per SM


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable"]}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # the host-side wire expanders of co-located ranks share the host's cores
    nloc = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    if nloc > 1 and "WHEELSIEVE_HOST_THREADS" not in os.environ:
        os.environ["WHEELSIEVE_HOST_THREADS"] = str(max(1, len(os.sched_getaffinity(0)) // nloc))
    return ws, rank, local


class Plumbing:
    """Host-side plumbing of a multi-process run (torchrun): gloo for the
    NCCL id broadcast, the barrier and the max-over-ranks of the timings.
    The data-path collective is the library's own NCCL all-gather."""

    def __init__(self, world: int, rank: int):
        self.world, self.rank = world, rank
        if world > 1:
            import torch.distributed as tdist
            tdist.init_process_group("gloo")
            self.d = tdist

    def barrier(self):
        if self.world > 1:
            self.d.barrier()

    def bcast(self, obj):
        if self.world == 1:
            return obj
        box = [obj]
        self.d.broadcast_object_list(box, src=0)
        return box[0]

    def reduce(self, v: float, op: str) -> float:
        if self.world == 1:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.d.all_reduce(t, op=self.d.ReduceOp.MAX if op == "max" else self.d.ReduceOp.SUM)
        return float(t.item())


def open_sieve(args, world, rank, local, pl):
    """The library context for this process: `--gpus N` devices of this
    process (single process), or this rank's device in a world of torchrun
    ranks.  Always an NCCL context, so every N takes the same code path."""
    import torch

    import paper_2310_17746_b200 as ws
    ndev = torch.cuda.device_count()
    if world > 1:
        dev = local % ndev
        torch.cuda.set_device(dev)
        nid = pl.bcast(ws.nccl_unique_id() if rank == 0 else None)
        return ws.Sieve(devices=[dev], world=world, rank=rank, nccl_id=nid), [dev]
    if args.gpus > ndev:
        raise SystemExit(f"--gpus {args.gpus}: only {ndev} CUDA devices visible")
    devs = list(range(args.gpus))
    torch.cuda.set_device(devs[0])
    return ws.Sieve(devices=devs), devs


def run_ours(args, cfg, world, rank, local):
    import torch

    import paper_2310_17746_b200 as ws

    pl = Plumbing(world, rank)
    sv, devs = open_sieve(args, world, rank, local, pl)
    nshards = sv.num_shards
    kind = cfg["kind"]
    streams = [torch.cuda.ExternalStream(st, device=torch.device("cuda", d))
               for st, d in zip(sv.streams, devs)]
    nccl = [dict(zip(("nranks", "rank"), sv.comm_info(i)), device=d) for i, d in enumerate(devs)]
    L, R = cfg.get("L"), cfg.get("R")
    shard0 = ws.partition(L, R, rank * len(devs), nshards, SEG) if L is not None else (None, None)

    # ---- per-config steps: the whole job through the library (it shards) ----
    if kind == "enumerate":  # strong: every device enumerates its shard into its own HBM
        outs = []
        for i, d in enumerate(devs):
            lo, hi = ws.partition(L, R, rank * len(devs) + i, nshards, SEG)
            outs.append(torch.empty(max(1, ws.prime_count_bound(lo, hi) + 2), dtype=torch.int64,
                                    device=f"cuda:{d}"))

        shard_counts = [0]

        def step():
            cnt, c = sv.enumerate_shards(L, R, outs, fresh_base=True)
            shard_counts[0] = cnt[0]
            return c
        units = None  # primes, known after the first step
    elif kind in ("count", "checks"):
        nseg = sv.num_segments(L, R)
        ps_dev = (torch.zeros(max(1, nseg), dtype=torch.int32, device=f"cuda:{devs[0]}")
                  if args.config == "c1" else None)

        def step():
            return sv.count_range(L, R, checks=(kind == "checks"), per_seg=ps_dev,
                                  fresh_base=True)
        units = R - L
    else:  # intervals: interval i -> shard i mod N inside the library
        Ls = splitmix_starts(42, 4096, 2**32, 2**44)
        width = 2**24

        def step():
            counts, sums, xors = sv.count_intervals(Ls, width, fresh_base=True)
            return ws.Checks(int(counts.astype(np.uint64).sum()),
                             int(sums.sum(dtype=np.uint64)),
                             int(np.bitwise_xor.reduce(xors)) if xors.size else 0, 0)
        units = int(Ls.size) * width

    for _ in range(args.warmup):
        c = step()
    if kind == "enumerate":
        units = c.count
    for d in devs:
        torch.cuda.synchronize(d)
    pl.barrier()
    for d in devs:
        torch.cuda.synchronize(d)
    sieve_ms, dev0_ms, launches = [], [], 0
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in devs]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in devs]
    with ClockSampler(devs[0]) as clk:
        for e, st in zip(ev0, streams):
            e.record(st)
        for _ in range(args.steps):
            c = step()
            t = sv.timing()
            sieve_ms.append(t.sieve_ms)
            dev0_ms.append(sv.device_timing(0).sieve_ms)
            launches += t.launches
        for e, st in zip(ev1, streams):
            e.record(st)
        for e in ev1:
            e.synchronize()
    for d in devs:
        torch.cuda.synchronize(d)
    local_ms = max(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    tot_ms = pl.reduce(local_ms, "max")
    launches = int(pl.reduce(launches, "sum"))
    checks = c  # the library already combined every shard
    ms_per_step = tot_ms / args.steps
    value = units / (ms_per_step / 1e3)

    # ---- e2e: same public API, host buffers, D2H inside the timed call ------
    k_e2e = max(2, min(args.steps, 10))
    e2e = {"unit": cfg["unit"], "steps": k_e2e, "timer": "host wall clock per call, max over ranks",
           "inputs": "two scalars (L, R) by value: no host->device input bytes"}
    if kind == "enumerate":
        cap = ws.prime_count_bound(L, R)
        if cap * 8 <= 8 << 30:
            host = torch.empty(cap, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        else:  # c4e: 23 GB; the wire path writes it with CPU stores, so pageable + pre-touched
            host = np.empty(units + 64, np.uint64)
            host.fill(0)
        sv.enumerate_range(L, R, out=host, fresh_base=True)
        pl.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            _, n, ce = sv.enumerate_range(L, R, out=host, fresh_base=True)
        e_ms = pl.reduce((time.perf_counter() - t0) * 1e3 / k_e2e, "max")
        assert ce.count == c.count and ce.sum == c.sum and ce.xor == c.xor
        tm = sv.timing()
        hv = host[:n]  # this process's part of the sorted enumeration, in host memory
        if world == 1:
            host_ok = (int(hv.sum(dtype=np.uint64)) == ce.sum and
                       int(np.bitwise_xor.reduce(hv)) == ce.xor and int(hv[-1]) == ce.largest)
            if not host_ok:
                raise SystemExit("e2e: host output disagrees with the device checksums")
        wire = os.environ.get("WHEELSIEVE_HOST_WIRE", "1") != "0" and tm.d2h_bytes < 4 * n
        e2e.update({"outputs": "the sorted uint64 primes in host memory (re-verified: sum, xor, "
                               "largest)",
                    "transfer": ("8-bit wire entries + per-block counts, widened on the host "
                                 "(ws_wire.cpp)") if wire else "uint64 values",
                    "host_expander_threads_per_rank": os.environ.get(
                        "WHEELSIEVE_HOST_THREADS",
                        f"{len(os.sched_getaffinity(0))} CPUs / {len(devs)} devices")})
    elif kind in ("count", "checks"):
        per = np.zeros(max(1, sv.num_segments(L, R)), np.uint32)
        pl.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            ce = sv.count_range(L, R, checks=(kind == "checks"), per_seg=per, fresh_base=True)
        e_ms = pl.reduce((time.perf_counter() - t0) * 1e3 / k_e2e, "max")
        assert ce.count == c.count
        tm = sv.timing()
        e2e["outputs"] = (f"count{' + sum/xor' if kind == 'checks' else ''} + largest, and the "
                          f"{per.size} per-segment uint32 counts in host memory")
    else:
        pl.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            step()
        e_ms = pl.reduce((time.perf_counter() - t0) * 1e3 / k_e2e, "max")
        tm = sv.timing()
        e2e["inputs"] = "4096 uint64 interval starts (host array, read on the host)"
        e2e["outputs"] = "per-interval uint32 counts + uint64 sums + uint64 xors in host memory"
    e2e.update({"value": units / (e_ms / 1e3), "ms_per_step": e_ms,
                "h2d_bytes_per_step": int(pl.reduce(tm.h2d_bytes, "sum")),
                "d2h_bytes_per_step": int(pl.reduce(tm.d2h_bytes, "sum"))})

    if rank != 0:
        sv.close()
        return None
    peaks, peak_src = load_peaks()
    props = torch.cuda.get_device_properties(devs[0])
    avg_sieve_ms = float(np.mean(dev0_ms))  # device 0's kernel time for shard 0
    clocks = clk.summary()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and nshards == 1:
        with open(tpath) as f:
            traffic = json.load(f).get(args.config, {}).get("traffic_bytes_per_launch")
    # algorithmic bytes of the dominant kernel over shard 0 (the whole job at N=1)
    lo0, hi0 = shard0
    if kind == "intervals":
        mine = Ls[0::nshards]
        hits = sum(bucket_hits(int(x), int(x) + 2**24) for x in mine[:64]) * (mine.size / 64)
        b_smem = sum(smem_bytes(int(x), int(x) + 2**24) for x in mine[:64]) * (mine.size / 64)
        primes0 = 0
    else:
        hits = bucket_hits(lo0, hi0)
        b_smem = smem_bytes(lo0, hi0)
        primes0 = shard_counts[0] if kind == "enumerate" else 0  # device 0's shard
    # count launches long enough take the wide kernel (3 segments per unit, one
    # 1024-thread CTA per SM); WHEELSIEVE_WIDE=0 keeps the per-segment kernel
    wide_on = os.environ.get("WHEELSIEVE_WIDE", "3") not in ("0", "1")
    count_kernel = ("sieve_wide_kernel" if wide_on and args.config in ("c3", "c4", "c5")
                    else "sieve_kernel")
    alg = 8.0 * primes0 + 8.0 * hits
    roof = None
    if alg > 0:
        achieved = alg / (avg_sieve_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "kernel": ("sieve_kernel<kEnumerate>" if kind == "enumerate" else count_kernel)
                          + (" + bucket_fill_kernel" if hits else ""),
                "algorithmic_bytes_per_launch": alg,
                "model": ("8 B x primes written" if kind == "enumerate" else "")
                         + (" + " if kind == "enumerate" and hits else "")
                         + (f"8 B x {hits:.4g} bucketed hits (p >= 2S)" if hits else ""),
                "avg_launch_ms": avg_sieve_ms,
                "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs (copy)"}
    smax = peaks.get("sm_max_mhz", 1965.0)
    speak = smem_peak_gbs(props.multi_processor_count, smax)
    sach = b_smem / (avg_sieve_ms / 1e3) / 1e9
    roof_smem = {"bound": "smem", "achieved": sach, "peak": speak, "unit": "GB/s",
                 "frac": sach / speak, "algorithmic_bytes_per_launch": b_smem,
                 "traffic": traffic if kind != "enumerate" else None,
                 "avg_launch_ms": avg_sieve_ms,
                 "kernel": "sieve_kernel<kEnumerate>" if kind == "enumerate" else count_kernel,
                 "model": "SURVEY 8d: 4 B x [2W + sum_{17<=p<=sqrt R} min(hits_p, W)]",
                 "peak_source": f"{props.multi_processor_count} SMs x 128 B/clk x {smax} MHz"}
    roof_hbm = roof
    if roof is None or (b_smem / speak > alg / peaks["hbm_gbs"]):
        roof = roof_smem
    if nshards > 1:
        for r_ in (roof, roof_smem, roof_hbm):
            if r_:
                r_["scope"] = f"device 0, shard 0 of {nshards}"
    line = {
        "metric": cfg["metric"], "value": value, "unit": cfg["unit"], "n_gpus": nshards,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (deterministic ranges; c5 seeded splitmix64)",
        "config": {"workload": cfg["workload"], "L": L, "R": R, "segment_slots": SEG,
                   "l2": L2_NOTE[kind], "parallelism": f"dp{nshards}",
                   "sharding": "ws_partition contiguous super-ranges per device"
                               if kind != "intervals" else "interval i -> device i mod N",
                   "launch": "torchrun, one process per GPU" if world > 1
                             else f"one process, {len(devs)} device(s)",
                   "base_primes": "re-sieved on device every step (WS_FRESH_BASE)"},
        "result": {"count": checks.count,
                   "sum": checks.sum if kind not in ("count",) else None,
                   "xor": checks.xor if kind not in ("count",) else None,
                   "largest": checks.largest if kind != "intervals" else None},
        "e2e": e2e, "roofline": roof, "roofline_smem": roof_smem, "roofline_hbm": roof_hbm,
        "gpu_launches": launches, "clocks": clocks,
        "nccl": {"collective": "one ncclAllGather of 32-byte shard records per call "
                               "(inside libwheelsieve_cuda.so)", "comms": nccl},
        "integers_per_s": ((R - L) if kind != "intervals" else units) / (ms_per_step / 1e3),
    }
    line["result_check"] = check_result(args.config, checks)
    if nshards == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    sv.close()
    return line


def check_result(config, c):
    """Compare the run's result with the reference goldens committed under
    tests/golden (produced by the reference library, oracle/gen_golden.py).
    Every config is strong-scaled, so the golden is the same at every N."""
    gdir = os.path.join(ROOT, "tests", "golden")
    try:
        if config == "c2":
            g = json.load(open(os.path.join(gdir, "reference_goldens.json")))
            r = [p for p in g["prefixes"] if p["limit"] == 10**10 - 1][0]
            ok = (c.count, c.sum, c.xor, c.largest) == (r["count"], r["sum"], r["xor"], r["largest"])
        elif config == "c1":
            r = json.load(open(os.path.join(gdir, "c1_per_segment.json")))
            ok = (c.count, c.largest) == (r["count"], r["largest"])
        elif config == "c3":
            r = json.load(open(os.path.join(gdir, "reference_big.json")))["pi_1000000000000"]
            ok = (c.count, c.largest) == (r["count"], r["largest"])
        elif config in ("c4", "c4e"):
            r = json.load(open(os.path.join(gdir, "reference_big.json")))["c4"]
            ok = (c.count, c.sum, c.xor, c.largest) == (r["count"], r["sum"], r["xor"], r["largest"])
        elif config == "c5":
            r = json.load(open(os.path.join(gdir, "c5_intervals.json")))
            ok = (c.count, c.sum, c.xor) == (r["total_count"], r["total_sum"], r["total_xor"])
        else:
            return "no golden for this configuration"
    except Exception as e:  # noqa: BLE001
        return f"golden unavailable: {e}"
    return "match reference golden" if ok else "MISMATCH vs reference golden"


def cpu_baseline(cfg):
    """The reference library (oracle/_ref) on a bounded sample, all host threads."""
    try:
        from oracle.oracle import Reference
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unavailable": str(e)}
    T = os.cpu_count() or 1
    kind = cfg["kind"]
    if kind == "enumerate" and cfg["L"] >= 10**15:  # c4e
        sample = ("reference composition (SURVEY 3.3) over [1e15, 1e15+1e9) visiting every "
                  "survivor (sum/xor), primes per second")
        r = ref.range(10**15, 10**15 + 10**9, T)
        val = r["count"] / (r["wall_ms"] / 1e3)
    elif kind == "enumerate":
        sample = "reference run() with a sum/xor PrimeSink over [0, 1e9] (prefix of c2), best of 3"
        best = min(ref.run_checks(10**9, T)["wall_ms"] for _ in range(3))
        val = 50_847_534 / (best / 1e3)
    elif kind == "count" and cfg["R"] <= 10**9 + 1:
        sample = "reference run() with a CountSink over [0, 1e9] (the full c1), best of 3"
        best = min(ref.pi(10**9, T)["wall_ms"] for _ in range(3))
        val = 1e9 / (best / 1e3)
    elif kind == "count":
        # BASELINE.json config 3: time the CPU at N = 1e11 and extrapolate per
        # integer.  This flatters the CPU: its integers/s falls with N (the
        # survey measured 3.62e9 at 1e11 vs 2.10e9 at the full 1e12)
        sample = ("reference run() with a CountSink over [0, 1e11], extrapolated per integer "
                  "to c3's 1e12 (flatters the CPU: per-integer cost grows with N)")
        r = ref.pi(10**11, T)
        if r["count"] != 4_118_054_813:
            return {"value": None, "unavailable": f"reference pi(1e11) = {r['count']}"}
        val = 1e11 / (r["wall_ms"] / 1e3)
    elif kind == "checks":
        sample = "reference composition (SURVEY 3.3) over [1e15, 1e15+1e9) with sum/xor"
        r = ref.range(10**15, 10**15 + 10**9, T)
        val = 1e9 / (r["wall_ms"] / 1e3)
    else:
        Ls = splitmix_starts(42, 4096, 2**32, 2**44)[:128]
        sample = "reference composition over the first 128 of the 4096 c5 intervals"
        _, _, _, ms = ref.intervals(Ls, 2**24, T)
        val = 128 * 2**24 / (ms / 1e3)
    return {"value": val, "unit": cfg["unit"], "cores": T, "kind": "reference",
            "sample": sample}


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU implementation, all host threads."""
    if rank != 0:
        return None
    from oracle.oracle import Reference
    try:
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        return {"impl": "reference", "unavailable": f"reference library not built: {e}"}
    T = os.cpu_count() or 1
    kind = cfg["kind"]
    if kind == "enumerate" and cfg["L"] >= 10**15:  # c4e
        sample = ("reference composition over [1e15, 1e15+1e9) visiting every survivor "
                  "(1% sample of c4e)")

        def step():
            r = ref.range(10**15, 10**15 + 10**9, T)
            return r["count"], r["wall_ms"]
    elif kind == "enumerate":
        sample = "reference run() with a sum/xor PrimeSink over [0, 1e10) (the full c2)"

        def step():
            r = ref.run_checks(10**10 - 1, T)
            return r["count"], r["wall_ms"]
    elif kind == "count" and cfg["R"] <= 10**9 + 1:
        sample = "reference run() with a CountSink over [0, 1e9] (the full c1)"

        def step():
            r = ref.pi(10**9, T)
            return 10**9, r["wall_ms"]
    elif kind == "count":
        # BASELINE.json config 3: the CPU is timed on N = 1e11, extrapolated per
        # integer.  The K timed steps cover [0, 1e11] together: step k counts
        # its 1/K slice with the reference's composition, so the
        # run stays within minutes for any K and the sum is exactly pi(1e11).
        edges = [10**11 * k // args.steps for k in range(args.steps + 1)]
        sample = (f"reference composition (threaded SegmentBitmap + sieve_segment) over [0, 1e11] "
                  f"in {args.steps} contiguous slices (one per step), extrapolated per integer to "
                  f"c3's 1e12 (flatters the CPU: per-integer cost grows with N); warm-up steps "
                  f"run() pi(1e9)")
        it = iter(range(args.steps))
        warm = [args.warmup]

        def step():
            if warm[0] > 0:
                warm[0] -= 1
                r = ref.pi(10**9, T)
                return 10**9, r["wall_ms"]
            k = next(it)
            r = ref.range(edges[k], edges[k + 1], T)
            step.count += r["count"]
            return edges[k + 1] - edges[k], r["wall_ms"]
        step.count = 0
    elif kind == "checks":
        sample = "reference composition over [1e15, 1e15+1e9) (1% sample of c4)"

        def step():
            r = ref.range(10**15, 10**15 + 10**9, T)
            return 10**9, r["wall_ms"]
    else:
        Ls = splitmix_starts(42, 4096, 2**32, 2**44)[:128]
        sample = "reference composition over the first 128 c5 intervals"

        def step():
            _, _, _, ms = ref.intervals(Ls, 2**24, T)
            return 128 * 2**24, ms
    for _ in range(args.warmup):
        step()
    units, ms = 0, 0.0
    for _ in range(args.steps):
        u, m = step()
        units += u
        ms += m
    value = units / (ms / 1e3)
    if kind == "count" and cfg["R"] > 10**9 + 1 and step.count != 4_118_054_813:
        return {"impl": "reference", "unavailable": f"reference slices sum to {step.count}"}
    return {"impl": "reference", "metric": cfg["metric"], "value": value, "unit": cfg["unit"],
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "none (CPU)",
            "note": "rank 0 alone runs the CPU reference; other ranks exit without work",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "sample": sample},
            "cpu_baseline": {"value": value, "unit": cfg["unit"], "cores": T,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": cfg["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    # NCCL's banner and init log go to stderr (stdout carries the one JSON
    # line); INFO makes every communicator's rank count visible there
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_env()
    cfg = CONFIGS[args.config]
    # stdout carries exactly one JSON line: while the run goes on, fd 1 (which
    # native code such as NCCL's version banner writes to) points at stderr
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        if args.impl == "reference":
            line = run_reference(args, cfg, world, rank)
        else:
            line = run_ours(args, cfg, world, rank, local)
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
