"""TEST INFRASTRUCTURE ONLY -- ctypes front for the two CPU checkers.

* ``Port``      : oracle/_build/libwsoracle.so, the plain-C restatement
                  (oracle/ws_oracle.c) of the reference algorithm.
* ``Reference`` : oracle/_ref/libwsref.so, the UNMODIFIED reference library
                  compiled from /root/reference/proj/src by oracle/Makefile,
                  driven through its own public API by oracle/ref_driver.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libwsoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwsref.so")
REF_SRC = "/root/reference/proj"

u64 = C.c_uint64
u32 = C.c_uint32
P64 = C.POINTER(C.c_uint64)
P32 = C.POINTER(C.c_uint32)
PD = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    """Compile the checkers (oracle/Makefile).  The reference library is only
    (re)built where /root/reference exists (this container); the GPU box uses
    the prebuilt oracle/_ref/libwsref.so shipped with the snapshot."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(P64)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(P32)


class _Acc(C.Structure):
    _fields_ = [("count", u64), ("sum", u64), ("xr", u64), ("largest", u64)]


class Port:
    """The plain-C restatement (single-threaded)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = L = C.CDLL(path)
        L.wso_isqrt.restype = u64
        L.wso_isqrt.argtypes = [u64]
        L.wso_ceil_sqrt.restype = u64
        L.wso_ceil_sqrt.argtypes = [u64]
        L.wso_naive_sieve.restype = C.c_int64
        L.wso_naive_sieve.argtypes = [u64, P64, u64]
        L.wso_start_offsets.restype = C.c_int
        L.wso_start_offsets.argtypes = [u64, u64, P64, P64]
        L.wso_range.restype = C.c_int
        L.wso_range.argtypes = [u64, u64, u64, C.POINTER(_Acc), P32, u64, P64, P64, u64, P64]
        L.wso_intervals.restype = C.c_int
        L.wso_intervals.argtypes = [P64, u64, u64, u64, P32, P64, P64]
        L.wso_splitmix_starts.restype = None
        L.wso_splitmix_starts.argtypes = [u64, u64, u64, u64, P64]

    def isqrt(self, n: int) -> int:
        return self.lib.wso_isqrt(n)

    def naive_sieve(self, n: int) -> np.ndarray:
        c = self.lib.wso_naive_sieve(n, None, 0)
        if c < 0:
            raise ValueError("naive_sieve: empty range")
        out = np.empty(c, dtype=np.uint64)
        self.lib.wso_naive_sieve(n, _p64(out), c)
        return out

    def start_offsets(self, p: int, start: int):
        a, b = u64(), u64()
        rc = self.lib.wso_start_offsets(p, start, C.byref(a), C.byref(b))
        if rc:
            raise ValueError(f"start_offsets rc={rc}")
        return a.value, b.value

    def range(self, L: int, R: int, seg_slots: int = 1 << 18, per_seg: bool = False,
              values: bool = False):
        """Returns dict(count, sum, xor, largest[, per_seg][, values])."""
        acc = _Acc()
        nseg_cap = max(1, ((R - L // 6 * 6 + 5) // 6 + seg_slots - 1) // seg_slots) if R > L else 1
        ps = np.zeros(nseg_cap, dtype=np.uint32) if per_seg else None
        nseg = u64()
        out = None
        nout = u64()
        if values:
            acc0 = _Acc()
            rc = self.lib.wso_range(L, R, seg_slots, C.byref(acc0), None, 0, None, None, 0, None)
            if rc:
                raise RuntimeError("oracle range failed")
            out = np.empty(max(1, acc0.count), dtype=np.uint64)
        rc = self.lib.wso_range(L, R, seg_slots, C.byref(acc), _p32(ps) if per_seg else None,
                                nseg_cap if per_seg else 0, C.byref(nseg),
                                _p64(out) if values else None, out.size if values else 0,
                                C.byref(nout))
        if rc:
            raise RuntimeError("oracle range failed")
        r = dict(count=acc.count, sum=acc.sum, xor=acc.xr, largest=acc.largest)
        if per_seg:
            r["per_seg"] = ps[: nseg.value].copy()
        if values:
            r["values"] = out[: nout.value].copy()
        return r

    def intervals(self, Ls: np.ndarray, width: int, seg_slots: int = 1 << 18):
        Ls = np.ascontiguousarray(Ls, dtype=np.uint64)
        n = Ls.size
        counts = np.zeros(n, np.uint32)
        sums = np.zeros(n, np.uint64)
        xors = np.zeros(n, np.uint64)
        rc = self.lib.wso_intervals(_p64(Ls), n, width, seg_slots, _p32(counts), _p64(sums),
                                    _p64(xors))
        if rc:
            raise RuntimeError("oracle intervals failed")
        return counts, sums, xors

    def splitmix_starts(self, seed: int, n: int, lo: int, hi: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.wso_splitmix_starts(seed, n, lo, hi, _p64(out))
        return out


class Reference:
    """The reference library itself (threaded where the reference is)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_SRC):
                build(ref=True)
            else:
                raise FileNotFoundError(f"{path} not built and {REF_SRC} absent")
        self.lib = L = C.CDLL(path)
        L.wsref_run_count.argtypes = [u64, C.c_uint, u64, P64, P64, PD]
        L.wsref_run_checks.argtypes = [u64, C.c_uint, u64, P64, P64, P64, P64, PD]
        L.wsref_run_values.argtypes = [u64, C.c_uint, u64, P64, u64, P64]
        L.wsref_range.argtypes = [u64, u64, C.c_uint, u64, P64, P64, P64, P64, P32, u64, P64, PD]
        L.wsref_range_values.argtypes = [u64, u64, u64, P64, u64, P64]
        L.wsref_intervals.argtypes = [P64, u64, u64, C.c_uint, u64, P32, P64, P64, PD]
        L.wsref_start_offsets.argtypes = [u64, u64, P64, P64]
        L.wsref_naive_sieve.argtypes = [u64, P64, u64, P64]
        L.wsref_bootstrap.argtypes = [u64, P64, u64, P64, P64]
        L.wsref_hw_threads.restype = C.c_uint
        L.wsref_sieve_segment.argtypes = [u64, u64, P64, P64]
        L.wsref_store_run.argtypes = [u64, C.c_uint, C.c_char_p, C.c_int, u64]
        L.wsref_read_back.argtypes = [C.c_char_p, u64, u64, P64, u64, P64]
        L.wsref_verify_store.argtypes = [C.c_char_p]
        for f in ("wsref_run_count", "wsref_run_checks", "wsref_run_values", "wsref_range",
                  "wsref_range_values", "wsref_intervals", "wsref_start_offsets",
                  "wsref_naive_sieve", "wsref_bootstrap", "wsref_sieve_segment",
                  "wsref_store_run", "wsref_read_back", "wsref_verify_store"):
            getattr(L, f).restype = C.c_int

    @staticmethod
    def _ok(rc: int, what: str):
        if rc:
            raise RuntimeError(f"reference {what} failed: status {rc}")

    def hw_threads(self) -> int:
        return self.lib.wsref_hw_threads()

    def pi(self, limit: int, threads: int = 0, seg_slots: int = 1 << 18):
        c, lg, ms = u64(), u64(), C.c_double()
        self._ok(self.lib.wsref_run_count(limit, threads, seg_slots, C.byref(c), C.byref(lg),
                                          C.byref(ms)), "run(count)")
        return dict(count=c.value, largest=lg.value, wall_ms=ms.value)

    def run_checks(self, limit: int, threads: int = 0, seg_slots: int = 1 << 18):
        c, s, x, lg, ms = u64(), u64(), u64(), u64(), C.c_double()
        self._ok(self.lib.wsref_run_checks(limit, threads, seg_slots, C.byref(c), C.byref(s),
                                           C.byref(x), C.byref(lg), C.byref(ms)), "run(checks)")
        return dict(count=c.value, sum=s.value, xor=x.value, largest=lg.value,
                    wall_ms=ms.value)

    def run_values(self, limit: int, threads: int = 1, seg_slots: int = 1 << 18):
        cap = int(1.3 * limit / max(1.0, np.log(max(limit, 3)))) + 16
        out = np.empty(cap, np.uint64)
        n = u64()
        self._ok(self.lib.wsref_run_values(limit, threads, seg_slots, _p64(out), cap,
                                           C.byref(n)), "run(values)")
        return out[: n.value].copy()

    def range(self, L: int, R: int, threads: int = 0, seg_slots: int = 1 << 18,
              per_seg: bool = False):
        nseg_cap = max(1, ((R - L // 6 * 6 + 5) // 6 + seg_slots - 1) // seg_slots) if R > L else 1
        ps = np.zeros(nseg_cap, np.uint32) if per_seg else None
        c, s, x, lg, ns, ms = u64(), u64(), u64(), u64(), u64(), C.c_double()
        self._ok(self.lib.wsref_range(L, R, threads, seg_slots, C.byref(c), C.byref(s),
                                      C.byref(x), C.byref(lg), _p32(ps) if per_seg else None,
                                      nseg_cap if per_seg else 0, C.byref(ns), C.byref(ms)),
                 "range")
        r = dict(count=c.value, sum=s.value, xor=x.value, largest=lg.value, wall_ms=ms.value)
        if per_seg:
            r["per_seg"] = ps[: ns.value].copy()
        return r

    def range_values(self, L: int, R: int, seg_slots: int = 1 << 18):
        cap = int(1.3 * (R - L) / max(1.0, np.log(max(L, 3)))) + 64
        out = np.empty(cap, np.uint64)
        n = u64()
        self._ok(self.lib.wsref_range_values(L, R, seg_slots, _p64(out), cap, C.byref(n)),
                 "range_values")
        return out[: n.value].copy()

    def intervals(self, Ls: np.ndarray, width: int, threads: int = 0,
                  seg_slots: int = 1 << 18):
        Ls = np.ascontiguousarray(Ls, dtype=np.uint64)
        n = Ls.size
        counts = np.zeros(n, np.uint32)
        sums = np.zeros(n, np.uint64)
        xors = np.zeros(n, np.uint64)
        ms = C.c_double()
        self._ok(self.lib.wsref_intervals(_p64(Ls), n, width, threads, seg_slots, _p32(counts),
                                          _p64(sums), _p64(xors), C.byref(ms)), "intervals")
        return counts, sums, xors, ms.value

    def sieve_segment(self, start: int, length: int):
        nw = (length + 63) // 64
        r1 = np.zeros(nw, np.uint64)
        r5 = np.zeros(nw, np.uint64)
        self._ok(self.lib.wsref_sieve_segment(start, length, _p64(r1), _p64(r5)), "sieve_segment")
        return r1, r5

    def store_run(self, limit: int, dir: str, binary: bool, primes_per_file: int,
                  threads: int = 0):
        self._ok(self.lib.wsref_store_run(limit, threads, dir.encode(), int(binary),
                                          primes_per_file), "store_run")

    def read_back(self, dir: str, lo: int, hi: int):
        """Returns (status, values): status 0 ok, else 1 + Errc."""
        cap = max(16, hi - lo)
        cap = min(cap, 1 << 26)
        out = np.empty(cap, np.uint64)
        n = u64()
        rc = self.lib.wsref_read_back(dir.encode(), lo, hi, _p64(out), cap, C.byref(n))
        return rc, out[: min(cap, n.value)].copy()

    def verify_store(self, dir: str) -> int:
        return self.lib.wsref_verify_store(dir.encode())

    def start_offsets(self, p: int, start: int):
        a, b = u64(), u64()
        self._ok(self.lib.wsref_start_offsets(p, start, C.byref(a), C.byref(b)),
                 "start_offsets")
        return a.value, b.value

    def naive_sieve(self, n: int) -> np.ndarray:
        cap = int(1.3 * n / max(1.0, np.log(max(n, 3)))) + 16
        out = np.empty(cap, np.uint64)
        c = u64()
        self._ok(self.lib.wsref_naive_sieve(n, _p64(out), cap, C.byref(c)), "naive_sieve")
        return out[: c.value].copy()

    def bootstrap(self, hint: int):
        cap = 1 << 22
        out = np.empty(cap, np.uint64)
        n, f = u64(), u64()
        self._ok(self.lib.wsref_bootstrap(hint, _p64(out), cap, C.byref(n), C.byref(f)),
                 "bootstrap")
        return out[: min(cap, n.value)].copy(), f.value


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h
