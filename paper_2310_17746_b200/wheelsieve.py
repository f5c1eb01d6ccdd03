"""Python mirror of the reference's sieve entry points over the GPU C ABI.

Names and semantics follow /root/reference/proj/include/wheelsieve:

* ``Errc`` / ``Error``            -- errors.hpp:9-32 (status = 1 + Errc)
* ``isqrt``, ``start_offsets``     -- wheel.hpp:50-81 (wheel.cpp:25-33, 96-106)
* ``round_segment_span``, ``plan_iteration`` -- engine.hpp:69-76 (engine.cpp:311-342)
* ``run(SieveConfig)``             -- engine.hpp:83: pi / enumeration of [0, limit]
  into a ``PrimeSink`` (sink.hpp:18-66: ``CountSink``, ``MemorySink``), with the
  ascending-emission contract enforced by ``PrimeSink.emit`` (sink.cpp:14-37)
* ``Sieve.count_range / enumerate_range / count_intervals`` -- the [L, R)
  entry points the reference composes from bootstrap + SegmentBitmap +
  sieve_segment, as single device calls
* ``partition``                    -- contiguous per-GPU super-ranges (§8e)

All compute goes through libwheelsieve_cuda.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (WS_FRESH_BASE, WS_MAX_DEVICES, WS_NCCL_ID_BYTES, WS_OUT_DEVICE, WS_WANT_CHECKS,
                   WsChecks, WsOpts, WsTiming)

lib = _lib.lib

K_MAX_WHEEL_INDEX = (2**64 - 1 - 5) // 6          # wheel.hpp:33
K_MAX_SEGMENT_END = 6 * (K_MAX_WHEEL_INDEX + 1)   # wheel.hpp:37
DEFAULT_SEGMENT_SLOTS = 1 << 18


class Errc(enum.IntEnum):
    """errors.hpp:9-23 (same order), plus device-side codes."""
    NotOnWheel = 0
    Overflow = 1
    EmptyRange = 2
    Capacity = 3
    Domain = 4
    Alignment = 5
    BadConfig = 6
    IncompleteBase = 7
    Ordering = 8
    Io = 9
    BadManifest = 10
    ChecksumMismatch = 11
    BeyondFrontier = 12
    Cuda = 99
    NoDevice = 100
    OutOfMemory = 101
    Nccl = 102


class Error(RuntimeError):
    """wheelsieve::Error (errors.hpp:25-32): carries an Errc."""

    def __init__(self, code: Errc, what: str):
        super().__init__(what)
        self.code = code


def _errc(status: int) -> Errc:
    return Errc(status - 1)


def _check(status: int, ctx=None, what: str = "") -> None:
    if status == 0:
        return
    msg = ""
    if ctx is not None:
        msg = (lib.ws_last_error(ctx) or b"").decode()
    name = (lib.ws_status_name(status) or b"?").decode()
    raise Error(_errc(status), f"{what}: {name}: {msg}".strip(": "))


def isqrt(n: int) -> int:
    return int(lib.ws_isqrt(n))


def ceil_sqrt(n: int) -> int:  # wheel.cpp:35-38
    r = isqrt(n)
    return r if r * r == n else r + 1


R1, R5 = 1, 5  # ResidueClass (wheel.hpp:13) as the residue itself


def value_of(index: int, residue: int) -> int:  # wheel.cpp:8-13
    if index > K_MAX_WHEEL_INDEX:
        raise Error(Errc.Overflow, f"wheel index {index} exceeds the 64-bit value range")
    return 6 * index + residue


def coord_of(n: int):  # wheel.cpp:15-23 -> (index, residue)
    if n % 6 not in (1, 5):
        raise Error(Errc.NotOnWheel, f"{n} is divisible by 2 or 3, not on the wheel")
    return n // 6, n % 6


def start_offsets(p: int, segment_start: int):
    """wheel.cpp:96-106 -> (id1, id5)."""
    a, b = C.c_uint64(), C.c_uint64()
    _check(lib.ws_start_offsets(p, segment_start, C.byref(a), C.byref(b)), what="start_offsets")
    return a.value, b.value


def read_back(dir: str, lo: int, hi: int) -> np.ndarray:
    """sink.cpp:306-321: primes in [lo, hi) of a chunked store, CRC-verified."""
    if hi <= lo:
        return np.zeros(0, np.uint64)
    n = C.c_uint64()
    st = lib.ws_read_back(str(dir).encode(), lo, hi, None, 0, C.byref(n))
    if st not in (0, 4):  # 4 = Capacity: just sizing
        _check(st, what="read_back")
    out = np.empty(max(1, n.value), np.uint64)
    _check(lib.ws_read_back(str(dir).encode(), lo, hi, out.ctypes.data, out.size, C.byref(n)),
           what="read_back")
    return out[: n.value].copy()


def verify_store(dir: str) -> None:
    """sink.cpp:323-342; raises Error on the first mismatch."""
    _check(lib.ws_verify_store(str(dir).encode()), what="verify_store")


def prime_count_bound(L: int, R: int) -> int:
    return int(lib.ws_prime_count_bound(L, R))


def partition(L: int, R: int, rank: int, world: int,
              segment_slots: int = DEFAULT_SEGMENT_SLOTS):
    lo, hi = C.c_uint64(), C.c_uint64()
    _check(lib.ws_partition(L, R, segment_slots, rank, world, C.byref(lo), C.byref(hi)),
           what="partition")
    return lo.value, hi.value


@dataclass
class Checks:
    count: int
    sum: int
    xor: int
    largest: int

    @staticmethod
    def of(c: WsChecks) -> "Checks":
        return Checks(c.count, c.sum, c.xor_, c.largest)

    def raw(self) -> WsChecks:
        M = (1 << 64) - 1
        return WsChecks(self.count & M, self.sum & M, self.xor & M, self.largest & M)


def combine_checks(records: Sequence[Checks]) -> Checks:
    """ws_combine_checks: the fold a multi-device context applies to the
    gathered per-shard records (count and sum add mod 2^64, xor folds,
    largest is the maximum)."""
    arr = (WsChecks * max(1, len(records)))(*[r.raw() for r in records])
    out = WsChecks()
    _check(lib.ws_combine_checks(C.addressof(arr), len(records), C.byref(out)),
           what="combine_checks")
    return Checks.of(out)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (WS_NCCL_ID_BYTES bytes) for a multi-process
    context; made on rank 0 and broadcast to the other ranks' Sieve(...)."""
    buf = (C.c_uint8 * WS_NCCL_ID_BYTES)()
    _check(lib.ws_nccl_unique_id(C.addressof(buf)), what="nccl_unique_id")
    return bytes(buf)


def _ptr(a) -> int:
    """Data pointer of a numpy array or a torch tensor."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _is_device(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


class Sieve:
    """A GPU context (device buffers, streams, resident base-prime tables).

    ``Sieve(device=d)`` drives one device with no NCCL.  ``Sieve(devices=[...])``
    drives several devices of this process, one shard each, combined by one
    NCCL all-gather inside the library; with ``world > 1`` (one Sieve per
    process, ``nccl_id`` from ``nccl_unique_id()`` on rank 0) the shards of
    all processes form one job.  Not reentrant: one Sieve per
    host thread."""

    def __init__(self, device: int = -1, segment_slots: int = DEFAULT_SEGMENT_SLOTS,
                 devices: Optional[Sequence[int]] = None, world: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None):
        o = WsOpts()
        lib.ws_opts_default(C.byref(o))
        o.segment_slots = segment_slots
        o.device = device
        if devices is not None:
            devices = list(devices)
            if not 1 <= len(devices) <= WS_MAX_DEVICES:
                raise Error(Errc.BadConfig, f"1..{WS_MAX_DEVICES} devices, got {len(devices)}")
            o.n_devices = len(devices)
            for i, d in enumerate(devices):
                o.device_ids[i] = d
            o.world = world
            o.rank = rank
            if world > 1 and nccl_id is None:
                raise Error(Errc.BadConfig, "world > 1 needs the rank-0 nccl_unique_id()")
            if nccl_id is not None:  # communicators by ncclCommInitRank with this id
                if len(nccl_id) != WS_NCCL_ID_BYTES:
                    raise Error(Errc.BadConfig, f"an NCCL id has {WS_NCCL_ID_BYTES} bytes")
                for i, b in enumerate(nccl_id):
                    o.nccl_id[i] = b
        elif world != 1:
            raise Error(Errc.BadConfig, "a multi-process context needs devices=[...]")
        h = C.c_void_p()
        _check(lib.ws_ctx_create(C.byref(o), C.byref(h)), what="ws_ctx_create")
        self._h = h
        self.segment_slots = segment_slots

    @property
    def num_devices(self) -> int:
        return int(lib.ws_ctx_num_devices(self._h))

    @property
    def num_shards(self) -> int:
        return int(lib.ws_ctx_num_shards(self._h))

    @property
    def devices(self) -> List[int]:
        return [int(lib.ws_ctx_device(self._h, i)) for i in range(self.num_devices)]

    @property
    def streams(self) -> List[int]:
        return [lib.ws_ctx_device_stream(self._h, i) or 0 for i in range(self.num_devices)]

    def device_timing(self, i: int) -> WsTiming:
        t = WsTiming()
        _check(lib.ws_device_timing(self._h, i, C.byref(t)), self._h, "device_timing")
        return t

    def comm_info(self, i: int = 0):
        """(ranks in local device i's NCCL communicator, its rank there)."""
        n, r = C.c_int32(), C.c_int32()
        _check(lib.ws_ctx_comm_info(self._h, i, C.byref(n), C.byref(r)), self._h, "comm_info")
        return n.value, r.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.ws_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self) -> int:
        return lib.ws_ctx_stream(self._h) or 0

    def timing(self) -> WsTiming:
        t = WsTiming()
        _check(lib.ws_last_timing(self._h, C.byref(t)), self._h, "timing")
        return t

    # -- [L, R) entry points -------------------------------------------------
    def count_range(self, L: int, R: int, checks: bool = False, per_seg=None,
                    fresh_base: bool = False):
        """Primes in [L, R).  per_seg: None, True (returns a new uint32 array)
        or a preallocated numpy / CUDA tensor of uint32 (int32) counts."""
        out = WsChecks()
        n = C.c_uint64()
        flags = (WS_WANT_CHECKS if checks else 0) | (WS_FRESH_BASE if fresh_base else 0)
        ps_ptr, cap, ret = None, 0, None
        if per_seg is True:
            nseg = self.num_segments(L, R)
            ret = np.zeros(max(1, nseg), np.uint32)
            ps_ptr, cap = ret.ctypes.data, ret.size
        elif per_seg is not None:
            ps_ptr, cap = _ptr(per_seg), per_seg.numel() if _is_device(per_seg) else per_seg.size
            if _is_device(per_seg):
                flags |= WS_OUT_DEVICE
        _check(lib.ws_count_range(self._h, L, R, flags, C.byref(out), ps_ptr, cap, C.byref(n)),
               self._h, "count_range")
        res = Checks.of(out)
        if per_seg is True:
            return res, ret[: n.value]
        return res

    def enumerate_range(self, L: int, R: int, out=None, fresh_base: bool = False):
        """Sorted primes of [L, R).  out: None (a new numpy array is returned),
        a numpy uint64 array, or a CUDA tensor (int64/uint64) on the ctx device.
        Returns (values_or_out, n, Checks)."""
        flags = WS_FRESH_BASE if fresh_base else 0
        own = out is None
        if own:
            out = np.empty(max(1, prime_count_bound(L, R)), np.uint64)
        if _is_device(out):
            flags |= WS_OUT_DEVICE
            cap = out.numel()
        else:
            cap = out.size
        n = C.c_uint64()
        chk = WsChecks()
        _check(lib.ws_enumerate_range(self._h, L, R, flags, _ptr(out), cap, C.byref(n),
                                      C.byref(chk)), self._h, "enumerate_range")
        if own:
            # a view (no multi-GB copy) unless the capacity bound was much
            # larger than the result
            v = out[: n.value]
            return (v if 2 * n.value >= out.size else v.copy()), n.value, Checks.of(chk)
        return out, n.value, Checks.of(chk)

    def count_intervals(self, Ls, width: int, want_sums: bool = True, want_xors: bool = True,
                        fresh_base: bool = False):
        """Per-interval (counts uint32, sums uint64, xors uint64) of [L_i, L_i + width)."""
        Ls = np.ascontiguousarray(Ls, dtype=np.uint64)
        n = Ls.size
        counts = np.zeros(n, np.uint32)
        sums = np.zeros(n, np.uint64) if want_sums else None
        xors = np.zeros(n, np.uint64) if want_xors else None
        flags = WS_FRESH_BASE if fresh_base else 0
        _check(lib.ws_count_intervals(self._h, Ls.ctypes.data, n, width, flags,
                                      counts.ctypes.data,
                                      sums.ctypes.data if sums is not None else None,
                                      xors.ctypes.data if xors is not None else None),
               self._h, "count_intervals")
        return counts, sums, xors

    def enumerate_shards(self, L: int, R: int, outs, fresh_base: bool = False):
        """Multi-device: local device i enumerates its shard of [L, R) into
        outs[i] (a CUDA tensor on that device).  Returns (counts, Checks)."""
        n = self.num_devices
        if len(outs) != n:
            raise Error(Errc.BadConfig, f"{n} output tensors needed")
        ptrs = (C.c_uint64 * n)(*[o.data_ptr() for o in outs])
        caps = (C.c_uint64 * n)(*[o.numel() for o in outs])
        counts = (C.c_uint64 * n)()
        chk = WsChecks()
        _check(lib.ws_enumerate_shards(self._h, L, R, WS_FRESH_BASE if fresh_base else 0,
                                       C.addressof(ptrs), C.addressof(caps), C.addressof(counts),
                                       C.byref(chk)), self._h, "enumerate_shards")
        return [int(c) for c in counts], Checks.of(chk)

    def count_ranges(self, Ls, Rs, checks: bool = False, fresh_base: bool = False):
        """Per-range Checks of [Ls[i], Rs[i]) (each sieved independently; the
        per-worker-tile counts of run())."""
        Ls = np.ascontiguousarray(Ls, dtype=np.uint64)
        Rs = np.ascontiguousarray(Rs, dtype=np.uint64)
        if Ls.shape != Rs.shape:
            raise Error(Errc.BadConfig, "Ls and Rs differ in length")
        n = Ls.size
        out = (WsChecks * max(1, n))()
        flags = (WS_WANT_CHECKS if checks else 0) | (WS_FRESH_BASE if fresh_base else 0)
        _check(lib.ws_count_ranges(self._h, Ls.ctypes.data, Rs.ctypes.data, n, flags,
                                   C.addressof(out)),
               self._h, "count_ranges")
        return [Checks.of(out[i]) for i in range(n)]

    def base_primes(self, B: int, fresh_base: bool = False) -> np.ndarray:
        """BasePrimeStore::bootstrap entries: wheel primes 5 <= p <= B (device-sieved)."""
        out = np.empty(max(1, prime_count_bound(0, B + 1)), np.uint64)
        n = C.c_uint64()
        _check(lib.ws_base_primes(self._h, B, WS_FRESH_BASE if fresh_base else 0,
                                  out.ctypes.data, out.size, C.byref(n)), self._h, "base_primes")
        return out[: n.value].copy()

    def sieve_segment(self, start: int, length: int):
        """SegmentBitmap(start, length) after sieve_segment: (r1_words, r5_words),
        uint64 FlagArray Bit layout, value 1 left set like the reference."""
        nw = (length + 63) // 64
        r1 = np.zeros(max(1, nw), np.uint64)
        r5 = np.zeros(max(1, nw), np.uint64)
        _check(lib.ws_sieve_segment(self._h, start, length, 0, r1.ctypes.data, r5.ctypes.data),
               self._h, "sieve_segment")
        return r1[:nw], r5[:nw]

    def store_range(self, L: int, R: int, dir: str, binary: bool = True,
                    primes_per_file: int = 125_000_000) -> int:
        """ChunkedFileSink-format store of the primes of [L, R) (frontier R)."""
        n = C.c_uint64()
        _check(lib.ws_store_range(self._h, L, R, str(dir).encode(), 1 if binary else 0,
                                  primes_per_file, C.byref(n)), self._h, "store_range")
        return n.value

    def num_segments(self, L: int, R: int) -> int:
        if R <= L:
            return 0
        lo0 = L // 6 * 6
        slots = (R - lo0 + 5) // 6
        return (slots + self.segment_slots - 1) // self.segment_slots


# ---------------------------------------------------------------------------
# run(SieveConfig) drop-in (engine.hpp:13-89, sink.hpp:18-66)

class PrimeSink:
    """sink.hpp:18-43: strictly ascending batches; emit_count for count sinks."""

    def __init__(self):
        self._count = 0
        self._largest = 0

    def emit(self, batch) -> None:  # sink.cpp:14-26
        batch = np.asarray(batch, dtype=np.uint64)
        if batch.size == 0:
            return
        if int(batch[0]) <= self._largest or (batch.size > 1 and not bool(np.all(batch[1:] > batch[:-1]))):
            raise Error(Errc.Ordering, f"emit batch not strictly ascending past {self._largest}")
        self.accept(batch)
        self._count += int(batch.size)
        self._largest = int(batch[-1])

    def emit_count(self, n: int, largest: int) -> None:  # sink.cpp:28-37
        if n == 0:
            return
        if self.wants_values():
            raise Error(Errc.Domain, "sink needs the values; count-only emission not possible")
        if largest <= self._largest:
            raise Error(Errc.Ordering, f"count batch ends at {largest}, not above {self._largest}")
        self._count += n
        self._largest = largest

    def flush(self) -> None:
        pass

    def wants_values(self) -> bool:
        return True

    def count(self) -> int:
        return self._count

    def largest(self) -> int:
        return self._largest

    def accept(self, batch) -> None:
        raise NotImplementedError


class CountSink(PrimeSink):
    def wants_values(self) -> bool:
        return False

    def accept(self, batch) -> None:
        pass


class MemorySink(PrimeSink):
    def __init__(self):
        super().__init__()
        self._chunks: List[np.ndarray] = []

    def accept(self, batch) -> None:
        self._chunks.append(np.array(batch, dtype=np.uint64))

    def primes(self) -> np.ndarray:
        return np.concatenate(self._chunks) if self._chunks else np.zeros(0, np.uint64)


@dataclass
class SieveConfig:
    """engine.hpp:13-29.  `threads` is kept for signature parity (the device
    decides its own parallelism); segment_span still sets the iteration
    size used for emission batches and the SieveReport accounting."""
    limit: Optional[int] = None
    threads: int = 1
    segment_span: int = 6_000_000
    flag_width: int = 0
    sink: Optional[PrimeSink] = None
    spawn_per_iteration: bool = False
    thread_cap: int = 1024


@dataclass
class SieveReport:  # engine.hpp:42-55
    prime_count: int = 0
    largest_prime: int = 0
    iterations: int = 0
    wall_ms: float = 0.0
    peak_flag_bytes: int = 0
    peak_flag_entries: int = 0
    sieved_to: int = 0
    stopped: bool = False
    overflowed: bool = False


class SinkFailure(Error):
    def __init__(self, code, what, partial: SieveReport):
        super().__init__(code, what)
        self.partial = partial


def round_segment_span(span: int, threads: int) -> int:  # engine.cpp:311-320
    if threads == 0:
        raise Error(Errc.BadConfig, "thread count must be positive")
    align = 6 * threads
    if span == 0:
        return align
    if span % align == 0:
        return span
    if span > 2**64 - 1 - align:
        raise Error(Errc.Overflow, "segment span exceeds the 64-bit value range")
    return (span // align + 1) * align


def _validate(config: SieveConfig, bounded: bool = True) -> None:  # engine.cpp:119-143
    if config.sink is None:
        raise Error(Errc.BadConfig, "config has no sink")
    if config.threads == 0:
        raise Error(Errc.BadConfig, "thread count must be positive")
    if config.threads > config.thread_cap:
        raise Error(Errc.BadConfig, "thread count exceeds the cap")
    align = 6 * config.threads
    if config.segment_span == 0 or config.segment_span % align:
        raise Error(Errc.BadConfig, f"segment span {config.segment_span} is not a positive multiple of {align}")
    if config.segment_span > K_MAX_SEGMENT_END:
        raise Error(Errc.BadConfig, "segment span exceeds the 64-bit value range")
    if bounded:
        if config.limit is None:
            raise Error(Errc.BadConfig, "bounded run requires a limit")
        if config.limit < 2:
            raise Error(Errc.EmptyRange, "no primes below 2")
        if config.limit > K_MAX_SEGMENT_END - 1:
            raise Error(Errc.Overflow, "limit exceeds the sievable 64-bit range")
    elif config.limit is not None:
        raise Error(Errc.BadConfig, "unbounded run cannot take a limit")


_default_sieve: Optional[Sieve] = None


def _sieve() -> Sieve:
    global _default_sieve
    if _default_sieve is None:
        _default_sieve = Sieve()
    return _default_sieve


_WIDTH_BYTES = {0: lambda n: (n + 7) // 8, 1: lambda n: n, 2: lambda n: 4 * n}
_CALL_VALUES = 1 << 28   # integers enumerated per device call for value sinks
_CALL_COUNT = 1 << 36    # integers counted per device call for count sinks ...
_CALL_TILES = 1 << 16    # ... and at most this many worker tiles per call


@dataclass
class WorkerAssignment:  # engine.hpp:34-40
    iteration: int
    worker: int
    lo: int
    hi: int


def plan_iteration(config: SieveConfig, iteration: int) -> List[WorkerAssignment]:
    """engine.cpp:322-342: iteration i = [i S, (i+1) S) cut into `threads`
    equal tiles in worker order."""
    if config.threads == 0 or config.threads > config.thread_cap:
        raise Error(Errc.BadConfig, "invalid thread count")
    span, align = config.segment_span, 6 * config.threads
    if span == 0 or span % align or span > K_MAX_SEGMENT_END:
        raise Error(Errc.BadConfig, f"segment span {span} is not a positive multiple of {align}")
    if iteration > K_MAX_SEGMENT_END // span - 1:
        raise Error(Errc.Overflow, f"iteration {iteration} leaves the 64-bit value range")
    sub = span // config.threads
    return [WorkerAssignment(iteration, j, iteration * span + j * sub,
                             iteration * span + (j + 1) * sub) for j in range(config.threads)]


def _tiles(config: SieveConfig, seg_lo: int, seg_hi: int):
    """The non-empty worker tiles of one iteration, clipped to seg_hi
    (engine.cpp:233-241)."""
    sub = config.segment_span // config.threads
    out = []
    for j in range(config.threads):
        lo = seg_lo + j * sub
        if lo >= seg_hi:
            break
        out.append((lo, seg_hi if sub > seg_hi - lo else lo + sub))
    return out


def _account(config: SieveConfig, tiles, rep: SieveReport) -> None:
    """Analytic flag-storage accounting of one iteration (engine.cpp:218-230)."""
    ent = byt = 0
    for lo, hi in tiles:
        n = (hi - lo) // 6
        ent += 2 * n
        byt += 2 * _WIDTH_BYTES[config.flag_width](n)
    rep.peak_flag_entries = max(rep.peak_flag_entries, ent)
    rep.peak_flag_bytes = max(rep.peak_flag_bytes, byt)


def _run_loop(config: SieveConfig, stop, sv: Sieve) -> SieveReport:
    """engine.cpp:149-307 on the device, with the reference's emission
    granularity: 2 and 3 first, then for every iteration one batch per
    non-empty worker tile in worker order -- ``emit(values)`` for value
    sinks, ``emit_count(count, largest)`` for count sinks (engine.cpp:277-288).
    The device sieves a block of iterations per call (every tile of the block
    as one ws_count_ranges batch, or one ordered enumeration cut at the tile
    borders on the host); emission and the stop check still go iteration by
    iteration, so a sink sees exactly the reference's batches."""
    bounded = stop is None
    _validate(config, bounded)
    sink = config.sink
    t0 = time.perf_counter()
    span = config.segment_span
    limit = config.limit if bounded else 0
    limit_end = (limit // 6 + 1) * 6 if bounded else K_MAX_SEGMENT_END
    total_iters = limit_end // span + (limit_end % span != 0) if bounded else None
    top_value = limit + 1 if bounded else K_MAX_SEGMENT_END
    rep = SieveReport()
    want_values = sink.wants_values()
    if want_values:
        per_call = max(1, _CALL_VALUES // span)
    else:
        per_call = max(1, min(_CALL_COUNT // span, _CALL_TILES // config.threads))
    block: dict = {}
    block_end = 0
    i = 0
    seg_lo = 0
    try:
        while True:
            if bounded and i >= total_iters:
                break
            if stop is not None and stop():
                rep.stopped = True
                break
            if not bounded and seg_lo > K_MAX_SEGMENT_END - span:
                rep.overflowed = True
                break
            seg_hi = limit_end if (bounded and span > limit_end - seg_lo) else seg_lo + span
            tiles = _tiles(config, seg_lo, seg_hi)
            _account(config, tiles, rep)
            if i >= block_end:  # sieve the next block of iterations on the device
                n_it = min(per_call, (K_MAX_SEGMENT_END - seg_lo) // span)
                if bounded:
                    n_it = min(n_it, total_iters - i)
                bhi = min(seg_lo + n_it * span, limit_end)
                blk_tiles = [t for k in range(n_it)
                             for t in _tiles(config, seg_lo + k * span,
                                             min(seg_lo + (k + 1) * span, bhi))]
                if want_values:
                    lo_v, hi_v = max(seg_lo, 4), min(bhi, top_value)
                    vals = sv.enumerate_range(lo_v, hi_v)[0] if lo_v < hi_v else \
                        np.zeros(0, np.uint64)
                    block = {"vals": vals}
                else:
                    Ls = [max(lo, 4) for lo, _ in blk_tiles]
                    Rs = [max(max(lo, 4), min(hi, top_value)) for lo, hi in blk_tiles]
                    res = sv.count_ranges(Ls, Rs)
                    block = {(lo, hi): r for (lo, hi), r in zip(blk_tiles, res)}
                block_end = i + n_it
            if i == 0:  # engine.cpp:268-276
                n = 2 if (not bounded or limit >= 3) else 1
                if want_values:
                    sink.emit(np.array([2, 3][:n], np.uint64))
                else:
                    sink.emit_count(n, 3 if n == 2 else 2)
            for lo, hi in tiles:
                if want_values:
                    v = block["vals"]
                    a = int(np.searchsorted(v, np.uint64(lo), side="left"))
                    b = int(np.searchsorted(v, np.uint64(min(hi, top_value)), side="left"))
                    if b > a:
                        sink.emit(v[a:b])
                else:
                    r = block[(lo, hi)]
                    if r.count:
                        sink.emit_count(r.count, r.largest)
            rep.iterations = i + 1
            rep.sieved_to = seg_hi
            i += 1
            seg_lo += span
    except Error as e:
        if isinstance(e, SinkFailure) or e.code in (Errc.Cuda, Errc.NoDevice, Errc.OutOfMemory,
                                                     Errc.Nccl):
            raise
        rep.prime_count = sink.count()
        rep.largest_prime = sink.largest()
        rep.wall_ms = (time.perf_counter() - t0) * 1e3
        raise SinkFailure(e.code, str(e), rep) from e
    if bounded:
        rep.sieved_to = limit + 1
    rep.prime_count = sink.count()
    rep.largest_prime = sink.largest()
    rep.wall_ms = (time.perf_counter() - t0) * 1e3
    return rep


def run(config: SieveConfig, sieve: Optional[Sieve] = None) -> SieveReport:
    """engine.hpp:83 on the GPU: every prime <= limit into config.sink."""
    return _run_loop(config, None, sieve or _sieve())


def run_unbounded(config: SieveConfig, stop, sieve: Optional[Sieve] = None) -> SieveReport:
    """engine.hpp:89 on the GPU.  `stop` is a zero-argument callable (or an
    object with is_set(), e.g. threading.Event) checked between iterations."""
    fn = stop.is_set if hasattr(stop, "is_set") else stop
    return _run_loop(config, fn, sieve or _sieve())


class PrimeStream:
    """stream.hpp:16-46 on the GPU: 2, 3, then every wheel prime ascending;
    each refill sieves `segments_per_refill` segments of segment_wheel_len
    slots on the device.  next() returns None once the 64-bit range is
    exhausted (overflowed() then stays true)."""

    def __init__(self, segment_wheel_len: int, sieve: Optional[Sieve] = None,
                 segments_per_refill: int = 64):
        if segment_wheel_len == 0:
            raise Error(Errc.Domain, "segment must span at least one wheel index")
        if segment_wheel_len > K_MAX_SEGMENT_END // 6:
            raise Error(Errc.Overflow, "segment span exceeds the 64-bit value range")
        self._sv = sieve or _sieve()
        self._len = segment_wheel_len
        # refills batch whole segments up to a value budget (a single segment
        # may exceed it, as the reference's own buffer would)
        per = max(1, min(segments_per_refill, _CALL_VALUES // (6 * segment_wheel_len)))
        self._span = 6 * segment_wheel_len * per
        self._next = 0
        self._buf = np.zeros(0, np.uint64)
        self._pos = 0
        self._prelude = 0
        self._overflowed = False

    @staticmethod
    def segment_would_overflow(start: int, wheel_len: int) -> bool:  # stream.cpp:24-26
        return start >= K_MAX_SEGMENT_END or wheel_len > (K_MAX_SEGMENT_END - start) // 6

    def overflowed(self) -> bool:
        return self._overflowed

    def _refill(self):
        if self.segment_would_overflow(self._next, self._len):
            self._overflowed = True
            return
        end = self._next + self._span
        if self.segment_would_overflow(self._next, self._span // 6):
            end = self._next + 6 * self._len * ((K_MAX_SEGMENT_END - self._next) // (6 * self._len))
        self._buf = self._sv.enumerate_range(max(self._next, 4), end)[0]
        self._pos = 0
        self._next = end

    def next(self):
        if self._prelude < 2:
            self._prelude += 1
            return 2 if self._prelude == 1 else 3
        while self._pos == self._buf.size:
            if self._overflowed:
                return None
            self._refill()
        v = int(self._buf[self._pos])
        self._pos += 1
        return v

    def __iter__(self):
        return self

    def __next__(self):
        v = self.next()
        if v is None:
            raise StopIteration
        return v
