"""GPU: seeded fuzz of every range entry point against the oracle, across
segment sizes, bucket policies and ragged interval batches."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2310_17746_b200 as ws

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _t(c):
    return (c.count, c.sum, c.xor, c.largest)


@pytest.mark.parametrize("slots", [1 << 12, 1 << 13, 1 << 15, 1 << 17, 1 << 18])
def test_fuzz_segment_sizes(port, slots):
    rng = np.random.default_rng(slots)
    with ws.Sieve(segment_slots=slots) as sv:
        for _ in range(12):
            L = int(rng.choice([rng.integers(0, 10**4), rng.integers(0, 10**10),
                                rng.integers(10**13, 10**15)]))
            W = int(rng.integers(1, 3 * slots * 6))
            ref = port.range(L, L + W, seg_slots=slots, per_seg=True, values=True)
            c, ps = sv.count_range(L, L + W, checks=True, per_seg=True)
            assert _t(c) == (ref["count"], ref["sum"], ref["xor"], ref["largest"]), (slots, L, W)
            assert np.array_equal(ps, ref["per_seg"])
            v, n, ce = sv.enumerate_range(L, L + W)
            assert np.array_equal(v, ref["values"]) and _t(ce) == _t(c)


def test_fuzz_intervals_ragged(port):
    rng = np.random.default_rng(99)
    with ws.Sieve() as sv:
        for width in (1, 5, 6, 7, 1000, 123_457, 2_000_003):
            Ls = rng.integers(0, 10**12, size=17).astype(np.uint64)
            Ls[0] = 0
            Ls[1] = 1
            counts, sums, xors = sv.count_intervals(Ls, width)
            for i, L in enumerate(Ls):
                r = port.range(int(L), int(L) + width)
                assert (int(counts[i]), int(sums[i]), int(xors[i])) == (r["count"], r["sum"],
                                                                         r["xor"]), (width, L)


BUCKET_FUZZ = r"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2310_17746_b200 as ws
from oracle.oracle import Port
port = Port()
rng = np.random.default_rng(5)
with ws.Sieve() as sv:
    for _ in range(10):
        L = int(rng.integers(10**11, 10**15))
        W = int(rng.integers(10**5, 4 * 10**6))
        r = port.range(L, L + W, per_seg=True)
        c, ps = sv.count_range(L, L + W, checks=True, per_seg=True)
        assert (c.count, c.sum, c.xor, c.largest) == (r["count"], r["sum"], r["xor"], r["largest"]), (L, W)
        assert np.array_equal(ps, r["per_seg"])
    Ls = rng.integers(2**32, 2**40, size=9).astype(np.uint64)
    counts, sums, xors = sv.count_intervals(Ls, 3 * 10**6)
    for i, L in enumerate(Ls):
        r = port.range(int(L), int(L) + 3 * 10**6)
        assert (int(counts[i]), int(sums[i]), int(xors[i])) == (r["count"], r["sum"], r["xor"])
print("ok")
"""


@pytest.mark.parametrize("env", [{"WHEELSIEVE_BUCKET_RATIO": "1", "WHEELSIEVE_BUCKET_PMIN": "1"},
                                 {"WHEELSIEVE_BUCKET_RATIO": "1", "WHEELSIEVE_BUCKET_PMIN": "3",
                                  "WHEELSIEVE_FILL_PIECE": "7",
                                  "WHEELSIEVE_BUCKET_BUDGET": str(3 << 20)},
                                 {"WHEELSIEVE_BUCKET_RATIO": "1", "WHEELSIEVE_BUCKET_CAP": "100",
                                  "WHEELSIEVE_BUCKET_CTAS": "1"},
                                 # the carried-offset fill for p >= run length: off, and
                                 # with short runs taken three at a time
                                 {"WHEELSIEVE_BUCKET_RATIO": "1", "WHEELSIEVE_FILL_HUGE": "0"},
                                 {"WHEELSIEVE_BUCKET_RATIO": "1", "WHEELSIEVE_FILL_PIECE": "5",
                                  "WHEELSIEVE_HUGE_STEP": "3",
                                  "WHEELSIEVE_BUCKET_BUDGET": str(5 << 20)}])
def test_fuzz_bucket_policies(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", BUCKET_FUZZ], cwd=ROOT, env=e, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_abi_error_paths(sieve, tmp_path):
    import ctypes as C
    from paper_2310_17746_b200 import _lib
    lib = _lib.lib
    n = C.c_uint64()
    # null outputs / contexts are rejected, never crash
    assert lib.ws_count_range(None, 0, 10, 0, None, None, 0, None) == 7
    assert lib.ws_count_range(sieve._h, 0, 10, 0, None, None, 0, None) == 7
    assert lib.ws_enumerate_range(sieve._h, 0, 100, 0, None, 5, C.byref(n), None) == 7
    assert lib.ws_count_intervals(sieve._h, None, 3, 10, 0, None, None, None) == 7
    Ls = np.array([10, 20], np.uint64)
    counts = np.zeros(2, np.uint32)
    assert lib.ws_count_intervals(sieve._h, Ls.ctypes.data, 2, 0, 0, counts.ctypes.data,
                                  None, None) == 3  # EmptyRange
    assert lib.ws_count_intervals(sieve._h, Ls.ctypes.data, 0, 10, 0, counts.ctypes.data,
                                  None, None) == 0
    assert lib.ws_partition(0, 10, 1 << 18, 2, 2, C.byref(n), C.byref(n)) == 7
    assert lib.ws_store_range(sieve._h, 0, 10, None, 0, 10, C.byref(n)) == 7
    assert lib.ws_store_range(sieve._h, 0, 10, str(tmp_path).encode(), 2, 10, C.byref(n)) == 7
    assert lib.ws_read_back(str(tmp_path / "nope").encode(), 0, 10, None, 0, C.byref(n)) == 11
    assert lib.ws_verify_store(str(tmp_path / "nope").encode()) == 11
    # the context stays usable after errors
    assert sieve.count_range(0, 101).count == 25
    t = sieve.timing()
    assert t.total_ms >= 0
    assert (lib.ws_last_error(sieve._h) or b"") == b""


def test_context_lifecycle_releases_device_memory():
    """Every path's scratch (wire ring, bucket windows, interval jobs, segment
    export) is released by ws_ctx_destroy: device memory returns to baseline
    over repeated create / use / destroy cycles."""
    import torch

    def cycle():
        with ws.Sieve() as s:
            v, n, _ = s.enumerate_range(10**12, 10**12 + 3 * 10**8)  # wire path
            assert n == v.size > 0
            s.count_range(10**15, 10**15 + 2 * 10**9, checks=True)  # bucket windows
            s.count_intervals(np.arange(5, dtype=np.uint64) * 2**30 + 2**40, 2**20)
            s.sieve_segment(6 * 10**9, 4096)
        torch.cuda.synchronize()

    cycle()  # first use: CUDA context, module load
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(4):
        cycle()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, (free0, free1)


def test_concurrent_contexts_in_threads():
    """One context per host thread (the ABI's threading rule): four threads
    enumerating (wire path) and counting concurrently get exactly the results
    a single thread gets."""
    import threading

    jobs = [(10**12 + k * 10**9, 3 * 10**8) for k in range(4)]
    want = {}
    with ws.Sieve() as s:
        for L, W in jobs:
            v, n, c = s.enumerate_range(L, L + W)
            want[L] = (n, c.sum, c.xor, int(v.sum(dtype=np.uint64)), s.count_range(L, L + W).count)
    got, errs = {}, []

    def work(L, W):
        try:
            with ws.Sieve() as s:
                for _ in range(2):
                    v, n, c = s.enumerate_range(L, L + W)
                    cnt = s.count_range(L, L + W).count
                got[L] = (n, c.sum, c.xor, int(v.sum(dtype=np.uint64)), cnt)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=j) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert got == want


def test_repeated_calls_reuse_launch_state(port):
    """Launch state that kernels reset themselves (segment tickets: the last
    CTA out zeroes them) and epoch-tagged small-base counts stay consistent
    over many back-to-back calls whose grids, windows, job counts and base
    builds differ from call to call."""
    rng = np.random.default_rng(77)
    cases = [(0, 10**6 + 1), (10**9, 10**9 + 3 * 10**7), (10**15, 10**15 + 10**8),
             (2**40, 2**40 + 5 * 10**6), (12345, 12346 + 6 * 2**18 * 7), (10**12 - 7, 10**12 + 10**7)]
    want = {}
    for L, R in cases:
        r = port.range(L, R)
        want[(L, R)] = (r["count"], r["sum"], r["xor"], r["largest"])
    Ls = np.array([2**33 + 977 * k for k in range(37)], np.uint64)
    ic, isum, ixor = port.intervals(Ls, 10**5)
    with ws.Sieve() as s:
        for it in range(60):
            L, R = cases[int(rng.integers(len(cases)))]
            fresh = bool(rng.integers(2))
            if it % 5 == 4:
                c, sm, x = s.count_intervals(Ls, 10**5, fresh_base=fresh)
                assert [int(v) for v in c] == [int(v) for v in ic], it
                assert [int(v) for v in sm] == [int(v) for v in isum], it
            elif it % 3 == 0 and R - L <= 3 * 10**7:
                v, n, c = s.enumerate_range(L, R, fresh_base=fresh)
                assert (n, c.sum, c.xor) == want[(L, R)][:3], (it, L, R)
            else:
                c = s.count_range(L, R, checks=True, fresh_base=fresh)
                assert _t(c) == want[(L, R)], (it, L, R, fresh)
