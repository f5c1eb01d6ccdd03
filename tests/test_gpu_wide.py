"""GPU: the wide count kernel (sieve_wide_kernel: one 1024-thread CTA per SM
sieving 3 segments as one unit) against the goldens, the oracle and the
per-segment kernel.  WHEELSIEVE_WIDE_MIN_UNITS=0 routes every eligible count
launch -- however short -- through it, so the unit edges (clipped last unit,
ranges shorter than a unit, value 1, the stamped primes of the first words),
the unit tables of bucket windows and of several jobs, and bucket-list
overflow are all exercised at sizes the oracle checks in seconds."""
import os

import numpy as np
import pytest

import paper_2310_17746_b200 as ws
from conftest import load_golden

pytestmark = pytest.mark.gpu


def _t(c):
    return (c.count, c.sum, c.xor, c.largest)


class _Env:
    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _wide(width=3, **kv):
    """A context whose count launches all take the wide kernel (the knobs are
    read when the context is created)."""
    env = dict(WHEELSIEVE_WIDE=width, WHEELSIEVE_WIDE_BUCKET=width, WHEELSIEVE_WIDE_MULTI=width,
               WHEELSIEVE_WIDE_MIN_UNITS=0)
    env.update(kv)
    with _Env(**env):
        return ws.Sieve()


def _narrow():
    with _Env(WHEELSIEVE_WIDE=0, WHEELSIEVE_WIDE_BUCKET=0, WHEELSIEVE_WIDE_MULTI=0):
        return ws.Sieve()


@pytest.mark.parametrize("width", [2, 3])
def test_wide_window_goldens_per_segment(golden, width):
    with _wide(width) as sv:
        for rec in golden["windows"]:
            c, ps = sv.count_range(rec["L"], rec["R"], checks=True, per_seg=True)
            assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec
            assert [int(x) for x in ps] == rec["seg18"], (rec["L"], rec["R"])
            c2 = sv.count_range(rec["L"], rec["R"])
            assert (c2.count, c2.largest) == (rec["count"], rec["largest"])
        for rec in golden["prefixes"]:
            c = sv.count_range(0, rec["limit"] + 1, checks=True)
            assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec["limit"]
        assert sv.timing().launches >= 1


def test_wide_tiny_ranges_exhaustive(port):
    with _wide() as sv:
        for L in range(0, 40):
            for R in range(L, 64):
                ref = port.range(L, R)
                c = sv.count_range(L, R, checks=True)
                assert _t(c) == (ref["count"], ref["sum"], ref["xor"], ref["largest"]), (L, R)


def test_wide_config1_per_segment_golden():
    g = load_golden("c1_per_segment.json")
    with _wide() as sv:
        c, ps = sv.count_range(0, 10**9 + 1, per_seg=True)
        assert c.count == g["count"] and c.largest == g["largest"]
        assert [int(x) for x in ps] == g["seg18"]


def test_wide_unit_edges_against_oracle(port):
    """Ranges of 1..7 segments +- a few slots: every clipped-unit shape."""
    S6 = 6 * (1 << 18)
    rng = np.random.default_rng(7)
    with _wide() as sv:
        for nseg in (1, 2, 3, 4, 5, 6, 7):
            for delta in (-7, -1, 0, 1, 5):
                L = int(rng.integers(0, 10**11))
                R = L + nseg * S6 + delta
                ref = port.range(L, R, per_seg=True)
                c, ps = sv.count_range(L, R, checks=True, per_seg=True)
                assert _t(c) == (ref["count"], ref["sum"], ref["xor"], ref["largest"]), (L, R)
                assert np.array_equal(ps, ref["per_seg"]), (L, R)


def test_wide_equals_per_segment_kernel_large_windows():
    """Windows too long for the oracle: both kernels, every accumulator and
    every per-segment count (high offsets take the 64-bit Barrett path)."""
    rng = np.random.default_rng(11)
    with _wide() as a, _narrow() as b:
        for base, width in ((10**10, 10**9), (10**12, 10**9), (10**15, 5 * 10**8),
                            (10**17, 3 * 10**7)):
            L = base + int(rng.integers(0, 10**6))
            R = L + int(rng.integers(width // 2, width))
            ca, pa = a.count_range(L, R, checks=True, per_seg=True)
            cb, pb = b.count_range(L, R, checks=True, per_seg=True)
            assert _t(ca) == _t(cb), (L, R)
            assert np.array_equal(pa, pb), (L, R)


def test_wide_bucket_window_golden_and_overflow():
    """C4's window (bucket lists, unit table) against the reference golden;
    then with a list capacity so small that every list overflows (the unit
    falls back to its primes' direct path) and with short windows."""
    g = load_golden("reference_big.json")["c4"]
    L, R = g["L"], g["R"]
    with _wide() as sv:
        c = sv.count_range(L, R, checks=True)
        assert _t(c) == (g["count"], g["sum"], g["xor"], g["largest"])
    with _wide(WHEELSIEVE_BUCKET_CAP=64) as sv:
        c = sv.count_range(L, L + 2 * 10**8, checks=True)
    with _narrow() as nv:
        ref = nv.count_range(L, L + 2 * 10**8, checks=True)
    assert _t(c) == _t(ref)
    with _wide(WHEELSIEVE_BUCKET_BUDGET=1 << 22) as sv:  # windows of a few segments
        c = sv.count_range(L, L + 2 * 10**8, checks=True)
    assert _t(c) == _t(ref)


def test_wide_interval_batches_and_range_batches(port):
    """Several jobs per launch: C5-style intervals (bucket windows whose units
    stop at job borders) against the golden, ragged ranges against the oracle."""
    g = load_golden("c5_intervals.json")
    Ls = np.array(g["L"][:512], dtype=np.uint64)
    with _wide() as sv:
        counts, sums, xors = sv.count_intervals(Ls, g["width"])
        assert [int(x) for x in counts] == g["counts"][:512]
        assert [int(x) for x in sums] == g["sums"][:512]
        rng = np.random.default_rng(5)
        lo = rng.integers(0, 10**10, size=9).astype(np.uint64)
        hi = lo + rng.integers(1, 4 * 10**7, size=9).astype(np.uint64)
        res = sv.count_ranges(lo, hi, checks=True)
        for L, R, c in zip(lo, hi, res):
            ref = port.range(int(L), int(R))
            assert _t(c) == (ref["count"], ref["sum"], ref["xor"], ref["largest"]), (L, R)
