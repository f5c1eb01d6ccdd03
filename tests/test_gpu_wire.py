"""Host-bound enumeration through the 8-bit wire format (kEnumWire +
csrc/ws_wire.cpp): every multi-chunk host enumeration takes this path, so its
VALUES (not only the device-side checksums) are checked here -- against the
oracle on multi-chunk windows at segment sizes 2^12, 2^16 and 2^18 (32, 512
and 2048 128-slot wire blocks per segment; clipped last segments), against
the reference goldens on [0, 1e10), under a truncating capacity, and against
the uint64 D2H path."""
import os

import numpy as np
import pytest

import paper_2310_17746_b200 as ws

pytestmark = pytest.mark.gpu


def _host_checks(v):
    v = np.asarray(v, dtype=np.uint64)
    return (int(v.size), int(v.sum(dtype=np.uint64)) if v.size else 0,
            int(np.bitwise_xor.reduce(v)) if v.size else 0, int(v[-1]) if v.size else 0)


@pytest.mark.parametrize("slots,L,W", [
    (1 << 12, 10**12 - 7, 3 * 10**7),        # 1221 segments
    (1 << 16, 2**40 + 1, 2 * 10**8),
    (1 << 18, 10**15, 4 * 10**8),            # 255 segments
    (1 << 18, 0, 3 * 10**8 + 1),             # dense start (2, 3 prelude + wire)
])
def test_multichunk_windows_vs_oracle(port, slots, L, W):
    s = ws.Sieve(segment_slots=slots)
    assert s.num_segments(L, L + W) >= 128  # several chunks -> wire path
    vals, n, c = s.enumerate_range(L, L + W)
    r = port.range(L, L + W)
    assert n == r["count"] == vals.size
    assert (c.count, c.sum, c.xor, c.largest) == (r["count"], r["sum"], r["xor"], r["largest"])
    assert _host_checks(vals) == (r["count"], r["sum"], r["xor"], r["largest"])
    assert bool(np.all(vals[1:] > vals[:-1]))
    s.close()


def test_config2_host_values_match_golden(sieve, golden):
    rec = [p for p in golden["prefixes"] if p["limit"] == 10**10 - 1][0]
    out = np.empty(455_052_511 + 64, np.uint64)
    for off in (0, 3):  # output alignment inside a cache line
        o = out[off:]
        _, n, c = sieve.enumerate_range(0, 10**10, out=o)
        assert n == rec["count"]
        assert _host_checks(o[:n]) == (rec["count"], rec["sum"], rec["xor"], rec["largest"])
        assert int(o[0]) == 2 and int(o[1]) == 3 and int(o[2]) == 5


def test_truncating_capacity(sieve, port):
    L, W = 10**13, 3 * 10**8
    full, n, _ = sieve.enumerate_range(L, L + W)
    for cap in (1, n // 3 + 1, n - 1):
        out = np.full(cap + 8, 7, np.uint64)
        with pytest.raises(ws.Error) as ei:
            sieve.enumerate_range(L, L + W, out=out[:cap])
        assert ei.value.code == ws.Errc.Capacity
        assert np.array_equal(out[:cap], full[:cap])
        assert bool(np.all(out[cap:] == 7))  # nothing past cap


def test_wire_equals_u64_path(port):
    L, W = 123_456_789_012, 5 * 10**8
    os.environ["WHEELSIEVE_HOST_WIRE"] = "0"
    try:
        plain = ws.Sieve()
    finally:
        del os.environ["WHEELSIEVE_HOST_WIRE"]
    wire = ws.Sieve()
    a, na, ca = plain.enumerate_range(L, L + W)
    b, nb, cb = wire.enumerate_range(L, L + W)
    assert na == nb and np.array_equal(a, b)
    assert (ca.count, ca.sum, ca.xor, ca.largest) == (cb.count, cb.sum, cb.xor, cb.largest)
    plain.close()
    wire.close()
