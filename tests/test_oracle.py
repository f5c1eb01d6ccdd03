"""CPU: pin the oracle.  The plain-C restatement (oracle/ws_oracle.c) must
agree with (a) the known answers in the reference's own tests, (b) the golden
vectors produced by running the reference (tests/golden/), and (c) the
reference library itself where it is built (oracle/_ref)."""
import os

import numpy as np
import pytest

from conftest import load_golden

# Known answers copied from the reference's own test suite (file:line).
KNOWN_PI = [
    (30, 10, None),            # test_cli.cpp:75
    (100, 25, None),           # test_wheel.cpp:101-104
    (1000, 168, None),         # test_cli.cpp:198
    (10_000, 1229, None),      # test_wheel.cpp:112
    (5999, 783, 5987),         # test_engine.cpp:258-259
    (100_000, 9592, 99991),    # test_cli.cpp:171
    (123_456, 11601, 123_449), # test_engine.cpp:179-180
    (1_000_000, 78498, 999_983),  # test_engine.cpp:139-140
    (10_000_000, 664_579, None),  # acceptance.cpp:214
]


@pytest.mark.parametrize("n,count,largest", KNOWN_PI)
def test_port_known_pi(port, n, count, largest):
    r = port.range(0, n + 1)
    assert r["count"] == count
    if largest is not None:
        assert r["largest"] == largest


def test_port_pi_1e8(port):
    assert port.range(0, 10**8 + 1)["count"] == 5_761_455  # acceptance.cpp:312


def test_port_100000th_prime(port):
    v = port.range(0, 1_300_000, values=True)["values"]
    assert int(v[99_999]) == 1_299_709  # acceptance.cpp:374


def test_port_segment_slices(port):
    # test_segment.cpp:135-173
    v = set(int(x) for x in port.range(12_000, 18_000, values=True)["values"])
    assert 14443 not in v and 14417 not in v and 12007 in v and max(v) == 17989
    assert port.range(10_200, 10_206)["count"] == 0  # 10201 = 101^2, 10205 composite
    v = port.range(168, 174, values=True)["values"]
    assert list(v) == [173]
    naive = port.naive_sieve(6000)
    assert list(port.range(0, 6000, values=True)["values"]) == list(naive)


def test_port_table1(port, golden):
    for rec in golden["start_offsets"]:
        assert port.start_offsets(rec["p"], rec["start"]) == (rec["id1"], rec["id5"])
    assert port.start_offsets(13, 14400) == (2407, 2402)  # acceptance.cpp:181-201


def test_port_table1_bruteforce(port):
    # acceptance.cpp:138-177 (reduced): brute-force smallest multiple per class
    rng = np.random.default_rng(20260816)
    for p in [int(x) for x in port.naive_sieve(600) if x >= 5]:
        for _ in range(20):
            start = 6 * int(rng.integers(p // 6 + 1, 166_666))
            i1, i5 = port.start_offsets(p, start)
            for res, idx in ((1, i1), (5, i5)):
                q = (start + p - 1) // p * p
                while q % 6 != res:
                    q += p
                assert 6 * idx + res == q


def test_port_isqrt(port):
    for n in [0, 1, 2, 3, 4, 15, 16, 17, 10**12, 2**52 - 1, 2**62, 2**64 - 1]:
        r = port.isqrt(n)
        assert r * r <= n < (r + 1) ** 2
    assert port.isqrt(2**64 - 1) == 4294967295  # test_wheel.cpp:76-99


def test_port_prefix_goldens(port, golden):
    for rec in golden["prefixes"]:
        if rec["limit"] > 10**8:
            continue
        r = port.range(0, rec["limit"] + 1)
        assert (r["count"], r["sum"], r["xor"], r["largest"]) == (
            rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec["limit"]


def test_port_window_goldens(port, golden):
    for rec in golden["windows"]:
        if rec["R"] - rec["L"] > 2 * 10**7:
            continue
        r = port.range(rec["L"], rec["R"], per_seg=True)
        assert (r["count"], r["sum"], r["xor"], r["largest"]) == (
            rec["count"], rec["sum"], rec["xor"], rec["largest"]), (rec["L"], rec["R"])
        assert list(r["per_seg"]) == rec["seg18"]
        if "seg12" in rec:
            r12 = port.range(rec["L"], rec["R"], seg_slots=1 << 12, per_seg=True)
            assert list(r12["per_seg"]) == rec["seg12"]


def test_port_c5_subset(port):
    g = load_golden("c5_intervals.json")
    Ls = port.splitmix_starts(g["seed"], g["n"], g["lo"], g["hi"])
    assert [int(x) for x in Ls] == g["L"]
    idx = [0, 1, 2, 4095]
    counts, sums, xors = port.intervals(Ls[idx], g["width"])
    assert [int(x) for x in counts] == [g["counts"][i] for i in idx]
    assert [int(x) for x in sums] == [g["sums"][i] for i in idx]
    assert [int(x) for x in xors] == [g["xors"][i] for i in idx]


def test_golden_consistency():
    c1 = load_golden("c1_per_segment.json")
    assert len(c1["seg18"]) == 636 and sum(c1["seg18"]) + 2 == c1["count"] == 50_847_534
    assert c1["seg18"][:3] == [119_266, 107_281, 103_628] and c1["seg18"][-1] == 59_150
    g = load_golden("c5_intervals.json")
    assert g["L"][0] == 378_761_080_469 and g["counts"][0] == 628_905
    assert sum(g["counts"]) == g["total_count"] == 2_331_645_558


REF_SO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "oracle", "_ref", "libwsref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built")
def test_port_matches_reference_random_windows(port):
    from oracle.oracle import Reference
    ref = Reference()
    rng = np.random.default_rng(7)
    for _ in range(40):
        L = int(rng.integers(0, 10**13))
        if rng.random() < 0.3:
            L = int(rng.integers(0, 10**6))
        W = int(rng.integers(1, 300_000))
        a = port.range(L, L + W, seg_slots=1 << 12, per_seg=True)
        b = ref.range(L, L + W, 1, 1 << 12, per_seg=True)
        assert (a["count"], a["sum"], a["xor"], a["largest"]) == (
            b["count"], b["sum"], b["xor"], b["largest"])
        assert list(a["per_seg"]) == list(b["per_seg"])


def test_scale_goldens_consistent(golden):
    """The weak-scaling c2 goldens (reference run() over [0, N*1e10)) extend
    the config-2 golden: counts grow, and pi(2e10) is the published value."""
    from conftest import load_golden
    g = load_golden("reference_scale.json")["c2_weak"]
    c2 = [p for p in golden["prefixes"] if p["limit"] == 10**10 - 1][0]
    counts = [c2["count"]] + [r["count"] for r in sorted(g, key=lambda r: r["gpus"])]
    assert counts == sorted(counts) and len(set(counts)) == 4
    assert g[0]["gpus"] == 2 and g[0]["count"] == 882_206_716
