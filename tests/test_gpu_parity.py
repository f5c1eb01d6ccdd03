"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference goldens.  Bar: bit-exact counts, per-segment counts, Σ mod 2^64, ⊕,
largest prime and enumerated values."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _tuple(c):
    return (c.count, c.sum, c.xor, c.largest)


def test_prefix_goldens(sieve, golden):
    for rec in golden["prefixes"]:
        c = sieve.count_range(0, rec["limit"] + 1, checks=True)
        assert _tuple(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec["limit"]
        c2 = sieve.count_range(0, rec["limit"] + 1)
        assert (c2.count, c2.largest) == (rec["count"], rec["largest"])


def test_window_goldens_per_segment(sieve, sieve12, golden):
    for rec in golden["windows"]:
        c, ps = sieve.count_range(rec["L"], rec["R"], checks=True, per_seg=True)
        assert _tuple(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec
        assert [int(x) for x in ps] == rec["seg18"], (rec["L"], rec["R"])
        if "seg12" in rec:
            c12, ps12 = sieve12.count_range(rec["L"], rec["R"], checks=True, per_seg=True)
            assert _tuple(c12) == _tuple(c)
            assert [int(x) for x in ps12] == rec["seg12"], (rec["L"], rec["R"])


def test_window_enumeration_goldens(sieve, golden, port):
    for rec in golden["windows"]:
        if rec["R"] - rec["L"] > 2 * 10**7:
            continue
        vals, n, c = sieve.enumerate_range(rec["L"], rec["R"])
        assert _tuple(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"])
        assert n == rec["count"]
        ref = port.range(rec["L"], rec["R"], values=True)["values"]
        assert np.array_equal(vals, ref), (rec["L"], rec["R"])


def test_config1_per_segment_golden(sieve):
    g = load_golden("c1_per_segment.json")
    c, ps = sieve.count_range(0, 10**9 + 1, per_seg=True)
    assert c.count == g["count"] == 50_847_534
    assert c.largest == g["largest"]
    assert [int(x) for x in ps] == g["seg18"]


def test_config2_enumeration_checksums(sieve, golden):
    rec = [p for p in golden["prefixes"] if p["limit"] == 10**10 - 1][0]
    import torch
    n_bound = 455_052_511 + 1024
    out = torch.empty(n_bound, dtype=torch.int64, device="cuda")
    _, n, c = sieve.enumerate_range(0, 10**10, out=out)
    assert _tuple(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"])
    v = out[:n]
    assert bool((v[1:] > v[:-1]).all())  # strictly ascending
    # the device array carries exactly the primes the checksums describe
    assert int(v[-1].item()) == rec["largest"] and int(v[0].item()) == 2
    host = v.cpu().numpy().view(np.uint64)
    assert int(host.sum(dtype=np.uint64)) == rec["sum"]
    assert int(np.bitwise_xor.reduce(host)) == rec["xor"]


def test_config3_pi_1e12(sieve):
    c = sieve.count_range(0, 10**12 + 1)
    assert c.count == 37_607_912_018  # SURVEY Appendix A (reference run(), 477 s @8T)
    assert c.largest == 999_999_999_989


def test_config5_intervals_golden(sieve):
    g = load_golden("c5_intervals.json")
    counts, sums, xors = sieve.count_intervals(np.array(g["L"], np.uint64), g["width"])
    assert [int(x) for x in counts] == g["counts"]
    assert [int(x) for x in sums] == g["sums"]
    assert [int(x) for x in xors] == g["xors"]


def test_c4_slice_golden(sieve, golden):
    rec = [w for w in golden["windows"] if (w["L"], w["R"]) == (10**15, 10**15 + 10**8)][0]
    c = sieve.count_range(rec["L"], rec["R"], checks=True)
    assert _tuple(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"])


def test_random_windows_vs_oracle(sieve, sieve12, port):
    rng = np.random.default_rng(1234)
    for i in range(60):
        kind = i % 4
        if kind == 0:
            L = int(rng.integers(0, 3000))
        elif kind == 1:
            L = int(rng.integers(0, 10**9))
        elif kind == 2:
            L = int(rng.integers(0, 10**14))
        else:
            L = int(rng.integers(10**15, 10**16 - 10**7))
        W = int(rng.integers(1, 4_000_000 if kind < 3 else 400_000))
        ref = port.range(L, L + W, seg_slots=1 << 12, per_seg=True, values=True)
        for sv in (sieve, sieve12):
            c, ps = sv.count_range(L, L + W, checks=True, per_seg=True)
            assert _tuple(c) == (ref["count"], ref["sum"], ref["xor"], ref["largest"]), (L, W)
            if sv is sieve12:
                assert [int(x) for x in ps] == [int(x) for x in ref["per_seg"]], (L, W)
        vals, n, c = sieve.enumerate_range(L, L + W)
        assert np.array_equal(vals, ref["values"]), (L, W)


def test_tiny_ranges_exhaustive(sieve, port):
    for L in range(0, 60):
        for R in range(L, 80):
            c = sieve.count_range(L, R, checks=True)
            r = port.range(L, R)
            assert _tuple(c) == (r["count"], r["sum"], r["xor"], r["largest"]), (L, R)


def test_base_table_growth_and_fresh(port):
    import paper_2310_17746_b200 as ws
    with ws.Sieve() as s:
        a = s.count_range(10**6, 10**6 + 10**5, checks=True)       # small base
        b = s.count_range(10**14, 10**14 + 10**6, checks=True)     # grows the table
        c = s.count_range(10**6, 10**6 + 10**5, checks=True)       # reuses the larger one
        d = s.count_range(10**6, 10**6 + 10**5, checks=True, fresh_base=True)
        assert _tuple(a) == _tuple(c) == _tuple(d)
        r = port.range(10**14, 10**14 + 10**6)
        assert _tuple(b) == (r["count"], r["sum"], r["xor"], r["largest"])


def test_errors(sieve):
    import paper_2310_17746_b200 as ws
    K = ws.wheelsieve.K_MAX_SEGMENT_END
    with pytest.raises(ws.Error) as e:
        sieve.count_range(0, K + 1)
    assert e.value.code == ws.Errc.Overflow
    assert sieve.count_range(100, 100).count == 0
    assert sieve.count_range(100, 50).count == 0
    out = np.zeros(3, np.uint64)
    with pytest.raises(ws.Error) as e:
        sieve.enumerate_range(0, 100, out=out)
    assert e.value.code == ws.Errc.Capacity
    assert list(out) == [2, 3, 5]
    with pytest.raises(ws.Error):
        ws.Sieve(segment_slots=1000)


def test_device_per_segment_and_timing(sieve):
    import torch
    nseg = sieve.num_segments(0, 10**9 + 1)
    ps = torch.zeros(nseg, dtype=torch.int32, device="cuda")
    c = sieve.count_range(0, 10**9 + 1, per_seg=ps)
    assert int(ps.sum().item()) + 2 == c.count
    t = sieve.timing()
    assert t.sieve_ms > 0 and t.segments == nseg and t.launches >= 1


def _run_isolated(code, env):
    """Run `code` in a fresh interpreter (the bucket knobs are read when a
    context is created)."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


BUCKET_CODE = r"""
import sys, json
sys.path.insert(0, '.')
import numpy as np
import paper_2310_17746_b200 as ws
from oracle.oracle import Port
port = Port()
s = ws.Sieve()
out = []
for L, R in [(10**15, 10**15 + 3 * 10**7), (2**43 - 10**6, 2**43 + 2**24), (10**12 - 7, 10**12 + 4 * 10**7 + 1)]:
    c, ps = s.count_range(L, R, checks=True, per_seg=True)
    r = port.range(L, R, per_seg=True)
    assert (c.count, c.sum, c.xor, c.largest) == (r["count"], r["sum"], r["xor"], r["largest"]), (L, R)
    assert np.array_equal(ps, r["per_seg"]), (L, R)
    v, n, ce = s.enumerate_range(L, R)
    assert n == r["count"] and ce.sum == r["sum"]
print("ok")
"""


@pytest.mark.parametrize("env", [{"WHEELSIEVE_BUCKET_BUDGET": str(1 << 20), "WHEELSIEVE_BUCKET_RATIO": "1"},
                                 {"WHEELSIEVE_BUCKET_CAP": "64", "WHEELSIEVE_BUCKET_RATIO": "1"},
                                 {"WHEELSIEVE_FILL_PIECE": "3", "WHEELSIEVE_BUCKET_RATIO": "1"},
                                 {}])
def test_bucket_windows_and_overflow(env):
    assert "ok" in _run_isolated(BUCKET_CODE, env)


def _is_prime_mr(n):
    """Deterministic Miller-Rabin for n < 3.3e24 (independent checker for
    ranges above the reference's 1e16 naive-sieve cap, wheel.hpp:40)."""
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@pytest.mark.parametrize("L,W", [(10**18, 40_000), (2**63 - 20_000, 40_000),
                                 (18446744073709551612 - 30_000, 30_000)])
def test_top_of_64bit_range_vs_miller_rabin(sieve, L, W):
    R = L + W
    vals, n, c = sieve.enumerate_range(L, R)
    expected = [v for v in range(L | 1, R, 2) if v % 3 and _is_prime_mr(v)]
    assert [int(x) for x in vals] == expected
    cc = sieve.count_range(L, R, checks=True)
    assert cc.count == len(expected) == n
    assert cc.sum == sum(expected) % 2**64 and cc.xor == c.xor
    assert cc.largest == (expected[-1] if expected else 0)


def test_sieve_segment_flag_words_match_reference():
    """ws_sieve_segment returns exactly the reference's FlagArray words after
    SegmentBitmap + sieve_segment (segment.cpp:93-188), golden from the
    reference library (tests/golden/reference_segments.json)."""
    import paper_2310_17746_b200 as ws
    from oracle.oracle import fnv1a64
    g = load_golden("reference_segments.json")
    for sv in (ws.Sieve(), ws.Sieve(segment_slots=1 << 12)):
        for rec in g["segments"]:
            r1, r5 = sv.sieve_segment(rec["start"], rec["len"])
            if rec["r1"] is not None:
                assert [int(x) for x in r1] == rec["r1"], (rec["start"], rec["len"])
                assert [int(x) for x in r5] == rec["r5"], (rec["start"], rec["len"])
            assert fnv1a64(r1.astype("<u8").tobytes()) == rec["fnv_r1"]
            assert fnv1a64(r5.astype("<u8").tobytes()) == rec["fnv_r5"]
        sv.close()


def test_sieve_segment_errors(sieve):
    import paper_2310_17746_b200 as ws
    for args, code in (((10, 5), ws.Errc.Alignment), ((12, 0), ws.Errc.Domain),
                       ((ws.wheelsieve.K_MAX_SEGMENT_END, 1), ws.Errc.Overflow)):
        with pytest.raises(ws.Error) as e:
            sieve.sieve_segment(*args)
        assert e.value.code == code  # test_segment.cpp:100-120


def test_base_primes_match_bootstrap(sieve):
    """ws_base_primes(B) == BasePrimeStore::bootstrap(hint).entries with
    B = ceil_sqrt(hint) (base_store.cpp:34-42)."""
    import paper_2310_17746_b200 as ws
    from oracle.oracle import fnv1a64
    g = load_golden("reference_segments.json")
    for rec in g["bootstrap"]:
        assert ws.ceil_sqrt(rec["hint"]) == rec["frontier"]
        e = sieve.base_primes(rec["frontier"])
        assert e.size == rec["n"] and [int(x) for x in e[:5]] == rec["first"]
        assert int(e[-1]) == rec["last"] and fnv1a64(e.astype("<u8").tobytes()) == rec["fnv"]
    assert sieve.base_primes(4).size == 0
    with pytest.raises(ws.Error) as e:
        sieve.base_primes(1)
    assert e.value.code == ws.Errc.EmptyRange


@pytest.mark.parametrize("B", [53, 54, 1000, 31623, 2**18 - 1, 2**18, 2**18 + 1, 10**6])
def test_base_table_one_block_and_two_level_builds(B, port):
    """Fresh table builds either side of the one-block bound (kTinyMax = 2^18)
    against a numpy sieve, and a prime count that uses each table."""
    import paper_2310_17746_b200 as ws
    comp = np.zeros(B + 1, dtype=bool)
    comp[:2] = True
    for q in range(2, int(B**0.5) + 1):
        if not comp[q]:
            comp[q * q::q] = True
    want = np.nonzero(~comp)[0]
    want = want[want >= 5]
    s = ws.Sieve()
    try:
        got = s.base_primes(B)
        assert got.size == want.size and np.array_equal(got.astype(np.int64), want)
    finally:
        s.close()
    # a window whose base bound is about B: [B^2 - 10^6, B^2)
    R = B * B
    L = max(0, R - 10**6)
    s = ws.Sieve()
    try:
        c = s.count_range(L, R, checks=True)
    finally:
        s.close()
    o = port.range(L, R)
    assert (c.count, c.sum, c.xor, c.largest) == (o["count"], o["sum"], o["xor"], o["largest"])


def test_repeated_fresh_base_with_buckets():
    """Regression: repeated WS_FRESH_BASE calls on a bucketed range (the base
    sieve and the main launch stage their uploads through pinned memory)."""
    import paper_2310_17746_b200 as ws
    g = load_golden("reference_goldens.json")
    rec = [w for w in g["windows"] if (w["L"], w["R"]) == (10**15, 10**15 + 10**8)][0]
    with ws.Sieve() as s:
        for _ in range(4):
            c = s.count_range(rec["L"], rec["R"], checks=True, fresh_base=True)
            assert (c.count, c.sum, c.xor) == (rec["count"], rec["sum"], rec["xor"])
        for _ in range(2):
            v, n, c = s.enumerate_range(rec["L"], rec["R"], fresh_base=True)
            assert (n, c.sum, c.xor) == (rec["count"], rec["sum"], rec["xor"])


def test_config4_full_window_reference_golden(sieve):
    """[1e15, 1e15 + 1e11): count, sum, xor, largest from the reference
    library's --big golden run (oracle/gen_golden.py --big, 262 s on 8 threads)."""
    big = load_golden("reference_big.json")["c4"]
    for fresh in (False, True):
        c = sieve.count_range(big["L"], big["R"], checks=True, fresh_base=fresh)
        assert (c.count, c.sum, c.xor, c.largest) == (big["count"], big["sum"], big["xor"],
                                                      big["largest"])


def test_config4_full_window_enumeration():
    """Config 4 "count and enumerate": all 2,895,317,534 primes of
    [1e15, 1e15 + 1e11) enumerated into HBM (23.2 GB), ascending, with the
    reference's count / sum / xor / largest."""
    import torch

    import paper_2310_17746_b200 as ws
    r = load_golden("reference_big.json")["c4"]
    L, R = 10**15, 10**15 + 10**11
    s = ws.Sieve()
    out = torch.empty(r["count"] + 64, dtype=torch.int64, device="cuda")
    _, n, c = s.enumerate_range(L, R, out=out)
    assert (n, c.sum, c.xor, c.largest) == (r["count"], r["sum"], r["xor"], r["largest"])
    v = out[:n]
    assert bool((v[1:] > v[:-1]).all())
    assert int(v[0]) > L and int(v[-1]) == r["largest"]
    # the array itself carries the checksums (int64 wrap = mod 2^64)
    assert int(v.sum()) % 2**64 == r["sum"]
    s.close()
    del out


@pytest.mark.parametrize("N,pi", [(2**32, 203_280_221), (2**40, 41_203_088_796),
                                  (10**13, 346_065_536_839), (10**14, 3_204_941_750_802)])
def test_published_prime_counts(sieve, N, pi):
    """Beyond the reference goldens (which stop at 1e12): standard published
    values of pi(x) (e.g. OEIS A006880 / A007053), up to 1e14."""
    assert sieve.count_range(0, N + 1).count == pi


EXTEND_CODE = r"""
import sys, json
sys.path.insert(0, ".")
import numpy as np
import paper_2310_17746_b200 as ws
s = ws.Sieve()
out = []
# bounds grow 1e3 -> 1e5 -> 1e6 -> 3.2e7: each call extends the resident table
for L, R in [(0, 10**6), (0, 10**10), (10**12 - 10**8, 10**12 + 10**8),
             (10**15, 10**15 + 3 * 10**8), (2**40, 2**40 + 10**8)]:
    c = s.count_range(L, R, checks=True)
    v, n, ce = s.enumerate_range(L, min(R, L + 10**8))
    out.append([c.count, c.sum, c.xor, c.largest, n, ce.sum, int(v[-1])])
print(json.dumps(out))
"""


def test_base_extension_matches_rebuild():
    """Device-side BasePrimeStore::extend (the table grows by sieving only the
    new range) gives exactly the results of rebuilding the table each time."""
    import json
    a = json.loads(_run_isolated(EXTEND_CODE, {"WHEELSIEVE_BASE_EXTEND": "1"}).strip().splitlines()[-1])
    b = json.loads(_run_isolated(EXTEND_CODE, {"WHEELSIEVE_BASE_EXTEND": "0"}).strip().splitlines()[-1])
    assert a == b
    assert a[1][0] == 455_052_511  # pi(1e10 - 1)
