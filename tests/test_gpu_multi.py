"""GPU: the multi-device path (ws_opts.n_devices >= 1: NCCL communicators,
ws_partition shards, one ncclAllGather of the shard records) against the
reference goldens, and the N-way shard decomposition of the multi-GPU configs.

Only one GPU is reachable here, so N > 1 is exercised the way the library
composes it: the N ws_partition shares (C3, C4) or the i mod N interval
subsets (C5) are sieved one after another on the device and folded with
ws_combine_checks -- the same fold the library applies to the records its
allgather returns.  The NCCL path itself runs with n_devices = 1 (a real
communicator of one rank): the collective, the record layout and the fold
are the ones an 8-GPU context uses."""
import numpy as np
import pytest

import paper_2310_17746_b200 as ws
from conftest import load_golden

pytestmark = pytest.mark.gpu

S = 1 << 18


def _t(c):
    return (c.count, c.sum, c.xor, c.largest)


@pytest.fixture(scope="module")
def multi():
    import torch
    s = ws.Sieve(devices=[torch.cuda.current_device()])
    yield s
    s.close()


@pytest.fixture(scope="module")
def big():
    return load_golden("reference_big.json")


def test_nccl_context_shape(multi):
    assert multi.num_devices == 1 and multi.num_shards == 1
    assert multi.comm_info(0) == (1, 0)  # a real NCCL communicator: 1 rank, rank 0


def test_nccl_path_prefix_and_window_goldens(multi, golden):
    for rec in golden["prefixes"]:
        c = multi.count_range(0, rec["limit"] + 1, checks=True)
        assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec["limit"]
    for rec in golden["windows"]:
        c, ps = multi.count_range(rec["L"], rec["R"], checks=True, per_seg=True)
        assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"])
        assert [int(x) for x in ps] == rec["seg18"]


def test_nccl_path_c1_c3(multi):
    g = load_golden("c1_per_segment.json")
    c, ps = multi.count_range(0, 10**9 + 1, per_seg=True)
    assert (c.count, c.largest) == (g["count"], g["largest"])
    assert [int(x) for x in ps] == g["seg18"]
    c3 = multi.count_range(0, 10**12 + 1)
    assert (c3.count, c3.largest) == (37_607_912_018, 999_999_999_989)
    t = multi.timing()
    assert t.sieve_ms > 0 and multi.device_timing(0).sieve_ms == pytest.approx(t.sieve_ms)


def test_nccl_path_c4_window(multi, big):
    r = big["c4"]
    c = multi.count_range(r["L"], r["R"], checks=True)
    assert _t(c) == (r["count"], r["sum"], r["xor"], r["largest"])


def test_nccl_path_c5_intervals(multi):
    g = load_golden("c5_intervals.json")
    counts, sums, xors = multi.count_intervals(np.array(g["L"], np.uint64), g["width"])
    assert [int(x) for x in counts] == g["counts"]
    assert [int(x) for x in sums] == g["sums"]
    assert [int(x) for x in xors] == g["xors"]


def test_nccl_path_enumeration(multi, golden, port):
    import torch
    rec = [p for p in golden["prefixes"] if p["limit"] == 10**10 - 1][0]
    out = torch.empty(455_052_511 + 1024, dtype=torch.int64, device="cuda")
    counts, c = multi.enumerate_shards(0, 10**10, [out])
    assert counts == [rec["count"]]
    assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"])
    host = out[: counts[0]].cpu().numpy().view(np.uint64)
    assert int(host.sum(dtype=np.uint64)) == rec["sum"]
    assert int(np.bitwise_xor.reduce(host)) == rec["xor"]
    # host and device output through ws_enumerate_range's multi-device path
    L, R = 10**13 - 12_345_677, 10**13 + 7_654_321
    ref = port.range(L, R, values=True)
    vals, n, ce = multi.enumerate_range(L, R)
    assert n == ref["count"] and np.array_equal(vals, ref["values"])
    dev = torch.zeros(n + 8, dtype=torch.int64, device="cuda")
    _, n2, _ = multi.enumerate_range(L, R, out=dev)
    assert n2 == n and np.array_equal(dev[:n].cpu().numpy().view(np.uint64), ref["values"])
    with pytest.raises(ws.Error) as e:  # capacity below the count
        multi.enumerate_range(L, R, out=np.zeros(n - 1, np.uint64))
    assert e.value.code == ws.Errc.Capacity


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c3_shards_combine(sieve, world):
    """BASELINE config 3 at 2/4/8 GPUs: the ws_partition shares of [0, 1e12],
    each counted alone, folded by ws_combine_checks."""
    L, R = 0, 10**12 + 1
    recs = []
    for r in range(world):
        lo, hi = ws.partition(L, R, r, world, S)
        recs.append(sieve.count_range(lo, hi, checks=True))
    c = ws.combine_checks(recs)
    assert (c.count, c.largest) == (37_607_912_018, 999_999_999_989)
    assert c == sieve.count_range(L, R, checks=True)


@pytest.mark.parametrize("world", [2, 8])
def test_c4_shards_combine(sieve, big, world):
    r = big["c4"]
    recs = [sieve.count_range(*ws.partition(r["L"], r["R"], k, world, S), checks=True)
            for k in range(world)]
    assert _t(ws.combine_checks(recs)) == (r["count"], r["sum"], r["xor"], r["largest"])


def test_c1_shards_per_segment(sieve):
    """Per-segment counts of 8 shards concatenate to the unsharded golden."""
    g = load_golden("c1_per_segment.json")
    parts = []
    for k in range(8):
        lo, hi = ws.partition(0, 10**9 + 1, k, 8, S)
        _, ps = sieve.count_range(lo, hi, per_seg=True)
        parts.extend(int(x) for x in ps)
    assert parts == g["seg18"]


def test_c5_interval_subsets(sieve):
    """Config 5 on 8 GPUs: interval i on GPU i mod 8; the per-GPU subsets
    reassemble to the golden arrays and the totals fold like the library's."""
    g = load_golden("c5_intervals.json")
    Ls = np.array(g["L"], np.uint64)
    counts = np.zeros(Ls.size, np.uint32)
    sums = np.zeros(Ls.size, np.uint64)
    xors = np.zeros(Ls.size, np.uint64)
    recs = []
    for k in range(8):
        c, s, x = sieve.count_intervals(Ls[k::8], g["width"])
        counts[k::8], sums[k::8], xors[k::8] = c, s, x
        recs.append(ws.Checks(int(c.astype(np.uint64).sum()), int(s.sum(dtype=np.uint64)),
                              int(np.bitwise_xor.reduce(x)), 0))
    assert [int(x) for x in counts] == g["counts"]
    assert [int(x) for x in sums] == g["sums"]
    t = ws.combine_checks(recs)
    assert (t.count, t.sum, t.xor) == (g["total_count"], g["total_sum"], g["total_xor"])


def test_count_ranges_matches_oracle(multi, sieve, port):
    rng = np.random.default_rng(7)
    Ls, Rs = [0, 1, 2, 3, 4, 5, 10**6, 2**40, 10**15], [10, 2, 3, 4, 5, 6, 10**6 + 3, 2**40 + 10**7,
                                                        10**15 + 10**6]
    for _ in range(40):
        a = int(rng.integers(0, 2**50))
        Ls.append(a)
        Rs.append(a + int(rng.integers(0, 3 * 10**6)))
    Ls.append(50)
    Rs.append(40)  # empty
    for sv in (sieve, multi):
        res = sv.count_ranges(Ls, Rs, checks=True)
        for L, R, c in zip(Ls, Rs, res):
            if R <= L:
                assert _t(c) == (0, 0, 0, 0)
                continue
            r = port.range(L, R)
            assert _t(c) == (r["count"], r["sum"], r["xor"], r["largest"]), (L, R)


def test_duplicate_devices_rejected():
    import torch
    d = torch.cuda.current_device()
    with pytest.raises(ws.Error) as e:
        ws.Sieve(devices=[d, d])
    assert e.value.code == ws.Errc.BadConfig


def test_multiprocess_init_path_one_rank():
    """The communicator path of a multi-process job (an id from
    ws_nccl_unique_id, ncclCommInitRank inside an NCCL group), as one rank."""
    import torch
    nid = ws.nccl_unique_id()
    assert len(nid) == 128 and any(nid)
    with ws.Sieve(devices=[torch.cuda.current_device()], world=1, rank=0, nccl_id=nid) as s:
        assert s.comm_info(0) == (1, 0) and s.num_shards == 1
        c = s.count_range(0, 10**9 + 1, checks=True)
        assert (c.count, c.largest) == (50_847_534, 999_999_937)
        counts, sums, _ = s.count_intervals(np.array([2**40, 2**41], np.uint64), 10**6)
        assert counts.tolist() == [s.count_range(2**40, 2**40 + 10**6).count,
                                   s.count_range(2**41, 2**41 + 10**6).count]


def test_bad_multi_configs():
    with pytest.raises(ws.Error) as e:
        ws.Sieve(devices=[0], world=2, rank=0)  # no NCCL id
    assert e.value.code == ws.Errc.BadConfig
    with pytest.raises(ws.Error) as e:
        ws.Sieve(devices=[0], world=2, rank=2, nccl_id=bytes(128))  # rank >= world
    assert e.value.code == ws.Errc.BadConfig
