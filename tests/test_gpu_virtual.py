"""GPU: the multi-device path with N > 1 shards, run as N "virtual devices"
on the one reachable GPU (WHEELSIEVE_VIRTUAL_SHARDS=1: duplicate device ids
allowed, one DevCtx + worker thread per shard, the 32-byte shard records
gathered through the host instead of by NCCL, which refuses two ranks on one
device).  Everything else -- ws_partition shards, per-segment offsets,
interval i -> shard i mod N, contiguous range blocks, the enumeration count
pass + offsets, ws_enumerate_shards, the combine -- is the code an N-GPU
context runs, checked here bit-exact against the reference goldens."""
import os

import numpy as np
import pytest

import paper_2310_17746_b200 as ws
from conftest import load_golden

pytestmark = pytest.mark.gpu


def _t(c):
    return (c.count, c.sum, c.xor, c.largest)


@pytest.fixture(scope="module", params=[2, 3, 8])
def virt(request):
    import torch
    d = torch.cuda.current_device()
    old = {k: os.environ.get(k) for k in ("WHEELSIEVE_VIRTUAL_SHARDS", "WHEELSIEVE_BUCKET_BUDGET")}
    os.environ["WHEELSIEVE_VIRTUAL_SHARDS"] = "1"
    os.environ["WHEELSIEVE_BUCKET_BUDGET"] = str(1 << 30)  # N contexts share the GPU's memory
    s = ws.Sieve(devices=[d] * request.param)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    yield s
    s.close()


def test_virtual_context_shape(virt):
    n = virt.num_shards
    assert virt.num_devices == n and n > 1
    assert [virt.comm_info(i) for i in range(n)] == [(n, i) for i in range(n)]


def test_sharded_counts_match_goldens(virt, golden):
    for rec in golden["prefixes"]:
        c = virt.count_range(0, rec["limit"] + 1, checks=True)
        assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec["limit"]
    for rec in golden["windows"]:  # many have fewer segments than shards: empty shards
        c, ps = virt.count_range(rec["L"], rec["R"], checks=True, per_seg=True)
        assert _t(c) == (rec["count"], rec["sum"], rec["xor"], rec["largest"]), rec
        assert [int(x) for x in ps] == rec["seg18"], (rec["L"], rec["R"])


def test_sharded_c1_c3(virt):
    g = load_golden("c1_per_segment.json")
    c, ps = virt.count_range(0, 10**9 + 1, per_seg=True)
    assert (c.count, c.largest) == (g["count"], g["largest"])
    assert [int(x) for x in ps] == g["seg18"]
    c3 = virt.count_range(0, 10**12 + 1)
    assert (c3.count, c3.largest) == (37_607_912_018, 999_999_999_989)


def test_sharded_bucket_window(virt, sieve):
    L, R = 10**15, 10**15 + 2 * 10**10  # bucket windows on every shard
    assert _t(virt.count_range(L, R, checks=True)) == _t(sieve.count_range(L, R, checks=True))


def test_sharded_intervals_c5(virt):
    g = load_golden("c5_intervals.json")
    counts, sums, xors = virt.count_intervals(np.array(g["L"], np.uint64), g["width"])
    assert [int(x) for x in counts] == g["counts"]
    assert [int(x) for x in sums] == g["sums"]
    assert [int(x) for x in xors] == g["xors"]


def test_sharded_count_ranges(virt, port):
    rng = np.random.default_rng(11)
    Ls, Rs = [0, 3, 100], [2, 10**6, 50]
    for _ in range(37):
        a = int(rng.integers(0, 2**45))
        Ls.append(a)
        Rs.append(a + int(rng.integers(0, 2 * 10**6)))
    for L, R, c in zip(Ls, Rs, virt.count_ranges(Ls, Rs, checks=True)):
        if R <= L:
            assert _t(c) == (0, 0, 0, 0)
            continue
        r = port.range(L, R)
        assert _t(c) == (r["count"], r["sum"], r["xor"], r["largest"]), (L, R)


def test_sharded_enumeration(virt, port, golden):
    import torch
    for L, R in [(0, 3 * 10**7), (10**13 - 12_345_677, 10**13 + 27_654_321), (2, 4), (5, 100)]:
        ref = port.range(L, R, values=True)
        vals, n, c = virt.enumerate_range(L, R)  # count pass, offsets, per-shard pipelines
        assert n == ref["count"] and np.array_equal(vals, ref["values"]), (L, R)
        assert _t(c) == (ref["count"], ref["sum"], ref["xor"], ref["largest"])
        dev = torch.zeros(n + 8, dtype=torch.int64, device="cuda")
        _, n2, _ = virt.enumerate_range(L, R, out=dev)
        assert n2 == n and np.array_equal(dev[:n].cpu().numpy().view(np.uint64), ref["values"])
    with pytest.raises(ws.Error) as e:
        virt.enumerate_range(0, 3 * 10**7, out=np.zeros(1000, np.uint64))
    assert e.value.code == ws.Errc.Capacity
    # c2 with every shard's primes left in its own buffer
    rec = [p for p in golden["prefixes"] if p["limit"] == 10**10 - 1][0]
    outs = []
    for k in range(virt.num_shards):
        lo, hi = ws.partition(0, 10**10, k, virt.num_shards)
        outs.append(torch.empty(ws.prime_count_bound(lo, hi) + 2, dtype=torch.int64, device="cuda"))
    counts, c = virt.enumerate_shards(0, 10**10, outs)
    assert sum(counts) == rec["count"] and _t(c) == (rec["count"], rec["sum"], rec["xor"],
                                                      rec["largest"])
    allv = np.concatenate([o[:k].cpu().numpy().view(np.uint64) for o, k in zip(outs, counts)])
    assert bool(np.all(allv[1:] > allv[:-1])) and int(allv[0]) == 2
    assert int(allv.sum(dtype=np.uint64)) == rec["sum"]


def test_sharded_run_emission(virt, port):
    """run() on a multi-shard context: per-tile batches identical to one device."""
    class Rec(ws.CountSink):
        def __init__(self):
            super().__init__()
            self.b = []

        def emit_count(self, n, largest):
            super().emit_count(n, largest)
            self.b.append((n, largest))

    a, b = Rec(), Rec()
    ws.run(ws.SieveConfig(10**7, 3, ws.round_segment_span(600_000, 3), 0, a), sieve=virt)
    ws.run(ws.SieveConfig(10**7, 3, ws.round_segment_span(600_000, 3), 0, b))
    assert a.b == b.b and a.count() == 664_579
