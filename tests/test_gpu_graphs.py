"""CUDA-graph replay of repeated small count calls (ws_abi.cu, graph_or_run).

The second identical small count call is captured into a graph and later ones
replay it.  Every replay must give the reference's results (count, largest,
per-segment counts), keep the timing counters meaningful, and a changed
input, buffer or resident table must never replay a stale graph."""
import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu

C1 = load_golden("c1_per_segment.json")
PI_1E9 = 50_847_534


def _c1_calls(sv, k, per_seg, fresh):
    for _ in range(k):
        if isinstance(per_seg, np.ndarray):
            per_seg[:] = 0
        else:
            per_seg.zero_()
        c = sv.count_range(0, 10**9 + 1, per_seg=per_seg, fresh_base=fresh)
        got = per_seg.cpu().numpy() if torch.is_tensor(per_seg) else per_seg
        assert c.count == PI_1E9 and c.largest == C1["largest"]
        assert [int(x) for x in got.astype(np.uint32)] == C1["seg18"]
        t = sv.timing()
        assert t.sieve_ms > 0 and t.segments == len(C1["seg18"]) and t.launches >= 1


@pytest.mark.parametrize("multi", [False, True])
@pytest.mark.parametrize("fresh", [True, False])
def test_replayed_c1_matches_golden(multi, fresh):
    import paper_2310_17746_b200 as ws
    sv = ws.Sieve(devices=[0]) if multi else ws.Sieve(device=0)
    try:
        dev = torch.zeros(len(C1["seg18"]), dtype=torch.int32, device="cuda")
        host = np.zeros(len(C1["seg18"]), np.uint32)
        _c1_calls(sv, 5, dev, fresh)   # run, capture, replay x3
        _c1_calls(sv, 4, host, fresh)  # host output: the direct path
        _c1_calls(sv, 3, dev, fresh)
    finally:
        sv.close()


def test_interleaved_keys_and_reallocation(golden):
    import paper_2310_17746_b200 as ws
    sv = ws.Sieve(device=0)
    try:
        recs = [r for r in golden["windows"] if r["R"] - r["L"] < 10**8][:4]
        ps = torch.zeros(len(C1["seg18"]), dtype=torch.int32, device="cuda")
        for rnd in range(4):
            for rec in recs:  # each window's call repeats, interleaved with others
                for _ in range(2):
                    c, seg = sv.count_range(rec["L"], rec["R"], per_seg=True, fresh_base=True)
                    assert c.count == rec["count"] and c.largest == rec["largest"]
                    assert [int(x) for x in seg] == rec["seg18"]
            c = sv.count_range(0, 10**9 + 1, per_seg=ps, fresh_base=True)
            assert c.count == PI_1E9
            assert [int(x) for x in ps.cpu().numpy().astype(np.uint32)] == C1["seg18"]
            if rnd == 1:  # a large call reallocates buffers: graphs must not replay stale pointers
                big = sv.count_range(10**15, 10**15 + 10**9, checks=True)
                assert big.count > 0
    finally:
        sv.close()


def test_graphs_off_is_the_same_path(monkeypatch):
    import paper_2310_17746_b200 as ws
    monkeypatch.setenv("WHEELSIEVE_GRAPHS", "0")
    sv = ws.Sieve(device=0)
    try:
        dev = torch.zeros(len(C1["seg18"]), dtype=torch.int32, device="cuda")
        _c1_calls(sv, 3, dev, True)
    finally:
        sv.close()
