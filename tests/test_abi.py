"""CPU: the C-ABI library loads, exports every symbol include/wheelsieve/gpu.h
declares, and its host-only helpers agree with the oracle.  No compute call
is made without a GPU (context creation must fail loudly instead)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "wheelsieve", "gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ws_[a-z_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2310_17746_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_sm100a_only_cubin():
    import subprocess
    so = os.path.join(ROOT, "paper_2310_17746_b200", "libwheelsieve_cuda.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_device_fails_loudly():
    import torch
    import paper_2310_17746_b200 as ws
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ws.Error) as e:
        ws.Sieve()
    assert e.value.code == ws.Errc.NoDevice


def test_isqrt_and_table1(port):
    import paper_2310_17746_b200 as ws
    for n in [0, 1, 24, 25, 26, 10**12, 2**64 - 1, 2**63 + 12345]:
        assert ws.isqrt(n) == port.isqrt(n)
    for p in [5, 7, 11, 13, 101, 997, 10007, 65521]:
        for start in [p // 6 * 6 + 6, 14400 // 6 * 6 * 7, 6 * 10**9, 6 * 123457]:
            if start <= p:
                continue
            assert ws.start_offsets(p, start) == port.start_offsets(p, start)
    with pytest.raises(ws.Error) as e:
        ws.start_offsets(9, 60)
    assert e.value.code == ws.Errc.Domain
    with pytest.raises(ws.Error) as e:
        ws.start_offsets(7, 61)
    assert e.value.code == ws.Errc.Alignment


@pytest.mark.parametrize("L,R,world", [(0, 10**12 + 1, 8), (10**15, 10**15 + 10**11, 8),
                                       (0, 1000, 4), (17, 6 * (1 << 18) * 5 + 3, 3),
                                       (5, 6, 2), (0, 10**9 + 1, 1)])
def test_partition_tiles_range(L, R, world):
    import paper_2310_17746_b200 as ws
    S = 1 << 18
    parts = [ws.partition(L, R, r, world, S) for r in range(world)]
    assert parts[0][0] == L and parts[-1][1] == R
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c
    lo0 = L // 6 * 6
    for a, b in parts[1:]:
        if L < a < R:
            assert (a - lo0) % (6 * S) == 0  # interior borders on segment borders
    nseg = ((R - lo0 + 5) // 6 + S - 1) // S
    sizes = [((b - a) + 6 * S - 1) // (6 * S) for a, b in parts]
    if nseg >= world:
        assert max(sizes) - min(sizes) <= 1


def test_prime_count_bound_is_upper_bound(golden):
    import paper_2310_17746_b200 as ws
    for rec in golden["windows"] + [dict(L=0, R=p["limit"] + 1, count=p["count"])
                                    for p in golden["prefixes"]]:
        assert ws.prime_count_bound(rec["L"], rec["R"]) >= rec["count"]


def test_wheel_coordinates():  # test_wheel.cpp:30-74
    import numpy as np
    import paper_2310_17746_b200 as ws
    assert ws.value_of(0, ws.R1) == 1 and ws.value_of(0, ws.R5) == 5
    assert ws.coord_of(25) == (4, 1) and ws.coord_of(35) == (5, 5)
    rng = np.random.default_rng(42)
    for _ in range(2000):
        k = int(rng.integers(0, ws.wheelsieve.K_MAX_WHEEL_INDEX))
        for r in (ws.R1, ws.R5):
            assert ws.coord_of(ws.value_of(k, r)) == (k, r)
    for bad in (0, 2, 3, 4, 6):
        with pytest.raises(ws.Error) as e:
            ws.coord_of(bad)
        assert e.value.code == ws.Errc.NotOnWheel
    with pytest.raises(ws.Error) as e:
        ws.value_of(ws.wheelsieve.K_MAX_WHEEL_INDEX + 1, ws.R1)
    assert e.value.code == ws.Errc.Overflow
    assert [ws.ceil_sqrt(n) for n in (0, 1, 2, 4, 5, 24, 25, 26)] == [0, 1, 2, 2, 3, 5, 5, 6]
