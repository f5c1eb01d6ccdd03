"""GPU: the chunked prime store -- byte-identical to the
reference's ChunkedFileSink output for the same range (reference library,
oracle/_ref, driven like its CLI: tools/wheelsieve.cpp:139-168), readable by
the reference's read_back/verify_store and vice versa, with the reference's
fault behaviour (test_sink.cpp)."""
import os

import numpy as np
import pytest

import paper_2310_17746_b200 as ws

pytestmark = pytest.mark.gpu


def _files(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


@pytest.mark.parametrize("limit,binary,ppf", [(97, False, 10), (97, True, 10), (2, True, 5),
                                              (30, False, 10), (1_000_000, True, 10_000),
                                              (1_000_000, False, 78_498),
                                              (10**8, True, 1_000_000)])
def test_store_byte_identical_to_reference(tmp_path, sieve, limit, binary, ppf):
    from oracle.oracle import Reference
    ref = Reference()
    ours, theirs = str(tmp_path / "gpu"), str(tmp_path / "ref")
    n = sieve.store_range(0, limit + 1, ours, binary=binary, primes_per_file=ppf)
    ref.store_run(limit, theirs, binary, ppf)
    a, b = _files(ours), _files(theirs)
    assert sorted(a) == sorted(b)
    for name in b:
        assert a[name] == b[name], name
    ws.verify_store(ours)
    assert ref.verify_store(ours) == 0
    lo, hi = limit // 3, limit // 2 + 1
    rc, vals = ref.read_back(ours, lo, hi)
    assert rc == 0
    assert np.array_equal(ws.read_back(theirs, lo, hi), vals)
    assert n == sum(int(x) for x in [len(ws.read_back(ours, 0, limit + 1))])


def test_store_window_and_faults(tmp_path, sieve, port):  # test_sink.cpp:153-278
    d = str(tmp_path / "w")
    L, R = 10**12, 10**12 + 2_000_003
    n = sieve.store_range(L, R, d, binary=True, primes_per_file=10_000)
    ref = port.range(L, R, values=True)["values"]
    assert n == ref.size and np.array_equal(ws.read_back(d, L, R), ref)
    assert np.array_equal(ws.read_back(d, L + 12345, L + 777_777),
                          ref[(ref >= L + 12345) & (ref < L + 777_777)])
    with pytest.raises(ws.Error) as e:
        ws.read_back(d, L, R + 1)
    assert e.value.code == ws.Errc.BeyondFrontier
    # corrupt one byte of the second chunk -> checksum mismatch on touch
    name = sorted(f for f in os.listdir(d) if f.endswith(".bin"))[1]
    p = os.path.join(d, name)
    raw = bytearray(open(p, "rb").read())
    raw[13] ^= 0x40
    open(p, "wb").write(bytes(raw))
    with pytest.raises(ws.Error) as e:
        ws.verify_store(d)
    assert e.value.code == ws.Errc.ChecksumMismatch
    # a range that avoids the corrupted file still reads
    first = sorted(f for f in os.listdir(d) if f.endswith(".bin"))[0]
    assert ws.read_back(d, L, L + 1000).size > 0
    os.remove(os.path.join(d, "manifest.json"))
    with pytest.raises(ws.Error) as e:
        ws.read_back(d, L, L + 10)
    assert e.value.code == ws.Errc.BadManifest
    with pytest.raises(ws.Error) as e:
        sieve.store_range(0, 100, str(tmp_path / "z"), primes_per_file=0)
    assert e.value.code == ws.Errc.Domain
    assert first
