"""CPU: the streaming chunk writer (ws_store_*, the engine behind
wheelsieve::ChunkedFileSink and ws_store_range) writes files byte-identical
to the reference's ChunkedFileSink (oracle/_ref: the reference library's own
sink driven by its CLI's recipe), for batches of every size, including the
parallel text encoding of large batches.  No GPU: the values come from the
oracle and are appended through the C ABI."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2310_17746_b200 import _lib

lib = _lib.lib


def _files(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))}


def _write(d, values, binary, ppf, batches, frontier):
    st = C.c_void_p()
    assert lib.ws_store_open(str(d).encode(), 1 if binary else 0, ppf, C.byref(st)) == 0
    cuts = np.linspace(0, values.size, batches + 1).astype(np.int64)
    for a, b in zip(cuts, cuts[1:]):
        part = np.ascontiguousarray(values[a:b])
        assert lib.ws_store_append(st, part.ctypes.data, part.size) == 0
    assert lib.ws_store_set_frontier(st, frontier) == 0
    assert lib.ws_store_close(st) == 0


@pytest.mark.parametrize("limit,binary,ppf,batches", [
    (97, False, 10, 3), (1_000_000, True, 10_000, 7), (1_000_000, False, 78_498, 1),
    (30_000_000, False, 700_000, 1),     # batches >= 2^20 values: parallel text encoding
    (30_000_000, True, 1_000_000, 2)])
def test_writer_matches_reference_sink(tmp_path, port, limit, binary, ppf, batches):
    from oracle.oracle import Reference
    try:
        ref = Reference()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"reference library unavailable: {e}")
    values = port.naive_sieve(limit).astype(np.uint64)
    ours, theirs = tmp_path / "ours", tmp_path / "ref"
    _write(ours, values, binary, ppf, batches, limit + 1)
    ref.store_run(limit, str(theirs), binary, ppf)
    a, b = _files(ours), _files(theirs)
    assert sorted(a) == sorted(b)
    for name in b:
        assert a[name] == b[name], name
    assert ref.verify_store(str(ours)) == 0
    assert lib.ws_verify_store(str(ours).encode()) == 0


def test_writer_durability_and_errors(tmp_path):
    st = C.c_void_p()
    assert lib.ws_store_open(str(tmp_path / "s").encode(), 1, 0, C.byref(st)) == 5  # Domain
    assert lib.ws_store_open(str(tmp_path / "s").encode(), 1, 4, C.byref(st)) == 0
    v = np.array([2, 3, 5, 7, 11, 13, 17], np.uint64)
    assert lib.ws_store_append(st, v.ctypes.data, 5) == 0   # one file closed at 4
    assert lib.ws_store_durable_count(st) == 4
    assert lib.ws_store_append(st, v[5:].ctypes.data, 2) == 0
    assert lib.ws_store_set_frontier(st, 17) == 5          # does not cover 17: Domain
    assert lib.ws_store_flush(st) == 0
    assert lib.ws_store_durable_count(st) == 7
    assert lib.ws_store_close(st) == 0
    assert sorted(os.listdir(tmp_path / "s")) == ["manifest.json", "primes_00000.bin",
                                                   "primes_00001.bin"]


@pytest.mark.parametrize("binary", [True, False])
def test_large_batches_write_in_parallel_pieces(tmp_path, binary):
    """Batches above 64 MB go out as parallel pwrite()s (and, in text, parallel
    encoding): the files equal those of many small sequential batches, and
    their recorded CRC-32s verify."""
    rng = np.random.default_rng(3)
    values = np.cumsum(rng.integers(1, 40, 9_000_000, dtype=np.uint64)).astype(np.uint64)
    big, small = tmp_path / "big", tmp_path / "small"
    _write(big, values, binary, 5_000_000, 1, int(values[-1]) + 1)
    _write(small, values, binary, 5_000_000, 97, int(values[-1]) + 1)
    a, b = _files(big), _files(small)
    assert sorted(a) == sorted(b) == ["manifest.json", f"primes_00000.{'bin' if binary else 'txt'}",
                                       f"primes_00001.{'bin' if binary else 'txt'}"]
    for name in a:
        assert a[name] == b[name], name
    assert lib.ws_verify_store(str(big).encode()) == 0
