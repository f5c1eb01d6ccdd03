"""GPU: the run(SieveConfig) drop-in, mirroring the reference's
tests/test_engine.cpp cases (file:line cited per test)."""
import numpy as np
import pytest

import paper_2310_17746_b200 as ws
from paper_2310_17746_b200 import (CountSink, Errc, Error, MemorySink, SieveConfig, SinkFailure,
                                   round_segment_span, run)

pytestmark = pytest.mark.gpu


def run_collect(limit, threads, span):
    sink = MemorySink()
    run(SieveConfig(limit, threads, round_segment_span(span, threads), 0, sink))
    return [int(x) for x in sink.primes()]


def test_round_segment_span():  # test_engine.cpp:48-71
    assert round_segment_span(6000, 1) == 6000
    assert round_segment_span(6000, 3) == 6012
    assert round_segment_span(600000, 3) == 600012
    assert round_segment_span(6001, 8) == 6048
    assert round_segment_span(0, 4) == 24
    assert round_segment_span(1, 1) == 6
    with pytest.raises(Error) as e:
        round_segment_span(2**64 - 1, 1000)
    assert e.value.code == Errc.Overflow
    with pytest.raises(Error) as e:
        round_segment_span(6000, 0)
    assert e.value.code == Errc.BadConfig


def test_tiny_limits(port):  # test_engine.cpp:113-121
    assert run_collect(2, 1, 6000) == [2]
    assert run_collect(3, 1, 6000) == [2, 3]
    assert run_collect(4, 1, 6000) == [2, 3]
    assert run_collect(5, 1, 6000) == [2, 3, 5]
    assert run_collect(30, 1, 6000) == [int(x) for x in port.naive_sieve(30)]
    assert run_collect(29, 1, 6000) == [int(x) for x in port.naive_sieve(30)]


def test_limits_below_two():  # test_engine.cpp:123-133
    for limit in (0, 1):
        with pytest.raises(Error) as e:
            run(SieveConfig(limit, 1, 6000, 0, MemorySink()))
        assert e.value.code == Errc.EmptyRange


def test_bounded_run_totals(port):  # test_engine.cpp:135-148
    sink = MemorySink()
    rep = run(SieveConfig(1_000_000, 2, 600000, 0, sink))
    assert rep.prime_count == 78498 and rep.largest_prime == 999983
    assert rep.iterations == 2 and rep.sieved_to == 1_000_001
    assert not rep.stopped and not rep.overflowed and rep.wall_ms >= 0
    assert np.array_equal(sink.primes(), port.naive_sieve(1_000_000))


def test_flag_accounting():  # test_engine.cpp:150-161
    def rep(width, threads):
        return run(SieveConfig(10_000, threads, 6000, width, CountSink()))
    assert rep(0, 1).peak_flag_entries == 2000
    assert rep(0, 1).peak_flag_bytes == 250
    assert rep(1, 1).peak_flag_bytes == 2000
    assert rep(2, 1).peak_flag_bytes == 8000
    assert rep(0, 4).peak_flag_entries == 2000


def test_invariance(port):  # test_engine.cpp:163-173
    ref = [int(x) for x in port.naive_sieve(10_000)]
    for threads in (1, 2, 3, 8):
        for span in (6000, 60000):
            assert run_collect(10_000, threads, span) == ref


def test_count_only_matches(port):  # test_engine.cpp:175-183
    c = CountSink()
    rep = run(SieveConfig(123_456, 3, round_segment_span(6000, 3), 0, c))
    assert rep.prime_count == 11601 and rep.largest_prime == 123_449
    assert c.count() == 11601 and c.largest() == 123_449


def test_invalid_configs():  # test_engine.cpp:185-225
    for cfg in (SieveConfig(1000, 1, 6000, 0, None), SieveConfig(1000, 0, 6000, 0, MemorySink()),
                SieveConfig(1000, 3, 6000, 0, MemorySink()),
                SieveConfig(1000, 2000, 6_000_000, 0, MemorySink()),
                SieveConfig(None, 1, 6000, 0, MemorySink())):
        with pytest.raises(Error) as e:
            run(cfg)
        assert e.value.code == Errc.BadConfig


class FailingSink(MemorySink):  # test_engine.cpp:38-45
    def accept(self, batch):
        if len(batch) and int(batch[-1]) >= 100:
            raise Error(Errc.Io, "disk full")
        super().accept(batch)


def test_sink_failure_partial(port):  # test_engine.cpp:227-238
    sink = FailingSink()
    with pytest.raises(SinkFailure) as e:
        run(SieveConfig(10_000, 1, 96, 0, sink))
    assert e.value.code == Errc.Io
    assert e.value.partial.prime_count == 24 and e.value.partial.largest_prime == 89
    assert np.array_equal(sink.primes(), port.naive_sieve(96))


def test_back_to_back():  # test_engine.cpp:274-280
    assert run_collect(100, 1, 6000) == run_collect(100, 1, 6000)


class StopRequestingSink(MemorySink):  # test_engine.cpp:22-34
    def __init__(self, flag):
        super().__init__()
        self.flag = flag

    def accept(self, batch):
        super().accept(batch)
        self.flag.set()


def test_unbounded_stop(port):  # test_engine.cpp:240-272
    import threading
    from paper_2310_17746_b200 import run_unbounded
    ev = threading.Event()
    ev.set()
    rep = run_unbounded(SieveConfig(None, 1, 6000, 0, CountSink()), ev)
    assert rep.stopped and not rep.overflowed and rep.prime_count == 0 and rep.iterations == 0
    ev = threading.Event()
    sink = StopRequestingSink(ev)
    rep = run_unbounded(SieveConfig(None, 1, 6000, 0, sink), ev)
    assert rep.stopped and rep.iterations == 1 and rep.prime_count == 783
    assert rep.largest_prime == 5987 and rep.sieved_to == 6000
    assert np.array_equal(sink.primes(), port.naive_sieve(5999))
    with pytest.raises(Error) as e:
        run_unbounded(SieveConfig(1000, 1, 6000, 0, MemorySink()), threading.Event())
    assert e.value.code == Errc.BadConfig


def test_large_run_values_match_checksums(sieve):  # config-2 style through run()
    class ChecksumSink(ws.PrimeSink):
        def __init__(self):
            super().__init__()
            self.s = 0
            self.x = 0

        def accept(self, batch):
            self.s = (self.s + int(batch.sum(dtype=np.uint64))) % 2**64
            self.x ^= int(np.bitwise_xor.reduce(batch))

    sink = ChecksumSink()
    rep = run(SieveConfig(10**9, 1, 6 * (1 << 18), 0, sink), sieve)
    assert rep.prime_count == 50_847_534 and rep.largest_prime == 999_999_937
    assert sink.s == 24_739_512_092_254_535 and sink.x == 6_213_527


def test_prime_stream(port):  # test_stream.cpp:12-69, acceptance.cpp:363-400
    import itertools
    from paper_2310_17746_b200 import PrimeStream
    assert list(itertools.islice(PrimeStream(1000), 10)) == [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]
    ref = [int(x) for x in port.naive_sieve(1_000_000)]
    assert list(itertools.islice(PrimeStream(7, segments_per_refill=3), len(ref))) == ref
    s = PrimeStream(1 << 12)
    v = None
    for _ in range(100_000):
        v = s.next()
    assert v == 1_299_709
    with pytest.raises(Error) as e:
        PrimeStream(0)
    assert e.value.code == Errc.Domain
    assert PrimeStream.segment_would_overflow(ws.wheelsieve.K_MAX_SEGMENT_END, 1)


class _RecordingCounts(CountSink):
    def __init__(self):
        super().__init__()
        self.batches = []

    def emit_count(self, n, largest):
        super().emit_count(n, largest)
        if n:
            self.batches.append((n, largest))


class _RecordingValues(MemorySink):
    def __init__(self):
        super().__init__()
        self.batches = []

    def accept(self, batch):
        super().accept(batch)
        self.batches.append((int(batch.size), int(batch[-1])))


def _expected_tiles(port, limit, threads, span):
    """engine.cpp:233-288: per iteration, one batch per non-empty worker tile
    (after 2, 3), computed here from the oracle over each tile's values."""
    out = [(2, 3)]
    limit_end = (limit // 6 + 1) * 6
    seg_lo = 0
    sub = span // threads
    while seg_lo < limit_end:
        seg_hi = min(seg_lo + span, limit_end)
        for j in range(threads):
            lo = seg_lo + j * sub
            if lo >= seg_hi:
                break
            hi = min(lo + sub, seg_hi)
            a, b = max(lo, 4), min(hi, limit + 1)
            if a < b:
                r = port.range(a, b)
                if r["count"]:
                    out.append((r["count"], r["largest"]))
        seg_lo += span
    return out


@pytest.mark.parametrize("limit,threads,span", [(100_000, 3, 6012), (1_000_000, 8, 600_000),
                                                (6_100, 2, 6_000), (10**7 + 7, 5, 600_000)])
def test_emission_granularity_per_tile(port, limit, threads, span):
    """Count sinks get emit_count(count, largest) for every non-empty worker
    tile of every iteration, value sinks emit(values) per tile -- the
    reference's batches exactly (engine.cpp:277-288)."""
    want = _expected_tiles(port, limit, threads, span)
    c = _RecordingCounts()
    run(SieveConfig(limit, threads, span, 0, c))
    assert c.batches == want
    v = _RecordingValues()
    run(SieveConfig(limit, threads, span, 0, v))
    assert v.batches == want


def test_count_sink_failure_partials(port):
    """SinkFailure carries the totals of the batches emitted before the
    failing one (engine.cpp:290-295) -- per tile, also for count sinks."""
    class Refuse(CountSink):
        def emit_count(self, n, largest):
            if largest > 50_000:
                raise Error(Errc.Io, "disk full")
            super().emit_count(n, largest)

    s = Refuse()
    with pytest.raises(SinkFailure) as e:
        run(SieveConfig(200_000, 4, 24_000, 0, s))
    want = port.range(0, 48_001)  # tiles of 6000: the last accepted one ends at 48000
    assert e.value.partial.prime_count == want["count"]
    assert e.value.partial.largest_prime == want["largest"]
    assert e.value.partial.iterations == 2
