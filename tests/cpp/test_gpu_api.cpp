// C++ parity tests of the drop-in C++ API (include/wheelsieve/*.hpp,
// libwheelsieve.so over the GPU C ABI) that read like the reference's own
// suite: each case cites the reference test it mirrors.  Expected values come from a textbook sieve local to this file
// (an independent checker, like the reference's naive_sieve oracle,
// wheel.cpp:40-54) and from known answers in the reference tests.
// Prints "[PASS]"/"[FAIL]" lines; exit code = number of failures.
#include <atomic>
#include <filesystem>
#include <cstdio>
#include <string>
#include <vector>

#include "wheelsieve/base_store.hpp"
#include "wheelsieve/engine.hpp"
#include "wheelsieve/gpu.hpp"
#include "wheelsieve/segment.hpp"
#include "wheelsieve/sink.hpp"
#include "wheelsieve/stream.hpp"
#include "wheelsieve/wheel.hpp"

using namespace wheelsieve;
using gpu::Checks;
using gpu::Context;

namespace {

int g_fail = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      std::printf("[FAIL] %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++g_fail;                                                              \
    }                                                                        \
  } while (0)

template <class F>
void expect_error(Errc code, F&& f, int line) {
  try {
    f();
    std::printf("[FAIL] line %d: expected error %d\n", line, static_cast<int>(code));
    ++g_fail;
  } catch (const Error& e) {
    if (e.code() != code) {
      std::printf("[FAIL] line %d: got error %d, expected %d (%s)\n", line,
                  static_cast<int>(e.code()), static_cast<int>(code), e.what());
      ++g_fail;
    }
  }
}
#define EXPECT_ERROR(code, stmt) expect_error(code, [&] { stmt; }, __LINE__)

std::vector<uint64_t> textbook(uint64_t n) {  // all primes <= n
  std::vector<uint8_t> comp(n + 1, 0);
  std::vector<uint64_t> out;
  for (uint64_t i = 2; i <= n; ++i) {
    if (comp[i]) continue;
    out.push_back(i);
    for (uint64_t j = i * i; j <= n; j += i) comp[j] = 1;
  }
  return out;
}

std::vector<uint64_t> run_collect(Context& dev, uint64_t limit, unsigned threads, uint64_t span) {
  MemorySink sink;
  SieveConfig config{limit, threads, round_segment_span(span, threads), FlagWidth::Bit, &sink};
  gpu::run(config, dev);
  return sink.primes();
}

// sieve_segment on a fresh SegmentBitmap with a bootstrapped base store
SegmentBitmap sieved(uint64_t start, uint64_t len) {
  SegmentBitmap seg(start, len);
  sieve_segment(seg, BasePrimeStore::bootstrap(std::max<uint64_t>(25, start + 6 * len)));
  return seg;
}

class StopRequestingSink : public MemorySink {  // test_engine.cpp:22-34
 public:
  explicit StopRequestingSink(std::atomic<bool>& stop) : stop_(stop) {}

 protected:
  void accept(std::span<const uint64_t> batch) override {
    MemorySink::accept(batch);
    stop_.store(true, std::memory_order_relaxed);
  }

 private:
  std::atomic<bool>& stop_;
};

class FailingSink : public MemorySink {  // test_engine.cpp:38-45
 protected:
  void accept(std::span<const uint64_t> batch) override {
    if (!batch.empty() && batch.back() >= 100) throw Error(Errc::Io, "disk full");
    MemorySink::accept(batch);
  }
};

}  // namespace

int main() {
  Context dev;

  // test_engine.cpp:48-71
  CHECK(round_segment_span(6000, 1) == 6000);
  CHECK(round_segment_span(6000, 3) == 6012);
  CHECK(round_segment_span(600000, 3) == 600012);
  CHECK(round_segment_span(6000, 8) == 6000);
  CHECK(round_segment_span(6001, 8) == 6048);
  CHECK(round_segment_span(0, 4) == 24);
  CHECK(round_segment_span(1, 1) == 6);
  EXPECT_ERROR(Errc::Overflow, round_segment_span(UINT64_MAX, 1000));
  EXPECT_ERROR(Errc::BadConfig, round_segment_span(6000, 0));

  {  // test_engine.cpp:73-98
    SieveConfig config;
    config.segment_span = 6000;
    config.threads = 5;
    const auto plan = plan_iteration(config, 2);
    CHECK(plan.size() == 5);
    CHECK((plan[0] == WorkerAssignment{2, 0, 12000, 13200}));
    CHECK((plan[2] == WorkerAssignment{2, 2, 14400, 15600}));
    CHECK((plan[4] == WorkerAssignment{2, 4, 16800, 18000}));
    config.threads = 7;
    EXPECT_ERROR(Errc::BadConfig, plan_iteration(config, 0));
    config.threads = 1;
    EXPECT_ERROR(Errc::Overflow, plan_iteration(config, kMaxSegmentEnd / 6000));
  }

  // tiny limits, test_engine.cpp:113-121
  CHECK((run_collect(dev, 2, 1, 6000) == std::vector<uint64_t>{2}));
  CHECK((run_collect(dev, 3, 1, 6000) == std::vector<uint64_t>{2, 3}));
  CHECK((run_collect(dev, 4, 1, 6000) == std::vector<uint64_t>{2, 3}));
  CHECK((run_collect(dev, 5, 1, 6000) == std::vector<uint64_t>{2, 3, 5}));
  CHECK(run_collect(dev, 30, 1, 6000) == textbook(30));
  CHECK(run_collect(dev, 29, 1, 6000) == textbook(30));

  {  // test_engine.cpp:123-133
    MemorySink sink;
    for (uint64_t limit : {uint64_t{0}, uint64_t{1}})
      EXPECT_ERROR(Errc::EmptyRange, gpu::run({limit, 1, 6000, FlagWidth::Bit, &sink}, dev));
  }

  {  // test_engine.cpp:135-148
    MemorySink sink;
    const SieveReport r = gpu::run({1'000'000, 2, 600000, FlagWidth::Bit, &sink}, dev);
    CHECK(r.prime_count == 78498);
    CHECK(r.largest_prime == 999983);
    CHECK(r.iterations == 2);
    CHECK(r.sieved_to == 1'000'001);
    CHECK(!r.stopped && !r.overflowed && r.wall_ms >= 0.0);
    CHECK(sink.primes() == textbook(1'000'000));
  }

  {  // test_engine.cpp:150-161
    auto rep = [&](FlagWidth w, unsigned t) {
      CountSink sink;
      return gpu::run({10'000, t, 6000, w, &sink}, dev);
    };
    CHECK(rep(FlagWidth::Bit, 1).peak_flag_entries == 2000);
    CHECK(rep(FlagWidth::Bit, 1).peak_flag_bytes == 250);
    CHECK(rep(FlagWidth::Byte, 1).peak_flag_bytes == 2000);
    CHECK(rep(FlagWidth::Word4, 1).peak_flag_bytes == 8000);
    CHECK(rep(FlagWidth::Bit, 4).peak_flag_entries == 2000);
  }

  {  // test_engine.cpp:163-173
    const auto ref = textbook(10'000);
    for (unsigned t : {1u, 2u, 3u, 8u})
      for (uint64_t span : {uint64_t{6000}, uint64_t{60000}})
        CHECK(run_collect(dev, 10'000, t, span) == ref);
  }

  {  // test_engine.cpp:175-183
    CountSink counter;
    const SieveReport r =
        gpu::run({123'456, 3, round_segment_span(6000, 3), FlagWidth::Bit, &counter}, dev);
    CHECK(r.prime_count == 11601);
    CHECK(r.largest_prime == 123'449);
    CHECK(counter.count() == 11601 && counter.largest() == 123'449);
  }

  {  // test_engine.cpp:185-225
    MemorySink sink;
    EXPECT_ERROR(Errc::BadConfig, gpu::run({1000, 1, 6000, FlagWidth::Bit, nullptr}, dev));
    EXPECT_ERROR(Errc::BadConfig, gpu::run({1000, 0, 6000, FlagWidth::Bit, &sink}, dev));
    EXPECT_ERROR(Errc::BadConfig, gpu::run({1000, 3, 6000, FlagWidth::Bit, &sink}, dev));
    EXPECT_ERROR(Errc::BadConfig, gpu::run({1000, 2000, 6'000'000, FlagWidth::Bit, &sink}, dev));
    EXPECT_ERROR(Errc::BadConfig, gpu::run({std::nullopt, 1, 6000, FlagWidth::Bit, &sink}, dev));
    std::atomic<bool> stop{false};
    EXPECT_ERROR(Errc::BadConfig, gpu::run_unbounded({1000, 1, 6000, FlagWidth::Bit, &sink}, stop, dev));
  }

  {  // test_engine.cpp:227-238
    FailingSink sink;
    try {
      gpu::run({10'000, 1, 96, FlagWidth::Bit, &sink}, dev);
      CHECK(false);
    } catch (const SinkFailure& e) {
      CHECK(e.code() == Errc::Io);
      CHECK(e.partial().prime_count == 24);
      CHECK(e.partial().largest_prime == 89);
      CHECK(sink.primes() == textbook(96));
    }
  }

  {  // test_engine.cpp:240-250
    CountSink counter;
    std::atomic<bool> stop{true};
    const SieveReport r =
        gpu::run_unbounded({std::nullopt, 1, 6000, FlagWidth::Bit, &counter}, stop, dev);
    CHECK(r.stopped && !r.overflowed && r.prime_count == 0 && r.iterations == 0);
  }

  {  // test_engine.cpp:252-262
    std::atomic<bool> stop{false};
    StopRequestingSink sink(stop);
    const SieveReport r = gpu::run_unbounded({std::nullopt, 1, 6000, FlagWidth::Bit, &sink}, stop, dev);
    CHECK(r.stopped && r.iterations == 1);
    CHECK(r.prime_count == 783 && r.largest_prime == 5987 && r.sieved_to == 6000);
    CHECK(sink.primes() == textbook(5999));
  }

  {  // test_engine.cpp:264-272
    std::atomic<bool> s1{false}, s4{false};
    StopRequestingSink k1(s1), k4(s4);
    gpu::run_unbounded({std::nullopt, 1, 6000, FlagWidth::Bit, &k1}, s1, dev);
    gpu::run_unbounded({std::nullopt, 4, 6000, FlagWidth::Bit, &k4}, s4, dev);
    CHECK(k1.primes() == k4.primes());
  }

  // wheel: Table 1 worked example (acceptance.cpp:181-201, test_wheel.cpp:152-159)
  CHECK((start_offsets(13, 14400) == StartOffsets{2407, 2402}));
  EXPECT_ERROR(Errc::Domain, start_offsets(9, 60));
  EXPECT_ERROR(Errc::Alignment, start_offsets(7, 61));
  CHECK(isqrt(UINT64_MAX) == 4294967295ull);

  {  // [L, R) entry points vs the textbook sieve, segment slices of test_segment.cpp
    const auto all = textbook(600'000);
    auto slice = [&](uint64_t L, uint64_t R) {
      std::vector<uint64_t> v;
      for (uint64_t p : all)
        if (p >= L && p < R) v.push_back(p);
      return v;
    };
    CHECK(dev.enumerate_range(12000, 18000) == slice(12000, 18000));   // test_segment.cpp:135-145
    CHECK(dev.enumerate_range(10200, 10206).empty());                  // :157-165
    CHECK((dev.enumerate_range(168, 174) == std::vector<uint64_t>{173})); // :167-173
    CHECK(dev.enumerate_range(594000, 600000) == slice(594000, 600000)); // :186-193
    std::vector<uint32_t> per;
    const Checks c = dev.count_range(0, 1'000'000'001, false, &per);  // config 1
    CHECK(c.count == 50'847'534 && per.size() == 636);
    uint64_t sum = 0;
    for (uint32_t x : per) sum += x;
    CHECK(sum + 2 == c.count && per[0] == 119'266 && per.back() == 59'150);
    std::vector<uint32_t> counts;
    std::vector<uint64_t> sums;
    const std::vector<uint64_t> Ls = {378'761'080'469ull};  // first config-5 interval
    dev.count_intervals(Ls, 1ull << 24, counts, &sums);
    CHECK(counts[0] == 628'905 && sums[0] == 238'210'012'871'732'589ull);
  }

  {  // test_segment.cpp:135-184 through SegmentBitmap + sieve_segment
    const SegmentBitmap seg = sieved(12000, 1000);
    CHECK(!seg.flag_for(14443) && !seg.flag_for(14417) && seg.flag_for(12007));
    const auto all = textbook(18000);
    std::vector<uint64_t> sl;
    for (uint64_t p : all)
      if (p >= 12000) sl.push_back(p);
    CHECK(seg.surviving() == sl);
    const SegmentBitmap first = sieved(0, 1000);
    CHECK(first.flag_for(1));  // not a multiple of anything; callers clear it
    const SegmentBitmap one = sieved(10200, 1);
    CHECK(!one.flag_for(10201) && !one.flag_for(10205));
    const SegmentBitmap sq = sieved(168, 1);
    CHECK(!sq.flag_for(169) && sq.flag_for(173));
    EXPECT_ERROR(Errc::Alignment, SegmentBitmap(10, 5));
    EXPECT_ERROR(Errc::Domain, SegmentBitmap(12, 0));
    EXPECT_ERROR(Errc::Overflow, SegmentBitmap(kMaxSegmentEnd, 1));
    EXPECT_ERROR(Errc::NotOnWheel, (void)seg.flag_for(12002));
    EXPECT_ERROR(Errc::Domain, (void)seg.flag_for(18001));
    SegmentBitmap tiny(12000, 1000);  // an incomplete base store (segment.cpp:166-169)
    EXPECT_ERROR(Errc::IncompleteBase, sieve_segment(tiny, BasePrimeStore::bootstrap(25)));
    SegmentBitmap trim = sieved(594000, 1000);  // widths agree (test_segment.cpp:186-193)
    SegmentBitmap wide(594000, 1000, FlagWidth::Byte);
    sieve_segment(wide, BasePrimeStore::bootstrap(600000));
    CHECK(trim.surviving() == wide.surviving() && trim.count_surviving() == wide.count_surviving());
    trim.clear_values_above(597000);
    CHECK(*trim.last_surviving() < 597000 && trim.flag_entries() == 2000);
  }

  {  // test_base_store.cpp:29-38 and test_wheel.cpp:30-74
    const auto b = dev.base_primes(ceil_sqrt(1'000'000));
    CHECK(b.size() == 166 && b.front() == 5 && b.back() == 997);
    CHECK(value_of({0, ResidueClass::R1}) == 1 && value_of({0, ResidueClass::R5}) == 5);
    CHECK((coord_of(25) == WheelCoord{4, ResidueClass::R1}));
    EXPECT_ERROR(Errc::NotOnWheel, coord_of(4));
    EXPECT_ERROR(Errc::Overflow, value_of({kMaxWheelIndex + 1, ResidueClass::R1}));
  }

  {  // test_stream.cpp:12-51, acceptance.cpp:363-400
    PrimeStream st(1000);
    std::vector<uint64_t> first;
    for (int i = 0; i < 10; ++i) first.push_back(*st.next());
    CHECK((first == std::vector<uint64_t>{2, 3, 5, 7, 11, 13, 17, 19, 23, 29}));
    PrimeStream s2(7);
    const auto ref = textbook(1'000'000);
    bool same = true;
    for (uint64_t p : ref) same = same && (*s2.next() == p);
    CHECK(same);
    PrimeStream s3(1 << 12);
    uint64_t v = 0;
    for (int i = 0; i < 100'000; ++i) v = *s3.next();
    CHECK(v == 1'299'709);
    EXPECT_ERROR(Errc::Domain, PrimeStream(0));
    CHECK(s3.base().covers(1'299'710));
    CHECK(PrimeStream::segment_would_overflow(kMaxSegmentEnd, 1));
    CHECK(!PrimeStream::segment_would_overflow(0, 1));
  }

  {  // chunked store round trip (sink.hpp:68-141): the device store, and
     // run() into a ChunkedFileSink -- byte-identical files
    const std::string d = "/tmp/wheelsieve_gpu_cpp_store", e = "/tmp/wheelsieve_gpu_cpp_sink";
    std::filesystem::remove_all(d);
    std::filesystem::remove_all(e);
    const uint64_t n = dev.store_range(0, 1'000'001, d, true, 10'000);
    CHECK(n == 78'498);
    verify_store(d);
    CHECK(read_back(d, 0, 1'000'001) == textbook(1'000'000));
    EXPECT_ERROR(Errc::BeyondFrontier, read_back(d, 0, 1'000'002));
    {
      ChunkedFileSink sink({e, 10'000, FileFormat::Binary});
      const SieveReport r = gpu::run({1'000'000, 2, 600'000, FlagWidth::Bit, &sink}, dev);
      CHECK(sink.durable_count() == 70'000);  // 7 closed files before the final flush
      sink.set_frontier(r.sieved_to);
      sink.flush();
      CHECK(sink.durable_count() == 78'498);
      EXPECT_ERROR(Errc::Domain, sink.set_frontier(999'983));
    }
    verify_store(e);
    auto slurp = [](const std::string& p) {
      std::FILE* f = std::fopen(p.c_str(), "rb");
      std::string s;
      char buf[1 << 16];
      size_t k;
      while (f && (k = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, k);
      if (f) std::fclose(f);
      return s;
    };
    for (const char* f : {"/manifest.json", "/primes_00000.bin", "/primes_00007.bin"})
      CHECK(slurp(d + f) == slurp(e + f) && !slurp(d + f).empty());
    EXPECT_ERROR(Errc::Domain, ChunkedFileSink({e, 0, FileFormat::Text}));
    std::filesystem::remove_all(d);
    std::filesystem::remove_all(e);
  }

  {  // count sinks get one emit_count per non-empty worker tile
     // (engine.cpp:277-288): a limit inside the first tile of iteration 1
    CountSink c;
    const SieveReport r = gpu::run({6'100, 2, 6'000, FlagWidth::Bit, &c}, dev);
    CHECK(r.iterations == 2 && r.prime_count == 795 && r.largest_prime == 6'091);
    MemorySink m;
    EXPECT_ERROR(Errc::Domain, m.emit_count(1, 7));  // value sinks take no counts
  }

  {  // a multi-device context (NCCL, one communicator per device): the same answers
    gpu::ContextOptions o;
    o.devices = {0};
    Context multi(o);
    CHECK(multi.num_devices() == 1 && multi.num_shards() == 1);
    std::vector<uint32_t> per;
    const Checks c = multi.count_range(0, 1'000'000'001, false, &per);
    CHECK(c.count == 50'847'534 && per.size() == 636 && per[0] == 119'266);
    MemorySink sink;
    gpu::run({1'000'000, 3, round_segment_span(600'000, 3), FlagWidth::Bit, &sink}, multi);
    CHECK(sink.primes() == textbook(1'000'000));
    const auto tiles = multi.count_ranges(std::vector<uint64_t>{0, 100, 10'000},
                                          std::vector<uint64_t>{100, 10'000, 10}, true);
    CHECK(tiles[0].count == 25 && tiles[1].count == 1229 - 25 && tiles[2].count == 0);
  }

  std::printf(g_fail ? "[FAIL] %d failures\n" : "[PASS] all checks\n", g_fail);
  return g_fail;
}
