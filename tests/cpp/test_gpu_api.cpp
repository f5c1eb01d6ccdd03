// C++ parity tests of wheelsieve::gpu (include/wheelsieve/gpu.hpp) that read
// like the reference's own suite: each case cites the reference test it
// mirrors.  Expected values come from a textbook sieve local to this file
// (an independent checker, like the reference's naive_sieve oracle,
// wheel.cpp:40-54) and from known answers in the reference tests.
// Prints "[PASS]"/"[FAIL]" lines; exit code = number of failures.
#include <atomic>
#include <filesystem>
#include <cstdio>
#include <string>
#include <vector>

#include "wheelsieve/gpu.hpp"

using namespace wheelsieve::gpu;

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

std::vector<uint64_t> run_collect(Device& dev, uint64_t limit, unsigned threads, uint64_t span) {
  MemorySink sink;
  SieveConfig config{limit, threads, round_segment_span(span, threads), FlagWidth::Bit, &sink};
  run(config, dev);
  return sink.primes();
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
  Device dev;

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
      EXPECT_ERROR(Errc::EmptyRange, run({limit, 1, 6000, FlagWidth::Bit, &sink}, dev));
  }

  {  // test_engine.cpp:135-148
    MemorySink sink;
    const SieveReport r = run({1'000'000, 2, 600000, FlagWidth::Bit, &sink}, dev);
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
      return run({10'000, t, 6000, w, &sink}, dev);
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
        run({123'456, 3, round_segment_span(6000, 3), FlagWidth::Bit, &counter}, dev);
    CHECK(r.prime_count == 11601);
    CHECK(r.largest_prime == 123'449);
    CHECK(counter.count() == 11601 && counter.largest() == 123'449);
  }

  {  // test_engine.cpp:185-225
    MemorySink sink;
    EXPECT_ERROR(Errc::BadConfig, run({1000, 1, 6000, FlagWidth::Bit, nullptr}, dev));
    EXPECT_ERROR(Errc::BadConfig, run({1000, 0, 6000, FlagWidth::Bit, &sink}, dev));
    EXPECT_ERROR(Errc::BadConfig, run({1000, 3, 6000, FlagWidth::Bit, &sink}, dev));
    EXPECT_ERROR(Errc::BadConfig, run({1000, 2000, 6'000'000, FlagWidth::Bit, &sink}, dev));
    EXPECT_ERROR(Errc::BadConfig, run({std::nullopt, 1, 6000, FlagWidth::Bit, &sink}, dev));
    std::atomic<bool> stop{false};
    EXPECT_ERROR(Errc::BadConfig, run_unbounded({1000, 1, 6000, FlagWidth::Bit, &sink}, stop, dev));
  }

  {  // test_engine.cpp:227-238
    FailingSink sink;
    try {
      run({10'000, 1, 96, FlagWidth::Bit, &sink}, dev);
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
        run_unbounded({std::nullopt, 1, 6000, FlagWidth::Bit, &counter}, stop, dev);
    CHECK(r.stopped && !r.overflowed && r.prime_count == 0 && r.iterations == 0);
  }

  {  // test_engine.cpp:252-262
    std::atomic<bool> stop{false};
    StopRequestingSink sink(stop);
    const SieveReport r = run_unbounded({std::nullopt, 1, 6000, FlagWidth::Bit, &sink}, stop, dev);
    CHECK(r.stopped && r.iterations == 1);
    CHECK(r.prime_count == 783 && r.largest_prime == 5987 && r.sieved_to == 6000);
    CHECK(sink.primes() == textbook(5999));
  }

  {  // test_engine.cpp:264-272
    std::atomic<bool> s1{false}, s4{false};
    StopRequestingSink k1(s1), k4(s4);
    run_unbounded({std::nullopt, 1, 6000, FlagWidth::Bit, &k1}, s1, dev);
    run_unbounded({std::nullopt, 4, 6000, FlagWidth::Bit, &k4}, s4, dev);
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

  {  // test_segment.cpp:135-184 against the SegmentBitmap mirror
    const SegmentFlags seg = dev.sieve_segment(12000, 1000);
    CHECK(!seg.flag_for(14443) && !seg.flag_for(14417) && seg.flag_for(12007));
    const auto all = textbook(18000);
    std::vector<uint64_t> sl;
    for (uint64_t p : all)
      if (p >= 12000) sl.push_back(p);
    CHECK(seg.surviving() == sl);
    const SegmentFlags first = dev.sieve_segment(0, 1000);
    CHECK(first.flag_for(1));  // not a multiple of anything; callers clear it
    const SegmentFlags one = dev.sieve_segment(10200, 1);
    CHECK(!one.flag_for(10201) && !one.flag_for(10205));
    const SegmentFlags sq = dev.sieve_segment(168, 1);
    CHECK(!sq.flag_for(169) && sq.flag_for(173));
    EXPECT_ERROR(Errc::Alignment, dev.sieve_segment(10, 5));
    EXPECT_ERROR(Errc::Domain, dev.sieve_segment(12, 0));
    EXPECT_ERROR(Errc::Overflow, dev.sieve_segment(kMaxSegmentEnd, 1));
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
    PrimeStream st(1000, dev);
    std::vector<uint64_t> first;
    for (int i = 0; i < 10; ++i) first.push_back(*st.next());
    CHECK((first == std::vector<uint64_t>{2, 3, 5, 7, 11, 13, 17, 19, 23, 29}));
    PrimeStream s2(7, dev);
    const auto ref = textbook(1'000'000);
    bool same = true;
    for (uint64_t p : ref) same = same && (*s2.next() == p);
    CHECK(same);
    PrimeStream s3(1 << 12, dev);
    uint64_t v = 0;
    for (int i = 0; i < 100'000; ++i) v = *s3.next();
    CHECK(v == 1'299'709);
    EXPECT_ERROR(Errc::Domain, PrimeStream(0, dev));
    CHECK(PrimeStream::segment_would_overflow(kMaxSegmentEnd, 1));
    CHECK(!PrimeStream::segment_would_overflow(0, 1));
  }

  {  // chunked store round trip through the C++ mirror (sink.hpp:68-141)
    const std::string d = "/tmp/wheelsieve_gpu_cpp_store";
    std::filesystem::remove_all(d);
    const uint64_t n = dev.store_range(0, 1'000'001, d, true, 10'000);
    CHECK(n == 78'498);
    verify_store(d);
    CHECK(read_back(d, 0, 1'000'001) == textbook(1'000'000));
    EXPECT_ERROR(Errc::BeyondFrontier, read_back(d, 0, 1'000'002));
    std::filesystem::remove_all(d);
  }

  std::printf(g_fail ? "[FAIL] %d failures\n" : "[PASS] all checks\n", g_fail);
  return g_fail;
}
