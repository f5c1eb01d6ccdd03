// wheelsieve::gpu -- C++20 host API of the B200 sieve, layered on the C ABI
// of wheelsieve/gpu.h (libwheelsieve_cuda.so).  Header-only.
//
// Drop-in mirror of the reference's public C++ surface for the sieve path
// (/root/reference/proj/include/wheelsieve):
//
//   errors.hpp:9-32     Errc, Error                      -> same names/values
//   sink.hpp:18-66      PrimeSink / CountSink / MemorySink (ascending-batch
//                       contract, count-only emit_count)  -> same semantics
//   engine.hpp:13-89    SieveConfig, WorkerAssignment, SieveReport, SinkFailure,
//                       round_segment_span, plan_iteration, run, run_unbounded
//   wheel.hpp:13-81     ResidueClass, WheelCoord, value_of, coord_of, isqrt,
//                       ceil_sqrt, start_offsets
//   segment.hpp:90-168  SegmentBitmap + sieve_segment -> Device::sieve_segment
//   base_store.hpp:25   BasePrimeStore::bootstrap     -> Device::base_primes
//   (new)               Device::count_range / enumerate_range / count_intervals
//                       for [L, R) (the SURVEY §3.3 composition as one call)
//
// Switching a caller of the reference engine over is a namespace change:
// `using namespace wheelsieve;` -> `using namespace wheelsieve::gpu;`.
// run() keeps the reference's emission granularity (one ascending batch per
// segment_span iteration, 2 and 3 first), its validation order and error
// codes, and its SinkFailure partial totals; the device sieves many
// iterations per call and the batches are cut on the host.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "wheelsieve/gpu.h"

namespace wheelsieve::gpu {

// errors.hpp:9-23 (same enumerators, same order) + device-side codes
enum class Errc : uint8_t {
  NotOnWheel,
  Overflow,
  EmptyRange,
  Capacity,
  Domain,
  Alignment,
  BadConfig,
  IncompleteBase,
  Ordering,
  Io,
  BadManifest,
  ChecksumMismatch,
  BeyondFrontier,
  Cuda = 99,
  NoDevice = 100,
  OutOfMemory = 101,
};

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

inline void check(ws_status s, const ws_ctx* ctx, const char* what) {
  if (s == WS_OK) return;
  std::string msg = std::string(what) + ": " + ws_status_name(s);
  if (ctx) msg += std::string(": ") + ws_last_error(ctx);
  throw Error(static_cast<Errc>(static_cast<int>(s) - 1), msg);
}

inline constexpr uint64_t kMaxWheelIndex = (UINT64_MAX - 5) / 6;        // wheel.hpp:33
inline constexpr uint64_t kMaxSegmentEnd = 6 * (kMaxWheelIndex + 1);    // wheel.hpp:37

inline uint64_t isqrt(uint64_t n) { return ws_isqrt(n); }

inline uint64_t ceil_sqrt(uint64_t n) {  // wheel.cpp:35-38
  const uint64_t r = isqrt(n);
  return r * r == n ? r : r + 1;
}

enum class ResidueClass : uint8_t { R1, R5 };  // wheel.hpp:13

struct WheelCoord {  // wheel.hpp:17-22
  uint64_t index;
  ResidueClass residue;
  bool operator==(const WheelCoord&) const = default;
};

inline uint64_t value_of(WheelCoord c) {  // wheel.cpp:8-13
  if (c.index > kMaxWheelIndex)
    throw Error(Errc::Overflow, "wheel index " + std::to_string(c.index) +
                                    " exceeds the 64-bit value range");
  return 6 * c.index + (c.residue == ResidueClass::R1 ? 1 : 5);
}

inline WheelCoord coord_of(uint64_t n) {  // wheel.cpp:15-23
  switch (n % 6) {
    case 1: return {n / 6, ResidueClass::R1};
    case 5: return {n / 6, ResidueClass::R5};
    default:
      throw Error(Errc::NotOnWheel, std::to_string(n) + " is divisible by 2 or 3, not on the wheel");
  }
}

struct StartOffsets {  // wheel.hpp:26-30
  uint64_t id1;
  uint64_t id5;
  bool operator==(const StartOffsets&) const = default;
};

inline StartOffsets start_offsets(uint64_t p, uint64_t segment_start) {
  StartOffsets o{};
  check(ws_start_offsets(p, segment_start, &o.id1, &o.id5), nullptr, "start_offsets");
  return o;
}

// ---------------------------------------------------------------- sinks ----
class PrimeSink {  // sink.hpp:18-43, sink.cpp:14-37
 public:
  virtual ~PrimeSink() = default;

  void emit(std::span<const uint64_t> batch) {
    if (batch.empty()) return;
    uint64_t prev = largest_;
    for (uint64_t v : batch) {
      if (v <= prev)
        throw Error(Errc::Ordering, "emit batch not strictly ascending past " +
                                        std::to_string(prev) + " (got " + std::to_string(v) + ")");
      prev = v;
    }
    accept(batch);
    count_ += batch.size();
    largest_ = batch.back();
  }

  void emit_count(uint64_t n, uint64_t largest) {
    if (n == 0) return;
    if (wants_values())
      throw Error(Errc::Domain, "sink needs the values; count-only emission not possible");
    if (largest <= largest_)
      throw Error(Errc::Ordering, "count batch ends at " + std::to_string(largest) +
                                      ", not above " + std::to_string(largest_));
    count_ += n;
    largest_ = largest;
  }

  virtual void flush() {}
  virtual bool wants_values() const { return true; }
  uint64_t count() const { return count_; }
  uint64_t largest() const { return largest_; }

 protected:
  virtual void accept(std::span<const uint64_t> batch) = 0;

 private:
  uint64_t count_ = 0;
  uint64_t largest_ = 0;
};

class CountSink : public PrimeSink {
 public:
  bool wants_values() const override { return false; }

 protected:
  void accept(std::span<const uint64_t>) override {}
};

class MemorySink : public PrimeSink {
 public:
  const std::vector<uint64_t>& primes() const { return primes_; }

 protected:
  void accept(std::span<const uint64_t> batch) override {
    primes_.insert(primes_.end(), batch.begin(), batch.end());
  }

 private:
  std::vector<uint64_t> primes_;
};

// --------------------------------------------------------------- device ----
struct Checks {
  uint64_t count = 0, sum = 0, xr = 0, largest = 0;
};

// Flag arrays of one sieved segment in FlagArray's Bit layout (segment.hpp:34-84):
// bit i of words[i >> 6], LSB-first, tail bits zero; the value 1 left set.
struct SegmentFlags {
  uint64_t start = 0, len = 0;
  std::vector<uint64_t> r1, r5;
  bool test(ResidueClass r, uint64_t i) const {
    const auto& w = r == ResidueClass::R1 ? r1 : r5;
    return (w[i >> 6] >> (i & 63)) & 1;
  }
  bool flag_for(uint64_t value) const {  // segment.cpp:112-124 (unchecked range)
    const WheelCoord c = coord_of(value);
    return test(c.residue, c.index - start / 6);
  }
  std::vector<uint64_t> surviving() const {  // segment.hpp:123-146 order
    std::vector<uint64_t> v;
    for (size_t wi = 0; wi < r1.size(); ++wi) {
      uint64_t m1 = r1[wi], m5 = r5[wi], both = m1 | m5;
      while (both) {
        const int bit = __builtin_ctzll(both);
        both &= both - 1;
        const uint64_t k = (uint64_t{wi} << 6) | static_cast<uint64_t>(bit);
        if ((m1 >> bit) & 1) v.push_back(start + 6 * k + 1);
        if ((m5 >> bit) & 1) v.push_back(start + 6 * k + 5);
      }
    }
    return v;
  }
};

// One GPU context (device buffers, stream, resident base-prime table).  Not
// reentrant: one Device per host thread.
class Device {
 public:
  explicit Device(int device = -1, uint32_t segment_slots = 1u << 18) {
    ws_opts o;
    ws_opts_default(&o);
    o.device = device;
    o.segment_slots = segment_slots;
    check(ws_ctx_create(&o, &ctx_), nullptr, "ws_ctx_create");
    slots_ = segment_slots;
  }
  ~Device() { ws_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  uint32_t segment_slots() const { return slots_; }
  ws_ctx* handle() { return ctx_; }

  Checks count_range(uint64_t L, uint64_t R, bool checksums = false,
                     std::vector<uint32_t>* per_segment = nullptr) {
    ws_checks c{};
    uint64_t nseg = 0;
    if (per_segment) {
      const uint64_t lo0 = L / 6 * 6;
      const uint64_t slots = R > L ? (R - lo0 + 5) / 6 : 0;
      per_segment->assign((slots + slots_ - 1) / slots_, 0);
    }
    check(ws_count_range(ctx_, L, R, checksums ? WS_WANT_CHECKS : 0u, &c,
                         per_segment ? per_segment->data() : nullptr,
                         per_segment ? per_segment->size() : 0, &nseg),
          ctx_, "ws_count_range");
    return {c.count, c.sum, c.xor_, c.largest};
  }

  std::vector<uint64_t> enumerate_range(uint64_t L, uint64_t R, Checks* checks = nullptr) {
    std::vector<uint64_t> out(std::max<uint64_t>(1, ws_prime_count_bound(L, R)));
    uint64_t n = 0;
    ws_checks c{};
    check(ws_enumerate_range(ctx_, L, R, 0u, out.data(), out.size(), &n, &c), ctx_,
          "ws_enumerate_range");
    out.resize(n);
    if (checks) *checks = {c.count, c.sum, c.xor_, c.largest};
    return out;
  }

  // BasePrimeStore::bootstrap entries: the wheel primes 5 <= p <= B.
  std::vector<uint64_t> base_primes(uint64_t B) {
    std::vector<uint64_t> out(std::max<uint64_t>(1, ws_prime_count_bound(0, B + 1)));
    uint64_t n = 0;
    check(ws_base_primes(ctx_, B, 0u, out.data(), out.size(), &n), ctx_, "ws_base_primes");
    out.resize(n);
    return out;
  }

  // SegmentBitmap(start, len) + sieve_segment (segment.cpp:93-188).
  SegmentFlags sieve_segment(uint64_t start, uint64_t len) {
    SegmentFlags f;
    f.start = start;
    f.len = len;
    const uint64_t nw = (len + 63) / 64;
    f.r1.assign(std::max<uint64_t>(nw, 1), 0);
    f.r5.assign(std::max<uint64_t>(nw, 1), 0);
    check(ws_sieve_segment(ctx_, start, len, 0u, f.r1.data(), f.r5.data()), ctx_,
          "ws_sieve_segment");
    f.r1.resize(nw);
    f.r5.resize(nw);
    return f;
  }

  // ChunkedFileSink-format store of the primes of [L, R) (frontier R).
  uint64_t store_range(uint64_t L, uint64_t R, const std::string& dir, bool binary,
                       uint64_t primes_per_file = 125'000'000) {
    uint64_t n = 0;
    check(ws_store_range(ctx_, L, R, dir.c_str(), binary ? WS_STORE_BINARY : WS_STORE_TEXT,
                         primes_per_file, &n),
          ctx_, "ws_store_range");
    return n;
  }

  void count_intervals(std::span<const uint64_t> Ls, uint64_t width, std::vector<uint32_t>& counts,
                       std::vector<uint64_t>* sums = nullptr,
                       std::vector<uint64_t>* xors = nullptr) {
    counts.assign(Ls.size(), 0);
    if (sums) sums->assign(Ls.size(), 0);
    if (xors) xors->assign(Ls.size(), 0);
    check(ws_count_intervals(ctx_, Ls.data(), Ls.size(), width, 0u, counts.data(),
                             sums ? sums->data() : nullptr, xors ? xors->data() : nullptr),
          ctx_, "ws_count_intervals");
  }

 private:
  ws_ctx* ctx_ = nullptr;
  uint32_t slots_ = 0;
};

// read_back / verify_store (sink.cpp:306-342) over a chunked store.
inline std::vector<uint64_t> read_back(const std::string& dir, uint64_t lo, uint64_t hi) {
  uint64_t n = 0;
  const ws_status s = ws_read_back(dir.c_str(), lo, hi, nullptr, 0, &n);
  if (s != WS_OK && s != WS_CAPACITY) check(s, nullptr, "read_back");
  std::vector<uint64_t> v(n);
  check(ws_read_back(dir.c_str(), lo, hi, v.data(), v.size(), &n), nullptr, "read_back");
  return v;
}
inline void verify_store(const std::string& dir) {
  check(ws_verify_store(dir.c_str()), nullptr, "verify_store");
}

// Unbounded incremental enumerator (stream.hpp:16-46): 2, 3, then every wheel
// prime ascending; the device sieves `block` values per refill (a multiple of
// 6 * segment_wheel_len) and the base primes grow with it (the store's
// incremental growth, base_store.cpp:44-76).  nullopt once the 64-bit range
// is exhausted (overflowed() then stays true).
class PrimeStream {
 public:
  explicit PrimeStream(uint64_t segment_wheel_len, Device& dev,
                       uint64_t segments_per_refill = 64)
      : dev_(dev), wheel_len_(segment_wheel_len) {
    if (segment_wheel_len == 0)
      throw Error(Errc::Domain, "segment must span at least one wheel index");
    if (segment_wheel_len > kMaxSegmentEnd / 6)
      throw Error(Errc::Overflow, "segment span exceeds the 64-bit value range");
    span_ = 6 * segment_wheel_len * std::max<uint64_t>(1, segments_per_refill);
    if (span_ / 6 / segments_per_refill != segment_wheel_len) span_ = 6 * segment_wheel_len;
  }

  std::optional<uint64_t> next() {
    if (prelude_ < 2) return prelude_++ == 0 ? 2 : 3;
    while (pos_ == buf_.size()) {
      if (overflowed_) return std::nullopt;
      refill();
    }
    return buf_[pos_++];
  }
  bool overflowed() const { return overflowed_; }
  uint64_t segment_wheel_len() const { return wheel_len_; }

  static bool segment_would_overflow(uint64_t start, uint64_t wheel_len) {  // stream.cpp:24-26
    return start >= kMaxSegmentEnd || wheel_len > (kMaxSegmentEnd - start) / 6;
  }

 private:
  void refill() {
    if (segment_would_overflow(next_start_, wheel_len_)) {
      overflowed_ = true;
      return;
    }
    uint64_t end = next_start_ + span_;
    if (segment_would_overflow(next_start_, span_ / 6)) {
      end = next_start_ + 6 * wheel_len_ * ((kMaxSegmentEnd - next_start_) / (6 * wheel_len_));
    }
    buf_ = dev_.enumerate_range(std::max<uint64_t>(next_start_, 4), end);
    pos_ = 0;
    next_start_ = end;
  }

  Device& dev_;
  uint64_t wheel_len_;
  uint64_t span_ = 0;
  uint64_t next_start_ = 0;
  std::vector<uint64_t> buf_;
  size_t pos_ = 0;
  uint8_t prelude_ = 0;
  bool overflowed_ = false;
};

// --------------------------------------------------------------- engine ----
enum class FlagWidth : uint8_t { Bit, Byte, Word4 };  // segment.hpp:20

constexpr uint64_t flag_payload_bytes(uint64_t count, FlagWidth width) {  // segment.hpp:23-30
  switch (width) {
    case FlagWidth::Bit: return (count + 7) / 8;
    case FlagWidth::Byte: return count;
    case FlagWidth::Word4: return 4 * count;
  }
  return 0;
}

struct SieveConfig {  // engine.hpp:13-29
  std::optional<uint64_t> limit;
  unsigned threads = 1;
  uint64_t segment_span = 6'000'000;
  FlagWidth flag_width = FlagWidth::Bit;
  PrimeSink* sink = nullptr;
  bool spawn_per_iteration = false;
  unsigned thread_cap = 1024;
};

struct WorkerAssignment {  // engine.hpp:34-40
  uint64_t iteration;
  unsigned worker;
  uint64_t lo;
  uint64_t hi;
  bool operator==(const WorkerAssignment&) const = default;
};

struct SieveReport {  // engine.hpp:42-55
  uint64_t prime_count = 0;
  uint64_t largest_prime = 0;
  uint64_t iterations = 0;
  double wall_ms = 0.0;
  uint64_t peak_flag_bytes = 0;
  uint64_t peak_flag_entries = 0;
  uint64_t sieved_to = 0;
  bool stopped = false;
  bool overflowed = false;
};

class SinkFailure : public Error {  // engine.hpp:59-67
 public:
  SinkFailure(Errc code, const std::string& what, SieveReport partial)
      : Error(code, what), partial_(partial) {}
  const SieveReport& partial() const { return partial_; }

 private:
  SieveReport partial_;
};

inline uint64_t round_segment_span(uint64_t span, unsigned threads) {  // engine.cpp:311-320
  if (threads == 0) throw Error(Errc::BadConfig, "thread count must be positive");
  const uint64_t align = 6ull * threads;
  if (span == 0) return align;
  if (span % align == 0) return span;
  if (span > UINT64_MAX - align)
    throw Error(Errc::Overflow, "segment span exceeds the 64-bit value range");
  return (span / align + 1) * align;
}

inline std::vector<WorkerAssignment> plan_iteration(const SieveConfig& config,
                                                    uint64_t iteration) {  // engine.cpp:322-342
  if (config.threads == 0 || config.threads > config.thread_cap)
    throw Error(Errc::BadConfig, "invalid thread count");
  const uint64_t span = config.segment_span;
  const uint64_t align = 6ull * config.threads;
  if (span == 0 || span % align != 0 || span > kMaxSegmentEnd)
    throw Error(Errc::BadConfig, "segment span " + std::to_string(span) +
                                     " is not a positive multiple of " + std::to_string(align));
  if (iteration > kMaxSegmentEnd / span - 1)
    throw Error(Errc::Overflow, "iteration " + std::to_string(iteration) +
                                    " leaves the 64-bit value range");
  const uint64_t sub = span / config.threads;
  std::vector<WorkerAssignment> plan;
  plan.reserve(config.threads);
  for (unsigned j = 0; j < config.threads; ++j) {
    const uint64_t lo = iteration * span + j * sub;
    plan.push_back({iteration, j, lo, lo + sub});
  }
  return plan;
}

namespace detail {

inline void validate(const SieveConfig& config, bool bounded) {  // engine.cpp:119-143
  if (config.sink == nullptr) throw Error(Errc::BadConfig, "config has no sink");
  if (config.threads == 0) throw Error(Errc::BadConfig, "thread count must be positive");
  if (config.threads > config.thread_cap)
    throw Error(Errc::BadConfig, "thread count " + std::to_string(config.threads) +
                                     " exceeds the cap " + std::to_string(config.thread_cap));
  const uint64_t align = 6ull * config.threads;
  if (config.segment_span == 0 || config.segment_span % align != 0)
    throw Error(Errc::BadConfig, "segment span " + std::to_string(config.segment_span) +
                                     " is not a positive multiple of " + std::to_string(align));
  if (config.segment_span > kMaxSegmentEnd)
    throw Error(Errc::BadConfig, "segment span exceeds the 64-bit value range");
  if (bounded) {
    if (!config.limit) throw Error(Errc::BadConfig, "bounded run requires a limit");
    if (*config.limit < 2) throw Error(Errc::EmptyRange, "no primes below 2");
    if (*config.limit > kMaxSegmentEnd - 1)
      throw Error(Errc::Overflow, "limit exceeds the sievable 64-bit range");
  } else if (config.limit) {
    throw Error(Errc::BadConfig, "unbounded run cannot take a limit");
  }
}

// Analytic flag-storage accounting of the widest iteration (engine.cpp:218-230).
inline void account(const SieveConfig& config, uint64_t seg_lo, uint64_t seg_hi,
                    SieveReport& rep) {
  const uint64_t sub = config.segment_span / config.threads;
  uint64_t entries = 0, bytes = 0;
  for (unsigned j = 0; j < config.threads; ++j) {
    const uint64_t lo = seg_lo + j * sub;
    if (lo >= seg_hi) break;
    const uint64_t hi = sub > seg_hi - lo ? seg_hi : lo + sub;
    const uint64_t len = (hi - lo) / 6;
    entries += 2 * len;
    bytes += 2 * flag_payload_bytes(len, config.flag_width);
  }
  rep.peak_flag_entries = std::max(rep.peak_flag_entries, entries);
  rep.peak_flag_bytes = std::max(rep.peak_flag_bytes, bytes);
}

// Values per device call when emitting into a value sink.
inline constexpr uint64_t kChunkValues = uint64_t{1} << 28;

inline SieveReport run_loop(const SieveConfig& config, const std::atomic<bool>* stop,
                            Device& dev) {
  validate(config, stop == nullptr);
  PrimeSink& sink = *config.sink;
  const auto t0 = std::chrono::steady_clock::now();
  const bool bounded = stop == nullptr;
  const uint64_t span = config.segment_span;
  const uint64_t limit = bounded ? *config.limit : 0;
  const uint64_t limit_end = bounded ? (limit / 6 + 1) * 6 : kMaxSegmentEnd;  // engine.cpp:160
  const uint64_t total_iterations = bounded ? limit_end / span + (limit_end % span != 0) : 0;
  SieveReport rep;
  auto finish = [&] {
    rep.wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  const bool want_values = sink.wants_values();
  // iterations per device call
  const uint64_t per_call = std::max<uint64_t>(1, kChunkValues / span);
  std::vector<uint64_t> vals;
  uint64_t vpos = 0;
  bool prelude_pending = true;
  uint64_t count_total = 0, count_largest = 0;
  if (bounded && !want_values) {
    // count-only: one device pass over [0, limit] (engine.cpp:252-253 per tile)
    const Checks c = dev.count_range(0, limit + 1);
    count_total = c.count;
    count_largest = c.largest;
  }
  try {
    for (uint64_t i = 0, seg_lo = 0;; ++i, seg_lo += span) {
      if (bounded && i >= total_iterations) break;
      if (stop && stop->load(std::memory_order_acquire)) {
        rep.stopped = true;
        break;
      }
      if (!bounded && seg_lo > kMaxSegmentEnd - span) {
        rep.overflowed = true;
        break;
      }
      const uint64_t seg_hi = (bounded && span > limit_end - seg_lo) ? limit_end : seg_lo + span;
      account(config, seg_lo, seg_hi, rep);
      if (prelude_pending) {  // engine.cpp:268-276
        prelude_pending = false;
        static constexpr uint64_t kPrelude[2] = {2, 3};
        const size_t n = (!bounded || limit >= 3) ? 2 : 1;
        if (want_values)
          sink.emit({kPrelude, n});
        else
          sink.emit_count(n, kPrelude[n - 1]);
      }
      if (want_values) {
        if (i % per_call == 0) {  // sieve the next block of iterations on the device
          const uint64_t blo = std::max<uint64_t>(seg_lo, 4);
          uint64_t bhi = seg_lo + std::min<uint64_t>(per_call, (kMaxSegmentEnd - seg_lo) / span) * span;
          if (bounded) bhi = std::min(bhi, limit + 1);
          vals = blo < bhi ? dev.enumerate_range(blo, bhi) : std::vector<uint64_t>{};
          vpos = 0;
        }
        const uint64_t top = bounded ? std::min(seg_hi, limit + 1) : seg_hi;
        const uint64_t end =
            std::lower_bound(vals.begin() + vpos, vals.end(), top) - vals.begin();
        if (end > vpos) sink.emit({vals.data() + vpos, end - vpos});
        vpos = end;
      } else if (bounded && i + 1 == total_iterations && count_total > 2) {
        sink.emit_count(count_total - std::min<uint64_t>(2, count_total), count_largest);
      } else if (!bounded) {
        const Checks c = dev.count_range(std::max<uint64_t>(seg_lo, 4), seg_hi);
        if (c.count) sink.emit_count(c.count, c.largest);
      }
      rep.iterations = i + 1;
      rep.sieved_to = seg_hi;
    }
  } catch (const Error& e) {
    if (e.code() == Errc::Cuda || e.code() == Errc::NoDevice || e.code() == Errc::OutOfMemory)
      throw;
    rep.prime_count = sink.count();
    rep.largest_prime = sink.largest();
    finish();
    throw SinkFailure(e.code(), e.what(), rep);
  }
  if (bounded) rep.sieved_to = limit + 1;
  rep.prime_count = sink.count();
  rep.largest_prime = sink.largest();
  finish();
  return rep;
}

}  // namespace detail

// engine.hpp:83 on the GPU.
inline SieveReport run(const SieveConfig& config, Device& dev) {
  return detail::run_loop(config, nullptr, dev);
}
inline SieveReport run(const SieveConfig& config) {
  Device dev;
  return run(config, dev);
}

// engine.hpp:89 on the GPU.
inline SieveReport run_unbounded(const SieveConfig& config, const std::atomic<bool>& stop,
                                 Device& dev) {
  return detail::run_loop(config, &stop, dev);
}
inline SieveReport run_unbounded(const SieveConfig& config, const std::atomic<bool>& stop) {
  Device dev;
  return run_unbounded(config, stop, dev);
}

}  // namespace wheelsieve::gpu
