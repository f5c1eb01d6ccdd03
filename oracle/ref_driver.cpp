// TEST INFRASTRUCTURE ONLY (oracle). Never linked into or called by the
// product path; only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it.
//
// extern "C" driver over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libwsref.so).  Every entry point composes the reference's own
// public API exactly as SURVEY.md §3.3 / §8c describe:
//   * prefixes   -> wheelsieve::run()            (engine.hpp:83, engine.cpp:344)
//   * [L, R)     -> BasePrimeStore::bootstrap + SegmentBitmap + sieve_segment
//                   (base_store.cpp:34, segment.cpp:93, segment.cpp:164)
//                   + clear_value(1) when lo == 0 (engine.cpp:244)
//                   + for_each_surviving filtered to [L, R) (segment.hpp:123)
//                   + 2 and 3 when in range (engine.cpp:268-276)
// Status returns: 0 ok, 1 + int(Errc) for a wheelsieve::Error, 99 other.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <thread>
#include <vector>

#include "wheelsieve/base_store.hpp"
#include "wheelsieve/engine.hpp"
#include "wheelsieve/segment.hpp"
#include "wheelsieve/sink.hpp"
#include "wheelsieve/wheel.hpp"

using namespace wheelsieve;

namespace {

// PrimeSink whose accept() (the protected extension point, sink.hpp:38)
// folds every emitted value into Σ mod 2^64 and ⊕.
class ChecksumSink : public PrimeSink {
 public:
  uint64_t sum = 0, xr = 0;

 protected:
  void accept(std::span<const uint64_t> batch) override {
    for (uint64_t v : batch) {
      sum += v;
      xr ^= v;
    }
  }
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    return 1 + static_cast<int>(e.code());
  } catch (...) {
    return 99;
  }
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct RangeAcc {
  uint64_t count = 0, sum = 0, xr = 0, largest = 0;
};

// One 6-aligned segment of the §3.3 composition.  Returns survivors in
// [L, R) (2 and 3 are never on the wheel).
RangeAcc sieve_one(uint64_t lo, uint64_t slots, uint64_t L, uint64_t R,
                   const BasePrimeStore& base, bool want_checks, std::vector<uint64_t>* out) {
  SegmentBitmap seg(lo, slots);
  sieve_segment(seg, base);
  if (lo == 0) seg.clear_value(1);
  RangeAcc a;
  seg.for_each_surviving([&](uint64_t v) {
    if (v < L || v >= R) return;
    ++a.count;
    a.largest = v;
    if (want_checks) {
      a.sum += v;
      a.xr ^= v;
    }
    if (out) out->push_back(v);
  });
  return a;
}

uint64_t nthreads_or_hw(unsigned t) {
  if (t) return t;
  unsigned h = std::thread::hardware_concurrency();
  return h ? h : 1;
}

}  // namespace

extern "C" {

// π over [0, limit] through the reference engine with a CountSink.
// segment_span = round_segment_span(6 * seg_slots * T, T).
int wsref_run_count(uint64_t limit, unsigned threads, uint64_t seg_slots, uint64_t* count,
                    uint64_t* largest, double* wall_ms) {
  return guarded([&] {
    CountSink sink;
    const unsigned t = static_cast<unsigned>(nthreads_or_hw(threads));
    SieveConfig cfg{limit, t, round_segment_span(6 * seg_slots * t, t), FlagWidth::Bit, &sink};
    SieveReport r = run(cfg);
    *count = r.prime_count;
    *largest = r.largest_prime;
    if (wall_ms) *wall_ms = r.wall_ms;
  });
}

// Full enumeration over [0, limit] through run() into a checksum sink.
int wsref_run_checks(uint64_t limit, unsigned threads, uint64_t seg_slots, uint64_t* count,
                     uint64_t* sum, uint64_t* xr, uint64_t* largest, double* wall_ms) {
  return guarded([&] {
    ChecksumSink sink;
    const unsigned t = static_cast<unsigned>(nthreads_or_hw(threads));
    SieveConfig cfg{limit, t, round_segment_span(6 * seg_slots * t, t), FlagWidth::Bit, &sink};
    SieveReport r = run(cfg);
    *count = r.prime_count;
    *sum = sink.sum;
    *xr = sink.xr;
    *largest = r.largest_prime;
    if (wall_ms) *wall_ms = r.wall_ms;
  });
}

// Enumeration over [0, limit] into a caller buffer (MemorySink).
int wsref_run_values(uint64_t limit, unsigned threads, uint64_t seg_slots, uint64_t* out,
                     uint64_t cap, uint64_t* n) {
  return guarded([&] {
    MemorySink sink;
    const unsigned t = static_cast<unsigned>(nthreads_or_hw(threads));
    SieveConfig cfg{limit, t, round_segment_span(6 * seg_slots * t, t), FlagWidth::Bit, &sink};
    run(cfg);
    const auto& p = sink.primes();
    *n = p.size();
    std::memcpy(out, p.data(), std::min<uint64_t>(cap, p.size()) * sizeof(uint64_t));
  });
}

// [L, R) through the per-segment composition, threaded: each
// thread owns its SegmentBitmap, the BasePrimeStore is shared read-only
// (SPEC.md:199).  per_seg (nullable) receives survivor counts per segment
// of seg_slots wheel slots starting at floor(L/6)*6 (2 and 3 excluded).
int wsref_range(uint64_t L, uint64_t R, unsigned threads, uint64_t seg_slots, uint64_t* count,
                uint64_t* sum, uint64_t* xr, uint64_t* largest, uint32_t* per_seg,
                uint64_t per_seg_cap, uint64_t* n_seg, double* wall_ms) {
  return guarded([&] {
    const double t0 = now_ms();
    *count = *sum = *xr = *largest = 0;
    if (n_seg) *n_seg = 0;
    if (R <= L) {
      if (wall_ms) *wall_ms = now_ms() - t0;
      return;
    }
    const uint64_t lo0 = L / 6 * 6;
    const uint64_t total_slots = (R - lo0 + 5) / 6;
    const uint64_t nseg = (total_slots + seg_slots - 1) / seg_slots;
    const uint64_t aligned_end = lo0 + 6 * total_slots;
    const BasePrimeStore base = BasePrimeStore::bootstrap(std::max<uint64_t>(25, aligned_end));
    const uint64_t T = nthreads_or_hw(threads);
    std::vector<RangeAcc> acc(T);
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::atomic<bool> failed{false};
    for (uint64_t t = 0; t < T; ++t)
      pool.emplace_back([&, t] {
        try {
          for (;;) {
            const uint64_t s = next.fetch_add(1);
            if (s >= nseg || failed.load()) break;
            const uint64_t lo = lo0 + 6 * seg_slots * s;
            const uint64_t slots = std::min(seg_slots, total_slots - s * seg_slots);
            RangeAcc a = sieve_one(lo, slots, L, R, base, true, nullptr);
            if (per_seg && s < per_seg_cap) per_seg[s] = static_cast<uint32_t>(a.count);
            acc[t].count += a.count;
            acc[t].sum += a.sum;
            acc[t].xr ^= a.xr;
            acc[t].largest = std::max(acc[t].largest, a.largest);
          }
        } catch (...) {
          failed = true;
          err = std::current_exception();
        }
      });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
    for (const RangeAcc& a : acc) {
      *count += a.count;
      *sum += a.sum;
      *xr ^= a.xr;
      *largest = std::max(*largest, a.largest);
    }
    for (uint64_t v : {uint64_t{2}, uint64_t{3}})
      if (v >= L && v < R) {
        *count += 1;
        *sum += v;
        *xr ^= v;
        *largest = std::max(*largest, v);
      }
    if (n_seg) *n_seg = nseg;
    if (wall_ms) *wall_ms = now_ms() - t0;
  });
}

// Sorted values of [L, R) via the composition (single thread, small ranges).
int wsref_range_values(uint64_t L, uint64_t R, uint64_t seg_slots, uint64_t* out, uint64_t cap,
                       uint64_t* n) {
  return guarded([&] {
    std::vector<uint64_t> vals;
    for (uint64_t v : {uint64_t{2}, uint64_t{3}})
      if (v >= L && v < R) vals.push_back(v);
    if (R > L) {
      const uint64_t lo0 = L / 6 * 6;
      const uint64_t total_slots = (R - lo0 + 5) / 6;
      const uint64_t aligned_end = lo0 + 6 * total_slots;
      const BasePrimeStore base =
          BasePrimeStore::bootstrap(std::max<uint64_t>(25, aligned_end));
      for (uint64_t s = 0; s * seg_slots < total_slots; ++s) {
        const uint64_t lo = lo0 + 6 * seg_slots * s;
        const uint64_t slots = std::min(seg_slots, total_slots - s * seg_slots);
        sieve_one(lo, slots, L, R, base, false, &vals);
      }
    }
    *n = vals.size();
    std::memcpy(out, vals.data(), std::min<uint64_t>(cap, vals.size()) * sizeof(uint64_t));
  });
}

// Batch of intervals [Ls[i], Ls[i] + width): one shared base store
// bootstrapped past the largest end, intervals distributed over threads.
int wsref_intervals(const uint64_t* Ls, uint64_t n, uint64_t width, unsigned threads,
                    uint64_t seg_slots, uint32_t* counts, uint64_t* sums, uint64_t* xors,
                    double* wall_ms) {
  return guarded([&] {
    const double t0 = now_ms();
    uint64_t max_end = 25;
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t lo0 = Ls[i] / 6 * 6;
      const uint64_t slots = (Ls[i] + width - lo0 + 5) / 6;
      max_end = std::max(max_end, lo0 + 6 * slots);
    }
    const BasePrimeStore base = BasePrimeStore::bootstrap(max_end);
    const uint64_t T = nthreads_or_hw(threads);
    std::atomic<uint64_t> next{0};
    std::exception_ptr err;
    std::vector<std::thread> pool;
    for (uint64_t t = 0; t < T; ++t)
      pool.emplace_back([&] {
        try {
          for (;;) {
            const uint64_t i = next.fetch_add(1);
            if (i >= n) break;
            const uint64_t L = Ls[i], R = Ls[i] + width;
            const uint64_t lo0 = L / 6 * 6;
            const uint64_t total_slots = (R - lo0 + 5) / 6;
            RangeAcc tot;
            for (uint64_t s = 0; s * seg_slots < total_slots; ++s) {
              const uint64_t lo = lo0 + 6 * seg_slots * s;
              const uint64_t slots = std::min(seg_slots, total_slots - s * seg_slots);
              RangeAcc a = sieve_one(lo, slots, L, R, base, true, nullptr);
              tot.count += a.count;
              tot.sum += a.sum;
              tot.xr ^= a.xr;
            }
            for (uint64_t v : {uint64_t{2}, uint64_t{3}})
              if (v >= L && v < R) {
                ++tot.count;
                tot.sum += v;
                tot.xr ^= v;
              }
            counts[i] = static_cast<uint32_t>(tot.count);
            sums[i] = tot.sum;
            if (xors) xors[i] = tot.xr;
          }
        } catch (...) {
          err = std::current_exception();
        }
      });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
    if (wall_ms) *wall_ms = now_ms() - t0;
  });
}

// Table 1 probe: start_offsets(p, segment_start) (wheel.cpp:96-106).
int wsref_start_offsets(uint64_t p, uint64_t segment_start, uint64_t* id1, uint64_t* id5) {
  return guarded([&] {
    StartOffsets o = start_offsets(p, segment_start);
    *id1 = o.id1;
    *id5 = o.id5;
  });
}

// naive_sieve(n) (wheel.cpp:40-54) into a caller buffer.
int wsref_naive_sieve(uint64_t n, uint64_t* out, uint64_t cap, uint64_t* count) {
  return guarded([&] {
    std::vector<uint64_t> v = naive_sieve(n);
    *count = v.size();
    std::memcpy(out, v.data(), std::min<uint64_t>(cap, v.size()) * sizeof(uint64_t));
  });
}

// BasePrimeStore::bootstrap(hint) (base_store.cpp:34-42): entries and frontier.
int wsref_bootstrap(uint64_t hint, uint64_t* out, uint64_t cap, uint64_t* n, uint64_t* frontier) {
  return guarded([&] {
    BasePrimeStore b = BasePrimeStore::bootstrap(hint);
    *n = b.size();
    *frontier = b.frontier();
    uint64_t i = 0;
    for (const BasePrime& e : b.entries())
      if (i < cap) out[i++] = e.value;
  });
}

// SegmentBitmap(start, len) + sieve_segment with a store bootstrapped past
// the segment end: the raw FlagArray words of both classes (segment.hpp:75).
int wsref_sieve_segment(uint64_t start, uint64_t len, uint64_t* r1, uint64_t* r5) {
  return guarded([&] {
    const BasePrimeStore base =
        BasePrimeStore::bootstrap(std::max<uint64_t>(25, start + 6 * len));
    SegmentBitmap seg(start, len);
    sieve_segment(seg, base);
    auto w1 = seg.marks(ResidueClass::R1).bit_words();
    auto w5 = seg.marks(ResidueClass::R5).bit_words();
    std::memcpy(r1, w1.data(), w1.size() * 8);
    std::memcpy(r5, w5.data(), w5.size() * 8);
  });
}

// The reference CLI's store path (tools/wheelsieve.cpp:139-168): run() over
// [0, limit] into a ChunkedFileSink, set_frontier(sieved_to), flush.
int wsref_store_run(uint64_t limit, unsigned threads, const char* dir, int binary,
                    uint64_t primes_per_file) {
  return guarded([&] {
    ChunkedFileSink sink(ChunkedFileOptions{dir, primes_per_file,
                                            binary ? FileFormat::Binary : FileFormat::Text});
    const unsigned t = static_cast<unsigned>(nthreads_or_hw(threads));
    SieveConfig cfg{limit, t, round_segment_span(6 * (1u << 18) * t, t), FlagWidth::Bit, &sink};
    const SieveReport r = run(cfg);
    sink.set_frontier(r.sieved_to);
    sink.flush();
  });
}

int wsref_read_back(const char* dir, uint64_t lo, uint64_t hi, uint64_t* out, uint64_t cap,
                    uint64_t* n) {
  return guarded([&] {
    const std::vector<uint64_t> v = read_back(dir, lo, hi);
    *n = v.size();
    std::memcpy(out, v.data(), std::min<uint64_t>(cap, v.size()) * 8);
  });
}

int wsref_verify_store(const char* dir) {
  return guarded([&] { verify_store(dir); });
}

unsigned wsref_hw_threads(void) { return static_cast<unsigned>(nthreads_or_hw(0)); }

}  // extern "C"
