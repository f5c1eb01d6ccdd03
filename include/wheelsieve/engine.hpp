// The sieve engine, GPU edition (drop-in for the reference's
// wheelsieve/engine.hpp; semantics of /root/reference/proj/src/engine.cpp).
//
// run() keeps the reference's observable behaviour -- validation order and
// error codes, the iteration / worker-tile structure of segment_span and
// threads, the emission sequence (2 and 3 first, then one batch per
// non-empty worker tile in worker order: emit(values) for value sinks,
// emit_count(count, largest) for count sinks), SinkFailure's partial report
// and the analytic flag accounting -- while the sieving runs on the GPU(s)
// of a wheelsieve::gpu::Context: a block of iterations per device call
// (every tile of the block counted as one ws_count_ranges batch, or one
// ordered ws_enumerate_range cut at the tile borders).  The stop flag is
// still checked between iterations and every sink sees exactly the
// reference's batches.  `threads` shapes the tiles; the parallelism is the
// context's devices (wheelsieve/gpu.hpp).
#pragma once

#include <atomic>
#include <cstdint>
#include <optional>
#include <vector>

#include "wheelsieve/segment.hpp"
#include "wheelsieve/sink.hpp"

namespace wheelsieve {

struct SieveConfig {
  std::optional<uint64_t> limit;          // inclusive bound; nullopt = unbounded
  unsigned threads = 1;                   // worker tiles per iteration
  uint64_t segment_span = 6'000'000;      // values per iteration, a multiple of 6 * threads
  FlagWidth flag_width = FlagWidth::Bit;  // footprint accounting only
  PrimeSink* sink = nullptr;
  bool spawn_per_iteration = false;       // accepted for compatibility (no host workers)
  unsigned thread_cap = 1024;             // threads above this are rejected
};

// Worker `worker`'s tile [lo, hi) of iteration `iteration`.
struct WorkerAssignment {
  uint64_t iteration;
  unsigned worker;
  uint64_t lo;
  uint64_t hi;
  bool operator==(const WorkerAssignment&) const = default;
};

struct SieveReport {
  uint64_t prime_count = 0;
  uint64_t largest_prime = 0;
  uint64_t iterations = 0;
  double wall_ms = 0.0;
  uint64_t peak_flag_bytes = 0;    // widest iteration, all tiles (analytic)
  uint64_t peak_flag_entries = 0;
  uint64_t sieved_to = 0;          // exclusive bound fully emitted
  bool stopped = false;            // run_unbounded honoured the stop flag
  bool overflowed = false;         // ran into the end of the 64-bit range
};

// A sink failure mid-run, with the totals that had been emitted before it.
class SinkFailure : public Error {
 public:
  SinkFailure(Errc code, const std::string& what, SieveReport partial)
      : Error(code, what), partial_(partial) {}
  const SieveReport& partial() const { return partial_; }

 private:
  SieveReport partial_;
};

// span rounded up to a multiple of 6 * threads (6 * threads for span 0).
uint64_t round_segment_span(uint64_t span, unsigned threads);

// The tiles of one iteration (pure).  Errc::BadConfig / Errc::Overflow.
std::vector<WorkerAssignment> plan_iteration(const SieveConfig& config, uint64_t iteration);

// 2, 3 and every wheel prime <= *config.limit into config.sink, on
// wheelsieve::gpu::default_context().
SieveReport run(const SieveConfig& config);

// Until `stop` is seen between iterations (the current one completes and
// emits) or the 64-bit range ends; config.limit must be nullopt.
SieveReport run_unbounded(const SieveConfig& config, const std::atomic<bool>& stop);

}  // namespace wheelsieve
