// wheelsieve::gpu -- the GPU-specific half of the C++ API (libwheelsieve.so,
// layered on the C ABI of wheelsieve/gpu.h).
//
// The reference's own interface -- Errc/Error, the sinks, SieveConfig /
// SieveReport / run / run_unbounded, PrimeStream, BasePrimeStore,
// SegmentBitmap / sieve_segment and the wheel functions -- lives in the
// reference-named headers next to this one (errors.hpp, sink.hpp, engine.hpp,
// stream.hpp, base_store.hpp, segment.hpp, wheel.hpp), implemented by this
// library: a reference caller switches by compiling against these headers
// and linking -lwheelsieve instead of the CPU library, subclasses of
// wheelsieve::PrimeSink included.
//
// This header adds what has no reference counterpart:
//   * Context: a device context -- one GPU, or several GPUs of this process
//     (and optionally of other processes) with NCCL communicators, where one
//     call is split into contiguous per-device super-ranges and the per-shard
//     records are combined by one ncclAllGather (SieveConfig::threads spreads
//     a reference run over CPU workers; a Context spreads it over GPUs);
//   * the [L, R) entry points the reference composes by hand (count_range,
//     enumerate_range, count_intervals, count_ranges) as single calls;
//   * default_context(): the context run(), sieve_segment() and the
//     stream use -- the current device, or every device listed in
//     WHEELSIEVE_DEVICES ("0,1,2,3" or "all") as one NCCL context.
#pragma once

#include <atomic>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "wheelsieve/engine.hpp"
#include "wheelsieve/errors.hpp"
#include "wheelsieve/gpu.h"

namespace wheelsieve::gpu {

// ws_status -> wheelsieve::Error (status = 1 + Errc); ctx (nullable) adds
// ws_last_error's message.
void check(ws_status status, const ws_ctx* ctx, const char* what);

struct Checks {
  uint64_t count = 0, sum = 0, xr = 0, largest = 0;
  bool operator==(const Checks&) const = default;
};

struct ContextOptions {
  std::vector<int> devices;           // empty: one device (`device`), no NCCL
  int device = -1;                    // -1: the calling thread's current device
  uint32_t segment_slots = 1u << 18;  // power of two in [2^12, 2^18]
  uint32_t world = 1;                 // processes sharing each call (NCCL)
  uint32_t rank = 0;
  std::string nccl_id;                // world > 1: nccl_unique_id() of rank 0
};

// A fresh ncclUniqueId (WS_NCCL_ID_BYTES bytes) to broadcast to the ranks.
std::string nccl_unique_id();

class Context {
 public:
  Context() : Context(ContextOptions{}) {}
  explicit Context(int device, uint32_t segment_slots = 1u << 18);
  explicit Context(const ContextOptions& options);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  ws_ctx* handle() { return ctx_; }
  uint32_t segment_slots() const { return slots_; }
  uint32_t num_devices() const { return ws_ctx_num_devices(ctx_); }
  uint32_t num_shards() const { return ws_ctx_num_shards(ctx_); }
  ws_timing timing() const;

  Checks count_range(uint64_t L, uint64_t R, bool checksums = false,
                     std::vector<uint32_t>* per_segment = nullptr);
  std::vector<uint64_t> enumerate_range(uint64_t L, uint64_t R, Checks* checks = nullptr);
  std::vector<Checks> count_ranges(std::span<const uint64_t> Ls, std::span<const uint64_t> Rs,
                                   bool checksums = false);
  void count_intervals(std::span<const uint64_t> Ls, uint64_t width, std::vector<uint32_t>& counts,
                       std::vector<uint64_t>* sums = nullptr,
                       std::vector<uint64_t>* xors = nullptr);
  // BasePrimeStore::bootstrap's entries: the wheel primes 5 <= p <= B.
  std::vector<uint64_t> base_primes(uint64_t B);
  // The two flag arrays of a sieved segment, FlagArray Bit layout (value 1 left set).
  void sieve_segment_words(uint64_t start, uint64_t len, uint64_t* r1_words, uint64_t* r5_words);
  // ChunkedFileSink-format store of [L, R) (frontier R), streamed in windows.
  uint64_t store_range(uint64_t L, uint64_t R, const std::string& dir, bool binary,
                       uint64_t primes_per_file = 125'000'000);

 private:
  ws_ctx* ctx_ = nullptr;
  uint32_t slots_ = 1u << 18;
};

// The context behind run(), run_unbounded(), sieve_segment(), PrimeStream
// and BasePrimeStore: created on first use (WHEELSIEVE_DEVICES or the
// current device) unless set_default_context() installed one.
Context& default_context();
void set_default_context(Context* ctx);  // nullptr: back to the lazily created one

SieveReport run(const SieveConfig& config, Context& ctx);
SieveReport run_unbounded(const SieveConfig& config, const std::atomic<bool>& stop, Context& ctx);

}  // namespace wheelsieve::gpu
