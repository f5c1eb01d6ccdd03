// The sieving-prime store, GPU edition (drop-in for the reference's
// wheelsieve/base_store.hpp; semantics of /root/reference/proj/src/base_store.cpp).
//
// The store is a host-side view of the primes 5 <= p <= frontier; they are
// produced on the device (ws_base_primes / ws_enumerate_range), where the
// sieve kernels keep their own resident table.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "wheelsieve/errors.hpp"

namespace wheelsieve {

// A sieving prime and its square, saturated to UINT64_MAX when p * p does
// not fit (such a prime never activates inside the 64-bit range).
struct BasePrime {
  uint64_t value;
  uint64_t square;
};

class BasePrimeStore {
 public:
  // Seeded for sieving up to limit_hint: the primes 5..ceil(sqrt(limit_hint)),
  // sieved on the GPU.  Errc::Domain below 25 (an empty store).
  static BasePrimeStore bootstrap(uint64_t limit_hint);

  // Grows the frontier to at least max(new_frontier, 2 * frontier) -- the
  // geometric policy that keeps repeated small requests cheap -- by sieving
  // the gap on the GPU.  No-op when already covered; Errc::Overflow past the
  // sievable range.
  void extend(uint64_t new_frontier);

  // Appends primes the caller produced: ascending, in (frontier, new_frontier],
  // complete up to new_frontier; values at or below the frontier are skipped.
  // Errc::Domain (beyond the new frontier, or a frontier moving back),
  // Errc::Ordering (not ascending).
  void absorb(std::span<const uint64_t> primes, uint64_t new_frontier);

  uint64_t frontier() const { return frontier_; }
  // frontier >= isqrt(segment_end - 1): enough primes for a segment ending there.
  bool covers(uint64_t segment_end) const;

  std::span<const BasePrime> entries() const { return primes_; }
  size_t size() const { return primes_.size(); }

 private:
  BasePrimeStore() = default;
  void push(uint64_t p, uint64_t bound);

  std::vector<BasePrime> primes_;
  uint64_t frontier_ = 0;
};

}  // namespace wheelsieve
