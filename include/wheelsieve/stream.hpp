// Unbounded prime enumeration, GPU edition (drop-in for the reference's
// wheelsieve/stream.hpp; semantics of /root/reference/proj/src/stream.cpp).
//
// next() yields 2, 3 and then every wheel prime in ascending order, without
// an upper bound fixed in advance.  Each refill enumerates a block of
// segments of segment_wheel_len slots on the GPU (bounded to ~2^28 values,
// never less than one segment) -- the same sequence the reference's
// one-segment refills produce -- and base() grows with the stream as the
// reference's store does.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "wheelsieve/base_store.hpp"
#include "wheelsieve/segment.hpp"

namespace wheelsieve {

class PrimeStream {
 public:
  // Errc::Domain for 0, Errc::Overflow if one segment leaves the 64-bit range.
  explicit PrimeStream(uint64_t segment_wheel_len, FlagWidth width = FlagWidth::Bit);

  // nullopt once the 64-bit range is exhausted (then overflowed() is true).
  std::optional<uint64_t> next();

  bool overflowed() const { return overflowed_; }
  uint64_t segment_wheel_len() const { return len_; }
  const BasePrimeStore& base() const { return base_; }

  static bool segment_would_overflow(uint64_t segment_start, uint64_t wheel_len);

 private:
  void refill();

  uint64_t len_;
  FlagWidth width_;
  BasePrimeStore base_;
  uint64_t next_ = 0;
  std::vector<uint64_t> buf_;
  size_t pos_ = 0;
  uint8_t prelude_ = 0;
  bool overflowed_ = false;
};

}  // namespace wheelsieve
