// Mod-6 wheel arithmetic, GPU edition (drop-in for the reference's
// wheelsieve/wheel.hpp; semantics of /root/reference/proj/src/wheel.cpp).
//
// Only integers coprime to 6 carry sieve flags: 6k+1 (class R1) and 6k+5
// (class R5), k being the wheel index.  These are small host-side pure
// functions; the sieve itself evaluates the same arithmetic on the device
// (libwheelsieve_cuda.so, paper Table 1 in its k-residue form).
#pragma once

#include <cstdint>
#include <vector>

#include "wheelsieve/errors.hpp"

namespace wheelsieve {

enum class ResidueClass : uint8_t { R1, R5 };

// value = 6 * index + (1 or 5); (0, R1) is the non-prime 1, (0, R5) is 5.
struct WheelCoord {
  uint64_t index;
  ResidueClass residue;
  bool operator==(const WheelCoord&) const = default;
};

// Absolute wheel indices of a prime's next multiple in each class.
struct StartOffsets {
  uint64_t id1;  // the 6k+1 multiple
  uint64_t id5;  // the 6k+5 multiple
  bool operator==(const StartOffsets&) const = default;
};

// The largest index whose 6k+5 value fits in 64 bits, and the first
// multiple of 6 past every representable wheel value.
inline constexpr uint64_t kMaxWheelIndex = (UINT64_MAX - 5) / 6;
inline constexpr uint64_t kMaxSegmentEnd = 6 * (kMaxWheelIndex + 1);
// Bound on naive_sieve's dense byte array.
inline constexpr uint64_t kDefaultNaiveCap = 100'000'000;

uint64_t value_of(WheelCoord coord);  // Errc::Overflow past kMaxWheelIndex
WheelCoord coord_of(uint64_t n);      // Errc::NotOnWheel unless n = 1, 5 (mod 6)

uint64_t isqrt(uint64_t n);      // floor(sqrt(n)), exact over all of uint64
uint64_t ceil_sqrt(uint64_t n);  // ceil(sqrt(n)), exact

// The textbook dense sieve of [0, n] (primes from 2 up).  Kept as the
// reference's independent checker: it shares nothing with the GPU path.
// Errc::EmptyRange for n < 2, Errc::Capacity above cap.
std::vector<uint64_t> naive_sieve(uint64_t n, uint64_t cap = kDefaultNaiveCap);

// p * floor((m - 1) / p): the last multiple of p below m (Errc::Domain when
// m <= p).
uint64_t greatest_multiple_below(uint64_t p, uint64_t m);

// Wheel indices of the first multiples of p strictly above `anchor` (a
// multiple of p; p coprime to 6).  Constant time.
StartOffsets start_offsets_after(uint64_t p, uint64_t anchor);

// Wheel indices of the first multiples of p at or beyond segment_start
// (a positive multiple of 6 above p): Errc::Domain / Errc::Alignment.
StartOffsets start_offsets(uint64_t p, uint64_t segment_start);

}  // namespace wheelsieve
