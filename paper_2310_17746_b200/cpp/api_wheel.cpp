// Wheel arithmetic (wheelsieve/wheel.hpp).  Semantics of the reference's
// wheel.cpp:8-106; Table 1 of the paper is used in its k-residue form (the
// same form the device kernels evaluate): a multiple p*k of p = +-1 (mod 6)
// lies in class r exactly when k = r * (p mod 6) (mod 6).
#include <cmath>
#include <string>

#include "wheelsieve/gpu.h"
#include "wheelsieve/wheel.hpp"

namespace wheelsieve {

uint64_t value_of(WheelCoord coord) {
  if (coord.index > kMaxWheelIndex)
    throw Error(Errc::Overflow, "wheel index " + std::to_string(coord.index) +
                                    " is past the last 64-bit wheel value");
  return 6 * coord.index + (coord.residue == ResidueClass::R5 ? 5 : 1);
}

WheelCoord coord_of(uint64_t n) {
  const uint64_t r = n % 6;
  if (r != 1 && r != 5)
    throw Error(Errc::NotOnWheel, std::to_string(n) + " is not coprime to 6");
  return {n / 6, r == 1 ? ResidueClass::R1 : ResidueClass::R5};
}

uint64_t isqrt(uint64_t n) { return ws_isqrt(n); }

uint64_t ceil_sqrt(uint64_t n) {
  const uint64_t r = ws_isqrt(n);
  return r * r == n ? r : r + 1;
}

std::vector<uint64_t> naive_sieve(uint64_t n, uint64_t cap) {
  // The independent checker of the API (not the GPU path): a byte per
  // integer, every prime crossing off from its square.
  if (n < 2) throw Error(Errc::EmptyRange, "there are no primes below 2");
  if (n > cap || n == UINT64_MAX)
    throw Error(Errc::Capacity, "dense sieve bound " + std::to_string(n) + " is above the cap " +
                                    std::to_string(cap));
  std::vector<uint8_t> crossed(n + 1, 0);
  std::vector<uint64_t> primes;
  for (uint64_t i = 2; i <= n; ++i) {
    if (crossed[i]) continue;
    primes.push_back(i);
    if (i <= n / i)
      for (uint64_t j = i * i; j <= n; j += i) crossed[j] = 1;
  }
  return primes;
}

uint64_t greatest_multiple_below(uint64_t p, uint64_t m) {
  if (p == 0 || m <= p)
    throw Error(Errc::Domain, "no positive multiple of " + std::to_string(p) + " lies below " +
                                  std::to_string(m));
  return (m - 1) / p * p;
}

StartOffsets start_offsets_after(uint64_t p, uint64_t anchor) {
  // anchor = p * k0; the next multiple in class r is anchor + c * p with the
  // least c in 1..6 putting it on r, i.e. wheel index
  // anchor / 6 + (anchor % 6 + c * p - r) / 6 (no overflow before the sum).
  const uint64_t q = anchor % 6, pm = p % 6;
  auto next_in = [&](uint64_t r) {
    uint64_t c = 1;
    while ((q + c * pm) % 6 != r) ++c;
    return anchor / 6 + (q + c * p - r) / 6;
  };
  return {next_in(1), next_in(5)};
}

StartOffsets start_offsets(uint64_t p, uint64_t segment_start) {
  if (p % 6 != 1 && p % 6 != 5)
    throw Error(Errc::Domain, std::to_string(p) + " is not coprime to 6");
  if (segment_start % 6 != 0)
    throw Error(Errc::Alignment, "segment start " + std::to_string(segment_start) +
                                     " is not a multiple of 6");
  if (segment_start <= p)
    throw Error(Errc::Domain, "segment start " + std::to_string(segment_start) +
                                  " must exceed the prime " + std::to_string(p));
  return start_offsets_after(p, greatest_multiple_below(p, segment_start));
}

}  // namespace wheelsieve
