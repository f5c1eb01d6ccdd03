// Segment containers and the GPU per-segment sieve (wheelsieve/segment.hpp);
// container semantics of the reference's segment.cpp:12-162.
#include <algorithm>
#include <bit>
#include <string>

#include "wheelsieve/base_store.hpp"
#include "wheelsieve/gpu.hpp"
#include "wheelsieve/segment.hpp"

namespace wheelsieve {

namespace {

uint64_t words_for(uint64_t size, FlagWidth width) {
  return (flag_payload_bytes(size, width) + 7) / 8;
}

}  // namespace

FlagArray::FlagArray(uint64_t size, FlagWidth width)
    : size_(size), width_(width), words_(words_for(size, width)) {
  fill_true();
}

void FlagArray::fill_true() {
  if (width_ != FlagWidth::Bit) {
    std::fill(words_.begin(), words_.end(), 0);
    if (width_ == FlagWidth::Byte)
      std::fill(byte_data(), byte_data() + size_, uint8_t{1});
    else
      std::fill(u32_data(), u32_data() + size_, uint32_t{1});
    return;
  }
  std::fill(words_.begin(), words_.end(), ~uint64_t{0});
  if (size_ % 64 && !words_.empty()) words_.back() = (uint64_t{1} << (size_ % 64)) - 1;
}

void FlagArray::clear_stride(uint64_t first, uint64_t step) {
  if (step == 0) throw Error(Errc::Domain, "stride must be positive");
  for (uint64_t i = first; i < size_; i += step) clear(i);
}

uint64_t FlagArray::count_true() const {
  uint64_t n = 0;
  if (width_ == FlagWidth::Bit) {
    for (uint64_t w : words_) n += static_cast<uint64_t>(std::popcount(w));
  } else {
    for (uint64_t i = 0; i < size_; ++i) n += test(i);
  }
  return n;
}

std::optional<uint64_t> FlagArray::last_true() const {
  if (width_ == FlagWidth::Bit) {
    for (size_t w = words_.size(); w-- > 0;)
      if (words_[w]) return (uint64_t{w} << 6) + 63 - std::countl_zero(words_[w]);
    return std::nullopt;
  }
  for (uint64_t i = size_; i-- > 0;)
    if (test(i)) return i;
  return std::nullopt;
}

void FlagArray::keep_only(std::span<const uint64_t> bits) {
  if (width_ == FlagWidth::Bit) {
    for (size_t w = 0; w < words_.size() && w < bits.size(); ++w) words_[w] &= bits[w];
    return;
  }
  for (uint64_t i = 0; i < size_; ++i)
    if (!((bits[i >> 6] >> (i & 63)) & 1u)) clear(i);
}

SegmentBitmap::SegmentBitmap(uint64_t segment_start, uint64_t wheel_len, FlagWidth width)
    : start_(segment_start),
      len_(wheel_len),
      width_(width),
      one_((segment_start % 6 || wheel_len == 0 ||
            wheel_len > (kMaxSegmentEnd - std::min(segment_start, kMaxSegmentEnd)) / 6)
               ? 0
               : wheel_len,
           width),
      five_(one_.size(), width) {
  if (segment_start % 6 != 0)
    throw Error(Errc::Alignment, "segment start " + std::to_string(segment_start) +
                                     " is not a multiple of 6");
  if (wheel_len == 0) throw Error(Errc::Domain, "a segment needs at least one wheel slot");
  if (segment_start >= kMaxSegmentEnd || wheel_len > (kMaxSegmentEnd - segment_start) / 6)
    throw Error(Errc::Overflow, "segment end is past the 64-bit value range");
}

uint64_t SegmentBitmap::slot_of(uint64_t value, ResidueClass* r) const {
  const WheelCoord c = coord_of(value);
  if (value < start_ || c.index - first_index() >= len_)
    throw Error(Errc::Domain, std::to_string(value) + " lies outside the segment");
  *r = c.residue;
  return c.index - first_index();
}

bool SegmentBitmap::flag_for(uint64_t value) const {
  ResidueClass r;
  const uint64_t k = slot_of(value, &r);
  return marks(r).test(k);
}

void SegmentBitmap::clear_value(uint64_t value) {
  ResidueClass r;
  const uint64_t k = slot_of(value, &r);
  marks(r).clear(k);
}

void SegmentBitmap::clear_values_above(uint64_t bound) {
  if (bound >= end_value()) return;
  // slot k of class c holds start + 6k + c: cleared once that exceeds bound
  for (const auto& [cls, res] : {std::pair{ResidueClass::R1, 1u}, std::pair{ResidueClass::R5, 5u}}) {
    FlagArray& f = marks(cls);
    const uint64_t first =
        bound < start_ + res ? 0 : (bound - start_ - res) / 6 + 1;  // first slot above bound
    for (uint64_t k = first; k < len_; ++k) f.clear(k);
  }
}

uint64_t SegmentBitmap::count_surviving() const { return one_.count_true() + five_.count_true(); }

std::optional<uint64_t> SegmentBitmap::last_surviving() const {
  const auto a = one_.last_true(), b = five_.last_true();
  if (!a && !b) return std::nullopt;
  const uint64_t va = a ? start_ + 6 * *a + 1 : 0, vb = b ? start_ + 6 * *b + 5 : 0;
  return std::max(va, vb);
}

std::vector<uint64_t> SegmentBitmap::surviving() const {
  std::vector<uint64_t> out;
  for_each_surviving([&](uint64_t v) { out.push_back(v); });
  return out;
}

void sieve_segment(SegmentBitmap& segment, const BasePrimeStore& base) {
  if (!base.covers(segment.end_value()))
    throw Error(Errc::IncompleteBase,
                "base primes reach " + std::to_string(base.frontier()) + ", the segment ending at " +
                    std::to_string(segment.end_value()) + " needs isqrt(end - 1) = " +
                    std::to_string(isqrt(segment.end_value() - 1)));
  const uint64_t nw = (segment.wheel_len() + 63) / 64;
  std::vector<uint64_t> r1(nw), r5(nw);
  gpu::default_context().sieve_segment_words(segment.segment_start(), segment.wheel_len(),
                                             r1.data(), r5.data());
  segment.marks(ResidueClass::R1).keep_only(r1);
  segment.marks(ResidueClass::R5).keep_only(r5);
}

}  // namespace wheelsieve
