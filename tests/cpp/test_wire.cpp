// Host wire-format expander (paper_2310_17746_b200/csrc/ws_wire.cpp) against a
// direct widening of every entry: random segments of random block counts
// (empty blocks, full-range counts, realistic ~35-entry blocks), every output
// alignment, partial ranges (skip, n) and pooled splits with tickets.  Run
// with the AVX-512+IFMA path, WHEELSIEVE_HOST_NO_IFMA=1 and
// WHEELSIEVE_HOST_SCALAR=1.
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "ws_wire.h"

namespace {

struct Case {
  std::vector<uint8_t> cnt, e;
  std::vector<uint64_t> seg_off, want;
  wswire::WireChunk ch{};
};

Case make_case(std::mt19937_64& rng, uint64_t nseg, uint64_t bps, uint64_t slot0, int flavour) {
  Case c;
  c.seg_off.push_back(0);
  for (uint64_t s = 0; s < nseg; ++s) {
    for (uint64_t b = 0; b < bps; ++b) {
      uint32_t k;
      if (flavour == 0) k = rng() % 5 == 0 ? 0 : rng() % 256;
      else if (flavour == 1) k = 25 + rng() % 21;
      else k = rng() % 3;
      c.cnt.push_back(static_cast<uint8_t>(k));
      const uint64_t blk = s * bps + b;
      for (uint32_t i = 0; i < k; ++i) {
        const uint8_t x = static_cast<uint8_t>(rng());
        c.e.push_back(x);
        c.want.push_back(6 * (slot0 + blk * wswire::kBlockSlots) + 3 * uint64_t{x} + 1 + (x & 1));
      }
    }
    c.seg_off.push_back(c.e.size());
  }
  c.e.resize(c.e.size() + 64);
  c.ch = wswire::WireChunk{c.cnt.data(), c.seg_off.data(), nseg, bps, slot0};
  return c;
}

}  // namespace

int main() {
  std::mt19937_64 rng(12345);
  int fails = 0;
  for (int trial = 0; trial < 400 && fails == 0; ++trial) {
    const uint64_t nseg = 1 + rng() % 6, bps = 1 + rng() % 40;
    const uint64_t slot0 = trial % 3 == 0 ? (rng() >> 12) : rng() % 1000000;
    Case c = make_case(rng, nseg, bps, slot0, trial % 3);
    const uint64_t total = c.want.size();
    const uint64_t skip = total ? rng() % (total + 1) : 0;
    const uint64_t n = total - skip ? rng() % (total - skip + 1) : 0;
    const uint64_t align = rng() % 8;
    std::vector<uint64_t> buf(total + 32, ~0ull);
    uint64_t* out = buf.data() + align;
    wswire::expand_range(c.ch, c.e.data() + skip, skip, n, out);
    for (uint64_t i = 0; i < n; ++i)
      if (out[i] != c.want[skip + i]) {
        std::printf("trial %d: value %llu mismatch\n", trial, (unsigned long long)i);
        ++fails;
        break;
      }
    for (uint64_t i = n; i + align < buf.size(); ++i)
      if (out[i] != ~0ull) {
        std::printf("trial %d: write past n at %llu\n", trial, (unsigned long long)i);
        ++fails;
        break;
      }
    for (uint64_t i = 0; i < align; ++i)
      if (buf[i] != ~0ull) {
        std::printf("trial %d: write before out\n", trial);
        ++fails;
        break;
      }
  }
  {  // pooled splits of a large chunk, two submissions with tickets
    wswire::Pool* pool = wswire::pool_create(4);
    Case c = make_case(rng, 40, 2048, 7, 1);
    const uint64_t total = c.want.size(), n = total - 5, h = n / 3;
    std::vector<uint64_t> buf(total + 1, 0);
    wswire::Ticket t1, t2;
    wswire::submit_expand(pool, c.ch, c.e.data(), 0, h, buf.data() + 1, &t1);
    wswire::submit_expand(pool, c.ch, c.e.data() + h, h, n - h, buf.data() + 1 + h, &t2);
    wswire::ticket_wait(pool, &t2);
    wswire::ticket_wait(pool, &t1);
    wswire::pool_wait(pool);
    for (uint64_t k = 0; k < n; ++k)
      if (buf[1 + k] != c.want[k]) {
        std::printf("pool: mismatch at %llu\n", (unsigned long long)k);
        ++fails;
        break;
      }
    if (buf[0] != 0 || buf[n + 1] != 0) ++fails, std::printf("pool: out of range write\n");
    wswire::pool_destroy(pool);
  }
  std::printf(fails ? "FAIL\n" : "OK\n");
  return fails ? 1 : 0;
}
