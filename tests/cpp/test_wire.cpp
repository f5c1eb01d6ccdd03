// Host wire-format expander (paper_2310_17746_b200/csrc/ws_wire.cpp) against a
// direct widening of every entry: random block counts (including empty
// blocks), every output alignment, partial ranges (skip, n) and the pooled
// split.  Run once with the AVX-512 path and once with WHEELSIEVE_HOST_SCALAR=1.
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "ws_wire.h"

int main() {
  std::mt19937_64 rng(12345);
  int fails = 0;
  for (int trial = 0; trial < 300; ++trial) {
    const uint64_t nblk = 1 + rng() % 40;
    const uint64_t bslots = uint64_t{1} << (12 + rng() % 4);
    const uint64_t slot0 = (trial % 3 == 0) ? (rng() >> 8) : rng() % 1000000;
    std::vector<uint32_t> cnt(nblk);
    std::vector<uint16_t> e;
    for (uint64_t b = 0; b < nblk; ++b) {
      const uint32_t c = (rng() % 5 == 0) ? 0 : rng() % (trial % 7 == 0 ? 9000 : 300);
      cnt[b] = c;
      std::vector<uint16_t> v;
      for (uint32_t i = 0; i < c; ++i) v.push_back(static_cast<uint16_t>(rng() % (2 * bslots)));
      e.insert(e.end(), v.begin(), v.end());
    }
    const uint64_t total = e.size();
    e.resize(total + 32);
    std::vector<uint64_t> want;
    for (uint64_t b = 0, k = 0; b < nblk; ++b)
      for (uint32_t i = 0; i < cnt[b]; ++i, ++k) {
        const uint64_t x = e[k];
        want.push_back(6 * (slot0 + b * bslots) + 3 * x + 1 + (x & 1));
      }
    const uint64_t skip = total ? rng() % (total + 1) : 0;
    const uint64_t n = (total - skip) ? rng() % (total - skip + 1) : 0;
    const uint64_t align = rng() % 8;
    std::vector<uint64_t> buf(total + 32, ~0ull);
    uint64_t* out = buf.data() + align;
    wswire::expand_range(e.data() + skip, cnt.data(), nblk, slot0, bslots, skip, n, out);
    for (uint64_t i = 0; i < n; ++i)
      if (out[i] != want[skip + i]) {
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
  // pooled split of a large range
  {
    wswire::Pool* pool = wswire::pool_create(4);
    const uint64_t nblk = 300, bslots = 1 << 15;
    std::vector<uint32_t> cnt(nblk);
    std::vector<uint16_t> e;
    for (uint64_t b = 0; b < nblk; ++b) {
      cnt[b] = rng() % 9000;
      for (uint32_t i = 0; i < cnt[b]; ++i) e.push_back(static_cast<uint16_t>(rng()));
    }
    const uint64_t total = e.size();
    std::vector<uint64_t> buf(total + 1, 0);
    wswire::Ticket t1, t2;
    const uint64_t h = (total - 5) / 3;
    wswire::submit_expand(pool, e.data(), cnt.data(), nblk, 7, bslots, 0, h, buf.data() + 1, &t1);
    wswire::submit_expand(pool, e.data() + h, cnt.data(), nblk, 7, bslots, h, total - 5 - h,
                          buf.data() + 1 + h, &t2);
    wswire::ticket_wait(pool, &t2);
    wswire::ticket_wait(pool, &t1);
    wswire::pool_wait(pool);
    for (uint64_t b = 0, k = 0; b < nblk && !fails; ++b)
      for (uint32_t i = 0; i < cnt[b] && k < total - 5; ++i, ++k) {
        const uint64_t x = e[k];
        if (buf[1 + k] != 6 * (7 + b * bslots) + 3 * x + 1 + (x & 1)) {
          std::printf("pool: mismatch at %llu\n", (unsigned long long)k);
          ++fails;
          break;
        }
      }
    if (buf[0] != 0 || buf[total - 4] != 0) ++fails, std::printf("pool: out of range write\n");
    wswire::pool_destroy(pool);
  }
  std::printf(fails ? "FAIL\n" : "OK\n");
  return fails ? 1 : 0;
}
