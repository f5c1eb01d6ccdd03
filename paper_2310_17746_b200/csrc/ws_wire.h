// Host expansion of the 16-bit enumeration wire format (see ws_wire.cpp).
#pragma once
#include <atomic>
#include <cstdint>

namespace wswire {

struct Pool;
Pool* pool_create(unsigned nthreads);  // 0 = hardware threads (WHEELSIEVE_HOST_THREADS)
void pool_destroy(Pool* p);
unsigned pool_size(const Pool* p);
void pool_wait(Pool* p);  // until every submitted expansion has finished

// Completion of one submission (its tasks decrement `left`).
struct Ticket {
  std::atomic<uint32_t> left{0};
};
void ticket_wait(Pool* p, Ticket* t);

// Blocks [0, nblk) of bslots wheel slots each, block b starting at wheel
// slot slot0 + b * bslots, holding cnt[b] entries each, in order: widens
// entries skip .. skip + n - 1 (e points at entry `skip`) into out[0 .. n).
void expand_range(const uint16_t* e, const uint32_t* cnt, uint64_t nblk, uint64_t slot0,
                  uint64_t bslots, uint64_t skip, uint64_t n, uint64_t* out);
// expand_range split into tasks on the pool
// (async; `t`, nullable, counts the tasks still running).
void submit_expand(Pool* pool, const uint16_t* e, const uint32_t* cnt, uint64_t nblk,
                   uint64_t slot0, uint64_t bslots, uint64_t skip, uint64_t n, uint64_t* out,
                   Ticket* t = nullptr);

}  // namespace wswire
