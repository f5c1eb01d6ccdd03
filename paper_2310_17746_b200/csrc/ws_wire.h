// Host expansion of the 8-bit enumeration wire format (see ws_wire.cpp).
#pragma once
#include <atomic>
#include <cstdint>

namespace wswire {

constexpr uint64_t kBlockSlots = 128;  // wheel slots per wire block (4 interleaved words)

// One pipeline chunk on the host: blocks in slot order, block b starting at
// wheel slot slot0 + b * kBlockSlots with cnt[b] entries; segment s owns
// blocks [s * bps, (s + 1) * bps) and entries [seg_off[s], seg_off[s + 1]).
struct WireChunk {
  const uint8_t* cnt;
  const uint64_t* seg_off;  // nseg + 1 offsets
  uint64_t nseg;
  uint64_t bps;
  uint64_t slot0;
};

struct Pool;
Pool* pool_create(unsigned nthreads);  // 0 = the process's CPUs (WHEELSIEVE_HOST_THREADS)
void pool_destroy(Pool* p);
unsigned pool_size(const Pool* p);
void pool_wait(Pool* p);  // until every submitted expansion has finished

// Completion of one submission (its tasks decrement `left`).
struct Ticket {
  std::atomic<uint32_t> left{0};
};
void ticket_wait(Pool* p, Ticket* t);

// Widens entries skip .. skip + n - 1 of the chunk (e points at entry
// `skip`) into out[0 .. n):  value = 6 * block_slot + 3e + 1 + (e & 1).
void expand_range(const WireChunk& ch, const uint8_t* e, uint64_t skip, uint64_t n,
                  uint64_t* out);
// expand_range split into tasks on the pool (async; `t`, nullable, counts the
// tasks still running).  `ch` is copied; the arrays it points to must live
// until the tasks finish.
void submit_expand(Pool* pool, const WireChunk& ch, const uint8_t* e, uint64_t skip, uint64_t n,
                   uint64_t* out, Ticket* t = nullptr);

}  // namespace wswire
