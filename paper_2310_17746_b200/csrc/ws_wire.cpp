// Host side of the 8-bit wire format (kEnumWire, ws_internal.h).
//
// For host-bound enumeration the PCIe link and the host's memory, not the
// sieve, are the bound: the primes below 1e10 are 3.64 GB as uint64 (65 ms at
// the measured 56 GB/s D2H) against 2.5 ms of sieving.  The kernel therefore
// ships every prime as one byte -- its bit position e in the interleaved
// survivor masks of its 128-slot block -- plus one count byte per block and
// the per-segment totals (0.47 GB at c2), and the host widens
//     value = 6 * block_first_slot + 3e + 1 + (e & 1)
// straight into the caller's buffer with non-temporal AVX-512 stores (IFMA
// where present), split over a small persistent thread pool and overlapped
// piece by piece with the D2H of later pieces.
//
// Order, count and checksums are fixed on the device; the host only widens
// entries.  Built with g++ (AVX-512 through target attributes and a runtime
// CPU check; a scalar path otherwise).
#include "ws_wire.h"

#include <immintrin.h>
#include <sched.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace wswire {

struct Pool {
  std::vector<std::thread> threads;
  std::mutex m;
  std::condition_variable cv, idle, progress;
  std::deque<std::function<void()>> q;
  size_t busy = 0;
  bool stop = false;

  explicit Pool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) threads.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : threads) t.join();
  }
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> g(m);
        cv.wait(g, [this] { return stop || !q.empty(); });
        if (q.empty()) return;
        f = std::move(q.front());
        q.pop_front();
        ++busy;
      }
      f();
      {
        std::lock_guard<std::mutex> g(m);
        --busy;
        if (q.empty() && busy == 0) idle.notify_all();
      }
      progress.notify_all();
    }
  }
  void submit(std::vector<std::function<void()>>& fs) {
    {
      std::lock_guard<std::mutex> g(m);
      for (auto& f : fs) q.push_back(std::move(f));
    }
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> g(m);
    idle.wait(g, [this] { return q.empty() && busy == 0; });
  }
  void wait(Ticket* t) {
    std::unique_lock<std::mutex> g(m);
    progress.wait(g, [t] { return t->left.load(std::memory_order_acquire) == 0; });
  }
};

namespace {

unsigned default_threads() {
  if (const char* e = std::getenv("WHEELSIEVE_HOST_THREADS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v > 0) return static_cast<unsigned>(std::min<long>(v, 256));
  }
  // the CPUs this process may run on (affinity / cgroup), not the machine's
  cpu_set_t set;
  unsigned h = 0;
  if (sched_getaffinity(0, sizeof set, &set) == 0) h = static_cast<unsigned>(CPU_COUNT(&set));
  if (!h) h = std::thread::hardware_concurrency();
  // one CPU stays with the calling thread, which spins on the ring's copy
  // events (c2 e2e on 16 vCPUs: 24.3 ms with 16 expanders, 23.2-23.7 with 14-15)
  if (h > 4) --h;
  return std::max(1u, std::min(h ? h : 4u, 64u));
}

// Locates entry `skip`: its block b and its offset inside that block.
void locate(const WireChunk& ch, uint64_t skip, uint64_t& b, uint64_t& off) {
  const uint64_t s = static_cast<uint64_t>(
      std::upper_bound(ch.seg_off, ch.seg_off + ch.nseg + 1, skip) - ch.seg_off - 1);
  off = skip - ch.seg_off[s];
  b = s * ch.bps;
  while (off >= ch.cnt[b]) off -= ch.cnt[b++];
}

// ---- scalar expansion ------------------------------------------------------
void expand_scalar(const WireChunk& ch, const uint8_t* e, uint64_t skip, uint64_t n,
                   uint64_t* out) {
  uint64_t b, off, done = 0;
  locate(ch, skip, b, off);
  for (; done < n; ++b) {
    const uint64_t base1 = 6 * (ch.slot0 + b * kBlockSlots) + 1;
    const uint64_t m = std::min<uint64_t>(ch.cnt[b] - off, n - done);
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t x = e[done + i];
      out[done + i] = base1 + 3 * x + (x & 1);
    }
    done += m;
    off = 0;
  }
}

// ---- AVX-512 expansion -----------------------------------------------------
// Eight entries at a time are widened in registers and appended to a carry
// register holding the 0..7 values of the current output cache line; each
// completed line leaves as one aligned 64-byte streaming store (the head
// line, shared with the caller's preceding data, and the tail line use
// masked ordinary stores).  IFMA (madd52lo) forms base + 3x in one op.
struct LaneTables {
  alignas(64) uint64_t merge[8][8];  // lanes < na from the carry, then the new vector
  alignas(64) uint64_t rest[8][8];   // new-vector lanes 8 - na .. 7 -> carry lanes 0 .. na-1
  LaneTables() {
    for (int na = 0; na < 8; ++na)
      for (int i = 0; i < 8; ++i) {
        merge[na][i] = i < na ? i : 8 + (i - na);
        rest[na][i] = (8 - na + i) & 7;
      }
  }
};
const LaneTables kLanes;

template <bool IFMA>
__attribute__((target("avx512f,avx512bw,avx512vl,avx512ifma"))) inline __m512i widen8(
    __m128i raw, __m512i base1) {
  const __m512i x = _mm512_cvtepu8_epi64(raw);
  const __m512i one = _mm512_set1_epi64(1);
  if constexpr (IFMA)
    return _mm512_madd52lo_epu64(_mm512_add_epi64(_mm512_and_si512(x, one), base1), x,
                                 _mm512_set1_epi64(3));
  else
    return _mm512_add_epi64(_mm512_add_epi64(_mm512_slli_epi64(x, 1), x),
                            _mm512_add_epi64(_mm512_and_si512(x, one), base1));
}

template <bool IFMA>
__attribute__((target("avx512f,avx512bw,avx512vl,avx512ifma"))) void expand_avx512(
    const WireChunk& ch, const uint8_t* e, uint64_t skip, uint64_t n, uint64_t* out) {
  if (n == 0) return;
  uint64_t b, off;
  locate(ch, skip, b, off);
  uint64_t* line = reinterpret_cast<uint64_t*>(reinterpret_cast<uintptr_t>(out) & ~uintptr_t{63});
  const uint32_t head = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(out) >> 3) & 7u);
  // carry: the current output line's first na values (lanes 0 .. na-1); the
  // head lanes of the first line are not ours and are never stored
  uint32_t na = head;
  bool first = true;
  __m512i carry = _mm512_setzero_si512();
  uint64_t left = n;
  for (; left; ++b) {
    const uint64_t m = std::min<uint64_t>(ch.cnt[b] - off, left);
    const __m512i base1 =
        _mm512_set1_epi64(static_cast<long long>(6 * (ch.slot0 + b * kBlockSlots) + 1));
    uint64_t i = 0;
    if (m >= 8) {
      // full vectors keep na fixed: the lane maps are loaded once per block
      const __m512i im = _mm512_load_si512(kLanes.merge[na]);
      const __m512i ir = _mm512_load_si512(kLanes.rest[na]);
      if (first) {  // the head line is shared with the caller's preceding data
        const __m512i v = widen8<IFMA>(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(e)), base1);
        _mm512_mask_storeu_epi64(line, static_cast<__mmask8>(0xFFu << head),
                                 _mm512_permutex2var_epi64(carry, im, v));
        carry = _mm512_permutexvar_epi64(ir, v);
        line += 8;
        first = false;
        i = 8;
      }
      for (; i + 8 <= m; i += 8) {
        const __m512i v =
            widen8<IFMA>(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(e + i)), base1);
        _mm512_stream_si512(reinterpret_cast<__m512i*>(line),
                            _mm512_permutex2var_epi64(carry, im, v));
        carry = _mm512_permutexvar_epi64(ir, v);
        line += 8;
      }
    }
    if (i < m) {  // the block's ragged tail: k < 8 values
      const uint32_t k = static_cast<uint32_t>(m - i);
      const __m512i v = widen8<IFMA>(
          _mm_maskz_loadu_epi8(static_cast<__mmask16>((1u << k) - 1), e + i), base1);
      const __m512i comb =
          _mm512_permutex2var_epi64(carry, _mm512_load_si512(kLanes.merge[na]), v);
      if (na + k >= 8) {
        if (first)
          _mm512_mask_storeu_epi64(line, static_cast<__mmask8>(0xFFu << head), comb);
        else
          _mm512_stream_si512(reinterpret_cast<__m512i*>(line), comb);
        first = false;
        line += 8;
        carry = _mm512_permutexvar_epi64(_mm512_load_si512(kLanes.rest[na]), v);
        na = na + k - 8;
      } else {
        carry = comb;
        na += k;
      }
    }
    left -= m;
    e += m;
    off = 0;
  }
  const uint32_t lo = first ? head : 0u;
  if (na > lo)
    _mm512_mask_storeu_epi64(line, static_cast<__mmask8>(((1u << na) - 1u) & (0xFFu << lo)), carry);
  _mm_sfence();
}

// 0 = scalar, 1 = AVX-512, 2 = AVX-512 + IFMA (WHEELSIEVE_HOST_SCALAR=1 forces 0)
int isa_level() {
  static const int lvl = [] {
    if (const char* s = std::getenv("WHEELSIEVE_HOST_SCALAR"))
      if (std::atoi(s)) return 0;
    __builtin_cpu_init();
    if (!(__builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
          __builtin_cpu_supports("avx512vl")))
      return 0;
    if (const char* s = std::getenv("WHEELSIEVE_HOST_NO_IFMA"))
      if (std::atoi(s)) return 1;
    return __builtin_cpu_supports("avx512ifma") ? 2 : 1;
  }();
  return lvl;
}

}  // namespace

Pool* pool_create(unsigned n) { return new Pool(n ? n : default_threads()); }
void pool_destroy(Pool* p) { delete p; }
unsigned pool_size(const Pool* p) { return static_cast<unsigned>(p->threads.size()); }
void pool_wait(Pool* p) { p->wait(); }
void ticket_wait(Pool* p, Ticket* t) { p->wait(t); }

void expand_range(const WireChunk& ch, const uint8_t* e, uint64_t skip, uint64_t n,
                  uint64_t* out) {
  if (n == 0) return;
  switch (isa_level()) {
    case 2: expand_avx512<true>(ch, e, skip, n, out); break;
    case 1: expand_avx512<false>(ch, e, skip, n, out); break;
    default: expand_scalar(ch, e, skip, n, out); break;
  }
}

void submit_expand(Pool* pool, const WireChunk& ch, const uint8_t* e, uint64_t skip, uint64_t n,
                   uint64_t* out, Ticket* t) {
  if (n == 0) return;
  // equal shares of the values; each task finds its first entry through the
  // segment offsets and at most one segment's block counts
  const uint64_t per = std::max<uint64_t>(uint64_t{1} << 16, n / (2 * pool_size(pool)) + 1);
  std::vector<std::function<void()>> fs;
  for (uint64_t a = 0; a < n; a += per) {
    const uint64_t m = std::min(per, n - a);
    fs.emplace_back([=] {
      expand_range(ch, e + a, skip + a, m, out + a);
      if (t) t->left.fetch_sub(1, std::memory_order_release);
    });
  }
  if (t) t->left.fetch_add(static_cast<uint32_t>(fs.size()), std::memory_order_relaxed);
  pool->submit(fs);
}

}  // namespace wswire
