// C-ABI host layer of libwheelsieve_cuda.so (declared in include/wheelsieve/gpu.h).
//
// Orchestration that the reference does in run_loop (engine.cpp:149-307) and
// BasePrimeStore::bootstrap (base_store.cpp:34-42) is redone device-first:
//   1. base primes <= isqrt(R - 1) are sieved on the device (bounds up to
//      2^18 by small_base_kernel alone; above, it gives level 0, the primes
//      <= sqrt(B), and the main sieve kernel enumerates [0, B] as level 1);
//      the table is kept resident and only re-sieved
//      when a call needs a larger bound (the reference's incremental base
//      store, base_store.cpp:44-76) or WS_FRESH_BASE is set;
//   2. one launch of the segment kernel covers every segment of every
//      requested range (no per-iteration barrier, engine.cpp:257-262);
//   3. only the results cross back: counts, checksums, per-segment counts or
//      the enumerated values.
// No exception crosses the ABI; errors become ws_status + ws_last_error.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "wheelsieve/gpu.h"
#include "ws_internal.h"
#include "ws_wire.h"

namespace {

constexpr uint64_t kMaxWheelIndex = (UINT64_MAX - 5) / 6;       // wheel.hpp:33
constexpr uint64_t kMaxSegmentEnd = 6 * (kMaxWheelIndex + 1);   // wheel.hpp:37

uint64_t isqrt_u64(uint64_t n) {  // wheel.cpp:25-33 semantics (exact)
  if (n == 0) return 0;
  uint64_t r = static_cast<uint64_t>(std::sqrt(static_cast<double>(n)));
  while (r > 0 && r > n / r) --r;
  while (r + 1 <= n / (r + 1)) ++r;
  return r;
}

struct Fail {
  ws_status code;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    throw Fail{WS_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e)};
  if (e != cudaSuccess) throw Fail{WS_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  void reserve(size_t n, const char* what) {
    if (n <= cap) return;
    release();
    ck(cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T)), what);
    cap = n;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
  // grow to n elements keeping the first `keep` (stream-ordered copy)
  void grow(size_t n, size_t keep, cudaStream_t st, const char* what) {
    if (n <= cap) return;
    T* q = nullptr;
    ck(cudaMalloc(&q, n * sizeof(T)), what);
    if (keep && ptr) {
      const cudaError_t e = cudaMemcpyAsync(q, ptr, std::min(keep, cap) * sizeof(T),
                                            cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) {
        cudaFree(q);
        ck(e, what);
      }
      ck(cudaStreamSynchronize(st), what);  // the old buffer is freed next
    }
    release();
    ptr = q;
    cap = n;
  }
};

// Growable page-locked host staging (async H2D/D2H without staging copies).
struct PinnedBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* reserve(size_t n, const char* what) {
    if (n <= bytes) return ptr;
    release();
    ck(cudaMallocHost(&ptr, std::max<size_t>(n, 64)), what);
    bytes = n;
    return ptr;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

// Per-call bump arena of pinned staging for async uploads.  A region is
// never reused within a call (its copy may still be pending); offsets reset
// at the start of the next call, which is safe because every call ends with
// a stream synchronisation.
struct PinnedArena {
  std::vector<PinnedBuf> blocks;
  size_t cur = 0, off = 0;
  void reset() {
    cur = 0;
    off = 0;
  }
  void* alloc(size_t n, const char* what) {
    n = (n + 255) / 256 * 256;
    while (cur < blocks.size() && off + n > blocks[cur].bytes) {
      ++cur;
      off = 0;
    }
    if (cur == blocks.size()) {
      blocks.emplace_back();
      blocks.back().reserve(std::max<size_t>(n, 1 << 20), what);
      off = 0;
    }
    void* p = static_cast<char*>(blocks[cur].ptr) + off;
    off += n;
    return p;
  }
  void release() {
    for (auto& b : blocks) b.release();
    blocks.clear();
    reset();
  }
};

uint64_t small_primes_upto(uint64_t B) {  // |{5,7,...,47} ∩ [5, B]| (the stamped primes)
  static const uint32_t sp[] = {5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47};
  uint64_t c = 0;
  for (uint32_t q : sp) c += q <= B;
  return c;
}

}  // namespace

struct ws_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t S = 1u << 18;
  int sms = 148;
  int bps[wsk::kNumModes] = {2, 2, 2, 2};  // resident blocks per SM per mode
  std::string err;
  ws_timing timing{};
  cudaEvent_t ev[4] = {};

  PinnedArena pin_up;  // async upload staging (jobs, runs), reset per call
  PinnedBuf pin_out;   // results, read after the call's synchronisation
  DevBuf<uint32_t> d_tabn;  // exact base-table size, written on device by prepare_table
  DevBuf<uint32_t> d_tabn_old;  // its value before an extension (append_table reads it)
  bool base_extend = true;      // grow the table incrementally (WHEELSIEVE_BASE_EXTEND=0: rebuild)
  DevBuf<uint32_t> small_tab;  // small-prime pattern tables

  // resident base-prime table: every prime in [53, base_B]
  bool base_valid = false;
  bool base_built = false;  // the last call (re)built the table
  uint64_t base_B = 0;
  uint32_t nprimes = 0;              // upper bound on the table size (host)
  const uint32_t* nprimes_dev = nullptr;  // exact size on device (nullable)
  DevBuf<uint32_t> tab_p;
  DevBuf<unsigned long long> tab_m;
  DevBuf<double> tab_inv;

  uint32_t* words_out[2] = {nullptr, nullptr};  // SegmentBitmap export (ws_sieve_segment)
  uint32_t n_below_S = 0;  // table primes (>= 37) below bucket_pmin: in-kernel; the rest bucketed
  uint32_t bucket_pmin = 0;
  uint32_t n_S = 0;        // table primes (>= 37) below S
  uint32_t n_wc = 161;     // table primes below the warp-cooperative limit (1024)
  // bytes of bucket lists per window buffer (two buffers): 8 GiB puts C4 in
  // 7 windows instead of 41, with fewer fill / sieve tails (C4 56.8 -> 53.5 ms;
  // 16 GiB is no faster: 32-bit entry indices cap a window near 2^32 entries)
  size_t bucket_budget = 8ull << 30;
  uint32_t cap_override = 0;           // test knob (WHEELSIEVE_BUCKET_CAP)
  uint32_t piece_override = 0;         // tuning knob (WHEELSIEVE_FILL_PIECE)
  bool fill_huge = true;               // carried-offset fill for p >= run length (WHEELSIEVE_FILL_HUGE)
  uint32_t huge_step = 1;              // runs per histogram step there (WHEELSIEVE_HUGE_STEP)
  uint32_t huge_from = 0;              // its lower bound in units of S (0: the run length)
  uint64_t huge_thr = 0;               // the run length in slots the count below is for
  uint32_t n_below_huge = 0;           // table primes (>= 53) below huge_thr
  uint32_t bucket_min_ratio = 8;       // buckets iff largest base prime >= ratio * S
  uint32_t bucket_ctas_per_sm = 0;     // tuning knob (WHEELSIEVE_BUCKET_CTAS)
  uint32_t ctas_per_sm = 0;            // tuning knob, all launches (WHEELSIEVE_CTAS_PER_SM)

  // scratch
  DevBuf<uint32_t> bucket[2];  // double-buffered window lists (fill w+1 || sieve w)
  DevBuf<uint32_t> bcount[2];
  cudaStream_t fstream = nullptr;  // bucket-fill stream
  // small base builds (B <= 2^18) run on their own stream, overlapping the call's
  // uploads and resets; the first launch that reads the table joins it
  cudaStream_t bstream = nullptr;
  cudaEvent_t ev_fork = nullptr;
  bool base_pending = false;
  DevBuf<unsigned long long> base_scratch;  // small_base_kernel's epoch-tagged block counts
  uint32_t base_epoch = 0;
  const unsigned long long* ticket_zeroed = nullptr;  // ticket buffer known to be zero
  size_t ticket_zeroed_cap = 0;
  cudaStream_t cstream = nullptr;  // device->host copy stream (chunked enumeration)
  cudaEvent_t ev_order = nullptr;
  static constexpr int kMaxChunks = 16;
  cudaEvent_t chunk_done[kMaxChunks] = {};
  // host-bound enumeration through the 8-bit wire format (ws_wire.cpp);
  // WHEELSIEVE_HOST_WIRE=0 ships uint64 values instead
  bool host_wire = true;
  wswire::Pool* pool = nullptr;  // host expansion threads (created on first use)
  DevBuf<uint8_t> wire;          // wire entries of every chunk
  DevBuf<uint8_t> wblk;          // survivors per wire block
  PinnedBuf pin_wire, pin_wblk;
  // a 6 MB ring stays in the host's last-level cache (60 MB L3 on the B200 box),
  // so the payload crosses DRAM only once, as output (c2 e2e 26.4 -> 25.2 ms)
  uint64_t wire_piece = 1u << 21;  // entries (bytes) per ring slot (WHEELSIEVE_WIRE_PIECE)
  uint64_t wire_ring = 3;          // ring slots (WHEELSIEVE_WIRE_RING)
  std::vector<cudaEvent_t> ring_ev;
  cudaEvent_t fill_done[2] = {}, sieve_done[2] = {};
  DevBuf<wsk::Run> runs;
  DevBuf<wsk::Job> jobs;
  DevBuf<wsk::JobAcc> acc;
  DevBuf<unsigned long long> ticket;
  DevBuf<uint32_t> per_seg;
  DevBuf<unsigned long long> status;
  DevBuf<unsigned long long> vals;  // enumeration scratch (base primes / host-bound output)
  DevBuf<uint32_t> l0_p;
  DevBuf<unsigned long long> l0_m;
  DevBuf<double> l0_inv;
  DevBuf<uint32_t> l0_n;
  std::vector<wsk::Job> h_jobs;

  ~ws_ctx() {
    cudaSetDevice(device);
    if (pool) wswire::pool_destroy(pool);
    wire.release();
    wblk.release();
    pin_wire.release();
    pin_wblk.release();
    for (cudaEvent_t e : ring_ev) cudaEventDestroy(e);
    for (auto* b : {&tab_p, &per_seg, &l0_p, &l0_n, &bucket[0], &bucket[1], &bcount[0], &bcount[1]})
      b->release();
    runs.release();
    tab_inv.release();
    l0_inv.release();
    d_tabn.release();
    d_tabn_old.release();
    small_tab.release();
    pin_up.release();
    pin_out.release();
    for (int i = 0; i < 2; ++i) {
      if (fill_done[i]) cudaEventDestroy(fill_done[i]);
      if (sieve_done[i]) cudaEventDestroy(sieve_done[i]);
    }
    if (fstream) cudaStreamDestroy(fstream);
    if (bstream) cudaStreamDestroy(bstream);
    base_scratch.release();
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (cstream) cudaStreamDestroy(cstream);
    if (ev_order) cudaEventDestroy(ev_order);
    for (cudaEvent_t e : chunk_done)
      if (e) cudaEventDestroy(e);
    for (auto* b : {&tab_m, &ticket, &status, &vals, &l0_m}) b->release();
    jobs.release();
    acc.release();
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// Every host<->device copy goes through these, so ws_timing reports the
// bytes that crossed PCIe in the last call.
cudaError_t copy_async(ws_ctx* c, void* dst, const void* src, size_t n, cudaMemcpyKind k,
                       cudaStream_t st) {
  if (k == cudaMemcpyHostToDevice) c->timing.h2d_bytes += n;
  if (k == cudaMemcpyDeviceToHost) c->timing.d2h_bytes += n;
  return cudaMemcpyAsync(dst, src, n, k, st);
}
cudaError_t copy_sync(ws_ctx* c, void* dst, const void* src, size_t n, cudaMemcpyKind k) {
  if (k == cudaMemcpyHostToDevice) c->timing.h2d_bytes += n;
  if (k == cudaMemcpyDeviceToHost) c->timing.d2h_bytes += n;
  return cudaMemcpy(dst, src, n, k);
}

uint64_t prime_count_bound(uint64_t L, uint64_t R) {
  if (R <= L) return 0;
  const double y = static_cast<double>(R - L);
  const uint64_t slots = (R - L) / 3 + 4;  // wheel slots + 2, 3 and rounding
  double b;
  // prefix: pi(x) < 1.25506 x / ln x (Rosser-Schoenfeld, x > 1)
  const double x = static_cast<double>(R);
  double pref = x < 17 ? 8.0 : 1.25506 * x / std::log(x) + 8;
  // window: pi(L + y) - pi(L) <= 2 y / ln y (Montgomery-Vaughan, y > 1)
  double win = y < 17 ? 8.0 : 2.0 * y / std::log(y) + 8;
  b = std::min(pref, win);
  const uint64_t bb = static_cast<uint64_t>(b) + 16;
  return std::min<uint64_t>(bb, slots);
}

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double ms() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
        .count();
  }
};

// Geometry of [L, R): K0 = floor(L/6), slots = ceil((R - 6 K0)/6).
wsk::Job make_job(uint64_t L, uint64_t R, uint32_t S, uint64_t seg_begin) {
  wsk::Job j{};
  j.L = L;
  j.R = R;
  j.K0 = L / 6;
  j.nslots = R > L ? (R - 6 * j.K0 + 5) / 6 : 0;
  j.seg_begin = seg_begin;
  j.nseg = (j.nslots + S - 1) / S;
  return j;
}

void validate_range(uint64_t L, uint64_t R) {
  if (R > kMaxSegmentEnd)
    throw Fail{WS_OVERFLOW, "range end " + std::to_string(R) +
                                " exceeds the sievable 64-bit range (engine.cpp:139)"};
  (void)L;
}

// Expected large-prime hits per segment: 2 S sum_{S <= p <= P} 1/p, by
// Mertens' estimate sum 1/p over [a, b] ~ ln(ln b / ln a).
double expected_large_hits(uint32_t pmin, uint32_t S, double pmax) {
  if (pmax <= pmin) return 0;
  return 2.0 * S * std::log(std::log(pmax) / std::log(static_cast<double>(pmin)));
}

// The segment kernel over every segment of ctx->h_jobs.  Without large
// primes this is one launch; otherwise the segments are processed in windows
// of W segments: bucket_fill (large-prime hit lists) then the sieve kernel.
// Table primes (>= 53) below x, by an odd-only host sieve; cached per context
// and per process (x is the fill's run length in slots, 2^23 at the default
// 32 x 2^18, so the sieve runs once).
uint32_t table_primes_below(ws_ctx* c, uint64_t x) {
  if (c->huge_thr == x) return c->n_below_huge;
  static std::mutex mu;
  static std::vector<std::pair<uint64_t, uint32_t>> memo;
  uint32_t n = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    bool found = false;
    for (const auto& e : memo)
      if (e.first == x) n = e.second, found = true;
    if (!found) {
      std::vector<uint8_t> comp(x / 2 + 1, 0);  // comp[i] <-> 2i + 1
      for (uint64_t i = 1; 2 * i + 1 < x; ++i) {
        if (comp[i]) continue;
        const uint64_t q = 2 * i + 1;
        if (q >= wsk::kFirstTablePrime) ++n;
        for (uint64_t j = q * q; j < x; j += 2 * q) comp[j / 2] = 1;
      }
      memo.emplace_back(x, n);
    }
  }
  c->huge_thr = x;
  c->n_below_huge = n;
  return n;
}

// Order the main stream after a pending small base build (bstream).
void join_base(ws_ctx* c) {
  if (!c->base_pending) return;
  ck(cudaStreamWaitEvent(c->stream, c->ev[1], 0), "base join");
  c->base_pending = false;
}

struct WireArgs {  // kEnumWire outputs
  uint8_t* entries;
  uint8_t* blk8;
};

void run_sieve(ws_ctx* c, int mode, uint32_t* per_seg_dev, unsigned long long* out,
               unsigned long long out_cap, bool timed, uint32_t acc_base = 0,
               bool record_start = true, const WireArgs* wire = nullptr) {
  uint64_t nseg = 0;
  for (const auto& j : c->h_jobs) nseg += j.nseg;
  const size_t nj = c->h_jobs.size();
  c->jobs.reserve(nj, "jobs");
  // + 1: the slot after the accumulators receives the exact table size
  if (c->acc.cap < acc_base + nj + 1) {  // grow without losing accumulators of earlier chunks
    if (acc_base) ck(cudaStreamSynchronize(c->stream), "sync");
    DevBuf<wsk::JobAcc> bigger;
    bigger.reserve(std::max<size_t>(acc_base + nj + 1, 16), "acc");
    if (acc_base)
      ck(cudaMemcpy(bigger.ptr, c->acc.ptr, acc_base * sizeof(wsk::JobAcc), cudaMemcpyDeviceToDevice),
         "acc");
    std::swap(c->acc, bigger);
    bigger.release();
  }
  if (nj > 1) {  // a single job travels in the kernel parameters
    void* hj = c->pin_up.alloc(nj * sizeof(wsk::Job), "pinned jobs");
    std::memcpy(hj, c->h_jobs.data(), nj * sizeof(wsk::Job));
    ck(copy_async(c, c->jobs.ptr, hj, nj * sizeof(wsk::Job), cudaMemcpyHostToDevice, c->stream),
       "upload jobs");
  }
  ck(cudaMemsetAsync(c->acc.ptr + acc_base, 0, nj * sizeof(wsk::JobAcc), c->stream), "zero acc");
  if (mode >= wsk::kEnumerate) {
    c->status.reserve(nseg, "status");
    ck(cudaMemsetAsync(c->status.ptr, 0, nseg * sizeof(unsigned long long), c->stream),
       "zero status");
  }
  if (nseg == 0) return;
  wsk::SieveParams p{};
  p.small_tab = c->small_tab.ptr;
  p.jobs = nj > 1 ? c->jobs.ptr : nullptr;
  if (nj == 1) p.job0 = c->h_jobs[0];
  p.njobs = static_cast<uint32_t>(nj);
  p.tabn_out = reinterpret_cast<uint32_t*>(c->acc.ptr + acc_base + nj);
  p.nseg_total = nseg;
  p.S = c->S;
  p.prime_p = c->tab_p.ptr;
  p.prime_m = c->tab_m.ptr;
  p.prime_inv = c->tab_inv.ptr;
  p.nprimes = c->nprimes;
  p.nprimes_dev = c->nprimes_dev;
  // warp-cooperative loop for primes below 1024 (>= 256 hits per class per
  // 2^18-slot segment): 161 table entries; one thread per prime above
  p.n_wc = std::min<uint32_t>(c->n_wc, c->nprimes);
  p.n_mid = std::min<uint32_t>(std::max(c->n_below_S, p.n_wc), c->nprimes);
  p.n_S = std::min<uint32_t>(std::max(c->n_S, p.n_wc), p.n_mid);
  p.acc = c->acc.ptr + acc_base;
  p.per_seg = per_seg_dev;
  p.status = c->status.ptr;
  p.out = out;
  p.out_cap = out_cap;
  p.words1 = c->words_out[0];
  p.words5 = c->words_out[1];
  if (wire) {
    p.out8 = wire->entries;
    p.blk8 = wire->blk8;
  }
  uint64_t max_grid = static_cast<uint64_t>(c->sms) * c->bps[mode];
  if (c->ctas_per_sm)
    max_grid = std::min<uint64_t>(max_grid, static_cast<uint64_t>(c->sms) * c->ctas_per_sm);
  // Buckets pay off only when most large primes are far above S (c4: up to
  // 120 S, c5: 16 S); up to a few S (c3: 3.8 S) the per-(prime, segment)
  // offset check in the kernel is cheaper than fill + apply + windowing.
  const bool buckets = c->nprimes > p.n_mid && c->base_B > c->bucket_pmin &&
                       c->base_B >= static_cast<uint64_t>(c->bucket_min_ratio) * c->S;
  uint64_t W = nseg;
  uint32_t cap = 0;
  if (buckets) {
    const double E = expected_large_hits(c->bucket_pmin, c->S, static_cast<double>(c->base_B));
    cap = static_cast<uint32_t>(1.1 * E + 8.0 * std::sqrt(E) + 1024);
    cap = (cap + 31) / 32 * 32;
    if (c->cap_override) cap = c->cap_override;
    W = std::max<uint64_t>(8, c->bucket_budget / (4ull * cap));
    W = std::min<uint64_t>({W, wsk::kMaxWindow, nseg});
    // the fill kernel indexes a window's lists with 32-bit entry indices
    W = std::min<uint64_t>(W, ((1ull << 32) - (1ull << 26)) / cap - 1);
    for (int b = 0; b < 2; ++b) {
      c->bucket[b].reserve(W * cap, "bucket lists");
      c->bcount[b].reserve(W, "bucket counts");
      ck(cudaMemsetAsync(c->bcount[b].ptr, 0, W * sizeof(uint32_t), c->stream), "zero bcount");
    }
  }
  const uint64_t nwin = (nseg + W - 1) / W;
  // one {counter, exits} pair per window; kernels leave them zero
  c->ticket.reserve(2 * nwin, "tickets");
  if (c->ticket_zeroed != c->ticket.ptr || c->ticket_zeroed_cap != c->ticket.cap) {
    ck(cudaMemsetAsync(c->ticket.ptr, 0, c->ticket.cap * sizeof(unsigned long long), c->stream),
       "zero tickets");
    c->ticket_zeroed = c->ticket.ptr;
    c->ticket_zeroed_cap = c->ticket.cap;
  }
  // runs of every window, uploaded once
  std::vector<wsk::Run> runs;
  std::vector<uint32_t> run_off(nwin + 1, 0);
  uint64_t piece = W;
  if (buckets) {
    // optional cap on sieve CTAs per SM to leave room for fill CTAs (measured: no gain)
    if (c->bucket_ctas_per_sm)
      max_grid = std::min<uint64_t>(max_grid, static_cast<uint64_t>(c->sms) * c->bucket_ctas_per_sm);
    // runs are cut into 32-segment pieces: short per-thread hit loops and a
    // fill grid that covers the GPU (measured best for c4 and c5)
    piece = c->piece_override ? c->piece_override : 32;
    piece = std::min<uint64_t>(piece, W);
    size_t j = 0;
    for (uint64_t w = 0; w < nwin; ++w) {
      const uint64_t ws = w * W, we = std::min(nseg, ws + W);
      while (j < nj && c->h_jobs[j].seg_begin + c->h_jobs[j].nseg <= ws) ++j;
      for (size_t q = j; q < nj && c->h_jobs[q].seg_begin < we; ++q) {
        const wsk::Job& J = c->h_jobs[q];
        const uint64_t a0 = std::max(ws, J.seg_begin), b0 = std::min(we, J.seg_begin + J.nseg);
        // runs are cut into pieces of at most `piece` segments so the fill
        // grid scales with the window when there are few large primes
        for (uint64_t x = a0; x < b0; x += piece) {
          const uint64_t y = std::min<uint64_t>(b0, x + piece);
          wsk::Run r{};
          r.k_lo = J.K0 + (x - J.seg_begin) * c->S;
          r.k_hi = std::min(J.K0 + (y - J.seg_begin) * c->S, J.K0 + J.nslots);
          r.seg0 = static_cast<uint32_t>(x - ws);
          r.nseg = static_cast<uint32_t>(y - x);
          runs.push_back(r);
        }
      }
      run_off[w + 1] = static_cast<uint32_t>(runs.size());
    }
    c->runs.reserve(runs.size(), "runs");
    void* hr = c->pin_up.alloc(runs.size() * sizeof(wsk::Run), "pinned runs");
    std::memcpy(hr, runs.data(), runs.size() * sizeof(wsk::Run));
    ck(copy_async(c, c->runs.ptr, hr, runs.size() * sizeof(wsk::Run), cudaMemcpyHostToDevice,
                  c->stream), "upload runs");
  }
  // ev[2] (call start) / ev[4] order the fill stream after everything queued so far
  join_base(c);
  if (record_start) ck(cudaEventRecord(c->ev[2], c->stream), "event");
  if (buckets) {
    ck(cudaEventRecord(c->ev_order, c->stream), "event");
    ck(cudaStreamWaitEvent(c->fstream, c->ev_order, 0), "fill wait");
  }
  // primes of at least the run length take the carried-offset fill when every
  // run is a piece of the one job (consecutive in wheel slots)
  uint32_t huge_begin = c->nprimes;
  const uint64_t huge_from = (c->huge_from ? c->huge_from : piece) * c->S;
  if (buckets && c->fill_huge && nj == 1 && c->base_B >= huge_from)
    huge_begin = std::max(p.n_mid, table_primes_below(c, huge_from));
  // with the large-prime fill that heavy (half of a C4 window), two sieve CTAs
  // per SM leave room for fill blocks to run alongside (C4 53.6 -> 53.1 ms,
  // C4e 60.6 -> 58.3 ms; multi-job windows such as C5's lose with it)
  if (huge_begin < c->nprimes && c->bucket_ctas_per_sm == 0)
    max_grid = std::min<uint64_t>(max_grid, 2ull * c->sms);
  for (uint64_t w = 0; w < nwin; ++w) {
    const uint64_t ws = w * W, we = std::min(nseg, ws + W);
    const int b = static_cast<int>(w & 1);
    if (buckets) {
      // fill window w into buffer b on the fill stream, once the sieve of
      // window w-2 has released it; it overlaps the sieve of window w-1
      if (w >= 2) ck(cudaStreamWaitEvent(c->fstream, c->sieve_done[b], 0), "fill wait");
      wsk::FillParams f{};
      f.runs = c->runs.ptr + run_off[w];
      f.nruns = run_off[w + 1] - run_off[w];
      f.prime_p = c->tab_p.ptr;
      f.prime_m = c->tab_m.ptr;
      f.prime_inv = c->tab_inv.ptr;
      f.nprimes_dev = c->nprimes_dev;
      f.p_begin = p.n_mid;
      f.p_end = c->nprimes;
      f.log2S = static_cast<uint32_t>(__builtin_ctz(c->S));
      f.bucket = c->bucket[b].ptr;
      f.bcount = c->bcount[b].ptr;
      f.bcap = cap;
      f.max_run_segs = static_cast<uint32_t>(piece);
      if (huge_begin < c->nprimes) {
        // p >= run length: at most one hit per class per run; offsets are
        // carried across runs (bucket_fill_huge_kernel)
        wsk::FillParams fh = f;
        fh.p_begin = huge_begin;
        f.p_end = huge_begin;
        const uint32_t nbx = (c->nprimes - huge_begin + wsk::kFillPrimesPerBlock - 1) /
                             wsk::kFillPrimesPerBlock;
        // enough block rows to cover the GPU ~12 blocks per SM, and a group
        // span below 2^31 slots
        const uint32_t rows = std::max<uint32_t>(1, (12u * c->sms + nbx - 1) / nbx);
        uint32_t g = (fh.nruns + rows - 1) / rows;
        g = std::max<uint32_t>(1, std::min<uint32_t>(g, ((1u << 31) - 1) / (piece * c->S)));
        fh.group_runs = g;
        fh.huge_step = c->huge_step;
        fh.max_run_segs = static_cast<uint32_t>(piece) * c->huge_step;
        ck(wsk::launch_bucket_fill_huge(fh, c->fstream), "bucket fill (huge primes)");
        c->timing.launches += 1;
      }
      ck(wsk::launch_bucket_fill(f, c->fstream), "bucket fill");
      ck(cudaEventRecord(c->fill_done[b], c->fstream), "event");
      ck(cudaStreamWaitEvent(c->stream, c->fill_done[b], 0), "sieve wait");
      c->timing.launches += 1;
      p.bucket = c->bucket[b].ptr;
      p.bcount = c->bcount[b].ptr;
      p.bcap = cap;
    }
    p.s_begin = ws;
    p.s_count = we - ws;
    p.ticket = c->ticket.ptr + 2 * w;
    const int grid = static_cast<int>(std::min<uint64_t>(we - ws, max_grid));
    ck(wsk::launch_sieve(mode, p, grid, c->stream), "sieve launch");
    if (buckets) ck(cudaEventRecord(c->sieve_done[b], c->stream), "event");
    c->timing.launches += 1;
  }
  (void)timed;
  ck(cudaEventRecord(c->ev[3], c->stream), "event");
  c->timing.segments += nseg;
}

// Make the resident table cover every prime in [37, B].  No host round
// trip: the level-0 count and the table size stay on the device and the
// kernels read them (SieveParams::nprimes_dev); the host keeps upper bounds.
// Device-side BasePrimeStore::extend (base_store.cpp:44-69): the resident
// table [53, base_B] already covers sqrt(B), so only (base_B, B] is sieved --
// with that table -- and appended; the table size stays on the device.
void extend_base(ws_ctx* c, uint64_t B) {
  join_base(c);
  ck(cudaEventRecord(c->ev[0], c->stream), "event");
  const uint64_t lo = c->base_B + 1;
  const uint64_t cap = prime_count_bound(lo, B + 1);
  const uint64_t need = static_cast<uint64_t>(c->nprimes) + cap;
  c->tab_p.grow(need, c->nprimes, c->stream, "base table");
  c->tab_m.grow(need, c->nprimes, c->stream, "base table");
  c->tab_inv.grow(need, c->nprimes, c->stream, "base table");
  c->vals.reserve(std::max<uint64_t>(cap, 1), "base values");
  c->d_tabn_old.reserve(1, "table size");
  // the extension's segments are small so a short range spreads over the GPU
  const uint32_t S_main = c->S;
  uint32_t S_ext = 1u << 12;
  while (S_ext < S_main && ((B - lo) / 6) / S_ext > 4ull * c->sms) S_ext <<= 1;
  c->S = S_ext;
  c->h_jobs.assign(1, make_job(lo, B + 1, c->S, 0));
  try {
    run_sieve(c, wsk::kEnumerate, nullptr, c->vals.ptr, cap, false);
  } catch (...) {
    c->S = S_main;
    throw;
  }
  c->S = S_main;
  ck(cudaMemcpyAsync(c->d_tabn_old.ptr, c->nprimes_dev, sizeof(uint32_t),
                     cudaMemcpyDeviceToDevice, c->stream), "table size");
  ck(wsk::launch_append_table(c->vals.ptr, &c->acc.ptr[0].count, cap, c->tab_p.ptr, c->tab_m.ptr,
                              c->tab_inv.ptr, c->d_tabn.ptr, c->d_tabn_old.ptr, c->stream),
     "append table");
  c->timing.launches += 1;
  c->nprimes = static_cast<uint32_t>(need);
  c->base_B = B;
  c->base_built = true;
  c->base_valid = true;
  ck(cudaEventRecord(c->ev[1], c->stream), "event");
}

cudaError_t launch_small_base(ws_ctx* c, uint32_t n, uint32_t* p, unsigned long long* m,
                              double* inv, uint32_t* count, cudaStream_t st) {
  if (!c->base_scratch.ptr) {
    c->base_scratch.reserve(64, "base scratch");
    ck(cudaMemset(c->base_scratch.ptr, 0, 64 * sizeof(unsigned long long)), "base scratch");
  }
  if (++c->base_epoch == 0) ++c->base_epoch;  // 0 marks "never written"
  return wsk::launch_small_base(n, p, m, inv, count, c->base_scratch.ptr, c->base_epoch, st);
}

void ensure_base(ws_ctx* c, uint64_t B, bool fresh) {
  c->base_built = false;
  join_base(c);
  if (c->base_valid && c->base_B >= B && !fresh) return;
  if (c->base_extend && c->base_valid && !fresh && c->nprimes_dev == c->d_tabn.ptr &&
      c->base_B >= wsk::kFirstTablePrime && isqrt_u64(B) <= c->base_B && B <= 0xFFFFFFFFull &&
      static_cast<uint64_t>(c->nprimes) + prime_count_bound(c->base_B + 1, B + 1) < 0xFFFFFFFFull)
    return extend_base(c, B);
  c->base_built = true;
  c->base_valid = false;
  if (B < wsk::kFirstTablePrime) {
    ck(cudaEventRecord(c->ev[0], c->stream), "event");
    c->nprimes = 0;
    c->nprimes_dev = nullptr;
    c->base_B = B;
    c->base_valid = true;
    ck(cudaEventRecord(c->ev[1], c->stream), "event");
    return;
  }
  if (B > 0xFFFFFFFFull) throw Fail{WS_OVERFLOW, "base bound exceeds 2^32"};
  if (B > wsk::kTinyMax) ck(cudaEventRecord(c->ev[0], c->stream), "event");
  if (B <= wsk::kTinyMax) {  // the whole table from one small_base launch, on bstream
    const uint64_t cap = prime_count_bound(0, B + 1);
    c->tab_p.reserve(cap, "base table");
    c->tab_m.reserve(cap, "base table");
    c->tab_inv.reserve(cap, "base table");
    c->d_tabn.reserve(1, "table size");
    // after everything queued so far (earlier launches read the old table);
    // ev[1] (the build's end, for base_ms) is also what the first reader joins
    ck(cudaEventRecord(c->ev_fork, c->stream), "event");
    ck(cudaStreamWaitEvent(c->bstream, c->ev_fork, 0), "base fork");
    ck(cudaEventRecord(c->ev[0], c->bstream), "event");
    ck(launch_small_base(c, static_cast<uint32_t>(B), c->tab_p.ptr, c->tab_m.ptr, c->tab_inv.ptr,
                         c->d_tabn.ptr, c->bstream), "small base");
    ck(cudaEventRecord(c->ev[1], c->bstream), "event");
    c->base_pending = true;
    c->timing.launches += 1;
    const uint64_t skip = small_primes_upto(B);
    c->nprimes = static_cast<uint32_t>(cap > skip ? cap - skip : 0);
    c->nprimes_dev = c->d_tabn.ptr;
    c->base_B = B;
    c->base_valid = true;
    return;
  }
  // level 0: primes in [37, isqrt(B)] (isqrt(B) < 2^16: at most 6542 - 11)
  const uint64_t B0 = isqrt_u64(B);
  c->l0_p.reserve(7000, "l0");
  c->l0_m.reserve(7000, "l0");
  c->l0_inv.reserve(7000, "l0");
  c->l0_n.reserve(1, "l0");
  ck(launch_small_base(c, static_cast<uint32_t>(B0), c->l0_p.ptr, c->l0_m.ptr, c->l0_inv.ptr,
                       c->l0_n.ptr, c->stream), "small base");
  c->timing.launches += 1;
  // level 1: enumerate [0, B + 1) with the level-0 table
  const uint64_t cap = prime_count_bound(0, B + 1);
  c->vals.reserve(cap, "base values");
  c->tab_p.reserve(cap, "base table");
  c->tab_m.reserve(cap, "base table");
  c->tab_inv.reserve(cap, "base table");
  c->d_tabn.reserve(1, "table size");
  std::swap(c->tab_p, c->l0_p);  // run_sieve reads the table from tab_*
  std::swap(c->tab_m, c->l0_m);
  std::swap(c->tab_inv, c->l0_inv);
  c->nprimes = 7000;
  c->nprimes_dev = c->l0_n.ptr;
  // small segments so the (short) base range spreads over many CTAs
  const uint32_t S_main = c->S;
  uint32_t S_base = 1u << 12;
  while (S_base < S_main && (B / 6) / S_base > 4ull * c->sms) S_base <<= 1;
  c->S = S_base;
  c->h_jobs.assign(1, make_job(0, B + 1, c->S, 0));
  try {
    run_sieve(c, wsk::kEnumerate, nullptr, c->vals.ptr, cap, false);
  } catch (...) {
    c->S = S_main;
    throw;
  }
  c->S = S_main;
  std::swap(c->tab_p, c->l0_p);
  std::swap(c->tab_m, c->l0_m);
  std::swap(c->tab_inv, c->l0_inv);
  const uint64_t skip = small_primes_upto(B);
  ck(wsk::launch_prepare_table(c->vals.ptr, skip, &c->acc.ptr[0].count, cap, c->tab_p.ptr,
                               c->tab_m.ptr, c->tab_inv.ptr, c->d_tabn.ptr, c->stream),
     "prepare table");
  c->timing.launches += 1;
  c->nprimes = static_cast<uint32_t>(cap > skip ? cap - skip : 0);
  c->nprimes_dev = c->d_tabn.ptr;
  c->base_B = B;
  c->base_valid = true;
  ck(cudaEventRecord(c->ev[1], c->stream), "event");
}

// Copy the n job accumulators and, from the slot after them, the exact table
// size (stored by the kernel: run_sieve's tabn_out) to pinned host memory in
// one copy, and wait: the one synchronisation of a call.
const wsk::JobAcc* fetch_results(ws_ctx* c, size_t n) {
  char* h = static_cast<char*>(c->pin_out.reserve((n + 1) * sizeof(wsk::JobAcc), "pinned out"));
  ck(copy_async(c, h, c->acc.ptr, (n + 1) * sizeof(wsk::JobAcc), cudaMemcpyDeviceToHost,
                c->stream), "results");
  ck(cudaStreamSynchronize(c->stream), "sync");
  ck(cudaGetLastError(), "kernel");
  const uint32_t tabn = *reinterpret_cast<const uint32_t*>(h + n * sizeof(wsk::JobAcc));
  c->timing.base_primes = tabn + small_primes_upto(c->base_B);
  return reinterpret_cast<const wsk::JobAcc*>(h);
}

float event_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0;
  return ms;
}

template <class F>
ws_status guarded(ws_ctx* c, F&& f) {
  if (!c) return WS_BAD_CONFIG;
  Timer t;
  c->err.clear();
  c->timing = ws_timing{};
  c->pin_up.reset();
  try {
    if (cudaSetDevice(c->device) != cudaSuccess) throw Fail{WS_NO_DEVICE, "cudaSetDevice"};
    f();
  } catch (const Fail& e) {
    c->err = e.msg;
    cudaGetLastError();
    c->ticket_zeroed = nullptr;  // a failed call may leave launch state behind: re-zero
    return e.code;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    c->ticket_zeroed = nullptr;
    return WS_OUT_OF_MEMORY;
  } catch (...) {
    c->err = "unknown failure";
    c->ticket_zeroed = nullptr;
    return WS_CUDA;
  }
  c->timing.total_ms = t.ms();
  return WS_OK;
}

void add_prelude(uint64_t L, uint64_t R, ws_checks* o) {  // engine.cpp:268-276
  for (uint64_t v : {uint64_t{2}, uint64_t{3}})
    if (v >= L && v < R) {
      o->count += 1;
      o->sum += v;
      o->xor_ ^= v;
      o->largest = std::max(o->largest, v);
    }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Host-output enumeration as a pipeline: [L, R) is cut into up to
// kMaxChunks chunks on segment borders; every chunk's sieve launch is queued
// at once on the compute stream, and as each chunk finishes its values are
// copied device->host on the copy stream while later chunks still sieve, so
// the PCIe transfer (the bound for large outputs) hides the kernels.
// Wire variant of the pipeline (ws_wire.cpp): the chunks' kernels write one
// byte per prime + one count byte per 128-slot block + per-segment totals;
// each chunk crosses PCIe at ~1 byte per prime and the host pool widens it
// into `out` while later pieces copy.
void enumerate_wire(ws_ctx* c, uint64_t nseg, uint64_t nch, const std::vector<uint64_t>& lo,
                    const std::vector<uint64_t>& hi, const std::vector<uint64_t>& boff,
                    uint64_t* out, uint64_t cap, ws_checks* chk) {
  const uint64_t bps = c->S / wsk::kWireBlockSlots;
  c->wire.reserve(boff[nch] + 64, "wire entries");
  c->wblk.reserve(nseg * bps, "wire block counts");
  c->per_seg.reserve(nseg, "per-segment counts");
  uint8_t* pb = static_cast<uint8_t*>(c->pin_wblk.reserve(nseg * bps + 64, "pinned wire"));
  const size_t acc_bytes = (nch * sizeof(wsk::JobAcc) + 63) / 64 * 64;
  char* hout = static_cast<char*>(c->pin_out.reserve(acc_bytes + nseg * 4 + 64, "pinned out"));
  wsk::JobAcc* hacc = reinterpret_cast<wsk::JobAcc*>(hout);
  uint32_t* hseg = reinterpret_cast<uint32_t*>(hout + acc_bytes);  // per-segment totals
  std::vector<uint64_t> seg0(nch + 1), k0(nch);
  for (uint64_t k = 0; k <= nch; ++k) seg0[k] = k * nseg / nch;
  // blocks past a clipped last segment are never written
  ck(cudaMemsetAsync(c->wblk.ptr, 0, nseg * bps, c->stream), "zero wire counts");
  for (uint64_t k = 0; k < nch; ++k) {
    const wsk::Job J = make_job(lo[k], hi[k], c->S, 0);
    k0[k] = J.K0;
    c->h_jobs.assign(1, J);
    WireArgs wa{c->wire.ptr + boff[k], c->wblk.ptr + seg0[k] * bps};
    run_sieve(c, wsk::kEnumWire, c->per_seg.ptr + seg0[k], nullptr, boff[k + 1] - boff[k], true,
              static_cast<uint32_t>(k), k == 0, &wa);
    // accumulators and segment totals straight into mapped pinned memory: no
    // copy-engine entry on the compute stream to queue behind earlier
    // chunks' payload copies
    const uint32_t ns = static_cast<uint32_t>(seg0[k + 1] - seg0[k]);
    ck(wsk::launch_acc_to_host(c->acc.ptr + k, hacc + k, 1, c->stream), "chunk acc");
    ck(wsk::launch_u32_to_host(c->per_seg.ptr + seg0[k], hseg + seg0[k], ns, c->stream),
       "chunk totals");
    c->timing.launches += 2;
    c->timing.d2h_bytes += sizeof(wsk::JobAcc) + 4ull * ns;
    ck(cudaEventRecord(c->chunk_done[k], c->stream), "event");
  }
  if (!c->pool) c->pool = wswire::pool_create(0);
  // Payload pieces of `piece` entries cross into a ring of `ring` pinned
  // slots, each expanded as soon as it lands and reused once expanded: a
  // small reused staging set instead of one buffer of the whole payload
  // leaves more of the host's memory bandwidth to the 8-byte output.
  const uint64_t piece = c->wire_piece, ring = c->wire_ring;
  uint8_t* slots = static_cast<uint8_t*>(c->pin_wire.reserve(piece * ring + 64, "pinned wire ring"));
  while (c->ring_ev.size() < ring) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    c->ring_ev.push_back(e);
  }
  std::vector<wswire::Ticket> tickets(ring);
  std::vector<uint64_t> opos(nch, 0), take(nch, 0);
  std::vector<std::vector<uint64_t>> seg_off(nch);
  std::vector<wswire::WireChunk> chunks(nch);
  struct Piece {
    uint64_t k, a, m, slot;
  };
  std::vector<Piece> issued;
  uint64_t kc = 0, ac = 0, pos = 0;
  bool started = false;
  // issues the next piece's D2H into the next ring slot; false when done
  auto issue_next = [&]() -> bool {
    while (kc < nch) {
      if (!started) {
        ck(cudaEventSynchronize(c->chunk_done[kc]), "chunk");
        const uint64_t n = hacc[kc].count;
        if (n > boff[kc + 1] - boff[kc]) throw Fail{WS_CUDA, "wire chunk exceeds its bound"};
        const uint64_t ns = seg0[kc + 1] - seg0[kc];
        seg_off[kc].assign(ns + 1, 0);
        for (uint64_t s = 0; s < ns; ++s) seg_off[kc][s + 1] = seg_off[kc][s] + hseg[seg0[kc] + s];
        if (seg_off[kc][ns] != n) throw Fail{WS_CUDA, "wire segment totals disagree"};
        chunks[kc] = wswire::WireChunk{pb + seg0[kc] * bps, seg_off[kc].data(), ns, bps, k0[kc]};
        take[kc] = pos < cap ? std::min(n, cap - pos) : 0;
        opos[kc] = pos;
        pos += n;
        chk->count += n;
        chk->sum += hacc[kc].sum;
        chk->xor_ ^= hacc[kc].xr;
        chk->largest = std::max<uint64_t>(chk->largest, hacc[kc].largest);
        if (take[kc])
          ck(copy_async(c, pb + seg0[kc] * bps, c->wblk.ptr + seg0[kc] * bps, ns * bps,
                        cudaMemcpyDeviceToHost, c->cstream), "wire d2h");
        started = true;
        ac = 0;
      }
      if (ac < take[kc]) {
        const uint64_t slot = issued.size() % ring;
        if (issued.size() >= ring) wswire::ticket_wait(c->pool, &tickets[slot]);  // slot free
        const uint64_t m = std::min(piece, take[kc] - ac);
        ck(copy_async(c, slots + slot * piece, c->wire.ptr + boff[kc] + ac, m,
                      cudaMemcpyDeviceToHost, c->cstream), "wire d2h");
        ck(cudaEventRecord(c->ring_ev[slot], c->cstream), "event");
        issued.push_back(Piece{kc, ac, m, slot});
        ac += m;
        return true;
      }
      ++kc;
      started = false;
    }
    return false;
  };
  try {
    for (uint64_t r = 0; r + 1 < ring && issue_next(); ++r) {
    }
    for (size_t j = 0; j < issued.size(); ++j) {
      const Piece pc = issued[j];
      ck(cudaEventSynchronize(c->ring_ev[pc.slot]), "wire d2h");
      // the piece holds entries [a, a + m) of chunk k
      wswire::submit_expand(c->pool, chunks[pc.k], slots + pc.slot * piece, pc.a, pc.m,
                            out + opos[pc.k] + pc.a, &tickets[pc.slot]);
      issue_next();  // into the slot of piece j + 1 - ring (waits for its expansion)
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    ck(cudaGetLastError(), "kernel");
  } catch (...) {
    wswire::pool_wait(c->pool);  // no task may outlive the call
    throw;
  }
  wswire::pool_wait(c->pool);
  c->timing.base_primes = c->nprimes + small_primes_upto(c->base_B);
}

void enumerate_to_host(ws_ctx* c, uint64_t L, uint64_t R, uint64_t* out, uint64_t cap,
                       ws_checks* chk) {
  const wsk::Job whole = make_job(L, R, c->S, 0);
  const uint64_t nseg = whole.nseg;
  const uint64_t nch = std::max<uint64_t>(1, std::min<uint64_t>(ws_ctx::kMaxChunks, nseg / 64));
  std::vector<uint64_t> lo(nch), hi(nch), boff(nch + 1, 0);
  const uint64_t lo0 = L / 6 * 6;
  for (uint64_t k = 0; k < nch; ++k) {
    const uint64_t a = k * nseg / nch, b = (k + 1) * nseg / nch;
    lo[k] = k == 0 ? L : std::min<uint64_t>(R, lo0 + 6ull * c->S * a);
    hi[k] = k + 1 == nch ? R : std::min<uint64_t>(R, lo0 + 6ull * c->S * b);
    boff[k + 1] = boff[k] + prime_count_bound(lo[k], hi[k]);
  }
  // large outputs (several chunks) cross PCIe in the wire format
  if (c->host_wire && nch > 1)
    return enumerate_wire(c, nseg, nch, lo, hi, boff, out, cap, chk);
  c->vals.reserve(std::max<uint64_t>(boff[nch], 1), "enumeration buffer");
  wsk::JobAcc* hacc = static_cast<wsk::JobAcc*>(
      c->pin_out.reserve(nch * sizeof(wsk::JobAcc) + 16, "pinned out"));
  for (uint64_t k = 0; k < nch; ++k) {
    c->h_jobs.assign(1, make_job(lo[k], hi[k], c->S, 0));
    run_sieve(c, wsk::kEnumerate, nullptr, c->vals.ptr + boff[k], boff[k + 1] - boff[k], true,
              static_cast<uint32_t>(k), k == 0);
    // accumulators straight into mapped pinned memory: no copy-engine entry
    // on the compute stream to queue behind earlier chunks' payload copies
    ck(wsk::launch_acc_to_host(c->acc.ptr + k, hacc + k, 1, c->stream), "chunk acc");
    c->timing.launches += 1;
    c->timing.d2h_bytes += sizeof(wsk::JobAcc);
    ck(cudaEventRecord(c->chunk_done[k], c->stream), "event");
  }
  uint64_t pos = 0;
  for (uint64_t k = 0; k < nch; ++k) {
    ck(cudaEventSynchronize(c->chunk_done[k]), "chunk");
    const uint64_t n = hacc[k].count;
    const uint64_t take = pos < cap ? std::min(n, cap - pos) : 0;
    if (take)
      ck(copy_async(c, out + pos, c->vals.ptr + boff[k], take * 8, cudaMemcpyDeviceToHost,
                    c->cstream), "d2h");
    pos += n;
    chk->count += n;
    chk->sum += hacc[k].sum;
    chk->xor_ ^= hacc[k].xr;
    chk->largest = std::max<uint64_t>(chk->largest, hacc[k].largest);
  }
  ck(cudaStreamSynchronize(c->cstream), "d2h sync");
  ck(cudaStreamSynchronize(c->stream), "sync");
  ck(cudaGetLastError(), "kernel");
  c->timing.base_primes = c->nprimes + small_primes_upto(c->base_B);
}

}  // namespace

extern "C" {

const char* ws_version(void) { return "wheelsieve-b200 0.1 (sm_100a)"; }

void ws_opts_default(ws_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->struct_size = sizeof(ws_opts);
  o->segment_slots = 1u << 18;
  o->device = -1;
}

const char* ws_status_name(ws_status s) {
  switch (s) {
    case WS_OK: return "ok";
    case WS_NOT_ON_WHEEL: return "NotOnWheel";
    case WS_OVERFLOW: return "Overflow";
    case WS_EMPTY_RANGE: return "EmptyRange";
    case WS_CAPACITY: return "Capacity";
    case WS_DOMAIN: return "Domain";
    case WS_ALIGNMENT: return "Alignment";
    case WS_BAD_CONFIG: return "BadConfig";
    case WS_INCOMPLETE_BASE: return "IncompleteBase";
    case WS_ORDERING: return "Ordering";
    case WS_IO: return "Io";
    case WS_BAD_MANIFEST: return "BadManifest";
    case WS_CHECKSUM_MISMATCH: return "ChecksumMismatch";
    case WS_BEYOND_FRONTIER: return "BeyondFrontier";
    case WS_CUDA: return "Cuda";
    case WS_NO_DEVICE: return "NoDevice";
    case WS_OUT_OF_MEMORY: return "OutOfMemory";
  }
  return "unknown";
}

ws_status ws_ctx_create(const ws_opts* opts, ws_ctx** out) {
  if (!out) return WS_BAD_CONFIG;
  *out = nullptr;
  ws_opts o;
  ws_opts_default(&o);
  if (opts) {
    if (opts->struct_size != sizeof(ws_opts)) return WS_BAD_CONFIG;
    o = *opts;
  }
  const uint32_t S = o.segment_slots;
  if (S < (1u << 12) || S > (1u << 18) || (S & (S - 1))) return WS_BAD_CONFIG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return WS_NO_DEVICE;
  }
  int dev = o.device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return WS_NO_DEVICE;
  if (dev >= ndev) return WS_NO_DEVICE;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return WS_NO_DEVICE;
  if (prop.major != 10) return WS_NO_DEVICE;  // built for sm_100a only
  ws_ctx* c = new (std::nothrow) ws_ctx;
  if (!c) return WS_OUT_OF_MEMORY;
  c->device = dev;
  c->S = S;
  {  // primes in [37, S): the in-kernel share of the table; and the warp-
     // cooperative share [37, wc_limit)
    // primes below bucket_pmin = ratio * S stay in the kernel even when the
    // large ones are bucketed (p in [S, pmin) through the loop-free one-hit
    // path): a bucketed hit costs ~90 instructions (fill + apply); measured
    // optimum ratio 2 for c4 and c5 (sweep over 1..8)
    uint32_t wc_limit = 1024, pmin_ratio = 2;
    if (const char* e = std::getenv("WHEELSIEVE_WC_LIMIT")) wc_limit = std::strtoul(e, nullptr, 10);
    if (const char* e = std::getenv("WHEELSIEVE_BUCKET_PMIN")) pmin_ratio = std::strtoul(e, nullptr, 10);
    const uint32_t pmin = S * std::max<uint32_t>(1, pmin_ratio);
    const uint32_t n_max = std::max(pmin, wc_limit);
    std::vector<uint8_t> comp(n_max, 0);
    uint32_t n = 0, nw = 0, ns = 0;
    for (uint32_t i = 2; i < n_max; ++i) {
      if (comp[i]) continue;
      if (i >= wsk::kFirstTablePrime && i < pmin) ++n;
      if (i >= wsk::kFirstTablePrime && i < S) ++ns;
      if (i >= wsk::kFirstTablePrime && i < wc_limit) ++nw;
      for (uint64_t j = static_cast<uint64_t>(i) * i; j < n_max; j += i) comp[j] = 1;
    }
    c->n_below_S = n;
    c->n_S = ns;
    c->n_wc = nw;
    c->bucket_pmin = pmin;
  }
  // test / tuning knobs: bucket-list capacity per segment and window budget
  if (const char* e = std::getenv("WHEELSIEVE_BUCKET_CAP")) c->cap_override = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_BUCKET_BUDGET")) c->bucket_budget = std::strtoull(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_FILL_PIECE")) c->piece_override = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_FILL_HUGE")) c->fill_huge = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_HUGE_FROM")) c->huge_from = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_HUGE_STEP"))
    c->huge_step = std::max<uint32_t>(1, std::min<uint32_t>(64, std::strtoul(e, nullptr, 10)));
  if (const char* e = std::getenv("WHEELSIEVE_BUCKET_RATIO")) c->bucket_min_ratio = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_BUCKET_CTAS")) c->bucket_ctas_per_sm = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_CTAS_PER_SM")) c->ctas_per_sm = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_HOST_WIRE")) c->host_wire = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_BASE_EXTEND")) c->base_extend = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_WIRE_PIECE"))
    c->wire_piece = std::max<uint64_t>(1024, std::strtoull(e, nullptr, 10));
  if (const char* e = std::getenv("WHEELSIEVE_WIRE_RING"))
    c->wire_ring = std::max<uint64_t>(2, std::strtoull(e, nullptr, 10));
  c->sms = prop.multiProcessorCount;
  if (cudaSetDevice(dev) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      wsk::sieve_configure(c->bps) != cudaSuccess) {
    delete c;
    cudaGetLastError();
    return WS_CUDA;
  }
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) {
      delete c;
      return WS_CUDA;
    }
  bool ok = cudaStreamCreateWithFlags(&c->fstream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->bstream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_order, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; i < ws_ctx::kMaxChunks && ok; ++i)
    ok = cudaEventCreateWithFlags(&c->chunk_done[i], cudaEventDisableTiming) == cudaSuccess;
  if (ok) {
    std::vector<uint32_t> tab(wsk::small_table_words());
    wsk::build_small_tables(tab.data());
    try {
      c->small_tab.reserve(tab.size(), "small tables");
    } catch (const Fail&) {
      ok = false;
    }
    ok = ok && cudaMemcpy(c->small_tab.ptr, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) ==
                   cudaSuccess;
  }
  for (int i = 0; i < 2 && ok; ++i)
    ok = cudaEventCreateWithFlags(&c->fill_done[i], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->sieve_done[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    delete c;
    return WS_CUDA;
  }
  *out = c;
  return WS_OK;
}

void ws_ctx_destroy(ws_ctx* ctx) { delete ctx; }

const char* ws_last_error(const ws_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* ws_ctx_stream(ws_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

ws_status ws_last_timing(const ws_ctx* ctx, ws_timing* out) {
  if (!ctx || !out) return WS_BAD_CONFIG;
  *out = ctx->timing;
  return WS_OK;
}

uint64_t ws_isqrt(uint64_t n) { return isqrt_u64(n); }

uint64_t ws_prime_count_bound(uint64_t L, uint64_t R) { return prime_count_bound(L, R); }

ws_status ws_start_offsets(uint64_t p, uint64_t start, uint64_t* id1, uint64_t* id5) {
  // wheel.cpp:96-106 semantics; computed with the k-residue form of Table 1
  if (!id1 || !id5) return WS_BAD_CONFIG;
  if (p % 6 != 1 && p % 6 != 5) return WS_DOMAIN;
  if (start % 6 != 0) return WS_ALIGNMENT;
  if (start <= p) return WS_DOMAIN;
  const uint64_t R6 = p / 6;
  const uint64_t t1 = p % 6 == 1 ? R6 : 5 * R6 + 4;
  const uint64_t t5 = p % 6 == 1 ? 5 * R6 : R6;
  const uint64_t k0 = start / 6;
  const uint64_t r = k0 % p;
  *id1 = k0 + (t1 >= r ? t1 - r : t1 + p - r);
  *id5 = k0 + (t5 >= r ? t5 - r : t5 + p - r);
  return WS_OK;
}

ws_status ws_partition(uint64_t L, uint64_t R, uint32_t S, uint32_t rank, uint32_t world,
                       uint64_t* lo, uint64_t* hi) {
  if (!lo || !hi || world == 0 || rank >= world || S == 0) return WS_BAD_CONFIG;
  if (R <= L) {
    *lo = *hi = L;
    return WS_OK;
  }
  if (R > kMaxSegmentEnd) return WS_OVERFLOW;
  const uint64_t lo0 = L / 6 * 6;
  const uint64_t nslots = (R - lo0 + 5) / 6;
  const uint64_t nseg = (nslots + S - 1) / S;
  auto seg_at = [&](uint64_t r) {  // balanced: floor(r * nseg / world)
    const unsigned __int128 x = static_cast<unsigned __int128>(r) * nseg / world;
    return static_cast<uint64_t>(x);
  };
  const uint64_t a = seg_at(rank), b = seg_at(rank + 1ull);
  *lo = rank == 0 ? L : std::min<uint64_t>(R, lo0 + 6ull * S * a);
  *hi = rank + 1 == world ? R : std::min<uint64_t>(R, lo0 + 6ull * S * b);
  if (*lo < L) *lo = L;
  if (*hi < *lo) *hi = *lo;
  return WS_OK;
}

ws_status ws_count_range(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, ws_checks* out,
                         uint32_t* per_seg, uint64_t per_seg_cap, uint64_t* n_seg) {
  return guarded(ctx, [&] {
    if (!out) throw Fail{WS_BAD_CONFIG, "null output"};
    *out = ws_checks{};
    if (n_seg) *n_seg = 0;
    if (R <= L) return;
    validate_range(L, R);
    const bool fresh = flags & WS_FRESH_BASE;
    ensure_base(ctx, R >= 2 ? isqrt_u64(R - 1) : 0, fresh);
    ctx->h_jobs.assign(1, make_job(L, R, ctx->S, 0));
    const uint64_t nseg = ctx->h_jobs[0].nseg;
    uint32_t* dps = nullptr;
    const bool dev_out = flags & WS_OUT_DEVICE;
    if (per_seg) {
      if (dev_out) {
        if (per_seg_cap < nseg) throw Fail{WS_CAPACITY, "per_seg capacity below segment count"};
        dps = per_seg;
      } else {
        ctx->per_seg.reserve(nseg, "per_seg");
        dps = ctx->per_seg.ptr;
      }
    }
    const int mode = (flags & WS_WANT_CHECKS) ? wsk::kCountChecks : wsk::kCount;
    run_sieve(ctx, mode, dps, nullptr, 0, true);
    if (per_seg && !dev_out)
      ck(copy_async(ctx, per_seg, dps, std::min(nseg, per_seg_cap) * sizeof(uint32_t),
                         cudaMemcpyDeviceToHost, ctx->stream), "per_seg");
    const wsk::JobAcc a = *fetch_results(ctx, 1);
    out->count = a.count;
    out->sum = a.sum;
    out->xor_ = a.xr;
    out->largest = a.largest;
    add_prelude(L, R, out);
    if (n_seg) *n_seg = nseg;
    ctx->timing.base_ms = ctx->base_built ? event_ms(ctx->ev[0], ctx->ev[1]) : 0.0;
    ctx->timing.sieve_ms = event_ms(ctx->ev[2], ctx->ev[3]);
  });
}

ws_status ws_enumerate_range(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, uint64_t* out,
                             uint64_t cap, uint64_t* n_out, ws_checks* checks) {
  ws_status st = guarded(ctx, [&] {
    if (!n_out) throw Fail{WS_BAD_CONFIG, "null n_out"};
    *n_out = 0;
    ws_checks chk{};
    if (checks) *checks = chk;
    if (R <= L) return;
    if (!out && cap) throw Fail{WS_BAD_CONFIG, "null output with nonzero capacity"};
    validate_range(L, R);
    ensure_base(ctx, R >= 2 ? isqrt_u64(R - 1) : 0, flags & WS_FRESH_BASE);
    uint64_t pre[2];
    uint64_t npre = 0;
    for (uint64_t v : {uint64_t{2}, uint64_t{3}})
      if (v >= L && v < R) pre[npre++] = v;
    ctx->h_jobs.assign(1, make_job(L, R, ctx->S, 0));
    const bool dev_out = flags & WS_OUT_DEVICE;
    if (dev_out && out && !is_device_ptr(out))
      throw Fail{WS_BAD_CONFIG, "WS_OUT_DEVICE with a non-device pointer"};
    unsigned long long* dst;
    uint64_t dcap;
    if (dev_out) {
      dst = reinterpret_cast<unsigned long long*>(out) + std::min(npre, cap);
      dcap = cap > npre ? cap - npre : 0;
      if (npre && cap)
        ck(copy_async(ctx, out, pre, std::min(npre, cap) * 8, cudaMemcpyHostToDevice,
                      ctx->stream), "prelude");
    } else {
      for (uint64_t i = 0; i < npre && i < cap; ++i) out[i] = pre[i];
      enumerate_to_host(ctx, L, R, out + std::min(npre, cap), cap > npre ? cap - npre : 0, &chk);
      add_prelude(L, R, &chk);
      *n_out = chk.count;
      if (checks) *checks = chk;
      ctx->timing.base_ms = ctx->base_built ? event_ms(ctx->ev[0], ctx->ev[1]) : 0.0;
      ctx->timing.sieve_ms = event_ms(ctx->ev[2], ctx->ev[3]);
      if (chk.count > cap) throw Fail{WS_CAPACITY, "output capacity below the prime count"};
      return;
    }
    run_sieve(ctx, wsk::kEnumerate, nullptr, dst, dcap, true);
    const wsk::JobAcc a = *fetch_results(ctx, 1);
    chk.count = a.count;
    chk.sum = a.sum;
    chk.xor_ = a.xr;
    chk.largest = a.largest;
    add_prelude(L, R, &chk);
    *n_out = chk.count;
    if (checks) *checks = chk;
    ctx->timing.base_ms = ctx->base_built ? event_ms(ctx->ev[0], ctx->ev[1]) : 0.0;
    ctx->timing.sieve_ms = event_ms(ctx->ev[2], ctx->ev[3]);
    if (chk.count > cap) throw Fail{WS_CAPACITY, "output capacity below the prime count"};
  });
  return st;
}

ws_status ws_base_primes(ws_ctx* ctx, uint64_t B, uint32_t flags, uint64_t* out, uint64_t cap,
                         uint64_t* n) {
  return guarded(ctx, [&] {
    if (!n) throw Fail{WS_BAD_CONFIG, "null n"};
    *n = 0;
    if (B < 2) throw Fail{WS_EMPTY_RANGE, "no primes below 2"};  // wheel.cpp:41
    if (B > 0xFFFFFFFFull) throw Fail{WS_CAPACITY, "base bound above 2^32"};
    // the store's entries are the wheel primes 5 <= p <= B (base_store.cpp:34-42):
    // enumerate [5, B + 1) on the device
    if (B < 5) return;
    ws_checks chk{};
    const uint32_t f = (flags & (WS_OUT_DEVICE | WS_FRESH_BASE));
    const ws_status st = ws_enumerate_range(ctx, 5, B + 1, f, out, cap, n, &chk);
    if (st != WS_OK) throw Fail{st, ctx->err};
  });
}

ws_status ws_sieve_segment(ws_ctx* ctx, uint64_t start, uint64_t len, uint32_t flags,
                           uint64_t* r1_words, uint64_t* r5_words) {
  return guarded(ctx, [&] {
    // SegmentBitmap checks, segment.cpp:101-110
    if (start % 6 != 0) throw Fail{WS_ALIGNMENT, "segment start is not a multiple of 6"};
    if (len == 0) throw Fail{WS_DOMAIN, "segment must span at least one wheel index"};
    if (len > (kMaxSegmentEnd - start) / 6)
      throw Fail{WS_OVERFLOW, "segment end exceeds the 64-bit value range"};
    if (!r1_words || !r5_words) throw Fail{WS_BAD_CONFIG, "null output"};
    const uint64_t end = start + 6 * len;
    ensure_base(ctx, isqrt_u64(end - 1), flags & WS_FRESH_BASE);
    ctx->h_jobs.assign(1, make_job(start, end, ctx->S, 0));
    const uint64_t nseg = ctx->h_jobs[0].nseg;
    const uint64_t words32 = nseg * (ctx->S / 32);
    const uint64_t out64 = (len + 63) / 64;
    const bool dev_out = flags & WS_OUT_DEVICE;
    DevBuf<uint32_t> tmp;
    tmp.reserve(2 * words32 + 2, "bitmap words");
    ctx->words_out[0] = tmp.ptr;
    ctx->words_out[1] = tmp.ptr + words32;
    try {
      run_sieve(ctx, wsk::kCount, nullptr, nullptr, 0, true);
    } catch (...) {
      ctx->words_out[0] = ctx->words_out[1] = nullptr;
      tmp.release();
      throw;
    }
    ctx->words_out[0] = ctx->words_out[1] = nullptr;
    // uint32 LSB-first words are byte-identical to FlagArray's uint64 words
    const cudaMemcpyKind k = dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    ck(copy_async(ctx, r1_words, tmp.ptr, out64 * 8, k, ctx->stream), "r1 words");
    ck(copy_async(ctx, r5_words, tmp.ptr + words32, out64 * 8, k, ctx->stream), "r5 words");
    fetch_results(ctx, 1);
    tmp.release();
    // sieve_segment leaves the value 1 set; callers clear it (engine.cpp:244)
    if (start == 0) {
      if (dev_out) {
        uint64_t w0 = 0;
        ck(copy_sync(ctx, &w0, r1_words, 8, cudaMemcpyDeviceToHost), "w0");
        w0 |= 1;
        ck(copy_sync(ctx, r1_words, &w0, 8, cudaMemcpyHostToDevice), "w0");
      } else {
        r1_words[0] |= 1;
      }
    }
    ctx->timing.sieve_ms = event_ms(ctx->ev[2], ctx->ev[3]);
  });
}

ws_status ws_count_intervals(ws_ctx* ctx, const uint64_t* Ls, uint64_t n, uint64_t width,
                             uint32_t flags, uint32_t* counts, uint64_t* sums, uint64_t* xors) {
  return guarded(ctx, [&] {
    if (n == 0) return;
    if (!Ls || !counts) throw Fail{WS_BAD_CONFIG, "null interval arrays"};
    if (width == 0) throw Fail{WS_EMPTY_RANGE, "zero-width intervals"};
    const bool dev_out = flags & WS_OUT_DEVICE;
    std::vector<uint64_t> hL;
    const uint64_t* L = Ls;
    if (dev_out) {
      hL.resize(n);
      ck(copy_sync(ctx, hL.data(), Ls, n * 8, cudaMemcpyDeviceToHost), "intervals in");
      L = hL.data();
    }
    uint64_t maxR = 0, seg = 0;
    ctx->h_jobs.clear();
    ctx->h_jobs.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
      if (L[i] > kMaxSegmentEnd - width) throw Fail{WS_OVERFLOW, "interval end overflows"};
      const uint64_t R = L[i] + width;
      maxR = std::max(maxR, R);
      ctx->h_jobs.push_back(make_job(L[i], R, ctx->S, seg));
      seg += ctx->h_jobs.back().nseg;
    }
    ensure_base(ctx, maxR >= 2 ? isqrt_u64(maxR - 1) : 0, flags & WS_FRESH_BASE);
    // ensure_base may have used h_jobs for the base sieve: rebuild
    ctx->h_jobs.clear();
    seg = 0;
    for (uint64_t i = 0; i < n; ++i) {
      ctx->h_jobs.push_back(make_job(L[i], L[i] + width, ctx->S, seg));
      seg += ctx->h_jobs.back().nseg;
    }
    const bool checks = sums || xors;
    run_sieve(ctx, checks ? wsk::kCountChecks : wsk::kCount, nullptr, nullptr, 0, true);
    const wsk::JobAcc* acc = fetch_results(ctx, n);
    std::vector<uint32_t> hc(n);
    std::vector<uint64_t> hs(n), hx(n);
    for (uint64_t i = 0; i < n; ++i) {
      ws_checks o{acc[i].count, acc[i].sum, acc[i].xr, acc[i].largest};
      add_prelude(L[i], L[i] + width, &o);
      hc[i] = static_cast<uint32_t>(o.count);
      hs[i] = o.sum;
      hx[i] = o.xor_;
    }
    if (dev_out) {
      ck(copy_sync(ctx, counts, hc.data(), n * 4, cudaMemcpyHostToDevice), "counts");
      if (sums) ck(copy_sync(ctx, sums, hs.data(), n * 8, cudaMemcpyHostToDevice), "sums");
      if (xors) ck(copy_sync(ctx, xors, hx.data(), n * 8, cudaMemcpyHostToDevice), "xors");
    } else {
      std::memcpy(counts, hc.data(), n * 4);
      if (sums) std::memcpy(sums, hs.data(), n * 8);
      if (xors) std::memcpy(xors, hx.data(), n * 8);
    }
    ctx->timing.base_ms = ctx->base_built ? event_ms(ctx->ev[0], ctx->ev[1]) : 0.0;
    ctx->timing.sieve_ms = event_ms(ctx->ev[2], ctx->ev[3]);
  });
}

}  // extern "C"
