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
#include <dlfcn.h>

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
#include "ws_host.h"
#include "ws_internal.h"
#include "ws_wire.h"

namespace wsh {

const NcclApi* nccl_api() {
  static const NcclApi* api = [] () -> const NcclApi* {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return nullptr;
    static NcclApi a;
    bool ok = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      ok = ok && fn != nullptr;
    };
    get(a.GetUniqueId, "ncclGetUniqueId");
    get(a.CommInitAll, "ncclCommInitAll");
    get(a.CommInitRank, "ncclCommInitRank");
    get(a.CommDestroy, "ncclCommDestroy");
    get(a.GroupStart, "ncclGroupStart");
    get(a.GroupEnd, "ncclGroupEnd");
    get(a.AllGather, "ncclAllGather");
    get(a.CommCount, "ncclCommCount");
    get(a.CommUserRank, "ncclCommUserRank");
    get(a.GetErrorString, "ncclGetErrorString");
    return ok ? &a : nullptr;
  }();
  return api;
}

}  // namespace wsh

using namespace wsh;

namespace {

// Every host<->device copy goes through these, so ws_timing reports the
// bytes that crossed PCIe in the last call.
cudaError_t copy_async(DevCtx* c, void* dst, const void* src, size_t n, cudaMemcpyKind k,
                       cudaStream_t st) {
  if (k == cudaMemcpyHostToDevice) c->timing.h2d_bytes += n;
  if (k == cudaMemcpyDeviceToHost) c->timing.d2h_bytes += n;
  return cudaMemcpyAsync(dst, src, n, k, st);
}
cudaError_t copy_sync(DevCtx* c, void* dst, const void* src, size_t n, cudaMemcpyKind k) {
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
uint32_t table_primes_below(DevCtx* c, uint64_t x) {
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
void join_base(DevCtx* c) {
  if (!c->base_pending) return;
  ck(cudaStreamWaitEvent(c->stream, c->ev[1], 0), "base join");
  c->base_pending = false;
}

struct WireArgs {  // kEnumWire outputs
  uint8_t* entries;
  uint8_t* blk8;
};

// A call's timing events (ev[2] start, ev[3] end of the sieve): while the
// stream is being captured into a graph they become event-record nodes, so a
// replayed call still times its sieve.
void record_timing_event(DevCtx* c, cudaEvent_t e) {
  ck(c->capturing ? cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal)
                  : cudaEventRecord(e, c->stream),
     "event");
}

void run_sieve(DevCtx* c, int mode, uint32_t* per_seg_dev, unsigned long long* out,
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
  p.single_pred = c->single_pred;
  p.mid_bitaddr = c->mid_bitaddr;
  p.miss_lane = c->miss_lane;
  p.skip5_max = c->skip5_max;
  p.seg_trans = c->seg_trans;
  p.trans_min = c->seg_trans_min;
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
  uint64_t pmin = c->bucket_pmin;
  bool buckets = c->nprimes > p.n_mid && c->base_B > pmin &&
                 c->base_B >= static_cast<uint64_t>(c->bucket_min_ratio) * c->S;
  // wide units (sieve_wide_kernel): single-job count launches without bucket
  // lists, long enough to keep every SM's lone CTA busy for many units
  const uint32_t wide_want = buckets ? c->wide_bucket : (nj > 1 ? c->wide_multi : c->wide);
  if (wide_want > 1 && mode <= wsk::kCountChecks && c->S == (1u << 18) &&
      c->words_out[0] == nullptr && nseg < (1ull << 28) && nseg >= 6 * nj &&
      nseg >= static_cast<uint64_t>(c->wide_min_units) * wide_want * c->sms) {
    p.wide = std::min<uint32_t>(wide_want, wsk::kWideMax);
    p.n_S = std::min<uint32_t>(
        std::max(table_primes_below(c, static_cast<uint64_t>(p.wide) * c->S), p.n_wc), c->nprimes);
    if (c->wide_double) {  // primes of at least half a unit: at most 2 hits per class, no loop
      const uint64_t unit = static_cast<uint64_t>(p.wide) * c->S;
      p.n_dbl = p.n_S;
      p.n_S = std::min<uint32_t>(std::max(table_primes_below(c, (unit + 1) / 2), p.n_wc), p.n_dbl);
    }
    // a unit pays the in-kernel visit of a large prime once per three segments,
    // so bucketing starts higher: 6 S instead of 2 S (C4 47.4 -> 43.0 ms, C5
    // 20.6 -> 19.4 ms; sweep over 2..16 S)
    const uint64_t pmin_w = static_cast<uint64_t>(c->wide_pmin_ratio) * c->S;
    if (buckets && pmin_w > pmin) {
      pmin = pmin_w;
      p.n_mid = std::min<uint32_t>(std::max(table_primes_below(c, pmin), p.n_wc), c->nprimes);
      buckets = c->nprimes > p.n_mid && c->base_B > pmin;
    }
    if (!buckets) p.n_mid = c->nprimes;
    p.miss_lane = 1;
    p.skip5_max = c->wide_skip5;
    p.trans_min = c->trans_min;
    p.seg_trans = 0;
    if (c->wide_n_wc) p.n_wc = std::min<uint32_t>(c->wide_n_wc, p.n_S);
    max_grid = c->sms;
  }
  uint64_t W = nseg;
  uint32_t cap = 0;
  if (buckets) {
    const double E = expected_large_hits(static_cast<uint32_t>(pmin), c->S,
                                         static_cast<double>(c->base_B));
    cap = static_cast<uint32_t>(1.1 * E + 8.0 * std::sqrt(E) + 1024);
    cap = (cap + 31) / 32 * 32;
    if (c->cap_override) cap = c->cap_override;
    W = std::max<uint64_t>(8, c->bucket_budget / (4ull * cap));
    W = std::min<uint64_t>({W, wsk::kMaxWindow, nseg});
    // the fill kernel indexes a window's lists with 32-bit entry indices
    const uint64_t w32 = ((1ull << 32) - (1ull << 26)) / cap;
    if (w32 < 2) throw Fail{WS_BAD_CONFIG, "bucket list capacity too large for 32-bit entry indices"};
    W = std::max<uint64_t>(1, std::min<uint64_t>(W, w32 - 1));
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
  bool staged = false;
  if (buckets) {
    // optional cap on sieve CTAs per SM to leave room for fill CTAs (measured: no gain)
    if (c->bucket_ctas_per_sm)
      max_grid = std::min<uint64_t>(max_grid, static_cast<uint64_t>(c->sms) * c->bucket_ctas_per_sm);
    // runs are cut into 32-segment pieces: short per-thread hit loops and a
    // fill grid that covers the GPU (measured best for c4 and c5)
    // (64 with the staged fills of a single-job window: their queues flush
    // whole chunks, so longer pieces keep write locality -- C4 51.3 -> 50.4 ms;
    // multi-job windows such as C5's keep the two-pass fills, where staging
    // measured slower: 22.5 vs 24.2 ms)
    staged = nj == 1 && c->stage_cap > 0;
    piece = c->piece_override ? c->piece_override : (staged ? 64 : 32);
    piece = std::min<uint64_t>(piece, W);
    // a run's span in slots is indexed in 32 bits by the fill kernels
    piece = std::max<uint64_t>(1, std::min<uint64_t>(piece, (0xFFFFFFFFull / c->S) - 1));
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
  // wide units over windows or several jobs: the launch's unit table
  std::vector<uint32_t> unit_off(nwin + 1, 0);
  if (p.wide > 1 && (buckets || nj > 1)) {
    std::vector<uint32_t> units;
    units.reserve(nseg / p.wide + nj + nwin);
    size_t j = 0;
    for (uint64_t w = 0; w < nwin; ++w) {
      const uint64_t ws = w * W, we = std::min(nseg, ws + W);
      while (j < nj && c->h_jobs[j].seg_begin + c->h_jobs[j].nseg <= ws) ++j;
      for (size_t q = j; q < nj && c->h_jobs[q].seg_begin < we; ++q) {
        const wsk::Job& J = c->h_jobs[q];
        const uint64_t a0 = std::max(ws, J.seg_begin), b0 = std::min(we, J.seg_begin + J.nseg);
        for (uint64_t x = a0; x < b0; x += p.wide)
          units.push_back(static_cast<uint32_t>(x - ws) |
                          static_cast<uint32_t>(std::min<uint64_t>(p.wide, b0 - x)) << 28);
      }
      unit_off[w + 1] = static_cast<uint32_t>(units.size());
    }
    c->units.reserve(std::max<size_t>(units.size(), 1), "units");
    void* hu = c->pin_up.alloc(units.size() * sizeof(uint32_t) + 4, "pinned units");
    std::memcpy(hu, units.data(), units.size() * sizeof(uint32_t));
    ck(copy_async(c, c->units.ptr, hu, units.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                  c->stream), "upload units");
  }
  // ev[2] (call start) / ev[4] order the fill stream after everything queued so far
  join_base(c);
  if (record_start) record_timing_event(c, c->ev[2]);
  if (buckets) {
    ck(cudaEventRecord(c->ev_order, c->stream), "event");
    ck(cudaStreamWaitEvent(c->fstream, c->ev_order, 0), "fill wait");
  }
  // primes of at least the run length take the carried-offset fill when every
  // run is a piece of the one job (consecutive in wheel slots)
  uint32_t huge_begin = c->nprimes;
  // (the one-check kernels -- the default -- take primes of at least the run
  // length only: a smaller WHEELSIEVE_HUGE_FROM needs WHEELSIEVE_HUGE_LOOP=1)
  uint64_t huge_segs = c->huge_from ? c->huge_from : piece;
  if (!c->huge_loop && c->huge_step == 1) huge_segs = std::max<uint64_t>(huge_segs, piece);
  const uint64_t huge_from = huge_segs * c->S;
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
      f.w_unroll = c->w_unroll;
      f.stage_cap = staged ? c->stage_cap : 0;
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
        fh.huge_loop = c->huge_loop;
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
    uint64_t units = p.wide > 1 ? (we - ws + p.wide - 1) / p.wide : we - ws;
    if (unit_off[nwin]) {
      p.units = c->units.ptr + unit_off[w];
      p.nunits = unit_off[w + 1] - unit_off[w];
      units = p.nunits;
    }
    const int grid = static_cast<int>(std::min<uint64_t>(units, max_grid));
    ck(wsk::launch_sieve(mode, p, grid, c->stream), "sieve launch");
    if (buckets) ck(cudaEventRecord(c->sieve_done[b], c->stream), "event");
    c->timing.launches += 1;
  }
  (void)timed;
  record_timing_event(c, c->ev[3]);
  c->timing.segments += nseg;
}

// Make the resident table cover every prime in [53, B].  No host round
// trip: the level-0 count and the table size stay on the device and the
// kernels read them (SieveParams::nprimes_dev); the host keeps upper bounds.
// Device-side BasePrimeStore::extend (base_store.cpp:44-69): the resident
// table [53, base_B] already covers sqrt(B), so only (base_B, B] is sieved --
// with that table -- and appended; the table size stays on the device.
void extend_base(DevCtx* c, uint64_t B) {
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

cudaError_t launch_small_base(DevCtx* c, uint32_t n, uint32_t* p, unsigned long long* m,
                              double* inv, uint32_t* count, cudaStream_t st) {
  if (!c->base_scratch.ptr) {
    c->base_scratch.reserve(64, "base scratch");
    ck(cudaMemset(c->base_scratch.ptr, 0, 64 * sizeof(unsigned long long)), "base scratch");
  }
  if (++c->base_epoch == 0) ++c->base_epoch;  // 0 marks "never written"
  return wsk::launch_small_base(n, p, m, inv, count, c->base_scratch.ptr, c->base_epoch, st);
}

void ensure_base(DevCtx* c, uint64_t B, bool fresh) {
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
  // level 0: primes in [53, isqrt(B)] (isqrt(B) < 2^16: at most 6542 - 11)
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
const wsk::JobAcc* fetch_results(DevCtx* c, size_t n) {
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
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();  // an unrecorded event is not a failure of the next call
    return 0;
  }
  return ms;
}

void reset_after_failure(ws_ctx* ctx) {
  cudaGetLastError();
  // a failed call may leave launch state behind: re-zero the tickets
  for (DevCtx* d : ctx->devs) d->ticket_zeroed = nullptr;
}

// Runs f() with the context's per-call state reset; a Fail (or any other
// exception) becomes a status + ws_last_error.  The caller's current device
// is restored on return.  ctx->timing aggregates the devices' timings (bytes,
// launches and segments summed; device times the maximum over devices).
template <class F>
ws_status guarded(ws_ctx* ctx, F&& f) {
  if (!ctx || ctx->devs.empty()) return WS_BAD_CONFIG;
  Timer t;
  ctx->err.clear();
  ctx->timing = ws_timing{};
  for (DevCtx* d : ctx->devs) {
    d->err.clear();
    d->timing = ws_timing{};
    d->pin_up.reset();
  }
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) {
    cudaGetLastError();
    prev = -1;
  }
  ws_status st = WS_OK;
  try {
    if (cudaSetDevice(ctx->devs[0]->device) != cudaSuccess) throw Fail{WS_NO_DEVICE, "cudaSetDevice"};
    f();
  } catch (const Fail& e) {
    ctx->err = e.msg;
    st = e.code;
  } catch (const std::bad_alloc&) {
    ctx->err = "host allocation failed";
    st = WS_OUT_OF_MEMORY;
  } catch (...) {
    ctx->err = "unknown failure";
    st = WS_CUDA;
  }
  if (st != WS_OK) reset_after_failure(ctx);
  ws_timing& T = ctx->timing;
  for (DevCtx* d : ctx->devs) {
    T.base_ms = std::max(T.base_ms, d->timing.base_ms);
    T.sieve_ms = std::max(T.sieve_ms, d->timing.sieve_ms);
    T.launches += d->timing.launches;
    T.segments += d->timing.segments;
    T.base_primes = std::max(T.base_primes, d->timing.base_primes);
    T.h2d_bytes += d->timing.h2d_bytes;
    T.d2h_bytes += d->timing.d2h_bytes;
  }
  T.total_ms = t.ms();
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

// fn(device context, local index) on every local device: inline for one
// device, else concurrently on the per-device worker threads.  Every device
// runs to completion before the first failure (by device order) is rethrown,
// so no device is left inside a collective its peers never enter.
void on_devices(ws_ctx* ctx, const std::function<void(DevCtx*, size_t)>& fn) {
  const size_t n = ctx->devs.size();
  if (n == 1 || !ctx->workers) {
    for (size_t i = 0; i < n; ++i) {
      ck(cudaSetDevice(ctx->devs[i]->device), "cudaSetDevice");
      fn(ctx->devs[i], i);
    }
    return;
  }
  std::vector<std::exception_ptr> errs(n);
  ctx->workers->run([&](size_t i) {
    try {
      ck(cudaSetDevice(ctx->devs[i]->device), "cudaSetDevice");
      fn(ctx->devs[i], i);
    } catch (...) {
      errs[i] = std::current_exception();
    }
  });
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void nccl_ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Fail{WS_NCCL, std::string(what) + ": " + nccl_api()->GetErrorString(r)};
}

// The context's one collective: every shard contributes n_per 32-byte
// JobAcc records (send[i]: device array of local device i, stream-ordered
// after the kernels that wrote it) and every device receives all
// nshards * n_per of them (shard-major) with one ncclAllGather per
// communicator, issued as one NCCL group from this thread.  Returns the
// gathered records on the host (device 0's copy).
std::vector<wsk::JobAcc> allgather_records(ws_ctx* ctx, const std::vector<const wsk::JobAcc*>& send,
                                           uint64_t n_per) {
  const uint64_t total = n_per * ctx->nshards;
  if (ctx->virt) {  // test mode: the same records, gathered through the host
    std::vector<wsk::JobAcc> all(total);
    for (size_t i = 0; i < ctx->devs.size(); ++i) {
      DevCtx* d = ctx->devs[i];
      ck(cudaSetDevice(d->device), "cudaSetDevice");
      auto* h = static_cast<wsk::JobAcc*>(d->pin_gather.reserve(n_per * sizeof(wsk::JobAcc), "pinned gather"));
      ck(copy_async(d, h, send[i], n_per * sizeof(wsk::JobAcc), cudaMemcpyDeviceToHost, d->stream),
         "gather readback");
      ck(cudaStreamSynchronize(d->stream), "gather sync");
      ck(cudaGetLastError(), "kernel");
      std::copy(h, h + n_per, all.begin() + ctx->shard_of(i) * n_per);
    }
    return all;
  }
  for (DevCtx* d : ctx->devs) {
    ck(cudaSetDevice(d->device), "cudaSetDevice");
    d->gather.reserve(total, "gather buffer");
  }
  nccl_ck(nccl_api()->GroupStart(), "ncclGroupStart");
  for (size_t i = 0; i < ctx->devs.size(); ++i) {
    DevCtx* d = ctx->devs[i];
    ck(cudaSetDevice(d->device), "cudaSetDevice");
    const ncclResult_t r = nccl_api()->AllGather(send[i], d->gather.ptr, 4 * n_per, ncclUint64,
                                                 ctx->comms[i], d->stream);
    if (r != ncclSuccess) {
      nccl_api()->GroupEnd();
      nccl_ck(r, "ncclAllGather");
    }
  }
  nccl_ck(nccl_api()->GroupEnd(), "ncclGroupEnd");
  DevCtx* d0 = ctx->devs[0];
  ck(cudaSetDevice(d0->device), "cudaSetDevice");
  auto* h = static_cast<wsk::JobAcc*>(d0->pin_gather.reserve(total * sizeof(wsk::JobAcc), "pinned gather"));
  ck(copy_async(d0, h, d0->gather.ptr, total * sizeof(wsk::JobAcc), cudaMemcpyDeviceToHost,
                d0->stream), "gather readback");
  for (DevCtx* d : ctx->devs) {
    ck(cudaSetDevice(d->device), "cudaSetDevice");
    ck(cudaStreamSynchronize(d->stream), "collective sync");
    ck(cudaGetLastError(), "kernel");
  }
  ck(cudaSetDevice(d0->device), "cudaSetDevice");
  return std::vector<wsk::JobAcc>(h, h + total);
}

// ws_combine_checks: the fold applied to the gathered per-shard records
// (count and sum wrap mod 2^64, xor folds, largest is the maximum).
ws_checks combine(const ws_checks* r, uint64_t n) {
  ws_checks o{};
  for (uint64_t i = 0; i < n; ++i) {
    o.count += r[i].count;
    o.sum += r[i].sum;
    o.xor_ ^= r[i].xor_;
    o.largest = std::max(o.largest, r[i].largest);
  }
  return o;
}

ws_checks to_checks(const wsk::JobAcc& a) { return ws_checks{a.count, a.sum, a.xr, a.largest}; }

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
void enumerate_wire(DevCtx* c, uint64_t nseg, uint64_t nch, const std::vector<uint64_t>& lo,
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
  if (!c->pool) c->pool = wswire::pool_create(c->host_threads);
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

void enumerate_to_host(DevCtx* c, uint64_t L, uint64_t R, uint64_t* out, uint64_t cap,
                       ws_checks* chk) {
  const wsk::Job whole = make_job(L, R, c->S, 0);
  const uint64_t nseg = whole.nseg;
  const uint64_t nch = std::max<uint64_t>(1, std::min<uint64_t>(DevCtx::kMaxChunks, nseg / 64));
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

// ---- shared bodies of the entry points -----------------------------------

ws_status partition_impl(uint64_t L, uint64_t R, uint32_t S, uint32_t rank, uint32_t world,
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

// Shard g's share of [L, R) and the global index of its first segment.
struct Shard {
  uint64_t lo = 0, hi = 0, seg0 = 0, nseg = 0;
};

Shard shard_of(const ws_ctx* ctx, uint32_t g, uint64_t L, uint64_t R) {
  Shard s;
  const uint32_t S = ctx->S;
  if (partition_impl(L, R, S, g, ctx->nshards, &s.lo, &s.hi) != WS_OK)
    throw Fail{WS_OVERFLOW, "range end exceeds the sievable 64-bit range"};
  if (s.hi > s.lo) {
    s.seg0 = (s.lo - L / 6 * 6) / (6ull * S);
    s.nseg = make_job(s.lo, s.hi, S, 0).nseg;
  }
  return s;
}

// ---- CUDA-graph replay of repeated small count calls ----------------------
// A count call's device work (a fresh base build, the accumulator reset, the
// sieve launch, the per-segment copy) is about ten API calls, a tenth of a
// small call such as C1 (0.2 ms).  When the same call repeats, the second one
// is captured into a graph and every later one replays it with a single
// cudaGraphLaunch.  Small single-pass count calls qualify, with a fresh base
// or a resident one that already covers them: their work is then fully
// determined by the CallKey (inputs, buffers, the resident table, and the
// allocation generation: any reallocation invalidates the graph).  The replay restores the host-side state the captured call left
// (resident-table bounds, counters).  Anything that fails during capture
// falls back to running the work directly.
constexpr uint64_t kGraphMaxSegs = 8192;

bool graph_eligible(const DevCtx* d, uint64_t lo, uint64_t hi, bool fresh) {
  if (!d->graphs || hi <= lo) return false;
  const uint64_t B = hi >= 2 ? isqrt_u64(hi - 1) : 0;
  // a cached base must already cover B (else the call extends or rebuilds it)
  if (!fresh && !(d->base_valid && d->base_B >= B)) return false;
  // no bucket windows (their fill pipeline spans streams and windows)
  if (B >= static_cast<uint64_t>(d->bucket_min_ratio) * d->S) return false;
  return make_job(lo, hi, d->S, 0).nseg <= kGraphMaxSegs;
}

template <class F>
void graph_or_run(DevCtx* d, CallKey key, bool fresh, F&& enqueue) {
  key.fresh = fresh;
  if (!fresh) {  // the resident table the captured launches read
    key.base_B = d->base_B;
    key.nprimes = d->nprimes;
    key.nprimes_dev = d->nprimes_dev;
  }
  key.gen = g_alloc_gen.load();
  CallGraph& g = d->cg;
  if (g.valid && g.key == key) {
    ck(cudaGraphLaunch(g.exec, d->stream), "graph launch");
    d->timing.launches += g.timing.launches;
    d->timing.segments += g.timing.segments;
    d->timing.h2d_bytes += g.timing.h2d_bytes;
    d->timing.d2h_bytes += g.timing.d2h_bytes;
    d->base_valid = g.base_valid;
    d->base_built = g.base_built;
    d->base_B = g.base_B;
    d->nprimes = g.nprimes;
    d->nprimes_dev = g.nprimes_dev;
    d->base_pending = false;
    return;
  }
  if (!(g.seen && g.key == key)) {  // first sighting: run it, remember it
    g.seen = true;
    g.valid = false;
    g.key = key;
    enqueue();
    return;
  }
  const ws_timing before = d->timing;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaError_t e = cudaStreamBeginCapture(d->stream, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    d->capturing = true;
    bool ok = true;
    try {
      enqueue();
    } catch (...) {
      ok = false;
    }
    d->capturing = false;
    e = cudaStreamEndCapture(d->stream, &graph);
    if (ok && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    if (!ok && e == cudaSuccess) e = cudaErrorStreamCaptureInvalidated;
    if (graph) cudaGraphDestroy(graph);
  }
  if (e != cudaSuccess || key.gen != g_alloc_gen.load()) {
    // not capturable (or it allocated): run directly from now on
    cudaGetLastError();
    if (exec) cudaGraphExecDestroy(exec);
    g.seen = false;
    d->timing = before;
    enqueue();
    return;
  }
  if (g.exec) cudaGraphExecDestroy(g.exec);
  g.exec = exec;
  g.valid = true;
  g.timing = ws_timing{};
  g.timing.launches = d->timing.launches - before.launches;
  g.timing.segments = d->timing.segments - before.segments;
  g.timing.h2d_bytes = d->timing.h2d_bytes - before.h2d_bytes;
  g.timing.d2h_bytes = d->timing.d2h_bytes - before.d2h_bytes;
  g.base_valid = d->base_valid;
  g.base_built = d->base_built;
  g.base_B = d->base_B;
  g.nprimes = d->nprimes;
  g.nprimes_dev = d->nprimes_dev;
  ck(cudaGraphLaunch(exec, d->stream), "graph launch");
}

// Queues the count of [lo, hi) on one device (its accumulator d->acc[0]; the
// per-segment counts into the device array dps when non-null).  An empty
// range leaves a zero accumulator.
void queue_count(DevCtx* d, uint64_t lo, uint64_t hi, int mode, bool fresh, uint32_t* dps) {
  if (hi <= lo) {
    d->acc.reserve(2, "acc");
    ck(cudaEventRecord(d->ev[2], d->stream), "event");
    ck(cudaMemsetAsync(d->acc.ptr, 0, sizeof(wsk::JobAcc), d->stream), "zero acc");
    ck(cudaEventRecord(d->ev[3], d->stream), "event");
    return;
  }
  validate_range(lo, hi);
  ensure_base(d, hi >= 2 ? isqrt_u64(hi - 1) : 0, fresh);
  d->h_jobs.assign(1, make_job(lo, hi, d->S, 0));
  run_sieve(d, mode, dps, nullptr, 0, true);
}

void record_device_times(DevCtx* d) {
  d->timing.base_ms = d->base_built ? event_ms(d->ev[0], d->ev[1]) : 0.0;
  d->timing.sieve_ms = event_ms(d->ev[2], d->ev[3]);
}

void count_range_single(DevCtx* d, uint64_t L, uint64_t R, uint32_t flags, ws_checks* out,
                        uint32_t* per_seg, uint64_t per_seg_cap, uint64_t* n_seg) {
  validate_range(L, R);
  const bool fresh = flags & WS_FRESH_BASE;
  const uint64_t nseg = make_job(L, R, d->S, 0).nseg;
  uint32_t* dps = nullptr;
  const bool dev_out = flags & WS_OUT_DEVICE;
  if (per_seg) {
    if (dev_out) {
      if (per_seg_cap < nseg) throw Fail{WS_CAPACITY, "per_seg capacity below segment count"};
      dps = per_seg;
    } else {
      d->per_seg.reserve(nseg, "per_seg");
      dps = d->per_seg.ptr;
    }
  }
  const int mode = (flags & WS_WANT_CHECKS) ? wsk::kCountChecks : wsk::kCount;
  auto enqueue = [&] {
    ensure_base(d, R >= 2 ? isqrt_u64(R - 1) : 0, fresh);
    d->h_jobs.assign(1, make_job(L, R, d->S, 0));
    run_sieve(d, mode, dps, nullptr, 0, true);
    if (per_seg && !dev_out)
      ck(copy_async(d, per_seg, dps, std::min(nseg, per_seg_cap) * sizeof(uint32_t),
                    cudaMemcpyDeviceToHost, d->stream), "per_seg");
  };
  // (a copy into pageable host memory inside a graph is slower than a direct
  // one: host per-segment outputs take the direct path)
  if (graph_eligible(d, L, R, fresh) && (!per_seg || dev_out)) {
    CallKey k;
    k.lo = L;
    k.hi = R;
    k.mode = mode;
    k.dps = dps;
    k.dst = (per_seg && !dev_out) ? per_seg : nullptr;
    k.kind = static_cast<int>(per_seg ? std::min(nseg, per_seg_cap) : 0) * 2 + (dev_out ? 1 : 0);
    k.S = d->S;
    graph_or_run(d, k, fresh, enqueue);
  } else {
    enqueue();
  }
  *out = to_checks(*fetch_results(d, 1));
  add_prelude(L, R, out);
  if (n_seg) *n_seg = nseg;
  record_device_times(d);
}

// Multi-device count: shard g = ws_partition(L, R, g, nshards); one allgather.
void count_range_multi(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, ws_checks* out,
                       uint32_t* per_seg, uint64_t per_seg_cap, uint64_t* n_seg) {
  validate_range(L, R);
  const uint64_t nseg = make_job(L, R, ctx->S, 0).nseg;
  const bool dev_out = flags & WS_OUT_DEVICE;
  if (per_seg && dev_out && per_seg_cap < nseg)
    throw Fail{WS_CAPACITY, "per_seg capacity below segment count"};
  const int mode = (flags & WS_WANT_CHECKS) ? wsk::kCountChecks : wsk::kCount;
  on_devices(ctx, [&](DevCtx* d, size_t i) {
    const Shard sh = shard_of(ctx, ctx->shard_of(i), L, R);
    uint32_t* dps = nullptr;
    if (per_seg && sh.nseg) {
      d->per_seg.reserve(sh.nseg, "per_seg");
      dps = d->per_seg.ptr;
    }
    auto enqueue = [&] {
      queue_count(d, sh.lo, sh.hi, mode, flags & WS_FRESH_BASE, dps);
      if (dps && per_seg_cap > sh.seg0) {
        const uint64_t n = std::min(sh.nseg, per_seg_cap - sh.seg0);
        ck(copy_async(d, per_seg + sh.seg0, dps, n * sizeof(uint32_t),
                      dev_out ? cudaMemcpyDefault : cudaMemcpyDeviceToHost, d->stream),
           "per_seg");
      }
    };
    if (ctx->devs.size() == 1 && graph_eligible(d, sh.lo, sh.hi, flags & WS_FRESH_BASE) &&
        (!per_seg || dev_out)) {
      CallKey k;
      k.lo = sh.lo;
      k.hi = sh.hi;
      k.mode = mode;
      k.dps = dps;
      k.dst = (dps && per_seg_cap > sh.seg0) ? per_seg + sh.seg0 : nullptr;
      k.kind = static_cast<int>(dps && per_seg_cap > sh.seg0
                                    ? std::min(sh.nseg, per_seg_cap - sh.seg0) : 0) * 2 +
               (dev_out ? 1 : 0);
      k.S = d->S;
      graph_or_run(d, k, flags & WS_FRESH_BASE, enqueue);
    } else {
      enqueue();
    }
  });
  std::vector<const wsk::JobAcc*> send;
  for (DevCtx* d : ctx->devs) send.push_back(d->acc.ptr);
  const std::vector<wsk::JobAcc> rec = allgather_records(ctx, send, 1);
  std::vector<ws_checks> c(rec.size());
  for (size_t g = 0; g < rec.size(); ++g) c[g] = to_checks(rec[g]);
  *out = combine(c.data(), c.size());
  add_prelude(L, R, out);
  if (n_seg) *n_seg = nseg;
  for (DevCtx* d : ctx->devs) record_device_times(d);
}

// Per-job results of a batch (count_intervals / count_ranges): job j of the
// batch is ranges[j]; shard g sieves the jobs of owner(j) == g.  Single
// device: one launch, results straight from the accumulators.  Multi-device:
// each shard's accumulators are padded to n_per records and gathered.
void count_jobs(ws_ctx* ctx, const std::vector<std::pair<uint64_t, uint64_t>>& ranges, bool checks,
                bool fresh, const std::function<uint32_t(uint64_t)>& owner, uint64_t n_per,
                const std::function<uint64_t(uint64_t)>& slot, std::vector<ws_checks>& res) {
  const uint64_t n = ranges.size();
  res.assign(n, ws_checks{});
  const int mode = checks ? wsk::kCountChecks : wsk::kCount;
  std::vector<const wsk::JobAcc*> send(ctx->devs.size(), nullptr);
  std::vector<std::vector<uint64_t>> mine(ctx->devs.size());
  for (size_t i = 0; i < ctx->devs.size(); ++i) {
    const uint32_t g = ctx->shard_of(i);
    for (uint64_t j = 0; j < n; ++j)
      if (owner(j) == g) mine[i].push_back(j);
  }
  on_devices(ctx, [&](DevCtx* d, size_t i) {
    const std::vector<uint64_t>& js = mine[i];
    uint64_t maxR = 0;
    for (uint64_t j : js)
      if (ranges[j].second > ranges[j].first) maxR = std::max(maxR, ranges[j].second);
    auto build = [&] {
      d->h_jobs.clear();
      d->h_jobs.reserve(js.size());
      uint64_t seg = 0;
      for (uint64_t j : js) {
        const auto [lo, hi] = ranges[j];
        d->h_jobs.push_back(make_job(lo, std::max(lo, hi), d->S, seg));
        seg += d->h_jobs.back().nseg;
      }
    };
    if (!js.empty()) ensure_base(d, maxR >= 2 ? isqrt_u64(maxR - 1) : 0, fresh);
    build();  // after ensure_base, which may sieve the base through h_jobs
    if (js.empty()) {
      d->acc.reserve(2, "acc");
      ck(cudaEventRecord(d->ev[2], d->stream), "event");
      ck(cudaEventRecord(d->ev[3], d->stream), "event");
    } else {
      run_sieve(d, mode, nullptr, nullptr, 0, true);
    }
    if (!ctx->nccl) return;
    d->gsend.reserve(std::max<uint64_t>(n_per, 1), "gather send");
    ck(cudaMemsetAsync(d->gsend.ptr, 0, n_per * sizeof(wsk::JobAcc), d->stream), "zero send");
    if (!js.empty())
      ck(cudaMemcpyAsync(d->gsend.ptr, d->acc.ptr, js.size() * sizeof(wsk::JobAcc),
                         cudaMemcpyDeviceToDevice, d->stream), "send records");
    send[i] = d->gsend.ptr;
  });
  if (!ctx->nccl) {
    DevCtx* d = ctx->devs[0];
    const wsk::JobAcc* acc = fetch_results(d, mine[0].size());
    for (size_t k = 0; k < mine[0].size(); ++k) res[mine[0][k]] = to_checks(acc[k]);
  } else {
    const std::vector<wsk::JobAcc> rec = allgather_records(ctx, send, n_per);
    for (uint64_t j = 0; j < n; ++j) res[j] = to_checks(rec[owner(j) * n_per + slot(j)]);
  }
  for (uint64_t j = 0; j < n; ++j) add_prelude(ranges[j].first, ranges[j].second, &res[j]);
  for (DevCtx* d : ctx->devs) record_device_times(d);
}

void enumerate_single(DevCtx* d, uint64_t L, uint64_t R, uint32_t flags, uint64_t* out,
                      uint64_t cap, uint64_t* n_out, ws_checks* checks) {
  ws_checks chk{};
  validate_range(L, R);
  ensure_base(d, R >= 2 ? isqrt_u64(R - 1) : 0, flags & WS_FRESH_BASE);
  uint64_t pre[2];
  uint64_t npre = 0;
  for (uint64_t v : {uint64_t{2}, uint64_t{3}})
    if (v >= L && v < R) pre[npre++] = v;
  d->h_jobs.assign(1, make_job(L, R, d->S, 0));
  const bool dev_out = flags & WS_OUT_DEVICE;
  if (dev_out && out && !is_device_ptr(out))
    throw Fail{WS_BAD_CONFIG, "WS_OUT_DEVICE with a non-device pointer"};
  if (!dev_out) {
    for (uint64_t i = 0; i < npre && i < cap; ++i) out[i] = pre[i];
    enumerate_to_host(d, L, R, out + std::min(npre, cap), cap > npre ? cap - npre : 0, &chk);
  } else {
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(out) + std::min(npre, cap);
    const uint64_t dcap = cap > npre ? cap - npre : 0;
    if (npre && cap)
      ck(copy_async(d, out, pre, std::min(npre, cap) * 8, cudaMemcpyHostToDevice, d->stream),
         "prelude");
    run_sieve(d, wsk::kEnumerate, nullptr, dst, dcap, true);
    chk = to_checks(*fetch_results(d, 1));
  }
  add_prelude(L, R, &chk);
  *n_out = chk.count;
  if (checks) *checks = chk;
  record_device_times(d);
  if (chk.count > cap) throw Fail{WS_CAPACITY, "output capacity below the prime count"};
}

int device_of_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ? a.device : -1;
}

// Multi-device enumeration: a count pass on every shard, one allgather of
// the shard records (offsets and totals), then every device writes its shard
// at its offset.
void enumerate_multi(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, uint64_t* out,
                     uint64_t cap, uint64_t* n_out, ws_checks* checks) {
  validate_range(L, R);
  const bool dev_out = flags & WS_OUT_DEVICE;
  const int out_dev = dev_out && out ? device_of_ptr(out) : -1;
  if (dev_out && out && out_dev < 0)
    throw Fail{WS_BAD_CONFIG, "WS_OUT_DEVICE with a non-device pointer"};
  on_devices(ctx, [&](DevCtx* d, size_t i) {
    const Shard sh = shard_of(ctx, ctx->shard_of(i), L, R);
    queue_count(d, sh.lo, sh.hi, wsk::kCountChecks, flags & WS_FRESH_BASE, nullptr);
  });
  std::vector<const wsk::JobAcc*> send;
  for (DevCtx* d : ctx->devs) send.push_back(d->acc.ptr);
  const std::vector<wsk::JobAcc> rec = allgather_records(ctx, send, 1);
  std::vector<ws_checks> c(rec.size());
  for (size_t g = 0; g < rec.size(); ++g) c[g] = to_checks(rec[g]);
  ws_checks total = combine(c.data(), c.size());
  add_prelude(L, R, &total);
  uint64_t pre[2];
  uint64_t npre = 0;
  for (uint64_t v : {uint64_t{2}, uint64_t{3}})
    if (v >= L && v < R) pre[npre++] = v;
  // global offset of every shard; this process owns shards [first, first + k)
  std::vector<uint64_t> off(ctx->nshards + 1, npre);
  for (uint32_t g = 0; g < ctx->nshards; ++g) off[g + 1] = off[g] + c[g].count;
  const uint32_t first = ctx->shard_of(0);
  const uint64_t local_base = first == 0 ? 0 : off[first];
  const uint64_t local_end = off[first + ctx->devs.size()];
  const uint64_t local_n = local_end - local_base;
  if (first == 0 && npre && cap) {
    if (dev_out)
      ck(cudaMemcpy(out, pre, std::min(npre, cap) * 8, cudaMemcpyHostToDevice), "prelude");
    else
      for (uint64_t i = 0; i < npre && i < cap; ++i) out[i] = pre[i];
  }
  on_devices(ctx, [&](DevCtx* d, size_t i) {
    const uint32_t g = ctx->shard_of(i);
    const Shard sh = shard_of(ctx, g, L, R);
    const uint64_t pos = off[g] - local_base;
    const uint64_t room = cap > pos ? cap - pos : 0;
    if (sh.hi <= sh.lo || !out) return;
    ws_checks chk{};
    if (!dev_out) {
      enumerate_to_host(d, sh.lo, sh.hi, out + pos, room, &chk);
    } else {
      d->h_jobs.assign(1, make_job(sh.lo, sh.hi, d->S, 0));
      const uint64_t n = c[g].count;
      if (out_dev == d->device) {
        run_sieve(d, wsk::kEnumerate, nullptr, reinterpret_cast<unsigned long long*>(out + pos),
                  room, true);
      } else {  // another device's memory: enumerate locally, then one copy over NVLink
        d->vals.reserve(std::max<uint64_t>(n, 1), "shard values");
        run_sieve(d, wsk::kEnumerate, nullptr, d->vals.ptr, n, true);
        if (room)
          ck(cudaMemcpyAsync(out + pos, d->vals.ptr, std::min(n, room) * 8, cudaMemcpyDefault,
                             d->stream), "shard copy");
      }
      chk = to_checks(*fetch_results(d, 1));
    }
    if (chk.count != c[g].count || chk.sum != c[g].sum || chk.xor_ != c[g].xor_)
      throw Fail{WS_CUDA, "shard enumeration disagrees with its count pass"};
  });
  *n_out = local_n;
  if (checks) *checks = total;
  for (DevCtx* d : ctx->devs) record_device_times(d);
  if (local_n > cap) throw Fail{WS_CAPACITY, "output capacity below the prime count"};
}

// Every local device enumerates its shard into its own memory: one pass,
// then one allgather of the shard records for the totals.
void enumerate_shards(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, uint64_t* const* outs,
                      const uint64_t* caps, uint64_t* counts, ws_checks* checks) {
  validate_range(L, R);
  const uint32_t first = ctx->shard_of(0);
  uint64_t npre = 0;
  uint64_t pre[2];
  for (uint64_t v : {uint64_t{2}, uint64_t{3}})
    if (v >= L && v < R) pre[npre++] = v;
  std::vector<uint64_t> got(ctx->devs.size(), 0);
  on_devices(ctx, [&](DevCtx* d, size_t i) {
    const uint32_t g = ctx->shard_of(i);
    const Shard sh = shard_of(ctx, g, L, R);
    if (outs[i] && device_of_ptr(outs[i]) != d->device)
      throw Fail{WS_BAD_CONFIG, "outs[i] must be memory of local device i"};
    if (!outs[i] && caps[i]) throw Fail{WS_BAD_CONFIG, "null output with nonzero capacity"};
    // shard 0 carries the prelude 2, 3
    const uint64_t np = g == 0 ? npre : 0;
    if (np && caps[i])
      ck(copy_async(d, outs[i], pre, std::min(np, caps[i]) * 8, cudaMemcpyHostToDevice, d->stream),
         "prelude");
    const uint64_t room = caps[i] > np ? caps[i] - np : 0;
    if (sh.hi <= sh.lo) {
      queue_count(d, sh.lo, sh.hi, wsk::kCount, false, nullptr);
    } else {
      ensure_base(d, sh.hi >= 2 ? isqrt_u64(sh.hi - 1) : 0, flags & WS_FRESH_BASE);
      d->h_jobs.assign(1, make_job(sh.lo, sh.hi, d->S, 0));
      run_sieve(d, wsk::kEnumerate, nullptr,
                reinterpret_cast<unsigned long long*>(outs[i] + std::min(np, caps[i])), room, true);
    }
    got[i] = np;
  });
  std::vector<const wsk::JobAcc*> send;
  for (DevCtx* d : ctx->devs) send.push_back(d->acc.ptr);
  const std::vector<wsk::JobAcc> rec = allgather_records(ctx, send, 1);
  std::vector<ws_checks> c(rec.size());
  for (size_t g = 0; g < rec.size(); ++g) c[g] = to_checks(rec[g]);
  ws_checks total = combine(c.data(), c.size());
  add_prelude(L, R, &total);
  bool short_cap = false;
  for (size_t i = 0; i < ctx->devs.size(); ++i) {
    counts[i] = got[i] + c[first + i].count;
    short_cap = short_cap || counts[i] > caps[i];
  }
  if (checks) *checks = total;
  for (DevCtx* d : ctx->devs) record_device_times(d);
  if (short_cap) throw Fail{WS_CAPACITY, "a shard's output capacity is below its prime count"};
}

// One device context on CUDA device `dev` (everything but NCCL).
ws_status make_dev(int dev, uint32_t S, DevCtx** out) {
  *out = nullptr;
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    return WS_NO_DEVICE;
  }
  if (prop.major != 10) return WS_NO_DEVICE;  // built for sm_100a only
  DevCtx* c = new (std::nothrow) DevCtx;
  if (!c) return WS_OUT_OF_MEMORY;
  c->device = dev;
  c->S = S;
  {  // primes in [53, S): the in-kernel share of the table; and the warp-
     // cooperative share [53, wc_limit)
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
  if (const char* e = std::getenv("WHEELSIEVE_SINGLE_PRED")) c->single_pred = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_MID_BITADDR")) c->mid_bitaddr = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_HUGE_LOOP")) c->huge_loop = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_FILL_UNROLL")) c->w_unroll = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_STAGE_CAP")) c->stage_cap = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_GRAPHS")) c->graphs = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_MISS_LANE")) c->miss_lane = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_SKIP5")) c->skip5_max = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_WIDE")) c->wide = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_PMIN")) c->wide_pmin_ratio = std::max<uint32_t>(1, std::strtoul(e, nullptr, 10));
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_BUCKET")) c->wide_bucket = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_MULTI")) c->wide_multi = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_SEG_TRANS")) c->seg_trans = std::atoi(e) != 0;
  if (const char* e = std::getenv("WHEELSIEVE_SEG_TRANS_MIN")) c->seg_trans_min = std::max<uint32_t>(32, std::strtoul(e, nullptr, 10));
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_DOUBLE")) c->wide_double = std::strtoul(e, nullptr, 10);
  if (const char* e = std::getenv("WHEELSIEVE_TRANS_MIN")) c->trans_min = std::max<uint32_t>(32, std::strtoul(e, nullptr, 10));
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_SKIP5")) c->wide_skip5 = std::strtoul(e, nullptr, 10);
  // wide units mark primes below 1280 warp-cooperatively (1024 .. 1536 within 0.6%)
  c->wide_n_wc = table_primes_below(c, 1280);
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_WC_LIMIT"))
    c->wide_n_wc = table_primes_below(c, std::strtoul(e, nullptr, 10));
  if (const char* e = std::getenv("WHEELSIEVE_WIDE_MIN_UNITS"))
    c->wide_min_units = std::strtoul(e, nullptr, 10);
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
  for (int i = 0; i < DevCtx::kMaxChunks && ok; ++i)
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

}  // namespace

extern "C" {

const char* ws_version(void) { return "wheelsieve-b200 0.2 (sm_100a, NCCL multi-device)"; }

void ws_opts_default(ws_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->struct_size = sizeof(ws_opts);
  o->segment_slots = 1u << 18;
  o->device = -1;
  o->world = 1;
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
    case WS_NCCL: return "Nccl";
  }
  return "unknown";
}

ws_status ws_nccl_unique_id(uint8_t* id) {
  if (!id) return WS_BAD_CONFIG;
  static_assert(sizeof(ncclUniqueId) == WS_NCCL_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  if (!nccl_api() || nccl_api()->GetUniqueId(&u) != ncclSuccess) return WS_NCCL;
  std::memcpy(id, &u, sizeof u);
  return WS_OK;
}

ws_status ws_ctx_create(const ws_opts* opts, ws_ctx** out) {
  if (!out) return WS_BAD_CONFIG;
  *out = nullptr;
  ws_opts o;
  ws_opts_default(&o);
  if (opts) {
    constexpr uint32_t kV1 = 16;  // {struct_size, segment_slots, device, reserved}
    if (opts->struct_size == kV1) {
      std::memcpy(&o, opts, kV1);
      if (o.n_devices != 0) return WS_BAD_CONFIG;  // v1's reserved word must be zero
      o.struct_size = sizeof(ws_opts);
    } else if (opts->struct_size == sizeof(ws_opts)) {
      o = *opts;
    } else {
      return WS_BAD_CONFIG;
    }
  }
  const uint32_t S = o.segment_slots;
  if (S < (1u << 12) || S > (1u << 18) || (S & (S - 1))) return WS_BAD_CONFIG;
  if (o.world == 0) o.world = 1;
  if (o.rank >= o.world || o.n_devices > WS_MAX_DEVICES) return WS_BAD_CONFIG;
  if (o.world > 1 && o.n_devices == 0) return WS_BAD_CONFIG;  // multi-process needs NCCL
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return WS_NO_DEVICE;
  }
  std::vector<int> devices;
  if (o.n_devices == 0) {
    int dev = o.device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return WS_NO_DEVICE;
    devices.push_back(dev);
  } else {
    for (uint32_t i = 0; i < o.n_devices; ++i) devices.push_back(o.device_ids[i]);
  }
  const char* virt_env = std::getenv("WHEELSIEVE_VIRTUAL_SHARDS");
  const bool virt = o.n_devices > 0 && o.world == 1 && virt_env && std::atoi(virt_env) != 0;
  for (size_t i = 0; i < devices.size(); ++i) {
    if (devices[i] < 0 || devices[i] >= ndev) return WS_NO_DEVICE;
    for (size_t j = 0; j < i && !virt; ++j)
      if (devices[j] == devices[i]) return WS_BAD_CONFIG;  // one shard per device
  }
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  ws_ctx* c = new (std::nothrow) ws_ctx;
  if (!c) return WS_OUT_OF_MEMORY;
  c->nccl = o.n_devices > 0;
  c->S = S;
  c->world = o.world;
  c->rank = o.rank;
  c->nshards = c->nccl ? o.world * static_cast<uint32_t>(devices.size()) : 1;
  const unsigned cpus = std::max(1u, std::thread::hardware_concurrency());
  for (size_t i = 0; i < devices.size(); ++i) {
    DevCtx* d = nullptr;
    const ws_status st = make_dev(devices[i], S, &d);
    if (st != WS_OK) {
      delete c;
      if (prev >= 0) cudaSetDevice(prev);
      return st;
    }
    d->shard = c->shard_of(i);
    // co-resident devices split the host's cores between their wire expanders
    if (devices.size() > 1 && !std::getenv("WHEELSIEVE_HOST_THREADS"))
      d->host_threads = std::max(1u, cpus / static_cast<unsigned>(devices.size()));
    c->devs.push_back(d);
  }
  c->virt = virt;
  if (c->nccl && virt && devices.size() > 1) c->workers = new (std::nothrow) DevWorkers(devices);
  if (c->nccl && !virt && !nccl_api()) {
    delete c;
    if (prev >= 0) cudaSetDevice(prev);
    return WS_NCCL;
  }
  if (c->nccl && !virt) {
    const NcclApi* N = nccl_api();
    const int k = static_cast<int>(devices.size());
    c->comms.assign(devices.size(), nullptr);
    ncclResult_t r;
    bool have_id = false;
    for (uint8_t b : o.nccl_id) have_id = have_id || b != 0;
    if (o.world == 1 && !have_id) {
      r = N->CommInitAll(c->comms.data(), k, devices.data());
    } else {  // a job shared with other processes (or a caller-made id)
      ncclUniqueId id;
      std::memcpy(&id, o.nccl_id, sizeof id);
      r = N->GroupStart();
      for (int i = 0; i < k && r == ncclSuccess; ++i) {
        cudaSetDevice(devices[i]);
        r = N->CommInitRank(&c->comms[i], static_cast<int>(o.world) * k, id,
                            static_cast<int>(o.rank) * k + i);
      }
      const ncclResult_t r2 = N->GroupEnd();
      if (r == ncclSuccess) r = r2;
    }
    if (r != ncclSuccess) {
      c->comms.clear();
      delete c;
      if (prev >= 0) cudaSetDevice(prev);
      return WS_NCCL;
    }
    if (devices.size() > 1) c->workers = new (std::nothrow) DevWorkers(devices);
  }
  if (prev >= 0) cudaSetDevice(prev);
  *out = c;
  return WS_OK;
}

void ws_ctx_destroy(ws_ctx* ctx) { delete ctx; }

const char* ws_last_error(const ws_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* ws_ctx_stream(ws_ctx* ctx) {
  return ctx && !ctx->devs.empty() ? static_cast<void*>(ctx->devs[0]->stream) : nullptr;
}

uint32_t ws_ctx_num_devices(const ws_ctx* ctx) {
  return ctx ? static_cast<uint32_t>(ctx->devs.size()) : 0;
}

uint32_t ws_ctx_num_shards(const ws_ctx* ctx) { return ctx ? ctx->nshards : 0; }

int32_t ws_ctx_device(const ws_ctx* ctx, uint32_t i) {
  return ctx && i < ctx->devs.size() ? ctx->devs[i]->device : -1;
}

void* ws_ctx_device_stream(ws_ctx* ctx, uint32_t i) {
  return ctx && i < ctx->devs.size() ? static_cast<void*>(ctx->devs[i]->stream) : nullptr;
}

ws_status ws_last_timing(const ws_ctx* ctx, ws_timing* out) {
  if (!ctx || !out) return WS_BAD_CONFIG;
  *out = ctx->timing;
  return WS_OK;
}

ws_status ws_device_timing(const ws_ctx* ctx, uint32_t i, ws_timing* out) {
  if (!ctx || !out || i >= ctx->devs.size()) return WS_BAD_CONFIG;
  *out = ctx->devs[i]->timing;
  out->total_ms = ctx->timing.total_ms;
  return WS_OK;
}

ws_status ws_ctx_comm_info(const ws_ctx* ctx, uint32_t i, int32_t* nranks, int32_t* comm_rank) {
  if (ctx && ctx->virt && nranks && comm_rank && i < ctx->devs.size()) {  // test mode: no NCCL
    *nranks = static_cast<int32_t>(ctx->nshards);
    *comm_rank = static_cast<int32_t>(ctx->shard_of(i));
    return WS_OK;
  }
  if (!ctx || !nranks || !comm_rank || !ctx->nccl || i >= ctx->comms.size()) return WS_BAD_CONFIG;
  int n = 0, r = 0;
  if (nccl_api()->CommCount(ctx->comms[i], &n) != ncclSuccess ||
      nccl_api()->CommUserRank(ctx->comms[i], &r) != ncclSuccess)
    return WS_NCCL;
  *nranks = n;
  *comm_rank = r;
  return WS_OK;
}

ws_status ws_combine_checks(const ws_checks* records, uint64_t n, ws_checks* out) {
  if (!out || (n && !records)) return WS_BAD_CONFIG;
  *out = combine(records, n);
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
  return partition_impl(L, R, S, rank, world, lo, hi);
}

ws_status ws_count_range(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, ws_checks* out,
                         uint32_t* per_seg, uint64_t per_seg_cap, uint64_t* n_seg) {
  return guarded(ctx, [&] {
    if (!out) throw Fail{WS_BAD_CONFIG, "null output"};
    *out = ws_checks{};
    if (n_seg) *n_seg = 0;
    if (R <= L) return;
    if (ctx->nccl)
      count_range_multi(ctx, L, R, flags, out, per_seg, per_seg_cap, n_seg);
    else
      count_range_single(ctx->devs[0], L, R, flags, out, per_seg, per_seg_cap, n_seg);
  });
}

ws_status ws_enumerate_range(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, uint64_t* out,
                             uint64_t cap, uint64_t* n_out, ws_checks* checks) {
  return guarded(ctx, [&] {
    if (!n_out) throw Fail{WS_BAD_CONFIG, "null n_out"};
    *n_out = 0;
    if (checks) *checks = ws_checks{};
    if (R <= L) return;
    if (!out && cap) throw Fail{WS_BAD_CONFIG, "null output with nonzero capacity"};
    if (ctx->nccl)
      enumerate_multi(ctx, L, R, flags, out, cap, n_out, checks);
    else
      enumerate_single(ctx->devs[0], L, R, flags, out, cap, n_out, checks);
  });
}

ws_status ws_enumerate_shards(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags,
                              uint64_t* const* outs, const uint64_t* caps, uint64_t* counts,
                              ws_checks* checks) {
  return guarded(ctx, [&] {
    if (!outs || !caps || !counts) throw Fail{WS_BAD_CONFIG, "null shard arrays"};
    for (size_t i = 0; i < ctx->devs.size(); ++i) counts[i] = 0;
    if (checks) *checks = ws_checks{};
    if (!ctx->nccl) throw Fail{WS_BAD_CONFIG, "ws_enumerate_shards needs a multi-device context"};
    if (R <= L) return;
    enumerate_shards(ctx, L, R, flags, outs, caps, counts, checks);
  });
}

ws_status ws_base_primes(ws_ctx* ctx, uint64_t B, uint32_t flags, uint64_t* out, uint64_t cap,
                         uint64_t* n) {
  return guarded(ctx, [&] {
    if (!n) throw Fail{WS_BAD_CONFIG, "null n"};
    *n = 0;
    if (B < 2) throw Fail{WS_EMPTY_RANGE, "no primes below 2"};  // wheel.cpp:41
    if (B > 0xFFFFFFFFull) throw Fail{WS_CAPACITY, "base bound above 2^32"};
    // the store's entries are the wheel primes 5 <= p <= B (base_store.cpp:34-42):
    // enumerate [5, B + 1) on the (first) device
    if (B < 5) return;
    if (!out && cap) throw Fail{WS_BAD_CONFIG, "null output with nonzero capacity"};
    ws_checks chk{};
    enumerate_single(ctx->devs[0], 5, B + 1, flags & (WS_OUT_DEVICE | WS_FRESH_BASE), out, cap, n,
                     &chk);
  });
}

ws_status ws_sieve_segment(ws_ctx* ctx, uint64_t start, uint64_t len, uint32_t flags,
                           uint64_t* r1_words, uint64_t* r5_words) {
  return guarded(ctx, [&] {
    DevCtx* d = ctx->devs[0];
    // SegmentBitmap checks, segment.cpp:101-110
    if (start % 6 != 0) throw Fail{WS_ALIGNMENT, "segment start is not a multiple of 6"};
    if (len == 0) throw Fail{WS_DOMAIN, "segment must span at least one wheel index"};
    if (len > (kMaxSegmentEnd - start) / 6)
      throw Fail{WS_OVERFLOW, "segment end exceeds the 64-bit value range"};
    if (!r1_words || !r5_words) throw Fail{WS_BAD_CONFIG, "null output"};
    const uint64_t end = start + 6 * len;
    ensure_base(d, isqrt_u64(end - 1), flags & WS_FRESH_BASE);
    d->h_jobs.assign(1, make_job(start, end, d->S, 0));
    const uint64_t nseg = d->h_jobs[0].nseg;
    const uint64_t words32 = nseg * (d->S / 32);
    const uint64_t out64 = (len + 63) / 64;
    const bool dev_out = flags & WS_OUT_DEVICE;
    DevBuf<uint32_t> tmp;
    tmp.reserve(2 * words32 + 2, "bitmap words");
    d->words_out[0] = tmp.ptr;
    d->words_out[1] = tmp.ptr + words32;
    try {
      run_sieve(d, wsk::kCount, nullptr, nullptr, 0, true);
    } catch (...) {
      d->words_out[0] = d->words_out[1] = nullptr;
      tmp.release();
      throw;
    }
    d->words_out[0] = d->words_out[1] = nullptr;
    // uint32 LSB-first words are byte-identical to FlagArray's uint64 words
    const cudaMemcpyKind k = dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    ck(copy_async(d, r1_words, tmp.ptr, out64 * 8, k, d->stream), "r1 words");
    ck(copy_async(d, r5_words, tmp.ptr + words32, out64 * 8, k, d->stream), "r5 words");
    fetch_results(d, 1);
    tmp.release();
    // sieve_segment leaves the value 1 set; callers clear it (engine.cpp:244)
    if (start == 0) {
      if (dev_out) {
        uint64_t w0 = 0;
        ck(copy_sync(d, &w0, r1_words, 8, cudaMemcpyDeviceToHost), "w0");
        w0 |= 1;
        ck(copy_sync(d, r1_words, &w0, 8, cudaMemcpyHostToDevice), "w0");
      } else {
        r1_words[0] |= 1;
      }
    }
    d->timing.sieve_ms = event_ms(d->ev[2], d->ev[3]);
  });
}

ws_status ws_count_intervals(ws_ctx* ctx, const uint64_t* Ls, uint64_t n, uint64_t width,
                             uint32_t flags, uint32_t* counts, uint64_t* sums, uint64_t* xors) {
  return guarded(ctx, [&] {
    if (n == 0) return;
    if (!Ls || !counts) throw Fail{WS_BAD_CONFIG, "null interval arrays"};
    if (width == 0) throw Fail{WS_EMPTY_RANGE, "zero-width intervals"};
    const bool dev_out = flags & WS_OUT_DEVICE;
    if (dev_out && ctx->nccl)
      throw Fail{WS_BAD_CONFIG, "WS_OUT_DEVICE intervals need a single-device context"};
    DevCtx* d0 = ctx->devs[0];
    std::vector<uint64_t> hL;
    const uint64_t* L = Ls;
    if (dev_out) {
      hL.resize(n);
      ck(copy_sync(d0, hL.data(), Ls, n * 8, cudaMemcpyDeviceToHost), "intervals in");
      L = hL.data();
    }
    std::vector<std::pair<uint64_t, uint64_t>> ranges(n);
    for (uint64_t i = 0; i < n; ++i) {
      if (L[i] > kMaxSegmentEnd - width) throw Fail{WS_OVERFLOW, "interval end overflows"};
      ranges[i] = {L[i], L[i] + width};
    }
    const uint64_t G = ctx->nshards;
    std::vector<ws_checks> res;
    // interval i -> shard i mod G, at slot i / G of that shard's records
    count_jobs(ctx, ranges, sums || xors, flags & WS_FRESH_BASE,
               [G](uint64_t i) { return static_cast<uint32_t>(i % G); }, (n + G - 1) / G,
               [G](uint64_t i) { return i / G; }, res);
    std::vector<uint32_t> hc(n);
    std::vector<uint64_t> hs(n), hx(n);
    for (uint64_t i = 0; i < n; ++i) {
      hc[i] = static_cast<uint32_t>(res[i].count);
      hs[i] = res[i].sum;
      hx[i] = res[i].xor_;
    }
    if (dev_out) {
      ck(copy_sync(d0, counts, hc.data(), n * 4, cudaMemcpyHostToDevice), "counts");
      if (sums) ck(copy_sync(d0, sums, hs.data(), n * 8, cudaMemcpyHostToDevice), "sums");
      if (xors) ck(copy_sync(d0, xors, hx.data(), n * 8, cudaMemcpyHostToDevice), "xors");
    } else {
      std::memcpy(counts, hc.data(), n * 4);
      if (sums) std::memcpy(sums, hs.data(), n * 8);
      if (xors) std::memcpy(xors, hx.data(), n * 8);
    }
  });
}

ws_status ws_count_ranges(ws_ctx* ctx, const uint64_t* Ls, const uint64_t* Rs, uint64_t n,
                          uint32_t flags, ws_checks* out) {
  return guarded(ctx, [&] {
    if (n == 0) return;
    if (!Ls || !Rs || !out) throw Fail{WS_BAD_CONFIG, "null range arrays"};
    std::vector<std::pair<uint64_t, uint64_t>> ranges(n);
    for (uint64_t i = 0; i < n; ++i) {
      if (Rs[i] > Ls[i]) validate_range(Ls[i], Rs[i]);
      ranges[i] = {Ls[i], Rs[i]};
    }
    // contiguous blocks: shard g takes ranges [floor(g n / G), floor((g+1) n / G))
    const uint64_t G = ctx->nshards;
    auto first = [n, G](uint64_t g) {
      return static_cast<uint64_t>(static_cast<unsigned __int128>(g) * n / G);
    };
    auto owner = [n, G, first](uint64_t i) {
      uint64_t g = static_cast<uint64_t>(static_cast<unsigned __int128>(i) * G / n);
      while (g + 1 < G && first(g + 1) <= i) ++g;
      while (g > 0 && first(g) > i) --g;
      return static_cast<uint32_t>(g);
    };
    std::vector<ws_checks> res;
    count_jobs(ctx, ranges, flags & WS_WANT_CHECKS, flags & WS_FRESH_BASE, owner,
               (n + G - 1) / G, [&](uint64_t i) { return i - first(owner(i)); }, res);
    std::memcpy(out, res.data(), n * sizeof(ws_checks));
  });
}

}  // extern "C"
