// The engine (wheelsieve/engine.hpp, wheelsieve/gpu.hpp): the reference's
// run loop (engine.cpp:149-307) with the sieving on the GPU.
//
// Iterations are still the unit of emission and of the stop check, and each
// iteration's tiles are the reference's (engine.cpp:233-241).  The device
// work is batched: a block of iterations is sieved per call -- for value
// sinks one ordered enumeration of the block, cut at the tile borders on the
// host; for count sinks one ws_count_ranges batch with every tile of the
// block as its own range, so each tile's (count, largest) comes from the
// device exactly as the reference's per-tile count_surviving /
// last_surviving do (engine.cpp:251-253).  Emission then walks the block
// iteration by iteration: 2 and 3 first, then one batch per non-empty tile.
#include <algorithm>
#include <chrono>
#include <string>
#include <utility>

#include "wheelsieve/engine.hpp"
#include "wheelsieve/gpu.hpp"

namespace wheelsieve {

namespace {

constexpr uint64_t kValueBlock = uint64_t{1} << 28;  // integers per call (value sinks)
constexpr uint64_t kCountBlock = uint64_t{1} << 36;  // integers per call (count sinks) ...
constexpr uint64_t kTileBlock = uint64_t{1} << 16;   // ... and at most this many tiles

void validate(const SieveConfig& c, bool bounded) {  // the reference's order, engine.cpp:119-143
  if (!c.sink) throw Error(Errc::BadConfig, "SieveConfig::sink is null");
  if (c.threads == 0) throw Error(Errc::BadConfig, "threads must be at least 1");
  if (c.threads > c.thread_cap)
    throw Error(Errc::BadConfig, std::to_string(c.threads) + " threads exceed thread_cap " +
                                     std::to_string(c.thread_cap));
  const uint64_t align = 6ull * c.threads;
  if (c.segment_span == 0 || c.segment_span % align)
    throw Error(Errc::BadConfig, "segment_span " + std::to_string(c.segment_span) +
                                     " must be a positive multiple of " + std::to_string(align));
  if (c.segment_span > kMaxSegmentEnd)
    throw Error(Errc::BadConfig, "segment_span is past the 64-bit value range");
  if (bounded) {
    if (!c.limit) throw Error(Errc::BadConfig, "run() needs a limit");
    if (*c.limit < 2) throw Error(Errc::EmptyRange, "there are no primes below 2");
    if (*c.limit > kMaxSegmentEnd - 1)
      throw Error(Errc::Overflow, "limit is past the sievable 64-bit range");
  } else if (c.limit) {
    throw Error(Errc::BadConfig, "run_unbounded() takes no limit");
  }
}

struct Tile {
  uint64_t lo, hi;
};

// The non-empty tiles of the iteration [seg_lo, seg_hi).
void tiles_of(const SieveConfig& c, uint64_t seg_lo, uint64_t seg_hi, std::vector<Tile>& out) {
  const uint64_t sub = c.segment_span / c.threads;
  for (unsigned j = 0; j < c.threads; ++j) {
    const uint64_t lo = seg_lo + j * sub;
    if (lo >= seg_hi) break;
    out.push_back({lo, sub > seg_hi - lo ? seg_hi : lo + sub});
  }
}

SieveReport run_loop(const SieveConfig& config, const std::atomic<bool>* stop,
                     gpu::Context& ctx) {
  validate(config, stop == nullptr);
  PrimeSink& sink = *config.sink;
  const auto t0 = std::chrono::steady_clock::now();
  const bool bounded = stop == nullptr;
  const uint64_t span = config.segment_span;
  const uint64_t limit = bounded ? *config.limit : 0;
  const uint64_t limit_end = bounded ? (limit / 6 + 1) * 6 : kMaxSegmentEnd;
  const uint64_t total = bounded ? limit_end / span + (limit_end % span != 0) : 0;
  const uint64_t top = bounded ? limit + 1 : kMaxSegmentEnd;  // values kept below this
  const bool values = sink.wants_values();
  const uint64_t per_call =
      values ? std::max<uint64_t>(1, kValueBlock / span)
             : std::max<uint64_t>(1, std::min<uint64_t>(kCountBlock / span,
                                                        kTileBlock / config.threads));
  SieveReport rep;
  auto stamp = [&] {
    rep.wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  // the block of iterations sieved by the last device call ends at blk_end
  uint64_t blk_end = 0;
  std::vector<uint64_t> vals;       // value sinks: the block's primes
  std::vector<Tile> blk_tiles;      // count sinks: the block's tiles ...
  std::vector<gpu::Checks> counts;  // ... and their results
  size_t tile_cursor = 0;
  std::vector<Tile> tiles;
  // one iteration's batches in worker order: 2 and 3 first (engine.cpp:268-276),
  // then one per non-empty tile; a sink error becomes SinkFailure with the
  // totals emitted before it (engine.cpp:264-296)
  auto emit_iteration = [&](uint64_t i) {
    try {
      if (i == 0) {
        static constexpr uint64_t kFirst[2] = {2, 3};
        const size_t n = (!bounded || limit >= 3) ? 2 : 1;
        if (values)
          sink.emit({kFirst, n});
        else
          sink.emit_count(n, kFirst[n - 1]);
      }
      for (const Tile& t : tiles) {
        if (values) {
          const auto a = std::lower_bound(vals.begin(), vals.end(), t.lo);
          const auto b = std::lower_bound(a, vals.end(), std::min(t.hi, top));
          if (b > a) sink.emit({&*a, static_cast<size_t>(b - a)});
        } else {
          const gpu::Checks& r = counts[tile_cursor++];
          if (r.count) sink.emit_count(r.count, r.largest);
        }
      }
    } catch (const Error& e) {
      rep.prime_count = sink.count();
      rep.largest_prime = sink.largest();
      stamp();
      throw SinkFailure(e.code(), e.what(), rep);
    }
  };
  for (uint64_t i = 0, seg_lo = 0;; ++i, seg_lo += span) {
    if (bounded && i >= total) break;
    if (stop && stop->load(std::memory_order_acquire)) {
      rep.stopped = true;
      break;
    }
    if (!bounded && seg_lo > kMaxSegmentEnd - span) {
      rep.overflowed = true;
      break;
    }
    const uint64_t seg_hi = (bounded && span > limit_end - seg_lo) ? limit_end : seg_lo + span;
    tiles.clear();
    tiles_of(config, seg_lo, seg_hi, tiles);
    {  // analytic flag accounting of this iteration (engine.cpp:218-230)
      uint64_t entries = 0, bytes = 0;
      for (const Tile& t : tiles) {
        const uint64_t len = (t.hi - t.lo) / 6;
        entries += 2 * len;
        bytes += 2 * flag_payload_bytes(len, config.flag_width);
      }
      rep.peak_flag_entries = std::max(rep.peak_flag_entries, entries);
      rep.peak_flag_bytes = std::max(rep.peak_flag_bytes, bytes);
    }
    if (i >= blk_end) {  // the next block of iterations on the device
      uint64_t n = std::min(per_call, (kMaxSegmentEnd - seg_lo) / span);
      if (bounded) n = std::min(n, total - i);
      const uint64_t bhi = std::min(seg_lo + n * span, limit_end);
      if (values) {
        const uint64_t a = std::max<uint64_t>(seg_lo, 4), b = std::min(bhi, top);
        vals = a < b ? ctx.enumerate_range(a, b) : std::vector<uint64_t>{};
      } else {
        blk_tiles.clear();
        for (uint64_t k = 0; k < n; ++k)
          tiles_of(config, seg_lo + k * span, std::min(seg_lo + (k + 1) * span, bhi), blk_tiles);
        std::vector<uint64_t> Ls(blk_tiles.size()), Rs(blk_tiles.size());
        for (size_t t = 0; t < blk_tiles.size(); ++t) {
          Ls[t] = std::max<uint64_t>(blk_tiles[t].lo, 4);
          Rs[t] = std::max(Ls[t], std::min(blk_tiles[t].hi, top));
        }
        counts = ctx.count_ranges(Ls, Rs);
        tile_cursor = 0;
      }
      blk_end = i + n;
    }
    emit_iteration(i);
    rep.iterations = i + 1;
    rep.sieved_to = seg_hi;
  }
  if (bounded) rep.sieved_to = limit + 1;
  rep.prime_count = sink.count();
  rep.largest_prime = sink.largest();
  stamp();
  return rep;
}

}  // namespace

uint64_t round_segment_span(uint64_t span, unsigned threads) {
  if (threads == 0) throw Error(Errc::BadConfig, "threads must be at least 1");
  const uint64_t align = 6ull * threads;
  if (span == 0) return align;
  if (span % align == 0) return span;
  if (span > UINT64_MAX - align)
    throw Error(Errc::Overflow, "segment_span is past the 64-bit value range");
  return (span / align + 1) * align;
}

std::vector<WorkerAssignment> plan_iteration(const SieveConfig& config, uint64_t iteration) {
  if (config.threads == 0 || config.threads > config.thread_cap)
    throw Error(Errc::BadConfig, "invalid thread count");
  const uint64_t span = config.segment_span;
  const uint64_t align = 6ull * config.threads;
  if (span == 0 || span % align || span > kMaxSegmentEnd)
    throw Error(Errc::BadConfig, "segment_span " + std::to_string(span) +
                                     " must be a positive multiple of " + std::to_string(align));
  if (iteration > kMaxSegmentEnd / span - 1)
    throw Error(Errc::Overflow, "iteration " + std::to_string(iteration) +
                                    " is past the 64-bit value range");
  const uint64_t sub = span / config.threads;
  std::vector<WorkerAssignment> plan(config.threads);
  for (unsigned j = 0; j < config.threads; ++j)
    plan[j] = {iteration, j, iteration * span + j * sub, iteration * span + (j + 1) * sub};
  return plan;
}

// A bad config is reported before any device is touched, as the reference does.
SieveReport run(const SieveConfig& config) {
  validate(config, true);
  return gpu::run(config, gpu::default_context());
}

SieveReport run_unbounded(const SieveConfig& config, const std::atomic<bool>& stop) {
  validate(config, false);
  return gpu::run_unbounded(config, stop, gpu::default_context());
}

namespace gpu {

SieveReport run(const SieveConfig& config, Context& ctx) { return run_loop(config, nullptr, ctx); }

SieveReport run_unbounded(const SieveConfig& config, const std::atomic<bool>& stop, Context& ctx) {
  return run_loop(config, &stop, ctx);
}

}  // namespace gpu

}  // namespace wheelsieve
