// Sinks and the chunked store (wheelsieve/sink.hpp).  The emission contract
// follows the reference's sink.cpp:14-37; ChunkedFileSink, read_back and
// verify_store go through the library's store (ws_store_*, ws_read_back,
// ws_verify_store in wheelsieve/gpu.h), which writes the reference's format.
#include <string>

#include "wheelsieve/gpu.hpp"
#include "wheelsieve/sink.hpp"

namespace wheelsieve {

void PrimeSink::emit(std::span<const uint64_t> batch) {
  if (batch.empty()) return;
  uint64_t after = last_;
  for (uint64_t v : batch) {
    if (v <= after)
      throw Error(Errc::Ordering, "batch value " + std::to_string(v) + " does not ascend past " +
                                      std::to_string(after));
    after = v;
  }
  accept(batch);
  total_ += batch.size();
  last_ = batch.back();
}

void PrimeSink::emit_count(uint64_t n, uint64_t largest) {
  if (n == 0) return;
  if (wants_values())
    throw Error(Errc::Domain, "this sink needs values, not counts");
  if (largest <= last_)
    throw Error(Errc::Ordering, "count batch ending at " + std::to_string(largest) +
                                    " does not ascend past " + std::to_string(last_));
  total_ += n;
  last_ = largest;
}

namespace {

void store_check(ws_status s, const ws_store* st, const char* what) {
  if (s == WS_OK) return;
  std::string msg = std::string(what) + ": " + ws_status_name(s);
  if (st && *ws_store_last_error(st)) msg += std::string(": ") + ws_store_last_error(st);
  throw Error(static_cast<Errc>(static_cast<int>(s) - 1), msg);
}

}  // namespace

ChunkedFileSink::ChunkedFileSink(ChunkedFileOptions options) : options_(std::move(options)) {
  if (options_.primes_per_file == 0) throw Error(Errc::Domain, "primes_per_file must be positive");
  const ws_status s =
      ws_store_open(options_.dir.c_str(),
                    options_.format == FileFormat::Binary ? WS_STORE_BINARY : WS_STORE_TEXT,
                    options_.primes_per_file, &store_);
  if (s == WS_IO)
    throw Error(Errc::Io, "cannot create output directory " + options_.dir.string());
  store_check(s, nullptr, "ChunkedFileSink");
}

ChunkedFileSink::~ChunkedFileSink() {
  // best effort, as a destructor must be; flush() reports failures
  ws_store_close(store_);
}

void ChunkedFileSink::accept(std::span<const uint64_t> batch) {
  store_check(ws_store_append(store_, batch.data(), batch.size()), store_, "ChunkedFileSink");
}

void ChunkedFileSink::flush() { store_check(ws_store_flush(store_), store_, "flush"); }

void ChunkedFileSink::set_frontier(uint64_t frontier) {
  store_check(ws_store_set_frontier(store_, frontier), store_, "set_frontier");
}

uint64_t ChunkedFileSink::durable_count() const { return ws_store_durable_count(store_); }

std::vector<uint64_t> read_back(const std::filesystem::path& dir, uint64_t lo, uint64_t hi) {
  uint64_t n = 0;
  ws_status s = ws_read_back(dir.c_str(), lo, hi, nullptr, 0, &n);
  if (s != WS_OK && s != WS_CAPACITY) gpu::check(s, nullptr, "read_back");
  std::vector<uint64_t> out(n);
  s = ws_read_back(dir.c_str(), lo, hi, out.data(), out.size(), &n);
  gpu::check(s, nullptr, "read_back");
  out.resize(n);
  return out;
}

void verify_store(const std::filesystem::path& dir) {
  gpu::check(ws_verify_store(dir.c_str()), nullptr, "verify_store");
}

}  // namespace wheelsieve
