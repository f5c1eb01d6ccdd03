// wheelsieve::gpu::Context and the default context (wheelsieve/gpu.hpp):
// thin C++ ownership over the C ABI of libwheelsieve_cuda.so.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>

#include "wheelsieve/gpu.hpp"

namespace wheelsieve::gpu {

void check(ws_status status, const ws_ctx* ctx, const char* what) {
  if (status == WS_OK) return;
  std::string msg = std::string(what) + ": " + ws_status_name(status);
  if (ctx && *ws_last_error(ctx)) msg += std::string(": ") + ws_last_error(ctx);
  throw Error(static_cast<Errc>(static_cast<int>(status) - 1), msg);
}

std::string nccl_unique_id() {
  std::string id(WS_NCCL_ID_BYTES, '\0');
  check(ws_nccl_unique_id(reinterpret_cast<uint8_t*>(id.data())), nullptr, "nccl_unique_id");
  return id;
}

Context::Context(int device, uint32_t segment_slots)
    : Context(ContextOptions{{}, device, segment_slots, 1, 0, {}}) {}

Context::Context(const ContextOptions& o) : slots_(o.segment_slots) {
  ws_opts w;
  ws_opts_default(&w);
  w.segment_slots = o.segment_slots;
  w.device = o.device;
  if (o.devices.size() > WS_MAX_DEVICES)
    throw Error(Errc::BadConfig, "at most " + std::to_string(WS_MAX_DEVICES) + " devices");
  w.n_devices = static_cast<uint32_t>(o.devices.size());
  std::copy(o.devices.begin(), o.devices.end(), w.device_ids);
  w.world = o.world;
  w.rank = o.rank;
  if (o.world > 1) {
    if (o.nccl_id.size() != WS_NCCL_ID_BYTES)
      throw Error(Errc::BadConfig, "a multi-process context needs rank 0's nccl_unique_id()");
    std::memcpy(w.nccl_id, o.nccl_id.data(), WS_NCCL_ID_BYTES);
  }
  check(ws_ctx_create(&w, &ctx_), nullptr, "ws_ctx_create");
}

Context::~Context() { ws_ctx_destroy(ctx_); }

ws_timing Context::timing() const {
  ws_timing t{};
  check(ws_last_timing(ctx_, &t), ctx_, "ws_last_timing");
  return t;
}

Checks Context::count_range(uint64_t L, uint64_t R, bool checksums,
                            std::vector<uint32_t>* per_segment) {
  ws_checks c{};
  uint64_t nseg = 0;
  if (per_segment) {
    const uint64_t slots = R > L ? (R - L / 6 * 6 + 5) / 6 : 0;
    per_segment->assign((slots + slots_ - 1) / slots_, 0);
  }
  check(ws_count_range(ctx_, L, R, checksums ? WS_WANT_CHECKS : 0u, &c,
                       per_segment ? per_segment->data() : nullptr,
                       per_segment ? per_segment->size() : 0, &nseg),
        ctx_, "ws_count_range");
  return {c.count, c.sum, c.xor_, c.largest};
}

std::vector<uint64_t> Context::enumerate_range(uint64_t L, uint64_t R, Checks* checks) {
  std::vector<uint64_t> out(std::max<uint64_t>(1, ws_prime_count_bound(L, R)));
  uint64_t n = 0;
  ws_checks c{};
  check(ws_enumerate_range(ctx_, L, R, 0u, out.data(), out.size(), &n, &c), ctx_,
        "ws_enumerate_range");
  out.resize(n);
  if (checks) *checks = {c.count, c.sum, c.xor_, c.largest};
  return out;
}

std::vector<Checks> Context::count_ranges(std::span<const uint64_t> Ls,
                                          std::span<const uint64_t> Rs, bool checksums) {
  if (Ls.size() != Rs.size()) throw Error(Errc::BadConfig, "range bounds differ in length");
  std::vector<ws_checks> raw(Ls.size());
  check(ws_count_ranges(ctx_, Ls.data(), Rs.data(), Ls.size(), checksums ? WS_WANT_CHECKS : 0u,
                        raw.data()),
        ctx_, "ws_count_ranges");
  std::vector<Checks> out(raw.size());
  for (size_t i = 0; i < raw.size(); ++i)
    out[i] = {raw[i].count, raw[i].sum, raw[i].xor_, raw[i].largest};
  return out;
}

void Context::count_intervals(std::span<const uint64_t> Ls, uint64_t width,
                              std::vector<uint32_t>& counts, std::vector<uint64_t>* sums,
                              std::vector<uint64_t>* xors) {
  counts.assign(Ls.size(), 0);
  if (sums) sums->assign(Ls.size(), 0);
  if (xors) xors->assign(Ls.size(), 0);
  check(ws_count_intervals(ctx_, Ls.data(), Ls.size(), width, 0u, counts.data(),
                           sums ? sums->data() : nullptr, xors ? xors->data() : nullptr),
        ctx_, "ws_count_intervals");
}

std::vector<uint64_t> Context::base_primes(uint64_t B) {
  std::vector<uint64_t> out(std::max<uint64_t>(1, ws_prime_count_bound(0, B + 1)));
  uint64_t n = 0;
  check(ws_base_primes(ctx_, B, 0u, out.data(), out.size(), &n), ctx_, "ws_base_primes");
  out.resize(n);
  return out;
}

void Context::sieve_segment_words(uint64_t start, uint64_t len, uint64_t* r1_words,
                                  uint64_t* r5_words) {
  check(ws_sieve_segment(ctx_, start, len, 0u, r1_words, r5_words), ctx_, "ws_sieve_segment");
}

uint64_t Context::store_range(uint64_t L, uint64_t R, const std::string& dir, bool binary,
                              uint64_t primes_per_file) {
  uint64_t n = 0;
  check(ws_store_range(ctx_, L, R, dir.c_str(), binary ? WS_STORE_BINARY : WS_STORE_TEXT,
                       primes_per_file, &n),
        ctx_, "ws_store_range");
  return n;
}

namespace {

std::mutex g_mu;
std::unique_ptr<Context> g_owned;
Context* g_installed = nullptr;

// WHEELSIEVE_DEVICES: "all", or a comma list of CUDA ordinals.
ContextOptions options_from_env() {
  ContextOptions o;
  const char* env = std::getenv("WHEELSIEVE_DEVICES");
  if (!env || !*env) return o;
  const std::string s(env);
  if (s == "all") {
    int n = 0;
    for (; n < WS_MAX_DEVICES; ++n) {
      ws_opts probe;
      ws_opts_default(&probe);
      probe.device = n;
      ws_ctx* c = nullptr;
      if (ws_ctx_create(&probe, &c) != WS_OK) break;
      ws_ctx_destroy(c);
    }
    for (int i = 0; i < n; ++i) o.devices.push_back(i);
    return o;
  }
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) o.devices.push_back(std::stoi(item));
  return o;
}

}  // namespace

Context& default_context() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_installed) return *g_installed;
  if (!g_owned) g_owned = std::make_unique<Context>(options_from_env());
  return *g_owned;
}

void set_default_context(Context* ctx) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_installed = ctx;
}

}  // namespace wheelsieve::gpu
