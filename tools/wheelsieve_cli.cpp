// wheelsieve (GPU): the reference CLI's three subcommands
// (/root/reference/proj/tools/wheelsieve.cpp) with the same flags, output
// lines, CSV and exit codes (0 ok, 1 error / verify mismatch, 2 usage),
// built on the drop-in C++ API (include/wheelsieve/*.hpp, libwheelsieve.so):
// run(), run_unbounded(), CountSink, ChunkedFileSink and a buffered stdout
// sink.  `--threads` shapes the worker tiles as in the reference; the
// sieving runs on the GPUs of the default context (WHEELSIEVE_DEVICES).
//
//   wheelsieve sieve  --limit N|unbounded [--threads T] [--segment S]
//                     [--flag-width bit|byte|word4] [--count-only | --out DIR]
//                     [--format text|binary] [--primes-per-file K] [--spawn-per-iteration]
//   wheelsieve verify --limit N [--threads T] [--segment S] [--flag-width W] [--poison P]
//   wheelsieve bench  --limits a,b,.. [--threads ..] [--segments ..] [--flag-widths ..]
//                     [--repeats R] [--csv PATH]
#include <algorithm>
#include <atomic>
#include <charconv>
#include <csignal>
#include <ctime>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "wheelsieve/engine.hpp"
#include "wheelsieve/sink.hpp"
#include "wheelsieve/wheel.hpp"

using namespace wheelsieve;

namespace {

std::atomic<bool> g_stop{false};
std::atomic<long long> g_first_sigint_ms{0};

// A second ^C aborts at once -- but only one that comes a while after the
// first: `timeout -s INT` signals the child and then its whole process group,
// so one interruption can arrive as two back-to-back SIGINTs.
extern "C" void on_sigint(int) {
  g_stop.store(true);
  timespec ts{};
  clock_gettime(CLOCK_MONOTONIC, &ts);  // async-signal-safe
  const long long now = ts.tv_sec * 1000LL + ts.tv_nsec / 1000000 + 1;
  long long first = 0;
  if (g_first_sigint_ms.compare_exchange_strong(first, now)) return;
  if (now - first > 500) std::_Exit(130);
}

struct Usage {
  std::string msg;
};

template <class T>
T parse_uint(const std::string& flag, const std::string& s) {
  T v{};
  auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc{} || end != s.data() + s.size())
    throw Usage{flag + " expects an unsigned integer, got '" + s + "'"};
  return v;
}

template <class T>
std::vector<T> parse_list(const std::string& flag, const std::string& s) {
  std::vector<T> out;
  size_t a = 0;
  while (a <= s.size()) {
    const size_t b = std::min(s.find(',', a), s.size());
    out.push_back(parse_uint<T>(flag, s.substr(a, b - a)));
    a = b + 1;
  }
  return out;
}

FlagWidth parse_width(const std::string& s) {
  std::string l = s;
  for (char& c : l) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  if (l == "bit") return FlagWidth::Bit;
  if (l == "byte") return FlagWidth::Byte;
  if (l == "word4") return FlagWidth::Word4;
  throw Usage{"--flag-width must be bit, byte or word4, got '" + s + "'"};
}

const char* width_text(FlagWidth w) {
  return w == FlagWidth::Bit ? "bit" : w == FlagWidth::Byte ? "byte" : "word4";
}

unsigned threads_default() {
  if (const char* e = std::getenv("WHEELSIEVE_THREADS")) {
    char* end = nullptr;
    const unsigned long v = std::strtoul(e, &end, 10);
    if (end != e && *end == '\0' && v >= 1 && v <= 1024) return static_cast<unsigned>(v);
    std::cerr << "warning: ignoring invalid WHEELSIEVE_THREADS='" << e << "'\n";
  }
  return std::max(1u, std::thread::hardware_concurrency());
}

uint64_t span_for(uint64_t requested, unsigned threads) {
  const uint64_t s = round_segment_span(requested, threads);
  if (s != requested)
    std::cerr << "warning: segment span rounded up to " << s << " (multiple of 6*" << threads
              << ")\n";
  return s;
}

// flag -> value over argv[from..]; flags listed in `bare` take no value
std::map<std::string, std::string> options(int argc, char** argv, int from,
                                           const std::vector<std::string>& valued,
                                           const std::vector<std::string>& bare) {
  std::map<std::string, std::string> o;
  for (int i = from; i < argc; ++i) {
    std::string a = argv[i], v;
    const size_t eq = a.find('=');
    if (eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    if (std::find(bare.begin(), bare.end(), a) != bare.end()) {
      o[a] = "1";
      continue;
    }
    if (std::find(valued.begin(), valued.end(), a) == valued.end()) throw Usage{"unknown option " + a};
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw Usage{a + " needs a value"};
      v = argv[++i];
    }
    o[a] = v;
  }
  return o;
}

// One decimal per line, written in ~1 MB chunks.
class StdoutSink final : public PrimeSink {
 public:
  ~StdoutSink() override { drain(); }
  void flush() override {
    drain();
    std::fflush(stdout);
  }

 protected:
  void accept(std::span<const uint64_t> batch) override {
    char d[24];
    for (uint64_t v : batch) {
      const auto r = std::to_chars(d, d + sizeof d, v);
      text_.append(d, r.ptr);
      text_.push_back('\n');
    }
    if (text_.size() >= (1u << 20)) drain();
  }

 private:
  void drain() {
    if (!text_.empty()) std::fwrite(text_.data(), 1, text_.size(), stdout);
    text_.clear();
  }
  std::string text_;
};

void summary(const SieveReport& r) {
  std::printf("count=%llu largest=%llu ms=%.3f\n", static_cast<unsigned long long>(r.prime_count),
              static_cast<unsigned long long>(r.largest_prime), r.wall_ms);
}

int cmd_sieve(int argc, char** argv) {
  auto o = options(argc, argv, 2,
                   {"--limit", "--threads", "--segment", "--flag-width", "--out", "--format",
                    "--primes-per-file"},
                   {"--count-only", "--spawn-per-iteration"});
  if (!o.count("--limit")) throw Usage{"--limit is required"};
  if (o.count("--count-only") && o.count("--out"))
    throw Usage{"--count-only excludes --out"};
  const bool unbounded = o["--limit"] == "unbounded";
  SieveConfig c;
  if (!unbounded) c.limit = parse_uint<uint64_t>("--limit", o["--limit"]);
  c.threads = o.count("--threads") ? parse_uint<unsigned>("--threads", o["--threads"])
                                   : threads_default();
  const uint64_t seg =
      o.count("--segment") ? parse_uint<uint64_t>("--segment", o["--segment"]) : 6'000'000;
  if (o.count("--flag-width")) c.flag_width = parse_width(o["--flag-width"]);
  c.spawn_per_iteration = o.count("--spawn-per-iteration") > 0;
  FileFormat fmt = FileFormat::Text;
  if (o.count("--format")) {
    if (o["--format"] == "binary")
      fmt = FileFormat::Binary;
    else if (o["--format"] != "text")
      throw Usage{"--format must be text or binary"};
  }
  const uint64_t per_file = o.count("--primes-per-file")
                                ? parse_uint<uint64_t>("--primes-per-file", o["--primes-per-file"])
                                : 125'000'000;
  c.segment_span = span_for(seg, c.threads);
  std::unique_ptr<PrimeSink> sink;
  ChunkedFileSink* files = nullptr;
  if (o.count("--count-only")) {
    sink = std::make_unique<CountSink>();
  } else if (o.count("--out")) {
    auto f = std::make_unique<ChunkedFileSink>(ChunkedFileOptions{o["--out"], per_file, fmt});
    files = f.get();
    sink = std::move(f);
  } else {
    sink = std::make_unique<StdoutSink>();
  }
  c.sink = sink.get();
  SieveReport r;
  if (unbounded) {
    std::signal(SIGINT, on_sigint);
    r = run_unbounded(c, g_stop);
    std::signal(SIGINT, SIG_DFL);
  } else {
    r = run(c);
  }
  if (files) files->set_frontier(r.sieved_to);
  sink->flush();
  if (r.overflowed) std::cerr << "note: enumeration reached the end of the 64-bit range\n";
  summary(r);
  return 0;
}

int cmd_verify(int argc, char** argv) {
  auto o = options(argc, argv, 2, {"--limit", "--threads", "--segment", "--flag-width", "--poison"},
                   {});
  if (!o.count("--limit")) throw Usage{"--limit is required"};
  const uint64_t limit = parse_uint<uint64_t>("--limit", o["--limit"]);
  const std::vector<uint64_t> want = naive_sieve(limit);
  MemorySink sink;
  SieveConfig c;
  c.limit = limit;
  c.threads = o.count("--threads") ? parse_uint<unsigned>("--threads", o["--threads"])
                                   : threads_default();
  c.segment_span = span_for(
      o.count("--segment") ? parse_uint<uint64_t>("--segment", o["--segment"]) : 6'000'000,
      c.threads);
  if (o.count("--flag-width")) c.flag_width = parse_width(o["--flag-width"]);
  c.sink = &sink;
  run(c);
  std::vector<uint64_t> got = sink.primes();
  if (o.count("--poison")) {  // drop one prime, as a wrongly cleared flag would
    const uint64_t p = parse_uint<uint64_t>("--poison", o["--poison"]);
    const auto it = std::find(got.begin(), got.end(), p);
    if (it != got.end()) got.erase(it);
  }
  const size_t n = std::min(want.size(), got.size());
  size_t i = 0;
  while (i < n && want[i] == got[i]) ++i;
  if (i == n && want.size() == got.size()) {
    std::printf("PASS count=%zu limit=%llu threads=%u segment=%llu\n", got.size(),
                static_cast<unsigned long long>(limit), c.threads,
                static_cast<unsigned long long>(c.segment_span));
    return 0;
  }
  if (i < n)
    std::printf("FAIL first divergence at index %zu: expected %llu, got %llu\n", i,
                static_cast<unsigned long long>(want[i]), static_cast<unsigned long long>(got[i]));
  else if (want.size() > got.size())
    std::printf("FAIL pipeline output ends early at index %zu: expected %llu\n", i,
                static_cast<unsigned long long>(want[i]));
  else
    std::printf("FAIL pipeline emitted extra value %llu at index %zu\n",
                static_cast<unsigned long long>(got[i]), i);
  return 1;
}

int cmd_bench(int argc, char** argv) {
  auto o = options(argc, argv, 2,
                   {"--limits", "--threads", "--segments", "--flag-widths", "--repeats", "--csv"},
                   {});
  if (!o.count("--limits")) throw Usage{"--limits is required"};
  const auto limits = parse_list<uint64_t>("--limits", o["--limits"]);
  const auto threads = o.count("--threads") ? parse_list<unsigned>("--threads", o["--threads"])
                                            : std::vector<unsigned>{threads_default()};
  const auto segments = o.count("--segments")
                            ? parse_list<uint64_t>("--segments", o["--segments"])
                            : std::vector<uint64_t>{6'000'000};
  std::vector<FlagWidth> widths{FlagWidth::Bit};
  if (o.count("--flag-widths")) {
    widths.clear();
    std::string s = o["--flag-widths"];
    size_t a = 0;
    while (a <= s.size()) {
      const size_t b = std::min(s.find(',', a), s.size());
      widths.push_back(parse_width(s.substr(a, b - a)));
      a = b + 1;
    }
  }
  const unsigned repeats = o.count("--repeats") ? parse_uint<unsigned>("--repeats", o["--repeats"]) : 1;
  if (repeats == 0) {
    std::cerr << "error: --repeats must be positive\n";
    return 2;
  }
  std::string csv =
      "threads,limit,segment_span,flag_width,wall_ms,iterations,peak_flag_bytes,prime_count\n";
  std::map<uint64_t, uint64_t> count_of;
  for (uint64_t limit : limits)
    for (unsigned t : threads)
      for (uint64_t seg : segments) {
        const uint64_t span = round_segment_span(seg, t);
        for (FlagWidth w : widths) {
          SieveReport best;
          for (unsigned r = 0; r < repeats; ++r) {
            CountSink sink;
            const SieveReport rep = run({limit, t, span, w, &sink});
            if (r == 0 || rep.wall_ms < best.wall_ms) best = rep;
          }
          const auto [it, fresh] = count_of.emplace(limit, best.prime_count);
          if (!fresh && it->second != best.prime_count) {
            std::cerr << "error: prime count " << best.prime_count << " for limit " << limit
                      << " disagrees with an earlier run (" << it->second << ")\n";
            return 1;
          }
          char row[200];
          std::snprintf(row, sizeof row, "%u,%llu,%llu,%s,%.3f,%llu,%llu,%llu\n", t,
                        static_cast<unsigned long long>(limit),
                        static_cast<unsigned long long>(span), width_text(w), best.wall_ms,
                        static_cast<unsigned long long>(best.iterations),
                        static_cast<unsigned long long>(best.peak_flag_bytes),
                        static_cast<unsigned long long>(best.prime_count));
          csv += row;
        }
      }
  if (!o.count("--csv") || o["--csv"] == "-" || o["--csv"].empty()) {
    std::fputs(csv.c_str(), stdout);
    return 0;
  }
  std::ofstream out(o["--csv"], std::ios::binary | std::ios::trunc);
  out << csv;
  if (!out) {
    std::cerr << "error: cannot write csv to " << o["--csv"] << "\n";
    return 1;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw Usage{"a subcommand is required: sieve, verify or bench"};
    const std::string cmd = argv[1];
    if (cmd == "sieve") return cmd_sieve(argc, argv);
    if (cmd == "verify") return cmd_verify(argc, argv);
    if (cmd == "bench") return cmd_bench(argc, argv);
    throw Usage{"unknown subcommand " + cmd};
  } catch (const Usage& u) {
    std::cerr << "usage error: " << u.msg << "\n";
    return 2;
  } catch (const SinkFailure& e) {
    std::cerr << "error: " << e.what() << " (" << e.partial().prime_count
              << " primes emitted before the failure)\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
