// Chunked prime store: the reference's ChunkedFileSink on-disk
// format (sink.hpp:68-141, sink.cpp:39-344) written from device-enumerated
// primes, byte-identical to what the reference CLI writes for the same range
// (`wheelsieve sieve --out`, tools/wheelsieve.cpp:139-168):
//   primes_%05llu.txt  one decimal value per line        (sink.cpp:66-73)
//   primes_%05llu.bin  8-byte little-endian words        (sink.cpp:74-78)
//   manifest.json      nlohmann dump(2), sorted keys, crc32 as 8 hex digits,
//                      written to manifest.json.tmp then renamed (sink.cpp:242-277)
// The binary chunks' CRC-32s are computed on the device (ws_crc.cu) over the
// enumerated words and combined per file with zlib's crc32_combine.
// read_back / verify_store (sink.cpp:306-342) read either implementation's stores.
#include <cuda_runtime.h>
#include <zlib.h>

#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <new>

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "wheelsieve/gpu.h"
#include "ws_internal.h"

namespace fs = std::filesystem;

namespace {

struct StoreFail {
  ws_status code;
  std::string msg;
};

struct FileEntry {
  std::string name;
  uint64_t count = 0, min = 0, max = 0;
  uint32_t crc32 = 0;
};

struct Manifest {
  int format = 0;  // 0 text, 1 binary
  uint64_t primes_per_file = 0, frontier = 0, total_count = 0;
  std::vector<FileEntry> files;
};

std::string chunk_name(uint64_t seq, int format) {  // sink.cpp:48-53
  char buf[48];
  std::snprintf(buf, sizeof buf, "primes_%05llu.%s", static_cast<unsigned long long>(seq),
                format ? "bin" : "txt");
  return buf;
}

std::string crc_hex(uint32_t crc) {  // sink.cpp:55-59
  char buf[16];
  std::snprintf(buf, sizeof buf, "%08x", crc);
  return buf;
}

// nlohmann::json::dump(2) of the manifest object (keys sorted), plus '\n'.
std::string manifest_text(const Manifest& m) {
  std::string s = "{\n  \"files\": [";
  for (size_t i = 0; i < m.files.size(); ++i) {
    const FileEntry& f = m.files[i];
    s += i ? ",\n    {\n" : "\n    {\n";
    s += "      \"count\": " + std::to_string(f.count) + ",\n";
    s += "      \"crc32\": \"" + crc_hex(f.crc32) + "\",\n";
    s += "      \"max\": " + std::to_string(f.max) + ",\n";
    s += "      \"min\": " + std::to_string(f.min) + ",\n";
    s += "      \"name\": \"" + f.name + "\"\n    }";
  }
  s += m.files.empty() ? "],\n" : "\n  ],\n";
  s += std::string("  \"format\": \"") + (m.format ? "binary" : "text") + "\",\n";
  s += "  \"frontier\": " + std::to_string(m.frontier) + ",\n";
  s += "  \"primes_per_file\": " + std::to_string(m.primes_per_file) + ",\n";
  s += "  \"total_count\": " + std::to_string(m.total_count) + "\n}\n";
  return s;
}

// ---- minimal JSON reader for the manifest schema --------------------------
struct Json {
  enum Kind { Null, Num, Str, Arr, Obj } kind = Null;
  uint64_t num = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const char* k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  [[noreturn]] void bad() { throw StoreFail{WS_BAD_MANIFEST, "manifest.json unreadable"}; }
  std::string string() {
    if (p >= e || *p != '"') bad();
    std::string s;
    for (++p; p < e && *p != '"'; ++p) {
      if (*p == '\\') {
        if (++p >= e) bad();
      }
      s.push_back(*p);
    }
    if (p >= e) bad();
    ++p;
    return s;
  }
  Json value() {
    ws();
    if (p >= e) bad();
    Json j;
    if (*p == '{') {
      j.kind = Json::Obj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return j;
      }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (p >= e || *p != ':') bad();
        ++p;
        j.obj.emplace_back(std::move(k), value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return j;
        }
        bad();
      }
    }
    if (*p == '[') {
      j.kind = Json::Arr;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return j;
      }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return j;
        }
        bad();
      }
    }
    if (*p == '"') {
      j.kind = Json::Str;
      j.str = string();
      return j;
    }
    if (*p >= '0' && *p <= '9') {
      j.kind = Json::Num;
      auto [n, ec] = std::from_chars(p, e, j.num);
      if (ec != std::errc{}) bad();
      p = n;
      return j;
    }
    bad();
  }
};

Manifest load_manifest(const fs::path& dir) {  // sink.cpp:113-159
  std::ifstream in(dir / "manifest.json", std::ios::binary);
  if (!in) throw StoreFail{WS_BAD_MANIFEST, "no manifest.json under " + dir.string()};
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  Parser ps{text.data(), text.data() + text.size()};
  const Json j = ps.value();
  auto need = [&](const Json* v, Json::Kind k, const char* what) {
    if (!v || v->kind != k)
      throw StoreFail{WS_BAD_MANIFEST, std::string("manifest.json incomplete: ") + what};
    return v;
  };
  Manifest m;
  const std::string fmt = need(j.get("format"), Json::Str, "format")->str;
  if (fmt == "text")
    m.format = 0;
  else if (fmt == "binary")
    m.format = 1;
  else
    throw StoreFail{WS_BAD_MANIFEST, "unknown format '" + fmt + "' in manifest"};
  m.primes_per_file = need(j.get("primes_per_file"), Json::Num, "primes_per_file")->num;
  m.frontier = need(j.get("frontier"), Json::Num, "frontier")->num;
  m.total_count = need(j.get("total_count"), Json::Num, "total_count")->num;
  for (const Json& f : need(j.get("files"), Json::Arr, "files")->arr) {
    FileEntry fe;
    fe.name = need(f.get("name"), Json::Str, "name")->str;
    fe.count = need(f.get("count"), Json::Num, "count")->num;
    fe.min = need(f.get("min"), Json::Num, "min")->num;
    fe.max = need(f.get("max"), Json::Num, "max")->num;
    const std::string crc = need(f.get("crc32"), Json::Str, "crc32")->str;
    char* endp = nullptr;
    fe.crc32 = static_cast<uint32_t>(std::strtoul(crc.c_str(), &endp, 16));
    if (crc.empty() || *endp) throw StoreFail{WS_BAD_MANIFEST, "manifest.json malformed crc32"};
    m.files.push_back(std::move(fe));
  }
  return m;
}

void encode_text(std::string& out, const uint64_t* v, uint64_t n) {  // sink.cpp:66-73
  char digits[24];
  for (uint64_t i = 0; i < n; ++i) {
    auto [end, ec] = std::to_chars(digits, digits + sizeof digits, v[i]);
    out.append(digits, end);
    out.push_back('\n');
  }
}

uint32_t crc_extend(uint32_t crc, const std::string& bytes) {
  uLong c = crc;
  for (size_t off = 0; off < bytes.size(); off += (1u << 30))
    c = ::crc32(c, reinterpret_cast<const Bytef*>(bytes.data() + off),
                static_cast<uInt>(std::min<size_t>(1u << 30, bytes.size() - off)));
  return static_cast<uint32_t>(c);
}

std::vector<uint64_t> load_and_verify(const fs::path& dir, const FileEntry& f, int format) {
  std::ifstream in(dir / f.name, std::ios::binary);  // sink.cpp:161-183
  if (!in) throw StoreFail{WS_BAD_MANIFEST, "manifest lists missing chunk file " + f.name};
  std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  uLong c = ::crc32(0, Z_NULL, 0);
  for (size_t off = 0; off < bytes.size(); off += (1u << 30))
    c = ::crc32(c, reinterpret_cast<const Bytef*>(bytes.data() + off),
                static_cast<uInt>(std::min<size_t>(1u << 30, bytes.size() - off)));
  const uint32_t crc = static_cast<uint32_t>(c);
  if (crc != f.crc32)
    throw StoreFail{WS_CHECKSUM_MISMATCH, "chunk file " + f.name +
                                              " does not match its recorded crc32 " +
                                              crc_hex(f.crc32)};
  std::vector<uint64_t> v;
  if (format == 0) {
    const char* p = bytes.data();
    const char* e = p + bytes.size();
    while (p < e) {
      uint64_t x = 0;
      auto [next, ec] = std::from_chars(p, e, x);
      if (ec != std::errc{} || next == e || *next != '\n')
        throw StoreFail{WS_BAD_MANIFEST, "chunk file " + f.name + " is not well-formed text"};
      v.push_back(x);
      p = next + 1;
    }
  } else {
    if (bytes.size() % 8)
      throw StoreFail{WS_BAD_MANIFEST, "chunk file " + f.name + " is not a whole number of words"};
    v.resize(bytes.size() / 8);
    std::memcpy(v.data(), bytes.data(), bytes.size());  // little-endian host
  }
  if (v.size() != f.count)
    throw StoreFail{WS_BAD_MANIFEST, "chunk file " + f.name + " holds " + std::to_string(v.size()) +
                                         " values, manifest says " + std::to_string(f.count)};
  return v;
}

void write_file(const fs::path& path, const void* data, size_t bytes) {
  std::FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) throw StoreFail{WS_IO, "cannot open chunk file " + path.filename().string()};
  const size_t w = bytes ? std::fwrite(data, 1, bytes, fp) : 0;
  const bool ok = std::fclose(fp) == 0 && w == bytes;
  if (!ok) throw StoreFail{WS_IO, "write to " + path.filename().string() + " failed"};
}

void write_manifest(const fs::path& dir, const Manifest& m) {  // sink.cpp:242-277
  const std::string text = manifest_text(m);
  const fs::path tmp = dir / "manifest.json.tmp";
  write_file(tmp, text.data(), text.size());
  std::error_code ec;
  fs::rename(tmp, dir / "manifest.json", ec);
  if (ec) throw StoreFail{WS_IO, "replacing manifest failed: " + ec.message()};
}

}  // namespace

// Device half of the store: CRC-32 of byte ranges of device-resident values.
namespace wsk {
cudaError_t launch_crc32_ranges(const void* data, const uint64_t* begin, const uint64_t* len,
                                uint32_t n, uint32_t* out, cudaStream_t st);
}

// The streaming writer behind ws_store_* and ws_store_range: the
// ChunkedFileSink life cycle (sink.cpp:185-304) -- files opened on demand,
// closed at primes_per_file values, the manifest rewritten (write-then-
// rename) at every rollover and on flush, so everything it lists is durable.
struct ws_store {
  fs::path dir;
  int format = 0;
  uint64_t per_file = 0;
  std::vector<FileEntry> closed;
  std::FILE* fp = nullptr;
  FileEntry cur;  // the open file (count 0 until its first value)
  uint64_t next_seq = 0;
  uint64_t largest = 0;
  uint64_t frontier = 0;
  bool frontier_set = false;
  uint64_t durable = 0;
  std::string err;
  std::string text;  // text-format encoding buffer

  std::string durable_note() const { return " (" + std::to_string(durable) + " primes durable)"; }

  void open_next() {
    cur = FileEntry{};
    cur.name = chunk_name(next_seq++, format);
    fp = std::fopen((dir / cur.name).c_str(), "wb");
    if (!fp) throw StoreFail{WS_IO, "cannot open chunk file " + cur.name + durable_note()};
    cur.crc32 = static_cast<uint32_t>(::crc32(0, Z_NULL, 0));
  }

  void write_at(const std::vector<std::pair<const char*, size_t>>& parts) {
    // sequential: writes to one file serialise on its inode anyway (parallel
    // pwrite()s measured no faster, C4e store 2.7 vs 3.2 GB/s)
    for (const auto& pr : parts)
      if (pr.second && std::fwrite(pr.first, 1, pr.second, fp) != pr.second)
        throw StoreFail{WS_IO, "write to " + cur.name + " failed" + durable_note()};
  }

  void write_bytes(const void* p, size_t n) { write_at({{static_cast<const char*>(p), n}}); }


  // n ascending values into the open file; crc_known: the CRC-32 of their
  // little-endian bytes, computed on the device (binary format only)
  void put(const uint64_t* v, uint64_t n, const uint32_t* crc_known) {
    if (format == 1) {
      write_bytes(v, n * 8);  // little-endian host: the words are the bytes
      if (crc_known) {
        cur.crc32 = static_cast<uint32_t>(
            ::crc32_combine(cur.crc32, *crc_known, static_cast<z_off_t>(n * 8)));
      } else {
        uLong c = cur.crc32;
        const auto* b = reinterpret_cast<const Bytef*>(v);
        for (uint64_t off = 0; off < n * 8; off += (1u << 30))
          c = ::crc32(c, b + off, static_cast<uInt>(std::min<uint64_t>(1u << 30, n * 8 - off)));
        cur.crc32 = static_cast<uint32_t>(c);
      }
    } else if (n < (1u << 20)) {
      text.clear();
      encode_text(text, v, n);
      write_bytes(text.data(), text.size());
      cur.crc32 = crc_extend(cur.crc32, text);
    } else {
      // large batches: decimal encoding and CRC in parallel pieces (the
      // encoding, not the disk, bounds a text store), written in order and
      // the pieces' CRCs chained with crc32_combine
      const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
      std::vector<std::string> piece(T);
      std::vector<uint32_t> pcrc(T, 0);
      std::vector<std::thread> th;
      for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const uint64_t a = n * t / T, b = n * (t + 1) / T;
          piece[t].reserve((b - a) * 17);
          encode_text(piece[t], v + a, b - a);
          pcrc[t] = crc_extend(static_cast<uint32_t>(::crc32(0, Z_NULL, 0)), piece[t]);
        });
      for (auto& x : th) x.join();
      std::vector<std::pair<const char*, size_t>> parts;
      for (unsigned t = 0; t < T; ++t) {
        parts.emplace_back(piece[t].data(), piece[t].size());
        cur.crc32 = static_cast<uint32_t>(
            ::crc32_combine(cur.crc32, pcrc[t], static_cast<z_off_t>(piece[t].size())));
      }
      write_at(parts);
    }
    if (cur.count == 0) cur.min = v[0];
    cur.max = v[n - 1];
    cur.count += n;
    largest = v[n - 1];
  }

  void close_file() {
    if (!fp) return;
    const bool ok = std::fclose(fp) == 0;
    fp = nullptr;
    if (!ok) throw StoreFail{WS_IO, "closing " + cur.name + " failed" + durable_note()};
    closed.push_back(cur);
    manifest();
  }

  void manifest() {
    Manifest m;
    m.format = format;
    m.primes_per_file = per_file;
    m.files = closed;
    for (const FileEntry& f : closed) m.total_count += f.count;
    m.frontier = frontier_set ? frontier : (largest == 0 ? 0 : largest + 1);
    write_manifest(dir, m);
    durable = m.total_count;
  }

  // values split at file boundaries; crcs (nullable): one per piece the split
  // produces, in order (the caller computed them with the same split)
  void append(const uint64_t* v, uint64_t n, const uint32_t* crcs) {
    while (n) {
      if (!fp) open_next();
      const uint64_t take = std::min(n, per_file - cur.count);
      put(v, take, crcs);
      if (crcs) ++crcs;
      v += take;
      n -= take;
      if (cur.count == per_file) close_file();
    }
  }

  void flush() {
    if (fp)
      close_file();
    else
      manifest();
  }
};

namespace {

template <class F>
ws_status store_guard(ws_store* st, F&& f) {
  if (!st) return WS_BAD_CONFIG;
  st->err.clear();
  try {
    f();
  } catch (const StoreFail& e) {
    st->err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    st->err = e.what();
    return WS_IO;
  }
  return WS_OK;
}

}  // namespace

extern "C" {

ws_status ws_store_open(const char* dir, uint32_t format, uint64_t primes_per_file,
                        ws_store** out) {
  if (!dir || !out) return WS_BAD_CONFIG;
  *out = nullptr;
  if (primes_per_file == 0) return WS_DOMAIN;  // sink.cpp:187-188
  if (format > 1) return WS_BAD_CONFIG;
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec) return WS_IO;
  ws_store* st = new (std::nothrow) ws_store;
  if (!st) return WS_OUT_OF_MEMORY;
  st->dir = dir;
  st->format = static_cast<int>(format);
  st->per_file = primes_per_file;
  *out = st;
  return WS_OK;
}

ws_status ws_store_append(ws_store* st, const uint64_t* values, uint64_t n) {
  return store_guard(st, [&] {
    if (n && !values) throw StoreFail{WS_BAD_CONFIG, "null values"};
    st->append(values, n, nullptr);
  });
}

ws_status ws_store_set_frontier(ws_store* st, uint64_t frontier) {
  return store_guard(st, [&] {
    if (frontier <= st->largest && st->largest != 0)  // sink.cpp:296-302
      throw StoreFail{WS_DOMAIN, "frontier " + std::to_string(frontier) +
                                     " does not cover the emitted prime " +
                                     std::to_string(st->largest)};
    st->frontier = frontier;
    st->frontier_set = true;
  });
}

ws_status ws_store_flush(ws_store* st) { return store_guard(st, [&] { st->flush(); }); }

uint64_t ws_store_durable_count(const ws_store* st) { return st ? st->durable : 0; }

const char* ws_store_last_error(const ws_store* st) { return st ? st->err.c_str() : "null store"; }

ws_status ws_store_close(ws_store* st) {
  if (!st) return WS_OK;
  const ws_status s = store_guard(st, [&] { st->flush(); });
  if (st->fp) std::fclose(st->fp);
  delete st;
  return s;
}

// [L, R) enumerated on the device in value windows of bounded size; each
// window's values are CRC'd on the device piece by piece (binary format),
// copied to a pinned staging buffer and appended to the streaming writer.
ws_status ws_store_range(ws_ctx* ctx, uint64_t L, uint64_t R, const char* dir, uint32_t format,
                         uint64_t primes_per_file, uint64_t* n_out) {
  if (!ctx || !dir || !n_out) return WS_BAD_CONFIG;
  *n_out = 0;
  if (primes_per_file == 0) return WS_DOMAIN;  // sink.cpp:187-188
  if (format > 1) return WS_BAD_CONFIG;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  const int dev0 = ws_ctx_device(ctx, 0);
  ws_store* st = nullptr;
  uint64_t* dbuf = nullptr;
  uint64_t* hbuf = nullptr;
  uint64_t* d_rng = nullptr;
  uint32_t* d_crc = nullptr;
  auto cleanup = [&] {
    if (dbuf) cudaFree(dbuf);
    if (hbuf) cudaFreeHost(hbuf);
    if (d_rng) cudaFree(d_rng);
    if (d_crc) cudaFree(d_crc);
    if (st) {
      if (st->fp) std::fclose(st->fp);
      delete st;
    }
    if (prev >= 0) cudaSetDevice(prev);
  };
  ws_status code = WS_OK;
  try {
    if (cudaSetDevice(dev0) != cudaSuccess) throw StoreFail{WS_NO_DEVICE, "cudaSetDevice"};
    ws_status s = ws_store_open(dir, format, primes_per_file, &st);
    if (s != WS_OK) throw StoreFail{s, std::string("cannot create output directory ") + dir};
    // value windows of whole segments, at most ~2^30 integers: the densest
    // window (the first) bounds the buffers, 8 B per prime on each side
    const uint64_t span = 6ull * (1u << 18) * 682;
    const uint64_t lo0 = L / 6 * 6;
    uint64_t cap = 1;
    for (uint64_t a = L; a < R;) {
      const uint64_t b = (R - lo0 > (a - lo0) + span) ? lo0 + ((a - lo0) / span + 1) * span : R;
      cap = std::max(cap, ws_prime_count_bound(a, b));
      break;  // the first window is the densest
    }
    constexpr uint64_t kPiece = 8192;  // values per device CRC range
    const uint64_t max_ranges = cap / kPiece + 2 * (cap / primes_per_file + 2) + 4;
    if (cudaMalloc(&dbuf, cap * 8) != cudaSuccess ||
        cudaMalloc(&d_rng, 2 * max_ranges * 8) != cudaSuccess ||
        cudaMalloc(&d_crc, max_ranges * 4) != cudaSuccess)
      throw StoreFail{WS_OUT_OF_MEMORY, "store window buffers"};
    if (cudaMallocHost(&hbuf, cap * 8) != cudaSuccess)
      throw StoreFail{WS_OUT_OF_MEMORY, "store host staging"};
    cudaStream_t strm = static_cast<cudaStream_t>(ws_ctx_stream(ctx));
    std::vector<uint64_t> begin, len, cuts;
    std::vector<uint32_t> crc, piece_crc;
    uint64_t total = 0;
    for (uint64_t a = L; a < R;) {
      const uint64_t b = (R - lo0 > (a - lo0) + span) ? lo0 + ((a - lo0) / span + 1) * span : R;
      uint64_t n = 0;
      ws_checks chk{};
      s = ws_enumerate_range(ctx, a, b, WS_OUT_DEVICE, dbuf, cap, &n, &chk);
      if (s != WS_OK) throw StoreFail{s, ws_last_error(ctx)};
      if (cudaSetDevice(dev0) != cudaSuccess) throw StoreFail{WS_NO_DEVICE, "cudaSetDevice"};
      if (n) {
        // the pieces append() will cut this window into: file boundaries
        cuts.assign(1, 0);
        uint64_t room = st->fp ? primes_per_file - st->cur.count : primes_per_file;
        for (uint64_t x = 0; x < n;) {
          const uint64_t t = std::min(n - x, room);
          x += t;
          cuts.push_back(x);
          room = primes_per_file;
        }
        const uint64_t np = cuts.size() - 1;
        piece_crc.assign(np, 0);
        if (format == 1) {  // device CRC of every <= 64 KiB range inside each piece
          begin.clear();
          len.clear();
          std::vector<uint64_t> first(np + 1, 0);
          for (uint64_t p = 0; p < np; ++p) {
            first[p] = begin.size();
            for (uint64_t x = cuts[p]; x < cuts[p + 1]; x += kPiece) {
              begin.push_back(8 * x);
              len.push_back(8 * (std::min(cuts[p + 1], x + kPiece) - x));
            }
          }
          first[np] = begin.size();
          const uint64_t nr = begin.size();
          if (nr > max_ranges) throw StoreFail{WS_CUDA, "store range table overflow"};
          crc.resize(nr);
          if (cudaMemcpyAsync(d_rng, begin.data(), nr * 8, cudaMemcpyHostToDevice, strm) !=
                  cudaSuccess ||
              cudaMemcpyAsync(d_rng + nr, len.data(), nr * 8, cudaMemcpyHostToDevice, strm) !=
                  cudaSuccess ||
              wsk::launch_crc32_ranges(dbuf, d_rng, d_rng + nr, static_cast<uint32_t>(nr), d_crc,
                                       strm) != cudaSuccess ||
              cudaMemcpyAsync(crc.data(), d_crc, nr * 4, cudaMemcpyDeviceToHost, strm) !=
                  cudaSuccess)
            throw StoreFail{WS_CUDA, "device crc"};
          if (cudaMemcpyAsync(hbuf, dbuf, n * 8, cudaMemcpyDeviceToHost, strm) != cudaSuccess ||
              cudaStreamSynchronize(strm) != cudaSuccess)
            throw StoreFail{WS_CUDA, "values readback"};
          for (uint64_t p = 0; p < np; ++p) {
            uLong c = ::crc32(0, Z_NULL, 0);
            for (uint64_t r = first[p]; r < first[p + 1]; ++r)
              c = ::crc32_combine(c, crc[r], static_cast<z_off_t>(len[r]));
            piece_crc[p] = static_cast<uint32_t>(c);
          }
          st->append(hbuf, n, piece_crc.data());
        } else {
          if (cudaMemcpyAsync(hbuf, dbuf, n * 8, cudaMemcpyDeviceToHost, strm) != cudaSuccess ||
              cudaStreamSynchronize(strm) != cudaSuccess)
            throw StoreFail{WS_CUDA, "values readback"};
          st->append(hbuf, n, nullptr);
        }
      }
      total += n;
      a = b;
    }
    // the CLI records the sieved-through bound (wheelsieve.cpp:167)
    st->frontier = R;
    st->frontier_set = true;
    st->flush();
    *n_out = total;
  } catch (const StoreFail& e) {
    code = e.code;
  } catch (...) {
    code = WS_IO;
  }
  cleanup();
  return code;
}

ws_status ws_read_back(const char* dir, uint64_t lo, uint64_t hi, uint64_t* out, uint64_t cap,
                       uint64_t* n_out) {  // sink.cpp:306-321
  if (!dir || !n_out) return WS_BAD_CONFIG;
  *n_out = 0;
  if (lo >= hi) return WS_OK;
  try {
    const Manifest m = load_manifest(dir);
    if (hi > m.frontier) return WS_BEYOND_FRONTIER;
    uint64_t n = 0;
    for (const FileEntry& f : m.files) {
      if (f.count == 0 || f.max < lo || f.min >= hi) continue;
      for (uint64_t v : load_and_verify(dir, f, m.format))
        if (lo <= v && v < hi) {
          if (out && n < cap) out[n] = v;
          ++n;
        }
    }
    *n_out = n;
    return n > cap ? WS_CAPACITY : WS_OK;
  } catch (const StoreFail& e) {
    return e.code;
  } catch (...) {
    return WS_IO;
  }
}

ws_status ws_verify_store(const char* dir) {  // sink.cpp:323-342
  if (!dir) return WS_BAD_CONFIG;
  try {
    const Manifest m = load_manifest(dir);
    uint64_t total = 0, prev = 0;
    for (const FileEntry& f : m.files) {
      const std::vector<uint64_t> v = load_and_verify(dir, f, m.format);
      if (!v.empty() && (v.front() != f.min || v.back() != f.max)) return WS_BAD_MANIFEST;
      for (uint64_t x : v) {
        if (x <= prev) return WS_BAD_MANIFEST;
        prev = x;
      }
      total += v.size();
    }
    return total == m.total_count ? WS_OK : WS_BAD_MANIFEST;
  } catch (const StoreFail& e) {
    return e.code;
  } catch (...) {
    return WS_IO;
  }
}

}  // extern "C"
