/*
 * wheelsieve GPU C ABI -- the drop-in boundary for the B200 segmented
 * mod-6 wheel sieve (libwheelsieve_cuda.so).
 *
 * The reference (/root/reference/proj) is a C++20 library with no C ABI; its
 * sieve is reached through these C++ entry points, which this ABI replaces:
 *
 *   wheelsieve::run(const SieveConfig&)          engine.hpp:83, engine.cpp:344
 *       -> ws_count_range / ws_enumerate_range on [0, limit + 1)
 *   sieve_segment + count_surviving / surviving   segment.hpp:168, segment.cpp:141-162
 *       -> batched: every segment of a range in one device pass
 *   [L, R) count / enumerate (SURVEY §3.3 composition; no single reference call)
 *       -> ws_count_range / ws_enumerate_range / ws_count_intervals
 *   engine tiling plan_iteration / round_segment_span  engine.cpp:311-342
 *       -> ws_partition (contiguous per-GPU super-ranges)
 *   start_offsets (paper Table 1)                 wheel.cpp:96-106  -> ws_start_offsets
 *   BasePrimeStore::bootstrap / naive_sieve       base_store.cpp:34, wheel.cpp:40 -> ws_base_primes
 *   SegmentBitmap + sieve_segment (flag arrays)   segment.cpp:93-188 -> ws_sieve_segment
 *   ChunkedFileSink / read_back / verify_store    sink.cpp:39-344 -> ws_store_range,
 *                                                 ws_read_back, ws_verify_store
 *   isqrt                                         wheel.cpp:25-33   -> ws_isqrt
 *
 * Conventions (mirroring the reference):
 *   - every value range is half-open [L, R); pi(N) is [0, N + 1);
 *   - 2 and 3 are added when in range (engine.cpp:268-276); 1 is never prime
 *     (engine.cpp:244);
 *   - a "segment" is `segment_slots` wheel slots per residue class (6k+1 and
 *     6k+5), spanning 6 * segment_slots values; segment i of [L, R) starts at
 *     floor(L / 6) * 6 + 6 * segment_slots * i and the last one is clipped;
 *     per-segment counts exclude 2 and 3;
 *   - sums are mod 2^64; enumeration output is strictly ascending;
 *   - status codes are 1 + wheelsieve::Errc (errors.hpp:9-23), no exception
 *     ever crosses this ABI; device/runtime failures map to WS_CUDA etc.
 *   - one host thread per context (the engine is not reentrant per run,
 *     SPEC.md:268); a context owns its device buffers and CUDA streams.
 *
 * Multi-GPU (SieveConfig::threads spreads one run() over worker threads,
 * engine.hpp:13-29 / engine.cpp:179-262; here one call spreads over GPUs):
 * a context created with ws_opts.n_devices = k >= 1 owns k devices, one
 * worker thread and one NCCL communicator per device.  With world = W
 * processes (each with the same k) the job is cut into W * k shards; local
 * device i of process `rank` is shard (NCCL rank) rank * k + i.  A range
 * [L, R) is split by ws_partition into contiguous per-shard super-ranges on
 * segment borders, interval batches go interval i -> shard i mod (W k), and
 * range batches (ws_count_ranges) in contiguous blocks.  Each device sieves
 * its shard with no data-path exchange; the per-shard 32-byte records
 * {count, sum, xor, largest} (per-interval records for batches) are
 * combined after exactly one ncclAllGather over NVLink (NCCL has no XOR
 * reduction) with the fold of ws_combine_checks.  Every process receives the
 * combined totals; per-segment counts and enumerated values stay with the
 * process that owns the shard (see ws_enumerate_range).
 */
#ifndef WHEELSIEVE_GPU_H_
#define WHEELSIEVE_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ws_status {
  WS_OK = 0,
  /* 1 + wheelsieve::Errc, errors.hpp:9-23 */
  WS_NOT_ON_WHEEL = 1,
  WS_OVERFLOW = 2,
  WS_EMPTY_RANGE = 3,
  WS_CAPACITY = 4,
  WS_DOMAIN = 5,
  WS_ALIGNMENT = 6,
  WS_BAD_CONFIG = 7,
  WS_INCOMPLETE_BASE = 8,
  WS_ORDERING = 9,
  WS_IO = 10,
  WS_BAD_MANIFEST = 11,
  WS_CHECKSUM_MISMATCH = 12,
  WS_BEYOND_FRONTIER = 13,
  /* device side */
  WS_CUDA = 100,     /* a CUDA runtime call or kernel failed */
  WS_NO_DEVICE = 101, /* no usable sm_100 device */
  WS_OUT_OF_MEMORY = 102,
  WS_NCCL = 103      /* an NCCL call failed (multi-device contexts) */
} ws_status;

/* Flags for the range calls. */
#define WS_WANT_CHECKS 0x1u  /* compute Σ mod 2^64 and ⊕ of the primes (count calls) */
#define WS_OUT_DEVICE 0x2u   /* output pointers are device pointers on the ctx device */
#define WS_FRESH_BASE 0x4u   /* re-sieve the base primes even if cached */

typedef struct ws_ctx ws_ctx;

#define WS_MAX_DEVICES 16
#define WS_NCCL_ID_BYTES 128 /* sizeof(ncclUniqueId) */

/* Version 2 (sizeof(ws_opts)).  Version 1 -- the first 16 bytes, with
 * n_devices then named `reserved` and required to be 0 -- is still accepted
 * (struct_size == 16). */
typedef struct ws_opts {
  uint32_t struct_size;   /* sizeof(ws_opts) */
  uint32_t segment_slots; /* wheel slots per class per segment: power of two in
                             [2^12, 2^18]; default 2^18 (64 KiB of flags) */
  int32_t device;         /* n_devices == 0: CUDA device ordinal, -1 = current device */
  uint32_t n_devices;     /* 0: single-device context on `device`, no NCCL;
                             k in [1, WS_MAX_DEVICES]: device_ids[0..k) with NCCL */
  int32_t device_ids[WS_MAX_DEVICES];
  uint32_t world;         /* processes sharing each job (0 or 1: this one alone) */
  uint32_t rank;          /* this process's rank in [0, world) */
  uint8_t nccl_id[WS_NCCL_ID_BYTES]; /* world > 1: the id ws_nccl_unique_id made on rank 0
                                        (ncclCommInitRank); all zero with world 1:
                                        ncclCommInitAll over device_ids */
} ws_opts;

typedef struct ws_checks {
  uint64_t count;   /* primes in [L, R), 2 and 3 included */
  uint64_t sum;     /* Σ mod 2^64 (0 unless requested / enumerated) */
  uint64_t xor_;    /* ⊕ (0 unless requested / enumerated) */
  uint64_t largest; /* largest prime in range, 0 if none */
} ws_checks;

typedef struct ws_timing {
  double base_ms;    /* device time of base-prime generation in the last call (0 if cached) */
  double sieve_ms;   /* device time of the main sieve kernel(s) of the last call */
  double total_ms;   /* host wall time of the last call */
  uint64_t launches; /* kernels launched by the last call */
  uint64_t segments; /* segments sieved by the main kernel in the last call */
  uint64_t base_primes; /* sieving primes (>= 5) used by the last call */
  uint64_t h2d_bytes;   /* bytes copied host->device by the last call */
  uint64_t d2h_bytes;   /* bytes copied device->host by the last call (host-bound
                           enumeration ships ~1 byte per prime, see ws_enumerate_range) */
} ws_timing;

void ws_opts_default(ws_opts* opts);
const char* ws_status_name(ws_status s);

ws_status ws_ctx_create(const ws_opts* opts, ws_ctx** out);
void ws_ctx_destroy(ws_ctx* ctx);
/* Message of the last failure on this context ("" if none). */
const char* ws_last_error(const ws_ctx* ctx);
/* The cudaStream_t the context launches on (local device 0's; for events /
 * interop). */
void* ws_ctx_stream(ws_ctx* ctx);
ws_status ws_last_timing(const ws_ctx* ctx, ws_timing* out);

/* Count primes in [L, R).  Replaces run() with a CountSink (engine.hpp:83)
 * for L = 0, and the SURVEY §3.3 composition otherwise.
 * per_seg (nullable, host unless WS_OUT_DEVICE): survivor count per segment,
 * at most per_seg_cap written; *n_seg (nullable) = number of segments.
 * Multi-device contexts: each shard writes its own segments' counts (with
 * world > 1 only this process's shards are written); *out is the whole range. */
ws_status ws_count_range(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, ws_checks* out,
                         uint32_t* per_seg, uint64_t per_seg_cap, uint64_t* n_seg);

/* Enumerate the primes of [L, R) in ascending order into out[0 .. *n_out).
 * Replaces run() with a value sink (MemorySink, sink.hpp:55-66).  Σ and ⊕
 * are always computed.  Multi-device contexts count every shard first (the
 * one collective gives each shard's offset and the totals), then each device
 * writes its shard at its offset -- host output in parallel pipelines,
 * device output (any device's memory, UVA) by a device-to-device copy from
 * devices that do not own `out`.  With world > 1, `out` receives this
 * process's shards only (*n_out = their count) while *checks holds the
 * whole range.  If the primes do not fit in cap, nothing is written
 * past cap, *n_out is the full count and WS_CAPACITY is returned.
 * Host output of more than one pipeline chunk (>= 128 segments) crosses PCIe
 * in an 8-bit wire format -- each prime as its bit position in its 128-slot
 * block, one count byte per block and per-segment totals -- and is widened on
 * the host by a pool of threads (WHEELSIEVE_HOST_THREADS, default the CPUs of
 * the process's affinity mask; WHEELSIEVE_HOST_WIRE=0 ships uint64 values
 * instead); order, count and checksums come from the device. */
ws_status ws_enumerate_range(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags, uint64_t* out,
                             uint64_t cap, uint64_t* n_out, ws_checks* checks);

/* Multi-device contexts: every local device i enumerates its ws_partition
 * shard of [L, R) into outs[i] (memory of that device, capacity caps[i];
 * shard 0 starts with 2 and 3 when in range) -- the enumerated arrays stay
 * on their GPU, in shard order the concatenation is the sorted enumeration.
 * counts[i] = primes of local shard i; *checks (nullable) = the whole range
 * after the one allgather.  WS_CAPACITY if a shard exceeds its capacity
 * (nothing is written past it). */
ws_status ws_enumerate_shards(ws_ctx* ctx, uint64_t L, uint64_t R, uint32_t flags,
                              uint64_t* const* outs, const uint64_t* caps, uint64_t* counts,
                              ws_checks* checks);

/* Count primes in each interval [Ls[i], Ls[i] + width), i < n, each sieved
 * independently (BASELINE config 5).  counts/sums/xors (nullable sums/xors)
 * receive per-interval results; Ls and outputs are host arrays unless
 * WS_OUT_DEVICE (single-device contexts only).  Multi-device contexts sieve
 * interval i on shard i mod (world * n_devices); every process receives all
 * n results. */
ws_status ws_count_intervals(ws_ctx* ctx, const uint64_t* Ls, uint64_t n, uint64_t width,
                             uint32_t flags, uint32_t* counts, uint64_t* sums, uint64_t* xors);

/* BasePrimeStore::bootstrap / entries (base_store.cpp:34-42, naive_sieve
 * wheel.cpp:40-54): the wheel primes 5 <= p <= B, ascending, sieved on the
 * device (B <= 2^32).  *n = count; WS_CAPACITY if cap is too small. */
ws_status ws_base_primes(ws_ctx* ctx, uint64_t B, uint32_t flags, uint64_t* out, uint64_t cap,
                         uint64_t* n);

/* SegmentBitmap(start, len) + sieve_segment (segment.hpp:90-168,
 * segment.cpp:93-188): the two flag arrays after sieving, in FlagArray's Bit
 * layout -- bit i of words[i / 64], LSB-first, tail bits zero -- for the 6k+1
 * class (r1_words) and the 6k+5 class (r5_words), ceil(len / 64) words each.
 * As in the reference the value 1 is left set (callers clear it,
 * engine.cpp:244).  Errors: WS_ALIGNMENT (start % 6), WS_DOMAIN (len == 0),
 * WS_OVERFLOW (end beyond the 64-bit range). */
ws_status ws_sieve_segment(ws_ctx* ctx, uint64_t start, uint64_t len, uint32_t flags,
                           uint64_t* r1_words, uint64_t* r5_words);

/* Chunked prime store (ChunkedFileSink, sink.hpp:68-141):
 * enumerate [L, R) on the device -- in value windows of ~2^30 integers, so
 * device and pinned host memory stay bounded (~0.5 GB each) at any range --
 * and stream primes_%05llu.{txt,bin} chunk
 * files of primes_per_file values plus manifest.json (count/min/max/crc32 per
 * file, format, total_count, frontier = R), byte-identical to the reference
 * CLI's `sieve --out` for [0, limit + 1).  Binary chunks' CRC-32s are
 * computed on the device.  WS_DOMAIN if primes_per_file == 0, WS_IO on
 * filesystem errors. */
#define WS_STORE_TEXT 0u
#define WS_STORE_BINARY 1u
ws_status ws_store_range(ws_ctx* ctx, uint64_t L, uint64_t R, const char* dir, uint32_t format,
                         uint64_t primes_per_file, uint64_t* n_out);
/* Streaming chunk writer (ChunkedFileSink, sink.hpp:68-141, sink.cpp:185-304):
 * chunk files are opened on demand and closed at primes_per_file values; the
 * manifest is rewritten (write-then-rename) at every rollover and on flush,
 * so what it lists is durable.  Memory is bounded by one batch.  Values
 * must ascend across appends (the caller's sink checks it).  The manifest
 * frontier is one past the largest value unless set.  ws_store_range uses
 * the same writer for device-enumerated windows of bounded size (binary
 * CRCs computed on the device). */
typedef struct ws_store ws_store;
ws_status ws_store_open(const char* dir, uint32_t format, uint64_t primes_per_file,
                        ws_store** out);
ws_status ws_store_append(ws_store* st, const uint64_t* values, uint64_t n);
ws_status ws_store_set_frontier(ws_store* st, uint64_t frontier);
ws_status ws_store_flush(ws_store* st);
uint64_t ws_store_durable_count(const ws_store* st);
const char* ws_store_last_error(const ws_store* st);
/* flushes (best effort: the status reports a failure) and frees */
ws_status ws_store_close(ws_store* st);

/* read_back (sink.cpp:306-321): primes in [lo, hi) of a store, every touched
 * file verified against its crc32 and count; WS_BEYOND_FRONTIER if hi exceeds
 * the recorded frontier, WS_CHECKSUM_MISMATCH / WS_BAD_MANIFEST / WS_IO. */
ws_status ws_read_back(const char* dir, uint64_t lo, uint64_t hi, uint64_t* out, uint64_t cap,
                       uint64_t* n_out);
/* verify_store (sink.cpp:323-342): every file vs the manifest, global order. */
ws_status ws_verify_store(const char* dir);

/* Count each range [Ls[i], Rs[i]), i < n, independently (the per-worker-tile
 * counts of run(), engine.cpp:233-288): out[i] receives count, Σ/⊕ (with
 * WS_WANT_CHECKS) and the largest prime of range i, 2 and 3 included when in
 * range.  Empty ranges (R <= L) give zeros.  Host arrays.  Multi-device
 * contexts split the batch into contiguous blocks of ranges per shard. */
ws_status ws_count_ranges(ws_ctx* ctx, const uint64_t* Ls, const uint64_t* Rs, uint64_t n,
                          uint32_t flags, ws_checks* out);

/* ---- multi-device contexts ---------------------------------------------- */
/* Fills id (WS_NCCL_ID_BYTES) with a fresh ncclUniqueId, on rank 0 of a
 * multi-process job; the caller broadcasts it to the other ranks' ws_opts. */
ws_status ws_nccl_unique_id(uint8_t* id);
/* Local devices of the context (1 for single-device contexts). */
uint32_t ws_ctx_num_devices(const ws_ctx* ctx);
/* Shards each job is split into (world * local devices; 1 without NCCL). */
uint32_t ws_ctx_num_shards(const ws_ctx* ctx);
/* CUDA ordinal and launch stream of local device i. */
int32_t ws_ctx_device(const ws_ctx* ctx, uint32_t i);
void* ws_ctx_device_stream(ws_ctx* ctx, uint32_t i);
/* Timing of the last call on local device i alone (ws_last_timing reports
 * the maximum device times and summed counters over the devices). */
ws_status ws_device_timing(const ws_ctx* ctx, uint32_t i, ws_timing* out);
/* NCCL communicator of local device i: ranks in the communicator and this
 * device's rank (WS_BAD_CONFIG for contexts without NCCL). */
ws_status ws_ctx_comm_info(const ws_ctx* ctx, uint32_t i, int32_t* nranks, int32_t* comm_rank);
/* The fold applied to the gathered per-shard records: count and Σ add mod
 * 2^64, ⊕ folds, largest is the maximum.  Pure function: combining the
 * ws_checks of ws_partition's shards of [L, R) (each counted alone) gives
 * exactly the ws_checks of [L, R). */
ws_status ws_combine_checks(const ws_checks* records, uint64_t n, ws_checks* out);

/* Upper bound on the number of primes in [L, R) (capacity helper). */
uint64_t ws_prime_count_bound(uint64_t L, uint64_t R);

/* Multi-GPU partitioner: rank's contiguous share [*lo, *hi) of [L, R), with
 * interior boundaries on multiples of 6 * segment_slots values counted from
 * floor(L / 6) * 6 (so every rank's segments coincide with the single-GPU
 * segmentation); rank r gets segments [floor(r n / world), floor((r+1) n / world))
 * of the n segments, clipped to [L, R).  Pure function. */
ws_status ws_partition(uint64_t L, uint64_t R, uint32_t segment_slots, uint32_t rank,
                       uint32_t world, uint64_t* lo, uint64_t* hi);

/* Paper Table 1 / wheel.cpp:96-106: wheel indices of the first multiples of
 * p at or beyond segment_start in the 6k+1 and 6k+5 classes. */
ws_status ws_start_offsets(uint64_t p, uint64_t segment_start, uint64_t* id1, uint64_t* id5);

/* floor(sqrt(n)), exact (wheel.cpp:25-33). */
uint64_t ws_isqrt(uint64_t n);

/* Library version string. */
const char* ws_version(void);

#ifdef __cplusplus
}
#endif

#endif /* WHEELSIEVE_GPU_H_ */
