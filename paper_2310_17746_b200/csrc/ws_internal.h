// Internal interface between the C-ABI host layer (ws_abi.cu) and the
// sm_100a kernels (ws_sieve.cu).  Plain structs, no torch types.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wsk {

constexpr int kThreads = 512;            // threads per sieve block
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kFirstTablePrime = 53; // primes 5..47 are stamped from pattern tables
constexpr uint32_t kTinyMax = 1u << 18;  // small_base_kernel bound (at most 33 blocks)

// One half-open value range [L, R) sieved as nseg segments of S wheel slots
// per residue class starting at wheel index K0 = floor(L / 6)
// (SURVEY §3.3 geometry: segment i starts at 6*K0 + 6*S*i).
struct Job {
  uint64_t L, R;
  uint64_t K0;        // first wheel index
  uint64_t nslots;    // wheel slots per class over the whole range
  uint64_t seg_begin; // index of the job's first segment in the launch
  uint64_t nseg;
};

// Per-job results, combined with 64-bit atomics (sum wraps mod 2^64).
struct JobAcc {
  unsigned long long count, sum, xr, largest;
};

// kEnumWire: ordered enumeration into the 8-bit host wire format -- each
// prime as its bit position e in the interleaved survivor masks of its
// 128-slot (4-word) block (value = 6 * block_first_slot + 3e + 1 + (e & 1)),
// one survivor-count byte per block (a block spans 768 integers, far fewer
// than 255 primes) and the per-segment totals; the host widens it
// (ws_wire.cpp).
enum Mode : int { kCount = 0, kCountChecks = 1, kEnumerate = 2, kEnumWire = 3 };
constexpr int kNumModes = 4;
constexpr uint32_t kWideMax = 3;  // segments per unit of the wide count kernel (192 KiB)
constexpr uint32_t kWireBlockSlots = 128;

// Large-prime buckets: per window of segments, the hits of every prime
// p >= S (at most one per class per segment) are scattered into per-segment
// lists of uint32 entries (slot | class * S: the bit index into the CTA's
// contiguous [6k+1 | 6k+5] bitmap) by bucket_fill_kernel and
// applied by the sieve kernel.  A list that overflows its capacity is
// detected by the sieve kernel, which then processes that segment's large
// primes directly (correct, just slower).
struct Run {             // a maximal run of window segments of one job
  uint64_t k_lo, k_hi;   // wheel-slot range [k_lo, k_hi) of the run
  uint32_t seg0;         // window-local index of the run's first segment
  uint32_t nseg;
};

struct SieveParams {
  const uint32_t* small_tab;  // small-prime pattern tables (built once per context)
  const Job* jobs;                   // njobs > 1 (device copy)
  Job job0;                          // njobs == 1: the job itself (no upload)
  uint32_t njobs;
  uint32_t* tabn_out;                // nullable: CTA 0 stores the exact table size
  uint64_t nseg_total;   // segments of all jobs
  uint64_t s_begin;      // this launch sieves segments [s_begin, s_begin + s_count)
  uint64_t s_count;
  uint32_t S;                        // wheel slots per class per segment (power of two)
  const uint32_t* prime_p;           // sieving primes >= 53 (kFirstTablePrime), ascending
  const unsigned long long* prime_m; // floor((2^64-1)/p), Barrett reciprocal (ks >= 2^53)
  const double* prime_inv;           // fl(1/p), FP64 quotient estimate (ks < 2^53)
  uint32_t nprimes;                  // host-side upper bound on the table size
  const uint32_t* nprimes_dev;       // nullable: exact table size, written on device
  uint32_t n_wc;                     // primes [0, n_wc) use the warp-cooperative loop
  uint32_t n_S;                      // primes [n_wc, n_S): one thread per prime, hit loop
                                     // (p < S; wide units: p < half a unit)
  uint32_t n_dbl;                    // wide: [n_S, n_dbl) straight-line, <= 2 hits per class
                                     // (half a unit <= p < a unit); 0 otherwise
  uint32_t n_mid;                    // [max(n_S, n_dbl), n_mid): one thread per prime, <= 1 hit
                                     // per class; [n_mid, nprimes) from buckets (directly if
                                     // bucket == null or a list overflowed)
  const uint32_t* bucket;            // window lists: bucket[(s - s_begin) * bcap + i]
  uint32_t* bcount;                  // entries per window segment (reset after use)
  uint32_t bcap;
  unsigned long long* ticket;        // {segment counter, exits}: zero at launch; the last
                                     // CTA out resets both for the next launch
  JobAcc* acc;                       // njobs accumulators (zeroed per launch)
  uint32_t* per_seg;                 // nullable, nseg_total counts
  unsigned long long* status;        // enumeration look-back words (zeroed)
  unsigned long long* out;           // enumeration output (after 2 and 3)
  unsigned long long out_cap;
  uint8_t* out8;                     // kEnumWire: entries (same positions as `out`)
  uint8_t* blk8;                     // kEnumWire: survivors per block, segment s at s * S / 128
  uint32_t single_pred;              // single-hit primes: predicated atomics (else OR 0 on a miss)
  uint32_t mid_bitaddr;              // mid-prime loop on shared bit addresses
  uint32_t miss_lane;                // single-hit misses OR 0 into word `lane` (else a word from h)
  uint32_t skip5_max;                // mid primes below it skip their hits on multiples of 5
  uint32_t wide;                     // > 1: sieve_wide_kernel, this many segments per unit
  uint32_t seg_trans;                // per-segment count kernels: transposed warp-cooperative marking
  uint32_t trans_min;                // shortest partial superblock marked transposed (mark_transposed)
  const uint32_t* units;             // wide launches over windows or several jobs: per unit,
  uint32_t nunits;                   //   first window-local segment | segment count << 28
  uint32_t* words1;                  // nullable (count modes): survivor flag words of
  uint32_t* words5;                  // each class, segment s at word s * S / 32
};

size_t sieve_smem_bytes(uint32_t S, int mode);
uint32_t small_table_words();
void build_small_tables(uint32_t* out);  // host
// blocks_per_sm[mode] for the kNumModes modes
cudaError_t sieve_configure(int* blocks_per_sm);
cudaError_t launch_sieve(int mode, const SieveParams& p, int grid, cudaStream_t st);
cudaError_t launch_acc_to_host(const JobAcc* acc, JobAcc* host_mapped, uint32_t n,
                               cudaStream_t st);
// n words to mapped pinned host memory with plain stores (see acc_to_host_kernel)
cudaError_t launch_u32_to_host(const uint32_t* src, uint32_t* host_mapped, uint32_t n,
                               cudaStream_t st);

struct FillParams {
  const Run* runs;
  uint32_t nruns;
  const uint32_t* prime_p;
  const unsigned long long* prime_m;
  const double* prime_inv;
  const uint32_t* nprimes_dev;  // exact table size (p_end is an upper bound)
  uint32_t p_begin, p_end;  // large primes [p_begin, p_end) of the table
  uint32_t log2S;
  uint32_t* bucket;
  uint32_t* bcount;
  uint32_t bcap;
  uint32_t max_run_segs;    // histogram size (dynamic shared memory)
  uint32_t group_runs;      // bucket_fill_huge_kernel: consecutive runs per block row
  uint32_t huge_step;       // ... and runs per histogram step (max_run_segs covers them)
  uint32_t huge_loop;       // 1: the hit-loop kernel even for one run per step (A/B knob)
  uint32_t w_unroll;        // bucket_fill_kernel pass 2: both classes, 2 hits each per step
  uint32_t stage_cap;       // > 0: staged fills, per-segment shared-memory queues of this
                            // many entries flushed as contiguous chunks (0: two-pass fills)
};
constexpr int kFillThreads = 256;
constexpr int kFillPrimesPerThread = 16;
constexpr int kFillPrimesPerBlock = kFillThreads * kFillPrimesPerThread;
constexpr uint32_t kMaxWindow = 16384;  // segments per window (run spans stay below 2^32 slots)
cudaError_t launch_bucket_fill(const FillParams& f, cudaStream_t st);
// Primes of at least the run length (at most one hit per class per run) over
// runs that are consecutive pieces of one job: first hits computed once per
// group of runs and carried from run to run in shared memory.
cudaError_t launch_bucket_fill_huge(const FillParams& f, cudaStream_t st);

// Appends the enumerated primes vals[0, min(*n_dev, cap)) to a table of
// *old_n_dev entries and sets *out_n (device-side BasePrimeStore::extend).
cudaError_t launch_append_table(const unsigned long long* vals, const unsigned long long* n_dev,
                                uint64_t cap, uint32_t* out_p, unsigned long long* out_m,
                                double* out_inv, uint32_t* out_n, const uint32_t* old_n_dev,
                                cudaStream_t st);

// Small base tables: all primes in [53, n] (n <= kTinyMax), ascending, with
// their Barrett constants; scratch holds >= 64 words (zeroed once), epoch is
// nonzero and differs from the previous launch's on the same scratch.
cudaError_t launch_small_base(uint32_t n, uint32_t* out_p, unsigned long long* out_m,
                              double* out_inv, uint32_t* out_count, unsigned long long* scratch,
                              uint32_t epoch, cudaStream_t st);
// Table preparation: vals[i] (uint64 primes, ascending) -> p / Barrett m for
// i in [skip, n).
// n_dev: number of values (device); out_n = n - skip (device).  cap bounds n.
cudaError_t launch_prepare_table(const unsigned long long* vals, uint64_t skip,
                                 const unsigned long long* n_dev, uint64_t cap, uint32_t* out_p,
                                 unsigned long long* out_m, double* out_inv, uint32_t* out_n,
                                 cudaStream_t st);

}  // namespace wsk
