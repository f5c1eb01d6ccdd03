// Host-side internals of libwheelsieve_cuda.so shared by ws_abi.cu (the C ABI)
// and ws_store.cu (the chunked store): per-device engine state (DevCtx) and
// the multi-device context behind the opaque ws_ctx handle.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "wheelsieve/gpu.h"
#include "ws_internal.h"
#include "ws_wire.h"

namespace wsh {

inline constexpr uint64_t kMaxWheelIndex = (UINT64_MAX - 5) / 6;       // wheel.hpp:33
inline constexpr uint64_t kMaxSegmentEnd = 6 * (kMaxWheelIndex + 1);   // wheel.hpp:37

inline uint64_t isqrt_u64(uint64_t n) {  // wheel.cpp:25-33 semantics (exact)
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

inline void ck(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    throw Fail{WS_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e)};
  if (e != cudaSuccess) throw Fail{WS_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Bumped by every (re)allocation or release of a device / pinned buffer: a
// captured CUDA graph (CallGraph) holds raw pointers and is valid only while
// this is unchanged.
inline std::atomic<uint64_t> g_alloc_gen{0};

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  void reserve(size_t n, const char* what) {
    if (n <= cap) return;
    release();
    ++g_alloc_gen;
    ck(cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T)), what);
    cap = n;
  }
  void release() {
    if (ptr) {
      cudaFree(ptr);
      ++g_alloc_gen;
    }
    ptr = nullptr;
    cap = 0;
  }
  // grow to n elements keeping the first `keep` (stream-ordered copy)
  void grow(size_t n, size_t keep, cudaStream_t st, const char* what) {
    if (n <= cap) return;
    ++g_alloc_gen;
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
    ++g_alloc_gen;
    ck(cudaMallocHost(&ptr, std::max<size_t>(n, 64)), what);
    bytes = n;
    return ptr;
  }
  void release() {
    if (ptr) {
      cudaFreeHost(ptr);
      ++g_alloc_gen;
    }
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

inline uint64_t small_primes_upto(uint64_t B) {  // |{5,7,...,47} ∩ [5, B]| (the stamped primes)
  static const uint32_t sp[] = {5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47};
  uint64_t c = 0;
  for (uint32_t q : sp) c += q <= B;
  return c;
}

// Everything a small count call's captured device work depends on.
struct CallKey {
  uint64_t lo = 0, hi = 0;
  int mode = -1;
  const void* dps = nullptr;  // device per-segment counts (nullable)
  const void* dst = nullptr;  // their copy destination (nullable)
  int kind = 0;               // its cudaMemcpyKind
  uint32_t S = 0;
  bool fresh = false;         // the call rebuilds the base table
  uint64_t base_B = 0;        // else: the resident table it reads
  uint32_t nprimes = 0;
  const void* nprimes_dev = nullptr;
  uint64_t gen = 0;           // g_alloc_gen at capture
  bool operator==(const CallKey& o) const {
    return lo == o.lo && hi == o.hi && mode == o.mode && dps == o.dps && dst == o.dst &&
           kind == o.kind && S == o.S && fresh == o.fresh && base_B == o.base_B &&
           nprimes == o.nprimes && nprimes_dev == o.nprimes_dev && gen == o.gen;
  }
};

// CUDA-graph replay of a repeated small count call (ws_abi.cu, graph_or_run):
// the second identical call is captured, later ones are one cudaGraphLaunch.
struct CallGraph {
  bool seen = false, valid = false;
  CallKey key;
  cudaGraphExec_t exec = nullptr;
  ws_timing timing{};  // the captured call's counters (launches, segments, bytes)
  bool base_valid = false, base_built = false;
  uint64_t base_B = 0;
  uint32_t nprimes = 0;
  const uint32_t* nprimes_dev = nullptr;
};

struct DevCtx {
  int device = 0;
  uint32_t shard = 0;   // this device's shard of a multi-device job (global NCCL rank)
  unsigned host_threads = 0;  // wire expander threads (0: the process's CPUs)
  cudaStream_t stream = nullptr;
  uint32_t S = 1u << 18;
  int sms = 148;
  int bps[wsk::kNumModes] = {2, 2, 2, 2};  // resident blocks per SM per mode
  uint32_t wide = 3;            // > 1: long count launches sieve this many segments per unit (WHEELSIEVE_WIDE)
  uint32_t wide_bucket = 3;     // ... in bucket windows (WHEELSIEVE_WIDE_BUCKET; C4 -4.8%, C5 -7.4%)
  uint32_t wide_pmin_ratio = 6; // ... where primes below this many S stay in the kernel (WHEELSIEVE_WIDE_PMIN)
  uint32_t wide_multi = 3;      // ... in launches over several jobs without buckets (WHEELSIEVE_WIDE_MULTI);
                                // several jobs: only when they average at least 6 segments
  uint32_t trans_min = 768;     // wide units: shortest partial superblock marked transposed
                                // (WHEELSIEVE_TRANS_MIN; 192..768 measured within 2%, 768 best)
  uint32_t seg_trans = 1;       // per-segment count kernels: transposed warp-cooperative marking (WHEELSIEVE_SEG_TRANS)
  uint32_t seg_trans_min = 768; // ... its shortest transposed partial superblock
  uint32_t wide_double = 1;     // wide units: straight-line marking for primes of at least half a
                                // unit (WHEELSIEVE_WIDE_DOUBLE; c3s -1.9%; a third: no further gain)
  uint32_t wide_skip5 = 49152;  // wide units: skip5_max (3x the hits per visit; WHEELSIEVE_WIDE_SKIP5)
  uint32_t wide_n_wc = 0;       // wide units: warp-cooperative primes (0: the context's n_wc)
  uint32_t wide_min_units = 2;  // ... when every SM gets at least this many units (pi(3e9): -11% at 4.3; C1 at 1.4: no gain)
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
  uint32_t n_below_S = 0;  // table primes (>= 53) below bucket_pmin: in-kernel; the rest bucketed
  uint32_t bucket_pmin = 0;
  uint32_t n_S = 0;        // table primes (>= 53) below S
  uint32_t n_wc = 161;     // table primes below the warp-cooperative limit (1024)
  // bytes of bucket lists per window buffer (two buffers): 8 GiB puts C4 in
  // 7 windows instead of 41, with fewer fill / sieve tails (C4 56.8 -> 53.5 ms;
  // 16 GiB is no faster: 32-bit entry indices cap a window near 2^32 entries)
  size_t bucket_budget = 8ull << 30;
  uint32_t cap_override = 0;           // test knob (WHEELSIEVE_BUCKET_CAP)
  uint32_t piece_override = 0;         // tuning knob (WHEELSIEVE_FILL_PIECE)
  bool fill_huge = true;               // carried-offset fill for p >= run length (WHEELSIEVE_FILL_HUGE)
  uint32_t huge_step = 1;              // runs per histogram step there (WHEELSIEVE_HUGE_STEP)
  uint32_t huge_loop = 0;              // WHEELSIEVE_HUGE_LOOP=1: the hit-loop kernel at step 1
  // WHEELSIEVE_FILL_UNROLL=1: fill pass 2 runs both classes, two hits each, per
  // step (independent cursor atomics); measured slower (C5 23.6 vs 23.3 ms,
  // C4 51.7 vs 50.9 ms): the predicated lanes cost more than the overlap wins
  uint32_t w_unroll = 0;
  uint32_t stage_cap = 256;            // WHEELSIEVE_STAGE_CAP: staged fill queue entries (0: two-pass fills)
  uint32_t huge_from = 0;              // its lower bound in units of S (0: the run length)
  uint64_t huge_thr = 0;               // the run length in slots the count below is for
  uint32_t n_below_huge = 0;           // table primes (>= 53) below huge_thr
  uint32_t bucket_min_ratio = 8;       // buckets iff largest base prime >= ratio * S
  uint32_t bucket_ctas_per_sm = 0;     // tuning knob (WHEELSIEVE_BUCKET_CTAS)
  uint32_t ctas_per_sm = 0;            // tuning knob, all launches (WHEELSIEVE_CTAS_PER_SM)
  // predicated single-hit atomics (WHEELSIEVE_SINGLE_PRED=1): 17% fewer shared
  // wavefronts at C3 but no faster (204.4 ms either way; C4 +0.2 ms), so off
  uint32_t single_pred = 0;
  uint32_t mid_bitaddr = 1;            // WHEELSIEVE_MID_BITADDR
  uint32_t miss_lane = 1;              // WHEELSIEVE_MISS_LANE
  uint32_t skip5_max = 16384;          // WHEELSIEVE_SKIP5: mid primes below it skip multiples of 5
  bool graphs = true;                  // WHEELSIEVE_GRAPHS=0: no graph replay of small calls
  bool capturing = false;              // the stream is being captured (timing events external)
  CallGraph cg;

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
  DevBuf<uint32_t> units;  // wide launches over windows / several jobs: unit table
  DevBuf<wsk::Job> jobs;
  DevBuf<wsk::JobAcc> acc;
  DevBuf<wsk::JobAcc> gather;   // multi-device: every shard's records after the allgather
  DevBuf<wsk::JobAcc> gsend;    // multi-device: this shard's padded records
  PinnedBuf pin_gather;
  DevBuf<unsigned long long> ticket;
  DevBuf<uint32_t> per_seg;
  DevBuf<unsigned long long> status;
  DevBuf<unsigned long long> vals;  // enumeration scratch (base primes / host-bound output)
  DevBuf<uint32_t> l0_p;
  DevBuf<unsigned long long> l0_m;
  DevBuf<double> l0_inv;
  DevBuf<uint32_t> l0_n;
  std::vector<wsk::Job> h_jobs;

  ~DevCtx() {
    cudaSetDevice(device);
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
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
    gather.release();
    gsend.release();
    pin_gather.release();
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};


}  // namespace wsh

namespace wsh {

// NCCL, loaded on first use (dlopen of libnccl.so.2 -- or the copy already in
// the process, e.g. PyTorch's): single-device users never pay for mapping the
// ~400 MB library, and a multi-device context fails with WS_NCCL, not the
// whole library with a load error, where NCCL is missing.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int*);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
  const char* (*GetErrorString)(ncclResult_t);
};
const NcclApi* nccl_api();  // nullptr when libnccl.so.2 cannot be loaded

// One host thread per local device of a multi-device context.  run(fn)
// executes fn(i) on worker i for every device concurrently and returns when
// all have finished; each worker keeps its device current.
class DevWorkers {
 public:
  explicit DevWorkers(const std::vector<int>& devices) : n_(devices.size()) {
    for (size_t i = 0; i < n_; ++i)
      threads_.emplace_back([this, i, dev = devices[i]] { loop(i, dev); });
  }
  ~DevWorkers() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  void run(const std::function<void(size_t)>& fn) {
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &fn;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(size_t i, int dev) {
    cudaSetDevice(dev);
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(size_t)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
        job = job_;
      }
      (*job)(i);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  size_t n_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t)>* job_ = nullptr;
  uint64_t gen_ = 0;
  size_t pending_ = 0;
  bool quit_ = false;
};

}  // namespace wsh

// The opaque handle of gpu.h.  A single-device context (ws_opts.n_devices ==
// 0) is exactly one DevCtx driven from the caller's thread.  A multi-device
// context owns one DevCtx per local device, a worker thread per device and
// one NCCL communicator per device; the job is split into world * n_local
// shards (shard = NCCL rank = rank * n_local + i), each device sieves its
// shard and the per-shard 32-byte records {count, sum, xor, largest} are
// combined after one ncclAllGather.
struct ws_ctx {
  std::vector<wsh::DevCtx*> devs;
  bool nccl = false;
  // test mode (WHEELSIEVE_VIRTUAL_SHARDS=1): several shards on one GPU, the
  // shard records gathered on the host instead of by NCCL (which refuses two
  // ranks on one device); everything else is the multi-device path
  bool virt = false;
  uint32_t world = 1, rank = 0;  // processes sharing a job, and this one's rank
  uint32_t nshards = 1;          // world * devs.size()
  uint32_t S = 1u << 18;         // segment slots (DevCtx::S is swapped during base builds,
                                 // so other threads read this immutable copy)
  std::vector<ncclComm_t> comms;
  wsh::DevWorkers* workers = nullptr;
  std::string err;
  ws_timing timing{};
  ~ws_ctx() {
    delete workers;
    for (ncclComm_t c : comms)
      if (c && wsh::nccl_api()) wsh::nccl_api()->CommDestroy(c);
    for (wsh::DevCtx* d : devs) delete d;
  }
  uint32_t shard_of(size_t i) const { return rank * static_cast<uint32_t>(devs.size()) + static_cast<uint32_t>(i); }
};
