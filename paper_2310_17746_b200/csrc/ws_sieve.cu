// sm_100a kernels of the B200 segmented mod-6 wheel sieve.
//
// Reference hot path (CPU, scalar): sieve_segment (segment.cpp:164-188) ->
// FlagArray::clear_stride (segment.cpp:49-69) per base prime and residue
// class, then count_surviving / for_each_surviving (segment.cpp:141-162,
// segment.hpp:123-146).  Here one thread block owns one segment at a time
// (persistent CTAs, 3 per SM in every mode, segments claimed from a ticket):
//
//   shared memory:  two uint32 bitmaps (6k+1 and 6k+5 classes), S/32 words each,
//                   bit k of class c <-> value 6*(ks + k) + c (LSB-first, the
//                   reference's bit layout, segment.hpp:46-50).  Flags are
//                   COMPOSITE bits (the complement of FlagArray), so crossing
//                   off is one ATOMS.OR.  No bank swizzle: simulated and
//                   measured conflicts of the strided loop are lower with the
//                   natural layout (2.4-way vs 2.8-way for p in [53, 1024)).
//   stamp:          primes 5..47 are never looped: their combined periodic
//                   patterns (5*7*11*13, 17*19*23, 29*31, 37*41, 43*47) are
//                   read through L1 and each word is five funnel-shifted table
//                   reads ANDed with the [L, R) trim mask.
//   medium primes:  53 <= p < wc_limit: warp-cooperative strided clear (lane l
//                   takes hits rel + l*p, rel + (l+32)*p, ...).
//   other primes:   one thread per prime (p < S: hit loop; p >= S: at most one
//                   hit per class), p and 1/p loaded one iteration ahead;
//                   p >= 2S from bucket lists when the base table is large.
//   offsets:        the first hit of p in each class is recomputed per
//                   (prime, segment) from ks mod p by one FP64 FMA (64-bit
//                   Barrett above 2^53) -- no divide, no carried state, so
//                   segments can be claimed dynamically (ticket counter),
//                   which the ordered enumeration look-back relies on.  The
//                   reference's activation rule (first hit at p*p,
//                   segment.cpp:178-183) is applied when p*p lies ahead.
//   finish:         __popc + warp/block reductions (count), optional
//                   sum/xor checksums, or ordered enumeration: per-warp
//                   prefix sums + a decoupled look-back across segments for
//                   the global output offset, then coalesced uint64 stores
//                   (or the 8-bit host wire format, ws_wire.cpp).
//
// sieve_wide_kernel (long count launches): one 1024-thread CTA per SM owns
// three consecutive segments as one unit -- per-(prime, unit) work is paid
// once per three segments, count and next-unit stamping are one pass (two
// barriers per unit), and the warp-cooperative primes are marked in
// conflict-free transposed superblocks (mark_transposed).
//
// Other kernels here: bucket_fill_kernel (large-prime hit lists per window,
// one launch per window) and bucket_fill_huge_kernel (primes of at least the
// run length, first hits carried across runs); small_base_kernel (base tables
// up to 2^18 in one launch); prepare/append_table_kernel (table entries from
// enumerated primes); acc/u32_to_host_kernel (results to mapped host memory).
#include <cstdint>
#include <type_traits>

#include "ws_internal.h"

namespace wsk {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Wheel helpers.  For a prime p coprime to 6, p = 6R + r, its multiples in
// class c sit at wheel indices k == t_c (mod p):
//   r == 1:  t1 = R,       t5 = 5R
//   r == 5:  t1 = 5R + 4,  t5 = R
// (the k-residue form of paper Table 1 / kStartIncrements, wheel.cpp:77-82).
__host__ __device__ constexpr uint32_t target1(uint32_t p) {
  return p % 6 == 1 ? p / 6 : 5 * (p / 6) + 4;
}
__host__ __device__ constexpr uint32_t target5(uint32_t p) {
  return p % 6 == 1 ? 5 * (p / 6) : p / 6;
}
// Both targets in the per-(prime, segment) loops: p == 1 (mod 6) iff
// p * 3^-1 (mod 2^32) >= 3^-1 (for p == 1 (mod 3) the product is k + 3^-1
// without wrapping), and t1 + t5 == p - 1 (both are the residues of -1/6 and
// -5/6 mod p) -- 7 instructions instead of 8 with the branchy select pair.
__device__ __forceinline__ void targets(uint32_t p, uint32_t& t1, uint32_t& t5) {
  const uint32_t q = p / 6u;
  const bool one = p * 0xAAAAAAABu >= 0xAAAAAAABu;
  t1 = one ? q : 5u * q + 4u;
  t5 = p - 1u - t1;
}

// x mod p for any 64-bit x, m = floor((2^64 - 1) / p).  q underestimates
// x / p by at most 2, so two conditional subtractions finish it.
__device__ __forceinline__ uint32_t mod_barrett(uint64_t x, uint32_t p, uint64_t m) {
  const uint64_t q = __umul64hi(x, m);
  uint64_t r = x - q * p;
  if (r >= p) r -= p;
  if (r >= p) r -= p;
  return static_cast<uint32_t>(r);
}

// ks mod p for every sieving prime of a segment.  For ks < 2^53 (values
// below 5.4e16, every BASELINE config) one FP64 FMA gives the quotient:
// fma(ks, 1/p, 1.5*2^52) holds round(ks/p) in its low mantissa word; with
// |ks * fl(1/p) - ks/p| < 1/37 the estimate is q or q+1, so one conditional
// add of p fixes the 32-bit remainder.  Larger ks use the 64-bit Barrett.
struct ModCtx {
  uint64_t ks;
  double ksd;
  uint32_t kslo;
  bool fast;
};

__device__ __forceinline__ ModCtx mod_ctx(uint64_t ks) {
  ModCtx c;
  c.ks = ks;
  c.fast = ks < (1ull << 53);
  c.ksd = static_cast<double>(ks);
  c.kslo = static_cast<uint32_t>(ks);
  return c;
}


// 32-bit shared-window address of a shared-memory pointer
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void atom_or_shared(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// 1 << (pos & 31) as one BMSK (no constant register, no separate mask of pos)
__device__ __forceinline__ uint32_t bit_of(uint32_t pos) {
  uint32_t m;
  asm("bmsk.wrap.b32 %0, %1, 1;" : "=r"(m) : "r"(pos));
  return m;
}

// bits [a, b) of a 32-bit word, a and b clamped to [0, 32]
__device__ __forceinline__ uint32_t range_mask(int64_t a, int64_t b) {
  a = a < 0 ? 0 : (a > 32 ? 32 : a);
  b = b < 0 ? 0 : (b > 32 ? 32 : b);
  if (b <= a) return 0u;
  const uint32_t hi = b == 32 ? kFull : ((1u << b) - 1u);
  const uint32_t lo = a == 32 ? kFull : ((1u << a) - 1u);
  return hi & ~lo;
}

// ---------------------------------------------------------------------------
// Small-prime pattern tables.  Group g has modulus Q_g; table word i of class
// c holds bits for wheel indices 32i .. 32i+31 (mod Q_g), bit set when the
// index is NOT a multiple-position of any prime of the group.  Stored
// wrap-extended so a funnel shift at any offset < Q_g reads 32 valid bits.
// groups: 5*7*11*13 = 5005, 17*19*23 = 7429, 29*31 = 899, 37*41 = 1517,
// 43*47 = 2021 -- every prime below kFirstTablePrime (53) is stamped
constexpr int kGroups = 5;
__host__ __device__ constexpr uint32_t group_prime(int g, int j) {
  return g == 0 ? (j == 0 ? 5 : j == 1 ? 7 : j == 2 ? 11 : 13)
       : g == 1 ? (j == 0 ? 17 : j == 1 ? 19 : 23)
       : g == 2 ? (j == 0 ? 29 : 31)
       : g == 3 ? (j == 0 ? 37 : 41)
                : (j == 0 ? 43 : 47);
}
__host__ __device__ constexpr int group_size(int g) { return g == 0 ? 4 : g == 1 ? 3 : 2; }
__host__ __device__ constexpr uint32_t group_mod(int g) {
  return g == 0 ? 5005 : g == 1 ? 7429 : g == 2 ? 899 : g == 3 ? 1517 : 2021;
}
constexpr uint32_t tab_words(uint32_t Q) { return (Q + 31) / 32 + 2; }
__host__ __device__ constexpr uint32_t tab_off(int g) {
  return g == 0 ? 0 : tab_off(g - 1) + tab_words(group_mod(g - 1));
}
constexpr uint32_t kTabPerClass = tab_off(kGroups);
constexpr uint32_t kTabWords = 2 * kTabPerClass;

// One table word (class cls, group g, word i): bit b set when index
// 32 i + b is not a multiple-position of any prime of the group.
__host__ __device__ uint32_t table_word(uint32_t idx) {
  const uint32_t cls = idx / kTabPerClass;  // 0 -> 6k+1, 1 -> 6k+5
  const uint32_t rem = idx % kTabPerClass;
  int g = 0;
  while (g + 1 < kGroups && rem >= tab_off(g + 1)) ++g;
  const uint32_t i = rem - tab_off(g);
  uint32_t word = 0;
  for (uint32_t b = 0; b < 32; ++b) {
    const uint32_t pos = 32 * i + b;
    bool keep = true;
    for (int j = 0; j < group_size(g); ++j) {
      const uint32_t q = group_prime(g, j);
      const uint32_t t = cls ? target5(q) : target1(q);
      keep = keep && (pos % q != t);
    }
    word |= static_cast<uint32_t>(keep) << b;
  }
  return word;
}

// The device copy stores each table word together with its successor (one
// 64-bit load per read); 32 bits at any bit offset < Q are one funnel shift.
__device__ __forceinline__ uint32_t tab_read(const uint2* t, uint32_t off) {
  const uint2 v = __ldg(t + (off >> 5));
  return __funnelshift_r(v.x, v.y, off & 31u);
}

// ---------------------------------------------------------------------------
struct SegInfo {
  uint64_t s;      // global segment index (>= nseg_total: done)
  uint32_t job;
  uint64_t ks;     // absolute wheel index of slot 0
  uint32_t len;    // slots in this segment
  uint32_t lo1, hi1, lo5, hi5;  // valid slot bounds per class
  uint32_t nwords; // words per class actually used (ceil(len / 32), rounded to 32)
  uint32_t t_lo;   // primes p <= t_lo: p*p below the segment (no activation)
  uint32_t t_hi;   // primes p > t_hi: p*p beyond the segment (inactive)
};

// floor(sqrt(n)) for 64-bit n, saturated to 2^32 - 1
__device__ __forceinline__ uint32_t isqrt64(uint64_t n) {
  uint64_t r = static_cast<uint64_t>(sqrt(static_cast<double>(n)));
  if (r > 0xFFFFFFFFull) r = 0xFFFFFFFFull;
  while (r * r > n) --r;
  while (r < 0xFFFFFFFFull && (r + 1) * (r + 1) <= n) ++r;
  return static_cast<uint32_t>(r);
}

__device__ __forceinline__ uint32_t first_valid(uint64_t ks, uint32_t c, uint64_t L) {
  const uint64_t v0 = 6 * ks + c;
  return v0 >= L ? 0u : static_cast<uint32_t>((L - v0 + 5) / 6);
}
__device__ __forceinline__ uint32_t end_valid(uint64_t ks, uint32_t c, uint64_t R, uint32_t len) {
  const uint64_t v0 = 6 * ks + c;
  if (v0 >= R) return 0u;
  const uint64_t n = (R - v0 + 5) / 6;
  return n < len ? static_cast<uint32_t>(n) : len;
}

__device__ void fetch_segment(const SieveParams& P, SegInfo& si) {
  const unsigned long long t = atomicAdd(P.ticket, 1ull);
  si.s = t < P.s_count ? P.s_begin + t : ~0ull;
  if (t >= P.s_count) {
    // every CTA draws exactly one failing ticket; after the last one no CTA
    // draws again, so it resets the pair for the next launch (no memset)
    if (atomicAdd(P.ticket + 1, 1ull) == gridDim.x - 1) {
      P.ticket[0] = 0;
      P.ticket[1] = 0;
    }
    return;
  }
  const uint64_t s = si.s;
  uint32_t lo = 0;
  Job J;
  if (P.njobs == 1) {
    J = P.job0;
  } else {
    uint32_t hi = P.njobs;  // last job with seg_begin <= s
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (P.jobs[mid].seg_begin <= s) lo = mid; else hi = mid;
    }
    J = P.jobs[lo];
  }
  si.job = lo;
  const uint64_t local = s - J.seg_begin;
  si.ks = J.K0 + local * P.S;
  const uint64_t rem = J.nslots - local * P.S;
  si.len = rem < P.S ? static_cast<uint32_t>(rem) : P.S;
  si.lo1 = first_valid(si.ks, 1, J.L);
  if (si.ks == 0 && si.lo1 < 1) si.lo1 = 1;  // value 1 is not prime (engine.cpp:244)
  si.lo5 = first_valid(si.ks, 5, J.L);
  si.hi1 = end_valid(si.ks, 1, J.R, si.len);
  si.hi5 = end_valid(si.ks, 5, J.R, si.len);
  si.nwords = ((si.len + 1023u) / 1024u) * 32u;
  // activation thresholds: p*p = 6*ksq + 1 is at or past slot ks iff
  // p > isqrt(6 ks), and before the segment end iff p <= isqrt(6 (ks + len))
  si.t_lo = isqrt64(6 * si.ks);
  si.t_hi = isqrt64(6 * (si.ks + si.len));
}

// Phase 1: stamp primes 5..47 and the [L, R) trim into every word.  The
// bitmaps hold COMPOSITE flags (bit set = crossed off or outside [L, R)):
// the complement of the reference's FlagArray, so crossing off is a single
// ATOMS.OR and survivors are ~word.
// Stamps the small-prime patterns into the segment: one 32-bit word per
// thread and iteration (a warp writes 128 contiguous bytes = one shared
// wavefront, and its table reads are conflict-free; 4-word-per-lane 128-bit
// stores move the same bytes but make the lanes' table reads 4-way bank
// conflicted).  Table phases are carried incrementally (+32 * kThreads mod Q
// per iteration) instead of a modulo per word.
__device__ __forceinline__ uint32_t phase_step(uint32_t a, uint32_t step, uint32_t Q) {
  a += step;
  return a >= Q ? a - Q : a;
}

__device__ __forceinline__ void init_words(const SegInfo& si, const uint2* tab, uint32_t* bm1,
                                           uint32_t* bm5) {
  constexpr uint32_t kStride = 32u * kThreads;
  uint32_t a0 = static_cast<uint32_t>((si.ks + 32u * threadIdx.x) % 5005u);
  uint32_t a1 = static_cast<uint32_t>((si.ks + 32u * threadIdx.x) % 7429u);
  uint32_t a2 = static_cast<uint32_t>((si.ks + 32u * threadIdx.x) % 899u);
  uint32_t a3 = static_cast<uint32_t>((si.ks + 32u * threadIdx.x) % 1517u);
  uint32_t a4 = static_cast<uint32_t>((si.ks + 32u * threadIdx.x) % 2021u);
  const uint2* t1 = tab;
  const uint2* t5 = tab + kTabPerClass;
  // only a range's first and last segments are trimmed (and only the first
  // segment of [0, ...) keeps the stamped primes): interior segments skip
  // both with one block-uniform test
  const uint32_t full = 32u * si.nwords;
  const bool edge =
      si.lo1 != 0 || si.lo5 != 0 || si.hi1 != full || si.hi5 != full || si.ks < 8;
  for (uint32_t w = threadIdx.x; w < si.nwords; w += kThreads) {
    uint32_t m1 = tab_read(t1, a0) & tab_read(t1 + tab_off(1), a1) & tab_read(t1 + tab_off(2), a2) &
                  tab_read(t1 + tab_off(3), a3) & tab_read(t1 + tab_off(4), a4);
    uint32_t m5 = tab_read(t5, a0) & tab_read(t5 + tab_off(1), a1) & tab_read(t5 + tab_off(2), a2) &
                  tab_read(t5 + tab_off(3), a3) & tab_read(t5 + tab_off(4), a4);
    a0 = phase_step(a0, kStride % 5005u, 5005u);
    a1 = phase_step(a1, kStride % 7429u, 7429u);
    a2 = phase_step(a2, kStride % 899u, 899u);
    a3 = phase_step(a3, kStride % 1517u, 1517u);
    a4 = phase_step(a4, kStride % 2021u, 2021u);
    if (edge) {
      if (w == 0 && si.ks < 8) {
        // the stamped primes themselves survive: 7, 13, 19, 31, 37, 43 at
        // class-1 indices 1, 2, 3, 5, 6, 7 and 5, 11, 17, 23, 29, 41, 47 at
        // class-5 indices 0..4, 6, 7
        m1 |= 0xEEu >> si.ks;
        m5 |= 0xDFu >> si.ks;
      }
      const int64_t base = 32 * static_cast<int64_t>(w);
      m1 &= range_mask(static_cast<int64_t>(si.lo1) - base, static_cast<int64_t>(si.hi1) - base);
      m5 &= range_mask(static_cast<int64_t>(si.lo5) - base, static_cast<int64_t>(si.hi5) - base);
    }
    bm1[w] = ~m1;
    bm5[w] = ~m5;
  }
}

// ks mod p from the FP64 quotient estimate (1/p comes preloaded: the prime
// loops load it together with p, one iteration ahead); Barrett above 2^53
__device__ __forceinline__ uint32_t mod_p(const ModCtx& c, uint32_t p, double inv_p,
                                          const unsigned long long* m, uint32_t i) {
  if (c.fast) {
    const double t = __fma_rn(c.ksd, inv_p, 6755399441055744.0);
    const uint32_t q = static_cast<uint32_t>(__double2loint(t));
    uint32_t r = c.kslo - q * p;
    if (static_cast<int32_t>(r) < 0) r += p;
    return r;
  }
  return mod_barrett(c.ks, p, __ldg(m + i));
}

// First hits (segment-relative) of prime p in both classes, or false when
// p is not yet active in this segment (p*p beyond its end; since primes
// ascend, no later prime is active either).  The activation test is two
// 32-bit compares against the segment's thresholds.
__device__ __forceinline__ bool prime_offsets(uint32_t p, double inv_p, uint32_t i,
                                              const unsigned long long* m, const ModCtx& mc,
                                              uint32_t t_lo, uint32_t t_hi, uint32_t& rel1,
                                              uint32_t& rel5) {
  if (p > t_hi) return false;
  uint32_t t1, t5;
  targets(p, t1, t5);
  if (p > t_lo) {
    // activation segment: class 1 starts exactly at p*p, class 5 at the
    // first multiple above it (anchor p*(p-1), segment.cpp:182)
    const uint64_t ksq = (static_cast<uint64_t>(p) * p - 1) / 6;
    rel1 = static_cast<uint32_t>(ksq - mc.ks);
    rel5 = rel1 + (t5 >= t1 ? t5 - t1 : t5 + p - t1);
  } else {
    const uint32_t r = mod_p(mc, p, inv_p, m, i);
    rel1 = t1 >= r ? t1 - r : t1 + p - r;
    rel5 = t5 >= r ? t5 - r : t5 + p - r;
  }
  return true;
}

// prime_offsets with the quotient path fixed at compile time (FAST: the FP64
// estimate, ks < 2^53), for loops unswitched on the segment-uniform flag
template <bool FAST>
__device__ __forceinline__ bool prime_offsets_t(uint32_t p, double inv_p, uint32_t i,
                                                const unsigned long long* m, const ModCtx& mc,
                                                uint32_t t_lo, uint32_t t_hi, uint32_t& rel1,
                                                uint32_t& rel5) {
  if (p > t_hi) return false;
  uint32_t t1, t5;
  targets(p, t1, t5);
  if (p > t_lo) {  // activation segment (see prime_offsets)
    const uint64_t ksq = (static_cast<uint64_t>(p) * p - 1) / 6;
    rel1 = static_cast<uint32_t>(ksq - mc.ks);
    rel5 = rel1 + (t5 >= t1 ? t5 - t1 : t5 + p - t1);
  } else {
    uint32_t r;
    if constexpr (FAST) {
      const double t = __fma_rn(mc.ksd, inv_p, 6755399441055744.0);
      r = mc.kslo - static_cast<uint32_t>(__double2loint(t)) * p;
      if (static_cast<int32_t>(r) < 0) r += p;
    } else {
      r = mod_barrett(mc.ks, p, __ldg(m + i));
    }
    rel1 = t1 >= r ? t1 - r : t1 + p - r;
    rel5 = t5 >= r ? t5 - r : t5 + p - r;
  }
  return true;
}


// ... if h < len, branch-free: a miss ORs 0 into the word picked by h's own
// bits under wmask (spread over the banks, always inside the bitmap)
__device__ __forceinline__ void mark_or(uint32_t a0, uint32_t h, uint32_t len, uint32_t wmask) {
  atom_or_shared(a0 + (((h >> 5) & wmask) << 2), h < len ? 1u << (h & 31u) : 0u);
}

// ... the miss going to word `lane` (bank `lane`) instead: a miss then adds at
// most one access to a bank a hit uses, rather than one at a random bank
// (modelled: 3.09 vs 3.53 wavefronts per warp op at a 50% hit rate)
__device__ __forceinline__ void mark_or_lane(uint32_t a0, uint32_t h, uint32_t len, uint32_t lane) {
  const bool hit = h < len;
  atom_or_shared(a0 + ((hit ? h >> 5 : lane) << 2), hit ? bit_of(h) : 0u);
}

// cross off the bit at shared-memory bit address hb
__device__ __forceinline__ void mark_bitaddr(uint32_t hb) {
  atom_or_shared((hb >> 3) & ~3u, bit_of(hb));
}

// Mid-prime hits with the multiples of 5 skipped.  Hit j of prime p in class
// c sits at wheel index K_j = K_0 + j p and has value 6 K_j + c = p m_j; it is
// a multiple of 5 -- a slot the stamped prime 5 has already crossed off --
// exactly when K_j == -c (mod 5), i.e. for every fifth j from j0 on (p is
// coprime to 5).  From hb (shared bit address of hit 0) below lim: hits
// 0 .. j0-1, then groups of four with the fifth skipped.
__device__ __forceinline__ void mark_skip5(uint32_t hb, uint32_t lim, uint32_t p, uint32_t j0) {
  for (; j0 > 0 && hb < lim; --j0, hb += p) mark_bitaddr(hb);
  hb += p;  // hit j0: a multiple of 5
  const uint32_t p2 = 2 * p, p3 = 3 * p, p5 = 5 * p;
  for (; hb + p3 < lim; hb += p5) {
    mark_bitaddr(hb);
    mark_bitaddr(hb + p);
    mark_bitaddr(hb + p2);
    mark_bitaddr(hb + p3);
  }
  for (uint32_t k = 0; k < 3 && hb < lim; ++k, hb += p) mark_bitaddr(hb);
}

// j0 of class c (cmod = (-c) mod 5: 4 for 6k+1, 0 for 6k+5) for a first hit at
// wheel index K0 (K0 mod 5 = k05) of a prime with 1/p mod 5 = inv5
__device__ __forceinline__ uint32_t skip5_phase(uint32_t k05, uint32_t cmod, uint32_t inv5) {
  const uint32_t d = cmod + 5u - k05;  // 1..9: (cmod - K0) mod 5 after one reduction
  const uint32_t dm = d >= 5u ? d - 5u : d;
  const uint32_t x = dm * inv5;  // <= 16
  return x - 5u * ((x * 13u) >> 6);  // x mod 5 for x <= 16
}

// cross off bit h of the bitmap at shared address a0
__device__ __forceinline__ void mark(uint32_t a0, uint32_t h) {
  atom_or_shared(a0 + ((h >> 5) << 2), bit_of(h));
}

// ... only if h < len, as a predicated atomic (no branch / reconvergence)
__device__ __forceinline__ void mark_if(uint32_t a0, uint32_t h, uint32_t len) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.lt.u32 q, %2, %3;\n\t@q red.shared.or.b32 [%0], %1;\n\t}"
      ::"r"(a0 + ((h >> 5) << 2)), "r"(bit_of(h)), "r"(h), "r"(len)
      : "memory");
}

// Warp-cooperative strided marking of one class: lane l takes hits
// h0 + l*p, h0 + (l+32)*p, ...  Consecutive hits of a lane are 32*p bits
// apart, i.e. exactly p words, so the bit within the word is loop-invariant
// and the loop only steps a shared byte address by 4p.
__device__ __forceinline__ void mark_strided(uint32_t a0, uint32_t h0, uint32_t p, uint32_t len,
                                             uint32_t lane) {
  const uint32_t h = h0 + lane * p;
  if (h >= len) return;
  const uint32_t bit = 1u << (h & 31u);
  const uint32_t alim = a0 + (((len - (h & 31u) + 31u) >> 5) << 2);
  const uint32_t step = 4 * p;
  uint32_t a = a0 + ((h >> 5) << 2);
  for (; a + 3 * step < alim; a += 4 * step) {
    atom_or_shared(a, bit);
    atom_or_shared(a + step, bit);
    atom_or_shared(a + 2 * step, bit);
    atom_or_shared(a + 3 * step, bit);
  }
  for (; a < alim; a += step) atom_or_shared(a, bit);
}

// Transposed warp-cooperative marking of one class: hits are taken in
// superblocks of 1024, lane l owning hits 32 l .. 32 l + 31 of the superblock
// and warp op i marking hit 32 l + i in every lane.  The lanes of an op are
// then exactly 32 p bits = p words apart -- p is odd, so the 32 words fall in
// 32 different banks (one wavefront per op, where consecutive hits per op
// average 2.5) -- and they share the bit within the word.  In a last partial
// superblock of at least tmin hits the lanes whose 32 hits all fit run the
// same way; shorter tails use the strided loop.
__device__ __forceinline__ void mark_transposed(uint32_t a0, uint32_t rel, uint32_t p,
                                                uint32_t len, uint32_t lane, uint32_t tmin) {
  const uint32_t lane_off = a0 + 4u * lane * p;
  // word address of the lane's hit at superblock-relative position pos: one
  // shift and one multiply-add
  auto mark_at = [&](uint32_t pos) {
    uint32_t addr;
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(addr) : "r"(pos >> 5), "r"(lane_off));
    atom_or_shared(addr, bit_of(pos));
  };
  uint32_t pos = rel;
  while (pos + 1023u * p < len) {
#pragma unroll 8
    for (uint32_t i = 0; i < 32; ++i) {
      mark_at(pos);
      pos += p;
    }
    pos += 992u * p;
  }
  if (pos + (tmin - 1u) * p < len) {
    // last, partial superblock: the lanes whose 32 hits all lie below len run
    // the same 32 ops under ONE branch (no per-op predicate); the hits after
    // them -- fewer than 32 -- are one strided op
    const bool full = pos + 32u * lane * p + 31u * p < len;
    const uint32_t nfull = __popc(__ballot_sync(kFull, full));
    if (full) {
      uint32_t q = pos;
#pragma unroll 8
      for (uint32_t i = 0; i < 32; ++i) {
        mark_at(q);
        q += p;
      }
    }
    pos += 32u * nfull * p;
  }
  if (pos < len) mark_strided(a0, pos, p, len, lane);
}

// Phase 2: medium and large primes (NT threads per block).
template <int NT, bool WC_LAST = false, bool WCT = false, bool BK = true>
__device__ __forceinline__ void sieve_primes(const SieveParams& P, const SegInfo& si,
                                             uint32_t* bm1, uint32_t* bm5, uint32_t* wc_ctr,
                                             uint32_t nprimes) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t len = si.len;
  const uint64_t ks = si.ks;
  const uint32_t a1 = smem_addr(bm1), a5 = smem_addr(bm5);
  const uint32_t t_lo = si.t_lo, t_hi = si.t_hi;
  const ModCtx mc = mod_ctx(ks);
  const uint32_t ks5 = static_cast<uint32_t>(ks % 5u);  // for the multiple-of-5 skips
  const uint32_t n_wc = min(P.n_wc, nprimes), n_mid = min(P.n_mid, nprimes);
  const uint32_t n_S = min(P.n_S, nprimes);  // (mid_end below caps it when bucketing)
  // warp-cooperative primes, handed out dynamically (largest work first); the
  // next prime is claimed and its p and 1/p loaded while the current one is
  // marked
  auto claim = [&](uint32_t& i, uint32_t& p, double& ip) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(wc_ctr, 1u);
    i = __shfl_sync(kFull, k, 0);
    if (i < n_wc) {
      p = __ldg(P.prime_p + i);
      ip = __ldg(P.prime_inv + i);
    }
  };
  auto wc_phase = [&]() {
    uint32_t wi, wp = 0;
    double wip = 0.0;
    claim(wi, wp, wip);
    while (wi < n_wc) {
      const uint32_t i = wi, p = wp;
      const double ip = wip;
      claim(wi, wp, wip);
      uint32_t rel1, rel5;
      if (!prime_offsets(p, ip, i, P.prime_m, mc, t_lo, t_hi, rel1, rel5)) break;
      if (WCT) {
        mark_transposed(a1, rel1, p, len, lane, P.trans_min);
        mark_transposed(a5, rel5, p, len, lane, P.trans_min);
      } else {
        mark_strided(a1, rel1, p, len, lane);
        mark_strided(a5, rel5, p, len, lane);
      }
    }
  };
  // WC_LAST (a lone CTA per SM): the dynamically claimed primes come after the
  // static chunks, smallest tasks last, so they even out the warps' finish
  // times before the closing barrier
  if (!WC_LAST) wc_phase();
  // large primes come from the window's bucket list unless it overflowed
  // (a wide unit: every one of its segments' lists)
  const uint32_t nparts = WC_LAST ? (len + P.S - 1) / P.S : 1u;
  bool use_bucket = BK && P.bucket != nullptr;  // BK false: a launch without bucket lists
  if (use_bucket)
    for (uint32_t part = 0; part < nparts; ++part)
      use_bucket = use_bucket && P.bcount[si.s - P.s_begin + part] <= P.bcap;
  const uint32_t lp_end = use_bucket ? n_mid : nprimes;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t mid_end = n_S < lp_end ? n_S : lp_end;
  // The per-thread prime loops below load p and 1/p one iteration ahead: the
  // loads are independent of the segment, and issuing them together and early
  // turns two dependent global round trips per (prime, segment) into none on
  // the critical path.
  constexpr uint32_t kStride = NT;  // 32 primes per warp and round
  auto load = [&](uint32_t idx, uint32_t end, uint32_t& p, double& ip) {
    if (idx < end) {
      p = __ldg(P.prime_p + idx);
      ip = __ldg(P.prime_inv + idx);
    } else {
      p = 0xFFFFFFFFu;
      ip = 0.0;
    }
  };
  // p < S: one thread per prime, static warp-sized chunks (round robin);
  // both classes advance together (their hits are the same stride p apart)
  {
    // bit addresses fit 32 bits while the bitmaps sit below 2^28 in the
    // shared window (always, for unclustered launches)
    const bool bitaddr = P.mid_bitaddr && a1 < (1u << 28) && a5 < (1u << 28);
    const uint32_t b1 = a1 << 3, b5 = a5 << 3;
    // primes below skip5_max: class loops that skip the multiples of 5
    const uint32_t skip_max = bitaddr ? P.skip5_max : 0u;
    uint32_t base = n_wc + 32 * warp;
    uint32_t pn;
    double ipn;
    load(base + lane, mid_end, pn, ipn);
    for (; base < mid_end; base += kStride) {
      const uint32_t p = pn, i = base + lane;
      const double ip = ipn;
      load(base + kStride + lane, mid_end, pn, ipn);
      if (__shfl_sync(kFull, p, 0) > t_hi) break;  // primes ascend: the rest is inactive
      uint32_t rel1, rel5;
      if (!prime_offsets(p, ip, i, P.prime_m, mc, t_lo, t_hi, rel1, rel5)) continue;
      if (p < skip_max) {
        const uint32_t inv5 = (0x42310u >> (4u * (p % 5u))) & 7u;  // 1/p mod 5
        mark_skip5(b1 + rel1, b1 + len, p, skip5_phase((ks5 + rel1) % 5u, 4u, inv5));
        mark_skip5(b5 + rel5, b5 + len, p, skip5_phase((ks5 + rel5) % 5u, 0u, inv5));
        continue;
      }
      const int32_t d = static_cast<int32_t>(rel5 - rel1);
      const uint32_t dpos = d > 0 ? static_cast<uint32_t>(d) : 0u;
      uint32_t h = rel1;
      if (bitaddr) {
        // the hits as shared-memory BIT addresses: word address (hb >> 3) & ~3
        // and bit hb & 31 with no base add, and the loop bound precomputed
        // (12 instructions per pair of marks instead of 14)
        const uint32_t dd = (a5 << 3) - b1 + static_cast<uint32_t>(d);
        const uint32_t lim = len > dpos ? b1 + (len - dpos) : 0u;
        uint32_t hb = b1 + h;
        for (; hb < lim; hb += p) {
          mark_bitaddr(hb);
          mark_bitaddr(hb + dd);
        }
        h = hb - b1;
      } else {
        for (; h + dpos < len; h += p) {
          mark(a1, h);
          mark(a5, h + d);
        }
      }
      mark_if(a1, h, len);
      mark_if(a5, h + d, d < 0 ? len : 0u);
    }
  }
  // p >= len / HITS: at most HITS hits per class -- no loop, no branch;
  // unswitched on the quotient path (ks < 2^53 everywhere but the very top).
  // HITS == 2 (wide units, primes of at least half the unit): the second hit
  // is p further on.  (Three hits for primes of a third measured no faster.)
  auto few_hits = [&](auto fast, auto hits, uint32_t begin, uint32_t end) {
    uint32_t base = begin + 32 * warp;
    uint32_t pn;
    double ipn;
    load(base + lane, end, pn, ipn);
    for (; base < end; base += kStride) {
      const uint32_t p = pn, i = base + lane;
      const double ip = ipn;
      load(base + kStride + lane, end, pn, ipn);
      if (__shfl_sync(kFull, p, 0) > t_hi) break;
      uint32_t rel1 = len, rel5 = len;
      prime_offsets_t<decltype(fast)::value>(p, ip, i, P.prime_m, mc, t_lo, t_hi, rel1, rel5);
      if (P.single_pred) {
        // predicated: lanes without a hit issue no shared-memory access, so
        // the warp's conflict degree is that of its hitting lanes only
        mark_if(a1, rel1, len);
        mark_if(a5, rel5, len);
      } else if (P.miss_lane) {
        mark_or_lane(a1, rel1, len, lane);
        mark_or_lane(a5, rel5, len, lane);
      } else {
        mark_or(a1, rel1, len, P.S / 32 - 1);
        mark_or(a5, rel5, len, P.S / 32 - 1);
      }
      if (decltype(hits)::value >= 2) {  // (wide launches set miss_lane)
        // min: rel + p must not wrap for the out-of-range sentinel p = 2^32 - 1
        const uint32_t step = min(p, len);
        mark_or_lane(a1, rel1 + step, len, lane);
        mark_or_lane(a5, rel5 + step, len, lane);
      }
    }
  };
  const uint32_t dbl_end = max(mid_end, min(P.n_dbl, lp_end));
  auto few_all = [&](auto fast) {
    if (dbl_end > mid_end) few_hits(fast, std::integral_constant<int, 2>{}, mid_end, dbl_end);
    few_hits(fast, std::integral_constant<int, 1>{}, dbl_end, lp_end);
  };
  if (mc.fast)
    few_all(std::true_type{});
  else
    few_all(std::false_type{});
  if (use_bucket) {
    // an entry is the bit index into [bm1 | bm5] (class at bit log2 S), so a
    // hit is shift + atomic; lists are read 4 entries per 128-bit streamed
    // load, two loads in flight per thread.  In a wide unit the classes are
    // P.wide * S bits apart and segment `part` starts S * part bits in:
    // entry e -> e + part S + (e >> log2 S) (wide - 1) S.
    const uint32_t log2S = 31u - __clz(P.S);
    const uint32_t wm1S = WC_LAST ? (P.wide - 1u) * P.S : 0u;
    for (uint32_t part = 0; part < nparts; ++part) {
      const uint32_t partS = part * P.S;
      auto put = [&](uint32_t e) {
        if (WC_LAST)
          mark(a1, e + partS + (e >> log2S) * wm1S);
        else
          mark(a1, e);
      };
      const uint64_t ls = si.s - P.s_begin + part;
      const uint32_t n = P.bcount[ls];
      const uint32_t* list = P.bucket + ls * P.bcap;  // 128 B aligned (bcap % 32 == 0)
      const uint4* list4 = reinterpret_cast<const uint4*>(list);
      const uint32_t n4 = n >> 2;
      uint32_t i = threadIdx.x;
      for (; i + NT < n4; i += 2 * NT) {
        const uint4 x = __ldcs(list4 + i), y = __ldcs(list4 + i + NT);
        put(x.x);
        put(x.y);
        put(x.z);
        put(x.w);
        put(y.x);
        put(y.y);
        put(y.z);
        put(y.w);
      }
      if (i < n4) {
        const uint4 x = __ldcs(list4 + i);
        put(x.x);
        put(x.y);
        put(x.z);
        put(x.w);
      }
      for (uint32_t j = 4 * n4 + threadIdx.x; j < n; j += NT) put(__ldcs(list + j));
    }
  }
  if (WC_LAST) wc_phase();
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_xor64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_max64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(kFull, v, o);
    v = u > v ? u : v;
  }
  return v;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(kFull, v, o);
    if (lane >= static_cast<uint32_t>(o)) v += u;
  }
  return v;
}

// spread the low 16 bits of x to the even bit positions of a 32-bit word
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kValMask = (1ull << 62) - 1;

// Decoupled look-back (warp 0): exclusive prefix of survivor counts over all
// segments before s.  Segments are claimed in ticket order, so every
// predecessor is owned by a running block and the wait terminates.
__device__ unsigned long long lookback(unsigned long long* status, uint64_t s,
                                       unsigned long long total) {
  const uint32_t lane = threadIdx.x & 31u;
  if (s == 0) {
    if (lane == 0) st_release(status, kIncl | total);
    return 0;
  }
  if (lane == 0) st_release(status + s, kAgg | total);
  unsigned long long prefix = 0;
  int64_t j = static_cast<int64_t>(s) - 1;
  for (;;) {
    const int64_t idx = j - static_cast<int64_t>(lane);
    unsigned long long v = kIncl;  // before segment 0: inclusive prefix 0
    if (idx >= 0) {
      do {
        v = ld_acquire(status + idx);
      } while ((v >> 62) == 0);
    }
    const unsigned incl = __ballot_sync(kFull, (v >> 62) == 2);
    if (incl) {
      const int k = __ffs(incl) - 1;  // nearest inclusive predecessor
      const unsigned long long mine = lane <= static_cast<uint32_t>(k) ? (v & kValMask) : 0ull;
      prefix += warp_sum64(mine);
      break;
    }
    prefix += warp_sum64(v & kValMask);
    j -= 32;
  }
  if (lane == 0) st_release(status + s, kIncl | (prefix + total));
  return prefix;
}

// Emission staging: per warp, a window of up to kStage 16-bit survivor
// positions of one 32-word round (bit 64*lane + b of the interleaved masks).
// 320 is the largest window that keeps 3 CTAs per SM (3 x (64 KiB bitmap +
// 10 KiB stage + static + reserved) <= 228 KiB); a C2 round averages ~280.
constexpr uint32_t kStage = 320;

// The segment's largest survivor (0 if none), in every lane of the calling
// warp: the top nonzero word of the bitmap, found 32 words at a time from the
// end (the job's largest is its last segment's; one step almost always).
__device__ __forceinline__ unsigned long long segment_largest(const SegInfo& si,
                                                              const uint32_t* bm1,
                                                              const uint32_t* bm5,
                                                              unsigned long long vbase,
                                                              uint32_t lane) {
  for (int32_t top = static_cast<int32_t>(si.nwords) - 1; top >= 0; top -= 32) {
    const int32_t w = top - static_cast<int32_t>(lane);
    uint32_t m1 = 0, m5 = 0;
    if (w >= 0) {
      m1 = ~bm1[w];
      m5 = ~bm5[w];
    }
    const uint32_t any = __ballot_sync(0xffffffffu, (m1 | m5) != 0u);
    if (any) {
      unsigned long long lg = 0;
      if (lane == static_cast<uint32_t>(__ffs(any) - 1)) {
        const unsigned long long wb = vbase + 192ull * static_cast<uint32_t>(w);
        const unsigned long long v1 = m1 ? wb + 6ull * (31 - __clz(m1)) + 1 : 0;
        const unsigned long long v5 = m5 ? wb + 6ull * (31 - __clz(m5)) + 5 : 0;
        lg = v1 > v5 ? v1 : v5;
      }
      return __shfl_sync(0xffffffffu, lg, __ffs(any) - 1);
    }
  }
  return 0;
}

template <int MODE>
constexpr size_t mode_smem_extra() {
  return MODE >= kEnumerate ? kWarps * kStage * sizeof(uint16_t) : 0;
}

// ---------------------------------------------------------------------------
template <int MODE, bool WCT = false>
__global__ void __launch_bounds__(kThreads, 3) sieve_kernel(const SieveParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* bm1 = smem;
  uint32_t* bm5 = smem + P.S / 32;
  const uint2* tab = reinterpret_cast<const uint2*>(P.small_tab);  // 8.7 KB, L1-resident
  uint16_t* stage_all = reinterpret_cast<uint16_t*>(smem + 2 * (P.S / 32));
  __shared__ SegInfo si;
  __shared__ unsigned long long red_a[kWarps], red_b[kWarps], red_c[kWarps];
  __shared__ uint32_t red_n[kWarps];
  __shared__ uint32_t wc_ctr;
  __shared__ unsigned long long seg_base;
  __shared__ uint32_t seg_total;
  constexpr bool kWire = MODE == kEnumWire;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;

  const uint32_t nprimes = P.nprimes_dev ? min(P.nprimes, *P.nprimes_dev) : P.nprimes;
  if (P.tabn_out != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *P.tabn_out = nprimes;
  for (;;) {
    __syncthreads();  // bitmap / si reuse guard
    if (threadIdx.x == 0) {
      fetch_segment(P, si);
      wc_ctr = 0;
    }
    __syncthreads();
    if (si.s == ~0ull) break;
    init_words(si, tab, bm1, bm5);
    __syncthreads();
    sieve_primes<kThreads, false, WCT>(P, si, bm1, bm5, &wc_ctr, nprimes);
    __syncthreads();
    if (P.bucket != nullptr && threadIdx.x == 0) P.bcount[si.s - P.s_begin] = 0;

    const uint64_t vbase = 6 * si.ks;
    if (MODE < kEnumerate && P.words1 != nullptr) {  // SegmentBitmap export
      const uint64_t wb = si.s * (P.S / 32);  // single-job launches
      const uint32_t nw = (si.len + 63) / 64 * 2;  // whole uint64 FlagArray words
      for (uint32_t w = threadIdx.x; w < nw; w += kThreads) {
        P.words1[wb + w] = ~bm1[w];
        P.words5[wb + w] = ~bm5[w];
      }
    }
    if (MODE < kEnumerate) {
      uint32_t cnt = 0;
      unsigned long long lg = 0, sum = 0, xr = 0;
      for (uint32_t wp = threadIdx.x; wp < si.nwords; wp += kThreads) {
        const uint32_t m1 = ~bm1[wp], m5 = ~bm5[wp];
        cnt += __popc(m1) + __popc(m5);
        if (MODE == kCountChecks && (m1 | m5)) {
          const unsigned long long wb = vbase + 192ull * wp;
          for (uint32_t x = m1; x; x &= x - 1) {
            const unsigned long long v = wb + 6ull * (__ffs(x) - 1) + 1;
            sum += v;
            xr ^= v;
          }
          for (uint32_t x = m5; x; x &= x - 1) {
            const unsigned long long v = wb + 6ull * (__ffs(x) - 1) + 5;
            sum += v;
            xr ^= v;
          }
        }
      }
      cnt = __reduce_add_sync(kFull, cnt);
      if (warp == 0) lg = segment_largest(si, bm1, bm5, vbase, lane);
      if (MODE == kCountChecks) {
        sum = warp_sum64(sum);
        xr = warp_xor64(xr);
      }
      if (lane == 0) {
        red_n[warp] = cnt;
        red_a[warp] = lg;
        red_b[warp] = sum;
        red_c[warp] = xr;
      }
      __syncthreads();
      if (warp == 0) {
        uint32_t c = lane < kWarps ? red_n[lane] : 0u;
        unsigned long long l = lane < kWarps ? red_a[lane] : 0ull;
        unsigned long long su = lane < kWarps ? red_b[lane] : 0ull;
        unsigned long long x = lane < kWarps ? red_c[lane] : 0ull;
        c = __reduce_add_sync(kFull, c);
        l = warp_max64(l);
        if (MODE == kCountChecks) {
          su = warp_sum64(su);
          x = warp_xor64(x);
        }
        if (lane == 0) {
          JobAcc& A = P.acc[si.job];
          if (P.per_seg) P.per_seg[si.s] = c;
          if (c) {
            atomicAdd(&A.count, static_cast<unsigned long long>(c));
            atomicMax(&A.largest, l);
            if (MODE == kCountChecks) {
              atomicAdd(&A.sum, su);
              atomicXor(&A.xr, x);
            }
          }
        }
      }
    } else {
      // ---- ordered enumeration ----
      // warp `warp` owns logical words [w_begin, w_end), in word order; the
      // shares are whole 32-word rounds so that no round straddles a wire
      // block (1024 words) even in a clipped last segment
      const uint32_t wpw = (si.nwords + 32 * kWarps - 1) / (32 * kWarps) * 32;
      const uint32_t w_begin = min(warp * wpw, si.nwords);
      const uint32_t w_end = min(w_begin + wpw, si.nwords);
      uint32_t cnt = 0;
      for (uint32_t w = w_begin + lane; w < w_end; w += 32)
        cnt += __popc(~bm1[w]) + __popc(~bm5[w]);
      cnt = __reduce_add_sync(kFull, cnt);
      if (lane == 0) red_n[warp] = cnt;
      __syncthreads();
      if (warp == 0) {
        const uint32_t c = lane < kWarps ? red_n[lane] : 0u;
        const uint32_t incl = warp_incl_scan(c, lane);
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        if (lane < kWarps) red_n[lane] = incl - c;
        const unsigned long long base = lookback(P.status, si.s, total);
        if (lane == 0) {
          seg_base = base;
          seg_total = total;
          if (P.per_seg) P.per_seg[si.s] = total;
          if (total) atomicAdd(&P.acc[si.job].count, static_cast<unsigned long long>(total));
        }
      }
      __syncthreads();
      unsigned long long pos = seg_base + red_n[warp];
      const bool seg_fits = seg_base + seg_total <= P.out_cap;
      unsigned long long sum = 0, xr = 0, lg = 0;
      uint16_t* stage = stage_all + warp * kStage;
      for (uint32_t w0 = w_begin; w0 < w_end; w0 += 32) {
        const uint32_t w = w0 + lane;
        uint32_t a = 0, b = 0;
        if (w < w_end) {
          a = ~bm1[w];
          b = ~bm5[w];
        }
        // ascending value order interleaves the classes: bit 2j <- 6k+1, 2j+1 <- 6k+5
        const uint32_t lo = spread16(a) | (spread16(b) << 1);
        const uint32_t hi = spread16(a >> 16) | (spread16(b >> 16) << 1);
        const uint32_t c = __popc(lo) + __popc(hi);
        const uint32_t incl = warp_incl_scan(c, lane);
        const uint32_t rtotal = __shfl_sync(kFull, incl, 31);
        const unsigned long long rbase = vbase + 192ull * w0;  // value base of the round
        if (kWire) {  // survivors per 4-word wire block (lanes 4k .. 4k+3), one byte each
          uint32_t bc = c + __shfl_down_sync(kFull, c, 1, 4);
          bc += __shfl_down_sync(kFull, bc, 2, 4);
          if ((lane & 3u) == 0 && w < w_end)
            P.blk8[si.s * (P.S / 128) + (w >> 2)] = static_cast<uint8_t>(bc);
        }
        if (rtotal == 0) continue;
        // The round's survivors go out in windows of kStage positions: each
        // pass, lanes drop their survivors that fall in the window into the
        // stage (in ascending order), then lane i writes window entries i,
        // i+32, ... coalesced.  Almost every round is one window; dense ones
        // (small values) take a few.  The stage holds positions 64*lane + b
        // (bit b of the interleaved masks); a survivor's value offset from
        // rbase is 192*lane + 3b + 1 + (b & 1) < 6144.
        const uint32_t eb = lane << 6, ob = 192u * lane;
        // the round's values share rbase's high word unless its low word is
        // within 6144 of wrapping (once in ~7e5 rounds): 32-bit arithmetic
        const uint32_t rlo = static_cast<uint32_t>(rbase);
        const uint32_t rhi = static_cast<uint32_t>(rbase >> 32);
        const bool nocarry = rlo < 0xFFFFFFFFu - 6144u;
#pragma unroll 1
        for (uint32_t wlo = 0; wlo < rtotal; wlo += kStage) {
          const uint32_t wn = min(kStage, rtotal - wlo);
          // stage entry of interleaved bit position t (0..63) of this lane:
          // the wire byte source (64 * lane + t) for the wire, else the value
          // offset from rbase, 192 * lane + 3t + 1 + (t & 1) < 6144
          auto enc = [&](uint32_t t) -> uint16_t {
            if (kWire) return static_cast<uint16_t>(eb | t);
            return static_cast<uint16_t>(ob + 3u * t + 1u + (t & 1u));
          };
          if (rtotal <= kStage) {  // one window (warp-uniform): no position test
            uint16_t* sp = stage + (incl - c);
#pragma unroll 1
            for (uint32_t x = lo; x; x &= x - 1) *sp++ = enc(__ffs(x) - 1);
#pragma unroll 1
            for (uint32_t x = hi; x; x &= x - 1) *sp++ = enc(31u + __ffs(x));
          } else if (incl > wlo && incl - c < wlo + wn) {  // lane has entries in the window
            uint32_t q = incl - c - wlo;  // window-relative position (wraps below 0)
#pragma unroll 1
            for (uint32_t x = lo; x; x &= x - 1, ++q)
              if (q < wn) stage[q] = enc(__ffs(x) - 1);
#pragma unroll 1
            for (uint32_t x = hi; x; x &= x - 1, ++q)
              if (q < wn) stage[q] = enc(31u + __ffs(x));
          }
          __syncwarp();
          const unsigned long long wpos = pos + wlo;
          // values this lane writes in the window: i = lane, lane + 32, ... < wn
          const uint32_t n = wn > lane ? (wn - 1 - lane) / 32 + 1 : 0u;
          uint32_t soff = 0;
          if (kWire) {
            // entry = the survivor's bit position in its 4-word block's
            // interleaved masks: the low byte of 64 * lane + bit
            uint8_t* dst8 = P.out8 + wpos;
#pragma unroll 4
            for (uint32_t i = lane; i < wn; i += 32) {
              const uint32_t e = stage[i];
              const uint32_t bb = e & 63u;
              const uint32_t off = 192u * (e >> 6) + 3u * bb + 1u + (bb & 1u);
              if (seg_fits || wpos + i < P.out_cap) dst8[i] = static_cast<uint8_t>(e);
              soff += off;
              xr ^= rbase + off;
            }
          } else if (seg_fits && nocarry) {
            uint2* dst = reinterpret_cast<uint2*>(P.out + wpos);
            uint32_t xlo = 0;
#pragma unroll 4
            for (uint32_t i = lane; i < wn; i += 32) {
              const uint32_t off = stage[i];
              const uint32_t vlo = rlo + off;
              dst[i] = make_uint2(vlo, rhi);
              soff += off;
              xlo ^= vlo;
            }
            xr ^= (static_cast<unsigned long long>(n & 1u ? rhi : 0u) << 32) | xlo;
          } else {
            unsigned long long* dst = P.out + wpos;
            for (uint32_t i = lane; i < wn; i += 32) {
              const uint32_t off = stage[i];
              const unsigned long long v = rbase + off;
              if (seg_fits || wpos + i < P.out_cap) dst[i] = v;
              soff += off;
              xr ^= v;
            }
          }
          sum += rbase * n + soff;
          __syncwarp();
        }
        pos += rtotal;
      }
      if (warp == 0) lg = segment_largest(si, bm1, bm5, vbase, lane);
      sum = warp_sum64(sum);
      xr = warp_xor64(xr);
      lg = warp_max64(lg);
      if (lane == 0) {
        red_a[warp] = sum;
        red_b[warp] = xr;
        red_c[warp] = lg;
      }
      __syncthreads();
      if (warp == 0) {
        unsigned long long su = lane < kWarps ? red_a[lane] : 0ull;
        unsigned long long x = lane < kWarps ? red_b[lane] : 0ull;
        unsigned long long l = lane < kWarps ? red_c[lane] : 0ull;
        su = warp_sum64(su);
        x = warp_xor64(x);
        l = warp_max64(l);
        if (lane == 0) {
          JobAcc& A = P.acc[si.job];
          atomicAdd(&A.sum, su);
          atomicXor(&A.xr, x);
          if (l) atomicMax(&A.largest, l);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Wide count kernel: one 1024-thread CTA per SM owns P.wide consecutive
// segments (2 or 3: 128 or 192 KiB of flags) as ONE sieving unit, so every
// per-(prime, unit) cost -- offsets, loop set-up, the single-hit checks, the
// p and 1/p loads -- is paid once per P.wide segments.  A lone CTA per SM has
// no sibling to cover its barriers, so the unit loop is cut to two barriers:
//   A: flags stamped          -> mark (sieve_primes)
//   B: marks complete         -> count unit u and stamp unit u+1 in ONE pass
//                                (each thread reads word w of u, then overwrites
//                                it with u+1's pattern: no barrier in between)
// The next unit's ticket and geometry are fetched by thread 0 during the
// marking, and the unit's totals gather in shared accumulators that thread 0
// flushes after barrier A.  Per-segment counts stay per S-slot segment.
// Count modes only (host-side gate).  Launches over bucket windows or several
// jobs bring a unit table (units never straddle a job or a window); a unit
// applies the bucket lists of each of its segments.
constexpr int kWideThreads = 1024;

__device__ void fetch_unit(const SieveParams& P, SegInfo& si) {
  const uint64_t nunits = P.units ? P.nunits : (P.s_count + P.wide - 1) / P.wide;
  const unsigned long long t = atomicAdd(P.ticket, 1ull);
  if (t >= nunits) {
    si.s = ~0ull;
    if (atomicAdd(P.ticket + 1, 1ull) == gridDim.x - 1) {  // see fetch_segment
      P.ticket[0] = 0;
      P.ticket[1] = 0;
    }
    return;
  }
  // the unit's first segment and segment count: analytic for one job without
  // windows, else from the launch's unit table (units never straddle a job
  // or a window): first window-local segment | count << 28
  uint64_t first = t * P.wide;
  uint32_t cnt = P.wide;
  if (P.units) {
    const uint32_t e = __ldg(P.units + t);
    first = e & 0x0FFFFFFFu;
    cnt = e >> 28;
  }
  const uint64_t s = P.s_begin + first;
  uint32_t lo = 0;
  Job J;
  if (P.njobs == 1) {
    J = P.job0;
  } else {
    uint32_t hi = P.njobs;  // last job with seg_begin <= s
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (P.jobs[mid].seg_begin <= s) lo = mid; else hi = mid;
    }
    J = P.jobs[lo];
  }
  si.s = s;
  si.job = lo;
  const uint64_t local = s - J.seg_begin;
  si.ks = J.K0 + local * P.S;
  const uint64_t rem = J.nslots - local * P.S;
  const uint64_t cap = static_cast<uint64_t>(cnt) * P.S;
  si.len = rem < cap ? static_cast<uint32_t>(rem) : static_cast<uint32_t>(cap);
  si.lo1 = first_valid(si.ks, 1, J.L);
  if (si.ks == 0 && si.lo1 < 1) si.lo1 = 1;
  si.lo5 = first_valid(si.ks, 5, J.L);
  si.hi1 = end_valid(si.ks, 1, J.R, si.len);
  si.hi5 = end_valid(si.ks, 5, J.R, si.len);
  si.nwords = ((si.len + 1023u) / 1024u) * 32u;
  si.t_lo = isqrt64(6 * si.ks);
  si.t_hi = isqrt64(6 * (si.ks + si.len));
}

struct WideAcc {
  unsigned long long lg, sum, xr;
  uint32_t cnt[4];
};

template <int MODE, bool BK>
__global__ void __launch_bounds__(kWideThreads, 1) sieve_wide_kernel(const SieveParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t wps = P.S / 32;  // words per class per segment (a multiple of kWideThreads)
  uint32_t* bm1 = smem;
  uint32_t* bm5 = smem + P.wide * wps;
  const uint2* tab1 = reinterpret_cast<const uint2*>(P.small_tab);
  const uint2* tab5 = tab1 + kTabPerClass;
  __shared__ SegInfo sis[2];
  __shared__ WideAcc acc;
  __shared__ uint32_t wc_ctr;
  const uint32_t lane = threadIdx.x & 31u;
  constexpr uint32_t kStride = 32u * kWideThreads;

  const uint32_t nprimes = P.nprimes_dev ? min(P.nprimes, *P.nprimes_dev) : P.nprimes;
  if (P.tabn_out != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *P.tabn_out = nprimes;
  if (threadIdx.x == 0) {
    fetch_unit(P, sis[0]);
    wc_ctr = 0;
    acc.lg = acc.sum = acc.xr = 0;
    acc.cnt[0] = acc.cnt[1] = acc.cnt[2] = acc.cnt[3] = 0;
  }
  __syncthreads();
  if (sis[0].s == ~0ull) return;

  // counts unit `o` (if any) and stamps unit `n` (if any) in one pass
  auto count_and_stamp = [&](const SegInfo* o, const SegInfo* n) {
    const uint32_t o_words = o ? o->nwords : 0u, n_words = n ? n->nwords : 0u;
    uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
    bool edge = false;
    if (n) {
      const uint64_t k = n->ks + 32u * threadIdx.x;
      a0 = static_cast<uint32_t>(k % 5005u);
      a1 = static_cast<uint32_t>(k % 7429u);
      a2 = static_cast<uint32_t>(k % 899u);
      a3 = static_cast<uint32_t>(k % 1517u);
      a4 = static_cast<uint32_t>(k % 2021u);
      const uint32_t full = 32u * n_words;
      edge = n->lo1 != 0 || n->lo5 != 0 || n->hi1 != full || n->hi5 != full || n->ks < 8;
    }
    const unsigned long long vbase = o ? 6 * o->ks : 0ull;
    unsigned long long sum = 0, xr = 0;
    uint32_t top_w = 0, top1 = 0, top5 = 0;  // the thread's last word with a survivor
    const uint32_t end_words = max(o_words, n_words);
    for (uint32_t part = 0; part * wps < end_words; ++part) {
      uint32_t cnt = 0;
      const uint32_t w_end = min((part + 1) * wps, end_words);
      for (uint32_t w = part * wps + threadIdx.x; w < w_end; w += kWideThreads) {
        if (w < o_words) {
          const uint32_t m1 = ~bm1[w], m5 = ~bm5[w];
          cnt += __popc(m1) + __popc(m5);
          if (m1 | m5) {
            top_w = w;
            top1 = m1;
            top5 = m5;
            if (MODE == kCountChecks) {
              const unsigned long long wb = vbase + 192ull * w;
              for (uint32_t x = m1; x; x &= x - 1) {
                const unsigned long long v = wb + 6ull * (__ffs(x) - 1) + 1;
                sum += v;
                xr ^= v;
              }
              for (uint32_t x = m5; x; x &= x - 1) {
                const unsigned long long v = wb + 6ull * (__ffs(x) - 1) + 5;
                sum += v;
                xr ^= v;
              }
            }
          }
        }
        if (w < n_words) {  // see init_words
          uint32_t m1 = tab_read(tab1, a0) & tab_read(tab1 + tab_off(1), a1) &
                        tab_read(tab1 + tab_off(2), a2) & tab_read(tab1 + tab_off(3), a3) &
                        tab_read(tab1 + tab_off(4), a4);
          uint32_t m5 = tab_read(tab5, a0) & tab_read(tab5 + tab_off(1), a1) &
                        tab_read(tab5 + tab_off(2), a2) & tab_read(tab5 + tab_off(3), a3) &
                        tab_read(tab5 + tab_off(4), a4);
          a0 = phase_step(a0, kStride % 5005u, 5005u);
          a1 = phase_step(a1, kStride % 7429u, 7429u);
          a2 = phase_step(a2, kStride % 899u, 899u);
          a3 = phase_step(a3, kStride % 1517u, 1517u);
          a4 = phase_step(a4, kStride % 2021u, 2021u);
          if (edge) {
            if (w == 0 && n->ks < 8) {
              m1 |= 0xEEu >> n->ks;
              m5 |= 0xDFu >> n->ks;
            }
            const int64_t base = 32 * static_cast<int64_t>(w);
            m1 &= range_mask(static_cast<int64_t>(n->lo1) - base,
                             static_cast<int64_t>(n->hi1) - base);
            m5 &= range_mask(static_cast<int64_t>(n->lo5) - base,
                             static_cast<int64_t>(n->hi5) - base);
          }
          bm1[w] = ~m1;
          bm5[w] = ~m5;
        }
      }
      if (o) {
        cnt = __reduce_add_sync(kFull, cnt);
        if (lane == 0 && cnt) atomicAdd(&acc.cnt[part], cnt);
      }
    }
    if (o) {
      unsigned long long lg = 0;
      if (top1 | top5) {
        const unsigned long long wb = vbase + 192ull * top_w;
        const unsigned long long v1 = top1 ? wb + 6ull * (31 - __clz(top1)) + 1 : 0;
        const unsigned long long v5 = top5 ? wb + 6ull * (31 - __clz(top5)) + 5 : 0;
        lg = v1 > v5 ? v1 : v5;
      }
      lg = warp_max64(lg);
      if (MODE == kCountChecks) {
        sum = warp_sum64(sum);
        xr = warp_xor64(xr);
      }
      if (lane == 0) {
        if (lg) atomicMax(&acc.lg, lg);
        if (MODE == kCountChecks) {
          atomicAdd(&acc.sum, sum);
          atomicXor(&acc.xr, xr);
        }
      }
    }
  };
  // thread 0: the finished unit's totals to the job accumulators
  auto flush = [&](const SegInfo& o) {
    JobAcc& A = P.acc[o.job];
    unsigned long long total = 0;
    for (uint32_t part = 0; part < P.wide; ++part) {
      if (part * P.S < o.len) {
        if (P.per_seg) P.per_seg[o.s + part] = acc.cnt[part];
        if (BK && P.bucket) P.bcount[o.s - P.s_begin + part] = 0;  // list consumed
        total += acc.cnt[part];
      }
      acc.cnt[part] = 0;
    }
    if (total) {
      atomicAdd(&A.count, total);
      atomicMax(&A.largest, acc.lg);
      if (MODE == kCountChecks) {
        atomicAdd(&A.sum, acc.sum);
        atomicXor(&A.xr, acc.xr);
      }
    }
    acc.lg = acc.sum = acc.xr = 0;
  };

  count_and_stamp(nullptr, &sis[0]);
  uint32_t cur = 0;
  bool pending = false;  // thread 0: unit cur^1 is counted but not flushed
  for (;;) {
    __syncthreads();  // A
    if (threadIdx.x == 0) {
      if (pending) flush(sis[cur ^ 1]);
      fetch_unit(P, sis[cur ^ 1]);
    }
    sieve_primes<kWideThreads, true, true, BK>(P, sis[cur], bm1, bm5, &wc_ctr, nprimes);
    __syncthreads();  // B
    const bool more = sis[cur ^ 1].s != ~0ull;
    if (threadIdx.x == 0) wc_ctr = 0;
    count_and_stamp(&sis[cur], more ? &sis[cur ^ 1] : nullptr);
    pending = true;
    cur ^= 1;
    if (!more) break;
  }
  __syncthreads();
  if (threadIdx.x == 0) flush(sis[cur ^ 1]);
}

// ---------------------------------------------------------------------------
// Large-prime bucket fill.  blockIdx.y = run, blockIdx.x = chunk of
// kFillThreads * kFillPrimesPerThread primes.  Two passes over the same hits:
// (1) per-segment histogram in shared memory, (2) one global atomicAdd per
// (block, segment) reserves a contiguous slice of that segment's list, then
// every hit is written into it.  First hits use the same Barrett offsets and
// p*p activation rule as the sieve kernel.
__global__ void __launch_bounds__(kFillThreads) bucket_fill_kernel(const FillParams F) {
  extern __shared__ uint32_t fill_smem[];
  uint32_t* hist = fill_smem;                       // max_run_segs counters
  uint32_t* first1 = fill_smem + F.max_run_segs;    // per prime: first hit (run-relative)
  uint32_t* first5 = first1 + kFillPrimesPerBlock;  // UINT32_MAX = no hit in this run
  const Run run = F.runs[blockIdx.y];
  const uint32_t S = 1u << F.log2S;
  const uint32_t span = static_cast<uint32_t>(run.k_hi - run.k_lo);  // <= kMaxWindow * S
  // activation thresholds of the run (see fetch_segment)
  const uint32_t t_lo = isqrt64(6 * run.k_lo), t_hi = isqrt64(6 * run.k_hi);
  const uint32_t first = F.p_begin + blockIdx.x * kFillPrimesPerBlock;
  const uint32_t p_end = F.nprimes_dev ? min(F.p_end, *F.nprimes_dev) : F.p_end;
  // primes ascend: a block whose first prime is not active anywhere in the
  // run (p*p beyond its end) has no hits -- common when the jobs of a window
  // need different base bounds (c5's intervals)
  if (first >= p_end || __ldg(F.prime_p + first) > t_hi) return;
  const ModCtx mc = mod_ctx(run.k_lo);
  for (uint32_t i = threadIdx.x; i < run.nseg; i += kFillThreads) hist[i] = 0;
  __syncthreads();
  // pass 1: first hits (Barrett, p*p activation) + per-segment histogram;
  // p and 1/p are loaded one prime ahead (independent of the run)
  uint32_t pn = 0;
  double ipn = 0.0;
  if (first + threadIdx.x < p_end) {
    pn = __ldg(F.prime_p + first + threadIdx.x);
    ipn = __ldg(F.prime_inv + first + threadIdx.x);
  }
#pragma unroll 1
  for (int j = 0; j < kFillPrimesPerThread; ++j) {
    const uint32_t li = j * kFillThreads + threadIdx.x;
    const uint32_t i = first + li;
    uint32_t r1 = 0xFFFFFFFFu, r5 = 0xFFFFFFFFu;
    const uint32_t p = pn;
    const double ip = ipn;
    if (i + kFillThreads < p_end && j + 1 < kFillPrimesPerThread) {
      pn = __ldg(F.prime_p + i + kFillThreads);
      ipn = __ldg(F.prime_inv + i + kFillThreads);
    }
    if (i < p_end) {
      uint32_t q1, q5;
      if (prime_offsets(p, ip, i, F.prime_m, mc, t_lo, t_hi, q1, q5)) {
        if (q1 < span) r1 = q1;
        if (q5 < span) r5 = q5;
        if (p <= 0xFFFFFFFFu - span) {  // 32-bit stepping cannot wrap
          for (uint32_t h = r1; h < span; h += p) atomicAdd(hist + (h >> F.log2S), 1u);
          for (uint32_t h = r5; h < span; h += p) atomicAdd(hist + (h >> F.log2S), 1u);
        } else {  // p within `span` of 2^32 (top of the 64-bit value range)
          for (uint64_t h = r1; h < span; h += p) atomicAdd(hist + (h >> F.log2S), 1u);
          for (uint64_t h = r5; h < span; h += p) atomicAdd(hist + (h >> F.log2S), 1u);
        }
      }
    }
    first1[li] = r1;
    first5[li] = r5;
  }
  __syncthreads();
  // reserve one contiguous slice per (block, segment); the cursor becomes
  // the slice's window-global entry index (the window holds < 2^32 entries)
  for (uint32_t i = threadIdx.x; i < run.nseg; i += kFillThreads) {
    const uint32_t c = hist[i];
    hist[i] = (run.seg0 + i) * F.bcap + (c ? atomicAdd(F.bcount + run.seg0 + i, c) : 0u);
  }
  __syncthreads();
  // pass 2: write the entries; p is loaded one prime ahead (a plain load at
  // the point of use stalled every prime's first hit on global latency)
  uint32_t pw = first + threadIdx.x < p_end ? __ldg(F.prime_p + first + threadIdx.x) : 0u;
#pragma unroll 1
  for (int j = 0; j < kFillPrimesPerThread; ++j) {
    const uint32_t li = j * kFillThreads + threadIdx.x;
    const uint32_t i = first + li;
    if (i >= p_end) break;
    const uint32_t p = pw;
    if (i + kFillThreads < p_end && j + 1 < kFillPrimesPerThread)
      pw = __ldg(F.prime_p + i + kFillThreads);
    uint32_t h1 = first1[li], h5 = first5[li];
    if (h1 == 0xFFFFFFFFu && h5 == 0xFFFFFFFFu) continue;
    // an entry is written while its segment's list has room: index below
    // the end of the segment's list (overflow is detected by the sieve)
    auto put = [&](uint32_t seg, uint32_t entry) {
      const uint32_t idx = atomicAdd(hist + seg, 1u);
      if (idx < (run.seg0 + seg + 1) * F.bcap) F.bucket[idx] = entry;
    };
    if (p <= 0xFFFFFFFFu - span && !F.w_unroll) {
      for (uint32_t h = h1; h < span; h += p) put(h >> F.log2S, h & (S - 1));
      for (uint32_t h = h5; h < span; h += p) put(h >> F.log2S, (h & (S - 1)) | S);
    } else if (p <= 0xFFFFFFFFu - span) {
      // both classes and two hits of each per step: p >= 2S puts consecutive
      // hits in different segments, so the four cursor atomics are
      // independent and their round trips overlap (one at a time, every
      // store waited for its own atomic)
      while (h1 < span || h5 < span) {
        const bool a = h1 < span, b = h5 < span;
        const uint32_t g1 = h1 + p, g5 = h5 + p;  // no wrap: h < span <= 2^32 - 1 - p
        const bool a2 = a && g1 < span, b2 = b && g5 < span;
        uint32_t i1 = 0, j1 = 0, i5 = 0, j5 = 0;
        if (a) i1 = atomicAdd(hist + (h1 >> F.log2S), 1u);
        if (a2) j1 = atomicAdd(hist + (g1 >> F.log2S), 1u);
        if (b) i5 = atomicAdd(hist + (h5 >> F.log2S), 1u);
        if (b2) j5 = atomicAdd(hist + (g5 >> F.log2S), 1u);
        auto store = [&](bool ok, uint32_t idx, uint32_t h, uint32_t cls) {
          if (ok && idx < (run.seg0 + (h >> F.log2S) + 1) * F.bcap)
            F.bucket[idx] = (h & (S - 1)) | cls;
        };
        store(a, i1, h1, 0u);
        store(a2, j1, g1, 0u);
        store(b, i5, h5, S);
        store(b2, j5, g5, S);
        h1 = a2 ? g1 + p : 0xFFFFFFFFu;  // g1 < span: g1 + p cannot wrap either
        h5 = b2 ? g5 + p : 0xFFFFFFFFu;
      }
    } else {
      const uint32_t r1 = h1, r5 = h5;
      for (uint64_t h = r1; h < span; h += p)
        put(static_cast<uint32_t>(h >> F.log2S), static_cast<uint32_t>(h) & (S - 1));
      for (uint64_t h = r5; h < span; h += p)
        put(static_cast<uint32_t>(h >> F.log2S), (static_cast<uint32_t>(h) & (S - 1)) | S);
    }
  }
}

// ---------------------------------------------------------------------------
// Bucket fill for primes p >= the run length (runs of 32 segments: p >= 32 S),
// which hit a run at most once per class.  bucket_fill_kernel would redo the
// per-(prime, run) setup -- loads, first-hit arithmetic, two passes of loop
// control -- for ~1 hit; here blockIdx.y takes F.group_runs consecutive runs
// of one job, the first hits are computed once at the group's start, kept in
// shared memory and advanced by p after each hit.  Per run: a histogram pass,
// one reservation per segment, a write pass -- the same per-run write locality
// as bucket_fill_kernel.
__global__ void __launch_bounds__(kFillThreads) bucket_fill_huge_kernel(const FillParams F) {
  extern __shared__ uint32_t fill_smem[];
  uint32_t* hist = fill_smem;                       // max_run_segs counters
  uint32_t* next1 = fill_smem + F.max_run_segs;     // per prime: next hit (group-relative)
  uint32_t* next5 = next1 + kFillPrimesPerBlock;    // UINT32_MAX = none in this group
  const uint32_t r_begin = blockIdx.y * F.group_runs;
  const uint32_t r_end = min(F.nruns, r_begin + F.group_runs);
  const uint64_t g_lo = F.runs[r_begin].k_lo, g_hi = F.runs[r_end - 1].k_hi;
  const uint32_t S = 1u << F.log2S;
  const uint32_t t_lo = isqrt64(6 * g_lo), t_hi = isqrt64(6 * g_hi);
  const ModCtx mc = mod_ctx(g_lo);
  const uint32_t gspan = static_cast<uint32_t>(g_hi - g_lo);  // < 2^31 (host bound)
  const uint32_t first = F.p_begin + blockIdx.x * kFillPrimesPerBlock;
  const uint32_t p_end = F.nprimes_dev ? min(F.p_end, *F.nprimes_dev) : F.p_end;
  uint32_t pp[kFillPrimesPerThread];  // the thread's primes stay in registers
#pragma unroll
  for (int j = 0; j < kFillPrimesPerThread; ++j) {
    const uint32_t li = j * kFillThreads + threadIdx.x;
    const uint32_t i = first + li;
    uint32_t r1 = 0xFFFFFFFFu, r5 = 0xFFFFFFFFu;
    pp[j] = 0;
    if (i < p_end) {
      pp[j] = __ldg(F.prime_p + i);
      uint32_t q1, q5;
      if (prime_offsets(pp[j], __ldg(F.prime_inv + i), i, F.prime_m, mc, t_lo, t_hi, q1, q5)) {
        if (q1 < gspan) r1 = q1;
        if (q5 < gspan) r5 = q5;
      }
    }
    next1[li] = r1;
    next5[li] = r5;
  }
  // F.huge_step consecutive runs at a time (one histogram over their
  // segments): at most huge_step hits per class per step
#pragma unroll 1
  for (uint32_t r = r_begin; r < r_end; r += F.huge_step) {
    const uint32_t r2 = min(r_end, r + F.huge_step) - 1;
    Run run = F.runs[r];
    run.k_hi = F.runs[r2].k_hi;
    run.nseg = F.runs[r2].seg0 + F.runs[r2].nseg - run.seg0;
    const uint32_t lo = static_cast<uint32_t>(run.k_lo - g_lo);
    const uint32_t hi = static_cast<uint32_t>(run.k_hi - g_lo);
    for (uint32_t k = threadIdx.x; k < run.nseg; k += kFillThreads) hist[k] = 0;
    __syncthreads();  // also orders the previous step's reservations
#pragma unroll
    for (int j = 0; j < kFillPrimesPerThread; ++j) {
      const uint32_t li = j * kFillThreads + threadIdx.x;
      // h < hi < 2^31 and p < 2^32: the 64-bit step cannot wrap
      for (uint64_t h = next1[li]; h < hi; h += pp[j]) atomicAdd(hist + ((h - lo) >> F.log2S), 1u);
      for (uint64_t h = next5[li]; h < hi; h += pp[j]) atomicAdd(hist + ((h - lo) >> F.log2S), 1u);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < run.nseg; k += kFillThreads) {
      const uint32_t c = hist[k];
      hist[k] = (run.seg0 + k) * F.bcap + (c ? atomicAdd(F.bcount + run.seg0 + k, c) : 0u);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kFillPrimesPerThread; ++j) {
      const uint32_t li = j * kFillThreads + threadIdx.x;
#pragma unroll
      for (int cls = 0; cls < 2; ++cls) {
        uint32_t* slot = (cls ? next5 : next1) + li;
        uint32_t h = *slot;
        if (h < hi) {
          do {
            const uint32_t seg = (h - lo) >> F.log2S;
            const uint32_t idx = atomicAdd(hist + seg, 1u);
            if (idx < (run.seg0 + seg + 1) * F.bcap)
              F.bucket[idx] = ((h - lo) & (S - 1)) | (cls ? S : 0u);
            const uint32_t n = h + pp[j];  // next hit, or none in this group
            h = n >= h && n < gspan ? n : 0xFFFFFFFFu;
          } while (h < hi);
          *slot = h;
        }
      }
    }
    __syncthreads();  // hist is reset for the next run
  }
}

// bucket_fill_huge_kernel for one run per step (the default): a prime of at
// least the run length hits a run at most once per class, so each (prime,
// class) is one predicated check per run -- no hit loop, so no warp runs to
// the busiest lane's trip count -- and the next hits stay in registers
// (16 primes x 2 classes per thread) instead of shared memory.
__global__ void __launch_bounds__(kFillThreads) bucket_fill_huge1_kernel(const FillParams F) {
  extern __shared__ uint32_t fill_smem[];
  uint32_t* hist = fill_smem;  // max_run_segs counters, then the run's list cursors
  const uint32_t r_begin = blockIdx.y * F.group_runs;
  const uint32_t r_end = min(F.nruns, r_begin + F.group_runs);
  const uint64_t g_lo = F.runs[r_begin].k_lo, g_hi = F.runs[r_end - 1].k_hi;
  const uint32_t S = 1u << F.log2S;
  const uint32_t t_lo = isqrt64(6 * g_lo), t_hi = isqrt64(6 * g_hi);
  const ModCtx mc = mod_ctx(g_lo);
  const uint32_t gspan = static_cast<uint32_t>(g_hi - g_lo);  // < 2^31 (host bound)
  const uint32_t first = F.p_begin + blockIdx.x * kFillPrimesPerBlock;
  const uint32_t p_end = F.nprimes_dev ? min(F.p_end, *F.nprimes_dev) : F.p_end;
  uint32_t pp[kFillPrimesPerThread], n1[kFillPrimesPerThread], n5[kFillPrimesPerThread];
#pragma unroll
  for (int j = 0; j < kFillPrimesPerThread; ++j) {
    const uint32_t i = first + j * kFillThreads + threadIdx.x;
    pp[j] = 0;
    n1[j] = n5[j] = 0xFFFFFFFFu;
    if (i < p_end) {
      pp[j] = __ldg(F.prime_p + i);
      uint32_t q1, q5;
      if (prime_offsets(pp[j], __ldg(F.prime_inv + i), i, F.prime_m, mc, t_lo, t_hi, q1, q5)) {
        if (q1 < gspan) n1[j] = q1;
        if (q5 < gspan) n5[j] = q5;
      }
    }
  }
#pragma unroll 1
  for (uint32_t r = r_begin; r < r_end; ++r) {
    const Run run = F.runs[r];
    const uint32_t lo = static_cast<uint32_t>(run.k_lo - g_lo);
    const uint32_t hi = static_cast<uint32_t>(run.k_hi - g_lo);
    for (uint32_t k = threadIdx.x; k < run.nseg; k += kFillThreads) hist[k] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kFillPrimesPerThread; ++j) {
      if (n1[j] < hi) atomicAdd(hist + ((n1[j] - lo) >> F.log2S), 1u);
      if (n5[j] < hi) atomicAdd(hist + ((n5[j] - lo) >> F.log2S), 1u);
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < run.nseg; k += kFillThreads) {
      const uint32_t c = hist[k];
      hist[k] = (run.seg0 + k) * F.bcap + (c ? atomicAdd(F.bcount + run.seg0 + k, c) : 0u);
    }
    __syncthreads();
    auto put = [&](uint32_t& h, uint32_t p, uint32_t cls_bit) {
      if (h < hi) {
        const uint32_t rel = h - lo;
        const uint32_t seg = rel >> F.log2S;
        const uint32_t idx = atomicAdd(hist + seg, 1u);
        if (idx < (run.seg0 + seg + 1) * F.bcap) F.bucket[idx] = (rel & (S - 1)) | cls_bit;
        const uint32_t n = h + p;  // the next hit is past this run (p >= its span)
        h = n >= h && n < gspan ? n : 0xFFFFFFFFu;
      }
    };
#pragma unroll
    for (int j = 0; j < kFillPrimesPerThread; ++j) {
      put(n1[j], pp[j], 0u);
      put(n5[j], pp[j], S);
    }
    __syncthreads();  // every cursor is used before the next run clears hist
  }
}

// ---------------------------------------------------------------------------
// Staged fills.  The two-pass fills above store every hit straight to its
// segment's list: the 32 lanes of a store hit 32 different lists, so each
// warp store is 32 separate L1 wavefronts and 32 partial L2 sectors -- about
// one data-pipe wavefront per 4-byte entry.  The staged fills queue a batch's
// hits per segment in shared memory (one returning shared atomic + one
// shared store each) and then flush every queue as one contiguous chunk: one
// global reservation (atomicAdd on the segment's count) per (batch, segment)
// and coalesced stores, ~1/32 wavefront per entry.  No histogram pass: the
// reservation happens at flush time.  A queue that fills up sends its extra
// hits down the direct path (one global atomic each), so any cap is correct.
// bcount[s] still counts every hit of segment s, written or not, so an
// overflowed list is detected by the sieve exactly as before.

// queue entry `entry` for window segment gseg (run-local seg)
__device__ __forceinline__ void stage_put(const FillParams& F, uint32_t* scnt, uint32_t* stage,
                                          uint32_t cap, uint32_t seg, uint32_t gseg,
                                          uint32_t entry) {
  const uint32_t idx = atomicAdd(scnt + seg, 1u);
  if (idx < cap) {
    stage[seg * cap + idx] = entry;
  } else {
    const uint32_t g = atomicAdd(F.bcount + gseg, 1u);
    if (g < F.bcap) F.bucket[gseg * F.bcap + g] = entry;
  }
}

// every queue of the run's nseg segments to its list, queues left empty.
// Called by the whole block right after a __syncthreads that ends the puts.
// Reservations first, all in flight together (one global atomic per
// non-empty queue, one thread each: a single round trip), then every warp
// copies whole queues with coalesced stores.  sbase: nseg words of scratch.
// Ends with a __syncthreads (the queues are empty for the next puts).
__device__ __forceinline__ void stage_flush(const FillParams& F, uint32_t* scnt, uint32_t* sbase,
                                            const uint32_t* stage, uint32_t cap, uint32_t seg0,
                                            uint32_t nseg) {
  for (uint32_t s = threadIdx.x; s < nseg; s += kFillThreads) {
    const uint32_t c = scnt[s];
    const uint32_t n = c < cap ? c : cap;
    scnt[s] = n;
    sbase[s] = n ? atomicAdd(F.bcount + seg0 + s, n) : 0u;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint32_t s = warp; s < nseg; s += kFillThreads / 32) {
    const uint32_t n = scnt[s], base = sbase[s];
    if (base >= F.bcap) continue;
    const uint32_t lim = F.bcap - base < n ? F.bcap - base : n;
    uint32_t* dst = F.bucket + (seg0 + s) * F.bcap + base;
    const uint32_t* src = stage + s * cap;
    for (uint32_t i = lane; i < lim; i += 32) dst[i] = src[i];
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < nseg; s += kFillThreads) scnt[s] = 0;
  __syncthreads();  // the queues are empty again
}

// bucket_fill_kernel, staged: a batch is one prime per thread (256 primes);
// each batch's hits over the run are queued, then flushed.
__global__ void __launch_bounds__(kFillThreads) bucket_fill_staged_kernel(const FillParams F) {
  extern __shared__ uint32_t fill_smem[];
  uint32_t* scnt = fill_smem;                        // max_run_segs queue lengths
  uint32_t* sbase = fill_smem + F.max_run_segs;      // ... and their list reservations
  uint32_t* stage = fill_smem + 2 * F.max_run_segs;  // max_run_segs queues of stage_cap entries
  const uint32_t cap = F.stage_cap;
  const Run run = F.runs[blockIdx.y];
  const uint32_t S = 1u << F.log2S;
  const uint32_t span = static_cast<uint32_t>(run.k_hi - run.k_lo);  // < 2^32 (host bound)
  const uint32_t t_lo = isqrt64(6 * run.k_lo), t_hi = isqrt64(6 * run.k_hi);
  const uint32_t first = F.p_begin + blockIdx.x * kFillPrimesPerBlock;
  const uint32_t p_end = F.nprimes_dev ? min(F.p_end, *F.nprimes_dev) : F.p_end;
  if (first >= p_end || __ldg(F.prime_p + first) > t_hi) return;  // see bucket_fill_kernel
  const ModCtx mc = mod_ctx(run.k_lo);
  for (uint32_t i = threadIdx.x; i < run.nseg; i += kFillThreads) scnt[i] = 0;
  uint32_t pn = 0;
  double ipn = 0.0;
  if (first + threadIdx.x < p_end) {
    pn = __ldg(F.prime_p + first + threadIdx.x);
    ipn = __ldg(F.prime_inv + first + threadIdx.x);
  }
  // primes per thread per batch: a batch of kb * 256 primes from p0 up puts
  // at most kb * 256 * 2S / p0 hits in a segment's queue on average; keep that
  // near 3/4 of the capacity
  const uint32_t p0 = __ldg(F.prime_p + first);
  const uint32_t kb = max(1u, min(static_cast<uint32_t>(kFillPrimesPerThread),
                                  static_cast<uint32_t>((3ull * cap * p0) / (2048ull * S))));
  __syncthreads();  // the queues are empty
#pragma unroll 1
  for (int j = 0; j < kFillPrimesPerThread; ++j) {
    const uint32_t b0 = first + j * kFillThreads;  // this step's first prime (block-uniform)
    const uint32_t i = b0 + threadIdx.x;
    const uint32_t p = pn;
    const double ip = ipn;
    // primes ascend: once a step's first prime is inactive in the run, so is the rest
    if (b0 >= p_end || __ldg(F.prime_p + b0) > t_hi) break;
    if (i + kFillThreads < p_end && j + 1 < kFillPrimesPerThread) {
      pn = __ldg(F.prime_p + i + kFillThreads);
      ipn = __ldg(F.prime_inv + i + kFillThreads);
    }
    uint32_t q1, q5;
    if (i < p_end && prime_offsets(p, ip, i, F.prime_m, mc, t_lo, t_hi, q1, q5)) {
      if (p <= 0xFFFFFFFFu - span) {  // 32-bit stepping cannot wrap
        for (uint32_t h = q1; h < span; h += p)
          stage_put(F, scnt, stage, cap, h >> F.log2S, run.seg0 + (h >> F.log2S), h & (S - 1));
        for (uint32_t h = q5; h < span; h += p)
          stage_put(F, scnt, stage, cap, h >> F.log2S, run.seg0 + (h >> F.log2S),
                    (h & (S - 1)) | S);
      } else {  // p within `span` of 2^32 (top of the 64-bit value range)
        for (uint64_t h = q1; h < span; h += p) {
          const uint32_t seg = static_cast<uint32_t>(h >> F.log2S);
          stage_put(F, scnt, stage, cap, seg, run.seg0 + seg, static_cast<uint32_t>(h) & (S - 1));
        }
        for (uint64_t h = q5; h < span; h += p) {
          const uint32_t seg = static_cast<uint32_t>(h >> F.log2S);
          stage_put(F, scnt, stage, cap, seg, run.seg0 + seg,
                    (static_cast<uint32_t>(h) & (S - 1)) | S);
        }
      }
    }
    // flush after every kb-th prime, and after the block's last active one
    const bool last = j + 1 == kFillPrimesPerThread || b0 + kFillThreads >= p_end ||
                      __ldg(F.prime_p + b0 + kFillThreads) > t_hi;
    if ((j + 1) % kb == 0 || last) {
      __syncthreads();
      stage_flush(F, scnt, sbase, stage, cap, run.seg0, run.nseg);
    }
  }
}

// bucket_fill_huge1_kernel, staged: per run, the block's <= 2 hits per prime
// are queued, then flushed (no histogram pass, no reservation pass).
__global__ void __launch_bounds__(kFillThreads) bucket_fill_huge1_staged_kernel(const FillParams F) {
  extern __shared__ uint32_t fill_smem[];
  uint32_t* scnt = fill_smem;
  uint32_t* sbase = fill_smem + F.max_run_segs;
  uint32_t* stage = fill_smem + 2 * F.max_run_segs;
  const uint32_t cap = F.stage_cap;
  const uint32_t r_begin = blockIdx.y * F.group_runs;
  const uint32_t r_end = min(F.nruns, r_begin + F.group_runs);
  const uint64_t g_lo = F.runs[r_begin].k_lo, g_hi = F.runs[r_end - 1].k_hi;
  const uint32_t S = 1u << F.log2S;
  const uint32_t t_lo = isqrt64(6 * g_lo), t_hi = isqrt64(6 * g_hi);
  const ModCtx mc = mod_ctx(g_lo);
  const uint32_t gspan = static_cast<uint32_t>(g_hi - g_lo);  // < 2^31 (host bound)
  const uint32_t first = F.p_begin + blockIdx.x * kFillPrimesPerBlock;
  const uint32_t p_end = F.nprimes_dev ? min(F.p_end, *F.nprimes_dev) : F.p_end;
  uint32_t pp[kFillPrimesPerThread], n1[kFillPrimesPerThread], n5[kFillPrimesPerThread];
#pragma unroll
  for (int j = 0; j < kFillPrimesPerThread; ++j) {
    const uint32_t i = first + j * kFillThreads + threadIdx.x;
    pp[j] = 0;
    n1[j] = n5[j] = 0xFFFFFFFFu;
    if (i < p_end) {
      pp[j] = __ldg(F.prime_p + i);
      uint32_t q1, q5;
      if (prime_offsets(pp[j], __ldg(F.prime_inv + i), i, F.prime_m, mc, t_lo, t_hi, q1, q5)) {
        if (q1 < gspan) n1[j] = q1;
        if (q5 < gspan) n5[j] = q5;
      }
    }
  }
  for (uint32_t k = threadIdx.x; k < F.max_run_segs; k += kFillThreads) scnt[k] = 0;
  __syncthreads();
#pragma unroll 1
  for (uint32_t r = r_begin; r < r_end; ++r) {
    const Run run = F.runs[r];
    const uint32_t lo = static_cast<uint32_t>(run.k_lo - g_lo);
    const uint32_t hi = static_cast<uint32_t>(run.k_hi - g_lo);
    auto put = [&](uint32_t& h, uint32_t p, uint32_t cls_bit) {
      if (h < hi) {
        const uint32_t rel = h - lo;
        const uint32_t seg = rel >> F.log2S;
        stage_put(F, scnt, stage, cap, seg, run.seg0 + seg, (rel & (S - 1)) | cls_bit);
        const uint32_t n = h + p;  // the next hit is past this run (p >= its span)
        h = n >= h && n < gspan ? n : 0xFFFFFFFFu;
      }
    };
#pragma unroll
    for (int j = 0; j < kFillPrimesPerThread; ++j) {
      put(n1[j], pp[j], 0u);
      put(n5[j], pp[j], S);
    }
    __syncthreads();
    stage_flush(F, scnt, sbase, stage, cap, run.seg0, run.nseg);
  }
}

// ---------------------------------------------------------------------------
// Small base tables: a dense sieve of [0, n] (n <= kTinyMax = 2^18) writing
// the primes >= 53 in ascending order with their Barrett constants
// (naive_sieve, wheel.cpp:40-54).  Used as level 0 of the two-level base build
// and, when the whole base bound fits, as the entire build.
// the 95 primes in [5, 512) (sqrt of kTinyMax); 2 and 3 never need marking
// because the compaction keeps only 6k +- 1
constexpr uint32_t kTinyPrimeCount = 95;
__constant__ uint32_t kTinyPrimes[kTinyPrimeCount] = {
      5,   7,  11,  13,  17,  19,  23,  29,  31,  37,  41,  43,  47,  53,  59,  61,
     67,  71,  73,  79,  83,  89,  97, 101, 103, 107, 109, 113, 127, 131, 137, 139,
    149, 151, 157, 163, 167, 173, 179, 181, 191, 193, 197, 199, 211, 223, 227, 229,
    233, 239, 241, 251, 257, 263, 269, 271, 277, 281, 283, 293, 307, 311, 313, 317,
    331, 337, 347, 349, 353, 359, 367, 373, 379, 383, 389, 397, 401, 409, 419, 421,
    431, 433, 439, 443, 449, 457, 461, 463, 467, 479, 487, 491, 499, 503, 509,};

// bit b of word w <-> x = 32 w + b; 32 w = 2 w (mod 6), so the 6k +- 1 mask
// depends on w mod 3
constexpr uint32_t wheel_mask(uint32_t ph) {
  uint32_t m = 0;
  for (uint32_t b = 0; b < 32; ++b) {
    const uint32_t r = (2 * ph + b) % 6;
    if (r == 1 || r == 5) m |= 1u << b;
  }
  return m;
}
constexpr uint32_t kWheelMask0 = wheel_mask(0), kWheelMask1 = wheel_mask(1),
                   kWheelMask2 = wheel_mask(2);

// Block b owns the 8192 numbers [8192 b, 8192 (b + 1)): it crosses off odd
// multiples of the primes up to sqrt(n) in a shared-memory bitmap (one warp
// per prime, lanes on consecutive multiples), publishes its survivor count,
// sums its predecessors' counts (all blocks publish without waiting, so
// there is no chain) and writes its primes at that offset.  Counts are tagged
// with the call's epoch, so the scratch words never need clearing.
constexpr uint32_t kBaseBlockWords = 256;  // 8192 numbers per block, one word per thread

__global__ void __launch_bounds__(kBaseBlockWords) small_base_kernel(
    uint32_t n, uint32_t* out_p, unsigned long long* out_m, double* out_inv,
    uint32_t* out_count, unsigned long long* scratch, uint32_t epoch) {
  __shared__ uint32_t comp[kBaseBlockWords];
  __shared__ uint32_t wsum[kBaseBlockWords / 32];
  __shared__ uint32_t s_prefix;
  const uint32_t b = blockIdx.x, t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  const uint32_t lo = b * 32u * kBaseBlockWords;
  const uint32_t hi = min(lo + 32u * kBaseBlockWords, n + 1);  // numbers [lo, hi)
  comp[t] = 0;
  __syncthreads();
#pragma unroll 1
  for (uint32_t k = warp; k < kTinyPrimeCount; k += kBaseBlockWords / 32) {
    const uint32_t q = kTinyPrimes[k];
    if (q * q > n) break;
    uint32_t j = (lo + q - 1) / q * q;  // first multiple >= lo, made odd, at least q*q
    if (!(j & 1u)) j += q;
    j = max(j, q * q);
    for (j += 2 * q * lane; j < hi; j += 64 * q) atomicOr(&comp[(j - lo) >> 5], 1u << (j & 31u));
  }
  __syncthreads();
  const uint32_t w = lo / 32 + t;  // global word of this thread
  uint32_t v = 0;
  if (32 * w <= n) {
    const uint32_t ph = w % 3;
    v = ~comp[t] & (ph == 0 ? kWheelMask0 : ph == 1 ? kWheelMask1 : kWheelMask2);
    if (w == 0) v = 0;
    if (w == 1) v &= ~((1u << (kFirstTablePrime - 32)) - 1);  // x >= 53
    if (w == n / 32) v &= (2u << (n & 31)) - 1;              // x <= n
  }
  const uint32_t c = __popc(v);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += u;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t ws = lane < kBaseBlockWords / 32 ? wsum[lane] : 0u;
    uint32_t wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= static_cast<uint32_t>(o)) wi += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, wi, 31);
    if (lane < kBaseBlockWords / 32) wsum[lane] = wi - ws;  // exclusive warp offsets
    if (lane == 0)
      st_release(scratch + b, (static_cast<unsigned long long>(epoch) << 32) | total);
    // predecessors' counts (at most 32 blocks precede: n <= 2^18)
    uint32_t pc = 0;
    if (lane < b) {
      unsigned long long x;
      do {
        x = ld_acquire(scratch + lane);
      } while (static_cast<uint32_t>(x >> 32) != epoch);
      pc = static_cast<uint32_t>(x);
    }
    pc = __reduce_add_sync(0xffffffffu, pc);
    if (lane == 0) {
      s_prefix = pc;
      if (b == gridDim.x - 1) *out_count = pc + total;
    }
  }
  __syncthreads();
  uint32_t pos = s_prefix + wsum[warp] + incl - c;
  for (; v; v &= v - 1) {
    const uint32_t x = 32 * w + __ffs(v) - 1;
    out_p[pos] = x;
    out_m[pos] = ~0ull / x;
    out_inv[pos] = 1.0 / static_cast<double>(x);
    ++pos;
  }
}

__global__ void prepare_table_kernel(const unsigned long long* vals, uint64_t skip,
                                     const unsigned long long* n_dev, uint64_t cap,
                                     uint32_t* out_p, unsigned long long* out_m, double* out_inv,
                                     uint32_t* out_n) {
  const uint64_t n = *n_dev < cap ? static_cast<uint64_t>(*n_dev) : cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_n = static_cast<uint32_t>(n > skip ? n - skip : 0);
  for (uint64_t i = skip + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = static_cast<uint32_t>(vals[i]);
    out_p[i - skip] = p;
    out_m[i - skip] = ~0ull / p;
    out_inv[i - skip] = 1.0 / static_cast<double>(p);
  }
}

}  // namespace

// device layout: (word i, word i + 1) pairs, 2 * kTabWords uint32
uint32_t small_table_words() { return 2 * kTabWords; }
void build_small_tables(uint32_t* out) {
  for (uint32_t i = 0; i < kTabWords; ++i) {
    out[2 * i] = table_word(i);
    out[2 * i + 1] = i + 1 < kTabWords ? table_word(i + 1) : 0u;
  }
}

size_t sieve_smem_bytes(uint32_t S, int mode) {
  const size_t base = 2 * (S / 32) * sizeof(uint32_t);
  return base + (mode >= kEnumerate ? mode_smem_extra<kEnumerate>() : 0);
}

cudaError_t sieve_configure(int* blocks_per_sm) {
  cudaError_t e;
  const void* fns[kNumModes] = {reinterpret_cast<const void*>(sieve_kernel<kCount>),
                                reinterpret_cast<const void*>(sieve_kernel<kCountChecks>),
                                reinterpret_cast<const void*>(sieve_kernel<kEnumerate>),
                                reinterpret_cast<const void*>(sieve_kernel<kEnumWire>)};
  const void* fns_t[kNumModes] = {reinterpret_cast<const void*>(sieve_kernel<kCount, true>),
                                  reinterpret_cast<const void*>(sieve_kernel<kCountChecks, true>),
                                  nullptr, nullptr};
  for (int m = 0; m < kNumModes; ++m) {
    const size_t smem = sieve_smem_bytes(1u << 18, m);
    e = cudaFuncSetAttribute(fns[m], cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (fns_t[m] != nullptr) {
      e = cudaFuncSetAttribute(fns_t[m], cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    int b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fns[m], kThreads, smem);
    if (e != cudaSuccess) return e;
    blocks_per_sm[m] = b < 1 ? 1 : b;
  }
  for (const void* f : {reinterpret_cast<const void*>(sieve_wide_kernel<kCount, false>),
                        reinterpret_cast<const void*>(sieve_wide_kernel<kCountChecks, false>),
                        reinterpret_cast<const void*>(sieve_wide_kernel<kCount, true>),
                        reinterpret_cast<const void*>(sieve_wide_kernel<kCountChecks, true>)}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kWideMax * sieve_smem_bytes(1u << 18, kCount)));
    if (e != cudaSuccess) return e;
  }
  // the fill kernels' histograms + per-prime state can pass the 48 KB default
  // (runs up to 4096 segments with WHEELSIEVE_FILL_PIECE)
  for (const void* f : {reinterpret_cast<const void*>(bucket_fill_kernel),
                        reinterpret_cast<const void*>(bucket_fill_huge_kernel),
                        reinterpret_cast<const void*>(bucket_fill_huge1_kernel),
                        reinterpret_cast<const void*>(bucket_fill_staged_kernel),
                        reinterpret_cast<const void*>(bucket_fill_huge1_staged_kernel)}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_sieve(int mode, const SieveParams& p, int grid, cudaStream_t st) {
  if (p.wide > 1) {  // count modes only (host-side gate)
    const size_t wsmem = static_cast<size_t>(p.wide) * sieve_smem_bytes(p.S, kCount);
    if (p.bucket != nullptr) {
      if (mode == kCount)
        sieve_wide_kernel<kCount, true><<<grid, kWideThreads, wsmem, st>>>(p);
      else
        sieve_wide_kernel<kCountChecks, true><<<grid, kWideThreads, wsmem, st>>>(p);
    } else {
      if (mode == kCount)
        sieve_wide_kernel<kCount, false><<<grid, kWideThreads, wsmem, st>>>(p);
      else
        sieve_wide_kernel<kCountChecks, false><<<grid, kWideThreads, wsmem, st>>>(p);
    }
    return cudaGetLastError();
  }
  const size_t smem = sieve_smem_bytes(p.S, mode);
  // count modes: transposed warp-cooperative marking (C1 kernel 0.148 -> 0.138 ms; the
  // enumerate kernels measured no gain: C2 +-0, C4e +0.5%)
  if (p.seg_trans && mode <= kCountChecks) {
    if (mode == kCount)
      sieve_kernel<kCount, true><<<grid, kThreads, smem, st>>>(p);
    else
      sieve_kernel<kCountChecks, true><<<grid, kThreads, smem, st>>>(p);
    return cudaGetLastError();
  }
  switch (mode) {
    case kCount: sieve_kernel<kCount><<<grid, kThreads, smem, st>>>(p); break;
    case kCountChecks: sieve_kernel<kCountChecks><<<grid, kThreads, smem, st>>>(p); break;
    case kEnumerate: sieve_kernel<kEnumerate><<<grid, kThreads, smem, st>>>(p); break;
    default: sieve_kernel<kEnumWire><<<grid, kThreads, smem, st>>>(p); break;
  }
  return cudaGetLastError();
}

// staged fills: the queue capacity that fits the dynamic shared-memory limit
// (kFillSmemMax) with the run's queue lengths, 0 = use the two-pass kernels
constexpr size_t kFillSmemMax = 96 * 1024;
uint32_t stage_cap_for(const FillParams& f) {
  if (f.stage_cap == 0 || f.max_run_segs == 0) return 0;
  const size_t words = kFillSmemMax / sizeof(uint32_t);
  if (words <= 2 * f.max_run_segs) return 0;
  const size_t fit = (words - 2 * f.max_run_segs) / f.max_run_segs;
  const uint32_t cap = static_cast<uint32_t>(fit < f.stage_cap ? fit : f.stage_cap);
  return cap >= 32 ? cap : 0;
}
size_t stage_smem(const FillParams& f) {
  return static_cast<size_t>(f.max_run_segs) * (2 + f.stage_cap) * sizeof(uint32_t);
}

cudaError_t launch_bucket_fill_huge(const FillParams& f, cudaStream_t st) {
  const uint32_t per_block = kFillThreads * kFillPrimesPerThread;
  const uint32_t nb = f.p_end > f.p_begin ? (f.p_end - f.p_begin + per_block - 1) / per_block : 0;
  if (nb == 0 || f.nruns == 0 || f.group_runs == 0) return cudaSuccess;
  dim3 grid(nb, (f.nruns + f.group_runs - 1) / f.group_runs);
  if (f.huge_step == 1 && !f.huge_loop) {
    if (const uint32_t cap = stage_cap_for(f)) {
      FillParams g = f;
      g.stage_cap = cap;
      bucket_fill_huge1_staged_kernel<<<grid, kFillThreads, stage_smem(g), st>>>(g);
      return cudaGetLastError();
    }
    bucket_fill_huge1_kernel<<<grid, kFillThreads, f.max_run_segs * sizeof(uint32_t), st>>>(f);
    return cudaGetLastError();
  }
  const size_t smem = (f.max_run_segs + 2 * kFillPrimesPerBlock) * sizeof(uint32_t);
  bucket_fill_huge_kernel<<<grid, kFillThreads, smem, st>>>(f);
  return cudaGetLastError();
}

cudaError_t launch_bucket_fill(const FillParams& f, cudaStream_t st) {
  const uint32_t per_block = kFillThreads * kFillPrimesPerThread;
  const uint32_t nb = (f.p_end - f.p_begin + per_block - 1) / per_block;
  if (nb == 0 || f.nruns == 0) return cudaSuccess;
  dim3 grid(nb, f.nruns);
  if (const uint32_t cap = stage_cap_for(f)) {
    FillParams g = f;
    g.stage_cap = cap;
    bucket_fill_staged_kernel<<<grid, kFillThreads, stage_smem(g), st>>>(g);
    return cudaGetLastError();
  }
  const size_t smem = (f.max_run_segs + 2 * kFillPrimesPerBlock) * sizeof(uint32_t);
  bucket_fill_kernel<<<grid, kFillThreads, smem, st>>>(f);
  return cudaGetLastError();
}

// Copies n job accumulators to mapped pinned host memory with plain stores
// (no copy engine: the pipelined enumeration keeps the D2H engine busy with
// chunk payloads, and a queued 32-byte copy would stall the compute stream).
__global__ void acc_to_host_kernel(const JobAcc* a, JobAcc* host, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) host[i] = a[i];
}

cudaError_t launch_acc_to_host(const JobAcc* acc, JobAcc* host_mapped, uint32_t n,
                               cudaStream_t st) {
  acc_to_host_kernel<<<1, 32, 0, st>>>(acc, host_mapped, n);
  return cudaGetLastError();
}

__global__ void u32_to_host_kernel(const uint32_t* src, uint32_t* host, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    host[i] = src[i];
}

cudaError_t launch_u32_to_host(const uint32_t* src, uint32_t* host_mapped, uint32_t n,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  u32_to_host_kernel<<<(n + 255) / 256 < 64 ? (n + 255) / 256 : 64, 256, 0, st>>>(src, host_mapped, n);
  return cudaGetLastError();
}

// BasePrimeStore::extend (base_store.cpp:44-69) on the device: the primes
// enumerated from (old bound, new bound] are appended to the resident table
// after its old_n entries (old_n read from a device copy, so the update of
// out_n cannot race with the readers).
__global__ void append_table_kernel(const unsigned long long* vals,
                                    const unsigned long long* n_dev, uint64_t cap,
                                    uint32_t* out_p, unsigned long long* out_m, double* out_inv,
                                    uint32_t* out_n, const uint32_t* old_n_dev) {
  const uint64_t n = *n_dev < cap ? static_cast<uint64_t>(*n_dev) : cap;
  const uint64_t base = *old_n_dev;
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_n = static_cast<uint32_t>(base + n);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = static_cast<uint32_t>(vals[i]);
    out_p[base + i] = p;
    out_m[base + i] = ~0ull / p;
    out_inv[base + i] = 1.0 / static_cast<double>(p);
  }
}

cudaError_t launch_append_table(const unsigned long long* vals, const unsigned long long* n_dev,
                                uint64_t cap, uint32_t* out_p, unsigned long long* out_m,
                                double* out_inv, uint32_t* out_n, const uint32_t* old_n_dev,
                                cudaStream_t st) {
  const int grid = static_cast<int>(cap / 256 + 1 < 4096 ? cap / 256 + 1 : 4096);
  append_table_kernel<<<grid, 256, 0, st>>>(vals, n_dev, cap, out_p, out_m, out_inv, out_n,
                                            old_n_dev);
  return cudaGetLastError();
}

cudaError_t launch_small_base(uint32_t n, uint32_t* out_p, unsigned long long* out_m,
                              double* out_inv, uint32_t* out_count, unsigned long long* scratch,
                              uint32_t epoch, cudaStream_t st) {
  if (n > kTinyMax || epoch == 0) return cudaErrorInvalidValue;
  const uint32_t grid = n / (32 * kBaseBlockWords) + 1;
  small_base_kernel<<<grid, kBaseBlockWords, 0, st>>>(n, out_p, out_m, out_inv, out_count,
                                                      scratch, epoch);
  return cudaGetLastError();
}

cudaError_t launch_prepare_table(const unsigned long long* vals, uint64_t skip,
                                 const unsigned long long* n_dev, uint64_t cap, uint32_t* out_p,
                                 unsigned long long* out_m, double* out_inv, uint32_t* out_n,
                                 cudaStream_t st) {
  const uint64_t cnt = cap > skip ? cap - skip : 1;
  const int grid = static_cast<int>(cnt / 256 + 1 < 4096 ? cnt / 256 + 1 : 4096);
  prepare_table_kernel<<<grid, 256, 0, st>>>(vals, skip, n_dev, cap, out_p, out_m, out_inv, out_n);
  return cudaGetLastError();
}

}  // namespace wsk
