/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.
 *
 * A plain-C restatement of the reference's segmented mod-6 wheel sieve
 * (/root/reference/proj), used by tests/ (parity checker), by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg.  The product
 * (paper_2310_17746_b200/, libwheelsieve_cuda.so) never links or calls it:
 * the GPU path fails loudly when its CUDA extension is missing.
 *
 * Parity is PINNED: tests/test_oracle.py checks this restatement against the
 * reference library itself (oracle/_ref/libwsref.so, compiled from the
 * reference sources by oracle/Makefile) and against the golden vectors
 * committed under tests/golden/ (generated from the reference by
 * oracle/gen_golden.py, plus the known answers in the reference's own tests).
 *
 * Each function cites the reference file:line it restates.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* wheel.hpp:33-37 */
#define WSO_MAX_WHEEL_INDEX ((UINT64_MAX - 5) / 6)
#define WSO_MAX_SEGMENT_END (6 * (WSO_MAX_WHEEL_INDEX + 1))

/* isqrt: wheel.cpp:25-33 (double estimate, exact fix-up by division). */
uint64_t wso_isqrt(uint64_t n) {
  if (n == 0) return 0;
  uint64_t r = (uint64_t)sqrt((double)n);
  while (r > 0 && r > n / r) --r;
  while (r + 1 <= n / (r + 1)) ++r;
  return r;
}

/* ceil_sqrt: wheel.cpp:35-38 */
uint64_t wso_ceil_sqrt(uint64_t n) {
  uint64_t r = wso_isqrt(n);
  return r * r == n ? r : r + 1;
}

/* naive_sieve: wheel.cpp:40-54.  Dense byte sieve of [0, n], crossing off
 * from i*i.  Writes min(count, cap) primes; returns the count, or -1 when
 * n < 2 (Errc::EmptyRange) / allocation fails. */
int64_t wso_naive_sieve(uint64_t n, uint64_t* out, uint64_t cap) {
  if (n < 2) return -1;
  uint8_t* comp = (uint8_t*)calloc(n + 1, 1);
  if (!comp) return -1;
  for (uint64_t i = 2; i <= n / i; ++i) {
    if (comp[i]) continue;
    for (uint64_t j = i * i; j <= n; j += i) comp[j] = 1;
  }
  int64_t c = 0;
  for (uint64_t i = 2; i <= n; ++i)
    if (!comp[i]) {
      if ((uint64_t)c < cap && out) out[c] = i;
      ++c;
    }
  free(comp);
  return c;
}

/* Table 1 (paper Table 1; kStartIncrements wheel.cpp:77-82): row = p mod 6
 * is 5, column = anchor mod 6; {id1_coeff, id1_add, id5_coeff, id5_add}. */
static const uint32_t kInc[2][6][4] = {
    {{1, 0, 5, 0}, {6, 1, 4, 0}, {5, 1, 3, 0}, {4, 1, 2, 0}, {3, 1, 1, 0}, {2, 1, 6, 1}},
    {{5, 4, 1, 0}, {6, 5, 2, 1}, {1, 1, 3, 2}, {2, 2, 4, 3}, {3, 3, 5, 4}, {4, 4, 6, 5}},
};

/* start_offsets_after: wheel.cpp:86-94. */
void wso_start_offsets_after(uint64_t p, uint64_t anchor, uint64_t* id1, uint64_t* id5) {
  const uint64_t base = anchor / 6, r = p / 6;
  const uint32_t* c = kInc[p % 6 == 5][anchor % 6];
  *id1 = base + c[0] * r + c[1];
  *id5 = base + c[2] * r + c[3];
}

/* start_offsets: wheel.cpp:96-106 (checked).  Returns 0 ok, else the
 * 1 + Errc code (Domain = 5, Alignment = 6). */
int wso_start_offsets(uint64_t p, uint64_t start, uint64_t* id1, uint64_t* id5) {
  if (p % 6 != 1 && p % 6 != 5) return 5;
  if (start % 6 != 0) return 6;
  if (start <= p) return 5;
  wso_start_offsets_after(p, p * ((start - 1) / p), id1, id5); /* wheel.cpp:56-61 */
  return 0;
}

/* ---- Segment bitmap (segment.hpp:34-160, segment.cpp:12-162), Bit mode. */
typedef struct {
  uint64_t start, len, k0;
  uint64_t* w1; /* class 6k+1, LSB-first, tail bits zero (segment.cpp:34-35) */
  uint64_t* w5; /* class 6k+5 */
  uint64_t nwords;
} wso_seg;

static void seg_fill(uint64_t* w, uint64_t nwords, uint64_t len) { /* segment.cpp:28-47 */
  memset(w, 0xff, nwords * 8);
  if (len & 63) w[nwords - 1] = (UINT64_C(1) << (len & 63)) - 1;
}

static int seg_init(wso_seg* s, uint64_t start, uint64_t len) { /* segment.cpp:93-110 */
  s->start = start;
  s->len = len;
  s->k0 = start / 6;
  s->nwords = (len + 63) / 64;
  s->w1 = (uint64_t*)malloc(s->nwords * 8);
  s->w5 = (uint64_t*)malloc(s->nwords * 8);
  if (!s->w1 || !s->w5) return -1;
  seg_fill(s->w1, s->nwords, len);
  seg_fill(s->w5, s->nwords, len);
  return 0;
}

static void seg_free(wso_seg* s) {
  free(s->w1);
  free(s->w5);
}

/* clear_stride: segment.cpp:49-57 (Bit branch). */
static void clear_stride(uint64_t* w, uint64_t size, uint64_t first, uint64_t step) {
  for (uint64_t i = first; i < size; i += step) w[i >> 6] &= ~(UINT64_C(1) << (i & 63));
}

/* sieve_segment: segment.cpp:164-188.  `primes` are the base primes >= 5 in
 * ascending order (BasePrimeStore::entries, base_store.hpp:52). */
static void sieve_segment(wso_seg* s, const uint64_t* primes, uint64_t np) {
  const uint64_t end = s->start + 6 * s->len;
  for (uint64_t i = 0; i < np; ++i) {
    const uint64_t p = primes[i];
    const uint64_t sq = p * p;
    if (sq >= end) break; /* segment.cpp:176 */
    /* anchor rule, segment.cpp:178-183 */
    const uint64_t anchor = sq >= s->start ? p * (p - 1) : p * ((s->start - 1) / p);
    uint64_t id1, id5;
    wso_start_offsets_after(p, anchor, &id1, &id5);
    if (id1 - s->k0 < s->len) clear_stride(s->w1, s->len, id1 - s->k0, p);
    if (id5 - s->k0 < s->len) clear_stride(s->w5, s->len, id5 - s->k0, p);
  }
}

/* clear_value for value 1 (engine.cpp:244, segment.cpp:126-130). */
static void clear_one(wso_seg* s) {
  if (s->start == 0) s->w1[0] &= ~UINT64_C(1);
}

/* Wheel primes >= 5 up to ceil_sqrt(hint): BasePrimeStore::bootstrap,
 * base_store.cpp:34-42.  Returns count (malloc'd into *out). */
static int64_t bootstrap(uint64_t hint, uint64_t** out) {
  if (hint < 25) hint = 25;
  const uint64_t f = wso_ceil_sqrt(hint);
  int64_t n = wso_naive_sieve(f, NULL, 0);
  if (n < 0) return -1;
  uint64_t* all = (uint64_t*)malloc((size_t)n * 8);
  wso_naive_sieve(f, all, (uint64_t)n);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (all[i] >= 5) all[m++] = all[i];
  *out = all;
  return m;
}

typedef struct {
  uint64_t count, sum, xr, largest;
} wso_acc;

/* for_each_surviving (segment.hpp:123-146): ascending, 6k+1 before 6k+5;
 * filtered to [L, R). */
static void visit(const wso_seg* s, uint64_t L, uint64_t R, wso_acc* a, uint64_t* out,
                  uint64_t cap, uint64_t* n_out) {
  for (uint64_t wi = 0; wi < s->nwords; ++wi) {
    uint64_t m1 = s->w1[wi], m5 = s->w5[wi], both = m1 | m5;
    while (both) {
      const int bit = __builtin_ctzll(both);
      both &= both - 1;
      const uint64_t k = (wi << 6) | (uint64_t)bit;
      for (int c = 0; c < 2; ++c) {
        if (!(((c ? m5 : m1) >> bit) & 1)) continue;
        const uint64_t v = s->start + 6 * k + (c ? 5 : 1);
        if (v < L || v >= R) continue;
        a->count++;
        a->sum += v;
        a->xr ^= v;
        a->largest = v;
        if (out) {
          if (*n_out < cap) out[*n_out] = v;
          (*n_out)++;
        }
      }
    }
  }
}

static void add_prelude(uint64_t L, uint64_t R, wso_acc* a, uint64_t* out, uint64_t cap,
                        uint64_t* n_out) {
  for (uint64_t v = 2; v <= 3; ++v)
    if (v >= L && v < R) {
      a->count++;
      a->sum += v;
      a->xr ^= v;
      if (v > a->largest) a->largest = v;
      if (out) {
        if (*n_out < cap) out[*n_out] = v;
        (*n_out)++;
      }
    }
}

/* The [L, R) composition of SURVEY §3.3: segments of seg_slots wheel slots
 * from floor(L/6)*6, last one clipped to ceil((R-lo)/6) slots, 1 cleared at
 * lo == 0, survivors filtered to [L, R), 2 and 3 added when in range.
 * per_seg (nullable) gets survivors per segment excluding 2 and 3.
 * out (nullable) receives the sorted values.  Returns 0, or -1 on error. */
int wso_range(uint64_t L, uint64_t R, uint64_t seg_slots, wso_acc* acc, uint32_t* per_seg,
              uint64_t per_seg_cap, uint64_t* n_seg, uint64_t* out, uint64_t cap,
              uint64_t* n_out) {
  memset(acc, 0, sizeof *acc);
  if (n_seg) *n_seg = 0;
  if (n_out) *n_out = 0;
  uint64_t dummy = 0;
  if (!n_out) n_out = &dummy;
  if (R <= L) return 0;
  if (seg_slots == 0) return -1;
  add_prelude(L, R, acc, out, cap, n_out);
  const uint64_t lo0 = L / 6 * 6;
  const uint64_t total = (R - lo0 + 5) / 6;
  uint64_t* primes = NULL;
  const int64_t np = bootstrap(lo0 + 6 * total, &primes);
  if (np < 0) return -1;
  uint64_t s = 0;
  for (; s * seg_slots < total; ++s) {
    const uint64_t lo = lo0 + 6 * seg_slots * s;
    const uint64_t len = total - s * seg_slots < seg_slots ? total - s * seg_slots : seg_slots;
    wso_seg seg;
    if (seg_init(&seg, lo, len)) {
      free(primes);
      return -1;
    }
    sieve_segment(&seg, primes, (uint64_t)np);
    clear_one(&seg);
    wso_acc a;
    memset(&a, 0, sizeof a);
    visit(&seg, L, R, &a, out, cap, n_out);
    seg_free(&seg);
    if (per_seg && s < per_seg_cap) per_seg[s] = (uint32_t)a.count;
    acc->count += a.count;
    acc->sum += a.sum;
    acc->xr ^= a.xr;
    if (a.count) acc->largest = a.largest;
  }
  if (n_seg) *n_seg = s;
  free(primes);
  return 0;
}

/* Batch of intervals [Ls[i], Ls[i]+width) (BASELINE config 5). */
int wso_intervals(const uint64_t* Ls, uint64_t n, uint64_t width, uint64_t seg_slots,
                  uint32_t* counts, uint64_t* sums, uint64_t* xors) {
  for (uint64_t i = 0; i < n; ++i) {
    wso_acc a;
    if (wso_range(Ls[i], Ls[i] + width, seg_slots, &a, NULL, 0, NULL, NULL, 0, NULL)) return -1;
    counts[i] = (uint32_t)a.count;
    sums[i] = a.sum;
    if (xors) xors[i] = a.xr;
  }
  return 0;
}

/* Config-5 input generator (our convention, not the
 * reference's): splitmix64 from seed s, L_i = lo + z_i mod (hi - lo). */
void wso_splitmix_starts(uint64_t seed, uint64_t n, uint64_t lo, uint64_t hi, uint64_t* out) {
  uint64_t x = seed;
  for (uint64_t i = 0; i < n; ++i) {
    x += UINT64_C(0x9E3779B97F4A7C15);
    uint64_t z = x;
    z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
    z ^= z >> 31;
    out[i] = lo + z % (hi - lo);
  }
}
