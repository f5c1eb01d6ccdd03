// Global (L2) RED.OR throughput on one B200 -- evidence for the choice
// between bucket lists in HBM and an L2-resident window bitmap for the large
// primes.  Not part of the product.
//
// Patterns, every op a `red.global.or.b32` on a bitmap of B bytes:
//   random    per-thread pseudo-random words (xorshift), the floor
//   primes    thread t owns a "prime" p_t (odd, in [pmin, pmax) slots) and
//             crosses off h, h + p, h + 2p, ... inside the window, the large-
//             prime marking loop of a window bitmap (two classes interleaved)
// and, for comparison, plain st.global.b32 with the random pattern.
// Reported: operations per second and per SM-clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mla tools/microbench_l2_atomics.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>

template <int OP>
__global__ void random_ops(uint32_t* bm, uint32_t words_mask, uint32_t iters) {
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
#pragma unroll 4
  for (uint32_t i = 0; i < iters; ++i) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    uint32_t* a = bm + (x & words_mask);
    if (OP == 0)
      asm volatile("red.global.or.b32 [%0], %1;" ::"l"(a), "r"(1u << (x >> 27)) : "memory");
    else
      asm volatile("st.global.b32 [%0], %1;" ::"l"(a), "r"(1u << (x >> 27)) : "memory");
  }
}

// thread t: prime p (slots), two classes, marks every hit in [0, span)
__global__ void prime_ops(uint32_t* bm, uint64_t span, uint32_t pmin, uint32_t pmax,
                          unsigned long long* nops) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  // primes ascend with t (a warp holds neighbours, like the sieve's table)
  const uint32_t p = (pmin + static_cast<uint32_t>((static_cast<uint64_t>(pmax - pmin) * t) /
                                                   (gridDim.x * blockDim.x))) | 1u;
  uint64_t h1 = (t * 7919ull) % p, h5 = (t * 104729ull) % p;
  const uint64_t half = span / 2;  // class 1 in [0, half), class 5 in [half, span)
  uint32_t n = 0;
  for (; h1 < half; h1 += p, ++n)
    asm volatile("red.global.or.b32 [%0], %1;" ::"l"(bm + (h1 >> 5)), "r"(1u << (h1 & 31)) : "memory");
  for (; h5 < half; h5 += p, ++n) {
    const uint64_t b = half + h5;
    asm volatile("red.global.or.b32 [%0], %1;" ::"l"(bm + (b >> 5)), "r"(1u << (b & 31)) : "memory");
  }
  atomicAdd(nops, static_cast<unsigned long long>(n));
}

int main() {
  int sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const size_t maxb = 1ull << 30;
  uint32_t* bm;
  unsigned long long* nops;
  cudaMalloc(&bm, maxb);
  cudaMalloc(&nops, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("B200: %d SMs, %.0f MHz\n", sms, clk_khz / 1e3);
  for (size_t mb : {16, 32, 64, 96, 128, 1024}) {
    const size_t bytes = mb << 20;
    // round down to a power of two words for the mask
    uint32_t words = 1;
    while (2ull * words * 4 <= bytes) words *= 2;
    for (int op = 0; op < 2; ++op) {
      const uint32_t iters = 4096;
      const int grid = sms * 8, block = 256;
      cudaMemset(bm, 0, bytes);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (op == 0)
          random_ops<0><<<grid, block>>>(bm, words - 1, iters);
        else
          random_ops<1><<<grid, block>>>(bm, words - 1, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = static_cast<double>(grid) * block * iters;
        if (rep == 2)
          printf("random %-6s bitmap %5zu MB (%u words): %.3f ms  %.3e ops/s  %.2f ops/SM/clk\n",
                 op == 0 ? "RED.OR" : "STG", mb, words, ms, ops / (ms * 1e-3),
                 ops / (ms * 1e-3) / sms / (clk_khz * 1e3));
      }
    }
  }
  // window bitmaps of the large-prime design: spans in slots (bits) per class
  struct Case {
    uint64_t span_bits;
    uint32_t pmin, pmax;
    const char* what;
  } cases[] = {
      {2ull * 750 * 262144, 524288, 31622777, "c4-like: 750 segments, p in [2S, 3.16e7)"},
      {2ull * 1500 * 262144, 524288, 31622777, "c4-like: 1500 segments, p in [2S, 3.16e7)"},
      {2ull * 1500 * 262144, 262144, 1000000, "c3-like: 1500 segments, p in [S, 1e6)"},
      {2ull * 3000 * 262144, 262144, 1000000, "c3-like: 3000 segments, p in [S, 1e6)"},
  };
  for (const Case& c : cases) {
    const size_t bytes = c.span_bits / 8;
    const int block = 256;
    // one thread per prime: ~pi(pmax) - pi(pmin) threads
    const double nprimes = c.pmax / std::log(static_cast<double>(c.pmax)) -
                           c.pmin / std::log(static_cast<double>(c.pmin));
    const int grid = static_cast<int>(nprimes / block) + 1;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(bm, 0, bytes);
      cudaMemset(nops, 0, 8);
      cudaEventRecord(e0);
      prime_ops<<<grid, block>>>(bm, c.span_bits, c.pmin, c.pmax, nops);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long n = 0;
      cudaMemcpy(&n, nops, 8, cudaMemcpyDeviceToHost);
      if (rep == 2)
        printf("primes %-44s bitmap %6.1f MB: %.3f ms  %llu ops  %.3e ops/s  %.2f ops/SM/clk\n",
               c.what, bytes / 1048576.0, ms, n, n / (ms * 1e-3),
               n / (ms * 1e-3) / sms / (clk_khz * 1e3));
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
