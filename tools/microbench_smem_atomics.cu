// Shared-memory atomic throughput on one B200 (evidence for DESIGN.md §3's
// marking bound; not part of the product).  Each CTA owns a 64 KiB bitmap
// like the sieve kernel; 3 CTAs x 512 threads per SM.  Patterns:
//   conflict-free  lane l touches word (base + l) -- one wavefront per warp op
//   stride-p       lane l touches word (l * p / 32 + base) like the sieve's
//                  warp-cooperative loop (p = 37 and p = 1021 bits)
//   random         per-lane pseudo-random words (the mid-prime loop's pattern)
// Every op is one instruction (immediate address offsets), so the rates are
// the shared-memory pipe's, not the issue rate's.
// for red.shared.or.b32 (no return), atom.shared.or.b32 (return used) and a
// plain st.shared.b32, reported as lane operations per SM per clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/msa tools/microbench_smem_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kThreads = 512, kWords = 16384, kIters = 4096;

template <int OP, int PAT>
__global__ void __launch_bounds__(kThreads, 3) bench(uint32_t* sink) {
  extern __shared__ uint32_t bm[];
  for (int i = threadIdx.x; i < kWords; i += kThreads) bm[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // a lane's word in the first 2 KiB row; op k adds k rows (immediate offsets),
  // so every op is one instruction
  const uint32_t w0 = PAT == 0   ? lane
                      : PAT == 1 ? ((lane * 1021u) >> 5) & 511u
                      : PAT == 2 ? ((lane * 37u) >> 5) & 511u
                                 : ((threadIdx.x * 2654435761u + blockIdx.x * 40503u) >> 9) & 511u;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(bm)) + 4 * w0 +
                        (warp & 1) * 2048u;
  const uint32_t v = 1u << (threadIdx.x & 31);
  uint32_t acc = 0;
#pragma unroll 1
  for (int it = 0; it < kIters / 32; ++it) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint32_t a = base + (k & 15) * 4096u;
      if (OP == 0) {
        asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
      } else if (OP == 1) {
        uint32_t r;
        asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
        acc += r;
      } else {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
      }
    }
  }
  __syncthreads();
  if (acc == 0x12345678u) sink[0] = bm[threadIdx.x];
}

template <int OP, int PAT>
void run(const char* name, int sms, int clk_khz, uint32_t* sink) {
  auto k = bench<OP, PAT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4);
  const int grid = sms * 3 * 8;
  k<<<grid, kThreads, kWords * 4>>>(sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, kThreads, kWords * 4>>>(sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = static_cast<double>(grid) * kThreads * kIters;
  const double per_sm_clk = ops / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("%-34s %8.3f ms  %7.2f lane-ops/SM/clk  (%.2f warp-ops/SM/clk)\n", name, ms, per_sm_clk,
         per_sm_clk / 32);
}

int main() {
  cudaDeviceProp p{};
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s: %d SMs, max clock %d MHz (rates below use the max clock)\n", p.name,
         p.multiProcessorCount, clk / 1000);
  uint32_t* sink;
  cudaMalloc(&sink, 64);
  const int n = p.multiProcessorCount;
  run<0, 0>("red.shared.or   conflict-free", n, clk, sink);
  run<0, 2>("red.shared.or   stride-37 (wc p=37)", n, clk, sink);
  run<0, 1>("red.shared.or   stride-1021 (wc p=1021)", n, clk, sink);
  run<0, 3>("red.shared.or   random", n, clk, sink);
  run<1, 0>("atom.shared.or  conflict-free", n, clk, sink);
  run<1, 3>("atom.shared.or  random", n, clk, sink);
  run<2, 0>("st.shared       conflict-free", n, clk, sink);
  run<2, 3>("st.shared       random", n, clk, sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
