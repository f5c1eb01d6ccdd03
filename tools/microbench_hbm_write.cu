// HBM write-only bandwidth on one B200 (evidence for DESIGN.md's enumeration
// roofline; not part of the product): grid-stride 16-byte and 8-byte stores
// over 4 GiB, CUDA events, best of 10, against a 16-byte copy for reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbmw tools/microbench_hbm_write.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void write16(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = make_uint4(uint32_t(i), 1, 2, 3);
}
__global__ void write8(unsigned long long* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = i;
}
__global__ void copy16(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

template <class F>
float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float bestms = 1e30f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < bestms) bestms = ms;
  }
  return bestms;
}

int main() {
  const size_t bytes = size_t(4) << 30;
  void *x, *y;
  cudaMalloc(&x, bytes);
  cudaMalloc(&y, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {4, 8, 16}) {
    const int grid = sms * per_sm;
    float t16 = best([&] { write16<<<grid, 512>>>((uint4*)x, bytes / 16); });
    float t8 = best([&] { write8<<<grid, 512>>>((unsigned long long*)x, bytes / 8); });
    float tc = best([&] { copy16<<<grid, 512>>>((const uint4*)x, (uint4*)y, bytes / 16); });
    printf("blocks/SM %2d: write 16 B %7.1f GB/s  write 8 B %7.1f GB/s  copy 16 B %7.1f GB/s (read+write)\n",
           per_sm, bytes / t16 / 1e6, bytes / t8 / 1e6, 2 * bytes / tc / 1e6);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
