// CRC-32 (zlib polynomial 0xEDB88320, reflected, init/final xor ~0) of byte
// ranges of a device buffer: one thread per range, slice-by-8 tables in
// shared memory.  The chunk store (ws_store.cpp) computes each binary chunk
// file's CRC from its ranges with zlib's crc32_combine, so the 8-byte words
// never have to be scanned on the host (sink.cpp:61-64, 220-221 compute them
// with zlib's crc32 over the encoded buffer).
#include <cstdint>

#include "ws_internal.h"

namespace wsk {
namespace {

__global__ void __launch_bounds__(256) crc32_ranges_kernel(const uint8_t* data,
                                                            const uint64_t* begin,
                                                            const uint64_t* len, uint32_t n,
                                                            uint32_t* out) {
  __shared__ uint32_t T[8][256];
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    T[0][i] = c;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = T[0][i];
    for (int t = 1; t < 8; ++t) {
      c = T[0][c & 0xFFu] ^ (c >> 8);
      T[t][i] = c;
    }
  }
  __syncthreads();
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint8_t* p = data + begin[r];
  uint64_t m = len[r];
  uint32_t c = 0xFFFFFFFFu;
  // ranges start on 8-byte boundaries (whole uint64 words) except the tail
  while (m && (reinterpret_cast<uintptr_t>(p) & 7u)) {
    c = T[0][(c ^ *p++) & 0xFFu] ^ (c >> 8);
    --m;
  }
  const uint64_t* q = reinterpret_cast<const uint64_t*>(p);
  for (; m >= 8; m -= 8) {
    const uint64_t v = *q++;
    const uint32_t lo = static_cast<uint32_t>(v) ^ c, hi = static_cast<uint32_t>(v >> 32);
    c = T[7][lo & 0xFFu] ^ T[6][(lo >> 8) & 0xFFu] ^ T[5][(lo >> 16) & 0xFFu] ^ T[4][lo >> 24] ^
        T[3][hi & 0xFFu] ^ T[2][(hi >> 8) & 0xFFu] ^ T[1][(hi >> 16) & 0xFFu] ^ T[0][hi >> 24];
  }
  p = reinterpret_cast<const uint8_t*>(q);
  while (m--) c = T[0][(c ^ *p++) & 0xFFu] ^ (c >> 8);
  out[r] = c ^ 0xFFFFFFFFu;
}

}  // namespace

cudaError_t launch_crc32_ranges(const void* data, const uint64_t* begin, const uint64_t* len,
                                uint32_t n, uint32_t* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  crc32_ranges_kernel<<<(n + 255) / 256, 256, 0, st>>>(static_cast<const uint8_t*>(data), begin,
                                                        len, n, out);
  return cudaGetLastError();
}

}  // namespace wsk
