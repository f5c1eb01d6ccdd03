// CPU test of the multi-device context's host threading (ws_host.h): the
// per-device worker pool runs fn(i) exactly once per device per run(), runs
// them concurrently, and a run() returns only after every worker finished.
// cudaSetDevice fails harmlessly without a GPU; no CUDA work is issued.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

#include "ws_host.h"

int main() {
  int fails = 0;
  for (size_t n : {1u, 2u, 3u, 8u}) {
    std::vector<int> devs(n);
    for (size_t i = 0; i < n; ++i) devs[i] = static_cast<int>(i);
    wsh::DevWorkers w(devs);
    std::vector<std::atomic<int>> hits(n);
    for (int round = 0; round < 2000; ++round) {
      std::atomic<int> inside{0};
      std::atomic<int> peak{0};
      w.run([&](size_t i) {
        const int now = ++inside;
        int p = peak.load();
        while (now > p && !peak.compare_exchange_weak(p, now)) {
        }
        if (round % 500 == 0) std::this_thread::sleep_for(std::chrono::milliseconds(2));
        hits[i].fetch_add(1);
        --inside;
      });
      if (inside.load() != 0) ++fails;  // run() returned before a worker finished
      if (round % 500 == 0 && n > 1 && peak.load() < 2) ++fails;  // workers overlap
    }
    for (size_t i = 0; i < n; ++i)
      if (hits[i].load() != 2000) {
        std::printf("device %zu ran %d times\n", i, hits[i].load());
        ++fails;
      }
  }
  std::printf(fails ? "[FAIL] %d\n" : "[PASS] workers\n", fails);
  return fails;
}
