// CPU random-row gather rate: T threads copy random R-byte rows of a big buffer into a contiguous
// staging buffer (software prefetch ahead).  Prints one JSON object per thread count.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  size_t GB = atoll(argv[1]); int R = atoi(argv[2]);
  size_t bytes = GB << 30; int64_t nrows = bytes / R;
  char* src = (char*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(src, bytes, MADV_HUGEPAGE);
  { std::vector<std::thread> th; for (int t = 0; t < 16; t++) th.emplace_back([=] { size_t a = bytes / 16 * t; memset(src + a, t, bytes / 16); }); for (auto& x : th) x.join(); }
  const int64_t n = 1 << 22;
  std::vector<int64_t> idx(n); uint64_t x = 88172645463325252ull;
  for (auto& v : idx) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = x % nrows; }
  char* dst = (char*)aligned_alloc(4096, (size_t)n * R);
  memset(dst, 0, (size_t)n * R);
  for (int T : {1, 2, 4, 8, 12, 16}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++)
      th.emplace_back([&, t] {
        int64_t lo = n * t / T, hi = n * (t + 1) / T;
        for (int64_t i = lo; i < hi; i++) {
          if (i + 8 < hi) { const char* p = src + idx[i + 8] * (int64_t)R; for (int c = 0; c < R; c += 64) __builtin_prefetch(p + c); }
          memcpy(dst + i * (int64_t)R, src + idx[i] * (int64_t)R, R);
        }
      });
    for (auto& y : th) y.join();
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("{\"threads\": %d, \"R\": %d, \"region_gb\": %zu, \"Mrows_s\": %.1f, \"gbs\": %.2f}\n", T, R, GB, n / dt / 1e6, n * (double)R / dt / 1e9);
  }
  return 0;
}
