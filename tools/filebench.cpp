// Random-read throughput of a file with `threads` workers doing pread of `bs` bytes at random
// bs-aligned offsets (O_DIRECT when possible) for `secs` seconds.  Prints one JSON object.
// Used by bench.py as the file-tier roofline denominator (same access pattern as the IO workers).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fcntl.h>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>
int main(int argc, char** argv) {
  if (argc < 5) { fprintf(stderr, "usage: filebench path bs threads secs [header]\n"); return 2; }
  const char* path = argv[1];
  int64_t bs = atoll(argv[2]);
  int T = atoi(argv[3]);
  double secs = atof(argv[4]);
  int64_t hdr = argc > 5 ? atoll(argv[5]) : 0;
  struct stat st;
  if (stat(path, &st) != 0) { perror("stat"); return 1; }
  int64_t nblocks = (st.st_size - hdr) / bs;
  int fd = open(path, O_RDONLY | O_DIRECT);
  bool direct = fd >= 0;
  if (!direct) fd = open(path, O_RDONLY);
  std::atomic<int64_t> ops{0};
  std::atomic<bool> stop{false};
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++)
    th.emplace_back([&, t] {
      void* buf = nullptr;
      if (posix_memalign(&buf, 4096, bs)) return;
      uint64_t x = 0x9E3779B97F4A7C15ull * (t + 1);
      int64_t n = 0;
      while (!stop.load(std::memory_order_relaxed)) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        int64_t blk = (int64_t)(x % (uint64_t)nblocks);
        if (pread(fd, buf, bs, hdr + blk * bs) != bs) break;
        n++;
      }
      ops += n;
      free(buf);
    });
  auto t0 = std::chrono::steady_clock::now();
  std::this_thread::sleep_for(std::chrono::duration<double>(secs));
  stop = true;
  for (auto& x : th) x.join();
  double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("{\"bs\": %lld, \"threads\": %d, \"direct\": %s, \"iops\": %.0f, \"gbs\": %.4f}\n", (long long)bs, T,
         direct ? "true" : "false", ops / dt, ops * (double)bs / dt / 1e9);
  return 0;
}
