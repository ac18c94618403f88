// tests/native/stager_harness.cpp — TEST INFRASTRUCTURE ONLY (tests/test_host_protocols.py).
//
// CPU fake-producer harness for the staged host tier's chunk-claim protocol (the host side of
// HELIOS_CACHE_HOST_STAGED, paper_2310_00837_b200/csrc/staging.cu, compiled in unchanged): host
// threads stand in for the GPU.  Per batch and context, a "lookup" thread writes a random host list
// and posts the mailbox {seq, n_host} with a release store (as k_stage_publish does); "host warp"
// threads then take chunks from the list's front exactly as gather.cu's host_rows_dyn does
// (take a 64-row chunk from the front, publish the front hint, read its state word; wait a bounded
// time for a claimed chunk; copy a published chunk from staging, any other from the host tier) while the real
// stager threads claim chunks from the back.  Every output row is compared with its source row, so a
// lost, duplicated-into-the-wrong-place or stale chunk fails; built with -fsanitize=thread it also
// checks the protocol's memory ordering.  Prints one JSON line.
// The reservation rule (stage_reserve > 0: the last chunks wait a bounded time for a stager before
// the GPU takes them) is mirrored too.
//   stager_harness <contexts> <batches> <n_host> <stage_workers> <gpu_threads> <frac> [steal_us] [reserve]
//                  [reserve_us]
#include "../../paper_2310_00837_b200/csrc/staging.cu"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

using namespace helios;

int main(int argc, char** argv) {
  const int n_ctx = argc > 1 ? atoi(argv[1]) : 3;
  const int batches = argc > 2 ? atoi(argv[2]) : 50;
  const int64_t n_host_max = argc > 3 ? atoll(argv[3]) : 5000;
  const int workers = argc > 4 ? atoi(argv[4]) : 4;
  const int gpu_threads = argc > 5 ? atoi(argv[5]) : 4;
  const float frac = argc > 6 ? (float)atof(argv[6]) : 1.0f;
  const int steal_us = argc > 7 ? atoi(argv[7]) : 100;   // the GPU's kStageStealNs (0: never wait)
  const float reserve = argc > 8 ? (float)atof(argv[8]) : 0.0f;  // stage_reserve
  const int reserve_us = argc > 9 ? atoi(argv[9]) : 200;  // the GPU's kStageReserveNs
  const int32_t R = 64;        // row bytes (the protocol is independent of R)
  const int64_t S = 20000;     // host-tier rows
  std::vector<char> tier((size_t)S * R);
  for (int64_t s = 0; s < S; s++)
    for (int k = 0; k < R; k++) tier[(size_t)s * R + k] = (char)((s * 131 + k * 7) & 0xFF);

  helios_cache c;
  c.host_tier = tier.data();
  c.R = R;
  c.stage_workers = workers;
  c.stage_frac = frac;
  stager_start(&c);

  const int64_t chunks = (n_host_max + kStageChunk - 1) / kStageChunk;
  struct Ctx {
    GatherWS w;
    std::vector<int64_t> li;
    std::vector<uint64_t> lw;
    std::vector<char> stage, out;
    std::vector<unsigned long long> chunk;
    uint32_t mail[4] = {0, 0, 0, 0};
    unsigned long long hint = 0;
  };
  std::vector<Ctx> ctx(n_ctx);
  for (auto& x : ctx) {
    x.li.resize(n_host_max);
    x.lw.resize(n_host_max);
    x.w.stage_rows = std::min<int64_t>(kStageCapRows, chunks * kStageChunk);
    x.stage.resize((size_t)x.w.stage_rows * R);
    x.out.resize((size_t)n_host_max * R);
    x.chunk.assign(chunks, 0);
    x.w.h_host_w = x.lw.data();
    x.w.h_stage = x.stage.data();
    x.w.h_chunk = x.chunk.data();
    x.w.h_mail = x.mail;
    x.w.h_hint = &x.hint;
    stager_register(&c, x.w);
  }
  std::atomic<int64_t> bad{0}, rows_gpu{0}, rows_staged{0};
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> drivers;
  for (int ci = 0; ci < n_ctx; ci++)
    drivers.emplace_back([&, ci]() {
      Ctx& x = ctx[ci];
      std::mt19937_64 rng(1234 + ci);
      for (uint32_t seq = 1; seq <= (uint32_t)batches; seq++) {
        const int64_t n = 1 + (int64_t)(rng() % n_host_max);
        for (int64_t j = 0; j < n; j++) {  // the GPU's k_lookup writes the mirror (relaxed: see staging.cu)
          __atomic_store_n(&x.lw[j], (1ull << 62) | (rng() % S), __ATOMIC_RELAXED);
          x.li[j] = j;
        }
        // k_stage_publish: mailbox {seq, n_host}, seq last with release
        __atomic_store_n(&x.mail[1], (uint32_t)n, __ATOMIC_RELAXED);
        __atomic_store_n(&x.mail[0], seq, __ATOMIC_RELEASE);
        std::atomic<int64_t> ticket{0};
        const int64_t n_chunks = (n + kStageChunk - 1) / kStageChunk;
        const int64_t n_res = std::min<int64_t>(std::min<int64_t>(n_chunks, x.w.stage_rows / kStageChunk),
                                                (int64_t)std::ceil(reserve * (float)n_chunks));
        const int64_t c_res = n_chunks - n_res;
        std::vector<std::thread> warps;
        for (int t = 0; t < gpu_threads; t++)
          warps.emplace_back([&]() {
            for (;;) {
              const int64_t j0 = ticket.fetch_add(kStageChunk);
              if (j0 >= n) break;
              const int64_t cc = j0 / kStageChunk;
              const int64_t j1 = std::min<int64_t>(n, j0 + kStageChunk);
              const unsigned long long claimed = ((unsigned long long)seq << 2) | kChunkClaimed;
              const unsigned long long done = ((unsigned long long)seq << 2) | kChunkDone;
              unsigned long long st = __atomic_load_n(&x.chunk[cc], __ATOMIC_ACQUIRE);
              if (cc >= c_res && st != claimed && st != done) {  // reserved: wait for a stager to claim it
                auto w0 = std::chrono::steady_clock::now();
                while (st != claimed && st != done &&
                       std::chrono::steady_clock::now() - w0 < std::chrono::microseconds(reserve_us)) {
                  std::this_thread::yield();
                  st = __atomic_load_n(&x.chunk[cc], __ATOMIC_ACQUIRE);
                }
              }
              if (st != claimed && st != done)  // this "warp" copies the chunk: stagers stop at the front
                __atomic_store_n(&x.hint, ((unsigned long long)seq << 32) | (unsigned long long)cc, __ATOMIC_RELAXED);
              if (st == claimed) {  // bounded wait, then take the chunk back (as host_rows_dyn)
                auto w0 = std::chrono::steady_clock::now();
                while (st == claimed && std::chrono::steady_clock::now() - w0 < std::chrono::microseconds(steal_us)) {
                  std::this_thread::yield();
                  st = __atomic_load_n(&x.chunk[cc], __ATOMIC_ACQUIRE);
                }
              }
              if (st != done) {  // not staged: zero-copy
                for (int64_t j = j0; j < j1; j++)
                  memcpy(&x.out[(size_t)x.li[j] * R], &tier[(size_t)(__atomic_load_n(&x.lw[j], __ATOMIC_RELAXED) & ((1ull << 56) - 1)) * R], R);
                rows_gpu += j1 - j0;
                continue;
              }
              const int64_t srow0 = (n_chunks - 1 - cc) * kStageChunk + (j0 - cc * kStageChunk);
              for (int64_t j = j0; j < j1; j++)
                memcpy(&x.out[(size_t)x.li[j] * R], &x.stage[(size_t)(srow0 + (j - j0)) * R], R);
              rows_staged += j1 - j0;
            }
          });
        for (auto& t : warps) t.join();
        for (int64_t j = 0; j < n; j++)
          if (memcmp(&x.out[(size_t)j * R], &tier[(size_t)(x.lw[j] & ((1ull << 56) - 1)) * R], R) != 0) bad++;
      }
    });
  for (auto& t : drivers) t.join();
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const int64_t staged_by_cpu = c.stager->rows.load();
  stager_stop(&c);
  printf("{\"bad_rows\": %lld, \"rows_gpu\": %lld, \"rows_staged_used\": %lld, \"rows_staged_by_cpu\": %lld, "
         "\"seconds\": %.4f, \"batches\": %d, \"contexts\": %d}\n",
         (long long)bad.load(), (long long)rows_gpu.load(), (long long)rows_staged.load(), (long long)staged_by_cpu, secs,
         batches, n_ctx);
  return bad.load() == 0 ? 0 : 1;
}
