// tests/native/ring_harness.cpp — TEST INFRASTRUCTURE ONLY (tests/test_host_protocols.py).
//
// CPU fake-producer harness for the file tier's SQ/CQ rings: the real host IO workers
// (paper_2310_00837_b200/csrc/io_workers.cu, compiled in unchanged) drain the rings while host threads
// play k_io's roles (gather.cu): submitters take request tickets, wait until their ring slot's previous
// occupant was consumed (free_seq), write the 32-byte descriptor and publish seq last with a release
// store; completers take tickets, wait for the CQ entry (acquire), check the staged row against the
// file bytes it must hold, count the completion and free the slot.  Requests m -> ring m % rings,
// sequence base + m / rings + 1, slot (seq - 1) & (depth - 1), as in the kernel.  Reports submitted /
// completed / missing / duplicate requests, wrong bytes and IO errors as one JSON line; built with
// -fsanitize=thread it also checks the rings' memory ordering.
//   ring_harness <rings> <depth> <producers> <requests> <fault_at (0 = none)>
#include "../../paper_2310_00837_b200/csrc/io_workers.cu"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <random>
#include <string>

using namespace helios;

int main(int argc, char** argv) {
  const int rings = argc > 1 ? atoi(argv[1]) : 2;
  const int depth = argc > 2 ? atoi(argv[2]) : 4;
  const int producers = argc > 3 ? atoi(argv[3]) : 2;
  const int64_t M = argc > 4 ? atoll(argv[4]) : 1000;
  const int64_t fault_at = argc > 5 ? atoll(argv[5]) : 0;
  const int32_t R = 512, stride = 512;
  const int64_t V = 4096, header = 4096;
  // the feature file: row v = bytes (v * 131 + k * 7) & 0xFF
  std::string path = "/tmp/ring_harness_" + std::to_string(getpid()) + ".bin";
  {
    std::vector<char> buf(header + V * stride, 0);
    for (int64_t v = 0; v < V; v++)
      for (int k = 0; k < R; k++) buf[header + v * stride + k] = (char)((v * 131 + k * 7) & 0xFF);
    FILE* f = fopen(path.c_str(), "wb");
    fwrite(buf.data(), 1, buf.size(), f);
    fclose(f);
  }
  helios_cache c;
  c.R = R;
  IoRings& io = c.io;
  io.rings = rings;
  io.depth = depth;
  io.slot_bytes = 4096;
  io.fault_at = fault_at;
  io.fd = open(path.c_str(), O_RDONLY);
  const int64_t n = (int64_t)rings * depth;
  std::vector<SqEntry> sq(n);
  std::vector<CqEntry> cq(n);
  std::vector<char> staging((size_t)n * io.slot_bytes);
  memset(sq.data(), 0, n * sizeof(SqEntry));
  memset(cq.data(), 0, n * sizeof(CqEntry));
  io.sq = sq.data();
  io.cq = cq.data();
  io.staging = staging.data();
  std::vector<uint32_t> free_seq(n, 0);  // the device-side ring state of k_io
  for (int r = 0; r < rings; r++) io.workers.emplace_back(io_worker, &c, r);

  // requests: random file rows
  std::vector<int64_t> row(M);
  std::mt19937_64 rng(7);
  for (auto& x : row) x = (int64_t)(rng() % V);
  std::atomic<int64_t> sub_ticket{0}, cmp_ticket{0}, bad{0}, io_errors{0}, submitted{0};
  std::vector<std::atomic<int>> seen(M);
  for (auto& s : seen) s = 0;
  auto slot_of = [&](int64_t m, uint32_t* seq) {
    const int r = (int)(m % rings);
    *seq = (uint32_t)(m / rings) + 1u;  // base_seq = 0: one batch
    return (int64_t)r * depth + ((*seq - 1u) & (uint32_t)(depth - 1));
  };
  std::vector<std::thread> th;
  for (int p = 0; p < producers; p++) {
    th.emplace_back([&]() {  // submitter role (one request per ticket; the kernel's lanes)
      for (;;) {
        const int64_t m = sub_ticket.fetch_add(1);
        if (m >= M) break;
        uint32_t seq;
        const int64_t idx = slot_of(m, &seq);
        while ((int32_t)(seq - (uint32_t)depth - __atomic_load_n(&free_seq[idx], __ATOMIC_ACQUIRE)) > 0)
          std::this_thread::yield();
        SqEntry* e = &sq[idx];
        e->file_off = (uint64_t)(header + row[m] * stride);
        e->len = (uint32_t)stride;
        e->slot = (uint32_t)idx;
        e->out_row = (uint64_t)m;
        __atomic_store_n(&e->seq, seq, __ATOMIC_RELEASE);
        submitted++;
      }
    });
    th.emplace_back([&]() {  // completer role (one request per ticket; the kernel's warps)
      for (;;) {
        const int64_t m = cmp_ticket.fetch_add(1);
        if (m >= M) break;
        uint32_t seq;
        const int64_t idx = slot_of(m, &seq);
        while (__atomic_load_n(&cq[idx].seq, __ATOMIC_ACQUIRE) != seq) std::this_thread::yield();
        if (__atomic_load_n(&cq[idx].status, __ATOMIC_RELAXED) != 0) {
          io_errors++;
        } else {
          const char* s = &staging[(size_t)idx * io.slot_bytes];
          for (int k = 0; k < R; k++)
            if (s[k] != (char)((row[m] * 131 + k * 7) & 0xFF)) {
              bad++;
              break;
            }
        }
        seen[m]++;
        __atomic_store_n(&free_seq[idx], seq, __ATOMIC_RELEASE);
      }
    });
  }
  for (auto& t : th) t.join();
  io.stop = true;
  for (auto& t : io.workers) t.join();
  close(io.fd);
  unlink(path.c_str());
  int64_t missing = 0, dup = 0, completed = 0;
  for (auto& s : seen) {
    missing += s.load() == 0;
    dup += s.load() > 1;
    completed += s.load() > 0;
  }
  printf("{\"submitted\": %lld, \"completed\": %lld, \"missing\": %lld, \"duplicates\": %lld, \"bad_bytes\": %lld, "
         "\"io_errors\": %lld, \"reads\": %lld}\n",
         (long long)submitted.load(), (long long)completed, (long long)missing, (long long)dup, (long long)bad.load(),
         (long long)io_errors.load(), (long long)io.reads.load());
  return 0;
}
