// io_workers.cu — host IO worker threads of the file tier: each drains one SQ ring
// in pinned memory, reads the requested bytes from the feature file with pread (O_DIRECT when the
// filesystem allows it) into the request's pinned staging slot and publishes the CQ entry.  The GPU
// side of the rings (thread-level submission, asynchronous completion; §3.1) is
// k_io in gather.cu.  Host-only code (no kernels): tests/native/ring_harness.cpp compiles it in with a
// CPU fake producer.
#include <cerrno>
#include <immintrin.h>
#include <unistd.h>

#include "internal.cuh"

namespace helios {

void io_worker(helios_cache* c, int r) {
  IoRings& io = c->io;
  uint32_t next = 1;
  int idle = 0;
  while (!io.stop.load(std::memory_order_relaxed)) {
    const int64_t idx = (int64_t)r * io.depth + ((next - 1u) & (uint32_t)(io.depth - 1));
    SqEntry* e = io.sq + idx;
    uint32_t s = __atomic_load_n(&e->seq, __ATOMIC_ACQUIRE);  // the producer's release store of seq
    if (s != next) {
      if (++idle < 2000) _mm_pause();
      else if (idle < 4000) std::this_thread::yield();
      else usleep(50);
      continue;
    }
    idle = 0;
    const uint64_t off = e->file_off;
    const uint32_t len = e->len;
    const uint32_t slot = e->slot;
    char* dst = io.staging + (int64_t)slot * io.slot_bytes;
    int32_t status = 0;
    int64_t k = io.read_counter.fetch_add(1) + 1;
    if (io.fault_at > 0 && k == io.fault_at) {
      status = HELIOS_E_IO;
    } else {
      uint32_t done = 0;
      while (done < len) {
        ssize_t got = pread(io.fd, dst + done, len - done, (off_t)(off + done));
        if (got < 0 && errno == EINTR) continue;
        if (got <= 0) break;
        done += (uint32_t)got;
      }
      // a short read is an error only if it does not cover the row bytes
      if (done < (uint32_t)c->R) status = HELIOS_E_IO;
    }
    if (status) io.host_err.store(status);
    io.reads.fetch_add(1, std::memory_order_relaxed);
    CqEntry* q = io.cq + idx;
    __atomic_store_n(&q->status, status, __ATOMIC_RELAXED);
    __atomic_store_n(&q->seq, next, __ATOMIC_RELEASE);  // the completion, published last
    next++;
  }
}

}  // namespace helios
