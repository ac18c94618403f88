// staging.cu — host stager threads for HELIOS_CACHE_HOST_STAGED (a platform adaptation of the
// pinned-host tier; DESIGN.md §3 reading 14, §7).
//
// The paper reads its CPU cache with GPU threads over UVA (§3.2.2).  On this platform
// random zero-copy reads of 512 B rows are capped near 48-50 M rows/s by a per-access host-side
// translation cost (profiles/links_r01.json), while sequential zero-copy reads reach the link.
// In staged mode the GPU still initiates everything: the lookup kernel writes the host-row list into
// pinned memory and a publish kernel posts a per-batch mailbox {seq, n_host}.  The GPU's host-row
// warps take rows from the FRONT of the list (zero-copy); these threads claim 64-row chunks from the
// BACK (state[c] = seq|CLAIMED), copy them into a contiguous pinned staging buffer and publish them
// (state[c] = seq|DONE); GPU warps that reach a published chunk stream it from staging, wait a
// bounded time for a claimed one and read any other chunk zero-copy (gather.cu, host_rows_dyn).  The
// split point is where the two sides meet, so it adapts to the rates of both.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <immintrin.h>
#include <mutex>
#include <shared_mutex>
#include <unistd.h>

#include "internal.cuh"

namespace helios {

// Chunk distribution word: (seq << 32) | (limit << 16) | next.  The next claim takes chunk
// n_chunks - 1 - next while next < limit; the CAS checks seq, limit and next in one word, so a
// worker holding a stale view can never take (or lose) a chunk of another batch.  `inflight` counts
// workers between their claim attempt and the chunk's completion: a new batch's word is published
// only once it is 0, so no copy of an earlier batch can still be writing the staging buffer (the GPU
// does not wait for chunks it copied itself, so such copies can outlive their batch).
struct StageCtx {
  GatherWS* w = nullptr;
  std::mutex mu;
  std::atomic<uint32_t> cur_seq{0};  // written under mu, read without it (a stale read only re-checks)
  int64_t n_host = 0, n_chunks = 0;  // of cur_seq; changed only with inflight == 0
  std::atomic<uint64_t> word{0};
  std::atomic<int> inflight{0};
};

struct Stager {
  std::vector<std::thread> threads;
  std::atomic<bool> stop{false};
  std::shared_mutex mu;  // guards ctxs (exclusive for (un)registration, shared for the scan)
  std::vector<StageCtx*> ctxs;
  const char* host_tier = nullptr;
  int32_t R = 0;
  float frac = 1.0f;     // share of a batch's chunks the stagers may claim at most
  std::atomic<int64_t> rows{0};
};

// A new batch was posted on x's mailbox: close the old word, wait for in-flight copies, open the new.
static void stage_open(Stager* S, StageCtx* x, uint32_t seq) {
  GatherWS& w = *x->w;
  x->word.store((uint64_t)x->cur_seq.load() << 32, std::memory_order_seq_cst);  // limit 0: no more claims
  while (x->inflight.load(std::memory_order_seq_cst) != 0) _mm_pause();
  x->n_host = __atomic_load_n(&w.h_mail[1], __ATOMIC_ACQUIRE);
  x->n_chunks = (x->n_host + kStageChunk - 1) / kStageChunk;
  int64_t lim = std::min<int64_t>(x->n_chunks, w.stage_rows / kStageChunk);
  lim = std::min<int64_t>(lim, (int64_t)std::ceil((double)S->frac * (double)x->n_chunks));
  x->cur_seq = seq;
  x->word.store(((uint64_t)seq << 32) | ((uint64_t)lim << 16), std::memory_order_seq_cst);
}

// Claims and copies chunks of x's current batch until none is left; returns whether it copied any.
static bool stage_claim_loop(Stager* S, StageCtx* x) {
  GatherWS& w = *x->w;
  bool did = false;
  for (;;) {
    {  // cheap check first: idle workers must not keep the inflight counter busy while stage_open waits
      const uint64_t peek = x->word.load(std::memory_order_acquire);
      if ((peek & 0xFFFF) >= ((peek >> 16) & 0xFFFF)) return did;
    }
    x->inflight.fetch_add(1, std::memory_order_seq_cst);
    uint64_t cur = x->word.load(std::memory_order_seq_cst);
    const uint32_t seq = (uint32_t)(cur >> 32);
    const int64_t lim = (int64_t)((cur >> 16) & 0xFFFF), next = (int64_t)(cur & 0xFFFF);
    if (next >= lim) {
      x->inflight.fetch_sub(1, std::memory_order_seq_cst);
      return did;
    }
    const int64_t c = x->n_chunks - 1 - next;  // stable: the word is open, so n_chunks belongs to seq
    const unsigned long long h = __atomic_load_n(w.h_hint, __ATOMIC_ACQUIRE);
    if ((uint32_t)(h >> 32) == seq && (int64_t)(h & 0xFFFFFFFFu) >= c) {  // the GPU's front reached c: stop
      x->word.compare_exchange_strong(cur, (cur & ~0xFFFF0000ull) | ((uint64_t)next << 16));
      x->inflight.fetch_sub(1, std::memory_order_seq_cst);
      return did;
    }
    if (!x->word.compare_exchange_weak(cur, cur + 1, std::memory_order_seq_cst)) {
      x->inflight.fetch_sub(1, std::memory_order_seq_cst);
      continue;
    }
    __atomic_store_n(&w.h_chunk[c], ((unsigned long long)seq << 2) | kChunkClaimed, __ATOMIC_RELAXED);
    const int64_t j0 = c * kStageChunk, j1 = std::min<int64_t>(x->n_host, j0 + kStageChunk);
    char* dst = w.h_stage + next * kStageChunk * (int64_t)S->R;
    const uint64_t* hw = w.h_host_w;
    // the mirror is written by the GPU (k_lookup of a LATER batch can overwrite it while a copy of
    // an abandoned chunk still reads it: that copy lands in staging nobody reads), so relaxed loads
    auto slot_of = [&](int64_t j) { return (int64_t)(__atomic_load_n(&hw[j], __ATOMIC_RELAXED) & ((1ull << 56) - 1)); };
    constexpr int kAhead = 12;  // rows prefetched ahead: random DRAM rows, latency-bound per thread
    for (int64_t j = j0; j < std::min<int64_t>(j1, j0 + kAhead); j++) {
      const char* p = S->host_tier + slot_of(j) * S->R;
      for (int q = 0; q < S->R; q += 64) __builtin_prefetch(p + q);
    }
    for (int64_t j = j0; j < j1; j++) {
      if (j + kAhead < j1) {
        const char* p = S->host_tier + slot_of(j + kAhead) * S->R;
        for (int q = 0; q < S->R; q += 64) __builtin_prefetch(p + q);
      }
      memcpy(dst + (j - j0) * S->R, S->host_tier + slot_of(j) * S->R, S->R);
    }
    __atomic_store_n(&w.h_chunk[c], ((unsigned long long)seq << 2) | kChunkDone, __ATOMIC_RELEASE);
    S->rows.fetch_add(j1 - j0, std::memory_order_relaxed);
    x->inflight.fetch_sub(1, std::memory_order_seq_cst);
    did = true;
  }
}

static void stager_worker(Stager* S) {
  int idle = 0;
  while (!S->stop.load(std::memory_order_relaxed)) {
    bool did = false;
    {
      std::shared_lock<std::shared_mutex> lk(S->mu);
      for (StageCtx* x : S->ctxs) {
        GatherWS& w = *x->w;
        if (__atomic_load_n(&w.h_mail[0], __ATOMIC_ACQUIRE) != x->cur_seq.load(std::memory_order_relaxed)) {
          std::lock_guard<std::mutex> g(x->mu);
          const uint32_t seq = __atomic_load_n(&w.h_mail[0], __ATOMIC_ACQUIRE);  // latest, re-read under lock
          if (seq != x->cur_seq.load()) stage_open(S, x, seq);  // a new batch was posted
        }
        did |= stage_claim_loop(S, x);
      }
    }
    if (did) {
      idle = 0;
    } else if (++idle < 4000) {
      _mm_pause();
    } else if (idle < 8000) {
      std::this_thread::yield();
    } else {
      usleep(20);
    }
  }
}

helios_status stager_start(helios_cache* c) {
  Stager* S = new Stager();
  S->host_tier = c->host_tier;
  S->R = c->R;
  S->frac = c->stage_frac;
  c->stager = S;
  for (int t = 0; t < c->stage_workers; t++) S->threads.emplace_back(stager_worker, S);
  return HELIOS_OK;
}

int64_t stager_rows(const helios_cache* c) { return c->stager ? c->stager->rows.load() : 0; }

void stager_stop(helios_cache* c) {
  Stager* S = c->stager;
  if (!S) return;
  S->stop = true;
  for (auto& t : S->threads) t.join();
  for (StageCtx* x : S->ctxs) delete x;
  delete S;
  c->stager = nullptr;
}

helios_status stager_register(helios_cache* c, GatherWS& w) {
  if (!c->stager) return HELIOS_OK;
  StageCtx* x = new StageCtx();
  x->w = &w;
  x->cur_seq = w.h_mail[0];
  x->word.store((uint64_t)x->cur_seq.load() << 32);  // limit 0 until the first batch is posted
  {
    std::unique_lock<std::shared_mutex> lk(c->stager->mu);
    c->stager->ctxs.push_back(x);
  }
  w.sctx = x;
  return HELIOS_OK;
}

void stager_unregister(helios_cache* c, GatherWS& w) {
  if (!c || !c->stager || !w.sctx) return;
  {
    std::unique_lock<std::shared_mutex> lk(c->stager->mu);
    auto& v = c->stager->ctxs;
    v.erase(std::remove(v.begin(), v.end(), w.sctx), v.end());
  }
  delete w.sctx;
  w.sctx = nullptr;
}

}  // namespace helios
