// staging.cu — host stager threads for HELIOS_CACHE_HOST_STAGED (a platform adaptation of the
// pinned-host tier).
//
// The paper reads its CPU cache with GPU threads over UVA (§3.2.2).  On this platform
// random zero-copy reads of 512 B rows are capped near 48-50 M rows/s by a per-access host-side
// translation cost (profiles/links_r01.json), while sequential zero-copy reads reach the link.
// In staged mode the GPU still initiates everything: the lookup kernel writes the host-row list into
// pinned memory and a publish kernel posts a per-batch mailbox {seq, n_host, n_gpu, n_stage};
// rows [0, n_gpu) keep the zero-copy path, and these threads copy rows [n_gpu, n_host) into a
// contiguous pinned staging buffer in chunks of kStageChunk rows, publishing each chunk's
// completion (release); GPU stage warps wait for a chunk (acquire, system scope) and stream it
// into the feature buffer.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <immintrin.h>
#include <mutex>
#include <shared_mutex>
#include <unistd.h>

#include "internal.cuh"

namespace helios {

// Chunk distribution word: (seq << 32) | (n_chunks << 16) | next.  A chunk (seq, c) is claimed by a
// CAS that checks seq and next < n_chunks in the same word, so a worker holding a stale view can
// never take (or lose) a chunk of another batch.  While a claimed chunk is outstanding the GPU is
// waiting for it, so the mailbox (n_gpu, n_stage) cannot change under the worker.
struct StageCtx {
  GatherWS* w = nullptr;
  std::mutex mu;
  uint32_t cur_seq = 0;
  std::atomic<uint64_t> word{0};
};

struct Stager {
  std::vector<std::thread> threads;
  std::atomic<bool> stop{false};
  std::shared_mutex mu;  // guards ctxs (exclusive for (un)registration, shared for the scan)
  std::vector<StageCtx*> ctxs;
  const char* host_tier = nullptr;
  int32_t R = 0;
  std::atomic<int64_t> rows{0};
};

static void stager_worker(Stager* S) {
  int idle = 0;
  while (!S->stop.load(std::memory_order_relaxed)) {
    bool did = false;
    {
      std::shared_lock<std::shared_mutex> lk(S->mu);
      for (StageCtx* x : S->ctxs) {
        GatherWS& w = *x->w;
        if (__atomic_load_n(&w.h_mail[0], __ATOMIC_ACQUIRE) != x->cur_seq) {  // a new batch was posted
          std::lock_guard<std::mutex> g(x->mu);
          const uint32_t seq = __atomic_load_n(&w.h_mail[0], __ATOMIC_ACQUIRE);  // latest, re-read under lock
          if (seq != x->cur_seq) {
            const uint64_t n_chunks = (w.h_mail[3] + kStageChunk - 1) / kStageChunk;
            x->word.store(((uint64_t)seq << 32) | (n_chunks << 16), std::memory_order_release);
            x->cur_seq = seq;
          }
        }
        for (;;) {
          uint64_t cur = x->word.load(std::memory_order_acquire);
          const uint32_t seq = (uint32_t)(cur >> 32);
          const int64_t n_chunks = (int64_t)((cur >> 16) & 0xFFFF), chunk = (int64_t)(cur & 0xFFFF);
          if (chunk >= n_chunks) break;
          if (!x->word.compare_exchange_weak(cur, cur + 1, std::memory_order_acq_rel)) continue;
          // (seq, chunk) is ours and outstanding: the mailbox of `seq` is stable
          const int64_t n_gpu = w.h_mail[2], n_stage = w.h_mail[3];
          const int64_t j0 = chunk * kStageChunk, j1 = std::min<int64_t>(n_stage, j0 + kStageChunk);
          const uint64_t* hw = w.h_host_w + n_gpu;
          for (int64_t j = j0; j < j1; j++) {
            if (j + 4 < j1) {
              const char* p = S->host_tier + (int64_t)(hw[j + 4] & ((1ull << 56) - 1)) * S->R;
              for (int q = 0; q < S->R; q += 64) __builtin_prefetch(p + q);
            }
            memcpy(w.h_stage + j * S->R, S->host_tier + (int64_t)(hw[j] & ((1ull << 56) - 1)) * S->R, S->R);
          }
          __atomic_store_n(&w.h_done[chunk], seq, __ATOMIC_RELEASE);
          S->rows.fetch_add(j1 - j0, std::memory_order_relaxed);
          did = true;
        }
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
  c->stager = S;
  for (int t = 0; t < c->stage_workers; t++) S->threads.emplace_back(stager_worker, S);
  return HELIOS_OK;
}

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
  x->word.store((uint64_t)x->cur_seq << 32);
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
