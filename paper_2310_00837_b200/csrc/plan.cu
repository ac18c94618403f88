// plan.cu — execution plan: per-slot workspaces + CUDA graphs of a whole mini-batch.
//
// The paper's runtime splits a training iteration into GPU-initiated operators, builds an intra-
// and inter-mini-batch pipeline plan and launches the operators on asynchronous streams
// (§3.3, Fig. pipeline_design).  Here a plan slot is one in-flight mini-batch:
// its sampling operators (K1/K2) and lookup/gather operator (K3/K4) are captured once into two CUDA
// graphs and replayed for every batch on the slot's stream; slots run concurrently, so the
// sampling of batch i+1 overlaps the gather of batch i (the inter-mini-batch pipeline).  File-tier
// IO operators (K5/K6) are launched per batch behind the graphs (they wait on cross-stream events).
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace helios {

void plan_free_impl(helios_plan* p) {
  cudaDeviceSynchronize();
  for (auto& s : p->slots) {
    ws_free(s.ws);
    gws_free(s.gws);
    if (s.mem) cudaFree(s.mem);
    if (s.feats) cudaFree(s.feats);
    if (s.g_sample) cudaGraphExecDestroy(s.g_sample);
    if (s.g_gather) cudaGraphExecDestroy(s.g_gather);
    if (s.g_all) cudaGraphExecDestroy(s.g_all);
    for (cudaEvent_t e : {s.ev_caller, s.ev_end})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : s.ring)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : s.ev_fork)
      if (e) cudaEventDestroy(e);
    if (s.ev_join) cudaEventDestroy(s.ev_join);
    if (s.s_side) cudaStreamDestroy(s.s_side);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  p->slots.clear();
  if (p->ev_gather_chain) cudaEventDestroy(p->ev_gather_chain);
  p->ev_gather_chain = nullptr;
}

template <typename F>
static helios_status capture(cudaStream_t st, cudaGraphExec_t* out, F&& body) {
  HCUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  helios_status s = body();
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(st, &graph);
  if (s != HELIOS_OK) {
    if (graph) cudaGraphDestroy(graph);
    return s;
  }
  if (e != cudaSuccess) return fail(HELIOS_E_CUDA, "stream capture failed: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(out, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(HELIOS_E_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
  return HELIOS_OK;
}

helios_status plan_create_impl(helios_plan* p) {
  helios_graph* g = p->g;
  const helios_plan_desc& d = p->d;
  int64_t lvl[HELIOS_MAX_HOPS + 1], edg[HELIOS_MAX_HOPS];
  helios_status s = sample_bounds(d.max_seeds, d.fanouts, d.L, g->V, g->E, &p->maxn, lvl, edg);
  if (s != HELIOS_OK) return s;
  p->slots.resize(d.depth);
  HCUDA(cudaEventCreateWithFlags(&p->ev_gather_chain, cudaEventDisableTiming));
  for (int k = 0; k < d.depth; k++) {
    PlanSlot& sl = p->slots[k];
    // output blocks: one allocation
    size_t bytes = p->maxn * 8 + (d.L + 1) * 8 + HELIOS_MAX_HOPS * 8 + 256;
    for (int h = 0; h < d.L; h++) bytes += ((lvl[h] + 1) * 4 + 255) / 256 * 256 + (edg[h] * 4 + 255) / 256 * 256;
    HCUDA(cudaMalloc(&sl.mem, bytes));
    char* q = (char*)sl.mem;
    sl.blocks.nodes = (int64_t*)q;
    sl.blocks.nodes_cap = std::max<int64_t>(p->maxn, 1);
    q += (p->maxn * 8 + 255) / 256 * 256;
    sl.blocks.level_counts = (int64_t*)q;
    q += 128;
    sl.blocks.edge_counts = (int64_t*)q;
    q += 128;
    for (int h = 0; h < d.L; h++) {
      sl.blocks.block_indptr[h] = (int32_t*)q;
      sl.blocks.indptr_cap[h] = lvl[h] + 1;
      q += ((lvl[h] + 1) * 4 + 255) / 256 * 256;
      sl.blocks.block_indices[h] = (int32_t*)q;
      sl.blocks.edges_cap[h] = edg[h];
      q += (edg[h] * 4 + 255) / 256 * 256;
    }
    HCUDA(cudaMemset(sl.blocks.level_counts, 0, 256));
    if (p->c) {
      HCUDA(cudaMalloc(&sl.feats, std::max<int64_t>(p->maxn, 1) * (int64_t)p->c->R));
      HCUDA(cudaMalloc(&sl.stats, sizeof(helios_gather_stats)));
      HCUDA(cudaMemset(sl.stats, 0, sizeof(helios_gather_stats)));
      s = gws_ensure(p->c, sl.gws, sl.blocks.nodes_cap);
      if (s != HELIOS_OK) return s;
    }
    s = ws_ensure(g, sl.ws, d.max_seeds, d.fanouts, d.L);
    if (s != HELIOS_OK) return s;
    HCUDA(cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking));
    HCUDA(cudaEventCreateWithFlags(&sl.ev_caller, cudaEventDisableTiming));
    HCUDA(cudaEventCreateWithFlags(&sl.ev_end, cudaEventDisableTiming));
    sl.ring.assign(3 * PlanSlot::kRing, nullptr);
    for (auto& e : sl.ring) HCUDA(cudaEventCreate(&e));
    if (p->graphs) {
      auto sample_ops = [&]() { return sample_launch(g, sl.ws, d.max_seeds, d.fanouts, d.L, &sl.blocks, sl.stream); };
      auto gather_ops = [&]() {
        return gather_launch(p->c, sl.gws, sl.blocks.nodes, sl.blocks.level_counts + d.L, sl.blocks.nodes_cap,
                             sl.feats, sl.stats, sl.stream);
      };
      s = capture(sl.stream, &sl.g_sample, sample_ops);
      if (s != HELIOS_OK) return s;
      if (p->c) {
        s = capture(sl.stream, &sl.g_gather, gather_ops);
        if (s != HELIOS_OK) return s;
      }
      if (p->intra && p->c) {
        // intra-batch pipeline: a lookup+gather pass per new node range forks
        // onto the side stream as soon as that range is final, while the next hop samples
        HCUDA(cudaStreamCreateWithFlags(&sl.s_side, cudaStreamNonBlocking));
        for (auto& e : sl.ev_fork) HCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        HCUDA(cudaEventCreateWithFlags(&sl.ev_join, cudaEventDisableTiming));
        std::function<helios_status(int)> hook = [&](int stage) -> helios_status {
          HCUDA(cudaEventRecord(sl.ev_fork[stage], sl.stream));
          HCUDA(cudaStreamWaitEvent(sl.s_side, sl.ev_fork[stage], 0));
          const int64_t* lo = stage == 0 ? nullptr : sl.blocks.level_counts + stage - 1;
          return gather_range_launch(p->c, sl.gws, sl.blocks.nodes, lo, sl.blocks.level_counts + stage,
                                     sl.blocks.nodes_cap, sl.feats, sl.stats, stage == 0, sl.s_side);
        };
        s = capture(sl.stream, &sl.g_all, [&]() -> helios_status {
          HCUDA(cudaMemsetAsync(sl.stats, 0, sizeof(helios_gather_stats), sl.stream));
          helios_status r = sample_launch(g, sl.ws, d.max_seeds, d.fanouts, d.L, &sl.blocks, sl.stream, &hook);
          HCUDA(cudaEventRecord(sl.ev_join, sl.s_side));
          HCUDA(cudaStreamWaitEvent(sl.stream, sl.ev_join, 0));
          return r;
        });
      } else {
        s = capture(sl.stream, &sl.g_all, [&]() {  // the whole batch in one graph (untimed submits)
          helios_status r = sample_ops();
          return (r == HELIOS_OK && p->c) ? gather_ops() : r;
        });
      }
      if (s != HELIOS_OK) return s;
    }
  }
  HCUDA(cudaDeviceSynchronize());
  return HELIOS_OK;
}

helios_status plan_submit_impl(helios_plan* p, int32_t slot, const int64_t* seeds, int64_t n, uint64_t key, uint32_t flags,
                               cudaStream_t caller) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  HCHECK(n >= 0 && n <= p->d.max_seeds, HELIOS_E_CAPACITY, "n_seeds %lld > plan capacity %lld", (long long)n,
         (long long)p->d.max_seeds);
  HCHECK(n == 0 || seeds, HELIOS_E_INVALID, "null seeds");
  PlanSlot& sl = p->slots[slot];
  HCUDA(cudaEventRecord(sl.ev_caller, caller));
  HCUDA(cudaStreamWaitEvent(sl.stream, sl.ev_caller, 0));
  helios_status s = ws_upload_params(sl.ws, key, n, seeds, (flags & HELIOS_SUBMIT_SEEDS_HOST) != 0, sl.stream);
  if (s != HELIOS_OK) return s;
  const bool timed = (flags & HELIOS_SUBMIT_TIMING) != 0;
  cudaEvent_t* ev = &sl.ring[3 * (sl.tcount % PlanSlot::kRing)];
  if (timed) HCUDA(cudaEventRecord(ev[0], sl.stream));
  const bool chain = p->serial_gather && p->c && !p->intra;
  if (p->graphs && p->intra && p->c) {  // one graph; timed submits time the whole overlapped batch
    HCUDA(cudaGraphLaunch(sl.g_all, sl.stream));
    if (timed) HCUDA(cudaEventRecord(ev[1], sl.stream));
  } else if (p->graphs && !timed && !chain) {
    HCUDA(cudaGraphLaunch(sl.g_all, sl.stream));
  } else {
    if (p->graphs) {
      HCUDA(cudaGraphLaunch(sl.g_sample, sl.stream));
    } else {
      s = sample_launch(p->g, sl.ws, p->d.max_seeds, p->d.fanouts, p->d.L, &sl.blocks, sl.stream);
      if (s != HELIOS_OK) return s;
    }
    if (chain && p->gather_chained) HCUDA(cudaStreamWaitEvent(sl.stream, p->ev_gather_chain, 0));
    if (timed) HCUDA(cudaEventRecord(ev[1], sl.stream));
    if (p->c) {
      if (p->graphs) {
        HCUDA(cudaGraphLaunch(sl.g_gather, sl.stream));
      } else {
        s = gather_launch(p->c, sl.gws, sl.blocks.nodes, sl.blocks.level_counts + p->d.L, sl.blocks.nodes_cap,
                          sl.feats, sl.stats, sl.stream);
        if (s != HELIOS_OK) return s;
      }
    }
  }
  if (p->c) {
    s = io_launch(p->c, sl.gws, sl.feats, sl.stream);
    if (s != HELIOS_OK) return s;
  }
  if (chain) {
    HCUDA(cudaEventRecord(p->ev_gather_chain, sl.stream));
    p->gather_chained = true;
  }
  if (timed) {
    HCUDA(cudaEventRecord(ev[2], sl.stream));
    sl.tcount++;
  }
  HCUDA(cudaEventRecord(sl.ev_end, sl.stream));
  sl.count++;
  sl.submitted = true;
  return HELIOS_OK;
}

helios_status plan_wait_impl(helios_plan* p, int32_t slot, cudaStream_t st) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  PlanSlot& sl = p->slots[slot];
  if (!sl.submitted) return HELIOS_OK;
  HCUDA(cudaStreamWaitEvent(st, sl.ev_end, 0));
  return HELIOS_OK;
}

helios_status plan_timing_impl(helios_plan* p, int32_t slot, int32_t back, float* sample_ms, float* gather_ms) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  PlanSlot& sl = p->slots[slot];
  HCHECK(back >= 0 && back < PlanSlot::kRing && back < sl.tcount, HELIOS_E_RANGE,
         "slot %d: timed batch -%d not recorded", slot, back);
  cudaEvent_t* ev = &sl.ring[3 * ((sl.tcount - 1 - back) % PlanSlot::kRing)];
  HCUDA(cudaEventSynchronize(ev[2]));
  float a = 0, b = 0;
  HCUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
  HCUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
  if (sample_ms) *sample_ms = a;
  if (gather_ms) *gather_ms = b;
  return HELIOS_OK;
}

helios_status plan_outputs_impl(helios_plan* p, int32_t slot, helios_blocks* blocks, void** features,
                                helios_gather_stats** stats) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  PlanSlot& sl = p->slots[slot];
  if (blocks) *blocks = sl.blocks;
  if (features) *features = sl.feats;
  if (stats) *stats = sl.stats;
  return HELIOS_OK;
}

}  // namespace helios
