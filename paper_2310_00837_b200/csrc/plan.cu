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
#include <cstdlib>
#include <cstring>
#include <vector>
#include <unistd.h>

#include "internal.cuh"

namespace helios {

void plan_free_impl(helios_plan* p) {
  cudaDeviceSynchronize();
  for (auto& s : p->slots) {
    ws_free(s.ws);
    gws_free(s.gws);
    if (s.mem) cudaFree(s.mem);
    if (s.h_rb) cudaFreeHost(s.h_rb);
    if (s.d_trace) cudaFree(s.d_trace);
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
    if (s.ev_lk) cudaEventDestroy(s.ev_lk);
    if (s.ev_host) cudaEventDestroy(s.ev_host);
    if (s.s_side) cudaStreamDestroy(s.s_side);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  p->slots.clear();
  for (auto& l : p->s_link) {
    if (l) cudaStreamDestroy(l);
    l = nullptr;
  }
  if (p->ev_ref) cudaEventDestroy(p->ev_ref);
  p->ev_ref = nullptr;
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

// PDL for a plan's kernels: on, except when the cache has a host tier.  There the gathers wait on
// PCIe and the stagers for most of a batch, and dependents launched early (programmatic launch) sit in
// griddepcontrol.wait holding SM slots that the other slots' kernels need: C3 at 24 slots 6,845-6,895
// batches/s without vs 6,672-6,722 with; C2 (HBM only) 29.8 k with vs 29.2 k without
// (profiles/r02/pdl_on_off.jsonl).  HELIOS_PLAN_PDL=1 / 0 forces it.
static bool plan_pdl(const helios_plan* p) {
  if (const char* e = getenv("HELIOS_PLAN_PDL")) return atoi(e) != 0;
  return !(p->c && p->c->S > 0);
}

helios_status plan_create_impl(helios_plan* p) {
  PdlScope pdl_scope(plan_pdl(p));
  helios_graph* g = p->g;
  const helios_plan_desc& d = p->d;
  int64_t lvl[HELIOS_MAX_HOPS + 1], edg[HELIOS_MAX_HOPS];
  helios_status s = sample_bounds(d.max_seeds, d.fanouts, d.L, g->V, g->E, &p->maxn, lvl, edg);
  if (s != HELIOS_OK) return s;
  const int G = p->G;
  p->slots.resize((size_t)d.depth * G);
  HCUDA(cudaEventCreateWithFlags(&p->ev_gather_chain, cudaEventDisableTiming));
  HCUDA(cudaEventCreate(&p->ev_ref));
  if (p->link) {
    int least = 0, greatest = 0;
    HCUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    if (const char* e = getenv("HELIOS_PLAN_LINKS")) p->n_links = std::max(1, std::min(atoi(e), helios_plan::kMaxLinks));
    for (int i = 0; i < p->n_links; i++) HCUDA(cudaStreamCreateWithPriority(&p->s_link[i], cudaStreamNonBlocking, greatest));
  }
  for (int k = 0; k < d.depth * G; k++) {  // per position: workspaces and outputs
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
      sl.gws.ctl_preset = !p->intra;
    }
    s = ws_ensure(g, sl.ws, d.max_seeds, d.fanouts, d.L);
    if (s != HELIOS_OK) return s;
    HCUDA(cudaHostAlloc(&sl.h_rb, (HELIOS_MAX_HOPS + 1 + 4) * sizeof(int64_t), cudaHostAllocDefault));
  }
  for (int k = 0; k < d.depth * G; k += G) {  // per slot (group leader): stream, events, graphs
    PlanSlot& sl = p->slots[k];
    SampleWS* gws_s[kMaxGroup];
    const helios_blocks* gblk[kMaxGroup];
    GatherWS* ggw[kMaxGroup];
    const int64_t* gnodes[kMaxGroup];
    const int64_t* gnn[kMaxGroup];
    void* gfeat[kMaxGroup];
    helios_gather_stats* gst[kMaxGroup];
    for (int j = 0; j < G; j++) {
      PlanSlot& m = p->slots[k + j];
      gws_s[j] = &m.ws;
      gblk[j] = &m.blocks;
      ggw[j] = &m.gws;
      gnodes[j] = m.blocks.nodes;
      gnn[j] = m.blocks.level_counts + d.L;
      gfeat[j] = m.feats;
      gst[j] = m.stats;
    }
    HCUDA(cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking));
    if (p->trace) {
      const size_t row = (size_t)(3 * d.L + 4) * 16;
      HCUDA(cudaMalloc(&sl.d_trace, PlanSlot::kTraceRing * row));
      HCUDA(cudaMemset(sl.d_trace, 0xFF, PlanSlot::kTraceRing * row));
      sl.gws.trace_params = sl.ws.d_params;  // before capture: the gather kernels take it by value
      sl.gws.trace_idx = 3 * d.L + 2;
    }
    HCUDA(cudaEventCreateWithFlags(&sl.ev_caller, cudaEventDisableTiming));
    HCUDA(cudaEventCreateWithFlags(&sl.ev_end, cudaEventDisableTiming));
    sl.ring.assign(PlanSlot::kEv * PlanSlot::kRing, nullptr);
    for (auto& e : sl.ring) HCUDA(cudaEventCreate(&e));
    if (p->link) {
      HCUDA(cudaEventCreateWithFlags(&sl.ev_lk, cudaEventDisableTiming));
      HCUDA(cudaEventCreateWithFlags(&sl.ev_host, cudaEventDisableTiming));
    }
    if (p->graphs) {
      auto sample_ops = [&]() -> helios_status {
        // the gather's control words are zeroed at the batch start, off the sampling -> lookup edge
        for (int j = 0; j < G; j++)
          if (ggw[j]->ctl_preset)
            HCUDA(cudaMemsetAsync(ggw[j]->d_ctl, 0, kCtlWords * sizeof(unsigned long long), sl.stream));
        return sample_launch_group(g, gws_s, gblk, G, d.max_seeds, d.fanouts, d.L, sl.stream);
      };
      auto gather_ops = [&]() {  // link mode: lookup + HBM rows only (host rows: link stream)
        if (p->link)
          return gather_hbm_launch(p->c, sl.gws, sl.blocks.nodes, sl.blocks.level_counts + d.L, sl.blocks.nodes_cap,
                                   sl.feats, sl.stats, sl.stream);
        return gather_launch_group(p->c, ggw, gnodes, gnn, G, sl.blocks.nodes_cap, gfeat, gst, sl.stream);
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

// Launches slot gi's group (G positions, leader gi*G) with the parameters already uploaded; positions
// not submitted since the last launch run as empty batches.
static helios_status launch_group(helios_plan* p, int gi, uint32_t flags) {
  PdlScope pdl_scope(plan_pdl(p));
  const int G = p->G;
  PlanSlot& sl = p->slots[(size_t)gi * G];
  helios_status s = HELIOS_OK;
  for (int j = 0; j < G; j++) {
    PlanSlot& m = p->slots[(size_t)gi * G + j];
    if (!m.staged) {
      s = ws_upload_params(m.ws, 0, 0, nullptr, false, sl.stream, nullptr);
      if (s != HELIOS_OK) return s;
      m.rb_req = false;
    }
  }
  const bool timed = (flags & HELIOS_SUBMIT_TIMING) != 0;
  cudaEvent_t* ev = &sl.ring[PlanSlot::kEv * (sl.tcount % PlanSlot::kRing)];
  if (timed) HCUDA(cudaEventRecord(ev[0], sl.stream));
  const bool chain = p->serial_gather && p->c && !p->intra;
  if (p->graphs && p->intra && p->c) {  // one graph; timed submits time the whole overlapped batch
    HCUDA(cudaGraphLaunch(sl.g_all, sl.stream));
    if (timed) HCUDA(cudaEventRecord(ev[1], sl.stream));
  } else if (p->graphs && !timed && !chain && !p->two_graphs) {
    HCUDA(cudaGraphLaunch(sl.g_all, sl.stream));
  } else {
    SampleWS* gws_s[kMaxGroup];
    const helios_blocks* gblk[kMaxGroup];
    GatherWS* ggw[kMaxGroup];
    const int64_t* gnodes[kMaxGroup];
    const int64_t* gnn[kMaxGroup];
    void* gfeat[kMaxGroup];
    helios_gather_stats* gst[kMaxGroup];
    for (int j = 0; j < G; j++) {
      PlanSlot& m = p->slots[(size_t)gi * G + j];
      gws_s[j] = &m.ws;
      gblk[j] = &m.blocks;
      ggw[j] = &m.gws;
      gnodes[j] = m.blocks.nodes;
      gnn[j] = m.blocks.level_counts + p->d.L;
      gfeat[j] = m.feats;
      gst[j] = m.stats;
    }
    if (p->graphs) {
      HCUDA(cudaGraphLaunch(sl.g_sample, sl.stream));
    } else {
      for (int j = 0; j < G; j++)
        if (ggw[j]->ctl_preset)
          HCUDA(cudaMemsetAsync(ggw[j]->d_ctl, 0, kCtlWords * sizeof(unsigned long long), sl.stream));
      s = sample_launch_group(p->g, gws_s, gblk, G, p->d.max_seeds, p->d.fanouts, p->d.L, sl.stream);
      if (s != HELIOS_OK) return s;
    }
    if (chain && p->gather_chained) HCUDA(cudaStreamWaitEvent(sl.stream, p->ev_gather_chain, 0));
    if (timed) HCUDA(cudaEventRecord(ev[1], sl.stream));
    if (p->c) {
      if (p->graphs) {
        HCUDA(cudaGraphLaunch(sl.g_gather, sl.stream));
      } else if (p->link) {
        s = gather_hbm_launch(p->c, sl.gws, sl.blocks.nodes, sl.blocks.level_counts + p->d.L, sl.blocks.nodes_cap,
                              sl.feats, sl.stats, sl.stream);
        if (s != HELIOS_OK) return s;
      } else {
        s = gather_launch_group(p->c, ggw, gnodes, gnn, G, sl.blocks.nodes_cap, gfeat, gst, sl.stream);
        if (s != HELIOS_OK) return s;
      }
    }
  }
  if (p->link) {  // host rows on the link stream, one batch at a time, in submission order
    HCUDA(cudaEventRecord(sl.ev_lk, sl.stream));
    cudaStream_t ls = p->s_link[p->link_count++ % p->n_links];
    HCUDA(cudaStreamWaitEvent(ls, sl.ev_lk, 0));
    if (timed) HCUDA(cudaEventRecord(ev[3], ls));
    s = gather_host_launch(p->c, sl.gws, sl.feats, ls);
    if (s != HELIOS_OK) return s;
    if (timed) HCUDA(cudaEventRecord(ev[4], ls));
    HCUDA(cudaEventRecord(sl.ev_host, ls));
    HCUDA(cudaStreamWaitEvent(sl.stream, sl.ev_host, 0));
  }
  if (p->c) {
    for (int j = 0; j < G; j++) {
      PlanSlot& m = p->slots[(size_t)gi * G + j];
      s = io_launch(p->c, m.gws, m.feats, sl.stream);
      if (s != HELIOS_OK) return s;
    }
  }
  if (chain) {
    HCUDA(cudaEventRecord(p->ev_gather_chain, sl.stream));
    p->gather_chained = true;
  }
  if (timed) {
    HCUDA(cudaEventRecord(ev[2], sl.stream));
    sl.tcount++;
  }
  const int L = p->d.L;
  for (int j = 0; j < G; j++) {
    PlanSlot& m = p->slots[(size_t)gi * G + j];
    m.rb_valid = m.rb_req;
    if (m.rb_valid) {
      HCUDA(cudaMemcpyAsync(m.h_rb, m.blocks.level_counts, (L + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, sl.stream));
      if (p->c) HCUDA(cudaMemcpyAsync(m.h_rb + L + 1, m.stats, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, sl.stream));
    }
    m.staged = false;
    m.submitted = true;
  }
  HCUDA(cudaEventRecord(sl.ev_end, sl.stream));
  sl.count++;
  return HELIOS_OK;
}

// Stages one batch at position `slot` (uploads its parameters on the group's stream) and launches
// the group when the position is the group's last one (or on HELIOS_SUBMIT_FLUSH); G = 1: every
// submit launches.
helios_status plan_submit_impl(helios_plan* p, int32_t slot, const int64_t* seeds, int64_t n, uint64_t key, uint32_t flags,
                               cudaStream_t caller) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  HCHECK(n >= 0 && n <= p->d.max_seeds, HELIOS_E_CAPACITY, "n_seeds %lld > plan capacity %lld", (long long)n,
         (long long)p->d.max_seeds);
  HCHECK(n == 0 || seeds, HELIOS_E_INVALID, "null seeds");
  HCHECK(!p->c || !p->c->broken, HELIOS_E_STATE, "cache unusable after an IO / staging watchdog timeout");
  const int G = p->G;
  const int gi = slot / G;
  PlanSlot& sl = p->slots[(size_t)gi * G];  // the group's leader: stream, graphs, events
  PlanSlot& me = p->slots[slot];
  HCHECK(!me.staged, HELIOS_E_STATE, "position %d already holds a batch that was not launched", slot);
  HCUDA(cudaEventRecord(sl.ev_caller, caller));
  HCUDA(cudaStreamWaitEvent(sl.stream, sl.ev_caller, 0));
  void* trace_row = nullptr;
  if (p->trace) {
    const size_t row = (size_t)(3 * p->d.L + 4) * 16;
    trace_row = (char*)sl.d_trace + (sl.count % PlanSlot::kTraceRing) * row;
    HCUDA(cudaMemsetAsync(trace_row, 0xFF, row, sl.stream));
  }
  helios_status s = ws_upload_params(me.ws, key, n, seeds, (flags & HELIOS_SUBMIT_SEEDS_HOST) != 0, sl.stream,
                                     trace_row);
  if (s != HELIOS_OK) return s;
  me.staged = true;
  me.rb_req = (flags & HELIOS_SUBMIT_READBACK) != 0;
  if (slot % G == G - 1 || (flags & HELIOS_SUBMIT_FLUSH)) return launch_group(p, gi, flags);
  return HELIOS_OK;
}

// The group of position `slot` is launched first if that position holds a staged (not yet launched)
// batch; otherwise the position's last batch belongs to the group's last launch, which is what the
// caller waits for (batches staged at the group's other positions stay staged).
static helios_status flush_group(helios_plan* p, int32_t slot) {
  if (!p->slots[slot].staged) return HELIOS_OK;
  return launch_group(p, slot / p->G, 0);
}

helios_status plan_wait_impl(helios_plan* p, int32_t slot, cudaStream_t st) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  helios_status s = flush_group(p, slot);
  if (s != HELIOS_OK) return s;
  PlanSlot& sl = p->slots[(size_t)(slot / p->G) * p->G];
  if (!p->slots[slot].submitted) return HELIOS_OK;
  HCUDA(cudaStreamWaitEvent(st, sl.ev_end, 0));
  return HELIOS_OK;
}

helios_status plan_readback_impl(helios_plan* p, int32_t slot, int64_t* out) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  HCHECK(out, HELIOS_E_INVALID, "null readback output");
  helios_status s = flush_group(p, slot);
  if (s != HELIOS_OK) return s;
  PlanSlot& sl = p->slots[slot];
  HCHECK(sl.submitted && sl.rb_valid, HELIOS_E_STATE, "slot %d: last batch not submitted with HELIOS_SUBMIT_READBACK", slot);
  // wait by polling with short sleeps rather than cudaEventSynchronize's spin: the host stager threads
  // (HOST_STAGED) share these cores, and a spinning waiter takes one from them
  cudaEvent_t ev = p->slots[(size_t)(slot / p->G) * p->G].ev_end;
  for (unsigned us = 2;; us = std::min(us * 2, 50u)) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) return fail(HELIOS_E_CUDA, "helios_plan_readback: %s", cudaGetErrorString(e));
    usleep(us);
  }
  const int L = p->d.L;
  memcpy(out, sl.h_rb, (L + 1) * sizeof(int64_t));
  for (int q = 0; q < 4; q++) out[L + 1 + q] = p->c ? sl.h_rb[L + 1 + q] : 0;
  return HELIOS_OK;
}

helios_status plan_timing_impl(helios_plan* p, int32_t slot, int32_t back, helios_batch_timing* out) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  HCHECK(out, HELIOS_E_INVALID, "null timing output");
  PlanSlot& sl = p->slots[(size_t)(slot / p->G) * p->G];  // timing is per group (its leader's events)
  HCHECK(back >= 0 && back < PlanSlot::kRing && back < sl.tcount, HELIOS_E_RANGE,
         "slot %d: timed batch -%d not recorded", slot, back);
  cudaEvent_t* ev = &sl.ring[PlanSlot::kEv * ((sl.tcount - 1 - back) % PlanSlot::kRing)];
  HCUDA(cudaEventSynchronize(ev[2]));
  helios_batch_timing t{0, 0, -1.0f, -1.0f, -1.0f, -1.0f};
  HCUDA(cudaEventElapsedTime(&t.sample_ms, ev[0], ev[1]));
  HCUDA(cudaEventElapsedTime(&t.gather_ms, ev[1], ev[2]));
  if (p->link) HCUDA(cudaEventElapsedTime(&t.link_ms, ev[3], ev[4]));
  if (p->marked) {
    HCUDA(cudaEventElapsedTime(&t.t_start, p->ev_ref, ev[0]));
    HCUDA(cudaEventElapsedTime(&t.t_gather, p->ev_ref, ev[1]));
    HCUDA(cudaEventElapsedTime(&t.t_end, p->ev_ref, ev[2]));
  }
  *out = t;
  return HELIOS_OK;
}

helios_status plan_trace_impl(helios_plan* p, int32_t slot, int32_t back, uint64_t* out, int32_t cap,
                              int32_t* n_out) {
  HCHECK(slot >= 0 && slot < (int32_t)p->slots.size(), HELIOS_E_INVALID, "slot %d of %zu", slot, p->slots.size());
  HCHECK(p->trace, HELIOS_E_STATE, "plan created without HELIOS_PLAN_TRACE");
  PlanSlot& sl = p->slots[slot];
  HCHECK(back >= 0 && back < PlanSlot::kTraceRing && back < sl.count, HELIOS_E_RANGE, "slot %d: batch -%d not traced",
         slot, back);
  const int K = 3 * p->d.L + 4;
  HCHECK(out && cap >= 2 * K, HELIOS_E_CAPACITY, "trace output needs %d words", 2 * K);
  HCUDA(cudaEventSynchronize(sl.ev_end));
  std::vector<uint64_t> row(2 * K);
  HCUDA(cudaMemcpy(row.data(), (char*)sl.d_trace + ((sl.count - 1 - back) % PlanSlot::kTraceRing) * (size_t)K * 16,
                   (size_t)K * 16, cudaMemcpyDeviceToHost));
  for (int k = 0; k < K; k++) {
    const bool ran = row[2 * k] != ~0ull;
    out[2 * k] = ran ? row[2 * k] : 0;
    out[2 * k + 1] = ran ? ~row[2 * k + 1] : 0;
  }
  if (n_out) *n_out = K;
  return HELIOS_OK;
}

helios_status plan_mark_impl(helios_plan* p, cudaStream_t st) {
  HCUDA(cudaEventRecord(p->ev_ref, st));
  p->marked = true;
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
