// abi.cu — extern "C" entry points of libhelios.so (declared and documented in include/helios.h).
#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <new>

#include "internal.cuh"

namespace helios {

static thread_local std::string g_last_error;

void set_error(const std::string& s) { g_last_error = s; }

// Programmatic dependent launch: on unless HELIOS_NO_PDL=1; a scope (PdlScope) can turn it off for the
// launches it encloses (plans whose cache has a host tier).
static thread_local int g_pdl_scope = -1;
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HELIOS_NO_PDL");
    return !(e && atoi(e) != 0);
  }();
  return on && g_pdl_scope != 0;
}
PdlScope::PdlScope(bool enable) : prev(g_pdl_scope) { g_pdl_scope = enable ? 1 : 0; }
PdlScope::~PdlScope() { g_pdl_scope = prev; }

helios_status fail(helios_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

helios_status cache_build_impl(helios_graph* g, const helios_cache_desc* d, helios_cache* c);
void cache_free_impl(helios_cache* c);
void plan_free_impl(helios_plan* p);
helios_status plan_create_impl(helios_plan* p);
helios_status plan_submit_impl(helios_plan* p, int32_t slot, const int64_t* seeds, int64_t n, uint64_t key, uint32_t flags,
                               cudaStream_t caller);
helios_status plan_wait_impl(helios_plan* p, int32_t slot, cudaStream_t st);
helios_status plan_timing_impl(helios_plan* p, int32_t slot, int32_t back, helios_batch_timing* out);
helios_status plan_mark_impl(helios_plan* p, cudaStream_t st);
helios_status plan_trace_impl(helios_plan* p, int32_t slot, int32_t back, uint64_t* out, int32_t cap, int32_t* n_out);
helios_status plan_readback_impl(helios_plan* p, int32_t slot, int64_t* out);
helios_status plan_outputs_impl(helios_plan* p, int32_t slot, helios_blocks* blocks, void** features,
                                helios_gather_stats** stats);

// helios_sample on the graph's default sampling context.
static helios_status sample_default(helios_graph* g, const int64_t* seeds, int64_t B, const int32_t* fanouts, int32_t L,
                                    uint64_t key, const helios_blocks* out, cudaStream_t st) {
  helios_status s = sample_check_out(g, B, fanouts, L, out);
  if (s != HELIOS_OK) return s;
  HCHECK(B == 0 || seeds, HELIOS_E_INVALID, "null seeds");
  s = ws_ensure(g, g->ws, B, fanouts, L);
  if (s != HELIOS_OK) return s;
  s = ws_upload_params(g->ws, key, B, seeds, false, st);
  if (s != HELIOS_OK) return s;
  return sample_launch(g, g->ws, B, fanouts, L, out, st);
}

static helios_status read_latched(int* d_err, helios_status* out) {
  int h = 0;
  HCUDA(cudaMemcpy(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) HCUDA(cudaMemset(d_err, 0, sizeof(int)));
  *out = (helios_status)h;
  return HELIOS_OK;
}

}  // namespace helios

using namespace helios;

#define GUARD_BEGIN try {
#define GUARD_END                                                   \
  }                                                                 \
  catch (const std::bad_alloc&) {                                   \
    return fail(HELIOS_E_NOMEM, "host allocation failed");          \
  }                                                                 \
  catch (...) {                                                     \
    return fail(HELIOS_E_STATE, "unexpected C++ exception");        \
  }

extern "C" {

int helios_abi_version(void) { return HELIOS_ABI_VERSION; }

const char* helios_last_error(void) { return helios::g_last_error.c_str(); }

helios_status helios_graph_load(int device, int64_t V, int64_t E, const int64_t* indptr, const int32_t* indices,
                                uint32_t flags, helios_graph** out) {
  GUARD_BEGIN
  HCHECK(out, HELIOS_E_INVALID, "out is NULL");
  *out = nullptr;
  HCHECK((flags & ~HELIOS_GRAPH_TOPO_HOST) == 0, HELIOS_E_INVALID, "unknown graph flags 0x%x", flags);
  HCHECK(V >= 1 && V < (1ll << 31), HELIOS_E_INVALID, "V=%lld out of [1, 2^31)", (long long)V);
  HCHECK(E >= 0 && indptr && (E == 0 || indices), HELIOS_E_INVALID, "bad E / null arrays");
  HCHECK(indptr[0] == 0 && indptr[V] == E, HELIOS_E_INVALID, "indptr[0]=%lld indptr[V]=%lld E=%lld",
         (long long)indptr[0], (long long)indptr[V], (long long)E);
  int ndev = 0;
  HCUDA(cudaGetDeviceCount(&ndev));
  HCHECK(device >= 0 && device < ndev, HELIOS_E_INVALID, "device %d of %d", device, ndev);
  DeviceGuard dg(device);
  helios_graph* g = new helios_graph();
  g->device = device;
  g->V = V;
  g->E = E;
  g->topo_host = (flags & HELIOS_GRAPH_TOPO_HOST) != 0;
  cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, device);
  auto cleanup = [&](helios_status st) {
    if (g->topo_host) {
      if (g->h_indptr) cudaFreeHost(g->h_indptr);
      if (g->h_indices) cudaFreeHost(g->h_indices);
    } else {
      if (g->indptr) cudaFree(g->indptr);
      if (g->indices) cudaFree(g->indices);
    }
    if (g->d_err) cudaFree(g->d_err);
    delete g;
    return st;
  };
  if (g->topo_host) {  // pinned, mapped host copy; kernels use the device aliases (zero-copy)
    if (cudaHostAlloc(&g->h_indptr, (V + 1) * 8, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostAlloc(&g->h_indices, std::max<int64_t>(E, 1) * 4, cudaHostAllocMapped) != cudaSuccess ||
        cudaMalloc(&g->d_err, sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return cleanup(fail(HELIOS_E_NOMEM, "pinned allocation of the CSR (%lld B) failed", (long long)(V * 8 + E * 4)));
    }
    memcpy(g->h_indptr, indptr, (V + 1) * 8);
    if (E > 0) memcpy(g->h_indices, indices, E * 4);
    if (cudaHostGetDevicePointer((void**)&g->indptr, g->h_indptr, 0) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&g->indices, g->h_indices, 0) != cudaSuccess ||
        cudaMemset(g->d_err, 0, sizeof(int)) != cudaSuccess)
      return cleanup(fail(HELIOS_E_CUDA, "mapping the host CSR failed: %s", cudaGetErrorString(cudaGetLastError())));
  } else {
    if (cudaMalloc(&g->indptr, (V + 1) * 8) != cudaSuccess ||
        cudaMalloc(&g->indices, std::max<int64_t>(E, 1) * 4) != cudaSuccess ||
        cudaMalloc(&g->d_err, sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return cleanup(fail(HELIOS_E_NOMEM, "device allocation of the CSR (%lld B) failed", (long long)(V * 8 + E * 4)));
    }
    if (cudaMemcpy(g->indptr, indptr, (V + 1) * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        (E > 0 && cudaMemcpy(g->indices, indices, E * 4, cudaMemcpyHostToDevice) != cudaSuccess) ||
        cudaMemset(g->d_err, 0, sizeof(int)) != cudaSuccess)
      return cleanup(fail(HELIOS_E_CUDA, "CSR upload failed: %s", cudaGetErrorString(cudaGetLastError())));
  }
  helios_status st = validate_csr_device(g->indptr, g->indices, V, E, g->d_err, 0);
  if (st != HELIOS_OK) return cleanup(st);
  helios_status lat = HELIOS_OK;
  if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(HELIOS_E_CUDA, "validate: %s", cudaGetErrorString(cudaGetLastError())));
  st = read_latched(g->d_err, &lat);
  if (st != HELIOS_OK) return cleanup(st);
  if (lat != HELIOS_OK)
    return cleanup(fail(lat, lat == HELIOS_E_RANGE ? "CSR index >= V" : "CSR indptr not monotone / inconsistent"));
  *out = g;
  return HELIOS_OK;
  GUARD_END
}

void helios_graph_free(helios_graph* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  cudaDeviceSynchronize();
  if (g->topo_host) {
    cudaFreeHost(g->h_indptr);
    cudaFreeHost(g->h_indices);
  } else {
    cudaFree(g->indptr);
    cudaFree(g->indices);
  }
  cudaFree(g->d_err);
  ws_free(g->ws);
  if (g->pre_mem) cudaFree(g->pre_mem);
  delete g;
}

helios_status helios_graph_info(const helios_graph* g, int64_t* V, int64_t* E, int* device) {
  HCHECK(g, HELIOS_E_INVALID, "null graph");
  if (V) *V = g->V;
  if (E) *E = g->E;
  if (device) *device = g->device;
  return HELIOS_OK;
}

helios_status helios_graph_device_csr(const helios_graph* g, const int64_t** indptr, const int32_t** indices) {
  HCHECK(g, HELIOS_E_INVALID, "null graph");
  if (indptr) *indptr = g->indptr;
  if (indices) *indices = g->indices;
  return HELIOS_OK;
}

helios_status helios_sample_bounds(int64_t n_seeds, const int32_t* fanouts, int32_t L, int64_t V, int64_t E,
                                   int64_t* max_nodes, int64_t* max_level_nodes, int64_t* max_edges) {
  GUARD_BEGIN
  return sample_bounds(n_seeds, fanouts, L, V, E, max_nodes, max_level_nodes, max_edges);
  GUARD_END
}

helios_status helios_sample(helios_graph* g, const int64_t* seeds, int64_t n_seeds, const int32_t* fanouts, int32_t L,
                            uint64_t key, const helios_blocks* out, void* stream) {
  GUARD_BEGIN
  HCHECK(g, HELIOS_E_INVALID, "null graph");
  DeviceGuard dg(g->device);
  return sample_default(g, seeds, n_seeds, fanouts, L, key, out, (cudaStream_t)stream);
  GUARD_END
}

helios_status helios_graph_probe_random(helios_graph* g, int64_t n_reads, int32_t reps, float* ms) {
  GUARD_BEGIN
  HCHECK(g, HELIOS_E_INVALID, "null graph");
  DeviceGuard dg(g->device);
  return probe_random_impl(g, n_reads, reps, ms);
  GUARD_END
}

helios_status helios_graph_sync(helios_graph* g, void* stream) {
  GUARD_BEGIN
  HCHECK(g, HELIOS_E_INVALID, "null graph");
  DeviceGuard dg(g->device);
  HCUDA(cudaStreamSynchronize((cudaStream_t)stream));
  helios_status lat = HELIOS_OK;
  helios_status st = read_latched(g->d_err, &lat);
  if (st != HELIOS_OK) return st;
  if (lat != HELIOS_OK) return fail(lat, "latched device error %d (seed out of range / duplicate seed)", (int)lat);
  return HELIOS_OK;
  GUARD_END
}

helios_status helios_presample(helios_graph* g, const int64_t* seeds, int64_t n_seeds, int32_t batch,
                               const int32_t* fanouts, int32_t L, const uint64_t* keys, uint64_t* hotness, void* stream) {
  GUARD_BEGIN
  HCHECK(g && hotness && keys && batch > 0 && (n_seeds == 0 || seeds), HELIOS_E_INVALID, "bad presample arguments");
  DeviceGuard dg(g->device);
  cudaStream_t st = (cudaStream_t)stream;
  int64_t maxn, lvl[HELIOS_MAX_HOPS + 1], edg[HELIOS_MAX_HOPS];
  helios_status s = sample_bounds(batch, fanouts, L, g->V, g->E, &maxn, lvl, edg);
  if (s != HELIOS_OK) return s;
  bool same = (g->pre_mem && g->pre_cap_B >= batch && g->pre_L == L);
  for (int h = 0; same && h < L; h++) same = (g->pre_fan[h] == fanouts[h]);
  if (!same) {
    HCUDA(cudaDeviceSynchronize());
    if (g->pre_mem) cudaFree(g->pre_mem);
    g->pre_mem = nullptr;
    size_t bytes = maxn * 8 + (L + 1) * 8 + HELIOS_MAX_HOPS * 8;
    for (int h = 0; h < L; h++) bytes += (lvl[h] + 1) * 4 + edg[h] * 4 + 64;
    HCUDA(cudaMalloc(&g->pre_mem, bytes));
    char* p = (char*)g->pre_mem;
    helios_blocks& b = g->pre_blocks;
    b = helios_blocks{};
    b.nodes = (int64_t*)p;
    b.nodes_cap = maxn;
    p += maxn * 8;
    b.level_counts = (int64_t*)p;
    p += (L + 1) * 8;
    b.edge_counts = (int64_t*)p;
    p += HELIOS_MAX_HOPS * 8;
    for (int h = 0; h < L; h++) {
      b.block_indptr[h] = (int32_t*)p;
      b.indptr_cap[h] = lvl[h] + 1;
      p += ((lvl[h] + 1) * 4 + 31) / 32 * 32;
      b.block_indices[h] = (int32_t*)p;
      b.edges_cap[h] = edg[h];
      p += (edg[h] * 4 + 31) / 32 * 32;
    }
    g->pre_cap_B = batch;
    g->pre_L = L;
    for (int h = 0; h < L; h++) g->pre_fan[h] = fanouts[h];
  }
  for (int64_t b = 0, i = 0; i < n_seeds; b++, i += batch) {
    int64_t nb = std::min<int64_t>(batch, n_seeds - i);
    s = sample_default(g, seeds + i, nb, fanouts, L, keys[b], &g->pre_blocks, st);
    if (s != HELIOS_OK) return s;
    s = hot_count_enqueue(g->pre_blocks.nodes, g->pre_blocks.level_counts + L, maxn, g->V, hotness, g->sms, st);
    if (s != HELIOS_OK) return s;
  }
  return HELIOS_OK;
  GUARD_END
}

helios_status helios_cache_build(helios_graph* g, const helios_cache_desc* d, helios_cache** out) {
  GUARD_BEGIN
  HCHECK(g && d && out, HELIOS_E_INVALID, "null argument");
  *out = nullptr;
  HCHECK(d->row_bytes > 0 && d->row_bytes % 16 == 0, HELIOS_E_INVALID, "row_bytes %d not a positive multiple of 16",
         d->row_bytes);
  HCHECK(d->world_size >= 1 && d->world_size <= HELIOS_MAX_RANKS && d->rank >= 0 && d->rank < d->world_size,
         HELIOS_E_INVALID, "rank %d / world_size %d", d->rank, d->world_size);
  HCHECK(d->hbm_rows >= 0 && d->host_rows >= 0, HELIOS_E_INVALID, "negative tier size");
  HCHECK(d->hotness, HELIOS_E_INVALID, "hotness is NULL");
  DeviceGuard dg(g->device);
  helios_cache* c = new helios_cache();
  helios_status st = cache_build_impl(g, d, c);
  if (st != HELIOS_OK) {
    std::string keep = helios_last_error();
    cache_free_impl(c);
    delete c;
    set_error(keep);
    return st;
  }
  *out = c;
  return HELIOS_OK;
  GUARD_END
}

void helios_cache_free(helios_cache* c) {
  if (!c) return;
  DeviceGuard dg(c->device);
  cache_free_impl(c);
  delete c;
}

helios_status helios_cache_query(const helios_cache* c, helios_cache_info* o) {
  HCHECK(c && o, HELIOS_E_INVALID, "null argument");
  o->dir = c->dir;
  o->hbm_tier = c->hbm;
  o->host_tier = c->host_tier;
  o->V = c->V;
  o->hbm_rows = c->H;
  o->host_rows = c->S;
  o->file_rows = c->file_rows;
  o->row_bytes = c->R;
  o->world_size = c->world;
  o->rank = c->world_rank;
  o->peers_attached = c->peers_attached;
  o->io_rings = c->io.rings;
  o->ring_depth = c->io.depth;
  o->direct_io = c->io.direct ? 1 : 0;
  o->io_reads = c->io.reads.load();
  o->staged_rows = stager_rows(c);
  o->io_sms = c->green_sms;
  return HELIOS_OK;
}

struct ExportBlob {
  uint32_t magic;
  int32_t rank, world, R;
  int64_t H;
  cudaIpcMemHandle_t handle;
};

helios_status helios_cache_export(helios_cache* c, void* blob, size_t* bytes) {
  GUARD_BEGIN
  HCHECK(c && bytes, HELIOS_E_INVALID, "null argument");
  if (!blob) {
    *bytes = sizeof(ExportBlob);
    return HELIOS_OK;
  }
  HCHECK(*bytes >= sizeof(ExportBlob), HELIOS_E_CAPACITY, "blob capacity %zu < %zu", *bytes, sizeof(ExportBlob));
  DeviceGuard dg(c->device);
  ExportBlob b{};
  b.magic = 0x48454C31u;
  b.rank = c->rank;
  b.world = c->G;
  b.R = c->R;
  b.H = c->H;
  HCUDA(cudaIpcGetMemHandle(&b.handle, c->hbm));
  memcpy(blob, &b, sizeof(b));
  *bytes = sizeof(b);
  return HELIOS_OK;
  GUARD_END
}

helios_status helios_cache_attach_peers(helios_cache* c, const void* blobs, size_t blob_bytes) {
  GUARD_BEGIN
  HCHECK(c && blobs && blob_bytes >= sizeof(ExportBlob), HELIOS_E_INVALID, "bad attach arguments");
  DeviceGuard dg(c->device);
  for (int r = 0; r < c->G; r++) {
    ExportBlob b;
    memcpy(&b, (const char*)blobs + (size_t)r * blob_bytes, sizeof(b));
    HCHECK(b.magic == 0x48454C31u && b.rank == r && b.world == c->G && b.R == c->R && b.H == c->H, HELIOS_E_INVALID,
           "blob %d inconsistent (rank %d world %d R %d H %lld)", r, b.rank, b.world, b.R, (long long)b.H);
    if (r == c->rank) continue;
    if (c->peer_ptrs[r]) continue;
    void* p = nullptr;
    HCUDA(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess));
    c->peer_ptrs[r] = (char*)p;
  }
  HCUDA(cudaMemcpy(c->d_peers, c->peer_ptrs, HELIOS_MAX_RANKS * sizeof(char*), cudaMemcpyHostToDevice));
  c->peers_attached = 1;
  return HELIOS_OK;
  GUARD_END
}

helios_status helios_gather(helios_cache* c, const int64_t* nodes, const int64_t* n_nodes, int64_t max_nodes, void* out,
                            helios_gather_stats* stats, void* stream) {
  GUARD_BEGIN
  HCHECK(c, HELIOS_E_INVALID, "null cache");
  DeviceGuard dg(c->device);
  helios_status st = gws_ensure(c, c->gws, max_nodes);
  if (st != HELIOS_OK) return st;
  st = gather_launch(c, c->gws, nodes, n_nodes, max_nodes, out, stats, (cudaStream_t)stream);
  if (st != HELIOS_OK) return st;
  return io_launch(c, c->gws, out, (cudaStream_t)stream);
  GUARD_END
}

helios_status helios_cache_probe_host(helios_cache* c, int64_t n_rows, uint64_t seed, int32_t reps, float* ms) {
  GUARD_BEGIN
  HCHECK(c, HELIOS_E_INVALID, "null cache");
  DeviceGuard dg(c->device);
  return probe_host_impl(c, n_rows, seed, reps, ms);
  GUARD_END
}

helios_status helios_cache_probe_link(helios_cache* c, int64_t n_rows, uint64_t seed, int32_t reps, float* ms,
                                      int32_t* best_depth) {
  GUARD_BEGIN
  HCHECK(c, HELIOS_E_INVALID, "null cache");
  DeviceGuard dg(c->device);
  return probe_link_impl(c, n_rows, seed, reps, ms, best_depth);
  GUARD_END
}

helios_status helios_batch_prepare(helios_graph* g, helios_cache* c, const int64_t* seeds, int64_t n_seeds,
                                   const int32_t* fanouts, int32_t L, uint64_t key, const helios_blocks* out,
                                   void* features, helios_gather_stats* stats, void* stream) {
  GUARD_BEGIN
  HCHECK(g && c && out, HELIOS_E_INVALID, "null argument");
  HCHECK(c->g == g, HELIOS_E_INVALID, "cache was built on another graph");
  DeviceGuard dg(g->device);
  cudaStream_t st = (cudaStream_t)stream;
  helios_status s = sample_default(g, seeds, n_seeds, fanouts, L, key, out, st);
  if (s != HELIOS_OK) return s;
  s = gws_ensure(c, c->gws, out->nodes_cap);
  if (s != HELIOS_OK) return s;
  s = gather_launch(c, c->gws, out->nodes, out->level_counts + L, out->nodes_cap, features, stats, st);
  if (s != HELIOS_OK) return s;
  return io_launch(c, c->gws, features, st);
  GUARD_END
}

helios_status helios_plan_create(helios_graph* g, helios_cache* c, const helios_plan_desc* d, helios_plan** out) {
  GUARD_BEGIN
  HCHECK(g && d && out, HELIOS_E_INVALID, "null argument");
  *out = nullptr;
  HCHECK(!c || c->g == g, HELIOS_E_INVALID, "cache was built on another graph");
  HCHECK(d->depth >= 1 && d->depth <= 32, HELIOS_E_INVALID, "plan depth %d not in [1,32]", d->depth);
  HCHECK(d->max_seeds >= 0, HELIOS_E_INVALID, "max_seeds < 0");
  DeviceGuard dg(g->device);
  helios_plan* p = new helios_plan();
  p->g = g;
  p->c = c;
  p->d = *d;
  p->graphs = !(d->flags & HELIOS_PLAN_NO_GRAPH);
  p->serial_gather = (d->flags & HELIOS_PLAN_SERIAL_GATHER) != 0;
  p->intra = (d->flags & HELIOS_PLAN_INTRA_BATCH) != 0;
  p->trace = (d->flags & HELIOS_PLAN_TRACE) != 0;
#ifndef HELIOS_TRACE
  if (p->trace) {
    delete p;
    return fail(HELIOS_E_INVALID, "HELIOS_PLAN_TRACE needs the traced build (libhelios_trace.so, HELIOS_LIB=trace)");
  }
#endif
  p->link = c && c->S > 0 && !p->intra && !p->serial_gather && (d->flags & HELIOS_PLAN_LINK_STREAM);
  HCHECK(!p->intra || p->graphs, HELIOS_E_INVALID, "HELIOS_PLAN_INTRA_BATCH needs CUDA graphs");
  p->G = d->group > 0 ? d->group : 1;
  if (const char* e = getenv("HELIOS_PLAN_TWO_GRAPHS")) p->two_graphs = atoi(e) != 0;
  if (p->G < 1 || p->G > kMaxGroup || (p->G > 1 && (p->intra || p->link || p->trace))) {
    const int G = p->G;
    delete p;
    return fail(HELIOS_E_INVALID, "plan group %d (need 1..%d, and 1 with INTRA_BATCH / LINK_STREAM / TRACE)", G,
                kMaxGroup);
  }
  helios_status st = plan_create_impl(p);
  if (st != HELIOS_OK) {
    std::string keep = helios_last_error();
    plan_free_impl(p);
    delete p;
    set_error(keep);
    return st;
  }
  *out = p;
  return HELIOS_OK;
  GUARD_END
}

void helios_plan_free(helios_plan* p) {
  if (!p) return;
  DeviceGuard dg(p->g->device);
  plan_free_impl(p);
  delete p;
}

helios_status helios_plan_outputs(helios_plan* p, int32_t slot, helios_blocks* blocks, void** features,
                                  helios_gather_stats** stats) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  return plan_outputs_impl(p, slot, blocks, features, stats);
  GUARD_END
}

helios_status helios_plan_submit(helios_plan* p, int32_t slot, const int64_t* seeds, int64_t n_seeds, uint64_t key,
                                 uint32_t flags, void* stream) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  DeviceGuard dg(p->g->device);
  return plan_submit_impl(p, slot, seeds, n_seeds, key, flags, (cudaStream_t)stream);
  GUARD_END
}

helios_status helios_plan_wait(helios_plan* p, int32_t slot, void* stream) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  DeviceGuard dg(p->g->device);
  return plan_wait_impl(p, slot, (cudaStream_t)stream);
  GUARD_END
}

helios_status helios_plan_timing(helios_plan* p, int32_t slot, int32_t back, helios_batch_timing* out) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  DeviceGuard dg(p->g->device);
  return plan_timing_impl(p, slot, back, out);
  GUARD_END
}

helios_status helios_plan_readback(helios_plan* p, int32_t slot, int64_t* out) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  DeviceGuard dg(p->g->device);
  return plan_readback_impl(p, slot, out);
  GUARD_END
}

helios_status helios_plan_trace(helios_plan* p, int32_t slot, int32_t back, uint64_t* out, int32_t cap,
                                int32_t* n_kernels) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  DeviceGuard dg(p->g->device);
  return plan_trace_impl(p, slot, back, out, cap, n_kernels);
  GUARD_END
}

helios_status helios_plan_mark(helios_plan* p, void* stream) {
  GUARD_BEGIN
  HCHECK(p, HELIOS_E_INVALID, "null plan");
  DeviceGuard dg(p->g->device);
  return plan_mark_impl(p, (cudaStream_t)stream);
  GUARD_END
}

helios_status helios_sync(helios_cache* c, void* stream) {
  GUARD_BEGIN
  HCHECK(c, HELIOS_E_INVALID, "null cache");
  DeviceGuard dg(c->device);
  HCUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (c->s_submit) HCUDA(cudaStreamSynchronize(c->s_submit));
  helios_status a = HELIOS_OK, b = HELIOS_OK;
  helios_status st = read_latched(c->d_err, &a);
  if (st != HELIOS_OK) return st;
  st = read_latched(c->g->d_err, &b);
  if (st != HELIOS_OK) return st;
  int host = c->io.host_err.exchange(0);
  if (a == HELIOS_E_TIMEOUT) c->broken = true;  // ring sequences / staging hand-offs are out of step
  if (a != HELIOS_OK) return fail(a, "latched cache error %d (IO failure or ring watchdog)", (int)a);
  if (host != 0) return fail((helios_status)host, "IO worker reported error %d", host);
  if (b != HELIOS_OK) return fail(b, "latched sampling error %d (seed out of range / duplicate seed)", (int)b);
  return HELIOS_OK;
  GUARD_END
}

}  // extern "C"
