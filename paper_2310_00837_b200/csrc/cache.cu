// cache.cu — heterogeneous cache construction (§3.2) and the host side of the
// IO rings (host IO workers draining the SQ rings with pread).
//
// Cache initialisation: hotness from a pre-sampling epoch (helios_presample), then
// "uses GPU to sort all vertices by their hotness in descending order" (stable radix sort on the
// GPU, ties by ascending id — reading 9), then the hottest rows fill the HBM tier (sharded
// round-robin by hot rank across world_size GPUs), the next S rows the pinned-host tier, and the
// rest stay in the feature file.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <sys/mman.h>
#include <immintrin.h>
#include <unistd.h>

#include "device.cuh"

namespace helios {

__global__ void k_iota_i32(int32_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (int32_t)i;
}

// Directory word of the vertex at hot rank r.
__global__ void k_make_dir(const int32_t* __restrict__ order, int64_t V, int32_t G, int64_t H, int64_t S,
                           int host_slot_is_id, int64_t* __restrict__ dir) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < V; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = order[r];
    uint64_t w;
    if (r < (int64_t)G * H) w = ((uint64_t)(r % G) << 56) | (uint64_t)(r / G);
    else if (r < (int64_t)G * H + S) w = (1ull << 62) | (uint64_t)(host_slot_is_id ? v : r - (int64_t)G * H);
    else w = (2ull << 62) | (uint64_t)v;
    dir[v] = (int64_t)w;
  }
}

// ids of this rank's HBM shard, in slot order: slot s <-> hot rank s*G + rank.
__global__ void k_shard_ids(const int32_t* __restrict__ order, int64_t n, int32_t G, int32_t rank,
                            int32_t* __restrict__ ids) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    ids[s] = order[s * G + rank];
}

helios_status cache_sort_and_dir(helios_cache* c, const uint64_t* hot, int32_t* d_order) {
  const int64_t V = c->V;
  HCHECK(V < (1ll << 31), HELIOS_E_INVALID, "V too large");
  uint64_t* keys_out = nullptr;
  int32_t* ids_in = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  HCUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp_bytes, (const uint64_t*)hot, keys_out,
                                                  (const int32_t*)ids_in, d_order, (int)V));
  HCUDA(cudaMalloc(&keys_out, V * 8));
  HCUDA(cudaMalloc(&ids_in, V * 4));
  HCUDA(cudaMalloc(&tmp, tmp_bytes));
  k_iota_i32<<<c->sms * 8, 256>>>(ids_in, V);
  // stable LSD radix sort: equal hotness keeps ascending id order
  HCUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, hot, keys_out, ids_in, d_order, (int)V));
  k_make_dir<<<c->sms * 8, 256>>>(d_order, V, c->G, c->H, c->S, (c->flags & HELIOS_CACHE_HOST_ALIAS) ? 1 : 0, c->dir);
  HCUDA(cudaGetLastError());
  HCUDA(cudaDeviceSynchronize());
  cudaFree(keys_out);
  cudaFree(ids_in);
  cudaFree(tmp);
  return HELIOS_OK;
}

// ---- host IO workers (io_workers.cu) ------------------------------------------------------

helios_status io_start(helios_cache* c, const helios_cache_desc* d) {
  IoRings& io = c->io;
  HCHECK(d->io_rings >= 1 && d->io_rings <= 256, HELIOS_E_INVALID, "io_rings %d", d->io_rings);
  HCHECK(d->ring_depth >= 2 && (d->ring_depth & (d->ring_depth - 1)) == 0, HELIOS_E_INVALID,
         "ring_depth %d not a power of two >= 2", d->ring_depth);
  HCHECK(c->stride >= c->R, HELIOS_E_INVALID, "file_stride < row_bytes");
  io.rings = d->io_rings;
  io.depth = d->ring_depth;
  io.slot_bytes = (c->stride + 4095) / 4096 * 4096;
  io.fault_at = (d->flags & HELIOS_CACHE_IO_FAULT_AT) ? d->io_fault_at : 0;
  const int64_t n = (int64_t)io.rings * io.depth;
  io.direct = false;
  if (!(d->flags & HELIOS_CACHE_NO_DIRECT_IO) && (c->stride % 512 == 0) && (c->header % 512 == 0)) {
    io.fd = open(c->path.c_str(), O_RDONLY | O_DIRECT);
    if (io.fd >= 0) io.direct = true;
  }
  if (io.fd < 0) io.fd = open(c->path.c_str(), O_RDONLY);
  HCHECK(io.fd >= 0, HELIOS_E_IO, "open(%s): %s", c->path.c_str(), strerror(errno));
  HCUDA(cudaHostAlloc(&io.sq, n * sizeof(SqEntry), cudaHostAllocMapped));
  HCUDA(cudaHostAlloc(&io.cq, n * sizeof(CqEntry), cudaHostAllocMapped));
  HCUDA(cudaHostAlloc(&io.staging, n * io.slot_bytes + 4096, cudaHostAllocMapped));
  memset(io.sq, 0, n * sizeof(SqEntry));
  memset(io.cq, 0, n * sizeof(CqEntry));
  HCUDA(cudaHostGetDevicePointer((void**)&io.d_sq, io.sq, 0));
  HCUDA(cudaHostGetDevicePointer((void**)&io.d_cq, io.cq, 0));
  HCUDA(cudaHostGetDevicePointer((void**)&io.d_staging, io.staging, 0));
  HCUDA(cudaMalloc(&io.d_free_seq, n * 4));
  HCUDA(cudaMemset(io.d_free_seq, 0, n * 4));
  HCUDA(cudaMalloc(&io.d_base_seq, io.rings * 4));
  HCUDA(cudaMemset(io.d_base_seq, 0, io.rings * 4));
  // O_DIRECT probe: one aligned read; fall back to buffered IO if the filesystem refuses it
  if (io.direct) {
    ssize_t got = pread(io.fd, io.staging, io.slot_bytes < 4096 ? 4096 : 4096, 0);
    if (got < 0) {
      close(io.fd);
      io.fd = open(c->path.c_str(), O_RDONLY);
      io.direct = false;
      HCHECK(io.fd >= 0, HELIOS_E_IO, "open(%s): %s", c->path.c_str(), strerror(errno));
    }
  }
  helios_status pst = io_preload_kernels();
  if (pst != HELIOS_OK) return pst;
  io.stop = false;
  for (int r = 0; r < io.rings; r++) io.workers.emplace_back(io_worker, c, r);
  return HELIOS_OK;
}

void io_stop(helios_cache* c) {
  IoRings& io = c->io;
  io.stop = true;
  for (auto& t : io.workers) t.join();
  io.workers.clear();
  if (io.fd >= 0) close(io.fd);
  io.fd = -1;
  if (io.sq) cudaFreeHost(io.sq);
  if (io.cq) cudaFreeHost(io.cq);
  if (io.staging) cudaFreeHost(io.staging);
  if (io.d_free_seq) cudaFree(io.d_free_seq);
  if (io.d_base_seq) cudaFree(io.d_base_seq);
  io.sq = nullptr;
  io.cq = nullptr;
  io.staging = nullptr;
  io.d_free_seq = io.d_base_seq = nullptr;
}

// ---- file reads for setup (tier fill) ------------------------------------------------------

static helios_status read_rows_from_file(const helios_cache* c, const int32_t* ids, int64_t n, char* dst_host) {
  int fd = open(c->path.c_str(), O_RDONLY);
  HCHECK(fd >= 0, HELIOS_E_IO, "open(%s): %s", c->path.c_str(), strerror(errno));
  std::atomic<int> bad{0};
  const int T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++)
    th.emplace_back([&, t]() {
      for (int64_t i = t; i < n; i += T) {
        ssize_t got = pread(fd, dst_host + i * c->R, c->R, (off_t)(c->header + (int64_t)ids[i] * c->stride));
        if (got != c->R) bad = 1;
      }
    });
  for (auto& x : th) x.join();
  close(fd);
  HCHECK(!bad, HELIOS_E_IO, "short read filling a tier from %s", c->path.c_str());
  return HELIOS_OK;
}

static helios_status fill_tier_from_file(helios_cache* c, const int32_t* h_ids, int64_t n, char* dst, bool dst_is_device) {
  const int64_t chunk = std::max<int64_t>(1, (256ll << 20) / c->R);
  char* buf = nullptr;
  if (dst_is_device) HCUDA(cudaHostAlloc(&buf, chunk * c->R, cudaHostAllocDefault));
  for (int64_t s = 0; s < n; s += chunk) {
    int64_t m = std::min(chunk, n - s);
    char* target = dst_is_device ? buf : dst + s * c->R;
    helios_status st = read_rows_from_file(c, h_ids + s, m, target);
    if (st != HELIOS_OK) {
      if (buf) cudaFreeHost(buf);
      return st;
    }
    if (dst_is_device) HCUDA(cudaMemcpy(dst + s * c->R, buf, m * c->R, cudaMemcpyHostToDevice));
  }
  if (buf) cudaFreeHost(buf);
  return HELIOS_OK;
}

// HBM tier fill from the (unregistered) canonical host table: host threads gather the rows of ids
// into one of two pinned chunks while the other chunk's copy to the GPU is in flight.
static helios_status fill_hbm_from_table(helios_cache* c, const int32_t* h_ids, int64_t n, char* dst) {
  const int64_t chunk_rows = std::max<int64_t>(1, (64ll << 20) / c->R);
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  helios_status s = HELIOS_OK;
  auto run = [&]() -> helios_status {
    for (int b = 0; b < 2; b++) {
      HCUDA(cudaHostAlloc(&buf[b], chunk_rows * (int64_t)c->R, cudaHostAllocDefault));
      HCUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    HCUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (int64_t k = 0, i0 = 0; i0 < n; k++, i0 += chunk_rows) {
      const int b = (int)(k & 1);
      const int64_t m = std::min(chunk_rows, n - i0);
      HCUDA(cudaEventSynchronize(ev[b]));  // the copy that last read this chunk is done
      std::vector<std::thread> th;
      for (int t = 0; t < T; t++)
        th.emplace_back([&, t]() {
          for (int64_t j = m * t / T; j < m * (t + 1) / T; j++)
            memcpy(buf[b] + j * c->R, (const char*)c->host_table + (int64_t)h_ids[i0 + j] * c->R, c->R);
        });
      for (auto& x : th) x.join();
      HCUDA(cudaMemcpyAsync(dst + i0 * (int64_t)c->R, buf[b], m * (int64_t)c->R, cudaMemcpyHostToDevice, st));
      HCUDA(cudaEventRecord(ev[b], st));
    }
    HCUDA(cudaStreamSynchronize(st));
    return HELIOS_OK;
  };
  s = run();
  if (st) cudaStreamSynchronize(st);
  for (int b = 0; b < 2; b++) {
    if (ev[b]) cudaEventDestroy(ev[b]);
    if (buf[b]) cudaFreeHost(buf[b]);
  }
  if (st) cudaStreamDestroy(st);
  return s;
}

helios_status cache_build_impl(helios_graph* g, const helios_cache_desc* d, helios_cache* c) {
  c->g = g;
  c->device = g->device;
  c->sms = g->sms;
  c->V = g->V;
  c->R = d->row_bytes;
  c->G = d->world_size;
  c->rank = d->rank;
  c->world = d->world_size;
  c->world_rank = d->rank;
  if (d->flags & HELIOS_CACHE_HBM_REPLICATED) {  // C5-rep: every rank holds the same hottest H rows, so
    c->G = 1;                                     // the directory is the single-GPU one (no peers)
    c->rank = 0;
  }
  c->H = d->hbm_rows;
  c->S = d->host_rows;
  c->flags = d->flags;
  c->host_table = d->host_table;
  c->path = d->feature_path ? d->feature_path : "";
  c->header = d->header_bytes;
  c->stride = d->file_stride > 0 ? d->file_stride : c->R;
  c->io_ctas = d->io_ctas > 0 ? d->io_ctas : 32;
  c->staged = (d->flags & HELIOS_CACHE_HOST_STAGED) != 0;
  c->io_sync = (d->flags & HELIOS_CACHE_IO_SYNC) != 0;
  c->stage_workers = d->stage_workers > 0 ? d->stage_workers : 8;
  c->stage_frac = d->stage_frac > 0.f ? std::min(d->stage_frac, 1.0f) : 1.0f;
  c->stage_reserve = d->stage_reserve > 0.f ? std::min(d->stage_reserve, c->stage_frac) : 0.0f;
  const int64_t V = c->V;
  // clamp tiers to V
  const int64_t GH = std::min<int64_t>((int64_t)c->G * c->H, V);
  c->S = std::min<int64_t>(c->S, V - GH);
  c->file_rows = V - GH - c->S;
  c->has_file = c->file_rows > 0;
  HCHECK(!c->has_file || !c->path.empty(), HELIOS_E_INVALID, "%lld FILE-tier rows but no feature_path",
         (long long)c->file_rows);
  const bool alias = (c->flags & HELIOS_CACHE_HOST_ALIAS) != 0;
  HCHECK(!alias || c->host_table, HELIOS_E_INVALID, "HOST_ALIAS needs host_table");
  HCHECK(c->host_table || !c->path.empty() || (c->H == 0 && c->S == 0), HELIOS_E_INVALID,
         "tiers need a source: host_table or feature_path");

  HCUDA(cudaMalloc(&c->d_err, sizeof(int)));
  HCUDA(cudaMemset(c->d_err, 0, sizeof(int)));
  HCUDA(cudaMalloc(&c->dir, V * 8));
  int32_t* d_order = nullptr;
  HCUDA(cudaMalloc(&d_order, V * 4));
  helios_status st = cache_sort_and_dir(c, d->hotness, d_order);
  if (st != HELIOS_OK) {
    cudaFree(d_order);
    return st;
  }
  // register the canonical host table (zero-copy source for fills and, with ALIAS, the host tier)
  char* table_dev = nullptr;
  // The canonical table is registered (pinned + mapped) only when the GPU reads it zero-copy, i.e. when
  // the host tier aliases it (HOST_ALIAS) or the caller mapped it already (TABLE_MAPPED).  Otherwise
  // the HBM shard is filled by host threads gathering its rows into pinned chunks copied to the GPU,
  // so a rank never pins the whole table (57 GB at C3) just to read its 1/G share of the hottest rows.
  if (c->host_table && (alias || (c->flags & HELIOS_CACHE_TABLE_MAPPED))) {
    if (!(c->flags & HELIOS_CACHE_TABLE_MAPPED)) {
      cudaError_t e = cudaHostRegister((void*)c->host_table, (size_t)V * c->R,
                                       cudaHostRegisterMapped | cudaHostRegisterReadOnly);
      if (e != cudaSuccess && e != cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        e = cudaHostRegister((void*)c->host_table, (size_t)V * c->R, cudaHostRegisterMapped);
      }
      if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();  // registered by the caller or another cache: borrow it, do not unregister
      } else if (e != cudaSuccess) {
        cudaFree(d_order);
        return fail(HELIOS_E_CUDA, "cudaHostRegister(host_table, %lld B): %s", (long long)V * c->R,
                    cudaGetErrorString(e));
      } else {
        c->host_registered = true;
      }
    }
    HCUDA(cudaHostGetDevicePointer((void**)&table_dev, (void*)c->host_table, 0));
  }
  // HBM shard: slots s with s*G + rank < G*H
  const int64_t H_eff = (GH > c->rank) ? (GH - c->rank + c->G - 1) / c->G : 0;
  HCUDA(cudaMalloc(&c->hbm, std::max<int64_t>(1, c->H) * (int64_t)c->R));
  if (H_eff > 0) {
    int32_t* d_ids = nullptr;
    HCUDA(cudaMalloc(&d_ids, H_eff * 4));
    k_shard_ids<<<c->sms * 4, 256>>>(d_order, H_eff, c->G, c->rank, d_ids);
    if (table_dev) {
      st = gather_rows_by_id(table_dev, c->R, d_ids, H_eff, c->hbm, c->sms, 0);
    } else if (c->host_table) {
      std::vector<int32_t> h_ids(H_eff);
      HCUDA(cudaMemcpy(h_ids.data(), d_ids, H_eff * 4, cudaMemcpyDeviceToHost));
      st = fill_hbm_from_table(c, h_ids.data(), H_eff, c->hbm);
    } else {
      std::vector<int32_t> h_ids(H_eff);
      HCUDA(cudaMemcpy(h_ids.data(), d_ids, H_eff * 4, cudaMemcpyDeviceToHost));
      st = fill_tier_from_file(c, h_ids.data(), H_eff, c->hbm, true);
    }
    HCUDA(cudaDeviceSynchronize());
    cudaFree(d_ids);
    if (st != HELIOS_OK) {
      cudaFree(d_order);
      return st;
    }
  }
  // host tier
  if (c->S > 0) {
    if (alias) {
      c->host_tier = (char*)c->host_table;
      c->d_host_tier = table_dev;
    } else {
      const size_t tier_bytes = (size_t)c->S * c->R;
      if (d->host_tier) {
        c->host_tier = (char*)d->host_tier;
        if (!(c->flags & HELIOS_CACHE_HOST_TIER_MAPPED)) {
          cudaError_t e = cudaHostRegister(c->host_tier, tier_bytes, cudaHostRegisterMapped);
          if (e == cudaErrorHostMemoryAlreadyRegistered) cudaGetLastError();
          else if (e != cudaSuccess) {
            cudaFree(d_order);
            return fail(HELIOS_E_CUDA, "cudaHostRegister(host_tier, %zu B): %s", tier_bytes, cudaGetErrorString(e));
          } else {
            c->host_tier_registered = true;
          }
        }
      } else {
        // anonymous memory with transparent huge pages, then pinned + mapped: the GPU reads it
        // zero-copy, and the host stagers' random row copies (HOST_STAGED) take 2 MB TLB entries
        // instead of a 4 KB page walk per row over the 51 GB tier
        void* m = mmap(nullptr, tier_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        HCHECK(m != MAP_FAILED, HELIOS_E_NOMEM, "mmap of the host tier (%zu B) failed", tier_bytes);
        madvise(m, tier_bytes, MADV_HUGEPAGE);
        cudaError_t e = cudaHostRegister(m, tier_bytes, cudaHostRegisterMapped);
        if (e != cudaSuccess) {
          munmap(m, tier_bytes);
          cudaGetLastError();
          return fail(HELIOS_E_NOMEM, "cudaHostRegister(host tier, %zu B): %s", tier_bytes, cudaGetErrorString(e));
        }
        c->host_tier = (char*)m;
        c->host_owned = true;
      }
      HCUDA(cudaHostGetDevicePointer((void**)&c->d_host_tier, c->host_tier, 0));
      if (!d->host_tier || (c->flags & HELIOS_CACHE_HOST_FILL)) {
        // packed in hot-rank order: slot s holds the vertex at hot rank G*H + s (reading 9), so the
        // warmest host rows share pages (translation locality of zero-copy reads)
        std::vector<int32_t> h_ids(c->S);
        HCUDA(cudaMemcpy(h_ids.data(), d_order + GH, c->S * 4, cudaMemcpyDeviceToHost));
        if (c->host_table) {
          const int T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
          std::vector<std::thread> th;
          for (int t = 0; t < T; t++)
            th.emplace_back([&, t]() {
              const int64_t lo = c->S * t / T, hi = c->S * (t + 1) / T;
              for (int64_t s = lo; s < hi; s++)
                memcpy(c->host_tier + s * c->R, (const char*)c->host_table + (int64_t)h_ids[s] * c->R, c->R);
            });
          for (auto& x : th) x.join();
        } else {
          st = fill_tier_from_file(c, h_ids.data(), c->S, c->host_tier, false);
          if (st != HELIOS_OK) {
            cudaFree(d_order);
            return st;
          }
        }
      }
    }
  }
  cudaFree(d_order);
  // peer table (self only until attach)
  HCUDA(cudaMalloc(&c->d_peers, HELIOS_MAX_RANKS * sizeof(char*)));
  HCUDA(cudaMemset(c->d_peers, 0, HELIOS_MAX_RANKS * sizeof(char*)));
  c->peer_ptrs[c->rank] = c->hbm;
  HCUDA(cudaMemcpy(c->d_peers, c->peer_ptrs, HELIOS_MAX_RANKS * sizeof(char*), cudaMemcpyHostToDevice));
  c->peers_attached = (c->G == 1);
  // streams / events for the IO kernels
  int lo, hi;
  HCUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  if (d->io_sms > 0 && c->has_file) {  // IO kernels confined to an SM partition (green context)
    int dev = 0;
    HCUDA(cudaGetDevice(&dev));
    st = green_io_start(c, dev, d->io_sms, hi);
    if (st != HELIOS_OK) return st;
  } else {
    HCUDA(cudaStreamCreateWithPriority(&c->s_submit, cudaStreamNonBlocking, hi));
  }
  HCUDA(cudaEventCreateWithFlags(&c->ev_lookup, cudaEventDisableTiming));
  HCUDA(cudaEventCreateWithFlags(&c->ev_submit, cudaEventDisableTiming));
  HCUDA(cudaEventCreateWithFlags(&c->ev_io_done, cudaEventDisableTiming));
  if (c->has_file) {
    st = io_start(c, d);
    if (st != HELIOS_OK) return st;
  }
  {  // K4 grid: one CTA per SM.  With host rows the gather is PCIe-latency bound; HBM-only, 2 CTAs per
     // SM make K4 alone faster (C2: 22.5 vs 30.6 us per launch) but the whole pipeline slower (C2
     // 28.6 k vs 30.2 k batches/s, profiles/r02/bench_c2_gather_grid.jsonl): the smaller footprint
     // leaves SM slots to the other batches' sampling kernels.
    int per_sm = 1;
    if (const char* e = getenv("HELIOS_GATHER_CTAS_PER_SM")) per_sm = std::max(1, std::min(atoi(e), 4));
    if (const char* e = getenv("HELIOS_GATHER_BULK")) c->gather_bulk = atoi(e) != 0;
    if (const char* e = getenv("HELIOS_GATHER_VU")) {
      const int v = atoi(e);
      c->gather_vu = (v == 16 || v == 4 || v == 2) ? v : 8;
    }
    if (const char* e = getenv("HELIOS_GATHER_SPLIT_HOST")) c->split_host = atoi(e) != 0;
    if (const char* e = getenv("HELIOS_GATHER_DIRECT")) c->direct = atoi(e) != 0;
    if (const char* e = getenv("HELIOS_GATHER_EVICT")) c->gather_evict = atoi(e) != 0;
    if (const char* e = getenv("HELIOS_GATHER_EVICT_LISTS")) c->gather_evict_lists = atoi(e) != 0;
    if (const char* e = getenv("HELIOS_GATHER_ASYNC")) c->gather_async = std::max(0, std::min(atoi(e), 8));
    if (c->gather_bulk) per_sm = 1;  // 192 KB of shared memory per CTA
    c->gather_ctas = c->sms * per_sm;
  }
  c->staged = c->staged && c->S > 0;
  if (c->staged) {
    st = stager_start(c);
    if (st != HELIOS_OK) return st;
  }
  return HELIOS_OK;
}

void cache_free_impl(helios_cache* c) {
  cudaDeviceSynchronize();
  io_stop(c);
  gws_free(c->gws);
  stager_stop(c);
  for (int r = 0; r < HELIOS_MAX_RANKS; r++)
    if (r != c->rank && c->peer_ptrs[r]) cudaIpcCloseMemHandle(c->peer_ptrs[r]);
  if (c->host_registered) cudaHostUnregister((void*)c->host_table);
  if (c->host_owned && c->host_tier) {
    cudaHostUnregister(c->host_tier);
    munmap(c->host_tier, (size_t)c->S * c->R);
  }
  if (c->host_tier_registered) cudaHostUnregister(c->host_tier);
  if (c->hbm) cudaFree(c->hbm);
  if (c->dir) cudaFree(c->dir);
  if (c->d_peers) cudaFree(c->d_peers);
  if (c->d_err) cudaFree(c->d_err);
  if (c->green) green_io_stop(c);
  if (c->s_submit) cudaStreamDestroy(c->s_submit);
  if (c->ev_lookup) cudaEventDestroy(c->ev_lookup);
  if (c->ev_submit) cudaEventDestroy(c->ev_submit);
  if (c->ev_io_done) cudaEventDestroy(c->ev_io_done);
}

}  // namespace helios
