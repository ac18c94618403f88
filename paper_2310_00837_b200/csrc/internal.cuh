// internal.cuh — shared internals of libhelios.so (device helpers, handle structs, error plumbing).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <functional>
#include <utility>
#include <cstdint>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "../../include/helios.h"

namespace helios {

// ---- error plumbing --------------------------------------------------------------------------
void set_error(const std::string& s);
helios_status fail(helios_status st, const char* fmt, ...);

#define HCUDA(call)                                                                           \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return ::helios::fail(HELIOS_E_CUDA, "%s:%d %s -> %s", __FILE__, __LINE__, #call,       \
                            cudaGetErrorString(e_));                                          \
  } while (0)

#define HCHECK(cond, st, ...)                                  \
  do {                                                         \
    if (!(cond)) return ::helios::fail((st), __VA_ARGS__);     \
  } while (0)

// Scoped "make device current" for entry points.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Programmatic dependent launch (sm_90+): the kernel may start launching while its predecessor in
// the stream drains; it must execute griddepcontrol.wait (pdl_wait) before touching the
// predecessor's results.  Captured into CUDA graphs as programmatic edges.
// HELIOS_NO_PDL=1 (read once): plain stream-ordered launches instead (ablation).
bool pdl_enabled();
struct PdlScope {  // launches inside the scope use PDL iff `enable` (and HELIOS_NO_PDL is not set)
  explicit PdlScope(bool enable);
  ~PdlScope();
  int prev;
};
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

constexpr int kMaxGroup = 4;                // batches per plan-slot group (one launch of each kernel)
constexpr uint32_t kEmpty = 0xFFFFFFFFu;  // empty hash key / unassigned local id / no minpos
constexpr int kScanBlock = 256;
#ifndef HELIOS_SCAN_ITEMS
#define HELIOS_SCAN_ITEMS 4  // items per thread of the count-scan / assign tiles (A/B builds: -DHELIOS_SCAN_ITEMS=n)
#endif
constexpr int kScanItems = HELIOS_SCAN_ITEMS;
constexpr int kScanTile = kScanBlock * kScanItems;

// Per-scan decoupled look-back state (reset to all-ones bytes before use).
struct ScanState {
  unsigned long long* status;  // [tiles]: all-ones = invalid; bit 62 set = inclusive; else aggregate
  unsigned int* counter;       // tile ticket (all-ones -> first ticket is 0)
};

// One slot of the per-batch open-addressing table (array of structs: an insert, its atomicMin and
// the later local-id reads all touch one 16 B slot, i.e. one 32 B sector, not three arrays).
// key and minpos share one 64-bit word (key in the high half): the insert's CAS claims a free slot
// with the edge position already in it, and a later occurrence lowers minpos with one 64-bit
// atomicMin (same key, so the word order is the position order) issued only when the word it read
// holds a larger position -- no separate read of `local` on the insert path.
struct alignas(16) TableSlot {
  unsigned long long km;  // (key << 32) | minpos; all-ones = free.  minpos: first edge position of an
                          // id new at this hop (meaningless once `local` is set)
  uint32_t local;         // local id in N_L once assigned, kEmpty = not yet
  uint32_t pad;
};
constexpr unsigned long long kEmptyKM = ~0ull;

// Sampling workspace: one per sampling context (the graph's default context, and one per plan
// slot so that consecutive batches can be in flight concurrently).
struct SampleWS {
  int64_t cap_edges = 0, cap_tiles_rows = 0, cap_tiles_edges = 0, cap_seeds = 0;
  uint32_t table_size = 0;   // power of two
  // one allocation: table | scan status | tile counters | barrier (table memset once, scan part per batch)
  char* reset_base = nullptr;
  size_t reset_bytes = 0;
  TableSlot* table = nullptr;
  ScanState row_scan[HELIOS_MAX_HOPS];
  ScanState edge_scan[HELIOS_MAX_HOPS];
  uint32_t* slot_of = nullptr;  // [cap_edges] hash slot of each sampled edge of the current hop
  uint32_t* node_slot = nullptr;  // [cap_nodes] hash slot of every node of the batch (table clear)
  int64_t cap_nodes = 0;
  // The table is all-EMPTY between batches: it is memset once at allocation and every batch
  // clears exactly the slots it occupied (k_table_clear); only the small scan-state region
  // [scan_base, scan_base + scan_bytes) is memset per batch.
  char* scan_base = nullptr;
  size_t scan_bytes = 0;
  unsigned* bar = nullptr;       // persistent-sampler grid barrier {arrivals, generation} (in the scan region)
  uint32_t* home = nullptr;      // home-region mask of the batch table (adaptive; written by the clear kernel)
  int cluster = 0;              // > 0: the whole batch in one launch of a cluster of this many CTAs
                                // (HELIOS_SAMPLE_MODE=cluster|cluster16|chain)
  // shared-memory tile dedup (HELIOS_SAMPLE_DEDUP=smem|global): hop h runs tiled when tile_rows[h] > 0
  int32_t tile_rows[HELIOS_MAX_HOPS] = {};
  uint2* elist = nullptr;        // [cap_edges] per-tile distinct entries {global slot, tile minpos}
  uint32_t* ndist = nullptr;     // [tiles] distinct ids per tile
  bool fill_seg = true;         // fill with f-lane segments (HELIOS_FILL_SEG=0: power-of-two lane groups)
  bool persistent = false;      // one cooperative kernel per batch instead of the 2+3L-kernel chain
                                // (HELIOS_SAMPLE_PERSISTENT=1; measured slower)
  // per-batch parameters, read by the kernels from device memory so that a captured CUDA graph
  // can be replayed for every batch: [0] key, [1] n_seeds, [2] seeds device pointer, [3] reserved,
  // [4, 4 + cap_seeds) inline seeds (host-seed submits: one H2D copy carries parameters + seeds)
  int64_t* d_params = nullptr;
  int64_t* h_params = nullptr;  // pinned staging for the parameter upload
  cudaEvent_t params_ev = nullptr;
};

// Per-gather bookkeeping (one per gather context): per-tier work lists written by the lookup
// kernel, and the ticket / count words shared with the gather and IO kernels.
enum : int { kListLocal = 0, kListPeer = 1, kListHost = 2, kListFile = 3, kLists = 4 };
enum : int { kCtlSubmit = 4, kCtlComplete = 5, kCtlStageSeq = 6, kCtlHostTicket = 7, kCtlDone = 8, kCtlWords = 9 };
// Which rows a k_gather_lists launch copies: every tier (one kernel), only the HBM tiers (local +
// peer), or only the host tier (zero-copy + staged rows; the plan's link stream).
enum : int { kPartAll = 0, kPartHbm = 1, kPartHost = 2 };
constexpr int kStageChunk = 64;              // rows per staging chunk (one state word each)
constexpr unsigned long long kChunkClaimed = 1, kChunkDone = 2;  // chunk state word: (seq << 2) | state
constexpr int64_t kStageCapRows = 1 << 16;   // staged rows per batch at most (the rest: zero-copy)
struct StageCtx;
struct Stager;
struct GatherWS {
  int64_t cap = 0;                      // rows per list
  int64_t* d_list_i = nullptr;          // [kLists * cap] output row of each entry
  uint64_t* d_list_w = nullptr;         // [kLists * cap] directory word of each entry
  unsigned long long* d_ctl = nullptr;  // [kCtlWords]: counts per list, IO tickets, staging split
  // HELIOS_CACHE_HOST_STAGED: the host list's directory words are mirrored into pinned memory for the
  // host stager threads, which copy 64-row chunks claimed from the list's end into a contiguous
  // pinned buffer.
  helios_cache* owner = nullptr;
  uint64_t* h_host_w = nullptr;         // pinned [cap] mirror of the host list's directory words (the
  uint64_t* d_host_w = nullptr;         //   stagers read it; device alias d_host_w, written by k_lookup)
  char* h_stage = nullptr;              // pinned [stage_rows, R]: chunk k from the list's end at row 64k
  char* d_stage = nullptr;
  int64_t stage_rows = 0;
  unsigned long long* h_chunk = nullptr;  // pinned [chunks]: (seq << 2) | kChunkClaimed / kChunkDone
  unsigned long long* d_chunk = nullptr;
  uint32_t* h_mail = nullptr;           // pinned {seq, n_host, -, -}, published by the GPU
  uint32_t* d_mail = nullptr;
  unsigned long long* h_hint = nullptr; // pinned (seq << 32) | chunk the GPU's host warps reached
  unsigned long long* d_hint = nullptr;
  uint32_t* d_seq = nullptr;            // device batch counter of this context
  bool ctl_preset = false;              // the plan zeroes d_ctl at the batch start (off the K2 -> K3 edge)
  const int64_t* trace_params = nullptr;  // HELIOS_PLAN_TRACE: the slot's parameter block (params[3] = trace row)
  int trace_idx = 0;                    // kernel position of K3 in the trace row (K4: +1)
  StageCtx* sctx = nullptr;
};

}  // namespace helios

struct helios_graph {
  int device = 0;
  int sms = 148;
  int64_t V = 0, E = 0;
  int64_t* indptr = nullptr;   // device [V+1] (device alias of pinned host memory with TOPO_HOST)
  int32_t* indices = nullptr;  // device [E]
  bool topo_host = false;      // CSR lives in pinned host memory (h_indptr / h_indices)
  int64_t* h_indptr = nullptr;
  int32_t* h_indices = nullptr;
  int* d_err = nullptr;        // device latched error (0 = none)
  helios::SampleWS ws;
  // presample scratch (lazily allocated)
  helios_blocks pre_blocks{};
  int64_t pre_cap_B = 0;
  int pre_L = -1;
  int32_t pre_fan[HELIOS_MAX_HOPS] = {};
  void* pre_mem = nullptr;
};

namespace helios {

// IO ring entry (SQ): 32 bytes, `seq` published last with release semantics (system scope).
struct alignas(32) SqEntry {
  uint64_t file_off;
  uint32_t len;
  uint32_t slot;
  uint64_t out_row;
  uint32_t seq;
  uint32_t rsvd;
};
struct alignas(8) CqEntry {
  uint32_t seq;     // == SqEntry.seq once the read landed in staging
  int32_t status;   // 0 ok, else HELIOS_E_IO
};

struct IoRings {
  int rings = 0, depth = 0;
  int64_t slot_bytes = 0;       // staging stride per slot (4096-aligned)
  SqEntry* sq = nullptr;        // pinned mapped [rings*depth]
  CqEntry* cq = nullptr;        // pinned mapped [rings*depth]
  char* staging = nullptr;      // pinned mapped [rings*depth*slot_bytes] (4096-aligned)
  SqEntry* d_sq = nullptr;      // device aliases of the above
  CqEntry* d_cq = nullptr;
  char* d_staging = nullptr;
  // device-side ring state
  uint32_t* d_free_seq = nullptr;   // [rings*depth] last sequence consumed by io_complete per slot
  uint32_t* d_base_seq = nullptr;   // [rings] sequences issued before the current batch
  // host workers
  std::vector<std::thread> workers;
  std::atomic<bool> stop{false};
  std::atomic<int> host_err{0};
  std::atomic<int64_t> reads{0};
  int fd = -1;
  bool direct = false;
  int64_t fault_at = 0;  // 1-based global read index to fail (tests), 0 = off
  std::atomic<int64_t> read_counter{0};
};

}  // namespace helios

struct helios_cache {
  helios_graph* g = nullptr;
  int device = 0;
  int sms = 148;
  int64_t V = 0;
  int32_t R = 0;
  int32_t G = 1, rank = 0;
  int64_t H = 0, S = 0, file_rows = 0;
  uint32_t flags = 0;
  int64_t* dir = nullptr;         // device [V]
  char* hbm = nullptr;            // device [H, R]
  char* host_tier = nullptr;      // host pointer
  char* d_host_tier = nullptr;    // device-mapped alias
  bool host_owned = false;        // packed host tier allocated by us
  bool host_tier_registered = false;  // we registered a caller-provided host tier
  bool host_registered = false;   // we registered host_table
  const void* host_table = nullptr;
  char** d_peers = nullptr;       // device [G] HBM shard base per rank (self included)
  char* peer_ptrs[HELIOS_MAX_RANKS] = {};
  int peers_attached = 0;
  int* d_err = nullptr;           // device latched error
  std::string path;
  int64_t header = 0, stride = 0;
  int world = 1, world_rank = 0;    // the caller's world size / rank (G, rank: the directory's)
  int io_ctas = 32;
  int gather_ctas = 148;            // K4 grid (one CTA per SM with a host tier, more for HBM-only caches)
  bool direct = true;               // HBM-only caches: lookup fused into the gather (HELIOS_GATHER_DIRECT=0: K3 + K4)
  bool split_host = true;           // host-tier rows in their own small kernel (HELIOS_GATHER_SPLIT_HOST=0: the
                                    // combined kernel, 2 host warps per 8)
  int gather_vu = 4;                // HBM / peer rows: 16-byte loads in flight per lane (HELIOS_GATHER_VU = 2/4/8/16;
                                    // 4: 80 registers, the footprint that leaves the sampler most room)
  bool gather_evict = true;         // HBM-only fused gather: evict-first L2 policy on its loads and stores (HELIOS_GATHER_EVICT=0: off)
  bool gather_evict_lists = false;  // K4 (tier lists): evict-first L2 policy on HBM / peer row copies (HELIOS_GATHER_EVICT_LISTS=1)
  int gather_async = 0;             // HBM-only fused gather: loads staged through a D-stage shared ring (HELIOS_GATHER_ASYNC=D, 4 or 8)
  bool gather_bulk = false;         // HELIOS_GATHER_BULK=1: HBM rows by cp.async.bulk (ablation)
  bool io_sync = false;            // HELIOS_CACHE_IO_SYNC ablation
  bool broken = false;             // a ring / staging watchdog fired: ring state is no longer consistent
  helios::IoRings io;
  bool has_file = false;
  // host staging (HELIOS_CACHE_HOST_STAGED)
  bool staged = false;
  float stage_frac = 1.0f;          // HOST_STAGED: share of a batch's host chunks the stagers may claim at most
  float stage_reserve = 0.0f;       // HOST_STAGED: share (from the list's end) the GPU leaves to the stagers
  int stage_workers = 8;
  helios::Stager* stager = nullptr;
  helios::GatherWS gws;            // default gather context (helios_gather / helios_batch_prepare)
  cudaStream_t s_submit = nullptr;  // IO stream: k_io of successive batches, serialised (ring sequences)
  void* green = nullptr;            // CUgreenCtx of the IO SM partition (io_sms > 0), s_submit belongs to it
  int green_sms = 0;                // SMs actually provisioned for it
  cudaEvent_t ev_lookup = nullptr, ev_submit = nullptr, ev_io_done = nullptr;
  bool io_pending = false;         // ev_io_done recorded at least once
};

#include <vector>
namespace helios {

struct PlanSlot {
  SampleWS ws;
  GatherWS gws;
  helios_blocks blocks{};
  void* mem = nullptr;
  char* feats = nullptr;
  helios_gather_stats* stats = nullptr;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t g_sample = nullptr, g_gather = nullptr, g_all = nullptr;
  cudaEvent_t ev_caller = nullptr, ev_end = nullptr;
  cudaStream_t s_side = nullptr;                        // intra-batch gather passes
  cudaEvent_t ev_fork[HELIOS_MAX_HOPS + 1] = {};
  cudaEvent_t ev_join = nullptr;
  cudaEvent_t ev_lk = nullptr, ev_host = nullptr;  // link mode: lookup done (slot) / host rows done (link)
  static constexpr int kRing = 1024;
  static constexpr int kEv = 5;   // per timed batch: {start, sampled, end} on the slot stream,
                                  // {host start, host end} on the link stream
  std::vector<cudaEvent_t> ring;  // kRing x kEv timing events (timed submits only)
  int64_t* h_rb = nullptr;        // pinned readback {level_counts[L+1], stats[4]} (HELIOS_SUBMIT_READBACK)
  static constexpr int kTraceRing = 256;
  void* d_trace = nullptr;        // HELIOS_PLAN_TRACE: kTraceRing rows of (3L+4) TraceRec
  bool rb_valid = false;          // the last submit requested a readback
  int64_t count = 0;              // batches submitted to this slot
  int64_t tcount = 0;             // timed batches submitted to this slot
  bool submitted = false;
  // plan groups (desc.group G > 1): every position has its own workspaces and outputs (above); the
  // group's first position (the leader) owns the stream, graphs and events used for all G.
  bool staged = false;            // parameters uploaded, group not launched yet
  bool rb_req = false;            // readback requested by this position's pending submit
};

}  // namespace helios

struct helios_plan {
  helios_graph* g = nullptr;
  helios_cache* c = nullptr;
  helios_plan_desc d{};
  int64_t maxn = 0;
  bool graphs = true;
  bool serial_gather = false;
  bool intra = false;  // HELIOS_PLAN_INTRA_BATCH
  // Link mode (HELIOS_PLAN_LINK_STREAM, opt-in ablation): the host-tier rows of every batch are
  // copied by one k_gather_lists<kPartHost> launch on a high-priority stream shared by all slots, so
  // the PCIe link serves one batch at a time; HBM rows stay on the slot stream.  Measured slower
  // than letting each slot's gather kernel read its own host rows.
  bool trace = false;  // HELIOS_PLAN_TRACE
  bool link = false;
  static constexpr int kMaxLinks = 4;
  int n_links = 1;                    // link streams used round-robin (HELIOS_PLAN_LINKS, 1..4)
  int64_t link_count = 0;             // batches submitted to the link streams
  cudaStream_t s_link[kMaxLinks] = {};
  cudaEvent_t ev_gather_chain = nullptr;  // last gather submitted (HELIOS_PLAN_SERIAL_GATHER)
  cudaEvent_t ev_ref = nullptr;           // helios_plan_mark: origin of the t_* timings
  bool marked = false;
  bool gather_chained = false;
  int G = 1;                              // batches per slot (desc.group); slots = depth x G positions
  bool two_graphs = false;                // HELIOS_PLAN_TWO_GRAPHS=1: untimed submits also launch the sampling
                                          // and gather graphs separately (as timed submits do)
  std::vector<helios::PlanSlot> slots;
};

namespace helios {

// Launch helpers implemented in the .cu files.
helios_status sample_bounds(int64_t n_seeds, const int32_t* fanouts, int32_t L, int64_t V, int64_t E,
                            int64_t* max_nodes, int64_t* level, int64_t* edges);
helios_status sample_check_out(const helios_graph* g, int64_t B, const int32_t* fanouts, int32_t L,
                               const helios_blocks* out);
helios_status ws_ensure(helios_graph* g, SampleWS& w, int64_t B, const int32_t* fanouts, int32_t L);
void ws_free(SampleWS& w);
// Uploads (key, n_seeds, seeds) into w.d_params on `st` with ONE copy (not capturable; done before
// a graph replay).  seeds_host: copy the seeds inline (host memory), else pass the device pointer.
helios_status ws_upload_params(SampleWS& w, uint64_t key, int64_t B, const int64_t* seeds, bool seeds_host,
                               cudaStream_t st, void* trace_row = nullptr);
// Enqueues the sampling kernels; they read key / n_seeds / seeds from w.d_params.  B_max sizes the grids.
// stage_hook (optional, multi-kernel path): called after the stream position where N_0 (stage 0) or
// N_{h+1} (stage h+1) is final, to fork per-range work (the intra-batch pipeline).
helios_status sample_launch(helios_graph* g, SampleWS& w, int64_t B_max, const int32_t* fanouts, int32_t L,
                            const helios_blocks* out, cudaStream_t st,
                            const std::function<helios_status(int)>* stage_hook = nullptr);
// n batches (1..kMaxGroup) in one launch of each kernel (gridDim.y = n); ws[b] / outs[b] per batch.
helios_status sample_launch_group(helios_graph* g, SampleWS* const* ws, const helios_blocks* const* outs, int n,
                                  int64_t B_max, const int32_t* fanouts, int32_t L, cudaStream_t st,
                                  const std::function<helios_status(int)>* hook = nullptr);
helios_status hot_count_enqueue(const int64_t* nodes, const int64_t* n_nodes, int64_t max_nodes, int64_t V, uint64_t* hot,
                                int sms, cudaStream_t st);
helios_status gws_ensure(helios_cache* c, GatherWS& w, int64_t max_nodes);
void gws_free(GatherWS& w);
// K3 lookup (per-tier lists) + K4 gather of the HBM / host tiers; FILE-tier rows stay in w's
// file list for io_launch.
helios_status gather_launch(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* n_nodes, int64_t max_nodes,
                            void* out, helios_gather_stats* stats, cudaStream_t st);
// The same for the n batches of a plan-slot group (one launch of each kernel, gridDim.y = n).
helios_status gather_launch_group(helios_cache* c, GatherWS* const* ws, const int64_t* const* nodes,
                                  const int64_t* const* n_nodes, int n, int64_t max_nodes, void* const* out,
                                  helios_gather_stats* const* stats, cudaStream_t st);
// Link mode, first half (slot stream): K3 lookup + K4 over the HBM tiers only (stats written).
helios_status gather_hbm_launch(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* n_nodes,
                                int64_t max_nodes, void* out, helios_gather_stats* stats, cudaStream_t st);
// Link mode, second half (link stream, after the first half): K4 over the host tier only.
helios_status gather_host_launch(helios_cache* c, GatherWS& w, void* out, cudaStream_t st);
// Intra-batch pipeline pass: lookup + gather of rows [*lo, *hi) (lo = NULL: from 0); stats
// accumulate, the file list accumulates (first = true resets everything).
helios_status gather_range_launch(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* lo,
                                  const int64_t* hi, int64_t max_rows, void* out, helios_gather_stats* stats, bool first,
                                  cudaStream_t st);
// Random-sector probe: mean device time (ms) of n uniformly random 4 B loads over the CSR indices.
helios_status probe_random_impl(helios_graph* g, int64_t n, int32_t reps, float* ms);
// Host-link probe: mean device time (ms) of K4's host part over n uniformly random host-tier rows.
helios_status probe_host_impl(helios_cache* c, int64_t n, uint64_t seed, int32_t reps, float* ms);
// Independent host-link probe (not K4): loads-only random-row kernel, best of 4 in-flight depths.
helios_status probe_link_impl(helios_cache* c, int64_t n, uint64_t seed, int32_t reps, float* ms, int32_t* best_depth);
// IO rings for the misses of the last gather_launch on `st` (not capturable: cross-stream events).
helios_status io_launch(helios_cache* c, GatherWS& w, void* out, cudaStream_t st);
helios_status validate_csr_device(const int64_t* indptr, const int32_t* indices, int64_t V, int64_t E, int* d_flag,
                                  cudaStream_t st);
helios_status cache_sort_and_dir(helios_cache* c, const uint64_t* hot, int32_t* d_order /*[V]*/);
helios_status gather_rows_by_id(const char* src_dev, int32_t R, const int32_t* ids, int64_t n, char* dst, int sms,
                                cudaStream_t st);
helios_status io_start(helios_cache* c, const helios_cache_desc* d);
void io_worker(helios_cache* c, int ring);  // host IO worker draining SQ ring `ring` (io_workers.cu)
helios_status io_preload_kernels();
void io_stop(helios_cache* c);
helios_status green_io_start(helios_cache* c, int device, int io_sms, int priority);  // green.cu
void green_io_stop(helios_cache* c);
helios_status stager_start(helios_cache* c);
void stager_stop(helios_cache* c);
int64_t stager_rows(const helios_cache* c);  // rows the stagers copied since build (0 without stagers)
helios_status stager_register(helios_cache* c, GatherWS& w);
void stager_unregister(helios_cache* c, GatherWS& w);

}  // namespace helios
