/* helios.h — C ABI v2 of libhelios.so: the B200 mini-batch preparation hot path of Helios
 * (arXiv 2310.00837): multi-hop uniform neighbour sampling over a CSR graph, dedup/relabel into
 * per-hop block CSRs, and feature extraction through a GPU-managed heterogeneous cache
 * (HBM tier, pinned-host tier read zero-copy, file tier served by GPU-initiated IO rings).
 *
 * Citations are PAPER.md line (= LaTeX paragraph) numbers with their section; "reading N" refers to
 * the numbered readings of the paper in DESIGN.md §Readings.
 *
 * Conventions for every entry point:
 *   - Plain pointers and sizes only.  "device" = CUDA device memory of the handle's device,
 *     "host" = ordinary host memory.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).
 *   - Ownership: inputs of *_load / *_build are copied (or, where stated, registered and borrowed);
 *     every output buffer is caller-owned and sized with helios_sample_bounds(); the library
 *     writes only within the capacities it is given.
 *   - Stream semantics: helios_sample / helios_gather / helios_batch_prepare / helios_presample
 *     only ENQUEUE work on `stream` (internal side streams are joined back with events);
 *     helios_graph_load / helios_cache_build / export / attach / *_sync / *_free block.
 *   - Errors: synchronous argument checks return immediately with a status; device-detected
 *     problems (seed out of range, duplicate seed, IO error, ring watchdog) are LATCHED in the
 *     handle and returned by the next helios_graph_sync / helios_sync — that batch's outputs are
 *     then undefined.  helios_last_error() gives a thread-local detail string.  No exception
 *     crosses the ABI; the library never calls exit().
 *   - Handles are not thread-safe: one handle per (process, device); calls on one handle must be
 *     issued from one host thread, and sample calls on one graph handle must be stream-ordered
 *     (they share the graph's sampling workspace).
 *   - IDs: int64 at the ABI (reading 11); V < 2^31 and CSR indices are int32.
 */
#ifndef HELIOS_H_
#define HELIOS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HELIOS_ABI_VERSION 2  /* 2: round 2 appended stage_reserve and io_sms to helios_cache_desc, io_sms to
                                  helios_cache_info and group to helios_plan_desc */
#define HELIOS_MAX_HOPS 8
#define HELIOS_MAX_RANKS 64

typedef enum {
  HELIOS_OK = 0,
  HELIOS_E_INVALID = 1,  /* malformed argument (bad CSR, row_bytes % 16, duplicate seed, ...) */
  HELIOS_E_RANGE = 2,    /* an id >= V */
  HELIOS_E_CAPACITY = 3, /* a caller buffer is smaller than helios_sample_bounds() requires */
  HELIOS_E_NOMEM = 4,    /* device / pinned allocation failed */
  HELIOS_E_CUDA = 5,     /* a CUDA runtime call failed (detail in helios_last_error) */
  HELIOS_E_IO = 6,       /* feature-file read failed or was short */
  HELIOS_E_TIMEOUT = 7,  /* IO ring watchdog fired (no completion within the bound) */
  HELIOS_E_STATE = 8     /* handle unusable after an earlier latched failure / wrong call order */
} helios_status;

typedef struct helios_graph helios_graph; /* opaque: device CSR + sampling workspace + latched error */
typedef struct helios_cache helios_cache; /* opaque: directory, tiers, IO rings, IO worker threads */

int helios_abi_version(void);
/* Thread-local detail of the last failing call on this thread ("" if none). */
const char* helios_last_error(void);

/* ---- Graph ---------------------------------------------------------------------------------
 * helios_graph_load: validates and uploads the CSR topology (the paper keeps "the entire topology
 * data" resident, §3.2.1; we keep it in HBM by default).
 *   device   CUDA device ordinal the handle lives on (made current for the call).
 *   V, E     vertex / edge counts; 1 <= V < 2^31, 0 <= E.
 *   indptr   host int64[V+1]: indptr[0] = 0, non-decreasing, indptr[V] = E  (else E_INVALID).
 *   indices  host int32[E]: neighbour ids, each in [0, V)  (else E_RANGE).  Copied.
 *   flags    0: the CSR is copied into HBM (default);
 *            HELIOS_GRAPH_TOPO_HOST: the CSR is copied into pinned, mapped host memory and the
 *            sampling kernels read it zero-copy over PCIe ("the entire topology data in the CPU
 *            cache", sampling via UVA: PAPER.md:206 §3.2.1, :215 §3.2.2).
 *   out      receives the handle (free with helios_graph_free).
 * Blocking.  Validation runs on the GPU after the copy. */
#define HELIOS_GRAPH_TOPO_HOST 0x1u
helios_status helios_graph_load(int device, int64_t V, int64_t E, const int64_t* indptr, const int32_t* indices,
                                uint32_t flags, helios_graph** out);
void helios_graph_free(helios_graph* g);
helios_status helios_graph_info(const helios_graph* g, int64_t* V, int64_t* E, int* device);
/* Device pointers of the resident CSR (for tests / zero-copy consumers); borrowed, valid until free. */
helios_status helios_graph_device_csr(const helios_graph* g, const int64_t** indptr, const int32_t** indices);

/* ---- Sampling (K1 sample_hop + K2 dedup_relabel) ------------------------------------------
 * Worst-case output sizes for a batch of n_seeds seeds with the given fanouts (f_h = -1: all
 * neighbours):  n_0 = n_seeds,  e_h <= min(n_h * f_h, E),  n_{h+1} <= min(V, n_h + e_h).
 *   max_level_nodes [L+1] host out: bound on n_h;  max_edges [L] host out: bound on e_h.
 *   *max_nodes = max_level_nodes[L]. */
helios_status helios_sample_bounds(int64_t n_seeds, const int32_t* fanouts, int32_t L, int64_t V, int64_t E,
                                   int64_t* max_nodes, int64_t* max_level_nodes, int64_t* max_edges);

/* Output of one sampled mini-batch ("batch generation", §3.3).  All
 * pointers are caller-owned DEVICE buffers; caps are element counts.
 *   nodes            int64[nodes_cap]: N_L — N_0 = seeds, then every newly reached id in
 *                    first-occurrence order over (hop, row, slot) (readings 5-6); N_h is a prefix.
 *   level_counts     int64[L+1]: n_0..n_L (device scalars written by the kernels).
 *   edge_counts      int64[L]: e_0..e_{L-1}.
 *   block_indptr[h]  int32[indptr_cap[h]] (>= n_h + 1): row i of hop h = frontier node N_h[i].
 *   block_indices[h] int32[edges_cap[h]]: local ids (rows of N_{h+1}) of the sampled neighbours,
 *                    slot order j = 0..k-1 within each row. */
typedef struct {
  int64_t* nodes;
  int64_t nodes_cap;
  int64_t* level_counts;
  int64_t* edge_counts;
  int32_t* block_indptr[HELIOS_MAX_HOPS];
  int64_t indptr_cap[HELIOS_MAX_HOPS];
  int32_t* block_indices[HELIOS_MAX_HOPS];
  int64_t edges_cap[HELIOS_MAX_HOPS];
} helios_blocks;

/* helios_sample: L-hop uniform neighbour sampling without replacement ("2-hop random neighbor
 * sampling", PAPER.md:292 §4.1; GPU sampling operator PAPER.md:215 §3.2.2, :239 §3.3).
 * For hop h and every row i < n_h (frontier = all of N_h, reading 5), v = N_h[i], d = deg(v),
 * k = min(d, f_h): all neighbours in CSR order if k == d, else Floyd's k-subset (reading 3) with
 * draws t_j = mulhi32(Philox4x32-10(ctr={j>>2, h, lo32 v, hi32 v}, key={lo32 key, hi32 key})[j&3],
 * d-k+j+1) (reading 2).  Then dedup/relabel into N_{h+1} (reading 6).
 *   g        graph handle.
 *   seeds    device int64[n_seeds], distinct, each < V (violations latched: E_INVALID / E_RANGE).
 *   fanouts  host int32[L], each >= 1 or -1.  L in [0, HELIOS_MAX_HOPS].
 *   key      64-bit batch key (keys are inputs; bench/test keys come from synth.batch_key).
 *   out      caller buffers with caps >= helios_sample_bounds() (else E_CAPACITY, nothing enqueued).
 * Enqueue-only on `stream`.  The graph's sampling workspace is allocated on first use for the
 * largest bounds seen (that first call synchronises the device). */
helios_status helios_sample(helios_graph* g, const int64_t* seeds, int64_t n_seeds, const int32_t* fanouts, int32_t L,
                            uint64_t key, const helios_blocks* out, void* stream);

/* Waits for `stream`, then returns and clears the graph's latched device error (HELIOS_OK if none). */
helios_status helios_graph_sync(helios_graph* g, void* stream);
/* Measurement aid (blocking): the random-sector ceiling the sampler sees.  `reps` launches of n_reads
 * independent uniformly random 4 B loads over the graph's CSR indices array (each touches one 32 B
 * sector; fresh positions every launch); *ms = mean device time per launch.  E_INVALID for
 * n_reads <= 0 or reps <= 0. */
helios_status helios_graph_probe_random(helios_graph* g, int64_t n_reads, int32_t reps, float* ms);

/* helios_presample: one pass of pre-sampling that "collects all vertices' hotness" (PAPER.md:212
 * §3.2.2 Cache Initialization; reading 8).  Seeds are split into consecutive batches of `batch`
 * (last one may be short); batch b is sampled with keys[b]; hotness[v] += 1 for every v in that
 * batch's N_L.
 *   seeds     device int64[n_seeds];  keys host uint64[ceil(n_seeds / batch)].
 *   hotness   device uint64[V], ACCUMULATED (zero it first; all-reduce across ranks if the
 *             presample pass is split over ranks — the Python layer does that over NCCL).
 * Enqueue-only. */
helios_status helios_presample(helios_graph* g, const int64_t* seeds, int64_t n_seeds, int32_t batch,
                               const int32_t* fanouts, int32_t L, const uint64_t* keys, uint64_t* hotness, void* stream);

/* ---- Heterogeneous cache (§3.2) ------------------------------------------
 * Directory word per vertex (int64): bits 63..62 tier (0 HBM, 1 HOST, 2 FILE),
 * bits 61..56 owner rank (HBM tier), bits 55..0 slot (HBM/HOST) or file row (FILE).
 * Placement (reading 9): order = vertices sorted by hotness desc, id asc; hot rank r:
 *   r <  G*H        -> HBM(owner = r mod G, slot = r div G)      G = world_size, H = hbm_rows
 *   r <  G*H + S    -> HOST(slot = (flags & HOST_ALIAS) ? v : r - G*H)            S = host_rows
 *   otherwise       -> FILE(row = v): bytes [header + v*stride, +row_bytes) of feature_path. */
#define HELIOS_CACHE_HOST_ALIAS 0x1u     /* host tier IS host_table (slot = v); no second copy   */
#define HELIOS_CACHE_TABLE_MAPPED 0x2u   /* host_table is already cudaHostRegister'ed + mapped   */
#define HELIOS_CACHE_NO_DIRECT_IO 0x4u   /* open feature_path without O_DIRECT                    */
#define HELIOS_CACHE_HOST_FILL 0x8u      /* fill the caller-provided host_tier (else assumed filled) */
#define HELIOS_CACHE_HOST_TIER_MAPPED 0x10u /* caller-provided host_tier already registered + mapped */
#define HELIOS_CACHE_HOST_STAGED 0x20u  /* dynamic split of every batch's host-tier rows: the GPU reads rows
                                           zero-copy from the front of the batch's host list while host
                                           stager threads copy 64-row chunks from its end into a contiguous
                                           pinned staging buffer that the GPU streams (
                                           reading 14).  The GPU still initiates every request. */
#define HELIOS_CACHE_IO_SYNC 0x40u      /* ablation: GIDS/BaM-style coupled IO, one warp per request does
                                           submit + completion poll + copy (§2.2)   */
#define HELIOS_CACHE_HBM_REPLICATED 0x200u /* C5-rep ablation: every rank's HBM tier holds the
                                           same hottest hbm_rows rows (directory of world_size 1: no peer
                                           rows, no NVLink traffic); host_rows then count from hot rank H */
#define HELIOS_CACHE_IO_FAULT_AT 0x100u  /* test builds: IO workers fail the io_fault_at-th read  */

typedef struct {
  int32_t row_bytes;          /* R = dim * 4 for fp32 features; multiple of 16 (else E_INVALID) */
  int32_t world_size, rank;   /* HBM tier sharded round-robin by hot rank over world_size GPUs  */
  int64_t hbm_rows;           /* H: HBM-tier rows held by EACH rank                              */
  int64_t host_rows;          /* S: pinned-host-tier rows (one shared tier)                      */
  const uint64_t* hotness;    /* device uint64[V] (helios_presample output, already all-reduced) */
  const void* host_table;     /* host: canonical rows, row v at host_table + v*R (V*R bytes), or NULL;
                                 borrowed (registered + mapped unless TABLE_MAPPED); must outlive the cache */
  const char* feature_path;   /* canonical feature file or NULL; required when G*H + S < V (FILE-tier rows
                                 are always read from it) or when no host_table is given to fill the tiers */
  int64_t header_bytes;       /* file: byte offset of row 0                                      */
  int64_t file_stride;        /* file: bytes between rows (>= R; 512-multiple for O_DIRECT)      */
  int32_t io_rings;           /* number of SQ/CQ ring pairs = host IO worker threads (>= 1)      */
  int32_t ring_depth;         /* entries per ring, power of two                                  */
  int32_t io_ctas;            /* CTA budget of each IO kernel (submit / complete); paper: 32 */
  int32_t io_fault_at;        /* with HELIOS_CACHE_IO_FAULT_AT: 1-based read index that fails   */
  uint32_t flags;
  void* host_tier;            /* optional caller-provided packed host tier (S*R bytes, e.g. a shared-memory
                                 mapping used by every rank): row s = vertex at hot rank G*H + s.  Filled by
                                 the library iff HELIOS_CACHE_HOST_FILL; registered unless HOST_TIER_MAPPED.
                                 NULL: the library allocates (pinned) and fills it.  Ignored with HOST_ALIAS. */
  int32_t stage_workers;      /* HOST_STAGED: host stager threads (0 = 8)                                */
  float stage_frac;           /* HOST_STAGED: cap on the share of each batch's host-row chunks the stagers
                                 may claim (0 = 1.0: no cap beyond the 2^16-row staging buffer)       */
  float stage_reserve;        /* HOST_STAGED: share of each batch's host-row chunks, counted from the list's
                                 end, that the GPU's host-row warps leave to the stagers: a warp reaching
                                 such a chunk waits up to 200 us for a stager to claim it (and the steal
                                 timeout for a claimed one) before copying it zero-copy itself.  0 = none:
                                 the pure dynamic split (whoever reaches a chunk first copies it).   */
  int32_t io_sms;             /* > 0 (with a file tier): run the IO kernel on a CUDA green context holding
                                 this many SMs (rounded up to the driver's granularity, 8 on sm_100), the
                                 in-process analog of the paper's MPS cap on operator SMs (PAPER.md:244,
                                 :352-357); everything else keeps the whole GPU.  0 = no partition.
                                 E_INVALID if the device cannot be split so; helios_cache_query reports
                                 the SMs provisioned. */
} helios_cache_desc;

/* Builds the directory and fills the tiers (blocking).  The HBM tier is filled from host_table
 * when given, else from feature_path; a packed host tier likewise.  Starts the IO workers when
 * any vertex is FILE-tier.  The graph handle must outlive the cache. */
helios_status helios_cache_build(helios_graph* g, const helios_cache_desc* desc, helios_cache** out);
void helios_cache_free(helios_cache* c);

typedef struct {
  const int64_t* dir;         /* device int64[V] directory                                      */
  const void* hbm_tier;       /* device [hbm_rows, R] this rank's shard                         */
  const void* host_tier;      /* host pointer of the host tier (alias of host_table or packed)   */
  int64_t V, hbm_rows, host_rows, file_rows;
  int32_t row_bytes, world_size, rank, peers_attached;
  int32_t io_rings, ring_depth, direct_io;
  int64_t io_reads;           /* file reads completed by the IO workers since build */
  int64_t staged_rows;        /* HOST_STAGED: host-tier rows copied by the stager threads since build */
  int32_t io_sms;             /* SMs of the IO green context (0 = the IO kernel may use every SM)   */
} helios_cache_info;
helios_status helios_cache_query(const helios_cache* c, helios_cache_info* out);

/* Multi-GPU: export this rank's HBM shard (CUDA IPC handle + sizes) into `blob`
 * (*bytes in: capacity, out: size; call with blob = NULL to get the size), all-gather the blobs
 * (Python layer, NCCL), then attach: blobs = world_size consecutive blobs of `blob_bytes` each, in
 * rank order.  After attach, HBM rows owned by peers are read directly over NVLink. */
helios_status helios_cache_export(helios_cache* c, void* blob, size_t* bytes);
helios_status helios_cache_attach_peers(helios_cache* c, const void* blobs, size_t blob_bytes);

/* ---- Feature extraction (K3 lookup + K4 gather + K5/K6 IO rings) -------------------------
 * out[i, :] = row(nodes[i]) for i < *n_nodes, byte for byte.
 *   nodes     device int64[max_nodes];  n_nodes device int64 scalar (e.g. level_counts + L).
 *   out       device [max_nodes, row_bytes];  stats device helios_gather_stats or NULL (overwritten).
 * Enqueue-only; FILE-tier rows go through the rings (thread-level submission, PAPER.md:167-172
 * §3.1.1; asynchronous completion, §3.1.2) on internal streams joined back. */
typedef struct {
  int64_t rows_hbm_local, rows_hbm_peer, rows_host, rows_file;
} helios_gather_stats;
/* Measurement aid (blocking): the host-link ceiling K4 sees for random host-tier rows.  Runs K4's
 * host-row part `reps` times, each over n_rows rows drawn uniformly from the host tier's address
 * range (fresh rows every rep, so no L2 reuse), into a scratch buffer; *ms = mean device time per
 * rep (CUDA events around the kernel).  E_INVALID for n_rows <= 0 or reps <= 0, E_STATE without a
 * host tier.  Library-owned scratch is freed before return. */
helios_status helios_cache_probe_host(helios_cache* c, int64_t n_rows, uint64_t seed, int32_t reps, float* ms);
/* Measurement aid (blocking): the same ceiling measured by a kernel that is NOT K4 — a loads-only
 * microkernel (no lists, no stores, no warp roles) reading n_rows uniformly random host-tier rows
 * (fresh rows every launch), swept over 8 settings of grid size x loads in flight per thread (about
 * 150 to 40 k rows in flight), `reps` launches each; *ms = the best mean device time per launch,
 * *best_depth (may be NULL) = the rows in flight of that setting.
 * E_INVALID for n_rows <= 0 or reps <= 0, E_STATE without a host tier. */
helios_status helios_cache_probe_link(helios_cache* c, int64_t n_rows, uint64_t seed, int32_t reps, float* ms,
                                      int32_t* best_depth);
helios_status helios_gather(helios_cache* c, const int64_t* nodes, const int64_t* n_nodes, int64_t max_nodes, void* out,
                            helios_gather_stats* stats, void* stream);

/* One whole mini-batch: helios_sample followed by helios_gather of N_L into `features`
 * (device [out->nodes_cap, row_bytes]).  Enqueue-only. */
helios_status helios_batch_prepare(helios_graph* g, helios_cache* c, const int64_t* seeds, int64_t n_seeds,
                                   const int32_t* fanouts, int32_t L, uint64_t key, const helios_blocks* out,
                                   void* features, helios_gather_stats* stats, void* stream);

/* ---- Execution plan: CUDA-graph replay + in-flight batch slots ------------------------------
 * The paper's runtime "decomposes GNN model execution into a sequence of GPU-initiated operators"
 * and builds an intra- and inter-mini-batch pipeline plan (§3.3).  A plan owns
 * `depth` slots; each slot has its own sampling workspace, output buffers, stream and a CUDA graph
 * of the whole batch (sampling kernels + lookup/gather), captured once at creation and replayed per
 * batch (key and n_seeds are read from device memory).  Batches submitted to different slots run
 * concurrently (sampling of batch i+1 overlaps the gather of batch i); FILE-tier IO of successive
 * batches is serialised on the cache's IO streams.
 *   desc.max_seeds   B: capacity of every slot (n_seeds <= B per submit).
 *   desc.L, fanouts  hops and fanouts (as helios_sample).
 *   desc.depth       number of slots, 1..32 (with CUDA_DEVICE_MAX_CONNECTIONS=32 every slot stream gets its own hardware queue).
 *   desc.flags       HELIOS_PLAN_NO_GRAPH: launch the kernels directly on every submit;
 *                    HELIOS_PLAN_SERIAL_GATHER: chain the gathers of successive submits;
 *                    HELIOS_PLAN_INTRA_BATCH: per-hop gather passes overlapping the sampling;
 *                    HELIOS_PLAN_LINK_STREAM: host rows on a shared link stream (see below).
 *   c                cache, or NULL for a sampling-only plan (no features / stats).
 * Link stream (HELIOS_PLAN_LINK_STREAM, when c has a host tier, without SERIAL_GATHER / INTRA_BATCH):
 * the host-tier rows of every batch are copied by one kernel on a high-priority stream shared by all
 * slots, in submission order, so the PCIe link serves one batch at a time with all of that batch's
 * reads in flight (PCIe is the host tier's bottleneck); the lookup and HBM rows stay
 * on the slot's stream.  An ablation: measured slower than the default.
 * Blocking create/free. */
#define HELIOS_PLAN_NO_GRAPH 0x1u
#define HELIOS_PLAN_SERIAL_GATHER 0x2u  /* gathers of successive batches run one at a time (sampling
                                           still overlaps): the link is not split between gathers */
#define HELIOS_PLAN_INTRA_BATCH 0x4u    /* intra-batch pipeline: a lookup + gather pass
                                           per new node range (N_0, then N_{h+1} \ N_h) forks onto a
                                           side stream while the next hop samples; timed submits then
                                           report the whole batch as the sampling phase */
#define HELIOS_PLAN_LINK_STREAM 0x8u    /* ablation: host-tier rows of every batch on a shared link stream */
#define HELIOS_PLAN_TRACE 0x10u         /* per-kernel device timeline of every batch (helios_plan_trace);
                                           only in the traced build libhelios_trace.so, else E_INVALID */
#define HELIOS_SUBMIT_SEEDS_HOST 0x1u  /* seeds pointer is host memory (copied with the parameters, H2D) */
#define HELIOS_SUBMIT_TIMING 0x2u      /* record device timing events around the sample / gather phases */
#define HELIOS_SUBMIT_READBACK 0x4u    /* copy the batch's level counts and tier stats to plan-owned pinned
                                          host memory at its end (read with helios_plan_readback) */
#define HELIOS_SUBMIT_FLUSH 0x8u       /* group > 1: launch the position's group now, even if not full */
typedef struct helios_plan helios_plan;
typedef struct {
  int64_t max_seeds;
  int32_t L;
  int32_t fanouts[HELIOS_MAX_HOPS];
  int32_t depth;
  uint32_t flags;
  int32_t group;   /* batches per slot, 1..4 (0 = 1).  With group G > 1 the plan has depth x G batch
                      POSITIONS (the `slot` argument of every plan call below is a position): positions
                      g*G .. g*G+G-1 form slot g, whose batches run as one group, each kernel of the
                      chain launched once for all G of them (gridDim.y = G, every batch with its own
                      table, scan state and outputs: results are those of G separate submits).  A
                      submit to the slot's last position launches the group, as does
                      HELIOS_SUBMIT_FLUSH or a helios_plan_wait on a position of a partly submitted
                      group (positions not submitted run as empty batches).  Timing is per group.
                      Not combinable with INTRA_BATCH, LINK_STREAM or TRACE (E_INVALID). */
} helios_plan_desc;
helios_status helios_plan_create(helios_graph* g, helios_cache* c, const helios_plan_desc* desc, helios_plan** out);
/* Free a plan before the cache and graph it was created on. */
void helios_plan_free(helios_plan* p);
/* Plan-owned DEVICE outputs of `slot` (valid until helios_plan_free): the slot's blocks, its
 * feature buffer [blocks->nodes_cap, row_bytes] (NULL without cache) and its gather stats. */
helios_status helios_plan_outputs(helios_plan* p, int32_t slot, helios_blocks* blocks, void** features,
                                  helios_gather_stats** stats);
/* Enqueue one batch into `slot`: ordered after all work already enqueued on `stream` (so the
 * caller may produce the seeds there and must have enqueued its consumption of the slot's previous
 * outputs there) and after the slot's previous batch.  seeds: device int64[n_seeds] (or host with
 * HELIOS_SUBMIT_SEEDS_HOST; copied before return is NOT guaranteed for device seeds — keep them
 * alive until the batch completes).  n_seeds <= desc.max_seeds (else E_CAPACITY). */
helios_status helios_plan_submit(helios_plan* p, int32_t slot, const int64_t* seeds, int64_t n_seeds, uint64_t key,
                                 uint32_t flags, void* stream);
/* Blocks until the last batch submitted to `slot` (with HELIOS_SUBMIT_READBACK) is done, then writes
 * its level counts and tier stats to host `out`: int64[L + 1 + 4] = n_0..n_L, rows_hbm_local,
 * rows_hbm_peer, rows_host, rows_file (stats 0 for a sample-only plan).  E_STATE if that batch was
 * not submitted with HELIOS_SUBMIT_READBACK. */
helios_status helios_plan_readback(helios_plan* p, int32_t slot, int64_t* out);
/* Makes `stream` wait for the last batch submitted to `slot`. */
helios_status helios_plan_wait(helios_plan* p, int32_t slot, void* stream);
/* Device timing of a batch submitted to `slot` with HELIOS_SUBMIT_TIMING: back = 0 is the slot's
 * last timed batch, back = k the k-th before it (k < 1024; CUDA events recorded around the two graph
 * segments, which are then launched as two graphs instead of one).  All values in ms:
 *   sample_ms   start of sampling -> end of sampling (slot stream);
 *   gather_ms   end of sampling -> end of the batch (lookup + gather + IO; in link mode including
 *               the wait for the link stream);
 *   link_ms     the batch's host-row kernel on the link stream, -1 without a link stream;
 *   t_start, t_gather, t_end   the batch's start / end of sampling / end, relative to the last
 *               helios_plan_mark (-1 if the plan was never marked), so a caller can form the union
 *               of busy intervals of overlapping batches.
 * Blocks until that batch is done; E_RANGE if it is not recorded. */
typedef struct {
  float sample_ms, gather_ms, link_ms;
  float t_start, t_gather, t_end;
} helios_batch_timing;
helios_status helios_plan_timing(helios_plan* p, int32_t slot, int32_t back, helios_batch_timing* out);
/* Device timeline of a batch of a plan created with HELIOS_PLAN_TRACE (tracing subsystem; nsys-free):
 * back = 0 is the slot's last batch, back = k the k-th before it (k < 256).  Blocks until the slot's
 * last batch is done.  out[2k], out[2k+1] = %globaltimer ns of the earliest warp start (after its
 * programmatic-dependency wait) and the latest warp end of kernel position k, 0 if it did not run:
 * k = 3h + {0, 1, 2} = count scan / fill / dedup-assign of hop h, 3L relabel, 3L+1 table clear,
 * 3L+2 lookup (K3), 3L+3 gather (K4).  *n_kernels = 3L + 4; E_CAPACITY if cap < 2 * (3L + 4),
 * E_STATE without HELIOS_PLAN_TRACE, E_RANGE if the batch is not in the ring. */
helios_status helios_plan_trace(helios_plan* p, int32_t slot, int32_t back, uint64_t* out, int32_t cap,
                                int32_t* n_kernels);
/* Records the plan's reference event on `stream` (the origin of helios_batch_timing's t_* values). */
helios_status helios_plan_mark(helios_plan* p, void* stream);

/* Waits for `stream` and the cache's IO streams; returns and clears latched errors of the cache
 * and its graph (E_IO, E_TIMEOUT, E_INVALID, E_RANGE).  After E_TIMEOUT the cache's ring state is
 * inconsistent and every later gather returns E_STATE (rebuild the cache). */
helios_status helios_sync(helios_cache* c, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HELIOS_H_ */
