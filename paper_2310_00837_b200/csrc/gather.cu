// gather.cu — K3 cache_lookup fused with K4 gather_rows, and the K5/K6 IO rings.
//
// k_lookup_gather<VPL,U>: one warp per row, U rows in flight per warp, VPL 16-byte vectors per lane
//   per row.  dir[v] resolves the row to its tier ("GPU threads directly access the
//   cached data in CPU memory by UVA ... or in GPU memory"): HBM (local shard or a peer shard read
//   over NVLink), HOST (pinned, mapped, read zero-copy over PCIe), or FILE (appended to the miss
//   list for the IO rings).  Per-tier row counts are warp-reduced into helios_gather_stats.
// k_io: the IO-request producer/consumer pair in one warp-specialised grid.  Submitter warps do
//   thread-level parallel IO command submission (§3.1.1) — every lane owns one
//   request, requests are striped over several SQ rings, the descriptor carries the file offset (the
//   "SSD logic block") and the staging slot (the "temporary IO buffer").  Completer warps do the
//   asynchronous completion handling (§3.1.2) — each warp claims a request, polls
//   its CQ entry (acquire, system scope), then moves the row from the staging slot into the output
//   feature buffer and frees the slot.
#include <algorithm>
#include <cstdlib>

#include "device.cuh"

namespace helios {

__device__ __forceinline__ void st_global_v4(int4* p, int4 v) {  // STG, not a generic ST (shuffled pointers)
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Evict-first variants (L2 cache policy from createpolicy): the gather's 2 x R bytes per row stream
// through L2 once, so marking them first-to-evict leaves the L2 to the sampler's tables and CSR sectors
// of the other batches in flight (HELIOS_GATHER_EVICT=1, HBM-only fused gather).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int4 ld_stream_ef(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_global_v4_ef(int4* p, int4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w),
               "l"(pol)
               : "memory");
}

// Base pointers of the four tier lists (device memory).  In staged mode the host list's directory
// words are mirrored into pinned memory (host_w_mirror) for the host stager threads.
struct ListPtrs {
  int64_t* i[kLists];
  uint64_t* w[kLists];
  uint64_t* host_w_mirror;
};

// K3: one thread per row of N_L: dir[v] -> tier list (local HBM / peer HBM / host / file), appended
// with warp-aggregated atomics.  The list counts are the per-tier row counts.
// Rows [*lo, *hi) of N_L (lo = NULL: from 0); the intra-batch pipeline runs one pass per node range.
struct LookupArgs {
  const int64_t* nodes;
  const int64_t* lo_ptr;
  const int64_t* n_nodes;
  const int64_t* dir;
  int64_t V;
  int32_t rank;
  ListPtrs L;
  unsigned long long* ctl;
  int* err;
  const int64_t* trace_params;
  int trace_idx;
};
struct LookupGroup {  // the batches of one launch (gridDim.y), as SampleGroup
  LookupArgs a[kMaxGroup];
};
__global__ void __launch_bounds__(256) k_lookup(const __grid_constant__ LookupGroup P) {
  const LookupArgs& A = P.a[blockIdx.y];
  const int64_t* __restrict__ nodes = A.nodes;
  const int64_t* __restrict__ dir = A.dir;
  const int64_t* lo_ptr = A.lo_ptr;
  const ListPtrs& L = A.L;
  unsigned long long* ctl = A.ctl;
  const int64_t V = A.V;
  const int32_t rank = A.rank;
  int* err = A.err;
  pdl_wait();  // N_L is final once the sampling chain's last kernel has completed
  pdl_trigger();
  TraceScope ts(A.trace_params, A.trace_idx);
  const int lane = threadIdx.x & 31;
  const int64_t lo = lo_ptr ? *lo_ptr : 0;
  const int64_t n = *A.n_nodes - lo;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < n; base += stride) {
    const int64_t i = lo + base + lane;
    int t = -1;
    uint64_t w = 0;
    if (base + lane < n) {
      const int64_t v = nodes[i];
      if ((uint64_t)v < (uint64_t)V) {
        w = (uint64_t)dir[v];
        const uint32_t tier = (uint32_t)(w >> 62);
        t = tier == 0 ? ((int)((w >> 56) & 63) == rank ? kListLocal : kListPeer) : (tier == 1 ? kListHost : kListFile);
      } else {  // a seed out of range (latched by the sampler too) or a bad id passed to helios_gather:
        latch(err, HELIOS_E_RANGE);  // no directory read, no row copied; the batch's output is undefined
      }
    }
#pragma unroll
    for (int q = 0; q < kLists; q++) {
      const unsigned m = __ballot_sync(0xFFFFFFFFu, t == q);
      if (m) {
        const int leader = __ffs(m) - 1;
        unsigned long long b = 0;
        if (lane == leader) b = atomicAdd(&ctl[q], (unsigned long long)__popc(m));
        b = __shfl_sync(0xFFFFFFFFu, b, leader);
        if (t == q) {
          const int64_t pos = (int64_t)b + __popc(m & ((1u << lane) - 1u));
          L.i[q][pos] = i;
          L.w[q][pos] = w;
          if (q == kListHost && L.host_w_mirror) L.host_w_mirror[pos] = w;
        }
      }
    }
  }
}

__device__ __forceinline__ void st_release_sys_u32_(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Staged mode (dynamic split): post the batch's mailbox {seq, n_host} (release,
// system scope) for the host stagers, which then claim 64-row chunks of the host list from its END
// while the GPU's host-row warps take rows from its FRONT (host_rows_dyn).
struct PublishGroup {
  unsigned long long* ctl[kMaxGroup];
  uint32_t* seq[kMaxGroup];
  uint32_t* mail[kMaxGroup];
};
__global__ void k_stage_publish(const __grid_constant__ PublishGroup P) {
  unsigned long long* ctl = P.ctl[blockIdx.y];
  uint32_t* seq_ctr = P.seq[blockIdx.y];
  uint32_t* mail = P.mail[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  const int64_t n_host = (int64_t)ctl[kListHost];
  const uint32_t seq = *seq_ctr + 1u;
  *seq_ctr = seq;
  ctl[kCtlStageSeq] = seq;
  mail[1] = (uint32_t)n_host;
  __threadfence_system();
  st_release_sys_u32_(&mail[0], seq);
}

struct GatherArgs {
  char* out;
  int32_t R;
  ListPtrs L;
  unsigned long long* ctl;  // list counts, staging split, host / stage row tickets
  int part;                 // kPartAll / kPartHbm / kPartHost
  int host_warps;           // kPartAll: zero-copy host-row warps per 8 warps
  bool staged;
  bool accumulate;          // intra-batch passes: add this pass's row counts to stats
  const char* stage;        // device alias of the pinned staging rows (chunk k from the list's end at row 64k)
  const unsigned long long* chunk;  // device alias of the per-chunk state words ((seq << 2) | CLAIMED / DONE)
  unsigned long long* hint; // device alias of the pinned front hint ((seq << 32) | chunk the GPU reached)
  float stage_reserve;      // share of the batch's chunks (from the list's end) left to the stagers
  int64_t stage_max_chunks; // chunks the staging buffer holds (the stagers never claim more)
  bool vu16;                // HBM / peer rows: 16 (else 8) 16-byte loads in flight per lane
  bool vu4;                 // HBM / peer rows: 4 loads in flight per lane (smaller register footprint)
  bool vu2;                 // HBM / peer rows: 2 loads in flight per lane
  bool evict;               // HBM / peer rows: evict-first L2 policy on the row loads and stores
  int* err;
  const char* hbm;          // this rank's shard
  char* const* peers;       // device [G]
  const char* host_dev;     // device alias of the host tier
  helios_gather_stats* stats;
  const int64_t* trace_params;  // HELIOS_PLAN_TRACE (nullptr: off)
  int trace_idx;
};

// Copies rows [j0, j0+U) of list q (warp-cooperative, VPL 16 B vectors per lane per row, all loads
// issued before the stores).
template <int VPL, int U>
__device__ __forceinline__ void copy_rows(const GatherArgs& a, int q, int64_t j0, int64_t cnt, int lane, int nvec) {
  for (int c0 = 0; c0 < nvec; c0 += 32 * VPL) {
    int4 r[U][VPL];
    const int4* src[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      src[u] = nullptr;
      if (j0 + u < cnt) {
        const uint64_t w = a.L.w[q][j0 + u];
        const int64_t slot = (int64_t)(w & ((1ull << 56) - 1));
        const char* base = q == kListLocal ? a.hbm : (q == kListPeer ? a.peers[(w >> 56) & 63] : a.host_dev);
        src[u] = (const int4*)(base + slot * a.R);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (src[u]) {
#pragma unroll
        for (int k = 0; k < VPL; k++) {
          const int idx = c0 + lane + 32 * k;
          if (idx < nvec) r[u][k] = ld_stream(src[u] + idx);
        }
      }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (src[u]) {
        int4* d = (int4*)(a.out + a.L.i[q][j0 + u] * (int64_t)a.R);
#pragma unroll
        for (int k = 0; k < VPL; k++) {
          const int idx = c0 + lane + 32 * k;
          if (idx < nvec) d[idx] = r[u][k];
        }
      }
  }
}

// HBM / NVLink-peer rows, flat mapping: a warp takes rw rows at a time and spreads their rw*nvec
// 16-byte vectors over its 32 lanes x VU registers (vector f -> row f / nvec, column f % nvec), so
// every lane is busy whatever the row size (R = 400 B: 25 vectors per row, 10 rows = 250 of 256
// slots) and each lane has VU independent loads in flight before its stores.  Lanes < rw resolve
// one row's source / destination pointers (list entry -> tier slot) and the others get them by
// shuffle; the list entries of the warp's NEXT group are loaded before this group's rows, so the
// list-read latency overlaps the row loads instead of preceding them.  rw = max(1, 32*VU/nvec); rows
// longer than 32*VU vectors take several passes.  inv = ceil(2^20 / nvec) (exact division for
// f * nvec < 2^20, which holds whenever rw > 1).
template <int VU>
__device__ __forceinline__ void flat_rows(const GatherArgs& a, int q, int64_t cnt, int64_t dw, int64_t n_dw, int lane,
                                          int nvec) {
  const int rw = max(1, 32 * VU / nvec);
  const uint32_t inv = ((1u << 20) + (uint32_t)nvec - 1u) / (uint32_t)nvec;
  const int64_t step = n_dw * rw;
  int64_t j0 = dw * rw;
  if (j0 >= cnt) return;
  const uint64_t* __restrict__ lw = a.L.w[q];
  const int64_t* __restrict__ li = a.L.i[q];
  auto resolve = [&](int64_t j, const char** sp, char** dp) {
    if (lane < rw && j + lane < cnt) {
      const uint64_t w = lw[j + lane];
      const char* base = q == kListLocal ? a.hbm : a.peers[(w >> 56) & 63];
      *sp = base + (int64_t)(w & ((1ull << 56) - 1)) * a.R;
      *dp = a.out + li[j + lane] * (int64_t)a.R;
    }
  };
  const char* sp = nullptr;
  char* dp = nullptr;
  resolve(j0, &sp, &dp);
  for (; j0 < cnt; j0 += step) {
    const char* sp_n = nullptr;
    char* dp_n = nullptr;
    if (j0 + step < cnt) resolve(j0 + step, &sp_n, &dp_n);  // next group's list entries, in flight now
    const int nrows = (int)min((int64_t)rw, cnt - j0);
    const int nv = nrows * nvec;
    for (int b0 = 0; b0 < nv; b0 += 32 * VU) {
      int4 r[VU];
#pragma unroll
      for (int k = 0; k < VU; k++) {
        const int f = b0 + lane + 32 * k;
        const int row = (rw == 1) ? 0 : min((int)(((uint32_t)f * inv) >> 20), rw - 1);
        const char* src = (const char*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)sp, row);
        if (f < nv) r[k] = a.evict ? ld_stream_ef((const int4*)src + (f - row * nvec), policy_evict_first())
                                   : ld_stream((const int4*)src + (f - row * nvec));
      }
#pragma unroll
      for (int k = 0; k < VU; k++) {
        const int f = b0 + lane + 32 * k;
        const int row = (rw == 1) ? 0 : min((int)(((uint32_t)f * inv) >> 20), rw - 1);
        char* dst = (char*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)dp, row);
        if (f < nv) {
          if (a.evict) st_global_v4_ef((int4*)dst + (f - row * nvec), r[k], policy_evict_first());
          else st_global_v4((int4*)dst + (f - row * nvec), r[k]);
        }
      }
    }
    sp = sp_n;
    dp = dp_n;
  }
}

// ---- fused lookup + gather for caches whose rows all live in HBM (C2: no host or file tier) -----------
// K3 exists to split N_L into per-tier lists; with every row in the HBM tier (local or a peer shard)
// there is nothing to split, so one kernel resolves dir[v] and copies the row, with K4's flat 16-byte
// mapping: lanes < rw read nodes[lo + j] and dir[v] of the warp's next rows (in flight while the current
// rows load), and out row = lo + j.  Per-tier row counts go to the ctl words (one atomic per warp
// group); the last CTA to finish writes the stats.  Out-of-range ids latch E_RANGE and copy nothing,
// as k_lookup does.
struct DirectArgs {
  const int64_t* nodes;
  const int64_t* lo_ptr;
  const int64_t* n_nodes;
  const int64_t* dir;
  int64_t V;
  int32_t rank;
};
struct DirectGroup {
  GatherArgs a[kMaxGroup];
  DirectArgs d[kMaxGroup];
};
// Per-tier counts of a fused lookup + gather: warp sums, one atomic per warp, then the last CTA
// publishes the stats.
__device__ __forceinline__ void direct_counts_publish(const GatherArgs& a, unsigned long long n_local,
                                                      unsigned long long n_peer, int lane) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_local += __shfl_xor_sync(0xFFFFFFFFu, n_local, o);
    n_peer += __shfl_xor_sync(0xFFFFFFFFu, n_peer, o);
  }
  if (lane == 0) {
    if (n_local) atomicAdd(&a.ctl[kListLocal], n_local);
    if (n_peer) atomicAdd(&a.ctl[kListPeer], n_peer);
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.stats) {
    __threadfence();
    const unsigned long long t = atomicAdd(&a.ctl[kCtlDone], 1ull);
    if (t == gridDim.x - 1) {  // every CTA's counts are in
      __threadfence();
      const int64_t nl = (int64_t)ld_volatile_u64(&a.ctl[kListLocal]), np = (int64_t)ld_volatile_u64(&a.ctl[kListPeer]);
      if (a.accumulate) {
        a.stats->rows_hbm_local += nl;
        a.stats->rows_hbm_peer += np;
      } else {
        a.stats->rows_hbm_local = nl;
        a.stats->rows_hbm_peer = np;
        a.stats->rows_host = 0;
      }
      a.stats->rows_file = 0;
    }
  }
}

template <int VU, bool EF>
__global__ void __launch_bounds__(256, VU == 4 ? 3 : 2) k_gather_direct(const __grid_constant__ DirectGroup P) {
  const GatherArgs& a = P.a[blockIdx.y];
  const DirectArgs& D = P.d[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(a.trace_params, a.trace_idx);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nvec = a.R >> 4;
  const int64_t lo = D.lo_ptr ? *D.lo_ptr : 0;
  const int64_t cnt = *D.n_nodes - lo;
  const int rw = max(1, 32 * VU / nvec);
  const uint32_t inv = ((1u << 20) + (uint32_t)nvec - 1u) / (uint32_t)nvec;
  const int64_t step = nw * rw;
  const uint64_t pol = EF ? policy_evict_first() : 0;
  unsigned long long n_local = 0, n_peer = 0;
  auto resolve = [&](int64_t j, const char** sp, char** dp) {
    *sp = nullptr;
    *dp = nullptr;
    if (lane < rw && j + lane < cnt) {
      const int64_t i = lo + j + lane;
      const int64_t v = D.nodes[i];
      if ((uint64_t)v < (uint64_t)D.V) {
        const uint64_t w = (uint64_t)D.dir[v];
        const int owner = (int)((w >> 56) & 63);
        const char* base = owner == D.rank ? a.hbm : a.peers[owner];
        *sp = base + (int64_t)(w & ((1ull << 56) - 1)) * a.R;
        *dp = a.out + i * (int64_t)a.R;
        if (owner == D.rank) n_local++;
        else n_peer++;
      } else {
        latch(a.err, HELIOS_E_RANGE);
      }
    }
  };
  int64_t j0 = gw * rw;
  const char* sp = nullptr;
  char* dp = nullptr;
  if (j0 < cnt) resolve(j0, &sp, &dp);
  for (; j0 < cnt; j0 += step) {
    const char* sp_n = nullptr;
    char* dp_n = nullptr;
    if (j0 + step < cnt) resolve(j0 + step, &sp_n, &dp_n);
    const int nrows = (int)min((int64_t)rw, cnt - j0);
    const int nv = nrows * nvec;
    for (int b0 = 0; b0 < nv; b0 += 32 * VU) {
      int4 r[VU];
#pragma unroll
      for (int k = 0; k < VU; k++) {
        const int f = b0 + lane + 32 * k;
        const int row = (rw == 1) ? 0 : min((int)(((uint32_t)f * inv) >> 20), rw - 1);
        const char* src = (const char*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)sp, row);
        if (f < nv && src) r[k] = EF ? ld_stream_ef((const int4*)src + (f - row * nvec), pol) : ld_stream((const int4*)src + (f - row * nvec));
      }
#pragma unroll
      for (int k = 0; k < VU; k++) {
        const int f = b0 + lane + 32 * k;
        const int row = (rw == 1) ? 0 : min((int)(((uint32_t)f * inv) >> 20), rw - 1);
        char* dst = (char*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)dp, row);
        if (f < nv && dst) {
          if (EF) st_global_v4_ef((int4*)dst + (f - row * nvec), r[k], pol);
          else st_global_v4((int4*)dst + (f - row * nvec), r[k]);
        }
      }
    }
    sp = sp_n;
    dp = dp_n;
  }
  direct_counts_publish(a, n_local, n_peer, lane);
}

// ---- fused lookup + gather with the loads staged through shared memory (HELIOS_GATHER_ASYNC=D) --------
// The same flat 16-byte mapping as k_gather_direct<VU>, but the loads are cp.async (SASS LDGSTS) into a
// per-warp shared-memory ring of D stages instead of registers: a lane keeps D x VU 16-byte loads in
// flight (D = 4, VU = 4: 256 B per lane, 64 KB per 256-thread CTA, four times the register path's)
// while holding only the D groups' destination pointers in registers.  Group t is issued into stage
// t mod D; once D groups are committed the oldest is complete (cp.async.wait_group D-1) and each lane
// stores the vectors IT loaded (no cross-lane shared-memory traffic, so no barrier).  Node ids of
// group t+2 and directory words of group t+1 are loaded while group t's rows are issued.  Requires
// nvec <= 32 * VU (one pass per group: R <= 2 KB at VU = 4); larger rows take k_gather_direct.
// Measured (C2, profiles/r02/k4_async.jsonl, gather_async_window_c2.jsonl): alone no faster than the
// register path at the same grid (30.6 vs 30.5 us at 1 CTA per SM, 21.3 vs 20.3 at 2), and the whole
// C2 step drops from 33.0 k to 20.6 k (D = 4) / 24.9 k (D = 8) batches/s: a 74-147 KB shared-memory
// CTA needs an SM carve-out the sampler kernels' CTAs (little shared memory) do not share, so they
// stop co-residing with the gather.  Kept as an opt-in ablation.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ int4 ld_shared_v4(const int4* p) {
  int4 r;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return r;
}

template <int VU, int D>
__global__ void __launch_bounds__(256, 3) k_gather_direct_async(const __grid_constant__ DirectGroup P) {
  extern __shared__ int4 s_ring[];  // [warp][D][VU][32] row vectors, then [warp][D][32] destination rows
  const GatherArgs& a = P.a[blockIdx.y];
  const DirectArgs& Dg = P.d[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(a.trace_params, a.trace_idx);
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  int4* ring = s_ring + wid * (D * VU * 32);
  char** s_dst = reinterpret_cast<char**>(s_ring + (blockDim.x >> 5) * (D * VU * 32)) + wid * (D * 32);
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nvec = a.R >> 4;
  const int64_t lo = Dg.lo_ptr ? *Dg.lo_ptr : 0;
  const int64_t cnt = *Dg.n_nodes - lo;
  const int rw = max(1, 32 * VU / nvec);
  const uint32_t inv = ((1u << 20) + (uint32_t)nvec - 1u) / (uint32_t)nvec;
  const int64_t step = nw * rw;
  const int64_t j0 = gw * rw;
  const int64_t ng = (j0 < cnt) ? (cnt - j0 + step - 1) / step : 0;  // groups of this warp
  unsigned long long n_local = 0, n_peer = 0;
  // row of group t owned by this lane (lanes < rw): node id 2 groups ahead, pointers 1 group ahead
  auto node_of = [&](int64_t t) -> int64_t {
    const int64_t j = j0 + t * step + lane;
    return (t < ng && lane < rw && j < cnt) ? Dg.nodes[lo + j] : -1;
  };
  auto resolve = [&](int64_t t, int64_t v, const char** sp, char** dp) {
    *sp = nullptr;
    *dp = nullptr;
    const int64_t j = j0 + t * step + lane;
    if (t < ng && lane < rw && j < cnt) {
      if ((uint64_t)v < (uint64_t)Dg.V) {
        const uint64_t w = (uint64_t)Dg.dir[v];
        const int owner = (int)((w >> 56) & 63);
        const char* base = owner == Dg.rank ? a.hbm : a.peers[owner];
        *sp = base + (int64_t)(w & ((1ull << 56) - 1)) * a.R;
        *dp = a.out + (lo + j) * (int64_t)a.R;
        if (owner == Dg.rank) n_local++;
        else n_peer++;
      } else {
        latch(a.err, HELIOS_E_RANGE);
      }
    }
  };
  const char* sp = nullptr;
  char* dp = nullptr;
  resolve(0, node_of(0), &sp, &dp);
  int64_t v_n = node_of(1);
  int s = 0;  // stage of group t
  for (int64_t t = 0; t < ng + D - 1; t++) {
    if (t < ng) {  // issue group t into stage s
      const int64_t v_nn = node_of(t + 2);
      const char* sp_n;
      char* dp_n;
      resolve(t + 1, v_n, &sp_n, &dp_n);
      const int nv = (int)min((int64_t)rw, cnt - (j0 + t * step)) * nvec;
      int4* st = ring + s * (VU * 32);
#pragma unroll
      for (int k = 0; k < VU; k++) {
        const int f = lane + 32 * k;
        const int row = (rw == 1) ? 0 : min((int)(((uint32_t)f * inv) >> 20), rw - 1);
        const char* src = (const char*)__shfl_sync(0xFFFFFFFFu, (unsigned long long)sp, row);
        if (f < nv && src) cp_async16(st + lane + 32 * k, (const int4*)src + (f - row * nvec));
      }
      if (lane < rw) s_dst[s * 32 + lane] = dp;
      sp = sp_n;
      dp = dp_n;
      v_n = v_nn;
    }
    cp_async_commit();
    s = (s + 1 == D) ? 0 : s + 1;  // = the stage of group t - (D - 1), the oldest in flight
    const int64_t tc = t - (D - 1);
    if (tc >= 0) {  // complete and store group tc (tc < ng always: t < ng + D - 1)
      cp_async_wait<D - 1>();
      __syncwarp();
      const int nv = (int)min((int64_t)rw, cnt - (j0 + tc * step)) * nvec;
      const int4* st = ring + s * (VU * 32);
#pragma unroll
      for (int k = 0; k < VU; k++) {
        const int f = lane + 32 * k;
        const int row = (rw == 1) ? 0 : min((int)(((uint32_t)f * inv) >> 20), rw - 1);
        char* dst = s_dst[s * 32 + row];
        if (f < nv && dst) st_global_v4((int4*)dst + (f - row * nvec), ld_shared_v4(st + lane + 32 * k));
      }
      __syncwarp();
    }
  }
  cp_async_wait<0>();
  direct_counts_publish(a, n_local, n_peer, lane);
}

// ---- bulk-copy (TMA engine) variant of the HBM / peer row copy (HELIOS_GATHER_BULK=1) ----------
// Rows move global -> shared -> global with cp.async.bulk (SASS UBLKCP): no register staging, and up
// to kBulkWarpBytes per warp in flight per direction.  Lane l of a warp owns row slot l of each of
// the warp's two shared-memory stages: it issues that row's bulk load (completing on the stage's
// mbarrier, armed with the group's byte count by lane 0) and, once the mbarrier phase completes,
// the row's bulk store; the stage is reloaded only after the lane's own earlier store finished
// reading it (cp.async.bulk.wait_group.read).  Loads of group g+1 overlap the stores of group g.
constexpr int kBulkWarpBytes = 12 * 1024;   // per stage; 8 warps x 2 stages = 192 KB per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Rows of list q in groups of G = min(32, kBulkWarpBytes / R); this warp takes groups dw, dw + n_dw, ...
__device__ __forceinline__ void bulk_rows(const GatherArgs& a, int q, int64_t cnt, int64_t dw, int64_t n_dw, int lane,
                                          char* stage0, uint64_t* bars, uint32_t* phase) {
  const int G = max(1, min(32, kBulkWarpBytes / a.R));
  const int64_t ngroups = (cnt + G - 1) / G;
  int64_t g = dw;
  if (g >= ngroups) return;
  auto issue = [&](int64_t grp, int st) {
    const int64_t j = grp * G + lane;
    const int n = (int)min((int64_t)G, cnt - grp * G);
    if (lane == 0) mbar_expect_tx(bars + st, (uint32_t)(n * a.R));
    __syncwarp();
    if (lane < n) {
      const uint64_t w = a.L.w[q][j];
      const char* base = q == kListLocal ? a.hbm : a.peers[(w >> 56) & 63];
      bulk_load(stage0 + (size_t)st * kBulkWarpBytes + lane * a.R, base + (int64_t)(w & ((1ull << 56) - 1)) * a.R,
                (uint32_t)a.R, bars + st);
    }
  };
  int st = 0;
  issue(g, 0);
  for (; g < ngroups; g += n_dw) {
    const int64_t nxt = g + n_dw;
    if (nxt < ngroups) {
      bulk_wait_read0();  // this lane's store from stage st^1 has finished reading it
      __syncwarp();
      issue(nxt, st ^ 1);
    }
    mbar_wait(bars + st, phase[st]);
    phase[st] ^= 1u;
    const int n = (int)min((int64_t)G, cnt - g * G);
    if (lane < n)
      bulk_store(a.out + a.L.i[q][g * G + lane] * (int64_t)a.R, stage0 + (size_t)st * kBulkWarpBytes + lane * a.R,
                 (uint32_t)a.R);
    bulk_commit();
    st ^= 1;
  }
}

// K4: warp-specialised gather.
//   kPartAll (one kernel, every tier): when the host list is non-empty one warp in 8 (two in staged
//     mode) serves host rows (zero-copy over PCIe, or the dynamic zero-copy / staged split) while the
//     others copy peer (NVLink) then local HBM rows.
//   kPartHbm: every warp copies peer then local rows (link mode, slot stream).
//   kPartHost: every warp serves host rows (link mode: the plan's link stream).
// Host rows are taken by ticket (UH rows per grab), not by a static split: CTAs that become resident
// late (SMs busy with other batches' sampling) then take less work instead of stretching the tail of
// the link transfer.
__device__ __forceinline__ uint32_t ld_acquire_sys_u32_(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int4 ld_volatile_v4_(const int4* p) {
  int4 r;
  asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
constexpr uint64_t kStageWatchdogNs = 30ull * 1000000000ull;

__device__ __forceinline__ int64_t warp_ticket(unsigned long long* ctr, int n, int lane) {
  unsigned long long t = 0;
  if (lane == 0) t = atomicAdd(ctr, (unsigned long long)n);
  return (int64_t)__shfl_sync(0xFFFFFFFFu, t, 0);
}

// Zero-copy host rows [0, n), UH rows per ticket.
template <int VPL, int UH>
__device__ __forceinline__ void host_rows(const GatherArgs& a, int64_t n, int lane, int nvec) {
  for (;;) {
    const int64_t j0 = warp_ticket(&a.ctl[kCtlHostTicket], UH, lane);
    if (j0 >= n) break;
    copy_rows<VPL, UH>(a, kListHost, j0, n, lane, nvec);
  }
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Staged mode: the GPU's host-row warps and the host stagers split the batch's host list [0, n_host)
// dynamically, in 64-row chunks.  The warps take chunks from the front (one device-side ticket, a
// posted write of the front hint, one relaxed system-scope read of the chunk's state word); the
// stagers claim chunks from the back (state = seq|CLAIMED), copy the rows into the contiguous pinned
// staging buffer and publish them (state = seq|DONE, release).  A published chunk is streamed from
// staging (one acquire orders the rows after the state word); a claimed one is waited for up to
// kStageStealNs and then copied zero-copy by the GPU itself; an unclaimed one is read zero-copy
// right away.  So the CPU's share is what it claims before the GPU's front arrives (capped by
// stage_frac), and a slow or descheduled stager costs at most the steal timeout.  A chunk both sides
// copy is copied twice (identical bytes; the staged copy is unused): no exclusivity is needed, only
// "every row by at least one side", and the GPU alone decides which rows it still has to copy.  The
// list the warps read is in device memory; the stagers read its pinned mirror.
// Reserved chunks (stage_reserve > 0): the last ceil(stage_reserve * n_chunks) chunks of the list are
// left to the stagers.  A warp reaching an unclaimed reserved chunk does not advance the front hint;
// it polls the chunk's state for up to kStageReserveNs (the stagers claim from the back, so they get
// there late in the batch) and only then takes the chunk itself (hint, zero-copy), so a stall of the
// host threads still costs a bounded wait, never a hang.
constexpr uint64_t kStageStealNs = 100000;
constexpr uint64_t kStageReserveNs = 200000;
template <int VPL, int UH>
__device__ __forceinline__ void host_rows_dyn(const GatherArgs& a, int64_t n_host, int lane, int nvec) {
  const uint32_t seq = (uint32_t)a.ctl[kCtlStageSeq];
  const unsigned long long claimed = ((unsigned long long)seq << 2) | kChunkClaimed;
  const unsigned long long done = ((unsigned long long)seq << 2) | kChunkDone;
  const int64_t n_chunks = (n_host + kStageChunk - 1) / kStageChunk;
  const int64_t n_res = min(min(n_chunks, a.stage_max_chunks), (int64_t)ceilf(a.stage_reserve * (float)n_chunks));
  const int64_t c_res = n_chunks - n_res;  // chunks [c_res, n_chunks) are reserved for the stagers
  for (;;) {
    const int64_t j0 = warp_ticket(&a.ctl[kCtlHostTicket], kStageChunk, lane);
    if (j0 >= n_host) break;
    const int64_t c = j0 / kStageChunk;
    const int64_t j1 = min(n_host, j0 + kStageChunk);
    unsigned long long st = 0;
    if (lane == 0) {
      st = ld_relaxed_sys_u64(&a.chunk[c]);
      if (c >= c_res && st != claimed && st != done) {  // reserved: give the stagers time to claim it
        const uint64_t t0 = globaltimer();
        unsigned backoff = 512;
        while (st != claimed && st != done && globaltimer() - t0 < kStageReserveNs) {
          __nanosleep(backoff);
          backoff = min(backoff * 2u, 8192u);
          st = ld_relaxed_sys_u64(&a.chunk[c]);
        }
      }
      if (st != claimed && st != done)  // this warp copies the chunk: stagers stop at the front
        st_relaxed_sys_u64(a.hint, ((unsigned long long)seq << 32) | (unsigned long long)c);
      if (st == claimed) {  // a stager is copying it: wait a bounded time, then take it back
        const uint64_t t0 = globaltimer();
        unsigned backoff = 256;
        while (st == claimed && globaltimer() - t0 < kStageStealNs) {
          __nanosleep(backoff);
          backoff = min(backoff * 2u, 4096u);
          st = ld_relaxed_sys_u64(&a.chunk[c]);
        }
      }
      if (st == done) (void)ld_acquire_sys_u64(&a.chunk[c]);  // orders the staged rows after the state word
    }
    st = __shfl_sync(0xFFFFFFFFu, st, 0);
    if (st != done) {  // not staged: read the chunk's rows zero-copy
      for (int64_t j = j0; j < j1; j += UH) copy_rows<VPL, UH>(a, kListHost, j, j1, lane, nvec);
      continue;
    }
    __syncwarp();
    // chunk c is staged at chunk position n_chunks - 1 - c of the staging buffer, rows contiguous
    const char* sbase = a.stage + (n_chunks - 1 - c) * kStageChunk * (int64_t)a.R;
    for (int64_t j = j0; j < j1; j += UH) {
      int4 r[UH][VPL];
#pragma unroll
      for (int u = 0; u < UH; u++)
        if (j + u < j1) {
#pragma unroll
          for (int k = 0; k < VPL; k++) {
            const int idx = lane + 32 * k;
            if (idx < nvec) r[u][k] = ld_volatile_v4_((const int4*)(sbase + (j + u - j0) * (int64_t)a.R) + idx);
          }
        }
#pragma unroll
      for (int u = 0; u < UH; u++)
        if (j + u < j1) {
          int4* dst = (int4*)(a.out + a.L.i[kListHost][j + u] * (int64_t)a.R);
#pragma unroll
          for (int k = 0; k < VPL; k++) {
            const int idx = lane + 32 * k;
            if (idx < nvec) dst[idx] = r[u][k];
          }
        }
    }
  }
}

// HOST = false: the instantiation for caches without a host tier (no host-row code, so the HBM copy
// loop alone sets the register budget).
struct GatherGroup {  // the batches of one launch (gridDim.y), as SampleGroup
  GatherArgs a[kMaxGroup];
};
// VU: 16-byte loads in flight per lane for HBM / peer rows.  The default 4 (80 registers) is slower
// than 8 (113 registers) for K4 alone but faster in the pipeline, where K4's register footprint decides
// how many of the other batches' sampler CTAs fit beside it; 2, 8 and 16
// (HELIOS_GATHER_VU) are the measured alternatives.
template <int VPL, int UH, bool BULK, bool HOST, int VU>
__global__ void __launch_bounds__(256, VU > 8 ? 1 : (VU == 4 ? 3 : (VU == 2 ? 4 : 2))) k_gather_lists(const __grid_constant__ GatherGroup P) {
  const GatherArgs& a = P.a[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(a.part == kPartHost ? nullptr : a.trace_params, a.trace_idx);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nvec = a.R >> 4;
  const int64_t n_local = (int64_t)a.ctl[kListLocal], n_peer = (int64_t)a.ctl[kListPeer],
                n_host = (int64_t)a.ctl[kListHost];
  if (HOST && a.part == kPartHost) {
    if (a.staged) host_rows_dyn<VPL, UH>(a, n_host, lane, nvec);
    else host_rows<VPL, UH>(a, n_host, lane, nvec);
    return;
  }
  if (a.stats && gw == 0 && lane == 0) {
    if (a.accumulate) {
      a.stats->rows_hbm_local += n_local;
      a.stats->rows_hbm_peer += n_peer;
      a.stats->rows_host += n_host;
    } else {
      a.stats->rows_hbm_local = n_local;
      a.stats->rows_hbm_peer = n_peer;
      a.stats->rows_host = n_host;
    }
    a.stats->rows_file = (int64_t)a.ctl[kListFile];  // the file list accumulates over passes
  }
  // kPartAll warp roles: r = gw % 8.  r < host_warps: host rows (zero-copy, or the dynamic
  // zero-copy / staged split); other warps: peer then local HBM rows.
  const int nspecial = (HOST && a.part == kPartAll && n_host > 0) ? a.host_warps : 0;
  const int r = (int)(gw & 7);
  if (HOST && r < nspecial) {
    if (a.staged) host_rows_dyn<VPL, UH>(a, n_host, lane, nvec);
    else host_rows<VPL, UH>(a, n_host, lane, nvec);
    return;
  }
  const int64_t dw = (gw >> 3) * (8 - nspecial) + (r - nspecial);  // index among data warps
  const int64_t n_dw = (nw >> 3) * (8 - nspecial);
  if constexpr (BULK) {
    extern __shared__ __align__(128) char bulk_smem[];
    __shared__ uint64_t bars[8][2];
    const int wi = threadIdx.x >> 5;
    uint32_t phase[2] = {0u, 0u};
    if (lane == 0) {
      mbar_init(&bars[wi][0], 1);
      mbar_init(&bars[wi][1], 1);
    }
    __syncwarp();
    char* stage0 = bulk_smem + (size_t)wi * 2 * kBulkWarpBytes;
    bulk_rows(a, kListPeer, n_peer, dw, n_dw, lane, stage0, bars[wi], phase);
    bulk_wait_read0();
    __syncwarp();
    bulk_rows(a, kListLocal, n_local, dw, n_dw, lane, stage0, bars[wi], phase);
    bulk_wait0();  // this lane's row stores are complete before the kernel ends
  } else {
    flat_rows<VU>(a, kListPeer, n_peer, dw, n_dw, lane, nvec);
    flat_rows<VU>(a, kListLocal, n_local, dw, n_dw, lane, nvec);
  }
}

// Split host part (the default; HELIOS_GATHER_SPLIT_HOST=0 = combined kernel): the host-tier rows of a batch in their
// own small kernel (64-thread CTAs, host-row code only) launched right behind the HBM part
// (k_gather_lists, kPartHbm) on the same stream.  A host-row warp spends most of its life waiting on
// PCIe reads and on the stagers; in the combined kernel it keeps a whole 256-thread CTA (and its
// registers) resident after the data warps are done, which takes SM slots from the other batches'
// sampling.  No griddepcontrol.wait: this grid is launched as the HBM part's programmatic dependent,
// whose CTAs trigger only after their own wait on the lookup / publish kernels has returned, so the
// lists, counts and mailbox it reads are complete.
template <int VPL, int UH>
__global__ void __launch_bounds__(64) k_gather_host(const __grid_constant__ GatherGroup P) {
  const GatherArgs& a = P.a[blockIdx.y];
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int nvec = a.R >> 4;
  const int64_t n_host = (int64_t)a.ctl[kListHost];
  if (a.staged) host_rows_dyn<VPL, UH>(a, n_host, lane, nvec);
  else host_rows<VPL, UH>(a, n_host, lane, nvec);
}

// Plain row copy by id (setup: HBM-tier fill from a mapped host table).
__global__ void k_rows_by_id(const char* __restrict__ src, int32_t R, const int32_t* __restrict__ ids, int64_t n,
                             char* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nvec = R >> 4;
  for (int64_t i = warp; i < n; i += nwarps) {
    const int4* s = (const int4*)(src + (int64_t)ids[i] * R);
    int4* d = (int4*)(dst + i * (int64_t)R);
    for (int k = lane; k < nvec; k += 32) d[k] = ld_stream(s + k);
  }
}

helios_status gather_rows_by_id(const char* src_dev, int32_t R, const int32_t* ids, int64_t n, char* dst, int sms,
                                cudaStream_t st) {
  if (n <= 0) return HELIOS_OK;
  k_rows_by_id<<<sms * 8, 256, 0, st>>>(src_dev, R, ids, n, dst);
  HCUDA(cudaGetLastError());
  return HELIOS_OK;
}

// ---- IO rings --------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int4 ld_volatile_v4(const int4* p) {
  int4 r;
  asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

constexpr uint64_t kWatchdogNs = 30ull * 1000000000ull;

struct IoArgs {
  const int64_t* miss_out;   // file list: output rows
  const uint64_t* miss_w;    // file list: directory words (slot bits = file row)
  unsigned long long* ctl;   // [kListFile] misses, [kCtlSubmit] / [kCtlComplete] tickets
  SqEntry* sq;               // device alias of pinned SQ
  CqEntry* cq;               // device alias of pinned CQ
  const char* staging;       // device alias of pinned staging
  uint32_t* free_seq;
  const uint32_t* base_seq;
  int rings, depth;
  int64_t slot_bytes, header, stride;
  int32_t len, R;
  char* out;
  int* err;
};

// K5 + K6 in ONE warp-specialised grid: in every CTA the first kIoSubmitWarps
// warps are submitters (thread-level submission, §3.1.1: each lane takes one request by ticket,
// waits for its ring slot to be free, writes the descriptor, publishes seq with st.release.sys) and
// the other warps are completers (asynchronous completion, §3.1.2: a warp takes one request by
// ticket, polls its CQ entry with ld.acquire.sys, moves the row staging -> out and frees the slot).
// Tickets are taken only by running warps, and every wait is on a strictly smaller ticket (a slot
// waits for request m - ring_size, a completion for its own submission), so the kernel makes progress
// with any number of its CTAs resident — also when it is serialised against every other kernel
// (ncu, CUDA_LAUNCH_BLOCKING, an SM-capped partition).  Watchdogs restart at every wait.
constexpr int kIoSubmitWarps = 2;

__device__ __forceinline__ void io_submit_warp(const IoArgs& a, int lane) {
  const unsigned long long M = a.ctl[kListFile];
  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(&a.ctl[kCtlSubmit], 32ull);
    tk = __shfl_sync(0xFFFFFFFFu, tk, 0);
    if (tk >= M) break;
    const unsigned long long m = tk + lane;
    if (m < M) {
      const int r = (int)(m % a.rings);
      const uint32_t p = (uint32_t)(m / a.rings);
      const uint32_t seq = a.base_seq[r] + p + 1u;
      const uint32_t slot = (seq - 1u) & (uint32_t)(a.depth - 1);
      const int64_t idx = (int64_t)r * a.depth + slot;
      bool ok = true;
      // slot reusable once its previous occupant (seq - depth) was consumed by a completer
      const uint64_t t0 = globaltimer();
      while ((int32_t)(seq - (uint32_t)a.depth - ld_acquire_gpu_u32(a.free_seq + idx)) > 0) {
        if (globaltimer() - t0 > kWatchdogNs) {
          latch(a.err, HELIOS_E_TIMEOUT);
          ok = false;
          break;
        }
        __nanosleep(256);
      }
      if (ok) {
        SqEntry* e = a.sq + idx;
        e->file_off = (uint64_t)(a.header + (int64_t)(a.miss_w[m] & ((1ull << 56) - 1)) * a.stride);
        e->len = (uint32_t)a.len;
        e->slot = (uint32_t)idx;
        e->out_row = (uint64_t)a.miss_out[m];
        __threadfence_system();
        st_release_sys_u32(&e->seq, seq);
      }
    }
  }
}

__device__ __forceinline__ void io_complete_warp(const IoArgs& a, int lane) {
  const unsigned long long M = a.ctl[kListFile];
  const int nvec = a.R >> 4;
  for (;;) {
    unsigned long long m = 0;
    if (lane == 0) m = atomicAdd(&a.ctl[kCtlComplete], 1ull);
    m = __shfl_sync(0xFFFFFFFFu, m, 0);
    if (m >= M) break;
    const int r = (int)(m % a.rings);
    const uint32_t p = (uint32_t)(m / a.rings);
    const uint32_t seq = a.base_seq[r] + p + 1u;
    const uint32_t slot = (seq - 1u) & (uint32_t)(a.depth - 1);
    const int64_t idx = (int64_t)r * a.depth + slot;
    bool ok = true;
    const uint64_t t0 = globaltimer();
    // every lane polls (one coalesced 32 B system-memory read per poll); the backoff grows to 8 us, far
    // below a storage read's latency, so polls do not eat PCIe read bandwidth (profiles/r02/ncu_io_summary.json)
    unsigned backoff = 256;
    while (ld_acquire_sys_u32(&a.cq[idx].seq) != seq) {
      if (globaltimer() - t0 > kWatchdogNs) {
        ok = false;
        break;
      }
      __nanosleep(backoff);
      backoff = min(backoff * 2u, 8192u);
    }
    ok = __all_sync(0xFFFFFFFFu, ok);
    if (!ok) {
      if (lane == 0) latch(a.err, HELIOS_E_TIMEOUT);
      break;
    }
    const int st = *(volatile const int32_t*)&a.cq[idx].status;
    if (st != 0) {
      if (lane == 0) latch(a.err, HELIOS_E_IO);
    } else {
      const int4* s = (const int4*)(a.staging + idx * a.slot_bytes);
      int4* d = (int4*)(a.out + a.miss_out[m] * (int64_t)a.R);
      for (int k = lane; k < nvec; k += 32) d[k] = ld_volatile_v4(s + k);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      st_release_gpu_u32(a.free_seq + idx, seq);
    }
  }
}

__global__ void __launch_bounds__(256) k_io(IoArgs a) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) < kIoSubmitWarps) io_submit_warp(a, lane);
  else io_complete_warp(a, lane);
}

// Ablation (HELIOS_CACHE_IO_SYNC): the synchronous IO stack the paper measures GIDS/BaM with
// (§2.2, Fig. iostack_bam): each warp owns one request end to end — its leader
// reserves a ring slot and submits, the warp then spins on the completion and finally copies the
// row — so a warp is tied up for the whole IO latency and at most one request per warp is in
// flight.  Same rings and host workers as the decoupled submit / complete roles of k_io.
__global__ void __launch_bounds__(256) k_io_sync(IoArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned long long M = a.ctl[kListFile];
  const int nvec = a.R >> 4;
  for (;;) {
    unsigned long long m = 0;
    if (lane == 0) m = atomicAdd(&a.ctl[kCtlSubmit], 1ull);
    m = __shfl_sync(0xFFFFFFFFu, m, 0);
    if (m >= M) break;
    const int r = (int)(m % a.rings);
    const uint32_t p = (uint32_t)(m / a.rings);
    const uint32_t seq = a.base_seq[r] + p + 1u;
    const uint32_t slot = (seq - 1u) & (uint32_t)(a.depth - 1);
    const int64_t idx = (int64_t)r * a.depth + slot;
    bool ok = true;
    uint64_t t0 = globaltimer();
    if (lane == 0) {
      while ((int32_t)(seq - (uint32_t)a.depth - ld_acquire_gpu_u32(a.free_seq + idx)) > 0) {
        if (globaltimer() - t0 > kWatchdogNs) {
          ok = false;
          break;
        }
        __nanosleep(256);
      }
      if (ok) {
        SqEntry* e = a.sq + idx;
        e->file_off = (uint64_t)(a.header + (int64_t)(a.miss_w[m] & ((1ull << 56) - 1)) * a.stride);
        e->len = (uint32_t)a.len;
        e->slot = (uint32_t)idx;
        e->out_row = (uint64_t)a.miss_out[m];
        __threadfence_system();
        st_release_sys_u32(&e->seq, seq);
      }
    }
    ok = __shfl_sync(0xFFFFFFFFu, ok, 0);
    t0 = globaltimer();
    while (ok && ld_acquire_sys_u32(&a.cq[idx].seq) != seq) {
      if (globaltimer() - t0 > kWatchdogNs) ok = false;
      else __nanosleep(128);
    }
    if (!__all_sync(0xFFFFFFFFu, ok)) {
      if (lane == 0) latch(a.err, HELIOS_E_TIMEOUT);
      break;
    }
    if (*(volatile const int32_t*)&a.cq[idx].status != 0) {
      if (lane == 0) latch(a.err, HELIOS_E_IO);
    } else {
      const int4* s = (const int4*)(a.staging + idx * a.slot_bytes);
      int4* d = (int4*)(a.out + a.miss_out[m] * (int64_t)a.R);
      for (int k = lane; k < nvec; k += 32) d[k] = ld_volatile_v4(s + k);
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      st_release_gpu_u32(a.free_seq + idx, seq);
    }
  }
}

__global__ void k_io_finish(unsigned long long* ctl, uint32_t* base_seq, int rings) {
  const unsigned long long M = ctl[kListFile];
  for (int r = threadIdx.x; r < rings; r += blockDim.x)
    base_seq[r] += (uint32_t)(M / rings + ((unsigned long long)r < M % rings ? 1 : 0));
}

// The IO kernels spin on host workers, so they are loaded up front rather than lazily (CUDA 12
// lazy loading of a kernel may wait for running work).
helios_status io_preload_kernels() {
  cudaFuncAttributes fa;
  HCUDA(cudaFuncGetAttributes(&fa, k_io));
  HCUDA(cudaFuncGetAttributes(&fa, k_io_finish));
  HCUDA(cudaFuncGetAttributes(&fa, k_io_sync));
  return HELIOS_OK;
}

// Persistent grid (8 warps per CTA; one in 8 serves host rows when the batch has any).  With a host
// tier: one CTA per SM — a gather waits on PCIe reads for most of its life, so a smaller resident
// footprint leaves SM slots to the other in-flight batches' sampling (measured against 4 CTAs per
// SM: C3 +6 %, C2 +6 %; 74-296 CTAs within noise on C3; 2 or 4 host warps per 8 are slower,
// DESIGN.md §11).  HBM-only caches use c->gather_ctas CTAs (K4 grid sweep).
// HELIOS_GATHER_BULK=1 (read at cache build; the bulk-copy ablation): one CTA per SM
// with 192 KB of dynamic shared memory.
constexpr int kBulkSmem = 8 * 2 * kBulkWarpBytes;

template <int VPL, int UH, bool HOST>
static void launch_gather(const GatherGroup& P, int n, int grid, bool bulk, cudaStream_t st) {
  if (bulk) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_gather_lists<VPL, UH, true, HOST, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kBulkSmem);
      attr = true;
    }
    launch_pdl_smem(k_gather_lists<VPL, UH, true, HOST, 8>, dim3(grid, n), dim3(256), kBulkSmem, st, P);
  } else if (P.a[0].vu16) {
    launch_pdl(k_gather_lists<VPL, UH, false, HOST, 16>, dim3(grid, n), dim3(256), st, P);
  } else if (P.a[0].vu4) {
    launch_pdl(k_gather_lists<VPL, UH, false, HOST, 4>, dim3(grid, n), dim3(256), st, P);
  } else if (P.a[0].vu2) {
    launch_pdl(k_gather_lists<VPL, UH, false, HOST, 2>, dim3(grid, n), dim3(256), st, P);
  } else {
    launch_pdl(k_gather_lists<VPL, UH, false, HOST, 8>, dim3(grid, n), dim3(256), st, P);
  }
}

template <bool HOST>
static void launch_gather_rows(const GatherGroup& P, int n, int grid, bool bulk, cudaStream_t st) {
  const int nvec = P.a[0].R / 16;
  if (nvec <= 32) launch_gather<1, 8, HOST>(P, n, grid, bulk, st);
  else if (nvec <= 64) launch_gather<2, 4, HOST>(P, n, grid, bulk, st);
  else if (nvec <= 128) launch_gather<4, 2, HOST>(P, n, grid, bulk, st);
  else launch_gather<8, 1, HOST>(P, n, grid, bulk, st);
}

// host: the cache has a host tier (else the lean HBM-only instantiation)
static void launch_gather_any(const GatherGroup& P, int n, int grid, bool bulk, bool host, cudaStream_t st) {
  if (host) launch_gather_rows<true>(P, n, grid, bulk, st);
  else launch_gather_rows<false>(P, n, grid, bulk, st);
}
static void launch_gather_host(const GatherGroup& P, int n, int grid, cudaStream_t st) {
  const int nvec = P.a[0].R / 16;
  if (nvec <= 32) launch_pdl(k_gather_host<1, 8>, dim3(grid, n), dim3(64), st, P);
  else if (nvec <= 64) launch_pdl(k_gather_host<2, 4>, dim3(grid, n), dim3(64), st, P);
  else if (nvec <= 128) launch_pdl(k_gather_host<4, 2>, dim3(grid, n), dim3(64), st, P);
  else launch_pdl(k_gather_host<8, 1>, dim3(grid, n), dim3(64), st, P);
}
static void launch_gather_any(const GatherArgs& a, int grid, bool bulk, bool host, cudaStream_t st) {
  GatherGroup P{};
  P.a[0] = a;
  launch_gather_any(P, 1, grid, bulk, host, st);
}

void gws_free(GatherWS& w) {
  stager_unregister(w.owner, w);
  if (w.d_list_i) cudaFree(w.d_list_i);
  if (w.d_list_w) cudaFree(w.d_list_w);
  if (w.d_ctl) cudaFree(w.d_ctl);
  if (w.h_host_w) cudaFreeHost(w.h_host_w);
  if (w.h_stage) cudaFreeHost(w.h_stage);
  if (w.h_chunk) cudaFreeHost(w.h_chunk);
  if (w.h_hint) cudaFreeHost(w.h_hint);
  if (w.h_mail) cudaFreeHost(w.h_mail);
  if (w.d_seq) cudaFree(w.d_seq);
  w = GatherWS{};
}

helios_status gws_ensure(helios_cache* c, GatherWS& w, int64_t max_nodes) {
  if (w.d_ctl && max_nodes <= w.cap) return HELIOS_OK;
  HCUDA(cudaDeviceSynchronize());
  gws_free(w);
  const int64_t cap = std::max<int64_t>(max_nodes, 1);
  HCUDA(cudaMalloc(&w.d_list_i, kLists * cap * 8));
  HCUDA(cudaMalloc(&w.d_list_w, kLists * cap * 8));
  HCUDA(cudaMalloc(&w.d_ctl, kCtlWords * sizeof(unsigned long long)));
  HCUDA(cudaMemset(w.d_ctl, 0, kCtlWords * sizeof(unsigned long long)));
  w.cap = cap;
  w.owner = c;
  if (c->staged) {
    const int64_t chunks = (cap + kStageChunk - 1) / kStageChunk;  // state words per list chunk
    HCHECK(chunks < 65536, HELIOS_E_CAPACITY, "staged host tier: %lld rows per batch exceed 2^22", (long long)cap);
    w.stage_rows = std::min<int64_t>(kStageCapRows, chunks * kStageChunk);
    HCUDA(cudaHostAlloc(&w.h_host_w, cap * 8, cudaHostAllocMapped));
    HCUDA(cudaHostAlloc(&w.h_stage, w.stage_rows * (int64_t)c->R, cudaHostAllocMapped));
    HCUDA(cudaHostAlloc(&w.h_chunk, chunks * 8, cudaHostAllocMapped));
    HCUDA(cudaHostAlloc(&w.h_mail, 16, cudaHostAllocMapped));
    HCUDA(cudaHostAlloc(&w.h_hint, 8, cudaHostAllocMapped));
    memset(w.h_chunk, 0, chunks * 8);
    memset(w.h_mail, 0, 16);
    memset(w.h_hint, 0, 8);
    HCUDA(cudaHostGetDevicePointer((void**)&w.d_host_w, w.h_host_w, 0));
    HCUDA(cudaHostGetDevicePointer((void**)&w.d_stage, w.h_stage, 0));
    HCUDA(cudaHostGetDevicePointer((void**)&w.d_chunk, w.h_chunk, 0));
    HCUDA(cudaHostGetDevicePointer((void**)&w.d_mail, w.h_mail, 0));
    HCUDA(cudaHostGetDevicePointer((void**)&w.d_hint, w.h_hint, 0));
    HCUDA(cudaMalloc(&w.d_seq, 4));
    HCUDA(cudaMemset(w.d_seq, 0, 4));
    helios_status st = stager_register(c, w);
    if (st != HELIOS_OK) return st;
  }
  return HELIOS_OK;
}

static GatherArgs make_args(helios_cache* c, GatherWS& w, void* out, helios_gather_stats* stats, bool accumulate,
                            int part) {
  GatherArgs a;
  for (int q = 0; q < kLists; q++) {
    a.L.i[q] = w.d_list_i + q * w.cap;
    a.L.w[q] = w.d_list_w + q * w.cap;
  }
  const bool staged = c->staged && w.d_host_w;
  a.L.host_w_mirror = staged ? w.d_host_w : nullptr;
  a.out = (char*)out;
  a.R = c->R;
  a.ctl = w.d_ctl;
  a.part = part;
  a.host_warps = staged ? 2 : 1;
  a.staged = staged;
  a.accumulate = accumulate;
  a.stage = w.d_stage;
  a.chunk = w.d_chunk;
  a.hint = w.d_hint;
  a.stage_reserve = c->stage_reserve;
  a.stage_max_chunks = w.stage_rows / kStageChunk;
  a.vu16 = c->gather_vu == 16;
  a.vu4 = c->gather_vu == 4;
  a.vu2 = c->gather_vu == 2;
  a.evict = c->gather_evict_lists;
  a.err = c->d_err;
  a.hbm = c->hbm;
  a.peers = c->d_peers;
  a.host_dev = c->d_host_tier;
  a.stats = stats;
  a.trace_params = w.trace_params;
  a.trace_idx = w.trace_idx + 1;
  return a;
}

template <int VU, int D>
static cudaError_t launch_direct_async(const DirectGroup& DP, int n, int ctas, cudaStream_t st) {
  constexpr size_t smem = (size_t)8 * D * 32 * (VU * sizeof(int4) + sizeof(char*));  // 8 warps x D stages
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_gather_direct_async<VU, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (attr != cudaSuccess) return attr;
  launch_pdl_smem(k_gather_direct_async<VU, D>, dim3(ctas, n), dim3(256), smem, st, DP);
  return cudaGetLastError();
}

// One lookup + gather pass over rows [*lo, *n_nodes) (lo = NULL: all) of each of the n batches of a
// group (one launch of each kernel, gridDim.y = n).  first: reset every count; otherwise (later
// intra-batch passes, n = 1) only the per-pass tier counts and row tickets are reset, so the file
// list and the stats accumulate over the passes of a batch.
static helios_status gather_pass_group(helios_cache* c, GatherWS* const* ws, const int64_t* const* nodes,
                                       const int64_t* lo, const int64_t* const* n_nodes, int n, int64_t max_rows,
                                       void* const* out, helios_gather_stats* const* stats, bool first, bool accumulate,
                                       int part, cudaStream_t st) {
  HCHECK(!c->broken, HELIOS_E_STATE, "cache unusable after an IO / staging watchdog timeout");
  HCHECK(n >= 1 && n <= kMaxGroup, HELIOS_E_INVALID, "group of %d batches (1..%d)", n, kMaxGroup);
  LookupGroup LP{};
  GatherGroup GP{};
  PublishGroup PP{};
  bool staged = false;
  for (int b = 0; b < n; b++) {
    GatherWS& w = *ws[b];
    if (first) {
      if (!w.ctl_preset) HCUDA(cudaMemsetAsync(w.d_ctl, 0, kCtlWords * sizeof(unsigned long long), st));
    } else {
      HCUDA(cudaMemsetAsync(w.d_ctl, 0, kListFile * sizeof(unsigned long long), st));
      HCUDA(cudaMemsetAsync(w.d_ctl + kCtlHostTicket, 0, sizeof(unsigned long long), st));
    }
    GP.a[b] = make_args(c, w, out[b], stats[b], accumulate, part);
    LP.a[b] = LookupArgs{nodes[b], lo, n_nodes[b], (const int64_t*)c->dir, c->V, c->rank, GP.a[b].L, w.d_ctl,
                         c->d_err, w.trace_params, w.trace_idx};
    PP.ctl[b] = w.d_ctl;
    PP.seq[b] = w.d_seq;
    PP.mail[b] = w.d_mail;
    staged = GP.a[b].staged;
  }
  if (c->direct && c->S == 0 && !c->has_file && part == kPartAll && !c->gather_bulk) {  // every row in HBM
    DirectGroup DP{};
    for (int b = 0; b < n; b++) {
      DP.a[b] = GP.a[b];
      DP.d[b] = DirectArgs{nodes[b], lo, n_nodes[b], (const int64_t*)c->dir, c->V, c->rank};
      if (!first) HCUDA(cudaMemsetAsync(ws[b]->d_ctl + kCtlDone, 0, sizeof(unsigned long long), st));
    }
    if (c->gather_async && c->R / 16 <= 32 * 4) {  // loads staged through shared memory (cp.async)
      const cudaError_t e = c->gather_async >= 8 ? launch_direct_async<4, 8>(DP, n, c->gather_ctas, st)
                                                 : launch_direct_async<4, 4>(DP, n, c->gather_ctas, st);
      HCUDA(e);
    } else if (c->gather_vu == 8) {
      if (c->gather_evict) launch_pdl(k_gather_direct<8, true>, dim3(c->gather_ctas, n), dim3(256), st, DP);
      else launch_pdl(k_gather_direct<8, false>, dim3(c->gather_ctas, n), dim3(256), st, DP);
    } else {
      if (c->gather_evict) launch_pdl(k_gather_direct<4, true>, dim3(c->gather_ctas, n), dim3(256), st, DP);
      else launch_pdl(k_gather_direct<4, false>, dim3(c->gather_ctas, n), dim3(256), st, DP);
    }
    HCUDA(cudaGetLastError());
    return HELIOS_OK;
  }
  const int lg = (int)std::min<int64_t>(std::max<int64_t>(1, (max_rows + 255) / 256), (int64_t)c->sms * 2);
  launch_pdl(k_lookup, dim3(lg, n), dim3(256), st, LP);
  if (staged) launch_pdl(k_stage_publish, dim3(1, n), dim3(1), st, PP);
  if (c->split_host && c->S > 0 && part == kPartAll) {  // HBM part, then the host part in its own small kernel
    for (int b = 0; b < n; b++) GP.a[b].part = kPartHbm;
    launch_gather_any(GP, n, c->gather_ctas, c->gather_bulk, false, st);
    for (int b = 0; b < n; b++) GP.a[b].part = kPartHost;
    launch_gather_host(GP, n, c->sms, st);
  } else {
    launch_gather_any(GP, n, c->gather_ctas, c->gather_bulk, c->S > 0, st);
  }
  HCUDA(cudaGetLastError());
  return HELIOS_OK;
}

static helios_status gather_pass(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* lo,
                                 const int64_t* n_nodes, int64_t max_rows, void* out, helios_gather_stats* stats,
                                 bool first, bool accumulate, int part, cudaStream_t st) {
  GatherWS* ws[1] = {&w};
  const int64_t* nd[1] = {nodes};
  const int64_t* nn[1] = {n_nodes};
  void* o[1] = {out};
  helios_gather_stats* sts[1] = {stats};
  return gather_pass_group(c, ws, nd, lo, nn, 1, max_rows, o, sts, first, accumulate, part, st);
}

helios_status gather_launch_group(helios_cache* c, GatherWS* const* ws, const int64_t* const* nodes,
                                  const int64_t* const* n_nodes, int n, int64_t max_nodes, void* const* out,
                                  helios_gather_stats* const* stats, cudaStream_t st) {
  HCHECK(c->G == 1 || c->peers_attached, HELIOS_E_STATE, "world_size %d but peers not attached", c->G);
  for (int b = 0; b < n; b++) {
    HCHECK(nodes[b] && n_nodes[b] && (out[b] || max_nodes == 0), HELIOS_E_INVALID, "null gather argument");
    HCHECK(ws[b]->d_ctl && max_nodes <= ws[b]->cap, HELIOS_E_CAPACITY, "max_nodes %lld > gather list cap %lld",
           (long long)max_nodes, (long long)ws[b]->cap);
  }
  return gather_pass_group(c, ws, nodes, nullptr, n_nodes, n, max_nodes, out, stats, true, false, kPartAll, st);
}

helios_status gather_launch(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* n_nodes, int64_t max_nodes,
                            void* out, helios_gather_stats* stats, cudaStream_t st) {
  HCHECK(nodes && n_nodes && (out || max_nodes == 0), HELIOS_E_INVALID, "null gather argument");
  HCHECK(c->G == 1 || c->peers_attached, HELIOS_E_STATE, "world_size %d but peers not attached", c->G);
  HCHECK(w.d_ctl && max_nodes <= w.cap, HELIOS_E_CAPACITY, "max_nodes %lld > gather list cap %lld",
         (long long)max_nodes, (long long)w.cap);
  return gather_pass(c, w, nodes, nullptr, n_nodes, max_nodes, out, stats, true, false, kPartAll, st);
}

helios_status gather_hbm_launch(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* n_nodes,
                                int64_t max_nodes, void* out, helios_gather_stats* stats, cudaStream_t st) {
  HCHECK(nodes && n_nodes && (out || max_nodes == 0), HELIOS_E_INVALID, "null gather argument");
  HCHECK(c->G == 1 || c->peers_attached, HELIOS_E_STATE, "world_size %d but peers not attached", c->G);
  HCHECK(w.d_ctl && max_nodes <= w.cap, HELIOS_E_CAPACITY, "max_nodes %lld > gather list cap %lld",
         (long long)max_nodes, (long long)w.cap);
  return gather_pass(c, w, nodes, nullptr, n_nodes, max_nodes, out, stats, true, false, kPartHbm, st);
}

helios_status gather_host_launch(helios_cache* c, GatherWS& w, void* out, cudaStream_t st) {
  HCHECK(!c->broken, HELIOS_E_STATE, "cache unusable after an IO / staging watchdog timeout");
  const GatherArgs a = make_args(c, w, out, nullptr, false, kPartHost);
  launch_gather_any(a, c->gather_ctas, false, true, st);
  HCUDA(cudaGetLastError());
  return HELIOS_OK;
}

helios_status gather_range_launch(helios_cache* c, GatherWS& w, const int64_t* nodes, const int64_t* lo,
                                  const int64_t* hi, int64_t max_rows, void* out, helios_gather_stats* stats, bool first,
                                  cudaStream_t st) {
  HCHECK(c->G == 1 || c->peers_attached, HELIOS_E_STATE, "world_size %d but peers not attached", c->G);
  return gather_pass(c, w, nodes, lo, hi, max_rows, out, stats, first, true, kPartAll, st);
}

// ---- host-link probe (measurement) --------------------------------------------------------------
// Fills a host list with n uniformly random rows of the host tier's address range (fresh per rep,
// SplitMix64 of (seed, rep, i)) and the ctl words the host part of K4 reads.
__global__ void k_probe_list(int64_t* li, uint64_t* lw, unsigned long long* ctl, int64_t n, int64_t range, uint64_t seed) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = t; i < n; i += nt) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    li[i] = i;
    lw[i] = (1ull << 62) | (uint64_t)__umul64hi(z, (uint64_t)range);
  }
  if (t == 0) {
    for (int q = 0; q < kCtlWords; q++) ctl[q] = 0;
    ctl[kListHost] = (unsigned long long)n;
  }
}

helios_status probe_host_impl(helios_cache* c, int64_t n, uint64_t seed, int32_t reps, float* ms) {
  HCHECK(n > 0 && reps > 0 && ms, HELIOS_E_INVALID, "probe: n_rows %lld, reps %d", (long long)n, reps);
  HCHECK(c->S > 0 && c->d_host_tier, HELIOS_E_STATE, "probe: the cache has no host tier");
  const int64_t range = (c->flags & HELIOS_CACHE_HOST_ALIAS) ? c->V : c->S;
  GatherWS w;
  HCUDA(cudaMalloc(&w.d_list_i, kLists * n * 8));
  HCUDA(cudaMalloc(&w.d_list_w, kLists * n * 8));
  HCUDA(cudaMalloc(&w.d_ctl, kCtlWords * sizeof(unsigned long long)));
  w.cap = n;
  char* out = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaStream_t st = nullptr;
  helios_status s = HELIOS_OK;
  float tot = 0;
  auto run = [&]() -> helios_status {
    HCUDA(cudaMalloc(&out, n * (int64_t)c->R));
    HCUDA(cudaEventCreate(&e0));
    HCUDA(cudaEventCreate(&e1));
    HCUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    GatherArgs a = make_args(c, w, out, nullptr, false, kPartHost);
    a.staged = false;
    a.L.i[kListHost] = w.d_list_i + kListHost * n;
    a.L.w[kListHost] = w.d_list_w + kListHost * n;
    for (int r = 0; r < reps; r++) {
      k_probe_list<<<c->sms * 4, 256, 0, st>>>(a.L.i[kListHost], a.L.w[kListHost], w.d_ctl, n, range,
                                                seed ^ (0x5851F42D4C957F2Dull * (uint64_t)(r + 1)));
      HCUDA(cudaEventRecord(e0, st));
      launch_gather_any(a, c->sms, false, true, st);  // the host part: one CTA per SM as in the pipeline
      HCUDA(cudaEventRecord(e1, st));
      HCUDA(cudaEventSynchronize(e1));
      float t = 0;
      HCUDA(cudaEventElapsedTime(&t, e0, e1));
      tot += t;
    }
    return HELIOS_OK;
  };
  s = run();
  if (st) cudaStreamSynchronize(st);
  if (out) cudaFree(out);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  cudaFree(w.d_list_i);
  cudaFree(w.d_list_w);
  cudaFree(w.d_ctl);
  w = GatherWS{};
  if (s == HELIOS_OK) *ms = tot / reps;
  return s;
}

// ---- independent host-link probe (measurement; not K4) --------------------------------------------
// Loads only: warp w of the grid reads D x 32 consecutive 16-byte vectors of the flattened sequence
// of random rows (load k of lane l: vector f = (w*D + k)*32 + l, i.e. vector f mod nvec of random row
// f / nvec), so every load instruction covers 512 contiguous bytes of rows, as a coalesced gather
// would; rows are drawn uniformly (SplitMix64 of (seed, row)) over the host tier; no stores, no
// lists, no warp roles.  D (loads in flight per lane) is swept by the host together with the grid
// size (rows in flight) and the best rate kept, so this is the ceiling of random R-byte zero-copy
// reads on this platform, independent of K4's code.
template <int D>
__global__ void k_probe_link(const char* __restrict__ host, int64_t range, int32_t R, int64_t n_rows, uint64_t seed,
                             int* sink) {
  const int nvec = R >> 4;
  const int64_t total = n_rows * nvec;
  int acc = 0;
  const int lane = threadIdx.x & 31;
  for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32 * D; base < total;
       base += (int64_t)gridDim.x * blockDim.x * D) {
    int4 r[D];
#pragma unroll
    for (int k = 0; k < D; k++) {
      const int64_t f = base + 32 * k + lane;
      r[k] = make_int4(0, 0, 0, 0);
      if (f < total) {
        const int64_t row = f / nvec;
        uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(row + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const int64_t slot = (int64_t)__umul64hi(z, (uint64_t)range);
        r[k] = ld_stream((const int4*)(host + slot * R) + (f - row * nvec));
      }
    }
#pragma unroll
    for (int k = 0; k < D; k++) acc ^= r[k].x ^ r[k].w;
  }
  if (acc == 0x7FFFFFFF) *sink = acc;
}

helios_status probe_link_impl(helios_cache* c, int64_t n, uint64_t seed, int32_t reps, float* ms, int32_t* best_depth) {
  HCHECK(n > 0 && reps > 0 && ms, HELIOS_E_INVALID, "probe: n_rows %lld, reps %d", (long long)n, reps);
  HCHECK(c->S > 0 && c->d_host_tier, HELIOS_E_STATE, "probe: the cache has no host tier");
  const int64_t range = (c->flags & HELIOS_CACHE_HOST_ALIAS) ? c->V : c->S;
  int* sink = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  HCUDA(cudaMalloc(&sink, sizeof(int)));
  HCUDA(cudaEventCreate(&e0));
  HCUDA(cudaEventCreate(&e1));
  float best = 1e30f;
  int bd = 0;
  uint64_t salt = seed;
  cudaError_t err = cudaSuccess;
  // rows in flight = threads * d / nvec: swept from ~300 to ~19 k rows at R = 512 (random zero-copy
  // rows slow down when far too many are outstanding, so the sweep covers both sides of the optimum)
  const int nvec = c->R / 16;
  for (int cfg = 0; cfg < 16; cfg++) {
    const int d = 1 << (cfg & 3);                                // 1, 2, 4, 8 loads in flight per lane
    const int grid_c = std::max(1, (c->sms / 4) << (cfg >> 2));  // 37, 74, 148, 296 CTAs (B200)
    float tot = 0;
    for (int r = 0; r < reps && err == cudaSuccess; r++) {
      salt = salt * 0x5851F42D4C957F2Dull + 0x14057B7EF767814Full;  // fresh rows every launch (no L2 reuse)
      cudaEventRecord(e0, 0);
      if (d == 1) k_probe_link<1><<<grid_c, 256>>>(c->d_host_tier, range, c->R, n, salt, sink);
      else if (d == 2) k_probe_link<2><<<grid_c, 256>>>(c->d_host_tier, range, c->R, n, salt, sink);
      else if (d == 4) k_probe_link<4><<<grid_c, 256>>>(c->d_host_tier, range, c->R, n, salt, sink);
      else k_probe_link<8><<<grid_c, 256>>>(c->d_host_tier, range, c->R, n, salt, sink);
      cudaEventRecord(e1, 0);
      err = cudaEventSynchronize(e1);
      float t = 0;
      if (err == cudaSuccess) err = cudaEventElapsedTime(&t, e0, e1);
      tot += t;
    }
    if (err == cudaSuccess && tot / reps < best) {
      best = tot / reps;
      bd = (int)((int64_t)grid_c * 256 * d / std::max(1, nvec));  // rows in flight of the best setting
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return fail(HELIOS_E_CUDA, "probe_link: %s", cudaGetErrorString(err));
  *ms = best;
  if (best_depth) *best_depth = bd;
  return HELIOS_OK;
}

// K5 / K6 on the cache's IO streams for the misses recorded in w by the preceding gather_launch on
// `st`.  IO batches are serialised across gather contexts through ev_io_done (ring sequence
// numbers advance per batch in k_io_finish).
helios_status io_launch(helios_cache* c, GatherWS& w, void* out, cudaStream_t st) {
  if (!c->has_file) return HELIOS_OK;
  IoArgs io;
  io.miss_out = w.d_list_i + kListFile * w.cap;
  io.miss_w = w.d_list_w + kListFile * w.cap;
  io.ctl = w.d_ctl;
  io.sq = c->io.d_sq;
  io.cq = c->io.d_cq;
  io.staging = c->io.d_staging;
  io.free_seq = c->io.d_free_seq;
  io.base_seq = c->io.d_base_seq;
  io.rings = c->io.rings;
  io.depth = c->io.depth;
  io.slot_bytes = c->io.slot_bytes;
  io.header = c->header;
  io.stride = c->stride;
  io.len = (int32_t)c->stride;
  io.R = c->R;
  io.out = (char*)out;
  io.err = c->d_err;
  HCHECK(!c->broken, HELIOS_E_STATE, "cache unusable after an IO / staging watchdog timeout");
  HCUDA(cudaEventRecord(c->ev_lookup, st));
  HCUDA(cudaStreamWaitEvent(c->s_submit, c->ev_lookup, 0));
  if (c->io_pending) HCUDA(cudaStreamWaitEvent(c->s_submit, c->ev_io_done, 0));
  if (c->io_sync) k_io_sync<<<c->io_ctas, 256, 0, c->s_submit>>>(io);
  else k_io<<<c->io_ctas, 256, 0, c->s_submit>>>(io);
  HCUDA(cudaGetLastError());
  HCUDA(cudaEventRecord(c->ev_submit, c->s_submit));
  HCUDA(cudaStreamWaitEvent(st, c->ev_submit, 0));
  k_io_finish<<<1, 64, 0, st>>>(w.d_ctl, c->io.d_base_seq, c->io.rings);
  HCUDA(cudaGetLastError());
  HCUDA(cudaEventRecord(c->ev_io_done, st));
  c->io_pending = true;
  return HELIOS_OK;
}

}  // namespace helios
