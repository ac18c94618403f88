// device.cuh — device-side primitives: Philox4x32-10, hash probing, decoupled look-back tile scan.
#pragma once

#include <cub/block/block_scan.cuh>

#include "internal.cuh"

namespace helios {

// Philox4x32-10 (Salmon et al., SC'11), reading 2: counter {j>>2, h, lo32 v, hi32 v}, key = batch key.
__device__ __forceinline__ uint32_t philox_word(uint64_t key, uint32_t h, uint64_t v, uint32_t j) {
  uint32_t c0 = j >> 2, c1 = h, c2 = (uint32_t)v, c3 = (uint32_t)(v >> 32);
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  uint32_t w = j & 3;
  return w == 0 ? c0 : (w == 1 ? c1 : (w == 2 ? c2 : c3));
}

// PDL: wait for the predecessor grid's completion + memory flush / let dependents start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Pipeline trace (HELIOS_PLAN_TRACE): params[3] of a batch points at its row of TraceRec, one per
// kernel position (3h + {0,1,2} = count scan / fill / assign of hop h, 3L relabel, 3L+1 table clear,
// 3L+2 lookup, 3L+3 gather).  The row is preset to all-ones; every warp records, after its PDL wait,
// the earliest start (atomicMin) and, when it leaves the kernel, the latest end (atomicMin of ~t).
struct TraceRec {
  unsigned long long start, end_inv;
};
#ifdef HELIOS_TRACE
struct TraceScope {
  TraceRec* r = nullptr;
  __device__ __forceinline__ TraceScope(const int64_t* params, int idx) {
    TraceRec* row = params ? reinterpret_cast<TraceRec*>(params[3]) : nullptr;
    if (row) {
      r = row + idx;
      if ((threadIdx.x & 31) == 0) atomicMin(&r->start, (unsigned long long)globaltimer());
    }
  }
  __device__ __forceinline__ ~TraceScope() {
    if (r && (threadIdx.x & 31) == 0) atomicMin(&r->end_inv, ~(unsigned long long)globaltimer());
  }
};
#else
// Default build: no tracing code in the kernels (even a disabled scope cost C2 13 %); the traced
// build is libhelios_trace.so (-DHELIOS_TRACE), loaded with HELIOS_LIB=trace.
struct TraceScope {
  __device__ __forceinline__ TraceScope(const int64_t*, int) {}
};
#endif

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_volatile_v4u32(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Open-addressing (linear probing) insert-or-find of key u at edge position e: returns the slot,
// *fresh = created here (with minpos = e); an existing slot's minpos is lowered to e if larger.
// Keys are homed in the table's first hmask+1 slots (hmask <= mask, both 2^k - 1) and probe on through
// the whole table (wrapping at mask), so any home region is correct at any load (the table is sized
// for the worst case); a home region sized to the batch keeps its slots dense in L2 lines.
__device__ __forceinline__ uint32_t table_insert(TableSlot* tab, uint32_t mask, uint32_t hmask, uint32_t u, uint32_t e,
                                                 bool* fresh) {
  const unsigned long long want = ((unsigned long long)u << 32) | e;
  uint32_t s = hash32(u) & hmask;
  for (;;) {
    unsigned long long w = ld_volatile_u64(&tab[s].km);
    if ((uint32_t)(w >> 32) == kEmpty) {
      w = atomicCAS(&tab[s].km, kEmptyKM, want);
      if (w == kEmptyKM) {
        *fresh = true;
        return s;
      }
    }
    if ((uint32_t)(w >> 32) == u) {
      if ((uint32_t)w > e) atomicMin(&tab[s].km, want);
      *fresh = false;
      return s;
    }
    s = (s + 1) & mask;
  }
}

// CSR index read with an evict-first L2 policy (sampled adjacency positions are rarely re-read within
// a batch; the default keeps them from displacing the batch tables in L2, HELIOS_SAMPLE_IDX_EVICT=0: off).
__device__ __forceinline__ int32_t ld_index_ef(const int32_t* p) {
  uint64_t pol;
  int32_t v;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void latch(int* err, int code) {
  if (code) atomicCAS(err, 0, code);
}

constexpr unsigned long long kStatusInvalid = ~0ull;
constexpr unsigned long long kStatusIncl = 1ull << 62;

// Tile ticket: counter starts at all-ones, so the first ticket is 0.  Call from every thread.
__device__ __forceinline__ unsigned tile_ticket(const ScanState& s, unsigned* sm) {
  if (threadIdx.x == 0) *sm = atomicAdd(s.counter, 1u) + 1u;
  __syncthreads();
  return *sm;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Decoupled look-back (Merrill & Garland 2016): publish this tile's aggregate, then warp 0 inspects
// 32 predecessors per step (closest first) until one carries an inclusive prefix, and publishes
// this tile's inclusive prefix.  Returns the exclusive prefix of the tile to every thread.
__device__ __forceinline__ long long tile_lookback(const ScanState& s, unsigned tile, long long agg, long long* sm) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(&s.status[0], kStatusIncl | (unsigned long long)agg);
    } else {
      if (lane == 0) atomicExch(&s.status[tile], (unsigned long long)agg);
      long long acc = 0;
      for (long long base = (long long)tile - 1;; base -= 32) {
        const long long j = base - lane;
        unsigned long long w = (j >= 0) ? ld_volatile_u64(&s.status[j]) : kStatusIncl;  // before tile 0: 0
        while (__any_sync(0xFFFFFFFFu, w == kStatusInvalid))
          if (w == kStatusInvalid) w = ld_volatile_u64(&s.status[j]);
        const unsigned incl = __ballot_sync(0xFFFFFFFFu, (w & kStatusIncl) != 0);
        long long v = (long long)(w & ~kStatusIncl);
        if (incl) {
          const int stop = __ffs(incl) - 1;  // closest predecessor with an inclusive prefix
          acc += warp_sum_ll(lane <= stop ? v : 0);
          break;
        }
        acc += warp_sum_ll(v);
      }
      prefix = acc;
      if (lane == 0) atomicExch(&s.status[tile], kStatusIncl | (unsigned long long)(acc + agg));
    }
    if (lane == 0) *sm = prefix;
  }
  __syncthreads();
  return *sm;
}

}  // namespace helios
