// sample.cu — K1 sample_hop and K2 dedup_relabel, the neighbour-sampling
// operator of PAPER.md:215 (§3.2.2) / :239 (§3.3), "2-hop random neighbor sampling" PAPER.md:292.
//
// A batch is 2 + 3L kernels (all enqueue-only; grids sized from host bounds, actual counts read
// from device memory, so the whole sequence is captured once into a CUDA graph and replayed):
//   per hop h:
//   k_row_count_scan   k_i = min(deg(N_h[i]), f_h); block_indptr[h] = exclusive scan (single-pass
//                      decoupled look-back), e_h = total.  Side job: relabel hop h-1's edges (h > 0)
//                      or insert N_0 = seeds into the batch hash table (h = 0: k_seed_count_scan).
//   k_fill_insert<G>   one G-lane group per row: copy the whole adjacency when k == d, else Floyd's
//                      k-subset with Philox draws resolved by group ballots; every sampled id is
//                      inserted into the open-addressing table right away (slot kept per edge) and
//                      atomicMin records the first edge position of ids new at this hop.
//   k_dedup_assign     flag = "this edge is the first occurrence of a new id"; a single-pass scan of
//                      the flags numbers the new ids n_h, n_h+1, ... in first-occurrence order and
//                      appends them to N_{h+1}.
//   k_relabel          (last hop only) block_indices[L-1][e] = local id of the edge's slot.
//   k_table_clear      resets the slots of N_L so the table is all-EMPTY for the next batch.
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <cstring>

#include "device.cuh"

namespace helios {

__global__ void k_validate_csr(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t V,
                               int64_t E, int* flag) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = tid; v < V; v += nt)
    if (indptr[v + 1] < indptr[v]) atomicCAS(flag, 0, HELIOS_E_INVALID);
  for (int64_t e = tid; e < E; e += nt) {
    int32_t u = indices[e];
    if (u < 0 || (int64_t)u >= V) atomicCAS(flag, 0, HELIOS_E_RANGE);
  }
  if (tid == 0 && (indptr[0] != 0 || indptr[V] != E)) atomicCAS(flag, 0, HELIOS_E_INVALID);
}

helios_status validate_csr_device(const int64_t* indptr, const int32_t* indices, int64_t V, int64_t E, int* d_flag,
                                  cudaStream_t st) {
  int dev, sms;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_validate_csr<<<sms * 8, 256, 0, st>>>(indptr, indices, V, E, d_flag);
  HCUDA(cudaGetLastError());
  return HELIOS_OK;
}

// Everything a batch's sampling kernels need, passed by value (one struct for every kernel).
struct SampleCtx {
  const int64_t* indptr;
  const int32_t* indices;
  int64_t V;
  const int64_t* params;  // [0] key, [1] n_seeds, [2] seeds pointer (device)
  int* err;
  TableSlot* tab;
  uint32_t mask;
  uint32_t* slot_of;
  uint32_t* node_slot;
  int64_t* nodes;
  int64_t* level_counts;
  int64_t* edge_counts;
  int32_t* bp[HELIOS_MAX_HOPS];
  int32_t* bi[HELIOS_MAX_HOPS];
  ScanState row_scan[HELIOS_MAX_HOPS];
  ScanState edge_scan[HELIOS_MAX_HOPS];
  int32_t fan[HELIOS_MAX_HOPS];
  int32_t L;
  unsigned* bar;  // grid barrier {arrivals, generation} (reset with the scan state every batch)
  // home region of the batch table (table_insert): *home & mask, written by the previous batch's clear
  // from its node count (adaptive); home_fixed != 0 overrides it (HELIOS_TABLE_HOME)
  const uint32_t* home;
  uint32_t* home_next;
  uint32_t home_fixed;
  // shared-memory tile dedup: tile_rows[h] > 0 = hop h runs the tiled fill / assign /
  // relabel; elist[E0 + j] = {global slot, tile minpos} of the tile's j-th distinct id, ndist[t] = count
  int32_t tile_rows[HELIOS_MAX_HOPS];
  uint2* elist;
  uint32_t* ndist;
  int32_t fill_seg;  // fill with f-lane segments (default; HELIOS_FILL_SEG=0: power-of-two groups)
  int32_t idx_ef;    // evict-first L2 policy on the fill's CSR index reads (default; HELIOS_SAMPLE_IDX_EVICT=0: off)
};

// The batches of one launch (a plan slot's group): the chain's kernels run with
// gridDim.y = n and CTA row y works on batch y; every batch keeps its own table, scan state and
// outputs, so a group is exactly n independent batches sharing each kernel launch.
struct SampleGroup {
  SampleCtx c[kMaxGroup];
};

// N_0 = seeds: copy into nodes, insert into the table with local id = position.  Duplicate or
// out-of-range seeds are latched (reading 7).
__device__ __forceinline__ uint32_t home_mask(const SampleCtx& c) {
  return c.home_fixed ? c.home_fixed : (ld_volatile_u32(c.home) & c.mask);
}

__device__ __forceinline__ void insert_seed(const SampleCtx& c, int64_t i, const int64_t* __restrict__ seeds,
                                            uint32_t hm) {
  const int64_t u = seeds[i];
  c.nodes[i] = u;
  c.node_slot[i] = kEmpty;
  if (u < 0 || u >= c.V) {
    latch(c.err, HELIOS_E_RANGE);
    return;
  }
  bool fresh;
  const uint32_t s = table_insert(c.tab, c.mask, hm, (uint32_t)u, kEmpty, &fresh);
  c.node_slot[i] = s;
  if (!fresh) {
    latch(c.err, HELIOS_E_INVALID);
    return;
  }
  c.tab[s].local = (uint32_t)i;
}

// ---- shared-memory tile dedup (north_star: "warp-cooperative dedup/relabel via a shared-memory hash
// plus radix compaction") ----------------------------------------------------------------------------
// Hop h's frontier rows are cut into tiles of tile_rows[h] consecutive rows, so a tile's sampled
// edges are the consecutive positions [E0, E1) = [bp[r0], bp[r1]) (at most kTileEdges).  The fill
// dedups a tile's ids in a shared-memory hash first (key, tile-minimum position) and touches the
// global table once per DISTINCT id of the tile (insert + minpos lowering) instead of once per
// edge; every edge keeps the index of its tile-distinct entry (slot_of[e] = E0 + j).  The assign
// reads the tile's distinct entries (not its edges), marks the first occurrences of ids new at this
// hop in a shared bitmap over the tile's edge positions, ranks them by popcount prefix (the radix
// compaction: rank = position order within the tile) and takes the tile's offset from a decoupled
// look-back over tiles in order, so new ids are numbered exactly in first-occurrence order (the
// oracle's).  The relabel reads the local ids of a tile's distinct entries into shared memory once
// and writes the tile's block indices from there.
constexpr int kTileEdges = 1024;            // sampled edges per tile at most (tile_rows * f_h)
constexpr int kTileSlots = 2 * kTileEdges;  // shared hash slots (load <= 0.5)

__device__ __forceinline__ int64_t tile_count(const SampleCtx& c, int h) {
  const int64_t n = c.level_counts[h];
  return (n + c.tile_rows[h] - 1) / c.tile_rows[h];
}

// Relabel of hop h, tiled: block indices from the local ids of each tile's distinct entries.
__device__ __forceinline__ void dev_relabel_tile(const SampleCtx& c, int h) {
  __shared__ uint32_t s_loc[kTileEdges];
  const int TR = c.tile_rows[h];
  const int64_t n = c.level_counts[h];
  const int64_t nt = tile_count(c, h);
  const int32_t* __restrict__ bp = c.bp[h];
  int32_t* __restrict__ bi = c.bi[h];
  for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const int64_t r0 = t * TR;
    const int64_t E0 = bp[r0], E1 = bp[min(n, r0 + TR)];
    const uint32_t nd = c.ndist[t];
    for (uint32_t j = threadIdx.x; j < nd; j += blockDim.x) s_loc[j] = c.tab[c.elist[E0 + j].x].local;
    __syncthreads();
    for (int64_t e = E0 + threadIdx.x; e < E1; e += blockDim.x) bi[e] = (int32_t)s_loc[c.slot_of[e] - (uint32_t)E0];
    __syncthreads();
  }
}

__device__ __forceinline__ void dev_relabel_any(const SampleCtx& c, int h) {
  if (c.tile_rows[h] > 0) {
    dev_relabel_tile(c, h);
    return;
  }
  const int64_t ep = c.edge_counts[h];
  int32_t* __restrict__ bi = c.bi[h];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ep; e += (int64_t)gridDim.x * blockDim.x)
    bi[e] = (int32_t)c.tab[c.slot_of[e]].local;
}

// Hop h degree scan: k_i = min(deg(N_h[i]), f_h), block_indptr[h] = exclusive scan (persistent tile
// loop + decoupled look-back), e_h = total.  Hop 0 reads N_0 = seeds from the parameters and inserts
// them into the table on the side; hop h > 0 relabels hop h-1's edges on the side.
template <int BLK>
__device__ __forceinline__ void dev_count_scan(const SampleCtx& c, int h) {
  constexpr int kTile = BLK * kScanItems;
  using BS = cub::BlockScan<long long, BLK>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned s_tile;
  __shared__ long long s_prefix;
  const int32_t f = c.fan[h];
  const int64_t* seeds = (const int64_t*)c.params[2];
  const int64_t* rows = (h == 0) ? seeds : c.nodes;
  const int64_t n = (h == 0) ? c.params[1] : c.level_counts[h];
  const ScanState& ss = c.row_scan[h];
  int32_t* __restrict__ bp = c.bp[h];
  for (;;) {  // tiles are taken in ticket order until they pass n
    const unsigned tile = tile_ticket(ss, &s_tile);
    const int64_t base = (int64_t)tile * kTile;
    if (tile > 0 && base >= n) break;
    if (h == 0 && tile == 0 && threadIdx.x == 0) c.level_counts[0] = n;
    long long k[kScanItems];
    long long sum = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; q++) {
      const int64_t i = base + threadIdx.x * kScanItems + q;
      k[q] = 0;
      if (i < n) {
        const int64_t v = rows[i];
        if ((uint64_t)v < (uint64_t)c.V) {
          const int64_t d = c.indptr[v + 1] - c.indptr[v];
          k[q] = (f < 0) ? d : min(d, (int64_t)f);
        }
      }
      sum += k[q];
    }
    long long excl, agg;
    BS(tmp).ExclusiveSum(sum, excl, agg);
    const long long prefix = tile_lookback(ss, tile, agg, &s_prefix);
    long long run = prefix + excl;
#pragma unroll
    for (int q = 0; q < kScanItems; q++) {
      const int64_t i = base + threadIdx.x * kScanItems + q;
      if (i < n) bp[i] = (int32_t)run;
      run += k[q];
    }
    if (threadIdx.x == 0 && ((n == 0 && tile == 0) || (base < n && n <= base + kTile))) {
      bp[n] = (int32_t)(prefix + agg);
      c.edge_counts[h] = prefix + agg;
    }
    __syncthreads();
  }
  if (h == 0) {  // side job: N_0 = seeds into the table, spread over the whole grid
    const uint32_t hm = home_mask(c);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      insert_seed(c, i, seeds, hm);
  }
  if (h > 0) dev_relabel_any(c, h - 1);  // side job: hop h-1's local ids are final (its assign has completed)
}

__device__ __forceinline__ void insert_edge(const SampleCtx& c, int64_t e, uint32_t u, uint32_t hm) {
  bool fresh;
  c.slot_of[e] = table_insert(c.tab, c.mask, hm, u, (uint32_t)e, &fresh);
}

// Hop h fill: one G-lane group per frontier row (G = power of two >= min(f, 32), >= 4).  Copy the
// whole adjacency when k == d; else Floyd's k-subset, lane j owning draw j and the sequential
// resolution done with group ballots.  Every sampled id is inserted into the table right away and
// atomicMin records the first edge position of ids new at this hop.
template <int G>
__device__ __forceinline__ void dev_fill_insert(const SampleCtx& c, int h) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const unsigned gmask = (G == 32) ? 0xFFFFFFFFu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int32_t f = c.fan[h];
  const uint64_t key = (uint64_t)c.params[0];
  const int64_t n = c.level_counts[h];
  const int32_t* __restrict__ bp = c.bp[h];
  int32_t* scratch = c.bi[h];
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
  const uint32_t hm = home_mask(c);
  for (int64_t i = grp; i < n; i += ngrp) {
    const int64_t v = c.nodes[i];
    int64_t base = 0, d = 0;
    if ((uint64_t)v < (uint64_t)c.V) {
      base = c.indptr[v];
      d = c.indptr[v + 1] - base;
    }
    const int64_t off = bp[i];
    const int64_t k = (f < 0) ? d : min(d, (int64_t)f);
    if (k == d) {  // every neighbour, CSR order, no RNG consumed
      for (int64_t p = gl; p < d; p += G)
        insert_edge(c, off + p, (uint32_t)(c.idx_ef ? ld_index_ef(c.indices + base + p) : c.indices[base + p]), hm);
    } else if (k <= G) {
      uint32_t t = 0, m = 0;
      if (gl < k) {
        m = (uint32_t)(d - k + gl + 1);
        t = __umulhi(philox_word(key, (uint32_t)h, (uint64_t)v, (uint32_t)gl), m);
      }
      uint32_t P = 0;
      for (int j = 0; j < (int)k; j++) {
        const uint32_t tj = __shfl_sync(gmask, t, j, G);
        const unsigned hit = __ballot_sync(gmask, gl < j && P == tj);
        if (gl == j) P = hit ? (m - 1) : tj;
      }
      if (gl < k) insert_edge(c, off + gl, (uint32_t)(c.idx_ef ? ld_index_ef(c.indices + base + P) : c.indices[base + P]), hm);
    } else {  // k > G (fanout > 32): leader runs Floyd serially, positions kept in the scratch row
      if (gl == 0) {
        for (int64_t j = 0; j < k; j++) {
          const uint32_t m = (uint32_t)(d - k + j + 1);
          const uint32_t tj = __umulhi(philox_word(key, (uint32_t)h, (uint64_t)v, (uint32_t)j), m);
          bool seen = false;
          for (int64_t q = 0; q < j; q++)
            if ((uint32_t)scratch[off + q] == tj) {
              seen = true;
              break;
            }
          scratch[off + j] = (int32_t)(seen ? m - 1 : tj);
        }
      }
      __syncwarp(gmask);
      for (int64_t j = gl; j < k; j += G) insert_edge(c, off + j, (uint32_t)c.indices[base + scratch[off + j]], hm);
      __syncwarp(gmask);
    }
  }
}

// Tiled fill of hop h (see the tile dedup comment above): the sampling of every row is that of
// dev_fill_insert (same draws, same positions); only the table insert differs.
template <int G>
__device__ __forceinline__ void dev_fill_tile(const SampleCtx& c, int h) {
  __shared__ uint32_t s_key[kTileSlots], s_min[kTileSlots], s_li[kTileSlots];
  __shared__ uint16_t s_eslot[kTileEdges];
  __shared__ uint32_t s_cnt;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const unsigned gmask = (G == 32) ? 0xFFFFFFFFu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const int32_t f = c.fan[h];
  const uint64_t key = (uint64_t)c.params[0];
  const int TR = c.tile_rows[h];
  const int64_t n = c.level_counts[h];
  const int64_t nt = tile_count(c, h);
  const int32_t* __restrict__ bp = c.bp[h];
  int32_t* scratch = c.bi[h];
  for (int p = threadIdx.x; p < kTileSlots; p += blockDim.x) {
    s_key[p] = kEmpty;
    s_min[p] = kEmpty;
  }
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int grp = threadIdx.x / G, ngrp = blockDim.x / G;
  for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const int64_t r0 = t * TR, r1 = min(n, r0 + TR);
    const int64_t E0 = bp[r0], E1 = bp[r1];
    auto ins = [&](int64_t e, uint32_t u) {  // shared-memory insert-or-find, tile-minimum position
      uint32_t q = hash32(u) & (kTileSlots - 1);
      for (;;) {
        const uint32_t k = atomicCAS(&s_key[q], kEmpty, u);
        if (k == kEmpty || k == u) break;
        q = (q + 1) & (kTileSlots - 1);
      }
      atomicMin(&s_min[q], (uint32_t)e);
      s_eslot[e - E0] = (uint16_t)q;
    };
    for (int64_t i = r0 + grp; i < r1; i += ngrp) {
      const int64_t v = c.nodes[i];
      int64_t base = 0, d = 0;
      if ((uint64_t)v < (uint64_t)c.V) {
        base = c.indptr[v];
        d = c.indptr[v + 1] - base;
      }
      const int64_t off = bp[i];
      const int64_t k = min(d, (int64_t)f);
      if (k == d) {
        for (int64_t p = gl; p < d; p += G) ins(off + p, (uint32_t)c.indices[base + p]);
      } else if (k <= G) {
        uint32_t tt = 0, m = 0;
        if (gl < k) {
          m = (uint32_t)(d - k + gl + 1);
          tt = __umulhi(philox_word(key, (uint32_t)h, (uint64_t)v, (uint32_t)gl), m);
        }
        uint32_t P = 0;
        for (int j = 0; j < (int)k; j++) {
          const uint32_t tj = __shfl_sync(gmask, tt, j, G);
          const unsigned hit = __ballot_sync(gmask, gl < j && P == tj);
          if (gl == j) P = hit ? (m - 1) : tj;
        }
        if (gl < k) ins(off + gl, (uint32_t)c.indices[base + P]);
      } else {  // k > G: serial Floyd in the scratch row (as dev_fill_insert)
        if (gl == 0) {
          for (int64_t j = 0; j < k; j++) {
            const uint32_t m = (uint32_t)(d - k + j + 1);
            const uint32_t tj = __umulhi(philox_word(key, (uint32_t)h, (uint64_t)v, (uint32_t)j), m);
            bool seen = false;
            for (int64_t q = 0; q < j; q++)
              if ((uint32_t)scratch[off + q] == tj) {
                seen = true;
                break;
              }
            scratch[off + j] = (int32_t)(seen ? m - 1 : tj);
          }
        }
        __syncwarp(gmask);
        for (int64_t j = gl; j < k; j += G) ins(off + j, (uint32_t)c.indices[base + scratch[off + j]]);
        __syncwarp(gmask);
      }
    }
    __syncthreads();
    // one global insert per distinct id of the tile, with the tile's first position of it
    const uint32_t hm = home_mask(c);
    for (int q = threadIdx.x; q < kTileSlots; q += blockDim.x) {
      const uint32_t u = s_key[q];
      if (u != kEmpty) {
        bool fresh;
        const uint32_t mp = s_min[q];
        const uint32_t gs = table_insert(c.tab, c.mask, hm, u, mp, &fresh);
        const uint32_t j = atomicAdd(&s_cnt, 1u);
        c.elist[E0 + j] = make_uint2(gs, mp);
        s_li[q] = j;
        s_key[q] = kEmpty;
        s_min[q] = kEmpty;
      }
    }
    __syncthreads();
    for (int64_t e = E0 + threadIdx.x; e < E1; e += blockDim.x) c.slot_of[e] = (uint32_t)E0 + s_li[s_eslot[e - E0]];
    if (threadIdx.x == 0) {
      c.ndist[t] = s_cnt;
      s_cnt = 0;
    }
    __syncthreads();
  }
}

// Tiled assign of hop h: tiles in ticket (= edge position) order; first occurrences of new ids are
// ranked inside the tile by a popcount prefix over a shared bitmap of the tile's edge positions.
template <int BLK>
__device__ __forceinline__ void dev_assign_tile(const SampleCtx& c, int h) {
  constexpr int kWords = kTileEdges / 32;
  __shared__ uint32_t s_bits[kWords], s_wpre[kWords];
  __shared__ uint32_t s_total;
  __shared__ unsigned s_tile;
  __shared__ long long s_prefix;
  const int TR = c.tile_rows[h];
  const int64_t n = c.level_counts[h];
  const int64_t nt = tile_count(c, h);
  const int64_t nh = n;
  const int32_t* __restrict__ bp = c.bp[h];
  const ScanState& ss = c.edge_scan[h];
  if (threadIdx.x < kWords) s_bits[threadIdx.x] = 0;
  __syncthreads();
  for (;;) {
    const unsigned tile = tile_ticket(ss, &s_tile);
    if (tile > 0 && (int64_t)tile >= nt) break;
    const bool real = (int64_t)tile < nt;
    const int64_t E0 = real ? bp[(int64_t)tile * TR] : 0;
    const uint32_t nd = real ? c.ndist[tile] : 0;
    for (uint32_t j = threadIdx.x; j < nd; j += BLK) {
      const uint2 ent = c.elist[E0 + j];
      const uint4 t = ld_volatile_v4u32(&c.tab[ent.x]);  // {minpos, key, local, pad}
      if (t.z == kEmpty && t.x == ent.y) {
        const uint32_t r = ent.y - (uint32_t)E0;
        atomicOr(&s_bits[r >> 5], 1u << (r & 31));
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // word prefix of the popcounts (kWords == 32)
      const uint32_t v = __popc(s_bits[threadIdx.x]);
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)threadIdx.x >= o) incl += y;
      }
      s_wpre[threadIdx.x] = incl - v;
      if (threadIdx.x == 31) s_total = incl;
    }
    __syncthreads();
    const long long prefix = tile_lookback(ss, tile, (long long)s_total, &s_prefix);
    for (uint32_t j = threadIdx.x; j < nd; j += BLK) {
      const uint2 ent = c.elist[E0 + j];
      const uint32_t r = ent.y - (uint32_t)E0;
      if (r < (uint32_t)kTileEdges) {
        const uint32_t w = s_bits[r >> 5];
        if ((w >> (r & 31)) & 1u) {  // this entry holds the first occurrence of an id new at hop h
          const int64_t id = nh + prefix + s_wpre[r >> 5] + __popc(w & ((1u << (r & 31)) - 1u));
          c.nodes[id] = (int64_t)(c.tab[ent.x].km >> 32);
          c.node_slot[id] = ent.x;
          c.tab[ent.x].local = (uint32_t)id;
        }
      }
    }
    if (threadIdx.x == 0 && ((nt == 0 && tile == 0) || (int64_t)tile == nt - 1)) c.level_counts[h + 1] = nh + prefix + s_total;
    __syncthreads();
    if (threadIdx.x < kWords) s_bits[threadIdx.x] = 0;
    __syncthreads();
  }
}

// Hop h fill with S-lane segments, S = f_h (1 <= f_h <= 32; the default, HELIOS_FILL_SEG=0 disables): a warp samples
// floor(32 / S) rows at once instead of 32 / G with G the power of two >= f (f = 5: 6 rows on 30 busy
// lanes instead of 4 rows on 20; f = 10: 3 instead of 2), so the same rows hold a third fewer warp
// slots.  Same draws, positions and inserts as dev_fill_insert (k <= f = S, so the serial path never
// applies); shuffles and ballots use the segment's lane mask with explicit source lanes.
__device__ __forceinline__ void dev_fill_seg(const SampleCtx& c, int h) {
  const int lane = threadIdx.x & 31;
  const int32_t f = c.fan[h];
  const int S = f;
  const int rpw = 32 / S;
  const int seg = lane / S;
  if (seg >= rpw) return;  // spare lanes (32 mod S of them); they take part in no shuffle
  const int sl = lane - seg * S;
  const int bl = seg * S;
  const unsigned smask = (S == 32) ? 0xFFFFFFFFu : (((1u << S) - 1u) << bl);
  const uint64_t key = (uint64_t)c.params[0];
  const int64_t n = c.level_counts[h];
  const int32_t* __restrict__ bp = c.bp[h];
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t hm = home_mask(c);
  for (int64_t i = warp * rpw + seg; i < n; i += nwarps * rpw) {
    const int64_t v = c.nodes[i];
    int64_t base = 0, d = 0;
    if ((uint64_t)v < (uint64_t)c.V) {
      base = c.indptr[v];
      d = c.indptr[v + 1] - base;
    }
    const int64_t off = bp[i];
    const int64_t k = min(d, (int64_t)f);
    if (k == d) {  // every neighbour, CSR order, no RNG consumed
      for (int64_t p = sl; p < d; p += S)
        insert_edge(c, off + p, (uint32_t)(c.idx_ef ? ld_index_ef(c.indices + base + p) : c.indices[base + p]), hm);
    } else {  // Floyd's k-subset, lane sl owning draw sl
      uint32_t t = 0, m = 0;
      if (sl < k) {
        m = (uint32_t)(d - k + sl + 1);
        t = __umulhi(philox_word(key, (uint32_t)h, (uint64_t)v, (uint32_t)sl), m);
      }
      uint32_t P = 0;
      for (int j = 0; j < (int)k; j++) {
        const uint32_t tj = __shfl_sync(smask, t, bl + j);
        const unsigned hit = __ballot_sync(smask, sl < j && P == tj);
        if (sl == j) P = hit ? (m - 1) : tj;
      }
      if (sl < k) insert_edge(c, off + sl, (uint32_t)(c.idx_ef ? ld_index_ef(c.indices + base + P) : c.indices[base + P]), hm);
    }
  }
}

__device__ __forceinline__ int fill_group(int32_t f) { return (f < 0 || f > 16) ? 32 : (f > 8 ? 16 : (f > 4 ? 8 : 4)); }

// Hop h dedup/relabel: flag = "this edge is the first occurrence of an id new at this hop"; the
// scan of the flags numbers the new ids n_h, n_h+1, ... in first-occurrence order and appends them
// to N_{h+1} (persistent tile loop + decoupled look-back).
template <int BLK>
__device__ __forceinline__ void dev_assign(const SampleCtx& c, int h) {
  constexpr int kTile = BLK * kScanItems;
  using BS = cub::BlockScan<int, BLK>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned s_tile;
  __shared__ long long s_prefix;
  const int64_t eh = c.edge_counts[h];
  const int64_t nh = c.level_counts[h];
  const ScanState& ss = c.edge_scan[h];
  for (;;) {
    const unsigned tile = tile_ticket(ss, &s_tile);
    const int64_t base = (int64_t)tile * kTile;
    if (tile > 0 && base >= eh) break;
    int flag[kScanItems];
    uint32_t slot[kScanItems];
    int sum = 0;
#pragma unroll
    for (int q = 0; q < kScanItems; q++) {
      const int64_t e = base + threadIdx.x * kScanItems + q;
      flag[q] = 0;
      slot[q] = 0;
      if (e < eh) {
        slot[q] = c.slot_of[e];
        const uint4 t = ld_volatile_v4u32(&c.tab[slot[q]]);  // {minpos, key, local, pad}
        flag[q] = (t.z == kEmpty && t.x == (uint32_t)e) ? 1 : 0;
      }
      sum += flag[q];
    }
    int excl, agg;
    BS(tmp).ExclusiveSum(sum, excl, agg);
    const long long prefix = tile_lookback(ss, tile, agg, &s_prefix);
    long long run = prefix + excl;
#pragma unroll
    for (int q = 0; q < kScanItems; q++) {
      if (flag[q]) {
        const int64_t id = nh + run;
        c.nodes[id] = (int64_t)(c.tab[slot[q]].km >> 32);
        c.node_slot[id] = slot[q];
        c.tab[slot[q]].local = (uint32_t)id;
        run++;
      }
    }
    if (threadIdx.x == 0 && ((eh == 0 && tile == 0) || (base < eh && eh <= base + kTile)))
      c.level_counts[h + 1] = nh + prefix + agg;
    __syncthreads();
  }
}

__device__ __forceinline__ void dev_relabel(const SampleCtx& c, int h) { dev_relabel_any(c, h); }

// Returns the batch hash table to all-EMPTY by clearing exactly the slots of the batch's nodes
// (every occupied slot belongs to one node of N_L).
__device__ __forceinline__ void dev_table_clear(const SampleCtx& c) {
  const int64_t n = c.level_counts[c.L];
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the next batch's home region: 2^k >= 2.5 n, at least 1/8 of the
    // worst-case table and at least half of this batch's region (it shrinks one halving per batch), which
    // bounds the probe runs of a batch much larger than its predecessor
    uint32_t hm = max(max(1023u, c.mask >> 3), (ld_volatile_u32(c.home) & c.mask) >> 1);
    while (hm < c.mask && (int64_t)hm + 1 < n * 5 / 2) hm = hm * 2 + 1;
    *c.home_next = hm & c.mask;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = c.node_slot[i];
    if (s != kEmpty) {
      *reinterpret_cast<uint4*>(&c.tab[s]) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    }
  }
}

__device__ __forceinline__ void dev_insert_seeds(const SampleCtx& c) {  // L = 0
  const int64_t B = c.params[1];
  const int64_t* seeds = (const int64_t*)c.params[2];
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i0 == 0) c.level_counts[0] = B;
  const uint32_t hm = home_mask(c);
  for (int64_t i = i0; i < B; i += (int64_t)gridDim.x * blockDim.x) insert_seed(c, i, seeds, hm);
}

// ---- multi-kernel path: one kernel per phase, chained with programmatic dependent launch ----
// blockIdx.y selects the batch of the group.
__global__ void __launch_bounds__(kScanBlock) k_count_scan(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  if (h > 0) pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * h);
  dev_count_scan<kScanBlock>(c, h);
}
template <int G>
__global__ void __launch_bounds__(256) k_fill_insert(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * h + 1);
  dev_fill_insert<G>(c, h);
}
template <int G>
__global__ void __launch_bounds__(256) k_fill_tile(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * h + 1);
  dev_fill_tile<G>(c, h);
}
__global__ void __launch_bounds__(256) k_fill_seg(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * h + 1);
  dev_fill_seg(c, h);
}
__global__ void __launch_bounds__(kScanBlock) k_assign_tile(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * h + 2);
  dev_assign_tile<kScanBlock>(c, h);
}
__global__ void __launch_bounds__(kScanBlock) k_dedup_assign(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * h + 2);
  dev_assign<kScanBlock>(c, h);
}
__global__ void __launch_bounds__(256) k_relabel(const __grid_constant__ SampleGroup P, int h) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * c.L);
  dev_relabel(c, h);
}
__global__ void __launch_bounds__(256) k_table_clear(const __grid_constant__ SampleGroup P) {
  const SampleCtx& c = P.c[blockIdx.y];
  pdl_wait();
  pdl_trigger();
  TraceScope ts(c.params, 3 * c.L + 1);
  dev_table_clear(c);
}
__global__ void __launch_bounds__(256) k_insert_seeds(const __grid_constant__ SampleGroup P) {
  dev_insert_seeds(P.c[blockIdx.y]);
}

// ---- persistent path: the whole batch in one cooperative kernel, phases separated by a grid
// barrier (3 per hop + 1), so a batch costs one launch instead of 2 + 3L ----
constexpr uint64_t kBarrierTimeoutNs = 10ull * 1000000000ull;

// Generation barrier over the cooperative grid.  bar[0] counts arrivals (all-ones = none: the scan
// state memset resets it every batch), bar[1] is the generation.  A watchdog latches E_TIMEOUT
// instead of hanging if the grid is ever not co-resident.
__device__ __forceinline__ bool grid_sync(const SampleCtx& c) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1;
    const unsigned gen = ld_volatile_u32(c.bar + 1);
    __threadfence();
    const unsigned arrived = atomicAdd(c.bar, 1u) + 2u;  // all-ones + 1 arrival -> 1
    if (arrived == gridDim.x) {
      atomicExch(c.bar, 0xFFFFFFFFu);
      __threadfence();
      atomicAdd(c.bar + 1, 1u);
    } else {
      const uint64_t t0 = globaltimer();
      while (ld_volatile_u32(c.bar + 1) == gen) {
        if (globaltimer() - t0 > kBarrierTimeoutNs) {
          latch(c.err, HELIOS_E_TIMEOUT);
          ok = 0;
          break;
        }
        __nanosleep(20);
      }
    }
    __threadfence();
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

__global__ void __launch_bounds__(256, 2) k_sample_batch(SampleCtx c) {
  if (c.L == 0) {
    dev_insert_seeds(c);
    if (!grid_sync(c)) return;
  }
  for (int h = 0; h < c.L; h++) {
    dev_count_scan<kScanBlock>(c, h);
    if (!grid_sync(c)) return;
    switch (fill_group(c.fan[h])) {
      case 4: dev_fill_insert<4>(c, h); break;
      case 8: dev_fill_insert<8>(c, h); break;
      case 16: dev_fill_insert<16>(c, h); break;
      default: dev_fill_insert<32>(c, h); break;
    }
    if (!grid_sync(c)) return;
    dev_assign<kScanBlock>(c, h);
    if (!grid_sync(c)) return;
  }
  if (c.L > 0) {
    dev_relabel(c, c.L - 1);
    if (!grid_sync(c)) return;
  }
  dev_table_clear(c);
}

// ---- cluster path (default): the whole batch in ONE launch of one thread-block cluster ------------
// The cluster's CTAs are co-scheduled by the hardware (on one GPC) and its barrier
// (barrier.cluster.arrive.release / wait.acquire) is a hardware barrier with cluster-scope memory
// ordering, so the 3L + 1 phase boundaries cost no kernel launches, no PDL waits and no software
// grid barrier; batches of different plan slots run as independent clusters side by side.  The
// phases are the chain's device functions (same code, same results) on BLK-thread CTAs.
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int BLK>
__global__ void __launch_bounds__(BLK, 1) k_sample_cluster(SampleCtx c) {
  if (c.L == 0) {
    dev_insert_seeds(c);
    cluster_sync();
  }
  for (int h = 0; h < c.L; h++) {
    dev_count_scan<BLK>(c, h);
    cluster_sync();
    switch (fill_group(c.fan[h])) {
      case 4: dev_fill_insert<4>(c, h); break;
      case 8: dev_fill_insert<8>(c, h); break;
      case 16: dev_fill_insert<16>(c, h); break;
      default: dev_fill_insert<32>(c, h); break;
    }
    cluster_sync();
    dev_assign<BLK>(c, h);
    cluster_sync();
  }
  if (c.L > 0) {
    dev_relabel(c, c.L - 1);
    cluster_sync();
  }
  dev_table_clear(c);
}

// hot[v] += 1 for every v of the batch's N_L.  An out-of-range id (a bad presample seed, already
// latched E_RANGE by insert_seed) is skipped rather than counted out of bounds.
__global__ void k_hot_count(const int64_t* __restrict__ nodes, const int64_t* __restrict__ n_nodes, int64_t V,
                            uint64_t* hot) {
  const int64_t n = *n_nodes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = nodes[i];
    if ((uint64_t)v < (uint64_t)V) atomicAdd((unsigned long long*)&hot[v], 1ull);
  }
}

helios_status hot_count_enqueue(const int64_t* nodes, const int64_t* n_nodes, int64_t max_nodes, int64_t V, uint64_t* hot,
                                int sms, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((max_nodes + 255) / 256, (int64_t)sms * 8);
  k_hot_count<<<std::max(grid, 1), 256, 0, st>>>(nodes, n_nodes, V, hot);
  HCUDA(cudaGetLastError());
  return HELIOS_OK;
}

// ---- random-sector probe (measurement) --------------------------------------------------------
// Every thread issues `per` independent loads at SplitMix64-random positions of indices[E].
__global__ void k_probe_random(const int32_t* __restrict__ a, int64_t E, int per, uint64_t seed, int* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  int acc = 0;
  for (int k = 0; k < per; k++) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (t * (uint64_t)per + k + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    acc += __ldcg(a + (int64_t)__umul64hi(z, (uint64_t)E));
  }
  if (acc == 0x7FFFFFFF) *sink = acc;
}

helios_status probe_random_impl(helios_graph* g, int64_t n, int32_t reps, float* ms) {
  HCHECK(n > 0 && reps > 0 && ms, HELIOS_E_INVALID, "probe: n_reads %lld, reps %d", (long long)n, reps);
  HCHECK(g->E > 0 && !g->topo_host, HELIOS_E_STATE, "probe: no HBM-resident CSR indices");
  const int per = 16;
  const int64_t threads = (n + per - 1) / per;
  const int grid = (int)std::max<int64_t>(1, (threads + 255) / 256);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int* sink = nullptr;
  HCUDA(cudaMalloc(&sink, sizeof(int)));
  HCUDA(cudaEventCreate(&e0));
  HCUDA(cudaEventCreate(&e1));
  float tot = 0;
  cudaError_t err = cudaSuccess;
  for (int r = 0; r < reps && err == cudaSuccess; r++) {
    cudaEventRecord(e0, 0);
    k_probe_random<<<grid, 256>>>(g->indices, g->E, per, 0xA5A5A5A5ull * (uint64_t)(r + 1), sink);
    cudaEventRecord(e1, 0);
    err = cudaEventSynchronize(e1);
    float t = 0;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&t, e0, e1);
    tot += t;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return fail(HELIOS_E_CUDA, "probe_random: %s", cudaGetErrorString(err));
  *ms = tot / reps * (float)n / (float)(threads * per);  // per n reads
  return HELIOS_OK;
}

// ---- host side --------------------------------------------------------------------------------

helios_status sample_bounds(int64_t n_seeds, const int32_t* fanouts, int32_t L, int64_t V, int64_t E, int64_t* max_nodes,
                            int64_t* level, int64_t* edges) {
  HCHECK(L >= 0 && L <= HELIOS_MAX_HOPS, HELIOS_E_INVALID, "L=%d out of [0,%d]", L, HELIOS_MAX_HOPS);
  HCHECK(n_seeds >= 0, HELIOS_E_INVALID, "n_seeds < 0");
  int64_t n = n_seeds;
  if (level) level[0] = n;
  for (int h = 0; h < L; h++) {
    HCHECK(fanouts && (fanouts[h] >= 1 || fanouts[h] == -1), HELIOS_E_INVALID, "fanout[%d]=%d (need >=1 or -1)", h,
           fanouts ? fanouts[h] : 0);
    const int64_t e = (fanouts[h] < 0) ? E : std::min<int64_t>(n * (int64_t)fanouts[h], E);
    if (edges) edges[h] = e;
    n = std::min<int64_t>(V, n + e);
    if (level) level[h + 1] = n;
  }
  if (max_nodes) *max_nodes = n;
  return HELIOS_OK;
}

helios_status sample_check_out(const helios_graph* g, int64_t B, const int32_t* fanouts, int32_t L,
                               const helios_blocks* out) {
  int64_t maxn, lvl[HELIOS_MAX_HOPS + 1], edg[HELIOS_MAX_HOPS];
  helios_status s = sample_bounds(B, fanouts, L, g->V, g->E, &maxn, lvl, edg);
  if (s != HELIOS_OK) return s;
  HCHECK(out && out->nodes && out->level_counts && (L == 0 || out->edge_counts), HELIOS_E_INVALID, "null output");
  HCHECK(out->nodes_cap >= maxn, HELIOS_E_CAPACITY, "nodes_cap %lld < bound %lld", (long long)out->nodes_cap,
         (long long)maxn);
  for (int h = 0; h < L; h++) {
    HCHECK(out->block_indptr[h] && out->block_indices[h], HELIOS_E_INVALID, "null block buffer for hop %d", h);
    HCHECK(out->indptr_cap[h] >= lvl[h] + 1, HELIOS_E_CAPACITY, "indptr_cap[%d] %lld < %lld", h,
           (long long)out->indptr_cap[h], (long long)lvl[h] + 1);
    HCHECK(out->edges_cap[h] >= edg[h], HELIOS_E_CAPACITY, "edges_cap[%d] %lld < %lld", h, (long long)out->edges_cap[h],
           (long long)edg[h]);
    HCHECK(edg[h] < (1ll << 31), HELIOS_E_CAPACITY, "hop %d edge bound %lld exceeds int32 block indices", h,
           (long long)edg[h]);
  }
  return HELIOS_OK;
}

static uint64_t pow2_at_least(int64_t x) {
  uint64_t p = 1024;
  while ((int64_t)p < x) p <<= 1;
  return p;
}

void ws_free(SampleWS& w) {
  if (w.reset_base) cudaFree(w.reset_base);
  if (w.slot_of) cudaFree(w.slot_of);
  if (w.node_slot) cudaFree(w.node_slot);
  if (w.elist) cudaFree(w.elist);
  if (w.ndist) cudaFree(w.ndist);
  if (w.d_params) cudaFree(w.d_params);
  if (w.h_params) cudaFreeHost(w.h_params);
  if (w.params_ev) cudaEventDestroy(w.params_ev);
  w = SampleWS{};
}

static bool cluster_fits(int cl);

helios_status ws_ensure(helios_graph* g, SampleWS& w, int64_t B, const int32_t* fanouts, int32_t L) {
  int64_t maxn, lvl[HELIOS_MAX_HOPS + 1], edg[HELIOS_MAX_HOPS];
  helios_status s = sample_bounds(B, fanouts, L, g->V, g->E, &maxn, lvl, edg);
  if (s != HELIOS_OK) return s;
  // shared-memory tile dedup for hops with a bounded fanout (HELIOS_SAMPLE_DEDUP=smem)
  bool tiled = false;
  if (const char* e = getenv("HELIOS_SAMPLE_DEDUP")) tiled = !strcmp(e, "smem");
  int32_t trows[HELIOS_MAX_HOPS] = {};
  int64_t max_e = 1, tiles_r = 1, tiles_e = 1, tiles_t = 1;
  for (int h = 0; h < L; h++) {
    max_e = std::max(max_e, edg[h]);
    tiles_r = std::max(tiles_r, (lvl[h] + kScanTile - 1) / kScanTile);
    tiles_e = std::max(tiles_e, (edg[h] + kScanTile - 1) / kScanTile);
    if (tiled && fanouts[h] > 0 && fanouts[h] <= kTileEdges) {
      trows[h] = kTileEdges / fanouts[h];
      tiles_t = std::max(tiles_t, (lvl[h] + trows[h] - 1) / trows[h]);
    }
  }
  tiles_e = std::max(tiles_e, tiles_t);  // the tiled assign's look-back uses the edge scan state
  // worst-case load <= 0.8 (n_L bound / table); the typical batch fills a few percent of it
  const uint64_t T64 = pow2_at_least(std::min<int64_t>(g->V, std::max<int64_t>(maxn, 1)) * 5 / 4);
  // slots are u32-indexed with kEmpty = 2^32-1 reserved: at most 2^31 slots
  HCHECK(T64 <= (1ull << 31), HELIOS_E_CAPACITY, "batch hash table of %llu slots exceeds 2^31 (V=%lld, node bound %lld)",
         (unsigned long long)T64, (long long)g->V, (long long)maxn);
  const uint32_t T = (uint32_t)T64;
  const int64_t max_nodes = std::max<int64_t>(maxn, 1);
  if (w.reset_base && T <= w.table_size && max_e <= w.cap_edges && tiles_r <= w.cap_tiles_rows &&
      tiles_e <= w.cap_tiles_edges && max_nodes <= w.cap_nodes && B <= w.cap_seeds && (!tiled || w.elist)) {
    for (int h = 0; h < HELIOS_MAX_HOPS; h++) w.tile_rows[h] = h < L ? trows[h] : 0;
    return HELIOS_OK;
  }
  HCUDA(cudaDeviceSynchronize());
  ws_free(w);
  const size_t table_bytes = (size_t)T * sizeof(TableSlot);
  const size_t status_bytes = (size_t)(tiles_r + tiles_e) * HELIOS_MAX_HOPS * 8;
  const size_t counter_bytes = (size_t)2 * HELIOS_MAX_HOPS * 4 + 8 + 8;  // + barrier, + home word
  w.reset_bytes = table_bytes + status_bytes + counter_bytes;
  HCUDA(cudaMalloc(&w.reset_base, w.reset_bytes));
  HCUDA(cudaMalloc(&w.slot_of, (size_t)max_e * 4));
  HCUDA(cudaMalloc(&w.node_slot, (size_t)max_nodes * 4));
  if (tiled) {
    HCUDA(cudaMalloc(&w.elist, (size_t)max_e * sizeof(uint2)));
    HCUDA(cudaMalloc(&w.ndist, (size_t)tiles_e * 4));
  }
  for (int h = 0; h < HELIOS_MAX_HOPS; h++) w.tile_rows[h] = h < L ? trows[h] : 0;
  w.cap_nodes = max_nodes;
  w.cap_seeds = std::max<int64_t>(B, 1);
  HCUDA(cudaMalloc(&w.d_params, (4 + w.cap_seeds) * sizeof(int64_t)));
  HCUDA(cudaHostAlloc(&w.h_params, (4 + w.cap_seeds) * sizeof(int64_t), cudaHostAllocDefault));
  HCUDA(cudaEventCreateWithFlags(&w.params_ev, cudaEventDisableTiming));
  w.table_size = T;
  w.cap_edges = max_e;
  w.cap_tiles_rows = tiles_r;
  w.cap_tiles_edges = tiles_e;
  char* p = w.reset_base;
  w.table = (TableSlot*)p;
  p += table_bytes;
  w.scan_base = p;
  for (int h = 0; h < HELIOS_MAX_HOPS; h++) {
    w.row_scan[h].status = (unsigned long long*)p;
    p += tiles_r * 8;
    w.edge_scan[h].status = (unsigned long long*)p;
    p += tiles_e * 8;
  }
  for (int h = 0; h < HELIOS_MAX_HOPS; h++) {
    w.row_scan[h].counter = (unsigned*)p;
    p += 4;
    w.edge_scan[h].counter = (unsigned*)p;
    p += 4;
  }
  w.bar = (unsigned*)p;
  p += 8;
  w.scan_bytes = (size_t)(p - w.scan_base);
  w.home = (uint32_t*)p;  // outside the per-batch reset; all-ones at allocation = home the whole table
  p += 8;
  if (const char* e = getenv("HELIOS_SAMPLE_PERSISTENT")) w.persistent = atoi(e) != 0;
  if (const char* e = getenv("HELIOS_FILL_SEG")) w.fill_seg = atoi(e) != 0;
  if (const char* e = getenv("HELIOS_SAMPLE_MODE")) {
    if (!strcmp(e, "cluster")) w.cluster = 8;
    else if (!strcmp(e, "cluster16")) w.cluster = 16;
    else if (!strcmp(e, "chain")) w.cluster = 0;
  }
  if (w.cluster) {  // a cluster of this size must be schedulable, else the chain is used
    static int ok8 = -1, ok16 = -1;
    int& ok = (w.cluster == 16) ? ok16 : ok8;
    if (ok < 0) ok = cluster_fits(w.cluster) ? 1 : 0;
    if (!ok) w.cluster = 0;
  }
  HCUDA(cudaMemset(w.reset_base, 0xFF, w.reset_bytes));  // the table starts all-EMPTY
  return HELIOS_OK;
}

helios_status ws_upload_params(SampleWS& w, uint64_t key, int64_t B, const int64_t* seeds, bool seeds_host,
                               cudaStream_t st, void* trace_row) {
  HCHECK(B <= w.cap_seeds, HELIOS_E_CAPACITY, "n_seeds %lld > workspace capacity %lld", (long long)B,
         (long long)w.cap_seeds);
  HCUDA(cudaEventSynchronize(w.params_ev));  // the previous upload has been consumed
  w.h_params[0] = (int64_t)key;
  w.h_params[1] = B;
  w.h_params[3] = (int64_t)(uintptr_t)trace_row;  // HELIOS_PLAN_TRACE row of this batch, or 0
  size_t bytes = 4 * sizeof(int64_t);
  if (seeds_host) {
    if (B > 0) memcpy(w.h_params + 4, seeds, B * sizeof(int64_t));
    w.h_params[2] = (int64_t)(uintptr_t)(w.d_params + 4);
    bytes += B * sizeof(int64_t);
  } else {
    w.h_params[2] = (int64_t)(uintptr_t)seeds;
  }
  HCUDA(cudaMemcpyAsync(w.d_params, w.h_params, bytes, cudaMemcpyHostToDevice, st));
  HCUDA(cudaEventRecord(w.params_ev, st));
  return HELIOS_OK;
}

static SampleCtx make_ctx(const helios_graph* g, const SampleWS& w, const int32_t* fanouts, int32_t L,
                          const helios_blocks* out) {
  SampleCtx c{};
  c.indptr = g->indptr;
  c.indices = g->indices;
  c.V = g->V;
  c.params = w.d_params;
  c.err = g->d_err;
  c.tab = w.table;
  c.mask = w.table_size - 1;
  c.slot_of = w.slot_of;
  c.node_slot = w.node_slot;
  c.nodes = out->nodes;
  c.level_counts = out->level_counts;
  c.edge_counts = out->edge_counts;
  for (int h = 0; h < L; h++) {
    c.bp[h] = out->block_indptr[h];
    c.bi[h] = out->block_indices[h];
    c.row_scan[h] = w.row_scan[h];
    c.edge_scan[h] = w.edge_scan[h];
    c.fan[h] = fanouts[h];
  }
  c.L = L;
  c.bar = w.bar;
  c.home = w.home;
  c.home_next = w.home;
  c.home_fixed = 0;
  if (const char* e = getenv("HELIOS_TABLE_HOME")) {  // fixed home region (0: the whole table, no adaptation)
    const long long v = atoll(e);
    uint32_t hm = 1023;
    while (hm < c.mask && (long long)hm + 1 < v) hm = hm * 2 + 1;
    c.home_fixed = (v <= 0) ? c.mask : (hm & c.mask);
  }
  const bool chain = !w.cluster && !w.persistent;  // the one-launch samplers run the global-table phases
  for (int h = 0; h < HELIOS_MAX_HOPS; h++) c.tile_rows[h] = (chain && h < L) ? w.tile_rows[h] : 0;
  c.elist = w.elist;
  c.ndist = w.ndist;
  c.fill_seg = w.fill_seg ? 1 : 0;
  c.idx_ef = 1;  // C2 +3.8 %, C3 within noise (profiles/r02/l2_policy_c2_c3.jsonl)
  if (const char* e = getenv("HELIOS_SAMPLE_IDX_EVICT")) c.idx_ef = atoi(e) != 0;
  return c;
}

template <int G>
static void launch_fill(const helios_graph* g, const SampleGroup& P, int n, int h, int64_t rows, cudaStream_t st) {
  const int TR = P.c[0].tile_rows[h];
  if (TR > 0) {  // tiled: one CTA per tile (tiles taken grid-stride)
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(1, (rows + TR - 1) / TR), (int64_t)g->sms * 4);
    launch_pdl(k_fill_tile<G>, dim3(grid, n), dim3(256), st, P, h);
    return;
  }
  static const int per_sm = [] {  // fill CTAs per SM at most (HELIOS_FILL_CTAS_PER_SM, default 4; 2 was best
    const char* e = getenv("HELIOS_FILL_CTAS_PER_SM");  // before the tables stayed L2-resident)
    return e ? std::max(1, std::min(atoi(e), 8)) : 4;
  }();
  const int32_t f = P.c[0].fan[h];
  if (P.c[0].fill_seg && f >= 1 && f <= 32) {  // S-lane segments, floor(32 / f) rows per warp
    const int64_t warps = (std::max<int64_t>(rows, 1) + 32 / f - 1) / (32 / f);
    const int grid = (int)std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)g->sms * per_sm);
    launch_pdl(k_fill_seg, dim3(grid, n), dim3(256), st, P, h);
    return;
  }
  const int64_t threads = std::max<int64_t>(rows, 1) * G;
  const int grid = (int)std::min<int64_t>((threads + 255) / 256, (int64_t)g->sms * per_sm);
  launch_pdl(k_fill_insert<G>, dim3(grid, n), dim3(256), st, P, h);
}

static int persistent_grid(int sms) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sample_batch, 256, 0);
    per_sm = std::max(1, std::min(per_sm, 2));
  }
  return sms * per_sm;
}

constexpr int kClusterBlock = 1024;

static cudaLaunchConfig_t cluster_cfg(int cl, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(kClusterBlock);
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// Whether a cluster of `cl` kClusterBlock-thread CTAs can be resident (16 needs the non-portable
// cluster size attribute).
static bool cluster_fits(int cl) {
  if (cl > 8 && cudaFuncSetAttribute(k_sample_cluster<kClusterBlock>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                    cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cluster_cfg(cl, nullptr, attr);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_sample_cluster<kClusterBlock>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

helios_status sample_launch_group(helios_graph* g, SampleWS* const* ws, const helios_blocks* const* outs, int n,
                                  int64_t B_max, const int32_t* fanouts, int32_t L, cudaStream_t st,
                                  const std::function<helios_status(int)>* hook) {
  int64_t maxn, lvl[HELIOS_MAX_HOPS + 1], edg[HELIOS_MAX_HOPS];
  helios_status s = sample_bounds(B_max, fanouts, L, g->V, g->E, &maxn, lvl, edg);
  if (s != HELIOS_OK) return s;
  HCHECK(n >= 1 && n <= kMaxGroup, HELIOS_E_INVALID, "group of %d batches (1..%d)", n, kMaxGroup);
  HCHECK(n == 1 || !hook, HELIOS_E_INVALID, "stage hooks need a group of one batch");
  SampleGroup P{};
  for (int b = 0; b < n; b++) {
    P.c[b] = make_ctx(g, *ws[b], fanouts, L, outs[b]);
    HCUDA(cudaMemsetAsync(ws[b]->scan_base, 0xFF, ws[b]->scan_bytes, st));
  }
  const SampleCtx& c = P.c[0];
  SampleWS& w = *ws[0];
  if (n == 1 && w.cluster && !hook) {  // the whole batch: one cluster, one launch
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = cluster_cfg(w.cluster, st, attr);
    HCUDA(cudaLaunchKernelEx(&cfg, k_sample_cluster<kClusterBlock>, c));
    return HELIOS_OK;
  }
  if (n == 1 && w.persistent && !hook) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(persistent_grid(g->sms));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HCUDA(cudaLaunchKernelEx(&cfg, k_sample_batch, c));
    return HELIOS_OK;
  }
  if (L == 0)
    k_insert_seeds<<<dim3((unsigned)std::max<int64_t>(1, (B_max + 255) / 256), n), 256, 0, st>>>(P);
  for (int h = 0; h < L; h++) {
    const int32_t f = fanouts[h];
    // persistent tile loops: a grid of at most one CTA per SM, tiles taken by ticket
    const int rt = (int)std::min<int64_t>(std::max<int64_t>(1, (lvl[h] + kScanTile - 1) / kScanTile), g->sms);
    // hop 0: enough CTAs for one seed insert per thread (the scan itself uses ceil(B/tile) tiles)
    if (h == 0) {
      const int g0 = std::max<int>(rt, (int)std::min<int64_t>((B_max + 255) / 256, g->sms));
      k_count_scan<<<dim3(g0, n), kScanBlock, 0, st>>>(P, 0);
      if (hook) {
        helios_status hs = (*hook)(0);
        if (hs != HELIOS_OK) return hs;
      }
    } else {
      launch_pdl(k_count_scan, dim3(rt, n), dim3(kScanBlock), st, P, h);
    }
    if (f < 0 || f > 16) launch_fill<32>(g, P, n, h, lvl[h], st);
    else if (f > 8) launch_fill<16>(g, P, n, h, lvl[h], st);
    else if (f > 4) launch_fill<8>(g, P, n, h, lvl[h], st);
    else launch_fill<4>(g, P, n, h, lvl[h], st);
    if (c.tile_rows[h] > 0) {
      const int TR = c.tile_rows[h];
      const int at = (int)std::min<int64_t>(std::max<int64_t>(1, (lvl[h] + TR - 1) / TR), g->sms);
      launch_pdl(k_assign_tile, dim3(at, n), dim3(kScanBlock), st, P, h);
    } else {
      const int et = (int)std::min<int64_t>(std::max<int64_t>(1, (edg[h] + kScanTile - 1) / kScanTile), g->sms);
      launch_pdl(k_dedup_assign, dim3(et, n), dim3(kScanBlock), st, P, h);
    }
    if (hook) {
      helios_status hs = (*hook)(h + 1);
      if (hs != HELIOS_OK) return hs;
    }
  }
  static const int tail_per_sm = [] {  // relabel / clear CTAs per SM at most (HELIOS_TAIL_CTAS_PER_SM, default 2)
    const char* e = getenv("HELIOS_TAIL_CTAS_PER_SM");
    return e ? std::max(1, std::min(atoi(e), 8)) : 2;
  }();
  if (L > 0) {
    const int ge = (int)std::min<int64_t>(std::max<int64_t>(1, (edg[L - 1] + 255) / 256), (int64_t)g->sms * tail_per_sm);
    launch_pdl(k_relabel, dim3(ge, n), dim3(256), st, P, L - 1);
  }
  const int gc = (int)std::min<int64_t>(std::max<int64_t>(1, (maxn + 255) / 256), (int64_t)g->sms * tail_per_sm);
  launch_pdl(k_table_clear, dim3(gc, n), dim3(256), st, P);
  HCUDA(cudaGetLastError());
  return HELIOS_OK;
}

helios_status sample_launch(helios_graph* g, SampleWS& w, int64_t B_max, const int32_t* fanouts, int32_t L,
                            const helios_blocks* out, cudaStream_t st, const std::function<helios_status(int)>* hook) {
  SampleWS* ws[1] = {&w};
  const helios_blocks* outs[1] = {out};
  return sample_launch_group(g, ws, outs, 1, B_max, fanouts, L, st, hook);
}

}  // namespace helios
