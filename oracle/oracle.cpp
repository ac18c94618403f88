// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU implementation of what the Helios mini-batch preparation
// path computes (§3.1-§3.2, arXiv 2310.00837), used to prove the CUDA path correct.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
// load this library.  It shares no code with paper_2310_00837_b200/csrc: its own Philox, its own
// hash map (std::unordered_map), its own directory encoder.  No blocking, fusion or reordering
// beyond what SURVEY.md §8(c)'s step-by-step algorithm states.
//
// Functions and the passage each follows:
//   oracle_philox4x32_10  Philox4x32-10 (Salmon et al., SC'11) — reading 2.
//                         Pinned: Random123 known-answer vectors (tests/golden/philox_kat.txt).
//   oracle_floyd          Floyd's k-subset algorithm (Bentley & Floyd, CACM 1987) on explicit draws —
//                         reading 3.  Pinned: exhaustive enumeration (every k-subset k! times).
//   oracle_sample         "2-hop random neighbor sampling" (§4.1), GPU neighbour
//                         sampling operator, readings 1,3-7.  Pinned: scipy BFS
//                         order for f=-1, closed forms (star, path, isolated), fanout bound, edge
//                         existence, dedup invariants, Monte-Carlo uniformity.
//   oracle_presample      "run an epoch of pre-sampling ... collects all vertices' hotness"
//                         (PAPER.md:212), reading 8.  Pinned: brute-force set recount.
//   oracle_cache_dir      "sort all vertices by their hotness in descending order ... hottest
//                         features to fill up the GPU cache and the second-hottest ... the CPU
//                         cache", reading 9.  Pinned: tier-order
//                         invariant, all-equal hotness -> ascending ids, caps.
//   oracle_gather         feature extraction into the "feature buffer":
//                         out[i] = row(N_L[i]) byte for byte.  Pinned: synth_feature closed form,
//                         file bytes, tiers-on == tiers-off.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstring>
#include <fcntl.h>
#include <numeric>
#include <unistd.h>
#include <unordered_map>
#include <vector>

namespace {

enum { OK = 0, E_INVALID = 1, E_RANGE = 2, E_CAPACITY = 3, E_NOMEM = 4, E_CUDA = 5, E_IO = 6 };

// ---- Philox4x32-10 --------------------------------------------------------------------------
// Round: (L0,R0,L1,R1) -> (hi(M1*L1) ^ R0 ^ k0, lo(M1*L1), hi(M0*L0) ^ R1 ^ k1, lo(M0*L0)),
// with ctr = (L0,R0,L1,R1) = (c0,c1,c2,c3); key bumped by the Weyl constants between rounds.
void philox4x32_10(const uint32_t in[4], const uint32_t k_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint32_t k0 = k_in[0], k1 = k_in[1];
  for (int round = 0; round < 10; round++) {
    if (round > 0) { k0 += W0; k1 += W1; }
    uint64_t p0 = (uint64_t)M0 * c0;
    uint64_t p1 = (uint64_t)M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// philox_u32(key, h, v, j) = Philox4x32-10(ctr = {j>>2, h, lo32(v), hi32(v)},
//                                          key = {lo32(key), hi32(key)}).word[j & 3]
uint32_t philox_u32(uint64_t key, int32_t h, int64_t v, int64_t j) {
  uint32_t ctr[4] = {(uint32_t)((uint64_t)j >> 2), (uint32_t)h, (uint32_t)(uint64_t)v, (uint32_t)((uint64_t)v >> 32)};
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  uint32_t o[4];
  philox4x32_10(ctr, k, o);
  return o[j & 3];
}

// Floyd: for j = 0..k-1, m = d-k+j+1, draw t in [0, m-1]; append m-1 if t already chosen else t.
void floyd(int64_t d, int64_t k, const uint32_t* t, int64_t* P) {
  for (int64_t j = 0; j < k; j++) {
    int64_t m = d - k + j + 1;
    int64_t tj = (int64_t)t[j];
    bool seen = false;
    for (int64_t q = 0; q < j; q++)
      if (P[q] == tj) { seen = true; break; }
    P[j] = seen ? m - 1 : tj;
  }
}

}  // namespace

extern "C" {

int oracle_abi_version(void) { return 1; }

void oracle_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }
uint32_t oracle_philox_u32(uint64_t key, int32_t h, int64_t v, int64_t j) { return philox_u32(key, h, v, j); }
void oracle_floyd(int64_t d, int64_t k, const uint32_t* t, int64_t* P) { floyd(d, k, t, P); }

// Positions (0-based, within v's adjacency) chosen for one row at hop h: k = min(d, f) (all if
// f == -1); every position in CSR order when k == d (no RNG consumed), else Floyd with
// t_j = mulhi32(philox_u32(key,h,v,j), m_j) (Lemire range reduction).  Returns k.
int64_t oracle_sample_row(uint64_t key, int32_t h, int64_t v, int64_t d, int64_t f, int64_t* P) {
  int64_t k = (f < 0) ? d : std::min(d, f);
  if (k == d) {
    for (int64_t p = 0; p < d; p++) P[p] = p;
    return k;
  }
  std::vector<uint32_t> t(k);
  for (int64_t j = 0; j < k; j++) {
    uint64_t m = (uint64_t)(d - k + j + 1);
    t[j] = (uint32_t)(((uint64_t)philox_u32(key, h, v, j) * m) >> 32);
  }
  floyd(d, k, t.data(), P);
  return k;
}

// ORACLE_SAMPLE.  Outputs:
//   nodes[n_L]                     N_0 = seeds, then new ids in first-occurrence order (h, i, j)
//   level_counts[L+1]              n_0 .. n_L
//   edge_counts[L]                 e_0 .. e_{L-1}
//   block_indptr (concatenated)    hop h: n_h + 1 int32 offsets (starts at sum_{g<h} (n_g + 1))
//   block_indices (concatenated)   hop h: e_h int32 local ids into N_{h+1} (starts at sum_{g<h} e_g)
// Returns OK, E_INVALID (duplicate seed / bad fanout), E_RANGE (seed >= V), E_CAPACITY.
int oracle_sample(int64_t V, const int64_t* indptr, const int32_t* indices, const int64_t* seeds, int64_t n_seeds,
                  const int32_t* fanouts, int32_t L, uint64_t key, int64_t nodes_cap, int64_t* nodes,
                  int64_t* level_counts, int64_t* edge_counts, int64_t bp_cap, int32_t* block_indptr,
                  int64_t bi_cap, int32_t* block_indices) {
  if (L < 0 || n_seeds < 0) return E_INVALID;
  for (int32_t h = 0; h < L; h++)
    if (fanouts[h] < -1 || fanouts[h] == 0) return E_INVALID;
  std::vector<int64_t> N;
  std::unordered_map<int64_t, int64_t> pos;
  for (int64_t i = 0; i < n_seeds; i++) {
    int64_t s = seeds[i];
    if (s < 0 || s >= V) return E_RANGE;
    if (pos.count(s)) return E_INVALID;
    pos[s] = (int64_t)N.size();
    N.push_back(s);
  }
  level_counts[0] = (int64_t)N.size();
  int64_t bp_off = 0, bi_off = 0;
  std::vector<int64_t> P;
  for (int32_t h = 0; h < L; h++) {
    int64_t n_h = (int64_t)N.size();  // frontier = ALL of N_h (reading 5: MFG blocks)
    if (bp_off + n_h + 1 > bp_cap) return E_CAPACITY;
    int32_t* bp = block_indptr + bp_off;
    int32_t* bi = block_indices + bi_off;
    int64_t e = 0;
    bp[0] = 0;
    for (int64_t i = 0; i < n_h; i++) {
      int64_t v = N[i];
      int64_t base = indptr[v], d = indptr[v + 1] - base;
      P.resize(std::max<int64_t>(d, 1));
      int64_t k = oracle_sample_row(key, h, v, d, fanouts[h], P.data());
      for (int64_t j = 0; j < k; j++) {  // slot order j = 0..k-1
        int64_t u = indices[base + P[j]];
        auto it = pos.find(u);
        int64_t lid;
        if (it == pos.end()) {
          lid = (int64_t)N.size();
          pos[u] = lid;
          N.push_back(u);
        } else {
          lid = it->second;
        }
        if (bi_off + e >= bi_cap) return E_CAPACITY;
        bi[e++] = (int32_t)lid;
      }
      bp[i + 1] = (int32_t)e;
    }
    edge_counts[h] = e;
    level_counts[h + 1] = (int64_t)N.size();
    bp_off += n_h + 1;
    bi_off += e;
  }
  if ((int64_t)N.size() > nodes_cap) return E_CAPACITY;
  std::copy(N.begin(), N.end(), nodes);
  return OK;
}

// hot[v] += number of presample batches b whose N_L(b) contains v (reading 8).  Batch b's seeds
// are seeds[offs[b] .. offs[b+1]), its key keys[b].
int oracle_presample(int64_t V, const int64_t* indptr, const int32_t* indices, const int64_t* seeds,
                     const int64_t* offs, int64_t n_batches, const uint64_t* keys, const int32_t* fanouts, int32_t L,
                     uint64_t* hot) {
  for (int64_t b = 0; b < n_batches; b++) {
    int64_t B = offs[b + 1] - offs[b];
    // capacity bound n_L <= B * prod(1 + f_h) (clamped to V), e_h <= n_h * f_h
    int64_t cap = B, ecap = 0, bcap = 0, n = B;
    for (int32_t h = 0; h < L; h++) {
      int64_t f = fanouts[h] < 0 ? V : fanouts[h];
      bcap += n + 1;
      int64_t eh = (fanouts[h] < 0) ? indptr[V] : std::min<int64_t>(n * f, indptr[V]);
      ecap += eh;
      n = std::min<int64_t>(V, n + eh);
      cap = n;
    }
    std::vector<int64_t> nodes(cap + 1), lc(L + 1), ec(L + 1);
    std::vector<int32_t> bp(bcap + 1), bi(ecap + 1);
    int rc = oracle_sample(V, indptr, indices, seeds + offs[b], B, fanouts, L, keys[b], cap + 1, nodes.data(), lc.data(),
                           ec.data(), bcap + 1, bp.data(), ecap + 1, bi.data());
    if (rc != OK) return rc;
    for (int64_t i = 0; i < lc[L]; i++) hot[nodes[i]] += 1;
  }
  return OK;
}

// Directory word: bits 63..62 tier (0 HBM, 1 HOST, 2 FILE), 61..56 owner rank,
// 55..0 slot / row.  order = stable sort of 0..V-1 by hot desc (ties: id asc).  Hot rank r:
//   r <  G*H          -> HBM(owner = r mod G, slot = r div G)
//   r <  G*H + S      -> HOST(slot = host_slot_is_id ? v : r - G*H)
//   otherwise         -> FILE(row = v)
// Also writes order[V] (the sorted vertex list) when order != NULL.
int oracle_cache_dir(int64_t V, const uint64_t* hot, int32_t G, int64_t H, int64_t S, int32_t host_slot_is_id,
                     int64_t* dir, int64_t* order_out) {
  if (G < 1 || G > 63 || H < 0 || S < 0) return E_INVALID;
  std::vector<int64_t> order(V);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return hot[a] > hot[b]; });
  for (int64_t r = 0; r < V; r++) {
    int64_t v = order[r];
    uint64_t w;
    if (r < (int64_t)G * H) {
      w = (0ull << 62) | ((uint64_t)(r % G) << 56) | (uint64_t)(r / G);
    } else if (r < (int64_t)G * H + S) {
      w = (1ull << 62) | (uint64_t)(host_slot_is_id ? v : r - (int64_t)G * H);
    } else {
      w = (2ull << 62) | (uint64_t)v;
    }
    dir[v] = (int64_t)w;
    if (order_out) order_out[r] = v;
  }
  return OK;
}

// Per-tier row counts for a node list under `dir`, as seen from rank `rank`:
// counts = {hbm_local, hbm_peer, host, file}.
void oracle_lookup_counts(const int64_t* dir, const int64_t* nodes, int64_t n, int32_t rank, int64_t* counts) {
  counts[0] = counts[1] = counts[2] = counts[3] = 0;
  for (int64_t i = 0; i < n; i++) {
    uint64_t w = (uint64_t)dir[nodes[i]];
    uint32_t tier = (uint32_t)(w >> 62), owner = (uint32_t)((w >> 56) & 63);
    if (tier == 0) counts[owner == (uint32_t)rank ? 0 : 1]++;
    else if (tier == 1) counts[2]++;
    else counts[3]++;
  }
}

// out[i] = row(nodes[i]) byte for byte, R bytes per row.  Source of row(v): the canonical host
// table (row v at table + v*R) when table != NULL and v is not FILE-tier under dir; otherwise the
// canonical feature file (pread of R bytes at header + v*stride).  Returns OK or E_IO.
int oracle_gather(const int64_t* nodes, int64_t n, int32_t R, const void* table, const char* path, int64_t header,
                  int64_t stride, const int64_t* dir, void* out) {
  int fd = -1;
  if (path && path[0]) {
    fd = open(path, O_RDONLY);
    if (fd < 0) return E_IO;
  }
  int rc = OK;
  for (int64_t i = 0; i < n; i++) {
    int64_t v = nodes[i];
    char* dst = (char*)out + i * (int64_t)R;
    bool from_file = (table == nullptr) || (dir && ((uint64_t)dir[v] >> 62) == 2);
    if (!from_file) {
      std::memcpy(dst, (const char*)table + v * (int64_t)R, R);
    } else {
      if (fd < 0) { rc = E_IO; break; }
      ssize_t got = pread(fd, dst, R, header + v * stride);
      if (got != R) { rc = E_IO; break; }
    }
  }
  if (fd >= 0) close(fd);
  return rc;
}

}  // extern "C"
