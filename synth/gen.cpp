// synth/gen.cpp — seeded synthetic INPUT generators shared by the oracle and the CUDA path.
//
// This module holds none of the method's arithmetic (no Philox, no sampling, no dedup, no cache
// policy): it only manufactures inputs — a power-law CSR graph, canonical feature rows, the
// training set, per-epoch seed batches and 64-bit batch keys.  Both sides receive its outputs as
// plain arrays.  Recipe: DESIGN.md "Input recipe".
//
// Random source: SplitMix64's finaliser mix64 (Steele et al., 2014), used as a counter-based hash
// u(seed, stream, i) = mix64(mix64(seed ^ stream) + i).  Sampling itself uses Philox4x32-10,
// which deliberately does not appear here.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <functional>
#include <thread>
#include <unistd.h>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t urand(uint64_t seed, uint64_t stream, uint64_t i) { return mix64(mix64(seed ^ stream) + i); }

int g_threads = 0;
int nthreads() {
  if (g_threads > 0) return g_threads;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

// Static-chunked parallel for over [0, n).
void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& body) {
  int T = nthreads();
  if (n < 4096 || T == 1) { body(0, n); return; }
  std::vector<std::thread> th;
  int64_t chunk = (n + T - 1) / T;
  for (int t = 0; t < T; t++) {
    int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back(body, lo, hi);
  }
  for (auto& x : th) x.join();
}
// Dynamic (work-stealing by atomic counter) parallel for, for skewed per-row work.
void parallel_for_dyn(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)>& body) {
  int T = nthreads();
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t lo = next.fetch_add(grain);
      if (lo >= n) break;
      body(lo, std::min(n, lo + grain));
    }
  };
  if (T == 1) { worker(); return; }
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++) th.emplace_back(worker);
  for (auto& x : th) x.join();
}

// ---- R-MAT-marginal (Kronecker) vertex labelling -------------------------------------------
// Vertex v in [0,V) sits at Kronecker position x = perm(v) in [0, 2^scale); its weight is the
// R-MAT marginal  w(x) = p1^popcount(x) * (1-p1)^(scale - popcount(x))  (Graph500's
// a,b,c,d = .57,.19,.19,.05 gives p1 = c+d = .24; larger p1 = less skew).  Row (out-degree) and
// column (destination) marginals coincide (b = c).
// perm is a bijection of [0, 2^scale) (xor-shift / odd-multiply rounds) that scatters hubs.
struct Perm {
  int scale;
  uint64_t mask, c0, m1, m1inv, m2, m2inv;
  int s1, s2;
  static uint64_t inv_odd(uint64_t a) {  // a^-1 mod 2^64 (Newton)
    uint64_t x = a;
    for (int i = 0; i < 6; i++) x *= 2 - a * x;
    return x;
  }
  Perm(int sc, uint64_t seed) : scale(sc) {
    mask = (sc >= 64) ? ~0ull : ((1ull << sc) - 1);
    c0 = urand(seed, 0x5045524Dull, 0) & mask;
    m1 = urand(seed, 0x5045524Dull, 1) | 1;
    m2 = urand(seed, 0x5045524Dull, 2) | 1;
    m1inv = inv_odd(m1);
    m2inv = inv_odd(m2);
    s1 = std::max(1, sc / 2 + 1);
    s2 = std::max(1, sc / 3 + 1);
  }
  static uint64_t xs_inv(uint64_t y, int s, uint64_t mask) {
    uint64_t x = y;
    for (int i = 0; i < 64 / s + 1; i++) x = y ^ (x >> s);
    return x & mask;
  }
  uint64_t fwd(uint64_t x) const {
    x ^= c0;
    x = (x * m1) & mask;
    x ^= x >> s1;
    x = (x * m2) & mask;
    x ^= x >> s2;
    return x & mask;
  }
  uint64_t inv(uint64_t y) const {
    uint64_t x = xs_inv(y, s2, mask);
    x = (x * m2inv) & mask;
    x = xs_inv(x, s1, mask);
    x = (x * m1inv) & mask;
    return x ^ c0;
  }
};


inline int scale_of(int64_t V) {
  int s = 1;
  while ((1ll << s) < V) s++;
  return s;
}

}  // namespace

extern "C" {

void synth_set_threads(int t) { g_threads = t; }
int synth_get_threads(void) { return nthreads(); }
uint64_t synth_mix64(uint64_t x) { return mix64(x); }

// Bijection self-check helpers (tests): forward / inverse of the vertex permutation.
uint64_t synth_perm_fwd(int scale, uint64_t seed, uint64_t x) { return Perm(scale, seed).fwd(x); }
uint64_t synth_perm_inv(int scale, uint64_t seed, uint64_t y) { return Perm(scale, seed).inv(y); }

// Phase 1: target out-degree of every vertex, deg[v] = floor(E * w(perm v) / W + U_v).
// Returns sum of target degrees (the provisional edge count before row dedup).
int64_t synth_graph_degrees(int64_t V, int64_t E_target, uint64_t seed, double p1, int64_t* deg) {
  if (V < 2 || E_target < 0) return -1;
  int scale = scale_of(V);
  Perm P(scale, seed);
  // W = sum_v w(perm v): weights depend only on popcount -> histogram.
  std::vector<std::vector<int64_t>> hist(nthreads(), std::vector<int64_t>(65, 0));
  std::atomic<int> tid{0};
  parallel_for(V, [&](int64_t lo, int64_t hi) {
    int t = tid.fetch_add(1);
    auto& h = hist[t % hist.size()];
    for (int64_t v = lo; v < hi; v++) h[__builtin_popcountll(P.fwd((uint64_t)v))]++;
  });
  std::vector<double> wpop(65);
  for (int k = 0; k <= scale; k++) wpop[k] = std::pow(p1, k) * std::pow(1.0 - p1, scale - k);
  double W = 0;
  for (auto& h : hist)
    for (int k = 0; k <= scale; k++) W += (double)h[k] * wpop[k];
  std::atomic<int64_t> total{0};
  parallel_for(V, [&](int64_t lo, int64_t hi) {
    int64_t s = 0;
    for (int64_t v = lo; v < hi; v++) {
      double ex = (double)E_target * wpop[__builtin_popcountll(P.fwd((uint64_t)v))] / W;
      double u = (double)(urand(seed, 0x444547ull, (uint64_t)v) >> 11) * 0x1.0p-53;
      int64_t d = (int64_t)std::floor(ex + u);
      deg[v] = d;
      s += d;
    }
    total += s;
  });
  return total.load();
}

// Phase 2: draw each row's destinations from the Kronecker column marginal, then sort, drop
// duplicates and self-loops.  prov_indptr = exclusive scan of deg (V+1 entries, caller-computed);
// prov (int32[prov_indptr[V]]) is scratch; final_len[v] receives the deduplicated row length and
// rows are left sorted at the front of their provisional slice.
int synth_graph_fill(int64_t V, uint64_t seed, double p1, const int64_t* prov_indptr, int32_t* prov, int64_t* final_len) {
  int scale = scale_of(V);
  const uint32_t p1q16 = (uint32_t)std::lround(p1 * 65536.0);  // P(bit = 1) per Kronecker level
  Perm P(scale, seed);
  parallel_for_dyn(V, 256, [&](int64_t lo, int64_t hi) {
    for (int64_t v = lo; v < hi; v++) {
      int64_t b = prov_indptr[v], d = prov_indptr[v + 1] - b;
      uint64_t ctr = 0;
      for (int64_t j = 0; j < d; j++) {
        for (;;) {  // rejection: positions >= V are not vertices
          uint64_t x = 0;
          for (int l = 0; l < scale; l += 4) {
            uint64_t r = urand(seed ^ ((uint64_t)v << 1), 0x445354ull, ctr++);
            for (int q = 0; q < 4 && l + q < scale; q++)
              if ((uint32_t)((r >> (16 * q)) & 0xFFFF) < p1q16) x |= 1ull << (l + q);
          }
          uint64_t u = P.inv(x);
          if ((int64_t)u < V) { prov[b + j] = (int32_t)u; break; }
        }
      }
      int32_t* row = prov + b;
      std::sort(row, row + d);
      int64_t w = 0;
      for (int64_t j = 0; j < d; j++) {
        if (row[j] == (int32_t)v) continue;           // self-loop
        if (w > 0 && row[w - 1] == row[j]) continue;  // duplicate (src,dst)
        row[w++] = row[j];
      }
      final_len[v] = w;
    }
  });
  return 0;
}

// Phase 3: compact rows into the final CSR (indptr = exclusive scan of final_len, caller-computed).
int synth_graph_compact(int64_t V, const int64_t* prov_indptr, const int32_t* prov, const int64_t* indptr,
                        int32_t* indices) {
  parallel_for_dyn(V, 4096, [&](int64_t lo, int64_t hi) {
    for (int64_t v = lo; v < hi; v++)
      std::memcpy(indices + indptr[v], prov + prov_indptr[v], sizeof(int32_t) * (indptr[v + 1] - indptr[v]));
  });
  return 0;
}

// Canonical feature rows (SPEC.md:61-69 synth_feature, made exact):
//   row(v)[j] = (float)(mix64(v*dim + j) >> 40) * 2^-24   — exact in fp32, in [0,1).
void synth_features(int64_t v0, int64_t n, int32_t dim, float* out) {
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
      uint64_t base = (uint64_t)(v0 + i) * (uint64_t)dim;
      float* r = out + i * (int64_t)dim;
      for (int32_t j = 0; j < dim; j++) r[j] = (float)(mix64(base + (uint64_t)j) >> 40) * 0x1.0p-24f;
    }
  });
}

// Gathered variant: out[i] = row(ids[i]) (used to build tier contents / test expectations without
// materialising the whole table).
void synth_features_at(const int64_t* ids, int64_t n, int32_t dim, float* out) {
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
      uint64_t base = (uint64_t)ids[i] * (uint64_t)dim;
      float* r = out + i * (int64_t)dim;
      for (int32_t j = 0; j < dim; j++) r[j] = (float)(mix64(base + (uint64_t)j) >> 40) * 0x1.0p-24f;
    }
  });
}

// Feature file: `header_bytes` of header ("HLSF" magic, version, V, dim, stride), then row v at
// header_bytes + v*stride, padded with zeros to stride (PAPER.md:205 fn: 512 B).
// Rows [v0, v0+n) only when n >= 0 (n < 0: all V).  Returns 0 or -errno.
int synth_write_feature_file(const char* path, int64_t V, int32_t dim, int64_t header_bytes, int64_t stride) {
  int64_t R = (int64_t)dim * 4;
  if (stride < R || header_bytes < 64) return -22;
  int fd = open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
  if (fd < 0) return -1;
  std::vector<char> hdr(header_bytes, 0);
  std::memcpy(hdr.data(), "HLSF", 4);
  uint32_t ver = 1;
  std::memcpy(hdr.data() + 4, &ver, 4);
  std::memcpy(hdr.data() + 8, &V, 8);
  std::memcpy(hdr.data() + 16, &dim, 4);
  std::memcpy(hdr.data() + 24, &stride, 8);
  if (pwrite(fd, hdr.data(), header_bytes, 0) != header_bytes) { close(fd); return -5; }
  if (ftruncate(fd, header_bytes + V * stride) != 0) { close(fd); return -5; }
  std::atomic<int> err{0};
  parallel_for_dyn(V, 8192, [&](int64_t lo, int64_t hi) {
    std::vector<char> buf((hi - lo) * stride, 0);
    for (int64_t v = lo; v < hi; v++) {
      float* r = (float*)(buf.data() + (v - lo) * stride);
      uint64_t base = (uint64_t)v * (uint64_t)dim;
      for (int32_t j = 0; j < dim; j++) r[j] = (float)(mix64(base + (uint64_t)j) >> 40) * 0x1.0p-24f;
    }
    int64_t off = header_bytes + lo * stride, len = (hi - lo) * stride, done = 0;
    while (done < len) {
      ssize_t w = pwrite(fd, buf.data() + done, len - done, off + done);
      if (w <= 0) { err = 1; return; }
      done += w;
    }
  });
  fsync(fd);
  close(fd);
  return err ? -5 : 0;
}

// Training set: 1% of vertices, uniform: { v : mix64(seed ^ 0x7472 ^ v) % 100 < pct }.
// out may be NULL (count only).  Returns the count, ascending ids.
int64_t synth_train_set(int64_t V, uint64_t seed, int32_t pct, int64_t* out) {
  int64_t c = 0;
  for (int64_t v = 0; v < V; v++)
    if (pct >= 100 || (int64_t)(mix64(seed ^ 0x7472ull ^ (uint64_t)v) % 100) < pct) {
      if (out) out[c] = v;
      c++;
    }
  return c;
}

// Epoch order: the train set sorted by (mix64(seed ^ mix64(epoch) ^ t), t); batch b is chunk b.
void synth_epoch_order(const int64_t* train, int64_t n, uint64_t seed, int64_t epoch, int64_t* out) {
  std::vector<std::pair<uint64_t, int64_t>> k(n);
  uint64_t e = mix64((uint64_t)epoch);
  for (int64_t i = 0; i < n; i++) k[i] = {mix64(seed ^ e ^ (uint64_t)train[i]), train[i]};
  std::sort(k.begin(), k.end());
  for (int64_t i = 0; i < n; i++) out[i] = k[i].second;
}

// Batch keys: key_b = mix64(global_seed ^ mix64((epoch << 32) | b)).
// Presample keys use ~global_seed and epoch 0.
uint64_t synth_batch_key(uint64_t global_seed, int64_t epoch, int64_t b) {
  return mix64(global_seed ^ mix64(((uint64_t)epoch << 32) | (uint64_t)b));
}

}  // extern "C"
