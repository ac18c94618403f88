// Host-tier read order study: zero-copy gather of the REAL per-batch host-tier slot lists of C3
// (tools/host_slots.py) from a pinned region of the host tier's size, in several issue orders and
// concurrencies.  Answers whether ordering the host reads (page locality for the host-side IOMMU
// translation cache) raises the random-row ceiling.  One JSON line per case.
// usage: hostorder <prefix> <S rows> <R bytes>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

template <int U>
__global__ void gather(const char* __restrict__ src, const int64_t* __restrict__ idx, char* __restrict__ dst, int64_t n, int R) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int nv = R / 16;
  for (int64_t b = w * U; b < n; b += nw * U) {
    for (int c = 0; c < nv; c += 32) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; u++) if (b + u < n && c + lane < nv) v[u] = ((const int4*)(src + idx[b + u] * (int64_t)R))[c + lane];
#pragma unroll
      for (int u = 0; u < U; u++) if (b + u < n && c + lane < nv) ((int4*)(dst + (b + u) * (int64_t)R))[c + lane] = v[u];
    }
  }
}

// Background load shaped like the sampler: random 4 B reads over a multi-GB HBM array plus
// random atomics, until *stop is set (run on a second stream while the gathers are timed).
__global__ void noise(const int* __restrict__ big, int64_t n, unsigned* tab, uint32_t mask, volatile int* stop) {
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  unsigned acc = 0;
  while (!*stop) {
    for (int k = 0; k < 64; k++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      acc += big[x % n];
      atomicAdd(&tab[(x >> 20) & mask], 1u);
    }
  }
  if (acc == 0xFFFFFFFFu) tab[0] = acc;
}

static std::vector<int64_t> readbin(const char* p) {
  FILE* f = fopen(p, "rb");
  if (!f) { perror(p); exit(1); }
  fseek(f, 0, SEEK_END); long n = ftell(f) / 8; fseek(f, 0, SEEK_SET);
  std::vector<int64_t> v(n);
  if (fread(v.data(), 8, n, f) != (size_t)n) exit(1);
  fclose(f);
  return v;
}

int main(int argc, char** argv) {
  char a[512], b[512];
  snprintf(a, sizeof a, "%s.slots.bin", argv[1]);
  snprintf(b, sizeof b, "%s.offs.bin", argv[1]);
  std::vector<int64_t> slots = readbin(a), offs = readbin(b);
  const int64_t S = atoll(argv[2]);
  const int R = atoi(argv[3]);
  const int nb = (int)offs.size() - 1;
  char* h = nullptr;
  CK(cudaHostAlloc(&h, (size_t)S * R, cudaHostAllocMapped));
  char* hd;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  int64_t* di; char* out;
  CK(cudaMalloc(&di, slots.size() * 8));
  CK(cudaMalloc(&out, slots.size() * (size_t)R));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int noise_ctas = argc > 4 ? atoi(argv[4]) : 0;   // background sampler-like load (CTAs of 256)
  int* big = nullptr; unsigned* tab = nullptr; int* stop = nullptr;
  const int64_t nbig = 7ll << 28;                         // 7.5 GB of int32, like C3's CSR
  cudaStream_t sn, sg;
  int least, greatest;
  CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  CK(cudaStreamCreateWithPriority(&sn, cudaStreamNonBlocking, least));
  CK(cudaStreamCreateWithPriority(&sg, cudaStreamNonBlocking, greatest));
  {  // no lazy loading: a kernel loaded while the spinning noise kernel runs could wait for it
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, gather<1>));
    CK(cudaFuncGetAttributes(&fa, gather<4>));
    CK(cudaFuncGetAttributes(&fa, gather<8>));
    CK(cudaFuncGetAttributes(&fa, noise));
  }
  if (noise_ctas) {
    CK(cudaMalloc(&big, nbig * 4));
    CK(cudaMemset(big, 1, nbig * 4));
    CK(cudaMalloc(&tab, (1 << 23) * 4));
    CK(cudaMemset(tab, 0, (1 << 23) * 4));
    CK(cudaHostAlloc(&stop, 4, cudaHostAllocMapped));
    *stop = 0;
  }
  // orders: 0 = lookup order; 1 = sorted within each batch; then W-batch windows (launch per window)
  struct Case { const char* name; int window; bool sort; };
  Case cases[] = {{"batch_lookup_order", 1, false}, {"batch_sorted", 1, true},
                  {"win6_lookup_order", 6, false}, {"win6_sorted", 6, true}};
  const int ncases = noise_ctas ? 2 : 4;
  for (int ci = 0; ci < ncases; ci++) {
    const Case& cs = cases[ci];
    std::vector<int64_t> v = slots;
    std::vector<std::pair<int64_t, int64_t>> launches;
    for (int i = 0; i < nb; i += cs.window) {
      int64_t lo = offs[i], hi = offs[std::min(nb, i + cs.window)];
      if (cs.sort) std::sort(v.begin() + lo, v.begin() + hi);
      launches.push_back({lo, hi - lo});
    }
    CK(cudaMemcpy(di, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    for (int warps : {37888, 4736, 1184, 592, 296, 148}) {   // 148 SMs x {256, 32, 8, 4, 2, 1} warps
      for (int U : {1, 4, 8}) {
        if (noise_ctas) {
          *(volatile int*)stop = 0;
          noise<<<noise_ctas, 256, 0, sn>>>(big, nbig, tab, (1 << 23) - 1, stop);
        }
        const int blocks = std::max(1, warps / 8);
        float best = 1e30f;
        for (int rep = 0; rep < 3; rep++) {
          cudaEventRecord(e0, sg);
          for (auto& l : launches) {
            if (U == 1) gather<1><<<blocks, 256, 0, sg>>>(hd, di + l.first, out, l.second, R);
            else if (U == 4) gather<4><<<blocks, 256, 0, sg>>>(hd, di + l.first, out, l.second, R);
            else gather<8><<<blocks, 256, 0, sg>>>(hd, di + l.first, out, l.second, R);
          }
          cudaEventRecord(e1, sg);
          CK(cudaEventSynchronize(e1));
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          best = std::min(best, ms);
        }
        if (noise_ctas) {
          *(volatile int*)stop = 1;
          CK(cudaStreamSynchronize(sn));
        }
        CK(cudaGetLastError());
        printf("{\"noise_ctas\": %d, \"order\": \"%s\", \"warps\": %d, \"U\": %d, \"rows\": %zu, \"Mrows_s\": %.1f, \"gbs\": %.2f, \"us_per_batch\": %.1f}\n",
               noise_ctas, cs.name, blocks * 8, U, slots.size(), slots.size() / best / 1e3, slots.size() * (double)R / best / 1e6,
               best * 1e3 / nb);
        fflush(stdout);
      }
    }
  }
  return 0;
}
