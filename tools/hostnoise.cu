// What slows zero-copy host-row reads down when other kernels run next to them?  Gathers the real
// C3 host-tier slot lists (tools/host_slots.py) from a pinned region of the host tier's size, alone
// and next to a background kernel of one of several access shapes (random reads over a large or a
// small HBM region, with or without atomics, streaming reads), with plain and .nc loads.
// usage: hostnoise <prefix> <S rows> <R bytes> [noise CTAs]
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <unistd.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int U, bool NC>
__global__ void gather(const char* __restrict__ src, const int64_t* __restrict__ idx, char* __restrict__ dst, int64_t n, int R) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int nv = R / 16;
  for (int64_t b = w * U; b < n; b += nw * U) {
    for (int c = 0; c < nv; c += 32) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; u++)
        if (b + u < n && c + lane < nv) {
          const int4* p = ((const int4*)(src + idx[b + u] * (int64_t)R)) + c + lane;
          v[u] = NC ? ld_nc(p) : *p;
        }
#pragma unroll
      for (int u = 0; u < U; u++) if (b + u < n && c + lane < nv) ((int4*)(dst + (b + u) * (int64_t)R))[c + lane] = v[u];
    }
  }
}

// Ticketed variant: UH rows per atomicAdd ticket (the library's host-row kernel schedule).
template <int U>
__global__ void gather_dyn(const char* __restrict__ src, const int64_t* __restrict__ idx, char* __restrict__ dst, int64_t n,
                           int R, unsigned long long* ticket) {
  int lane = threadIdx.x & 31;
  int nv = R / 16;
  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, (unsigned long long)U);
    const int64_t b = (int64_t)__shfl_sync(0xFFFFFFFFu, t, 0);
    if (b >= n) break;
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) if (b + u < n && lane < nv) v[u] = ((const int4*)(src + idx[b + u] * (int64_t)R))[lane];
#pragma unroll
    for (int u = 0; u < U; u++) if (b + u < n && lane < nv) ((int4*)(dst + (b + u) * (int64_t)R))[lane] = v[u];
  }
}

// One short burst of random reads (run between batches: evicts TLB / L2 state like the sampler).
__global__ void burst(const int* __restrict__ big, int64_t n, unsigned* sink, int iters) {
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  unsigned acc = 0;
  for (int k = 0; k < iters; k++) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    acc += big[x % n];
  }
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

// Compute-only spin for `ns` nanoseconds (between batches: SM activity without memory traffic).
__global__ void spin(int64_t ns, unsigned* sink) {
  const uint64_t t0 = clock64();
  uint64_t x = threadIdx.x;
  while ((int64_t)(clock64() - t0) < ns * 2) x = x * 6364136223846793005ull + 1;  // ~2 GHz
  if (x == 42) sink[0] = (unsigned)x;
}
// Streaming writes of `n` ints (between batches: write-only HBM traffic).
__global__ void wburst(int* big, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) big[i] = (int)i;
}

// mode 1: random 4 B reads over 7.5 GB + random atomics over 32 MB
// mode 2: random 4 B reads over 7.5 GB only
// mode 3: random 4 B reads over 64 MB only (L2-resident, few TLB entries)
// mode 4: random atomics over 32 MB only
// mode 5: streaming 16 B reads over 7.5 GB
// mode 6: random 4 B reads over 7.5 GB, one lane per warp (light, latency-bound)
__global__ void noise(const int* __restrict__ big, int64_t n, unsigned* tab, uint32_t mask, volatile int* stop, int mode) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  uint64_t x = 0x9E3779B97F4A7C15ull * (tid + 1);
  unsigned acc = 0;
  int64_t pos = tid * 4;
  while (!*stop) {
    for (int k = 0; k < 64; k++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      if (mode == 1) { acc += big[x % n]; atomicAdd(&tab[(x >> 20) & mask], 1u); }
      else if (mode == 2) acc += big[x % n];
      else if (mode == 3) acc += big[x & ((16 << 20) - 1)];
      else if (mode == 4) atomicAdd(&tab[(x >> 20) & mask], 1u);
      else if (mode == 5) { int4 v = *(const int4*)(big + pos); acc += v.x ^ v.w; pos += nt * 4; if (pos + 4 > n) pos = tid * 4; }
      else if (mode == 6) { if ((threadIdx.x & 31) == 0) acc += big[x % n]; }
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
  const int nctas = argc > 4 ? atoi(argv[4]) : 148;
  const int nb = (int)offs.size() - 1;
  cudaFuncAttributes fa;  // no lazy loading next to the spinning noise kernel
  CK(cudaFuncGetAttributes(&fa, gather<8, false>));
  CK(cudaFuncGetAttributes(&fa, gather<8, true>));
  CK(cudaFuncGetAttributes(&fa, noise));
  char* h = nullptr;
  CK(cudaHostAlloc(&h, (size_t)S * R, cudaHostAllocMapped));
  char* hd;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  int64_t* di; char* out;
  CK(cudaMalloc(&di, slots.size() * 8));
  CK(cudaMalloc(&out, slots.size() * (size_t)R));
  CK(cudaMemcpy(di, slots.data(), slots.size() * 8, cudaMemcpyHostToDevice));
  const int64_t nbig = 7ll << 28;
  int* big; unsigned* tab; int* stop;
  CK(cudaMalloc(&big, nbig * 4));
  CK(cudaMemset(big, 1, nbig * 4));
  CK(cudaMalloc(&tab, (1 << 23) * 4));
  CK(cudaMemset(tab, 0, (1 << 23) * 4));
  CK(cudaMalloc(&stop, 4));   // device flag: polling a host flag would itself load the PCIe path
  int* h_one; int* h_zero;
  CK(cudaHostAlloc(&h_one, 4, 0)); CK(cudaHostAlloc(&h_zero, 4, 0));
  *h_one = 1; *h_zero = 0;
  cudaStream_t sn, sg, sc;
  CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  int least, greatest;
  CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  CK(cudaStreamCreateWithPriority(&sn, cudaStreamNonBlocking, least));
  CK(cudaStreamCreateWithPriority(&sg, cudaStreamNonBlocking, greatest));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  unsigned long long* tickets;
  CK(cudaMalloc(&tickets, nb * 8 * 8));
  CK(cudaFuncGetAttributes(&fa, gather_dyn<8>));
  CK(cudaFuncGetAttributes(&fa, burst));
  CK(cudaFuncGetAttributes(&fa, spin));
  CK(cudaFuncGetAttributes(&fa, wburst));
  // cases: {noise mode, noise CTAs (0 = none), between-batch burst (0 none, 1 over 7.5 GB, 2 over 64 MB)}
  struct Case { const char* name; int mode, ctas, burst_kind; };
  Case cases[] = {{"none", 0, 0, 0}, {"concurrent rand7.5GB x148", 2, 148, 0}, {"concurrent rand7.5GB x16", 2, 16, 0},
                  {"concurrent stream7.5GB x148", 5, 148, 0}, {"burst rand7.5GB between batches", 0, 0, 1},
                  {"burst rand64MB between batches", 0, 0, 2}, {"spin 20us between batches", 0, 0, 3},
                  {"write 64MB between batches", 0, 0, 4}, {"host sleep 50us between batches", 0, 0, 5}};
  for (const Case& cs : cases) {
    for (int dyn = 0; dyn < 2; dyn++) {
      if (cs.mode) {
        CK(cudaMemcpyAsync(stop, h_zero, 4, cudaMemcpyHostToDevice, sc));
        CK(cudaStreamSynchronize(sc));
        noise<<<cs.ctas, 256, 0, sn>>>(big, nbig, tab, (1 << 23) - 1, stop, cs.mode);
      }
      float best = 1e30f;
      for (int rep = 0; rep < 3; rep++) {
        CK(cudaMemsetAsync(tickets, 0, nb * 8 * 8, sg));
        float tot = 0;
        for (int i = 0; i < nb; i++) {
          if (cs.burst_kind == 1 || cs.burst_kind == 2)
            burst<<<148 * 4, 256, 0, sg>>>(big, cs.burst_kind == 1 ? nbig : (16 << 20), tab, 32);
          else if (cs.burst_kind == 3) spin<<<148 * 4, 256, 0, sg>>>(20000, tab);
          else if (cs.burst_kind == 4) wburst<<<148 * 4, 256, 0, sg>>>(big, 16 << 20);
          else if (cs.burst_kind == 5) usleep(50);
          cudaEventRecord(e0, sg);
          if (dyn) gather_dyn<8><<<148, 256, 0, sg>>>(hd, di + offs[i], out, offs[i + 1] - offs[i], R, tickets + 8 * i);
          else gather<8, false><<<148, 256, 0, sg>>>(hd, di + offs[i], out, offs[i + 1] - offs[i], R);
          cudaEventRecord(e1, sg);
          CK(cudaEventSynchronize(e1));
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          tot += ms;
        }
        best = std::min(best, tot);
      }
      if (cs.mode) {
        CK(cudaMemcpyAsync(stop, h_one, 4, cudaMemcpyHostToDevice, sc));
        CK(cudaStreamSynchronize(sn));
      }
      CK(cudaGetLastError());
      printf("{\"case\": \"%s\", \"tickets\": %d, \"warps\": 1184, \"Mrows_s\": %.1f, \"us_per_batch\": %.1f}\n",
             cs.name, dyn, slots.size() / best / 1e3, best * 1e3 / nb);
      fflush(stdout);
    }
  }
  return 0;
}
