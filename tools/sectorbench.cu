// Random-sector ceiling of HBM3e for the sampler's access shape: every thread issues independent
// uniformly random 4 B loads (one 32 B sector each) over an array of a given size, with 1..8 loads
// in flight per thread.  Prints G sectors/s per (array size, loads in flight).  usage: sectorbench
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); return 1;} }while(0)

template <int ILP>
__global__ void rnd(const int* __restrict__ a, int64_t n, int iters, unsigned* sink) {
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + 1);
  unsigned acc = 0;
  for (int it = 0; it < iters; it++) {
    int64_t idx[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      idx[k] = (int64_t)__umul64hi(x, (uint64_t)n);
    }
#pragma unroll
    for (int k = 0; k < ILP; k++) acc += __ldcg(a + idx[k]);
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  const int64_t maxn = 7ll << 28;  // 7.5 GB of int32
  int* a;
  unsigned* sink;
  CK(cudaMalloc(&a, maxn * 4));
  CK(cudaMemset(a, 1, maxn * 4));
  CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int64_t mb : {64ll, 256ll, 1024ll, 7168ll}) {
    const int64_t n = mb << 18;
    for (int ilp : {1, 2, 4, 8}) {
      const int blocks = 148 * 8, iters = 64 / ilp;
      float best = 1e30f;
      for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        if (ilp == 1) rnd<1><<<blocks, 256>>>(a, n, iters, sink);
        else if (ilp == 2) rnd<2><<<blocks, 256>>>(a, n, iters, sink);
        else if (ilp == 4) rnd<4><<<blocks, 256>>>(a, n, iters, sink);
        else rnd<8><<<blocks, 256>>>(a, n, iters, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      const double loads = (double)blocks * 256 * iters * ilp;
      printf("{\"array_mb\": %lld, \"ilp\": %d, \"Gsectors_s\": %.2f, \"GBs_at_32B\": %.1f}\n", (long long)mb, ilp,
             loads / best / 1e6, loads * 32 / best / 1e6);
    }
  }
  return 0;
}
