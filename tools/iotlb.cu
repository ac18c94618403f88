// Host-side translation locality of zero-copy reads: random 512 B rows from a pinned region of the
// C3 host tier's size, (a) uniformly within windows of W GB, (b) in clusters of K rows that share
// one 4 KB page / one 2 MB page.  Fresh rows every launch (no L2 reuse across launches).
// usage: iotlb <region GB>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Row j of launch `seed`: cluster c = j / K picks a random unit of `unit_rows` rows inside the window,
// member j % K a random row inside that unit (unit_rows = 1: plain uniform rows).
__global__ void gen(int64_t* idx, int64_t n, int64_t window_rows, int64_t unit_rows, int K, uint64_t seed) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t units = window_rows / unit_rows;
    const int64_t u = (int64_t)__umul64hi(mix(seed + 0x9E3779B97F4A7C15ull * (uint64_t)(j / K + 1)), (uint64_t)units);
    const int64_t r = unit_rows > 1 ? (int64_t)__umul64hi(mix(seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(j + 1))), (uint64_t)unit_rows) : 0;
    idx[j] = u * unit_rows + r;
  }
}

__global__ void gather(const char* __restrict__ src, const int64_t* __restrict__ idx, char* __restrict__ dst, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w * 8; b < n; b += nw * 8) {
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) if (b + u < n) v[u] = ((const int4*)(src + idx[b + u] * 512))[lane];
#pragma unroll
    for (int u = 0; u < 8; u++) if (b + u < n) ((int4*)(dst + (b + u) * 512))[lane] = v[u];
  }
}

int main(int argc, char** argv) {
  const int64_t gb = argc > 1 ? atoll(argv[1]) : 51;
  const int64_t rows = (gb << 30) / 512;
  char* h;
  CK(cudaHostAlloc(&h, (size_t)rows * 512, cudaHostAllocMapped));
  char* hd;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  const int64_t n = 1 << 18;
  int64_t* idx;
  char* out;
  CK(cudaMalloc(&idx, n * 8));
  CK(cudaMalloc(&out, n * 512));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case { const char* name; double window_gb; int64_t unit_rows; int K; };
  Case cases[] = {{"uniform", 51, 1, 1},      {"uniform", 32, 1, 1},      {"uniform", 16, 1, 1},
                  {"uniform", 8, 1, 1},       {"uniform", 4, 1, 1},       {"uniform", 2, 1, 1},
                  {"4KB-page clusters", 51, 8, 2},   {"4KB-page clusters", 51, 8, 4},   {"4KB-page clusters", 51, 8, 8},
                  {"2MB-page clusters", 51, 4096, 2}, {"2MB-page clusters", 51, 4096, 4}, {"2MB-page clusters", 51, 4096, 8},
                  {"2MB-page clusters", 51, 4096, 32}, {"64KB-page clusters", 51, 128, 4}, {"64KB-page clusters", 51, 128, 16}};
  uint64_t seed = 1;
  for (const Case& c : cases) {
    const int64_t wrows = std::min<int64_t>(rows, (int64_t)(c.window_gb * (1ll << 30) / 512));
    float tot = 0;
    const int reps = 8;
    for (int r = 0; r < reps; r++) {
      gen<<<148 * 4, 256>>>(idx, n, wrows, c.unit_rows, c.K, seed++ * 0x2545F4914F6CDD1Dull);
      cudaEventRecord(e0);
      gather<<<148, 256>>>(hd, idx, out, n);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    printf("{\"case\": \"%s\", \"window_gb\": %.0f, \"K\": %d, \"Mrows_s\": %.1f, \"gbs\": %.2f}\n", c.name, c.window_gb, c.K,
           n * reps / tot / 1e3, n * reps * 512.0 / tot / 1e6);
    fflush(stdout);
  }
  return 0;
}
