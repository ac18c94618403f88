// Step-0 link microbenchmarks: HBM copy, pinned H2D/D2H copy, zero-copy reads of
// pinned host memory (sequential and random R-byte rows), random R-byte row gather from HBM.
// Best of 10, CUDA events. Prints one JSON object.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)

__global__ void copy16(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i];
}
// one warp per row; rows picked by idx[]; R bytes per row (R % 16 == 0, R/16 <= 32*V)
template <int V>
__global__ void gather_rows(const char* __restrict__ src, const int64_t* __restrict__ idx, char* __restrict__ dst,
                            int64_t nrows, int R) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int nv = R / 16;
  for (int64_t r = w; r < nrows; r += nw) {
    const int4* s = (const int4*)(src + idx[r] * (int64_t)R);
    int4* d = (int4*)(dst + r * (int64_t)R);
    int4 v[V];
#pragma unroll
    for (int k = 0; k < V; k++) if (lane + 32 * k < nv) v[k] = s[lane + 32 * k];
#pragma unroll
    for (int k = 0; k < V; k++) if (lane + 32 * k < nv) d[lane + 32 * k] = v[k];
  }
}
static float best_ms(int reps, auto fn) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float best = 1e30f;
  for (int i = 0; i < reps; i++) { cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
  CK(cudaGetLastError()); return best;
}
int main(int argc, char** argv) {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = 4ull << 30;
  char *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 1, bytes));
  float ms = best_ms(10, [&]{ copy16<<<sms * 8, 512>>>((int4*)a, (int4*)b, bytes / 16); });
  printf("{\"sms\": %d, \"hbm_copy_gbs\": %.1f", sms, 2.0 * bytes / ms / 1e6);
  size_t hb = 8ull << 30; char* h; CK(cudaHostAlloc(&h, hb, cudaHostAllocMapped)); memset(h, 2, hb);
  ms = best_ms(5, [&]{ cudaMemcpyAsync(a, h, 2ull << 30, cudaMemcpyHostToDevice); });
  printf(", \"h2d_copy_gbs\": %.2f", (2ull << 30) / ms / 1e6);
  ms = best_ms(5, [&]{ cudaMemcpyAsync(h, a, 2ull << 30, cudaMemcpyDeviceToHost); });
  printf(", \"d2h_copy_gbs\": %.2f", (2ull << 30) / ms / 1e6);
  char* hd; CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  int Rs[3] = {400, 512, 4096};
  for (int R : Rs) {
    int64_t nrows_src = hb / R, n = std::min<int64_t>(1 << 20, (2ull << 30) / R);
    std::vector<int64_t> seq(n), rnd(n); uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < n; i++) { seq[i] = i; x ^= x << 13; x ^= x >> 7; x ^= x << 17; rnd[i] = x % nrows_src; }
    int64_t* di; CK(cudaMalloc(&di, n * 8));
    for (int mode = 0; mode < 2; mode++) {
      CK(cudaMemcpy(di, mode ? rnd.data() : seq.data(), n * 8, cudaMemcpyHostToDevice));
      for (int grid_mul : {4, 16}) {
        auto run = [&](const char* src) { if (R <= 512) gather_rows<1><<<sms * grid_mul, 256>>>(src, di, b, n, R);
                                          else gather_rows<8><<<sms * grid_mul, 256>>>(src, di, b, n, R); };
        ms = best_ms(5, [&]{ run(hd); });
        printf(", \"zc_%s_R%d_g%d_gbs\": %.2f", mode ? "rand" : "seq", R, grid_mul, (double)n * R / ms / 1e6);
      }
      int64_t* dj; CK(cudaMalloc(&dj, n * 8));
      std::vector<int64_t> r2(n); for (int64_t i = 0; i < n; i++) r2[i] = rnd[i] % ((bytes / 2) / R);
      CK(cudaMemcpy(dj, mode ? r2.data() : seq.data(), n * 8, cudaMemcpyHostToDevice));
      ms = best_ms(10, [&]{ if (R <= 512) gather_rows<1><<<sms * 16, 256>>>(a, dj, b + (bytes / 2), n, R);
                            else gather_rows<8><<<sms * 16, 256>>>(a, dj, b + bytes / 2, n, R); });
      printf(", \"hbm_gather_%s_R%d_gbs\": %.1f", mode ? "rand" : "seq", R, 2.0 * n * R / ms / 1e6);
      cudaFree(dj);
    }
    cudaFree(di);
  }
  printf("}\n");
  return 0;
}
