// Zero-copy random-row read throughput from pinned host memory vs allocation method / region size /
// access skew (tier layout study for the host tier).  Prints one JSON object per case.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <thread>
#include <algorithm>
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
static void fill(char* p, size_t n) {
  int T = 16; std::vector<std::thread> th;
  for (int t = 0; t < T; t++) th.emplace_back([=]{ size_t a = n / T * t, b = (t == T-1) ? n : n / T * (t+1); memset(p + a, t + 1, b - a); });
  for (auto& x : th) x.join();
}
static void print_huge() {
  FILE* f = fopen("/proc/self/smaps_rollup", "r"); char line[256];
  while (f && fgets(line, sizeof line, f)) if (strstr(line, "AnonHuge") || strstr(line, "Rss:")) fprintf(stdout, "%s", line);
  if (f) fclose(f);
}
int main(int argc, char** argv) {
  size_t GB = atoll(argv[1]); int method = atoi(argv[2]); int R = argc > 3 ? atoi(argv[3]) : 512;
  size_t bytes = GB << 30; int64_t nrows_src = bytes / R;
  char* h = nullptr;
  double t0 = 0;
  if (method == 0) { CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped)); }
  else {
    h = (char*)mmap(nullptr, bytes, PROT_READ|PROT_WRITE, MAP_PRIVATE|MAP_ANONYMOUS, -1, 0);
    madvise(h, bytes, method == 1 ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
    fill(h, bytes);
    print_huge();
    CK(cudaHostRegister(h, bytes, cudaHostRegisterMapped | (method == 3 ? cudaHostRegisterReadOnly : 0)));
  }
  char* hd; CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  int sms = 148;
  int64_t n = std::min<int64_t>(1 << 20, (1ll << 31) / R);
  int64_t* di; char* out; CK(cudaMalloc(&di, n * 8)); CK(cudaMalloc(&out, n * R));
  std::vector<int64_t> idx(n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"cudaHostAlloc", "mmap+THP+register", "mmap+noTHP+register", "mmap+THP+register(RO)"};
  for (double frac : {1.0, 0.1}) {
    uint64_t x = 88172645463325252ull;
    int64_t range = std::max<int64_t>(1, (int64_t)(nrows_src * frac));
    for (int64_t i = 0; i < n; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; idx[i] = x % range; }
    CK(cudaMemcpy(di, idx.data(), n * 8, cudaMemcpyHostToDevice));
    for (int U : {1, 4}) {
      float best = 1e9;
      for (int r = 0; r < 5; r++) {
        cudaEventRecord(a);
        if (U == 1) gather<1><<<sms * 8, 256>>>(hd, di, out, n, R); else gather<4><<<sms * 8, 256>>>(hd, di, out, n, R);
        cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
      }
      CK(cudaGetLastError());
      printf("{\"method\": \"%s\", \"region_gb\": %zu, \"R\": %d, \"range_frac\": %g, \"U\": %d, \"gbs\": %.2f, \"Mrows_s\": %.1f}\n", names[method], GB, R, frac, U, (double)n * R / best / 1e6, n / best / 1e3);
      fflush(stdout);
    }
  }
  return 0;
}
