// Random zero-copy row reads from host memory mapped through the CUDA VMM API (cuMemCreate with a
// HOST_NUMA location, mapped at the allocation granularity) vs cudaHostAlloc.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <thread>
#include <algorithm>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); exit(1);} }while(0)
#define CU(x) do{CUresult r=(x); if(r!=CUDA_SUCCESS){const char* s; cuGetErrorString(r,&s); fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,s); exit(1);} }while(0)

__global__ void gather(const char* __restrict__ src, const int64_t* __restrict__ idx, char* __restrict__ dst, int64_t n, int R) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int nv = R / 16;
  for (int64_t b = w; b < n; b += nw)
    for (int c = lane; c < nv; c += 32) ((int4*)(dst + b * (int64_t)R))[c] = ((const int4*)(src + idx[b] * (int64_t)R))[c];
}
int main(int argc, char** argv) {
  size_t GB = atoll(argv[1]); int R = argc > 2 ? atoi(argv[2]) : 512;
  size_t bytes = GB << 30;
  CK(cudaFree(0));
  CUdevice dev; CU(cuDeviceGet(&dev, 0));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = 0;
  size_t gran = 0, rgran = 0;
  CU(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CU(cuMemGetAllocationGranularity(&rgran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("granularity min %zu recommended %zu\n", gran, rgran);
  size_t g = std::max(gran, rgran);
  bytes = (bytes + g - 1) / g * g;
  CUmemGenericAllocationHandle h;
  CU(cuMemCreate(&h, bytes, &prop, 0));
  CUdeviceptr va;
  CU(cuMemAddressReserve(&va, bytes, g, 0, 0));
  CU(cuMemMap(va, bytes, 0, h, 0));
  CUmemAccessDesc acc[2] = {};
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc[0].location.id = 0; acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA; acc[1].location.id = 0; acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUresult r2 = cuMemSetAccess(va, bytes, acc, 2);
  bool host_ok = (r2 == CUDA_SUCCESS);
  if (!host_ok) { printf("host access not granted (%d); device only\n", (int)r2); CU(cuMemSetAccess(va, bytes, acc, 1)); }
  char* p = (char*)va;
  if (host_ok) {  // CPU writes through the same VA
    int T = 16; std::vector<std::thread> th;
    for (int t = 0; t < T; t++) th.emplace_back([=]{ size_t a = bytes / T * t, b = (t == T - 1) ? bytes : bytes / T * (t + 1); memset(p + a, t + 1, b - a); });
    for (auto& x : th) x.join();
    printf("cpu fill ok\n");
  } else {
    CK(cudaMemset(p, 7, bytes));
  }
  int64_t nrows = bytes / R, n = std::min<int64_t>(1 << 20, (1ll << 31) / R);
  std::vector<int64_t> idx(n); uint64_t x = 88172645463325252ull;
  int64_t* di; char* out; CK(cudaMalloc(&di, n * 8)); CK(cudaMalloc(&out, n * R));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (double frac : {1.0, 0.1}) {
    int64_t range = (int64_t)(nrows * frac);
    for (int64_t i = 0; i < n; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; idx[i] = x % range; }
    CK(cudaMemcpy(di, idx.data(), n * 8, cudaMemcpyHostToDevice));
    float best = 1e9;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(a); gather<<<148 * 8, 256>>>(p, di, out, n, R); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    if (host_ok && frac == 1.0) {  // verify a row from the CPU view
      std::vector<char> row(R); CK(cudaMemcpy(row.data(), out, R, cudaMemcpyDeviceToHost));
      printf("row check %s\n", memcmp(row.data(), p + idx[0] * R, R) == 0 ? "ok" : "MISMATCH");
    }
    printf("{\"method\": \"vmm-host-numa\", \"region_gb\": %zu, \"R\": %d, \"range_frac\": %g, \"gbs\": %.2f, \"Mrows_s\": %.1f}\n",
           GB, R, frac, (double)n * R / best / 1e6, n / best / 1e3);
  }
  return 0;
}
