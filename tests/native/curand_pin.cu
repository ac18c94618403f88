// tests/native/curand_pin.cu — TEST INFRASTRUCTURE ONLY (tests/test_gpu_rng.py).
//
// Library pin of reading 2 (SURVEY.md §8(c) "Library pin"): cuRAND's device
// Philox4x32-10 with curand_init(seed = key, subsequence = v, offset = (h << 34) | j) starts at
// counter {j>>2, h, lo32 v, hi32 v} (skipahead_sequence adds v to ctr.z/w, skipahead adds
// offset/4 to ctr.x/y and keeps offset&3 as the output word), so its first curand() is the
// oracle's philox_u32(key, h, v, j).  Nothing here is shared with the product or the oracle.
#include <curand_kernel.h>
#include <cstdint>

__global__ void k_curand_first(const unsigned long long* key, const unsigned long long* v, const unsigned long long* off,
                               unsigned int* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  curandStatePhilox4_32_10_t s;
  curand_init(key[i], v[i], off[i], &s);
  out[i] = curand(&s);
}

extern "C" int curand_pin_first(const unsigned long long* key, const unsigned long long* v,
                                const unsigned long long* off, unsigned int* out, int n) {
  unsigned long long *dk, *dv, *doff;
  unsigned int* dout;
  if (cudaMalloc(&dk, n * 8) || cudaMalloc(&dv, n * 8) || cudaMalloc(&doff, n * 8) || cudaMalloc(&dout, n * 4)) return 1;
  cudaMemcpy(dk, key, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(doff, off, n * 8, cudaMemcpyHostToDevice);
  k_curand_first<<<(n + 127) / 128, 128>>>(dk, dv, doff, dout, n);
  cudaError_t e = cudaMemcpy(out, dout, n * 4, cudaMemcpyDeviceToHost);
  cudaFree(dk);
  cudaFree(dv);
  cudaFree(doff);
  cudaFree(dout);
  return e == cudaSuccess ? 0 : 2;
}
