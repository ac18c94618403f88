// green.cu — SM partition for the IO operators through a CUDA green context.
//
// The paper confines its GPU-initiated IO operators to a fraction of the GPU: the operators' SM
// usage is capped by their grid size and by MPS, and ~30 % of the SMs (32 IO blocks) suffice for
// full IO bandwidth (PAPER.md:244 §3.3, :352-357 §4).  On Blackwell the in-process analog of an MPS
// SM cap is a green context: cuDevSmResourceSplitByCount carves `io_sms` SMs out of the device,
// cuGreenCtxCreate provisions them, and a stream created in that green context runs the IO kernel
// (k_io / k_io_sync) on those SMs only.  Everything else (sampling, lookup, gather) stays on the
// primary context and the whole GPU; the two sides synchronise through ordinary CUDA events.
// The driver entry points are resolved at run time (cudaGetDriverEntryPointByVersion), so the
// library does not link libcuda directly.
#include <cuda.h>

#include "internal.cuh"

namespace helios {

namespace {
using PFN_getres = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using PFN_split = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
using PFN_gendesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
using PFN_gcreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
using PFN_gdestroy = CUresult (*)(CUgreenCtx);
using PFN_gstream = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);

template <typename F>
helios_status entry(const char* sym, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  HCUDA(cudaGetDriverEntryPointByVersion(sym, &p, CUDART_VERSION, cudaEnableDefault, &q));
  HCHECK(q == cudaDriverEntryPointSuccess && p, HELIOS_E_CUDA, "driver entry point %s unavailable", sym);
  *fn = reinterpret_cast<F>(p);
  return HELIOS_OK;
}
}  // namespace

helios_status green_io_start(helios_cache* c, int device, int io_sms, int priority) {
  PFN_getres getres;
  PFN_split split;
  PFN_gendesc gendesc;
  PFN_gcreate gcreate;
  PFN_gstream gstream;
  helios_status s;
  if ((s = entry("cuDeviceGetDevResource", &getres)) != HELIOS_OK) return s;
  if ((s = entry("cuDevSmResourceSplitByCount", &split)) != HELIOS_OK) return s;
  if ((s = entry("cuDevResourceGenerateDesc", &gendesc)) != HELIOS_OK) return s;
  if ((s = entry("cuGreenCtxCreate", &gcreate)) != HELIOS_OK) return s;
  if ((s = entry("cuGreenCtxStreamCreate", &gstream)) != HELIOS_OK) return s;
  CUdevResource all{}, part{}, rest{};
  CUresult r = getres((CUdevice)device, &all, CU_DEV_RESOURCE_TYPE_SM);
  HCHECK(r == CUDA_SUCCESS, HELIOS_E_CUDA, "cuDeviceGetDevResource: %d", (int)r);
  unsigned n = 1;
  r = split(&part, &n, &all, &rest, 0, (unsigned)io_sms);
  HCHECK(r == CUDA_SUCCESS && n == 1, HELIOS_E_INVALID, "cannot split %d SMs off the device for IO (CUresult %d)",
         io_sms, (int)r);
  CUdevResourceDesc desc = nullptr;
  r = gendesc(&desc, &part, 1);
  HCHECK(r == CUDA_SUCCESS, HELIOS_E_CUDA, "cuDevResourceGenerateDesc: %d", (int)r);
  CUgreenCtx g = nullptr;
  r = gcreate(&g, desc, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM);
  HCHECK(r == CUDA_SUCCESS, HELIOS_E_CUDA, "cuGreenCtxCreate: %d", (int)r);
  c->green = g;
  c->green_sms = (int)part.sm.smCount;
  CUstream st = nullptr;
  r = gstream(&st, g, CU_STREAM_NON_BLOCKING, priority);
  HCHECK(r == CUDA_SUCCESS, HELIOS_E_CUDA, "cuGreenCtxStreamCreate: %d", (int)r);
  c->s_submit = (cudaStream_t)st;
  return HELIOS_OK;
}

void green_io_stop(helios_cache* c) {
  if (!c->green) return;
  PFN_gdestroy gdestroy;
  if (c->s_submit) {
    cudaStreamSynchronize(c->s_submit);
    cudaStreamDestroy(c->s_submit);
    c->s_submit = nullptr;
  }
  if (entry("cuGreenCtxDestroy", &gdestroy) == HELIOS_OK) gdestroy((CUgreenCtx)c->green);
  c->green = nullptr;
}

}  // namespace helios
