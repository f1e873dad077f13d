// partition.cu — spatial SM partition for the streaming driver (green contexts).
//
// Streaming (a long video processed as independent consecutive batches) mixes
// two kinds of work: the full-resolution passes (sketch, modes, foreground), which are
// HBM- or tensor-bound persistent kernels that want every SM, and the small solve
// (cdmd_fit), a chain of ~20 latency-bound kernels on a handful of SMs.  Sharing SMs,
// every kernel of the solve waits for a persistent kernel to drain before it gets an
// SM, so the solve's latency under load grows 3-4x and bounds throughput.  Here the
// device's SMs are split once into two green contexts: `fit_sms` SMs (rounded up to
// the hardware granularity, 8 on sm_100) that only the solves use, and the rest for
// the passes; persistent kernels then size their grids to the pass partition.
#include <cudaTypedefs.h>

#include "common.cuh"

namespace cdmd {
int g_persist_limit = 0;   // > 0: persistent grids use at most this many CTAs
}

namespace {

template <class F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

CUgreenCtx g_ctx[2] = {nullptr, nullptr};

}  // namespace

extern "C" cdmd_status cdmd_sm_partition(int device, int fit_sms, int n_streams, void** pass_streams,
                                         void** fit_streams, int* sms) {
  if (fit_sms <= 0 || n_streams <= 0 || !pass_streams || !fit_streams || !sms) return CDMD_ERR_ARG;
  if (g_ctx[0]) return CDMD_ERR_ARG;   // one partition per process
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess) return CDMD_ERR_CUDA;
  auto devGet = entry<PFN_cuDeviceGet_v2000>("cuDeviceGet");
  auto getRes = entry<PFN_cuDeviceGetDevResource_v12040>("cuDeviceGetDevResource");
  auto split = entry<PFN_cuDevSmResourceSplitByCount_v12040>("cuDevSmResourceSplitByCount");
  auto gen = entry<PFN_cuDevResourceGenerateDesc_v12040>("cuDevResourceGenerateDesc");
  auto create = entry<PFN_cuGreenCtxCreate_v12040>("cuGreenCtxCreate");
  auto screate = entry<PFN_cuGreenCtxStreamCreate_v12050>("cuGreenCtxStreamCreate");
  if (!devGet || !getRes || !split || !gen || !create || !screate) return CDMD_ERR_UNSUPPORTED;
  CUdevice dev;
  if (devGet(&dev, device) != CUDA_SUCCESS) return CDMD_ERR_CUDA;
  CUdevResource all, parts[2];
  if (getRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return CDMD_ERR_CUDA;
  unsigned int groups = 1;
  if (split(&parts[0], &groups, &all, &parts[1], 0, (unsigned)fit_sms) != CUDA_SUCCESS || groups != 1)
    return CDMD_ERR_CUDA;
  if (parts[1].sm.smCount == 0) return CDMD_ERR_RANGE;
  for (int g = 0; g < 2; ++g) {
    CUdevResourceDesc desc;
    if (gen(&desc, &parts[g], 1) != CUDA_SUCCESS) return CDMD_ERR_CUDA;
    if (create(&g_ctx[g], desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return CDMD_ERR_CUDA;
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  for (int i = 0; i < n_streams; ++i) {
    CUstream s;
    if (screate(&s, g_ctx[1], CU_STREAM_NON_BLOCKING, lo) != CUDA_SUCCESS) return CDMD_ERR_CUDA;
    pass_streams[i] = s;
    if (screate(&s, g_ctx[0], CU_STREAM_NON_BLOCKING, hi) != CUDA_SUCCESS) return CDMD_ERR_CUDA;
    fit_streams[i] = s;
  }
  sms[0] = (int)parts[0].sm.smCount;   // solve partition
  sms[1] = (int)parts[1].sm.smCount;   // pass partition
  cdmd::g_persist_limit = sms[1];
  return CDMD_OK;
}
