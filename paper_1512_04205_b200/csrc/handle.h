// handle.h — per-device state of libcdmd (internal).
#pragma once
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <vector>

#include "common.cuh"

struct cdmd_handle_s {
  int device = 0;
  int sm_count = 0;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cusolverDnParams_t params = nullptr;
  uint16_t* gauss_table = nullptr;   // device, 65536 bf16 bit patterns (immutable)
  int32_t* host_info = nullptr;      // pinned, 16 words for fit read-back
  int* sched = nullptr;              // device, tile counters of the persistent kernels (0 modes, 1 foreground)
  std::vector<char> host_ws;         // cuSOLVER host workspace (fit only)
  double omega_eps = 0.0;            // > 0: background by |omega| < omega_eps, else OMP
};

namespace cdmd {
cdmd_status fit_impl(cdmd_handle h, const void* Y, int64_t ldy, int kind, int64_t p, int64_t m,
                     int k, int K, double dt, cdmd_model* model, void* ws, size_t ws_bytes,
                     cudaStream_t st);
size_t fit_ws_bytes(cdmd_handle h, int64_t p, int64_t m, int k);
}  // namespace cdmd
