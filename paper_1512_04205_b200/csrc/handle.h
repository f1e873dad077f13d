// handle.h — per-device state of libcdmd (internal).
#pragma once
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <atomic>
#include <map>
#include <array>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace cdmd {
// pixel-sorted entries of a sparse C (sparse_csc.cu): pos ascending, rs = row << 1 | negative
struct SparseCsc {
  int32_t* pos = nullptr;
  int32_t* rs = nullptr;
  int nent = 0;
};
}  // namespace cdmd

struct cdmd_handle_s {
  int device = 0;
  int sm_count = 0;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cusolverDnParams_t params = nullptr;
  uint16_t* gauss_table = nullptr;   // device, 65536 bf16 bit patterns (immutable)
  uint16_t* srft_table = nullptr;    // device, 16385 fp16 bit patterns of the SRFT quarter wave (immutable)
  int32_t* host_info = nullptr;      // pinned, 16 words for fit read-back
  // device, CDMD_SCHED_SLOTS tile counters of the persistent kernels (dynamic tile
  // schedule).  Every launch takes the next slot, so persistent launches of one handle
  // on different streams never share a counter (up to CDMD_SCHED_SLOTS in flight).
  int* sched = nullptr;
  std::atomic<uint32_t> sched_next{0};
  // sparse plans (n, p, s, seed) whose index lists were checked once against their ELL
  // capacity (cdmd_sketch syncs the first time a plan is seen, never afterwards)
  std::set<std::tuple<int64_t, int64_t, double, uint64_t>> sparse_checked;
  std::map<std::tuple<int64_t, int64_t, double, uint64_t>, cdmd::SparseCsc> sparse_csc;   // plan -> sorted C
  std::mutex mu;
  std::vector<char> host_ws;         // cuSOLVER host workspace (fit only)
  double omega_eps = 0.0;            // > 0: background by |omega| < omega_eps, else OMP
  // cuSOLVER workspace sizes per (p, m, k) (sy_dev, sy_host, ge_dev, ge_host): queried once,
  // so a fit under stream capture needs no cuSOLVER call
  std::map<std::tuple<int64_t, int64_t, int>, std::array<size_t, 4>> fit_ws_sizes;
  // (m - 1, k) shapes whose last eager fit fell back from Lanczos: a fit captured into a
  // graph for them takes the Householder solver directly, as the eager fit ended up doing
  std::set<std::pair<int64_t, int>> lz_fell_back;
  std::atomic<uint64_t> lz_runs{0};       // cdmd_fit calls whose eigenpairs came from Lanczos
  std::atomic<uint64_t> lz_fallbacks{0};  // ... of which failed the residual test (Householder reran)
};

#define CDMD_SCHED_SLOTS 64

namespace cdmd {
// a tile counter of its own for one persistent launch (reset on the launch's stream)
inline int* sched_slot(cdmd_handle h) {
  return h->sched + (h->sched_next.fetch_add(1, std::memory_order_relaxed) % CDMD_SCHED_SLOTS);
}
const SparseCsc* sparse_csc_get(cdmd_handle h, const SensingPlan& P, uint64_t seed, const int32_t* ell,
                                const int32_t* counts, cudaStream_t st, cudaError_t* err);
bool sketch_sparse_sorted_supported(int64_t p);
cudaError_t launch_sketch_sparse_sorted(const cdmd_video& v, const SensingPlan& P, const int32_t* pos,
                                        const int32_t* rs, int nent, int32_t* Y, int64_t ldy, cudaStream_t st);
cdmd_status fit_impl(cdmd_handle h, const void* Y, int64_t ldy, int kind, int64_t p, int64_t m,
                     int k, int K, double dt, cdmd_model* model, void* ws, size_t ws_bytes,
                     cudaStream_t st);
size_t fit_ws_bytes(cdmd_handle h, int64_t p, int64_t m, int k);
}  // namespace cdmd
