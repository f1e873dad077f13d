// sparse_csc.cu — the pixel-sorted form of a sparse sensing matrix C, built once per
// sensing plan (n, p, s, seed) and cached by the handle for sketch_sparse_sorted_kernel.
// The ELL rows from sensing.cu (the stream layout of DESIGN.md §3) become
// (pixel, row << 1 | negative) pairs, radix-sorted by pixel (CUB, one-time
// preprocessing of C's structure, not the per-call data path).
#include <cub/device/device_radix_sort.cuh>

#include "handle.h"

namespace cdmd {

cudaError_t launch_sparse_ell_to_pairs(const SensingPlan& P, const int32_t* ell, const int32_t* counts, int32_t* key,
                                       int32_t* val, cudaStream_t st);

// Returns the cached entry of (P, seed) or builds it from the ELL lists just generated
// on `st` (synchronises `st` once while building).
const SparseCsc* sparse_csc_get(cdmd_handle h, const SensingPlan& P, uint64_t seed, const int32_t* ell,
                                const int32_t* counts, cudaStream_t st, cudaError_t* err) {
  *err = cudaSuccess;
  const auto key = std::make_tuple(P.n, P.p, P.s, seed);
  {
    std::lock_guard<std::mutex> g(h->mu);
    auto it = h->sparse_csc.find(key);
    if (it != h->sparse_csc.end()) return &it->second;
  }
  if (!ell) return nullptr;   // not built yet and no lists to build from
  const int64_t N = P.p * P.cap;
  int32_t *kin = nullptr, *vin = nullptr, *kout = nullptr, *vout = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cudaMalloc(&kin, sizeof(int32_t) * N);
  if (e == cudaSuccess) e = cudaMalloc(&vin, sizeof(int32_t) * N);
  if (e == cudaSuccess) e = cudaMalloc(&kout, sizeof(int32_t) * N);
  if (e == cudaSuccess) e = cudaMalloc(&vout, sizeof(int32_t) * N);
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, vin, vout, (int)N, 0, 24, st);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes + 16);
  if (e == cudaSuccess) e = launch_sparse_ell_to_pairs(P, ell, counts, kin, vin, st);
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, (int)N, 0, 24, st);
  std::vector<int32_t> cnt(P.p);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(cnt.data(), counts, sizeof(int32_t) * P.p, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(kin);
  cudaFree(vin);
  cudaFree(tmp);
  if (e != cudaSuccess) {
    cudaFree(kout);
    cudaFree(vout);
    *err = e;
    return nullptr;
  }
  int64_t nent = 0;
  for (int32_t c : cnt) nent += c;
  std::lock_guard<std::mutex> g(h->mu);
  SparseCsc& c = h->sparse_csc[key];
  c.pos = kout;
  c.rs = vout;
  c.nent = (int)nent;
  return &c;
}

}  // namespace cdmd
