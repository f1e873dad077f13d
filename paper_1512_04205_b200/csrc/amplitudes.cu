// amplitudes.cu — full-state amplitudes b = lstsq(Phi, x_1) (Alg. 1 step 9).
//
// Phi arrives folded (cdmd_modes): real columns F, a real mode j -> F_j = phi_j, a
// conjugate pair (j, j+1) -> F_j = Re phi_j, F_{j+1} = Im phi_j.  x_1 is real, so the
// complex least-squares problem min ||x_1 - Phi b|| is the real one min ||x_1 - F c||
// with b_j = c_j (real mode) and b_j = (c_j - i c_{j+1}) / 2, b_{j+1} = conj(b_j)
// (pair), because phi_j b_j + conj(phi_j b_j) = 2 (F_j Re b_j - F_{j+1} Im b_j).
//
// Two phases so a pixel-row-sharded run only exchanges k (k + 1) doubles:
//   gram : G = [F^T F | F^T x_1] of the slab (HBM pass over Phi, fp64 accumulation of
//          exact fp32 x fp32 products, fixed-order block reduction: deterministic);
//   solve: Cholesky of F^T F in fp64 on one CTA, two triangular solves, unfold to b.
// The caller sums G over slabs (all-reduce) between the two calls.
#include "handle.h"

namespace cdmd {
namespace {

constexpr int kAmpThreads = 512;
constexpr int kAmpTile = 64;  // pixels per shared-memory tile

__host__ __device__ inline int amp_entries(int k) { return k * (k + 1) / 2 + k; }

// Entry e of the upper triangle of the (k+1) x (k+1) matrix [F x_1]^T [F x_1] without
// its (k, k) corner, row-major over i: (i, j) with i <= j <= k, i < k.
__device__ inline void amp_entry(int e, int k, int& i, int& j) {
  // row i holds k + 1 - i entries
  int r = 0, base = 0;
  while (e >= base + (k + 1 - r)) { base += k + 1 - r; ++r; }
  i = r;
  j = r + (e - base);
}

template <int NQ>
__global__ void __launch_bounds__(kAmpThreads)
amp_gram_kernel(const float* __restrict__ Phi, int64_t ldphi, const uint8_t* __restrict__ x1,
                int64_t n_local, int k, double* __restrict__ part) {
  extern __shared__ float sF[];  // (k + 1) rows of kAmpTile + 1 floats; row k = x_1
  constexpr int LD = kAmpTile + 1;
  const int E = amp_entries(k);
  double acc[NQ];
  int off_i[NQ], off_j[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    acc[q] = 0.0;
    const int e = threadIdx.x + q * kAmpThreads;
    int i = 0, j = 0;
    if (e < E) amp_entry(e, k, i, j);
    off_i[q] = i * LD;
    off_j[q] = j * LD;
  }
  const int64_t ntiles = (n_local + kAmpTile - 1) / kAmpTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kAmpTile;
    __syncthreads();
    for (int idx = threadIdx.x; idx < (k + 1) * kAmpTile; idx += kAmpThreads) {
      const int c = idx / kAmpTile, p = idx % kAmpTile;
      const int64_t j = p0 + p;
      float v = 0.f;
      if (j < n_local) v = c < k ? __ldg(Phi + (int64_t)c * ldphi + j) : (float)__ldg(x1 + j);
      sF[c * LD + p] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int p = 0; p < kAmpTile; ++p) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        acc[q] = fma((double)sF[off_i[q] + p], (double)sF[off_j[q] + p], acc[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int e = threadIdx.x + q * kAmpThreads;
    if (e < E) part[(int64_t)blockIdx.x * E + e] = acc[q];
  }
}

// Fixed-order sum of the block partials; writes G (k x (k+1), column-major, ld k)
// with both triangles of F^T F and column k = F^T x_1.
__global__ void amp_reduce_kernel(const double* __restrict__ part, int nblocks, int k,
                                  double* __restrict__ G) {
  const int E = amp_entries(k);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += part[(int64_t)b * E + e];
  int i, j;
  amp_entry(e, k, i, j);
  G[i + (int64_t)j * k] = s;
  if (j < k) G[j + (int64_t)i * k] = s;
}

// One CTA: Cholesky F^T F = L L^T (fp64, lower triangle in shared memory), L y = r,
// L^T c = y, then unfold c to the complex amplitudes.  A pivot d^2 <= kAmpPivotRtol *
// (F^T F)_jj (column j dependent on the earlier ones to ~1e-6 in norm, below the fp32
// resolution of Phi) drops column j: c_j = 0, still a least-squares solution
// (reading R24).
constexpr double kAmpPivotRtol = 1e-12;

__global__ void amp_solve_kernel(const double* __restrict__ G, int k, const int32_t* __restrict__ pair,
                                 double* __restrict__ b, int32_t* __restrict__ dropped) {
  extern __shared__ double sA[];  // k x k (column-major), then r[k], then diag0[k]
  double* r = sA + (size_t)k * k;
  double* d0 = r + k;
  __shared__ int s_drop[128];
  __shared__ int s_ndrop;
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) sA[idx] = G[idx];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    r[i] = G[i + (int64_t)k * k];
    d0[i] = G[i + (int64_t)i * k];
    s_drop[i] = 0;
  }
  if (threadIdx.x == 0) s_ndrop = 0;
  __syncthreads();
  for (int c = 0; c < k; ++c) {
    const double d2 = sA[c + c * k];
    const bool drop = !(d2 > kAmpPivotRtol * d0[c]) || !(d0[c] > 0.0);
    const double inv = drop ? 0.0 : rsqrt(d2);
    __syncthreads();
    if (threadIdx.x == 0) {
      sA[c + c * k] = drop ? 0.0 : sqrt(d2);
      if (drop) { s_drop[c] = 1; ++s_ndrop; }
    }
    for (int i = c + 1 + threadIdx.x; i < k; i += blockDim.x) sA[i + c * k] *= inv;
    __syncthreads();
    // trailing update of the lower triangle: A_ij -= L_ic L_jc, c < j <= i
    const int rem = k - c - 1;
    for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
      const int i = c + 1 + idx / rem, j = c + 1 + idx % rem;
      if (j <= i) sA[i + j * k] -= sA[i + c * k] * sA[j + c * k];
    }
    __syncthreads();
  }
  // forward: L y = r (y overwrites r); dropped rows give y = 0
  for (int c = 0; c < k; ++c) {
    if (threadIdx.x == 0) r[c] = s_drop[c] ? 0.0 : r[c] / sA[c + c * k];
    __syncthreads();
    for (int i = c + 1 + threadIdx.x; i < k; i += blockDim.x) r[i] -= sA[i + c * k] * r[c];
    __syncthreads();
  }
  // backward: L^T c = y
  for (int c = k - 1; c >= 0; --c) {
    if (threadIdx.x == 0) r[c] = s_drop[c] ? 0.0 : r[c] / sA[c + c * k];
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += blockDim.x) r[i] -= sA[c + i * k] * r[c];
    __syncthreads();
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double re, im;
    if (pair[j] == 0) {
      re = r[j]; im = 0.0;
    } else if (pair[j] > 0) {
      re = 0.5 * r[j]; im = -0.5 * r[j + 1];
    } else {
      re = 0.5 * r[j - 1]; im = 0.5 * r[j];
    }
    b[2 * j] = re;
    b[2 * j + 1] = im;
  }
  if (threadIdx.x == 0 && dropped) *dropped = s_ndrop;
}

}  // namespace

int amp_gram_blocks(int sms) { return 2 * (sms > 0 ? sms : 148); }

size_t amp_gram_ws_bytes(int sms, int k) {
  return (size_t)amp_gram_blocks(sms) * (size_t)amp_entries(k) * sizeof(double);
}

size_t amp_solve_smem_bytes(int k) { return ((size_t)k * k + 2 * (size_t)k) * sizeof(double); }

cudaError_t launch_amp_gram(int sms, const float* Phi, int64_t ldphi, const uint8_t* x1, int64_t n_local,
                            int k, double* ws, double* G, cudaStream_t st) {
  const int E = amp_entries(k);
  const int64_t ntiles = (n_local + kAmpTile - 1) / kAmpTile;
  int blocks = amp_gram_blocks(sms);
  if ((int64_t)blocks > ntiles) blocks = (int)ntiles;
  const size_t smem = (size_t)(k + 1) * (kAmpTile + 1) * sizeof(float);
  const int nq = (E + kAmpThreads - 1) / kAmpThreads;
  note_launch();
  if (nq <= 1) amp_gram_kernel<1><<<blocks, kAmpThreads, smem, st>>>(Phi, ldphi, x1, n_local, k, ws);
  else if (nq <= 2) amp_gram_kernel<2><<<blocks, kAmpThreads, smem, st>>>(Phi, ldphi, x1, n_local, k, ws);
  else if (nq <= 4) amp_gram_kernel<4><<<blocks, kAmpThreads, smem, st>>>(Phi, ldphi, x1, n_local, k, ws);
  else if (nq <= 8) amp_gram_kernel<8><<<blocks, kAmpThreads, smem, st>>>(Phi, ldphi, x1, n_local, k, ws);
  else amp_gram_kernel<17><<<blocks, kAmpThreads, smem, st>>>(Phi, ldphi, x1, n_local, k, ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  note_launch();
  amp_reduce_kernel<<<(E + 255) / 256, 256, 0, st>>>(ws, blocks, k, G);
  return cudaGetLastError();
}

cudaError_t launch_amp_solve(const double* G, int k, const int32_t* pair, double* b, int32_t* dropped,
                             cudaStream_t st) {
  const size_t smem = amp_solve_smem_bytes(k);
  cudaError_t e = cudaFuncSetAttribute(amp_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  note_launch();
  amp_solve_kernel<<<1, 256, smem, st>>>(G, k, pair, b, dropped);
  return cudaGetLastError();
}

}  // namespace cdmd
