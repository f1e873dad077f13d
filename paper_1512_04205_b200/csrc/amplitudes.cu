// amplitudes.cu — full-state amplitudes b = lstsq(Phi, x_1) (Alg. 1 step 9).
//
// Phi arrives folded (cdmd_modes): real columns F, a real mode j -> F_j = phi_j, a
// conjugate pair (j, j+1) -> F_j = Re phi_j, F_{j+1} = Im phi_j.  x_1 is real, so the
// complex least-squares problem min ||x_1 - Phi b|| is the real one min ||x_1 - F c||
// with b_j = c_j (real mode) and b_j = (c_j - i c_{j+1}) / 2, b_{j+1} = conj(b_j)
// (pair), because phi_j b_j + conj(phi_j b_j) = 2 (F_j Re b_j - F_{j+1} Im b_j).
//
// Two phases so a pixel-row-sharded run only exchanges k (k + 1) doubles:
//   gram : G = [F^T F | F^T x_1] of the slab (one pass over Phi; register-blocked fp32
//          FMAs within a 128-pixel tile, fp64 across tiles; fixed-order reduction of
//          the per-CTA partials: deterministic);
//   solve: Cholesky of F^T F in fp64 on one CTA, two triangular solves, unfold to b.
// The caller sums G over slabs (all-reduce) between the two calls.
#include "handle.h"

namespace cdmd {
namespace {

constexpr int kAmpTile = 128;  // pixels per shared-memory tile

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

// Shared row stride: 16-byte aligned and = 4 (mod 8) words (4-way store conflicts at worst).
__host__ __device__ inline int amp_ldc(int nb) { return (4 * nb) % 8 == 0 ? 4 * nb + 4 : 4 * nb + 8; }

// Row-major offset of entry (i, j), i <= j, in the list above.
__host__ __device__ inline int amp_entry_index(int i, int j, int k) {
  return i * (k + 1) - i * (i - 1) / 2 + (j - i);
}

__device__ inline void cp_async4(float* dst, const float* src, bool valid) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}

// Register-blocked Gram pass.  Shared tile: kAmpTile pixels x ldc floats, pixel-
// major (row p = the k folded mode values of pixel p, then x_1, zero-padded to a
// multiple of 4), so a thread's 4 + 4 operands are two 16-byte loads.  Tiles are
// double-buffered: cp.async (4-byte, transposing, zero-filled past n_local) fills the
// next tile while the current one is consumed; x_1 (bytes) goes through a register.
// Each thread of a group owns one 4 x 4 micro-tile (bi <= bj) of the upper block
// triangle of [F x_1]^T [F x_1]; the NG (a power of two) groups of a CTA split the tile's pixels into contiguous runs.
// Products are summed in fp32 over one tile (<= kAmpTile / NG terms), then added to
// fp64 totals, so fp32 rounding stays per-tile.  Partials: one row of E doubles per
// (CTA, group), summed in fixed order by amp_reduce_kernel.
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
amp_gram_kernel(const float* __restrict__ Phi, int64_t ldphi, const uint8_t* __restrict__ x1,
                int64_t n_local, int k, int nb, int nmt, int tg, int ng, double* __restrict__ part) {
  extern __shared__ __align__(16) float sF[];
  const int ldc = amp_ldc(nb);
  const int stage_floats = kAmpTile * ldc;
  const int E = amp_entries(k);
  const int g = threadIdx.x / tg, t = threadIdx.x % tg;
  int bi = 0, bj = 0;
  {  // micro-tile t -> (bi, bj), bi <= bj, row-major over the block triangle
    int r = 0, base = 0;
    while (r < nb && t >= base + (nb - r)) { base += nb - r; ++r; }
    bi = r;
    bj = r + (t - base);
  }
  const bool active = t < nmt;
  // zero the padding columns k+1 .. 4nb-1 of both stages once
  const int npad = 4 * nb - (k + 1);
  for (int idx = threadIdx.x; idx < 2 * kAmpTile * npad; idx += blockDim.x) {
    const int st = idx / (kAmpTile * npad), r = idx % (kAmpTile * npad);
    sF[st * stage_floats + (r / npad) * ldc + k + 1 + r % npad] = 0.f;
  }
  double tot[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) tot[q] = 0.0;
  const int64_t ntiles = (n_local + kAmpTile - 1) / kAmpTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  auto issue = [&](int64_t tile, int st) {
    const int64_t p0 = tile * kAmpTile;
    float* dst = sF + st * stage_floats;
    if (p0 + kAmpTile <= n_local) {  // full tile: no bounds tests, pointer strides only
      const float* src = Phi + (int64_t)warp * ldphi + p0 + lane;
      float* d = dst + lane * ldc + warp;
      const int64_t sstep = (int64_t)nwarps * ldphi;
      for (int c = warp; c < k; c += nwarps, src += sstep, d += nwarps) {
#pragma unroll
        for (int j = 0; j < kAmpTile / 32; ++j) cp_async4(d + j * 32 * ldc, src + j * 32, true);
      }
    } else {
      for (int c = warp; c < k; c += nwarps) {
        const float* src = Phi + (int64_t)c * ldphi + p0;
#pragma unroll
        for (int p = lane; p < kAmpTile; p += 32) {
          const bool ok = p0 + p < n_local;
          cp_async4(dst + p * ldc + c, src + (ok ? p : 0), ok);
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  float xreg = 0.f;
  auto load_x = [&](int64_t tile) {
    const int64_t j = tile * kAmpTile + threadIdx.x;
    xreg = (threadIdx.x < kAmpTile && j < n_local) ? (float)__ldg(x1 + j) : 0.f;
  };
  int64_t tile = blockIdx.x;
  int st = 0;
  if (tile < ntiles) { issue(tile, 0); load_x(tile); }
  for (; tile < ntiles; tile += gridDim.x, st ^= 1) {
    if (threadIdx.x < kAmpTile) sF[st * stage_floats + threadIdx.x * ldc + k] = xreg;
    const int64_t nxt = tile + gridDim.x;
    if (nxt < ntiles) {
      issue(nxt, st ^ 1);
      load_x(nxt);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    if (active) {
      const float* cur = sF + st * stage_floats;
      float acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = 0.f;
      const int ppg = kAmpTile / ng;  // each group: a contiguous run of the tile's pixels
      const float* pa = cur + g * ppg * ldc + 4 * bi;
      const float* pb = cur + g * ppg * ldc + 4 * bj;
#pragma unroll 4
      for (int p = 0; p < ppg; ++p, pa += ldc, pb += ldc) {
        const float4 a = *reinterpret_cast<const float4*>(pa);
        const float4 b = *reinterpret_cast<const float4*>(pb);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) acc[u * 4 + w] = fmaf(av[u], bv[w], acc[u * 4 + w]);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) tot[q] += (double)acc[q];
    }
    __syncthreads();  // stage st is refilled by the next iteration's issue
  }
  if (!active) return;
  double* row = part + ((int64_t)blockIdx.x * ng + g) * E;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int i = 4 * bi + u, j = 4 * bj + w;
      if (i <= j && i < k && j <= k) row[amp_entry_index(i, j, k)] = tot[u * 4 + w];
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
// (reading R23).
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

struct AmpGramShape {
  int nb, nmt, tg, ng, threads;
};

AmpGramShape amp_gram_shape(int k) {
  AmpGramShape g;
  g.nb = (k + 1 + 3) / 4;
  g.nmt = g.nb * (g.nb + 1) / 2;
  g.tg = (g.nmt + 31) / 32 * 32;
  g.ng = 1;  // a power of two dividing kAmpTile
  while (g.ng < 16 && g.tg * g.ng * 2 <= 256) g.ng *= 2;
  g.threads = g.tg * g.ng;
  return g;
}

int amp_gram_blocks(int sms) { return 3 * (sms > 0 ? sms : 148); }

size_t amp_gram_ws_bytes(int sms, int k) {
  return (size_t)amp_gram_blocks(sms) * amp_gram_shape(k).ng * (size_t)amp_entries(k) * sizeof(double);
}

size_t amp_solve_smem_bytes(int k) { return ((size_t)k * k + 2 * (size_t)k) * sizeof(double); }

cudaError_t launch_amp_gram(int sms, const float* Phi, int64_t ldphi, const uint8_t* x1, int64_t n_local,
                            int k, double* ws, double* G, cudaStream_t st) {
  const int E = amp_entries(k);
  const AmpGramShape sh = amp_gram_shape(k);
  const int64_t ntiles = (n_local + kAmpTile - 1) / kAmpTile;
  int blocks = amp_gram_blocks(sms);
  if ((int64_t)blocks > ntiles) blocks = (int)ntiles;
  const size_t smem = 2 * (size_t)kAmpTile * amp_ldc(sh.nb) * sizeof(float);
  // <= 192 threads (k <= 62): three resident CTAs per SM (measured: 2 x 384 threads 0.41 ms,
  // 3 x 192 0.38 ms, 4 x 192 on 64-pixel tiles 0.39 ms at c4)
  const bool two = sh.threads <= 192;
  auto kern = two ? amp_gram_kernel<192, 3> : amp_gram_kernel<576, 1>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return e;
  note_launch();
  kern<<<blocks, sh.threads, smem, st>>>(Phi, ldphi, x1, n_local, k, sh.nb, sh.nmt, sh.tg, sh.ng, ws);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  note_launch();
  amp_reduce_kernel<<<(E + 255) / 256, 256, 0, st>>>(ws, blocks * sh.ng, k, G);
  return cudaGetLastError();
}

cudaError_t launch_amp_solve(const double* G, int k, const int32_t* pair, double* b, int32_t* dropped,
                             cudaStream_t st) {
  const size_t smem = amp_solve_smem_bytes(k);
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(amp_solve_kernel));
  if (e != cudaSuccess) return e;
  note_launch();
  amp_solve_kernel<<<1, 256, smem, st>>>(G, k, pair, b, dropped);
  return cudaGetLastError();
}

}  // namespace cdmd
