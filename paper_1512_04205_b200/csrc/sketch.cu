// sketch.cu — Y_full = C D (Alg. 1 step 3; Eq. P:286-288) for the four
// measurement matrices.  C is never materialised (north_star): single pixel and
// sparse C are index lists produced by sensing.cu; Rademacher / Gaussian entries
// are regenerated from Philox inside the kernels.
//
// Single pixel / sparse: HBM sector-gather bound (one 32-B sector per (entry,
// frame)); integer sums are exact in int32 (|Y| <= 255 n < 2^31 for n <= 8.4e6).
// Rademacher: int8 x uint8 dot products (dp4a here; tcgen05 kind::i8 in
// sketch_tc.cu).  Gaussian: exact bf16 x uint8 products, fp32 partial sums over
// short pixel chunks accumulated in fp64, one rounding to fp32 Y at the end.
#include <stdlib.h>

#include "common.cuh"

namespace cdmd {

// ------------------------------------------------------------ single pixel
// Y[r, t] = D[row_r, t] if row_r lies in this slab, else 0 (partial sums of a
// pixel-sharded run add up to the full sketch).
__global__ void sketch_spixel_kernel(const uint8_t* __restrict__ X, int64_t ld, int64_t pix0,
                                     int64_t n_local, int64_t m, int64_t p,
                                     const int32_t* __restrict__ rows, int32_t* __restrict__ Y,
                                     int64_t ldy) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p) return;
  const int64_t j = (int64_t)rows[r] - pix0;
  const bool in = j >= 0 && j < n_local;
  const int64_t t0 = (int64_t)blockIdx.y * 64;
  const int64_t t1 = t0 + 64 < m ? t0 + 64 : m;
#pragma unroll 8
  for (int64_t t = t0; t < t1; ++t) Y[r + t * ldy] = in ? (int32_t)__ldg(X + t * ld + j) : 0;
}

cudaError_t launch_sketch_spixel(const cdmd_video& v, const SensingPlan& P, const int32_t* rows,
                                 int32_t* Y, int64_t ldy, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(P.p, 128), (unsigned)ceil_div(v.m, 64));
  note_launch();
  sketch_spixel_kernel<<<grid, 128, 0, st>>>(v.X, v.ld, v.pix0, v.n_local, v.m, P.p, rows, Y, ldy);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ sparse
// One warp per row r of C, one lane per frame: lane t accumulates
// sum_e sign_e * D[pos_e, t] over the row's ELL entries (warp-uniform trip
// count; the entry list is a broadcast load).  8 gathers in flight per lane.
__global__ void __launch_bounds__(256) sketch_sparse_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t pix0, int64_t n_local, int64_t m, int64_t p,
    const int32_t* __restrict__ ell, const int32_t* __restrict__ counts, int64_t cap,
    int32_t* __restrict__ Y, int64_t ldy) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + warp;
  if (r >= p) return;
  const int64_t t = (int64_t)blockIdx.y * 32 + lane;
  const bool tok = t < m;
  const uint8_t* __restrict__ xt = X + (tok ? t : 0) * ld - pix0;
  const int32_t* __restrict__ e = ell + r * cap;
  const int cnt = counts[r];
  int32_t acc = 0;
  int i = 0;
  for (; i + 8 <= cnt; i += 8) {
    int32_t ent[8], val[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ent[u] = __ldg(e + i + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t pos = (int64_t)(ent[u] >> 1);
      const bool in = tok && pos >= pix0 && pos < pix0 + n_local;
      val[u] = in ? (int32_t)__ldg(xt + pos) : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += (ent[u] & 1) ? -val[u] : val[u];
  }
  for (; i < cnt; ++i) {
    const int32_t en = __ldg(e + i);
    const int64_t pos = (int64_t)(en >> 1);
    const bool in = tok && pos >= pix0 && pos < pix0 + n_local;
    const int32_t vv = in ? (int32_t)__ldg(xt + pos) : 0;
    acc += (en & 1) ? -vv : vv;
  }
  if (tok) Y[r + t * ldy] = acc;
}

cudaError_t launch_sketch_sparse(const cdmd_video& v, const SensingPlan& P, const int32_t* ell,
                                 const int32_t* counts, int32_t* Y, int64_t ldy, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(P.p, 8), (unsigned)ceil_div(v.m, 32));
  note_launch();
  sketch_sparse_kernel<<<grid, 256, 0, st>>>(v.X, v.ld, v.pix0, v.n_local, v.m, P.p, ell, counts,
                                             P.cap, Y, ldy);
  return cudaGetLastError();
}

// ------------------------------------------------------- sparse, pixel-sorted
// The same sum Y[r, t] = sum_e sign_e D[pos_e, t], reorganised so that X is read once
// per touched 32-B sector and frame in address order: the (pos, row, sign) entries of
// C are sorted by pixel once per sensing plan (cached by the handle, sparse_csc_build),
// a CTA owns SK_TF frames and walks the whole sorted list for them, scattering
// sign * x into its frames' column of Y kept in shared memory (int32 atomics: exact
// and order-independent), then writes those columns of Y.  No global atomics.
constexpr int SK_TF = 4;        // frames per CTA
constexpr int SK_T = 512;

__global__ void __launch_bounds__(SK_T) sketch_sparse_sorted_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t pix0, int64_t n_local, int64_t m, int64_t p,
    const int32_t* __restrict__ pos, const int32_t* __restrict__ rs, int nent, int32_t* __restrict__ Y,
    int64_t ldy) {
  extern __shared__ int32_t ys[];                 // [p][SK_TF]
  __shared__ int range[2];
  const int64_t t0 = (int64_t)blockIdx.x * SK_TF;
  const int nt = (int)(m - t0 < SK_TF ? m - t0 : SK_TF);
  for (int64_t i = threadIdx.x; i < p * SK_TF; i += SK_T) ys[i] = 0;
  if (threadIdx.x < 2) {   // entries of this slab: [first pos >= pix0, first pos >= pix0 + n_local)
    const int64_t key = threadIdx.x == 0 ? pix0 : pix0 + n_local;
    int lo = 0, hi = nent;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int64_t)pos[mid] < key) lo = mid + 1; else hi = mid;
    }
    range[threadIdx.x] = lo;
  }
  __syncthreads();
  const int e0 = range[0], e1 = range[1];
  const uint8_t* __restrict__ xt = X + t0 * ld - pix0;
  int e = e0 + (int)threadIdx.x;
  // two entries per iteration: 2 x SK_TF independent gathers in flight per thread
  for (; e + SK_T < e1; e += 2 * SK_T) {
    const int64_t pa = pos[e], pb = pos[e + SK_T];
    const int ra = rs[e], rb = rs[e + SK_T];
    int va[SK_TF], vb[SK_TF];
#pragma unroll
    for (int tt = 0; tt < SK_TF; ++tt) {
      va[tt] = tt < nt ? (int)__ldg(xt + tt * ld + pa) : 0;
      vb[tt] = tt < nt ? (int)__ldg(xt + tt * ld + pb) : 0;
    }
#pragma unroll
    for (int tt = 0; tt < SK_TF; ++tt) {
      atomicAdd(&ys[(ra >> 1) * SK_TF + tt], (ra & 1) ? -va[tt] : va[tt]);
      atomicAdd(&ys[(rb >> 1) * SK_TF + tt], (rb & 1) ? -vb[tt] : vb[tt]);
    }
  }
  for (; e < e1; e += SK_T) {
    const int64_t pa = pos[e];
    const int ra = rs[e];
#pragma unroll
    for (int tt = 0; tt < SK_TF; ++tt) {
      const int v = tt < nt ? (int)__ldg(xt + tt * ld + pa) : 0;
      atomicAdd(&ys[(ra >> 1) * SK_TF + tt], (ra & 1) ? -v : v);
    }
  }
  __syncthreads();
  for (int tt = 0; tt < nt; ++tt)
    for (int64_t r = threadIdx.x; r < p; r += SK_T) Y[r + (t0 + tt) * ldy] = ys[r * SK_TF + tt];
}

bool sketch_sparse_sorted_supported(int64_t p) { return (size_t)p * SK_TF * sizeof(int32_t) <= 160 * 1024; }

cudaError_t launch_sketch_sparse_sorted(const cdmd_video& v, const SensingPlan& P, const int32_t* pos,
                                        const int32_t* rs, int nent, int32_t* Y, int64_t ldy, cudaStream_t st) {
  const size_t smem = (size_t)P.p * SK_TF * sizeof(int32_t);
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(sketch_sparse_sorted_kernel));
  if (e != cudaSuccess) return e;
  note_launch();
  sketch_sparse_sorted_kernel<<<(unsigned)ceil_div(v.m, SK_TF), SK_T, smem, st>>>(v.X, v.ld, v.pix0, v.n_local, v.m,
                                                                                 P.p, pos, rs, nent, Y, ldy);
  return cudaGetLastError();
}

// ELL rows -> (key = pos or 0xFFFFFF for an unused slot, value = row << 1 | negative)
__global__ void sparse_ell_to_pairs_kernel(const int32_t* __restrict__ ell, const int32_t* __restrict__ counts,
                                           int64_t p, int64_t cap, int32_t* __restrict__ key,
                                           int32_t* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p * cap) return;
  const int64_t r = i / cap, c = i % cap;
  const int32_t en = ell[i];
  const bool used = c < counts[r];
  key[i] = used ? (en >> 1) : 0xFFFFFF;
  val[i] = used ? (int32_t)((r << 1) | (en & 1)) : 0;
}

cudaError_t launch_sparse_ell_to_pairs(const SensingPlan& P, const int32_t* ell, const int32_t* counts, int32_t* key,
                                       int32_t* val, cudaStream_t st) {
  const int64_t N = P.p * P.cap;
  note_launch();
  sparse_ell_to_pairs_kernel<<<(unsigned)ceil_div(N, 256), 256, 0, st>>>(ell, counts, P.p, P.cap, key, val);
  return cudaGetLastError();
}

// -------------------------------------------------------- Rademacher (SIMT)
// Block tile: 64 rows of C x 64 frames; K loop over 128-pixel chunks aligned to
// the global 128-pixel grid (pix0 % 128 == 0), so one Philox call yields the
// 128 sign bits of (row, chunk).  dp4a.u32.s32: 4 uint8 pixels x 4 int8 signs.
__device__ __forceinline__ int32_t dp4a_us(uint32_t a_u8, uint32_t b_s8, int32_t c) {
  int32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8), "r"(b_s8), "r"(c));
  return d;
}

__global__ void __launch_bounds__(256) sketch_rademacher_simt_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t pix0, int64_t n_local, int64_t m, int64_t p,
    uint32_t k0, uint32_t k1, int32_t* __restrict__ Y, int64_t ldy) {
  __shared__ uint32_t cb[64][5];        // sign bits of 64 rows x 128 pixels
  __shared__ uint32_t xs[64][33];       // 64 frames x 128 pixels (32 words)
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  const int64_t r0 = (int64_t)blockIdx.x * 64, f0 = (int64_t)blockIdx.y * 64;
  int32_t acc[4][4] = {};
  // nibble -> 4 int8 signs (bit 0 -> +1, bit 1 -> -1)
  auto expand = [](uint32_t nib) -> uint32_t {
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) w |= (((nib >> b) & 1u) ? 0xFFu : 0x01u) << (8 * b);
    return w;
  };
  for (int64_t c0 = 0; c0 < n_local; c0 += 128) {
    __syncthreads();
    if (tid < 64) {
      const int64_t r = r0 + tid;
      uint4 w = make_uint4(0, 0, 0, 0);
      if (r < p) w = philox(make_uint4((uint32_t)((pix0 + c0) >> 7), (uint32_t)r, 0u, TAG_RADEMACHER), k0, k1);
      cb[tid][0] = w.x; cb[tid][1] = w.y; cb[tid][2] = w.z; cb[tid][3] = w.w;
    }
    for (int i = tid; i < 64 * 32; i += 256) {
      const int f = i >> 5, q = i & 31;
      const int64_t t = f0 + f, j = c0 + 4 * q;
      uint32_t val = 0;
      if (t < m) {
        if (j + 3 < n_local) {
          val = *reinterpret_cast<const uint32_t*>(X + t * ld + j);
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (j + b < n_local) val |= (uint32_t)X[t * ld + j + b] << (8 * b);
        }
      }
      xs[f][q] = val;
    }
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < 32; ++q) {
      uint32_t sg[4], xv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) sg[a] = expand((cb[ty * 4 + a][q >> 3] >> (4 * (q & 7))) & 15u);
#pragma unroll
      for (int b = 0; b < 4; ++b) xv[b] = xs[tx * 4 + b][q];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = dp4a_us(xv[b], sg[a], acc[a][b]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t r = r0 + ty * 4 + a, t = f0 + tx * 4 + b;
      if (r < p && t < m) Y[r + t * ldy] = acc[a][b];
    }
}

bool sketch_rademacher_tc_supported(const cdmd_video& v);
cudaError_t launch_sketch_rademacher_tc(const cdmd_video& v, const SensingPlan& P, int32_t* Y, int64_t ldy,
                                        cudaStream_t st);

cudaError_t launch_sketch_rademacher(const cdmd_video& v, const SensingPlan& P, int32_t* Y,
                                     int64_t ldy, cudaStream_t st) {
  if (sketch_rademacher_tc_supported(v) && !getenv("CDMD_SIMT_SKETCH"))
    return launch_sketch_rademacher_tc(v, P, Y, ldy, st);
  dim3 grid((unsigned)ceil_div(P.p, 64), (unsigned)ceil_div(v.m, 64));
  note_launch();
  sketch_rademacher_simt_kernel<<<grid, 256, 0, st>>>(v.X, v.ld, v.pix0, v.n_local, v.m, P.p, P.k0,
                                                      P.k1, Y, ldy);
  return cudaGetLastError();
}

// ---------------------------------------------------------- Gaussian (SIMT)
// Block tile: 64 rows x 64 frames; K loop over 32-pixel chunks (4 Philox calls
// per row give 8 table indices each).  fp32 FMA of exact products.
__global__ void __launch_bounds__(256) sketch_gaussian_simt_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t pix0, int64_t n_local, int64_t m, int64_t p,
    uint32_t k0, uint32_t k1, const uint16_t* __restrict__ table, float* __restrict__ Y,
    int64_t ldy) {
  __shared__ float cs[32][65];   // [pixel][row]
  __shared__ float xs[32][65];   // [pixel][frame]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t r0 = (int64_t)blockIdx.x * 64, f0 = (int64_t)blockIdx.y * 64;
  double acc64[4][4] = {};
  for (int64_t c0 = 0; c0 < n_local; c0 += 32) {
    float acc[4][4] = {};
    __syncthreads();
    {  // 64 rows x 4 groups of 8 pixels: one Philox call per thread
      const int rr = tid >> 2, g = tid & 3;
      const int64_t r = r0 + rr;
      const int64_t gi = pix0 + c0 + 8 * g;  // global pixel of slot 0 (multiple of 8)
      uint4 w = make_uint4(0, 0, 0, 0);
      if (r < p) w = philox(make_uint4((uint32_t)(gi >> 3), (uint32_t)r, 0u, TAG_GAUSSIAN), k0, k1);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int sl = 0; sl < 8; ++sl) {
        const uint32_t u16 = (ws[sl >> 1] >> (16 * (sl & 1))) & 0xFFFFu;
        const float c = __uint_as_float((uint32_t)__ldg(table + u16) << 16);
        cs[8 * g + sl][rr] = (r < p && c0 + 8 * g + sl < n_local) ? c : 0.f;
      }
    }
    for (int i = tid; i < 64 * 32; i += 256) {
      const int f = i >> 5, q = i & 31;
      const int64_t t = f0 + f, j = c0 + q;
      xs[q][f] = (t < m && j < n_local) ? (float)X[t * ld + j] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      float a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = cs[q][ty * 4 + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = xs[q][tx * 4 + u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) acc[u][w2] = fmaf(a[u], b[w2], acc[u][w2]);
    }
    // fp32 partial sums of 32 exact products, accumulated across chunks in fp64
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int w2 = 0; w2 < 4; ++w2) acc64[u][w2] += (double)acc[u][w2];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t r = r0 + ty * 4 + a, t = f0 + tx * 4 + b;
      if (r < p && t < m) Y[r + t * ldy] = (float)acc64[a][b];
    }
}

bool sketch_gaussian_tc_supported(const cdmd_video& v);
int gaussian_tc_splits(const cdmd_video& v, int64_t p);
cudaError_t launch_sketch_gaussian_tc(const cdmd_video& v, const SensingPlan& P, const uint16_t* table, float* part,
                                      int* splits_out, cudaStream_t st);
bool sketch_gaussian_tc2_supported(const cdmd_video& v);
int gaussian_tc2_splits(const cdmd_video& v, int64_t p);
cudaError_t launch_sketch_gaussian_tc2(const cdmd_video& v, const SensingPlan& P, const uint16_t* table, float* part,
                                       int* splits_out, cudaStream_t st);

// Y = sum over the split-K partial sums, in split order, in fp64 (deterministic)
__global__ void __launch_bounds__(256) split_reduce_kernel(const float* __restrict__ part, int splits, int64_t p,
                                                           int64_t m, float* __restrict__ Y, int64_t ldy) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p * m) return;
  const int64_t r = idx % p, t = idx / p;
  double s = 0.0;
  for (int q = 0; q < splits; ++q) s += (double)part[((int64_t)q * m + t) * p + r];
  Y[r + t * ldy] = (float)s;
}

cudaError_t launch_sketch_tc2(const cdmd_video& v, const SensingPlan& P, const uint16_t* table, float* part,
                              int* splits_out, const int32_t* freqs, cudaStream_t st);

bool sketch_srft_supported(const cdmd_video& v) { return sketch_gaussian_tc2_supported(v); }

// SRFT (reading R25): the Gaussian pair kernel with the SRFT generator, then the same
// fixed-order split reduction
cudaError_t launch_sketch_srft(const cdmd_video& v, const SensingPlan& P, const int32_t* freqs,
                               const uint16_t* table, float* Y, int64_t ldy, float* part, cudaStream_t st) {
  int splits = 0;
  cudaError_t e = launch_sketch_tc2(v, P, table, part, &splits, freqs, st);
  if (e != cudaSuccess) return e;
  const int64_t total = P.p * v.m;
  note_launch();
  split_reduce_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(part, splits, P.p, v.m, Y, ldy);
  return cudaGetLastError();
}

int64_t gaussian_part_floats(const cdmd_video& v, int64_t p) {
  const int s1 = gaussian_tc_splits(v, p), s2 = gaussian_tc2_splits(v, p);
  return (int64_t)(s1 > s2 ? s1 : s2) * v.m * p;
}

cudaError_t launch_sketch_gaussian(const cdmd_video& v, const SensingPlan& P, const uint16_t* table,
                                   float* Y, int64_t ldy, float* part, cudaStream_t st) {
  if (!getenv("CDMD_SIMT_SKETCH") && part) {
    // CTA pairs (sketch_tc2.cu) by default; CDMD_GAUSS_1CTA selects the single-CTA kernel
    int splits = 0;
    cudaError_t e = cudaErrorNotSupported;
    if (sketch_gaussian_tc2_supported(v) && !getenv("CDMD_GAUSS_1CTA"))
      e = launch_sketch_gaussian_tc2(v, P, table, part, &splits, st);
    else if (sketch_gaussian_tc_supported(v))
      e = launch_sketch_gaussian_tc(v, P, table, part, &splits, st);
    if (e != cudaErrorNotSupported) {
      if (e != cudaSuccess) return e;
      const int64_t total = P.p * v.m;
      note_launch();
      split_reduce_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, st>>>(part, splits, P.p, v.m, Y, ldy);
      return cudaGetLastError();
    }
  }
  dim3 grid((unsigned)ceil_div(P.p, 64), (unsigned)ceil_div(v.m, 64));
  note_launch();
  sketch_gaussian_simt_kernel<<<grid, 256, 0, st>>>(v.X, v.ld, v.pix0, v.n_local, v.m, P.p, P.k0,
                                                    P.k1, table, Y, ldy);
  return cudaGetLastError();
}

}  // namespace cdmd
