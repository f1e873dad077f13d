// sensing.cu — on-device generation of the measurement matrix C from
// Philox4x32-10, following the stream layouts of DESIGN.md §3.  C itself is never
// materialised: single pixel and sparse C become index lists (p and ~p ln n
// entries), Rademacher and Gaussian entries are regenerated inside the sketch
// kernels.  Cost is O(p) / O(p ln n) threads of Philox work per call.
#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"

namespace cdmd {

SensingPlan make_plan(int64_t n_total, const cdmd_sensing* c) {
  SensingPlan P{};
  P.kind = c->kind;
  P.n = n_total;
  P.p = c->p;
  P.k0 = (uint32_t)(c->seed & 0xffffffffu);
  P.k1 = (uint32_t)(c->seed >> 32);
  // sparse rate: default s = n / ln n, natural log, global n (reading R6)
  P.s = c->s > 0 ? c->s : (double)n_total / log((double)n_total);
  P.lq = log1p(-1.0 / P.s);
  int bits = 1;
  while (bits < 63 && (((int64_t)1 << bits) < n_total)) ++bits;  // bits to hold n-1
  if (n_total <= 1) bits = 1;
  P.h = (bits + 1) / 2;
  const double mu = (double)n_total / P.s;  // expected non-zeros per sparse row
  P.cap = (int64_t)ceil(mu + 12.0 * sqrt(mu) + 16.0);
  return P;
}

size_t sensing_ws_bytes(const SensingPlan& P) {
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  if (P.kind == CDMD_SPIXEL) return al(sizeof(int32_t) * P.p);
  if (P.kind == CDMD_SRFT) return al(sizeof(int32_t) * (P.p / 2 + 1));
  if (P.kind == CDMD_SPARSE)
    return al(sizeof(int32_t) * P.p * P.cap) + al(sizeof(int32_t) * P.p) + al(16);
  return 256;
}

// ------------------------------------------------------------- single pixel
// Row r of C = R is the pixel pi(r), pi a bijection of [0, n): a 6-round balanced
// Feistel network on 2h-bit words (round i: F_i(R) = Philox(R, i, 0, TAG)[0] mod 2^h)
// restricted to [0, n) by cycle walking.  Distinct rows = sampling without
// replacement.
__global__ void spixel_rows_kernel(int64_t n, int64_t p, int h, uint32_t k0, uint32_t k1,
                                   int32_t* __restrict__ rows, uint32_t tag) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p) return;
  const uint64_t mask = (1ull << h) - 1ull;
  uint64_t x = (uint64_t)r;
  do {
    uint64_t L = x >> h, R = x & mask;
#pragma unroll 1
    for (uint32_t i = 0; i < 6; ++i) {
      const uint64_t f = (uint64_t)philox(make_uint4((uint32_t)R, i, 0u, tag), k0, k1).x & mask;
      const uint64_t nl = R;
      R = L ^ f;
      L = nl;
    }
    x = (L << h) | R;
  } while (x >= (uint64_t)n);
  rows[r] = (int32_t)x;
}

cudaError_t launch_spixel_rows(const SensingPlan& P, int32_t* rows, cudaStream_t st) {
  const int T = 128;
  note_launch();
  spixel_rows_kernel<<<(unsigned)ceil_div(P.p, T), T, 0, st>>>(P.n, P.p, P.h, P.k0, P.k1, rows, TAG_SPIXEL);
  return cudaGetLastError();
}

// SRFT (reading R25): R = p/2 distinct frequencies, the same Feistel
// bijection with its own tag
cudaError_t launch_srft_freqs(const SensingPlan& P, int32_t* freqs, cudaStream_t st) {
  const int T = 128;
  const int64_t nf = P.p / 2;
  note_launch();
  spixel_rows_kernel<<<(unsigned)ceil_div(nf, T), T, 0, st>>>(P.n, nf, P.h, P.k0, P.k1, freqs, TAG_SRFT);
  return cudaGetLastError();
}

// Q[r] = fp16_RNE(cos(2 pi r / 2^16)), r = 0 .. 2^14 (fp64 cos, one rounding)
__global__ void srft_table_kernel(uint16_t* __restrict__ table) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > 16384) return;
  table[r] = __half_as_ushort(__double2half(cos(2.0 * 3.141592653589793238 * (double)r / 65536.0)));
}

cudaError_t launch_srft_table(uint16_t* table, cudaStream_t st) {
  note_launch();
  srft_table_kernel<<<(16385 + 255) / 256, 256, 0, st>>>(table);
  return cudaGetLastError();
}

// -------------------------------------------------------------------- sparse
// Row r: non-zeros of an i.i.d. row with P(c != 0) = 1/s found by
// geometric skips.  Draw j: w = Philox(j, r, 0, TAG); U = 53 random bits,
// u = (U + 1/2) 2^-53 in (0,1); gap g = floor(log u / log(1 - 1/s)); position =
// previous + 1 + g; sign from bit 0 of w2.  ELL entry = pos << 1 | (sign < 0).
__global__ void sparse_rows_kernel(int64_t n, int64_t p, double lq, int64_t cap, uint32_t k0,
                                   uint32_t k1, int32_t* __restrict__ ell,
                                   int32_t* __restrict__ counts, int32_t* __restrict__ flags) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= p) return;
  int64_t prev = -1, cnt = 0;
  for (uint32_t j = 0;; ++j) {
    const uint4 w = philox(make_uint4(j, (uint32_t)r, 0u, TAG_SPARSE), k0, k1);
    const uint64_t U = ((uint64_t)(w.y & 0x1FFFFFu) << 32) | (uint64_t)w.x;
    const double u = ((double)U + 0.5) * 0x1p-53;
    const double g = floor(log(u) / lq);
    if ((double)prev + 1.0 + g >= (double)n) break;
    const int64_t pos = prev + 1 + (int64_t)g;
    if (cnt < cap) ell[r * cap + cnt] = (int32_t)((pos << 1) | (int64_t)(w.z & 1u));
    ++cnt;
    prev = pos;
  }
  counts[r] = (int32_t)(cnt < cap ? cnt : cap);
  if (cnt > cap) atomicOr(flags, FLAG_SPARSE_OVERFLOW);
}

cudaError_t launch_sparse_rows(const SensingPlan& P, int32_t* ell, int32_t* counts, int32_t* flags,
                               cudaStream_t st) {
  const int T = 64;
  note_launch();
  sparse_rows_kernel<<<(unsigned)ceil_div(P.p, T), T, 0, st>>>(P.n, P.p, P.lq, P.cap, P.k0, P.k1,
                                                               ell, counts, flags);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Gaussian
// T[j] = bf16_RNE(Phi^-1((j + 1/2) / 2^16)) (P:374 N(0,1); reading R7), computed
// once per handle in fp64 with the CUDA inverse normal CDF and rounded to 8
// significant bits, ties to even.
__global__ void gaussian_table_kernel(uint16_t* __restrict__ table) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= 65536) return;
  const double x = normcdfinv(((double)j + 0.5) * 0x1p-16);
  int e;
  const double mant = frexp(x, &e);          // x = mant 2^e, 0.5 <= |mant| < 1
  const double y = ldexp(rint(mant * 256.0), e - 8);  // rint: round half to even
  table[j] = (uint16_t)(__float_as_uint((float)y) >> 16);  // y is exact in bf16
}

cudaError_t launch_gaussian_table(uint16_t* table, cudaStream_t st) {
  note_launch();
  gaussian_table_kernel<<<256, 256, 0, st>>>(table);
  return cudaGetLastError();
}

__global__ void philox_test_kernel(const uint32_t* __restrict__ ctr, uint32_t k0, uint32_t k1,
                                   uint32_t* __restrict__ out, int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
  const uint4 w = philox(c, k0, k1);
  out[4 * i] = w.x;
  out[4 * i + 1] = w.y;
  out[4 * i + 2] = w.z;
  out[4 * i + 3] = w.w;
}

cudaError_t launch_philox_test(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                               int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  note_launch();
  philox_test_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, st>>>(ctr, k0, k1, out, count);
  return cudaGetLastError();
}

}  // namespace cdmd
