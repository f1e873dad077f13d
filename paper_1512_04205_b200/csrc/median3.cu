// median3.cu — 3x3 median post-filter of the bit-packed foreground mask (Fig. 7,
// P:582; reading R22).  One thread per output word: the nine shifted
// 32-pixel neighbour words (rows y-1, y, y+1; columns x-1, x, x+1) are assembled
// with funnel shifts from the packed rows, the bits that would wrap across an image
// row are cleared, and a bit-sliced carry-save adder tree gives "at least 5 of 9"
// for all 32 pixels at once.
#include "common.cuh"

namespace cdmd {

namespace {

// 32 mask bits starting at pixel s of one frame (pixels outside [0, n) read as 0)
__device__ __forceinline__ uint32_t bits32(const uint32_t* __restrict__ f, int64_t s, int64_t n, int64_t nw) {
  if (s + 32 <= 0 || s >= n) return 0u;
  const int64_t q = s >> 5;                     // floor division (s may be negative)
  const int r = (int)(s & 31);
  const uint32_t lo = (q >= 0 && q < nw) ? __ldg(f + q) : 0u;
  const uint32_t hi = (q + 1 >= 0 && q + 1 < nw) ? __ldg(f + q + 1) : 0u;
  uint32_t v = (uint32_t)((((uint64_t)hi << 32) | lo) >> r);
  if (s < 0) v &= ~0u << (uint32_t)(-s);        // pixels before 0
  const int64_t past = s + 32 - n;              // pixels at or beyond n
  if (past > 0) v &= past >= 32 ? 0u : (~0u >> (uint32_t)past);
  return v;
}

__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& co) {
  s = a ^ b ^ c;
  co = (a & b) | (a & c) | (b & c);
}

}  // namespace

__global__ void __launch_bounds__(256) mask_median3_kernel(const uint32_t* __restrict__ in, int64_t ldw,
                                                           int64_t W, int64_t H, uint32_t* __restrict__ out) {
  const int64_t n = W * H, nw = (n + 31) >> 5;
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  const int64_t t = blockIdx.y;
  const uint32_t* f = in + t * ldw;
  const int64_t j0 = w << 5;
  // bits whose pixel is in column 0 (no left neighbour) or column W-1 (no right one)
  uint32_t first = 0u, last = 0u;
  for (int64_t i = (W - j0 % W) % W; i < 32; i += W) first |= 1u << i;
  for (int64_t i = (W - 1 - j0 % W + W) % W; i < 32; i += W) last |= 1u << i;
  uint32_t x[9];
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int64_t s = j0 + dy * W;
    x[3 * (dy + 1) + 0] = bits32(f, s - 1, n, nw) & ~first;   // left neighbours
    x[3 * (dy + 1) + 1] = bits32(f, s, n, nw);
    x[3 * (dy + 1) + 2] = bits32(f, s + 1, n, nw) & ~last;    // right neighbours
  }
  // count of the nine bits per position: CSA tree -> (b3 b2 b1 b0), majority = count >= 5
  uint32_t s1, c1, s2, c2, s3, c3, s4, c4, s5, c5;
  fa(x[0], x[1], x[2], s1, c1);
  fa(x[3], x[4], x[5], s2, c2);
  fa(x[6], x[7], x[8], s3, c3);
  fa(s1, s2, s3, s4, c4);        // weight 1: s4; weight 2: c1 c2 c3 c4
  fa(c1, c2, c3, s5, c5);        // weight 2: s5 (+ c4); weight 4: c5
  const uint32_t b1 = s5 ^ c4, c6 = s5 & c4;     // weight 2 total bit; carry to weight 4
  const uint32_t b2 = c5 ^ c6, b3 = c5 & c6;     // weight 4 bit; weight 8 bit
  uint32_t r = b3 | (b2 & (b1 | s4));
  const int64_t tail = n - j0;                   // pixels of this word inside the frame
  if (tail < 32) r &= (1u << tail) - 1u;
  out[t * ldw + w] = r;
}

cudaError_t launch_mask_median3(const uint32_t* in, int64_t ldw, int64_t W, int64_t H, int64_t m, uint32_t* out,
                                cudaStream_t st) {
  const int64_t nw = (W * H + 31) >> 5;
  dim3 grid((unsigned)ceil_div(nw, 256), (unsigned)m);
  note_launch();
  mask_median3_kernel<<<grid, 256, 0, st>>>(in, ldw, W, H, out);
  return cudaGetLastError();
}

}  // namespace cdmd
