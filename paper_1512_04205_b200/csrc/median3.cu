// median3.cu — 3x3 median post-filter of the bit-packed foreground mask (Fig. 7,
// P:582; reading R22).  Per output word the nine shifted 32-pixel neighbour
// words (rows y-1, y, y+1; columns x-1, x, x+1) are assembled with funnel shifts from
// the packed rows, the bits that would wrap across an image row are cleared, and a
// bit-sliced carry-save adder tree gives "at least 5 of 9" for all 32 pixels at once.
#include <stdlib.h>

#include "common.cuh"

namespace cdmd {

namespace {

__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& co) {
  s = a ^ b ^ c;
  co = (a & b) | (a & c) | (b & c);
}


}  // namespace

// Each thread produces MW consecutive output words.  For image row offset dy the
// neighbour windows start at pixel j0 + dy W - 1 + {0, 1, 2}: the same bit offset r_dy
// for every word of the thread (and every thread), so three words per row slide along
// and each new output word costs one load per row plus funnel shifts.  32-bit pixel
// indices (whole frames of < 2^31 pixels).
template <int MW>   // output words per thread (consecutive pixels of one frame)
__global__ void __launch_bounds__(256) mask_median3_kernel(const uint32_t* __restrict__ in, int64_t ldw,
                                                           int W, int H, uint32_t* __restrict__ out) {
  const int n = W * H, nw = (n + 31) >> 5;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) * MW;
  if (w0 >= nw) return;
  const int64_t t = blockIdx.y;
  const uint32_t* f = in + t * ldw;
  const uint32_t lastmask = (n & 31) ? ((1u << (n & 31)) - 1u) : ~0u;   // valid bits of word nw - 1
  auto word = [&](int q) -> uint32_t {
    if (q < 0 || q >= nw) return 0u;
    const uint32_t v = __ldg(f + q);
    return q == nw - 1 ? v & lastmask : v;
  };
  // per row: bit offset r; every word the thread's MW outputs need (MW + 2 per row) is
  // loaded up front, so all 3 (MW + 2) loads are in flight at once
  int q[3];
  uint32_t r[3], v[3][MW + 2];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int s = (w0 << 5) + (d - 1) * W - 1;     // may be negative
    q[d] = s >> 5;
    r[d] = (uint32_t)s & 31u;
#pragma unroll
    for (int u = 0; u < MW + 2; ++u) v[d][u] = word(q[d] + u);
  }
  int x0 = (w0 << 5) % W;                          // column of the word's first pixel
#pragma unroll
  for (int u = 0; u < MW; ++u) {
    const int w = w0 + u;
    if (w >= nw) break;
    uint32_t first = 0u, last = 0u;                // pixels in column 0 / column W-1
    if (W >= 32) {                                 // at most one of each per word
      const int i0 = x0 == 0 ? 0 : W - x0, i1 = W - 1 - x0;
      if (i0 < 32) first = 1u << i0;
      if (i1 < 32) last = 1u << i1;
    } else {
      for (int i = (W - x0) % W; i < 32; i += W) first |= 1u << i;
      for (int i = (2 * W - 1 - x0) % W; i < 32; i += W) last |= 1u << i;
    }
    uint32_t x[9];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const uint32_t rr = r[d];
      const uint32_t wa = v[d][u], wb = v[d][u + 1], wc = v[d][u + 2];
      const uint32_t L = __funnelshift_r(wa, wb, rr);
      const uint32_t Cc = rr == 31u ? wb : __funnelshift_r(wa, wb, rr + 1u);
      const uint32_t R = rr >= 30u ? __funnelshift_r(wb, wc, rr - 30u) : __funnelshift_r(wa, wb, rr + 2u);
      x[3 * d + 0] = L & ~first;
      x[3 * d + 1] = Cc;
      x[3 * d + 2] = R & ~last;
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
    uint32_t res = b3 | (b2 & (b1 | s4));
    if (w == nw - 1) res &= lastmask;
    out[t * ldw + w] = res;
    x0 += 32;
    while (x0 >= W) x0 -= W;
  }
}

// Word-aligned rows (W % 128 == 0, 16-B aligned frames and ldw % 4 == 0: 1080p, 4K): a
// thread owns four consecutive words of MR consecutive image rows.  Each image row is
// read as ONE coalesced 16-B load per thread, in a sliding window of three rows (MR + 2
// loads for MR output rows, so L2 serves each word ~(MR + 2)/MR times instead of three);
// the word before and after the thread's four come from the neighbouring lanes by
// shuffles (lanes 0 and 31 load them).  Rows start at word boundaries, so the horizontal
// neighbours are one-bit shifts across adjacent words, and the word across an image-row
// boundary is replaced by zero (zero padding, reading R22) -- which also discards what the
// shuffle brings from a lane in another row.
constexpr int MED_MR = 8;   // image rows per thread

__global__ void __launch_bounds__(256) mask_median3_w32_kernel(const uint32_t* __restrict__ in, int64_t ldw,
                                                               int nwr, int H, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int G = nwr >> 2;                                   // 4-word groups per image row
  const int nbands = (H + MED_MR - 1) / MED_MR;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = tid < G * nbands;
  const int g = act ? tid % G : 0, band = act ? tid / G : 0;
  const int y0 = band * MED_MR;
  const int64_t t = blockIdx.y;
  const uint32_t* f = in + t * ldw;
  uint32_t* o = out + t * ldw;
  // one image row y of this thread's column group: 4 words + the word before / after
  auto load_row = [&](int y, uint32_t (&c)[4], uint32_t& lw, uint32_t& rw) {
    const bool ok = act && y >= 0 && y < H;
    const int64_t q = (int64_t)y * nwr + 4 * g;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (ok) v = __ldg(reinterpret_cast<const uint4*>(f + q));
    c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
    lw = __shfl_up_sync(0xffffffffu, v.w, 1);
    rw = __shfl_down_sync(0xffffffffu, v.x, 1);
    if (lane == 0) lw = (ok && g > 0) ? __ldg(f + q - 1) : 0u;
    if (lane == 31) rw = (ok && g < G - 1) ? __ldg(f + q + 4) : 0u;
  };
  // (measured at 1080p x 500: a 3-row sliding window 0.071 ms; every row's loads issued
  // first 0.103 ms (MR = 8) / 0.089 ms (MR = 4); MR = 16 0.077 ms; the generic kernel 0.168 ms)
  uint32_t c[3][4], lw[3], rw[3];
  load_row(y0 - 1, c[0], lw[0], rw[0]);
  load_row(y0, c[1], lw[1], rw[1]);
#pragma unroll
  for (int i = 0; i < MED_MR; ++i) {
    const int y = y0 + i;
    load_row(y + 1, c[(i + 2) % 3], lw[(i + 2) % 3], rw[(i + 2) % 3]);
    if (act && y < H) {
      uint32_t res[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t x[9];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int rr = (i + d) % 3;                        // rows y - 1, y, y + 1
          const uint32_t cc = c[rr][u];
          const uint32_t l = (u == 0) ? (g == 0 ? 0u : lw[rr]) : c[rr][u - 1];
          const uint32_t r = (u == 3) ? (g == G - 1 ? 0u : rw[rr]) : c[rr][u + 1];
          x[3 * d + 0] = (cc << 1) | (l >> 31);              // pixel x - 1
          x[3 * d + 1] = cc;
          x[3 * d + 2] = (cc >> 1) | (r << 31);              // pixel x + 1
        }
        uint32_t s1, c1, s2, c2, s3, c3, s4, c4, s5, c5;
        fa(x[0], x[1], x[2], s1, c1);
        fa(x[3], x[4], x[5], s2, c2);
        fa(x[6], x[7], x[8], s3, c3);
        fa(s1, s2, s3, s4, c4);
        fa(c1, c2, c3, s5, c5);
        const uint32_t b1 = s5 ^ c4, c6 = s5 & c4;
        const uint32_t b2 = c5 ^ c6, b3 = c5 & c6;
        res[u] = b3 | (b2 & (b1 | s4));
      }
      *reinterpret_cast<uint4*>(o + (int64_t)y * nwr + 4 * g) = make_uint4(res[0], res[1], res[2], res[3]);
    }
  }
}

cudaError_t launch_mask_median3(const uint32_t* in, int64_t ldw, int64_t W, int64_t H, int64_t m, uint32_t* out,
                                cudaStream_t st) {
  if (W * H >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
  if (W % 128 == 0 && ldw % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0 && !getenv("CDMD_MEDIAN_GENERIC")) {
    const int nwr = (int)(W / 32);
    const int64_t threads = (int64_t)(nwr / 4) * ceil_div(H, MED_MR);
    dim3 grid((unsigned)ceil_div(threads, 256), (unsigned)m);
    note_launch();
    mask_median3_w32_kernel<<<grid, 256, 0, st>>>(in, ldw, nwr, (int)H, out);
    return cudaGetLastError();
  }
  const int64_t nw = (W * H + 31) >> 5;
  static int mw = -1;   // words per thread (CDMD_MEDIAN_MW: 1, 2, 4 or 8)
  if (mw < 0) {
    const char* e = getenv("CDMD_MEDIAN_MW");
    mw = e ? atoi(e) : 8;   // measured at 1080p x 500: 1 / 2 / 4 / 8 -> 0.29 / 0.22 / 0.171 / 0.167 ms
    if (mw != 1 && mw != 2 && mw != 4 && mw != 8) mw = 8;
  }
  dim3 grid((unsigned)ceil_div(ceil_div(nw, mw), 256), (unsigned)m);
  note_launch();
  switch (mw) {
    case 1: mask_median3_kernel<1><<<grid, 256, 0, st>>>(in, ldw, (int)W, (int)H, out); break;
    case 4: mask_median3_kernel<4><<<grid, 256, 0, st>>>(in, ldw, (int)W, (int)H, out); break;
    case 2: mask_median3_kernel<2><<<grid, 256, 0, st>>>(in, ldw, (int)W, (int)H, out); break;
    default: mask_median3_kernel<8><<<grid, 256, 0, st>>>(in, ldw, (int)W, (int)H, out); break;
  }
  return cudaGetLastError();
}

}  // namespace cdmd
