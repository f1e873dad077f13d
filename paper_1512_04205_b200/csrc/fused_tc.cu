// fused_tc.cu — N11, the fused single pass: modes of the OMP
// support, dynamic background, residual, threshold and bit-pack from ONE read of X.
//
// "The computation of the full modes Phi ... remain[s] the only computational expensive
// step ... embarrassingly parallel".  The background (Eq. DMDTerms)
// needs only the n_coef folded columns of Phi the support touches, Phi_F = X' M_F
// (Eq. cDMDModes P:318-321 restricted to those columns), so a CTA that holds a 128-pixel
// slab of X (all m frames, 64 KB at m = 500) computes Phi_F for its pixels on tensor
// cores and then thresholds the same bytes:
//   phase A  D1[px, l*16 + f] = sum_t X[t, px] Mq'[t, l, f]    tcgen05 kind::i8, M = 128
//            pixels (TMEM lanes), N = 4 limbs x 16 columns; Mq' = the int8 limbs of M for
//            the support columns shifted by one frame (Mq'[0] = 0, Mq'[t] = Mq[t - 1]), so
//            the X stages of frames 0..m-1 serve as X' = frames 1..m-1 (exact int32);
//   convert  one thread per pixel: the exact limb recombination (as cdmd_modes:
//            bit-identical Phi_F), split into three bf16 terms, written as the B operand
//            of phase B;
//   phase B  L[t, px] = sum_f H[t, f] Phi_F[px, f]  (six kind::f16 MMAs on the bf16 x 3
//            splits, M = 128 frames, N = 128 pixels, as foreground_tc.cu), fp32 in TMEM;
//   mask     one thread per frame, as foreground_tc.cu: d = x - L, t = d^2 - tau'^2
//            (tau'^2 the float above tau^2), the sign bits funnel-shifted into the word
//            (strict >, Eq. thres).
// X is read from HBM once; the full Phi is never written (Alg. 1's Phi output is
// cdmd_modes' job).  The X stages of a tile stay resident from phase A to the mask,
// two tiles in flight (8 stages of 16 KB at m <= 512).  Warp roles: 0 TMA producer,
// 1 TMEM owner + phase A issuer, 2-5 convert, 6-13 mask, 14 phase B issuer; the
// producer starts loading while the other warps build the resident operands.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

// fused_fg_kernel<true> (static background) ends its per-tile loop body with `continue`
// before the dynamic path: "loop is not reachable" there is expected
#pragma nv_diag_suppress 128

namespace cdmd {

constexpr int FU_BM = 128;                 // pixels per tile (phase A M, phase B N)
constexpr int FU_BK = 128;                 // frames per stage (phase B M)
constexpr int FU_STAGE = FU_BM * FU_BK;    // 16 KB of X per stage
constexpr int FU_NC = 16;                  // folded support columns (n_coef <= 16)
constexpr int FU_NA = CDMD_LIMBS * FU_NC;  // phase A N
constexpr int FU_MASK_WARPS = 8;         // 4 TMEM lane quarters x 2 slices of 64 pixels
constexpr int FU_PW = FU_BM / (FU_MASK_WARPS / 4);   // pixels per mask warp
constexpr int FU_NW = FU_PW / 32;          // mask words per thread per stage
constexpr int FU_MASK_WARP0 = 6;           // warps 6..13: quarters (warp % 4) x 2 pixel slices
constexpr int FU_BWARP = FU_MASK_WARP0 + FU_MASK_WARPS;   // phase B issuer (warp 14)
constexpr int FU_THREADS = 32 * (FU_BWARP + 1);
constexpr int FU_MAX_FB = 4;               // m <= 512

__device__ __forceinline__ uint32_t fu_km_off(int r, int c, int KP) {
  return (uint32_t)((r >> 3) * (16 * KP) + c * 128 + (r & 7) * 16);
}
__device__ __forceinline__ uint64_t fu_desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ unsigned long long fu_sub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fu_fma2(unsigned long long a, unsigned long long b,
                                                      unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__device__ __forceinline__ unsigned long long fu_add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 32 mask bits of one frame (as foreground_tc.cu's mask32): the uint8 pixel becomes an
// exact float through 2^23 + x (byte permute into the mantissa) minus 2^23, d = x - L,
// t = d^2 - tau'^2 with tau'^2 the float above tau^2 (t >= 0 exactly when |d| > tau),
// the sign bit of t funnel-shifted into the word, complemented at the end.
__device__ __forceinline__ uint32_t fu_mask32(const uint32_t (&xw)[8], const uint32_t (&L)[32],
                                              unsigned long long ntau2) {
  const unsigned long long bias = 0xCB000000CB000000ull;   // (-2^23, -2^23)
  uint32_t word = 0;
#pragma unroll
  for (int i = 30; i >= 0; i -= 2) {
    const uint32_t a = __byte_perm(xw[i >> 2], 0x4B000000u, 0x7540u + (i & 3));
    const uint32_t b = __byte_perm(xw[i >> 2], 0x4B000000u, 0x7540u + ((i + 1) & 3));
    const unsigned long long x2 = fu_add2(((unsigned long long)b << 32) | a, bias);
    const unsigned long long l2 = (unsigned long long)L[i] | ((unsigned long long)L[i + 1] << 32);
    const unsigned long long d2 = fu_sub2(x2, l2);
    const unsigned long long t2 = fu_fma2(d2, d2, ntau2);
    word = __funnelshift_l((uint32_t)(t2 >> 32), word, 1);
    word = __funnelshift_l((uint32_t)t2, word, 1);
  }
  return ~word;
}

// ---- the fused 3x3 median post-filter (Fig. 7; reading R22: 3x3, zero padding)
// (a) After the 8 mask warps wrote a tile's raw mask words, the tile counts towards its
//     image rows y-1, y, y+1 (release atomics after a barrier: the CTA's words first).
// (b) Once a CTA's tiles are exhausted, its convert, mask and phase-B warps filter
//     (image row, 32-frame block) tasks claimed from a second counter in row order: each
//     waits (acquire) until the rows y-1, y, y+1 of its row are complete, then consecutive threads take
//     8-word runs of one frame row (all 30 loads of a run in flight), the neighbour bits by
//     one-bit shifts across adjacent words (zero outside the frame), and the bit-sliced
//     carry-save count "at least 5 of 9", as median3.cu.  Rows are filtered while other
//     CTAs still process tiles.
__device__ __forceinline__ void fu_fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& co) {
  s = a ^ b ^ c;
  co = (a & b) | (a & c) | (b & c);
}

__device__ __forceinline__ void fu_count_tile(int tile, int H, int ncw, int* cnt, int mw, int lane) {
  asm volatile("bar.sync 2, 256;" ::: "memory");   // every mask thread's raw words of the tile are written
  if (mw == 0 && lane < 3) {
    const int yy = tile / ncw + lane - 1;
    if (yy >= 0 && yy < H)
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt + yy) : "memory");
  }
}

// phase (b): nthr threads (tid 0 .. nthr-1) of warps 2..14, named barrier 3
__device__ __noinline__ void fu_median_rows(int64_t m, int64_t ldw, int W, int H, int ncw, const uint32_t* raw,
                                            uint32_t* out, int* cnt, int* rowq, int tid, int nthr, int& rowsh) {
  const int nwr = W >> 5;                          // words per image row
  constexpr int MT = 8;                            // output words per run
  const int tpr = (nwr + MT - 1) / MT;             // runs per frame row
  constexpr int FBT = 32;                          // frames per task
  const int nfbt = (int)((m + FBT - 1) / FBT);
  for (;;) {
    if (tid == 0) {
      const int task = atomicAdd(rowq, 1);         // tasks in row order: (row, frame block)
      const int Y = task / nfbt;
      rowsh = task;
      if (Y < H) {   // wait until rows Y-1, Y, Y+1 are complete
        for (int d = -1; d <= 1; ++d) {
          const int yy = Y + d;
          if (yy < 0 || yy >= H) continue;
          const int need = ncw * ((yy > 0) + 1 + (yy < H - 1));
          int c;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(c) : "l"(cnt + yy) : "memory");
            if (c >= need) break;
            __nanosleep(256);
          }
        }
      }
    }
    asm volatile("bar.sync 3, %0;" ::"r"(nthr) : "memory");
    const int task = rowsh;
    asm volatile("bar.sync 3, %0;" ::"r"(nthr) : "memory");
    const int Y = task / nfbt;
    if (Y >= H) break;
    const int t0 = (task - Y * nfbt) * FBT;
    const int nt = (int)(m - t0 < FBT ? m - t0 : FBT);
    const int total = nt * tpr;
    for (int idx = tid; idx < total; idx += nthr) {
      const int t = t0 + idx / tpr, w0 = (idx % tpr) * MT;
      const uint32_t* rt = raw + (int64_t)t * ldw;
      uint32_t v[3][MT + 2];   // words w0 - 1 .. w0 + MT of rows Y-1, Y, Y+1
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int yy = Y + d - 1;
        const bool rowok = yy >= 0 && yy < H;
        const uint32_t* rw = rt + (int64_t)(rowok ? yy : 0) * nwr;
#pragma unroll
        for (int u = 0; u < MT + 2; ++u) {
          const int w = w0 + u - 1;
          v[d][u] = (rowok && w >= 0 && w < nwr) ? __ldcg(rw + w) : 0u;
        }
      }
      uint32_t* ot = out + (int64_t)t * ldw + (int64_t)Y * nwr;
#pragma unroll
      for (int u = 0; u < MT; ++u) {
        if (w0 + u >= nwr) break;
        uint32_t x[9];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const uint32_t a = v[d][u], b = v[d][u + 1], c = v[d][u + 2];
          x[3 * d + 0] = (b << 1) | (a >> 31);   // pixel x - 1
          x[3 * d + 1] = b;
          x[3 * d + 2] = (b >> 1) | (c << 31);   // pixel x + 1
        }
        uint32_t s1, c1, s2, c2, s3, c3, s4, c4, s5, c5;
        fu_fa(x[0], x[1], x[2], s1, c1);
        fu_fa(x[3], x[4], x[5], s2, c2);
        fu_fa(x[6], x[7], x[8], s3, c3);
        fu_fa(s1, s2, s3, s4, c4);
        fu_fa(c1, c2, c3, s5, c5);
        const uint32_t b1 = s5 ^ c4, c6 = s5 & c4;
        const uint32_t b2 = c5 ^ c6, b3 = c5 & c6;
        ot[w0 + u] = b3 | (b2 & (b1 | s4));
      }
    }
  }
}

// phase (b) for word-aligned rows (W % 128 == 0, 16-B aligned masks, ldw % 4 == 0): tasks
// are bands of FU_MB image rows over ALL frames (one task per CTA at 1080p), so the
// claim / wait / barrier overhead is paid ~once per CTA; within a band a thread takes
// (4-word group g, frame t) items and slides a three-row window down the band's rows,
// one coalesced 16-B load per row, the side words from the neighbouring lanes (as
// median3.cu's word-aligned kernel; the words across an image-row boundary are zero).
constexpr int FU_MB = 8;
__device__ __noinline__ void fu_median_bands(int64_t m, int64_t ldw, int W, int H, int ncw, const uint32_t* raw,
                                             uint32_t* out, int* cnt, int* rowq, int tid, int nthr, int& rowsh) {
  const int nwr = W >> 5, G = nwr >> 2;
  const int nb = (H + FU_MB - 1) / FU_MB;
  const int lane = tid & 31;
  for (;;) {
    if (tid == 0) {
      const int b = atomicAdd(rowq, 1);
      rowsh = b;
      if (b < nb) {   // wait until every row of the band (and so its neighbours) is complete
        for (int yy = b * FU_MB; yy < min(H, (b + 1) * FU_MB); ++yy) {
          const int need = ncw * ((yy > 0) + 1 + (yy < H - 1));
          int c;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(c) : "l"(cnt + yy) : "memory");
            if (c >= need) break;
            __nanosleep(256);
          }
        }
      }
    }
    asm volatile("bar.sync 3, %0;" ::"r"(nthr) : "memory");
    const int b = rowsh;
    asm volatile("bar.sync 3, %0;" ::"r"(nthr) : "memory");
    if (b >= nb) break;
    const int y0 = b * FU_MB;
    const int64_t items = (int64_t)G * m;
    for (int64_t i0 = 0; i0 < items; i0 += nthr) {       // warp-uniform trip count (shuffles)
      const int64_t it = i0 + tid;
      const bool act = it < items;
      const int g = act ? (int)(it % G) : 0;
      const int64_t t = act ? it / G : 0;
      const uint32_t* f = raw + t * ldw;
      uint32_t* o = out + t * ldw;
      auto load_row = [&](int y, uint32_t (&c)[4], uint32_t& lw, uint32_t& rw) {
        const bool ok = act && y >= 0 && y < H;
        const int64_t q = (int64_t)y * nwr + 4 * g;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (ok) v = __ldcg(reinterpret_cast<const uint4*>(f + q));
        c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
        lw = __shfl_up_sync(0xffffffffu, v.w, 1);
        rw = __shfl_down_sync(0xffffffffu, v.x, 1);
        if (lane == 0) lw = (ok && g > 0) ? __ldcg(f + q - 1) : 0u;
        if (lane == 31) rw = (ok && g < G - 1) ? __ldcg(f + q + 4) : 0u;
      };
      // all FU_MB + 2 rows in flight at once: one CTA per SM runs this trailing phase, so
      // the loads of a thread are what hides the L2 latency
      uint32_t c[FU_MB + 2][4], lw[FU_MB + 2], rw[FU_MB + 2];
#pragma unroll
      for (int i = 0; i < FU_MB + 2; ++i) load_row(y0 - 1 + i, c[i], lw[i], rw[i]);
#pragma unroll
      for (int i = 0; i < FU_MB; ++i) {
        const int y = y0 + i;
        if (act && y < H) {
          uint32_t res[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint32_t x[9];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const int rr = i + d;
              const uint32_t cc = c[rr][u];
              const uint32_t l = (u == 0) ? (g == 0 ? 0u : lw[rr]) : c[rr][u - 1];
              const uint32_t r = (u == 3) ? (g == G - 1 ? 0u : rw[rr]) : c[rr][u + 1];
              x[3 * d + 0] = (cc << 1) | (l >> 31);
              x[3 * d + 1] = cc;
              x[3 * d + 2] = (cc >> 1) | (r << 31);
            }
            uint32_t s1, c1, s2, c2, s3, c3, s4, c4, s5, c5;
            fu_fa(x[0], x[1], x[2], s1, c1);
            fu_fa(x[3], x[4], x[5], s2, c2);
            fu_fa(x[6], x[7], x[8], s3, c3);
            fu_fa(s1, s2, s3, s4, c4);
            fu_fa(c1, c2, c3, s5, c5);
            const uint32_t b1 = s5 ^ c4, c6 = s5 & c4;
            const uint32_t b2 = c5 ^ c6, b3 = c5 & c6;
            res[u] = b3 | (b2 & (b1 | s4));
          }
          *reinterpret_cast<uint4*>(o + (int64_t)y * nwr + 4 * g) = make_uint4(res[0], res[1], res[2], res[3]);
        }
      }
    }
  }
}

// STATIC (template ST): no phase B; the convert warps reduce Phi_F of each
// pixel to its static background L = sum_f Phi_F[f] c_f(1) (the fmaf order of
// foreground.cu's static kernel) and the integer bounds x > floor(L + tau), x <
// ceil(L - tau) (bytes, plus an "always" bit); the mask warps compare four pixels per
// byte-SIMD instruction against them.
__device__ __forceinline__ uint32_t fu_movemask4(uint32_t v) {  // bytes 0x00/0xFF -> 4 bits
  return ((v & 0x01010101u) * 0x10204080u) >> 28;
}

template <bool ST>
__global__ void __launch_bounds__(FU_THREADS, 1) fused_fg_kernel(
    const __grid_constant__ CUtensorMap mapX, int64_t n_local, int64_t m, int nfb, int64_t mpad, int kpad,
    const int8_t* __restrict__ Mq, const double* __restrict__ Mq_scale, const float* __restrict__ coef,
    const int32_t* __restrict__ coef_col, int n_coef, float tau, uint32_t* __restrict__ mask, int64_t ldw,
    int num_tiles, int stages, int* __restrict__ tile_counter, int imgW, int imgH, int ncw,
    uint32_t* __restrict__ medout, int* __restrict__ medcnt) {
  // imgW > 0: the 3x3 median post-filter is fused (Fig. 7): tile = (image row y,
  // 128-pixel chunk c) of whole frames (imgW % 32 == 0), the raw mask goes to `mask`
  // (workspace) and the filtered one to `medout`; a tile's median is computed by the
  // CTA that completes the last of its (up to) nine neighbour tiles (counters medcnt).
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  const int mA = nfb * FU_BK;
  constexpr int PART_B = FU_BM * FU_NC * 2;   // one bf16 part of Phi_F (phase B operand)
  const int PART_A = mA * FU_NC * 2;           // one bf16 part of H
  uint8_t* sX = smem;                                            // stages x 16 KB, SW128
  uint8_t* sQ = sX + (size_t)stages * FU_STAGE;                  // Mq' panels: nfb x (64 rows x 128 B), SW128
  uint8_t* sH = sQ + (size_t)nfb * FU_NA * FU_BK;                // H: 3 parts x mA x 16 bf16
  uint8_t* sP = sH + 3 * (size_t)PART_A;                         // Phi_F: 3 parts x 128 x 16 bf16
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sP + 3 * PART_B);
  uint64_t* xempty = xfull + stages;
  uint64_t* afull = xempty + stages;    // [2] phase A accumulator ready
  uint64_t* aempty = afull + 2;         // [2] phase A accumulator drained (convert warps)
  uint64_t* pfull = aempty + 2;         // Phi_F operand written (convert warps)
  uint64_t* pempty = pfull + 1;         // Phi_F operand consumed (phase B MMAs done)
  uint64_t* bfull = pempty + 1;         // [2] phase B accumulator ready
  uint64_t* bempty = bfull + 2;         // [2] phase B accumulator drained (mask warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 2);
  __shared__ int tq_id[tc::TQ_N];
  __shared__ uint64_t tq_bar[2 * tc::TQ_N];
  __shared__ float sScale[FU_NC];
  __shared__ float sC0[FU_NC];                              // ST: c_f(1)
  __shared__ __align__(16) uint8_t sHi[2][FU_BM], sLo[2][FU_BM];   // ST: per-pixel byte bounds, by tile parity
  __shared__ uint32_t sAlw[2][FU_BM / 32];                  // ST: pixels outside [0, 255] +- tau: always set
  __shared__ uint64_t bnd_full[2], bnd_empty[2];
  __shared__ int rowsh;                                     // median: the row being filtered
  const tc::TileQueue tq{tq_id, tq_bar, tq_bar + tc::TQ_N};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // first pixel and length of a tile
  auto tile_base = [&](int tile) -> int64_t {
    return imgW > 0 ? (int64_t)(tile / ncw) * imgW + (int64_t)(tile % ncw) * FU_BM : (int64_t)tile * FU_BM;
  };
  auto tile_len = [&](int tile) -> int {
    const int64_t rest = imgW > 0 ? (int64_t)imgW - (int64_t)(tile % ncw) * FU_BM : n_local - (int64_t)tile * FU_BM;
    return rest < FU_BM ? (int)rest : FU_BM;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], FU_MASK_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&afull[b], 1);
      tc::mbar_init(&aempty[b], 4);
      tc::mbar_init(&bfull[b], 1);
      tc::mbar_init(&bempty[b], FU_MASK_WARPS);
    }
    tc::mbar_init(pfull, 4);
    tc::mbar_init(pempty, 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&bnd_full[b], 4);
      tc::mbar_init(&bnd_empty[b], FU_MASK_WARPS);
    }
    tc::tq_init(tq, (ST ? 1 : 2) + 4 + FU_MASK_WARPS);   // A issuer, [B issuer,] convert, mask
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapX);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the TMA producer starts right away; every other warp builds the resident operands
  // (the shifted limbs Mq' and the split H) and meets the others at named barrier 1
  if (warp != 0) {
    const int ntb = blockDim.x - 32, t0 = threadIdx.x - 32;
    for (int f = t0; f < FU_NC; f += ntb) {
      sScale[f] = f < n_coef ? (float)Mq_scale[coef_col[f]] : 0.f;
      sC0[f] = f < n_coef ? coef[(int64_t)f * m] : 0.f;
    }
    const int nchunks = FU_NA * nfb * 8;          // 16-B chunks of Mq'
    for (int q = t0; q < nchunks; q += ntb) {
      const int row = q / (nfb * 8), rest = q % (nfb * 8);
      const int kb = rest >> 3, c = rest & 7;
      const int l = row / FU_NC, f = row % FU_NC;
      const int8_t* src = (f < n_coef) ? Mq + ((int64_t)l * kpad + coef_col[f]) * mpad : nullptr;
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const int64_t t = (int64_t)kb * FU_BK + c * 16 + b;    // frame of X (X' frame t - 1)
        const uint32_t v = (src && t >= 1 && t <= m - 1) ? (uint32_t)(uint8_t)__ldg(src + t - 1) : 0u;
        w[b >> 2] |= v << (8 * (b & 3));
      }
      *reinterpret_cast<uint4*>(sQ + (size_t)kb * FU_NA * FU_BK + row * 128 + ((c ^ (row & 7)) << 4)) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (int idx = t0; idx < (ST ? 0 : mA * FU_NC); idx += ntb) {
      const int t = idx / FU_NC, f = idx % FU_NC;
      const float v = (t < m && f < n_coef) ? coef[(int64_t)f * m + t] : 0.f;
      const __nv_bfloat16 a = __float2bfloat16_rn(v);
      const float r1 = v - __bfloat162float(a);
      const __nv_bfloat16 b = __float2bfloat16_rn(r1);
      const __nv_bfloat16 c = __float2bfloat16_rn(r1 - __bfloat162float(b));
      const uint32_t off = fu_km_off(t, f >> 3, FU_NC) + (f & 7) * 2;
      *reinterpret_cast<__nv_bfloat16*>(sH + off) = a;
      *reinterpret_cast<__nv_bfloat16*>(sH + PART_A + off) = b;
      *reinterpret_cast<__nv_bfloat16*>(sH + 2 * PART_A + off) = c;
    }
    tc::fence_proxy_async();   // generic-proxy smem writes (Mq', H) -> async proxy (MMA)
    asm volatile("bar.sync 1, %0;" ::"r"(ntb) : "memory");
  }
  // TMEM columns: phase A accumulators [0, 64) and [64, 128); phase B [128, 256), [256, 384)

  if (warp == 0) {
    if (lane == 0) {  // -------------------------------------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0;; ++k) {
        const int tile = tc::tq_publish(tq, k, tile_counter, num_tiles);
        if (tile < 0) break;
        for (int fb = 0; fb < nfb; ++fb) {
          tc::mbar_wait(&xempty[stage], phase ^ 1u);
          tc::mbar_arrive_expect_tx(&xfull[stage], FU_STAGE);
          tc::tma_load_2d(sX + (size_t)stage * FU_STAGE, &mapX, &xfull[stage], (int32_t)tile_base(tile), fb * FU_BK);
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // --------------------------------------------- MMA issuer
      constexpr uint32_t IDA = tc::idesc_i8(FU_BM, FU_NA, false, true, true, false);
      const uint32_t xBase = tc::smem_u32(sX), qBase = tc::smem_u32(sQ);
      int stage = 0;
      uint32_t phase = 0;
      for (int ti = 0;; ++ti) {   // phase A only: phase B has an issuer of its own
        if (tc::tq_take(tq, ti) < 0) break;
        const int ab = ti & 1;
        tc::mbar_wait(&aempty[ab], ((uint32_t)(ti >> 1) & 1u) ^ 1u);
        tc::fence_after();
        const uint32_t d = tmem_base + (uint32_t)(ab * FU_NA);
        for (int fb = 0; fb < nfb; ++fb) {
          tc::mbar_wait(&xfull[stage], phase);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < FU_BK / 32; ++kk) {
            const uint64_t ad = tc::smem_desc_sw128(xBase + stage * FU_STAGE + kk * 32 * 128, FU_STAGE, 1024);
            const uint64_t bd = tc::smem_desc_sw128(qBase + fb * FU_NA * FU_BK + kk * 32, 0, 1024);
            tc::mma_i8(d, ad, bd, IDA, (fb | kk) != 0);
          }
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
        tc::mma_commit(&afull[ab]);
      }
    }
  } else if (warp == FU_BWARP) {
    if (lane == 0 && !ST) {  // ------------------------------------ phase B issuer
      constexpr uint32_t IDB = tc::idesc_f16(FU_BK, FU_BM, true, true, false, false);
      const uint32_t hBase = tc::smem_u32(sH), pBase = tc::smem_u32(sP);
      int itB = 0;
      for (int u = 0;; ++u) {
        if (tc::tq_take(tq, u) < 0) break;
        tc::mbar_wait(pfull, (uint32_t)u & 1u);   // Phi_F of tile u split into sP
        tc::fence_after();
        for (int fb = 0; fb < nfb; ++fb, ++itB) {
          const int bb = itB & 1;
          tc::mbar_wait(&bempty[bb], ((uint32_t)(itB >> 1) & 1u) ^ 1u);
          tc::fence_after();
          const uint32_t d = tmem_base + 128u + (uint32_t)(bb * FU_BM);
          int first = 1;
#pragma unroll
          for (int pi = 0; pi < 3; ++pi)
#pragma unroll
            for (int pj = 0; pj < 3 - pi; ++pj) {
              const uint64_t ad = fu_desc_nosw(hBase + pi * PART_A + fb * (FU_BK / 8) * (16 * FU_NC), 128, 16 * FU_NC);
              const uint64_t bd = fu_desc_nosw(pBase + pj * PART_B, 128, 16 * FU_NC);
              tc::mma_f16(d, ad, bd, IDB, first ? 0u : 1u);
              first = 0;
            }
          tc::mma_commit(&bfull[bb]);
        }
        tc::mma_commit(pempty);
      }
    }
  } else if (warp < FU_MASK_WARP0) {  // ------------------------------ convert (2..5)
    const int q = warp & 3;
    const int row = q * 32 + lane;              // pixel of the tile (TMEM lane)
    for (int ti = 0;; ++ti) {
      const int tile = tc::tq_take_warp(tq, ti);
      if (tile < 0) break;
      const int ab = ti & 1;
      tc::mbar_wait(&afull[ab], (uint32_t)(ti >> 1) & 1u);
      tc::fence_after();
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * FU_NA);
      uint32_t h0[8], h1[8], h2[8];
      float phif[FU_NC];
#pragma unroll
      for (int half = 0; half < 2; ++half) {   // columns 8 half .. 8 half + 7
        uint32_t r0[8], r1[8], r2[8], r3[8];
        tc::tmem_ld8(ta + 0 * FU_NC + 8 * half, r0);
        tc::tmem_ld8(ta + 1 * FU_NC + 8 * half, r1);
        tc::tmem_ld8(ta + 2 * FU_NC + 8 * half, r2);
        tc::tmem_ld8(ta + 3 * FU_NC + 8 * half, r3);
        tc::tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < 8; g += 2) {
          const int f = 8 * half + g;
          const float v0 = combine_limbs(r0[g], r1[g], r2[g], r3[g], sScale[f]);
          const float v1 = combine_limbs(r0[g + 1], r1[g + 1], r2[g + 1], r3[g + 1], sScale[f + 1]);
          phif[f] = v0;
          phif[f + 1] = v1;
          const __nv_bfloat162 a = __floats2bfloat162_rn(v0, v1);
          const float2 af = __bfloat1622float2(a);
          const float e0 = v0 - af.x, e1 = v1 - af.y;
          const __nv_bfloat162 b = __floats2bfloat162_rn(e0, e1);
          const float2 bf = __bfloat1622float2(b);
          const __nv_bfloat162 c = __floats2bfloat162_rn(e0 - bf.x, e1 - bf.y);
          h0[f / 2] = *reinterpret_cast<const uint32_t*>(&a);
          h1[f / 2] = *reinterpret_cast<const uint32_t*>(&b);
          h2[f / 2] = *reinterpret_cast<const uint32_t*>(&c);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&aempty[ab]);
      if (ST) {   // static background and integer bounds of pixel `row`
        float L = 0.f;
#pragma unroll
        for (int f = 0; f < FU_NC; ++f)
          if (f < n_coef) L = fmaf(phif[f], sC0[f], L);   // the static kernel's order
        const int bb = ti & 1;
        tc::mbar_wait(&bnd_empty[bb], ((uint32_t)(ti >> 1) & 1u) ^ 1u);
        const float fh = floorf(L + tau), fl = ceilf(L - tau);
        const bool alw = row < tile_len(tile) && (fh < 0.f || fl > 255.f);
        sHi[bb][row] = (uint8_t)fminf(fmaxf(fh, 0.f), 255.f);
        sLo[bb][row] = (uint8_t)fminf(fmaxf(fl, 0.f), 255.f);
        const uint32_t bal = __ballot_sync(0xffffffffu, alw);
        if (lane == 0) sAlw[bb][q] = bal;
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bnd_full[bb]);
        continue;
      }
      tc::mbar_wait(pempty, ((uint32_t)ti & 1u) ^ 1u);   // phase B of the previous tile is done with sP
#pragma unroll
      for (int c8 = 0; c8 < 2; ++c8) {
        const uint32_t off = fu_km_off(row, c8, FU_NC);
        *reinterpret_cast<uint4*>(sP + off) = make_uint4(h0[4 * c8], h0[4 * c8 + 1], h0[4 * c8 + 2], h0[4 * c8 + 3]);
        *reinterpret_cast<uint4*>(sP + PART_B + off) =
            make_uint4(h1[4 * c8], h1[4 * c8 + 1], h1[4 * c8 + 2], h1[4 * c8 + 3]);
        *reinterpret_cast<uint4*>(sP + 2 * PART_B + off) =
            make_uint4(h2[4 * c8], h2[4 * c8 + 1], h2[4 * c8 + 2], h2[4 * c8 + 3]);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(pfull);
    }
  } else if (warp < FU_BWARP) {  // ---------------------------------------- mask
    const int mw = warp - FU_MASK_WARP0;
    const int q = warp & 3;                // TMEM lane quarter: frames 32q .. 32q + 31 of a stage
    const int sl = mw >> 2;                // pixels [FU_PW sl, FU_PW (sl + 1)) of the tile
    const int r = q * 32 + lane;           // frame within the stage (TMEM lane)
    const float nt2 = -__uint_as_float(__float_as_uint(tau * tau) + 1u);   // -(next float above tau^2)
    const unsigned long long ntau2 =
        (unsigned long long)__float_as_uint(nt2) | ((unsigned long long)__float_as_uint(nt2) << 32);
    int stage = 0;
    uint32_t phase = 0;
    int itB = 0;
    for (int ti = 0;; ++ti) {
      const int tile = tc::tq_take_warp(tq, ti);
      if (tile < 0) break;
      const int64_t w0 = (tile_base(tile) + sl * FU_PW) >> 5;   // this thread's first mask word
      const int tlen = tile_len(tile);                             // pixels of the tile (multiple of 32 unless ragged)
      if (ST) {   // ------------------------------ static: byte bounds, all frames of the tile
        const int tb = ti & 1;
        tc::mbar_wait(&bnd_full[tb], (uint32_t)(ti >> 1) & 1u);
        uint32_t hiw[FU_NW][8], low[FU_NW][8], alw[FU_NW], valid[FU_NW];
#pragma unroll
        for (int w = 0; w < FU_NW; ++w) {
          const int p0 = sl * FU_PW + 32 * w;
          const uint4 h0 = *reinterpret_cast<const uint4*>(&sHi[tb][p0]);
          const uint4 h1 = *reinterpret_cast<const uint4*>(&sHi[tb][p0 + 16]);
          const uint4 l0 = *reinterpret_cast<const uint4*>(&sLo[tb][p0]);
          const uint4 l1 = *reinterpret_cast<const uint4*>(&sLo[tb][p0 + 16]);
          hiw[w][0] = h0.x; hiw[w][1] = h0.y; hiw[w][2] = h0.z; hiw[w][3] = h0.w;
          hiw[w][4] = h1.x; hiw[w][5] = h1.y; hiw[w][6] = h1.z; hiw[w][7] = h1.w;
          low[w][0] = l0.x; low[w][1] = l0.y; low[w][2] = l0.z; low[w][3] = l0.w;
          low[w][4] = l1.x; low[w][5] = l1.y; low[w][6] = l1.z; low[w][7] = l1.w;
          alw[w] = sAlw[tb][p0 >> 5];
          valid[w] = (p0 + 32 <= tlen) ? 0xffffffffu : (p0 < tlen ? ((1u << (tlen - p0)) - 1u) : 0u);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bnd_empty[tb]);
        for (int fb = 0; fb < nfb; ++fb) {
          tc::mbar_wait(&xfull[stage], phase);
          const uint8_t* rowp = sX + (size_t)stage * FU_STAGE + r * 128;
          uint32_t words[FU_NW];
#pragma unroll
          for (int w = 0; w < FU_NW; ++w) {
            const int c = (sl * FU_PW + 32 * w) >> 4;
            const uint4 a = *reinterpret_cast<const uint4*>(rowp + ((c ^ (r & 7)) << 4));
            const uint4 b = *reinterpret_cast<const uint4*>(rowp + (((c + 1) ^ (r & 7)) << 4));
            const uint32_t xw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint32_t word = alw[w];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              word |= fu_movemask4(__vcmpgtu4(xw[u], hiw[w][u]) | __vcmpltu4(xw[u], low[w][u])) << (4 * u);
            words[w] = word & valid[w];
          }
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&xempty[stage]);
          if (++stage == stages) { stage = 0; phase ^= 1u; }
          const int64_t t = (int64_t)fb * FU_BK + r;
          if (t < m) {
            uint32_t* dst = mask + t * ldw + w0;
#pragma unroll
            for (int w = 0; w < FU_NW; ++w)
              if (sl * FU_PW + 32 * w < tlen) dst[w] = words[w];
          }
        }
        if (imgW > 0) fu_count_tile(tile, imgH, ncw, medcnt, mw, lane);
        continue;
      }
      for (int fb = 0; fb < nfb; ++fb, ++itB) {
        const int bb = itB & 1;
        tc::mbar_wait(&bfull[bb], (uint32_t)(itB >> 1) & 1u);
        tc::mbar_wait(&xfull[stage], phase);
        tc::fence_after();
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + 128u + (uint32_t)(bb * FU_BM) + sl * FU_PW;
        const uint8_t* rowp = sX + (size_t)stage * FU_STAGE + r * 128;
        uint32_t words[FU_NW];
        uint32_t La[32], Lb[32];
        tc::tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(&La[0]));
        tc::tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&La[16]));
#pragma unroll
        for (int w = 0; w < FU_NW; ++w) {
          uint32_t (&L)[32] = (w & 1) ? Lb : La;
          uint32_t (&Ln)[32] = (w & 1) ? La : Lb;
          const int c = (sl * FU_PW + 32 * w) >> 4;    // 16-B chunk of the 128-B frame row
          const uint4 a = *reinterpret_cast<const uint4*>(rowp + ((c ^ (r & 7)) << 4));
          const uint4 b = *reinterpret_cast<const uint4*>(rowp + (((c + 1) ^ (r & 7)) << 4));
          const uint32_t xw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          tc::tmem_ld_wait();
          if (w + 1 < FU_NW) {
            tc::tmem_ld16(ta + 32 * (w + 1), *reinterpret_cast<uint32_t(*)[16]>(&Ln[0]));
            tc::tmem_ld16(ta + 32 * (w + 1) + 16, *reinterpret_cast<uint32_t(*)[16]>(&Ln[16]));
          }
          words[w] = fu_mask32(xw, L, ntau2);
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&bempty[bb]);
          tc::mbar_arrive(&xempty[stage]);
        }
        if (++stage == stages) { stage = 0; phase ^= 1u; }
        const int64_t t = (int64_t)fb * FU_BK + r;
        if (t < m) {
          uint32_t* dst = mask + t * ldw + w0;
          if (FU_NW == 2 && ((ldw | w0) & 1) == 0 && sl * FU_PW + 32 < tlen) {   // 8-B aligned pair
            *reinterpret_cast<uint2*>(dst) = make_uint2(words[0], words[FU_NW - 1]);
          } else {
#pragma unroll
            for (int w = 0; w < FU_NW; ++w)
              if (sl * FU_PW + 32 * w < tlen) dst[w] = words[w];
          }
        }
      }
      if (imgW > 0) fu_count_tile(tile, imgH, ncw, medcnt, mw, lane);
    }
  }
  // phase (b): warps 2 .. FU_BWARP filter whole image rows (median fused)
  if (imgW > 0 && warp >= 2)
    if (imgW % 128 == 0 && ldw % 4 == 0 && ((reinterpret_cast<uintptr_t>(mask) | reinterpret_cast<uintptr_t>(medout)) & 15) == 0)
      fu_median_bands(m, ldw, imgW, imgH, ncw, mask, medout, medcnt, medcnt + imgH, threadIdx.x - 64,
                      blockDim.x - 64, rowsh);
    else
      fu_median_rows(m, ldw, imgW, imgH, ncw, mask, medout, medcnt, medcnt + imgH, threadIdx.x - 64,
                   blockDim.x - 64, rowsh);
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 512);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 fu_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static size_t fu_smem_bytes(int nfb, int stages) {
  return 1024 + (size_t)stages * FU_STAGE + (size_t)nfb * FU_NA * FU_BK + 3 * (size_t)nfb * FU_BK * FU_NC * 2 +
         3 * (size_t)FU_BM * FU_NC * 2 + 256;
}

static int fu_stages(int nfb) {
  // two whole tiles resident (phase A of tile i + 1 overlaps the mask of tile i)
  int s = 2 * nfb;
  while (s > nfb && fu_smem_bytes(nfb, s) > 225 * 1024) --s;
  return s;
}

bool fused_supported(const cdmd_video& v, const cdmd_model& M, int mode) {
  if (mode != CDMD_BG_DYNAMIC && mode != CDMD_BG_STATIC) return false;
  if (M.n_coef < 1 || M.n_coef > FU_NC || !fu_encode_fn()) return false;
  const int nfb = (int)ceil_div(v.m, FU_BK);
  if (nfb > FU_MAX_FB || M.mpad > (int64_t)nfb * FU_BK) return false;
  return fu_smem_bytes(nfb, fu_stages(nfb)) <= 225 * 1024 && fu_stages(nfb) >= nfb + 1 && (v.ld % 16) == 0;
}

cudaError_t launch_fused_fg(const cdmd_video& v, const cdmd_model& M, int mode, float tau, uint32_t* mask,
                            int64_t ldw, int* tile_counter, cudaStream_t st) {
  return launch_fused_fg_median(v, M, mode, tau, mask, ldw, tile_counter, 0, 0, nullptr, nullptr, st);
}

cudaError_t launch_fused_fg_median(const cdmd_video& v, const cdmd_model& M, int mode, float tau, uint32_t* mask,
                                   int64_t ldw, int* tile_counter, int imgW, int imgH, uint32_t* medout, int* medcnt,
                                   cudaStream_t st) {
  auto kern = mode == CDMD_BG_STATIC ? fused_fg_kernel<true> : fused_fg_kernel<false>;
  const int nfb = (int)ceil_div(v.m, FU_BK);
  CUtensorMap mapX;
  cuuint64_t dims[2] = {(cuuint64_t)v.n_local, (cuuint64_t)v.m};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld};
  cuuint32_t box[2] = {FU_BM, FU_BK};
  cuuint32_t estr[2] = {1, 1};
  if (fu_encode_fn()(&mapX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int stages = fu_stages(nfb);
  const size_t smem = fu_smem_bytes(nfb, stages);
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ncw = imgW > 0 ? (int)ceil_div(imgW, FU_BM) : 0;
  const int num_tiles = imgW > 0 ? imgH * ncw : (int)ceil_div(v.n_local, FU_BM);
  const int pc = persistent_ctas(sms);
  const int grid = num_tiles < pc ? num_tiles : pc;
  e = cudaMemsetAsync(tile_counter, 0, sizeof(int), st);
  if (e == cudaSuccess && imgW > 0) e = cudaMemsetAsync(medcnt, 0, sizeof(int) * ((size_t)imgH + 1), st);
  if (e != cudaSuccess) return e;
  note_launch();
  kern<<<grid, FU_THREADS, smem, st>>>(mapX, v.n_local, v.m, nfb, M.mpad, M.kpad, M.Mq, M.Mq_scale,
                                                  M.coef, M.coef_col, M.n_coef, tau, mask, ldw, num_tiles, stages,
                                                  tile_counter, imgW, imgH, ncw, medout, medcnt);
  return cudaGetLastError();
}

}  // namespace cdmd
