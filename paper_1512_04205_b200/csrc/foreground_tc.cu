// foreground_tc.cu — fused dynamic background + residual + threshold + bit-pack on
// tcgen05 tensor cores (Eq. DMDTerms P:185-193 with Eq. thres).
//
// The dynamic background of a 256-pixel tile over a 128-frame unit is the rank-NC
// product L^T = H (128 frames x NC) . Phi_F^T (NC x 256 pixels) of the coefficient
// table h_f(t) = Re/Im of beta_p lambda_p^(t-1) and the folded support modes.  On
// CUDA cores that is NC FMAs per pixel-frame (ALU-bound above HBM speed); here it is
// six kind::f16 MMAs (M = 128 frames, N = 256 pixels) on bf16 three-term splits
//   H = A0 + A1 + A2,  Phi_F = B0 + B1 + B2  (24 significant bits each),
//   L^T ~= sum_{i + j <= 2} A_i B_j^T  accumulated in fp32 in TMEM,
// followed by an epilogue in which each thread owns one frame (TMEM lane) and reads
// 32 consecutive pixels' backgrounds (TMEM columns) and bytes (two 16-B loads from
// the SWIZZLE_128B TMA tile), builds the 32-bit mask word in registers (f32x2 packed
// subtractions) and stores whole words.  Persistent CTAs with a dynamic tile schedule
// (tc::TileQueue: tiles claimed from a counter); warp 0 TMA producer,
// warp 1 TMEM owner + MMA issuer, warps 2..17 epilogue (they also split Phi_F of the
// next tile into the B operand).  One read of X, one write of the mask.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

namespace cdmd {

constexpr int FG_BN = 256;          // pixels per tile (UMMA N, TMEM columns per buffer)
constexpr int FG_BM = 128;          // frames per unit (UMMA M, TMEM lanes)
constexpr int FG_XSTAGE = FG_BM * FG_BN;   // bytes of X per unit (two 128x128 SW128 boxes)
// epilogue warps EW (template): 4 TMEM lane quarters x EW/4 pixel slices of 1024/EW
// pixels; each thread builds 1024/EW/32 mask words per unit
#ifdef CDMD_ABLATIONS
#define FG_ABL(x) (x)
#else
#define FG_ABL(x) false
#endif

// no-swizzle K-major core-matrix layout: row r, 16-B chunk c at
// (r / 8) * SBO + c * 128 + (r % 8) * 16, SBO = 16 * KP
__device__ __forceinline__ uint32_t km_off(int r, int c, int KP) {
  return (uint32_t)((r >> 3) * (16 * KP) + c * 128 + (r & 7) * 16);
}

__device__ __forceinline__ void split3(float v, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  a = __float2bfloat16_rn(v);
  const float r1 = v - __bfloat162float(a);
  b = __float2bfloat16_rn(r1);
  c = __float2bfloat16_rn(r1 - __bfloat162float(b));
}

__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100); layout type 0 = SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// 32 mask bits of one frame: pixels of 8 byte-words xw (4 pixels each) against 32
// background values L; bit i = |x_i - L_i| > tau.  The uint8 pixel becomes an exact
// float through 2^23 + x (byte permute into the mantissa) minus 2^23, one packed
// f32x2 add per two pixels; d = x - L is one packed subtraction and t = d^2 - tau'^2
// one packed FMA, with tau'^2 the float just above tau^2 so that t >= 0 exactly when
// d^2 > tau^2 (strict >).  A funnel shift moves the sign bit of t into the word
// (pixels taken from 31 down to 0); the word is complemented once at the end.
__device__ __forceinline__ uint32_t mask32(const uint32_t (&xw)[8], const uint32_t (&L)[32], float tau) {
  const unsigned long long bias = f2pack(-8388608.0f, -8388608.0f);
  const float nt2 = -__uint_as_float(__float_as_uint(tau * tau) + 1u);   // -(next float above tau^2)
  const unsigned long long ntau2 = f2pack(nt2, nt2);
  uint32_t word = 0;
#pragma unroll
  for (int i = 30; i >= 0; i -= 2) {
    const uint32_t a = __byte_perm(xw[i >> 2], 0x4B000000u, 0x7540u + (i & 3));
    const uint32_t b = __byte_perm(xw[i >> 2], 0x4B000000u, 0x7540u + ((i + 1) & 3));
    const unsigned long long x2 = fadd2(((unsigned long long)b << 32) | a, bias);                  // exact x
    const unsigned long long l2 = (unsigned long long)L[i] | ((unsigned long long)L[i + 1] << 32);
    const unsigned long long d2 = fsub2(x2, l2);
    const unsigned long long t2 = ffma2(d2, d2, ntau2);
    word = __funnelshift_l((uint32_t)(t2 >> 32), word, 1);   // bit i + 1 (complemented)
    word = __funnelshift_l((uint32_t)t2, word, 1);           // bit i (complemented)
  }
  return ~word;
}

template <int KP, int EW>
__global__ void __launch_bounds__(32 * (2 + EW), 1) foreground_tc_kernel(
    const __grid_constant__ CUtensorMap mapX, int64_t n_local, int64_t m, int nfb,
    const float* __restrict__ Phi, int64_t ldphi, const float* __restrict__ coef,
    const int32_t* __restrict__ coef_col, int n_coef, float tau, uint32_t* __restrict__ mask,
    int64_t ldw, int num_tiles, int stages, int dbg, int* __restrict__ tile_counter) {
  constexpr int PART_B = FG_BN * KP * 2;  // bytes of one split part of Phi_F (B)
  constexpr int FG_EPI_WARPS = EW;
  constexpr int FG_PW = FG_BN / (EW / 4);  // pixels per epilogue warp per unit
  constexpr int NW = FG_PW / 32;           // mask words per thread per unit
  extern __shared__ __align__(1024) uint8_t smem_raw[];   // 1024-B aligned: SWIZZLE_128B atoms
  uint8_t* smem = smem_raw;                                  // (keeps the shared address space visible)
  const int mA = nfb * FG_BM;
  const int PART_A = mA * KP * 2;
  uint8_t* sX = smem;                                          // stages x 32 KB (SW128 boxes)
  uint8_t* sA = sX + (size_t)stages * FG_XSTAGE;               // H: 3 parts x mA frames x KP
  uint8_t* sB = sA + 3 * (size_t)PART_A;                       // Phi_F: 2 buffers x 3 parts
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sB + 2 * 3 * PART_B);
  uint64_t* xempty = xfull + stages;
  uint64_t* bfull = xempty + stages;
  uint64_t* bempty = bfull + 2;
  uint64_t* tfull = bempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ int tq_id[tc::TQ_N];
  __shared__ uint64_t tq_bar[2 * tc::TQ_N];
  const tc::TileQueue tq{tq_id, tq_bar, tq_bar + tc::TQ_N};

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int idx = threadIdx.x; idx < 2 * 3 * PART_B / 16; idx += blockDim.x)   // B buffers: zero columns stay zero
    reinterpret_cast<uint4*>(sB)[idx] = make_uint4(0, 0, 0, 0);
  // ---- coefficient table H (frames x KP), split in three bf16 parts, resident
  for (int idx = threadIdx.x; idx < mA * KP; idx += blockDim.x) {
    const int t = idx / KP, f = idx % KP;
    const float v = (t < m && f < n_coef) ? coef[(int64_t)f * m + t] : 0.f;
    __nv_bfloat16 b0, b1, b2;
    split3(v, b0, b1, b2);
    const uint32_t off = km_off(t, f >> 3, KP) + (f & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = b0;
    *reinterpret_cast<__nv_bfloat16*>(sA + PART_A + off) = b1;
    *reinterpret_cast<__nv_bfloat16*>(sA + 2 * PART_A + off) = b2;
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], FG_EPI_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&bfull[b], FG_EPI_WARPS);
      tc::mbar_init(&bempty[b], 1);
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], FG_EPI_WARPS);
    }
    tc::tq_init(tq, 1 + FG_EPI_WARPS);   // MMA issuer + epilogue warps
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapX);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * FG_BN);
  tc::fence_proxy_async();  // generic-proxy smem writes (H) -> async proxy (MMA)
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      // tiles are published two ahead of this thread's own loads: the epilogue
      // prefetches Phi_F of tile k + 2 while it works on tile k
      int pub = 0;
      bool ended = false;
      for (int k = 0;; ++k) {
        while (!ended && pub <= k + 2) ended = tc::tq_publish(tq, pub++, tile_counter, num_tiles) < 0;
        const int tile = tq_id[k % tc::TQ_N];   // published by this thread, not yet reusable
        if (tile < 0) break;
        for (int fb = 0; fb < nfb; ++fb) {
          tc::mbar_wait(&xempty[stage], phase ^ 1u);
          tc::mbar_arrive_expect_tx(&xfull[stage], FG_XSTAGE);
          uint8_t* dst = sX + (size_t)stage * FG_XSTAGE;
          tc::tma_load_2d(dst, &mapX, &xfull[stage], tile * FG_BN, fb * FG_BM);
          tc::tma_load_2d(dst + FG_XSTAGE / 2, &mapX, &xfull[stage], tile * FG_BN + 128, fb * FG_BM);
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      constexpr uint32_t IDESC = tc::idesc_f16(FG_BM, FG_BN, true, true, false, false);
      const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
      int it = 0, ti = 0;
      for (;; ++ti) {
        if (tc::tq_take(tq, ti) < 0) break;
        const int bb = ti & 1;
        tc::mbar_wait(&bfull[bb], (uint32_t)(ti >> 1) & 1u);
        tc::fence_after();
        for (int fb = 0; fb < nfb; ++fb, ++it) {
          const int tb = it & 1;
          tc::mbar_wait(&tempty[tb], ((uint32_t)(it >> 1) & 1u) ^ 1u);
          tc::fence_after();
          const uint32_t d = tmem_base + (uint32_t)(tb * FG_BN);
          int first = 1;
#pragma unroll
          for (int pi = 0; pi < 3; ++pi)
#pragma unroll
            for (int pj = 0; pj < 3 - pi; ++pj)
#pragma unroll
              for (int kk = 0; kk < KP / 16; ++kk) {
                const uint64_t ad =
                    desc_nosw(aBase + pi * PART_A + fb * (FG_BM / 8) * (16 * KP) + kk * 256, 128, 16 * KP);
                const uint64_t bd = desc_nosw(bBase + (bb * 3 + pj) * PART_B + kk * 256, 128, 16 * KP);
                if (!FG_ABL(dbg & 2)) tc::mma_f16(d, ad, bd, IDESC, first ? 0u : 1u);
                first = 0;
              }
          tc::mma_commit(&tfull[tb]);
        }
        tc::mma_commit(&bempty[bb]);
      }
    }
  } else {  // ---------------------------------------------------------- epilogue
    const int ew = warp - 2;          // 0 .. FG_EPI_WARPS-1
    const int q = warp & 3;           // TMEM lane quarter: frames 32q .. 32q+31 of a unit
    const int sl = ew >> 2;           // pixel slice [sl*FG_PW, (sl+1)*FG_PW) of a tile
    const int r = q * 32 + lane;      // frame within the unit (= TMEM lane)
    const int etid = ew * 32 + lane;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ti = 0;
    // Phi_F of a tile (B operand), prefetched into registers one tile ahead
    // (consecutive threads own consecutive pixels: coalesced) and split into smem
    // when its buffer is free.
    const int br = etid & (FG_BN - 1);
    const int bfh = etid >> 8;                    // which part of the KP columns
    constexpr int BH = KP * FG_BN / (32 * EW);    // columns of Phi_F per thread
    float pv[BH];
    auto load_phi = [&](int tile) {
      const int64_t j = (int64_t)tile * FG_BN + br;
#pragma unroll
      for (int u = 0; u < BH; ++u) {
        const int f = bfh * BH + u;
        pv[u] = (tile >= 0 && f < n_coef && j < n_local) ? __ldg(Phi + j + (int64_t)coef_col[f] * ldphi) : 0.f;
      }
    };
    auto build_b = [&](int tix) {
      const int bb = tix & 1;
      tc::mbar_wait(&bempty[bb], ((uint32_t)(tix >> 1) & 1u) ^ 1u);
      uint8_t* pb = sB + (size_t)bb * 3 * PART_B;
      if (bfh * BH < n_coef) {   // chunks of columns >= n_coef stay zero (written once)
        // three-term bf16 split, two columns per conversion; a thread's BH columns of
        // pixel br are whole 16-B chunks of the K-major layout: one 16-B store per part
        uint32_t q0[BH / 2], q1[BH / 2], q2[BH / 2];
#pragma unroll
        for (int u = 0; u < BH; u += 2) {
          const __nv_bfloat162 a = __floats2bfloat162_rn(pv[u], pv[u + 1]);
          const float2 af = __bfloat1622float2(a);
          const float r0 = pv[u] - af.x, r1 = pv[u + 1] - af.y;
          const __nv_bfloat162 b = __floats2bfloat162_rn(r0, r1);
          const float2 bf = __bfloat1622float2(b);
          const __nv_bfloat162 c = __floats2bfloat162_rn(r0 - bf.x, r1 - bf.y);
          q0[u / 2] = *reinterpret_cast<const uint32_t*>(&a);
          q1[u / 2] = *reinterpret_cast<const uint32_t*>(&b);
          q2[u / 2] = *reinterpret_cast<const uint32_t*>(&c);
        }
#pragma unroll
        for (int c8 = 0; c8 < BH / 8; ++c8) {
          const uint32_t off = km_off(br, (bfh * BH) / 8 + c8, KP);
          *reinterpret_cast<uint4*>(pb + off) = make_uint4(q0[4 * c8], q0[4 * c8 + 1], q0[4 * c8 + 2], q0[4 * c8 + 3]);
          *reinterpret_cast<uint4*>(pb + PART_B + off) =
              make_uint4(q1[4 * c8], q1[4 * c8 + 1], q1[4 * c8 + 2], q1[4 * c8 + 3]);
          *reinterpret_cast<uint4*>(pb + 2 * PART_B + off) =
              make_uint4(q2[4 * c8], q2[4 * c8 + 1], q2[4 * c8 + 2], q2[4 * c8 + 3]);
        }
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bfull[bb]);
    };
    // tile ids in order from the queue: this tile, the next (B being built), the one after
    int tile = tc::tq_take_warp(tq, 0);
    load_phi(tile);
    if (tile >= 0) build_b(0);
    int tnext = tile >= 0 ? tc::tq_take_warp(tq, 1) : -1;
    load_phi(tnext);
    for (; tile >= 0; ++ti) {
      int tafter = -1;
      if (tnext >= 0) {
        build_b(ti + 1);
        tafter = tc::tq_take_warp(tq, ti + 2);
        load_phi(tafter);
      }
      for (int fb = 0; fb < nfb; ++fb, ++it) {
        const int tb = it & 1;
        tc::mbar_wait(&tfull[tb], (uint32_t)(it >> 1) & 1u);
        tc::mbar_wait(&xfull[stage], phase);
        tc::fence_after();
        const uint8_t* xs = sX + (size_t)stage * FG_XSTAGE;
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(tb * FG_BN);
        const int64_t t = (int64_t)fb * FG_BM + r;
        uint32_t words[NW];
        // TMEM loads of word w + 1 in flight while word w is built (tcgen05.wait::ld
        // waits for all of this thread's loads, so it is issued before the arithmetic)
        uint32_t La[32], Lb[32];
        tc::tmem_ld16(ta + sl * FG_PW, *reinterpret_cast<uint32_t(*)[16]>(&La[0]));
        tc::tmem_ld16(ta + sl * FG_PW + 16, *reinterpret_cast<uint32_t(*)[16]>(&La[16]));
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const int j0 = sl * FG_PW + 32 * w;       // pixel offset in the tile
          uint32_t (&L)[32] = (w & 1) ? Lb : La;
          uint32_t (&Ln)[32] = (w & 1) ? La : Lb;
          // pixels j0..j0+31 of frame r: box j0/128, 16-B chunks c, c+1 XOR-swizzled by r%8
          const uint8_t* row = xs + (j0 >> 7) * (FG_XSTAGE / 2) + r * 128;
          const int c = (j0 & 127) >> 4;
          const uint4 a = *reinterpret_cast<const uint4*>(row + (((c) ^ (r & 7)) << 4));
          const uint4 b = *reinterpret_cast<const uint4*>(row + (((c + 1) ^ (r & 7)) << 4));
          const uint32_t xw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          tc::tmem_ld_wait();
          if (w + 1 < NW) {
            tc::tmem_ld16(ta + j0 + 32, *reinterpret_cast<uint32_t(*)[16]>(&Ln[0]));
            tc::tmem_ld16(ta + j0 + 48, *reinterpret_cast<uint32_t(*)[16]>(&Ln[16]));
          }
          words[w] = FG_ABL(dbg & 1) ? 0u : mask32(xw, L, tau);
        }
        // the stage goes back only after the words are built: the shared loads have
        // then completed (handing it back right after issuing them raced with the
        // producer's next TMA write into the stage -- rare mask errors under load)
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&tempty[tb]);
          tc::mbar_arrive(&xempty[stage]);
        }
        if (++stage == stages) { stage = 0; phase ^= 1u; }
        const int64_t w0 = ((int64_t)tile * FG_BN + sl * FG_PW) >> 5;   // first mask word
        if (t < m) {
          uint32_t* dst = mask + t * ldw + w0;
          if (32 * (w0 + NW) <= n_local + 31 && 32 * (w0 + NW - 1) < n_local && (ldw & 3) == 0 && NW == 4) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(words[0], words[1 % NW], words[2 % NW], words[3 % NW]);
          } else {
#pragma unroll
            for (int w = 0; w < NW; ++w)
              if (32 * (w0 + w) < n_local) dst[w] = words[w];
          }
        }
      }
      tile = tnext;
      tnext = tafter;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 2 * FG_BN);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 fg_encode_fn() {
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

static size_t fg_smem_bytes(int KP, int nfb, int stages) {
  return 1024 + (size_t)stages * FG_XSTAGE + 3 * (size_t)nfb * FG_BM * KP * 2 + 2 * 3 * (size_t)FG_BN * KP * 2 +
         512;
}

// ablation switches exist only in builds with -DCDMD_ABLATIONS;
// the release kernel always runs the MMAs and the mask arithmetic
#ifdef CDMD_ABLATIONS
static int dbg_mode() {
  const char* e = getenv("CDMD_FG_DBG");
  return e ? atoi(e) : 0;
}
#else
static int dbg_mode() { return 0; }
#endif

static int fg_kp(int n_coef) { return n_coef <= 16 ? 16 : (n_coef <= 32 ? 32 : 0); }

bool foreground_tc_supported(const cdmd_video& v, const cdmd_model& M) {
  const int KP = fg_kp(M.n_coef);
  if (!KP || !fg_encode_fn()) return false;
  const int nfb = (int)ceil_div(v.m, FG_BM);
  return fg_smem_bytes(KP, nfb, 2) <= 226 * 1024 && (v.ld % 16) == 0;   // 1 KB: static smem
}

template <int KP, int EW>
static cudaError_t launch_kp(const cdmd_video& v, const cdmd_model& M, const float* Phi, int64_t ldphi,
                             float tau, uint32_t* mask, int64_t ldw, int* tile_counter, cudaStream_t st) {
  const int nfb = (int)ceil_div(v.m, FG_BM);
  CUtensorMap mapX;
  cuuint64_t dims[2] = {(cuuint64_t)v.n_local, (cuuint64_t)v.m};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld};
  cuuint32_t box[2] = {128, FG_BM};
  cuuint32_t estr[2] = {1, 1};
  if (fg_encode_fn()(&mapX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  // 3 X stages measured faster than 4 (0.319 vs 0.329 ms at c4) and 2 (0.322 ms)
  int stages = 3;
  if (const char* e = getenv("CDMD_FG_STAGES")) { const int q = atoi(e); if (q >= 2 && q <= 4) stages = q; }
  while (stages > 2 && fg_smem_bytes(KP, nfb, stages) > 226 * 1024) --stages;
  const size_t smem = fg_smem_bytes(KP, nfb, stages);
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(foreground_tc_kernel<KP, EW>));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int num_tiles = (int)ceil_div(v.n_local, FG_BN);
  const int pc = persistent_ctas(sms);
  const int grid = num_tiles < pc ? num_tiles : pc;
  e = cudaMemsetAsync(tile_counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  note_launch();
  foreground_tc_kernel<KP, EW><<<grid, 32 * (2 + EW), smem, st>>>(
      mapX, v.n_local, v.m, nfb, Phi, ldphi, M.coef, M.coef_col, M.n_coef, tau, mask, ldw, num_tiles, stages, dbg_mode(),
      tile_counter);
  return cudaGetLastError();
}

cudaError_t launch_foreground_tc(const cdmd_video& v, const cdmd_model& M, const float* Phi, int64_t ldphi,
                                 float tau, uint32_t* mask, int64_t ldw, int* tile_counter, cudaStream_t st) {
  static int ew = -1;
  if (ew < 0) {   // epilogue warps (CDMD_FG_EW = 8 or 16; measured in DESIGN.md §5.4)
    const char* e = getenv("CDMD_FG_EW");
    ew = (e && atoi(e) == 16) ? 16 : 8;
  }
  if (fg_kp(M.n_coef) == 16)
    return ew == 16 ? launch_kp<16, 16>(v, M, Phi, ldphi, tau, mask, ldw, tile_counter, st)
                    : launch_kp<16, 8>(v, M, Phi, ldphi, tau, mask, ldw, tile_counter, st);
  return ew == 16 ? launch_kp<32, 16>(v, M, Phi, ldphi, tau, mask, ldw, tile_counter, st)
                  : launch_kp<32, 8>(v, M, Phi, ldphi, tau, mask, ldw, tile_counter, st);
}

}  // namespace cdmd
