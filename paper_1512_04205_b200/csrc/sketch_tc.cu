// sketch_tc.cu — dense sketches on tcgen05 tensor cores (Alg. 1 step 3, P:336;
// "computing Y = CX using unstructured dense matrices has a time complexity of
// O(pnm)").
//
// Rademacher: Y[r, t] = sum_i c_ri X[t, i] with c_ri = +-1 as one
// split-K int8 GEMM, D[rows x frames] = C[rows x pixels] . X[frames x pixels]^T:
//   A = C tile, 128 rows x 128 pixels of s8, regenerated from Philox in SMEM by four
//       generator warps (one Philox call = the 128 sign bits of (row, 128-px chunk))
//       in the SWIZZLE_128B K-major layout;
//   B = X tile, <= 256 frames x 128 pixels of u8 -- the stored frame-major layout is
//       already K-major -- TMA-staged with SWIZZLE_128B;
//   D = int32 accumulators in TMEM for the CTA's (row block, frame block), summed
//       over its pixel range.  kind::i8 takes u8 x s8 directly, so no -128 shift is
//       needed; every product and sum is exact (|Y| <= 255 n < 2^31).
// Pixel ranges are split across CTAs and the partial sums meet in Y through int32
// atomics (exact and order-independent).  Warp roles: 0 TMA producer, 1 TMEM owner +
// MMA issuer, 2..5 C generators and then the epilogue.
#include <cstdio>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace cdmd {

constexpr int SK_BM = 128;   // rows of C per CTA (UMMA M)
constexpr int SK_BK = 128;   // pixels per stage (one Philox call per row)
constexpr int SK_CST = SK_BM * SK_BK;  // bytes of a C stage

__global__ void __launch_bounds__(192, 1) sketch_rademacher_tc_kernel(
    const __grid_constant__ CUtensorMap mapX, int64_t pix0, int64_t n_local, int64_t m, int64_t p,
    uint32_t k0, uint32_t k1, int fbn, int nchunks_total, int chunks_per_split, int stages,
    int32_t* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];   // 1024-B aligned: SWIZZLE_128B atoms
  uint8_t* smem = smem_raw;                                  // (keeps the shared address space visible)
  const int xst = fbn * SK_BK;                    // bytes of an X stage
  uint8_t* sX = smem;
  uint8_t* sC = sX + (size_t)stages * xst;
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sC + (size_t)stages * SK_CST);
  uint64_t* xempty = xfull + stages;
  uint64_t* cfull = xempty + stages;
  uint64_t* cempty = cfull + stages;
  uint64_t* tfull = cempty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * SK_BM;     // first row of C
  const int64_t f0 = (int64_t)blockIdx.y * fbn;       // first frame
  const int c_begin = blockIdx.z * chunks_per_split;  // 128-pixel chunks of this split
  const int c_end = min(nchunks_total, c_begin + chunks_per_split);
  const int nch = c_end - c_begin;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 1);
      tc::mbar_init(&cfull[s], 4);
      tc::mbar_init(&cempty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapX);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 256);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int c = c_begin; c < c_end; ++c) {
        tc::mbar_wait(&xempty[stage], phase ^ 1u);
        tc::mbar_arrive_expect_tx(&xfull[stage], (uint32_t)xst);
        tc::tma_load_2d(sX + (size_t)stage * xst, &mapX, &xfull[stage], c * SK_BK, (int32_t)f0);
        if (++stage == stages) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      const uint32_t idesc = tc::idesc_i8(SK_BM, fbn, /*a_signed=*/true, /*b_signed=*/false, false, false);
      const uint32_t xBase = tc::smem_u32(sX), cBase = tc::smem_u32(sC);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nch; ++i) {
        tc::mbar_wait(&xfull[stage], phase);
        tc::mbar_wait(&cfull[stage], phase);
        tc::fence_after();
#pragma unroll
        for (int kk = 0; kk < SK_BK / 32; ++kk) {
          const uint64_t ad = tc::smem_desc_sw128(cBase + stage * SK_CST + kk * 32, 0, 1024);
          const uint64_t bd = tc::smem_desc_sw128(xBase + stage * xst + kk * 32, 0, 1024);
          tc::mma_i8(tmem_base, ad, bd, idesc, (i | kk) != 0);
        }
        tc::mma_commit(&xempty[stage]);
        tc::mma_commit(&cempty[stage]);
        if (++stage == stages) { stage = 0; phase ^= 1u; }
      }
      tc::mma_commit(tfull);
    }
  } else {  // ------------------------------------------ C generators + epilogue
    const int g = threadIdx.x - 64;             // 0..127: the row of C this thread generates
    const int64_t row = r0 + g;
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < nch; ++i) {
      const int c = c_begin + i;
      uint4 w = make_uint4(0, 0, 0, 0);
      if (row < p) w = philox(make_uint4((uint32_t)((pix0 >> 7) + c), (uint32_t)row, 0u, TAG_RADEMACHER), k0, k1);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      tc::mbar_wait(&cempty[stage], phase ^ 1u);
      uint8_t* dst = sC + (size_t)stage * SK_CST + g * 128;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {           // 16 pixels per 16-B chunk
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t nib = (ws[ch >> 1] >> (16 * (ch & 1) + 4 * q)) & 0xFu;
          const uint32_t spread = (nib * 0x00204081u) & 0x01010101u;  // bit b -> byte b
          v[q] = 0x01010101u + spread * 0xFEu;                        // bit 1 -> -1, 0 -> +1
        }
        *reinterpret_cast<uint4*>(dst + ((ch ^ (g & 7)) << 4)) = make_uint4(v[0], v[1], v[2], v[3]);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&cfull[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1u; }
    }
    // epilogue: TMEM lane = row of C, columns = frames; int32 atomics into Y
    tc::mbar_wait(tfull, 0);
    tc::fence_after();
    const int q = warp & 3;
    const int64_t rr = r0 + q * 32 + lane;
    const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16);
    const int fvalid = (int)min((int64_t)fbn, m - f0);
    for (int c0 = 0; c0 < fbn; c0 += 16) {
      uint32_t v[16];
      tc::tmem_ld16(ta + c0, v);
      tc::tmem_ld_wait();
      if (rr < p && nch > 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c0 + i < fvalid) atomicAdd(Y + rr + (f0 + c0 + i) * ldy, (int32_t)v[i]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 256);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 sk_encode_fn() {
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

bool sketch_rademacher_tc_supported(const cdmd_video& v) { return sk_encode_fn() != nullptr && (v.ld % 16) == 0; }

cudaError_t launch_sketch_rademacher_tc(const cdmd_video& v, const SensingPlan& P, int32_t* Y, int64_t ldy,
                                        cudaStream_t st) {
  // frame blocks of at most 256 (UMMA N), multiple of 16
  const int nfb = (int)ceil_div(v.m, 256);
  const int fbn = (int)round_up(ceil_div(v.m, nfb), 16);
  const int nrb = (int)ceil_div(P.p, SK_BM);
  const int nchunks = (int)ceil_div(v.n_local, SK_BK);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // split the pixel range so the grid covers ~2 waves of 148 SMs
  int splits = (int)ceil_div(2 * sms, (int64_t)nrb * nfb);
  if (splits > nchunks) splits = nchunks;
  if (splits < 1) splits = 1;
  const int cps = (int)ceil_div(nchunks, splits);
  splits = (int)ceil_div(nchunks, cps);
  CUtensorMap mapX;
  cuuint64_t dims[2] = {(cuuint64_t)v.n_local, (cuuint64_t)v.m};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld};
  cuuint32_t box[2] = {SK_BK, (cuuint32_t)fbn};
  cuuint32_t estr[2] = {1, 1};
  if (sk_encode_fn()(&mapX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int xst = fbn * SK_BK;
  int stages = 4;
  auto smem_of = [&](int s) { return (size_t)1024 + (size_t)s * (xst + SK_CST) + 512; };
  while (stages > 2 && smem_of(stages) > 110 * 1024) --stages;  // two CTAs per SM
  const size_t smem = smem_of(stages);
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(sketch_rademacher_tc_kernel));
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(Y, 0, sizeof(int32_t) * (size_t)ldy * v.m, st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)nrb, (unsigned)nfb, (unsigned)splits);
  note_launch();
  sketch_rademacher_tc_kernel<<<grid, 192, smem, st>>>(mapX, v.pix0, v.n_local, v.m, P.p, P.k0, P.k1, fbn,
                                                       nchunks, cps, stages, Y, ldy);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------ Gaussian
// Y = C D with c_ri = T[u16] (bf16-valued N(0,1)) as one split-K
// kind::f16 GEMM with fp32 accumulation in TMEM (north_star: "bf16 x uint8-exact
// operands accumulate in fp32 on tensor cores"):
//   A = C tile, 128 rows x 32 pixels of fp16 (every table value is exact in fp16),
//       regenerated in SMEM by eight generator warps: one Philox call -> eight 16-bit
//       table indices -> one 16-B chunk; the table's positive half (32768 fp16) is
//       resident in SMEM (T is odd-symmetric);
//   B = X tile, <= 512 frames x 32 pixels (TMA-staged uint8, 4 stages deep), converted
//       in SMEM by eight warps from uint8 to the
//       exact fp16 value x - 128 (centred: 4x smaller partial sums); one spare frame row
//       of ones yields sum_i c_ri, and the epilogue adds back 128 * sum_i c_ri;
//   D = fp32 in TMEM (M = 128, N <= 512 over two MMAs), split-K partial sums meet in Y
//       through fp32 atomics.
#ifdef CDMD_GS_PROF
__device__ long long gs_prof[8 * 16];
#define GS_T(ii, slot)                                                                               \
  if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x & 31) == 0 && (ii) >= 100 && (ii) < 108 && \
      (warp <= 1 || warp == 1 + GS_GEN_WARPS || warp == GS_GEN_WARPS + GS_CVT_WARPS || warp == 1 + GS_GEN_WARPS + GS_CVT_WARPS)) \
    gs_prof[((ii) - 100) * 16 + (slot)] = clock64();
#else
#define GS_T(ii, slot)
#endif
constexpr int GS_BM = 128;            // rows of C per CTA
constexpr int GS_BK = 32;             // pixels per stage (64-B fp16 rows, SWIZZLE_64B)
constexpr int GS_A = GS_BM * GS_BK * 2;   // bytes of an A stage (8 KB)
constexpr int GS_XK = 64;             // pixels per uint8 X stage (64-B TMA rows)
constexpr int GS_XS = 2;              // uint8 X stages (TMA)
#ifndef GS_GEN_WARPS_DEF
#define GS_GEN_WARPS_DEF 8
#endif
constexpr int GS_GEN_WARPS = GS_GEN_WARPS_DEF;   // 4, 8 or 16: thread = (row, 8-pixel chunks) of the A stage
constexpr int GS_CVT_WARPS = 8;
constexpr int GS_THREADS = 32 * (2 + GS_GEN_WARPS + GS_CVT_WARPS);

__global__ void __launch_bounds__(GS_THREADS, 1) sketch_gaussian_tc_kernel(
    const __grid_constant__ CUtensorMap mapX, int64_t pix0, int64_t n_local, int64_t m, int64_t p,
    uint32_t k0, uint32_t k1, const uint16_t* __restrict__ table_bf16, int npad, int nchunks_total,
    int chunks_per_split, int xbox, float* __restrict__ part) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];   // 1024-B aligned: swizzle atoms
  uint8_t* smem = smem_raw;
  const int BST = npad * GS_BK * 2;                     // bytes of a B stage (fp16)
  const int XST = npad * GS_XK;                         // bytes of an X stage (uint8)
  uint8_t* sA = smem;                                   // 2 x 8 KB
  uint8_t* sB = sA + 2 * GS_A;                          // 2 x BST
  uint8_t* sX = sB + 2 * (size_t)BST;                   // GS_XS x XST
  uint16_t* htab = reinterpret_cast<uint16_t*>(sX + (size_t)GS_XS * XST);   // 32768 fp16 bits
  uint64_t* afull = reinterpret_cast<uint64_t*>(htab + 32768);
  uint64_t* bfull = afull + 2;
  uint64_t* sempty = bfull + 2;
  uint64_t* xfull = sempty + 2;
  uint64_t* xempty = xfull + GS_XS;
  uint64_t* tfull = xempty + GS_XS;
  uint64_t* bhi = tfull + 1;      // B frames [256, npad) of a stage converted
  uint64_t* slo = bhi + 2;        // the stage's MMAs on frames [0, 256) done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slo + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * GS_BM;
  const int c_begin = blockIdx.y * chunks_per_split;
  const int c_end = min(nchunks_total, c_begin + chunks_per_split);
  const int nch = c_end - c_begin;
  for (int j = threadIdx.x; j < 32768; j += blockDim.x) {   // positive half of T as fp16 bits
    const float v = __uint_as_float((uint32_t)table_bf16[32768 + j] << 16);
    htab[j] = __half_as_ushort(__float2half_rn(v));         // exact: 8 significant bits
  }
  if (warp == 0 && lane == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&afull[b], GS_GEN_WARPS);
      tc::mbar_init(&bfull[b], GS_CVT_WARPS / 2);
      tc::mbar_init(&bhi[b], GS_CVT_WARPS / 2);
      tc::mbar_init(&sempty[b], 1);
      tc::mbar_init(&slo[b], 1);
    }
    for (int b = 0; b < GS_XS; ++b) {
      tc::mbar_init(&xfull[b], 1);
      tc::mbar_init(&xempty[b], GS_CVT_WARPS);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapX);
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int wtma = 1 + GS_GEN_WARPS + GS_CVT_WARPS;       // the TMA warp

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
      for (int i = 0; i < nch; ++i) {
        const int st = i & 1;
        const uint32_t ph = (uint32_t)(i >> 1) & 1u;
        tc::mbar_wait(&afull[st], ph);
        GS_T(i, 0)
        tc::mbar_wait(&bfull[st], ph);
        GS_T(i, 1)
        tc::fence_after();
        // frames [0, 256) as soon as their converter half is done, then [256, npad)
        for (int nb = 0; nb < npad; nb += 256) {
          if (nb) {
            tc::mma_commit(&slo[st]);
            tc::mbar_wait(&bhi[st], ph);
            tc::fence_after();
          }
          const int nn = npad - nb < 256 ? npad - nb : 256;
          const uint32_t idesc = tc::idesc_f16(GS_BM, nn, false, false, false, false);
#pragma unroll
          for (int kk = 0; kk < GS_BK / 16; ++kk) {
            const uint64_t ad = tc::smem_desc(aBase + st * GS_A + kk * 32, 0, 512, 4);
            const uint64_t bd = tc::smem_desc(bBase + st * BST + nb * 64 + kk * 32, 0, 512, 4);
            tc::mma_f16(tmem_base + (uint32_t)nb, ad, bd, idesc, (i | kk) != 0);
          }
        }
        if (npad <= 256) tc::mma_commit(&slo[st]);
        tc::mma_commit(&sempty[st]);
        GS_T(i, 2)
      }
      tc::mma_commit(tfull);
    }
  } else if (warp == wtma) {
    if (lane == 0) {  // ---------------------------------------- TMA producer (X uint8)
      const int nx = (nch + 1) >> 1;   // X stages of GS_XK = 2 GS_BK pixels (64-B rows)
      for (int i = 0; i < nx; ++i) {
        const int xs = i % GS_XS;
        const uint32_t ph = (uint32_t)(i / GS_XS) & 1u;
        tc::mbar_wait(&xempty[xs], ph ^ 1u);
        tc::mbar_arrive_expect_tx(&xfull[xs], (uint32_t)XST);
        GS_T(2 * i, 15)
        const int px = (c_begin + 2 * i) * GS_BK;
        for (int fb = 0; fb < npad; fb += xbox)   // boxes of xbox frame rows tile npad exactly
          tc::tma_load_2d(sX + (size_t)xs * XST + (size_t)fb * GS_XK, &mapX, &xfull[xs], px, fb);
      }
    }
  } else if (warp <= GS_GEN_WARPS) {  // ---------------- C generators, then epilogue
    constexpr int GS_NQ = 16 / GS_GEN_WARPS;    // 16-B chunks (8 pixels, one Philox call) per thread and stage
    const int g = threadIdx.x - 32;            // 0..32 GS_GEN_WARPS - 1
    const int rr = g & (GS_BM - 1);            // row of the tile
    const int q0 = g >> 7;                     // chunks q0 + (GS_GEN_WARPS / 4) c of the stage's four
    const int64_t row = r0 + rr;
    const int swz = (rr >> 1) & 3;             // SWIZZLE_64B chunk permutation of this row
    const uint32_t ctr0 = (uint32_t)(pix0 >> 3) + (uint32_t)(c_begin * (GS_BK / 8) + q0);
    for (int i = 0; i < nch; ++i) {
      const int st = i & 1;
      const uint32_t ph = (uint32_t)(i >> 1) & 1u;
      uint32_t h2[GS_NQ][4];
#pragma unroll
      for (int c = 0; c < GS_NQ; ++c) {
        uint4 w = make_uint4(0, 0, 0, 0);   // one Philox call = eight 16-bit table indices
        if (row < p)
          w = philox(make_uint4(ctr0 + (uint32_t)(i * (GS_BK / 8) + c * (GS_GEN_WARPS / 4)), (uint32_t)row, 0u, TAG_GAUSSIAN),
                     k0, k1);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // both 16-bit indices at once: T[u] = +H[u - 32768] (u >= 32768), -H[u ^ 0x7FFF] otherwise
          const uint32_t wq = ws[q];
          const uint32_t sg = ~wq & 0x80008000u;
          const uint32_t idx = (wq ^ (sg - (sg >> 15))) & 0x7FFF7FFFu;
          const uint32_t h0 = htab[idx & 0xFFFFu], h1 = htab[idx >> 16];
          h2[c][q] = (h0 | (h1 << 16)) ^ sg;
        }
      }
      GS_T(i, 3)
      tc::mbar_wait(&sempty[st], ph ^ 1u);
      GS_T(i, 4)
#pragma unroll
      for (int c = 0; c < GS_NQ; ++c) {
        const int q8 = q0 + c * (GS_GEN_WARPS / 4);
        *reinterpret_cast<uint4*>(sA + st * GS_A + rr * 64 + ((q8 ^ swz) << 4)) = make_uint4(h2[c][0], h2[c][1], h2[c][2], h2[c][3]);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&afull[st]);
      GS_T(i, 5)
    }
    if (warp <= 4) {  // epilogue: TMEM lane = row of C, column t = frame, column m = sum_i c_ri
      tc::mbar_wait(tfull, 0);
      tc::fence_after();
      const int q = warp & 3;
      const int64_t ry = r0 + q * 32 + lane;
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16);
      uint32_t rs[16];
      tc::tmem_ld16(ta + (uint32_t)(m & ~15), rs);
      tc::tmem_ld_wait();
      const float rowsum = __uint_as_float(rs[m & 15]);
      for (int c0 = 0; c0 < (int)m; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(ta + c0, v);
        tc::tmem_ld_wait();
        if (ry < p && nch > 0) {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (c0 + t < m) part[((int64_t)blockIdx.y * m + c0 + t) * p + ry] = fmaf(128.0f, rowsum, __uint_as_float(v[t]));
        }
      }
    }
  } else {  // --------------------------- X converters: uint8 (SMEM) -> fp16 x - 128
    // thread = (16-pixel half hf, frames fr0 + 64 u of its 256-frame group): all four frame rows are read and
    // converted into registers before the B slot is awaited, so the conversion overlaps
    // the MMA that still reads the slot; the ragged last chunk of the slab and the row
    // of ones take a per-element path
    const int cthr = threadIdx.x - 32 * (1 + GS_GEN_WARPS);   // 0..255
    const int grp = cthr >> 7;                                  // frames [256 grp, 256 grp + 256)
    const int hf = cthr & 1, fr0 = 256 * grp + ((cthr & 127) >> 1);   // half, first frame
    const __half2 c1152 = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
    const int mi = (int)m;
    for (int i = 0; i < nch; ++i) {
      const int st = i & 1;
      const uint32_t ph = (uint32_t)(i >> 1) & 1u;
      const int xi = i >> 1, xs = xi % GS_XS;                   // one X stage = two B stages
      if ((i & 1) == 0) tc::mbar_wait(&xfull[xs], (uint32_t)(xi / GS_XS) & 1u);
      const uint8_t* xt = sX + (size_t)xs * XST + GS_BK * (i & 1) + 16 * hf;
      const int64_t jx = (int64_t)(c_begin + i) * GS_BK + 16 * hf;   // first local pixel of the half
      const int64_t rem = n_local - jx;
      const int valid = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
      uint32_t hw[4][8];
      if (valid == 16) {   // branch-free: four predicated 16-B loads in flight, then convert
        uint4 xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int f = fr0 + 64 * u;
          xv[u] = f < mi ? *reinterpret_cast<const uint4*>(xt + f * GS_XK) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int f = fr0 + 64 * u;
          const uint32_t xw[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
          const uint32_t fill = f == mi ? 0x3C003C00u : 0u;   // the row of ones: D[:, m] = sum_i c_ri
#pragma unroll
          for (int b = 0; b < 8; ++b) {   // two pixels -> half2 (1024 + x) - 1152 = x - 128, exact
            const uint32_t pr = __byte_perm(xw[b >> 1], 0x64646464u, (b & 1) ? 0x7372u : 0x5150u);
            __half2 hh = __hsub2(*reinterpret_cast<const __half2*>(&pr), c1152);
            hw[u][b] = f < mi ? *reinterpret_cast<uint32_t*>(&hh) : fill;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int f = fr0 + 64 * u;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            uint32_t w = 0u;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int q = 2 * b + e;
              uint32_t h = 0u;
              if (q < valid) {
                if (f < mi) h = __half_as_ushort(__int2half_rn((int)xt[f * GS_XK + q] - 128));
                else if (f == mi) h = 0x3C00u;   // the row of ones: D[:, m] = sum_i c_ri
              }
              w |= h << (16 * e);
            }
            hw[u][b] = w;
          }
        }
      }
      GS_T(i, 9 + (warp == 1 + GS_GEN_WARPS ? 0 : 3))
      tc::mbar_wait(grp ? &sempty[st] : &slo[st], ph ^ 1u);
      GS_T(i, 10 + (warp == 1 + GS_GEN_WARPS ? 0 : 3))
      uint8_t* bst = sB + (size_t)st * BST;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = fr0 + 64 * u;
        if (f < npad) {
          uint8_t* rowp = bst + f * 64;
          const int swz = (f >> 1) & 3;
          *reinterpret_cast<uint4*>(rowp + (((2 * hf) ^ swz) << 4)) = make_uint4(hw[u][0], hw[u][1], hw[u][2], hw[u][3]);
          *reinterpret_cast<uint4*>(rowp + (((2 * hf + 1) ^ swz) << 4)) = make_uint4(hw[u][4], hw[u][5], hw[u][6], hw[u][7]);
        }
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if ((i & 1) || i == nch - 1) tc::mbar_arrive(&xempty[xs]);
        if (grp == 0 || npad > 256) tc::mbar_arrive(grp ? &bhi[st] : &bfull[st]);
      GS_T(i, 11 + (warp == 1 + GS_GEN_WARPS ? 0 : 3))
      }
    }
  }
  __syncthreads();
#ifdef CDMD_GS_PROF
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const long long t0 = gs_prof[0];
    for (int r = 0; r < 8; ++r) {
      printf("GSPROF stage %d:", 100 + r);
      for (int c = 0; c < 16; ++c) printf(" %lld", gs_prof[r * 16 + c] - t0);
      printf("\n");
    }
  }
#endif
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 512);
  }
}

bool sketch_gaussian_tc_supported(const cdmd_video& v) { return v.m + 1 <= 512 && (v.ld % 16) == 0 && sk_encode_fn() != nullptr; }

int gaussian_tc_splits(const cdmd_video& v, int64_t p) {
  const int nrb = (int)ceil_div(p, GS_BM);
  const int nchunks = (int)ceil_div(v.n_local, GS_BK);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int splits = sms / nrb;   // one CTA per SM: a single wave
  if (splits > nchunks) splits = nchunks;
  if (splits < 1) splits = 1;
  return (int)ceil_div(nchunks, ceil_div(nchunks, splits));
}

// part: splits x m x p fp32 partial sums (reduced by the caller)
cudaError_t launch_sketch_gaussian_tc(const cdmd_video& v, const SensingPlan& P, const uint16_t* table, float* part,
                                      int* splits_out, cudaStream_t st) {
  const int npad = (int)round_up(v.m + 1, 16);     // frames + the row of ones
  const int nrb = (int)ceil_div(P.p, GS_BM);
  const int nchunks = (int)ceil_div(v.n_local, GS_BK);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int splits = sms / nrb;   // one CTA per SM: a single wave
  if (splits > nchunks) splits = nchunks;
  if (splits < 1) splits = 1;
  const int cps = (int)ceil_div(nchunks, splits);
  splits = (int)ceil_div(nchunks, cps);
  CUtensorMap mapX;
  cuuint64_t dims[2] = {(cuuint64_t)v.n_local, (cuuint64_t)v.m};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld};
  // frame rows per TMA box: a multiple of 16 that divides npad, at most 256
  int xbox = npad;
  if (xbox > 256) {
    int q = npad / 16, kk = 16;
    while (q % kk) --kk;
    xbox = 16 * kk;
  }
  cuuint32_t box[2] = {GS_XK, (cuuint32_t)xbox};
  cuuint32_t estr[2] = {1, 1};
  if (sk_encode_fn()(&mapX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const size_t smem = 1024 + 2 * (size_t)GS_A + 2 * (size_t)npad * GS_BK * 2 + (size_t)GS_XS * npad * GS_XK + 65536 + 512;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(sketch_gaussian_tc_kernel));
  if (e != cudaSuccess) return e;
  *splits_out = splits;
  dim3 grid((unsigned)nrb, (unsigned)splits);
  note_launch();
  sketch_gaussian_tc_kernel<<<grid, GS_THREADS, smem, st>>>(mapX, v.pix0, v.n_local, v.m, P.p, P.k0, P.k1, table, npad,
                                                            nchunks, cps, xbox, part);
  return cudaGetLastError();
}

}  // namespace cdmd
