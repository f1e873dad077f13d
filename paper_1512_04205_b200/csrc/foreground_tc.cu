// foreground_tc.cu — fused dynamic background + residual + threshold + bit-pack on
// tcgen05 tensor cores (Eq. DMDTerms P:185-193 with Eq. thres).
//
// The dynamic background of a 128-pixel tile over 256 frames is the rank-NC
// product L = Phi_F (128 x NC) . H^T (NC x 256) of the folded support modes and the
// coefficient table h_f(t) = Re/Im of beta_p lambda_p^(t-1).  On CUDA cores that is
// NC FMAs per pixel-frame (ALU-bound above HBM speed); here it is six
// kind::f16 MMAs per (tile, frame block) on bf16 three-term splits of both factors
//   Phi_F = A0 + A1 + A2,  H = B0 + B1 + B2  (24 significant bits each),
//   L ~= sum_{i + j <= 2} A_i B_j^T  accumulated in fp32 in TMEM,
// followed by an epilogue that reads L from TMEM (lane = pixel), compares with the
// uint8 pixels of the TMA-staged X tile and ballots 32 pixels into one mask word.
// Persistent CTAs; warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps 2..9
// epilogue (also build the A splits of each tile from Phi).  One read of X, one
// write of the mask, Phi_F read once.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace cdmd {

constexpr int FG_BM = 128;         // pixels per tile (UMMA M, TMEM lanes)
constexpr int FG_BN = 256;         // frames per unit (UMMA N, TMEM columns per buffer)
constexpr int FG_XSTAGE = FG_BM * FG_BN;  // bytes of X per unit
constexpr int FG_FSPLIT = 4;                 // frame slices per unit (per TMEM lane quarter)
constexpr int FG_EPI_WARPS = 4 * FG_FSPLIT;   // epilogue warps
constexpr int FG_FW = FG_BN / FG_FSPLIT;      // frames per epilogue warp per unit

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

template <int KP>
__global__ void __launch_bounds__(32 * (2 + FG_EPI_WARPS), 1) foreground_tc_kernel(
    const __grid_constant__ CUtensorMap mapX, int64_t n_local, int64_t m, int nfb,
    const float* __restrict__ Phi, int64_t ldphi, const float* __restrict__ coef,
    const int32_t* __restrict__ coef_col, int n_coef, float tau, uint32_t* __restrict__ mask,
    int64_t ldw, int num_tiles, int stages) {
  constexpr int PART_A = FG_BM * KP * 2;  // bytes of one split part of A
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int mB = nfb * FG_BN;
  const int PART_B = mB * KP * 2;
  uint8_t* sX = smem;                                          // stages x 32 KB
  uint8_t* sB = sX + (size_t)stages * FG_XSTAGE;               // 3 parts x mB rows x KP
  uint8_t* sA = sB + 3 * (size_t)PART_B;                       // 2 buffers x 3 parts
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sA + 2 * 3 * PART_A);
  uint64_t* xempty = xfull + stages;
  uint64_t* afull = xempty + stages;
  uint64_t* aempty = afull + 2;
  uint64_t* tfull = aempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- coefficient table H (frames x KP), split in three bf16 parts, resident
  for (int idx = threadIdx.x; idx < mB * KP; idx += blockDim.x) {
    const int t = idx / KP, f = idx % KP;
    const float v = (t < m && f < n_coef) ? coef[(int64_t)f * m + t] : 0.f;
    __nv_bfloat16 b0, b1, b2;
    split3(v, b0, b1, b2);
    const uint32_t off = km_off(t, f >> 3, KP) + (f & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = b0;
    *reinterpret_cast<__nv_bfloat16*>(sB + PART_B + off) = b1;
    *reinterpret_cast<__nv_bfloat16*>(sB + 2 * PART_B + off) = b2;
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], FG_EPI_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&afull[b], FG_EPI_WARPS);
      tc::mbar_init(&aempty[b], 1);
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], FG_EPI_WARPS);
    }
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
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x)
        for (int fb = 0; fb < nfb; ++fb) {
          tc::mbar_wait(&xempty[stage], phase ^ 1u);
          tc::mbar_arrive_expect_tx(&xfull[stage], FG_XSTAGE);
          tc::tma_load_2d(sX + (size_t)stage * FG_XSTAGE, &mapX, &xfull[stage], tile * FG_BM, fb * FG_BN);
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      constexpr uint32_t IDESC = tc::idesc_f16(FG_BM, FG_BN, true, true, false, false);
      const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
      int it = 0, ti = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ti) {
        const int ab = ti & 1;
        tc::mbar_wait(&afull[ab], (uint32_t)(ti >> 1) & 1u);
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
                const uint64_t ad = desc_nosw(aBase + (ab * 3 + pi) * PART_A + kk * 256, 128, 16 * KP);
                const uint64_t bd =
                    desc_nosw(bBase + pj * PART_B + fb * (FG_BN / 8) * (16 * KP) + kk * 256, 128, 16 * KP);
                tc::mma_f16(d, ad, bd, IDESC, first ? 0u : 1u);
                first = 0;
              }
          tc::mma_commit(&tfull[tb]);
        }
        tc::mma_commit(&aempty[ab]);
      }
    }
  } else {  // ---------------------------------------------------------- epilogue
    const int ew = warp - 2;          // 0..7
    const int q = warp & 3;           // TMEM lane quarter
    const int half = ew >> 2;         // frame slice [half*FG_FW, (half+1)*FG_FW) of a unit
    const int row = q * 32 + lane;    // pixel within the tile
    const int etid = ew * 32 + lane;  // 0 .. 32*FG_EPI_WARPS-1
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ti = 0;
    // A = Phi_F of a tile, prefetched into registers one tile ahead (coalesced:
    // consecutive lanes own consecutive pixels) and split into smem when its
    // buffer is free, so the MMA of tile i+1 never waits for the epilogue.
    const int ar = etid & (FG_BM - 1);
    const int afh = etid >> 7;                   // which KP/FG_FSPLIT columns of A
    constexpr int AH = KP / FG_FSPLIT;
    float pv[AH];
    auto load_phi = [&](int tile) {
      const int64_t j = (int64_t)tile * FG_BM + ar;
#pragma unroll
      for (int u = 0; u < AH; ++u) {
        const int f = afh * AH + u;
        pv[u] = (tile < num_tiles && f < n_coef && j < n_local) ? __ldg(Phi + j + (int64_t)coef_col[f] * ldphi) : 0.f;
      }
    };
    auto build_a = [&](int tix) {
      const int ab = tix & 1;
      tc::mbar_wait(&aempty[ab], ((uint32_t)(tix >> 1) & 1u) ^ 1u);
      uint8_t* pa = sA + (size_t)ab * 3 * PART_A;
#pragma unroll
      for (int u = 0; u < AH; ++u) {
        const int f = afh * AH + u;
        __nv_bfloat16 a0, a1, a2;
        split3(pv[u], a0, a1, a2);
        const uint32_t off = km_off(ar, f >> 3, KP) + (f & 7) * 2;
        *reinterpret_cast<__nv_bfloat16*>(pa + off) = a0;
        *reinterpret_cast<__nv_bfloat16*>(pa + PART_A + off) = a1;
        *reinterpret_cast<__nv_bfloat16*>(pa + 2 * PART_A + off) = a2;
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&afull[ab]);
    };
    load_phi(blockIdx.x);
    if ((int)blockIdx.x < num_tiles) build_a(0);
    load_phi(blockIdx.x + gridDim.x);
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++ti) {
      if (tile + (int)gridDim.x < num_tiles) {
        build_a(ti + 1);
        load_phi(tile + 2 * gridDim.x);
      }
      const int64_t wi = (int64_t)tile * (FG_BM / 32) + q;  // mask word of this warp's 32 pixels
      const bool wvalid = 32 * wi < n_local;
      for (int fb = 0; fb < nfb; ++fb, ++it) {
        const int tb = it & 1;
        tc::mbar_wait(&tfull[tb], (uint32_t)(it >> 1) & 1u);
        tc::mbar_wait(&xfull[stage], phase);
        tc::fence_after();
        const uint8_t* xs = sX + (size_t)stage * FG_XSTAGE;
        const uint32_t tb_addr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(tb * FG_BN + half * FG_FW);
        // 32 frames per group: one ballot per frame gives the warp's mask word;
        // lane i keeps frame i's word and the group is stored with one instruction
        uint32_t* mrow = mask + ((int64_t)fb * FG_BN + half * FG_FW) * ldw + wi;
        for (int c32 = 0; c32 < FG_FW; c32 += 32) {
          uint32_t Lr[32];
          tc::tmem_ld16(tb_addr + c32, *reinterpret_cast<uint32_t(*)[16]>(&Lr[0]));
          tc::tmem_ld16(tb_addr + c32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&Lr[16]));
          tc::tmem_ld_wait();
          const uint8_t* xr = xs + (half * FG_FW + c32) * FG_BM + row;
          uint32_t myword = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = __uint_as_float(0x4B000000u | (uint32_t)xr[i * FG_BM]) - 8388608.0f;
            const uint32_t word = __ballot_sync(0xffffffffu, fabsf(x - __uint_as_float(Lr[i])) > tau);
            myword = (lane == i) ? word : myword;
          }
          const int64_t t = (int64_t)fb * FG_BN + half * FG_FW + c32 + lane;
          if (wvalid && t < m) mrow[(int64_t)(c32 + lane) * ldw] = myword;
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(&tempty[tb]);
          tc::mbar_arrive(&xempty[stage]);
        }
        if (++stage == stages) { stage = 0; phase ^= 1u; }
      }
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
  return 1024 + (size_t)stages * FG_XSTAGE + 3 * (size_t)nfb * FG_BN * KP * 2 + 2 * 3 * (size_t)FG_BM * KP * 2 +
         512;
}

static int fg_kp(int n_coef) { return n_coef <= 16 ? 16 : (n_coef <= 32 ? 32 : 0); }

bool foreground_tc_supported(const cdmd_video& v, const cdmd_model& M) {
  const int KP = fg_kp(M.n_coef);
  if (!KP || !fg_encode_fn()) return false;
  const int nfb = (int)ceil_div(v.m, FG_BN);
  return fg_smem_bytes(KP, nfb, 2) <= 227 * 1024;
}

template <int KP>
static cudaError_t launch_kp(const cdmd_video& v, const cdmd_model& M, const float* Phi, int64_t ldphi,
                             float tau, uint32_t* mask, int64_t ldw, cudaStream_t st) {
  const int nfb = (int)ceil_div(v.m, FG_BN);
  CUtensorMap mapX;
  cuuint64_t dims[2] = {(cuuint64_t)v.n_local, (cuuint64_t)v.m};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld};
  cuuint32_t box[2] = {FG_BM, FG_BN};
  cuuint32_t estr[2] = {1, 1};
  if (fg_encode_fn()(&mapX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  int stages = 4;
  while (stages > 2 && fg_smem_bytes(KP, nfb, stages) > 227 * 1024) --stages;
  const size_t smem = fg_smem_bytes(KP, nfb, stages);
  cudaError_t e = cudaFuncSetAttribute(foreground_tc_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int num_tiles = (int)ceil_div(v.n_local, FG_BM);
  const int grid = num_tiles < sms ? num_tiles : sms;
  foreground_tc_kernel<KP><<<grid, 32 * (2 + FG_EPI_WARPS), smem, st>>>(
      mapX, v.n_local, v.m, nfb, Phi, ldphi, M.coef, M.coef_col, M.n_coef, tau, mask, ldw, num_tiles, stages);
  return cudaGetLastError();
}

cudaError_t launch_foreground_tc(const cdmd_video& v, const cdmd_model& M, const float* Phi, int64_t ldphi,
                                 float tau, uint32_t* mask, int64_t ldw, cudaStream_t st) {
  if (fg_kp(M.n_coef) == 16) return launch_kp<16>(v, M, Phi, ldphi, tau, mask, ldw, st);
  return launch_kp<32>(v, M, Phi, ldphi, tau, mask, ldw, st);
}

}  // namespace cdmd
