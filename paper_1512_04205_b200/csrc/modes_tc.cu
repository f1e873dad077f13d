// modes_tc.cu — Phi = X' M on 5th-generation tensor cores (tcgen05, kind::i8).
//
// Eq. cDMDModes as D[pixel, n] = sum_t X'[t, pixel] * Mq[n, t] with
//   A = X' tile: 128 pixels x 128 frames of uint8, MN-major (pixels contiguous, as
//       stored), TMA-staged with SWIZZLE_128B;
//   B = the int8 limbs of M: n = limb * kpad + column, K-major, loaded ONCE per CTA
//       by TMA and kept resident in shared memory;
//   D = int32 in TMEM (exact: |D| <= (m-1) 255 127 < 2^31), two accumulator
//       buffers so the epilogue of tile i overlaps the MMAs of tile i+1.
// Persistent CTAs (one per SM) claiming tiles dynamically (tc::TileQueue), warp roles: warp 0 TMA producer, warp 1 TMEM
// allocator + single-thread MMA issuer, warps 2-9 epilogue (TMEM -> registers ->
// exact limb recombination in int64 -> fp32 Phi, coalesced stores).
// The result is bit-identical to modes.cu's dp4a kernel (both accumulate exactly).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace cdmd {

constexpr int TC_BM = 128;      // pixels per tile (UMMA M)
constexpr int TC_BK = 128;      // frames per TMA stage
constexpr int TC_STAGE = TC_BM * TC_BK;  // bytes per A stage

template <int NT>
__global__ void __launch_bounds__(320, 1) modes_tc_kernel(
    const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t n_local,
    int nkb, int stages, int kpad, int k_eff, const double* __restrict__ scale, float* __restrict__ Phi,
    int64_t ldphi, int num_tiles, uint32_t tmem_cols, int* __restrict__ tile_counter) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];   // 1024-B aligned: SWIZZLE_128B atoms
  uint8_t* smem = smem_raw;                                  // (keeps the shared address space visible)
  uint8_t* sB = smem;                                   // NT x (nkb * 128) bytes, panel-major
  uint8_t* sA = sB + (size_t)NT * nkb * TC_BK;          // stages x 16 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + (size_t)stages * TC_STAGE);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  __shared__ float sScale[256];
  __shared__ int tq_id[tc::TQ_N];
  __shared__ uint64_t tq_bar[2 * tc::TQ_N];
  const tc::TileQueue tq{tq_id, tq_bar, tq_bar + tc::TQ_N};

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < kpad; c += blockDim.x) sScale[c] = (float)scale[c];
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&tfull[0], 1);
    tc::mbar_init(&tfull[1], 1);
    tc::mbar_init(&tempty[0], 8);
    tc::mbar_init(&tempty[1], 8);
    tc::mbar_init(bfull, 1);
    tc::tq_init(tq, 1 + 8);   // MMA issuer + 8 epilogue warps
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapA);
    tc::tma_prefetch(&mapB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, tmem_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------- TMA producer
      tc::mbar_arrive_expect_tx(bfull, (uint32_t)(NT * nkb * TC_BK));
      for (int kb = 0; kb < nkb; ++kb) tc::tma_load_2d(sB + (size_t)kb * NT * TC_BK, &mapB, bfull, kb * TC_BK, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0;; ++k) {
        const int tile = tc::tq_publish(tq, k, tile_counter, num_tiles);
        if (tile < 0) break;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1u);
          tc::mbar_arrive_expect_tx(&full[stage], TC_STAGE);
          tc::tma_load_2d(sA + (size_t)stage * TC_STAGE, &mapA, &full[stage], tile * TC_BM, kb * TC_BK);
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------- MMA issuer
      constexpr uint32_t IDESC = tc::idesc_i8(TC_BM, NT, /*a_signed=*/false, /*b_signed=*/true,
                                              /*a_mn=*/true, /*b_mn=*/false);
      tc::mbar_wait(bfull, 0);
      tc::fence_after();
      const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (;; ++it) {
        if (tc::tq_take(tq, it) < 0) break;
        const int acc = it & 1;
        const uint32_t acc_phase = (uint32_t)(it >> 1) & 1u;
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1u);
        tc::fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * NT);
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < TC_BK / 32; ++kk) {
            // A: MN-major SW128 -- 8-frame groups of 128-B rows every 1024 B (SBO)
            const uint64_t ad = tc::smem_desc_sw128(aBase + stage * TC_STAGE + kk * 32 * 128, TC_STAGE, 1024);
            // B: K-major SW128 -- rows of 128 frames, 8-row groups every 1024 B;
            //    K advances by 32 B inside the swizzled row
            const uint64_t bd = tc::smem_desc_sw128(bBase + kb * NT * TC_BK + kk * 32, 0, 1024);
            tc::mma_i8(d, ad, bd, IDESC, (kb | kk) != 0);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
  } else {  // ------------------------------------------------------ epilogue
    // 8 warps: warp w reads TMEM lane quarter (w % 4) and every other 16-column chunk
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int cpar = (warp - 2) >> 2;      // which 16-column chunks (0: even, 1: odd)
    const int row = q * 32 + lane;         // pixel within the tile
    int it = 0;
    for (;; ++it) {
      const int tile = tc::tq_take_warp(tq, it);
      if (tile < 0) break;
      const int acc = it & 1;
      const uint32_t acc_phase = (uint32_t)(it >> 1) & 1u;
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after();
      const int64_t j = (int64_t)tile * TC_BM + row;
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NT);
      float* __restrict__ out = Phi + j;
      for (int c0 = 16 * cpar; c0 < k_eff; c0 += 32) {
        uint32_t r0[16], r1[16], r2[16], r3[16];
        tc::tmem_ld16(tb + 0 * kpad + c0, r0);
        tc::tmem_ld16(tb + 1 * kpad + c0, r1);
        tc::tmem_ld16(tb + 2 * kpad + c0, r2);
        tc::tmem_ld16(tb + 3 * kpad + c0, r3);
        tc::tmem_ld_wait();
        const int nc = k_eff - c0 < 16 ? k_eff - c0 : 16;
        if (j < n_local) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nc) out[(int64_t)(c0 + i) * ldphi] = combine_limbs(r0[i], r1[i], r2[i], r3[i], sScale[c0 + i]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, tmem_cols);
  }
}

// ------------------------------------------------------------------ wide M (kpad > 64)
// With more than 64 columns the int8 limbs of M no longer fit one CTA (N <= 256, and
// B stays resident in shared memory).  A cluster of MC_G = 4 CTAs then shares each
// X' tile: CTA r TMA-loads frames [32r, 32r + 32) of every 128-frame stage and
// multicasts them into the same offset of all four CTAs, so X' leaves L2 once per
// cluster; CTA g owns columns [32g, 32g + 32) (all four limbs: N = 128, its B slice
// resident) and its own TMEM accumulators.  A stage is reused once all four CTAs'
// MMAs have read it (each MMA thread commits to the stage's empty barrier in every CTA).
// Tiles are assigned to clusters statically (all four CTAs walk the same sequence).
constexpr int MC_G = 4;                    // CTAs per cluster (column groups)
constexpr int MC_CG = 32;                  // columns per CTA
constexpr int MC_NT = CDMD_LIMBS * MC_CG;  // UMMA N per CTA

__global__ void __cluster_dims__(MC_G, 1, 1) __launch_bounds__(320, 1) modes_tc_mc_kernel(
    const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int64_t n_local,
    int nkb, int stages, int kpad, int k_eff, const double* __restrict__ scale, float* __restrict__ Phi,
    int64_t ldphi, int num_tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint8_t* sB = smem;                                       // nkb panels of MC_NT rows x 128 B
  uint8_t* sA = sB + (size_t)MC_NT * nkb * TC_BK;           // stages x 16 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + (size_t)stages * TC_STAGE);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  __shared__ float sScale[MC_CG];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = (int)tc::cluster_ctarank();
  const int cid = blockIdx.x / MC_G, ncl = gridDim.x / MC_G;
  for (int c = threadIdx.x; c < MC_CG; c += blockDim.x) sScale[c] = g * MC_CG + c < kpad ? (float)scale[g * MC_CG + c] : 0.f;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], MC_G);
    }
    tc::mbar_init(&tfull[0], 1);
    tc::mbar_init(&tfull[1], 1);
    tc::mbar_init(&tempty[0], 8);
    tc::mbar_init(&tempty[1], 8);
    tc::mbar_init(bfull, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapA);
    tc::tma_prefetch(&mapB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * MC_NT);
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();   // every CTA's barriers exist before any multicast or remote arrive
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------- TMA producer
      tc::mbar_arrive_expect_tx(bfull, (uint32_t)(MC_NT * nkb * TC_BK));
      for (int kb = 0; kb < nkb; ++kb)
        for (int l = 0; l < CDMD_LIMBS; ++l)   // rows l*kpad + 32g .. +31 (past the last limb: zero fill)
          tc::tma_load_2d(sB + (size_t)kb * MC_NT * TC_BK + l * MC_CG * TC_BK, &mapB, bfull, kb * TC_BK,
                          l * kpad + g * MC_CG);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1u);   // all four CTAs are done with this stage
          tc::mbar_arrive_expect_tx(&full[stage], TC_STAGE);
          tc::tma_load_2d_mc(sA + (size_t)stage * TC_STAGE + g * (TC_STAGE / MC_G), &mapA, &full[stage],
                             tile * TC_BM, kb * TC_BK + g * (TC_BK / MC_G), (uint16_t)((1u << MC_G) - 1));
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
      }
      // drain: every CTA's final commits have reached this CTA's empty barriers
      for (int s = 0; s < stages; ++s) {
        tc::mbar_wait(&empty[stage], phase ^ 1u);
        if (++stage == stages) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------- MMA issuer
      constexpr uint32_t IDESC = tc::idesc_i8(TC_BM, MC_NT, false, true, true, false);
      tc::mbar_wait(bfull, 0);
      tc::fence_after();
      const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
        const int acc = it & 1;
        tc::mbar_wait(&tempty[acc], (((uint32_t)(it >> 1)) & 1u) ^ 1u);
        tc::fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * MC_NT);
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
#pragma unroll
          for (int kk = 0; kk < TC_BK / 32; ++kk) {
            const uint64_t ad = tc::smem_desc_sw128(aBase + stage * TC_STAGE + kk * 32 * 128, TC_STAGE, 1024);
            const uint64_t bd = tc::smem_desc_sw128(bBase + kb * MC_NT * TC_BK + kk * 32, 0, 1024);
            tc::mma_i8(d, ad, bd, IDESC, (kb | kk) != 0);
          }
          tc::mma_commit_multicast(&empty[stage], (uint16_t)((1u << MC_G) - 1));
          if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
  } else {  // ------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int c0 = 16 * ((warp - 2) >> 2);   // this warp's 16 of the CTA's 32 columns
    const int row = q * 32 + lane;
    int it = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl, ++it) {
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], ((uint32_t)(it >> 1)) & 1u);
      tc::fence_after();
      const int64_t j = (int64_t)tile * TC_BM + row;
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * MC_NT);
      const int gc = g * MC_CG + c0;   // first global column of this warp
      if (gc < k_eff) {
        uint32_t r0[16], r1[16], r2[16], r3[16];
        tc::tmem_ld16(tb + 0 * MC_CG + c0, r0);
        tc::tmem_ld16(tb + 1 * MC_CG + c0, r1);
        tc::tmem_ld16(tb + 2 * MC_CG + c0, r2);
        tc::tmem_ld16(tb + 3 * MC_CG + c0, r3);
        tc::tmem_ld_wait();
        const int nc = k_eff - gc < 16 ? k_eff - gc : 16;
        if (j < n_local) {
          float* __restrict__ out = Phi + j;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nc) out[(int64_t)(gc + i) * ldphi] = combine_limbs(r0[i], r1[i], r2[i], r3[i], sScale[c0 + i]);
        }
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::tmem_dealloc(tmem_base, 2 * MC_NT);
  }
  tc::cluster_sync_all();   // no CTA leaves while a peer may still signal its barriers
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

static bool make_map_u8(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t stride1,
                        uint32_t b0, uint32_t b1) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {stride1};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NT>
static cudaError_t launch_nt(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi,
                             int* tile_counter, cudaStream_t st) {
  const int64_t n1 = v.m - 1;
  const int nkb = (int)(M.mpad / TC_BK);
  CUtensorMap mapA, mapB;
  if (!make_map_u8(&mapA, v.X + v.ld, (uint64_t)v.n_local, (uint64_t)n1, (uint64_t)v.ld, TC_BM, TC_BK))
    return cudaErrorInvalidValue;
  if (!make_map_u8(&mapB, M.Mq, (uint64_t)M.mpad, (uint64_t)NT, (uint64_t)M.mpad, TC_BK, NT))
    return cudaErrorInvalidValue;
  const size_t bbytes = (size_t)NT * nkb * TC_BK;
  const size_t max_smem = 225 * 1024;   // 227 KB less the static shared arrays (sScale, tile queue)
  const size_t fixed = bbytes + 1024 + 512;
  int stages = (int)((max_smem - fixed) / TC_STAGE);
  if (stages > 8) stages = 8;
  if (const char* e = getenv("CDMD_MODES_STAGES")) { const int q = atoi(e); if (q >= 2 && q < stages) stages = q; }
  const size_t smem = fixed + (size_t)stages * TC_STAGE;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(modes_tc_kernel<NT>));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int num_tiles = (int)ceil_div(v.n_local, TC_BM);
  const int pc = persistent_ctas(sms);
  const int grid = num_tiles < pc ? num_tiles : pc;
  uint32_t cols = 32;
  while (cols < 2u * NT) cols <<= 1;
  e = cudaMemsetAsync(tile_counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  note_launch();
  modes_tc_kernel<NT><<<grid, 320, smem, st>>>(mapA, mapB, v.n_local, nkb, stages, M.kpad, M.k_eff,
                                                M.Mq_scale, Phi, ldphi, num_tiles, cols, tile_counter);
  return cudaGetLastError();
}

static bool modes_mc_supported(const cdmd_model& M) {
  return M.kpad > 64 && M.kpad <= MC_G * MC_CG && (size_t)MC_NT * M.mpad + 2 * TC_STAGE + 2048 <= 225 * 1024;
}

static cudaError_t launch_mc(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi, cudaStream_t st) {
  const int64_t n1 = v.m - 1;
  const int nkb = (int)(M.mpad / TC_BK);
  CUtensorMap mapA, mapB;
  if (!make_map_u8(&mapA, v.X + v.ld, (uint64_t)v.n_local, (uint64_t)n1, (uint64_t)v.ld, TC_BM, TC_BK / MC_G))
    return cudaErrorInvalidValue;
  if (!make_map_u8(&mapB, M.Mq, (uint64_t)M.mpad, (uint64_t)M.kpad * CDMD_LIMBS, (uint64_t)M.mpad, TC_BK, MC_CG))
    return cudaErrorInvalidValue;
  const size_t fixed = (size_t)MC_NT * nkb * TC_BK + 1024 + 512;
  int stages = (int)((225 * 1024 - fixed) / TC_STAGE);
  if (stages > 8) stages = 8;
  if (const char* e = getenv("CDMD_MODES_STAGES")) { const int q = atoi(e); if (q >= 2 && q < stages) stages = q; }
  const size_t smem = fixed + (size_t)stages * TC_STAGE;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(modes_tc_mc_kernel));
  if (e != cudaSuccess) return e;
  const int num_tiles = (int)ceil_div(v.n_local, TC_BM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(MC_G * 64, 1, 1);
  cfg.blockDim = dim3(320, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  int clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&clusters, modes_tc_mc_kernel, &cfg);
  if (e != cudaSuccess || clusters < 1) clusters = 32;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = persistent_ctas(sms) / MC_G;
  if (clusters > cap && cap >= 1) clusters = cap;
  if (clusters > num_tiles) clusters = num_tiles;
  note_launch();
  modes_tc_mc_kernel<<<MC_G * clusters, 320, smem, st>>>(mapA, mapB, v.n_local, nkb, stages, M.kpad, M.k_eff,
                                                         M.Mq_scale, Phi, ldphi, num_tiles);
  return cudaGetLastError();
}

bool modes_tc_supported(const cdmd_model& M) {
  const int NT = M.kpad * CDMD_LIMBS;
  if (modes_mc_supported(M)) return true;
  if (NT > 256 || (NT % 64) != 0) return false;
  return (size_t)NT * M.mpad + 2 * TC_STAGE + 2048 <= 225 * 1024;
}

cudaError_t launch_modes_tc(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi,
                            int* tile_counter, cudaStream_t st) {
  if (!modes_tc_supported(M) || !encode_fn()) return launch_modes_simt(v, M, Phi, ldphi, st);
  if (M.kpad > 64 && !getenv("CDMD_MODES_NO_MC")) return launch_mc(v, M, Phi, ldphi, st);
  switch (M.kpad * CDMD_LIMBS) {
    case 64: return launch_nt<64>(v, M, Phi, ldphi, tile_counter, st);
    case 128: return launch_nt<128>(v, M, Phi, ldphi, tile_counter, st);
    case 192: return launch_nt<192>(v, M, Phi, ldphi, tile_counter, st);
    case 256: return launch_nt<256>(v, M, Phi, ldphi, tile_counter, st);
  }
  return launch_modes_simt(v, M, Phi, ldphi, st);
}

}  // namespace cdmd
