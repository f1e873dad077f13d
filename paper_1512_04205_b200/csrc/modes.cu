// modes.cu — Phi = X' V S^-1 W = X' M (Alg. 1 step 8, Eq. cDMDModes).
//
// Numerics: X' is uint8 (exact), M is represented by CDMD_LIMBS
// balanced base-128 int8 limbs per column (cdmd_fit writes them), so every
// partial product sum_t X'[t,j] d_l[t,c] is an EXACT int32 (|.| <= (m-1) 255 127);
// the limbs are recombined exactly in int64, converted once to fp32 and scaled.  The only
// error is the quantisation of M (2^-28 of the column maximum for 4 limbs).
// This file holds the CUDA-core (dp4a) kernel; modes_tc.cu holds the tcgen05
// kernel, which produces bit-identical output.
#include "common.cuh"

namespace cdmd {

__device__ __forceinline__ int32_t dp4a_us2(uint32_t a_u8, uint32_t b_s8, int32_t c) {
  int32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8), "r"(b_s8), "r"(c));
  return d;
}

// Block: 64 pixels x 16 columns (x 4 limbs); frames in chunks of 64.
// Thread (tx, ty): pixels 4tx..4tx+3, column c0+ty, all limbs.
__global__ void __launch_bounds__(256) modes_simt_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t n_local, int64_t m,
    const int8_t* __restrict__ Mq, const double* __restrict__ scale, int kpad, int64_t mpad,
    int k_eff, float* __restrict__ Phi, int64_t ldphi) {
  __shared__ uint32_t xs[64][17];                 // [pixel][4-frame word]
  __shared__ uint32_t ms[CDMD_LIMBS][16][17];     // [limb][col][4-frame word]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t px0 = (int64_t)blockIdx.x * 64;
  const int c0 = blockIdx.y * 16;
  const int64_t n1 = m - 1;
  int32_t acc[CDMD_LIMBS][4] = {};
  for (int64_t f0 = 0; f0 < n1; f0 += 64) {
    __syncthreads();
    // X' tile: frames f0..f0+63 (X' frame f = X frame f+1), pixels px0..px0+63
    for (int i = tid; i < 64 * 16; i += 256) {
      const int px = i & 63, w = i >> 6;
      uint32_t v = 0;
      const int64_t j = px0 + px;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t f = f0 + 4 * w + b;
        if (j < n_local && f < n1) v |= (uint32_t)__ldg(X + (f + 1) * ld + j) << (8 * b);
      }
      xs[px][w] = v;
    }
    for (int i = tid; i < CDMD_LIMBS * 16 * 16; i += 256) {
      const int w = i & 15, c = (i >> 4) & 15, l = i >> 8;
      ms[l][c][w] = *reinterpret_cast<const uint32_t*>(
          Mq + ((int64_t)l * kpad + c0 + c) * mpad + f0 + 4 * w);
    }
    __syncthreads();
#pragma unroll 4
    for (int w = 0; w < 16; ++w) {
      uint32_t xv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = xs[tx * 4 + a][w];
#pragma unroll
      for (int l = 0; l < CDMD_LIMBS; ++l) {
        const uint32_t mv = ms[l][ty][w];
#pragma unroll
        for (int a = 0; a < 4; ++a) acc[l][a] = dp4a_us2(xv[a], mv, acc[l][a]);
      }
    }
  }
  const int c = c0 + ty;
  if (c >= k_eff) return;
  const float sc = (float)scale[c];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t j = px0 + tx * 4 + a;
    if (j >= n_local) continue;
    Phi[j + (int64_t)c * ldphi] =
        combine_limbs((uint32_t)acc[0][a], (uint32_t)acc[1][a], (uint32_t)acc[2][a], (uint32_t)acc[3][a], sc);
  }
}

cudaError_t launch_modes_simt(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi,
                              cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(v.n_local, 64), (unsigned)(M.kpad / 16));
  note_launch();
  modes_simt_kernel<<<grid, 256, 0, st>>>(v.X, v.ld, v.n_local, v.m, M.Mq, M.Mq_scale, M.kpad,
                                          M.mpad, M.k_eff, Phi, ldphi);
  return cudaGetLastError();
}

}  // namespace cdmd
