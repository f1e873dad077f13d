// foreground.cu — background reconstruction + residual + threshold + bit-pack
// (Eq. DMDTerms, x_BG = Phi beta P:206-208, Eq. thres).
//
// The background of pixel j at frame t is a short real dot product over the
// folded Phi columns the OMP support touches (cdmd_fit's coefficient table):
//   L_jt = sum_f Phi[j, F_f] h_f(t),  h_f(t) = sum of Re / -sg Im of beta_p lambda_p^(t-1)
// STATIC uses h_f(1) for every t.  mask_jt = [ |x_jt - L_jt| > tau ].
// Layout: each lane owns pixels base + lane + 32 i (i < 4), so a warp ballot per
// slot i yields one mask word (32 consecutive pixels) directly; X reads are
// 32-B coalesced per slot.  One pass over X, mask written once.
#include "common.cuh"

namespace cdmd {

constexpr int FG_FRAMES = 64;   // frames per block (grid y)

template <int NC>
__global__ void __launch_bounds__(256) foreground_dynamic_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t n_local, int64_t m,
    const float* __restrict__ Phi, int64_t ldphi, const float* __restrict__ coef,
    const int32_t* __restrict__ coef_col, int n_coef, float tau, uint32_t* __restrict__ mask,
    int64_t ldw) {
  __shared__ float h[FG_FRAMES][NC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = ((int64_t)blockIdx.x * 8 + warp) * 128;
  const int64_t t0 = (int64_t)blockIdx.y * FG_FRAMES;
  const int nt = (int)(m - t0 < FG_FRAMES ? m - t0 : FG_FRAMES);
  for (int i = threadIdx.x; i < FG_FRAMES * NC; i += blockDim.x) {
    const int tt = i / NC, f = i % NC;
    h[tt][f] = (f < n_coef && tt < nt) ? coef[(int64_t)f * m + t0 + tt] : 0.f;
  }
  float ph[4][NC];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int64_t j = base + lane + 32 * s;
#pragma unroll
    for (int f = 0; f < NC; ++f)
      ph[s][f] = (f < n_coef && j < n_local) ? __ldg(Phi + j + (int64_t)coef_col[f] * ldphi) : 0.f;
  }
  __syncthreads();
  if (base >= n_local) return;
  for (int tt = 0; tt < nt; ++tt) {
    const int64_t t = t0 + tt;
    const uint8_t* __restrict__ xt = X + t * ld;
    float xv[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int64_t j = base + lane + 32 * s;
      xv[s] = j < n_local ? (float)__ldg(xt + j) : 0.f;
    }
    float L[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int f = 0; f < NC; ++f) {
      const float hf = h[tt][f];
#pragma unroll
      for (int s = 0; s < 4; ++s) L[s] = fmaf(ph[s][f], hf, L[s]);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const unsigned word = __ballot_sync(0xffffffffu, fabsf(xv[s] - L[s]) > tau);
      const int64_t wi = (base >> 5) + s;
      if (lane == s && 32 * wi < n_local) mask[t * ldw + wi] = word;
    }
  }
}

// STATIC: the background is one value per pixel, so the threshold
// test reduces to integer bounds: with integer x,
//   x > L + tau  <=>  x > floor(L + tau)      x < L - tau  <=>  x < ceil(L - tau).
// Each thread owns one mask word (32 consecutive pixels): per frame it loads 32
// bytes (2 x 16 B, the warp reads 1 KB contiguous), compares four pixels per
// byte-SIMD instruction and stores one coalesced word.  HBM-bound.
__device__ __forceinline__ uint32_t movemask4(uint32_t v) {  // bytes 0x00/0xFF -> 4 bits
  return ((v & 0x01010101u) * 0x10204080u) >> 28;
}

__global__ void __launch_bounds__(256) foreground_static_kernel(
    const uint8_t* __restrict__ X, int64_t ld, int64_t n_local, int64_t m,
    const float* __restrict__ Phi, int64_t ldphi, const float* __restrict__ coef,
    const int32_t* __restrict__ coef_col, int n_coef, float tau, uint32_t* __restrict__ mask,
    int64_t ldw, int64_t frames_per_block) {
  // static background of the block's 8192 pixels, computed with coalesced Phi
  // reads into shared memory (stored [b][thread] so the per-thread reads below
  // are conflict-free), then converted to per-pixel integer bounds
  __shared__ float Ls[32][257];
  const int64_t jb = (int64_t)blockIdx.x * blockDim.x * 32;
  {
    float Lacc[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) Lacc[u] = 0.f;
    for (int f = 0; f < n_coef; ++f) {  // 32 independent coalesced loads in flight per column
      const float* col = Phi + (int64_t)coef_col[f] * ldphi + jb + threadIdx.x;
      const float c = coef[(int64_t)f * m];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const int64_t j = jb + threadIdx.x + 256 * u;
        Lacc[u] = fmaf(j < n_local ? __ldg(col + 256 * u) : 0.f, c, Lacc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int i = threadIdx.x + 256 * u;
      Ls[i & 31][i >> 5] = Lacc[u];
    }
  }
  __syncthreads();
  const int64_t wi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j0 = wi * 32;
  if (j0 >= n_local) return;
  const int64_t t0 = (int64_t)blockIdx.y * frames_per_block;
  const int64_t t1 = t0 + frames_per_block < m ? t0 + frames_per_block : m;
  uint32_t hiw[8], low[8], always = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    uint32_t hw = 0, lw = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t j = j0 + 4 * w + b;
      const float L = Ls[4 * w + b][threadIdx.x];
      const float fh = floorf(L + tau), fl = ceilf(L - tau);
      if (j < n_local && (fh < 0.f || fl > 255.f)) always |= 1u << (4 * w + b);
      hw |= (uint32_t)fminf(fmaxf(fh, 0.f), 255.f) << (8 * b);
      lw |= (uint32_t)fminf(fmaxf(fl, 0.f), 255.f) << (8 * b);
    }
    hiw[w] = hw;
    low[w] = lw;
  }
  const uint32_t valid = (j0 + 32 <= n_local) ? 0xffffffffu : ((1u << (n_local - j0)) - 1u);
  const bool full = j0 + 32 <= n_local;
  const uint8_t* __restrict__ xp = X + j0;
#pragma unroll 2
  for (int64_t t = t0; t < t1; ++t) {
    uint32_t xw[8];
    if (full) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(xp + t * ld));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(xp + t * ld + 16));
      xw[0] = a.x; xw[1] = a.y; xw[2] = a.z; xw[3] = a.w;
      xw[4] = b.x; xw[5] = b.y; xw[6] = b.z; xw[7] = b.w;
    } else {
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b)
          if (j0 + 4 * w + b < n_local) v |= (uint32_t)xp[t * ld + 4 * w + b] << (8 * b);
        xw[w] = v;
      }
    }
    uint32_t word = always;
#pragma unroll
    for (int w = 0; w < 8; ++w)
      word |= movemask4(__vcmpgtu4(xw[w], hiw[w]) | __vcmpltu4(xw[w], low[w])) << (4 * w);
    mask[t * ldw + wi] = word & valid;
  }
}

template <int NC>
static cudaError_t launch_dyn(const cdmd_video& v, const cdmd_model& M, const float* Phi,
                              int64_t ldphi, float tau, uint32_t* mask, int64_t ldw, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(v.n_local, 1024), (unsigned)ceil_div(v.m, FG_FRAMES));
  note_launch();
  foreground_dynamic_kernel<NC><<<grid, 256, 0, st>>>(v.X, v.ld, v.n_local, v.m, Phi, ldphi, M.coef,
                                                      M.coef_col, M.n_coef, tau, mask, ldw);
  return cudaGetLastError();
}

bool foreground_tc_supported(const cdmd_video& v, const cdmd_model& M);
cudaError_t launch_foreground_tc(const cdmd_video& v, const cdmd_model& M, const float* Phi, int64_t ldphi,
                                 float tau, uint32_t* mask, int64_t ldw, int* tile_counter, cudaStream_t st);

cudaError_t launch_foreground(const cdmd_video& v, const cdmd_model& M, const float* Phi,
                              int64_t ldphi, int mode, float tau, uint32_t* mask, int64_t ldw,
                              int* tile_counter, cudaStream_t st) {
  if (mode == CDMD_BG_STATIC) {
    // one thread per mask word; frames split so the grid covers >= 4 waves
    const int64_t words = ceil_div(v.n_local, 32);
    const int64_t bx = ceil_div(words, 256);
    int64_t fpb = v.m;
    while (fpb > 64 && bx * ceil_div(v.m, fpb) < 2 * 148) fpb = (fpb + 1) / 2;
    dim3 grid((unsigned)bx, (unsigned)ceil_div(v.m, fpb));
    note_launch();
    foreground_static_kernel<<<grid, 256, 0, st>>>(v.X, v.ld, v.n_local, v.m, Phi, ldphi, M.coef,
                                                   M.coef_col, M.n_coef, tau, mask, ldw, fpb);
    return cudaGetLastError();
  }
  if (foreground_tc_supported(v, M))
    return launch_foreground_tc(v, M, Phi, ldphi, tau, mask, ldw, tile_counter, st);
  const int nc = M.n_coef;
  if (nc <= 4) return launch_dyn<4>(v, M, Phi, ldphi, tau, mask, ldw, st);
  if (nc <= 8) return launch_dyn<8>(v, M, Phi, ldphi, tau, mask, ldw, st);
  if (nc <= 12) return launch_dyn<12>(v, M, Phi, ldphi, tau, mask, ldw, st);
  if (nc <= 16) return launch_dyn<16>(v, M, Phi, ldphi, tau, mask, ldw, st);
  if (nc <= 24) return launch_dyn<24>(v, M, Phi, ldphi, tau, mask, ldw, st);
  if (nc <= 32) return launch_dyn<32>(v, M, Phi, ldphi, tau, mask, ldw, st);
  return launch_dyn<64>(v, M, Phi, ldphi, tau, mask, ldw, st);
}

// Background frames t0+1 .. t0+nt (inspection path of cdmd_background).
__global__ void background_kernel(const float* __restrict__ Phi, int64_t ldphi, int64_t n_local,
                                  int64_t m, const float* __restrict__ coef,
                                  const int32_t* __restrict__ coef_col, int n_coef, int dynamic,
                                  int64_t t0, int64_t nt, float* __restrict__ L, int64_t ldl) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tt = blockIdx.y;
  if (j >= n_local || tt >= nt) return;
  const int64_t t = dynamic ? t0 + tt : 0;
  float acc = 0.f;
  for (int f = 0; f < n_coef; ++f) acc = fmaf(Phi[j + (int64_t)coef_col[f] * ldphi], coef[(int64_t)f * m + t], acc);
  L[tt * ldl + j] = acc;
}

cudaError_t launch_background(const float* Phi, int64_t ldphi, int64_t n_local, const cdmd_model& M,
                              int mode, int64_t t0, int64_t nt, float* L, int64_t ldl,
                              cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(n_local, 256), (unsigned)nt);
  note_launch();
  background_kernel<<<grid, 256, 0, st>>>(Phi, ldphi, n_local, M.m, M.coef, M.coef_col, M.n_coef,
                                          mode == CDMD_BG_DYNAMIC, t0, nt, L, ldl);
  return cudaGetLastError();
}

}  // namespace cdmd
