// common.cuh — shared device helpers of libcdmd (sm_100a).  Product code: no
// oracle code is included or mirrored here.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <stdint.h>

#include "../../include/cdmd.h"

#define CDMD_LIMBS 4        // int8 limbs of the fixed-point M
#define CDMD_KBLK 128       // frames per K block of the modes GEMM (mpad granularity)
#define CDMD_NBLK 16        // kpad granularity (tcgen05 N step for M=128)

namespace cdmd {

// every libcdmd kernel launch site calls note_launch() (cdmd_kernel_launches)
inline std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> n{0};
  return n;
}
inline void note_launch() { launch_counter().fetch_add(1, std::memory_order_relaxed); }

// Opt kernel `kern` into the device's whole shared memory per block (minus its static
// shared memory), once per (device, kernel).  The attribute is per function: setting it
// to each launch's own size would let one host thread lower it under another's launch.
cudaError_t smem_optin(const void* kern);

// CTAs of the persistent full-resolution kernels (modes, foreground): all SMs, or
// fewer with CDMD_PERSIST_RESERVE=R (R SMs left to other streams' small solves)
int persistent_ctas(int sms);
extern int g_persist_limit;   // set by cdmd_sm_partition (partition.cu)


// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. SC'11 (the generator DESIGN.md §3.1 fixes for C): per round
// (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2, c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0);
// key += (W0, W1) between rounds.
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Exact recombination of the int8-limb partial sums of the modes GEMM
// (DESIGN.md §5.3): tot = sum_l acc_l 128^(3-l) in int64 (exact), then one
// conversion to fp32 and one fp32 multiply by the column scale.  Shared by the
// dp4a and tcgen05 kernels so their outputs are bit-identical.
__device__ __forceinline__ float combine_limbs(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               float scale) {
  const long long tot = ((long long)(int32_t)a0 << 21) + ((long long)(int32_t)a1 << 14) +
                        ((long long)(int32_t)a2 << 7) + (long long)(int32_t)a3;
  return (float)tot * scale;
}

// Philox counter word c3 tags the use of the stream.
enum : uint32_t { TAG_SPIXEL = 1, TAG_SPARSE = 2, TAG_RADEMACHER = 3, TAG_GAUSSIAN = 4, TAG_SRFT = 5,
                  TAG_SRFT_PHASE = 6 };

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// dev_info words written by kernels (read back by cdmd_fit)
enum { INFO_K_EFF = 0, INFO_K_SEL = 1, INFO_N_COEF = 2, INFO_FLAGS = 3 };
enum { FLAG_SPARSE_OVERFLOW = 1, FLAG_NONFINITE = 2, FLAG_EIG_PAIRING = 4, FLAG_OMP_CHOL = 8, FLAG_GRAPH_STALE = 16 };

}  // namespace cdmd

// ------------------------------------------------------- internal host interface
struct cdmd_handle_s;

namespace cdmd {

struct SensingPlan {            // resolved sensing parameters
  int kind;
  int64_t n, p;
  double s, lq;                  // sparse rate and log1p(-1/s)
  uint32_t k0, k1;
  int h;                         // Feistel half width (single pixel)
  int64_t cap;                   // ELL capacity (sparse)
};

SensingPlan make_plan(int64_t n_total, const cdmd_sensing* c);
size_t sensing_ws_bytes(const SensingPlan& P);

// launchers (return cudaGetLastError())
cudaError_t launch_spixel_rows(const SensingPlan& P, int32_t* rows, cudaStream_t st);
// SRFT: the p/2 frequencies of R (the Feistel bijection with tag TAG_SRFT)
cudaError_t launch_srft_freqs(const SensingPlan& P, int32_t* freqs, cudaStream_t st);
cudaError_t launch_srft_table(uint16_t* table, cudaStream_t st);
cudaError_t launch_sketch_srft(const cdmd_video& v, const SensingPlan& P, const int32_t* freqs,
                               const uint16_t* table, float* Y, int64_t ldy, float* part, cudaStream_t st);
bool sketch_srft_supported(const cdmd_video& v);
cudaError_t launch_sparse_rows(const SensingPlan& P, int32_t* ell, int32_t* counts,
                               int32_t* flags, cudaStream_t st);
cudaError_t launch_gaussian_table(uint16_t* table, cudaStream_t st);
cudaError_t launch_philox_test(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out,
                               int64_t count, cudaStream_t st);

cudaError_t launch_sketch_spixel(const cdmd_video& v, const SensingPlan& P, const int32_t* rows,
                                 int32_t* Y, int64_t ldy, cudaStream_t st);
cudaError_t launch_sketch_sparse(const cdmd_video& v, const SensingPlan& P, const int32_t* ell,
                                 const int32_t* counts, int32_t* Y, int64_t ldy, cudaStream_t st);
cudaError_t launch_sketch_rademacher(const cdmd_video& v, const SensingPlan& P, int32_t* Y,
                                     int64_t ldy, cudaStream_t st);
// Gaussian: split-K partial sums go to `part` (gaussian_part_floats(v, p) floats of
// the sketch workspace) and are reduced in a fixed order (deterministic Y)
int64_t gaussian_part_floats(const cdmd_video& v, int64_t p);
cudaError_t launch_sketch_gaussian(const cdmd_video& v, const SensingPlan& P, const uint16_t* table,
                                   float* Y, int64_t ldy, float* part, cudaStream_t st);

cudaError_t launch_modes_simt(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi,
                              cudaStream_t st);
// tile_counter: one device int of the handle (dynamic persistent tile schedule)
cudaError_t launch_modes_tc(const cdmd_video& v, const cdmd_model& M, float* Phi, int64_t ldphi,
                            int* tile_counter, cudaStream_t st);

size_t amp_gram_ws_bytes(int sms, int k);
cudaError_t launch_amp_gram(int sms, const float* Phi, int64_t ldphi, const uint8_t* x1, int64_t n_local,
                            int k, double* ws, double* G, cudaStream_t st);
cudaError_t launch_amp_solve(const double* G, int k, const int32_t* pair, double* b, int32_t* dropped,
                             cudaStream_t st);
cudaError_t launch_background(const float* Phi, int64_t ldphi, int64_t n_local, const cdmd_model& M,
                              int mode, int64_t t0, int64_t nt, float* L, int64_t ldl,
                              cudaStream_t st);
cudaError_t launch_foreground(const cdmd_video& v, const cdmd_model& M, const float* Phi,
                              int64_t ldphi, int mode, float tau, uint32_t* mask, int64_t ldw,
                              int* tile_counter, cudaStream_t st);

// N11 fused single pass (fused_tc.cu): dynamic or static background, n_coef <= 16, m <= 512
bool fused_supported(const cdmd_video& v, const cdmd_model& M, int mode);
cudaError_t launch_fused_fg(const cdmd_video& v, const cdmd_model& M, int mode, float tau, uint32_t* mask,
                            int64_t ldw, int* tile_counter, cudaStream_t st);
// ... with the 3x3 median fused (whole frames, imgW % 32 == 0): raw mask -> mask, filtered -> medout
cudaError_t launch_fused_fg_median(const cdmd_video& v, const cdmd_model& M, int mode, float tau, uint32_t* mask,
                                   int64_t ldw, int* tile_counter, int imgW, int imgH, uint32_t* medout, int* medcnt,
                                   cudaStream_t st);

cudaError_t launch_mask_median3(const uint32_t* in, int64_t ldw, int64_t W, int64_t H, int64_t m, uint32_t* out,
                                cudaStream_t st);

bool modes_tc_supported(const cdmd_model& M);
bool foreground_tc_supported(const cdmd_video& v, const cdmd_model& M);

}  // namespace cdmd
