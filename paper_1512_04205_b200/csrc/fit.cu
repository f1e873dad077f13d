// fit.cu — the small cDMD solve on the sketch (not HBM-bound; O(p m^2 + m^3)).
//
// Alg. 1 on Y_full = C D (p x m), Y = Y_full[:, :m-1], Y' = Y_full[:, 1:]:
//   G = Y_full^T Y_full (m x m, fp64; one cuBLAS DGEMM) holds every inner
//   product the solve needs: Y^T Y = G[0:m-1, 0:m-1], Y^T Y' = G[0:m-1, 1:m],
//   Y'^T Y' = G[1:m, 1:m], Y'^T y1 = G[1:m, 0], ||y1||^2 = G[0, 0].
//   step 4  truncated SVD of Y (Eq. svd) by the method of
//           snapshots: Y^T Y = V S^2 V^T (cuSOLVER syevd), top k, sigma_j kept iff
//           sigma_j > 1e-6 sigma_1 (reading R10)
//   step 6  A~ = U^T Y' V S^-1 = S^-1 V^T (Y^T Y') V S^-1
//   step 7  A~ W = W Lambda (cuSOLVER geev), canonical order/phase
//   step 8' M = V S^-1 W (P:346 without X'), kept conjugate-folded (real columns)
//   Rem. 3  beta = omp(Phi_Y, y1) with Phi_Y = Y' M, in the Gram form of
//           Rubinstein et al.: Phi_Y^H Phi_Y = M^H (Y'^T Y') M, Phi_Y^H y1 =
//           M^H (Y'^T y1) -- identical selections, residual norms from the Gram
//           omega = log(lambda)/dt; coefficient table of the background
//           L_jt = Re sum_{p in S} beta_p phi_jp lambda_p^(t-1)
//   modes   int8 fixed-point limbs of M for cdmd_modes
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "handle.h"

namespace cdmd {

static constexpr double RANK_RTOL = 1e-6;  // reading R10
static constexpr double OMP_STOP = 1e-6;   // reading R12: stop when ||r|| <= 1e-6 ||y1||
static constexpr double TIE_RTOL = 1e-9;   // reading R13

struct FitWs {
  double *Yd, *G, *A, *w, *V, *T, *B, *VR, *Wc, *SW, *T2, *Gf, *cf, *ehw, *Es;
  int* dinfo;
  void* sy_dev;
  size_t sy_dev_bytes, sy_host_bytes;
  void* ge_dev;
  size_t ge_dev_bytes, ge_host_bytes;
  size_t total;
};

size_t hqr_smem_bytes(int k);
bool eh_supported(int n, int k);
void eh_prof_read(unsigned long long* out);
void hqr_prof_read(unsigned long long* out);
size_t eh_work_doubles(int n, int k);
cudaError_t launch_eh(int n, int k, const double* G, int64_t ldg, double* lam, double* Zout, double* work,
                      int* info, int med_cnt, double* med, cudaStream_t st);

bool lz_supported(int n, int k);
cudaError_t launch_eh_lz(int n, int k, const double* G, int64_t ldg, double* lam, double* Zout, double* work,
                         int* info, int* flag, cudaStream_t st);

// symmetric eigensolver: Lanczos on a 16-CTA cluster (lanczos.cu, default where it fits;
// its residual test falls back to the next), the 8-CTA Householder cluster solver
// (eigh.cu, n1 <= 510), else cuSOLVER syevdx.  CDMD_SYEV=h -> Householder cluster solver,
// CDMD_SYEV=d -> cuSOLVER syevd, CDMD_SYEV=dx -> cuSOLVER syevdx
static int syev_mode(int n1, int k) {
  const char* e = getenv("CDMD_SYEV");
  if (e && e[0] == 'd' && e[1] == 0) return 1;
  if (e && e[0] == 'd' && e[1] == 'x') return 2;
  if (!(e && e[0] == 'h') && lz_supported(n1, k)) return 3;
  return eh_supported(n1, k) ? 0 : 2;
}
cudaError_t launch_hqr_eig(int k, const double* A, double* W, double* VR, int* info, double* scratch,
                           cudaStream_t st);

static bool use_device_eig(int k) {
  const char* e = getenv("CDMD_GEEV");
  if (e && e[0] == 'c') return false;
  return hqr_smem_bytes(k) <= 227 * 1024;
}

static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

static cdmd_status layout_ws(cdmd_handle h, int64_t p, int64_t m, int k, char* base, FitWs* W) {
  const int64_t n1 = m - 1;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* ptr = base ? base + off : nullptr;
    off += al(bytes);
    return ptr;
  };
  W->Yd = (double*)take(sizeof(double) * p * m);
  W->G = (double*)take(sizeof(double) * m * m);
  W->A = (double*)take(sizeof(double) * n1 * n1);
  W->w = (double*)take(sizeof(double) * n1);
  W->V = (double*)take(sizeof(double) * n1 * k);
  W->T = (double*)take(sizeof(double) * n1 * k);
  W->B = (double*)take(sizeof(double) * k * k);
  W->VR = (double*)take(sizeof(double) * k * k);
  W->Es = (double*)take(sizeof(double) * 2 * k * k);   // eig scratch: Hessenberg form and Q
  W->Wc = (double*)take(sizeof(double) * 2 * k);
  W->SW = (double*)take(sizeof(double) * k * k);
  W->T2 = (double*)take(sizeof(double) * n1 * k);
  W->Gf = (double*)take(sizeof(double) * k * k);
  W->cf = (double*)take(sizeof(double) * k);
  W->dinfo = (int*)take(sizeof(int) * 16);
  W->ehw = (double*)take(sizeof(double) * eh_work_doubles((int)n1, k));
  // solver workspaces (queried with the final dimensions, once per handle and shape)
  std::array<size_t, 4> sz{};
  bool have = false;
  {
    std::lock_guard<std::mutex> g(h->mu);
    auto it = h->fit_ws_sizes.find({p, m, k});
    if (it != h->fit_ws_sizes.end()) {
      sz = it->second;
      have = true;
    }
  }
  if (!have) {   // (not under stream capture: cdmd_fit_workspace_bytes or an eager fit fills the cache)
    size_t d = 0, hb = 0;
    if (cusolverDnXsyevd_bufferSize(h->solver, h->params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n1,
                                    CUDA_R_64F, W->A, n1, CUDA_R_64F, W->w, CUDA_R_64F, &d,
                                    &hb) != CUSOLVER_STATUS_SUCCESS)
      return CDMD_ERR_CUDA;
    {
      size_t d2 = 0, hb2 = 0;
      int64_t meig = 0;
      double vl = 0.0, vu = 0.0;
      if (cusolverDnXsyevdx_bufferSize(h->solver, h->params, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                                       CUBLAS_FILL_MODE_LOWER, n1, CUDA_R_64F, W->A, n1, &vl, &vu, n1 - k + 1, n1,
                                       &meig, CUDA_R_64F, W->w, CUDA_R_64F, &d2, &hb2) != CUSOLVER_STATUS_SUCCESS)
        return CDMD_ERR_CUDA;
      if (d2 > d) d = d2;
      if (hb2 > hb) hb = hb2;
    }
    size_t gd = 0, ghb = 0;
    if (cusolverDnXgeev_bufferSize(h->solver, h->params, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, k,
                                   CUDA_R_64F, W->B, k, CUDA_C_64F, W->Wc, CUDA_R_64F, nullptr, k, CUDA_R_64F, W->VR,
                                   k, CUDA_R_64F, &gd, &ghb) != CUSOLVER_STATUS_SUCCESS)
      return CDMD_ERR_CUDA;
    sz = {d, hb, gd, ghb};
    std::lock_guard<std::mutex> g(h->mu);
    h->fit_ws_sizes[{p, m, k}] = sz;
  }
  W->sy_dev_bytes = sz[0];
  W->sy_host_bytes = sz[1];
  W->sy_dev = take(sz[0] + 16);
  W->ge_dev_bytes = sz[2];
  W->ge_host_bytes = sz[3];
  W->ge_dev = take(sz[2] + 16);
  W->total = off;
  return CDMD_OK;
}

size_t fit_ws_bytes(cdmd_handle h, int64_t p, int64_t m, int k) {
  FitWs W{};
  if (layout_ws(h, p, m, k, nullptr, &W) != CDMD_OK) return 0;
  return W.total;
}

// ------------------------------------------------------------------ kernels
template <typename T>
__global__ void to_f64_kernel(const T* __restrict__ Y, int64_t ldy, int64_t p, int64_t m,
                              double* __restrict__ Yd) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p * m) return;
  const int64_t r = i % p, t = i / p;
  Yd[i] = (double)Y[r + t * ldy];
}

// sigma_j = sqrt(w), descending; V = matching eigenvectors; k_eff.  Eigen-pairs
// are ascending in (w, A); the largest sits at index `top`.
// gd_omega > 0: also keep only sigma_j > gd_omega * median(sigma) (Gavish-Donoho optimal
// hard threshold, Remark 2), the median of the med_cnt largest eigenvalues'
// square roots taken from med[0..1] (or, med == nullptr, from the full ascending w)
__global__ void select_topk_kernel(const double* __restrict__ A, const double* __restrict__ w,
                                   int64_t n1, int64_t top, int k, double* __restrict__ V,
                                   double* __restrict__ sigma, int* __restrict__ dinfo, double gd_omega,
                                   int med_cnt, const double* __restrict__ med) {
  const int c = blockIdx.x;  // output column
  const int64_t src = top - c;
  const double s0 = sqrt(fmax(w[top], 0.0));
  for (int64_t i = threadIdx.x; i < n1; i += blockDim.x) V[i + c * n1] = A[i + src * n1];
  if (threadIdx.x == 0) {
    const double s = sqrt(fmax(w[src], 0.0));
    sigma[c] = s;
    if (c == 0) {
      double thr = RANK_RTOL * s0;
      if (gd_omega > 0.0) {
        double ma, mb;   // eigenvalues of descending ranks (cnt-1)/2 and cnt/2
        if (med) { ma = med[0]; mb = med[1]; }
        else { ma = w[n1 - 1 - (med_cnt - 1) / 2]; mb = w[n1 - 1 - med_cnt / 2]; }
        const double msig = 0.5 * (sqrt(fmax(ma, 0.0)) + sqrt(fmax(mb, 0.0)));
        thr = fmax(thr, gd_omega * msig);
      }
      int ke = 0;
      for (int j = 0; j < k; ++j)
        if (sqrt(fmax(w[top - j], 0.0)) > thr) ++ke; else break;
      if (gd_omega > 0.0 && ke == 0 && s0 > 0.0) ke = 1;   // at least one (the rule's floor)
      dinfo[INFO_K_EFF] = ke;
    }
  }
}

__global__ void scale_atilde_kernel(double* __restrict__ B, const double* __restrict__ sigma, int k) {
  const int i = threadIdx.x, j = blockIdx.x;
  if (i < k) B[i + j * k] /= sigma[i] * sigma[j];
}

// canonical eigen-order and phase (reading R11) + folded S^-1 W + lambda/omega/pair.
// One block: thread 0 forms and sorts the units (real eigenvalue / conjugate pair,
// LAPACK layout of real geev output); one warp per unit normalises its vector.
__global__ void __launch_bounds__(256) canonicalize_kernel(
    int k, const double* __restrict__ Wc, const double* __restrict__ VR, const double* __restrict__ sigma,
    double dt, double* __restrict__ lam_out, double* __restrict__ om_out, int32_t* __restrict__ pair_out,
    double* __restrict__ SW, int* __restrict__ dinfo) {
  __shared__ int ufirst[256], upair[256], ucol[256];
  __shared__ int f0[256], p0[256];
  __shared__ double m0[256], wsh[2 * 256];
  __shared__ int nu_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2 * k && i < 2 * 256; i += blockDim.x) wsh[i] = Wc[i];   // staged once
  __syncthreads();
  if (tid == 0) {   // the units (a real eigenvalue or a conjugate pair), in eig's order
    int nu = 0, flags = 0;
    for (int j = 0; j < k && nu < 256;) {
      const double re = wsh[2 * j], im = wsh[2 * j + 1];
      int pr = 0;
      if (im != 0.0) {
        if (im > 0.0 && j + 1 < k && wsh[2 * j + 2] == re && wsh[2 * j + 3] == -im) pr = 1;
        else flags |= FLAG_EIG_PAIRING;
      }
      f0[nu] = j; p0[nu] = pr; m0[nu] = hypot(re, pr ? im : 0.0); ++nu;
      j += pr ? 2 : 1;
    }
    nu_sh = nu;
    if (flags) atomicOr(&dinfo[INFO_FLAGS], flags);
  }
  __syncthreads();
  {  // stable order by (|lambda| desc, real before pair): each unit's rank counted in parallel
    const int nu = nu_sh;
    for (int a = tid; a < nu; a += blockDim.x) {
      const double ka = isnan(m0[a]) ? -1.0 : m0[a];
      const int pa = p0[a];
      int rk = 0;
      for (int b = 0; b < nu; ++b) {
        const double kb = isnan(m0[b]) ? -1.0 : m0[b];
        rk += (kb > ka || (kb == ka && (p0[b] < pa || (p0[b] == pa && b < a)))) ? 1 : 0;
      }
      ufirst[rk] = f0[a]; upair[rk] = pa;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int c = 0;
    for (int u = 0; u < nu_sh; ++u) { ucol[u] = c; c += upair[u] ? 2 : 1; }
  }
  __syncthreads();
  const int nu = nu_sh;
  for (int u = warp; u < nu; u += blockDim.x / 32) {
    const int j = ufirst[u], pr = upair[u], c = ucol[u];
    const double* va = VR + (int64_t)j * k;
    const double* vb = VR + (int64_t)(j + 1) * k;
    // unit 2-norm
    double nrm = 0.0;
    for (int i = lane; i < k; i += 32) {
      const double a = va[i], b = pr ? vb[i] : 0.0;
      nrm += a * a + b * b;
    }
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    nrm = sqrt(nrm);
    // largest |component| (first index on ties)
    double amax = -1.0;
    int imax = 0x7fffffff;
    for (int i = lane; i < k; i += 32) {
      const double a = va[i] / nrm, b = pr ? vb[i] / nrm : 0.0;
      const double mg = hypot(a, b);
      if (mg > amax) { amax = mg; imax = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double oa = __shfl_xor_sync(0xffffffffu, amax, o);
      const int oi = __shfl_xor_sync(0xffffffffu, imax, o);
      if (oa > amax || (oa == amax && oi < imax)) { amax = oa; imax = oi; }
    }
    const double pa = va[imax] / nrm, pb = pr ? vb[imax] / nrm : 0.0;
    const double pm = hypot(pa, pb);
    const double cr = pa / pm, ci = -pb / pm;  // conj(phase)
    for (int i = lane; i < k; i += 32) {
      const double a = va[i] / nrm, b = pr ? vb[i] / nrm : 0.0;
      SW[i + (int64_t)c * k] = (a * cr - b * ci) / sigma[i];
      if (pr) SW[i + (int64_t)(c + 1) * k] = (a * ci + b * cr) / sigma[i];
    }
    if (lane == 0) {
      const double lr = Wc[2 * j], li = pr ? Wc[2 * j + 1] : 0.0;
      const double lmod = hypot(lr, li), larg = atan2(li, lr);
      lam_out[2 * c] = lr; lam_out[2 * c + 1] = li;
      om_out[2 * c] = log(lmod) / dt; om_out[2 * c + 1] = larg / dt;
      pair_out[c] = pr ? 1 : 0;
      if (pr) {
        lam_out[2 * c + 2] = lr; lam_out[2 * c + 3] = -li;
        om_out[2 * c + 2] = log(lmod) / dt; om_out[2 * c + 3] = -larg / dt;
        pair_out[c + 1] = -1;
      }
    }
  }
}

// complex helpers
struct cplx { double r, i; };
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ cplx cconjmul(cplx a, cplx b) { return {a.r * b.r + a.i * b.i, a.r * b.i - a.i * b.r}; }  // conj(a) b

__device__ __forceinline__ void mode_rep(const int32_t* pair, int j, int& ra, int& rb, double& sg) {
  const int pj = pair[j];
  if (pj == 0) { ra = j; rb = j; sg = 0.0; }
  else if (pj > 0) { ra = j; rb = j + 1; sg = 1.0; }
  else { ra = j - 1; rb = j; sg = -1.0; }
}

// <phi_i, phi_j> = phi_i^H phi_j from the fold Gram Gf = F^T F (phi = f_ra + i sg f_rb)
__device__ __forceinline__ cplx gram_c(const double* Gf, int k, const int32_t* pair, int i, int j) {
  int ai, bi, aj, bj;
  double si, sj;
  mode_rep(pair, i, ai, bi, si);
  mode_rep(pair, j, aj, bj, sj);
  const double re = Gf[ai + aj * k] + si * sj * Gf[bi + bj * k];
  const double im = sj * Gf[ai + bj * k] - si * Gf[bi + aj * k];
  return {re, im};
}

// OMP (Remark 3 P:363-369) in Gram form + background coefficient table.
// One block.  corr_j = phi_j^H r = alpha_j - sum_{s in S} <phi_j, phi_s> beta_s.
__device__ unsigned long long g_omp_prof[4];   // cycles: staging, selection, outputs, coefficient table
__global__ void __launch_bounds__(256) omp_kernel(
    int k, int K, int64_t m, const double* __restrict__ Gf_g, const double* __restrict__ cf,
    const double* __restrict__ G, const int32_t* __restrict__ pair_g, const double* __restrict__ lam_g,
    double* __restrict__ beta_out, int32_t* __restrict__ support_out, float* __restrict__ coef,
    int32_t* __restrict__ coef_col, int* __restrict__ dinfo, double omega_eps, double dt, int staged) {
  // staged: Gf (k x k), lambda (2k) and the pairing (k) copied to shared memory first --
  // the selection loop and the Cholesky read them one element at a time on serial chains
  extern __shared__ double omp_dyn[];
  const unsigned long long tp0 = clock64();
  const double* Gf = Gf_g;
  const double* lam = lam_g;
  const int32_t* pair = pair_g;
  cplx* Gc = nullptr;   // staged: the complex Gram <phi_i, phi_j> of the modes, k x k
  if (staged) {
    Gc = reinterpret_cast<cplx*>(omp_dyn);
    double* ls = omp_dyn + 2 * (size_t)k * k;
    int32_t* ps = reinterpret_cast<int32_t*>(ls + 2 * k);
    for (int i = threadIdx.x; i < 2 * k; i += blockDim.x) ls[i] = lam_g[i];
    for (int i = threadIdx.x; i < k; i += blockDim.x) ps[i] = pair_g[i];
    __syncthreads();
    lam = ls;
    pair = ps;
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) Gc[idx] = gram_c(Gf_g, k, pair, idx / k, idx % k);
    __syncthreads();
  }
  auto gram = [&](int i, int j) -> cplx { return Gc ? Gc[i * k + j] : gram_c(Gf, k, pair, i, j); };
  const unsigned long long tp1 = clock64();
  __shared__ double sc[512];
  __shared__ double red[256];
  __shared__ int redi[256];
  __shared__ int S[32];
  __shared__ cplx alpha[512];
  __shared__ cplx beta[32];
  __shared__ cplx Lc[32 * 32];  // Cholesky factor of Gc[S,S]
  __shared__ double Linv[32];   // 1 / its real diagonal (thread 0's serial chain multiplies)
  __shared__ int nS_sh, stop_sh;
  __shared__ int F[128];
  __shared__ int nF_sh;
  const int tid = threadIdx.x;
  const double y1n2 = G[0];
  for (int j = tid; j < k; j += blockDim.x) {
    int ra, rb;
    double sg;
    mode_rep(pair, j, ra, rb, sg);
    alpha[j] = {cf[ra], -sg * cf[rb]};
  }
  // frequency selection: the columns with |omega| = |log lambda| / dt < omega_eps,
  // in index order, at most K (the model's support capacity; reading R24); each is added
  // as a forced "OMP step" (same least squares)
  __shared__ int T[32];
  __shared__ int nT_sh;
  if (tid == 0) {
    nS_sh = 0; stop_sh = 0; nT_sh = 0;
    if (omega_eps > 0.0) {
      const int cap = K < 32 ? K : 32;   // beta/support hold K entries, coef 2K rows
      for (int j = 0; j < k && nT_sh < cap; ++j) {
        const double lr = lam[2 * j], li = lam[2 * j + 1];
        const double om = hypot(log(hypot(lr, li)), atan2(li, lr)) / dt;
        if (om < omega_eps) T[nT_sh++] = j;
      }
    }
  }
  __syncthreads();
  const bool by_freq = omega_eps > 0.0;
  const int Kmax = by_freq ? nT_sh : (K < k ? K : k);
  for (int it = 0; it < Kmax; ++it) {
    const int nS = nS_sh;
    if (tid == 0 && !by_freq) {
      double rn2 = y1n2;
      for (int s = 0; s < nS; ++s) {
        const cplx t = cconjmul(alpha[S[s]], beta[s]);
        rn2 -= t.r;
      }
      if (!(y1n2 > 0.0) || rn2 <= OMP_STOP * OMP_STOP * y1n2) stop_sh = 1;
    }
    __syncthreads();
    if (stop_sh) break;
    double best = -1.0;
    for (int j = tid; j < k; j += blockDim.x) {
      bool in = false;
      for (int s = 0; s < nS; ++s) in |= (S[s] == j);
      const cplx gjj = gram(j, j);
      double score = -1.0;
      if (!in && gjj.r > 0.0) {
        cplx c = alpha[j];
        for (int s = 0; s < nS; ++s) {
          const cplx g = gram(j, S[s]);
          const cplx t = cmul(g, beta[s]);
          c.r -= t.r; c.i -= t.i;
        }
        score = hypot(c.r, c.i) / sqrt(gjj.r);
      }
      sc[j] = score;
      best = fmax(best, score);
    }
    // max score and the lowest index within the tie band: warp shuffles, then one value per
    // warp (two block barriers per iteration instead of a 256-wide tree each)
    const int nwarp = (int)(blockDim.x >> 5), wl = tid & 31, wi = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (wl == 0) red[wi] = best;
    __syncthreads();
    double bmax = red[0];
    for (int w = 1; w < nwarp; ++w) bmax = fmax(bmax, red[w]);
    int cand = 1 << 30;
    for (int j = tid; j < k; j += blockDim.x)
      if (sc[j] >= bmax * (1.0 - TIE_RTOL) && j < cand) cand = j;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cand = min(cand, __shfl_xor_sync(0xffffffffu, cand, o));
    if (wl == 0) redi[wi] = cand;
    __syncthreads();
    if (tid == 0) {
      int jbest = redi[0];
      for (int w = 1; w < nwarp; ++w) jbest = min(jbest, redi[w]);
      const int js = by_freq ? T[it] : jbest;
      if ((!by_freq && (!(bmax > 0.0) || !isfinite(bmax))) || js >= k || nS >= 32) {
        stop_sh = 1;
      } else {
        S[nS] = js;
        const int n = nS + 1;
        // complex Cholesky of Gc[S,S] (Hermitian positive definite): rows 0..n-2 are the
        // previous iteration's factor (the same support), only row n-1 is new
        bool ok = true;
        for (int a = n - 1; a < n && ok; ++a) {
          for (int b = 0; b <= a; ++b) {
            cplx s = gram(S[a], S[b]);  // <phi_a, phi_b>: row a, col b
            for (int q = 0; q < b; ++q) {
              const cplx t = cmul(Lc[a * 32 + q], cplx{Lc[b * 32 + q].r, -Lc[b * 32 + q].i});
              s.r -= t.r; s.i -= t.i;
            }
            if (a == b) {
              if (!(s.r > 0.0)) { ok = false; break; }
              const double dg = sqrt(s.r);
              Lc[a * 32 + a] = {dg, 0.0};
              Linv[a] = 1.0 / dg;
            } else {
              const double id = Linv[b];
              Lc[a * 32 + b] = {s.r * id, s.i * id};
            }
          }
        }
        if (!ok) {
          stop_sh = 1;
          atomicOr(&dinfo[INFO_FLAGS], 8);
        } else {
          // Normal equations: Gc beta = alpha with Gc[a][b] = <phi_a, phi_b>.
          // L computed above satisfies L L^H = H with H[a][b] = <phi_a, phi_b>.
          cplx z[32];
          for (int a = 0; a < n; ++a) {  // L z = alpha_S
            cplx s = alpha[S[a]];
            for (int q = 0; q < a; ++q) {
              const cplx t = cmul(Lc[a * 32 + q], z[q]);
              s.r -= t.r; s.i -= t.i;
            }
            z[a] = {s.r * Linv[a], s.i * Linv[a]};
          }
          for (int a = n - 1; a >= 0; --a) {  // L^H beta = z
            cplx s = z[a];
            for (int q = a + 1; q < n; ++q) {
              const cplx lq = {Lc[q * 32 + a].r, -Lc[q * 32 + a].i};
              const cplx t = cmul(lq, beta[q]);
              s.r -= t.r; s.i -= t.i;
            }
            beta[a] = {s.r * Linv[a], s.i * Linv[a]};
          }
          nS_sh = n;
        }
      }
    }
    __syncthreads();
    if (stop_sh) break;
  }
  __syncthreads();
  const unsigned long long tp2 = clock64();
  const int nS = nS_sh;
  // outputs + used fold columns (sorted, unique)
  if (tid == 0) {
    int nF = 0;
    for (int s = 0; s < nS; ++s) {
      support_out[s] = S[s];
      beta_out[2 * s] = beta[s].r;
      beta_out[2 * s + 1] = beta[s].i;
      int ra, rb;
      double sg;
      mode_rep(pair, S[s], ra, rb, sg);
      const int cols[2] = {ra, rb};
      for (int q = 0; q < (sg != 0.0 ? 2 : 1); ++q) {
        bool have = false;
        for (int f = 0; f < nF; ++f) have |= (F[f] == cols[q]);
        if (!have && nF < 128) F[nF++] = cols[q];
      }
    }
    for (int a = 1; a < nF; ++a) {
      const int v = F[a];
      int b = a - 1;
      while (b >= 0 && F[b] > v) { F[b + 1] = F[b]; --b; }
      F[b + 1] = v;
    }
    for (int f = 0; f < nF; ++f) coef_col[f] = F[f];
    nF_sh = nF;
    dinfo[INFO_K_SEL] = nS;
    dinfo[INFO_N_COEF] = nF;
  }
  __syncthreads();
  const unsigned long long tp3 = clock64();
  const int nF = nF_sh;
  // coef[f][t] = sum over support modes touching fold column F[f] of
  //   Re(beta lambda^t) (the f_ra part) or -sg Im(beta lambda^t) (the f_rb part)
  // (per frame t: beta_s lambda_s^t of each support mode once, then the fold columns'
  // sums in support order)
  __shared__ double llog[32], larg_s[32];
  __shared__ int sra[32], srb[32];
  __shared__ double ssg[32];
  if (tid < nS) {
    const double lr = lam[2 * S[tid]], li = lam[2 * S[tid] + 1];
    llog[tid] = log(hypot(lr, li));
    larg_s[tid] = atan2(li, lr);
    int ra, rb;
    double sg;
    mode_rep(pair, S[tid], ra, rb, sg);
    sra[tid] = ra;
    srb[tid] = rb;
    ssg[tid] = sg;
  }
  __syncthreads();
  for (int64_t t = tid; t < m; t += blockDim.x) {
    cplx cs_[32];
    for (int s = 0; s < nS; ++s) {
      const double mag = exp((double)t * llog[s]);
      double sn, cs;
      sincos((double)t * larg_s[s], &sn, &cs);
      cs_[s] = cmul(beta[s], cplx{mag * cs, mag * sn});
    }
    for (int f = 0; f < nF; ++f) {
      double acc = 0.0;
      for (int s = 0; s < nS; ++s) {
        const int ra = sra[s], rb = srb[s];
        const double sg = ssg[s];
        if (ra != F[f] && !(sg != 0.0 && rb == F[f])) continue;
        if (ra == F[f]) acc += cs_[s].r;
        if (sg != 0.0 && rb == F[f]) acc += -sg * cs_[s].i;
      }
      coef[f * m + t] = (float)acc;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    g_omp_prof[0] = tp1 - tp0;
    g_omp_prof[1] = tp2 - tp1;
    g_omp_prof[2] = tp3 - tp2;
    g_omp_prof[3] = clock64() - tp3;
  }
}
void omp_prof_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_omp_prof, sizeof(unsigned long long) * 4); }

// int8 limbs of M: Q = rint(M / s_c * 126 * 128^(L-1)),
// balanced base-128 digits, Mq[(l*kpad + c) * mpad + t]; scale = s_c / (126 128^(L-1)).
__global__ void quantize_kernel(const double* __restrict__ Mf, int64_t n1, int k_eff, int kpad,
                                int64_t mpad, int8_t* __restrict__ Mq, double* __restrict__ scale) {
  const int c = blockIdx.x;
  __shared__ double red[256];
  double mx = 0.0;
  if (c < k_eff)
    for (int64_t t = threadIdx.x; t < n1; t += blockDim.x) mx = fmax(mx, fabs(Mf[t + c * n1]));
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  const double sc = red[0];
  const double full = 126.0 * 2097152.0;  // 126 * 128^(L-1), L = 4
  const double mul = sc > 0.0 ? full / sc : 0.0;
  if (threadIdx.x == 0) scale[c] = sc > 0.0 ? sc / full : 0.0;
  for (int64_t t = threadIdx.x; t < mpad; t += blockDim.x) {
    long long Q = (c < k_eff && t < n1) ? llrint(Mf[t + c * n1] * mul) : 0;
    int8_t d[CDMD_LIMBS];
#pragma unroll
    for (int l = CDMD_LIMBS - 1; l >= 1; --l) {
      const long long q = (Q + 64) >> 7;  // floor((Q + 64) / 128)
      d[l] = (int8_t)(Q - (q << 7));
      Q = q;
    }
    d[0] = (int8_t)Q;
#pragma unroll
    for (int l = 0; l < CDMD_LIMBS; ++l) Mq[((int64_t)l * kpad + c) * mpad + t] = d[l];
  }
}

// Optional substep timing (env CDMD_PROFILE_FIT=1): CUDA events, printed to stderr.
struct FitProf {
  bool on = false;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[16];
  const char* name[16];
  int n = 0;
  void mark(const char* nm) {
    if (!on || n >= 16) return;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], st);
    name[n++] = nm;
  }
  void report() {
    if (!on || n < 2) return;
    cudaEventSynchronize(ev[n - 1]);
    for (int i = 1; i < n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, "[cdmd_fit] %-12s %8.3f ms\n", name[i], ms);
    }
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    n = 0;
  }
};

#define BL(x)                                                                                   \
  do {                                                                                          \
    const cublasStatus_t b_ = (x);                                                              \
    if (b_ != CUBLAS_STATUS_SUCCESS) {                                                          \
      if (getenv("CDMD_DEBUG")) fprintf(stderr, "[cdmd_fit] %s:%d %s: cuBLAS status %d\n", __FILE__, __LINE__, #x, \
                                        (int)b_);                                               \
      return CDMD_ERR_CUDA;                                                                     \
    }                                                                                           \
  } while (0)
// CDMD_DEBUG=1: name the failing call and the CUDA error on stderr
#define CU(x)                                                                               \
  do {                                                                                      \
    const cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                                \
      if (getenv("CDMD_DEBUG")) fprintf(stderr, "[cdmd_fit] %s:%d %s: %s\n", __FILE__, __LINE__, #x, \
                                        cudaGetErrorString(e_));                            \
      return CDMD_ERR_CUDA;                                                                 \
    }                                                                                       \
  } while (0)

// graph capture: the sizes a replay assumes (the previous eager fit's) against this run's
__global__ void graph_check_kernel(int* __restrict__ dinfo, int ke, int K_sel, int n_coef) {
  if (threadIdx.x != 0) return;
  const bool bad = dinfo[INFO_K_EFF] != ke || dinfo[INFO_K_SEL] != K_sel || dinfo[INFO_N_COEF] != n_coef ||
                   dinfo[8] != 0 || dinfo[9] != 0 || dinfo[10] != 0;
  if (bad) dinfo[INFO_FLAGS] |= FLAG_GRAPH_STALE;
}

cdmd_status fit_impl(cdmd_handle h, const void* Y, int64_t ldy, int kind, int64_t p, int64_t m,
                     int k, int K, double dt, cdmd_model* model, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  // k < 0: the Gavish-Donoho optimal hard-threshold rank (Remark 2), at most -k
  const bool gd = k < 0;
  if (gd) k = -k;
  FitWs W{};
  cdmd_status s0 = layout_ws(h, p, m, k, (char*)ws, &W);
  if (s0 != CDMD_OK) return s0;
  if (ws_bytes < W.total) return CDMD_ERR_WORKSPACE;
  const int64_t n1 = m - 1;
  // Stream capture (a CUDA graph of the whole step): no host read-backs -- the sizes come
  // from the previous eager fit of this model, and the graph_check kernel flags a replay
  // whose run disagrees (dev_info[INFO_FLAGS] & FLAG_GRAPH_STALE) so the caller refits eagerly
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(st, &cst));
  const bool cap = cst != cudaStreamCaptureStatusNone;
  if (cap && (gd || model->k_eff < 1)) return CDMD_ERR_UNSUPPORTED;
  FitProf prof;
  prof.on = !cap && getenv("CDMD_PROFILE_FIT") != nullptr;
  prof.st = st;
  prof.mark("start");
  BL(cublasSetStream(h->blas, st));
  if (cusolverDnSetStream(h->solver, st) != CUSOLVER_STATUS_SUCCESS) return CDMD_ERR_CUDA;
  CU(cudaMemsetAsync(W.dinfo, 0, sizeof(int) * 16, st));
  CU(cudaMemsetAsync(model->dev_info, 0, sizeof(int32_t) * 8, st));
  // Y -> fp64
  {
    const int64_t N = p * m;
    note_launch();
    if (kind == CDMD_GAUSSIAN || kind == CDMD_SRFT)
      to_f64_kernel<float><<<(unsigned)ceil_div(N, 256), 256, 0, st>>>((const float*)Y, ldy, p, m, W.Yd);
    else
      to_f64_kernel<int32_t><<<(unsigned)ceil_div(N, 256), 256, 0, st>>>((const int32_t*)Y, ldy, p, m, W.Yd);
    CU(cudaGetLastError());
  }
  const double one = 1.0, zero = 0.0;
  prof.mark("to_f64");
  // G = Y_full^T Y_full
  BL(cublasDgemm(h->blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)m, (int)m, (int)p, &one, W.Yd, (int)p,
                 W.Yd, (int)p, &zero, W.G, (int)m));
  // A = Y^T Y = G[0:m-1, 0:m-1]
  CU(cudaMemcpy2DAsync(W.A, sizeof(double) * n1, W.G, sizeof(double) * m, sizeof(double) * n1, n1,
                       cudaMemcpyDeviceToDevice, st));
  prof.mark("gram");
  size_t hneed = W.sy_host_bytes > W.ge_host_bytes ? W.sy_host_bytes : W.ge_host_bytes;
  if (h->host_ws.size() < hneed + 16) h->host_ws.resize(hneed + 16);
  int64_t top = n1 - 1;
  // Gavish-Donoho needs every singular value of Y (the median): beyond the cluster
  // solver's size (n1 > 510, C5) it takes cuSOLVER's full syevd instead of syevdx
  int smode = syev_mode((int)n1, k);
  if (gd && smode == 2) smode = 1;
  if (gd && smode == 3) smode = eh_supported((int)n1, k) ? 0 : 1;   // the median needs every eigenvalue
  // the median singular value runs over all min(p, m-1) singular values of Y
  const int med_cnt = gd ? (int)(p < n1 ? p : n1) : 0;
  const double beta = (double)(p < n1 ? p : n1) / (double)(p < n1 ? n1 : p);
  const double gd_omega = gd ? 0.56 * beta * beta * beta - 0.95 * beta * beta + 1.82 * beta + 1.43 : 0.0;
  double* med = W.ehw + eh_work_doubles((int)n1, k) - 8;   // two doubles of the eigh workspace slack
  if (cap && smode == 3) {   // mirror the eager path: Householder where Lanczos last fell back
    std::lock_guard<std::mutex> g(h->mu);
    if (h->lz_fell_back.count({n1, k})) smode = eh_supported((int)n1, k) ? 0 : 2;
  }
  if (cap && smode != 0 && smode != 3) return CDMD_ERR_UNSUPPORTED;   // cuSOLVER's host workspaces
  if (smode == 3) {
    // Lanczos: k largest pairs written ascending into (W.w, W.A); dinfo[10] = not converged
    cudaError_t le = launch_eh_lz((int)n1, k, W.G, m, W.w, W.A, W.ehw, W.dinfo + 8, W.dinfo + 10, st);
    if (le == cudaErrorNotSupported) {
      (void)cudaGetLastError();
      smode = eh_supported((int)n1, k) ? 0 : 2;
    } else {
      CU(le);
    }
    top = k - 1;
  }
  if (smode == 0) {
    // cluster tridiagonalisation + bisection + inverse iteration; k largest pairs
    // written ascending into (W.w, W.A) like syevdx
    CU(launch_eh((int)n1, k, W.G, m, W.w, W.A, W.ehw, W.dinfo + 8, med_cnt, med, st));
    top = k - 1;
  } else if (smode == 3) {
  } else if (smode == 2) {
    // only the k largest eigenpairs (1-based indices n1-k+1 .. n1, ascending)
    int64_t meig = 0;
    double vl = 0.0, vu = 0.0;
    if (cusolverDnXsyevdx(h->solver, h->params, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                          CUBLAS_FILL_MODE_LOWER, n1, CUDA_R_64F, W.A, n1, &vl, &vu, n1 - k + 1, n1, &meig,
                          CUDA_R_64F, W.w, CUDA_R_64F, W.sy_dev, W.sy_dev_bytes,
                          W.sy_host_bytes ? h->host_ws.data() : nullptr, W.sy_host_bytes,
                          W.dinfo + 8) != CUSOLVER_STATUS_SUCCESS)
      return CDMD_ERR_CUDA;
    top = k - 1;
  } else {
    if (cusolverDnXsyevd(h->solver, h->params, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n1,
                         CUDA_R_64F, W.A, n1, CUDA_R_64F, W.w, CUDA_R_64F, W.sy_dev, W.sy_dev_bytes,
                         W.sy_host_bytes ? h->host_ws.data() : nullptr, W.sy_host_bytes,
                         W.dinfo + 8) != CUSOLVER_STATUS_SUCCESS)
      return CDMD_ERR_CUDA;
  }
  prof.mark("syevd");
  note_launch();
  select_topk_kernel<<<k, 128, 0, st>>>(W.A, W.w, n1, top, k, W.V, model->sigma, W.dinfo, gd_omega, med_cnt,
                                        smode == 0 ? med : nullptr);
  CU(cudaGetLastError());
  if (!cap) {
    CU(cudaMemcpyAsync(h->host_info, W.dinfo, sizeof(int) * 16, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  if (smode == 3 && !cap) {
    h->lz_runs.fetch_add(1);
    std::lock_guard<std::mutex> g(h->mu);
    if (h->host_info[10] != 0) h->lz_fell_back.insert({n1, k});
    else h->lz_fell_back.erase({n1, k});
  }
  if (smode == 3 && !cap && h->host_info[10] != 0) {
    // a Ritz pair failed the residual test: the Householder solver decides
    h->lz_fallbacks.fetch_add(1);
    if (eh_supported((int)n1, k)) {
      CU(launch_eh((int)n1, k, W.G, m, W.w, W.A, W.ehw, W.dinfo + 8, 0, nullptr, st));
    } else {
      CU(cudaMemcpy2DAsync(W.A, sizeof(double) * n1, W.G, sizeof(double) * m, sizeof(double) * n1, n1,
                           cudaMemcpyDeviceToDevice, st));
      int64_t meig = 0;
      double vl = 0.0, vu = 0.0;
      if (cusolverDnXsyevdx(h->solver, h->params, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I,
                            CUBLAS_FILL_MODE_LOWER, n1, CUDA_R_64F, W.A, n1, &vl, &vu, n1 - k + 1, n1, &meig,
                            CUDA_R_64F, W.w, CUDA_R_64F, W.sy_dev, W.sy_dev_bytes,
                            W.sy_host_bytes ? h->host_ws.data() : nullptr, W.sy_host_bytes,
                            W.dinfo + 8) != CUSOLVER_STATUS_SUCCESS)
        return CDMD_ERR_CUDA;
    }
    note_launch();
    select_topk_kernel<<<k, 128, 0, st>>>(W.A, W.w, n1, top, k, W.V, model->sigma, W.dinfo, gd_omega, med_cnt,
                                          nullptr);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(h->host_info, W.dinfo, sizeof(int) * 16, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  prof.mark("select+sync");
  if (!cap && h->host_info[8] != 0) {
    model->info = h->host_info[8];
    return CDMD_ERR_NUMERIC;
  }
  const int ke = cap ? model->k_eff : h->host_info[INFO_K_EFF];
  model->k_eff = ke;
  if (ke < 1) return CDMD_ERR_NUMERIC;
  // A~ = S^-1 V^T (Y^T Y') V S^-1, Y^T Y' = G[0:m-1, 1:m] = G + m (ld m)
  BL(cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n1, ke, (int)n1, &one, W.G + m, (int)m,
                 W.V, (int)n1, &zero, W.T, (int)n1));
  BL(cublasDgemm(h->blas, CUBLAS_OP_T, CUBLAS_OP_N, ke, ke, (int)n1, &one, W.V, (int)n1, W.T,
                 (int)n1, &zero, W.B, ke));
  note_launch();
  scale_atilde_kernel<<<ke, ke <= 1024 ? ((ke + 31) / 32) * 32 : 1024, 0, st>>>(W.B, model->sigma, ke);
  CU(cudaGetLastError());
  prof.mark("atilde");
  // eig(A~): real nonsymmetric, LAPACK-style output (pairs as Re/Im columns).
  // Default: the single-warp on-device Hessenberg + Francis QR solver (eig.cu);
  // cuSOLVER's hybrid geev for k > 118 or with CDMD_GEEV=cusolver.
  if (use_device_eig(ke)) {
    CU(launch_hqr_eig(ke, W.B, W.Wc, W.VR, W.dinfo + 9, W.Es, st));
  } else if (cap) {
    return CDMD_ERR_UNSUPPORTED;   // cuSOLVER geev's host workspace
  } else {
    size_t d = 0, hb = 0;
    if (cusolverDnXgeev_bufferSize(h->solver, h->params, CUSOLVER_EIG_MODE_NOVECTOR,
                                   CUSOLVER_EIG_MODE_VECTOR, ke, CUDA_R_64F, W.B, ke, CUDA_C_64F,
                                   W.Wc, CUDA_R_64F, nullptr, ke, CUDA_R_64F, W.VR, ke,
                                   CUDA_R_64F, &d, &hb) != CUSOLVER_STATUS_SUCCESS)
      return CDMD_ERR_CUDA;
    if (d > W.ge_dev_bytes) return CDMD_ERR_WORKSPACE;
    if (h->host_ws.size() < hb + 16) h->host_ws.resize(hb + 16);
    if (cusolverDnXgeev(h->solver, h->params, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR,
                        ke, CUDA_R_64F, W.B, ke, CUDA_C_64F, W.Wc, CUDA_R_64F, nullptr, ke,
                        CUDA_R_64F, W.VR, ke, CUDA_R_64F, W.ge_dev, d,
                        hb ? h->host_ws.data() : nullptr, hb, W.dinfo + 9) != CUSOLVER_STATUS_SUCCESS)
      return CDMD_ERR_CUDA;
  }
  prof.mark("geev");
  note_launch();
  canonicalize_kernel<<<1, 256, 0, st>>>(ke, W.Wc, W.VR, model->sigma, dt, model->lambda,
                                        model->omega, model->pair, W.SW, W.dinfo);
  CU(cudaGetLastError());
  // M (folded) = V S^-1 W
  BL(cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n1, ke, ke, &one, W.V, (int)n1, W.SW, ke,
                 &zero, model->Mfold, (int)n1));
  // Gf = M^T (Y'^T Y') M, cf = M^T (Y'^T y1): Y'^T Y' = G + m + 1, Y'^T y1 = G + 1
  BL(cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n1, ke, (int)n1, &one, W.G + m + 1, (int)m,
                 model->Mfold, (int)n1, &zero, W.T2, (int)n1));
  BL(cublasDgemm(h->blas, CUBLAS_OP_T, CUBLAS_OP_N, ke, ke, (int)n1, &one, model->Mfold, (int)n1,
                 W.T2, (int)n1, &zero, W.Gf, ke));
  BL(cublasDgemv(h->blas, CUBLAS_OP_T, (int)n1, ke, &one, model->Mfold, (int)n1, W.G + 1, 1, &zero,
                 W.cf, 1));
  prof.mark("canon+M+gram");
  note_launch();
  {
    const size_t osm = sizeof(double) * (2 * (size_t)ke * ke + 2 * (size_t)ke) + sizeof(int32_t) * (size_t)ke + 16;
    const int staged = osm <= 160 * 1024;
    if (staged) CU(smem_optin(reinterpret_cast<const void*>(omp_kernel)));
    omp_kernel<<<1, 256, staged ? osm : 0, st>>>(ke, K, m, W.Gf, W.cf, W.G, model->pair, model->lambda,
                                                 model->beta, model->support, model->coef, model->coef_col,
                                                 W.dinfo, h->omega_eps, dt, staged);
  }
  CU(cudaGetLastError());
  prof.mark("omp+coef");
  note_launch();
  quantize_kernel<<<model->kpad, 256, 0, st>>>(model->Mfold, n1, ke, model->kpad, model->mpad,
                                               model->Mq, model->Mq_scale);
  CU(cudaGetLastError());
  if (cap) {   // a replay checks itself against the sizes it was captured with
    note_launch();
    graph_check_kernel<<<1, 32, 0, st>>>(W.dinfo, ke, model->K_eff, model->n_coef);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(model->dev_info, W.dinfo, sizeof(int32_t) * 8, cudaMemcpyDeviceToDevice, st));
    return CDMD_OK;
  }
  CU(cudaMemcpyAsync(model->dev_info, W.dinfo, sizeof(int32_t) * 8, cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(h->host_info, W.dinfo, sizeof(int) * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  prof.mark("quant+sync");
  prof.report();
  if (prof.on) {
    unsigned long long t[12];
    hqr_prof_read(t);
    fprintf(stderr, "[cdmd_hqr] orthes %llu  ortran %llu  deflation %llu  m-search %llu  bulges %llu  iters %llu  steps %llu (cycles)\n",
            t[0], t[1], t[2], t[3], t[4], t[5], t[6]);
    unsigned long long o[4];
    omp_prof_read(o);
    fprintf(stderr, "[cdmd_omp] staging %llu  selection %llu  outputs %llu  coef table %llu (cycles)\n", o[0], o[1],
            o[2], o[3]);
    if (t[8] && t[6])   // built with -DCDMD_HQR_PROF2
      fprintf(stderr, "[cdmd_hqr] per bulge step: chain %llu  row update %llu  column update %llu (cycles)\n",
              t[8] / t[6], t[9] / t[6], t[10] / t[6]);
  }
  model->K_eff = h->host_info[INFO_K_SEL];
  model->n_coef = h->host_info[INFO_N_COEF];
  model->dt = dt;
  model->info = h->host_info[9];
  if (h->host_info[9] != 0) return CDMD_ERR_NUMERIC;
  if (h->host_info[INFO_FLAGS] & FLAG_EIG_PAIRING) return CDMD_ERR_NUMERIC;
  return CDMD_OK;
}

}  // namespace cdmd
