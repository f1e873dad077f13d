// eigh.cu — top-k eigenpairs of the symmetric Gram Y^T Y (the truncated SVD of Alg. 1
// step 4, by the method of snapshots) on the device, for n1 = m-1 <= 510.
//
//   1. tridiagonalisation A = Q T Q^T (Householder, LAPACK dsytd2 "lower" order) by
//      ONE 8-CTA thread-block cluster: the lower triangle lives in the CTAs' shared
//      memory (row i on CTA i % 8), vectors move through distributed shared memory,
//      three cluster barriers per column;
//   2. the k largest eigenvalues of T by Sturm-count bisection (one thread each);
//   3. their eigenvectors of T by inverse iteration with partial-pivoting LU of
//      T - lambda I, clusters of close eigenvalues re-orthogonalised (as LAPACK dstein);
//   4. back transformation Z <- Q Z with the stored reflectors (one warp per column).
// It uses 8 SMs for the O(n^3) phase, so several batches' fits overlap (streaming).
#include <cooperative_groups.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"

namespace cg = cooperative_groups;

namespace cdmd {

constexpr int EH_CL = 8;        // CTAs per cluster
constexpr int EH_T = 512;       // threads per CTA
constexpr int EH_NMAX = 510;    // largest n1 whose lower triangle fits in 8 x 227 KB

__host__ __device__ inline int64_t eh_rows(int n, int rank) { return rank < n ? (n - rank + EH_CL - 1) / EH_CL : 0; }
__host__ __device__ inline int64_t eh_asz(int n, int rank) {
  const int64_t nr = eh_rows(n, rank);
  return nr > 0 ? nr * (rank + 1) + 4 * nr * (nr - 1) : 0;
}
// identical shared-memory layout on every CTA (DSMEM addresses map 1:1)
__host__ __device__ inline int64_t eh_asz_max(int n) {
  int64_t mx = 0;
  for (int r = 0; r < EH_CL; ++r) mx = eh_asz(n, r) > mx ? eh_asz(n, r) : mx;
  return mx;
}
// offset of local row slot s (global row i = rank + 8 s, holding columns 0..i)
__device__ __forceinline__ int eh_off(int rank, int s) { return s * (rank + 1) + 4 * s * (s - 1); }

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (warp == 0) {
    s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// G: n x n column-major (ld = ldg), symmetric.  Outputs d[n], e[n-1], tau[n],
// V: n x n column-major holding reflector j in column j (entries j+1 .. n-1, v[j+1] = 1).
__device__ unsigned long long g_eh_prof[8];

// DSMEM exchange primitives: st.async stores into another CTA's shared memory signal
// that CTA's mbarrier (complete_tx); the receiver arms the barrier with the byte count
// it expects.  No cluster-wide barrier (and no GPU-scope fence) per exchange.
__device__ __forceinline__ uint32_t eh_mapa(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void eh_st_async(uint32_t addr, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(mbar)
               : "memory");
}

__global__ void __cluster_dims__(EH_CL, 1, 1) __launch_bounds__(EH_T, 1)
    eh_tridiag_kernel(int n, const double* __restrict__ G, int64_t ldg, double* __restrict__ d,
                      double* __restrict__ e, double* __restrict__ tau_out, double* __restrict__ V) {
  unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tq = clock64();
#ifdef CDMD_EH_PROF
#define EH_TICK(k) do { if (threadIdx.x == 0) { const unsigned long long t_ = clock64(); tp[k] += t_ - tq; tq = t_; } } while (0)
#else
#define EH_TICK(k) do { (void)tq; } while (0)
#endif
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ double sm[];
  const int nr = (int)eh_rows(n, rank);
  const int stride = (n + EH_CL - 1) / EH_CL + 1;     // cbuf row stride (max rows per CTA + 1)
  double* Aloc = sm;                                   // lower-triangle rows of this CTA
  double* xbuf2 = Aloc + eh_asz_max(n);                // [2][n] column below the diagonal (received)
  double* pbuf2 = xbuf2 + 2 * n;                       // [2][n] p = tau A v (received)
  double* cbuf2 = pbuf2 + 2 * n;                       // [2][8][stride] column parts (received)
  double* nrm2 = cbuf2 + 2 * EH_CL * stride;           // [2][8] partial squared norms (received)
  double* kpart2 = nrm2 + 2 * EH_CL;                   // [2][8] partial p.v (received)
  double* v = kpart2 + 2 * EH_CL;                      // [n]
  double* w = v + n;                                   // [n]
  double* rowp = w + n;                                // [stride] row parts of own rows
  double* red = rowp + stride;                         // [40]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 40);   // barX[2], barC[2], barP[2]
  double* cpart = reinterpret_cast<double*>(bars + 8);      // [16 warps][n] column partial sums
  uint64_t* barX = bars;
  uint64_t* barC = bars + 2;
  uint64_t* barP = bars + 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t s_x = tc::smem_u32(xbuf2), s_p = tc::smem_u32(pbuf2), s_c = tc::smem_u32(cbuf2);
  const uint32_t s_n = tc::smem_u32(nrm2), s_k = tc::smem_u32(kpart2), s_b = tc::smem_u32(bars);
  // load own rows (lower part) from G
  for (int s = 0; s < nr; ++s) {
    const int i = rank + EH_CL * s;
    double* row = Aloc + eh_off(rank, s);
    for (int c = tid; c <= i; c += EH_T) row[c] = G[i + (int64_t)c * ldg];
  }
  for (int i = tid; i < (EH_T / 32) * n; i += EH_T) cpart[i] = 0.0;
  if (tid == 0) {
    for (int q = 0; q < 6; ++q) tc::mbar_init(&bars[q], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  cluster.sync();   // barriers initialised and every CTA resident before any DSMEM traffic
  // push own entries of column c (rows l > c) and the partial |x[1:]|^2 to every CTA
  auto push_column = [&](int c) {
    const int b = c & 1;
    double part = 0.0;
    for (int s = tid; s < nr; s += EH_T) {
      const int l = rank + EH_CL * s;
      if (l > c) {
        const double xl = Aloc[eh_off(rank, s) + c];
        if (l > c + 1) part += xl * xl;
        for (int r = 0; r < EH_CL; ++r)
          eh_st_async(eh_mapa(s_x + 8u * (uint32_t)(b * n + l), r), xl, eh_mapa(s_b + 8u * (uint32_t)(0 + b), r));
      }
    }
    part = block_sum(part, red);
    if (tid == 0)
      for (int r = 0; r < EH_CL; ++r)
        eh_st_async(eh_mapa(s_n + 8u * (uint32_t)(b * EH_CL + rank), r), part, eh_mapa(s_b + 8u * (uint32_t)b, r));
  };
  push_column(0);
  int own_gt = nr;                 // own rows l > j (updated as j advances)
  uint32_t phC[2] = {0u, 0u}, phP[2] = {0u, 0u};
  EH_TICK(0);
  for (int j = 0; j < n - 1; ++j) {
    const int b = j & 1;
    if (own_gt > 0 && rank + EH_CL * (nr - own_gt) <= j) --own_gt;   // own row j left the trailing block
    if (tid == 0) tc::mbar_arrive_expect_tx(&barX[b], 8u * (uint32_t)(n - j - 1) + 8u * EH_CL);
    tc::mbar_wait(&barX[b], (uint32_t)(j >> 1) & 1u);
    EH_TICK(2);
    const double* xbuf = xbuf2 + b * n;
    const double* nrm = nrm2 + b * EH_CL;
    double* pbuf = pbuf2 + b * n;
    const double* kpart = kpart2 + b * EH_CL;
    const double* cbuf = cbuf2 + b * EH_CL * stride;
    // (b) Householder reflector (redundantly on every CTA): H = I - tau v v^T
    double xn2 = 0.0;
    for (int r = 0; r < EH_CL; ++r) xn2 += nrm[r];
    const double alpha = xbuf[j + 1];
    const double xnorm = sqrt(xn2);
    double beta = alpha, tau = 0.0;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int i = j + 1 + tid; i < n; i += EH_T) v[i] = (i == j + 1) ? 1.0 : xbuf[i] * scal;
    }
    if (rank == 0 && tid == 0) {
      e[j] = beta;
      tau_out[j] = tau;
    }
    if (rank == (j % EH_CL) && tid == 0) d[j] = Aloc[eh_off(rank, j / EH_CL) + j];
    __syncthreads();
    EH_TICK(1);
    if (tau == 0.0) {   // column j + 1 is already final
      if (j + 1 < n - 1) push_column(j + 1);
      continue;
    }
    for (int i = j + 1 + tid; i < n; i += EH_T)
      if ((i % EH_CL) == rank) V[i + (int64_t)j * n] = v[i];   // reflector for the back transform
    // (c) p = tau A v on the trailing block, one sweep over the own rows (warp per
    //     row): the row part s_l = sum_{i<=l} A[l][i] v_i and the column part
    //     c_i += A[l][i] v_l (per-warp partials), then the column sums go to the
    //     rows' owners
    {
      double* cw = cpart + warp * n;
      for (int s = warp; s < nr; s += EH_T / 32) {
        const int l = rank + EH_CL * s;
        if (l <= j) continue;
        const double* row = Aloc + eh_off(rank, s);
        const double vl = v[l];
        double acc = 0.0;
        for (int i = j + 1 + lane; i < l; i += 32) {
          const double a = row[i];
          acc += a * v[i];
          cw[i] += a * vl;
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) rowp[s] = acc + row[l] * vl;   // own-row partial incl. the diagonal
      }
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < n; i += EH_T) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < EH_T / 32; ++q) {
        acc += cpart[q * n + i];
        cpart[q * n + i] = 0.0;
      }
      const int o = i % EH_CL;   // owner of row i: slot (source rank, local row i / 8)
      eh_st_async(eh_mapa(s_c + 8u * (uint32_t)((b * EH_CL + rank) * stride + i / EH_CL), o), acc,
                  eh_mapa(s_b + 8u * (uint32_t)(2 + b), o));
    }
    if (tid == 0) tc::mbar_arrive_expect_tx(&barC[b], 8u * EH_CL * (uint32_t)own_gt);
    EH_TICK(3);
    tc::mbar_wait(&barC[b], phC[b]);
    phC[b] ^= 1u;
    EH_TICK(2);
    // (d) owners complete p for their rows and send it everywhere; partial p.v
    double kp = 0.0;
    for (int s = tid; s < nr; s += EH_T) {
      const int l = rank + EH_CL * s;
      if (l <= j) continue;
      double pl = rowp[s];
      for (int r = 0; r < EH_CL; ++r) pl += cbuf[r * stride + s];
      pl *= tau;
      kp += pl * v[l];
      for (int r = 0; r < EH_CL; ++r)
        eh_st_async(eh_mapa(s_p + 8u * (uint32_t)(b * n + l), r), pl, eh_mapa(s_b + 8u * (uint32_t)(4 + b), r));
    }
    kp = block_sum(kp, red);
    if (tid == 0) {
      for (int r = 0; r < EH_CL; ++r)
        eh_st_async(eh_mapa(s_k + 8u * (uint32_t)(b * EH_CL + rank), r), kp, eh_mapa(s_b + 8u * (uint32_t)(4 + b), r));
      tc::mbar_arrive_expect_tx(&barP[b], 8u * (uint32_t)(n - j - 1) + 8u * EH_CL);
    }
    EH_TICK(4);
    tc::mbar_wait(&barP[b], phP[b]);
    phP[b] ^= 1u;
    EH_TICK(2);
    // (e) w = p - (tau/2)(p.v) v; rank-2 update of own rows: A -= v w^T + w v^T
    double pv = 0.0;
    for (int r = 0; r < EH_CL; ++r) pv += kpart[r];
    const double K = -0.5 * tau * pv;
    for (int i = j + 1 + tid; i < n; i += EH_T) w[i] = pbuf[i] + K * v[i];
    __syncthreads();
    for (int s = warp; s < nr; s += EH_T / 32) {
      const int l = rank + EH_CL * s;
      if (l <= j) continue;
      double* row = Aloc + eh_off(rank, s);
      const double vl = v[l], wl = w[l];
      for (int i = j + 1 + lane; i <= l; i += 32) row[i] -= vl * w[i] + wl * v[i];
    }
    __syncthreads();
    if (j + 1 < n - 1) push_column(j + 1);
    EH_TICK(5);
  }
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0)
    for (int k = 0; k < 8; ++k) g_eh_prof[k] = tp[k];
  if (rank == ((n - 1) % EH_CL) && tid == 0) d[n - 1] = Aloc[eh_off(rank, (n - 1) / EH_CL) + (n - 1)];
}

// Gershgorin bounds, ||T||, pivmin and e^2 (one block; min / max reductions over the
// threads, exact in any order)
__global__ void eh_prep_kernel(int n, const double* __restrict__ d, const double* __restrict__ e,
                               double* __restrict__ e2, double* __restrict__ bounds) {
  __shared__ double rgl[32], rgu[32], rtn[32], rem[32];
  double gl = INFINITY, gu = -INFINITY, tn = 0.0, emax2 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double ei = i < n - 1 ? e[i] : 0.0;
    e2[i] = ei * ei;
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + fabs(ei);
    gl = fmin(gl, d[i] - r);
    gu = fmax(gu, d[i] + r);
    tn = fmax(tn, fabs(d[i]) + r);
    emax2 = fmax(emax2, ei * ei);
  }
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
    tn = fmax(tn, __shfl_xor_sync(0xffffffffu, tn, o));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
  }
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) {
    rgl[w] = gl;
    rgu[w] = gu;
    rtn[w] = tn;
    rem[w] = emax2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int v = 1; v < nw; ++v) {
      gl = fmin(gl, rgl[v]);
      gu = fmax(gu, rgu[v]);
      tn = fmax(tn, rtn[v]);
      emax2 = fmax(emax2, rem[v]);
    }
    const double pivmin = fmax(2.2250738585072014e-308 * fmax(emax2, 1.0), 1e-300);
    const double pad = 2.0 * 2.220446049250313e-16 * tn * n + 2.0 * pivmin;
    bounds[0] = gl - pad;
    bounds[1] = gu + pad;
    bounds[2] = tn;
    bounds[3] = pivmin;
  }
}

// reciprocal: hardware approximation + one third-order correction r (1 + e + e^2),
// e = 1 - x r (about 1 ulp; used on serial chains -- the inverse iteration's LU --
// where IEEE division is several times longer)
__device__ __forceinline__ double eh_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Sturm counts at EH_NP points at once (independent chains interleave).
// Division-free: the leading principal minors p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}
// (the ratio recurrence q_i = p_i / p_{i-1} multiplied through, so the dependent chain
// is one FMA per step instead of a reciprocal); the count is the number of negative
// ratios, i.e. of sign changes between consecutive minors.  A ratio of magnitude below
// pivmin is replaced by -pivmin as in the ratio form (LAPACK dlaebz); every 8 steps the
// pair (p_{i-1}, p_i) is rescaled by a power of two (signs and ratios unchanged).
constexpr int EH_NP = 4;
__device__ __forceinline__ double eh_pow2_norm(double a) {   // 2^-e with |a| 2^-e in [1, 2)
  const long long bits = __double_as_longlong(a);
  const int ex = (int)((bits >> 52) & 0x7ff);
  return __longlong_as_double((long long)(2046 - ex) << 52);
}
__device__ __forceinline__ void eh_sturm_step(double di, double ei, const double (&x)[EH_NP], double pivmin,
                                              double (&p0)[EH_NP], double (&p1)[EH_NP], int (&cnt)[EH_NP]) {
#pragma unroll
  for (int u = 0; u < EH_NP; ++u) {
    double pn = fma(di - x[u], p1[u], -ei * p0[u]);
    if (fabs(pn) < pivmin * fabs(p1[u])) pn = -pivmin * p1[u];   // ratio clamp
    cnt[u] += ((__double_as_longlong(pn) ^ __double_as_longlong(p1[u])) < 0) ? 1 : 0;
    p0[u] = p1[u];
    p1[u] = pn;
  }
}
// d, e2 in shared memory (uniform across the warp: broadcast loads); the steps come in
// groups of 8 whose operands are loaded before the group, off the dependent chain
__device__ __forceinline__ void eh_sturm_multi(int n, const double* __restrict__ d, const double* __restrict__ e2,
                                               const double (&x)[EH_NP], double pivmin, int (&cnt)[EH_NP]) {
  double p0[EH_NP], p1[EH_NP];   // p_{i-1}, p_i
#pragma unroll
  for (int u = 0; u < EH_NP; ++u) {
    double q = d[0] - x[u];
    if (fabs(q) < pivmin) q = -pivmin;
    p0[u] = 1.0;
    p1[u] = q;
    cnt[u] = q < 0 ? 1 : 0;
  }
  int i = 1;
  for (; i + 8 <= n; i += 8) {
    double dv[8], ev[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      dv[s] = d[i + s];
      ev[s] = e2[i + s - 1];
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) eh_sturm_step(dv[s], ev[s], x, pivmin, p0, p1, cnt);
#pragma unroll
    for (int u = 0; u < EH_NP; ++u) {   // rescale by a power of two every 8 steps
      const double sc = eh_pow2_norm(fabs(p1[u]) > fabs(p0[u]) ? p1[u] : p0[u]);
      p0[u] *= sc;
      p1[u] *= sc;
    }
  }
  for (; i < n; ++i) eh_sturm_step(d[i], e2[i - 1], x, pivmin, p0, p1, cnt);
}

// One warp per wanted eigenvalue: 128-point multisection (7 bits per round; four
// points per lane) on Sturm counts.  The (r+1)-th largest eigenvalue (ascending
// index n-1-r) goes to lam[k-1-r].
// Blocks k and k + 1 (when med_cnt > 0) compute the eigenvalues of descending rank
// (med_cnt - 1) / 2 and med_cnt / 2 into med[0], med[1]: the median of the med_cnt
// largest eigenvalues (Gavish-Donoho rank, Remark 2).
constexpr int EH_BW = 8;   // warps per CTA; BW of them per eigenvalue (8 / BW eigenvalues per CTA)
template <int BW>
__global__ void __launch_bounds__(32 * EH_BW) eh_bisect_kernel(int n, int k, const double* d, const double* e2,
                                                               const double* __restrict__ bounds,
                                                               double* __restrict__ lam, int med_cnt,
                                                               double* __restrict__ med) {
  constexpr int NG = EH_BW / BW;   // eigenvalues per CTA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gi = warp / BW, gt = tid - gi * 32 * BW;   // group, thread within the group
  const int r0 = blockIdx.x * NG + gi;
  extern __shared__ double bsm[];     // d[n], e2[n]
  __shared__ int wsum[NG][2][BW];
  for (int i = tid; i < n; i += 32 * EH_BW) {
    bsm[i] = d[i];
    bsm[n + i] = e2[i];
  }
  __syncthreads();
  if (r0 >= k + (med_cnt > 0 ? 2 : 0)) return;   // a whole group (named barriers below)
  d = bsm;
  e2 = bsm + n;
  const int r = r0 < k ? r0 : (r0 == k ? (med_cnt - 1) / 2 : med_cnt / 2);
  const int idx = n - 1 - r;
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[3];
  constexpr int NPT = 32 * BW * EH_NP;   // points per round, at lo + (hi - lo) t / (NPT + 1)
  for (int round = 0; round < 60; ++round) {
    // stop at 2^-44 relative (sigma = sqrt(theta) to ~1e-14, far inside every use; the
    // inverse iteration refines the vectors): one multisection round fewer than 2 eps at c4
    if (hi - lo <= 0x1p-44 * fmax(fabs(lo), fabs(hi)) + pivmin) break;   // uniform across the group
    double x[EH_NP];
    int c[EH_NP];
#pragma unroll
    for (int u = 0; u < EH_NP; ++u) x[u] = lo + (hi - lo) * (double)(EH_NP * gt + u + 1) / (double)(NPT + 1);
    eh_sturm_multi(n, d, e2, x, pivmin, c);
    // points with count <= idx lie below the eigenvalue; counts are monotone in the
    // point index, so the number below is the total over threads and chains
    int nbl = 0;
#pragma unroll
    for (int u = 0; u < EH_NP; ++u) nbl += c[u] <= idx ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nbl += __shfl_xor_sync(0xffffffffu, nbl, o);
    if (lane == 0) wsum[gi][round & 1][warp - gi * BW] = nbl;
    if (BW > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "r"(32 * BW) : "memory");
    else __syncwarp();
    nbl = 0;
#pragma unroll
    for (int w = 0; w < BW; ++w) nbl += wsum[gi][round & 1][w];
    const double nlo = nbl > 0 ? lo + (hi - lo) * (double)nbl / (double)(NPT + 1) : lo;
    const double nhi = nbl < NPT ? lo + (hi - lo) * (double)(nbl + 1) / (double)(NPT + 1) : hi;
    lo = nlo;
    hi = nhi;
  }
  if (gt == 0) {
    if (r0 < k) lam[k - 1 - r] = 0.5 * (lo + hi);
    else med[r0 - k] = 0.5 * (lo + hi);
  }
}

// Inverse iteration on T - lambda I (LU with partial pivoting), one warp per group
// of eigenvalues closer than 1e-7 ||T|| (re-orthogonalised with modified Gram-Schmidt,
// as LAPACK dstein does for clusters).  lam ascending (k largest); Z[:, q] <-> lam[q].
__global__ void __launch_bounds__(128) eh_invit_kernel(int n, int k, const double* __restrict__ d,
                                                      const double* __restrict__ e,
                                                      const double* __restrict__ bounds,
                                                      const double* __restrict__ lam, double* __restrict__ Z,
                                                      int* __restrict__ info) {
  // one warp (CTA) per group of (numerically) equal eigenvalues; the LU factors and
  // the iterate live in shared memory.  Lane 0 runs the two sequential recurrences
  // (multiplying by stored reciprocal pivots); the lanes share the vector operations.
  extern __shared__ double ismv[];
  const int wid = threadIdx.x >> 5;
  double* ism = ismv + (size_t)wid * (7 * (size_t)n + (n + 7) / 8 + 2);   // this warp's slice
  double* ui = ism;               // 1 / pivot
  double* u1 = ui + n;
  double* u2 = u1 + n;
  double* lm = u2 + n;
  double* z = lm + n;
  double* ds = z + n;             // d, e staged: lane 0's LU reads them on a serial chain
  double* es = ds + n;
  uint8_t* pv = reinterpret_cast<uint8_t*>(es + n);   // rows i, i+1 swapped
  const int lane = threadIdx.x & 31;
  const int grp = blockIdx.x * (int)(blockDim.x >> 5) + wid;   // this warp's group of eigenvalues
  for (int i = lane; i < n; i += 32) {
    ds[i] = d[i];
    es[i] = e[i];
  }
  __syncwarp();
  d = ds;
  e = es;
  const double tnorm = bounds[2];
  const double eps = 2.220446049250313e-16;
  // group c of the descending order r = 0 .. k-1 (q = k-1-r): [r0, r1)
  int g = -1, r0 = 0, r1 = 0;
  for (int r = 0; r < k; ++r) {
    if (r == 0 || fabs(lam[k - r] - lam[k - 1 - r]) > 1e-7 * tnorm) {
      if (g == grp) break;
      ++g;
      r0 = r;
    }
    r1 = r + 1;
  }
  if (g != grp) return;
  auto warp_sum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  for (int r = r0; r < r1; ++r) {
    const int q = k - 1 - r;
    const double lambda = lam[q];
    const double tiny = eps * tnorm;
    if (lane == 0) {   // LU of T - lambda I with partial pivoting
      double a = d[0] - lambda, b = n > 1 ? e[0] : 0.0;
      for (int i = 0; i < n - 1; ++i) {
        const double sub = e[i];
        const double dnext = d[i + 1] - lambda;
        const double enext = (i + 1 < n - 1) ? e[i + 1] : 0.0;
        if (fabs(a) >= fabs(sub)) {
          const double piv = (a != 0.0) ? a : tiny;
          const double ip = eh_rcp(piv);   // the chain multiplies by it (no division subroutine)
          const double mult = (a != 0.0) ? sub * ip : 0.0;
          pv[i] = 0;
          lm[i] = mult;
          ui[i] = ip;
          u1[i] = b;
          u2[i] = 0.0;
          a = dnext - mult * b;
          b = enext;
        } else {
          const double ip = eh_rcp(sub);
          const double mult = a * ip;
          pv[i] = 1;
          lm[i] = mult;
          ui[i] = ip;
          u1[i] = dnext;
          u2[i] = enext;
          a = b - mult * dnext;
          b = -mult * enext;
        }
      }
      ui[n - 1] = 1.0 / ((fabs(a) > tiny) ? a : (a >= 0 ? tiny : -tiny));
      u1[n - 1] = 0.0;
      u2[n - 1] = 0.0;
    }
    for (int i = lane; i < n; i += 32) z[i] = 1.0 + 0.5 * sin(1.0 + 0.713 * i + 0.37 * r);
    __syncwarp();
    for (int it = 0; it < 3; ++it) {
      if (lane == 0) {
        double zc = z[0];                  // forward: row swaps and multipliers
        for (int i = 0; i < n - 1; ++i) {
          const double zn = z[i + 1];
          if (pv[i]) {
            z[i] = zn;
            zc = zc - lm[i] * zn;
          } else {
            z[i] = zc;
            zc = zn - lm[i] * zc;
          }
        }
        z[n - 1] = zc;
        double z1 = 0.0, z2 = 0.0;         // backward: U z = z
        for (int i = n - 1; i >= 0; --i) {
          const double zi = (z[i] - u1[i] * z1 - u2[i] * z2) * ui[i];
          z[i] = zi;
          z2 = z1;
          z1 = zi;
        }
      }
      __syncwarp();
      for (int rr = r0; rr < r; ++rr) {   // orthogonalise within the group (MGS)
        const double* zq = Z + (int64_t)(k - 1 - rr) * n;
        double dot = 0.0;
        for (int i = lane; i < n; i += 32) dot += zq[i] * z[i];
        dot = warp_sum(dot);
        for (int i = lane; i < n; i += 32) z[i] -= dot * zq[i];
        __syncwarp();
      }
      double nn = 0.0;
      for (int i = lane; i < n; i += 32) nn += z[i] * z[i];
      const double inv = 1.0 / sqrt(warp_sum(nn));
      for (int i = lane; i < n; i += 32) z[i] *= inv;
      __syncwarp();
    }
    // sign: the largest-magnitude entry (first on ties) positive
    double best = -1.0;
    int im = n;
    for (int i = lane; i < n; i += 32) {
      const double v = fabs(z[i]);
      if (v > best) { best = v; im = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, im, o);
      if (ob > best || (ob == best && oi < im)) { best = ob; im = oi; }
    }
    const double sg = z[im] < 0 ? -1.0 : 1.0;
    for (int i = lane; i < n; i += 32) Z[i + (int64_t)q * n] = sg * z[i];
    __syncwarp();
  }
  if (grp == 0 && lane == 0) *info = 0;
}

// Z <- Q Z, Q = H_0 H_1 ... H_{n-3} (applied last to first): one warp per column of
// Z, the column in registers (element i = lane + 32 t), the next reflector's
// entries loaded while the current one is applied.
constexpr int EH_ZR = (EH_NMAX + 31) / 32;
__global__ void __launch_bounds__(128) eh_backtransform_kernel(int n, int k, const double* __restrict__ V,
                                                               const double* __restrict__ tau,
                                                               double* __restrict__ Z) {
  const int lane = threadIdx.x & 31;
  const int col = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (col >= k) return;
  double z[EH_ZR], vn[EH_ZR];
  double* zc = Z + (int64_t)col * n;
#pragma unroll
  for (int t = 0; t < EH_ZR; ++t) {
    const int i = lane + 32 * t;
    z[t] = i < n ? zc[i] : 0.0;
  }
  auto load_v = [&](int j) {
#pragma unroll
    for (int t = 0; t < EH_ZR; ++t) {
      const int i = lane + 32 * t;
      vn[t] = (j >= 0 && i > j && i < n) ? __ldg(V + (int64_t)j * n + i) : 0.0;
    }
  };
  int j = n - 2;
  load_v(j);
  for (; j >= 0; --j) {
    double v[EH_ZR];
#pragma unroll
    for (int t = 0; t < EH_ZR; ++t) v[t] = vn[t];
    const double tj = __ldg(tau + j);
    load_v(j - 1);
    if (j >= 4 && 16 * lane < n) {   // reflector j - 4 into L1: one 128-B line per lane
      const double* pf = V + (int64_t)(j - 4) * n + 16 * lane;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(pf));
    }
    if (tj == 0.0) continue;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int t = 0; t < EH_ZR; t += 2) {
      s0 = fma(v[t], z[t], s0);
      if (t + 1 < EH_ZR) s1 = fma(v[t + 1], z[t + 1], s1);
    }
    double sacc = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    sacc *= tj;
#pragma unroll
    for (int t = 0; t < EH_ZR; ++t) z[t] = fma(-sacc, v[t], z[t]);
  }
#pragma unroll
  for (int t = 0; t < EH_ZR; ++t) {
    const int i = lane + 32 * t;
    if (i < n) zc[i] = z[t];
  }
}

// eh_invit_kernel: EH_IW warps per CTA, a group of eigenvalues each, with their own slice
constexpr int EH_IW = 4;
static size_t eh_invit_smem(int n) { return sizeof(double) * EH_IW * (7 * (size_t)n + (n + 7) / 8 + 2); }

size_t eh_tridiag_smem(int n) {
  const int64_t stride = (n + EH_CL - 1) / EH_CL + 1;
  return sizeof(double) * ((size_t)eh_asz_max(n) + 6 * (size_t)n + 2 * EH_CL * stride + 4 * EH_CL + stride + 40 +
                           8 + (size_t)(EH_T / 32) * n);
}

bool eh_supported(int n, int k) { return n >= 3 && n <= EH_NMAX && k <= 256 && eh_tridiag_smem(n) <= 227 * 1024; }

size_t eh_work_doubles(int n, int k) {
  return (size_t)n * n + 7 * (size_t)n + (size_t)n * k + 128;
}

// G (n x n, ld ldg) -> lam[k] (ascending: the k largest), Zout (n x k column-major, ld n).
void eh_prof_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_eh_prof, sizeof(unsigned long long) * 8); }

// med_cnt > 0: also the median of the med_cnt largest eigenvalues into med[0..1]
cudaError_t launch_eh(int n, int k, const double* G, int64_t ldg, double* lam, double* Zout, double* work,
                      int* info, int med_cnt, double* med, cudaStream_t st) {
  double* V = work;
  double* d = V + (size_t)n * n;
  double* e = d + n;
  double* tau = e + n;
  double* wk = tau + n;
  cudaError_t err;
  // CDMD_PROFILE_FIT: CUDA events between the solver's kernels, printed to stderr
  cudaStreamCaptureStatus cst_ = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cst_);
  const bool prof = cst_ == cudaStreamCaptureStatusNone && getenv("CDMD_PROFILE_FIT") != nullptr;
  cudaEvent_t ev[6];
  if (prof) for (int i = 0; i < 6; ++i) { cudaEventCreate(&ev[i]); }
  auto mark = [&](int i) { if (prof) cudaEventRecord(ev[i], st); };
  mark(0);
  {
    const size_t smem = eh_tridiag_smem(n);
    err = smem_optin(reinterpret_cast<const void*>(eh_tridiag_kernel));
    if (err != cudaSuccess) return err;
    note_launch();
    eh_tridiag_kernel<<<EH_CL, EH_T, smem, st>>>(n, G, ldg, d, e, tau, V);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
  }
  mark(1);
  double* e2 = wk;
  double* bounds = e2 + n;
  note_launch();
  eh_prep_kernel<<<1, 256, 0, st>>>(n, d, e, e2, bounds);
  note_launch();
  eh_bisect_kernel<EH_BW><<<k + (med_cnt > 0 ? 2 : 0), 32 * EH_BW, sizeof(double) * 2 * (size_t)n, st>>>(
      n, k, d, e2, bounds, lam, med_cnt, med);
  mark(2);
  note_launch();
  err = smem_optin(reinterpret_cast<const void*>(eh_invit_kernel));
  if (err != cudaSuccess) return err;
  eh_invit_kernel<<<(unsigned)ceil_div(k, EH_IW), 32 * EH_IW, eh_invit_smem(n), st>>>(n, k, d, e, bounds, lam, Zout,
                                                                                      info);
  mark(3);
  note_launch();
  eh_backtransform_kernel<<<(unsigned)ceil_div(k, 4), 128, 0, st>>>(n, k, V, tau, Zout);
  mark(4);
  if (prof) {
    cudaEventSynchronize(ev[4]);
    float t[4];
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    fprintf(stderr, "[cdmd_eh] tridiag %.3f  bisect %.3f  invit %.3f  backtransform %.3f ms\n", t[0], t[1], t[2],
            t[3]);
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  }
  return cudaGetLastError();
}

// Lanczos variant (lanczos.cu): the same outputs as launch_eh (k largest pairs ascending
// in lam, Zout) from a Krylov space of J = lz_steps(n, k) << n; *flag = 0 when every Ritz
// pair passed the residual test, else the caller reruns launch_eh.  The returned error
// is cudaErrorNotSupported when this device cannot co-schedule the 16-CTA cluster.
bool lz_supported(int n, int k);
int lz_steps(int n, int k);
void lz_prof_read(unsigned long long* out);
cudaError_t launch_lz(int n, int J, const double* G, int64_t ldg, double* alpha, double* beta, double* Q, int* jdone,
                      cudaStream_t st);
cudaError_t launch_lz_check(int J, int k, const double* beta, const double* lam1, const double* S, const int* jdone,
                            int* flag, cudaStream_t st);
cudaError_t launch_lz_ritz(int n, int J, int k, const double* Q, const double* S, const double* lam1, double* lam,
                           double* Z, cudaStream_t st);

cudaError_t launch_eh_lz(int n, int k, const double* G, int64_t ldg, double* lam, double* Zout, double* work,
                         int* info, int* flag, cudaStream_t st) {
  const int J = lz_steps(n, k);
  // work: Q (n x J) | alpha, beta, e2 (J each) | bounds (8) | lam1 (k + 1) | S (J x (k + 1)) | jdone
  double* Q = work;
  double* al = Q + (size_t)n * J;
  double* be = al + J;
  double* e2 = be + J;
  double* bounds = e2 + J;
  double* lam1 = bounds + 8;
  double* S = lam1 + (k + 1);
  int* jdone = reinterpret_cast<int*>(S + (size_t)J * (k + 1));
  cudaError_t err;
  cudaStreamCaptureStatus cst_ = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cst_);
  const bool prof = cst_ == cudaStreamCaptureStatusNone && getenv("CDMD_PROFILE_FIT") != nullptr;
  cudaEvent_t ev[6];
  if (prof) for (int i = 0; i < 6; ++i) cudaEventCreate(&ev[i]);
  auto mark = [&](int i) { if (prof) cudaEventRecord(ev[i], st); };
  mark(0);
  if ((err = launch_lz(n, J, G, ldg, al, be, Q, jdone, st)) != cudaSuccess) return err;
  mark(1);
  note_launch();
  eh_prep_kernel<<<1, 256, 0, st>>>(J, al, be, e2, bounds);
  mark(4);
  note_launch();
  // eight warps per eigenvalue (lowest latency; packing four eigenvalues to a CTA with
  // eh_bisect_kernel<2> holds a quarter of the SMs but measured +30 us and no streaming gain)
  eh_bisect_kernel<EH_BW><<<(unsigned)(k + 1), 32 * EH_BW, sizeof(double) * 2 * (size_t)J, st>>>(
      J, k + 1, al, e2, bounds, lam1, 0, nullptr);
  mark(5);
  if ((err = smem_optin(reinterpret_cast<const void*>(eh_invit_kernel))) != cudaSuccess) return err;
  note_launch();
  eh_invit_kernel<<<(unsigned)ceil_div(k + 1, EH_IW), 32 * EH_IW, eh_invit_smem(J), st>>>(J, k + 1, al, be, bounds,
                                                                                          lam1, S, info);
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  mark(2);
  if ((err = launch_lz_check(J, k, be, lam1, S, jdone, flag, st)) != cudaSuccess) return err;
  if ((err = launch_lz_ritz(n, J, k, Q, S, lam1, lam, Zout, st)) != cudaSuccess) return err;
  mark(3);
  if (prof) {
    cudaEventSynchronize(ev[3]);
    float t[3];
    for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    float tp = 0.f, tb = 0.f;
    cudaEventElapsedTime(&tp, ev[1], ev[4]);
    cudaEventElapsedTime(&tb, ev[4], ev[5]);
    fprintf(stderr, "[cdmd_lz] J %d  lanczos %.3f  tridiag eig %.3f (prep %.3f bisect %.3f)  ritz %.3f ms\n", J, t[0],
            t[1], tp, tb, t[2]);
    unsigned long long pc[12];
    lz_prof_read(pc);
    if (pc[0])   // built with -DCDMD_LZ_PROF
      fprintf(stderr, "[cdmd_lz] cycles/step: matvec %llu sendA %llu h1 %llu z1 %llu sendB %llu h2 %llu z2 %llu xQ %llu\n",
              pc[0] / J, pc[1] / J, pc[2] / J, pc[3] / J, pc[4] / J, pc[5] / J, pc[6] / J, pc[7] / J);
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  }
  return cudaSuccess;
}

}  // namespace cdmd
