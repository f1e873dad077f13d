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

#include "common.cuh"

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
__device__ __forceinline__ int64_t eh_off(int rank, int64_t s) { return s * (rank + 1) + 4 * s * (s - 1); }

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
__global__ void __cluster_dims__(EH_CL, 1, 1) __launch_bounds__(EH_T, 1)
    eh_tridiag_kernel(int n, const double* __restrict__ G, int64_t ldg, double* __restrict__ d,
                      double* __restrict__ e, double* __restrict__ tau_out, double* __restrict__ V) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  extern __shared__ double sm[];
  const int64_t nr = eh_rows(n, rank);
  const int64_t stride = (n + EH_CL - 1) / EH_CL + 1;  // cbuf row stride (max rows per CTA + 1)
  double* Aloc = sm;                                   // lower-triangle rows of this CTA
  double* xbuf = Aloc + eh_asz_max(n);                 // [n] column below the diagonal
  double* pbuf = xbuf + n;                             // [n] p = tau A v
  double* cbuf = pbuf + n;                             // [8][stride] column contributions
  double* nrm = cbuf + EH_CL * stride;                 // [8] partial squared norms
  double* kpart = nrm + EH_CL;                         // [8] partial p.v
  double* v = kpart + EH_CL;                           // [n]
  double* w = v + n;                                   // [n]
  double* red = w + n;                                 // [33]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // load own rows (lower part) from G
  for (int64_t s = 0; s < nr; ++s) {
    const int64_t i = rank + EH_CL * s;
    double* row = Aloc + eh_off(rank, s);
    for (int64_t c = tid; c <= i; c += EH_T) row[c] = G[i + c * ldg];
  }
  __syncthreads();
  cluster.sync();
  for (int j = 0; j < n - 1; ++j) {
    // (a) push own entries of column j (rows i > j) and the partial norm of x[1:]
    double part = 0.0;
    for (int64_t s = tid; s < nr; s += EH_T) {
      const int64_t i = rank + EH_CL * s;
      if (i > j) {
        const double xi = Aloc[eh_off(rank, s) + j];
        if (i > j + 1) part += xi * xi;
        for (int r = 0; r < EH_CL; ++r) cluster.map_shared_rank(xbuf, r)[i] = xi;
      }
    }
    part = block_sum(part, red);
    if (tid == 0)
      for (int r = 0; r < EH_CL; ++r) cluster.map_shared_rank(nrm, r)[rank] = part;
    cluster.sync();
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
    if (tau != 0.0) {
      for (int i = j + 1 + tid; i < n; i += EH_T)
        if ((i % EH_CL) == rank) V[i + (int64_t)j * n] = v[i];   // reflector for the back transform
      // (c) p = tau A v on the trailing block: own-row part (warp per row) and
      //     column contributions to every row (thread per column), reduce-scattered
      for (int64_t s = warp; s < nr; s += EH_T / 32) {
        const int64_t l = rank + EH_CL * s;
        if (l <= j) continue;
        const double* row = Aloc + eh_off(rank, s);
        double acc = 0.0;
        for (int64_t i = j + 1 + lane; i <= l; i += 32) acc += row[i] * v[i];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) pbuf[l] = acc;   // own-row partial (only own rows are read)
      }
      for (int i = j + 1 + tid; i < n; i += EH_T) {
        double acc = 0.0;
        int64_t s0 = (i - rank) / EH_CL + 1;   // first own row l > i
        if (i < rank) s0 = 0;
        for (int64_t s = s0; s < nr; ++s) {
          const int64_t l = rank + EH_CL * s;
          if (l > i) acc += Aloc[eh_off(rank, s) + i] * v[l];
        }
        // to the owner of row i, slot (source rank, local row i / 8)
        cluster.map_shared_rank(cbuf, i % EH_CL)[(int64_t)rank * stride + i / EH_CL] = acc;
      }
      cluster.sync();
      // (d) owners complete p for their rows and push it; partial p.v
      double kp = 0.0;
      for (int64_t s = tid; s < nr; s += EH_T) {
        const int64_t l = rank + EH_CL * s;
        if (l <= j) continue;
        double pl = pbuf[l];
        for (int r = 0; r < EH_CL; ++r) pl += cbuf[(int64_t)r * stride + s];
        pl *= tau;
        kp += pl * v[l];
        for (int r = 0; r < EH_CL; ++r) cluster.map_shared_rank(pbuf, r)[l] = pl;
      }
      kp = block_sum(kp, red);
      if (tid == 0)
        for (int r = 0; r < EH_CL; ++r) cluster.map_shared_rank(kpart, r)[rank] = kp;
      cluster.sync();
      // (e) w = p - (tau/2)(p.v) v; rank-2 update of own rows: A -= v w^T + w v^T
      double pv = 0.0;
      for (int r = 0; r < EH_CL; ++r) pv += kpart[r];
      const double K = -0.5 * tau * pv;
      for (int i = j + 1 + tid; i < n; i += EH_T) w[i] = pbuf[i] + K * v[i];
      __syncthreads();
      for (int64_t s = warp; s < nr; s += EH_T / 32) {
        const int64_t l = rank + EH_CL * s;
        if (l <= j) continue;
        double* row = Aloc + eh_off(rank, s);
        const double vl = v[l], wl = w[l];
        for (int64_t i = j + 1 + lane; i <= l; i += 32) row[i] -= vl * w[i] + wl * v[i];
      }
      __syncthreads();
    }
    cluster.sync();   // buffers (xbuf, nrm, v) are rewritten by the next column
  }
  if (rank == ((n - 1) % EH_CL) && tid == 0) d[n - 1] = Aloc[eh_off(rank, (n - 1) / EH_CL) + (n - 1)];
}

// Sturm count: number of eigenvalues of T(d, e) smaller than x
__device__ int eh_sturm(int n, const double* d, const double* e2, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  if (q < 0) ++cnt;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) ++cnt;
  }
  return cnt;
}

// One block.  The (r+1)-th largest eigenvalue of T goes to lam[k-1-r] (ascending
// output, as syevd) and its eigenvector to Z[:, k-1-r]
// eigenvector of T (unit norm).  Clusters (relative gap <= 1e-3 of ||T||) are
// handled by one thread with modified Gram-Schmidt between inverse iterations.
__global__ void __launch_bounds__(256) eh_tridiag_eig_kernel(int n, int k, const double* __restrict__ d,
                                                             const double* __restrict__ e, double* __restrict__ lam,
                                                             double* __restrict__ Z, double* __restrict__ work,
                                                             int* __restrict__ info) {
  extern __shared__ double sh[];
  double* sd = sh;            // n
  double* se = sd + n;        // n
  double* se2 = se + n;       // n
  double* slam = se2 + n;     // k
  __shared__ double tnorm_s, pivmin_s, gl_s, gu_s;
  __shared__ int cstart[256];
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += blockDim.x) {
    sd[i] = d[i];
    se[i] = i < n - 1 ? e[i] : 0.0;
    se2[i] = se[i] * se[i];
  }
  __syncthreads();
  if (tid == 0) {
    double gl = sd[0], gu = sd[0], tn = 0.0, emax2 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double r = (i > 0 ? fabs(se[i - 1]) : 0.0) + (i < n - 1 ? fabs(se[i]) : 0.0);
      gl = fmin(gl, sd[i] - r);
      gu = fmax(gu, sd[i] + r);
      tn = fmax(tn, fabs(sd[i]) + r);
      emax2 = fmax(emax2, se2[i]);
    }
    tnorm_s = tn;
    pivmin_s = fmax(2.2250738585072014e-308 * fmax(emax2, 1.0), 1e-300);
    const double pad = 2.0 * 2.220446049250313e-16 * tn * n + 2.0 * pivmin_s;
    gl_s = gl - pad;
    gu_s = gu + pad;
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  // ---- bisection: eigenvalue with ascending index n-1-r
  for (int r = tid; r < k; r += blockDim.x) {
    const int idx = n - 1 - r;  // want count(< x) = idx at the lower end
    double lo = gl_s, hi = gu_s;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (hi - lo <= 2.0 * eps * fmax(fabs(lo), fabs(hi)) + pivmin_s) break;
      if (eh_sturm(n, sd, se2, mid, pivmin_s) > idx) hi = mid;
      else lo = mid;
    }
    slam[r] = 0.5 * (lo + hi);
  }
  __syncthreads();
  // ---- clusters (descending order): start indices
  if (tid == 0) {
    int nc = 0;
    for (int r = 0; r < k; ++r)
      if (r == 0 || fabs(slam[r - 1] - slam[r]) > 1e-3 * tnorm_s) cstart[nc++] = r;
    cstart[nc] = k;
    cstart[255] = nc;
  }
  __syncthreads();
  const int ncl = cstart[255];
  // ---- inverse iteration, one thread per cluster; work: 6 n doubles per thread
  for (int c = tid; c < ncl; c += blockDim.x) {
    double* wk = work + (int64_t)c * 6 * n;
    double* u = wk;            // U diagonal
    double* u1 = u + n;        // first superdiagonal
    double* u2 = u1 + n;       // second superdiagonal
    double* lm = u2 + n;       // multipliers
    double* z = lm + n;        // iterate
    double* piv = z + n;       // row interchange flags
    for (int r = cstart[c]; r < cstart[c + 1]; ++r) {
      const double lambda = slam[r];
      // LU with partial pivoting of T - lambda I (rows i, i+1 may swap)
      const double tiny = eps * tnorm_s;
      double a = sd[0] - lambda, b = n > 1 ? se[0] : 0.0;
      for (int i = 0; i < n - 1; ++i) {
        const double sub = se[i];            // T[i+1][i]
        const double dnext = sd[i + 1] - lambda;
        const double enext = (i + 1 < n - 1) ? se[i + 1] : 0.0;
        if (fabs(a) >= fabs(sub)) {          // no interchange
          piv[i] = 0.0;
          const double mult = (a != 0.0) ? sub / a : 0.0;
          lm[i] = mult;
          u[i] = (a != 0.0) ? a : tiny;
          u1[i] = b;
          u2[i] = 0.0;
          a = dnext - mult * b;
          b = enext;
        } else {                             // interchange rows i and i+1
          piv[i] = 1.0;
          const double mult = a / sub;
          lm[i] = mult;
          u[i] = sub;
          u1[i] = dnext;
          u2[i] = enext;
          a = b - mult * dnext;
          b = -mult * enext;
        }
      }
      u[n - 1] = (fabs(a) > tiny) ? a : (a >= 0 ? tiny : -tiny);
      // start vector (deterministic, non-degenerate)
      for (int i = 0; i < n; ++i) z[i] = 1.0 + 0.5 * sin(1.0 + 0.713 * i + 0.37 * r);
      for (int it = 0; it < 6; ++it) {
        // forward: apply the row interchanges and multipliers (L^-1 P)
        for (int i = 0; i < n - 1; ++i) {
          if (piv[i] != 0.0) {
            const double t = z[i];
            z[i] = z[i + 1];
            z[i + 1] = t - lm[i] * z[i];
          } else {
            z[i + 1] -= lm[i] * z[i];
          }
        }
        // back substitution with U (diag u, super u1, u2)
        for (int i = n - 1; i >= 0; --i) {
          double s = z[i];
          if (i + 1 < n) s -= u1[i] * z[i + 1];
          if (i + 2 < n) s -= u2[i] * z[i + 2];
          z[i] = s / u[i];
        }
        // re-orthogonalise against the earlier members of the cluster
        for (int q = cstart[c]; q < r; ++q) {
          double dot = 0.0;
          const double* zq = Z + (int64_t)(k - 1 - q) * n;
          for (int i = 0; i < n; ++i) dot += zq[i] * z[i];
          for (int i = 0; i < n; ++i) z[i] -= dot * zq[i];
        }
        double nn = 0.0;
        for (int i = 0; i < n; ++i) nn += z[i] * z[i];
        const double inv = 1.0 / sqrt(nn);
        for (int i = 0; i < n; ++i) z[i] *= inv;
      }
      // sign convention: largest component positive
      int im = 0;
      for (int i = 1; i < n; ++i)
        if (fabs(z[i]) > fabs(z[im])) im = i;
      const double sg = z[im] < 0 ? -1.0 : 1.0;
      for (int i = 0; i < n; ++i) Z[i + (int64_t)(k - 1 - r) * n] = sg * z[i];
      lam[k - 1 - r] = slam[r];
    }
  }
  if (tid == 0) *info = 0;
}

// Z <- Q Z, Q = H_0 H_1 ... H_{n-2}; one warp per column of Z (k columns).
__global__ void __launch_bounds__(512) eh_backtransform_kernel(int n, int k, const double* __restrict__ V,
                                                               const double* __restrict__ tau,
                                                               double* __restrict__ Z) {
  const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= k) return;
  double* z = Z + (int64_t)col * n;
  for (int j = n - 2; j >= 0; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;
    const double* vj = V + (int64_t)j * n;
    double s = 0.0;
    for (int i = j + 1 + lane; i < n; i += 32) s += vj[i] * z[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    s *= tj;
    for (int i = j + 1 + lane; i < n; i += 32) z[i] -= s * vj[i];
    __syncwarp();
  }
}

size_t eh_tridiag_smem(int n) {
  const int64_t stride = (n + EH_CL - 1) / EH_CL + 1;
  return sizeof(double) * ((size_t)eh_asz_max(n) + 4 * (size_t)n + EH_CL * stride + 2 * EH_CL + 40);
}

bool eh_supported(int n, int k) { return n >= 3 && n <= EH_NMAX && k <= 256 && eh_tridiag_smem(n) <= 227 * 1024; }

size_t eh_work_doubles(int n, int k) {
  return (size_t)n * n + 3 * (size_t)n + (size_t)n * k + 6 * (size_t)n * k + 64;
}

// G (n x n, ld ldg) -> lam[k] (ascending: the k largest), Zout (n x k column-major, ld n).
cudaError_t launch_eh(int n, int k, const double* G, int64_t ldg, double* lam, double* Zout, double* work,
                      int* info, cudaStream_t st) {
  double* V = work;
  double* d = V + (size_t)n * n;
  double* e = d + n;
  double* tau = e + n;
  double* wk = tau + n;
  const size_t smem = eh_tridiag_smem(n);
  cudaError_t err = cudaFuncSetAttribute(eh_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  eh_tridiag_kernel<<<EH_CL, EH_T, smem, st>>>(n, G, ldg, d, e, tau, V);
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  const size_t smem2 = sizeof(double) * (3 * (size_t)n + k);
  err = cudaFuncSetAttribute(eh_tridiag_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  if (err != cudaSuccess) return err;
  eh_tridiag_eig_kernel<<<1, 256, smem2, st>>>(n, k, d, e, lam, Zout, wk, info);
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  eh_backtransform_kernel<<<(unsigned)ceil_div(k, 16), 512, 0, st>>>(n, k, V, tau, Zout);
  return cudaGetLastError();
}

}  // namespace cdmd
