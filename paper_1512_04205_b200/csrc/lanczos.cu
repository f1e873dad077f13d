// lanczos.cu — the k largest eigenpairs of the symmetric Gram Y^T Y (Alg. 1 step 4,
// P:339, by the method of snapshots) by Lanczos with full reorthogonalisation, on ONE
// 16-CTA thread-block cluster.
//
// The one-stage Householder tridiagonalisation (eigh.cu) is a chain of n - 2 dependent
// column steps, each a trailing matvec plus cluster exchanges.  The top k eigenpairs of
// the snapshot Gram converge in a Krylov space of about 2.2 k (measured on the c4 sketch:
// Ritz values to 2e-13 and every Ritz vector to 1e-11 of LAPACK's after 125 steps for
// k = 50, n = 499), so Lanczos reaches the same result in J << n steps:
//   z = G q_j                           (G rows resident in shared memory, 32 per CTA)
//   h1 = Q^T z, z -= Q h1               (two-pass classical Gram-Schmidt against the whole
//   h2 = Q^T z, z -= Q h2                basis; Q's rows resident with their G rows)
//   alpha_j = h1_j + h2_j, beta_j = ||z|| (||z||^2 = ||z_1||^2 - ||h2||^2), q_{j+1} = z / beta_j
// with three cluster exchanges per step (the partial sums of h1; of h2 and ||z_1||^2;
// the rows of q_{j+1}), bulk DSMEM copies issued by sixteen lanes in parallel.  The
// tridiagonal T_J = tridiag(alpha, beta) then goes through eigh.cu's bisection and
// inverse iteration for its k + 1 largest pairs, V = Q S (cuBLAS DGEMM), and the
// Lanczos residual |beta_{J-1}| |s_{J-1,i}| = ||G v_i - theta_i v_i|| decides whether the
// Ritz pairs are converged (relative to the gap to theta_k); if not, cdmd_fit falls back
// to the Householder solver.
#include <atomic>
#include <cooperative_groups.h>
#include <math.h>

#include "common.cuh"
#include "tc.cuh"

namespace cg = cooperative_groups;

namespace cdmd {

constexpr int LZ_CL = 16;       // CTAs per cluster
constexpr int LZ_T = 512;       // threads per CTA
// per-phase cycle totals of CTA 0's thread 0 (built with -DCDMD_LZ_PROF; printed by
// launch_eh_lz under CDMD_PROFILE_FIT)
__device__ unsigned long long g_lz_prof[12];
void lz_prof_read(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_lz_prof, sizeof(unsigned long long) * 12); }
#ifdef CDMD_LZ_PROF
#define LZ_TICK(k)                                   \
  do {                                               \
    if (tid == 0) {                                  \
      const unsigned long long t_ = clock64();       \
      tps[k] += t_ - tq;                             \
      tq = t_;                                       \
    }                                                \
  } while (0)
#else
#define LZ_TICK(k) \
  do {             \
  } while (0)
#endif

__device__ __forceinline__ void lz_st_async(uint32_t cluster_addr, double v, uint32_t cluster_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(cluster_addr),
               "l"(__double_as_longlong(v)), "r"(cluster_mbar)
               : "memory");
}

// entries c < count owned by CTA t (c % 16 == t)
__device__ __forceinline__ int lz_owned(int count, int t) { return count > t ? (count - 1 - t) / LZ_CL + 1 : 0; }

// The two variants: SMALL (n <= 512: 32 rows per CTA, the rows of G in registers, 32
// doubles per thread, kept in the exchange order of q) and BIG (n <= 1024: 64 rows per
// CTA, the rows of G streamed from L2 every step -- 8 MB of G stay L2-resident -- against
// q reassembled in natural order in shared memory).
template <bool BIG>
struct LzCfg {
  static constexpr int R = BIG ? 64 : 32;      // rows per CTA (row l on CTA l % 16, slot l / 16)
  static constexpr int NMAX = LZ_CL * R;       // 512 / 1024
  static constexpr int JM = BIG ? 288 : 144;   // Krylov dimension cap (2.25 k + 9 <= JM)
  static constexpr int NS = JM / LZ_CL + 1;    // slots per owner: entries c = 16 slot + owner, c <= JM
  static constexpr int AS = NS + 1;            // gathered row: the owner's slots and its sum of squares
  static constexpr int QLD = BIG ? R + 1 : R;  // row stride of qp (padded: conflict-free reassembly)
  static constexpr int RH = R / 32;            // rows per half-warp
};

// dynamic shared memory: Qs[R][JM] | rsA[16][NS] | agA[16][AS] | rsB[16][NS] | agB[16][AS] |
// qp[16][QLD] | qn[NMAX] (BIG) | zsh[R] | bars[5].  The two projections h1 = Q^T z,
// h2 = Q^T z1 are cluster all-reduces done as reduce-scatter + all-gather with st.async
// (entry c is summed by CTA c % 16, from the 16 partials it receives in rs*, then sent to
// every CTA's ag*): a few hundred bytes per CTA per hop instead of every partial vector to
// every CTA.  qp holds q_j in the exchange's order, qp[QLD r + s] = q_j[r + 16 s] (CTA r's
// slot s) -- SMALL keeps its register copy of G in that order; BIG reassembles q_j in
// natural order (qn) for the streamed rows.  Barriers: RS_A, AG_A, RS_B, AG_B, Q, each
// completing once per step (parity j & 1); B carries ||z1||^2 as entry nc.
template <bool BIG>
size_t lz_smem_bytes_t() {
  using C = LzCfg<BIG>;
  return sizeof(double) * ((size_t)C::R * C::JM + 2 * (size_t)LZ_CL * (C::NS + C::AS) + (size_t)LZ_CL * C::QLD +
                           (BIG ? (size_t)C::NMAX : 0) + C::R) +
         64;
}

template <bool BIG>
__global__ void __launch_bounds__(LZ_T, 1)
    lz_kernel(int n, const double* __restrict__ G, int64_t ldg, int J, double* __restrict__ alpha,
              double* __restrict__ beta, double* __restrict__ Qout, int* __restrict__ jdone) {
  using C = LzCfg<BIG>;
  constexpr int R = C::R, JM = C::JM, NS = C::NS, AS = C::AS, QLD = C::QLD;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) double lsm[];
  double* Qs = lsm;                                   // [R][JM] local rows of the basis
  double* rsA = Qs + (size_t)R * JM;                  // [16 senders][NS] partials of my entries
  double* agA = rsA + LZ_CL * NS;                     // [16 owners][AS] h1, gathered
  double* rsB = agA + LZ_CL * AS;
  double* agB = rsB + LZ_CL * NS;                     // h2 and ||z1||^2 (entry nc), sums of squares
  double* qp = agB + LZ_CL * AS;                      // [16][QLD] q_j, exchange order
  double* qn = qp + LZ_CL * QLD;                      // BIG: [NMAX] q_j, natural order
  double* zsh = qn + (BIG ? C::NMAX : 0);             // [R]
  uint64_t* bars = reinterpret_cast<uint64_t*>(zsh + R);   // RS_A, AG_A, RS_B, AG_B, Q
  __shared__ double red2[LZ_T / 32];
  const uint32_t s_rsA = tc::smem_u32(rsA), s_agA = tc::smem_u32(agA), s_rsB = tc::smem_u32(rsB);
  const uint32_t s_agB = tc::smem_u32(agB), s_qp = tc::smem_u32(qp), s_bar = tc::smem_u32(bars);
  const int s_row = warp * 2 + (lane >> 4), g = lane & 15;   // half-warp per local row (+ 32 rr)
  // SMALL: row l = rank + 16 s_row of G (symmetric: row l = column l) in qp's order,
  // greg[2t + e] = G[l][t + 16 (2g + e)]
  double greg[BIG ? 1 : 32];
  if (!BIG) {
    const int l = rank + LZ_CL * s_row;
#pragma unroll
    for (int t = 0; t < 16; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = t + LZ_CL * (2 * g + e);
        greg[2 * t + e] = (l < n && i < n) ? __ldg(G + i + (int64_t)l * ldg) : 0.0;
      }
  }
  // BIG: double2 loads of the streamed rows when every row starts 16-B aligned
  const bool al2 = BIG && ((ldg & 1) == 0) && ((reinterpret_cast<uintptr_t>(G) & 15) == 0);
  for (int idx = tid; idx < R * JM; idx += LZ_T) Qs[idx] = 0.0;
  // q_0: a fixed pseudo-random unit vector (identical on every CTA, no exchange)
  {
    double nq = 0.0;
    for (int P = tid; P < C::NMAX; P += LZ_T) {
      const int l = BIG ? P : (P >> 5) + LZ_CL * (P & 31);   // SMALL: qp position P
      double v = 0.0;
      if (l < n) {
        const uint4 w = philox(make_uint4((uint32_t)l, 0u, 0u, 0x4C5Au), 0x1234567u, 0x89ABCDEu);
        v = ((double)w.x + 0.5) * 0x1p-32 - 0.5;
      }
      nq = fma(v, v, nq);
      if (BIG) qn[P] = v; else qp[P] = v;
    }
    for (int o = 16; o > 0; o >>= 1) nq += __shfl_xor_sync(0xffffffffu, nq, o);
    if (lane == 0) red2[warp] = nq;
    __syncthreads();
    double nq2 = 0.0;
    for (int w = 0; w < LZ_T / 32; ++w) nq2 += red2[w];
    const double inq = 1.0 / sqrt(nq2);
    for (int P = tid; P < C::NMAX; P += LZ_T) {
      if (BIG) qn[P] *= inq; else qp[P] *= inq;
    }
  }
  if (tid == 0) {
    for (int q = 0; q < 5; ++q) tc::mbar_init(&bars[q], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  if (tid < R) Qs[tid * JM + 0] = BIG ? qn[rank + LZ_CL * tid] : qp[rank * QLD + tid];
  cluster.sync();
  int jend = J;
#ifdef CDMD_LZ_PROF
  __shared__ unsigned long long tps[12];   // phase cycle totals (thread 0)
  if (tid < 12) tps[tid] = 0;
  __syncthreads();
  unsigned long long tq = clock64();
#endif
  for (int j = 0; j < J; ++j) {
    const uint32_t par = (uint32_t)j & 1u;
    const int nc = j + 1, ncb = nc + 1;   // basis columns 0..j; B's entries (h2, ||z1||^2)
    // (1) z = G q_j on the local rows
    if (!BIG) {   // registers x broadcast shared loads
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int t = 0; t < 16; t += 2) {
        const double2 q0 = *reinterpret_cast<const double2*>(qp + 32 * t + 2 * g);
        const double2 q1 = *reinterpret_cast<const double2*>(qp + 32 * (t + 1) + 2 * g);
        a0 = fma(greg[2 * t], q0.x, a0);
        a1 = fma(greg[2 * t + 1], q0.y, a1);
        a2 = fma(greg[2 * t + 2], q1.x, a2);
        a3 = fma(greg[2 * t + 3], q1.y, a3);
      }
      double a = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (g == 0) zsh[s_row] = a;
    } else {      // two streamed rows per half-warp (L2-resident G)
      const int l0 = rank + LZ_CL * s_row, l1 = l0 + LZ_CL * 32;
      const double* r0 = G + (int64_t)(l0 < n ? l0 : 0) * ldg;
      const double* r1 = G + (int64_t)(l1 < n ? l1 : 0) * ldg;
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      if (al2) {
        const int n2 = n & ~1;
#pragma unroll 4
        for (int i = 2 * g; i < n2; i += 32) {
          const double2 q = *reinterpret_cast<const double2*>(qn + i);
          const double2 x0 = __ldg(reinterpret_cast<const double2*>(r0 + i));
          const double2 x1 = __ldg(reinterpret_cast<const double2*>(r1 + i));
          a0 = fma(x0.x, q.x, a0);
          a1 = fma(x0.y, q.y, a1);
          b0 = fma(x1.x, q.x, b0);
          b1 = fma(x1.y, q.y, b1);
        }
        if ((n & 1) && g == 0) {
          a0 = fma(__ldg(r0 + n - 1), qn[n - 1], a0);
          b0 = fma(__ldg(r1 + n - 1), qn[n - 1], b0);
        }
      } else {
#pragma unroll 4
        for (int i = g; i < n; i += 16) {
          const double q = qn[i];
          a0 = fma(__ldg(r0 + i), q, a0);
          b0 = fma(__ldg(r1 + i), q, b0);
        }
      }
      double a = a0 + a1, b = b0 + b1;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (g == 0) {
        zsh[s_row] = l0 < n ? a : 0.0;
        zsh[s_row + 32] = l1 < n ? b : 0.0;
      }
    }
    if (tid < 5) {   // this step's expected bytes (each barrier's previous phase is complete)
      const uint32_t bytes = tid == 0   ? 8u * LZ_CL * lz_owned(nc, rank)
                             : tid == 1 ? 8u * nc
                             : tid == 2 ? 8u * LZ_CL * lz_owned(ncb, rank)
                             : tid == 3 ? 8u * (ncb + LZ_CL)
                                        : 8u * LZ_CL * R;
      tc::mbar_arrive_expect_tx(&bars[tid], bytes);
    }
    __syncthreads();
    LZ_TICK(0);
    // (2) partial h1_c = Q_loc[:, c]^T z -> owner c % 16
    if (tid < nc) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int s = 0; s < R; s += 4) {
        a0 = fma(Qs[s * JM + tid], zsh[s], a0);
        a1 = fma(Qs[(s + 1) * JM + tid], zsh[s + 1], a1);
        a2 = fma(Qs[(s + 2) * JM + tid], zsh[s + 2], a2);
        a3 = fma(Qs[(s + 3) * JM + tid], zsh[s + 3], a3);
      }
      const uint32_t o = (uint32_t)(tid & (LZ_CL - 1));
      lz_st_async(tc::mapa(s_rsA + 8u * (uint32_t)(rank * NS + tid / LZ_CL), o), (a0 + a1) + (a2 + a3),
                  tc::mapa(s_bar, o));
    }
    LZ_TICK(1);
    // (3) owners (warp 0, lane = slot): sum the 16 partials in a fixed order, send to all
    if (warp == 0) {
      tc::mbar_wait(&bars[0], par);
      const int c = LZ_CL * lane + rank;
      if (lane < NS && c < nc) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int r = 0; r < LZ_CL; r += 4) {
          a0 += rsA[r * NS + lane];
          a1 += rsA[(r + 1) * NS + lane];
          a2 += rsA[(r + 2) * NS + lane];
          a3 += rsA[(r + 3) * NS + lane];
        }
        const double v = (a0 + a1) + (a2 + a3);
        const uint32_t off = 8u * (uint32_t)(rank * AS + lane);
#pragma unroll 4
        for (int t = 0; t < LZ_CL; ++t) lz_st_async(tc::mapa(s_agA + off, t), v, tc::mapa(s_bar + 8u, t));
      }
    }
    tc::mbar_wait(&bars[1], par);
    LZ_TICK(2);
    // (4) z1 = z - Q h1 on the local rows (h1_c = agA[(c % 16) AS + c / 16]), local ||z1||^2
    {
      const double* hg = agA + g * AS;
      double sq = 0.0;
#pragma unroll
      for (int rr = 0; rr < C::RH; ++rr) {
        const int s = s_row + 32 * rr;
        const double* qr = Qs + s * JM;
        double a = 0.0, b = 0.0;
        int i = 0;
        for (; LZ_CL * (i + 1) + g < nc; i += 2) {
          a = fma(qr[LZ_CL * i + g], hg[i], a);
          b = fma(qr[LZ_CL * (i + 1) + g], hg[i + 1], b);
        }
        if (LZ_CL * i + g < nc) a = fma(qr[LZ_CL * i + g], hg[i], a);
        a += b;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const double z1 = zsh[s] - a;
        sq = fma(z1, z1, sq);
        __syncwarp();
        if (g == 0) zsh[s] = z1;
      }
      sq += __shfl_xor_sync(0xffffffffu, sq, 16);   // the warp's rows
      if (lane == 0) red2[warp] = sq;
    }
    __syncthreads();
    LZ_TICK(3);
    // (5) partial h2_c = Q_loc[:, c]^T z1 and (entry nc) ||z1_loc||^2 -> owners
    if (tid <= nc) {
      double v;
      if (tid < nc) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int s = 0; s < R; s += 4) {
          a0 = fma(Qs[s * JM + tid], zsh[s], a0);
          a1 = fma(Qs[(s + 1) * JM + tid], zsh[s + 1], a1);
          a2 = fma(Qs[(s + 2) * JM + tid], zsh[s + 2], a2);
          a3 = fma(Qs[(s + 3) * JM + tid], zsh[s + 3], a3);
        }
        v = (a0 + a1) + (a2 + a3);
      } else {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int w = 0; w < LZ_T / 32; w += 2) {
          a0 += red2[w];
          a1 += red2[w + 1];
        }
        v = a0 + a1;
      }
      const uint32_t o = (uint32_t)(tid & (LZ_CL - 1));
      lz_st_async(tc::mapa(s_rsB + 8u * (uint32_t)(rank * NS + tid / LZ_CL), o), v, tc::mapa(s_bar + 16u, o));
    }
    LZ_TICK(4);
    // (6) owners: sums, and the sum of squares of my h2 entries (not of the norm entry)
    if (warp == 0) {
      tc::mbar_wait(&bars[2], par);
      const int c = LZ_CL * lane + rank;
      double v = 0.0;
      if (lane < NS && c < ncb) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int r = 0; r < LZ_CL; r += 4) {
          a0 += rsB[r * NS + lane];
          a1 += rsB[(r + 1) * NS + lane];
          a2 += rsB[(r + 2) * NS + lane];
          a3 += rsB[(r + 3) * NS + lane];
        }
        v = (a0 + a1) + (a2 + a3);
        const uint32_t off = 8u * (uint32_t)(rank * AS + lane);
#pragma unroll 4
        for (int t = 0; t < LZ_CL; ++t) lz_st_async(tc::mapa(s_agB + off, t), v, tc::mapa(s_bar + 24u, t));
      }
      double sq = c < nc && lane < NS ? v * v : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane < LZ_CL)
        lz_st_async(tc::mapa(s_agB + 8u * (uint32_t)(rank * AS + NS), lane), sq, tc::mapa(s_bar + 24u, lane));
    }
    tc::mbar_wait(&bars[3], par);
    LZ_TICK(5);
    // (7) z2 = z1 - Q h2; alpha_j, beta_j; q_{j+1} = z2 / beta_j.  ||h2||^2 is the 16 owners'
    // sums of squares added by a 16-lane butterfly: bitwise identical in every lane and CTA.
    double nh2 = agB[(lane & 15) * AS + NS];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) nh2 += __shfl_xor_sync(0xffffffffu, nh2, o);
    const double nz1 = agB[(nc & (LZ_CL - 1)) * AS + nc / LZ_CL];
    const double b2 = nz1 - nh2;
    const double bj = b2 > 0.0 ? sqrt(b2) : 0.0;
    const double aj = agA[(j & (LZ_CL - 1)) * AS + j / LZ_CL] + agB[(j & (LZ_CL - 1)) * AS + j / LZ_CL];
    const bool stop = !(bj > 1e-13 * fabs(aj) + 1e-300) || j + 1 == J;   // invariant subspace / last step
    const double ib = stop ? 0.0 : 1.0 / bj;
    {
      const double* hg = agB + g * AS;
#pragma unroll
      for (int rr = 0; rr < C::RH; ++rr) {
        const int s = s_row + 32 * rr;
        const double* qr = Qs + s * JM;
        double a = 0.0, b = 0.0;
        int i = 0;
        for (; LZ_CL * (i + 1) + g < nc; i += 2) {
          a = fma(qr[LZ_CL * i + g], hg[i], a);
          b = fma(qr[LZ_CL * (i + 1) + g], hg[i + 1], b);
        }
        if (LZ_CL * i + g < nc) a = fma(qr[LZ_CL * i + g], hg[i], a);
        a += b;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const double qv = (zsh[s] - a) * ib;   // the same in all 16 lanes of the half-warp
        if (!stop) {
          // lane g sends the row to CTA g
          lz_st_async(tc::mapa(s_qp + 8u * (uint32_t)(rank * QLD + s), g), qv, tc::mapa(s_bar + 32u, g));
          if (g == 0) Qs[s * JM + j + 1] = qv;
        }
      }
    }
    if (rank == 0 && tid == 0) {
      alpha[j] = aj;
      beta[j] = bj;
    }
    if (stop) {
      jend = j + 1;
      if (rank == 0)
        for (int jj = jend + tid; jj < J; jj += LZ_T) alpha[jj] = beta[jj] = 0.0;   // T padded block-diagonal
      break;
    }
    LZ_TICK(6);
    tc::mbar_wait(&bars[4], par);
    if (BIG) {   // q_{j+1} in natural order for the streamed rows
      for (int i = tid; i < C::NMAX; i += LZ_T) qn[i] = i < n ? qp[(i & (LZ_CL - 1)) * QLD + i / LZ_CL] : 0.0;
      __syncthreads();
    }
    LZ_TICK(7);
  }
  // the basis, n x jend column-major
  __syncthreads();
  for (int idx = tid; idx < R * jend; idx += LZ_T) {
    const int s = idx / jend, c = idx % jend, l = rank + LZ_CL * s;
    if (l < n) Qout[l + (int64_t)c * n] = Qs[s * JM + c];
  }
  if (rank == 0 && tid == 0) {
    *jdone = jend;
#ifdef CDMD_LZ_PROF
    for (int q = 0; q < 8; ++q) g_lz_prof[q] = tps[q];
#endif
  }
  cluster.sync();   // no CTA leaves while a peer may still write into it
}

// Convergence of the k largest Ritz pairs (of the k + 1 computed, ascending lam1[0..k],
// S: jend x (k + 1) eigenvectors of T, column q <-> lam1[q]): ||G v_i - theta_i v_i|| =
// |beta_{J-1}| |S[J-1, i]| <= LZ_TOL (theta_i - theta_k) for the k largest.
// flag: 0 converged, 1 not.  The gap bound sin(v_i, u_i) <= r_i / gap_i keeps every Ritz
// vector within LZ_TOL of the eigenvector (and |theta_i - lambda_i| <= r_i <= LZ_TOL theta_i).
constexpr double LZ_TOL = 1e-9;
__global__ void lz_check_kernel(int J, int k, const double* __restrict__ beta, const double* __restrict__ lam1,
                                const double* __restrict__ S, const int* __restrict__ jdone, int* __restrict__ flag) {
  if (threadIdx.x != 0) return;
  const double bl = fabs(beta[J - 1]);
  int bad = *jdone != J;   // stopped early (an invariant subspace of dimension < J): Householder decides
  for (int q = 1; q <= k; ++q) {
    const double r = bl * fabs(S[(int64_t)(J - 1) + (int64_t)q * J]);
    const double gap = lam1[q] - lam1[0];
    if (!(r <= LZ_TOL * gap)) bad = 1;
  }
  *flag = bad;
}

// 1 when this device co-schedules the variant's 16-CTA cluster at its shared-memory size
template <bool BIG>
static int lz_cluster_ok() {
  static std::atomic<int> okd[64];   // per device: 0 unknown, 1 yes, 2 no
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  const int known = okd[dev].load();
  if (known) return known == 1 ? 1 : 0;
  int ok;
  const size_t smem = lz_smem_bytes_t<BIG>();
  cudaError_t e = cudaFuncSetAttribute(lz_kernel<BIG>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) e = smem_optin(reinterpret_cast<const void*>(lz_kernel<BIG>));
  int nc = 0;
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(LZ_CL, 1, 1);
    cfg.blockDim = dim3(LZ_T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = LZ_CL;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    e = cudaOccupancyMaxActiveClusters(&nc, lz_kernel<BIG>, &cfg);
  }
  if (e != cudaSuccess) (void)cudaGetLastError();
  ok = (e == cudaSuccess && nc > 0) ? 1 : 0;
  okd[dev].store(ok ? 1 : 2);
  return ok;
}

static bool lz_big(int n) { return n > LzCfg<false>::NMAX; }

int lz_steps(int n, int k) {
  const int J = 9 * k / 4 + 9;   // 2.25 k + 9 (tools/lanczos_sim.py: converged by ~2.2 k + 5)
  return J < n ? J : n;
}

bool lz_supported(int n, int k) {
  if (n < 8 || n > LzCfg<true>::NMAX || k < 1 || k + 1 > n) return false;
  if (lz_big(n)) return lz_steps(n, k) <= LzCfg<true>::JM && lz_cluster_ok<true>() == 1;
  return lz_steps(n, k) <= LzCfg<false>::JM && lz_cluster_ok<false>() == 1;
}

// Krylov dimension cap of the variant that serves n (workspace sizing)
int lz_jmax(int n) { return lz_big(n) ? LzCfg<true>::JM : LzCfg<false>::JM; }

template <bool BIG>
static cudaError_t launch_lz_t(int n, int J, const double* G, int64_t ldg, double* alpha, double* beta, double* Q,
                               int* jdone, cudaStream_t st) {
  if (lz_cluster_ok<BIG>() != 1) return cudaErrorNotSupported;   // also sets the function attributes
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(LZ_CL, 1, 1);
  cfg.blockDim = dim3(LZ_T, 1, 1);
  cfg.dynamicSmemBytes = lz_smem_bytes_t<BIG>();
  cfg.stream = st;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = LZ_CL;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  note_launch();
  const cudaError_t e = cudaLaunchKernelEx(&cfg, lz_kernel<BIG>, n, G, ldg, J, alpha, beta, Q, jdone);
  if (e == cudaErrorInvalidClusterSize) {   // e.g. a green context with fewer SMs than one cluster
    (void)cudaGetLastError();
    return cudaErrorNotSupported;
  }
  return e;
}

cudaError_t launch_lz(int n, int J, const double* G, int64_t ldg, double* alpha, double* beta, double* Q, int* jdone,
                      cudaStream_t st) {
  return lz_big(n) ? launch_lz_t<true>(n, J, G, ldg, alpha, beta, Q, jdone, st)
                   : launch_lz_t<false>(n, J, G, ldg, alpha, beta, Q, jdone, st);
}

cudaError_t launch_lz_check(int J, int k, const double* beta, const double* lam1, const double* S, const int* jdone,
                            int* flag, cudaStream_t st) {
  note_launch();
  lz_check_kernel<<<1, 32, 0, st>>>(J, k, beta, lam1, S, jdone, flag);
  return cudaGetLastError();
}

// Ritz vectors Zout[:, q] = Q S[:, q + 1] (q < k; S: J x (k + 1), the k largest are columns 1..k)
__global__ void lz_ritz_kernel(int n, int J, int k, const double* __restrict__ Q, const double* __restrict__ S,
                               const double* __restrict__ lam1, double* __restrict__ lam, double* __restrict__ Z) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < k) lam[idx] = lam1[idx + 1];
  if (idx >= (int64_t)n * k) return;
  const int i = (int)(idx % n), q = (int)(idx / n);
  const double* sc = S + (int64_t)(q + 1) * J;
  double a0 = 0.0, a1 = 0.0;
  int c = 0;
  for (; c + 1 < J; c += 2) {
    a0 = fma(__ldg(Q + i + (int64_t)c * n), __ldg(sc + c), a0);
    a1 = fma(__ldg(Q + i + (int64_t)(c + 1) * n), __ldg(sc + c + 1), a1);
  }
  if (c < J) a0 = fma(__ldg(Q + i + (int64_t)c * n), __ldg(sc + c), a0);
  Z[idx] = a0 + a1;
}

cudaError_t launch_lz_ritz(int n, int J, int k, const double* Q, const double* S, const double* lam1, double* lam,
                           double* Z, cudaStream_t st) {
  note_launch();
  lz_ritz_kernel<<<(unsigned)ceil_div((int64_t)n * k, 256), 256, 0, st>>>(n, J, k, Q, S, lam1, lam, Z);
  return cudaGetLastError();
}

}  // namespace cdmd
