// sketch_tc2.cu — the Gaussian sketch Y = C D on CTA pairs (tcgen05 cta_group::2).
//
// Same arithmetic as sketch_tc.cu's single-CTA kernel: c_ri = T[u16]
// is bf16-valued (exact in fp16), X - 128 is exact in fp16, fp32 accumulation in TMEM,
// a row of ones yields sum_i c_ri and the epilogue adds 128 sum_i c_ri, split-K partial
// sums meet in Y through fp32 atomics.  What changes is the operand split:
//   * a cluster of two CTAs (one TPC) owns 256 rows of C: each CTA generates its own
//     128 rows (A, 8 KB per 32-pixel stage) and accumulates them in its own TMEM;
//   * the pair shares B: each CTA converts and holds only half of the frames of every
//     N = 256 MMA (16 KB per stage instead of 32 KB), and TMA-loads only those frames;
//   * the leader CTA issues tcgen05.mma.cta_group::2 (M = 256) once both CTAs' A and B
//     halves of a stage are in place (their producer warps arrive on the leader's
//     barriers), and tcgen05.commit multicasts the stage's release to both CTAs.
// Halving the per-CTA B traffic and buffer lets five stages stay in flight (the
// single-CTA kernel fits two), which hides the producer/MMA round trip.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc.cuh"

namespace cdmd {

namespace {

constexpr int G2_BM = 128;                 // rows of C per CTA (the pair: 256)
constexpr int G2_BK = 32;                  // pixels per stage (64-B fp16 rows, SWIZZLE_64B)
constexpr int G2_A = G2_BM * G2_BK * 2;    // bytes of an A stage (8 KB)
constexpr int G2_XK = 64;                  // pixels per uint8 X stage (64-B TMA rows)
constexpr int G2_XS = 2;                   // X stages
#ifndef G2_GRP_DEF
#define G2_GRP_DEF 2
#endif
constexpr int G2_GRP = G2_GRP_DEF;         // stages per producer->MMA hand-off
#ifndef G2_S_DEF
#define G2_S_DEF 4
#endif
constexpr int G2_S = G2_S_DEF;             // A/B stages
constexpr int G2_NG = G2_S / G2_GRP;       // hand-off groups in flight
constexpr int G2_GEN = 8;                  // generator warps
constexpr int G2_CVT = 8;                  // converter warps
constexpr int G2_THREADS = 32 * (2 + G2_GEN + G2_CVT);

PFN_cuTensorMapEncodeTiled_v12000 g2_encode_fn() {
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

}  // namespace

// npad: frames + the row of ones, rounded up to 32.  MMA h (h = 0, 1) covers frames
// [256 h, 256 h + N_h), N_0 = min(256, npad), N_1 = npad - N_0; CTA r of the pair holds
// frames 256 h + r N_h / 2 + [0, N_h / 2) of it (B rows: h = 0 first, then h = 1).
// SRFT (template SR = true, reading R25): the same pipeline with another generator.
// A CTA's 128 rows of C are the Re (rows 0..63) and Im (rows 64..127) parts of 64
// frequencies f of R; a generator thread owns one frequency and one 8-pixel chunk of
// every 32-pixel stage and writes both rows.  Entry phase index q = phi_i - b_i (mod
// 2^16) with b_i = floor(2^16 ((f i) mod n) / n) advanced by an exact integer
// recurrence (b += floor(2^16 f / n), rem += 2^16 f mod n, carry at n), phi_i from
// Philox(i / 8, 0, 0, TAG_SRFT_PHASE); the values come from the fp16 quarter-wave
// table in shared memory.
template <bool SR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G2_THREADS, 1) sketch_gaussian_tc2_kernel(
    const __grid_constant__ CUtensorMap mapX0, const __grid_constant__ CUtensorMap mapX1, int64_t pix0,
    int64_t n_local, int64_t m, int64_t p, uint32_t k0, uint32_t k1, const uint16_t* __restrict__ table_bf16,
    int npad, int nchunks_total, int chunks_per_split, float* __restrict__ part, int64_t n_total,
    const int32_t* __restrict__ freqs) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  const int N0 = npad < 256 ? npad : 256, N1 = npad - N0;
  const int h0r = N0 / 2, h1r = N1 / 2;         // this CTA's B rows per MMA half
  const int brows = h0r + h1r;
  const int BST = brows * G2_BK * 2;            // bytes of a B stage (fp16)
  const int XST = brows * G2_XK;                // bytes of an X stage (uint8)
  uint8_t* sA = smem;                           // G2_S x 8 KB
  uint8_t* sB = sA + G2_S * G2_A;               // G2_S x BST
  uint8_t* sX = sB + (size_t)G2_S * BST;        // G2_XS x XST
  uint16_t* htab = reinterpret_cast<uint16_t*>(sX + (size_t)G2_XS * XST);   // 32768 fp16 bits
  uint64_t* afull = reinterpret_cast<uint64_t*>(htab + 32768);   // leader: both CTAs' A halves written
  uint64_t* bfull = afull + G2_S;               // leader: both CTAs' B halves written
  uint64_t* sempty = bfull + G2_S;              // both CTAs: the stage's MMAs done (multicast commit)
  uint64_t* xfull = sempty + G2_S;
  uint64_t* xempty = xfull + G2_XS;
  uint64_t* tfull = xempty + G2_XS;
  uint64_t* lfullA = tfull + 1;                 // peer: its A half written (relayed to the leader)
  uint64_t* lfullB = lfullA + G2_S;             // peer: its B half written (relayed to the leader)
  uint64_t* pfull = lfullB + G2_S;              // leader: the peer's A and B halves written (relay)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfull + G2_S);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = tc::cluster_ctarank();   // 0 = leader
  const int64_t r0 = (int64_t)blockIdx.x * G2_BM;
  const int c_begin = blockIdx.y * chunks_per_split;
  const int c_end = min(nchunks_total, c_begin + chunks_per_split);
  const int nch = c_end - c_begin;
  if (SR) {
    for (int j = threadIdx.x; j <= 16384; j += blockDim.x) htab[j] = table_bf16[j];   // fp16 quarter wave
  } else {
    for (int j = threadIdx.x; j < 32768; j += blockDim.x) {   // positive half of T as fp16 bits
      const float v = __uint_as_float((uint32_t)table_bf16[32768 + j] << 16);
      htab[j] = __half_as_ushort(__float2half_rn(v));         // exact: 8 significant bits
    }
  }
  if (warp == 0 && lane == 0) {
    for (int b = 0; b < G2_S; ++b) {
      // leader: its own producer warps + one relayed arrival from the peer
      tc::mbar_init(&afull[b], G2_GEN);
      tc::mbar_init(&bfull[b], G2_CVT);
      tc::mbar_init(&pfull[b], 1);
      tc::mbar_init(&sempty[b], 1);
      tc::mbar_init(&lfullA[b], G2_GEN);
      tc::mbar_init(&lfullB[b], G2_CVT);
    }
    for (int b = 0; b < G2_XS; ++b) {
      tc::mbar_init(&xfull[b], 1);
      tc::mbar_init(&xempty[b], G2_CVT);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_mbar_init();
    tc::tma_prefetch(&mapX0);
    tc::tma_prefetch(&mapX1);
  }
  if (warp == 0) tc::tmem_alloc2(tmem_slot, 512);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();   // both CTAs' barriers initialised before any remote arrive
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int wtma = 1 + G2_GEN + G2_CVT;

  if (warp == 0) {
    if (lane == 0 && crank == 0) {  // ------------------------- MMA issuer (leader)
      const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB);
      for (int i = 0; i < nch; ++i) {
        const int st = i % G2_S;
        const int gs = (i / G2_GRP) % G2_NG;
        const uint32_t ph = (uint32_t)(i / (G2_GRP * G2_NG)) & 1u;
        if (i % G2_GRP == 0) {   // a group of G2_GRP stages is handed over at once
          tc::mbar_wait(&afull[gs], ph);
          tc::mbar_wait(&bfull[gs], ph);
          tc::mbar_wait(&pfull[gs], ph);
          tc::fence_after();
        }
        for (int h = 0; h < (N1 > 0 ? 2 : 1); ++h) {
          const int nn = h ? N1 : N0;
          const uint32_t idesc = tc::idesc_f16(2 * G2_BM, nn, false, false, false, false);
#pragma unroll
          for (int kk = 0; kk < G2_BK / 16; ++kk) {
            const uint64_t ad = tc::smem_desc(aBase + st * G2_A + kk * 32, 0, 512, 4);
            const uint64_t bd = tc::smem_desc(bBase + st * BST + (h ? h0r * 64 : 0) + kk * 32, 0, 512, 4);
            tc::mma2_f16(tmem_base + (uint32_t)(256 * h), ad, bd, idesc, (i | kk) != 0);
          }
        }
        if (i % G2_GRP == G2_GRP - 1 || i == nch - 1) tc::mma2_commit_multicast(&sempty[gs], 0x3);
      }
      tc::mma2_commit_multicast(tfull, 0x3);
    } else if (lane == 0) {  // --------- peer: relay its stage readiness to the leader (one
      //                                  cluster-scope release per stage and operand)
      const uint32_t pf = tc::mapa(tc::smem_u32(pfull), 0);
      for (int gi = 0; gi * G2_GRP < nch; ++gi) {
        const int gs = gi % G2_NG;
        const uint32_t ph = (uint32_t)(gi / G2_NG) & 1u;
        tc::mbar_wait(&lfullA[gs], ph);
        tc::mbar_wait(&lfullB[gs], ph);
        tc::mbar_arrive_cluster(pf + 8u * (uint32_t)gs);   // one cluster-scope release per group
      }
    }
  } else if (warp == wtma) {
    if (lane == 0) {  // ------------------------------------ TMA producer (this CTA's frames)
      const int nx = (nch + 1) >> 1;   // X stages of G2_XK = 2 G2_BK pixels
      for (int i = 0; i < nx; ++i) {
        const int xs = i % G2_XS;
        const uint32_t ph = (uint32_t)(i / G2_XS) & 1u;
        tc::mbar_wait(&xempty[xs], ph ^ 1u);
        tc::mbar_arrive_expect_tx(&xfull[xs], (uint32_t)XST);
        const int px = (c_begin + 2 * i) * G2_BK;
        uint8_t* dst = sX + (size_t)xs * XST;
        tc::tma_load_2d(dst, &mapX0, &xfull[xs], px, (int)crank * h0r);
        if (h1r) tc::tma_load_2d(dst + (size_t)h0r * G2_XK, &mapX1, &xfull[xs], px, 256 + (int)crank * h1r);
      }
    }
  } else if (warp <= G2_GEN && SR) {  // ------------------- SRFT generators, then epilogue
    const int g = threadIdx.x - 32;
    const int fr = g & 63, cq = g >> 6;         // frequency of the CTA, 8-pixel chunk of a stage
    const int64_t nf = p / 2;
    const int64_t fi = (int64_t)blockIdx.x * 64 + fr;
    const bool fok = fi < nf;
    const uint64_t n = (uint64_t)n_total;
    const uint64_t f = fok ? (uint64_t)freqs[fi] : 0ull;
    const uint32_t Qf = (uint32_t)((65536ull * f) / n), Rf = (uint32_t)((65536ull * f) % n);
    const uint32_t Q24 = (uint32_t)((65536ull * 24ull * f) / n), R24 = (uint32_t)((65536ull * 24ull * f) % n);
    const uint32_t nn = (uint32_t)n;
    const uint64_t P0 = (uint64_t)pix0 + (uint64_t)c_begin * G2_BK + 8ull * cq;
    const uint64_t a0 = (f * P0) % n;
    uint32_t b = (uint32_t)((65536ull * a0) / n), rem = (uint32_t)((65536ull * a0) % n);
    const int swzr = (fr >> 1) & 3, swzi = ((64 + fr) >> 1) & 3;
    auto cosq = [&](uint32_t q) -> uint32_t {   // fp16 bits of cos(2 pi q / 2^16)
      const uint32_t qd = (q >> 14) & 3u, r = q & 16383u;
      const uint32_t idx = (qd & 1u) ? 16384u - r : r;
      return (uint32_t)htab[idx] ^ ((((qd + 1u) >> 1) & 1u) << 15);
    };
    for (int i = 0; i < nch; ++i) {
      const int st = i % G2_S;
      const int gs = (i / G2_GRP) % G2_NG;
      const uint32_t ph = (uint32_t)(i / (G2_GRP * G2_NG)) & 1u;
      const bool gend = i % G2_GRP == G2_GRP - 1 || i == nch - 1;
      const uint64_t Pc = (uint64_t)pix0 + (uint64_t)(c_begin + i) * G2_BK + 8ull * cq;   // multiple of 8
      const uint4 w = philox(make_uint4((uint32_t)(Pc >> 3), 0u, 0u, TAG_SRFT_PHASE), k0, k1);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      uint32_t re[4], im[4];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t phi = (ws[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
        const uint32_t q = (phi - b) & 0xFFFFu;
        const uint32_t c = fok ? cosq(q) : 0u, sn = fok ? cosq((q - 16384u) & 0xFFFFu) : 0u;
        if (u & 1) { re[u >> 1] |= c << 16; im[u >> 1] |= sn << 16; }
        else { re[u >> 1] = c; im[u >> 1] = sn; }
        b += Qf;                      // i -> i + 1
        rem += Rf;
        if (rem >= nn) { rem -= nn; ++b; }
      }
      b += Q24;                       // i + 8 -> i + 32: this thread's chunk of the next stage
      rem += R24;
      if (rem >= nn) { rem -= nn; ++b; }
      if (i % G2_GRP == 0) tc::mbar_wait(&sempty[gs], ph ^ 1u);
      *reinterpret_cast<uint4*>(sA + st * G2_A + fr * 64 + ((cq ^ swzr) << 4)) = make_uint4(re[0], re[1], re[2], re[3]);
      *reinterpret_cast<uint4*>(sA + st * G2_A + (64 + fr) * 64 + ((cq ^ swzi) << 4)) =
          make_uint4(im[0], im[1], im[2], im[3]);
      if (gend) {
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(crank == 0 ? &afull[gs] : &lfullA[gs]);
      }
    }
    if (warp <= 4) {  // epilogue: TMEM lane = row of the tile (Re 0..63, Im 64..127)
      tc::mbar_wait(tfull, 0);
      tc::fence_after();
      const int q = warp & 3;
      const int rr = q * 32 + lane;
      const int64_t fq = (int64_t)blockIdx.x * 64 + (rr & 63);
      const int64_t ry = rr < 64 ? fq : nf + fq;
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16);
      uint32_t rs[16];
      tc::tmem_ld16(ta + (uint32_t)(m & ~15), rs);
      tc::tmem_ld_wait();
      const float rowsum = __uint_as_float(rs[m & 15]);
      for (int c0 = 0; c0 < (int)m; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(ta + c0, v);
        tc::tmem_ld_wait();
        if (fq < nf && nch > 0) {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (c0 + t < m) part[((int64_t)blockIdx.y * m + c0 + t) * p + ry] = fmaf(128.0f, rowsum, __uint_as_float(v[t]));
        }
      }
    }
  } else if (warp <= G2_GEN) {  // ---------------------------- C generators, then epilogue
    constexpr int NQ = 16 / G2_GEN;             // 16-B chunks (8 pixels, one Philox call) per thread and stage
    const int g = threadIdx.x - 32;
    const int rr = g & (G2_BM - 1);             // row of the tile
    const int q0 = g >> 7;
    const int64_t row = r0 + rr;
    const int swz = (rr >> 1) & 3;              // SWIZZLE_64B chunk permutation of this row
    const uint32_t ctr0 = (uint32_t)(pix0 >> 3) + (uint32_t)(c_begin * (G2_BK / 8) + q0);
    for (int i = 0; i < nch; ++i) {
      const int st = i % G2_S;
      const int gs = (i / G2_GRP) % G2_NG;
      const uint32_t ph = (uint32_t)(i / (G2_GRP * G2_NG)) & 1u;
      const bool gend = i % G2_GRP == G2_GRP - 1 || i == nch - 1;
      uint32_t h2[NQ][4];
#pragma unroll
      for (int c = 0; c < NQ; ++c) {
        uint4 w = make_uint4(0, 0, 0, 0);   // one Philox call = eight 16-bit table indices
        if (row < p)
          w = philox(make_uint4(ctr0 + (uint32_t)(i * (G2_BK / 8) + c * (G2_GEN / 4)), (uint32_t)row, 0u, TAG_GAUSSIAN),
                     k0, k1);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // both 16-bit indices at once: T[u] = +H[u - 32768] (u >= 32768), -H[u ^ 0x7FFF] otherwise
          const uint32_t wq = ws[q];
          const uint32_t sg = ~wq & 0x80008000u;
          const uint32_t idx = (wq ^ (sg - (sg >> 15))) & 0x7FFF7FFFu;
          const uint32_t e0 = htab[idx & 0xFFFFu], e1 = htab[idx >> 16];
          h2[c][q] = (e0 | (e1 << 16)) ^ sg;
        }
      }
      if (i % G2_GRP == 0) tc::mbar_wait(&sempty[gs], ph ^ 1u);
#pragma unroll
      for (int c = 0; c < NQ; ++c) {
        const int q8 = q0 + c * (G2_GEN / 4);
        *reinterpret_cast<uint4*>(sA + st * G2_A + rr * 64 + ((q8 ^ swz) << 4)) =
            make_uint4(h2[c][0], h2[c][1], h2[c][2], h2[c][3]);
      }
      if (gend) {
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(crank == 0 ? &afull[gs] : &lfullA[gs]);
      }
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
  } else {  // ------------------ X converters: uint8 (SMEM) -> fp16 x - 128, this CTA's frames
    // thread = (16-pixel half hf, B row fl of each MMA half): the X rows are read and
    // converted into registers before the B slot is awaited; the ragged last chunk of
    // the slab and the row of ones take a per-element path
    const int cthr = threadIdx.x - 32 * (1 + G2_GEN);   // 0..255
    const int hf = cthr & 1, fl = cthr >> 1;            // half, row within an MMA half (0..127)
    const __half2 c1152 = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
    const int mi = (int)m;
    int frame[2], brow[2];
    frame[0] = fl < h0r ? (int)crank * h0r + fl : -1;
    brow[0] = fl;
    frame[1] = fl < h1r ? 256 + (int)crank * h1r + fl : -1;
    brow[1] = h0r + fl;
    for (int i = 0; i < nch; ++i) {
      const int st = i % G2_S;
      const int gs = (i / G2_GRP) % G2_NG;
      const uint32_t ph = (uint32_t)(i / (G2_GRP * G2_NG)) & 1u;
      const bool gend = i % G2_GRP == G2_GRP - 1 || i == nch - 1;
      const int xi = i >> 1, xs = xi % G2_XS;
      if ((i & 1) == 0) tc::mbar_wait(&xfull[xs], (uint32_t)(xi / G2_XS) & 1u);
      const uint8_t* xt = sX + (size_t)xs * XST + G2_BK * (i & 1) + 16 * hf;
      const int64_t jx = (int64_t)(c_begin + i) * G2_BK + 16 * hf;   // first local pixel of the half
      const int64_t rem = n_local - jx;
      const int valid = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
      uint32_t hw[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int f = frame[u];
        if (valid == 16) {
          uint4 xv = make_uint4(0, 0, 0, 0);
          if (f >= 0 && f < mi) xv = *reinterpret_cast<const uint4*>(xt + brow[u] * G2_XK);
          const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
          const uint32_t fill = f == mi ? 0x3C003C00u : 0u;   // the row of ones: D[:, m] = sum_i c_ri
#pragma unroll
          for (int b = 0; b < 8; ++b) {   // two pixels -> half2 (1024 + x) - 1152 = x - 128, exact
            const uint32_t pr = __byte_perm(xw[b >> 1], 0x64646464u, (b & 1) ? 0x7372u : 0x5150u);
            __half2 hh = __hsub2(*reinterpret_cast<const __half2*>(&pr), c1152);
            hw[u][b] = (f >= 0 && f < mi) ? *reinterpret_cast<uint32_t*>(&hh) : fill;
          }
        } else {
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            uint32_t w = 0u;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int q = 2 * b + e;
              uint32_t h = 0u;
              if (q < valid && f >= 0) {
                if (f < mi) h = __half_as_ushort(__int2half_rn((int)xt[brow[u] * G2_XK + q] - 128));
                else if (f == mi) h = 0x3C00u;
              }
              w |= h << (16 * e);
            }
            hw[u][b] = w;
          }
        }
      }
      if (i % G2_GRP == 0) tc::mbar_wait(&sempty[gs], ph ^ 1u);
      uint8_t* bst = sB + (size_t)st * BST;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (frame[u] < 0) continue;
        uint8_t* rowp = bst + brow[u] * 64;
        const int swz = (brow[u] >> 1) & 3;
        *reinterpret_cast<uint4*>(rowp + (((2 * hf) ^ swz) << 4)) = make_uint4(hw[u][0], hw[u][1], hw[u][2], hw[u][3]);
        *reinterpret_cast<uint4*>(rowp + (((2 * hf + 1) ^ swz) << 4)) = make_uint4(hw[u][4], hw[u][5], hw[u][6], hw[u][7]);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if ((i & 1) || i == nch - 1) tc::mbar_arrive(&xempty[xs]);
        if (gend) tc::mbar_arrive(crank == 0 ? &bfull[gs] : &lfullB[gs]);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync_all();   // both CTAs done with the pair's TMEM
  if (warp == 0) {
    tc::fence_after();
    tc::tmem_dealloc2(tmem_base, 512);
  }
}

bool sketch_gaussian_tc2_supported(const cdmd_video& v) {
  return v.m + 1 <= 512 && (v.ld % 16) == 0 && g2_encode_fn() != nullptr;
}

int gaussian_tc2_splits(const cdmd_video& v, int64_t p) {
  const int npairs = (int)ceil_div(p, 2 * G2_BM);
  const int nchunks = (int)ceil_div(v.n_local, G2_BK);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int splits = sms / (2 * npairs);   // one CTA per SM: a single wave
  if (splits > nchunks) splits = nchunks;
  if (splits < 1) splits = 1;
  return (int)ceil_div(nchunks, ceil_div(nchunks, splits));
}

// part: splits x m x p fp32 partial sums (reduced by the caller)
cudaError_t launch_sketch_tc2(const cdmd_video& v, const SensingPlan& P, const uint16_t* table, float* part,
                              int* splits_out, const int32_t* freqs, cudaStream_t st) {
  const bool sr = P.kind == CDMD_SRFT;
  const int npad = (int)round_up(v.m + 1, 32);     // frames + the row of ones
  const int N0 = npad < 256 ? npad : 256, N1 = npad - N0;
  const int npairs = (int)ceil_div(P.p, 2 * G2_BM);
  const int nchunks = (int)ceil_div(v.n_local, G2_BK);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int splits = sms / (2 * npairs);   // one CTA per SM: a single wave
  if (splits > nchunks) splits = nchunks;
  if (splits < 1) splits = 1;
  const int cps = (int)ceil_div(nchunks, splits);
  splits = (int)ceil_div(nchunks, cps);
  CUtensorMap mapX0, mapX1;
  cuuint64_t dims[2] = {(cuuint64_t)v.n_local, (cuuint64_t)v.m};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld};
  cuuint32_t estr[2] = {1, 1};
  cuuint32_t box0[2] = {G2_XK, (cuuint32_t)(N0 / 2)};
  cuuint32_t box1[2] = {G2_XK, (cuuint32_t)(N1 > 0 ? N1 / 2 : 16)};
  if (g2_encode_fn()(&mapX0, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box0, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      g2_encode_fn()(&mapX1, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(v.X), dims, strides, box1, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const size_t brows = (size_t)(N0 + N1) / 2;
  const size_t smem = 1024 + (size_t)G2_S * (G2_A + brows * G2_BK * 2) + (size_t)G2_XS * brows * G2_XK + 65536 + 768;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = sr ? sketch_gaussian_tc2_kernel<true> : sketch_gaussian_tc2_kernel<false>;
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return e;
  *splits_out = splits;
  dim3 grid((unsigned)(2 * npairs), (unsigned)splits);
  note_launch();
  kern<<<grid, G2_THREADS, smem, st>>>(mapX0, mapX1, v.pix0, v.n_local, v.m, P.p, P.k0, P.k1, table, npad, nchunks,
                                       cps, part, P.n, freqs);
  return cudaGetLastError();
}

cudaError_t launch_sketch_gaussian_tc2(const cdmd_video& v, const SensingPlan& P, const uint16_t* table, float* part,
                                       int* splits_out, cudaStream_t st) {
  return launch_sketch_tc2(v, P, table, part, splits_out, nullptr, st);
}

}  // namespace cdmd
