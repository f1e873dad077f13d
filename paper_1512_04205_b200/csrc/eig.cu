// eig.cu — eigen-decomposition of the small real nonsymmetric A~ (Alg. 1 step 7,
// P:344) on the device, replacing cuSOLVER's hybrid geev for k <= 118.
//
// One warp, the matrix and the Schur vectors resident in shared memory (fp64):
//   1. Householder reduction to upper Hessenberg form, accumulating Q
//      (EISPACK orthes / ortran);
//   2. Francis double-shift QR iteration with Wilkinson / exceptional shifts,
//      accumulating the Schur vectors (EISPACK hqr2);
//   3. back substitution for the eigenvectors of the quasi-triangular Schur form
//      and back transformation with the Schur vectors (hqr2).
// The scalar control flow runs redundantly (uniformly) on all 32 lanes; every row /
// column / Schur-vector update loop and every dot product is split across lanes.
// Output follows the LAPACK real-geev convention the canonicalisation expects:
// lambda_j = (wr, wi) with each complex pair listed (+im, -im) consecutively and
// exactly conjugate, VR column j = Re v, column j+1 = Im v for the pair.
#include <math.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cdmd {

namespace {

struct Warp {
  int lane;
  __device__ __forceinline__ void sync() const { __syncwarp(); }
  __device__ __forceinline__ double sum(double v) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  }
};

// complex division (a + ib) / (c + id) (Smith's algorithm)
__device__ __forceinline__ void cdiv(double xr, double xi, double yr, double yi, double& cr, double& ci) {
  double r, d;
  if (fabs(yr) > fabs(yi)) {
    r = yi / yr;
    d = yr + r * yi;
    cr = (xr + r * xi) / d;
    ci = (xi - r * xr) / d;
  } else {
    r = yr / yi;
    d = yi + r * yr;
    cr = (r * xr + xi) / d;
    ci = (r * xi - xr) / d;
  }
}

// (x / y) complex through one reciprocal of |y|^2 (no division subroutine and its branches
// on the inverse iteration's serial chain); Smith's algorithm where |y|^2 could underflow or
// overflow.  rcp_hc is defined below.
__device__ __forceinline__ double rcp_hc(double x);
__device__ __forceinline__ void cdiv_fast(double xr, double xi, double yr, double yi, double& cr, double& ci) {
  const double d = fma(yr, yr, yi * yi);
  if (!(d >= 1e-280 && d <= 1e280)) {
    cdiv(xr, xi, yr, yi, cr, ci);
    return;
  }
  const double id = rcp_hc(d);
  cr = fma(xr, yr, xi * yi) * id;
  ci = fma(xi, yr, -(xr * yi)) * id;
}

// reciprocal and reciprocal square root: hardware approximation + two Newton steps
// (about 1 ulp; the Francis step's scalar chain is latency-bound, IEEE division and
// sqrt are several times longer)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
// The same to full precision in fewer dependent steps (the Francis step's scalar chain):
// one third-order correction from the hardware approximation (relative error e0 ~ 2^-22
// -> ~e0^3): reciprocal r (1 + e + e^2), e = 1 - x r; reciprocal square root
// y (1 + e/2 + 3 e^2 / 8), e = 1 - x y^2.
__device__ __forceinline__ double rcp_hc(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double rsqrt_hc(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}

}  // namespace

// A: k x k column-major (device); outputs W (2k: re, im), VR (k x k column-major).
// par3: shared memory holds 32 lane-private vector pairs (2 nn doubles each) and the
// eigenvectors of the Schur form are back-substituted one per lane.
__global__ void __launch_bounds__(32) hqr_eig_kernel(int nn, const double* __restrict__ A,
                                                    double* __restrict__ W, double* __restrict__ VR,
                                                    int* __restrict__ info, int par3) {
  extern __shared__ double sm[];
  const int ld = nn + 1;
  double* H = sm;                 // nn x ld, row-major: H[i * ld + j]
  double* V = H + nn * ld;        // Schur vectors, row-major
  double* ort = V + nn * ld;      // nn
  double* d = ort + nn;           // nn real parts
  double* e = d + nn;             // nn imaginary parts
  double* xbuf = e + nn;          // par3: [32][2 nn] lane-private (Re, Im) vectors
  const Warp wp{(int)(threadIdx.x & 31)};
  const int lane = wp.lane;
#define Hx(i, j) H[(i) * ld + (j)]
#define Vx(i, j) V[(i) * ld + (j)]
  for (int idx = lane; idx < nn * nn; idx += 32) {
    const int i = idx % nn, j = idx / nn;  // A column-major
    Hx(i, j) = A[idx];
    Vx(i, j) = (i == j) ? 1.0 : 0.0;
  }
  wp.sync();
  const int low = 0, high = nn - 1;
#ifdef CDMD_EIG_PROF
  long long tp[6];
  tp[0] = clock64();
#define EIG_T(i) tp[i] = clock64();
#else
#define EIG_T(i)
#endif
  // ------------------------------------------------ 1. orthes (Hessenberg)
  for (int m = low + 1; m <= high - 1; ++m) {
    double scale = 0.0;
    for (int i = m + lane; i <= high; i += 32) scale += fabs(Hx(i, m - 1));
    scale = wp.sum(scale);
    if (scale != 0.0) {
      double h = 0.0;
      for (int i = m + lane; i <= high; i += 32) {
        const double o = Hx(i, m - 1) / scale;
        ort[i] = o;
        h += o * o;
      }
      h = wp.sum(h);
      wp.sync();
      const double om = ort[m];
      const double g = om > 0 ? -sqrt(h) : sqrt(h);
      h = h - om * g;
      wp.sync();
      if (lane == 0) ort[m] = om - g;
      wp.sync();
      // H = (I - u u'/h) H: columns j = m .. nn-1
      for (int j = m + lane; j < nn; j += 32) {
        double f = 0.0;
        for (int i = high; i >= m; --i) f += ort[i] * Hx(i, j);
        f = f / h;
        for (int i = m; i <= high; ++i) Hx(i, j) -= f * ort[i];
      }
      wp.sync();
      // H = H (I - u u'/h): rows i = 0 .. high
      for (int i = lane; i <= high; i += 32) {
        double f = 0.0;
        for (int j = high; j >= m; --j) f += ort[j] * Hx(i, j);
        f = f / h;
        for (int j = m; j <= high; ++j) Hx(i, j) -= f * ort[j];
      }
      wp.sync();
      if (lane == 0) {
        ort[m] = scale * ort[m];
        Hx(m, m - 1) = scale * g;
      }
      wp.sync();
    }
  }
  EIG_T(1)
  // ortran: accumulate the transformations into V
  for (int m = high - 1; m >= low + 1; --m) {
    if (Hx(m, m - 1) != 0.0) {
      for (int i = m + 1 + lane; i <= high; i += 32) ort[i] = Hx(i, m - 1);
      wp.sync();
      for (int j = m + lane; j <= high; j += 32) {
        double g = 0.0;
        for (int i = m; i <= high; ++i) g += ort[i] * Vx(i, j);
        g = (g / ort[m]) / Hx(m, m - 1);  // double division avoids underflow
        for (int i = m; i <= high; ++i) Vx(i, j) += g * ort[i];
      }
      wp.sync();
    }
  }
  EIG_T(2)
  // ------------------------------------------------------- 2. hqr2 (Schur)
  int n = nn - 1;
  const double eps = 0x1p-52;
  double exshift = 0.0;
  double p = 0, q = 0, r = 0, s = 0, z = 0, t, w, x, y;
  double norm = 0.0;
  for (int i = lane; i < nn; i += 32)
    for (int j = (i > 0 ? i - 1 : 0); j < nn; ++j) norm += fabs(Hx(i, j));
  norm = wp.sum(norm);
  int iter = 0, total_iter = 0, fail = 0;
#ifdef CDMD_EIG_PROF
  long long qa = 0, qb = 0, qc = 0, qsteps = 0, t_a = 0;
#define QT(acc) { const long long t_ = clock64(); acc += t_ - t_a; t_a = t_; }
#else
#define QT(acc)
#endif
  while (n >= low) {
#ifdef CDMD_EIG_PROF
    t_a = clock64();
#endif
    int l = n;
    while (l > low) {
      s = fabs(Hx(l - 1, l - 1)) + fabs(Hx(l, l));
      if (s == 0.0) s = norm;
      if (fabs(Hx(l, l - 1)) < eps * s) break;
      l--;
    }
    if (l == n) {  // one root found
      const double hn = Hx(n, n) + exshift;
      wp.sync();
      if (lane == 0) {
        Hx(n, n) = hn;
        d[n] = hn;
        e[n] = 0.0;
      }
      wp.sync();
      n--;
      iter = 0;
    } else if (l == n - 1) {  // two roots found
      w = Hx(n, n - 1) * Hx(n - 1, n);
      p = (Hx(n - 1, n - 1) - Hx(n, n)) / 2.0;
      q = p * p + w;
      z = sqrt(fabs(q));
      const double hnn = Hx(n, n) + exshift, hn1 = Hx(n - 1, n - 1) + exshift;
      wp.sync();
      if (lane == 0) {
        Hx(n, n) = hnn;
        Hx(n - 1, n - 1) = hn1;
      }
      wp.sync();
      x = hnn;
      if (q >= 0) {  // real pair
        z = (p >= 0) ? p + z : p - z;
        double dn1 = x + z, dn = dn1;
        if (z != 0.0) dn = x - w / z;
        x = Hx(n, n - 1);
        s = fabs(x) + fabs(z);
        p = x / s;
        q = z / s;
        r = sqrt(p * p + q * q);
        p = p / r;
        q = q / r;
        wp.sync();
        if (lane == 0) {
          d[n - 1] = dn1;
          d[n] = dn;
          e[n - 1] = 0.0;
          e[n] = 0.0;
        }
        for (int j = n - 1 + lane; j < nn; j += 32) {  // row modification
          const double zz = Hx(n - 1, j);
          Hx(n - 1, j) = q * zz + p * Hx(n, j);
          Hx(n, j) = q * Hx(n, j) - p * zz;
        }
        wp.sync();
        for (int i = lane; i <= n; i += 32) {  // column modification
          const double zz = Hx(i, n - 1);
          Hx(i, n - 1) = q * zz + p * Hx(i, n);
          Hx(i, n) = q * Hx(i, n) - p * zz;
        }
        for (int i = low + lane; i <= high; i += 32) {  // accumulate
          const double zz = Vx(i, n - 1);
          Vx(i, n - 1) = q * zz + p * Vx(i, n);
          Vx(i, n) = q * Vx(i, n) - p * zz;
        }
        wp.sync();
      } else {  // complex pair
        wp.sync();
        if (lane == 0) {
          d[n - 1] = x + p;
          d[n] = x + p;
          e[n - 1] = z;
          e[n] = -z;
        }
        wp.sync();
      }
      n = n - 2;
      iter = 0;
    } else {  // no convergence yet: form shift
      QT(qa)
      x = Hx(n, n);
      y = 0.0;
      w = 0.0;
      if (l < n) {
        y = Hx(n - 1, n - 1);
        w = Hx(n, n - 1) * Hx(n - 1, n);
      }
      if (iter == 10) {  // Wilkinson's original ad hoc shift
        exshift += x;
        wp.sync();
        for (int i = low + lane; i <= n; i += 32) Hx(i, i) -= x;
        wp.sync();
        s = fabs(Hx(n, n - 1)) + fabs(Hx(n - 1, n - 2));
        x = y = 0.75 * s;
        w = -0.4375 * s * s;
      }
      if (iter == 30) {  // MATLAB's ad hoc shift
        s = (y - x) / 2.0;
        s = s * s + w;
        if (s > 0) {
          s = sqrt(s);
          if (y < x) s = -s;
          s = x - w / ((y - x) / 2.0 + s);
          wp.sync();
          for (int i = low + lane; i <= n; i += 32) Hx(i, i) -= s;
          wp.sync();
          exshift += s;
          x = y = w = 0.964;
        }
      }
      iter++;
      if (++total_iter > 60 * nn) {
        fail = 1;
        break;
      }
      int m = n - 2;  // look for two consecutive small sub-diagonal elements
      // (p, q, r) are carried multiplied by h = H(m+1, m): the test below is homogeneous
      // in them and the first reflector is scale-invariant, so no divisions in the loop
      while (m >= l) {
        z = Hx(m, m);
        r = x - z;
        s = y - z;
        const double h = Hx(m + 1, m);
        p = (r * s - w) + Hx(m, m + 1) * h;
        q = (Hx(m + 1, m + 1) - z - r - s) * h;
        r = Hx(m + 2, m + 1) * h;
        if (m == l) break;
        if (fabs(Hx(m, m - 1)) * (fabs(q) + fabs(r)) <
            eps * (fabs(p) * (fabs(Hx(m - 1, m - 1)) + fabs(z) + fabs(Hx(m + 1, m + 1)))))
          break;
        m--;
      }
      {
        const double sc = fabs(p) + fabs(q) + fabs(r);
        if (sc != 0.0) {
          const double isc = rcp_nr(sc);
          p *= isc;
          q *= isc;
          r *= isc;
        }
      }
      QT(qb)
      wp.sync();
      for (int i = m + 2 + lane; i <= n; i += 32) {
        Hx(i, i - 2) = 0.0;
        if (i > m + 2) Hx(i, i - 3) = 0.0;
      }
      wp.sync();
      for (int kk = m; kk <= n - 1; ++kk) {  // double QR step, rows l:n, columns m:n
#ifdef CDMD_EIG_PROF
        ++qsteps;
#endif
        const bool notlast = (kk != n - 1);
        if (kk != m) {
          p = Hx(kk, kk - 1);
          q = Hx(kk + 1, kk - 1);
          r = notlast ? Hx(kk + 2, kk - 1) : 0.0;
          x = fabs(p) + fabs(q) + fabs(r);
          if (x == 0.0) continue;
          if (x < 1e-140 || x > 1e140) {   // EISPACK's scaling, only where squares could under/overflow
            const double ix = 1.0 / x;
            p = p * ix;
            q = q * ix;
            r = r * ix;
          } else {
            x = 1.0;                        // the reflector is scale-invariant; s below is unscaled
          }
        }
        const double ss = p * p + q * q + r * r;
        s = ss > 0.0 ? ss * rsqrt_nr(ss) : 0.0;
        if (p < 0) s = -s;
        if (s != 0) {
          double newsub = 0.0;
          bool setsub = false;
          if (kk != m) {
            newsub = -s * x;
            setsub = true;
          } else if (l != m) {
            newsub = -Hx(kk, kk - 1);
            setsub = true;
          }
          wp.sync();
          if (setsub && lane == 0) Hx(kk, kk - 1) = newsub;
          wp.sync();
          p = p + s;
          const double is = rcp_nr(s), ip = rcp_nr(p);
          x = p * is;
          y = q * is;
          z = r * is;
          q = q * ip;
          r = r * ip;
          for (int j = kk + lane; j < nn; j += 32) {  // row modification
            double pp = Hx(kk, j) + q * Hx(kk + 1, j);
            if (notlast) {
              pp = pp + r * Hx(kk + 2, j);
              Hx(kk + 2, j) = Hx(kk + 2, j) - pp * z;
            }
            Hx(kk, j) = Hx(kk, j) - pp * x;
            Hx(kk + 1, j) = Hx(kk + 1, j) - pp * y;
          }
          wp.sync();
          const int imax = n < kk + 3 ? n : kk + 3;
          const double zn = notlast ? z : 0.0;
          // column modification of H (rows 0..imax) and accumulation into V (all rows),
          // as one loop: with r = 0 the third column is left unchanged when last
          for (int i = lane; i <= high; i += 32) {
            double* hr = &Hx(i, kk);
            double* vr = &Vx(i, kk);
            const double v0 = vr[0], v1 = vr[1], v2 = notlast ? vr[2] : 0.0;
            const double pv = x * v0 + y * v1 + zn * v2;
            vr[0] = v0 - pv;
            vr[1] = v1 - pv * q;
            if (notlast) vr[2] = v2 - pv * r;
            if (i <= imax) {
              const double h0 = hr[0], h1 = hr[1], h2 = notlast ? hr[2] : 0.0;
              const double ph = x * h0 + y * h1 + zn * h2;
              hr[0] = h0 - ph;
              hr[1] = h1 - ph * q;
              if (notlast) hr[2] = h2 - ph * r;
            }
          }
          wp.sync();
        }
      }
      QT(qc)
    }
  }
#ifdef CDMD_EIG_PROF
  if (lane == 0) printf("EIGQR deflate+1/2-root %lld shift+msearch %lld sweep(+rest) %lld steps %lld\n", qa, qb, qc, qsteps);
#endif
  if (fail) {
    if (lane == 0) *info = 1;
    return;
  }
  EIG_T(3)
  // ------------------------------------- 3. eigenvectors of the Schur form
  if (norm != 0.0 && par3) {
    // One eigenvector (real) or pair (complex) per lane, 32 at a time in decreasing n:
    // a round reads only columns <= its own n of the Schur form, so the lanes solve
    // into private buffers and write their columns back after the round.
    int nitems = 0;
    for (int c = nn - 1; c >= 0; --c)
      if (e[c] <= 0.0) ++nitems;
    double* xr = xbuf + (size_t)lane * 2 * nn;
    double* xi = xr + nn;
    for (int r0 = 0; r0 < nitems; r0 += 32) {
      // this lane's item: the (r0 + lane)-th index c (descending) with e[c] <= 0
      int my = -1;
      {
        int cnt = 0;
        for (int c = nn - 1; c >= 0; --c)
          if (e[c] <= 0.0) {
            if (cnt == r0 + lane) { my = c; break; }
            ++cnt;
          }
      }
      if (my >= 0) {
        const int n3 = my;
        const double p3 = d[n3], q3 = e[n3];
        double z3 = 0.0, r3 = 0.0, s3 = 0.0;
        if (q3 == 0.0) {   // real vector
          int l = n3;
          xr[n3] = 1.0;
          for (int i = n3 - 1; i >= 0; i--) {
            const double w3 = Hx(i, i) - p3;
            double rr = 0.0;
            for (int j = l; j <= n3; ++j) rr += Hx(i, j) * xr[j];
            if (e[i] < 0.0) {
              z3 = w3;
              s3 = rr;
            } else {
              l = i;
              if (e[i] == 0.0) {
                xr[i] = (w3 != 0.0) ? -rr / w3 : -rr / (eps * norm);
              } else {   // solve real equations
                const double x3 = Hx(i, i + 1), y3 = Hx(i + 1, i);
                const double qq = (d[i] - p3) * (d[i] - p3) + e[i] * e[i];
                const double t3 = (x3 * s3 - z3 * rr) / qq;
                xr[i] = t3;
                xr[i + 1] = (fabs(x3) > fabs(z3)) ? (-rr - w3 * t3) / x3 : (-s3 - y3 * t3) / z3;
              }
              const double t3 = fabs(xr[i]);   // overflow control
              if ((eps * t3) * t3 > 1)
                for (int j = i; j <= n3; ++j) xr[j] /= t3;
            }
          }
        } else {   // complex vector (columns n-1 = Re, n = Im)
          int l = n3 - 1;
          if (fabs(Hx(n3, n3 - 1)) > fabs(Hx(n3 - 1, n3))) {
            xr[n3 - 1] = q3 / Hx(n3, n3 - 1);
            xi[n3 - 1] = -(Hx(n3, n3) - p3) / Hx(n3, n3 - 1);
          } else {
            cdiv(0.0, -Hx(n3 - 1, n3), Hx(n3 - 1, n3 - 1) - p3, q3, xr[n3 - 1], xi[n3 - 1]);
          }
          xr[n3] = 0.0;
          xi[n3] = 1.0;
          for (int i = n3 - 2; i >= 0; i--) {
            double ra = 0.0, sa = 0.0;
            for (int j = l; j <= n3; ++j) {
              ra += Hx(i, j) * xr[j];
              sa += Hx(i, j) * xi[j];
            }
            const double w3 = Hx(i, i) - p3;
            if (e[i] < 0.0) {
              z3 = w3;
              r3 = ra;
              s3 = sa;
            } else {
              l = i;
              if (e[i] == 0) {
                cdiv(-ra, -sa, w3, q3, xr[i], xi[i]);
              } else {   // solve complex equations
                const double x3 = Hx(i, i + 1), y3 = Hx(i + 1, i);
                double vr = (d[i] - p3) * (d[i] - p3) + e[i] * e[i] - q3 * q3;
                const double vi = (d[i] - p3) * 2.0 * q3;
                if (vr == 0.0 && vi == 0.0)
                  vr = eps * norm * (fabs(w3) + fabs(q3) + fabs(x3) + fabs(y3) + fabs(z3));
                double c0, c1;
                cdiv(x3 * r3 - z3 * ra + q3 * sa, x3 * s3 - z3 * sa - q3 * ra, vr, vi, c0, c1);
                xr[i] = c0;
                xi[i] = c1;
                if (fabs(x3) > (fabs(z3) + fabs(q3))) {
                  xr[i + 1] = (-ra - w3 * c0 + q3 * c1) / x3;
                  xi[i + 1] = (-sa - w3 * c1 - q3 * c0) / x3;
                } else {
                  cdiv(-r3 - y3 * c0, -s3 - y3 * c1, z3, q3, xr[i + 1], xi[i + 1]);
                }
              }
              const double t3 = fmax(fabs(xr[i]), fabs(xi[i]));   // overflow control
              if ((eps * t3) * t3 > 1)
                for (int j = i; j <= n3; ++j) {
                  xr[j] /= t3;
                  xi[j] /= t3;
                }
            }
          }
        }
      }
      wp.sync();   // every lane of the round has read the Schur form: write the columns
      if (my >= 0) {
        if (e[my] == 0.0) {
          for (int j = 0; j <= my; ++j) Hx(j, my) = xr[j];
        } else {
          for (int j = 0; j <= my; ++j) {
            Hx(j, my - 1) = xr[j];
            Hx(j, my) = xi[j];
          }
          Hx(my, my - 1) = 0.0;
        }
      }
      wp.sync();
    }
  } else if (norm != 0.0) {
    for (n = nn - 1; n >= 0; n--) {
      p = d[n];
      q = e[n];
      if (q == 0) {  // real vector
        int l = n;
        wp.sync();
        if (lane == 0) Hx(n, n) = 1.0;
        wp.sync();
        for (int i = n - 1; i >= 0; i--) {
          w = Hx(i, i) - p;
          double rr = 0.0;
          for (int j = l + lane; j <= n; j += 32) rr += Hx(i, j) * Hx(j, n);
          r = wp.sum(rr);
          if (e[i] < 0.0) {
            z = w;
            s = r;
          } else {
            l = i;
            double v0, v1 = 0.0;
            bool two = false;
            if (e[i] == 0.0) {
              v0 = (w != 0.0) ? -r / w : -r / (eps * norm);
            } else {  // solve real equations
              x = Hx(i, i + 1);
              y = Hx(i + 1, i);
              q = (d[i] - p) * (d[i] - p) + e[i] * e[i];
              t = (x * s - z * r) / q;
              v0 = t;
              v1 = (fabs(x) > fabs(z)) ? (-r - w * t) / x : (-s - y * t) / z;
              two = true;
            }
            wp.sync();
            if (lane == 0) {
              Hx(i, n) = v0;
              if (two) Hx(i + 1, n) = v1;
            }
            wp.sync();
            t = fabs(Hx(i, n));  // overflow control
            if ((eps * t) * t > 1) {
              for (int j = i + lane; j <= n; j += 32) Hx(j, n) = Hx(j, n) / t;
              wp.sync();
            }
          }
        }
      } else if (q < 0) {  // complex vector (columns n-1 = Re, n = Im)
        int l = n - 1;
        double a0, a1;
        if (fabs(Hx(n, n - 1)) > fabs(Hx(n - 1, n))) {
          a0 = q / Hx(n, n - 1);
          a1 = -(Hx(n, n) - p) / Hx(n, n - 1);
        } else {
          cdiv(0.0, -Hx(n - 1, n), Hx(n - 1, n - 1) - p, q, a0, a1);
        }
        wp.sync();
        if (lane == 0) {
          Hx(n - 1, n - 1) = a0;
          Hx(n - 1, n) = a1;
          Hx(n, n - 1) = 0.0;
          Hx(n, n) = 1.0;
        }
        wp.sync();
        for (int i = n - 2; i >= 0; i--) {
          double ra = 0.0, sa = 0.0;
          for (int j = l + lane; j <= n; j += 32) {
            ra += Hx(i, j) * Hx(j, n - 1);
            sa += Hx(i, j) * Hx(j, n);
          }
          ra = wp.sum(ra);
          sa = wp.sum(sa);
          w = Hx(i, i) - p;
          if (e[i] < 0.0) {
            z = w;
            r = ra;
            s = sa;
          } else {
            l = i;
            double c0, c1, c2 = 0.0, c3 = 0.0;
            bool two = false;
            if (e[i] == 0) {
              cdiv(-ra, -sa, w, q, c0, c1);
            } else {  // solve complex equations
              x = Hx(i, i + 1);
              y = Hx(i + 1, i);
              double vr = (d[i] - p) * (d[i] - p) + e[i] * e[i] - q * q;
              const double vi = (d[i] - p) * 2.0 * q;
              if (vr == 0.0 && vi == 0.0)
                vr = eps * norm * (fabs(w) + fabs(q) + fabs(x) + fabs(y) + fabs(z));
              cdiv(x * r - z * ra + q * sa, x * s - z * sa - q * ra, vr, vi, c0, c1);
              if (fabs(x) > (fabs(z) + fabs(q))) {
                c2 = (-ra - w * c0 + q * c1) / x;
                c3 = (-sa - w * c1 - q * c0) / x;
              } else {
                cdiv(-r - y * c0, -s - y * c1, z, q, c2, c3);
              }
              two = true;
            }
            wp.sync();
            if (lane == 0) {
              Hx(i, n - 1) = c0;
              Hx(i, n) = c1;
              if (two) {
                Hx(i + 1, n - 1) = c2;
                Hx(i + 1, n) = c3;
              }
            }
            wp.sync();
            t = fmax(fabs(Hx(i, n - 1)), fabs(Hx(i, n)));  // overflow control
            if ((eps * t) * t > 1) {
              for (int j = i + lane; j <= n; j += 32) {
                Hx(j, n - 1) = Hx(j, n - 1) / t;
                Hx(j, n) = Hx(j, n) / t;
              }
              wp.sync();
            }
          }
        }
      }
    }
  }
  if (norm != 0.0) {
    EIG_T(4)
    // back transformation: V = V * (upper triangular part of H)
    for (int j = nn - 1; j >= low; j--) {
      for (int i = low + lane; i <= high; i += 32) {
        double zz = 0.0;
        const int kmax = j < high ? j : high;
        for (int kx = low; kx <= kmax; ++kx) zz += Vx(i, kx) * Hx(kx, j);
        Vx(i, j) = zz;
      }
      wp.sync();
    }
  }
  for (int j = lane; j < nn; j += 32) {
    W[2 * j] = d[j];
    W[2 * j + 1] = e[j];
  }
  for (int idx = lane; idx < nn * nn; idx += 32) {
    const int i = idx % nn, j = idx / nn;
    VR[idx] = Vx(i, j);
  }
  if (lane == 0) *info = 0;
#ifdef CDMD_EIG_PROF
  EIG_T(5)
  if (lane == 0)
    printf("EIGPROF n=%d orthes %lld ortran %lld qr %lld (iters %d) backsub %lld backtr+out %lld\n", nn, tp[1] - tp[0],
           tp[2] - tp[1], tp[3] - tp[2], total_iter, tp[4] - tp[3], tp[5] - tp[4]);
#endif
#undef Hx
#undef Vx
}


// ======================================================================== v2
// Eigenvalues by the Francis QR without Schur vectors (EISPACK hqr: updates confined
// to the active block), then every eigenvector at once by inverse iteration on the
// Hessenberg matrix (one warp per real eigenvalue / conjugate pair) and the back
// transformation with Q from orthes.  The sequential QR sweep does about half the
// work of hqr2's, and the eigenvectors leave the serial chain.
//
// hqrv_kernel: A (k x k column-major) -> W (wr, wi pairs as hqr2), H0 (the Hessenberg
// form, row-major k x k) and Q (row-major k x k) for hinvit_kernel.
__device__ unsigned long long g_hqr_prof[8];   // orthes, ortran, deflation search, m search, bulge steps, iterations, steps
__device__ unsigned long long g_hqr_prof2[4];  // CDMD_HQR_PROF2: bulge step = scalar chain, row update, column update
void hqr_prof_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_hqr_prof, sizeof(unsigned long long) * 8);
  cudaMemcpyFromSymbol(out + 8, g_hqr_prof2, sizeof(unsigned long long) * 4);
}

constexpr int HQ_WARPS = 8;   // warps of hqrv_kernel: all reduce to Hessenberg form, warp 0 runs hqr

template <bool BIG>   // BIG: more than 64 rows (slots beyond two per lane in the bulge step)
__global__ void __launch_bounds__(32 * HQ_WARPS, 1) hqrv_kernel(int nn, const double* __restrict__ A,
                                                            double* __restrict__ W, double* __restrict__ H0,
                                                            double* __restrict__ Qout, int* __restrict__ info,
                                                            int ovl) {
  // ovl: the shared block also holds a copy R of H after orthes and a separate scratch
  // block, so warps 4..7 accumulate Q (ortran, from R) while warp 0 already runs hqr
  extern __shared__ double sm[];
  const int ld = nn + 1;
  double* H = sm;                 // nn x ld, row-major
  double* V = H + nn * ld;        // Q, row-major
  const int vsz = nn * ld > 3 * ld + 80 ? nn * ld : 3 * ld + 80;
  double* ort = V + vsz;          // nn
  double* d = ort + nn;           // nn real parts
  double* e = d + nn;             // nn imaginary parts
  const Warp wp{(int)(threadIdx.x & 31)};
  const int lane = wp.lane, warp = (int)(threadIdx.x >> 5), tid = (int)threadIdx.x;
  constexpr int NT = 32 * HQ_WARPS;
#define Hx(i, j) H[(i) * ld + (j)]
#define Vx(i, j) V[(i) * ld + (j)]
  for (int idx = tid; idx < nn * nn; idx += NT) {
    const int i = idx % nn, j = idx / nn;  // A column-major
    Hx(i, j) = A[idx];
    Vx(i, j) = (i == j) ? 1.0 : 0.0;
  }
  // the padding column and the bulge step's scratch block hold zeros (finite: the step
  // multiplies them by zero coefficients)
  for (int i = tid; i < nn; i += NT) Hx(i, nn) = 0.0;
  __syncthreads();
  unsigned long long pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long tq = clock64();
#define HQ_TICK(k) do { const unsigned long long t_ = clock64(); pr[k] += t_ - tq; tq = t_; } while (0)
  const int low = 0, high = nn - 1;
  // ------------------------------------------------ orthes (Hessenberg), all warps.
  // Thread t = (c, g): c = t % 64 a column (left update) or row (right update), g = t / 64
  // one of four interleaved slices of the dot product; the four partials meet in part[]
  // and every thread of the column/row then updates its slice.
  double* part = e + nn;          // [4][64] partial dots (e's tail of the shared block)
  double* scr = V;                // 3 x ld + 80 (V's storage once Q is copied out): where the
                                  // bulge step's idle lanes load and store
  const int tc_ = tid & 63, tg = tid >> 6;
  for (int m = low + 1; m <= high - 1; ++m) {
    // the reflector from column m - 1 (every warp redundantly: no barrier for the scalars)
    double scale = 0.0;
    for (int i = m + lane; i <= high; i += 32) scale += fabs(Hx(i, m - 1));
    scale = wp.sum(scale);
    if (scale == 0.0) continue;   // uniform across the CTA
    const double isc = rcp_hc(scale);
    double h = 0.0;
    for (int i = m + lane; i <= high; i += 32) {
      const double o = Hx(i, m - 1) * isc;
      h += o * o;
    }
    h = wp.sum(h);
    const double om = Hx(m, m - 1) * isc;
    const double sq = h * rsqrt_hc(h);   // h > 0: the column below the subdiagonal is not all zero
    const double g = om > 0 ? -sq : sq;
    h = h - om * g;
    const double ih = rcp_hc(h);
    __syncthreads();   // every warp has read column m - 1
    if (tid <= high - m) ort[m + tid] = tid == 0 ? om - g : Hx(m + tid, m - 1) * isc;
    __syncthreads();
    // H = (I - u u'/h) H: f_j = u' H(:, j), j = m .. nn-1
    for (int j0 = m; j0 < nn; j0 += 64) {
      const int j = j0 + tc_;
      double f0 = 0.0, f1 = 0.0;
      if (j < nn) {
        int i = m + tg;
        for (; i + 4 <= high; i += 8) {
          f0 = fma(ort[i], Hx(i, j), f0);
          f1 = fma(ort[i + 4], Hx(i + 4, j), f1);
        }
        if (i <= high) f0 = fma(ort[i], Hx(i, j), f0);
        part[tg * 64 + tc_] = f0 + f1;
      }
      __syncthreads();
      if (j < nn) {
        const double f = ((part[tc_] + part[64 + tc_]) + (part[128 + tc_] + part[192 + tc_])) * ih;
        for (int i = m + tg; i <= high; i += 4) Hx(i, j) -= f * ort[i];
      }
      __syncthreads();
    }
    // H = H (I - u u'/h): g_i = H(i, :) u, i = 0 .. high
    for (int i0 = 0; i0 <= high; i0 += 64) {
      const int i = i0 + tc_;
      double f0 = 0.0, f1 = 0.0;
      if (i <= high) {
        int j = m + tg;
        for (; j + 4 <= high; j += 8) {
          f0 = fma(ort[j], Hx(i, j), f0);
          f1 = fma(ort[j + 4], Hx(i, j + 4), f1);
        }
        if (j <= high) f0 = fma(ort[j], Hx(i, j), f0);
        part[tg * 64 + tc_] = f0 + f1;
      }
      __syncthreads();
      if (i <= high) {
        const double f = ((part[tc_] + part[64 + tc_]) + (part[128 + tc_] + part[192 + tc_])) * ih;
        for (int j = m + tg; j <= high; j += 4) Hx(i, j) -= f * ort[j];
      }
      __syncthreads();
    }
    if (tid == 0) {
      ort[m] = scale * ort[m];
      Hx(m, m - 1) = scale * g;
    }
    __syncthreads();
  }
  HQ_TICK(0);
  if (ovl) {
    double* R = part + 256;          // nn x ld: H as orthes left it (ortran's reflectors)
    double* scr2 = R + nn * ld;      // 3 ld + 80: hqr's scratch block
    for (int idx = tid; idx < nn * nn; idx += NT) {
      const int i = idx / nn, j = idx % nn;
      const double h = Hx(i, j);
      H0[idx] = (i > j + 1) ? 0.0 : h;
      R[i * ld + j] = h;
    }
    for (int i = tid; i < 3 * ld + 80; i += NT) scr2[i] = 0.0;
    __syncthreads();
    if (warp >= 4) {   // ortran on 128 threads (32 columns x 4 slices), named barrier 1
      const int t = tid - 128, tc = t & 31, ts = t >> 5;
      for (int m = high - 1; m >= low + 1; --m) {
        const double hm = R[m * ld + m - 1];
        if (hm == 0.0) continue;   // uniform
        if (t >= 1 && t <= high - m) ort[m + t] = R[(m + t) * ld + m - 1];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const double iom = rcp_hc(ort[m] * hm);
        for (int j0 = m; j0 <= high; j0 += 32) {
          const int j = j0 + tc;
          double f0 = 0.0, f1 = 0.0;
          if (j <= high) {
            int i = m + ts;
            for (; i + 4 <= high; i += 8) {
              f0 = fma(ort[i], Vx(i, j), f0);
              f1 = fma(ort[i + 4], Vx(i + 4, j), f1);
            }
            if (i <= high) f0 = fma(ort[i], Vx(i, j), f0);
            part[ts * 32 + tc] = f0 + f1;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (j <= high) {
            const double f = ((part[tc] + part[32 + tc]) + (part[64 + tc] + part[96 + tc])) * iom;
            for (int i = m + ts; i <= high; i += 4) Vx(i, j) += f * ort[i];
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
      }
      for (int idx = t; idx < nn * nn; idx += 128) Qout[idx] = Vx(idx / nn, idx % nn);
      return;
    }
    if (warp != 0) return;
    scr = scr2;
  } else {
  // ortran: Q explicitly, V(:, j) += g_j u with g_j = u' V(:, j) / (u_m H(m, m-1)),
  // the same (column, slice) thread map
  for (int m = high - 1; m >= low + 1; --m) {
    const double hm = Hx(m, m - 1);
    if (hm == 0.0) continue;   // uniform
    if (tid >= 1 && tid <= high - m) ort[m + tid] = Hx(m + tid, m - 1);
    __syncthreads();
    const double iom = rcp_hc(ort[m] * hm);
    for (int j0 = m; j0 <= high; j0 += 64) {
      const int j = j0 + tc_;
      double f0 = 0.0, f1 = 0.0;
      if (j <= high) {
        int i = m + tg;
        for (; i + 4 <= high; i += 8) {
          f0 = fma(ort[i], Vx(i, j), f0);
          f1 = fma(ort[i + 4], Vx(i + 4, j), f1);
        }
        if (i <= high) f0 = fma(ort[i], Vx(i, j), f0);
        part[tg * 64 + tc_] = f0 + f1;
      }
      __syncthreads();
      if (j <= high) {
        const double f = ((part[tc_] + part[64 + tc_]) + (part[128 + tc_] + part[192 + tc_])) * iom;
        for (int i = m + tg; i <= high; i += 4) Vx(i, j) += f * ort[i];
      }
      __syncthreads();
    }
  }
  // the Hessenberg form and Q for the inverse iteration (below-subdiagonal entries are
  // orthes' workspace: zero them in the copy)
  for (int idx = tid; idx < nn * nn; idx += NT) {
    const int i = idx / nn, j = idx % nn;
    H0[idx] = (i > j + 1) ? 0.0 : Hx(i, j);
    Qout[idx] = Vx(i, j);
  }
  __syncthreads();   // Q copied out: V's storage becomes the scratch block
  for (int i = tid; i < 3 * ld + 80; i += NT) scr[i] = 0.0;
  __syncthreads();
  if (warp != 0) return;   // hqr below is one warp's: no CTA barrier after this point
  }
  // ------------------------------------------------------- hqr (values only)
  int n = nn - 1;
  const double eps = 0x1p-52;
  double exshift = 0.0;
  double p = 0, q = 0, r = 0, s = 0, z = 0, w, x, y;
  double norm = 0.0;
  for (int i = lane; i < nn; i += 32)
    for (int j = (i > 0 ? i - 1 : 0); j < nn; ++j) norm += fabs(Hx(i, j));
  norm = wp.sum(norm);
  int iter = 0, total_iter = 0, fail = 0;
#ifdef CDMD_HQR_PROF2
  unsigned long long pb[3] = {0, 0, 0};
#endif
  HQ_TICK(1);
  while (n >= low) {
    // deflation search, 32 candidates per round: the largest l in (low, n] with a
    // negligible subdiagonal H(l, l-1) (the sequential scan's first hit), else low
    int l = low;
    for (int base = n; base > low; base -= 32) {
      const int cand = base - lane;
      bool hit = false;
      if (cand > low) {
        double sl = fabs(Hx(cand - 1, cand - 1)) + fabs(Hx(cand, cand));
        if (sl == 0.0) sl = norm;
        hit = fabs(Hx(cand, cand - 1)) < eps * sl;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (bal) {
        l = base - (__ffs(bal) - 1);
        break;
      }
    }
    HQ_TICK(2);
    if (l == n) {  // one root
      if (lane == 0) {
        d[n] = Hx(n, n) + exshift;
        e[n] = 0.0;
      }
      n--;
      iter = 0;
    } else if (l == n - 1) {  // two roots
      w = Hx(n, n - 1) * Hx(n - 1, n);
      p = (Hx(n - 1, n - 1) - Hx(n, n)) / 2.0;
      q = p * p + w;
      z = sqrt(fabs(q));
      x = Hx(n, n) + exshift;
      if (q >= 0) {
        z = (p >= 0) ? p + z : p - z;
        double dn = x + z;
        if (z != 0.0) dn = x - w / z;
        if (lane == 0) {
          d[n - 1] = x + z;
          d[n] = dn;
          e[n - 1] = 0.0;
          e[n] = 0.0;
        }
      } else if (lane == 0) {
        d[n - 1] = x + p;
        d[n] = x + p;
        e[n - 1] = z;
        e[n] = -z;
      }
      n = n - 2;
      iter = 0;
    } else {  // shift
      x = Hx(n, n);
      y = 0.0;
      w = 0.0;
      if (l < n) {
        y = Hx(n - 1, n - 1);
        w = Hx(n, n - 1) * Hx(n - 1, n);
      }
      if (iter == 10) {
        exshift += x;
        wp.sync();
        for (int i = low + lane; i <= n; i += 32) Hx(i, i) -= x;
        wp.sync();
        s = fabs(Hx(n, n - 1)) + fabs(Hx(n - 1, n - 2));
        x = y = 0.75 * s;
        w = -0.4375 * s * s;
      }
      if (iter == 30) {
        s = (y - x) / 2.0;
        s = s * s + w;
        if (s > 0) {
          s = sqrt(s);
          if (y < x) s = -s;
          s = x - w / ((y - x) / 2.0 + s);
          wp.sync();
          for (int i = low + lane; i <= n; i += 32) Hx(i, i) -= s;
          wp.sync();
          exshift += s;
          x = y = w = 0.964;
        }
      }
      iter++;
      if (++total_iter > 60 * nn) {
        fail = 1;
        break;
      }
      pr[5]++;
      // start of the bulge, 32 candidates per round: the largest m in [l, n-2] where two
      // consecutive small subdiagonals allow splitting (or m = l), with its (p, q, r)
      // carried multiplied by H(m+1, m) (no divisions), as the sequential scan
      int m = l;
      for (int base = n - 2; base >= l; base -= 32) {
        const int cand = base - lane;
        bool hit = false;
        double pp = 0.0, qq = 0.0, rr = 0.0;
        if (cand >= l) {
          const double zz = Hx(cand, cand);
          const double r_ = x - zz, s_ = y - zz;
          const double h = Hx(cand + 1, cand);
          pp = (r_ * s_ - w) + Hx(cand, cand + 1) * h;
          qq = (Hx(cand + 1, cand + 1) - zz - r_ - s_) * h;
          rr = Hx(cand + 2, cand + 1) * h;
          hit = (cand == l) || (fabs(Hx(cand, cand - 1)) * (fabs(qq) + fabs(rr)) <
                                eps * (fabs(pp) * (fabs(Hx(cand - 1, cand - 1)) + fabs(zz) + fabs(Hx(cand + 1, cand + 1)))));
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (bal) {
          const int src = __ffs(bal) - 1;
          m = base - src;
          p = __shfl_sync(0xffffffffu, pp, src);
          q = __shfl_sync(0xffffffffu, qq, src);
          r = __shfl_sync(0xffffffffu, rr, src);
          break;
        }
      }
      {
        const double sc = fabs(p) + fabs(q) + fabs(r);
        if (sc != 0.0) {
          const double isc = rcp_nr(sc);
          p *= isc;
          q *= isc;
          r *= isc;
        }
      }
      HQ_TICK(3);
      wp.sync();
      for (int i = m + 2 + lane; i <= n; i += 32) {
        Hx(i, i - 2) = 0.0;
        if (i > m + 2) Hx(i, i - 3) = 0.0;
      }
      // EISPACK negates H(m, m-1) at the first bulge step when the bulge starts below l;
      // it does not depend on the reflector, so it is done here, off the step loop
      const double hneg = (l != m) ? -Hx(m, m - 1) : 0.0;
      wp.sync();
      if (l != m && lane == 0) Hx(m, m - 1) = hneg;
      wp.sync();
      pr[6] += n - m;
#ifdef CDMD_HQR_PROF2
      unsigned long long tb_prev = clock64();
#endif
      // Each step splits into the 3 x 3 block B = H(kk..kk+2, kk..kk+2) and row kk+3 of
      // columns kk..kk+2, which every lane updates redundantly in registers (they hold the
      // next step's p, q, r: no shuffle or shared-memory round trip on the chain), and the
      // rest -- rows kk..kk+2 of columns kk+3..n, columns kk..kk+2 of rows l..kk-1 -- one
      // column / row per lane slot.  Every operand is loaded at the top of the step, before
      // the reflector is known.  Idle lanes and the absent row / column kk+2 of the last
      // step (r = z = 0) use the scratch block: scr[0..2] stays zero, scr[4..6] is the
      // column-update dummy, scr[8 + lane + {0, ld, 2 ld}] the row-update dummies.
      double* const Z0 = scr;
      double* const CD = scr + 4;
      // (p, q, r) of every step come from registers: the bulge start's for kk = m, the
      // previous step's updated block otherwise, or -- after a skipped step -- column kk of H
      double pn = p, qn = q, rn = r;
      for (int kk = m; kk <= n - 1; ++kk) {  // double QR step on the active block l..n
        const bool notlast = (kk != n - 1);
        // ---- operands (independent of this step's reflector)
        double* bp[3][3];
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int c = 0; c < 3; ++c) bp[t][c] = (notlast || (t < 2 && c < 2)) ? &Hx(kk + t, kk + c) : Z0;
        double B[3][3];
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int c = 0; c < 3; ++c) B[t][c] = *bp[t][c];
        const bool has3 = kk + 3 <= n;
        const double* r3l = has3 ? &Hx(kk + 3, kk) : Z0;
        double* r3s = has3 ? &Hx(kk + 3, kk) : CD;
        double r30 = r3l[0], r31 = r3l[1], r32 = notlast ? r3l[2] : 0.0;
        const int j0 = kk + 3 + lane, j1 = j0 + 32;
        double* rb0 = j0 <= n ? &Hx(kk, j0) : scr + 8 + lane;
        double* rb1 = j1 <= n ? &Hx(kk, j1) : scr + 40 + lane;
        double u0 = rb0[0], u1 = rb0[ld], u2 = rb0[2 * ld];
        double w0 = rb1[0], w1 = rb1[ld], w2 = rb1[2 * ld];
        const int i0 = l + lane, i1 = i0 + 32;
        double* cb0 = i0 <= kk - 1 ? &Hx(i0, kk) : CD;
        double* cb1 = i1 <= kk - 1 ? &Hx(i1, kk) : CD;
        double g00 = cb0[0], g01 = cb0[1], g02 = cb0[2];
        double g10 = cb1[0], g11 = cb1[1], g12 = cb1[2];
        // ---- the reflector
        p = pn;
        q = qn;
        r = notlast ? rn : 0.0;
        // EISPACK scales (p, q, r) by |p| + |q| + |r|; the scaling only matters near under- or
        // overflow, so the range test is taken on p^2 + q^2 + r^2 (needed anyway) and the
        // abs-sum stays off the step's dependent chain (x = 1 otherwise, as before)
        double ss = p * p + q * q + r * r;
        double is = rsqrt_hc(ss);   // 1 / s, s = sign(p) ||(p, q, r)|| (issued before the range test)
        x = 1.0;
        if (!(ss >= 1e-280 && ss <= 1e280)) {   // rare: one branch per step for every special case
          // a skipped step hands the next one column kk of H as its (p, q, r)
          auto skip_operands = [&]() {
            if (kk + 1 <= n - 1) {
              pn = Hx(kk + 1, kk);
              qn = Hx(kk + 2, kk);
              rn = (kk + 3 <= n) ? Hx(kk + 3, kk) : 0.0;
            }
          };
          if (kk != m) {
            x = fabs(p) + fabs(q) + fabs(r);
            if (x == 0.0) { skip_operands(); continue; }
            const double ix = 1.0 / x;
            p = p * ix;
            q = q * ix;
            r = r * ix;
            ss = p * p + q * q + r * r;
            is = rsqrt_hc(ss);
          }
          if (ss == 0.0) { skip_operands(); continue; }
        }
        if (p < 0) is = -is;
        s = ss * is;
        if (kk != m) Hx(kk, kk - 1) = -s * x;   // every lane the same value; read by no lane this step
#ifdef CDMD_HQR_PROF2
        unsigned long long tb0 = clock64();
#endif
        p = fma(ss, is, p);   // p + s
        const double ip = rcp_hc(p);
        x = p * is;
        y = q * is;
        z = r * is;
        q = q * ip;
        r = r * ip;
        // ---- block and row kk+3 (every lane): rows from the left, then columns from the right
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double pp = fma(r, B[2][c], fma(q, B[1][c], B[0][c]));
          B[0][c] -= pp * x;
          B[1][c] -= pp * y;
          B[2][c] -= pp * z;
        }
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const double pp = fma(z, B[t][2], fma(y, B[t][1], x * B[t][0]));
          B[t][0] -= pp;
          B[t][1] -= pp * q;
          B[t][2] -= pp * r;
        }
        {
          const double pp = fma(z, r32, fma(y, r31, x * r30));
          r30 -= pp;
          r31 -= pp * q;
          r32 -= pp * r;
        }
        // ---- the rest, a column / row per lane slot
        {
          const double pu = fma(r, u2, fma(q, u1, u0));
          const double pw = fma(r, w2, fma(q, w1, w0));
          u0 -= pu * x;
          u1 -= pu * y;
          u2 -= pu * z;
          w0 -= pw * x;
          w1 -= pw * y;
          w2 -= pw * z;
          const double pg = fma(z, g02, fma(y, g01, x * g00));
          const double ph = fma(z, g12, fma(y, g11, x * g10));
          g00 -= pg;
          g01 -= pg * q;
          g02 -= pg * r;
          g10 -= ph;
          g11 -= ph * q;
          g12 -= ph * r;
        }
#ifdef CDMD_HQR_PROF2
        unsigned long long tb1 = clock64();
#endif
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
          for (int c = 0; c < 3; ++c) *bp[t][c] = B[t][c];
        r3s[0] = r30;
        r3s[1] = r31;
        if (notlast) r3s[2] = r32;
        rb0[0] = u0;
        rb0[ld] = u1;
        rb0[2 * ld] = u2;
        rb1[0] = w0;
        rb1[ld] = w1;
        rb1[2 * ld] = w2;
        cb0[0] = g00;
        cb0[1] = g01;
        cb0[2] = g02;
        cb1[0] = g10;
        cb1[1] = g11;
        cb1[2] = g12;
        // slots beyond two (n > 64): plain loops, behind warp-uniform guards (one test per
        // step when the matrix has at most 64 rows)
        if (BIG || nn > 64) {   // (the run-time test in the small instantiation measured faster
                                // than removing the loops at compile time: 1.17 M vs 1.26 M cycles)
        if (kk + 3 + 64 <= n)
        for (int j = j1 + 32; j <= n; j += 32) {
          double pp = Hx(kk, j) + q * Hx(kk + 1, j);
          if (notlast) {
            pp = pp + r * Hx(kk + 2, j);
            Hx(kk + 2, j) = Hx(kk + 2, j) - pp * z;
          }
          Hx(kk, j) = Hx(kk, j) - pp * x;
          Hx(kk + 1, j) = Hx(kk + 1, j) - pp * y;
        }
        if (l + 64 <= kk - 1)
        for (int i = i1 + 32; i <= kk - 1; i += 32) {
          double pp = x * Hx(i, kk) + y * Hx(i, kk + 1);
          if (notlast) {
            pp = pp + z * Hx(i, kk + 2);
            Hx(i, kk + 2) = Hx(i, kk + 2) - pp * r;
          }
          Hx(i, kk) = Hx(i, kk) - pp;
          Hx(i, kk + 1) = Hx(i, kk + 1) - pp * q;
        }
        }
        pn = B[1][0];
        qn = B[2][0];
        rn = r30;
        wp.sync();
#ifdef CDMD_HQR_PROF2
        unsigned long long tb2 = clock64();
        pb[0] += tb0 - tb_prev;
        pb[1] += tb1 - tb0;
        pb[2] += tb2 - tb1;
        tb_prev = tb2;
#endif
      }
      HQ_TICK(4);
    }
  }
  wp.sync();
  if (lane == 0) {
    for (int k2 = 0; k2 < 7; ++k2) g_hqr_prof[k2] = pr[k2];
#ifdef CDMD_HQR_PROF2
    for (int k2 = 0; k2 < 3; ++k2) g_hqr_prof2[k2] = pb[k2];
#endif
  }
#undef HQ_TICK
  if (fail) {
    if (lane == 0) *info = 1;
    return;
  }
  for (int j = lane; j < nn; j += 32) {
    W[2 * j] = d[j];
    W[2 * j + 1] = e[j];
  }
  if (lane == 0) *info = 0;
#undef Hx
#undef Vx
}

// Inverse iteration on the Hessenberg H0 for eigenvalue j (a warp per CTA; the
// complex conjugate pair (wi > 0, then wi < 0) is solved once, in complex arithmetic,
// by the CTA of its first member).  LU of H0 - lambda I with partial pivoting between
// adjacent rows (Hessenberg), a first solve U x = eps3 (EISPACK invit), one more
// inverse-iteration step, then v = Q x.  VR column j = Re v (and j+1 = Im v for a
// pair); canonicalize_kernel normalises and phases it.
constexpr int HI_WARPS = 4;   // eigenvalues per CTA of hinvit_kernel (a warp each, own shared slice)

__global__ void __launch_bounds__(32 * HI_WARPS) hinvit_kernel(int nn, const double* __restrict__ W,
                                                              const double* __restrict__ H0,
                                                              const double* __restrict__ Q,
                                                              double* __restrict__ VR, size_t warp_doubles) {
  extern __shared__ double smv[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j = blockIdx.x * (int)(blockDim.x >> 5) + wid;
  if (j >= nn) return;
  double* sm = smv + (size_t)wid * warp_doubles;
  const double wr = W[2 * j], wi = W[2 * j + 1];
  if (wi < 0.0) return;   // second member of a pair
  const bool cx = wi != 0.0;
  const int ld = nn + 1;
  double* Br = sm;                    // nn x ld (row-major), becomes U
  double* Bi = Br + nn * ld;          // imaginary part (pairs)
  double* xr = Bi + nn * ld;          // nn
  double* xi = xr + nn;               // nn
  double* mr = xi + nn;               // multipliers (nn)
  double* mi = mr + nn;
  uint8_t* sw = reinterpret_cast<uint8_t*>(mi + nn);   // row swap flags
  double norm = 0.0;
  for (int idx = lane; idx < nn * nn; idx += 32) {
    const int i = idx / nn, c = idx % nn;
    const double h = H0[idx];
    norm += fabs(h);
    Br[i * ld + c] = h - (i == c ? wr : 0.0);
    Bi[i * ld + c] = (i == c) ? -wi : 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) norm += __shfl_xor_sync(0xffffffffu, norm, o);
  if (norm == 0.0) norm = 1.0;
  const double eps3 = norm * 0x1p-52;   // replaces zero pivots, seeds the first solve
  __syncwarp();
  // LU with partial pivoting between rows k and k+1
  for (int k = 0; k < nn - 1; ++k) {
    const double ar = Br[k * ld + k], ai = Bi[k * ld + k];
    const double br = Br[(k + 1) * ld + k], bi = Bi[(k + 1) * ld + k];
    const bool swp = fabs(br) + fabs(bi) > fabs(ar) + fabs(ai);
    double pr = swp ? br : ar, pi = swp ? bi : ai;   // pivot
    const double lr = swp ? ar : br, li = swp ? ai : bi;   // eliminated
    if (pr == 0.0 && pi == 0.0) pr = eps3;
    double cr, ci;   // multiplier l / p
    cdiv_fast(lr, li, pr, pi, cr, ci);
    __syncwarp();
    for (int c = k + lane; c < nn; c += 32) {
      double ur = Br[k * ld + c], ui = Bi[k * ld + c];
      double vr = Br[(k + 1) * ld + c], vi = Bi[(k + 1) * ld + c];
      if (swp) {
        const double tr = ur, ti = ui;
        ur = vr; ui = vi; vr = tr; vi = ti;
      }
      if (c == k) { ur = pr; ui = pi; }
      Br[k * ld + c] = ur;
      Bi[k * ld + c] = ui;
      Br[(k + 1) * ld + c] = vr - (cr * ur - ci * ui);
      Bi[(k + 1) * ld + c] = vi - (cr * ui + ci * ur);
    }
    if (lane == 0) {
      mr[k] = cr;
      mi[k] = ci;
      sw[k] = swp ? 1 : 0;
    }
    __syncwarp();
  }
  if (lane == 0 && Br[(nn - 1) * ld + nn - 1] == 0.0 && Bi[(nn - 1) * ld + nn - 1] == 0.0)
    Br[(nn - 1) * ld + nn - 1] = eps3;
  for (int i = lane; i < nn; i += 32) {
    xr[i] = eps3;
    xi[i] = 0.0;
  }
  __syncwarp();
  for (int it = 0; it < 2; ++it) {
    if (it > 0 && lane == 0) {   // apply L^-1 (row swaps and multipliers) to x
      for (int k = 0; k < nn - 1; ++k) {
        double ar = xr[k], ai = xi[k], br = xr[k + 1], bi = xi[k + 1];
        if (sw[k]) {
          const double tr = ar, ti = ai;
          ar = br; ai = bi; br = tr; bi = ti;
        }
        xr[k] = ar;
        xi[k] = ai;
        xr[k + 1] = br - (mr[k] * ar - mi[k] * ai);
        xi[k + 1] = bi - (mr[k] * ai + mi[k] * ar);
      }
    }
    __syncwarp();
    // U x = rhs, column-oriented back substitution
    for (int i = nn - 1; i >= 0; --i) {
      double ur = Br[i * ld + i], ui = Bi[i * ld + i];
      if (ur == 0.0 && ui == 0.0) ur = eps3;
      double vr, vi;
      cdiv_fast(xr[i], xi[i], ur, ui, vr, vi);
      __syncwarp();
      for (int r2 = lane; r2 < i; r2 += 32) {
        const double cr = Br[r2 * ld + i], ci = Bi[r2 * ld + i];
        xr[r2] -= cr * vr - ci * vi;
        xi[r2] -= cr * vi + ci * vr;
      }
      if (lane == 0) {
        xr[i] = vr;
        xi[i] = vi;
      }
      __syncwarp();
    }
    // rescale (inverse iteration grows the vector by ~1 / dist(lambda, spectrum))
    double mx = 0.0;
    for (int i = lane; i < nn; i += 32) mx = fmax(mx, fabs(xr[i]) + fabs(xi[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
    for (int i = lane; i < nn; i += 32) {
      xr[i] *= sc;
      xi[i] *= sc;
    }
    __syncwarp();
  }
  // v = Q x
  for (int i = lane; i < nn; i += 32) {
    double ar = 0.0, ai = 0.0;
    const double* qrow = Q + (int64_t)i * nn;
    for (int c = 0; c < nn; ++c) {
      const double qv = __ldg(qrow + c);
      ar = fma(qv, xr[c], ar);
      ai = fma(qv, xi[c], ai);
    }
    VR[(int64_t)j * nn + i] = ar;
    if (cx) VR[(int64_t)(j + 1) * nn + i] = ai;
  }
}

// hqrv: H | V (at least the bulge step's 3 (k+1) + 64 scratch) | ort, d, e | part[256]
static size_t hqr_vsz(int k) {
  const size_t a = (size_t)k * (k + 1), b = 3 * ((size_t)k + 1) + 80;
  return a > b ? a : b;
}
size_t hqr_smem_bytes(int k) { return sizeof(double) * ((size_t)k * (k + 1) + hqr_vsz(k) + 3 * (size_t)k + 256); }
static size_t hqr_smem_par3(int k) { return hqr_smem_bytes(k) + sizeof(double) * 64 * (size_t)k; }

static size_t hinvit_smem(int k) { return sizeof(double) * ((size_t)2 * k * (k + 1) + 4 * (size_t)k) + k + 16; }

// scratch: >= 2 k^2 doubles (the Hessenberg form and Q of the v2 path)
cudaError_t launch_hqr_eig(int k, const double* A, double* W, double* VR, int* info, double* scratch,
                           cudaStream_t st) {
  if (scratch && hinvit_smem(k) <= 226 * 1024 && !getenv("CDMD_EIG_V1")) {
    double* H0 = scratch;
    double* Q = scratch + (size_t)k * k;
    const size_t smem = hqr_smem_bytes(k);
    auto kern = k > 64 ? hqrv_kernel<true> : hqrv_kernel<false>;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern));
    if (e != cudaSuccess) return e;
    // Q accumulated beside hqr when the copy of H and a separate scratch block fit
    const size_t smem_ovl = smem + sizeof(double) * ((size_t)k * (k + 1) + 3 * ((size_t)k + 1) + 80);
    const int ovl = (smem_ovl <= 226 * 1024 && !getenv("CDMD_HQR_SEQ")) ? 1 : 0;
    note_launch();
    kern<<<1, 32 * HQ_WARPS, ovl ? smem_ovl : smem, st>>>(k, A, W, H0, Q, info, ovl);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // a warp per eigenvalue, HI_WARPS to a CTA when their shared slices fit (fewer SMs held
    // while the streaming lanes' passes run)
    const size_t wd = (hinvit_smem(k) + 15) / 8;
    const int per = sizeof(double) * wd * HI_WARPS <= 200 * 1024 ? HI_WARPS : 1;
    e = smem_optin(reinterpret_cast<const void*>(hinvit_kernel));
    if (e != cudaSuccess) return e;
    note_launch();
    if (per == HI_WARPS)
      hinvit_kernel<<<(unsigned)ceil_div(k, HI_WARPS), 32 * HI_WARPS, sizeof(double) * wd * HI_WARPS, st>>>(k, W, H0, Q,
                                                                                                        VR, wd);
    else
      hinvit_kernel<<<(unsigned)k, 32, sizeof(double) * wd, st>>>(k, W, H0, Q, VR, wd);
    return cudaGetLastError();
  }
  const int par3 = hqr_smem_par3(k) <= 226 * 1024;
  const size_t smem = par3 ? hqr_smem_par3(k) : hqr_smem_bytes(k);
  cudaError_t e = smem_optin(reinterpret_cast<const void*>(hqr_eig_kernel));
  if (e != cudaSuccess) return e;
  note_launch();
  hqr_eig_kernel<<<1, 32, smem, st>>>(k, A, W, VR, info, par3);
  return cudaGetLastError();
}

}  // namespace cdmd
