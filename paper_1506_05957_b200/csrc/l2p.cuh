// Streaming L2P: evaluates a half-stored local expansion (and its gradient)
// at one point without materialising R_n^m: the regular harmonics are
// generated column by column (fixed m, increasing n) with the recurrences of
// harmonics.py:38-59 and consumed immediately.
//
//   phi      = Re sum_{n,m} L_n^m R_n^m          (harmonics.py:258-270)
//   d_z phi  = sum L_{n+1}^m R_n^m               (dz R_n^m = R_{n-1}^m)
//   (d_x + i d_y) phi = sum L_{n+1}^{m-1} R_n^m  ((dx+idy) R_n^m = R_{n-1}^{m+1})
// Real symmetry folds the m < 0 half into the m >= 0 terms.
#pragma once

#include "common.cuh"

namespace fmmbem {

// (m0, mstep): only the columns m = m0, m0 + mstep, ... (split over threads)
template <int C, bool GRAD>
__device__ __forceinline__ void l2p_eval(const double2* __restrict__ L, int H, int p, double x,
                                         double y, double z, double* pot, double* grad,
                                         const double* __restrict__ rec, int m0 = 0, int mstep = 1) {
  const double rho2 = x * x + y * y + z * z;
  double zr[C], zi[C], gz[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { zr[c] = 0.0; zi[c] = 0.0; gz[c] = 0.0; }
  double2 diag = make_double2(1.0, 0.0);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) diag = cscale(cmul(make_double2(x, y), diag), __ldg(rec + REC_DIAG + m));
    if (m < m0 || (m - m0) % mstep) continue;
    double2 prev2 = make_double2(0.0, 0.0), cur = diag;
    const double w = m == 0 ? 1.0 : 2.0;
    for (int n = m; n <= p; ++n) {
      if (n == m + 1) {
        prev2 = cur;
        cur = cscale(cur, z);
      } else if (n > m + 1) {
        const double inv = __ldg(rec + n * (P_MAX + 1) + m);
        double2 nx;
        nx.x = ((2 * n - 1) * z * cur.x - rho2 * prev2.x) * inv;
        nx.y = ((2 * n - 1) * z * cur.y - rho2 * prev2.y) * inv;
        prev2 = cur;
        cur = nx;
      }
      const int i0 = hidx(n, m);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double2 l = L[c * H + i0];
        pot[c] = fma(w, fma(l.x, cur.x, -l.y * cur.y), pot[c]);
      }
      if (GRAD && n < p) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double2* Lc = L + c * H;
          const double2 lz = Lc[hidx(n + 1, m)];
          gz[c] = fma(w, fma(lz.x, cur.x, -lz.y * cur.y), gz[c]);
          // L_{n+1}^{m-1} R_n^m, with L^{-1} = -conj(L^1)
          double2 a = (m > 0) ? Lc[hidx(n + 1, m - 1)] : Lc[hidx(n + 1, 1)];
          if (m == 0) a = make_double2(-a.x, a.y);
          double2 t = cmul(a, cur);
          zr[c] += t.x;
          zi[c] += t.y;
          if (m > 0) {
            // - conj(L_{n+1}^{m+1} R_n^m)
            const double2 u = cmul(Lc[hidx(n + 1, m + 1)], cur);
            zr[c] -= u.x;
            zi[c] += u.y;
          }
        }
      }
    }
  }
  if (GRAD) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      grad[3 * c + 0] += zr[c];
      grad[3 * c + 1] += zi[c];
      grad[3 * c + 2] += gz[c];
    }
  }
}

// One-channel potential-only L2P for 4 column slices (warp-uniform): slice k evaluates the
// columns m with (m mod 8) in {k, 7 - k} (column m has p + 1 - m terms: near-equal shares).
// Each column starts from R_m^m = c_m (x + i y)^m, c_m = prod_{j <= m} -1/(2j)
// (harmonics.py:50-52), by binary powering, and runs the n-recurrence with the coefficients
// (2n-1)/((n+m)(n-m)) and 1/((n+m)(n-m)) from constant memory (warp-uniform (n, m)).
struct L2PConst {
  double diag[P_MAX + 1];
  double ra[(P_MAX + 1) * (P_MAX + 1)];  // [n][m] (2n - 1) / ((n + m)(n - m))
  double rb[(P_MAX + 1) * (P_MAX + 1)];  // [n][m] 1 / ((n + m)(n - m))
};
// (one copy per translation unit: no relocatable device code; operator.cu uploads its own)
static __constant__ L2PConst c_l2p;

__device__ __forceinline__ double2 cpow_int(double2 w, int m) {
  double2 r = make_double2(1.0, 0.0);
  while (m) {
    if (m & 1) r = cmul(r, w);
    m >>= 1;
    if (m) w = cmul(w, w);
  }
  return r;
}

__device__ __forceinline__ double l2p_eval1(const double2* __restrict__ L, int p, double x, double y,
                                            double z, int slice) {
  const double rho2 = x * x + y * y + z * z;
  const double2 w = make_double2(x, y);
  double acc = 0.0;
  for (int m0 = 0; m0 <= p; m0 += 8) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = m0 + (h ? 7 - slice : slice);
      if (m > p) continue;
      double2 cur = cscale(cpow_int(w, m), c_l2p.diag[m]), prev2 = make_double2(0.0, 0.0);
      int i = hidx(m, m);
      double col = fma(L[i].x, cur.x, -L[i].y * cur.y);
      if (m < p) {
        prev2 = cur;
        cur = cscale(cur, z);
        i += m + 1;
        col = fma(L[i].x, cur.x, fma(-L[i].y, cur.y, col));
      }
      for (int n = m + 2; n <= p; ++n) {
        const double az = c_l2p.ra[n * (P_MAX + 1) + m] * z, b = c_l2p.rb[n * (P_MAX + 1) + m] * rho2;
        const double2 nx = make_double2(fma(az, cur.x, -b * prev2.x), fma(az, cur.y, -b * prev2.y));
        prev2 = cur;
        cur = nx;
        i += n;
        col = fma(L[i].x, cur.x, fma(-L[i].y, cur.y, col));
      }
      acc = m == 0 ? acc + col : fma(2.0, col, acc);
    }
  }
  return acc;
}

}  // namespace fmmbem
