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

}  // namespace fmmbem
