// Single-expansion operators on the device: the reference's Expansion / p2m / m2m / m2l /
// l2l / m2p / l2p (pkg/src/fmmbem/fmm.py:36-81) over harmonics.particle_to_multipole,
// translation_matrix, multipole_to_point and local_to_point (harmonics.py:201-270).
//
// These act on ONE expansion (C channels) in the reference's FULL flat layout
// idx(n, m) = n^2 + n + m, complex as interleaved (re, im) doubles, so arbitrary complex
// coefficient sets (not only real-field ones) go through unchanged.  They are not on the
// apply path (the plan kernels use half storage and batched tables); they give the
// per-operator unit checks of the reference's test_harmonics.py / acceptance criterion 7
// a device counterpart.  Every sum runs in a fixed order per output (no atomics).
#include "kernels.cuh"

namespace fmmbem {
namespace {

__device__ __forceinline__ int fidx(int n, int m) { return n * n + n + m; }

// R_n^m(x, y, z) for one (n, m), |m| <= n, by the recurrences of harmonics.regular
// (harmonics.py:38-59): sectoral, then n = m+1, then the two-term recurrence in n.
__device__ double2 reg_nm(double x, double y, double z, int n, int m) {
  const int am = m < 0 ? -m : m;
  if (am > n || n < 0) return make_double2(0.0, 0.0);
  const double rho2 = x * x + y * y + z * z;
  double2 s = make_double2(1.0, 0.0);
  for (int k = 1; k <= am; ++k) s = cmul(make_double2(-x / (2 * k), -y / (2 * k)), s);
  double2 prev = make_double2(0.0, 0.0), cur = s;
  for (int k = am + 1; k <= n; ++k) {
    double2 nxt;
    if (k == am + 1) {
      nxt = cscale(cur, z);
    } else {
      nxt.x = ((2 * k - 1) * z * cur.x - rho2 * prev.x) / ((double)(k + am) * (k - am));
      nxt.y = ((2 * k - 1) * z * cur.y - rho2 * prev.y) / ((double)(k + am) * (k - am));
    }
    prev = cur;
    cur = nxt;
  }
  if (m < 0) {
    cur = cconj(cur);
    if (am & 1) cur = make_double2(-cur.x, -cur.y);
  }
  return cur;
}

// full tables R_n^m or I_n^m (n <= p) in `out`, by harmonics.regular / irregular (:38-85)
__device__ void table_full(double x, double y, double z, int p, bool irr, double2* out) {
  const double rho2 = x * x + y * y + z * z;
  out[0] = make_double2(irr ? 1.0 / sqrt(rho2) : 1.0, 0.0);
  for (int m = 1; m <= p; ++m) {
    const double2 f = irr ? make_double2(-(2 * m - 1) * x / rho2, -(2 * m - 1) * y / rho2)
                          : make_double2(-x / (2 * m), -y / (2 * m));
    out[fidx(m, m)] = cmul(f, out[fidx(m - 1, m - 1)]);
  }
  for (int m = 0; m < p; ++m)
    out[fidx(m + 1, m)] = cscale(out[fidx(m, m)], irr ? (2 * m + 1) * z / rho2 : z);
  for (int m = 0; m <= p; ++m)
    for (int n = m + 2; n <= p; ++n) {
      const double2 a = out[fidx(n - 1, m)], b = out[fidx(n - 2, m)];
      if (irr) {
        const double c = (double)((n - 1) * (n - 1) - m * m);
        out[fidx(n, m)] = make_double2(((2 * n - 1) * z * a.x - c * b.x) / rho2,
                                       ((2 * n - 1) * z * a.y - c * b.y) / rho2);
      } else {
        const double d = (double)(n + m) * (n - m);
        out[fidx(n, m)] = make_double2(((2 * n - 1) * z * a.x - rho2 * b.x) / d,
                                       ((2 * n - 1) * z * a.y - rho2 * b.y) / d);
      }
    }
  for (int n = 1; n <= p; ++n)
    for (int m = 1; m <= n; ++m) {
      const double2 v = cconj(out[fidx(n, m)]);
      out[fidx(n, -m)] = (m & 1) ? make_double2(-v.x, -v.y) : v;
    }
}

__device__ __forceinline__ double2 tget(const double2* t, int p, int n, int m) {
  return (n >= 0 && n <= p && (m < 0 ? -m : m) <= n) ? t[fidx(n, m)] : make_double2(0.0, 0.0);
}

// harmonics.particle_to_multipole: thread = (channel, coefficient), sources in order
__global__ void k_exp_p2m(int64_t N, int C, int p, const double* __restrict__ rel,
                          const double* __restrict__ q, const double* __restrict__ d,
                          double2* __restrict__ out) {
  const int S = (p + 1) * (p + 1);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= C * S) return;
  const int c = t / S, i = t % S;
  const int n = (int)sqrt((double)i + 0.5);
  const int m = i - n * n - n;
  double2 acc = make_double2(0.0, 0.0);
  double2 dip = make_double2(0.0, 0.0);
  for (int64_t j = 0; j < N; ++j) {
    const double x = rel[3 * j], y = rel[3 * j + 1], z = rel[3 * j + 2];
    if (q) {
      const double2 r = reg_nm(x, y, z, n, m);
      acc.x += q[(size_t)c * N + j] * r.x;
      acc.y += q[(size_t)c * N + j] * r.y;
    }
    if (d && n >= 1) {
      // d . grad R = 1/2 (dx - i dy) R_{n-1}^{m+1} - 1/2 (dx + i dy) R_{n-1}^{m-1} + dz R_{n-1}^m
      const double* dd = d + ((size_t)c * N + j) * 3;
      const double2 a = reg_nm(x, y, z, n - 1, m + 1), b = reg_nm(x, y, z, n - 1, m - 1);
      const double2 g = reg_nm(x, y, z, n - 1, m);
      // gx = (a - b)/2, gy = (a + b)/(2i) with b the raw R_{n-1}^{m-1} (shift rule sign folded)
      const double2 gx = make_double2(0.5 * (a.x - b.x), 0.5 * (a.y - b.y));
      const double2 gy = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x + b.x));
      dip.x += dd[0] * gx.x + dd[1] * gy.x + dd[2] * g.x;
      dip.y += dd[0] * gx.y + dd[1] * gy.y + dd[2] * g.y;
    }
  }
  out[t] = make_double2(acc.x + dip.x, acc.y + dip.y);
}

// translation_matrix('m2m' | 'l2l' | 'm2l', d, p) applied: one CTA per channel,
// thread per output coefficient; the R (order p) or I (order 2p) table of d in shared memory
__global__ void k_exp_translate(int kind, int C, int p, double dx, double dy, double dz,
                                const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ double2 tab[];
  const int S = (p + 1) * (p + 1);
  const int tp = kind == 1 ? 2 * p : p;
  if (threadIdx.x == 0) table_full(dx, dy, dz, tp, kind == 1, tab);
  __syncthreads();
  const double2* cin = in + (size_t)blockIdx.x * S;
  for (int o = threadIdx.x; o < S; o += blockDim.x) {
    const int n = (int)sqrt((double)o + 0.5), m = o - n * n - n;
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j <= p; ++j)
      for (int k = -j; k <= j; ++k) {
        const double2 v = cin[fidx(j, k)];
        if (kind == 0) {          // M2M: R_{n-j}^{m-k}, j <= n, |m-k| <= n-j
          if (j > n) continue;
          acc = cfma(v, tget(tab, tp, n - j, m - k), acc);
        } else if (kind == 2) {   // L2L: R_{j-n}^{k-m}, j >= n, |k-m| <= j-n
          if (j < n) continue;
          acc = cfma(v, tget(tab, tp, j - n, k - m), acc);
        } else {                  // M2L: (-1)^n conj(I_{j+n}^{k+m}) (output (n, m), input (j, k))
          acc = cfma(v, cconj(tab[fidx(j + n, k + m)]), acc);
        }
      }
    if (kind == 1 && (n & 1)) acc = make_double2(-acc.x, -acc.y);
    out[(size_t)blockIdx.x * S + o] = acc;
  }
}

// multipole_to_point / local_to_point (harmonics.py:238-270): thread per target
__global__ void k_exp_eval(int kind, int C, int p, int64_t N, const double* __restrict__ rel,
                           const double2* __restrict__ coeffs, int want_grad,
                           double* __restrict__ pot, double* __restrict__ grad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= N) return;
  double2 tab[(P_MAX + 2) * (P_MAX + 2)];
  const bool irr = kind == 0;
  const int tp = (irr && want_grad) ? p + 1 : p;
  table_full(rel[3 * t], rel[3 * t + 1], rel[3 * t + 2], tp, irr, tab);
  const int S = (p + 1) * (p + 1);
  for (int c = 0; c < C; ++c) {
    const double2* cc = coeffs + (size_t)c * S;
    double ph = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int n = 0; n <= p; ++n)
      for (int m = -n; m <= n; ++m) {
        const double2 v = cc[fidx(n, m)];
        // pot: Re(c conj(I)) for M2P, Re(c R) for L2P
        const double2 h = tab[fidx(n, m)];
        ph += irr ? v.x * h.x + v.y * h.y : v.x * h.x - v.y * h.y;
        if (!want_grad) continue;
        double2 a, b, g;
        if (irr) {  // irregular_gradient: a = I_{n+1}^{m+1}, b = -I_{n+1}^{m-1}, gz = -I_{n+1}^m
          a = tget(tab, tp, n + 1, m + 1);
          const double2 bm = tget(tab, tp, n + 1, m - 1);
          b = make_double2(-bm.x, -bm.y);
          const double2 zz = tget(tab, tp, n + 1, m);
          g = make_double2(-zz.x, -zz.y);
        } else {    // regular_gradient: a = R_{n-1}^{m+1}, b = -R_{n-1}^{m-1}, gz = R_{n-1}^m
          a = tget(tab, tp, n - 1, m + 1);
          const double2 bm = tget(tab, tp, n - 1, m - 1);
          b = make_double2(-bm.x, -bm.y);
          g = tget(tab, tp, n - 1, m);
        }
        const double2 hx = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));   // (a + b) / 2
        const double2 hy = make_double2(0.5 * (a.y - b.y), -0.5 * (a.x - b.x));  // (a - b) / 2i
        if (irr) {
          gx += v.x * hx.x + v.y * hx.y;
          gy += v.x * hy.x + v.y * hy.y;
          gz += v.x * g.x + v.y * g.y;
        } else {
          gx += v.x * hx.x - v.y * hx.y;
          gy += v.x * hy.x - v.y * hy.y;
          gz += v.x * g.x - v.y * g.y;
        }
      }
    pot[(size_t)c * N + t] = ph;
    if (want_grad) {
      double* gg = grad + ((size_t)c * N + t) * 3;
      gg[0] = gx;
      gg[1] = gy;
      gg[2] = gz;
    }
  }
}

}  // namespace

void expansion_p2m(const double* rel, int64_t N, const double* q, const double* d, int C, int p,
                   double* coeffs, cudaStream_t s) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
  FMM_REQUIRE(C >= 1 && N >= 0 && (q || d), "p2m needs charges or dipoles");
  const int S = (p + 1) * (p + 1);
  DevBuf<double> drel, dq, dd;
  DevBuf<double2> out(C * S);
  drel.upload(rel, 3 * N, s);
  if (q) dq.upload(q, (size_t)C * N, s);
  if (d) dd.upload(d, (size_t)C * N * 3, s);
  k_exp_p2m<<<grid_for((int64_t)C * S, 128), 128, 0, s>>>(N, C, p, drel.get(), q ? dq.get() : nullptr,
                                                         d ? dd.get() : nullptr, out.get());
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaMemcpyAsync(coeffs, out.get(), (size_t)C * S * sizeof(double2), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
}

void expansion_translate(int kind, const double* dvec, int C, int p, const double* in, double* out,
                         cudaStream_t s) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
  FMM_REQUIRE(kind >= 0 && kind <= 2 && C >= 1, "unknown translation kind");
  if (kind == 1)
    FMM_REQUIRE(dvec[0] != 0.0 || dvec[1] != 0.0 || dvec[2] != 0.0, "M2L offset must be nonzero");
  const int S = (p + 1) * (p + 1);
  const int tp = kind == 1 ? 2 * p : p;
  DevBuf<double2> din, dout(C * S);
  din.upload(reinterpret_cast<const double2*>(in), (size_t)C * S, s);
  const size_t smem = (size_t)(tp + 1) * (tp + 1) * sizeof(double2);
  k_exp_translate<<<C, 256, smem, s>>>(kind, C, p, dvec[0], dvec[1], dvec[2], din.get(), dout.get());
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaMemcpyAsync(out, dout.get(), (size_t)C * S * sizeof(double2), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
}

void expansion_evaluate(int kind, const double* coeffs, int C, int p, const double* rel, int64_t N,
                        bool want_grad, double* pot, double* grad, cudaStream_t s) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
  FMM_REQUIRE(kind == 0 || kind == 1, "unknown evaluation kind");
  const int S = (p + 1) * (p + 1);
  DevBuf<double2> dc;
  DevBuf<double> drel, dpot((size_t)C * std::max<int64_t>(N, 1)), dgrad;
  dc.upload(reinterpret_cast<const double2*>(coeffs), (size_t)C * S, s);
  drel.upload(rel, 3 * N, s);
  if (want_grad) dgrad.resize((size_t)C * std::max<int64_t>(N, 1) * 3);
  if (N > 0) {
    // the per-thread table lives in local memory: small blocks keep the stack footprint low
    k_exp_eval<<<grid_for(N, 64), 64, 0, s>>>(kind, C, p, N, drel.get(), dc.get(), want_grad ? 1 : 0,
                                             dpot.get(), want_grad ? dgrad.get() : nullptr);
    FMM_LAUNCH_CHECK();
    FMM_CUDA(cudaMemcpyAsync(pot, dpot.get(), (size_t)C * N * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (want_grad)
      FMM_CUDA(cudaMemcpyAsync(grad, dgrad.get(), (size_t)C * N * 3 * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
  }
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fmmbem
