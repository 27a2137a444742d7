// M2L by rotation ("point and shoot"): O(p^3) instead of O(p^4) per pair.
//
// The reference's M2L (harmonics.py:180-198, fmm.py:292-314)
//     L_j^k = (-1)^j sum_{n<=p,m} M_n^m conj(I_{n+j}^{m+k}(D))
// is a linear map that commutes with rotations.  With Q the rotation taking
// D to |D| z (Q = R_y(-theta) R_z(-phi)), regular harmonics transform degree
// by degree, R_n^m(Q y) = sum_k A^n_{mk} R_n^k(y), with
//     A^n_{mk} = sqrt((n+k)!(n-k)! / ((n+m)!(n-m)!)) d^n_{mk}(-theta) e^{-ik phi}
// (d = Wigner small-d), so the same truncated operator factors exactly as
//     M' = A M,   L'_j^k = (-1)^j sum_{n>=|k|} M'_n^{-k} (n+j)! / |D|^{n+j+1},
//     L_j^k = e^{-ik phi} sum_l a^j_{lk} L'_j^l          (a = A without the phase)
// because I_N^mu(|D| z) vanishes unless mu = 0.  Per pair and channel this is
// ~7k DFMA at p = 12 instead of ~62k for the dense contraction; parity with
// the reference is exact up to roundoff.
//
// The real matrices a^n (n <= p_tab) of every distinct M2L offset are built
// once at setup from the single-term start values d^{j0}_{mk}, j0 = max(|m|,|k|),
// and the stable three-term recursion in the degree.  One CTA per
// (offset, <= 8 pairs) stages them in shared memory and runs the three stages
// for up to 8 vectors (pairs x channels) at once; results go to the per-pair
// slots that k_m2l_gather adds per target cell in a fixed order.
#include <map>
#include <utility>

#include "kernels.cuh"

namespace fmmbem {

__host__ __device__ __forceinline__ int rot_base(int n) { return n * (4 * n * n - 1) / 3; }
__host__ __device__ __forceinline__ int rot_size(int p) { return rot_base(p + 1); }

namespace {

__device__ double dfact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}

// one thread per (offset, m, k): d^j_{mk}(-theta) for j = max(|m|,|k|) .. P, scaled
__global__ void k_rot_tables(const double* __restrict__ off, int n_off, int P, double* __restrict__ out,
                             double* __restrict__ geo) {
  const int W = 2 * P + 1;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n_off * W * W) return;
  const int u = (int)(gid / (W * W));
  const int mk = (int)(gid % (W * W));
  const int m = mk / W - P, k = mk % W - P;
  const double x = off[3 * u], y = off[3 * u + 1], z = off[3 * u + 2];
  const double r = sqrt(x * x + y * y + z * z);
  const double th = acos(fmin(1.0, fmax(-1.0, z / r)));
  if (mk == 0) {
    geo[3 * u] = r;
    geo[3 * u + 1] = th;
    geo[3 * u + 2] = atan2(y, x);
  }
  const double beta = -th;
  const double c = cos(0.5 * beta), s = sin(0.5 * beta), cb = cos(beta);
  const int j0 = max(abs(m), abs(k));
  double* base = out + (size_t)u * rot_size(P);
  // start value: the single surviving term of Wigner's formula at j = j0
  double d0 = 0.0;
  {
    const int j = j0;
    for (int ss = 0; ss <= 2 * j; ++ss) {
      const int a1 = j + k - ss, a3 = m - k + ss, a4 = j - m - ss;
      if (a1 < 0 || a3 < 0 || a4 < 0) continue;
      const double num = sqrt(dfact(j + k) * dfact(j - k) * dfact(j + m) * dfact(j - m));
      const double den = dfact(a1) * dfact(ss) * dfact(a3) * dfact(a4);
      const double sg = ((m - k + ss) & 1) ? -1.0 : 1.0;
      d0 += sg * num / den * pow(c, 2 * j + k - m - 2 * ss) * pow(s, m - k + 2 * ss);
    }
  }
  double prev2 = 0.0, prev1 = d0;
  for (int j = j0; j <= P; ++j) {
    double cur;
    if (j == j0) {
      cur = d0;
    } else if (j == 1) {  // from j0 = 0 (m = k = 0)
      cur = cb;
    } else {
      const double a = sqrt((double)(j * j - m * m) * (double)(j * j - k * k)) * (j - 1);
      const double b = (2.0 * j - 1.0) * (j * (j - 1.0) * cb - (double)m * k);
      const double cc = j * sqrt((double)((j - 1) * (j - 1) - m * m) * (double)((j - 1) * (j - 1) - k * k));
      cur = (b * prev1 - cc * prev2) / a;
    }
    if (j != j0) {
      prev2 = prev1;
      prev1 = cur;
    }
    const double scale = sqrt(dfact(j + k) * dfact(j - k) / (dfact(j + m) * dfact(j - m)));
    base[rot_base(j) + (m + j) * (2 * j + 1) + (k + j)] = scale * cur;
  }
}

// ---- FP64 tensor-core (DMMA m8n8k4) formulation -------------------------
//
// With the real-field symmetries M_n^{-k} = (-1)^k conj(M_n^k) (also for the
// phased M, M' and L'), each stage splits into two real products of order
// (n+1) x (n+1), one on the real parts and one on the imaginary parts:
//   A:  Re M'_n^m = sum_{k>=0} SA_re[m][k] Re Mf_n^k,   SA_re = a_{m,k} + (-1)^k a_{m,-k} (k>0)
//       Im M'_n^m = sum_{k>=0} SA_im[m][k] Im Mf_n^k,   SA_im = a_{m,k} - (-1)^k a_{m,-k}
//   B:  L'_j^k    = (-1)^(j+k) sum_{n>=k} z_{n+j} conj(M'_n^k)            (Hankel in z)
//   C:  Re L~_j^k = sum_{l>=0} SC_re[k][l] Re L'_j^l,   SC_re = a_{l,k} + (-1)^l a_{-l,k}
//       Im L~_j^k = sum_{l>=0} SC_im[k][l] Im L'_j^l,   L_j^k = e^{-ik phi} L~_j^k
// A warp takes 8 vectors (pairs x channels) of one offset; the vectors are
// the n = 8 columns of mma.sync.m8n8k4.f64, the real matrices SA/SC the row
// operand (pre-swizzled per 8x4 tile into lane order at setup, so a fragment
// is one coalesced 256-byte load), stage B's Hankel operand is formed from z.

__host__ __device__ constexpr int frag_mt(int n) { return (n + 8) >> 3; }
__host__ __device__ constexpr int frag_ks(int n) { return (n + 4) >> 2; }
__host__ __device__ constexpr int aux_stride(int P) { return 4 * P + 4; }
__host__ __device__ constexpr int frag_base(int n) {  // tiles of degrees < n
  int b = 0;
  for (int i = 0; i < n; ++i) b += frag_mt(i) * frag_ks(i);
  return b;
}

// one thread per (offset, table, tile, lane)
__global__ void k_rot_frag(const double* __restrict__ rot, int n_off, int P, int ttot,
                           double* __restrict__ out) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n_off * 4 * ttot * 32) return;
  const int lane = (int)(gid & 31);
  int64_t r = gid >> 5;
  const int t = (int)(r % ttot);
  r /= ttot;
  const int which = (int)(r & 3);
  const int u = (int)(r >> 2);
  int n = 0;
  while (n < P && frag_base(n + 1) <= t) ++n;
  const int lt = t - frag_base(n), ks = frag_ks(n);
  const int row = (lt / ks) * 8 + (lane >> 2), col = (lt % ks) * 4 + (lane & 3);
  double v = 0.0;
  if (row <= n && col <= n) {
    const double* a = rot + (size_t)u * rot_size(P) + rot_base(n) + n * (2 * n + 1) + n;
    const int W = 2 * n + 1;  // a(m, k) = a[m * W + k], m, k in [-n, n]
    if (which < 2) {  // SA: row m, col k
      const int m = row, k = col;
      v = a[m * W + k];
      if (k > 0) v += ((which == 0) == !(k & 1) ? 1.0 : -1.0) * a[m * W - k];
    } else {  // SC: row k, col l
      const int k = row, l = col;
      v = a[l * W + k];
      if (l > 0) v += ((which == 2) == !(l & 1) ? 1.0 : -1.0) * a[-l * W + k];
    }
  }
  out[gid] = v;
}

__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d.x), "+d"(d.y)
               : "d"(a), "d"(b));
}

#ifndef ROT_WARPS_N
#define ROT_WARPS_N 2
#endif
constexpr int ROT_WARPS = ROT_WARPS_N;  // warp units per CTA of the per-warp rotation kernels
constexpr int FRAG_KS_MAX = (P_MAX + 4) / 4;  // k-steps of the largest degree
static_assert((P_MAX + 8) / 8 <= 3, "row tiles per degree");

struct Frag {
  double r[3][FRAG_KS_MAX], i[3][FRAG_KS_MAX];
};

// per offset: e^{-ik phi} (k <= P) and z_N = N! / |D|^(N+1) (N <= 2P)
__global__ void k_rot_aux(const double* __restrict__ geo, int n_off, int P, double* __restrict__ aux) {
  const int stride = aux_stride(P);
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n_off * stride) return;
  const int u = (int)(gid / stride), i = (int)(gid % stride);
  const double r = geo[3 * u], phi = geo[3 * u + 2];
  double v = 0.0;
  if (i < 2 * (P + 1)) {
    double sn, cs;
    sincos(-(double)(i >> 1) * phi, &sn, &cs);
    v = (i & 1) ? sn : cs;
  } else if (i - 2 * (P + 1) <= 2 * P) {
    const int N = i - 2 * (P + 1);
    double f = 1.0, rp = 1.0 / r;
    for (int t = 1; t <= N; ++t) {
      f *= t;
      rp /= r;
    }
    v = f * rp;
  }
  aux[gid] = v;
}

// warp unit = (item, octet of vectors); vector v of an item = (pair v / C, channel v % C).
// Everything is unrolled for the compile-time order P; the next degree's operator
// fragments are loaded while the current degree multiplies.
// CLS: the item's vectors may come from different offsets of one class (same polar-angle
// tables and |D|): the azimuthal phases are read per vector into registers; otherwise the
// item shares one offset and its phases are read once into shared memory.
// One warp unit of the rotation M2L: the three stages for 8 vectors whose offsets share the
// polar-angle tables `tabs` (4 tables, tstride doubles apart) and |D|.  The caller has filled
// the unit's buffers wsh: zz (and ph when !CLS); inputs per lane:
//   !SH: msrc = the multipole of vector fr = lane >> 2 (null: none), read from global memory
//        degree by degree;  SH: the 8 multipoles are already staged in bre / bim ([H][8] planes)
//        and the tables are in shared memory
//   paA  = (CLS) the phases e^{-ik phi} of vector fr's offset
//   dst0/dst1, po0/po1 = the result slots and phases of vectors 2 fc and 2 fc + 1 (fc = lane & 3)
//   after(j) runs once stage C has read degree j's rows of the planes (they are free from then on)
template <int P, bool CLS, bool SH, class After>
__device__ __forceinline__ void
m2l_rot_core(double* __restrict__ wsh, const int lane, const double* __restrict__ tabs, const size_t tstride,
             const double2* __restrict__ msrc, const double2* __restrict__ paA, double2* __restrict__ dst0,
             double2* __restrict__ dst1, const double2* __restrict__ po0, const double2* __restrict__ po1,
             After&& after) {
  constexpr int H = hcount(P);
  double* bre = wsh;                                       // [H][8] real parts
  double* bim = bre + 8 * H;                               // [H][8] imaginary parts
  double2* ph = reinterpret_cast<double2*>(bim + 8 * H);   // [P+1] e^{-ik phi}
  double* zz = reinterpret_cast<double*>(ph + P + 1);      // [2P+1] N! / r^(N+1)
  const int fr = lane >> 2, fc = lane & 3;  // fragment row / column-in-k
  const double* T = tabs + lane;
  auto load = [&](Frag& f, int tab, int n) {
    const int mt = frag_mt(n), ks = frag_ks(n);
    const double* tr = T + (SH ? 0 : tab) * tstride + (size_t)frag_base(n) * 32;
    const double* ti = tr + tstride;
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int t = 0; t < FRAG_KS_MAX; ++t)
        if (q < mt && t < ks) {
          if constexpr (SH) {
            if (tab == 0) {
              f.r[q][t] = tr[(q * ks + t) * 32];
              f.i[q][t] = ti[(q * ks + t) * 32];
            } else {
              // stage C's operators are the transposes of stage A's (SC[k][l] = SA[l][k], from
              // d_{-l,k} = (-1)^(l+k) d_{l,-k}): element (8q + fr, 4t + fc) of the transpose is
              // lane (4 (t & 1) + fc, fr & 3) of SA's tile (row tile t / 2, k-step 2q + fr / 4) --
              // two tiles at the same bank offsets, conflict-free.  Rows past the degree (k-step
              // clamped) only feed result rows that are dropped.
              const int kk = min(2 * q + (lane >> 4), ks - 1);
              const int o = ((t >> 1) * ks + kk) * 32 + (4 * (t & 1) + (lane & 3)) * 4 + ((lane >> 2) & 3) - lane;
              f.r[q][t] = tr[o];
              f.i[q][t] = ti[o];
            }
          } else {
            f.r[q][t] = __ldg(tr + (q * ks + t) * 32);
            f.i[q][t] = __ldg(ti + (q * ks + t) * 32);
          }
        }
  };
  // stage A: Re/Im M'_n^m = SA_re/im[m][k] Re/Im (e^{-ik phi} M_n^k); the B operand
  // (k = 4t + fc, vector fr) comes straight from global memory (or the staged planes), so the
  // degrees are independent and need no synchronisation; next degree's operands are in flight
  // azimuthal phases e^{-ik phi} of each vector's own offset (the item's pairs share the
  // polar-angle tables and |D|, not necessarily phi): stage A's column fr, outputs 2fc, 2fc+1
  double2 phA[CLS ? FRAG_KS_MAX : 1];  // (CLS) e^{-ik phi} of column fr's offset at k = 4t + fc
  if constexpr (CLS) {
#pragma unroll
    for (int t = 0; t < FRAG_KS_MAX; ++t)
      phA[t] = 4 * t + fc <= P ? __ldg(paA + 4 * t + fc) : make_double2(0.0, 0.0);
  }
  __syncwarp();  // ph, zz
  struct BIn {
    double2 m[FRAG_KS_MAX];
  };
  auto load_b = [&](BIn& b, int n) {
    const int ks = frag_ks(n), hb = n * (n + 1) / 2;
#pragma unroll
    for (int t = 0; t < FRAG_KS_MAX; ++t)
      if (t < ks) {
        const int col = t * 4 + fc;
        if constexpr (SH)
          b.m[t] = col <= n ? make_double2(bre[(hb + col) * 8 + fr], bim[(hb + col) * 8 + fr]) : make_double2(0.0, 0.0);
        else
          b.m[t] = (msrc && col <= n) ? __ldg(msrc + hb + col) : make_double2(0.0, 0.0);
      }
  };
  double2 ar[3], ai[3];
  auto mult_a = [&](const Frag& f, const BIn& b, int n) {
    const int mt = frag_mt(n), ks = frag_ks(n);
#pragma unroll
    for (int q = 0; q < 3; ++q) ar[q] = ai[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < FRAG_KS_MAX; ++t)
      if (t < ks) {
        const int col = t * 4 + fc;
        const double2 x = col <= n ? cmul(CLS ? phA[CLS ? t : 0] : ph[col], b.m[t]) : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (q < mt) {
            dmma(ar[q], f.r[q][t], x.x);
            dmma(ai[q], f.i[q][t], x.y);
          }
      }
  };
  {
    Frag cur;
    BIn bc;
    load(cur, 0, 0);
    load_b(bc, 0);
#pragma unroll
    for (int n = 0; n <= P; ++n) {
      Frag nxt;
      BIn bn;
      if (n < P) {
        load(nxt, 0, n + 1);
        load_b(bn, n + 1);
      }
      mult_a(cur, bc, n);
      const int hb = n * (n + 1) / 2;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int m = q * 8 + fr;
        if (q < frag_mt(n) && m <= n) {
          *reinterpret_cast<double2*>(bre + (hb + m) * 8 + 2 * fc) = ar[q];
          *reinterpret_cast<double2*>(bim + (hb + m) * 8 + 2 * fc) = ai[q];
        }
      }
      if (n < P) {
        cur = nxt;
        bc = bn;
      }
    }
  }
  Frag cur;
  load(cur, 2, 0);  // stage C's first degree lands during stage B
  __syncwarp();
  // stage B, two orders per pass: rows j = k..P, reduction over n = k..P, Hankel
  // operand (-1)^(j+k) z_{n+j} (negated for the conjugated imaginary part)
#pragma unroll
  for (int k0 = 0; k0 <= P; k0 += 2) {
    double2 br_[2][3], bi_[2][3];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int k = k0 + w;
#pragma unroll
      for (int q = 0; q < 3; ++q) br_[w][q] = bi_[w][q] = make_double2(0.0, 0.0);
      if (k > P) continue;
      const int L = P + 1 - k, jt = (L + 7) >> 3, ks = (L + 3) >> 2;
#pragma unroll
      for (int t = 0; t < FRAG_KS_MAX; ++t)
        if (t < ks) {
          const int n = k + t * 4 + fc;
          const bool ok = n <= P;
          const int hn = n * (n + 1) / 2 + k;
          const double vr = ok ? bre[hn * 8 + fr] : 0.0;
          const double vi = ok ? bim[hn * 8 + fr] : 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (q < jt) {
              const int j = k + q * 8 + fr;
              double a = (ok && j <= P) ? zz[j + n] : 0.0;
              if ((j + k) & 1) a = -a;
              dmma(br_[w][q], a, vr);
              dmma(bi_[w][q], -a, vi);
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int k = k0 + w;
      if (k > P) continue;
      const int jt = (P + 1 - k + 7) >> 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int j = k + q * 8 + fr;
        if (q < jt && j <= P) {
          const int hj = j * (j + 1) / 2 + k;
          // (SH: stage C runs on the transposed stage-A tables, whose column l = 0 is twice
          // SC's: SC_re[k][0] = a_{0,k} = SA_re[0][k] / 2 -- folded in here)
          if (SH && k == 0) br_[w][q] = make_double2(0.5 * br_[w][q].x, 0.5 * br_[w][q].y);
          *reinterpret_cast<double2*>(bre + hj * 8 + 2 * fc) = br_[w][q];
          *reinterpret_cast<double2*>(bim + hj * 8 + 2 * fc) = bi_[w][q];
        }
      }
    }
    __syncwarp();
  }
  // stage C (tables 2, 3): Re/Im L~_j^k = SC_re/im[k][l] Re/Im L'_j^l
  auto mult = [&](const Frag& f, int n) {
    const int mt = frag_mt(n), ks = frag_ks(n), hb = n * (n + 1) / 2;
#pragma unroll
    for (int q = 0; q < 3; ++q) ar[q] = ai[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < FRAG_KS_MAX; ++t)
      if (t < ks) {
        const int col = t * 4 + fc;
        const double br = col <= n ? bre[(hb + col) * 8 + fr] : 0.0;
        const double bi = col <= n ? bim[(hb + col) * 8 + fr] : 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (q < mt) {
            dmma(ar[q], f.r[q][t], br);
            dmma(ai[q], f.i[q][t], bi);
          }
      }
  };
  // stage C and the output phase; lane owns vectors 2 fc and 2 fc + 1
  double2* dst[2] = {dst0, dst1};
  double2 phO[2][CLS ? 3 : 1];  // (CLS) e^{-ik phi} of output vector 2 fc + w at k = 8 q + fr
  if constexpr (CLS) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      phO[0][q] = 8 * q + fr <= P ? __ldg(po0 + 8 * q + fr) : make_double2(0.0, 0.0);
      phO[1][q] = 8 * q + fr <= P ? __ldg(po1 + 8 * q + fr) : make_double2(0.0, 0.0);
    }
  }
#pragma unroll
  for (int j = 0; j <= P; ++j) {
    Frag nxt;
    if (j < P) load(nxt, 2, j + 1);
    mult(cur, j);
    after(j);
    const int hb = j * (j + 1) / 2;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int k = q * 8 + fr;
      if (q < frag_mt(j) && k <= j) {
        const double2 e0 = CLS ? phO[0][CLS ? q : 0] : ph[k], e1 = CLS ? phO[1][CLS ? q : 0] : ph[k];
        double2 o0 = make_double2(ar[q].x, ai[q].x), o1 = make_double2(ar[q].y, ai[q].y);
        if (SH && k == 0) {
          // transposed tables: SC_re[0][l] = 2 SA_re[l][0] (l > 0; the l = 0 half is folded into
          // stage B), SC_im[0][l] = 0 (the order-0 coefficients of a real field are real)
          o0 = make_double2(2.0 * o0.x, 0.0);
          o1 = make_double2(2.0 * o1.x, 0.0);
        }
        if (dst[0]) dst[0][hb + k] = cmul(e0, o0);
        if (dst[1]) dst[1][hb + k] = cmul(e1, o1);
      }
    }
    if (j < P) cur = nxt;
  }
}

// v1: one warp unit per warp, two units per CTA, the tables read from L2 by every warp
// (also the offset-grouped mode, CLS = false: one offset and one phase table per item)
template <int P, bool CLS>
__global__ void __launch_bounds__(ROT_WARPS * 32)
k_m2l_rot(const int4* __restrict__ items, int n_items, const int* __restrict__ gpair,
          const int* __restrict__ pair_src, const int* __restrict__ pair_off, const double* __restrict__ frag,
          const int* __restrict__ dir, int ttot,
          const double* __restrict__ aux, int aux_p, const double2* __restrict__ M, int C,
          double2* __restrict__ pout) {
  constexpr int H = hcount(P);
  constexpr int WS = 16 * H + 4 * P + 4;
  extern __shared__ double sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * ROT_WARPS + warp;
  const int item = unit / C, oct = unit % C;
  if (item >= n_items) return;
  const int4 it = items[item];
  const int nvec = (it.z - it.y) * C, v0 = oct * 8;
  if (v0 >= nvec) return;
  double* wsh = sh + (size_t)warp * WS;
  double* sp = wsh + 16 * H;      // [P+1] e^{-ik phi} as (re, im)
  double* zz = sp + 2 * (P + 1);  // [2P+1] N! / r^(N+1)
  const int u = it.x, astr = aux_stride(aux_p);
  {
    const double* A = aux + (size_t)u * astr;
#pragma unroll
    for (int i = lane; i < 2 * (P + 1); i += 32) sp[i] = A[i];
#pragma unroll
    for (int i = lane; i <= 2 * P; i += 32) zz[i] = A[2 * (aux_p + 1) + i];
  }
  const int fr = lane >> 2, fc = lane & 3;
  const double2* msrc = nullptr;
  int uo = u;
  {
    const int vg = v0 + fr;
    if (vg < nvec) {
      const int pr = gpair[it.y + vg / C];
      msrc = M + ((size_t)pair_src[pr] * C + vg % C) * H;
      uo = pair_off[pr];
    }
  }
  double2* dst[2];
  const double2* po[2];
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const int vg = v0 + 2 * fc + w;
    const int pr = vg < nvec ? gpair[it.y + vg / C] : 0;
    dst[w] = vg < nvec ? pout + ((size_t)pr * C + vg % C) * H : nullptr;
    po[w] = reinterpret_cast<const double2*>(aux + (size_t)((CLS && vg < nvec) ? pair_off[pr] : u) * astr);
  }
  m2l_rot_core<P, CLS, false>(wsh, lane, frag + (size_t)dir[u] * 4 * ttot * 32, (size_t)ttot * 32, msrc,
                              reinterpret_cast<const double2*>(aux + (size_t)uo * astr), dst[0], dst[1], po[0],
                              po[1], [](int) {});
}

// ---- v2: the direction's tables staged once per CTA by bulk async copies (TMA) --------------
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "MBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBW_%=;\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (16-byte aligned, a multiple of 16 bytes), completion on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}

constexpr int ROT2_GROUP = 24;  // items per CTA group (divisible by every ROT2 warp count)
__host__ __device__ constexpr size_t rot2_tab_doubles(int P) { return (size_t)2 * frag_base(P + 1) * 32; }
__host__ __device__ constexpr size_t rot2_ws_doubles(int P) { return (size_t)16 * hcount(P) + 4 * P + 4; }
__host__ __device__ constexpr size_t rot2_smem(int P, int W) {
  return (rot2_tab_doubles(P) + (size_t)W * rot2_ws_doubles(P)) * sizeof(double) + 16;
}
// warps per CTA: the most of {12, 8, 6, 4, 3, 2, 1} whose buffers fit beside the tables; low
// orders take 8 (several CTAs per SM)
__host__ __device__ constexpr int rot2_warps(int P) {
  constexpr int cand[7] = {12, 8, 6, 4, 3, 2, 1};
  if (P <= 10) return 8;
  for (int i = 0; i < 7; ++i)
    if (rot2_smem(P, cand[i]) <= (size_t)227 * 1024) return cand[i];
  return 1;
}

// group = (direction table, first item, end item) of class-grouped items whose offsets share one
// polar angle; the CTA's warps take the items' warp units (item x channel octet) round robin.
// vecs[8 item + a] = (pair slot, source cell, offset id, 0) of the item's a-th pair (slot -1:
// none): one independent load per unit (fetched one unit ahead), then all the unit's multipoles
// are read in one burst into the stage planes -- no dependent global loads inside the stages.
template <int P, int W, bool ASYNC>
__global__ void __launch_bounds__(W * 32)
k_m2l_rot2(const int4* __restrict__ groups, const int4* __restrict__ vecs, const double* __restrict__ frag,
           int ttot, const double* __restrict__ aux, int aux_p, const double2* __restrict__ M, int C,
           double2* __restrict__ pout) {
  constexpr int H = hcount(P);
  constexpr int NT = frag_base(P + 1);  // tiles per table up to degree P
  constexpr size_t WS = rot2_ws_doubles(P);
  extern __shared__ __align__(128) double sh[];
  double* tabs = sh;                                 // [2][NT * 32]: SA_re, SA_im (stage C reads them transposed)
  double* wbuf = sh + rot2_tab_doubles(P);           // [W][WS]
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(wbuf + (size_t)W * WS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 g = groups[blockIdx.x];
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, 2u * NT * 32u * (unsigned)sizeof(double));
    const double* src = frag + (size_t)g.x * 4 * ttot * 32;
#pragma unroll
    for (int t = 0; t < 2; ++t)
      bulk_g2s(tabs + (size_t)t * NT * 32, src + (size_t)t * ttot * 32, NT * 32u * (unsigned)sizeof(double), bar);
  }
  __syncthreads();  // the barrier is initialised before anyone polls it
  double* wsh = wbuf + (size_t)warp * WS;
  double* bre = wsh;
  double* bim = wsh + 8 * H;
  double* zz = wsh + 16 * H + 2 * (P + 1);
  const int astr = aux_stride(aux_p);
  const int va = lane & 7, fr = lane >> 2, fc = lane & 3;
  // lane's vector in the load role: va of the unit's octet
  auto fetch = [&](int unit) -> int4 {  // x = -2: no such unit
    if (unit >= g.z * C) return make_int4(-2, 0, 0, 0);
    const int vg = (unit % C) * 8 + va;  // vector of the item = (pair vg / C, channel vg % C)
    int4 e = __ldg(vecs + (size_t)(unit / C) * 8 + vg / C);
    e.w = vg % C;
    return e;
  };
  // degree j of a unit's 8 multipoles into the planes, asynchronously: lane's vector va,
  // coefficients i = hb + (lane >> 3) + 4 r; a missing vector's rows are zero-filled.  Each
  // 16-byte coefficient goes as two 8-byte copies (the planes split real and imaginary parts).
  auto prefetch = [&](const int4& rec, int j) {
    if (rec.x == -2) return;  // no such unit
    const double2* mv = M + ((size_t)rec.y * C + rec.w) * H;
    const unsigned sz = rec.x >= 0 ? 8u : 0u;
    const int hb = j * (j + 1) / 2;
    for (int i = hb + (lane >> 3); i <= hb + j; i += 4) {
      const double* s = reinterpret_cast<const double*>(mv + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(bre + i * 8 + va)),
                   "l"(s), "r"(sz)
                   : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(bim + i * 8 + va)),
                   "l"(s + 1), "r"(sz)
                   : "memory");
    }
  };
  // !ASYNC: the unit's multipoles in one burst of 16-byte loads (all in flight together), then
  // stored into the planes
  auto burst = [&](const int4& rec) {
    const double2* mv = rec.x >= 0 ? M + ((size_t)rec.y * C + rec.w) * H : nullptr;
    constexpr int NL = (H + 3) / 4, B = 10;
#pragma unroll
    for (int j0 = 0; j0 < NL; j0 += B) {
      double2 v[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int i = (lane >> 3) + 4 * (j0 + j);
        v[j] = (mv && j0 + j < NL && i < H) ? __ldg(mv + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const int i = (lane >> 3) + 4 * (j0 + j);
        if (j0 + j < NL && i < H) {
          bre[i * 8 + va] = v[j].x;
          bim[i * 8 + va] = v[j].y;
        }
      }
    }
  };
  int unit = g.y * C + warp;
  int4 cur = fetch(unit);
  if (ASYNC && cur.x != -2) {
#pragma unroll
    for (int j = 0; j <= P; ++j) prefetch(cur, j);
  }
  bool first = true;
  for (; unit < g.z * C; unit += W) {
    int4 nxt = fetch(unit + W);
    if (__shfl_sync(0xffffffffu, nxt.x, 0) == -1) nxt.x = -2;  // an octet past the item's vectors: skipped
    if (__shfl_sync(0xffffffffu, cur.x, 0) < 0) {  // a skipped octet: burst-load the one after it
      cur = nxt;
      if (ASYNC && cur.x != -2) {
#pragma unroll
        for (int j = 0; j <= P; ++j) prefetch(cur, j);
      }
      continue;
    }
    // the unit's |D| factors, from any member offset (the octet's first vector exists)
    const int u0 = __shfl_sync(0xffffffffu, cur.z, 0);
    {
      const double* A = aux + (size_t)u0 * astr + 2 * (aux_p + 1);
#pragma unroll
      for (int i = lane; i <= 2 * P; i += 32) zz[i] = A[i];
    }
    if constexpr (!ASYNC) burst(cur);
    // roles of the stages: column fr (stage A), outputs 2 fc and 2 fc + 1 (stage C)
    const int offA = __shfl_sync(0xffffffffu, cur.z, fr);
    int prO[2], offO[2], chO[2];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      prO[w] = __shfl_sync(0xffffffffu, cur.x, 2 * fc + w);
      offO[w] = __shfl_sync(0xffffffffu, cur.z, 2 * fc + w);
      chO[w] = __shfl_sync(0xffffffffu, cur.w, 2 * fc + w);
    }
    double2* d0 = prO[0] >= 0 ? pout + ((size_t)prO[0] * C + chO[0]) * H : nullptr;
    double2* d1 = prO[1] >= 0 ? pout + ((size_t)prO[1] * C + chO[1]) * H : nullptr;
    if (first) {
      mbar_wait(bar, 0);  // the tables have landed
      first = false;
    }
    if constexpr (ASYNC) asm volatile("cp.async.wait_all;" ::: "memory");  // this unit's multipoles are in the planes
    __syncwarp();
    // (ASYNC) the next unit's multipoles follow stage C through the planes, degree by degree
    m2l_rot_core<P, true, true>(wsh, lane, tabs, (size_t)NT * 32, nullptr,
                                reinterpret_cast<const double2*>(aux + (size_t)offA * astr), d0, d1,
                                reinterpret_cast<const double2*>(aux + (size_t)offO[0] * astr),
                                reinterpret_cast<const double2*>(aux + (size_t)offO[1] * astr),
                                [&](int j) {
                                  if constexpr (ASYNC) prefetch(nxt, j);
                                });
    __syncwarp();  // the planes are free again
    cur = nxt;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int P>
void launch_rot_p(const Plan& plan, const int4* gitems, const int* gpair, int n_items, int C,
                  const double2* M, double2* pout, cudaStream_t st, bool cls, const int4* groups, int n_groups,
                  const int4* vecs) {
  constexpr int H = hcount(P);
  // the shared-table kernel is opt-in (FMMBEM_M2L_SHARED=1; 1a = with the cp.async multipole
  // prefetch): both kernels are bound by the LSU data pipe (operand wavefronts per DMMA: 83 % of
  // its peak in ncu), not by L2 or latency, and the per-warp kernel measured as fast or faster
  // (cfg5 p = 14 apply 2.461 vs 2.474 / 2.503 ms, cfg2 5 829 vs 5 739 / 5 658 mat-vecs/s)
  const char* sel = std::getenv("FMMBEM_M2L_SHARED");
  if (cls && groups && vecs && n_groups > 0 && sel && sel[0] == '1') {
    constexpr int W = rot2_warps(P);
    constexpr size_t smem2 = rot2_smem(P, W);
    static DeviceOnce attr2;
    if (attr2.first()) {
      FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot2<P, W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot2<P, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      attr2.mark();
    }
    auto kern2 = sel[1] == 'a' ? k_m2l_rot2<P, W, true> : k_m2l_rot2<P, W, false>;  // "1a": cp.async prefetch
    kern2<<<(unsigned)n_groups, W * 32, smem2, st>>>(
        groups, vecs, plan.rotf.get(), frag_base(plan.rot_p + 1), plan.rot_aux.get(), plan.rot_p, M, C, pout);
    FMM_LAUNCH_CHECK();
    return;
  }
  const size_t smem = (size_t)ROT_WARPS * (16 * H + 4 * P + 4) * sizeof(double);
  static DeviceOnce attr;
  if (attr.first()) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    // FMMBEM_M2L_CARVEOUT=percent: shared-memory share of the SM for this kernel (fewer resident
    // CTAs, more L1 for the table fragments); default: the driver's choice
    if (const char* e = std::getenv("FMMBEM_M2L_CARVEOUT")) {
      FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot<P, false>, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e)));
      FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot<P, true>, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e)));
    }
    attr.mark();
  }
  const int64_t units = (int64_t)n_items * C;
  auto kern = cls ? k_m2l_rot<P, true> : k_m2l_rot<P, false>;
  kern<<<(unsigned)((units + ROT_WARPS - 1) / ROT_WARPS), ROT_WARPS * 32, smem, st>>>(
      gitems, n_items, gpair, plan.m2l_src.get(), plan.m2l_off.get(), plan.rotf.get(), plan.rot_dir.get(),
      frag_base(plan.rot_p + 1),
      plan.rot_aux.get(), plan.rot_p, M, C, pout);
  FMM_LAUNCH_CHECK();
}

template <int... Ps>
void launch_rot_dispatch(std::integer_sequence<int, Ps...>, int p, const Plan& plan,
                         const int4* gitems, const int* gpair, int n_items, int C,
                         const double2* M, double2* pout, cudaStream_t st, bool cls, const int4* groups,
                         int n_groups, const int4* vecs) {
  bool done = false;
  ((p == Ps + M2L_ROT_MIN_P && !done
        ? (launch_rot_p<Ps + M2L_ROT_MIN_P>(plan, gitems, gpair, n_items, C, M, pout, st, cls, groups, n_groups,
                                            vecs),
           done = true)
        : false),
   ...);
  FMM_REQUIRE(done, "rotation M2L order out of range");
}


// ---- M2M by rotation --------------------------------------------------------------------
// The reference's M2M (harmonics.py:156-177, fmm.py:268-290)
//     M'_n^m = sum_{j<=n, k} M_j^k R_{n-j}^{m-k}(d),   d = c_child - c_parent
// factors like the M2L: rotate d onto +z (A = a E, the same tables), translate along z, where
// R_l^mu(|d| z) = |d|^l / l! delta_{mu 0} leaves, per order k, the lower-triangular Toeplitz
//     M''_n^k = sum_{j=k..n} |d|^{n-j} / (n-j)! M'_j^k,
// and rotate back with A^{-1} = E^{-1} a~, a~_{mk} = (-1)^{m-k} a_{mk} (the Wigner small-d
// symmetry d_{km} = (-1)^{k-m} d_{mk}).  In the real split a~ is a with a checkerboard sign, so
// the back rotation reuses the stage-A fragments with (-1)^k on the input, (-1)^m on the output
// and the phase e^{+im phi}.  M2M is exact in the reference too, so this agrees with the dense
// operator to roundoff.
// per rtab id: e^{-ik phi} (k <= P) and t_l = |d|^l / l! (l <= P)
__global__ void k_m2m_aux(const double* __restrict__ geo, int n_off, int P, double* __restrict__ aux) {
  const int stride = aux_stride(P);
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)n_off * stride) return;
  const int u = (int)(gid / stride), i = (int)(gid % stride);
  const double r = geo[3 * u], phi = geo[3 * u + 2];
  double v = 0.0;
  if (i < 2 * (P + 1)) {
    double sn, cs;
    sincos(-(double)(i >> 1) * phi, &sn, &cs);
    v = (i & 1) ? sn : cs;
  } else if (i - 2 * (P + 1) <= P) {
    const int l = i - 2 * (P + 1);
    double f = 1.0;
    for (int t = 1; t <= l; ++t) f *= r / t;
    v = f;
  }
  aux[gid] = v;
}

// warp unit = (item, octet of vectors); vector v of an item = (child v / C, channel v % C);
// the item's children share one rtab id (level, octant): one direction, phase and |d|.
// LOCAL = false: M2M (above), the child's multipole -> its contribution to the parent's,
//                written to the child's slot of cout (k_children_sum adds them in order).
// LOCAL = true:  L2L, the parent's local expansion -> ADDED to the child's (harmonics.py:
//   175-176): rotate the local with (A^{-1})^T = a~^T E^{+} (SC tables, checkerboard sign,
//   input phase e^{+ik phi}), translate along z with the upper-triangular Toeplitz
//   L''_n^k = sum_{j>=n} |d|^{j-n}/(j-n)! L'_j^k, and rotate back with A^T = E a^T (the M2L's
//   stage C).
// The M2M instance is bounded to 128 registers per thread (8 CTAs of 64 threads per SM; 24-32
// bytes of spills at the high orders, 254 registers uncapped): its levels run beside the
// persistent near field, which leaves 16 K registers per SM -- two M2M CTAs instead of one, and
// the chain ends under the near field instead of after it.  The L2L instance runs after the
// near field and keeps the whole register file.
#ifndef VROT_M2M_MIN_BLOCKS
#define VROT_M2M_MIN_BLOCKS 8
#endif
template <int P, bool LOCAL>
__global__ void __launch_bounds__(ROT_WARPS * 32, LOCAL ? 1 : VROT_M2M_MIN_BLOCKS)
k_vrot(const int4* __restrict__ items, int n_items, const int* __restrict__ child,
       const int* __restrict__ parent, const double* __restrict__ frag, const int* __restrict__ dir,
       int ttot, const double* __restrict__ aux, int aux_p, const double2* __restrict__ in, int C,
       double2* __restrict__ out) {
  constexpr int H = hcount(P);
  constexpr int WS = 16 * H + 4 * P + 4;
  constexpr int TAB_IN = LOCAL ? 2 : 0;   // fragments of the first rotation
  constexpr int TAB_OUT = LOCAL ? 2 : 0;  // and of the back rotation
  extern __shared__ double sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * ROT_WARPS + warp;
  const int item = unit / C, oct = unit % C;
  if (item >= n_items) return;
  const int4 it = items[item];
  const int nvec = (it.z - it.y) * C, v0 = oct * 8;
  if (v0 >= nvec) return;
  double* bre = sh + (size_t)warp * WS;                    // [H][8] real parts
  double* bim = bre + 8 * H;                               // [H][8] imaginary parts
  double2* ph = reinterpret_cast<double2*>(bim + 8 * H);   // [P+1] e^{-ik phi}
  double* tt = reinterpret_cast<double*>(ph + P + 1);      // [P+1] |d|^l / l!
  const int u = it.x;
  {
    const double* A = aux + (size_t)u * aux_stride(aux_p);
    double* sp = reinterpret_cast<double*>(ph);
#pragma unroll
    for (int i = lane; i < 2 * (P + 1); i += 32) sp[i] = A[i];
#pragma unroll
    for (int i = lane; i <= P; i += 32) tt[i] = A[2 * (aux_p + 1) + i];
  }
  const int fr = lane >> 2, fc = lane & 3;
  const double* T = frag + (size_t)dir[u] * 4 * ttot * 32 + lane;
  auto load = [&](Frag& f, int tab, int n) {
    const int mt = frag_mt(n), ks = frag_ks(n);
    const double* tr = T + (size_t)(tab * ttot + frag_base(n)) * 32;
    const double* ti = tr + (size_t)ttot * 32;
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int t = 0; t < FRAG_KS_MAX; ++t)
        if (q < mt && t < ks) {
          f.r[q][t] = __ldg(tr + (q * ks + t) * 32);
          f.i[q][t] = __ldg(ti + (q * ks + t) * 32);
        }
  };
  const double2* vsrc = nullptr;
  {
    const int vg = v0 + fr;
    if (vg < nvec) {
      const int c = child[it.y + vg / C];
      vsrc = in + ((size_t)(LOCAL ? parent[c] : c) * C + vg % C) * H;
    }
  }
  __syncwarp();  // ph, tt
  double2 ar[3], ai[3];
  // stage 1: first rotation, degree by degree
  {
    Frag cur;
    double2 bc[FRAG_KS_MAX];
    auto load_b = [&](double2* b, int n) {
      const int ks = frag_ks(n), hb = n * (n + 1) / 2;
#pragma unroll
      for (int t = 0; t < FRAG_KS_MAX; ++t)
        if (t < ks) {
          const int col = t * 4 + fc;
          b[t] = (vsrc && col <= n) ? __ldg(vsrc + hb + col) : make_double2(0.0, 0.0);
        }
    };
    load(cur, TAB_IN, 0);
    load_b(bc, 0);
#pragma unroll
    for (int n = 0; n <= P; ++n) {
      Frag nxt;
      double2 bn[FRAG_KS_MAX];
      if (n < P) {
        load(nxt, TAB_IN, n + 1);
        load_b(bn, n + 1);
      }
      const int mt = frag_mt(n), ks = frag_ks(n);
#pragma unroll
      for (int q = 0; q < 3; ++q) ar[q] = ai[q] = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < FRAG_KS_MAX; ++t)
        if (t < ks) {
          const int col = t * 4 + fc;
          double2 x = make_double2(0.0, 0.0);
          if (col <= n) {
            // M2M: e^{-ik phi} M; L2L: (-1)^k e^{+ik phi} L
            x = LOCAL ? cmul(cconj(ph[col]), bc[t]) : cmul(ph[col], bc[t]);
            if (LOCAL && (col & 1)) x = make_double2(-x.x, -x.y);
          }
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (q < mt) {
              dmma(ar[q], cur.r[q][t], x.x);
              dmma(ai[q], cur.i[q][t], x.y);
            }
        }
      const int hb = n * (n + 1) / 2;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int m = q * 8 + fr;
        if (q < mt && m <= n) {
          double2 r = ar[q], i = ai[q];
          if (LOCAL && (m & 1)) {  // output checkerboard sign of a~^T
            r = make_double2(-r.x, -r.y);
            i = make_double2(-i.x, -i.y);
          }
          *reinterpret_cast<double2*>(bre + (hb + m) * 8 + 2 * fc) = r;
          *reinterpret_cast<double2*>(bim + (hb + m) * 8 + 2 * fc) = i;
        }
      }
      if (n < P) {
        cur = nxt;
#pragma unroll
        for (int t = 0; t < FRAG_KS_MAX; ++t) bc[t] = bn[t];
      }
    }
  }
  Frag cur;
  load(cur, TAB_OUT, 0);  // the back rotation's first degree lands during stage 2
  __syncwarp();
  // stage 2: z translation per order k, rows n = k..P (output degree), columns j (input degree):
  // M2M lower-triangular t_{n-j} (j <= n), L2L upper-triangular t_{j-n} (j >= n)
#pragma unroll
  for (int k0 = 0; k0 <= P; k0 += 2) {
    double2 br_[2][3], bi_[2][3];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int k = k0 + w;
#pragma unroll
      for (int q = 0; q < 3; ++q) br_[w][q] = bi_[w][q] = make_double2(0.0, 0.0);
      if (k > P) continue;
      const int L = P + 1 - k, jt = (L + 7) >> 3, ks = (L + 3) >> 2;
#pragma unroll
      for (int t = 0; t < FRAG_KS_MAX; ++t)
        if (t < ks) {
          const int j = k + t * 4 + fc;
          const bool ok = j <= P;
          const int hn = j * (j + 1) / 2 + k;
          const double vr = ok ? bre[hn * 8 + fr] : 0.0;
          const double vi = ok ? bim[hn * 8 + fr] : 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (q < jt) {
              const int n = k + q * 8 + fr;
              double a = 0.0;
              if (ok && n <= P) {
                if (LOCAL) a = j >= n ? tt[j - n] : 0.0;
                else a = j <= n ? tt[n - j] : 0.0;
              }
              dmma(br_[w][q], a, vr);
              dmma(bi_[w][q], a, vi);
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int k = k0 + w;
      if (k > P) continue;
      const int jt = (P + 1 - k + 7) >> 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int n = k + q * 8 + fr;
        if (q < jt && n <= P) {
          const int hj = n * (n + 1) / 2 + k;
          *reinterpret_cast<double2*>(bre + hj * 8 + 2 * fc) = br_[w][q];
          *reinterpret_cast<double2*>(bim + hj * 8 + 2 * fc) = bi_[w][q];
        }
      }
    }
    __syncwarp();
  }
  // stage 3: back rotation; lane owns vectors v0 + 2 fc and v0 + 2 fc + 1
  // M2M: (-1)^m e^{+im phi} (SA with (-1)^k on the input), written to the child's slot;
  // L2L: e^{-ik phi} (SC), added to the child's local expansion
  double2* dst[2];
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const int vg = v0 + 2 * fc + w;
    dst[w] = vg < nvec ? out + ((size_t)child[it.y + vg / C] * C + vg % C) * H : nullptr;
  }
#pragma unroll
  for (int n = 0; n <= P; ++n) {
    Frag nxt;
    if (n < P) load(nxt, TAB_OUT, n + 1);
    const int mt = frag_mt(n), ks = frag_ks(n), hb = n * (n + 1) / 2;
#pragma unroll
    for (int q = 0; q < 3; ++q) ar[q] = ai[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int t = 0; t < FRAG_KS_MAX; ++t)
      if (t < ks) {
        const int col = t * 4 + fc;
        const double sg = (!LOCAL && (col & 1)) ? -1.0 : 1.0;
        const double br = col <= n ? sg * bre[(hb + col) * 8 + fr] : 0.0;
        const double bi = col <= n ? sg * bim[(hb + col) * 8 + fr] : 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (q < mt) {
            dmma(ar[q], cur.r[q][t], br);
            dmma(ai[q], cur.i[q][t], bi);
          }
      }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int m = q * 8 + fr;
      if (q < mt && m <= n) {
        if (LOCAL) {
          const double2 e = ph[m];
          if (dst[0]) dst[0][hb + m] = cadd(dst[0][hb + m], cmul(e, make_double2(ar[q].x, ai[q].x)));
          if (dst[1]) dst[1][hb + m] = cadd(dst[1][hb + m], cmul(e, make_double2(ar[q].y, ai[q].y)));
        } else {
          const double2 e = cconj(ph[m]);
          const double sg = (m & 1) ? -1.0 : 1.0;
          if (dst[0]) dst[0][hb + m] = cscale(cmul(e, make_double2(ar[q].x, ai[q].x)), sg);
          if (dst[1]) dst[1][hb + m] = cscale(cmul(e, make_double2(ar[q].y, ai[q].y)), sg);
        }
      }
    }
    if (n < P) cur = nxt;
  }
}

struct VrotTabs {  // one tree's rotation tables (Plan::m2m_* or Plan::l2l_*)
  const int4* items;
  const int* child;
  const int* parent;
  const double* frag;
  const int* dir;
  const double* aux;
  int p;
};

template <int P, bool LOCAL>
void launch_vrot_p(const VrotTabs& t, int ia, int n_items, int C, const double2* in, double2* out,
                   cudaStream_t st) {
  constexpr int H = hcount(P);
  const size_t smem = (size_t)ROT_WARPS * (16 * H + 4 * P + 4) * sizeof(double);
  static DeviceOnce attr;
  if (attr.first()) {
    FMM_CUDA(cudaFuncSetAttribute(k_vrot<P, LOCAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr.mark();
  }
  const int64_t units = (int64_t)n_items * C;
  k_vrot<P, LOCAL><<<(unsigned)((units + ROT_WARPS - 1) / ROT_WARPS), ROT_WARPS * 32, smem, st>>>(
      t.items + ia, n_items, t.child, t.parent, t.frag, t.dir, frag_base(t.p + 1), t.aux, t.p, in, C, out);
  FMM_LAUNCH_CHECK();
}

template <bool LOCAL, int... Ps>
void launch_vrot_dispatch(std::integer_sequence<int, Ps...>, int p, const VrotTabs& t, int ia,
                          int n_items, int C, const double2* in, double2* out, cudaStream_t st) {
  bool done = false;
  ((p == Ps + M2L_ROT_MIN_P && !done
        ? (launch_vrot_p<Ps + M2L_ROT_MIN_P, LOCAL>(t, ia, n_items, C, in, out, st), done = true)
        : false),
   ...);
  FMM_REQUIRE(done, "rotation M2M/L2L order out of range");
}

}  // namespace

void compute_rot_tables(const double* d_off, int n_off, int P, double* out, double* geo,
                        cudaStream_t s) {
  const int W = 2 * P + 1;
  const int64_t n = (int64_t)n_off * W * W;
  if (n) k_rot_tables<<<grid_for(n, 128), 128, 0, s>>>(d_off, n_off, P, out, geo);
  FMM_LAUNCH_CHECK();
}

size_t rot_table_size(int P) { return (size_t)rot_size(P); }

size_t rot_frag_size(int P) { return (size_t)4 * frag_base(P + 1) * 32; }

void build_rot_frag(const double* rot, int n_off, int P, double* out, cudaStream_t s) {
  const int ttot = frag_base(P + 1);
  const int64_t n = (int64_t)n_off * 4 * ttot * 32;
  if (n) k_rot_frag<<<grid_for(n, 256), 256, 0, s>>>(rot, n_off, P, ttot, out);
  FMM_LAUNCH_CHECK();
}

void build_rot_aux(const double* geo, int n_off, int P, double* aux, cudaStream_t s) {
  const int64_t n = (int64_t)n_off * aux_stride(P);
  if (n) k_rot_aux<<<grid_for(n, 128), 128, 0, s>>>(geo, n_off, P, aux);
  FMM_LAUNCH_CHECK();
}

void launch_m2l_rot(const Plan& plan, const int4* gitems, const int* gpair, int n_items, int p,
                    int C, const double2* M, double2* pout, cudaStream_t st, bool cls, const RotGroups* rg) {
  if (n_items <= 0) return;
  FMM_REQUIRE(p <= plan.rot_p, "rotation tables not prepared for this order");
  launch_rot_dispatch(std::make_integer_sequence<int, P_MAX - M2L_ROT_MIN_P + 1>{}, p, plan, gitems,
                      gpair, n_items, C, M, pout, st, cls, rg ? rg->groups.get() : nullptr, rg ? rg->n_groups : 0,
                      rg ? rg->vecs.get() : nullptr);
}

// CTA groups of the shared-table rotation M2L: consecutive class-grouped items of one direction
// table, <= ROT2_GROUP items each, cut evenly; and the items' pairs as (slot, source cell,
// offset id, 0) records, 8 per item
void RotGroups::build(const std::vector<int4>& items, const std::vector<int>& cpair, const std::vector<int>& pair_src,
                      const std::vector<int>& pair_off, const std::vector<int>& dir_of_off, cudaStream_t s) {
  std::vector<int4> g, v(std::max<size_t>(items.size(), 1) * 8, make_int4(-1, 0, 0, 0));
  for (size_t i = 0; i < items.size();) {
    size_t j = i;
    const int d = dir_of_off[items[i].x];
    while (j < items.size() && dir_of_off[items[j].x] == d) ++j;
    const int64_t u0 = (int64_t)i, len = (int64_t)(j - i), nch = (len + ROT2_GROUP - 1) / ROT2_GROUP;
    for (int64_t q = 0; q < nch; ++q)
      g.push_back(make_int4(d, (int)(u0 + len * q / nch), (int)(u0 + len * (q + 1) / nch), 0));
    i = j;
  }
  for (size_t i = 0; i < items.size(); ++i) {
    FMM_REQUIRE(items[i].z - items[i].y <= 8 && items[i].z > items[i].y, "rotation M2L item size");
    for (int k = items[i].y; k < items[i].z; ++k) {
      const int pr = cpair[k];
      v[i * 8 + (k - items[i].y)] = make_int4(pr, pair_src[pr], pair_off[pr], 0);
    }
  }
  n_groups = (int)g.size();
  groups.upload(g.empty() ? std::vector<int4>(1) : g, s);
  vecs.upload(v, s);
}

namespace {

// per rtab id (level * 8 + octant) of one tree: d = c_child - c_parent = (+-h, +-h, +-h),
// h = the child level's half width; fragments per distinct polar angle, (phase, |d|^l/l!) rows
void build_vrot_tables(const Tree& tr, int p, DevBuf<double>& frag_out, DevBuf<int>& dir_out,
                       DevBuf<double>& aux_out, cudaStream_t s) {
  const int nl = std::max(tr.n_levels, 1), n_off = nl * 8;
  std::vector<double> off(3 * (size_t)n_off);
  for (int l = 0; l < nl; ++l)
    for (int o = 0; o < 8; ++o) {
      const double h = l < (int)tr.level_half.size() ? tr.level_half[l] : 1.0;
      double* d = &off[3 * (size_t)(l * 8 + o)];
      d[0] = (o & 1) ? h : -h;
      d[1] = (o & 2) ? h : -h;
      d[2] = (o & 4) ? h : -h;
    }
  std::map<double, int> dirs;
  std::vector<int> dir(n_off);
  std::vector<double> rep;
  for (int u = 0; u < n_off; ++u) {
    const double x = off[3 * u], y = off[3 * u + 1], z = off[3 * u + 2];
    const double key = z / std::sqrt(x * x + y * y + z * z);
    auto it = dirs.find(key);
    if (it == dirs.end()) {
      it = dirs.emplace(key, (int)dirs.size()).first;
      rep.insert(rep.end(), {x, y, z});
    }
    dir[u] = it->second;
  }
  const int nd = (int)dirs.size();
  DevBuf<double> d_rep, d_off, geo_rep, geo, one, rot;
  d_rep.upload(rep, s);
  d_off.upload(off, s);
  dir_out.upload(dir, s);
  rot.resize((size_t)nd * rot_size(p));
  geo_rep.resize((size_t)nd * 3);
  compute_rot_tables(d_rep.get(), nd, p, rot.get(), geo_rep.get(), s);
  geo.resize((size_t)n_off * 3);
  one.resize((size_t)n_off);
  compute_rot_tables(d_off.get(), n_off, 0, one.get(), geo.get(), s);
  frag_out.resize((size_t)nd * rot_frag_size(p));
  build_rot_frag(rot.get(), nd, p, frag_out.get(), s);
  aux_out.resize((size_t)n_off * rot_aux_size(p));
  const int64_t n = (int64_t)n_off * aux_stride(p);
  k_m2m_aux<<<grid_for(n, 128), 128, 0, s>>>(geo.get(), n_off, p, aux_out.get());
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void plan_ensure_m2m_rot(Plan& plan, int p, cudaStream_t s) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p out of range [0, 20]");
  if (plan.m2m_rot_p >= p) return;
  build_vrot_tables(plan.src, p, plan.m2m_rotf, plan.m2m_dir, plan.m2m_aux, s);
  build_vrot_tables(plan.tgt, p, plan.l2l_rotf, plan.l2l_dir, plan.l2l_aux, s);
  plan.m2m_rot_p = p;
}

void launch_m2m_rot(const Plan& plan, int p, int C, double2* M, double2* cout, cudaStream_t st) {
  FMM_REQUIRE(p >= M2L_ROT_MIN_P && p <= plan.m2m_rot_p, "rotation M2M tables not prepared");
  const int CH = C * hcount(p);
  const VrotTabs t{plan.d_m2m_ritems.get(), plan.m2m_rchild.get(), plan.src.parent.get(),
                   plan.m2m_rotf.get(), plan.m2m_dir.get(), plan.m2m_aux.get(), plan.m2m_rot_p};
  for (int l = (int)plan.m2m_level_off.size() - 2; l >= 0; --l) {
    const int np = plan.m2m_level_off[l + 1] - plan.m2m_level_off[l];
    if (np <= 0) continue;
    const int ia = plan.m2m_ritem_off[l], ib = plan.m2m_ritem_off[l + 1];
    if (ib > ia)
      launch_vrot_dispatch<false>(std::make_integer_sequence<int, P_MAX - M2L_ROT_MIN_P + 1>{}, p, t,
                                  ia, ib - ia, C, M, cout, st);
    launch_children_sum(plan, l, CH, cout, M, st);
  }
}

void launch_l2l_rot(const Plan& plan, int p, int C, double2* L, cudaStream_t st, int l0, int l1) {
  FMM_REQUIRE(p >= M2L_ROT_MIN_P && p <= plan.m2m_rot_p, "rotation L2L tables not prepared");
  const VrotTabs t{plan.d_l2l_ritems.get(), plan.l2l_rchild.get(), plan.tgt.parent.get(),
                   plan.l2l_rotf.get(), plan.l2l_dir.get(), plan.l2l_aux.get(), plan.m2m_rot_p};
  for (int l = std::max(l0, 0); l + 1 < (int)plan.l2l_ritem_off.size() && l < l1; ++l) {  // top-down
    const int ia = plan.l2l_ritem_off[l], ib = plan.l2l_ritem_off[l + 1];
    if (ib > ia)
      launch_vrot_dispatch<true>(std::make_integer_sequence<int, P_MAX - M2L_ROT_MIN_P + 1>{}, p, t,
                                 ia, ib - ia, C, L, L, st);
  }
}
}  // namespace fmmbem
