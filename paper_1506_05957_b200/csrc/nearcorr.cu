// Near-singular / singular correction assembly on device (setup, p-independent).
//
// Reference: BemOperator._find_near_pairs (bemop.py:95-101), _pair_rule_sums
// (bemop.py:104-125), _correction_matrix (bemop.py:127-184) and the Hess-Smith
// polar singular integrals (quadrature.py:175-247).
//
//   near pairs : (target i, source panel j) with |c_i - c_j| <= near_factor * sqrt(2 S_j)
//                (cKDTree.query_ball_point, inclusive) - here a uniform grid whose
//                cell edge is the largest cutoff, so the 27 neighbouring cells hold
//                every candidate; distances use the same unfused arithmetic.
//   value      : fine(19-pt) - coarse(4-pt, centroid point dropped by the d2>0 mask)
//   self pairs : + singular - fine for the even kernels, - fine for the odd ones.
// Output is CSR by target panel with columns ascending; Stokes kernels store
// one 3x3 block per pair (row-major), i.e. block-CSR.
#include <cub/cub.cuh>

#include "operator.cuh"

namespace fmmbem {
namespace {

constexpr double FOUR_PI = 12.566370614359172;  // 4.0 * np.pi

__global__ void k_cutoffs(int64_t P, const double* area, double factor, double* cut) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < P) cut[j] = __dmul_rn(factor, sqrt(__dmul_rn(2.0, area[j])));
}

struct Grid {
  double lo[3];
  double h;
  int dim[3];
};

__device__ __forceinline__ int cell_coord(double v, double lo, double h, int dim) {
  int c = (int)floor((v - lo) / h);
  return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__global__ void k_grid_keys(int64_t P, const double* cen, Grid g, int* key, int* idx) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= P) return;
  const int a = cell_coord(cen[3 * j], g.lo[0], g.h, g.dim[0]);
  const int b = cell_coord(cen[3 * j + 1], g.lo[1], g.h, g.dim[1]);
  const int c = cell_coord(cen[3 * j + 2], g.lo[2], g.h, g.dim[2]);
  key[j] = (c * g.dim[1] + b) * g.dim[0] + a;
  idx[j] = (int)j;
}

__global__ void k_cell_ranges(int64_t P, const int* skey, int* cstart, int* cend) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int k = skey[i];
  if (i == 0 || skey[i - 1] != k) cstart[k] = (int)i;
  if (i == P - 1 || skey[i + 1] != k) cend[k] = (int)i + 1;
}

// pass 0: count; pass 1: fill (then each row is sorted by column)
template <bool FILL>
__global__ void k_near(int64_t P, const double* cen, const double* cut, Grid g, const int* sidx,
                       const int* cstart, const int* cend, int* count, const int* rowptr,
                       int* cols) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  const double x = cen[3 * i], y = cen[3 * i + 1], z = cen[3 * i + 2];
  const int a = cell_coord(x, g.lo[0], g.h, g.dim[0]);
  const int b = cell_coord(y, g.lo[1], g.h, g.dim[1]);
  const int c = cell_coord(z, g.lo[2], g.h, g.dim[2]);
  int n = 0;
  const int base = FILL ? rowptr[i] : 0;
  for (int dc = -1; dc <= 1; ++dc) {
    const int cc = c + dc;
    if (cc < 0 || cc >= g.dim[2]) continue;
    for (int db = -1; db <= 1; ++db) {
      const int bb = b + db;
      if (bb < 0 || bb >= g.dim[1]) continue;
      for (int da = -1; da <= 1; ++da) {
        const int aa = a + da;
        if (aa < 0 || aa >= g.dim[0]) continue;
        const int k = (cc * g.dim[1] + bb) * g.dim[0] + aa;
        for (int e = cstart[k]; e < cend[k]; ++e) {
          const int j = sidx[e];
          const double dx = __dadd_rn(x, -cen[3 * j]);
          const double dy = __dadd_rn(y, -cen[3 * j + 1]);
          const double dz = __dadd_rn(z, -cen[3 * j + 2]);
          const double d2 =
              __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
          const double r = cut[j];
          if (d2 <= __dmul_rn(r, r)) {
            if (FILL) cols[base + n] = j;
            ++n;
          }
        }
      }
    }
  }
  if (!FILL) {
    count[i] = n;
  } else {
    int* row = cols + base;
    for (int u = 1; u < n; ++u) {  // insertion sort: rows hold a few dozen entries
      const int v = row[u];
      int w = u - 1;
      while (w >= 0 && row[w] > v) { row[w + 1] = row[w]; --w; }
      row[w + 1] = v;
    }
  }
}

// Sum of kernel x rule over one source panel seen from target x (bemop.py:104-125)
template <int KIND>
__device__ void rule_sum(double x, double y, double z, const double* pts, const double* wts, int K,
                         const double* nrm, double* out) {
  double s = 0.0;
  double o[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = 0; k < K; ++k) {
    const double rx = x - pts[3 * k], ry = y - pts[3 * k + 1], rz = z - pts[3 * k + 2];
    const double d2 = rx * rx + ry * ry + rz * rz;
    const double inv = d2 > 0.0 ? 1.0 / sqrt(d2) : 0.0;
    const double w = wts[k];
    if (KIND == 0) {  // Laplace single
      s += w * inv;
    } else if (KIND == 1) {  // Laplace double
      const double rn = rx * nrm[0] + ry * nrm[1] + rz * nrm[2];
      s += w * rn * inv * inv * inv;
    } else {
      const double r[3] = {rx, ry, rz};
      double f;
      if (KIND == 2) {  // stokeslet: I sum w/r + sum w r r^T / r^3
        s += w * inv;
        f = w * inv * inv * inv;
      } else {  // stresslet: 6 sum w (r.n) r r^T / r^5
        const double rn = rx * nrm[0] + ry * nrm[1] + rz * nrm[2];
        const double i2 = inv * inv;
        f = 6.0 * w * rn * i2 * i2 * inv;
      }
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) o[3 * a + b] += f * r[a] * r[b];
    }
  }
  if (KIND <= 1) {
    out[0] = s / FOUR_PI;
  } else {
    for (int a = 0; a < 9; ++a) out[a] = o[a];
    if (KIND == 2) { out[0] += s; out[4] += s; out[8] += s; }
  }
}

// Hess-Smith polar integral about the centroid (quadrature.py:175-247).
// Returns the scalar Laplace value (already / 4 pi) or the 3x3 stokeslet block.
template <int KIND>
__device__ void singular_integral(const double* v, const double* gx, const double* gw, int ng,
                                  double* out) {
  // panel_geometry centroid (mean) and normal
  double cen[3], e1[3], e2[3], nrm[3], uv[3][2];
  for (int d = 0; d < 3; ++d) cen[d] = (v[d] + v[3 + d] + v[6 + d]) / 3.0;
  const double a1[3] = {v[3] - v[0], v[4] - v[1], v[5] - v[2]};
  const double a2[3] = {v[6] - v[0], v[7] - v[1], v[8] - v[2]};
  double cr[3] = {a1[1] * a2[2] - a1[2] * a2[1], a1[2] * a2[0] - a1[0] * a2[2],
                  a1[0] * a2[1] - a1[1] * a2[0]};
  double cn = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
  for (int d = 0; d < 3; ++d) nrm[d] = cr[d] / cn;
  const double en = a1[0] * nrm[0] + a1[1] * nrm[1] + a1[2] * nrm[2];
  for (int d = 0; d < 3; ++d) e1[d] = a1[d] - en * nrm[d];
  const double e1n = sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
  for (int d = 0; d < 3; ++d) e1[d] /= e1n;
  e2[0] = nrm[1] * e1[2] - nrm[2] * e1[1];
  e2[1] = nrm[2] * e1[0] - nrm[0] * e1[2];
  e2[2] = nrm[0] * e1[1] - nrm[1] * e1[0];
  for (int k = 0; k < 3; ++k) {
    const double r[3] = {v[3 * k] - cen[0], v[3 * k + 1] - cen[1], v[3 * k + 2] - cen[2]};
    uv[k][0] = r[0] * e1[0] + r[1] * e1[1] + r[2] * e1[2];
    uv[k][1] = r[0] * e2[0] + r[1] * e2[1] + r[2] * e2[2];
  }
  double scalar = 0.0, b00 = 0.0, b01 = 0.0, b11 = 0.0;
  for (int i = 0; i < 3; ++i) {
    const double* a = uv[i];
    const double* b = uv[(i + 1) % 3];
    const double ta = atan2(a[1], a[0]);
    double tb = atan2(b[1], b[0]);
    if (tb <= ta) tb += 2.0 * 3.141592653589793;
    double ne0 = b[1] - a[1], ne1 = -(b[0] - a[0]);
    const double nl = sqrt(ne0 * ne0 + ne1 * ne1);
    ne0 /= nl;
    ne1 /= nl;
    double de = ne0 * a[0] + ne1 * a[1];
    if (de < 0.0) { ne0 = -ne0; ne1 = -ne1; de = -de; }
    const double half_span = 0.5 * (tb - ta), mid = 0.5 * (tb + ta);
    for (int k = 0; k < ng; ++k) {
      const double phi = half_span * gx[k] + mid;
      const double wphi = half_span * gw[k];
      double sn, cs;
      sincos(phi, &sn, &cs);
      const double R = de / (cs * ne0 + sn * ne1);
      scalar += wphi * R;
      if (KIND == 2) {
        b00 += wphi * (R * cs * cs);
        b01 += wphi * (R * cs * sn);
        b11 += wphi * (R * sn * sn);
      }
    }
  }
  if (KIND == 0) {
    out[0] = scalar / FOUR_PI;
    return;
  }
  // frame rows (e1, e2, n); result = F^T local F
  const double F[3][3] = {{e1[0], e1[1], e1[2]}, {e2[0], e2[1], e2[2]}, {nrm[0], nrm[1], nrm[2]}};
  const double loc[3][3] = {{scalar + b00, b01, 0.0}, {b01, scalar + b11, 0.0}, {0.0, 0.0, scalar}};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) acc += F[k][a] * loc[k][l] * F[l][b];
      out[3 * a + b] = acc;
    }
}

template <int KIND>
__global__ void k_corr_values(int64_t P, const int* rowptr, const int* cols, const double* cen,
                              const double* gpos, const double* gw, const double* fpos,
                              const double* fw, const double* nrm, const double* pverts,
                              const double* lgx, const double* lgw, int ng, double* vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P) return;
  constexpr int NV = KIND <= 1 ? 1 : 9;
  const double x = cen[3 * i], y = cen[3 * i + 1], z = cen[3 * i + 2];
  for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
    const int j = cols[e];
    double coarse[9], fine[9], d[9];
    rule_sum<KIND>(x, y, z, gpos + 12 * (int64_t)j, gw + 4 * (int64_t)j, 4, nrm + 3 * (int64_t)j, coarse);
    rule_sum<KIND>(x, y, z, fpos + 57 * (int64_t)j, fw + 19 * (int64_t)j, 19, nrm + 3 * (int64_t)j, fine);
    for (int a = 0; a < NV; ++a) d[a] = fine[a] - coarse[a];
    if (j == i) {
      if (KIND == 0 || KIND == 2) {
        double sg[9];
        singular_integral<KIND>(pverts + 9 * (int64_t)j, lgx, lgw, ng, sg);
        for (int a = 0; a < NV; ++a) d[a] += sg[a];
      }
      for (int a = 0; a < NV; ++a) d[a] -= fine[a];
    }
    for (int a = 0; a < NV; ++a) vals[(int64_t)e * NV + a] = d[a];
  }
}

}  // namespace

void build_near_pairs(BemOp& op, cudaStream_t s) {
  const int64_t P = op.n_panels;
  const int B = 256;
  DevBuf<double> cut(P);
  k_cutoffs<<<grid_for(P, B), B, 0, s>>>(P, op.area.get(), op.near_factor, cut.get());
  FMM_LAUNCH_CHECK();
  const std::vector<double> hcut = cut.download(s);
  const std::vector<double> hcen = op.centroid.download(s);
  Grid g;
  double hi[3];
  for (int d = 0; d < 3; ++d) { g.lo[d] = hcen[d]; hi[d] = hcen[d]; }
  for (int64_t j = 0; j < P; ++j)
    for (int d = 0; d < 3; ++d) {
      g.lo[d] = std::min(g.lo[d], hcen[3 * j + d]);
      hi[d] = std::max(hi[d], hcen[3 * j + d]);
    }
  double hmax = 0.0;
  for (double c : hcut) hmax = std::max(hmax, c);
  g.h = hmax > 0.0 ? hmax : 1.0;
  while (true) {
    int64_t tot = 1;
    for (int d = 0; d < 3; ++d) {
      g.dim[d] = (int)std::floor((hi[d] - g.lo[d]) / g.h) + 1;
      tot *= g.dim[d];
    }
    if (tot <= (int64_t)1 << 24) break;
    g.h *= 2.0;  // still >= every cutoff, so 27 neighbours stay sufficient
  }
  const int ncell = g.dim[0] * g.dim[1] * g.dim[2];
  DevBuf<int> key(P), idx(P), skey(P), sidx(P), cstart(ncell), cend(ncell);
  k_grid_keys<<<grid_for(P, B), B, 0, s>>>(P, op.centroid.get(), g, key.get(), idx.get());
  {
    size_t bytes = 0;
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.get(), skey.get(), idx.get(),
                                             sidx.get(), (int)P, 0, 32, s));
    DevBuf<unsigned char> tmp(bytes ? bytes : 1);
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, key.get(), skey.get(), idx.get(),
                                             sidx.get(), (int)P, 0, 32, s));
  }
  cstart.zero(s);
  cend.zero(s);
  k_cell_ranges<<<grid_for(P, B), B, 0, s>>>(P, skey.get(), cstart.get(), cend.get());
  DevBuf<int> count(P + 1);
  count.zero(s);
  k_near<false><<<grid_for(P, B), B, 0, s>>>(P, op.centroid.get(), cut.get(), g, sidx.get(),
                                             cstart.get(), cend.get(), count.get(), nullptr, nullptr);
  FMM_LAUNCH_CHECK();
  op.near_rowptr.resize(P + 1);
  {
    size_t bytes = 0;
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, count.get(), op.near_rowptr.get(),
                                           (int)(P + 1), s));
    DevBuf<unsigned char> tmp(bytes ? bytes : 1);
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, count.get(), op.near_rowptr.get(),
                                           (int)(P + 1), s));
  }
  int nnz = 0;
  FMM_CUDA(cudaMemcpyAsync(&nnz, op.near_rowptr.get() + P, sizeof(int), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  op.near_nnz = nnz;
  op.near_cols.resize(std::max(nnz, 1));
  k_near<true><<<grid_for(P, B), B, 0, s>>>(P, op.centroid.get(), cut.get(), g, sidx.get(),
                                            cstart.get(), cend.get(), nullptr,
                                            op.near_rowptr.get(), op.near_cols.get());
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaStreamSynchronize(s));
}

void build_correction(BemOp& op, int kind, Correction& out, cudaStream_t s) {
  const int64_t P = op.n_panels;
  const int B = 128;
  out.kind = kind;
  out.block = kind <= 1 ? 1 : 9;
  out.vals.resize((size_t)std::max(op.near_nnz, 1) * out.block);
#define CORR_CASE(K)                                                                           \
  case K:                                                                                      \
    k_corr_values<K><<<grid_for(P, B), B, 0, s>>>(                                             \
        P, op.near_rowptr.get(), op.near_cols.get(), op.centroid.get(), op.gauss_pos.get(),    \
        op.gauss_w.get(), op.fine_pos.get(), op.fine_w.get(), op.normal.get(),                 \
        op.panel_verts.get(), op.leg_x.get(), op.leg_w.get(), op.n_gauss_singular,             \
        out.vals.get());                                                                       \
    break;
  switch (kind) {
    CORR_CASE(0)
    CORR_CASE(1)
    CORR_CASE(2)
    CORR_CASE(3)
    default: throw ArgumentError("unknown correction kernel");
  }
#undef CORR_CASE
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fmmbem
