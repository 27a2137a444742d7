// P2M as a geometry-only operator applied to the densities.
//
// Reference: FmmPlan._upward leaf part (fmm.py:235-257) with
// harmonics.particle_to_multipole (harmonics.py:221-235):
//   M_leaf = sum_g q_g R(y_g - c) + sum_g d_g . grad R(y_g - c).
// For the BEM system operator the Gauss-point strengths are a fixed
// geometric factor times one entry of x (bemop.py:188-203, 213-216):
//   Laplace 1st kind  q_g = w_g x[panel]          -> B_g = w_g R(y_g - c)
//   Laplace 2nd kind  d_g = w_g x[panel] n_g      -> B_g = w_g (n_g . grad) R(y_g - c)
//   Stokes            q_c = w_g t_c[panel], q_3 = y_g . (w_g t[panel]) -> B_g = w_g R
// so M_leaf,c = sum_g s_c(g) B_g with s read from x.  B (coefficient-major,
// [hidx][sorted source], orders up to p_tab, prefix-compatible in p) is built
// once per operator; every apply is a coalesced streaming reduction over it:
// one warp per (leaf, coefficient), lanes over the leaf's Gauss points,
// shuffle-tree reduction in a fixed order.
#include "operator.cuh"

namespace fmmbem {
namespace {

__global__ void k_basis_build(int64_t ns, int ptab, int kind, const double* __restrict__ px,
                              const double* __restrict__ py, const double* __restrict__ pz,
                              const int* __restrict__ leaf_of_body, const double* __restrict__ cx,
                              const double* __restrict__ cy, const double* __restrict__ cz,
                              const double* __restrict__ s_w, const int* __restrict__ s_panel,
                              const double* __restrict__ nrm, const double* __restrict__ rec,
                              double2* __restrict__ B) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const int leaf = leaf_of_body[i];
  double2 R[hcount(P_MAX)];
  regular_half(px[i] - cx[leaf], py[i] - cy[leaf], pz[i] - cz[leaf], ptab, R, rec);
  const double w = s_w[i];
  const int H = hcount(ptab);
  if (kind != K_LAP_DOUBLE) {
    for (int idx = 0; idx < H; ++idx) B[(size_t)idx * ns + i] = cscale(R[idx], w);
    return;
  }
  const int pn = s_panel[i];
  const double dx = 0.5 * w * nrm[3 * pn], dy = 0.5 * w * nrm[3 * pn + 1], dz = w * nrm[3 * pn + 2];
  for (int n = 0; n <= ptab; ++n)
    for (int m = 0; m <= n; ++m) {
      // 1/2 (dx - i dy) R_{n-1}^{m+1} - 1/2 (dx + i dy) R_{n-1}^{m-1} + dz R_{n-1}^m
      double2 a = make_double2(0.0, 0.0);
      if (n >= 1) {
        if (m + 1 <= n - 1) a = cfma(make_double2(dx, -dy), R[hidx(n - 1, m + 1)], a);
        if (m - 1 >= -(n - 1)) a = cfma(make_double2(-dx, -dy), hget(R, n - 1, m - 1), a);
        if (m <= n - 1) {
          const double2 r = R[hidx(n - 1, m)];
          a.x = fma(dz, r.x, a.x);
          a.y = fma(dz, r.y, a.y);
        }
      }
      B[(size_t)hidx(n, m) * ns + i] = a;
    }
}

// per-Gauss-point channel scalars s_c(g) (sorted source order)
template <int C>
__device__ __forceinline__ void basis_scalars(int kind, int64_t i, const int* s_panel,
                                              const double* x, const double* px, const double* py,
                                              const double* pz, double* s) {
  const int pn = s_panel[i];
  if (C == 1) {
    s[0] = x[pn];
  } else {
    const double t0 = x[3 * pn], t1 = x[3 * pn + 1], t2 = x[3 * pn + 2];
    s[0] = t0;
    s[1] = t1;
    s[2] = t2;
    s[3] = px[i] * t0 + py[i] * t1 + pz[i] * t2;
  }
}

template <int C>
__global__ void __launch_bounds__(256)
k_p2m_basis(const int* __restrict__ leaves, const int* __restrict__ body_start,
            const int* __restrict__ body_count, int64_t ns, int H, int kind,
            const double2* __restrict__ B, const int* __restrict__ s_panel,
            const double* __restrict__ x, const double* __restrict__ px,
            const double* __restrict__ py, const double* __restrict__ pz,
            double2* __restrict__ M) {
  const int leaf = leaves[blockIdx.x];
  const int b0 = body_start[leaf], nb = body_count[leaf];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int idx = warp; idx < H; idx += nw) {
    double2 acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = make_double2(0.0, 0.0);
    const double2* Bi = B + (size_t)idx * ns + b0;
    for (int b = lane; b < nb; b += 32) {
      double s[C == 1 ? 1 : 4];
      basis_scalars<C>(kind, b0 + b, s_panel, x, px, py, pz, s);
      const double2 v = Bi[b];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        acc[c].x = fma(s[c], v.x, acc[c].x);
        acc[c].y = fma(s[c], v.y, acc[c].y);
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      for (int o = 16; o > 0; o >>= 1) {
        acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, o);
        acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, o);
      }
    }
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < C; ++c) M[((size_t)leaf * C + c) * H + idx] = acc[c];
  }
}

// clustered columns (Laplace kinds, one channel), cluster-major Bc[c][h]:
// M_leaf[h] = sum over the leaf's clusters of Bc[c][h] x[panel(c)], one thread per h
__global__ void __launch_bounds__(128)
k_p2m_basis_cl(const int* __restrict__ leaves, const int2* __restrict__ cl_range, int Hp, int H,
               const double2* __restrict__ B, const int* __restrict__ cl_panel,
               const double* __restrict__ x, double2* __restrict__ M) {
  const int leaf = leaves[blockIdx.x];
  const int2 cr = cl_range[leaf];
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int c = cr.x; c < cr.y; ++c) {
      const double s = __ldg(x + __ldg(cl_panel + c));
      const double2 v = __ldg(B + (size_t)c * Hp + h);
      acc.x = fma(s, v.x, acc.x);
      acc.y = fma(s, v.y, acc.y);
    }
    M[(size_t)leaf * H + h] = acc;
  }
}

// Bc[c][h] = sum over the cluster's Gauss points (in sorted order) of B[h][i]
__global__ void k_basis_cluster_sum(int64_t ns, int ncl, int H, const int* __restrict__ cl_src,
                                    const double2* __restrict__ B, double2* __restrict__ Bc) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)ncl * H) return;
  const int h = (int)(gid % H), c = (int)(gid / H);
  double2 a = make_double2(0.0, 0.0);
  for (int i = cl_src[c]; i < cl_src[c + 1]; ++i) a = cadd(a, B[(size_t)h * ns + i]);
  Bc[(size_t)c * H + h] = a;
}

}  // namespace

bool ensure_p2m_basis(BemOp& op, int p, cudaStream_t s) {
  if (op.basis_p >= p) return true;
  const int64_t ns = op.plan.src.n_points;
  // grow to the operator's largest useful order at once (prefix-compatible in p)
  const int ptab = std::max(p, std::min(P_MAX, std::max(op.basis_p, 12)));
  constexpr double BUDGET = 24e9;  // bytes of HBM this table may take
  if ((double)hcount(ptab) * ns * sizeof(double2) > BUDGET) return false;
  const Tree& S = op.plan.src;
  const bool cluster = op.basis_kind_for_sys == K_LAP_SINGLE || op.basis_kind_for_sys == K_LAP_DOUBLE;
  DevBuf<double2> per_source;
  DevBuf<double2>& B = cluster ? per_source : op.p2m_basis;
  B.resize((size_t)hcount(ptab) * ns);
  k_basis_build<<<grid_for(ns, 128), 128, 0, s>>>(ns, ptab, op.basis_kind_for_sys, S.px.get(),
                                                  S.py.get(), S.pz.get(), S.leaf_of_body.get(),
                                                  S.cx.get(), S.cy.get(), S.cz.get(),
                                                  op.s_weight.get(), op.s_panel.get(),
                                                  op.normal.get(), S.rec, B.get());
  FMM_LAUNCH_CHECK();
  op.basis_clustered = cluster;
  op.basis_cols = (int)ns;
  if (cluster) {
    // clusters: maximal runs of sorted Gauss points with the same (leaf, panel)
    const std::vector<int> leaf = S.leaf_of_body.download(s), pan = op.s_panel.download(s);
    std::vector<int> src_begin, cpanel, range(2 * (size_t)S.n_cells, 0);
    for (int64_t i = 0; i < ns; ++i) {
      if (i == 0 || leaf[i] != leaf[i - 1] || pan[i] != pan[i - 1]) {
        if (i == 0 || leaf[i] != leaf[i - 1]) range[2 * (size_t)leaf[i]] = (int)src_begin.size();
        src_begin.push_back((int)i);
        cpanel.push_back(pan[i]);
      }
      range[2 * (size_t)leaf[i] + 1] = (int)src_begin.size();
    }
    const int ncl = (int)cpanel.size();
    src_begin.push_back((int)ns);
    DevBuf<int> d_src;
    d_src.upload(src_begin, s);
    op.cl_panel.upload(cpanel, s);
    op.cl_range.upload(range, s);
    op.p2m_basis.resize((size_t)hcount(ptab) * ncl);
    const int64_t n = (int64_t)ncl * hcount(ptab);
    k_basis_cluster_sum<<<grid_for(n, 256), 256, 0, s>>>(ns, ncl, hcount(ptab), d_src.get(),
                                                          per_source.get(), op.p2m_basis.get());
    FMM_LAUNCH_CHECK();
    op.basis_cols = ncl;
  }
  FMM_CUDA(cudaStreamSynchronize(s));
  op.basis_p = ptab;
  return true;
}

void launch_p2m_basis(BemOp& op, int p, int C, const double* x, double2* M, cudaStream_t s,
                      const int* leaves, int n_leaves) {
  const Tree& S = op.plan.src;
  const int H = hcount(p);
  if (!leaves) {
    leaves = S.leaves.get();
    n_leaves = S.n_leaves;
  }
  if (n_leaves <= 0) return;
  if (op.basis_clustered) {
    FMM_REQUIRE(C == 1, "clustered P2M basis is single-channel");
    k_p2m_basis_cl<<<n_leaves, 128, 0, s>>>(leaves, reinterpret_cast<const int2*>(op.cl_range.get()),
                                             hcount(op.basis_p), H, op.p2m_basis.get(), op.cl_panel.get(),
                                             x, M);
  } else if (C == 1)
    k_p2m_basis<1><<<n_leaves, 256, 0, s>>>(leaves, S.body_start.get(), S.body_count.get(),
                                              S.n_points, H, op.basis_kind_for_sys,
                                              op.p2m_basis.get(), op.s_panel.get(), x, S.px.get(),
                                              S.py.get(), S.pz.get(), M);
  else
    k_p2m_basis<4><<<n_leaves, 256, 0, s>>>(leaves, S.body_start.get(), S.body_count.get(),
                                              S.n_points, H, op.basis_kind_for_sys,
                                              op.p2m_basis.get(), op.s_panel.get(), x, S.px.get(),
                                              S.py.get(), S.pz.get(), M);
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmbem
