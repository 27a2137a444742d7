// BemOperator.apply / dense_apply / assemble_rhs on device.
//
// Reference: BemOperator._layer_apply (bemop.py:192-232), _apply (280-288),
// assemble_rhs (290-310), _gauss_density (188-190), the Stokes channel maps
// (fmm.py:422-453).  One layer application is
//
//   density gather  ->  [stream B]  P2P items ------------------------------+
//                   ->  [stream A]  P2M -> M2M -> M2L -> L2L --------------+-> epilogue
//
// and the epilogue fuses L2P (+ gradients), the sum of the P2P item
// partials, the near/singular correction SpMV, the Stokes/stresslet
// recombination, the 1/(4 pi) or 1/(8 pi mu) factors and the 0.5 x term.
// apply(x, p) is captured once per p into a CUDA graph and replayed.
#include "operator.cuh"
#include "l2p.cuh"

namespace fmmbem {

void upload_index_tables();

void upload_l2p_constants() {
  static DeviceOnce done;
  if (!done.first()) return;
  static L2PConst h;
  h.diag[0] = 1.0;
  for (int m = 1; m <= P_MAX; ++m) h.diag[m] = h.diag[m - 1] * (-1.0 / (2.0 * m));
  for (int n = 0; n <= P_MAX; ++n)
    for (int m = 0; m <= P_MAX; ++m) {
      const double d = (double)(n + m) * (double)(n - m);
      h.ra[n * (P_MAX + 1) + m] = (n >= m + 2) ? (2.0 * n - 1.0) / d : 0.0;
      h.rb[n * (P_MAX + 1) + m] = (n >= m + 2) ? 1.0 / d : 0.0;
    }
  FMM_CUDA(cudaMemcpyToSymbol(c_l2p, &h, sizeof(h)));
  done.mark();
}

namespace {

constexpr double FOUR_PI = 12.566370614359172;

__global__ void k_sorted_sources(int64_t ns, const int* perm, const double* gw, double* s_w,
                                 int* s_panel, const int* tgt_perm_inv, int* self_src) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const int o = perm[i];
  s_w[i] = gw[o];
  s_panel[i] = o / 4;  // 4 far-rule points per panel, panel-major (bemop.py:68-70)
  // Gauss point 0 of panel j is bitwise its collocation point (bemop.py:64-67)
  if (o % 4 == 0) self_src[tgt_perm_inv[o / 4]] = (int)i;
}

// double-layer near-field source records (x, y), (z, w n_x), (w n_y, w n_z), sorted order
__global__ void k_source_records(int64_t ns, const double* px, const double* py, const double* pz,
                                 const double* s_w, const int* s_panel, const double* nrm, double2* srec) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const double w = s_w[i];
  const int pn = s_panel[i];
  srec[3 * i] = make_double2(px[i], py[i]);
  srec[3 * i + 1] = make_double2(pz[i], w * nrm[3 * pn]);
  srec[3 * i + 2] = make_double2(w * nrm[3 * pn + 1], w * nrm[3 * pn + 2]);
}

__global__ void k_row_ranges(int64_t n, const int* perm, const int* rowptr, int2* rows) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) rows[i] = make_int2(rowptr[perm[i]], rowptr[perm[i] + 1]);
}

__global__ void k_invert_perm(int64_t n, const int* perm, int* inv) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = (int)i;
}

// Gauss-point densities w_g * x[panel(g)] in sorted source order (bemop.py:188-190)
template <int KIND>
__global__ void k_density(int64_t ns, const double* __restrict__ s_w, const int* __restrict__ s_panel,
                          const double* __restrict__ px, const double* __restrict__ py,
                          const double* __restrict__ pz, const double* __restrict__ nrm,
                          const double* __restrict__ x, double* q, double* dip, double* wsrc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const int pn = s_panel[i];
  const double w = s_w[i];
  if (KIND == K_LAP_SINGLE) {
    q[i] = w * x[pn];
  } else if (KIND == K_LAP_DOUBLE) {
    const double v = w * x[pn];
    const double d0 = v * nrm[3 * pn], d1 = v * nrm[3 * pn + 1], d2 = v * nrm[3 * pn + 2];
    dip[3 * i] = d0;
    dip[3 * i + 1] = d1;
    dip[3 * i + 2] = d2;
  } else {
    const double f0 = w * x[3 * pn], f1 = w * x[3 * pn + 1], f2 = w * x[3 * pn + 2];
    const double yf = px[i] * f0 + py[i] * f1 + pz[i] * f2;
    if (KIND == K_STOKESLET) {
      // channels (f_x, f_y, f_z, y.f) (fmm.py:422-425)
      q[i] = f0;
      q[ns + i] = f1;
      q[2 * ns + i] = f2;
      q[3 * ns + i] = yf;
      wsrc[3 * i] = f0;
      wsrc[3 * i + 1] = f1;
      wsrc[3 * i + 2] = f2;
    } else {
      // seven dipole channels Phi_c = f_c n, Lambda_c = n_c f, Psi = (y.f) n (fmm.py:436-445)
      const double n0 = nrm[3 * pn], n1 = nrm[3 * pn + 1], n2 = nrm[3 * pn + 2];
      const double f[3] = {f0, f1, f2}, nn[3] = {n0, n1, n2};
      for (int c = 0; c < 3; ++c)
        for (int k = 0; k < 3; ++k) {
          dip[(c * ns + i) * 3 + k] = f[c] * nn[k];
          dip[((3 + c) * ns + i) * 3 + k] = nn[c] * f[k];
        }
      for (int k = 0; k < 3; ++k) dip[(6 * ns + i) * 3 + k] = yf * nn[k];
      for (int k = 0; k < 3; ++k) {
        wsrc[6 * i + k] = f[k];
        wsrc[6 * i + 3 + k] = nn[k];
      }
    }
  }
}

template <int KIND> struct EpiTraits;
template <> struct EpiTraits<K_LAP_SINGLE> { static constexpr int C = 1, NC = 1; static constexpr bool GRAD = false; };
template <> struct EpiTraits<K_LAP_DOUBLE> { static constexpr int C = 1, NC = 1; static constexpr bool GRAD = false; };
template <> struct EpiTraits<K_STOKESLET> { static constexpr int C = 4, NC = 3; static constexpr bool GRAD = true; };
template <> struct EpiTraits<K_STRESSLET> { static constexpr int C = 7, NC = 3; static constexpr bool GRAD = true; };

struct EpiArgs {
  const int* leaves;
  const int* item_begin;
  const P2PItem* items;
  const double* part;
  const double2* L;
  const int* path_off;  // per target cell: the cells whose local expansions reach its targets
  const int* path;
  int max_path;
  int p;
  const int* rowptr;
  const int2* rows;  // per sorted target: [start, end) of its correction row (no perm lookup)
  const int* cols;
  const double* vals;
  const double* x;
  double alpha, beta;
  double* y;
  double* ysorted;  // sharded: write (target body - tbody_a) * NC + c instead of y[panel]
  int tbody_a;
  // 0 = whole layer; 1 = near part only (near-field partials + correction,
  // y = alpha x + beta (near / 4 pi + corr)); 2 = far part only, added: y += beta pot / 4 pi
  int mode = 0;
};

// NS threads per target (NS > 1 for the one-channel kinds): slice k takes the
// L2P columns m = k mod NS, every NS-th near-field item and correction entry;
// the slices' partials are added in slice order.
template <int KIND> constexpr int epi_slices() { return EpiTraits<KIND>::C == 1 ? 4 : 1; }
constexpr int EPI_TGT = 128;  // targets per CTA (blockIdx.y: the leaf's target tile)

template <int KIND, bool FAR>
__global__ void __launch_bounds__(EPI_TGT * epi_slices<KIND>()) k_epilogue(TreeDev T, EpiArgs a) {
  using Tr = EpiTraits<KIND>;
  constexpr int C = Tr::C, NC = Tr::NC, NS = epi_slices<KIND>();
  extern __shared__ double2 sL[];  // [path cell][C][H], then the slice partials
  const int li = blockIdx.x;
  const int leaf = a.leaves[li];
  const int H = hcount(a.p);
  const int pb = FAR ? a.path_off[leaf] : 0, np = FAR ? a.path_off[leaf + 1] - pb : 0;
  double* red = reinterpret_cast<double*>(sL + (FAR ? (size_t)a.max_path * C * H : 0));  // [NS][EPI_TGT][2]
  const int t0 = T.body_start[leaf], nt = T.body_count[leaf];
  const int ib = a.item_begin[li], ie = a.item_begin[li + 1];
  const int tl = threadIdx.x % EPI_TGT, slice = threadIdx.x / EPI_TGT;
  if ((int)blockIdx.y * EPI_TGT >= nt) return;  // (uniform over the CTA, before any barrier)
  // every path cell's local expansion (the leaf, then its ancestors with M2L terms) and its
  // centre, staged once (the L2P loop below then touches no global memory)
  __shared__ double s_cc[3 * 24];
  pdl_wait();  // L (the M2L gather) and the partials are complete past this point
  for (int i = threadIdx.x; i < np * C * H; i += blockDim.x) {
    const int k = i / (C * H), r = i - k * (C * H);
    sL[i] = a.L[(size_t)a.path[pb + k] * C * H + r];
  }
  if (FAR && threadIdx.x < np) {
    const int cell = a.path[pb + threadIdx.x];
    s_cc[3 * threadIdx.x] = T.cx[cell];
    s_cc[3 * threadIdx.x + 1] = T.cy[cell];
    s_cc[3 * threadIdx.x + 2] = T.cz[cell];
  }
  {
    const int base = blockIdx.y * EPI_TGT;
    const int lt = base + tl;
    const bool valid = lt < nt;
    const int ti = t0 + (valid ? lt : 0);
    const int pn = T.perm[ti];
    const double tx = T.px[ti], ty = T.py[ti], tz = T.pz[ti];
    // near-field partials and the correction row first: their loads overlap the L2P below
    double near[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) near[c] = 0.0;
    // a leaf's items are consecutive with out_off advancing by nt (plan_make_items)
    const int oo = ib < ie ? a.items[ib].out_off : 0;
    const bool near_part = a.mode != 2;
    if (valid && near_part)
      for (int it = ib + slice; it < ie; it += NS) {
        const double* pp = a.part + (size_t)(oo + (it - ib) * nt + lt) * NC;
#pragma unroll
        for (int c = 0; c < NC; ++c) near[c] += pp[c];
      }
    double corr1 = 0.0;
    if ((KIND == K_LAP_SINGLE || KIND == K_LAP_DOUBLE) && valid && near_part) {
      const int2 rr = a.rows[ti];
#pragma unroll 4
      for (int e = rr.x + slice; e < rr.y; e += NS) corr1 = fma(a.vals[e], a.x[a.cols[e]], corr1);
    }
    double pot[C], grad[3 * C];
#pragma unroll
    for (int c = 0; c < C; ++c) { pot[c] = 0.0; grad[3 * c] = grad[3 * c + 1] = grad[3 * c + 2] = 0.0; }
    if (FAR) {
      __syncthreads();  // (first pass: the staged expansions)
      if (valid)
        for (int k = 0; k < np; ++k) {
          const double dx = tx - s_cc[3 * k], dy = ty - s_cc[3 * k + 1], dz = tz - s_cc[3 * k + 2];
          if (C == 1)
            pot[0] += l2p_eval1(sL + (size_t)k * H, a.p, dx, dy, dz, slice);
          else
            l2p_eval<C, Tr::GRAD>(sL + (size_t)k * C * H, H, a.p, dx, dy, dz, pot, grad, T.rec, slice, NS);
        }
    }
    if (KIND == K_LAP_SINGLE || KIND == K_LAP_DOUBLE) {
      double corr = corr1;
      double far_near = pot[0] + near[0];
      if (NS > 1) {
        red[(slice * EPI_TGT + tl) * 2] = far_near;
        red[(slice * EPI_TGT + tl) * 2 + 1] = corr;
        __syncthreads();
        if (slice == 0)
          for (int k = 1; k < NS; ++k) {
            far_near += red[(k * EPI_TGT + tl) * 2];
            corr += red[(k * EPI_TGT + tl) * 2 + 1];
          }
        __syncthreads();
      }
      if (slice == 0 && valid) {
        double* yy = a.ysorted ? a.ysorted + (ti - a.tbody_a) : a.y + pn;
        if (a.mode == 2) {
          *yy += a.beta * (far_near / FOUR_PI);
        } else {
          const double layer = far_near / FOUR_PI + corr;
          *yy = a.alpha * a.x[pn] + a.beta * layer;
        }
      }
    } else if (valid) {
      const double xt[3] = {tx, ty, tz};
      double u[3];
      for (int i = 0; i < 3; ++i) {
        if (KIND == K_STOKESLET) {
          // u_i = phi_i - x_c d_i phi_c + d_i psi (fmm.py:428-433)
          double v = pot[i];
          for (int c = 0; c < 3; ++c) v -= xt[c] * grad[3 * c + i];
          u[i] = v + grad[3 * 3 + i];
        } else {
          // u_i = 2 Lambda_i - 2 x_c d_i Phi_c + 2 d_i Psi (fmm.py:448-453)
          double v = 2.0 * pot[3 + i];
          for (int c = 0; c < 3; ++c) v -= 2.0 * xt[c] * grad[3 * c + i];
          u[i] = v + 2.0 * grad[3 * 6 + i];
        }
        u[i] += near[i];
      }
      if (a.mode == 2) {  // far part only: the near part (k_block_near) already wrote y
        for (int r = 0; r < 3; ++r) {
          double* yy = a.ysorted ? a.ysorted + 3 * (ti - a.tbody_a) + r : a.y + 3 * pn + r;
          *yy += a.beta * u[r];
        }
        return;
      }
      double corr[3] = {0.0, 0.0, 0.0};
      for (int e = a.rowptr[pn]; e < a.rowptr[pn + 1]; ++e) {
        const double* blk = a.vals + (size_t)e * 9;
        const double* xs = a.x + 3 * (size_t)a.cols[e];
        for (int r = 0; r < 3; ++r)
          corr[r] = fma(blk[3 * r], xs[0], fma(blk[3 * r + 1], xs[1], fma(blk[3 * r + 2], xs[2], corr[r])));
      }
      for (int r = 0; r < 3; ++r) {
        const double v = a.alpha * a.x[3 * pn + r] + a.beta * (u[r] + corr[r]);
        if (a.ysorted) a.ysorted[3 * (ti - a.tbody_a) + r] = v;
        else a.y[3 * pn + r] = v;
      }
    }
  }
}

// Near part of the 3-component (Stokes) layers, y = alpha x + beta (near + C x): one warp per
// target, its lanes over the near-field item partials and the 3x3 correction blocks of its
// row (a streaming block-CSR row product instead of one thread walking the whole row), the
// lanes' sums combined by a fixed xor-shuffle tree (bitwise reproducible).  Runs on the near
// stream beside the far field; the far epilogue (mode 2) then adds beta * u_far.
constexpr int BN_WARPS = 8;
__global__ void __launch_bounds__(BN_WARPS * 32) k_block_near(TreeDev T, EpiArgs a) {
  const int li = blockIdx.x, leaf = a.leaves[li];
  const int t0 = T.body_start[leaf], nt = T.body_count[leaf];
  const int lt = blockIdx.y * BN_WARPS + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (lt >= nt) return;  // warp-uniform
  const int ti = t0 + lt;
  const int ib = a.item_begin[li], ie = a.item_begin[li + 1];
  const int oo = ib < ie ? a.items[ib].out_off : 0;
  double v[3] = {0.0, 0.0, 0.0};
  for (int it = ib + lane; it < ie; it += 32) {
    const double* pp = a.part + (size_t)(oo + (it - ib) * nt + lt) * 3;
    v[0] += pp[0];
    v[1] += pp[1];
    v[2] += pp[2];
  }
  const int2 rr = a.rows[ti];
  for (int e = rr.x + lane; e < rr.y; e += 32) {
    const double* blk = a.vals + (size_t)e * 9;
    const double* xs = a.x + 3 * (size_t)a.cols[e];
    const double x0 = xs[0], x1 = xs[1], x2 = xs[2];
#pragma unroll
    for (int r = 0; r < 3; ++r) v[r] = fma(blk[3 * r], x0, fma(blk[3 * r + 1], x1, fma(blk[3 * r + 2], x2, v[r])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int r = 0; r < 3; ++r) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
  if (lane < 3) {
    const int pn = T.perm[ti];
    const double val = a.alpha * a.x[3 * pn + lane] + a.beta * (lane == 0 ? v[0] : lane == 1 ? v[1] : v[2]);
    if (a.ysorted) a.ysorted[3 * (ti - a.tbody_a) + lane] = val;
    else a.y[3 * pn + lane] = val;
  }
}

template <int KIND>
void launch_density(BemOp& op, const double* x, cudaStream_t s) {
  const int64_t ns = op.plan.src.n_points;
  k_density<KIND><<<grid_for(ns, 256), 256, 0, s>>>(
      ns, op.s_weight.get(), op.s_panel.get(), op.plan.src.px.get(), op.plan.src.py.get(),
      op.plan.src.pz.get(), op.normal.get(), x, op.q.get(), op.dip.get(), op.wsrc.get());
  FMM_LAUNCH_CHECK();
}

template <int KIND>
void launch_epilogue(BemOp& op, const EpiArgs& a, bool far, cudaStream_t s, int nl) {
  constexpr int C = EpiTraits<KIND>::C, NS = epi_slices<KIND>();
  const size_t red = NS > 1 ? (size_t)NS * EPI_TGT * 2 * sizeof(double) : 0;
  const size_t lbytes = (size_t)std::max(a.max_path, 1) * C * sizeof(double2);
  const size_t smem = (far ? lbytes * hcount(a.p) : 0) + red;
  if (nl <= 0) return;
  const int tiles = (std::max(op.plan.tgt.max_leaf_count, 1) + EPI_TGT - 1) / EPI_TGT;
  if (far) {
    const size_t most = lbytes * hcount(P_MAX) + red;
    FMM_REQUIRE(smem <= 227 * 1024, "epilogue: root paths too long for shared memory");
    FMM_CUDA(cudaFuncSetAttribute(k_epilogue<KIND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::min<size_t>(most, 227 * 1024)));
    launch_pdl(k_epilogue<KIND, true>, dim3(nl, tiles), dim3(EPI_TGT * NS), smem, s, tree_dev(op.plan.tgt), a);
  } else {
    k_epilogue<KIND, false><<<dim3(nl, tiles), EPI_TGT * NS, smem, s>>>(tree_dev(op.plan.tgt), a);
  }
  FMM_LAUNCH_CHECK();
}


// Far part of the one-channel epilogue when each leaf holds its complete local expansion (the
// L2L mode): one thread per target, the whole L2P of the leaf's expansion (harmonics.py:
// 258-270), y[panel] += beta phi / (4 pi).  Fully unrolled for the order P, so the columns'
// n-recurrences (serial within a column) interleave across columns; the leaf's expansion is
// staged once per CTA.  Replaces the path-walk epilogue's 4 column slices, whose lanes sat
// idle on the ~80-target leaves of cfg5.
constexpr int L2PL_THREADS = 128;

template <int P>
__global__ void __launch_bounds__(L2PL_THREADS) k_leaf_l2p(TreeDev T, const int* __restrict__ leaves,
                                                           const int* __restrict__ has_far,
                                                           const double2* __restrict__ L, double beta,
                                                           double* __restrict__ y, double* __restrict__ ysorted,
                                                           int tbody_a) {
  constexpr int H = hcount(P);
  __shared__ double2 sL[H];
  const int leaf = leaves[blockIdx.x];
  if (has_far[leaf + 1] == has_far[leaf]) return;  // no local expansion reaches this leaf
  const int nt = T.body_count[leaf];
  const int lt = blockIdx.y * L2PL_THREADS + threadIdx.x;
  if ((int)blockIdx.y * L2PL_THREADS >= nt) return;
  pdl_wait();  // L (the L2L levels) is complete past this point
  for (int i = threadIdx.x; i < H; i += L2PL_THREADS) sL[i] = L[(size_t)leaf * H + i];
  __syncthreads();
  if (lt >= nt) return;
  const int ti = T.body_start[leaf] + lt;
  const double x = T.px[ti] - T.cx[leaf], yy = T.py[ti] - T.cy[leaf], z = T.pz[ti] - T.cz[leaf];
  const double rho2 = x * x + yy * yy + z * z;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // independent partial sums (m mod 4)
  double2 diag = make_double2(1.0, 0.0);
#pragma unroll
  for (int m = 0; m <= P; ++m) {
    if (m > 0) diag = cscale(cmul(make_double2(x, yy), diag), -1.0 / (2.0 * m));  // R_m^m (harmonics.py:50-52)
    double2 cur = diag, prev2 = make_double2(0.0, 0.0);
    int i = hidx(m, m);
    double col = fma(sL[i].x, cur.x, -sL[i].y * cur.y);
#pragma unroll
    for (int n = m + 1; n <= P; ++n) {
      double2 nx;
      if (n == m + 1) {
        nx = cscale(cur, z);
      } else {
        const double az = c_l2p.ra[n * (P_MAX + 1) + m] * z, b = c_l2p.rb[n * (P_MAX + 1) + m] * rho2;
        nx = make_double2(fma(az, cur.x, -b * prev2.x), fma(az, cur.y, -b * prev2.y));
      }
      prev2 = cur;
      cur = nx;
      i += n;
      col = fma(sL[i].x, cur.x, fma(-sL[i].y, cur.y, col));
    }
    acc[m & 3] = m == 0 ? acc[0] + col : fma(2.0, col, acc[m & 3]);
  }
  const double phi = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  double* dst = ysorted ? ysorted + (ti - tbody_a) : y + T.perm[ti];
  *dst += beta * (phi / FOUR_PI);
}

template <int P>
void launch_leaf_l2p_p(BemOp& op, const double* L, double beta, double* y, cudaStream_t s) {
  const Tree& T = op.plan.tgt;
  const int tiles = (std::max(T.max_leaf_count, 1) + L2PL_THREADS - 1) / L2PL_THREADS;
  if (T.n_leaves > 0)
    launch_pdl(k_leaf_l2p<P>, dim3(T.n_leaves, tiles), dim3(L2PL_THREADS), 0, s, tree_dev(T),
               (const int*)T.leaves.get(), (const int*)op.plan.epi_leaf_off.get(),
               reinterpret_cast<const double2*>(L), beta, y, (double*)nullptr, 0);
  FMM_LAUNCH_CHECK();
}

template <int... Ps>
void launch_leaf_l2p(std::integer_sequence<int, Ps...>, int p, BemOp& op, const double2* L,
                     double beta, double* y, cudaStream_t s) {
  bool done = false;
  ((p == Ps && !done ? (launch_leaf_l2p_p<Ps>(op, reinterpret_cast<const double*>(L), beta, y, s), done = true)
                     : false),
   ...);
  FMM_REQUIRE(done, "leaf L2P: order out of range");
}

int layer_channels(int kind) { return kind == K_STOKESLET ? 4 : kind == K_STRESSLET ? 7 : 1; }

void ensure_dense(BemOp& op) {
  if (op.dense_ready) return;
  std::vector<int> row, srcl, ib;
  plan_dense_items(op.plan, op.dense_items_h, row, srcl, ib, op.dense_part_len);
  op.dense_items.upload(op.dense_items_h);
  op.dense_src.upload(srcl);
  op.dense_item_begin.upload(ib);
  op.dense_max_sources = 0;
  for (const auto& it : op.dense_items_h) {
    int acc = 0;
    for (int k = it.pair_begin; k < it.pair_end; ++k) acc += op.plan.src.h_body_count[srcl[k]];
    op.dense_max_sources = std::max(op.dense_max_sources, acc);
  }
  FMM_CUDA(cudaDeviceSynchronize());
  op.dense_ready = true;
}

void clear_graphs(BemOp& op) {
  for (auto& kv : op.graphs) cudaGraphExecDestroy(kv.second);
  op.graphs.clear();
  op.graph_kernels.clear();
}

// M2M levels above the leaves: rotation (DMMA, O(p^3)) from p = 3, octant-grouped dense below
// (FMMBEM_M2M=grouped forces the dense kernel)
bool m2m_rot_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FMMBEM_M2M");
    return !(e && std::string(e) == "grouped");
  }();
  return on;
}

// downward pass: rotation L2L down the target tree, then each leaf's own expansion at its
// targets (the reference's L2L + L2P, fmm.py:280-336), or (FMMBEM_DOWN=path, the sharded
// path, p < 3) every path cell's expansion evaluated at the leaf's targets (L2L is exact)
// The L2L levels are a chain of short, latency-bound launches (~15-20 us each at p = 14); they
// pay off only when the path epilogue's per-target work is large: cfg5 (4 088 target leaves,
// ~80 targets each): 0.29 -> 0.11 + 0.10 ms per p = 14 apply; cfg2 / cfg3 (272 leaves): slower.
constexpr int L2L_MIN_TGT_LEAVES = 1024;
constexpr int L2L_ROT_MIN_CELLS = 2048;  // levels with at least this many cells take the rotation L2L

bool l2l_rot_mode(const BemOp& op, int p, bool sharded, bool dense) {
  static const int force = [] {  // FMMBEM_DOWN=l2l | path
    const char* e = std::getenv("FMMBEM_DOWN");
    return !e ? -1 : std::string(e) == "path" ? 0 : 1;
  }();
  const bool want = force >= 0 ? force == 1 : op.plan.tgt.n_leaves >= L2L_MIN_TGT_LEAVES;
  return want && !sharded && !dense && m2m_rot_enabled() && p >= M2L_ROT_MIN_P &&
         op.plan.m2m_rot_p >= p;
}

void launch_upward_m2m(BemOp& op, int p, int C, cudaStream_t s) {
  Plan& pl = op.plan;
  if (m2m_rot_enabled() && p >= M2L_ROT_MIN_P && pl.m2m_rot_p >= p)
    launch_m2m_rot(pl, p, C, op.M.get(), op.m2m_cout.get(), s);
  else
    launch_m2m_grouped(pl, p, C, pl.rshift_src.get(), op.M.get(), op.m2m_cout.get(), s);
}

// allocations and p-dependent tables; never called inside a stream capture.
void prepare(BemOp& op, int kind, int p, bool dense) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");

  const int C = layer_channels(kind);
  const int64_t ns = op.plan.src.n_points;
  op.q.ensure((size_t)ns * (kind == K_STOKESLET ? 4 : 1));
  op.dip.ensure((size_t)ns * 3 * (kind == K_STRESSLET ? 7 : 1));
  op.wsrc.ensure((size_t)ns * 6);
  if (dense) {
    ensure_dense(op);
    op.part_dense.ensure((size_t)std::max<int64_t>(op.dense_part_len, 1) * 3);
  } else {
    op.part.ensure((size_t)std::max<int64_t>(op.plan.part_len, 1) * 3);
    op.M.ensure((size_t)op.plan.src.n_cells * C * hcount(p));
    op.m2m_cout.ensure((size_t)op.plan.src.n_cells * C * hcount(p));
    op.L.ensure((size_t)op.plan.tgt.n_cells * C * hcount(p));
    op.m2l_part.ensure((size_t)std::max(op.plan.n_m2l, 1) * C * hcount(p));
    plan_ensure_igrid(op.plan, p, op.s_main);
    if (op.plan.use_rot) plan_ensure_rot(op.plan, p, op.s_main);
    if (m2m_rot_enabled()) plan_ensure_m2m_rot(op.plan, p, op.s_main);
    if (op.shard.active && !op.shard.virtual_mode) {  // exchange buffers (no allocation in a capture)
      const size_t per = (size_t)op.shard.max_sleaves * C * hcount(p);
      op.shard.mleaf_send.ensure(std::max<size_t>(per, 1));
      op.shard.mleaf_recv.ensure(std::max<size_t>(per * op.shard.world, 1));
    }
    if (kind == op.basis_kind_for_sys) op.use_basis = ensure_p2m_basis(op, p, op.s_main);
  }
}

bool timeline_on() {
  static const bool on = std::getenv("FMMBEM_TIMELINE") != nullptr;
  return on;
}

void mark(BemOp& op, int i, cudaStream_t s) {
  if (op.timing && timeline_on())
    FMM_CUDA(cudaEventRecordWithFlags(op.ev_tl[i], s, cudaEventRecordExternal));
}

void record(BemOp& op, int stage, bool end, cudaStream_t s) {
  // External: inside a stream capture this becomes a real event-record node
  if (op.timing)
    FMM_CUDA(cudaEventRecordWithFlags(op.ev[2 * stage + (end ? 1 : 0)], s, cudaEventRecordExternal));
}

}  // namespace

BemOp::~BemOp() {
  for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
  if (mbox_h) cudaFreeHost(mbox_h);
  if (xpin_h) cudaFreeHost(xpin_h);
  if (ypin_h) cudaFreeHost(ypin_h);
  if (mflag_h) cudaFreeHost(mflag_h);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev_tl)
    if (e) cudaEventDestroy(e);
  for (auto& e : call_ev)
    if (e) cudaEventDestroy(e);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_enter) cudaEventDestroy(ev_enter);
  if (ev_basis) cudaEventDestroy(ev_basis);
  if (ev_m2l2) cudaEventDestroy(ev_m2l2);
  if (s_far2) cudaStreamDestroy(s_far2);
  if (ev_leave) cudaEventDestroy(ev_leave);
  if (s_main) cudaStreamDestroy(s_main);
  if (s_near) cudaStreamDestroy(s_near);
}

void op_init(BemOp& op, const double* panel_vertices, int64_t P, const double* gauss_pts,
             const double* gauss_wts, const double* fine_pts, const double* fine_wts,
             const double* normals, const double* areas, const double* leg_x, const double* leg_w,
             int n_gauss_singular, int formulation, double theta, int n_crit, double mu,
             double near_factor, int max_depth) {
  FMM_REQUIRE(P > 0, "mesh must have panels");
  FMM_REQUIRE(formulation >= 0 && formulation <= 2, "unknown formulation");
  FMM_REQUIRE(n_gauss_singular >= 1, "n_gauss_singular must be >= 1");
  upload_index_tables();
  upload_l2p_constants();
  op.formulation = formulation;
  op.mu = mu;
  op.near_factor = near_factor;
  op.n_gauss_singular = n_gauss_singular;
  op.n_panels = P;
  op.n = formulation == STOKES ? 3 * P : P;
  // the far-field chain (many short, dependent launches) gets the higher priority;
  // the near field (one large, independent launch) fills the remaining SMs
  int prio_lo = 0, prio_hi = 0;
  FMM_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const bool near_hi = std::getenv("FMMBEM_NEAR_PRIO_HIGH") != nullptr;
  FMM_CUDA(cudaStreamCreateWithPriority(&op.s_main, cudaStreamNonBlocking, near_hi ? prio_lo : prio_hi));
  FMM_CUDA(cudaStreamCreateWithPriority(&op.s_near, cudaStreamNonBlocking, near_hi ? prio_hi : prio_lo));
  FMM_CUDA(cudaEventCreateWithFlags(&op.ev_fork, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&op.ev_join, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&op.ev_enter, cudaEventDisableTiming));
  // (low priority: the latency-bound M2M levels on s_main must not wait for the leaf M2L's CTAs)
  FMM_CUDA(cudaStreamCreateWithPriority(&op.s_far2, cudaStreamNonBlocking, prio_lo));
  FMM_CUDA(cudaEventCreateWithFlags(&op.ev_basis, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&op.ev_m2l2, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&op.ev_leave, cudaEventDisableTiming));
  for (auto& e : op.ev) FMM_CUDA(cudaEventCreate(&e));
  for (auto& e : op.ev_tl) FMM_CUDA(cudaEventCreate(&e));
  for (auto& e : op.call_ev) FMM_CUDA(cudaEventCreate(&e));
  cudaStream_t s = op.s_main;
  // collocation points are bitwise the centroid Gauss point (bemop.py:64-67)
  std::vector<double> cen(3 * P);
  for (int64_t j = 0; j < P; ++j)
    for (int d = 0; d < 3; ++d) cen[3 * j + d] = gauss_pts[12 * j + d];
  op.centroid.upload(cen, s);
  op.normal.upload(normals, 3 * P, s);
  op.area.upload(areas, P, s);
  op.panel_verts.upload(panel_vertices, 9 * P, s);
  op.gauss_pos.upload(gauss_pts, 12 * P, s);
  op.gauss_w.upload(gauss_wts, 4 * P, s);
  op.fine_pos.upload(fine_pts, 57 * P, s);
  op.fine_w.upload(fine_wts, 19 * P, s);
  op.leg_x.upload(leg_x, n_gauss_singular, s);
  op.leg_w.upload(leg_w, n_gauss_singular, s);
  // large double-layer systems: 1 024-source items for the persistent near-field kernel (fewer
  // item hand-overs; 896 is the better tile below ~100 k panels and for the other kernels)
  if (formulation == LAPLACE_SECOND && 4 * P >= 400000 && !std::getenv("FMMBEM_P2P_ITEM")) op.plan.p2p_item_src = 1024;
  plan_build(op.plan, gauss_pts, 4 * P, cen.data(), P, n_crit, theta, max_depth, s);
  const int64_t ns = op.plan.src.n_points;
  op.s_weight.resize(ns);
  op.s_panel.resize(ns);
  op.self_src.resize(P);
  op.p2p_sched.resize(2);
  op.p2p_sched.zero(s);
  {
    DevBuf<int> tinv;
    tinv.resize(P);
    k_invert_perm<<<grid_for(P, 256), 256, 0, s>>>(P, op.plan.tgt.perm.get(), tinv.get());
    FMM_LAUNCH_CHECK();
    k_sorted_sources<<<grid_for(ns, 256), 256, 0, s>>>(ns, op.plan.src.perm.get(), op.gauss_w.get(),
                                                        op.s_weight.get(), op.s_panel.get(), tinv.get(),
                                                        op.self_src.get());
    FMM_LAUNCH_CHECK();
    op.srec.resize((size_t)ns * 3);
    k_source_records<<<grid_for(ns, 256), 256, 0, s>>>(ns, op.plan.src.px.get(), op.plan.src.py.get(),
                                                        op.plan.src.pz.get(), op.s_weight.get(),
                                                        op.s_panel.get(), op.normal.get(), op.srec.get());
    FMM_LAUNCH_CHECK();
    FMM_CUDA(cudaStreamSynchronize(s));
    op.h_self_src = op.self_src.download(s);
  }
  op.p2p_aux.build(op.plan.src, op.plan.tgt, op.plan.items, op.plan.h_p2p_src, op.h_self_src, s);
  op.max_item_sources = 0;
  for (const auto& it : op.plan.items) {
    int acc = 0;
    for (int k = it.pair_begin; k < it.pair_end; ++k) acc += op.plan.src.h_body_count[op.plan.h_p2p_src[k]];
    op.max_item_sources = std::max(op.max_item_sources, acc);
  }
  build_near_pairs(op, s);
  op.near_rows.resize(P);
  k_row_ranges<<<grid_for(P, 256), 256, 0, s>>>(P, op.plan.tgt.perm.get(), op.near_rowptr.get(), op.near_rows.get());
  FMM_LAUNCH_CHECK();
  int sys_kind, rhs_kind;
  if (formulation == LAPLACE_FIRST) { sys_kind = K_LAP_SINGLE; rhs_kind = K_LAP_DOUBLE; }
  else if (formulation == LAPLACE_SECOND) { sys_kind = K_LAP_DOUBLE; rhs_kind = K_LAP_SINGLE; }
  else { sys_kind = K_STOKESLET; rhs_kind = K_STRESSLET; }
  op.basis_kind_for_sys = sys_kind;
  build_correction(op, sys_kind, op.c_sys, s);
  build_correction(op, rhs_kind, op.c_rhs, s);
  op.x_in.resize(op.n);
  op.y_out.resize(op.n);
  // size the apply workspaces for the largest order up front (graphs bake in addresses)
  prepare(op, sys_kind, P_MAX, false);
  FMM_CUDA(cudaStreamSynchronize(s));
}

void launch_layer_epilogue(BemOp& op, const LayerCall& c, bool sharded, cudaStream_t s, int mode) {
  Plan& pl = op.plan;
  ShardWork& sw = op.shard;
  EpiArgs a;
  a.mode = mode;
  a.leaves = sharded ? sw.epi_leaves.get() : pl.tgt.leaves.get();
  a.item_begin = c.dense ? op.dense_item_begin.get() : sharded ? sw.item_begin.get() : pl.tleaf_item_begin.get();
  a.items = c.dense ? op.dense_items.get() : sharded ? sw.items.get() : pl.d_items.get();
  a.ysorted = (sharded && !sw.virtual_mode) ? sw.ysend.get() : nullptr;
  a.tbody_a = sw.tbody_a;
  const int n_epi = sharded ? sw.n_epi_leaves : pl.tgt.n_leaves;
  a.part = c.dense ? op.part_dense.get() : op.part.get();
  a.L = op.L.get();
  const bool l2l = l2l_rot_mode(op, c.p, sharded, c.dense);
  a.path_off = l2l ? pl.epi_leaf_off.get() : pl.epi_path_off.get();
  a.path = l2l ? pl.epi_leaf.get() : pl.epi_path.get();
  a.max_path = l2l ? 1 : pl.max_path;
  a.p = c.p;
  a.rowptr = op.near_rowptr.get();
  a.rows = op.near_rows.get();
  a.cols = op.near_cols.get();
  a.vals = c.corr->vals.get();
  a.x = c.x;
  a.alpha = c.alpha;
  a.beta = c.beta;
  a.y = c.y;
  if (mode != 1) record(op, ST_EPI, false, s);
  const bool far = !c.dense && mode != 1;
  if (mode == 1 && c.kind == K_STOKESLET) {
    const int tiles = (std::max(op.plan.tgt.max_leaf_count, 1) + BN_WARPS - 1) / BN_WARPS;
    if (n_epi > 0) k_block_near<<<dim3(n_epi, tiles), BN_WARPS * 32, 0, s>>>(tree_dev(op.plan.tgt), a);
    FMM_LAUNCH_CHECK();
    return;
  }
  if (mode == 2 && l2l && (c.kind == K_LAP_SINGLE || c.kind == K_LAP_DOUBLE) && !a.ysorted) {
    launch_leaf_l2p(std::make_integer_sequence<int, P_MAX + 1>{}, c.p, op, op.L.get(), c.beta, c.y, s);
    return;
  }
  switch (c.kind) {
    case K_LAP_SINGLE: launch_epilogue<K_LAP_SINGLE>(op, a, far, s, n_epi); break;
    case K_LAP_DOUBLE: launch_epilogue<K_LAP_DOUBLE>(op, a, far, s, n_epi); break;
    case K_STOKESLET: launch_epilogue<K_STOKESLET>(op, a, far, s, n_epi); break;
    default: launch_epilogue<K_STRESSLET>(op, a, far, s, n_epi); break;
  }
}

void op_layer(BemOp& op, const LayerCall& c, cudaStream_t s, bool sharded) {
  Plan& pl = op.plan;
  ShardWork& sw = op.shard;
  sharded = sharded && sw.active && !c.dense;
  const int C = layer_channels(c.kind);
  const TreeDev S = tree_dev(pl.src), T = tree_dev(pl.tgt);
  record(op, ST_TOTAL, false, s);
  mark(op, 0, s);
  // the double layer's persistent near field reads x through static source records and the
  // basis upward pass reads x directly: the Gauss-point densities are only needed otherwise
  const bool basis_up = c.kind == op.basis_kind_for_sys && op.use_basis && op.basis_p >= c.p;
  const bool lapd_near = c.kind == K_LAP_DOUBLE && !c.dense &&
                         p2p_lapd_usable(sharded ? &sw.p2p_aux : &op.p2p_aux,
                                         sharded ? sw.max_item_sources : op.max_item_sources);
  const bool need_density = !(lapd_near && basis_up);
  if (need_density) switch (c.kind) {
    case K_LAP_SINGLE: launch_density<K_LAP_SINGLE>(op, c.x, s); break;
    case K_LAP_DOUBLE: launch_density<K_LAP_DOUBLE>(op, c.x, s); break;
    case K_STOKESLET: launch_density<K_STOKESLET>(op, c.x, s); break;
    default: launch_density<K_STRESSLET>(op, c.x, s); break;
  }
  const double* w = c.kind == K_LAP_SINGLE ? op.q.get() : c.kind == K_LAP_DOUBLE ? op.dip.get()
                                                                                : op.wsrc.get();
  // M2L split by source cell: the pairs with leaf sources run on a third stream as soon as the
  // leaf basis stream is done, beside the (latency-bound) M2M levels; the rest after the M2M
  // (FMMBEM_M2L_SPLIT=1; off by default: measured slower on cfg5, 445 vs 451 mat-vecs/s —
  // the leaf M2L's long CTAs hold the SMs and each M2M level waits for slots, at any stream
  // priority); the gather waits for both
  static const bool split_env = std::getenv("FMMBEM_M2L_SPLIT") && std::string(std::getenv("FMMBEM_M2L_SPLIT")) == "1";
  const bool split_m2l = split_env && !c.dense && !sharded && pl.use_rot && c.p >= M2L_ROT_MIN_P &&
                         pl.rot_p >= c.p && !pl.m2l_ci_leaf.empty() &&
                         !(op.basis_clustered && !op.basis_leaf_only && c.kind == op.basis_kind_for_sys &&
                           op.use_basis && op.basis_p >= c.p);  // (direct basis: no M2M to hide)
  bool leaf_m2l_forked = false;
  auto fork_leaf_m2l = [&]() {
    if (!split_m2l) return;
    FMM_CUDA(cudaEventRecord(op.ev_basis, s));
    FMM_CUDA(cudaStreamWaitEvent(op.s_far2, op.ev_basis, 0));
    launch_m2l_rot(pl, pl.d_m2l_ci_leaf.get(), pl.m2l_cp_leaf.get(), (int)pl.m2l_ci_leaf.size(), c.p, C,
                   op.M.get(), op.m2l_part.get(), op.s_far2, true, &pl.m2l_rg_leaf);
    FMM_CUDA(cudaEventRecord(op.ev_m2l2, op.s_far2));
    leaf_m2l_forked = true;
  };
  // far-field stages as steps; FMMBEM_AHEAD=1 (upward) / 2 (upward + M2L) issues them before
  // the near field is forked (scheduling experiments; default 0: all after the fork)
  auto upward = [&]() {
    const double* q = (c.kind == K_LAP_SINGLE || c.kind == K_STOKESLET) ? op.q.get() : nullptr;
    const double* d = (c.kind == K_LAP_DOUBLE || c.kind == K_STRESSLET) ? op.dip.get() : nullptr;
    record(op, ST_UP, false, s);
    const bool own_only = sharded && !sw.virtual_mode;  // P2M of own leaves, then all-gather
    const int* lv = own_only ? sw.p2m_leaves.get() : pl.src.leaves.get();
    const int nlv = own_only ? sw.n_p2m_leaves : pl.src.n_leaves;
    const bool basis = c.kind == op.basis_kind_for_sys && op.use_basis && op.basis_p >= c.p;
    if (basis && op.basis_clustered && !own_only) {
      // every multipole straight from the sources (no M2M levels), or the leaves' multipoles
      // and the M2M chain above them
      launch_p2m_basis(op, c.p, C, c.x, op.M.get(), s, nullptr, 0);
      mark(op, 1, s);
      if (op.basis_leaf_only) {
        fork_leaf_m2l();
        launch_upward_m2m(op, c.p, C, s);
      }
      mark(op, 2, s);
    } else {
      if (basis)
        launch_p2m_basis(op, c.p, C, c.x, op.M.get(), s, lv, nlv);
      else
        launch_p2m(S, lv, nlv, c.p, C, q, d, op.M.get(), s);
      if (own_only) shard_exchange_multipoles(op, C, c.p, s);
      fork_leaf_m2l();
      launch_upward_m2m(op, c.p, C, s);
    }
    record(op, ST_UP, true, s);
  };
  auto m2l = [&]() {
    record(op, ST_M2L, false, s);
    if (split_m2l) {
      launch_m2l_rot(pl, pl.d_m2l_ci_rest.get(), pl.m2l_cp_rest.get(), (int)pl.m2l_ci_rest.size(), c.p, C,
                     op.M.get(), op.m2l_part.get(), s, true, &pl.m2l_rg_rest);
      if (leaf_m2l_forked)
        FMM_CUDA(cudaStreamWaitEvent(s, op.ev_m2l2, 0));
      else  // (the upward path did not fork it)
        launch_m2l_rot(pl, pl.d_m2l_ci_leaf.get(), pl.m2l_cp_leaf.get(), (int)pl.m2l_ci_leaf.size(), c.p, C,
                       op.M.get(), op.m2l_part.get(), s, true, &pl.m2l_rg_leaf);
      launch_m2l_gather(pl, c.p, C, op.m2l_part.get(), op.L.get(), s);
    } else if (sharded)
      launch_m2l(pl, c.p, C, op.M.get(), op.L.get(), op.m2l_part.get(), s, sw.gitems.get(),
                 (int)sw.gitems_h.size(), sw.gather_cells.get(), sw.n_gather_cells, sw.gpair.get(),
                 sw.citems.get(), sw.n_citems, sw.cpair.get(), &sw.rg);
    else
      launch_m2l(pl, c.p, C, op.M.get(), op.L.get(), op.m2l_part.get(), s);
    record(op, ST_M2L, true, s);
    mark(op, 3, s);
  };
  static const int ahead_env = std::getenv("FMMBEM_AHEAD") ? std::atoi(std::getenv("FMMBEM_AHEAD")) : 0;
  const int ahead = c.dense ? 0 : ahead_env;
  if (ahead >= 1) upward();
  if (ahead >= 2) m2l();
  // near field on the second stream
  // near field on the second stream (concurrent with the far field), or in line
  const bool serial = op.serial_near;
  cudaStream_t sn = serial ? s : op.s_near;
  if (!serial) {
    FMM_CUDA(cudaEventRecord(op.ev_fork, s));
    FMM_CUDA(cudaStreamWaitEvent(op.s_near, op.ev_fork, 0));
  }
  record(op, ST_P2P, false, sn);
  if (c.dense)
    launch_p2p((P2PKind)c.kind, S, T, op.dense_items.get(), (int)op.dense_items_h.size(),
               op.dense_src.get(), op.dense_max_sources, w, op.part_dense.get(), sn,
               nullptr);
  else if (sharded)
    launch_p2p((P2PKind)c.kind, S, T, sw.items.get(), (int)sw.items_h.size(), pl.p2p_src.get(),
               sw.max_item_sources, w, op.part.get(), sn, sw.p2p_order.get(), &sw.p2p_aux,
               op.p2p_sched.get(), op.srec.get(), op.s_panel.get(), c.x);
  else
    launch_p2p((P2PKind)c.kind, S, T, pl.d_items.get(), (int)pl.items.size(), pl.p2p_src.get(),
               op.max_item_sources, w, op.part.get(), sn, pl.p2p_order.get(), &op.p2p_aux,
               op.p2p_sched.get(), op.srec.get(), op.s_panel.get(), c.x);
  // one-channel kinds: the near part of the epilogue (item partials + correction rows) runs
  // right behind the near field, concurrently with the far field
  record(op, ST_P2P, true, sn);
  mark(op, 5, sn);
  const bool split_epi = !c.dense && (c.kind == K_LAP_SINGLE || c.kind == K_LAP_DOUBLE || c.kind == K_STOKESLET);
  if (split_epi) launch_layer_epilogue(op, c, sharded, sn, 1);
  if (!serial) FMM_CUDA(cudaEventRecord(op.ev_join, op.s_near));
  // far field on the main stream
  if (!c.dense) {
    if (ahead < 1) upward();
    if (ahead < 2) m2l();

    record(op, ST_DOWN, false, s);
    if (l2l_rot_mode(op, c.p, sharded, c.dense)) {
      // per level: few cells -> the dense one-CTA-per-cell kernel (shorter critical path); many
      // cells (the bottom levels of a large tree) -> the O(p^3) DMMA rotation kernel, one warp per
      // 8 cells (cfg5 p = 14: 3 560 cells 68 us dense vs ~15 us).  FMMBEM_L2L=rot | dense forces one.
      static const int mode = [] {
        const char* e = std::getenv("FMMBEM_L2L");
        return !e ? 0 : std::string(e) == "rot" ? 1 : std::string(e) == "dense" ? 2 : 0;
      }();
      const int nl = (int)pl.l2l_level_off.size() - 1;
      for (int l = 1; l < nl; ++l) {
        const int cells = pl.l2l_level_off[l + 1] - pl.l2l_level_off[l];
        if (cells <= 0) continue;
        static const int min_cells =
            std::getenv("FMMBEM_L2L_ROT_MIN") ? std::atoi(std::getenv("FMMBEM_L2L_ROT_MIN")) : L2L_ROT_MIN_CELLS;
        const bool rot = mode == 1 || (mode == 0 && cells >= min_cells);
        if (rot)
          launch_l2l_rot(pl, c.p, C, op.L.get(), s, l, l + 1);
        else
          launch_l2l(pl.tgt, pl.l2l_level_off, pl.l2l_cells.get(), c.p, C, pl.rshift_tgt.get(), op.L.get(), s, l,
                     l + 1);
      }
    }
    record(op, ST_DOWN, true, s);
    mark(op, 4, s);
  }
  if (!serial) FMM_CUDA(cudaStreamWaitEvent(s, op.ev_join, 0));
  launch_layer_epilogue(op, c, sharded, s, split_epi ? 2 : 0);
  const bool ysorted_out = sharded && !sw.virtual_mode;
  if (ysorted_out && !sw.local_vectors)
    shard_exchange_y(op, c.kind == K_LAP_SINGLE || c.kind == K_LAP_DOUBLE ? 1 : 3, c.y, s);
  record(op, ST_EPI, true, s);
  record(op, ST_TOTAL, true, s);
  mark(op, 6, s);
}

namespace {

void sys_call(BemOp& op, int p, bool dense, const double* x, double* y, LayerCall& c) {
  c.p = p;
  c.dense = dense;
  c.corr = &op.c_sys;
  c.x = x;
  c.y = y;
  if (op.formulation == LAPLACE_FIRST) { c.kind = K_LAP_SINGLE; c.alpha = 0.0; c.beta = 1.0; }
  else if (op.formulation == LAPLACE_SECOND) { c.kind = K_LAP_DOUBLE; c.alpha = 0.5; c.beta = -1.0; }
  else { c.kind = K_STOKESLET; c.alpha = 0.0; c.beta = 1.0 / (8.0 * 3.141592653589793 * op.mu); }
}

void accumulate_stage_times(BemOp& op) {
  if (!op.timing) return;
  if (timeline_on()) {
    float t[7];
    for (int i = 0; i < 7; ++i)
      if (cudaEventElapsedTime(&t[i], op.ev_tl[0], op.ev_tl[i]) != cudaSuccess) {
        cudaGetLastError();
        t[i] = -1.f;
      }
    std::fprintf(stderr, "TIMELINE basis %.3f m2m %.3f m2l %.3f l2l %.3f p2p %.3f end %.3f\n", t[1], t[2],
                 t[3], t[4], t[5], t[6]);
  }
  for (int st = 0; st < N_STAGES; ++st) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, op.ev[2 * st], op.ev[2 * st + 1]) == cudaSuccess)
      op.stage_ms[st] += ms;
    else
      cudaGetLastError();
  }
  op.stage_calls++;
}

}  // namespace

// y = A x for device vectors (x, y may alias nothing in the op)
void op_apply_device(BemOp& op, const double* x, double* y, int p) {
  LayerCall c;
  sys_call(op, p, false, op.x_in.get(), op.y_out.get(), c);
  prepare(op, c.kind, p, false);
  cudaStream_t s = op.s_main;
  if (x) FMM_CUDA(cudaMemcpyAsync(op.x_in.get(), x, op.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const bool sharded = op.shard.active;
  // graphs: unsharded, virtual and NCCL shards (NCCL collectives are captured); the host
  // transport blocks the host inside every collective and runs eagerly
  if (op.use_graphs && !(sharded && op.shard.transport == ShardWork::T_HOST)) {
    // captured graphs bake in buffer addresses: any reallocation invalidates them
    const std::vector<const void*> sig = {op.q.get(), op.dip.get(), op.wsrc.get(), op.srec.get(), op.part.get(),
                                          op.M.get(), op.L.get(), op.plan.igrid.get(),
                                          op.x_in.get(), op.y_out.get(), op.m2l_part.get(),
                                          op.p2m_basis.get(), op.m2m_cout.get(), op.plan.rotf.get(),
                                          op.plan.rot_aux.get(), op.plan.rot_dir.get(), op.cl_panel.get(),
                                          op.p2m_items.d.get(), op.p2m_reduce.d.get(), op.p2m_part.get(),
                                          // table LAYOUTS baked into the captured kernel arguments
                                          // (a regrown table may come back at the same address)
                                          (const void*)(intptr_t)op.plan.rot_p,
                                          (const void*)(intptr_t)op.plan.igrid_p,
                                          (const void*)(intptr_t)op.basis_p,
                                          (const void*)(intptr_t)op.plan.n_rot_dirs,
                                          (const void*)(intptr_t)op.basis_cols,
                                          op.plan.m2m_rotf.get(), op.plan.m2m_aux.get(),
                                          op.plan.l2l_rotf.get(), op.plan.l2l_aux.get(),
                                          (const void*)(intptr_t)op.plan.m2m_rot_p,
                                          op.shard.mleaf_send.get(), op.shard.mleaf_recv.get(),
                                          op.shard.ysend.get(), op.shard.yrecv.get()};
    if (sig != op.graph_sig) {
      clear_graphs(op);
      op.graph_sig = sig;
    }
    const int key = p * 8 + (op.timing ? 1 : 0) + (op.serial_near ? 2 : 0) + (op.shard.local_vectors ? 4 : 0);
    auto it = op.graphs.find(key);
    if (it == op.graphs.end()) {
      cudaGraph_t g;
      FMM_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        op_layer(op, c, s, sharded);
      } catch (...) {
        cudaStreamEndCapture(s, &g);
        throw;
      }
      FMM_CUDA(cudaStreamEndCapture(s, &g));
      size_t nn = 0;
      FMM_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      if (nn) FMM_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
      int nk = 0;
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        FMM_CUDA(cudaGraphNodeGetType(nd, &ty));
        nk += ty == cudaGraphNodeTypeKernel ? 1 : 0;
      }
      cudaGraphExec_t ex;
      FMM_CUDA(cudaGraphInstantiate(&ex, g, 0));
      cudaGraphDestroy(g);
      it = op.graphs.emplace(key, ex).first;
      op.graph_kernels[key] = nk;
    }
    FMM_CUDA(cudaGraphLaunch(it->second, s));
    op.kernel_launches += op.graph_kernels[key];
    op.applies += 1;
  } else {
    op_layer(op, c, s, sharded);
    op.applies += 1;
  }
  if (y) FMM_CUDA(cudaMemcpyAsync(y, op.y_out.get(), op.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

// stage timers of the last apply; call only after the op's stream has been synchronised
void op_collect_stage_times(BemOp& op) { accumulate_stage_times(op); }

void op_dense_apply_device(BemOp& op, const double* x, double* y) {
  LayerCall c;
  sys_call(op, 0, true, x, y, c);
  prepare(op, c.kind, 0, true);
  op_layer(op, c, op.s_main);
  FMM_CUDA(cudaStreamSynchronize(op.s_main));
}

void op_rhs_device(BemOp& op, const double* data, double* b, int p, bool dense) {
  LayerCall c;
  c.p = p;
  c.dense = dense;
  c.corr = &op.c_rhs;
  c.x = data;
  c.y = b;
  if (op.formulation == LAPLACE_FIRST) { c.kind = K_LAP_DOUBLE; c.alpha = 0.5; c.beta = -1.0; }
  else if (op.formulation == LAPLACE_SECOND) { c.kind = K_LAP_SINGLE; c.alpha = 0.0; c.beta = 1.0; }
  else { c.kind = K_STRESSLET; c.alpha = 0.5; c.beta = -1.0 / (8.0 * 3.141592653589793); }
  prepare(op, c.kind, p, dense);
  op_layer(op, c, op.s_main);
  FMM_CUDA(cudaStreamSynchronize(op.s_main));
}

// ------------------------------------------------------- FmmPlan far/near (generic)
namespace {
__global__ void k_permute_channels(int64_t ns, int C, int width, const int* perm, const double* in,
                                   double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const int o = perm[i];
  for (int c = 0; c < C; ++c)
    for (int k = 0; k < width; ++k) out[((size_t)c * ns + i) * width + k] = in[((size_t)c * ns + o) * width + k];
}
}  // namespace

void plan_evaluate(Plan& plan, int C, const double* q_orig, const double* d_orig, int p,
                   bool want_grad, int parts, double* pot, double* grad, cudaStream_t s) {
  upload_index_tables();
  FMM_REQUIRE(C == 1 || C == 4 || C == 7, "channel count must be 1, 4 or 7");
  FMM_REQUIRE(q_orig || d_orig, "charges or dipoles required");
  const int64_t ns = plan.src.n_points;
  DevBuf<double>&qs = plan.eval.qs, &ds = plan.eval.ds;
  if (q_orig) {
    qs.ensure((size_t)C * ns);
    k_permute_channels<<<grid_for(ns, 256), 256, 0, s>>>(ns, C, 1, plan.src.perm.get(), q_orig, qs.get());
  }
  if (d_orig) {
    ds.ensure((size_t)C * ns * 3);
    k_permute_channels<<<grid_for(ns, 256), 256, 0, s>>>(ns, C, 3, plan.src.perm.get(), d_orig, ds.get());
  }
  FMM_LAUNCH_CHECK();
  const TreeDev S = tree_dev(plan.src), T = tree_dev(plan.tgt);
  if (parts & 1) {
    plan_ensure_igrid(plan, p, s);
    if (plan.use_rot) plan_ensure_rot(plan, p, s);
    DevBuf<double2>&M = plan.eval.M, &L = plan.eval.L, &part = plan.eval.part;
    M.ensure((size_t)plan.src.n_cells * C * hcount(p));
    L.ensure((size_t)plan.tgt.n_cells * C * hcount(p));
    part.ensure((size_t)std::max(plan.n_m2l, 1) * C * hcount(p));
    launch_p2m(S, plan.src.leaves.get(), plan.src.n_leaves, p, C, q_orig ? qs.get() : nullptr,
               d_orig ? ds.get() : nullptr, M.get(), s);
    launch_m2m(plan.src, plan.m2m_level_off, plan.m2m_cells.get(), p, C, plan.rshift_src.get(), M.get(), s);
    launch_m2l(plan, p, C, M.get(), L.get(), part.get(), s);
    launch_l2l(plan.tgt, plan.l2l_level_off, plan.l2l_cells.get(), p, C, plan.rshift_tgt.get(), L.get(), s);
    launch_l2p_channels(T, plan.tgt.leaves.get(), plan.tgt.n_leaves, p, C, want_grad, L.get(), pot,
                        grad, s);
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  if (parts & 2) {
    launch_p2p_channels(S, T, plan, C, q_orig ? qs.get() : nullptr, d_orig ? ds.get() : nullptr,
                        want_grad, pot, grad, s);
  }
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fmmbem
