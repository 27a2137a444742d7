// Near field (P2P) kernels.
//
// Reference: FmmPlan.near_field (fmm.py:356-419) over the per-target-leaf
// source lists (fmm.py:161-167, p2p_items 351-354).  Coincident source /
// target pairs contribute exactly zero (the d2 > 0 mask, fmm.py:394,403): the
// BEM collocation point is bitwise the centroid Gauss point.
//
// Work decomposition: a work item is (target leaf, slice of its source-leaf
// list holding <= ~1024 sources).  The item's sources are staged once in
// shared memory (SoA, coalesced), targets stay in registers, and when a leaf
// has fewer targets than threads the CTA splits the sources over thread
// groups and reduces them in a fixed order.  Each item writes its own partial
// sums; the epilogue adds the items of a leaf in item order, so the result
// is bitwise reproducible without atomics.
//
// Stokes uses the direct stokeslet G f = f/r + r (r.f)/r^3 (kernels.py:42-48)
// instead of the reference's four-channel decomposition of the near field;
// the two agree to ~1e-13 and the direct form is cheaper.
#include "kernels.cuh"
#include "l2p.cuh"

namespace fmmbem {

constexpr int P2P_THREADS = 256;

template <P2PKind K>
struct P2PTraits;
template <> struct P2PTraits<P2PKind::LAP_Q> { static constexpr int NW = 1, NC = 1, TPT = 2; };
template <> struct P2PTraits<P2PKind::LAP_D> { static constexpr int NW = 3, NC = 1, TPT = 4; };
template <> struct P2PTraits<P2PKind::STOKESLET> { static constexpr int NW = 3, NC = 3, TPT = 2; };
template <> struct P2PTraits<P2PKind::STRESSLET> { static constexpr int NW = 6, NC = 3, TPT = 2; };

// 1/sqrt(x) for x > 0 to ~1 ulp: the SFU's double-precision seed (MUFU.RSQ64H,
// ~2^-22) plus one third-order Newton step, y (1 + e/2 + 3e^2/8), e = 1 - x y^2:
// 5 DP instructions and no slow-path branch (the libdevice rsqrt carries one).
// x == 0 yields inf/NaN and is masked by the caller (the reference's d2 > 0 rule).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// Second-order Newton step on the same seed, y (1 + (1 - x y^2) / 2): relative
// error ~1.5 (2^-22.9)^2 ~ 3e-14, used by the double layer (4 DP instructions).
__device__ __forceinline__ double rsqrt_nr2(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return fma(y, fma(-0.5 * x * y, y, 0.5), y);
}

template <P2PKind K>
__device__ __forceinline__ void interact(double rx, double ry, double rz, const double* wv,
                                         double* acc) {
  if (K == P2PKind::LAP_D) {
    // d2 + 1e-200: a coincident pair (r = 0) gives r.n = 0 times a finite
    // 1e300 instead of the masked branch; for any other pair the bias is far
    // below one ulp of d2.
    const double d2 = fma(rx, rx, fma(ry, ry, fma(rz, rz, 1e-200)));
    // r^-3 from the seed y directly: with e = 1 - d2 y^2, (y (1 + e/2))^3 =
    // y^3 (1 + 3e/2 + O(e^2)), relative error ~7.5 (2^-22.9)^2 ~ 1e-13
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d2));
    const double y2 = y * y;
    const double y3 = y2 * y;
    const double e = fma(-d2, y2, 1.0);
    const double rn = fma(rx, wv[0], fma(ry, wv[1], rz * wv[2]));
    acc[0] = fma(rn, fma(1.5 * e, y3, y3), acc[0]);
    return;
  }
  const double d2 = fma(rx, rx, fma(ry, ry, rz * rz));
  const double inv = d2 > 0.0 ? rsqrt_nr(d2) : 0.0;
  if (K == P2PKind::LAP_Q) {
    acc[0] = fma(wv[0], inv, acc[0]);
  } else if (K == P2PKind::LAP_D) {
    const double rn = fma(rx, wv[0], fma(ry, wv[1], rz * wv[2]));
    const double inv3 = inv * inv * inv;
    acc[0] = fma(rn, inv3, acc[0]);
  } else if (K == P2PKind::STOKESLET) {
    const double rf = fma(rx, wv[0], fma(ry, wv[1], rz * wv[2]));
    const double s = rf * (inv * inv * inv);
    acc[0] = fma(wv[0], inv, fma(rx, s, acc[0]));
    acc[1] = fma(wv[1], inv, fma(ry, s, acc[1]));
    acc[2] = fma(wv[2], inv, fma(rz, s, acc[2]));
  } else {
    // stresslet contracted with the source normal: 6 r (r.f)(r.n) / r^5 (kernels.py:51-58)
    const double rf = fma(rx, wv[0], fma(ry, wv[1], rz * wv[2]));
    const double rn = fma(rx, wv[3], fma(ry, wv[4], rz * wv[5]));
    const double inv2 = inv * inv;
    const double s = 6.0 * rf * rn * (inv2 * inv2 * inv);
    acc[0] = fma(rx, s, acc[0]);
    acc[1] = fma(ry, s, acc[1]);
    acc[2] = fma(rz, s, acc[2]);
  }
}

// sources staged as double2 planes: (x, y), (z, w0), (w1, w2), (w3, w4), (w5, -)
template <int NW> struct SrcPlanes { static constexpr int N = (3 + NW + 1) / 2; };

template <P2PKind K>
__global__ void __launch_bounds__(P2P_THREADS, 4)
k_p2p(TreeDev S, TreeDev T, const P2PItem* __restrict__ items, const int* __restrict__ order,
      const int* __restrict__ p2p_src,
      int max_src, const double* __restrict__ w, double* __restrict__ part) {
  constexpr int NW = P2PTraits<K>::NW, NC = P2PTraits<K>::NC;
  constexpr int NPL = SrcPlanes<NW>::N;
  constexpr int TPT = P2PTraits<K>::TPT;  // targets per thread: each staged source is reused TPT times
  extern __shared__ double2 sh2[];
  const P2PItem it = items[order ? order[blockIdx.x] : (int)blockIdx.x];
  int ns = 0;
  for (int k = it.pair_begin; k < it.pair_end; ++k) {
    const int leaf = p2p_src[k];
    const int s0 = S.body_start[leaf], cnt = S.body_count[leaf];
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      double v[2 * NPL];
      v[0] = S.px[s0 + i];
      v[1] = S.py[s0 + i];
      v[2] = S.pz[s0 + i];
#pragma unroll
      for (int q = 0; q < NW; ++q) v[3 + q] = w[(size_t)(s0 + i) * NW + q];
#pragma unroll
      for (int q = 3 + NW; q < 2 * NPL; ++q) v[q] = 0.0;
#pragma unroll
      for (int pl = 0; pl < NPL; ++pl) sh2[pl * max_src + ns + i] = make_double2(v[2 * pl], v[2 * pl + 1]);
    }
    ns += cnt;
  }
  __syncthreads();
  const int t0 = T.body_start[it.tgt_leaf], nt = T.body_count[it.tgt_leaf];
  const int nslot = (nt + TPT - 1) / TPT;
  for (int sbase = 0; sbase < nslot; sbase += blockDim.x) {
    const int nsl = min(nslot - sbase, (int)blockDim.x);
    const int G = blockDim.x / nsl;
    const int sl = threadIdx.x % nsl, g = threadIdx.x / nsl;
    double acc[TPT][NC];
    double tx[TPT], ty[TPT], tz[TPT];
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
      const int lt = min(sbase + sl + q * nslot, nt - 1);
      tx[q] = T.px[t0 + lt];
      ty[q] = T.py[t0 + lt];
      tz[q] = T.pz[t0 + lt];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[q][c] = 0.0;
    }
    if (g < G) {
      for (int j = g; j < ns; j += G) {
        double v[2 * NPL];
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl) {
          const double2 u = sh2[pl * max_src + j];
          v[2 * pl] = u.x;
          v[2 * pl + 1] = u.y;
        }
#pragma unroll
        for (int q = 0; q < TPT; ++q) interact<K>(tx[q] - v[0], ty[q] - v[1], tz[q] - v[2], v + 3, acc[q]);
      }
    }
    __syncthreads();  // the source tile is no longer read: reuse it for the group reduction
    double* red = reinterpret_cast<double*>(sh2);
    if (g < G)
#pragma unroll
      for (int q = 0; q < TPT; ++q)
#pragma unroll
        for (int c = 0; c < NC; ++c) red[((g * TPT + q) * nsl + sl) * NC + c] = acc[q][c];
    __syncthreads();
    if (g == 0) {
#pragma unroll
      for (int q = 0; q < TPT; ++q) {
        const int lt = sbase + sl + q * nslot;
        if (lt >= nt) continue;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double r = 0.0;
          for (int gg = 0; gg < G; ++gg) r += red[((gg * TPT + q) * nsl + sl) * NC + c];
          part[(size_t)(it.out_off + lt) * NC + c] = r;
        }
      }
    }
    __syncthreads();
  }
}

template <P2PKind K>
void launch_p2p_t(const TreeDev& S, const TreeDev& T, const P2PItem* items, int n_items,
                  const int* p2p_src, int max_src, const double* w, double* part, cudaStream_t st,
                  const int* order) {
  constexpr int NPL = SrcPlanes<P2PTraits<K>::NW>::N;
  // shared memory: the staged sources, or the group reduction (threads * TPT * comps)
  const size_t smem = std::max((size_t)max_src * NPL * sizeof(double2),
                               (size_t)P2P_THREADS * P2PTraits<K>::TPT * P2PTraits<K>::NC * sizeof(double));
  FMM_REQUIRE(smem <= 227 * 1024, "P2P: source slice too large for shared memory");
  FMM_CUDA(cudaFuncSetAttribute(k_p2p<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (n_items)
    k_p2p<K><<<n_items, P2P_THREADS, smem, st>>>(S, T, items, order, p2p_src, max_src, w, part);
  FMM_LAUNCH_CHECK();
}

void launch_p2p(P2PKind kind, const TreeDev& S, const TreeDev& T, const P2PItem* items,
                int n_items, const int* p2p_src, int max_sources, const double* w, double* part,
                cudaStream_t st, const int* order) {
  const int ms = std::max(max_sources, 1);
  switch (kind) {
    case P2PKind::LAP_Q: return launch_p2p_t<P2PKind::LAP_Q>(S, T, items, n_items, p2p_src, ms, w, part, st, order);
    case P2PKind::LAP_D: return launch_p2p_t<P2PKind::LAP_D>(S, T, items, n_items, p2p_src, ms, w, part, st, order);
    case P2PKind::STOKESLET: return launch_p2p_t<P2PKind::STOKESLET>(S, T, items, n_items, p2p_src, ms, w, part, st, order);
    case P2PKind::STRESSLET: return launch_p2p_t<P2PKind::STRESSLET>(S, T, items, n_items, p2p_src, ms, w, part, st, order);
  }
}

// ----------------------------------------------------- generic channel forms (FmmPlan API)
template <int C, bool HQ, bool HD, bool GRAD>
__global__ void k_p2p_channels(TreeDev S, TreeDev T, const int* tleaves, const int* row,
                               const int* srcl, const double* __restrict__ q,
                               const double* __restrict__ d, double* pot, double* grad) {
  const int leaf = tleaves[blockIdx.x];
  const int t0 = T.body_start[leaf], nt = T.body_count[leaf];
  const int64_t ns = S.n_points, ntot = T.n_points;
  for (int lt = threadIdx.x; lt < nt; lt += blockDim.x) {
    const int ti = t0 + lt;
    const double tx = T.px[ti], ty = T.py[ti], tz = T.pz[ti];
    double ap[C], ag[C][3];
#pragma unroll
    for (int c = 0; c < C; ++c) { ap[c] = 0; ag[c][0] = ag[c][1] = ag[c][2] = 0; }
    for (int e = row[leaf]; e < row[leaf + 1]; ++e) {
      const int sl = srcl[e];
      const int s0 = S.body_start[sl], sn = S.body_count[sl];
      for (int j = s0; j < s0 + sn; ++j) {
        const double rx = tx - S.px[j], ry = ty - S.py[j], rz = tz - S.pz[j];
        const double d2 = rx * rx + ry * ry + rz * rz;
        if (!(d2 > 0.0)) continue;
        const double inv = 1.0 / sqrt(d2);
        const double inv3 = inv * inv * inv;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if (HQ) {
            const double qq = q[c * ns + j];
            ap[c] += qq * inv;
            if (GRAD) {
              ag[c][0] -= qq * rx * inv3;
              ag[c][1] -= qq * ry * inv3;
              ag[c][2] -= qq * rz * inv3;
            }
          }
          if (HD) {
            const double* dd = d + (c * ns + j) * 3;
            const double rn = rx * dd[0] + ry * dd[1] + rz * dd[2];
            ap[c] += rn * inv3;
            if (GRAD) {
              const double f5 = 3.0 * rn * inv3 * inv * inv;
              ag[c][0] += dd[0] * inv3 - f5 * rx;
              ag[c][1] += dd[1] * inv3 - f5 * ry;
              ag[c][2] += dd[2] * inv3 - f5 * rz;
            }
          }
        }
      }
    }
    const int o = T.perm[ti];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      pot[c * ntot + o] += ap[c];
      if (GRAD)
        for (int k = 0; k < 3; ++k) grad[(c * ntot + o) * 3 + k] += ag[c][k];
    }
  }
}

template <int C, bool HQ, bool HD>
void p2p_channels_t(const TreeDev& S, const TreeDev& T, const Plan& plan, bool g, const double* q,
                    const double* d, double* pot, double* grad, cudaStream_t st) {
  const int n = plan.tgt.n_leaves;
  if (!n) return;
  if (g)
    k_p2p_channels<C, HQ, HD, true><<<n, 128, 0, st>>>(S, T, plan.tgt.leaves.get(), plan.p2p_row.get(),
                                                       plan.p2p_src.get(), q, d, pot, grad);
  else
    k_p2p_channels<C, HQ, HD, false><<<n, 128, 0, st>>>(S, T, plan.tgt.leaves.get(), plan.p2p_row.get(),
                                                        plan.p2p_src.get(), q, d, pot, grad);
  FMM_LAUNCH_CHECK();
}

void launch_p2p_channels(const TreeDev& S, const TreeDev& T, const Plan& plan, int C,
                         const double* q, const double* d, bool want_grad, double* pot,
                         double* grad, cudaStream_t st) {
  const bool hq = q != nullptr, hd = d != nullptr;
#define PC_CASE(CC)                                                                   \
  if (C == CC) {                                                                      \
    if (hq && hd) return p2p_channels_t<CC, true, true>(S, T, plan, want_grad, q, d, pot, grad, st); \
    if (hq) return p2p_channels_t<CC, true, false>(S, T, plan, want_grad, q, d, pot, grad, st);     \
    return p2p_channels_t<CC, false, true>(S, T, plan, want_grad, q, d, pot, grad, st);            \
  }
  PC_CASE(1)
  PC_CASE(4)
  PC_CASE(7)
#undef PC_CASE
  throw ArgumentError("near_field: unsupported channel count");
}

template <int C, bool GRAD>
__global__ void k_l2p_channels(TreeDev T, const int* leaves, int p, const double2* __restrict__ L,
                               double* pot, double* grad) {
  extern __shared__ double2 sL[];
  const int H = hcount(p);
  const int leaf = leaves[blockIdx.x];
  for (int i = threadIdx.x; i < C * H; i += blockDim.x) sL[i] = L[(size_t)leaf * C * H + i];
  __syncthreads();
  const int t0 = T.body_start[leaf], nt = T.body_count[leaf];
  const double cx = T.cx[leaf], cy = T.cy[leaf], cz = T.cz[leaf];
  const int64_t ntot = T.n_points;
  for (int lt = threadIdx.x; lt < nt; lt += blockDim.x) {
    const int ti = t0 + lt;
    double ph[C], gr[3 * C];
#pragma unroll
    for (int c = 0; c < C; ++c) { ph[c] = 0; gr[3 * c] = gr[3 * c + 1] = gr[3 * c + 2] = 0; }
    l2p_eval<C, GRAD>(sL, H, p, T.px[ti] - cx, T.py[ti] - cy, T.pz[ti] - cz, ph, gr, T.rec);
    const int o = T.perm[ti];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      pot[c * ntot + o] += ph[c];
      if (GRAD)
        for (int k = 0; k < 3; ++k) grad[(c * ntot + o) * 3 + k] += gr[3 * c + k];
    }
  }
}

void launch_l2p_channels(const TreeDev& T, const int* leaves, int n_leaves, int p, int C,
                         bool want_grad, const double2* L, double* pot, double* grad,
                         cudaStream_t st) {
  if (!n_leaves) return;
  const size_t smem = (size_t)C * hcount(p) * sizeof(double2);
#define L2P_CASE(CC)                                                                         \
  if (C == CC) {                                                                             \
    if (want_grad) {                                                                         \
      FMM_CUDA(cudaFuncSetAttribute(k_l2p_channels<CC, true>,                                \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
      k_l2p_channels<CC, true><<<n_leaves, 128, smem, st>>>(T, leaves, p, L, pot, grad);      \
    } else {                                                                                 \
      FMM_CUDA(cudaFuncSetAttribute(k_l2p_channels<CC, false>,                               \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
      k_l2p_channels<CC, false><<<n_leaves, 128, smem, st>>>(T, leaves, p, L, pot, grad);     \
    }                                                                                        \
    FMM_LAUNCH_CHECK();                                                                      \
    return;                                                                                  \
  }
  L2P_CASE(1)
  L2P_CASE(4)
  L2P_CASE(7)
#undef L2P_CASE
  throw ArgumentError("far_field: unsupported channel count");
}

}  // namespace fmmbem
