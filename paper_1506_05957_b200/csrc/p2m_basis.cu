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
#include <algorithm>

#include <string>
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

// The same sums with the leaf's channel scalars staged once in shared memory (the kernel above
// recomputes them for every coefficient: ~25 instructions per 16-byte table entry) and two
// coefficient rows per warp in flight, up to 4 entries per lane each.  Per-lane order and the
// lane reduction are those of k_p2m_basis, so the results are bit-identical.
template <int C>
__global__ void __launch_bounds__(256)
k_p2m_basis_st(const int* __restrict__ leaves, const int* __restrict__ body_start,
               const int* __restrict__ body_count, int64_t ns, int H, int kind,
               const double2* __restrict__ B, const int* __restrict__ s_panel,
               const double* __restrict__ x, const double* __restrict__ px,
               const double* __restrict__ py, const double* __restrict__ pz,
               double2* __restrict__ M, int max_nb) {
  extern __shared__ double p2m_ss[];  // [C][max_nb]
  const int leaf = leaves[blockIdx.x];
  const int b0 = body_start[leaf], nb = body_count[leaf];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    double s[C == 1 ? 1 : 4];
    basis_scalars<C>(kind, b0 + b, s_panel, x, px, py, pz, s);
#pragma unroll
    for (int c = 0; c < C; ++c) p2m_ss[c * max_nb + b] = s[c];
  }
  __syncthreads();
  constexpr int U = 4;  // entries per lane in flight per row
  for (int idx = warp; idx < H; idx += 2 * nw) {
    const int idx2 = idx + nw;
    const bool two = idx2 < H;
    double2 acc[2][C];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[r][c] = make_double2(0.0, 0.0);
    const double2* B0 = B + (size_t)idx * ns + b0;
    const double2* B1 = B + (size_t)(two ? idx2 : idx) * ns + b0;
    for (int bb = lane; bb < nb; bb += 32 * U) {
      double2 v0[U], v1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = bb + 32 * u;
        v0[u] = b < nb ? __ldg(B0 + b) : make_double2(0.0, 0.0);
        v1[u] = (two && b < nb) ? __ldg(B1 + b) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = bb + 32 * u;
        if (b < nb) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const double sc = p2m_ss[c * max_nb + b];
            acc[0][c].x = fma(sc, v0[u].x, acc[0][c].x);
            acc[0][c].y = fma(sc, v0[u].y, acc[0][c].y);
            acc[1][c].x = fma(sc, v1[u].x, acc[1][c].x);
            acc[1][c].y = fma(sc, v1[u].y, acc[1][c].y);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
        for (int o = 16; o > 0; o >>= 1) {
          acc[r][c].x += __shfl_xor_sync(0xffffffffu, acc[r][c].x, o);
          acc[r][c].y += __shfl_xor_sync(0xffffffffu, acc[r][c].y, o);
        }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        M[((size_t)leaf * C + c) * H + idx] = acc[0][c];
        if (two) M[((size_t)leaf * C + c) * H + idx2] = acc[1][c];
      }
    }
  }
}

// clustered entries (Laplace kinds, one channel), entry-major Bd[e][h]: work item
// (cell, entry range, slot): acc[h] = sum_e Bd[e][h] x[panel(e)], one thread per h;
// slot < 0 writes the cell's multipole, else a partial that k_p2m_reduce adds in order
// 4 warps split the item's (<= 32) entries, lanes run over h (NJ = ceil(H/32)
// per lane, every row load a coalesced 512 B), the warps' sums are added in
// warp order through shared memory.
constexpr int P2M_CHUNK = 64;
// direct upward pass only while it streams at most this many times the leaf table
// (cfg2: 3.1x, direct measured faster; cfg5: see DESIGN.md section 4)
constexpr double UPWARD_DIRECT_MAX_RATIO = 3.5;

template <int NJ>
__global__ void __launch_bounds__(128)
k_p2m_basis_cl(const int4* __restrict__ items, const int* __restrict__ red_of,
               const int4* __restrict__ reds, unsigned* arrive, int Hp, int H,
               const double2* __restrict__ B, const int* __restrict__ e_panel,
               const double* __restrict__ x, double2* __restrict__ M, double2* __restrict__ part) {
  __shared__ double sx[P2M_CHUNK];
  __shared__ double2 red[4][NJ * 32];
  const int4 it = items[blockIdx.x];
  const int len = it.z - it.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < len) sx[threadIdx.x] = __ldg(x + __ldg(e_panel + it.y + threadIdx.x));
  __syncthreads();
  double2 acc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j] = make_double2(0.0, 0.0);
  // batches of P2M_BATCH rows: all their loads are issued before the first use
  // (memory-level parallelism: the stream is latency-bound otherwise)
  constexpr int P2M_BATCH = 4;
#pragma unroll
  for (int k0 = 0; k0 < P2M_CHUNK / 4; k0 += P2M_BATCH) {
    double2 v[P2M_BATCH][NJ];
#pragma unroll
    for (int u = 0; u < P2M_BATCH; ++u) {
      const int e = warp + 4 * (k0 + u);
      const double2* row = B + (size_t)(it.y + min(e, len - 1)) * Hp;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int h = lane + 32 * j;
        v[u][j] = (e < len && h < H) ? __ldg(row + h) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < P2M_BATCH; ++u) {
      const int e = warp + 4 * (k0 + u);
      const double s = e < len ? sx[e] : 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        acc[j].x = fma(s, v[u][j].x, acc[j].x);
        acc[j].y = fma(s, v[u][j].y, acc[j].y);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) red[warp][lane + 32 * j] = acc[j];
  __syncthreads();
  double2* out = it.w < 0 ? M + (size_t)it.x * H : part + (size_t)it.w * H;
  for (int h = threadIdx.x; h < H; h += blockDim.x)
    out[h] = cadd(cadd(cadd(red[0][h], red[1][h]), red[2][h]), red[3][h]);
  if (it.w < 0) return;
  // a cell split over several items: the last one to finish adds the partials in slot order
  const int r = red_of[blockIdx.x];
  const int4 rc = reds[r];
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(arrive + r, 1u) == (unsigned)rc.z - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    double2 acc = __ldcg(part + (size_t)rc.y * H + h);
    for (int k = 1; k < rc.z; ++k) acc = cadd(acc, __ldcg(part + (size_t)(rc.y + k) * H + h));
    M[(size_t)rc.x * H + h] = acc;
  }
  if (threadIdx.x == 0) arrive[r] = 0u;
}

// The same stream through the TMA: one thread arms an mbarrier and issues bulk async copies of
// P2M_TMA_ROWS rows at a time into a two-deep shared-memory ring; the CTA's threads (one per
// coefficient column) accumulate the rows in entry order.  The copy engine generates the
// addresses, so the stream needs almost no issue slots -- it runs beside the persistent near
// field, whose warps otherwise starve a load-issuing kernel (basis stream 0.98 ms beside the
// near field with k_p2m_basis_cl).
#ifndef P2M_TMA_ROWS_N
#define P2M_TMA_ROWS_N 8
#endif
constexpr int P2M_TMA_ROWS = P2M_TMA_ROWS_N;

template <int NJ>
__global__ void __launch_bounds__(128)
k_p2m_basis_tma(const int4* __restrict__ items, const int* __restrict__ red_of,
                const int4* __restrict__ reds, unsigned* arrive, int Hp, int H,
                const double2* __restrict__ B, const int* __restrict__ e_panel,
                const double* __restrict__ x, double2* __restrict__ M, double2* __restrict__ part) {
  constexpr int R = P2M_TMA_ROWS;
  extern __shared__ __align__(128) unsigned char p2m_smem[];
  double2* buf = reinterpret_cast<double2*>(p2m_smem);  // [2][R][H]
  __shared__ double sx[P2M_CHUNK];
  __shared__ unsigned long long full[2];
  const int4 it = items[blockIdx.x];
  const int len = it.z - it.y, tid = threadIdx.x;
  if (tid < len) sx[tid] = __ldg(x + __ldg(e_panel + it.y + tid));
  if (tid == 0) {
    tma_bar_init(&full[0], 1);
    tma_bar_init(&full[1], 1);
    tma_bar_init_fence();
  }
  __syncthreads();
  const int nchunk = (len + R - 1) / R;
  auto issue = [&](int c) {  // (thread 0) chunk c into ring slot c & 1
    const int r0 = c * R, nr = min(R, len - r0);
    unsigned long long* bar = &full[c & 1];
    double2* dst = buf + (size_t)(c & 1) * R * H;
    const double2* src = B + (size_t)(it.y + r0) * Hp;
    tma_bar_expect(bar, (unsigned)(nr * H * sizeof(double2)));
    if (H == Hp) {
      tma_load_1d(dst, src, (unsigned)(nr * H * sizeof(double2)), bar);
    } else {
      for (int r = 0; r < nr; ++r)
        tma_load_1d(dst + (size_t)r * H, src + (size_t)r * Hp, (unsigned)(H * sizeof(double2)), bar);
    }
  };
  if (tid == 0) {
    issue(0);
    if (nchunk > 1) issue(1);
  }
  double2 acc[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j] = make_double2(0.0, 0.0);
  for (int c = 0; c < nchunk; ++c) {
    tma_bar_wait(&full[c & 1], (unsigned)(c >> 1) & 1u);
    const double2* b = buf + (size_t)(c & 1) * R * H;
    const int nr = min(R, len - c * R);
    for (int r = 0; r < nr; ++r) {
      const double s = sx[c * R + r];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int h = tid + 128 * j;
        if (h < H) {
          const double2 v = b[(size_t)r * H + h];
          acc[j].x = fma(s, v.x, acc[j].x);
          acc[j].y = fma(s, v.y, acc[j].y);
        }
      }
    }
    __syncthreads();  // the ring slot is consumed
    if (tid == 0 && c + 2 < nchunk) {
      tma_fence_proxy();
      issue(c + 2);
    }
  }
  double2* out = it.w < 0 ? M + (size_t)it.x * H : part + (size_t)it.w * H;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int h = tid + 128 * j;
    if (h < H) out[h] = acc[j];
  }
  if (it.w < 0) return;
  // a cell split over several items: the last one to finish adds the partials in slot order
  const int r = red_of[blockIdx.x];
  const int4 rc = reds[r];
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(arrive + r, 1u) == (unsigned)rc.z - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int h = tid; h < H; h += blockDim.x) {
    double2 a = __ldcg(part + (size_t)rc.y * H + h);
    for (int k = 1; k < rc.z; ++k) a = cadd(a, __ldcg(part + (size_t)(rc.y + k) * H + h));
    M[(size_t)rc.x * H + h] = a;
  }
  if (tid == 0) arrive[r] = 0u;
}

// Direct upward basis: entry e = (cell, cluster in the cell's subtree),
// Bd[e][h] = sum over the cluster's Gauss points (sorted order) of the kernel's
// P2M basis about the CELL's centre.  M2M of a regular-harmonic expansion is
// exact (degree j of the parent only needs degrees <= j of the child), so this
// is the multipole the M2M chain would produce, with no level dependencies.
__global__ void k_basis_build_entries(int ne, int ptab, int kind, const int* __restrict__ e_cell,
                                      const int* __restrict__ e_cluster, const int* __restrict__ cl_src,
                                      const double* __restrict__ px, const double* __restrict__ py,
                                      const double* __restrict__ pz, const double* __restrict__ cx,
                                      const double* __restrict__ cy, const double* __restrict__ cz,
                                      const double* __restrict__ s_w, const int* __restrict__ s_panel,
                                      const double* __restrict__ nrm, const double* __restrict__ rec,
                                      double2* __restrict__ B) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int cell = e_cell[e], cl = e_cluster[e];
  const int H = hcount(ptab);
  double2 R[hcount(P_MAX)], acc[hcount(P_MAX)];
  for (int h = 0; h < H; ++h) acc[h] = make_double2(0.0, 0.0);
  for (int i = cl_src[cl]; i < cl_src[cl + 1]; ++i) {
    regular_half(px[i] - cx[cell], py[i] - cy[cell], pz[i] - cz[cell], ptab, R, rec);
    const double w = s_w[i];
    if (kind != K_LAP_DOUBLE) {
      for (int h = 0; h < H; ++h) acc[h] = cadd(acc[h], cscale(R[h], w));
      continue;
    }
    const int pn = s_panel[i];
    const double dx = 0.5 * w * nrm[3 * pn], dy = 0.5 * w * nrm[3 * pn + 1], dz = w * nrm[3 * pn + 2];
    for (int n = 1; n <= ptab; ++n)
      for (int m = 0; m <= n; ++m) {
        double2 a = make_double2(0.0, 0.0);
        if (m + 1 <= n - 1) a = cfma(make_double2(dx, -dy), R[hidx(n - 1, m + 1)], a);
        if (m - 1 >= -(n - 1)) a = cfma(make_double2(-dx, -dy), hget(R, n - 1, m - 1), a);
        if (m <= n - 1) {
          const double2 r = R[hidx(n - 1, m)];
          a.x = fma(dz, r.x, a.x);
          a.y = fma(dz, r.y, a.y);
        }
        acc[hidx(n, m)] = cadd(acc[hidx(n, m)], a);
      }
  }
  for (int h = 0; h < H; ++h) B[(size_t)e * H + h] = acc[h];
}

}  // namespace

// work items over the entries of the given cells, <= P2M_CHUNK entries each
void set_p2m_items(BemOp& op, const std::vector<int>& cells, const std::vector<int>& range,
                   P2MItems& items, P2MItems& reduce, int& n_slots) {
  std::vector<int4> it, red;
  std::vector<int> red_of;
  int slot = 0;
  for (int c : cells) {
    const int e0 = range[2 * (size_t)c], e1 = range[2 * (size_t)c + 1], len = e1 - e0;
    const int nch = std::max(1, (len + P2M_CHUNK - 1) / P2M_CHUNK);
    if (nch == 1) {
      it.push_back(make_int4(c, e0, e1, -1));
      red_of.push_back(-1);
      continue;
    }
    red.push_back(make_int4(c, slot, nch, 0));
    for (int q = 0; q < nch; ++q) {
      it.push_back(make_int4(c, e0 + (int)((int64_t)len * q / nch), e0 + (int)((int64_t)len * (q + 1) / nch),
                             slot++));
      red_of.push_back((int)red.size() - 1);
    }
  }
  items.red_of.upload(red_of.empty() ? std::vector<int>(1, -1) : red_of);
  items.arrive.resize(std::max<size_t>(red.size(), 1));
  items.arrive.zero();
  items.n = (int)it.size();
  items.d.upload(it.empty() ? std::vector<int4>(1) : it);
  reduce.n = (int)red.size();
  reduce.d.upload(red.empty() ? std::vector<int4>(1) : red);
  n_slots = slot;
}

bool ensure_p2m_basis(BemOp& op, int p, cudaStream_t s) {
  if (op.basis_p >= p) return true;
  const int64_t ns = op.plan.src.n_points;
  // grow to the operator's largest useful order at once (prefix-compatible in p)
  const int ptab = std::max(p, std::min(P_MAX, std::max(op.basis_p, 12)));
  constexpr double BUDGET = 24e9;  // bytes of HBM this table may take
  if ((double)hcount(ptab) * ns * sizeof(double2) > BUDGET) return false;
  const Tree& S = op.plan.src;
  const bool cluster = op.basis_kind_for_sys == K_LAP_SINGLE || op.basis_kind_for_sys == K_LAP_DOUBLE;
  op.basis_clustered = cluster;
  if (!cluster) {
    op.p2m_basis.resize((size_t)hcount(ptab) * ns);
    k_basis_build<<<grid_for(ns, 128), 128, 0, s>>>(ns, ptab, op.basis_kind_for_sys, S.px.get(),
                                                    S.py.get(), S.pz.get(), S.leaf_of_body.get(),
                                                    S.cx.get(), S.cy.get(), S.cz.get(),
                                                    op.s_weight.get(), op.s_panel.get(),
                                                    op.normal.get(), S.rec, op.p2m_basis.get());
    FMM_LAUNCH_CHECK();
    op.basis_cols = (int)ns;
  } else {
    // clusters: maximal runs of sorted Gauss points with the same (leaf, panel)
    const std::vector<int> leaf = S.leaf_of_body.download(s), pan = op.s_panel.download(s);
    std::vector<int> src_begin, cpanel;
    for (int64_t i = 0; i < ns; ++i)
      if (i == 0 || leaf[i] != leaf[i - 1] || pan[i] != pan[i - 1]) {
        src_begin.push_back((int)i);
        cpanel.push_back(pan[i]);
      }
    src_begin.push_back((int)ns);
    // cells with a multipole: every M2L source and every leaf (the sharded path's P2M)
    const Plan& pl = op.plan;
    std::vector<char> need(S.n_cells, 0);
    for (int c : pl.h_m2l_src) need[c] = 1;
    for (int c = 0; c < S.n_cells; ++c)
      if (S.h_n_child[c] == 0) need[c] = 1;
    // entries of the direct table vs the leaf table: the direct pass streams every cluster once
    // per needed ancestor.  FMMBEM_UPWARD=direct|leaf overrides the choice.
    {
      auto count = [&](int c) {
        const int b0 = S.h_body_start[c], b1 = b0 + S.h_body_count[c];
        return (int64_t)(std::lower_bound(src_begin.begin(), src_begin.end(), b1) -
                         std::lower_bound(src_begin.begin(), src_begin.end(), b0));
      };
      int64_t e_direct = 0, e_leaf = 0;
      for (int c = 0; c < S.n_cells; ++c) {
        if (!need[c]) continue;
        const int64_t k = count(c);
        e_direct += k;
        if (S.h_n_child[c] == 0) e_leaf += k;
      }
      const char* env = std::getenv("FMMBEM_UPWARD");
      const bool leaf = env ? std::string(env) == "leaf"
                            : (double)e_direct > UPWARD_DIRECT_MAX_RATIO * (double)e_leaf;
      op.basis_leaf_only = leaf;
      if (leaf)
        for (int c = 0; c < S.n_cells; ++c) need[c] = S.h_n_child[c] == 0;
    }
    std::vector<int> cells, e_cell, e_cl, e_panel, range(2 * (size_t)S.n_cells, 0);
    for (int c = 0; c < S.n_cells; ++c) {
      if (!need[c]) continue;
      cells.push_back(c);
      const int b0 = S.h_body_start[c], b1 = b0 + S.h_body_count[c];
      const int k0 = (int)(std::lower_bound(src_begin.begin(), src_begin.end(), b0) - src_begin.begin());
      const int k1 = (int)(std::lower_bound(src_begin.begin(), src_begin.end(), b1) - src_begin.begin());
      range[2 * (size_t)c] = (int)e_cell.size();
      for (int k = k0; k < k1; ++k) {
        e_cell.push_back(c);
        e_cl.push_back(k);
        e_panel.push_back(cpanel[k]);
      }
      range[2 * (size_t)c + 1] = (int)e_cell.size();
    }
    const int ne = (int)e_cell.size();
    if ((double)hcount(ptab) * ne * sizeof(double2) > BUDGET) return false;
    DevBuf<int> d_src, d_cell, d_cl;
    d_src.upload(src_begin, s);
    d_cell.upload(e_cell, s);
    d_cl.upload(e_cl, s);
    op.cl_panel.upload(e_panel, s);
    op.h_cl_range = range;
    set_p2m_items(op, cells, range, op.p2m_items, op.p2m_reduce, op.n_p2m_slots);
    op.p2m_part.ensure((size_t)std::max(op.n_p2m_slots, 1) * hcount(P_MAX));
    op.p2m_leaf_list = nullptr;
    op.p2m_basis.resize((size_t)hcount(ptab) * ne);
    k_basis_build_entries<<<grid_for(ne, 64), 64, 0, s>>>(
        ne, ptab, op.basis_kind_for_sys, d_cell.get(), d_cl.get(), d_src.get(), S.px.get(),
        S.py.get(), S.pz.get(), S.cx.get(), S.cy.get(), S.cz.get(), op.s_weight.get(),
        op.s_panel.get(), op.normal.get(), S.rec, op.p2m_basis.get());
    FMM_LAUNCH_CHECK();
    op.basis_cols = ne;
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  FMM_CUDA(cudaStreamSynchronize(s));
  op.basis_p = ptab;
  return true;
}

// the work items of a shard's own leaves for the clustered basis (host data: call outside a
// stream capture, e.g. when the shard is set up)
void prepare_p2m_leaf_items(BemOp& op, const int* leaves, int n_leaves) {
  if (!op.basis_clustered || leaves == op.p2m_leaf_list) return;
  std::vector<int> lv(n_leaves);
  if (n_leaves)
    FMM_CUDA(cudaMemcpy(lv.data(), leaves, n_leaves * sizeof(int), cudaMemcpyDeviceToHost));
  set_p2m_items(op, lv, op.h_cl_range, op.p2m_leaf_items, op.p2m_leaf_reduce, op.n_p2m_leaf_slots);
  op.p2m_part.ensure((size_t)std::max(op.n_p2m_leaf_slots, 1) * hcount(P_MAX));
  op.p2m_leaf_list = leaves;
}

void launch_p2m_basis(BemOp& op, int p, int C, const double* x, double2* M, cudaStream_t s,
                      const int* leaves, int n_leaves) {
  const Tree& S = op.plan.src;
  const int H = hcount(p);
  if (op.basis_clustered) {
    FMM_REQUIRE(C == 1, "clustered P2M basis is single-channel");
    const bool direct = leaves == nullptr;  // all multipoles, else the given leaves
    if (!direct && leaves != op.p2m_leaf_list) prepare_p2m_leaf_items(op, leaves, n_leaves);
    const P2MItems& it = direct ? op.p2m_items : op.p2m_leaf_items;
    const P2MItems& red = direct ? op.p2m_reduce : op.p2m_leaf_reduce;
    FMM_REQUIRE(op.p2m_part.size() >= (size_t)std::max(op.n_p2m_slots, op.n_p2m_leaf_slots) * H,
                "P2M partial buffer not sized");
    // the TMA stream from 1 024 items up (small problems are latency-bound: the load-issuing
    // kernel starts faster, cfg1 18.5 k vs 17.9 k mat-vecs/s); FMMBEM_P2M=ldg | tma forces one
    static const int force = [] {
      const char* e = std::getenv("FMMBEM_P2M");
      return !e ? 0 : std::string(e) == "ldg" ? 1 : std::string(e) == "tma" ? 2 : 0;
    }();
    const bool use_tma = force == 2 || (force == 0 && it.n >= 1024);
    if (it.n && use_tma) {
      const int Hp = hcount(op.basis_p);
      const size_t smem = (size_t)2 * P2M_TMA_ROWS * H * sizeof(double2);
      static DeviceOnce attr;
      if (attr.first()) {
        FMM_CUDA(cudaFuncSetAttribute(k_p2m_basis_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        FMM_CUDA(cudaFuncSetAttribute(k_p2m_basis_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr.mark();
      }
      if (H <= 128)
        k_p2m_basis_tma<1><<<it.n, 128, smem, s>>>(it.d.get(), it.red_of.get(), red.d.get(), it.arrive.get(), Hp,
                                                   H, op.p2m_basis.get(), op.cl_panel.get(), x, M,
                                                   op.p2m_part.get());
      else
        k_p2m_basis_tma<2><<<it.n, 128, smem, s>>>(it.d.get(), it.red_of.get(), red.d.get(), it.arrive.get(), Hp,
                                                   H, op.p2m_basis.get(), op.cl_panel.get(), x, M,
                                                   op.p2m_part.get());
    } else if (it.n) {
      const int nj = (H + 31) / 32, Hp = hcount(op.basis_p);
#define P2M_CL(NJ)                                                                              \
  case NJ:                                                                                      \
    k_p2m_basis_cl<NJ><<<it.n, 128, 0, s>>>(it.d.get(), it.red_of.get(), red.d.get(),          \
                                            it.arrive.get(), Hp, H, op.p2m_basis.get(),         \
                                            op.cl_panel.get(), x, M, op.p2m_part.get());        \
    break;
      switch (nj) {
        P2M_CL(1) P2M_CL(2) P2M_CL(3) P2M_CL(4) P2M_CL(5) P2M_CL(6) P2M_CL(7) P2M_CL(8)
        default: FMM_REQUIRE(false, "P2M: order out of range");
      }
#undef P2M_CL
    }
  } else {
    if (!leaves) {
      leaves = S.leaves.get();
      n_leaves = S.n_leaves;
    }
    if (n_leaves <= 0) return;
    const int max_nb = std::max(S.max_leaf_count, 1);
    const size_t ss_bytes = (size_t)C * max_nb * sizeof(double);
    static const bool old_kernel = std::getenv("FMMBEM_P2M_BASIS") && std::string(std::getenv("FMMBEM_P2M_BASIS")) == "old";
    if (ss_bytes <= 48 * 1024 && !old_kernel) {
      if (C == 1)
        k_p2m_basis_st<1><<<n_leaves, 256, ss_bytes, s>>>(leaves, S.body_start.get(), S.body_count.get(), S.n_points,
                                                           H, op.basis_kind_for_sys, op.p2m_basis.get(),
                                                           op.s_panel.get(), x, S.px.get(), S.py.get(), S.pz.get(), M,
                                                           max_nb);
      else
        k_p2m_basis_st<4><<<n_leaves, 256, ss_bytes, s>>>(leaves, S.body_start.get(), S.body_count.get(), S.n_points,
                                                           H, op.basis_kind_for_sys, op.p2m_basis.get(),
                                                           op.s_panel.get(), x, S.px.get(), S.py.get(), S.pz.get(), M,
                                                           max_nb);
      FMM_LAUNCH_CHECK();
      return;
    }
    if (C == 1)
    k_p2m_basis<1><<<n_leaves, 256, 0, s>>>(leaves, S.body_start.get(), S.body_count.get(),
                                              S.n_points, H, op.basis_kind_for_sys,
                                              op.p2m_basis.get(), op.s_panel.get(), x, S.px.get(),
                                              S.py.get(), S.pz.get(), M);
  else
    k_p2m_basis<4><<<n_leaves, 256, 0, s>>>(leaves, S.body_start.get(), S.body_count.get(),
                                              S.n_points, H, op.basis_kind_for_sys,
                                              op.p2m_basis.get(), op.s_panel.get(), x, S.px.get(),
                                              S.py.get(), S.pz.get(), M);
  }
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmbem
