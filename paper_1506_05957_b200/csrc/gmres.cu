// Relaxed GMRES with the Krylov basis resident in HBM.
//
// Reference: solver.gmres (solver.py:69-134), RelaxationSchedule / schedule_p /
// relax_eps (solver.py:20-47).  Unrestarted, modified Gram-Schmidt Arnoldi and
// Givens rotations, residual estimate |g[k+1]| / ||b||, stop when < tol, then
// y = H^{-1} g and x = sum y_j v_j.  The mat-vec, the MGS dot/axpy sweeps, the
// norm and the basis update run on the device; the O(k) Givens/Hessenberg
// scalar work and the order schedule run on the host from one (k+2)-double
// read-back per iteration, which is also the only host synchronisation.
// Reductions are two-level with a fixed combination order (bitwise
// reproducible from run to run).
#include <cooperative_groups.h>

#include <cmath>

#include "operator.cuh"

namespace fmmbem {
namespace {

constexpr int RT = 256;   // threads per reduction block
constexpr int RB = 296;   // blocks (2 per SM)

__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

// finish: the last block to arrive adds the block partials (fixed assignment
// of partials to threads and a fixed reduction tree: deterministic)
__device__ void finish(double part, double* partials, unsigned* counter, double* out, bool do_sqrt,
                       double* sh, double* mbox = nullptr, unsigned long long* mflag = nullptr,
                       unsigned long long seq = 0) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = part;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) t += __ldcg(partials + b);
  t = block_sum(t, sh);
  if (threadIdx.x == 0) {
    *out = do_sqrt ? sqrt(t) : t;
    *counter = 0u;
    if (mbox) {
      mbox[0] = *out;
      __threadfence_system();
    }
    if (mflag) *reinterpret_cast<volatile unsigned long long*>(mflag) = seq;
  }
}

// w -= h_prev * v_prev (if v_prev); out = v . w      (solver.py:100-102)
__global__ void __launch_bounds__(RT) k_mgs(int64_t n, const double* __restrict__ v, double* w,
                                            const double* __restrict__ vprev, const double* hprev,
                                            double* partials, unsigned* counter, double* out) {
  __shared__ double sh[RT / 32];
  const double h = vprev ? *hprev : 0.0;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double wi = w[i];
    if (vprev) {
      wi = wi - h * vprev[i];
      w[i] = wi;
    }
    acc = fma(v[i], wi, acc);
  }
  finish(block_sum(acc, sh), partials, counter, out, false, sh);
}

// w -= h * v; out = ||w||    (solver.py:102-103)
__global__ void __launch_bounds__(RT) k_norm(int64_t n, double* w, const double* __restrict__ v,
                                             const double* hv, double* partials, unsigned* counter,
                                             double* out, double* mbox = nullptr,
                                             unsigned long long* mflag = nullptr,
                                             unsigned long long seq = 0) {
  __shared__ double sh[RT / 32];
  const double h = v ? *hv : 0.0;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double wi = w[i];
    if (v) {
      wi = wi - h * v[i];
      w[i] = wi;
    }
    acc = fma(wi, wi, acc);
  }
  finish(block_sum(acc, sh), partials, counter, out, true, sh, mbox, mflag, seq);
}

// v = w / h (or zeros on breakdown)    (solver.py:104-107)
__global__ void k_normalize(int64_t n, double* w, const double* h) {
  const double d = *h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = d > 0.0 ? w[i] / d : 0.0;
}

// x = sum_j y_j v_j in basis order    (solver.py:130-133)
__global__ void k_combine(int64_t n, int m, const double* __restrict__ V, const double* __restrict__ y,
                          double* x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc += y[j] * V[(size_t)j * n + i];
    x[i] = acc;
  }
}

__global__ void k_scale(int64_t n, const double* b, const double* nb, double* v, double* v2) {
  const double d = *nb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = v2[i] = d > 0.0 ? b[i] / d : 0.0;  // (b = 0: the host returns x = 0 after the first column)
}

// One Arnoldi step in a single cooperative launch (grid-wide barriers between
// the MGS sweeps): for j = 0..k, w -= h_{j-1} v_{j-1} fused with h_j = v_j . w;
// then w -= h_k v_k, h_{k+1} = ||w||, v_{k+1} = w / h_{k+1}.  Block partials
// are written per sweep and every block adds them in the same fixed order,
// so all blocks hold bitwise the same h_j.
constexpr int AB = 148;  // blocks (one per SM)

__device__ double grid_total(double part, double* partials, double* sh) {
  namespace cg = cooperative_groups;
  if (threadIdx.x == 0) partials[blockIdx.x] = part;
  cg::this_grid().sync();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) t += __ldcg(partials + b);
  t = block_sum(t, sh);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = t;
  __syncthreads();
  return bc;
}

// (w0: the mat-vec result, read in the first sweep; w: the new basis vector;
// xnext: a second copy of it, the next mat-vec's input)
__global__ void __launch_bounds__(RT) k_arnoldi(int64_t n, int k, const double* __restrict__ V,
                                                const double* __restrict__ w0, double* w,
                                                double* xnext, double* partials, double* hd,
                                                double* mbox, unsigned long long* mflag,
                                                unsigned long long seq) {
  __shared__ double sh[RT / 32];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double h = 0.0;
  for (int j = 0; j <= k + 1; ++j) {
    const double* vprev = j ? V + (size_t)(j - 1) * n : nullptr;
    const double* v = j <= k ? V + (size_t)j * n : nullptr;
    double acc = 0.0;
    for (int64_t i = i0; i < n; i += stride) {
      double wi = j ? w[i] : w0[i];
      if (vprev) wi = wi - h * vprev[i];
      if (!j || vprev) w[i] = wi;
      acc = v ? fma(v[i], wi, acc) : fma(wi, wi, acc);
    }
    // alternate two partial arrays so a fast block cannot overwrite a slow block's read
    h = grid_total(block_sum(acc, sh), partials + (j & 1) * gridDim.x, sh);
    if (j > k) h = sqrt(h);
    if (i0 == 0) {
      hd[j] = h;
      mbox[j] = h;
    }
  }
  if (i0 == 0) {  // the column is complete: post it to the host
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(mflag) = seq;
  }
  for (int64_t i = i0; i < n; i += stride) w[i] = xnext[i] = h > 0.0 ? w[i] / h : 0.0;
}

// The grid-wide step with w held in registers (GE elements per thread) and the next basis
// vector prefetched before each grid barrier: a sweep reads v_j once instead of reading v_j
// and reading + writing w (n up to AB * GT * GE).
constexpr int GT = 512;  // threads per CTA

template <int GE>
__global__ void __launch_bounds__(GT) k_arnoldi_reg(int64_t n, int k, const double* __restrict__ V,
                                                    const double* __restrict__ w0, double* w,
                                                    double* xnext, double* partials, double* hd,
                                                    double* mbox, unsigned long long* mflag,
                                                    unsigned long long seq) {
  __shared__ double sh[GT / 32];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double wr[GE], vc[GE], vn[GE];
#pragma unroll
  for (int e = 0; e < GE; ++e) {
    const int64_t i = i0 + e * stride;
    wr[e] = i < n ? w0[i] : 0.0;
    vn[e] = i < n ? V[i] : 0.0;
  }
  double h = 0.0;
  for (int j = 0; j <= k + 1; ++j) {
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < GE; ++e) {
      if (j) wr[e] = fma(-h, vc[e], wr[e]);  // w -= h_{j-1} v_{j-1}
      vc[e] = vn[e];
    }
    if (j + 1 <= k) {
#pragma unroll
      for (int e = 0; e < GE; ++e) {
        const int64_t i = i0 + e * stride;
        vn[e] = i < n ? V[(size_t)(j + 1) * n + i] : 0.0;
      }
    }
#pragma unroll
    for (int e = 0; e < GE; ++e) acc = j <= k ? fma(vc[e], wr[e], acc) : fma(wr[e], wr[e], acc);
    h = grid_total(block_sum(acc, sh), partials + (j & 1) * gridDim.x, sh);
    if (j > k) h = sqrt(h);
    if (i0 == 0) {
      hd[j] = h;
      mbox[j] = h;
    }
  }
  if (i0 == 0) {  // the column is complete: post it to the host
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(mflag) = seq;
  }
#pragma unroll
  for (int e = 0; e < GE; ++e) {
    const int64_t i = i0 + e * stride;
    if (i < n) w[i] = xnext[i] = h > 0.0 ? wr[e] / h : 0.0;
  }
}

// The same Arnoldi step for n <= ACL * ACT * AE on one thread-block cluster: w stays in
// registers (AE elements per thread), each sweep's CTA partials are exchanged through
// distributed shared memory and added in rank order by every CTA (bitwise-identical h_j),
// so a sweep costs one cluster barrier instead of a grid-wide one.
constexpr int ACL = 8;     // CTAs per cluster (portable size)
constexpr int ACT = 1024;  // threads per CTA
constexpr int AE = 4;      // elements per thread: n <= 32 768

__global__ void __launch_bounds__(ACT) k_arnoldi_cluster(int n, int k, const double* __restrict__ V,
                                                         const double* __restrict__ w0, double* w,
                                                         double* xnext, double* hd, double* mbox,
                                                         unsigned long long* mflag,
                                                         unsigned long long seq) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double sh[ACT / 32];
  __shared__ double part[2 * ACL];
  const int rank = (int)cluster.block_rank();
  const int t = rank * ACT + threadIdx.x;  // element t + e * ACL * ACT
  // registers: w, the current basis vector v_j (v_{j-1} of the next sweep) and v_{j+1},
  // prefetched before the sweep's cluster barrier
  double wr[AE], vc[AE], vn[AE];
#pragma unroll
  for (int e = 0; e < AE; ++e) {
    const int i = t + e * ACL * ACT;
    wr[e] = i < n ? w0[i] : 0.0;
    vn[e] = i < n ? V[i] : 0.0;
  }
  double h = 0.0;
  for (int j = 0; j <= k + 1; ++j) {
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < AE; ++e) {
      if (j) wr[e] = fma(-h, vc[e], wr[e]);  // w -= h_{j-1} v_{j-1}
      vc[e] = vn[e];
    }
    if (j + 1 <= k) {
#pragma unroll
      for (int e = 0; e < AE; ++e) {
        const int i = t + e * ACL * ACT;
        vn[e] = i < n ? V[(size_t)(j + 1) * n + i] : 0.0;
      }
    }
#pragma unroll
    for (int e = 0; e < AE; ++e) acc = j <= k ? fma(vc[e], wr[e], acc) : fma(wr[e], wr[e], acc);
    const double bs = block_sum(acc, sh);
    // push this CTA's partial into every CTA's slot [j & 1][rank] (remote stores are
    // posted; the barrier's release/acquire makes them visible), then read locally
    if (threadIdx.x == 0)  // (block_sum's total lives in thread 0)
#pragma unroll
      for (int r = 0; r < ACL; ++r) *cluster.map_shared_rank(part + (j & 1) * ACL + rank, r) = bs;
    cluster.sync();
    double tot = 0.0;
#pragma unroll
    for (int r = 0; r < ACL; ++r) tot += part[(j & 1) * ACL + r];
    h = j > k ? sqrt(tot) : tot;
    if (t == 0) {
      hd[j] = h;
      mbox[j] = h;
    }
  }
  if (t == 0) {  // the column is complete: post it to the host
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(mflag) = seq;
  }
#pragma unroll
  for (int e = 0; e < AE; ++e) {
    const int i = t + e * ACL * ACT;
    if (i < n) w[i] = xnext[i] = h > 0.0 ? wr[e] / h : 0.0;
  }
  cluster.sync();  // no CTA may exit while others still read its shared memory
}

// ||b|| on one cluster (n <= ACL * ACT * AE): written to the device scalar and posted to the
// host mailbox slot, read by the host together with the first Arnoldi column
__global__ void __launch_bounds__(ACT) k_norm_cluster(int n, const double* __restrict__ b, double* out,
                                                      double* mbox, double* v, double* v2) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double sh[ACT / 32];
  __shared__ double part[ACL];
  const int rank = (int)cluster.block_rank();
  const int t = rank * ACT + threadIdx.x;
  double br[AE];
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < AE; ++e) {
    const int i = t + e * ACL * ACT;
    br[e] = i < n ? b[i] : 0.0;
    acc = fma(br[e], br[e], acc);
  }
  const double bs = block_sum(acc, sh);
  if (threadIdx.x == 0)
#pragma unroll
    for (int r = 0; r < ACL; ++r) *cluster.map_shared_rank(part + rank, r) = bs;
  cluster.sync();
  double tot = 0.0;
#pragma unroll
  for (int r = 0; r < ACL; ++r) tot += part[r];
  const double nb = sqrt(tot);
  if (t == 0) {
    *out = mbox[0] = nb;
    __threadfence_system();
  }
  // v_0 = b / ||b|| (and the first mat-vec's input), as k_scale (b = 0: zeros)
#pragma unroll
  for (int e = 0; e < AE; ++e) {
    const int i = t + e * ACL * ACT;
    if (i < n) v[i] = v2[i] = nb > 0.0 ? br[e] / nb : 0.0;
  }
}

double relax_eps(double r, double eta) { return std::min(eta / std::min(std::max(r, eta), 1.0), 1.0); }

int schedule_p(double r, double eta, int p_initial, int p_min) {
  const double eps = relax_eps(r, eta);
  const int p = eps < 1.0 ? (int)std::ceil(-std::log2(eps)) : p_min;
  return std::min(p_initial, std::max(p_min, p));
}


// ---- partitioned GMRES (a real shard, one process per GPU) ----------------
// Each rank keeps only its own rows of the Krylov vectors (sorted target order, as the sharded
// epilogue writes them).  Per iteration: all-gather of v_k into the apply's input, the apply
// (own rows of w), classical Gram-Schmidt with one re-orthogonalisation (CGS2: two batched
// all-reduces of k+1 local dot products, then one of ||w||^2), and the same Givens update on
// every rank (bitwise-equal H after the all-reduces).  CGS2 replaces the reference's MGS
// (solver.py:100-103) by an algebraically equal, roundoff-level different sweep.
constexpr int SB = 256, SG = 2 * 148;  // threads / blocks of the partitioned vector kernels

__device__ double block_sum_sb(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < SB / 32; ++i) t += sh[i];
  __syncthreads();
  return t;
}

// part[j * SG + block] = partial dot of V_j and w (grid (SG, k1))
__global__ void __launch_bounds__(SB) k_sh_dots(int64_t n, const double* __restrict__ V,
                                                const double* __restrict__ w, double* __restrict__ part) {
  __shared__ double sh[SB / 32];
  const int j = blockIdx.y;
  const double* v = V + (size_t)j * n;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)SB + threadIdx.x; i < n; i += (int64_t)SG * SB)
    acc = fma(v[i], w[i], acc);
  acc = block_sum_sb(acc, sh);
  if (threadIdx.x == 0) part[(size_t)j * SG + blockIdx.x] = acc;
}

// h[j] = sum of the partials in block order (fixed: identical on every call)
__global__ void k_sh_finish(int k1, const double* __restrict__ part, double* __restrict__ h) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k1) return;
  double t = 0.0;
  for (int b = 0; b < SG; ++b) t += part[(size_t)j * SG + b];
  h[j] = t;
}

// w -= sum_j h_j V_j
__global__ void k_sh_update(int64_t n, int k1, const double* __restrict__ V, const double* __restrict__ h,
                            double* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = w[i];
    for (int j = 0; j < k1; ++j) acc = fma(-h[j], V[(size_t)j * n + i], acc);
    w[i] = acc;
  }
}

__global__ void k_sh_scale(int64_t n, const double* __restrict__ w, double inv, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = w[i] * inv;
}

GmresResult op_gmres_sharded(BemOp& op, const double* b, double tol, double eta, int p_initial,
                             int p_min, bool relaxed, int max_iter, double* x, GmresCallback cb,
                             void* user) {
  ShardWork& sw = op.shard;
  GmresResult res;
  cudaStream_t s = op.s_main;
  const int nc = op.formulation == STOKES ? 3 : 1;
  const int64_t nl = (int64_t)(sw.tbody_b - sw.tbody_a) * nc;  // own rows
  const int64_t nv = std::max<int64_t>(nl, 1);
  DevBuf<double>& V = op.g_basis;
  V.ensure((size_t)(max_iter + 2) * nv);
  DevBuf<double>& part = op.g_partials;
  part.ensure((size_t)SG * (max_iter + 1));
  DevBuf<double>& scal = op.g_scal;
  scal.ensure(2 * (size_t)(max_iter + 2));
  double* h1 = scal.get();
  double* h2 = scal.get() + (max_iter + 2);
  double* w = V.get() + (size_t)(max_iter + 1) * nv;  // scratch column
  auto dots = [&](const double* Vb, int k1, const double* vec, double* h) {
    if (nl > 0) k_sh_dots<<<dim3(SG, k1), SB, 0, s>>>(nl, Vb, vec, part.get());
    else FMM_CUDA(cudaMemsetAsync(part.get(), 0, (size_t)SG * k1 * sizeof(double), s));
    k_sh_finish<<<grid_for(k1, 128), 128, 0, s>>>(k1, part.get(), h);
    FMM_LAUNCH_CHECK();
    shard_allreduce(op, h, k1, s);
  };
  auto read = [&](const double* d, int k1, double* hst) {
    FMM_CUDA(cudaMemcpyAsync(hst, d, k1 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  };
  // own rows of b, ||b||
  shard_pack_rows(op, nc, b, w, s);
  double nb2 = 0.0;
  dots(w, 1, w, h1);
  read(h1, 1, &nb2);
  const double norm_b = std::sqrt(nb2);
  if (norm_b == 0.0 || max_iter == 0) {
    FMM_CUDA(cudaMemsetAsync(x, 0, op.n * sizeof(double), s));
    FMM_CUDA(cudaStreamSynchronize(s));
    res.converged = norm_b == 0.0;
    return res;
  }
  k_sh_scale<<<RB, RT, 0, s>>>(nl, w, 1.0 / norm_b, V.get());
  FMM_LAUNCH_CHECK();
  std::vector<double> H((size_t)(max_iter + 1) * max_iter, 0.0);
  auto Hat = [&](int i, int j) -> double& { return H[(size_t)i * max_iter + j]; };
  std::vector<double> cs(max_iter), sn(max_iter), g(max_iter + 1, 0.0), ha(max_iter + 1), hb(max_iter + 1);
  g[0] = norm_b;
  double residual = 1.0;
  int prev_p = p_initial;
  sw.local_vectors = true;
  try {
    for (int k = 0; k < max_iter; ++k) {
      const int p = relaxed ? std::min(schedule_p(residual, eta, p_initial, p_min), prev_p) : p_initial;
      prev_p = p;
      const double* vk = V.get() + (size_t)k * nv;
      double* vk1 = V.get() + (size_t)(k + 1) * nv;
      // all-gather v_k into the apply's (panel-order) input; the apply leaves w's own rows in ysend
      shard_gather_rows(op, nc, vk, op.x_in.get(), s);
      op_apply_device(op, nullptr, nullptr, p);
      if (nl > 0)
        FMM_CUDA(cudaMemcpyAsync(w, sw.ysend.get(), nl * sizeof(double), cudaMemcpyDeviceToDevice, s));
      // CGS2
      dots(V.get(), k + 1, w, h1);
      k_sh_update<<<RB, RT, 0, s>>>(nl, k + 1, V.get(), h1, w);
      dots(V.get(), k + 1, w, h2);
      k_sh_update<<<RB, RT, 0, s>>>(nl, k + 1, V.get(), h2, w);
      double ww = 0.0;
      dots(w, 1, w, h2 + k + 1);
      read(h1, k + 1, ha.data());
      read(h2, k + 2, hb.data());
      ww = hb[k + 1];
      const double hk1 = std::sqrt(ww);
      k_sh_scale<<<RB, RT, 0, s>>>(nl, w, hk1 > 0.0 ? 1.0 / hk1 : 0.0, vk1);
      FMM_LAUNCH_CHECK();
      op.kernel_launches += 8;
      for (int j = 0; j <= k; ++j) Hat(j, k) = ha[j] + hb[j];
      Hat(k + 1, k) = hk1;
      for (int j = 0; j < k; ++j) {
        const double t1 = cs[j] * Hat(j, k) + sn[j] * Hat(j + 1, k);
        Hat(j + 1, k) = -sn[j] * Hat(j, k) + cs[j] * Hat(j + 1, k);
        Hat(j, k) = t1;
      }
      const double denom = std::hypot(Hat(k, k), Hat(k + 1, k));
      cs[k] = Hat(k, k) / denom;
      sn[k] = Hat(k + 1, k) / denom;
      Hat(k, k) = denom;
      Hat(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      residual = std::fabs(g[k + 1]) / norm_b;
      res.residuals.push_back(residual);
      res.orders.push_back(p);
      if (cb && cb(k + 1, residual, p, user) != 0) {
        res.stopped = true;
        break;
      }
      if (residual < tol) {
        res.converged = true;
        break;
      }
    }
  } catch (...) {
    sw.local_vectors = false;
    throw;
  }
  sw.local_vectors = false;
  const int m = (int)res.orders.size();
  std::vector<double> y(std::max(m, 1), 0.0);
  for (int i = m - 1; i >= 0; --i) {
    double t = g[i];
    for (int j = i + 1; j < m; ++j) t -= Hat(i, j) * y[j];
    y[i] = t / Hat(i, i);
  }
  DevBuf<double>& yd = op.g_y;
  yd.upload(y, s);
  k_combine<<<RB, RT, 0, s>>>(nl, m, V.get(), yd.get(), w);
  FMM_LAUNCH_CHECK();
  shard_gather_rows(op, nc, w, x, s);  // every rank returns the whole solution
  op.kernel_launches += 2;
  return res;
}
}  // namespace

GmresResult op_gmres(BemOp& op, const double* b, double tol, double eta, int p_initial, int p_min,
                     bool relaxed, int max_iter, double* x, GmresCallback cb, void* user) {
  // eta drives the order (RelaxationSchedule.order, solver.py:41-47), tol the stop test (:124)
  FMM_REQUIRE(eta > 0.0, "eta must be positive");
  FMM_REQUIRE(max_iter >= 0, "max_iter must be >= 0");
  FMM_REQUIRE(p_initial >= 0 && p_initial <= P_MAX, "p_initial must be in [0, 20]");
  FMM_REQUIRE(!(op.shard.active && op.shard.virtual_mode),
              "GMRES needs full mat-vecs: a virtual shard only computes its own rows");
  FMM_REQUIRE(max_iter >= 0, "max_iter must be >= 0");
  if (op.shard.active)
    return op_gmres_sharded(op, b, tol, eta, p_initial, p_min, relaxed, max_iter, x, cb, user);
  GmresResult res;
  const int64_t n = op.n;
  cudaStream_t s = op.s_main;
  // workspaces live in the operator (grow-only): no allocation inside a solve
  DevBuf<double>& partials = op.g_partials;
  DevBuf<double>& scal = op.g_scal;
  DevBuf<unsigned>& counter = op.g_counter;
  partials.ensure(std::max(RB, 2 * AB));
  scal.ensure(max_iter + 3);
  if (!counter.size()) {
    counter.ensure(1);
    counter.zero(s);
  }
  if (op.mbox_cap < max_iter + 3) {
    if (op.mbox_h) FMM_CUDA(cudaFreeHost(op.mbox_h));
    op.mbox_cap = max_iter + 3;
    FMM_CUDA(cudaHostAlloc(&op.mbox_h, op.mbox_cap * sizeof(double), cudaHostAllocMapped));
    FMM_CUDA(cudaHostGetDevicePointer((void**)&op.mbox_d, op.mbox_h, 0));
  }
  if (!op.mflag_h) {
    FMM_CUDA(cudaHostAlloc(&op.mflag_h, sizeof(unsigned long long), cudaHostAllocMapped));
    FMM_CUDA(cudaHostGetDevicePointer((void**)&op.mflag_d, op.mflag_h, 0));
    *op.mflag_h = op.mbox_seq;
  }
  // wait for the kernel that posts sequence `seq` (spin on pinned memory; a
  // failed stream surfaces through cudaStreamQuery)
  auto wait_post = [&](unsigned long long seq) {
    const volatile unsigned long long* f = op.mflag_h;
    for (long spins = 0; *f != seq; ++spins) {
      if ((spins & 1023) == 1023) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e != cudaSuccess && e != cudaErrorNotReady) FMM_CUDA(e);
        if (e == cudaSuccess && *f != seq) throw CudaFailure("GMRES mailbox: stream idle without a post");
      }
    }
  };
  // ||b||: device scalar for k_scale, and mailbox slot max_iter + 2 for the host, read with the
  // first Arnoldi column (no round trip before the first mat-vec)
  double* nb = scal.get() + max_iter + 2;
  double* nb_box = op.mbox_d + max_iter + 2;
  auto cluster_cfg = [&](cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ACL);
    cfg.blockDim = dim3(ACT);
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ACL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
  };
  DevBuf<double>& V = op.g_basis;
  V.ensure((size_t)(max_iter + 1) * n);
  bool fused_scale = false;  // the cluster norm also writes v_0 (k_scale otherwise)
  if (n <= (int64_t)ACL * ACT * AE) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = cluster_cfg(at);
    FMM_CUDA(cudaLaunchKernelEx(&cfg, k_norm_cluster, (int)n, b, nb, nb_box, V.get(), op.x_in.get()));
    fused_scale = true;
  } else {
    k_norm<<<RB, RT, 0, s>>>(n, const_cast<double*>(b), nullptr, nullptr, partials.get(), counter.get(), nb,
                             nb_box, nullptr, 0);
  }
  FMM_LAUNCH_CHECK();
  op.kernel_launches += 1;
  double norm_b = -1.0;  // known after the first column
  auto read_norm_b = [&]() {
    norm_b = op.mbox_h[max_iter + 2];
    if (norm_b == 0.0) {
      FMM_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
      FMM_CUDA(cudaStreamSynchronize(s));
      res.converged = true;
      return true;
    }
    return false;
  };
  if (max_iter == 0) {
    FMM_CUDA(cudaStreamSynchronize(s));
    if (read_norm_b()) return res;
  }
  if (!fused_scale) {
    k_scale<<<RB, RT, 0, s>>>(n, b, nb, V.get(), op.x_in.get());
    op.kernel_launches += 1;
  }
  std::vector<double> H((size_t)(max_iter + 1) * std::max(max_iter, 1), 0.0);
  auto Hat = [&](int i, int j) -> double& { return H[(size_t)i * max_iter + j]; };
  std::vector<double> cs(max_iter), sn(max_iter), g(max_iter + 1, 0.0), hcol(max_iter + 2);
  if (norm_b > 0.0) g[0] = norm_b;
  double residual = 1.0;
  int prev_p = p_initial;
  double* hd = scal.get();  // H column k on device: hd[0..k+1]
  for (int k = 0; k < max_iter; ++k) {
    int p = relaxed ? std::min(schedule_p(residual, eta, p_initial, p_min), prev_p) : p_initial;
    prev_p = p;
    double* w = V.get() + (size_t)(k + 1) * n;
    op_apply_device(op, nullptr, nullptr, p);  // x_in holds v_k (k_scale / k_arnoldi)
    {
      const double* Vc = V.get();
      double* pp = partials.get();
      int kk = k;
      int64_t nn = n;
      double* mb = op.mbox_d;
      unsigned long long* mf = op.mflag_d;
      unsigned long long sq = ++op.mbox_seq;
      const double* w0 = op.y_out.get();
      double* xn = op.x_in.get();
      if (n <= (int64_t)ACL * ACT * AE) {
        cudaLaunchAttribute at[1];
        cudaLaunchConfig_t cfg = cluster_cfg(at);
        FMM_CUDA(cudaLaunchKernelEx(&cfg, k_arnoldi_cluster, (int)n, kk, Vc, w0, w, xn, hd, mb, mf, sq));
      } else {
        void* args[] = {&nn, &kk, &Vc, &w0, &w, &xn, &pp, &hd, &mb, &mf, &sq};
        const int64_t cap = (int64_t)AB * GT;
        const void* kern = n <= cap ? (const void*)k_arnoldi_reg<1>
                         : n <= 2 * cap ? (const void*)k_arnoldi_reg<2>
                         : n <= 4 * cap ? (const void*)k_arnoldi_reg<4>
                         : n <= 8 * cap ? (const void*)k_arnoldi_reg<8> : nullptr;
        if (kern)
          FMM_CUDA(cudaLaunchCooperativeKernel(kern, dim3(AB), dim3(GT), args, 0, s));
        else
          FMM_CUDA(cudaLaunchCooperativeKernel((const void*)k_arnoldi, dim3(AB), dim3(RT), args, 0, s));
      }
    }
    FMM_LAUNCH_CHECK();
    op.kernel_launches += 1;
    wait_post(op.mbox_seq);
    if (k == 0) {
      if (read_norm_b()) return res;
      g[0] = norm_b;
    }
    for (int j = 0; j <= k + 1; ++j) hcol[j] = op.mbox_h[j];
    if (op.timing) {
      FMM_CUDA(cudaStreamSynchronize(s));
      op_collect_stage_times(op);
    }
    for (int j = 0; j <= k + 1; ++j) Hat(j, k) = hcol[j];
    for (int j = 0; j < k; ++j) {
      const double h1 = cs[j] * Hat(j, k) + sn[j] * Hat(j + 1, k);
      Hat(j + 1, k) = -sn[j] * Hat(j, k) + cs[j] * Hat(j + 1, k);
      Hat(j, k) = h1;
    }
    const double denom = std::hypot(Hat(k, k), Hat(k + 1, k));
    cs[k] = Hat(k, k) / denom;
    sn[k] = Hat(k + 1, k) / denom;
    Hat(k, k) = denom;
    Hat(k + 1, k) = 0.0;
    g[k + 1] = -sn[k] * g[k];
    g[k] = cs[k] * g[k];
    residual = std::fabs(g[k + 1]) / norm_b;
    res.residuals.push_back(residual);
    res.orders.push_back(p);
    if (cb && cb(k + 1, residual, p, user) != 0) {  // the caller asked to stop (e.g. it raised)
      res.stopped = true;
      break;
    }
    if (residual < tol) {
      res.converged = true;
      break;
    }
  }
  const int m = (int)res.orders.size();
  // back substitution on the triangular H[:m,:m] (np.linalg.solve in the reference)
  std::vector<double> y(std::max(m, 1), 0.0);
  for (int i = m - 1; i >= 0; --i) {
    double t = g[i];
    for (int j = i + 1; j < m; ++j) t -= Hat(i, j) * y[j];
    y[i] = t / Hat(i, i);
  }
  DevBuf<double>& yd = op.g_y;
  yd.ensure(y.size());
  if (op.ypin_cap < (int)y.size()) {  // pinned: the copy is truly asynchronous
    if (op.ypin_h) FMM_CUDA(cudaFreeHost(op.ypin_h));
    op.ypin_cap = std::max((int)y.size(), max_iter);
    FMM_CUDA(cudaHostAlloc(&op.ypin_h, op.ypin_cap * sizeof(double), cudaHostAllocDefault));
  }
  std::copy(y.begin(), y.end(), op.ypin_h);
  FMM_CUDA(cudaMemcpyAsync(yd.get(), op.ypin_h, y.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  k_combine<<<RB, RT, 0, s>>>(n, m, V.get(), yd.get(), x);
  FMM_LAUNCH_CHECK();
  op.kernel_launches += 1;
  // x is complete in stream order on op.s_main; the callers (capi.cu) record their end event,
  // queue the D2H copy if any and synchronise once
  return res;
}

}  // namespace fmmbem
