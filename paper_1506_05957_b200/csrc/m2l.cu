// M2L on device: warp-per-(pair, channel) register-tiled contraction.
//
// Reference: FmmPlan._m2l_sweep (fmm.py:292-314) with the M2L gather map
// (harmonics.py:180-198):
//     L_j^k = (-1)^j sum_{n<=p} sum_{|m|<=n} M_n^m conj(I_{n+j}^{m+k}(D)),  D = c_t - c_s.
// The reference groups pairs by offset and runs one zgemm per group.  Here a
// work item is (target cell, slice of <= 16 of its interaction pairs); each
// warp of the CTA streams (pair, channel) units through its own shared-memory
// slot (the full I(D) grid of order 2p and the full-storage multipole) and
// accumulates in registers.  Lane l owns output column k and BJ consecutive
// rows j0..j0+BJ-1 (half storage: k <= j <= p).  For fixed m the I rows it
// needs, n+j0 .. n+j0+BJ-1, slide by one row per step in n, so every step is
// one new shared-memory load plus one broadcast M load for BJ complex FMAs
// (4 DFMA each); the window is rotated by unrolling, not by register moves.
// Items write partial L blocks that a second kernel adds per cell in item
// order: deterministic, no atomics.
#include "kernels.cuh"

namespace fmmbem {

constexpr int M2L_WARPS = 4;

// smallest tile height BJ whose tiles fit one warp
__host__ __device__ constexpr int m2l_tiles(int p, int bj) {
  int t = 0;
  for (int k = 0; k <= p; ++k) t += (p - k + 1 + bj - 1) / bj;
  return t;
}
__host__ __device__ constexpr int m2l_bj(int p) {
  int bj = 1;
  while (m2l_tiles(p, bj) > 32) ++bj;
  return bj;
}

// I_n^m(D) in FULL flat storage n^2+n+m for n <= order (setup)
__global__ void k_igrid_full(const double* off, int n_off, int order, double2* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_off) return;
  const double x = off[3 * i], y = off[3 * i + 1], z = off[3 * i + 2];
  double2* o = out + (size_t)i * (order + 1) * (order + 1);
  const double rho2 = x * x + y * y + z * z;
  const double inv_r2 = 1.0 / rho2;
  double2 diag = make_double2(1.0 / sqrt(rho2), 0.0);
  auto put = [&](int n, int m, double2 v) {
    o[n * n + n + m] = v;
    if (m > 0) o[n * n + n - m] = (m & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
  };
  for (int m = 0; m <= order; ++m) {
    if (m > 0) diag = cscale(cmul(make_double2(x, y), diag), -(2.0 * m - 1.0) * inv_r2);
    put(m, m, diag);
    if (m + 1 <= order) {
      double2 prev2 = diag;
      double2 prev1 = cscale(diag, (2.0 * m + 1.0) * z * inv_r2);
      put(m + 1, m, prev1);
      for (int n = m + 2; n <= order; ++n) {
        const double a = (2 * n - 1) * z;
        const double b = (double)((n - 1) * (n - 1) - m * m);
        double2 cur;
        cur.x = (a * prev1.x - b * prev2.x) * inv_r2;
        cur.y = (a * prev1.y - b * prev2.y) * inv_r2;
        put(n, m, cur);
        prev2 = prev1;
        prev1 = cur;
      }
    }
  }
}

void compute_igrid_full(const double* d_off, int n_off, int order, double2* out, cudaStream_t s) {
  if (n_off) k_igrid_full<<<grid_for(n_off, 64), 64, 0, s>>>(d_off, n_off, order, out);
  FMM_LAUNCH_CHECK();
}

template <int P>
__global__ void __launch_bounds__(M2L_WARPS * 32)
k_m2l_tiled(const int4* __restrict__ items, const int* __restrict__ srcs,
            const int* __restrict__ offs, const double2* __restrict__ igrid, int igrid_stride,
            int Ck, int Ctot, int cbase, const double2* __restrict__ M, double2* __restrict__ part) {
  constexpr int BJ = m2l_bj(P);
  constexpr int H = (P + 1) * (P + 2) / 2;
  constexpr int S = (P + 1) * (P + 1);
  constexpr int Q = 2 * P;
  constexpr int QQ = (Q + 1) * (Q + 1);
  extern __shared__ double2 sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sI = sh + warp * (QQ + S);
  double2* sM = sI + QQ;
  const int4 it = items[blockIdx.x];  // (target cell, pair begin, pair end, item id)
  // lane -> (k, j0)
  int k = -1, j0 = 0;
  {
    int cum = 0;
    for (int kk = 0; kk <= P; ++kk) {
      const int nt = (P - kk + 1 + BJ - 1) / BJ;
      if (k < 0 && lane < cum + nt) {
        k = kk;
        j0 = kk + (lane - cum) * BJ;
      }
      cum += nt;
    }
  }
  const bool active = k >= 0;
  double2 acc[BJ];
#pragma unroll
  for (int t = 0; t < BJ; ++t) acc[t] = make_double2(0.0, 0.0);
  const int nunits = (it.z - it.y) * Ck;
  for (int u = warp; u < nunits; u += M2L_WARPS) {
    const int e = it.y + u / Ck, c = cbase + u % Ck;
    const double2* Ig = igrid + (size_t)offs[e] * igrid_stride;
    for (int i = lane; i < QQ; i += 32) sI[i] = Ig[i];
    const double2* Ms = M + ((size_t)srcs[e] * Ctot + c) * H;
    for (int f = lane; f < S; f += 32) {
      const int n = (int)sqrtf((float)f + 0.5f);
      sM[f] = hget(Ms, n, f - n * n - n);
    }
    __syncwarp();
    if (active) {
      for (int m = -P; m <= P; ++m) {
        const int n0 = m < 0 ? -m : m;
        const int col = m + k;
        double2 w[BJ];
        // rows n0 + j0 + t, clamped to the grid (clamped rows only feed rows j > p, discarded)
#pragma unroll
        for (int t = 0; t < BJ; ++t) {
          const int N = min(n0 + j0 + t, Q);
          w[t] = sI[N * N + N + col];
        }
        int nlead = n0 + j0 + BJ;  // next row to enter the window
        const double2* mp = sM + n0 * n0 + n0 + m;
        int mstep = 2 * n0 + 2;
        int n = n0;
        // unrolled by BJ: the window slot holding row n+j0+t is (q + t) % BJ
        for (; n + BJ - 1 <= P; n += BJ) {
#pragma unroll
          for (int q = 0; q < BJ; ++q) {
            const double2 mv = *mp;
            mp += mstep;
            mstep += 2;
#pragma unroll
            for (int t = 0; t < BJ; ++t) acc[t] = cfma_conj(mv, w[(q + t) % BJ], acc[t]);
            const int N = min(nlead, Q);
            w[q] = sI[N * N + N + col];
            ++nlead;
          }
        }
        // remainder steps (fewer than BJ), window slots continue the rotation
#pragma unroll
        for (int q = 0; q < BJ - 1; ++q) {
          if (n + q <= P) {
            const double2 mv = *mp;
            mp += mstep;
            mstep += 2;
#pragma unroll
            for (int t = 0; t < BJ; ++t) acc[t] = cfma_conj(mv, w[(q + t) % BJ], acc[t]);
            const int N = min(nlead, Q);
            w[q] = sI[N * N + N + col];
            ++nlead;
          }
        }
      }
    }
    __syncwarp();
  }
  // cross-warp reduction (warps w and w + Ck hold the same channel), fixed order
  __syncthreads();
  double2* red = sh;  // [M2L_WARPS][32][BJ]
#pragma unroll
  for (int t = 0; t < BJ; ++t) red[(warp * 32 + lane) * BJ + t] = acc[t];
  __syncthreads();
  if (warp < Ck && active) {
    const int c = cbase + warp;
#pragma unroll
    for (int t = 0; t < BJ; ++t) {
      const int j = j0 + t;
      if (j > P) continue;
      double2 s = make_double2(0.0, 0.0);
      for (int w2 = warp; w2 < M2L_WARPS; w2 += Ck) s = cadd(s, red[(w2 * 32 + lane) * BJ + t]);
      const double sg = (j & 1) ? -1.0 : 1.0;
      part[((size_t)it.w * Ctot + c) * H + j * (j + 1) / 2 + k] = cscale(s, sg);
    }
  }
}

// L[cell] = sum of its items' partial blocks (cells without items get zeros)
__global__ void k_m2l_reduce(int n_cells, const int* __restrict__ cell_items, int CH,
                             const double2* __restrict__ part, double2* __restrict__ L) {
  const int cell = blockIdx.x;
  const int i0 = cell_items[cell], i1 = cell_items[cell + 1];
  for (int t = threadIdx.x; t < CH; t += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int i = i0; i < i1; ++i) s = cadd(s, part[(size_t)i * CH + t]);
    L[(size_t)cell * CH + t] = s;
  }
}

template <int P>
void launch_m2l_p(const Plan& plan, int Ctot, const double2* M, double2* part, cudaStream_t st) {
  constexpr int S = (P + 1) * (P + 1);
  constexpr int QQ = (2 * P + 1) * (2 * P + 1);
  constexpr int RED = 32 * m2l_bj(P);
  const size_t smem = (size_t)M2L_WARPS * (QQ + S > RED ? QQ + S : RED) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2l_tiled<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  const int n = (int)plan.m2l_items.size();
  const int stride = (2 * plan.igrid_p + 1) * (2 * plan.igrid_p + 1);
  // channel groups whose size divides the warp count
  for (int cb = 0; cb < Ctot;) {
    const int rem = Ctot - cb;
    const int ck = rem >= 4 ? 4 : rem >= 2 ? 2 : 1;
    k_m2l_tiled<P><<<n, M2L_WARPS * 32, smem, st>>>(plan.d_m2l_items.get(), plan.m2l_src.get(),
                                                    plan.m2l_off.get(), plan.igrid.get(), stride,
                                                    ck, Ctot, cb, M, part);
    cb += ck;
  }
  FMM_LAUNCH_CHECK();
}

void launch_m2l(const Plan& plan, int p, int C, const double2* M, double2* L, double2* part,
                cudaStream_t st) {
  const int H = hcount(p);
  if (!plan.m2l_items.empty()) {
    switch (p) {
#define M2L_CASE(PP) case PP: launch_m2l_p<PP>(plan, C, M, part, st); break;
      M2L_CASE(0) M2L_CASE(1) M2L_CASE(2) M2L_CASE(3) M2L_CASE(4) M2L_CASE(5) M2L_CASE(6)
      M2L_CASE(7) M2L_CASE(8) M2L_CASE(9) M2L_CASE(10) M2L_CASE(11) M2L_CASE(12) M2L_CASE(13)
      M2L_CASE(14) M2L_CASE(15) M2L_CASE(16) M2L_CASE(17) M2L_CASE(18) M2L_CASE(19) M2L_CASE(20)
#undef M2L_CASE
      default: throw ArgumentError("M2L: expansion order out of range");
    }
  }
  k_m2l_reduce<<<plan.tgt.n_cells, 128, 0, st>>>(plan.tgt.n_cells, plan.m2l_cell_items.get(), C * H,
                                                 part, L);
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmbem
