// Far-field operators: P2M, M2M, M2L, L2L on device (fp64, SIMT).
//
// Reference math (harmonics.py):
//   P2M  M = sum q R(y - c) + sum d . grad R(y - c)         fmm.py:235-257
//   M2M  M'_n^m = sum_{j,k} M_j^k R_{n-j}^{m-k}(child - parent)   fmm.py:268-290
//   M2L  L_j^k = (-1)^j sum_{n<=p,m} M_n^m conj(I_{n+j}^{m+k}(D))  fmm.py:292-314
//   L2L  L'_n^m = sum_{j>=n,k} L_j^k R_{j-n}^{k-m}(child - parent)
// Every expansion is stored half (m >= 0, see common.cuh); per-cell blocks
// are [cell][channel][hcount(p)] double2.  The reference batches these as
// zgemm over offset groups; here one CTA owns one output cell, so every
// accumulation runs in a fixed order and no atomics are needed.
#include "kernels.cuh"

namespace fmmbem {

__constant__ short c_n_of[hcount(P_MAX)];
__constant__ short c_m_of[hcount(P_MAX)];

void upload_index_tables() {
  static bool done = false;
  if (done) return;
  short n_of[hcount(P_MAX)], m_of[hcount(P_MAX)];
  for (int n = 0; n <= P_MAX; ++n)
    for (int m = 0; m <= n; ++m) {
      n_of[hidx(n, m)] = (short)n;
      m_of[hidx(n, m)] = (short)m;
    }
  FMM_CUDA(cudaMemcpyToSymbol(c_n_of, n_of, sizeof(n_of)));
  FMM_CUDA(cudaMemcpyToSymbol(c_m_of, m_of, sizeof(m_of)));
  done = true;
}

// ------------------------------------------------------------------ P2M
// one CTA per source leaf; bodies processed CHUNK at a time: the first CHUNK
// threads evaluate R for one body each into shared memory, then every thread
// reduces the chunk into its own coefficients.
constexpr int P2M_THREADS = 128;
constexpr int P2M_CHUNK = 32;
constexpr int P2M_SLOTS = (hcount(P_MAX) + P2M_THREADS - 1) / P2M_THREADS;

template <int C, bool HQ, bool HD>
__global__ void __launch_bounds__(P2M_THREADS)
k_p2m(TreeDev S, const int* leaves, int p, const double* __restrict__ q,
      const double* __restrict__ d, double2* __restrict__ M) {
  extern __shared__ double2 sh_r[];  // [P2M_CHUNK][H]
  __shared__ double s_q[HQ ? C : 1][P2M_CHUNK];
  __shared__ double s_d[HD ? C : 1][P2M_CHUNK][3];
  const int H = hcount(p);
  const int leaf = leaves[blockIdx.x];
  const int b0 = S.body_start[leaf], nb = S.body_count[leaf];
  const double cx = S.cx[leaf], cy = S.cy[leaf], cz = S.cz[leaf];
  const int64_t ns = S.n_points;
  double2 acc[P2M_SLOTS][C];
#pragma unroll
  for (int s = 0; s < P2M_SLOTS; ++s)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[s][c] = make_double2(0.0, 0.0);

  for (int base = 0; base < nb; base += P2M_CHUNK) {
    const int cnt = min(P2M_CHUNK, nb - base);
    if (threadIdx.x < cnt) {
      const int i = b0 + base + threadIdx.x;
      regular_half(S.px[i] - cx, S.py[i] - cy, S.pz[i] - cz, p, sh_r + threadIdx.x * H);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (HQ) s_q[c][threadIdx.x] = q[c * ns + i];
        if (HD) {
          s_d[c][threadIdx.x][0] = d[(c * ns + i) * 3 + 0];
          s_d[c][threadIdx.x][1] = d[(c * ns + i) * 3 + 1];
          s_d[c][threadIdx.x][2] = d[(c * ns + i) * 3 + 2];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < P2M_SLOTS; ++s) {
      const int idx = threadIdx.x + s * P2M_THREADS;
      if (idx < H) {
        const int n = c_n_of[idx], m = c_m_of[idx];
        // gradient-shift sources R_{n-1}^{m+1}, R_{n-1}^{m-1}, R_{n-1}^m (harmonics.py:128-140)
        const bool has_up = n >= 1 && m + 1 <= n - 1;
        const bool has_dn = n >= 1 && m - 1 >= -(n - 1);
        const bool has_z = n >= 1 && m <= n - 1;
        for (int b = 0; b < cnt; ++b) {
          const double2* R = sh_r + b * H;
          double2 rv, ra, rb, rz;
          if (HQ) rv = R[idx];
          if (HD) {
            ra = has_up ? R[hidx(n - 1, m + 1)] : make_double2(0.0, 0.0);
            rb = has_dn ? hget(R, n - 1, m - 1) : make_double2(0.0, 0.0);
            rz = has_z ? R[hidx(n - 1, m)] : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int c = 0; c < C; ++c) {
            double2 a = acc[s][c];
            if (HQ) {
              const double w = s_q[c][b];
              a.x = fma(w, rv.x, a.x);
              a.y = fma(w, rv.y, a.y);
            }
            if (HD) {
              const double dx = 0.5 * s_d[c][b][0], dy = 0.5 * s_d[c][b][1], dz = s_d[c][b][2];
              // 1/2 (dx - i dy) R^{m+1} - 1/2 (dx + i dy) R^{m-1} + dz R^m
              a = cfma(make_double2(dx, -dy), ra, a);
              a = cfma(make_double2(-dx, -dy), rb, a);
              a.x = fma(dz, rz.x, a.x);
              a.y = fma(dz, rz.y, a.y);
            }
            acc[s][c] = a;
          }
        }
      }
    }
    __syncthreads();
  }
  double2* out = M + (size_t)leaf * C * H;
#pragma unroll
  for (int s = 0; s < P2M_SLOTS; ++s) {
    const int idx = threadIdx.x + s * P2M_THREADS;
    if (idx < H)
#pragma unroll
      for (int c = 0; c < C; ++c) out[c * H + idx] = acc[s][c];
  }
}

template <int C, bool HQ, bool HD>
void launch_p2m_t(const TreeDev& S, const int* leaves, int n_leaves, int p, const double* q,
                  const double* d, double2* M, cudaStream_t st) {
  const size_t smem = (size_t)P2M_CHUNK * hcount(p) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    FMM_CUDA(cudaFuncSetAttribute(k_p2m<C, HQ, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(P2M_CHUNK * hcount(P_MAX) * sizeof(double2))));
    attr = true;
  }
  if (n_leaves) k_p2m<C, HQ, HD><<<n_leaves, P2M_THREADS, smem, st>>>(S, leaves, p, q, d, M);
  FMM_LAUNCH_CHECK();
}

void launch_p2m(const TreeDev& S, const int* leaves, int n_leaves, int p, int C, const double* q,
                const double* d, double2* M, cudaStream_t st) {
  const bool hq = q != nullptr, hd = d != nullptr;
#define P2M_CASE(CC)                                                               \
  if (C == CC) {                                                                   \
    if (hq && hd) return launch_p2m_t<CC, true, true>(S, leaves, n_leaves, p, q, d, M, st);  \
    if (hq) return launch_p2m_t<CC, true, false>(S, leaves, n_leaves, p, q, d, M, st);       \
    return launch_p2m_t<CC, false, true>(S, leaves, n_leaves, p, q, d, M, st);               \
  }
  P2M_CASE(1)
  P2M_CASE(4)
  P2M_CASE(7)
#undef P2M_CASE
  throw ArgumentError("P2M: unsupported channel count");
}

// ------------------------------------------------------------------ M2M
// one CTA per cell of `level`; internal cells gather their children.
constexpr int VERT_THREADS = 256;

__global__ void __launch_bounds__(VERT_THREADS)
k_m2m(TreeDev S, int cell0, int cell1, int p, int C, const double2* __restrict__ rshift,
      double2* __restrict__ M) {
  extern __shared__ double2 sh[];  // [C*H] child coefficients + [H] R(d)
  const int cell = cell0 + blockIdx.x;
  if (cell >= cell1 || S.is_leaf[cell]) return;
  const int H = hcount(p);
  double2* sM = sh;
  double2* sR = sh + C * H;
  const int nout = C * H;
  double2 acc[8];
  for (int s = 0; s < 8; ++s) acc[s] = make_double2(0.0, 0.0);
  const int fc = S.first_child[cell], nc = S.n_child[cell];
  for (int k = 0; k < nc; ++k) {
    const int ch = fc + k;
    const int o = (S.cx[ch] > S.cx[cell] ? 1 : 0) | (S.cy[ch] > S.cy[cell] ? 2 : 0) |
                  (S.cz[ch] > S.cz[cell] ? 4 : 0);
    const double2* R = rshift + ((size_t)S.level[ch] * 8 + o) * hcount(P_MAX);
    for (int i = threadIdx.x; i < nout; i += blockDim.x) sM[i] = M[(size_t)ch * nout + i];
    for (int i = threadIdx.x; i < H; i += blockDim.x) sR[i] = R[i];
    __syncthreads();
    for (int s = 0, t = threadIdx.x; t < nout; ++s, t += blockDim.x) {
      const int c = t / H, idx = t - c * H;
      const int n = c_n_of[idx], m = c_m_of[idx];
      const double2* Mc = sM + c * H;
      double2 a = acc[s];
      for (int j = 0; j <= n; ++j) {
        const int kmin = max(-j, m - (n - j)), kmax = min(j, m + (n - j));
        for (int kk = kmin; kk <= kmax; ++kk) a = cfma(hget(Mc, j, kk), hget(sR, n - j, m - kk), a);
      }
      acc[s] = a;
    }
    __syncthreads();
  }
  for (int s = 0, t = threadIdx.x; t < nout; ++s, t += blockDim.x) M[(size_t)cell * nout + t] = acc[s];
}

void launch_m2m(const TreeDev& S, const Tree& host, int p, int C, const double2* rshift,
                double2* M, cudaStream_t st) {
  const int H = hcount(p);
  FMM_REQUIRE(C * H <= 8 * VERT_THREADS, "M2M: too many coefficients per cell");
  const size_t smem = (size_t)(C + 1) * H * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2m, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(8 * hcount(P_MAX) * sizeof(double2))));
    attr = true;
  }
  for (int l = host.n_levels - 2; l >= 0; --l) {
    const int a = host.level_start[l], b = host.level_start[l + 1];
    if (b > a) k_m2m<<<b - a, VERT_THREADS, smem, st>>>(S, a, b, p, C, rshift, M);
  }
  FMM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ L2L
__global__ void __launch_bounds__(VERT_THREADS)
k_l2l(TreeDev T, int cell0, int cell1, int p, int C, const double2* __restrict__ rshift,
      double2* __restrict__ L) {
  extern __shared__ double2 sh[];
  const int cell = cell0 + blockIdx.x;
  if (cell >= cell1) return;
  const int H = hcount(p);
  const int nout = C * H;
  const int par = T.parent[cell];
  const int o = (T.cx[cell] > T.cx[par] ? 1 : 0) | (T.cy[cell] > T.cy[par] ? 2 : 0) |
                (T.cz[cell] > T.cz[par] ? 4 : 0);
  const double2* R = rshift + ((size_t)T.level[cell] * 8 + o) * hcount(P_MAX);
  double2* sL = sh;
  double2* sR = sh + nout;
  for (int i = threadIdx.x; i < nout; i += blockDim.x) sL[i] = L[(size_t)par * nout + i];
  for (int i = threadIdx.x; i < H; i += blockDim.x) sR[i] = R[i];
  __syncthreads();
  for (int t = threadIdx.x; t < nout; t += blockDim.x) {
    const int c = t / H, idx = t - c * H;
    const int n = c_n_of[idx], m = c_m_of[idx];
    const double2* Lc = sL + c * H;
    double2 a = make_double2(0.0, 0.0);
    for (int j = n; j <= p; ++j) {
      const int kmin = max(-j, m - (j - n)), kmax = min(j, m + (j - n));
      for (int kk = kmin; kk <= kmax; ++kk) a = cfma(hget(Lc, j, kk), hget(sR, j - n, kk - m), a);
    }
    double2 v = L[(size_t)cell * nout + t];
    L[(size_t)cell * nout + t] = cadd(v, a);
  }
}

void launch_l2l(const TreeDev& T, const Tree& host, int p, int C, const double2* rshift,
                double2* L, cudaStream_t st) {
  const int H = hcount(p);
  const size_t smem = (size_t)(C + 1) * H * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    FMM_CUDA(cudaFuncSetAttribute(k_l2l, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(8 * hcount(P_MAX) * sizeof(double2))));
    attr = true;
  }
  for (int l = 1; l < host.n_levels; ++l) {
    const int a = host.level_start[l], b = host.level_start[l + 1];
    if (b > a) k_l2l<<<b - a, VERT_THREADS, smem, st>>>(T, a, b, p, C, rshift, L);
  }
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmbem
