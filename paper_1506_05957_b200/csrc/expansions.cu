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
  static DeviceOnce done;
  if (!done.first()) return;
  short n_of[hcount(P_MAX)], m_of[hcount(P_MAX)];
  for (int n = 0; n <= P_MAX; ++n)
    for (int m = 0; m <= n; ++m) {
      n_of[hidx(n, m)] = (short)n;
      m_of[hidx(n, m)] = (short)m;
    }
  FMM_CUDA(cudaMemcpyToSymbol(c_n_of, n_of, sizeof(n_of)));
  FMM_CUDA(cudaMemcpyToSymbol(c_m_of, m_of, sizeof(m_of)));
  done.mark();
}

// ------------------------------------------------------------------ P2M
// One CTA per source leaf; bodies processed CHUNK at a time.  Phase A: eight
// threads per body generate R (interleaved columns m) into shared memory.
// Phase B: thread groups each reduce a strided subset of the chunk's bodies
// into their own coefficient (all threads busy even at low p); groups are
// added in a fixed order at the end.
constexpr int P2M_THREADS = 256;
constexpr int P2M_CHUNK = 32;

template <int C, bool HQ, bool HD>
__global__ void __launch_bounds__(P2M_THREADS)
k_p2m(TreeDev S, const int* leaves, int p, const double* __restrict__ q,
      const double* __restrict__ d, double2* __restrict__ M) {
  extern __shared__ double2 sh_r[];  // [P2M_CHUNK][H], later the group reduction
  __shared__ double s_q[HQ ? C : 1][P2M_CHUNK];
  __shared__ double s_d[HD ? C : 1][P2M_CHUNK][3];
  const int H = hcount(p);
  const int leaf = leaves[blockIdx.x];
  const int b0 = S.body_start[leaf], nb = S.body_count[leaf];
  const double cx = S.cx[leaf], cy = S.cy[leaf], cz = S.cz[leaf];
  const int64_t ns = S.n_points;
  const int G = H <= P2M_THREADS ? P2M_THREADS / H : 1;  // H <= 231 < 256 always
  const int idx = threadIdx.x % H, g = threadIdx.x / H;
  const bool active = g < G;
  const int n = c_n_of[idx], m = c_m_of[idx];
  const bool has_up = n >= 1 && m + 1 <= n - 1;
  const bool has_dn = n >= 1 && m - 1 >= -(n - 1);
  const bool has_z = n >= 1 && m <= n - 1;
  double2 acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = make_double2(0.0, 0.0);

  for (int base = 0; base < nb; base += P2M_CHUNK) {
    const int cnt = min(P2M_CHUNK, nb - base);
    const int bl = threadIdx.x >> 3, part = threadIdx.x & 7;
    if (bl < cnt) {
      const int i = b0 + base + bl;
      regular_half_cols(S.px[i] - cx, S.py[i] - cy, S.pz[i] - cz, p, sh_r + bl * H, part, 8, S.rec);
      if (part == 0) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if (HQ) s_q[c][bl] = q[c * ns + i];
          if (HD) {
            s_d[c][bl][0] = d[(c * ns + i) * 3 + 0];
            s_d[c][bl][1] = d[(c * ns + i) * 3 + 1];
            s_d[c][bl][2] = d[(c * ns + i) * 3 + 2];
          }
        }
      }
    }
    __syncthreads();
    if (active) {
      for (int b = g; b < cnt; b += G) {
        const double2* R = sh_r + b * H;
        double2 rv, ra, rb, rz;
        if (HQ) rv = R[idx];
        if (HD) {
          // gradient-shift sources R_{n-1}^{m+1}, R_{n-1}^{m-1}, R_{n-1}^m (harmonics.py:128-140)
          ra = has_up ? R[hidx(n - 1, m + 1)] : make_double2(0.0, 0.0);
          rb = has_dn ? hget(R, n - 1, m - 1) : make_double2(0.0, 0.0);
          rz = has_z ? R[hidx(n - 1, m)] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double2 a = acc[c];
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
          acc[c] = a;
        }
      }
    }
    __syncthreads();
  }
  // groups -> fixed-order sum
  if (active)
#pragma unroll
    for (int c = 0; c < C; ++c) sh_r[(g * C + c) * H + idx] = acc[c];
  __syncthreads();
  double2* out = M + (size_t)leaf * C * H;
  for (int t = threadIdx.x; t < C * H; t += blockDim.x) {
    const int c = t / H, ii = t - c * H;
    double2 s = make_double2(0.0, 0.0);
    for (int gg = 0; gg < G; ++gg) s = cadd(s, sh_r[(gg * C + c) * H + ii]);
    out[c * H + ii] = s;
  }
}

template <int C, bool HQ, bool HD>
void launch_p2m_t(const TreeDev& S, const int* leaves, int n_leaves, int p, const double* q,
                  const double* d, double2* M, cudaStream_t st) {
  const int H = hcount(p);
  const int G = P2M_THREADS / H;
  const size_t smem = (size_t)std::max(P2M_CHUNK * H, G * C * H) * sizeof(double2);
  static DeviceOnce attr;
  if (attr.first()) {
    FMM_CUDA(cudaFuncSetAttribute(k_p2m<C, HQ, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(P2M_CHUNK * hcount(P_MAX) * sizeof(double2))));
    attr.mark();
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

}  // namespace fmmbem
