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

constexpr int ROT_THREADS = 256;
constexpr int ROT_V = 8;  // vectors (pairs x channels) per pass

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

__global__ void __launch_bounds__(ROT_THREADS)
k_m2l_rot(const int4* __restrict__ items, const int* __restrict__ gpair,
          const int* __restrict__ pair_src, const double* __restrict__ rot, int rot_stride,
          const double* __restrict__ geo, int p, const double2* __restrict__ M, int Ctot, int C,
          double2* __restrict__ pout) {
  extern __shared__ double2 sh2[];
  const int H = hcount(p), S = (p + 1) * (p + 1), RS = rot_size(p);
  double2* sPh = sh2;                       // [2p+1] e^{-ik phi}, k = -p..p
  double2* sMf = sPh + (2 * p + 1);         // [V][S] e^{-ik phi} M_n^k
  double2* sMp = sMf + ROT_V * S;           // [V][H] M'
  double2* sLp = sMp + ROT_V * H;           // [V][H] L'
  double* sZ = reinterpret_cast<double*>(sLp + ROT_V * H);  // [2p+1] N! / r^(N+1)
  double* sA = sZ + (2 * p + 2);                            // rotation matrices, 8-byte aligned
  const int4 it = items[blockIdx.x];
  const int u = it.x;
  {
    const double* A = rot + (size_t)u * rot_stride;
    for (int i = threadIdx.x; i < RS; i += blockDim.x) cp_async8(sA + i, A + i);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  const double r = geo[3 * u], ph = geo[3 * u + 2];
  for (int k = threadIdx.x; k < 2 * p + 1; k += blockDim.x) {
    double sn, cs;
    sincos(-(double)(k - p) * ph, &sn, &cs);
    sPh[k] = make_double2(cs, sn);
  }
  if (threadIdx.x == 0) {
    double f = 1.0, rp = 1.0 / r;  // N! / r^(N+1)
    for (int N = 0; N <= 2 * p; ++N) {
      if (N > 0) {
        f *= N;
        rp /= r;
      }
      sZ[N] = f * rp;
    }
  }
  const int vpp = C;                        // vectors per pair (channels)
  const int ppass = ROT_V / vpp > 0 ? ROT_V / vpp : 1;
  for (int e0 = it.y; e0 < it.z; e0 += ppass) {
    const int np = min(ppass, it.z - e0);
    const int nv = np * vpp;
    __syncthreads();
    for (int f = threadIdx.x; f < nv * S; f += blockDim.x) {
      const int v = f / S, g = f - v * S;
      const int e = gpair[e0 + v / vpp], c = v % vpp;
      const int n = (int)__fsqrt_rz((float)g), k = g - n * n - n;
      const double2 mv = hget(M + ((size_t)pair_src[e] * Ctot + c) * H, n, k);
      sMf[v * S + g] = cmul(sPh[k + p], mv);
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // stage A: M'_n^m = sum_k a^n_{mk} (e^{-ik phi} M_n^k), m >= 0, 4 vectors per item
    const int ngrp = (nv + 3) / 4;
    for (int w = threadIdx.x; w < H * ngrp; w += blockDim.x) {
      const int idx = w % H, vg = w / H;
      const int n = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
      const int m = idx - n * (n + 1) / 2;
      const double* arow = sA + rot_base(n) + (m + n) * (2 * n + 1) + n;  // a[k] at arow[k]
      double2 acc[4] = {};
      for (int k = -n; k <= n; ++k) {
        const double aa = arow[k];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 mv = sMf[(vg * 4 + q) * S + n * n + n + k];
          acc[q].x = fma(aa, mv.x, acc[q].x);
          acc[q].y = fma(aa, mv.y, acc[q].y);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (vg * 4 + q < nv) sMp[(vg * 4 + q) * H + idx] = acc[q];
    }
    __syncthreads();
    // stage B: L'_j^k = (-1)^j sum_{n>=k} M'_n^{-k} z_{n+j},  M'_n^{-k} = (-1)^k conj(M'_n^k)
    for (int w = threadIdx.x; w < H * ngrp; w += blockDim.x) {
      const int idx = w % H, vg = w / H;
      const int j = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
      const int k = idx - j * (j + 1) / 2;
      double2 acc[4] = {};
      for (int n = k; n <= p; ++n) {
        const double zz = sZ[n + j];
        const int hi = n * (n + 1) / 2 + k;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 mv = sMp[(vg * 4 + q) * H + hi];
          acc[q].x = fma(zz, mv.x, acc[q].x);
          acc[q].y = fma(-zz, mv.y, acc[q].y);  // conj
        }
      }
      const double sg = ((j + k) & 1) ? -1.0 : 1.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (vg * 4 + q < nv) sLp[(vg * 4 + q) * H + idx] = cscale(acc[q], sg);
    }
    __syncthreads();
    // stage C: L_j^k = e^{-ik phi} sum_l a^j_{lk} L'_j^l (l < 0 via real symmetry)
    for (int w = threadIdx.x; w < H * ngrp; w += blockDim.x) {
      const int idx = w % H, vg = w / H;
      const int j = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
      const int k = idx - j * (j + 1) / 2;
      const double* acol = sA + rot_base(j) + (k + j);  // a[l][k] at acol[(l + j) * (2j + 1)]
      const int stride = 2 * j + 1;
      double2 acc[4] = {};
      for (int l = -j; l <= j; ++l) {
        const double aa = acol[(l + j) * stride];
        const int al = l < 0 ? -l : l;
        const int hi = j * (j + 1) / 2 + al;
        const bool neg = l < 0, odd = (al & 1) != 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double2 lv = sLp[(vg * 4 + q) * H + hi];
          if (neg) lv = odd ? make_double2(-lv.x, lv.y) : make_double2(lv.x, -lv.y);
          acc[q].x = fma(aa, lv.x, acc[q].x);
          acc[q].y = fma(aa, lv.y, acc[q].y);
        }
      }
      const double2 phs = sPh[k + p];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int v = vg * 4 + q;
        if (v >= nv) continue;
        const int e = gpair[e0 + v / vpp], c = v % vpp;
        pout[((size_t)e * Ctot + c) * H + idx] = cmul(phs, acc[q]);
      }
    }
  }
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

void launch_m2l_rot(const Plan& plan, const int4* gitems, const int* gpair, int n_items, int p,
                    int C, const double2* M, double2* pout, cudaStream_t st) {
  if (n_items <= 0) return;
  const int H = hcount(p), S = (p + 1) * (p + 1);
  const size_t smem = (size_t)(2 * p + 1 + ROT_V * S + 2 * ROT_V * H) * sizeof(double2) +
                      (size_t)(2 * p + 2 + rot_size(p)) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2l_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  FMM_REQUIRE(smem <= 227 * 1024, "rotation M2L tiles exceed shared memory");
  k_m2l_rot<<<n_items, ROT_THREADS, smem, st>>>(gitems, gpair, plan.m2l_src.get(), plan.rot.get(),
                                               rot_size(plan.rot_p), plan.rot_geo.get(), p, M, C, C,
                                               pout);
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmbem
