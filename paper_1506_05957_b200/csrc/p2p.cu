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
#include <algorithm>
#include <cstdio>

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
  // d2 >= +0 always: the coincident-pair mask (fmm.py:403) as an integer compare of the bit
  // pattern (integer pipe) instead of a DSETP on the FP64 pipe
  const double inv = __double_as_longlong(d2) > 0 ? rsqrt_nr2(d2) : 0.0;  // ~3e-14 relative
  if (K == P2PKind::LAP_Q) {
    acc[0] = fma(wv[0], inv, acc[0]);
  } else if (K == P2PKind::LAP_D) {
    const double rn = fma(rx, wv[0], fma(ry, wv[1], rz * wv[2]));
    const double inv3 = inv * inv * inv;
    acc[0] = fma(rn, inv3, acc[0]);
  } else if (K == P2PKind::STOKESLET) {
    // f / r + r (r.f) / r^3 = (f + r (r.f) / r^2) / r: 8 DP instructions after inv
    const double rf = fma(rx, wv[0], fma(ry, wv[1], rz * wv[2]));
    const double t = rf * (inv * inv);
    acc[0] = fma(fma(rx, t, wv[0]), inv, acc[0]);
    acc[1] = fma(fma(ry, t, wv[1]), inv, acc[1]);
    acc[2] = fma(fma(rz, t, wv[2]), inv, acc[2]);
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

// ------------------------------------------------------------------ double layer, expanded form
// Laplace double-layer potential sum_j d_j.(t - y_j) / |t - y_j|^3 (fmm.py:399-419) in
// coordinates centred on the target leaf (t' = t - c, s' = y - c):
//   |t - y|^2 = |t'|^2 + |s'|^2 - 2 t'.s'      (1 DADD + 3 DFMA instead of 3 DADD + 3 DFMA)
//   d.(t - y) = d.t' - d.s'                    (3 DFMA)
// with the per-source parts (-2 s', |s'|^2, d, -d.s') staged once per item.  Centring on the
// leaf keeps |t'|, |s'| at the size of the near region, so the cancellation in |t - y|^2 costs
// ~eps R^2 / r^2 <= ~1e-12 relative on the closest pairs.  The coincident pair (the target is
// Gauss point 0 of its own panel, bemop.py:64-67; the reference's d2 > 0 mask, fmm.py:403) is
// removed by index: its slot in the staged tile gets d2 = ~1e300, so r^-3 underflows to 0.
// 12 DP instructions per interaction (15 in the difference form).
//
// Persistent and warp-specialised: one CTA per SM; LAPD_PROD producer warps take items in
// largest-first order from a global counter and stage item k+1 (leaf table, transformed
// sources, every target's own-source slot) into one of two shared-memory stages while the
// LAPD_CONS consumer threads run the interaction loop on item k.  Stages are handed over
// through barriers: FULL is a shared-memory mbarrier per stage (every producer thread arrives,
// consumer warps only wait on its phase, so no consumer warp waits for another — the last
// warp's reduction of item k overlaps the other warps' item k + 1); EMPTY is a named barrier
// (consumers arrive, producers sync).
constexpr int LAPD_TPT = 4;
#ifndef LAPD_CONS_N
#define LAPD_CONS_N 256
#endif
constexpr int LAPD_CONS = LAPD_CONS_N;  // consumer threads (tools: -DLAPD_CONS_N=384)
#ifndef LAPD_PROD_N
#define LAPD_PROD_N 128
#endif
constexpr int LAPD_PROD = LAPD_PROD_N;
#ifndef LAPD_SPT
#define LAPD_SPT 2  // sources per trip of the consumer loop (tools: -DLAPD_SPT=3)
#endif
#ifndef LAPD_SPR
#define LAPD_SPR 4
#endif
constexpr int SPR = LAPD_SPR;  // sources per staging thread per round (loads in flight)
enum : int { BAR_FULL0 = 1, BAR_EMPTY0 = 5, BAR_PROD = 9 };  // up to 4 stages

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "MBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBW_%=;\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct LapdStage {  // shared-memory stage layout (offsets in bytes from the stage base)
  size_t planes, tgt, ltab, slot, spec, bytes;
  __host__ __device__ LapdStage(int max_src, int max_leaves, int max_tgt) {
    planes = 0;
    tgt = (size_t)4 * max_src * sizeof(double2);        // [2][max_tgt] double2: (x', y'), (z', |t'|^2)
    ltab = tgt + (size_t)2 * max_tgt * sizeof(double2);
    slot = ltab + (size_t)max_leaves * sizeof(int4);
    spec = slot + (size_t)max_tgt * sizeof(int);
    bytes = (spec + (size_t)max_tgt * sizeof(int) + 8 * sizeof(int) + 15) / 16 * 16;
  }
};

struct LapdSrc {
  double2 ab, cs, dxy, dzs;  // (-2x', -2y'), (-2z', |s'|^2), (d_x, d_y), (d_z, -d.s')
};

__device__ __forceinline__ LapdSrc lapd_load(const double2* __restrict__ sh2, int max_src, int j) {
  return LapdSrc{sh2[j], sh2[max_src + j], sh2[2 * max_src + j], sh2[3 * max_src + j]};
}

template <int TPT, bool MASK>
__device__ __forceinline__ void lapd_body(const LapdSrc& u, int j, const double* tx, const double* ty,
                                          const double* tz, const double* tt, const int* self,
                                          double* acc) {
#pragma unroll
  for (int q = 0; q < TPT; ++q) {
    double d2 = fma(tx[q], u.ab.x, fma(ty[q], u.ab.y, fma(tz[q], u.cs.x, u.cs.y + tt[q])));
    // coincident pair: hi word of ~1e300 (the lo word is irrelevant), so r^-3 underflows to 0
    if (MASK) d2 = __hiloint2double(j == self[q] ? 0x7E37E43C : __double2hiint(d2), __double2loint(d2));
    // seed: MUFU.RSQ64H (an fp32 MUFU.RSQ seed through F2F conversions measured 16 % slower
    // on cfg5: the conversions cost more FP64-pipe time than the fp64 seed)
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d2));
    // r^-3 = y^3 (1 + 3/2 e), e = 1 - d2 y^2, = -3/2 y^3 g with g = d2 y^2 - 5/3; the -3/2
    // is folded into the staged dipoles (rn below is -3/2 d.(t - y)): 12 DP instructions
    const double y2 = y * y;
    const double g = fma(d2, y2, -5.0 / 3.0);
    const double y3 = y2 * y;
    const double rn = fma(u.dxy.x, tx[q], fma(u.dxy.y, ty[q], fma(u.dzs.x, tz[q], u.dzs.y)));
    acc[q] = fma(rn * y3, g, acc[q]);
  }
}

// Panel-shared dipole term.  The far rule's Gauss points of one panel lie in the panel's plane
// and carry the same normal and density, so d.(t - y_j) = d.t' - d.s'_j is the same for every
// point j of the panel (d.s'_j = d.s'_0 exactly for a flat panel), and the three outer points
// share one weight (quadrature.py:47-52: -27/48 at the centroid, 25/48 at the others).  The
// outer points of one panel inside one source leaf therefore form a cluster of C <= 3 points:
//   sum_j d.(t - y_j) / r_j^3 = (d.(t - y_0)) * sum_j r_j^-3
// costs 8 C + 4 DP instructions instead of 12 C.  The centroids and lone outer points stay
// single points (12 instructions); measured on a synthetic tile (tools/p2p_cluster_probe.cu):
// 32.4 (single) / 26.8 (C = 2) / 23.8 (C = 3) cycles per warp-interaction.
template <int C>
struct LapdCl {
  double2 ab[C], cs[C], dxy, dzs;
};

template <int C>
__device__ __forceinline__ LapdCl<C> lapd_load_cl(const double2* __restrict__ sh2, int max_src, int rec, int pt) {
  LapdCl<C> u;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    u.ab[i] = sh2[pt + i];
    u.cs[i] = sh2[max_src + pt + i];
  }
  u.dxy = sh2[2 * max_src + rec];
  u.dzs = sh2[3 * max_src + rec];
  return u;
}

template <int TPT, int C>
__device__ __forceinline__ void lapd_body_cl(const LapdCl<C>& u, const double* tx, const double* ty,
                                             const double* tz, const double* tt, double* acc) {
#pragma unroll
  for (int q = 0; q < TPT; ++q) {
    const double rn = fma(u.dxy.x, tx[q], fma(u.dxy.y, ty[q], fma(u.dzs.x, tz[q], u.dzs.y)));
    double k = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const double d2 = fma(tx[q], u.ab[i].x, fma(ty[q], u.ab[i].y, fma(tz[q], u.cs[i].x, u.cs[i].y + tt[q])));
      double y;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d2));
      const double y2 = y * y;
      const double g = fma(d2, y2, -5.0 / 3.0);
      const double y3 = y2 * y;
      k = i == 0 ? y3 * g : fma(y3, g, k);
    }
    acc[q] = fma(rn, k, acc[q]);
  }
}

// the clusters of one tile section: records [rec0, rec0 + n), points from pt0 (C per cluster);
// thread group g of G takes the records r = g (mod G), so the groups' shares stay balanced
// across the sections; the next cluster is read while this one is used
template <int TPT, int C>
__device__ __forceinline__ void lapd_run_clusters(const double2* __restrict__ sh2, int max_src, int rec0, int pt0,
                                                  int n, int g, int G, const double* tx, const double* ty,
                                                  const double* tz, const double* tt, double* acc) {
  int c = (g - rec0 % G + G) % G;
  if (c >= n) return;
  LapdCl<C> u = lapd_load_cl<C>(sh2, max_src, rec0 + c, pt0 + C * c);
  for (; c + G < n; c += G) {
    const LapdCl<C> v = lapd_load_cl<C>(sh2, max_src, rec0 + c + G, pt0 + C * (c + G));
    lapd_body_cl<TPT, C>(u, tx, ty, tz, tt, acc);
    u = v;
  }
  lapd_body_cl<TPT, C>(u, tx, ty, tz, tt, acc);
}

// The launch bound is 128 threads above the launched count, which caps the kernel at 128
// registers per thread (no spills; 149 uncapped).  Alone the kernel is 1.6 % slower (1.482 vs
// 1.458 ms on cfg5), but the 16 K registers it leaves per SM let the far-field CTAs (basis
// stream, rotation M2M, M2L) co-reside: the upward pass ends under the near field instead of
// 0.19 ms after it (cfg5 465 -> 473 mat-vecs/s, cfg2 5 850 -> 6 050; 96 registers spill: 408).
#ifndef LAPD_BOUND_EXTRA
#define LAPD_BOUND_EXTRA 128
#endif
template <int NCT, int NSTG>
__global__ void __launch_bounds__(NCT + LAPD_PROD + LAPD_BOUND_EXTRA, 1)
k_p2p_lapd(TreeDev T, const LapdHdr* __restrict__ hdrs, int n_items, const int4* __restrict__ gl_ltab,
           const int* __restrict__ gl_slot, const int* __restrict__ gl_spec, int max_src, int max_leaves, int max_tgt,
           const double2* __restrict__ srec, const int* __restrict__ s_panel, const int* __restrict__ s_code,
           const double* __restrict__ xd, double* __restrict__ part, unsigned* __restrict__ sched,
           long long* __restrict__ trace) {
  constexpr int TPT = LAPD_TPT, NPT = LAPD_PROD, ALL = NCT + NPT;
  // optional per-item clock trace (FMMBEM_P2P_TRACE): [cta][item < 32][8]
#define TR(k, j)                                                              \
  if (trace && (k) < 32) trace[((size_t)blockIdx.x * 32 + (k)) * 8 + (j)] = (long long)globaltimer_ns()
  extern __shared__ __align__(16) unsigned char smem[];
  const LapdStage L(max_src, max_leaves, max_tgt);
  double* red = reinterpret_cast<double*>(smem + NSTG * L.bytes);  // [NSTG][NCT * TPT] group partials
  __shared__ int s_idx;
  __shared__ unsigned s_done[NSTG];  // consumer warps done with the stage's item
  __shared__ unsigned long long s_full[NSTG];  // FULL mbarriers (NPT arrivals per phase)
  if (threadIdx.x < NSTG) {
    s_done[threadIdx.x] = 0u;
    mbar_init(&s_full[threadIdx.x], NPT);
  }
  __syncthreads();
  // stage item `cur` into stage st with threads tid < nthr (false: the schedule is exhausted)
  auto stage = [&](int cur, int st, int tid, int nthr, bool all) -> bool {
    unsigned char* base = smem + st * L.bytes;
    double2* sh2 = reinterpret_cast<double2*>(base);
    int4* ltab = reinterpret_cast<int4*>(base + L.ltab);
    int* slot = reinterpret_cast<int*>(base + L.slot);
    double2* tg = reinterpret_cast<double2*>(base + L.tgt);
    int* spec = slot + max_tgt;  // tile positions (item order) of the targets' own sources
    int* hdr = spec + max_tgt;   // live (0: done), ns, nt, out_off, nspec, n1, n2, n3
    if (cur >= n_items) {
      if (tid == 0) hdr[0] = 0;
      return false;
    }
    const LapdHdr H = hdrs[cur];
    for (int q = tid; q < H.nl; q += nthr) ltab[q] = gl_ltab[H.pair_begin + q];
    for (int lt = tid; lt < H.nt; lt += nthr) {
      slot[lt] = gl_slot[H.out_off + lt];
      if (lt < H.nspec) spec[lt] = gl_spec[H.out_off + lt];
      const double x = T.px[H.t0 + lt] - H.cx, y = T.py[H.t0 + lt] - H.cy, z = T.pz[H.t0 + lt] - H.cz;
      tg[lt] = make_double2(x, y);
      tg[max_tgt + lt] = make_double2(z, fma(x, x, fma(y, y, z * z)));
    }
    if (tid == 0) {
      hdr[0] = 1;
      hdr[1] = H.ns;
      hdr[2] = H.nt;
      hdr[3] = H.out_off;
      hdr[4] = H.nspec;
      hdr[5] = H.n1;
      hdr[6] = H.n2;
      hdr[7] = H.n3;
    }
    if (all) __syncthreads();
    else bar_sync(BAR_PROD, NPT);
    // flattened over the tile: SPR sources per thread per round, loads issued before use
    for (int i0 = tid; i0 < H.ns; i0 += SPR * nthr) {
      double2 v[SPR][3];
      int pn[SPR], cd[SPR], o12[SPR], o3[SPR];
#pragma unroll
      for (int u = 0; u < SPR; ++u) {
        const int i = min(i0 + u * nthr, H.ns - 1);
        int lo = 0, hi = H.nl - 1;  // last leaf with offset <= i
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ltab[mid].z <= i) lo = mid;
          else hi = mid - 1;
        }
        const int4 e = ltab[lo];
        const int gi = e.x + i - e.z;
        const size_t g = (size_t)gi * 3;
        v[u][0] = srec[g];
        v[u][1] = srec[g + 1];
        v[u][2] = srec[g + 2];
        pn[u] = s_panel[gi];
        cd[u] = s_code[gi];
        o12[u] = e.y;
        o3[u] = e.w;
      }
      double xv[SPR];
#pragma unroll
      for (int u = 0; u < SPR; ++u) xv[u] = xd[pn[u]];
#pragma unroll
      for (int u = 0; u < SPR; ++u) {
        const int i = i0 + u * nthr;
        if (i >= H.ns) break;
        const int sec = cd[u] & 3, pos = (cd[u] >> 2) & 3, rank = cd[u] >> 4;
        int pt, rec;  // slots in the point planes (0, 1) and the record planes (2, 3)
        if (sec == 0) {
          // single point: own sources first (rank among them), the rest compacted after
          const int sidx = (o12[u] & 0xffff) + rank;
          int r = 0, hi = H.nspec;  // r = number of own sources at single positions < sidx
          while (r < hi) {
            const int mid = (r + hi) >> 1;
            if (spec[mid] < sidx) r = mid + 1;
            else hi = mid;
          }
          pt = rec = (r < H.nspec && spec[r] == sidx) ? r : H.nspec + sidx - r;
        } else if (sec == 1) {
          const int c = (o12[u] >> 16) + rank;
          pt = H.n1 + 2 * c + pos;
          rec = H.n1 + c;
        } else {
          const int c = o3[u] + rank;
          pt = H.n1 + 2 * H.n2 + 3 * c + pos;
          rec = H.n1 + H.n2 + c;
        }
        const double sx = v[u][0].x - H.cx, sy = v[u][0].y - H.cy, sz = v[u][1].x - H.cz;
        const double ss = fma(sx, sx, fma(sy, sy, sz * sz));
        sh2[pt] = make_double2(-2.0 * sx, -2.0 * sy);
        sh2[max_src + pt] = make_double2(-2.0 * sz, ss);
        if (pos == 0) {
          // dipole d = (w n) x[panel] (bemop.py:188-203, 213-216), times the -3/2 of the
          // interaction body's r^-3 = -3/2 y^3 g; a cluster's first point writes the shared one
          const double xs = -1.5 * xv[u];
          const double dx = v[u][1].y * xs, dy = v[u][2].x * xs, dz = v[u][2].y * xs;
          const double ds = fma(dx, sx, fma(dy, sy, dz * sz));
          sh2[2 * max_src + rec] = make_double2(dx, dy);
          sh2[3 * max_src + rec] = make_double2(dz, -ds);
        }
      }
    }
    return true;
  };
  // prologue: the whole CTA stages its first item (nothing to overlap it with yet); the
  // producers then hand it over through FULL like every later item
  unsigned nxt = 0;
  if (threadIdx.x == NCT) {
    TR(0, 0);
    nxt = atomicAdd(sched, 1u);
  }
  const bool live0 = stage(blockIdx.x, 0, threadIdx.x, ALL, true);
  __syncthreads();
  if (threadIdx.x >= NCT) {
    // ------------------------------------------------------------------ producers
    // schedule position blockIdx.x first, then positions gridDim.x + atomicAdd(sched) (the next
    // one requested while the current item is staged)
    const int pt = threadIdx.x - NCT;
    if (pt == 0) {
      TR(0, 1);
      TR(0, 2);
    }
    mbar_arrive(&s_full[0]);
    int k = 1;
    if (live0) {
      for (;; ++k) {
        const int st = k % NSTG;
        if (pt == 0) TR(k, 0);
        if (k >= NSTG) bar_sync(BAR_EMPTY0 + st, ALL);
        if (pt == 0) TR(k, 1);
        if (pt == 0) s_idx = (int)(gridDim.x + nxt);
        bar_sync(BAR_PROD, NPT);
        const int cur = s_idx;
        if (pt == 0) nxt = atomicAdd(sched, 1u);
        const bool live = stage(cur, st, pt, NPT, false);
        if (live && pt == 0) TR(k, 2);
        mbar_arrive(&s_full[st]);
        if (!live) break;
      }
    } else {
      k = 0;
    }
    // match the consumers' EMPTY arrivals of the last NSTG - 1 items
    for (int j = max(0, k - NSTG + 1); j < k; ++j) bar_sync(BAR_EMPTY0 + j % NSTG, ALL);
    __syncwarp();
    if (threadIdx.x == NCT) {
      // the last CTA out resets the schedule for the next launch
      __threadfence();
      if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {
        sched[0] = 0u;
        sched[1] = 0u;
        __threadfence();
      }
    }
    return;
  }
  // -------------------------------------------------------------------- consumers
  for (int k = 0;; ++k) {
    const int st = k % NSTG;
    const unsigned char* base = smem + st * L.bytes;
    const double2* sh2 = reinterpret_cast<const double2*>(base);
    const int* slot = reinterpret_cast<const int*>(base + L.slot);
    const double2* tg = reinterpret_cast<const double2*>(base + L.tgt);
    const int* hdr = slot + 2 * max_tgt;
    if (threadIdx.x == 0) TR(k, 3);
    mbar_wait(&s_full[st], (unsigned)(k / NSTG) & 1u);
    if (threadIdx.x == 0) TR(k, 4);
    if (hdr[0] == 0) break;
    const int nt = hdr[2], out_off = hdr[3], nspec = hdr[4];
    const int ns = hdr[5], n2 = hdr[6], n3 = hdr[7];  // (ns: the single points; then the clusters)
    // thread groups: nsl target slots (TPT targets each) x G source groups
    const int nsl = (nt + TPT - 1) / TPT;
    const int G = NCT / nsl;
    const int sl = threadIdx.x % nsl, g = threadIdx.x / nsl;
    double acc[TPT], tx[TPT], ty[TPT], tz[TPT], tt[TPT];
    int self[TPT];
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
      const int lt = min(sl + q * nsl, nt - 1);
      const double2 xy = tg[lt], zt = tg[max_tgt + lt];
      tx[q] = xy.x;
      ty[q] = xy.y;
      tz[q] = zt.x;
      tt[q] = zt.y;
      acc[q] = 0.0;
      self[q] = slot[lt];
    }
    if (g < G) {
      // the self mask costs 2 issue slots per interaction: only the (at most TPT) iterations
      // that meet a target's own source run the masked body; the loop is split around them
      // the tile holds the item's targets' own sources first (j < nspec): only those iterations
      // need the self mask (2 issue slots per interaction)
      int j = g;
      for (; j < nspec; j += G) lapd_body<TPT, true>(lapd_load(sh2, max_src, j), j, tx, ty, tz, tt, self, acc);
      // software-pipelined: the next source's tile entry is read while this one is used
      if (j < ns) {
#if LAPD_SPT == 3
        // three sources per trip: 3 TPT independent chains in flight
        for (; j + 2 * G < ns; j += 3 * G) {
          const LapdSrc u = lapd_load(sh2, max_src, j);
          const LapdSrc v = lapd_load(sh2, max_src, j + G);
          const LapdSrc w2 = lapd_load(sh2, max_src, j + 2 * G);
          lapd_body<TPT, false>(u, j, tx, ty, tz, tt, self, acc);
          lapd_body<TPT, false>(v, j + G, tx, ty, tz, tt, self, acc);
          lapd_body<TPT, false>(w2, j + 2 * G, tx, ty, tz, tt, self, acc);
        }
        for (; j < ns; j += G) lapd_body<TPT, false>(lapd_load(sh2, max_src, j), j, tx, ty, tz, tt, self, acc);
#else
        LapdSrc u = lapd_load(sh2, max_src, j);
        for (; j + G < ns; j += 2 * G) {
          // two sources per trip: 2 TPT independent chains in flight
          const LapdSrc v = lapd_load(sh2, max_src, j + G);
          const LapdSrc w2 = lapd_load(sh2, max_src, min(j + 2 * G, ns - 1));
          lapd_body<TPT, false>(u, j, tx, ty, tz, tt, self, acc);
          lapd_body<TPT, false>(v, j + G, tx, ty, tz, tt, self, acc);
          u = w2;
        }
        if (j < ns) lapd_body<TPT, false>(u, j, tx, ty, tz, tt, self, acc);
#endif
      }
      lapd_run_clusters<TPT, 2>(sh2, max_src, ns, ns, n2, g, G, tx, ty, tz, tt, acc);
      lapd_run_clusters<TPT, 3>(sh2, max_src, ns + n2, ns + 2 * n2, n3, g, G, tx, ty, tz, tt, acc);
    }
    if (threadIdx.x == 0) TR(k, 5);
    if (threadIdx.x == NCT - 32) TR(k, 6);
    // group partials into this stage's reduction area; the last warp to finish sums them in
    // group order (deterministic) while the others move on to the next stage
    double* rd = red + st * NCT * TPT;
    if (g < G)
#pragma unroll
      for (int q = 0; q < TPT; ++q) rd[(g * TPT + q) * nsl + sl] = acc[q];
    __threadfence_block();
    __syncwarp();
    unsigned last = 0;
    if ((threadIdx.x & 31) == 0) last = atomicAdd(&s_done[st], 1u) == NCT / 32 - 1;
    if (__shfl_sync(0xffffffffu, last, 0)) {
      __threadfence_block();
      for (int lt = threadIdx.x & 31; lt < nt; lt += 32) {
        const int q = lt / nsl, s2 = lt - q * nsl;
        double r = 0.0;
        for (int gg = 0; gg < G; ++gg) r += rd[(gg * TPT + q) * nsl + s2];
        part[out_off + lt] = r;
      }
      if ((threadIdx.x & 31) == 0) s_done[st] = 0u;
      __syncwarp();
    }
    bar_arrive(BAR_EMPTY0 + st, ALL);  // stage (and, for the last warp, its reduction area) released
    if (threadIdx.x == 0) TR(k, 7);
  }
}

long long* p2p_trace_buffer();

bool p2p_lapd_usable(const P2PAux* aux, int max_sources) {
  const int ms = std::max(max_sources, 1);
  return aux && aux->ready && aux->max_tgt <= LAPD_CONS * LAPD_TPT &&
         2 * (LapdStage(ms, aux->max_leaves, aux->max_tgt).bytes + (size_t)384 * LAPD_TPT * sizeof(double)) <=
             227 * 1024;
}

void P2PAux::build(const Tree& S, const Tree& T, const std::vector<P2PItem>& items,
                   const std::vector<int>& p2p_src, const std::vector<int>& self_src_sorted,
                   cudaStream_t st) {
  // tile sections per source leaf (see lapd_body_cl): the outer far-rule points of one panel
  // inside one leaf form a cluster of 2 or 3; centroids (Gauss point 0, bemop.py:64-70) and lone
  // outer points stay singles.  FMMBEM_P2P_CLUSTER=0 keeps every point single.
  static const bool cluster = !(std::getenv("FMMBEM_P2P_CLUSTER") && std::atoi(std::getenv("FMMBEM_P2P_CLUSTER")) == 0);
  const std::vector<int> perm = S.perm.download(st);
  std::vector<int> cd(std::max<size_t>(perm.size(), 1), 0);
  std::vector<int> c1(S.n_cells, 0), c2(S.n_cells, 0), c3(S.n_cells, 0);
  {
    std::vector<std::pair<int, int>> pts;  // (original index = 4 panel + k, sorted index)
    for (const int leaf : S.h_leaves) {
      const int s0 = S.h_body_start[leaf], cnt = S.h_body_count[leaf];
      pts.clear();
      for (int i = 0; i < cnt; ++i) pts.emplace_back(perm[s0 + i], s0 + i);
      std::sort(pts.begin(), pts.end());
      int r1 = 0, r2 = 0, r3 = 0;
      for (size_t a = 0; a < pts.size();) {
        size_t b = a;
        while (b < pts.size() && pts[b].first / 4 == pts[a].first / 4) ++b;
        size_t o = a;  // the panel's outer points [o, b)
        if (pts[a].first % 4 == 0) cd[pts[o++].second] = 0 | (r1++ << 4);
        const int m = (int)(b - o);
        if (!cluster || m == 1) {
          for (; o < b; ++o) cd[pts[o].second] = 0 | (r1++ << 4);
        } else if (m == 2) {
          for (int q = 0; q < 2; ++q) cd[pts[o + q].second] = 1 | (q << 2) | (r2 << 4);
          ++r2;
        } else if (m == 3) {
          for (int q = 0; q < 3; ++q) cd[pts[o + q].second] = 2 | (q << 2) | (r3 << 4);
          ++r3;
        }
        a = b;
      }
      c1[leaf] = r1;
      c2[leaf] = r2;
      c3[leaf] = r3;
    }
  }
  std::vector<int4> lt(std::max<size_t>(p2p_src.size(), 1), make_int4(0, 0, 0, 0));
  int64_t part_len = 0;
  for (const auto& it : items) part_len = std::max<int64_t>(part_len, it.out_off + T.h_body_count[it.tgt_leaf]);
  std::vector<int> sl(std::max<int64_t>(part_len, 1), -1), sp(std::max<int64_t>(part_len, 1), 0);
  std::vector<int> nspec_of(items.size(), 0);
  std::vector<int4> sect(items.size(), make_int4(0, 0, 0, 0));  // (n1, n2, n3, ns) per item
  max_leaves = 1;
  max_tgt = 1;
  for (const auto& it : items) {
    int off = 0, o1 = 0, o2 = 0, o3 = 0;
    for (int k = it.pair_begin; k < it.pair_end; ++k) {
      const int leaf = p2p_src[k];
      FMM_REQUIRE(o1 < 65536 && o2 < 32768, "P2P: item too large for the packed section offsets");
      lt[k] = make_int4(S.h_body_start[leaf], o1 | (o2 << 16), off, o3);
      off += S.h_body_count[leaf];
      o1 += c1[leaf];
      o2 += c2[leaf];
      o3 += c3[leaf];
    }
    sect[&it - items.data()] = make_int4(o1, o2, o3, off);
    const int t0 = T.h_body_start[it.tgt_leaf], nt = T.h_body_count[it.tgt_leaf];
    std::vector<std::pair<int, int>> own;  // (position among the item's singles, target)
    for (int l = 0; l < nt; ++l) {
      const int gs = self_src_sorted[t0 + l];
      for (int k = it.pair_begin; k < it.pair_end; ++k) {
        const int leaf = p2p_src[k];
        if (gs >= lt[k].x && gs < lt[k].x + S.h_body_count[leaf]) own.emplace_back((lt[k].y & 0xffff) + (cd[gs] >> 4), l);
      }
    }
    std::sort(own.begin(), own.end());
    for (size_t r = 0; r < own.size(); ++r) {
      sl[it.out_off + own[r].second] = (int)r;  // the own source sits at tile slot r
      sp[it.out_off + r] = own[r].first;
    }
    nspec_of[&it - items.data()] = (int)own.size();
    max_leaves = std::max(max_leaves, it.pair_end - it.pair_begin);
    max_tgt = std::max(max_tgt, nt);
  }
  const std::vector<int> ord = p2p_schedule(T, S, items, p2p_src);
  std::vector<LapdHdr> h(std::max<size_t>(ord.size(), 1));
  for (size_t r = 0; r < ord.size(); ++r) {
    const P2PItem& it = items[ord[r]];
    LapdHdr& e = h[r];
    e.pair_begin = it.pair_begin;
    e.nl = it.pair_end - it.pair_begin;
    e.ns = sect[ord[r]].w;
    e.n1 = sect[ord[r]].x;
    e.n2 = sect[ord[r]].y;
    e.n3 = sect[ord[r]].z;
    e.t0 = T.h_body_start[it.tgt_leaf];
    e.nt = T.h_body_count[it.tgt_leaf];
    e.out_off = it.out_off;
    e.nspec = nspec_of[ord[r]];
    e.cx = T.h_cx[it.tgt_leaf];
    e.cy = T.h_cy[it.tgt_leaf];
    e.cz = T.h_cz[it.tgt_leaf];
  }
  n_items = (int)items.size();
  if (std::getenv("FMMBEM_P2P_STATS")) {
    double w1 = 0, w2 = 0, w3 = 0, wspec = 0;
    for (size_t i = 0; i < items.size(); ++i) {
      const double nt = T.h_body_count[items[i].tgt_leaf];
      w1 += nt * sect[i].x, w2 += nt * 2.0 * sect[i].y, w3 += nt * 3.0 * sect[i].z, wspec += nt * nspec_of[i];
    }
    std::fprintf(stderr, "[fmmbem] P2P tile sections by interactions: singles %.4f (own %.4f) pairs %.4f triples %.4f of %.4g\n",
                 w1 / (w1 + w2 + w3), wspec / (w1 + w2 + w3), w2 / (w1 + w2 + w3), w3 / (w1 + w2 + w3), w1 + w2 + w3);
  }
  p2p_trace_buffer();  // (allocated here, outside any stream capture)
  hdr.upload(h, st);
  ltab.upload(lt, st);
  slot.upload(sl, st);
  spec.upload(sp, st);
  code.upload(cd, st);
  ready = true;
}

// FMMBEM_P2P_TRACE=1: a per-item clock trace of the double-layer kernel, read by fmmbem_debug_p2p_trace
long long* p2p_trace_buffer() {
  static long long* buf = nullptr;
  if (!buf && std::getenv("FMMBEM_P2P_TRACE")) {
    FMM_CUDA(cudaMalloc(&buf, (size_t)1024 * 32 * 8 * sizeof(long long)));
    FMM_CUDA(cudaMemset(buf, 0, (size_t)1024 * 32 * 8 * sizeof(long long)));
  }
  return buf;
}

void launch_p2p_lapd(const TreeDev& T, const P2PAux& aux, int max_src, const double2* srec,
                     const int* s_panel, const double* x, double* part, cudaStream_t st, unsigned* sched) {
  const LapdStage L(max_src, aux.max_leaves, aux.max_tgt);
  constexpr int nct = LAPD_CONS;
  const size_t per = L.bytes + (size_t)nct * LAPD_TPT * sizeof(double);
  // 2 stages: measured faster than 3 inside the concurrent step (the far-field kernels share the
  // SMs' shared memory with this persistent kernel); FMMBEM_P2P_STAGES=3 for a deeper ring
  static const int want = std::getenv("FMMBEM_P2P_STAGES") ? std::atoi(std::getenv("FMMBEM_P2P_STAGES")) : 2;
  const int nstg = (want >= 3 && 3 * per <= 227 * 1024) ? 3 : 2;
  const size_t smem = nstg * per;
  FMM_REQUIRE(smem <= 227 * 1024, "P2P: source slice too large for shared memory");
  FMM_REQUIRE(sched != nullptr, "P2P: the double-layer kernel needs its schedule counter");
  auto kern = nstg == 3 ? k_p2p_lapd<LAPD_CONS, 3> : k_p2p_lapd<LAPD_CONS, 2>;
  const int nthr = LAPD_CONS + LAPD_PROD;
  FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // shared-memory carveout of the SMs this persistent kernel occupies: the far-field kernels
  // launched beside it can only co-reside in what the configuration leaves over
  // (FMMBEM_P2P_CARVEOUT=percent, -1 = driver default)
  // default: the maximum -- with the driver's choice (164 KB for this kernel's 150 KB) a far-field
  // CTA that needs more than ~12 KB of shared memory cannot be placed beside it
  static const int carve = std::getenv("FMMBEM_P2P_CARVEOUT") ? std::atoi(std::getenv("FMMBEM_P2P_CARVEOUT")) : 100;
  if (carve >= 0)
    FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  int dev = 0, sms = 0;
  FMM_CUDA(cudaGetDevice(&dev));
  FMM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // FMMBEM_P2P_RESERVE=k leaves k SMs without a near-field CTA (for the far-field chain)
  static const int reserve = std::getenv("FMMBEM_P2P_RESERVE") ? std::atoi(std::getenv("FMMBEM_P2P_RESERVE")) : 0;
  const int grid = std::min(aux.n_items, std::max(1, sms - reserve));
  if (grid > 0)
    kern<<<grid, nthr, smem, st>>>(T, aux.hdr.get(), aux.n_items, aux.ltab.get(), aux.slot.get(),
                                   aux.spec.get(), max_src,
                                   aux.max_leaves, aux.max_tgt, srec, s_panel, aux.code.get(), x, part, sched,
                                   p2p_trace_buffer());
  FMM_LAUNCH_CHECK();
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
                cudaStream_t st, const int* order, const P2PAux* aux, unsigned* sched,
                const double2* srec, const int* s_panel, const double* x) {
  const int ms = std::max(max_sources, 1);
  switch (kind) {
    case P2PKind::LAP_Q: return launch_p2p_t<P2PKind::LAP_Q>(S, T, items, n_items, p2p_src, ms, w, part, st, order);
    case P2PKind::LAP_D:
      if (p2p_lapd_usable(aux, ms) && sched && srec && s_panel && x)
        return launch_p2p_lapd(T, *aux, ms, srec, s_panel, x, part, st, sched);
      return launch_p2p_t<P2PKind::LAP_D>(S, T, items, n_items, p2p_src, ms, w, part, st, order);
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

extern "C" int fmmbem_debug_p2p_trace(long long* host, int64_t n) {
  long long* b = fmmbem::p2p_trace_buffer();
  if (!b) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  const size_t m = std::min<size_t>((size_t)n, (size_t)1024 * 32 * 8);
  return cudaMemcpy(host, b, m * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 3;
}
