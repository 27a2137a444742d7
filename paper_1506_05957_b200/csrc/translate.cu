// Expansion translations (M2L, M2M, L2L) on one register-tiled engine.
//
// Reference operators (harmonics.py:156-218, applied in fmm.py:268-314):
//   M2L  L_j^k  += (-1)^j sum_{n<=p,|m|<=n} M_n^m conj(I_{n+j}^{m+k}(D))   D = c_t - c_s
//   M2M  M'_n^m += sum_{j<=n,k} M_j^k R_{n-j}^{m-k}(d)                     d = c_child - c_parent
//   L2L  L'_n^m += sum_{j>=n,k} L_j^k R_{j-n}^{k-m}(d)                     d = c_child - c_parent
// (the reference applies them as zgemm with dense (p+1)^2 x (p+1)^2 operators).
//
// One CTA owns one output expansion.  M2L / L2L: 4 warps stream the input
// expansions ("pairs") through double-buffered shared memory - the operator
// table (the full conj(I(D)) grid of order 2p, or the R(d) grid of order p)
// arrives by cp.async while the previous pair is being contracted - and split
// the input orders among themselves.  M2M: one warp per child, each with its
// own buffer.  Lane l owns output order oc(l) and BJ consecutive output
// degrees r0(l)..r0+BJ-1.
// For a fixed input order, the table rows each lane needs slide by one row per
// input degree, so every step is one shared-memory load of the operator, one
// broadcast load of the input coefficient per channel, and BJ*CK complex FMAs;
// the window rotates through registers by unrolling.  Warps are summed in a
// fixed order at the end: deterministic, no atomics.  Outputs are half-stored
// (m >= 0); inputs are expanded to full storage while staging.
#include "kernels.cuh"

namespace fmmbem {

enum TMode : int { T_M2L = 0, T_M2M = 1, T_L2L = 2 };
constexpr int TR_WARPS = 4;

__host__ __device__ constexpr int tr_tiles(int p, int bj) {
  int t = 0;
  for (int k = 0; k <= p; ++k) t += (p - k + 1 + bj - 1) / bj;
  return t;
}
__host__ __device__ constexpr int tr_bj(int p) {
  int bj = 1;
  while (tr_tiles(p, bj) > 32) ++bj;
  return bj;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

struct TrArgs {
  const int4* items;        // M2L: (out cell, pair begin, pair end, item id)
  const int* cells;         // M2M / L2L: output cells
  const int* pair_in;       // M2L: source cell per pair
  const int* pair_tab;      // M2L: offset id per pair
  const int* first_child;   // M2M
  const int* n_child;       // M2M
  const int* parent;        // L2L
  const int* rtab;          // M2M / L2L: (level * 8 + octant) per cell
  const double2* table;     // operator tables
  int table_stride;         // complex per table entry
  const double2* in;        // input expansions [cell][Ctot][H]
  double2* out;             // M2L: partial blocks [item][Ctot][H]; else [cell][Ctot][H]
  int Ctot, cbase;
};

template <int MODE> struct TrCfg {
  static constexpr bool SPLIT_PAIRS = MODE == T_M2M;   // warps per input expansion (child)
  static constexpr int MSPLIT = MODE == T_M2M ? 2 : 1;  // warps sharing one child
  static constexpr int WARPS = MODE == T_M2M ? 16 : TR_WARPS;
};

template <int P, int CK, int MODE>
__global__ void __launch_bounds__(TrCfg<MODE>::WARPS * 32) k_translate(TrArgs a) {
  constexpr int BJ = tr_bj(P);
  constexpr int H = (P + 1) * (P + 2) / 2;
  constexpr int S = (P + 1) * (P + 1);
  constexpr int TQ = MODE == T_M2L ? 2 * P : P;  // table order
  constexpr bool SPLIT_PAIRS = TrCfg<MODE>::SPLIT_PAIRS;
  constexpr int NW = TrCfg<MODE>::WARPS;
  const int TT = tab_size(TQ);                    // entries copied per pair
  // M2L reads rows up to 2p + BJ - 1 unclamped: rows past 2p only ever feed
  // output degrees > p (discarded), so the slack rows are left uninitialised
  const int TA = MODE == T_M2L ? tab_size(TQ + BJ) : TT;
  const int BUF = TA + CK * S;
  extern __shared__ double2 sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- this CTA's output and its list of inputs
  int out_cell, e0, e1, item_id = 0;
  if (MODE == T_M2L) {
    const int4 it = a.items[blockIdx.x];
    out_cell = it.x;
    e0 = it.y;
    e1 = it.z;
    item_id = it.w;
  } else if (MODE == T_M2M) {
    out_cell = a.cells[blockIdx.x];
    e0 = a.first_child[out_cell];
    e1 = e0 + a.n_child[out_cell];
  } else {
    out_cell = a.cells[blockIdx.x];
    e0 = 0;
    e1 = 1;
  }
  auto in_cell = [&](int e) {
    return MODE == T_M2L ? a.pair_in[e] : MODE == T_M2M ? e : a.parent[out_cell];
  };
  auto tab_id = [&](int e) {
    return MODE == T_M2L ? a.pair_tab[e] : MODE == T_M2M ? a.rtab[e] : a.rtab[out_cell];
  };
  // stage pair e into buf with `nthr` cooperating threads (thread index tid)
  auto stage = [&](int e, double2* buf, int tid, int nthr) {
    const double2* T = a.table + (size_t)tab_id(e) * a.table_stride;
    for (int i = tid; i < TT; i += nthr) cp_async16(buf + i, T + i);
    cp_async_commit();
    const double2* src = a.in + ((size_t)in_cell(e) * a.Ctot + a.cbase) * H;
    for (int f = tid; f < CK * S; f += nthr) {
      const int c = f / S, g = f - c * S;
      const int n = (int)__fsqrt_rz((float)g);
      buf[TA + f] = hget(src + c * H, n, g - n * n - n);
    }
  };

  // ---- lane tile, tile-major so that consecutive lanes hold consecutive oc
  int oc = -1, r0 = 0;
  {
    int cum = 0;
    for (int tau = 0; tau * BJ <= P; ++tau) {
      const int nt = P - tau * BJ + 1;  // oc = 0 .. P - tau*BJ
      if (oc < 0 && lane < cum + nt) {
        oc = lane - cum;
        r0 = oc + tau * BJ;
      }
      cum += nt;
    }
  }
  const bool active = oc >= 0;
  double2 acc[CK][BJ];
#pragma unroll
  for (int c = 0; c < CK; ++c)
#pragma unroll
    for (int t = 0; t < BJ; ++t) acc[c][t] = make_double2(0.0, 0.0);

  // contract one staged pair over input orders am = -P + ai, ai = a0, a0 + astep, ...
  auto contract = [&](const double2* sT, const double2* sIn, int a0, int astep) {
    for (int ai = a0; ai < 2 * P + 1; ai += astep) {
      const int am = ai - P;
      const int b0 = am < 0 ? -am : am;
      const int col = MODE == T_M2L ? am + oc : MODE == T_M2M ? oc - am : am - oc;
      const int acol = col < 0 ? -col : col;
      auto tval = [&](int row) -> double2 {  // M2M / L2L: masked, clamped
        const int N = min(max(row, 0), TQ);
        const double2 v = sT[pidx(N, max(min(col, N), -N))];
        return row >= acol ? v : make_double2(0.0, 0.0);
      };
      double2 w[BJ];
      int lead = 0, off = 0, dn = 0;
      if (MODE == T_M2L) {
        // rows b0 + r0 + t of conj(I); the entering row's offset is advanced incrementally
#pragma unroll
        for (int t = 0; t < BJ; ++t) w[t] = sT[pidx(b0 + r0 + t, col)];
        lead = b0 + r0 + BJ;
        off = pidx(lead, col);
        dn = 2 * lead + 2;
      } else if (MODE == T_M2M) {
#pragma unroll
        for (int t = 0; t < BJ; ++t) w[t] = tval(r0 + t - b0);
        lead = r0 - b0 - 1;
      } else {
#pragma unroll
        for (int t = 0; t < BJ; ++t) w[t] = tval(b0 - r0 - t);
        lead = b0 + 1 - r0;
      }
      const double2* ip = sIn + b0 * b0 + b0 + am;
      int istep = 2 * b0 + 2;
      int b = b0;
      auto step = [&](int q) {
        double2 mv[CK];
#pragma unroll
        for (int c = 0; c < CK; ++c) mv[c] = ip[c * S];
        ip += istep;
        istep += 2;
#pragma unroll
        for (int t = 0; t < BJ; ++t) {
          const int slot = MODE == T_M2L ? (q + t) % BJ : (t + BJ - q) % BJ;
#pragma unroll
          for (int c = 0; c < CK; ++c) acc[c][t] = cfma(mv[c], w[slot], acc[c][t]);
        }
        if (MODE == T_M2L) {
          w[q] = sT[off];
          off += dn;
          dn += 2;
        } else {
          w[(BJ - 1 - q) % BJ] = tval(lead);
          lead += MODE == T_M2M ? -1 : 1;
        }
      };
      for (; b + BJ - 1 <= P; b += BJ) {
        if (MODE == T_M2L) {
          // issue the block's shared-memory loads first (inputs and entering
          // operator rows), then run its BJ steps: hides the LDS latency
          double2 mvb[BJ][CK], nw[BJ];
#pragma unroll
          for (int q = 0; q < BJ; ++q) {
#pragma unroll
            for (int c = 0; c < CK; ++c) mvb[q][c] = ip[c * S];
            ip += istep;
            istep += 2;
            nw[q] = sT[off];
            off += dn;
            dn += 2;
          }
#pragma unroll
          for (int q = 0; q < BJ; ++q) {
#pragma unroll
            for (int t = 0; t < BJ; ++t)
#pragma unroll
              for (int c = 0; c < CK; ++c) acc[c][t] = cfma(mvb[q][c], w[(q + t) % BJ], acc[c][t]);
            w[q] = nw[q];
          }
        } else {
#pragma unroll
          for (int q = 0; q < BJ; ++q) step(q);
        }
      }
#pragma unroll
      for (int q = 0; q < BJ - 1; ++q)
        if (b + q <= P) step(q);
    }
  };

  if (SPLIT_PAIRS) {
    // every child staged at once (<= 8), then MSPLIT warps per child split its input orders
    constexpr int MS = TrCfg<MODE>::MSPLIT;
    for (int e = e0; e < e1; ++e) stage(e, sh + (e - e0) * BUF, threadIdx.x, blockDim.x);
    cp_async_wait_all();
    __syncthreads();
    const int g = warp / MS;
    if (active && e0 + g < e1) contract(sh + g * BUF, sh + g * BUF + TA, warp % MS, MS);
  } else {
    if (e1 > e0) stage(e0, sh, threadIdx.x, blockDim.x);
    for (int e = e0; e < e1; ++e) {
      double2* cur = sh + ((e - e0) & 1) * BUF;
      cp_async_wait_all();
      __syncthreads();
      if (e + 1 < e1) stage(e + 1, sh + ((e + 1 - e0) & 1) * BUF, threadIdx.x, blockDim.x);
      if (active) contract(cur, cur + TA, warp, NW);
    }
  }
  // ---- fixed-order reduction over the warps
  __syncthreads();
  double2* red = sh;  // [NW][32][CK][BJ]
#pragma unroll
  for (int c = 0; c < CK; ++c)
#pragma unroll
    for (int t = 0; t < BJ; ++t) red[((warp * 32 + lane) * CK + c) * BJ + t] = acc[c][t];
  __syncthreads();
  if (warp == 0 && active) {
#pragma unroll
    for (int c = 0; c < CK; ++c)
#pragma unroll
      for (int t = 0; t < BJ; ++t) {
        const int r = r0 + t;
        if (r > P) continue;
        double2 s = red[(lane * CK + c) * BJ + t];
        for (int w2 = 1; w2 < NW; ++w2) s = cadd(s, red[((w2 * 32 + lane) * CK + c) * BJ + t]);
        const int idx = r * (r + 1) / 2 + oc;
        if (MODE == T_M2L) {
          if (r & 1) s = make_double2(-s.x, -s.y);
          a.out[((size_t)item_id * a.Ctot + a.cbase + c) * H + idx] = s;
        } else if (MODE == T_M2M) {
          a.out[((size_t)out_cell * a.Ctot + a.cbase + c) * H + idx] = s;
        } else {
          double2* d = a.out + ((size_t)out_cell * a.Ctot + a.cbase + c) * H + idx;
          *d = cadd(*d, s);
        }
      }
  }
}

template <int P, int CK, int MODE>
size_t tr_smem() {
  constexpr int S = (P + 1) * (P + 1);
  constexpr int TQ = MODE == T_M2L ? 2 * P : P;
  const size_t one = (size_t)((MODE == T_M2L ? tab_size(TQ + tr_bj(P)) : tab_size(TQ)) + CK * S);
  const size_t buf = TrCfg<MODE>::SPLIT_PAIRS ? 8 * one : 2 * one;
  const size_t red = (size_t)TrCfg<MODE>::WARPS * 32 * CK * tr_bj(P);
  return std::max(buf, red) * sizeof(double2);
}

template <int P, int CK, int MODE>
void tr_launch_one(int nblocks, const TrArgs& a, cudaStream_t st) {
  const size_t sm = tr_smem<P, CK, MODE>();
  static DeviceOnce attr;
  if (attr.first()) {
    FMM_CUDA(cudaFuncSetAttribute(k_translate<P, CK, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sm));
    attr.mark();
  }
  k_translate<P, CK, MODE><<<nblocks, TrCfg<MODE>::WARPS * 32, sm, st>>>(a);
}

template <int P, int MODE>
void tr_launch_groups(int nblocks, TrArgs a, cudaStream_t st) {
  constexpr size_t LIMIT = 227 * 1024;
  // channel groups of 4 / 2 / 1 (Ctot = 1, 4 or 7), as large as shared memory allows -- and as
  // the register file allows: the 4-channel kernels of orders >= 16 and the 2-channel one of
  // order 20 spilled 39-62 KB per thread, so those orders take narrower groups
  constexpr int CK_MAX = P >= 20 ? 1 : P >= 16 ? 2 : 4;
  for (int cb = 0; cb < a.Ctot;) {
    const int rem = a.Ctot - cb;
    a.cbase = cb;
    if constexpr (CK_MAX >= 4) {
      if (rem >= 4 && tr_smem<P, 4, MODE>() <= LIMIT) {
        tr_launch_one<P, 4, MODE>(nblocks, a, st);
        cb += 4;
        continue;
      }
    }
    if constexpr (CK_MAX >= 2) {
      if (rem >= 2 && tr_smem<P, 2, MODE>() <= LIMIT) {
        tr_launch_one<P, 2, MODE>(nblocks, a, st);
        cb += 2;
        continue;
      }
    }
    {
      const bool fits = tr_smem<P, 1, MODE>() <= LIMIT;
      FMM_REQUIRE(fits, "translation tiles exceed shared memory");
      tr_launch_one<P, 1, MODE>(nblocks, a, st);
      cb += 1;
    }
  }
  FMM_LAUNCH_CHECK();
}

template <int MODE>
void tr_dispatch(int p, int nblocks, const TrArgs& a, cudaStream_t st) {
  if (nblocks <= 0) return;
  switch (p) {
#define TR_CASE(PP) case PP: tr_launch_groups<PP, MODE>(nblocks, a, st); break;
    TR_CASE(0) TR_CASE(1) TR_CASE(2) TR_CASE(3) TR_CASE(4) TR_CASE(5) TR_CASE(6)
    TR_CASE(7) TR_CASE(8) TR_CASE(9) TR_CASE(10) TR_CASE(11) TR_CASE(12) TR_CASE(13)
    TR_CASE(14) TR_CASE(15) TR_CASE(16) TR_CASE(17) TR_CASE(18) TR_CASE(19) TR_CASE(20)
#undef TR_CASE
    default: throw ArgumentError("translation: expansion order out of range");
  }
}

// ------------------------------------------------------------------ I grids (setup)
// conj(I_n^m(D)) in FULL flat storage n^2+n+m for n <= order
__global__ void k_igrid_full(const double* off, int n_off, int order, double2* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_off) return;
  const double x = off[3 * i], y = off[3 * i + 1], z = off[3 * i + 2];
  double2* o = out + (size_t)i * tab_size(order);
  const double rho2 = x * x + y * y + z * z;
  const double inv_r2 = 1.0 / rho2;
  double2 diag = make_double2(1.0 / sqrt(rho2), 0.0);
  auto put = [&](int n, int m, double2 v) {
    // stored conjugated: the M2L contraction uses conj(I) (harmonics.py:180-198)
    o[pidx(n, m)] = make_double2(v.x, -v.y);
    if (m > 0) o[pidx(n, -m)] = (m & 1) ? make_double2(-v.x, -v.y) : v;
  };
  for (int m = 0; m <= order; ++m) {
    if (m > 0) diag = cscale(cmul(make_double2(x, y), diag), -(2.0 * m - 1.0) * inv_r2);
    put(m, m, diag);
    if (m + 1 <= order) {
      double2 prev2 = diag;
      double2 prev1 = cscale(diag, (2.0 * m + 1.0) * z * inv_r2);
      put(m + 1, m, prev1);
      for (int n = m + 2; n <= order; ++n) {
        const double aa = (2 * n - 1) * z;
        const double bb = (double)((n - 1) * (n - 1) - m * m);
        double2 cur;
        cur.x = (aa * prev1.x - bb * prev2.x) * inv_r2;
        cur.y = (aa * prev1.y - bb * prev2.y) * inv_r2;
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

// L[cell] = sum of its M2L items' partial blocks (cells without items get zeros)
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

// ------------------------------------------------------------------ M2L, offset-grouped
// One CTA per (translation offset, <= 8 pairs): the conj(I(D)) grid is staged
// once and applied to NV = 4 input vectors at a time (4 pairs x 1 channel, or
// 1 pair x 4 channels), so every gathered operator value feeds 4*BJ complex
// FMAs; the 4 warps split the input orders.  Each pair's result is written to
// its CSR slot and a second kernel adds a target's pairs in CSR order
// (deterministic).
template <int P, int CK>
__global__ void __launch_bounds__(TR_WARPS * 32)
k_m2l_grouped(const int4* __restrict__ items, const int* __restrict__ gpair,
              const int* __restrict__ pair_src, const double2* __restrict__ table, int table_stride,
              const double2* __restrict__ M, int Ctot, int cbase, double2* __restrict__ pout) {
  constexpr int BJ = tr_bj(P);
  constexpr int H = (P + 1) * (P + 2) / 2;
  constexpr int S = (P + 1) * (P + 1);
  constexpr int TQ = 2 * P;
  constexpr int NV = 4;            // vectors per contraction pass
  constexpr int NP = NV / CK;      // pairs per pass
  const int TT = tab_size(TQ), TA = tab_size(TQ + BJ);
  extern __shared__ double2 sh[];
  double2* sT = sh;
  double2* sM = sh + TA;           // [NV][S]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 it = items[blockIdx.x];
  {
    const double2* T = table + (size_t)it.x * table_stride;
    for (int i = threadIdx.x; i < TT; i += blockDim.x) cp_async16(sT + i, T + i);
    cp_async_commit();
  }
  int oc = -1, r0 = 0;
  {
    int cum = 0;
    for (int kk = 0; kk <= P; ++kk) {
      const int nt = (P - kk + 1 + BJ - 1) / BJ;
      if (oc < 0 && lane < cum + nt) {
        oc = kk;
        r0 = kk + (lane - cum) * BJ;
      }
      cum += nt;
    }
  }
  const bool active = oc >= 0;
  for (int e0 = it.y; e0 < it.z; e0 += NP) {
    const int np = min(NP, it.z - e0);
    const int nv = np * CK;
    __syncthreads();  // previous pass done with sM
    for (int f = threadIdx.x; f < NV * S; f += blockDim.x) {
      const int v = f / S, g = f - v * S;
      double2 val = make_double2(0.0, 0.0);
      if (v < nv) {
        const int e = gpair[e0 + v / CK], c = cbase + v % CK;
        const int n = (int)__fsqrt_rz((float)g);
        val = hget(M + ((size_t)pair_src[e] * Ctot + c) * H, n, g - n * n - n);
      }
      sM[f] = val;
    }
    cp_async_wait_all();
    __syncthreads();
    double2 acc[NV][BJ];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int t = 0; t < BJ; ++t) acc[v][t] = make_double2(0.0, 0.0);
    if (active) {
      for (int ai = warp; ai < 2 * P + 1; ai += TR_WARPS) {
        const int am = ai - P;
        const int b0 = am < 0 ? -am : am;
        const int col = am + oc;
        double2 w[BJ];
#pragma unroll
        for (int t = 0; t < BJ; ++t) w[t] = sT[pidx(b0 + r0 + t, col)];
        int off = pidx(b0 + r0 + BJ, col), dn = 2 * (b0 + r0 + BJ) + 2;
        const double2* ip = sM + b0 * b0 + b0 + am;
        int istep = 2 * b0 + 2;
        auto step = [&](int q) {
          double2 mv[NV];
#pragma unroll
          for (int v = 0; v < NV; ++v) mv[v] = ip[v * S];
          const double2 nw = sT[off];
          ip += istep;
          istep += 2;
          off += dn;
          dn += 2;
#pragma unroll
          for (int t = 0; t < BJ; ++t)
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v][t] = cfma(mv[v], w[(q + t) % BJ], acc[v][t]);
          w[q] = nw;
        };
        int b = b0;
        for (; b + BJ - 1 <= P; b += BJ) {
#pragma unroll
          for (int q = 0; q < BJ; ++q) step(q);
        }
#pragma unroll
        for (int q = 0; q < BJ - 1; ++q)
          if (b + q <= P) step(q);
      }
    }
    // fixed-order reduction over the 4 warps, one vector at a time
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      __syncthreads();
      double2* red = sM;  // reuse: [4 warps][32][BJ] <= NV * S
#pragma unroll
      for (int t = 0; t < BJ; ++t) red[(warp * 32 + lane) * BJ + t] = acc[v][t];
      __syncthreads();
      if (warp == 0 && active && v < nv) {
        const int e = gpair[e0 + v / CK], c = cbase + v % CK;
#pragma unroll
        for (int t = 0; t < BJ; ++t) {
          const int r = r0 + t;
          if (r > P) continue;
          double2 sum = red[lane * BJ + t];
          for (int w2 = 1; w2 < TR_WARPS; ++w2) sum = cadd(sum, red[(w2 * 32 + lane) * BJ + t]);
          if (r & 1) sum = make_double2(-sum.x, -sum.y);
          pout[((size_t)e * Ctot + c) * H + r * (r + 1) / 2 + oc] = sum;
        }
      }
    }
  }
}

// L[cell] = sum over the cell's M2L pairs (CSR order) of their results: 64
// coefficients x 4 pair slices per CTA, slices added in a fixed order
__global__ void __launch_bounds__(256)
k_m2l_gather(const int* __restrict__ cells, const int* __restrict__ row, int CH,
             const double2* __restrict__ pout, double2* __restrict__ L) {
  __shared__ double2 red[4][64];
  const int cell = cells ? cells[blockIdx.x] : blockIdx.x;
  const int t = blockIdx.y * 64 + (threadIdx.x & 63), q = threadIdx.x >> 6;
  const int i0 = row[cell], i1 = row[cell + 1];
  double2 s = make_double2(0.0, 0.0);
  pdl_wait();  // the M2L results are complete past this point
  if (t < CH)
    for (int i = i0 + q; i < i1; i += 4) s = cadd(s, pout[(size_t)i * CH + t]);
  red[q][threadIdx.x & 63] = s;
  __syncthreads();
  if (q == 0 && t < CH) {
    const int l = threadIdx.x;
    L[(size_t)cell * CH + t] = cadd(cadd(red[0][l], red[1][l]), cadd(red[2][l], red[3][l]));
  }
}

template <int P, int CK>
size_t m2lg_smem() {
  constexpr int S = (P + 1) * (P + 1);
  const size_t red = (size_t)TR_WARPS * 32 * tr_bj(P);
  return ((size_t)tab_size(2 * P + tr_bj(P)) + std::max((size_t)4 * S, red)) * sizeof(double2);
}

template <int P>
void m2lg_launch(const Plan& plan, const int4* gitems, const int* gpair, int n, int C,
                 const double2* M, double2* pout, cudaStream_t st) {
  if (n <= 0) return;
  const int stride = tab_size(2 * plan.igrid_p);
  for (int cb = 0; cb < C;) {
    const int rem = C - cb;
    if (rem >= 4) {
      static DeviceOnce a4;
      if (a4.first()) {
        FMM_CUDA(cudaFuncSetAttribute(k_m2l_grouped<P, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)m2lg_smem<P, 4>()));
        a4.mark();
      }
      k_m2l_grouped<P, 4><<<n, TR_WARPS * 32, m2lg_smem<P, 4>(), st>>>(
          gitems, gpair, plan.m2l_src.get(), plan.igrid.get(), stride,
          M, C, cb, pout);
      cb += 4;
    } else if (rem >= 2) {
      static DeviceOnce a2;
      if (a2.first()) {
        FMM_CUDA(cudaFuncSetAttribute(k_m2l_grouped<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)m2lg_smem<P, 2>()));
        a2.mark();
      }
      k_m2l_grouped<P, 2><<<n, TR_WARPS * 32, m2lg_smem<P, 2>(), st>>>(
          gitems, gpair, plan.m2l_src.get(), plan.igrid.get(), stride,
          M, C, cb, pout);
      cb += 2;
    } else {
      static DeviceOnce a1;
      if (a1.first()) {
        FMM_CUDA(cudaFuncSetAttribute(k_m2l_grouped<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)m2lg_smem<P, 1>()));
        a1.mark();
      }
      k_m2l_grouped<P, 1><<<n, TR_WARPS * 32, m2lg_smem<P, 1>(), st>>>(
          gitems, gpair, plan.m2l_src.get(), plan.igrid.get(), stride,
          M, C, cb, pout);
      cb += 1;
    }
  }
  FMM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ launchers
void launch_m2l(const Plan& plan, int p, int C, const double2* M, double2* L, double2* part,
                cudaStream_t st, const int4* gitems, int n_gitems, const int* cells, int n_cells,
                const int* gpair, const int4* citems, int n_citems, const int* cpair, const RotGroups* rg) {
  // part holds one result block per M2L pair (CSR order): n_m2l * C * hcount(p)
  if (n_cells < 0) n_cells = plan.tgt.n_cells;
  if (plan.use_rot && p >= M2L_ROT_MIN_P && plan.rot_p >= p) {
    // class-grouped items: shared polar-angle tables and |D|, per-vector azimuthal phases;
    // ~30 % fewer warp units than grouping by offset (cfg2 p=12: 41.4 -> 33.2 us with 2-warp CTAs)
    if (!citems) {
      citems = plan.d_m2l_citems.get();
      n_citems = (int)plan.m2l_citems.size();
      cpair = plan.m2l_cpair.get();
      rg = &plan.m2l_rg;
    }
    launch_m2l_rot(plan, citems, cpair, n_citems, p, C, M, part, st, true, rg);
  } else {
  if (!gpair) gpair = plan.m2l_gpair.get();
  if (!gitems) {
    gitems = plan.d_m2l_gitems.get();
    n_gitems = (int)plan.m2l_gitems.size();
  }
  switch (p) {
#define G_CASE(PP) case PP: m2lg_launch<PP>(plan, gitems, gpair, n_gitems, C, M, part, st); break;
    G_CASE(0) G_CASE(1) G_CASE(2) G_CASE(3) G_CASE(4) G_CASE(5) G_CASE(6)
    G_CASE(7) G_CASE(8) G_CASE(9) G_CASE(10) G_CASE(11) G_CASE(12) G_CASE(13)
    G_CASE(14) G_CASE(15) G_CASE(16) G_CASE(17) G_CASE(18) G_CASE(19) G_CASE(20)
#undef G_CASE
    default: throw ArgumentError("M2L: expansion order out of range");
  }
  }
  if (n_cells > 0) {
    const int CH = C * hcount(p);
    dim3 grid(n_cells, (CH + 63) / 64);
    launch_pdl(k_m2l_gather, grid, dim3(256), 0, st, cells, plan.m2l_row.get(), CH, (const double2*)part, L);
  }
  FMM_LAUNCH_CHECK();
}

// L[cell] for every target cell from the per-pair slots (the second half of launch_m2l)
void launch_m2l_gather(const Plan& plan, int p, int C, const double2* part, double2* L, cudaStream_t st) {
  const int CH = C * hcount(p);
  dim3 grid(plan.tgt.n_cells, (CH + 63) / 64);
  if (plan.tgt.n_cells > 0)
    launch_pdl(k_m2l_gather, grid, dim3(256), 0, st, (const int*)nullptr, plan.m2l_row.get(), CH, part, L);
  FMM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ M2M, octant-grouped
// Children at one level that sit in the same octant of their parents share
// R(d): one CTA per (level, octant, <= 8 children) applies it to 4 child
// vectors per pass (same scheme as k_m2l_grouped, with the M2M index map and
// the j <= n, |m-k| <= n-j mask); every child's contribution goes to its own
// slot and k_children_sum adds the children of each parent in octant order.
constexpr int M2M_WARPS = 8;  // warps splitting the input orders of one M2M item

template <int P, int CK>
__global__ void __launch_bounds__(M2M_WARPS * 32)
k_m2m_grouped(const int4* __restrict__ items, const int* __restrict__ gchild,
              const double2* __restrict__ table, int table_stride, const double2* __restrict__ M,
              int Ctot, int cbase, double2* __restrict__ cout) {
  constexpr int BJ = tr_bj(P);
  constexpr int H = (P + 1) * (P + 2) / 2;
  constexpr int S = (P + 1) * (P + 1);
  constexpr int NV = 4;
  constexpr int NP = NV / CK;
  extern __shared__ double2 sh[];
  double2* sT = sh;
  double2* sM = sh + S;  // [NV][S]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 it = items[blockIdx.x];
  {
    const double2* T = table + (size_t)it.x * table_stride;
    for (int i = threadIdx.x; i < S; i += blockDim.x) cp_async16(sT + i, T + i);
    cp_async_commit();
  }
  int oc = -1, r0 = 0;
  {
    int cum = 0;
    for (int kk = 0; kk <= P; ++kk) {
      const int nt = (P - kk + 1 + BJ - 1) / BJ;
      if (oc < 0 && lane < cum + nt) {
        oc = kk;
        r0 = kk + (lane - cum) * BJ;
      }
      cum += nt;
    }
  }
  const bool active = oc >= 0;
  for (int e0 = it.y; e0 < it.z; e0 += NP) {
    const int np = min(NP, it.z - e0);
    const int nv = np * CK;
    __syncthreads();
    for (int f = threadIdx.x; f < NV * S; f += blockDim.x) {
      const int v = f / S, g = f - v * S;
      double2 val = make_double2(0.0, 0.0);
      if (v < nv) {
        const int ch = gchild[e0 + v / CK], c = cbase + v % CK;
        const int n = (int)__fsqrt_rz((float)g);
        val = hget(M + ((size_t)ch * Ctot + c) * H, n, g - n * n - n);
      }
      sM[f] = val;
    }
    cp_async_wait_all();
    __syncthreads();
    double2 acc[NV][BJ];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int t = 0; t < BJ; ++t) acc[v][t] = make_double2(0.0, 0.0);
    if (active) {
      for (int ai = warp; ai < 2 * P + 1; ai += M2M_WARPS) {
        const int am = ai - P;
        const int b0 = am < 0 ? -am : am;
        const int col = oc - am;
        const int acol = col < 0 ? -col : col;
        auto tval = [&](int row) -> double2 {  // R_{row}^{col}, zero outside the triangle
          const int N = min(max(row, 0), P);
          const double2 v = sT[pidx(N, max(min(col, N), -N))];
          return row >= acol ? v : make_double2(0.0, 0.0);
        };
        double2 w[BJ];
#pragma unroll
        for (int t = 0; t < BJ; ++t) w[t] = tval(r0 + t - b0);
        int lead = r0 - b0 - 1;
        const double2* ip = sM + b0 * b0 + b0 + am;
        int istep = 2 * b0 + 2;
        auto step = [&](int q) {
          double2 mv[NV];
#pragma unroll
          for (int v = 0; v < NV; ++v) mv[v] = ip[v * S];
          const double2 nw = tval(lead);
          ip += istep;
          istep += 2;
          --lead;
#pragma unroll
          for (int t = 0; t < BJ; ++t)
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v][t] = cfma(mv[v], w[(t + BJ - q) % BJ], acc[v][t]);
          w[(BJ - 1 - q) % BJ] = nw;
        };
        int b = b0;
        for (; b + BJ - 1 <= P; b += BJ) {
#pragma unroll
          for (int q = 0; q < BJ; ++q) step(q);
        }
#pragma unroll
        for (int q = 0; q < BJ - 1; ++q)
          if (b + q <= P) step(q);
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      __syncthreads();
      double2* red = sM;
#pragma unroll
      for (int t = 0; t < BJ; ++t) red[(warp * 32 + lane) * BJ + t] = acc[v][t];
      __syncthreads();
      if (warp == 0 && active && v < nv) {
        const int ch = gchild[e0 + v / CK], c = cbase + v % CK;
#pragma unroll
        for (int t = 0; t < BJ; ++t) {
          const int r = r0 + t;
          if (r > P) continue;
          double2 sum = red[lane * BJ + t];
          for (int w2 = 1; w2 < M2M_WARPS; ++w2) sum = cadd(sum, red[(w2 * 32 + lane) * BJ + t]);
          cout[((size_t)ch * Ctot + c) * H + r * (r + 1) / 2 + oc] = sum;
        }
      }
    }
  }
}

// M[parent] = sum of its children's contributions in octant order
__global__ void k_children_sum(const int* __restrict__ parents, const int* __restrict__ first_child,
                               const int* __restrict__ n_child, int CH,
                               const double2* __restrict__ cout, double2* __restrict__ M) {
  const int par = parents[blockIdx.x];
  const int f = first_child[par], nc = n_child[par];
  for (int t = threadIdx.x; t < CH; t += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < nc; ++k) s = cadd(s, cout[(size_t)(f + k) * CH + t]);
    M[(size_t)par * CH + t] = s;
  }
}

template <int P, int CK>
size_t m2mg_smem() {
  constexpr int S = (P + 1) * (P + 1);
  const size_t red = (size_t)M2M_WARPS * 32 * tr_bj(P);
  return ((size_t)S + std::max((size_t)4 * S, red)) * sizeof(double2);
}

template <int P, int CK>
void m2mg_launch_one(const int4* items, int n, const int* gchild, const double2* rfull,
                     const double2* M, int C, int cb, double2* cout, cudaStream_t st) {
  static DeviceOnce attr;
  if (attr.first()) {
    FMM_CUDA(cudaFuncSetAttribute(k_m2m_grouped<P, CK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)m2mg_smem<P, CK>()));
    attr.mark();
  }
  k_m2m_grouped<P, CK><<<n, M2M_WARPS * 32, m2mg_smem<P, CK>(), st>>>(items, gchild, rfull, tab_size(P_MAX),
                                                                     M, C, cb, cout);
}

template <int P>
void m2mg_launch(const int4* items, int n, const int* gchild, const double2* rfull, const double2* M,
                 int C, double2* cout, cudaStream_t st) {
  if (n <= 0) return;
  for (int cb = 0; cb < C;) {
    const int rem = C - cb;
    if (rem >= 4) { m2mg_launch_one<P, 4>(items, n, gchild, rfull, M, C, cb, cout, st); cb += 4; }
    else if (rem >= 2) { m2mg_launch_one<P, 2>(items, n, gchild, rfull, M, C, cb, cout, st); cb += 2; }
    else { m2mg_launch_one<P, 1>(items, n, gchild, rfull, M, C, cb, cout, st); cb += 1; }
  }
  FMM_LAUNCH_CHECK();
}

void launch_m2m_grouped(const Plan& plan, int p, int C, const double2* rfull, double2* M,
                        double2* cout, cudaStream_t st) {
  const Tree& S = plan.src;
  const int CH = C * hcount(p);
  for (int l = (int)plan.m2m_level_off.size() - 2; l >= 0; --l) {
    const int np = plan.m2m_level_off[l + 1] - plan.m2m_level_off[l];
    if (np <= 0) continue;
    const int ia = plan.m2m_gitem_off[l], ib = plan.m2m_gitem_off[l + 1];
    const int4* items = plan.d_m2m_gitems.get() + ia;
    switch (p) {
#define MG_CASE(PP) case PP: m2mg_launch<PP>(items, ib - ia, plan.m2m_gchild.get(), rfull, M, C, cout, st); break;
      MG_CASE(0) MG_CASE(1) MG_CASE(2) MG_CASE(3) MG_CASE(4) MG_CASE(5) MG_CASE(6)
      MG_CASE(7) MG_CASE(8) MG_CASE(9) MG_CASE(10) MG_CASE(11) MG_CASE(12) MG_CASE(13)
      MG_CASE(14) MG_CASE(15) MG_CASE(16) MG_CASE(17) MG_CASE(18) MG_CASE(19) MG_CASE(20)
#undef MG_CASE
      default: throw ArgumentError("M2M: expansion order out of range");
    }
    k_children_sum<<<np, 128, 0, st>>>(plan.m2m_cells.get() + plan.m2m_level_off[l], S.first_child.get(),
                                       S.n_child.get(), CH, cout, M);
    FMM_LAUNCH_CHECK();
  }
}

void launch_children_sum(const Plan& plan, int l, int CH, const double2* cout, double2* M,
                         cudaStream_t st) {
  const int np = plan.m2m_level_off[l + 1] - plan.m2m_level_off[l];
  if (np <= 0) return;
  k_children_sum<<<np, 128, 0, st>>>(plan.m2m_cells.get() + plan.m2m_level_off[l],
                                     plan.src.first_child.get(), plan.src.n_child.get(), CH, cout, M);
  FMM_LAUNCH_CHECK();
}

void launch_m2m(const Tree& S, const std::vector<int>& level_off, const int* cells, int p, int C,
                const double2* rfull, double2* M, cudaStream_t st) {
  TrArgs a{};
  a.first_child = S.first_child.get();
  a.n_child = S.n_child.get();
  a.rtab = S.rtab.get();
  a.table = rfull;
  a.table_stride = tab_size(P_MAX);
  a.in = M;
  a.out = M;
  a.Ctot = C;
  for (int l = (int)level_off.size() - 2; l >= 0; --l) {
    a.cells = cells + level_off[l];
    tr_dispatch<T_M2M>(p, level_off[l + 1] - level_off[l], a, st);
  }
}

void launch_l2l(const Tree& T, const std::vector<int>& level_off, const int* cells, int p, int C,
                const double2* rfull, double2* L, cudaStream_t st, int l0, int l1) {
  TrArgs a{};
  a.parent = T.parent.get();
  a.rtab = T.rtab.get();
  a.table = rfull;
  a.table_stride = tab_size(P_MAX);
  a.in = L;
  a.out = L;
  a.Ctot = C;
  for (int l = std::max(l0, 1); l + 1 < (int)level_off.size() && l < l1; ++l) {
    a.cells = cells + level_off[l];
    tr_dispatch<T_L2L>(p, level_off[l + 1] - level_off[l], a, st);
  }
}

}  // namespace fmmbem
