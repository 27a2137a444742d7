// Dual-tree traversal on device, plus the per-apply work lists.
//
// Reference: dual_traversal (fmm.py:84-125).  A (source, target) cell pair is
// accepted for M2L when d > 0 and (r_s + r_t) < theta * d with r = half width
// (CELL_RADIUS_FACTOR = 1, fmm.py:26); otherwise leaf-leaf pairs go to P2P and
// the source is split iff it is internal and (the target is a leaf or
// hw_s >= hw_t) (fmm.py:117).  The reference walks a stack; here the frontier
// is expanded level-synchronously on the GPU, which yields the same pair sets.
// Pairs are then sorted by (target, source) so every later accumulation has
// a fixed order (bitwise-reproducible mat-vecs).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <tuple>

#include "kernels.cuh"

namespace fmmbem {

void build_trees(Plan& plan, const double* src_xyz, int64_t ns, const double* tgt_xyz, int64_t nt,
                 cudaStream_t s);

namespace {

struct TreeView {
  const double *cx, *cy, *cz, *half;
  const uint8_t* is_leaf;
  const int *first_child, *n_child;
};

TreeView view(const Tree& t) {
  return TreeView{t.cx.get(), t.cy.get(), t.cz.get(), t.half.get(), t.is_leaf.get(),
                  t.first_child.get(), t.n_child.get()};
}

__global__ void k_traverse(const int2* front, int nf, TreeView S, TreeView T, double theta,
                           int2* next, int* n_next, int2* m2l, int* n_m2l, int2* p2p, int* n_p2p) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const int s = front[i].x, t = front[i].y;
  const double dx = __dadd_rn(S.cx[s], -T.cx[t]);
  const double dy = __dadd_rn(S.cy[s], -T.cy[t]);
  const double dz = __dadd_rn(S.cz[s], -T.cz[t]);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double d = sqrt(d2);
  const double rs = S.half[s], rt = T.half[t];
  if (d > 0.0 && __dadd_rn(rs, rt) < __dmul_rn(theta, d)) {
    int k = atomicAdd(n_m2l, 1);
    m2l[k] = make_int2(s, t);
    return;
  }
  const bool sl = S.is_leaf[s], tl = T.is_leaf[t];
  if (sl && tl) {
    int k = atomicAdd(n_p2p, 1);
    p2p[k] = make_int2(s, t);
    return;
  }
  const bool split_src = !sl && (tl || rs >= rt);
  if (split_src) {
    const int f = S.first_child[s], nc = S.n_child[s];
    int k = atomicAdd(n_next, nc);
    for (int c = 0; c < nc; ++c) next[k + c] = make_int2(f + c, t);
  } else {
    const int f = T.first_child[t], nc = T.n_child[t];
    int k = atomicAdd(n_next, nc);
    for (int c = 0; c < nc; ++c) next[k + c] = make_int2(s, f + c);
  }
}

void sort_pairs_tgt_major(std::vector<int2>& v) {
  std::sort(v.begin(), v.end(), [](const int2& a, const int2& b) {
    return a.y != b.y ? a.y < b.y : a.x < b.x;
  });
}

void traverse(Plan& plan, std::vector<int2>& m2l, std::vector<int2>& p2p, cudaStream_t s) {
  const int B = 256;
  TreeView S = view(plan.src), T = view(plan.tgt);
  std::vector<int2> front_h(1, make_int2(0, 0));
  DevBuf<int2> front, next, dm2l, dp2p;
  DevBuf<int> counters(3);
  front.upload(front_h, s);
  int nf = 1;
  while (nf > 0) {
    next.ensure((size_t)nf * 8);
    dm2l.ensure(nf);
    dp2p.ensure(nf);
    counters.zero(s);
    k_traverse<<<grid_for(nf, B), B, 0, s>>>(front.get(), nf, S, T, plan.theta, next.get(),
                                             counters.get(), dm2l.get(), counters.get() + 1,
                                             dp2p.get(), counters.get() + 2);
    FMM_LAUNCH_CHECK();
    int c[3];
    FMM_CUDA(cudaMemcpyAsync(c, counters.get(), sizeof(c), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    if (c[1]) {
      size_t o = m2l.size();
      m2l.resize(o + c[1]);
      FMM_CUDA(cudaMemcpy(m2l.data() + o, dm2l.get(), c[1] * sizeof(int2), cudaMemcpyDeviceToHost));
    }
    if (c[2]) {
      size_t o = p2p.size();
      p2p.resize(o + c[2]);
      FMM_CUDA(cudaMemcpy(p2p.data() + o, dp2p.get(), c[2] * sizeof(int2), cudaMemcpyDeviceToHost));
    }
    std::swap(front, next);
    nf = c[0];
  }
  sort_pairs_tgt_major(m2l);
  sort_pairs_tgt_major(p2p);
}

// R_n^m(d) in FULL storage for the 8 child offsets (+-h, +-h, +-h) of every
// level (the M2M / L2L operators; fmm.py:268-290 uses the first cell's offset
// of each octant group, here the exact lattice offset)
__global__ void k_rshift(const double* child_half, int n_levels, double2* out,
                         const double* rec) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_levels * 8) return;
  const int l = i / 8, o = i % 8;
  const double h = child_half[l];
  double2* dst = out + (size_t)i * tab_size(P_MAX);
  double2 tmp[hcount(P_MAX)];
  regular_half((o & 1) ? h : -h, (o & 2) ? h : -h, (o & 4) ? h : -h, P_MAX, tmp, rec);
  for (int n = 0; n <= P_MAX; ++n)
    for (int m = -n; m <= n; ++m) dst[pidx(n, m)] = hget(tmp, n, m);
}

void build_rshift(const Tree& t, DevBuf<double2>& out, cudaStream_t s) {
  // entry l holds offsets of level-l cells from their parent: half width of level l
  std::vector<double> ch(std::max(t.n_levels, 1));
  for (int l = 0; l < t.n_levels; ++l) ch[l] = t.level_half[l];
  DevBuf<double> d;
  d.upload(ch, s);
  out.resize((size_t)ch.size() * 8 * tab_size(P_MAX));
  k_rshift<<<grid_for(ch.size() * 8, 64), 64, 0, s>>>(d.get(), (int)ch.size(), out.get(), t.rec);
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

void plan_make_items(const Tree& tgt, const Tree& src, const std::vector<int>& row,
                     const std::vector<int>& srcl, int chunk, std::vector<P2PItem>& items,
                     std::vector<int>& item_begin, int64_t& part_len, int64_t& interactions) {
  items.clear();
  item_begin.assign(tgt.n_leaves + 1, 0);
  part_len = 0;
  interactions = 0;
  for (int li = 0; li < tgt.n_leaves; ++li) {
    const int t = tgt.h_leaves[li];
    const int nt = tgt.h_body_count[t];
    item_begin[li] = (int)items.size();
    int b = row[t];
    const int e = row[t + 1];
    while (b < e) {
      int acc = 0, k = b;
      while (k < e && (acc == 0 || acc + src.h_body_count[srcl[k]] <= chunk)) {
        acc += src.h_body_count[srcl[k]];
        ++k;
      }
      items.push_back(P2PItem{t, b, k, (int)part_len});
      part_len += nt;
      interactions += (int64_t)acc * nt;
      b = k;
    }
  }
  item_begin[tgt.n_leaves] = (int)items.size();
}

void plan_dense_items(const Plan& plan, std::vector<P2PItem>& items, std::vector<int>& row,
                      std::vector<int>& srcl, std::vector<int>& item_begin, int64_t& part_len) {
  const Tree& T = plan.tgt;
  const Tree& S = plan.src;
  row.assign(T.n_cells + 1, 0);
  srcl.clear();
  for (int c = 0; c < T.n_cells; ++c) {
    row[c] = (int)srcl.size();
    if (T.h_is_leaf[c])
      for (int sl : S.h_leaves) srcl.push_back(sl);
  }
  row[T.n_cells] = (int)srcl.size();
  int64_t inter = 0;
  plan_make_items(T, S, row, srcl, 2048, items, item_begin, part_len, inter);
}

void plan_ensure_igrid(Plan& plan, int p, cudaStream_t s) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p out of range [0, 20]");
  if (plan.igrid_p >= p) return;
  const int order = 2 * p;
  plan.igrid.resize((size_t)std::max(plan.n_offsets, 1) * tab_size(order));
  compute_igrid_full(plan.off_d.get(), plan.n_offsets, order, plan.igrid.get(), s);
  FMM_CUDA(cudaStreamSynchronize(s));
  plan.igrid_p = p;
}

std::vector<int> p2p_schedule(const Tree& T, const Tree& S, const std::vector<P2PItem>& items,
                              const std::vector<int>& p2p_src) {
  std::vector<int64_t> cost(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    int64_t ns = 0;
    for (int k = items[i].pair_begin; k < items[i].pair_end; ++k) ns += S.h_body_count[p2p_src[k]];
    cost[i] = ns * T.h_body_count[items[i].tgt_leaf];
  }
  std::vector<int> ord(items.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  return ord;
}

void plan_ensure_rot(Plan& plan, int p, cudaStream_t s) {
  FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p out of range [0, 20]");
  if (plan.rot_p >= p) return;
  // one table per distinct polar angle (the offsets are lattice-exact, so equal
  // directions give bitwise-equal z / |D|)
  std::map<double, int> dirs;
  std::vector<int> dir(plan.n_offsets);
  std::vector<double> rep;
  for (int u = 0; u < plan.n_offsets; ++u) {
    const double x = plan.h_off[3 * u], y = plan.h_off[3 * u + 1], z = plan.h_off[3 * u + 2];
    const double key = z / std::sqrt(x * x + y * y + z * z);
    auto it = dirs.find(key);
    if (it == dirs.end()) {
      it = dirs.emplace(key, (int)dirs.size()).first;
      rep.insert(rep.end(), {x, y, z});
    }
    dir[u] = it->second;
  }
  plan.n_rot_dirs = (int)dirs.size();
  plan.rot_dir.upload(dir.empty() ? std::vector<int>(1, 0) : dir, s);
  plan.h_rot_dir = dir;
  DevBuf<double> d_rep, geo_rep, one;
  d_rep.upload(rep.empty() ? std::vector<double>(3, 1.0) : rep, s);
  const int nd = std::max(plan.n_rot_dirs, 1);
  plan.rot.resize((size_t)nd * rot_table_size(p));
  geo_rep.resize((size_t)nd * 3);
  compute_rot_tables(d_rep.get(), plan.n_rot_dirs, p, plan.rot.get(), geo_rep.get(), s);
  // (|D|, theta, phi) of every offset (order-0 tables are a by-product)
  plan.rot_geo.resize((size_t)std::max(plan.n_offsets, 1) * 3);
  one.resize((size_t)std::max(plan.n_offsets, 1));
  compute_rot_tables(plan.off_d.get(), plan.n_offsets, 0, one.get(), plan.rot_geo.get(), s);
  if (plan.m2l_citems.empty() && plan.n_m2l > 0) {
    // classes: (polar-angle table, |D| as the device computed it) -- the members differ only in
    // the azimuth and share bitwise the same Hankel factors N!/|D|^(N+1)
    const std::vector<double> geo = plan.rot_geo.download(s);
    std::map<std::pair<int, double>, int> cls;
    std::vector<int> cls_of(plan.n_offsets);
    for (int u = 0; u < plan.n_offsets; ++u)
      cls_of[u] = cls.emplace(std::make_pair(dir[u], geo[3 * u]), (int)cls.size()).first->second;
    std::vector<int> gp(plan.n_m2l);
    for (int k = 0; k < plan.n_m2l; ++k) gp[k] = k;
    std::stable_sort(gp.begin(), gp.end(), [&](int a, int b) {
      // by direction table first: the shared-table kernel stages one table per CTA group
      const int oa = plan.h_m2l_off[a], ob = plan.h_m2l_off[b];
      if (dir[oa] != dir[ob]) return dir[oa] < dir[ob];
      const int ca = cls_of[oa], cb = cls_of[ob];
      return ca != cb ? ca < cb : oa < ob;
    });
    for (size_t i = 0; i < gp.size();) {
      size_t j = i;
      const int c0 = cls_of[plan.h_m2l_off[gp[i]]];
      while (j < gp.size() && cls_of[plan.h_m2l_off[gp[j]]] == c0) ++j;
      const int len = (int)(j - i), nch = (len + 7) / 8;
      for (int q = 0; q < nch; ++q) {
        const int lo = (int)i + (int)((int64_t)len * q / nch), hi = (int)i + (int)((int64_t)len * (q + 1) / nch);
        plan.m2l_citems.push_back(make_int4(plan.h_m2l_off[gp[lo]], lo, hi, 0));
      }
      i = j;
    }
    plan.h_m2l_cpair = gp;
    plan.d_m2l_citems.upload(plan.m2l_citems, s);
    plan.m2l_cpair.upload(gp, s);
    std::vector<int> cpl_all, cpr_all;
    {
      std::vector<int>&cpl = cpl_all, &cpr = cpr_all;
      plan.m2l_ci_leaf.clear();
      plan.m2l_ci_rest.clear();
      auto cut = [&](std::vector<int>& cp, std::vector<int4>& items, size_t start) {
        const int len = (int)(cp.size() - start), nch = (len + 7) / 8;
        for (int q = 0; q < nch; ++q) {
          const int lo = (int)start + (int)((int64_t)len * q / nch);
          const int hi = (int)start + (int)((int64_t)len * (q + 1) / nch);
          items.push_back(make_int4(plan.h_m2l_off[cp[lo]], lo, hi, 0));
        }
      };
      for (size_t i = 0; i < gp.size();) {
        size_t j = i;
        const int c0 = cls_of[plan.h_m2l_off[gp[i]]];
        while (j < gp.size() && cls_of[plan.h_m2l_off[gp[j]]] == c0) ++j;
        const size_t sl = cpl.size(), sr = cpr.size();
        for (size_t k = i; k < j; ++k)
          (plan.src.h_n_child[plan.h_m2l_src[gp[k]]] == 0 ? cpl : cpr).push_back(gp[k]);
        cut(cpl, plan.m2l_ci_leaf, sl);
        cut(cpr, plan.m2l_ci_rest, sr);
        i = j;
      }
      plan.d_m2l_ci_leaf.upload(plan.m2l_ci_leaf.empty() ? std::vector<int4>(1) : plan.m2l_ci_leaf, s);
      plan.d_m2l_ci_rest.upload(plan.m2l_ci_rest.empty() ? std::vector<int4>(1) : plan.m2l_ci_rest, s);
      plan.m2l_cp_leaf.upload(cpl.empty() ? std::vector<int>(1, 0) : cpl, s);
      plan.m2l_cp_rest.upload(cpr.empty() ? std::vector<int>(1, 0) : cpr, s);
    }
    plan.m2l_rg.build(plan.m2l_citems, gp, plan.h_m2l_src, plan.h_m2l_off, dir, s);
    plan.m2l_rg_leaf.build(plan.m2l_ci_leaf, cpl_all, plan.h_m2l_src, plan.h_m2l_off, dir, s);
    plan.m2l_rg_rest.build(plan.m2l_ci_rest, cpr_all, plan.h_m2l_src, plan.h_m2l_off, dir, s);
  }

  plan.rotf.resize((size_t)nd * rot_frag_size(p));
  build_rot_frag(plan.rot.get(), plan.n_rot_dirs, p, plan.rotf.get(), s);
  plan.rot_aux.resize((size_t)std::max(plan.n_offsets, 1) * rot_aux_size(p));
  build_rot_aux(plan.rot_geo.get(), plan.n_offsets, p, plan.rot_aux.get(), s);
  FMM_CUDA(cudaStreamSynchronize(s));
  plan.rot_p = p;
}

void plan_build(Plan& plan, const double* src_xyz, int64_t ns, const double* tgt_xyz, int64_t nt,
                int n_crit, double theta, int max_depth, cudaStream_t s) {
  FMM_REQUIRE(ns > 0 && nt > 0, "points must be nonempty (N, 3) arrays");
  FMM_REQUIRE(ns < (1ll << 31) && nt < (1ll << 31), "too many points");
  FMM_REQUIRE(n_crit >= 1, "n_crit must be >= 1");
  FMM_REQUIRE(theta > 0.0 && theta < 1.0, "theta must be in (0, 1)");
  FMM_REQUIRE(max_depth >= 1 && max_depth <= MAX_DEPTH_LIMIT, "max_depth must be in [1, 21]");
  plan.n_crit = n_crit;
  plan.theta = theta;
  plan.use_rot = std::getenv("FMMBEM_DENSE_M2L") == nullptr;
  plan.max_depth = max_depth;
  plan.recip.upload(make_recip_table(), s);
  build_trees(plan, src_xyz, ns, tgt_xyz, nt, s);
  plan.src.rec = plan.recip.get();
  plan.tgt.rec = plan.recip.get();

  std::vector<int2> m2l, p2p;
  traverse(plan, m2l, p2p, s);
  const Tree& S = plan.src;
  const Tree& T = plan.tgt;

  // M2L CSR by target cell and the distinct-offset table.  Offsets between
  // cell centres are exact multiples of the smaller half width (centres sit
  // at odd multiples of their half width from the root corner), so the key
  // (level_s, level_t, round(D / h_min)) identifies the translation; the
  // reference groups the same pairs by D rounded to half * 2^-(max_depth+2)
  // (fmm.py:144-159), which lands on the same lattice vectors.
  plan.n_m2l = (int)m2l.size();
  plan.h_m2l_row.assign(T.n_cells + 1, 0);
  plan.h_m2l_src.resize(m2l.size());
  std::vector<int> offid(m2l.size());
  std::map<std::tuple<int, int, long long, long long, long long>, int> offmap;
  std::vector<double> offd;
  for (size_t k = 0; k < m2l.size(); ++k) {
    const int sc = m2l[k].x, tc = m2l[k].y;
    plan.h_m2l_row[tc + 1]++;
    plan.h_m2l_src[k] = sc;
    const int ls = S.h_level[sc], lt = T.h_level[tc];
    // both trees share the root cube, so the finer cell's half width is exact
    const double hmin = std::ldexp(plan.root_half, -std::max(ls, lt));
    const double D[3] = {T.h_cx[tc] - S.h_cx[sc], T.h_cy[tc] - S.h_cy[sc], T.h_cz[tc] - S.h_cz[sc]};
    long long q[3];
    for (int d = 0; d < 3; ++d) q[d] = llround(D[d] / hmin);
    auto key = std::make_tuple(ls, lt, q[0], q[1], q[2]);
    auto it = offmap.find(key);
    if (it == offmap.end()) {
      it = offmap.emplace(key, (int)(offd.size() / 3)).first;
      for (int d = 0; d < 3; ++d) offd.push_back((double)q[d] * hmin);
    }
    offid[k] = it->second;
  }
  for (int c = 0; c < T.n_cells; ++c) plan.h_m2l_row[c + 1] += plan.h_m2l_row[c];
  plan.n_offsets = (int)(offd.size() / 3);
  plan.m2l_row.upload(plan.h_m2l_row, s);
  plan.m2l_src.upload(plan.h_m2l_src, s);
  plan.m2l_off.upload(offid, s);
  plan.h_m2l_off = offid;
  plan.m2l_citems.clear();
  plan.off_d.upload(offd, s);
  plan.h_off = offd;
  plan.m2l_tgt_cells.clear();
  for (int c = 0; c < T.n_cells; ++c)
    if (plan.h_m2l_row[c + 1] > plan.h_m2l_row[c]) plan.m2l_tgt_cells.push_back(c);
  plan.d_m2l_tgt_cells.upload(plan.m2l_tgt_cells, s);
  plan.igrid_p = -1;
  // M2L items: each target cell's list cut into near-equal slices of <= 16 pairs
  plan.m2l_items.clear();
  std::vector<int> cell_items(T.n_cells + 1, 0);
  for (int c = 0; c < T.n_cells; ++c) {
    cell_items[c] = (int)plan.m2l_items.size();
    const int b = plan.h_m2l_row[c], e = plan.h_m2l_row[c + 1], len = e - b;
    if (!len) continue;
    const int nch = (len + 15) / 16;
    for (int q = 0; q < nch; ++q) {
      const int lo = b + (int)((int64_t)len * q / nch), hi = b + (int)((int64_t)len * (q + 1) / nch);
      plan.m2l_items.push_back(make_int4(c, lo, hi, (int)plan.m2l_items.size()));
    }
  }
  cell_items[T.n_cells] = (int)plan.m2l_items.size();
  plan.d_m2l_items.upload(plan.m2l_items, s);
  plan.m2l_cell_items.upload(cell_items, s);
  {
    // offset-grouped work: pairs sharing a translation share its operator grid
    std::vector<int> gp(m2l.size());
    for (size_t k = 0; k < gp.size(); ++k) gp[k] = (int)k;
    std::stable_sort(gp.begin(), gp.end(), [&](int a, int b) { return offid[a] < offid[b]; });
    plan.m2l_gitems.clear();
    for (size_t i = 0; i < gp.size();) {
      size_t j = i;
      while (j < gp.size() && offid[gp[j]] == offid[gp[i]]) ++j;
      const int len = (int)(j - i), nch = (len + 7) / 8;
      for (int q = 0; q < nch; ++q) {
        const int lo = (int)i + (int)((int64_t)len * q / nch), hi = (int)i + (int)((int64_t)len * (q + 1) / nch);
        plan.m2l_gitems.push_back(make_int4(offid[gp[i]], lo, hi, 0));
      }
      i = j;
    }
    plan.d_m2l_gitems.upload(plan.m2l_gitems.empty() ? std::vector<int4>(1) : plan.m2l_gitems, s);
    plan.m2l_gpair.upload(gp.empty() ? std::vector<int>(1, 0) : gp, s);
  }

  // P2P CSR by target leaf and the balanced work items
  plan.n_p2p = (int)p2p.size();
  plan.h_p2p_row.assign(T.n_cells + 1, 0);
  plan.h_p2p_src.resize(p2p.size());
  for (size_t k = 0; k < p2p.size(); ++k) {
    plan.h_p2p_row[p2p[k].y + 1]++;
    plan.h_p2p_src[k] = p2p[k].x;
  }
  for (int c = 0; c < T.n_cells; ++c) plan.h_p2p_row[c + 1] += plan.h_p2p_row[c];
  plan.p2p_row.upload(plan.h_p2p_row, s);
  plan.p2p_src.upload(plan.h_p2p_src, s);
  std::vector<int> item_begin;
  plan_make_items(T, S, plan.h_p2p_row, plan.h_p2p_src, plan.item_sources(), plan.items, item_begin,
                  plan.part_len, plan.p2p_interactions);
  plan.d_items.upload(plan.items, s);
  {
    const std::vector<int> ord = p2p_schedule(T, S, plan.items, plan.h_p2p_src);
    plan.p2p_order.upload(ord.empty() ? std::vector<int>(1, 0) : ord, s);
  }
  plan.tleaf_item_begin.upload(item_begin, s);

  // needed(c): c is an M2L source or its parent's multipole is needed
  {
    std::vector<uint8_t> need(S.n_cells, 0), nz(T.n_cells, 0);
    for (int sc : plan.h_m2l_src) need[sc] = 1;
    for (int c = 1; c < S.n_cells; ++c)  // level-major numbering: parents come first
      if (need[S.h_parent[c]]) need[c] = 1;
    std::vector<int> cells;
    plan.m2m_level_off.assign(1, 0);
    for (int l = 0; l < S.n_levels; ++l) {
      for (int c = S.level_start[l]; c < S.level_start[l + 1]; ++c)
        if (!S.h_is_leaf[c] && need[c]) cells.push_back(c);
      plan.m2m_level_off.push_back((int)cells.size());
    }
    plan.m2m_cells.upload(cells.empty() ? std::vector<int>(1, 0) : cells, s);
    // children of those parents grouped by (level, octant) -> shared R(d)
    std::vector<int4> gitems, ritems;
    std::vector<int> gchild, rchild;
    plan.m2m_gitem_off.assign(1, 0);
    plan.m2m_ritem_off.assign(1, 0);
    for (int l = 0; l < S.n_levels; ++l) {
      std::vector<std::vector<int>> by_oct(8);
      for (int k = plan.m2m_level_off[l]; k < plan.m2m_level_off[l + 1]; ++k) {
        const int par = cells[k];
        for (int ch = S.h_first_child[par]; ch < S.h_first_child[par] + S.h_n_child[par]; ++ch) {
          const int o = (S.h_cx[ch] > S.h_cx[par] ? 1 : 0) | (S.h_cy[ch] > S.h_cy[par] ? 2 : 0) |
                        (S.h_cz[ch] > S.h_cz[par] ? 4 : 0);
          by_oct[o].push_back(ch);
        }
      }
      for (int o = 0; o < 8; ++o) {
        const auto& v = by_oct[o];
        for (size_t i = 0; i < v.size(); i += 4) {  // one 4-vector pass per CTA
          const int b = (int)gchild.size();
          for (size_t j = i; j < std::min(v.size(), i + 4); ++j) gchild.push_back(v[j]);
          gitems.push_back(make_int4((l + 1) * 8 + o, b, (int)gchild.size(), 0));
        }
        for (size_t i = 0; i < v.size(); i += 8) {  // rotation M2M: 8 vectors per warp
          const int b = (int)rchild.size();
          for (size_t j = i; j < std::min(v.size(), i + 8); ++j) rchild.push_back(v[j]);
          ritems.push_back(make_int4((l + 1) * 8 + o, b, (int)rchild.size(), 0));
        }
      }
      plan.m2m_gitem_off.push_back((int)gitems.size());
      plan.m2m_ritem_off.push_back((int)ritems.size());
    }
    plan.d_m2m_ritems.upload(ritems.empty() ? std::vector<int4>(1) : ritems, s);
    plan.m2m_rchild.upload(rchild.empty() ? std::vector<int>(1, 0) : rchild, s);
    plan.d_m2m_gitems.upload(gitems.empty() ? std::vector<int4>(1) : gitems, s);
    plan.m2m_gchild.upload(gchild.empty() ? std::vector<int>(1, 0) : gchild, s);
    for (int c = 0; c < T.n_cells; ++c)
      if (plan.h_m2l_row[c + 1] > plan.h_m2l_row[c]) nz[c] = 1;
    for (int c = 1; c < T.n_cells; ++c)
      if (nz[T.h_parent[c]]) nz[c] = 1;
    cells.clear();
    plan.l2l_level_off.assign(1, 0);
    for (int l = 0; l < T.n_levels; ++l) {
      if (l > 0)
        for (int c = T.level_start[l]; c < T.level_start[l + 1]; ++c)
          if (nz[T.h_parent[c]]) cells.push_back(c);
      plan.l2l_level_off.push_back((int)cells.size());
    }
    plan.l2l_cells.upload(cells.empty() ? std::vector<int>(1, 0) : cells, s);
    {
      std::vector<int4> ritems;
      std::vector<int> rchild;
      plan.l2l_ritem_off.assign(1, 0);
      for (int l = 0; l < T.n_levels; ++l) {
        std::vector<std::vector<int>> by_oct(8);
        for (int k = plan.l2l_level_off[l]; k < plan.l2l_level_off[l + 1]; ++k) {
          const int c = cells[k], par = T.h_parent[c];
          const int o = (T.h_cx[c] > T.h_cx[par] ? 1 : 0) | (T.h_cy[c] > T.h_cy[par] ? 2 : 0) |
                        (T.h_cz[c] > T.h_cz[par] ? 4 : 0);
          by_oct[o].push_back(c);
        }
        for (int o = 0; o < 8; ++o)
          for (size_t i = 0; i < by_oct[o].size(); i += 8) {
            const int b = (int)rchild.size();
            for (size_t j = i; j < std::min(by_oct[o].size(), i + 8); ++j) rchild.push_back(by_oct[o][j]);
            ritems.push_back(make_int4(l * 8 + o, b, (int)rchild.size(), 0));
          }
        plan.l2l_ritem_off.push_back((int)ritems.size());
      }
      plan.d_l2l_ritems.upload(ritems.empty() ? std::vector<int4>(1) : ritems, s);
      plan.l2l_rchild.upload(rchild.empty() ? std::vector<int>(1, 0) : rchild, s);
      std::vector<int> loff(T.n_cells + 1, 0), leaf;
      for (int c = 0; c < T.n_cells; ++c) {
        loff[c] = (int)leaf.size();
        if (T.h_n_child[c] == 0 && nz[c]) leaf.push_back(c);
      }
      loff[T.n_cells] = (int)leaf.size();
      plan.epi_leaf_off.upload(loff, s);
      plan.epi_leaf.upload(leaf.empty() ? std::vector<int>(1, 0) : leaf, s);
    }
    std::vector<int> poff(T.n_cells + 1, 0), path;
    for (int c = 0; c < T.n_cells; ++c) {
      poff[c] = (int)path.size();
      if (T.h_n_child[c] != 0) continue;
      for (int a = c; a >= 0; a = T.h_parent[a])
        if (plan.h_m2l_row[a + 1] > plan.h_m2l_row[a]) path.push_back(a);
    }
    poff[T.n_cells] = (int)path.size();
    plan.max_path = 0;
    for (int c = 0; c < T.n_cells; ++c) plan.max_path = std::max(plan.max_path, poff[c + 1] - poff[c]);
    plan.epi_path_off.upload(poff, s);
    plan.epi_path.upload(path.empty() ? std::vector<int>(1, 0) : path, s);
  }
  for (Tree* tr : {&plan.src, &plan.tgt}) {
    std::vector<int> rt(tr->n_cells, 0);
    for (int c = 1; c < tr->n_cells; ++c) {
      const int pa = tr->h_parent[c];
      const int o = (tr->h_cx[c] > tr->h_cx[pa] ? 1 : 0) | (tr->h_cy[c] > tr->h_cy[pa] ? 2 : 0) |
                    (tr->h_cz[c] > tr->h_cz[pa] ? 4 : 0);
      rt[c] = tr->h_level[c] * 8 + o;
    }
    tr->rtab.upload(rt, s);
  }
  build_rshift(S, plan.rshift_src, s);
  build_rshift(T, plan.rshift_tgt, s);
  FMM_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fmmbem
