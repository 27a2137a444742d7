// Octree + dual-traversal plan, resident in HBM.
//
// Replaces FmmPlan.__init__ (pkg/src/fmmbem/fmm.py:131-168), build_tree
// (octree.py:57-131), bounding_cube (octree.py:46-54) and dual_traversal
// (fmm.py:84-125).  Cells are numbered level by level and in Morton order
// inside a level (the reference numbers them depth-first); trees and pair
// sets are compared with the reference by content, never by index.
#pragma once

#include <cstdlib>

#include "common.cuh"

namespace fmmbem {

struct Tree {
  int64_t n_points = 0;
  int n_cells = 0;
  int n_levels = 0;  // levels present: 0 .. n_levels-1
  int n_leaves = 0;
  int max_leaf_count = 0;
  std::vector<int> level_start;  // host: cells of level l are [level_start[l], level_start[l+1])
  std::vector<double> level_half;  // host: half width per level (root_half * 0.5^l)

  // per cell (device)
  DevBuf<double> cx, cy, cz, half;
  DevBuf<int> level, parent, first_child, n_child, body_start, body_count;
  DevBuf<uint8_t> is_leaf;
  // leaves in body order (device) and per sorted body its leaf cell
  DevBuf<int> leaves, leaf_of_body;
  DevBuf<int> rtab;  // level * 8 + octant of each cell inside its parent (M2M/L2L table id)
  // sorted position -> original index, and sorted coordinates
  DevBuf<int> perm;
  DevBuf<double> px, py, pz;

  // host mirrors (small)
  std::vector<int> h_level, h_parent, h_first_child, h_n_child, h_body_start, h_body_count;
  std::vector<uint8_t> h_is_leaf;
  std::vector<int> h_leaves;
  std::vector<double> h_cx, h_cy, h_cz;
  const double* rec = nullptr;  // plan's reciprocal table (common.cuh)
};

constexpr int P2P_ITEM_SOURCES_DEFAULT = 896;  // sources per P2P work item (shared-memory tile)
// (FMMBEM_P2P_ITEM overrides it, for tuning)
inline int p2p_item_sources() {
  static const int v = std::getenv("FMMBEM_P2P_ITEM") ? std::atoi(std::getenv("FMMBEM_P2P_ITEM"))
                                                      : P2P_ITEM_SOURCES_DEFAULT;
  return v;
}

struct P2PItem {
  int tgt_leaf;   // target cell id
  int pair_begin; // range into p2p source-leaf list (CSR of the target leaf)
  int pair_end;
  int out_off;    // offset into the per-item partial buffer (in targets)
};

// Work lists of the shared-table rotation M2L (m2l_rot.cu, k_m2l_rot2) over one list of
// class-grouped items: CTA groups (direction table, first item, end item) and the items' pairs
// as (result slot, source cell, offset id, 0) records, 8 per item (slot -1: none)
struct RotGroups {
  DevBuf<int4> groups, vecs;
  int n_groups = 0;
  void build(const std::vector<int4>& items, const std::vector<int>& cpair, const std::vector<int>& pair_src,
             const std::vector<int>& pair_off, const std::vector<int>& dir_of_off, cudaStream_t s);
};

// grow-only device workspace of plan_evaluate / fmmbem_plan_evaluate (one per plan: repeated
// evaluations allocate nothing)
struct EvalWork {
  DevBuf<double> q, d, qs, ds, pot, grad;
  DevBuf<double2> M, L, part;
};

struct Plan {
  int device = 0;
  EvalWork eval;
  // sources per P2P work item: 0 = p2p_item_sources(); the operator sets 1 024 for large
  // double-layer systems (the persistent near-field kernel: cfg5 493.6 -> 500.3 mat-vecs/s)
  int p2p_item_src = 0;
  int item_sources() const { return p2p_item_src > 0 ? p2p_item_src : p2p_item_sources(); }
  int n_crit = 0;
  int max_depth = 20;
  double theta = 0.5;
  double root_c[3] = {0, 0, 0};
  double root_half = 0;
  Tree src, tgt;
  DevBuf<double> recip;  // make_recip_table() on device

  // M2L: CSR by target cell over (source cell, offset id)
  int n_m2l = 0;
  DevBuf<int> m2l_row;     // n_tgt_cells + 1
  DevBuf<int> m2l_src;     // n_m2l
  DevBuf<int> m2l_off;     // n_m2l, offset-table index
  std::vector<int> h_m2l_row, h_m2l_src;
  int n_offsets = 0;
  DevBuf<double> off_d;    // 3 * n_offsets, the (lattice-exact) translation vectors
  DevBuf<double2> igrid;   // n_offsets * (2 igrid_p + 1)^2, FULL flat storage n^2+n+m
  int igrid_p = -1;        // I tables hold orders up to 2 * igrid_p
  // rotation-based M2L (m2l_rot.cu): per offset the scaled Wigner matrices a^n, n <= rot_p,
  // and (|D|, theta, phi)
  // The a^n depend on the polar angle of D only: offsets with bitwise-equal
  // cos(theta) share one table (rot_dir maps offset -> table).
  DevBuf<double> rot, rot_geo;
  DevBuf<int> rot_dir;
  std::vector<int> h_rot_dir;
  int n_rot_dirs = 0;
  std::vector<double> h_off;  // 3 * n_offsets
  DevBuf<double> rot_aux;  // per offset e^{-ik phi} and N!/|D|^(N+1)
  DevBuf<double> rotf;  // the same operators as DMMA 8x4 row fragments (m2l_rot.cu)
  int rot_p = -1;
  bool use_rot = true;  // FMMBEM_DENSE_M2L=1 selects the dense contraction instead
  // M2L work items: (target cell, pair begin, pair end, item id), <= 16 pairs each
  std::vector<int4> m2l_items;
  DevBuf<int4> d_m2l_items;
  DevBuf<int> m2l_cell_items;  // n_tgt_cells + 1 offsets into m2l_items
  // offset-grouped M2L: pairs (CSR positions) sorted by offset, items of <= 8
  // pairs sharing one translation (off id, begin, end into m2l_gpair)
  std::vector<int4> m2l_gitems;
  DevBuf<int4> d_m2l_gitems;
  DevBuf<int> m2l_gpair;
  // rotation M2L: pairs grouped by CLASS (same polar-angle table and |D|: the offsets differ
  // only in the azimuth, applied per vector), items of <= 8 pairs; x = a member offset
  std::vector<int> h_m2l_off;  // offset id per CSR pair position
  std::vector<int4> m2l_citems;
  DevBuf<int4> d_m2l_citems;
  DevBuf<int> m2l_cpair;
  std::vector<int> h_m2l_cpair;
  // the same class-grouped items split by source cell: leaf sources (their multipoles exist as
  // soon as the leaf basis stream ends, so these run beside the M2M levels) and the rest
  std::vector<int4> m2l_ci_leaf, m2l_ci_rest;
  DevBuf<int4> d_m2l_ci_leaf, d_m2l_ci_rest;
  // CTA groups of the shared-table rotation M2L over each of the three item lists
  RotGroups m2l_rg, m2l_rg_leaf, m2l_rg_rest;
  DevBuf<int> m2l_cp_leaf, m2l_cp_rest;
  std::vector<int> m2l_tgt_cells;  // target cells with >= 1 M2L source
  DevBuf<int> d_m2l_tgt_cells;

  // P2P: CSR by target leaf (cell id) over source leaves
  int n_p2p = 0;
  DevBuf<int> p2p_row;     // n_tgt_cells + 1
  DevBuf<int> p2p_src;
  std::vector<int> h_p2p_row, h_p2p_src;
  std::vector<P2PItem> items;
  DevBuf<P2PItem> d_items;
  DevBuf<int> p2p_order;  // items by decreasing work (persistent P2P schedule)
  DevBuf<int> tleaf_item_begin;  // per target leaf index (body order) -> first item; n_leaves + 1
  int64_t part_len = 0;          // total targets over items
  int64_t p2p_interactions = 0;

  // pruned vertical passes: M2M only for parents whose multipole is needed by an
  // M2L (or an ancestor's), L2L only below cells that carry a local expansion
  // direct downward pass: per target leaf, the cells on its path to the root
  // (itself first) that receive M2L terms; the epilogue evaluates each one's
  // local expansion at the targets (L2L is exact, so this equals the L2L chain)
  DevBuf<int> epi_path_off;  // n_tgt_cells + 1 (empty for non-leaves)
  DevBuf<int> epi_path;
  int max_path = 0;          // longest such list
  std::vector<int> m2m_level_off, l2l_level_off;
  DevBuf<int> m2m_cells, l2l_cells;
  // octant-grouped M2M: items (rtab id, begin, end) into m2m_gchild, per parent level
  std::vector<int> m2m_gitem_off;
  DevBuf<int4> d_m2m_gitems;
  DevBuf<int> m2m_gchild;

  // rotation-based M2M (m2l_rot.cu): children grouped by (level, octant) in items of <= 8,
  // per parent level [m2m_ritem_off[l], m2m_ritem_off[l+1]); per rtab id (level * 8 + octant)
  // the rotation fragments of its direction and (e^{-ik phi}, |d|^l / l!)
  std::vector<int> m2m_ritem_off;
  DevBuf<int4> d_m2m_ritems;
  DevBuf<int> m2m_rchild;
  DevBuf<double> m2m_rotf, m2m_aux;
  DevBuf<int> m2m_dir;
  int m2m_rot_p = -1;  // (both trees' tables: M2M on the source tree, L2L on the target tree)
  // rotation-based L2L on the target tree: the cells of l2l_cells grouped by (level, octant),
  // items of <= 8, per level (top-down); with it the epilogue evaluates only each leaf's own
  // (complete) local expansion: epi_leaf_off / epi_leaf (the leaf, or nothing without far field)
  std::vector<int> l2l_ritem_off;
  DevBuf<int4> d_l2l_ritems;
  DevBuf<int> l2l_rchild;
  DevBuf<double> l2l_rotf, l2l_aux;
  DevBuf<int> l2l_dir;
  DevBuf<int> epi_leaf_off, epi_leaf;

  // M2M / L2L translation tables: R(d) for the 8 child octants of every level, up to igrid... P_MAX
  DevBuf<double2> rshift_src;  // [level][octant][(P_MAX+1)^2] full storage
  DevBuf<double2> rshift_tgt;
};

// builds both trees over a shared root cube, the traversal, and the work lists
void plan_build(Plan& plan, const double* src_xyz, int64_t ns, const double* tgt_xyz, int64_t nt,
                int n_crit, double theta, int max_depth, cudaStream_t s);
// (re)build the irregular-harmonic tables for M2L up to order 2p
void plan_ensure_igrid(Plan& plan, int p, cudaStream_t s);
void plan_ensure_rot(Plan& plan, int p, cudaStream_t s);
void plan_ensure_m2m_rot(Plan& plan, int p, cudaStream_t s);
// item indices by decreasing work (targets x sources), for the persistent P2P kernel
std::vector<int> p2p_schedule(const Tree& T, const Tree& S, const std::vector<P2PItem>& items,
                              const std::vector<int>& p2p_src);
// dense "every source leaf for every target leaf" item list (dense_apply)
void plan_dense_items(const Plan& plan, std::vector<P2PItem>& items, std::vector<int>& row,
                      std::vector<int>& src, std::vector<int>& item_begin, int64_t& part_len);
void plan_make_items(const Tree& tgt, const Tree& src, const std::vector<int>& row,
                     const std::vector<int>& srcl, int chunk, std::vector<P2PItem>& items,
                     std::vector<int>& item_begin, int64_t& part_len, int64_t& interactions);

}  // namespace fmmbem
