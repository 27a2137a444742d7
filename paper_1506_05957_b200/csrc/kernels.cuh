// Launch wrappers for the hot-path kernels (one translation unit each).
#pragma once

#include "plan.cuh"

namespace fmmbem {

// plain-pointer view of a Tree for kernel arguments
struct TreeDev {
  const double *px, *py, *pz;
  const double *cx, *cy, *cz, *half;
  const int *level, *parent, *first_child, *n_child, *body_start, *body_count, *perm;
  const uint8_t* is_leaf;
  int64_t n_points;
  const double* rec;
};

inline TreeDev tree_dev(const Tree& t) {
  return TreeDev{t.px.get(), t.py.get(), t.pz.get(), t.cx.get(), t.cy.get(), t.cz.get(),
                 t.half.get(), t.level.get(), t.parent.get(), t.first_child.get(),
                 t.n_child.get(), t.body_start.get(), t.body_count.get(), t.perm.get(),
                 t.is_leaf.get(), t.n_points, t.rec};
}

void upload_index_tables();

// far field
void launch_p2m(const TreeDev& S, const int* leaves, int n_leaves, int p, int C, const double* q,
                const double* d, double2* M, cudaStream_t st);
// M2M over the parents listed per level (cells[level_off[l] .. level_off[l+1]])
void launch_m2m(const Tree& S, const std::vector<int>& level_off, const int* cells, int p, int C,
                const double2* rfull, double2* M, cudaStream_t st);
// M2L into per-item partial blocks (part: n_items * C * hcount(p)) then reduced into L (all cells)
// (gitems, cells: optional restricted work lists for a shard; defaults = whole plan)
void launch_m2l(const Plan& plan, int p, int C, const double2* M, double2* L, double2* part,
                cudaStream_t st, const int4* gitems = nullptr, int n_gitems = -1,
                const int* cells = nullptr, int n_cells = -1, const int* gpair = nullptr,
                const int4* citems = nullptr, int n_citems = -1, const int* cpair = nullptr,
                const RotGroups* rg = nullptr);
void compute_igrid_full(const double* d_off, int n_off, int order, double2* out, cudaStream_t s);
void compute_rot_tables(const double* d_off, int n_off, int P, double* out, double* geo,
                        cudaStream_t s);
size_t rot_table_size(int P);
size_t rot_frag_size(int P);
inline size_t rot_aux_size(int P) { return (size_t)(4 * P + 4); }
void build_rot_aux(const double* geo, int n_off, int P, double* aux, cudaStream_t s);
void build_rot_frag(const double* rot, int n_off, int P, double* out, cudaStream_t s);
// rg (RotGroups over class-grouped items) and FMMBEM_M2L_SHARED=1: the shared-table kernel, one
// CTA per group with the direction's tables staged in shared memory by bulk async copies (TMA)
// and the multipoles prefetched by cp.async; otherwise the per-warp kernel that reads the tables
// from L2 (the default: measured 1-2 % faster, both are bound by shared/L1 operand bandwidth)
void launch_m2l_rot(const Plan& plan, const int4* gitems, const int* gpair, int n_items, int p,
                    int C, const double2* M, double2* pout, cudaStream_t st, bool cls,
                    const RotGroups* rg = nullptr);
constexpr int M2L_ROT_MIN_P = 3;  // rotation-based M2L from this order up
void launch_m2l_gather(const Plan& plan, int p, int C, const double2* part, double2* L, cudaStream_t st);
// M2M by rotation (point and shoot, DMMA): per-child contributions into cout, then the
// children of every parent summed in order (p >= M2L_ROT_MIN_P; plan_ensure_m2m_rot first)
void launch_m2m_rot(const Plan& plan, int p, int C, double2* M, double2* cout, cudaStream_t st);
// levels [l0, l1) of the target tree (default: all)
void launch_l2l_rot(const Plan& plan, int p, int C, double2* L, cudaStream_t st, int l0 = 0, int l1 = 1 << 30);
void launch_children_sum(const Plan& plan, int level, int CH, const double2* cout, double2* M,
                         cudaStream_t st);
// M2M through octant-grouped child translations (cout: per-cell child contributions)
void launch_m2m_grouped(const Plan& plan, int p, int C, const double2* rfull, double2* M,
                        double2* cout, cudaStream_t st);
// L2L into the cells listed per level whose parent has a nonzero local expansion
void launch_l2l(const Tree& T, const std::vector<int>& level_off, const int* cells, int p, int C,
                const double2* rfull, double2* L, cudaStream_t st, int l0 = 1, int l1 = 1 << 30);

// near field (P2P) kinds
enum class P2PKind : int { LAP_Q = 0, LAP_D = 1, STOKESLET = 2, STRESSLET = 3 };
inline int p2p_comps(P2PKind k) { return (k == P2PKind::LAP_Q || k == P2PKind::LAP_D) ? 1 : 3; }

// Writes per-item partial sums part[(item.out_off + local_target) * comps + comp].
// Source strengths (sorted source order): LAP_Q: w[ns]; LAP_D: w[ns*3] dipoles;
// STOKESLET: w[ns*3] forces; STRESSLET: w[ns*6] = (force, normal).
// CTA b takes item order[b] (largest work first), or item b when order is null.
// Per item list, for the persistent double-layer kernel: every item's source leaves as
// (start, count, tile offset) at their CSR position, and every item target's tile slot of
// its own centroid Gauss point (-1 if not in the item) at its partial-sum position.
struct LapdHdr {  // one P2P item in schedule (largest-first) order
  int pair_begin, nl, ns, t0, nt, out_off, nspec;
  // tile sections: n1 single points (own sources first), n2 clusters of 2 and n3 clusters of 3
  // points of one panel sharing the dipole term (ns = n1 + 2 n2 + 3 n3)
  int n1, n2, n3;
  double cx, cy, cz;  // target leaf centre
};
struct P2PAux {
  DevBuf<LapdHdr> hdr;
  int n_items = 0;
  // per item source leaf: (body start, singles offset | pair-cluster offset << 16, tile offset,
  // triple-cluster offset)
  DevBuf<int4> ltab;
  DevBuf<int> slot;  // per item target: its own source's tile slot (own sources first), or -1
  DevBuf<int> spec;  // per item: the own sources' positions among the item's singles, ascending
  // per sorted source: section (0 single, 1 pair, 2 triple) | position in its cluster << 2 |
  // rank inside its leaf's section << 4
  DevBuf<int> code;
  int max_leaves = 1, max_tgt = 1;
  bool ready = false;
  void build(const Tree& S, const Tree& T, const std::vector<P2PItem>& items,
             const std::vector<int>& p2p_src, const std::vector<int>& self_src_sorted, cudaStream_t st);
};
// aux (LAP_D) selects the persistent expanded-form double-layer kernel, which also needs a
// 2-uint schedule counter (zero before the first launch; self-resetting) and the sources as
// static records srec[3 i .. 3 i + 2] = (x, y), (z, w n_x), (w n_y, w n_z) in sorted order with
// the panel s_panel[i] whose density x[panel] scales the dipole; without them, or
// when the stages do not fit shared memory, the difference-form kernel runs.
void launch_p2p(P2PKind kind, const TreeDev& S, const TreeDev& T, const P2PItem* items,
                int n_items, const int* p2p_src, int max_sources, const double* w, double* part,
                cudaStream_t st, const int* order, const P2PAux* aux = nullptr,
                unsigned* sched = nullptr, const double2* srec = nullptr,
                const int* s_panel = nullptr, const double* x = nullptr);
bool p2p_lapd_usable(const P2PAux* aux, int max_sources);

// generic channel near field (FmmPlan.near_field): charges q[C][ns] and/or dipoles d[C][ns][3];
// accumulates into pot[C][nt] (+ grad[C][nt][3]) in ORIGINAL target order.
void launch_p2p_channels(const TreeDev& S, const TreeDev& T, const Plan& plan, int C,
                         const double* q, const double* d, bool want_grad, double* pot,
                         double* grad, cudaStream_t st);

// generic L2P (FmmPlan.far_field tail): pot[C][nt] (+ grad) in ORIGINAL target order
void launch_l2p_channels(const TreeDev& T, const int* leaves, int n_leaves, int p, int C,
                         bool want_grad, const double2* L, double* pot, double* grad,
                         cudaStream_t st);

}  // namespace fmmbem
