// BemOperator on device: plan + geometry + corrections + apply/GMRES.
#pragma once

#include <map>
#include <memory>

#include "kernels.cuh"

namespace fmmbem {

enum Formulation : int { LAPLACE_FIRST = 0, LAPLACE_SECOND = 1, STOKES = 2 };
// layer kernels, numbered like P2PKind
enum LayerKind : int { K_LAP_SINGLE = 0, K_LAP_DOUBLE = 1, K_STOKESLET = 2, K_STRESSLET = 3 };

struct Correction {
  int kind = -1;
  int block = 1;          // 1 (scalar) or 9 (3x3 block, row-major)
  DevBuf<double> vals;    // near_nnz * block
};

// stage timers captured with the apply (CUDA events on the launching streams)
enum Stage : int { ST_P2P = 0, ST_UP = 1, ST_M2L = 2, ST_DOWN = 3, ST_EPI = 4, ST_TOTAL = 5, N_STAGES = 6 };

// One rank's share of a partitioned apply (shard.cu): target leaves
// [tleaf_a, tleaf_b) and source leaves [sleaf_a, sleaf_b) in body order.
// host-staged collectives (fmmbem_op_shard_host): the caller's transport on host buffers
typedef int (*HostAllgather)(const double* send, double* recv, int64_t count, void* user);
typedef int (*HostAllreduce)(double* buf, int64_t count, void* user);

struct ShardWork {
  bool active = false;
  bool virtual_mode = false;  // no collectives: full upward pass, own y entries only (tests)
  // transport of a real shard: NCCL (device buffers, capturable in the per-p graphs) or the
  // caller's host callbacks (device <-> pinned host staging around each collective)
  enum Transport : int { T_VIRTUAL = 0, T_NCCL = 1, T_HOST = 2 };
  int transport = T_VIRTUAL;
  HostAllgather host_ag = nullptr;
  HostAllreduce host_ar = nullptr;
  void* host_user = nullptr;
  double* hstage = nullptr;  // pinned host staging of the host transport
  size_t hstage_cap = 0;
  // partitioned Krylov vectors (sharded GMRES): the apply consumes the gathered x_in and
  // leaves its own rows in ysend (sorted target order) instead of all-gathering y
  bool local_vectors = false;
  int rank = 0, world = 1;
  int tleaf_a = 0, tleaf_b = 0, tbody_a = 0, tbody_b = 0, max_tbody = 0;
  int sleaf_a = 0, sleaf_b = 0, max_sleaves = 0;
  DevBuf<int> epi_leaves;  // own target leaves (cell ids)
  int n_epi_leaves = 0;
  std::vector<P2PItem> items_h;
  DevBuf<P2PItem> items;
  DevBuf<int> p2p_order;
  P2PAux p2p_aux;
  DevBuf<int> item_begin;
  int64_t part_len = 0;
  int max_item_sources = 0;
  std::vector<int4> gitems_h;
  DevBuf<int4> gitems;
  DevBuf<int> gpair;
  DevBuf<int4> citems;  // class-grouped (rotation M2L) items restricted to the shard
  DevBuf<int> cpair;
  int n_citems = 0;
  RotGroups rg;  // their CTA groups and pair records (shared-table rotation M2L)
  DevBuf<int> gather_cells;
  int n_gather_cells = 0;
  std::vector<int> l2l_off;
  DevBuf<int> l2l_cells;
  DevBuf<int> p2m_leaves;
  int n_p2m_leaves = 0;
  DevBuf<int> leaf_owner_off;   // world + 1 source-leaf bounds
  DevBuf<int> body_owner_off;   // world + 1 target-body bounds
  DevBuf<double2> mleaf_send, mleaf_recv;
  DevBuf<double> ysend, yrecv;
  void* comm = nullptr;
};

struct P2MItems {
  DevBuf<int4> d;
  DevBuf<int> red_of;       // per item: its cell's reduce record, or -1
  DevBuf<unsigned> arrive;  // per reduce record: items done (self-resetting)
  int n = 0;
};

struct BemOp {
  int formulation = LAPLACE_SECOND;
  double mu = 1e-3;
  double near_factor = 2.0;
  int n_gauss_singular = 32;
  int64_t n_panels = 0;
  int64_t n = 0;  // unknowns
  int device = 0;
  Plan plan;
  cudaStream_t s_main = nullptr, s_near = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_enter = nullptr, ev_leave = nullptr;  // caller-stream ordering (capi.cu)
  // third stream: the M2L of leaf sources beside the M2M levels (fork after the basis stream)
  cudaStream_t s_far2 = nullptr;
  cudaEvent_t ev_basis = nullptr, ev_m2l2 = nullptr;

  // geometry, panel order
  DevBuf<double> centroid, normal, area, panel_verts, gauss_pos, gauss_w, fine_pos, fine_w;
  DevBuf<double> leg_x, leg_w;
  // per sorted source: weight, panel, absolute position is plan.src.p{x,y,z}
  DevBuf<double> s_weight;
  DevBuf<int> s_panel;
  DevBuf<int> self_src;  // per sorted target: sorted source index of its centroid Gauss point
  DevBuf<unsigned> p2p_sched;  // persistent P2P item counter + CTAs done (self-resetting)
  std::vector<int> h_self_src;
  P2PAux p2p_aux;  // plan items

  // near pairs (CSR by target panel) and the two corrections
  int near_nnz = 0;
  DevBuf<int> near_rowptr, near_cols;
  DevBuf<int2> near_rows;  // per sorted target: its correction row range
  Correction c_sys, c_rhs;

  // work buffers
  DevBuf<double2> srec;  // double-layer near-field source records (k_density)
  DevBuf<double> x_in, y_out, q, dip, wsrc, part, part_dense, stage_x, stage_y;
  DevBuf<double2> M, L, m2l_part, m2m_cout;
  int max_item_sources = 0;
  // dense (direct) P2P lists
  bool dense_ready = false;
  std::vector<P2PItem> dense_items_h;
  DevBuf<P2PItem> dense_items;
  DevBuf<int> dense_src, dense_item_begin;
  int64_t dense_part_len = 0;
  int dense_max_sources = 0;

  ShardWork shard;

  // precomputed P2M basis of the system kernel ([hidx][sorted source], p2m_basis.cu)
  int basis_kind_for_sys = -1;
  int basis_p = -1;
  bool use_basis = false;
  DevBuf<double2> p2m_basis;
  // Laplace kinds: the Gauss points of one panel inside one leaf share x[panel],
  // so their basis columns are pre-summed per (leaf, panel) cluster
  bool basis_clustered = false;
  // clustered kinds: entries for the leaves only, the upper multipoles by octant-grouped M2M
  // (chosen when the direct table, one entry per (cell, cluster of its subtree), would stream
  // several times the leaf table's bytes: deep trees such as cfg5)
  bool basis_leaf_only = false;
  int basis_cols = 0;            // columns of p2m_basis (clusters or sources)
  // direct upward pass (clustered kinds): basis entries (cell, cluster of its subtree)
  // for every M2L source cell and leaf, so the multipoles need no M2M
  std::vector<int> h_cl_range;   // per source cell: first entry, one past last (2 per cell)
  DevBuf<int> cl_panel;          // per entry: panel index
  P2MItems p2m_items, p2m_reduce;            // all multipoles (unsharded)
  P2MItems p2m_leaf_items, p2m_leaf_reduce;  // a shard's own leaves
  const int* p2m_leaf_list = nullptr;
  int n_p2m_slots = 0, n_p2m_leaf_slots = 0;
  DevBuf<double2> p2m_part;

  // GMRES workspaces (Krylov basis, reductions), grow-only
  DevBuf<double> g_basis, g_partials, g_scal, g_y;
  DevBuf<unsigned> g_counter;
  // host-mapped mailbox: the Arnoldi / norm kernels post their scalars and a
  // sequence number straight into pinned host memory; the host spins on it
  // instead of a copy + stream synchronisation per iteration
  double* mbox_h = nullptr;                 // [mbox_cap] values
  double* xpin_h = nullptr;                 // pinned staging of the host solution (n)
  double* ypin_h = nullptr;                 // pinned staging of the least-squares solution y
  int ypin_cap = 0;
  int64_t xpin_cap = 0;
  double* mbox_d = nullptr;
  unsigned long long* mflag_h = nullptr;    // sequence flag
  unsigned long long* mflag_d = nullptr;
  int mbox_cap = 0;
  unsigned long long mbox_seq = 0;

  // CUDA graphs of apply(p), one per order
  std::map<int, cudaGraphExec_t> graphs;
  std::map<int, int> graph_kernels;  // kernel nodes per captured graph
  std::vector<const void*> graph_sig;

  // launch accounting and whole-call device timing (bench instrumentation)
  int64_t kernel_launches = 0;
  int64_t applies = 0;
  cudaEvent_t call_ev[2] = {nullptr, nullptr};
  double last_call_ms = 0.0;
  bool use_graphs = true;
  bool serial_near = false;  // near field in line with the far field (isolated kernel timings)

  // stage timing
  bool timing = false;
  cudaEvent_t ev[2 * N_STAGES] = {};
  // FMMBEM_TIMELINE=1 (with timing on): marks inside the apply, printed per apply to stderr
  // (0 start, 1 basis stream done, 2 M2M done, 3 M2L done, 4 L2L done, 5 P2P done, 6 end)
  cudaEvent_t ev_tl[8] = {};
  double stage_ms[N_STAGES] = {};
  int64_t stage_calls = 0;

  ~BemOp();
};

struct LayerCall {
  int kind;             // LayerKind
  int p;
  bool dense;
  const Correction* corr;
  double alpha, beta;   // y = alpha * x + beta * layer(x)
  const double* x;      // device, panel order (n)
  double* y;            // device (n)
};

void op_init(BemOp& op, const double* panel_vertices, int64_t n_panels, const double* gauss_pts,
             const double* gauss_wts, const double* fine_pts, const double* fine_wts,
             const double* normals, const double* areas, const double* leg_x, const double* leg_w,
             int n_gauss_singular, int formulation, double theta, int n_crit, double mu,
             double near_factor, int max_depth);
void op_layer(BemOp& op, const LayerCall& call, cudaStream_t s, bool sharded = false);
// async on op.s_main; x == nullptr: the input is already in op.x_in, y == nullptr:
// leave the result in op.y_out
void op_apply_device(BemOp& op, const double* x, double* y, int p);
void op_collect_stage_times(BemOp& op);  // after a sync of op.s_main
void op_dense_apply_device(BemOp& op, const double* x, double* y);
void op_rhs_device(BemOp& op, const double* data, double* b, int p, bool dense);
void build_near_pairs(BemOp& op, cudaStream_t s);
bool ensure_p2m_basis(BemOp& op, int p, cudaStream_t s);  // false: over the memory budget
void prepare_p2m_leaf_items(BemOp& op, const int* leaves_dev, int n_leaves);
void launch_p2m_basis(BemOp& op, int p, int C, const double* x, double2* M, cudaStream_t s,
                      const int* leaves = nullptr, int n_leaves = -1);
void build_correction(BemOp& op, int kind, Correction& out, cudaStream_t s);

struct GmresResult {
  std::vector<double> residuals;
  std::vector<int> orders;
  bool converged = false;
  bool stopped = false;  // the progress callback asked to stop
};
// sharding (shard.cu)
void op_shard_setup(BemOp& op, int rank, int world, const int* tleaf_bounds,
                    const int* sleaf_bounds, const unsigned char* nccl_id);
void op_shard_release(BemOp& op);
void op_leaf_work(const BemOp& op, int which, double* w);
void shard_exchange_multipoles(BemOp& op, int C, int p, cudaStream_t s);
void shard_exchange_y(BemOp& op, int nc, double* y, cudaStream_t s);
// collectives of a real shard (NCCL or the host transport), stream-ordered on s
void shard_allgather(BemOp& op, const double* send, double* recv, size_t count, cudaStream_t s);
void shard_allreduce(BemOp& op, double* buf, size_t count, cudaStream_t s);
// own rows (sorted target order, nc per target) of a panel-order vector, and the inverse
// all-gather of every rank's rows into a panel-order vector
void shard_pack_rows(const BemOp& op, int nc, const double* full, double* local, cudaStream_t s);
void shard_gather_rows(BemOp& op, int nc, const double* local, double* full, cudaStream_t s);
void op_shard_setup_host(BemOp& op, int rank, int world, const int* tleaf_bounds,
                         const int* sleaf_bounds, HostAllgather ag, HostAllreduce ar, void* user);
void nccl_unique_id(unsigned char* out);

// per-iteration progress (solver.py:122-123): k (1-based), residual, p; nonzero return stops
typedef int (*GmresCallback)(int32_t k, double residual, int32_t p, void* user);
GmresResult op_gmres(BemOp& op, const double* b_dev, double tol, double eta, int p_initial,
                     int p_min, bool relaxed, int max_iter, double* x_dev,
                     GmresCallback cb = nullptr, void* user = nullptr);

// single-expansion API (expansion_api.cu, fmm.py:36-81); host buffers, full flat layout
void expansion_p2m(const double* rel, int64_t N, const double* q, const double* d, int C, int p,
                   double* coeffs, cudaStream_t s);
void expansion_translate(int kind, const double* dvec, int C, int p, const double* in, double* out,
                         cudaStream_t s);
void expansion_evaluate(int kind, const double* coeffs, int C, int p, const double* rel, int64_t N,
                        bool want_grad, double* pot, double* grad, cudaStream_t s);

// FmmPlan.far_field / near_field (generic channels, host-facing helper)
void plan_evaluate(Plan& plan, int C, const double* q_orig, const double* d_orig, int p,
                   bool want_grad, int parts, double* pot, double* grad, cudaStream_t s);

}  // namespace fmmbem
