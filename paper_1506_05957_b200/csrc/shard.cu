// Partitioned apply across GPUs (one process per GPU), SURVEY.md §8(e).
//
// Every rank holds the same plan (built deterministically from the same
// geometry).  Rank r owns a contiguous range of target leaves (body order,
// balanced by work) and of source leaves (balanced by bodies):
//   1. P2M of its own source leaves, NCCL all-gather of the leaf multipoles
//      (equal-size padded slices), then the (cheap) M2M on every rank;
//   2. M2L only for target cells that are ancestors-or-self of its
//      leaves, P2P items and epilogue only for its leaves -> its y entries;
//   3. NCCL all-gather of the y slices, scattered back to panel order.
// The Krylov vectors stay replicated, so GMRES (and the relaxed-p decisions)
// proceed identically on every rank without an all-reduce.  NCCL is loaded
// with dlopen on first use (the process's own libnccl.so.2, e.g. torch's), so
// the library has no link-time NCCL dependency.  A "virtual" shard (no
// collectives, full upward pass, own y entries only) lets one GPU check every
// rank's restricted work lists against the unpartitioned apply.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <set>

#include "operator.cuh"

namespace fmmbem {
namespace {

// ------------------------------------------------------------------ NCCL (dlopen)
typedef struct { char internal[128]; } NcclId;
typedef int (*fn_getid)(NcclId*);
typedef int (*fn_init)(void**, int, NcclId, int);
typedef int (*fn_allgather)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_destroy)(void*);
typedef const char* (*fn_errstr)(int);
constexpr int NCCL_DOUBLE = 8;  // ncclFloat64
constexpr int NCCL_SUM = 0;     // ncclSum

struct Nccl {
  void* h = nullptr;
  fn_getid get_id = nullptr;
  fn_init init = nullptr;
  fn_allgather allgather = nullptr;
  fn_allreduce allreduce = nullptr;
  fn_destroy destroy = nullptr;
  fn_errstr errstr = nullptr;
  void load() {
    if (h) return;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw CudaFailure(std::string("cannot load libnccl.so.2: ") + dlerror());
    get_id = (fn_getid)dlsym(h, "ncclGetUniqueId");
    init = (fn_init)dlsym(h, "ncclCommInitRank");
    allgather = (fn_allgather)dlsym(h, "ncclAllGather");
    allreduce = (fn_allreduce)dlsym(h, "ncclAllReduce");
    destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
    errstr = (fn_errstr)dlsym(h, "ncclGetErrorString");
    if (!get_id || !init || !allgather || !allreduce || !destroy)
      throw CudaFailure("libnccl.so.2 lacks symbols");
  }
  void check(int rc, const char* what) {
    if (rc) throw CudaFailure(std::string(what) + ": " + (errstr ? errstr(rc) : "nccl error"));
  }
};
Nccl g_nccl;

__global__ void k_pack_leaves(const int* __restrict__ leaves, int n, int CH,
                              const double2* __restrict__ M, double2* __restrict__ out) {
  const int j = blockIdx.x;
  if (j >= n) return;
  const double2* src = M + (size_t)leaves[j] * CH;
  for (int t = threadIdx.x; t < CH; t += blockDim.x) out[(size_t)j * CH + t] = src[t];
}

// M[leaf] for every source leaf from the gathered per-rank slices
__global__ void k_unpack_leaves(const int* __restrict__ leaves, int n_leaves,
                                const int* __restrict__ bounds, int world, int max_per, int CH,
                                const double2* __restrict__ recv, double2* __restrict__ M) {
  const int li = blockIdx.x;
  if (li >= n_leaves) return;
  int r = 0;
  while (r + 1 < world && bounds[r + 1] <= li) ++r;
  const double2* src = recv + ((size_t)r * max_per + (li - bounds[r])) * CH;
  double2* dst = M + (size_t)leaves[li] * CH;
  for (int t = threadIdx.x; t < CH; t += blockDim.x) dst[t] = src[t];
}

// own rows of a panel-order vector in sorted target order: local[i nc + c] = full[perm[a + i] nc + c]
__global__ void k_pack_rows(int64_t n_loc, const int* __restrict__ perm, int tbody_a, int nc,
                            const double* __restrict__ full, double* __restrict__ local) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const int pn = perm[tbody_a + i];
  for (int c = 0; c < nc; ++c) local[i * nc + c] = full[(size_t)pn * nc + c];
}

// y[panel] from the gathered per-rank slices (sorted target order)
__global__ void k_unpack_y(int64_t nt, const int* __restrict__ perm, const int* __restrict__ bounds,
                           int world, int max_per, int nc, const double* __restrict__ recv,
                           double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  int r = 0;
  while (r + 1 < world && bounds[r + 1] <= i) ++r;
  const double* src = recv + ((size_t)r * max_per + (i - bounds[r])) * nc;
  const int pn = perm[i];
  for (int c = 0; c < nc; ++c) y[(size_t)pn * nc + c] = src[c];
}

}  // namespace

void nccl_unique_id(unsigned char* out) {
  g_nccl.load();
  NcclId id;
  g_nccl.check(g_nccl.get_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void op_shard_release(BemOp& op) {
  if (op.shard.comm) {
    g_nccl.destroy(op.shard.comm);
    op.shard.comm = nullptr;
  }
  if (op.shard.hstage) {
    cudaFreeHost(op.shard.hstage);
    op.shard.hstage = nullptr;
    op.shard.hstage_cap = 0;
  }
  op.shard.active = false;
  op.shard.transport = ShardWork::T_VIRTUAL;
  op.shard.local_vectors = false;
}

namespace {
double* host_stage(ShardWork& sw, size_t n) {
  if (sw.hstage_cap < n) {
    if (sw.hstage) FMM_CUDA(cudaFreeHost(sw.hstage));
    sw.hstage_cap = std::max(n, (size_t)1 << 16);
    FMM_CUDA(cudaHostAlloc(&sw.hstage, sw.hstage_cap * sizeof(double), cudaHostAllocDefault));
  }
  return sw.hstage;
}
}  // namespace

void shard_allgather(BemOp& op, const double* send, double* recv, size_t count, cudaStream_t s) {
  ShardWork& sw = op.shard;
  if (sw.transport == ShardWork::T_NCCL) {
    g_nccl.check(g_nccl.allgather(send, recv, count, NCCL_DOUBLE, sw.comm, s), "ncclAllGather");
    return;
  }
  FMM_REQUIRE(sw.transport == ShardWork::T_HOST && sw.host_ag, "shard has no transport");
  double* h = host_stage(sw, count * (sw.world + 1));
  FMM_CUDA(cudaMemcpyAsync(h, send, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  if (sw.host_ag(h, h + count, (int64_t)count, sw.host_user) != 0)
    throw CudaFailure("host transport: all-gather failed");
  FMM_CUDA(cudaMemcpyAsync(recv, h + count, count * sw.world * sizeof(double), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaStreamSynchronize(s));  // the staging buffer is reused by the next collective
}

void shard_allreduce(BemOp& op, double* buf, size_t count, cudaStream_t s) {
  ShardWork& sw = op.shard;
  if (sw.transport == ShardWork::T_NCCL) {
    g_nccl.check(g_nccl.allreduce(buf, buf, count, NCCL_DOUBLE, NCCL_SUM, sw.comm, s), "ncclAllReduce");
    return;
  }
  FMM_REQUIRE(sw.transport == ShardWork::T_HOST && sw.host_ar, "shard has no transport");
  double* h = host_stage(sw, count);
  FMM_CUDA(cudaMemcpyAsync(h, buf, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  if (sw.host_ar(h, (int64_t)count, sw.host_user) != 0) throw CudaFailure("host transport: all-reduce failed");
  FMM_CUDA(cudaMemcpyAsync(buf, h, count * sizeof(double), cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaStreamSynchronize(s));
}

void shard_pack_rows(const BemOp& op, int nc, const double* full, double* local, cudaStream_t s) {
  const ShardWork& sw = op.shard;
  const int64_t nl = sw.tbody_b - sw.tbody_a;
  if (nl > 0)
    k_pack_rows<<<grid_for(nl, 256), 256, 0, s>>>(nl, op.plan.tgt.perm.get(), sw.tbody_a, nc, full, local);
  FMM_LAUNCH_CHECK();
}

void shard_gather_rows(BemOp& op, int nc, const double* local, double* full, cudaStream_t s) {
  ShardWork& sw = op.shard;
  const size_t per = (size_t)sw.max_tbody * nc;
  const int64_t nl = (int64_t)(sw.tbody_b - sw.tbody_a) * nc;
  if (nl > 0 && local != sw.ysend.get())
    FMM_CUDA(cudaMemcpyAsync(sw.ysend.get(), local, nl * sizeof(double), cudaMemcpyDeviceToDevice, s));
  shard_allgather(op, sw.ysend.get(), sw.yrecv.get(), per, s);
  const Tree& T = op.plan.tgt;
  k_unpack_y<<<grid_for(T.n_points, 256), 256, 0, s>>>(T.n_points, T.perm.get(), sw.body_owner_off.get(),
                                                       sw.world, sw.max_tbody, nc, sw.yrecv.get(), full);
  FMM_LAUNCH_CHECK();
}

// per-leaf work weights used by the host-side partitioner
void op_leaf_work(const BemOp& op, int which, double* w) {
  const Plan& pl = op.plan;
  if (which == 1) {  // source leaves: bodies (P2M) in body order
    for (int i = 0; i < pl.src.n_leaves; ++i) w[i] = pl.src.h_body_count[pl.src.h_leaves[i]];
    return;
  }
  // target leaves: P2P interactions (x 18 flop) + the M2L work of the leaf and a
  // share of its ancestors' (x 8 * hcount(12) * 169 flop per pair)
  const Tree& T = pl.tgt;
  std::vector<int> nleaf(T.n_cells, 0);
  for (int c : T.h_leaves)
    for (int a = c; a >= 0; a = T.h_parent[a]) nleaf[a]++;
  const double m2l_cost = 8.0 * hcount(12) * 169.0;
  for (int li = 0; li < T.n_leaves; ++li) {
    const int c = T.h_leaves[li];
    double inter = 0.0;
    for (int e = pl.h_p2p_row[c]; e < pl.h_p2p_row[c + 1]; ++e)
      inter += (double)pl.src.h_body_count[pl.h_p2p_src[e]] * T.h_body_count[c];
    double m2l = 0.0;
    for (int a = c; a >= 0; a = T.h_parent[a])
      m2l += (double)(pl.h_m2l_row[a + 1] - pl.h_m2l_row[a]) / nleaf[a];
    w[li] = 18.0 * inter + m2l_cost * m2l;
  }
}

void op_shard_setup(BemOp& op, int rank, int world, const int* tb, const int* sb,
                    const unsigned char* nccl_id) {
  const Plan& pl = op.plan;
  const Tree& T = pl.tgt;
  const Tree& S = pl.src;
  FMM_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
  FMM_REQUIRE(tb[0] == 0 && tb[world] == T.n_leaves && sb[0] == 0 && sb[world] == S.n_leaves,
              "leaf bounds must cover all leaves");
  for (int r = 0; r < world; ++r)
    FMM_REQUIRE(tb[r] <= tb[r + 1] && sb[r] <= sb[r + 1], "leaf bounds must be non-decreasing");
  op_shard_release(op);
  ShardWork& sw = op.shard;
  cudaStream_t s = op.s_main;
  sw.rank = rank;
  sw.world = world;
  sw.virtual_mode = nccl_id == nullptr;
  sw.tleaf_a = tb[rank];
  sw.tleaf_b = tb[rank + 1];
  sw.sleaf_a = sb[rank];
  sw.sleaf_b = sb[rank + 1];
  auto body_of = [&](int li) { return li < T.n_leaves ? T.h_body_start[T.h_leaves[li]] : (int)T.n_points; };
  std::vector<int> body_bounds(world + 1);
  for (int r = 0; r <= world; ++r) body_bounds[r] = body_of(tb[r]);
  sw.tbody_a = body_bounds[rank];
  sw.tbody_b = body_bounds[rank + 1];
  sw.max_tbody = 0;
  sw.max_sleaves = 0;
  for (int r = 0; r < world; ++r) {
    sw.max_tbody = std::max(sw.max_tbody, body_bounds[r + 1] - body_bounds[r]);
    sw.max_sleaves = std::max(sw.max_sleaves, sb[r + 1] - sb[r]);
  }
  // ---- target side: own leaves, P2P items, epilogue lists
  std::vector<int> own(T.h_leaves.begin() + sw.tleaf_a, T.h_leaves.begin() + sw.tleaf_b);
  sw.n_epi_leaves = (int)own.size();
  sw.epi_leaves.upload(own.empty() ? std::vector<int>(1, 0) : own, s);
  sw.items_h.clear();
  std::vector<int> ib(own.size() + 1, 0);
  sw.part_len = 0;
  sw.max_item_sources = 1;
  for (size_t li = 0; li < own.size(); ++li) {
    const int t = own[li], nt = T.h_body_count[t];
    ib[li] = (int)sw.items_h.size();
    int b = pl.h_p2p_row[t];
    const int e = pl.h_p2p_row[t + 1];
    while (b < e) {  // same slicing rule as plan_make_items (<= Plan::item_sources() sources)
      int acc = 0, k = b;
      while (k < e && (acc == 0 || acc + S.h_body_count[pl.h_p2p_src[k]] <= pl.item_sources())) {
        acc += S.h_body_count[pl.h_p2p_src[k]];
        ++k;
      }
      sw.items_h.push_back(P2PItem{t, b, k, (int)sw.part_len});
      sw.part_len += nt;
      sw.max_item_sources = std::max(sw.max_item_sources, acc);
      b = k;
    }
  }
  ib[own.size()] = (int)sw.items_h.size();
  sw.items.upload(sw.items_h.empty() ? std::vector<P2PItem>(1) : sw.items_h, s);
  {
    const std::vector<int> ord = p2p_schedule(op.plan.tgt, op.plan.src, sw.items_h, op.plan.h_p2p_src);
    sw.p2p_order.upload(ord.empty() ? std::vector<int>(1, 0) : ord, s);
  }
  sw.item_begin.upload(ib, s);
  sw.p2p_aux.build(op.plan.src, op.plan.tgt, sw.items_h, op.plan.h_p2p_src, op.h_self_src, s);
  op.part.ensure((size_t)std::max<int64_t>(std::max(sw.part_len, pl.part_len), 1) * 3);
  // needed target cells: ancestors-or-self of own leaves
  std::vector<uint8_t> need(T.n_cells, 0);
  for (int c : own)
    for (int a = c; a >= 0 && !need[a]; a = T.h_parent[a]) need[a] = 1;
  std::vector<int> cells;
  for (int c = 0; c < T.n_cells; ++c)
    if (need[c]) cells.push_back(c);
  sw.n_gather_cells = (int)cells.size();
  sw.gather_cells.upload(cells.empty() ? std::vector<int>(1, 0) : cells, s);
  // M2L: the plan's offset-sorted pairs restricted to needed targets, re-cut into <= 8-pair items
  std::vector<int> tgt_of(pl.n_m2l);
  for (int c = 0; c < T.n_cells; ++c)
    for (int e = pl.h_m2l_row[c]; e < pl.h_m2l_row[c + 1]; ++e) tgt_of[e] = c;
  std::vector<int> gp;
  std::vector<int4> gi;
  {
    std::vector<int> gp_all(std::max(pl.n_m2l, 1));
    if (pl.n_m2l)
      FMM_CUDA(cudaMemcpy(gp_all.data(), pl.m2l_gpair.get(), pl.n_m2l * sizeof(int), cudaMemcpyDeviceToHost));
    for (const int4& it : pl.m2l_gitems) {
      const int start = (int)gp.size();
      for (int i = it.y; i < it.z; ++i)
        if (need[tgt_of[gp_all[i]]]) gp.push_back(gp_all[i]);
      if ((int)gp.size() > start) gi.push_back(make_int4(it.x, start, (int)gp.size(), 0));
    }
  }
  sw.gitems_h = gi;
  sw.gitems.upload(gi.empty() ? std::vector<int4>(1) : gi, s);
  sw.gpair.upload(gp.empty() ? std::vector<int>(1, 0) : gp, s);
  // the same restriction of the class-grouped items (rotation M2L)
  {
    std::vector<int> cp;
    std::vector<int4> ci;
    for (const int4& it : pl.m2l_citems) {
      const int start = (int)cp.size();
      for (int i = it.y; i < it.z; ++i)
        if (need[tgt_of[pl.h_m2l_cpair[i]]]) cp.push_back(pl.h_m2l_cpair[i]);
      if ((int)cp.size() > start) ci.push_back(make_int4(pl.h_m2l_off[cp[start]], start, (int)cp.size(), 0));
    }
    sw.n_citems = (int)ci.size();
    sw.citems.upload(ci.empty() ? std::vector<int4>(1) : ci, s);
    sw.cpair.upload(cp.empty() ? std::vector<int>(1, 0) : cp, s);
    if (!ci.empty()) sw.rg.build(ci, cp, pl.h_m2l_src, pl.h_m2l_off, pl.h_rot_dir, s);
  }
  // L2L: needed cells whose parent carries a local expansion (plan's pruned lists)
  std::vector<int> l2l_all;
  if (!pl.l2l_level_off.empty() && pl.l2l_level_off.back() > 0) {
    l2l_all.resize(pl.l2l_level_off.back());
    FMM_CUDA(cudaMemcpy(l2l_all.data(), pl.l2l_cells.get(), l2l_all.size() * sizeof(int), cudaMemcpyDeviceToHost));
  }
  std::vector<int> lc;
  sw.l2l_off.assign(1, 0);
  for (size_t l = 0; l + 1 < pl.l2l_level_off.size(); ++l) {
    for (int k = pl.l2l_level_off[l]; k < pl.l2l_level_off[l + 1]; ++k)
      if (need[l2l_all[k]]) lc.push_back(l2l_all[k]);
    sw.l2l_off.push_back((int)lc.size());
  }
  sw.l2l_cells.upload(lc.empty() ? std::vector<int>(1, 0) : lc, s);
  // ---- source side
  std::vector<int> sl(S.h_leaves.begin() + sw.sleaf_a, S.h_leaves.begin() + sw.sleaf_b);
  sw.n_p2m_leaves = (int)sl.size();
  sw.p2m_leaves.upload(sl.empty() ? std::vector<int>(1, 0) : sl, s);
  std::vector<int> sbv(sb, sb + world + 1);
  sw.leaf_owner_off.upload(sbv, s);
  sw.body_owner_off.upload(body_bounds, s);
  sw.ysend.ensure((size_t)std::max(sw.max_tbody, 1) * 3);
  sw.yrecv.ensure((size_t)std::max(sw.max_tbody, 1) * 3 * world);
  // ---- communicator
  sw.transport = sw.virtual_mode ? ShardWork::T_VIRTUAL : ShardWork::T_NCCL;
  if (!sw.virtual_mode) {
    g_nccl.load();
    NcclId id;
    std::memcpy(id.internal, nccl_id, 128);
    FMM_CUDA(cudaSetDevice(op.device));
    g_nccl.check(g_nccl.init(&sw.comm, world, id, rank), "ncclCommInitRank");
  }
  FMM_CUDA(cudaStreamSynchronize(s));
  op.p2m_leaf_list = nullptr;  // (sw.p2m_leaves was reallocated)
  prepare_p2m_leaf_items(op, sw.p2m_leaves.get(), sw.n_p2m_leaves);
  // graphs were captured for the unpartitioned apply
  for (auto& kv : op.graphs) cudaGraphExecDestroy(kv.second);
  op.graphs.clear();
  op.graph_kernels.clear();
  op.graph_sig.clear();
  sw.active = true;
}

void op_shard_setup_host(BemOp& op, int rank, int world, const int* tb, const int* sb,
                         HostAllgather ag, HostAllreduce ar, void* user) {
  FMM_REQUIRE(ag && ar, "host transport needs all-gather and all-reduce callbacks");
  // the work split as for NCCL, built in virtual mode (no communicator), then switched over
  op_shard_setup(op, rank, world, tb, sb, nullptr);
  ShardWork& sw = op.shard;
  sw.virtual_mode = false;
  sw.transport = ShardWork::T_HOST;
  sw.host_ag = ag;
  sw.host_ar = ar;
  sw.host_user = user;
}

void shard_exchange_multipoles(BemOp& op, int C, int p, cudaStream_t s) {
  ShardWork& sw = op.shard;
  const int CH = C * hcount(p);
  const size_t per = (size_t)sw.max_sleaves * CH;
  sw.mleaf_send.ensure(std::max<size_t>(per, 1));
  sw.mleaf_recv.ensure(std::max<size_t>(per * sw.world, 1));
  if (sw.n_p2m_leaves)
    k_pack_leaves<<<sw.n_p2m_leaves, 128, 0, s>>>(sw.p2m_leaves.get(), sw.n_p2m_leaves, CH, op.M.get(),
                                                  sw.mleaf_send.get());
  FMM_LAUNCH_CHECK();
  shard_allgather(op, reinterpret_cast<const double*>(sw.mleaf_send.get()),
                  reinterpret_cast<double*>(sw.mleaf_recv.get()), per * 2, s);
  const Tree& S = op.plan.src;
  k_unpack_leaves<<<S.n_leaves, 128, 0, s>>>(S.leaves.get(), S.n_leaves, sw.leaf_owner_off.get(),
                                             sw.world, sw.max_sleaves, CH, sw.mleaf_recv.get(),
                                             op.M.get());
  FMM_LAUNCH_CHECK();
}

void shard_exchange_y(BemOp& op, int nc, double* y, cudaStream_t s) {
  ShardWork& sw = op.shard;
  const size_t per = (size_t)sw.max_tbody * nc;
  shard_allgather(op, sw.ysend.get(), sw.yrecv.get(), per, s);
  const Tree& T = op.plan.tgt;
  k_unpack_y<<<grid_for(T.n_points, 256), 256, 0, s>>>(T.n_points, T.perm.get(), sw.body_owner_off.get(),
                                                       sw.world, sw.max_tbody, nc, sw.yrecv.get(), y);
  FMM_LAUNCH_CHECK();
}

}  // namespace fmmbem
