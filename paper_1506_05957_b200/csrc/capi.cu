// extern "C" boundary (include/fmmbem_b200.h): argument checks, device
// selection, host<->device staging and error mapping.  No compute here.
#include <cstring>
#include <memory>

#include "../../include/fmmbem_b200.h"
#include "operator.cuh"

using namespace fmmbem;

struct fmmbem_plan {
  Plan* plan = nullptr;
  std::unique_ptr<Plan> owned;
  cudaStream_t stream = nullptr;
  int device = 0;
  ~fmmbem_plan() {
    if (stream) cudaStreamDestroy(stream);
  }
};

struct fmmbem_op {
  std::unique_ptr<BemOp> op;
  fmmbem_plan plan_view;  // borrowed view on op->plan
  int device = 0;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return FMMBEM_OK;
  } catch (const ArgumentError& e) {
    g_err = e.what();
    return FMMBEM_EINVAL;
  } catch (const CudaFailure& e) {
    g_err = e.what();
    return FMMBEM_ECUDA;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return FMMBEM_EINTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FMMBEM_EINTERNAL;
  }
}

void select(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw CudaFailure("no CUDA device available (the fmmbem_b200 path has no CPU fallback)");
  }
  FMM_REQUIRE(device >= 0 && device < n, "device index out of range");
  FMM_CUDA(cudaSetDevice(device));
}

__global__ void k_dfma_probe(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

// Stream ordering with the caller (include/fmmbem_b200.h): the op's own stream waits for
// the work already queued on the caller's stream (NULL = the legacy default stream, where
// torch queues by default), and the caller's stream waits for the op's work on the way out.
void enter_caller_stream(BemOp& op, cudaStream_t caller) {
  FMM_CUDA(cudaEventRecord(op.ev_enter, caller));
  FMM_CUDA(cudaStreamWaitEvent(op.s_main, op.ev_enter, 0));
}

void leave_caller_stream(BemOp& op, cudaStream_t caller) {
  FMM_CUDA(cudaEventRecord(op.ev_leave, op.s_main));
  FMM_CUDA(cudaStreamWaitEvent(caller, op.ev_leave, 0));
}

}  // namespace

extern "C" {

const char* fmmbem_last_error(void) { return g_err.c_str(); }

int fmmbem_version(void) { return 1; }

int fmmbem_expansion_p2m(const double* rel, int64_t n, const double* charges, const double* dipoles,
                         int C, int p, double* coeffs, int device) {
  return guarded([&] {
    FMM_REQUIRE(coeffs && (rel || n == 0), "null argument");
    select(device);
    expansion_p2m(rel, n, charges, dipoles, C, p, coeffs, 0);
  });
}

int fmmbem_expansion_translate(int kind, const double* d, int C, int p, const double* coeffs_in,
                               double* coeffs_out, int device) {
  return guarded([&] {
    FMM_REQUIRE(d && coeffs_in && coeffs_out, "null argument");
    select(device);
    expansion_translate(kind, d, C, p, coeffs_in, coeffs_out, 0);
  });
}

int fmmbem_expansion_evaluate(int kind, const double* coeffs, int C, int p, const double* rel,
                              int64_t n, int want_gradient, double* pot, double* grad, int device) {
  return guarded([&] {
    FMM_REQUIRE(coeffs && pot && (rel || n == 0) && (!want_gradient || grad), "null argument");
    FMM_REQUIRE(C >= 1 && n >= 0, "bad sizes");
    select(device);
    expansion_evaluate(kind, coeffs, C, p, rel, n, want_gradient != 0, pot, grad, 0);
  });
}

int fmmbem_device_count(int* count) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return FMMBEM_OK;
}

int fmmbem_fp64_peak(int device, double* tflops) {
  return guarded([&] {
    select(device);
    cudaDeviceProp prop;
    FMM_CUDA(cudaGetDeviceProperties(&prop, device));
    DevBuf<double> out(1);
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 2048;
    k_dfma_probe<<<blocks, threads>>>(out.get(), 64, 1.0000001, 1e-7);
    FMM_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    FMM_CUDA(cudaEventCreate(&e0));
    FMM_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      FMM_CUDA(cudaEventRecord(e0));
      k_dfma_probe<<<blocks, threads>>>(out.get(), iters, 1.0000001, 1e-7);
      FMM_CUDA(cudaEventRecord(e1));
      FMM_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      FMM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tflops = 2.0 * 8 * 16 * (double)iters * blocks * threads / (best * 1e-3) / 1e12;
  });
}

int fmmbem_plan_create(const double* src_xyz, int64_t ns, const double* tgt_xyz, int64_t nt,
                       int n_crit, double theta, int max_depth, int device, fmmbem_plan** out) {
  return guarded([&] {
    FMM_REQUIRE(out && src_xyz && tgt_xyz, "null argument");
    select(device);
    upload_index_tables();
    auto h = std::make_unique<fmmbem_plan>();
    h->owned = std::make_unique<Plan>();
    h->plan = h->owned.get();
    h->device = device;
    FMM_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    plan_build(*h->plan, src_xyz, ns, tgt_xyz, nt, n_crit, theta, max_depth, h->stream);
    *out = h.release();
  });
}

int fmmbem_plan_destroy(fmmbem_plan* plan) {
  return guarded([&] {
    if (!plan) return;
    if (plan->owned) cudaSetDevice(plan->device);
    delete plan;
  });
}

int fmmbem_plan_sizes(const fmmbem_plan* h, int64_t* sizes) {
  return guarded([&] {
    FMM_REQUIRE(h && sizes, "null argument");
    const Plan& p = *h->plan;
    sizes[0] = p.src.n_cells;
    sizes[1] = p.tgt.n_cells;
    sizes[2] = p.src.n_leaves;
    sizes[3] = p.tgt.n_leaves;
    sizes[4] = p.n_m2l;
    sizes[5] = p.n_p2p;
    sizes[6] = p.src.n_levels;
    sizes[7] = p.tgt.n_levels;
    sizes[8] = p.p2p_interactions;
    sizes[9] = p.n_offsets;
  });
}

int fmmbem_plan_tree(const fmmbem_plan* h, int which, int64_t* perm, double* center,
                     double* half_width, int32_t* level, int32_t* parent, int64_t* body_start,
                     int64_t* body_count, uint8_t* is_leaf) {
  return guarded([&] {
    FMM_REQUIRE(h && (which == 0 || which == 1), "bad tree selector");
    select(h->device);
    const Tree& t = which == 0 ? h->plan->src : h->plan->tgt;
    const int nc = t.n_cells;
    if (perm) {
      auto v = t.perm.download();
      for (int64_t i = 0; i < t.n_points; ++i) perm[i] = v[i];
    }
    if (center)
      for (int c = 0; c < nc; ++c) {
        center[3 * c] = t.h_cx[c];
        center[3 * c + 1] = t.h_cy[c];
        center[3 * c + 2] = t.h_cz[c];
      }
    if (half_width) {
      auto v = t.half.download();
      std::memcpy(half_width, v.data(), nc * sizeof(double));
    }
    for (int c = 0; c < nc; ++c) {
      if (level) level[c] = t.h_level[c];
      if (parent) parent[c] = t.h_parent[c];
      if (body_start) body_start[c] = t.h_body_start[c];
      if (body_count) body_count[c] = t.h_body_count[c];
      if (is_leaf) is_leaf[c] = t.h_is_leaf[c];
    }
  });
}

int fmmbem_plan_pairs(const fmmbem_plan* h, int which, int32_t* pairs) {
  return guarded([&] {
    FMM_REQUIRE(h && pairs && (which == 0 || which == 1), "bad pair selector");
    const Plan& p = *h->plan;
    const std::vector<int>& row = which == 0 ? p.h_m2l_row : p.h_p2p_row;
    const std::vector<int>& src = which == 0 ? p.h_m2l_src : p.h_p2p_src;
    for (int t = 0; t + 1 < (int)row.size(); ++t)
      for (int e = row[t]; e < row[t + 1]; ++e) {
        pairs[2 * e] = src[e];
        pairs[2 * e + 1] = t;
      }
  });
}

int fmmbem_plan_evaluate(fmmbem_plan* h, const double* charges, const double* dipoles, int C,
                         int p, int want_gradient, int parts, double* pot, double* grad) {
  return guarded([&] {
    FMM_REQUIRE(h && pot, "null argument");
    FMM_REQUIRE(parts >= 1 && parts <= 3, "parts must be 1 (far), 2 (near) or 3");
    FMM_REQUIRE(!want_gradient || grad, "gradient output required");
    FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
    select(h->device);
    Plan& pl = *h->plan;
    const int64_t ns = pl.src.n_points, nt = pl.tgt.n_points;
    cudaStream_t s = h->stream;
    EvalWork& w = pl.eval;  // grow-only: repeated evaluations allocate nothing
    DevBuf<double>&dq = w.q, &dd = w.d, &dpot = w.pot, &dgrad = w.grad;
    if (charges) dq.put(charges, (size_t)C * ns, s);
    if (dipoles) dd.put(dipoles, (size_t)C * ns * 3, s);
    dpot.zero_n((size_t)C * nt, s);
    dgrad.zero_n(want_gradient ? (size_t)C * nt * 3 : 1, s);
    plan_evaluate(pl, C, charges ? dq.get() : nullptr, dipoles ? dd.get() : nullptr, p,
                  want_gradient != 0, parts, dpot.get(), want_gradient ? dgrad.get() : nullptr, s);
    FMM_CUDA(cudaMemcpyAsync(pot, dpot.get(), (size_t)C * nt * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (want_gradient)
      FMM_CUDA(cudaMemcpyAsync(grad, dgrad.get(), (size_t)C * nt * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  });
}

int fmmbem_op_create(const double* panel_vertices, int64_t n_panels, const double* gauss_pts,
                     const double* gauss_wts, const double* fine_pts, const double* fine_wts,
                     const double* normals, const double* areas, const double* leg_x,
                     const double* leg_w, int n_gauss_singular, int formulation, double theta,
                     int n_crit, double mu, double near_factor, int max_depth, int device,
                     fmmbem_op** out) {
  return guarded([&] {
    FMM_REQUIRE(out && panel_vertices && gauss_pts && gauss_wts && fine_pts && fine_wts && normals &&
                    areas && leg_x && leg_w,
                "null argument");
    select(device);
    auto h = std::make_unique<fmmbem_op>();
    h->op = std::make_unique<BemOp>();
    h->device = device;
    h->op->device = device;
    op_init(*h->op, panel_vertices, n_panels, gauss_pts, gauss_wts, fine_pts, fine_wts, normals,
            areas, leg_x, leg_w, n_gauss_singular, formulation, theta, n_crit, mu, near_factor,
            max_depth);
    h->plan_view.plan = &h->op->plan;
    h->plan_view.device = device;
    FMM_CUDA(cudaStreamCreateWithFlags(&h->plan_view.stream, cudaStreamNonBlocking));
    *out = h.release();
  });
}

int fmmbem_op_destroy(fmmbem_op* op) {
  return guarded([&] {
    if (!op) return;
    cudaSetDevice(op->device);
    delete op;
  });
}

int fmmbem_op_size(const fmmbem_op* op, int64_t* n) {
  return guarded([&] {
    FMM_REQUIRE(op && n, "null argument");
    *n = op->op->n;
  });
}

int fmmbem_op_plan(fmmbem_op* op, fmmbem_plan** plan) {
  return guarded([&] {
    FMM_REQUIRE(op && plan, "null argument");
    *plan = &op->plan_view;
  });
}

int fmmbem_op_apply(fmmbem_op* h, const double* x, double* y, int p) {
  return guarded([&] {
    FMM_REQUIRE(h && x && y, "null argument");
    FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
    select(h->device);
    BemOp& op = *h->op;
    cudaStream_t s = op.s_main;
    op.stage_x.ensure(op.n);
    op.stage_y.ensure(op.n);
    FMM_CUDA(cudaMemcpyAsync(op.stage_x.get(), x, op.n * sizeof(double), cudaMemcpyHostToDevice, s));
    op_apply_device(op, op.stage_x.get(), op.stage_y.get(), p);
    FMM_CUDA(cudaMemcpyAsync(y, op.stage_y.get(), op.n * sizeof(double), cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    op_collect_stage_times(op);
  });
}

int fmmbem_op_apply_device(fmmbem_op* h, const double* x_dev, double* y_dev, int p, void* stream) {
  return guarded([&] {
    FMM_REQUIRE(h && x_dev && y_dev, "null argument");
    FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
    select(h->device);
    BemOp& op = *h->op;
    const cudaStream_t caller = (cudaStream_t)stream;
    enter_caller_stream(op, caller);
    op_apply_device(op, x_dev, y_dev, p);
    leave_caller_stream(op, caller);
    if (!caller || op.timing) {  // NULL stream: synchronous, like the host variant
      FMM_CUDA(cudaStreamSynchronize(op.s_main));
      op_collect_stage_times(op);
    }
  });
}

int fmmbem_op_dense_apply(fmmbem_op* h, const double* x, double* y) {
  return guarded([&] {
    FMM_REQUIRE(h && x && y, "null argument");
    select(h->device);
    BemOp& op = *h->op;
    DevBuf<double> dx, dy(op.n);
    dx.upload(x, op.n, op.s_main);
    op_dense_apply_device(op, dx.get(), dy.get());
    FMM_CUDA(cudaMemcpyAsync(y, dy.get(), op.n * sizeof(double), cudaMemcpyDeviceToHost, op.s_main));
    FMM_CUDA(cudaStreamSynchronize(op.s_main));
  });
}

int fmmbem_op_assemble_rhs(fmmbem_op* h, const double* data, int p, int dense, double* b) {
  return guarded([&] {
    FMM_REQUIRE(h && data && b, "null argument");
    FMM_REQUIRE(p >= 0 && p <= P_MAX, "expansion order p must be in [0, 20]");
    select(h->device);
    BemOp& op = *h->op;
    DevBuf<double> dd, db(op.n);
    dd.upload(data, op.n, op.s_main);
    op_rhs_device(op, dd.get(), db.get(), p, dense != 0);
    FMM_CUDA(cudaMemcpyAsync(b, db.get(), op.n * sizeof(double), cudaMemcpyDeviceToHost, op.s_main));
    FMM_CUDA(cudaStreamSynchronize(op.s_main));
  });
}

int fmmbem_op_correction(const fmmbem_op* h, int which, int64_t* nnz_pairs, int32_t* block,
                         int64_t* indptr, int64_t* indices, double* data) {
  return guarded([&] {
    FMM_REQUIRE(h && (which == 0 || which == 1), "bad correction selector");
    select(h->device);
    const BemOp& op = *h->op;
    const Correction& c = which == 0 ? op.c_sys : op.c_rhs;
    if (nnz_pairs) *nnz_pairs = op.near_nnz;
    if (block) *block = c.block;
    if (indptr) {
      auto v = op.near_rowptr.download();
      for (size_t i = 0; i < v.size(); ++i) indptr[i] = v[i];
    }
    if (indices) {
      auto v = op.near_cols.download();
      for (int i = 0; i < op.near_nnz; ++i) indices[i] = v[i];
    }
    if (data) {
      auto v = c.vals.download();
      std::memcpy(data, v.data(), (size_t)op.near_nnz * c.block * sizeof(double));
    }
  });
}

static void gmres_common(fmmbem_op* h, const double* b_dev, double tol, double eta, int p_initial,
                         int p_min, int relaxed, int max_iter, double* x_dev, double* residuals,
                         int32_t* orders, int32_t* n_iter, int32_t* converged,
                         fmmbem_gmres_callback cb, void* user) {
  GmresResult r = op_gmres(*h->op, b_dev, tol, eta, p_initial, p_min, relaxed != 0, max_iter,
                           x_dev, cb, user);
  for (size_t k = 0; k < r.orders.size(); ++k) {
    if (residuals) residuals[k] = r.residuals[k];
    if (orders) orders[k] = r.orders[k];
  }
  if (n_iter) *n_iter = (int32_t)r.orders.size();
  if (converged) *converged = r.converged ? 1 : 0;
}

int fmmbem_op_gmres(fmmbem_op* h, const double* b, double tol, double eta, int p_initial,
                    int p_min, int relaxed, int max_iter, double* x, double* residuals,
                    int32_t* orders, int32_t* n_iter, int32_t* converged,
                    fmmbem_gmres_callback cb, void* user) {
  return guarded([&] {
    FMM_REQUIRE(h && b && x, "null argument");
    select(h->device);
    BemOp& op = *h->op;
    op.stage_x.ensure(op.n);
    op.stage_y.ensure(op.n);
    FMM_CUDA(cudaEventRecord(op.call_ev[0], op.s_main));
    FMM_CUDA(cudaMemcpyAsync(op.stage_x.get(), b, op.n * sizeof(double), cudaMemcpyHostToDevice, op.s_main));
    gmres_common(h, op.stage_x.get(), tol, eta, p_initial, p_min, relaxed, max_iter,
                 op.stage_y.get(), residuals, orders, n_iter, converged, cb, user);
    // x straight into the caller's buffer when it is page-locked (the Python wrapper hands
    // out pinned arrays), else through a pinned staging buffer (a pageable D2H copy is
    // staged by the driver, slower)
    cudaPointerAttributes pa{};
    const bool x_pinned = cudaPointerGetAttributes(&pa, x) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    if (!x_pinned) cudaGetLastError();
    if (!x_pinned && op.xpin_cap < op.n) {
      if (op.xpin_h) FMM_CUDA(cudaFreeHost(op.xpin_h));
      FMM_CUDA(cudaHostAlloc(&op.xpin_h, op.n * sizeof(double), cudaHostAllocDefault));
      op.xpin_cap = op.n;
    }
    FMM_CUDA(cudaMemcpyAsync(x_pinned ? x : op.xpin_h, op.stage_y.get(), op.n * sizeof(double),
                             cudaMemcpyDeviceToHost, op.s_main));
    FMM_CUDA(cudaEventRecord(op.call_ev[1], op.s_main));
    FMM_CUDA(cudaStreamSynchronize(op.s_main));
    if (!x_pinned) std::memcpy(x, op.xpin_h, op.n * sizeof(double));
    float ms = 0.f;
    FMM_CUDA(cudaEventElapsedTime(&ms, op.call_ev[0], op.call_ev[1]));
    op.last_call_ms = ms;
  });
}

int fmmbem_op_gmres_device(fmmbem_op* h, const double* b_dev, double tol, double eta,
                           int p_initial, int p_min, int relaxed, int max_iter, double* x_dev,
                           double* residuals, int32_t* orders, int32_t* n_iter,
                           int32_t* converged, fmmbem_gmres_callback cb, void* user,
                           void* stream) {
  return guarded([&] {
    FMM_REQUIRE(h && b_dev && x_dev, "null argument");
    select(h->device);
    BemOp& op = *h->op;
    const cudaStream_t caller = (cudaStream_t)stream;
    enter_caller_stream(op, caller);
    FMM_CUDA(cudaEventRecord(op.call_ev[0], op.s_main));
    gmres_common(h, b_dev, tol, eta, p_initial, p_min, relaxed, max_iter, x_dev, residuals,
                 orders, n_iter, converged, cb, user);
    FMM_CUDA(cudaEventRecord(op.call_ev[1], op.s_main));
    leave_caller_stream(op, caller);
    FMM_CUDA(cudaStreamSynchronize(op.s_main));
    float ms = 0.f;
    FMM_CUDA(cudaEventElapsedTime(&ms, op.call_ev[0], op.call_ev[1]));
    op.last_call_ms = ms;
  });
}

int fmmbem_op_set_timing(fmmbem_op* h, int enable, int use_graphs) {
  return guarded([&] {
    FMM_REQUIRE(h, "null argument");
    h->op->timing = enable != 0;
    h->op->use_graphs = use_graphs != 0;
  });
}

int fmmbem_op_set_serial(fmmbem_op* h, int serial) {
  return guarded([&] {
    FMM_REQUIRE(h, "null argument");
    h->op->serial_near = serial != 0;
  });
}

int fmmbem_op_stage_times(fmmbem_op* h, double* ms6, int64_t* calls, int reset) {
  return guarded([&] {
    FMM_REQUIRE(h, "null argument");
    BemOp& op = *h->op;
    if (ms6)
      for (int i = 0; i < N_STAGES; ++i) ms6[i] = op.stage_ms[i];
    if (calls) *calls = op.stage_calls;
    if (reset) {
      for (auto& v : op.stage_ms) v = 0.0;
      op.stage_calls = 0;
    }
  });
}

int fmmbem_nccl_unique_id(unsigned char* out128) {
  return guarded([&] {
    FMM_REQUIRE(out128, "null argument");
    nccl_unique_id(out128);
  });
}

int fmmbem_op_leaf_work(const fmmbem_op* h, int which, double* w) {
  return guarded([&] {
    FMM_REQUIRE(h && w && (which == 0 || which == 1), "bad arguments");
    op_leaf_work(*h->op, which, w);
  });
}

int fmmbem_op_shard(fmmbem_op* h, int rank, int world, const int32_t* tleaf_bounds,
                    const int32_t* sleaf_bounds, const unsigned char* nccl_id) {
  return guarded([&] {
    FMM_REQUIRE(h && tleaf_bounds && sleaf_bounds, "null argument");
    select(h->device);
    op_shard_setup(*h->op, rank, world, tleaf_bounds, sleaf_bounds, nccl_id);
  });
}

int fmmbem_op_shard_host(fmmbem_op* h, int rank, int world, const int32_t* tleaf_bounds,
                         const int32_t* sleaf_bounds, fmmbem_allgather_fn allgather,
                         fmmbem_allreduce_fn allreduce, void* user) {
  return guarded([&] {
    FMM_REQUIRE(h && tleaf_bounds && sleaf_bounds && allgather && allreduce, "null argument");
    select(h->device);
    op_shard_setup_host(*h->op, rank, world, tleaf_bounds, sleaf_bounds, allgather, allreduce, user);
  });
}

int fmmbem_op_unshard(fmmbem_op* h) {
  return guarded([&] {
    FMM_REQUIRE(h, "null argument");
    select(h->device);
    op_shard_release(*h->op);
    BemOp& op = *h->op;
    for (auto& kv : op.graphs) cudaGraphExecDestroy(kv.second);
    op.graphs.clear();
    op.graph_kernels.clear();
    op.graph_sig.clear();
  });
}

int fmmbem_op_counters(fmmbem_op* h, int64_t* kernel_launches, int64_t* applies,
                       double* last_call_ms) {
  return guarded([&] {
    FMM_REQUIRE(h, "null argument");
    if (kernel_launches) *kernel_launches = h->op->kernel_launches;
    if (applies) *applies = h->op->applies;
    if (last_call_ms) *last_call_ms = h->op->last_call_ms;
  });
}

}  // extern "C"
