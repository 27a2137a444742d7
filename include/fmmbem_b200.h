/*
 * fmmbem_b200 — C ABI of the B200 (sm_100a) FMM-BEM hot path.
 *
 * The reference (arXiv:1506.05957 package, /root/reference/pkg/src/fmmbem) is
 * pure Python; its plug-in point for this path is a Python duck type, not an
 * FFI: solver.gmres(apply_fn, ...) calls apply_fn(x, p) (solver.py:69,99) and
 * solver.solve(operator, ...) passes operator.apply (solver.py:142).  Each
 * entry point below replaces one method of that surface; the ctypes binding
 * that mirrors the reference classes is paper_1506_05957_b200/_native.py and
 * INTEGRATION.md shows the binding a maintainer of the reference would add.
 *
 * Conventions: every function returns 0 on success, FMMBEM_EINVAL for invalid
 * arguments (the reference raises ValueError) and FMMBEM_ECUDA for device
 * failures; fmmbem_last_error() returns the thread's last message.  Arrays are
 * C-contiguous float64 / int64 in the reference's own shapes and orders.
 * "host" buffers are ordinary memory; *_device variants take device pointers.
 * Handles are not re-entrant (one stream per operator, like the reference's
 * sequential solver loop).
 */
#ifndef FMMBEM_B200_H
#define FMMBEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMMBEM_OK 0
#define FMMBEM_EINVAL 1
#define FMMBEM_ECUDA 2
#define FMMBEM_EINTERNAL 3

typedef struct fmmbem_plan fmmbem_plan;
typedef struct fmmbem_op fmmbem_op;

/* Formulation enum values (bemop.py:33-40). */
#define FMMBEM_LAPLACE_FIRST 0
#define FMMBEM_LAPLACE_SECOND 1
#define FMMBEM_STOKES 2

const char* fmmbem_last_error(void);
int fmmbem_version(void);
/* number of visible CUDA devices (0 on a CPU-only host; never an error) */
int fmmbem_device_count(int* count);
/* measured sm_100a DFMA throughput (TFLOP/s) of a dependent-chain microkernel */
int fmmbem_fp64_peak(int device, double* tflops);

/* ---------------------------------------------------------------- FmmPlan
 * Replaces fmm.FmmPlan.__init__ (fmm.py:131-168): shared bounding cube
 * (octree.bounding_cube, octree.py:46-54), both octrees (octree.build_tree,
 * octree.py:57-131) and the dual traversal (fmm.dual_traversal, fmm.py:84-125),
 * all built on the device.  src_xyz (ns,3), tgt_xyz (nt,3). */
int fmmbem_plan_create(const double* src_xyz, int64_t ns, const double* tgt_xyz, int64_t nt,
                       int n_crit, double theta, int max_depth, int device, fmmbem_plan** out);
int fmmbem_plan_destroy(fmmbem_plan* plan);
/* sizes[0..9] = src cells, tgt cells, src leaves, tgt leaves, m2l pairs, p2p pairs,
 *               src levels, tgt levels, p2p interactions, m2l offsets */
int fmmbem_plan_sizes(const fmmbem_plan* plan, int64_t* sizes);
/* Octree arrays of one tree (which = 0 source, 1 target), mirrors octree.Octree
 * (octree.py:6-43).  Cells are numbered level by level, Morton order inside a
 * level (the reference numbers depth-first); compare by content. Any output
 * pointer may be NULL. center (ncell,3). */
int fmmbem_plan_tree(const fmmbem_plan* plan, int which, int64_t* perm, double* center,
                     double* half_width, int32_t* level, int32_t* parent, int64_t* body_start,
                     int64_t* body_count, uint8_t* is_leaf);
/* Interaction lists (which = 0 M2L, 1 P2P) as (n,2) int32 (source cell, target cell),
 * like FmmPlan.m2l_pairs / p2p_pairs (fmm.py:141-143). */
int fmmbem_plan_pairs(const fmmbem_plan* plan, int which, int32_t* pairs);
/* FmmPlan.far_field (parts=1, fmm.py:203-233) and/or near_field (parts=2,
 * fmm.py:356-419) of the 1/r kernel with C in {1,4,7} channels of charges (C,ns)
 * and/or dipoles (C,ns,3).  pot (C,nt) and grad (C,nt,3, may be NULL) are
 * OVERWRITTEN with the requested parts' sum (no 1/4pi). Host buffers. */
int fmmbem_plan_evaluate(fmmbem_plan* plan, const double* charges, const double* dipoles, int C,
                         int p, int want_gradient, int parts, double* pot, double* grad);

/* ---------------------------------------------------------------- single expansions
 * The reference's one-expansion API (fmm.py:36-81: Expansion, p2m, m2m, m2l, l2l, m2p, l2p
 * over harmonics.py:201-270), on the device.  Coefficients use the reference's FULL flat
 * layout idx(n, m) = n^2 + n + m, complex128 as interleaved (re, im): coeffs (C, (p+1)^2).
 * Host buffers; `device` selects the GPU.
 *   p2m:       rel (N,3) = source - center; charges (C,N) and/or dipoles (C,N,3) (NULL = absent)
 *   translate: kind 0 = m2m (d = old center - new center, fmm.py:56-59),
 *              1 = m2l (d = target center - source center, :62-65), 2 = l2l (d = new - old, :68-71)
 *   evaluate:  kind 0 = m2p (multipole_to_point), 1 = l2p (local_to_point); rel (N,3) = target -
 *              center; pot (C,N), grad (C,N,3) or NULL */
int fmmbem_expansion_p2m(const double* rel, int64_t n, const double* charges, const double* dipoles,
                         int C, int p, double* coeffs, int device);
int fmmbem_expansion_translate(int kind, const double* d, int C, int p, const double* coeffs_in,
                               double* coeffs_out, int device);
int fmmbem_expansion_evaluate(int kind, const double* coeffs, int C, int p, const double* rel,
                              int64_t n, int want_gradient, double* pot, double* grad, int device);

/* ---------------------------------------------------------------- BemOperator
 * Replaces bemop.BemOperator.__init__ (bemop.py:50-82): geometry comes from the
 * host (quadrature.quadrature_points / panel_geometry, quadrature.py:86-121, so
 * it is bit-identical to the reference), the plan, the near-pair search
 * (bemop.py:95-101) and both correction matrices (bemop.py:127-184, including
 * the polar singular integrals quadrature.py:175-247) are built on the device.
 *   panel_vertices (P,3,3), gauss_pts (P,4,3), gauss_wts (P,4) — FAR_RULE;
 *   fine_pts (P,19,3), fine_wts (P,19) — NEAR_RULE; normals (P,3); areas (P);
 *   leg_x / leg_w — n_gauss_singular Gauss-Legendre nodes on [-1,1]. */
int fmmbem_op_create(const double* panel_vertices, int64_t n_panels, const double* gauss_pts,
                     const double* gauss_wts, const double* fine_pts, const double* fine_wts,
                     const double* normals, const double* areas, const double* leg_x,
                     const double* leg_w, int n_gauss_singular, int formulation, double theta,
                     int n_crit, double mu, double near_factor, int max_depth, int device,
                     fmmbem_op** out);
int fmmbem_op_destroy(fmmbem_op* op);
/* number of unknowns n (BemOperator.shape[0], bemop.py:89-92) */
int fmmbem_op_size(const fmmbem_op* op, int64_t* n);
/* borrowed plan handle of the operator (BemOperator.plan) — do not destroy */
int fmmbem_op_plan(fmmbem_op* op, fmmbem_plan** plan);
/* BemOperator.apply(x, p) (bemop.py:272-274), host x (n) -> host y (n) */
int fmmbem_op_apply(fmmbem_op* op, const double* x, double* y, int p);
/* same with device pointers.  Stream-ordered with the caller: the op's work starts after the
 * work already queued on `stream` and `stream` waits for it on return.  stream = NULL: after
 * the legacy default stream (torch's default), and the call synchronises before returning;
 * a non-NULL stream returns without a host synchronisation (y_dev is ready in `stream` order). */
int fmmbem_op_apply_device(fmmbem_op* op, const double* x_dev, double* y_dev, int p, void* stream);
/* BemOperator.dense_apply(x) (bemop.py:276-278) */
int fmmbem_op_dense_apply(fmmbem_op* op, const double* x, double* y);
/* BemOperator.assemble_rhs(data, p, dense) (bemop.py:290-310); data (P) or (P,3) */
int fmmbem_op_assemble_rhs(fmmbem_op* op, const double* data, int p, int dense, double* b);
/* Correction CSR (which = 0 C_sys, 1 C_rhs), rows = target panels, columns ascending,
 * block = 1 (Laplace) or 9 (Stokes 3x3 row-major).  Call with NULL arrays to get
 * nnz_pairs and block; indptr (P+1), indices (nnz), data (nnz*block). */
int fmmbem_op_correction(const fmmbem_op* op, int which, int64_t* nnz_pairs, int32_t* block,
                         int64_t* indptr, int64_t* indices, double* data);
/* Progress callback of the GMRES loop, called after every iteration like the reference's
 * callback(k, residual, p) (solver.py:122-123); k is 1-based.  Return 0 to continue; a nonzero
 * return stops the solve after this iteration (the Python binding uses it to re-raise an
 * exception the callback threw).  May be NULL. */
typedef int (*fmmbem_gmres_callback)(int32_t k, double residual, int32_t p, void* user);
/* solver.solve / solver.gmres with the relaxation schedule (solver.py:20-143) on the device.
 * tol is the stop test (|g_{k+1}|/||b|| < tol, solver.py:119,124); eta drives the order
 * (RelaxationSchedule.eta, solver.py:41-47; solve() passes eta = tol, solver.py:141-143).
 * Host b (n) -> host x (n); residuals / orders (max_iter) are filled for the n_iter
 * iterations done. */
int fmmbem_op_gmres(fmmbem_op* op, const double* b, double tol, double eta, int p_initial,
                    int p_min, int relaxed, int max_iter, double* x, double* residuals,
                    int32_t* orders, int32_t* n_iter, int32_t* converged,
                    fmmbem_gmres_callback callback, void* user);
/* device-pointer GMRES (b_dev, x_dev on the op's device), stream-ordered with `stream` like
 * fmmbem_op_apply_device (NULL = legacy default stream); always returns with x_dev complete. */
int fmmbem_op_gmres_device(fmmbem_op* op, const double* b_dev, double tol, double eta,
                           int p_initial, int p_min, int relaxed, int max_iter, double* x_dev,
                           double* residuals, int32_t* orders, int32_t* n_iter,
                           int32_t* converged, fmmbem_gmres_callback callback, void* user,
                           void* stream);
/* instrumentation: enable per-stage CUDA-event timing of every apply (0/1), read
 * the accumulated milliseconds per stage [p2p, p2m+m2m, m2l, l2l, epilogue, total]
 * and the number of timed applies, reset them; use_graphs toggles CUDA graphs. */
int fmmbem_op_set_timing(fmmbem_op* op, int enable, int use_graphs);
int fmmbem_op_stage_times(fmmbem_op* op, double* ms6, int64_t* calls, int reset);
/* serial = 1 runs the near field in line with the far field instead of on its own stream
 * (every kernel then has the GPU to itself: isolated per-stage timings); default 0. */
int fmmbem_op_set_serial(fmmbem_op* op, int serial);
/* cumulative kernel launches issued by the op (graph kernel nodes included), number of
 * graph-launched applies, and the CUDA-event duration of the last fmmbem_op_gmres*
 * call (for the host variant: H2D of b .. D2H of x inclusive). */
int fmmbem_op_counters(fmmbem_op* op, int64_t* kernel_launches, int64_t* applies,
                       double* last_call_ms);

/* ---------------------------------------------------------------- multi-GPU (one process per GPU)
 * rank r owns target leaves [tleaf_bounds[r], tleaf_bounds[r+1]) and source
 * leaves [sleaf_bounds[r], sleaf_bounds[r+1]) (leaf indices in body order, bounds of length
 * world+1).  Each apply does P2M of its source leaves, an NCCL all-gather of the leaf
 * multipoles, M2L/L2L/P2P/epilogue for its target leaves and (fmmbem_op_apply) an NCCL
 * all-gather of the result.  fmmbem_op_gmres on a sharded op partitions the Krylov vectors:
 * each rank keeps its own rows, all-gathers v_k before each apply and reduces the
 * Gram-Schmidt dot products with NCCL all-reduces (CGS2); x is returned whole on every rank.  nccl_id: 128 bytes from fmmbem_nccl_unique_id on rank
 * 0, shared by the caller (e.g. torch.distributed); NULL = "virtual" shard without
 * collectives that computes only its own rows (single-GPU check of the work split). */
int fmmbem_nccl_unique_id(unsigned char* out128);
/* per-leaf work weights (which = 0 target leaves: P2P + M2L flop estimate; 1 source leaves:
 * bodies), leaf order = body order, for the host-side partitioner */
int fmmbem_op_leaf_work(const fmmbem_op* op, int which, double* w);
int fmmbem_op_shard(fmmbem_op* op, int rank, int world, const int32_t* tleaf_bounds,
                    const int32_t* sleaf_bounds, const unsigned char* nccl_id);
int fmmbem_op_unshard(fmmbem_op* op);
/* The same partition with a caller-provided HOST transport instead of NCCL: every collective
 * of the sharded apply and GMRES copies its device buffer to pinned host memory, calls the
 * callback, and copies the result back.  allgather: recv (world * count) = every rank's send
 * (count) in rank order; allreduce: buf (count) summed over ranks in place.  Return 0 on
 * success.  Used for two processes sharing one GPU (tests, with torch.distributed/gloo behind
 * the callbacks) and for transports without NCCL; the apply then runs without CUDA graphs. */
typedef int (*fmmbem_allgather_fn)(const double* send, double* recv, int64_t count, void* user);
typedef int (*fmmbem_allreduce_fn)(double* buf, int64_t count, void* user);
int fmmbem_op_shard_host(fmmbem_op* op, int rank, int world, const int32_t* tleaf_bounds,
                         const int32_t* sleaf_bounds, fmmbem_allgather_fn allgather,
                         fmmbem_allreduce_fn allreduce, void* user);

#ifdef __cplusplus
}
#endif

#endif /* FMMBEM_B200_H */
