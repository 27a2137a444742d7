// Device octree build that reproduces the reference tree bit for bit.
//
// Reference: bounding_cube (octree.py:46-54) and build_tree (octree.py:57-131).
// The reference splits a cell when count > n_crit and level < max_depth,
// assigns octant (x>cx) + 2(y>cy) + 4(z>cz) with a STRICT '>' against the
// exact cell centre, and forms child centres as c + (+-h) with h = half/2.
// Points lying exactly on a split plane (hundreds of them on the symmetric
// icospheres) must take the same branch, so instead of quantised Morton
// codes every point replays those comparisons against the same floating-point
// centres (one 3-bit digit per level), giving a 3*max_depth-bit path key.
// One stable radix sort on the key groups every cell's bodies contiguously;
// cells are then discovered level by level from digit changes, and a second
// sort on (leaf start, original index) restores the reference's
// "input order inside a leaf" body permutation (octree.py:61-63).
#include <cub/cub.cuh>

#include "plan.cuh"

namespace fmmbem {
namespace {

__device__ __forceinline__ unsigned long long order_key(double v) {
  unsigned long long b = __double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double order_val(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(b);
}

// bbox[0..2] = min (as order keys), bbox[3..5] = max
__global__ void k_bbox(const double* xyz, int64_t n, unsigned long long* bbox) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int d = 0; d < 3; ++d) {
      unsigned long long k = order_key(xyz[3 * i + d]);
      lo[d] = k < lo[d] ? k : lo[d];
      hi[d] = k > hi[d] ? k : hi[d];
    }
  }
  for (int d = 0; d < 3; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long a = __shfl_xor_sync(0xffffffffu, lo[d], o);
      unsigned long long b = __shfl_xor_sync(0xffffffffu, hi[d], o);
      lo[d] = a < lo[d] ? a : lo[d];
      hi[d] = b > hi[d] ? b : hi[d];
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&bbox[d], lo[d]);
      atomicMax(&bbox[3 + d], hi[d]);
    }
  }
}

__global__ void k_path_keys(const double* xyz, int64_t n, double cx, double cy, double cz,
                            double half, int depth, unsigned long long* keys, int* idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
  double h = half;
  unsigned long long key = 0;
  for (int l = 0; l < depth; ++l) {
    const int o = (x > cx ? 1 : 0) | (y > cy ? 2 : 0) | (z > cz ? 4 : 0);
    key = (key << 3) | (unsigned long long)o;
    h = h * 0.5;
    cx = __dadd_rn(cx, (o & 1) ? h : -h);
    cy = __dadd_rn(cy, (o & 2) ? h : -h);
    cz = __dadd_rn(cz, (o & 4) ? h : -h);
  }
  keys[i] = key;
  idx[i] = (int)i;
}

__global__ void k_classify(int a, int b, int level, int n_crit, int depth, const int* count,
                           uint8_t* is_leaf) {
  int c = a + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= b) return;
  is_leaf[c] = (count[c] > n_crit && level < depth) ? 0 : 1;
}

__global__ void k_heads(int64_t n, int level, int depth, const unsigned long long* keys,
                        int* cell_of, int* leaf_of, const int* start, const uint8_t* is_leaf,
                        int* flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell_of[i];
  int f = 0;
  if (c >= 0) {
    if (is_leaf[c]) {
      leaf_of[i] = c;
      cell_of[i] = -1;
    } else {
      const int sh = 3 * (depth - 1 - level);
      const unsigned dg = (unsigned)((keys[i] >> sh) & 7ull);
      f = (i == start[c]) || (dg != (unsigned)((keys[i - 1] >> sh) & 7ull));
    }
  }
  flag[i] = f;
}

__global__ void k_emit(int64_t n, int level, int depth, int base, const unsigned long long* keys,
                       int* cell_of, const int* flag, const int* pos, int* start, int* parent,
                       int* lev, double* cx, double* cy, double* cz, double h) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cell_of[i];
  if (c < 0) return;
  const int nc = base + pos[i] + flag[i] - 1;
  if (flag[i]) {
    const int o = (int)((keys[i] >> (3 * (depth - 1 - level))) & 7ull);
    start[nc] = (int)i;
    parent[nc] = c;
    lev[nc] = level + 1;
    // child centre = c + (+-h) exactly as octree.py:105-112
    cx[nc] = __dadd_rn(cx[c], (o & 1) ? h : -h);
    cy[nc] = __dadd_rn(cy[c], (o & 2) ? h : -h);
    cz[nc] = __dadd_rn(cz[c], (o & 4) ? h : -h);
  }
  cell_of[i] = nc;
}

__global__ void k_child_counts(int base, int nc, const int* parent, const int* start, int* count,
                               int* first_child, int* n_child) {
  int id = base + blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= base + nc) return;
  const int p = parent[id];
  const bool last = !(id + 1 < base + nc && parent[id + 1] == p);
  const int end = last ? start[p] + count[p] : start[id + 1];
  count[id] = end - start[id];
  if (id == base || parent[id - 1] != p) first_child[p] = id;
  atomicAdd(&n_child[p], 1);
}

__global__ void k_leaf_keys(int64_t n, const int* leaf_of, const int* start, const int* idx,
                            unsigned long long* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = ((unsigned long long)(unsigned)start[leaf_of[i]] << 32) | (unsigned)idx[i];
}

__global__ void k_finish_bodies(int64_t n, const unsigned long long* sorted, const double* xyz,
                                int* perm, double* px, double* py, double* pz) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int o = (int)(sorted[j] & 0xffffffffull);
  perm[j] = o;
  px[j] = xyz[3 * (int64_t)o];
  py[j] = xyz[3 * (int64_t)o + 1];
  pz[j] = xyz[3 * (int64_t)o + 2];
}

__global__ void k_leaf_heads(int64_t n, const int* leaf_of, int* flag) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  flag[j] = (j == 0 || leaf_of[j] != leaf_of[j - 1]) ? 1 : 0;
}

__global__ void k_leaf_list(int64_t n, const int* leaf_of, const int* flag, const int* pos,
                            int* leaves) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (flag[j]) leaves[pos[j]] = leaf_of[j];
}

__global__ void k_fill_half(int n, const int* lev, const double* level_half, double* half) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) half[c] = level_half[lev[c]];
}

template <typename T>
void cub_exclusive_sum(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t bytes = 0;
  FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, s));
  DevBuf<unsigned char> tmp(bytes ? bytes : 1);
  FMM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, (int)n, s));
  FMM_CUDA(cudaStreamSynchronize(s));
}

void build_one_tree(Tree& t, const double* d_xyz, int64_t n, const double root_c[3],
                    double root_half, int n_crit, int depth, cudaStream_t s) {
  const int B = 256;
  t.n_points = n;
  DevBuf<unsigned long long> keys(n), keys_sorted(n);
  DevBuf<int> idx(n), idx_sorted(n);
  k_path_keys<<<grid_for(n, B), B, 0, s>>>(d_xyz, n, root_c[0], root_c[1], root_c[2], root_half,
                                           depth, keys.get(), idx.get());
  FMM_LAUNCH_CHECK();
  {
    size_t bytes = 0;
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), keys_sorted.get(),
                                             idx.get(), idx_sorted.get(), (int)n, 0, 3 * depth, s));
    DevBuf<unsigned char> tmp(bytes ? bytes : 1);
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), keys_sorted.get(),
                                             idx.get(), idx_sorted.get(), (int)n, 0, 3 * depth, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  // capacity: cells at level l+1 <= min(n, 8 * internal_l); internal_l <= n / (n_crit + 1)
  const int64_t per_level = std::min<int64_t>(n, 8 * (n / (n_crit + 1) + 1));
  const int64_t cap = 1 + per_level * (int64_t)depth;
  DevBuf<int> start(cap), count(cap), parent(cap), lev(cap), first_child(cap), n_child(cap);
  DevBuf<uint8_t> is_leaf(cap);
  DevBuf<double> cx(cap), cy(cap), cz(cap);
  FMM_CUDA(cudaMemsetAsync(first_child.get(), 0xff, cap * sizeof(int), s));
  n_child.zero(s);
  {
    int zero = 0, neg = -1, nn = (int)n;
    FMM_CUDA(cudaMemcpyAsync(start.get(), &zero, sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(count.get(), &nn, sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(parent.get(), &neg, sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(lev.get(), &zero, sizeof(int), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(cx.get(), &root_c[0], sizeof(double), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(cy.get(), &root_c[1], sizeof(double), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaMemcpyAsync(cz.get(), &root_c[2], sizeof(double), cudaMemcpyHostToDevice, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  DevBuf<int> cell_of(n), leaf_of(n), flag(n), pos(n);
  cell_of.zero(s);
  t.level_start.assign(1, 0);
  t.level_start.push_back(1);
  t.level_half.assign(1, root_half);
  int level = 0;
  while (true) {
    const int a = t.level_start[level], b = t.level_start[level + 1];
    k_classify<<<grid_for(b - a, B), B, 0, s>>>(a, b, level, n_crit, depth, count.get(),
                                               is_leaf.get());
    k_heads<<<grid_for(n, B), B, 0, s>>>(n, level, depth, keys_sorted.get(), cell_of.get(),
                                         leaf_of.get(), start.get(), is_leaf.get(), flag.get());
    FMM_LAUNCH_CHECK();
    cub_exclusive_sum(flag.get(), pos.get(), n, s);
    int last_pos = 0, last_flag = 0;
    FMM_CUDA(cudaMemcpy(&last_pos, pos.get() + n - 1, sizeof(int), cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(&last_flag, flag.get() + n - 1, sizeof(int), cudaMemcpyDeviceToHost));
    const int nc = last_pos + last_flag;
    if (nc == 0) break;
    FMM_REQUIRE(b + (int64_t)nc <= cap, "octree capacity exceeded");
    const double h = t.level_half[level] * 0.5;
    k_emit<<<grid_for(n, B), B, 0, s>>>(n, level, depth, b, keys_sorted.get(), cell_of.get(),
                                        flag.get(), pos.get(), start.get(), parent.get(),
                                        lev.get(), cx.get(), cy.get(), cz.get(), h);
    k_child_counts<<<grid_for(nc, B), B, 0, s>>>(b, nc, parent.get(), start.get(), count.get(),
                                                first_child.get(), n_child.get());
    FMM_LAUNCH_CHECK();
    t.level_start.push_back(b + nc);
    t.level_half.push_back(h);
    ++level;
  }
  t.n_levels = level + 1;
  const int ncell = t.level_start[t.n_levels];
  t.n_cells = ncell;
  // body permutation: (leaf start, original index) => input order inside each leaf
  DevBuf<unsigned long long> k2(n), k2s(n);
  k_leaf_keys<<<grid_for(n, B), B, 0, s>>>(n, leaf_of.get(), start.get(), idx_sorted.get(),
                                           k2.get());
  {
    size_t bytes = 0;
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, k2.get(), k2s.get(), (int)n, 0, 64, s));
    DevBuf<unsigned char> tmp(bytes ? bytes : 1);
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, k2.get(), k2s.get(), (int)n, 0, 64, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  t.perm.resize(n);
  t.px.resize(n);
  t.py.resize(n);
  t.pz.resize(n);
  k_finish_bodies<<<grid_for(n, B), B, 0, s>>>(n, k2s.get(), d_xyz, t.perm.get(), t.px.get(),
                                               t.py.get(), t.pz.get());
  FMM_LAUNCH_CHECK();
  // leaf of every sorted body: the leaf segments are identical in both orders
  t.leaf_of_body.resize(n);
  FMM_CUDA(cudaMemcpyAsync(t.leaf_of_body.get(), leaf_of.get(), n * sizeof(int),
                           cudaMemcpyDeviceToDevice, s));
  k_leaf_heads<<<grid_for(n, B), B, 0, s>>>(n, leaf_of.get(), flag.get());
  cub_exclusive_sum(flag.get(), pos.get(), n, s);
  int lp = 0, lf = 0;
  FMM_CUDA(cudaMemcpy(&lp, pos.get() + n - 1, sizeof(int), cudaMemcpyDeviceToHost));
  FMM_CUDA(cudaMemcpy(&lf, flag.get() + n - 1, sizeof(int), cudaMemcpyDeviceToHost));
  t.n_leaves = lp + lf;
  t.leaves.resize(t.n_leaves);
  k_leaf_list<<<grid_for(n, B), B, 0, s>>>(n, leaf_of.get(), flag.get(), pos.get(),
                                           t.leaves.get());
  FMM_LAUNCH_CHECK();

  // compact per-cell arrays to the final cell count
  auto shrink_i = [&](DevBuf<int>& src, DevBuf<int>& dst) {
    dst.resize(ncell);
    FMM_CUDA(cudaMemcpyAsync(dst.get(), src.get(), ncell * sizeof(int), cudaMemcpyDeviceToDevice, s));
  };
  auto shrink_d = [&](DevBuf<double>& src, DevBuf<double>& dst) {
    dst.resize(ncell);
    FMM_CUDA(cudaMemcpyAsync(dst.get(), src.get(), ncell * sizeof(double), cudaMemcpyDeviceToDevice, s));
  };
  shrink_i(start, t.body_start);
  shrink_i(count, t.body_count);
  shrink_i(parent, t.parent);
  shrink_i(lev, t.level);
  shrink_i(first_child, t.first_child);
  shrink_i(n_child, t.n_child);
  shrink_d(cx, t.cx);
  shrink_d(cy, t.cy);
  shrink_d(cz, t.cz);
  t.is_leaf.resize(ncell);
  FMM_CUDA(cudaMemcpyAsync(t.is_leaf.get(), is_leaf.get(), ncell, cudaMemcpyDeviceToDevice, s));
  DevBuf<double> lh;
  lh.upload(t.level_half, s);
  t.half.resize(ncell);
  k_fill_half<<<grid_for(ncell, B), B, 0, s>>>(ncell, t.level.get(), lh.get(), t.half.get());
  FMM_LAUNCH_CHECK();
  FMM_CUDA(cudaStreamSynchronize(s));

  t.h_body_start = t.body_start.download(s);
  t.h_body_count = t.body_count.download(s);
  t.h_parent = t.parent.download(s);
  t.h_level = t.level.download(s);
  t.h_first_child = t.first_child.download(s);
  t.h_n_child = t.n_child.download(s);
  t.h_is_leaf = t.is_leaf.download(s);
  t.h_leaves = t.leaves.download(s);
  t.h_cx = t.cx.download(s);
  t.h_cy = t.cy.download(s);
  t.h_cz = t.cz.download(s);
  t.max_leaf_count = 0;
  for (int c : t.h_leaves) t.max_leaf_count = std::max(t.max_leaf_count, t.h_body_count[c]);
}

}  // namespace

void build_trees(Plan& plan, const double* src_xyz, int64_t ns, const double* tgt_xyz, int64_t nt,
                 cudaStream_t s) {
  DevBuf<double> dsrc, dtgt;
  dsrc.upload(src_xyz, 3 * ns, s);
  dtgt.upload(tgt_xyz, 3 * nt, s);
  // root cube over vstack(src, tgt) (fmm.py:135) with bounding_cube's padding
  DevBuf<unsigned long long> bbox(6);
  unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
  FMM_CUDA(cudaMemcpyAsync(bbox.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
  k_bbox<<<296, 256, 0, s>>>(dsrc.get(), ns, bbox.get());
  k_bbox<<<296, 256, 0, s>>>(dtgt.get(), nt, bbox.get());
  FMM_LAUNCH_CHECK();
  unsigned long long hb[6];
  FMM_CUDA(cudaMemcpyAsync(hb, bbox.get(), sizeof(hb), cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    unsigned long long k = hb[d];
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    memcpy(&lo[d], &b, 8);
    k = hb[3 + d];
    b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    memcpy(&hi[d], &b, 8);
  }
  // octree.py:48-54 (host code is built with -ffp-contract=off)
  double ext = 0.0;
  for (int d = 0; d < 3; ++d) {
    volatile double sum = lo[d] + hi[d];
    plan.root_c[d] = 0.5 * sum;
    volatile double e = hi[d] - lo[d];
    ext = (d == 0 || e > ext) ? e : ext;
  }
  const double pad = 1e-6;
  volatile double half = 0.5 * ext;
  volatile double scaled = half * (1.0 + pad);
  plan.root_half = scaled + pad;
  build_one_tree(plan.src, dsrc.get(), ns, plan.root_c, plan.root_half, plan.n_crit,
                 plan.max_depth, s);
  build_one_tree(plan.tgt, dtgt.get(), nt, plan.root_c, plan.root_half, plan.n_crit,
                 plan.max_depth, s);
}

}  // namespace fmmbem
