// Shared device/host helpers for the B200 FMM-BEM hot path.
//
// Coefficient storage convention (differs from the reference on purpose):
// the reference keeps all (p+1)^2 complex coefficients per expansion in the
// flat n^2+n+m layout (harmonics.py:30-35).  Sources and densities are real,
// so M_n^{-m} = (-1)^m conj(M_n^m) (harmonics.py:56-58) and the same holds for
// local expansions and for R / I.  Here every expansion stores only m >= 0:
// index hidx(n, m) = n(n+1)/2 + m, count hcount(p) = (p+1)(p+2)/2, which halves
// memory traffic and M2L work.  Negative orders are reconstructed on the fly.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace fmmbem {

constexpr int P_MAX = 20;             // largest expansion order served (RHS uses 18)
constexpr int MAX_DEPTH_LIMIT = 21;   // 3 bits per level in a 64-bit key

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgumentError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

#define FMM_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t err__ = (call);                                                          \
    if (err__ != cudaSuccess)                                                            \
      throw ::fmmbem::CudaFailure(std::string(#call) + ": " + cudaGetErrorString(err__) + \
                                  " (" __FILE__ ":" + std::to_string(__LINE__) + ")");   \
  } while (0)

#define FMM_LAUNCH_CHECK() FMM_CUDA(cudaGetLastError())

// Programmatic dependent launch: a kernel launched with launch_pdl may start while the
// previous kernel on its stream drains; it must call pdl_wait() before reading that
// kernel's output (a no-op when launched normally).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FMMBEM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  FMM_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Per-device one-time setup (constant-memory tables, kernel attributes): both belong to the
// CURRENT device, so a process that drives several devices must redo them on each one.
//   static DeviceOnce once;  if (once.first()) { ...; once.mark(); }
struct DeviceOnce {
  unsigned long long mask = 0;  // bit d: done on device d
  bool first() const {
    int dev = 0;
    FMM_CUDA(cudaGetDevice(&dev));
    return !(__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & (1ull << (dev & 63)));
  }
  void mark() {
    int dev = 0;
    FMM_CUDA(cudaGetDevice(&dev));
    __atomic_fetch_or(&mask, 1ull << (dev & 63), __ATOMIC_RELEASE);
  }
};

#define FMM_REQUIRE(cond, msg)                  \
  do {                                          \
    if (!(cond)) throw ::fmmbem::ArgumentError(msg); \
  } while (0)

__host__ __device__ constexpr int hidx(int n, int m) { return n * (n + 1) / 2 + m; }
__host__ __device__ constexpr int hcount(int p) { return (p + 1) * (p + 2) / 2; }

// ---------------------------------------------------------------- complex on double2
__device__ __forceinline__ double2 cmake(double re, double im) { return make_double2(re, im); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a * b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc + a * conj(b)
__device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y);
  acc.y = fma(-a.x, b.y, acc.y);
  return acc;
}

// Full flat storage of operator tables (I grids, R grids): entry (N, c) at
// N^2 + N + c, prefix-compatible in N.
__host__ __device__ __forceinline__ int pidx(int N, int col) { return N * N + N + col; }
__host__ __device__ __forceinline__ int tab_size(int order) { return (order + 1) * (order + 1); }

// value of a half-stored real-symmetric expansion at (n, m), any sign of m
__device__ __forceinline__ double2 hget(const double2* c, int n, int m) {
  if (m >= 0) return c[hidx(n, m)];
  double2 v = c[hidx(n, -m)];
  return (m & 1) ? make_double2(-v.x, v.y) : make_double2(v.x, -v.y);
}

// ------------------------------------------------ solid harmonics (harmonics.py:38-85)
// Reciprocal table (device, read through the read-only cache) replacing the
// fp64 divisions of the recurrences: rec[n*(P_MAX+1)+m] = 1/((n+m)(n-m)) for
// n >= m+2, and rec[REC_DIAG+m] = -1/(2m) for m >= 1.
constexpr int REC_DIAG = (P_MAX + 1) * (P_MAX + 1);
constexpr int REC_SIZE = REC_DIAG + P_MAX + 1;
inline std::vector<double> make_recip_table() {
  std::vector<double> t(REC_SIZE, 0.0);
  for (int n = 0; n <= P_MAX; ++n)
    for (int m = 0; m + 2 <= n; ++m) t[n * (P_MAX + 1) + m] = 1.0 / (double)((n + m) * (n - m));
  for (int m = 1; m <= P_MAX; ++m) t[REC_DIAG + m] = -1.0 / (2.0 * m);
  return t;
}

// Regular R_n^m(r) = rho^n P_n^m e^{im b}/(n+m)!, m >= 0, n <= p, into out[hidx].
__device__ inline void regular_half(double x, double y, double z, int p, double2* out,
                                    const double* __restrict__ rec) {
  const double rho2 = x * x + y * y + z * z;
  double2 diag = make_double2(1.0, 0.0);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) {
      // R_m^m = -(x + i y) / (2m) * R_{m-1}^{m-1}
      diag = cscale(cmul(make_double2(x, y), diag), __ldg(rec + REC_DIAG + m));
    }
    out[hidx(m, m)] = diag;
    if (m + 1 <= p) {
      double2 prev2 = diag;
      double2 prev1 = cscale(diag, z);
      out[hidx(m + 1, m)] = prev1;
      for (int n = m + 2; n <= p; ++n) {
        const double inv = __ldg(rec + n * (P_MAX + 1) + m);
        double2 cur;
        cur.x = ((2 * n - 1) * z * prev1.x - rho2 * prev2.x) * inv;
        cur.y = ((2 * n - 1) * z * prev1.y - rho2 * prev2.y) * inv;
        out[hidx(n, m)] = cur;
        prev2 = prev1;
        prev1 = cur;
      }
    }
  }
}

// Same values as regular_half, but only the columns m = m0, m0 + mstep, ...
// (several threads cooperate on one point; the sectoral chain is cheap).
__device__ inline void regular_half_cols(double x, double y, double z, int p, double2* out,
                                         int m0, int mstep, const double* __restrict__ rec) {
  const double rho2 = x * x + y * y + z * z;
  double2 diag = make_double2(1.0, 0.0);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) diag = cscale(cmul(make_double2(x, y), diag), __ldg(rec + REC_DIAG + m));
    if (m < m0 || (m - m0) % mstep) continue;
    out[hidx(m, m)] = diag;
    if (m + 1 <= p) {
      double2 prev2 = diag;
      double2 prev1 = cscale(diag, z);
      out[hidx(m + 1, m)] = prev1;
      for (int n = m + 2; n <= p; ++n) {
        const double inv = __ldg(rec + n * (P_MAX + 1) + m);
        double2 cur;
        cur.x = ((2 * n - 1) * z * prev1.x - rho2 * prev2.x) * inv;
        cur.y = ((2 * n - 1) * z * prev1.y - rho2 * prev2.y) * inv;
        out[hidx(n, m)] = cur;
        prev2 = prev1;
        prev1 = cur;
      }
    }
  }
}

// Irregular I_n^m(r) = (n-m)! P_n^m e^{im b} / rho^(n+1), m >= 0, n <= p.
__device__ inline void irregular_half(double x, double y, double z, int p, double2* out) {
  const double rho2 = x * x + y * y + z * z;
  const double inv_r2 = 1.0 / rho2;
  double2 diag = make_double2(1.0 / sqrt(rho2), 0.0);
  for (int m = 0; m <= p; ++m) {
    if (m > 0) {
      // I_m^m = -(2m-1)(x + i y)/rho^2 * I_{m-1}^{m-1}
      const double s = -(2.0 * m - 1.0) * inv_r2;
      diag = cscale(cmul(make_double2(x, y), diag), s);
    }
    out[hidx(m, m)] = diag;
    if (m + 1 <= p) {
      double2 prev2 = diag;
      double2 prev1 = cscale(diag, (2.0 * m + 1.0) * z * inv_r2);
      out[hidx(m + 1, m)] = prev1;
      for (int n = m + 2; n <= p; ++n) {
        const double a = (2 * n - 1) * z;
        const double b = (double)((n - 1) * (n - 1) - m * m);
        double2 cur;
        cur.x = (a * prev1.x - b * prev2.x) * inv_r2;
        cur.y = (a * prev1.y - b * prev2.y) * inv_r2;
        out[hidx(n, m)] = cur;
        prev2 = prev1;
        prev1 = cur;
      }
    }
  }
}

// ---------------------------------------------------------------- bulk async copies (TMA)
// mbarrier + cp.async.bulk helpers (sm_90+): one thread arms the barrier with the byte count and
// issues the copies; every consumer polls the barrier's phase.
__device__ __forceinline__ void tma_bar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void tma_bar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_bar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "TMAW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TMAW_%=;\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}
// global -> shared, 16-byte aligned, a multiple of 16 bytes; completes on the mbarrier
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
// generic-proxy reads of a shared buffer are ordered before the async-proxy writes that refill it
__device__ __forceinline__ void tma_fence_proxy() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------- device buffer
template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr_(o.ptr_), n_(o.n_) { o.ptr_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); ptr_ = o.ptr_; n_ = o.n_; o.ptr_ = nullptr; o.n_ = 0; }
    return *this;
  }
  void resize(size_t n) {
    if (n == n_) return;
    release();
    if (n) FMM_CUDA(cudaMalloc(&ptr_, n * sizeof(T)));
    n_ = n;
  }
  void ensure(size_t n) { if (n > n_) resize(n); }
  void release() {
    if (ptr_) cudaFree(ptr_);
    ptr_ = nullptr;
    n_ = 0;
  }
  void zero(cudaStream_t s = 0) { if (n_) FMM_CUDA(cudaMemsetAsync(ptr_, 0, n_ * sizeof(T), s)); }
  void upload(const T* h, size_t n, cudaStream_t s = 0) {
    resize(n);
    if (n) FMM_CUDA(cudaMemcpyAsync(ptr_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s = 0) { upload(v.data(), v.size(), s); }
  // grow-only variants for reused workspaces: the first n elements are (re)written
  void put(const T* h, size_t n, cudaStream_t s = 0) {
    ensure(n);
    if (n) FMM_CUDA(cudaMemcpyAsync(ptr_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void zero_n(size_t n, cudaStream_t s = 0) {
    ensure(n);
    if (n) FMM_CUDA(cudaMemsetAsync(ptr_, 0, n * sizeof(T), s));
  }
  std::vector<T> download(cudaStream_t s = 0) const {
    std::vector<T> h(n_);
    if (n_) {
      FMM_CUDA(cudaMemcpyAsync(h.data(), ptr_, n_ * sizeof(T), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
    }
    return h;
  }
  T* get() const { return ptr_; }
  size_t size() const { return n_; }

 private:
  T* ptr_ = nullptr;
  size_t n_ = 0;
};

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }

}  // namespace fmmbem
