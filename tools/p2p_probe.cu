// Microbenchmark of the double-layer P2P inner loop (expanded form, 13 DP
// instructions per interaction) on synthetic shared-memory sources: how close
// to the FP64 pipe the loop runs as a function of targets per thread (TPT) and
// resident warps, with no staging, barriers or tail.  Also DFMA / MUFU.RSQ64H
// latencies.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe tools/p2p_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int NSRC = 512;

// MODE 0: production loop; 1: no self mask; 2: fp32 seed (F2F + MUFU.RSQ + F2F) instead of
// MUFU.RSQ64H; 3: no mask, seed = rsqrt of the previous source's d2 (no MUFU in the chain)
template <int TPT, int MODE = 0>
__global__ void lapd_loop(const double2* __restrict__ src, int reps, double* out, int Grt = 8, int nsrt = NSRC) {
  __shared__ double2 sh[4 * NSRC];
  for (int i = threadIdx.x; i < 4 * NSRC; i += blockDim.x) sh[i] = src[i];
  __syncthreads();
  double tx[TPT], ty[TPT], tz[TPT], tt[TPT], acc[TPT];
  int self[TPT];
#pragma unroll
  for (int q = 0; q < TPT; ++q) {
    tx[q] = 0.01 * (threadIdx.x + q);
    ty[q] = 0.02 - 1e-4 * q;
    tz[q] = 0.03 + 1e-5 * threadIdx.x;
    tt[q] = tx[q] * tx[q] + ty[q] * ty[q] + tz[q] * tz[q];
    acc[q] = 0.0;
    self[q] = (threadIdx.x * 7 + q) % NSRC;
  }
  const int G = MODE == 4 ? Grt : 8, g = threadIdx.x % G;  // lanes of a warp read 8 distinct sources
  const int nsl = MODE == 4 ? nsrt : NSRC;
  for (int r = 0; r < reps; ++r) {
    for (int j = g; j < nsl; j += G) {
      const double2 ab = sh[j], cs = sh[NSRC + j], dxy = sh[2 * NSRC + j], dzs = sh[3 * NSRC + j];
#pragma unroll
      for (int q = 0; q < TPT; ++q) {
        double d2 = fma(tx[q], ab.x, fma(ty[q], ab.y, fma(tz[q], cs.x, cs.y + tt[q])));
        if (MODE == 0 || MODE == 2)
          d2 = __hiloint2double(j == self[q] ? 0x7E37E43C : __double2hiint(d2), __double2loint(d2));
        double y;
        if (MODE == 2) y = (double)rsqrtf((float)d2);
        else asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d2));
        const double y2 = y * y;
        const double y3 = y2 * y;
        const double e = fma(-d2, y2, 1.0);
        const double rn = fma(dxy.x, tx[q], fma(dxy.y, ty[q], fma(dzs.x, tz[q], dzs.y)));
        acc[q] = fma(rn, fma(1.5 * e, y3, y3), acc[q]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < TPT; ++q) s += acc[q];
  if (s == 1.2345) out[0] = s;
}

__global__ void dfma_lat(double* out, int n, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / n; out[1] = x; }
}

__global__ void mufu_lat(double* out, int n) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y + 1.0;  // DADD in the chain
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (double)(t1 - t0) / n; out[1] = x; }
}

__global__ void mufu_tput(double* out, int n) {
  double x0 = 1.0 + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  double a = 0;
  for (int i = 0; i < n; ++i) {
    double y0, y1, y2, y3, y4, y5, y6, y7;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x0));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y1) : "d"(x1));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y2) : "d"(x2));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y3) : "d"(x3));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y4) : "d"(x4));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y5) : "d"(x5));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y6) : "d"(x6));
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y7) : "d"(x7));
    a += y0 + y1 + y2 + y3 + y4 + y5 + y6 + y7;
  }
  if (a == 1.2345) out[0] = a;
}

template <int TPT, int MODE = 0>
int run(const double2* src, double* out, int sms, int threads, int ctas_per_sm, double clk_ghz) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * ctas_per_sm, reps = 16;
  lapd_loop<TPT, MODE><<<blocks, threads>>>(src, 1, out);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    lapd_loop<TPT, MODE><<<blocks, threads>>>(src, reps, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lapd_loop<TPT, MODE>, threads, 0);
  const double inter = (double)blocks * threads * TPT * (NSRC / 8) * reps;
  const double dp = inter * 13.0;
  const double peak_dp = sms * 64.0 * clk_ghz * 1e9;
  printf("{\"mode\": %d, \"tpt\": %d, \"threads\": %d, \"ctas_per_sm\": %d, \"resident\": %d, \"ginter_per_s\": %.2f, "
         "\"alg_tflops\": %.2f, \"dp_pipe_frac\": %.3f}\n",
         MODE, TPT, threads, ctas_per_sm, occ, inter / (best * 1e-3) / 1e9, 18.0 * inter / (best * 1e-3) / 1e12,
         dp / (best * 1e-3) / peak_dp);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  double2* src;
  CK(cudaMalloc(&src, 4 * NSRC * sizeof(double2)));
  double2 h[4 * NSRC];
  for (int i = 0; i < 4 * NSRC; ++i) h[i] = make_double2(0.1 + 1e-3 * i, -0.2 + 1e-4 * i);
  for (int i = 0; i < NSRC; ++i) h[NSRC + i].y = 2.0 + 1e-3 * i;  // |s|^2 large enough for d2 > 0
  CK(cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice));
  double lat[2];
  dfma_lat<<<1, 32>>>(out, 4096, 1.0000001, 1e-9);
  CK(cudaMemcpy(lat, out, 16, cudaMemcpyDeviceToHost));
  printf("{\"dfma_latency_cycles\": %.2f}\n", lat[0]);
  mufu_lat<<<1, 32>>>(out, 4096);
  CK(cudaMemcpy(lat, out, 16, cudaMemcpyDeviceToHost));
  printf("{\"rsq64h_plus_dadd_latency_cycles\": %.2f}\n", lat[0]);
  const double clk = 1.965;
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mufu_tput<<<sms * 4, 256>>>(out, 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    mufu_tput<<<sms * 4, 256>>>(out, 2048);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double n = 8.0 * 2048 * sms * 4 * 256;
    printf("{\"rsq64h_per_clk_per_sm\": %.2f}\n", n / (ms * 1e-3) / (sms * clk * 1e9));
  }
  for (int c : {1, 3}) run<4, 0>(src, out, sms, 256, c, clk);
  for (int c : {1, 3}) run<4, 1>(src, out, sms, 256, c, clk);
  for (int c : {1, 3}) run<4, 4>(src, out, sms, 256, c, clk);
  return 0;
}
