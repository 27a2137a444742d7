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
  // MODE 5: the production mapping, nsl = Grt target slots, G = 256 / nsl groups, g = tid / nsl
  const int G = MODE == 4 ? Grt : MODE == 5 ? (int)blockDim.x / Grt : 8;
  const int g = MODE == 5 ? (int)threadIdx.x / Grt : (int)threadIdx.x % G;
  if (g >= G) return;
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
        else if (MODE == 6) {
          // fp32 seed on the XU: d2 -> float by bit surgery (integer pipe), MUFU.RSQ, back
          const int fb = __funnelshift_l(__double2loint(d2), __double2hiint(d2), 3) - (896 << 23);
          float yf;
          asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(__int_as_float(fb)));
          const int yb = __float_as_int(yf);
          y = __hiloint2double((yb >> 3) + (896 << 20), yb << 29);
        } else asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d2));
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
  // 8 independent chains y <- rsqrt(y + 1) (one DADD per MUFU, so the DP pipe is not the limit)
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = 1.0 + threadIdx.x + q;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[q]));
      x[q] = y + 1.0;
    }
  }
  double a = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) a += x[q];
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
    printf("{\"rsq64h_per_clk_per_sm\": %.2f, \"ms\": %.3f}\n", n / (ms * 1e-3) / (sms * clk * 1e9), ms);
  }
  for (int c : {1, 3}) run<4, 0>(src, out, sms, 256, c, clk);
  for (int c : {1, 3}) run<4, 1>(src, out, sms, 256, c, clk);
  for (int c : {1, 3}) run<4, 4>(src, out, sms, 256, c, clk);
  for (int c : {1, 3}) run<4, 6>(src, out, sms, 256, c, clk);
  for (int nsl : {19, 32, 64}) {
    printf("nsl %d: ", nsl);
    // (run<> prints one line)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 1, reps = 16;
    lapd_loop<4, 5><<<blocks, 256>>>(src, 1, out, nsl, NSRC);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    lapd_loop<4, 5><<<blocks, 256>>>(src, reps, out, nsl, NSRC);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const int G = 256 / nsl;
    const double inter = (double)blocks * G * nsl * 4 * ((NSRC + G - 1) / G) * reps;
    printf("{\"mode\": 5, \"nsl\": %d, \"dp_pipe_frac_active_threads\": %.3f}\n", nsl,
           inter * 13.0 / (ms * 1e-3) / (sms * 64.0 * clk * 1e9));
  }
  return 0;
}
