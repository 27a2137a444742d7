// FP64 peak probe for B200 (sm_100a): DFMA throughput, and the cost of the
// fp64 reciprocal-square-root variants the P2P kernel can use.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
__global__ void rsqrt_loop(double* out, int iters) {
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  double v0 = 1.0 + threadIdx.x * 1e-6, v1 = v0 + 0.25, v2 = v0 + 0.5, v3 = v0 + 0.75;
  for (int i = 0; i < iters; ++i) {
    double r0, r1, r2, r3;
    if (MODE == 0) { r0 = rsqrt(v0); r1 = rsqrt(v1); r2 = rsqrt(v2); r3 = rsqrt(v3); }
    else if (MODE == 1) { r0 = 1.0 / sqrt(v0); r1 = 1.0 / sqrt(v1); r2 = 1.0 / sqrt(v2); r3 = 1.0 / sqrt(v3); }
    else {
      // float seed + 2 Newton steps in fp64
      double vv[4] = {v0, v1, v2, v3}; double rr[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double y = (double)rsqrtf((float)vv[k]);
        double h = fma(-vv[k] * y, y, 1.0); y = fma(y * h, 0.5 + 0.375 * h, y);
        h = fma(-vv[k] * y, y, 1.0); y = fma(y * 0.5, h, y);
        rr[k] = y;
      }
      r0 = rr[0]; r1 = rr[1]; r2 = rr[2]; r3 = rr[3];
    }
    acc0 += r0; acc1 += r1; acc2 += r2; acc3 += r3;
    v0 += 1e-9; v1 += 1e-9; v2 += 1e-9; v3 += 1e-9;
  }
  double s = acc0 + acc1 + acc2 + acc3;
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d", prop.name, prop.multiProcessorCount, clk);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  dfma_chain<<<blocks, threads>>>(out, 64, 1.0000001, 1e-7); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); dfma_chain<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf(", \"dfma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  const char* names[3] = {"rsqrt_builtin", "one_over_sqrt", "f32seed_newton2"};
  for (int mode = 0; mode < 3; ++mode) {
    float bm = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      if (mode == 0) rsqrt_loop<0><<<blocks, threads>>>(out, 1024);
      if (mode == 1) rsqrt_loop<1><<<blocks, threads>>>(out, 1024);
      if (mode == 2) rsqrt_loop<2><<<blocks, threads>>>(out, 1024);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < bm) bm = ms;
    }
    double n = 4.0 * 1024 * blocks * threads;
    printf(", \"%s_grsqrt_per_s\": %.4e", names[mode], n / (bm * 1e-3) / 1e9);
  }
  printf("}\n");
  return 0;
}
