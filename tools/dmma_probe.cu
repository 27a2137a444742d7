// Do DMMA (FP64 tensor, mma.sync m8n8k4 f64) and DFMA (FP64 SIMT) share one pipe on sm_100a?
// Times a DFMA-only loop, a DMMA-only loop and loops that interleave both; if the mixed loop
// takes ~max(parts) the two issue to different units, if ~sum they share the FP64 pipe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}

// ND DMMA and NF DFMA per unrolled step, 8 independent DMMA accumulators, 8 DFMA chains
template <int ND, int NF>
__global__ void mix(double* out, int iters, double a, double b) {
  double2 acc[8];
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i] = make_double2(threadIdx.x * 1e-3 + i, 0.0); x[i] = threadIdx.x * 1e-3 + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int k = 0; k < ND; ++k) dmma(acc[(u + k) & 7], a, b);
#pragma unroll
      for (int k = 0; k < NF; ++k) x[(u + k) & 7] = fma(x[(u + k) & 7], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y + x[i];
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF>
void run(double* out, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  mix<ND, NF><<<blocks, threads>>>(out, 16, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mix<ND, NF><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32.0;
  const double steps = (double)iters * 8;
  const double dmma_flop = warps * steps * ND * 512.0;     // 8x8x4 FMAs x 2
  const double dfma_flop = warps * 32 * steps * NF * 2.0;
  printf("ND=%d NF=%d blocks=%d threads=%d: %.3f ms  dmma %.2f TF/s  dfma %.2f TF/s  total %.2f TF/s\n", ND, NF,
         blocks, threads, best, dmma_flop / best / 1e9, dfma_flop / best / 1e9,
         (dmma_flop + dfma_flop) / best / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {4, 8}) {
    const int blocks = sms * occ, threads = 256;
    run<0, 8>(out, blocks, threads);
    run<1, 0>(out, blocks, threads);
    run<2, 0>(out, blocks, threads);
    run<1, 8>(out, blocks, threads);
    run<1, 4>(out, blocks, threads);
    run<1, 16>(out, blocks, threads);
    run<2, 8>(out, blocks, threads);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
