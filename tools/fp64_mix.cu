// Do DFMA (FP64 vector pipe) and DMMA (mma.sync m8n8k4 f64) share hardware on
// B200?  Warps 0..W/2-1 run DFMA chains, the rest DMMA; compare the combined
// rate with each alone.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_work(double* out, int iters) {
  double x[8];
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], 1.0000001, 1e-7);
  double s = 0;
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
__device__ __forceinline__ void dmma_work(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}
// mode 0: all DFMA, 1: all DMMA, 2: half/half
__global__ void mix(double* out, int mode, int it_f, int it_m) {
  const int w = threadIdx.x >> 5;
  const bool do_m = mode == 1 || (mode == 2 && (w & 1));
  if (do_m) dmma_work(out, it_m); else dfma_work(out, it_f);
}
int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 512;
  const int it_f = 1 << 15, it_m = 1 << 13;
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<blocks, threads>>>(out, mode, 100, 100);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      mix<<<blocks, threads>>>(out, mode, it_f, it_m);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double warps = (double)blocks * threads / 32;
    double wf = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0);
    double wm = mode == 1 ? warps : (mode == 2 ? warps / 2 : 0);
    double flops = wf * 32 * 8.0 * it_f * 2 + wm * 4.0 * it_m * 512;
    printf("{\"mode\": %d, \"ms\": %.3f, \"tflops\": %.2f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f}\n", mode, best,
           flops / (best * 1e-3) / 1e12, wf * 32 * 8.0 * it_f * 2 / (best * 1e-3) / 1e12, wm * 4.0 * it_m * 512 / (best * 1e-3) / 1e12);
  }
  return 0;
}
