// FP64 roofline denominator: sustained DFMA and DMMA (mma.sync.m8n8k4.f64)
// throughput on this B200, measured with CUDA events over a multi-second loop.
// MEASURED_PEAKS.json has no FP64 figure; bench.py reads
// the JSON this prints (profiles/fp64_peak.json).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  // DFMA
  int iters = 1 << 16;
  dfma_loop<8><<<blocks, threads>>>(out, 1000, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  double best = 0, sustained = 0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * 8 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
    sustained = tf;
  }
  // DMMA
  double dbest = 0;
  int diters = 1 << 14;
  dmma_loop<<<blocks, threads>>>(out, 100);
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, diters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per warp per mma: 8*8*4 MACs = 512 flop
    double tf = 512.0 * 4 * (double)diters * blocks * (threads / 32) / (ms * 1e-3) / 1e12;
    if (tf > dbest) dbest = tf;
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"dfma_tflops_best\": %.3f, \"dfma_tflops_last\": %.3f, \"dmma_tflops_best\": %.3f, \"err\": \"%s\"}\n",
         sms, best, sustained, dbest, cudaGetErrorString(err));
  return 0;
}
