// Sustained FP64 peak: the DFMA loop of fp64_peak.cu launched back to back
// for ~6 s (CUDA events around the whole run), the FP64 analogue of the
// driver's "bf16_tflops_sustained" (MEASURED_PEAKS.json: matmuls back to back
// for 4 s).  A kernel timed inside a long step runs under the same power cap,
// so this is the denominator for the step-level FP64 fraction beside the
// burst figure (profiles/fp64_peak.json).  Run it with nvidia-smi sampling
// the SM clock (tools/fp64_sustained.sh).
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

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 17;
  const double flop = 2.0 * 8 * (double)iters * blocks * threads;
  cudaEvent_t e0, e1, a0, a1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&a0);
  cudaEventCreate(&a1);
  dfma_loop<8><<<blocks, threads>>>(out, 1000, 1.0000001, 1e-7);
  cudaDeviceSynchronize();
  // one launch alone (burst)
  cudaEventRecord(a0);
  dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
  cudaEventRecord(a1);
  cudaEventSynchronize(a1);
  float ms1;
  cudaEventElapsedTime(&ms1, a0, a1);
  const int reps = static_cast<int>(6000.0 / ms1) + 1;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"dfma_tflops_burst\": %.3f, \"dfma_tflops_sustained\": %.3f, \"seconds\": %.2f, \"launches\": %d, "
         "\"err\": \"%s\"}\n",
         sms, flop / (ms1 * 1e-3) / 1e12, flop * reps / (ms * 1e-3) / 1e12, ms * 1e-3, reps, cudaGetErrorString(err));
  return 0;
}
