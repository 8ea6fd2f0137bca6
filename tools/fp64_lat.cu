// DFMA latency and the ILP x warps needed to saturate the FP64 pipe on B200.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void chain(double* out, int iters, long long* cyc) {
  double x[ILP];
  for (int c = 0; c < ILP; ++c) x[c] = threadIdx.x * 1e-9 + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < ILP; ++c) x[c] = fma(x[c], 1.0000001, 1e-7);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < ILP; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMallocManaged(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  // latency: one warp, ILP 1
  chain<1><<<1, 32>>>(out, iters, cyc); cudaDeviceSynchronize();
  printf("{\"dfma_latency_cycles\": %.2f,\n", (double)cyc[0] / iters);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 1; warps <= 8; warps *= 2) {
#define RUN(ILP) { chain<ILP><<<sms, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize(); \
      cudaEventRecord(e0); chain<ILP><<<sms, warps * 32>>>(out, iters, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1); \
      float ms; cudaEventElapsedTime(&ms, e0, e1); \
      printf(" \"w%d_ilp%d_tflops\": %.2f,\n", warps, ILP, 2.0 * ILP * iters * sms * warps * 32 / (ms * 1e-3) / 1e12); }
    RUN(1) RUN(2) RUN(4) RUN(8)
  }
  printf(" \"end\": 0}\n");
  return 0;
}
