// Micro-benchmark: per-SM read/write throughput of tensor memory (tcgen05.ld /
// tcgen05.st, 32x32b shape = per-lane private rows) against shared memory
// LDS.64, and whether the two paths add up when mixed.  One CTA of 8 warps per
// SM (the tiled3d kernel's shape).  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tmem_bw tools/tmem_bw.cu
// Prints one JSON line per mode: bytes per SM-cycle at the measured clock.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a));
}
__device__ __forceinline__ void tm_st8(uint32_t a, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// mode 0: TMEM read, 1: LDS.64 read, 2: half/half mixed, 3: TMEM write,
// 4: warps 0-3 TMEM read / warps 4-7 LDS.64 read
__global__ void __launch_bounds__(256, 1) bw(int iters, int mode, unsigned* out) {
  __shared__ uint32_t taddr_s;
  extern __shared__ double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        static_cast<unsigned>(__cvta_generic_to_shared(&taddr_s))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  for (int i = tid; i < 8 * 32 * 64; i += 256) sm[i] = i * 0.5;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s + ((32u * (warp & 3)) << 16) + (warp >= 4 ? 256u : 0u);
  uint32_t r[8];
  for (int j = 0; j < 8; ++j) r[j] = tid * 8 + j;
  for (int c = 0; c < 16; ++c) tm_st8(base + c * 8, r);
  tm_wait_st();
  unsigned acc = 0;
  const double* sp = sm + warp * 32 * 64 + lane;
  double dacc = 0.0;
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        uint32_t a[8], b[8];
        tm_ld8(base + c * 8, a);
        tm_ld8(base + c * 8 + 8, b);
        tm_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) acc ^= a[j] + b[j];
      }
    } else if (mode == 1) {
#pragma unroll
      for (int c = 0; c < 64; ++c) dacc += sp[c * 32];
    } else if (mode == 2) {
#pragma unroll
      for (int c = 0; c < 8; c += 2) {
        uint32_t a[8], b[8];
        tm_ld8(base + c * 8, a);
        tm_ld8(base + c * 8 + 8, b);
        tm_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) acc ^= a[j] + b[j];
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) dacc += sp[c * 32];
    } else if (mode == 4) {
      // warps 0-3 read TMEM, warps 4-7 read shared memory (same bytes as modes 0/1 per warp)
      if (warp < 4) {
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          uint32_t a[8], b[8];
          tm_ld8(base + c * 8, a);
          tm_ld8(base + c * 8 + 8, b);
          tm_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) acc ^= a[j] + b[j];
        }
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) dacc += sp[c * 32];
      }
    } else {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        r[c & 7] += it;
        tm_st8(base + c * 8, r);
      }
      tm_wait_st();
    }
  }
  if (acc == 0x12345u && dacc == -1.0) out[0] = acc;  // keep the loads alive
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr_s));
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
  unsigned* out;
  cudaMalloc(&out, 4);
  const size_t smem = 8 * 32 * 64 * sizeof(double);
  cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const char* names[5] = {"tmem_ld", "lds64", "mixed_half_half", "tmem_st", "split_warps"};
  const int iters = 20000;
  for (int mode = 0; mode < 5; ++mode) {
    bw<<<sms, 256, smem>>>(100, mode, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bw<<<sms, 256, smem>>>(iters, mode, out);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // bytes per iteration per CTA: 8 warps x 32 lanes x 64 words (TMEM 4 B words = 16 cols x 8 = 128 cols? no: 16 x8 = 128 32-bit cols)
    double bytes_it = (mode == 1 || mode == 2) ? 8.0 * 32 * 64 * 8 : 8.0 * 32 * 128 * 4;
    if (mode == 2) bytes_it = 8.0 * 32 * (64 * 4 + 32 * 8);
    if (mode == 4) bytes_it = 4.0 * 32 * (128 * 4 + 64 * 8);
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("{\"mode\": \"%s\", \"err\": \"%s\", \"ms\": %.3f, \"bytes_per_sm_cycle_at_base_clock\": %.1f}\n", names[mode],
           cudaGetErrorString(err), ms, bytes_it * iters / cycles);
  }
  return 0;
}
