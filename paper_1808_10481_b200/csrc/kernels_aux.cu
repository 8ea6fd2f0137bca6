// Auxiliary device kernels: on-device exact-jet fill for separable trig data,
// z ghost mirroring for reflective walls, and the AoS <-> SoA conversions
// behind hlf_set_field / hlf_get_field.
#include "hlf_internal.cuh"

namespace hlfk {
namespace {

// field += amp * prod_ax sin_jet(1, w_ax, phase_ax, x_ax, h, m+1) (jet.cpp:65-74)
__global__ void fill_separable(const __grid_constant__ FillParams P) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(P.Nx) * P.Ny * P.Nz;
  if (tid >= total) return;
  const int ix = static_cast<int>(tid % P.Nx);
  const int64_t r = tid / P.Nx;
  const int iy = static_cast<int>(r % P.Ny);
  const int iz = static_cast<int>(r / P.Ny);
  const int idx[3] = {ix, iy, iz};
  const double pi = 3.141592653589793238462643383279502884;
  double jet[3][kMaxM + 1];
  for (int ax = 0; ax < 3; ++ax) {
    double base = ax == 0 ? P.amp : 1.0;
    const double x0 = P.x0[ax] + idx[ax] * P.h;
    for (int i = 0; i < P.n1; ++i) {
      jet[ax][i] = ax < P.d ? base * sin(P.w[ax] * x0 + P.phase[ax] + i * pi / 2.0) : (i == 0 ? base : 0.0);
      base *= P.h * P.w[ax] / static_cast<double>(i + 1);
    }
  }
  const int F = P.d == 1 ? P.n1 : (P.d == 2 ? P.n1 * P.n1 : P.n1 * P.n1 * P.n1);
  double* base = P.dst + static_cast<int64_t>(P.zoff + iz) * P.layer + static_cast<int64_t>(iy) * P.Nx + ix;
  for (int f = 0; f < F; ++f) {
    int a[3] = {0, 0, 0};
    int e = f;
    for (int ax = P.d - 1; ax >= 0; --ax) {
      a[ax] = e % P.n1;
      e /= P.n1;
    }
    double v = 1.0;
    for (int ax = P.d - 1; ax >= 0; --ax) v *= jet[ax][a[ax]];
    base[f * P.coef] += v;
  }
}

// Nodal error against separable trig data (the on-device counterpart of the
// host accessors l2_error_1d/2d, analysis.cpp:241-285, at the nodes instead of
// Gauss points): err[0] += sum over nodes of (value - exact)^2, err[1] = max
// over nodes and scaled jet coefficients of |jet - exact jet|.
__global__ void separable_error(const __grid_constant__ FillParams P) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(P.Nx) * P.Ny * P.Nz;
  double sq = 0.0, mx = 0.0;
  if (tid < total) {
    const int ix = static_cast<int>(tid % P.Nx);
    const int64_t r = tid / P.Nx;
    const int iy = static_cast<int>(r % P.Ny);
    const int iz = static_cast<int>(r / P.Ny);
    const int idx[3] = {ix, iy, iz};
    const double pi = 3.141592653589793238462643383279502884;
    double jet[3][kMaxM + 1];
    for (int ax = 0; ax < 3; ++ax) {
      double base = ax == 0 ? P.amp : 1.0;
      const double x0 = P.x0[ax] + idx[ax] * P.h;
      for (int i = 0; i < P.n1; ++i) {
        jet[ax][i] = ax < P.d ? base * sin(P.w[ax] * x0 + P.phase[ax] + i * pi / 2.0) : (i == 0 ? base : 0.0);
        base *= P.h * P.w[ax] / static_cast<double>(i + 1);
      }
    }
    const int F = P.d == 1 ? P.n1 : (P.d == 2 ? P.n1 * P.n1 : P.n1 * P.n1 * P.n1);
    const double* base = P.dst + static_cast<int64_t>(P.zoff + iz) * P.layer + static_cast<int64_t>(iy) * P.Nx + ix;
    for (int f = 0; f < F; ++f) {
      int a[3] = {0, 0, 0};
      int e = f;
      for (int ax = P.d - 1; ax >= 0; --ax) {
        a[ax] = e % P.n1;
        e /= P.n1;
      }
      double v = 1.0;
      for (int ax = P.d - 1; ax >= 0; --ax) v *= jet[ax][a[ax]];
      const double dv = base[f * P.coef] - v;
      if (f == 0) sq = dv * dv;
      mx = fmax(mx, fabs(dv));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_down_sync(0xffffffffu, sq, o);
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(P.err, sq);
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(P.err + 1), static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
}

// dst plane (coef-major [F][plane]) = sigma * (-1)^{a_z} src, a_z = last index
__global__ void mirror_layer(double* dst, const double* src, int64_t plane, int n1, int F,
                             double sigma) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= plane * F) return;
  const int f = static_cast<int>(tid / plane);
  const int az = f % n1;
  dst[tid] = (az & 1 ? -sigma : sigma) * src[tid];
}

// AoS chunk [count][F] for nodes node0.. (x-major: iz fastest) <-> SoA field
template <bool TO_SOA>
__global__ void aos_soa(const double* __restrict__ in, double* __restrict__ out, int64_t node0,
                        int64_t count, int F, int Nx, int Ny, int Nz, int64_t layer, int64_t coef,
                        int zoff) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= count * F) return;
  const int64_t local = tid / F;
  const int f = static_cast<int>(tid % F);
  const int64_t node = node0 + local;
  const int iz = static_cast<int>(node % Nz);
  const int64_t r = node / Nz;
  const int iy = static_cast<int>(r % Ny);
  const int ix = static_cast<int>(r / Ny);
  const int64_t soa = static_cast<int64_t>(zoff + iz) * layer + f * coef + static_cast<int64_t>(iy) * Nx + ix;
  if (TO_SOA) out[soa] = in[tid];
  else out[tid] = in[soa];
}

unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

int launch_error(const FillParams& p, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(p.Nx) * p.Ny * p.Nz;
  if (total == 0) return 0;
  separable_error<<<blocks_for(total, 128), 128, 0, st>>>(p);
  return 1;
}

int launch_fill(const FillParams& p, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(p.Nx) * p.Ny * p.Nz;
  if (total == 0) return 0;
  fill_separable<<<blocks_for(total, 128), 128, 0, st>>>(p);
  return 1;
}

int launch_mirror_layer(double* dst, const double* src, int64_t plane, int n1, int d, double sigma,
                        cudaStream_t st) {
  const int F = d == 1 ? n1 : (d == 2 ? n1 * n1 : n1 * n1 * n1);
  mirror_layer<<<blocks_for(plane * F, 256), 256, 0, st>>>(dst, src, plane, n1, F, sigma);
  return 1;
}

int launch_aos_to_soa(const double* aos, double* field, int64_t node0, int64_t count, int F, int Nx,
                      int Ny, int Nz, int64_t layer, int64_t coef, int zoff, cudaStream_t st) {
  if (count == 0) return 0;
  aos_soa<true><<<blocks_for(count * F, 256), 256, 0, st>>>(aos, field, node0, count, F, Nx, Ny, Nz,
                                                             layer, coef, zoff);
  return 1;
}

int launch_soa_to_aos(const double* field, double* aos, int64_t node0, int64_t count, int F, int Nx,
                      int Ny, int Nz, int64_t layer, int64_t coef, int zoff, cudaStream_t st) {
  if (count == 0) return 0;
  aos_soa<false><<<blocks_for(count * F, 256), 256, 0, st>>>(field, aos, node0, count, F, Nx, Ny, Nz,
                                                              layer, coef, zoff);
  return 1;
}

}  // namespace hlfk
