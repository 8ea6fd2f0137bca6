// Gauss-quadrature L2 error of a staggered field against separable trig data
// on the device: the counterpart of the reference's host accessors
// l2_error_1d (analysis.cpp:241-256) and l2_error_2d (:258-285), in d = 1..3.
//
// Cells are centred on the other grid's nodes (a primary-grid field: cells
// [x_j, x_j+1] around dual node j; a dual-grid field: [x_{j-1/2}, x_{j+1/2}]
// around primary node j).  Per cell the 2^d corner jets are stacked and
// reconstructed with M along every axis (reconstruct_cell_1d/2d,
// interpolation.cpp:63-113), the Hermite polynomial (scaled coefficients:
// value at offset xi h = sum_s ext[s] xi^s, jet_eval) is evaluated at the
// n-point Gauss rule of every axis (n = 2m+2, as gauss_rule(op.n)), and
// w (value - exact)^2 (h/2)^d is summed.  Accessor, not a hot path: one
// thread per cell, local arrays.
#include "hlf_internal.cuh"

namespace hlfk {
namespace {

template <int D>
__global__ void __launch_bounds__(128) l2_cells(const __grid_constant__ L2Params P) {
  constexpr int NMAX = D == 3 ? 10 : kMaxN;  // d = 3: m <= 4
  constexpr int EMAX = D == 1 ? NMAX : (D == 2 ? NMAX * NMAX : NMAX * NMAX * NMAX);
  const int n = P.n, n1 = P.n1;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(P.cells[0]) * P.cells[1] * P.cells[2];
  double acc = 0.0;
  if (tid < total) {
    int c[3];
    c[0] = static_cast<int>(tid % P.cells[0]);
    const int64_t rest = tid / P.cells[0];
    c[1] = static_cast<int>(rest % P.cells[1]);
    c[2] = static_cast<int>(rest / P.cells[1]);
    // corner node index per axis and side (wrap on periodic axes)
    int node[3][2];
    for (int ax = 0; ax < 3; ++ax)
      for (int side = 0; side < 2; ++side) {
        int q = c[ax] + side - P.shift;
        if (ax < D && P.wrap[ax]) {
          if (q < 0) q += P.cells[ax];
          if (q >= P.cells[ax]) q -= P.cells[ax];
        }
        node[ax][side] = ax < D ? q : 0;
      }
    double S[EMAX], T[EMAX];
    int stride[3] = {1, 1, 1};
    for (int ax = D - 2; ax >= 0; --ax) stride[ax] = stride[ax + 1] * n;
    const int E = D == 1 ? n : (D == 2 ? n * n : n * n * n);
    const int F = D == 1 ? n1 : (D == 2 ? n1 * n1 : n1 * n1 * n1);
    // stacked corners: index side * n1 + a per axis (x-major)
    for (int corner = 0; corner < (1 << D); ++corner) {
      const int sx = corner & 1, sy = (corner >> 1) & 1, sz = (corner >> 2) & 1;
      const int64_t nb = static_cast<int64_t>(P.zoff + node[2][sz]) * P.layer +
                         static_cast<int64_t>(node[1][sy]) * P.Nx + node[0][sx];
      for (int f = 0; f < F; ++f) {
        int a[3] = {0, 0, 0}, e = f;
        for (int ax = D - 1; ax >= 0; --ax) {
          a[ax] = e % n1;
          e /= n1;
        }
        const int side[3] = {sx, sy, sz};
        int idx = 0;
        for (int ax = 0; ax < D; ++ax) idx += (side[ax] * n1 + a[ax]) * stride[ax];
        S[idx] = P.src[nb + f * P.coef];
      }
    }
    // M along each axis (interpolation.cpp:87-112)
    for (int ax = 0; ax < D; ++ax) {
      const int st = stride[ax];
      for (int e = 0; e < E; ++e) {
        if ((e / st) % n != 0) continue;
        for (int r = 0; r < n; ++r) {
          double v = 0.0;
          for (int s = 0; s < n; ++s) v = fma(P.M[r * n + s], S[e + s * st], v);
          T[e + r * st] = v;
        }
      }
      for (int e = 0; e < E; ++e) S[e] = T[e];
    }
    // Gauss points: contract one axis at a time (x first), then the exact value
    double xc[3];
    for (int ax = 0; ax < 3; ++ax) xc[ax] = P.xc0[ax] + c[ax] * P.h;
    const double pi2 = 1.5707963267948966;
    (void)pi2;
    const int NQ = D == 1 ? n : (D == 2 ? n * n : n * n * n);
    for (int qi = 0; qi < NQ; ++qi) {
      int q[3] = {0, 0, 0}, e = qi;
      for (int ax = D - 1; ax >= 0; --ax) {
        q[ax] = e % n;
        e /= n;
      }
      // value = sum_s ext[s] prod_ax xi_ax^{s_ax}, Horner along the last axis first
      double val = 0.0;
      if (D == 1) {
        const double xi = 0.5 * P.gx[q[0]];
        for (int s = n - 1; s >= 0; --s) val = fma(val, xi, S[s]);
      } else if (D == 2) {
        const double xi = 0.5 * P.gx[q[0]], eta = 0.5 * P.gx[q[1]];
        for (int sx = n - 1; sx >= 0; --sx) {
          double row = 0.0;
          for (int sy = n - 1; sy >= 0; --sy) row = fma(row, eta, S[sx * n + sy]);
          val = fma(val, xi, row);
        }
      } else {
        const double xi = 0.5 * P.gx[q[0]], eta = 0.5 * P.gx[q[1]], zeta = 0.5 * P.gx[q[2]];
        for (int sx = n - 1; sx >= 0; --sx) {
          double pl = 0.0;
          for (int sy = n - 1; sy >= 0; --sy) {
            double row = 0.0;
            for (int sz = n - 1; sz >= 0; --sz) row = fma(row, zeta, S[(sx * n + sy) * n + sz]);
            pl = fma(pl, eta, row);
          }
          val = fma(val, xi, pl);
        }
      }
      double ex = P.amp, w = 1.0;
      for (int ax = 0; ax < D; ++ax) {
        const double x = xc[ax] + 0.5 * P.h * P.gx[q[ax]];
        ex *= sin(P.w[ax] * x + P.phase[ax]);
        w *= P.gw[q[ax]] * 0.5 * P.h;
      }
      const double diff = val - ex;
      acc = fma(w * diff, diff, acc);
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(P.out, acc);
}

// Discrete energy of the 1D leapfrog (conserved_q / conserved_r,
// analysis.cpp:221-239): E = |f - g(. + s)|^2_{m+1} + |f + g(. - s)|^2_{m+1}
// with f, g the piecewise Hermite interpolants of the two fields
// (interpolant_from_primary / _from_dual, analysis.cpp:35-86), s = c dt / 2
// and |.|_{m+1} the Sobolev seminorm of order m+1 (sobolev_seminorm).  One
// thread per cell of f: the shifted g has one breakpoint inside it (|s| < h/2),
// and each part is integrated exactly with the (m+1)-point Gauss rule (the
// integrand has degree 2m).  The reference's pw_shift / pw_combine split and
// recenter the same polynomials; this evaluates them in place.
__device__ double deriv_eval(const double* a, int n, int k, double xi, double inv_hk) {
  double v = 0.0;
  for (int i = n - 1; i >= k; --i) {
    double fac = 1.0;
    for (int q = 0; q < k; ++q) fac *= static_cast<double>(i - q);
    v = fma(v, xi, a[i] * fac);
  }
  return v * inv_hk;
}

__device__ void recon_1d(const EnergyParams& P, const double* jets, int l, int r, double* out) {
  double S[kMaxN];
  for (int a = 0; a < P.n1; ++a) {
    S[a] = jets[l + a * P.coef];
    S[P.n1 + a] = jets[r + a * P.coef];
  }
  for (int i = 0; i < P.n; ++i) {
    double v = 0.0;
    for (int q = 0; q < P.n; ++q) v = fma(P.M[i * P.n + q], S[q], v);
    out[i] = v;
  }
}

__global__ void __launch_bounds__(128) energy_1d(const __grid_constant__ EnergyParams P) {
  const int j = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (j < P.K) {
    const int K = P.K, n = P.n, k = P.n1;  // seminorm order m + 1
    const double h = P.h;
    // f cell: primary-based [x_j, x_j+1] around dual j, or dual-based
    // [x_j-1/2, x_j+1/2] around primary j; g cells left / right of its middle
    const double a0 = P.x0 + (P.f_primary ? j * h : (j - 0.5) * h);
    double fa[kMaxN], gl[kMaxN], gr[kMaxN];
    if (P.f_primary) recon_1d(P, P.f, j, (j + 1) % K, fa);
    else recon_1d(P, P.f, (j - 1 + K) % K, j, fa);
    recon_1d(P, P.g, (j - 1 + K) % K, j, gl);
    recon_1d(P, P.g, j, (j + 1) % K, gr);
    double inv_hk = 1.0;
    for (int q = 0; q < k; ++q) inv_hk /= h;
    const double cf = a0 + 0.5 * h;
    for (int sg = 0; sg < 2; ++sg) {
      const double sigma = sg == 0 ? 1.0 : -1.0;  // f - g(x + s), then f + g(x - s)
      const double bp = a0 + 0.5 * h - sigma * P.s;
      for (int part = 0; part < 2; ++part) {
        const double xl = part == 0 ? a0 : bp, xr = part == 0 ? bp : a0 + h;
        const double* gc = part == 0 ? gl : gr;
        const double cg = part == 0 ? a0 : a0 + h;
        const double half = 0.5 * (xr - xl), mid = 0.5 * (xr + xl);
        for (int q = 0; q < k; ++q) {
          const double x = mid + half * P.gx[q];
          const double df = deriv_eval(fa, n, k, (x - cf) / h, inv_hk);
          const double dg = deriv_eval(gc, n, k, (x + sigma * P.s - cg) / h, inv_hk);
          const double v = df - sigma * dg;
          acc = fma(P.gw[q] * half * v, v, acc);
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(P.out, acc);
}

}  // namespace

int launch_energy_1d(const EnergyParams& p, cudaStream_t st) {
  if (p.K <= 0) return 0;
  energy_1d<<<(p.K + 127) / 128, 128, 0, st>>>(p);
  return 1;
}

int launch_l2(const L2Params& p, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(p.cells[0]) * p.cells[1] * p.cells[2];
  if (total == 0) return 0;
  const unsigned blocks = static_cast<unsigned>((total + 127) / 128);
  switch (p.d) {
    case 1: l2_cells<1><<<blocks, 128, 0, st>>>(p); break;
    case 2: l2_cells<2><<<blocks, 128, 0, st>>>(p); break;
    case 3: l2_cells<3><<<blocks, 128, 0, st>>>(p); break;
    default: return -1;
  }
  return 1;
}

}  // namespace hlfk
