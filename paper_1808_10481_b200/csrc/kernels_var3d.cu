// 3D Hermite-leapfrog half steps with a spatially varying coefficient
// ap = -(c0 + c1 prod_ax sin(w_ax x_ax + phase_ax))  (ap = -c^2, c^2 separable),
// av a scalar, m = 1..3: the variable-coefficient CK recurrence of
// ck_recurrence_variable (stepper1d.cpp:22-38) generalised to d = 3 with
// truncated tensor products (tensor_multiply, jet.cpp:109-121).
//
// The ap jets are generated on the fly at every target node (no stored
// coefficient grids: the traffic stays the 24 B per DOF-update of the
// constant-coefficient kernels), and because the jet is
// e0 (-c0) plus an outer product (-c1 s_x (x) s_y (x) s_z), the truncated
// product ap (.) X is -c0 X - c1 S_x S_y S_z X with S_a the 1D truncated
// Cauchy product along axis a: 3 n^2 lines x n(n+1)/2 multiply-adds instead
// of the (n(n+1)/2)^3 of a general n^3 jet.
//
// One warp per target node, the node's n^3 tensors in padded shared memory
// (strides n+1 and n(n+1)+1 so that lines along every axis are bank
// friendly), lanes over lines (sweeps, products) or entries (derivatives).
// Per node, with P_r / V_r the CK tables (seed zero for the target's family):
//   pressure:  D = sum_c d_c recon(V_c);  P_1 = ap (.) D;  P_{r+2} = ap (.) (av Lap P_r)
//              p += sum_{r odd} w_r P_r           (advance_p, stepper1d.cpp:147-156)
//   velocity:  P_0 = recon(p);  V_c[r] = av d_c P_{r-1};  P_{r+1} = ap (.) (av Lap P_{r-1})
//              v_c += sum_{r odd} w_r V_c[r]      (advance_v, stepper1d.cpp:158-166)
// with d_c the truncated scaled derivative (jet_differentiate, jet.cpp:20-31)
// and Lap = sum_c d_c d_c (the two derivatives of the recurrence; av is a
// scalar).  Arithmetic is reordered against the oracle (FMA, separable
// products), so parity is at the 1e-12 bar, not bit-identical.
#include <type_traits>

#include "hlf_internal.cuh"

namespace hlfk {
namespace {

// compile-time loop: f(std::integral_constant<int, I>) for I = B .. E-1
template <int B, int E, class Fn>
__device__ __forceinline__ void static_for(Fn&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

constexpr int WARPS = 4;

template <int MM>
struct V3 {
  static constexpr int n1 = MM + 1, n = 2 * MM + 2, F = n1 * n1 * n1, E = n * n * n;
  // strides chosen by a bank-conflict search over the access patterns (lines
  // along each axis with lanes over the other two, entries with lanes over
  // z then y): 2, 4 and 2 wavefronts per 32-lane LDS.64 for x-, y- and z-lines
  // and 2 for entries at n = 8 (the first layout, SY = n+1 and SX = n(n+1)+1,
  // was 4 everywhere: ncu showed 50 % of the shared wavefronts as conflicts)
  static constexpr int SZ = 1, SY = n, SX = n * n + 1;
  static constexpr int T = n * SX;                                 // doubles per padded tensor
  static constexpr int NBUF = 3;
  static constexpr int SMEM = WARPS * NBUF * T;                    // doubles per CTA
};

template <int MM>
__device__ __forceinline__ int pidx(int qx, int qy, int qz) {
  return qx * V3<MM>::SX + qy * V3<MM>::SY + qz;
}

// line l (0 .. n^2-1) along axis ax: base offset and stride in the padded layout
template <int MM>
__device__ __forceinline__ void line_of(int ax, int l, int& base, int& stride) {
  constexpr int n = V3<MM>::n;
  const int a = l / n, b = l - (l / n) * n;
  if (ax == 0) {
    base = pidx<MM>(0, a, b);
    stride = V3<MM>::SX;
  } else if (ax == 1) {
    base = pidx<MM>(a, 0, b);
    stride = V3<MM>::SY;
  } else {
    base = pidx<MM>(b, a, 0);  // lanes run along x here (conflict-free with SX = n^2 + 1)
    stride = 1;
  }
}

// scaled jet of sin(w x + ph) at x, spacing h: s[k] = (w h)^k / k! sin(w x + ph + k pi/2) (sin_jet, jet.cpp)
template <int N>
__device__ __forceinline__ void sin_jet_dev(double w, double ph, double x, double h, double (&s)[N]) {
  double sn, cs;
  sincos(w * x + ph, &sn, &cs);
  double f = 1.0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int r = k & 3;
    s[k] = f * (r == 0 ? sn : (r == 1 ? cs : (r == 2 ? -sn : -cs)));
    f = f * (w * h) / (k + 1);
  }
}

struct V3Params {
  HalfParams hp;
  double c0, c1, w[3], ph[3];
  double x0[3];  // coordinate of target node 0 per axis
};

template <int MM, int KIND>
#ifndef HLF_V3_MINB
#define HLF_V3_MINB 2  // 8 warps per SM with the unrolled line loops beat 16 register-capped ones: 4.9 -> 7.4e9 DOF/s at 192^3 m = 3
#endif
#ifndef HLF_V3_MINB_M1
#define HLF_V3_MINB_M1 4  // m = 1: 16 warps per SM (<= 128 registers): 24.3 -> 22.9 ms/step at 192^3 (m = 2, 3: slower)
#endif
__global__ void __launch_bounds__(WARPS * 32, MM == 1 ? HLF_V3_MINB_M1 : HLF_V3_MINB) var3d(const __grid_constant__ V3Params Q) {
  using C = V3<MM>;
  constexpr int n1 = C::n1, n = C::n, F = C::F, E = C::E, T = C::T;
  constexpr int NOUT = KIND == VEL ? 3 : 1;
  constexpr int NSRC = KIND == VEL ? 1 : 3;
  constexpr int FL = (F + 31) / 32;  // output entries per lane
  const HalfParams& P = Q.hp;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* A = sm + warp * C::NBUF * T;
  double* B = A + T;
  double* Cb = B + T;
  const double inv_h = 1.0 / P.h;

  const int64_t total = static_cast<int64_t>(P.tNx) * P.tNy * P.tNz;
  const int64_t stride_nodes = static_cast<int64_t>(gridDim.x) * WARPS;
#pragma unroll 1
  for (int64_t node = static_cast<int64_t>(blockIdx.x) * WARPS + warp; node < total; node += stride_nodes) {
    int t[3];
    t[0] = static_cast<int>(node % P.tNx);
    const int64_t rest = node / P.tNx;
    t[1] = static_cast<int>(rest % P.tNy);
    t[2] = static_cast<int>(rest / P.tNy);
    const int64_t toff = static_cast<int64_t>(P.t_zoff + t[2]) * P.t_layer + static_cast<int64_t>(t[1]) * P.tNx + t[0];

    // per axis and side: the source node's offset and whether it is a wall
    // mirror (as half_generic's corner maps); a corner's address is the sum
    int64_t aoff[3][2];
    bool aflip[3][2];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        int q = KIND == VEL ? t[ax] + side : t[ax] - 1 + side;
        bool flip = false;
        if (ax < 2) {
          if (P.bnd[ax] == 0) {
            if (q >= P.K[ax]) q -= P.K[ax];
            if (q < 0) q += P.K[ax];
          } else if (KIND == PRE) {
            if (q < 0) {
              q = 0;
              flip = true;
            } else if (q >= P.K[ax]) {
              q = P.K[ax] - 1;
              flip = true;
            }
          }
        }
        aflip[ax][side] = flip;
        aoff[ax][side] = ax == 0 ? q : (ax == 1 ? static_cast<int64_t>(q) * P.sNx
                                                : static_cast<int64_t>(P.s_zoff + q) * P.s_layer);
      }

    // this node's separable ap: per-axis sin jets
    double sx[n], sy[n], sz[n];
    sin_jet_dev<n>(Q.w[0], Q.ph[0], Q.x0[0] + t[0] * P.h, P.h, sx);
    sin_jet_dev<n>(Q.w[1], Q.ph[1], Q.x0[1] + t[1] * P.h, P.h, sy);
    sin_jet_dev<n>(Q.w[2], Q.ph[2], Q.x0[2] + t[2] * P.h, P.h, sz);

    // targets of this lane's output entries
    double tgt[NOUT][FL];
#pragma unroll
    for (int c = 0; c < NOUT; ++c)
#pragma unroll
      for (int j = 0; j < FL; ++j) {
        const int f = lane + 32 * j;
        tgt[c][j] = f < F ? P.dst[c][toff + static_cast<int64_t>(f) * P.t_coef] : 0.0;
      }

    // ---- reconstruction of one source field into Cb (x, y, z sweeps of M)
    // gather of one source field's stacked corner tensor: this lane's E/32
    // entries are loaded into registers first (gather_load, issued one
    // component ahead so the loads overlap the previous component's sweeps)
    // and stored to A later (gather_store)
    constexpr int GL = (E + 31) / 32;
    auto gather_load = [&](int comp, double (&g)[GL]) {
      const double* src = P.src[comp];
#pragma unroll
      for (int j = 0; j < GL; ++j) {
        const int e = lane + 32 * j;
        if (e >= E) break;
        const int q[3] = {e / (n * n), (e / n) % n, e % n};
        int f = 0;
        int64_t off = 0;
        double sign = 1.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const int side = q[ax] >= n1, l = q[ax] - side * n1;
          f = f * n1 + l;
          off += side ? aoff[ax][1] : aoff[ax][0];
          if (side ? aflip[ax][1] : aflip[ax][0]) {
            if (l & 1) sign = -sign;
            if (comp != ax) sign = -sign;  // tangential velocity is odd across the wall
          }
        }
        g[j] = sign * __ldg(src + off + static_cast<int64_t>(f) * P.s_coef);
      }
    };
    auto gather_store = [&](const double (&g)[GL]) {
#pragma unroll
      for (int j = 0; j < GL; ++j) {
        const int e = lane + 32 * j;
        if (e >= E) break;
        A[pidx<MM>(e / (n * n), (e / n) % n, e % n)] = g[j];
      }
    };
    double gbuf[GL];
    // ---- reconstruction of the gathered field (gbuf) into Cb (x, y, z sweeps
    // of M); `next` >= 0 issues the gather of component `next` meanwhile
    auto reconstruct = [&](int next) {
      gather_store(gbuf);
      if (next >= 0) gather_load(next, gbuf);
      __syncwarp();
      double* in = A;
      double* out = Cb;
#pragma unroll 1
      for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
        for (int it = 0; it < (n * n + 31) / 32; ++it) {
          const int l = lane + 32 * it;
          if (l >= n * n) break;
          int base, st;
          line_of<MM>(ax, l, base, st);
          // parity split of M (M_R = diag((-1)^r) M_L diag((-1)^l), host-checked
          // m_mirror): out[r] = sum_l M[r][l] (L_l + (-1)^(r+l) R_l), and the
          // exact zeros M[r][0] (even r >= 2, m <= 3) skipped: 8 adds + 29
          // FMAs per line instead of 64 FMAs
          double sg[n1], df[n1];
#pragma unroll
          for (int l = 0; l < n1; ++l) {
            const double lo = in[base + l * st], hi = in[base + (n1 + l) * st];
            sg[l] = lo + hi;
            df[l] = lo - hi;
          }
#pragma unroll
          for (int r = 0; r < n; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < n1; ++l) {
              if (MM <= 3 && l == 0 && r >= 2 && (r & 1) == 0) continue;
              acc = fma(P.M[r * n + l], ((r + l) & 1) ? df[l] : sg[l], acc);
            }
            out[base + r * st] = acc;
          }
        }
        __syncwarp();
        double* tmp = in;
        in = out;
        out = tmp;
      }
      // after three sweeps the result is in A (in) -- copy pointer semantics:
      // sweeps A->Cb, Cb->A, A->Cb: the result sits in Cb
    };

    // X <- ap (.) X in place: X = -c0 X - c1 S_x S_y S_z X, with the S passes through B.
    // Only the box q <= lim (every axis) is computed: the truncated product at
    // q reads entries <= q, and the later levels and the target read no
    // entry outside the box of their level (lim from level_lim below)
    auto ap_times = [&](double* X, auto limc) {
      constexpr int lim = decltype(limc)::value;
      // z pass X -> B, y pass in B, x pass B -> X fused with -c0 X - c1 (.)
#pragma unroll
      for (int ax = 2; ax >= 0; --ax) {
        const double* s = ax == 0 ? sx : (ax == 1 ? sy : sz);  // compile-time after unrolling
        const double* in = ax == 2 ? X : B;
#pragma unroll
        for (int it = 0; it < (n * n + 31) / 32; ++it) {
          const int l = lane + 32 * it;
          if (l >= n * n) break;
          if (l / n > lim || l % n > lim) continue;  // the line's fixed coordinates
          int base, st;
          line_of<MM>(ax, l, base, st);
          double v[n];
#pragma unroll
          for (int i = 0; i < n; ++i) v[i] = i <= lim ? in[base + i * st] : 0.0;
#pragma unroll
          for (int i = n - 1; i >= 0; --i) {
            if (i > lim) continue;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j <= i; ++j) acc = fma(s[j], v[i - j], acc);
            if (ax == 0) X[base + i * st] = fma(-Q.c1, acc, -Q.c0 * X[base + i * st]);
            else B[base + i * st] = acc;
          }
        }
        __syncwarp();
      }
    };

    // Y <- av Lap X (truncated second derivatives, jet_differentiate twice per axis)
    auto av_lap = [&](const double* X, double* Y, auto limc) {
      constexpr int lim = decltype(limc)::value;
#pragma unroll 4
      for (int e = lane; e < E; e += 32) {
        const int q[3] = {e / (n * n), (e / n) % n, e % n};
        if (q[0] > lim || q[1] > lim || q[2] > lim) continue;
        double acc = 0.0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          if (q[ax] + 2 < n) {
            int r[3] = {q[0], q[1], q[2]};
            r[ax] += 2;
            acc = fma(static_cast<double>((q[ax] + 1) * (q[ax] + 2)) * inv_h * inv_h, X[pidx<MM>(r[0], r[1], r[2])], acc);
          }
        }
        Y[pidx<MM>(q[0], q[1], q[2])] = P.av * acc;
      }
      __syncwarp();
    };

    if constexpr (KIND == PRE) {
      // D = sum_c d_c recon(V_c), accumulated in B... B is the product scratch,
      // so D goes to A after the reconstructions (kept in registers meanwhile)
      double dsum[(E + 31) / 32];
#pragma unroll
      for (int j = 0; j < (E + 31) / 32; ++j) dsum[j] = 0.0;
      gather_load(0, gbuf);
#pragma unroll 1
      for (int comp = 0; comp < NSRC; ++comp) {
        reconstruct(comp + 1 < NSRC ? comp + 1 : -1);  // -> Cb (gather of comp + 1 in flight)
#pragma unroll
        for (int j = 0; j < (E + 31) / 32; ++j) {
          const int e = lane + 32 * j;
          if (e < E) {
            const int q[3] = {e / (n * n), (e / n) % n, e % n};
            if (q[comp] + 1 < n) {
              int r[3] = {q[0], q[1], q[2]};
              r[comp] += 1;
              dsum[j] = fma(static_cast<double>(q[comp] + 1) * inv_h, Cb[pidx<MM>(r[0], r[1], r[2])], dsum[j]);
            }
          }
        }
        __syncwarp();
      }
      // P_1 = ap (.) D, in A
#pragma unroll
      for (int j = 0; j < (E + 31) / 32; ++j) {
        const int e = lane + 32 * j;
        if (e < E) A[pidx<MM>(e / (n * n), (e / n) % n, e % n)] = dsum[j];
      }
      __syncwarp();
      // levels unrolled so that each level's box is a compile-time bound
      static_for<0, n / 2>([&](auto ri) {
        constexpr int r = 2 * decltype(ri)::value + 1;
        // P_r is read by the target (o <= m) and, through Lap, by P_{r+2}:
        // box q <= m + (n - 1 - r)
        constexpr int lim = (MM + (n - 1 - r)) < n - 1 ? MM + (n - 1 - r) : n - 1;
        using L = std::integral_constant<int, lim>;
        if constexpr (r > 1) {
          av_lap(A, Cb, L{});  // Cb = av Lap P_{r-2}
          double* tmp = A;
          A = Cb;
          Cb = tmp;
        }
        ap_times(A, L{});      // A = P_r
        const double w = P.w[r];
#pragma unroll
        for (int j = 0; j < FL; ++j) {
          const int f = lane + 32 * j;
          if (f < F) {
            const int o[3] = {f / (n1 * n1), (f / n1) % n1, f % n1};
            tgt[0][j] = fma(w, A[pidx<MM>(o[0], o[1], o[2])], tgt[0][j]);
          }
        }
      });
    } else {
      gather_load(0, gbuf);
      reconstruct(-1);  // P_0 in Cb
      double* Pc = Cb;
      double* Xs = A;
      static_for<0, n / 2>([&](auto ri) {
        constexpr int r = 2 * decltype(ri)::value + 1;
        // V_c[r] = av d_c P_{r-1}: this lane's output entries
        const double w = P.w[r];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int j = 0; j < FL; ++j) {
            const int f = lane + 32 * j;
            if (f < F) {
              int o[3] = {f / (n1 * n1), (f / n1) % n1, f % n1};
              const int qc = o[c];
              o[c] += 1;
              const double dv = static_cast<double>(qc + 1) * inv_h * Pc[pidx<MM>(o[0], o[1], o[2])];
              tgt[c][j] = fma(w, P.av * dv, tgt[c][j]);  // qc + 1 <= m + 1 < n: never truncated here
            }
          }
        if constexpr (r + 2 < n) {
          // P_{r+1} is read by V[r+2] = d_c P_{r+1} (o + e_c, o <= m) and,
          // through Lap, by P_{r+3}: box q <= m + 1 + (n - 2 - (r + 1))
          constexpr int lim = (MM + 1 + (n - 3 - r)) < n - 1 ? MM + 1 + (n - 3 - r) : n - 1;
          using L = std::integral_constant<int, lim>;
          av_lap(Pc, Xs, L{});   // Xs = av Lap P_{r-1}
          ap_times(Xs, L{});     // Xs = P_{r+1}
          double* tmp = Pc;
          Pc = Xs;
          Xs = tmp;
        }
      });
      // keep A/B/Cb roles consistent for the next node
      (void)Xs;
    }

    // store + finite flag
    bool bad = false;
#pragma unroll
    for (int c = 0; c < NOUT; ++c)
#pragma unroll
      for (int j = 0; j < FL; ++j) {
        const int f = lane + 32 * j;
        if (f < F) {
          bad |= !isfinite(tgt[c][j]);
          P.dst[c][toff + static_cast<int64_t>(f) * P.t_coef] = tgt[c][j];
        }
      }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && P.step >= 0) report_nonfinite(P.flag, P.step);
    // restore the buffer roles (the pressure loop may have swapped them)
    A = sm + warp * C::NBUF * T;
    B = A + T;
    Cb = B + T;
    __syncwarp();
  }
}

template <int MM>
int launch_m(HalfKind kind, const V3Params& q, cudaStream_t st) {
  const size_t smem = sizeof(double) * V3<MM>::SMEM;
  static std::atomic<unsigned long long> cfg_pre{0}, cfg_vel{0};
  const int64_t total = static_cast<int64_t>(q.hp.tNx) * q.hp.tNy * q.hp.tNz;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (total + WARPS - 1) / WARPS;
  const unsigned blocks = static_cast<unsigned>(want < 64LL * sms ? want : 64LL * sms);
  if (kind == VEL) {
    ensure_smem_opt_in(var3d<MM, VEL>, static_cast<int>(smem), cfg_vel);
    var3d<MM, VEL><<<blocks, WARPS * 32, smem, st>>>(q);
  } else {
    ensure_smem_opt_in(var3d<MM, PRE>, static_cast<int>(smem), cfg_pre);
    var3d<MM, PRE><<<blocks, WARPS * 32, smem, st>>>(q);
  }
  mark_launch(q.hp, st);
  return 1;
}

// separable coefficient jets on the nodes of one grid, stored like hlf_set_coeff's
// ([z][E][y][x]): jet = -(c0 e_0 + c1 s_x (x) s_y (x) s_z)
template <int D>
__global__ void fill_sep_coeff(double* dst, int Nx, int Ny, int Nz, int n, double h, double x0, double y0, double z0,
                               double c0, double c1, double wx, double wy, double wz, double px, double py,
                               double pz) {
  const int64_t total = static_cast<int64_t>(Nx) * Ny * Nz;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int ix = static_cast<int>(i % Nx);
  const int iy = static_cast<int>((i / Nx) % Ny);
  const int iz = static_cast<int>(i / (static_cast<int64_t>(Nx) * Ny));
  double s[3][kMaxN];
  const double w[3] = {wx, wy, wz}, ph[3] = {px, py, pz}, xx[3] = {x0 + ix * h, y0 + iy * h, z0 + iz * h};
  for (int ax = 0; ax < D; ++ax) {
    double sn, cs;
    sincos(w[ax] * xx[ax] + ph[ax], &sn, &cs);
    double f = 1.0;
    for (int k = 0; k < n; ++k) {
      const int r = k & 3;
      s[ax][k] = f * (r == 0 ? sn : (r == 1 ? cs : (r == 2 ? -sn : -cs)));
      f = f * (w[ax] * h) / (k + 1);
    }
  }
  const int64_t plane = static_cast<int64_t>(Nx) * Ny;
  const int E = D == 1 ? n : (D == 2 ? n * n : n * n * n);
  for (int e = 0; e < E; ++e) {
    int q[3] = {0, 0, 0}, r = e;
    for (int ax = D - 1; ax >= 0; --ax) {
      q[ax] = r % n;
      r /= n;
    }
    double prod = c1;
    for (int ax = 0; ax < D; ++ax) prod *= s[ax][q[ax]];
    const double v = -(prod + (e == 0 ? c0 : 0.0));
    dst[(static_cast<int64_t>(iz) * E + e) * plane + static_cast<int64_t>(iy) * Nx + ix] = v;
  }
}

}  // namespace

bool var3d_supported(int m) { return m >= 1 && m <= 3; }

int launch_half_var3d(int m, HalfKind kind, const HalfParams& p, const double* sep, const double* x0,
                      cudaStream_t st) {
  V3Params q;
  q.hp = p;
  q.c0 = sep[0];
  q.c1 = sep[1];
  for (int a = 0; a < 3; ++a) {
    q.w[a] = sep[2 + a];
    q.ph[a] = sep[5 + a];
    q.x0[a] = x0[a];
  }
  switch (m) {
    case 1: return launch_m<1>(kind, q, st);
    case 2: return launch_m<2>(kind, q, st);
    case 3: return launch_m<3>(kind, q, st);
    default: return -1;
  }
}

int launch_fill_sep_coeff(double* dst, int d, const int* N, int n, double h, const double* x0, const double* sep,
                          cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(N[0]) * N[1] * N[2];
  const unsigned blocks = static_cast<unsigned>((total + 127) / 128);
  if (d == 1)
    fill_sep_coeff<1><<<blocks, 128, 0, st>>>(dst, N[0], N[1], N[2], n, h, x0[0], x0[1], x0[2], sep[0], sep[1],
                                              sep[2], sep[3], sep[4], sep[5], sep[6], sep[7]);
  else if (d == 2)
    fill_sep_coeff<2><<<blocks, 128, 0, st>>>(dst, N[0], N[1], N[2], n, h, x0[0], x0[1], x0[2], sep[0], sep[1],
                                              sep[2], sep[3], sep[4], sep[5], sep[6], sep[7]);
  else
    fill_sep_coeff<3><<<blocks, 128, 0, st>>>(dst, N[0], N[1], N[2], n, h, x0[0], x0[1], x0[2], sep[0], sep[1],
                                              sep[2], sep[3], sep[4], sep[5], sep[6], sep[7]);
  return 1;
}

}  // namespace hlfk
