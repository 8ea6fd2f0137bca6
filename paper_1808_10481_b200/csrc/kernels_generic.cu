// Generic Hermite-leapfrog half-step kernels, any d in {1,2,3} and order m
// (d<=2: m<=8; d=3: m<=4).  One thread per target node; the stacked corner
// tensor and the reconstruction live in thread-local arrays.  This is the
// correctness path for every configuration and the production path for 1D;
// the 3D headline runs the tiled kernel in kernels_tiled3d.cu.  In 1D the
// same arithmetic runs fully unrolled in registers (half_1d).
//
// Per target node:
//   1. gather the (m+1)^d jets of the 2^d source corners into the stacked
//      n^d tensor, index side*(m+1)+l per axis (reconstruct_cell_1d/2d,
//      interpolation.cpp:63-113), mirroring ghosts across reflective walls;
//   2. apply M along x, then y, then z (interpolation.cpp:87-112);
//   3. the iterated, truncated CK recurrence of ck_recurrence_variable
//      (stepper1d.cpp:22-38) with scalar or per-node (tensor product,
//      jet.cpp:109-121) ap and the odd-level sum of leapfrog_half_update
//      (stepper1d.cpp:54-61), in the oracle's operation order;
//   4. in-place update of the target jet and the non-finite flag
//      (check_finite, stepper1d.cpp:121-129).
#include "hlf_internal.cuh"

namespace hlfk {
namespace {

__host__ __device__ constexpr int cpow(int b, int e) { return e == 0 ? 1 : b * cpow(b, e - 1); }

// x / h of jet_differentiate (jet.cpp:20-31).  When h is a power of two the
// quotient equals x * (1/h) bit for bit (both are the correctly rounded value
// of the same real number), so the faithful kernels skip the IEEE division.
template <class Params>
__device__ __forceinline__ double div_h(double x, const Params& P) {
  return P.pow2_h ? __dmul_rn(x, P.inv_h) : __ddiv_rn(x, P.h);
}

template <int D>
struct Idx {
  // tensor of extent N per axis, x-major: e = sum_ax q_ax N^(D-1-ax)
  template <int N>
  __device__ static __forceinline__ int flat(const int* q) {
    int e = 0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) e = e * N + q[ax];
    return e;
  }
  template <int N>
  __device__ static __forceinline__ void split(int e, int* q) {
#pragma unroll
    for (int ax = D - 1; ax >= 0; --ax) {
      q[ax] = e % N;
      e /= N;
    }
  }
};

// Entries of CK level k that any later level or the target reads: the target
// needs q <= m per axis at the odd levels, and each level reads the next one
// shifted by one unit along one axis (d_c T[q] = T[q + e_c] ...), so level k
// needs excess(q) = sum_c max(0, q_c - m) <= n - 1 - k.  The set is closed
// downwards, so the truncated products stay inside it.  Skipping the other
// entries changes no computed value (bit-identical results).
template <int D, int MM>
__device__ __forceinline__ int excess(int e) {
  constexpr int n = 2 * MM + 2;
  int x = 0;
#pragma unroll
  for (int ax = 0; ax < D; ++ax) {
    const int q = e % n;
    e /= n;
    x += q > MM ? q - MM : 0;
  }
  return x;
}

// FRC: a forcing table z_r (n^d jets, levels r = 0..2m) at the target nodes is
// added to every P level (ck_recurrence_variable's z, stepper1d.cpp:29-32,
// generalised to tensor jets): both tables are then live at every level.
template <int D, int MM, bool VAR, int KIND, bool FRC = false>
__global__ void __launch_bounds__(128) half_generic(const __grid_constant__ HalfParams P) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  constexpr int F = cpow(n1, D), E = cpow(n, D);
  constexpr int NSRC = KIND == VEL ? 1 : D;

  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(P.tNx) * P.tNy * P.tNz;
  if (tid >= total) return;
  int t[3];
  t[0] = static_cast<int>(tid % P.tNx);
  const int64_t rest = tid / P.tNx;
  t[1] = static_cast<int>(rest % P.tNy);
  t[2] = static_cast<int>(rest / P.tNy);

  // ---- corner addresses (plane offset + layer) and reflection flags ----
  // axes 0..min(D,2)-1 are in-plane (x, y); axis 2 (z, d = 3) uses layers
  int64_t coff[1 << D];
  int cflip[1 << D];  // bit ax set: mirrored across a wall normal to ax
#pragma unroll
  for (int corner = 0; corner < (1 << D); ++corner) {
    int s[3] = {0, 0, 0};
    int flip = 0;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const int side = (corner >> ax) & 1;
      int q = KIND == VEL ? t[ax] + side : t[ax] - 1 + side;
      if (ax < 2) {
        if (P.bnd[ax] == 0) {
          if (q >= P.K[ax]) q -= P.K[ax];
          if (q < 0) q += P.K[ax];
        } else if (KIND == PRE) {
          if (q < 0) {
            q = 0;
            flip |= 1 << ax;
          } else if (q >= P.K[ax]) {
            q = P.K[ax] - 1;
            flip |= 1 << ax;
          }
        }
      }
      s[ax] = q;
    }
    const int layer = D == 3 ? P.s_zoff + s[2] : 0;
    coff[corner] = static_cast<int64_t>(layer) * P.s_layer + static_cast<int64_t>(D >= 2 ? s[1] : 0) * P.sNx + s[0];
    cflip[corner] = flip;
  }

  const int64_t toff = static_cast<int64_t>(D == 3 ? P.t_zoff + t[2] : 0) * P.t_layer +
                       static_cast<int64_t>(D >= 2 ? t[1] : 0) * P.tNx + t[0];

  // Arithmetic below is "faithful": separate IEEE multiply/add/divide in the
  // oracle's order (no FMA contraction), so results equal the oracle and, in
  // 1D, the compiled reference bit for bit.  The reconstruction is
  // ill-conditioned (cond(A) = 429 at m = 3), so ANY reordering moves
  // long-run results by ~N cond(A) eps (compiling the reference itself with
  // -mfma moves config 1 by 1.2e-11); the fast tiled kernels trade this for
  // speed and are checked against the 1e-12 bar over short runs.
  double S[E];
  double Pt[E];
  double Vt[D * E];
  bool bad = false;
  if constexpr (FRC) {  // the seeded-zero table is read at level 0 (ck_recurrence_variable: P[0] / V[0])
#pragma unroll 1
    for (int e = 0; e < E; ++e) {
      if (KIND == VEL)
        for (int c = 0; c < D; ++c) Vt[c * E + e] = 0.0;
      else
        Pt[e] = 0.0;
    }
  }

#pragma unroll 1
  for (int comp = 0; comp < NSRC; ++comp) {
    const double* src = P.src[comp];
    // 1. stacked corners
#pragma unroll 1
    for (int corner = 0; corner < (1 << D); ++corner) {
#pragma unroll 1
      for (int f = 0; f < F; ++f) {
        int a[3];
        Idx<D>::template split<n1>(f, a);
        double sign = 1.0;
        int q[3];
#pragma unroll
        for (int ax = 0; ax < D; ++ax) {
          if ((cflip[corner] >> ax) & 1) {
            if (a[ax] & 1) sign = -sign;
            if (comp != ax) sign = -sign;  // tangential velocity is odd across the wall
          }
          q[ax] = ((corner >> ax) & 1) * n1 + a[ax];
        }
        S[Idx<D>::template flat<n>(q)] = sign * __ldg(src + coff[corner] + f * P.s_coef);
      }
    }
    // 2. tensor sweeps, x first (interpolation.cpp:53-61, 87-112)
#pragma unroll 1
    for (int ax = 0; ax < D; ++ax) {
      const int stride = cpow(n, D - 1 - ax);
#pragma unroll 1
      for (int e = 0; e < E; ++e) {
        if ((e / stride) % n != 0) continue;
        double in[n];
#pragma unroll
        for (int s = 0; s < n; ++s) in[s] = S[e + s * stride];
#pragma unroll
        for (int r = 0; r < n; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int s = 0; s < n; ++s) acc = __dadd_rn(acc, __dmul_rn(P.M[r * n + s], in[s]));
          S[e + r * stride] = acc;
        }
      }
    }
#pragma unroll 1
    for (int e = 0; e < E; ++e) {
      if (KIND == PRE) Vt[comp * E + e] = S[e];
      else Pt[e] = S[e];
    }
  }

  // 3. coupled CK recurrence, count = 2m+2 (stepper1d.cpp:22-38): with one
  //    field seeded zero only one table is live per level.
  //    P[r+1] = ap (.) sum_c d_c V_c[r];  V_c[r+1] = av d_c P[r]
  //    d_c T[q] = (T[q+e_c] (q_c+1)) / h, truncated (jet.cpp:123-135)
  constexpr int NOUT = KIND == VEL ? D : 1;
  double tgt[NOUT * F];
#pragma unroll 1
  for (int c = 0; c < NOUT; ++c)
#pragma unroll 1
    for (int f = 0; f < F; ++f) tgt[c * F + f] = P.dst[c][toff + f * P.t_coef];
  const double* apj = VAR ? P.coeff + static_cast<int64_t>(D == 3 ? t[2] : 0) * P.c_layer +
                                static_cast<int64_t>(D >= 2 ? t[1] : 0) * P.tNx + t[0]
                          : nullptr;
  double apl[VAR ? E : 1];  // this node's ap jet, loaded once for all CK levels
  if constexpr (VAR) {
#pragma unroll 1
    for (int e = 0; e < E; ++e) apl[e] = __ldg(apj + e * P.c_coef);
  }
  // forcing table of this node: [t_z][(r E + e)][t_y][t_x] (no ghost layers)
  const double* zf = FRC ? P.force + static_cast<int64_t>(D == 3 ? t[2] : 0) * P.f_layer +
                               static_cast<int64_t>(D >= 2 ? t[1] : 0) * P.tNx + t[0]
                         : nullptr;
#pragma unroll 1
  for (int r = 0; r + 1 < n; ++r) {
    const bool p_live = (KIND == VEL) == (r % 2 == 0);
    const int keep = n - 2 - r;  // level r + 1 entries with excess <= keep are read later
    if (FRC) {
      // both tables from level r: S = sum_c d_c V_c[r] first (old V), then
      // V_c[r+1] = av d_c P[r] (old P), then P[r+1] = ap (.) S + z_r
#pragma unroll 1
      for (int e = 0; e < E; ++e) S[e] = 0.0;
#pragma unroll 1
      for (int c = 0; c < D; ++c) {
        const int stride = cpow(n, D - 1 - c);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
          if (excess<D, MM>(e) > keep) continue;
          const int qc = (e / stride) % n;
          const double dv = qc + 1 < n ? div_h(__dmul_rn(Vt[c * E + e + stride], static_cast<double>(qc + 1)), P) : 0.0;
          S[e] = __dadd_rn(S[e], dv);
        }
      }
#pragma unroll 1
      for (int c = 0; c < D; ++c) {
        const int stride = cpow(n, D - 1 - c);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
          if (excess<D, MM>(e) > keep) continue;
          const int qc = (e / stride) % n;
          const double dv = qc + 1 < n ? div_h(__dmul_rn(Pt[e + stride], static_cast<double>(qc + 1)), P) : 0.0;
          Vt[c * E + e] = __dmul_rn(P.av, dv);
        }
      }
    }
    if (FRC) {
      // P[r+1] below (the p_live = false branch) from S
    } else if (p_live) {
#pragma unroll 1
      for (int c = 0; c < D; ++c) {
        const int stride = cpow(n, D - 1 - c);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
          if (excess<D, MM>(e) > keep) continue;
          const int qc = (e / stride) % n;
          const double dv = qc + 1 < n ? div_h(__dmul_rn(Pt[e + stride], static_cast<double>(qc + 1)), P) : 0.0;
          Vt[c * E + e] = __dmul_rn(P.av, dv);
        }
      }
    }
    if (FRC || !p_live) {
      // Pt <- ap (.) (sum_c d_c V_c); the sum goes through S as scratch
#pragma unroll 1
      for (int e = 0; e < E && !FRC; ++e) S[e] = 0.0;
#pragma unroll 1
      for (int c = 0; c < D && !FRC; ++c) {
        const int stride = cpow(n, D - 1 - c);
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
          if (excess<D, MM>(e) > keep) continue;
          const int qc = (e / stride) % n;
          const double dv = qc + 1 < n ? div_h(__dmul_rn(Vt[c * E + e + stride], static_cast<double>(qc + 1)), P) : 0.0;
          S[e] = __dadd_rn(S[e], dv);
        }
      }
      if (VAR) {
        // truncated tensor product, contributions in ascending order of the
        // ap index (jet.cpp:109-121): for output q only ap indices qi <= q
        // (per axis) contribute, visited as nested ascending loops, which is
        // the ascending flat order of the reference's full scan
#pragma unroll 1
        for (int e = 0; e < E; ++e) {
          if (excess<D, MM>(e) > keep) continue;
          int q[3] = {0, 0, 0};
          Idx<D>::template split<n>(e, q);
          double s = 0.0;
          if constexpr (D == 2) {
#pragma unroll 1
            for (int ix = 0; ix <= q[0]; ++ix)
#pragma unroll 1
              for (int iy = 0; iy <= q[1]; ++iy) {
                const double a = apl[ix * n + iy];
                if (a != 0.0) s = __dadd_rn(s, __dmul_rn(a, S[(q[0] - ix) * n + (q[1] - iy)]));
              }
          } else {
#pragma unroll 1
            for (int ix = 0; ix <= q[0]; ++ix)
#pragma unroll 1
              for (int iy = 0; iy <= q[1]; ++iy)
#pragma unroll 1
                for (int iz = 0; iz <= q[2]; ++iz) {
                  const double a = apl[(ix * n + iy) * n + iz];
                  if (a != 0.0) s = __dadd_rn(s, __dmul_rn(a, S[((q[0] - ix) * n + (q[1] - iy)) * n + (q[2] - iz)]));
                }
          }
          Pt[e] = s;
        }
      } else {
#pragma unroll 1
        for (int e = 0; e < E; ++e)
          if (excess<D, MM>(e) <= keep) Pt[e] = __dmul_rn(P.ap, S[e]);
      }
      if (FRC) {
#pragma unroll 1
        for (int e = 0; e < E; ++e)
          if (excess<D, MM>(e) <= keep) Pt[e] = __dadd_rn(Pt[e], __ldg(zf + (r * E + e) * P.f_coef));
      }
    }
    // leapfrog_half_update (stepper1d.cpp:54-61): odd levels of the target's table
    if ((r + 1) & 1) {
      const double w = P.w[r + 1];
#pragma unroll 1
      for (int c = 0; c < NOUT; ++c)
#pragma unroll 1
        for (int f = 0; f < F; ++f) {
          int o[3] = {0, 0, 0};
          Idx<D>::template split<n1>(f, o);
          const int e = Idx<D>::template flat<n>(o);
          const double tv = KIND == VEL ? Vt[c * E + e] : Pt[e];
          tgt[c * F + f] = __dadd_rn(tgt[c * F + f], __dmul_rn(w, tv));
        }
    }
  }
  // 4. in-place store + finite flag (check_finite, stepper1d.cpp:121-129)
#pragma unroll 1
  for (int c = 0; c < NOUT; ++c)
#pragma unroll 1
    for (int f = 0; f < F; ++f) {
      const double nv = tgt[c * F + f];
      bad |= !isfinite(nv);
      P.dst[c][toff + f * P.t_coef] = nv;
    }

  if (bad && P.step >= 0) report_nonfinite(P.flag, P.step);
}

// 1D: the same faithful arithmetic, operation for operation (so results stay
// bit-identical to half_generic<1,...>, the oracle and the compiled
// reference), but fully unrolled: every array index is a compile-time
// constant, the 2n stacked values, the two n-entry tables and the target jet
// live in registers, and the kernel streams at memory speed instead of
// spilling its tables to local memory.
//
// FRC: a forcing table z_r (ck_recurrence_variable's z, stepper1d.cpp:29-32)
// is added to every P level, so both tables are live at every level and the
// full coupled recurrence runs: P[r+1] = ap (.) D V[r] + z_r, V[r+1] = av D P[r].
template <int MM, bool VAR, int KIND, bool FRC = false>
__global__ void __launch_bounds__(128) half_1d(const __grid_constant__ HalfParams P) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  const int t0 = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t0 >= P.tNx) return;
  // corner nodes (same maps as half_generic)
  int q[2];
  bool flip[2];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    int qq = KIND == VEL ? t0 + side : t0 - 1 + side;
    flip[side] = false;
    if (P.bnd[0] == 0) {
      if (qq >= P.K[0]) qq -= P.K[0];
      if (qq < 0) qq += P.K[0];
    } else if (KIND == PRE) {
      if (qq < 0) {
        qq = 0;
        flip[side] = true;
      } else if (qq >= P.K[0]) {
        qq = P.K[0] - 1;
        flip[side] = true;
      }
    }
    q[side] = qq;
  }
  double S[n];
#pragma unroll
  for (int side = 0; side < 2; ++side)
#pragma unroll
    for (int a = 0; a < n1; ++a) {
      const double v = __ldg(P.src[0] + q[side] + a * P.s_coef);
      S[side * n1 + a] = (flip[side] && (a & 1)) ? -v : v;  // ghost = (-1)^a interior (normal velocity)
    }
  double T[n];  // M applied along x (interpolation.cpp:53-61)
#pragma unroll
  for (int r = 0; r < n; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < n; ++s2) acc = __dadd_rn(acc, __dmul_rn(P.M[r * n + s2], S[s2]));
    T[r] = acc;
  }
  double Pt[n], Vt[n];
#pragma unroll
  for (int e = 0; e < n; ++e) {
    Pt[e] = KIND == VEL ? T[e] : 0.0;
    Vt[e] = KIND == VEL ? 0.0 : T[e];
  }
  const int64_t toff = t0;
  double tgt[n1];
#pragma unroll
  for (int f = 0; f < n1; ++f) tgt[f] = P.dst[0][toff + f * P.t_coef];
  const double* apj = VAR ? P.coeff + t0 : nullptr;
  // CK recurrence, count = 2m+2 levels (stepper1d.cpp:22-38)
#pragma unroll
  for (int r = 0; FRC && r + 1 < n; ++r) {
    // P[r+1] = ap (.) D V[r] + z_r and V[r+1] = av (.) D P[r] (both from level r)
    double Pn[n], Vn[n];
#pragma unroll
    for (int e = 0; e < n; ++e) {
      const double dp = e + 1 < n ? div_h(__dmul_rn(Pt[e + 1 < n ? e + 1 : e], static_cast<double>(e + 1)), P) : 0.0;
      Vn[e] = __dadd_rn(0.0, __dmul_rn(P.av, dp));
    }
    double Sd[n];
#pragma unroll
    for (int e = 0; e < n; ++e)
      Sd[e] = e + 1 < n ? div_h(__dmul_rn(Vt[e + 1 < n ? e + 1 : e], static_cast<double>(e + 1)), P) : 0.0;
#pragma unroll
    for (int e = 0; e < n; ++e) {
      double sacc = 0.0;
      if (VAR) {
#pragma unroll
        for (int ei = 0; ei <= e; ++ei) {
          const double a = __ldg(apj + ei * P.c_coef);
          if (a != 0.0) sacc = __dadd_rn(sacc, __dmul_rn(a, Sd[e - ei]));
        }
      } else {
        sacc = __dadd_rn(0.0, __dmul_rn(P.ap, Sd[e]));
      }
      Pn[e] = __dadd_rn(sacc, __ldg(P.force + t0 + (r * n + e) * P.f_coef));
    }
#pragma unroll
    for (int e = 0; e < n; ++e) {
      Pt[e] = Pn[e];
      Vt[e] = Vn[e];
    }
    if ((r + 1) & 1) {  // leapfrog_half_update (stepper1d.cpp:54-61)
      const double w = P.w[r + 1];
#pragma unroll
      for (int f = 0; f < n1; ++f) tgt[f] = __dadd_rn(tgt[f], __dmul_rn(w, KIND == VEL ? Vt[f] : Pt[f]));
    }
  }
#pragma unroll
  for (int r = 0; !FRC && r + 1 < n; ++r) {
    const bool p_live = (KIND == VEL) == (r % 2 == 0);
    if (p_live) {
#pragma unroll
      for (int e = 0; e < n; ++e) {
        const double dv = e + 1 < n ? div_h(__dmul_rn(Pt[e + 1 < n ? e + 1 : e], static_cast<double>(e + 1)), P)
                                    : 0.0;
        Vt[e] = __dmul_rn(P.av, dv);
      }
    } else {
      double Sd[n];
#pragma unroll
      for (int e = 0; e < n; ++e) {
        const double dv = e + 1 < n ? div_h(__dmul_rn(Vt[e + 1 < n ? e + 1 : e], static_cast<double>(e + 1)), P)
                                    : 0.0;
        Sd[e] = __dadd_rn(0.0, dv);
      }
      if (VAR) {
#pragma unroll
        for (int e = 0; e < n; ++e) {
          double sacc = 0.0;
#pragma unroll
          for (int ei = 0; ei <= e; ++ei) {
            const double a = __ldg(apj + ei * P.c_coef);
            if (a != 0.0) sacc = __dadd_rn(sacc, __dmul_rn(a, Sd[e - ei]));
          }
          Pt[e] = sacc;
        }
      } else {
#pragma unroll
        for (int e = 0; e < n; ++e) Pt[e] = __dmul_rn(P.ap, Sd[e]);
      }
    }
    if ((r + 1) & 1) {  // leapfrog_half_update (stepper1d.cpp:54-61)
      const double w = P.w[r + 1];
#pragma unroll
      for (int f = 0; f < n1; ++f) tgt[f] = __dadd_rn(tgt[f], __dmul_rn(w, KIND == VEL ? Vt[f] : Pt[f]));
    }
  }
  bool bad = false;
#pragma unroll
  for (int f = 0; f < n1; ++f) {
    bad |= !isfinite(tgt[f]);
    P.dst[0][toff + f * P.t_coef] = tgt[f];
  }
  if (bad && P.step >= 0) report_nonfinite(P.flag, P.step);
}

template <int D, int MM>
int launch_dm(bool variable, HalfKind kind, const HalfParams& p, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(p.tNx) * p.tNy * p.tNz;
  const int threads = 128;
  const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
  if (blocks == 0) return 0;
  if constexpr (D == 1) {
    if (p.force) {
      if (kind == VEL) {
        if (variable) half_1d<MM, true, VEL, true><<<blocks, threads, 0, st>>>(p);
        else half_1d<MM, false, VEL, true><<<blocks, threads, 0, st>>>(p);
      } else {
        if (variable) half_1d<MM, true, PRE, true><<<blocks, threads, 0, st>>>(p);
        else half_1d<MM, false, PRE, true><<<blocks, threads, 0, st>>>(p);
      }
      return 1;
    }
    if (kind == VEL) {
      if (variable) half_1d<MM, true, VEL><<<blocks, threads, 0, st>>>(p);
      else half_1d<MM, false, VEL><<<blocks, threads, 0, st>>>(p);
    } else {
      if (variable) half_1d<MM, true, PRE><<<blocks, threads, 0, st>>>(p);
      else half_1d<MM, false, PRE><<<blocks, threads, 0, st>>>(p);
    }
    return 1;
  }
  if (p.force) {
    if (kind == VEL) {
      if (variable) half_generic<D, MM, true, VEL, true><<<blocks, threads, 0, st>>>(p);
      else half_generic<D, MM, false, VEL, true><<<blocks, threads, 0, st>>>(p);
    } else {
      if (variable) half_generic<D, MM, true, PRE, true><<<blocks, threads, 0, st>>>(p);
      else half_generic<D, MM, false, PRE, true><<<blocks, threads, 0, st>>>(p);
    }
    return 1;
  }
  if (kind == VEL) {
    if (variable) half_generic<D, MM, true, VEL><<<blocks, threads, 0, st>>>(p);
    else half_generic<D, MM, false, VEL><<<blocks, threads, 0, st>>>(p);
  } else {
    if (variable) half_generic<D, MM, true, PRE><<<blocks, threads, 0, st>>>(p);
    else half_generic<D, MM, false, PRE><<<blocks, threads, 0, st>>>(p);
  }
  return 1;
}

// ---- 1D alternative schemes (faithful arithmetic, reference operation order)

// both CK tables of ck_recurrence_variable (stepper1d.cpp:22-38) level by
// level from the reconstructions of the two fields; `sink(r, Pr, Vr)` sees
// every level r = 0..n-1 in order
template <int MM, typename Sink>
__device__ __forceinline__ void ck_tables_1d(const Scheme1dParams& P, const double (&Tp)[2 * MM + 2],
                                             const double (&Tv)[2 * MM + 2], Sink sink) {
  constexpr int n = 2 * MM + 2;
  double Pc[n], Vc[n];
#pragma unroll
  for (int e = 0; e < n; ++e) {
    Pc[e] = Tp[e];
    Vc[e] = Tv[e];
  }
  sink(0, Pc, Vc);
#pragma unroll
  for (int r = 0; r + 1 < n; ++r) {
    double Pn[n], Vn[n];
#pragma unroll
    for (int e = 0; e < n; ++e) {
      // jet_multiply(ap, jet_differentiate(V, 1, h)) with ap = [ap, 0, ...]:
      // out = 0.0 + ap * (V[e+1] * (e+1) / h)  (jet.cpp:8-31)
      const double dv = e + 1 < n ? div_h(__dmul_rn(Vc[e + 1 < n ? e + 1 : e], static_cast<double>(e + 1)), P) : 0.0;
      const double dp = e + 1 < n ? div_h(__dmul_rn(Pc[e + 1 < n ? e + 1 : e], static_cast<double>(e + 1)), P) : 0.0;
      Pn[e] = __dadd_rn(0.0, __dmul_rn(P.ap, dv));
      Vn[e] = __dadd_rn(0.0, __dmul_rn(P.av, dp));
    }
#pragma unroll
    for (int e = 0; e < n; ++e) {
      Pc[e] = Pn[e];
      Vc[e] = Vn[e];
    }
    sink(r + 1, Pc, Vc);
  }
}

// reconstruct_cell_1d + interp_apply (interpolation.cpp:53-75) for both fields
template <int MM>
__device__ __forceinline__ void reconstruct_pv_1d(const Scheme1dParams& P, int li, int ri, double (&Tp)[2 * MM + 2],
                                                  double (&Tv)[2 * MM + 2]) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  double Sp[n], Sv[n];
#pragma unroll
  for (int a = 0; a < n1; ++a) {
    Sp[a] = __ldg(P.src_p + li + a * P.K);
    Sp[n1 + a] = __ldg(P.src_p + ri + a * P.K);
    Sv[a] = __ldg(P.src_v + li + a * P.K);
    Sv[n1 + a] = __ldg(P.src_v + ri + a * P.K);
  }
#pragma unroll
  for (int r = 0; r < n; ++r) {
    double ap_ = 0.0, av_ = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < n; ++s2) {
      ap_ = __dadd_rn(ap_, __dmul_rn(P.M[r * n + s2], Sp[s2]));
      av_ = __dadd_rn(av_, __dmul_rn(P.M[r * n + s2], Sv[s2]));
    }
    Tp[r] = ap_;
    Tv[r] = av_;
  }
}

// one half of step_modified: out = modified_advance(prev, table) for p and v
// (stepper1d.cpp:73-91, 191-232)
template <int MM>
__global__ void __launch_bounds__(128) modified_1d(const __grid_constant__ Scheme1dParams P) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  const int j = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P.K) return;
  const int li = P.to_primary ? (j == 0 ? P.K - 1 : j - 1) : j;
  const int ri = P.to_primary ? j : (j + 1 == P.K ? 0 : j + 1);
  double Tp[n], Tv[n];
  reconstruct_pv_1d<MM>(P, li, ri, Tp, Tv);
  double op[n1], ov[n1];
#pragma unroll
  for (int s2 = 0; s2 < n1; ++s2) {
    const double pp = P.dst_p[j + s2 * P.K], pv = P.dst_v[j + s2 * P.K];
    op[s2] = s2 % 2 == 0 ? pp : -pp;
    ov[s2] = s2 % 2 == 0 ? pv : -pv;
  }
  double w = 2.0;  // w[0] = 2, w[r] = w[r-1] * dt / 2 / r
  ck_tables_1d<MM>(P, Tp, Tv, [&](int r, const double (&Pr)[n], const double (&Vr)[n]) {
    if (r > 0) w = __ddiv_rn(__dmul_rn(__dmul_rn(w, P.dt), 0.5), static_cast<double>(r));  // (w dt) / 2 == (w dt) * 0.5 exactly
#pragma unroll
    for (int s2 = 0; s2 < n1; ++s2) {
      if ((s2 % 2 == 0) == (r % 2 == 1)) {  // even s: odd levels; odd s: even levels
        op[s2] = __dadd_rn(op[s2], __dmul_rn(w, Pr[s2]));
        ov[s2] = __dadd_rn(ov[s2], __dmul_rn(w, Vr[s2]));
      }
    }
  });
  bool bad = false;
#pragma unroll
  for (int s2 = 0; s2 < n1; ++s2) {
    bad |= !isfinite(op[s2]) || !isfinite(ov[s2]);
    P.dst_p[j + s2 * P.K] = op[s2];
    P.dst_v[j + s2 * P.K] = ov[s2];
  }
  if (bad && P.step >= 0) report_nonfinite(P.flag, P.step);
}

// one pass of step_dual_hermite: taylor_advance by tau = dt/2 (stepper1d.cpp:63-71, 249-272)
template <int MM, int PASS>
__global__ void __launch_bounds__(128) dual_hermite_1d(const __grid_constant__ Scheme1dParams P) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  const int j = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P.K) return;
  const int li = PASS == 0 ? j : (j == 0 ? P.K - 1 : j - 1);
  const int ri = PASS == 0 ? (j + 1 == P.K ? 0 : j + 1) : j;
  double Tp[n], Tv[n];
  reconstruct_pv_1d<MM>(P, li, ri, Tp, Tv);
  const double tau = __dmul_rn(P.dt, 0.5);  // dt / 2 exactly
  double op[n1], ov[n1];
#pragma unroll
  for (int s2 = 0; s2 < n1; ++s2) op[s2] = ov[s2] = 0.0;
  double w = 1.0;
  ck_tables_1d<MM>(P, Tp, Tv, [&](int r, const double (&Pr)[n], const double (&Vr)[n]) {
    if (r > 0) w = __dmul_rn(w, __ddiv_rn(tau, static_cast<double>(r)));
#pragma unroll
    for (int s2 = 0; s2 < n1; ++s2) {
      op[s2] = __dadd_rn(op[s2], __dmul_rn(w, Pr[s2]));
      ov[s2] = __dadd_rn(ov[s2], __dmul_rn(w, Vr[s2]));
    }
  });
  bool bad = false;
#pragma unroll
  for (int s2 = 0; s2 < n1; ++s2) {
    bad |= !isfinite(op[s2]) || !isfinite(ov[s2]);
    P.dst_p[j + s2 * P.K] = op[s2];
    P.dst_v[j + s2 * P.K] = ov[s2];
  }
  if (PASS == 1 && bad && P.step >= 0) report_nonfinite(P.flag, P.step);
}

}  // namespace

int launch_modified_1d(int m, const Scheme1dParams& p, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>((p.K + 127) / 128);
  switch (m) {
#define HLF_M(MM) \
  case MM: modified_1d<MM><<<blocks, 128, 0, st>>>(p); return 1;
    HLF_M(0) HLF_M(1) HLF_M(2) HLF_M(3) HLF_M(4) HLF_M(5) HLF_M(6) HLF_M(7) HLF_M(8)
#undef HLF_M
    default: return -1;
  }
}

int launch_dual_hermite_1d(int m, int pass, const Scheme1dParams& p, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>((p.K + 127) / 128);
  switch (m) {
#define HLF_M(MM)                                                            \
  case MM:                                                                   \
    if (pass == 0) dual_hermite_1d<MM, 0><<<blocks, 128, 0, st>>>(p);        \
    else dual_hermite_1d<MM, 1><<<blocks, 128, 0, st>>>(p);                  \
    return 1;
    HLF_M(0) HLF_M(1) HLF_M(2) HLF_M(3) HLF_M(4) HLF_M(5) HLF_M(6) HLF_M(7) HLF_M(8)
#undef HLF_M
    default: return -1;
  }
}

int launch_half_generic(int d, int m, bool variable, HalfKind kind, const HalfParams& p,
                        cudaStream_t st) {
#define HLF_CASE(D, MM) \
  if (d == D && m == MM) return launch_dm<D, MM>(variable, kind, p, st);
  HLF_CASE(1, 0) HLF_CASE(1, 1) HLF_CASE(1, 2) HLF_CASE(1, 3) HLF_CASE(1, 4)
  HLF_CASE(1, 5) HLF_CASE(1, 6) HLF_CASE(1, 7) HLF_CASE(1, 8)
  HLF_CASE(2, 0) HLF_CASE(2, 1) HLF_CASE(2, 2) HLF_CASE(2, 3) HLF_CASE(2, 4)
  HLF_CASE(2, 5) HLF_CASE(2, 6) HLF_CASE(2, 7) HLF_CASE(2, 8)
  HLF_CASE(3, 0) HLF_CASE(3, 1) HLF_CASE(3, 2) HLF_CASE(3, 3) HLF_CASE(3, 4)
#undef HLF_CASE
  return -1;
}

}  // namespace hlfk
