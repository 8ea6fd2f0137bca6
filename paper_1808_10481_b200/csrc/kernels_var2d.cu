// 2D half-step kernel with per-node coefficient jets (variable ap = -c^2(x, y),
// SURVEY.md sec. 8(d) config 3 and sec. 8(f) item 1), m = 1..4, periodic or
// reflective walls.
//
// The reference's variable-coefficient CK (ck_recurrence_variable,
// stepper1d.cpp:22-38) multiplies by the ap jet with a truncated Cauchy
// product at every level (tensor_multiply, jet.cpp:109-121), so the closed
// forms of the tiled kernels do not apply.  With one field seeded zero and av a
// scalar, the live levels collapse to
//   PRE  (v -> p):  P_1 = ap (.) div V_0,   P_{k+2} = ap (.) (av Lap P_k)
//   VEL  (p -> v):  V_{k+1} = av grad P_k,  P_{k+2} = ap (.) (av Lap P_k)
// where div / grad / Lap are the truncated scaled-jet derivatives of
// jet_differentiate / tensor_dx,dy (jet.cpp:20-31, 123-135) and (.) is the
// truncated tensor product; the odd levels are summed into the target with
// the weights of leapfrog_half_update (stepper1d.cpp:54-61).
//
// Only the entries a later level (or the target) reads are computed: level k
// needs the region R_k (per jet row qx, the largest qy), derived at compile
// time from the target box by "grow" (Lap reads q + 2e_x and q + 2e_y); at
// m = 3 this is 2232 multiply-adds per pressure cell instead of 5184.
//
// Layout: two threads per cell, 16 cells per warp, 2 warps per CTA.  Thread t
// owns the jet rows qx = t, t + 2, t + 4, ... of every level, so the level
// P_k lives in its registers and Lap P_k (rows qx and qx + 2) is
// thread-local; only X (the operand of the next product, all rows) and the
// ap jet sit in shared memory (rows padded to an odd number of 16 B slots,
// cells 2 slots apart: the LDS.128 row loads of a warp are conflict-free).
// The product of a row is a sum of 1D causal convolutions of ap rows with X
// rows; every ap row a thread loads serves all of its output rows.  The x
// derivatives of the velocity outputs and of div V_0 read the partner
// thread's rows through one shuffle per value.  The reconstruction uses the
// sum/difference form of M (M_R = diag((-1)^r) M_L diag((-1)^l),
// interpolation.cpp:29-48).
#include <cstring>
#include <utility>

#include "hlf_internal.cuh"

namespace hlfk {
namespace v2d {
namespace {

constexpr int NTHREADS = 64;
constexpr unsigned FULL = 0xffffffffu;

template <int MM>
struct Shape {
  static constexpr int n1 = MM + 1, n = 2 * MM + 2;
  static constexpr int NJ = MM + 1;                              // rows per thread
  static constexpr int NS = MM / 2 + 1;                          // target rows per thread (max)
  static constexpr int RS = ((n + 2) / 2) % 2 ? n + 2 : n + 4;   // padded row: odd number of 16 B slots
  static constexpr int AS = n * RS;                              // one jet
  static constexpr int CS = (2 * AS + 15) / 16 * 16 + 4;         // cell stride: 2 slots mod 8
  static constexpr int CPW = 16;
  static constexpr int CPC = CPW * (NTHREADS / 32);
  static constexpr int SMEM = CPC * CS * 8;
};

// lim[k][r]: the largest qy of row r needed at level k (-1: row not needed)
template <int MM, int KIND>
struct Regions {
  static constexpr int n = 2 * MM + 2;
  int lim[n][n];
  __host__ __device__ constexpr Regions() : lim() {
    for (int k = 0; k < n; ++k)
      for (int r = 0; r < n; ++r) lim[k][r] = -1;
    // target box (PRE: P_k itself on q <= m) or the output footprint (VEL:
    // grad P_k on q <= m reads q + e_x, q + e_y)
    int base[n] = {};
    for (int r = 0; r < n; ++r)
      base[r] = KIND == PRE ? (r <= MM ? MM : -1) : (r <= MM ? MM + 1 : (r == MM + 1 ? MM : -1));
    const int top = KIND == PRE ? n - 1 : n - 2;
    for (int r = 0; r < n; ++r) lim[top][r] = base[r];
    for (int k = top - 2; k >= 0; k -= 2)
      for (int r = 0; r < n; ++r) {
        int v = base[r];
        const int own = lim[k + 2][r] >= 0 ? (lim[k + 2][r] + 2 < n - 1 ? lim[k + 2][r] + 2 : n - 1) : -1;
        if (own > v) v = own;
        if (r >= 2 && lim[k + 2][r - 2] > v) v = lim[k + 2][r - 2];
        lim[k][r] = v;
      }
  }
  // limit of thread-row j (rows 2j and 2j + 1 of the two threads)
  __host__ __device__ constexpr int row_pair(int k, int j) const {
    const int a = lim[k][2 * j], b = lim[k][2 * j + 1];
    return a > b ? a : b;
  }
  __host__ __device__ constexpr int last_row(int k) const {
    int r = -1;
    for (int q = 0; q < n; ++q)
      if (lim[k][q] >= 0) r = q;
    return r;
  }
};

// sum/difference form of one M application: out[r] = sum_l M[r][l] (L_l + (-1)^{r-l} R_l)
template <int MM>
__device__ __forceinline__ void apply_m(const HalfParams& P, const double (&lr)[2 * MM + 2],
                                        double (&out)[2 * MM + 2]) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  double sg[n1], df[n1];
#pragma unroll
  for (int l = 0; l < n1; ++l) {
    sg[l] = lr[l] + lr[n1 + l];
    df[l] = lr[l] - lr[n1 + l];
  }
#pragma unroll
  for (int r = 0; r < n; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < n1; ++l) acc = fma(P.M[r * n + l], ((r - l) & 1) ? df[l] : sg[l], acc);
    out[r] = acc;
  }
}

// the row-pair limits as compile-time constants (a constexpr table indexed by
// an unrolled loop variable would be materialised in local memory)
template <int MM, int KIND, int K, int J>
struct RowLim {
  static constexpr int v = Regions<MM, KIND>{}.row_pair(K, J);
  static constexpr int last = Regions<MM, KIND>{}.last_row(K);
};

// acc[J] (row 2J + t) += ap[IX] (*) X[row - IX] when the row is in R_K
template <int MM, int KIND, int K, int IX, int J>
__device__ __forceinline__ void product_row(const double (&av)[2 * MM + 4], const double* X, int t,
                                            double (&acc)[MM + 1][2 * MM + 2]) {
  using S = Shape<MM>;
  constexpr int Lj = RowLim<MM, KIND, K, J>::v, last = RowLim<MM, KIND, K, J>::last;
  if constexpr (Lj >= 0 && 2 * J + 1 >= IX) {
    const int r = 2 * J + t;
    if (r >= IX && r <= last) {
      double xv[S::n + 2];
#pragma unroll
      for (int i = 0; i <= Lj; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(X + (r - IX) * S::RS + i);
        xv[i] = v.x;
        xv[i + 1] = v.y;
      }
#pragma unroll
      for (int qy = 0; qy <= Lj; ++qy)
#pragma unroll
        for (int iy = 0; iy <= qy; ++iy) acc[J][qy] = fma(av[iy], xv[qy - iy], acc[J][qy]);
    }
  }
}

template <int MM, int KIND, int K, int IX, int... J>
__device__ __forceinline__ void product_rows(std::integer_sequence<int, J...>, const double (&av)[2 * MM + 4],
                                             const double* X, int t, double (&acc)[MM + 1][2 * MM + 2]) {
  (product_row<MM, KIND, K, IX, J>(av, X, t, acc), ...);
}

// for IX = 0.. : load ap row IX once, apply it to every row of the thread
template <int MM, int KIND, int K, int IX>
__device__ __forceinline__ void product_ix(const double* A, const double* X, int t,
                                           double (&acc)[MM + 1][2 * MM + 2]) {
  using S = Shape<MM>;
  constexpr int last = RowLim<MM, KIND, K, 0>::last;
  if constexpr (IX <= last) {
    constexpr int LA = RowLim<MM, KIND, K, IX / 2>::v;  // widest row that uses ap row IX
    double av[S::n + 2];
#pragma unroll
    for (int i = 0; i <= LA; i += 2) {
      const double2 v = *reinterpret_cast<const double2*>(A + IX * S::RS + i);
      av[i] = v.x;
      av[i + 1] = v.y;
    }
    product_rows<MM, KIND, K, IX>(std::make_integer_sequence<int, S::NJ>{}, av, X, t, acc);
    product_ix<MM, KIND, K, IX + 1>(A, X, t, acc);
  }
}

template <int MM, int KIND, int K>
__device__ __forceinline__ void product(const double* A, const double* X, int t, double (&acc)[MM + 1][2 * MM + 2]) {
  constexpr int n = 2 * MM + 2;
#pragma unroll
  for (int j = 0; j <= MM; ++j)
#pragma unroll
    for (int q = 0; q < n; ++q) acc[j][q] = 0.0;
  product_ix<MM, KIND, K, 0>(A, X, t, acc);
}

// ---- separable coefficient (hlf_set_coeff_separable): ap = -c0 e_0 - c1 sx (x) sy,
// so ap (.) X = -c0 X - c1 Sx(Sy(X)): Y = Sy(X) row by row (causal
// convolution with sy along qy, thread-local), then each output row mixes the
// rows below it with sx (all rows: Y goes through shared memory, buffer A)
template <int MM, int KIND, int K, int J>
__device__ __forceinline__ void sep_ysweep_row(const double (&sy)[2 * MM + 2], const double* X, double* Y, int t) {
  using S = Shape<MM>;
  constexpr int Lj = RowLim<MM, KIND, K, J>::v, last = RowLim<MM, KIND, K, J>::last;
  if constexpr (Lj >= 0) {
    const int r = 2 * J + t;
    if (r <= last) {
      double xv[S::n + 2], yv[S::n + 2];
#pragma unroll
      for (int i = 0; i <= Lj; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(X + r * S::RS + i);
        xv[i] = v.x;
        xv[i + 1] = v.y;
      }
#pragma unroll
      for (int qy = 0; qy <= Lj; ++qy) {
        double y = 0.0;
#pragma unroll
        for (int b = 0; b <= qy; ++b) y = fma(sy[b], xv[qy - b], y);
        yv[qy] = y;
      }
      yv[Lj + 1] = 0.0;
#pragma unroll
      for (int i = 0; i <= Lj; i += 2) *reinterpret_cast<double2*>(Y + r * S::RS + i) = make_double2(yv[i], yv[i + 1]);
    }
  }
}

template <int MM, int KIND, int K, int J>
__device__ __forceinline__ void sep_xcomb_row(const double (&nsx)[2 * MM + 2], double c0, const double* X,
                                              const double* Y, int t, double (&acc)[MM + 1][2 * MM + 2]) {
  using S = Shape<MM>;
  constexpr int Lj = RowLim<MM, KIND, K, J>::v, last = RowLim<MM, KIND, K, J>::last;
  if constexpr (Lj >= 0) {
    const int r = 2 * J + t;
    if (r <= last) {
#pragma unroll
      for (int i = 0; i <= Lj; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(X + r * S::RS + i);
        acc[J][i] = -c0 * v.x;
        if (i + 1 <= Lj) acc[J][i + 1 <= Lj ? i + 1 : i] = -c0 * v.y;
      }
#pragma unroll
      for (int a = 0; a <= 2 * J + 1; ++a) {
        if (a > r) break;
        const double* yr = Y + (r - a) * S::RS;
#pragma unroll
        for (int i = 0; i <= Lj; i += 2) {
          const double2 v = *reinterpret_cast<const double2*>(yr + i);
          acc[J][i] = fma(nsx[a], v.x, acc[J][i]);
          if (i + 1 <= Lj) acc[J][i + 1 <= Lj ? i + 1 : i] = fma(nsx[a], v.y, acc[J][i + 1 <= Lj ? i + 1 : i]);
        }
      }
    }
  }
}

template <int MM, int KIND, int K, int... J>
__device__ __forceinline__ void product_sep_(std::integer_sequence<int, J...>, const double (&nsx)[2 * MM + 2],
                                             const double (&sy)[2 * MM + 2], double c0, double* A, const double* X,
                                             int t, double (&acc)[MM + 1][2 * MM + 2]) {
  (sep_ysweep_row<MM, KIND, K, J>(sy, X, A, t), ...);
  __syncwarp();
  (sep_xcomb_row<MM, KIND, K, J>(nsx, c0, X, A, t, acc), ...);
}

// X_K = av Lap P_{K-2} on thread-row J (row r + 2 = acc[J + 1])
template <int MM, int KIND, int K, int J>
__device__ __forceinline__ void lap_row(double (&acc)[MM + 1][2 * MM + 2], int t, double c) {
  constexpr int n = 2 * MM + 2, NJ = MM + 1;
  constexpr int Lj = RowLim<MM, KIND, K, J>::v;
  if constexpr (Lj >= 0) {
    const int r = 2 * J + t;
    const double fx = static_cast<double>((r + 1) * (r + 2));
#pragma unroll
    for (int qy = 0; qy <= Lj; ++qy) {
      double v = J + 1 < NJ ? acc[J + 1 < NJ ? J + 1 : J][qy] * fx : 0.0;
      if (qy + 2 < n) v = fma(acc[J][qy + 2 < n ? qy + 2 : qy], static_cast<double>((qy + 1) * (qy + 2)), v);
      acc[J][qy] = v * c;
    }
  }
}

template <int MM, int KIND, int K, int J>
__device__ __forceinline__ void store_row(const double (&acc)[MM + 1][2 * MM + 2], double* X, int t) {
  using S = Shape<MM>;
  constexpr int Lj = RowLim<MM, KIND, K, J>::v, last = RowLim<MM, KIND, K, J>::last;
  if constexpr (Lj >= 0) {
    const int r = 2 * J + t;
    if (r <= last) {
#pragma unroll
      for (int i = 0; i <= Lj; i += 2)
        *reinterpret_cast<double2*>(X + r * S::RS + i) =
            make_double2(acc[J][i], i + 1 < S::n ? acc[J][i + 1 < S::n ? i + 1 : i] : 0.0);
    }
  }
}

// Lap in registers (ascending rows: row J + 1 is still P_{K-2} when row J
// reads it), then the store once the partner has finished reading X
template <int MM, int KIND, int K, int... J>
__device__ __forceinline__ void laplacian_store_(std::integer_sequence<int, J...>, double (&acc)[MM + 1][2 * MM + 2],
                                                 double* X, int t, double c) {
  (lap_row<MM, KIND, K, J>(acc, t, c), ...);
  __syncwarp();
  (store_row<MM, KIND, K, J>(acc, X, t), ...);
  __syncwarp();
}

template <int MM, int KIND, int K>
__device__ __forceinline__ void laplacian_store(double (&acc)[MM + 1][2 * MM + 2], double* X, int t, double c) {
  laplacian_store_<MM, KIND, K>(std::make_integer_sequence<int, MM + 1>{}, acc, X, t, c);
}

// the ap operand: stored jets in A (SEP = false) or the separable data
template <int MM, bool SEP>
struct Coef {
  double* A;                // stored jet rows (SEP: scratch for Sy(X))
  double nsx[2 * MM + 2];   // -c1 sx (SEP)
  double sy[2 * MM + 2];    // sy (SEP)
  double c0;
};

template <int MM, int KIND, int K, bool SEP>
__device__ __forceinline__ void product_any(Coef<MM, SEP>& C, const double* X, int t,
                                            double (&acc)[MM + 1][2 * MM + 2]) {
  if constexpr (SEP)
    product_sep_<MM, KIND, K>(std::make_integer_sequence<int, MM + 1>{}, C.nsx, C.sy, C.c0, C.A, X, t, acc);
  else
    product<MM, KIND, K>(C.A, X, t, acc);
}

// PRE levels K = 1, 3, .., n - 1: P_K = ap (.) X_K, target += w_K P_K,
// X_{K+2} = av Lap P_K
template <int MM, int K, bool SEP>
__device__ __forceinline__ void pre_levels(const HalfParams& P, Coef<MM, SEP>& A, double* X, int t, double c,
                                           double (&acc)[MM + 1][2 * MM + 2], double (&tgt)[MM / 2 + 1][MM + 1]) {
  product_any<MM, PRE, K>(A, X, t, acc);
#pragma unroll
  for (int s = 0; s <= MM / 2; ++s)
    if (2 * s + t <= MM) {
#pragma unroll
      for (int b = 0; b <= MM; ++b) tgt[s][b] = fma(P.w[K], acc[s][b], tgt[s][b]);
    }
  if constexpr (K + 2 < 2 * MM + 2) {
    laplacian_store<MM, PRE, K + 2>(acc, X, t, c);
    pre_levels<MM, K + 2, SEP>(P, A, X, t, c, acc, tgt);
  }
}

// VEL levels K = 0, 2, .., n - 2: target_c += w_{K+1} av d_c P_K on the
// target rows (d_x reads row r + 1, the partner's), then X_{K+2} = av Lap P_K
// and P_{K+2} = ap (.) X_{K+2}
template <int MM, int K, bool SEP>
__device__ __forceinline__ void vel_levels(const HalfParams& P, Coef<MM, SEP>& A, double* X, int t, double c,
                                           double inv_h, double (&acc)[MM + 1][2 * MM + 2],
                                           double (&tgt)[2][MM / 2 + 1][MM + 1]) {
  constexpr int NJ = MM + 1;
  const double wa = P.w[K + 1] * P.av * inv_h;
#pragma unroll
  for (int s = 0; s <= MM / 2; ++s) {
    const double fxr = static_cast<double>(2 * s + t + 1) * wa;
#pragma unroll
    for (int b = 0; b <= MM; ++b) {
      // row 2s + t + 1 is the partner's acc[s + t]; we send it our acc[s + 1 - t]
      const double hi = s + 1 < NJ ? acc[s + 1][b] : 0.0;
      const double up = __shfl_xor_sync(FULL, t ? acc[s][b] : hi, 1);
      if (2 * s + t <= MM) {
        tgt[0][s][b] = fma(up, fxr, tgt[0][s][b]);
        tgt[1][s][b] = fma(acc[s][b + 1], static_cast<double>(b + 1) * wa, tgt[1][s][b]);
      }
    }
  }
  if constexpr (K + 2 < 2 * MM + 1) {
    laplacian_store<MM, VEL, K + 2>(acc, X, t, c);
    product_any<MM, VEL, K + 2>(A, X, t, acc);
    vel_levels<MM, K + 2, SEP>(P, A, X, t, c, inv_h, acc, tgt);
  }
}

template <int MM, int KIND, bool SEP>
__global__ void __launch_bounds__(NTHREADS) var2d(const __grid_constant__ HalfParams P) {
  using S = Shape<MM>;
  constexpr int n1 = S::n1, n = S::n, NJ = S::NJ, NS = S::NS;
  constexpr int NSRC = KIND == VEL ? 1 : 2;
  constexpr int NOUT = KIND == VEL ? 2 : 1;
  extern __shared__ double smem[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane >> 1;
  const int t = lane & 1;
  const int64_t total = static_cast<int64_t>(P.tNx) * P.tNy;
  const int64_t cell = static_cast<int64_t>(blockIdx.x) * S::CPC + warp * S::CPW + q;
  const bool live = cell < total;
  double* A = smem + (warp * S::CPW + q) * S::CS;
  double* X = A + S::AS;

  const int tx = live ? static_cast<int>(cell % P.tNx) : 0;
  const int ty = live ? static_cast<int>(cell / P.tNx) : 0;
  const int64_t tnode = static_cast<int64_t>(ty) * P.tNx + tx;

  Coef<MM, SEP> coef;
  coef.A = A;
  if constexpr (SEP) {
    // ap = -(c0 + c1 sin(w_x x + ph_x) sin(w_y y + ph_y)) at the target node:
    // the reference's sin_jet (jet.cpp:65-74) per axis
    const double xx = P.sep_x0[0] + tx * P.h, yy = P.sep_x0[1] + ty * P.h;
    double sn, cs;
    sincos(P.sep[2] * xx + P.sep[5], &sn, &cs);
    double f = 1.0;
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const int r4 = k & 3;
      coef.nsx[k] = -P.sep[1] * f * (r4 == 0 ? sn : (r4 == 1 ? cs : (r4 == 2 ? -sn : -cs)));
      f = f * (P.sep[2] * P.h) / (k + 1);
    }
    sincos(P.sep[3] * yy + P.sep[6], &sn, &cs);
    f = 1.0;
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const int r4 = k & 3;
      coef.sy[k] = f * (r4 == 0 ? sn : (r4 == 1 ? cs : (r4 == 2 ? -sn : -cs)));
      f = f * (P.sep[3] * P.h) / (k + 1);
    }
    coef.c0 = P.sep[0];
  } else {
    // ap jet rows t, t + 2, .. -> A  ([E][y][x] planes, e = qx n + qy)
    const double* ap = P.coeff + tnode;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int r = 2 * j + t;
#pragma unroll
      for (int qy = 0; qy < n; qy += 2) {
        const double a0 = __ldg(ap + (r * n + qy) * P.c_coef);
        const double a1 = __ldg(ap + (r * n + qy + 1) * P.c_coef);
        *reinterpret_cast<double2*>(A + r * S::RS + qy) = make_double2(a0, a1);
      }
    }
  }
  // corner nodes and wall flips (as half_generic): VEL corners t + side,
  // PRE corners t - 1 + side (mirrored ghosts across reflective walls)
  int64_t cx[2], cy[2];
  int fx[2] = {0, 0}, fy[2] = {0, 0};
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    int qx = KIND == VEL ? tx + side : tx - 1 + side;
    int qy = KIND == VEL ? ty + side : ty - 1 + side;
    if (P.bnd[0] == 0) {
      if (qx >= P.K[0]) qx -= P.K[0];
      if (qx < 0) qx += P.K[0];
    } else if (KIND == PRE) {
      if (qx < 0) { qx = 0; fx[side] = 1; }
      else if (qx >= P.K[0]) { qx = P.K[0] - 1; fx[side] = 1; }
    }
    if (P.bnd[1] == 0) {
      if (qy >= P.K[1]) qy -= P.K[1];
      if (qy < 0) qy += P.K[1];
    } else if (KIND == PRE) {
      if (qy < 0) { qy = 0; fy[side] = 1; }
      else if (qy >= P.K[1]) { qy = P.K[1] - 1; fy[side] = 1; }
    }
    cx[side] = qx;
    cy[side] = static_cast<int64_t>(qy) * P.sNx;
  }

  // target rows 2s + t <= m (s < NS)
  double tgt[NOUT][NS][n1];
#pragma unroll
  for (int c = 0; c < NOUT; ++c)
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int b = 0; b < n1; ++b)
        tgt[c][s][b] = 2 * s + t <= MM ? P.dst[c][tnode + ((2 * s + t) * n1 + b) * P.t_coef] : 0.0;

  const double inv_h = P.inv_h;
  double acc[NJ][n];  // this thread's rows of the current level
  // ---- reconstruction (reconstruct_cell_2d, interpolation.cpp:77-113) ----
  const double sgn_t = t ? -1.0 : 1.0;  // (-1)^t
  double Mt[NJ][n1];                     // this thread's rows of M_L
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int l = 0; l < n1; ++l) Mt[j][l] = t ? P.M[(2 * j + 1) * n + l] : P.M[2 * j * n + l];
#pragma unroll
  for (int comp = 0; comp < NSRC; ++comp) {
    const double* src = P.src[comp];
    // x sweep in registers: Y[j][col] (row 2j + t) = sum_l M[2j+t][l] u_l with
    // u_l = L_l + (-1)^{t+l} R_l of the stacked column col = (side y, order b)
    double Y[NJ][n];
#pragma unroll
    for (int sy = 0; sy < 2; ++sy) {
      double sgy_c = 1.0;  // mirror signs (half_generic): per flipped axis
      if (KIND == PRE && fy[sy]) sgy_c = comp != 1 ? -1.0 : 1.0;  // (-1)^order, and -1 for the
#pragma unroll                                                      // tangential velocity
      for (int b = 0; b < n1; ++b) {
        const double sgy = (KIND == PRE && fy[sy] && (b & 1)) ? -sgy_c : sgy_c;
        double lr[n];
#pragma unroll
        for (int sx = 0; sx < 2; ++sx) {
          const double* base = src + cy[sy] + cx[sx];
          double sgx = 1.0;
          if (KIND == PRE && fx[sx]) sgx = comp != 0 ? -1.0 : 1.0;
#pragma unroll
          for (int a = 0; a < n1; ++a) {
            const double sa = (KIND == PRE && fx[sx] && (a & 1)) ? -sgx : sgx;
            lr[sx * n1 + a] = sa * sgy * __ldg(base + (a * n1 + b) * P.s_coef);
          }
        }
        double u[n1];
#pragma unroll
        for (int l = 0; l < n1; ++l) u[l] = fma((l & 1) ? -sgn_t : sgn_t, lr[n1 + l], lr[l]);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          double y = 0.0;
#pragma unroll
          for (int l = 0; l < n1; ++l) y = fma(Mt[j][l], u[l], y);
          Y[j][sy * n1 + b] = y;
        }
      }
    }
    // y sweep of the thread's rows
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      double out[n];
      apply_m<MM>(P, Y[j], out);
      if (KIND == VEL || comp == 0) {
#pragma unroll
        for (int c2 = 0; c2 < n; ++c2) acc[j][c2] = out[c2];
      } else {
        // div V_0, y term: d_y V_y[r][qy] = V_y[r][qy + 1] (qy + 1) / h
#pragma unroll
        for (int c2 = 0; c2 + 1 < n; ++c2)
          acc[j][c2] = fma(out[c2 + 1], static_cast<double>(c2 + 1) * inv_h, acc[j][c2]);
      }
    }
    if (KIND == PRE && comp == 0) {
      // div V_0, x term: d_x V_x[r] = V_x[r + 1] (r + 1) / h; row r + 1 is the
      // partner's acc[j + t] (zero past row n - 1), we send it acc[j + 1 - t];
      // ascending j keeps every row until it has been sent
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const double f = static_cast<double>(2 * j + t + 1) * inv_h;
#pragma unroll
        for (int c2 = 0; c2 < n; ++c2) {
          const double hi = j + 1 < NJ ? acc[j + 1][c2] : 0.0;
          const double up = __shfl_xor_sync(FULL, t ? acc[j][c2] : hi, 1);
          acc[j][c2] = up * f;
        }
      }
    }
    __syncwarp();
  }

  const double lap_c = P.av * inv_h * inv_h;
  if constexpr (KIND == PRE) {
    // X_1 = div V_0 -> shared memory (the last y sweep has read X: synced above)
    constexpr int last1 = RowLim<MM, PRE, 1, 0>::last;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int r = 2 * j + t;
      if (r <= last1) {
#pragma unroll
        for (int c2 = 0; c2 < n; c2 += 2)
          *reinterpret_cast<double2*>(X + r * S::RS + c2) = make_double2(acc[j][c2], acc[j][c2 + 1]);
      }
    }
    __syncwarp();
    pre_levels<MM, 1, SEP>(P, coef, X, t, lap_c, acc, tgt[0]);
  } else {
    vel_levels<MM, 0, SEP>(P, coef, X, t, lap_c, inv_h, acc, tgt);
  }

  // in-place store + finite flag (check_finite, stepper1d.cpp:121-129)
  if (live) {
    bool bad = false;
#pragma unroll
    for (int c = 0; c < NOUT; ++c)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (2 * s + t <= MM) {
#pragma unroll
          for (int b = 0; b < n1; ++b) {
            bad |= !isfinite(tgt[c][s][b]);
            P.dst[c][tnode + ((2 * s + t) * n1 + b) * P.t_coef] = tgt[c][s][b];
          }
        }
    if (bad && P.step >= 0) report_nonfinite(P.flag, P.step);
  }
}

template <int MM>
int launch_m(HalfKind kind, const HalfParams& p, cudaStream_t st) {
  using S = Shape<MM>;
  const int64_t total = static_cast<int64_t>(p.tNx) * p.tNy;
  const int64_t blocks = (total + S::CPC - 1) / S::CPC;
  if (blocks > 0x7fffffff) return -2;
  static std::atomic<unsigned long long> vel_ok{0}, pre_ok{0}, vel_sep{0}, pre_sep{0};
  if (p.sep_on) {
    if (kind == VEL) ensure_smem_opt_in(var2d<MM, VEL, true>, S::SMEM, vel_sep);
    else ensure_smem_opt_in(var2d<MM, PRE, true>, S::SMEM, pre_sep);
    if (kind == VEL)
      var2d<MM, VEL, true><<<static_cast<unsigned>(blocks), NTHREADS, S::SMEM, st>>>(p);
    else
      var2d<MM, PRE, true><<<static_cast<unsigned>(blocks), NTHREADS, S::SMEM, st>>>(p);
    return 1;
  }
  if (kind == VEL) ensure_smem_opt_in(var2d<MM, VEL, false>, S::SMEM, vel_ok);
  else ensure_smem_opt_in(var2d<MM, PRE, false>, S::SMEM, pre_ok);
  if (kind == VEL)
    var2d<MM, VEL, false><<<static_cast<unsigned>(blocks), NTHREADS, S::SMEM, st>>>(p);
  else
    var2d<MM, PRE, false><<<static_cast<unsigned>(blocks), NTHREADS, S::SMEM, st>>>(p);
  return 1;
}

}  // namespace
}  // namespace v2d

bool var2d_supported(int m) { return m >= 1 && m <= 4; }

int launch_half_var2d(int m, HalfKind kind, const HalfParams& p, cudaStream_t st) {
  switch (m) {
    case 1: return v2d::launch_m<1>(kind, p, st);
    case 2: return v2d::launch_m<2>(kind, p, st);
    case 3: return v2d::launch_m<3>(kind, p, st);
    case 4: return v2d::launch_m<4>(kind, p, st);
    default: return -1;
  }
}

}  // namespace hlfk
