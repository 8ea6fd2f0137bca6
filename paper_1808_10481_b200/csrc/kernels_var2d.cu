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
// Layout: G = m + 1 threads ("quad" at m = 3) per cell, 32 / G cells per warp,
// 4 warps per CTA, no inter-warp sharing (only __syncwarp).  Each cell owns
// three n x n jets in shared memory (ap, X = the derivative term, P = the
// level), rows padded to n + 2 doubles; thread t owns jet rows t and
// n - 1 - t, so the target rows 0..m are one per thread.  The product of a
// row is a sum of 1D causal convolutions of ap rows with X rows (rows in
// registers, LDS.128), the reconstruction uses the sum/difference form of M
// (M_R = diag((-1)^r) M_L diag((-1)^l), interpolation.cpp:29-48).
#include <cstring>

#include "hlf_internal.cuh"

namespace hlfk {
namespace v2d {
namespace {

constexpr int NTHREADS = 128;

template <int MM>
struct Shape {
  static constexpr int n1 = MM + 1, n = 2 * MM + 2, G = MM + 1;
  // Bank mapping: LDS.128 serves eight 16 B slots per wavefront.  Rows are an
  // odd number of slots apart (a cell's threads read distinct rows) and cells
  // an odd number of slots apart too (the broadcast ap rows of the 8 cells of
  // a warp and the 32 distinct X rows then spread evenly over the slots).
  static constexpr int RS = ((n + 2) / 2) % 2 ? n + 2 : n + 4;  // padded row (doubles)
  static constexpr int AS = n * RS;                              // one jet
  static constexpr int CS = (3 * AS + 15) / 16 * 16 + 2;         // cell stride: 16 B mod 128 B
  static constexpr int CPW = 32 / G;                      // cells per warp
  static constexpr int SPW = CPW + (32 % G ? 1 : 0);      // + a dummy slot for idle lanes
  static constexpr int CPC = CPW * (NTHREADS / 32);
  static constexpr int SMEM = (NTHREADS / 32) * SPW * CS * 8;
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
  __host__ __device__ constexpr int lo(int k) const { return lim[k][0]; }
  __host__ __device__ constexpr int hi(int k) const { return lim[k][n / 2]; }
  __host__ __device__ constexpr int last_row(int k) const {
    int r = -1;
    for (int q = 0; q < n; ++q)
      if (lim[k][q] >= 0) r = q;
    return r;
  }
};

// row-vector loads of L + 1 doubles (pairs; RS = n + 2 keeps the pad in range)
template <int L>
__device__ __forceinline__ void load_row(double (&v)[L + 2], const double* p) {
#pragma unroll
  for (int i = 0; i <= L; i += 2) {
    const double2 t = *reinterpret_cast<const double2*>(p + i);
    v[i] = t.x;
    v[i + 1] = t.y;
  }
}

// acc[qy] += sum_{iy <= qy} a[iy] x[qy - iy], qy <= L (truncated 1D product)
template <int L>
__device__ __forceinline__ void conv_row(double (&acc)[L + 1], const double* a, const double* x) {
  double av[L + 2], xv[L + 2];
  load_row<L>(av, a);
  load_row<L>(xv, x);
#pragma unroll
  for (int qy = 0; qy <= L; ++qy)
#pragma unroll
    for (int iy = 0; iy <= qy; ++iy) acc[qy] = fma(av[iy], xv[qy - iy], acc[qy]);
}

template <int L>
__device__ __forceinline__ void store_row(double* p, const double (&v)[L + 1]) {
#pragma unroll
  for (int i = 0; i <= L; ++i) p[i] = v[i];
}

// one level's product P = ap (.) X on the rows this thread owns
template <int MM, int KIND, int K>
__device__ __forceinline__ void product(const HalfParams& P, const double* A, const double* X, double* Pj,
                                        int t, double (&tgt)[MM + 1]) {
  using S = Shape<MM>;
  constexpr Regions<MM, KIND> R{};
  constexpr int Llo = R.lo(K), Lhi = R.hi(K), last = R.last_row(K);
  {
    double acc[Llo + 1];
#pragma unroll
    for (int i = 0; i <= Llo; ++i) acc[i] = 0.0;
    for (int ix = 0; ix <= t; ++ix) conv_row<Llo>(acc, A + ix * S::RS, X + (t - ix) * S::RS);
    store_row<Llo>(Pj + t * S::RS, acc);
    if constexpr (KIND == PRE && (K & 1)) {
#pragma unroll
      for (int b = 0; b <= MM; ++b) tgt[b] = fma(P.w[K], acc[b], tgt[b]);
    }
  }
  if constexpr (Lhi >= 0) {
    const int r = S::n - 1 - t;
    if (r <= last) {
      double acc[Lhi + 1];
#pragma unroll
      for (int i = 0; i <= Lhi; ++i) acc[i] = 0.0;
      for (int ix = 0; ix <= r; ++ix) conv_row<Lhi>(acc, A + ix * S::RS, X + (r - ix) * S::RS);
      store_row<Lhi>(Pj + r * S::RS, acc);
    }
  }
}

// X = av Lap P on one row r (qy <= L): (P[r+2][qy] (r+1)(r+2) + P[r][qy+2] (qy+1)(qy+2)) av / h^2
template <int MM, int L>
__device__ __forceinline__ void lap_row(const double* Pj, double* X, int r, double c) {
  using S = Shape<MM>;
  constexpr int n = S::n;
  constexpr int LO = L + 2 < n - 1 ? L + 2 : n - 1;  // own-row entries read
  double own[LO + 2];
  load_row<LO>(own, Pj + r * S::RS);
  double out[L + 1];
  const double fx = static_cast<double>((r + 1) * (r + 2));
  if (r + 2 < n) {
    double up[L + 2];
    load_row<L>(up, Pj + (r + 2) * S::RS);
#pragma unroll
    for (int qy = 0; qy <= L; ++qy) out[qy] = up[qy] * fx;
  } else {
#pragma unroll
    for (int qy = 0; qy <= L; ++qy) out[qy] = 0.0;
  }
#pragma unroll
  for (int qy = 0; qy <= L; ++qy)
    if (qy + 2 < n) out[qy] = fma(own[qy + 2], static_cast<double>((qy + 1) * (qy + 2)), out[qy]);
#pragma unroll
  for (int qy = 0; qy <= L; ++qy) out[qy] *= c;
  store_row<L>(X + r * S::RS, out);
}

template <int MM, int KIND, int K>
__device__ __forceinline__ void laplacian(const double* Pj, double* X, int t, double c) {
  using S = Shape<MM>;
  constexpr Regions<MM, KIND> R{};
  constexpr int Llo = R.lo(K), Lhi = R.hi(K), last = R.last_row(K);
  lap_row<MM, Llo>(Pj, X, t, c);
  if constexpr (Lhi >= 0) {
    const int r = S::n - 1 - t;
    if (r <= last) lap_row<MM, Lhi>(Pj, X, r, c);
  }
}

// PRE levels K = 1, 3, .., n - 1: P_K = ap (.) X_K, target += w_K P_K,
// X_{K+2} = av Lap P_K
template <int MM, int K>
__device__ __forceinline__ void pre_levels(const HalfParams& P, const double* A, double* X, double* Pj, int t,
                                           double c, double (&tgt)[MM + 1]) {
  product<MM, PRE, K>(P, A, X, Pj, t, tgt);
  if constexpr (K + 2 < 2 * MM + 2) {
    __syncwarp();
    laplacian<MM, PRE, K + 2>(Pj, X, t, c);
    __syncwarp();
    pre_levels<MM, K + 2>(P, A, X, Pj, t, c, tgt);
  }
}

// VEL levels K = 0, 2, .., n - 2: target_c += w_{K+1} av d_c P_K on the
// target rows, then X_{K+2} = av Lap P_K and P_{K+2} = ap (.) X_{K+2}
template <int MM, int K>
__device__ __forceinline__ void vel_levels(const HalfParams& P, const double* A, double* X, double* Pj, int t,
                                           double c, double inv_h, double (&tgt)[2][MM + 1]) {
  using S = Shape<MM>;
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  const double wa = P.w[K + 1] * P.av * inv_h;
  double up[n1 + 1], own[n1 + 3];
  load_row<n1 - 1>(up, Pj + (t + 1) * S::RS);
  load_row<n1 + 1>(own, Pj + t * S::RS);
  const double fxr = static_cast<double>(t + 1) * wa;
#pragma unroll
  for (int b = 0; b < n1; ++b) {
    tgt[0][b] = fma(up[b], fxr, tgt[0][b]);
    tgt[1][b] = fma(own[b + 1], static_cast<double>(b + 1) * wa, tgt[1][b]);
  }
  if constexpr (K + 2 < n - 1) {
    laplacian<MM, VEL, K + 2>(Pj, X, t, c);
    __syncwarp();
    double unused[MM + 1];
    product<MM, VEL, K + 2>(P, A, X, Pj, t, unused);
    __syncwarp();
    vel_levels<MM, K + 2>(P, A, X, Pj, t, c, inv_h, tgt);
  }
}

// sum/difference form of one M application: out[r] = sum_l M[r][l] (L_l + (-1)^{r-l} R_l)
template <int MM>
__device__ __forceinline__ void apply_m(const HalfParams& P, const double (&lr)[2 * MM + 2], double (&out)[2 * MM + 2]) {
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

template <int MM, int KIND>
__global__ void __launch_bounds__(NTHREADS) var2d(const __grid_constant__ HalfParams P) {
  using S = Shape<MM>;
  constexpr int n1 = S::n1, n = S::n, G = S::G;
  constexpr int NSRC = KIND == VEL ? 1 : 2;
  constexpr int NOUT = KIND == VEL ? 2 : 1;
  extern __shared__ double smem[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane / G;
  const int t = lane - q * G;
  const int64_t total = static_cast<int64_t>(P.tNx) * P.tNy;
  const int64_t cell = static_cast<int64_t>(blockIdx.x) * S::CPC + warp * S::CPW + q;
  const bool live = q < S::CPW && cell < total;
  double* A = smem + (warp * S::SPW + (q < S::CPW ? q : S::CPW)) * S::CS;
  double* X = A + S::AS;
  double* Pj = X + S::AS;

  const int tx = live ? static_cast<int>(cell % P.tNx) : 0;
  const int ty = live ? static_cast<int>(cell / P.tNx) : 0;
  const int64_t tnode = static_cast<int64_t>(ty) * P.tNx + tx;
  const int rl = t, rh = n - 1 - t;

  // ap jet rows rl, rh -> A  ([E][y][x] planes, e = qx n + qy)
  {
    const double* ap = P.coeff + tnode;
#pragma unroll
    for (int qy = 0; qy < n; ++qy) {
      A[rl * S::RS + qy] = __ldg(ap + (rl * n + qy) * P.c_coef);
      A[rh * S::RS + qy] = __ldg(ap + (rh * n + qy) * P.c_coef);
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

  double tgt[NOUT][n1];
#pragma unroll
  for (int c = 0; c < NOUT; ++c)
#pragma unroll
    for (int b = 0; b < n1; ++b) tgt[c][b] = P.dst[c][tnode + (rl * n1 + b) * P.t_coef];

  double vy[2][n];  // PRE: V_y rows rl, rh of the reconstruction
  // ---- reconstruction (reconstruct_cell_2d, interpolation.cpp:77-113) ----
#pragma unroll
  for (int comp = 0; comp < NSRC; ++comp) {
    const double* src = P.src[comp];
    // x sweep of stacked columns rl (sy = 0, b = t) and rh (sy = 1, b = m - t) -> X
#pragma unroll
    for (int side_y = 0; side_y < 2; ++side_y) {
      const int b = side_y == 0 ? t : MM - t;
      const int col = side_y == 0 ? rl : rh;
      double lr[n], out[n];
#pragma unroll
      for (int sx = 0; sx < 2; ++sx) {
        const double* base = src + cy[side_y] + cx[sx];
        // mirror signs (half_generic): per flipped axis (-1)^order, and -1 for
        // the velocity component tangential to that wall
        double sgx = 1.0;
        if (KIND == PRE && fx[sx]) sgx = comp != 0 ? -1.0 : 1.0;
        double sgy = 1.0;
        if (KIND == PRE && fy[side_y]) sgy = ((b & 1) ? -1.0 : 1.0) * (comp != 1 ? -1.0 : 1.0);
#pragma unroll
        for (int a = 0; a < n1; ++a) {
          const double sa = (KIND == PRE && fx[sx] && (a & 1)) ? -sgx : sgx;
          lr[sx * n1 + a] = sa * sgy * __ldg(base + (a * n1 + b) * P.s_coef);
        }
      }
      apply_m<MM>(P, lr, out);
#pragma unroll
      for (int r = 0; r < n; ++r) X[r * S::RS + col] = out[r];
    }
    __syncwarp();
    // y sweep of rows rl, rh
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = h == 0 ? rl : rh;
      double lr[n], out[n];
#pragma unroll
      for (int c = 0; c < n; ++c) lr[c] = X[r * S::RS + c];
      apply_m<MM>(P, lr, out);
      if (KIND == VEL || comp == 0) {
#pragma unroll
        for (int c = 0; c < n; ++c) Pj[r * S::RS + c] = out[c];
      } else {
#pragma unroll
        for (int c = 0; c < n; ++c) vy[h][c] = out[c];
      }
    }
    __syncwarp();
  }

  const double inv_h = P.inv_h;
  const double lap_c = P.av * inv_h * inv_h;
  if constexpr (KIND == PRE) {
    // X_1 = div V_0 on the rows this thread owns (all n entries)
    constexpr Regions<MM, PRE> R{};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = h == 0 ? rl : rh;
      if (h == 1 && r > R.last_row(1)) break;
      double out[n];
      if (r + 1 < n) {
        const double f = static_cast<double>(r + 1);
#pragma unroll
        for (int c = 0; c < n; ++c) out[c] = Pj[(r + 1) * S::RS + c] * f;
      } else {
#pragma unroll
        for (int c = 0; c < n; ++c) out[c] = 0.0;
      }
#pragma unroll
      for (int c = 0; c + 1 < n; ++c) out[c] = fma(vy[h][c + 1], static_cast<double>(c + 1), out[c]);
#pragma unroll
      for (int c = 0; c < n; ++c) X[r * S::RS + c] = out[c] * inv_h;
    }
    __syncwarp();
    pre_levels<MM, 1>(P, A, X, Pj, t, lap_c, tgt[0]);
  } else {
    vel_levels<MM, 0>(P, A, X, Pj, t, lap_c, inv_h, tgt);
  }

  // in-place store + finite flag (check_finite, stepper1d.cpp:121-129)
  if (live) {
    bool bad = false;
#pragma unroll
    for (int c = 0; c < NOUT; ++c)
#pragma unroll
      for (int b = 0; b < n1; ++b) {
        bad |= !isfinite(tgt[c][b]);
        P.dst[c][tnode + (rl * n1 + b) * P.t_coef] = tgt[c][b];
      }
    if (bad && P.step >= 0) atomicMin(P.flag, P.step);
  }
}

template <int MM>
int launch_m(HalfKind kind, const HalfParams& p, cudaStream_t st) {
  using S = Shape<MM>;
  const int64_t total = static_cast<int64_t>(p.tNx) * p.tNy;
  const int64_t blocks = (total + S::CPC - 1) / S::CPC;
  if (blocks > 0x7fffffff) return -2;
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(var2d<MM, VEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
    cudaFuncSetAttribute(var2d<MM, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
    init = true;
  }
  if (kind == VEL)
    var2d<MM, VEL><<<static_cast<unsigned>(blocks), NTHREADS, S::SMEM, st>>>(p);
  else
    var2d<MM, PRE><<<static_cast<unsigned>(blocks), NTHREADS, S::SMEM, st>>>(p);
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
