// 16-warp tiled 3D half-step kernel for m = 3 (constant coefficients).
//
// Same pipeline as kernels_tiled3d.cu (32 cells along x per CTA, z-marching,
// raw layer -> fused XY -> 2-layer ring -> Z + closed-form CK), reorganised so
// that a thread needs <= 128 registers and the SM runs 16 warps instead of 8
// (the 8-warp kernel is latency-bound: ncu shows the FP64 pipe ~38 % busy,
// stalls dominated by fixed-latency dependencies and shared-memory waits):
//   XY:   task = (l_z, q_x parity, cell half) -> 16 tasks; lane = (cell, source
//         row hi); the lane computes the half x-lines of its row, swaps them
//         with lane ^ 16 and computes the y half-lines of q_y parity hi.
//   Z+CK: warp = (parity class, column half h); each half computes P for 8 of
//         the class's 16 columns and a partial CK sum; the h = 0 warp adds its
//         partial into the staged target, a named barrier hands it to the
//         h = 1 warp, which adds its own and stores.
#include <cstring>

#include "hlf_internal.cuh"

namespace hlfk {
namespace v5 {
namespace {

constexpr int MM = 3;
constexpr int n1 = MM + 1, n = 2 * MM + 2, F = n1 * n1 * n1, nh = n / 2, jh = (n1 + 1) / 2;
constexpr int TXC = 32;
constexpr int RAWX = TXC + 1;
constexpr int NWARP = 16;
constexpr int NTHREADS = NWARP * 32;
constexpr int ZC = 32;
constexpr int kMaxB = 20;
constexpr int RAW = F * 2 * RAWX;
constexpr int RING = n * n * n1 * TXC;
constexpr int RAW_PER_THREAD = (RAW + NTHREADS - 1) / NTHREADS;

struct TParams {
  double ML[kMaxN * (kMaxM + 1)];  // s! * M[s][l] (left block)
  double GM[kMaxB];                // G_k * k!/b!
  const double* src;
  double* dst[3];
  int64_t s_layer, s_plane, t_layer, t_plane;
  int sNx, sNy, tNx, tNy, tNz, t_zoff;
  int K[2], bnd[2];
  int pre, comp, step;
  int* flag;
};

constexpr int bindex(int b0, int b1, int b2, int mm) {
  int idx = 0;
  for (int a0 = 0; a0 <= mm; ++a0)
    for (int a1 = 0; a1 <= mm - a0; ++a1)
      for (int a2 = 0; a2 <= mm - a0 - a1; ++a2) {
        if (a0 == b0 && a1 == b1 && a2 == b2) return idx;
        ++idx;
      }
  return -1;
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void pair_barrier(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id)); }

#include "tiled3d_v5_gen.cuh"

__device__ __forceinline__ double ifact(int k) { return k <= 1 ? 1.0 : (k == 2 ? 0.5 : 1.0 / 6.0); }

template <int NT>
__global__ void __launch_bounds__(NTHREADS, 1) tiled3d_v5(const __grid_constant__ TParams P) {
  extern __shared__ __align__(16) double smem[];
  double* raw = smem;
  double* ring0 = raw + RAW;
  double* ring1 = ring0 + RING;
  double* tgs = ring1 + RING;  // [t][f][cell]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TXC;
  const int ty = blockIdx.y;
  const int k0 = blockIdx.z * ZC;
  const int k1 = min(k0 + ZC, P.tNz);
  if (k0 >= k1) return;

  // raw-element offsets (constant over layers) and mirror signs
  int off[RAW_PER_THREAD];
  unsigned negmask = 0;
#pragma unroll
  for (int t = 0; t < RAW_PER_THREAD; ++t) {
    const int e = tid + t * NTHREADS;
    off[t] = -1;
    if (e >= RAW) continue;
    const int f = e / (2 * RAWX);
    const int r = e - f * 2 * RAWX;
    const int sy = r / RAWX, sx = r - sy * RAWX;
    int q0 = x0 + sx - P.pre, q1 = ty + sy - P.pre;
    bool neg = false;
    const int ax0 = f / (n1 * n1), ay0 = (f / n1) % n1;
    if (P.bnd[0] == 0) {
      if (q0 >= P.K[0]) q0 -= P.K[0];
      if (q0 < 0) q0 += P.K[0];
    } else if (P.pre && (q0 < 0 || q0 == P.K[0])) {
      q0 = q0 < 0 ? 0 : P.K[0] - 1;
      neg ^= (ax0 & 1) != 0;
      neg ^= P.comp != 0;
    }
    if (q0 >= P.sNx) q0 = P.sNx - 1;
    if (P.bnd[1] == 0) {
      if (q1 >= P.K[1]) q1 -= P.K[1];
      if (q1 < 0) q1 += P.K[1];
    } else if (P.pre && (q1 < 0 || q1 == P.K[1])) {
      q1 = q1 < 0 ? 0 : P.K[1] - 1;
      neg ^= (ay0 & 1) != 0;
      neg ^= P.comp != 1;
    }
    if (q1 >= P.sNy) q1 = P.sNy - 1;
    off[t] = static_cast<int>(f * P.s_plane + static_cast<int64_t>(q1) * P.sNx + q0);
    if (neg) negmask |= 1u << t;
  }

  // XY roles: task = warp = (l_z, q_x parity, cell half); lane = (cell, row)
  const int hi = lane >> 4;
  const int xy_lz = warp >> 2, xy_px = (warp >> 1) & 1, xy_cell = (warp & 1) * 16 + (lane & 15);
  const double g = hi ? -1.0 : 1.0;
  // Z+CK roles: class (PX, PY, PZ) = warp & 7, column half = warp >> 3
  const int w8 = warp & 7, half = warp >> 3;
  const int PX = (w8 >> 2) & 1, PY = (w8 >> 1) & 1, PZ = w8 & 1;
  const int cbase = ((PX * n + PY) * n1) * TXC + lane;
  const bool active = x0 + lane < P.tNx;

  auto issue_raw = [&](int layer) {
    const double* base = P.src + static_cast<int64_t>(layer) * P.s_layer;
#pragma unroll
    for (int t = 0; t < RAW_PER_THREAD; ++t)
      if (off[t] >= 0) cp_async8(raw + tid + t * NTHREADS, base + off[t]);
    cp_async_commit();
  };

  issue_raw(k0);
  double* ro = ring1;
  double* rn = ring0;
  bool bad = false;
#pragma unroll 1
  for (int k = k0 - 1; k < k1; ++k) {
    const bool work = k >= k0;
    cp_async_wait_all();
    if (negmask) {
#pragma unroll
      for (int t = 0; t < RAW_PER_THREAD; ++t)
        if ((negmask >> t) & 1u) raw[tid + t * NTHREADS] = -raw[tid + t * NTHREADS];
    }
    __syncthreads();
    if (work) {
      const int64_t lbase = static_cast<int64_t>(P.t_zoff + k) * P.t_layer + static_cast<int64_t>(ty) * P.tNx + x0;
#pragma unroll 1
      for (int e = tid; e < NT * F * TXC; e += NTHREADS) {
        const int c_ = e & (TXC - 1);
        const int tf = e >> 5;
        const int t = tf / F, f = tf - t * F;
        if (x0 + c_ < P.tNx) cp_async8(tgs + e, P.dst[t] + lbase + f * P.t_plane + c_);
      }
      cp_async_commit();
    }
    {
      // per-lane y coefficients (q_y parity hi), reloaded so they do not stay live
      double cy[nh][n1];
#pragma unroll
      for (int kk = 0; kk < nh; ++kk)
#pragma unroll
        for (int l = 0; l < n1; ++l) {
          const double mv = P.ML[(hi + 2 * kk) * n1 + l];
          cy[kk][l] = (hi && ((hi + l) & 1)) ? -mv : mv;
        }
      const double* rb = raw + (xy_lz * 2 + hi) * RAWX + xy_cell;
      double* wb = rn + (hi * n1 + xy_lz) * TXC + xy_cell;
      if (xy_px) v5_m3_xy_px1(P, rb, wb, cy, g);
      else v5_m3_xy_px0(P, rb, wb, cy, g);
    }
    cp_async_wait_all();
    __syncthreads();
    if (k + 1 < k1) issue_raw(k + 2);

    if (work) {
      double pt[2][nh][nh];
      if (PZ) {
        if (half) v5_m3_z_pz1_h1(P, ro + cbase, rn + cbase, pt);
        else v5_m3_z_pz1_h0(P, ro + cbase, rn + cbase, pt);
      } else {
        if (half) v5_m3_z_pz0_h1(P, ro + cbase, rn + cbase, pt);
        else v5_m3_z_pz0_h0(P, ro + cbase, rn + cbase, pt);
      }
      const int64_t obase = static_cast<int64_t>(P.t_zoff + k) * P.t_layer + static_cast<int64_t>(ty) * P.tNx + x0 + lane;
#pragma unroll 1
      for (int t = 0; t < NT; ++t) {
        const int c = NT == 3 ? t : P.comp;
        double acc[jh][jh][jh];
#pragma unroll
        for (int a = 0; a < jh; ++a)
#pragma unroll
          for (int b = 0; b < jh; ++b)
#pragma unroll
            for (int d = 0; d < jh; ++d) acc[a][b][d] = 0.0;
        const int sh = c == 0 ? 1 - PX : (c == 1 ? 1 - PY : 1 - PZ);
        switch ((c * 2 + sh) * 2 + half) {
          case 0: v5_m3_ck_c0_s0_h0(P, pt, acc); break;
          case 1: v5_m3_ck_c0_s0_h1(P, pt, acc); break;
          case 2: v5_m3_ck_c0_s1_h0(P, pt, acc); break;
          case 3: v5_m3_ck_c0_s1_h1(P, pt, acc); break;
          case 4: v5_m3_ck_c1_s0_h0(P, pt, acc); break;
          case 5: v5_m3_ck_c1_s0_h1(P, pt, acc); break;
          case 6: v5_m3_ck_c1_s1_h0(P, pt, acc); break;
          case 7: v5_m3_ck_c1_s1_h1(P, pt, acc); break;
          case 8: v5_m3_ck_c2_s0_h0(P, pt, acc); break;
          case 9: v5_m3_ck_c2_s0_h1(P, pt, acc); break;
          case 10: v5_m3_ck_c2_s1_h0(P, pt, acc); break;
          default: v5_m3_ck_c2_s1_h1(P, pt, acc); break;
        }
        const int tslot = NT == 3 ? c : 0;
        const int sx = (PX - (c == 0)) & 1, sy = (PY - (c == 1)) & 1, sz = (PZ - (c == 2)) & 1;
        if (half == 0) {
#pragma unroll
          for (int a = 0; a < jh; ++a)
#pragma unroll
            for (int b = 0; b < jh; ++b)
#pragma unroll
              for (int d = 0; d < jh; ++d) {
                const int ox = sx + 2 * a, oy = sy + 2 * b, oz = sz + 2 * d;
                const int f = (ox * n1 + oy) * n1 + oz;
                double* slot = tgs + (tslot * F + f) * TXC + lane;
                *slot = fma(acc[a][b][d], ifact(ox) * ifact(oy) * ifact(oz), *slot);
              }
        }
        pair_barrier(1 + w8);
        if (half == 1) {
          double* dstt = P.dst[tslot];
#pragma unroll
          for (int a = 0; a < jh; ++a)
#pragma unroll
            for (int b = 0; b < jh; ++b)
#pragma unroll
              for (int d = 0; d < jh; ++d) {
                const int ox = sx + 2 * a, oy = sy + 2 * b, oz = sz + 2 * d;
                const int f = (ox * n1 + oy) * n1 + oz;
                const double v = fma(acc[a][b][d], ifact(ox) * ifact(oy) * ifact(oz), tgs[(tslot * F + f) * TXC + lane]);
                bad |= !isfinite(v);
                if (active) dstt[obase + f * P.t_plane] = v;
              }
        }
      }
    }
    double* tmp = ro;
    ro = rn;
    rn = tmp;
  }
  if (bad && active && P.step >= 0) atomicMin(P.flag, P.step);
}

double host_fact(int k) {
  double r = 1.0;
  for (int t = 2; t <= k; ++t) r *= t;
  return r;
}

template <int NT>
int launch_one(const TParams& T, cudaStream_t st) {
  const size_t smem = sizeof(double) * (RAW + 2 * RING + NT * F * TXC);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tiled3d_v5<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured = true;
  }
  dim3 grid((T.tNx + TXC - 1) / TXC, T.tNy, (T.tNz + ZC - 1) / ZC);
  tiled3d_v5<NT><<<grid, NTHREADS, smem, st>>>(T);
  return 1;
}

}  // namespace

int launch(HalfKind kind, const HalfParams& p, cudaStream_t st) {
  TParams T;
  std::memset(&T, 0, sizeof(T));
  for (int s = 0; s < n; ++s)
    for (int l = 0; l < n1; ++l) T.ML[s * n1 + l] = host_fact(s) * p.M[s * n + l];
  for (int b0 = 0; b0 <= MM; ++b0)
    for (int b1 = 0; b1 <= MM - b0; ++b1)
      for (int b2 = 0; b2 <= MM - b0 - b1; ++b2) {
        const int k = b0 + b1 + b2;
        T.GM[bindex(b0, b1, b2, MM)] = p.G[k] * host_fact(k) / (host_fact(b0) * host_fact(b1) * host_fact(b2));
      }
  T.s_layer = p.s_layer;
  T.s_plane = p.s_coef;
  T.t_layer = p.t_layer;
  T.t_plane = p.t_coef;
  T.sNx = p.sNx;
  T.sNy = p.sNy;
  T.tNx = p.tNx;
  T.tNy = p.tNy;
  T.tNz = p.tNz;
  T.t_zoff = p.t_zoff;
  T.K[0] = p.K[0];
  T.K[1] = p.K[1];
  T.bnd[0] = p.bnd[0];
  T.bnd[1] = p.bnd[1];
  T.step = p.step;
  T.flag = p.flag;
  if (kind == VEL) {
    T.src = p.src[0];
    for (int t = 0; t < 3; ++t) T.dst[t] = p.dst[t];
    return launch_one<3>(T, st);
  }
  T.pre = 1;
  int launched = 0;
  for (int c = 0; c < 3; ++c) {
    T.comp = c;
    T.src = p.src[c];
    T.dst[0] = p.dst[0];
    launched += launch_one<1>(T, st);
  }
  return launched;
}

}  // namespace v5
}  // namespace hlfk
