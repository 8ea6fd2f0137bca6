// Tiled, y-marching 2D half-step kernel (d = 2, constant coefficients, m = 1..4).
//
// One CTA = 4 warps owns a row of TXC = 32 target cells along x (lane = cell)
// and marches over ZC target rows in y.  Per target row j:
//   (raw)  the next source row (all (m+1)^2 coefficients of the 33 source
//          nodes under the row) and the row's target jets stream into shared
//          memory with cp.async one row ahead (double-buffered; ~40 KB per
//          CTA, so several CTAs share an SM and keep HBM busy);
//   (X)    half x-lines of M (reconstruct_cell_2d's first sweep,
//          interpolation.cpp:87-99) into a 2-row ring;
//   (Y+CK) warp = parity class (q_x, q_y mod 2): y half-lines between ring rows
//          j and j+1 (interpolation.cpp:101-112), then the closed-form odd CK
//          sum of the leapfrog update (d = 2) for every
//          target component, added to the staged target and stored.
// VEL (p -> v, u) is one launch (NT = 2).  PRE (v, u -> p) at m <= 3 is one
// merged launch (NT = 3): P~ = My (Mx^{+1} V_x) + My^{+1} (Mx V_y), i.e. the
// index shift of each divergence term moves into that term's sweep rows, so
// both terms share one CK sum and one read-modify-write of p; at m = 4 it is
// one launch per component (NT = 1).
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "hlf_internal.cuh"

namespace hlfk {
namespace t2 {
namespace {

constexpr int TXC = 32;
constexpr int RAWX = TXC + 2;  // 33 source nodes used; 34 keeps TMA rows 16 B multiples
constexpr int NWARP = 4;
constexpr int NTHREADS = NWARP * 32;
constexpr int ZC = 32;  // rows per CTA (32: +14 % at 1024^2 m = 3 over 64, equal at 4096^2); see launch_one
constexpr int kMaxB2 = 15;  // |b| <= 4 in 2D

struct T2Params {
  CUtensorMap tmap[2];             // raw source tensors [coef][y][x], box (RAWX, 1, F)
  CUtensorMap tmapT[2];            // target tensors, box (TXC, 1, F)
  double ML[kMaxN * (kMaxM + 1)];  // s! M[s][l] (left block)
  double GM[kMaxB2];               // G_k k!/b!
  const double* src;
  const double* src2;              // NT == 3: the V_y source
  double* dst[2];
  int64_t s_plane, t_plane;        // coefficient strides (Nx * Ny)
  int sNx, sNy, tNx, tNy;
  int K[2], bnd[2];
  int pre, comp, step;
  int zc;                       // target rows per CTA
  int tma, tma_t;                  // tensor maps encoded (raw sources / targets)
  int* flag;
  unsigned long long* ctr;         // path counters of this half step (tests) or null
  const HalfParams* hp;            // host only: the caller's parameters (launch timing)
};

#include "tiled2d_gen.cuh"

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// one tensor box (x, y, coefficient plane 0) global -> shared, completing on the mbarrier
__device__ __forceinline__ void tma_box3(double* smem, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(0),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int MM>
__device__ __forceinline__ void x_task(int px, const T2Params& P, const double* rb, double* wb) {
  if constexpr (MM == 1) { if (px) t2_m1_x_px1(P, rb, wb); else t2_m1_x_px0(P, rb, wb); }
  else if constexpr (MM == 2) { if (px) t2_m2_x_px1(P, rb, wb); else t2_m2_x_px0(P, rb, wb); }
  else if constexpr (MM == 3) { if (px) t2_m3_x_px1(P, rb, wb); else t2_m3_x_px0(P, rb, wb); }
  else { if (px) t2_m4_x_px1(P, rb, wb); else t2_m4_x_px0(P, rb, wb); }
}

template <int MM>
__device__ __forceinline__ void x_task_sh(int px, const T2Params& P, const double* rb, double* wb) {
  if constexpr (MM == 1) { if (px) t2_m1_x_px1_sh(P, rb, wb); else t2_m1_x_px0_sh(P, rb, wb); }
  else if constexpr (MM == 2) { if (px) t2_m2_x_px1_sh(P, rb, wb); else t2_m2_x_px0_sh(P, rb, wb); }
  else if constexpr (MM == 3) { if (px) t2_m3_x_px1_sh(P, rb, wb); else t2_m3_x_px0_sh(P, rb, wb); }
  else { if (px) t2_m4_x_px1_sh(P, rb, wb); else t2_m4_x_px0_sh(P, rb, wb); }
}

template <int MM>
__device__ __forceinline__ void yck_merged(int w, const T2Params& P, const double* ro, const double* rn,
                                           const double* rob, const double* rnb, const double* tg, int lane,
                                           double* const* dptr, bool active, bool& bad) {
  if constexpr (MM == 1) t2_m1_prem(w, P, ro, rn, rob, rnb, tg, lane, dptr, active, bad);
  else if constexpr (MM == 2) t2_m2_prem(w, P, ro, rn, rob, rnb, tg, lane, dptr, active, bad);
  else if constexpr (MM == 3) t2_m3_prem(w, P, ro, rn, rob, rnb, tg, lane, dptr, active, bad);
  else t2_m4_prem(w, P, ro, rn, rob, rnb, tg, lane, dptr, active, bad);
}

template <int MM, int NT>
__device__ __forceinline__ void yck(int w, const T2Params& P, const double* ro, const double* rn, const double* tg,
                                    int lane, double* const* dptr, bool active, bool& bad) {
#define HLF_T2(M_)                                                                     \
  if (NT == 2) t2_m##M_##_vel(w, P, ro, rn, tg, lane, dptr, active, bad);              \
  else if (P.comp == 0) t2_m##M_##_pre0(w, P, ro, rn, tg, lane, dptr, active, bad);    \
  else t2_m##M_##_pre1(w, P, ro, rn, tg, lane, dptr, active, bad);
  if constexpr (MM == 1) { HLF_T2(1) }
  else if constexpr (MM == 2) { HLF_T2(2) }
  else if constexpr (MM == 3) { HLF_T2(3) }
  else { HLF_T2(4) }
#undef HLF_T2
}

template <int MM, int NT>
__global__ void __launch_bounds__(NTHREADS) tiled2d(const __grid_constant__ T2Params P) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2, F = n1 * n1;
  constexpr bool MX = NT == 3;         // merged pressure launch
  constexpr int NS = MX ? 2 : 1;       // raw sources
  constexpr int NTT = MX ? 1 : NT;     // target fields
  constexpr int RAW = F * RAWX;
  constexpr int RAWS = (RAW + 2 + 15) / 16 * 16;  // raw stage stride (128 B multiple, pre-shift spare)
  // raw stages per source: the merged launch (and m = 4) single-buffers its
  // sources so that one more CTA fits an SM; the next row is then issued after
  // the X stage (it lands during the Y + CK stage).  Merged m = 3: +7 %,
  // m = 4: +3 %; m <= 2 single launches keep two stages (-3 % otherwise).
  constexpr int RST = (MX || MM >= 4) ? 1 : 2;
  constexpr int RING = n * n1 * TXC;
  constexpr int TGT = NTT * F * TXC;
  extern __shared__ __align__(128) double smem_raw[];
  // 128 B aligned base by offset arithmetic (keeps the accesses LDS/STS)
  double* smem = smem_raw + ((128u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 127u)) & 127u) / 8u;
  double* rawbuf = smem + P.pre;       // [source][2 stages]; node 0 of a row at stage base + pre
  double* ring0 = smem + RST * NS * RAWS;
  double* ring1 = ring0 + RING;
  double* ringb0 = ring1 + RING;       // MX: x-lines of V_y (ring A = ring0/1 holds V_x's)
  double* ringb1 = ringb0 + (MX ? RING : 0);
  double* tgsbuf = ringb1 + (MX ? RING : 0);  // 2 stages [t][f][cell]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TXC;
  const int j0 = blockIdx.y * P.zc;
  const int j1 = min(j0 + P.zc, P.tNy);
  if (j0 >= j1) return;
  const bool active = x0 + lane < P.tNx;

  // x node map of this lane and of node 32 (wrap, or mirror at walls)
  auto xmap = [&](int sx, bool& mir) {
    int q = x0 + sx - P.pre;
    mir = false;
    if (P.bnd[0] == 0) {
      if (q >= P.K[0]) q -= P.K[0];
      if (q < 0) q += P.K[0];
    } else if (P.pre && (q < 0 || q == P.K[0])) {
      q = q < 0 ? 0 : P.K[0] - 1;
      mir = true;
    }
    return q >= P.sNx ? P.sNx - 1 : q;
  };
  auto ymap = [&](int r, bool& mir) {
    int q = r;
    mir = false;
    if (P.bnd[1] == 0) {
      if (q >= P.K[1]) q -= P.K[1];
      if (q < 0) q += P.K[1];
    } else if (P.pre && (q < 0 || q == P.K[1])) {
      q = q < 0 ? 0 : P.K[1] - 1;
      mir = true;
    }
    return q >= P.sNy ? P.sNy - 1 : q;
  };
  bool mx_lane, mx_last;
  const int xo_lane = xmap(lane, mx_lane);
  const int xo_last = xmap(TXC, mx_last);
  const bool xwall = __syncthreads_or(mx_lane || mx_last);
  // TMA rows: no x wrap / mirror inside the row (edge CTAs load per node)
  const bool tma_rows = P.tma && !xwall && (P.pre ? (x0 >= 2 && x0 + TXC <= P.sNx && x0 - 1 + TXC < P.K[0])
                                                  : (x0 + RAWX <= P.sNx && x0 + TXC < P.K[0]));
  __shared__ __align__(8) uint64_t rawbar[2], tgtbar[2];
  unsigned rphase = 0, tphase = 0;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&rawbar[i], 1);
      mbar_init(&tgtbar[i], 1);
    }
    fence_mbar_init();
    count_path(P.ctr, tma_rows, P.tma_t != 0);
  }
  __syncthreads();

  // source row sr (allocation row index of the source family) -> raw stage
  auto issue_raw = [&](int sr) {
    bool my;
    const int q = ymap(sr, my);
    if (tma_rows) {
      if (tid == 0) {
        mbar_expect_tx(&rawbar[sr & 1], NS * RAW * 8);
        fence_proxy_async();
#pragma unroll
        for (int si = 0; si < NS; ++si)
          tma_box3(rawbuf + (si * RST + (sr & (RST - 1))) * RAWS - P.pre, &P.tmap[si], x0 - 2 * P.pre, q,
                   &rawbar[sr & 1]);
      }
      cp_async_commit();
      return;
    }
#pragma unroll
    for (int si = 0; si < NS; ++si) {
      double* raw = rawbuf + (si * RST + (sr & (RST - 1))) * RAWS;
      const double* rowbase = (si ? P.src2 : P.src) + static_cast<int64_t>(q) * P.sNx;
      for (int f = warp; f < F; f += NWARP) cp_async8(raw + f * RAWX + lane, rowbase + f * P.s_plane + xo_lane);
      if (tid < F) cp_async8(raw + tid * RAWX + TXC, rowbase + tid * P.s_plane + xo_last);
    }
    cp_async_commit();
  };
  // mirror signs: ghost = sigma (-1)^{a_n} interior (zero-Dirichlet walls, PRE)
  auto fix_raw = [&](int sr) {
    bool my;
    (void)ymap(sr, my);
    if (!my && !xwall) return;
    for (int si = 0; si < NS; ++si) {
      double* raw = rawbuf + (si * RST + (sr & (RST - 1))) * RAWS;
      const int comp = MX ? si : P.comp;
      for (int e = tid; e < RAW; e += NTHREADS) {
        const int f = e / RAWX, sx = e - f * RAWX;
        bool mx;
        (void)xmap(sx, mx);
        bool neg = false;
        if (mx) neg ^= ((f / n1) & 1) ^ (comp != 0);
        if (my) neg ^= ((f % n1) & 1) ^ (comp != 1);
        if (neg) raw[e] = -raw[e];
      }
    }
    if (tma_rows) fence_proxy_async();  // generic writes before the next TMA refill of this stage
  };
  auto issue_targets = [&](int j) {
    double* tg = tgsbuf + (j & 1) * TGT;
    if (P.tma_t) {
      if (tid == 0) {
        mbar_expect_tx(&tgtbar[j & 1], TGT * 8);
        fence_proxy_async();
#pragma unroll
        for (int t = 0; t < NTT; ++t) tma_box3(tg + t * F * TXC, &P.tmapT[t], x0, j, &tgtbar[j & 1]);
      }
      cp_async_commit();
      return;
    }
    if (x0 + lane < P.tNx) {
      const int64_t rowoff = static_cast<int64_t>(j) * P.tNx + x0 + lane;
      for (int r = warp; r < NTT * F; r += NWARP) {
        const int t = r / F, f = r - t * F;
        cp_async8(tg + r * TXC + lane, P.dst[t] + rowoff + f * P.t_plane);
      }
    }
    cp_async_commit();
  };

  // source rows for target row j: j + s - pre, s = 0, 1
  issue_raw(j0 - P.pre);
  double* ro = ring1;
  double* rn = ring0;
  double* rob = ringb1;
  double* rnb = ringb0;
  bool bad = false;
  for (int j = j0 - 1; j < j1; ++j) {
    const bool work = j >= j0;
    const int snew = j + 1 - P.pre;  // source row entering the ring this iteration
    cp_async_wait_all();
    if (tma_rows) {
      mbar_wait(&rawbar[snew & 1], (rphase >> (snew & 1)) & 1);
      rphase ^= 1u << (snew & 1);
    }
    __syncthreads();
    fix_raw(snew);
    __syncthreads();
    if (RST == 2 && j + 1 < j1) issue_raw(snew + 1);
    if (j + 1 < j1) issue_targets(j + 1);
    const double* raw = rawbuf + (snew & (RST - 1)) * RAWS;
    if constexpr (MX) {
      // V_x with the shifted x rows into ring A, V_y into ring B
      for (int task = warp; task < 4 * n1; task += NWARP) {
        const int si = task >= 2 * n1, tk = task - si * 2 * n1, ly = tk >> 1, px = tk & 1;
        if (si) x_task<MM>(px, P, raw + RST * RAWS + ly * RAWX + lane, rnb + ly * TXC + lane);
        else x_task_sh<MM>(px, P, raw + ly * RAWX + lane, rn + ly * TXC + lane);
      }
    } else {
      for (int task = warp; task < 2 * n1; task += NWARP) {
        const int ly = task >> 1, px = task & 1;
        x_task<MM>(px, P, raw + ly * RAWX + lane, rn + ly * TXC + lane);
      }
    }
    __syncthreads();
    if (RST == 1 && j + 1 < j1) issue_raw(snew + 1);  // single raw stage: X is done with it
    if (work && P.tma_t) {
      mbar_wait(&tgtbar[j & 1], (tphase >> (j & 1)) & 1);
      tphase ^= 1u << (j & 1);
    }
    if (work) {
      double* dptr[NTT];
      for (int t = 0; t < NTT; ++t) dptr[t] = P.dst[t] + static_cast<int64_t>(j) * P.tNx + x0 + lane;
      if constexpr (MX)
        yck_merged<MM>(warp, P, ro + lane, rn + lane, rob + lane, rnb + lane, tgsbuf + (j & 1) * TGT, lane, dptr,
                       active, bad);
      else
        yck<MM, NT>(warp, P, ro + lane, rn + lane, tgsbuf + (j & 1) * TGT, lane, dptr, active, bad);
    }
    double* tmp = ro;
    ro = rn;
    rn = tmp;
    tmp = rob;
    rob = rnb;
    rnb = tmp;
  }
  if (bad && active && P.step >= 0) report_nonfinite(P.flag, P.step);
}

double host_fact(int k) {
  double r = 1.0;
  for (int t = 2; t <= k; ++t) r *= t;
  return r;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// [coef][y][x] tensor, box (bx, 1, F); false if not encodable (alignment, no driver entry)
bool encode_map(CUtensorMap* map, const double* base, int nx, int ny, int F, int64_t plane, int bx) {
  auto enc = tensor_map_encoder();
  if (enc == nullptr || base == nullptr || (reinterpret_cast<uintptr_t>(base) & 15) != 0 || nx % 2 || plane % 2)
    return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(nx), static_cast<cuuint64_t>(ny), static_cast<cuuint64_t>(F)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(nx) * 8, static_cast<cuuint64_t>(plane) * 8};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(bx), 1, static_cast<cuuint32_t>(F)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MM, int NT>
int launch_one(T2Params T, cudaStream_t st) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2, F = n1 * n1;
  constexpr int NS = NT == 3 ? 2 : 1, NTT = NT == 3 ? 1 : NT;
  constexpr int RAWS = (F * RAWX + 2 + 15) / 16 * 16;
  const bool want = std::getenv("HLF_NO_TMA") == nullptr;
  T.tma = want && encode_map(&T.tmap[0], T.src, T.sNx, T.sNy, F, T.s_plane, RAWX) &&
          (NS == 1 || encode_map(&T.tmap[1], T.src2, T.sNx, T.sNy, F, T.s_plane, RAWX));
  T.tma_t = want;
  for (int t = 0; t < NTT && T.tma_t; ++t) T.tma_t = encode_map(&T.tmapT[t], T.dst[t], T.tNx, T.tNy, F, T.t_plane, TXC);
  constexpr int RST = (NT == 3 || MM >= 4) ? 1 : 2;
  const size_t smem = sizeof(double) * (RST * NS * RAWS + 2 * NS * n * n1 * TXC + 2 * NTT * F * TXC) + 128;
  static std::atomic<unsigned long long> configured{0};
  ensure_smem_opt_in(tiled2d<MM, NT>, static_cast<int>(smem), configured);
  // rows per CTA: ZC, or shorter chunks when the grid has too few CTAs to
  // fill the SMs evenly (1024^2: m = 1 +7 % at 8 rows, m = 3 +9 % and m = 4
  // +11 % at 16, m = 2 equal; 4096^2 is best at 32); HLF_T2_ZC overrides
  static const int zc_env = std::getenv("HLF_T2_ZC") ? std::atoi(std::getenv("HLF_T2_ZC")) : 0;
  const int64_t ctas32 = static_cast<int64_t>((T.tNx + TXC - 1) / TXC) * ((T.tNy + ZC - 1) / ZC);
  T.zc = zc_env > 0 ? zc_env : (ctas32 >= 2048 ? ZC : (MM == 1 ? 8 : (MM == 2 ? ZC : 16)));
  dim3 grid((T.tNx + TXC - 1) / TXC, (T.tNy + T.zc - 1) / T.zc);
  tiled2d<MM, NT><<<grid, NTHREADS, smem, st>>>(T);
  mark_launch(*T.hp, st);
  return 1;
}

template <int MM>
int launch_m(HalfKind kind, const HalfParams& p, cudaStream_t st) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
  T2Params T;
  std::memset(&T, 0, sizeof(T));
  for (int s = 0; s < n; ++s)
    for (int l = 0; l < n1; ++l) T.ML[s * n1 + l] = host_fact(s) * p.M[s * n + l];
  int idx = 0;
  for (int b0 = 0; b0 <= MM; ++b0)
    for (int b1 = 0; b1 <= MM - b0; ++b1) {
      const int k = b0 + b1;
      T.GM[idx++] = p.G[k] * host_fact(k) / (host_fact(b0) * host_fact(b1));
    }
  T.s_plane = p.s_coef;
  T.t_plane = p.t_coef;
  T.sNx = p.sNx;
  T.sNy = p.sNy;
  T.tNx = p.tNx;
  T.tNy = p.tNy;
  T.K[0] = p.K[0];
  T.K[1] = p.K[1];
  T.bnd[0] = p.bnd[0];
  T.bnd[1] = p.bnd[1];
  T.step = p.step;
  T.flag = p.flag;
  T.ctr = p.path_ctr ? p.path_ctr + 3 * kind : nullptr;
  T.hp = &p;
  if (kind == VEL) {
    T.src = p.src[0];
    T.dst[0] = p.dst[0];
    T.dst[1] = p.dst[1];
    return launch_one<MM, 2>(T, st);
  }
  T.pre = 1;
  // merged launch, 4096^2 step times: m = 1 +13 %, m = 2 +9 %, m = 3 +9 %;
  // at m = 4 its larger shared footprint (two raw sources, four ring rows)
  // costs occupancy and it is 14 % slower, so there the per-component
  // launches stay (HLF_MERGE_ALL forces the merged launch for A/B runs)
  static const bool merge = std::getenv("HLF_NO_MERGE") == nullptr;
  static const bool merge_all = std::getenv("HLF_MERGE_ALL") != nullptr;
  if (merge && (MM <= 3 || merge_all)) {
    T.comp = -1;
    T.src = p.src[0];
    T.src2 = p.src[1];
    T.dst[0] = p.dst[0];
    return launch_one<MM, 3>(T, st);
  }
  int launched = 0;
  for (int c = 0; c < 2; ++c) {
    T.comp = c;
    T.src = p.src[c];
    T.dst[0] = p.dst[0];
    launched += launch_one<MM, 1>(T, st);
  }
  return launched;
}

}  // namespace
}  // namespace t2

bool tiled2d_supported(int m) { return m >= 1 && m <= 4; }

int launch_half_tiled2d(int m, HalfKind kind, const HalfParams& p, cudaStream_t st) {
  switch (m) {
    case 1: return t2::launch_m<1>(kind, p, st);
    case 2: return t2::launch_m<2>(kind, p, st);
    case 3: return t2::launch_m<3>(kind, p, st);
    case 4: return t2::launch_m<4>(kind, p, st);
    default: return -1;
  }
}

}  // namespace hlfk
