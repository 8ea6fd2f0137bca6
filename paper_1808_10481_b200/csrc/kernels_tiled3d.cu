// Tiled, z-marching 3D half-step kernel (d = 3, constant coefficients, m <= 3).
//
// One CTA = 8 warps owns a row of TXC = 32 target cells along x (lane = cell)
// and marches over a chunk of ZC target layers in z.  Per target layer k it
//   (raw)  streams the next source layer (all (m+1)^3 coefficients of the
//          33 x 2 source nodes under the row) into shared memory with cp.async,
//          one layer ahead of use;
//   (X)    applies M along x: 2 (m+1)^2 x-lines per cell, shared by the two
//          source rows (reconstruct_cell_2d's first sweep, interpolation.cpp:87-99);
//   (Y)    applies M along y: n (m+1) y-lines per cell (interpolation.cpp:101-112);
//          the result for source layer k+1 goes into a 2-layer ring;
//          m = 3 sweeps y first instead, once per source node, in place over
//          the raw stage, then x on neighbouring nodes ((m+1)^2 + n (m+1)
//          lines per cell instead of 2 (m+1)^2 + n (m+1));
//   (Z+CK) applies M along z between ring layers k and k+1 and immediately
//          contracts with the closed-form odd Cauchy-Kowalewski sum of the
//          leapfrog half update (stepper1d.cpp:22-61).
// Every line uses the parity split of M (out[s] couples to sigma_l = L_l + R_l
// for s+l even and to delta_l = R_l - L_l for s+l odd),
// with rows pre-scaled by s! so that the CK coefficients collapse to
// G_k k!/b! (host table GM) and a final 1/o! per output.
// Warps specialise by parity class in the Z+CK stage: warp w owns the P
// entries with (q_x, q_y, q_z) = (w>>2, w>>1, w) mod 2, which holds every P
// entry any of its 24 (velocity) or 8 (pressure) outputs needs, so the CK sum
// runs entirely in registers with compile-time indices.
//
// VEL (p -> v_x, v_y, v_z) is one launch; PRE (v -> p) is two: the V_x and
// V_y divergence terms merged (their index shifts moved into the x / y sweep
// rows, summed in the XY stage, one shift-free CK), and V_z (HLF_NO_MERGE:
// three launches, one per source component c, each adding the c-th
// divergence term (q_c+1) V_c[q+e_c] with target component c).
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "hlf_internal.cuh"

namespace hlfk {
namespace {

constexpr int TXC = 32;         // cells per CTA row (= lanes)
constexpr int RAWX = TXC + 2;   // source row stride: 33 nodes used, 34 = 17 x 16 B (TMA row copies)
constexpr int NWARP = 8;
constexpr int NTHREADS = NWARP * 32;
#ifndef HLF_ZC
#define HLF_ZC 64
#endif
#ifndef HLF_L2HINT
#define HLF_L2HINT 1  // evict-first L2 policy for the target loads and stores (velocity, V_z launches)
#endif
#ifndef HLF_ZSEL_SELECT
#define HLF_ZSEL_SELECT 0  // 1: the V_z launch shifts with per-column selects instead of shifted M rows
#endif
constexpr int ZC = HLF_ZC;      // target layers per CTA (with TMA loads: 64 +0.9 % over 128, 256 -1.5 %)
constexpr int kMaxB = 20;       // multi-indices |b| <= 3
constexpr int kRZ = 2 * 10 * 2 * 4;  // z-folded CK rows: [PZo][(a, b), a + b <= m][jzo][l] (sized for m = 3)

template <int MM>
struct Cfg {
  static constexpr int n1 = MM + 1, n = 2 * MM + 2, F = n1 * n1 * n1, nh = n / 2, jh = (n1 + 1) / 2;
  static constexpr int RAW = F * 2 * RAWX;
  // raw stage stride: one spare double each side for the pre shift, rounded
  // to 128 B (TMA tensor destinations must be 128 B aligned)
  static constexpr int RAWS = (RAW + 2 + 15) / 16 * 16;
  static constexpr int RING = n * n * n1 * TXC;
  // NT: 3 = velocity half (three targets), 1 = one pressure divergence term,
  // 2 = merged V_x + V_y pressure launch (two raw sources, one target),
  // 4 = the whole pressure half step (V_x + V_y merged as for 2, V_z in a
  // second ring; three raw sources, one target)
  template <int NT>
  static constexpr int NTGT = NT == 2 || NT == 4 ? 1 : NT;
  template <int NT>
  static constexpr int NSRC = NT == 2 ? 2 : (NT == 4 ? 3 : 1);  // raw sources per stage
  template <int NT>
  static constexpr int NRING = NT == 4 ? 4 : 2;  // ring layers
  template <int NT>
  static constexpr int TGT = NTGT<NT> * F * TXC;
  // Raw stages (RST) and target stages (TST): the TMA box of a source layer
  // is issued RST - 1/2 iterations and that of a target layer TST - 1
  // iterations ahead of use.  At m = 1 an iteration is short against the DRAM
  // round trip (the loads, not the arithmetic, set the pace), so the stages
  // are deep; at m = 3 there is no room for a second stage (and an iteration
  // covers the latency).  HLF_M1_RST / _TST, HLF_M2_RST / _TST override.
#ifndef HLF_M1_RST
#define HLF_M1_RST 2
#endif
#ifndef HLF_M1_TST
#define HLF_M1_TST 2
#endif
#ifndef HLF_M2_RST
#define HLF_M2_RST 1
#endif
#ifndef HLF_M2_TST
#define HLF_M2_TST 1
#endif
  template <int NT>
  static constexpr int RST = MM == 1 ? HLF_M1_RST : (MM == 2 ? HLF_M2_RST : 1);
  template <int NT>
  static constexpr int TST = MM == 1 ? HLF_M1_TST : (MM == 2 ? HLF_M2_TST : 1);
  template <int NT>
  static constexpr int SMEM_DOUBLES = NSRC<NT> * RST<NT> * RAWS + NRING<NT> * RING + TST<NT> * TGT<NT>;
};

struct TParams {
  CUtensorMap tmap[3];             // raw source tensors [layer][coef][y][x] for TMA box loads
  CUtensorMap tmapT[3];            // target tensors, box (32 cells, 1 row, F, 1 layer)
  double ML[kMaxN * (kMaxM + 1)];  // s! * M[s][l], l < m+1 (left block), row-major [s][l]
  double GM[kMaxB];                // G_k * k!/b!, indexed by bindex(b)
  double IF[kMaxM + 1];            // 1/o!
  double RZ[kRZ];                  // pressure launches, m = 2, 3: z sweep folded into the CK (rz_table)
  const double* src;               // source field base (layer 0 of the allocation)
  const double* src2;              // NT == 2, 4: the V_y source
  const double* src3;              // NT == 4: the V_z source
  double* dst[3];                  // target field bases, per target component
  int64_t s_layer, s_plane;        // source strides
  int64_t t_layer, t_plane;        // target strides
  int t_plane32;                   // t_plane as int (host-checked: F * t_plane < 2^31)
  int sNx, sNy;                    // source plane dims (row stride = sNx)
  int tNx, tNy, tNz;               // target nodes
  int t_zoff;                      // target layer index of z = 0
  int K[2], bnd[2];                // x, y cells and boundary kinds
  int pre;                         // 1: source is the dual family (x0 - 1 shift, mirrors)
  int comp;                        // source component (mirror parity), PRE only
  int step;
  int tma;                         // strides allow 16 B aligned TMA row copies
  int tma_t;                       // target tensor maps encoded
  int raster;                      // > 0: CTA rows launched in groups of `raster` y rows (below)
  int* flag;
  unsigned long long* ctr;         // path counters of this half step (tests) or null
  const HalfParams* hp;            // host only: the caller's parameters (launch timing)
};

__host__ __device__ constexpr int bindex(int b0, int b1, int b2, int mm) {
  // position of (b0, b1, b2) in the enumeration b0 <= mm, b1 <= mm-b0, b2 <= mm-b0-b1
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
// L2 policy for the streamed targets (read once by TMA, written once): evict
// first, so the source rows a neighbouring CTA row reads again stay in L2
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_global_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(__cvta_generic_to_global(p)), "d"(v), "l"(pol));
}
__device__ __forceinline__ void tma_box_hint(double* smem, const CUtensorMap* map, int x, int y, int layer, uint64_t* bar,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], "
      "[%6], %7;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(0), "r"(layer),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_global(double* p, double v) {
  asm volatile("st.global.f64 [%0], %1;\n" ::"l"(__cvta_generic_to_global(p)), "d"(v));
}
// cp.async that the compiler may not reorder with the surrounding shared-memory
// reads (the target slots are re-filled right after their last read)
__device__ __forceinline__ void cp_async8_ordered(double* smem, const double* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_group1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
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
// one tensor box global -> shared (x, y, coefficient plane 0, layer), completing on the mbarrier
__device__ __forceinline__ void tma_box(double* smem, const CUtensorMap* map, int x, int y, int layer, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(0), "r"(layer),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

#include "tiled3d_gen.cuh"
#include "tiled3d_v7_gen.cuh"
// m = 3 Z + CK with both q_z parities in one warp (lanes 16..31 = PZ 1 of the
// same 16 cells): the class-local CK body is picked by the warp-uniform
// shift along x / y; along z the PZ = 0 lanes shift pt by one in registers.
__device__ __forceinline__ void v7_ck(int c, int PX, int PY, int PZ, const TParams& P, double (&pt)[4][4][4],
                                      double (&acc)[2][2][2]) {
  if (c < 0) {
    v7_m3_ck_c0_s0(P, pt, acc);  // no shift (merged pressure launch)
  } else if (c == 0) {
    if (PX) v7_m3_ck_c0_s0(P, pt, acc); else v7_m3_ck_c0_s1(P, pt, acc);
  } else if (c == 1) {
    if (PY) v7_m3_ck_c1_s0(P, pt, acc); else v7_m3_ck_c1_s1(P, pt, acc);
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int d = 0; d < 4; ++d) pt[a][b][d] = PZ ? pt[a][b][d] : (d + 1 < 4 ? pt[a][b][d + 1] : 0.0);
    v7_m3_ck_c2_s0(P, pt, acc);
  }
}

// m = 3, V7 layout, streaming Z + CK (the z half line of each class column is
// folded into the accumulators right away; tiled3d_v7_gen.cuh v7_m3_zck_*)
__device__ __forceinline__ void v7_zck(int c, int PX, int PY, int PZ, const TParams& P, const double* ro,
                                       const double* rn, const double (&cz)[4][4], double g,
                                       double (&acc)[2][2][2]) {
  if (c < 0) {
    v7_m3_zck_c0_s0(P, ro, rn, cz, g, PZ, acc);  // no shift (merged pressure launch)
  } else if (c == 0) {
    if (PX) v7_m3_zck_c0_s0(P, ro, rn, cz, g, PZ, acc); else v7_m3_zck_c0_s1(P, ro, rn, cz, g, PZ, acc);
  } else if (c == 1) {
    if (PY) v7_m3_zck_c1_s0(P, ro, rn, cz, g, PZ, acc); else v7_m3_zck_c1_s1(P, ro, rn, cz, g, PZ, acc);
  } else {
#if HLF_ZSEL_SELECT
    v7_m3_zck_zsel(P, ro, rn, cz, g, PZ, acc);
#else
    v7_m3_zck_c0_s0(P, ro, rn, cz, g, PZ, acc);  // the z shift is in the PZ = 0 lanes' rows (cz)
#endif
  }
}

template <int MM>
__device__ __forceinline__ void xy_task(const TParams& P, int w, const double* raw, double* rn, int lane) {
  // task w = (l_z, q_x parity): fused X+Y stage into the ring layer rn
  constexpr int n1 = MM + 1;
  if (w >= 2 * n1) return;
  const int lz = w >> 1;
  const double* rb = raw + lz * 2 * RAWX + lane;
  double* wb = rn + lz * TXC + lane;
  if constexpr (MM == 1) {
    if (w & 1) m1_xy_px1(P, rb, wb); else m1_xy_px0(P, rb, wb);
  } else if constexpr (MM == 2) {
    if (w & 1) m2_xy_px1(P, rb, wb); else m2_xy_px0(P, rb, wb);
  } else {
    if (w & 1) m3_xy_px1(P, rb, wb); else m3_xy_px0(P, rb, wb);
  }
}

template <int MM>
__device__ __forceinline__ void z_stage(const TParams& P, int pz, const double* ro, const double* rn,
                                        double (&pt)[MM + 1][MM + 1][MM + 1]) {
  if constexpr (MM == 1) {
    if (pz) m1_z_pz1(P, ro, rn, pt); else m1_z_pz0(P, ro, rn, pt);
  } else if constexpr (MM == 2) {
    if (pz) m2_z_pz1(P, ro, rn, pt); else m2_z_pz0(P, ro, rn, pt);
  } else {
    if (pz) m3_z_pz1(P, ro, rn, pt); else m3_z_pz0(P, ro, rn, pt);
  }
}

template <int MM>
__device__ __forceinline__ void ck(int c, int w, const TParams& P, const double (&pt)[MM + 1][MM + 1][MM + 1],
                                   double (&acc)[(MM + 2) / 2][(MM + 2) / 2][(MM + 2) / 2]) {
  if constexpr (MM == 1) m1_ck(c, w, P, pt, acc);
  else if constexpr (MM == 2) m2_ck(c, w, P, pt, acc);
  else if (c < 0) m3_ck_1(P, pt, acc);  // merged pressure launch: no index shift (the shared shift-0 body)
  else m3_ck(c, w, P, pt, acc);
}

// merged pressure launch (c < 0): the index shift is in the sweep rows
template <int MM>
__device__ __forceinline__ void ck_any(int c, int w, const TParams& P, const double (&pt)[MM + 1][MM + 1][MM + 1],
                                       double (&acc)[(MM + 2) / 2][(MM + 2) / 2][(MM + 2) / 2]) {
  if constexpr (MM == 1) {
    if (c < 0) m1_ck_noshift(w, P, pt, acc); else m1_ck(c, w, P, pt, acc);
  } else if constexpr (MM == 2) {
    if (c < 0) m2_ck_noshift(w, P, pt, acc); else m2_ck(c, w, P, pt, acc);
  } else {
    ck<MM>(c, w, P, pt, acc);
  }
}

// merged XY task (V_x through rows q_x+1, V_y through rows q_y+1)
template <int MM>
__device__ __forceinline__ void xy_merged(int px, const TParams& P, const double* rbx, const double* rby,
                                          double* wb) {
  if constexpr (MM == 1) {
    if (px) m1_xy_px1_vxy(P, rbx, rby, wb); else m1_xy_px0_vxy(P, rbx, rby, wb);
  } else if constexpr (MM == 2) {
    if (px) m2_xy_px1_vxy(P, rbx, rby, wb); else m2_xy_px0_vxy(P, rbx, rby, wb);
  } else {
    if (px) m3_xy_px1_vxy(P, rbx, rby, wb); else m3_xy_px0_vxy(P, rbx, rby, wb);
  }
}

// 1/o! for o <= 3 without a dynamically indexed parameter load
__device__ __forceinline__ double ifact_s(int o) { return o <= 1 ? 1.0 : (o == 2 ? 0.5 : 1.0 / 6.0); }

template <int MM, int NT>
#ifndef HLF_M1_CTAS
#define HLF_M1_CTAS 3  // m = 1: 3 CTAs per SM (<= 85 registers): 19.5 -> 17.8 ms at 512x512x256
#endif
__global__ void __launch_bounds__(NTHREADS, MM == 1 ? HLF_M1_CTAS : (MM == 2 ? 2 : 1)) tiled3d(const __grid_constant__ TParams P) {
  using G = Cfg<MM>;
  constexpr int n1 = G::n1, n = G::n, F = G::F, nh = G::nh, jh = G::jh;
  static_assert(nh == MM + 1, "n/2 == m+1");
  constexpr int RST = G::template RST<NT>;   // raw stages
  constexpr int TST = G::template TST<NT>;   // target stages
  constexpr int NSRC = G::template NSRC<NT>;
  static_assert(RST >= 1 && RST <= 4 && TST >= 1 && TST <= 4, "stage counts");
  constexpr bool MX = NT == 2 || NT == 4;     // merged V_x + V_y pressure launch (NT = 4: and V_z)
  constexpr bool ALL3 = NT == 4;
  constexpr int NTT = G::template NTGT<NT>;   // target fields
#ifndef HLF_XY_XFIRST
  constexpr bool YF = MM == 3 && !ALL3;       // y-first XY stage (tiled3d_gen.cuh m3_yl / m3_xt)
#else
  constexpr bool YF = false;
#endif
  extern __shared__ __align__(128) double smem_raw[];
  // TMA tensor destinations must be 128 B aligned: align the base explicitly
  // (the launch requests 128 B of slack)
  // (offset arithmetic on smem_raw keeps the accesses LDS/STS; a pointer
  // rebuilt from an integer would turn them into generic loads)
  double* smem = smem_raw + ((128u - (static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 127u)) & 127u) / 8u;
  // raw stages (MX: raw V_x, raw V_y); node index 0 of a row sits at
  // stage base + pre so that TMA row copies start on a 16 B boundary
  double* rawbuf = smem + P.pre;
  double* ring0 = smem + NSRC * RST * G::RAWS;
  double* ring1 = ring0 + G::RING;
  double* tgs = ring0 + G::template NRING<NT> * G::RING;  // target stages [stage][t][f][cell] (lane-private path: stage 0)
  // NT = 4: the V_z ring (layers ring1 + RING, + 2 RING)
  double* raw = rawbuf;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // CTA order: a source row is read by cell rows ty and ty + 1; launched
  // x-fastest those two CTAs start gridDim.x apart and the second read misses
  // L2 part of the time.  With raster = G the rows of an x tile go in groups
  // of G consecutive CTAs (y fastest inside the group), x tiles next.
  int bx = blockIdx.x, ty = blockIdx.y;
  if (P.raster > 1) {
    const int lin = blockIdx.x + gridDim.x * blockIdx.y;
    const int grp = lin / (P.raster * gridDim.x), r = lin - grp * P.raster * gridDim.x;
    const int rows = min(P.raster, static_cast<int>(gridDim.y) - grp * P.raster);
    ty = grp * P.raster + r % rows;
    bx = r / rows;
  }
  const int x0 = bx * TXC;
  const int k0 = blockIdx.z * ZC;
  const int k1 = min(k0 + ZC, P.tNz);
  if (k0 >= k1) return;

  // Raw layer = 2 F rows (f, source row sy) of RAWX nodes; warp w streams rows
  // w, w+8, ... with lane = node sx (sx = 32 of every row by thread tid < 2F).
  // The x/y node maps (wrap, or mirror at walls) are the same for every row
  // and layer, so they are computed once.
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
  auto ymap = [&](int sy, bool& mir) {
    int q = ty + sy - P.pre;
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
  bool mx_lane, mx_last, my0, my1;
  const int xo_lane = xmap(lane, mx_lane);
  const int xo_last = xmap(TXC, mx_last);
  const int64_t yo0 = static_cast<int64_t>(ymap(0, my0)) * P.sNx;
  const int64_t yo1 = static_cast<int64_t>(ymap(1, my1)) * P.sNx;
  const bool walls = __syncthreads_or(mx_lane || mx_last || my0 || my1);
  __shared__ __align__(8) uint64_t rawbar[4];
  __shared__ __align__(8) uint64_t tgtbar[4];
  uint32_t rphase = 0, tphase = 0;
  // TMA boxes need: no x wrap / mirror inside the row, the two source rows
  // consecutive and unmirrored
  const bool xmirror = __syncthreads_or(mx_lane || mx_last);  // block-wide, evaluated by every thread
#ifdef HLF_EXP_NORAW
  const bool tma_rows = false;  // ablation build: no raw loads, so nothing to wait for
  (void)xmirror;
#else
  const bool tma_rows = P.tma && (P.pre ? (x0 >= 2 && x0 + TXC <= P.sNx) : (x0 + RAWX <= P.sNx)) && !xmirror &&
                        (P.pre ? x0 - 1 + TXC < P.K[0] : true) && !my0 && !my1 && yo1 == yo0 + P.sNx;
#endif
  // Edge CTAs whose row leaves the tensor in exactly one used node (pressure:
  // x0 = 0, node sx = 0 wraps or mirrors; velocity: the last periodic tile,
  // node sx = 32 wraps to 0) still load their rows as TMA boxes (the
  // out-of-range nodes are zero-filled) and patch that one node per row from
  // a register loaded one layer ahead (stored after the box has landed).
  const int psx = P.pre ? 0 : TXC;
  bool mx_psx;
  const int xo_psx = xmap(psx, mx_psx);
  const bool other_mirror = __syncthreads_or((mx_lane && lane != psx) || (mx_last && TXC != psx));
#ifdef HLF_EXP_NORAW
  const bool patch = false;
#else
  const bool patch = RST == 1 && !tma_rows && P.tma && !other_mirror && !my0 && !my1 && yo1 == yo0 + P.sNx &&
                     (P.pre ? (x0 == 0 && TXC - 1 < P.K[0] && TXC <= P.sNx)
                            : (P.bnd[0] == 0 && x0 + TXC == P.K[0] && x0 + TXC <= P.sNx));
#endif
  const bool box_rows = tma_rows || patch;
  double pv = 0.0;  // this thread's patch value (row tid % ROWS of source tid / ROWS)
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(&rawbar[i], 1);
      mbar_init(&tgtbar[i], 1);
    }
    fence_mbar_init();
    count_path(P.ctr, box_rows, P.tma_t != 0);
  }
  __syncthreads();
  constexpr int ROWS = 2 * F;
  // Interior CTAs (no wrap or mirror along x) load every raw row with one TMA
  // bulk copy (34 nodes = 272 B, 16 B aligned) completing on an mbarrier;
  // boundary CTAs and unaligned strides use per-node cp.async.
  auto issue_raw = [&](int layer) {
#ifdef HLF_EXP_NORAW
    cp_async_commit();
    return;
#endif
    if (box_rows) {
      // one 4D box (34 nodes x 2 rows x F coefficients x 1 layer) per source
      const int stage = layer % RST;
      if (patch && tid < NSRC * ROWS) {
        const int si = tid / ROWS, r = tid - si * ROWS;
        const double* base = (si == 0 ? P.src : si == 1 ? P.src2 : P.src3) + static_cast<int64_t>(layer) * P.s_layer;
        pv = __ldg(base + static_cast<int64_t>(r >> 1) * P.s_plane + ((r & 1) ? yo1 : yo0) + xo_psx);
      }
      if (tid == 0) {
        constexpr int NS = NSRC;
        mbar_expect_tx(&rawbar[stage], NSRC * G::RAW * 8);
        fence_proxy_async();
#pragma unroll
        for (int si = 0; si < NS; ++si)
          tma_box(rawbuf + (stage * NSRC + si) * G::RAWS - P.pre, &P.tmap[si], x0 - 2 * P.pre, ty - P.pre, layer,
                  &rawbar[stage]);
      }
      cp_async_commit();  // empty group: keeps the per-thread group pattern
      return;
    }
#pragma unroll
   for (int si = 0; si < NSRC; ++si) {
    double* raw = rawbuf + ((layer % RST) * NSRC + si) * G::RAWS;
    const double* base = (si == 0 ? P.src : si == 1 ? P.src2 : P.src3) + static_cast<int64_t>(layer) * P.s_layer;
    if constexpr (ROWS % NWARP == 0) {
      // row r = warp + 8 i: coefficient plane (warp >> 1) + 4 i, source row warp & 1
      const double* q = base + static_cast<int64_t>(warp >> 1) * P.s_plane + ((warp & 1) ? yo1 : yo0) + xo_lane;
      const int64_t step = (NWARP / 2) * P.s_plane;
#pragma unroll
      for (int i = 0; i < ROWS / NWARP; ++i) {
        cp_async8(raw + (warp + NWARP * i) * RAWX + lane, q);
        q += step;
      }
    } else {
#pragma unroll 4
      for (int r = warp; r < ROWS; r += NWARP) {
        const double* rowp = base + static_cast<int64_t>(r >> 1) * P.s_plane + ((r & 1) ? yo1 : yo0);
        cp_async8(raw + r * RAWX + lane, rowp + xo_lane);
      }
    }
    if (tid < ROWS) {
      const double* rowp = base + static_cast<int64_t>(tid >> 1) * P.s_plane + ((tid & 1) ? yo1 : yo0);
      cp_async8(raw + tid * RAWX + TXC, rowp + xo_last);
    }
   }
    cp_async_commit();
  };
  // mirror signs (zero-Dirichlet walls, PRE only): ghost = sigma (-1)^{a_n} interior
  auto fix_walls_buf = [&](double* raw, int comp) {
    for (int e = tid; e < G::RAW; e += NTHREADS) {
      const int r = e / RAWX, sx = e - r * RAWX;
      const int f = r >> 1, sy = r & 1;
      bool mx;
      bool my;
      (void)xmap(sx, mx);
      (void)ymap(sy, my);
      bool neg = false;
      if (mx) neg ^= (((f / (n1 * n1)) & 1) != 0) ^ (comp != 0);
      if (my) neg ^= ((((f / n1) % n1) & 1) != 0) ^ (comp != 1);
      if (neg) raw[e] = -raw[e];
    }
  };
  auto fix_walls = [&](int layer) {
    double* st0 = rawbuf + (layer % RST) * NSRC * G::RAWS;
    if constexpr (MX) {
      fix_walls_buf(st0, 0);
      fix_walls_buf(st0 + G::RAWS, 1);
      if constexpr (ALL3) fix_walls_buf(st0 + 2 * G::RAWS, 2);
    } else {
      fix_walls_buf(st0, P.comp);
    }
  };
  auto finish_raw = [&](int layer) {
    cp_async_wait_group1();  // this thread's raw(k+1) landed; its targets(k) may be in flight
    if (box_rows) {
      const int stage = layer % RST;
      mbar_wait(&rawbar[stage], (rphase >> stage) & 1);
      rphase ^= 1u << stage;
      if (patch && tid < NSRC * ROWS) {  // RST == 1
        const int si = tid / ROWS, r = tid - si * ROWS;
        rawbuf[(stage * NSRC + si) * G::RAWS + r * RAWX + psx] = pv;  // after the box: no race with its zero fill
      }
    }
    if (walls) {
      __syncthreads();
      fix_walls(layer);
      if (box_rows) fence_proxy_async();  // generic writes before the next TMA refill of this stage
    }
    __syncthreads();
  };
  // class of this warp in the Z + CK stage
  // V7: the two q_z parities of a class share a warp (lane halves).  With TMA
  // loads it still wins for the pressure launches (V_z launch 45.8 vs 47.6 ms)
  // but the velocity launch, with three CK bodies and the z-shift selects of
  // its z component, is faster in the plain one-class-per-warp layout
  // (62.2 vs 68.8 ms at 512x512x256).  HLF_NO_V7 / HLF_V7 force one layout.
  // ZF (m = 2, 3 pressure launches): the z sweep folded into the CK
  // (tiled3d_gen.cuh m3_zf_*: 4 FMAs per (ring column, output) from the
  // column's sum / difference values and the host rows RZ, instead of the z
  // half line plus the CK terms; one output class per warp, the plain
  // layout, warp-uniform rows as constant operands).  HLF_NO_ZF: V7 below.
#if defined(HLF_NO_ZF)
  constexpr bool ZF = false;
#else
  constexpr bool ZF = MM >= 2 && (NT == 1 || NT == 2);
#endif
#if defined(HLF_NO_V7)
  constexpr bool V7 = false;
#elif defined(HLF_V7)
  constexpr bool V7 = MM == 3 && !ZF;
#else
  constexpr bool V7 = MM == 3 && NT != 3 && !ZF;
#endif
  // V7S: the V7 Z stage and CK fused per class column (streaming; one column
  // of P~ live instead of 64).  HLF_V7_SPLIT keeps the two stages apart.
#if defined(HLF_V7_SPLIT)
  constexpr bool V7S = false;
#else
  constexpr bool V7S = V7;
#endif
  // V7 (m = 3): warp = (PX, PY, cell half), lane = (cell, PZ = lane >> 4)
  const int PX = (warp >> 2) & 1, PY = (warp >> 1) & 1;
  const int PZ = V7 ? (lane >> 4) : (warp & 1);
  const int zcell = V7 ? ((warp & 1) * 16 + (lane & 15)) : lane;
  const int cbase = ((PX * n + PY) * n1) * TXC + zcell;
  const bool zactive = x0 + zcell < P.tNx;
  double cz[nh][n1];
  const double zg = PZ ? -1.0 : 1.0;
  // V_z pressure launch (streaming): the PZ = 0 lanes read P~ one z index up
  // (the divergence term's shift); rows 2 iz + 2 have the class's own row
  // parity, so their z lines use the same sum / difference pattern and the
  // shift is just the next row of M (row 2m + 2 does not exist: zero)
  const bool zshift = V7S && NT == 1 && P.comp == 2 && PZ == 0 && !HLF_ZSEL_SELECT;
  if constexpr (V7) {
#pragma unroll
    for (int iz = 0; iz < nh; ++iz)
#pragma unroll
      for (int l = 0; l < n1; ++l) {
        const int row = PZ + 2 * iz + (zshift ? 2 : 0);
        cz[iz][l] = row < n ? P.ML[(row < n ? row : 0) * n1 + l] : 0.0;
      }
  }

  // Targets of layer kk for this lane's own outputs (the entries its epilogue
  // reads), staged with cp.async one iteration ahead.  Per-thread cp.async
  // groups: every iteration commits [raw(k+2)] then [targets(k+1)], so
  // wait_group 1 at the top (raw) and before the epilogue (targets) suffices.
  auto issue_own_targets = [&](int kk) {
    if (zactive && !P.tma_t) {
      const int64_t ob = static_cast<int64_t>(P.t_zoff + kk) * P.t_layer + static_cast<int64_t>(ty) * P.tNx + x0 + zcell;
#pragma unroll 1
      for (int t = 0; t < NTT; ++t) {
        const int c = MX || ZF ? -1 : (NT == 3 ? t : P.comp);  // ZF: class = output parity
        const int sx = (PX - (c == 0)) & 1, sy = (PY - (c == 1)) & 1, sz = (PZ - (c == 2)) & 1;
        const int f0 = (sx * n1 + sy) * n1 + sz;
        const double* q = P.dst[t] + ob + f0 * P.t_plane32;
        double* sp = tgs + (t * F + f0) * TXC + zcell;
#pragma unroll
        for (int a = 0; a < jh; ++a)
#pragma unroll
          for (int b = 0; b < jh; ++b)
#pragma unroll
            for (int d = 0; d < jh; ++d) {
              if (MM < 3 && (sx + 2 * a > MM || sy + 2 * b > MM || sz + 2 * d > MM)) continue;
              const int df = (2 * a * n1 + 2 * b) * n1 + 2 * d;
              cp_async8_ordered(sp + df * TXC, q + df * P.t_plane32);
            }
      }
    }
    cp_async_commit();
  };

  // evict-first targets: velocity and V_z launches -1.5 %; the merged launch
  // +1.5 % (kept on the default policy)
  constexpr bool L2H = HLF_L2HINT && NT != 2;
  const uint64_t l2pol = L2H ? evict_first_policy() : 0;
  // target boxes of layer kk into stage kk % TST (one per target field)
  auto issue_tgt = [&](int kk) {
    const int ts = kk % TST;
    mbar_expect_tx(&tgtbar[ts], NTT * F * TXC * 8);
    fence_proxy_async();
#pragma unroll
    for (int t = 0; t < NTT; ++t)
      if (L2H) tma_box_hint(tgs + (ts * NTT + t) * F * TXC, &P.tmapT[t], x0, ty, P.t_zoff + kk, &tgtbar[ts], l2pol);
      else tma_box(tgs + (ts * NTT + t) * F * TXC, &P.tmapT[t], x0, ty, P.t_zoff + kk, &tgtbar[ts]);
  };
  // iteration k0-1 is the prologue: it only builds ring layer k0.  The raw
  // layers k0 .. k0+RST-1 and the target layers k0 .. k0+TST-2 go out first.
  for (int l = k0; l < k0 + RST && l <= k1; ++l) issue_raw(l);
  cp_async_commit();  // (empty) targets group of the prologue
  if (P.tma_t && tid == 0)
    for (int l = k0; l < k0 + TST - 1 && l < k1; ++l) issue_tgt(l);
  double* ro = ring1;
  double* rn = ring0;
  double* roz = ring1 + 2 * G::RING;  // NT = 4 only
  double* rnz = ring0 + 2 * G::RING;
  int emax = 0;  // max |high word| of the written values (finite check)
#pragma unroll 1
  for (int k = k0 - 1; k < k1; ++k) {
    const bool work = k >= k0;
    raw = rawbuf + ((k + 1) % RST) * NSRC * G::RAWS;
    finish_raw(k + 1);  // raw(k+1) landed; every warp left the previous Z + CK stage
    if (P.tma_t && work && tid == 0 && k + TST - 1 < k1) {
      // targets of layer k + TST - 1 into the stage layer k - 1 used (its
      // epilogue is over: every warp passed the barrier in finish_raw)
      issue_tgt(k + TST - 1);
    }
#ifndef HLF_EXP_NOXY
    if constexpr (YF) {
      // y-first XY (m = 3): warps (q_z, w2) sweep y in place over the raw
      // stage (node = lane, q_x = 2 w2 + i; node 32 on lanes 0, 1), then the
      // warp pair of q_z syncs and each warp sweeps x for j_y = w2 mod 2
      const int qz = warp >> 1, w2 = warp & 1;
#pragma unroll
      for (int si = 0; si < NSRC; ++si) {
        double* sb = raw + si * G::RAWS + qz * 2 * RAWX;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double* yb = sb + (2 * w2 + i) * n1 * n1 * 2 * RAWX + lane;
          if (MX && si == 1) m3_yl_sh(P, yb); else m3_yl(P, yb);
        }
        if (lane < 2) {
          double* yb = sb + (2 * w2 + lane) * n1 * n1 * 2 * RAWX + TXC;
          if (MX && si == 1) m3_yl_sh(P, yb); else m3_yl(P, yb);
        }
      }
      asm volatile("bar.sync %0, 64;\n" ::"r"(1 + qz) : "memory");
      const double* xb = raw + qz * 2 * RAWX + lane;
      double* wb = rn + qz * TXC + lane;
      if constexpr (MX) {
        if (w2) m3_xt1_vxy(P, xb, xb + G::RAWS, wb); else m3_xt0_vxy(P, xb, xb + G::RAWS, wb);
      } else {
        if (w2) m3_xt1(P, xb, wb); else m3_xt0(P, xb, wb);
      }
    } else if constexpr (ALL3) {
      // tasks 0 .. 2 n1 - 1: merged V_x + V_y (l_z, q_x parity) into the
      // ring; 2 n1 .. 4 n1 - 1: V_z (plain rows) into the V_z ring
#pragma unroll 1
      for (int task = warp; task < 4 * n1; task += NWARP) {
        if (task < 2 * n1) {
          const int lz = task >> 1;
          const double* rbx = raw + lz * 2 * RAWX + lane;
          xy_merged<MM>(task & 1, P, rbx, rbx + G::RAWS, rn + lz * TXC + lane);
        } else {
          xy_task<MM>(P, task - 2 * n1, raw + 2 * G::RAWS, rnz, lane);
        }
      }
    } else if (MX && warp >= 2 * n1) {
      // m < 3: fewer (l_z, q_x parity) tasks than warps
    } else if constexpr (MX) {
      const int lz = warp >> 1;
      double* wb = rn + lz * TXC + lane;
      const double* rbx = raw + lz * 2 * RAWX + lane;
      const double* rby = rbx + G::RAWS;
#ifndef HLF_XY_RMW
      xy_merged<MM>(warp & 1, P, rbx, rby, wb);
#else
      if (warp & 1) {
        m3_xy_px1_vx(P, rbx, wb);
        m3_xy_px1_vy(P, rby, wb);
      } else {
        m3_xy_px0_vx(P, rbx, wb);
        m3_xy_px0_vy(P, rby, wb);
      }
#endif
    } else {
      xy_task<MM>(P, warp, raw, rn, lane);
    }
#endif
    __syncthreads();
    // the stage of raw(k+1) is free again: refill it with raw(k+1+RST)
    if (k + 1 + RST <= k1) issue_raw(k + 1 + RST); else cp_async_commit();

#ifdef HLF_EXP_NOZCK
    if (0) {
#else
    if (work) {
#endif
      // Z stage + CK for this warp's parity class
      double pt[nh][nh][nh];
      // ZF runs the merged launch and the V_z launch (the only pressure
      // launches at m = 2, 3 unless HLF_NO_ZF: launch_m ignores HLF_NO_MERGE)
      constexpr bool zf = ZF;
      if constexpr (V7 && !V7S) v7_m3_z(ro + cbase, rn + cbase, cz, zg, pt);
      else if constexpr (!V7) {
        if (!zf) z_stage<MM>(P, PZ, ro + cbase, rn + cbase, pt);
      }
      if constexpr (ALL3) {
        // + the V_z term: its divergence reads P~_z[q + e_z], i.e. the other
        // q_z class of the V_z ring, one class index up when PZ = 1 (warp-uniform)
        double pz[nh][nh][nh];
        z_stage<MM>(P, 1 - PZ, roz + cbase, rnz + cbase, pz);
        if (PZ) {
#pragma unroll
          for (int a = 0; a < nh; ++a)
#pragma unroll
            for (int b = 0; b < nh; ++b)
#pragma unroll
              for (int d = 0; d + 1 < nh; ++d) pt[a][b][d] += pz[a][b][d + 1];
        } else {
#pragma unroll
          for (int a = 0; a < nh; ++a)
#pragma unroll
            for (int b = 0; b < nh; ++b)
#pragma unroll
              for (int d = 0; d < nh; ++d) pt[a][b][d] += pz[a][b][d];
        }
      }
      const int64_t obase = static_cast<int64_t>(P.t_zoff + k) * P.t_layer + static_cast<int64_t>(ty) * P.tNx + x0 + zcell;
      if (P.tma_t) {
        const int ts = k % TST;
        mbar_wait(&tgtbar[ts], (tphase >> ts) & 1);
        tphase ^= 1u << ts;
      } else {
        cp_async_wait_group1();  // this lane's targets(k) landed; raw(k+2) may be in flight
      }
      // velocity launch, m = 3: the three components' CK sums are one shared
      // Q sum at shifted indices (v_c[o] = Q[o + e_c], GM does not depend on
      // c; tiled3d_gen.cuh m3_vel_qs): 2624 instead of 3360 FMAs per cell,
      // summed once per class before the epilogue (-1 %: the CK is not what
      // bounds this launch)
#ifndef HLF_VEL_PERCOMP
      constexpr bool VQ = NT == 3 && MM == 3 && !V7;
#else
      constexpr bool VQ = false;
#endif
      double accq[VQ ? 3 : 1][jh][jh][jh];
      if constexpr (VQ) {
        // one body for every class, then each component takes its entries
        // j + (1 - P_c) e_c (warp-uniform shifts).  Per-class bodies with
        // only the entries a class needs (1884 FMAs per cell) ran 28 % slower:
        // eight live code paths

        double Q[jh + 1][jh + 1][jh + 1];
        m3_vel_qs(P, pt, Q);
#pragma unroll
        for (int a = 0; a < jh; ++a)
#pragma unroll
          for (int b = 0; b < jh; ++b)
#pragma unroll
            for (int d = 0; d < jh; ++d) {
              accq[VQ ? 0 : 0][a][b][d] = PX ? Q[a][b][d] : Q[a + 1][b][d];
              accq[VQ ? 1 : 0][a][b][d] = PY ? Q[a][b][d] : Q[a][b + 1][d];
              accq[VQ ? 2 : 0][a][b][d] = PZ ? Q[a][b][d] : Q[a][b][d + 1];
            }
      }
      // the velocity launch's three components unrolled (their CK chains
      // interleave: 66.2 -> 63.4 ms at 512x512x256)
#pragma unroll
      for (int t = 0; t < NTT; ++t) {
        const int c = MX ? -1 : (NT == 3 ? t : P.comp);  // -1: shifts already in the XY rows
        const int ce = zf ? -1 : c;  // ZF: the warp's class is the output parity
        double acc[jh][jh][jh];
#pragma unroll
        for (int a = 0; a < jh; ++a)
#pragma unroll
          for (int b = 0; b < jh; ++b)
#pragma unroll
            for (int d = 0; d < jh; ++d) acc[a][b][d] = 0.0;
        // outputs o = s + 2j (s = the class's output parity for component c):
        // one base address per component, compile-time offsets per j
        const int sx = (PX - (ce == 0)) & 1, sy = (PY - (ce == 1)) & 1, sz = (PZ - (ce == 2)) & 1;
        const int f0 = (sx * n1 + sy) * n1 + sz;
        double* dp = P.dst[t] + obase + f0 * P.t_plane32;
        asm("" : "+l"(dp));  // keep dp a base register: one IMAD.WIDE per output address
        // TMA targets sit in stage k % TST; the lane-private cp.async path uses stage 0
        const double* tp = tgs + ((P.tma_t ? k % TST : 0) * NTT + t) * F * TXC + f0 * TXC + zcell;
#ifndef HLF_EXP_NOCK
        if constexpr (VQ) {
#pragma unroll
          for (int a = 0; a < jh; ++a)
#pragma unroll
            for (int b = 0; b < jh; ++b)
#pragma unroll
              for (int d = 0; d < jh; ++d) acc[a][b][d] = accq[VQ ? t : 0][a][b][d];
        } else if constexpr (V7S) v7_zck(c, PX, PY, PZ, P, ro + cbase, rn + cbase, cz, zg, acc);
        else if constexpr (V7) v7_ck(c, PX, PY, PZ, P, pt, acc);
        else if (zf) {
          if constexpr (ZF && MM == 3) {
            const double* a0 = ro + cbase;
            const double* a1 = rn + cbase;
            if (MX) {
              if (PZ) m3_zf_s0_pz1(P, a0, a1, acc); else m3_zf_s0_pz0(P, a0, a1, acc);
            } else {
              if (PZ) m3_zf_s1_pz1(P, a0, a1, acc); else m3_zf_s1_pz0(P, a0, a1, acc);
            }
          } else if constexpr (ZF && MM == 2) {
            const double* a0 = ro + cbase;
            const double* a1 = rn + cbase;
            if (MX) {
              if (PZ) m2_zf_s0_pz1(P, a0, a1, acc); else m2_zf_s0_pz0(P, a0, a1, acc);
            } else {
              if (PZ) m2_zf_s1_pz1(P, a0, a1, acc); else m2_zf_s1_pz0(P, a0, a1, acc);
            }
          }
        } else ck_any<MM>(c, warp, P, pt, acc);
#else
        acc[0][0][0] += pt[0][0][0] + pt[3][3][3] + pt[1][2][3];
#endif
        const double ix[2] = {ifact_s(sx), ifact_s(sx + 2)};
        const double iy[2] = {ifact_s(sy), ifact_s(sy + 2)};
        const double iz[2] = {ifact_s(sz), ifact_s(sz + 2)};
#pragma unroll
        for (int a = 0; a < jh; ++a) {
#pragma unroll
          for (int b = 0; b < jh; ++b) {
#pragma unroll
            for (int d = 0; d < jh; ++d) {
              if (MM < 3 && (sx + 2 * a > MM || sy + 2 * b > MM || sz + 2 * d > MM)) continue;
              const int df = (2 * a * n1 + 2 * b) * n1 + 2 * d;
              const double v = fma(acc[a][b][d], ix[a] * iy[b] * iz[d], tp[df * TXC]);
              emax = max(emax, __double2hiint(v) & 0x7fffffff);  // >= 0x7ff00000: inf / nan
              if (zactive) {
                if (L2H) st_global_hint(dp + df * P.t_plane32, v, l2pol);
                else st_global(dp + df * P.t_plane32, v);
              }
            }
          }
        }
      }
    }
#ifndef HLF_EXP_NOTGT
    if (k + 1 < k1 && !P.tma_t) issue_own_targets(k + 1); else cp_async_commit();
#else
    cp_async_commit();
#endif
    double* tmp = ro;
    ro = rn;
    rn = tmp;
    if constexpr (ALL3) {
      tmp = roz;
      roz = rnz;
      rnz = tmp;
    }
  }
  if (emax >= 0x7ff00000 && zactive && P.step >= 0) report_nonfinite(P.flag, P.step);
}

double host_fact(int k) {
  double r = 1.0;
  for (int t = 2; t <= k; ++t) r *= t;
  return r;
}

// Driver entry point for cuTensorMapEncodeTiled (no libcuda link dependency)
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

// raw source tensor [layer][coef][y][x] with box (RAWX, 2, F, 1); false if not encodable
template <int MM>
bool encode_raw_map(CUtensorMap* map, const double* base, const TParams& T, int layers) {
  auto enc = tensor_map_encoder();
  if (enc == nullptr || base == nullptr || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  constexpr int n1 = MM + 1, F = n1 * n1 * n1;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(T.sNx), static_cast<cuuint64_t>(T.sNy),
                              static_cast<cuuint64_t>(F), static_cast<cuuint64_t>(layers)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(T.sNx) * 8, static_cast<cuuint64_t>(T.s_plane) * 8,
                                 static_cast<cuuint64_t>(T.s_layer) * 8};
  const cuuint32_t box[4] = {RAWX, 2, F, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// target tensor [layer][coef][y][x] with box (TXC, 1, F, 1); out-of-range cells are zero-filled
template <int MM>
bool encode_tgt_map(CUtensorMap* map, const double* base, const TParams& T, int layers) {
  auto enc = tensor_map_encoder();
  if (enc == nullptr || base == nullptr || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if (T.tNx % 2 || T.t_plane % 2 || T.t_layer % 2) return false;
  constexpr int n1 = MM + 1, F = n1 * n1 * n1;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(T.tNx), static_cast<cuuint64_t>(T.tNy),
                              static_cast<cuuint64_t>(F), static_cast<cuuint64_t>(layers)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(T.tNx) * 8, static_cast<cuuint64_t>(T.t_plane) * 8,
                                 static_cast<cuuint64_t>(T.t_layer) * 8};
  const cuuint32_t box[4] = {TXC, 1, F, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MM, int NT>
int launch_one(TParams T, cudaStream_t st) {
  {
    constexpr int NTT = Cfg<MM>::template NTGT<NT>;
    bool ok = T.tma_t != 0;
    for (int t = 0; t < NTT && ok; ++t) ok = encode_tgt_map<MM>(&T.tmapT[t], T.dst[t], T, T.t_zoff + T.tNz + 2);
    T.tma_t = ok;
  }
  if (T.tma) {
    const int layers = T.tNz + 3;
    T.tma = encode_raw_map<MM>(&T.tmap[0], T.src, T, layers) &&
            (NT != 2 && NT != 4 || encode_raw_map<MM>(&T.tmap[1], T.src2, T, layers)) &&
            (NT != 4 || encode_raw_map<MM>(&T.tmap[2], T.src3, T, layers));
  }
  using G = Cfg<MM>;
  const size_t smem = sizeof(double) * G::template SMEM_DOUBLES<NT> + 128;
  static std::atomic<unsigned long long> configured{0};
  ensure_smem_opt_in(tiled3d<MM, NT>, static_cast<int>(smem), configured);
  // x-fastest rasterisation; y-fastest (neighbouring rows, which share a
  // source row, launched side by side) measured 1 % slower at 512x512x256
  dim3 grid((T.tNx + TXC - 1) / TXC, T.tNy, (T.tNz + ZC - 1) / ZC);
  tiled3d<MM, NT><<<grid, NTHREADS, smem, st>>>(T);
  mark_launch(*T.hp, st);
  return 1;
}

template <int MM>
int launch_m(HalfKind kind, const HalfParams& p, cudaStream_t st) {
  constexpr int n1 = MM + 1, n = 2 * MM + 2;
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
  for (int o = 0; o <= MM; ++o) T.IF[o] = 1.0 / host_fact(o);
  auto rz_table = [&](int sh) {
    // RZ[PZo][(a, b)][jzo][l] = sum_c GM[a, b, c] (+-) s! M[s][l], s = oz + 2c + sh
    // (oz = PZo + 2 jzo; + for s + l even (sum), - for odd (difference));
    // tools/gen_tiled3d.py gen_zf
    if constexpr (MM >= 2) {
      constexpr int nab = (MM + 1) * (MM + 2) / 2, jhh = (n1 + 1) / 2;
      int ab = 0;
      for (int a = 0; a <= MM; ++a)
        for (int b = 0; b <= MM - a; ++b, ++ab)
          for (int pzo = 0; pzo < 2; ++pzo)
            for (int jzo = 0; jzo < 2; ++jzo)
              for (int l = 0; l < n1; ++l) {
                double r = 0.0;
                const int oz = pzo + 2 * jzo;
                for (int c = 0; a + b + c <= MM; ++c) {
                  const int s = oz + 2 * c + sh;
                  if (s >= n) break;
                  r += T.GM[bindex(a, b, c, MM)] * (((s + l) & 1) ? -T.ML[s * n1 + l] : T.ML[s * n1 + l]);
                }
                T.RZ[((pzo * nab + ab) * jhh + jzo) * n1 + l] = r;
              }
    }
    (void)sh;
  };
  T.s_layer = p.s_layer;
  T.s_plane = p.s_coef;
  T.t_layer = p.t_layer;
  T.t_plane = p.t_coef;
  if (static_cast<int64_t>(n1 * n1 * n1) * p.t_coef >= (int64_t{1} << 31)) return -2;  // generic path
  T.t_plane32 = static_cast<int>(p.t_coef);
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
  T.ctr = p.path_ctr ? p.path_ctr + 3 * kind : nullptr;
  T.hp = &p;
  // TMA boxes: 16 B aligned strides and bases (checked again per tensor map)
  T.tma = std::getenv("HLF_NO_TMA") == nullptr && p.s_layer % 2 == 0 && p.s_coef % 2 == 0 && p.sNx % 2 == 0;
  T.tma_t = std::getenv("HLF_NO_TMA_T") == nullptr;
  {
    // m = 3: groups of 8 rows (merged pressure launch DRAM 2438 -> 2267 B per
    // cell, step -0.9 %; m = 1, 2 +-0: tools/raster_sweep.sh, raster_ab.sh)
    const char* e = std::getenv("HLF_RASTER");
    T.raster = e ? std::atoi(e) : (MM == 3 ? 8 : 0);
  }
  if (kind == VEL) {
    T.pre = 0;
    T.comp = 0;
    T.src = p.src[0];
    for (int t = 0; t < 3; ++t) T.dst[t] = p.dst[t];
    return launch_one<MM, 3>(T, st);
  }
  T.pre = 1;
  T.dst[0] = p.dst[0];
  int launched = 0;
  // m = 2, 3 with the z-folded CK have no single V_x / V_y pressure launches
  // (HLF_NO_MERGE applies to m = 1 and to HLF_NO_ZF builds)
  static const bool merge = std::getenv("HLF_NO_MERGE") == nullptr;
#ifdef HLF_NO_ZF
  constexpr bool force_merge = false;
#else
  constexpr bool force_merge = MM >= 2;
#endif
  static const bool all3 = std::getenv("HLF_NO_ALL3") == nullptr;
  {
    // merged V_x + V_y launch: m = 3 +5.9 %, m = 1 +19.5 %, m = 2 +20 % (the
    // p read-modify-write of one pressure launch saved)
    if constexpr (MM == 1) {
      if (merge && all3) {
        // m = 1: the whole pressure half step in one launch (three raw
        // sources, the V_z term through a second ring)
        T.comp = -1;
        T.src = p.src[0];
        T.src2 = p.src[1];
        T.src3 = p.src[2];
        return launch_one<MM, 4>(T, st);
      }
    }
    if (merge || force_merge) {
      // V_x and V_y divergence terms in one launch, V_z in a second
      T.comp = -1;
      T.src = p.src[0];
      T.src2 = p.src[1];
      rz_table(0);
      launched += launch_one<MM, 2>(T, st);
      T.comp = 2;
      T.src = p.src[2];
      rz_table(1);
      return launched + launch_one<MM, 1>(T, st);
    }
  }
  for (int c = 0; c < 3; ++c) {
    T.comp = c;
    T.src = p.src[c];
    if (c == 2) rz_table(1);
    launched += launch_one<MM, 1>(T, st);
  }
  return launched;
}

}  // namespace

bool tiled3d_supported(int m) { return m >= 1 && m <= 3; }

int launch_half_tiled3d(int m, HalfKind kind, const HalfParams& p, cudaStream_t st) {
  switch (m) {
    case 1: return launch_m<1>(kind, p, st);
    case 2: return launch_m<2>(kind, p, st);
    case 3: return launch_m<3>(kind, p, st);
    default: return -1;
  }
}

}  // namespace hlfk
