// Internal declarations shared by the host orchestration (hlf_capi.cu) and the
// kernels.  Everything is FP64; the method is arXiv 1808.10481's
// Hermite-leapfrog scheme (reference: /root/reference/proj, 1D only; the d-dim
// generalization follows SURVEY.md App. A.3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace hlfk {

constexpr int kMaxM = 8;                 // SchemeConfig::m_cap (config.hpp:31)
constexpr int kMaxN = 2 * kMaxM + 2;     // 2m+2

// Which staggered half step a launch performs.
//   VEL: target = dual nodes (velocity), source = p at the 2^d primary corners
//        (Stepper1d::advance_v, stepper1d.cpp:158-166)
//   PRE: target = primary nodes (pressure), source = v at the 2^d dual corners
//        (Stepper1d::advance_p, stepper1d.cpp:147-156)
enum HalfKind { VEL = 0, PRE = 1 };

// Kernel parameters, passed by value (lives in the constant parameter bank, so
// M and the CK weights are free DFMA operands).
struct HalfParams {
  double M[kMaxN * kMaxN];      // interpolation operator, row-major (interpolation.cpp:42-44)
  // Closed-form CK weights for constant coefficients:
  //   G[k] = w_{2k+1} / h^{2k+1} * (VEL: av^{k+1} ap^k | PRE: ap^{k+1} av^k)
  // with w_r = 2 prod_{q<=r} (dt/2)/q (leapfrog_half_update, stepper1d.cpp:54-61)
  double G[kMaxM + 1];
  double w[kMaxN];              // w_r for the iterated (variable-coefficient) form
  double inv_h, h;
  int pow2_h;                   // h is a power of two: x / h == x * inv_h exactly (faithful kernels)
  double ap, av;
  const double* src[3];         // source field bases (layer 0 of the allocation)
  double* dst[3];               // target field bases
  const double* coeff;          // per-target-node ap jets [z][E][y][x] or null
  int64_t s_layer, s_coef;      // source strides (elements)
  int64_t t_layer, t_coef;      // target strides
  int64_t c_layer, c_coef;      // coefficient-jet strides
  const double* force;          // forcing table z_r at the target nodes, [z][(r n^d + e)][y][x], or null
  int64_t f_coef;               // plane of the target grid
  int64_t f_layer;              // (n - 1) n^d planes
  int sNx, sNy;                 // source plane size
  int tNx, tNy, tNz;            // target nodes to update
  int t_zoff;                   // layer index of target z = 0 (p: 0, v: 1)
  int s_zoff;                   // layer index of source z = 0
  int K[3];
  int bnd[3];                   // 0 periodic, 1 reflective (x, y in-kernel; z via ghost layers)
  int step;                     // step index for the finite flag, -1 = do not record
  int* flag;                    // [first non-finite step (atomicMin), graph step base]
  // optional path counters (tests; null in production): per HalfKind
  // [CTAs, CTAs that loaded their source rows by TMA, CTAs that loaded their targets by TMA]
  unsigned long long* path_ctr;
  // optional per-launch timing (hlf_time_launches): event launch_ev[i + 1] is
  // recorded after the i-th kernel of this half step (launch_ev[0] before it)
  cudaEvent_t* launch_ev;
  int* launch_idx;
  // separable coefficient generated in the kernel (var2d; var3d reads its own copy):
  // ap = -(sep[0] + sep[1] prod sin(sep[2+a] x_a + sep[5+a])), sep_x0 = target node 0
  int sep_on;
  double sep[8];
  double sep_x0[3];
};

// record the "after launch" event of a timed half step (no-op otherwise)
inline void mark_launch(const HalfParams& p, cudaStream_t st) {
  if (p.launch_ev != nullptr && *p.launch_idx < 3) cudaEventRecord(p.launch_ev[++*p.launch_idx], st);
}

// per-CTA path accounting of the tiled kernels (counters enabled by hlf_enable_path_counters)
__device__ __forceinline__ void count_path(unsigned long long* ctr, bool tma_rows, bool tma_t) {
  if (ctr == nullptr) return;
  atomicAdd(ctr, 1ull);
  if (tma_rows) atomicAdd(ctr + 1, 1ull);
  if (tma_t) atomicAdd(ctr + 2, 1ull);
}

struct FillParams {
  double* dst;
  int64_t layer, coef;
  int Nx, Ny, Nz, zoff;
  int d, n1;
  double x0[3];                 // coordinate of node 0 along each axis
  double h, amp;
  double w[3], phase[3];
  double* err;                  // launch_error: [sum of squared value errors, max |jet error|]
};

// Gauss-quadrature L2 error of one field against amp prod sin(w x + phase)
struct L2Params {
  double M[kMaxN * kMaxN];
  double gx[kMaxN], gw[kMaxN];  // n-point Gauss-Legendre rule on [-1, 1]
  const double* src;            // field base (layer 0 of the allocation)
  int64_t layer, coef;
  int zoff;
  int Nx;                       // field nodes along x (row stride)
  int cells[3];                 // cells per axis (1 for unused axes)
  int wrap[3];                  // periodic axis
  int shift;                    // 0: corners j, j+1 (primary field); 1: j-1, j (dual field)
  double xc0[3];                // centre of cell 0 per axis
  double h;
  int n, n1, d;
  double amp, w[3], phase[3];
  double* out;                  // += sum of w (value - exact)^2 (h/2)^d
};

// 1D discrete energy (conserved_q / conserved_r): f, g = the two fields
struct EnergyParams {
  double M[kMaxN * kMaxN];
  double gx[kMaxN], gw[kMaxN];  // (m+1)-point Gauss-Legendre rule
  const double* f;              // field whose cells are integrated ([coef][node], stride coef)
  const double* g;              // the other field (shifted by -+ s)
  int64_t coef;
  int f_primary;                // f on the primary grid (conserved_q) or the dual grid (conserved_r)
  int K, n, n1;
  double x0, h, s;
  double* out;
};

// 1D alternative schemes of the reference Stepper1d (periodic, constant
// ap / av): the modified Hermite-leapfrog half pass (step_modified,
// stepper1d.cpp:191-232) and the two passes of the classic two-half-step
// Hermite scheme (step_dual_hermite, stepper1d.cpp:249-272).
struct Scheme1dParams {
  double M[kMaxN * kMaxN];
  double h, ap, av, dt;
  double inv_h;
  int pow2_h;                   // h is a power of two: x / h == x * inv_h exactly
  int K;                        // nodes per grid (periodic)
  int to_primary;               // modified: 1 = dual -> primary half, 0 = primary -> dual
  const double* src_p;          // the two fields of the source grid [coef][node]
  const double* src_v;
  double* dst_p;                // targets (modified: updated in place from their previous value)
  double* dst_v;
  int step;
  int* flag;
};

// First non-finite step: flag[0] = min over reports, flag[1] = the step base
// of a replayed CUDA graph (kernels captured in one carry the step offset
// within it; 0 for direct launches).  Read only on the failure path.
__device__ __forceinline__ void report_nonfinite(int* flag, int step) {
  atomicMin(flag, step + *reinterpret_cast<volatile int*>(flag + 1));
}

// The dynamic shared-memory opt-in (cudaFuncSetAttribute) is per device:
// set it once per kernel and device (devices 0..63), thread-safely.
template <class Kernel>
inline void ensure_smem_opt_in(Kernel kernel, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess)
    done.fetch_or(bit, std::memory_order_release);
}

// launchers (return the number of kernels launched)
int launch_modified_1d(int m, const Scheme1dParams& p, cudaStream_t st);
// pass 0: dual midpoints from the primary grid; pass 1: primary from the midpoints
int launch_dual_hermite_1d(int m, int pass, const Scheme1dParams& p, cudaStream_t st);
int launch_half_generic(int d, int m, bool variable, HalfKind kind, const HalfParams& p,
                        cudaStream_t st);
int launch_half_tiled3d(int m, HalfKind kind, const HalfParams& p, cudaStream_t st);
bool tiled3d_supported(int m);
int launch_half_tiled2d(int m, HalfKind kind, const HalfParams& p, cudaStream_t st);
bool tiled2d_supported(int m);
// 3D with ap = -(c0 + c1 prod sin(w x + ph)) generated on the fly, m = 1..3;
// sep = {c0, c1, w[3], phase[3]}, x0 = coordinates of target node 0
int launch_half_var3d(int m, HalfKind kind, const HalfParams& p, const double* sep, const double* x0,
                      cudaStream_t st);
bool var3d_supported(int m);
// the same coefficient as stored per-node jets ([z][E][y][x]) of one grid
int launch_fill_sep_coeff(double* dst, int d, const int* N, int n, double h, const double* x0, const double* sep,
                          cudaStream_t st);
// 2D with per-node ap jets (variable c^2), m = 1..4
int launch_half_var2d(int m, HalfKind kind, const HalfParams& p, cudaStream_t st);
bool var2d_supported(int m);
int launch_fill(const FillParams& p, cudaStream_t st);
int launch_l2(const L2Params& p, cudaStream_t st);
int launch_energy_1d(const EnergyParams& p, cudaStream_t st);
// field - amp prod sin_jet -> err[0] += sum of squared value errors, err[1] = max |jet error|
int launch_error(const FillParams& p, cudaStream_t st);
// z ghost mirror for the dual family: dst layer = sign * (-1)^{c_z} src layer
int launch_mirror_layer(double* dst, const double* src, int64_t plane, int n1, int d, double sigma,
                        cudaStream_t st);
// AoS [node][coef] chunk <-> SoA field (x-major node order)
int launch_aos_to_soa(const double* aos, double* field, int64_t node0, int64_t count, int F,
                      int Nx, int Ny, int Nz, int64_t layer, int64_t coef, int zoff, cudaStream_t st);
int launch_soa_to_aos(const double* field, double* aos, int64_t node0, int64_t count, int F,
                      int Nx, int Ny, int Nz, int64_t layer, int64_t coef, int zoff, cudaStream_t st);

}  // namespace hlfk
