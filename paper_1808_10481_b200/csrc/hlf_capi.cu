// Host orchestration behind the C-ABI in include/hlf_b200.h.
//
// Owns the device-resident staggered state (SoA [layer][coef][y][x] per
// field), the CK weights for the current dt, the z ghost layers, and the
// fused non-finite flag.  Mirrors the reference's Stepper1d semantics
// (proj/src/stepper1d.cpp): advance_p then advance_v, time stamps advanced by
// += dt on the host (:155, :165), InstabilityError carrying the step index
// (:121-129), ConfigError for bad m / grid / field count (config.cpp:27-32,
// grid.cpp:10-26).
#include <climits>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hlf_b200.h"
#include "hlf_internal.cuh"

using hlfk::HalfParams;

struct hlf_solver {
  int d = 1, m = 0, n1 = 1, n = 2, F = 1, E = 1;
  int K[3] = {1, 1, 1};
  int bnd[3] = {0, 0, 0};
  int Np[3] = {1, 1, 1}, Nd[3] = {1, 1, 1};
  double x_min[3] = {0, 0, 0};
  double h = 1.0, ap = -1.0, av = -1.0;
  bool variable = false;
  // CUDA graph of graph_chunk leapfrog steps, replayed by hlf_advance_n
  // (small grids are launch bound); rebuilt when dt, the kernel variant or a
  // kernel pointer (gen) changes
  int graph_chunk = 32;
  cudaGraphExec_t graph_exec = nullptr;
  int graph_steps = 0, graph_variant = -1, graph_kernels = 0;
  double graph_dt = 0.0;
  uint64_t gen = 1, graph_gen = 0;
  bool m_mirror = true;  // M_R = diag((-1)^r) M_L diag((-1)^l): the fast kernels use M_L only
  bool z_slab = false;
  int scheme = HLF_SCHEME_LEAPFROG;
  int nfields = 2;              // d + 1, or 4 for the 1D alternative schemes
  double t_p = 0.0, t_v = 0.0, dt = 0.0;
  std::vector<double> M;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // fields: 0 = p, 1..d = v components
  double* field[4] = {nullptr, nullptr, nullptr, nullptr};
  int layers[4] = {1, 1, 1, 1};
  int64_t plane[4] = {1, 1, 1, 1};
  double* coeff[2] = {nullptr, nullptr};
  // hlf_set_coeff_separable: ap = -(c0 + c1 prod sin(w x + ph)); 3D m <= 3
  // generates the jets inside the var3d kernel (no stored grids)
  bool sep3d = false;
  double sep[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // c0, c1, w[3], phase[3]
  bool coeff_ready(int grid) const { return coeff[grid] != nullptr || sep3d; }
  double* force[2] = {nullptr, nullptr};  // 1D forcing tables [(r n + s)][x] per target grid
  bool force_on = false;
  bool force_fresh[2] = {false, false};
  int* flag = nullptr;
  int* flag_host = nullptr;
  unsigned long long* path_ctr = nullptr;  // hlf_enable_path_counters (tests)
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};  // hlf_time_launches
  bool timing = false;
  int tev_idx = 0;
  double* errbuf = nullptr;     // hlf_error_separable accumulator (device) and its host copy
  double* errbuf_host = nullptr;
  double* staging[2] = {nullptr, nullptr};  // double-buffered host-transfer staging
  size_t staging_bytes = 0;
  cudaStream_t xstream = nullptr;           // copy stream of hlf_set_field / hlf_get_field
  cudaEvent_t copy_done[2] = {nullptr, nullptr}, perm_done[2] = {nullptr, nullptr};
  int64_t launches = 0;
  int variant = 0;
  std::string err;

  int64_t layer_stride(int f) const { return plane[f] * F; }
  int zoff(int f) const { return (d == 3 && f > 0) ? 1 : 0; }
  // leapfrog: p primary, v dual; alternative schemes: even fields primary, odd dual
  int grid_of(int f) const {
    return (scheme == HLF_SCHEME_LEAPFROG ? f == 0 : f % 2 == 0) ? HLF_PRIMARY : HLF_DUAL;
  }
  const int* nodes_of(int f) const { return grid_of(f) == HLF_PRIMARY ? Np : Nd; }
  int64_t num_nodes(int grid) const {
    const int* N = grid == HLF_PRIMARY ? Np : Nd;
    return static_cast<int64_t>(N[0]) * N[1] * N[2];
  }
};

namespace {

thread_local std::string g_create_error;

hlf_status fail(hlf_solver* s, hlf_status st, const std::string& msg) {
  if (s) s->err = msg;
  else g_create_error = msg;
  return st;
}

hlf_status cuda_fail(hlf_solver* s, cudaError_t e, const char* what) {
  return fail(s, HLF_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

#define HLF_CUDA(s, call)                                      \
  do {                                                         \
    cudaError_t hlf_e_ = (call);                               \
    if (hlf_e_ != cudaSuccess) return cuda_fail((s), hlf_e_, #call); \
  } while (0)

double binom(int s, int l) {
  double b = 1.0;
  for (int q = 0; q < l; ++q) b = b * (s - q) / (q + 1);
  return b;
}

// M = A^{-1} by Gauss-Jordan with partial pivoting (the algorithm of
// Eigen::PartialPivLU::inverse used at interpolation.cpp:40).
void build_M(int m, std::vector<double>& M, double* cond) {
  const int n = 2 * m + 2;
  std::vector<double> A(static_cast<size_t>(n) * n, 0.0), W, inv(static_cast<size_t>(n) * n, 0.0);
  for (int half = 0; half < 2; ++half) {
    const double xi = half == 0 ? -0.5 : 0.5;
    for (int l = 0; l <= m; ++l) {
      const int row = half * (m + 1) + l;
      for (int s = l; s < n; ++s) A[row * n + s] = binom(s, l) * std::pow(xi, s - l);
    }
  }
  W = A;
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(W[r * n + col]) > std::abs(W[piv * n + col])) piv = r;
    if (piv != col)
      for (int j = 0; j < n; ++j) {
        std::swap(W[piv * n + j], W[col * n + j]);
        std::swap(inv[piv * n + j], inv[col * n + j]);
      }
    const double dd = W[col * n + col];
    for (int j = 0; j < n; ++j) {
      W[col * n + j] /= dd;
      inv[col * n + j] /= dd;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = W[r * n + col];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        W[r * n + j] -= f * W[col * n + j];
        inv[r * n + j] -= f * inv[col * n + j];
      }
    }
  }
  M = inv;
  if (cond) {
    auto norm1 = [n](const std::vector<double>& X) {
      double best = 0.0;
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += std::abs(X[i * n + j]);
        best = s > best ? s : best;
      }
      return best;
    };
    *cond = norm1(A) * norm1(inv);
  }
}

int ipow(int b, int e) {
  int r = 1;
  while (e-- > 0) r *= b;
  return r;
}

bool valid_field(const hlf_solver* s, int f) { return f >= 0 && f < s->nfields; }

hlf_status ensure_staging(hlf_solver* s, size_t bytes) {
  if (!s->xstream) {
    HLF_CUDA(s, cudaStreamCreateWithFlags(&s->xstream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      HLF_CUDA(s, cudaEventCreateWithFlags(&s->copy_done[b], cudaEventDisableTiming));
      HLF_CUDA(s, cudaEventCreateWithFlags(&s->perm_done[b], cudaEventDisableTiming));
    }
  }
  if (s->staging_bytes >= bytes) return HLF_OK;
  for (double*& b : s->staging) {
    if (b) cudaFree(b);
    b = nullptr;
  }
  s->staging_bytes = 0;
  HLF_CUDA(s, cudaMalloc(&s->staging[0], bytes));
  HLF_CUDA(s, cudaMalloc(&s->staging[1], bytes));
  s->staging_bytes = bytes;
  return HLF_OK;
}

constexpr size_t kChunkBytes = size_t(256) << 20;

// host AoS [node][per] <-> device SoA [zoff+z][per][y][x], through two device
// staging chunks: the PCIe copy of chunk i (copy stream) overlaps the permute
// kernel of chunk i-1 (solver stream), ordered by per-buffer events
hlf_status transfer(hlf_solver* s, double* dev, const int* N, int per, int64_t layer, int zoff,
                    double* host, bool to_device) {
  const int64_t nodes = static_cast<int64_t>(N[0]) * N[1] * N[2];
  const int64_t chunk_nodes = std::max<int64_t>(1, static_cast<int64_t>(kChunkBytes / (sizeof(double) * per)));
  hlf_status st = ensure_staging(s, std::min<int64_t>(nodes, chunk_nodes) * per * sizeof(double));
  if (st != HLF_OK) return st;
  const int64_t coef = static_cast<int64_t>(N[0]) * N[1];
  // both buffers start free (and, for downloads, after the work queued on the solver stream)
  for (int b = 0; b < 2; ++b) {
    HLF_CUDA(s, cudaEventRecord(s->perm_done[b], s->stream));
    HLF_CUDA(s, cudaEventRecord(s->copy_done[b], s->stream));
  }
  int i = 0;
  for (int64_t n0 = 0; n0 < nodes; n0 += chunk_nodes, ++i) {
    const int b = i & 1;
    double* stg = s->staging[b];
    const int64_t cnt = std::min(chunk_nodes, nodes - n0);
    const size_t bytes = static_cast<size_t>(cnt) * per * sizeof(double);
    if (to_device) {
      HLF_CUDA(s, cudaStreamWaitEvent(s->xstream, s->perm_done[b], 0));  // buffer b consumed
      HLF_CUDA(s, cudaMemcpyAsync(stg, host + n0 * per, bytes, cudaMemcpyHostToDevice, s->xstream));
      HLF_CUDA(s, cudaEventRecord(s->copy_done[b], s->xstream));
      HLF_CUDA(s, cudaStreamWaitEvent(s->stream, s->copy_done[b], 0));
      s->launches += hlfk::launch_aos_to_soa(stg, dev, n0, cnt, per, N[0], N[1], N[2], layer, coef, zoff,
                                             s->stream);
      HLF_CUDA(s, cudaEventRecord(s->perm_done[b], s->stream));
    } else {
      HLF_CUDA(s, cudaStreamWaitEvent(s->stream, s->copy_done[b], 0));  // buffer b drained to the host
      s->launches += hlfk::launch_soa_to_aos(dev, stg, n0, cnt, per, N[0], N[1], N[2], layer, coef, zoff,
                                             s->stream);
      HLF_CUDA(s, cudaEventRecord(s->perm_done[b], s->stream));
      HLF_CUDA(s, cudaStreamWaitEvent(s->xstream, s->perm_done[b], 0));
      HLF_CUDA(s, cudaMemcpyAsync(host + n0 * per, stg, bytes, cudaMemcpyDeviceToHost, s->xstream));
      HLF_CUDA(s, cudaEventRecord(s->copy_done[b], s->xstream));
    }
    HLF_CUDA(s, cudaGetLastError());
  }
  HLF_CUDA(s, cudaStreamSynchronize(s->xstream));
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  return HLF_OK;
}

// z ghost layers for d = 3 (skipped in slab mode: the caller exchanges halos)
hlf_status fill_ghosts(hlf_solver* s, bool for_pressure) {
  if (s->d != 3 || s->z_slab) return HLF_OK;
  const int Kz = s->K[2];
  if (!for_pressure) {
    // velocity half step reads p layer Kz: periodic wrap = copy of layer 0
    if (s->bnd[2] == HLF_PERIODIC) {
      const int64_t L = s->layer_stride(0);
      HLF_CUDA(s, cudaMemcpyAsync(s->field[0] + Kz * L, s->field[0], L * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s->stream));
    }
    return HLF_OK;
  }
  for (int c = 1; c <= 3; ++c) {
    const int64_t L = s->layer_stride(c);
    double* base = s->field[c];
    if (s->bnd[2] == HLF_PERIODIC) {
      // ghost index 0 (z = -1) = layer z = Kz-1 (index Kz)
      HLF_CUDA(s, cudaMemcpyAsync(base, base + Kz * L, L * sizeof(double), cudaMemcpyDeviceToDevice,
                                  s->stream));
    } else {
      const double sigma = (c - 1) == 2 ? 1.0 : -1.0;  // wall-normal v_z even, tangential odd
      s->launches += hlfk::launch_mirror_layer(base, base + L, s->plane[c], s->n1, 3, sigma, s->stream);
      s->launches += hlfk::launch_mirror_layer(base + (Kz + 1) * L, base + Kz * L, s->plane[c], s->n1, 3,
                                               sigma, s->stream);
    }
  }
  HLF_CUDA(s, cudaGetLastError());
  return HLF_OK;
}

void fill_weights(const hlf_solver* s, hlfk::HalfKind kind, HalfParams& P) {
  std::memcpy(P.M, s->M.data(), sizeof(double) * s->M.size());
  // w_r = 2 prod_{q<=r} (dt/2)/q, exactly as leapfrog_half_update (stepper1d.cpp:57-58)
  for (int r = 0; r < s->n && r < hlfk::kMaxN; ++r) {
    double w = 2.0;
    for (int q = 1; q <= r; ++q) w *= s->dt / 2.0 / q;
    P.w[r] = w;
  }
  for (int k = 0; k <= s->m; ++k) {
    const int r = 2 * k + 1;
    double g = P.w[r];
    for (int q = 0; q < r; ++q) g /= s->h;
    const double a_pow = kind == hlfk::VEL ? std::pow(s->av, k + 1) * std::pow(s->ap, k)
                                           : std::pow(s->ap, k + 1) * std::pow(s->av, k);
    P.G[k] = g * a_pow;
  }
  P.inv_h = 1.0 / s->h;
  P.h = s->h;
  {
    int e2 = 0;
    P.pow2_h = std::frexp(s->h, &e2) == 0.5;
  }
  P.ap = s->ap;
  P.av = s->av;
}

// zlo/zhi: target layers [zlo, zhi) of a 3D half step (-1: all).  A range is
// the full launch with both field bases shifted by zlo layers, so every kernel
// runs it unchanged.
// variant 1 = the fast kernels: tiled3d / tiled2d (constant coefficients),
// var2d (2D with per-node ap jets)
bool tiled_available(const hlf_solver* s) {
  if (!s->m_mirror) return false;
  if (s->variable) return (s->d == 2 && hlfk::var2d_supported(s->m)) || (s->d == 3 && s->sep3d);  // sep3d: the coefficient lives in the kernel
  return (s->d == 3 && hlfk::tiled3d_supported(s->m)) || (s->d == 2 && hlfk::tiled2d_supported(s->m));
}

hlf_status launch_half(hlf_solver* s, hlfk::HalfKind kind, int step, int zlo = 0, int zhi = -1) {
  if (s->scheme != HLF_SCHEME_LEAPFROG)
    return fail(s, HLF_CONFIG_ERROR, "half steps belong to the leapfrog scheme; use hlf_step");
  hlf_status st = fill_ghosts(s, kind == hlfk::PRE);
  if (st != HLF_OK) return st;
  HalfParams P;
  std::memset(&P, 0, sizeof(P));
  fill_weights(s, kind, P);
  const int tf = kind == hlfk::VEL ? 1 : 0;  // first target field
  const int sf = kind == hlfk::VEL ? 0 : 1;  // first source field
  const int* tN = s->nodes_of(tf);
  const int* sN = s->nodes_of(sf);
  for (int c = 0; c < 3; ++c) {
    P.src[c] = c < (kind == hlfk::VEL ? 1 : s->d) ? s->field[sf + c] : nullptr;
    P.dst[c] = c < (kind == hlfk::VEL ? s->d : 1) ? s->field[tf + c] : nullptr;
    P.K[c] = s->K[c];
    P.bnd[c] = s->bnd[c];
  }
  P.s_layer = s->layer_stride(sf);
  P.s_coef = s->plane[sf];
  P.t_layer = s->layer_stride(tf);
  P.t_coef = s->plane[tf];
  P.sNx = sN[0];
  P.sNy = sN[1];
  P.tNx = tN[0];
  P.tNy = tN[1];
  P.tNz = tN[2];
  P.t_zoff = s->zoff(tf);
  P.s_zoff = s->zoff(sf);
  P.coeff = s->variable ? s->coeff[s->grid_of(tf)] : nullptr;
  P.c_coef = s->plane[tf];
  P.c_layer = s->plane[tf] * s->E;
  P.step = step;
  P.flag = s->flag;
  P.path_ctr = s->path_ctr;
  if (s->timing) {
    s->tev_idx = 0;
    P.launch_ev = s->tev;
    P.launch_idx = &s->tev_idx;
    HLF_CUDA(s, cudaEventRecord(s->tev[0], s->stream));
  }
  const int fg = s->grid_of(tf);
  if (s->force_on) {
    if (!s->force_fresh[fg])
      return fail(s, HLF_CONFIG_ERROR,
                  "forcing mode: set this half step's table with hlf_set_forcing (or hlf_clear_forcing)");
    P.force = s->force[fg];
    P.f_coef = s->plane[tf];
    P.f_layer = s->plane[tf] * (s->n - 1) * s->E;
  }
  if (zhi < 0) zhi = P.tNz;
  if (zlo < 0 || zhi > P.tNz || zlo > zhi || (s->d != 3 && (zlo != 0 || zhi != P.tNz)))
    return fail(s, HLF_INVALID_ARGUMENT, "layer range outside the target field (ranges are 3D only)");
  if (zlo == zhi) return HLF_OK;
  if (zlo > 0 || zhi < P.tNz) {
    for (int c = 0; c < 3; ++c)
      if (P.src[c]) P.src[c] += static_cast<int64_t>(zlo) * P.s_layer;
    if (P.coeff) P.coeff += static_cast<int64_t>(zlo) * P.c_layer;
    if (P.force) P.force += static_cast<int64_t>(zlo) * P.f_layer;
    P.t_zoff += zlo;
    P.tNz = zhi - zlo;
  }
  int launched = -1;
  if (s->variable && s->sep3d) {
    // coordinates of target node 0 (primary: x_min, dual: x_min + h/2; z from the layer range)
    for (int ax = 0; ax < 3; ++ax) P.sep_x0[ax] = s->x_min[ax] + (fg == HLF_DUAL ? 0.5 * s->h : 0.0);
    P.sep_x0[2] += zlo * s->h;
    std::memcpy(P.sep, s->sep, sizeof(P.sep));
    P.sep_on = 1;
  }
  if (P.force) {
    // forced half steps: the faithful kernels (the tiled / var kernels have no forcing term)
  } else if (s->variant == 1 && s->variable && s->sep3d && s->d == 3) {
    launched = hlfk::launch_half_var3d(s->m, kind, P, s->sep, P.sep_x0, s->stream);
  } else if (s->variant == 1 && !s->variable && s->d == 3 && hlfk::tiled3d_supported(s->m))
    launched = hlfk::launch_half_tiled3d(s->m, kind, P, s->stream);
  else if (s->variant == 1 && !s->variable && s->d == 2 && hlfk::tiled2d_supported(s->m))
    launched = hlfk::launch_half_tiled2d(s->m, kind, P, s->stream);
  else if (s->variant == 1 && s->variable && s->d == 2 && hlfk::var2d_supported(s->m))
    launched = hlfk::launch_half_var2d(s->m, kind, P, s->stream);
  if (launched < 0 && s->variable && s->sep3d)
    return fail(s, HLF_CONFIG_ERROR,
                "on-the-fly separable coefficients need the var2d / var3d kernel (variant 1)");
  if (launched == -2 || launched < 0 && (s->variant != 1 || P.force))  // -2: custom M / planes too large for the tiled kernel
    launched = hlfk::launch_half_generic(s->d, s->m, s->variable, kind, P, s->stream);
  if (launched < 0) return fail(s, HLF_CONFIG_ERROR, "no device kernel for this (dim, m)");
  if (s->timing && s->tev_idx == 0) mark_launch(P, s->stream);  // kernels without their own marks
  s->launches += launched;
  HLF_CUDA(s, cudaGetLastError());
  if (s->force_on) s->force_fresh[fg] = false;
  return HLF_OK;
}

hlf_status read_flag(hlf_solver* s, int* bad) {
  HLF_CUDA(s, cudaMemcpyAsync(s->flag_host, s->flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  *bad = *s->flag_host == INT_MAX ? -1 : *s->flag_host;
  return HLF_OK;
}

hlf_status instability(hlf_solver* s, int step) {
  return fail(s, HLF_INSTABILITY, "solution became non-finite at step " + std::to_string(step));
}

}  // namespace

extern "C" {

int hlf_abi_version(void) { return HLF_B200_ABI_VERSION; }

hlf_status hlf_build_interp_operator(int m, double* M_out, double* condition_out) {
  if (m < 0 || m > hlfk::kMaxM)
    return fail(nullptr, HLF_CONFIG_ERROR, "interpolation order m must be in [0, 8]");
  std::vector<double> M;
  build_M(m, M, condition_out);
  if (M_out) std::memcpy(M_out, M.data(), sizeof(double) * M.size());
  return HLF_OK;
}

hlf_status hlf_create(const hlf_desc* desc, hlf_solver** out) {
  if (!desc || !out) return fail(nullptr, HLF_INVALID_ARGUMENT, "null descriptor");
  *out = nullptr;
  const int d = desc->dim;
  if (d < 1 || d > 3) return fail(nullptr, HLF_CONFIG_ERROR, "dim must be 1, 2 or 3");
  if (desc->m < 0 || desc->m > hlfk::kMaxM)
    return fail(nullptr, HLF_CONFIG_ERROR, "scheme order m must be in [0, 8]");
  if (d == 3 && desc->m > 4)
    return fail(nullptr, HLF_CONFIG_ERROR, "3D device kernels support m <= 4");
  if (!(desc->h > 0.0) || !std::isfinite(desc->h))
    return fail(nullptr, HLF_CONFIG_ERROR, "grid spacing must be positive");
  for (int ax = 0; ax < d; ++ax) {
    if (desc->K[ax] < 2) return fail(nullptr, HLF_CONFIG_ERROR, "grid needs K >= 2");
    if (desc->boundary[ax] != HLF_PERIODIC && desc->boundary[ax] != HLF_REFLECTIVE)
      return fail(nullptr, HLF_CONFIG_ERROR, "unknown boundary kind");
  }
  if (desc->z_slab && (d != 3 || desc->boundary[2] != HLF_PERIODIC))
    return fail(nullptr, HLF_CONFIG_ERROR, "z slabs need d = 3 with a periodic z axis");
  if (desc->scheme < HLF_SCHEME_LEAPFROG || desc->scheme > HLF_SCHEME_MODIFIED_ADVECTION)
    return fail(nullptr, HLF_CONFIG_ERROR, "unknown time scheme");
  if (desc->scheme != HLF_SCHEME_LEAPFROG &&
      (d != 1 || desc->boundary[0] != HLF_PERIODIC || desc->variable_ap || desc->z_slab))
    return fail(nullptr, HLF_CONFIG_ERROR,
                "the modified and dual-Hermite schemes run in 1D, periodic, with constant coefficients");

  hlf_solver* s = new hlf_solver;
  s->d = d;
  s->m = desc->m;
  s->n1 = desc->m + 1;
  s->n = 2 * desc->m + 2;
  s->F = ipow(s->n1, d);
  s->E = ipow(s->n, d);
  s->h = desc->h;
  s->ap = desc->ap;
  s->av = desc->av;
  s->variable = desc->variable_ap != 0;
  s->z_slab = desc->z_slab != 0;
  s->scheme = desc->scheme;
  s->nfields = desc->scheme == HLF_SCHEME_LEAPFROG ? d + 1 : (desc->scheme == HLF_SCHEME_MODIFIED_ADVECTION ? 2 : 4);
  s->device = desc->device;
  for (int ax = 0; ax < 3; ++ax) {
    const bool used = ax < d;
    s->K[ax] = used ? desc->K[ax] : 1;
    s->bnd[ax] = used ? desc->boundary[ax] : HLF_PERIODIC;
    s->x_min[ax] = used ? desc->x_min[ax] : 0.0;
    s->Nd[ax] = s->K[ax];
    s->Np[ax] = used && s->bnd[ax] == HLF_REFLECTIVE ? s->K[ax] + 1 : s->K[ax];
  }
  if (desc->M) {
    s->M.assign(desc->M, desc->M + s->n * s->n);
  } else {
    build_M(s->m, s->M, nullptr);
  }
  {
    // a caller-supplied M without the mirror symmetry of A (interpolation.cpp:29-38)
    // runs on the generic kernel, which applies all n x n entries
    double mx = 0.0, dev = 0.0;
    for (double v : s->M) mx = std::max(mx, std::fabs(v));
    for (int r = 0; r < s->n; ++r)
      for (int l = 0; l < s->n1; ++l) {
        const double sg = ((r + l) & 1) ? -1.0 : 1.0;
        dev = std::max(dev, std::fabs(s->M[r * s->n + s->n1 + l] - sg * s->M[r * s->n + l]));
      }
    // the generated sweeps of the tiled kernels also omit the terms of the
    // entries that are exactly zero for the reference's M (even rows r >= 2,
    // l = 0, m <= 3; tools/gen_tiled3d.py mzero)
    bool zeros = true;
    for (int r = 2; r < s->n && s->m <= 3; r += 2) zeros = zeros && s->M[r * s->n] == 0.0;
    s->m_mirror = dev <= 1e-13 * mx && zeros;
  }
  auto bail = [&](hlf_status st) {
    g_create_error = s->err;
    hlf_destroy(s);
    return st;
  };
  cudaError_t e = cudaSetDevice(s->device);
  if (e != cudaSuccess) return bail(cuda_fail(s, e, "cudaSetDevice"));
  if (desc->stream) {
    s->stream = static_cast<cudaStream_t>(desc->stream);
  } else {
    e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(cuda_fail(s, e, "cudaStreamCreate"));
    s->own_stream = true;
  }
  for (int f = 0; f < s->nfields; ++f) {
    const int* N = s->nodes_of(f);
    s->plane[f] = static_cast<int64_t>(N[0]) * N[1];
    // d = 3: p gets one upper ghost/halo layer unless the z walls already
    // provide node Kz; every v component gets a ghost layer on each side
    s->layers[f] = d == 3 ? (f == 0 ? s->K[2] + 1 : s->K[2] + 2) : 1;
    const size_t bytes = static_cast<size_t>(s->layers[f]) * s->layer_stride(f) * sizeof(double);
    e = cudaMalloc(&s->field[f], bytes);
    if (e != cudaSuccess) return bail(cuda_fail(s, e, "cudaMalloc(field)"));
    e = cudaMemsetAsync(s->field[f], 0, bytes, s->stream);
    if (e != cudaSuccess) return bail(cuda_fail(s, e, "cudaMemset(field)"));
  }
  e = cudaMalloc(&s->flag, 2 * sizeof(int));
  if (e != cudaSuccess) return bail(cuda_fail(s, e, "cudaMalloc(flag)"));
  e = cudaMallocHost(&s->flag_host, sizeof(int));
  if (e != cudaSuccess) return bail(cuda_fail(s, e, "cudaMallocHost(flag)"));
  const int init_flag[2] = {INT_MAX, 0};  // [first bad step, graph step base]
  e = cudaMemcpyAsync(s->flag, init_flag, sizeof(init_flag), cudaMemcpyHostToDevice, s->stream);
  if (e != cudaSuccess) return bail(cuda_fail(s, e, "flag init"));
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return bail(cuda_fail(s, e, "sync"));
  s->variant = tiled_available(s) ? 1 : 0;
  *out = s;
  return HLF_OK;
}

void hlf_destroy(hlf_solver* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (double*& f : s->field)
    if (f) cudaFree(f);
  for (double*& c : s->coeff)
    if (c) cudaFree(c);
  for (double*& c : s->force)
    if (c) cudaFree(c);
  if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
  if (s->flag) cudaFree(s->flag);
  if (s->path_ctr) cudaFree(s->path_ctr);
  for (cudaEvent_t e : s->tev)
    if (e) cudaEventDestroy(e);
  if (s->flag_host) cudaFreeHost(s->flag_host);
  if (s->errbuf) cudaFree(s->errbuf);
  if (s->errbuf_host) cudaFreeHost(s->errbuf_host);
  for (double* b : s->staging)
    if (b) cudaFree(b);
  if (s->xstream) cudaStreamDestroy(s->xstream);
  for (int b = 0; b < 2; ++b) {
    if (s->copy_done[b]) cudaEventDestroy(s->copy_done[b]);
    if (s->perm_done[b]) cudaEventDestroy(s->perm_done[b]);
  }
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

const char* hlf_last_error(const hlf_solver* s) { return s ? s->err.c_str() : g_create_error.c_str(); }

int64_t hlf_num_nodes(const hlf_solver* s, int grid) { return s ? s->num_nodes(grid) : -1; }
int hlf_num_coeffs(const hlf_solver* s) { return s ? s->F : -1; }

hlf_status hlf_set_field(hlf_solver* s, int field, const double* host_aos) {
  if (!s || !valid_field(s, field) || !host_aos) return fail(s, HLF_INVALID_ARGUMENT, "bad field or buffer");
  cudaSetDevice(s->device);
  return transfer(s, s->field[field], s->nodes_of(field), s->F, s->layer_stride(field), s->zoff(field),
                  const_cast<double*>(host_aos), true);
}

hlf_status hlf_get_field(hlf_solver* s, int field, double* host_aos) {
  if (!s || !valid_field(s, field) || !host_aos) return fail(s, HLF_INVALID_ARGUMENT, "bad field or buffer");
  cudaSetDevice(s->device);
  return transfer(s, s->field[field], s->nodes_of(field), s->F, s->layer_stride(field), s->zoff(field),
                  host_aos, false);
}

hlf_status hlf_set_coeff(hlf_solver* s, int grid, const double* host_jets) {
  if (!s || (grid != HLF_PRIMARY && grid != HLF_DUAL) || !host_jets)
    return fail(s, HLF_INVALID_ARGUMENT, "bad grid or buffer");
  if (!s->variable) return fail(s, HLF_CONFIG_ERROR, "solver was created with constant coefficients");
  cudaSetDevice(s->device);
  if (s->sep3d) {
    s->sep3d = false;  // back to stored jets
    ++s->gen;
    if (s->d == 3) s->variant = tiled_available(s) ? 1 : 0;
  }
  const int* N = grid == HLF_PRIMARY ? s->Np : s->Nd;
  const int64_t plane = static_cast<int64_t>(N[0]) * N[1];
  if (!s->coeff[grid]) {
    const size_t bytes = static_cast<size_t>(s->num_nodes(grid)) * s->E * sizeof(double);
    HLF_CUDA(s, cudaMalloc(&s->coeff[grid], bytes));
    ++s->gen;
  }
  return transfer(s, s->coeff[grid], N, s->E, plane * s->E, 0, const_cast<double*>(host_jets), true);
}

hlf_status hlf_set_coeff_separable(hlf_solver* s, double c0, double c1, const double* w, const double* phase) {
  if (!s || !w || !phase) return HLF_INVALID_ARGUMENT;
  if (!s->variable) return fail(s, HLF_CONFIG_ERROR, "solver was created with constant coefficients");
  if (s->scheme != HLF_SCHEME_LEAPFROG) return fail(s, HLF_CONFIG_ERROR, "variable coefficients: leapfrog scheme only");
  cudaSetDevice(s->device);
  s->sep[0] = c0;
  s->sep[1] = c1;
  for (int a = 0; a < 3; ++a) {
    s->sep[2 + a] = a < s->d ? w[a] : 0.0;
    s->sep[5 + a] = a < s->d ? phase[a] : 0.0;
  }
  ++s->gen;
  if (((s->d == 3 && hlfk::var3d_supported(s->m)) || (s->d == 2 && hlfk::var2d_supported(s->m))) && s->m_mirror &&
      !s->force_on) {
    s->sep3d = true;  // generated inside the var3d / var2d kernel: nothing stored
    s->variant = 1;   // (the generic kernel reads stored jets)
    return HLF_OK;
  }
  s->sep3d = false;
  // other (d, m): expand into the stored per-node jets the var2d / generic kernels read
  for (int grid = 0; grid < 2; ++grid) {
    const int* N = grid == HLF_PRIMARY ? s->Np : s->Nd;
    if (!s->coeff[grid]) {
      const size_t bytes = static_cast<size_t>(s->num_nodes(grid)) * s->E * sizeof(double);
      HLF_CUDA(s, cudaMalloc(&s->coeff[grid], bytes));
    }
    double x0[3];
    for (int a = 0; a < 3; ++a) x0[a] = s->x_min[a] + (grid == HLF_DUAL ? 0.5 * s->h : 0.0);
    hlfk::launch_fill_sep_coeff(s->coeff[grid], s->d, N, s->n, s->h, x0, s->sep, s->stream);
    HLF_CUDA(s, cudaGetLastError());
  }
  return HLF_OK;
}

hlf_status hlf_set_forcing(hlf_solver* s, int grid, const double* host_table) {
  if (!s || (grid != HLF_PRIMARY && grid != HLF_DUAL) || !host_table)
    return fail(s, HLF_INVALID_ARGUMENT, "bad grid or buffer");
  if (s->scheme != HLF_SCHEME_LEAPFROG)
    return fail(s, HLF_CONFIG_ERROR, "forcing tables are supported for the leapfrog scheme");
  cudaSetDevice(s->device);
  if (s->sep3d) {
    // forced runs go through the generic kernel, which reads stored ap jets
    s->sep3d = false;
    for (int g = 0; g < 2; ++g) {
      const int* Ng = g == HLF_PRIMARY ? s->Np : s->Nd;
      if (!s->coeff[g]) {
        const size_t bytes = static_cast<size_t>(s->num_nodes(g)) * s->E * sizeof(double);
        HLF_CUDA(s, cudaMalloc(&s->coeff[g], bytes));
      }
      double x0[3];
      for (int a = 0; a < 3; ++a) x0[a] = s->x_min[a] + (g == HLF_DUAL ? 0.5 * s->h : 0.0);
      hlfk::launch_fill_sep_coeff(s->coeff[g], s->d, Ng, s->n, s->h, x0, s->sep, s->stream);
      HLF_CUDA(s, cudaGetLastError());
    }
  }
  const int* N = grid == HLF_PRIMARY ? s->Np : s->Nd;
  const int per = (s->n - 1) * s->E;
  if (!s->force[grid]) {
    const size_t bytes = static_cast<size_t>(s->num_nodes(grid)) * per * sizeof(double);
    HLF_CUDA(s, cudaMalloc(&s->force[grid], bytes));
  }
  const int64_t plane = static_cast<int64_t>(N[0]) * N[1];
  hlf_status st = transfer(s, s->force[grid], N, per, plane * per, 0, const_cast<double*>(host_table), true);
  if (st != HLF_OK) return st;
  s->force_on = true;
  s->force_fresh[grid] = true;
  return HLF_OK;
}

hlf_status hlf_clear_forcing(hlf_solver* s) {
  if (!s) return HLF_INVALID_ARGUMENT;
  s->force_on = false;
  s->force_fresh[0] = s->force_fresh[1] = false;
  return HLF_OK;
}

hlf_status hlf_set_times(hlf_solver* s, double t_p, double t_v, double dt) {
  if (!s) return fail(s, HLF_INVALID_ARGUMENT, "null solver");
  s->t_p = t_p;
  s->t_v = t_v;
  s->dt = dt;
  return HLF_OK;
}

hlf_status hlf_get_times(const hlf_solver* s, double* t_p, double* t_v, double* dt) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (t_p) *t_p = s->t_p;
  if (t_v) *t_v = s->t_v;
  if (dt) *dt = s->dt;
  return HLF_OK;
}

hlf_status hlf_set_dt(hlf_solver* s, double dt) {
  if (!s) return HLF_INVALID_ARGUMENT;
  s->dt = dt;
  return HLF_OK;
}

hlf_status hlf_advance_p(hlf_solver* s) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (s->variable && !s->coeff_ready(HLF_PRIMARY)) return fail(s, HLF_CONFIG_ERROR, "primary-grid ap jets not set");
  cudaSetDevice(s->device);
  hlf_status st = launch_half(s, hlfk::PRE, -1);
  if (st != HLF_OK) return st;
  s->t_p += s->dt;
  return HLF_OK;
}

hlf_status hlf_advance_v(hlf_solver* s) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (s->variable && !s->coeff_ready(HLF_DUAL)) return fail(s, HLF_CONFIG_ERROR, "dual-grid ap jets not set");
  cudaSetDevice(s->device);
  hlf_status st = launch_half(s, hlfk::VEL, -1);
  if (st != HLF_OK) return st;
  s->t_v += s->dt;
  return HLF_OK;
}

hlf_status hlf_advance_p_indexed(hlf_solver* s, int step_index) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (s->variable && !s->coeff_ready(HLF_PRIMARY)) return fail(s, HLF_CONFIG_ERROR, "primary-grid ap jets not set");
  cudaSetDevice(s->device);
  hlf_status st = launch_half(s, hlfk::PRE, step_index);
  if (st != HLF_OK) return st;
  s->t_p += s->dt;
  return HLF_OK;
}

hlf_status hlf_advance_v_indexed(hlf_solver* s, int step_index) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (s->variable && !s->coeff_ready(HLF_DUAL)) return fail(s, HLF_CONFIG_ERROR, "dual-grid ap jets not set");
  cudaSetDevice(s->device);
  hlf_status st = launch_half(s, hlfk::VEL, step_index);
  if (st != HLF_OK) return st;
  s->t_v += s->dt;
  return HLF_OK;
}

hlf_status hlf_advance_layers(hlf_solver* s, int half, int step_index, int z_begin, int z_end) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (half != 0 && half != 1) return fail(s, HLF_INVALID_ARGUMENT, "half must be 0 (pressure) or 1 (velocity)");
  if (s->variable && !s->coeff_ready(half == 0 ? HLF_PRIMARY : HLF_DUAL))
    return fail(s, HLF_CONFIG_ERROR, "ap jets not set");
  cudaSetDevice(s->device);
  return launch_half(s, half == 0 ? hlfk::PRE : hlfk::VEL, step_index, z_begin, z_end);
}

hlf_status hlf_commit_half(hlf_solver* s, int half) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (half == 0) s->t_p += s->dt;
  else if (half == 1) s->t_v += s->dt;
  else return fail(s, HLF_INVALID_ARGUMENT, "half must be 0 (pressure) or 1 (velocity)");
  return HLF_OK;
}

// one step of the 1D modified / dual-Hermite scheme (stepper1d.cpp:191-272)
static hlf_status scheme1d_step(hlf_solver* s, int step_index) {
  hlfk::Scheme1dParams P;
  std::memset(&P, 0, sizeof(P));
  std::memcpy(P.M, s->M.data(), sizeof(double) * s->M.size());
  P.h = s->h;
  P.inv_h = 1.0 / s->h;
  {
    int e2 = 0;
    P.pow2_h = std::frexp(s->h, &e2) == 0.5;
  }
  P.ap = s->ap;
  P.av = s->av;
  P.dt = s->dt;
  P.K = s->K[0];
  P.step = step_index;
  P.flag = s->flag;
  int launched = 0;
  if (s->scheme == HLF_SCHEME_MODIFIED_ADVECTION) {
    // the single-field branch of step_modified (stepper1d.cpp:205-209):
    // ck_advection's recurrence U_{r+1} = a D U_r (:40-52) is the two-table
    // recurrence with both tables seeded by the same reconstruction and
    // av = ap (the tables stay equal level by level, value for value), so the
    // two-field kernel runs it with the second field aliased to the first
    P.av = s->ap;
    P.to_primary = 1;
    P.src_p = P.src_v = s->field[1];
    P.dst_p = P.dst_v = s->field[0];
    launched += hlfk::launch_modified_1d(s->m, P, s->stream);
    P.to_primary = 0;
    P.src_p = P.src_v = s->field[0];
    P.dst_p = P.dst_v = s->field[1];
    launched += hlfk::launch_modified_1d(s->m, P, s->stream);
  } else if (s->scheme == HLF_SCHEME_MODIFIED) {
    // primary update from the dual copies, then dual update from the new primary
    P.to_primary = 1;
    P.src_p = s->field[3];
    P.src_v = s->field[1];
    P.dst_p = s->field[0];
    P.dst_v = s->field[2];
    launched += hlfk::launch_modified_1d(s->m, P, s->stream);
    P.to_primary = 0;
    P.src_p = s->field[0];
    P.src_v = s->field[2];
    P.dst_p = s->field[3];
    P.dst_v = s->field[1];
    launched += hlfk::launch_modified_1d(s->m, P, s->stream);
  } else {
    P.src_p = s->field[0];
    P.src_v = s->field[2];
    P.dst_p = s->field[1];
    P.dst_v = s->field[3];
    launched += hlfk::launch_dual_hermite_1d(s->m, 0, P, s->stream);
    P.src_p = s->field[1];
    P.src_v = s->field[3];
    P.dst_p = s->field[0];
    P.dst_v = s->field[2];
    launched += hlfk::launch_dual_hermite_1d(s->m, 1, P, s->stream);
  }
  s->launches += launched;
  HLF_CUDA(s, cudaGetLastError());
  s->t_p += s->dt;
  s->t_v = s->scheme == HLF_SCHEME_DUAL_HERMITE ? s->t_p : s->t_p + s->dt / 2.0;
  return HLF_OK;
}

static hlf_status step_async(hlf_solver* s, int step_index) {
  if (s->scheme != HLF_SCHEME_LEAPFROG) return scheme1d_step(s, step_index);
  if (s->variable && (!s->coeff_ready(0) || !s->coeff_ready(1))) return fail(s, HLF_CONFIG_ERROR, "ap jets not set");
  hlf_status st = launch_half(s, hlfk::PRE, step_index);
  if (st != HLF_OK) return st;
  s->t_p += s->dt;
  st = launch_half(s, hlfk::VEL, step_index);
  if (st != HLF_OK) return st;
  s->t_v += s->dt;
  return HLF_OK;
}

__global__ void set_graph_step_base(int* flag, int base) { flag[1] = base; }
// flag[0] = INT_MAX (no non-finite value seen): every hlf_step / hlf_advance_n
// checks only the steps it runs, as check_finite (stepper1d.cpp:121-129) looks
// only at the current state
__global__ void reset_finite_flag(int* flag) { flag[0] = INT_MAX; }

static hlf_status reset_flag(hlf_solver* s) {
  reset_finite_flag<<<1, 1, 0, s->stream>>>(s->flag);
  s->launches += 1;
  HLF_CUDA(s, cudaGetLastError());
  return HLF_OK;
}

// host time stamps of one step, as step_async / scheme1d_step advance them
static void advance_times(hlf_solver* s) {
  s->t_p += s->dt;
  if (s->scheme == HLF_SCHEME_LEAPFROG) s->t_v += s->dt;
  else s->t_v = s->scheme == HLF_SCHEME_DUAL_HERMITE ? s->t_p : s->t_p + s->dt / 2.0;
}

// capture `chunk` steps (step offsets 0..chunk-1) into s->graph_exec; on any
// capture problem graphs are switched off and the caller launches directly
static void ensure_graph(hlf_solver* s, int chunk) {
  if (s->graph_exec && s->graph_steps == chunk && s->graph_dt == s->dt && s->graph_variant == s->variant &&
      s->graph_gen == s->gen)
    return;
  if (s->graph_exec) cudaGraphExecDestroy(s->graph_exec);
  s->graph_exec = nullptr;
  const double t_p = s->t_p, t_v = s->t_v;
  const int64_t launches = s->launches;
  hlf_status st = HLF_OK;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
    for (int k = 0; k < chunk && st == HLF_OK; ++k) st = step_async(s, k);
    if (cudaStreamEndCapture(s->stream, &g) != cudaSuccess) st = HLF_CUDA_ERROR;
  } else {
    st = HLF_CUDA_ERROR;
  }
  s->t_p = t_p;
  s->t_v = t_v;
  s->graph_kernels = static_cast<int>(s->launches - launches);
  s->launches = launches;
  if (st == HLF_OK && g && cudaGraphInstantiate(&s->graph_exec, g, 0) == cudaSuccess) {
    s->graph_steps = chunk;
    s->graph_dt = s->dt;
    s->graph_variant = s->variant;
    s->graph_gen = s->gen;
  } else {
    s->graph_exec = nullptr;
    s->graph_chunk = 0;  // fall back to direct launches for this solver
  }
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
}

hlf_status hlf_set_graph_steps(hlf_solver* s, int steps) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (steps < 0) return fail(s, HLF_INVALID_ARGUMENT, "negative graph chunk");
  s->graph_chunk = steps;
  return HLF_OK;
}

hlf_status hlf_step(hlf_solver* s, int step_index) {
  if (!s) return HLF_INVALID_ARGUMENT;
  cudaSetDevice(s->device);
  hlf_status st = reset_flag(s);
  if (st != HLF_OK) return st;
  st = step_async(s, step_index);
  if (st != HLF_OK) return st;
  int bad = -1;
  st = read_flag(s, &bad);
  if (st != HLF_OK) return st;
  return bad >= 0 ? instability(s, bad) : HLF_OK;
}

hlf_status hlf_advance_n(hlf_solver* s, int n, int first_step) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (n < 0) return fail(s, HLF_INVALID_ARGUMENT, "negative step count");
  cudaSetDevice(s->device);
  {
    hlf_status st = reset_flag(s);
    if (st != HLF_OK) return st;
  }
  int i = 0;
  const int chunk = s->graph_chunk;
  if (chunk > 0 && n >= 2 * chunk && !s->force_on && !s->z_slab) {
    // the first step runs directly (one-time launch set-up stays out of the
    // capture), then whole chunks replay the graph with their step base
    hlf_status st = step_async(s, first_step);
    if (st != HLF_OK) return st;
    i = 1;
    ensure_graph(s, chunk);
    if (s->graph_exec) {
      for (; n - i >= chunk; i += chunk) {
        set_graph_step_base<<<1, 1, 0, s->stream>>>(s->flag, first_step + i);
        HLF_CUDA(s, cudaGraphLaunch(s->graph_exec, s->stream));
        for (int k = 0; k < chunk; ++k) advance_times(s);
        s->launches += s->graph_kernels + 1;
      }
      set_graph_step_base<<<1, 1, 0, s->stream>>>(s->flag, 0);
      s->launches += 1;
      HLF_CUDA(s, cudaGetLastError());
    }
  }
  for (; i < n; ++i) {
    hlf_status st = step_async(s, first_step + i);
    if (st != HLF_OK) return st;
  }
  int bad = -1;
  hlf_status st = read_flag(s, &bad);
  if (st != HLF_OK) return st;
  return bad >= 0 ? instability(s, bad) : HLF_OK;
}

hlf_status hlf_plan_steps(double T, double dt_nominal, int* n_out, double* dt_out) {
  // step_count (config.cpp:34-38) and the caller's dt = T / n (tests/test_stepper1d.cpp:33-35)
  if (!(T > 0.0)) return fail(nullptr, HLF_CONFIG_ERROR, "final time must be positive");
  if (!(dt_nominal > 0.0)) return fail(nullptr, HLF_CONFIG_ERROR, "nominal dt must be positive");
  const double q = std::ceil(T / dt_nominal);
  if (!(q < 2147483647.0)) return fail(nullptr, HLF_CONFIG_ERROR, "step count overflows int");
  const int n = static_cast<int>(q);
  if (n_out) *n_out = n;
  if (dt_out) *dt_out = T / n;
  return HLF_OK;
}

hlf_status hlf_advance_to(hlf_solver* s, double T, int first_step, int* steps_out) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (steps_out) *steps_out = 0;
  const double span = T - s->t_p;
  if (!(s->dt != 0.0) || !std::isfinite(s->dt) || !std::isfinite(T))
    return fail(s, HLF_CONFIG_ERROR, "advance_to needs a finite nonzero dt and T");
  const double q = span / s->dt;
  if (q < -1e-9) return fail(s, HLF_CONFIG_ERROR, "T lies behind the state's time in the direction of dt");
  const double nr = std::nearbyint(q);
  // the staggered partner was initialised half a step of this dt away
  // (init_leapfrog, stepper1d.cpp:131-145): dt cannot change here, so it has
  // to divide the remaining time
  if (std::fabs(q - nr) > 1e-9 * std::max(1.0, std::fabs(q)) || nr > 2147483647.0)
    return fail(s, HLF_CONFIG_ERROR,
                "dt does not divide T - t_p; initialise the state with dt = T / step_count(T, dt_nominal)");
  const int n = static_cast<int>(nr);
  hlf_status st = hlf_advance_n(s, n, first_step);
  if (steps_out) *steps_out = n;
  return st;
}

hlf_status hlf_poll_finite(hlf_solver* s, int* first_bad_step) {
  if (!s || !first_bad_step) return HLF_INVALID_ARGUMENT;
  cudaSetDevice(s->device);
  return read_flag(s, first_bad_step);
}

hlf_status hlf_clear_finite(hlf_solver* s) {
  if (!s) return HLF_INVALID_ARGUMENT;
  cudaSetDevice(s->device);
  *s->flag_host = INT_MAX;
  HLF_CUDA(s, cudaMemcpyAsync(s->flag, s->flag_host, sizeof(int), cudaMemcpyHostToDevice, s->stream));
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  return HLF_OK;
}

hlf_status hlf_synchronize(hlf_solver* s) {
  if (!s) return HLF_INVALID_ARGUMENT;
  cudaSetDevice(s->device);
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  return HLF_OK;
}

hlf_status hlf_field_device(hlf_solver* s, int field, double** dev_ptr, int64_t* layer_stride,
                            int64_t* coef_stride, int* layers) {
  if (!s || !valid_field(s, field)) return fail(s, HLF_INVALID_ARGUMENT, "bad field");
  if (dev_ptr) *dev_ptr = s->field[field];
  if (layer_stride) *layer_stride = s->layer_stride(field);
  if (coef_stride) *coef_stride = s->plane[field];
  if (layers) *layers = s->layers[field];
  return HLF_OK;
}

hlf_status hlf_fill_separable(hlf_solver* s, int field, double amp, const double* w, const double* phase) {
  if (!s || !valid_field(s, field) || !w || !phase) return fail(s, HLF_INVALID_ARGUMENT, "bad field");
  cudaSetDevice(s->device);
  hlfk::FillParams P;
  std::memset(&P, 0, sizeof(P));
  const int* N = s->nodes_of(field);
  P.dst = s->field[field];
  P.layer = s->layer_stride(field);
  P.coef = s->plane[field];
  P.Nx = N[0];
  P.Ny = N[1];
  P.Nz = N[2];
  P.zoff = s->zoff(field);
  P.d = s->d;
  P.n1 = s->n1;
  P.h = s->h;
  P.amp = amp;
  for (int ax = 0; ax < 3; ++ax) {
    P.x0[ax] = s->x_min[ax] + (field == 0 ? 0.0 : 0.5 * s->h);
    P.w[ax] = ax < s->d ? w[ax] : 0.0;
    P.phase[ax] = ax < s->d ? phase[ax] : 0.0;
  }
  s->launches += hlfk::launch_fill(P, s->stream);
  HLF_CUDA(s, cudaGetLastError());
  return HLF_OK;
}

hlf_status hlf_error_separable(hlf_solver* s, int field, double amp, const double* w, const double* phase,
                               double* rms_value, double* max_jet) {
  if (!s || !valid_field(s, field) || !w || !phase || !rms_value || !max_jet)
    return fail(s, HLF_INVALID_ARGUMENT, "bad argument");
  cudaSetDevice(s->device);
  if (!s->errbuf) {
    HLF_CUDA(s, cudaMalloc(&s->errbuf, 2 * sizeof(double)));
    HLF_CUDA(s, cudaMallocHost(&s->errbuf_host, 2 * sizeof(double)));
  }
  hlfk::FillParams P;
  std::memset(&P, 0, sizeof(P));
  const int* N = s->nodes_of(field);
  P.dst = s->field[field];
  P.layer = s->layer_stride(field);
  P.coef = s->plane[field];
  P.Nx = N[0];
  P.Ny = N[1];
  P.Nz = N[2];
  P.zoff = s->zoff(field);
  P.d = s->d;
  P.n1 = s->n1;
  P.h = s->h;
  P.amp = amp;
  P.err = s->errbuf;
  for (int ax = 0; ax < 3; ++ax) {
    P.x0[ax] = s->x_min[ax] + (field == 0 ? 0.0 : 0.5 * s->h);
    P.w[ax] = ax < s->d ? w[ax] : 0.0;
    P.phase[ax] = ax < s->d ? phase[ax] : 0.0;
  }
  HLF_CUDA(s, cudaMemsetAsync(s->errbuf, 0, 2 * sizeof(double), s->stream));
  s->launches += hlfk::launch_error(P, s->stream);
  HLF_CUDA(s, cudaGetLastError());
  HLF_CUDA(s, cudaMemcpyAsync(s->errbuf_host, s->errbuf, 2 * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  const double nodes = static_cast<double>(N[0]) * N[1] * N[2];
  *rms_value = std::sqrt(s->errbuf_host[0] / nodes);
  *max_jet = s->errbuf_host[1];
  return HLF_OK;
}

// n-point Gauss-Legendre rule on [-1, 1] (Newton on P_n; gauss_rule,
// analysis.cpp:15-33, takes the same nodes from GSL)
static void gauss_legendre(int n, double* x, double* w) {
  const double pi = 3.141592653589793238462643383279502884;
  for (int i = 0; i < n; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) p0 = 1.0;
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[n - 1 - i] = z;
    w[n - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

hlf_status hlf_l2_error_separable(hlf_solver* s, int field, double amp, const double* w, const double* phase,
                                  double* l2) {
  if (!s || !valid_field(s, field) || !w || !phase || !l2) return fail(s, HLF_INVALID_ARGUMENT, "bad argument");
  const int grid = s->grid_of(field);
  if (s->z_slab) return fail(s, HLF_CONFIG_ERROR, "the Gauss L2 accessor runs on whole (non-slab) domains");
  for (int ax = 0; ax < s->d; ++ax)
    if (grid == HLF_DUAL && s->bnd[ax] != HLF_PERIODIC)
      return fail(s, HLF_CONFIG_ERROR,
                  "the Gauss L2 of a dual-grid field needs periodic axes (wall cells are clipped)");
  if (s->d == 3 && s->m > 4) return fail(s, HLF_CONFIG_ERROR, "3D: m <= 4");
  cudaSetDevice(s->device);
  if (!s->errbuf) {
    HLF_CUDA(s, cudaMalloc(&s->errbuf, 2 * sizeof(double)));
    HLF_CUDA(s, cudaMallocHost(&s->errbuf_host, 2 * sizeof(double)));
  }
  hlfk::L2Params P;
  std::memset(&P, 0, sizeof(P));
  std::memcpy(P.M, s->M.data(), sizeof(double) * s->M.size());
  gauss_legendre(s->n, P.gx, P.gw);
  P.src = s->field[field];
  P.layer = s->layer_stride(field);
  P.coef = s->plane[field];
  P.zoff = s->zoff(field);
  P.Nx = s->nodes_of(field)[0];
  P.shift = grid == HLF_PRIMARY ? 0 : 1;
  P.h = s->h;
  P.n = s->n;
  P.n1 = s->n1;
  P.d = s->d;
  P.amp = amp;
  P.out = s->errbuf;
  for (int ax = 0; ax < 3; ++ax) {
    const bool used = ax < s->d;
    P.cells[ax] = used ? s->K[ax] : 1;
    P.wrap[ax] = used && s->bnd[ax] == HLF_PERIODIC;
    P.xc0[ax] = used ? s->x_min[ax] + (grid == HLF_PRIMARY ? 0.5 * s->h : 0.0) : 0.0;
    P.w[ax] = used ? w[ax] : 0.0;
    P.phase[ax] = used ? phase[ax] : 0.0;
  }
  HLF_CUDA(s, cudaMemsetAsync(s->errbuf, 0, sizeof(double), s->stream));
  s->launches += hlfk::launch_l2(P, s->stream);
  HLF_CUDA(s, cudaGetLastError());
  HLF_CUDA(s, cudaMemcpyAsync(s->errbuf_host, s->errbuf, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  *l2 = std::sqrt(s->errbuf_host[0]);
  return HLF_OK;
}

hlf_status hlf_energy_1d(hlf_solver* s, int kind, double c, double* energy) {
  if (!s || !energy || (kind != 0 && kind != 1)) return fail(s, HLF_INVALID_ARGUMENT, "bad argument");
  if (s->d != 1 || s->bnd[0] != HLF_PERIODIC || s->scheme != HLF_SCHEME_LEAPFROG)
    return fail(s, HLF_CONFIG_ERROR, "the discrete energy is defined for the 1D periodic leapfrog");
  const double sh = c * s->dt / 2.0;
  if (!(std::fabs(sh) < 0.5 * s->h)) return fail(s, HLF_CONFIG_ERROR, "|c dt / 2| must be below h / 2");
  cudaSetDevice(s->device);
  if (!s->errbuf) {
    HLF_CUDA(s, cudaMalloc(&s->errbuf, 2 * sizeof(double)));
    HLF_CUDA(s, cudaMallocHost(&s->errbuf_host, 2 * sizeof(double)));
  }
  hlfk::EnergyParams P;
  std::memset(&P, 0, sizeof(P));
  std::memcpy(P.M, s->M.data(), sizeof(double) * s->M.size());
  gauss_legendre(s->n1, P.gx, P.gw);
  P.f = s->field[kind == 0 ? 0 : 1];
  P.g = s->field[kind == 0 ? 1 : 0];
  P.coef = s->plane[0];
  P.f_primary = kind == 0;
  P.K = s->K[0];
  P.n = s->n;
  P.n1 = s->n1;
  P.x0 = s->x_min[0];
  P.h = s->h;
  P.s = sh;
  P.out = s->errbuf;
  HLF_CUDA(s, cudaMemsetAsync(s->errbuf, 0, sizeof(double), s->stream));
  s->launches += hlfk::launch_energy_1d(P, s->stream);
  HLF_CUDA(s, cudaGetLastError());
  HLF_CUDA(s, cudaMemcpyAsync(s->errbuf_host, s->errbuf, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  *energy = s->errbuf_host[0];
  return HLF_OK;
}

hlf_status hlf_zero_field(hlf_solver* s, int field) {
  if (!s || !valid_field(s, field)) return fail(s, HLF_INVALID_ARGUMENT, "bad field");
  cudaSetDevice(s->device);
  const size_t bytes = static_cast<size_t>(s->layers[field]) * s->layer_stride(field) * sizeof(double);
  HLF_CUDA(s, cudaMemsetAsync(s->field[field], 0, bytes, s->stream));
  return HLF_OK;
}

hlf_status hlf_halo_send_ptr(hlf_solver* s, int kind, int comp, double** dev_ptr, int64_t* count) {
  if (!s || s->d != 3 || (kind == 1 && (comp < 0 || comp > 2)))
    return fail(s, HLF_INVALID_ARGUMENT, "halos exist for d = 3 only");
  const int Kz = s->K[2];
  if (kind == 0) {
    *dev_ptr = s->field[0];  // p layer 0 -> previous rank's layer Kz
    *count = s->layer_stride(0);
  } else {
    *dev_ptr = s->field[1 + comp] + Kz * s->layer_stride(1 + comp);  // v layer Kz-1 -> next rank's ghost
    *count = s->layer_stride(1 + comp);
  }
  return HLF_OK;
}

hlf_status hlf_halo_recv_ptr(hlf_solver* s, int kind, int comp, double** dev_ptr, int64_t* count) {
  if (!s || s->d != 3 || (kind == 1 && (comp < 0 || comp > 2)))
    return fail(s, HLF_INVALID_ARGUMENT, "halos exist for d = 3 only");
  const int Kz = s->K[2];
  if (kind == 0) {
    *dev_ptr = s->field[0] + Kz * s->layer_stride(0);
    *count = s->layer_stride(0);
  } else {
    *dev_ptr = s->field[1 + comp];
    *count = s->layer_stride(1 + comp);
  }
  return HLF_OK;
}

int64_t hlf_launch_count(const hlf_solver* s) { return s ? s->launches : -1; }
void* hlf_get_stream(const hlf_solver* s) { return s ? static_cast<void*>(s->stream) : nullptr; }

hlf_status hlf_enable_path_counters(hlf_solver* s, int on) {
  if (!s) return HLF_INVALID_ARGUMENT;
  cudaSetDevice(s->device);
  if (on) {
    if (!s->path_ctr) HLF_CUDA(s, cudaMalloc(&s->path_ctr, 6 * sizeof(unsigned long long)));
    HLF_CUDA(s, cudaMemsetAsync(s->path_ctr, 0, 6 * sizeof(unsigned long long), s->stream));
  } else if (s->path_ctr) {
    HLF_CUDA(s, cudaStreamSynchronize(s->stream));
    cudaFree(s->path_ctr);
    s->path_ctr = nullptr;
  }
  s->gen++;  // a captured graph holds the old parameter blocks
  return HLF_OK;
}

hlf_status hlf_time_launches(hlf_solver* s, int steps, int first_step, double* ms_out, int* launches_out) {
  if (!s || !ms_out || steps <= 0) return HLF_INVALID_ARGUMENT;
  if (s->scheme != HLF_SCHEME_LEAPFROG) return fail(s, HLF_CONFIG_ERROR, "launch timing covers the leapfrog scheme");
  cudaSetDevice(s->device);
  for (cudaEvent_t& e : s->tev)
    if (!e) HLF_CUDA(s, cudaEventCreate(&e));
  double acc[2][3] = {{0, 0, 0}, {0, 0, 0}};
  int nl[2] = {0, 0};
  s->timing = true;
  hlf_status st = HLF_OK;
  for (int i = 0; i < steps && st == HLF_OK; ++i) {
    // step_system order: pressure (advance_p) then velocity (advance_v)
    for (int half = 0; half < 2 && st == HLF_OK; ++half) {
      const hlfk::HalfKind kind = half == 0 ? hlfk::PRE : hlfk::VEL;
      st = launch_half(s, kind, first_step + i);
      if (st != HLF_OK) break;
      if (half == 0) s->t_p += s->dt;
      else s->t_v += s->dt;
      const int k = kind == hlfk::VEL ? 0 : 1;
      nl[k] = s->tev_idx;
      if (cudaEventSynchronize(s->tev[s->tev_idx]) != cudaSuccess) {
        st = cuda_fail(s, cudaGetLastError(), "launch timing");
        break;
      }
      for (int j = 0; j < s->tev_idx; ++j) {
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, s->tev[j], s->tev[j + 1]);
        acc[k][j] += ms;
      }
    }
  }
  s->timing = false;
  if (st != HLF_OK) return st;
  for (int k = 0; k < 2; ++k)
    for (int j = 0; j < 3; ++j) ms_out[3 * k + j] = j < nl[k] ? acc[k][j] / steps : 0.0;
  if (launches_out) {
    launches_out[0] = nl[0];
    launches_out[1] = nl[1];
  }
  return HLF_OK;
}

hlf_status hlf_read_path_counters(hlf_solver* s, int64_t* out6) {
  if (!s || !out6) return HLF_INVALID_ARGUMENT;
  cudaSetDevice(s->device);
  unsigned long long h[6] = {0, 0, 0, 0, 0, 0};
  if (s->path_ctr) {
    HLF_CUDA(s, cudaMemcpyAsync(h, s->path_ctr, sizeof(h), cudaMemcpyDeviceToHost, s->stream));
    HLF_CUDA(s, cudaStreamSynchronize(s->stream));
  }
  for (int i = 0; i < 6; ++i) out6[i] = static_cast<int64_t>(h[i]);
  return HLF_OK;
}
int hlf_kernel_variant(const hlf_solver* s) { return s ? s->variant : -1; }

hlf_status hlf_set_kernel_variant(hlf_solver* s, int variant) {
  if (!s) return HLF_INVALID_ARGUMENT;
  if (variant == 1 && !tiled_available(s))
    return fail(s, HLF_CONFIG_ERROR, "tiled kernel not available for this configuration");
  if (variant != 0 && variant != 1) return fail(s, HLF_INVALID_ARGUMENT, "unknown variant");
  s->variant = variant;
  ++s->gen;
  return HLF_OK;
}

}  // extern "C"
