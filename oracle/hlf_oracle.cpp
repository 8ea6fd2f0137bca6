// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// CPU restatement of the Hermite-leapfrog staggered half steps of
// arXiv 1808.10481 for d = 1, 2, 3, written in the reference's own idiom so it
// can serve as the parity checker for the CUDA path.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg load this library.
//
// What it follows (reference = /root/reference):
//   * scaled jets u_i = h^i/i! d^i u                      proj/include/hlf/jet.hpp:7-9
//   * tensor jets, x-major row order                       proj/include/hlf/jet.hpp:34-46
//   * M = A^{-1}, A[h(m+1)+l][s] = C(s,l) (-/+1/2)^{s-l}   proj/src/interpolation.cpp:21-51
//   * 1D matvec                                            proj/src/interpolation.cpp:53-61
//   * tensor reconstruction: sweep x, then y (then z)      proj/src/interpolation.cpp:77-113
//   * truncated tensor derivative / product                proj/src/jet.cpp:109-135
//   * coupled CK recurrence, count = 2m+2                  proj/src/stepper1d.cpp:22-38, 94
//     P[r+1] = ap (.) sum_c d_c V_c[r],  V_c[r+1] = av (.) d_c P[r]
//     (1D: P[r+1] = ap (.) D V[r], V[r+1] = av (.) D P[r])
//   * odd-r leapfrog weights w_r = 2 prod_{q<=r} (dt/2)/q    proj/src/stepper1d.cpp:54-61
//   * advance_p then advance_v, then finite check          proj/src/stepper1d.cpp:147-172
//   * coefficient jets taken at the target node            proj/src/stepper1d.cpp:103-110,150-164
//   * reflective walls on primary lines, one mirrored ghost dual layer per wall,
//     ghost = sigma (-1)^{i_n} interior  (
//     sigma = +1 wall-normal velocity, -1 tangential)
// The reference ships no d>1 stepper; d = 1 is pinned
// against the compiled reference (oracle/_ref) and d > 1 through dimensional
// reduction, polynomial exactness and the paper's rates (tests/).
//
// Host layout (shared with the product's set/get_field): node (ix, iy, iz) is
// row ((ix * Ny) + iy) * Nz + iz (x-major, as PiecewiseTensor::cell,
// proj/include/hlf/interpolation.hpp:50-52); coefficient (a, b, c) is
// (a * n1 + b) * n1 + c (x-major, as TensorJet::at, jet.hpp:43-44).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

double binom(int s, int l) {
  double b = 1.0;
  for (int q = 0; q < l; ++q) b = b * (s - q) / (q + 1);
  return b;
}

// Gauss-Jordan with partial pivoting: the same elimination the shim gives the
// compiled reference (oracle/shim/Eigen/Dense), so M agrees with it bit for bit.
std::vector<double> build_M(int m) {
  const int n = 2 * m + 2;
  std::vector<double> A(static_cast<size_t>(n) * n, 0.0), inv(static_cast<size_t>(n) * n, 0.0);
  for (int half = 0; half < 2; ++half) {
    const double xi = half == 0 ? -0.5 : 0.5;
    for (int l = 0; l <= m; ++l) {
      const int row = half * (m + 1) + l;
      for (int s = l; s < n; ++s) A[row * n + s] = binom(s, l) * std::pow(xi, s - l);
    }
  }
  for (int i = 0; i < n; ++i) inv[i * n + i] = 1.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(A[r * n + col]) > std::abs(A[piv * n + col])) piv = r;
    if (piv != col)
      for (int j = 0; j < n; ++j) {
        std::swap(A[piv * n + j], A[col * n + j]);
        std::swap(inv[piv * n + j], inv[col * n + j]);
      }
    const double dd = A[col * n + col];
    for (int j = 0; j < n; ++j) {
      A[col * n + j] /= dd;
      inv[col * n + j] /= dd;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = A[r * n + col];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        A[r * n + j] -= f * A[col * n + j];
        inv[r * n + j] -= f * inv[col * n + j];
      }
    }
  }
  return inv;
}

int ipow(int b, int e) {
  int r = 1;
  while (e-- > 0) r *= b;
  return r;
}

struct Oracle {
  int d = 1, m = 0, n1 = 1, n = 2;
  int K[3] = {1, 1, 1};
  int bnd[3] = {0, 0, 0};  // 0 periodic, 1 reflective
  int Np[3] = {1, 1, 1}, Nd[3] = {1, 1, 1};
  double h = 1.0;
  double ap = -1.0, av = -1.0;
  int nthreads = 1;
  std::vector<double> M;
  int F = 1, E = 1;  // n1^d and n^d
  std::vector<double> p;            // [primary node][F]
  std::vector<double> v[3];         // [dual node][F]
  std::vector<double> cj[2][2];     // [grid][ap/av] per-node n^d jets (empty = constant)
  std::vector<double> fz[2];        // [grid] forcing levels z(r), [node][r = 0..n-2][n^d] (empty = none)
  // z-slab mode (d = 3, periodic z across ranks): z neighbours beyond the slab
  // come from halo layers set by the caller, [ix][iy][F]
  bool slab = false;
  std::vector<double> p_halo;       // primary layer z = Kz (next rank's layer 0)
  std::vector<double> v_halo[3];    // dual layer z = -1 (previous rank's layer Kz-1)
  double t_p = 0.0, t_v = 0.0, dt = 0.0;

  size_t nodes(int grid) const {
    const int* N = grid == 0 ? Np : Nd;
    return static_cast<size_t>(N[0]) * N[1] * N[2];
  }
  size_t node_index(int grid, const int* idx) const {
    const int* N = grid == 0 ? Np : Nd;
    return (static_cast<size_t>(idx[0]) * N[1] + idx[1]) * N[2] + idx[2];
  }
  void unravel(int grid, size_t node, int* idx) const {
    const int* N = grid == 0 ? Np : Nd;
    idx[2] = static_cast<int>(node % N[2]);
    node /= N[2];
    idx[1] = static_cast<int>(node % N[1]);
    idx[0] = static_cast<int>(node / N[1]);
  }

  // strides of an extent-n (or n1) x-major tensor of dimension d
  void strides(int ext, int* st) const {
    st[d - 1] = 1;
    for (int ax = d - 2; ax >= 0; --ax) st[ax] = st[ax + 1] * ext;
  }

  // --- jet arithmetic on n^d tensors (proj/src/jet.cpp:109-135) ---
  // out = d/dx_ax of t (scaled), truncated: out[i] = t[i+1] (i+1) / h
  void tensor_d(const double* t, int ax, double* out) const {
    int st[3];
    strides(n, st);
    for (int e = 0; e < E; ++e) {
      const int i = (e / st[ax]) % n;
      out[e] = i + 1 < n ? t[e + st[ax]] * (i + 1) / h : 0.0;
    }
  }
  // truncated tensor product, skipping zero entries of a (jet.cpp:109-121)
  void tensor_mul(const double* a, const double* b, double* out) const {
    int st[3];
    strides(n, st);
    for (int e = 0; e < E; ++e) out[e] = 0.0;
    for (int ea = 0; ea < E; ++ea) {
      const double c = a[ea];
      if (c == 0.0) continue;
      int ia[3] = {0, 0, 0};
      for (int ax = 0; ax < d; ++ax) ia[ax] = (ea / st[ax]) % n;
      for (int eb = 0; eb < E; ++eb) {
        bool ok = true;
        int eo = 0;
        for (int ax = 0; ax < d; ++ax) {
          const int k = (eb / st[ax]) % n;
          if (ia[ax] + k >= n) {
            ok = false;
            break;
          }
          eo += (ia[ax] + k) * st[ax];
        }
        if (ok) out[eo] += c * b[eb];
      }
    }
  }

  // --- reconstruction (proj/src/interpolation.cpp:53-113) ---
  // corners[c] (c's bit ax = high side along ax) hold n1^d jets; result is the
  // n^d extended jet at the cell center.  Stacked index along every axis is
  // side*(m+1) + l, exactly the reference's `stacked` vector, and M is applied
  // axis by axis starting with x, as reconstruct_cell_2d does.
  void reconstruct(const double* const* corners, double* ext) const {
    int sn[3], s1[3];
    strides(n, sn);
    strides(n1, s1);
    std::vector<double> a(E), b(E);
    for (int e = 0; e < E; ++e) {
      int corner = 0, src = 0;
      for (int ax = 0; ax < d; ++ax) {
        const int q = (e / sn[ax]) % n;
        const int side = q / n1, l = q % n1;
        corner |= side << ax;
        src += l * s1[ax];
      }
      a[e] = corners[corner][src];
    }
    for (int ax = 0; ax < d; ++ax) {
      for (int e = 0; e < E; ++e) {
        const int i = (e / sn[ax]) % n;
        if (i != 0) continue;
        // line through e along ax: out[r] = sum_s M[r][s] stacked[s]
        for (int r = 0; r < n; ++r) {
          const double* row = M.data() + static_cast<size_t>(r) * n;
          double acc = 0.0;
          for (int s = 0; s < n; ++s) acc += row[s] * a[e + s * sn[ax]];
          b[e + r * sn[ax]] = acc;
        }
      }
      a.swap(b);
    }
    std::memcpy(ext, a.data(), sizeof(double) * E);
  }

  // (m+1)^d corner of an n^d tensor -> F-entry jet update with leapfrog weights
  // target[s] += sum_{r odd < count} w_r table[r][s]   (stepper1d.cpp:54-61)
  void leapfrog(double* target, const std::vector<std::vector<double>>& table) const {
    int sn[3], s1[3];
    strides(n, sn);
    strides(n1, s1);
    const int count = static_cast<int>(table.size());
    for (int r = 1; r < count; r += 2) {
      double w = 2.0;
      for (int q = 1; q <= r; ++q) w *= dt / 2.0 / q;
      for (int f = 0; f < F; ++f) {
        int e = 0;
        for (int ax = 0; ax < d; ++ax) e += ((f / s1[ax]) % n1) * sn[ax];
        target[f] += w * table[r][e];
      }
    }
  }

  // ghost handling for the dual (velocity) family: returns the jet to use for
  // dual index idx (may be -1 or K along reflective axes) of component comp
  void dual_jet(int comp, const int* idx_in, double* out) const {
    if (slab && d == 3 && idx_in[2] < 0) {
      int ix = idx_in[0] % K[0], iy = idx_in[1] % K[1];
      ix = ix < 0 ? ix + K[0] : ix;
      iy = iy < 0 ? iy + K[1] : iy;
      const double* src = v_halo[comp].data() + (static_cast<size_t>(ix) * Nd[1] + iy) * F;
      std::memcpy(out, src, sizeof(double) * F);
      return;
    }
    int idx[3] = {idx_in[0], idx_in[1], idx_in[2]};
    int flip[3] = {0, 0, 0};
    double sigma = 1.0;
    for (int ax = 0; ax < d; ++ax) {
      if (bnd[ax] == 0) {
        int r = idx[ax] % K[ax];
        idx[ax] = r < 0 ? r + K[ax] : r;
      } else if (idx[ax] < 0 || idx[ax] >= K[ax]) {
        idx[ax] = idx[ax] < 0 ? 0 : K[ax] - 1;
        flip[ax] = 1;
        sigma *= comp == ax ? 1.0 : -1.0;
      }
    }
    const double* src = v[comp].data() + node_index(1, idx) * F;
    int s1[3];
    strides(n1, s1);
    for (int f = 0; f < F; ++f) {
      double s = sigma;
      for (int ax = 0; ax < d; ++ax)
        if (flip[ax] && ((f / s1[ax]) % n1) % 2 == 1) s = -s;
      out[f] = s * src[f];
    }
  }

  const double* forcing(int grid, size_t node) const {
    return fz[grid].empty() ? nullptr : fz[grid].data() + node * static_cast<size_t>(n - 1) * E;
  }

  const double* coeff(int grid, int which, size_t node) const {
    const auto& c = cj[grid][which];
    return c.empty() ? nullptr : c.data() + node * E;
  }

  // one CK iteration level, both tables (stepper1d.cpp:22-38 generalized):
  // P[r+1] = ap (.) sum_c d_c V_c[r];  V_c[r+1] = av (.) d_c P[r]
  // With a forcing table zt (the node's levels z(r), stepper1d.cpp:29-32)
  // z(r) is added to P[r+1] after the product, as the reference does.
  void ck(std::vector<std::vector<double>>& P, std::vector<std::vector<double>> (&V)[3],
          const double* apj, const double* avj, const double* zt = nullptr) const {
    std::vector<double> tmp(E), acc(E);
    for (int r = 0; r + 1 < n; ++r) {
      for (int e = 0; e < E; ++e) acc[e] = 0.0;
      for (int c = 0; c < d; ++c) {
        tensor_d(V[c][r].data(), c, tmp.data());
        for (int e = 0; e < E; ++e) acc[e] += tmp[e];
      }
      if (apj) {
        tensor_mul(apj, acc.data(), P[r + 1].data());
      } else {
        for (int e = 0; e < E; ++e) P[r + 1][e] = ap * acc[e];
      }
      if (zt)
        for (int e = 0; e < E; ++e) P[r + 1][e] += zt[static_cast<size_t>(r) * E + e];
      for (int c = 0; c < d; ++c) {
        tensor_d(P[r].data(), c, tmp.data());
        if (avj) {
          tensor_mul(avj, tmp.data(), V[c][r + 1].data());
        } else {
          for (int e = 0; e < E; ++e) V[c][r + 1][e] = av * tmp[e];
        }
      }
    }
  }

  void advance_p() {
    const size_t N = nodes(0);
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (long long node = 0; node < static_cast<long long>(N); ++node) {
      int idx[3];
      unravel(0, static_cast<size_t>(node), idx);
      const int nc = 1 << d;
      std::vector<std::vector<double>> cs(nc, std::vector<double>(F));
      std::vector<const double*> cp(nc);
      std::vector<std::vector<double>> P(n, std::vector<double>(E, 0.0));
      std::vector<std::vector<double>> V[3];
      for (int c = 0; c < d; ++c) {
        V[c].assign(n, std::vector<double>(E, 0.0));
        // p cell at primary node i spans dual neighbours i-1 (low), i (high)
        for (int corner = 0; corner < nc; ++corner) {
          int di[3] = {0, 0, 0};
          for (int ax = 0; ax < d; ++ax) di[ax] = idx[ax] - 1 + ((corner >> ax) & 1);
          dual_jet(c, di, cs[corner].data());
          cp[corner] = cs[corner].data();
        }
        reconstruct(cp.data(), V[c][0].data());
      }
      ck(P, V, coeff(0, 0, node), coeff(0, 1, node), forcing(0, node));
      leapfrog(p.data() + static_cast<size_t>(node) * F, P);
    }
    t_p += dt;
  }

  void advance_v() {
    const size_t N = nodes(1);
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
    for (long long node = 0; node < static_cast<long long>(N); ++node) {
      int idx[3];
      unravel(1, static_cast<size_t>(node), idx);
      const int nc = 1 << d;
      std::vector<const double*> cp(nc);
      for (int corner = 0; corner < nc; ++corner) {
        int pi[3] = {0, 0, 0};
        bool halo = false;
        for (int ax = 0; ax < d; ++ax) {
          int q = idx[ax] + ((corner >> ax) & 1);
          if (slab && ax == 2 && q == K[2]) halo = true;
          if (bnd[ax] == 0) q %= K[ax];
          pi[ax] = q;
        }
        cp[corner] = halo ? p_halo.data() + (static_cast<size_t>(pi[0]) * Np[1] + pi[1]) * F
                          : p.data() + node_index(0, pi) * F;
      }
      std::vector<std::vector<double>> P(n, std::vector<double>(E, 0.0));
      std::vector<std::vector<double>> V[3];
      for (int c = 0; c < d; ++c) V[c].assign(n, std::vector<double>(E, 0.0));
      reconstruct(cp.data(), P[0].data());
      ck(P, V, coeff(1, 0, node), coeff(1, 1, node), forcing(1, node));
      for (int c = 0; c < d; ++c) leapfrog(v[c].data() + static_cast<size_t>(node) * F, V[c]);
    }
    t_v += dt;
  }

  bool all_finite() const {
    for (double x : p)
      if (!std::isfinite(x)) return false;
    for (int c = 0; c < d; ++c)
      for (double x : v[c])
        if (!std::isfinite(x)) return false;
    return true;
  }
};

// scaled jet of amp * sin(w x + phase) at x0 (proj/src/jet.cpp:65-74)
void sin_jet(double amp, double w, double phase, double x0, double h, int n, double* out) {
  double base = amp;
  const double pi = std::acos(-1.0);
  for (int i = 0; i < n; ++i) {
    out[i] = base * std::sin(w * x0 + phase + i * pi / 2.0);
    base *= h * w / static_cast<double>(i + 1);
  }
}

}  // namespace

extern "C" {

void* orc_create(int d, int m, const int* K, const int* bnd, double h, double ap, double av,
                 int nthreads) {
  if (d < 1 || d > 3 || m < 0 || m > 8) return nullptr;
  Oracle* o = new Oracle;
  o->d = d;
  o->m = m;
  o->n1 = m + 1;
  o->n = 2 * m + 2;
  o->h = h;
  o->ap = ap;
  o->av = av;
  o->nthreads = nthreads > 0 ? nthreads : 1;
  for (int ax = 0; ax < 3; ++ax) {
    o->K[ax] = ax < d ? K[ax] : 1;
    o->bnd[ax] = ax < d ? bnd[ax] : 0;
    o->Nd[ax] = o->K[ax];
    o->Np[ax] = ax < d && o->bnd[ax] == 1 ? o->K[ax] + 1 : o->K[ax];
  }
  o->F = ipow(o->n1, d);
  o->E = ipow(o->n, d);
  o->M = build_M(m);
  o->p.assign(o->nodes(0) * o->F, 0.0);
  for (int c = 0; c < d; ++c) o->v[c].assign(o->nodes(1) * o->F, 0.0);
  return o;
}

void orc_destroy(void* h) { delete static_cast<Oracle*>(h); }

void orc_get_M(int m, double* out) {
  std::vector<double> M = build_M(m);
  std::memcpy(out, M.data(), sizeof(double) * M.size());
}

void orc_set_M(void* h, const double* M) {
  Oracle* o = static_cast<Oracle*>(h);
  std::memcpy(o->M.data(), M, sizeof(double) * o->M.size());
}

long long orc_num_nodes(void* h, int grid) { return static_cast<long long>(static_cast<Oracle*>(h)->nodes(grid)); }

void orc_set_field(void* h, int field, const double* src) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<double>& dst = field == 0 ? o->p : o->v[field - 1];
  std::memcpy(dst.data(), src, sizeof(double) * dst.size());
}

void orc_get_field(void* h, int field, double* out) {
  Oracle* o = static_cast<Oracle*>(h);
  const std::vector<double>& src = field == 0 ? o->p : o->v[field - 1];
  std::memcpy(out, src.data(), sizeof(double) * src.size());
}

// per-node n^d coefficient jets; which = 0 (ap) or 1 (av); null clears
void orc_set_coeff(void* h, int grid, int which, const double* jets) {
  Oracle* o = static_cast<Oracle*>(h);
  auto& c = o->cj[grid][which];
  if (!jets) {
    c.clear();
    return;
  }
  c.assign(jets, jets + o->nodes(grid) * o->E);
}

// forcing levels for the half steps updating `grid` (0 primary, 1 dual):
// [node][r = 0..2m][n^d]; null clears (hlf_set_forcing's table)
void orc_set_forcing(void* h, int grid, const double* table) {
  auto* o = static_cast<Oracle*>(h);
  if (!table) {
    o->fz[grid].clear();
    return;
  }
  o->fz[grid].assign(table, table + o->nodes(grid) * static_cast<size_t>(o->n - 1) * o->E);
}

void orc_set_times(void* h, double t_p, double t_v, double dt) {
  Oracle* o = static_cast<Oracle*>(h);
  o->t_p = t_p;
  o->t_v = t_v;
  o->dt = dt;
}

void orc_get_times(void* h, double* out) {
  Oracle* o = static_cast<Oracle*>(h);
  out[0] = o->t_p;
  out[1] = o->t_v;
  out[2] = o->dt;
}

void orc_advance_p(void* h) { static_cast<Oracle*>(h)->advance_p(); }
void orc_advance_v(void* h) { static_cast<Oracle*>(h)->advance_v(); }

// step_system (stepper1d.cpp:168-172): returns -1, or the step index at which
// the state became non-finite (InstabilityError::step)
int orc_advance_n(void* h, int nsteps, int first_step) {
  Oracle* o = static_cast<Oracle*>(h);
  for (int i = 0; i < nsteps; ++i) {
    o->advance_p();
    o->advance_v();
    if (!o->all_finite()) return first_step + i;
  }
  return -1;
}

// z-slab mode: halos replace the periodic z wrap (d = 3)
void orc_set_slab(void* h, int on) {
  Oracle* o = static_cast<Oracle*>(h);
  o->slab = on != 0;
  const size_t plane_p = static_cast<size_t>(o->Np[0]) * o->Np[1] * o->F;
  const size_t plane_d = static_cast<size_t>(o->Nd[0]) * o->Nd[1] * o->F;
  o->p_halo.assign(plane_p, 0.0);
  for (int c = 0; c < 3; ++c) o->v_halo[c].assign(plane_d, 0.0);
}

// copy z-layer z of a field out as [ix][iy][F]
void orc_get_layer(void* h, int field, int z, double* out) {
  Oracle* o = static_cast<Oracle*>(h);
  const int grid = field == 0 ? 0 : 1;
  const int* N = grid == 0 ? o->Np : o->Nd;
  const std::vector<double>& src = field == 0 ? o->p : o->v[field - 1];
  for (int ix = 0; ix < N[0]; ++ix)
    for (int iy = 0; iy < N[1]; ++iy) {
      const int idx[3] = {ix, iy, z};
      std::memcpy(out + (static_cast<size_t>(ix) * N[1] + iy) * o->F, src.data() + o->node_index(grid, idx) * o->F,
                  sizeof(double) * o->F);
    }
}

// kind 0: p halo (layer Kz); kind 1: v halo of component comp (layer -1)
void orc_set_halo(void* h, int kind, int comp, const double* in) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<double>& dst = kind == 0 ? o->p_halo : o->v_halo[comp];
  std::memcpy(dst.data(), in, sizeof(double) * dst.size());
}

// reconstruct one cell from 2^d corner jets (for direct reconstruction tests)
void orc_reconstruct(void* h, const double* corners, double* ext) {
  Oracle* o = static_cast<Oracle*>(h);
  const int nc = 1 << o->d;
  std::vector<const double*> cp(nc);
  for (int c = 0; c < nc; ++c) cp[c] = corners + static_cast<size_t>(c) * o->F;
  o->reconstruct(cp.data(), ext);
}

// Adds amp * prod_ax sin(w_ax x_ax + phase_ax) as scaled jets of `len` entries
// per axis at the nodes of a grid with N[ax] nodes starting at
// x0[ax] (+ offset * h): out[node][coef], node/coef x-major.  The exact data of
// every built-in wave problem is a short sum of such separable terms
// (proj/src/problems.cpp:140-160 and the 3D analogue).
void orc_add_separable(int d, const int* N, const double* x0, double h, double offset, int len,
                       double amp, const double* w, const double* phase, double* out) {
  const int Fl = ipow(len, d);
  std::vector<double> jets[3];
  long long total = 1;
  for (int ax = 0; ax < d; ++ax) total *= N[ax];
  int Nn[3] = {1, 1, 1};
  for (int ax = 0; ax < d; ++ax) Nn[ax] = N[ax];
  for (int ax = 0; ax < d; ++ax) {
    jets[ax].resize(static_cast<size_t>(Nn[ax]) * len);
    for (int i = 0; i < Nn[ax]; ++i)
      sin_jet(ax == 0 ? amp : 1.0, w[ax], phase[ax], x0[ax] + (i + offset) * h, h, len,
              jets[ax].data() + static_cast<size_t>(i) * len);
  }
  for (long long node = 0; node < total; ++node) {
    int idx[3] = {0, 0, 0};
    long long r = node;
    for (int ax = d - 1; ax >= 0; --ax) {
      idx[ax] = static_cast<int>(r % Nn[ax]);
      r /= Nn[ax];
    }
    for (int f = 0; f < Fl; ++f) {
      int rem = f;
      double val = 1.0;
      for (int ax = d - 1; ax >= 0; --ax) {
        const int a = rem % len;
        rem /= len;
        val *= jets[ax][static_cast<size_t>(idx[ax]) * len + a];
      }
      out[static_cast<size_t>(node) * Fl + f] += val;
    }
  }
}

}  // extern "C"
