// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// C-ABI shim over the COMPILED REFERENCE (sources under /root/reference/proj,
// built unchanged by oracle/Makefile into oracle/_ref/).  It lets the Python
// tests and bench.py's reference arm drive the reference's own Stepper1d,
// build_interp_operator, reconstruct_cell_2d, analysis accessors and problem
// providers.  Nothing in the product links this file.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hlf/analysis.hpp"
#include "hlf/config.hpp"
#include "hlf/grid.hpp"
#include "hlf/interpolation.hpp"
#include "hlf/jet.hpp"
#include "hlf/problem.hpp"
#include "hlf/stepper1d.hpp"

using namespace hlf;

namespace {

// tests/test_stepper1d.cpp:17-27
Problem1d zero_problem() {
  Problem1d p;
  p.name = "zero";
  p.x_min = -1.0;
  p.x_max = 1.0;
  p.c_max = 1.0;
  p.ap = [](double, double, int n) { return constant_jet(-1.0, n); };
  p.av = [](double, double, int n) { return constant_jet(-1.0, n); };
  p.exact = [](int, double, double, double, int n) { return Jet(n, 0.0); };
  return p;
}

bool make_problem(const char* name, unsigned seed, Problem1d& out) {
  const std::string s(name);
  if (s == "standing-wave") out = standing_wave_problem();
  else if (s == "variable-speed") out = variable_speed_problem();
  else if (s == "pv") out = pv_problem();
  else if (s == "random-wave") out = random_wave_problem(seed);
  else if (s == "zero") out = zero_problem();
  else return false;
  return true;
}

struct Ref1d {
  std::unique_ptr<Stepper1d> stepper;
  State1d st;
  ModifiedState1d mst;  // step_modified state (stepper1d.cpp:174-232)
  DualState1d dst;      // step_dual_hermite state (stepper1d.cpp:235-272)
};

}  // namespace

extern "C" {

int ref_build_interp(int m, double* M_out, double* cond_out) {
  try {
    InterpOperator op = build_interp_operator(m);
    std::memcpy(M_out, op.M.data(), sizeof(double) * op.M.size());
    if (cond_out) *cond_out = op.condition;
    return 0;
  } catch (const ConfigError&) {
    return 1;
  }
}

// reconstruct_cell_2d (proj/src/interpolation.cpp:77-113); corners (m+1)^2 each
void ref_reconstruct_2d(int m, const double* c00, const double* c10, const double* c01,
                        const double* c11, double* out) {
  InterpOperator op = build_interp_operator(m);
  auto tj = [m](const double* a) {
    TensorJet t(m + 1, m + 1);
    std::memcpy(t.a.data(), a, sizeof(double) * t.a.size());
    return t;
  };
  TensorJet r = reconstruct_cell_2d(op, tj(c00), tj(c10), tj(c01), tj(c11));
  std::memcpy(out, r.a.data(), sizeof(double) * r.a.size());
}

void ref_reconstruct_1d(int m, const double* left, const double* right, double* out) {
  InterpOperator op = build_interp_operator(m);
  Jet l(left, left + m + 1), r(right, right + m + 1);
  Jet e = reconstruct_cell_1d(op, l, r);
  std::memcpy(out, e.data(), sizeof(double) * e.size());
}

void* ref1d_create(const char* problem, unsigned seed, int m, int K) {
  Problem1d prob;
  if (!make_problem(problem, seed, prob)) return nullptr;
  try {
    Grid1d g = Grid1d::over(prob.x_min, prob.x_max, K);
    Ref1d* r = new Ref1d;
    r->stepper = std::make_unique<Stepper1d>(prob, g, m);
    return r;
  } catch (...) {
    return nullptr;
  }
}

void ref1d_destroy(void* h) { delete static_cast<Ref1d*>(h); }

// x_min, x_max, c_max, h
void ref1d_info(void* h, double* out) {
  const Stepper1d& s = *static_cast<Ref1d*>(h)->stepper;
  out[0] = s.problem().x_min;
  out[1] = s.problem().x_max;
  out[2] = s.problem().c_max;
  out[3] = s.grid().h;
}

void ref1d_init(void* h, double dt, double t0) {
  Ref1d* r = static_cast<Ref1d*>(h);
  r->st = r->stepper->init_leapfrog(dt, t0);
}

// p, v: [K][m+1]; times: t_p, t_v, dt
void ref1d_get(void* h, double* p, double* v, double* times) {
  Ref1d* r = static_cast<Ref1d*>(h);
  const int n1 = r->stepper->m() + 1;
  for (size_t j = 0; j < r->st.p.size(); ++j) {
    if (p) std::memcpy(p + j * n1, r->st.p[j].data(), sizeof(double) * n1);
    if (v) std::memcpy(v + j * n1, r->st.v[j].data(), sizeof(double) * n1);
  }
  if (times) {
    times[0] = r->st.t_p;
    times[1] = r->st.t_v;
    times[2] = r->st.dt;
  }
}

void ref1d_set(void* h, const double* p, const double* v, const double* times) {
  Ref1d* r = static_cast<Ref1d*>(h);
  const int n1 = r->stepper->m() + 1;
  const int K = r->stepper->grid().K;
  r->st.p.assign(K, Jet(n1, 0.0));
  r->st.v.assign(K, Jet(n1, 0.0));
  for (int j = 0; j < K; ++j) {
    std::memcpy(r->st.p[j].data(), p + static_cast<size_t>(j) * n1, sizeof(double) * n1);
    std::memcpy(r->st.v[j].data(), v + static_cast<size_t>(j) * n1, sizeof(double) * n1);
  }
  r->st.t_p = times[0];
  r->st.t_v = times[1];
  r->st.dt = times[2];
}

void ref1d_set_dt(void* h, double dt) { static_cast<Ref1d*>(h)->st.dt = dt; }
void ref1d_advance_p(void* h) { static_cast<Ref1d*>(h)->stepper->advance_p(static_cast<Ref1d*>(h)->st); }
void ref1d_advance_v(void* h) { static_cast<Ref1d*>(h)->stepper->advance_v(static_cast<Ref1d*>(h)->st); }

// loops step_system like tests/test_stepper1d.cpp:38; returns -1 or the
// InstabilityError step
int ref1d_steps(void* h, int n, int first) {
  Ref1d* r = static_cast<Ref1d*>(h);
  try {
    for (int i = 0; i < n; ++i) r->stepper->step_system(r->st, first + i);
  } catch (const InstabilityError& e) {
    return e.step;
  }
  return -1;
}

// tests/test_stepper1d.cpp:39-40
double ref1d_l2_p(void* h) {
  Ref1d* r = static_cast<Ref1d*>(h);
  const Stepper1d& s = *r->stepper;
  const double t = r->st.t_p;
  return l2_error_1d(r->st.p, s.grid(), s.op(), true,
                     [&](double x) { return s.problem().exact_value(0, x, t); });
}

double ref1d_l2_v(void* h) {
  Ref1d* r = static_cast<Ref1d*>(h);
  const Stepper1d& s = *r->stepper;
  const double t = r->st.t_v;
  return l2_error_1d(r->st.v, s.grid(), s.op(), false,
                     [&](double x) { return s.problem().exact_value(1, x, t); });
}

double ref1d_conserved_q(void* h, double c) {
  Ref1d* r = static_cast<Ref1d*>(h);
  return conserved_q(r->st.p, r->st.v, r->stepper->grid(), r->stepper->op(), c, r->st.dt);
}

double ref1d_conserved_r(void* h, double c) {
  Ref1d* r = static_cast<Ref1d*>(h);
  return conserved_r(r->st.v, r->st.p, r->stepper->grid(), r->stepper->op(), c, r->st.dt);
}

// coefficient jets the stepper evaluates at construction (stepper1d.cpp:103-110):
// which 0 = ap, 1 = av; on_dual selects the grid; out [K][2m+2]
void ref1d_coeff(void* h, int which, int on_dual, double* out) {
  const Stepper1d& s = *static_cast<Ref1d*>(h)->stepper;
  const int n = 2 * s.m() + 2;
  for (int j = 0; j < s.grid().K; ++j) {
    const double x = on_dual ? s.grid().dual(j) : s.grid().primary(j);
    Jet c = which == 0 ? s.problem().ap(x, s.grid().h, n) : s.problem().av(x, s.grid().h, n);
    std::memcpy(out + static_cast<size_t>(j) * n, c.data(), sizeof(double) * n);
  }
}

// the forcing levels forcing_at(x, t)(r), r = 0..2m (stepper1d.cpp:113-119),
// at every node of one grid: out [K][2m+1][2m+2] (zero without a forcing)
void ref1d_forcing(void* h, int on_dual, double t, double* out) {
  const Stepper1d& s = *static_cast<Ref1d*>(h)->stepper;
  const int n = 2 * s.m() + 2;
  const auto& fz = s.problem().forcing;
  for (int j = 0; j < s.grid().K; ++j) {
    const double x = on_dual ? s.grid().dual(j) : s.grid().primary(j);
    for (int r = 0; r + 1 < n; ++r) {
      double* o = out + (static_cast<size_t>(j) * (n - 1) + r) * n;
      if (!fz) {
        std::memset(o, 0, sizeof(double) * n);
        continue;
      }
      Jet z = fz(r, x, t, s.grid().h, n);
      for (int i = 0; i < n; ++i) o[i] = i < static_cast<int>(z.size()) ? z[i] : 0.0;
    }
  }
}

int ref1d_has_forcing(void* h) { return static_cast<bool>(static_cast<Ref1d*>(h)->stepper->problem().forcing); }

// Problem2d exact jets at one point (proj/src/problems.cpp:140-199):
// name = acoustics-periodic | acoustics-reflective | gaussian-pulse | maxwell-tm
int ref2d_exact(const char* name, int f, double x, double y, double t, double h, int n,
                double* out) {
  const std::string s(name);
  Problem2d p;
  if (s == "acoustics-periodic") p = acoustics_mode_problem(Boundary::periodic);
  else if (s == "acoustics-reflective") p = acoustics_mode_problem(Boundary::reflective);
  else if (s == "gaussian-pulse") p = gaussian_pulse_problem();
  else if (s == "maxwell-tm") p = maxwell_cavity_problem();
  else return 1;
  TensorJet tj = p.exact(f, x, y, t, h, n);
  std::memcpy(out, tj.a.data(), sizeof(double) * tj.a.size());
  return 0;
}

// l2_error_2d over a PiecewiseTensor (analysis.cpp:259-285): cells given as
// n^2 jets row-major ix*ny+iy with centers/bounds; exact = acoustics mode
// (periodic, field f, time t)
double ref2d_l2_acoustics(int nx, int ny, double h, const double* cx, const double* cy,
                          const double* lo_x, const double* hi_x, const double* lo_y,
                          const double* hi_y, int n, const double* ext, int f, double t) {
  PiecewiseTensor pt;
  pt.nx = nx;
  pt.ny = ny;
  pt.h = h;
  pt.cx.assign(cx, cx + nx);
  pt.cy.assign(cy, cy + ny);
  pt.lo_x.assign(lo_x, lo_x + nx);
  pt.hi_x.assign(hi_x, hi_x + nx);
  pt.lo_y.assign(lo_y, lo_y + ny);
  pt.hi_y.assign(hi_y, hi_y + ny);
  pt.ext.resize(static_cast<size_t>(nx) * ny);
  for (size_t c = 0; c < pt.ext.size(); ++c) {
    pt.ext[c] = TensorJet(n, n);
    std::memcpy(pt.ext[c].a.data(), ext + c * n * n, sizeof(double) * n * n);
  }
  Problem2d p = acoustics_mode_problem(Boundary::periodic);
  return l2_error_2d(pt, [&](double x, double y) { return p.exact_value(f, x, y, t); });
}

double ref_convergence_rate(int count, const double* hs, const double* es) {
  std::vector<double> h(hs, hs + count), e(es, es + count);
  try {
    return convergence_rate(h, e).rate;
  } catch (...) {
    return NAN;
  }
}

double ref_dt_nominal(int dim, double cfl, double h, double c_max) {
  SchemeConfig cfg;
  cfg.cfl = cfl;
  return dim == 1 ? cfg.dt_nominal_1d(h, c_max) : cfg.dt_nominal_2d(h, c_max);
}

int ref_step_count(double T, double dt) { return step_count(T, dt); }

// ---- the reference's alternative time schemes: jets flat [node][coef]
void ref1d_init_modified(void* h, double dt, double t0) {
  Ref1d* r = static_cast<Ref1d*>(h);
  r->mst = r->stepper->init_modified(dt, t0);
}
// fields in the order p primary, v primary, p dual, v dual; tdt = {t, dt}
void ref1d_get_modified(void* h, double* pp, double* vp, double* pd, double* vd, double* tdt) {
  const ModifiedState1d& st = static_cast<Ref1d*>(h)->mst;
  double* outs[4] = {pp, vp, pd, vd};
  const std::vector<Jet>* ins[4] = {&st.prim[0], &st.prim[1], &st.dual[0], &st.dual[1]};
  for (int f = 0; f < 4; ++f) {
    size_t k = 0;
    for (const Jet& j : *ins[f])
      for (double x : j) outs[f][k++] = x;
  }
  tdt[0] = st.t;
  tdt[1] = st.dt;
}
int ref1d_steps_modified(void* h, int n, int first) {
  Ref1d* r = static_cast<Ref1d*>(h);
  try {
    for (int i = 0; i < n; ++i) r->stepper->step_modified(r->mst, first + i);
  } catch (const InstabilityError& e) {
    return e.step;
  }
  return -1;
}
void ref1d_init_dual(void* h, double dt, double t0) {
  Ref1d* r = static_cast<Ref1d*>(h);
  r->dst = r->stepper->init_dual_hermite(dt, t0);
}
void ref1d_get_dual(void* h, double* p, double* v, double* tdt) {
  const DualState1d& st = static_cast<Ref1d*>(h)->dst;
  size_t k = 0;
  for (const Jet& j : st.p)
    for (double x : j) p[k++] = x;
  k = 0;
  for (const Jet& j : st.v)
    for (double x : j) v[k++] = x;
  tdt[0] = st.t;
  tdt[1] = st.dt;
}
int ref1d_steps_dual(void* h, int n, int first) {
  Ref1d* r = static_cast<Ref1d*>(h);
  try {
    for (int i = 0; i < n; ++i) r->stepper->step_dual_hermite(r->dst, first + i);
  } catch (const InstabilityError& e) {
    return e.step;
  }
  return -1;
}

}  // extern "C"
