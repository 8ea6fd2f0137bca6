// The 2D drop-in hlf::b200::Stepper2d (include/hlf/b200/stepper2d.hpp) driven
// through the reference's own 2D types and analysis code: Problem2d /
// Grid2d / TensorJet / PiecewiseTensor, reconstruct_cell_2d, l2_error_2d and
// convergence_rate (linked from oracle/_ref/libhlf_ref.a).  The checks are the
// stepper2d module's examples and invariants and the 2D acceptance criteria
// of the reference's specification:
//   * dimensional reduction: a y-independent 2D problem evolves every x row
//     exactly like the reference's own Stepper1d (1e-12);
//   * the paper's 2D rates at CFL 0.9, m = 0..3, within +-0.4;
//   * reflective walls: p = 0 on every wall at the Gauss points after every
//     step (1e-10), and the Gaussian pulse stays bounded for 1000 steps;
//   * Maxwell TM cavity, m = 4, CFL 0.8, a 3-point sweep: >= 4 orders;
//   * zero data stays zero, instability carries the step index, bad m is a
//     ConfigError.
// Built by oracle/Makefile (`make -C oracle dropin`), run on the GPU by
// tests/test_cpp_dropin.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "hlf/analysis.hpp"
#include "hlf/b200/stepper2d.hpp"
#include "hlf/config.hpp"
#include "hlf/problem.hpp"
#include "hlf/stepper1d.hpp"

using namespace hlf;
using hlf::b200::State2d;
using hlf::b200::Stepper2d;

namespace {
const double pi = std::acos(-1.0);

double dt_for(const Grid2d& g, int m, double cfl, double T, int* nsteps) {
  SchemeConfig cfg;
  cfg.m = m;
  cfg.cfl = cfl;
  *nsteps = step_count(T, cfg.dt_nominal_2d(g.h, 1.0));
  return T / *nsteps;
}

double p_l2(const Stepper2d& s, const State2d& st) {
  const Problem2d& prob = s.problem();
  const double t = st.t_p;
  return l2_error_2d(s.cells(st), [&](double x, double y) { return prob.exact_value(0, x, y, t); });
}

double max_abs_p(const State2d& st) {
  double mx = 0.0;
  for (const TensorJet& j : st.p)
    for (double a : j.a) mx = std::max(mx, std::fabs(a));
  return mx;
}
}  // namespace

TEST_CASE("zero data stays zero") {
  Problem2d prob = acoustics_mode_problem(Boundary::periodic);
  prob.exact = [](int, double, double, double, double, int n) { return TensorJet(n, n); };
  Grid2d g = Grid2d::over(-1.0, 1.0, -1.0, 1.0, 12);
  Stepper2d s(prob, g, 3);
  State2d st = s.init_leapfrog(0.05);
  s.advance_n(st, 10, 0);
  CHECK(max_abs_p(st) == 0.0);
  for (const TensorJet& j : st.v)
    for (double a : j.a) CHECK(a == 0.0);
}

TEST_CASE("a y-independent problem is the reference's 1D stepper (dimensional reduction)") {
  // tensor consistency to 1e-12 against the compiled reference
  for (int m : {1, 2, 3}) {
    const int K = 20;
    Problem1d p1 = standing_wave_problem();
    Problem2d p2;
    p2.name = "y-independent standing wave";
    p2.boundary = Boundary::periodic;
    p2.x_min = p1.x_min;
    p2.x_max = p1.x_max;
    p2.y_min = -1.0;
    p2.y_max = p2.y_min + (p1.x_max - p1.x_min);
    p2.exact = [p1](int f, double x, double, double t, double h, int n) {
      Jet one(n, 0.0);
      one[0] = 1.0;
      if (f == 2) return TensorJet(n, n);  // no y velocity
      return tensor_outer(p1.exact(f, x, t, h, n), one);
    };
    Grid1d g1 = Grid1d::over(p1.x_min, p1.x_max, K);
    Grid2d g2 = Grid2d::over(p2.x_min, p2.x_max, p2.y_min, p2.y_max, K);
    const double dt = 0.9 * g1.h / 2.0;
    Stepper1d ref(p1, g1, m);
    State1d r = ref.init_leapfrog(dt);
    Stepper2d dev(p2, g2, m);
    State2d st = dev.init_leapfrog(dt);
    for (int i = 0; i < 25; ++i) ref.step_system(r, i);
    dev.advance_n(st, 25, 0);
    CHECK(st.t_p == r.t_p);
    double scale = 0.0, err = 0.0;
    for (int ix = 0; ix < K; ++ix)
      for (int iy = 0; iy < K; ++iy)
        for (int a = 0; a <= m; ++a)
          for (int b = 0; b <= m; ++b) {
            const double want_p = b == 0 ? r.p[ix][a] : 0.0;
            const double want_v = b == 0 ? r.v[ix][a] : 0.0;
            scale = std::max({scale, std::fabs(want_p), std::fabs(want_v)});
            err = std::max(err, std::fabs(st.p[static_cast<size_t>(ix) * K + iy].at(a, b) - want_p));
            err = std::max(err, std::fabs(st.v[static_cast<size_t>(ix) * K + iy].at(a, b) - want_v));
            err = std::max(err, std::fabs(st.u[static_cast<size_t>(ix) * K + iy].at(a, b)));
          }
    CAPTURE(m);
    CHECK(err <= 1e-12 * scale);
  }
}

TEST_CASE("2D acoustics rates match the paper at CFL 0.9 (m = 0..3)") {
  // PAPER.md:1098 (Hermite-leapfrog, C_CFL = 0.9): 1.86, 1.88, 6.01, 6.74;
  // SPEC.md:516 acceptance band +-0.4.  L2 of p on the dual cells by the
  // reference's l2_error_2d, slope by its convergence_rate.  The paper does
  // not state the 2D final time; T = 4.13 is the final time of its 1D
  // convergence study (Table 1, test_stepper1d.cpp:323-330), and K = 10..80
  // keeps m = 3 above the roundoff floor (at K = 160 its error is ~1e-13).
  const double paper[4] = {1.86, 1.88, 6.01, 6.74};
  const double T = 4.13;
  const std::vector<int> Ks = {10, 20, 40, 80};
  Problem2d prob = acoustics_mode_problem(Boundary::periodic);
  for (int m = 0; m <= 3; ++m) {
    std::vector<double> hs, es;
    for (int K : Ks) {
      Grid2d g = Grid2d::over(-1.0, 1.0, -1.0, 1.0, K);
      int n = 0;
      const double dt = dt_for(g, m, 0.9, T, &n);
      Stepper2d s(prob, g, m);
      State2d st = s.init_leapfrog(dt);
      CHECK(s.advance_to(st, T) == n);
      hs.push_back(g.h);
      es.push_back(p_l2(s, st));
    }
    const RateFit fit = convergence_rate(hs, es);
    CAPTURE(m);
    CAPTURE(fit.rate);
    MESSAGE("m=" << m << " rate " << fit.rate << " (paper " << paper[m] << ")");
    CHECK(fit.points_used >= 3);
    CHECK(std::fabs(fit.rate - paper[m]) <= 0.4);
  }
}

TEST_CASE("reflective walls: p vanishes on every wall at the Gauss points after every step") {
  // SPEC.md:331 (Eq. 80 conditions at quadrature points, 1e-10): the
  // reconstructed p on the wall edges of the boundary cells
  Problem2d prob = gaussian_pulse_problem();
  for (int m : {1, 2, 3}) {
    const int K = 24;
    Grid2d g = Grid2d::over(prob.x_min, prob.x_max, prob.y_min, prob.y_max, K);
    Stepper2d s(prob, g, m);
    State2d st = s.init_leapfrog(0.5 * g.h / std::sqrt(2.0));
    double worst = 0.0;
    const int nq = 2 * m + 2;
    for (int step = 0; step < 30; ++step) {
      s.step_system(st, step);
      const PiecewiseTensor pw = s.cells(st);
      const double scale = std::max(max_abs_p(st), 1e-300);
      for (int k = 0; k < K; ++k)
        for (int q = 0; q < nq; ++q) {
          const double t = -0.5 + (q + 0.5) / nq;  // points along the wall edge
          // x walls (xi = -1/2 at ix = 0, +1/2 at ix = K-1), y walls likewise
          worst = std::max(worst, std::fabs(tensor_eval(pw.cell(0, k), -0.5, t)) / scale);
          worst = std::max(worst, std::fabs(tensor_eval(pw.cell(K - 1, k), 0.5, t)) / scale);
          worst = std::max(worst, std::fabs(tensor_eval(pw.cell(k, 0), t, -0.5)) / scale);
          worst = std::max(worst, std::fabs(tensor_eval(pw.cell(k, K - 1), t, 0.5)) / scale);
        }
    }
    CAPTURE(m);
    CHECK(worst <= 1e-10);
  }
}

TEST_CASE("the Gaussian pulse with reflective walls stays bounded for 1000 steps") {
  // SPEC.md stepper2d example (Fig. 6 setup, qualitative): stable, bounded
  Problem2d prob = gaussian_pulse_problem();
  const int K = 64, m = 3;
  Grid2d g = Grid2d::over(prob.x_min, prob.x_max, prob.y_min, prob.y_max, K);
  Stepper2d s(prob, g, m);
  SchemeConfig cfg;
  cfg.m = m;
  State2d st = s.init_leapfrog(cfg.dt_nominal_2d(g.h, 1.0));
  const double p0 = max_abs_p(st);
  s.advance_n(st, 1000, 0);
  CHECK(std::isfinite(max_abs_p(st)));
  CHECK(max_abs_p(st) <= 2.0 * p0);
}

TEST_CASE("Maxwell TM cavity: m = 4, CFL 0.8, 3-point sweep, >= 4 orders of decay") {
  // SPEC.md:520 (Fig. 8 trend): omega_x = omega_y = 8 pi, PEC walls
  Problem2d prob = maxwell_cavity_problem();
  const int m = 4;
  const double T = 0.25;
  std::vector<double> es;
  for (int K : {16, 32, 64}) {
    Grid2d g = Grid2d::over(prob.x_min, prob.x_max, prob.y_min, prob.y_max, K);
    int n = 0;
    const double dt = dt_for(g, m, 0.8, T, &n);
    Stepper2d s(prob, g, m);
    State2d st = s.init_leapfrog(dt);
    CHECK(s.advance_to(st, T) == n);
    es.push_back(p_l2(s, st));
    MESSAGE("Maxwell K=" << K << " L2(Ez) " << es.back());
  }
  CHECK(es[1] < es[0]);
  CHECK(es[2] < es[1]);
  CHECK(es[0] / es[2] >= 1e4);
}

TEST_CASE("instability carries the step index; bad orders are configuration errors") {
  Problem2d prob = acoustics_mode_problem(Boundary::periodic);
  Grid2d g = Grid2d::over(-1.0, 1.0, -1.0, 1.0, 12);
  Stepper2d s(prob, g, 2);
  State2d st = s.init_leapfrog(3.0 * g.h);
  bool blew = false;
  for (int i = 0; i < 3000 && !blew; ++i) {
    try {
      s.step_system(st, i);
    } catch (const InstabilityError& e) {
      blew = true;
      CHECK(e.step == i);
      CHECK(std::string(e.what()).find(std::to_string(i)) != std::string::npos);
    }
  }
  CHECK(blew);
  CHECK_THROWS_AS(Stepper2d(prob, g, 9), ConfigError);
  State2d ok = s.init_leapfrog(0.2 * g.h);
  CHECK_NOTHROW(s.advance_n(ok, 10, 0));
}
