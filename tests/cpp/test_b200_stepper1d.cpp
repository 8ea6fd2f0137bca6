// The reference's Stepper1d test cases (proj/tests/test_stepper1d.cpp:208-417)
// re-targeted at the drop-in hlf::b200::Stepper1d: only the stepper type
// changes; problems, grids, states, analysis accessors and error types are
// the reference's own (linked from oracle/_ref/libhlf_ref.a).  Built by
// oracle/Makefile (`make -C oracle dropin`), run by tests/test_cpp_dropin.py
// on the GPU.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <vector>

#include "hlf/analysis.hpp"
#include "hlf/b200/stepper1d.hpp"
#include "hlf/config.hpp"
#include "hlf/problem.hpp"
#include "hlf/stepper1d.hpp"

using namespace hlf;
using DeviceStepper1d = hlf::b200::Stepper1d;

namespace {
const double pi = std::acos(-1.0);

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

// variable speed without forcing: ap = -c^2(x), c^2 = 1 + sin(x)/2 (problems.cpp:45-49)
Problem1d variable_unforced_problem() {
  Problem1d p = variable_speed_problem();
  p.forcing = nullptr;
  return p;
}

// tests/test_stepper1d.cpp:29-41 with the device stepper
double leapfrog_l2(const Problem1d& prob, int m, double cfl, int K, double T) {
  Grid1d g = Grid1d::over(prob.x_min, prob.x_max, K);
  SchemeConfig cfg;
  cfg.m = m;
  cfg.cfl = cfl;
  const int nsteps = step_count(T, cfg.dt_nominal_1d(g.h, prob.c_max));
  const double dt = T / nsteps;
  DeviceStepper1d stepper(prob, g, m);
  State1d st = stepper.init_leapfrog(dt);
  for (int i = 0; i < nsteps; ++i) stepper.step_system(st, i);
  return l2_error_1d(st.p, g, stepper.op(), true,
                     [&](double x) { return prob.exact_value(0, x, st.t_p); });
}

double max_rel(const std::vector<Jet>& a, const std::vector<Jet>& b) {
  double d = 0.0, s = 0.0;
  for (size_t j = 0; j < a.size(); ++j)
    for (size_t i = 0; i < a[j].size(); ++i) {
      d = std::max(d, std::abs(a[j][i] - b[j][i]));
      s = std::max(s, std::abs(b[j][i]));
    }
  return s > 0 ? d / s : d;
}
}  // namespace

TEST_CASE("zero data stays zero") {
  Problem1d prob = zero_problem();
  Grid1d g = Grid1d::over(-1.0, 1.0, 8);
  DeviceStepper1d stepper(prob, g, 2);
  State1d lf = stepper.init_leapfrog(0.05);
  for (int i = 0; i < 10; ++i) stepper.step_system(lf, i);
  for (int j = 0; j < g.K; ++j) {
    for (double x : lf.p[j]) CHECK(x == 0.0);
    for (double x : lf.v[j]) CHECK(x == 0.0);
  }
}

TEST_CASE("stepping is linear in the state") {
  Problem1d prob = standing_wave_problem();
  Grid1d g = Grid1d::over(-1.0, 1.0, 8);
  const int m = 2;
  DeviceStepper1d stepper(prob, g, m);
  const double dt = 0.08;
  auto fill = [&](State1d& st, double mix) {
    for (int j = 0; j < g.K; ++j)
      for (int s = 0; s <= m; ++s) {
        st.p[j][s] = std::sin(1.7 * j + mix + 0.3 * s);
        st.v[j][s] = std::cos(0.9 * j - 2.0 * mix + 0.7 * s);
      }
  };
  State1d a = stepper.init_leapfrog(dt), b = stepper.init_leapfrog(dt), ab = stepper.init_leapfrog(dt);
  fill(a, 0.4);
  fill(b, 1.9);
  const double al = 0.6, be = -1.3;
  for (int j = 0; j < g.K; ++j)
    for (int s = 0; s <= m; ++s) {
      ab.p[j][s] = al * a.p[j][s] + be * b.p[j][s];
      ab.v[j][s] = al * a.v[j][s] + be * b.v[j][s];
    }
  stepper.step_system(a, 0);
  stepper.step_system(b, 0);
  stepper.step_system(ab, 0);
  for (int j = 0; j < g.K; ++j)
    for (int s = 0; s <= m; ++s) {
      CHECK(ab.p[j][s] == doctest::Approx(al * a.p[j][s] + be * b.p[j][s]).epsilon(1e-12));
      CHECK(ab.v[j][s] == doctest::Approx(al * a.v[j][s] + be * b.v[j][s]).epsilon(1e-12));
    }
}

TEST_CASE("leapfrog steps reverse exactly") {
  Problem1d prob = standing_wave_problem();
  Grid1d g = Grid1d::over(-1.0, 1.0, 10);
  const int m = 2;
  DeviceStepper1d stepper(prob, g, m);
  const double dt = 0.07;
  State1d st = stepper.init_leapfrog(dt);
  State1d ref = st;
  const int nsteps = 20;
  for (int i = 0; i < nsteps; ++i) stepper.step_system(st, i);
  st.dt = -dt;
  for (int i = 0; i < nsteps; ++i) {
    stepper.advance_v(st);
    stepper.advance_p(st);
  }
  for (int j = 0; j < g.K; ++j)
    for (int s = 0; s <= m; ++s) {
      CHECK(st.p[j][s] == doctest::Approx(ref.p[j][s]).epsilon(1e-11));
      CHECK(st.v[j][s] == doctest::Approx(ref.v[j][s]).epsilon(1e-11));
    }
  CHECK(st.t_p == doctest::Approx(0.0).epsilon(1e-12));
}

TEST_CASE("running past the stability limit raises an instability error") {
  Problem1d prob = standing_wave_problem();
  Grid1d g = Grid1d::over(-1.0, 1.0, 16);
  DeviceStepper1d stepper(prob, g, 2);
  SchemeConfig cfg;
  cfg.m = 2;
  cfg.cfl = 2.5;
  State1d st = stepper.init_leapfrog(cfg.dt_nominal_1d(g.h, prob.c_max));
  // the reference's own stepper on the same data fixes the expected step
  Stepper1d refstep(prob, g, 2);
  State1d rst = refstep.init_leapfrog(cfg.dt_nominal_1d(g.h, prob.c_max));
  int expected = -1;
  for (int i = 0; i < 5000 && expected < 0; ++i) {
    try {
      refstep.step_system(rst, i);
    } catch (const InstabilityError& e) {
      expected = e.step;
    }
  }
  REQUIRE(expected > 0);
  bool blew_up = false;
  for (int i = 0; i < 5000 && !blew_up; ++i) {
    try {
      stepper.step_system(st, i);
    } catch (const InstabilityError& e) {
      blew_up = true;
      CHECK(e.step == i);
      CHECK(e.step == expected);
      CHECK(std::string(e.what()).find(std::to_string(i)) != std::string::npos);
    }
  }
  CHECK(blew_up);
}

TEST_CASE("after an instability a re-initialised state steps cleanly") {
  // check_finite (stepper1d.cpp:121-129) looks at the current state only:
  // the same stepper object must not report a stale step afterwards
  Problem1d prob = standing_wave_problem();
  Grid1d g = Grid1d::over(-1.0, 1.0, 16);
  DeviceStepper1d stepper(prob, g, 2);
  SchemeConfig cfg;
  cfg.m = 2;
  cfg.cfl = 2.5;
  State1d st = stepper.init_leapfrog(cfg.dt_nominal_1d(g.h, prob.c_max));
  CHECK_THROWS_AS(stepper.advance_n(st, 5000, 0), InstabilityError);
  cfg.cfl = 0.5;
  State1d ok = stepper.init_leapfrog(cfg.dt_nominal_1d(g.h, prob.c_max));
  CHECK_NOTHROW(stepper.advance_n(ok, 20, 0));
  CHECK_NOTHROW(stepper.step_system(ok, 20));
  for (const Jet& j : ok.p) CHECK(std::isfinite(j[0]));
}

TEST_CASE("advance_to is the caller loop of leapfrog_l2") {
  // tests/test_stepper1d.cpp:29-41 with the loop replaced by advance_to
  Problem1d prob = standing_wave_problem();
  for (int K : {10, 20, 40}) {
    Grid1d g = Grid1d::over(prob.x_min, prob.x_max, K);
    SchemeConfig cfg;
    cfg.m = 2;
    cfg.cfl = 0.9;
    const double T = 4.13;
    const int nsteps = step_count(T, cfg.dt_nominal_1d(g.h, prob.c_max));
    const double dt = T / nsteps;
    Stepper1d ref(prob, g, 2);
    State1d rst = ref.init_leapfrog(dt);
    for (int i = 0; i < nsteps; ++i) ref.step_system(rst, i);
    DeviceStepper1d dev(prob, g, 2);
    State1d st = dev.init_leapfrog(dt);
    CHECK(dev.advance_to(st, T) == nsteps);
    CHECK(st.t_p == rst.t_p);
    CHECK(st.t_v == rst.t_v);
    for (int j = 0; j < K; ++j)
      for (int s = 0; s <= 2; ++s) {
        CHECK(st.p[j][s] == doctest::Approx(rst.p[j][s]).epsilon(1e-12));
        CHECK(st.v[j][s] == doctest::Approx(rst.v[j][s]).epsilon(1e-12));
      }
    State1d bad = dev.init_leapfrog(dt);
    CHECK_THROWS_AS(dev.advance_to(bad, T + 0.5 * dt), ConfigError);
  }
}

TEST_CASE("standing wave convergence, Hermite-leapfrog") {
  // tests/test_stepper1d.cpp:323-339 (values pinned to 5 digits there)
  Problem1d prob = standing_wave_problem();
  const double T = 4.13, cfl = 0.9;
  std::vector<int> Ks = {10, 20, 40, 80};
  std::vector<double> expect = {1.5081e-04, 2.3521e-06, 3.6708e-08, 5.7460e-10};
  std::vector<double> hs, es;
  for (size_t i = 0; i < Ks.size(); ++i) {
    const double e = leapfrog_l2(prob, 2, cfl, Ks[i], T);
    CHECK(std::abs(e / expect[i] - 1.0) < 2e-4);
    hs.push_back(2.0 / Ks[i]);
    es.push_back(e);
  }
  RateFit fit = convergence_rate(hs, es);
  CHECK(fit.points_used == 4);
  CHECK(std::abs(fit.rate - 6.00) < 0.3);
}

TEST_CASE("variable speed convergence with forcing, Hermite-leapfrog") {
  // tests/test_stepper1d.cpp:341-353 with the device stepper: c^2(x) jets and
  // the forcing provider of variable_speed_problem (problems.cpp:37-61)
  Problem1d prob = variable_speed_problem();
  const double T = 3.2, cfl = 0.9;
  std::vector<int> Ks = {10, 20, 40, 80};
  std::vector<double> expect = {5.3628e-06, 8.0000e-08, 1.2426e-09, 1.9781e-11};
  std::vector<double> hs, es;
  for (size_t i = 0; i < Ks.size(); ++i) {
    const double e = leapfrog_l2(prob, 2, cfl, Ks[i], T);
    CHECK(e == doctest::Approx(expect[i]).epsilon(0.02));
    hs.push_back(2.0 * pi / Ks[i]);
    es.push_back(e);
  }
  RateFit fit = convergence_rate(hs, es);
  CHECK(std::abs(fit.rate - 6.02) < 0.3);
}

TEST_CASE("device matches the reference stepper state, constant and variable ap") {
  for (int variant = 0; variant < 3; ++variant) {
    Problem1d prob = variant == 0 ? standing_wave_problem()
                     : variant == 1 ? variable_unforced_problem() : variable_speed_problem();
    for (int m = 0; m <= 5; ++m) {
      Grid1d g = Grid1d::over(prob.x_min, prob.x_max, 32);
      Stepper1d ref(prob, g, m);
      DeviceStepper1d dev(prob, g, m);
      const double dt = 0.5 * g.h / prob.c_max;
      State1d a = ref.init_leapfrog(dt), b = dev.init_leapfrog(dt);
      for (int i = 0; i < 40; ++i) ref.step_system(a, i);
      dev.advance_n(b, 40, 0);
      CHECK(max_rel(b.p, a.p) <= 1e-12);
      CHECK(max_rel(b.v, a.v) <= 1e-12);
      CHECK(b.t_p == a.t_p);
      CHECK(b.t_v == a.t_v);
    }
  }
}

TEST_CASE("discrete invariants hold across steps and orders") {
  // tests/test_stepper1d.cpp:389-417
  Problem1d prob = random_wave_problem(1234);
  Grid1d g = Grid1d::over(-1.0, 1.0, 16);
  const int nsteps = 100;
  for (int m = 0; m <= 3; ++m) {
    for (double cfl : {0.1, 0.5, 0.9}) {
      SchemeConfig cfg;
      cfg.m = m;
      cfg.cfl = cfl;
      const double dt = cfg.dt_nominal_1d(g.h, prob.c_max);
      DeviceStepper1d stepper(prob, g, m);
      State1d st = stepper.init_leapfrog(dt);
      const double q0 = conserved_r(st.v, st.p, g, stepper.op(), 1.0, dt);
      REQUIRE(q0 > 0.0);
      double drift = 0.0;
      for (int i = 0; i < nsteps; ++i) {
        stepper.advance_p(st);
        const double q = conserved_q(st.p, st.v, g, stepper.op(), 1.0, dt);
        drift = std::max(drift, std::abs(q / q0 - 1.0));
        stepper.advance_v(st);
        const double r = conserved_r(st.v, st.p, g, stepper.op(), 1.0, dt);
        drift = std::max(drift, std::abs(r / q0 - 1.0));
      }
      CHECK(drift < 1e-10);
    }
  }
}

TEST_CASE("unsupported problem features are configuration errors") {
  Grid1d g = Grid1d::over(0.0, 2.0 * pi, 16);
  CHECK_THROWS_AS(DeviceStepper1d(standing_wave_problem(), g, 9), ConfigError);   // m cap
}

TEST_CASE("a one-field problem runs only the modified scheme") {
  // the leapfrog and Dual-Hermite initialisers throw like the reference's
  // (stepper1d.cpp:132-133, 236-237)
  Grid1d g = Grid1d::over(0.0, 2.0 * pi, 16);
  Problem1d adv = advection_problem();
  DeviceStepper1d dev(adv, g, 2);
  CHECK_THROWS_AS(dev.init_leapfrog(0.1), ConfigError);
  CHECK_THROWS_AS(dev.init_dual_hermite(0.1), ConfigError);
}

TEST_CASE("modified scheme advection convergence (single field) on the device") {
  // tests/test_stepper1d.cpp:357-371 (PAPER Table 3) with the device stepper:
  // the reference's own goldens and rate band
  Problem1d prob = advection_problem();
  const double T = 4.13, cfl = 0.9;
  std::vector<int> Ks = {10, 20, 40};
  std::vector<double> expect = {1.298e-03, 2.212e-05, 3.541e-07};
  std::vector<double> hs, es;
  for (size_t i = 0; i < Ks.size(); ++i) {
    Grid1d g = Grid1d::over(prob.x_min, prob.x_max, Ks[i]);
    SchemeConfig cfg;
    cfg.m = 2;
    cfg.cfl = cfl;
    const int nsteps = step_count(T, cfg.dt_nominal_1d(g.h, prob.c_max));
    const double dt = T / nsteps;
    DeviceStepper1d stepper(prob, g, 2);
    ModifiedState1d st = stepper.init_modified(dt);
    for (int k = 0; k < nsteps; ++k) stepper.step_modified(st, k);
    const double e = l2_error_1d(st.prim[0], g, stepper.op(), true,
                                 [&](double x) { return prob.exact_value(0, x, st.t); });
    CHECK(e == doctest::Approx(expect[i]).epsilon(0.02));
    hs.push_back(2.0 / Ks[i]);
    es.push_back(e);
  }
  RateFit fit = convergence_rate(hs, es);
  CHECK(std::abs(fit.rate - 5.98) < 0.4);
}

TEST_CASE("single-field modified scheme matches the reference bit for bit") {
  Problem1d prob = advection_problem();
  for (int m = 0; m <= 5; ++m) {
    Grid1d g = Grid1d::over(prob.x_min, prob.x_max, 24);
    Stepper1d ref(prob, g, m);
    DeviceStepper1d dev(prob, g, m);
    const double dt = 0.4 * g.h / prob.c_max;
    ModifiedState1d a = ref.init_modified(dt), b = dev.init_modified(dt);
    for (int i = 0; i < 30; ++i) {
      ref.step_modified(a, i);
      dev.step_modified(b, i);
    }
    CHECK(max_rel(b.prim[0], a.prim[0]) == 0.0);
    CHECK(max_rel(b.dual[0], a.dual[0]) == 0.0);
    CHECK(b.t == a.t);
  }
}

TEST_CASE("modified and Dual-Hermite variants match the reference bit for bit") {
  // stepper1d.cpp:174-272 on the device (constant coefficients)
  for (const Problem1d& prob : {standing_wave_problem(), random_wave_problem(1234)}) {
    for (int m = 0; m <= 4; ++m) {
      Grid1d g = Grid1d::over(prob.x_min, prob.x_max, 24);
      Stepper1d ref(prob, g, m);
      DeviceStepper1d dev(prob, g, m);
      const double dt = 0.5 * g.h / prob.c_max;
      ModifiedState1d a = ref.init_modified(dt), b = dev.init_modified(dt);
      for (int i = 0; i < 25; ++i) {
        ref.step_modified(a, i);
        dev.step_modified(b, i);
      }
      for (int f = 0; f < 2; ++f) {
        CHECK(max_rel(b.prim[f], a.prim[f]) == 0.0);
        CHECK(max_rel(b.dual[f], a.dual[f]) == 0.0);
      }
      CHECK(b.t == a.t);
      DualState1d c = ref.init_dual_hermite(dt), d = dev.init_dual_hermite(dt);
      for (int i = 0; i < 25; ++i) {
        ref.step_dual_hermite(c, i);
        dev.step_dual_hermite(d, i);
      }
      CHECK(max_rel(d.p, c.p) == 0.0);
      CHECK(max_rel(d.v, c.v) == 0.0);
      CHECK(d.t == c.t);
    }
  }
}
