// Drop-in replacement for the reference's hlf::Stepper1d
// (proj/include/hlf/stepper1d.hpp:66-96) that runs the half steps on the B200
// through the C-ABI (hlf_b200.h).  It is written against the reference's own
// public types -- Problem1d, Grid1d, State1d, InterpOperator, ConfigError,
// InstabilityError -- so a caller swaps
//     hlf::Stepper1d stepper(prob, g, m);
// for
//     hlf::b200::Stepper1d stepper(prob, g, m);
// and keeps the rest of its code (tests/cpp/test_b200_stepper1d.cpp is the
// reference's test_stepper1d.cpp re-targeted this way).
//
// State1d stays caller-owned and host-resident, exactly as in the reference
// (stepper1d.hpp:49-52): advance_p/advance_v/step_system upload the jets,
// run on the device and download them.  advance_n (an extension) keeps the
// state on the device for n steps and is the call to use for long runs.
//
// Coverage: the Hermite-leapfrog variant (step_system) and, for constant
// coefficients, the modified (init_modified / step_modified) and classic
// Dual-Hermite (init_dual_hermite / step_dual_hermite) variants, bit-identical
// to the reference.  Coefficient jets are taken from the problem at
// construction like the reference (stepper1d.cpp:103-110): constant ap/av run
// the constant-coefficient kernels, a varying ap runs the per-node ap-jet
// kernels (leapfrog only; av must be constant).  A forcing provider
// (Problem1d::forcing, stepper1d.cpp:113-119) is evaluated on the host at the
// nodes and times the reference uses and handed to the device per half step
// (hlf_set_forcing; leapfrog only).  A varying av is rejected with ConfigError
// (the reference's CPU Stepper1d still covers it).
#pragma once

#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hlf/b200/device_stepper.hpp"
#include "hlf/config.hpp"
#include "hlf/grid.hpp"
#include "hlf/interpolation.hpp"
#include "hlf/problem.hpp"
#include "hlf/stepper1d.hpp"

namespace hlf::b200 {

class Stepper1d {
 public:
  Stepper1d(Problem1d prob, Grid1d grid, int m) : prob_(std::move(prob)), grid_(grid), m_(m), n_(2 * m + 2) {
    SchemeConfig guard;  // stepper1d.cpp:95-97
    guard.m = m;
    guard.validate();
    // one field (scalar advection, problem.hpp:16-17) runs only the modified
    // scheme (step_modified's n_fields == 1 branch, stepper1d.cpp:205-209)
    if (prob_.n_fields != 1 && prob_.n_fields != 2) throw ConfigError("the device path needs one or two fields");
    one_field_ = prob_.n_fields == 1;
    op_ = build_interp_operator(m);  // the host operator, handed to the device unchanged
    std::vector<double> ap_prim, ap_dual;
    bool ap_const = true, av_const = true;
    double ap0 = 0.0, av0 = 0.0;
    for (int j = 0; j < grid_.K; ++j) {
      for (int on_dual = 0; on_dual < 2; ++on_dual) {
        const double x = on_dual ? grid_.dual(j) : grid_.primary(j);
        Jet ap = prob_.ap(x, grid_.h, n_);
        Jet av = one_field_ ? constant_jet(0.0, n_) : prob_.av(x, grid_.h, n_);
        if (j == 0 && on_dual == 0) {
          ap0 = ap[0];
          av0 = av[0];
        }
        for (int s = 0; s < n_; ++s) {
          if (ap[s] != (s == 0 ? ap0 : 0.0)) ap_const = false;
          if (av[s] != (s == 0 ? av0 : 0.0)) av_const = false;
        }
        (on_dual ? ap_dual : ap_prim).insert((on_dual ? ap_dual : ap_prim).end(), ap.begin(), ap.end());
      }
    }
    if (!av_const) throw ConfigError("a spatially varying av is not supported on the device path");
    hlf_desc d{};
    d.dim = 1;
    d.m = m;
    d.K[0] = grid_.K;
    d.x_min[0] = grid_.x_min;
    d.h = grid_.h;
    d.boundary[0] = HLF_PERIODIC;
    d.ap = ap0;
    d.av = av0;
    d.variable_ap = ap_const ? 0 : 1;
    d.M = op_.M.data();
    dev_ = std::make_unique<DeviceStepper>(d);
    if (!ap_const) {
      dev_->set_coeff(HLF_PRIMARY, ap_prim);
      dev_->set_coeff(HLF_DUAL, ap_dual);
    }
    desc_ = d;
    ap_const_ = ap_const;
  }

  bool one_field() const { return one_field_; }

  // stepper1d.cpp:131-145
  State1d init_leapfrog(double dt, double t0 = 0.0) const {
    if (one_field_) throw ConfigError("init_leapfrog requires a two-field system");  // stepper1d.cpp:132-133
    State1d st;
    st.dt = dt;
    st.t_p = t0;
    st.t_v = t0 + dt / 2.0;
    st.p.resize(grid_.K);
    st.v.resize(grid_.K);
    for (int j = 0; j < grid_.K; ++j) {
      st.p[j] = prob_.exact(0, grid_.primary(j), t0, grid_.h, m_ + 1);
      st.v[j] = prob_.exact(1, grid_.dual(j), st.t_v, grid_.h, m_ + 1);
    }
    return st;
  }

  // forcing levels: advance_p at (primary x_j, t_v), advance_v at (dual x_j,
  // t_p) (stepper1d.cpp:152, 162)
  void advance_p(State1d& st) const {
    upload(st);
    if (prob_.forcing) dev_->set_forcing(HLF_PRIMARY, forcing_table(false, st.t_v));
    guarded([&] { dev_->advance_p(); }, st);
    download(st);
  }
  void advance_v(State1d& st) const {
    upload(st);
    if (prob_.forcing) dev_->set_forcing(HLF_DUAL, forcing_table(true, st.t_p));
    guarded([&] { dev_->advance_v(); }, st);
    download(st);
  }
  // stepper1d.cpp:168-172: throws InstabilityError(step_index) like check_finite
  void step_system(State1d& st, int step_index) const {
    upload(st);
    guarded([&] { forced_or_plain_steps(st, 1, step_index); }, st);
    download(st);
  }
  // extension: n steps with the state resident on the device
  void advance_n(State1d& st, int n, int first_step = 0) const {
    upload(st);
    guarded([&] { forced_or_plain_steps(st, n, first_step); }, st);
    download(st);
  }
  // extension: from st.t_p to T in steps of st.dt, i.e. the caller loop of
  // test_stepper1d.cpp:33-38 (dt = T / step_count(T, dt_nominal) chosen before
  // init_leapfrog); returns the steps run.  ConfigError when st.dt does not
  // divide T - t_p (the staggered v sits half a step of that dt away).
  int advance_to(State1d& st, double T, int first_step = 0) const {
    if (prob_.forcing) {
      // forcing tables are evaluated per half step on the host: the same
      // step rule as hlf_advance_to, then the forced steps one by one
      const double q = st.dt != 0.0 ? (T - st.t_p) / st.dt : -1.0;
      const double nr = std::nearbyint(q);
      if (!(q > -1e-9) || std::fabs(q - nr) > 1e-9 * std::fmax(1.0, std::fabs(q)))
        throw ConfigError("dt does not divide T - t_p; initialise the state with dt = T / step_count(T, dt_nominal)");
      advance_n(st, static_cast<int>(nr), first_step);
      return static_cast<int>(nr);
    }
    upload(st);
    int n = 0;
    guarded([&] { n = dev_->advance_to(T, first_step); }, st);
    download(st);
    return n;
  }

  // ---- modified Hermite-leapfrog (stepper1d.cpp:174-232)
  ModifiedState1d init_modified(double dt, double t0 = 0.0) const {
    ModifiedState1d st;
    st.dt = dt;
    st.t = t0;
    st.prim.resize(prob_.n_fields);
    st.dual.resize(prob_.n_fields);
    for (int f = 0; f < prob_.n_fields; ++f) {
      st.prim[f].resize(grid_.K);
      st.dual[f].resize(grid_.K);
      for (int j = 0; j < grid_.K; ++j) {
        st.prim[f][j] = prob_.exact(f, grid_.primary(j), t0, grid_.h, m_ + 1);
        st.dual[f][j] = prob_.exact(f, grid_.dual(j), t0 + dt / 2.0, grid_.h, m_ + 1);
      }
    }
    return st;
  }
  void step_modified(ModifiedState1d& st, int step_index) const {
    if (one_field_) {
      // device fields: 0 = u primary (t), 1 = u dual (t + dt/2)
      DeviceStepper& dev = alt(HLF_SCHEME_MODIFIED_ADVECTION);
      dev.set_field(0, flat(st.prim[0]));
      dev.set_field(1, flat(st.dual[0]));
      dev.set_times(st.t, st.t + st.dt / 2.0, st.dt);
      auto down = [&] {
        unflat(dev.get_field(0), st.prim[0]);
        unflat(dev.get_field(1), st.dual[0]);
        double tv = 0.0, dt = 0.0;
        dev.times(st.t, tv, dt);
      };
      alt_guarded([&] { dev.step(step_index); }, down);
      down();
      return;
    }
    DeviceStepper& dev = alt(HLF_SCHEME_MODIFIED);
    // device fields: 0 = p primary, 1 = v dual, 2 = v primary, 3 = p dual
    const std::vector<Jet>* in[4] = {&st.prim[0], &st.dual[1], &st.prim[1], &st.dual[0]};
    for (int f = 0; f < 4; ++f) dev.set_field(f, flat(*in[f]));
    dev.set_times(st.t, st.t + st.dt / 2.0, st.dt);
    auto down = [&] {
      std::vector<Jet>* out[4] = {&st.prim[0], &st.dual[1], &st.prim[1], &st.dual[0]};
      for (int f = 0; f < 4; ++f) unflat(dev.get_field(f), *out[f]);
      double tv = 0.0, dt = 0.0;
      dev.times(st.t, tv, dt);
    };
    alt_guarded([&] { dev.step(step_index); }, down);
    down();
  }

  // ---- classic two-half-step Hermite baseline (stepper1d.cpp:235-272)
  DualState1d init_dual_hermite(double dt, double t0 = 0.0) const {
    if (one_field_) throw ConfigError("the classic Hermite baseline needs a two-field system");  // stepper1d.cpp:236-237
    DualState1d st;
    st.dt = dt;
    st.t = t0;
    st.p.resize(grid_.K);
    st.v.resize(grid_.K);
    for (int j = 0; j < grid_.K; ++j) {
      st.p[j] = prob_.exact(0, grid_.primary(j), t0, grid_.h, m_ + 1);
      st.v[j] = prob_.exact(1, grid_.primary(j), t0, grid_.h, m_ + 1);
    }
    return st;
  }
  void step_dual_hermite(DualState1d& st, int step_index) const {
    DeviceStepper& dev = alt(HLF_SCHEME_DUAL_HERMITE);
    dev.set_field(0, flat(st.p));
    dev.set_field(2, flat(st.v));
    dev.set_times(st.t, st.t, st.dt);
    auto down = [&] {
      unflat(dev.get_field(0), st.p);
      unflat(dev.get_field(2), st.v);
      double tv = 0.0, dt = 0.0;
      dev.times(st.t, tv, dt);
    };
    alt_guarded([&] { dev.step(step_index); }, down);
    down();
  }

  const Problem1d& problem() const { return prob_; }
  const Grid1d& grid() const { return grid_; }
  const InterpOperator& op() const { return op_; }
  int m() const { return m_; }

 private:
  Problem1d prob_;
  Grid1d grid_;
  int m_, n_;
  InterpOperator op_;
  std::unique_ptr<DeviceStepper> dev_;
  hlf_desc desc_{};
  bool ap_const_ = true;
  bool one_field_ = false;
  mutable std::unique_ptr<DeviceStepper> alt_dev_[4];  // per alternative scheme, created on first use

  DeviceStepper& alt(int scheme) const {
    if (!ap_const_) throw ConfigError("the modified / Dual-Hermite device path needs constant coefficients");
    if (prob_.forcing) throw ConfigError("the modified / Dual-Hermite device path has no forcing");
    if (!alt_dev_[scheme]) {
      hlf_desc d = desc_;
      d.scheme = scheme;
      d.variable_ap = 0;
      try {
        alt_dev_[scheme] = std::make_unique<DeviceStepper>(d);
      } catch (const Error& e) {
        if (e.status == HLF_CONFIG_ERROR) throw ConfigError(e.what());
        throw;
      }
    }
    return *alt_dev_[scheme];
  }
  // forcing_at(x_j, t)(r), r = 0..n-2, at every node of one grid: [K][n-1][n]
  std::vector<double> forcing_table(bool dual, double t) const {
    std::vector<double> out(static_cast<size_t>(grid_.K) * (n_ - 1) * n_, 0.0);
    for (int j = 0; j < grid_.K; ++j) {
      const double x = dual ? grid_.dual(j) : grid_.primary(j);
      for (int r = 0; r + 1 < n_; ++r) {
        const Jet z = prob_.forcing(r, x, t, grid_.h, n_);
        for (int i = 0; i < n_ && i < static_cast<int>(z.size()); ++i)
          out[(static_cast<size_t>(j) * (n_ - 1) + r) * n_ + i] = z[i];
      }
    }
    return out;
  }
  // n leapfrog steps on the device; with a forcing provider each step gets
  // its two tables (p at t_v, v at t_p + dt: the reference's t_p after
  // advance_p) and runs as one hlf_step
  void forced_or_plain_steps(const State1d& st, int n, int first_step) const {
    if (!prob_.forcing) {
      dev_->advance_n(n, first_step);
      return;
    }
    double t_p = st.t_p, t_v = st.t_v, dt = st.dt;
    for (int i = 0; i < n; ++i) {
      dev_->set_forcing(HLF_PRIMARY, forcing_table(false, t_v));
      dev_->set_forcing(HLF_DUAL, forcing_table(true, t_p + dt));
      dev_->step(first_step + i);
      dev_->times(t_p, t_v, dt);
    }
  }
  std::vector<double> flat(const std::vector<Jet>& jets) const {
    const int n1 = m_ + 1;
    if (static_cast<int>(jets.size()) != grid_.K) throw std::invalid_argument("one jet per node expected");
    std::vector<double> out(static_cast<size_t>(grid_.K) * n1);
    for (int j = 0; j < grid_.K; ++j) {
      if (static_cast<int>(jets[j].size()) != n1) throw std::invalid_argument("jets must hold m+1 entries");
      std::memcpy(out.data() + static_cast<size_t>(j) * n1, jets[j].data(), sizeof(double) * n1);
    }
    return out;
  }
  void unflat(const std::vector<double>& in, std::vector<Jet>& jets) const {
    const int n1 = m_ + 1;
    for (int j = 0; j < grid_.K; ++j)
      std::memcpy(jets[j].data(), in.data() + static_cast<size_t>(j) * n1, sizeof(double) * n1);
  }
  template <class Fn, class Down>
  void alt_guarded(Fn&& fn, Down&& down) const {
    try {
      fn();
    } catch (const Error& e) {
      if (e.status == HLF_INSTABILITY) {
        down();
        throw InstabilityError(instability_step(e.what()), e.what());
      }
      if (e.status == HLF_CONFIG_ERROR) throw ConfigError(e.what());
      throw;
    }
  }

  void upload(const State1d& st) const {
    if (one_field_) throw ConfigError("the Hermite-leapfrog half steps require a two-field system");
    const int n1 = m_ + 1;
    if (static_cast<int>(st.p.size()) != grid_.K || static_cast<int>(st.v.size()) != grid_.K)
      throw std::invalid_argument("State1d must hold one jet per node");
    std::vector<double> p(static_cast<size_t>(grid_.K) * n1), v(p.size());
    for (int j = 0; j < grid_.K; ++j) {
      if (static_cast<int>(st.p[j].size()) != n1 || static_cast<int>(st.v[j].size()) != n1)
        throw std::invalid_argument("State1d jets must hold m+1 entries");
      std::memcpy(p.data() + static_cast<size_t>(j) * n1, st.p[j].data(), sizeof(double) * n1);
      std::memcpy(v.data() + static_cast<size_t>(j) * n1, st.v[j].data(), sizeof(double) * n1);
    }
    dev_->set_field(0, p);
    dev_->set_field(1, v);
    dev_->set_times(st.t_p, st.t_v, st.dt);
  }
  void download(State1d& st) const {
    const int n1 = m_ + 1;
    const std::vector<double> p = dev_->get_field(0), v = dev_->get_field(1);
    for (int j = 0; j < grid_.K; ++j) {
      std::memcpy(st.p[j].data(), p.data() + static_cast<size_t>(j) * n1, sizeof(double) * n1);
      std::memcpy(st.v[j].data(), v.data() + static_cast<size_t>(j) * n1, sizeof(double) * n1);
    }
    dev_->times(st.t_p, st.t_v, st.dt);
  }
  // the reference updates the state before check_finite throws
  // (stepper1d.cpp:168-172), so the instability path still downloads it
  template <class Fn>
  void guarded(Fn&& fn, State1d& st) const {
    try {
      fn();
    } catch (const Error& e) {
      if (e.status == HLF_INSTABILITY) {
        download(st);
        throw InstabilityError(instability_step(e.what()), e.what());
      }
      if (e.status == HLF_CONFIG_ERROR) throw ConfigError(e.what());
      if (e.status == HLF_INVALID_ARGUMENT) throw std::invalid_argument(e.what());
      throw;
    }
  }
};

}  // namespace hlf::b200
