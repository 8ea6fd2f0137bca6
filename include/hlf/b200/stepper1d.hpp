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
// Coverage: the Hermite-leapfrog variant (step_system).  Coefficient jets are
// taken from the problem at construction like the reference (stepper1d.cpp:
// 103-110): constant ap/av run the constant-coefficient kernels, a varying ap
// runs the per-node ap-jet kernels (av must be constant).  Problems with a
// forcing provider, a varying av, or the modified / Dual-Hermite variants are
// rejected with ConfigError (the reference's CPU Stepper1d still covers them).
#pragma once

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
    if (prob_.n_fields != 2) throw ConfigError("the staggered scheme needs a two-field system");
    if (prob_.forcing) throw ConfigError("forcing providers are not supported on the device path");
    op_ = build_interp_operator(m);  // the host operator, handed to the device unchanged
    std::vector<double> ap_prim, ap_dual;
    bool ap_const = true, av_const = true;
    double ap0 = 0.0, av0 = 0.0;
    for (int j = 0; j < grid_.K; ++j) {
      for (int on_dual = 0; on_dual < 2; ++on_dual) {
        const double x = on_dual ? grid_.dual(j) : grid_.primary(j);
        Jet ap = prob_.ap(x, grid_.h, n_);
        Jet av = prob_.av(x, grid_.h, n_);
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
  }

  // stepper1d.cpp:131-145
  State1d init_leapfrog(double dt, double t0 = 0.0) const {
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

  void advance_p(State1d& st) const {
    upload(st);
    guarded([&] { dev_->advance_p(); }, st);
    download(st);
  }
  void advance_v(State1d& st) const {
    upload(st);
    guarded([&] { dev_->advance_v(); }, st);
    download(st);
  }
  // stepper1d.cpp:168-172: throws InstabilityError(step_index) like check_finite
  void step_system(State1d& st, int step_index) const {
    upload(st);
    guarded([&] { dev_->step(step_index); }, st);
    download(st);
  }
  // extension: n steps with the state resident on the device
  void advance_n(State1d& st, int n, int first_step = 0) const {
    upload(st);
    guarded([&] { dev_->advance_n(n, first_step); }, st);
    download(st);
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

  void upload(const State1d& st) const {
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
