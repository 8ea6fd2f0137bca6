// Drop-in 2D stepper over the reference's own 2D types (Problem2d, Grid2d,
// TensorJet, PiecewiseTensor: proj/include/hlf/problem.hpp:34-55,
// grid.hpp:24-39, jet.hpp:34-46, interpolation.hpp:43-55), running the
// half steps on the B200 through the C-ABI (hlf_b200.h).
//
// The reference specifies but does not implement the 2D stepper
// (module stepper2d); this class is that module's
// interface in the reference's idiom, shaped like its Stepper1d
// (stepper1d.hpp:66-96):
//   * State2d (SPEC.md "StaggeredState2d"): caller-owned, host-resident,
//     p on the primary grid at t_p, the velocities (v along x, u along y;
//     Problem2d field order p, v, u, problem.hpp:41-46) on the dual grid at
//     t_v = t_p + dt/2; one TensorJet of (m+1) x (m+1) scaled coefficients per
//     node, nodes row-major ix * Ny + iy (PiecewiseTensor::cell's order);
//   * init_leapfrog(dt, t0) from Problem2d::exact like Stepper1d::init_leapfrog
//     (stepper1d.cpp:131-145); advance_p / advance_v / step_system; advance_n
//     and advance_to keep the state on the device for the whole run;
//   * reflective problems (Problem2d::boundary) put the walls on primary-grid
//     lines: K + 1 primary nodes per axis;
//   * Maxwell TM (Problem2d::System::maxwell_tm, fields Ez, Hx, Hy) runs on the
//     acoustic kernels with p = Ez, v = -Hy, u = Hx (problem.hpp:34-37);
//   * cells(state) builds the PiecewiseTensor of p on the dual cells with the
//     reference's own reconstruct_cell_2d, so the reference's l2_error_2d
//     (analysis.hpp:65-66) measures the device state unchanged.
// Exceptions: ConfigError (bad m, non-square grid handled by Grid2d::over),
// InstabilityError{step} (check_finite's message), std::invalid_argument.
#pragma once

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hlf/b200/device_stepper.hpp"
#include "hlf/config.hpp"
#include "hlf/grid.hpp"
#include "hlf/interpolation.hpp"
#include "hlf/jet.hpp"
#include "hlf/problem.hpp"

namespace hlf::b200 {

struct State2d {
  double t_p = 0.0, t_v = 0.0, dt = 0.0;
  std::vector<TensorJet> p, v, u;  // p: primary nodes; v (x-velocity), u (y-velocity): dual nodes
};

class Stepper2d {
 public:
  Stepper2d(Problem2d prob, Grid2d grid, int m) : prob_(std::move(prob)), grid_(grid), m_(m), n1_(m + 1) {
    SchemeConfig guard;
    guard.m = m;
    guard.validate();
    walls_ = prob_.boundary == Boundary::reflective;
    maxwell_ = prob_.system == Problem2d::System::maxwell_tm;
    op_ = build_interp_operator(m);
    hlf_desc d{};
    d.dim = 2;
    d.m = m;
    d.K[0] = d.K[1] = grid_.K;
    d.x_min[0] = grid_.x_min;
    d.x_min[1] = grid_.y_min;
    d.h = grid_.h;
    d.boundary[0] = d.boundary[1] = walls_ ? HLF_REFLECTIVE : HLF_PERIODIC;
    d.ap = -1.0;  // dp/dt = -(dv/dx + du/dy), dv/dt = -dp/dx, du/dt = -dp/dy (problem.hpp:34-36)
    d.av = -1.0;
    d.M = op_.M.data();
    try {
      dev_ = std::make_unique<DeviceStepper>(d);
    } catch (const Error& e) {
      if (e.status == HLF_CONFIG_ERROR) throw ConfigError(e.what());
      throw;
    }
  }

  int primary_nodes() const { return grid_.K + (walls_ ? 1 : 0); }  // per axis
  int dual_nodes() const { return grid_.K; }

  // exact jets of p at (primary, t0), velocities at (dual, t0 + dt/2)
  State2d init_leapfrog(double dt, double t0 = 0.0) const {
    State2d st;
    st.dt = dt;
    st.t_p = t0;
    st.t_v = t0 + dt / 2.0;
    const int Np = primary_nodes(), Nd = dual_nodes();
    st.p.reserve(static_cast<size_t>(Np) * Np);
    for (int i = 0; i < Np; ++i)
      for (int j = 0; j < Np; ++j)
        st.p.push_back(prob_.exact(0, grid_.primary_x(i), grid_.primary_y(j), t0, grid_.h, n1_));
    st.v.reserve(static_cast<size_t>(Nd) * Nd);
    st.u.reserve(static_cast<size_t>(Nd) * Nd);
    for (int i = 0; i < Nd; ++i)
      for (int j = 0; j < Nd; ++j) {
        st.v.push_back(prob_.exact(1, grid_.dual_x(i), grid_.dual_y(j), st.t_v, grid_.h, n1_));
        st.u.push_back(prob_.exact(2, grid_.dual_x(i), grid_.dual_y(j), st.t_v, grid_.h, n1_));
      }
    return st;
  }

  void advance_p(State2d& st) const {
    upload(st);
    guarded([&] { dev_->advance_p(); }, st);
    download(st);
  }
  void advance_v(State2d& st) const {
    upload(st);
    guarded([&] { dev_->advance_v(); }, st);
    download(st);
  }
  void step_system(State2d& st, int step_index) const {
    upload(st);
    guarded([&] { dev_->step(step_index); }, st);
    download(st);
  }
  void advance_n(State2d& st, int n, int first_step = 0) const {
    upload(st);
    guarded([&] { dev_->advance_n(n, first_step); }, st);
    download(st);
  }
  // from st.t_p to T in steps of st.dt (the caller loop, test_stepper1d.cpp:33-38);
  // returns the steps run; ConfigError when st.dt does not divide T - t_p
  int advance_to(State2d& st, double T, int first_step = 0) const {
    upload(st);
    int n = 0;
    guarded([&] { n = dev_->advance_to(T, first_step); }, st);
    download(st);
    return n;
  }

  // p on the dual cells (centred on dual nodes, corners the four primary
  // nodes), reconstructed by the reference's reconstruct_cell_2d
  // (interpolation.cpp:77-113): input of the reference's l2_error_2d
  PiecewiseTensor cells(const State2d& st) const {
    const int K = grid_.K, Np = primary_nodes();
    PiecewiseTensor pw;
    pw.nx = pw.ny = K;
    pw.h = grid_.h;
    for (int i = 0; i < K; ++i) {
      pw.cx.push_back(grid_.dual_x(i));
      pw.cy.push_back(grid_.dual_y(i));
      pw.lo_x.push_back(grid_.primary_x(i));
      pw.hi_x.push_back(grid_.primary_x(i + 1));
      pw.lo_y.push_back(grid_.primary_y(i));
      pw.hi_y.push_back(grid_.primary_y(i + 1));
    }
    auto node = [&](int i, int j) -> const TensorJet& {
      if (!walls_) {
        i = grid_.wrap(i);
        j = grid_.wrap(j);
      }
      return st.p[static_cast<size_t>(i) * Np + j];
    };
    pw.ext.reserve(static_cast<size_t>(K) * K);
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < K; ++j)
        pw.ext.push_back(reconstruct_cell_2d(op_, node(i, j), node(i + 1, j), node(i, j + 1), node(i + 1, j + 1)));
    return pw;
  }

  const Problem2d& problem() const { return prob_; }
  const Grid2d& grid() const { return grid_; }
  const InterpOperator& op() const { return op_; }
  int m() const { return m_; }

 private:
  Problem2d prob_;
  Grid2d grid_;
  int m_, n1_;
  bool walls_ = false, maxwell_ = false;
  InterpOperator op_;
  std::unique_ptr<DeviceStepper> dev_;

  std::vector<double> flat(const std::vector<TensorJet>& jets, size_t count, double sign) const {
    if (jets.size() != count) throw std::invalid_argument("State2d: one TensorJet per node expected");
    const size_t F = static_cast<size_t>(n1_) * n1_;
    std::vector<double> out(count * F);
    for (size_t k = 0; k < count; ++k) {
      if (jets[k].nx != n1_ || jets[k].ny != n1_) throw std::invalid_argument("State2d jets must be (m+1)^2");
      for (size_t e = 0; e < F; ++e) out[k * F + e] = sign * jets[k].a[e];
    }
    return out;
  }
  void unflat(const std::vector<double>& in, std::vector<TensorJet>& jets, double sign) const {
    const size_t F = static_cast<size_t>(n1_) * n1_;
    for (size_t k = 0; k < jets.size(); ++k)
      for (size_t e = 0; e < F; ++e) jets[k].a[e] = sign * in[k * F + e];
  }
  // device field 1 = velocity along x, 2 = along y; Maxwell TM: (Hx, Hy) ->
  // (-Hy, Hx) on the device
  void upload(const State2d& st) const {
    const size_t Np = static_cast<size_t>(primary_nodes()) * primary_nodes();
    const size_t Nd = static_cast<size_t>(dual_nodes()) * dual_nodes();
    dev_->set_field(0, flat(st.p, Np, 1.0));
    if (maxwell_) {
      dev_->set_field(1, flat(st.u, Nd, -1.0));  // -Hy
      dev_->set_field(2, flat(st.v, Nd, 1.0));   // Hx
    } else {
      dev_->set_field(1, flat(st.v, Nd, 1.0));
      dev_->set_field(2, flat(st.u, Nd, 1.0));
    }
    dev_->set_times(st.t_p, st.t_v, st.dt);
  }
  void download(State2d& st) const {
    unflat(dev_->get_field(0), st.p, 1.0);
    if (maxwell_) {
      unflat(dev_->get_field(1), st.u, -1.0);
      unflat(dev_->get_field(2), st.v, 1.0);
    } else {
      unflat(dev_->get_field(1), st.v, 1.0);
      unflat(dev_->get_field(2), st.u, 1.0);
    }
    dev_->times(st.t_p, st.t_v, st.dt);
  }
  template <class Fn>
  void guarded(Fn&& fn, State2d& st) const {
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
