// Header-only C++ RAII wrapper over the C-ABI in hlf_b200.h (no reference
// types needed).  Errors become exceptions; the drop-in for the reference's
// own types (hlf::Stepper1d etc.) is hlf/b200/stepper1d.hpp.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "hlf_b200.h"

namespace hlf::b200 {

struct Error : std::runtime_error {
  hlf_status status;
  Error(hlf_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

// throws on any non-OK status; callers that need the reference's exception
// types translate (see stepper1d.hpp)
inline void check(hlf_status st, const hlf_solver* s) {
  if (st != HLF_OK) throw Error(st, hlf_last_error(s));
}

// step index carried by an HLF_INSTABILITY message ("... at step N")
inline int instability_step(const std::string& what) {
  const auto pos = what.find_last_of(' ');
  return pos == std::string::npos ? -1 : std::stoi(what.substr(pos + 1));
}

class DeviceStepper {
 public:
  explicit DeviceStepper(const hlf_desc& desc) {
    hlf_solver* s = nullptr;
    check(hlf_create(&desc, &s), nullptr);
    s_ = s;
    F_ = hlf_num_coeffs(s_);
    dim_ = desc.dim;
    scheme_ = desc.scheme;
  }
  ~DeviceStepper() { hlf_destroy(s_); }
  DeviceStepper(const DeviceStepper&) = delete;
  DeviceStepper& operator=(const DeviceStepper&) = delete;

  int coeffs() const { return F_; }
  int dim() const { return dim_; }
  int64_t nodes(int grid) const { return hlf_num_nodes(s_, grid); }
  // leapfrog: p primary, v dual; the alternative 1D schemes: even fields primary, odd dual
  int64_t field_nodes(int f) const {
    const bool primary = scheme_ == HLF_SCHEME_LEAPFROG ? f == 0 : f % 2 == 0;
    return nodes(primary ? HLF_PRIMARY : HLF_DUAL);
  }

  void set_field(int f, const std::vector<double>& aos) {
    if (static_cast<int64_t>(aos.size()) != field_nodes(f) * F_)
      throw std::invalid_argument("set_field: buffer must hold nodes x (m+1)^d entries");
    check(hlf_set_field(s_, f, aos.data()), s_);
  }
  std::vector<double> get_field(int f) const {
    std::vector<double> out(static_cast<size_t>(field_nodes(f) * F_));
    check(hlf_get_field(s_, f, out.data()), s_);
    return out;
  }
  void set_coeff(int grid, const std::vector<double>& jets) { check(hlf_set_coeff(s_, grid, jets.data()), s_); }
  void set_forcing(int grid, const std::vector<double>& table) {
    check(hlf_set_forcing(s_, grid, table.data()), s_);
  }
  void clear_forcing() { check(hlf_clear_forcing(s_), s_); }
  // advance_n replays chunks of `steps` steps as one CUDA graph (0: off)
  void set_graph_steps(int steps) { check(hlf_set_graph_steps(s_, steps), s_); }
  // on-device accessors (analysis.cpp:221-285)
  double l2_error_separable(int field, double amp, const double* w, const double* phase) {
    double l2 = 0.0;
    check(hlf_l2_error_separable(s_, field, amp, w, phase, &l2), s_);
    return l2;
  }
  double energy_1d(int kind, double c) {
    double e = 0.0;
    check(hlf_energy_1d(s_, kind, c, &e), s_);
    return e;
  }
  void set_times(double t_p, double t_v, double dt) { check(hlf_set_times(s_, t_p, t_v, dt), s_); }
  void times(double& t_p, double& t_v, double& dt) const { check(hlf_get_times(s_, &t_p, &t_v, &dt), s_); }
  void set_dt(double dt) { check(hlf_set_dt(s_, dt), s_); }

  void advance_p() { check(hlf_advance_p(s_), s_); }
  void advance_v() { check(hlf_advance_v(s_), s_); }
  void step(int step_index) { check(hlf_step(s_, step_index), s_); }
  void advance_n(int n, int first_step) { check(hlf_advance_n(s_, n, first_step), s_); }
  // from t_p to T in steps of the current dt (hlf_advance_to); returns the steps run
  int advance_to(double T, int first_step) {
    int n = 0;
    check(hlf_advance_to(s_, T, first_step, &n), s_);
    return n;
  }
  void synchronize() { check(hlf_synchronize(s_), s_); }

  hlf_solver* handle() const { return s_; }

 private:
  hlf_solver* s_ = nullptr;
  int F_ = 0, dim_ = 0, scheme_ = HLF_SCHEME_LEAPFROG;
};

}  // namespace hlf::b200
