// The multi-GPU z-slab path driven from a C++ host through the C-ABI only
// (hlf_slabs_*, include/hlf_b200.h): a periodic 3D box split into z slabs,
// each slab filled with the exact standing mode on the device, stepped with
// the library's own halo exchange, and compared bit for bit with one solver
// over the whole box.  One GPU: several slabs share device 0 (peer-copy
// transport) and one slab exercises the NCCL transport (self send/recv).
// Built by oracle/Makefile (`make -C oracle dropin`), run by
// tests/test_cpp_dropin.py on the GPU.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "hlf_b200.h"

namespace {
const double pi = std::acos(-1.0);

hlf_desc box_desc(int K0, int K1, int K2, int m, std::vector<double>& M) {
  M.assign(static_cast<size_t>((2 * m + 2) * (2 * m + 2)), 0.0);
  REQUIRE(hlf_build_interp_operator(m, M.data(), nullptr) == HLF_OK);
  hlf_desc d;
  std::memset(&d, 0, sizeof(d));
  d.dim = 3;
  d.m = m;
  d.K[0] = K0;
  d.K[1] = K1;
  d.K[2] = K2;
  d.x_min[0] = d.x_min[1] = d.x_min[2] = -1.0;
  d.h = 2.0 / K0;
  d.ap = d.av = -1.0;
  d.M = M.data();
  return d;
}

// p = cos(wt t) prod sin(w_a x_a), v_c = -(w_c/wt) sin(wt t) cos(w_c x_c) prod_{a != c} sin (t = dt/2 for v)
void fill_mode(hlf_solver* s, const hlf_desc& d, double dt) {
  double w[3], ph0[3] = {0, 0, 0};
  double wt2 = 0.0;
  for (int a = 0; a < 3; ++a) {
    w[a] = 2.0 * pi / (d.K[a] * d.h);
    wt2 += w[a] * w[a];
  }
  const double wt = std::sqrt(wt2);
  for (int f = 0; f < 4; ++f) REQUIRE(hlf_zero_field(s, f) == HLF_OK);
  REQUIRE(hlf_fill_separable(s, 0, 1.0, w, ph0) == HLF_OK);
  for (int c = 0; c < 3; ++c) {
    double ph[3] = {0, 0, 0};
    ph[c] = pi / 2;
    REQUIRE(hlf_fill_separable(s, 1 + c, -(w[c] / wt) * std::sin(wt * dt / 2), w, ph) == HLF_OK);
  }
}

std::vector<double> field(hlf_solver* s, int f) {
  const int64_t n = hlf_num_nodes(s, f == 0 ? HLF_PRIMARY : HLF_DUAL) * hlf_num_coeffs(s);
  std::vector<double> out(static_cast<size_t>(n));
  REQUIRE(hlf_get_field(s, f, out.data()) == HLF_OK);
  return out;
}

void run_case(int nslabs, int transport) {
  const int K0 = 64, K1 = 4, K2 = 12, m = 3, steps = 5;
  std::vector<double> M;
  hlf_desc d = box_desc(K0, K1, K2, m, M);
  const double dt = 0.9 * d.h / std::sqrt(3.0);
  // one solver over the whole box
  hlf_solver* full = nullptr;
  REQUIRE(hlf_create(&d, &full) == HLF_OK);
  fill_mode(full, d, dt);
  REQUIRE(hlf_set_times(full, 0.0, dt / 2, dt) == HLF_OK);
  REQUIRE(hlf_advance_n(full, steps, 0) == HLF_OK);
  // the slab group: each slab fills its part of the same global mode (x_min
  // of slab r is shifted by r kz h, so the separable fill is the global one)
  std::vector<int> devs(static_cast<size_t>(nslabs), 0);
  hlf_slab_group* g = nullptr;
  REQUIRE(hlf_slabs_create(&d, nslabs, devs.data(), transport, &g) == HLF_OK);
  CHECK(hlf_slabs_transport(g) == transport);
  for (int r = 0; r < nslabs; ++r) {
    hlf_desc dr = d;  // fill_mode needs the global periods
    fill_mode(hlf_slabs_solver(g, r), dr, dt);
  }
  REQUIRE(hlf_slabs_set_times(g, 0.0, dt / 2, dt) == HLF_OK);
  REQUIRE(hlf_slabs_advance_n(g, steps, 0) == HLF_OK);
  const int kz = K2 / nslabs;
  const int F = hlf_num_coeffs(full);
  for (int f = 0; f < 4; ++f) {
    const std::vector<double> ref = field(full, f);
    for (int r = 0; r < nslabs; ++r) {
      const std::vector<double> got = field(hlf_slabs_solver(g, r), f);
      // host AoS is x-major [x][y][z][coef]: slab r holds z in [r kz, (r+1) kz)
      bool same = true;
      for (int x = 0; x < K0 && same; ++x)
        for (int y = 0; y < K1 && same; ++y)
          for (int z = 0; z < kz && same; ++z)
            for (int c = 0; c < F; ++c) {
              const size_t gi = ((static_cast<size_t>(x) * K1 + y) * K2 + (r * kz + z)) * F + c;
              const size_t li = ((static_cast<size_t>(x) * K1 + y) * kz + z) * F + c;
              if (got[li] != ref[gi]) {
                same = false;
                break;
              }
            }
      CAPTURE(f);
      CAPTURE(r);
      CHECK(same);
    }
  }
  double tp = 0, tv = 0, dtt = 0, tp2 = 0, tv2 = 0, dt2 = 0;
  hlf_get_times(full, &tp, &tv, &dtt);
  hlf_get_times(hlf_slabs_solver(g, 0), &tp2, &tv2, &dt2);
  CHECK(tp == tp2);
  CHECK(tv == tv2);
  hlf_slabs_destroy(g);
  hlf_destroy(full);
}
}  // namespace

TEST_CASE("three slabs on one device (peer copies) equal one solver bit for bit") { run_case(3, HLF_TRANSPORT_COPY); }

TEST_CASE("four slabs on one device (peer copies) equal one solver bit for bit") { run_case(4, HLF_TRANSPORT_COPY); }

TEST_CASE("one slab through NCCL (self send / receive) equals one solver bit for bit") {
  run_case(1, HLF_TRANSPORT_NCCL);
}

TEST_CASE("bad splits are configuration errors") {
  std::vector<double> M;
  hlf_desc d = box_desc(64, 4, 12, 3, M);
  int devs[5] = {0, 0, 0, 0, 0};
  hlf_slab_group* g = nullptr;
  CHECK(hlf_slabs_create(&d, 5, devs, HLF_TRANSPORT_COPY, &g) == HLF_CONFIG_ERROR);
  CHECK(std::string(hlf_slabs_last_error(nullptr)).size() > 0);
  CHECK(hlf_slabs_create(&d, 2, devs, HLF_TRANSPORT_NCCL, &g) == HLF_CONFIG_ERROR);
}
