// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Stand-in for GSL's fixed Gauss-Legendre tables (`find_package(GSL)`,
// reference proj/CMakeLists.txt:14), the only GSL entry points the reference
// calls (proj/src/analysis.cpp:21-29).  Nodes are the roots of P_n found by
// Newton iteration from the Chebyshev guess, weights 2/((1-x^2) P_n'(x)^2);
// gsl_integration_glfixed_point returns node i in ascending order mapped to
// [a, b], as GSL documents.  Pinned through the reference's L2 goldens
// (proj/tests/test_stepper1d.cpp:323-387), which the compiled reference
// reproduces with this shim.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdlib>

typedef struct {
  size_t n;
  double* x;  // ascending nodes on [-1, 1]
  double* w;
} gsl_integration_glfixed_table;

static inline gsl_integration_glfixed_table* gsl_integration_glfixed_table_alloc(size_t n) {
  gsl_integration_glfixed_table* t =
      static_cast<gsl_integration_glfixed_table*>(std::malloc(sizeof(gsl_integration_glfixed_table)));
  t->n = n;
  t->x = static_cast<double*>(std::malloc(n * sizeof(double)));
  t->w = static_cast<double*>(std::malloc(n * sizeof(double)));
  const double pi = std::acos(-1.0);
  for (size_t i = 0; i < n; ++i) {
    // i-th root counted from the top, then stored ascending
    double x = std::cos(pi * (static_cast<double>(i) + 0.75) / (static_cast<double>(n) + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (size_t k = 2; k <= n; ++k) {
        const double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / static_cast<double>(k);
        p0 = p1;
        p1 = pk;
      }
      if (n == 1) {
        p1 = x;
        p0 = 1.0;
      }
      dp = static_cast<double>(n) * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-16) break;
    }
    // recompute the derivative at the converged root
    {
      double p0 = 1.0, p1 = x;
      for (size_t k = 2; k <= n; ++k) {
        const double pk = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / static_cast<double>(k);
        p0 = p1;
        p1 = pk;
      }
      dp = n == 1 ? 1.0 : static_cast<double>(n) * (x * p1 - p0) / (x * x - 1.0);
    }
    t->x[n - 1 - i] = x;
    t->w[n - 1 - i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
  return t;
}

static inline int gsl_integration_glfixed_point(double a, double b, size_t i, double* xi,
                                                double* wi, const gsl_integration_glfixed_table* t) {
  if (i >= t->n) return 1;
  const double A = 0.5 * (b - a), B = 0.5 * (b + a);
  *xi = B + A * t->x[i];
  *wi = A * t->w[i];
  return 0;
}

static inline void gsl_integration_glfixed_table_free(gsl_integration_glfixed_table* t) {
  if (!t) return;
  std::free(t->x);
  std::free(t->w);
  std::free(t);
}
