// Host-only plan helpers that need more than double precision (binary128 via
// libquadmath).  Compiled by the host compiler with -ffp-contract=off.
//
// alpha = beta = 1/2: the Hahn expansion (PAPER.md, asymptotics.py:36-75)
// terminates after its m = 0 term, P_n(cos phi) = k_n sin((n+1) phi) / sin phi
// with k_n = P_n(1) / (n+1).  The reference nevertheless plans no asymptotic
// blocks for this pair (g_M == 0 gives n_M = 0 and tbar = 0, asymptotics.py:
// 123-124, 238-250) and evaluates P_n by recurrence at every Lobatto row, at
// the point its libm angles define: x_p = cos(theta_p) in the interior, and
// 1 + xm_p / -1 + xm_p with the half-angle xm_p near +-1 (_kernels_cy.pyx:
// 27, 58-64).  Those points sit a few 1e-16 off the ideal angles pi p / G, and
// the (conditioning-limited) inverse inherits that offset.  The
// tables below let the device evaluate the closed form at exactly those
// points: phi_p = theta*_p + delta_p with theta*_p = pi p / G, and to first
// order in (n+1) delta_p (<= 1e-10 here, so the neglected term is ~1e-21)
//   sin((n+1) phi_p) = sin((n+1) theta*_p) + (n+1) delta_p cos((n+1) theta*_p).

#include <quadmath.h>
#include <stdint.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/cjt.h"

namespace {

// (no Q literal suffix: -std=c++17 without GNU extensions)
const __float128 kOne = 1, kTwo = 2, kHalf = 0.5;
const __float128 kPi = 4 * atanq(kOne);   // M_PIq uses the Q suffix

__float128 effective_angle(double x, double xm, int8_t region) {
  if (region == 1) return kTwo * asinq(sqrtq(-(__float128)xm / kTwo));              // x = 1 + xm
  if (region == -1) return kPi - kTwo * asinq(sqrtq((__float128)xm / kTwo));      // x = -1 + xm
  return acosq((__float128)x);
}

}  // namespace

extern "C" int cjt_host_half_exact(const double* x, const double* xm, const int8_t* regions, int64_t G,
                                   int64_t n, double* k, double* inv_sin, double* delta_over_sin) {
  // inv_sin == delta_over_sin == nullptr: only k (the forward plan needs no row tables)
  const bool want_rows = inv_sin || delta_over_sin;
  if (n < 0 || !k) return CJT_EINVAL;
  if (want_rows && (G < 1 || !x || !xm || !regions || !inv_sin || !delta_over_sin)) return CJT_EINVAL;
  // P_m(1) = Gamma(m + 3/2) / (Gamma(3/2) m!): P_m(1) = P_{m-1}(1) (m + 1/2) / m
  __float128 p1 = kOne;
  for (int64_t m = 0; m <= n; ++m) {
    if (m > 0) p1 = p1 * ((__float128)m + kHalf) / (__float128)m;
    k[m] = (double)(p1 / (__float128)(m + 1));
  }
  if (!want_rows) return CJT_OK;
  auto rows = [&](int64_t p0, int64_t p1) {
    for (int64_t p = p0; p < p1; ++p) {
      if (p == 0 || p == G) {
        inv_sin[p] = 0.0;
        delta_over_sin[p] = 0.0;
        continue;
      }
      const __float128 phi = effective_angle(x[p], xm[p], regions[p]);
      const __float128 ideal = kPi * (__float128)p / (__float128)G;
      const __float128 s = sinq(phi);
      inv_sin[p] = (double)(kOne / s);
      delta_over_sin[p] = (double)((phi - ideal) / s);
    }
  };
  // binary128 is software arithmetic (~1 us per row): large grids on threads
  const int64_t nrow = G + 1;
  const int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                        std::max<int64_t>(1, nrow / 8192));
  if (nt <= 1) {
    rows(0, nrow);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(rows, nrow * t / nt, nrow * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
  return CJT_OK;
}
