/*
 * ORACLE - TEST INFRASTRUCTURE ONLY.  Not part of the product; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Plain-C restatement of the reference's two recurrence kernels
 * (/root/reference/pkg/src/chebjac/_kernels_cy.pyx):
 *   oracle_clenshaw_points       _kernels_cy.pyx:83-122 (helpers 17-80)
 *   oracle_transpose_accumulate  _kernels_cy.pyx:201-237 (helpers 125-198)
 * Same grouping into runs of equal (cut, region), same lanes of 8, same
 * operation order, libm cos/sin; compiled with -ffp-contract=off so no FMA
 * contraction changes the rounding.
 */
#include <math.h>
#include <stdint.h>

#define LANES 8

static void clenshaw_plain(const double* A, const double* B, const double* C,
                           const double* coeffs, int64_t nloc, const double* th,
                           double* out, int64_t w) {
  double x[LANES], u1[LANES], u2[LANES];
  for (int64_t l = 0; l < w; ++l) {
    x[l] = cos(th[l]);
    u1[l] = 0.0;
    u2[l] = 0.0;
  }
  for (int64_t n = nloc; n >= 0; --n) {
    const double an = A[n], bn = B[n], cn1 = C[n + 1], fn = coeffs[n];
    for (int64_t l = 0; l < w; ++l) {
      const double u0 = (an * x[l] + bn) * u1[l] - cn1 * u2[l] + fn;
      u2[l] = u1[l];
      u1[l] = u0;
    }
  }
  for (int64_t l = 0; l < w; ++l) out[l] = u1[l];
}

static void clenshaw_reinsch(const double* A, const double* C, const double* rb,
                             const double* rbi, const double* coeffs, int64_t nloc,
                             const double* th, int plus_end, double* out, int64_t w) {
  double xm[LANES], u[LANES], d[LANES];
  for (int64_t l = 0; l < w; ++l) {
    if (plus_end) {
      const double h = sin(0.5 * th[l]);
      xm[l] = -2.0 * h * h;
    } else {
      const double h = cos(0.5 * th[l]);
      xm[l] = 2.0 * h * h;
    }
    u[l] = 0.0;
    d[l] = 0.0;
  }
  for (int64_t n = nloc; n > 0; --n) {
    const double an = A[n], cn1 = C[n + 1], fn = coeffs[n], rn = rb[n], rin = rbi[n];
    for (int64_t l = 0; l < w; ++l) {
      d[l] = (an * xm[l] * u[l] + cn1 * d[l] + fn) * rn;
      u[l] = (u[l] + d[l]) * rin;
    }
  }
  for (int64_t l = 0; l < w; ++l) out[l] = A[0] * xm[l] * u[l] + C[1] * d[l] + coeffs[0];
}

void oracle_clenshaw_points(const double* A, const double* B, const double* C,
                            const double* rbp, const double* rbm, const double* rbpi,
                            const double* rbmi, const double* coeffs, const double* thetas,
                            const int64_t* cuts, const int8_t* regions, double* out,
                            int64_t npts) {
  int64_t start = 0;
  while (start < npts) {
    const int64_t nc = cuts[start];
    const int8_t reg = regions[start];
    int64_t stop = start + 1;
    while (stop < npts && cuts[stop] == nc && regions[stop] == reg) ++stop;
    if (nc <= 0) {
      for (int64_t i = start; i < stop; ++i) out[i] = 0.0;
    } else {
      for (int64_t base = start; base < stop; base += LANES) {
        const int64_t w = (stop - base > LANES) ? LANES : stop - base;
        if (reg == 0)
          clenshaw_plain(A, B, C, coeffs, nc - 1, thetas + base, out + base, w);
        else if (reg == 1)
          clenshaw_reinsch(A, C, rbp, rbpi, coeffs, nc - 1, thetas + base, 1, out + base, w);
        else
          clenshaw_reinsch(A, C, rbm, rbmi, coeffs, nc - 1, thetas + base, 0, out + base, w);
      }
    }
    start = stop;
  }
}

static void accumulate_plain(const double* A, const double* B, const double* C,
                             const double* wv, int64_t nc, const double* th, double* out,
                             int64_t w) {
  double x[LANES], pp[LANES], pc[LANES];
  for (int64_t l = 0; l < w; ++l) {
    x[l] = cos(th[l]);
    pp[l] = 0.0;
    pc[l] = 1.0;
    out[0] += wv[l];
  }
  for (int64_t n = 1; n < nc; ++n) {
    const double an = A[n - 1], bn = B[n - 1], cn = C[n - 1];
    double acc = 0.0;
    for (int64_t l = 0; l < w; ++l) {
      const double pn = (an * x[l] + bn) * pc[l] - cn * pp[l];
      pp[l] = pc[l];
      pc[l] = pn;
      acc += wv[l] * pn;
    }
    out[n] += acc;
  }
}

static void accumulate_reinsch(const double* A, const double* C, const double* rf,
                               const double* rfi, const double* wv, int64_t nc,
                               const double* th, int plus_end, double* out, int64_t w) {
  double xm[LANES], pc[LANES], d[LANES];
  for (int64_t l = 0; l < w; ++l) {
    if (plus_end) {
      const double h = sin(0.5 * th[l]);
      xm[l] = -2.0 * h * h;
    } else {
      const double h = cos(0.5 * th[l]);
      xm[l] = 2.0 * h * h;
    }
    pc[l] = 1.0;
    d[l] = 0.0;
    out[0] += wv[l];
  }
  for (int64_t n = 0; n < nc - 1; ++n) {
    const double an = A[n], cn = C[n], rn = rf[n], rin = rfi[n];
    double acc = 0.0;
    for (int64_t l = 0; l < w; ++l) {
      d[l] = (an * xm[l] * pc[l] + cn * d[l]) * rin;
      pc[l] = (pc[l] + d[l]) * rn;
      acc += wv[l] * pc[l];
    }
    out[n + 1] += acc;
  }
}

void oracle_transpose_accumulate(const double* A, const double* B, const double* C,
                                 const double* rfp, const double* rfm, const double* rfpi,
                                 const double* rfmi, const double* wv, const double* thetas,
                                 const int64_t* cuts, const int8_t* regions, double* out,
                                 int64_t npts) {
  int64_t start = 0;
  while (start < npts) {
    const int64_t nc = cuts[start];
    const int8_t reg = regions[start];
    int64_t stop = start + 1;
    while (stop < npts && cuts[stop] == nc && regions[stop] == reg) ++stop;
    if (nc > 0) {
      for (int64_t base = start; base < stop; base += LANES) {
        const int64_t w = (stop - base > LANES) ? LANES : stop - base;
        if (reg == 0)
          accumulate_plain(A, B, C, wv + base, nc, thetas + base, out, w);
        else if (reg == 1)
          accumulate_reinsch(A, C, rfp, rfpi, wv + base, nc, thetas + base, 1, out, w);
        else
          accumulate_reinsch(A, C, rfm, rfmi, wv + base, nc, thetas + base, 0, out, w);
      }
    }
    start = stop;
  }
}
