// Integer parameter shifts of Jacobi coefficient vectors (engine.py:232-292):
// increment_beta / decrement_beta and their alpha versions, conjugated by the
// parity map c_n -> (-1)^n c_n with alpha <-> beta (engine.py:270-286).
//
// * increments are the bidiagonal product, one thread per coefficient, in the
//   reference's operation order (NumPy, engine.py:243-248) -> bit-identical;
// * decrements are the bidiagonal back-substitution (engine.py:258-267), a
//   first-order linear recurrence run from the top degree down.  One CTA per
//   vector: each thread composes the affine map x_i = p_i + q_i x_{i+1} over
//   its contiguous chunk, one thread chains the chunk boundaries, then every
//   chunk is re-run with the reference's exact formula from its (chained)
//   top value.  Only the chunk-boundary values carry the composition's
//   rounding.
#include "cjt_internal.cuh"

namespace cjt {
namespace {

// diag_k = (a + b + k + 1) / (a + b + 2k + 1), diag_0 = 1; same rounding as
// NumPy's left-to-right evaluation of `a + b + k + 1.0` with scalar a, b
__device__ __forceinline__ double shift_diag(double ab, int64_t k) {
  if (k == 0) return 1.0;
  const double kd = (double)k;
  return __ddiv_rn(__dadd_rn(__dadd_rn(ab, kd), 1.0), __dadd_rn(__dadd_rn(ab, __dmul_rn(2.0, kd)), 1.0));
}
// (a + k + 1) / (a + b + 2k + 3)
__device__ __forceinline__ double shift_upper_num(double a, int64_t k) {
  return __dadd_rn(__dadd_rn(a, (double)k), 1.0);
}
__device__ __forceinline__ double shift_upper_den(double ab, int64_t k) {
  return __dadd_rn(__dadd_rn(ab, __dmul_rn(2.0, (double)k)), 3.0);
}

// out = B(a, b) in: out_k = diag_k d_k + d_{k+1} (a+k+1) / (a+b+2k+3);
// FLIP: d_k = (-1)^k in_k and out_k (-1)^k (the alpha shift)
template <bool FLIP>
__global__ void k_shift_inc(const double* __restrict__ in, double* __restrict__ out, int64_t n,
                            int64_t batch, double a, double b) {
  const int64_t n1 = n + 1;
  const int64_t total = n1 * batch;
  const double ab = __dadd_rn(a, b);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = idx % n1;
    double dk = in[idx];
    if (FLIP && (k & 1)) dk = -dk;
    double r = __dmul_rn(shift_diag(ab, k), dk);
    if (k < n) {
      double dn = in[idx + 1];
      if (FLIP && ((k + 1) & 1)) dn = -dn;
      r = __dadd_rn(r, __ddiv_rn(__dmul_rn(dn, shift_upper_num(a, k)), shift_upper_den(ab, k)));
    }
    out[idx] = (FLIP && (k & 1)) ? -r : r;
  }
}

constexpr int DEC_T = 256;

// back-substitution out_n = d_n / diag_n, out_i = (d_i - upper_i out_{i+1}) / diag_i
// for the TARGET parameters (a, b); one CTA per vector
template <bool FLIP>
__global__ void __launch_bounds__(DEC_T) k_shift_dec(const double* __restrict__ in,
                                                     double* __restrict__ out, int64_t n, double a,
                                                     double b) {
  __shared__ double Ps[DEC_T], Qs[DEC_T], Xs[DEC_T + 1];
  const int64_t n1 = n + 1;
  const double* d = in + (int64_t)blockIdx.x * n1;
  double* o = out + (int64_t)blockIdx.x * n1;
  const double ab = __dadd_rn(a, b);
  const int t = threadIdx.x;
  const int64_t chunk = (n1 + DEC_T - 1) / DEC_T;
  const int64_t i0 = min(n1, t * chunk), i1 = min(n1, i0 + chunk);
  auto dval = [&](int64_t i) {
    const double v = d[i];
    return (FLIP && (i & 1)) ? -v : v;
  };
  // phase 1: x_{i0} = P + Q x_{i1} over this chunk (x_{n+1} := 0)
  double P = 0.0, Q = 1.0;
  for (int64_t i = i1 - 1; i >= i0; --i) {
    const double g = shift_diag(ab, i);
    const double u = __ddiv_rn(shift_upper_num(a, i), shift_upper_den(ab, i));
    const double p = dval(i) / g, q = -u / g;
    P = fma(q, P, p);
    Q = q * Q;
  }
  Ps[t] = P;
  Qs[t] = Q;
  __syncthreads();
  // phase 2: chunk tops from the last chunk down
  if (t == 0) {
    double x = 0.0;
    Xs[DEC_T] = 0.0;
    for (int c = DEC_T - 1; c >= 0; --c) {
      Xs[c + 1] = x;   // value just above chunk c
      x = fma(Qs[c], x, Ps[c]);
    }
  }
  __syncthreads();
  // phase 3: the reference's recurrence over the chunk from its top value
  double x = Xs[t + 1];
  for (int64_t i = i1 - 1; i >= i0; --i) {
    const double g = shift_diag(ab, i);
    const double u = __ddiv_rn(shift_upper_num(a, i), shift_upper_den(ab, i));
    // top degree: out_n = d_n / diag_n exactly (x = 0 there)
    x = (i == n) ? __ddiv_rn(dval(i), g) : __ddiv_rn(__dsub_rn(dval(i), __dmul_rn(u, x)), g);
    o[i] = (FLIP && (i & 1)) ? -x : x;
  }
}

}  // namespace

int launch_shift(int op, double alpha, double beta, const double* in, double* out, int64_t n,
                 int64_t batch, cudaStream_t st) {
  if (batch <= 0) return CJT_OK;
  const int64_t total = (n + 1) * batch;
  const int T = 256;
  const unsigned grid = (unsigned)std::min<int64_t>((total + T - 1) / T, 148 * 32);
  switch (op) {
    case CJT_SHIFT_INC_BETA:
      k_shift_inc<false><<<grid, T, 0, st>>>(in, out, n, batch, alpha, beta);
      break;
    case CJT_SHIFT_INC_ALPHA:   // parity-conjugated beta shift with (beta, alpha)
      k_shift_inc<true><<<grid, T, 0, st>>>(in, out, n, batch, beta, alpha);
      break;
    case CJT_SHIFT_DEC_BETA:    // target (alpha, beta - 1)
      k_shift_dec<false><<<(unsigned)batch, DEC_T, 0, st>>>(in, out, n, alpha, beta - 1.0);
      break;
    case CJT_SHIFT_DEC_ALPHA:   // target of the swapped system: (beta, alpha - 1)
      k_shift_dec<true><<<(unsigned)batch, DEC_T, 0, st>>>(in, out, n, beta, alpha - 1.0);
      break;
    default:
      return fail(CJT_EINVAL, "unknown shift operation");
  }
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

}  // namespace cjt
