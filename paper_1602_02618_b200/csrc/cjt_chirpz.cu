// Batched chirp-z (Bluestein) transforms with fused diagonal scalings.
//
// Every DCT-I / bordered DST-I of the reference execution (engine.py:163-227,
// trig.py:35-63) is one real part of
//     z_q = sum_p exp(i pi p q / G) pre_m[p] x[p],   out[q] (+)= sum_m Re(post_m[q] z_q),
// evaluated as chirp * (cyclic convolution of length L = 2^k) * chirp.  The
// chirps and the diagonals (C_{n,m}, u_m - i v_m, CC weights, 2/G) are folded
// into the per-plan complex tables pre/post (planner.py: chirpz), so one kernel
// shape serves blocks, analysis and synthesis.
//
//   L <= 8192: one fused kernel per batch of vectors; FFT, spectrum product and
//              inverse FFT stay in shared memory (no HBM traffic besides the
//              real input slice and the real output slice).
//   L >  8192: three passes of a four-step FFT (L = L1 x L2): column FFTs with
//              the input diagonal fused into the load and the inter-step
//              twiddle into the store; row FFT -> spectrum product -> row
//              inverse FFT fused in one pass; column inverse FFTs with the
//              output diagonal and the sum over m fused into the store.
#include "cjt_internal.cuh"

namespace cjt {

namespace {

template <int LOGL>
struct FusedCfg {
  static constexpr int L = 1 << LOGL;
  static constexpr int E = (L >= 4096) ? L : 4096;  // complex elements per CTA
  static constexpr int NG = E / L;                  // vectors per CTA
  static constexpr int T = E / 16;                  // threads per CTA
  static constexpr int SMEM = NG * padded_len(L) * 16;
};

template <int LOGL>
__global__ void __launch_bounds__(FusedCfg<LOGL>::T)
    k_chirpz_fused(ChirpZDev cz, const double2* __restrict__ tw, const double* __restrict__ x,
                   int64_t ldx, double* __restrict__ out, int64_t ldo, int64_t batch) {
  using Cfg = FusedCfg<LOGL>;
  constexpr int L = Cfg::L;
  constexpr int TPG = L / 16;
  extern __shared__ double2 smem[];
  const int grp = threadIdx.x / TPG;
  const int t = threadIdx.x % TPG;
  const int64_t b = (int64_t)blockIdx.x * Cfg::NG + grp;
  const bool valid = b < batch;
  double2* s = smem + grp * padded_len(L);
  const double* xb = x + (valid ? b : 0) * ldx + cz.p0;

  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;

  for (int m = 0; m < cz.m_count; ++m) {
    const double2* pre = cz.pre + (int64_t)m * cz.width;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = t + i * TPG;
      double2 v = make_double2(0.0, 0.0);
      if (valid && e < cz.width) {
        const double xv = __ldg(xb + e);
        const double2 p = __ldg(pre + e);
        v = make_double2(xv * p.x, xv * p.y);
      }
      s[pad16(e)] = v;
    }
    __syncthreads();
    fft_smem<LOGL, -1>(s, t, tw);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = t + i * TPG;
      s[pad16(e)] = cmul(s[pad16(e)], __ldg(cz.khat + e));
    }
    __syncthreads();
    fft_smem<LOGL, +1>(s, t, tw);
    const double2* post = cz.post + (int64_t)m * cz.count;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = t + i * TPG;
      if (e < cz.count) {
        const double2 y = s[pad16(e)];
        const double2 q = __ldg(post + e);
        acc[i] += fma(q.x, y.x, -q.y * y.y);
      }
    }
    __syncthreads();
  }
  if (!valid) return;
  double* ob = out + b * ldo + cz.q0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = t + i * TPG;
    if (e < cz.count) ob[e] = cz.accumulate ? ob[e] + acc[i] : acc[i];
  }
}

// W_L^t = exp(-2 pi i t / L) from the two-level table (t < L)
__device__ __forceinline__ double2 twiddle_L(const ChirpZDev& cz, int64_t t) {
  return cmul(__ldg(cz.tw_hi + (t >> 12)), __ldg(cz.tw_lo + (t & 4095)));
}

template <int LOG1>
struct ColCfg {
  static constexpr int L1 = 1 << LOG1;
  static constexpr int E = (L1 >= 4096) ? L1 : 4096;
  static constexpr int NC = E / L1;                  // columns per CTA
  static constexpr int T = E / 16;
  static constexpr int CS = padded_len(L1) + 1;      // odd column stride (conflict-free transpose)
  static constexpr int SMEM = NC * CS * 16;
};

// pass 1: x (real slice) * pre_m -> column FFTs over n1 -> * W_L^{n2 k1} -> buf[b][m][k1][n2]
template <int LOG1>
__global__ void __launch_bounds__(ColCfg<LOG1>::T)
    k_chirpz_cols_fwd(ChirpZDev cz, const double2* __restrict__ tw, const double* __restrict__ x,
                      int64_t ldx, double2* __restrict__ buf) {
  using Cfg = ColCfg<LOG1>;
  constexpr int L1 = Cfg::L1, NC = Cfg::NC, T = Cfg::T, CS = Cfg::CS;
  extern __shared__ double2 smem[];
  const int64_t L2 = (int64_t)1 << cz.log2;
  const int64_t L = cz.length;
  const int64_t c0 = (int64_t)blockIdx.x * NC;
  const int64_t b = blockIdx.y;
  const double* xb = x + b * ldx + cz.p0;
  const int grp = threadIdx.x / (L1 / 16);
  const int t = threadIdx.x % (L1 / 16);
  for (int m = 0; m < cz.m_count; ++m) {
    const double2* pre = cz.pre + (int64_t)m * cz.width;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int idx = threadIdx.x + i * T;
      const int c = idx % NC, n1 = idx / NC;
      const int64_t pidx = (int64_t)n1 * L2 + c0 + c;
      double2 v = make_double2(0.0, 0.0);
      if (pidx < cz.width) {
        const double xv = __ldg(xb + pidx);
        const double2 p = __ldg(pre + pidx);
        v = make_double2(xv * p.x, xv * p.y);
      }
      smem[c * CS + pad16(n1)] = v;
    }
    __syncthreads();
    fft_smem<LOG1, -1>(smem + grp * CS, t, tw);
    double2* bm = buf + (b * cz.m_count + m) * L;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int idx = threadIdx.x + i * T;
      const int c = idx % NC, k1 = idx / NC;
      const int64_t n2 = c0 + c;
      bm[(int64_t)k1 * L2 + n2] = cmul(smem[c * CS + pad16(k1)], twiddle_L(cz, n2 * k1));
    }
    __syncthreads();
  }
}

template <int LOG2>
struct RowCfg {
  static constexpr int L2 = 1 << LOG2;
  static constexpr int E = (L2 >= 4096) ? L2 : 4096;
  static constexpr int NR = E / L2;
  static constexpr int T = E / 16;
  static constexpr int SMEM = NR * padded_len(L2) * 16;
};

// pass 2: rows k1 of buf: FFT over n2 -> * khat[k1][k2] -> inverse FFT over k2
template <int LOG2>
__global__ void __launch_bounds__(RowCfg<LOG2>::T)
    k_chirpz_rows(ChirpZDev cz, const double2* __restrict__ tw, double2* __restrict__ buf) {
  using Cfg = RowCfg<LOG2>;
  constexpr int L2 = Cfg::L2, NR = Cfg::NR;
  constexpr int TPG = L2 / 16;
  extern __shared__ double2 smem[];
  const int grp = threadIdx.x / TPG;
  const int t = threadIdx.x % TPG;
  const int64_t k1 = (int64_t)blockIdx.x * NR + grp;
  const int64_t L = cz.length;
  double2* row = buf + (int64_t)blockIdx.y * L + k1 * L2;
  const double2* kh = cz.khat + k1 * L2;
  double2* s = smem + grp * padded_len(L2);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = t + i * TPG;
    s[pad16(e)] = row[e];
  }
  __syncthreads();
  fft_smem<LOG2, -1>(s, t, tw);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = t + i * TPG;
    s[pad16(e)] = cmul(s[pad16(e)], __ldg(kh + e));
  }
  __syncthreads();
  fft_smem<LOG2, +1>(s, t, tw);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = t + i * TPG;
    row[e] = s[pad16(e)];
  }
}

// pass 3: columns n2: * W_L^{-n2 k1} -> inverse FFT over k1 -> sum_m Re(post_m * y) -> out
template <int LOG1>
__global__ void __launch_bounds__(ColCfg<LOG1>::T)
    k_chirpz_cols_inv(ChirpZDev cz, const double2* __restrict__ tw,
                      const double2* __restrict__ buf, double* __restrict__ out, int64_t ldo) {
  using Cfg = ColCfg<LOG1>;
  constexpr int L1 = Cfg::L1, NC = Cfg::NC, T = Cfg::T, CS = Cfg::CS;
  extern __shared__ double2 smem[];
  const int64_t L2 = (int64_t)1 << cz.log2;
  const int64_t L = cz.length;
  const int64_t c0 = (int64_t)blockIdx.x * NC;
  const int64_t b = blockIdx.y;
  const int grp = threadIdx.x / (L1 / 16);
  const int t = threadIdx.x % (L1 / 16);
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int m = 0; m < cz.m_count; ++m) {
    const double2* bm = buf + (b * cz.m_count + m) * L;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int idx = threadIdx.x + i * T;
      const int c = idx % NC, k1 = idx / NC;
      const int64_t n2 = c0 + c;
      double2 w = twiddle_L(cz, n2 * k1);
      w.y = -w.y;
      smem[c * CS + pad16(k1)] = cmul(bm[(int64_t)k1 * L2 + n2], w);
    }
    __syncthreads();
    fft_smem<LOG1, +1>(smem + grp * CS, t, tw);
    const double2* post = cz.post + (int64_t)m * cz.count;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int idx = threadIdx.x + i * T;
      const int c = idx % NC, n1 = idx / NC;
      const int64_t sidx = (int64_t)n1 * L2 + c0 + c;
      if (sidx < cz.count) {
        const double2 y = smem[c * CS + pad16(n1)];
        const double2 q = __ldg(post + sidx);
        acc[i] += fma(q.x, y.x, -q.y * y.y);
      }
    }
    __syncthreads();
  }
  double* ob = out + b * ldo + cz.q0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int idx = threadIdx.x + i * T;
    const int c = idx % NC, n1 = idx / NC;
    const int64_t sidx = (int64_t)n1 * L2 + c0 + c;
    if (sidx < cz.count) ob[sidx] = cz.accumulate ? ob[sidx] + acc[i] : acc[i];
  }
}

template <typename K>
int set_smem(K kernel, int bytes) {
  static_assert(sizeof(K) > 0, "");
  CJT_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return CJT_OK;
}

template <int LOGL>
int run_fused(const ChirpZDev& cz, const double2* tw, const double* x, int64_t ldx, double* out,
              int64_t ldo, int64_t batch, cudaStream_t st) {
  using Cfg = FusedCfg<LOGL>;
  static bool init = false;
  if (!init) {
    if (int rc = set_smem(k_chirpz_fused<LOGL>, Cfg::SMEM)) return rc;
    init = true;
  }
  dim3 grid((unsigned)((batch + Cfg::NG - 1) / Cfg::NG));
  k_chirpz_fused<LOGL><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, x, ldx, out, ldo, batch);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

template <int LOG1>
int run_cols_fwd(const ChirpZDev& cz, const double2* tw, const double* x, int64_t ldx,
                 double2* buf, int64_t batch, cudaStream_t st) {
  using Cfg = ColCfg<LOG1>;
  static bool init = false;
  if (!init) {
    if (int rc = set_smem(k_chirpz_cols_fwd<LOG1>, Cfg::SMEM)) return rc;
    init = true;
  }
  const int64_t L2 = (int64_t)1 << cz.log2;
  dim3 grid((unsigned)(L2 / Cfg::NC), (unsigned)batch);
  k_chirpz_cols_fwd<LOG1><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, x, ldx, buf);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

template <int LOG2>
int run_rows(const ChirpZDev& cz, const double2* tw, double2* buf, int64_t batch, cudaStream_t st) {
  using Cfg = RowCfg<LOG2>;
  static bool init = false;
  if (!init) {
    if (int rc = set_smem(k_chirpz_rows<LOG2>, Cfg::SMEM)) return rc;
    init = true;
  }
  const int64_t L1 = (int64_t)1 << cz.log1;
  dim3 grid((unsigned)(L1 / Cfg::NR), (unsigned)(batch * cz.m_count));
  k_chirpz_rows<LOG2><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, buf);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

template <int LOG1>
int run_cols_inv(const ChirpZDev& cz, const double2* tw, const double2* buf, double* out,
                 int64_t ldo, int64_t batch, cudaStream_t st) {
  using Cfg = ColCfg<LOG1>;
  static bool init = false;
  if (!init) {
    if (int rc = set_smem(k_chirpz_cols_inv<LOG1>, Cfg::SMEM)) return rc;
    init = true;
  }
  const int64_t L2 = (int64_t)1 << cz.log2;
  dim3 grid((unsigned)(L2 / Cfg::NC), (unsigned)batch);
  k_chirpz_cols_inv<LOG1><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, buf, out, ldo);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

}  // namespace

int launch_chirpz(const ChirpZDev& cz, const double2* tw8192, const double* x, int64_t ldx,
                  double* out, int64_t ldo, int64_t batch, double2* scratch, cudaStream_t st,
                  int* launches) {
  if (batch <= 0) return CJT_OK;
  const int lg = cz.log2len;
  if (lg <= 13) {
    *launches += 1;
    switch (lg) {
      case 4: return run_fused<4>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 5: return run_fused<5>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 6: return run_fused<6>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 7: return run_fused<7>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 8: return run_fused<8>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 9: return run_fused<9>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 10: return run_fused<10>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 11: return run_fused<11>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 12: return run_fused<12>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 13: return run_fused<13>(cz, tw8192, x, ldx, out, ldo, batch, st);
      default: return fail(CJT_EINVAL, "chirp-z length below 16");
    }
  }
  *launches += 3;
  int rc = CJT_OK;
  switch (cz.log1) {
#define CJT_COLF(K) case K: rc = run_cols_fwd<K>(cz, tw8192, x, ldx, scratch, batch, st); break;
    CJT_COLF(7) CJT_COLF(8) CJT_COLF(9) CJT_COLF(10) CJT_COLF(11) CJT_COLF(12) CJT_COLF(13)
#undef CJT_COLF
    default: return fail(CJT_EINVAL, "chirp-z column length out of range");
  }
  if (rc) return rc;
  switch (cz.log2) {
#define CJT_ROW(K) case K: rc = run_rows<K>(cz, tw8192, scratch, batch, st); break;
    CJT_ROW(7) CJT_ROW(8) CJT_ROW(9) CJT_ROW(10) CJT_ROW(11) CJT_ROW(12) CJT_ROW(13)
#undef CJT_ROW
    default: return fail(CJT_EINVAL, "chirp-z row length out of range");
  }
  if (rc) return rc;
  switch (cz.log1) {
#define CJT_COLI(K) case K: rc = run_cols_inv<K>(cz, tw8192, scratch, out, ldo, batch, st); break;
    CJT_COLI(7) CJT_COLI(8) CJT_COLI(9) CJT_COLI(10) CJT_COLI(11) CJT_COLI(12) CJT_COLI(13)
#undef CJT_COLI
    default: return fail(CJT_EINVAL, "chirp-z column length out of range");
  }
  return rc;
}

}  // namespace cjt
