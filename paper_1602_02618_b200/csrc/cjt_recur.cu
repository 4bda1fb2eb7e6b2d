// Recurrence region of the transform: the rows/degrees of the (degree x angle)
// plane that the certified asymptotic blocks do not cover.
//
// Reference: clenshaw_points / transpose_accumulate (_kernels_cy.pyx:17-237,
// _kernels_np.py:22-97).  The reference evaluates every (row, vector) pair with
// its own Clenshaw-Smith chain (forward) or forward recurrence (inverse).  Here
// P_n(x_i) does not depend on the vector, so both directions become contractions
// with a *generated* operand:
//
//   forward  values[b, i] = sum_{n < cut_i} P_n(x_i) c[b, n]          (K1)
//   inverse  out[b, n]    = sum_{i : n < cut_i} P_n(x_i) wv[b, i]     (K2)
//
// P_n(x_i) is produced on the fly by the reference's forward recurrences
// (plain three-term in the interior, Reinsch-modified with the endpoint
// ratios near x = +-1, _kernels_cy.pyx:125-198), with every multiply/add
// rounded exactly as the reference (no FMA contraction), so the generated
// values are bit-identical to the reference's inverse kernel.  Long rows are
// split into degree segments that restart from per-plan checkpoints of the
// recurrence state (every CK degrees), which keeps the values bit-identical
// while exposing parallelism; partial sums are reduced in a fixed order
// (deterministic, no atomics).
#include "cjt_internal.cuh"

namespace cjt {

namespace {

// state at degree n: plain (P_{n-1}, P_n), Reinsch (pi_n, d_n)
__device__ __forceinline__ void rec_init(int reg, double& s0, double& s1) {
  if (reg == 0) {
    s0 = 0.0;
    s1 = 1.0;
  } else {
    s0 = 1.0;
    s1 = 0.0;
  }
}
__device__ __forceinline__ double rec_value(int reg, double s0, double s1) {
  return reg == 0 ? s1 : s0;
}
// degree n -> n+1 (reference arithmetic, _kernels_cy.pyx:144-147, 186-188)
__device__ __forceinline__ void rec_step(int reg, double x, double xm, const RecTablesDev& t,
                                         int64_t n, double& s0, double& s1) {
  const double a = __ldg(t.A + n);
  const double c = __ldg(t.C + n);
  if (reg == 0) {
    const double bb = __ldg(t.B + n);
    const double pn = __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(a, x), bb), s1), __dmul_rn(c, s0));
    s0 = s1;
    s1 = pn;
  } else {
    const double rf = __ldg((reg > 0 ? t.rfp : t.rfm) + n);
    const double rfi = __ldg((reg > 0 ? t.rfpi : t.rfmi) + n);
    const double d = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, xm), s0), __dmul_rn(c, s1)), rfi);
    s0 = __dmul_rn(__dadd_rn(s0, d), rf);
    s1 = d;
  }
}

__device__ __forceinline__ void load_state(const RecRowsDev& rows, const int64_t* ck_off,
                                           const double2* ck, int64_t i, int64_t n0, int reg,
                                           double& s0, double& s1) {
  if (n0 == 0) {
    rec_init(reg, s0, s1);
  } else {
    const double2 st = ck[ck_off[i] + n0 / CK - 1];
    s0 = st.x;
    s1 = st.y;
  }
}

__global__ void k_checkpoints(RecRowsDev rows, RecTablesDev tab, const int64_t* __restrict__ ck_off,
                              double2* __restrict__ ck) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows.nrows) return;
  const int reg = rows.reg[i];
  const double x = rows.x[i], xm = rows.xm[i];
  const int64_t nc = rows.cut[i];
  double s0, s1;
  rec_init(reg, s0, s1);
  double2* out = ck + ck_off[i];
  for (int64_t n = 0; n + 1 < nc; ++n) {
    rec_step(reg, x, xm, tab, n, s0, s1);
    if (((n + 1) % CK) == 0) out[(n + 1) / CK - 1] = make_double2(s0, s1);
  }
}

// K1: one lane per grid row, FWD_VT vectors per lane, coefficients staged in
// shared memory and read as warp-wide broadcasts.
__global__ void __launch_bounds__(FWD_ROWS)
    k_rec_forward(RecRowsDev rows, RecTablesDev tab, const int64_t* __restrict__ ck_off,
                  const double2* __restrict__ ck, const FwdItem* __restrict__ items,
                  const double* __restrict__ c, int64_t ldc, int64_t ncoef, int64_t batch,
                  double* __restrict__ part) {
  __shared__ __align__(16) double cs[FWD_CH][FWD_VT];
  const FwdItem it = items[blockIdx.x];
  const int64_t b0 = (int64_t)blockIdx.y * FWD_VT;
  const int lr = threadIdx.x;
  const int64_t i = it.row0 + lr;
  const bool live = lr < it.nrows;
  int reg = 0;
  double x = 0.0, xm = 0.0;
  int64_t cut = 0;
  if (live) {
    reg = rows.reg[i];
    x = rows.x[i];
    xm = rows.xm[i];
    cut = rows.cut[i];
  }
  double s0 = 0.0, s1 = 0.0;
  if (live && cut > it.n_begin) load_state(rows, ck_off, ck, i, it.n_begin, reg, s0, s1);
  double acc[FWD_VT];
#pragma unroll
  for (int v = 0; v < FWD_VT; ++v) acc[v] = 0.0;

  for (int64_t n0 = it.n_begin; n0 < it.n_end; n0 += FWD_CH) {
    // stage c[b0 .. b0+VT)[n0 .. n0+CH) transposed: cs[k][v]
#pragma unroll
    for (int q = 0; q < (FWD_CH * FWD_VT) / FWD_ROWS; ++q) {
      const int idx = threadIdx.x + q * FWD_ROWS;
      const int k = idx % FWD_CH, v = idx / FWD_CH;
      const int64_t bb = b0 + v, n = n0 + k;
      cs[k][v] = (bb < batch && n < ncoef) ? __ldg(c + bb * ldc + n) : 0.0;
    }
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < FWD_CH; ++k) {
      const int64_t n = n0 + k;
      const double p = (n < cut) ? rec_value(reg, s0, s1) : 0.0;
      const double2* row = reinterpret_cast<const double2*>(&cs[k][0]);
#pragma unroll
      for (int v = 0; v < FWD_VT / 2; ++v) {
        const double2 cv = row[v];
        acc[2 * v] = fma(p, cv.x, acc[2 * v]);
        acc[2 * v + 1] = fma(p, cv.y, acc[2 * v + 1]);
      }
      if (n + 1 < cut) rec_step(reg, x, xm, tab, n, s0, s1);
    }
    __syncthreads();
  }
  if (!live) return;
  double* dst = part + (int64_t)it.slot * batch * FWD_ROWS;
#pragma unroll
  for (int v = 0; v < FWD_VT; ++v) {
    const int64_t bb = b0 + v;
    if (bb < batch) dst[bb * FWD_ROWS + lr] = acc[v];
  }
}

__global__ void k_rec_forward_reduce(const int32_t* __restrict__ tile_slot0,
                                     const int32_t* __restrict__ tile_nslot, int64_t nrows,
                                     const double* __restrict__ part, double* __restrict__ vals,
                                     int64_t ldv, int64_t batch) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (i >= nrows) return;
  const int64_t tile = i / FWD_ROWS, lr = i % FWD_ROWS;
  const int32_t s0 = tile_slot0[tile], ns = tile_nslot[tile];
  double acc = 0.0;
  for (int s = 0; s < ns; ++s) acc += part[((int64_t)(s0 + s) * batch + b) * FWD_ROWS + lr];
  vals[b * ldv + i] = acc;
}

// K2: degrees x vectors output tile, reduction over grid rows; P tiles are
// generated into shared memory (two threads per row, CK degrees each) and
// contracted with the staged wv tile.  16-byte chunks are XOR-swizzled by
// row so the row-strided staging stores and the GEMM's 128-bit loads are both
// nearly conflict-free.
__device__ __forceinline__ int swz(int row, int col) {  // col in doubles, 64 per row
  return row * 64 + ((((col >> 1) ^ (row & 7))) << 1) + (col & 1);
}

__global__ void __launch_bounds__(256)
    k_rec_inverse(RecRowsDev rows, RecTablesDev tab, const int64_t* __restrict__ ck_off,
                  const double2* __restrict__ ck, const InvItem* __restrict__ items,
                  const int32_t* __restrict__ tile_ids, const double* __restrict__ wv,
                  int64_t ldw, int64_t batch, double* __restrict__ part) {
  extern __shared__ __align__(16) double sm_inv[];
  double* Ps = sm_inv;                      // [INV_RT][64] P_n(x_i), swizzled
  double* Ws = sm_inv + INV_RT * 64;        // [INV_RT][64] wv, swizzled
  const InvItem it = items[blockIdx.x];
  const int64_t b0 = (int64_t)blockIdx.y * INV_VT;
  const int tid = threadIdx.x;
  const int td = tid >> 4, tv = tid & 15;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q] = 0.0;

  for (int tt = 0; tt < it.t_count; ++tt) {
    const int64_t r0 = (int64_t)tile_ids[it.t_begin + tt] * INV_RT;
    // generate P for rows r0 + (tid & 127), degrees n0 + 32*(tid >> 7) .. +32
    {
      const int lr = tid & (INV_RT - 1);
      const int half = tid >> 7;
      const int64_t i = r0 + lr;
      const int64_t nstart = it.n0 + half * CK;
      int64_t cut = 0;
      int reg = 0;
      double x = 0.0, xm = 0.0, s0 = 0.0, s1 = 0.0;
      if (i < rows.nrows) {
        cut = rows.cut[i];
        reg = rows.reg[i];
        x = rows.x[i];
        xm = rows.xm[i];
        if (cut > nstart) load_state(rows, ck_off, ck, i, nstart, reg, s0, s1);
      }
#pragma unroll 4
      for (int k = 0; k < CK; ++k) {
        const int64_t n = nstart + k;
        Ps[swz(lr, half * CK + k)] = (n < cut) ? rec_value(reg, s0, s1) : 0.0;
        if (n + 1 < cut) rec_step(reg, x, xm, tab, n, s0, s1);
      }
    }
    // stage wv[b0 + v][r0 + row] -> Ws[row][v]
#pragma unroll 4
    for (int q = 0; q < (INV_RT * INV_VT) / 256; ++q) {
      const int idx = tid + q * 256;
      const int row = idx % INV_RT, v = idx / INV_RT;
      const int64_t bb = b0 + v, i = r0 + row;
      Ws[swz(row, v)] = (bb < batch && i < rows.nrows) ? __ldg(wv + bb * ldw + i) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int row = 0; row < INV_RT; ++row) {
      const int sw = row & 7;
      const double2 p01 = *reinterpret_cast<const double2*>(&Ps[row * 64 + (((2 * td) ^ sw) << 1)]);
      const double2 p23 = *reinterpret_cast<const double2*>(&Ps[row * 64 + (((2 * td + 1) ^ sw) << 1)]);
      const double2 w01 = *reinterpret_cast<const double2*>(&Ws[row * 64 + (((2 * tv) ^ sw) << 1)]);
      const double2 w23 = *reinterpret_cast<const double2*>(&Ws[row * 64 + (((2 * tv + 1) ^ sw) << 1)]);
      const double pp[4] = {p01.x, p01.y, p23.x, p23.y};
      const double ww[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = fma(pp[a], ww[q], acc[a][q]);
    }
    __syncthreads();
  }
  double* dst = part + (int64_t)it.slot * batch * INV_DT;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t bb = b0 + 4 * tv + q;
    if (bb >= batch) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) dst[bb * INV_DT + 4 * td + a] = acc[a][q];
  }
}

__global__ void k_inverse_finish(const int32_t* __restrict__ dt_slot0,
                                 const int32_t* __restrict__ dt_nslot, int64_t ndeg,
                                 const double* __restrict__ part,
                                 const double* __restrict__ blocks_acc,
                                 const double* __restrict__ scal, double* __restrict__ out,
                                 int64_t ldo, int64_t batch) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (n >= ndeg) return;
  const int64_t d = n / INV_DT, k = n % INV_DT;
  const int32_t s0 = dt_slot0[d], ns = dt_nslot[d];
  double acc = blocks_acc ? blocks_acc[b * ldo + n] : 0.0;
  for (int s = 0; s < ns; ++s) acc += part[((int64_t)(s0 + s) * batch + b) * INV_DT + k];
  out[b * ldo + n] = acc * scal[n];
}

// Reference-signature Clenshaw-Smith / Reinsch evaluation, one thread per
// point, the reference's exact operation order (_kernels_cy.pyx:17-80).
__global__ void k_clenshaw_points(RecTablesDev tab, const double* __restrict__ rbp,
                                  const double* __restrict__ rbm, const double* __restrict__ rbpi,
                                  const double* __restrict__ rbmi,
                                  const double* __restrict__ coeffs, const double* __restrict__ xs,
                                  const double* __restrict__ xms, const int8_t* __restrict__ regs,
                                  const int64_t* __restrict__ cuts, double* __restrict__ out,
                                  int64_t npts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  const int64_t nc = cuts[i];
  if (nc <= 0) {
    out[i] = 0.0;
    return;
  }
  const int reg = regs[i];
  if (reg == 0) {
    const double x = xs[i];
    double u1 = 0.0, u2 = 0.0;
    for (int64_t n = nc - 1; n >= 0; --n) {
      const double t1 = __dmul_rn(__dadd_rn(__dmul_rn(tab.A[n], x), tab.B[n]), u1);
      const double u0 = __dadd_rn(__dsub_rn(t1, __dmul_rn(tab.C[n + 1], u2)), coeffs[n]);
      u2 = u1;
      u1 = u0;
    }
    out[i] = u1;
  } else {
    const double xm = xms[i];
    const double* rb = reg > 0 ? rbp : rbm;
    const double* rbi = reg > 0 ? rbpi : rbmi;
    double u = 0.0, d = 0.0;
    for (int64_t n = nc - 1; n > 0; --n) {
      const double t = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(tab.A[n], xm), u),
                                           __dmul_rn(tab.C[n + 1], d)), coeffs[n]);
      d = __dmul_rn(t, rb[n]);
      u = __dmul_rn(__dadd_rn(u, d), rbi[n]);
    }
    out[i] = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(tab.A[0], xm), u), __dmul_rn(tab.C[1], d)),
                       coeffs[0]);
  }
}

}  // namespace

int launch_checkpoints(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                       double2* ck, cudaStream_t st) {
  if (rows.nrows <= 0) return CJT_OK;
  const int T = 128;
  k_checkpoints<<<(unsigned)((rows.nrows + T - 1) / T), T, 0, st>>>(rows, tab, ck_off, ck);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_rec_forward(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                       const double2* ck, const FwdItem* items, int64_t n_items, const double* c,
                       int64_t ldc, int64_t ncoef, int64_t batch, double* part, cudaStream_t st) {
  if (n_items <= 0 || batch <= 0) return CJT_OK;
  dim3 grid((unsigned)n_items, (unsigned)((batch + FWD_VT - 1) / FWD_VT));
  k_rec_forward<<<grid, FWD_ROWS, 0, st>>>(rows, tab, ck_off, ck, items, c, ldc, ncoef, batch, part);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_rec_forward_reduce(const int32_t* tile_slot0, const int32_t* tile_nslot, int64_t nrows,
                              const double* part, double* vals, int64_t ldv, int64_t batch,
                              cudaStream_t st) {
  const int T = 256;
  dim3 grid((unsigned)((nrows + T - 1) / T), (unsigned)batch);
  k_rec_forward_reduce<<<grid, T, 0, st>>>(tile_slot0, tile_nslot, nrows, part, vals, ldv, batch);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_rec_inverse(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                       const double2* ck, const InvItem* items, int64_t n_items,
                       const int32_t* tile_ids, const double* wv, int64_t ldw, int64_t batch,
                       double* part, cudaStream_t st) {
  if (n_items <= 0 || batch <= 0) return CJT_OK;
  const int smem = 2 * INV_RT * 64 * (int)sizeof(double);
  static bool init = false;
  if (!init) {
    CJT_CUDA_TRY(cudaFuncSetAttribute(k_rec_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    init = true;
  }
  dim3 grid((unsigned)n_items, (unsigned)((batch + INV_VT - 1) / INV_VT));
  k_rec_inverse<<<grid, 256, smem, st>>>(rows, tab, ck_off, ck, items, tile_ids, wv, ldw, batch, part);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_inverse_finish(const int32_t* dt_slot0, const int32_t* dt_nslot, int64_t ndeg,
                          const double* part, const double* blocks_acc, const double* scal,
                          double* out, int64_t ldo, int64_t batch, cudaStream_t st) {
  const int T = 256;
  dim3 grid((unsigned)((ndeg + T - 1) / T), (unsigned)batch);
  k_inverse_finish<<<grid, T, 0, st>>>(dt_slot0, dt_nslot, ndeg, part, blocks_acc, scal, out, ldo, batch);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_clenshaw_points(const RecTablesDev& tab, const double* rbp, const double* rbm,
                           const double* rbpi, const double* rbmi, const double* coeffs,
                           const double* x, const double* xm, const int8_t* reg,
                           const int64_t* cut, double* out, int64_t npts, cudaStream_t st) {
  if (npts <= 0) return CJT_OK;
  const int T = 128;
  k_clenshaw_points<<<(unsigned)((npts + T - 1) / T), T, 0, st>>>(tab, rbp, rbm, rbpi, rbmi, coeffs,
                                                                  x, xm, reg, cut, out, npts);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

}  // namespace cjt
