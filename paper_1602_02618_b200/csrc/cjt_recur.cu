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
#include <algorithm>
#include <cstdlib>
#include <type_traits>


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

// Generation arithmetic of the contraction kernels (FMA form; gen_chain,
// gen_chain_g below).  The reference's rounding (rec_step) is kept where its
// exact values are the contract: plan-time checkpoints and the Clenshaw plugin.  The P values the
// transforms contract with are generated with the same recurrences in FMA
// form, whose dependency chain is two operations per degree instead of five
// (Reinsch) or two instead of three (three-term), with a' = A / rf, c' = C / rf
// tabulated per degree:
//   three-term: p_{n+1} = fma(fma(A x, 1, B), p_n, -(C p_{n-1}))
//   Reinsch:    d = fma(a' xm, s0, c' s1);  s0 <- fma(rf, d, rf s0);  s1 <- d
// (algebraically identical to _kernels_cy.pyx:144-147 / 186-188; differs by
// rounding only, well inside the transform tolerance).

// Recurrence tables of a degree window staged in shared memory:
// rows 0..8 = A, B, C, rf+, rf-, A/rf+, A/rf-, C/rf+, C/rf- (REC_WIN_ROWS),
// each `span` entries from n_lo.
__device__ __forceinline__ const double* table_row(const RecTablesDev& t, int r) {
  switch (r) {
    case 0: return t.A;
    case 1: return t.B;
    case 2: return t.C;
    case 3: return t.rfp;
    case 4: return t.rfm;
    case 5: return t.Ap;
    case 6: return t.Am;
    case 7: return t.Cp;
    default: return t.Cm;
  }
}
// K consecutive degrees of one recurrence chain from a shared-memory table
// window (rows A, B, C, rf+, rf-, A/rf+, A/rf-, C/rf+, C/rf- at stride
// STRIDE, entry k of this chain at tb[r STRIDE + k]): st(k, P_k) for
// k < K (0 from degree nval on), advancing the state while k + 1 < nval
// (nval = cut - first degree, clamped to [0, K + 1]: K + 1 hands the state on
// to the next stage).
// The region branch is taken once per call and every table read has a
// compile-time offset: the loop is issue-bound, not latency-bound.
template <int K, int STRIDE, class Store>
__device__ __forceinline__ void gen_chain(int reg, double xx, const double* tb, int nval, double& s0,
                                          double& s1, const Store& st) {
  if (nval > K) {
    // full stage (the common case): no predicates, so each 8-degree chunk's
    // table reads and chain-independent products are issued ahead of the
    // chain; the dependency chain is one DFMA (three-term) or two (Reinsch)
    // per degree instead of a shared-memory load latency per degree
    constexpr int CH = 8;
    if (reg == 0) {
#pragma unroll
      for (int k0 = 0; k0 < K; k0 += CH) {
        double t[CH], c[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          t[j] = fma(tb[k0 + j], xx, tb[STRIDE + k0 + j]);
          c[j] = tb[2 * STRIDE + k0 + j];
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          st(k0 + j, s1);
          const double pn = fma(t[j], s1, -(c[j] * s0));
          s0 = s1;
          s1 = pn;
        }
      }
    } else {
      const int o = reg > 0 ? 0 : 1;
      const double* rf = tb + (3 + o) * STRIDE;
      const double* ap = tb + (5 + o) * STRIDE;
      const double* cp = tb + (7 + o) * STRIDE;
#pragma unroll
      for (int k0 = 0; k0 < K; k0 += CH) {
        double a[CH], c[CH], r[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          a[j] = ap[k0 + j] * xx;
          c[j] = cp[k0 + j];
          r[j] = rf[k0 + j];
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          st(k0 + j, s0);
          const double d = fma(a[j], s0, c[j] * s1);
          s0 = fma(r[j], d, r[j] * s0);
          s1 = d;
        }
      }
    }
    return;
  }
  if (reg == 0) {
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
      st(k, k < nval ? s1 : 0.0);
      if (k + 1 < nval) {
        const double pn = fma(fma(tb[k], xx, tb[STRIDE + k]), s1, -(tb[2 * STRIDE + k] * s0));
        s0 = s1;
        s1 = pn;
      }
    }
  } else {
    const int o = reg > 0 ? 0 : 1;
    const double* rf = tb + (3 + o) * STRIDE;
    const double* ap = tb + (5 + o) * STRIDE;
    const double* cp = tb + (7 + o) * STRIDE;
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
      st(k, k < nval ? s0 : 0.0);
      if (k + 1 < nval) {
        const double d = fma(ap[k] * xx, s0, cp[k] * s1);
        s0 = fma(rf[k], d, rf[k] * s0);
        s1 = d;
      }
    }
  }
}

// The same chain with the tables read from global memory (L1-resident
// windows) from degree n0: pgen kernels of the two-pass contraction.
template <int K, class Store>
__device__ __forceinline__ void gen_chain_g(int reg, double xx, const RecTablesDev& t, int64_t n0,
                                            int nval, double& s0, double& s1, const Store& st) {
  if (reg == 0) {
    const double *A = t.A + n0, *B = t.B + n0, *C = t.C + n0;
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
      st(k, k < nval ? s1 : 0.0);
      if (k + 1 < nval) {
        const double pn = fma(fma(__ldg(A + k), xx, __ldg(B + k)), s1, -(__ldg(C + k) * s0));
        s0 = s1;
        s1 = pn;
      }
    }
  } else {
    const double* rf = (reg > 0 ? t.rfp : t.rfm) + n0;
    const double* ap = (reg > 0 ? t.Ap : t.Am) + n0;
    const double* cp = (reg > 0 ? t.Cp : t.Cm) + n0;
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
      st(k, k < nval ? s0 : 0.0);
      if (k + 1 < nval) {
        const double r = __ldg(rf + k);
        const double d = fma(__ldg(ap + k) * xx, s0, __ldg(cp + k) * s1);
        s0 = fma(r, d, r * s0);
        s1 = d;
      }
    }
  }
}

// Per-(row tile, generator thread) start state of K2, laid out densely in
// work-list order so the kernel streams it with one coalesced load per stage.
struct GenState {
  double s0, s1;   // recurrence state at degree nstart
  double xx;       // x (interior) or x - x0 (endpoint regions)
  int64_t cutreg;  // cut * 4 + (region + 1); cut = 0 marks an idle generator
};

__global__ void k_build_inv_gen(RecRowsDev rows, const int64_t* __restrict__ ck_off,
                                const double2* __restrict__ ck, const int32_t* __restrict__ ids,
                                const int32_t* __restrict__ gn0, int64_t total,
                                GenState* __restrict__ out) {
  const int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= total * 128) return;
  const int64_t g = gi / 128;
  const int tid = (int)(gi % 128);
  // chunk-major: generator tid = (chunk tid / 32, row tid % 32), so each
  // producer warp of K2 reads one degree window (broadcast table reads)
  const int64_t i = (int64_t)ids[g] * INV_RT + (tid & 31);
  const int64_t nstart = gn0[g] + CK * (tid >> 5);
  GenState st{0.0, 0.0, 0.0, 0};
  if (i < rows.nrows) {
    const int64_t cut = rows.cut[i];
    const int reg = rows.reg[i];
    if (cut > nstart) {
      load_state(rows, ck_off, ck, i, nstart, reg, st.s0, st.s1);
      st.xx = reg == 0 ? rows.x[i] : rows.xm[i];
      st.cutreg = cut * 4 + (reg + 1);
    }
  }
  out[gi] = st;
}

// Plan-time recurrence checkpoints (s0, s1) every CK degrees of every row,
// in the reference's exact rounding (rec_step).  Each row is a serial chain;
// the table entries of a window of degrees are staged in shared memory once
// per CTA (all its rows step through the same degrees), so a step costs the
// chain's own latency instead of a global load round trip.
constexpr int CKW = 256;   // degrees per staged window
__global__ void __launch_bounds__(128) k_checkpoints(RecRowsDev rows, RecTablesDev tab,
                                                     const int64_t* __restrict__ ck_off, double2* __restrict__ ck) {
  __shared__ double w[7][CKW];
  __shared__ int64_t s_max;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < rows.nrows;
  const int reg = live ? rows.reg[i] : 0;
  const double x = live ? rows.x[i] : 0.0, xm = live ? rows.xm[i] : 0.0;
  const int64_t nc = live ? rows.cut[i] : 0;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  atomicMax((unsigned long long*)&s_max, (unsigned long long)nc);
  __syncthreads();
  const int64_t top = s_max;   // the CTA's longest chain
  double s0, s1;
  rec_init(reg, s0, s1);
  double2* out = live ? ck + ck_off[i] : nullptr;
  const double* rf_t = reg > 0 ? &w[3][0] : &w[4][0];
  const double* rfi_t = reg > 0 ? &w[5][0] : &w[6][0];
  for (int64_t n0 = 0; n0 + 1 < top; n0 += CKW) {
    __syncthreads();
    for (int e = threadIdx.x; e < 7 * CKW; e += blockDim.x) {
      const int r = e / CKW, k = e % CKW;
      const int64_t n = n0 + k;
      const double* src = r == 0 ? tab.A : r == 1 ? tab.B : r == 2 ? tab.C : r == 3 ? tab.rfp
                        : r == 4 ? tab.rfm : r == 5 ? tab.rfpi : tab.rfmi;
      w[r][k] = n < tab.n_tab ? __ldg(src + n) : 0.0;
    }
    __syncthreads();
    const int64_t n1 = min(n0 + CKW, nc - 1);
    int64_t n = n0;
    // whole checkpoint intervals: CK steps fully unrolled (table reads hoisted
    // off the dependent chain, no per-step bounds or checkpoint tests); same
    // operations in the same order as the tail loop below (bit-identical)
    for (; n + CK <= n1; n += CK) {
      const int kb = (int)(n - n0);
      if (reg == 0) {
#pragma unroll
        for (int k = 0; k < CK; ++k) {
          const double pn = __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(w[0][kb + k], x), w[1][kb + k]), s1),
                                      __dmul_rn(w[2][kb + k], s0));
          s0 = s1;
          s1 = pn;
        }
      } else {
#pragma unroll
        for (int k = 0; k < CK; ++k) {
          const double d = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(w[0][kb + k], xm), s0), __dmul_rn(w[2][kb + k], s1)),
                                     rfi_t[kb + k]);
          s0 = __dmul_rn(__dadd_rn(s0, d), rf_t[kb + k]);
          s1 = d;
        }
      }
      out[(n + CK) / CK - 1] = make_double2(s0, s1);
    }
    for (; n < n1; ++n) {
      const int k = (int)(n - n0);
      const double a = w[0][k], c = w[2][k];
      if (reg == 0) {
        const double pn = __dsub_rn(__dmul_rn(__dadd_rn(__dmul_rn(a, x), w[1][k]), s1), __dmul_rn(c, s0));
        s0 = s1;
        s1 = pn;
      } else {
        const double d = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, xm), s0), __dmul_rn(c, s1)), rfi_t[k]);
        s0 = __dmul_rn(__dadd_rn(s0, d), rf_t[k]);
        s1 = d;
      }
      if (((n + 1) % CK) == 0) out[(n + 1) / CK - 1] = make_double2(s0, s1);
    }
  }
}

// ---------------------------------------------------------------------------
// DMMA helpers: mma.sync m8n8k4 f64 (the fp64 tensor path of sm_100a; tcgen05
// has no f64 kind).  Fragments: A[r][k] at lane 4r+k, B[k][n] at lane 4n+k,
// D[r][2c+j] at lane 4r+c.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// 8-byte async copy global -> shared, zero-filled when !valid
__device__ __forceinline__ void cp_async8(void* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0));
}
// 16-byte async copy global -> shared with zero fill beyond `bytes` (0, 8, 16)
__device__ __forceinline__ void cp_async16z(void* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Warp-specialised DMMA contractions (K1, K2).
//   consumers: NCW warps, 4 along M (32 rows/degrees each) x NCW/4 along N,
//              DMMA only (mma.sync m8n8k4 f64), accumulators in registers;
//   producers: 4 warps (128 threads) running the recurrence generators and
//              staging the other operand with cp.async, one stage ahead.
// Stages rotate through a ring of NBUF buffers handed over with named barriers:
//   FULL[b]  (ids 1..NBUF):        producers bar.arrive after filling buffer b,
//                                  consumers bar.sync before reading it;
//   EMPTY[b] (ids NBUF+1..2 NBUF): consumers bar.arrive after reading buffer b,
//                                  producers bar.sync before refilling it;
//   id 2 NBUF + 1: producer-only barrier (their private table buffers).
// On B200 DMMA and DMUL/DADD share the fp64 datapath, so the generators'
// serial chains are slowed by the consumers' DMMAs; NBUF = 3 gives them two
// consumer stages of slack instead of one.
#ifndef CJT_NCW8_MIN
#define CJT_NCW8_MIN 128
#endif
template <int VT>
struct WsCfg {
  static constexpr int NBUF = VT == 64 ? 3 : 2;      // P stage ring depth (small tiles: occupancy)
  // operand-tile ring (c / wv): one deeper than the P ring, so the producers
  // prefetch the next stage's tile while generating this stage's P (its
  // global-load latency is hidden behind the recurrence chains)
  static constexpr int NCB = NBUF + 1;
  static constexpr int NCW = VT >= CJT_NCW8_MIN ? 8 : 4;   // consumer warps
  static constexpr int NC = 32 * NCW;
  static constexpr int NP = 128;                     // producer threads
  static constexpr int NTH = NC + NP;
  static constexpr int NWN = NCW / 4;                // consumer warps along N
  static constexpr int NT = VT / 8 / NWN;            // 8-vector DMMA tiles per consumer warp
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
constexpr int RING_MAX = 3;
constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + RING_MAX, BAR_PROD = 1 + 2 * RING_MAX;

// K1 (forward): values[b][i] = sum_n P_n(x_i) c[b][n] over one item
// (128 rows x a degree segment) and one tile of VT vectors; stages of 32
// degrees.  Producer thread p owns row p's recurrence chain (state carried
// across stages in registers) and writes P^T[k][p].
// FOLD (alpha = beta, see cjt_plan::fold): the stage's 32 degrees are stored
// parity-sorted (slot k/2 for even k, 16 + k/2 for odd k) and contracted into
// two accumulator sets, E (even degrees) and O (odd degrees); the reduce
// writes E + O to row i and E - O to its mirror row G - i.
template <int VT, bool FOLD>
__global__ void __launch_bounds__(WsCfg<VT>::NTH)
    k_rec_forward_ws(RecRowsDev rows, RecTablesDev tab, const int64_t* __restrict__ ck_off,
                     const double2* __restrict__ ck, const FwdItem* __restrict__ items,
                     const double* __restrict__ c, int64_t ldc, int64_t ncoef, int64_t batch,
                     double* __restrict__ part, int dbg) {
  using W = WsCfg<VT>;
  constexpr int PT = FWD_ROWS + 4;   // P^T row stride (degrees x rows)
  constexpr int CS = FWD_KS + 4;     // staged c row stride (vectors x degrees)
  extern __shared__ __align__(16) double smem_rec[];
  double(*Pt)[FWD_KS][PT] = reinterpret_cast<double(*)[FWD_KS][PT]>(smem_rec);
  double(*Cs)[VT][CS] = reinterpret_cast<double(*)[VT][CS]>(smem_rec + W::NBUF * FWD_KS * PT);
  double(*Ts)[REC_WIN_ROWS * FWD_KS] =
      reinterpret_cast<double(*)[REC_WIN_ROWS * FWD_KS]>(smem_rec + W::NBUF * FWD_KS * PT + W::NCB * VT * CS);
  const FwdItem it = items[blockIdx.x];
  const int64_t b0 = (int64_t)blockIdx.y * VT;
  const int tid = threadIdx.x;
  const int nstages = (it.n_end - it.n_begin) / FWD_KS;

  if (tid >= W::NC) {
    // ------------------------------ producer ------------------------------
    const int p = tid - W::NC;
    const int64_t gi = it.row0 + p;
    int reg = 0;
    double xx = 0.0, s0 = 0.0, s1 = 0.0;
    int64_t cut = 0;
    if (p < it.nrows) {
      reg = rows.reg[gi];
      xx = reg == 0 ? rows.x[gi] : rows.xm[gi];
      cut = rows.cut[gi];
      if (cut > it.n_begin) load_state(rows, ck_off, ck, gi, it.n_begin, reg, s0, s1);
    }
    // table window: one 16-byte copy (two degrees) per producer thread
    // p < 144; the row pointer is fixed per thread
    // (144 copies: thread p copies chunk p and, for p < 16, chunk p + 128)
    constexpr int TCH = REC_WIN_ROWS * FWD_KS / 2;
    static_assert(TCH <= 2 * W::NP, "table window copies");
    const int tk = 2 * (p % (FWD_KS / 2));
    const int trow0 = p / (FWD_KS / 2), trow1 = (p + W::NP) / (FWD_KS / 2);
    const double* tsrc0 = table_row(tab, trow0);
    const double* tsrc1 = table_row(tab, min(trow1, REC_WIN_ROWS - 1));
    auto stage_tables = [&](int buf, int64_t n0) {
      const int64_t n = n0 + tk;
      const int bytes = n + 1 < tab.n_tab ? 16 : n < tab.n_tab ? 8 : 0;
      cp_async16z(&Ts[buf][trow0 * FWD_KS + tk], bytes ? tsrc0 + n : tsrc0, bytes);
      if (p + W::NP < TCH) cp_async16z(&Ts[buf][trow1 * FWD_KS + tk], bytes ? tsrc1 + n : tsrc1, bytes);
    };
    // stage c[b0 .. b0+VT)[n0 .. n0+32) into Cs[cb]: 16-byte copies when the
    // rows are 16-byte aligned (even ldc), else 8-byte copies
    const bool c16 = !FOLD && ((ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0);
    auto stage_c = [&](int cb, int64_t n0) {
      if (c16) {
#pragma unroll
        for (int q = 0; q < (VT * FWD_KS / 2) / W::NP; ++q) {
          const int idx = p + q * W::NP;
          const int v = idx / (FWD_KS / 2), k = 2 * (idx % (FWD_KS / 2));
          const int64_t bb = b0 + v, n = n0 + k;
          const int bytes = bb >= batch ? 0 : n + 1 < ncoef ? 16 : n < ncoef ? 8 : 0;
          cp_async16z(&Cs[cb][v][k], bytes ? c + bb * ldc + n : c, bytes);
        }
      } else {
#pragma unroll
        for (int q = 0; q < (VT * FWD_KS) / W::NP; ++q) {
          const int idx = p + q * W::NP;
          const int v = idx / FWD_KS, k = idx % FWD_KS;
          const int64_t bb = b0 + v, n = n0 + k;
          const bool ok = bb < batch && n < ncoef;
          const int slot = FOLD ? (k & 1) * (FWD_KS / 2) + (k >> 1) : k;
          cp_async8(&Cs[cb][v][slot], ok ? c + bb * ldc + n : c, ok);
        }
      }
    };
    stage_tables(0, it.n_begin);
    stage_c(0, it.n_begin);
    cp_async_commit();
    cp_async_wait_all();
    named_sync(BAR_PROD, W::NP);
    for (int sidx = 0; sidx < nstages; ++sidx) {
      const int buf = sidx % W::NBUF, tb = sidx & 1;
      const int64_t n0 = it.n_begin + (int64_t)sidx * FWD_KS;
      if (sidx >= W::NBUF) named_sync(BAR_EMPTY + buf, W::NTH);
      // next stage's c tile and tables (Cs[(sidx+1) % NCB] was last read by
      // stage sidx + 1 - NCB = sidx - NBUF, released by the EMPTY wait above)
      // (two groups: the tables, needed by the producers at the next stage,
      // then the c tile, needed by the consumers one stage later still)
      if (sidx + 1 < nstages) stage_tables(tb ^ 1, n0 + FWD_KS);
      cp_async_commit();
      if (sidx + 1 < nstages) stage_c((sidx + 1) % W::NCB, n0 + FWD_KS);
      cp_async_commit();
      const int nval = (int)max((int64_t)0, min((int64_t)FWD_KS + 1, cut - n0));
      if (dbg != 1)
        gen_chain<FWD_KS, FWD_KS>(reg, xx, Ts[tb], nval, s0, s1, [&](int k, double v) {
          Pt[buf][FOLD ? (k & 1) * (FWD_KS / 2) + (k >> 1) : k][p] = v;
        });
      // next stage's tables and this stage's c tile landed; the next c tile
      // (newest group) may stay in flight
      cp_async_wait<1>();
      named_sync(BAR_PROD, W::NP);            // next stage's tables visible to all producers
      named_arrive(BAR_FULL + buf, W::NTH);   // P^T and c tile of this stage are ready
    }
    return;
  }

  // ------------------------------ consumer --------------------------------
  const int lane = tid & 31, warp = (tid >> 5) & 3, wn = tid >> 7;
  const int ar = lane >> 2, ak = lane & 3;
  const int ntile0 = wn * W::NT;
  constexpr int NS = FOLD ? 2 : 1;   // accumulator sets (E, O)
  double acc[NS][4][W::NT][2];
#pragma unroll
  for (int h = 0; h < NS; ++h)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < W::NT; ++nt) acc[h][mt][nt][0] = acc[h][mt][nt][1] = 0.0;
  for (int sidx = 0; sidx < nstages; ++sidx) {
    const int buf = sidx % W::NBUF, cbuf = sidx % W::NCB;
    named_sync(BAR_FULL + buf, W::NTH);
    if (dbg != 2)
#pragma unroll
    for (int kk = 0; kk < FWD_KS / 4; ++kk) {
      // FOLD: slots 0..15 hold the even degrees (set E), 16..31 the odd (O)
      constexpr int KH = FWD_KS / 4 / 2;
      const int h = (FOLD && kk >= KH) ? 1 : 0;
      double a[4], bf[W::NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = Pt[buf][4 * kk + ak][32 * warp + 8 * mt + ar];
#pragma unroll
      for (int nt = 0; nt < W::NT; ++nt) bf[nt] = Cs[cbuf][8 * (ntile0 + nt) + ar][4 * kk + ak];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < W::NT; ++nt)
          dmma(acc[FOLD ? h : 0][mt][nt][0], acc[FOLD ? h : 0][mt][nt][1], a[mt], bf[nt]);
    }
    if (sidx + W::NBUF < nstages) named_arrive(BAR_EMPTY + buf, W::NTH);
  }
  // D[row][vec]: row = 32 warp + 8 mt + (lane>>2), vec = 8 (ntile0 + nt) + 2 (lane&3) + j
#pragma unroll
  for (int h = 0; h < NS; ++h) {
    double* dst = part + ((int64_t)it.slot * NS + h) * batch * FWD_ROWS;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < W::NT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int row = 32 * warp + 8 * mt + ar;
          const int64_t bb = b0 + 8 * (ntile0 + nt) + 2 * ak + j;
          if (bb < batch) dst[bb * FWD_ROWS + row] = acc[h][mt][nt][j];
        }
  }
}

// folded plans: rows i < nrows (= G/2 + 1) carry E (even degrees) and O (odd
// degrees) partials; row i gets E + O, its mirror G - i gets E - O
__global__ void k_rec_forward_reduce_fold(const int32_t* __restrict__ tile_slot0,
                                          const int32_t* __restrict__ tile_nslot, int64_t nrows,
                                          const double* __restrict__ part, double* __restrict__ vals,
                                          int64_t ldv, int64_t batch, int64_t G) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (i >= nrows) return;
  const int64_t tile = i / FWD_ROWS, lr = i % FWD_ROWS;
  const int32_t s0 = tile_slot0[tile], ns = tile_nslot[tile];
  double e = 0.0, o = 0.0;
#pragma unroll 4
  for (int s = 0; s < ns; ++s) {
    e += part[(((int64_t)(s0 + s) * 2 + 0) * batch + b) * FWD_ROWS + lr];
    o += part[(((int64_t)(s0 + s) * 2 + 1) * batch + b) * FWD_ROWS + lr];
  }
  vals[b * ldv + i] = e + o;
  if (G - i != i) vals[b * ldv + (G - i)] = e - o;
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
#pragma unroll 8   // independent loads in flight; the sum keeps its fixed order
  for (int s = 0; s < ns; ++s) acc += part[((int64_t)(s0 + s) * batch + b) * FWD_ROWS + lr];
  vals[b * ldv + i] = acc;
}

// K2 (inverse): out[b][n] = sum_i P_n(x_i) wv[b][i] for one item (128
// degrees x a list of 32-row tiles) and one tile of VT vectors; one stage per
// row tile.  Producer thread p = (row p/4, degree chunk p%4) restarts from the
// dense generator stream and writes P[row][deg]; producers also stage the
// wv tile.  The tables of the item's 128-degree window live in shared memory.
// FOLD (alpha = beta): rows i < nrows = G/2 + 1 only, degrees stored
// parity-sorted (window slot dl/2 for even dl, 64 + dl/2 for odd): consumer
// warps 0-1 contract the even degrees with wv_i + wv_{G-i}, warps 2-3 the odd
// degrees with wv_i - wv_{G-i} (the middle row i = G/2 counted once).
template <int VT, bool FOLD>
__global__ void __launch_bounds__(WsCfg<VT>::NTH)
    k_rec_inverse_ws(RecTablesDev tab, const GenState* __restrict__ gen, int64_t nrows,
                     const InvItem* __restrict__ items, const int32_t* __restrict__ tile_ids,
                     const double* __restrict__ wv, int64_t ldw, int64_t batch,
                     double* __restrict__ part, int dbg, int64_t G) {
  using W = WsCfg<VT>;
  // P stored degree-major, [degree slot][row] with row stride RS: a producer
  // warp (32 rows, one 32-degree chunk) stores 32 consecutive doubles per
  // degree, and the consumers' A fragments (rows 4 kk + ak, degrees 8 mt + ar)
  // hit bank pairs 4 ar + ak: conflict-free both ways
  constexpr int RS = INV_RT + 4;
  constexpr int WS = INV_RT + 4;
  constexpr int SPAN = INV_DT;      // table window: degrees n0 .. n0 + 127
  // window row stride with two pad slots per 32 degrees: chunk gq starts at slot 34 gq -- 16-byte
  // aligned (vector table loads) and in bank pair 2 gq (conflict-free)
  constexpr int SPANP = SPAN + 2 * (SPAN / 32);
  extern __shared__ __align__(16) double smem_rec[];
  double(*Ps)[INV_DT][RS] = reinterpret_cast<double(*)[INV_DT][RS]>(smem_rec);
  double(*Ws)[VT][WS] = reinterpret_cast<double(*)[VT][WS]>(smem_rec + W::NBUF * INV_DT * RS);
  // FOLD: the mirror rows' wv tile, ring after Ws
  double(*Wm)[VT][WS] = reinterpret_cast<double(*)[VT][WS]>(smem_rec + W::NBUF * INV_DT * RS + W::NCB * VT * WS);
  double* Tw = smem_rec + W::NBUF * INV_DT * RS + (FOLD ? 2 : 1) * W::NCB * VT * WS;   // [REC_WIN_ROWS][SPAN]
  const InvItem it = items[blockIdx.x];
  const int64_t b0 = (int64_t)blockIdx.y * VT;
  const int tid = threadIdx.x;

  if (tid >= W::NC) {
    // ------------------------------ producer ------------------------------
    const int p = tid - W::NC;
    const int grow = p & 31, gq = p >> 5;   // producer warp gq: degree chunk gq of all 32 rows
    for (int idx = p; idx < REC_WIN_ROWS * SPAN; idx += W::NP) {
      const int r = idx / SPAN, k = idx % SPAN;
      const int slot = r * SPANP + k + 2 * (k >> 5);
      const bool ok = it.n0 + k < tab.n_tab;
      const double* src = table_row(tab, r);
      cp_async8(&Tw[slot], ok ? src + it.n0 + k : src, ok);
    }
    // stage the wv tile of row tile tt into Ws[wb]
    auto stage_wv = [&](int wb, int tt) {
      const int64_t r0 = (int64_t)tile_ids[it.t_begin + tt] * INV_RT;
#pragma unroll
      for (int q = 0; q < (VT * INV_RT) / W::NP; ++q) {
        const int idx = p + q * W::NP;
        const int v = idx / INV_RT, k = idx % INV_RT;
        const int64_t bb = b0 + v, i = r0 + k;
        const bool ok = bb < batch && i < nrows;
        cp_async8(&Ws[wb][v][k], ok ? wv + bb * ldw + i : wv, ok);
        if constexpr (FOLD) {
          const bool okm = ok && G - i != i;   // the middle row is its own mirror
          cp_async8(&Wm[wb][v][k], okm ? wv + bb * ldw + (G - i) : wv, okm);
        }
      }
    };
    stage_wv(0, 0);
    cp_async_commit();
    cp_async_wait_all();
    named_sync(BAR_PROD, W::NP);
    const GenState* gbase = gen + (int64_t)it.t_begin * 128 + p;
    GenState nxt = gbase[0];
    const int nl0 = CK * gq;
    const int64_t nstart = it.n0 + nl0;
    for (int tt = 0; tt < it.t_count; ++tt) {
      const int buf = tt % W::NBUF;
      GenState g = nxt;
      if (tt + 1 < it.t_count) nxt = gbase[(int64_t)(tt + 1) * 128];   // prefetch
      if (tt >= W::NBUF) named_sync(BAR_EMPTY + buf, W::NTH);
      // next tile's wv (Ws[(tt+1) % NCB] last read at stage tt - NBUF, released above)
      if (tt + 1 < it.t_count) stage_wv((tt + 1) % W::NCB, tt + 1);
      cp_async_commit();
      const int64_t cut = g.cutreg >> 2;
      const int reg = (int)(g.cutreg & 3) - 1;
      const int nval = (int)max((int64_t)0, min((int64_t)CK + 1, cut - nstart));
      // this chunk's window: degrees nl0 + k at slot nl0 + k + 2 gq (pads per 32)
      if (dbg != 1)
        gen_chain<CK, SPANP>(reg, g.xx, Tw + nl0 + 2 * gq, nval, g.s0, g.s1, [&](int k, double v) {
          const int dl = nl0 + k;
          Ps[buf][FOLD ? (dl & 1) * (INV_DT / 2) + (dl >> 1) : dl][grow] = v;
        });
      // this stage's wv tile (committed one iteration ago) must have landed;
      // the next tile's copies (newest group) may stay in flight
      cp_async_wait<1>();
      named_arrive(BAR_FULL + buf, W::NTH);
    }
    return;
  }

  // ------------------------------ consumer --------------------------------
  const int lane = tid & 31, warp = (tid >> 5) & 3, wn = tid >> 7;
  const int ar = lane >> 2, ak = lane & 3;
  const int ntile0 = wn * W::NT;
  double acc[4][W::NT][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < W::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  for (int tt = 0; tt < it.t_count; ++tt) {
    const int buf = tt % W::NBUF, wbuf = tt % W::NCB;
    named_sync(BAR_FULL + buf, W::NTH);
    if (dbg != 2)
#pragma unroll
    for (int kk = 0; kk < INV_RT / 4; ++kk) {
      double a[4], bf[W::NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = Ps[buf][32 * warp + 8 * mt + ar][4 * kk + ak];
#pragma unroll
      for (int nt = 0; nt < W::NT; ++nt) {
        bf[nt] = Ws[wbuf][8 * (ntile0 + nt) + ar][4 * kk + ak];
        if constexpr (FOLD) {   // even-degree warps: wv_i + wv_{G-i}; odd: wv_i - wv_{G-i}
          const double m = Wm[wbuf][8 * (ntile0 + nt) + ar][4 * kk + ak];
          bf[nt] = warp < 2 ? bf[nt] + m : bf[nt] - m;
        }
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < W::NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[nt]);
    }
    if (tt + W::NBUF < it.t_count) named_arrive(BAR_EMPTY + buf, W::NTH);
  }
  double* dst = part + (int64_t)it.slot * batch * INV_DT;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < W::NT; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int slot = 32 * warp + 8 * mt + ar;
        const int deg = FOLD ? (slot < INV_DT / 2 ? 2 * slot : 2 * (slot - INV_DT / 2) + 1) : slot;
        const int64_t bb = b0 + 8 * (ntile0 + nt) + 2 * ak + j;
        if (bb < batch) dst[bb * INV_DT + deg] = acc[mt][nt][j];
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
#pragma unroll 8   // independent loads in flight; the sum keeps its fixed order
  for (int s = 0; s < ns; ++s) acc += part[((int64_t)(s0 + s) * batch + b) * INV_DT + k];
  out[b * ldo + n] = acc * scal[n];
}

// Reference-signature Clenshaw-Smith / Reinsch evaluation, one thread per
// point, the reference's exact operation order (_kernels_cy.pyx:17-80).
// DIV: the scalar Python form (recurrences.py:149) divides by rb[n] where
// the Cython kernel multiplies by the tabulated reciprocal.
template <bool DIV>
__global__ void k_clenshaw_points(RecTablesDev tab, const double* __restrict__ rbp,
                                  const double* __restrict__ rbm, const double* __restrict__ rbpi,
                                  const double* __restrict__ rbmi,
                                  const double* __restrict__ coeffs, int64_t ldc,
                                  const double* __restrict__ xs, const double* __restrict__ xms,
                                  const int8_t* __restrict__ regs, const int64_t* __restrict__ cuts,
                                  double* __restrict__ out, int64_t ldo, int64_t npts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  // batch: vector blockIdx.y (evaluate_expansion_batched); the plugin uses one
  coeffs += (int64_t)blockIdx.y * ldc;
  out += (int64_t)blockIdx.y * ldo;
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
      u = DIV ? __ddiv_rn(__dadd_rn(u, d), rb[n]) : __dmul_rn(__dadd_rn(u, d), rbi[n]);
    }
    out[i] = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(tab.A[0], xm), u), __dmul_rn(tab.C[1], d)),
                       coeffs[0]);
  }
}

// P_0 .. P_{n_max} at one point per thread (recurrences.py:74-112): the plain
// forward three-term recurrence (mode 0) or Reinsch's modified forward
// recurrence anchored at +1 / -1 (mode +1 / -1, rf = rf_plus / rf_minus), the
// reference's operation order and true division, so values are bit-identical.
// out: [npts][n_max + 1].
__global__ void k_jacobi_values(RecTablesDev tab, int64_t n_max, const double* __restrict__ xs,
                                const double* __restrict__ xms, const int8_t* __restrict__ mode,
                                double* __restrict__ out, int64_t npts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double* o = out + i * (n_max + 1);
  o[0] = 1.0;
  const int md = mode[i];
  if (md == 0) {
    const double x = xs[i];
    double p_prev = 0.0, p_cur = 1.0;
    for (int64_t n = 0; n < n_max; ++n) {
      const double t = __dmul_rn(__dadd_rn(__dmul_rn(tab.A[n], x), tab.B[n]), p_cur);
      const double p_next = __dsub_rn(t, __dmul_rn(tab.C[n], p_prev));
      p_prev = p_cur;
      p_cur = p_next;
      o[n + 1] = p_cur;
    }
  } else {
    const double xm = xms[i];
    const double* rf = md > 0 ? tab.rfp : tab.rfm;
    double pi_cur = 1.0, d = 0.0;
    for (int64_t n = 0; n < n_max; ++n) {
      const double num = __dadd_rn(__dmul_rn(__dmul_rn(tab.A[n], xm), pi_cur), __dmul_rn(tab.C[n], d));
      d = __ddiv_rn(num, rf[n]);
      pi_cur = __dmul_rn(__dadd_rn(pi_cur, d), rf[n]);
      o[n + 1] = pi_cur;
    }
  }
}


// ---------------------------------------------------------------------------
// Two-pass recurrence contraction (default when the P workspace fits):
//   pass 1  k_pgen_fwd / k_pgen_inv: generate every P_n(x_i) of the recurrence
//           region once per execution, fully row- and segment-parallel from the
//           per-plan checkpoints, into an HBM workspace laid out as the 32 x 128
//           blocks the contraction streams;
//   pass 2  k_rec_gemm: a cp.async-pipelined fp64 DMMA GEMM over those blocks.
// Generating in its own pass keeps the generators' DMUL/DADD chains off the
// fp64 datapath the DMMAs saturate (on B200 they share it).

// forward blocks: block (t, j) = P^T[k][row] for rows 128 t.. and degrees 32 j..
// (grid-stride over blocks: many resident warps hide the chains' latency)
__global__ void __launch_bounds__(128)
    k_pgen_fwd(RecRowsDev rows, RecTablesDev tab, const int64_t* __restrict__ ck_off,
               const double2* __restrict__ ck, const int2* __restrict__ blk_tj, int64_t nblk,
               double* __restrict__ P, int fold) {
  const int tid = threadIdx.x;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int2 tj = blk_tj[blk];
    const int64_t i = (int64_t)tj.x * FWD_ROWS + tid;
    const int64_t n0 = (int64_t)tj.y * FWD_KS;
    double* out = P + blk * (FWD_KS * FWD_ROWS) + tid;
    int64_t cut = 0;
    int reg = 0;
    double x = 0.0, xm = 0.0, s0 = 0.0, s1 = 0.0;
    if (i < rows.nrows) {
      cut = rows.cut[i];
      if (cut > n0) {
        reg = rows.reg[i];
        x = rows.x[i];
        xm = rows.xm[i];
        load_state(rows, ck_off, ck, i, n0, reg, s0, s1);
      }
    }
    const int nval = (int)max((int64_t)0, min((int64_t)FWD_KS + 1, cut - n0));
    // fold: parity-sorted degree slots (see k_rec_forward_ws)
    gen_chain_g<FWD_KS>(reg, reg == 0 ? x : xm, tab, n0, nval, s0, s1, [&](int k, double v) {
      out[(fold ? (k & 1) * (FWD_KS / 2) + (k >> 1) : k) * FWD_ROWS] = v;
    });
  }
}

// inverse blocks: block g = P[deg][row] (128 degrees x 32 rows) for work-list
// row tile g; thread (chunk q = tid/32, row = tid%32) runs degrees 32 q..32 q+31
// from the generator stream; each warp store is 32 consecutive doubles
__global__ void __launch_bounds__(128)
    k_pgen_inv(RecTablesDev tab, const GenState* __restrict__ gen, const int32_t* __restrict__ gn0,
               int64_t gbeg, int64_t gend, double* __restrict__ P) {
  const int tid = threadIdx.x;
  const int q = tid >> 5, row = tid & 31;
  for (int64_t g = gbeg + blockIdx.x; g < gend; g += gridDim.x) {
    GenState st = gen[g * 128 + q * 32 + row];
    const int64_t cut = st.cutreg >> 2;
    const int reg = (int)(st.cutreg & 3) - 1;
    const int64_t nstart = (int64_t)gn0[g] + CK * q;
    double* out = P + (g - gbeg) * (INV_RT * INV_DT) + (CK * q) * INV_RT + row;
    const int nval = (int)max((int64_t)0, min((int64_t)CK + 1, cut - nstart));
    gen_chain_g<CK>(reg, st.xx, tab, nstart, nval, st.s0, st.s1,
                    [&](int k, double v) { out[k * INV_RT] = v; });
  }
}

// 16-byte async copy (both addresses 16-byte aligned)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}

// A block in global memory: AMK = false -> [k 32][m 128] (forward P^T),
// AMK = true -> [m 128][k 32] (inverse P transposed for coalesced generation);
// the shared-memory copy keeps the same orientation with padded rows so the
// DMMA A-fragment loads are conflict-free either way.
template <int VT, bool AMK>
struct GemmCfg {
  static constexpr int NCW = VT >= 64 ? 8 : 4;    // warps: 4 along M x NCW/4 along N
  static constexpr int NTH = 32 * NCW;
  static constexpr int NWN = NCW / 4;
  static constexpr int NT = VT / 8 / NWN;
  static constexpr int STAGES = 3;
  static constexpr int AROWS = AMK ? 128 : 32;
  static constexpr int AS = AMK ? 32 + 4 : 128 + 4;   // A row stride
  static constexpr int XS = 32 + 4;
  static constexpr int SMEM = 8 * STAGES * (AROWS * AS + VT * XS);
};

// out[slot][b][m] = sum over the item's stages s, k < 32 of
//   A_s[k][m] * x[b][xoff(s) + k],  A_s = P block (p_block0 + s) (32 x 128),
// xoff(s) = x_off0 + 32 s (forward: contiguous degrees) or 32 * ids[ids_off + s]
// (inverse: the item's row tiles).
// FOLD (forward, alpha = beta): degree slots parity-sorted by k_pgen_fwd; two
// accumulator sets (even / odd degrees), partials [slot][2][batch][128]
template <int VT, bool AMK, bool FOLD = false>
__global__ void __launch_bounds__(GemmCfg<VT, AMK>::NTH)
    k_rec_gemm(const GemmItem* __restrict__ items, const double* __restrict__ P,
               const int32_t* __restrict__ ids, const double* __restrict__ x, int64_t ldx,
               int64_t xlen, int64_t batch, double* __restrict__ part) {
  using C = GemmCfg<VT, AMK>;
  extern __shared__ __align__(16) double smem_g[];
  double(*As)[C::AROWS][C::AS] = reinterpret_cast<double(*)[C::AROWS][C::AS]>(smem_g);
  double(*Xs)[VT][C::XS] = reinterpret_cast<double(*)[VT][C::XS]>(smem_g + C::STAGES * C::AROWS * C::AS);
  const GemmItem it = items[blockIdx.y];
  const int64_t b0 = (int64_t)blockIdx.x * VT;
  const int tid = threadIdx.x, lane = tid & 31, warp = (tid >> 5) & 3, wn = tid >> 7;
  const int ar = lane >> 2, ak = lane & 3;
  const int ntile0 = wn * C::NT;

  auto load_stage = [&](int buf, int sidx) {
    const double* a = P + (it.p_block0 + sidx) * (int64_t)(32 * 128);
    constexpr int CPR = (AMK ? 32 : 128) / 2;        // 16-byte chunks per A row
#pragma unroll
    for (int q = 0; q < (32 * 64) / C::NTH; ++q) {
      const int idx = tid + q * C::NTH;
      const int r = idx / CPR, ch = idx % CPR;
      cp_async16(&As[buf][r][2 * ch], a + r * (2 * CPR) + 2 * ch);
    }
    const int64_t xoff = it.ids_off >= 0 ? (int64_t)ids[it.ids_off + sidx] * 32 : it.x_off0 + 32 * (int64_t)sidx;
#pragma unroll
    for (int q = 0; q < (VT * 32) / C::NTH; ++q) {
      const int idx = tid + q * C::NTH;
      const int v = idx >> 5, k = idx & 31;
      const int64_t bb = b0 + v, kk = xoff + k;
      const bool ok = bb < batch && kk < xlen;
      const int ks = FOLD ? (k & 1) * 16 + (k >> 1) : k;
      cp_async8(&Xs[buf][v][ks], ok ? x + bb * ldx + kk : x, ok);
    }
  };

  constexpr int NS = FOLD ? 2 : 1;
  double acc[NS][4][C::NT][2];
#pragma unroll
  for (int h = 0; h < NS; ++h)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) acc[h][mt][nt][0] = acc[h][mt][nt][1] = 0.0;

  const int ns = it.nstages;
#pragma unroll
  for (int sidx = 0; sidx < C::STAGES - 1; ++sidx) {
    if (sidx < ns) load_stage(sidx, sidx);
    cp_async_commit();
  }
  for (int sidx = 0; sidx < ns; ++sidx) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    const int nxt = sidx + C::STAGES - 1;
    if (nxt < ns) load_stage(nxt % C::STAGES, nxt);
    cp_async_commit();
    const int buf = sidx % C::STAGES;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double a[4], bf[C::NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        a[mt] = AMK ? As[buf][32 * warp + 8 * mt + ar][4 * kk + ak] : As[buf][4 * kk + ak][32 * warp + 8 * mt + ar];
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) bf[nt] = Xs[buf][8 * (ntile0 + nt) + ar][4 * kk + ak];
      const int h = (FOLD && kk >= 4) ? 1 : 0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
          dmma(acc[FOLD ? h : 0][mt][nt][0], acc[FOLD ? h : 0][mt][nt][1], a[mt], bf[nt]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int h = 0; h < NS; ++h) {
    double* dst = part + ((int64_t)it.slot * NS + h) * batch * 128;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int m = 32 * warp + 8 * mt + ar;
          const int64_t bb = b0 + 8 * (ntile0 + nt) + 2 * ak + j;
          if (bb < batch) dst[bb * 128 + m] = acc[h][mt][nt][j];
        }
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

// $CJT_WS_DBG (experiments only): 1 = producers skip generation, 2 = consumers skip DMMA
static int ws_debug() {
  static const int v = [] {
    const char* e = getenv("CJT_WS_DBG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int launch_rec_forward(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                       const double2* ck, const FwdItem* items, int64_t n_items, const double* c,
                       int64_t ldc, int64_t ncoef, int64_t batch, int vt, bool fold, double* part,
                       cudaStream_t st) {
  if (n_items <= 0 || batch <= 0) return CJT_OK;
  dim3 grid((unsigned)n_items, (unsigned)((batch + vt - 1) / vt));
  if (fold && vt > 64) return fail(CJT_EINVAL, "folded contraction tiles hold at most 64 vectors");
  switch (vt) {
#define CJT_FWD_F(V, F)                                                                          \
  {                                                                                              \
    constexpr int R = WsCfg<V>::NBUF;                                                            \
    const int smem = 8 * (R * FWD_KS * (FWD_ROWS + 4) + (R + 1) * V * (FWD_KS + 4) + 2 * REC_WIN_ROWS * FWD_KS);  \
    static DeviceOnce once_;                                                                    \
    if (int rc_ = once_([&]() -> int {                                                                                 \
      CJT_CUDA_TRY(cudaFuncSetAttribute(k_rec_forward_ws<V, F>,                                  \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, smem));     \
      return CJT_OK;                                                                               \
    })) return rc_;                                                                                            \
    k_rec_forward_ws<V, F><<<grid, WsCfg<V>::NTH, smem, st>>>(rows, tab, ck_off, ck, items, c,   \
                                                              ldc, ncoef, batch, part, ws_debug()); \
  }
#define CJT_FWD(V)                                                                               \
  case V:                                                                                        \
    if (fold) CJT_FWD_F(V, true) else CJT_FWD_F(V, false)                                       \
    break;
    case 128: CJT_FWD_F(128, false) break;
    CJT_FWD(64) CJT_FWD(32) CJT_FWD(24) CJT_FWD(16)
#undef CJT_FWD
#undef CJT_FWD_F
    default: return fail(CJT_EINVAL, "bad vector tile");
  }
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_rec_forward_reduce(const int32_t* tile_slot0, const int32_t* tile_nslot, int64_t nrows,
                              const double* part, double* vals, int64_t ldv, int64_t batch,
                              int64_t G, bool fold, cudaStream_t st) {
  const int T = 256;
  dim3 grid((unsigned)((nrows + T - 1) / T), (unsigned)batch);
  if (fold)
    k_rec_forward_reduce_fold<<<grid, T, 0, st>>>(tile_slot0, tile_nslot, nrows, part, vals, ldv, batch, G);
  else
    k_rec_forward_reduce<<<grid, T, 0, st>>>(tile_slot0, tile_nslot, nrows, part, vals, ldv, batch);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_build_inv_gen(const RecRowsDev& rows, const int64_t* ck_off, const double2* ck,
                         const int32_t* ids, const int32_t* gn0, int64_t total, void* out,
                         cudaStream_t st) {
  if (total <= 0) return CJT_OK;
  const int T = 128;
  k_build_inv_gen<<<(unsigned)((total * 128 + T - 1) / T), T, 0, st>>>(rows, ck_off, ck, ids, gn0, total,
                                                                       (GenState*)out);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_rec_inverse(const RecTablesDev& tab, const void* gen, int64_t nrows, const InvItem* items,
                       int64_t n_items, const int32_t* tile_ids, const double* wv, int64_t ldw,
                       int64_t batch, int vt, bool fold, int64_t G, double* part, cudaStream_t st) {
  if (n_items <= 0 || batch <= 0) return CJT_OK;
  if (fold && vt > 64) return fail(CJT_EINVAL, "folded contraction tiles hold at most 64 vectors");
  dim3 grid((unsigned)n_items, (unsigned)((batch + vt - 1) / vt));
  const GenState* g = (const GenState*)gen;
  switch (vt) {
#define CJT_INV_F(V, F)                                                                          \
  {                                                                                              \
    constexpr int R = WsCfg<V>::NBUF;                                                            \
    const int smem = 8 * (R * INV_DT * (INV_RT + 4) + (F ? 2 : 1) * (R + 1) * V * (INV_RT + 4) + \
                          REC_WIN_ROWS * (INV_DT + 2 * (INV_DT / 32)));                          \
    static DeviceOnce once_;                                                                    \
    if (int rc_ = once_([&]() -> int {                                                                                 \
      CJT_CUDA_TRY(cudaFuncSetAttribute(k_rec_inverse_ws<V, F>,                                  \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, smem));     \
      return CJT_OK;                                                                               \
    })) return rc_;                                                                                            \
    k_rec_inverse_ws<V, F><<<grid, WsCfg<V>::NTH, smem, st>>>(tab, g, nrows, items, tile_ids, wv, \
                                                              ldw, batch, part, ws_debug(), G);  \
  }
#define CJT_INV(V)                                                                               \
  case V:                                                                                        \
    if (fold) CJT_INV_F(V, true) else CJT_INV_F(V, false)                                       \
    break;
    case 128: CJT_INV_F(128, false) break;
    CJT_INV(64) CJT_INV(32) CJT_INV(24) CJT_INV(16)
#undef CJT_INV
#undef CJT_INV_F
    default: return fail(CJT_EINVAL, "bad vector tile");
  }
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}


int launch_pgen_fwd(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                    const double2* ck, const int2* blk_tj, int64_t nblk, double* P, bool fold,
                    cudaStream_t st) {
  if (nblk <= 0) return CJT_OK;
  const int64_t grid = std::min<int64_t>(nblk, 148 * 16);
  k_pgen_fwd<<<(unsigned)grid, 128, 0, st>>>(rows, tab, ck_off, ck, blk_tj, nblk, P, fold ? 1 : 0);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_pgen_inv(const RecTablesDev& tab, const void* gen, const int32_t* gn0, int64_t gbeg,
                    int64_t gend, double* P, cudaStream_t st) {
  if (gend <= gbeg) return CJT_OK;
  const int64_t grid = std::min<int64_t>(gend - gbeg, 148 * 16);
  k_pgen_inv<<<(unsigned)grid, 128, 0, st>>>(tab, (const GenState*)gen, gn0, gbeg, gend, P);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_rec_gemm(const GemmItem* items, int64_t n_items, const double* P, const int32_t* ids,
                    const double* x, int64_t ldx, int64_t xlen, int64_t batch, int vt, bool amk,
                    bool fold, double* part, cudaStream_t st) {
  if (n_items <= 0 || batch <= 0) return CJT_OK;
  dim3 grid((unsigned)((batch + vt - 1) / vt), (unsigned)n_items);
#define CJT_GEMM(V, M, F)                                                                        \
  if (vt == V && amk == M && fold == F) {                                                        \
    using Cf = GemmCfg<V, M>;                                                                    \
    static DeviceOnce once_;                                                                    \
    if (int rc_ = once_([&]() -> int {                                                                                 \
      CJT_CUDA_TRY(cudaFuncSetAttribute(k_rec_gemm<V, M, F>,                                     \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM)); \
      return CJT_OK;                                                                               \
    })) return rc_;                                                                                            \
    k_rec_gemm<V, M, F><<<grid, Cf::NTH, Cf::SMEM, st>>>(items, P, ids, x, ldx, xlen, batch, part); \
    CJT_CUDA_TRY(cudaGetLastError());                                                            \
    return CJT_OK;                                                                               \
  }
  CJT_GEMM(128, false, false) CJT_GEMM(64, false, false) CJT_GEMM(32, false, false) CJT_GEMM(16, false, false)
  CJT_GEMM(128, true, false) CJT_GEMM(64, true, false) CJT_GEMM(32, true, false) CJT_GEMM(16, true, false)
  CJT_GEMM(64, false, true)
#undef CJT_GEMM
  return fail(CJT_EINVAL, "bad vector tile");
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
                           int64_t ldc, const double* x, const double* xm, const int8_t* reg,
                           const int64_t* cut, double* out, int64_t ldo, int64_t npts,
                           int64_t batch, bool divide, cudaStream_t st) {
  if (npts <= 0 || batch <= 0) return CJT_OK;
  if (batch > 65535) return fail(CJT_EINVAL, "clenshaw batch must be <= 65535 per call");
  const int T = 128;
  dim3 grid((unsigned)((npts + T - 1) / T), (unsigned)batch);
  auto kern = divide ? k_clenshaw_points<true> : k_clenshaw_points<false>;
  kern<<<grid, T, 0, st>>>(tab, rbp, rbm, rbpi, rbmi, coeffs, ldc, x, xm, reg, cut, out, ldo, npts);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_jacobi_values(const RecTablesDev& tab, int64_t n_max, const double* x, const double* xm,
                         const int8_t* mode, double* out, int64_t npts, cudaStream_t st) {
  if (npts <= 0) return CJT_OK;
  const int T = 128;
  k_jacobi_values<<<(unsigned)((npts + T - 1) / T), T, 0, st>>>(tab, n_max, x, xm, mode, out, npts);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

}  // namespace cjt
