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
//   2^14 <= L <= 2^17: one thread-block cluster of P CTAs per vector; each CTA
//              holds Q = L/P points in shared memory (decimated n = r + P n2),
//              runs a local Q-point FFT, and the P-point DFTs across the
//              cluster, the spectrum product and the inverse P-point DFTs run
//              over distributed shared memory, followed by the local inverse
//              FFT: the whole Bluestein product stays on chip.
//   L >  2^17: three passes of a four-step FFT (L = L1 x L2): column FFTs with
//              the input diagonal fused into the load and the inter-step
//              twiddle into the store; row FFT -> spectrum product -> row
//              inverse FFT fused in one pass; column inverse FFTs with the
//              output diagonal and the sum over m fused into the store.
#include <cooperative_groups.h>
#include <climits>
#include <cstdlib>

#include "cjt_internal.cuh"

namespace cjt {

namespace {

template <int LOGL>
struct FusedCfg {
  static constexpr int L = 1 << LOGL;
#ifndef CJT_FUSED13_TWSMEM
#define CJT_FUSED13_TWSMEM 0
#endif
#ifndef CJT_FUSED13_LEPT
#define CJT_FUSED13_LEPT 4
#endif
  // 8192 with radix-16 passes: 512 threads (16 warps) hide the global-load
  // latency of the fused first / last passes better than radix-32 with 8 warps
  static constexpr int LEPT = LOGL == 13 ? CJT_FUSED13_LEPT : 4;
  static constexpr int EPT = 1 << LEPT;             // elements per thread
#ifndef CJT_FUSED_LOGEMIN
#define CJT_FUSED_LOGEMIN 12
#endif
  static constexpr int EMIN = 1 << CJT_FUSED_LOGEMIN;
  static constexpr int E = (L >= EMIN) ? L : EMIN;  // complex elements per CTA
  static constexpr int NG = E / L;                  // vectors per CTA
  static constexpr int T = E / EPT;                 // threads per CTA
  // (build option, off: 8192-point tiles with the shared-memory twiddle table;
  // the packed global tables' coalesced loads win although only ~23 KB of L1
  // remain next to the FFT buffer and accumulator)
  static constexpr bool TW_SMEM = CJT_FUSED13_TWSMEM && LOGL == 13;
  static constexpr int SMEM = NG * padded_len(L) * 16 + E * 8 + (TW_SMEM ? 1024 * 16 : 0);
};

// Schedule of a fused chirp-z launch.  Work unit u = (vector group, output
// tile j, term m), u = (grp * n_out + j) * M + m; each unit is n_in forward
// FFTs (one per input tile, spectra summed) and one inverse FFT.
//   direct:   grid (groups, n_out), one CTA per (grp, j) runs all m and
//             accumulates the output tile in shared memory;
//   stream-K: P CTAs each take a contiguous range of the F = U * n_in
//             forward FFTs (f -> unit f / n_in, tile f % n_in); a unit cut by
//             a range boundary is finished by each CTA on its part (one extra
//             inverse FFT).  Every (CTA, unit) segment writes its output tile
//             to a partial slot; a fixed-order combine sums slots and terms
//             (deterministic).  Removes the wave-quantisation tail of small
//             grids (e.g. 448 CTAs on 148 SMs at one CTA per SM).
struct FusedSched {
  int streamk;       // 0: direct
  int64_t U, F;      // units, forward FFTs
  int64_t P;         // CTAs (stream-K)
  int64_t S;         // partial slots per CTA (stream-K)
  __host__ __device__ int64_t start(int64_t c) const { return F * c / P; }
  // CTA whose range holds forward FFT f
  __host__ __device__ int64_t cta_of(int64_t f) const { return ((f + 1) * P + F - 1) / F - 1; }
};

// two-level FFT (Fft2) for L >= 512; khat and the spectrum sums are then in
// the permuted order p = k1 S + k2 <-> natural k1 + 16 k2 (capi permutes khat)
template <int LOGL>
__host__ __device__ constexpr bool fused_fft2() { return fft2_used(LOGL); }

template <int LOGL, bool MULTI, class TW, class Sink>
__device__ __forceinline__ void fused_unit2(const ChirpZDev& cz, const TW& tw, double2* s, int t,
                                            bool valid, const double* xb, int j, int m, int ti0,
                                            int ti1, double2* specb, const Sink& sink) {
  using F = Fft2<LOGL>;
  constexpr int L = F::L;
  const double2* pre = cz.pre + (int64_t)m * cz.width;
  const int k1 = t / F::TPS;
  double2* reg = s + k1 * F::PS;
  double2* spr = specb ? specb + k1 * F::S : nullptr;
  for (int ti = ti0; ti < ti1; ++ti) {
    const int64_t to = cz.tin[2 * ti], tn = cz.tin[2 * ti + 1];
    auto load_x = [&](int e) -> double2 {
      if (valid && e < tn) {
        const double xv = __ldg(xb + to + e);
        const double2 p = __ldg(pre + to + e);
        return make_double2(xv * p.x, xv * p.y);
      }
      return make_double2(0.0, 0.0);
    };
    __syncthreads();   // previous readers of s are done
    fft2_first<LOGL>(s, t, tw, load_x);
    __syncthreads();
    const double2* kh = cz.khat + ((int64_t)j * cz.n_in + ti) * L + k1 * F::S;
    if constexpr (MULTI) {
      // spectrum product summed over the unit's tiles: running sum in spec
      // (L2), the last tile writes the total into shared memory
      const bool first = ti == ti0, last = ti == ti1 - 1;
      auto store_spec = [&](int e, double2 v) {
        double2 y = cmul(v, __ldg(kh + e));
        if (!first && valid) {
          const double2 a = __ldcg(spr + e);
          y.x += a.x;
          y.y += a.y;
        }
        if (last)
          reg[pad16(e)] = y;
        else if (valid)
          __stcg(spr + e, y);
      };
      fft2_sub<LOGL, -1>(s, t, tw, SmemLoad{reg}, store_spec);
    } else {
      // single-tile units: forward sub-FFT, spectrum product, inverse sub-FFT
      // with the forward's last pass and the inverse's first pass fused in
      // registers (a separate instantiation from the multi-tile code)
      auto spec_op = [&](int e, double2 v) -> double2 { return cmul(v, __ldg(kh + e)); };
      sub_conv<F::LOGS>(reg, t % F::TPS, tw, spec_op);
    }
  }
  if constexpr (MULTI) fft2_sub<LOGL, +1>(s, t, tw, SmemLoad{reg}, SmemStore{reg});
  __syncthreads();
  const int64_t so = cz.tout[2 * j], sc = cz.tout[2 * j + 1];
  const double2* post = cz.post + (int64_t)m * cz.count + so;
  auto store_out = [&](int e, double2 y) {
    if (e < sc) {
      const double2 q = __ldg(post + e);
      sink(e, fma(q.x, y.x, -q.y * y.y));
    }
  };
  fft2_last_inv<LOGL>(s, t, tw, store_out);
}

template <int LOGL, bool MULTI, class TW, class Sink>
__device__ __forceinline__ void fused_unit(const ChirpZDev& cz, const TW& tw, double2* s, int t,
                                           bool valid, const double* xb, int j, int m, int ti0,
                                           int ti1, double2* specb, const Sink& sink) {
  if constexpr (fused_fft2<LOGL>()) {
    fused_unit2<LOGL, MULTI>(cz, tw, s, t, valid, xb, j, m, ti0, ti1, specb, sink);
    return;
  }
  using Cfg = FusedCfg<LOGL>;
  constexpr int L = Cfg::L;
  const double2* pre = cz.pre + (int64_t)m * cz.width;
  for (int ti = ti0; ti < ti1; ++ti) {
    const int64_t to = cz.tin[2 * ti], tn = cz.tin[2 * ti + 1];
    // forward FFT straight from global: x * pre (zero padded)
    auto load_x = [&](int e) -> double2 {
      if (valid && e < tn) {
        const double xv = __ldg(xb + to + e);
        const double2 p = __ldg(pre + to + e);
        return make_double2(xv * p.x, xv * p.y);
      }
      return make_double2(0.0, 0.0);
    };
    // spectrum product fused into the last pass.  Input tiles are summed in
    // the frequency domain (one inverse FFT per unit, not per input tile):
    // the running sum lives in the L2-resident spec buffer, each element
    // owned by one thread (the last pass's output positions are fixed), and
    // the final tile writes the total into shared memory.
    const double2* kh = cz.khat + ((int64_t)j * cz.n_in + ti) * L;
    const bool first = ti == ti0, last = ti == ti1 - 1;
    auto store_spec = [&](int e, double2 v) {
      double2 y = cmul(v, __ldg(kh + e));
      if (!first && valid) {
        const double2 a = __ldcg(specb + e);
        y.x += a.x;
        y.y += a.y;
      }
      if (last)
        s[pad16(e)] = y;
      else if (valid)
        __stcg(specb + e, y);
    };
    fft_smem_io<LOGL, -1, decltype(load_x), decltype(store_spec), Cfg::LEPT>(s, t, tw, load_x, store_spec);
  }
  // inverse FFT: output diagonal fused into the last pass, value to the sink
  const int64_t so = cz.tout[2 * j], sc = cz.tout[2 * j + 1];
  const double2* post = cz.post + (int64_t)m * cz.count + so;
  auto store_out = [&](int e, double2 y) {
    if (e < sc) {
      const double2 q = __ldg(post + e);
      sink(e, fma(q.x, y.x, -q.y * y.y));
    }
  };
  fft_smem_io<LOGL, +1, SmemLoad, decltype(store_out), Cfg::LEPT>(s, t, tw, SmemLoad{s}, store_out);
}

template <int LOGL, bool MULTI, class TW>
__device__ __forceinline__ void fused_direct(const ChirpZDev& cz, const TW& tw, double2* s, double* acc,
                                             int t, int grp, const double* __restrict__ x, int64_t ldx,
                                             double* __restrict__ out, int64_t ldo, int64_t batch,
                                             double2* __restrict__ spec) {
  using Cfg = FusedCfg<LOGL>;
  constexpr int L = Cfg::L;
  constexpr int TPG = L / Cfg::EPT;
  const int64_t b = (int64_t)blockIdx.x * Cfg::NG + grp;
  const bool valid = b < batch;
  const double* xb = x + (valid ? b : 0) * ldx + cz.p0;
  const int j = blockIdx.y;
  const int64_t so = cz.tout[2 * j], sc = cz.tout[2 * j + 1];
  double2* specb = (cz.n_in > 1 && valid) ? spec + ((int64_t)blockIdx.x * gridDim.y + j) * Cfg::NG * L +
                                                 (int64_t)grp * L
                                          : nullptr;
#pragma unroll
  for (int i = 0; i < Cfg::EPT; ++i) acc[t + i * TPG] = 0.0;
  auto sink = [&](int e, double v) { acc[e] += v; };
  for (int m = 0; m < cz.m_count; ++m) fused_unit<LOGL, MULTI>(cz, tw, s, t, valid, xb, j, m, 0, cz.n_in, specb, sink);
  __syncthreads();
  if (!valid) return;
  double* ob = out + b * ldo + cz.qout + so;
#pragma unroll
  for (int i = 0; i < Cfg::EPT; ++i) {
    const int e = t + i * TPG;
    if (e < sc) ob[e] = cz.accumulate ? ob[e] + acc[e] : acc[e];
  }
}

template <int LOGL, bool MULTI, class TW>
__device__ __forceinline__ void fused_streamk(const ChirpZDev& cz, const TW& tw, double2* s, double* acc,
                                              int t, int grp, const double* __restrict__ x, int64_t ldx,
                                              int64_t batch, double* __restrict__ part,
                                              double2* __restrict__ spec, const FusedSched& sk) {
  using Cfg = FusedCfg<LOGL>;
  constexpr int L = Cfg::L;
  constexpr int TPG = L / Cfg::EPT;
  const int64_t c = blockIdx.x;
  const int64_t f0 = sk.start(c), f1 = sk.start(c + 1);
  const int M = cz.m_count;
  const int64_t gj_first = f0 / cz.n_in / M;
  double2* specb = spec ? spec + (c * Cfg::NG + grp) * L : nullptr;
  // the output tile of one (group, j) accumulates over its terms m in shared
  // memory and is written once per (CTA, (group, j)) segment
#pragma unroll
  for (int i = 0; i < Cfg::EPT; ++i) acc[t + i * TPG] = 0.0;
  auto flush = [&](int64_t gj) {
    __syncthreads();
    const int j = (int)(gj % cz.n_out);
    const int64_t b = gj / cz.n_out * Cfg::NG + grp;
    const int64_t sc = cz.tout[2 * j + 1];
    double* slot = part + (((c * sk.S + (gj - gj_first)) * Cfg::NG) + grp) * cz.count_max;
#pragma unroll
    for (int i = 0; i < Cfg::EPT; ++i) {
      const int e = t + i * TPG;
      if (e < sc && b < batch) slot[e] = acc[e];
      acc[e] = 0.0;
    }
  };
  int64_t cur = f0 / cz.n_in / M;
  for (int64_t f = f0; f < f1;) {
    const int64_t u = f / cz.n_in;
    const int ti0 = (int)(f % cz.n_in);
    const int ti1 = (int)min((int64_t)cz.n_in, (int64_t)ti0 + (f1 - f));
    const int64_t gj = u / M;
    const int m = (int)(u % M);
    if (gj != cur) {
      flush(cur);
      cur = gj;
    }
    const int64_t g = gj / cz.n_out;
    const int j = (int)(gj % cz.n_out);
    const int64_t b = g * Cfg::NG + grp;
    const bool valid = b < batch;
    const double* xb = x + (valid ? b : 0) * ldx + cz.p0;
    auto sink = [&](int e, double v) { acc[e] += v; };
    fused_unit<LOGL, MULTI>(cz, tw, s, t, valid, xb, j, m, ti0, ti1, specb, sink);
    f += ti1 - ti0;
  }
  flush(cur);
}

// grid: direct (groups, n_out) or stream-K (P); see FusedSched.
template <int LOGL, bool MULTI>
__global__ void __launch_bounds__(FusedCfg<LOGL>::T, (LOGL <= 12) ? 512 / FusedCfg<LOGL>::T : 1)
    k_chirpz_fused(ChirpZDev cz, const double2* __restrict__ tw, const double* __restrict__ x,
                   int64_t ldx, double* __restrict__ out, int64_t ldo, int64_t batch,
                   double* __restrict__ part, double2* __restrict__ spec, FusedSched sk) {
  using Cfg = FusedCfg<LOGL>;
  constexpr int L = Cfg::L;
  constexpr int TPG = L / Cfg::EPT;
  extern __shared__ double2 smem[];
  const int grp = threadIdx.x / TPG;
  const int t = threadIdx.x % TPG;
  double2* s = smem + grp * padded_len(L);
  double* acc = reinterpret_cast<double*>(smem + Cfg::NG * padded_len(L)) + grp * L;
  if constexpr (Cfg::TW_SMEM) {
    const TwSmem tws = tw_smem_init(reinterpret_cast<double2*>(acc + Cfg::E), tw);
    if (sk.streamk)
      fused_streamk<LOGL, MULTI>(cz, tws, s, acc, t, grp, x, ldx, batch, part, spec, sk);
    else
      fused_direct<LOGL, MULTI>(cz, tws, s, acc, t, grp, x, ldx, out, ldo, batch, spec);
  } else {
    if (sk.streamk)
      fused_streamk<LOGL, MULTI>(cz, tw, s, acc, t, grp, x, ldx, batch, part, spec, sk);
    else
      fused_direct<LOGL, MULTI>(cz, tw, s, acc, t, grp, x, ldx, out, ldo, batch, spec);
  }
}

// stream-K combine: out[b][q0 + so_j + e] (+)= sum over the CTAs whose
// ranges cover (group, j) of their slot for it (fixed order).
// grid (e chunks, n_out, batch).
__global__ void __launch_bounds__(256) k_chirpz_combine_sk(ChirpZDev cz, const double* __restrict__ part,
                                                           FusedSched sk, int ng, double* __restrict__ out,
                                                           int64_t ldo) {
  const int j = blockIdx.y;
  const int64_t b = blockIdx.z;
  const int64_t g = b / ng, gi = b % ng;
  const int64_t so = __ldg(cz.tout + 2 * j), sc = __ldg(cz.tout + 2 * j + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= sc) return;
  const int64_t gj = g * cz.n_out + j;
  const int64_t per_gj = (int64_t)cz.m_count * cz.n_in;   // forward FFTs of one (group, j)
  const int64_t ca = sk.cta_of(gj * per_gj), cb = sk.cta_of(gj * per_gj + per_gj - 1);
  const int64_t stride = (int64_t)ng * cz.count_max;
  const double* pe = part + gi * cz.count_max + e;
  // the first CTA may hold earlier segments (slot k_a); every later one
  // starts inside this (group, j) and holds it in its slot 0
  const int64_t ka = gj - sk.start(ca) / cz.n_in / cz.m_count;
  double v = pe[(ca * sk.S + ka) * stride];
  for (int64_t c = ca + 1; c <= cb; ++c) v += pe[c * sk.S * stride];
  double* o = out + b * ldo + cz.qout + so + e;
  *o = cz.accumulate ? *o + v : v;
}

// W_L^t = exp(-2 pi i t / L) from the two-level table (t < L)
__device__ __forceinline__ double2 twiddle_L(const ChirpZDev& cz, int64_t t) {
  return cmul(__ldg(cz.tw_hi + (t >> 12)), __ldg(cz.tw_lo + (t & 4095)));
}

template <int LOGQ, int P>
struct ClusterCfg {
  static constexpr int Q = 1 << LOGQ;
  static constexpr int T = Q / 16;
  static constexpr int SMEM = padded_len(Q) * 16 + Q * 8;   // FFT buffer + output accumulator
};

template <int LOGQ, int P>
__global__ void __launch_bounds__(ClusterCfg<LOGQ, P>::T, 1)
    k_chirpz_cluster(ChirpZDev cz, const double2* __restrict__ tw, const double* __restrict__ x,
                     int64_t ldx, double* __restrict__ out, int64_t ldo) {
  namespace cg = cooperative_groups;
  using Cfg = ClusterCfg<LOGQ, P>;
  constexpr int Q = Cfg::Q, T = Cfg::T, NCOL = 16 / P;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double2 smem[];
  double2* s = smem;
  double* acc = reinterpret_cast<double*>(smem + padded_len(Q));  // [Q], thread-private slots
  const int r = (int)cluster.block_rank();   // n1: this CTA's residue class
  const int64_t b = blockIdx.x / P;
  const int t = threadIdx.x;
  const double* xb = x + b * ldx + cz.p0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[t + i * T] = 0.0;

  for (int m = 0; m < cz.m_count; ++m) {
    const double2* pre = cz.pre + (int64_t)m * cz.width;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n2 = t + i * T;
      const int64_t pidx = r + (int64_t)P * n2;
      double2 v = make_double2(0.0, 0.0);
      if (pidx < cz.width) {
        const double xv = __ldg(xb + pidx);
        const double2 pp = __ldg(pre + pidx);
        v = make_double2(xv * pp.x, xv * pp.y);
      }
      s[pad16(n2)] = v;
    }
    __syncthreads();
    fft_smem<LOGQ, -1>(s, t, tw);
    if (r > 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k2 = t + i * T;
        s[pad16(k2)] = cmul(s[pad16(k2)], twiddle_L(cz, (int64_t)r * k2));
      }
    }
    cluster.sync();
    // P-point DFT across the cluster, spectrum product, inverse P-point DFT
#pragma unroll
    for (int j = 0; j < NCOL; ++j) {
      const int k2 = r * (Q / P) + t + j * T;
      double2 v[P];
#pragma unroll
      for (int q = 0; q < P; ++q) v[q] = cluster.map_shared_rank(s, q)[pad16(k2)];
      dft_reg<P, -1>(v);
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) v[k1] = cmul(v[k1], __ldg(cz.khat + k2 + (int64_t)Q * k1));
      dft_reg<P, +1>(v);
#pragma unroll
      for (int q = 0; q < P; ++q) cluster.map_shared_rank(s, q)[pad16(k2)] = v[q];
    }
    cluster.sync();
    if (r > 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k2 = t + i * T;
        double2 w = twiddle_L(cz, (int64_t)r * k2);
        w.y = -w.y;
        s[pad16(k2)] = cmul(s[pad16(k2)], w);
      }
    }
    __syncthreads();
    fft_smem<LOGQ, +1>(s, t, tw);
    const double2* post = cz.post + (int64_t)m * cz.count;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n2 = t + i * T;
      const int64_t sidx = r + (int64_t)P * n2;
      if (sidx < cz.count) {
        const double2 y = s[pad16(n2)];
        const double2 q = __ldg(post + sidx);
        acc[n2] += fma(q.x, y.x, -q.y * y.y);
      }
    }
  }
  double* ob = out + b * ldo + cz.qout;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int n2 = t + i * T;
    const int64_t sidx = r + (int64_t)P * n2;
    if (sidx < cz.count) ob[sidx] = cz.accumulate ? ob[sidx] + acc[n2] : acc[n2];
  }
}

// (build option, off: column FFT twiddles from the shared-memory table, see CJT_ROWS_TWSMEM)
#ifndef CJT_COLS_TWSMEM
#define CJT_COLS_TWSMEM 0
#endif
template <int LOG1>
struct ColCfg {
  static constexpr int L1 = 1 << LOG1;
#ifndef CJT_COLS_EMIN
#define CJT_COLS_EMIN 2048
#endif
  static constexpr int E = (L1 >= CJT_COLS_EMIN) ? L1 : CJT_COLS_EMIN;   // complex elements per CTA
  static constexpr int NC = E / L1;                  // columns per CTA
  static constexpr int T = E / 16;
  static constexpr int CS = padded_len(L1) + 1;      // odd column stride (conflict-free transpose)
  // + per-thread four-step twiddles (W_L^{n2 k1_0}, W_L^{n2 T/NC}), looked up once for all terms
  static constexpr int TWO = NC * CS + (CJT_COLS_TWSMEM ? 1024 : 0);   // offset (double2) of that table
  static constexpr int SMEM = (TWO + 2 * T) * 16;
};

// pass 1: x (real slice) * pre_m -> column FFTs over n1 -> * W_L^{n2 k1} -> buf[b][m][k1][n2]
template <int LOG1>
__global__ void __launch_bounds__(ColCfg<LOG1>::T, (ColCfg<LOG1>::T >= 512) ? 1 : 512 / ColCfg<LOG1>::T)
    k_chirpz_cols_fwd(ChirpZDev cz, const double2* __restrict__ twg, const double* __restrict__ x,
                      int64_t ldx, double2* __restrict__ buf) {
  using Cfg = ColCfg<LOG1>;
  constexpr int L1 = Cfg::L1, NC = Cfg::NC, T = Cfg::T, CS = Cfg::CS;
  extern __shared__ double2 smem[];
#if CJT_COLS_TWSMEM
  const TwSmem tw = tw_smem_init(smem + NC * CS, twg);
#else
  const double2* tw = twg;
#endif
  const int64_t L2 = (int64_t)1 << cz.log2;
  const int64_t L = cz.length;
  // consecutive CTAs share a column tile across vectors: the pre table stays in L2
  const int64_t c0 = (int64_t)blockIdx.y * NC;
  const int64_t b = blockIdx.x;
  // input tile blockIdx.z (tiled multi-pass): columns of x[to .. to + tn)
  const int64_t to = __ldg(cz.tin + 2 * blockIdx.z), tn = __ldg(cz.tin + 2 * blockIdx.z + 1);
  const int nslot = max(cz.n_in, cz.n_out);
  const double* xb = x + b * ldx + cz.p0 + to;
  const int grp = threadIdx.x / (L1 / 16);
  const int t = threadIdx.x % (L1 / 16);
  // this thread's column n2 is fixed and k1 = k1_0 + i T/NC: twiddles
  // W_L^{n2 k1} by a running product from two table values, looked up once
  // for all terms (scattered loads: one cache line per lane)
  // (kept in shared memory: eight more live registers across the FFT spill)
  double2* tws = smem + Cfg::TWO + 2 * threadIdx.x;
  tws[0] = twiddle_L(cz, (c0 + threadIdx.x % NC) * (threadIdx.x / NC));
  tws[1] = twiddle_L(cz, (c0 + threadIdx.x % NC) * (T / NC));
  for (int m = 0; m < cz.m_count; ++m) {
    const double2* pre = cz.pre + (int64_t)m * cz.width + to;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int idx = threadIdx.x + i * T;
      const int c = idx % NC, n1 = idx / NC;
      const int64_t pidx = (int64_t)n1 * L2 + c0 + c;
      double2 v = make_double2(0.0, 0.0);
      if (pidx < tn) {
        const double xv = __ldg(xb + pidx);
        const double2 p = __ldg(pre + pidx);
        v = make_double2(xv * p.x, xv * p.y);
      }
      smem[c * CS + pad16(n1)] = v;
    }
    __syncthreads();
    fft_smem<LOG1, -1, 4, FftSync<LOG1, 4>>(smem + grp * CS, t, tw);
    __syncthreads();   // the transposed store reads other warps' columns
    double2* bm = buf + ((b * cz.m_count + m) * nslot + blockIdx.z) * L;
    const int c = threadIdx.x % NC;
    const int64_t n2 = c0 + c;
    const int k10 = threadIdx.x / NC;
    double2 w = tws[0];
    const double2 ws = tws[1];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k1 = k10 + i * (T / NC);
      bm[(int64_t)k1 * L2 + n2] = cmul(smem[c * CS + pad16(k1)], w);
      w = cmul(w, ws);
    }
    __syncthreads();
  }
}

// Short columns (L1 <= 32): one thread per column n2, the L1-point DFT in
// registers -- no shared memory, no barriers; x and the twiddles W_L^{n2 k1}
// are loaded once and reused for every term m.  Loads and stores of
// consecutive threads are consecutive n2 (coalesced).
constexpr int COLR_T = 128;

// W_L^{n2 k}, k < R, from W_L^{n2 2^j} (at most three rounded products each)
template <int R>
__device__ __forceinline__ void column_twiddles(const ChirpZDev& cz, int64_t n2, double2* w) {
  w[0] = make_double2(1.0, 0.0);
  // W_L^{n2 2^p} from the per-length column table: consecutive threads read
  // consecutive entries (the two-level table costs a cache line per lane)
  const int64_t L2 = (int64_t)1 << cz.log2;
#pragma unroll
  for (int j = 1, p = 0; j < R; j <<= 1, ++p) w[j] = __ldg(cz.tw_col + p * L2 + n2);
#pragma unroll
  for (int k = 3; k < R; ++k) {
    if ((k & (k - 1)) != 0) {
      const int hi = 1 << (31 - __clz(k));
      w[k] = cmul(w[hi], w[k - hi]);
    }
  }
}

template <int LOG1>
__global__ void __launch_bounds__(COLR_T, (LOG1 <= 4) ? 4 : 1)
    k_chirpz_cols_fwd_reg(ChirpZDev cz, const double* __restrict__ x, int64_t ldx,
                          double2* __restrict__ buf) {
  constexpr int L1 = 1 << LOG1;
  const int64_t L2 = (int64_t)1 << cz.log2;
  const int64_t L = cz.length;
  const int64_t n2 = (int64_t)blockIdx.y * COLR_T + threadIdx.x;
  const int64_t b = blockIdx.x;
  // blockIdx.z = (input tile, term): x[to .. to + tn) * pre_m -> slot (m, tile);
  // one term per thread keeps the kernel at 4 CTAs / SM (x and the twiddles
  // are re-read / recomputed per term from L2 instead of held for all terms)
  const int m = (int)(blockIdx.z % cz.m_count);
  const int tile = (int)(blockIdx.z / cz.m_count);
  const int64_t to = __ldg(cz.tin + 2 * tile), tn = __ldg(cz.tin + 2 * tile + 1);
  const int nslot = max(cz.n_in, cz.n_out);
  const double* xb = x + b * ldx + cz.p0 + to;
  double xv[L1];
#pragma unroll
  for (int r = 0; r < L1; ++r) {
    const int64_t pidx = r * L2 + n2;
    xv[r] = pidx < tn ? __ldg(xb + pidx) : 0.0;
  }
  double2 w[L1];
  column_twiddles<L1>(cz, n2, w);
  {
    const double2* pre = cz.pre + (int64_t)m * cz.width + to;
    double2 v[L1];
#pragma unroll
    for (int r = 0; r < L1; ++r) {
      const int64_t pidx = r * L2 + n2;
      const double2 p = pidx < tn ? __ldg(pre + pidx) : make_double2(0.0, 0.0);
      v[r] = make_double2(xv[r] * p.x, xv[r] * p.y);
    }
    dft_reg<L1, -1>(v);
    double2* bm = buf + ((b * cz.m_count + m) * nslot + tile) * L + n2;
#pragma unroll
    for (int k = 0; k < L1; ++k) bm[k * L2] = cmul(v[k], w[k]);
  }
}

template <int LOG1>
__global__ void __launch_bounds__(COLR_T, (LOG1 <= 4) ? 4 : 1)
    k_chirpz_cols_inv_reg(ChirpZDev cz, const double2* __restrict__ buf, double* __restrict__ out,
                          int64_t ldo) {
  constexpr int L1 = 1 << LOG1;
  const int64_t L2 = (int64_t)1 << cz.log2;
  const int64_t L = cz.length;
  const int64_t n2 = (int64_t)blockIdx.y * COLR_T + threadIdx.x;
  const int64_t b = blockIdx.x;
  // output tile blockIdx.z (tiled multi-pass): slot blockIdx.z -> out[so .. so + sc)
  const int64_t so = __ldg(cz.tout + 2 * blockIdx.z), sc = __ldg(cz.tout + 2 * blockIdx.z + 1);
  const int nslot = max(cz.n_in, cz.n_out);
  double acc[L1];
#pragma unroll
  for (int r = 0; r < L1; ++r) acc[r] = 0.0;
  // per term: the column and the output diagonal are loaded together (one
  // latency per term); the twiddle W_L^{-n2 k1} was applied by the row pass
  const double2* bcol = buf + (b * cz.m_count * nslot + blockIdx.z) * L + n2;
  for (int m = 0; m < cz.m_count; ++m) {
    const double2* post = cz.post + (int64_t)m * cz.count + so;
    double2 v[L1], pq[L1];
#pragma unroll
    for (int k = 0; k < L1; ++k) v[k] = __ldcs(bcol + (int64_t)m * nslot * L + k * L2);
#pragma unroll
    for (int r = 0; r < L1; ++r) {
      const int64_t q = r * L2 + n2;
      pq[r] = q < sc ? __ldg(post + q) : make_double2(0.0, 0.0);
    }
    dft_reg<L1, +1>(v);
#pragma unroll
    for (int r = 0; r < L1; ++r) acc[r] += fma(pq[r].x, v[r].x, -pq[r].y * v[r].y);
  }
  double* ob = out + b * ldo + cz.qout + so;
#pragma unroll
  for (int r = 0; r < L1; ++r) {
    const int64_t q = r * L2 + n2;
    if (q < sc) ob[q] = cz.accumulate ? ob[q] + acc[r] : acc[r];
  }
}

// (build option, off: row FFT twiddles from a 1024-entry shared-memory table
// (TwSmem).  It was the answer to the 8192-entry global table's scattered
// per-lane loads, but its strided reads are 8-way bank conflicts; the packed
// per-period tables (tw_pow, cjt_internal.cuh) are coalesced and faster)
#ifndef CJT_ROWS_TWSMEM
#define CJT_ROWS_TWSMEM 0
#endif
template <int LOG2>
struct RowCfg {
  static constexpr int L2 = 1 << LOG2;
  static constexpr int LEPT = (LOG2 == 13 && !fft2_used(LOG2)) ? 5 : 4;   // Fft2: 16 per thread
  static constexpr int EPT = 1 << LEPT;
#ifndef CJT_ROWS_EMIN
#define CJT_ROWS_EMIN 1024
#endif
  static constexpr int E = (L2 >= CJT_ROWS_EMIN) ? L2 : CJT_ROWS_EMIN;   // complex elements per CTA
  static constexpr int NR = E / L2;
  static constexpr int T = E / EPT;
  // (4096 / 8192-point rows only: A/B on configs 2, 4, 5 -- the 1024 / 2048
  // rows of config 2 lose ~1.5 %, the longer rows of configs 4 / 5 gain 1-3 %)
  static constexpr bool TWS = CJT_ROWS_TWSMEM && LOG2 >= 12;
  static constexpr int SMEM = NR * padded_len(L2) * 16 + (TWS ? 1024 * 16 : 0);
};

// pass 2: rows k1 of buf: FFT over n2 -> * khat[k1][k2] -> inverse FFT over k2
// (global load fused into the first forward pass, the spectrum product into
// the first inverse pass, the global store into the last inverse pass).
// Tiled multi-pass (n_in > 1 or n_out > 1; slots s < max(n_in, n_out) per
// (vector, term) in buf):
//   input tiles:  the row FFTs of slots 0..n_in-1 are multiplied by their
//                 spectra and summed (running sum in slot 0, each element
//                 owned by one thread), one inverse FFT -> slot 0;
//   output tiles: one forward FFT, its spectrum kept in slot n_out-1; per
//                 output tile j, spectrum * khat_j -> inverse FFT -> slot j.
template <int LOG2, int TM, class TW>
__device__ __forceinline__ void rows_impl(ChirpZDev cz, const TW& tw, double2* __restrict__ buf,
                                          double2* smem);

// TM (tiling mode): 0 untiled, 1 input tiles, 2 output tiles (separate
// instantiations keep the untiled kernel's register allocation unchanged)
#ifndef CJT_ROWS_MINB
#define CJT_ROWS_MINB 2
#endif
#ifndef CJT_ROWS12_MINB
#define CJT_ROWS12_MINB 2
#endif
template <int LOG2, int TM>
__global__ void __launch_bounds__(RowCfg<LOG2>::T, (LOG2 <= 11) ? CJT_ROWS_MINB * 256 / RowCfg<LOG2>::T : (LOG2 <= 12) ? CJT_ROWS12_MINB : 1)
    k_chirpz_rows(ChirpZDev cz, const double2* __restrict__ twg, double2* __restrict__ buf) {
  using Cfg = RowCfg<LOG2>;
  extern __shared__ double2 smem[];
  if constexpr (Cfg::TWS)
    rows_impl<LOG2, TM>(cz, tw_smem_init(smem + Cfg::NR * padded_len(Cfg::L2), twg), buf, smem);
  else
    rows_impl<LOG2, TM>(cz, twg, buf, smem);
}

template <int LOG2, int TM, class TW>
__device__ __forceinline__ void rows_impl(ChirpZDev cz, const TW& tw, double2* __restrict__ buf,
                                          double2* smem) {
  using Cfg = RowCfg<LOG2>;
  constexpr int L2 = Cfg::L2, NR = Cfg::NR;
  constexpr int TPG = L2 / Cfg::EPT;
  const int grp = threadIdx.x / TPG;
  const int t = threadIdx.x % TPG;
  // consecutive CTAs share spectrum rows across (vector, term): khat stays in L2
  const int64_t k1 = (int64_t)blockIdx.y * NR + grp;
  const int64_t L = cz.length;
  const int nslot = max(cz.n_in, cz.n_out);
  double2* row = buf + (int64_t)blockIdx.x * nslot * L + k1 * L2;   // slot s: row + s L
  const double2* kh = cz.khat + k1 * L2;                             // tile (j, i): kh + (j n_in + i) L
  double2* s = smem + grp * padded_len(L2);
  if constexpr (fft2_used(LOG2)) {
    // two-level FFT: khat rows are in the permuted order (capi)
    using F = Fft2<LOG2>;
    double2* reg = s + (t / F::TPS) * F::PS;
    const int kofs = (t / F::TPS) * F::S;
    // the register column pass (log1 <= 5) expects the four-step inverse
    // twiddle W_L^{-k1 e} from here: this thread stores e = t + S n1 for
    // n1 = 0, 1, ..., a running product from two lookups
    auto store_out = [&](double2* dst) {
      if (cz.log1 <= 5) {
        double2 w = twiddle_L(cz, k1 * t), ws = twiddle_L(cz, k1 * F::S);
        w.y = -w.y;
        ws.y = -ws.y;
        auto store_tw = [&](int e, double2 v) {
          dst[e] = cmul(v, w);
          w = cmul(w, ws);
        };
        fft2_last_inv<LOG2>(s, t, tw, store_tw);
      } else {
        auto store_row = [&](int e, double2 v) { dst[e] = v; };
        fft2_last_inv<LOG2>(s, t, tw, store_row);
      }
    };
    if constexpr (TM == 0) {
      auto load_row = [&](int e) -> double2 { return row[e]; };
      fft2_first<LOG2>(s, t, tw, load_row);
      __syncthreads();
      const double2* khr = kh + kofs;
      auto mul_spec = [&](int e, double2 v) -> double2 { return cmul(v, __ldg(khr + e)); };
      sub_conv<F::LOGS>(reg, t % F::TPS, tw, mul_spec);
      __syncthreads();
      store_out(row);
      return;
    }
    if constexpr (TM == 1) {
      double2* acc = row + kofs;   // running spectrum sum in slot 0 (thread-owned elements)
      for (int i = 0; i < cz.n_in; ++i) {
        const double2* src = row + (int64_t)i * L;
        auto load_row = [&](int e) -> double2 { return src[e]; };
        __syncthreads();   // previous readers of s are done
        fft2_first<LOG2>(s, t, tw, load_row);
        __syncthreads();   // (also: every load of slot 0 precedes the first acc store)
        const double2* khr = kh + (int64_t)i * L + kofs;
        const bool first = i == 0, last = i == cz.n_in - 1;
        auto store_spec = [&](int e, double2 v) {
          double2 y = cmul(v, __ldg(khr + e));
          if (!first) {
            const double2 a = __ldcg(acc + e);
            y.x += a.x;
            y.y += a.y;
          }
          if (last)
            reg[pad16(e)] = y;
          else
            __stcg(acc + e, y);
        };
        fft2_sub<LOG2, -1>(s, t, tw, SmemLoad{reg}, store_spec);
      }
      fft2_sub<LOG2, +1>(s, t, tw, SmemLoad{reg}, SmemStore{reg});
      __syncthreads();
      store_out(row);
      return;
    }
    // output tiles (TM == 2)
    {
      auto load_row = [&](int e) -> double2 { return row[e]; };
      fft2_first<LOG2>(s, t, tw, load_row);
      __syncthreads();
    }
    double2* keep = row + (int64_t)(cz.n_out - 1) * L + kofs;   // the forward spectrum
    const double2* kh0 = kh + kofs;
    auto store_spec0 = [&](int e, double2 v) {
      __stcg(keep + e, v);
      reg[pad16(e)] = cmul(v, __ldg(kh0 + e));
    };
    fft2_sub<LOG2, -1>(s, t, tw, SmemLoad{reg}, store_spec0);
    const int lt = t % F::TPS;
    for (int j = 0; j < cz.n_out; ++j) {
      if (j > 0) {
        __syncthreads();   // the previous tile's last pass has read every region
        const double2* khr = kh + (int64_t)j * cz.n_in * L + kofs;
        // the region's TPS threads share one warp: reload, then warp-sync
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int e = lt + k * F::TPS;
          reg[pad16(e)] = cmul(__ldcg(keep + e), __ldg(khr + e));
        }
        __syncwarp();
      }
      fft2_sub<LOG2, +1>(s, t, tw, SmemLoad{reg}, SmemStore{reg});
      __syncthreads();
      store_out(row + (int64_t)j * L);
    }
    return;
  } else {
  // single-level FFT (CJT_FFT2=0 builds): untiled only (capi rejects tiles)
  auto load_row = [&](int e) -> double2 { return row[e]; };
  fft_smem_io<LOG2, -1, decltype(load_row), SmemStore, Cfg::LEPT>(s, t, tw, load_row, SmemStore{s});
  auto load_spec = [&](int e) -> double2 { return cmul(s[pad16(e)], __ldg(kh + e)); };
  auto store_row = [&](int e, double2 v) { row[e] = v; };
  fft_smem_io<LOG2, +1, decltype(load_spec), decltype(store_row), Cfg::LEPT>(s, t, tw, load_spec, store_row);
  }
}

// pass 3: columns n2: * W_L^{-n2 k1} -> inverse FFT over k1 -> sum_m Re(post_m * y) -> out
template <int LOG1>
__global__ void __launch_bounds__(ColCfg<LOG1>::T, (ColCfg<LOG1>::T >= 512) ? 1 : 512 / ColCfg<LOG1>::T)
    k_chirpz_cols_inv(ChirpZDev cz, const double2* __restrict__ twg,
                      const double2* __restrict__ buf, double* __restrict__ out, int64_t ldo) {
  using Cfg = ColCfg<LOG1>;
  constexpr int L1 = Cfg::L1, NC = Cfg::NC, T = Cfg::T, CS = Cfg::CS;
  extern __shared__ double2 smem[];
#if CJT_COLS_TWSMEM
  const TwSmem tw = tw_smem_init(smem + NC * CS, twg);
#else
  const double2* tw = twg;
#endif
  const int64_t L2 = (int64_t)1 << cz.log2;
  const int64_t L = cz.length;
  const int64_t c0 = (int64_t)blockIdx.y * NC;
  const int64_t b = blockIdx.x;
  const int64_t so = __ldg(cz.tout + 2 * blockIdx.z), sc = __ldg(cz.tout + 2 * blockIdx.z + 1);
  const int nslot = max(cz.n_in, cz.n_out);
  const int grp = threadIdx.x / (L1 / 16);
  const int t = threadIdx.x % (L1 / 16);
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  // W_L^{n2 k1} running product, looked up once for all terms (see k_chirpz_cols_fwd)
  double2* tws = smem + Cfg::TWO + 2 * threadIdx.x;
  tws[0] = twiddle_L(cz, (c0 + threadIdx.x % NC) * (threadIdx.x / NC));
  tws[1] = twiddle_L(cz, (c0 + threadIdx.x % NC) * (T / NC));
  for (int m = 0; m < cz.m_count; ++m) {
    const double2* bm = buf + ((b * cz.m_count + m) * nslot + blockIdx.z) * L;
    {
      const int c = threadIdx.x % NC;
      const int64_t n2 = c0 + c;
      const int k10 = threadIdx.x / NC;
      double2 w = tws[0];
      const double2 ws = tws[1];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k1 = k10 + i * (T / NC);
        smem[c * CS + pad16(k1)] = cmul(bm[(int64_t)k1 * L2 + n2], make_double2(w.x, -w.y));
        w = cmul(w, ws);
      }
    }
    __syncthreads();
    fft_smem<LOG1, +1, 4, FftSync<LOG1, 4>>(smem + grp * CS, t, tw);
    __syncthreads();   // the transposed store reads other warps' columns
    const double2* post = cz.post + (int64_t)m * cz.count + so;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int idx = threadIdx.x + i * T;
      const int c = idx % NC, n1 = idx / NC;
      const int64_t sidx = (int64_t)n1 * L2 + c0 + c;
      if (sidx < sc) {
        const double2 y = smem[c * CS + pad16(n1)];
        const double2 q = __ldg(post + sidx);
        acc[i] += fma(q.x, y.x, -q.y * y.y);
      }
    }
    __syncthreads();
  }
  double* ob = out + b * ldo + cz.qout + so;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int idx = threadIdx.x + i * T;
    const int c = idx % NC, n1 = idx / NC;
    const int64_t sidx = (int64_t)n1 * L2 + c0 + c;
    if (sidx < sc) ob[sidx] = cz.accumulate ? ob[sidx] + acc[i] : acc[i];
  }
}

template <typename K>
int set_smem(K kernel, int bytes) {
  static_assert(sizeof(K) > 0, "");
  CJT_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return CJT_OK;
}

int fused_groups(int lg) { return lg >= CJT_FUSED_LOGEMIN ? 1 : (1 << (CJT_FUSED_LOGEMIN - lg)); }
// resident CTAs per SM (128 registers per thread: 512 threads)
int fused_ctas_per_sm(int lg) { return lg > 12 ? 1 : 512 / (((1 << lg) * fused_groups(lg)) / 16); }

// direct unless stream-K shortens the modelled critical path by > 10 %
// (time in forward-FFT units, inverse FFT ~ one unit; partial traffic ignored)
FusedSched fused_sched(const ChirpZDev& cz, int64_t batch) {
  const int ng = fused_groups(cz.log2len);
  const int64_t slots = 148 * fused_ctas_per_sm(cz.log2len);
  const int64_t gn = (batch + ng - 1) / ng * cz.n_out;
  FusedSched sk{0, gn * cz.m_count, gn * cz.m_count * cz.n_in, 0, 0};
  const int64_t t_direct = (gn + slots - 1) / slots * cz.m_count * (cz.n_in + 1);
  const int64_t P = std::min(slots, sk.F);
  const int64_t per = (sk.F + P - 1) / P;
  const int64_t segs = per / cz.n_in + 2;   // units a CTA range touches (upper bound)
  const int64_t t_sk = per + std::min(segs, per);
  const int64_t gsegs = segs / cz.m_count + 2;   // (group, j) segments a CTA range touches
  // $CJT_FUSED_SCHED (experiments): 1 forces direct, 2 stream-K
  static const int force = [] {
    const char* e = getenv("CJT_FUSED_SCHED");
    return e ? atoi(e) : 0;
  }();
  const bool pick = force ? force == 2 : 10 * t_sk < 9 * t_direct;
  if (pick && batch <= 65535) {
    sk.streamk = 1;
    sk.P = P;
    sk.S = gsegs;
  }
  return sk;
}

template <int LOGL>
int run_fused(const ChirpZDev& cz, const double2* tw, const double* x, int64_t ldx, double* out,
              int64_t ldo, int64_t batch, double* part, double2* spec, cudaStream_t st, int* launches) {
  using Cfg = FusedCfg<LOGL>;
  static_assert(Cfg::NG == (LOGL >= CJT_FUSED_LOGEMIN ? 1 : (1 << (CJT_FUSED_LOGEMIN - LOGL))), "fused_groups out of sync");
  static DeviceOnce once_;
  if (int rc_ = once_([&]() -> int {
    if (int rc = set_smem(k_chirpz_fused<LOGL, false>, Cfg::SMEM)) return rc;
    if (int rc = set_smem(k_chirpz_fused<LOGL, true>, Cfg::SMEM)) return rc;
    return CJT_OK;
  })) return rc_;
  const FusedSched sk = fused_sched(cz, batch);
  if (sk.streamk && batch > 65535) return fail(CJT_EINVAL, "chirp-z stream-K schedule out of range");
  if (cz.n_in > 1 && !spec) return fail(CJT_EINVAL, "chirp-z without spectrum workspace");
  if (sk.streamk && !part) return fail(CJT_EINVAL, "chirp-z without partial workspace");
  const int64_t groups = (batch + Cfg::NG - 1) / Cfg::NG;
  dim3 grid = sk.streamk ? dim3((unsigned)sk.P) : dim3((unsigned)groups, (unsigned)cz.n_out);
  if (cz.n_in > 1)
    k_chirpz_fused<LOGL, true><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, x, ldx, out, ldo, batch, part, spec, sk);
  else
    k_chirpz_fused<LOGL, false><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, x, ldx, out, ldo, batch, part, spec, sk);
  CJT_CUDA_TRY(cudaGetLastError());
  *launches += 1;
  if (sk.streamk) {
    dim3 g2((unsigned)((cz.count_max + 255) / 256), (unsigned)cz.n_out, (unsigned)batch);
    k_chirpz_combine_sk<<<g2, 256, 0, st>>>(cz, part, sk, Cfg::NG, out, ldo);
    CJT_CUDA_TRY(cudaGetLastError());
    *launches += 1;
  }
  return CJT_OK;
}

template <int LOGQ, int P>
int run_cluster(const ChirpZDev& cz, const double2* tw, const double* x, int64_t ldx, double* out,
                int64_t ldo, int64_t batch, cudaStream_t st) {
  using Cfg = ClusterCfg<LOGQ, P>;
  auto kern = k_chirpz_cluster<LOGQ, P>;
  static DeviceOnce once_;
  if (int rc_ = once_([&]() -> int {
    if (int rc = set_smem(kern, Cfg::SMEM)) return rc;
    if (P > 8) CJT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return CJT_OK;
  })) return rc_;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P * batch));
  cfg.blockDim = dim3(Cfg::T);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CJT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, cz, tw, x, ldx, out, ldo));
  return CJT_OK;
}

template <int LOG1>
int run_cols_fwd(const ChirpZDev& cz, const double2* tw, const double* x, int64_t ldx,
                 double2* buf, int64_t batch, cudaStream_t st) {
  using Cfg = ColCfg<LOG1>;
  static DeviceOnce once_;
  if (int rc_ = once_([&]() -> int {
    if (int rc = set_smem(k_chirpz_cols_fwd<LOG1>, Cfg::SMEM)) return rc;
    return CJT_OK;
  })) return rc_;
  const int64_t L2 = (int64_t)1 << cz.log2;
  if constexpr (LOG1 <= 5) {
    dim3 grid((unsigned)batch, (unsigned)(L2 / COLR_T), (unsigned)(cz.n_in * cz.m_count));
    k_chirpz_cols_fwd_reg<LOG1><<<grid, COLR_T, 0, st>>>(cz, x, ldx, buf);
    CJT_CUDA_TRY(cudaGetLastError());
    return CJT_OK;
  }
  dim3 grid((unsigned)batch, (unsigned)(L2 / Cfg::NC), (unsigned)cz.n_in);
  k_chirpz_cols_fwd<LOG1><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, x, ldx, buf);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

template <int LOG2>
int run_rows(const ChirpZDev& cz, const double2* tw, double2* buf, int64_t batch, cudaStream_t st) {
  using Cfg = RowCfg<LOG2>;
  static DeviceOnce once_;
  if (int rc_ = once_([&]() -> int {
    if (int rc = set_smem(k_chirpz_rows<LOG2, 0>, Cfg::SMEM)) return rc;
    if (int rc = set_smem(k_chirpz_rows<LOG2, 1>, Cfg::SMEM)) return rc;
    if (int rc = set_smem(k_chirpz_rows<LOG2, 2>, Cfg::SMEM)) return rc;
    return CJT_OK;
  })) return rc_;
  const int64_t L1 = (int64_t)1 << cz.log1;
  dim3 grid((unsigned)(batch * cz.m_count), (unsigned)(L1 / Cfg::NR));
  auto kern = cz.n_in > 1 ? k_chirpz_rows<LOG2, 1> : cz.n_out > 1 ? k_chirpz_rows<LOG2, 2> : k_chirpz_rows<LOG2, 0>;
  kern<<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, buf);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

template <int LOG1>
int run_cols_inv(const ChirpZDev& cz, const double2* tw, const double2* buf, double* out,
                 int64_t ldo, int64_t batch, cudaStream_t st) {
  using Cfg = ColCfg<LOG1>;
  static DeviceOnce once_;
  if (int rc_ = once_([&]() -> int {
    if (int rc = set_smem(k_chirpz_cols_inv<LOG1>, Cfg::SMEM)) return rc;
    return CJT_OK;
  })) return rc_;
  const int64_t L2 = (int64_t)1 << cz.log2;
  if constexpr (LOG1 <= 5) {
    dim3 grid((unsigned)batch, (unsigned)(L2 / COLR_T), (unsigned)cz.n_out);
    k_chirpz_cols_inv_reg<LOG1><<<grid, COLR_T, 0, st>>>(cz, buf, out, ldo);
    CJT_CUDA_TRY(cudaGetLastError());
    return CJT_OK;
  }
  dim3 grid((unsigned)batch, (unsigned)(L2 / Cfg::NC), (unsigned)cz.n_out);
  k_chirpz_cols_inv<LOG1><<<grid, Cfg::T, Cfg::SMEM, st>>>(cz, tw, buf, out, ldo);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

}  // namespace

void chirpz_workspace(const ChirpZDev& cz, int64_t batch, int64_t* part_elems, int64_t* spec_elems) {
  // sized for every execution batch up to the reserved one
  *part_elems = *spec_elems = 0;
  if (cz.length <= 0 || cz.log2len > 13) return;
  const int ng = fused_groups(cz.log2len);
  for (int64_t bb = 1; bb <= batch; ++bb) {
    const FusedSched sk = fused_sched(cz, bb);
    if (sk.streamk) {
      *part_elems = std::max(*part_elems, sk.P * sk.S * ng * cz.count_max);
      if (cz.n_in > 1) *spec_elems = std::max(*spec_elems, sk.P * ng * cz.length);
    } else if (cz.n_in > 1) {
      *spec_elems = std::max(*spec_elems, (bb + ng - 1) / ng * ng * cz.n_out * cz.length);
    }
  }
}

bool cluster_enabled() {
  static const bool on = [] {
    const char* e = getenv("CJT_CLUSTER");
    return e && e[0] == '1';
  }();
  return on;
}

int launch_chirpz(const ChirpZDev& cz, const double2* tw8192, const double* x, int64_t ldx,
                  double* out, int64_t ldo, int64_t batch, double2* scratch, double* part,
                  double2* spec, cudaStream_t st, int* launches) {
  if (batch <= 0) return CJT_OK;
  const int lg = cz.log2len;
  if (lg <= 13) {
    switch (lg) {
#define CJT_FUSED(K) case K: return run_fused<K>(cz, tw8192, x, ldx, out, ldo, batch, part, spec, st, launches);
      CJT_FUSED(4) CJT_FUSED(5) CJT_FUSED(6) CJT_FUSED(7) CJT_FUSED(8) CJT_FUSED(9) CJT_FUSED(10)
      CJT_FUSED(11) CJT_FUSED(12) CJT_FUSED(13)
#undef CJT_FUSED
      default: return fail(CJT_EINVAL, "chirp-z length below 16");
    }
  }
  if (lg <= 17 && cz.n_in == 1 && cz.n_out == 1 && cluster_enabled()) {   // (tiled products keep the multi-pass layout)
    *launches += 1;
    switch (lg) {
      case 14: return run_cluster<12, 4>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 15: return run_cluster<12, 8>(cz, tw8192, x, ldx, out, ldo, batch, st);
      case 16: return run_cluster<12, 16>(cz, tw8192, x, ldx, out, ldo, batch, st);
      default: return run_cluster<13, 16>(cz, tw8192, x, ldx, out, ldo, batch, st);
    }
  }
  *launches += 3;
  int rc = CJT_OK;
  // register column passes rely on the row pass applying the inverse twiddle
  if (cz.log1 <= 5 && !fft2_used(cz.log2)) return fail(CJT_EINVAL, "multi-pass split unsupported");
  if ((cz.n_in > 1 || cz.n_out > 1) && (!fft2_used(cz.log2) || (cz.n_in > 1 && cz.n_out > 1)))
    return fail(CJT_EINVAL, "tiled multi-pass chirp-z needs n_in == 1 or n_out == 1");
  switch (cz.log1) {
#define CJT_COLF(K) case K: rc = run_cols_fwd<K>(cz, tw8192, x, ldx, scratch, batch, st); break;
    CJT_COLF(4) CJT_COLF(5) CJT_COLF(6) CJT_COLF(7) CJT_COLF(8) CJT_COLF(9) CJT_COLF(10) CJT_COLF(11)
    CJT_COLF(12) CJT_COLF(13)
#undef CJT_COLF
    default: return fail(CJT_EINVAL, "chirp-z column length out of range");
  }
  if (rc) return rc;
  switch (cz.log2) {
#define CJT_ROW(K) case K: rc = run_rows<K>(cz, tw8192, scratch, batch, st); break;
    CJT_ROW(10) CJT_ROW(11) CJT_ROW(12) CJT_ROW(13)
#undef CJT_ROW
    default: return fail(CJT_EINVAL, "chirp-z row length out of range");
  }
  if (rc) return rc;
  switch (cz.log1) {
#define CJT_COLI(K) case K: rc = run_cols_inv<K>(cz, tw8192, scratch, out, ldo, batch, st); break;
    CJT_COLI(4) CJT_COLI(5) CJT_COLI(6) CJT_COLI(7) CJT_COLI(8) CJT_COLI(9) CJT_COLI(10) CJT_COLI(11)
    CJT_COLI(12) CJT_COLI(13)
#undef CJT_COLI
    default: return fail(CJT_EINVAL, "chirp-z column length out of range");
  }
  return rc;
}

}  // namespace cjt
