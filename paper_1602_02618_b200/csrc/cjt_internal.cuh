// Internal definitions shared by the CJT CUDA translation units (sm_100a).
//
// Data layout in HBM (all float64):
//   coefficient batches   [batch][N+1]            row-major, one vector per row
//   Lobatto values        [batch][G+1]
//   chirp-z scratch       [batch][m][L] complex    (multi-pass Bluestein only)
//   recurrence partials   [slot][batch][tile]      (deterministic split-K)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/cjt.h"

namespace cjt {

// One-time per-DEVICE initialisation (cudaFuncSetAttribute and friends act on
// the current device only): a process that drives several GPUs, or several
// host threads racing to the first launch, runs `f` exactly once per device.
struct DeviceOnce {
  std::atomic<uint64_t> done{0};
  std::mutex mu;
  template <typename F>
  int operator()(F&& f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      dev = 0;
    }
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return 0;
    std::lock_guard<std::mutex> lk(mu);
    if (done.load(std::memory_order_relaxed) & bit) return 0;
    const int rc = f();
    if (rc == 0) done.fetch_or(bit, std::memory_order_release);
    return rc;
  }
};

// ---------------------------------------------------------------------------
// errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
#define CJT_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t err__ = (expr);                                                   \
    if (err__ != cudaSuccess)                                                     \
      return ::cjt::fail(CJT_ECUDA, std::string(#expr " failed: ") +              \
                                        cudaGetErrorString(err__));               \
  } while (0)

// ---------------------------------------------------------------------------
// 1-D TMA (cp.async.bulk) global -> shared copies completed on an mbarrier
// (sm_90+; used by the streaming kernels).  Sizes and addresses: multiples
// of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// shared -> global bulk copy in the issuing thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the source reads of all committed bulk groups are done (the buffer may be reused)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk group has completed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * (DIR * i): DIR = -1 -> a * (-i), DIR = +1 -> a * i
template <int DIR>
__device__ __forceinline__ double2 cmul_i(double2 a) {
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

// padded shared-memory index: one slot of padding every 16 complex elements,
// which makes the stride-16 write of the first radix-16 pass conflict-free
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int l) { return l + l / 16; }

// ---------------------------------------------------------------------------
// in-register DFT of size R (2, 4, 8, 16), natural order in and out,
// X_k = sum_j v_j exp(DIR 2 pi i j k / R)

__device__ __forceinline__ double cos16(int j) {
  switch (j & 15) {
    case 0: return 1.0;
    case 1: return 0.92387953251128675613;
    case 2: return 0.70710678118654752440;
    case 3: return 0.38268343236508977173;
    case 4: return 0.0;
    case 5: return -0.38268343236508977173;
    case 6: return -0.70710678118654752440;
    case 7: return -0.92387953251128675613;
    case 8: return -1.0;
    case 9: return -0.92387953251128675613;
    case 10: return -0.70710678118654752440;
    case 11: return -0.38268343236508977173;
    case 12: return 0.0;
    case 13: return 0.38268343236508977173;
    case 14: return 0.70710678118654752440;
    default: return 0.92387953251128675613;
  }
}
__device__ __forceinline__ double sin16(int j) { return cos16(j - 4); }

__device__ __forceinline__ double cos32(int j) {
  switch (j & 31) {
    case 1: return 0.98078528040323044913;
    case 3: return 0.83146961230254523708;
    case 5: return 0.55557023301960222474;
    case 7: return 0.19509032201612826785;
    case 9: return -0.19509032201612826785;
    case 11: return -0.55557023301960222474;
    case 13: return -0.83146961230254523708;
    case 15: return -0.98078528040323044913;
    case 17: return -0.98078528040323044913;
    case 19: return -0.83146961230254523708;
    case 21: return -0.55557023301960222474;
    case 23: return -0.19509032201612826785;
    case 25: return 0.19509032201612826785;
    case 27: return 0.55557023301960222474;
    case 29: return 0.83146961230254523708;
    case 31: return 0.98078528040323044913;
    default: return cos16((j & 31) >> 1);
  }
}
__device__ __forceinline__ double sin32(int j) { return cos32(j - 8); }

// b * exp(DIR 2 pi i k / SZ), compile-time K and SZ after unrolling (SZ <= 32)
template <int DIR, int K, int SZ>
__device__ __forceinline__ double2 twiddle_const(double2 b) {
  if constexpr (K == 0) {
    return b;
  } else if constexpr (4 * K == SZ) {
    return cmul_i<DIR>(b);
  } else {
    constexpr int J = K * (32 / SZ);
    const double c = cos32(J);
    const double s = DIR * sin32(J);
    return make_double2(fma(b.x, c, -b.y * s), fma(b.x, s, b.y * c));
  }
}

__host__ __device__ constexpr int bitrev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

template <int DIR, int SZ, int ST, int K, int R>
__device__ __forceinline__ void dft_stage_k(double2* v) {
  if constexpr (K < SZ / 2) {
    double2 a = v[ST + K];
    double2 b = twiddle_const<DIR, K, SZ>(v[ST + K + SZ / 2]);
    v[ST + K] = cadd(a, b);
    v[ST + K + SZ / 2] = csub(a, b);
    dft_stage_k<DIR, SZ, ST, K + 1, R>(v);
  }
}
template <int DIR, int SZ, int ST, int R>
__device__ __forceinline__ void dft_stage(double2* v) {
  if constexpr (ST < R) {
    dft_stage_k<DIR, SZ, ST, 0, R>(v);
    dft_stage<DIR, SZ, ST + SZ, R>(v);
  }
}
template <int DIR, int SZ, int R>
__device__ __forceinline__ void dft_levels(double2* v) {
  if constexpr (SZ <= R) {
    dft_stage<DIR, SZ, 0, R>(v);
    dft_levels<DIR, SZ * 2, R>(v);
  }
}
template <int R, int DIR>
__device__ __forceinline__ void dft_reg(double2* v) {
  constexpr int BITS = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : (R == 16) ? 4 : 5;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int j = bitrev(i, BITS);
    if (j > i) {
      double2 t = v[i];
      v[i] = v[j];
      v[j] = t;
    }
  }
  dft_levels<DIR, 2, R>(v);
}


#ifndef CJT_TW_MODE
#define CJT_TW_MODE 1
#endif

// Twiddle sources: W^u = exp(-2 pi i u / 8192), 0 <= u < 8192.
// A plain pointer is the 8192-entry global table (read through L1).
__device__ __forceinline__ double2 tw_at(const double2* __restrict__ tw, int u) { return __ldg(&tw[u]); }

// TwSmem: 1024 entries W^r in shared memory and an octant rotation,
// W^(1024 o + r) = exp(-i pi o / 4) W^r.  For kernels whose shared memory
// leaves too little L1 to hold the global table's working set (an L2 round
// trip per twiddle otherwise dominates).
struct TwSmem {
  const double2* tab;
  __device__ __forceinline__ double2 operator()(int u) const {
    double2 a = tab[u & 1023];
    const int o = u >> 10;
    if (o & 1) {   // times (1 - i) / sqrt 2
      constexpr double c = 0.70710678118654752440;
      a = make_double2((a.x + a.y) * c, (a.y - a.x) * c);
    }
    const int q = o >> 1;   // times (-i)^q
    if (q & 1) a = make_double2(a.y, -a.x);
    if (q & 2) a = make_double2(-a.x, -a.y);
    return a;
  }
};
__device__ __forceinline__ double2 tw_at(const TwSmem& tw, int u) { return tw(u); }

// copy W^r, r < 1024, into shared memory (all threads of the CTA; syncs)
__device__ __forceinline__ TwSmem tw_smem_init(double2* tab, const double2* __restrict__ tw) {
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = __ldg(&tw[i]);
  __syncthreads();
  return TwSmem{tab};
}

// Packed power tables behind the 8192-entry table (shared_twiddles, capi):
//   tw[8192 + 2^c + k] = exp(-2 pi i k / 2^c),  c = 0..13, k < 2^c.
// The thread with butterfly index k of a size-2^A pass needs w^(2^p),
// w = exp(-2 pi i k / 2^A), i.e. entry k of table c = A - p: consecutive
// threads read consecutive entries (coalesced 16-byte loads, 4 wavefronts
// per warp) where the same values taken from the 8192-entry table are
// 2^(13 - A + p) entries apart (one cache line per lane, up to 32 wavefronts
// per load: measured 28 % of the row kernels' l1tex wavefronts).
constexpr int TW_PACKED_OFFSET = 8192;
constexpr int TW_TABLE_ENTRIES = 8192 + 16384;
template <int A, int P>
__device__ __forceinline__ double2 tw_pow(const double2* __restrict__ tw, int k) {
  static_assert(A - P >= 0 && A <= 13, "tw_pow: table out of range");
  return __ldg(&tw[TW_PACKED_OFFSET + (1 << (A - P)) + k]);
}
template <int A, int P>
__device__ __forceinline__ double2 tw_pow(const TwSmem& tw, int k) {
  return tw((k << (13 - A)) << P);
}

// v[r] *= w^r for r = 1..R-1 with w = exp(-2 pi i k / 2^A) (conjugated for
// DIR > 0), k < 2^A / R; w^(2^j) are read from the tables (tw_pow), the other
// powers are products of at most three of them.
template <int R, int DIR, int A, class TW>
__device__ __forceinline__ void twiddle_powers(double2* v, const TW& tw, int k) {
  double2 p[32];
  p[1] = tw_pow<A, 0>(tw, k);
  if constexpr (R > 2) p[2] = tw_pow<A, 1>(tw, k);
  if constexpr (R > 4) p[4] = tw_pow<A, 2>(tw, k);
  if constexpr (R > 8) p[8] = tw_pow<A, 3>(tw, k);
  if constexpr (R > 16) p[16] = tw_pow<A, 4>(tw, k);
  if constexpr (DIR > 0) {
#pragma unroll
    for (int j = 1; j < R; j <<= 1) p[j].y = -p[j].y;
  }
#pragma unroll
  for (int r = 1; r < R; ++r) {
    if ((r & (r - 1)) != 0) {  // not a power of two: r = hi + lo
      const int hi = 1 << (31 - __clz(r));
      p[r] = cmul(p[hi], p[r - hi]);
    }
    v[r] = cmul(v[r], p[r]);
  }
}

// ---------------------------------------------------------------------------
// Shared-memory Stockham FFT of length L = 2^LOGL (4 <= LOGL <= 13), executed
// by the L/EPT threads t of one group, EPT = 2^LEPT elements per thread (radix
// EPT passes, the last pass radix L / EPT^(passes-1)).  `tw` is the
// 8192-entry table exp(-2 pi i u / 8192).  Every thread of the CTA must call
// it with the same LOGL (it synchronises the CTA between passes).  Result in
// natural order.
// First-pass loader / last-pass storer hooks: the default reads and writes
// the shared buffer; fused kernels substitute global loads (with the input
// diagonal), the spectrum product, or the output accumulation, saving a
// shared-memory round trip each.
struct SmemLoad {
  const double2* s;
  __device__ __forceinline__ double2 operator()(int e) const { return s[pad16(e)]; }
};
struct SmemStore {
  double2* s;
  __device__ __forceinline__ void operator()(int e, double2 v) const { s[pad16(e)] = v; }
};

// Barrier policy of an FFT's passes: the whole CTA, or only the warp (for
// sub-FFTs owned by one warp or by a fraction of one)
struct SyncCTA {
  static __device__ __forceinline__ void sync() { __syncthreads(); }
};
struct SyncWarp {
  static __device__ __forceinline__ void sync() { __syncwarp(); }
};

template <int LOGL, int DIR, int LEPT, int PASS, class LoadF, class StoreF, class TW, class SY = SyncCTA>
__device__ __forceinline__ void fft_pass(double2* s, int t, const TW& tw,
                                         const LoadF& first_load, const StoreF& last_store) {
  constexpr int NP = (LOGL + LEPT - 1) / LEPT;
  if constexpr (PASS < NP) {
    constexpr int EPT = 1 << LEPT;
    constexpr int LR = (PASS < NP - 1) ? LEPT : (LOGL - LEPT * (NP - 1));
    constexpr int R = 1 << LR;
    constexpr int L = 1 << LOGL;
    constexpr int LNS = LEPT * PASS;
    constexpr int NS = 1 << LNS;
    constexpr int NBF = EPT / R;
    constexpr int STRIDE = L / R;
    constexpr int TPG = L / EPT;
    double2 v[EPT];
#pragma unroll
    for (int q = 0; q < NBF; ++q) {
      const int j = t + q * TPG;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (PASS == 0)
          v[q * R + r] = first_load(j + r * STRIDE);
        else
          v[q * R + r] = s[pad16(j + r * STRIDE)];
      }
    }
    SY::sync();
#pragma unroll
    for (int q = 0; q < NBF; ++q) {
      const int j = t + q * TPG;
      const int k = j & (NS - 1);
      if constexpr (PASS > 0) {
#if CJT_TW_MODE == 0
        constexpr int SH = 13 - (LNS + LR);
#pragma unroll
        for (int r = 1; r < R; ++r) {
          double2 w = tw_at(tw, (r * k) << SH);
          if (DIR > 0) w.y = -w.y;
          v[q * R + r] = cmul(v[q * R + r], w);
        }
#else
        // powers of w = W^k from the tabulated w, w^2, w^4, w^8 (at most three
        // rounded products per power)
        twiddle_powers<R, DIR, LNS + LR>(&v[q * R], tw, k);
#endif
      }
      dft_reg<R, DIR>(&v[q * R]);
      const int base = ((j - k) << LR) + k;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (PASS == NP - 1)
          last_store(base + r * NS, v[q * R + r]);
        else
          s[pad16(base + r * NS)] = v[q * R + r];
      }
    }
    SY::sync();
    fft_pass<LOGL, DIR, LEPT, PASS + 1, LoadF, StoreF, TW, SY>(s, t, tw, first_load, last_store);
  }
}

template <int LOGL, int DIR, int LEPT = 4, class SY = SyncCTA, class TW>
__device__ __forceinline__ void fft_smem(double2* s, int t, const TW& tw) {
  static_assert(LOGL >= LEPT && LOGL <= 13, "smem FFT length out of range");
  fft_pass<LOGL, DIR, LEPT, 0, SmemLoad, SmemStore, TW, SY>(s, t, tw, SmemLoad{s}, SmemStore{s});
}
// FFTs whose L / 2^LEPT threads sit inside one warp synchronise the warp only
template <int LOGL, int LEPT>
using FftSync = std::conditional_t<(LOGL - LEPT <= 5), SyncWarp, SyncCTA>;

// FFT with a custom first-pass source and last-pass sink (see SmemLoad/SmemStore)
template <int LOGL, int DIR, class LoadF, class StoreF, int LEPT = 4, class TW>
__device__ __forceinline__ void fft_smem_io(double2* s, int t, const TW& tw,
                                            const LoadF& ld, const StoreF& st) {
  static_assert(LOGL >= LEPT && LOGL <= 13, "smem FFT length out of range");
  fft_pass<LOGL, DIR, LEPT, 0>(s, t, tw, ld, st);
}

// ---------------------------------------------------------------------------
// Two-level FFT of length L = 16 S (512 <= L <= 8192, T = S threads per FFT):
//   fft2_first:    CTA-wide radix-16 DIF pass: thread n2 loads x[n2 + S n1]
//                  (n1 < 16) through the hook, DFT over n1, twiddle W_L^{n2 k1},
//                  writes sub-sequence k1 at region k1 (contiguous, padded);
//   sub-FFTs:      16 independent S-point FFTs over n2, one per region, each
//                  owned by S/16 consecutive threads (a warp or part of one) and
//                  synchronised with __syncwarp only;  X[k1 + 16 k2] = region
//                  k1 position k2 ("permuted" spectrum order);
//   fft2_last_inv: CTA-wide radix-16 DIT inverse pass from the permuted
//                  spectrum after the inverse sub-FFTs: thread n2 gathers
//                  region k1 position n2, twiddle W_L^{-n2 k1}, IDFT over k1,
//                  value y[n2 + S n1] to the hook.
// A forward FFT, spectrum product and inverse FFT thus need two CTA barriers
// instead of two per pass; warps drift apart and overlap shared-memory and
// FP64 phases.
#ifndef CJT_FFT2
#define CJT_FFT2 1
#endif
// lengths that run the two-level FFT (fused tiles and multi-pass rows); their
// spectra (khat) are stored in the permuted order k1 S + k2 <-> k1 + 16 k2
__host__ __device__ constexpr bool fft2_used(int lg) { return CJT_FFT2 && lg >= 9; }

template <int LOGL>
struct Fft2 {
  static constexpr int L = 1 << LOGL;
  static constexpr int LOGS = LOGL - 4;
  static constexpr int S = L / 16;
  static constexpr int PS = padded_len(S);   // region stride
  static constexpr int TPS = S / 16;         // threads per sub-FFT
};

template <int LOGL, class LoadF, class TW>
__device__ __forceinline__ void fft2_first(double2* s, int n2, const TW& tw, const LoadF& ld) {
  using F = Fft2<LOGL>;
  double2 v[16];
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) v[n1] = ld(n2 + F::S * n1);
  dft_reg<16, -1>(v);
  twiddle_powers<16, -1, LOGL>(v, tw, n2);
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) s[k1 * F::PS + pad16(n2)] = v[k1];
}

template <int LOGL, class StoreF, class TW>
__device__ __forceinline__ void fft2_last_inv(const double2* s, int n2, const TW& tw, const StoreF& st) {
  using F = Fft2<LOGL>;
  double2 v[16];
#pragma unroll
  for (int k1 = 0; k1 < 16; ++k1) v[k1] = s[k1 * F::PS + pad16(n2)];
  twiddle_powers<16, +1, LOGL>(v, tw, n2);
  dft_reg<16, +1>(v);
#pragma unroll
  for (int n1 = 0; n1 < 16; ++n1) st(n2 + F::S * n1, v[n1]);
}

// One warp-synchronous Stockham pass of radix 2^LR over an N = 2^LOGN region
// (LNS = log2 of the product of the previous radices), 16 elements per thread.
template <int LOGN, int DIR, int LR, int LNS, class LoadF, class StoreF, class TW>
__device__ __forceinline__ void sub_pass(double2* s, int t, const TW& tw, const LoadF& ld,
                                         const StoreF& st) {
  constexpr int N = 1 << LOGN, R = 1 << LR, NS = 1 << LNS;
  constexpr int NBF = 16 / R, STRIDE = N / R, TPG = N / 16;
  double2 v[16];
#pragma unroll
  for (int q = 0; q < NBF; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = ld(t + q * TPG + r * STRIDE);
  __syncwarp();
#pragma unroll
  for (int q = 0; q < NBF; ++q) {
    const int j = t + q * TPG;
    const int k = j & (NS - 1);
    if constexpr (LNS > 0) twiddle_powers<R, DIR, LNS + LR>(&v[q * R], tw, k);
    dft_reg<R, DIR>(&v[q * R]);
    const int base = ((j - k) << LR) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) st(base + r * NS, v[q * R + r]);
  }
  __syncwarp();
}

// COUNT consecutive passes of radix 2^LR starting at LNS (shared-memory in place)
template <int LOGN, int DIR, int LR, int LNS, int COUNT, class TW>
__device__ __forceinline__ void sub_passes(double2* s, int t, const TW& tw) {
  if constexpr (COUNT > 0) {
    sub_pass<LOGN, DIR, LR, LNS>(s, t, tw, SmemLoad{s}, SmemStore{s});
    sub_passes<LOGN, DIR, LR, LNS + LR, COUNT - 1>(s, t, tw);
  }
}

// Sub-FFT pass plan for N = 2^LOGN: FULL passes of radix 16, then a remainder
// radix 2^REM.  The inverse runs the radices in reverse order, so the forward's
// last pass and the inverse's first pass touch the same elements in the same
// thread: sub_middle does both in registers around the spectrum operation.
template <int LOGN>
struct SubPlan {
  static constexpr int FULL = (LOGN - 1) / 4;
  static constexpr int REM = LOGN - 4 * FULL;   // 1..4
};

// forward last pass (radix 2^REM at LNS = 4 FULL) -> op(e, X_e) at spectrum
// index e -> inverse first pass (radix 2^REM, no twiddle) -> shared memory
template <int LOGN, class SpecF, class TW>
__device__ __forceinline__ void sub_middle(double2* s, int t, const TW& tw, const SpecF& op) {
  constexpr int LR = SubPlan<LOGN>::REM, LNS = 4 * SubPlan<LOGN>::FULL;
  constexpr int N = 1 << LOGN, R = 1 << LR, NS = 1 << LNS;
  constexpr int NBF = 16 / R, TPG = N / 16;
  static_assert(NS * R == N, "sub_middle: pass plan");
  double2 v[16];
#pragma unroll
  for (int q = 0; q < NBF; ++q)
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = s[pad16(t + q * TPG + r * NS)];
  __syncwarp();
#pragma unroll
  for (int q = 0; q < NBF; ++q) {
    const int j = t + q * TPG;   // j < NS: this butterfly's outputs are j + r NS
    if constexpr (LNS > 0) twiddle_powers<R, -1, LNS + LR>(&v[q * R], tw, j);
    dft_reg<R, -1>(&v[q * R]);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q * R + r] = op(j + r * NS, v[q * R + r]);
    dft_reg<R, +1>(&v[q * R]);
    // R consecutive elements per thread: with pad16, the 16-byte bank groups of
    // neighbouring lanes collide in pairs for R = 8 (lanes j, j + 1) and R = 2
    // (lanes j, j + 4) -- ncu: 2-way conflicts, 11 % of the row kernels'
    // shared-memory wavefronts.  Those lanes store their elements in the order
    // r ^ R/2 instead (a register select), which makes every store conflict-free.
    constexpr bool SWZ = (LR == 3) || (LR == 1 && LOGN >= 7);
    if constexpr (SWZ) {
      const bool f = LR == 3 ? (j & 1) : ((j >> 2) & 1);
      const int x = f ? R / 2 : 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2 a = v[q * R + r], b = v[q * R + (r ^ (R / 2))];
        s[pad16((j << LR) + (r ^ x))] = f ? b : a;
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) s[pad16((j << LR) + r)] = v[q * R + r];
    }
  }
  __syncwarp();
}

// forward sub-FFT with the last pass's outputs sent to st(e, X_e) (natural e)
template <int LOGN, class StoreF, class TW>
__device__ __forceinline__ void sub_fft_fwd_to(double2* s, int t, const TW& tw, const StoreF& st) {
  using SP = SubPlan<LOGN>;
  sub_passes<LOGN, -1, 4, 0, SP::FULL>(s, t, tw);
  sub_pass<LOGN, -1, SP::REM, 4 * SP::FULL>(s, t, tw, SmemLoad{s}, st);
}

// forward sub-FFT, X_e <- op(e, X_e), inverse sub-FFT, natural order in place
template <int LOGN, class SpecF, class TW>
__device__ __forceinline__ void sub_conv(double2* s, int t, const TW& tw, const SpecF& op) {
  using SP = SubPlan<LOGN>;
  sub_passes<LOGN, -1, 4, 0, SP::FULL>(s, t, tw);
  sub_middle<LOGN>(s, t, tw, op);
  sub_passes<LOGN, +1, 4, SP::REM, SP::FULL>(s, t, tw);
}

// the sub-FFT of region k1 = n2 / TPS, local thread n2 % TPS (warp-synchronous)
template <int LOGL, int DIR, class LoadF, class StoreF, class TW>
__device__ __forceinline__ void fft2_sub(double2* s, int n2, const TW& tw, const LoadF& ld,
                                         const StoreF& st) {
  using F = Fft2<LOGL>;
  static_assert(F::TPS >= 1 && F::TPS <= 32, "sub-FFT must fit one warp");
  fft_pass<F::LOGS, DIR, 4, 0, LoadF, StoreF, TW, SyncWarp>(s + (n2 / F::TPS) * F::PS, n2 % F::TPS, tw,
                                                           ld, st);
}

// ---------------------------------------------------------------------------
// device-side descriptors

struct ChirpZDev {
  int64_t p0, width, q0, count, length;
  int64_t qout;                  // output index of q = q0 (q0 - out_shift)
  int32_t m_count, accumulate;
  int32_t log2len, log1, log2;   // multipass split L = L1 * L2 (log1 + log2 = log2len)
  const double2* pre;       // [m][width]
  const double2* post;      // [m][count]
  const double2* khat;      // fused: natural order; multipass: [k1][k2] = khat[k1 + L1 k2]
  const double2* tw_hi;     // multipass: exp(-2 pi i (a 4096) / L)
  const double2* tw_lo;     // multipass: exp(-2 pi i b / L), b < 4096
  const double2* tw_col;    // multipass, register columns (log1 <= 5): [p][n2] = exp(-2 pi i n2 2^p / L), p < log1
  int32_t n_in, n_out;      // tiling (fused path only; 1 x 1 otherwise)
  int64_t count_max;        // largest output tile
  const int64_t* tin;       // [n_in][2] (offset, width)
  const int64_t* tout;      // [n_out][2] (offset, count)
};

struct RecRowsDev {
  const double* x;
  const double* xm;
  const int8_t* reg;
  const int64_t* cut;
  int64_t nrows;
};

struct RecTablesDev {
  const double *A, *B, *C, *rfp, *rfm, *rfpi, *rfmi;
  int64_t n_tab;   // entries per table
  // FMA-form Reinsch tables (A, C scaled by 1/rf+-), see rec_step_fast
  const double *Ap = nullptr, *Am = nullptr, *Cp = nullptr, *Cm = nullptr;
};
constexpr int REC_WIN_ROWS = 9;   // A, B, C, rf+, rf-, A/rf+, A/rf-, C/rf+, C/rf-

// forward split-K work item: rows [row0, row0+nrows) x degrees [n_begin, n_end)
struct FwdItem {
  int32_t row0, nrows, n_begin, n_end, slot, pad;
};
// two-pass contraction item: stages s < nstages use P block p_block0 + s and
// operand columns x_off0 + 32 s (ids_off < 0) or 32 * ids[ids_off + s]
struct GemmItem {
  int64_t p_block0;
  int64_t x_off0;
  int32_t ids_off, nstages, slot, pad;
};
// inverse work item: degrees [n0, n0+64) x row tiles tile_ids[t_begin .. t_begin+t_count)
struct InvItem {
  int32_t n0, t_begin, t_count, slot;
};

constexpr int CK = 32;          // recurrence checkpoint spacing (degrees)
constexpr int FWD_ROWS = 128;   // grid rows per forward CTA tile (4 warps x 32 rows)
constexpr int FWD_KS = 32;      // degrees per forward pipeline stage
constexpr int INV_DT = 128;     // degrees per inverse CTA tile (4 warps x 32 degrees)
constexpr int INV_RT = 32;      // grid rows per inverse pipeline stage (= row tile)

// Cluster (DSMEM) chirp-z path for 2^14 <= L <= 2^17; opt-in (CJT_CLUSTER=1)
// until it beats the multi-pass path on the benchmark configurations.
bool cluster_enabled();

// vectors per CTA tile of the DMMA contractions, chosen from the batch size
// vector tile: one tile per batch up to 128 vectors (the recurrence is then
// generated once; the warp-specialised producers, not the DMMA width, bound
// the small tiles), 128 beyond
// (24: three 8-vector DMMA tiles per warp, for the 17..24-vector groups of
// ragged batches -- 25 % less padded contraction than a 32-vector tile)
inline int pick_vt(int64_t batch) {
  return batch <= 16 ? 16 : batch <= 24 ? 24 : batch <= 32 ? 32 : batch <= 64 ? 64 : 128;
}

// ---------------------------------------------------------------------------
// launchers (host)
// scratch: multi-pass buffer (batch x m x L complex); part: m-split partial
// sums (m x batch x count doubles), used when too few CTAs would run; spec:
// per-CTA spectrum sums of input-tiled fused chirp-z (chirpz_spec_elems).
// device-side planning of chirp-z products, cjt_plan_dev.cu
struct DevDiag {
  int kind;               // CJT_DIAG_ARRAY: host table; CJT_DIAG_MODULATION: u_m - i v_m of grid rows
  const double2* host;    // [m][len] (array kind)
  int64_t row0;           // modulation kind: grid row of index 0
};
struct PlanGrid {         // what the modulation kind needs (device pointers)
  const double* thetas = nullptr;
  const double* wa = nullptr;
  const double* wb = nullptr;
  double alpha = 0.0, beta = 0.0;
};
// diag[m][t] (from the host or the modulation functions) times chirp(base + t)
int build_device_diag(const DevDiag& dd, int64_t len, int m_count, int64_t base, int64_t G, const PlanGrid& grid,
                      std::vector<void*>& allocs, const double2** out);
// every tile's kernel spectrum, 1/L folded in, in the execution layout `mode`
// (0 natural, 1 two-level on-chip, 2 multi-pass rows, 3 multi-pass two-level rows)
int build_device_spectra(const ChirpZDev& cz, const int64_t* tin_dev, const int64_t* tout_dev, int64_t G,
                         int mode, std::vector<void*>& allocs, const double2** out);
// host natural-order spectra -> device, permuted into layout `mode`
int permute_spectra(const double2* natural_host, int64_t L, int ntile, int mode, int log1, int log2,
                    std::vector<void*>& allocs, const double2** out);

// alpha = beta = 1/2 inverse as exact conversion + bf16 tensor-core correction
// (half_gemm plans), cjt_half.cu.  X: [n1][n1] bf16 (X[k][m] = M[m][k]),
// tbf: [batch][n1] bf16 scratch, corr: [batch][n1] fp32 scratch.
int launch_transpose_bf16(const void* in, void* out, int64_t rows, int64_t cols, cudaStream_t st);
bool umma_half_supported(int64_t n1, int64_t batch);
bool umma_overlap_enabled();   // $CJT_HALF_OVERLAP=1: conversion overlapped with the GEMM (opt-in, slower)
int umma_half_inverse(const double* t, double* out, int64_t n1, int64_t batch, const void* Mrow, void* tbf,
                      const double* k, int* flags, cudaStream_t st);
int half_gemm_inverse(const double* t, double* out, int64_t n1, int64_t batch, const void* X, void* tbf,
                      float* corr, const double* k, cudaStream_t st);
int half_gemm_prepare(cudaStream_t st);   // cuBLAS handle of `st` (outside capture)
int launch_identity(double* buf, int64_t n1, int64_t b0, int64_t nb, cudaStream_t st);
int launch_to_bf16(const double* in, int64_t ldi, void* out, int64_t ldo, int64_t n1, int64_t rows, cudaStream_t st);

// alpha = beta = 1/2 forward (exact U -> T conversion), cjt_half.cu
int launch_half_forward(const double* c, int64_t ldc, double* out, int64_t ldo, const double* k,
                        int64_t n1, int64_t batch, double* scratch, cudaStream_t st);
int64_t half_forward_scratch(int64_t n1);   // doubles per vector (0: one chunk, no scratch)

int launch_chirpz(const ChirpZDev& cz, const double2* tw8192, const double* x, int64_t ldx,
                  double* out, int64_t ldo, int64_t batch, double2* scratch, double* part,
                  double2* spec, cudaStream_t st, int* launches);
// integer parameter shifts (cjt_shift.cu); op = CJT_SHIFT_*
int launch_shift(int op, double alpha, double beta, const double* in, double* out, int64_t n,
                 int64_t batch, cudaStream_t st);
// workspace of one chirp-z at this batch: partial outputs (doubles) and
// spectrum sums (complex elements)
void chirpz_workspace(const ChirpZDev& cz, int64_t batch, int64_t* part_elems, int64_t* spec_elems);

int launch_checkpoints(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                       double2* ck, cudaStream_t st);
// fold: parity-folded contraction (alpha = beta), partials [slot][2][batch][128]
int launch_rec_forward(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                       const double2* ck, const FwdItem* items, int64_t n_items,
                       const double* c, int64_t ldc, int64_t ncoef, int64_t batch, int vt,
                       bool fold, double* part, cudaStream_t st);
int launch_rec_forward_reduce(const int32_t* tile_slot0, const int32_t* tile_nslot,
                              int64_t nrows, const double* part, double* vals, int64_t ldv,
                              int64_t batch, int64_t G, bool fold, cudaStream_t st);
// K2 generator stream: 32 bytes per (work-list row tile, generator thread)
constexpr int GEN_STATE_BYTES = 32;
int launch_build_inv_gen(const RecRowsDev& rows, const int64_t* ck_off, const double2* ck,
                         const int32_t* ids, const int32_t* gn0, int64_t total, void* out,
                         cudaStream_t st);
// fold: parity-folded contraction (alpha = beta) over rows < nrows = G/2 + 1
int launch_rec_inverse(const RecTablesDev& tab, const void* gen, int64_t nrows, const InvItem* items,
                       int64_t n_items, const int32_t* tile_ids, const double* wv, int64_t ldw,
                       int64_t batch, int vt, bool fold, int64_t G, double* part, cudaStream_t st);
int launch_pgen_fwd(const RecRowsDev& rows, const RecTablesDev& tab, const int64_t* ck_off,
                    const double2* ck, const int2* blk_tj, int64_t nblk, double* P, bool fold,
                    cudaStream_t st);
int launch_pgen_inv(const RecTablesDev& tab, const void* gen, const int32_t* gn0, int64_t gbeg,
                    int64_t gend, double* P, cudaStream_t st);
int launch_rec_gemm(const GemmItem* items, int64_t n_items, const double* P, const int32_t* ids,
                    const double* x, int64_t ldx, int64_t xlen, int64_t batch, int vt, bool amk,
                    bool fold, double* part, cudaStream_t st);
int launch_inverse_finish(const int32_t* dt_slot0, const int32_t* dt_nslot, int64_t ndeg,
                          const double* part, const double* blocks_acc, const double* scal,
                          double* out, int64_t ldo, int64_t batch, cudaStream_t st);
int launch_clenshaw_points(const RecTablesDev& tab, const double* rbp, const double* rbm,
                           const double* rbpi, const double* rbmi, const double* coeffs,
                           int64_t ldc, const double* x, const double* xm, const int8_t* reg,
                           const int64_t* cut, double* out, int64_t ldo, int64_t npts,
                           int64_t batch, bool divide, cudaStream_t st);
int launch_jacobi_values(const RecTablesDev& tab, int64_t n_max, const double* x, const double* xm,
                         const int8_t* mode, double* out, int64_t npts, cudaStream_t st);

}  // namespace cjt
