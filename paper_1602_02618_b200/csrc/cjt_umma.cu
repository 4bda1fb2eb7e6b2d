// alpha = beta = 1/2 inverse on the 5th-generation tensor cores (sm_100a):
//
//   out[b][m] = u_m / k_m + sum_k M[m][k] t[b][k],   u = E t (exact T -> U)
//
// M is the plan's (N+1) x (N+1) first-order correction to the reference's
// evaluation points (cjt_half.cu, cjt_capi.cu: build_half_gemm_matrix), bf16,
// row-major [m][k]; t the Chebyshev input, fp64, and tbf its bf16 copy.  The
// correction is ~1e-12 ||t||_1, so bf16 operands with fp32 accumulation carry
// it to ~1e-15 ||t||_1; the exact part and the sum stay fp64.
//
// CTA pairs (clusters of 2, tcgen05 cta_group::2), one persistent CTA per
// SM, warp-specialised:
//   warp 0  TMA producer (both CTAs): this CTA's 128 x 64 tile of M (A,
//           K-major) and its half (128 x 64) of the pair's 256-vector bf16
//           tile (B), 128-byte swizzled, into a kStages ring; the bytes of
//           both CTAs complete the LEADER's full barrier;
//   warp 1  allocates 512 TMEM columns per CTA (two 128 x 256 fp32
//           accumulators); the leader's elected lane issues
//           tcgen05.mma.cta_group::2 (M = 256 over the pair's two A tiles,
//           N = 256 over both B halves, K = 16); tcgen05.commit multicasts
//           the stage release and the finished accumulator to both CTAs;
//   warps 2-17 epilogue, four groups of four warps (one per TMEM lane
//           quarter): tcgen05.ld (32x32b.x8) gives each thread one output
//           coefficient m (its TMEM lane) for 8 consecutive vectors b; the
//           fp64 rows t[b][m0 .. m0 + 129] of those vectors arrive by a TMA
//           tile load into the group's double buffer (one chunk ahead), the
//           exact part (two fp64 FMAs) is added and the result written
//           straight to HBM, coalesced across the warp, while the MMAs
//           already accumulate the next tile in the other TMEM buffer; the
//           threads of both CTAs release an accumulator on the leader's
//           barrier.
// Measured on B200 (config 3, N = 4095, 8192 vectors): 239 us; the MMA side
// alone (epilogue skipped, CJT_UMMA_DBG=1) 170 us = 1.62 PF/s (bf16 burst
// peak 1.65); one CTA per SM with cta_group::1 and 3 stages: 251 us (MMA
// side 195 us).
// Pair tiles: 256 output coefficients m x 256 vectors b, K = N + 1 in steps of 64.
#include <cuda_bf16.h>

#include <cstdlib>

#include "cjt_internal.cuh"
#include "cjt_tma.cuh"

namespace cjt {
namespace {

constexpr int kBM = 128;            // output coefficients per tile (TMEM lanes)
constexpr int kBK = 64;             // bf16 elements per 128-byte swizzled row
constexpr int kABytes = kBM * kBK * 2;    // 16 KB
constexpr int kEpiGroupsC = 4;
constexpr int kTW = kBM + 2;                              // t tile width: m0 .. m0 + 129
constexpr int kTRows = 8;                                 // vectors per epilogue chunk
constexpr int kTBytes = kTRows * kTW * 8;                 // 8.3 KB
constexpr int kEpiGroups = kEpiGroupsC;       // epilogue warp groups (4 warps: one per TMEM lane quarter)
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kThreads = 64 + 32 * kEpiWarps;

constexpr uint32_t kPeerMask = 0xFEFFFFFFu;   // shared::cluster address bit 24 = CTA rank in the pair

// per vector-tile width BN (256, or 128 for small batches: more pair tiles)
template <int BN>
struct UCfg {
  static constexpr int BBytes = (BN / 2) * kBK * 2;     // this CTA's half of the pair's B tile
  static constexpr int StageBytes = kABytes + BBytes;
  static constexpr int Stages = BN == 256 ? 4 : 6;
  static constexpr int Smem = Stages * StageBytes + kEpiGroupsC * 2 * kTBytes + 1024;
  static constexpr uint32_t TmemCols = 2 * BN;
  static constexpr uint32_t Idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)((2 * kBM) >> 4) << 24);
};

// shared-memory matrix descriptor, K-major, 128-byte swizzle: 8-row core
// groups 1024 bytes apart (SBO), version 1 (sm_100), layout type 2
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// both CTAs of the pair load into their own shared memory; the bytes are
// counted on the LEADER's (rank 0) barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar) & kPeerMask), "l"(policy)
      : "memory");
}

// L2 eviction policies: the operand tiles (M: re-read by every vector tile;
// the bf16 vectors: re-read by the 16 coefficient tiles of their vector tile)
// must stay in L2 while the epilogue streams t in and the result out
__device__ __forceinline__ uint64_t l2_policy(int kind) {   // 0 normal, 1 evict_last, 2 evict_first
  uint64_t p;
  if (kind == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 2)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// arrive on this barrier in both CTAs of the pair once the leader's MMAs completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void umma_bf16_pair(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// arrive on the leader CTA's copy of this barrier
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 8 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------------------
// fp64 -> bf16 conversion of the input, overlapped with the GEMM: the
// conversion kernel lets its dependent launch at once (programmatic dependent
// launch), walks the rows in order in units of kUnitElems elements and counts
// finished units per 128-row group; the GEMM's TMA producers wait for a group's
// count before their first load of its rows.  One persistent wave of small
// CTAs (no shared memory), which stay resident next to the GEMM's CTAs.
constexpr int kGroupRows = 128;
constexpr int kUnitElems = 16384;

__device__ __forceinline__ void wait_group(const int* flag, int need) {
  int v = 0;
  for (int spins = 0; spins < (1 << 22); ++spins) {   // (bounded: a lost signal must not hang the GPU)
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= need) break;
    __nanosleep(100);
  }
  asm volatile("fence.proxy.async;" ::: "memory");   // generic-proxy writes -> TMA (async proxy) reads
}

__global__ void __launch_bounds__(256) k_to_bf16_flagged(const double* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                                         int64_t n1, int64_t rows, int* __restrict__ flags) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t gelems = (int64_t)kGroupRows * n1, total = rows * n1;
  const int64_t upg = (gelems + kUnitElems - 1) / kUnitElems;
  const int64_t nunits = ((rows + kGroupRows - 1) / kGroupRows) * upg;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t g = u / upg, gbeg = g * gelems, gend = min(total, gbeg + gelems);
    const int64_t e0 = gbeg + (u % upg) * kUnitElems, e1 = min(gend, e0 + kUnitElems);
#pragma unroll 4
    for (int64_t q = e0 / 4 + threadIdx.x; q < e1 / 4; q += 256) {   // (N + 1) % 8 == 0: whole quads
      const double2 a = __ldcs(reinterpret_cast<const double2*>(in) + 2 * q);
      const double2 b = __ldcs(reinterpret_cast<const double2*>(in) + 2 * q + 1);
      __nv_bfloat162 lo, hi;
      lo.x = __double2bfloat16(a.x);
      lo.y = __double2bfloat16(a.y);
      hi.x = __double2bfloat16(b.x);
      hi.y = __double2bfloat16(b.y);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&lo);
      w.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out)[q] = w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(flags + g, 1);
    }
  }
}

template <int BN, int DBG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_half_inv_umma(const __grid_constant__ CUtensorMap map_m, const __grid_constant__ CUtensorMap map_t,
                    const __grid_constant__ CUtensorMap map_x,
                    const double* __restrict__ t, const double* __restrict__ kt, double* __restrict__ out, int n1,
                    int batch, int hints, const int* __restrict__ flags, int flag_need) {
  using C = UCfg<BN>;
  constexpr int kBN = BN, kStages = C::Stages, kStageBytes = C::StageBytes;
  constexpr uint32_t kTmemCols = C::TmemCols;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
  __shared__ __align__(8) uint64_t xbar[kEpiGroups][2];   // fp64 t tiles of the epilogue groups
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA pairs (clusters of 2): pair tile = 256 coefficients m x 256 vectors
  // b; CTA rank r owns m rows [m0 + 128 r, + 128) (its A tile, its TMEM
  // accumulator, its epilogue) and loads B rows [b0 + 128 r, + 128); the
  // leader (rank 0) issues the cta_group::2 MMAs over both CTAs' tiles
  const int rank = blockIdx.x & 1, cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int mpt = (n1 + 2 * kBM - 1) / (2 * kBM), bt = (batch + kBN - 1) / kBN;
  const int tiles = mpt * bt;
  const int kblocks = (n1 + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * 32 * kEpiWarps);   // (the leader's) both CTAs' epilogue threads
      for (int g = 0; g < kEpiGroups; ++g) mbar_init(&xbar[g][a], 1);
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_m)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_t)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();                            // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {
      // TMA producer
      int s = 0;
      uint32_t ph = 0;
      const uint64_t pol_a = l2_policy(hints & 3), pol_b = l2_policy((hints >> 2) & 3);
      for (int tile = cid; tile < tiles; tile += ncl) {
        const int m0 = (tile % mpt) * 2 * kBM + rank * kBM, b0 = (tile / mpt) * kBN + rank * (kBN / 2);
        // overlapped conversion (k_to_bf16_flagged runs concurrently): the bf16
        // rows of this tile's 128-row group must be complete
        if (flags && b0 < batch) wait_group(flags + b0 / kGroupRows, flag_need);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);      // the pair's MMAs are done with this stage
          uint8_t* sa = smem + s * kStageBytes;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * kStageBytes);   // both CTAs' bytes
          tma_load_2d_pair(sa, &map_m, kb * kBK, m0, &full[s], pol_a);
          tma_load_2d_pair(sa + kABytes, &map_t, kb * kBK, b0, &full[s], pol_b);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // MMA issuer (the pair's leader)
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = cid; tile < tiles; tile += ncl, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * kBN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          const uint64_t ad = sw128_desc(sa), bd = sw128_desc(sa + kABytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)   // 32 bytes along K per step: +2 in the 16-byte address field
            umma_bf16_pair(d, ad + 2 * k, bd + 2 * k, C::Idesc, (kb | k) != 0);
          umma_commit_pair(&empty[s]);         // the stage is free in both CTAs once these MMAs completed
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc]);         // both CTAs' accumulators complete
      }
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31; group g = (w - 2) / 4
    // takes the 16-vector chunks g, g + kEpiGroups, ... of every tile.  The
    // fp64 rows t[b][m0 .. m0 + 129] of a chunk arrive by one TMA tile load
    // into the group's double buffer (issued one chunk ahead), so the HBM
    // reads need no registers; the results go out as coalesced stores.
    const int q = warp & 3;
    const int grp = (warp - 2) >> 2;
    const bool leader = (warp == 2 + 4 * grp) && lane == 0;
    double* xb = reinterpret_cast<double*>(smem + kStages * kStageBytes + grp * 2 * kTBytes);
    constexpr int kChunks = kBN / (kTRows * kEpiGroups);   // per tile and group
    const int my_tiles = tiles > cid ? (tiles - 1 - cid) / ncl + 1 : 0;
    const int nseq = my_tiles * kChunks;
    const uint64_t pol_x = l2_policy((hints >> 4) & 3);
    auto issue_x = [&](int sq) {   // leader: t tile of chunk sq of this group's sequence
      if (sq >= nseq) return;
      const int tile = cid + (sq / kChunks) * ncl;
      const int c0 = kTRows * (grp + kEpiGroups * (sq % kChunks));
      uint64_t* br = &xbar[grp][sq & 1];
      mbar_expect_tx(br, kTBytes);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
          "%3}], [%4], %5;" ::"r"(smem_u32(xb + (sq & 1) * (kTRows * kTW))),
          "l"(reinterpret_cast<uint64_t>(&map_x)), "r"((tile % mpt) * 2 * kBM + rank * kBM),
          "r"((tile / mpt) * kBN + c0),
          "r"(smem_u32(br)), "l"(pol_x)
          : "memory");
    };
    if (leader && !(DBG & (5 | 64))) issue_x(0);
    int it = 0, sq = 0;
    for (int tile = cid; tile < tiles; tile += ncl, ++it) {
      const int acc = it & 1;
      const int m0 = (tile % mpt) * 2 * kBM + rank * kBM, b0 = (tile / mpt) * kBN;
      const int ml = q * 32 + lane;          // row of the t tile
      const int m = m0 + ml;
      const bool mv = m < n1;
      // out = c_t t_m - c_h t_{m+2} + corr: T_0 = U_0, T_j = (U_j - U_{j-2}) / 2
      const double inv_k = mv ? 1.0 / __ldg(kt + m) : 0.0;
      const double c_h = 0.5 * inv_k, c_t = m == 0 ? inv_k : c_h;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      if constexpr (DBG & 1) {   // timing experiment: accumulator read only, no HBM traffic
        float v[8];
        tmem_ld8(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kBN), v);
        if (v[0] == 12345.f) out[0] = v[1];
        tc_fence_before();
        mbar_arrive_leader(&tempty[acc]);
        sq += kChunks;
      } else {
#pragma unroll 1
      for (int c0 = kTRows * grp; c0 < kBN; c0 += kTRows * kEpiGroups, ++sq) {
        // (DBG bits, timing experiments only: 2 no result stores, 4 no t tiles,
        // 8 no fp64 arithmetic, 16 no accumulator loads)
        if (leader && !(DBG & (4 | 64))) issue_x(sq + 1);         // its buffer was released by the barrier below
        double gt[kTRows], gh[kTRows];
        if constexpr (DBG & 64) {   // experiment: t rows straight from global memory into registers
#pragma unroll
          for (int j = 0; j < kTRows; ++j) {
            const int b = b0 + c0 + j;
            const double* tp = t + (int64_t)b * n1 + m;
            gt[j] = (mv && b < batch) ? __ldg(tp) : 0.0;
            gh[j] = (m + 2 < n1 && b < batch) ? __ldg(tp + 2) : 0.0;
          }
        }
        float v[kTRows];
        if constexpr (DBG & 16) {
#pragma unroll
          for (int j = 0; j < kTRows; ++j) v[j] = (float)(c0 + j);
        } else {
          tmem_ld8(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * kBN + c0), v);
        }
        if constexpr (!(DBG & (4 | 64))) mbar_wait(&xbar[grp][sq & 1], (uint32_t)((sq >> 1) & 1));
        const double* xr = xb + (sq & 1) * (kTRows * kTW);
#pragma unroll
        for (int j = 0; j < kTRows; ++j) {
          const int b = b0 + c0 + j;
          double tm = 1.0, hi = 2.0;
          if constexpr (DBG & 64) {
            tm = gt[j];
            hi = gh[j];
          } else if constexpr (!(DBG & 4)) {
            tm = xr[j * kTW + ml];
            if constexpr (DBG & 32) {   // experiment: t_{m+2} from lane + 2 (shuffle), shared memory for the last two lanes
              const double hs = __shfl_down_sync(0xffffffffu, tm, 2);
              hi = hs;
              if (lane >= 30) hi = xr[j * kTW + ml + 2];
            } else {
              hi = xr[j * kTW + ml + 2];   // zero past N+1 (TMA fill)
            }
          }
          double r;
          if constexpr (DBG & 8)
            r = __hiloint2double(__double2hiint(tm) ^ __double2loint(hi), __double2loint(tm) ^ __float_as_int(v[j]));
          else
            r = fma(c_t, tm, fma(-c_h, hi, (double)v[j]));
          if constexpr (DBG & 2) {
            if (mv && b < batch && __double2loint(r) == 0x12345678 && __double2hiint(r) == 0x7654321)
              __stcs(out + (int64_t)b * n1 + m, r);
          } else {
            if (mv && b < batch) __stcs(out + (int64_t)b * n1 + m, r);
          }
        }
        if constexpr (!(DBG & 64))
          asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");   // the group is done with this buffer
      }
      tc_fence_before();
      mbar_arrive_leader(&tempty[acc]);   // the leader may reuse this accumulator (both CTAs)
      }
    }
  }
  tc_fence_before();
  cluster_sync();                            // no remote arrive or MMA still targets this CTA
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                 : "memory");
  }
}

// row-major [rows][cols] bf16, box = box_rows x 64, 128-byte swizzle
int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  return tmap_make(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// row-major [rows][cols] fp64, box = box_rows x box_cols, no swizzle
int make_map_f64(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows, int box_cols) {
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  return tmap_make(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

}  // namespace

bool umma_half_supported(int64_t n1, int64_t batch) {
  return n1 % 8 == 0 && n1 <= 0x7fffffff && batch <= 0x7fffffff && !getenv("CJT_HALF_CUBLAS");
}

template <int BN, int DBG>
int launch_umma_dbg(const CUtensorMap& mm, const void* tbf, const CUtensorMap& mx, const double* t, const double* k,
                    double* out, int64_t n1, int64_t batch, int sms, const int* flags, cudaStream_t st) {
  static DeviceOnce once;
  if (int rc = once([] {
        CJT_CUDA_TRY(cudaFuncSetAttribute(k_half_inv_umma<BN, DBG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          UCfg<BN>::Smem));
        return CJT_OK;
      }))
    return rc;
  CUtensorMap mt;
  if (int rc = make_map(&mt, tbf, batch, n1, BN / 2)) return rc;
  const int64_t tiles = ((n1 + 2 * kBM - 1) / (2 * kBM)) * ((batch + BN - 1) / BN);
  const unsigned grid = 2 * (unsigned)std::min<int64_t>(tiles, sms / 2);   // CTA pairs
  // L2 policies of the TMA loads: M | vectors << 2 | fp64 t tiles << 4 (0 normal, 1 evict_last, 2 evict_first)
  static const int hints = getenv("CJT_UMMA_HINTS") ? atoi(getenv("CJT_UMMA_HINTS")) : 37;
  const int need = (int)(((int64_t)kGroupRows * n1 + kUnitElems - 1) / kUnitElems);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = UCfg<BN>::Smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;   // start while the conversion kernel runs
  cfg.attrs = attr;
  cfg.numAttrs = flags ? 1 : 0;
  CJT_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_half_inv_umma<BN, DBG>, mm, mt, mx, t, k, out, (int)n1, (int)batch, hints,
                                  flags, need));
  return CJT_OK;
}

template <int BN>
int launch_umma(const CUtensorMap& mm, const void* tbf, const CUtensorMap& mx, const double* t, const double* k,
                double* out, int64_t n1, int64_t batch, int sms, const int* flags, cudaStream_t st) {
  // $CJT_UMMA_DBG (timing experiments): 1 = epilogue without HBM traffic;
  // builds with -DCJT_UMMA_DBG_BUILD also have the partial epilogues (bit mask, see the kernel)
  static const int dbg = getenv("CJT_UMMA_DBG") ? atoi(getenv("CJT_UMMA_DBG")) : 0;
  switch (dbg) {
#define CJT_UD(D) case D: return launch_umma_dbg<BN, D>(mm, tbf, mx, t, k, out, n1, batch, sms, flags, st);
    CJT_UD(1)
#ifdef CJT_UMMA_DBG_BUILD
    CJT_UD(2) CJT_UD(4) CJT_UD(6) CJT_UD(8) CJT_UD(12) CJT_UD(14) CJT_UD(16) CJT_UD(30) CJT_UD(10) CJT_UD(32) CJT_UD(64)
#endif
#undef CJT_UD
    default: return launch_umma_dbg<BN, 0>(mm, tbf, mx, t, k, out, n1, batch, sms, flags, st);
  }
}

bool umma_overlap_enabled() {
  // opt-in: measured slower on B200 (config 3: 0.420 vs 0.382 ms per step) -- the
  // conversion's HBM traffic slows the GEMM's operand and epilogue streams by
  // more than the 46 us it hides
  const char* e = getenv("CJT_HALF_OVERLAP");   // (read per call: tests switch it)
  return e && atoi(e) == 1;
}

// flags != nullptr: tbf is NOT converted yet -- the conversion runs here,
// overlapped with the GEMM (flags: one int per 128 vectors, scratch)
int umma_half_inverse(const double* t, double* out, int64_t n1, int64_t batch, const void* Mrow, void* tbf,
                      const double* k, int* flags, cudaStream_t st) {
  if (batch <= 0) return CJT_OK;
  if (((uintptr_t)t & 15) != 0) return fail(CJT_EINVAL, "umma_half_inverse: input must be 16-byte aligned");
  if (flags) {
    const int64_t ngroups = (batch + kGroupRows - 1) / kGroupRows;
    CJT_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)ngroups * sizeof(int), st));
    int dev0 = 0, sms0 = 148;
    CJT_CUDA_TRY(cudaGetDevice(&dev0));
    CJT_CUDA_TRY(cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0));
    const int64_t nunits = ngroups * (((int64_t)kGroupRows * n1 + kUnitElems - 1) / kUnitElems);
    k_to_bf16_flagged<<<(unsigned)std::min<int64_t>(nunits, 2 * sms0), 256, 0, st>>>(
        t, reinterpret_cast<__nv_bfloat16*>(tbf), n1, batch, flags);
    CJT_CUDA_TRY(cudaGetLastError());
  }
  CUtensorMap mm, mx;
  if (int rc = make_map(&mm, Mrow, n1, n1, kBM)) return rc;
  if (int rc = make_map_f64(&mx, t, batch, n1, kTRows, kTW)) return rc;
  int dev = 0, sms = 148;
  CJT_CUDA_TRY(cudaGetDevice(&dev));
  CJT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // 256-vector tiles, or 128 when they would leave CTA pairs idle (small
  // batches, e.g. one GPU's shard of a multi-GPU batch); the arithmetic of a
  // vector does not depend on the tile width (same K order, same epilogue)
  // (waves x tile time, tile time ~ width; ties go to the wider tile)
  const int64_t mpt = (n1 + 2 * kBM - 1) / (2 * kBM), pairs = std::max(1, sms / 2);
  const int64_t cost256 = 2 * ((mpt * ((batch + 255) / 256) + pairs - 1) / pairs);
  const int64_t cost128 = (mpt * ((batch + 127) / 128) + pairs - 1) / pairs;
  if (cost128 < cost256 && !getenv("CJT_UMMA_BN256"))
    return launch_umma<128>(mm, tbf, mx, t, k, out, n1, batch, sms, flags, st);
  return launch_umma<256>(mm, tbf, mx, t, k, out, n1, batch, sms, flags, st);
}

}  // namespace cjt
