// alpha = beta = 1/2 forward: the exact Jacobi -> Chebyshev conversion.
//
// P_n^{(1/2,1/2)} = k_n U_n with k_n = P_n(1)/(n+1), and
// U_n = sum_{j <= n, j = n mod 2} e_j T_j (e_0 = 1, e_j = 2), so
//   cheb_j = e_j sum_{n >= j, n = j (mod 2)} k_n c_n,
// two suffix sums (even / odd degrees) per vector.  This is the terminating
// m = 0 term of the Hahn expansion the reference's partition leaves unused
// for this pair (see cjt_host.cpp); the forward is insensitive to the
// reference's evaluation points (<= 2e-16 ||c||_1), so the
// closed form matches its results to rounding (tests/test_gpu_half.py).
//
// HBM-bound: 16 B per coefficient (read c, write cheb) plus the k table
// (L2-resident).  One CTA per vector walks the vector from the top in tiles
// of 4 * kThreads pairs: every thread forms the exact products k_n c_n
// (two_prod) and its local suffix sums in double-double, a block-wide
// exclusive suffix scan of the thread totals (warp shuffles + one shared
// exchange) adds the higher part, and the carry moves to the next tile; the
// result is rounded once.

#include <cublas_v2.h>
#include <cuda_bf16.h>

#include <map>
#include <mutex>

#include "cjt_internal.cuh"

namespace cjt {
namespace {

constexpr int kThreads = 256;
constexpr int kPairs = 4;              // (even, odd) coefficient pairs per thread per tile
constexpr int kTile = 2 * kPairs * kThreads;

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd dd_add(dd a, dd b) {
  const double s = a.hi + b.hi;
  const double bb = s - a.hi;
  double e = (a.hi - (s - bb)) + (b.hi - bb);
  e += a.lo + b.lo;
  const double h = s + e;
  return dd{h, e - (h - s)};
}

__device__ __forceinline__ dd dd_prod(double a, double b) {
  const double p = a * b;
  return dd{p, fma(a, b, -p)};
}

__device__ __forceinline__ dd shfl_down_dd(dd v, int d) {
  return dd{__shfl_down_sync(0xffffffffu, v.hi, d), __shfl_down_sync(0xffffffffu, v.lo, d)};
}

__global__ void __launch_bounds__(kThreads) k_half_forward(const double* __restrict__ c, int64_t ldc,
                                                           double* __restrict__ out, int64_t ldo,
                                                           const double* __restrict__ kt, int64_t n1) {
  const int64_t b = blockIdx.x;
  const double* cb = c + b * ldc;
  double* ob = out + b * ldo;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ dd s_warp[2][kThreads / 32];
  // thread-owned runs of 2 kPairs entries, padded to an odd stride (bank spread)
  constexpr int kRun = 2 * kPairs + 1;
  __shared__ double s_tile[kThreads * kRun];
  dd carry_e{0.0, 0.0}, carry_o{0.0, 0.0};   // sums of all higher tiles (even / odd degrees)
  const int64_t ntiles = (n1 + kTile - 1) / kTile;
  for (int64_t t = ntiles - 1; t >= 0; --t) {
    const int64_t t0 = t * kTile;
    // coalesced tile load, then each thread takes 2 kPairs consecutive entries
#pragma unroll
    for (int e = 0; e < 2 * kPairs; ++e) {
      const int64_t j = t0 + e * kThreads + threadIdx.x;
      const int l = e * kThreads + threadIdx.x;
      s_tile[(l / (2 * kPairs)) * kRun + l % (2 * kPairs)] = j < n1 ? cb[j] : 0.0;
    }
    __syncthreads();
    const int64_t base = t0 + (int64_t)threadIdx.x * (2 * kPairs);
    double v[2 * kPairs];
#pragma unroll
    for (int e = 0; e < 2 * kPairs; ++e) v[e] = s_tile[threadIdx.x * kRun + e];
    // local suffix sums, exact products
    dd se{0.0, 0.0}, so{0.0, 0.0};
    dd loc[2 * kPairs];
#pragma unroll
    for (int e = 2 * kPairs - 1; e >= 0; --e) {
      const int64_t j = base + e;
      const dd pr = j < n1 ? dd_prod(__ldg(kt + j), v[e]) : dd{0.0, 0.0};
      if (e & 1) {
        so = dd_add(so, pr);
        loc[e] = so;
      } else {
        se = dd_add(se, pr);
        loc[e] = se;
      }
    }
    // inclusive suffix scan of (se, so) over the threads of the block
    dd ie = se, io = so;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const dd ue = shfl_down_dd(ie, d), uo = shfl_down_dd(io, d);
      if (lane + d < 32) {
        ie = dd_add(ie, ue);
        io = dd_add(io, uo);
      }
    }
    if (lane == 0) {
      s_warp[0][warp] = ie;
      s_warp[1][warp] = io;
    }
    __syncthreads();
    // higher warps' totals and the carry of the higher tiles
    dd he = carry_e, ho = carry_o;
    for (int w = kThreads / 32 - 1; w > warp; --w) {
      he = dd_add(he, s_warp[0][w]);
      ho = dd_add(ho, s_warp[1][w]);
    }
    // exclusive (this thread's higher neighbours within the warp)
    const dd xe = shfl_down_dd(ie, 1), xo = shfl_down_dd(io, 1);
    if (lane < 31) {
      he = dd_add(he, xe);
      ho = dd_add(ho, xo);
    }
    __syncthreads();   // every thread has read its inputs from s_tile
#pragma unroll
    for (int e = 0; e < 2 * kPairs; ++e) {
      const int64_t j = base + e;
      const dd s = dd_add(loc[e], (e & 1) ? ho : he);
      s_tile[threadIdx.x * kRun + e] = (j == 0 ? 1.0 : 2.0) * s.hi;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 2 * kPairs; ++e) {
      const int64_t j = t0 + e * kThreads + threadIdx.x;
      const int l = e * kThreads + threadIdx.x;
      if (j < n1) ob[j] = s_tile[(l / (2 * kPairs)) * kRun + l % (2 * kPairs)];
    }
    // carry for the next (lower) tile: every warp's total
    dd te = carry_e, to = carry_o;
    for (int w = kThreads / 32 - 1; w >= 0; --w) {
      te = dd_add(te, s_warp[0][w]);
      to = dd_add(to, s_warp[1][w]);
    }
    carry_e = te;
    carry_o = to;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// alpha = beta = 1/2 inverse, small / moderate N (half_gemm plans):
//   out = E t + M t,
// E t the exact Chebyshev -> Jacobi conversion (T_0 = U_0, T_j = (U_j -
// U_{j-2}) / 2, c_m = u_m / k_m: two coefficients per output), and M the
// (N+1) x (N+1) first-order correction that moves the evaluation to the
// reference's points (cjt_host.cpp), built once per plan by running the
// synthesis + correction chirp-z products on the identity.  |M t| is ~1e-12
// ||t||_1 (the reference's own deviation from the exact transform at
// N = 4095), so M and t in bf16 with fp32 accumulation are ~1e3 x more
// accurate than needed: the contraction runs on the tensor cores (cuBLAS
// GemmEx; 2 (N+1)^2 flop per vector).

__global__ void k_to_bf16(const double* __restrict__ in, int64_t ldi, __nv_bfloat16* __restrict__ out,
                          int64_t ldo, int64_t n1, int64_t rows) {
  const int64_t total = n1 * rows;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n1, c = e % n1;
    out[r * ldo + c] = __double2bfloat16(in[r * ldi + c]);
  }
}

__global__ void k_identity(double* buf, int64_t n1, int64_t b0, int64_t nb) {
  const int64_t total = n1 * nb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n1, c = e % n1;
    buf[e] = (c == b0 + r) ? 1.0 : 0.0;
  }
}

__global__ void k_half_inv_finish(const double* __restrict__ t, int64_t ldt, const float* __restrict__ corr,
                                  int64_t ldc, const double* __restrict__ kt, double* __restrict__ out,
                                  int64_t ldo, int64_t n1, int64_t batch) {
  const int64_t total = n1 * batch;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / n1, m = e % n1;
    const double* tb = t + b * ldt;
    const double hi = m + 2 < n1 ? tb[m + 2] : 0.0;
    const double u = (m == 0 ? tb[0] - 0.5 * hi : 0.5 * (tb[m] - hi));
    out[b * ldo + m] = u / kt[m] + (double)corr[b * ldc + m];
  }
}

inline unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32); }

struct BlasKey {
  int dev;
  cudaStream_t st;
  bool operator<(const BlasKey& o) const { return dev != o.dev ? dev < o.dev : st < o.st; }
};

// one cuBLAS handle per (device, stream), with its own workspace so calls are
// capturable into CUDA graphs; created outside capture (first use / plan build)
int blas_handle(cudaStream_t st, cublasHandle_t* out) {
  static std::map<BlasKey, cublasHandle_t> handles;
  static std::mutex mu;
  int dev = 0;
  CJT_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = handles.find(BlasKey{dev, st});
  if (it != handles.end()) {
    *out = it->second;
    return CJT_OK;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone)
    return fail(CJT_EINVAL, "cuBLAS handle for this stream must exist before graph capture (run once uncaptured)");
  cublasHandle_t h;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return fail(CJT_ECUDA, "cublasCreate failed");
  void* ws = nullptr;
  const size_t wsb = size_t(32) << 20;
  CJT_CUDA_TRY(cudaMalloc(&ws, wsb));
  if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS || cublasSetWorkspace(h, ws, wsb) != CUBLAS_STATUS_SUCCESS)
    return fail(CJT_ECUDA, "cublasSetStream / cublasSetWorkspace failed");
  handles[BlasKey{dev, st}] = h;
  *out = h;
  return CJT_OK;
}

}  // namespace

int launch_identity(double* buf, int64_t n1, int64_t b0, int64_t nb, cudaStream_t st) {
  k_identity<<<grid_for(n1 * nb), 256, 0, st>>>(buf, n1, b0, nb);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int launch_to_bf16(const double* in, int64_t ldi, void* out, int64_t ldo, int64_t n1, int64_t rows, cudaStream_t st) {
  k_to_bf16<<<grid_for(n1 * rows), 256, 0, st>>>(in, ldi, (__nv_bfloat16*)out, ldo, n1, rows);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int half_gemm_inverse(const double* t, double* out, int64_t n1, int64_t batch, const void* X, void* tbf,
                      float* corr, const double* k, cudaStream_t st) {
  if (batch <= 0) return CJT_OK;
  if (int rc = launch_to_bf16(t, n1, tbf, n1, n1, batch, st)) return rc;
  cublasHandle_t h;
  if (int rc = blas_handle(st, &h)) return rc;
  const float one = 1.0f, zero = 0.0f;
  // column-major view: corr (n1 x B) = X^T-as-stored (n1 x n1, X[k][m] = M[m][k]) . t^T (n1 x B)
  if (cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)n1, (int)batch, (int)n1, &one, X, CUDA_R_16BF, (int)n1, tbf,
                   CUDA_R_16BF, (int)n1, &zero, corr, CUDA_R_32F, (int)n1, CUBLAS_COMPUTE_32F,
                   CUBLAS_GEMM_DEFAULT) != CUBLAS_STATUS_SUCCESS)
    return fail(CJT_ECUDA, "cublasGemmEx failed");
  k_half_inv_finish<<<grid_for(n1 * batch), 256, 0, st>>>(t, n1, corr, n1, k, out, n1, n1, batch);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

int half_gemm_prepare(cudaStream_t st) {
  cublasHandle_t h;
  return blas_handle(st, &h);
}

int launch_half_forward(const double* c, int64_t ldc, double* out, int64_t ldo, const double* k,
                        int64_t n1, int64_t batch, cudaStream_t st) {
  if (batch <= 0) return CJT_OK;
  if (batch > 0x7fffffffLL) return fail(CJT_EINVAL, "batch too large");
  k_half_forward<<<(unsigned)batch, kThreads, 0, st>>>(c, ldc, out, ldo, k, n1);
  CJT_CUDA_TRY(cudaGetLastError());
  return CJT_OK;
}

}  // namespace cjt
