// Device-side planning of the chirp-z products:
// chirp phases, the diagonal tables with their chirps folded in, the
// modulation functions u_m - i v_m of the asymptotic blocks
// (asymptotics.py:36-75), and the Bluestein kernel spectra of every tile
// (planner._spectrum; a radix-2 Stockham FFT at plan time), laid out in the order the
// execution kernels read them.  The host only decides the tiling.
//
// Numerics: chirp(k) = exp(i pi k^2 / (2G)) with k^2 reduced exactly mod 4G in
// integers and the phase r / (2G) split into a double-double before sincospi,
// so each chirp is within ~1 ulp; the modulation tables follow the reference's
// operation order in double.  Both enter the transforms as diagonal factors
// whose last-bit differences are far below the transform tolerance
// (tests/test_gpu_plan_dev.py compares device- and host-built plans).

#include <utility>

#include "cjt_internal.cuh"

namespace cjt {
namespace {

// exp(i pi k^2 / (2G)) (SIGN = +1) or its conjugate (SIGN = -1)
template <int SIGN>
__device__ __forceinline__ double2 chirp_dev(int64_t k, int64_t G) {
  const int64_t four_g = 4 * G;
  int64_t km = k % four_g;
  if (km < 0) km += four_g;
  // k^2 mod 4G without overflow: |km| < 4G <= 2^26 here, km^2 < 2^52
  const int64_t r = (int64_t)(((unsigned long long)km * (unsigned long long)km) % (unsigned long long)four_g);
  const double den = (double)(2 * G);
  const double hi = (double)r / den;                  // phase / pi = r / (2G) in [0, 2)
  const double lo = fma(-hi, den, (double)r) / den;   // exact remainder
  double s, c;
  sincospi(hi, &s, &c);
  const double pl = 3.141592653589793238462643383279502884 * lo;
  const double cs = fma(-s, pl, c), sn = fma(c, pl, s);
  return make_double2(cs, SIGN * sn);
}

// diag[m][t] *= chirp(base + t), in place
__global__ void k_fold_chirp(double2* diag, int64_t len, int m_count, int64_t base, int64_t G) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= len) return;
  const double2 ch = chirp_dev<1>(base + t, G);
  for (int m = 0; m < m_count; ++m) diag[m * len + t] = cmul(diag[m * len + t], ch);
}

// u_m(theta) - i v_m(theta) at grid rows row0 + t (asymptotics.py:36-75,
// engine.py:133-141), operation order of planner.modulation
__global__ void k_modulation(double2* out, int64_t len, int m_count, int64_t row0, const double* __restrict__ thetas,
                             double a, double b, const double* __restrict__ wa, const double* __restrict__ wb) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= len) return;
  const double th = thetas[row0 + t];
  const double sh = sin(0.5 * th), ch = cos(0.5 * th);
  const double phase = (a + b + 1.0) * 0.5 * th - (a + 0.5) * 0.5 * 3.141592653589793;
  double re = cos(phase), im = sin(phase);
  const double scale0 = 1.0 / (pow(sh, a + 0.5) * pow(ch, b + 0.5));
  for (int m = 0; m < m_count; ++m) {
    double cr = re, ci = im;
    double scale = scale0 * pow(ch, -(double)m);
    double um = 0.0, vm = 0.0;
    for (int l = 0; l <= m; ++l) {
      const double rho = wa[l] * wb[m - l];
      if (rho != 0.0) {
        um += rho * cr * scale;
        vm -= rho * ci * scale;
      }
      if (l < m) {
        const double tmp = cr;
        cr = ci;
        ci = -tmp;
        scale = scale * ch / sh;
      }
    }
    out[m * len + t] = make_double2(um, -vm);   // u - i v
    const double nre = re * ch - im * sh, nim = re * sh + im * ch;
    re = nre;
    im = nim;
  }
}

// Bluestein kernel of every tile (planner._spectrum before its FFT):
// ker[t] = conj(chirp(off + t)) for t < count_j, ker[L - w_i + 1 + u] =
// conj(chirp(off - (w_i - 1 - u))) for u < w_i - 1, zero elsewhere.
__global__ void k_spectrum_kernels(double2* ker, int64_t L, int n_in, int n_out, const int64_t* __restrict__ tin,
                                   const int64_t* __restrict__ tout, int64_t p0, int64_t q0, int64_t G) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int tile = blockIdx.y;   // j * n_in + i
  if (t >= L) return;
  const int j = tile / n_in, i = tile % n_in;
  const int64_t off = (q0 + tout[2 * j]) - (p0 + tin[2 * i]);
  const int64_t cnt = tout[2 * j + 1], w = tin[2 * i + 1];
  double2 v = make_double2(0.0, 0.0);
  if (t < cnt)
    v = chirp_dev<-1>(off + t, G);
  else if (t >= L - w + 1)
    v = chirp_dev<-1>(off - (L - t), G);
  ker[(int64_t)tile * L + t] = v;
}

// natural-order spectra (1/L folded in here) -> the execution kernels' layout
__global__ void k_permute_khat(const double2* __restrict__ src, double2* __restrict__ dst, int64_t L, int mode,
                               int log1, int log2, double scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tile = blockIdx.y;
  if (e >= L) return;
  const double2* s = src + tile * L;
  double2* d = dst + tile * L;
  int64_t from = e;
  if (mode == 1) {   // two-level on-chip FFT: position k1 S + k2 holds k1 + 16 k2
    const int64_t S = L / 16, k1 = e / S, k2 = e % S;
    from = k1 + 16 * k2;
  } else if (mode >= 2) {   // multi-pass rows: [k1][pos(k2)] holds k1 + L1 k2
    const int64_t L2 = (int64_t)1 << log2, L1 = (int64_t)1 << log1;
    const int64_t k1 = e / L2, pos = e % L2;
    int64_t k2 = pos;
    if (mode == 3) {   // rows run the two-level FFT: pos = (k2 % 16) S2 + k2 / 16
      const int64_t S2 = L2 / 16;
      k2 = (pos % S2) * 16 + pos / S2;
    }
    from = k1 + L1 * k2;
  }
  const double2 v = s[from];
  d[e] = make_double2(v.x * scale, v.y * scale);
}

// One radix-2 Stockham pass (forward, exp(-2 pi i ...)) over `ntile`
// independent transforms of length L = 2^n: pass with Ns = 2^p reads
// in[j], in[j + L/2] and writes the butterfly at (j / Ns) 2 Ns + j % Ns (+ Ns).
// Plan-time only (every tile's Bluestein kernel spectrum): log2 L launches,
// twiddles from sincospi, error O(log L) ulp like any radix-2 FFT.
__global__ void k_fft_r2_pass(const double2* __restrict__ in, double2* __restrict__ out, int64_t L, int64_t ns) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tile = blockIdx.y;
  const int64_t half = L / 2;
  if (j >= half) return;
  const double2* x = in + tile * L;
  double2* y = out + tile * L;
  const int64_t k = j & (ns - 1);
  double s, c;
  sincospi(-(double)k / (double)ns, &s, &c);
  const double2 v0 = x[j];
  const double2 v1 = cmul(x[j + half], make_double2(c, s));
  const int64_t d = (j - k) * 2 + k;
  y[d] = cadd(v0, v1);
  y[d + ns] = csub(v0, v1);
}

// per-thread grow-only scratch for the unpermuted spectra (no cudaFree, and
// with it no implicit device synchronisation, per plan build)
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = -1;
  ~Scratch() {
    if (p) cudaFree(p);
  }
};
int scratch(size_t bytes, void** out) {
  thread_local Scratch s;
  int dev = 0;
  CJT_CUDA_TRY(cudaGetDevice(&dev));
  if (s.bytes < bytes || s.dev != dev) {
    if (s.p) {
      int cur = dev;
      cudaSetDevice(s.dev);
      cudaFree(s.p);
      cudaSetDevice(cur);
    }
    s.p = nullptr;
    s.bytes = 0;
    CJT_CUDA_TRY(cudaMalloc(&s.p, bytes));
    s.bytes = bytes;
    s.dev = dev;
  }
  *out = s.p;
  return CJT_OK;
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

int dalloc_list(std::vector<void*>& list, void** p, size_t bytes) {
  *p = nullptr;
  cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CJT_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) + ") failed: " +
                                cudaGetErrorString(e));
  }
  list.push_back(*p);
  return CJT_OK;
}

}  // namespace

int build_device_diag(const DevDiag& dd, int64_t len, int m_count, int64_t base, int64_t G, const PlanGrid& grid,
                      std::vector<void*>& allocs, const double2** out) {
  void* p = nullptr;
  if (int rc = dalloc_list(allocs, &p, (size_t)m_count * len * sizeof(double2))) return rc;
  double2* d = (double2*)p;
  if (dd.kind == CJT_DIAG_MODULATION) {
    if (!grid.thetas || !grid.wa || !grid.wb) return fail(CJT_EINVAL, "modulation diagonal needs the plan grid");
    k_modulation<<<blocks_for(len, 128), 128, 0, cudaStreamPerThread>>>(d, len, m_count, dd.row0, grid.thetas, grid.alpha, grid.beta,
                                                 grid.wa, grid.wb);
    CJT_CUDA_TRY(cudaGetLastError());
  } else {
    CJT_CUDA_TRY(cudaMemcpyAsync(d, dd.host, (size_t)m_count * len * sizeof(double2), cudaMemcpyHostToDevice,
                                 cudaStreamPerThread));
  }
  k_fold_chirp<<<blocks_for(len, 256), 256, 0, cudaStreamPerThread>>>(d, len, m_count, base, G);
  CJT_CUDA_TRY(cudaGetLastError());
  *out = d;
  return CJT_OK;
}

int build_device_spectra(const ChirpZDev& cz, const int64_t* tin_dev, const int64_t* tout_dev, int64_t G,
                         int mode, std::vector<void*>& allocs, const double2** out) {
  const int64_t L = cz.length;
  const int ntile = cz.n_in * cz.n_out;
  const size_t elems = (size_t)ntile * L;
  void *kp = nullptr, *dp = nullptr;
  if (int rc = dalloc_list(allocs, &dp, elems * sizeof(double2))) return rc;
  if (int rc = scratch(2 * elems * sizeof(double2), &kp)) return rc;
  double2* a = (double2*)kp;
  double2* b = a + elems;
  cudaStream_t st = cudaStreamPerThread;
  dim3 g1(blocks_for(L, 256), (unsigned)ntile);
  k_spectrum_kernels<<<g1, 256, 0, st>>>(a, L, cz.n_in, cz.n_out, tin_dev, tout_dev, cz.p0, cz.q0, G);
  CJT_CUDA_TRY(cudaGetLastError());
  dim3 gh(blocks_for(L / 2, 256), (unsigned)ntile);
  for (int64_t ns = 1; ns < L; ns *= 2) {
    k_fft_r2_pass<<<gh, 256, 0, st>>>(a, b, L, ns);
    std::swap(a, b);
  }
  CJT_CUDA_TRY(cudaGetLastError());
  k_permute_khat<<<g1, 256, 0, st>>>(a, (double2*)dp, L, mode, cz.log1, cz.log2, 1.0 / (double)L);
  CJT_CUDA_TRY(cudaGetLastError());
  CJT_CUDA_TRY(cudaStreamSynchronize(st));   // the scratch is reused by this thread's next build
  *out = (const double2*)dp;
  return CJT_OK;
}

int permute_spectra(const double2* natural_host, int64_t L, int ntile, int mode, int log1, int log2,
                    std::vector<void*>& allocs, const double2** out) {
  void *sp = nullptr, *dp = nullptr;
  if (int rc = dalloc_list(allocs, &dp, (size_t)ntile * L * sizeof(double2))) return rc;
  if (mode == 0) {
    CJT_CUDA_TRY(cudaMemcpyAsync(dp, natural_host, (size_t)ntile * L * sizeof(double2), cudaMemcpyHostToDevice,
                                 cudaStreamPerThread));
    CJT_CUDA_TRY(cudaStreamSynchronize(cudaStreamPerThread));
    *out = (const double2*)dp;
    return CJT_OK;
  }
  if (int rc = scratch((size_t)ntile * L * sizeof(double2), &sp)) return rc;
  cudaStream_t st = cudaStreamPerThread;
  CJT_CUDA_TRY(cudaMemcpyAsync(sp, natural_host, (size_t)ntile * L * sizeof(double2), cudaMemcpyHostToDevice, st));
  dim3 g1(blocks_for(L, 256), (unsigned)ntile);
  k_permute_khat<<<g1, 256, 0, st>>>((const double2*)sp, (double2*)dp, L, mode, log1, log2, 1.0);
  CJT_CUDA_TRY(cudaGetLastError());
  CJT_CUDA_TRY(cudaStreamSynchronize(st));
  *out = (const double2*)dp;
  return CJT_OK;
}

}  // namespace cjt
