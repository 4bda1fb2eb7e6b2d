// Microbenchmark of the shared-memory Stockham FFT core (cjt_internal.cuh):
// NB batched 2^LOGL-point complex fp64 transforms, forward + inverse, REPS times,
// data resident in shared memory.  Reports element-passes per SM clock and the
// round-trip error (inverse(forward(x)) / L - x).
#include <cstdio>
#include <cmath>
#include <vector>
#include "../paper_1602_02618_b200/csrc/cjt_internal.cuh"
using namespace cjt;

#ifndef LEPT_B
#define LEPT_B 4
#endif
#ifndef MINB
#define MINB 1
#endif
constexpr int EPTB = 1 << LEPT_B;
#ifndef LOGL_B
#define LOGL_B 12
#endif
template <int LOGL>
__global__ void __launch_bounds__((1 << LOGL_B) / EPTB, MINB) k_fft_rt(double2* data, const double2* tw, int reps) {
  constexpr int L = 1 << LOGL, TPG = L / EPTB, NG = 1;
  extern __shared__ double2 sm[];
  const int grp = threadIdx.x / TPG, t = threadIdx.x % TPG;
  double2* s = sm + grp * padded_len(L);
  double2* g = data + ((size_t)blockIdx.x * NG + grp) * L;
  for (int i = 0; i < EPTB; ++i) s[pad16(t + i * TPG)] = g[t + i * TPG];
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    fft_smem<LOGL, -1, LEPT_B>(s, t, tw);
    fft_smem<LOGL, +1, LEPT_B>(s, t, tw);
    for (int i = 0; i < EPTB; ++i) { double2 v = s[pad16(t + i * TPG)]; s[pad16(t + i * TPG)] = make_double2(v.x / L, v.y / L); }
    __syncthreads();
  }
  for (int i = 0; i < EPTB; ++i) g[t + i * TPG] = s[pad16(t + i * TPG)];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::vector<double2> tw(8192);
  for (int u = 0; u < 8192; ++u) { long double a = -2.0L * 3.14159265358979323846264338327950288L * u / 8192; tw[u] = make_double2((double)cosl(a), (double)sinl(a)); }
  double2* dtw; cudaMalloc(&dtw, 8192 * 16); cudaMemcpy(dtw, tw.data(), 8192 * 16, cudaMemcpyHostToDevice);
  const int LOGL = LOGL_B, L = 1 << LOGL;
  const int blocks = sms * 8, n = blocks * L;
  std::vector<double2> h(n);
  for (int i = 0; i < n; ++i) h[i] = make_double2(sin(0.37 * i) , cos(1.3 * i + 0.1));
  double2* d; cudaMalloc(&d, (size_t)n * 16);
  cudaMemcpy(d, h.data(), (size_t)n * 16, cudaMemcpyHostToDevice);
  const int smem = padded_len(L) * 16;
  cudaFuncSetAttribute(k_fft_rt<LOGL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_fft_rt<LOGL><<<blocks, L / EPTB, smem>>>(d, dtw, 1);
  cudaDeviceSynchronize();
  std::vector<double2> o(n); cudaMemcpy(o.data(), d, (size_t)n * 16, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < n; ++i) err = fmax(err, fmax(fabs(o[i].x - h[i].x), fabs(o[i].y - h[i].y)));
  cudaMemcpy(d, h.data(), (size_t)n * 16, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 50;
  cudaEventRecord(e0); k_fft_rt<LOGL><<<blocks, L / EPTB, smem>>>(d, dtw, reps); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double passes = 2.0 * reps * ((LOGL + LEPT_B - 1) / LEPT_B);
  const double ep = passes * (double)n;
  printf("LEPT=%d MINB=%d LOGL=%d blocks=%d: %.3f ms, %.2f elem-passes/clk/SM (clk %d MHz), %.1f GFLOP/s nominal (5 L log2 L), rt err %.3e, %s\n",
         LEPT_B, MINB, LOGL, blocks, ms, ep / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000,
         2.0 * reps * 5.0 * LOGL * n / (ms * 1e-3) / 1e9, err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
