// Microbenchmark: dependent DFMA chain latency on one warp, alone and with
// DMMA-issuing warps on the same SM (is the recurrence producers' chain
// slowed by the consumers' tensor-pipe work?).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* sink, long long* clk, int iters, int dmma_warps) {
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    double x = threadIdx.x * 1e-9 + 0.5;
    const double m = 0.999999999, c = 1e-12;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int r = 0; r < 32; ++r) x = fma(x, m, c);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    if (x == 1234.5) sink[threadIdx.x] = x;
  } else if (warp <= dmma_warps) {
    double a = 1e-3 * (threadIdx.x & 31), b = 1.0 - 1e-6 * (threadIdx.x & 31);
    double c[8][2];
    for (int u = 0; u < 8; ++u) { c[u][0] = u; c[u][1] = -u; }
    for (int i = 0; i < iters * 4; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
    double s = 0; for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
    if (s == 1234.5) sink[threadIdx.x] = s;
  }
}

int main() {
  double* sink; long long* clk;
  cudaMalloc(&sink, 1 << 20); cudaMalloc(&clk, 1024 * 8);
  const int iters = 2000;
  for (int dw : {0, 1, 3, 7, 15}) {
    k_lat<<<148, 32 * (dw + 1)>>>(sink, clk, iters, dw);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("dmma warps %2d: dependent DFMA latency %.1f clk\n", dw, avg / (iters * 32.0));
  }
  return 0;
}
