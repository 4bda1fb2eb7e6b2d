// Microbenchmark: fp64 FMA (DFMA) vs fp64 MMA (mma.sync m8n8k4 f64, DMMA) throughput on one GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* sink, int iters) {
  double a[8];
  for (int u = 0; u < 8; ++u) a[u] = threadIdx.x * 1e-9 + u;
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = fma(a[u], m, c);
  }
  double s = 0; for (int u = 0; u < 8; ++u) s += a[u];
  if (s == 1234.5) sink[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma(double* sink, int iters) {
  double a = 1e-3 * (threadIdx.x & 31), b = 1.0 - 1e-6 * (threadIdx.x & 31);
  double c[NACC][2];
  for (int u = 0; u < NACC; ++u) { c[u][0] = u; c[u][1] = -u; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < NACC; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int u = 0; u < NACC; ++u) s += c[u][0] + c[u][1];
  if (s == 1234.5) sink[threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink; cudaMalloc(&sink, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int tpb : {256, 512}) {
    for (int bps : {2, 4, 8}) {
      int blocks = sms * bps, iters = 2048;
      k_dfma<<<blocks, tpb>>>(sink, 16);
      cudaEventRecord(e0); k_dfma<<<blocks, tpb>>>(sink, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * 8 * (double)iters * tpb * blocks;
      printf("DFMA tpb=%d blocks/SM=%d: %.2f TFLOP/s\n", tpb, bps, fl / ms / 1e9);
    }
  }
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, iters = 4096;
      k_dmma<8><<<blocks, tpb>>>(sink, 16);
      cudaEventRecord(e0); k_dmma<8><<<blocks, tpb>>>(sink, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 512.0 * 8 * (double)iters * (tpb / 32) * blocks;
      printf("DMMA(8 acc) tpb=%d blocks/SM=%d: %.2f TFLOP/s\n", tpb, bps, fl / ms / 1e9);
      k_dmma<2><<<blocks, tpb>>>(sink, 16);
      cudaEventRecord(e0); k_dmma<2><<<blocks, tpb>>>(sink, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 512.0 * 2 * (double)iters * (tpb / 32) * blocks;
      printf("DMMA(2 acc) tpb=%d blocks/SM=%d: %.2f TFLOP/s\n", tpb, bps, fl / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
