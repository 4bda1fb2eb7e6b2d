// Ceiling of the K1/K2 consumer loop: per k-step, 4 A + NT B fragments loaded
// from shared memory (same layouts/strides as the kernels) feeding 4 x NT
// DMMA m8n8k4 f64; no producers, no barriers inside the stage.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NT, int NWARPS, int SYNC>
__global__ void __launch_bounds__(NWARPS * 32) k(double* out, int stages) {
  constexpr int PT = 132, CS = 36;
  __shared__ double Pt[32][PT];
  __shared__ double Cs[32][CS];
  const int tid = threadIdx.x, lane = tid & 31, warp = (tid >> 5) & 3, wn = tid >> 7;
  for (int i = tid; i < 32 * PT; i += blockDim.x) (&Pt[0][0])[i] = 1e-3 * (i % 97);
  for (int i = tid; i < 32 * CS; i += blockDim.x) (&Cs[0][0])[i] = 1e-3 * (i % 89);
  __syncthreads();
  const int ar = lane >> 2, ak = lane & 3;
  double acc[4][NT][2] = {};
  for (int s = 0; s < stages; ++s) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      double a[4], b[NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = Pt[4 * kk + ak][32 * warp + 8 * mt + ar];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) b[nt] = Cs[((wn * NT + nt) * 8 + ar) & 31][4 * kk + ak];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    if (SYNC) __syncthreads();
  }
  double sum = 0;
  for (int mt = 0; mt < 4; ++mt) for (int nt = 0; nt < NT; ++nt) sum += acc[mt][nt][0] + acc[mt][nt][1];
  if (sum == 12345.0) out[tid] = sum;
}

template <int NT, int NWARPS, int SYNC>
void run(const char* name, int blocks_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8192 * 8);
  const int stages = 2000, blocks = sms * blocks_per_sm;
  k<NT, NWARPS, SYNC><<<blocks, NWARPS * 32>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<NT, NWARPS, SYNC><<<blocks, NWARPS * 32>>>(out, stages); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * 4 * NT * 8 * (double)stages * NWARPS * blocks;
  printf("%-28s blocks/SM=%d: %.2f TFLOP/s  %s\n", name, blocks_per_sm, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<8, 4, 0>("NT8 4warps nosync", 1);  run<8, 4, 0>("NT8 4warps nosync", 2);
  run<8, 8, 0>("NT8 8warps nosync", 1);  run<8, 8, 1>("NT8 8warps sync", 1);
  run<4, 8, 0>("NT4 8warps nosync", 1);  run<4, 8, 0>("NT4 8warps nosync", 2);
  run<4, 16, 0>("NT4 16warps nosync", 1); run<4, 16, 1>("NT4 16warps sync", 1);
  run<2, 8, 0>("NT2 8warps nosync", 2);
  return 0;
}
