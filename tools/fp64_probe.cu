// fp64 pipe throughput on the live GPU (why the K2T matrix epilogue avoids
// fp64): DFMA, DMUL and I2F.F64 warp-instructions per SM per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, double s) {
  double a[8];
  unsigned u = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001 + i;
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma(a[i], s, 0.5);
      else if (MODE == 1) a[i] = a[i] * s;
      else { a[i] += (double)(u + i); u = u * 3 + 1; }
    }
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 1.2345) out[0] = r;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[3] = {"DFMA", "DMUL", "I2F.F64+DADD"};
  for (int m = 0; m < 3; ++m) {
    const int iters = 4096, threads = 1024, blocks = sms * 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<blocks, threads>>>(d, iters, 1.0000001);
      if (m == 1) k<1><<<blocks, threads>>>(d, iters, 1.0000001);
      if (m == 2) k<2><<<blocks, threads>>>(d, iters, 1.0000001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 8;
    printf("%s: %.1f Gop/s = %.1f lane-ops/clk/SM at %d MHz\n", names[m], ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
