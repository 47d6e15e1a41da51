// Integer / half pipe-rate probe for the min-sum engine.
// Measures, on the live B200, warp-instructions issued per SM per cycle for the
// instruction mixes the dense min-sum of Eq. 1 can lower to:
//   VIMNMX.U16x2 (min.u16x2), HMNMX2 (min.f16x2 on count bit patterns),
//   IMAD (mad.lo with an opaque 1: an add on the FMA pipe), IADD3 (3-input add).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

#define VMIN(d, a, b) asm volatile("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b))
#define HMIN(d, a, b) asm volatile("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b))
#define IMAD(acc, m, one) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc) : "r"(m), "r"(one))
#define IADD3(acc, m1, m2) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(acc) : "r"(m1), "r"(m2))

// MODE (warp-instructions per inner step in kInstr): 0 VIMNMX+HMNMX2+IADD3+LOP3, 1 2xHMNMX2+IADD3,
//       2 IMAD only, 3 IADD3 only, 4 VIMNMX+IMAD+LOP3, 5 HMNMX2+IMAD+LOP3, 6 VIMNMX+HMNMX2+IADD3,
//       7 2xVIMNMX+IADD3, 8 mix 1 VIMNMX + 3 HMNMX2 + 2 IADD3 per 4 words
template <int MODE>
__global__ void __launch_bounds__(256) probe(uint32_t* out, uint64_t* cyc, uint64_t* ns, uint32_t one, int iters) {
  uint32_t a[8], b[8], acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * (i + 3); b[i] = threadIdx.x ^ (i * 77); acc[i] = i; }
  __syncthreads();
  uint64_t c0 = clock64(), t0 = gtime();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t m, m2;
        if (MODE == 0) { VMIN(m, a[i], b[i]); HMIN(m2, b[i], a[i]); IADD3(acc[i], m, m2); b[i] ^= acc[i]; }
        if (MODE == 1) { HMIN(m, a[i], b[i]); HMIN(m2, b[i], acc[i]); IADD3(acc[i], m, m2); }
        if (MODE == 2) { IMAD(acc[i], a[i], one); }
        if (MODE == 3) { IADD3(acc[i], a[i], b[i]); }
        if (MODE == 4) { VMIN(m, a[i], b[i]); IMAD(acc[i], m, one); b[i] ^= acc[i]; }
        if (MODE == 5) { HMIN(m, a[i], b[i]); IMAD(acc[i], m, one); b[i] ^= acc[i]; }
        if (MODE == 6) { VMIN(m, a[i], acc[i]); HMIN(m2, b[i], acc[i]); IADD3(acc[i], m, m2); }
        if (MODE == 7) { VMIN(m, a[i], b[i]); VMIN(m2, b[i], acc[i]); IADD3(acc[i], m, m2); }
        if (MODE == 8) {
          uint32_t m3, m4;
          VMIN(m, a[i], acc[i]); HMIN(m2, b[i], acc[i]); HMIN(m3, a[i], acc[i]); HMIN(m4, acc[i], b[i]);
          IADD3(acc[i], m, m2); IADD3(acc[i], m3, m4);
        }
      }
    }
  }
  uint64_t c1 = clock64(), t1 = gtime();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i] + b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[blockIdx.x] = c1 - c0; ns[blockIdx.x] = t1 - t0; }
}

// warp-instructions per inner (i) step of each mode, as counted in SASS terms
static const double kInstr[9] = {4, 3, 1, 1, 3, 3, 3, 3, 6};
static const char* kName[9] = {"VIMNMX+HMNMX2+IADD3+LOP3", "2xHMNMX2+IADD3", "IMAD(add)", "IADD3 (2 adds fused)",
                               "VIMNMX+IMAD+LOP3", "HMNMX2+IMAD+LOP3", "VIMNMX+HMNMX2+IADD3", "2xVIMNMX+IADD3",
                               "VIMNMX+3xHMNMX2+2xIADD3"};

template <int MODE>
int run(int sms, int occ, int threads) {
  int grid = sms * occ;
  uint32_t* out; uint64_t *cyc, *ns;
  CK(cudaMalloc(&out, grid * threads * 4)); CK(cudaMalloc(&cyc, grid * 8)); CK(cudaMalloc(&ns, grid * 8));
  int iters = 4096;
  probe<MODE><<<grid, threads>>>(out, cyc, ns, 1u, 16);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<grid, threads>>>(out, cyc, ns, 1u, iters);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  uint64_t hc[4096], hn[4096];
  CK(cudaMemcpy(hc, cyc, grid * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hn, ns, grid * 8, cudaMemcpyDeviceToHost));
  double cmax = 0, nmax = 0;
  for (int i = 0; i < grid; ++i) { if (hc[i] > cmax) cmax = hc[i]; if (hn[i] > nmax) nmax = hn[i]; }
  double mhz = cmax / nmax * 1e3;
  double warp_instr = (double)grid * threads / 32 * iters * 4 * 8 * kInstr[MODE];
  double per_sm_clk = warp_instr / sms / cmax;
  printf("{\"mode\": %d, \"name\": \"%s\", \"threads\": %d, \"occ\": %d, \"warp_instr_per_sm_clk\": %.3f, "
         "\"lane_ops_per_sm_clk\": %.1f, \"sm_mhz\": %.0f, \"ms\": %.3f}\n",
         MODE, kName[MODE], threads, occ, per_sm_clk, per_sm_clk * 32, mhz, ms);
  cudaFree(out); cudaFree(cyc); cudaFree(ns);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  int sms = p.multiProcessorCount;
  for (int occ : {2, 4}) {
    run<0>(sms, occ, 256); run<1>(sms, occ, 256); run<2>(sms, occ, 256); run<3>(sms, occ, 256);
    run<4>(sms, occ, 256); run<5>(sms, occ, 256); run<6>(sms, occ, 256); run<7>(sms, occ, 256);
    run<8>(sms, occ, 256);
  }
  return 0;
}
