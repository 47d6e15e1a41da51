// Exact-rank key terms shared by the min-sum engines (minsum.cu, minsum_tc.cu):
// key_i = sum_j floor(C_ij 2^64 / D_ij) (DESIGN.md §2 "Exact ranks", Eq. 3 in F
// form) with the reciprocal tables r_d = floor(2^64 / d),
// e_d = 2^64 mod d, so floor(C 2^64 / d) = C r_d + floor(C e_d / d) (C < d);
// the d^F term of SURVEY N1; 128-bit atomics.  The tables have internal
// linkage: each translation unit holds and initialises its own copy.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace sa {

static __device__ uint64_t g_rtab[65536];   // floor(2^64 / d), d >= 2
static __device__ uint32_t g_etab[65536];   // 2^64 mod d
static __device__ double g_rcp[65536];      // RN(1 / d), d >= 1

static __global__ void recip_kernel() {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= 65536) return;
  g_rcp[d] = d ? __drcp_rn((double)d) : 0.0;
  if (d < 2) { g_rtab[d] = 0; g_etab[d] = 0; return; }
  uint64_t r = ~0ull / (uint64_t)d;
  uint64_t e = ~0ull % (uint64_t)d + 1;   // (2^64 - 1) mod d + 1
  if (e == (uint64_t)d) { r += 1; e = 0; }
  g_rtab[d] = r;
  g_etab[d] = (uint32_t)e;
}

// Filled once per device (and per translation unit, which owns its copy of the
// tables), synchronously: the kernel runs on a private stream that is
// synchronised before any caller's work can read the tables, whatever stream
// that work is on (a stream-ordered fill raced with other streams).
static sa_status ensure_recip_tables_tu(cudaStream_t) {
  static DeviceOnce once;
  return once.run([]() -> sa_status {
    cudaStream_t s = nullptr;
    SA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    recip_kernel<<<256, 256, 0, s>>>();
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return fail(SA_E_CUDA, "reciprocal tables: %s", cudaGetErrorString(e));
    return SA_OK;
  });
}

// floor(C * 2^64 / D) accumulated into a 96-bit (lo, hi) register pair.
__device__ __forceinline__ void add_term(uint64_t& lo, uint32_t& hi, uint32_t C, uint32_t D) {
  if (D == 0 || C == 0) return;
  if (C == D) { hi += 1; return; }      // the term is exactly 2^64
  uint64_t t = (uint64_t)C * g_rtab[D] + (uint64_t)((C * g_etab[D]) / D);
  lo += t;
  hi += (lo < t) ? 1u : 0u;
}

// F = C / D rounded to nearest (Z19) without a division: with y = RN(1/D),
// q0 = RN(C y) is within an ulp of C/D, the remainder r = C - q0 D is exact
// (FMA) and RN(q0 + r y) is the correctly rounded quotient (Markstein's
// correction).  Verified against __ddiv_rn for every 0 <= C <= D <= 65535 by
// sa_selftest_f_division (tests/test_gpu_parity.py).
// The same with d = (double)D and y = RN(1/D) supplied (y = 0 for D = 0 gives 0).
__device__ __forceinline__ double f_ratio_y(uint32_t C, double d, double y) {
  // (double)C for C < 2^32 without the quarter-rate I2F.F64: 2^52 + C, minus 2^52 (exact)
  const double c = __hiloint2double(0x43300000, (int)C) - 4503599627370496.0;
  const double q0 = c * y;
  const double r = fma(-q0, d, c);
  return fma(r, y, q0);
}
__device__ __forceinline__ double f_ratio(uint32_t C, uint32_t D) {
  if (D == 0) return 0.0;
  return f_ratio_y(C, (double)D, g_rcp[D]);
}
__device__ __forceinline__ double rcp_of(int n) { return n > 0 ? g_rcp[n] : 0.0; }

// d^F key term: round(2^52 (ln(1+Delta) - ln(Delta + C/D))), F = 0 when D = 0.
__device__ __forceinline__ void add_dF_term(uint64_t& lo, uint32_t& hi, uint32_t C, uint32_t D, double delta,
                                            double ln1pd) {
  const double F = D > 0 ? __ddiv_rn((double)C, (double)D) : 0.0;
  double t = ln1pd - log(delta + F);
  t = t > 0.0 ? t : 0.0;
  const uint64_t q = __double2ull_rn(t * DF_SCALE);
  lo += q;
  hi += (lo < q) ? 1u : 0u;
}

__device__ __forceinline__ void atomic_add_key(sa_key128* k, uint64_t lo, uint64_t hi) {
  unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long*>(&k->lo), (unsigned long long)lo);
  uint64_t carry = ((uint64_t)old + lo < (uint64_t)old) ? 1ull : 0ull;
  uint64_t h = hi + carry;
  if (h) atomicAdd(reinterpret_cast<unsigned long long*>(&k->hi), (unsigned long long)h);
}

__device__ __forceinline__ void shfl_add(uint64_t& lo, uint32_t& hi, int mask) {
  uint64_t olo = __shfl_xor_sync(0xffffffffu, lo, mask);
  uint32_t ohi = __shfl_xor_sync(0xffffffffu, hi, mask);
  lo += olo;
  hi += ohi + ((lo < olo) ? 1u : 0u);
}

static inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

}  // namespace sa
