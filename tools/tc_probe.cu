// Standalone check of the tcgen05 kind::i8 GEMM core (csrc/tc_gemm.cuh):
// descriptors, TMA boxes, TMEM layout, the tile schedule and the pipeline,
// against a CPU product of random 0/1 matrices; then its throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -o tools/tc_probe tools/tc_probe.cu -lcuda
// Run:   tools/tc_probe [M N K density]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "../paper_0905_1744_b200/csrc/tc_gemm.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

using namespace sa::tc;

struct WriteEpi {
  int32_t* C;
  int64_t ldc;
  struct State {};
  static constexpr int TAB_BYTES = 16;
  __host__ __device__ static constexpr int xpose_bytes(int, bool, int) { return 0; }
  __device__ bool skip() const { return false; }
  __device__ void begin(State&, const Tile&, int, int, int, int, uint8_t*) const {}
  template <int CW, bool FP4, int CG>
  __device__ void chunk(State&, const Tile& T, int row, int col, const uint32_t (&v)[CW], int, const uint8_t*,
                        int, uint8_t*) const {
    if (row >= T.ra) return;
    const int pi = T.pi;
    int32_t* out = C + (int64_t)pi * 0 + (int64_t)(T.row0 + row) * ldc + T.col0 + col;
#pragma unroll
    for (int j = 0; j < CW; ++j)
      if (col + j < T.rb) out[j] = (int32_t)v[j];
  }
  template <int CW>
  __device__ void correct(State&, int, uint32_t (&)[CW]) const {}
  __device__ void end(State&, const Tile&, int) const {}
  __device__ void finish(int) const {}
};

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void make_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int64_t ld, int box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld};
  const cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)r); exit(1); }
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 300;
  const int N = argc > 2 ? atoi(argv[2]) : 700;
  const int K = argc > 3 ? atoi(argv[3]) : 1024;   // multiple of 128
  const double dens = argc > 4 ? atof(argv[4]) : 0.3;
  const int sym = argc > 5 ? atoi(argv[5]) : 0;
  const int Nb = sym ? M : N;
  std::vector<uint8_t> A((size_t)M * K), B((size_t)Nb * K);
  srand(1234);
  for (auto& x : A) x = (rand() / (double)RAND_MAX) < dens;
  for (auto& x : B) x = (rand() / (double)RAND_MAX) < dens;
  uint8_t *dA, *dB;
  int32_t *dC, *dkb;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dC, (size_t)M * Nb * 4));
  CK(cudaMalloc(&dkb, 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0xff, (size_t)M * Nb * 4));
  const int kb = K / BK;
  CK(cudaMemcpy(dkb, &kb, 4, cudaMemcpyHostToDevice));
  Batch batch{};
  batch.n = 1;
  batch.group = 8;
  Problem& P = batch.p[0];
  P.na = M;
  P.nb = Nb;
  P.sym = sym;
  P.tiles_n = (Nb + Geo<false>::BN - 1) / Geo<false>::BN;
  P.tile_begin = 0;
  P.kblocks = dkb;
  P.map = 0;
  Maps maps;
  memset(&maps, 0, sizeof maps);
  make_map(&maps.m[0], dA, M, K, BM);
  make_map(&maps.m[1], sym ? dA : dB, Nb, K, Geo<false>::BN);
  const int64_t tiles = problem_tiles<Geo<false>::BN>(M, Nb, sym);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(gemm_kernel<WriteEpi, 8, 32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_of(8, 32, false, 16, 0)));
  WriteEpi epi{dC, Nb};
  const int grid = (int)(tiles < sms ? tiles : sms);
  gemm_kernel<WriteEpi, 8, 32, false><<<grid, threads_of(8), smem_of(8, 32, false, 16, 0)>>>(batch, maps, tiles, epi);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> C((size_t)M * Nb);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  const uint8_t* Bh = sym ? A.data() : B.data();
  long bad = 0, checked = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < Nb; ++j) {
      if (sym && (j / Geo<false>::BN) < (i / BM) / 2) continue;   // tile not scheduled
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += A[(size_t)i * K + k] * Bh[(size_t)j * K + k];
      ++checked;
      if (C[(size_t)i * Nb + j] != ref) {
        if (bad < 10) printf("mismatch C[%d][%d] = %d, want %d\n", i, j, C[(size_t)i * Nb + j], ref);
        ++bad;
      }
    }
  printf("check M=%d N=%d K=%d sym=%d tiles=%lld: %ld / %ld wrong\n", M, Nb, K, sym, (long long)tiles, bad, checked);

  // throughput
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 5;
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) gemm_kernel<WriteEpi, 8, 32, false><<<grid, threads_of(8), smem_of(8, 32, false, 16, 0)>>>(batch, maps, tiles, epi);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double ops = 2.0 * tiles * BM * Geo<false>::BN * (double)K;
  printf("time %.3f ms, %.1f TOPS (tile ops incl. padding)\n", ms, ops / ms / 1e9);
  return bad ? 2 : 0;
}
