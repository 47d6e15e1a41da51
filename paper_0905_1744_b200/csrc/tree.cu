// N4 -- the guide tree of a bucket (PAPER.md P:133-136:
// "This similarity matrix is then used to build a guide tree"; SPEC.md
// build_guide_tree S:277-285: UPGMA, ties to the smaller (min id, max id)
// pair).  Readings T1-T3: d = 1 - F, cluster id = smallest
// member, F(ab, c) = RN(RN(RN(n_a F_ac) + RN(n_b F_bc)) / (n_a + n_b)),
// height = (1 - F_ab) / 2.
//
// Each row i of the working matrix keeps its best active partner
// (bval[i], bidx[i]): the largest F over active k != i, ties to the smallest
// k -- which is the smallest (min, max) pair for that row.  A merge is the
// best row-best (ties to the smallest pair), found by one block reduction;
// merging (a, b) rewrites row / column a with the size-weighted averages,
// rescans row a and every row whose best partner was a or b, and lets any
// other row adopt a if a's new entry beats its best.  So every merge costs
// O(n) plus one O(n) block scan per rescanned row, in one CTA (the merges are
// sequential); the first row-bests come from a grid-wide kernel.  A 12 500-row
// bucket takes ~1.5 s (tools/tree_bench.py): ~120 us per merge, three
// latency-bound passes over n entries on one SM.
#include "common.cuh"

namespace sa {

constexpr int UT = 1024;   // threads of the merge CTA

// (v1, k1) better than (v2, k2) for one row: larger F, ties to the smaller k
__device__ __forceinline__ bool row_better(double v1, int k1, double v2, int k2) {
  return v1 > v2 || (v1 == v2 && k1 < k2);
}
// the global order on candidate pairs (v, a < b)
__device__ __forceinline__ bool pair_better(double v1, int a1, int b1, double v2, int a2, int b2) {
  if (v1 != v2) return v1 > v2;
  if (a1 != a2) return a1 < a2;
  return b1 < b2;
}

// first row-bests: one warp per row
__global__ void upgma_init_kernel(const double* __restrict__ S, int n, int64_t ld, double* __restrict__ bval,
                                  int32_t* __restrict__ bidx) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double v = -1.0 / 0.0;
    int k = 0x7fffffff;
    for (int c = lane; c < n; c += 32) {
      if (c == i) continue;
      const double x = S[i * ld + c];
      if (row_better(x, c, v, k)) { v = x; k = c; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int ok = __shfl_xor_sync(0xffffffffu, k, o);
      if (row_better(ov, ok, v, k)) { v = ov; k = ok; }
    }
    if (lane == 0) {
      bval[i] = v;
      bidx[i] = k;
    }
  }
}

// block-wide best over a row's active columns (all threads call; returns to all)
__device__ void block_row_best(const double* __restrict__ row, int self, int n, const uint8_t* __restrict__ active,
                               double* s_v, int* s_k, double& bv, int& bk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double v = -1.0 / 0.0;
  int k = 0x7fffffff;
  for (int c = tid; c < n; c += UT) {
    if (c == self || !active[c]) continue;
    const double x = row[c];
    if (row_better(x, c, v, k)) { v = x; k = c; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int ok = __shfl_xor_sync(0xffffffffu, k, o);
    if (row_better(ov, ok, v, k)) { v = ov; k = ok; }
  }
  if (lane == 0) { s_v[warp] = v; s_k[warp] = k; }
  __syncthreads();
  if (warp == 0) {
    v = s_v[lane];
    k = s_k[lane];
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int ok = __shfl_xor_sync(0xffffffffu, k, o);
      if (row_better(ov, ok, v, k)) { v = ov; k = ok; }
    }
    if (lane == 0) { s_v[32] = v; s_k[32] = k; }
  }
  __syncthreads();
  bv = s_v[32];
  bk = s_k[32];
  __syncthreads();
}

__global__ void __launch_bounds__(UT) upgma_merge_kernel(double* __restrict__ S, int n, int64_t ld,
                                                         double* __restrict__ bval, int32_t* __restrict__ bidx,
                                                         int32_t* __restrict__ size, uint8_t* __restrict__ active,
                                                         int32_t* __restrict__ resc, int32_t* __restrict__ merges,
                                                         double* __restrict__ heights) {
  __shared__ double s_v[33];
  __shared__ int s_k[33], s_a[33], s_b[33];
  __shared__ int s_nres;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < n; i += UT) {
    active[i] = 1;
    size[i] = 1;
  }
  __syncthreads();
  for (int m = 0; m + 1 < n; ++m) {
    // 1. the best active pair
    double v = -1.0 / 0.0;
    int a = 0x7fffffff, b = 0x7fffffff;
    for (int i = tid; i < n; i += UT) {
      if (!active[i]) continue;
      const int k = bidx[i];
      const int lo = min(i, k), hi = max(i, k);
      if (pair_better(bval[i], lo, hi, v, a, b)) { v = bval[i]; a = lo; b = hi; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oa = __shfl_xor_sync(0xffffffffu, a, o), ob = __shfl_xor_sync(0xffffffffu, b, o);
      if (pair_better(ov, oa, ob, v, a, b)) { v = ov; a = oa; b = ob; }
    }
    if (lane == 0) { s_v[warp] = v; s_a[warp] = a; s_b[warp] = b; }
    if (tid == 0) s_nres = 0;
    __syncthreads();
    if (warp == 0) {
      v = s_v[lane];
      a = s_a[lane];
      b = s_b[lane];
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oa = __shfl_xor_sync(0xffffffffu, a, o), ob = __shfl_xor_sync(0xffffffffu, b, o);
        if (pair_better(ov, oa, ob, v, a, b)) { v = ov; a = oa; b = ob; }
      }
      if (lane == 0) { s_v[32] = v; s_a[32] = a; s_b[32] = b; }
    }
    __syncthreads();
    v = s_v[32];
    a = s_a[32];
    b = s_b[32];
    if (tid == 0) {
      merges[2 * m] = a;
      merges[2 * m + 1] = b;
      heights[m] = __dmul_rn(__dadd_rn(1.0, -v), 0.5);
    }
    // 2. row / column a <- the size-weighted averages of rows a and b
    const double na = (double)size[a], nb = (double)size[b], nab = (double)(size[a] + size[b]);
    for (int c = tid; c < n; c += UT) {
      if (!active[c] || c == a || c == b) continue;
      const double x = __ddiv_rn(__dadd_rn(__dmul_rn(na, S[(int64_t)a * ld + c]), __dmul_rn(nb, S[(int64_t)b * ld + c])), nab);
      S[(int64_t)a * ld + c] = x;
      S[(int64_t)c * ld + a] = x;
      // 3. row c's best partner: a rescan if it was a or b, else adopt a if better
      const int k = bidx[c];
      if (k == a || k == b) resc[atomicAdd(&s_nres, 1)] = c;
      else if (row_better(x, a, bval[c], k)) { bval[c] = x; bidx[c] = a; }
    }
    __syncthreads();
    if (tid == 0) {
      size[a] += size[b];
      active[b] = 0;
    }
    __syncthreads();
    // 4. rescans: row a, then the rows whose partner was a or b (few: one
    // block-wide scan each beats one warp per row, measured)
    const int nres = s_nres;
    for (int r = -1; r < nres; ++r) {
      const int row = r < 0 ? a : resc[r];
      double bv;
      int bk;
      block_row_best(S + (int64_t)row * ld, row, n, active, s_v, s_k, bv, bk);
      if (tid == 0) {
        bval[row] = bv;
        bidx[row] = bk;
      }
    }
    __syncthreads();
  }
}

sa_status upgma_launch(const double* F, int32_t n, int64_t ld, int32_t* merges, double* heights, cudaStream_t st) {
  if (n <= 1) return SA_OK;
  Scratch scratch(st);
  SA_ALLOC(S, double, (size_t)n * n);
  SA_ALLOC(bval, double, n);
  SA_ALLOC(bidx, int32_t, n);
  SA_ALLOC(size, int32_t, n);
  SA_ALLOC(active, uint8_t, n);
  SA_ALLOC(resc, int32_t, n);
  SA_CUDA(cudaMemcpy2DAsync(S, (size_t)n * sizeof(double), F, (size_t)ld * sizeof(double), (size_t)n * sizeof(double),
                            (size_t)n, cudaMemcpyDeviceToDevice, st));
  const int64_t warps = n;
  upgma_init_kernel<<<(unsigned)std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16), 256, 0, st>>>(S, n, n, bval,
                                                                                                  bidx);
  SA_LAUNCHED();
  upgma_merge_kernel<<<1, UT, 0, st>>>(S, n, n, bval, bidx, size, active, resc, merges, heights);
  SA_LAUNCHED();
  return SA_OK;
}

}  // namespace sa
