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
#include <algorithm>
#include <cmath>
#include <vector>

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

// ----------------------------------------------- d^F form (reading T4) ----
// The working matrix of the d^F tree holds S = -d = CR(ln(RN(Delta + F))):
// UPGMA's "smallest d" is then the same "largest S" the merge kernels look
// for, and negation commutes with every RN operation of the update, so the
// merges and heights (h0 = 0: height = -S / 2 = d / 2) are the d-space ones.
// ln in double-double: x = m 2^e, m in [1/sqrt2, sqrt2), ln m = 2 atanh(s),
// s = (m - 1) / (m + 1), |s| <= 0.1716, 21 terms of sum s^(2k+1) / (2k+1)
// (truncation < 2^-104 relative), plus e ln 2; every step an error-free
// transform or a double-double operation (relative error ~2^-104 each), so
// the result is within 2^-96 |ln x| (a generous bound) of the real value.
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b), bb = __dadd_rn(s, -a);
  return {s, __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb))};
}
__device__ __forceinline__ dd dd_fast_two_sum(double a, double b) {   // |a| >= |b|
  const double s = __dadd_rn(a, b);
  return {s, __dadd_rn(b, -__dadd_rn(s, -a))};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  const dd t = dd_two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = dd_fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return dd_fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = __dmul_rn(a.hi, b.hi);
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __fma_rn(a.hi, b.lo, e);
  e = __fma_rn(a.lo, b.hi, e);
  return dd_fast_two_sum(p, e);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = __ddiv_rn(a.hi, b.hi);
  dd r = dd_add(a, dd_mul(dd{-q1, 0.0}, b));
  const double q2 = __ddiv_rn(r.hi, b.hi);
  r = dd_add(r, dd_mul(dd{-q2, 0.0}, b));
  const double q3 = __ddiv_rn(r.hi, b.hi);
  return dd_add(dd_fast_two_sum(q1, q2), dd{q3, 0.0});
}

constexpr int LN_TERMS = 21;
__constant__ dd c_inv_odd[LN_TERMS];   // 1 / (2k + 1) in double-double
static DeviceOnce g_ln_once;

static sa_status ensure_ln_table() {
  return g_ln_once.run([]() -> sa_status {
    dd h[LN_TERMS];
    for (int k = 0; k < LN_TERMS; ++k) {
      const double d = 2.0 * k + 1.0;
      h[k].hi = 1.0 / d;
      h[k].lo = std::fma(-h[k].hi, d, 1.0) / d;   // the remainder 1 - hi d is exact
    }
    SA_CUDA(cudaMemcpyToSymbol(c_inv_odd, h, sizeof h));
    return SA_OK;
  });
}

// CR(ln x) for a finite x > 0; *certified = the rounding is proven correct
__device__ double cr_log(double x, bool* certified) {
  int e;
  double m = frexp(x, &e);   // [0.5, 1)
  if (m < 0.70710678118654752440) {
    m = __dmul_rn(m, 2.0);
    e -= 1;
  }
  const double num = __dadd_rn(m, -1.0);   // exact (Sterbenz)
  const dd s = dd_div(dd{num, 0.0}, dd_two_sum(m, 1.0));
  const dd s2 = dd_mul(s, s);
  dd p = c_inv_odd[LN_TERMS - 1];
  for (int k = LN_TERMS - 2; k >= 0; --k) p = dd_add(dd_mul(p, s2), c_inv_odd[k]);
  dd r = dd_mul(s, p);
  r.hi = __dmul_rn(r.hi, 2.0);
  r.lo = __dmul_rn(r.lo, 2.0);
  const dd ln2 = {6.93147180559945286227e-01, 2.31904681384629955842e-17};
  r = dd_add(dd_mul(ln2, dd{(double)e, 0.0}), r);
  // certified iff [r - E, r + E] stays between the midpoints around r.hi
  const double E = ldexp(fabs(r.hi), -96);
  const double up = __dadd_rn(nextafter(r.hi, 1.0 / 0.0), -r.hi);
  const double dn = __dadd_rn(r.hi, -nextafter(r.hi, -1.0 / 0.0));
  *certified = r.hi == 0.0 ? r.lo == 0.0
                           : (__dadd_rn(r.lo, E) < __dmul_rn(up, 0.5) && __dadd_rn(r.lo, -E) > -__dmul_rn(dn, 0.5));
  return r.hi;
}

__global__ void dF_matrix_kernel(const double* __restrict__ F, int64_t ldf, int n, double delta,
                                 double* __restrict__ S, int64_t lds, unsigned long long* __restrict__ unc) {
  unsigned long long bad = 0;
  const int64_t total = (int64_t)n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    double v = 0.0;
    if (i != j) {
      bool ok;
      v = cr_log(__dadd_rn(delta, F[i * ldf + j]), &ok);
      bad += ok ? 0 : 1;
    }
    S[i * lds + j] = v;
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(unc, bad);
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
                                                         double* __restrict__ heights, double h0) {
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
      heights[m] = __dmul_rn(__dadd_rn(h0, -v), 0.5);
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

__global__ void fill_ones_kernel(int32_t* __restrict__ p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 1;
}
static sa_status fill_ones_i32(int32_t* p, int n, cudaStream_t st) {
  fill_ones_kernel<<<(unsigned)std::min(1024, (n + 255) / 256), 256, 0, st>>>(p, n);
  SA_LAUNCHED();
  return SA_OK;
}

// ------------------------------------------------------------ grid-wide ----
// The same merges with every SM taking part (one cooperative launch, all
// blocks resident, two grid barriers per merge).  Block k owns rows / columns
// [k n / G, (k + 1) n / G).  Per merge m:
//   1. (every block, redundantly) finish merge m - 1: row a and the rows
//      that were rescanned take their best from the partials of steps 2 / 3;
//      then the global best active pair from those and the blocks' partials
//      of the other rows -- merge m's (a, b);
//   2. each block over its columns c: the size-weighted average x of rows a
//      and b (row / column a), adoption of a by row c when x beats its best,
//      a rescan flag when row c's best partner was a or b; its partial best
//      over its rows that are not being rescanned; its partial best of row a's
//      new entries;                                               [barrier]
//   3. the flagged rows' scans: q column chunks per row (ug_chunks), one
//      warp per (row, chunk), spread over the grid's warps.       [barrier]
// Every value is computed by the same IEEE operations in the same order as in
// upgma_merge_kernel, and every reduction uses the same total order (largest F,
// ties to the smaller index / pair), so the tree is identical.
struct GridBest {
  double v;
  int a, b;
};
constexpr int UG_T = 256;       // threads per block
constexpr int UG_W = UG_T / 32;

// step 3's work split for nf flagged rows: q column chunks per row, q * nf
// units spread over the grid's gw warps (at least 64 columns per chunk)
__device__ __forceinline__ int ug_chunks(int nf, int n, int gw) {
  return max(1, min(gw / max(nf, 1), n / 64));
}

__device__ __forceinline__ void warp_pair_best(double& v, int& a, int& b) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oa = __shfl_xor_sync(0xffffffffu, a, o), ob = __shfl_xor_sync(0xffffffffu, b, o);
    if (pair_better(ov, oa, ob, v, a, b)) { v = ov; a = oa; b = ob; }
  }
}
__device__ __forceinline__ void warp_row_best(double& v, int& k) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int ok = __shfl_xor_sync(0xffffffffu, k, o);
    if (row_better(ov, ok, v, k)) { v = ov; k = ok; }
  }
}

// One bucket's tree on blocks [g0, g0 + G) of the cooperative launch.
struct UgTask {
  double* S;
  int64_t ld;
  int n, g0, G;
  double* bval;
  int32_t* bidx;
  int32_t* size;
  uint8_t* active;
  int32_t* resc;     // [2][n] flagged rows by merge parity
  int32_t* nres;     // [2]
  GridBest* part;    // [2][2G]
  GridBest* fin;     // [n + G * UG_W]
  int32_t* merges;
  double* heights;
  unsigned* bar;     // [2] arrivals, generation
  double h0;         // height = (h0 - best) / 2: 1 for F (d = 1 - F), 0 for -d (d^F)
};

// barrier over one task's blocks (all resident: cooperative launch)
__device__ __forceinline__ void group_sync(unsigned* bar, int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == (unsigned)G - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      } while (g == gen);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(UG_T) upgma_grid_kernel(const UgTask* __restrict__ tasks, int ntasks,
                                                          unsigned long long* __restrict__ prof) {
  __shared__ double s_v[2][UG_W];
  __shared__ int s_a[2][UG_W], s_b[UG_W];
  int t = 0;
  while (t + 1 < ntasks && (int)blockIdx.x >= tasks[t + 1].g0) ++t;
  const UgTask T = tasks[t];
  double* __restrict__ S = T.S;
  const int64_t ld = T.ld;
  const int n = T.n;
  double* __restrict__ bval = T.bval;
  int32_t* __restrict__ bidx = T.bidx;
  int32_t* __restrict__ size = T.size;
  uint8_t* __restrict__ active = T.active;
  int32_t* __restrict__ resc = T.resc;
  int32_t* __restrict__ nres = T.nres;
  GridBest* __restrict__ part = T.part;
  GridBest* __restrict__ fin = T.fin;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = T.G, bid = (int)blockIdx.x - T.g0;
  if (bid >= G) return;   // spare blocks (none: the host assigns every block)
  const int r0 = (int)((int64_t)bid * n / G), r1 = (int)((int64_t)(bid + 1) * n / G);
  // partials of one merge: [0, G) the rows not rescanned (pairs), [G, 2G) row
  // a's new entries (two sets by merge parity); fin: q per flagged row
  const size_t pset = (size_t)2 * G;
  const int GW = G * UG_W;
  // the first row-bests as merge -1's partials (no flagged rows, no row a)
  {
    double v = -1.0 / 0.0;
    int a = 0x7fffffff, b = 0x7fffffff;
    for (int i = r0 + tid; i < r1; i += UG_T) {
      const int k = bidx[i];
      const int lo = min(i, k), hi = max(i, k);
      if (pair_better(bval[i], lo, hi, v, a, b)) { v = bval[i]; a = lo; b = hi; }
    }
    warp_pair_best(v, a, b);
    if (lane == 0) { s_v[0][warp] = v; s_a[0][warp] = a; s_b[warp] = b; }
    __syncthreads();
    if (warp == 0) {
      v = lane < UG_W ? s_v[0][lane] : -1.0 / 0.0;
      a = lane < UG_W ? s_a[0][lane] : 0x7fffffff;
      b = lane < UG_W ? s_b[lane] : 0x7fffffff;
      warp_pair_best(v, a, b);
      if (lane == 0) part[pset + bid] = GridBest{v, a, b};
    }
  }
  int pa = -1;   // row a of the previous merge
  group_sync(T.bar, G);
  unsigned long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  auto gtime = [] {
    unsigned long long x;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x));
    return x;
  };
  const bool timing = prof && blockIdx.x == 0 && tid == 0;
  for (int m = 0; m + 1 < n; ++m) {
    if (timing) t0 = gtime();
    const GridBest* prev = part + (size_t)((m + 1) & 1) * pset;
    GridBest* cur = part + (size_t)(m & 1) * pset;
    const int32_t* presc = resc + (size_t)((m + 1) & 1) * n;
    int32_t* mresc = resc + (size_t)(m & 1) * n;
    // ---- 1. finish merge m - 1 (rows of list L = [pa, flagged rows...]) and
    // find merge m's pair; warp 0 takes the other rows' partials, warp w >= 1
    // the list rows w - 1, w - 1 + (UG_W - 1), ...
    const int pn = nres[(m + 1) & 1];
    const int pq = ug_chunks(pn, n, GW);
    double v = -1.0 / 0.0;
    int a = 0x7fffffff, b = 0x7fffffff;
    if (warp == 0) {
      for (int i = lane; i < G; i += 32) {
        const GridBest p = prev[i];
        if (pair_better(p.v, p.a, p.b, v, a, b)) { v = p.v; a = p.a; b = p.b; }
      }
    } else if (pa >= 0) {
      for (int r = warp - 1; r <= pn; r += UG_W - 1) {
        const int row = r == 0 ? pa : presc[r - 1];
        double rv = -1.0 / 0.0;
        int rk = 0x7fffffff;
        const GridBest* pr = r == 0 ? prev + G : fin + (size_t)(r - 1) * pq;
        for (int i = lane; i < (r == 0 ? G : pq); i += 32)
          if (row_better(pr[i].v, pr[i].a, rv, rk)) { rv = pr[i].v; rk = pr[i].a; }
        warp_row_best(rv, rk);
        if (lane == 0 && row >= r0 && row < r1) {   // the owner keeps the row's best
          bval[row] = rv;
          bidx[row] = rk;
        }
        const int lo = min(row, rk), hi = max(row, rk);
        if (pair_better(rv, lo, hi, v, a, b)) { v = rv; a = lo; b = hi; }
      }
    }
    warp_pair_best(v, a, b);   // lanes agree after the butterfly
    if (lane == 0) { s_v[0][warp] = v; s_a[0][warp] = a; s_b[warp] = b; }
    __syncthreads();
    v = s_v[0][0];
    a = s_a[0][0];
    b = s_b[0];
    for (int w = 1; w < UG_W; ++w)
      if (pair_better(s_v[0][w], s_a[0][w], s_b[w], v, a, b)) { v = s_v[0][w]; a = s_a[0][w]; b = s_b[w]; }
    if (timing) t1 = gtime();
    if (bid == 0 && tid == 0) {
      T.merges[2 * m] = a;
      T.merges[2 * m + 1] = b;
      T.heights[m] = __dmul_rn(__dadd_rn(T.h0, -v), 0.5);
    }
    // ---- 2. this block's columns c: row / column a, adoption or a rescan
    // flag for row c, and the partials
    const double na = (double)size[a], nb = (double)size[b], nab = (double)(size[a] + size[b]);
    double av = -1.0 / 0.0, pv = -1.0 / 0.0;
    int ak = 0x7fffffff, p1 = 0x7fffffff, p2 = 0x7fffffff;
    for (int c = r0 + tid; c < r1; c += UG_T) {
      if (!active[c] || c == a || c == b) continue;
      const double x =
          __ddiv_rn(__dadd_rn(__dmul_rn(na, S[(int64_t)a * ld + c]), __dmul_rn(nb, S[(int64_t)b * ld + c])), nab);
      S[(int64_t)a * ld + c] = x;
      S[(int64_t)c * ld + a] = x;
      if (row_better(x, c, av, ak)) { av = x; ak = c; }
      int k = bidx[c];
      if (k == a || k == b) {
        mresc[atomicAdd(&nres[m & 1], 1)] = c;
        continue;
      }
      double bv = bval[c];
      if (row_better(x, a, bv, k)) { bv = x; k = a; bval[c] = x; bidx[c] = a; }
      const int lo = min(c, k), hi = max(c, k);
      if (pair_better(bv, lo, hi, pv, p1, p2)) { pv = bv; p1 = lo; p2 = hi; }
    }
    warp_row_best(av, ak);
    warp_pair_best(pv, p1, p2);
    __syncthreads();   // step 1's shared values are read
    if (lane == 0) { s_v[0][warp] = pv; s_a[0][warp] = p1; s_b[warp] = p2; s_v[1][warp] = av; s_a[1][warp] = ak; }
    __syncthreads();
    if (warp == 0) {
      pv = lane < UG_W ? s_v[0][lane] : -1.0 / 0.0;
      p1 = lane < UG_W ? s_a[0][lane] : 0x7fffffff;
      p2 = lane < UG_W ? s_b[lane] : 0x7fffffff;
      av = lane < UG_W ? s_v[1][lane] : -1.0 / 0.0;
      ak = lane < UG_W ? s_a[1][lane] : 0x7fffffff;
      warp_pair_best(pv, p1, p2);
      warp_row_best(av, ak);
      if (lane == 0) {
        cur[bid] = GridBest{pv, p1, p2};
        cur[G + bid] = GridBest{av, ak, 0};
      }
    }
    if (timing) t2 = gtime();
    group_sync(T.bar, G);
    if (timing) t3 = gtime();
    // ---- 3. the flagged rows' partial bests, q column chunks each
    if (bid == 0 && tid == 0) {   // read only after the next barrier
      size[a] += size[b];
      active[b] = 0;
      nres[(m + 1) & 1] = 0;      // merge m + 1's list (merge m - 1's was read in step 1)
    }
    {
      const int nf = nres[m & 1], q = ug_chunks(nf, n, GW);
      for (int u = bid * UG_W + warp; u < nf * q; u += GW) {
        const int r = u / q, ch = u - r * q;
        const int row = mresc[r];
        // even chunk bounds, 16-byte loads (ld is even)
        const int c0 = (int)(((int64_t)ch * n / q) & ~1ll), c1 = ch + 1 == q ? n : (int)(((int64_t)(ch + 1) * n / q) & ~1ll);
        const double* rp = S + (int64_t)row * ld;
        double rv = -1.0 / 0.0;
        int rk = 0x7fffffff;
#pragma unroll 4
        for (int c = c0 + 2 * lane; c < c1; c += 64) {
          const double2 x = *reinterpret_cast<const double2*>(rp + c);
          if (c != row && c != b && active[c] && row_better(x.x, c, rv, rk)) { rv = x.x; rk = c; }
          if (c + 1 < c1 && c + 1 != row && c + 1 != b && active[c + 1] && row_better(x.y, c + 1, rv, rk)) {
            rv = x.y;
            rk = c + 1;
          }
        }
        warp_row_best(rv, rk);
        if (lane == 0) fin[u] = GridBest{rv, rk, 0};
      }
    }
    pa = a;
    if (timing) {
      const unsigned long long t4 = gtime();
      prof[0] += t1 - t0;   // step 1
      prof[1] += t2 - t1;   // step 2
      prof[2] += t3 - t2;   // barrier after step 2 (incl. waiting for the slowest block)
      prof[3] += t4 - t3;   // step 3
      prof[5] += nres[m & 1];
      if (nres[m & 1] > (int)prof[6]) prof[6] = nres[m & 1];
    }
    group_sync(T.bar, G);
    if (timing) prof[4] += gtime() - t3;   // step 3 + the last barrier
  }
}

static bool upgma_grid_enabled(int32_t n) {
  const char* e = getenv("SA_UPGMA_GRID");   // 1: always, 0: never, default: n >= 1024
  if (e) return atoi(e) != 0;
  return n >= 1024;
}

template <class T>
static sa_status salloc(Scratch& scratch, T*& p, size_t n) {
  p = scratch.alloc<T>(n);
  if (!p) return fail(SA_E_NOMEM, "scratch allocation of %zu elements failed", n);
  return SA_OK;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Working copies and the first row-bests of one task.
static sa_status upgma_prepare(Scratch& scratch, const double* F, int32_t n, int64_t ld, const TreeForm& tf,
                               double*& S, int64_t& lds, double*& bval, int32_t*& bidx, cudaStream_t st) {
  lds = (n + 1) & ~1;   // even: 16-byte row starts for the grid loop's scans
  SA_TRY(salloc(scratch, S, (size_t)n * lds));
  SA_TRY(salloc(scratch, bval, (size_t)n));
  SA_TRY(salloc(scratch, bidx, (size_t)n));
  if (tf.form == SA_TREE_DF) {
    SA_TRY(ensure_ln_table());
    const int64_t total = (int64_t)n * n;
    dF_matrix_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)device_sms() * 8), 256, 0, st>>>(
        F, ld, n, tf.delta, S, lds, tf.unc);
    SA_LAUNCHED();
  } else {
    SA_CUDA(cudaMemcpy2DAsync(S, (size_t)lds * sizeof(double), F, (size_t)ld * sizeof(double),
                              (size_t)n * sizeof(double), (size_t)n, cudaMemcpyDeviceToDevice, st));
  }
  const int64_t warps = n;
  upgma_init_kernel<<<(unsigned)std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16), 256, 0, st>>>(S, n, lds, bval,
                                                                                                  bidx);
  SA_LAUNCHED();
  return SA_OK;
}

// Every task's tree in cooperative launches of `blocks` resident blocks, the
// blocks of one launch shared out in proportion to n^2 (the merges' work),
// at least one per task.
static sa_status upgma_grid_batch(int count, const double* const* F, const int32_t* n, const int64_t* ld,
                                  int32_t* const* merges, double* const* heights, const TreeForm& tf,
                                  cudaStream_t st) {
  int per_sm = 0;
  SA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, upgma_grid_kernel, UG_T, 0));
  const int bps = std::max(1, std::min(per_sm, env_int("SA_UPGMA_BPS", 1)));
  const int blocks = bps * device_sms();
  std::vector<int> idx;
  for (int i = 0; i < count; ++i)
    if (n[i] > 1) idx.push_back(i);
  const bool want_prof = env_int("SA_UPGMA_PROF", 0) != 0;   // block 0's phase times to stderr
  for (size_t w0 = 0; w0 < idx.size(); w0 += (size_t)blocks) {
    const size_t w1 = std::min(idx.size(), w0 + (size_t)blocks);
    const int nt = (int)(w1 - w0);
    Scratch scratch(st);
    // blocks per task: one each, the rest by largest remainder of n^2
    std::vector<int> g(nt, 1);
    double W = 0;
    for (int k = 0; k < nt; ++k) W += (double)n[idx[w0 + k]] * n[idx[w0 + k]];
    const int spare = blocks - nt;
    std::vector<std::pair<double, int>> rem;
    int given = 0;
    for (int k = 0; k < nt; ++k) {
      const double share = spare * ((double)n[idx[w0 + k]] * n[idx[w0 + k]] / W);
      const int whole = (int)share;
      g[k] += whole;
      given += whole;
      rem.push_back({share - whole, k});
    }
    std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first || (x.first == y.first && x.second < y.second); });
    for (int k = 0; given < spare && k < nt; ++k, ++given) ++g[rem[k].second];
    std::vector<UgTask> tasks(nt);
    int g0 = 0;
    for (int k = 0; k < nt; ++k) {
      const int i = idx[w0 + k];
      UgTask& T = tasks[k];
      T.n = n[i];
      T.G = std::min(g[k], std::max(1, (n[i] + 31) / 32));   // at least 32 rows per block
      T.g0 = g0;
      g0 += g[k];
      SA_TRY(upgma_prepare(scratch, F[i], n[i], ld[i], tf, T.S, T.ld, T.bval, T.bidx, st));
      T.h0 = tf.form == SA_TREE_DF ? 0.0 : 1.0;
      SA_TRY(salloc(scratch, T.size, (size_t)n[i]));
      SA_TRY(salloc(scratch, T.active, (size_t)n[i]));
      SA_TRY(salloc(scratch, T.resc, (size_t)2 * n[i]));
      SA_TRY(salloc(scratch, T.nres, 2));
      SA_TRY(salloc(scratch, T.part, (size_t)4 * T.G));
      SA_TRY(salloc(scratch, T.fin, (size_t)n[i] + (size_t)T.G * UG_W));
      SA_TRY(salloc(scratch, T.bar, 2));
      SA_CUDA(cudaMemsetAsync(T.active, 1, n[i], st));
      SA_CUDA(cudaMemsetAsync(T.nres, 0, 2 * sizeof(int32_t), st));
      SA_CUDA(cudaMemsetAsync(T.bar, 0, 2 * sizeof(unsigned), st));
      SA_TRY(fill_ones_i32(T.size, n[i], st));
      T.merges = merges[i];
      T.heights = heights[i];
    }
    UgTask* dtasks = nullptr;
    SA_TRY(salloc(scratch, dtasks, (size_t)nt));
    SA_CUDA(cudaMemcpyAsync(dtasks, tasks.data(), sizeof(UgTask) * nt, cudaMemcpyHostToDevice, st));
    unsigned long long* prof = nullptr;
    if (want_prof) {
      SA_TRY(salloc(scratch, prof, 8));
      SA_CUDA(cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), st));
    }
    int ntasks = nt;
    void* args[] = {&dtasks, &ntasks, &prof};
    SA_CUDA(cudaLaunchCooperativeKernel((const void*)upgma_grid_kernel, dim3(g0), dim3(UG_T), args, 0, st));
    SA_LAUNCHED();
    if (prof) {
      unsigned long long h[8];
      SA_CUDA(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr,
              "upgma_grid tasks=%d blocks=%d task0 n=%d G=%d: step1 %.0f ms, step2 %.0f ms, barrier2 %.0f ms, step3 %.0f "
              "ms, step3+barrier3 %.0f ms; flagged rows %llu (max %llu)\n",
              nt, g0, tasks[0].n, tasks[0].G, h[0] * 1e-6, h[1] * 1e-6, h[2] * 1e-6, h[3] * 1e-6, h[4] * 1e-6, h[5], h[6]);
    }
    // the host task table must outlive the copy
    SA_CUDA(cudaStreamSynchronize(st));
  }
  return SA_OK;
}

sa_status upgma_launch(const double* F, int32_t n, int64_t ld, int32_t* merges, double* heights, const TreeForm& tf,
                       cudaStream_t st) {
  if (tf.unc) SA_CUDA(cudaMemsetAsync(tf.unc, 0, sizeof(unsigned long long), st));
  if (n <= 1) return SA_OK;
  if (upgma_grid_enabled(n)) return upgma_grid_batch(1, &F, &n, &ld, &merges, &heights, tf, st);
  Scratch scratch(st);
  double *S, *bval;
  int32_t* bidx;
  int64_t lds;
  SA_TRY(upgma_prepare(scratch, F, n, ld, tf, S, lds, bval, bidx, st));
  SA_ALLOC(size, int32_t, n);
  SA_ALLOC(active, uint8_t, n);
  SA_ALLOC(resc, int32_t, n);
  upgma_merge_kernel<<<1, UT, 0, st>>>(S, n, lds, bval, bidx, size, active, resc, merges, heights,
                                       tf.form == SA_TREE_DF ? 0.0 : 1.0);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status upgma_launch_batch(int count, const double* const* F, const int32_t* n, const int64_t* ld,
                             int32_t* const* merges, double* const* heights, const TreeForm& tf, cudaStream_t st) {
  if (tf.unc) SA_CUDA(cudaMemsetAsync(tf.unc, 0, sizeof(unsigned long long), st));
  return upgma_grid_batch(count, F, n, ld, merges, heights, tf, st);
}

}  // namespace sa
