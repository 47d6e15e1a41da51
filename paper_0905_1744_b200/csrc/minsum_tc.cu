// K2T -- the min-sum engine on the tensor cores (SURVEY.md
// §8(f) N3(iii)).  The exact-rank key terms, reciprocal tables and 128-bit
// atomics are the ones K2 uses (keyterm.cuh).
//
// Eq. 1's numerator as an exact 0/1 contraction:
//     C_ij = sum_t min(c^i_t, c^j_t) = sum_t sum_{r>=1} [c^i_t >= r][c^j_t >= r]
// over the threshold layers r of every bin t.  A column (r, t) contributes to
// a pair only if both rows reach layer r in bin t, so each problem keeps only
// the columns that can contribute:
//   symmetric problem (A = B): columns reached by >= 2 rows (the diagonal
//     C_ii = nk_i is set in the epilogue);
//   rectangular problem: columns reached by >= 1 row of A and >= 1 row of B.
// On the BASELINE workloads layer 1 and most of layer 2 survive and almost
// nothing above (config 4 block: 8000 + 7999 + 209 + 1 columns), so
// K' ~ 16 k instead of the 8000 x max-count of the full unary expansion.
//
// Device-side pipeline per launch (no host synchronisation):
//   tc_hist_kernel   seen-once / seen-twice bit planes per (layer, bin) and
//                    side, built in shared memory (atomicOr) and merged into
//                    global planes; folds the largest count into state[0];
//   tc_select_kernel the column list of every problem, K' rounded up to 128,
//                    kblocks = K'/128; flags the launch infeasible (state[1])
//                    when a count exceeds TC_LCAP or K' exceeds TC_KCAP;
//   tc_build_kernel  A'[row][c] = [c_row(bin_c) >= layer_c] as uint8 rows of
//                    TC_KCAP bytes;
//   tc::gemm_kernel  the tcgen05 kind::i8 GEMM (tc_gemm.cuh) with KeyMatEpi:
//                    exact-rank keys (row sums, plus column sums for the
//                    mirrored pairs of symmetric problems) and / or the
//                    uint16 C / fp64 F matrices (mirrored for symmetric).
// When a launch is infeasible every K2T kernel returns at once and the
// guarded SAD / u16 engines (minsum.cu) run instead: exact in every case.
#include <atomic>
#include <cstring>

#include "common.cuh"
#include "keyterm.cuh"
#include "tc_gemm.cuh"
#include "tc_sparse.cuh"

namespace sa {

constexpr int TC_LCAP = 32;                    // threshold layers tracked
constexpr int TC_WPL = 256;                    // plane words per layer (bins <= 8192)
constexpr int TC_PLANE = TC_LCAP * TC_WPL;     // words per plane (32 KB)
constexpr int TC_KCAP = 32768;                 // columns (bytes) per operand row

// state words (ctx->dcount): [0] largest count, [1] K2T infeasible, [2] K2T enabled for this call
__device__ __forceinline__ bool tc_infeasible(const uint32_t* state) {
  return reinterpret_cast<const volatile uint32_t*>(state)[1] != 0u;
}

// Rows of all sides of a launch, flattened: side s = rows [row_begin[s], row_begin[s+1]).
struct TcSides {
  const uint16_t* rows[2 * tc::MAXPROB];
  int64_t row_begin[2 * tc::MAXPROB + 1];
  int n;
};

// ---------------------------------------------------------- histogram ----
// Thread w of a CTA owns plane word w (bins 32 w .. 32 w + 31) of every layer:
// for each of its rows it loads those 32 counts (64 bytes) and updates, per
// layer l reached, seen1 |= m, seen2 |= seen1_old & m with m = [count >= l]
// -- registers for the first TC_HREG layers, its own shared-memory words for
// deeper ones; no atomics until the flush into the global planes.
constexpr int TC_HREG = 8;
constexpr int TC_HIST_THREADS = TC_WPL;   // 256
constexpr int TC_HIST_ROWS = 4;

__device__ __forceinline__ uint32_t layer_mask(const uint32_t (&v)[16], uint32_t L2) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t c = __vsetgeu2(v[i], L2);   // 1 per half with count >= layer
    m |= ((c | (c >> 15)) & 3u) << (2 * i);
  }
  return m;
}

// Row outputs of the operand build (declared here: the histogram pass also
// writes the first dense layers, below).
struct TcOut {
  uint8_t* out[2 * tc::MAXPROB];
  int prob[2 * tc::MAXPROB];
};

// Per row, the histogram pass also stores its layer-2 and layer-3 masks
// ([c >= 2], [c >= 3]: 2 x 256 words, 2 KB, coalesced); the build then reads
// the listed layer-2 / layer-3 columns from them instead of gathering counts
// from the 16 KB profile row (one 32-byte DRAM sector per gathered count).
// After them, 8 summary words: bit j of word w is set when one of bins
// [1024 w + 32 j, + 32) reaches count 4, so the build skips the profile read
// of a listed layer >= 4 column whose 32-bin word has no count >= 4 (most).
// Rows [0, split) of a launch with a carried side use the carry's masks.
constexpr int TC_MW = TC_WPL;   // mask words per layer
constexpr int TC_MDEEP = 2 * TC_MW;        // offset of the count >= 4 summary words
constexpr int TC_MROW = 2 * TC_MW + 8;     // words per row
struct TcMasks {
  uint32_t* own;                // rows [split, R): row g at own + (g - split) * TC_MROW
  const uint32_t* carried;      // rows [0, split)
  int64_t split;
  int own_valid, carried_valid; // 0: not written (sparse launches skip them): the build reads the profile row
  __device__ __forceinline__ bool valid(int64_t g) const { return g < split ? carried_valid != 0 : own_valid != 0; }
  __device__ __forceinline__ const uint32_t* row(int64_t g) const {
    return g < split ? carried + g * TC_MROW : own + (g - split) * TC_MROW;
  }
};

// 32 layer-mask bits (bin i of the thread's word -> bit i) as operand columns:
// FP4: 16 bytes, column i = nibble i (e2m1 1.0 = 0b0010); u8: 32 bytes of 0/1.
template <bool FP4>
__device__ __forceinline__ void store_mask_columns(uint8_t* dst, uint32_t m, int ncols) {
  if constexpr (FP4) {
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t x = (m >> (8 * k)) & 0xffu;                // 8 bits -> 8 nibbles
      x = (x | (x << 12)) & 0x000F000Fu;
      x = (x | (x << 6)) & 0x03030303u;
      x = (x | (x << 3)) & 0x11111111u;
      o[k] = x << 1;
    }
    // 8-byte stores: a dense layer of dw (a multiple of 16) columns is a multiple of 8 bytes
    *reinterpret_cast<uint2*>(dst) = make_uint2(o[0], o[1]);
    if (ncols >= 32) *reinterpret_cast<uint2*>(dst + 8) = make_uint2(o[2], o[3]);
  } else {
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = (((m >> (4 * k)) & 0xfu) * 0x00204081u) & 0x01010101u;   // 4 bits -> 4 bytes
    *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
    if (ncols >= 32) *reinterpret_cast<uint4*>(dst + 16) = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

// The first `spec` dense layers (a launch parameter: 1 when the launch expects
// its problems to take the sparse path for layers >= 2, tc_sparse.cu, else 2)
// are written by the histogram pass itself (every bin of the layer, in bin
// order: the layout the column selection gives a dense layer), so the profile
// rows are read once for both: the selection later keeps nd dense layers;
// tc_dense_kernel adds layers spec + 1 .. nd when nd > spec, and
// tc_build_kernel overwrites the columns from nd * dw on when nd < spec.
constexpr int TC_SPEC_MAX = 2;

// Records for the sparse layers (tc_sparse.cu): every (row, bin) whose count
// reaches 2, as {row, bin | count << 16}, into this CTA's segment of
// `rec_seg` (seg_cap records; the count goes to seg_cnt[blockIdx.x], and a
// segment that overflows makes the whole launch dense).
struct TcRecOut {
  uint2* seg;
  uint32_t* cnt;
  uint32_t* povf;   // [MAXPROB]: the problem of a row whose record did not fit runs dense
  uint32_t* incomplete;
  uint32_t seg_cap;
  int on;
};

// DEEP = false: the sparse-path launch's lean instantiation (layer 1 and the
// records only; deep_planes must be 0): none of the deeper layers' code or
// shared memory, so the instruction stream fits the cache (the general kernel
// stalled 35% on instruction fetch on config 4, ncu) and more CTAs fit an SM.
#ifndef SA_HIST_LEAN_ROWS
#define SA_HIST_LEAN_ROWS 4
#endif
#ifndef SA_HIST_LEAN_MINB
#define SA_HIST_LEAN_MINB 2
#endif
#ifndef SA_HIST_LEAN_GRID
#define SA_HIST_LEAN_GRID 4   // CTAs per SM in the grid
#endif
template <bool DEEP>
__host__ __device__ constexpr int hist_rows() { return DEEP ? TC_HIST_ROWS : SA_HIST_LEAN_ROWS; }
template <bool FP4, bool DEEP>
__global__ void __launch_bounds__(TC_HIST_THREADS, DEEP ? 2 : SA_HIST_LEAN_MINB)   // two CTAs per SM (<= 128 registers)
tc_hist_kernel(const __grid_constant__ TcSides S, const __grid_constant__ TcOut O, int stride16, int bins,
               uint32_t* __restrict__ planes, uint32_t* __restrict__ state, int64_t hist_from, TcMasks mk, int spec,
               TcRecOut ro, int deep_planes, const int32_t* __restrict__ only_dense) {
  constexpr int TC_HIST_ROWS = hist_rows<DEEP>();
  if constexpr (!DEEP) deep_planes = 0;
  if (only_dense) {   // the planes pass after the plan: nothing to do when every problem runs sparse
    bool any_dense = false;
    for (int t = 0; t < S.n; ++t) any_dense = any_dense || only_dense[O.prob[t]] == 0;
    if (!any_dense) return;
  }
  __shared__ uint32_t s_nrec;
  if (threadIdx.x == 0) s_nrec = 0;
  __syncthreads();
  static_assert(tc::MAXPROB <= 32, "ovf_probs is a 32-bit problem mask");
  constexpr int64_t ROWB = FP4 ? TC_KCAP / 2 : TC_KCAP;
  const int dw = (bins + 15) & ~15;                      // columns per dense layer
  const int64_t layer_bytes = FP4 ? dw / 2 : dw;
  extern __shared__ uint32_t deep[];   // [2][TC_LCAP - TC_HREG][TC_WPL], word w owned by thread w
  constexpr int ND = TC_LCAP - TC_HREG;
  const int w = threadIdx.x;
  const bool active = w * 32 < stride16;
  if constexpr (DEEP)
    for (int l = 0; l < 2 * ND; ++l) deep[l * TC_WPL + w] = 0u;
  // rows [hist_from, R): a carried side (TcCarry) comes first and is skipped
  const int64_t R = S.row_begin[S.n] - hist_from;
  const int64_t r0 = hist_from + blockIdx.x * R / gridDim.x, r1 = hist_from + (blockIdx.x + 1) * R / gridDim.x;
  uint32_t s1[TC_HREG], s2[TC_HREG];
#pragma unroll
  for (int l = 0; l < TC_HREG; ++l) s1[l] = s2[l] = 0u;
  uint32_t mx = 0;
  uint32_t ovf_probs = 0;   // bit q: a record of problem q did not fit this CTA's segment
  bool seg_full = false;
  int side = -1, deepest = 0;
  auto flush = [&](int sd) {
    uint32_t* g1 = planes + (int64_t)sd * 2 * TC_PLANE;
    uint32_t* g2 = g1 + TC_PLANE;
#pragma unroll
    for (int l = 0; l < TC_HREG; ++l) {
      uint32_t t2 = s2[l];
      if (s1[l]) t2 |= atomicOr(&g1[l * TC_WPL + w], s1[l]) & s1[l];   // seen by another CTA too
      if (t2) atomicOr(&g2[l * TC_WPL + w], t2);
      s1[l] = s2[l] = 0u;
    }
    for (int l = 0; l < (DEEP ? deepest : 0); ++l) {
      const uint32_t d1 = deep[l * TC_WPL + w];
      uint32_t d2 = deep[(ND + l) * TC_WPL + w];
      if (d1) d2 |= atomicOr(&g1[(TC_HREG + l) * TC_WPL + w], d1) & d1;
      if (d2) atomicOr(&g2[(TC_HREG + l) * TC_WPL + w], d2);
      deep[l * TC_WPL + w] = deep[(ND + l) * TC_WPL + w] = 0u;
    }
    deepest = 0;
  };
  int64_t g = r0;
  while (g < r1) {
    int t = side < 0 ? 0 : side;
    while (g >= S.row_begin[t + 1]) ++t;
    if (t != side) {
      if (side >= 0 && active) flush(side);
      side = t;
    }
    const int cnt = (int)min((int64_t)TC_HIST_ROWS, min(r1, S.row_begin[t + 1]) - g);
    if (only_dense && only_dense[O.prob[t]]) {   // planes pass: rows of sparse problems need no deep planes
      g += cnt;
      continue;
    }
    bool deep4[TC_HIST_ROWS];
#pragma unroll
    for (int h = 0; h < TC_HIST_ROWS; ++h) deep4[h] = false;
    if (active) {
      uint4 raw[TC_HIST_ROWS][4];
      const uint16_t* base = S.rows[t] + (g - S.row_begin[t]) * (int64_t)stride16 + w * 32;
#pragma unroll
      for (int h = 0; h < TC_HIST_ROWS; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          raw[h][k] = h < cnt ? reinterpret_cast<const uint4*>(base + h * (int64_t)stride16)[k] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int h = 0; h < TC_HIST_ROWS; ++h) {
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[4 * k] = raw[h][k].x;
          v[4 * k + 1] = raw[h][k].y;
          v[4 * k + 2] = raw[h][k].z;
          v[4 * k + 3] = raw[h][k].w;
        }
        uint32_t vm = v[0];
#pragma unroll
        for (int i = 1; i < 16; ++i) vm = __vmaxu2(vm, v[i]);
        const uint32_t vmax = max(vm & 0xffffu, vm >> 16);
        mx = max(mx, vmax);
        deep4[h] = vmax >= 4u;
        const bool in_cols = w * 32 < dw;
        uint8_t* orow = O.out[t] + (g - S.row_begin[t] + h) * ROWB + (FP4 ? w * 16 : w * 32);
        uint32_t m23[2] = {0u, 0u};   // [c >= 2], [c >= 3] of the thread's 32 bins
        if (deep_planes) {
          // every layer's seen-once / seen-twice planes (the dense path's column
          // selection); a planes-only pass (only_dense) skips layer 1 and writes nothing
#pragma unroll
          for (int l = 0; l < TC_HREG; ++l) {
            const uint32_t m = (uint32_t)l < vmax ? layer_mask(v, (uint32_t)(l + 1) * 0x00010001u) : 0u;
            if (l < spec && h < cnt && in_cols && !only_dense)
              store_mask_columns<FP4>(orow + l * layer_bytes, m, dw - w * 32);
            if (l == 1 || l == 2) m23[l - 1] = m;
            if ((uint32_t)l >= vmax && l >= 3) break;   // layers 1-3: the masks above
            if (l == 0 && only_dense) continue;
            s2[l] |= s1[l] & m;
            s1[l] |= m;
          }
        } else {
          // sparse-path launch: layer 1 only (operand columns and its planes);
          // [c >= 2] just for the records, and only where a count reaches 2
          const uint32_t m = layer_mask(v, 0x00010001u);
          if (h < cnt && in_cols) store_mask_columns<FP4>(orow, m, dw - w * 32);
          s2[0] |= s1[0] & m;
          s1[0] |= m;
          if (vmax >= 2u) m23[0] = layer_mask(v, 0x00020002u);
        }
        if (h < cnt) {
          uint32_t* mr = mk.own + (g + h - hist_from) * TC_MROW;
          if (mk.own_valid) {
            mr[w] = m23[0];
            mr[TC_MW + w] = m23[1];
          }
          if (ro.on) {
            // records of the bins reaching 2 (sparse per row: ~8 of 8000 on
            // the protein workloads); the count is re-read from the row (L1)
            // A full segment stays full: from then on a row with records only
            // marks its problem, in a per-thread mask that reaches povf once,
            // at the end of the kernel (long sequences, config 5: ~500 records
            // per row against a budget of 48 -- one global atomic per lost
            // record on the same two words took 1.1 ms of a 1.15 ms pass).
            uint32_t m = m23[0];
            if (m) {
              if (!seg_full && *reinterpret_cast<volatile uint32_t*>(&s_nrec) >= ro.seg_cap) seg_full = true;
              if (seg_full) ovf_probs |= 1u << O.prob[t];
              else
                while (m) {
                  const int bit = __ffs(m) - 1;
                  m &= m - 1;
                  const uint32_t pos = atomicAdd(&s_nrec, 1u);
                  if (pos >= ro.seg_cap) {
                    ovf_probs |= 1u << O.prob[t];
                    seg_full = true;
                    break;
                  }
                  const uint32_t c = __ldg(base + h * (int64_t)stride16 + bit);
                  ro.seg[(int64_t)blockIdx.x * ro.seg_cap + pos] =
                      make_uint2((uint32_t)(g + h), (uint32_t)(w * 32 + bit) | (c << 16));
                }
            }
          }
        }
        const int top = DEEP && deep_planes ? (int)min(vmax, (uint32_t)TC_LCAP) : 0;
        for (int l = TC_HREG; l < top; ++l) {
          const uint32_t m = layer_mask(v, (uint32_t)(l + 1) * 0x00010001u);
          uint32_t* d1 = &deep[(l - TC_HREG) * TC_WPL + w];
          deep[(ND + l - TC_HREG) * TC_WPL + w] |= *d1 & m;
          *d1 |= m;
          deepest = max(deepest, l - TC_HREG + 1);
        }
      }
    }
    // the row's count >= 4 summary: one word per warp (all lanes take part)
#pragma unroll
    for (int h = 0; h < TC_HIST_ROWS; ++h) {
      const uint32_t b4 = __ballot_sync(0xffffffffu, deep4[h]);
      if ((w & 31) == 0 && h < cnt && mk.own_valid) mk.own[(g + h - hist_from) * TC_MROW + TC_MDEEP + (w >> 5)] = b4;
    }
    g += cnt;
  }
  if (side >= 0 && active) flush(side);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((w & 31) == 0 && mx) atomicMax(&state[0], mx);
  if (ro.on) {
    ovf_probs = __reduce_or_sync(0xffffffffu, ovf_probs);
    if ((w & 31) == 0 && ovf_probs) {
      for (uint32_t q = ovf_probs; q; q &= q - 1) atomicOr(&ro.povf[__ffs(q) - 1], 1u);
      atomicOr(ro.incomplete, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) ro.cnt[blockIdx.x] = s_nrec;
  }
}

// The hist CTAs' record segments -> one dense array after the carried
// launch's records (`carried`: [0] count, [2] incomplete flag), total[0] = the
// count.  A segment over its cap (a CTA whose rows repeat more bins than the
// budget) keeps its first seg_cap records; the hist pass marked the problems
// of the rows whose records did not fit (povf: they run dense).
struct TcRecOvf {
  int carried_prob;   // problem of the carried side 0
  uint32_t* povf;     // [MAXPROB], zeroed by the caller
};
__global__ void tc_rec_compact_kernel(const uint2* __restrict__ seg, const uint32_t* __restrict__ cnt, int nseg,
                                      uint32_t seg_cap, uint2* __restrict__ out, uint32_t out_cap,
                                      uint32_t* __restrict__ total, const uint32_t* __restrict__ carried,
                                      const TcRecOvf ov) {
  __shared__ uint32_t s_base;
  const int b = blockIdx.x;
  if (threadIdx.x < 32) {
    uint32_t sum = 0;
    for (int i = threadIdx.x; i < b; i += 32) sum += min(cnt[i], seg_cap);
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (threadIdx.x == 0) s_base = sum + (carried ? carried[0] : 0u);
  }
  __syncthreads();
  const uint32_t c = cnt[b], n = min(c, seg_cap);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t pos = s_base + i;
    if (pos < out_cap) out[pos] = seg[(int64_t)b * seg_cap + i];
  }
  if (threadIdx.x == 0) {
    (void)c;
    if (b == 0 && carried && carried[2]) {   // the carried side's records are incomplete
      atomicOr(&ov.povf[ov.carried_prob], 1u);
      atomicOr(&total[2], 1u);
    }
    if (b == nseg - 1) total[0] = min(s_base + n, out_cap);
  }
}

// OR of the seen-once planes of sides [0, nsides) (the carried query side of a
// later rectangular launch: a column can contribute if any of its rows reaches it)
__global__ void tc_or_planes_kernel(const uint32_t* __restrict__ planes, int nsides, uint32_t* __restrict__ out,
                                    const uint32_t* __restrict__ state) {
  if (tc_infeasible(state)) return;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < TC_PLANE; w += gridDim.x * blockDim.x) {
    uint32_t m = 0;
    for (int sd = 0; sd < nsides; ++sd) m |= planes[(int64_t)sd * 2 * TC_PLANE + w];
    out[w] = m;
  }
}

// Per-row epilogue info (TcEpiProb kinfo / yinfo) of every row of every side.
struct TcNk {
  const int32_t* nk[2 * tc::MAXPROB];
};
__global__ void tc_info_kernel(const __grid_constant__ TcSides S, const __grid_constant__ TcNk N,
                               uint4* __restrict__ kinfo, double2* __restrict__ yinfo, const uint32_t* __restrict__ state) {
  if (tc_infeasible(state)) return;
  const int64_t R = S.row_begin[S.n];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < R; g += (int64_t)gridDim.x * blockDim.x) {
    int t = 0;
    while (g >= S.row_begin[t + 1]) ++t;
    const int nk = N.nk[t][g - S.row_begin[t]];
    const int ns = nk > 0 ? nk : -1;
    const int d = ns > 0 ? ns : 0;
    const uint64_t r = g_rtab[d];
    kinfo[g] = make_uint4((uint32_t)r, (uint32_t)(r >> 32), g_etab[d], (uint32_t)ns);
    yinfo[g] = make_double2(g_rcp[d], (double)d);
  }
}

// ------------------------------------------------------ column select ----
struct TcSel {
  int side_a[tc::MAXPROB], side_b[tc::MAXPROB];   // side_b = -1: symmetric
  int n;
  int first;                                        // index of problem 0 in the whole call
};

// One CTA (1024 threads = 32 warps) per problem; warp w owns layer w + 1
// (256 plane words, 8 per thread).  Kept columns per layer never increase
// with the layer (a pair reaching layer l + 1 in a bin also reaches l), so the
// layers holding at least half of the bins form a prefix: those are stored
// "dense" -- every bin, in bin order, dw = round_up(bins, 16) columns per
// layer (a column no pair shares only adds zeros off the diagonal, which the
// epilogue overrides) -- and the build kernel encodes them with vector loads.
// The remaining layers list their kept (layer, bin) columns.
__global__ void __launch_bounds__(1024)
tc_select_kernel(const __grid_constant__ TcSel sel, const uint32_t* __restrict__ planes, int bins, int kbc,
                 uint32_t* __restrict__ collist, int32_t* __restrict__ kblocks, int32_t* __restrict__ ndense,
                 uint32_t* __restrict__ state, uint32_t* __restrict__ cols_out, const int32_t* __restrict__ spmode) {
  __shared__ uint32_t warp_cnt[32];
  __shared__ uint32_t warp_pos[32];
  __shared__ uint32_t s_total, s_nd;
  const int q = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int PER = TC_PLANE / 1024;   // 8 words per thread
  static_assert(TC_WPL == 32 * PER, "one warp per layer");
  const uint32_t* a = planes + (int64_t)sel.side_a[q] * 2 * TC_PLANE;
  const uint32_t* b = sel.side_b[q] >= 0 ? planes + (int64_t)sel.side_b[q] * 2 * TC_PLANE : nullptr;
  const int dw = (bins + 15) & ~15;
  uint32_t m[PER];
  uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int w = tid * PER + i;
    m[i] = b ? (a[w] & b[w]) : a[TC_PLANE + w];
    cnt += __popc(m[i]);
  }
  uint32_t x = cnt;   // inclusive scan inside the warp (= layer)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_cnt[wid] = x;
  __syncthreads();
  // sparse problems (tc_sparse.cu): layer 1 only, every bin (layers >= 2 are
  // the epilogue's correction entries)
  const bool sparse = spmode && spmode[q] != 0;
  if (tid == 0) {
    uint32_t nd = 0;
    while (nd < 32 && 2 * warp_cnt[nd] >= (uint32_t)bins && warp_cnt[nd] > 0) ++nd;
    if (sparse) nd = 1;
    uint32_t pos = nd * (uint32_t)dw;
    for (int w = 0; w < 32; ++w) {
      warp_pos[w] = w < (int)nd ? (uint32_t)w * dw : pos;
      if (w >= (int)nd && !sparse) pos += warp_cnt[w];
    }
    s_total = pos;
    s_nd = nd;
  }
  __syncthreads();
  const uint32_t total = s_total, nd = s_nd;
  if (tid == 0 && cols_out && sel.first + q < SA_TC_COLS_MAX) cols_out[sel.first + q] = total;
  const uint32_t kpad = max((uint32_t)kbc, (total + kbc - 1u) / kbc * kbc);   // kbc columns per K block
  const bool too_many = kpad > (uint32_t)TC_KCAP;
  const bool deep = !sparse && reinterpret_cast<const volatile uint32_t*>(state)[0] > (uint32_t)TC_LCAP;
  if (too_many || deep) {
    if (tid == 0) {
      atomicOr(&state[1], 1u);
      kblocks[q] = 1;
      ndense[q] = 0;
    }
    return;
  }
  uint32_t* out = collist + (int64_t)q * TC_KCAP;
  const uint32_t layer = (uint32_t)wid + 1u;
  if ((uint32_t)wid < nd) {
    for (int t = lane; t < dw; t += 32) out[wid * dw + t] = t < bins ? ((uint32_t)t | (layer << 16)) : 0u;
  } else if (!sparse) {
    uint32_t pos = warp_pos[wid] + x - cnt;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint32_t bin0 = (uint32_t)(lane * PER + i) * 32u;
      uint32_t mm = m[i];
      while (mm) {
        const int bpos = __ffs(mm) - 1;
        mm &= mm - 1;
        out[pos++] = (bin0 + (uint32_t)bpos) | (layer << 16);
      }
    }
  }
  for (uint32_t p = total + tid; p < kpad; p += blockDim.x) out[p] = 0u;   // layer 0: padding column
  if (tid == 0) {
    kblocks[q] = (int32_t)(kpad / (uint32_t)kbc);
    ndense[q] = (int32_t)nd;
  }
}

// ------------------------------------------------------- operand rows ----
// Row r of side s -> out[s] + r * TC_KCAP: the side's problem's columns.
// Dense layers (prefix): thread c of a row reads bins 16 c .. 16 c + 15 once
// (two 16-byte loads) and writes one 16-byte chunk per dense layer; listed
// (sparse) columns: 16 entries per chunk, the counts gathered from the row
// (L1 / L2).
__device__ __forceinline__ int TcOutProbs(const TcOut& O, int nsides) {
  int n = 0;
  for (int sd = 0; sd < nsides; ++sd) n = max(n, O.prob[sd] + 1);
  return n;
}

// Dense layers: one thread per (row, 16-bin chunk) of every side, all dense
// layers of that chunk from one 32-byte load.  Counts are <= TC_LCAP here (the
// launch is feasible), so for each u16 half h: h >= L <=> bit 15 of
// h + 0x8000 - L (no carry between the halves).
// FP4: two columns per byte, 1.0 = e2m1 0b0010 in the low (even column) or
// high (odd column) nibble; rows of TC_KCAP / 2 bytes.
template <bool FP4>
__global__ void __launch_bounds__(256)
tc_dense_kernel(const __grid_constant__ TcSides S, const __grid_constant__ TcOut O, int stride16, int bins,
                const int32_t* __restrict__ ndense, const uint32_t* __restrict__ state,
                const int32_t* __restrict__ carry_nd, int carry_np, int spec, int carry_spec) {
  constexpr int64_t ROWB = FP4 ? TC_KCAP / 2 : TC_KCAP;
  if (tc_infeasible(state)) return;
  int ndmax = 0;   // no problem keeps more dense layers than the histogram pass wrote: nothing to do
  for (int q = 0; q < TcOutProbs(O, S.n); ++q) ndmax = max(ndmax, ndense[q]);
  // a carried side 0 (TcCarry) holds the layers below min(its spec, nd of every
  // problem of the launch that built it): its build overwrote the rest
  int cfrom = carry_spec;
  for (int q = 0; q < carry_np; ++q) cfrom = min(cfrom, carry_nd[q]);
  if (ndmax <= spec && !(carry_np > 0 && cfrom < ndense[O.prob[0]])) return;
  const int dwc = ((bins + 15) & ~15) / 16;
  const int64_t items = S.row_begin[S.n] * dwc;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = it / dwc;
    const int c = (int)(it - g * dwc);
    int lo = 0, hi = S.n - 1;   // side of row g: last s with row_begin[s] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (S.row_begin[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    const int nd = ndense[O.prob[lo]];
    const int lfrom = (carry_np > 0 && lo == 0) ? cfrom : spec;
    if (nd <= lfrom) continue;
    const int64_t r = g - S.row_begin[lo];
    const uint4* src = reinterpret_cast<const uint4*>(S.rows[lo] + r * (int64_t)stride16 + c * 16);
    const uint4 v0 = src[0], v1 = src[1];
    const uint32_t vs[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint8_t* rowp = O.out[lo] + r * ROWB;
    for (int l = lfrom; l < nd; ++l) {   // layers 1 .. spec: written by tc_hist_kernel
      const uint32_t bias = (0x8000u - (uint32_t)(l + 1)) * 0x00010001u;
      uint32_t o[4];
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
        const uint32_t m0 = ((vs[2 * wd] + bias) >> 15) & 0x00010001u;   // bits 0, 16
        const uint32_t m1 = ((vs[2 * wd + 1] + bias) >> 15) & 0x00010001u;
        if constexpr (FP4) {
          const uint32_t x = (m0 | (m0 >> 12)) & 0x11u, y = (m1 | (m1 >> 12)) & 0x11u;   // bits 0, 4
          o[wd] = (x | (y << 8)) << 1;                                                     // 16 bits: 4 nibbles
        } else {
          o[wd] = __byte_perm(m0, m1, 0x6420);
        }
      }
      if constexpr (FP4)
        reinterpret_cast<uint2*>(rowp)[l * dwc + c] = make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
      else
        reinterpret_cast<uint4*>(rowp)[l * dwc + c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

constexpr int TC_BUILD_THREADS = 512;

// Listed (sparse) columns and the zero padding up to the 128-column K block:
// the CTA's rows are taken in batches that give every thread one (row, chunk)
// item: 16 entries from the column list (L1 / L2), 16 counts gathered from
// the row, one 16-byte store.
template <bool FP4>
__global__ void __launch_bounds__(TC_BUILD_THREADS)
tc_build_kernel(const __grid_constant__ TcSides S, const __grid_constant__ TcOut O, int stride16, int bins,
                const uint32_t* __restrict__ collist, const int32_t* __restrict__ kblocks,
                const int32_t* __restrict__ ndense, const uint32_t* __restrict__ state, TcMasks mk) {
  constexpr int64_t ROWB = FP4 ? TC_KCAP / 2 : TC_KCAP;
  constexpr int KBC = FP4 ? 256 : 128;   // columns per K block
  if (tc_infeasible(state)) return;
  const int64_t R = S.row_begin[S.n];
  const int64_t r0 = blockIdx.x * R / gridDim.x, r1 = (blockIdx.x + 1) * R / gridDim.x;
  const int tid = threadIdx.x;
  const int dwc = ((bins + 15) & ~15) / 16;   // chunks per dense layer
  int side = -1, c0 = 0, ns = 0, q = 0;
  int64_t g = r0;
  while (g < r1) {
    int t = side < 0 ? 0 : side;
    while (g >= S.row_begin[t + 1]) ++t;
    if (t != side) {
      side = t;
      q = O.prob[t];
      c0 = ndense[q] * dwc;                 // first listed chunk
      ns = kblocks[q] * (KBC / 16) - c0;    // listed + padding chunks per row (may be 0)
    }
    if (ns <= 0) {   // every column of this side is in a dense layer
      g = min(r1, S.row_begin[t + 1]);
      continue;
    }
    const int rows_per = max(1, TC_BUILD_THREADS / ns);
    const int cnt = (int)min((int64_t)rows_per, min(r1, S.row_begin[t + 1]) - g);
    const int64_t rbase = g - S.row_begin[t];
    const uint32_t* cl = collist + (int64_t)q * TC_KCAP;
    for (int item = tid; item < cnt * ns; item += TC_BUILD_THREADS) {
      const int h = item / ns, c = c0 + item % ns;
      const uint16_t* row = S.rows[t] + (rbase + h) * (int64_t)stride16;
      const uint32_t* mrow = mk.row(g + h);
      const bool mv = mk.valid(g + h);
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(cl + c * 16) + k);
        const uint32_t es[4] = {x.x, x.y, x.z, x.w};
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t layer = es[b] >> 16, bin = es[b] & 0xffffu;
          uint32_t bit;
          if (mv && (layer == 2u || layer == 3u))   // from the row's layer mask
            bit = (__ldg(mrow + (layer - 2u) * TC_MW + (bin >> 5)) >> (bin & 31u)) & 1u;
          else if (mv && layer >= 4u && !((__ldg(mrow + TC_MDEEP + (bin >> 10)) >> ((bin >> 5) & 31u)) & 1u))
            bit = 0u;                       // no count >= 4 in the bin's 32-bin word
          else
            bit = (layer != 0u && (uint32_t)__ldg(row + bin) >= layer) ? 1u : 0u;
          word |= FP4 ? (bit << (4 * b + 1)) : (bit << (8 * b));
        }
        o[k] = word;
      }
      uint8_t* rowp = O.out[t] + (rbase + h) * ROWB;
      if constexpr (FP4)
        reinterpret_cast<uint2*>(rowp)[c] = make_uint2(o[0] | (o[1] << 16), o[2] | (o[3] << 16));
      else
        reinterpret_cast<uint4*>(rowp)[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    g += cnt;
  }
}

// ------------------------------------------------------------ epilogue ----
struct TcEpiProb {
  const int32_t* nkA;
  const int32_t* nkB;
  // per row of each side, precomputed by tc_info_kernel (one 16-byte load in
  // the epilogue instead of nk -> dependent table gathers): keys {rl, rh, e, nk'},
  // F {RN(1/nk'), nk'} (nk' = nk if > 0, else -1 with zero tables)
  const uint4* kinfoA;
  const uint4* kinfoB;
  const double2* yinfoA;
  const double2* yinfoB;
  sa_key128* keyA;
  sa_key128* keyB;
  uint16_t* num;
  double* sim;
  int64_t ld;
  double delta, ln1pd;
  int32_t form;
  int32_t sym;
  // sparse layers >= 2 (tc_sparse.cuh): the correction entries of key
  // (row, column block) are ents[koff[key] .. koff[key + 1]), sorted by
  // column, kpart[key] = their count per epilogue slice; koff / kpart point at
  // this problem's keys (nullptr: no entries)
  const uint32_t* koff;
  const uint32_t* kpart;
  const uint32_t* ents;
  int32_t tn, slice, bn;
  int32_t tma;   // bit 0: matrices leave by TMA tensor stores (KeyMatEpi::tma_chunk; omap of this problem
                 // valid); bit 1: n % 8 == 0 (the boxes never cross a row end inside a 16-byte unit)
};

// Output matrices are written once and never re-read by the kernel: streaming
// stores (st.global.cs) keep them from evicting the operand rows the tiles
// re-read from L2.
__device__ __forceinline__ void st_out(uint16_t* p, uint16_t v) { __stcs(reinterpret_cast<unsigned short*>(p), v); }
__device__ __forceinline__ void st_out(double* p, double v) { __stcs(p, v); }
// experiment flavours (SA_K2T_DEBUG): 8 skip, 16 plain st.global, 32 st.global.L1::no_allocate, else .cs
__device__ __forceinline__ void st_out_if(int fl, uint16_t* p, uint16_t v) {
  if (fl == 0) st_out(p, v);
  else if (fl == 16) *p = v;
  else if (fl == 32) asm volatile("st.global.L1::no_allocate.b16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}
__device__ __forceinline__ void st_out_if(int fl, double* p, double v) {
  if (fl == 0) st_out(p, v);
  else if (fl == 16) *p = v;
  else if (fl == 32) asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// K2T's key accumulators: while its GEMM runs, a key's two 64-bit words hold
// (X, Y) with key = Y 2^32 + X, so a 96-bit partial sum hi 2^64 + lo goes in
// with two fire-and-forget adds, X += lo mod 2^32, Y += hi 2^32 + lo / 2^32
// (no returned value, no carry chain; X stays below 2^64 for any realistic
// number of partials: < 2^32 each).  tc_key_finalize_kernel turns (X, Y) into
// the 128-bit key after the launch.
__device__ __forceinline__ void red_add_key_xy(sa_key128* k, uint64_t lo, uint32_t hi) {
  const unsigned long long x = lo & 0xffffffffull, y = ((unsigned long long)hi << 32) | (lo >> 32);
  if (x) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(&k->lo), "l"(x) : "memory");
  if (y) asm volatile("red.global.add.u64 [%0], %1;" ::"l"(&k->hi), "l"(y) : "memory");
}
__global__ void tc_key_finalize_kernel(sa_key128* __restrict__ keys, int64_t n, const uint32_t* __restrict__ state) {
  if (reinterpret_cast<const volatile uint32_t*>(state)[1] != 0u) return;   // declined: the fallback wrote true keys
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = keys[i].lo, y = keys[i].hi;
    const uint64_t lo = x + (y << 32);
    keys[i] = sa_key128{lo, (y >> 32) + (lo < x ? 1ull : 0ull)};
  }
}

// 96-bit (lo, hi) add
__device__ __forceinline__ void add96(uint64_t& lo, uint32_t& hi, uint64_t blo, uint32_t bhi) {
  lo += blo;
  hi += bhi + ((lo < blo) ? 1u : 0u);
}

// floor(C 2^64 / D) mod 2^64 (the exact-rank key term) from the
// D-side reciprocal tables rl + 2^32 rh = r = floor(2^64 / D), e = 2^64 mod D
// (0 <= C <= D < 2^16):  C r + floor(C e / D).  The quotient x / D of
// x = C e < 2^32 is taken without a division: floor(x / D) = floor(x (r + 1) / 2^64),
// because r + 1 - 2^64 / D < 1 and x 2^-64 < 2^-32 < 1 / D keep x (r + 1) / 2^64
// inside [x / D, floor(x / D) + 1) (e = 0 gives x = 0).  C = D gives 2^64, which
// wraps to 0 here: the caller adds it to the high word.
__device__ __forceinline__ uint64_t key_term_lo(uint32_t C, uint32_t rl, uint32_t rh, uint32_t e) {
  const uint64_t p = (uint64_t)C * rl + ((uint64_t)(C * rh) << 32);
  const uint32_t x = C * e;
  const uint64_t p0 = (uint64_t)x * rl;
  const uint64_t p1 = (uint64_t)x * rh + (p0 >> 32);
  const uint32_t s = (uint32_t)p0 + x;
  const uint32_t q = (uint32_t)((p1 + (s < x ? 1ull : 0ull)) >> 32);
  return p + q;
}

// the d^F term out of line: its log keeps registers the F-form fast path needs
__device__ __noinline__ void dF_term_outlined(uint64_t& lo, uint32_t& hi, uint32_t C, uint32_t D, double delta,
                                              double ln1pd) {
  add_dF_term(lo, hi, C, D, delta, ln1pd);
}

// MODE: which outputs this instantiation can write (EPI_KEYS | EPI_NUM |
// EPI_SIM); a launch picks the smallest one covering its problems, so the
// key path and the matrix path each get their own register allocation.
enum { EPI_KEYS = 1, EPI_NUM = 2, EPI_SIM = 4, EPI_ALL = 7 };

// Per-tile tables.  Every epilogue warp stages, for each column of its slice,
// before the accumulator is ready (tc_gemm.cuh):
//   key entry  {rl, rh, e, nk'}  reciprocal tables of D = nk' (EPI_KEYS)
//   F entry    {y, d}  y = RN(1 / nk'), d = nk'         (EPI_SIM)
// with nk' = nk if the column exists and nk > 0, else -1 (tables of 0: r = e
// = y = 0).  A pair then takes D = min(nk'_row, nk'_col) and the tables of
// whichever side is smaller; the -1 sentinel makes every term of a missing or
// empty (n < k, Z4) row or column 0 with no extra test: r = e = 0 gives key
// term 0, C = D is impossible, y = 0 gives F = 0.  The lanes read the entries
// of the chunk's columns as shared-memory broadcasts.
// Output tensor maps of the TMA-store matrix epilogue, per problem (in the
// kernel's parameter space, as TMA requires): F direct (16 x 32 box, 128-byte
// swizzle), F mirrored (16 x 16), C direct (16 x 32), C mirrored (32 x 16).
enum { OM_FD = 0, OM_FM = 1, OM_CD = 2, OM_CM = 3, OM_N = 4 };

template <int MODE>
struct KeyMatEpi {
  CUtensorMap omap[OM_N * tc::MAXPROB];   // first member: 64-byte aligned
  TcEpiProb e[tc::MAXPROB];
  const uint32_t* state;
  int dbg;   // experiments only (SA_K2T_DEBUG bit 8: matrix stores skipped)

  static constexpr bool KEYS = (MODE & EPI_KEYS) != 0;
  static constexpr bool SIM = (MODE & EPI_SIM) != 0;
  static constexpr bool MATS = (MODE & (EPI_NUM | EPI_SIM)) != 0;
  static constexpr int KOFF = 0;
  static constexpr int YOFF = KEYS ? 16 : 0;
  static constexpr int TAB_BYTES = (KEYS && SIM) ? 32 : 16;
  // the per-warp 32 x CW uint16 transpose buffer of the matrix path, plus (F
  // with the e2m1 stage sizes, where it fits) a 32-row {y, d} table
  //   CTA pairs (CG = 2, small stages): F itself goes through a 32 x CW fp64
  //   transpose buffer, so each F is computed once (f_transposed);
  //   one CTA (CG = 1): F is recomputed in the transposed pass, with a
  //   32-row {y, d} table where it fits (e2m1 stage sizes).
  //   CTA pairs (CG = 2, 31 KB stages): F computed once per pair and staged
  //   half a chunk at a time (32 rows x 8 doubles) for 16-byte direct stores
  //   (vec_direct; rows padded to a multiple of 16, else the path below);
  //   otherwise F is recomputed in the transposed pass, with a 32-row {y, d}
  //   table where it fits (e2m1 stage sizes).
  __host__ __device__ static constexpr bool vec_direct(int CW, int CG) { return SIM && CG == 2 && CW == 16; }
  __host__ __device__ static constexpr bool row_table(bool FP4, int CW, int CG) {
    return SIM && FP4 && !vec_direct(CW, CG);
  }
  // TMA-store staging (CTA pairs, C and F): per warp, the direct half of a
  // chunk (tma_chunk), 5 KB; the vector-store buffers of the fallback path
  // (3 KB) fit inside
  __host__ __device__ static constexpr bool tma_out(int CW, int CG) {
    return MODE == (EPI_NUM | EPI_SIM) && CG == 2 && CW == 16;
  }
  __host__ __device__ static constexpr int xpose_bytes(int CW, bool FP4, int CG) {
    return tma_out(CW, CG) ? 5120
                           : (MATS ? 64 * CW : 0) + (vec_direct(CW, CG) ? 32 * 8 * 8 : 0) +
                                 (row_table(FP4, CW, CG) ? 32 * 16 : 0);
  }
  __device__ void finish(int lane) const {
    if (MATS && lane == 0) tc::bulk_wait0();   // TMA stores of the last chunks complete before exit
  }

  struct State {
    uint64_t lo;      // row key, 96 bits
    uint32_t hi;
    uint32_t q0, q1, q2, q3;   // the next correction entries of this thread's (row, slice), column order
    uint32_t ep, ee;           // further entries: ents[ep .. ee)
    int nk;           // nk' of the row (sentinel -1: no row or nk = 0)
    int nk0;          // nk of the row (0 if none): the diagonal numerator C_ii
    int row_g;
    bool rv;          // the row exists
    uint32_t rl, rh, ek;
    double y, d;      // RN(1 / nk') and nk' as doubles (0 for the sentinel)
  };

  __device__ bool skip() const { return tc_infeasible(state); }

  // The per-tile loads (row info, the correction queue's index, the column
  // tables) all issued together into registers (`prefetch`: the column
  // tables as 4 x 32 unrolled, independent loads per lane -- slices up to 128
  // columns, wider ones load the rest directly), then consumed (`begin_pf`).
  // (Issuing tile t + 1's loads at the start of tile t measured neutral on
  // S5; the unrolled form took the S2a GEMM 1.979 -> 1.956 ms.)
  static constexpr int PFK = 4;
  struct Pf {
    uint4 kcol[PFK];
    double2 ycol[PFK];
    uint4 krow;
    double2 yrow;
    int nk0;
    uint32_t kb, ke, pc;
  };
  __device__ __forceinline__ void prefetch(Pf& p, const tc::Tile& T, int row, int lane, int cbeg, int cend) const {
    const TcEpiProb& E = e[T.pi];
    const int row_g = T.row0 + row;
    const bool rv = row < T.ra;
    p.nk0 = rv ? __ldg(E.nkA + row_g) : 0;
    if constexpr (KEYS) p.krow = rv ? __ldg(E.kinfoA + row_g) : make_uint4(0u, 0u, 0u, 0xffffffffu);
    if constexpr (SIM) p.yrow = rv ? __ldg(E.yinfoA + row_g) : make_double2(0.0, 0.0);
    p.kb = p.ke = p.pc = 0u;
    if (E.koff && rv && !(dbg & 256)) {   // (SA_K2T_DEBUG 256: experiment, corrections skipped)
      const int64_t key = (int64_t)row_g * E.tn + T.col0 / E.bn;
      p.kb = __ldg(E.koff + key);
      p.ke = __ldg(E.koff + key + 1);
      p.pc = __ldg(E.kpart + key);
    }
#pragma unroll
    for (int k = 0; k < PFK; ++k) {
      const int c = cbeg + lane + 32 * k;
      const bool cv = c < cend && c < T.rb && !(dbg & 128);   // (SA_K2T_DEBUG 128: experiment, no column tables)
      if constexpr (KEYS) p.kcol[k] = cv ? __ldg(E.kinfoB + T.col0 + c) : make_uint4(0u, 0u, 0u, 0xffffffffu);
      if constexpr (SIM) p.ycol[k] = cv ? __ldg(E.yinfoB + T.col0 + c) : make_double2(0.0, 0.0);
    }
  }
  __device__ __forceinline__ void begin_pf(State& s, const tc::Tile& T, const Pf& p, int row, int lane, int cbeg,
                                           int cend, uint8_t* tab) const {
    const TcEpiProb& E = e[T.pi];
    s.lo = 0;
    s.hi = 0;
    s.row_g = T.row0 + row;
    s.rv = row < T.ra;
    s.nk0 = p.nk0;
    s.nk = s.nk0 > 0 ? s.nk0 : -1;
    if constexpr (KEYS) {
      s.rl = p.krow.x;
      s.rh = p.krow.y;
      s.ek = p.krow.z;
    }
    if constexpr (SIM) {
      s.y = p.yrow.x;
      s.d = p.yrow.y;
    }
    // correction entries of (row, column block, slice): the first four in
    // registers (independent loads, issued before the accumulator wait)
    s.ep = s.ee = 0;
    s.q0 = s.q1 = s.q2 = s.q3 = 0xFFFFFFFFu;
    if (E.koff && s.rv && !(dbg & 256)) {
      const uint32_t kb = p.kb, ke = p.ke, pc = p.pc;
      const uint32_t part = (uint32_t)(cbeg / E.slice);
      const uint32_t before = part == 0 ? 0u : __vsadu4(pc & ((1u << (8 * part)) - 1u), 0u);   // slices < part
      const uint32_t avail = ke - kb;
      const uint32_t n = before < avail ? min((pc >> (8 * part)) & 0xffu, avail - before) : 0u;
      const uint32_t b = kb + before, e = b + n;
      if (n > 0) s.q0 = __ldg(E.ents + b);
      if (n > 1) s.q1 = __ldg(E.ents + b + 1);
      if (n > 2) s.q2 = __ldg(E.ents + b + 2);
      if (n > 3) s.q3 = __ldg(E.ents + b + 3);
      s.ep = b + min(n, 4u);
      s.ee = e;
    }
    if constexpr (KEYS || SIM) {
#pragma unroll
      for (int k = 0; k < PFK; ++k) {
        const int c = cbeg + lane + 32 * k;
        if (c < cend) {
          uint8_t* ent = tab + (c - cbeg) * TAB_BYTES;
          if constexpr (KEYS) *reinterpret_cast<uint4*>(ent + KOFF) = p.kcol[k];
          if constexpr (SIM) *reinterpret_cast<double2*>(ent + YOFF) = p.ycol[k];
        }
      }
      for (int c = cbeg + 32 * PFK + lane; c < cend; c += 32) {   // slices wider than 128 columns
        const bool cv = c < T.rb && !(dbg & 128);
        uint8_t* ent = tab + (c - cbeg) * TAB_BYTES;
        if constexpr (KEYS)
          *reinterpret_cast<uint4*>(ent + KOFF) =
              cv ? __ldg(E.kinfoB + T.col0 + c) : make_uint4(0u, 0u, 0u, 0xffffffffu);
        if constexpr (SIM)
          *reinterpret_cast<double2*>(ent + YOFF) = cv ? __ldg(E.yinfoB + T.col0 + c) : make_double2(0.0, 0.0);
      }
    }
    __syncwarp();
  }
  __device__ void begin(State& s, const tc::Tile& T, int row, int lane, int cbeg, int cend, uint8_t* tab) const {
    Pf p;
    prefetch(p, T, row, lane, cbeg, cend);
    begin_pf(s, T, p, row, lane, cbeg, cend, tab);
  }

  // Layers >= 2 of the chunk's pairs (tc_sparse.cu): add the entries whose
  // column falls in [col, col + CW) to the accumulator values.  Warp-uniform
  // loop: one pass per entry depth any lane still has in the chunk (usually
  // none or one); a pass applies each lane's head entry with a predicated add
  // per column (no dynamic register indexing) and pops it.
  template <int CW>
  __device__ __forceinline__ void correct(State& s, int col, uint32_t (&v)[CW]) const {
    const uint32_t lim = (uint32_t)(col + CW) << 16;
    while (__any_sync(0xffffffffu, s.q0 < lim)) {
      if (s.q0 < lim) {
        const uint32_t jj = (s.q0 >> 16) - (uint32_t)col, d = s.q0 & 0xffffu;
#pragma unroll
        for (int j = 0; j < CW; ++j) v[j] += jj == (uint32_t)j ? d : 0u;
        s.q0 = s.q1;
        s.q1 = s.q2;
        s.q2 = s.q3;
        s.q3 = s.ep < s.ee ? __ldg(e[0].ents + s.ep) : 0xFFFFFFFFu;
        s.ep += s.ep < s.ee ? 1u : 0u;
      }
    }
  }

  // F = C / D (reading Z19, division-free) with D = min(nk'_row, nk'_col)
  // taken by comparing the reciprocals: y_c > y_r <=> nk'_c < nk'_r for
  // nk' >= 1 (RN(1/D) is strictly decreasing over D < 2^16); a sentinel side
  // (y = d = 0) meets C = 0 (an empty or missing row / column: zero profile or
  // TMA zero fill), and C = 0 gives +0 whatever side is taken.
  __device__ __forceinline__ static double fsel(uint32_t C, double yr, double dr, double yc, double dc) {
    // y > 0 (or the +0 sentinel) order like their bit patterns; distinct D < 2^16
    // differ in the high word (relative gap 1/D > 2^-20), so an integer compare
    // of the high words (ALU pipe) decides yc > yr
    const bool col = __double2hiint(yc) > __double2hiint(yr);
    return f_ratio_y(C, col ? dc : dr, col ? yc : yr);
  }
  // experiment (SA_K2T_DEBUG bit 64): a stand-in for F with no fp64 arithmetic
  __device__ __forceinline__ double fsel_dbg(uint32_t C, double yr, double dr, double yc, double dc) const {
    if (dbg & 64) return __hiloint2double((int)(C ^ __double2hiint(yc)), (int)C);
    return fsel(C, yr, dr, yc, dc);
  }

  // the exact-rank term of pair (row, column entry k), numerator C: 64 low bits + the 2^64 carry
  __device__ __forceinline__ void fterm(const State& s, const uint4& k, uint32_t C, uint64_t& t, uint32_t& cd) const {
    const int nkc = (int)k.w;
    const bool cm = nkc < s.nk;
    t = key_term_lo(C, cm ? k.x : s.rl, cm ? k.y : s.rh, cm ? k.z : s.ek);
    cd = ((int)C == min(s.nk, nkc)) ? 1u : 0u;
  }

  // column sums of 8 columns' terms over the 32 rows of the warp: butterfly
  // over lane bits 4, 3, 2 (8 -> 1 value per lane), then xor 2, 1; lanes
  // 4 m hold column m and add it to its key with a 128-bit atomic
  __device__ __forceinline__ static void colsum8(uint64_t (&tlo)[8], uint32_t (&thi)[8], int lane, sa_key128* keys,
                                                  int c0, int jbase, int ncols) {
#pragma unroll
    for (int sft = 4, half = 16; sft >= 1; sft >>= 1, half >>= 1) {
      const bool upper = (lane & half) != 0;
#pragma unroll
      for (int i = 0; i < sft; ++i) {
        const uint64_t slo = upper ? tlo[i] : tlo[i + sft];
        const uint32_t shi = upper ? thi[i] : thi[i + sft];
        uint64_t klo = upper ? tlo[i + sft] : tlo[i];
        uint32_t khi = upper ? thi[i + sft] : thi[i];
        const uint64_t rlo = __shfl_xor_sync(0xffffffffu, slo, half);
        const uint32_t rhi = __shfl_xor_sync(0xffffffffu, shi, half);
        add96(klo, khi, rlo, rhi);
        tlo[i] = klo;
        thi[i] = khi;
      }
    }
    uint64_t lo = tlo[0];
    uint32_t hi = thi[0];
    {
      uint64_t rlo = __shfl_xor_sync(0xffffffffu, lo, 2);
      uint32_t rhi = __shfl_xor_sync(0xffffffffu, hi, 2);
      add96(lo, hi, rlo, rhi);
      rlo = __shfl_xor_sync(0xffffffffu, lo, 1);
      rhi = __shfl_xor_sync(0xffffffffu, hi, 1);
      add96(lo, hi, rlo, rhi);
    }
    // lane bits 4,3,2 name the column: 4 * b4 + 2 * b3 + b2
    const int jc = jbase + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && (lo | hi) && jc < ncols) red_add_key_xy(keys + c0 + jc, lo, hi);
  }

  // CW columns [col, col + CW) of this thread's row; lanes = 32 consecutive rows.
  template <int CW, bool FP4, int CG>
  __device__ void chunk(State& s, const tc::Tile& T, int row, int col, const uint32_t (&v)[CW], int lane,
                        const uint8_t* tab, int tj, uint8_t* xp) const {
    static_assert(CW == 16 || CW == 32, "chunk width");
    const TcEpiProb& E = e[T.pi];
    const bool sym = E.sym != 0;
    const int c0 = T.col0 + col;                        // global column of j = 0
    const int wrow0 = s.row_g - lane;                   // the warp's first row
    const bool upper = !sym || c0 > wrow0 + 31;         // every pair strictly above the diagonal (warp-uniform)
    const int ncols = min(CW, T.rb - col);              // columns that exist
    const uint8_t* ent = tab + tj * TAB_BYTES;
    if constexpr (row_table(FP4, CW, CG)) {
      if (tj == 0) {                                    // the warp's rows' {y, d}, once per tile
        reinterpret_cast<double2*>(xp + 64 * CW)[lane] = make_double2(s.y, s.d);
        __syncwarp();
      }
    }
    if (sym && c0 + CW <= wrow0) return;                // every pair below the diagonal: counted by its mirror

    if (KEYS && E.keyA) {
      const bool colsum = sym && E.keyB;
      if (upper && E.form != SA_RANK_DF) {
        // ---- fast path: every pair counted for the row (and mirrored), sentinels mask the rest
#pragma unroll
        for (int g = 0; g < CW / 8; ++g) {
          uint64_t tlo[8];
          uint32_t thi[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int j = g * 8 + jj;
            const uint4 k = *reinterpret_cast<const uint4*>(ent + j * TAB_BYTES + KOFF);
            fterm(s, k, v[j], tlo[jj], thi[jj]);
            add96(s.lo, s.hi, tlo[jj], thi[jj]);
          }
          if (colsum) colsum8(tlo, thi, lane, E.keyB, c0, g * 8, ncols);
        }
      } else {
        // ---- diagonal chunks and the d^F form: explicit masks
#pragma unroll
        for (int g = 0; g < CW / 8; ++g) {
          uint64_t tlo[8];
          uint32_t thi[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int j = g * 8 + jj;
            const int gc = c0 + j;
            const uint4 k = *reinterpret_cast<const uint4*>(ent + j * TAB_BYTES + KOFF);
            const bool cv = j < ncols;
            const bool diag = sym && gc == s.row_g;
            const uint32_t C = diag ? (uint32_t)s.nk0 : v[j];
            uint64_t lo = 0;
            uint32_t hi = 0;
            if (s.rv && cv && (!sym || gc >= s.row_g)) {
              if (E.form == SA_RANK_DF) {
                const int nkc0 = max((int)k.w, 0);
                dF_term_outlined(lo, hi, C, (uint32_t)min(s.nk0, nkc0), E.delta, E.ln1pd);
              } else {
                fterm(s, k, C, lo, hi);
              }
            }
            add96(s.lo, s.hi, lo, hi);
            const bool mirror = sym && gc > s.row_g;
            tlo[jj] = mirror ? lo : 0ull;
            thi[jj] = mirror ? hi : 0u;
          }
          if (colsum) colsum8(tlo, thi, lane, E.keyB, c0, g * 8, ncols);
        }
      }
    }

    if constexpr (MATS) {
      if (sym) mats<true, CW, FP4, CG>(s, E, T, col, c0, wrow0, upper, ncols, v, lane, ent, tj, xp);
      else mats<false, CW, FP4, CG>(s, E, T, col, c0, wrow0, upper, ncols, v, lane, ent, tj, xp);
    }
  }

  // Fast path with vector direct stores (vec_direct; 16 columns, rows padded
  // to a multiple of 16 elements): lanes = rows compute every F once, store
  // the mirrored elements (lanes = consecutive rows: coalesced) and stage F
  // half a chunk at a time in a 32 x 8 fp64 buffer (16-byte unit u of row r
  // at u ^ ((r >> 1) & 3): conflict-free both ways) and C in the 32 x 16
  // uint16 buffer; the direct row segments then leave as 16-byte stores
  // (4 lanes per 64-byte F row segment, 2 per 32-byte C segment).
  template <bool SYM>
  __device__ __forceinline__ void fast_vec(const State& s, const TcEpiProb& E, int c0, int wrow0,
                                           const uint32_t (&v)[16], int lane, const uint8_t* ent, uint8_t* xp,
                                           int stores) const {
    constexpr bool want_num = (MODE & EPI_NUM) != 0;
    const int64_t ld = E.ld;   // 64-bit offsets: n_b * ld may exceed 2^31
    uint16_t* const num = E.num;
    double* const sim = E.sim;
    uint8_t* const fb = xp + 64 * 16;
    const bool vst = stores != 8;
    uint32_t w[8];
    int64_t om = (int64_t)c0 * ld + s.row_g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double Fp = 0.0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int j = h * 8 + jj;
        const uint32_t C = v[j];
        if (j & 1) w[j >> 1] |= C << 16;
        else w[j >> 1] = C;
        const double2 yd = *reinterpret_cast<const double2*>(ent + j * TAB_BYTES + YOFF);
        const double F = fsel_dbg(C, s.y, s.d, yd.x, yd.y);
        if constexpr (SYM) {
          if constexpr (want_num) st_out_if(stores, num + om, (uint16_t)C);
          st_out_if(stores, sim + om, F);
        }
        om += ld;
        if (jj & 1)
          *reinterpret_cast<double2*>(fb + lane * 64 + (((jj >> 1) ^ ((lane >> 1) & 3)) * 16)) = make_double2(Fp, F);
        else
          Fp = F;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int rho = (lane >> 2) + 8 * k, u = lane & 3;
        const double2 f2 = *reinterpret_cast<const double2*>(fb + rho * 64 + ((u ^ ((rho >> 1) & 3)) * 16));
        if (vst) __stcs(reinterpret_cast<double2*>(sim + (int64_t)(wrow0 + rho) * ld + c0 + h * 8 + u * 2), f2);
      }
      __syncwarp();
    }
    if constexpr (want_num) {
#pragma unroll
      for (int q = 0; q < 2; ++q)
        *reinterpret_cast<uint4*>(xp + lane * 32 + ((q ^ ((lane >> 2) & 1)) * 16)) =
            make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int rho = (lane >> 1) + 16 * k, u = lane & 1;
        const uint4 c8 = *reinterpret_cast<const uint4*>(xp + rho * 32 + ((u ^ ((rho >> 2) & 1)) * 16));
        if (vst) __stcs(reinterpret_cast<uint4*>(num + (int64_t)(wrow0 + rho) * ld + c0 + u * 8), c8);
      }
      __syncwarp();
    }
  }

  // The chunk's 32 x 16 pairs (lanes = rows, every pair strictly above the
  // diagonal).  The mirrored block (rows c0.., columns wrow0..) leaves straight
  // from registers: for each column j the warp's 32 lanes hold 32 consecutive
  // elements of mirrored row c0 + j, one coalesced store each (256 B of F,
  // 64 B of C, whole sectors).  The direct block (rows wrow0.., columns c0..)
  // has lanes = rows, so it goes through shared memory (F [32 rows][128 B],
  // 16-byte unit u of row r at u ^ (r & 7), SWIZZLE_128B; C [32 rows][32 B];
  // 5 KB per warp) and leaves by two TMA tensor stores.  Shared-memory bandwidth
  // is what the CTA shares with the MMA's operand reads and the TMA operand
  // loads, so only the half that needs a transpose is staged.  Lane 0 owns the
  // bulk group: before rewriting the buffer it waits until the previous
  // chunk's stores have read it.  (Measured, config 4 S5 GEMM: both halves
  // through shared memory, 8 warps 3.74 ms; 8-column halves, 16 warps 4.35 ms;
  // direct rows from registers + mirror by TMA, 16 warps 4.79 ms.)
  __device__ __forceinline__ void tma_chunk(const State& s, int pi, int c0, int wrow0, int ncols, const uint32_t (&v)[16],
                                            int lane, const uint8_t* ent, uint8_t* xp, const TcEpiProb& E) const {
    double F[16];
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t C = v[j];
      if (j & 1) w[j >> 1] |= C << 16;
      else w[j >> 1] = C;
      const double2 yd = *reinterpret_cast<const double2*>(ent + j * TAB_BYTES + YOFF);
      F[j] = fsel(C, s.y, s.d, yd.x, yd.y);   // (no per-pair run-time switch: it costs a branch per pair)
    }
    // the mirrored half (experiment builds: SA_MIRROR_V2 pairs lanes so that F leaves as 16-byte
    // stores, two rows of one mirrored row per lane; SA_MIRROR_LAST issues it after the TMA stores)
    auto mirror = [&]() {
#ifdef SA_MIRROR_V2
      if (ncols == 16 && __all_sync(0xffffffffu, s.rv) && !(dbg & (8 | 512))) {
        const int odd = lane & 1;
        double* fm2 = E.sim + (int64_t)(c0 + odd) * E.ld + (s.row_g - odd);
        uint16_t* cmr = E.num + (int64_t)c0 * E.ld + s.row_g;
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const double send = odd ? F[j] : F[j + 1];
          const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
          const double2 o = odd ? make_double2(recv, F[j + 1]) : make_double2(F[j], recv);
          __stcs(reinterpret_cast<double2*>(fm2 + (int64_t)j * E.ld), o);
          __stcs(reinterpret_cast<unsigned short*>(cmr + (int64_t)j * E.ld), (unsigned short)v[j]);
          __stcs(reinterpret_cast<unsigned short*>(cmr + (int64_t)(j + 1) * E.ld), (unsigned short)v[j + 1]);
        }
        return;
      }
#endif
      if (s.rv && !(dbg & (8 | 512))) {   // (SA_K2T_DEBUG 512: experiment, mirrored stores skipped)
        double* fm = E.sim + (int64_t)c0 * E.ld + s.row_g;
        uint16_t* cmr = E.num + (int64_t)c0 * E.ld + s.row_g;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < ncols) {
            __stcs(fm + (int64_t)j * E.ld, F[j]);
            __stcs(reinterpret_cast<unsigned short*>(cmr + (int64_t)j * E.ld), (unsigned short)v[j]);
          }
        }
      }
    };
#ifdef SA_MIRROR_LAST
    if (dbg & 4096) {
      mirror();
      return;
    }
#else
    mirror();
#endif
    if (dbg & 4096) return;   // (SA_K2T_DEBUG 4096: experiment, no staging / TMA stores of the direct half)
    if (lane == 0) tc::bulk_wait_read0();
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 8; ++u)
      *reinterpret_cast<double2*>(xp + lane * 128 + ((u ^ (lane & 7)) * 16)) = make_double2(F[2 * u], F[2 * u + 1]);
    *reinterpret_cast<uint4*>(xp + 4096 + lane * 32) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(xp + 4096 + lane * 32 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
    tc::fence_async_smem();
    __syncwarp();
    if (lane == 0 && !(dbg & 8)) {
      const uint32_t xs = tc::s_addr(xp);
      const CUtensorMap* om = omap + OM_N * pi;
      if (E.tma & 4) {   // evict-first: the output stream should not push the operand rows out of L2
        const uint64_t pol = tc::policy_evict_first();
        tc::tma_store_2d_hint(om + OM_FD, xs, c0, wrow0, pol);
        if (!(dbg & 1024)) tc::tma_store_2d_hint(om + OM_CD, xs + 4096, c0, wrow0, pol);
      } else {
        tc::tma_store_2d(om + OM_FD, xs, c0, wrow0);
        if (!(dbg & 1024)) tc::tma_store_2d(om + OM_CD, xs + 4096, c0, wrow0);
      }
      tc::bulk_commit();
    }
#ifdef SA_MIRROR_LAST
    mirror();
#endif
  }

  // the numerator / F matrices of a chunk (the host sets num (sim) on every
  // problem of a launch whose MODE has NUM (SIM))
  template <bool SYM, int CW, bool FP4, int CG>
  __device__ __forceinline__ void mats(State& s, const TcEpiProb& E, const tc::Tile& T, int col, int c0, int wrow0,
                                       bool upper, int ncols, const uint32_t (&v)[CW], int lane, const uint8_t* ent,
                                       int tj, uint8_t* xp) const {
    constexpr bool want_num = (MODE & EPI_NUM) != 0;
    constexpr bool want_sim = SIM;
    constexpr bool RT = row_table(FP4, CW, CG);
    constexpr bool VD = vec_direct(CW, CG);
    const bool rows_all = wrow0 + 32 <= T.row0 + T.ra;   // warp-uniform
    const double2* rtab = reinterpret_cast<const double2*>(xp + 64 * CW);   // written by chunk() at tj = 0
    if constexpr (SYM && tma_out(CW, CG)) {
      // every pair strictly above the diagonal: TMA tensor stores.  Ragged
      // rows and columns are clipped by the maps' bounds -- at 16-byte
      // granularity in the inner (column) dimension, so when a row's end is
      // not 16-byte aligned for uint16 (n % 8 != 0) the chunks that cross it
      // take the per-thread path, which never touches the padding columns.
      if (upper && E.tma && ((E.tma & 2) || c0 + CW <= T.col0 + T.rb)) {
        tma_chunk(s, T.pi, c0, wrow0, ncols, v, lane, ent, xp, E);
        return;
      }
      if (lane == 0) tc::bulk_wait_read0();   // the staging buffer is about to be reused by the path below
      __syncwarp();
    }
    if (upper && ncols == CW && rows_all) {
      const int stores = dbg & 56;
      // ---- fast path (all 32 rows and CW columns exist, no diagonal).
      // (1) lanes = rows: F of every pair; the mirrored element (gc, row)
      // with lanes = consecutive rows (coalesced); C staged in the warp's
      // 32 x CW uint16 transpose buffer (16-byte units XOR-swizzled by the
      // row: conflict-free both ways).  Element offsets fit 32 bits (n_b ld < 2^31).
      constexpr int Q = CW / 8;                          // 16-byte units per buffer row
      constexpr int QSH = CW == 16 ? 2 : 1;              // swizzle: unit ^ ((row >> QSH) % Q)
      const int64_t ld = E.ld;   // 64-bit offsets: n_b * ld may exceed 2^31
      uint16_t* const num = E.num;
      double* const sim = E.sim;
      if constexpr (VD) {
        if ((ld & 15) == 0) {
          fast_vec<SYM>(s, E, c0, wrow0, v, lane, ent, xp, stores);
          return;
        }
      }
      {
        uint32_t w[CW / 2];
        int64_t om = (int64_t)c0 * ld + s.row_g;
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const uint32_t C = v[j];
          if (j & 1) w[j >> 1] |= C << 16;
          else w[j >> 1] = C;
          if constexpr (SYM) {
            if constexpr (want_num) st_out_if(stores, num + om, (uint16_t)C);
            if constexpr (want_sim) {
              const double2 yd = *reinterpret_cast<const double2*>(ent + j * TAB_BYTES + YOFF);
              st_out_if(stores, sim + om, fsel_dbg(C, s.y, s.d, yd.x, yd.y));
            }
          }
          om += ld;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int qs = q ^ ((lane >> QSH) & (Q - 1));
          *reinterpret_cast<uint4*>(xp + lane * (CW * 2) + qs * 16) =
              make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
      }
      __syncwarp();
      // (2) lanes = columns: the direct row segments (row, c0 ..) from the
      // buffer, 32 / CW rows per pass; row data from the row table (or shuffles)
      const int cl = lane % CW;
      double yc = 0.0, dc = 0.0;
      if constexpr (want_sim) {
        const double2 yd = *reinterpret_cast<const double2*>(ent + cl * TAB_BYTES + YOFF);
        yc = yd.x;
        dc = yd.y;
      }
      constexpr int RPP = 32 / CW;
      int64_t od = (int64_t)(wrow0 + lane / CW) * ld + c0 + cl;
#pragma unroll
      for (int pss = 0; pss < CW; ++pss) {
        const int i = pss * RPP + lane / CW;              // buffer row = warp row
        const int qs = (cl >> 3) ^ ((i >> QSH) & (Q - 1));
        const uint32_t C = *reinterpret_cast<const uint16_t*>(xp + i * (CW * 2) + qs * 16 + (cl & 7) * 2);
        if constexpr (want_num) st_out_if(stores, num + od, (uint16_t)C);
        if constexpr (want_sim) {
          double y_i, d_i;
          if constexpr (RT) {
            const double2 r = rtab[i];
            y_i = r.x;
            d_i = r.y;
          } else {
            y_i = __shfl_sync(0xffffffffu, s.y, i);
            d_i = __shfl_sync(0xffffffffu, s.d, i);
          }
          st_out_if(stores, sim + od, fsel_dbg(C, y_i, d_i, yc, dc));
        }
        od += RPP * ld;
      }
      __syncwarp();
    } else {
      // ---- diagonal / ragged chunks: per-element masks
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int gc = c0 + j;
        if (!s.rv || j >= ncols || (SYM && gc < s.row_g)) continue;
        const bool diag = SYM && gc == s.row_g;
        const uint32_t C = diag ? (uint32_t)s.nk0 : v[j];
        double F = 0.0;
        if constexpr (want_sim) {
          const double2 yd = *reinterpret_cast<const double2*>(ent + j * TAB_BYTES + YOFF);
          F = fsel(C, s.y, s.d, yd.x, yd.y);
        }
        const int64_t od = (int64_t)s.row_g * E.ld + gc;
        if constexpr (want_num) st_out(E.num + od, (uint16_t)C);
        if constexpr (want_sim) st_out(E.sim + od, F);
        if (SYM && !diag) {
          const int64_t om = (int64_t)gc * E.ld + s.row_g;
          if constexpr (want_num) st_out(E.num + om, (uint16_t)C);
          if constexpr (want_sim) st_out(E.sim + om, F);
        }
      }
    }
  }

  __device__ void end(State& s, const tc::Tile& T, int row) const {
    const TcEpiProb& E = e[T.pi];
    if (KEYS && E.keyA && s.rv && (s.lo | s.hi)) red_add_key_xy(E.keyA + s.row_g, s.lo, s.hi);
    (void)row;
  }
};

// ------------------------------------------------------------- F pass ----
// F = C / min(nk_row, nk_col) elementwise over an na x nb numerator matrix
// (row stride ld), written as fp64 (Z19: IEEE RN, via f_ratio).  Used for
// S5's similarity matrix after a numerator-only GEMM epilogue: a coalesced
// HBM-bound pass (2 bytes read, 8 written per entry) at full occupancy instead
// of fp64 work inside the tensor-core kernel's epilogue.
__global__ void __launch_bounds__(256)
ratio_kernel(const uint16_t* __restrict__ num, const int32_t* __restrict__ nkA, const int32_t* __restrict__ nkB,
             int64_t na, int64_t nb, int64_t ld, double* __restrict__ sim, const uint32_t* __restrict__ state) {
  if (state && tc_infeasible(state)) return;   // K2T declined: the fallback engine wrote sim itself
  for (int64_t i = blockIdx.x; i < na; i += gridDim.x) {
    const int nki = nkA[i];
    const uint16_t* nr = num + i * ld;
    double* sr = sim + i * ld;
#pragma unroll 4
    for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) {
      const int D = min(nki, nkB[j]);
      sr[j] = D > 0 ? f_ratio(nr[j], (uint32_t)D) : 0.0;
    }
  }
}

sa_status ratio_launch(const uint16_t* num, const int32_t* nkA, const int32_t* nkB, int64_t na, int64_t nb,
                       int64_t ld, double* sim, cudaStream_t st, const uint32_t* state) {
  if (na <= 0 || nb <= 0) return SA_OK;
  SA_TRY(ensure_recip_tables_tu(st));
  const int64_t blocks = std::min<int64_t>(na, 148 * 8);
  ratio_kernel<<<(unsigned)blocks, 256, 0, st>>>(num, nkA, nkB, na, nb, ld, sim, state);
  SA_LAUNCHED();
  return SA_OK;
}

// ---------------------------------------------------- division self-test ----
__global__ void f_division_check_kernel(unsigned long long* bad) {
  const uint32_t D = blockIdx.x + 1;
  unsigned long long nb = 0;
  for (uint32_t C = threadIdx.x; C <= D; C += blockDim.x) {
    const double a = f_ratio(C, D), b = __ddiv_rn((double)C, (double)D);
    nb += (__double_as_longlong(a) != __double_as_longlong(b)) ? 1ull : 0ull;
  }
  if (nb) atomicAdd(bad, nb);
}

// Zero a key array when the launch was declined (see tc_launch).
__global__ void tc_reset_keys_kernel(sa_key128* __restrict__ keys, int64_t n, const uint32_t* __restrict__ state) {
  if (!tc_infeasible(state)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = sa_key128{0, 0};
}

// ------------------------------------------------------------- host ----
template <class Epi, int EW, int CW, bool FP4, int CG>
static sa_status tc_configure() {
  if constexpr (CG == 1) {
    static_assert(tc::smem_of(EW, CW, FP4, Epi::TAB_BYTES, Epi::xpose_bytes(CW, FP4, 1)) <= 232448, "shared memory");
    SA_CUDA(cudaFuncSetAttribute(tc::gemm_kernel<Epi, EW, CW, FP4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem_of(EW, CW, FP4, Epi::TAB_BYTES, Epi::xpose_bytes(CW, FP4, 1))));
  } else {
    static_assert(tc::smem2_of(EW, CW, FP4, Epi::TAB_BYTES, Epi::xpose_bytes(CW, FP4, 2)) <= 232448, "shared memory");
    SA_CUDA(cudaFuncSetAttribute(tc::gemm2_kernel<Epi, EW, CW, FP4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem2_of(EW, CW, FP4, Epi::TAB_BYTES, Epi::xpose_bytes(CW, FP4, 2))));
  }
  return SA_OK;
}
template <class Epi, int EW, int CW, bool FP4, int CG>
static void tc_gemm(int64_t grid, const tc::Batch& batch, const tc::Maps& maps, int64_t tiles,
                    const KeyMatEpi<EPI_ALL>& epi, cudaStream_t st) {
  Epi k;
  static_assert(sizeof k == sizeof epi, "epilogue layouts");
  std::memcpy(&k, &epi, sizeof k);
  if constexpr (CG == 1)
    tc::gemm_kernel<Epi, EW, CW, FP4><<<(unsigned)grid, tc::threads_of(EW),
                                         tc::smem_of(EW, CW, FP4, Epi::TAB_BYTES, Epi::xpose_bytes(CW, FP4, 1)), st>>>(
        batch, maps, tiles, k);
  else
    tc::gemm2_kernel<Epi, EW, CW, FP4><<<(unsigned)grid, tc::threads_of(EW),
                                          tc::smem2_of(EW, CW, FP4, Epi::TAB_BYTES, Epi::xpose_bytes(CW, FP4, 2)), st>>>(
        batch, maps, tiles, k);
}
// the (epilogue mode, geometry) instantiations a launch can pick.  Matrices
// (NUM | SIM): 8 (default) or 16 epilogue warps; on CTA pairs the direct halves
// leave by TMA tensor stores (5 KB of staging per warp).
template <bool FP4, int CG>
static sa_status tc_configure_all() {
  constexpr int CW_ALL = FP4 ? 16 : 32;
  sa_status cs = tc_configure<KeyMatEpi<EPI_KEYS>, 16, 16, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_KEYS>, 12, 16, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_KEYS>, 8, CW_ALL, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_NUM>, 16, 16, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_SIM>, 16, 16, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_NUM | EPI_SIM>, 16, 16, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_NUM | EPI_SIM>, 8, 16, FP4, CG>();
  if (cs == SA_OK) cs = tc_configure<KeyMatEpi<EPI_KEYS | EPI_NUM>, 8, CW_ALL, FP4, CG>();
  return cs;
}
template <bool FP4, int CG>
static void tc_gemm_mode(int mode, int keysw, int matsw, int64_t grid, const tc::Batch& batch, const tc::Maps& maps,
                         int64_t tiles, const KeyMatEpi<EPI_ALL>& epi, cudaStream_t st) {
  constexpr int CW_ALL = FP4 ? 16 : 32;
  if (mode == EPI_KEYS && keysw == 16) tc_gemm<KeyMatEpi<EPI_KEYS>, 16, 16, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else if (mode == EPI_KEYS && keysw == 12)
    tc_gemm<KeyMatEpi<EPI_KEYS>, 12, 16, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else if (mode == EPI_KEYS) tc_gemm<KeyMatEpi<EPI_KEYS>, 8, CW_ALL, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else if (mode == EPI_NUM) tc_gemm<KeyMatEpi<EPI_NUM>, 16, 16, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else if (mode == EPI_SIM) tc_gemm<KeyMatEpi<EPI_SIM>, 16, 16, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else if ((mode & EPI_KEYS) == 0 && matsw != 8)
    tc_gemm<KeyMatEpi<EPI_NUM | EPI_SIM>, 16, 16, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else if ((mode & EPI_KEYS) == 0)
    tc_gemm<KeyMatEpi<EPI_NUM | EPI_SIM>, 8, 16, FP4, CG>(grid, batch, maps, tiles, epi, st);
  else tc_gemm<KeyMatEpi<EPI_KEYS | EPI_NUM>, 8, CW_ALL, FP4, CG>(grid, batch, maps, tiles, epi, st);   // never with F
}

// Format / pair switches are read at every launch (a test can switch them);
// g_last_fp4 = the format of the last K2T launch in this process (sa_ctx_tc_operand).
static bool env_on(const char* name, bool dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) != 0 : dflt;
}
static std::atomic<int> g_last_fp4{1};
// CTA pairs (tcgen05 cta_group::2, tc_gemm.cuh) unless SA_K2T_PAIR=0
static bool tc_pairs() { return env_on("SA_K2T_PAIR", true); }

static sa_status tc_encode_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int box_rows, int64_t rowb) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)rowb, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)rowb};
  const cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled (K2T) failed (%d)", (int)r);
  return SA_OK;
}


// Output maps of the TMA-store matrix epilogue (KeyMatEpi::tma_chunk) for an
// na x nb matrix with row stride ld elements: columns are the inner dimension.
static sa_status tc_encode_out(CUtensorMap* m, void* base, CUtensorMapDataType dt, int esize, int64_t na, int64_t nb,
                               int64_t ld, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)nb, (cuuint64_t)na};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * esize)};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, dt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swz,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled (K2T output) failed (%d)", (int)r);
  return SA_OK;
}
// SA_K2T_STORE_HINT=1: the TMA tensor stores of the matrix epilogue carry an
// L2 evict-first policy (0: no hint)
static bool store_hint_setting() {
  const char* e = getenv("SA_K2T_STORE_HINT");
  return e ? atoi(e) != 0 : true;
}

// SA_K2T_TMA_STORE=0: the matrix epilogue's per-thread stores instead of TMA tensor stores
static bool tma_store_enabled() {
  const char* e = getenv("SA_K2T_TMA_STORE");
  return !(e && atoi(e) == 0);
}

// Epilogue geometry of a launch's MODE (mirrors tc_gemm_mode): epilogue warps
// and chunk width -> the column slice each warp owns (the sparse entries are
// keyed by it).
struct EpiGeo {
  int ew, cw;
};
static EpiGeo epi_geo(int mode, int keysw, int matsw, bool fp4, bool pairs) {
  const int cw_all = fp4 ? 16 : 32;
  if (mode == EPI_KEYS) return keysw == 16 ? EpiGeo{16, 16} : keysw == 12 ? EpiGeo{12, 16} : EpiGeo{8, cw_all};
  if (mode == EPI_NUM || mode == EPI_SIM) return {16, 16};
  if ((mode & EPI_KEYS) == 0) return matsw != 8 ? EpiGeo{16, 16} : EpiGeo{8, 16};
  return {8, cw_all};
}

// Sparse layers >= 2 (tc_sparse.cu): SA_K2T_SPARSE=0 disables them (every
// problem keeps its layers >= 2 as MMA columns, round-1 behaviour);
// SA_K2T_SPARSE_BUDGET = b: a problem goes sparse when its correction terms
// number at most pairs / b (default 8).
// SA_K2T_SPARSE=2 forces it (tests): every problem whose terms fit a large
// buffer (64 per pair, at most 2^28 in all) goes sparse.
static int sparse_setting() {
  const char* e = getenv("SA_K2T_SPARSE");
  return e ? atoi(e) : 1;
}
static bool sparse_enabled() { return sparse_setting() != 0; }
static int sparse_budget() {
  const char* e = getenv("SA_K2T_SPARSE_BUDGET");
  const int b = e ? atoi(e) : 8;
  return b >= 1 ? b : 8;
}
constexpr int SP_REC_PER_ROW = 48;   // record budget per row (overflow: the launch stays dense)

sa_status tc_launch(const std::vector<MsProblem>& probs_in, int ldw16, int32_t bins, uint32_t* state,
                    uint32_t* cols_out, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1, TcCarry* keep,
                    const TcCarry* use) {
  SA_TRY(ensure_recip_tables_tu(st));
  const int g_num_sms = device_sms();
  static DeviceOnce once;
  SA_TRY(once.run([]() -> sa_status {
    SA_CUDA(cudaFuncSetAttribute(tc_hist_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * (TC_LCAP - TC_HREG) * TC_WPL * 4));
    SA_CUDA(cudaFuncSetAttribute(tc_hist_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 2 * (TC_LCAP - TC_HREG) * TC_WPL * 4));
    sa_status cs = tc_configure_all<false, 1>();
    if (cs == SA_OK) cs = tc_configure_all<true, 1>();
    if (cs == SA_OK) cs = tc_configure_all<false, 2>();
    if (cs == SA_OK) cs = tc_configure_all<true, 2>();
    return cs;
  }));
  const int stride16 = 2 * ldw16;
  const bool fp4 = tc_fp4_operands();
  const bool pairs = tc_pairs();
  g_last_fp4.store(fp4 ? 1 : 0);
  const int64_t rowb = fp4 ? TC_KCAP / 2 : TC_KCAP;
  const int kbc = fp4 ? 256 : 128;
  const int BN = fp4 ? tc::Geo<true>::BN : tc::Geo<false>::BN;
  static const bool fpass = [] {
    const char* e = getenv("SA_K2T_FPASS");
    return e && atoi(e) != 0;
  }();
  static const int debug = [] {   // SA_K2T_DEBUG: component switches for experiments (tc_gemm.cuh, KeyMatEpi)
    const char* e = getenv("SA_K2T_DEBUG");
    return e ? atoi(e) : 0;
  }();
  // epilogue warps (16 for keys: with layer 1 alone the key epilogue, not the
  // MMA, bounds S2a / S2d, and more warps hide its latency -- config 4:
  // S2a GEMM 3.16 / 2.67 / 2.60 ms with 8 / 12 / 16; 12 for the matrices on
  // CTA pairs), read per launch
  const int keysw = [] {
    const char* e = getenv("SA_K2T_KEYSW");
    const int w = e ? atoi(e) : 16;
    return w == 8 || w == 12 ? w : 16;
  }();
  const int matsw = [] {   // matrix-epilogue warps: 8 (default; config 4 S5 GEMM 3.59 ms vs 3.92 with 16) or 16
    const char* e = getenv("SA_K2T_MATSW");
    const int w = e ? atoi(e) : 8;
    return w == 16 ? 16 : 8;
  }();
  const bool sp_on = sparse_enabled() && bins <= SP_BINS;
  const int spec = sp_on ? 1 : TC_SPEC_MAX;   // dense layers the histogram pass writes
  const int budget = sparse_budget();
  std::vector<MsProblem> probs;
  for (const auto& p : probs_in)
    if (p.na > 0 && p.nb > 0) probs.push_back(p);
  size_t i0 = 0;
  while (i0 < probs.size()) {
    const size_t i1 = std::min(probs.size(), i0 + (size_t)tc::MAXPROB);
    const int np = (int)(i1 - i0);
    Scratch scratch(st);
    // sides (A rows of every problem, plus B rows of rectangular ones) and selection
    TcSides sides{};
    TcOut outs{};
    TcSel sel{};
    sel.n = np;
    sel.first = (int)i0;
    std::vector<int64_t> side_n;
    auto add_side = [&](const uint32_t* rows, int64_t n, int q) {
      sides.rows[sides.n] = reinterpret_cast<const uint16_t*>(rows);
      sides.row_begin[sides.n + 1] = sides.row_begin[sides.n] + n;
      outs.prob[sides.n] = q;
      side_n.push_back(n);
      return sides.n++;
    };
    TcNk sides_nk{};
    for (int q = 0; q < np; ++q) {
      const MsProblem& P = probs[i0 + q];
      sel.side_a[q] = add_side(P.A, P.na, q);
      sides_nk.nk[sel.side_a[q]] = P.nkA;
      sel.side_b[q] = P.sym ? -1 : add_side(P.B, P.nb, q);
      if (!P.sym) sides_nk.nk[sel.side_b[q]] = P.nkB;
    }
    // the epilogue MODE of this launch (keys and F in one launch would need
    // both column tables: F then goes through the F pass -- numerators in the
    // epilogue, ratio_kernel after) and its geometry
    bool any_keys = false;
    for (int q = 0; q < np; ++q) any_keys = any_keys || probs[i0 + q].keyA;
    const bool fpass_here = fpass || any_keys;
    int mode = 0;
    bool all_sym = true;
    for (int q = 0; q < np; ++q) {
      const MsProblem& P = probs[i0 + q];
      mode |= (P.keyA ? EPI_KEYS : 0) | ((P.num || (fpass_here && P.sim)) ? EPI_NUM : 0) |
              ((!fpass_here && P.sim) ? EPI_SIM : 0);
      all_sym = all_sym && P.sym;
    }
    const EpiGeo geo = epi_geo(mode, keysw, matsw, fp4, pairs);
    const int slice = tc::slice_of(geo.ew, geo.cw, fp4);

    SA_ALLOC(planes, uint32_t, (size_t)sides.n * 2 * TC_PLANE);
    SA_ALLOC(collist, uint32_t, (size_t)np * TC_KCAP);
    SA_ALLOC(kblocks, int32_t, np);
    int32_t* ndense = (keep && keep->scratch && i0 == 0) ? keep->scratch->alloc<int32_t>(np) : scratch.alloc<int32_t>(np);
    if (!ndense) return fail(SA_E_NOMEM, "scratch allocation of K2T dense-layer counts failed");
    SA_CUDA(cudaMemsetAsync(planes, 0, (size_t)sides.n * 2 * TC_PLANE * 4, st));
    const int64_t R = sides.row_begin[sides.n];
    // operand rows: one output per side (its problem's column list).  A
    // keeping launch (S2a) puts all its sides (contiguous source rows) in one
    // buffer of the caller's scratch; a launch given a carry whose rows are
    // its first side (S2d's queries) reuses rows, dense layers and planes.
    const bool carried = use && use->valid && use->fp4 == fp4 && np == 1 && sides.n >= 1 &&
                         reinterpret_cast<const uint32_t*>(sides.rows[0]) == use->src && side_n[0] == use->nrows;
    bool keeping = keep && keep->scratch && i0 == 0 && probs.size() <= (size_t)tc::MAXPROB;
    for (int sd = 1; keeping && sd < sides.n; ++sd)
      keeping = sides.rows[sd] == sides.rows[0] + (sides.row_begin[sd] - sides.row_begin[0]) * (int64_t)stride16;
    Scratch* kscr = keeping ? keep->scratch : &scratch;   // where the carried state lives
    uint8_t* side_out[2 * tc::MAXPROB];
    uint8_t* kept = keeping ? keep->scratch->alloc<uint8_t>((size_t)R * rowb) : nullptr;
    if (keeping && !kept) return fail(SA_E_NOMEM, "scratch allocation of K2T operand rows failed");
    for (int sd = 0; sd < sides.n; ++sd) {
      uint8_t* o = nullptr;
      if (carried && sd == 0) o = use->rows;
      else if (kept) o = kept + sides.row_begin[sd] * rowb;
      else o = scratch.alloc<uint8_t>((size_t)side_n[sd] * rowb);
      if (!o) return fail(SA_E_NOMEM, "scratch allocation of K2T operand rows failed");
      side_out[sd] = outs.out[sd] = o;
    }
    if (carried)
      SA_CUDA(cudaMemcpyAsync(planes, use->seen1, TC_PLANE * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    const int64_t hfrom = carried ? sides.row_begin[1] : 0;
    // layer-2/3 masks of the rows this launch's histogram pass covers (a keeping
    // launch's live in the caller's scratch, for the next launch's carried side)
    TcMasks mk{};
    mk.split = hfrom;
    mk.carried = carried ? use->masks : nullptr;
    // the layer-2/3 masks serve the build of listed (dense-path) columns; a
    // launch expecting the sparse path skips them (a dense problem then reads
    // its counts from the profile rows)
    mk.own_valid = sp_on ? 0 : 1;
    mk.carried_valid = carried ? use->masks_valid : 0;
    mk.own = mk.own_valid ? kscr->alloc<uint32_t>((size_t)(R - hfrom) * TC_MROW) : nullptr;
    if (mk.own_valid && !mk.own) return fail(SA_E_NOMEM, "scratch allocation of K2T layer masks failed");
    const int hrows = sp_on ? hist_rows<false>() : TC_HIST_ROWS;   // rows per CTA iteration
    const int hx = (int)std::max<int64_t>(
        1, std::min<int64_t>((R - hfrom + hrows - 1) / hrows, (sp_on ? SA_HIST_LEAN_GRID : 4) * g_num_sms));
    const int hsm = 2 * (TC_LCAP - TC_HREG) * TC_WPL * 4;
    // sparse-layer records: per hist CTA a segment, then one dense array (after
    // the carried launch's records, when there are any)
    TcRecOut ro{};
    SpBuffers spb;
    uint32_t rec_cap = 0;
    if (sp_on) {
      const int64_t per_cta = (R - hfrom + hx - 1) / hx;
      const int rec_per_row = sparse_setting() == 2 ? 8 * SP_REC_PER_ROW : SP_REC_PER_ROW;
      ro.seg_cap = (uint32_t)(per_cta * rec_per_row + 64);
      ro.seg = scratch.alloc<uint2>((size_t)hx * ro.seg_cap);
      ro.cnt = scratch.alloc<uint32_t>(hx);
      ro.on = 1;
      const int64_t cap64 = (int64_t)hx * ro.seg_cap + (carried && use->recs ? use->rec_cap : 0);
      rec_cap = (uint32_t)std::min<int64_t>(cap64, (int64_t)1 << 31);
      spb.recs = kscr->alloc<uint2>(rec_cap);
      spb.nrec = kscr->alloc<uint32_t>(4);   // [0] records, [2] incomplete (some segment overflowed)
      spb.povf = scratch.alloc<uint32_t>(tc::MAXPROB);
      ro.povf = spb.povf;
      ro.incomplete = spb.nrec + 2;
      if (!ro.seg || !ro.cnt || !spb.recs || !spb.nrec || !spb.povf)
        return fail(SA_E_NOMEM, "scratch allocation of K2T sparse records failed");
      SA_CUDA(cudaMemsetAsync(spb.nrec, 0, 4 * sizeof(uint32_t), st));
      SA_CUDA(cudaMemsetAsync(spb.povf, 0, tc::MAXPROB * sizeof(uint32_t), st));
      if (carried && use->recs) SA_TRY(sp_copy_records(use->recs, use->nrec, use->rec_cap, spb.recs, spb.nrec + 1,
                                                       g_num_sms, st));
    }
    // sparse-path launches build layer 1 and the records only; the deeper
    // planes of the problems that end up dense come from a second, planes-only
    // pass over just their rows (after the plan)
    if (sp_on) {
      if (fp4)
        tc_hist_kernel<true, false><<<hx, TC_HIST_THREADS, 0, st>>>(sides, outs, stride16, bins, planes, state, hfrom,
                                                                     mk, spec, ro, 0, nullptr);
      else
        tc_hist_kernel<false, false><<<hx, TC_HIST_THREADS, 0, st>>>(sides, outs, stride16, bins, planes, state,
                                                                      hfrom, mk, spec, ro, 0, nullptr);
    } else if (fp4) {
      tc_hist_kernel<true, true><<<hx, TC_HIST_THREADS, hsm, st>>>(sides, outs, stride16, bins, planes, state, hfrom,
                                                                   mk, spec, ro, 1, nullptr);
    } else {
      tc_hist_kernel<false, true><<<hx, TC_HIST_THREADS, hsm, st>>>(sides, outs, stride16, bins, planes, state, hfrom,
                                                                    mk, spec, ro, 1, nullptr);
    }
    SA_LAUNCHED();
    if (sp_on) {
      // a carried side without records (its launch ran with sparse layers off) cannot go sparse
      const bool carry_ok = !carried || use->recs;
      TcRecOvf ov{};
      ov.carried_prob = outs.prob[0];
      ov.povf = spb.povf;
      tc_rec_compact_kernel<<<hx, 256, 0, st>>>(ro.seg, ro.cnt, hx, ro.seg_cap, spb.recs, rec_cap, spb.nrec,
                                                 carried ? spb.nrec + 1 : nullptr, ov);
      SA_LAUNCHED();
      if (!carry_ok) {   // carried rows without records (their launch ran with sparse layers off): dense
        SA_CUDA(cudaMemsetAsync(spb.povf, 0xFF, tc::MAXPROB * sizeof(uint32_t), st));
        SA_CUDA(cudaMemsetAsync(spb.nrec + 2, 0xFF, sizeof(uint32_t), st));
      }
    }
    if (kept) {
      uint32_t* s1 = keep->scratch->alloc<uint32_t>(TC_PLANE);
      if (!s1) return fail(SA_E_NOMEM, "scratch allocation of K2T planes failed");
      tc_or_planes_kernel<<<TC_PLANE / 256, 256, 0, st>>>(planes, sides.n, s1, state);
      SA_LAUNCHED();
      keep->valid = true;
      keep->src = reinterpret_cast<const uint32_t*>(sides.rows[0]);
      keep->nrows = R;
      keep->fp4 = fp4;
      keep->rows = kept;
      keep->seen1 = s1;
      keep->ndense = ndense;
      keep->np = np;
      keep->masks = mk.own;
      keep->masks_valid = mk.own_valid;
      keep->spec = spec;
      keep->recs = sp_on ? spb.recs : nullptr;
      keep->nrec = sp_on ? spb.nrec : nullptr;
      keep->rec_cap = rec_cap;
    }
    // plan of the sparse layers: which problems take them (device-decided)
    SpLaunch L{};
    if (sp_on) {
      for (int sd = 0; sd <= sides.n; ++sd) L.row_begin[sd] = sides.row_begin[sd];
      L.nsides = sides.n;
      L.nprob = np;
      uint64_t kb = 0, ecap = 0;
      int64_t na_all = 0;
      for (int q = 0; q < np; ++q) {
        const MsProblem& P = probs[i0 + q];
        L.side_a[q] = sel.side_a[q];
        L.side_b[q] = sel.side_b[q];
        L.tn[q] = (int32_t)((P.nb + BN - 1) / BN);
        L.key_base[q] = kb;
        L.abase[q] = na_all;
        na_all += P.na;
        kb += (uint64_t)P.na * L.tn[q];
        const uint64_t npair = P.sym ? (uint64_t)P.na * (P.na - 1) / 2 : (uint64_t)P.na * P.nb;
        L.cap[q] = sparse_setting() == 2 ? std::min<uint64_t>(npair * 64, (uint64_t)1 << 28) : npair / budget;
        if (L.tn[q] > SP_TN_MAX || P.nb >= (1 << 23)) L.cap[q] = 0;   // key / block-counter limits of the row build
        ecap += L.cap[q];
      }
      L.key_base[np] = kb;
      L.abase[np] = na_all;
      L.nkeys = (int64_t)kb;
      L.bn = BN;
      L.slice = slice;
      L.rec_cap = rec_cap;
      // kpart packs one 8-bit count per epilogue slice: at most 4 slices (the
      // 20-warp experiment geometry has 5 and stays dense)
      L.enabled = ecap < ((uint64_t)1 << 32) && kb < ((uint64_t)1 << 32) && (BN + slice - 1) / slice <= 4 ? 1 : 0;
      L.terms_out = (sel.first + np <= SA_TC_COLS_MAX && cols_out)
                        ? reinterpret_cast<unsigned long long*>(state + SA_TC_TERMS_AT) + sel.first
                        : nullptr;
      spb.bincnt = scratch.alloc<uint32_t>((size_t)sides.n * SP_BINS);
      spb.binoff = scratch.alloc<uint32_t>((size_t)sides.n * SP_BSTRIDE);
      spb.sidebase = scratch.alloc<uint32_t>(sides.n);
      spb.blist = scratch.alloc<uint2>(rec_cap);
      spb.sorted = scratch.alloc<uint2>(rec_cap);
      spb.bslot = scratch.alloc<uint32_t>(rec_cap);
      spb.spos = scratch.alloc<uint32_t>(rec_cap);
      spb.rcnt = scratch.alloc<uint32_t>((size_t)R);
      spb.rstart = scratch.alloc<uint32_t>((size_t)R + 1);
      spb.rlist = scratch.alloc<uint32_t>(rec_cap);
      spb.mode = scratch.alloc<int32_t>(np);
      spb.flags = scratch.alloc<uint32_t>(4);
      spb.rowcnt = scratch.alloc<uint32_t>((size_t)na_all);
      spb.rowoff = scratch.alloc<uint32_t>((size_t)na_all + 1);
      spb.koff = scratch.alloc<uint32_t>((size_t)kb + 1);
      spb.kpart = scratch.alloc<uint32_t>((size_t)kb + 1);
      spb.scan_tmp = scratch.alloc<uint32_t>((size_t)(std::max<int64_t>(R, na_all) / 4096) + 2);
      spb.ents = scratch.alloc<uint32_t>((size_t)std::max<uint64_t>(ecap, 1));
      if (!spb.bincnt || !spb.binoff || !spb.sidebase || !spb.blist || !spb.sorted || !spb.bslot || !spb.spos ||
          !spb.rcnt || !spb.rstart ||
          !spb.rlist || !spb.mode || !spb.flags || !spb.rowcnt || !spb.rowoff || !spb.koff || !spb.kpart ||
          !spb.scan_tmp || !spb.ents)
        return fail(SA_E_NOMEM, "scratch allocation of K2T sparse-layer buffers failed");
      SA_CUDA(cudaMemsetAsync(spb.bincnt, 0, (size_t)sides.n * SP_BINS * 4, st));
      SA_CUDA(cudaMemsetAsync(spb.flags, 0, 16, st));
      SA_CUDA(cudaMemsetAsync(spb.sidebase, 0, (size_t)sides.n * 4, st));
      SA_CUDA(cudaMemsetAsync(spb.rcnt, 0, (size_t)R * 4, st));
      SA_TRY(sp_build(L, spb, g_num_sms, st));
      {
        // the dense problems' planes for layers >= 2 (all rows, carried ones included)
        TcMasks mk0{};
        TcRecOut ro0{};
        const int hx0 = (int)std::max<int64_t>(1, std::min<int64_t>((R + TC_HIST_ROWS - 1) / TC_HIST_ROWS,
                                                                     4 * g_num_sms));
        if (fp4)
          tc_hist_kernel<true, true><<<hx0, TC_HIST_THREADS, hsm, st>>>(sides, outs, stride16, bins, planes, state, 0, mk0,
                                                                  spec, ro0, 1, spb.mode);
        else
          tc_hist_kernel<false, true><<<hx0, TC_HIST_THREADS, hsm, st>>>(sides, outs, stride16, bins, planes, state, 0,
                                                                   mk0, spec, ro0, 1, spb.mode);
        SA_LAUNCHED();
      }
      if (cols_out && sel.first + np <= SA_TC_COLS_MAX)
        SA_CUDA(cudaMemcpyAsync(state + SA_TC_MODE_AT + sel.first, spb.mode, np * 4, cudaMemcpyDeviceToDevice, st));
    } else if (cols_out && sel.first + np <= SA_TC_COLS_MAX) {
      SA_CUDA(cudaMemsetAsync(state + SA_TC_MODE_AT + sel.first, 0, np * 4, st));
    }
    tc_select_kernel<<<np, 1024, 0, st>>>(sel, planes, bins, kbc, collist, kblocks, ndense, state, cols_out,
                                          sp_on ? spb.mode : nullptr);
    SA_LAUNCHED();
    uint4* kinfo = scratch.alloc<uint4>((size_t)R);
    double2* yinfo = scratch.alloc<double2>((size_t)R);
    if (!kinfo || !yinfo) return fail(SA_E_NOMEM, "scratch allocation of K2T row info failed");
    tc_info_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((R + 255) / 256, 4 * g_num_sms)), 256, 0, st>>>(
        sides, sides_nk, kinfo, yinfo, state);
    SA_LAUNCHED();
    const int bx = (int)std::max<int64_t>(1, std::min<int64_t>(R, 4 * g_num_sms));
    const int32_t* cnd = carried ? use->ndense : nullptr;
    const int cnp = carried ? use->np : 0;
    const int cspec = carried ? use->spec : spec;
    if (fp4) {
      tc_dense_kernel<true><<<8 * g_num_sms, 256, 0, st>>>(sides, outs, stride16, bins, ndense, state, cnd, cnp, spec,
                                                           cspec);
      SA_LAUNCHED();
      tc_build_kernel<true><<<bx, TC_BUILD_THREADS, 0, st>>>(sides, outs, stride16, bins, collist, kblocks, ndense,
                                                             state, mk);
    } else {
      tc_dense_kernel<false><<<8 * g_num_sms, 256, 0, st>>>(sides, outs, stride16, bins, ndense, state, cnd, cnp, spec,
                                                            cspec);
      SA_LAUNCHED();
      tc_build_kernel<false><<<bx, TC_BUILD_THREADS, 0, st>>>(sides, outs, stride16, bins, collist, kblocks, ndense,
                                                              state, mk);
    }
    SA_LAUNCHED();
    if (sp_on) SA_TRY(sp_entries(L, spb, g_num_sms, st));
    // GEMM
    tc::Batch batch{};
    tc::Maps maps;
    std::memset(&maps, 0, sizeof maps);
    KeyMatEpi<EPI_ALL> epi{};
    epi.state = state;
    epi.dbg = debug;
    int64_t tiles = 0;
    for (int q = 0; q < np; ++q) {
      const MsProblem& P = probs[i0 + q];
      tc::Problem& T = batch.p[q];
      T.na = P.na;
      T.nb = P.nb;
      T.sym = P.sym;
      T.tiles_n = (P.nb + BN - 1) / BN;
      T.tile_begin = tiles;
      T.kblocks = kblocks + q;
      T.map = q;
      if (pairs)
        tiles += fp4 ? tc::problem_tiles<tc::Geo<true>::BN, tc::TBM2>(P.na, P.nb, P.sym != 0)
                     : tc::problem_tiles<tc::Geo<false>::BN, tc::TBM2>(P.na, P.nb, P.sym != 0);
      else
        tiles += fp4 ? tc::problem_tiles<tc::Geo<true>::BN>(P.na, P.nb, P.sym != 0)
                     : tc::problem_tiles<tc::Geo<false>::BN>(P.na, P.nb, P.sym != 0);
      const uint8_t* a = side_out[sel.side_a[q]];
      const uint8_t* b = P.sym ? a : side_out[sel.side_b[q]];
      SA_TRY(tc_encode_map(&maps.m[2 * q], a, P.na, tc::BM, rowb));
      SA_TRY(tc_encode_map(&maps.m[2 * q + 1], b, P.nb, pairs ? BN / 2 : BN, rowb));
      TcEpiProb& E = epi.e[q];
      E.nkA = P.nkA;
      E.nkB = P.nkB;
      {
        const int64_t ra = sides.row_begin[sel.side_a[q]];
        const int64_t rb = sides.row_begin[P.sym ? sel.side_a[q] : sel.side_b[q]];
        E.kinfoA = kinfo + ra;
        E.kinfoB = kinfo + rb;
        E.yinfoA = yinfo + ra;
        E.yinfoB = yinfo + rb;
      }
      E.keyA = P.keyA;
      E.keyB = P.sym ? P.keyB : nullptr;
      // S5's F: in the tensor-core epilogue (default), or (SA_K2T_FPASS=1) numerators
      // there and F by ratio_kernel after
      E.num = P.num;
      E.sim = fpass_here ? nullptr : P.sim;
      if (fpass_here && P.sim && !P.num) {
        E.num = scratch.alloc<uint16_t>((size_t)P.na * P.ld);
        if (!E.num) return fail(SA_E_NOMEM, "scratch allocation of K2T numerators failed");
      }
      E.ld = P.ld;
      E.form = P.form;
      E.delta = P.delta;
      E.ln1pd = P.ln1pd;
      E.sym = P.sym;
      if (sp_on) {
        E.koff = spb.koff + L.key_base[q];
        E.kpart = spb.kpart + L.key_base[q];
        E.ents = spb.ents;
        E.tn = L.tn[q];
        E.slice = slice;
        E.bn = BN;
      }
      // the matrices leave by TMA tensor stores (CTA pairs, NUM | SIM, symmetric,
      // rows a multiple of 16 bytes apart, 16-byte aligned bases)
      E.tma = 0;
      if (pairs && mode == (EPI_NUM | EPI_SIM) && P.sym && E.num && E.sim && tma_store_enabled() && P.ld % 8 == 0 &&
          (reinterpret_cast<uintptr_t>(E.num) & 15) == 0 && (reinterpret_cast<uintptr_t>(E.sim) & 15) == 0) {
        CUtensorMap* om = epi.omap + OM_N * q;
        SA_TRY(tc_encode_out(om + OM_FD, E.sim, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, P.na, P.nb, P.ld, 16, 32,
                             CU_TENSOR_MAP_SWIZZLE_128B));
        SA_TRY(tc_encode_out(om + OM_CD, E.num, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, P.na, P.nb, P.ld, 16, 32,
                             CU_TENSOR_MAP_SWIZZLE_NONE));
        // bit 1: every row end 16-byte aligned (no edge fallback); bit 2: evict-first stores
        E.tma = 1 | (P.nb % 8 == 0 ? 2 : 0) | (store_hint_setting() ? 4 : 0);
      }
    }
    // every problem of the launch gets every output its MODE writes (the
    // epilogue's fast paths test no pointer): scratch for a problem that did
    // not ask for one (only in mixed batches)
    for (int q = 0; q < np; ++q) {
      TcEpiProb& E = epi.e[q];
      const MsProblem& P = probs[i0 + q];
      if ((mode & EPI_NUM) && !E.num) E.num = scratch.alloc<uint16_t>((size_t)P.na * P.ld);
      if ((mode & EPI_SIM) && !E.sim) E.sim = scratch.alloc<double>((size_t)P.na * P.ld);
      if (((mode & EPI_NUM) && !E.num) || ((mode & EPI_SIM) && !E.sim))
        return fail(SA_E_NOMEM, "scratch allocation of K2T output matrices failed");
    }
    batch.n = np;
    static const int group = [] {   // SA_K2T_GROUP: row blocks per group of the tile order
      const char* e = getenv("SA_K2T_GROUP");
      const int g = e ? atoi(e) : 12;
      return g >= 1 && g <= 1024 ? g : 12;
    }();
    // SA_K2T_GROUP_KEYS: the same for a keys-only launch of symmetric problems
    // (S2a's blocks), default one group per problem (column-major over the
    // triangle: the whole A side stays in L2, nothing else streams through it).
    // Measured on config 4 (scripts/gpu_group_sweep.sh): S2a 3.75 -> 3.64 ms
    // with one group, while S2d and S5 (12.5 GB of output through L2) lose
    // with large groups and gain a little at 12 (S5 GEMM 4.80 -> 4.74 ms).
    static const int group_keys = [] {
      const char* e = getenv("SA_K2T_GROUP_KEYS");
      const int g = e ? atoi(e) : 1 << 20;
      return g >= 1 ? g : 1 << 20;
    }();
    batch.group = (mode == EPI_KEYS && all_sym) ? group_keys : group;
    // SA_K2T_EVICT_LAST: operand L2 policies (tc::side_policy bits: 1 / 2 the
    // A / B side evict_last, 4 / 8 evict_first, 0 no hint).  Default 1: the
    // group's A row band, re-read by every column block of the group, is kept
    // over the output stream (scripts/gpu_policy_sweep.sh, config 4: S5 GEMM
    // 4.75 -> 4.73 ms; any evict_first side is slower, up to +0.56 ms).
    // The one-CTA kernel applies evict_last to both sides for any non-zero value.
    static const int evict_last = [] {
      const char* e = getenv("SA_K2T_EVICT_LAST");
      return e ? atoi(e) : 1;
    }();
    batch.evict_last = evict_last;
    batch.debug = debug;
    static const int serp = [] {   // SA_K2T_SERP=0: plain group order (tc::serp_index)
      const char* e = getenv("SA_K2T_SERP");
      return e ? atoi(e) : 1;
    }();
    batch.serp = serp;
    // decoded tile table (every GEMM warp reads its tile's coordinates with one load)
    uint2* ttab = scratch.alloc<uint2>((size_t)std::max<int64_t>(tiles, 1));
    if (!ttab) return fail(SA_E_NOMEM, "scratch allocation of the K2T tile table failed");
    {
      const unsigned tb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tiles + 255) / 256, 4 * g_num_sms));
      if (pairs) {
        if (fp4) tc::tile_table_kernel<tc::Geo<true>::BN, tc::TBM2><<<tb, 256, 0, st>>>(batch, tiles, ttab);
        else tc::tile_table_kernel<tc::Geo<false>::BN, tc::TBM2><<<tb, 256, 0, st>>>(batch, tiles, ttab);
      } else {
        if (fp4) tc::tile_table_kernel<tc::Geo<true>::BN, tc::BM><<<tb, 256, 0, st>>>(batch, tiles, ttab);
        else tc::tile_table_kernel<tc::Geo<false>::BN, tc::BM><<<tb, 256, 0, st>>>(batch, tiles, ttab);
      }
      SA_LAUNCHED();
    }
    batch.table = ttab;
    const int64_t grid = pairs ? 2 * std::min<int64_t>(tiles, g_num_sms / 2) : std::min<int64_t>(tiles, g_num_sms);
    if (ev0) SA_CUDA(cudaEventRecord(ev0, st));   // the GEMM kernel alone (SA_PHASE_GEMM*)
    if (pairs) {
      if (fp4) tc_gemm_mode<true, 2>(mode, keysw, matsw, grid, batch, maps, tiles, epi, st);
      else tc_gemm_mode<false, 2>(mode, keysw, matsw, grid, batch, maps, tiles, epi, st);
    } else {
      if (fp4) tc_gemm_mode<true, 1>(mode, keysw, matsw, grid, batch, maps, tiles, epi, st);
      else tc_gemm_mode<false, 1>(mode, keysw, matsw, grid, batch, maps, tiles, epi, st);
    }
    SA_LAUNCHED();
    if (ev1) SA_CUDA(cudaEventRecord(ev1, st));
    for (int q = 0; q < np; ++q) {
      const MsProblem& P = probs[i0 + q];
      if (fpass_here && P.sim) SA_TRY(ratio_launch(epi.e[q].num, P.nkA, P.nkB, P.na, P.nb, P.ld, P.sim, st, state));
      // (X, Y) key accumulators -> 128-bit keys (a symmetric problem's column
      // sums go to the same array as its row sums)
      if (P.keyA) {
        tc_key_finalize_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((P.na + 255) / 256, 4 * g_num_sms)),
                                 256, 0, st>>>(P.keyA, P.na, state);
        SA_LAUNCHED();
      }
      if (P.sym && P.keyB && P.keyB != P.keyA) {
        tc_key_finalize_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((P.nb + 255) / 256, 4 * g_num_sms)),
                                 256, 0, st>>>(P.keyB, P.nb, state);
        SA_LAUNCHED();
      }
    }
    i0 = i1;
  }
  // A launch of more than MAXPROB problems runs chunk by chunk: if a later
  // chunk is declined (state[1]), the earlier chunks' GEMMs have already added
  // their key terms, and the fallback engine recomputes every problem -- so
  // the keys go back to zero first (device-guarded: nothing happens when K2T
  // completed the launch).  Matrices are overwritten by the fallback anyway.
  if (probs.size() > (size_t)tc::MAXPROB) {
    for (const auto& P : probs) {
      if (P.keyA) {
        tc_reset_keys_kernel<<<64, 256, 0, st>>>(P.keyA, P.na, state);
        SA_LAUNCHED();
      }
      if (P.sym && P.keyB && P.keyB != P.keyA) {
        tc_reset_keys_kernel<<<64, 256, 0, st>>>(P.keyB, P.nb, state);
        SA_LAUNCHED();
      }
    }
  }
  return SA_OK;
}

// Operand format of K2T: packed e2m1 0/1.0 columns on kind::mxf4 (default: twice
// the kind::i8 MMA rate, half the operand bytes; exact, tc_gemm.cuh) or u8 0/1
// columns on kind::i8 (SA_K2T_FP4=0).
bool tc_fp4_operands() { return env_on("SA_K2T_FP4", true); }
bool tc_last_fp4() { return g_last_fp4.load() != 0; }

sa_status f_division_selftest(int64_t* mismatches_h) {
  SA_TRY(ensure_recip_tables_tu(0));
  unsigned long long* d = nullptr;
  SA_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  SA_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
  f_division_check_kernel<<<65535, 256>>>(d);
  const cudaError_t e = cudaGetLastError();
  unsigned long long h = 0;
  if (e == cudaSuccess) cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(SA_E_CUDA, "division self-test launch: %s", cudaGetErrorString(e));
  SA_CUDA(cudaGetLastError());
  *mismatches_h = (int64_t)h;
  return SA_OK;
}

}  // namespace sa
