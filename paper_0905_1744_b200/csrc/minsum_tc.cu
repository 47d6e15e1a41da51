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
#include <cstring>

#include "common.cuh"
#include "keyterm.cuh"
#include "tc_gemm.cuh"

namespace sa {

constexpr int TC_LCAP = 32;                    // threshold layers tracked
constexpr int TC_WPL = 256;                    // plane words per layer (bins <= 8192)
constexpr int TC_PLANE = TC_LCAP * TC_WPL;     // words per plane (32 KB)
constexpr int TC_KCAP = 32768;                 // columns (bytes) per operand row

// state words (ctx->dcount): [0] largest count, [1] K2T infeasible, [2] K2T enabled for this call
__device__ __forceinline__ bool tc_infeasible(const uint32_t* state) {
  return reinterpret_cast<const volatile uint32_t*>(state)[1] != 0u;
}

struct TcSide {
  const uint16_t* rows;
  int64_t n;
};
struct TcSides {
  TcSide s[2 * tc::MAXPROB];
  int n;
};

// ---------------------------------------------------------- histogram ----
__global__ void __launch_bounds__(512)
tc_hist_kernel(const __grid_constant__ TcSides sides, int stride16, uint32_t* __restrict__ planes,
               uint32_t* __restrict__ state) {
  extern __shared__ uint32_t sp[];   // [2][TC_PLANE]
  const TcSide S = sides.s[blockIdx.y];
  for (int w = threadIdx.x; w < 2 * TC_PLANE; w += blockDim.x) sp[w] = 0u;
  __syncthreads();
  uint32_t mx = 0;
  const int chunks = stride16 / 8;
  for (int64_t r = blockIdx.x; r < S.n; r += gridDim.x) {
    const uint4* row = reinterpret_cast<const uint4*>(S.rows + r * (int64_t)stride16);
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
      const uint4 w4 = row[c];
      if ((w4.x | w4.y | w4.z | w4.w) == 0u) continue;
      const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t v = (ws[q >> 1] >> (16 * (q & 1))) & 0xffffu;
        if (!v) continue;
        mx = max(mx, v);
        const int t = c * 8 + q;
        const uint32_t bit = 1u << (t & 31);
        const int L = min((int)v, TC_LCAP);
        for (int l = 0; l < L; ++l) {
          const int word = l * TC_WPL + (t >> 5);
          const uint32_t old = atomicOr(&sp[word], bit);
          if (old & bit) atomicOr(&sp[TC_PLANE + word], bit);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&state[0], mx);
  __syncthreads();
  uint32_t* g1 = planes + (int64_t)blockIdx.y * 2 * TC_PLANE;
  uint32_t* g2 = g1 + TC_PLANE;
  for (int w = threadIdx.x; w < TC_PLANE; w += blockDim.x) {
    const uint32_t s1 = sp[w];
    uint32_t s2 = sp[TC_PLANE + w];
    if (s1) s2 |= atomicOr(&g1[w], s1) & s1;   // a bit another CTA already saw is now seen twice
    if (s2) atomicOr(&g2[w], s2);
  }
}

// ------------------------------------------------------ column select ----
struct TcSel {
  int side_a[tc::MAXPROB], side_b[tc::MAXPROB];   // side_b = -1: symmetric
  int n;
  int first;                                        // index of problem 0 in the whole call
};

__global__ void __launch_bounds__(1024)
tc_select_kernel(const __grid_constant__ TcSel sel, const uint32_t* __restrict__ planes,
                 uint32_t* __restrict__ collist, int32_t* __restrict__ kblocks, uint32_t* __restrict__ state,
                 uint32_t* __restrict__ cols_out) {
  __shared__ uint32_t warp_tot[32];
  const int q = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int PER = TC_PLANE / 1024;   // 8 words per thread
  const uint32_t* a = planes + (int64_t)sel.side_a[q] * 2 * TC_PLANE;
  const uint32_t* b = sel.side_b[q] >= 0 ? planes + (int64_t)sel.side_b[q] * 2 * TC_PLANE : nullptr;
  uint32_t m[PER];
  uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int w = tid * PER + i;
    m[i] = b ? (a[w] & b[w]) : a[TC_PLANE + w];
    cnt += __popc(m[i]);
  }
  // block exclusive scan of cnt
  uint32_t x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;   // inclusive
  }
  __syncthreads();
  const uint32_t total = warp_tot[31];
  if (tid == 0 && cols_out && sel.first + q < SA_TC_COLS_MAX) cols_out[sel.first + q] = total;
  uint32_t pos = x - cnt + (wid ? warp_tot[wid - 1] : 0u);
  const uint32_t kpad = max(128u, (total + 127u) & ~127u);
  const bool too_many = kpad > (uint32_t)TC_KCAP;
  const bool deep = reinterpret_cast<const volatile uint32_t*>(state)[0] > (uint32_t)TC_LCAP;
  if (too_many || deep) {
    if (tid == 0) {
      atomicOr(&state[1], 1u);
      kblocks[q] = 1;
    }
    return;
  }
  uint32_t* out = collist + (int64_t)q * TC_KCAP;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int w = tid * PER + i;
    const uint32_t layer = (uint32_t)(w / TC_WPL) + 1u;
    const uint32_t bin0 = (uint32_t)(w % TC_WPL) * 32u;
    uint32_t mm = m[i];
    while (mm) {
      const int bpos = __ffs(mm) - 1;
      mm &= mm - 1;
      out[pos++] = (bin0 + (uint32_t)bpos) | (layer << 16);
    }
  }
  for (uint32_t p = total + tid; p < kpad; p += blockDim.x) out[p] = 0u;   // layer 0: padding column
  if (tid == 0) kblocks[q] = (int32_t)(kpad / 128u);
}

// ------------------------------------------------------- operand rows ----
struct TcBuild {
  const uint16_t* rows[2 * tc::MAXPROB];
  uint8_t* out[2 * tc::MAXPROB];
  int64_t row_begin[2 * tc::MAXPROB + 1];   // prefix of row counts over targets
  int prob[2 * tc::MAXPROB];
  int n;
};

constexpr int TC_BUILD_THREADS = 512;

__global__ void __launch_bounds__(TC_BUILD_THREADS)
tc_build_kernel(const __grid_constant__ TcBuild B, int stride16, const uint32_t* __restrict__ collist,
                const int32_t* __restrict__ kblocks, const uint32_t* __restrict__ state) {
  if (tc_infeasible(state)) return;
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* cols = sm;                                          // TC_KCAP entries
  uint16_t* row = reinterpret_cast<uint16_t*>(sm + TC_KCAP);    // stride16 counts
  const int64_t R = B.row_begin[B.n];
  const int64_t r0 = blockIdx.x * R / gridDim.x, r1 = (blockIdx.x + 1) * R / gridDim.x;
  int tgt = -1, kpad = 0;
  for (int64_t g = r0; g < r1; ++g) {
    int t = tgt < 0 ? 0 : tgt;
    while (g >= B.row_begin[t + 1]) ++t;
    __syncthreads();   // previous row (and column list) fully consumed
    if (t != tgt) {
      tgt = t;
      const int q = B.prob[t];
      kpad = kblocks[q] * 128;
      const uint4* src = reinterpret_cast<const uint4*>(collist + (int64_t)q * TC_KCAP);
      for (int i = threadIdx.x; i < kpad / 4; i += blockDim.x) reinterpret_cast<uint4*>(cols)[i] = src[i];
    }
    const int64_t r = g - B.row_begin[t];
    const uint4* src = reinterpret_cast<const uint4*>(B.rows[t] + r * (int64_t)stride16);
    for (int i = threadIdx.x; i < stride16 / 8; i += blockDim.x) reinterpret_cast<uint4*>(row)[i] = src[i];
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(B.out[t] + r * (int64_t)TC_KCAP);
    for (int c = threadIdx.x; c < kpad / 16; c += blockDim.x) {
      uint32_t o[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint4 e = reinterpret_cast<const uint4*>(cols)[c * 4 + w];
        const uint32_t es[4] = {e.x, e.y, e.z, e.w};
        uint32_t word = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t layer = es[k] >> 16;
          const uint32_t bitv = (layer != 0u && (uint32_t)row[es[k] & 0xffffu] >= layer) ? 1u : 0u;
          word |= bitv << (8 * k);
        }
        o[w] = word;
      }
      dst[c] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// ------------------------------------------------------------ epilogue ----
struct TcEpiProb {
  const int32_t* nkA;
  const int32_t* nkB;
  sa_key128* keyA;
  sa_key128* keyB;
  uint16_t* num;
  double* sim;
  int64_t ld;
  double delta, ln1pd;
  int32_t form;
  int32_t sym;
};

// 96-bit (lo, hi) add
__device__ __forceinline__ void add96(uint64_t& lo, uint32_t& hi, uint64_t blo, uint32_t bhi) {
  lo += blo;
  hi += bhi + ((lo < blo) ? 1u : 0u);
}

struct KeyMatEpi {
  TcEpiProb e[tc::MAXPROB];
  const uint32_t* state;

  struct State {
    uint64_t lo;
    uint32_t hi;
    int nk_r;
    int row_g;
  };

  __device__ bool skip() const { return tc_infeasible(state); }

  __device__ void begin(State& s, const tc::Tile& T, int row) const {
    const TcEpiProb& E = e[T.pi];
    s.lo = 0;
    s.hi = 0;
    s.row_g = T.row0 + row;
    s.nk_r = row < T.ra ? E.nkA[s.row_g] : -1;
  }

  __device__ void chunk(State& s, const tc::Tile& T, int row, int col, const uint32_t (&v)[32], int lane,
                        uint32_t* xpose) const {
    const TcEpiProb& E = e[T.pi];
    const bool sym = E.sym != 0;
    const int c0 = T.col0 + col;                        // global column of j = 0
    const int nk_cl = (col + lane < T.rb) ? E.nkB[c0 + lane] : -1;   // column c0 + lane
    uint32_t C[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) C[j] = (sym && c0 + j == s.row_g) ? (uint32_t)s.nk_r : v[j];

    if (E.keyA) {
      const bool colsum = sym && E.keyB;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint64_t tlo[8];
        uint32_t thi[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = g * 8 + jj;
          const int nk_c = __shfl_sync(0xffffffffu, nk_cl, j);
          const int gc = c0 + j;
          uint64_t lo = 0;
          uint32_t hi = 0;
          if (s.nk_r >= 0 && nk_c >= 0 && (!sym || gc >= s.row_g))
            key_term_f(E, lo, hi, C[j], (uint32_t)min(s.nk_r, nk_c));
          add96(s.lo, s.hi, lo, hi);
          const bool mirror = colsum && gc > s.row_g;
          tlo[jj] = mirror ? lo : 0ull;
          thi[jj] = mirror ? hi : 0u;
        }
        if (colsum) {
          // reduce the 8 column terms over the 32 rows of the warp: butterfly
          // over lane bits 4, 3, 2 (8 -> 1 value per lane), then xor 2, 1
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
          const int jc = g * 8 + ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
          if ((lane & 3) == 0 && (lo | hi) && col + jc < T.rb) atomic_add_key(E.keyB + c0 + jc, lo, hi);
        }
      }
    }

    if (E.num || E.sim) {
      // mirrored half (symmetric): lanes = consecutive rows -> coalesced columns
      if (sym) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int nk_c = __shfl_sync(0xffffffffu, nk_cl, j);
          const int gc = c0 + j;
          if (s.nk_r < 0 || nk_c < 0 || gc <= s.row_g) continue;
          const int64_t o = (int64_t)gc * E.ld + s.row_g;
          if (E.num) E.num[o] = (uint16_t)C[j];
          if (E.sim) {
            const int D = min(s.nk_r, nk_c);
            E.sim[o] = D > 0 ? __ddiv_rn((double)C[j], (double)D) : 0.0;
          }
        }
      }
      // direct half through a 32 x 32 transpose: lanes = consecutive columns
#pragma unroll
      for (int j = 0; j < 32; ++j) xpose[lane * 33 + j] = C[j];
      __syncwarp();
      const int rbase = s.row_g - lane;
      const int gc = c0 + lane;
#pragma unroll 4
      for (int i = 0; i < 32; ++i) {
        const int nk_ri = __shfl_sync(0xffffffffu, s.nk_r, i);
        const int rg = rbase + i;
        if (nk_ri < 0 || nk_cl < 0 || (sym && gc < rg)) continue;
        const uint32_t Cv = xpose[i * 33 + lane];
        const int64_t o = (int64_t)rg * E.ld + gc;
        if (E.num) E.num[o] = (uint16_t)Cv;
        if (E.sim) {
          const int D = min(nk_ri, nk_cl);
          E.sim[o] = D > 0 ? __ddiv_rn((double)Cv, (double)D) : 0.0;
        }
      }
      __syncwarp();
    }
  }

  __device__ void end(State& s, const tc::Tile& T, int row) const {
    const TcEpiProb& E = e[T.pi];
    if (E.keyA && s.nk_r >= 0 && (s.lo | s.hi)) atomic_add_key(E.keyA + s.row_g, s.lo, s.hi);
    (void)row;
  }

  __device__ static void key_term_f(const TcEpiProb& E, uint64_t& lo, uint32_t& hi, uint32_t C, uint32_t D) {
    if (E.form == SA_RANK_DF) add_dF_term(lo, hi, C, D, E.delta, E.ln1pd);
    else add_term(lo, hi, C, D);
  }
};

// ------------------------------------------------------------- host ----
static sa_status tc_encode_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int box_rows);

sa_status tc_launch(const std::vector<MsProblem>& probs_in, int ldw16, int32_t bins, uint32_t* state,
                    uint32_t* cols_out, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
  (void)bins;
  SA_TRY(ensure_recip_tables_tu(st));
  static int g_num_sms = 0;
  if (g_num_sms == 0) {
    int dev = 0;
    SA_CUDA(cudaGetDevice(&dev));
    SA_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  static bool configured = false;
  if (!configured) {
    SA_CUDA(cudaFuncSetAttribute(tc_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TC_PLANE * 4));
    SA_CUDA(cudaFuncSetAttribute(tc_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 TC_KCAP * 4 + 8192 * 2));
    SA_CUDA(cudaFuncSetAttribute(tc::gemm_kernel<KeyMatEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM));
    configured = true;
  }
  const int stride16 = 2 * ldw16;
  std::vector<MsProblem> probs;
  for (const auto& p : probs_in)
    if (p.na > 0 && p.nb > 0) probs.push_back(p);
  if (ev0) SA_CUDA(cudaEventRecord(ev0, st));
  size_t i0 = 0;
  while (i0 < probs.size()) {
    const size_t i1 = std::min(probs.size(), i0 + (size_t)tc::MAXPROB);
    const int np = (int)(i1 - i0);
    Scratch scratch(st);
    // sides and selection
    TcSides sides{};
    TcSel sel{};
    sel.n = np;
    sel.first = (int)i0;
    for (int q = 0; q < np; ++q) {
      const MsProblem& P = probs[i0 + q];
      sel.side_a[q] = sides.n;
      sides.s[sides.n++] = TcSide{reinterpret_cast<const uint16_t*>(P.A), P.na};
      if (P.sym) {
        sel.side_b[q] = -1;
      } else {
        sel.side_b[q] = sides.n;
        sides.s[sides.n++] = TcSide{reinterpret_cast<const uint16_t*>(P.B), P.nb};
      }
    }
    SA_ALLOC(planes, uint32_t, (size_t)sides.n * 2 * TC_PLANE);
    SA_ALLOC(collist, uint32_t, (size_t)np * TC_KCAP);
    SA_ALLOC(kblocks, int32_t, np);
    SA_CUDA(cudaMemsetAsync(planes, 0, (size_t)sides.n * 2 * TC_PLANE * 4, st));
    int64_t maxn = 1;
    for (int s = 0; s < sides.n; ++s) maxn = std::max(maxn, sides.s[s].n);
    const int hx = (int)std::max<int64_t>(1, std::min<int64_t>(maxn, (3 * g_num_sms + sides.n - 1) / sides.n));
    tc_hist_kernel<<<dim3(hx, sides.n), 512, 2 * TC_PLANE * 4, st>>>(sides, stride16, planes, state);
    SA_LAUNCHED();
    tc_select_kernel<<<np, 1024, 0, st>>>(sel, planes, collist, kblocks, state, cols_out);
    SA_LAUNCHED();
    // operand rows: one target per side (the side's problem's column list)
    TcBuild bl{};
    uint8_t* side_out[2 * tc::MAXPROB];
    bl.row_begin[0] = 0;
    for (int q = 0; q < np; ++q) {
      const int sa_ = sel.side_a[q], sb = sel.side_b[q];
      for (int s : {sa_, sb}) {
        if (s < 0) continue;
        uint8_t* o = scratch.alloc<uint8_t>((size_t)sides.s[s].n * TC_KCAP);
        if (!o) return fail(SA_E_NOMEM, "scratch allocation of K2T operand rows failed");
        side_out[s] = o;
        bl.rows[bl.n] = sides.s[s].rows;
        bl.out[bl.n] = o;
        bl.prob[bl.n] = q;
        bl.row_begin[bl.n + 1] = bl.row_begin[bl.n] + sides.s[s].n;
        ++bl.n;
      }
    }
    const int64_t R = bl.row_begin[bl.n];
    const int bx = (int)std::min<int64_t>(R, 2 * g_num_sms);
    tc_build_kernel<<<bx, TC_BUILD_THREADS, TC_KCAP * 4 + 8192 * 2, st>>>(bl, stride16, collist, kblocks, state);
    SA_LAUNCHED();
    // GEMM
    tc::Batch batch{};
    tc::Maps maps;
    std::memset(&maps, 0, sizeof maps);
    KeyMatEpi epi{};
    epi.state = state;
    int64_t tiles = 0;
    for (int q = 0; q < np; ++q) {
      const MsProblem& P = probs[i0 + q];
      tc::Problem& T = batch.p[q];
      T.na = P.na;
      T.nb = P.nb;
      T.sym = P.sym;
      T.tiles_n = (P.nb + tc::BN - 1) / tc::BN;
      T.tile_begin = tiles;
      T.kblocks = kblocks + q;
      T.map = q;
      tiles += tc::problem_tiles(P.na, P.nb, P.sym != 0);
      const uint8_t* a = side_out[sel.side_a[q]];
      const uint8_t* b = P.sym ? a : side_out[sel.side_b[q]];
      SA_TRY(tc_encode_map(&maps.m[2 * q], a, P.na, tc::BM));
      SA_TRY(tc_encode_map(&maps.m[2 * q + 1], b, P.nb, tc::BN));
      TcEpiProb& E = epi.e[q];
      E.nkA = P.nkA;
      E.nkB = P.nkB;
      E.keyA = P.keyA;
      E.keyB = P.sym ? P.keyB : nullptr;
      E.num = P.num;
      E.sim = P.sim;
      E.ld = P.ld;
      E.form = P.form;
      E.delta = P.delta;
      E.ln1pd = P.ln1pd;
      E.sym = P.sym;
    }
    batch.n = np;
    const int64_t grid = tiles < g_num_sms ? tiles : g_num_sms;
    tc::gemm_kernel<KeyMatEpi><<<(unsigned)grid, tc::THREADS, tc::SMEM, st>>>(batch, maps, tiles, epi);
    SA_LAUNCHED();
    i0 = i1;
  }
  if (ev1) SA_CUDA(cudaEventRecord(ev1, st));
  return SA_OK;
}

static sa_status tc_encode_map(CUtensorMap* m, const uint8_t* base, int64_t rows, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)TC_KCAP, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)TC_KCAP};
  const cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled (K2T) failed (%d)", (int)r);
  return SA_OK;
}

}  // namespace sa
