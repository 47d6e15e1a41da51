// K2 -- the dense min-sum engine: C_ij = sum_t min(c^i_t, c^j_t), the numerator
// of Eq. 1, for every pair of a tile, with fused
// epilogues:
//   * exact-rank keys  key_i += floor(C_ij 2^64 / D_ij)  (S2a, S2d; Eq. 3 in
//     F form, readings Z1/Z10/Z11) -- row sums, plus column sums on
//     symmetric off-diagonal tiles;
//   * numerators C_ij (uint16) and F_ij = C_ij / D_ij in fp64 (S5),
//     mirrored for symmetric problems.
//
// Design: profiles are uint16 counts packed two bins per 32-bit
// word; one `min.u16x2` (SASS VIMNMX.U16x2) takes the min of two bins and one
// three-input add (IADD3) folds two of those into the packed accumulator.  The
// per-lane u16 sums cannot carry: each lane's sum <= C <= min(nk) <= 65535.
// A CTA owns a 128 x 128 pair tile; each of its 256 threads keeps an 8 x 8
// register block of packed accumulators and reads 8 + 8 rows with LDS.128
// (4 words = 8 bins per load), i.e. 16 loads per 256 VIMNMX.  Rows are staged
// 32 words (64 bins) at a time through a 4-stage cp.async ring with a padded
// row stride (36 words) that makes every LDS.128 conflict-free.  The grid is
// persistent: one CTA per SM strides over a flat list of tiles of up to 16
// problems (all local blocks of S2a, all buckets of S5).
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "keyterm.cuh"

namespace sa {

sa_status ensure_recip_tables(cudaStream_t st) { return ensure_recip_tables_tu(st); }

constexpr int MS_MAXPROB = 16;
struct MsBatch {
  MsProblem p[MS_MAXPROB];
  int n;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void key_term(const MsProblem& P, uint64_t& lo, uint32_t& hi, uint32_t C, uint32_t D) {
  if (P.form == SA_RANK_DF) add_dF_term(lo, hi, C, D, P.delta, P.ln1pd);
  else add_term(lo, hi, C, D);
}

// acc += sum over the 4 byte lanes of |a - b|  (one VABSDIFF4.U8.ACC)
__device__ __forceinline__ void vsad4_acc(uint32_t& acc, uint32_t a, uint32_t b) {
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(acc) : "r"(a), "r"(b));
}

// Numerator of one pair from its accumulator (see the ENC_* encodings).
template <int ENC>
__device__ __forceinline__ uint32_t acc_to_C(uint32_t acc, int nka, int nkb) {
  if (ENC == ENC_U8_SAD) return (uint32_t)(nka + nkb - (int)acc) >> 1;   // sum min = (sum a + sum b - sum|a-b|)/2
  return (acc & 0xffffu) + (acc >> 16);                                  // the two u16 lanes
}

// Device-side engine dispatch: both encodings are enqueued and each kernel
// returns at once unless the largest count (*guard, written by to_u8_kernel)
// selects it -- u8 SAD when every count is <= 255, u16 otherwise -- so the
// host never waits for the decision.
// guard[0] = largest count, guard[1] = the tensor-core engine (K2T) found the
// launch infeasible, guard[2] = K2T enabled for this call: when K2T ran, these
// engines return at once.
__device__ __forceinline__ bool tc_handled(const uint32_t* guard) {
  const volatile uint32_t* g = guard;
  return g[2] != 0u && g[1] == 0u;
}
template <int ENC>
__device__ __forceinline__ bool guard_skip(const uint32_t* guard) {
  if (!guard) return false;
  if (tc_handled(guard)) return true;
  const uint32_t m = *reinterpret_cast<const volatile uint32_t*>(guard);
  return (m <= 255u) != (ENC == ENC_U8_SAD);
}

template <int FW>
__device__ __forceinline__ void load_frag(uint32_t (&f)[FW], const uint32_t* p) {
  if constexpr (FW == 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
  } else {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    f[0] = v.x; f[1] = v.y;
  }
}

// One smem stage of the uint8 SAD engine with FW-word fragments (FW = 4: one
// LDS.128 = 16 bins per row; FW = 2: LDS.64 = 8 bins) and an UNR-way
// unrolled k loop.  The w-outer order puts 64 independent accumulators
// between two updates of the same one.
template <int FW, int UNR>
__device__ __forceinline__ void sad_stage(const uint32_t* __restrict__ As, const uint32_t* __restrict__ Bs, int ty,
                                          int tx, uint32_t (&acc)[8][8]) {
#pragma unroll UNR
  for (int kq = 0; kq < MS_BKW / FW; ++kq) {
    uint32_t a[8][FW], b[8][FW];
#pragma unroll
    for (int i = 0; i < 8; ++i) load_frag<FW>(a[i], As + (ty + 16 * i) * MS_LDW + kq * FW);
#pragma unroll
    for (int j = 0; j < 8; ++j) load_frag<FW>(b[j], Bs + (tx + 16 * j) * MS_LDW + kq * FW);
#pragma unroll
    for (int w = 0; w < FW; ++w)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) vsad4_acc(acc[i][j], a[i][w], b[j][w]);
  }
}

template <int ENC>
__device__ __forceinline__ void compute_stage_u4(const uint32_t* __restrict__ As, const uint32_t* __restrict__ Bs,
                                                 int ty, int tx, uint32_t (&acc)[8][8], uint32_t one);

// One smem stage (MS_BKW words of 128 A rows and 128 B rows) into the 8 x 8
// register block of packed accumulators.
template <int ENC, int VAR>
__device__ __forceinline__ void compute_stage(const uint32_t* __restrict__ As, const uint32_t* __restrict__ Bs,
                                              int ty, int tx, uint32_t (&acc)[8][8], uint32_t one) {
  if constexpr (ENC == ENC_U8_SAD && VAR != 0) {
    sad_stage<(VAR == 1 ? 4 : 2), (VAR == 3 ? 1 : 2)>(As, Bs, ty, tx, acc);
  } else {
    compute_stage_u4<ENC>(As, Bs, ty, tx, acc, one);
  }
}

template <int ENC>
__device__ __forceinline__ void compute_stage_u4(const uint32_t* __restrict__ As, const uint32_t* __restrict__ Bs,
                                                 int ty, int tx, uint32_t (&acc)[8][8], uint32_t one) {
#pragma unroll
  for (int kq = 0; kq < MS_BKW / 4; ++kq) {
    uint4 a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const uint4*>(As + (ty + 16 * i) * MS_LDW + kq * 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const uint4*>(Bs + (tx + 16 * j) * MS_LDW + kq * 4);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (ENC == ENC_U8_SAD) {
          // 16 bins: four VABSDIFF4.U8.ACC, |a-b| of 4 byte lanes summed into acc
          vsad4_acc(acc[i][j], a[i].x, b[j].x);
          vsad4_acc(acc[i][j], a[i].y, b[j].y);
          vsad4_acc(acc[i][j], a[i].z, b[j].z);
          vsad4_acc(acc[i][j], a[i].w, b[j].w);
        } else if constexpr (ENC == ENC_U16_MIN_IMAD) {
          // 8 bins: four VIMNMX.U16x2 (ALU pipe), adds as IMAD on the FMA pipe
          uint32_t m0 = __vminu2(a[i].x, b[j].x), m1 = __vminu2(a[i].y, b[j].y);
          uint32_t m2 = __vminu2(a[i].z, b[j].z), m3 = __vminu2(a[i].w, b[j].w);
          asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i][j]) : "r"(m0), "r"(one));
          asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i][j]) : "r"(m1), "r"(one));
          asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i][j]) : "r"(m2), "r"(one));
          asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i][j]) : "r"(m3), "r"(one));
        } else {
          // 8 bins: four VIMNMX.U16x2 + two IADD3
          acc[i][j] += __vminu2(a[i].x, b[j].x) + __vminu2(a[i].y, b[j].y);
          acc[i][j] += __vminu2(a[i].z, b[j].z) + __vminu2(a[i].w, b[j].w);
        }
      }
  }
}

struct TileInfo {
  int pi, ti, tj, row0, col0, ra, rb;
};

template <bool SYM>
__device__ __forceinline__ TileInfo decode_tile(const MsBatch& batch, int64_t tile) {
  TileInfo T;
  int pi = 0;
  while (pi + 1 < batch.n && batch.p[pi + 1].tile_begin <= tile) ++pi;
  const MsProblem& P = batch.p[pi];
  int64_t t = tile - P.tile_begin;
  if (SYM) {
    const int nt = P.tiles_b;
    int ti = 0;
    while (t >= nt - ti) { t -= nt - ti; ++ti; }
    T.ti = ti;
    T.tj = ti + (int)t;
  } else {
    T.ti = (int)(t / P.tiles_b);
    T.tj = (int)(t % P.tiles_b);
  }
  T.pi = pi;
  T.row0 = T.ti * MS_BM;
  T.col0 = T.tj * MS_BM;
  T.ra = min(MS_BM, P.na - T.row0);
  T.rb = min(MS_BM, P.nb - T.col0);
  return T;
}

// Fused epilogue of one tile: exact-rank keys and / or the C, F matrices.
template <bool SYM, int ENC, int TN = 8>
__device__ __forceinline__ void tile_epilogue(const MsProblem& P, const TileInfo& T, int ty, int tx, int lane,
                                              const uint32_t (&acc)[8][TN]) {
  constexpr int CS = MS_BM / TN;   // column stride of a thread's TN columns
  const bool offdiag = SYM && (T.ti != T.tj);
  const int row0 = T.row0, col0 = T.col0;
  int nkr[8], nkc[TN];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = ty + 16 * i;
    nkr[i] = (r < T.ra) ? P.nkA[row0 + r] : -1;
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const int c = tx + CS * j;
    nkc[j] = (c < T.rb) ? P.nkB[col0 + c] : -1;
  }
  if (P.keyA) {
    // row sums: key_i += sum_j floor(C_ij 2^64 / D_ij)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint64_t lo = 0;
      uint32_t hi = 0;
      if (nkr[i] >= 0) {
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          if (nkc[j] < 0) continue;
          const uint32_t C = acc_to_C<ENC>(acc[i][j], nkr[i], nkc[j]);
          key_term(P, lo, hi, C, (uint32_t)min(nkr[i], nkc[j]));
        }
      }
      shfl_add(lo, hi, 1);
      shfl_add(lo, hi, 2);
      shfl_add(lo, hi, 4);
      if ((lane & 7) == 0 && nkr[i] >= 0 && (lo | hi)) atomic_add_key(P.keyA + row0 + ty + 16 * i, lo, hi);
    }
    if (offdiag && P.keyB) {
      // column sums: the mirrored pairs (j, i) of an off-diagonal tile
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        uint64_t lo = 0;
        uint32_t hi = 0;
        if (nkc[j] >= 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (nkr[i] < 0) continue;
            const uint32_t C = acc_to_C<ENC>(acc[i][j], nkr[i], nkc[j]);
            key_term(P, lo, hi, C, (uint32_t)min(nkr[i], nkc[j]));
          }
        }
        shfl_add(lo, hi, 8);
        shfl_add(lo, hi, 16);
        if (lane < 8 && nkc[j] >= 0 && (lo | hi)) atomic_add_key(P.keyB + col0 + tx + CS * j, lo, hi);
      }
    }
  }
  if (P.num || P.sim) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (nkr[i] < 0) continue;
      const int64_t gr = row0 + ty + 16 * i;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        if (nkc[j] < 0) continue;
        const int64_t gc = col0 + tx + CS * j;
        const uint32_t C = acc_to_C<ENC>(acc[i][j], nkr[i], nkc[j]);
        const int D = min(nkr[i], nkc[j]);
        if (P.num) {
          P.num[gr * P.ld + gc] = (uint16_t)C;
          if (offdiag) P.num[gc * P.ld + gr] = (uint16_t)C;
        }
        if (P.sim) {
          const double F = D > 0 ? __ddiv_rn((double)C, (double)D) : 0.0;
          P.sim[gr * P.ld + gc] = F;
          if (offdiag) P.sim[gc * P.ld + gr] = F;
        }
      }
    }
  }
}

// ---------------------------------------------- engine A: cp.async ring ---
// Every thread copies 8 x 16 B per stage; a CTA-wide barrier per stage.
template <bool SYM, int ENC, int VAR>
__global__ void __launch_bounds__(MS_THREADS, 1)
minsum_kernel(const __grid_constant__ MsBatch batch, int64_t total_tiles, int ldw, uint32_t one,
              const uint32_t* __restrict__ guard) {
  if (guard_skip<ENC>(guard)) return;
  extern __shared__ __align__(16) uint32_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);  // row group 0..15: rows ty + 16 i
  const int tx = (warp & 1) * 8 + (lane & 7);     // col group 0..15: cols tx + 16 j
  const int nK = ldw / MS_BKW;
  constexpr int STAGE_W = 2 * MS_BM * MS_LDW;

  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const TileInfo T = decode_tile<SYM>(batch, tile);
    const MsProblem& P = batch.p[T.pi];
    const uint32_t* Ag = P.A + (int64_t)T.row0 * ldw;
    const uint32_t* Bg = P.B + (int64_t)T.col0 * ldw;

    auto load = [&](int stage, int kc) {
      uint32_t* sb = smem + stage * STAGE_W;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = tid + MS_THREADS * u;
        const int r = c >> 3, ch = c & 7;
        const bool isA = r < MS_BM;
        const int rr = isA ? r : r - MS_BM;
        const bool valid = rr < (isA ? T.ra : T.rb);
        const uint32_t* g = (isA ? Ag : Bg) + (int64_t)(valid ? rr : 0) * ldw + kc * MS_BKW + ch * 4;
        cp_async16(smem_u32(sb + r * MS_LDW + ch * 4), g, valid ? 16 : 0);
      }
    };

    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0u;

#pragma unroll
    for (int s = 0; s < MS_STAGES - 1; ++s) {
      if (s < nK) load(s, s);
      cp_commit();
    }
    for (int kc = 0; kc < nK; ++kc) {
      cp_wait<MS_STAGES - 2>();
      __syncthreads();
      {
        const int nxt = kc + MS_STAGES - 1;
        if (nxt < nK) load(nxt % MS_STAGES, nxt);
        cp_commit();
      }
      const uint32_t* As = smem + (kc % MS_STAGES) * STAGE_W;
      compute_stage<ENC, VAR>(As, As + MS_BM * MS_LDW, ty, tx, acc, one);
    }
    __syncthreads();   // smem is reloaded by the next tile
    tile_epilogue<SYM, ENC>(P, T, ty, tx, lane, acc);
  }
}

// ------------------------------------------- engine B: TMA + mbarrier ring --
// One elected thread (warp 0, lane 0) streams the 128-row A and B boxes of
// every stage of every tile of this CTA with two TMA tensor loads
// (cp.async.bulk.tensor.2d, SWIZZLE_128B, rows past the end zero-filled by
// the TMA unit), MS_TMA_STAGES - 2 stages ahead and across tile boundaries
// (the next tile's first stages land during this tile's epilogue).  Each warp
// waits on the stage's "full" mbarrier (TMA transaction count) and releases
// it on the stage's "empty" mbarrier: no CTA-wide barrier in the main loop.
// The 128-byte swizzle replaces the padded rows of engine A: reading 16-byte
// chunk c of row r at chunk position c ^ (r & 7) keeps every fragment load
// bank-conflict-free.
constexpr int MS_TMA_STAGES = 6;
constexpr int MS_TMA_ROW_W = MS_BKW;                       // 32 words = 128 B per row per stage
constexpr int MS_TMA_STAGE_W = 2 * MS_BM * MS_TMA_ROW_W;   // 8192 words = 32 KB
constexpr int MS_TMA_SMEM = MS_TMA_STAGES * MS_TMA_STAGE_W * 4 + 1024 + 2 * MS_TMA_STAGES * 8;

struct alignas(64) MsMaps {
  CUtensorMap m[2 * MS_MAXPROB];   // problem p: m[2p] = A rows, m[2p+1] = B rows
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// word pointer of 16-byte chunk c of row r in a SWIZZLE_128B box of 128-byte rows
__device__ __forceinline__ const uint32_t* swz(const uint32_t* base, int r, int c) {
  return base + r * MS_TMA_ROW_W + ((c ^ (r & 7)) << 2);
}

template <int ENC, int FW, int TN>
__device__ __forceinline__ void compute_stage_swz(const uint32_t* __restrict__ As, const uint32_t* __restrict__ Bs,
                                                  int ty, int tx, uint32_t (&acc)[8][TN], uint32_t one) {
  constexpr int CS = MS_BM / TN;
#pragma unroll
  for (int kq = 0; kq < MS_BKW / FW; ++kq) {
    const int o = kq * FW;
    uint32_t a[8][FW], b[TN][FW];
#pragma unroll
    for (int i = 0; i < 8; ++i) load_frag<FW>(a[i], swz(As, ty + 16 * i, o >> 2) + (o & 3));
#pragma unroll
    for (int j = 0; j < TN; ++j) load_frag<FW>(b[j], swz(Bs, tx + CS * j, o >> 2) + (o & 3));
    if constexpr (ENC == ENC_U8_SAD) {
#pragma unroll
      for (int w = 0; w < FW; ++w)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) vsad4_acc(acc[i][j], a[i][w], b[j][w]);
    } else {
#pragma unroll
      for (int w = 0; w < FW; w += 2)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            const uint32_t m0 = __vminu2(a[i][w], b[j][w]), m1 = __vminu2(a[i][w + 1], b[j][w + 1]);
            if constexpr (ENC == ENC_U16_MIN_IMAD) {
              asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i][j]) : "r"(m0), "r"(one));
              asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc[i][j]) : "r"(m1), "r"(one));
            } else {
              acc[i][j] += m0 + m1;
            }
          }
    }
  }
}

// TN = columns per thread: 8 -> 256 threads (8 warps, 8 x 8 blocks); 4 -> 512
// threads (16 warps, 8 x 4 blocks, <= 128 registers: twice the warps per
// scheduler to hide latency, 12 LDS.128 per 128 VABSDIFF4 instead of 16 per 256).
template <int TN>
__host__ __device__ constexpr int tma_threads() { return 16 * (MS_BM / TN); }

template <bool SYM, int ENC, int VAR, int TN>
__global__ void __launch_bounds__(tma_threads<TN>(), 1)
minsum_tma_kernel(const __grid_constant__ MsBatch batch, const __grid_constant__ MsMaps maps, int64_t total_tiles,
                  int ldw, uint32_t one, const uint32_t* __restrict__ guard) {
  if (guard_skip<ENC>(guard)) return;
  constexpr int NT = tma_threads<TN>();
  constexpr int WPR = (MS_BM / TN) / 8;     // warps per row group
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t base_s = (smem_u32(smem_raw) + 1023u) & ~1023u;     // SWIZZLE_128B wants 1 KB alignment
  uint32_t* smem = reinterpret_cast<uint32_t*>(smem_raw + (base_s - smem_u32(smem_raw)));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + MS_TMA_STAGES * MS_TMA_STAGE_W);
  uint64_t* empty = full + MS_TMA_STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ty = (warp / WPR) * 4 + (lane >> 3);
  const int tx = (warp % WPR) * 8 + (lane & 7);
  const int nK = ldw / MS_BKW;
  if (tid == 0) {
    for (int s = 0; s < MS_TMA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t my_tiles = total_tiles > blockIdx.x ? (total_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nstages = my_tiles * nK;
  const bool producer = (tid == 0);
  int64_t g_load = 0, ld_tile = blockIdx.x;
  int ld_kc = 0;
  TileInfo LT{};
  if (producer && my_tiles) LT = decode_tile<SYM>(batch, ld_tile);
  auto produce = [&]() {   // one thread: stage g_load into slot g_load % S
    const int slot = (int)(g_load % MS_TMA_STAGES);
    if (g_load >= MS_TMA_STAGES) mbar_wait(&empty[slot], (uint32_t)(((g_load / MS_TMA_STAGES) - 1) & 1));
    mbar_arrive_tx(&full[slot], MS_TMA_STAGE_W * 4);
    const uint32_t dst = smem_u32(smem + slot * MS_TMA_STAGE_W);
    tma_load_2d(dst, &maps.m[2 * LT.pi], ld_kc * MS_BKW, LT.row0, &full[slot]);
    tma_load_2d(dst + MS_BM * MS_TMA_ROW_W * 4, &maps.m[2 * LT.pi + 1], ld_kc * MS_BKW, LT.col0, &full[slot]);
    ++g_load;
    if (++ld_kc == nK) {
      ld_kc = 0;
      ld_tile += gridDim.x;
      if (ld_tile < total_tiles) LT = decode_tile<SYM>(batch, ld_tile);
    }
  };
  if (producer)
    while (g_load < nstages && g_load < MS_TMA_STAGES - 2) produce();

  int64_t g_use = 0;
  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const TileInfo T = decode_tile<SYM>(batch, tile);
    const MsProblem& P = batch.p[T.pi];
    uint32_t acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0u;
    for (int kc = 0; kc < nK; ++kc, ++g_use) {
      if (producer && g_load < nstages) produce();
      const int slot = (int)(g_use % MS_TMA_STAGES);
      mbar_wait(&full[slot], (uint32_t)((g_use / MS_TMA_STAGES) & 1));
      const uint32_t* As = smem + slot * MS_TMA_STAGE_W;
      compute_stage_swz<ENC, (ENC == ENC_U8_SAD && VAR >= 2) ? 2 : 4, TN>(As, As + MS_BM * MS_TMA_ROW_W, ty, tx,
                                                                           acc, one);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    tile_epilogue<SYM, ENC, TN>(P, T, ty, tx, lane, acc);
  }
}

// Pipeline of the engine (SA_K2_PIPE): "tma" (default) = TMA tensor loads +
// mbarrier ring (engine B), "cpasync" = per-thread cp.async + CTA barrier per
// stage (engine A).
static bool use_tma_pipe() {
  const char* e = getenv("SA_K2_PIPE");
  return !(e && !strcmp(e, "cpasync"));
}

// Thread layout of engine B (SA_K2_LAYOUT): 4 = 512 threads x 8x4 (default), 8 = 256 threads x 8x8.
static int tma_layout() {
  const char* e = getenv("SA_K2_LAYOUT");
  return (e && atoi(e) == 8) ? 8 : 4;
}

// 2-D map over `rows` rows of ldw 32-bit words: boxes of 32 words x 128 rows,
// 128-byte swizzle, rows past the end read as zeros.
static sa_status encode_rows_map(CUtensorMap* m, const uint32_t* base, int64_t rows, int ldw) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)ldw, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ldw * 4};
  const cuuint32_t box[2] = {(cuuint32_t)MS_BKW, (cuuint32_t)MS_BM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SA_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SA_OK;
}

template <bool SYM, int ENC, int VAR>
static sa_status launch_one(const MsBatch& b, int64_t tiles, int ldw, const uint32_t* guard, cudaStream_t st) {
  static DeviceOnce once;
  SA_TRY(once.run([]() -> sa_status {
    SA_CUDA(cudaFuncSetAttribute(minsum_kernel<SYM, ENC, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, MS_SMEM));
    SA_CUDA(cudaFuncSetAttribute(minsum_tma_kernel<SYM, ENC, VAR, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 MS_TMA_SMEM));
    SA_CUDA(cudaFuncSetAttribute(minsum_tma_kernel<SYM, ENC, VAR, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 MS_TMA_SMEM));
    return SA_OK;
  }));
  const int g_num_sms = device_sms();
  const int64_t grid = tiles < g_num_sms ? tiles : g_num_sms;
  if (use_tma_pipe()) {
    MsMaps maps;
    std::memset(&maps, 0, sizeof maps);
    for (int p = 0; p < b.n; ++p) {
      SA_TRY(encode_rows_map(&maps.m[2 * p], b.p[p].A, b.p[p].na, ldw));
      SA_TRY(encode_rows_map(&maps.m[2 * p + 1], b.p[p].B, b.p[p].nb, ldw));
    }
    if (tma_layout() == 4)
      minsum_tma_kernel<SYM, ENC, VAR, 4><<<(unsigned)grid, tma_threads<4>(), MS_TMA_SMEM, st>>>(b, maps, tiles, ldw,
                                                                                                1u, guard);
    else
      minsum_tma_kernel<SYM, ENC, VAR, 8><<<(unsigned)grid, tma_threads<8>(), MS_TMA_SMEM, st>>>(b, maps, tiles, ldw,
                                                                                                1u, guard);
  } else {
    minsum_kernel<SYM, ENC, VAR><<<(unsigned)grid, MS_THREADS, MS_SMEM, st>>>(b, tiles, ldw, 1u, guard);
  }
  SA_LAUNCHED();
  return SA_OK;
}

// SAD-engine inner-loop variant (SA_K2_VARIANT, default 0): 0 = uint4
// fragments, fully unrolled stage; 1 = uint4, 2-way unroll; 2 = uint2, 2-way;
// 3 = uint2, no unroll.
static int sad_variant() {
  const char* e = getenv("SA_K2_VARIANT");
  const int v = e ? atoi(e) : 0;
  return (v >= 0 && v <= 3) ? v : 0;
}

template <bool SYM>
static sa_status launch_enc(const MsBatch& b, int64_t tiles, int ldw, int enc, const uint32_t* guard,
                            cudaStream_t st) {
  if (enc == ENC_U8_SAD) {
    switch (sad_variant()) {
      case 1: return launch_one<SYM, ENC_U8_SAD, 1>(b, tiles, ldw, guard, st);
      case 2: return launch_one<SYM, ENC_U8_SAD, 2>(b, tiles, ldw, guard, st);
      case 3: return launch_one<SYM, ENC_U8_SAD, 3>(b, tiles, ldw, guard, st);
      default: return launch_one<SYM, ENC_U8_SAD, 0>(b, tiles, ldw, guard, st);
    }
  }
  if (enc == ENC_U16_MIN_IMAD) return launch_one<SYM, ENC_U16_MIN_IMAD, 0>(b, tiles, ldw, guard, st);
  return launch_one<SYM, ENC_U16_MIN, 0>(b, tiles, ldw, guard, st);
}

sa_status minsum_launch(const std::vector<MsProblem>& probs_in, int ldw, int enc, cudaStream_t st,
                        cudaEvent_t ev0, cudaEvent_t ev1, const uint32_t* guard) {
  if (ldw % MS_BKW != 0) return fail(SA_E_INVAL, "profile row stride must be a multiple of 64 bins");
  SA_TRY(ensure_recip_tables(st));
  // split into batches of at most MS_MAXPROB problems of the same symmetry
  std::vector<MsProblem> probs;
  for (const auto& p : probs_in)
    if (p.na > 0 && p.nb > 0) probs.push_back(p);
  if (ev0) SA_CUDA(cudaEventRecord(ev0, st));
  size_t i = 0;
  while (i < probs.size()) {
    MsBatch b{};
    b.n = 0;
    const int sym = probs[i].sym;
    int64_t tiles = 0;
    while (i < probs.size() && b.n < MS_MAXPROB && probs[i].sym == sym) {
      MsProblem q = probs[i++];
      q.tiles_b = (q.nb + MS_BM - 1) / MS_BM;
      const int64_t ta = (q.na + MS_BM - 1) / MS_BM;
      q.tile_begin = tiles;
      tiles += sym ? (int64_t)q.tiles_b * (q.tiles_b + 1) / 2 : ta * q.tiles_b;
      b.p[b.n++] = q;
    }
    const sa_status rs = sym ? launch_enc<true>(b, tiles, ldw, enc, guard, st)
                             : launch_enc<false>(b, tiles, ldw, enc, guard, st);
    if (rs != SA_OK) return rs;
  }
  if (ev1) SA_CUDA(cudaEventRecord(ev1, st));
  return SA_OK;
}

// ------------------------------------------------- u16 -> u8 operand rows --
// The SAD encoding needs every count <= 255; the conversion saturates and
// reports the largest count so the caller can fall back to the u16 engine.
__global__ void to_u8_kernel(const uint16_t* __restrict__ p16, int64_t n, int stride16, uint8_t* __restrict__ p8,
                             int stride8, uint32_t* __restrict__ maxc, bool guarded) {
  if (guarded && tc_handled(maxc)) return;   // maxc = the guard words (K2T ran: rows unused)
  const int chunks = stride8 / 8;
  uint32_t mx = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * chunks;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / chunks;
    const int t0 = (int)(idx % chunks) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t0 < stride16) v = *reinterpret_cast<const uint4*>(p16 + row * stride16 + t0);
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t out[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t lo = w[q] & 0xffffu, hi = w[q] >> 16;
      mx = max(mx, max(lo, hi));
      const uint32_t b = min(lo, 255u) | (min(hi, 255u) << 8);
      out[q >> 1] |= b << (16 * (q & 1));
    }
    *reinterpret_cast<uint2*>(p8 + row * stride8 + t0) = make_uint2(out[0], out[1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxc, mx);
}

sa_status to_u8_launch(const uint16_t* p16, int64_t n, int32_t stride16, int32_t bins, uint8_t* p8, int32_t stride8,
                       uint32_t* maxc, cudaStream_t st, bool guarded) {
  (void)bins;
  if (n <= 0) return SA_OK;
  const int64_t work = n * (stride8 / 8);
  const int64_t blocks = (work + 255) / 256;
  // a guarded conversion (the K2T fallback's rows) usually returns at once:
  // a small grid keeps that cheap (it strides over the rows when it does run)
  const int64_t cap = guarded ? 148 * 2 : 148 * 16;
  to_u8_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, st>>>(p16, n, stride16, p8, stride8, maxc, guarded);
  SA_LAUNCHED();
  return SA_OK;
}

// --------------------------------------------------------- keys -> fp64 --
__host__ __device__ inline double u128_to_double(uint64_t hi, uint64_t lo) {
  if (hi == 0) {
#ifdef __CUDA_ARCH__
    return __ull2double_rn(lo);
#else
    return (double)lo;
#endif
  }
#ifdef __CUDA_ARCH__
  const int s = 64 - __clzll((long long)hi);
#else
  const int s = 64 - __builtin_clzll(hi);
#endif
  uint64_t m, rest;
  if (s == 64) { m = hi; rest = lo; }
  else { m = (hi << (64 - s)) | (lo >> s); rest = lo & ((1ull << s) - 1); }
  m |= (rest != 0) ? 1ull : 0ull;   // sticky bit below the rounding position
#ifdef __CUDA_ARCH__
  return ldexp(__ull2double_rn(m), s);
#else
  return ldexp((double)m, s);
#endif
}

double u128_to_double_host(uint64_t hi, uint64_t lo) { return u128_to_double(hi, lo); }

__global__ void keys_to_f64_kernel(const sa_key128* __restrict__ keys, int64_t n, int form, double ln1pd,
                                   int64_t npool, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (form == SA_RANK_DF) {
      const double v = ldexp(u128_to_double(keys[i].hi, keys[i].lo), -52);
      out[i] = __ddiv_rn(v, (double)npool) - ln1pd;
    } else {
      const double v = ldexp(u128_to_double(keys[i].hi, keys[i].lo), -64);
      out[i] = __ddiv_rn(v, (double)npool);
    }
  }
}

sa_status keys_to_f64_launch(const sa_key128* keys, int64_t n, int64_t npool, double* out, cudaStream_t st,
                             int form, double ln1pd) {
  if (n <= 0) return SA_OK;
  const int64_t blocks = (n + 255) / 256;
  keys_to_f64_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(keys, n, form, ln1pd, npool, out);
  SA_LAUNCHED();
  return SA_OK;
}

}  // namespace sa

