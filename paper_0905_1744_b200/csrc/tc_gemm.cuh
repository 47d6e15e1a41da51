// K2T -- the tensor-core form of the min-sum engine (SURVEY.md §8(f) N3(iii),
// DESIGN.md §4b): Eq. 1's numerator C_ij = sum_t min(c^i_t, c^j_t)
// written as an exact 0/1 contraction over threshold
// layers,
//     min(a, b) = sum_{r >= 1} [a >= r] [b >= r],
// so C = A' B'^T with A'[i][(r, t)] = [c^i_t >= r] -- a dense u8 GEMM with s32
// accumulators (tcgen05.mma kind::i8).  Sums are integers < 2^31: exact.
//
// This header holds the device side shared by libsa (minsum_tc.cu) and the
// standalone descriptor probe (tools/tc_probe.cu): PTX wrappers, the tile
// schedule and the warp-specialised persistent kernel.  The epilogue is a
// template parameter.
//
// Kernel anatomy (one CTA per SM, 320 threads):
//   warp 8  lane 0: TMA producer -- per stage one 128-row x 128-byte box of A
//                   and one 256-row x 128-byte box of B (SWIZZLE_128B), into a
//                   4-stage ring guarded by full/empty mbarriers;
//   warp 9  lane 0: MMA issuer -- 4 x tcgen05.mma.cta_group::1.kind::i8
//                   (M=128, N=256, K=32) per stage into one of two TMEM
//                   accumulators (2 x 256 columns), tcgen05.commit frees the
//                   stage / publishes the accumulator;
//   warps 0-7:      epilogue -- warp w reads TMEM lanes 32(w%4).. (tile rows)
//                   and columns 128(w/4).. with tcgen05.ld.32x32b.x32, calls
//                   Epi::chunk for every 32 columns, then releases the buffer.
#pragma once
#include <cuda.h>
#include <cstdint>

namespace sa {
namespace tc {

constexpr int BM = 128;          // tile rows (UMMA M)
constexpr int BK = 128;          // bytes of K per stage (128 u8 columns, or 256 packed fp4 columns)
constexpr int UKB = 32;          // bytes of K per tcgen05.mma (kind::i8: K = 32; kind::mxf4: K = 64)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;
constexpr int TMEM_COLS = 512;
// Operand format: u8 0/1 columns (kind::i8, s32 accumulators, 128 x 256
// tiles) or packed e2m1 0/1.0 columns (kind::mxf4, block32 UE8M0 scale factors
// all 1.0, f32 accumulators -- exact: sums <= 32768 < 2^24 -- twice the MMA
// rate; 128 x 240 tiles so that two accumulators leave 32 TMEM columns for the
// scale factors).
template <bool FP4>
struct Geo {
  static constexpr int BN = FP4 ? 240 : 256;               // tile columns (UMMA N)
  static constexpr int B_BYTES = BN * BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;    // multiple of 1024 (SWIZZLE_128B atoms)
  static constexpr int SF_COL = 2 * BN;                    // first scale-factor TMEM column (FP4)
  static constexpr int COLS_PER_KB = FP4 ? 256 : 128;      // operand columns per 128-byte K block
};
static_assert(Geo<true>::STAGE_BYTES % 1024 == 0 && Geo<false>::STAGE_BYTES % 1024 == 0, "stage alignment");
// Epilogue geometry (template parameters of gemm_kernel): EW epilogue warps
// (a multiple of 4: warp w reads TMEM lanes 32 (w % 4) .. and the w / 4-th
// column slice of SLICE columns), CW columns per tcgen05.ld chunk (16 or 32).
// Each epilogue warp owns TB bytes of shared memory per slice column
// (Epi::TAB_BYTES: the per-tile column tables the epilogue stages before the
// accumulator is ready) plus XB scratch bytes (Epi::xpose_bytes(CW, FP4, CG)).
__host__ __device__ constexpr int threads_of(int EW) { return (EW + 2) * 32; }
__host__ __device__ constexpr int slice_of(int EW, int CW, bool FP4) {
  return (((FP4 ? 240 : 256) / (EW / 4) + CW - 1) / CW) * CW;
}
__host__ __device__ constexpr int smem_of(int EW, int CW, bool FP4, int TB, int XB) {
  return STAGES * (FP4 ? Geo<true>::STAGE_BYTES : Geo<false>::STAGE_BYTES) + 1024 + 256 +
         EW * (slice_of(EW, CW, FP4) * TB + XB);
}
constexpr int MAXPROB = 16;

// ----------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t s_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_addr(bar)), "r"(count));
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_addr(bar)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TC_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TC_WAIT_%=;\n"
      "}\n" ::"r"(s_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(s_addr(bar))
      : "memory");
}
// the same with an L2 eviction-priority policy (createpolicy): operand rows are
// re-read by many tiles, the output matrices stream past them
__device__ __forceinline__ void tma_2d_hint(uint32_t dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(s_addr(bar)), "l"(policy)
      : "memory");
}
// TMA tensor store shared -> global (bulk-group completion) and its fences
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
// ... with an L2 cache-eviction policy (createpolicy) on the written lines
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, uint32_t src, int x, int y,
                                                  uint64_t policy) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of every committed group have been read (the buffer is free again)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (TMA reads)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Batch::evict_last bits -> the policy of one operand side (A: shift 0, B: shift 1):
// bit 0/1 evict_last, bit 2/3 evict_first, else evict_normal
__device__ __forceinline__ uint64_t side_policy(int bits, int shift) {
  if (bits & (1 << shift)) return policy_evict_last();
  if (bits & (4 << shift)) return policy_evict_first();
  return policy_evict_normal();
}
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_addr(slot)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// D[tmem] (+)= A[smem] . B[smem]^T, u8 x u8 -> s32
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// D[tmem] (+)= (A[smem] x SFA) . (B[smem] x SFB)^T, packed e2m1, UE8M0 scale per 32 K
__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                         uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
               : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int CW>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[CW]) {
  if constexpr (CW == 16) tmem_ld16(taddr, v);
  else tmem_ld32(taddr, v);
}

// Shared-memory matrix descriptor of a K-major operand tile in the canonical
// SWIZZLE_128B layout TMA writes: rows of 128 bytes, 8-row (1024 B) atoms.
// LBO is unused for swizzled K-major layouts (1), SBO = 1024 B between 8-row
// groups, version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor: s32 accumulator, u8 x u8, both K-major, M = BM, N = 256.
__host__ __device__ constexpr uint32_t idesc_i8() {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(Geo<false>::BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
// Block-scaled descriptor: e2m1 x e2m1 (MXF4 format 1), UE8M0 scales (bit 23),
// scale-factor ids 0, dense K = 64, both K-major, M = BM, N = 240.
__host__ __device__ constexpr uint32_t idesc_mxf4() {
  return (1u << 7) | (1u << 10) | ((uint32_t)(Geo<true>::BN >> 3) << 17) | (1u << 23) | ((uint32_t)(BM >> 4) << 24);
}

// ------------------------------------------------------------ schedule ----
// One problem = rows [0, na) of A' against rows [0, nb) of B' over kblocks
// 128-byte K blocks (read from device memory: the column count is decided on
// the device).  sym: A' == B', only tiles touching the upper triangle
// (col block J >= I / 2 for 128-row / 256-column tiles).
struct Problem {
  int32_t na, nb;
  int32_t sym;
  int32_t tiles_n;            // ceil(nb / BN)
  int64_t tile_begin;         // first global tile of this problem
  const int32_t* kblocks;     // device: K' / 128 (>= 1)
  int32_t map;                // tensor maps m[2 map] (A rows, box 128) and m[2 map + 1] (B rows, box 256)
  int32_t pad_;
};
struct Batch {
  Problem p[MAXPROB];
  const uint2* table;   // nullable: decoded tiles (tile_table_kernel), {pi | ti << 8, tj} per tile
  int n;
  int group;        // GROUP: row blocks per group of the tile order (below)
  int evict_last;   // operand L2 policies (side_policy bits; 0: no hint)
  int debug;        // experiments only (SA_K2T_DEBUG): 1 no MMA, 2 no TMA loads, 4 no epilogue work, 8192 TMEM loads only
  int serp;         // serpentine group order (serp_index): odd groups run backwards
};
struct alignas(64) Maps {
  CUtensorMap m[2 * MAXPROB];
};

struct Tile {
  int pi, row0, col0, ra, rb;
};

// Tile order inside a problem: groups of GROUP (Batch::group) row blocks; in a group, column
// block by column block, the group's rows inside (column-major).  The ~148
// tiles in flight then share ~148 / GROUP column blocks of B and GROUP row
// blocks of A (config 4 bucket, GROUP = 12: ~38 MB + 25 MB, inside the 126 MB
// L2) instead of sweeping all of B every wave.  Symmetric problems keep the tiles with
// column block J >= I / 2.

// sum_{i < n} floor((a i + b) / m)  (the classic floor-sum recursion)
__host__ __device__ inline int64_t floor_sum(int64_t n, int64_t m, int64_t a, int64_t b) {
  int64_t ans = 0;
  while (true) {
    if (a >= m) { ans += (n - 1) * n / 2 * (a / m); a %= m; }
    if (b >= m) { ans += n * (b / m); b %= m; }
    const int64_t y = a * n + b;
    if (y < m) break;
    n = y / m;
    b = y % m;
    const int64_t t = m; m = a; a = t;
  }
  return ans;
}
// tiles of rows [0, i1) of a symmetric problem: row block i keeps column
// blocks j >= floor(i BM / BN) (the blocks holding some column >= a row)
// (TBM = tile rows: 128, or 256 for a CTA pair)
template <int BN, int TBM = BM>
__host__ __device__ inline int64_t sym_tiles_before(int i1, int tn) {
  return (int64_t)i1 * tn - floor_sum(i1, BN, TBM, 0);
}
template <int BN, int TBM = BM>
__host__ __device__ inline int64_t problem_tiles(int64_t na, int64_t nb, bool sym) {
  const int64_t tm = (na + TBM - 1) / TBM, tn = (nb + BN - 1) / BN;
  return sym ? sym_tiles_before<BN, TBM>((int)tm, (int)tn) : tm * tn;
}

template <int BN, int TBM = BM>
__device__ __forceinline__ Tile decode_slow(const Batch& b, int64_t tile);

// Tile of a flat tile index: from the launch's decoded table (one 8-byte load)
// when there is one, else computed (the group / triangle arithmetic below).
template <int BN, int TBM = BM>
__device__ __forceinline__ Tile decode(const Batch& b, int64_t tile) {
  if (!b.table) return decode_slow<BN, TBM>(b, tile);
  const uint2 e = b.table[tile];
  const int pi = (int)(e.x & 0xffu), ti = (int)(e.x >> 8), tj = (int)e.y;
  const Problem& P = b.p[pi];
  Tile T;
  T.pi = pi;
  T.row0 = ti * TBM;
  T.col0 = tj * BN;
  T.ra = min(TBM, P.na - T.row0);
  T.rb = min(BN, P.nb - T.col0);
  return T;
}
// Serpentine group order: the tiles of every odd group of a problem run in
// reverse, so a group's column sweep starts on the B column blocks the
// previous group touched last (still in L2) instead of on the ones it touched
// first (evicted first by the output stream).  Same tile set, same tiles per
// launch; only the position of a tile in the flat order changes.
template <int BN, int TBM>
__device__ __forceinline__ int64_t serp_index(const Batch& b, int64_t tile) {
  int pi = 0;
  while (pi + 1 < b.n && b.p[pi + 1].tile_begin <= tile) ++pi;
  const Problem& P = b.p[pi];
  const int64_t t = tile - P.tile_begin;
  const int tm = (P.na + TBM - 1) / TBM, tn = P.tiles_n;
  const int GROUP = b.group;
  int64_t gb, ge;
  int gi;
  if (!P.sym) {
    const int64_t full = (int64_t)GROUP * tn;
    gi = (int)(t / full);
    gb = (int64_t)gi * full;
    ge = min(gb + full, (int64_t)tm * tn);
  } else {
    int g0 = 0;
    while (g0 + GROUP < tm && sym_tiles_before<BN, TBM>(g0 + GROUP, tn) <= t) g0 += GROUP;
    gi = g0 / GROUP;
    gb = sym_tiles_before<BN, TBM>(g0, tn);
    ge = sym_tiles_before<BN, TBM>(min(g0 + GROUP, tm), tn);
  }
  return (gi & 1) ? P.tile_begin + gb + ge - 1 - t : tile;
}
template <int BN, int TBM>
__global__ void tile_table_kernel(const __grid_constant__ Batch b, int64_t total, uint2* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const Tile T = decode_slow<BN, TBM>(b, b.serp ? serp_index<BN, TBM>(b, t) : t);
    out[t] = make_uint2((uint32_t)T.pi | ((uint32_t)(T.row0 / TBM) << 8), (uint32_t)(T.col0 / BN));
  }
}

template <int BN, int TBM>
__device__ __forceinline__ Tile decode_slow(const Batch& b, int64_t tile) {
  int pi = 0;
  while (pi + 1 < b.n && b.p[pi + 1].tile_begin <= tile) ++pi;
  const Problem& P = b.p[pi];
  int64_t t = tile - P.tile_begin;
  const int tm = (P.na + TBM - 1) / TBM, tn = P.tiles_n;
  const int GROUP = b.group;
  int ti, tj;
  if (!P.sym) {
    const int64_t full = (int64_t)GROUP * tn;     // tiles of a full group
    const int g0 = (int)(t / full) * GROUP;
    const int64_t u = t - (int64_t)g0 / GROUP * full;
    const int rows = min(GROUP, tm - g0);
    ti = g0 + (int)(u % rows);
    tj = (int)(u / rows);
  } else {
    int g0 = 0;
    while (g0 + GROUP < tm && sym_tiles_before<BN, TBM>(g0 + GROUP, tn) <= t) g0 += GROUP;
    int64_t u = t - sym_tiles_before<BN, TBM>(g0, tn);
    const int g1 = min(g0 + GROUP, tm);
    // column j holds the group's rows i < ceil((j + 1) BN / BM)
    auto rows_at = [&](int j) { return min(g1, ((j + 1) * BN + TBM - 1) / TBM) - g0; };
    int j = (int)((int64_t)g0 * TBM / BN);
    for (;; ++j) {   // the first few columns hold fewer rows
      const int cnt = rows_at(j);
      if (cnt == g1 - g0 || u < cnt) break;
      u -= cnt;
    }
    const int cnt = rows_at(j);
    ti = g0 + (int)(u % cnt);
    tj = j + (int)(u / cnt);
  }
  Tile T;
  T.pi = pi;
  T.row0 = ti * TBM;
  T.col0 = tj * BN;
  T.ra = min(TBM, P.na - T.row0);
  T.rb = min(BN, P.nb - T.col0);
  return T;
}

// -------------------------------------------------------------- kernel ----
// Epi (const, a kernel parameter) must provide a per-thread `State` and
//   __device__ bool skip() const;                                  // device-side dispatch guard
//   __device__ void begin(State&, const Tile&, int row) const;     // per thread, per tile
//   static constexpr int TAB_BYTES;                                // table bytes per slice column
//   __device__ void begin(State&, const Tile&, int row, int lane, int cbeg, int cend,
//                         uint8_t* tab) const;                       // before the accumulator wait
//   template <int CW, bool FP4, int CG> __device__ void chunk(State&, const Tile&, int row, int col, const uint32_t (&v)[CW],
//                         int lane, const uint8_t* tab, int tj, uint8_t* xp) const;   // all lanes, converged
//   template <int CW> __device__ void correct(State&, int col, uint32_t (&v)[CW]) const;   // adjust the
//                         accumulator chunk before chunk() (sparse layers, tc_sparse.cu), all lanes converged
//   __device__ void end(State&, const Tile&, int row) const;
//   __device__ void finish(int lane) const;                        // once per epilogue warp, at exit
// row = tile row of this thread (0..127), [cbeg, cend) = the warp's column
// slice of the tile, col = first tile column of the chunk, tab = the warp's
// table (TAB_BYTES x SLICE bytes, 16-byte aligned), tj = col - cbeg, xp = the
// warp's xpose_bytes(CW) scratch.
template <class Epi, int EW, int CW, bool FP4>
__global__ void __launch_bounds__(threads_of(EW), 1)
gemm_kernel(const __grid_constant__ Batch batch, const __grid_constant__ Maps maps, int64_t total_tiles, Epi epi) {
  using G = Geo<FP4>;
  constexpr int BN = G::BN, STAGE_BYTES = G::STAGE_BYTES;
  static_assert(EW % 4 == 0 && BN % CW == 0, "epilogue geometry");
  constexpr int EPI_WARPS = EW;
  if (epi.skip()) return;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t raw_s = s_addr(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base_s - raw_s);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* tab_all = smem + STAGES * STAGE_BYTES + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == EPI_WARPS && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      bar_init(&tfull[b], 1);
      bar_init(&tempty[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == EPI_WARPS + 1) tmem_alloc(tmem_slot, TMEM_COLS);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  if constexpr (FP4) {
    // every UE8M0 scale factor = 2^0 (0x7F): columns [SF_COL, 512) of all 128 lanes
    if (warp < 4)
      for (int c = G::SF_COL; c < TMEM_COLS; c += 8) tmem_st8(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, 0x7F7F7F7Fu);
    fence_before();
    __syncthreads();
    fence_after();
  }

  if (warp == EPI_WARPS) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      const bool hint = batch.evict_last != 0;
      int64_t g = 0;
      for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const Tile T = decode<BN>(batch, tile);
        const Problem& P = batch.p[T.pi];
        const int nkb = *reinterpret_cast<const volatile int32_t*>(P.kblocks);
        const CUtensorMap* ma = &maps.m[2 * P.map];
        const CUtensorMap* mb = &maps.m[2 * P.map + 1];
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int slot = (int)(g % STAGES);
          if (g >= STAGES) bar_wait(&empty[slot], (uint32_t)(((g / STAGES) - 1) & 1));
          if (batch.debug & 2) {
            bar_arrive(&full[slot]);
            continue;
          }
          bar_arrive_tx(&full[slot], STAGE_BYTES);
          const uint32_t dst = base_s + slot * STAGE_BYTES;
          if (hint) {
            tma_2d_hint(dst, ma, kb * BK, T.row0, &full[slot], pol);
            tma_2d_hint(dst + A_BYTES, mb, kb * BK, T.col0, &full[slot], pol);
          } else {
            tma_2d(dst, ma, kb * BK, T.row0, &full[slot]);
            tma_2d(dst + A_BYTES, mb, kb * BK, T.col0, &full[slot]);
          }
        }
      }
    }
  } else if (warp == EPI_WARPS + 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = FP4 ? idesc_mxf4() : idesc_i8();
      const uint32_t sfa = tmem_base + (uint32_t)G::SF_COL, sfb = tmem_base + (uint32_t)G::SF_COL + 16u;
      int64_t g = 0, lt = 0;
      for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
        const Tile T = decode<BN>(batch, tile);
        const Problem& P = batch.p[T.pi];
        const int nkb = *reinterpret_cast<const volatile int32_t*>(P.kblocks);
        const int buf = (int)(lt & 1);
        if (lt >= 2) bar_wait(&tempty[buf], (uint32_t)(((lt >> 1) - 1) & 1));
        fence_after();
        const uint32_t d = tmem_base + (uint32_t)(buf * BN);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int slot = (int)(g % STAGES);
          bar_wait(&full[slot], (uint32_t)((g / STAGES) & 1));
          fence_after();
          const uint32_t sa_ = base_s + slot * STAGE_BYTES;
          const uint64_t da = sw128_desc(sa_), db = sw128_desc(sa_ + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UKB; ++k) {
            if (batch.debug & 1) break;
            const uint64_t off = (uint64_t)((k * UKB) >> 4);
            if constexpr (FP4) mma_mxf4(d, da + off, db + off, idesc, (kb | k) != 0, sfa, sfb);
            else mma_i8(d, da + off, db + off, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[slot]);
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps
    const int quad = warp & 3, part = warp >> 2;
    const int row = quad * 32 + lane;
    constexpr int SLICE = slice_of(EW, CW, FP4);
    constexpr int XB = Epi::xpose_bytes(CW, FP4, 1);
    uint8_t* tab = tab_all + warp * (SLICE * Epi::TAB_BYTES + XB);
    uint8_t* xp = tab + SLICE * Epi::TAB_BYTES;
    const int cbeg = part * SLICE, cend = min(cbeg + SLICE, BN);
    typename Epi::State es;
    int64_t lt = 0;
    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++lt) {
      const Tile T = decode<BN>(batch, tile);
      const int buf = (int)(lt & 1);
      epi.begin(es, T, row, lane, cbeg, cend, tab);   // row state and column tables while the MMA runs
      bar_wait(&tfull[buf], (uint32_t)((lt >> 1) & 1));
      fence_after();
#pragma unroll 1
      for (int col = cbeg; col < ((batch.debug & 4) ? cbeg : cend); col += CW) {
        uint32_t v[CW];
        tmem_ld<CW>(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + col), v);
        if constexpr (FP4) {
          // exact integer-valued f32 sums (< 2^23): add 2^23, keep the mantissa
#pragma unroll
          for (int j = 0; j < CW; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + 8388608.0f) & 0x7FFFFFu;
        }
        epi.template correct<CW>(es, col, v);
        epi.template chunk<CW, FP4, 1>(es, T, row, col, v, lane, tab, col - cbeg, xp);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(&tempty[buf]);
      epi.end(es, T, row);
    }
    epi.finish(lane);
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == EPI_WARPS + 1) tmem_dealloc(tmem_base, TMEM_COLS);
}


// ============================================================ CTA pair ====
// The same contraction with tcgen05.mma.cta_group::2 on a CTA pair (a
// cluster of 2 CTAs on the two SMs of a TPC): one MMA instruction computes a
// 256 x BN tile, each CTA holding 128 rows of A and BN / 2 rows of B in its
// own shared memory and its own 128 x BN accumulator in its own TMEM.  Each
// SM therefore streams 128 + BN / 2 operand rows per tile instead of
// 128 + BN -- a third less L2 -> SM traffic for the same tensor work -- and
// a stage is 31 (32) KB, so more stages fit.
//   both CTAs, warp EW lane 0: TMA loads of the CTA's A rows / B half into
//     its own stage slot, completing on the LEADER's full barrier (the
//     .cta_group::2 form; the leader alone posts expect_tx for both halves);
//   leader, warp EW+1 lane 0: waits full, issues 4 x tcgen05.mma.cta_group::2
//     per stage, commits (multicast to both CTAs) the stage's empty barriers
//     and, per tile, the accumulator's tfull barriers;
//   both CTAs, warps 0..EW-1: the epilogue on the CTA's own 128 rows; each
//     warp releases the accumulator on the leader's tempty barrier (2 EW
//     arrivals per tile, the peer's through its cluster address).
template <bool FP4>
struct Geo2 {
  static constexpr int BN = Geo<FP4>::BN;                 // tile columns (UMMA N, split over the pair)
  static constexpr int BNH = BN / 2;                      // B rows per CTA
  static constexpr int B_BYTES = BNH * BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // per CTA
  static constexpr int SF_COL = 2 * BN;
};
static_assert(Geo2<true>::STAGE_BYTES % 1024 == 0 && Geo2<false>::STAGE_BYTES % 1024 == 0, "stage alignment");
constexpr int TBM2 = 2 * BM;   // pair-tile rows

#ifndef SA_MAX_STAGES
#define SA_MAX_STAGES 8
#endif
__host__ __device__ constexpr int stages2_of(int EW, int CW, bool FP4, int TB, int XB) {
  return (232448 - 1024 - 512 - EW * (slice_of(EW, CW, FP4) * TB + XB)) /
                     (FP4 ? Geo2<true>::STAGE_BYTES : Geo2<false>::STAGE_BYTES) > SA_MAX_STAGES
             ? SA_MAX_STAGES
             : (232448 - 1024 - 512 - EW * (slice_of(EW, CW, FP4) * TB + XB)) /
                   (FP4 ? Geo2<true>::STAGE_BYTES : Geo2<false>::STAGE_BYTES);
}
__host__ __device__ constexpr int smem2_of(int EW, int CW, bool FP4, int TB, int XB) {
  return stages2_of(EW, CW, FP4, TB, XB) * (FP4 ? Geo2<true>::STAGE_BYTES : Geo2<false>::STAGE_BYTES) + 1024 + 512 +
         EW * (slice_of(EW, CW, FP4) * TB + XB);
}

// one lane of a converged warp (elect.sync): the warp-wide role loops keep
// their descriptors / coordinates warp-uniform (uniform registers), and only
// the elected lane issues the single-thread TMA / MMA / commit instructions
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Relaxed: the arrive only has to follow this warp's completed tcgen05.ld
// (tcgen05.wait::ld + fence::before_thread_sync); a .release arrive would also
// drain every outstanding global store of the warp (MEMBAR + ERRBAR) first.
__device__ __forceinline__ void bar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load into this CTA's shared memory, completing on the leader CTA's barrier
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
// the same with an L2 eviction-priority policy
__device__ __forceinline__ void tma_2d_pair_hint(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                 uint32_t leader_bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_addr(slot)), "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void mma2_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma2_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                          uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb));
}
// arrive on barrier `bar` (same offset) in both CTAs of the pair when the issued MMAs complete
__device__ __forceinline__ void mma_commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          s_addr(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// instruction descriptors with M = 256 (the pair)
__host__ __device__ constexpr uint32_t idesc2_i8() {
  return (2u << 4) | ((uint32_t)(Geo<false>::BN >> 3) << 17) | ((uint32_t)(TBM2 >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc2_mxf4() {
  return (1u << 7) | (1u << 10) | ((uint32_t)(Geo<true>::BN >> 3) << 17) | (1u << 23) | ((uint32_t)(TBM2 >> 4) << 24);
}

template <class Epi, int EW, int CW, bool FP4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(threads_of(EW), 1)
gemm2_kernel(const __grid_constant__ Batch batch, const __grid_constant__ Maps maps, int64_t total_tiles,
             const __grid_constant__ Epi epi) {
  using G = Geo2<FP4>;
  constexpr int BN = G::BN, BNH = G::BNH, STAGE_BYTES = G::STAGE_BYTES;
  constexpr int XB = Epi::xpose_bytes(CW, FP4, 2);
  constexpr int NST = stages2_of(EW, CW, FP4, Epi::TAB_BYTES, XB);
  static_assert(NST >= 3, "CTA-pair stages");
  static_assert(EW % 4 == 0 && BN % CW == 0, "epilogue geometry");
  // per-warp scratch of a multiple of 1024 bytes (the TMA-store staging of
  // the matrix epilogue: SWIZZLE_128B boxes need 1024-byte alignment) sits
  // right after the (1024-aligned) stages; otherwise after the tables
  constexpr bool XALIGN = XB > 0 && XB % 1024 == 0;
  constexpr int XFRONT = XALIGN ? EW * XB : 0;
  constexpr int EPI_WARPS = EW;
  if (epi.skip()) return;   // uniform over the grid (device state word)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t raw_s = s_addr(smem_raw);
  const uint32_t base_s = (raw_s + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base_s - raw_s);
  uint8_t* xp_all = smem + NST * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE_BYTES + XFRONT);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* tab_all = smem + NST * STAGE_BYTES + XFRONT + 512;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == EPI_WARPS && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      bar_init(&tfull[b], 1);
      bar_init(&tempty[b], 2 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == EPI_WARPS + 1) tmem_alloc2(tmem_slot, TMEM_COLS);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  if constexpr (FP4) {
    if (warp < 4)
      for (int c = G::SF_COL; c < TMEM_COLS; c += 8)
        tmem_st8(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, 0x7F7F7F7Fu);
    fence_before();
  }
  cluster_sync_all();   // barriers initialised and scale factors written in both CTAs
  fence_after();

  if (warp == EPI_WARPS) {
    // ------------------------------------------------ TMA producer (both CTAs, whole warp)
    {
      const uint32_t full0_leader = map_to_rank(s_addr(&full[0]), 0);   // the leader's full barriers
      const bool no_tma = (batch.debug & 2) != 0;
      const bool hint = batch.evict_last != 0;
      const uint64_t pol_a = side_policy(batch.evict_last, 0), pol_b = side_policy(batch.evict_last, 1);
      uint32_t g = 0;
      for (int64_t tile = pair; tile < total_tiles; tile += npairs) {
        const Tile T = decode<BN, TBM2>(batch, tile);
        const Problem& P = batch.p[T.pi];
        const int nkb = *reinterpret_cast<const volatile int32_t*>(P.kblocks);
        const CUtensorMap* ma = &maps.m[2 * P.map];
        const CUtensorMap* mb = &maps.m[2 * P.map + 1];
        const int arow = T.row0 + (int)rank * BM, brow = T.col0 + (int)rank * BNH;
        uint32_t slot = g % NST, phase = (g / NST) & 1u;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          if (g >= (uint32_t)NST) bar_wait(&empty[slot], phase ^ 1u);
          if (elect_one()) {
            if (no_tma) {
              if (leader) bar_arrive(&full[slot]);
            } else {
              if (leader) bar_arrive_tx(&full[slot], 2 * STAGE_BYTES);
              const uint32_t dst = base_s + slot * STAGE_BYTES;
              const uint32_t fb = full0_leader + slot * 8u;
              if (hint) {
                tma_2d_pair_hint(dst, ma, kb * BK, arow, fb, pol_a);
                tma_2d_pair_hint(dst + A_BYTES, mb, kb * BK, brow, fb, pol_b);
              } else {
                tma_2d_pair(dst, ma, kb * BK, arow, fb);
                tma_2d_pair(dst + A_BYTES, mb, kb * BK, brow, fb);
              }
            }
          }
          __syncwarp();
          if (++slot == (uint32_t)NST) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == EPI_WARPS + 1) {
    // ------------------------------------------------ MMA issuer (leader CTA, whole warp)
    if (leader) {
      constexpr uint32_t idesc = FP4 ? idesc2_mxf4() : idesc2_i8();
      const uint32_t sfa = tmem_base + (uint32_t)G::SF_COL, sfb = tmem_base + (uint32_t)G::SF_COL + 16u;
      const bool no_mma = (batch.debug & 1) != 0;
      uint32_t g = 0, lt = 0;
      for (int64_t tile = pair; tile < total_tiles; tile += npairs, ++lt) {
        const Tile T = decode<BN, TBM2>(batch, tile);
        const Problem& P = batch.p[T.pi];
        const int nkb = *reinterpret_cast<const volatile int32_t*>(P.kblocks);
        const uint32_t buf = lt & 1u;
        if (lt >= 2) bar_wait(&tempty[buf], ((lt >> 1) - 1) & 1u);
        fence_after();
        const uint32_t d = tmem_base + buf * (uint32_t)BN;
        uint32_t slot = g % NST, phase = (g / NST) & 1u;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          bar_wait(&full[slot], phase);
          fence_after();
          const uint32_t sa_ = base_s + slot * STAGE_BYTES;
          const uint64_t da = sw128_desc(sa_), db = sw128_desc(sa_ + A_BYTES);
          if (elect_one()) {
            if (!no_mma) {
#pragma unroll
              for (int k = 0; k < BK / UKB; ++k) {
                const uint64_t off = (uint64_t)((k * UKB) >> 4);
                if constexpr (FP4) mma2_mxf4(d, da + off, db + off, idesc, (kb | k) != 0, sfa, sfb);
                else mma2_i8(d, da + off, db + off, idesc, (kb | k) != 0);
              }
            }
            mma_commit2(&empty[slot]);
          }
          __syncwarp();
          if (++slot == (uint32_t)NST) {
            slot = 0;
            phase ^= 1u;
          }
        }
        if (elect_one()) mma_commit2(&tfull[buf]);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps (both CTAs)
    const int quad = warp & 3, part = warp >> 2;
    const int row = quad * 32 + lane;
    constexpr int SLICE = slice_of(EW, CW, FP4);
    uint8_t* tab = tab_all + warp * (SLICE * Epi::TAB_BYTES + (XALIGN ? 0 : XB));
    uint8_t* xp = XALIGN ? xp_all + warp * XB : tab + SLICE * Epi::TAB_BYTES;
    const int cbeg = part * SLICE, cend = min(cbeg + SLICE, BN);
    const uint32_t tempty_leader = map_to_rank(s_addr(&tempty[0]), 0);
    const bool no_epi = (batch.debug & 4) != 0;
    typename Epi::State es;
    uint32_t lt = 0;
    auto half_tile = [&](int64_t tile) {   // this CTA's half of the pair tile
      Tile T = decode<BN, TBM2>(batch, tile);
      T.row0 += (int)rank * BM;
      T.ra = max(0, min(BM, T.ra - (int)rank * BM));
      return T;
    };
    for (int64_t tile = pair; tile < total_tiles; tile += npairs, ++lt) {
      const Tile T = half_tile(tile);
      const uint32_t buf = lt & 1u;
      epi.begin(es, T, row, lane, cbeg, cend, tab);
      bar_wait(&tfull[buf], (lt >> 1) & 1u);
      fence_after();
#pragma unroll 1
      for (int col = cbeg; col < (no_epi ? cbeg : cend); col += CW) {
        uint32_t v[CW];
        tmem_ld<CW>(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(buf * BN + col), v);
        if constexpr (FP4) {
#pragma unroll
          for (int j = 0; j < CW; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + 8388608.0f) & 0x7FFFFFu;
        }
        if (batch.debug & 8192) continue;   // (experiment: the TMEM loads alone)
        epi.template correct<CW>(es, col, v);
        epi.template chunk<CW, FP4, 2>(es, T, row, col, v, lane, tab, col - cbeg, xp);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive_cluster(tempty_leader + buf * 8u);
      epi.end(es, T, row);
    }
    epi.finish(lane);
  }
  fence_before();
  __syncthreads();
  cluster_sync_all();   // no CTA leaves while its peer may still signal its barriers
  fence_after();
  if (warp == EPI_WARPS + 1) tmem_dealloc2(tmem_base, TMEM_COLS);
}

}  // namespace tc
}  // namespace sa
