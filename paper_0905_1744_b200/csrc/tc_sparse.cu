// K2T sparse layers: the exact correction for threshold layers >= 2
// (DESIGN.md §4c).  Eq. 1's numerator, split by layer:
//
//   C_ij = L1_ij + R_ij,   L1_ij = sum_t [c^i_t >= 1][c^j_t >= 1]
//                          R_ij  = sum_t (min(c^i_t, c^j_t) - 1)_+
//
// (min(a, b) = [a >= 1][b >= 1] + (min(a, b) - 1)_+ for a, b >= 0).  L1 is the
// dense 0/1 contraction over the 8000 bins the tensor cores compute; R only
// has terms where BOTH counts reach 2, and on the protein workloads a row has
// ~8 such bins of 8000 (SURVEY §8(d) probe; cfg4 buckets: 0.001-0.065 terms
// per pair).  So R is a sparse-sparse product: for every bin t, every pair of
// rows that both repeat t contributes min(c_i, c_j) - 1.  This file builds, per
// launch and on the device:
//
//   records   (row, bin, count) for every count >= 2, appended by the histogram
//             pass (minsum_tc.cu)
//   plan      per problem: E = the number of (pair, bin) terms, exactly
//             sum_t n_t (n_t - 1) / 2 (symmetric) or sum_t nA_t nB_t; the
//             problem runs SPARSE (tensor cores on layer 1 only) iff E fits
//             its entry budget, else DENSE (layers >= 2 as MMA columns)
//   bin lists per side: the rows repeating each bin, sorted by row
//   row lists the records of each row
//   entries   per row a of a problem's A side, a k-way merge (by partner row)
//             of the bin lists of a's repeated bins (partners b > a when
//             symmetric): one u32 per partner, (column within the tile's
//             column block << 16 | sum of min - 1 over the shared bins),
//             ordered by partner; koff / kpart index them by key (a, column
//             block) -- the pairs one epilogue thread owns in one tile
//
// The GEMM epilogue (KeyMatEpi::correct) adds the entries to its accumulator
// chunk before computing keys or F, so every downstream value sees the exact C.
#include "common.cuh"
#include "tc_sparse.cuh"

namespace sa {

__device__ __forceinline__ int sp_side_of(const SpLaunch& L, int64_t g) {
  int s = 0;
  while (s + 1 < L.nsides && L.row_begin[s + 1] <= g) ++s;
  return s;
}
__device__ __forceinline__ uint32_t sp_nrec(const SpLaunch& L, const uint32_t* nrec) {
  return min(*nrec, L.rec_cap);   // records of overflowed segments are partial: their problems run dense
}

// --------------------------------------------- bin counts, row counts ----
__global__ void sp_bincount_kernel(const SpLaunch L, const uint2* __restrict__ recs, const uint32_t* __restrict__ nrec,
                                   uint32_t* __restrict__ bincnt, uint32_t* __restrict__ sidetot,
                                   uint32_t* __restrict__ rcnt) {
  __shared__ uint32_t st[2 * tc::MAXPROB];
  if (threadIdx.x < 2 * tc::MAXPROB) st[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t n = sp_nrec(L, nrec);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 r = recs[i];
    const int s = sp_side_of(L, r.x);
    atomicAdd(&bincnt[s * SP_BINS + (r.y & 0xffffu)], 1u);
    atomicAdd(&rcnt[r.x], 1u);
    atomicAdd(&st[s], 1u);
  }
  __syncthreads();
  if (threadIdx.x < L.nsides && st[threadIdx.x]) atomicAdd(&sidetot[threadIdx.x], st[threadIdx.x]);
}

// ------------------------------------------------------------- planning --
// One CTA per problem: E = number of correction terms; sparse iff E <= cap and
// none of its rows' record segments overflowed (povf).  flags[0] |= 1 when any problem is sparse.
__global__ void __launch_bounds__(1024) sp_plan_kernel(const SpLaunch L, const uint32_t* __restrict__ bincnt,
                                                       const uint32_t* __restrict__ povf, int32_t* __restrict__ mode,
                                                       uint32_t* __restrict__ flags) {
  __shared__ unsigned long long part[32];
  const int q = blockIdx.x;
  const uint32_t* a = bincnt + L.side_a[q] * SP_BINS;
  const uint32_t* b = L.side_b[q] >= 0 ? bincnt + L.side_b[q] * SP_BINS : nullptr;
  unsigned long long e = 0;
  for (int t = threadIdx.x; t < SP_BINS; t += blockDim.x) {
    const unsigned long long na = a[t];
    e += b ? na * b[t] : na * (na - (na > 0 ? 1ull : 0ull)) / 2;
  }
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long E = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) E += part[w];
    const bool ok = L.enabled && !povf[q] && E <= (unsigned long long)L.cap[q];
    mode[q] = ok ? 1 : 0;
    if (ok) atomicOr(&flags[0], 1u);
    if (L.terms_out) L.terms_out[q] = E;
  }
}

// --------------------------------------------------- bin lists (per side) --
// One CTA per side: exclusive scan of its SP_BINS counts into
// binoff[side][0..SP_BINS] (bincnt keeps the counts: the scatter below
// consumes them with atomicSub).  Sides follow one another in the list array.
__global__ void __launch_bounds__(1024) sp_binscan_kernel(const uint32_t* __restrict__ bincnt,
                                                          uint32_t* __restrict__ binoff,
                                                          const uint32_t* __restrict__ flags,
                                                          const uint32_t* __restrict__ sidetot) {
  if (!(flags[0] & 1u)) return;
  __shared__ uint32_t wsum[32];
  const int s = blockIdx.x;
  constexpr int PER = SP_BINS / 1024;
  const uint32_t* c = bincnt + s * SP_BINS;
  uint32_t v[PER], tot = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = c[threadIdx.x * PER + i];
    tot += v[i];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t y = wsum[lane], z = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += t;
    }
    wsum[lane] = z - y;
  }
  __syncthreads();
  uint32_t sbase = 0;
  for (int i = 0; i < s; ++i) sbase += sidetot[i];
  uint32_t run = sbase + wsum[w] + x - tot;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    binoff[s * SP_BSTRIDE + threadIdx.x * PER + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 1023) binoff[s * SP_BSTRIDE + SP_BINS] = run;   // the side's end
}

// records -> bin lists (entry = (row within its side, count)) and row lists
// (entry = bin | count << 16); both in arbitrary order inside a list
__global__ void sp_scatter_kernel(const SpLaunch L, const uint2* __restrict__ recs, const uint32_t* __restrict__ nrec,
                                  uint32_t* __restrict__ bincnt, const uint32_t* __restrict__ binoff,
                                  uint2* __restrict__ blist, uint32_t* __restrict__ rcnt,
                                  const uint32_t* __restrict__ rstart, uint32_t* __restrict__ rlist,
                                  uint32_t* __restrict__ bslot, const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
  const uint32_t n = sp_nrec(L, nrec);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 r = recs[i];
    const int s = sp_side_of(L, r.x);
    const uint32_t bin = r.y & 0xffffu;
    const uint32_t pos = binoff[s * SP_BSTRIDE + bin] + atomicSub(&bincnt[s * SP_BINS + bin], 1u) - 1u;
    const uint32_t slot = rstart[r.x] + atomicSub(&rcnt[r.x], 1u) - 1u;
    blist[pos] = make_uint2((uint32_t)(r.x - L.row_begin[s]), r.y >> 16);
    bslot[pos] = slot;   // the record's row-list slot, for its position after the list sort
    rlist[slot] = r.y;
  }
}

// One warp per (side, bin) list: rank sort by row (rows are distinct inside a
// list), out of place; spos[row-list slot] = the sorted position of that
// record's own entry (a symmetric row's partners are the list's tail after it).  O(n^2 / 32) per list: the lists are short (a bin's
// rows with count >= 2; ~15 on the config-4 buckets).
__global__ void __launch_bounds__(256) sp_listsort_kernel(const SpLaunch L, const uint32_t* __restrict__ binoff,
                                                          const uint2* __restrict__ blist, uint2* __restrict__ sorted,
                                                          const uint32_t* __restrict__ bslot,
                                                          uint32_t* __restrict__ spos, const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < (int64_t)L.nsides * SP_BINS;
       item += nw) {
    const int s = (int)(item / SP_BINS), t = (int)(item % SP_BINS);
    const uint32_t b = binoff[s * SP_BSTRIDE + t], n = binoff[s * SP_BSTRIDE + t + 1] - b;
    if (n == 0) continue;
    if (n == 1) {
      if (lane == 0) {
        sorted[b] = blist[b];
        spos[bslot[b]] = b;
      }
      continue;
    }
    for (uint32_t i = lane; i < n; i += 32) {
      const uint2 x = blist[b + i];
      uint32_t rank = 0;
      for (uint32_t j = 0; j < n; ++j) rank += blist[b + j].x < x.x ? 1u : 0u;
      sorted[b + rank] = x;
      spos[bslot[b + i]] = b + rank;   // where the record's own row sits in its sorted list
    }
  }
}

// ------------------------------------------------------------ row merge --
struct SpRow {
  int q;          // problem
  uint32_t r;     // row within the problem's A side
  uint32_t g;     // row in the launch (flattened sides)
};
__device__ __forceinline__ SpRow sp_row_of(const SpLaunch& L, uint32_t ai) {
  int q = 0;
  while (q + 1 < L.nprob && (uint32_t)L.abase[q + 1] <= ai) ++q;
  SpRow R;
  R.q = q;
  R.r = ai - (uint32_t)L.abase[q];
  R.g = (uint32_t)L.row_begin[L.side_a[q]] + R.r;
  return R;
}
// first position in the sorted list [b, e) whose row exceeds r
__device__ __forceinline__ uint32_t sp_upper(const uint2* __restrict__ list, uint32_t b, uint32_t e, uint32_t r) {
  while (b < e) {
    const uint32_t m = (b + e) >> 1;
    if (list[m].x <= r) b = m + 1;
    else e = m;
  }
  return b;
}

// Terms of each A-side row (before merging the bins of one partner): one warp
// per row, lanes over the row's records.
constexpr int SP_FILL_WARPS = 4;
__global__ void __launch_bounds__(32 * SP_FILL_WARPS) sp_rowcount_kernel(
    const SpLaunch L, const int32_t* __restrict__ mode, const uint32_t* __restrict__ binoff,
    const uint32_t* __restrict__ spos, const uint32_t* __restrict__ rstart, const uint32_t* __restrict__ rlist,
    uint32_t* __restrict__ rowcnt, const uint32_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const bool any = (flags[0] & 1u) != 0;
  const uint32_t NA = (uint32_t)L.abase[L.nprob];
  const uint32_t nwarps = gridDim.x * SP_FILL_WARPS;
  for (uint32_t ai = blockIdx.x * SP_FILL_WARPS + (threadIdx.x >> 5); ai < NA; ai += nwarps) {
    const SpRow R = sp_row_of(L, ai);
    uint32_t cnt = 0;
    if (any && mode[R.q]) {
      const bool sym = L.side_b[R.q] < 0;
      const int ps = sym ? L.side_a[R.q] : L.side_b[R.q];
      for (uint32_t i = rstart[R.g] + lane; i < rstart[R.g + 1]; i += 32) {
        const uint32_t t = rlist[i] & 0xffffu;
        const uint32_t b = binoff[ps * SP_BSTRIDE + t], e = binoff[ps * SP_BSTRIDE + t + 1];
        cnt += e - (sym ? spos[i] + 1u : b);
      }
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) rowcnt[ai] = cnt;
  }
}

// Entries of each A-side row, one warp per row.  Raw terms (partner b,
// min(c_a, c_b) - 1) come from the tails of the sorted lists of the row's
// repeated bins (partners b > a when symmetric).  The entries are one u32 per
// distinct partner, (column within its column block << 16 | summed term), in
// partner order from rowoff[ai]; koff / kpart are written for every column
// block J of the row (empty blocks: position, 0); slots left by partners that
// share several bins hold SP_DEAD.  Two ways, by the row's raw term count:
//   <= SP_ROWBUF (nearly every row): raw terms into shared arrays, a warp
//      bitonic sort of the keys (partner << 9 | slot) -- in registers up to
//      128 terms --, one entry per run of equal partners, and the block counts
//      through a shared per-block counter array;
//   larger (long, repetitive sequences): a sweep over the column blocks the
//      partners fall in, each repeated bin a cursor kept in shared memory,
//      terms added into a per-column shared accumulator per block.
constexpr int SP_ROWBUF = 512;   // raw terms per warp buffer (power of two)
constexpr int SP_CURSORS = 128;   // cursor state of the sweep: 2.5 KB, inside the raw buffer
constexpr int SP_BN_MAX = 256;   // column-block width (240 e2m1, 256 u8)

// Ascending sort of the n <= 32 E keys key[0..n) by one warp in registers:
// bitonic network on 32 E slots (element t * 32 + lane in register t, pads
// 0xFFFFFFFF); strides below 32 exchange through shuffles, larger ones
// between a lane's registers.  The sorted keys go back to key[].
template <int E>
__device__ __forceinline__ void sp_warp_sort(uint32_t* key, uint32_t n, int lane) {
  uint32_t v[E];
#pragma unroll
  for (int t = 0; t < E; ++t) v[t] = (uint32_t)(t * 32 + lane) < n ? key[t * 32 + lane] : 0xFFFFFFFFu;
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int t2 = t ^ (stride >> 5);
          if (t2 > t) {
            const bool up = (((t * 32 + lane) & size) == 0);
            const uint32_t a = v[t], b = v[t2];
            if ((a > b) == up) {
              v[t] = b;
              v[t2] = a;
            }
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int i = t * 32 + lane;
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[t], stride);
          const bool up = (i & size) == 0, lower = (lane & stride) == 0;
          v[t] = (lower == up) ? min(v[t], o) : max(v[t], o);
        }
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < E; ++t)
    if ((uint32_t)(t * 32 + lane) < n) key[t * 32 + lane] = v[t];
  __syncwarp();
}

// Occupancy: the row fill is latency-bound (dependent gathers per row), so
// the per-warp counter array is sized by the launch (accw = max(tn, bn)
// words, dynamic shared memory) instead of SP_TN_MAX, and registers are
// capped for SA_FILL_MINB CTAs per SM.
#ifndef SA_FILL_MINB
#define SA_FILL_MINB 10
#endif
__global__ void __launch_bounds__(32 * SP_FILL_WARPS, SA_FILL_MINB) sp_rowfill_kernel(
    const SpLaunch L, const int32_t* __restrict__ mode, const uint32_t* __restrict__ binoff,
    const uint2* __restrict__ sorted, const uint32_t* __restrict__ spos, const uint32_t* __restrict__ rstart,
    const uint32_t* __restrict__ rlist,
    const uint32_t* __restrict__ rowoff, uint32_t* __restrict__ ents, uint32_t* __restrict__ koff,
    uint32_t* __restrict__ kpart, const uint32_t* __restrict__ flags, int accw) {
  __shared__ unsigned long long s_buf[SP_FILL_WARPS][SP_ROWBUF];   // raw terms; cursors of the sweep
  extern __shared__ uint32_t s_acc[];                              // [SP_FILL_WARPS][accw]: per-block counters; sweep accumulator
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned long long* buf = s_buf[wib];
  uint32_t* acc = s_acc + wib * accw;
  // the sweep's cursor state overlays the raw buffer (4 KB): position, end, own count, current partner
  uint32_t* cur = reinterpret_cast<uint32_t*>(buf);
  uint32_t* end = cur + SP_CURSORS;
  uint32_t* own = end + SP_CURSORS;
  uint2* val = reinterpret_cast<uint2*>(own + SP_CURSORS);
  const bool any = (flags[0] & 1u) != 0;
  const uint32_t bn = (uint32_t)L.bn, sl = (uint32_t)L.slice;
  const uint32_t NA = (uint32_t)L.abase[L.nprob];
  const uint32_t nwarps = gridDim.x * SP_FILL_WARPS;
  for (uint32_t c = lane; c < (uint32_t)accw; c += 32) acc[c] = 0u;
  __syncwarp();
  for (uint32_t ai = blockIdx.x * SP_FILL_WARPS + wib; ai < NA; ai += nwarps) {
    const SpRow R = sp_row_of(L, ai);
    const uint32_t tn = (uint32_t)L.tn[R.q];
    const uint64_t kbase = L.key_base[R.q] + (uint64_t)R.r * tn;
    const uint32_t p0 = rowoff[ai], p1 = rowoff[ai + 1], nraw = p1 - p0;
    uint32_t pos = p0, curJ = 0;   // (sweep) blocks < curJ are written
    const bool active = any && mode[R.q] && nraw > 0;
    const bool sym = L.side_b[R.q] < 0;
    const int ps = sym ? L.side_a[R.q] : L.side_b[R.q];
    const uint32_t r0 = rstart[R.g], k = rstart[R.g + 1] - r0;
    if (active && nraw <= (uint32_t)SP_ROWBUF) {
      // ---- raw terms -> shared arrays: key = partner << 9 | slot, term[slot]
      // (lanes take records; slots by a warp scan)
      uint32_t* key = reinterpret_cast<uint32_t*>(buf);
      uint32_t* term = key + SP_ROWBUF;
      uint32_t base = 0;
      for (uint32_t i0 = 0; i0 < k; i0 += 32) {
        const uint32_t i = i0 + lane;
        uint32_t pb = 0, pe = 0, o = 0;
        if (i < k) {
          const uint32_t rr = rlist[r0 + i];
          const uint32_t t = rr & 0xffffu;
          o = rr >> 16;
          pb = sym ? spos[r0 + i] + 1u : binoff[ps * SP_BSTRIDE + t];
          pe = binoff[ps * SP_BSTRIDE + t + 1];
        }
        const uint32_t len = pe - pb;
        uint32_t x = len;
        for (int sh = 1; sh < 32; sh <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, sh);
          if (lane >= sh) x += y;
        }
        // the chunk's raw terms spread over the lanes (consecutive terms of a
        // bin on consecutive lanes: independent, mostly coalesced loads); term
        // w's bin = the largest lane j whose start (exclusive prefix) is <= w
        const uint32_t start = x - len, total = __shfl_sync(0xffffffffu, x, 31);
        for (uint32_t w0 = 0; w0 < total; w0 += 32) {
          const uint32_t w = w0 + lane;
          int j = 0;
#pragma unroll
          for (int s = 16; s > 0; s >>= 1)
            if (__shfl_sync(0xffffffffu, start, j + s) <= w) j += s;
          const uint32_t pj = __shfl_sync(0xffffffffu, pb, j) + (w - __shfl_sync(0xffffffffu, start, j));
          const uint32_t oj = __shfl_sync(0xffffffffu, o, j);
          if (w < total) {
            const uint2 e = sorted[pj];
            key[base + w] = (e.x << 9) | (base + w);
            term[base + w] = min(oj, e.y) - 1u;
          }
        }
        base += total;
      }
      __syncwarp();
      // ---- sort the keys: in registers up to 128 (shuffle bitonic), else in shared memory
      if (nraw <= 32) sp_warp_sort<1>(key, nraw, lane);
      else if (nraw <= 64) sp_warp_sort<2>(key, nraw, lane);
      else if (nraw <= 128) sp_warp_sort<4>(key, nraw, lane);
      else {
        uint32_t n2 = 256;
        while (n2 < nraw) n2 <<= 1;
        for (uint32_t i = nraw + lane; i < n2; i += 32) key[i] = 0xFFFFFFFFu;
        __syncwarp();
        for (uint32_t size = 2; size <= n2; size <<= 1)
          for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t h = lane; h < n2 / 2; h += 32) {   // one compare-exchange per lane and pass
              const uint32_t i = ((h & ~(stride - 1)) << 1) | (h & (stride - 1)), j = i + stride;
              const uint32_t a = key[i], c = key[j];
              if ((a > c) == ((i & size) == 0)) {
                key[i] = c;
                key[j] = a;
              }
            }
            __syncwarp();
          }
      }
      // ---- one entry per distinct partner (run heads, ballot scan), each
      // head summing its run's terms; per-block slice counters
      uint32_t outn = 0;
      for (uint32_t i0 = 0; i0 < nraw; i0 += 32) {
        const uint32_t i = i0 + lane;
        bool head = false;
        uint32_t b = 0, d = 0;
        if (i < nraw) {
          const uint32_t kv = key[i];
          b = kv >> 9;
          head = i == 0 || (key[i - 1] >> 9) != b;
          if (head) {
            d = term[kv & 511u];
            for (uint32_t j = i + 1; j < nraw && (key[j] >> 9) == b; ++j) d += term[key[j] & 511u];
          }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, head);
        if (head) {
          const uint32_t J = b / bn, jl = b - J * bn;
          ents[p0 + outn + __popc(m & ((1u << lane) - 1u))] = (jl << 16) | d;
          atomicAdd(&acc[J], 1u << (8 * (jl / sl)));
        }
        outn += __popc(m);
      }
      __syncwarp();
      // ---- keys of every block: slice counts and a scan of the block totals
      uint32_t run = p0;
      for (uint32_t j0 = 0; j0 < tn; j0 += 32) {
        const uint32_t j = j0 + lane;
        const uint32_t pc = j < tn ? acc[j] : 0u;
        const uint32_t tot = __vsadu4(pc, 0u);
        uint32_t x = tot;
        for (int sh = 1; sh < 32; sh <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, sh);
          if (lane >= sh) x += y;
        }
        if (j < tn) {
          koff[kbase + j] = run + x - tot;
          kpart[kbase + j] = pc;
          acc[j] = 0u;
        }
        run += __shfl_sync(0xffffffffu, x, 31);
      }
      for (uint32_t i = p0 + outn + lane; i < p1; i += 32) ents[i] = SP_DEAD;
      __syncwarp();
      continue;
    }
    if (active) {
      // ---- long row: sweep over the column blocks
      const bool cached = k <= (uint32_t)SP_CURSORS;
      if (cached) {
        for (uint32_t i = lane; i < k; i += 32) {
          const uint32_t rr = rlist[r0 + i];
          const uint32_t t = rr & 0xffffu;
          const uint32_t b = binoff[ps * SP_BSTRIDE + t], e = binoff[ps * SP_BSTRIDE + t + 1];
          const uint32_t p = sym ? spos[r0 + i] + 1u : b;
          cur[i] = p;
          end[i] = e;
          own[i] = rr >> 16;
          val[i] = p < e ? sorted[p] : make_uint2(0xFFFFFFFFu, 0u);
        }
        __syncwarp();
      }
      while (true) {
        uint32_t mn = 0xFFFFFFFFu;   // the next block: the smallest current partner
        if (cached) {
          for (uint32_t i = lane; i < k; i += 32) mn = min(mn, val[i].x);
        } else {
          for (uint32_t i = lane; i < k; i += 32) {
            const uint32_t rr = rlist[r0 + i];
            const uint32_t t = rr & 0xffffu;
            const uint32_t b = binoff[ps * SP_BSTRIDE + t], e = binoff[ps * SP_BSTRIDE + t + 1];
            const uint32_t lo = sym ? max(curJ * bn, R.r + 1u) : curJ * bn;
            const uint32_t p = lo == 0 ? b : sp_upper(sorted, b, e, lo - 1u);
            if (p < e) mn = min(mn, sorted[p].x);
          }
        }
        for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if (mn == 0xFFFFFFFFu) break;
        const uint32_t J = mn / bn, lo_b = J * bn, hi_b = lo_b + bn;
        for (uint32_t j = curJ + lane; j < J; j += 32) {   // empty blocks before J
          koff[kbase + j] = pos;
          kpart[kbase + j] = 0u;
        }
        if (cached) {
          for (uint32_t i = lane; i < k; i += 32) {
            uint2 v = val[i];
            if (v.x >= hi_b) continue;
            uint32_t p = cur[i];
            const uint32_t e = end[i], o = own[i];
            while (v.x < hi_b) {
              atomicAdd(&acc[v.x - lo_b], min(o, v.y) - 1u);
              ++p;
              v = p < e ? sorted[p] : make_uint2(0xFFFFFFFFu, 0u);
            }
            cur[i] = p;
            val[i] = v;
          }
        } else {
          for (uint32_t i = lane; i < k; i += 32) {
            const uint32_t rr = rlist[r0 + i];
            const uint32_t t = rr & 0xffffu, o = rr >> 16;
            const uint32_t b = binoff[ps * SP_BSTRIDE + t], e = binoff[ps * SP_BSTRIDE + t + 1];
            const uint32_t lo = sym ? max(lo_b, R.r + 1u) : lo_b;
            for (uint32_t p = lo == 0 ? b : sp_upper(sorted, b, e, lo - 1u); p < e; ++p) {
              const uint2 v = sorted[p];
              if (v.x >= hi_b) break;
              atomicAdd(&acc[v.x - lo_b], min(o, v.y) - 1u);
            }
          }
        }
        __syncwarp();
        koff[kbase + J] = pos;
        uint32_t pc = 0;
        for (uint32_t c0 = 0; c0 < bn; c0 += 32) {
          const uint32_t c = c0 + lane;
          const uint32_t d = c < bn ? acc[c] : 0u;
          const uint32_t m = __ballot_sync(0xffffffffu, d != 0u);
          if (d) {
            ents[pos + __popc(m & ((1u << lane) - 1u))] = (c << 16) | d;
            acc[c] = 0u;
          }
          pc += d ? 1u << (8 * (c / sl)) : 0u;   // this lane's slice counts (<= 8 per slice: no carry)
          pos += __popc(m);
        }
        for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
        if (lane == 0) kpart[kbase + J] = pc;
        __syncwarp();
        curJ = J + 1;
      }
    }
    for (uint32_t j = curJ + lane; j < tn; j += 32) {
      koff[kbase + j] = pos;
      kpart[kbase + j] = 0u;
    }
    for (uint32_t i = pos + lane; i < p1; i += 32) ents[i] = SP_DEAD;
    __syncwarp();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) koff[L.nkeys] = rowoff[NA];
}

// ----------------------------------------------------------- u32 scan ----
// Exclusive scan of n u32 counts into out[0..n] (out[n] = total), 3 phases:
// per-4096 block sums, one CTA scanning the block sums, block-local scans.
constexpr int SP_SCAN_BLOCK = 4096;
__global__ void __launch_bounds__(1024) sp_scan_sums_kernel(const uint32_t* __restrict__ in, int64_t n,
                                                            uint32_t* __restrict__ sums) {
  const int64_t b0 = (int64_t)blockIdx.x * SP_SCAN_BLOCK;
  uint32_t s = 0;
  for (int64_t i = b0 + threadIdx.x; i < min(n, b0 + SP_SCAN_BLOCK); i += blockDim.x) s += in[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ uint32_t w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < 32; ++i) t += w[i];
    sums[blockIdx.x] = t;
  }
}
__global__ void __launch_bounds__(1024) sp_scan_top_kernel(uint32_t* __restrict__ sums, int64_t nb) {
  __shared__ uint32_t w[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? sums[i] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) w[wi] = x;
    __syncthreads();
    if (wi == 0) {
      const uint32_t y = w[lane];
      uint32_t z = y;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += t;
      }
      w[lane] = z - y;
    }
    __syncthreads();
    const uint32_t c = carry;
    if (i < nb) sums[i] = c + w[wi] + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + w[wi] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = carry;
}
__global__ void __launch_bounds__(1024) sp_scan_final_kernel(const uint32_t* __restrict__ in, int64_t n,
                                                             const uint32_t* __restrict__ sums,
                                                             uint32_t* __restrict__ out) {
  __shared__ uint32_t w[32];
  constexpr int PER = SP_SCAN_BLOCK / 1024;
  const int64_t b0 = (int64_t)blockIdx.x * SP_SCAN_BLOCK + threadIdx.x * PER;
  uint32_t v[PER], tot = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = b0 + i < n ? in[b0 + i] : 0u;
    tot += v[i];
  }
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  uint32_t x = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) w[wi] = x;
  __syncthreads();
  if (wi == 0) {
    const uint32_t y = w[lane];
    uint32_t z = y;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += t;
    }
    w[lane] = z - y;
  }
  __syncthreads();
  uint32_t run = sums[blockIdx.x] + w[wi] + x - tot;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    if (b0 + i < n) out[b0 + i] = run;
    run += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}

static sa_status scan_u32(const uint32_t* in, int64_t n, uint32_t* out, uint32_t* tmp, cudaStream_t st) {
  const int64_t nblk = std::max<int64_t>(1, (n + SP_SCAN_BLOCK - 1) / SP_SCAN_BLOCK);
  sp_scan_sums_kernel<<<(unsigned)nblk, 1024, 0, st>>>(in, n, tmp);
  SA_LAUNCHED();
  sp_scan_top_kernel<<<1, 1024, 0, st>>>(tmp, nblk);
  SA_LAUNCHED();
  sp_scan_final_kernel<<<(unsigned)nblk, 1024, 0, st>>>(in, n, tmp, out);
  SA_LAUNCHED();
  return SA_OK;
}

// carried records (a previous launch's, e.g. S2a's rows for S2d's query side)
// (nsrc: the carried launch's nrec words, [0] count, [2] incomplete; ndst =
// nrec + 1 of the new launch: its [1] carried count, [3] carried incomplete)
__global__ void sp_copy_records_kernel(const uint2* __restrict__ src, const uint32_t* __restrict__ nsrc,
                                       uint32_t src_cap, uint2* __restrict__ dst, uint32_t* __restrict__ ndst) {
  const uint32_t n = min(nsrc[0], src_cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ndst[0] = n;
    ndst[2] = nsrc[2];   // the carried launch's incomplete flag
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// ------------------------------------------------------------- host ----
sa_status sp_build(SpLaunch& L, SpBuffers& B, int sms, cudaStream_t st) {
  sp_bincount_kernel<<<sms * 4, 256, 0, st>>>(L, B.recs, B.nrec, B.bincnt, B.sidebase, B.rcnt);
  SA_LAUNCHED();
  sp_plan_kernel<<<L.nprob, 1024, 0, st>>>(L, B.bincnt, B.povf, B.mode, B.flags);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status sp_entries(SpLaunch& L, SpBuffers& B, int sms, cudaStream_t st) {
  sp_binscan_kernel<<<L.nsides, 1024, 0, st>>>(B.bincnt, B.binoff, B.flags, B.sidebase);
  SA_LAUNCHED();
  const int64_t R = L.row_begin[L.nsides];
  SA_TRY(scan_u32(B.rcnt, R, B.rstart, B.scan_tmp, st));
  sp_scatter_kernel<<<sms * 4, 256, 0, st>>>(L, B.recs, B.nrec, B.bincnt, B.binoff, B.blist, B.rcnt, B.rstart,
                                             B.rlist, B.bslot, B.flags);
  SA_LAUNCHED();
  sp_listsort_kernel<<<sms * 8, 256, 0, st>>>(L, B.binoff, B.blist, B.sorted, B.bslot, B.spos, B.flags);
  SA_LAUNCHED();
  const int64_t NA = L.abase[L.nprob];
  const unsigned fb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((NA + SP_FILL_WARPS - 1) / SP_FILL_WARPS,
                                                                       (int64_t)sms * 16));
  sp_rowcount_kernel<<<fb, 32 * SP_FILL_WARPS, 0, st>>>(L, B.mode, B.binoff, B.spos, B.rstart, B.rlist, B.rowcnt,
                                                        B.flags);
  SA_LAUNCHED();
  SA_TRY(scan_u32(B.rowcnt, NA, B.rowoff, B.scan_tmp, st));
  int accw = L.bn;
  for (int q = 0; q < L.nprob; ++q)
    if (L.cap[q] > 0) accw = std::max(accw, (int)L.tn[q]);   // problems that can run sparse: tn <= SP_TN_MAX
  accw = std::min((accw + 31) & ~31, SP_TN_MAX);
  sp_rowfill_kernel<<<fb, 32 * SP_FILL_WARPS, SP_FILL_WARPS * accw * 4, st>>>(
      L, B.mode, B.binoff, B.sorted, B.spos, B.rstart, B.rlist, B.rowoff, B.ents, B.koff, B.kpart, B.flags, accw);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status sp_copy_records(const uint2* src, const uint32_t* nsrc, uint32_t src_cap, uint2* dst, uint32_t* ndst,
                          int sms, cudaStream_t st) {
  sp_copy_records_kernel<<<sms * 2, 256, 0, st>>>(src, nsrc, src_cap, dst, ndst);
  SA_LAUNCHED();
  return SA_OK;
}

}  // namespace sa
