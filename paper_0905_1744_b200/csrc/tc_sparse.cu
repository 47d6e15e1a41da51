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
//   records   (row, bin, count) for every count >= 2 (appended by the histogram
//             pass, minsum_tc.cu)
//   bin lists per side: the rows repeating each bin (count + scan + scatter)
//   plan      per problem: E = the number of (pair, bin) terms, exactly
//             sum_t n_t (n_t - 1) / 2 (symmetric) or sum_t nA_t nB_t; the
//             problem runs SPARSE (tensor cores on layer 1 only) iff E fits
//             its entry budget, else DENSE (layers >= 2 as MMA columns)
//   entries   one u32 per term, (column within the tile's column block << 16 |
//             min - 1), grouped by key = (row, column block, epilogue slice)
//             -- exactly the set of pairs one epilogue thread owns in one tile
//             -- sorted by column, duplicates of a pair merged
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

// ---------------------------------------------------------- bin counts ----
__global__ void sp_bincount_kernel(const SpLaunch L, const uint2* __restrict__ recs, const uint32_t* __restrict__ nrec,
                                   uint32_t* __restrict__ bincnt) {
  const uint32_t n = min(*nrec, L.rec_cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 r = recs[i];
    const int s = sp_side_of(L, r.x);
    atomicAdd(&bincnt[s * SP_BINS + (r.y & 0xffffu)], 1u);
  }
}

// ------------------------------------------------------------- planning --
// One CTA per problem: E = number of correction terms; sparse iff E <= cap and
// the record buffer did not overflow.  flags[0] |= 1 when any problem is sparse.
__global__ void __launch_bounds__(1024) sp_plan_kernel(const SpLaunch L, const uint32_t* __restrict__ bincnt,
                                                       const uint32_t* __restrict__ nrec, int32_t* __restrict__ mode,
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
    const bool ok = L.enabled && *nrec <= L.rec_cap && E <= (unsigned long long)L.cap[q];
    mode[q] = ok ? 1 : 0;
    if (ok) atomicOr(&flags[0], 1u);
    if (L.terms_out) L.terms_out[q] = E;
  }
}

// --------------------------------------------------- bin lists (per side) --
// One CTA per side: exclusive scan of its SP_BINS counts into binoff[side][t]
// (bincnt keeps the counts: the scatter below consumes them with atomicSub).
__global__ void __launch_bounds__(1024) sp_binscan_kernel(const uint32_t* __restrict__ bincnt,
                                                          uint32_t* __restrict__ binoff,
                                                          const uint32_t* __restrict__ flags,
                                                          const uint32_t* __restrict__ base_dev) {
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
  // sides are laid out one after another in the list array: side s starts
  // after every record of sides < s (base_dev[s], from the side totals)
  uint32_t run = base_dev[s] + wsum[w] + x - tot;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    binoff[s * SP_BSTRIDE + threadIdx.x * PER + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 1023) binoff[s * SP_BSTRIDE + SP_BINS] = run;   // the side's end
}

// side totals -> side bases (one thread; at most 2 * MAXPROB sides)
__global__ void sp_sidebase_kernel(const SpLaunch L, const uint32_t* __restrict__ bincnt, uint32_t* __restrict__ base,
                                   const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
  __shared__ uint32_t tot[2 * tc::MAXPROB];
  const int s = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (s < L.nsides) {
    uint32_t t = 0;
    for (int b = lane; b < SP_BINS; b += 32) t += bincnt[s * SP_BINS + b];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) tot[s] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int i = 0; i < L.nsides; ++i) {
      base[i] = run;
      run += tot[i];
    }
  }
}

// records -> bin lists: list entry = (row within its side, count)
__global__ void sp_scatter_kernel(const SpLaunch L, const uint2* __restrict__ recs, const uint32_t* __restrict__ nrec,
                                  uint32_t* __restrict__ bincnt, const uint32_t* __restrict__ binoff,
                                  uint2* __restrict__ blist, const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
  const uint32_t n = min(*nrec, L.rec_cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 r = recs[i];
    const int s = sp_side_of(L, r.x);
    const uint32_t bin = r.y & 0xffffu;
    const uint32_t pos = binoff[s * SP_BSTRIDE + bin] + atomicSub(&bincnt[s * SP_BINS + bin], 1u) - 1u;
    blist[pos] = make_uint2((uint32_t)(r.x - L.row_begin[s]), r.y >> 16);
  }
}

// -------------------------------------------------------------- pairs ----
// One warp per (problem, bin) of the sparse problems.  FILL = false: count the
// terms per key; FILL = true: write them (kcnt is consumed by atomicSub, so
// the positions inside a key are arbitrary -- sp_sort_kernel orders them).
// Rows in a list are in scatter order; a symmetric pair is (min, max).
template <bool FILL>
__global__ void __launch_bounds__(256) sp_pairs_kernel(const SpLaunch L, const uint32_t* __restrict__ binoff,
                                                       const uint2* __restrict__ blist, const int32_t* __restrict__ mode,
                                                       uint32_t* __restrict__ kcnt, const uint32_t* __restrict__ koff,
                                                       uint32_t* __restrict__ ents, const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < (int64_t)L.nprob * SP_BINS;
       item += nw) {
    const int q = (int)(item / SP_BINS), t = (int)(item % SP_BINS);
    if (!mode[q]) continue;
    const int sa_ = L.side_a[q], sb = L.side_b[q];
    const uint32_t a0 = binoff[sa_ * SP_BSTRIDE + t];
    const uint32_t na = binoff[sa_ * SP_BSTRIDE + t + 1] - a0;
    if (na == 0) continue;
    const uint64_t key0 = L.key_base[q];
    const uint32_t tn = (uint32_t)L.tn[q], np = (uint32_t)L.nparts, bn = (uint32_t)L.bn, sl = (uint32_t)L.slice;
    uint32_t b0 = a0, nb = na;
    if (sb >= 0) {
      b0 = binoff[sb * SP_BSTRIDE + t];
      nb = binoff[sb * SP_BSTRIDE + t + 1] - b0;
    }
    // lanes take rows x of side A; symmetric problems pair x with the later
    // list entries only (each unordered pair once, as (min row, max row))
    for (uint32_t x = lane; x < na; x += 32) {
      const uint2 ex = blist[a0 + x];
      for (uint32_t y = sb < 0 ? x + 1 : 0; y < nb; ++y) {
        const uint2 ey = blist[b0 + y];
        const uint32_t ra = sb < 0 ? min(ex.x, ey.x) : ex.x, rb = sb < 0 ? max(ex.x, ey.x) : ey.x;
        const uint32_t jl = rb % bn;
        const uint64_t key = key0 + ((uint64_t)ra * tn + rb / bn) * np + jl / sl;
        if (FILL) {
          const uint32_t pos = koff[key] + atomicSub(&kcnt[key], 1u) - 1u;
          ents[pos] = (jl << 16) | (min(ex.y, ey.y) - 1u);
        } else {
          atomicAdd(&kcnt[key], 1u);
        }
      }
    }
  }
}

// ----------------------------------------------------------- key scan ----
// Exclusive scan of n u32 counts into out[0..n] (out[n] = total), 3 phases:
// per-4096 block sums, one CTA scanning the block sums, block-local scans.
constexpr int SP_SCAN_BLOCK = 4096;
__global__ void __launch_bounds__(1024) sp_scan_sums_kernel(const uint32_t* __restrict__ in, int64_t n,
                                                            uint32_t* __restrict__ sums,
                                                            const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
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
__global__ void __launch_bounds__(1024) sp_scan_top_kernel(uint32_t* __restrict__ sums, int64_t nb,
                                                           const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
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
                                                             uint32_t* __restrict__ out,
                                                             const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
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

// ------------------------------------------------------- sort + merge ----
// One thread per key: insertion sort of its entries by value (column, then
// term), terms of the same column summed into one entry (a pair sharing
// several repeated bins), the freed tail filled with SP_DEAD (never matched).
__global__ void sp_sort_kernel(const uint32_t* __restrict__ koff, int64_t nkeys, uint32_t* __restrict__ ents,
                               const uint32_t* __restrict__ flags) {
  if (!(flags[0] & 1u)) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nkeys; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = koff[k], e = koff[k + 1];
    if (e - b < 2) continue;
    for (uint32_t i = b + 1; i < e; ++i) {
      const uint32_t x = ents[i];
      uint32_t j = i;
      while (j > b && ents[j - 1] > x) {
        ents[j] = ents[j - 1];
        --j;
      }
      ents[j] = x;
    }
    uint32_t w = b;
    for (uint32_t i = b + 1; i < e; ++i) {
      if ((ents[i] >> 16) == (ents[w] >> 16)) ents[w] += ents[i] & 0xffffu;
      else ents[++w] = ents[i];
    }
    for (uint32_t i = w + 1; i < e; ++i) ents[i] = SP_DEAD;
  }
}

// carried records (a previous launch's, e.g. S2a's rows for S2d's query side)
__global__ void sp_copy_records_kernel(const uint2* __restrict__ src, const uint32_t* __restrict__ nsrc,
                                       uint32_t src_cap, uint2* __restrict__ dst, uint32_t* __restrict__ ndst) {
  const uint32_t n = min(*nsrc, src_cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) *ndst = *nsrc;   // overflow carries over
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// ------------------------------------------------------------- host ----
sa_status sp_build(SpLaunch& L, SpBuffers& B, int sms, cudaStream_t st) {
  const int nb_rec = sms * 4;
  sp_bincount_kernel<<<nb_rec, 256, 0, st>>>(L, B.recs, B.nrec, B.bincnt);
  SA_LAUNCHED();
  sp_plan_kernel<<<L.nprob, 1024, 0, st>>>(L, B.bincnt, B.nrec, B.mode, B.flags);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status sp_entries(SpLaunch& L, SpBuffers& B, int sms, cudaStream_t st) {
  sp_sidebase_kernel<<<1, 32 * 2 * tc::MAXPROB, 0, st>>>(L, B.bincnt, B.sidebase, B.flags);
  SA_LAUNCHED();
  sp_binscan_kernel<<<L.nsides, 1024, 0, st>>>(B.bincnt, B.binoff, B.flags, B.sidebase);
  SA_LAUNCHED();
  sp_scatter_kernel<<<sms * 4, 256, 0, st>>>(L, B.recs, B.nrec, B.bincnt, B.binoff, B.blist, B.flags);
  SA_LAUNCHED();
  // bincnt is now all zero again; binoff keeps the list starts
  const int pw = sms * 8;   // blocks of 8 warps
  sp_pairs_kernel<false><<<pw, 256, 0, st>>>(L, B.binoff, B.blist, B.mode, B.kcnt, nullptr, nullptr, B.flags);
  SA_LAUNCHED();
  const int64_t n = L.nkeys;
  const int64_t nblk = (n + SP_SCAN_BLOCK - 1) / SP_SCAN_BLOCK;
  sp_scan_sums_kernel<<<(unsigned)nblk, 1024, 0, st>>>(B.kcnt, n, B.scan_tmp, B.flags);
  SA_LAUNCHED();
  sp_scan_top_kernel<<<1, 1024, 0, st>>>(B.scan_tmp, nblk, B.flags);
  SA_LAUNCHED();
  sp_scan_final_kernel<<<(unsigned)nblk, 1024, 0, st>>>(B.kcnt, n, B.scan_tmp, B.koff, B.flags);
  SA_LAUNCHED();
  sp_pairs_kernel<true><<<pw, 256, 0, st>>>(L, B.binoff, B.blist, B.mode, B.kcnt, B.koff, B.ents, B.flags);
  SA_LAUNCHED();
  sp_sort_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, sms * 16), 256, 0, st>>>(B.koff, n, B.ents, B.flags);
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
