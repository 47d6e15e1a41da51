// K4-K6 -- ordering, sampling, pivot agreement, bucket assignment and the
// stable bucket scatter of the redistribution (§3.1.1-3.1.2,
// P:343-423; Algorithm 2 steps 3-11).
//
// Orders are by (exact rank, global index) (O4 / reading Z12).  On the device
// the rank is its 128-bit key; a comparison is certified when the keys differ
// by at least the pool size.  Every kernel that orders also
// flags the items whose order the keys do not certify, so the host can resolve
// them exactly (sa_partition's exact path).
#include <cstring>

#include "common.cuh"

namespace sa {

struct SegSpec {   // segment s = [ (q0+s)*N/P - base, (q0+s+1)*N/P - base )
  int64_t N, P, q0, base;
  __host__ __device__ int64_t begin(int64_t s) const { return (q0 + s) * N / P - base; }
};

__device__ __forceinline__ bool key_lt(const sa_key128& a, int64_t ga, const sa_key128& b, int64_t gb) {
  if (a.hi != b.hi) return a.hi < b.hi;
  if (a.lo != b.lo) return a.lo < b.lo;
  return ga < gb;
}
// |a - b| < window (128-bit)
__device__ __forceinline__ bool key_near(const sa_key128& a, const sa_key128& b, int64_t window) {
  uint64_t dlo, dhi;
  const bool a_ge = (a.hi > b.hi) || (a.hi == b.hi && a.lo >= b.lo);
  if (a_ge) { dlo = a.lo - b.lo; dhi = a.hi - b.hi - (a.lo < b.lo ? 1 : 0); }
  else      { dlo = b.lo - a.lo; dhi = b.hi - a.hi - (b.lo < a.lo ? 1 : 0); }
  return dhi == 0 && dlo < (uint64_t)window;
}

// Exact segment sort by (key, gid) in O(w) expected work per segment.  One CTA
// per segment:
//  1. d_i = RN(key_i) as a double and [min, max] over the segment;
//  2. bucket_i = floor((d_i - min) * nb / (max - min)) -- a monotone
//     non-decreasing function of the exact key, so every item of a lower
//     bucket precedes every item of a higher one;
//  3. counting sort of the buckets, then the position of i inside its bucket
//     = #{j in the bucket : (k_j, g_j) < (k_i, g_i)} by exact 128-bit compares.
// Ties and near-ties are exact (the compares use the full keys); skewed or
// constant keys degrade to quadratic work inside the crowded buckets only.
// Adjacent sorted keys closer than `window` (the pool size) are counted in
// *amb_count: the key order is then not certified.
constexpr int BS_THREADS = 1024;
constexpr int BS_MAXB = 4096;

__device__ __forceinline__ double key_to_double(const sa_key128& k) {
  if (k.hi == 0) return __ull2double_rn(k.lo);
  const int sh = 64 - __clzll((long long)k.hi);
  uint64_t m, rest;
  if (sh == 64) { m = k.hi; rest = k.lo; }
  else { m = (k.hi << (64 - sh)) | (k.lo >> sh); rest = k.lo & ((1ull << sh) - 1); }
  m |= (rest != 0) ? 1ull : 0ull;
  return ldexp(__ull2double_rn(m), sh);
}

__global__ void __launch_bounds__(BS_THREADS)
bucket_sort_kernel(const sa_key128* __restrict__ keys, const int64_t* __restrict__ gids, int64_t gid0, SegSpec sp,
                   int64_t window, int32_t* __restrict__ order_out, int32_t* __restrict__ bkt,
                   int32_t* __restrict__ list, uint32_t* __restrict__ amb_count) {
  __shared__ int32_t start[BS_MAXB + 1];
  __shared__ int32_t fill[BS_MAXB];
  __shared__ int32_t part[BS_THREADS];
  __shared__ double rmin[BS_THREADS / 32], rmax[BS_THREADS / 32];
  const int tid = threadIdx.x;
  const int64_t s = blockIdx.x;
  const int64_t b = sp.begin(s), e = sp.begin(s + 1), w = e - b;
  if (w <= 0) return;
  auto gid = [&](int64_t i) { return gids ? gids[i] : gid0 + i; };

  double mn = 1.0 / 0.0, mx = -1.0 / 0.0;
  for (int64_t i = b + tid; i < e; i += BS_THREADS) {
    const double d = key_to_double(keys[i]);
    mn = fmin(mn, d);
    mx = fmax(mx, d);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((tid & 31) == 0) { rmin[tid >> 5] = mn; rmax[tid >> 5] = mx; }
  __syncthreads();
  mn = rmin[0];
  mx = rmax[0];
  for (int t = 1; t < BS_THREADS / 32; ++t) { mn = fmin(mn, rmin[t]); mx = fmax(mx, rmax[t]); }
  const int64_t nb_want = w / 2 < 1 ? 1 : w / 2;
  const int nb = (int)(nb_want < BS_MAXB ? nb_want : BS_MAXB);
  const double scale = mx > mn ? (double)nb / (mx - mn) : 0.0;

  for (int t = tid; t < nb; t += BS_THREADS) start[t] = 0;
  __syncthreads();
  for (int64_t i = b + tid; i < e; i += BS_THREADS) {
    int bk = (int)((key_to_double(keys[i]) - mn) * scale);
    bk = min(max(bk, 0), nb - 1);
    bkt[i] = bk;
    atomicAdd(&start[bk], 1);
  }
  __syncthreads();
  // exclusive scan of the nb counts: 4 per thread, then a block scan
  int loc[4], sum = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int t = tid * 4 + q;
    loc[q] = t < nb ? start[t] : 0;
    sum += loc[q];
  }
  part[tid] = sum;
  __syncthreads();
  for (int o = 1; o < BS_THREADS; o <<= 1) {
    const int v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = part[tid] - sum;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int t = tid * 4 + q;
    if (t < nb) { start[t] = run; fill[t] = run; }
    run += loc[q];
  }
  if (tid == 0) start[nb] = (int)w;
  __syncthreads();
  for (int64_t i = b + tid; i < e; i += BS_THREADS) {
    const int slot = atomicAdd(&fill[bkt[i]], 1);
    list[b + slot] = (int32_t)(i - b);
  }
  __syncthreads();
  for (int64_t i = b + tid; i < e; i += BS_THREADS) {
    const int bk = bkt[i];
    const sa_key128 ki = keys[i];
    const int64_t gi = gid(i);
    int cnt = 0;
    for (int t = start[bk]; t < start[bk + 1]; ++t) {
      const int64_t j = b + list[b + t];
      cnt += (j != i && key_lt(keys[j], gid(j), ki, gi)) ? 1 : 0;
    }
    order_out[b + start[bk] + cnt] = (int32_t)(i - b);
  }
  __syncthreads();
  uint32_t near = 0;
  for (int64_t t = tid; t + 1 < w; t += BS_THREADS)
    near += key_near(keys[b + order_out[b + t]], keys[b + order_out[b + t + 1]], window) ? 1u : 0u;
  if (near) atomicAdd(amb_count, near);
}

// The same exact segment sort spread over the whole GPU (the one-CTA-per-
// segment kernel above leaves 140 of 148 SMs idle on p = 8 blocks): five
// grid-wide passes over all items of all segments -- (1) d_i = RN(key_i) and
// per-segment [min, max] (warp-reduced atomics on the doubles' bit patterns,
// which order like the non-negative doubles), (2) bucket_i and per-segment
// bucket counts, (3) one CTA per segment scans its counts, (4) bucket lists,
// (5) position inside the bucket by exact (key, gid) compares, then the
// uncertified-neighbour count over the sorted order.
constexpr int SS_NB = 16384;   // buckets per segment at most (w / 2 when smaller)

__device__ __forceinline__ int seg_of(const SegSpec& sp, int nseg, int64_t i) {
  int s = 0;
  while (s + 1 < nseg && sp.begin(s + 1) <= i) ++s;
  return s;
}

__global__ void ss_minmax_kernel(const sa_key128* __restrict__ keys, SegSpec sp, int nseg, int64_t total,
                                 double* __restrict__ dv, unsigned long long* __restrict__ mm) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool in = i < total;
  const int s = in ? seg_of(sp, nseg, i) : -1;
  double d = 0.0;
  if (in) {
    d = key_to_double(keys[i]);
    dv[i] = d;
  }
  unsigned long long lo = in ? (unsigned long long)__double_as_longlong(d) : ~0ull;
  unsigned long long hi = in ? lo : 0ull;
  const int s0 = __shfl_sync(0xffffffffu, s, 0);
  if (__all_sync(0xffffffffu, s == s0 || s < 0)) {   // warp inside one segment: reduce first
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0 && s0 >= 0) {
      atomicMin(&mm[2 * s0], lo);
      atomicMax(&mm[2 * s0 + 1], hi);
    }
  } else if (in) {
    atomicMin(&mm[2 * s], lo);
    atomicMax(&mm[2 * s + 1], hi);
  }
}

__device__ __forceinline__ void seg_scale(const SegSpec& sp, int s, const unsigned long long* mm, int& nb,
                                          double& mn, double& scale) {
  const int64_t w = sp.begin(s + 1) - sp.begin(s);
  const int64_t want = w / 2 < 1 ? 1 : w / 2;
  nb = (int)(want < SS_NB ? want : SS_NB);
  mn = __longlong_as_double((long long)mm[2 * s]);
  const double mx = __longlong_as_double((long long)mm[2 * s + 1]);
  scale = mx > mn ? (double)nb / (mx - mn) : 0.0;
}

__global__ void ss_bucket_kernel(SegSpec sp, int nseg, int64_t total, const double* __restrict__ dv,
                                 const unsigned long long* __restrict__ mm, int32_t* __restrict__ bkt,
                                 int32_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = seg_of(sp, nseg, i);
  int nb;
  double mn, scale;
  seg_scale(sp, s, mm, nb, mn, scale);
  int bk = (int)((dv[i] - mn) * scale);
  bk = min(max(bk, 0), nb - 1);
  bkt[i] = bk;
  atomicAdd(&cnt[(int64_t)s * (SS_NB + 1) + bk], 1);
}

// one CTA per segment: exclusive scan of its bucket counts -> start (in place) and fill
__global__ void __launch_bounds__(1024) ss_scan_kernel(SegSpec sp, const unsigned long long* __restrict__ mm,
                                                       int32_t* __restrict__ cnt, int32_t* __restrict__ fill) {
  __shared__ int32_t part[1024];
  const int s = blockIdx.x, tid = threadIdx.x;
  int nb;
  double mn, scale;
  seg_scale(sp, s, mm, nb, mn, scale);
  int32_t* c = cnt + (int64_t)s * (SS_NB + 1);
  int32_t* f = fill + (int64_t)s * SS_NB;
  constexpr int PER = SS_NB / 1024;
  int loc[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = tid * PER + q;
    loc[q] = t < nb ? c[t] : 0;
    sum += loc[q];
  }
  part[tid] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = part[tid] - sum;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int t = tid * PER + q;
    if (t < nb) {
      c[t] = run;
      f[t] = run;
    }
    run += loc[q];
  }
  if (tid == 0) c[nb] = (int)(sp.begin(s + 1) - sp.begin(s));
}

__global__ void ss_fill_kernel(SegSpec sp, int nseg, int64_t total, const int32_t* __restrict__ bkt,
                               int32_t* __restrict__ fill, int32_t* __restrict__ list) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = seg_of(sp, nseg, i);
  const int64_t b = sp.begin(s);
  const int slot = atomicAdd(&fill[(int64_t)s * SS_NB + bkt[i]], 1);
  list[b + slot] = (int32_t)(i - b);
}

__global__ void ss_rank_kernel(const sa_key128* __restrict__ keys, const int64_t* __restrict__ gids, int64_t gid0,
                               SegSpec sp, int nseg, int64_t total, const int32_t* __restrict__ bkt,
                               const int32_t* __restrict__ cnt, const int32_t* __restrict__ list,
                               int32_t* __restrict__ order_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int s = seg_of(sp, nseg, i);
  const int64_t b = sp.begin(s);
  auto gid = [&](int64_t x) { return gids ? gids[x] : gid0 + x; };
  const int32_t* c = cnt + (int64_t)s * (SS_NB + 1);
  const int bk = bkt[i];
  const sa_key128 ki = keys[i];
  const int64_t gi = gid(i);
  int r = 0;
  for (int t = c[bk]; t < c[bk + 1]; ++t) {
    const int64_t j = b + list[b + t];
    r += (j != i && key_lt(keys[j], gid(j), ki, gi)) ? 1 : 0;
  }
  order_out[b + c[bk] + r] = (int32_t)(i - b);
}

__global__ void ss_near_kernel(const sa_key128* __restrict__ keys, SegSpec sp, int nseg, int64_t total,
                               int64_t window, const int32_t* __restrict__ order, uint32_t* __restrict__ amb_count) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool near = false;
  if (t < total) {
    const int s = seg_of(sp, nseg, t);
    const int64_t b = sp.begin(s);
    if (t + 1 < sp.begin(s + 1)) near = key_near(keys[b + order[t]], keys[b + order[t + 1]], window);
  }
  const uint32_t m = __ballot_sync(0xffffffffu, near);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(amb_count, (uint32_t)__popc(m));
}

sa_status segsort_launch_impl(const sa_key128* keys, const int64_t* gids, int64_t gid0, SegSpec sp, int nseg,
                              int64_t total, int64_t window, int32_t* order_out, uint32_t* amb_count,
                              cudaStream_t st) {
  if (nseg <= 0 || total <= 0) return SA_OK;
  const char* env = getenv("SA_SEGSORT");   // SA_SEGSORT=cta: the one-CTA-per-segment kernel (read per call)
  const bool one_cta = env && !strcmp(env, "cta");
  if (one_cta) {
    void* scratch = nullptr;
    SA_CUDA(cudaMallocAsync(&scratch, (size_t)total * 8, st));
    int32_t* bkt = static_cast<int32_t*>(scratch);
    int32_t* list = bkt + total;
    bucket_sort_kernel<<<(unsigned)nseg, BS_THREADS, 0, st>>>(keys, gids, gid0, sp, window, order_out, bkt, list,
                                                              amb_count);
    const cudaError_t le = cudaGetLastError();
    count_launch();
    cudaFreeAsync(scratch, st);
    if (le != cudaSuccess) return fail(SA_E_CUDA, "bucket_sort_kernel launch: %s", cudaGetErrorString(le));
    return SA_OK;
  }
  Scratch scratch(st);
  SA_ALLOC(dv, double, total);
  SA_ALLOC(bkt, int32_t, total);
  SA_ALLOC(list, int32_t, total);
  SA_ALLOC(mm, unsigned long long, 2 * nseg);
  SA_ALLOC(cnt, int32_t, (size_t)nseg * (SS_NB + 1));
  SA_ALLOC(fill, int32_t, (size_t)nseg * SS_NB);
  SA_CUDA(cudaMemsetAsync(cnt, 0, (size_t)nseg * (SS_NB + 1) * sizeof(int32_t), st));
  // [min, max] init: min = all ones (above every double's bits), max = 0
  SA_CUDA(cudaMemsetAsync(mm, 0, 2 * nseg * sizeof(unsigned long long), st));
  for (int s = 0; s < nseg; ++s)
    SA_CUDA(cudaMemsetAsync(mm + 2 * s, 0xff, sizeof(unsigned long long), st));
  const unsigned g = (unsigned)((total + 255) / 256);
  ss_minmax_kernel<<<g, 256, 0, st>>>(keys, sp, nseg, total, dv, mm);
  SA_LAUNCHED();
  ss_bucket_kernel<<<g, 256, 0, st>>>(sp, nseg, total, dv, mm, bkt, cnt);
  SA_LAUNCHED();
  ss_scan_kernel<<<nseg, 1024, 0, st>>>(sp, mm, cnt, fill);
  SA_LAUNCHED();
  ss_fill_kernel<<<g, 256, 0, st>>>(sp, nseg, total, bkt, fill, list);
  SA_LAUNCHED();
  ss_rank_kernel<<<g, 256, 0, st>>>(keys, gids, gid0, sp, nseg, total, bkt, cnt, list, order_out);
  SA_LAUNCHED();
  ss_near_kernel<<<g, 256, 0, st>>>(keys, sp, nseg, total, window, order_out, amb_count);
  SA_LAUNCHED();
  return SA_OK;
}

// ------------------------------------------------------- sample picking --
// out[s*count + j] = gid of the item at sorted position floor((j+1) w_s / den)
// of segment s (den = count + 1 for the global sample, S:345 / P:348-352;
// den = p for regular samples).
__global__ void pick_kernel(const int32_t* __restrict__ order, SegSpec sp, int nseg, int count, int den,
                            int64_t gid0, int64_t* __restrict__ out_gid, int32_t* __restrict__ out_local) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseg * count) return;
  const int s = t / count, j = t % count;
  const int64_t b = sp.begin(s), w = sp.begin(s + 1) - b;
  const int64_t pos = ((int64_t)(j + 1) * w) / den;
  const int64_t local = b + order[b + pos];
  out_gid[t] = gid0 + local;
  if (out_local) out_local[t] = (int32_t)local;
}

// gather profile rows (stride elements) + nk of the selected local items
__global__ void gather_rows_kernel(const uint16_t* __restrict__ prof, const int32_t* __restrict__ nk,
                                   const int32_t* __restrict__ sel, int nsel, int stride,
                                   uint16_t* __restrict__ out, int32_t* __restrict__ out_nk) {
  for (int r = blockIdx.x; r < nsel; r += gridDim.x) {
    const int64_t src = sel[r];
    const uint4* a = reinterpret_cast<const uint4*>(prof + src * stride);
    uint4* o = reinterpret_cast<uint4*>(out + (int64_t)r * stride);
    for (int v = threadIdx.x; v < stride / 8; v += blockDim.x) o[v] = a[v];
    if (threadIdx.x == 0) out_nk[r] = nk[src];
  }
}

// regular-sample records (S3a): key, gid, nk, block
__global__ void make_records_kernel(const int32_t* __restrict__ local, const int64_t* __restrict__ gid,
                                    int n, const sa_key128* __restrict__ keys, const int32_t* __restrict__ nk,
                                    int count, int q0, sa_pivot* __restrict__ rec) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  sa_pivot r;
  r.key = keys[local[t]];
  r.global_idx = gid[t];
  r.nk = nk[local[t]];
  r.block = q0 + t / count;
  rec[t] = r;
}

__global__ void split_records_kernel(const sa_pivot* __restrict__ rec, int n, sa_key128* __restrict__ keys,
                                     int64_t* __restrict__ gids) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  keys[t] = rec[t].key;
  gids[t] = rec[t].global_idx;
}

// sorted Y and pivots = Y_{floor(p/2) + j p} (1-based), j = 0..p-2 (Z9)
__global__ void pivots_kernel(const sa_pivot* __restrict__ rec, const int32_t* __restrict__ order, int n, int p,
                              int64_t* __restrict__ y_sorted_gid, sa_pivot* __restrict__ pivots) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n && y_sorted_gid) y_sorted_gid[t] = rec[order[t]].global_idx;
  if (t < p - 1) pivots[t] = rec[order[p / 2 + t * p - 1]];
}

// ------------------------------------------------------ bucket assignment --
// bucket(i) = #{pivots strictly below (k_i, g_i)} = smallest b with
// (k_i, g_i) <= pivot_b.  Flags items whose comparison
// with some pivot is not certified by the keys.  Per-bucket counts and residue
// bytes are accumulated for the count exchange (C3).
__global__ void __launch_bounds__(256)
assign_kernel(const sa_key128* __restrict__ keys, int64_t gid0, int n, const sa_pivot* __restrict__ pivots, int p,
              int64_t window, const int64_t* __restrict__ offs, int32_t* __restrict__ bucket_of,
              uint8_t* __restrict__ amb, uint32_t* __restrict__ amb_count, unsigned long long* __restrict__ counts,
              unsigned long long* __restrict__ bytes) {
  extern __shared__ unsigned long long sh[];   // [2p]
  for (int b = threadIdx.x; b < 2 * p; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const sa_key128 k = keys[i];
    const int64_t g = gid0 + i;
    int bkt = 0;
    bool near = false;
    for (int b = 0; b < p - 1; ++b) {
      const sa_pivot pv = pivots[b];
      bkt += key_lt(pv.key, pv.global_idx, k, g) ? 1 : 0;
      near |= (pv.global_idx != g) && key_near(pv.key, k, window);
    }
    bucket_of[i] = bkt;
    if (amb) amb[i] = near ? 1 : 0;
    if (near) atomicAdd(amb_count, 1u);
    atomicAdd(&sh[bkt], 1ull);
    atomicAdd(&sh[p + bkt], (unsigned long long)(offs[i + 1] - offs[i]));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < p; b += blockDim.x) {
    if (sh[b]) atomicAdd(&counts[b], sh[b]);
    if (sh[p + b]) atomicAdd(&bytes[b], sh[p + b]);
  }
}

// --------------------------------------------------------- stable scatter --
// Chunked stable counting sort by bucket: chunk c holds items [256c, 256c+256).
__global__ void __launch_bounds__(256)
bucket_hist_kernel(const int32_t* __restrict__ bucket_of, int n, int p, int32_t* __restrict__ hist /*[nchunk][p]*/) {
  extern __shared__ int32_t hs[];
  for (int b = threadIdx.x; b < p; b += blockDim.x) hs[b] = 0;
  __syncthreads();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i < n) atomicAdd(&hs[bucket_of[i]], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < p; b += blockDim.x) hist[(int64_t)blockIdx.x * p + b] = hs[b];
}

// exclusive offsets, bucket-major then chunk: base[c][b] (one CTA: block scans
// of 4096-entry tiles of the (b, c) sequence, carried from tile to tile)
__global__ void __launch_bounds__(1024) bucket_scan_kernel(const int32_t* __restrict__ hist, int nchunk, int p,
                                                           int64_t* __restrict__ base) {
  __shared__ int64_t part[1024];
  __shared__ int64_t carry;
  const int tid = threadIdx.x;
  const int64_t total = (int64_t)nchunk * p;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < total; t0 += 4096) {
    int64_t loc[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t k = t0 + tid * 4 + q;   // k = b * nchunk + c
      loc[q] = k < total ? hist[(k % nchunk) * p + k / nchunk] : 0;
      sum += loc[q];
    }
    part[tid] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t v = tid >= o ? part[tid - o] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    int64_t run = carry + part[tid] - sum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t k = t0 + tid * 4 + q;
      if (k < total) base[(k % nchunk) * p + k / nchunk] = run;
      run += loc[q];
    }
    __syncthreads();
    if (tid == 1023) carry = run;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256)
bucket_scatter_kernel(const int32_t* __restrict__ bucket_of, int n, int p, const int64_t* __restrict__ base,
                      int32_t* __restrict__ perm /* perm[dst] = src */) {
  extern __shared__ int32_t wc[];   // [8][p]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < 8 * p; t += blockDim.x) wc[t] = 0;
  __syncthreads();
  const int i = blockIdx.x * 256 + threadIdx.x;
  const int b = i < n ? bucket_of[i] : -1 - lane;   // distinct sentinels never match
  const unsigned mask = __match_any_sync(0xffffffffu, b);
  const int rank = __popc(mask & ((1u << lane) - 1u));
  if (i < n && rank == 0) wc[warp * p + b] = __popc(mask);
  __syncthreads();
  if (i < n) {
    int64_t pos = base[(int64_t)blockIdx.x * p + b] + rank;
    for (int w = 0; w < warp; ++w) pos += wc[w * p + b];
    perm[pos] = i;
  }
}

// lens in permuted order -> lens_out[dst] = len(perm[dst])
__global__ void perm_meta_kernel(const int32_t* __restrict__ perm, int n, const int64_t* __restrict__ offs,
                                 const int32_t* __restrict__ bucket_of, int64_t gid0, int64_t* __restrict__ lens,
                                 int64_t* __restrict__ gid_out, int32_t* __restrict__ bkt_out) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int s = perm[d];
  lens[d] = offs[s + 1] - offs[s];
  if (gid_out) gid_out[d] = gid0 + s;
  if (bkt_out) bkt_out[d] = bucket_of[s];
}

// exclusive scan of int64 (3 phases)
__global__ void scan_partial_kernel(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ part) {
  __shared__ int64_t sh[256];
  const int64_t base = (int64_t)blockIdx.x * 1024;
  int64_t s = 0;
  for (int t = 0; t < 4; ++t) {
    const int64_t i = base + threadIdx.x * 4 + t;
    if (i < n) s += in[i];
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void scan_top_kernel(int64_t* __restrict__ part, int64_t nparts) {
  if (threadIdx.x != 0) return;
  int64_t run = 0;
  for (int64_t i = 0; i < nparts; ++i) { const int64_t v = part[i]; part[i] = run; run += v; }
  part[nparts] = run;
}
__global__ void scan_final_kernel(const int64_t* __restrict__ in, int64_t n, const int64_t* __restrict__ part,
                                  int64_t* __restrict__ out) {
  __shared__ int64_t sh[256];
  const int64_t base = (int64_t)blockIdx.x * 1024;
  int64_t v[4], s = 0;
  for (int t = 0; t < 4; ++t) {
    const int64_t i = base + threadIdx.x * 4 + t;
    v[t] = i < n ? in[i] : 0;
    s += v[t];
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {     // Hillis-Steele inclusive
    const int64_t x = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += x;
    __syncthreads();
  }
  int64_t run = part[blockIdx.x] + sh[threadIdx.x] - s;
  for (int t = 0; t < 4; ++t) {
    const int64_t i = base + threadIdx.x * 4 + t;
    if (i < n) out[i] = run;
    run += v[t];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = part[gridDim.x];
}

// copy residues of sequence perm[d] to dst + doff[d]  (one warp per sequence)
__global__ void copy_seqs_kernel(const int32_t* __restrict__ perm, int n, const uint8_t* __restrict__ src,
                                 const int64_t* __restrict__ soff, uint8_t* __restrict__ dst,
                                 const int64_t* __restrict__ doff) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int d = warp; d < n; d += nw) {
    const int s = perm ? perm[d] : d;
    const int64_t a = soff[s], len = soff[s + 1] - a, o = doff[d];
    for (int64_t u = lane; u < len; u += 32) dst[o + u] = src[a + u];
  }
}

// segment reorder after the all-to-all: seg t copies cnt[t] meta records and
// nbytes[t] residue bytes from (src_m, src_r) to (dst_m, dst_r)
struct SegCopy {
  int64_t src_m, dst_m, cnt, src_r, dst_r, nbytes;
};
__global__ void seg_copy_kernel(const SegCopy* __restrict__ segs, int nseg, const int64_t* __restrict__ meta_in,
                                int64_t* __restrict__ meta_out, const uint8_t* __restrict__ res_in,
                                uint8_t* __restrict__ res_out) {
  for (int t = blockIdx.y; t < nseg; t += gridDim.y) {
    const SegCopy sc = segs[t];
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < sc.cnt * 2; u += (int64_t)gridDim.x * blockDim.x)
      meta_out[sc.dst_m * 2 + u] = meta_in[sc.src_m * 2 + u];
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < sc.nbytes; u += (int64_t)gridDim.x * blockDim.x)
      res_out[sc.dst_r + u] = res_in[sc.src_r + u];
  }
}

// meta record = {int64 gid, int32 len, int32 bucket}
__global__ void pack_meta_kernel(const int32_t* __restrict__ perm, int n, const int64_t* __restrict__ offs,
                                 const int32_t* __restrict__ bucket_of, int64_t gid0, int64_t* __restrict__ meta) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int s = perm[d];
  meta[2 * d] = gid0 + s;
  const uint64_t lb = (uint64_t)(uint32_t)(offs[s + 1] - offs[s]) | ((uint64_t)(uint32_t)bucket_of[s] << 32);
  meta[2 * d + 1] = (int64_t)lb;
}
__global__ void unpack_meta_kernel(const int64_t* __restrict__ meta, int n, int64_t* __restrict__ gid,
                                   int64_t* __restrict__ lens, int32_t* __restrict__ bkt) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  gid[d] = meta[2 * d];
  const uint64_t lb = (uint64_t)meta[2 * d + 1];
  lens[d] = (int64_t)(uint32_t)(lb & 0xffffffffu);
  bkt[d] = (int32_t)(uint32_t)(lb >> 32);
}

// ------------------------------------------------------------- host glue --
static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

sa_status segment_sort_keys(const sa_key128* keys, int64_t gid0, int64_t N, int64_t P, int64_t q0, int64_t base,
                            int nseg, int64_t window, int32_t* order_out, uint8_t* amb, uint32_t* amb_count,
                            cudaStream_t st) {
  (void)amb;
  SegSpec sp{N, P, q0, base};
  return segsort_launch_impl(keys, nullptr, gid0, sp, nseg, sp.begin(nseg) - sp.begin(0), window, order_out,
                             amb_count, st);
}

sa_status sort_records(const sa_pivot* rec, int n, int64_t window, sa_key128* tmp_keys, int64_t* tmp_gid,
                       int32_t* order_out, uint8_t* amb, uint32_t* amb_count, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  split_records_kernel<<<cdiv(n, 256), 256, 0, st>>>(rec, n, tmp_keys, tmp_gid);
  SA_LAUNCHED();
  (void)amb;
  SegSpec sp{n, 1, 0, 0};
  return segsort_launch_impl(tmp_keys, tmp_gid, 0, sp, 1, n, window, order_out, amb_count, st);
}

sa_status pick_launch(const int32_t* order, int64_t N, int64_t P, int64_t q0, int64_t base, int nseg, int count,
                      int den, int64_t gid0, int64_t* out_gid, int32_t* out_local, cudaStream_t st) {
  const int tot = nseg * count;
  if (tot <= 0) return SA_OK;
  SegSpec sp{N, P, q0, base};
  pick_kernel<<<cdiv(tot, 128), 128, 0, st>>>(order, sp, nseg, count, den, gid0, out_gid, out_local);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status gather_rows_launch(const uint16_t* prof, const int32_t* nk, const int32_t* sel, int nsel, int stride,
                             uint16_t* out, int32_t* out_nk, cudaStream_t st) {
  if (nsel <= 0) return SA_OK;
  gather_rows_kernel<<<(unsigned)std::min(nsel, 4096), 256, 0, st>>>(prof, nk, sel, nsel, stride, out, out_nk);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status make_records_launch(const int32_t* local, const int64_t* gid, int n, const sa_key128* keys,
                              const int32_t* nk, int count, int q0, sa_pivot* rec, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  make_records_kernel<<<cdiv(n, 128), 128, 0, st>>>(local, gid, n, keys, nk, count, q0, rec);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status pivots_launch(const sa_pivot* rec, const int32_t* order, int n, int p, int64_t* y_sorted_gid,
                        sa_pivot* pivots, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  pivots_kernel<<<cdiv(n, 128), 128, 0, st>>>(rec, order, n, p, y_sorted_gid, pivots);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status assign_launch(const sa_key128* keys, int64_t gid0, int n, const sa_pivot* pivots, int p, int64_t window,
                        const int64_t* offs, int32_t* bucket_of, uint8_t* amb, uint32_t* amb_count,
                        unsigned long long* counts, unsigned long long* bytes, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  assign_kernel<<<cdiv(n, 256), 256, 2 * p * sizeof(unsigned long long), st>>>(
      keys, gid0, n, pivots, p, window, offs, bucket_of, amb, amb_count, counts, bytes);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status scan_launch(const int64_t* in, int64_t n, int64_t* out /*[n+1]*/, int64_t* part /*[cdiv(n,1024)+1]*/,
                      cudaStream_t st) {
  const int64_t np = (n + 1023) / 1024;
  if (n <= 0) {
    SA_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    return SA_OK;
  }
  scan_partial_kernel<<<(unsigned)np, 256, 0, st>>>(in, n, part);
  SA_LAUNCHED();
  scan_top_kernel<<<1, 32, 0, st>>>(part, np);
  SA_LAUNCHED();
  scan_final_kernel<<<(unsigned)np, 256, 0, st>>>(in, n, part, out);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status bucket_perm_launch(const int32_t* bucket_of, int n, int p, int32_t* hist, int64_t* base, int32_t* perm,
                             cudaStream_t st) {
  if (n <= 0) return SA_OK;
  const int nchunk = (int)cdiv(n, 256);
  bucket_hist_kernel<<<nchunk, 256, p * sizeof(int32_t), st>>>(bucket_of, n, p, hist);
  SA_LAUNCHED();
  bucket_scan_kernel<<<1, 1024, 0, st>>>(hist, nchunk, p, base);
  SA_LAUNCHED();
  bucket_scatter_kernel<<<nchunk, 256, 8 * p * sizeof(int32_t), st>>>(bucket_of, n, p, base, perm);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status perm_meta_launch(const int32_t* perm, int n, const int64_t* offs, const int32_t* bucket_of, int64_t gid0,
                           int64_t* lens, int64_t* gid_out, int32_t* bkt_out, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  perm_meta_kernel<<<cdiv(n, 256), 256, 0, st>>>(perm, n, offs, bucket_of, gid0, lens, gid_out, bkt_out);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status copy_seqs_launch(const int32_t* perm, int n, const uint8_t* src, const int64_t* soff, uint8_t* dst,
                           const int64_t* doff, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  copy_seqs_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 8), 148 * 16), 256, 0, st>>>(perm, n, src, soff, dst, doff);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status pack_meta_launch(const int32_t* perm, int n, const int64_t* offs, const int32_t* bucket_of, int64_t gid0,
                           int64_t* meta, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  pack_meta_kernel<<<cdiv(n, 256), 256, 0, st>>>(perm, n, offs, bucket_of, gid0, meta);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status unpack_meta_launch(const int64_t* meta, int n, int64_t* gid, int64_t* lens, int32_t* bkt, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  unpack_meta_kernel<<<cdiv(n, 256), 256, 0, st>>>(meta, n, gid, lens, bkt);
  SA_LAUNCHED();
  return SA_OK;
}

sa_status seg_copy_launch(const void* segs_dev, int nseg, const int64_t* meta_in, int64_t* meta_out,
                          const uint8_t* res_in, uint8_t* res_out, cudaStream_t st) {
  if (nseg <= 0) return SA_OK;
  dim3 grid(64, (unsigned)std::min(nseg, 1024));
  seg_copy_kernel<<<grid, 256, 0, st>>>(static_cast<const SegCopy*>(segs_dev), nseg, meta_in, meta_out, res_in,
                                        res_out);
  SA_LAUNCHED();
  return SA_OK;
}

size_t segcopy_size() { return sizeof(SegCopy); }
void segcopy_fill(void* dst, int t, int64_t src_m, int64_t dst_m, int64_t cnt, int64_t src_r, int64_t dst_r,
                  int64_t nbytes) {
  static_cast<SegCopy*>(dst)[t] = SegCopy{src_m, dst_m, cnt, src_r, dst_r, nbytes};
}

}  // namespace sa
