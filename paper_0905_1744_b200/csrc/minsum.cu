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
#include "common.cuh"

namespace sa {

__device__ uint64_t g_rtab[65536];   // floor(2^64 / d), d >= 2
__device__ uint32_t g_etab[65536];   // 2^64 mod d

constexpr int MS_MAXPROB = 16;
struct MsBatch {
  MsProblem p[MS_MAXPROB];
  int n;
};

__global__ void recip_kernel() {
  int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= 65536) return;
  if (d < 2) { g_rtab[d] = 0; g_etab[d] = 0; return; }
  uint64_t r = ~0ull / (uint64_t)d;
  uint64_t e = ~0ull % (uint64_t)d + 1;   // (2^64 - 1) mod d + 1
  if (e == (uint64_t)d) { r += 1; e = 0; }
  g_rtab[d] = r;
  g_etab[d] = (uint32_t)e;
}

sa_status ensure_recip_tables(cudaStream_t st) {
  static bool ready[64] = {};
  int dev = 0;
  SA_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && ready[dev]) return SA_OK;
  recip_kernel<<<256, 256, 0, st>>>();
  SA_LAUNCHED();
  if (dev < 64) ready[dev] = true;
  return SA_OK;
}

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

// floor(C * 2^64 / D) accumulated into a 96-bit (lo, hi) register pair.
__device__ __forceinline__ void add_term(uint64_t& lo, uint32_t& hi, uint32_t C, uint32_t D) {
  if (D == 0 || C == 0) return;
  if (C == D) { hi += 1; return; }      // the term is exactly 2^64
  uint64_t t = (uint64_t)C * g_rtab[D] + (uint64_t)((C * g_etab[D]) / D);
  lo += t;
  hi += (lo < t) ? 1u : 0u;
}

__device__ __forceinline__ void atomic_add_key(sa_key128* k, uint64_t lo, uint64_t hi) {
  unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long*>(&k->lo), (unsigned long long)lo);
  uint64_t carry = ((uint64_t)old + lo < (uint64_t)old) ? 1ull : 0ull;
  uint64_t h = hi + carry;
  if (h) atomicAdd(reinterpret_cast<unsigned long long*>(&k->hi), (unsigned long long)h);
}

__device__ __forceinline__ void shfl_add(uint64_t& lo, uint32_t& hi, int mask) {
  uint64_t olo = __shfl_xor_sync(0xffffffffu, lo, mask);
  uint32_t ohi = __shfl_xor_sync(0xffffffffu, hi, mask);
  lo += olo;
  hi += ohi + ((lo < olo) ? 1u : 0u);
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

template <bool SYM, int ENC, int VAR>
__global__ void __launch_bounds__(MS_THREADS, 1)
minsum_kernel(const __grid_constant__ MsBatch batch, int64_t total_tiles, int ldw, uint32_t one) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ty = (warp >> 1) * 4 + (lane >> 3);  // row group 0..15: rows ty + 16 i
  const int tx = (warp & 1) * 8 + (lane & 7);     // col group 0..15: cols tx + 16 j
  const int nK = ldw / MS_BKW;
  constexpr int STAGE_W = 2 * MS_BM * MS_LDW;

  for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    int pi = 0;
    while (pi + 1 < batch.n && batch.p[pi + 1].tile_begin <= tile) ++pi;
    const MsProblem& P = batch.p[pi];
    int64_t t = tile - P.tile_begin;
    int ti, tj;
    if (SYM) {
      const int T = P.tiles_b;
      ti = 0;
      while (t >= T - ti) { t -= T - ti; ++ti; }
      tj = ti + (int)t;
    } else {
      ti = (int)(t / P.tiles_b);
      tj = (int)(t % P.tiles_b);
    }
    const int row0 = ti * MS_BM, col0 = tj * MS_BM;
    const int ra = min(MS_BM, P.na - row0), rb = min(MS_BM, P.nb - col0);
    const uint32_t* Ag = P.A + (int64_t)row0 * ldw;
    const uint32_t* Bg = P.B + (int64_t)col0 * ldw;

    auto load = [&](int stage, int kc) {
      uint32_t* sb = smem + stage * STAGE_W;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = tid + MS_THREADS * u;
        const int r = c >> 3, ch = c & 7;
        const bool isA = r < MS_BM;
        const int rr = isA ? r : r - MS_BM;
        const bool valid = rr < (isA ? ra : rb);
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
      const uint32_t* Bs = As + MS_BM * MS_LDW;
      if (ENC == ENC_U8_SAD && VAR != 0) {
        sad_stage<(VAR == 1 ? 4 : 2), (VAR == 3 ? 1 : 2)>(As, Bs, ty, tx, acc);
        continue;
      }
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
            if (ENC == ENC_U8_SAD) {
              // 16 bins: four VABSDIFF4.U8.ACC, |a-b| of 4 byte lanes summed into acc
              vsad4_acc(acc[i][j], a[i].x, b[j].x);
              vsad4_acc(acc[i][j], a[i].y, b[j].y);
              vsad4_acc(acc[i][j], a[i].z, b[j].z);
              vsad4_acc(acc[i][j], a[i].w, b[j].w);
            } else if (ENC == ENC_U16_MIN_IMAD) {
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
    __syncthreads();   // smem is reloaded by the next tile

    // ------------------------------------------------------------ epilogue
    const bool offdiag = SYM && (ti != tj);
    int nkr[8], nkc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = ty + 16 * i;
      nkr[i] = (r < ra) ? P.nkA[row0 + r] : -1;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = tx + 16 * j;
      nkc[j] = (c < rb) ? P.nkB[col0 + c] : -1;
    }

    if (P.keyA) {
      // row sums: key_i += sum_j floor(C_ij 2^64 / D_ij)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint64_t lo = 0;
        uint32_t hi = 0;
        if (nkr[i] >= 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (nkc[j] < 0) continue;
            const uint32_t C = acc_to_C<ENC>(acc[i][j], nkr[i], nkc[j]);
            add_term(lo, hi, C, (uint32_t)min(nkr[i], nkc[j]));
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
        for (int j = 0; j < 8; ++j) {
          uint64_t lo = 0;
          uint32_t hi = 0;
          if (nkc[j] >= 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (nkr[i] < 0) continue;
              const uint32_t C = acc_to_C<ENC>(acc[i][j], nkr[i], nkc[j]);
              add_term(lo, hi, C, (uint32_t)min(nkr[i], nkc[j]));
            }
          }
          shfl_add(lo, hi, 8);
          shfl_add(lo, hi, 16);
          if (lane < 8 && nkc[j] >= 0 && (lo | hi)) atomic_add_key(P.keyB + col0 + tx + 16 * j, lo, hi);
        }
      }
    }
    if (P.num || P.sim) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (nkr[i] < 0) continue;
        const int64_t gr = row0 + ty + 16 * i;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (nkc[j] < 0) continue;
          const int64_t gc = col0 + tx + 16 * j;
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
}

static int g_num_sms = 0;

template <bool SYM, int ENC, int VAR>
static sa_status launch_one(const MsBatch& b, int64_t tiles, int ldw, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    SA_CUDA(cudaFuncSetAttribute(minsum_kernel<SYM, ENC, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, MS_SMEM));
    configured = true;
  }
  const int64_t grid = tiles < g_num_sms ? tiles : g_num_sms;
  minsum_kernel<SYM, ENC, VAR><<<(unsigned)grid, MS_THREADS, MS_SMEM, st>>>(b, tiles, ldw, 1u);
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
static sa_status launch_enc(const MsBatch& b, int64_t tiles, int ldw, int enc, cudaStream_t st) {
  if (enc == ENC_U8_SAD) {
    switch (sad_variant()) {
      case 1: return launch_one<SYM, ENC_U8_SAD, 1>(b, tiles, ldw, st);
      case 2: return launch_one<SYM, ENC_U8_SAD, 2>(b, tiles, ldw, st);
      case 3: return launch_one<SYM, ENC_U8_SAD, 3>(b, tiles, ldw, st);
      default: return launch_one<SYM, ENC_U8_SAD, 0>(b, tiles, ldw, st);
    }
  }
  if (enc == ENC_U16_MIN_IMAD) return launch_one<SYM, ENC_U16_MIN_IMAD, 0>(b, tiles, ldw, st);
  return launch_one<SYM, ENC_U16_MIN, 0>(b, tiles, ldw, st);
}

sa_status minsum_launch(const std::vector<MsProblem>& probs_in, int ldw, int enc, cudaStream_t st,
                        cudaEvent_t ev0, cudaEvent_t ev1) {
  if (ldw % MS_BKW != 0) return fail(SA_E_INVAL, "profile row stride must be a multiple of 64 bins");
  SA_TRY(ensure_recip_tables(st));
  if (g_num_sms == 0) {
    int dev = 0;
    SA_CUDA(cudaGetDevice(&dev));
    SA_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
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
    const sa_status rs = sym ? launch_enc<true>(b, tiles, ldw, enc, st) : launch_enc<false>(b, tiles, ldw, enc, st);
    if (rs != SA_OK) return rs;
  }
  if (ev1) SA_CUDA(cudaEventRecord(ev1, st));
  return SA_OK;
}

// ------------------------------------------------- u16 -> u8 operand rows --
// The SAD encoding needs every count <= 255; the conversion saturates and
// reports the largest count so the caller can fall back to the u16 engine.
__global__ void to_u8_kernel(const uint16_t* __restrict__ p16, int64_t n, int stride16, uint8_t* __restrict__ p8,
                             int stride8, uint32_t* __restrict__ maxc) {
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
                       uint32_t* maxc, cudaStream_t st) {
  (void)bins;
  if (n <= 0) return SA_OK;
  const int64_t work = n * (stride8 / 8);
  const int64_t blocks = (work + 255) / 256;
  to_u8_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(p16, n, stride16, p8, stride8, maxc);
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

__global__ void keys_to_f64_kernel(const sa_key128* __restrict__ keys, int64_t n, double inv_scale_den,
                                   int64_t npool, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = ldexp(u128_to_double(keys[i].hi, keys[i].lo), -64);
    out[i] = __ddiv_rn(v, (double)npool);
  }
}

sa_status keys_to_f64_launch(const sa_key128* keys, int64_t n, int64_t npool, double* out, cudaStream_t st) {
  if (n <= 0) return SA_OK;
  const int64_t blocks = (n + 255) / 256;
  keys_to_f64_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, st>>>(keys, n, 0.0, npool, out);
  SA_LAUNCHED();
  return SA_OK;
}

}  // namespace sa
