// K1 -- k-mer count profiles c^X (§3 "k-mer Rank").
//
// One CTA builds one profile at a time (persistent grid-stride over
// sequences): the profile lives in shared memory as packed u16x2 words
// (2 bins per 32-bit word, 16 KB for 20^3 bins), every k-mer occurrence is one
// shared-memory atomicAdd of 1 << 16*(id & 1) into word id >> 1 (a lane never
// carries into its neighbour: a count is <= nk <= 65535, checked), then the
// whole row -- including the zero padding up to the 64-bin row stride -- is
// streamed to HBM with 16-byte vector stores.  The kernel is bound by that
// 16 KB-per-sequence write (K1).  profiles_bulk_kernel (the
// default) hands that write to the TMA engine as one bulk copy per row and
// counts the next sequence into a second buffer meanwhile.
#include "common.cuh"

namespace sa {

__global__ void __launch_bounds__(256)
profiles_kernel(const uint8_t* __restrict__ res, const int64_t* __restrict__ offs, int32_t n, int32_t k,
                int32_t alphabet, int32_t stride, uint16_t* __restrict__ out, int32_t* __restrict__ nk_out,
                uint32_t* __restrict__ err, int cs) {
  extern __shared__ __align__(16) uint32_t hist[];   // stride / 2 words
  const int words = stride >> 1;
  const int vec = words >> 2;                         // uint4 per row (stride % 64 == 0)
  uint4* h4 = reinterpret_cast<uint4*>(hist);
  for (int v = threadIdx.x; v < vec; v += blockDim.x) h4[v] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // the copy-out of each row zeroes the histogram for the next one
  for (int64_t s = blockIdx.x; s < n; s += gridDim.x) {
    const int64_t b = offs[s], e = offs[s + 1];
    const int64_t len = e - b;
    const int64_t nk = len >= k ? len - k + 1 : 0;
    const uint8_t* x = res + b;
    uint32_t bad = 0;
    for (int64_t u = threadIdx.x; u < len; u += blockDim.x)
      if (x[u] >= alphabet) bad = 1;
    for (int64_t u = threadIdx.x; u < nk; u += blockDim.x) {
      uint32_t id = 0;
      bool ok = true;
      for (int t = 0; t < k; ++t) {
        const uint32_t r = x[u + t];
        ok &= r < (uint32_t)alphabet;
        id = id * (uint32_t)alphabet + r;
      }
      if (ok) atomicAdd(&hist[id >> 1], 1u << ((id & 1u) << 4));
    }
    if (bad) atomicOr(err, ERR_RESIDUE);
    if (threadIdx.x == 0) {
      if (nk > 65535) atomicOr(err, ERR_NK);
      nk_out[s] = (int32_t)nk;
    }
    __syncthreads();
    uint4* o4 = reinterpret_cast<uint4*>(out + s * (int64_t)stride);
    if (cs) {
      for (int v = threadIdx.x; v < vec; v += blockDim.x) {
        __stcs(o4 + v, h4[v]);
        h4[v] = make_uint4(0, 0, 0, 0);
      }
    } else {
      for (int v = threadIdx.x; v < vec; v += blockDim.x) {
        o4[v] = h4[v];
        h4[v] = make_uint4(0, 0, 0, 0);
      }
    }
    __syncthreads();
  }
}

// The same with the row copy-out as an asynchronous bulk copy (TMA engine,
// cp.async.bulk shared -> global) from one of two shared-memory histograms:
// the CTA counts row s + grid into the other buffer while row s streams out.
// Before a buffer is zeroed and reused, the bulk store issued from it two
// rows earlier must have finished reading it (wait_group.read 1).
__global__ void __launch_bounds__(256)
profiles_bulk_kernel(const uint8_t* __restrict__ res, const int64_t* __restrict__ offs, int32_t n, int32_t k,
                     int32_t alphabet, int32_t stride, uint16_t* __restrict__ out, int32_t* __restrict__ nk_out,
                     uint32_t* __restrict__ err) {
  extern __shared__ __align__(128) uint32_t hist2[];   // 2 x stride / 2 words
  const int words = stride >> 1;
  const int vec = words >> 2;
  const uint32_t row_bytes = (uint32_t)stride * 2u;
  int buf = 0;
  for (int64_t s = blockIdx.x; s < n; s += gridDim.x, buf ^= 1) {
    uint32_t* hist = hist2 + buf * words;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    uint4* h4 = reinterpret_cast<uint4*>(hist);
    for (int v = threadIdx.x; v < vec; v += blockDim.x) h4[v] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int64_t b = offs[s], e = offs[s + 1];
    const int64_t len = e - b;
    const int64_t nk = len >= k ? len - k + 1 : 0;
    const uint8_t* x = res + b;
    // every residue of a sequence with nk > 0 lies in some k-mer: the range
    // check rides on the k-mer reads (its own pass only when len < k)
    uint32_t bad = 0;
    if (nk == 0)
      for (int64_t u = threadIdx.x; u < len; u += blockDim.x)
        if (x[u] >= alphabet) bad = 1;
    for (int64_t u = threadIdx.x; u < nk; u += blockDim.x) {
      uint32_t id = 0;
      bool ok = true;
      for (int t = 0; t < k; ++t) {
        const uint32_t r = x[u + t];
        ok &= r < (uint32_t)alphabet;
        id = id * (uint32_t)alphabet + r;
      }
      if (ok) atomicAdd(&hist[id >> 1], 1u << ((id & 1u) << 4));
      else bad = 1;
    }
    if (bad) atomicOr(err, ERR_RESIDUE);
    if (threadIdx.x == 0) {
      if (nk > 65535) atomicOr(err, ERR_NK);
      nk_out[s] = (int32_t)nk;
    }
    // the histogram's generic-proxy writes before the async-proxy read
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(hist);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                   "cp.async.bulk.commit_group;"
                   :: "l"(out + s * (int64_t)stride), "r"(src), "r"(row_bytes) : "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

sa_status profiles_launch(const uint8_t* residues, const int64_t* offsets, int32_t n, int32_t k,
                          int32_t alphabet, int32_t stride, uint16_t* out, int32_t* nk, uint32_t* err_flag,
                          cudaStream_t st) {
  if (n <= 0) return SA_OK;
  const int smem = stride * 2;
  // both kernels may take up to 227 KB of dynamic shared memory (the attribute
  // is a per-device ceiling; each launch passes what it needs)
  static DeviceOnce once;
  SA_TRY(once.run([]() -> sa_status {
    SA_CUDA(cudaFuncSetAttribute(profiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    SA_CUDA(cudaFuncSetAttribute(profiles_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    return SA_OK;
  }));
  int dev = 0, sms = 0, per_sm = 0;
  SA_CUDA(cudaGetDevice(&dev));
  SA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, profiles_kernel, 256, smem));
  if (per_sm < 1) per_sm = 1;
  static const int cs = [] {   // streaming (evict-first) row stores unless SA_PROF_CS=0
    const char* e = getenv("SA_PROF_CS");
    return e ? atoi(e) : 1;
  }();
  static const int bulk = [] {   // SA_PROF_BULK=0: thread stores instead of bulk copies
    const char* e = getenv("SA_PROF_BULK");
    return e ? atoi(e) : 1;
  }();
  if (bulk && 2 * smem <= 227 * 1024) {   // two row buffers fit (bins <= 58 112)
    int per_sm_b = 0;
    SA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_b, profiles_bulk_kernel, 256, 2 * smem));
    if (per_sm_b < 1) per_sm_b = 1;
    const int64_t gb = (int64_t)sms * per_sm_b;
    profiles_bulk_kernel<<<(unsigned)(n < gb ? n : gb), 256, 2 * smem, st>>>(residues, offsets, n, k, alphabet, stride,
                                                                          out, nk, err_flag);
    SA_LAUNCHED();
    return SA_OK;
  }
  const int64_t grid = (int64_t)sms * per_sm;
  profiles_kernel<<<(unsigned)(n < grid ? n : grid), 256, smem, st>>>(residues, offsets, n, k, alphabet, stride, out,
                                                                     nk, err_flag, cs);
  SA_LAUNCHED();
  return SA_OK;
}

}  // namespace sa
