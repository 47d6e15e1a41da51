// libsa internal declarations shared by the .cu translation units.
// Product code only: nothing here is shared with oracle/ (DESIGN.md §1).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <string>
#include <chrono>
#include <vector>

#include "../../include/sa.h"

namespace sa {

// ------------------------------------------------------------- errors ----
void set_error(const char* fmt, ...);
sa_status fail(sa_status s, const char* fmt, ...);
void count_launch(int n = 1);

#define SA_CUDA(call)                                                                \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return ::sa::fail(SA_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,        \
                        cudaGetErrorString(e_));                                     \
  } while (0)

#define SA_TRY(expr)                 \
  do {                               \
    sa_status s_ = (expr);           \
    if (s_ != SA_OK) return s_;      \
  } while (0)

#define SA_LAUNCHED()                                                                \
  do {                                                                               \
    ::sa::count_launch();                                                            \
    cudaError_t e_ = cudaGetLastError();                                             \
    if (e_ != cudaSuccess)                                                           \
      return ::sa::fail(SA_E_CUDA, "%s:%d launch: %s", __FILE__, __LINE__,           \
                        cudaGetErrorString(e_));                                     \
  } while (0)

// Large scratch blocks kept by the library between calls (on by default;
// SA_SCRATCH_CACHE=0 turns it off).  The stream-ordered pool keeps freed memory too (release
// threshold, api.cu), but was seen to re-map a 328 MB block in the middle of a
// run (config 3, tenth timed step: cudaMallocAsync held the host 48-176 ms,
// DESIGN.md section 7).  A block returned here carries an event recorded on the
// stream that last used it; whoever takes it makes its stream wait on that
// event, so reuse is ordered after the earlier work on any stream.  Blocks are
// matched by exact size and device; the cache is bounded (count and bytes),
// the oldest block going back to the pool.
struct ScratchCache {
  struct Blk {
    void* p;
    size_t bytes;
    int dev;
    cudaEvent_t ev;
    cudaStream_t st;
  };
  static constexpr size_t MIN_BYTES = (size_t)1 << 20;
  static constexpr size_t MAX_BLOCKS = 96;
  static constexpr size_t MAX_BYTES = (size_t)24 << 30;
  std::mutex m;
  std::vector<Blk> blocks;
  size_t held = 0;
  static ScratchCache& get() {
    static ScratchCache c;
    return c;
  }
  static bool enabled() {
    static const bool on = [] {
      const char* e = getenv("SA_SCRATCH_CACHE");
      return !e || atoi(e) != 0;  // on unless SA_SCRATCH_CACHE=0
    }();
    return on;
  }
  void* take(size_t bytes, int dev, cudaStream_t st) {
    Blk b{};
    {
      std::lock_guard<std::mutex> g(m);
      size_t i = 0;
      for (; i < blocks.size(); ++i)
        if (blocks[i].bytes == bytes && blocks[i].dev == dev) break;
      if (i == blocks.size()) return nullptr;
      b = blocks[i];
      blocks.erase(blocks.begin() + (long)i);
      held -= b.bytes;
    }
    if (b.st != st) cudaStreamWaitEvent(st, b.ev, 0);
    cudaEventDestroy(b.ev);
    return b.p;
  }
  // every kept block back to the pool (an allocation failed: the memory may be needed elsewhere)
  bool flush(cudaStream_t st) {
    std::vector<Blk> drop;
    {
      std::lock_guard<std::mutex> g(m);
      drop.swap(blocks);
      held = 0;
    }
    for (const Blk& d : drop) {
      cudaStreamWaitEvent(st, d.ev, 0);
      cudaFreeAsync(d.p, st);
      cudaEventDestroy(d.ev);
    }
    return !drop.empty();
  }
  // false: not kept (the caller frees it)
  bool give(void* p, size_t bytes, int dev, cudaStream_t st) {
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, st) != cudaSuccess) {
      cudaGetLastError();
      if (ev) cudaEventDestroy(ev);
      return false;
    }
    std::vector<Blk> drop;
    {
      std::lock_guard<std::mutex> g(m);
      blocks.push_back(Blk{p, bytes, dev, ev, st});
      held += bytes;
      while (blocks.size() > MAX_BLOCKS || held > MAX_BYTES) {
        drop.push_back(blocks.front());
        held -= blocks.front().bytes;
        blocks.erase(blocks.begin());
      }
    }
    for (const Blk& d : drop) {   // back to the pool, after the work that last used it
      cudaStreamWaitEvent(st, d.ev, 0);
      cudaFreeAsync(d.p, st);
      cudaEventDestroy(d.ev);
    }
    return true;
  }
};

// Stream-ordered scratch: allocations are freed on the same stream when the
// Scratch goes out of scope, so kernels enqueued before still see them.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  std::vector<size_t> sizes;
  int dev = -1;
  bool oom = false;
  explicit Scratch(cudaStream_t s) : st(s) {
    if (ScratchCache::enabled() && cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      dev = -1;
    }
  }
  ~Scratch() {
    for (size_t i = 0; i < ptrs.size(); ++i) {
      if (dev >= 0 && sizes[i] >= ScratchCache::MIN_BYTES && ScratchCache::get().give(ptrs[i], sizes[i], dev, st))
        continue;
      cudaFreeAsync(ptrs[i], st);
    }
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
    if (dev >= 0 && bytes >= ScratchCache::MIN_BYTES && (p = ScratchCache::get().take(bytes, dev, st)) != nullptr) {
      ptrs.push_back(p);
      sizes.push_back(bytes);
      return static_cast<T*>(p);
    }
    // SA_TRACE_ALLOC=1 (diagnostics): report pool allocations that hold the host for more than 0.3 ms
    static const bool trace = [] {
      const char* e = getenv("SA_TRACE_ALLOC");
      return e && atoi(e) != 0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t rc = cudaMallocAsync(&p, bytes, st);
    if (rc != cudaSuccess && dev >= 0 && ScratchCache::get().flush(st)) {
      cudaGetLastError();
      rc = cudaMallocAsync(&p, bytes, st);
    }
    if (trace) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 0.3) fprintf(stderr, "[sa] cudaMallocAsync(%zu bytes) held the host %.2f ms\n", bytes, ms);
    }
    if (rc != cudaSuccess) {
      cudaGetLastError();
      oom = true;
      return nullptr;
    }
    ptrs.push_back(p);
    sizes.push_back(bytes);
    return static_cast<T*>(p);
  }
};

// One-time setup per (call site, device): kernel attributes
// (cudaFuncSetAttribute is per device) and device tables.  `f` runs under the
// site's mutex the first time a thread reaches the site with a given current
// device; concurrent contexts on several threads or devices are safe.
struct DeviceOnce {
  std::mutex m;
  bool done[64] = {};
  template <class F>
  sa_status run(F&& f) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      return fail(SA_E_CUDA, "cudaGetDevice failed");
    }
    std::lock_guard<std::mutex> g(m);
    if (dev < 64 && done[dev]) return SA_OK;
    const sa_status s = f();
    if (s == SA_OK && dev < 64) done[dev] = true;
    return s;
  }
};
// SM count of the current device (148 on B200).
inline int device_sms() {
  int dev = 0, s = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 148;
  }
  return s > 0 ? s : 148;
}

#define SA_ALLOC(var, T, n)                                                        \
  T* var = scratch.alloc<T>(n);                                                    \
  if (!var) return fail(SA_E_NOMEM, "scratch allocation of %zu x %s failed", (size_t)(n), #T)

// Error flags written by kernels (device-detected range errors).
enum : uint32_t { ERR_RESIDUE = 1u, ERR_NK = 2u };

// --------------------------------------------------- min-sum engine (K2) --
// Tile geometry: 128 x 128 pairs per CTA, 256 threads, 8 x 8 pairs per thread,
// 32 packed words (64 bins) per pipeline stage.
constexpr int MS_BM = 128;
constexpr int MS_THREADS = 256;
constexpr int MS_BKW = 32;
constexpr int MS_LDW = MS_BKW + 4;   // padded smem row (words): conflict-free LDS.128
constexpr int MS_STAGES = 4;
constexpr int MS_SMEM = MS_STAGES * 2 * MS_BM * MS_LDW * 4;

struct MsProblem {
  const uint32_t* A;       // packed u16x2 rows, stride ldw words
  const uint32_t* B;
  const int32_t* nkA;
  const int32_t* nkB;
  int32_t na, nb;
  int32_t sym;             // A == B: upper-triangle tiles only, mirrored outputs
  int32_t tiles_b;         // ceil(nb / 128)
  int64_t tile_begin;      // first global tile id of this problem
  sa_key128* keyA;         // row sums (nullable)
  sa_key128* keyB;         // column sums for sym off-diagonal tiles (nullable)
  uint16_t* num;           // [na][ld] numerators (nullable)
  double* sim;             // [na][ld] C/D (nullable)
  int64_t ld;
  int32_t form;            // SA_RANK_F: key += floor(C 2^64 / D); SA_RANK_DF: key += dF term (below)
  double delta;            // SA_RANK_DF: the Delta of Eq. 2
  double ln1pd;            // SA_RANK_DF: ln(1 + Delta) (host-computed)
};

// d^F key term (Eq. 2): round(2^52 (ln(1+Delta) - ln(Delta + F)))
// >= 0, so sum_j d^F(i, j) = key_i 2^-52 - npool ln(1+Delta).
constexpr double DF_SCALE = 4503599627370496.0;   // 2^52

// Profile encodings the engine reads:
//   ENC_U16_MIN       uint16 counts, 2 bins/word, VIMNMX.U16x2 + IADD3 (any count)
//   ENC_U16_MIN_IMAD  same, adds issued as IMAD on the FMA pipe (experiment)
//   ENC_U8_SAD        uint8 counts, 4 bins/word, C = (nk_a + nk_b - sum|a-b|)/2 with
//                     VABSDIFF4.U8.ACC (every count must be <= 255)
//   ENC_TC            0/1 threshold layers on the tensor cores (K2T, minsum_tc.cuh)
enum { ENC_U16_MIN = 0, ENC_U8_SAD = 1, ENC_U16_MIN_IMAD = 2, ENC_AUTO = 3, ENC_TC = 4 };
// Row strides: u16 rows are round_up(bins, 64) elements; u8 rows round_up(bins, 128) bytes.
inline int32_t stride_u16(int32_t bins) { return ((bins + 63) / 64) * 64; }
inline int32_t stride_u8(int32_t bins) { return ((bins + 127) / 128) * 128; }

// Launch the engine over `probs`; ldw = row stride in 32-bit words.
// guard (nullable): device counter holding the largest count; when set, the
// launch is a no-op on the device unless the counter selects `enc`.
sa_status minsum_launch(const std::vector<MsProblem>& probs, int ldw, int enc, cudaStream_t st,
                        cudaEvent_t ev0, cudaEvent_t ev1, const uint32_t* guard = nullptr);
// uint16 rows -> uint8 rows (zero padded) + atomicMax of every count into *maxc.
// guarded: skip when the tensor-core engine handled the call (maxc = guard words).
sa_status to_u8_launch(const uint16_t* p16, int64_t n, int32_t stride16, int32_t bins, uint8_t* p8,
                       int32_t stride8, uint32_t* maxc, cudaStream_t st, bool guarded = false);
// K2T: the tensor-core engine over `probs` (u16 operand rows, ldw16 words per
// row).  state = guard words [largest count, infeasible, enabled]; when the
// launch is infeasible (a count > 32 or too many layer columns) its kernels
// return at once and the guarded engines above must be enqueued after it.
// cols_out[i] (device, nullable) = kept layer columns K' of problem i (i < SA_TC_COLS_MAX).
constexpr int TC_MAX_BINS = 8192;
sa_status f_division_selftest(int64_t* mismatches_h);
// N4: UPGMA guide tree of an n x n similarity matrix (tree.cu)
// N4 distance form: SA_TREE_F (d = 1 - F) or SA_TREE_DF (d = CR(-ln(Delta + F)); uncertified
// correctly-rounded logs are counted into *unc)
struct TreeForm {
  int form = SA_TREE_F;
  double delta = 0.02;
  unsigned long long* unc = nullptr;
};
sa_status upgma_launch(const double* F, int32_t n, int64_t ld, int32_t* merges, double* heights, const TreeForm& tf,
                       cudaStream_t st);
sa_status upgma_launch_batch(int count, const double* const* F, const int32_t* n, const int64_t* ld,
                             int32_t* const* merges, double* const* heights, const TreeForm& tf, cudaStream_t st);
bool tc_fp4_operands();   // K2T operand format for the next launch: true = packed e2m1 (kind::mxf4), false = u8
bool tc_last_fp4();       // the format of the last K2T launch
// sim[i][j] = num[i][j] / min(nkA[i], nkB[j]) (fp64, IEEE RN; 0 when the min is 0), row stride ld.
sa_status ratio_launch(const uint16_t* num, const int32_t* nkA, const int32_t* nkB, int64_t na, int64_t nb,
                       int64_t ld, double* sim, cudaStream_t st, const uint32_t* state = nullptr);
constexpr int SA_STAGE_BYTES = 1 << 16;   // ctx->hstage: mapped pinned staging for d2h_small
// ctx->dcount: [0..3] guard words, [16..80) K2T column counts, [80..144) K2T
// sparse-layer mode per problem, [144..272) its correction terms (u64)
constexpr int SA_DCOUNT_WORDS = 512;
constexpr int SA_TC_COLS_AT = 16;
constexpr int SA_TC_COLS_MAX = 64;
constexpr int SA_TC_MODE_AT = 80;
constexpr int SA_TC_TERMS_AT = 144;
// Operand rows carried from one K2T launch to the next on the same u16 rows
// (sa_partition: S2a's blocks -> S2d's query side): the rows with their first
// dense layers already written and the OR of their seen-once planes.  The
// memory belongs to the caller's Scratch (it must outlive both launches).
struct TcCarry {
  Scratch* scratch = nullptr;        // where a keeping launch allocates (nullptr: nothing kept)
  bool valid = false;
  const uint32_t* src = nullptr;     // first u16 row they were built from
  int64_t nrows = 0;
  bool fp4 = false;
  uint8_t* rows = nullptr;           // [nrows][row bytes]
  uint32_t* seen1 = nullptr;         // seen-once planes (one plane, all layers)
  int32_t* ndense = nullptr;         // [np] dense layers each problem of the building launch kept
  int np = 0;
  uint32_t* masks = nullptr;         // [nrows][2][256] layer-2 / layer-3 masks (minsum_tc.cu TcMasks)
  int masks_valid = 1;               // its histogram pass wrote the layer masks
  int spec = 2;                      // dense layers its histogram pass wrote
  const uint2* recs = nullptr;       // its sparse-layer records (tc_sparse.cuh), nullptr when off
  const uint32_t* nrec = nullptr;
  uint32_t rec_cap = 0;
};
sa_status tc_launch(const std::vector<MsProblem>& probs, int ldw16, int32_t bins, uint32_t* state,
                    uint32_t* cols_out, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1,
                    TcCarry* keep = nullptr, const TcCarry* use = nullptr);
sa_status ensure_recip_tables(cudaStream_t st);

// ------------------------------------------------------ profiles (K1) --
sa_status profiles_launch(const uint8_t* residues, const int64_t* offsets, int32_t n, int32_t k,
                          int32_t alphabet, int32_t stride, uint16_t* out, int32_t* nk,
                          uint32_t* err_flag, cudaStream_t st);

// ---------------------------------------------------- ordering (K4-K6) --
// Sort each segment [seg[s], seg[s+1]) of `keys` by (key, gid) ascending
// where gid = gid0 + local index.  order_out[seg[s] + pos] = local index.
// amb[i] = 1 if item i has another item of its segment within `window` of
// its key (the key order is then not certified); *amb_count += flagged.
sa_status segment_sort_launch(const sa_key128* keys, int64_t gid0, const int64_t* seg_h, int nseg,
                              int64_t window, int32_t* order_out, uint8_t* amb, uint32_t* amb_count,
                              cudaStream_t st);
// Sort records (pivot candidates) by (key, global_idx): same contract.
sa_status record_sort_launch(const sa_pivot* rec, int n, int64_t window, int32_t* order_out,
                             uint8_t* amb, uint32_t* amb_count, cudaStream_t st);

double u128_to_double_host(uint64_t hi, uint64_t lo);

// keys -> fp64 ranks: RN(key) * 2^-64 / npool (F form) or
// RN(key) * 2^-52 / npool - ln(1+Delta) (d^F form).
sa_status keys_to_f64_launch(const sa_key128* keys, int64_t n, int64_t npool, double* out,
                             cudaStream_t st, int form = SA_RANK_F, double ln1pd = 0.0);

// ---------------------------------------------------- exact fallback ----
// Exact comparison of V_a = sum_j Ca_j / Da_j and V_b (rows over the same
// pool, D = min(nk_query, nk_j)).  Returns -1, 0, +1.
int exact_compare(const uint16_t* Ca, int32_t nka, const uint16_t* Cb, int32_t nkb,
                  const int32_t* nk_pool, int npool);

}  // namespace sa

struct sa_ctx {
  int device = 0;
  int nranks = 1;
  int rank = 0;
  sa_comm_ops comm{};
  bool has_comm = false;        // callbacks attached (sa_ctx_attach_comm)
  void* nccl = nullptr;         // libsa's own NCCL communicator (sa_ctx_attach_nccl)
  uint32_t* derr = nullptr;     // device: sticky error flags of the asynchronous calls (ERR_*)
  bool timing = false;
  // phase events: a ring of SA_PHASE_RING (begin, end) pairs per phase,
  // created on first use; ev_count = occurrences recorded, ev_cur = last slot
  cudaEvent_t ev[SA_PHASE_COUNT][SA_PHASE_RING][2] = {};
  int64_t ev_count[SA_PHASE_COUNT] = {};
  int ev_cur[SA_PHASE_COUNT] = {};
  int last_gemm_phase = -1;     // the specific phase of the last K2T GEMM record
  int last_enc = -1;            // ENC_* of the last min-sum call, or ENC_AUTO
  bool last_tc = false;         // the last auto call tried the tensor-core engine first
  int last_tc_probs = 0;        // problems of that K2T call
  int rank_form = SA_RANK_F;    // sa_ctx_set_rank_form
  double delta = 0.02;
  int tree_form = SA_TREE_F;    // sa_ctx_set_tree_form
  double tree_delta = 0.02;
  unsigned long long* tree_unc = nullptr;   // device (inside derr's block): uncertified d^F logs of the last tree call
  uint32_t* dcount = nullptr;   // device: largest count of the last auto-dispatched call
  uint32_t* hpinned = nullptr;  // pinned host word for small readbacks
  // mapped pinned staging for the hot path's small readbacks (d2h_small): a
  // kernel stores into it over PCIe, so the read never queues on the copy
  // engine behind a caller's large device-to-host copies
  uint8_t* hstage = nullptr;
  uint8_t* dstage = nullptr;
};
