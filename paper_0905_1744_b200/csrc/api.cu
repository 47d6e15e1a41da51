// libsa C ABI (include/sa.h): context, S1 profiles, S2 rank, S2-S3 partition,
// S4 redistribution, S5 bucket similarity.  Host orchestration of the kernels
// in profiles.cu / minsum.cu / order.cu; collectives through the caller's
// sa_comm_ops (torch.distributed / NCCL in the Python binding).
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "comm.h"

namespace sa {

// ------------------------------------------------------------- errors ----
static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}
sa_status fail(sa_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
void count_launch(int n) { g_launches += n; }

// ---------------------------------------------------- order.cu exports ----
sa_status segment_sort_keys(const sa_key128* keys, int64_t gid0, int64_t N, int64_t P, int64_t q0, int64_t base,
                            int nseg, int64_t window, int32_t* order_out, uint8_t* amb, uint32_t* amb_count,
                            cudaStream_t st);
sa_status sort_records(const sa_pivot* rec, int n, int64_t window, sa_key128* tmp_keys, int64_t* tmp_gid,
                       int32_t* order_out, uint8_t* amb, uint32_t* amb_count, cudaStream_t st);
sa_status pick_launch(const int32_t* order, int64_t N, int64_t P, int64_t q0, int64_t base, int nseg, int count,
                      int den, int64_t gid0, int64_t* out_gid, int32_t* out_local, cudaStream_t st);
sa_status gather_rows_launch(const uint16_t* prof, const int32_t* nk, const int32_t* sel, int nsel, int stride,
                             uint16_t* out, int32_t* out_nk, cudaStream_t st);
sa_status make_records_launch(const int32_t* local, const int64_t* gid, int n, const sa_key128* keys,
                              const int32_t* nk, int count, int q0, sa_pivot* rec, cudaStream_t st);
sa_status pivots_launch(const sa_pivot* rec, const int32_t* order, int n, int p, int64_t* y_sorted_gid,
                        sa_pivot* pivots, cudaStream_t st);
sa_status assign_launch(const sa_key128* keys, int64_t gid0, int n, const sa_pivot* pivots, int p, int64_t window,
                        const int64_t* offs, int32_t* bucket_of, uint8_t* amb, uint32_t* amb_count,
                        unsigned long long* counts, unsigned long long* bytes, cudaStream_t st);
sa_status scan_launch(const int64_t* in, int64_t n, int64_t* out, int64_t* part, cudaStream_t st);
sa_status bucket_perm_launch(const int32_t* bucket_of, int n, int p, int32_t* hist, int64_t* base, int32_t* perm,
                             cudaStream_t st);
sa_status perm_meta_launch(const int32_t* perm, int n, const int64_t* offs, const int32_t* bucket_of, int64_t gid0,
                           int64_t* lens, int64_t* gid_out, int32_t* bkt_out, cudaStream_t st);
sa_status copy_seqs_launch(const int32_t* perm, int n, const uint8_t* src, const int64_t* soff, uint8_t* dst,
                           const int64_t* doff, cudaStream_t st);
sa_status pack_meta_launch(const int32_t* perm, int n, const int64_t* offs, const int32_t* bucket_of, int64_t gid0,
                           int64_t* meta, cudaStream_t st);
sa_status unpack_meta_launch(const int64_t* meta, int n, int64_t* gid, int64_t* lens, int32_t* bkt, cudaStream_t st);
sa_status seg_copy_launch(const void* segs_dev, int nseg, const int64_t* meta_in, int64_t* meta_out,
                          const uint8_t* res_in, uint8_t* res_out, cudaStream_t st);
size_t segcopy_size();
void segcopy_fill(void* dst, int t, int64_t src_m, int64_t dst_m, int64_t cnt, int64_t src_r, int64_t dst_r,
                  int64_t nbytes);

// ---------------------------------------------------------- scratch ------
static inline int64_t block_begin(int64_t q, int64_t N, int64_t p) { return q * N / p; }

static int32_t profile_stride(int32_t bins) { return stride_u16(bins); }

// tree form of the context (sa_ctx_set_tree_form)
static inline TreeForm tree_form_of(const sa_ctx* c) {
  TreeForm t;
  t.form = c->tree_form;
  t.delta = c->tree_delta;
  t.unc = c->tree_unc;
  return t;
}

// rank form of the context onto a key-producing problem (sa_ctx_set_rank_form)
static inline void apply_form(const sa_ctx* c, MsProblem& pr) {
  pr.form = c->rank_form;
  pr.delta = c->delta;
  pr.ln1pd = std::log1p(c->delta);
}
// key distance below which an order is not certified: npool for exact F keys
// (2^64 V - npool < key <= 2^64 V); 32 npool for d^F keys (per-term log and
// rounding error <= 16 units of 2^-52 on either side, DESIGN.md §2 N1)
static inline int64_t window_of(const sa_ctx* c, int64_t npool) {
  return c->rank_form == SA_RANK_DF ? 32 * npool : npool;
}

// Engine choice: SA_ENGINE = auto | tc (default: the tensor-core engine K2T
// when the launch is feasible, else the u8 SAD engine when every count is
// <= 255, else u16) | sad / u8 (the same without K2T) | u16 | u16imad (forced).
struct EngineMode {
  int enc;    // ENC_AUTO or a forced ENC_*
  bool tc;    // auto mode: try K2T first
};
static EngineMode engine_mode() {
  const char* e = getenv("SA_ENGINE");
  if (!e || !*e || !strcmp(e, "auto") || !strcmp(e, "tc")) return {ENC_AUTO, true};
  if (!strcmp(e, "sad") || !strcmp(e, "u8")) return {ENC_AUTO, false};
  if (!strcmp(e, "u16imad")) return {ENC_U16_MIN_IMAD, false};
  return {ENC_U16_MIN, false};
}

// Operand rows the min-sum engine reads for a set of u16 profile rows.
struct Operand {
  const uint32_t* rows;
  int ldw;   // row stride in 32-bit words
};

// Engine operands of an A x B min-sum problem given its u16 profile rows.  In
// the auto modes every encoding is prepared and the choice is made on the
// device, with no host synchronisation: K2T's own kernels decide whether the
// launch fits it (minsum_tc.cuh), the u8 SAD rows are converted on the device
// and the largest count is folded into ctx->dcount, and launch_ops enqueues
// every engine, each guarded by those words.  With K2T the u8 conversions are
// deferred to launch_ops and guarded too (they are only read by the fallback).
struct EngineOps {
  Operand a16, b16, a8, b8;
  int mode;                     // ENC_U16_MIN / ENC_U16_MIN_IMAD (forced) or ENC_AUTO
  bool tc = false;              // auto mode: K2T first
  int32_t bins = 0;
  uint32_t* guard = nullptr;
  struct Conv {
    const uint16_t* p16;
    int64_t n;
    uint8_t* p8;
  };
  std::vector<Conv> conv;       // deferred (guarded) u8 conversions
};

// Build the u8 (SAD) operand rows of `n` u16 profile rows in scratch memory and
// fold the largest count into *maxc (device); with K2T the conversion is only
// recorded in E->conv.
static sa_status make_u8_rows(Scratch& scratch, const uint16_t* p16, int64_t n, int32_t bins, uint32_t* maxc,
                              Operand* out, cudaStream_t st, EngineOps* E) {
  const int32_t s8 = stride_u8(bins);
  uint8_t* p8 = scratch.alloc<uint8_t>((size_t)std::max<int64_t>(n, 1) * s8);
  if (!p8) return fail(SA_E_NOMEM, "scratch allocation of u8 operand rows failed");
  if (E && E->tc) E->conv.push_back({p16, n, p8});
  else SA_TRY(to_u8_launch(p16, n, stride_u16(bins), bins, p8, s8, maxc, st));
  out->rows = reinterpret_cast<const uint32_t*>(p8);
  out->ldw = s8 / 4;
  return SA_OK;
}

static sa_status prepare_ops(sa_ctx* c, Scratch& scratch, const uint16_t* A16, int64_t na, const uint16_t* B16,
                             int64_t nb, int32_t bins, bool reset_count, EngineOps* E, cudaStream_t st) {
  const int ldw16 = stride_u16(bins) / 2;
  E->a16 = Operand{reinterpret_cast<const uint32_t*>(A16), ldw16};
  E->b16 = Operand{reinterpret_cast<const uint32_t*>(B16), ldw16};
  E->bins = bins;
  const EngineMode m = engine_mode();
  if (m.enc != ENC_AUTO) {
    E->mode = m.enc;
    return SA_OK;
  }
  E->mode = ENC_AUTO;
  E->tc = m.tc && bins <= TC_MAX_BINS;
  E->guard = c->dcount;
  if (reset_count) SA_CUDA(cudaMemsetAsync(c->dcount, 0, 4 * sizeof(uint32_t), st));
  if (B16 == A16) {   // same rows (possibly different counts): convert the longer prefix once
    SA_TRY(make_u8_rows(scratch, A16, std::max(na, nb), bins, c->dcount, &E->a8, st, E));
    E->b8 = E->a8;
  } else {
    SA_TRY(make_u8_rows(scratch, A16, na, bins, c->dcount, &E->a8, st, E));
    SA_TRY(make_u8_rows(scratch, B16, nb, bins, c->dcount, &E->b8, st, E));
  }
  return SA_OK;
}

// packed upper triangle: one CTA per row, coalesced row-segment copy
template <class T>
__global__ void pack_upper_kernel(const T* __restrict__ m, int32_t n, int64_t ld, T* __restrict__ out) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const T* src = m + i * ld;
    T* dst = out + i * (int64_t)n - i * (i - 1) / 2 - i;   // = i*n - i*(i+1)/2, then column j at + j
    for (int64_t j = i + threadIdx.x; j < n; j += blockDim.x) dst[j] = src[j];
  }
}

static inline cudaEvent_t ev_begin(sa_ctx* c, int ph);
static inline cudaEvent_t ev_end(sa_ctx* c, int ph);

// Enqueue the problems (A / B pointers given into the u16 operands).
static sa_status launch_ops(sa_ctx* c, const EngineOps& E, const std::vector<MsProblem>& probs16, cudaStream_t st,
                            cudaEvent_t ev0, cudaEvent_t ev1, int gemm_phase, TcCarry* keep = nullptr,
                            const TcCarry* use = nullptr) {
  c->last_enc = E.mode;
  c->last_tc = E.tc;
  c->last_tc_probs = 0;
  if (E.mode != ENC_AUTO) return minsum_launch(probs16, E.a16.ldw, E.mode, st, ev0, ev1);
  if (ev0) SA_CUDA(cudaEventRecord(ev0, st));
  SA_CUDA(cudaMemsetAsync(E.guard + 2, E.tc ? 1 : 0, sizeof(uint32_t), st));
  if (E.tc) {
    c->last_tc_probs = (int)probs16.size();
    cudaEvent_t g0 = ev_begin(c, gemm_phase);
    cudaEvent_t g1 = ev_end(c, gemm_phase);
    if (g0) c->last_gemm_phase = gemm_phase;
    SA_TRY(tc_launch(probs16, E.a16.ldw, E.bins, E.guard, E.guard + SA_TC_COLS_AT, st, g0, g1, keep, use));
    for (const auto& cv : E.conv)
      SA_TRY(to_u8_launch(cv.p16, cv.n, stride_u16(E.bins), E.bins, cv.p8, stride_u8(E.bins), E.guard, st, true));
  }
  std::vector<MsProblem> p8 = probs16;
  for (auto& p : p8) {
    const int64_t ra = (p.A - E.a16.rows) / E.a16.ldw, rb = (p.B - E.b16.rows) / E.b16.ldw;
    p.A = E.a8.rows + ra * E.a8.ldw;
    p.B = E.b8.rows + rb * E.b8.ldw;
  }
  SA_TRY(minsum_launch(p8, E.a8.ldw, ENC_U8_SAD, st, nullptr, nullptr, E.guard));
  SA_TRY(minsum_launch(probs16, E.a16.ldw, ENC_U16_MIN, st, nullptr, nullptr, E.guard));
  if (ev1) SA_CUDA(cudaEventRecord(ev1, st));
  return SA_OK;
}

}  // namespace sa

using namespace sa;

// ============================================================= context ====
extern "C" {

const char* sa_last_error(void) { return g_err.c_str(); }
int64_t sa_launch_count(void) { return g_launches.load(); }
int32_t sa_profile_stride(int32_t bins) { return profile_stride(bins); }

int sa_exact_rank_compare(const uint16_t* Ca_h, int32_t nka, const uint16_t* Cb_h, int32_t nkb,
                          const int32_t* nk_pool_h, int32_t npool) {
  if (npool <= 0 || !Ca_h || !Cb_h || !nk_pool_h) return 0;
  return exact_compare(Ca_h, nka, Cb_h, nkb, nk_pool_h, npool);
}

sa_status sa_ctx_create(int cuda_device, sa_ctx** out) {
  g_err.clear();
  if (!out) return fail(SA_E_INVAL, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SA_E_CUDA, "no CUDA device available (%s); libsa has no CPU fallback",
                e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  }
  if (cuda_device < 0 || cuda_device >= ndev) return fail(SA_E_INVAL, "device %d out of range", cuda_device);
  SA_CUDA(cudaSetDevice(cuda_device));
  cudaDeviceProp prop;
  SA_CUDA(cudaGetDeviceProperties(&prop, cuda_device));
  if (prop.major != 10) return fail(SA_E_CUDA, "libsa is built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
  // Scratch comes from the device's stream-ordered pool; keep freed memory in
  // the pool instead of returning it to the driver at every synchronisation,
  // so steady-state calls never re-map device memory.
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  sa_ctx* c = new sa_ctx();
  c->device = cuda_device;
  if (cudaMalloc(&c->dcount, SA_DCOUNT_WORDS * 4) != cudaSuccess || cudaMalloc(&c->derr, 32) != cudaSuccess ||
      cudaMemset(c->derr, 0, 32) != cudaSuccess ||
      cudaHostAlloc(&c->hpinned, SA_DCOUNT_WORDS * 4, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(&c->hstage, SA_STAGE_BYTES, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dstage), c->hstage, 0) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return fail(SA_E_NOMEM, "context allocation failed");
  }
  c->tree_unc = reinterpret_cast<unsigned long long*>(c->derr + 4);
  *out = c;
  return SA_OK;
}

sa_status sa_ctx_attach_comm(sa_ctx* ctx, const sa_comm_ops* ops, int nranks, int rank) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SA_E_INVAL, "bad nranks/rank %d/%d", nranks, rank);
  if (nranks > 1 && (!ops || !ops->allgather || !ops->alltoallv))
    return fail(SA_E_INVAL, "nranks > 1 needs allgather and alltoallv callbacks");
  ctx->nranks = nranks;
  ctx->rank = rank;
  // attached callbacks are used even for one rank (exercises the collective
  // path end to end, e.g. a 1-rank NCCL group); without them, exchanges are
  // local copies
  ctx->has_comm = ops && ops->allgather && ops->alltoallv;
  if (ops) ctx->comm = *ops;
  return SA_OK;
}

sa_status sa_nccl_unique_id(void* id_h) {
  g_err.clear();
  if (!id_h) return fail(SA_E_INVAL, "id_h is NULL");
  return nccl_unique_id(id_h);
}

sa_status sa_ctx_attach_nccl(sa_ctx* ctx, const void* id_h, int nranks, int rank) {
  g_err.clear();
  if (!ctx || !id_h) return fail(SA_E_INVAL, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SA_E_INVAL, "bad nranks/rank %d/%d", nranks, rank);
  if (ctx->nccl) return fail(SA_E_STATE, "an NCCL communicator is already attached");
  SA_CUDA(cudaSetDevice(ctx->device));
  void* comm = nullptr;
  SA_TRY(nccl_init(&comm, id_h, nranks, rank));
  ctx->nccl = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->has_comm = false;   // the NCCL communicator takes precedence over callbacks
  return SA_OK;
}

sa_status sa_ctx_check(sa_ctx* ctx, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  SA_CUDA(cudaSetDevice(ctx->device));
  SA_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  uint32_t h = 0;
  SA_CUDA(cudaMemcpy(&h, ctx->derr, 4, cudaMemcpyDeviceToHost));
  if (h) SA_CUDA(cudaMemset(ctx->derr, 0, 4));
  if (ctx->nccl) SA_TRY(nccl_check(ctx->nccl));
  if (h & ERR_RESIDUE) return fail(SA_E_RANGE, "residue outside the alphabet (detected by sa_kmer_profiles)");
  if (h & ERR_NK) return fail(SA_E_RANGE, "a sequence has more than 65535 k-mers (detected by sa_kmer_profiles)");
  return SA_OK;
}

sa_status sa_ctx_destroy(sa_ctx* ctx) {
  if (!ctx) return SA_OK;
  cudaSetDevice(ctx->device);
  for (int i = 0; i < SA_PHASE_COUNT; ++i)
    for (int j = 0; j < SA_PHASE_RING; ++j)
      for (int b = 0; b < 2; ++b)
        if (ctx->ev[i][j][b]) cudaEventDestroy(ctx->ev[i][j][b]);
  if (ctx->nccl) nccl_destroy(ctx->nccl);
  if (ctx->dcount) cudaFree(ctx->dcount);
  if (ctx->derr) cudaFree(ctx->derr);
  if (ctx->hpinned) cudaFreeHost(ctx->hpinned);
  if (ctx->hstage) cudaFreeHost(ctx->hstage);
  delete ctx;
  return SA_OK;
}

sa_status sa_ctx_set_tree_form(sa_ctx* ctx, int form, double delta) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (form != SA_TREE_F && form != SA_TREE_DF) return fail(SA_E_INVAL, "unknown tree form %d", form);
  if (form == SA_TREE_DF && !(delta > 0.0 && std::isfinite(delta))) return fail(SA_E_INVAL, "Delta must be > 0");
  ctx->tree_form = form;
  if (form == SA_TREE_DF) ctx->tree_delta = delta;
  return SA_OK;
}

sa_status sa_ctx_tree_uncertified(sa_ctx* ctx, int64_t* count_h, void* stream) {
  g_err.clear();
  if (!ctx || !count_h) return fail(SA_E_INVAL, "NULL argument");
  SA_CUDA(cudaSetDevice(ctx->device));
  unsigned long long v = 0;
  SA_CUDA(cudaMemcpyAsync(&v, ctx->tree_unc, sizeof v, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  SA_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  *count_h = (int64_t)v;
  return SA_OK;
}

sa_status sa_ctx_set_rank_form(sa_ctx* ctx, int form, double delta) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (form != SA_RANK_F && form != SA_RANK_DF) return fail(SA_E_INVAL, "unknown rank form %d", form);
  if (form == SA_RANK_DF && !(delta > 0.0 && std::isfinite(delta))) return fail(SA_E_INVAL, "Delta must be > 0");
  ctx->rank_form = form;
  if (form == SA_RANK_DF) ctx->delta = delta;
  return SA_OK;
}

int sa_ctx_engine(const sa_ctx* ctx) {
  if (!ctx) return -1;
  if (ctx->last_enc != ENC_AUTO) return ctx->last_enc;
  // auto dispatch: the device words decided (blocking read)
  if (cudaSetDevice(ctx->device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(ctx->hpinned, ctx->dcount, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  if (ctx->hpinned[2] && !ctx->hpinned[1]) return ENC_TC;
  return ctx->hpinned[0] <= 255 ? ENC_U8_SAD : ENC_U16_MIN;
}

int sa_ctx_tc_operand(const sa_ctx* ctx) {
  if (!ctx || !ctx->last_tc) return -1;
  return tc_last_fp4() ? 1 : 0;
}

int32_t sa_ctx_tc_columns(const sa_ctx* ctx, int32_t* cols_h, int32_t max) {
  if (!ctx || !ctx->last_tc || ctx->last_tc_probs <= 0) return 0;
  if (cudaSetDevice(ctx->device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(ctx->hpinned, ctx->dcount, SA_DCOUNT_WORDS * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  if (!(ctx->hpinned[2] && !ctx->hpinned[1])) return 0;   // K2T declined: a fallback engine ran
  const int n = std::min(ctx->last_tc_probs, SA_TC_COLS_MAX);
  for (int i = 0; i < n && i < max; ++i) cols_h[i] = (int32_t)ctx->hpinned[SA_TC_COLS_AT + i];
  return n;
}

int32_t sa_ctx_tc_sparse(const sa_ctx* ctx, int32_t* mode_h, int64_t* terms_h, int32_t max) {
  if (!ctx || !mode_h || !ctx->last_tc || ctx->last_tc_probs <= 0) return 0;
  if (cudaSetDevice(ctx->device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(ctx->hpinned, ctx->dcount, SA_DCOUNT_WORDS * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  if (!(ctx->hpinned[2] && !ctx->hpinned[1])) return 0;   // K2T declined: a fallback engine ran
  const int n = std::min(ctx->last_tc_probs, SA_TC_COLS_MAX);
  for (int i = 0; i < n && i < max; ++i) {
    mode_h[i] = (int32_t)ctx->hpinned[SA_TC_MODE_AT + i];
    if (terms_h) {
      uint64_t t = 0;
      std::memcpy(&t, &ctx->hpinned[SA_TC_TERMS_AT + 2 * i], 8);
      terms_h[i] = (int64_t)t;
    }
  }
  return std::min(n, max);
}

sa_status sa_selftest_f_division(int32_t cuda_device, int64_t* mismatches_h) {
  g_err.clear();
  if (!mismatches_h) return fail(SA_E_INVAL, "NULL argument");
  SA_CUDA(cudaSetDevice(cuda_device));
  return f_division_selftest(mismatches_h);
}

sa_status sa_ctx_set_timing(sa_ctx* ctx, int enable) {
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  ctx->timing = enable != 0;
  for (int i = 0; i < SA_PHASE_COUNT; ++i) ctx->ev_count[i] = 0;
  ctx->last_gemm_phase = -1;
  return SA_OK;
}

static sa_status phase_slot_ms(sa_ctx* ctx, int ph, int slot, float* ms) {
  SA_CUDA(cudaEventSynchronize(ctx->ev[ph][slot][1]));
  SA_CUDA(cudaEventElapsedTime(ms, ctx->ev[ph][slot][0], ctx->ev[ph][slot][1]));
  return SA_OK;
}

sa_status sa_ctx_phase_ms(sa_ctx* ctx, float* ms_h) {
  g_err.clear();
  if (!ctx || !ms_h) return fail(SA_E_INVAL, "NULL argument");
  SA_CUDA(cudaSetDevice(ctx->device));
  for (int i = 0; i < SA_PHASE_COUNT; ++i) {
    ms_h[i] = 0.f;
    int ph = i;
    if (i == SA_PHASE_GEMM && ctx->last_gemm_phase >= 0) ph = ctx->last_gemm_phase;   // the last K2T GEMM of any call
    if (ctx->ev_count[ph] == 0) continue;
    SA_TRY(phase_slot_ms(ctx, ph, ctx->ev_cur[ph], &ms_h[i]));
  }
  return SA_OK;
}

int32_t sa_ctx_phase_history(sa_ctx* ctx, int32_t phase, float* ms_h, int32_t max) {
  g_err.clear();
  if (!ctx || !ms_h || phase < 0 || phase >= SA_PHASE_COUNT || max < 0) {
    fail(SA_E_INVAL, "bad argument");
    return -1;
  }
  if (cudaSetDevice(ctx->device) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  const int64_t cnt = ctx->ev_count[phase];
  const int n = (int)std::min<int64_t>(std::min<int64_t>(cnt, SA_PHASE_RING), max);
  for (int t = 0; t < n; ++t) {
    const int64_t occ = cnt - n + t;   // oldest kept first
    if (phase_slot_ms(ctx, phase, (int)(occ % SA_PHASE_RING), &ms_h[t]) != SA_OK) return -1;
  }
  return n;
}

}  // extern "C"

namespace sa {
// A new occurrence of phase ph: its begin event (nullptr when timing is off or
// the events cannot be created).  ev_end returns the end event of the same
// occurrence, so call ev_begin first.
static inline cudaEvent_t ev_begin(sa_ctx* c, int ph) {
  if (!c->timing) return nullptr;
  const int slot = (int)(c->ev_count[ph] % SA_PHASE_RING);
  for (int b = 0; b < 2; ++b)
    if (!c->ev[ph][slot][b] && cudaEventCreate(&c->ev[ph][slot][b]) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  c->ev_cur[ph] = slot;
  ++c->ev_count[ph];
  return c->ev[ph][slot][0];
}
static inline cudaEvent_t ev_end(sa_ctx* c, int ph) {
  return c->timing && c->ev_count[ph] > 0 ? c->ev[ph][c->ev_cur[ph]][1] : nullptr;
}
static inline sa_status rec(cudaEvent_t e, cudaStream_t st) {
  if (e) SA_CUDA(cudaEventRecord(e, st));
  return SA_OK;
}

static sa_status comm_allgather(sa_ctx* c, const void* send, void* recv, int64_t bytes, cudaStream_t st) {
  if (c->nccl) return nccl_allgather(c->nccl, send, recv, bytes, st);
  if (!c->has_comm) {
    if (send != recv && bytes > 0) SA_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
    return SA_OK;
  }
  if (c->comm.allgather(c->comm.user, send, recv, bytes, (void*)st) != 0)
    return fail(SA_E_COMM, "allgather callback failed (%lld bytes)", (long long)bytes);
  return SA_OK;
}

// numerator rows of selected query rows against a pool, to the host (exact path)
static sa_status numerator_rows_host(const uint16_t* prof, const int32_t* nk, const std::vector<int32_t>& rows,
                                     const uint16_t* pool, const int32_t* pool_nk, int npool, int stride,
                                     std::vector<uint16_t>& out, cudaStream_t st) {
  const int nq = (int)rows.size();
  out.assign((size_t)nq * npool, 0);
  if (nq == 0 || npool == 0) return SA_OK;
  Scratch scratch(st);
  SA_ALLOC(sel, int32_t, nq);
  SA_ALLOC(qp, uint16_t, (size_t)nq * stride);
  SA_ALLOC(qn, int32_t, nq);
  SA_ALLOC(num, uint16_t, (size_t)nq * npool);
  SA_CUDA(cudaMemcpyAsync(sel, rows.data(), nq * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  SA_TRY(gather_rows_launch(prof, nk, sel, nq, stride, qp, qn, st));
  MsProblem pr{};
  pr.A = reinterpret_cast<const uint32_t*>(qp);
  pr.B = reinterpret_cast<const uint32_t*>(pool);
  pr.nkA = qn;
  pr.nkB = pool_nk;
  pr.na = nq;
  pr.nb = npool;
  pr.sym = 0;
  pr.num = num;
  pr.ld = npool;
  SA_TRY(minsum_launch({pr}, stride / 2, ENC_U16_MIN, st, nullptr, nullptr));
  SA_CUDA(cudaMemcpyAsync(out.data(), num, out.size() * sizeof(uint16_t), cudaMemcpyDeviceToHost, st));
  SA_CUDA(cudaStreamSynchronize(st));
  return SA_OK;
}

static inline bool host_key_lt(const sa_key128& a, int64_t ga, const sa_key128& b, int64_t gb) {
  if (a.hi != b.hi) return a.hi < b.hi;
  if (a.lo != b.lo) return a.lo < b.lo;
  return ga < gb;
}
static inline bool host_key_near(const sa_key128& a, const sa_key128& b, int64_t window) {
  unsigned __int128 x = ((unsigned __int128)a.hi << 64) | a.lo, y = ((unsigned __int128)b.hi << 64) | b.lo;
  unsigned __int128 d = x >= y ? x - y : y - x;
  return d < (unsigned __int128)(uint64_t)window;
}

// Exact re-sort of the uncertified runs of each segment of a device order
// array (exact path).  Segments follow the block layout; the pool of segment s
// is either its own block (pool_is_block) or the shared pool (pool/pool_nk).
static sa_status resolve_segments(sa_ctx* c, const sa_key128* keys_d, int32_t* order_d, int64_t n_local,
                                  int64_t N, int64_t p, int64_t q0, int64_t first_global, int nseg, int64_t window,
                                  const uint16_t* prof, const int32_t* nk, int stride, bool pool_is_block,
                                  const uint16_t* pool, const int32_t* pool_nk, int npool, int* resolved,
                                  cudaStream_t st) {
  std::vector<sa_key128> keys(n_local);
  std::vector<int32_t> order(n_local);
  std::vector<int32_t> nk_h(n_local);
  SA_CUDA(cudaMemcpyAsync(keys.data(), keys_d, n_local * sizeof(sa_key128), cudaMemcpyDeviceToHost, st));
  SA_CUDA(cudaMemcpyAsync(order.data(), order_d, n_local * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SA_CUDA(cudaMemcpyAsync(nk_h.data(), nk, n_local * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> pool_nk_h;
  if (!pool_is_block) {
    pool_nk_h.resize(npool);
    SA_CUDA(cudaMemcpyAsync(pool_nk_h.data(), pool_nk, npool * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  SA_CUDA(cudaStreamSynchronize(st));
  bool changed = false;
  for (int s = 0; s < nseg; ++s) {
    const int64_t b = block_begin(q0 + s, N, p) - first_global, e = block_begin(q0 + s + 1, N, p) - first_global;
    int64_t pos = b;
    while (pos < e) {
      int64_t end = pos + 1;
      while (end < e && host_key_near(keys[b + order[end - 1]], keys[b + order[end]], window)) ++end;
      if (end - pos >= 2) {
        // run [pos, end): exact sort of these members
        std::vector<int32_t> rows;
        for (int64_t t = pos; t < end; ++t) rows.push_back((int32_t)(b + order[t]));
        std::vector<uint16_t> C;
        const uint16_t* pl = pool_is_block ? prof + b * stride : pool;
        const int32_t* pn = pool_is_block ? nk + b : pool_nk;
        const int np = pool_is_block ? (int)(e - b) : npool;
        SA_TRY(numerator_rows_host(prof, nk, rows, pl, pn, np, stride, C, st));
        std::vector<int32_t> pnh;
        if (pool_is_block) pnh.assign(nk_h.begin() + b, nk_h.begin() + e);
        const int32_t* pnk = pool_is_block ? pnh.data() : pool_nk_h.data();
        std::vector<int> idx(rows.size());
        std::iota(idx.begin(), idx.end(), 0);
        std::sort(idx.begin(), idx.end(), [&](int x, int y) {
          const int cmp = exact_compare(&C[(size_t)x * np], nk_h[rows[x]], &C[(size_t)y * np], nk_h[rows[y]], pnk, np);
          if (cmp != 0) return cmp < 0;
          return rows[x] < rows[y];   // equal ranks: ascending global index
        });
        for (size_t t = 0; t < idx.size(); ++t) {
          const int32_t v = (int32_t)(rows[idx[t]] - b);
          if (order[pos + t] != v) changed = true;
          order[pos + t] = v;
        }
        *resolved += (int)(end - pos);
      }
      pos = end;
    }
  }
  if (changed)
    SA_CUDA(cudaMemcpyAsync(order_d, order.data(), n_local * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  SA_CUDA(cudaStreamSynchronize(st));
  return SA_OK;
}

// Small device -> host readback on the hot path: one kernel copies the bytes
// into the context's mapped pinned staging buffer (stores over PCIe, no copy
// engine), then the stream is synchronised.  A cudaMemcpyAsync would queue on
// the device-to-host copy engine behind whatever large copies the caller has
// in flight on other streams (measured: a 4-byte read waits 23 ms behind
// 1.25 GB of result copies, tools/dma_probe.py).
__global__ void stage_copy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t bytes) {
  for (int64_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

static sa_status d2h_small(sa_ctx* c, void* h, const void* d, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return SA_OK;
  if (bytes > (size_t)SA_STAGE_BYTES) {
    SA_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
    SA_CUDA(cudaStreamSynchronize(st));
    return SA_OK;
  }
  stage_copy_kernel<<<1, 256, 0, st>>>(c->dstage, static_cast<const uint8_t*>(d), (int64_t)bytes);
  SA_LAUNCHED();
  SA_CUDA(cudaStreamSynchronize(st));
  std::memcpy(h, c->hstage, bytes);
  return SA_OK;
}

static sa_status read_u32(sa_ctx* c, const uint32_t* d, uint32_t* h, cudaStream_t st) {
  return d2h_small(c, h, d, sizeof(uint32_t), st);
}

struct PartArgs {
  int32_t p, kb;
  const uint16_t* prof;
  const int32_t* nk;
  const int64_t* offs;
  int32_t stride;
  int64_t N, first, nloc;
  int32_t* bucket_of;
  sa_pivot* pivots;
  int64_t* counts_h;
  int64_t* bytes_h;
  sa_partition_debug* dbg;
};

// One pass of Algorithm 2 steps 2-11.  exact=false: keys only, uncertified
// comparisons counted; exact=true: every uncertified comparison resolved.
// Returns through *amb_all the number of uncertified comparisons (all ranks).
static sa_status partition_pass(sa_ctx* c, const PartArgs& a, bool exact, int64_t* amb_all, int* resolved,
                                cudaStream_t st) {
  Scratch scratch(st);
  const int G = c->nranks, r = c->rank;
  const int pb = a.p / G;
  const int64_t q0 = (int64_t)r * pb;
  const int n = (int)a.nloc;
  const int ldw = a.stride / 2;
  const int s_loc = pb * a.kb, s_all = a.p * a.kb;
  int64_t wmax = 0;
  for (int q = 0; q < a.p; ++q) wmax = std::max(wmax, block_begin(q + 1, a.N, a.p) - block_begin(q, a.N, a.p));

  SA_ALLOC(amb_cnt, uint32_t, 4);
  SA_CUDA(cudaMemsetAsync(amb_cnt, 0, 4 * sizeof(uint32_t), st));
  SA_ALLOC(lkey, sa_key128, n);
  SA_ALLOC(gkey, sa_key128, n);
  SA_ALLOC(lorder, int32_t, n);
  SA_ALLOC(gorder, int32_t, n);
  SA_ALLOC(samp_gid, int64_t, s_loc);
  SA_ALLOC(samp_local, int32_t, s_loc);
  SA_ALLOC(s_prof_loc, uint16_t, (size_t)s_loc * a.stride);
  SA_ALLOC(s_nk_loc, int32_t, s_loc);
  SA_ALLOC(s_prof, uint16_t, (size_t)s_all * a.stride);
  SA_ALLOC(s_nk, int32_t, s_all);
  SA_ALLOC(s_gid, int64_t, s_all);
  SA_CUDA(cudaMemsetAsync(lkey, 0, n * sizeof(sa_key128), st));
  SA_CUDA(cudaMemsetAsync(gkey, 0, n * sizeof(sa_key128), st));

  // engine operands of the local rows (u8 SAD rows when every count fits,
  // decided on the device; see prepare_ops)
  EngineOps E;
  SA_TRY(prepare_ops(c, scratch, a.prof, n, a.prof, n, a.stride, true, &E, st));

  // K2T operand rows built for S2a's blocks are reused by S2d's query side
  // (the same rows: first dense layers and seen-once planes carried over)
  TcCarry carry;
  carry.scratch = &scratch;

  // ---- S2a: local rank of every member against its own block
  SA_TRY(rec(ev_begin(c, SA_PHASE_S2A), st));
  {
    std::vector<MsProblem> probs;
    for (int q = 0; q < pb; ++q) {
      const int64_t b = block_begin(q0 + q, a.N, a.p) - a.first;
      const int64_t e = block_begin(q0 + q + 1, a.N, a.p) - a.first;
      MsProblem pr{};
      pr.A = pr.B = E.a16.rows + b * E.a16.ldw;
      pr.nkA = pr.nkB = a.nk + b;
      pr.na = pr.nb = (int32_t)(e - b);
      pr.sym = 1;
      pr.keyA = pr.keyB = lkey + b;
      apply_form(c, pr);
      probs.push_back(pr);
    }
    SA_TRY(launch_ops(c, E, probs, st, nullptr, nullptr, SA_PHASE_GEMM_S2A, &carry));
  }
  SA_TRY(rec(ev_end(c, SA_PHASE_S2A), st));

  // ---- S2b: sort each block by (local rank, index); k_b samples
  SA_TRY(rec(ev_begin(c, SA_PHASE_S2B), st));
  SA_TRY(segment_sort_keys(lkey, a.first, a.N, a.p, q0, a.first, pb, window_of(c, wmax), lorder, nullptr,
                           amb_cnt + 0, st));
  if (exact) {
    uint32_t h = 0;
    SA_TRY(read_u32(c, amb_cnt + 0, &h, st));
    if (h)
      SA_TRY(resolve_segments(c, lkey, lorder, n, a.N, a.p, q0, a.first, pb, wmax, a.prof, a.nk, a.stride, true,
                              nullptr, nullptr, 0, resolved, st));
  }
  SA_TRY(pick_launch(lorder, a.N, a.p, q0, a.first, pb, a.kb, a.kb + 1, a.first, samp_gid, samp_local, st));
  SA_TRY(rec(ev_end(c, SA_PHASE_S2B), st));

  // ---- S2c: the global sample S replicated on every rank
  SA_TRY(rec(ev_begin(c, SA_PHASE_S2C), st));
  SA_TRY(gather_rows_launch(a.prof, a.nk, samp_local, s_loc, a.stride, s_prof_loc, s_nk_loc, st));
  SA_TRY(comm_allgather(c, s_prof_loc, s_prof, (int64_t)s_loc * a.stride * 2, st));
  SA_TRY(comm_allgather(c, s_nk_loc, s_nk, (int64_t)s_loc * 4, st));
  SA_TRY(comm_allgather(c, samp_gid, s_gid, (int64_t)s_loc * 8, st));
  SA_TRY(rec(ev_end(c, SA_PHASE_S2C), st));

  // ---- S2d: global rank against S
  {
    // the same local operands; the sample rows' counts fold into the same
    // device counter, so the engine is valid for both sides
    EngineOps E2 = E;
    E2.b16 = Operand{reinterpret_cast<const uint32_t*>(s_prof), ldw};
    if (E2.mode == ENC_AUTO) SA_TRY(make_u8_rows(scratch, s_prof, s_all, a.stride, c->dcount, &E2.b8, st, &E2));
    SA_TRY(rec(ev_begin(c, SA_PHASE_S2D), st));
    MsProblem pr{};
    pr.A = E2.a16.rows;
    pr.B = E2.b16.rows;
    pr.nkA = a.nk;
    pr.nkB = s_nk;
    pr.na = n;
    pr.nb = s_all;
    pr.sym = 0;
    pr.keyA = gkey;
    if (a.dbg && a.dbg->global_num) {   // parity artifact: the N x s numerator matrix
      pr.num = a.dbg->global_num;
      pr.ld = s_all;
    }
    apply_form(c, pr);
    SA_TRY(launch_ops(c, E2, {pr}, st, nullptr, nullptr, SA_PHASE_GEMM_S2D, nullptr, &carry));
  }
  SA_TRY(rec(ev_end(c, SA_PHASE_S2D), st));

  // ---- S3: block sort, regular samples, pivots, buckets
  SA_TRY(rec(ev_begin(c, SA_PHASE_S3), st));
  SA_TRY(segment_sort_keys(gkey, a.first, a.N, a.p, q0, a.first, pb, window_of(c, s_all), gorder, nullptr,
                           amb_cnt + 1, st));
  if (exact) {
    uint32_t h = 0;
    SA_TRY(read_u32(c, amb_cnt + 1, &h, st));
    if (h)
      SA_TRY(resolve_segments(c, gkey, gorder, n, a.N, a.p, q0, a.first, pb, s_all, a.prof, a.nk, a.stride, false,
                              s_prof, s_nk, s_all, resolved, st));
  }
  const int ncand_loc = pb * (a.p - 1), ncand = a.p * (a.p - 1);
  SA_ALLOC(counts_d, unsigned long long, 2 * a.p);
  SA_CUDA(cudaMemsetAsync(counts_d, 0, 2 * a.p * sizeof(unsigned long long), st));
  SA_ALLOC(y_gid, int64_t, std::max(ncand, 1));
  if (a.p > 1) {
    SA_ALLOC(cand_gid, int64_t, ncand_loc);
    SA_ALLOC(cand_local, int32_t, ncand_loc);
    SA_ALLOC(rec_loc, sa_pivot, ncand_loc);
    SA_ALLOC(rec_all, sa_pivot, ncand);
    SA_ALLOC(tmp_k, sa_key128, ncand);
    SA_ALLOC(tmp_g, int64_t, ncand);
    SA_ALLOC(yorder, int32_t, ncand);
    SA_TRY(pick_launch(gorder, a.N, a.p, q0, a.first, pb, a.p - 1, a.p, a.first, cand_gid, cand_local, st));
    SA_TRY(make_records_launch(cand_local, cand_gid, ncand_loc, gkey, a.nk, a.p - 1, (int)q0, rec_loc, st));
    SA_TRY(comm_allgather(c, rec_loc, rec_all, (int64_t)ncand_loc * sizeof(sa_pivot), st));
    SA_TRY(sort_records(rec_all, ncand, window_of(c, s_all), tmp_k, tmp_g, yorder, nullptr, amb_cnt + 2, st));

    std::vector<uint16_t> candC;        // exact path: C rows of every candidate vs S
    std::vector<sa_pivot> rec_h;
    std::vector<int32_t> s_nk_h;
    if (exact) {
      // C rows of the local candidates, gathered from every rank (collective)
      std::vector<int32_t> cl(ncand_loc);
      SA_CUDA(cudaMemcpyAsync(cl.data(), cand_local, ncand_loc * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaStreamSynchronize(st));
      std::vector<uint16_t> Cloc;
      SA_TRY(numerator_rows_host(a.prof, a.nk, cl, s_prof, s_nk, s_all, a.stride, Cloc, st));
      SA_ALLOC(cl_d, uint16_t, (size_t)ncand_loc * s_all);
      SA_ALLOC(call_d, uint16_t, (size_t)ncand * s_all);
      SA_CUDA(cudaMemcpyAsync(cl_d, Cloc.data(), Cloc.size() * 2, cudaMemcpyHostToDevice, st));
      SA_TRY(comm_allgather(c, cl_d, call_d, (int64_t)ncand_loc * s_all * 2, st));
      candC.resize((size_t)ncand * s_all);
      rec_h.resize(ncand);
      s_nk_h.resize(s_all);
      SA_CUDA(cudaMemcpyAsync(candC.data(), call_d, candC.size() * 2, cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaMemcpyAsync(rec_h.data(), rec_all, ncand * sizeof(sa_pivot), cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaMemcpyAsync(s_nk_h.data(), s_nk, s_all * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaStreamSynchronize(st));
      // exact sort of Y on the host (identical on every rank)
      std::vector<int32_t> yo(ncand);
      std::iota(yo.begin(), yo.end(), 0);
      std::sort(yo.begin(), yo.end(), [&](int x, int y) {
        const sa_pivot &X = rec_h[x], &Y = rec_h[y];
        int cmp;
        if (host_key_near(X.key, Y.key, s_all))
          cmp = exact_compare(&candC[(size_t)x * s_all], X.nk, &candC[(size_t)y * s_all], Y.nk, s_nk_h.data(), s_all);
        else
          cmp = host_key_lt(X.key, 0, Y.key, 1) ? -1 : 1;
        if (cmp != 0) return cmp < 0;
        return X.global_idx < Y.global_idx;
      });
      SA_CUDA(cudaMemcpyAsync(yorder, yo.data(), ncand * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    }
    SA_TRY(pivots_launch(rec_all, yorder, ncand, a.p, y_gid, a.pivots, st));
    SA_TRY(assign_launch(gkey, a.first, n, a.pivots, a.p, window_of(c, s_all), a.offs, a.bucket_of, nullptr,
                         amb_cnt + 3, counts_d, counts_d + a.p, st));
    if (exact) {
      uint32_t h = 0;
      SA_TRY(read_u32(c, amb_cnt + 3, &h, st));
      if (h) {
        // re-decide every item whose comparison with a pivot is uncertified
        std::vector<sa_pivot> piv(a.p - 1);
        std::vector<sa_key128> keys(n);
        std::vector<int32_t> bkt(n), nk_h(n);
        std::vector<int64_t> offs_h(n + 1);
        SA_CUDA(cudaMemcpyAsync(piv.data(), a.pivots, (a.p - 1) * sizeof(sa_pivot), cudaMemcpyDeviceToHost, st));
        SA_CUDA(cudaMemcpyAsync(keys.data(), gkey, n * sizeof(sa_key128), cudaMemcpyDeviceToHost, st));
        SA_CUDA(cudaMemcpyAsync(bkt.data(), a.bucket_of, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA(cudaMemcpyAsync(nk_h.data(), a.nk, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA(cudaMemcpyAsync(offs_h.data(), a.offs, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SA_CUDA(cudaStreamSynchronize(st));
        std::vector<int> pidx(a.p - 1);   // candidate slot of each pivot
        for (int b = 0; b < a.p - 1; ++b)
          for (int t = 0; t < ncand; ++t)
            if (rec_h[t].global_idx == piv[b].global_idx) pidx[b] = t;
        std::vector<int32_t> flagged;
        for (int i = 0; i < n; ++i)
          for (int b = 0; b < a.p - 1; ++b)
            if (piv[b].global_idx != a.first + i && host_key_near(piv[b].key, keys[i], s_all)) {
              flagged.push_back(i);
              break;
            }
        std::vector<uint16_t> Ci;
        SA_TRY(numerator_rows_host(a.prof, a.nk, flagged, s_prof, s_nk, s_all, a.stride, Ci, st));
        for (size_t f = 0; f < flagged.size(); ++f) {
          const int i = flagged[f];
          int bk = 0;
          for (int b = 0; b < a.p - 1; ++b) {
            bool less;   // pivot_b < item ?
            if (piv[b].global_idx == a.first + i) less = false;
            else if (host_key_near(piv[b].key, keys[i], s_all)) {
              const int cmp = exact_compare(&candC[(size_t)pidx[b] * s_all], piv[b].nk, &Ci[f * s_all], nk_h[i],
                                            s_nk_h.data(), s_all);
              less = cmp < 0 || (cmp == 0 && piv[b].global_idx < a.first + i);
            } else
              less = host_key_lt(piv[b].key, piv[b].global_idx, keys[i], a.first + i);
            bk += less ? 1 : 0;
          }
          bkt[i] = bk;
          ++*resolved;
        }
        std::vector<unsigned long long> cb(2 * a.p, 0);
        for (int i = 0; i < n; ++i) {
          cb[bkt[i]] += 1;
          cb[a.p + bkt[i]] += (unsigned long long)(offs_h[i + 1] - offs_h[i]);
        }
        SA_CUDA(cudaMemcpyAsync(a.bucket_of, bkt.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        SA_CUDA(cudaMemcpyAsync(counts_d, cb.data(), cb.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
        SA_CUDA(cudaStreamSynchronize(st));
      }
    }
  } else {
    // p == 1: a single bucket
    SA_CUDA(cudaMemsetAsync(a.bucket_of, 0, n * sizeof(int32_t), st));
    std::vector<int64_t> offs_h(2);
    SA_CUDA(cudaMemcpyAsync(&offs_h[0], a.offs, 8, cudaMemcpyDeviceToHost, st));
    SA_CUDA(cudaMemcpyAsync(&offs_h[1], a.offs + n, 8, cudaMemcpyDeviceToHost, st));
    SA_CUDA(cudaStreamSynchronize(st));
    unsigned long long cb[2] = {(unsigned long long)n, (unsigned long long)(offs_h[1] - offs_h[0])};
    SA_CUDA(cudaMemcpyAsync(counts_d, cb, sizeof cb, cudaMemcpyHostToDevice, st));
  }
  SA_TRY(rec(ev_end(c, SA_PHASE_S3), st));

  // ---- C3: count exchange (the one mandatory host block).  Each rank's record
  // is [p counts][p residue bytes][four u32 uncertified-comparison counters].
  // ... plus the rank's sticky error flags (sa_kmer_profiles), so that every
  // rank sees any rank's range error and all fail together
  const int recw = 2 * a.p + 3;
  SA_ALLOC(xrec, int64_t, recw);
  SA_ALLOC(xall, int64_t, (size_t)recw * G);
  SA_CUDA(cudaMemcpyAsync(xrec, counts_d, 2 * a.p * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  SA_CUDA(cudaMemcpyAsync(xrec + 2 * a.p, amb_cnt, 4 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  SA_CUDA(cudaMemcpyAsync(xrec + 2 * a.p + 2, c->derr, 8, cudaMemcpyDeviceToDevice, st));
  SA_TRY(comm_allgather(c, xrec, xall, (int64_t)recw * 8, st));
  std::vector<int64_t> xh((size_t)recw * G);
  SA_TRY(d2h_small(c, xh.data(), xall, xh.size() * 8, st));
  int64_t amb_total = 0;
  uint32_t errs = 0;
  for (int g = 0; g < G; ++g) {
    uint32_t e2[2];
    std::memcpy(e2, &xh[(size_t)g * recw + 2 * a.p + 2], sizeof e2);
    errs |= e2[0];
  }
  if (errs) {
    SA_CUDA(cudaMemsetAsync(c->derr, 0, 4, st));
    if (errs & ERR_RESIDUE) return fail(SA_E_RANGE, "residue outside the alphabet (sa_kmer_profiles, some rank)");
    return fail(SA_E_RANGE, "a sequence has more than 65535 k-mers (sa_kmer_profiles, some rank)");
  }
  for (int g = 0; g < G; ++g) {
    uint32_t cnt4[4];
    std::memcpy(cnt4, &xh[(size_t)g * recw + 2 * a.p], sizeof cnt4);
    for (int t = 0; t < 4; ++t) amb_total += cnt4[t];
    for (int b = 0; b < a.p; ++b) {
      a.counts_h[(size_t)g * a.p + b] = xh[(size_t)g * recw + b];
      a.bytes_h[(size_t)g * a.p + b] = xh[(size_t)g * recw + a.p + b];
    }
  }
  *amb_all = amb_total;

  // ---- debug artifacts
  if (a.dbg) {
    sa_partition_debug* d = a.dbg;
    if (d->local_key) SA_CUDA(cudaMemcpyAsync(d->local_key, lkey, n * sizeof(sa_key128), cudaMemcpyDeviceToDevice, st));
    if (d->global_key)
      SA_CUDA(cudaMemcpyAsync(d->global_key, gkey, n * sizeof(sa_key128), cudaMemcpyDeviceToDevice, st));
    if (d->local_f64 || d->global_f64) {
      for (int q = 0; q < pb; ++q) {
        const int64_t b = block_begin(q0 + q, a.N, a.p) - a.first;
        const int64_t e = block_begin(q0 + q + 1, a.N, a.p) - a.first;
        if (d->local_f64)
          SA_TRY(keys_to_f64_launch(lkey + b, e - b, e - b, d->local_f64 + b, st, c->rank_form, std::log1p(c->delta)));
      }
      if (d->global_f64)
        SA_TRY(keys_to_f64_launch(gkey, n, s_all, d->global_f64, st, c->rank_form, std::log1p(c->delta)));
    }
    if (d->local_order) {
      // order (segment offsets) -> global ids
      std::vector<int32_t> o(n);
      std::vector<int64_t> g(n);
      SA_CUDA(cudaMemcpyAsync(o.data(), lorder, n * 4, cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaStreamSynchronize(st));
      for (int q = 0; q < pb; ++q) {
        const int64_t b = block_begin(q0 + q, a.N, a.p) - a.first;
        const int64_t e = block_begin(q0 + q + 1, a.N, a.p) - a.first;
        for (int64_t t = b; t < e; ++t) g[t] = a.first + b + o[t];
      }
      SA_CUDA(cudaMemcpyAsync(d->local_order, g.data(), n * 8, cudaMemcpyHostToDevice, st));
      SA_CUDA(cudaStreamSynchronize(st));
    }
    if (d->global_order) {
      std::vector<int32_t> o(n);
      std::vector<int64_t> g(n);
      SA_CUDA(cudaMemcpyAsync(o.data(), gorder, n * 4, cudaMemcpyDeviceToHost, st));
      SA_CUDA(cudaStreamSynchronize(st));
      for (int q = 0; q < pb; ++q) {
        const int64_t b = block_begin(q0 + q, a.N, a.p) - a.first;
        const int64_t e = block_begin(q0 + q + 1, a.N, a.p) - a.first;
        for (int64_t t = b; t < e; ++t) g[t] = a.first + b + o[t];
      }
      SA_CUDA(cudaMemcpyAsync(d->global_order, g.data(), n * 8, cudaMemcpyHostToDevice, st));
      SA_CUDA(cudaStreamSynchronize(st));
    }
    if (d->sample_idx) SA_CUDA(cudaMemcpyAsync(d->sample_idx, s_gid, s_all * 8, cudaMemcpyDeviceToDevice, st));
    if (d->candidates && ncand > 0)
      SA_CUDA(cudaMemcpyAsync(d->candidates, y_gid, ncand * 8, cudaMemcpyDeviceToDevice, st));
  }
  return SA_OK;
}

}  // namespace sa

extern "C" {

sa_status sa_kmer_profiles(sa_ctx* ctx, const uint8_t* residues, const int64_t* offsets, int32_t n, int32_t k,
                           int32_t alphabet, uint16_t* profiles, int32_t* nkmers, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (n < 0) return fail(SA_E_INVAL, "n < 0");
  if (k < 1) return fail(SA_E_INVAL, "k < 1");
  if (alphabet < 2) return fail(SA_E_INVAL, "alphabet < 2");
  int64_t bins = 1;
  for (int t = 0; t < k; ++t) {
    bins *= alphabet;
    if (bins > 65536) return fail(SA_E_INVAL, "alphabet^k > 65536");
  }
  if (n == 0) return SA_OK;
  if (!offsets || !profiles || !nkmers) return fail(SA_E_INVAL, "NULL required pointer");
  cudaStream_t st = (cudaStream_t)stream;
  SA_CUDA(cudaSetDevice(ctx->device));
  // asynchronous: range errors go to the context's sticky device flags,
  // surfaced by sa_ctx_check or at sa_partition's count exchange
  SA_TRY(profiles_launch(residues, offsets, n, k, alphabet, profile_stride((int32_t)bins), profiles, nkmers, ctx->derr,
                         st));
  return SA_OK;
}

sa_status sa_kmer_rank(sa_ctx* ctx, const uint16_t* q_prof, const int32_t* q_nk, int32_t nq,
                       const uint16_t* pool_prof, const int32_t* pool_nk, int32_t npool, int32_t bins,
                       sa_key128* keys, double* rank_f64, uint16_t* numerators, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (npool <= 0) return fail(SA_E_INVAL, "empty pool");
  if (nq < 0 || bins < 1 || bins > 65536) return fail(SA_E_INVAL, "bad nq / bins");
  if (nq == 0) return SA_OK;
  if (!q_prof || !q_nk || !pool_prof || !pool_nk || !keys) return fail(SA_E_INVAL, "NULL required pointer");
  cudaStream_t st = (cudaStream_t)stream;
  SA_CUDA(cudaSetDevice(ctx->device));
  SA_CUDA(cudaMemsetAsync(keys, 0, (size_t)nq * sizeof(sa_key128), st));
  Scratch scratch(st);
  EngineOps E;
  SA_TRY(prepare_ops(ctx, scratch, q_prof, nq, pool_prof, npool, bins, true, &E, st));
  MsProblem pr{};
  pr.A = E.a16.rows;
  pr.B = E.b16.rows;
  pr.nkA = q_nk;
  pr.nkB = pool_nk;
  pr.na = nq;
  pr.nb = npool;
  // the pool is the query set itself (a block's local rank, or the centralized
  // rank of SURVEY N2): C is symmetric, so only the upper-triangle tiles run,
  // each adding its row sums to key_i and its column sums to key_j
  pr.sym = (q_prof == pool_prof && q_nk == pool_nk && nq == npool) ? 1 : 0;
  pr.keyA = keys;
  pr.keyB = pr.sym ? keys : nullptr;
  pr.num = numerators;
  pr.ld = npool;
  apply_form(ctx, pr);
  cudaEvent_t r0 = ev_begin(ctx, SA_PHASE_RANK);
  SA_TRY(launch_ops(ctx, E, {pr}, st, r0, ev_end(ctx, SA_PHASE_RANK), SA_PHASE_GEMM));
  if (rank_f64) SA_TRY(keys_to_f64_launch(keys, nq, npool, rank_f64, st, ctx->rank_form, std::log1p(ctx->delta)));
  return SA_OK;
}

sa_status sa_partition(sa_ctx* ctx, int32_t p, int32_t samples_per_block, const uint16_t* profiles,
                       const int32_t* nkmers, const int64_t* offsets, int32_t bins, int64_t n_total,
                       int64_t first_global, int32_t n_local, int32_t* bucket_of, sa_pivot* pivots, int64_t* counts_h,
                       int64_t* bytes_h, sa_partition_debug* dbg, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  const int G = ctx->nranks, r = ctx->rank;
  if (p < 1) return fail(SA_E_INVAL, "p < 1");
  if (n_total < p) return fail(SA_E_INVAL, "n_total < p");
  if (p % G != 0) return fail(SA_E_INVAL, "nranks (%d) must divide p (%d)", G, p);
  if (bins < 1 || bins > 65536) return fail(SA_E_INVAL, "bad bins");
  const int pb = p / G;
  const int64_t exp_first = block_begin((int64_t)r * pb, n_total, p);
  const int64_t exp_n = block_begin((int64_t)(r + 1) * pb, n_total, p) - exp_first;
  if (first_global != exp_first || n_local != exp_n)
    return fail(SA_E_INVAL, "shard [%lld, +%d) does not match blocks [%d, %d) = [%lld, +%lld)",
                (long long)first_global, n_local, r * pb, (r + 1) * pb, (long long)exp_first, (long long)exp_n);
  for (int q = 0; q < p; ++q) {
    const int64_t w = block_begin(q + 1, n_total, p) - block_begin(q, n_total, p);
    if (samples_per_block < 1 || samples_per_block > w)
      return fail(SA_E_INVAL, "samples_per_block (%d) must be in [1, block size %lld]", samples_per_block,
                  (long long)w);
  }
  if (!profiles || !nkmers || !offsets || !bucket_of || !counts_h || !bytes_h || (p > 1 && !pivots))
    return fail(SA_E_INVAL, "NULL required pointer");
  if ((int64_t)p * samples_per_block > (int64_t)1 << 30) return fail(SA_E_INVAL, "sample too large");
  cudaStream_t st = (cudaStream_t)stream;
  SA_CUDA(cudaSetDevice(ctx->device));
  PartArgs a{p, samples_per_block, profiles, nkmers, offsets, profile_stride(bins), n_total, first_global, n_local,
             bucket_of, pivots, counts_h, bytes_h, dbg};
  int64_t amb = 0;
  int resolved = 0;
  SA_TRY(partition_pass(ctx, a, false, &amb, &resolved, st));
  if (dbg && dbg->uncertified_h) *dbg->uncertified_h = ctx->rank_form == SA_RANK_DF ? (int32_t)amb : 0;
  if (amb > 0 && ctx->rank_form == SA_RANK_F) {
    // some order was not certified by the keys on some rank: redo the pass
    // with exact resolution everywhere (collectively -- every rank saw amb).
    SA_TRY(partition_pass(ctx, a, true, &amb, &resolved, st));
  }
  if (dbg && dbg->exact_fallbacks_h) *dbg->exact_fallbacks_h = resolved;
  return SA_OK;
}

sa_status sa_redistribute(sa_ctx* ctx, int32_t p, const uint8_t* residues, const int64_t* offsets, int32_t n_local,
                          int64_t first_global, const int32_t* bucket_of, const int64_t* counts_h,
                          const int64_t* bytes_h, uint8_t* recv_residues, int64_t* recv_offsets,
                          int64_t* recv_global_idx, int32_t* recv_bucket, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  const int G = ctx->nranks, r = ctx->rank;
  if (p < 1 || p % G != 0) return fail(SA_E_INVAL, "nranks must divide p");
  if (!counts_h || !bytes_h || !recv_offsets) return fail(SA_E_INVAL, "NULL required pointer");
  if (n_local > 0 && (!residues || !offsets || !bucket_of)) return fail(SA_E_INVAL, "NULL required pointer");
  const int pb = p / G;
  cudaStream_t st = (cudaStream_t)stream;
  SA_CUDA(cudaSetDevice(ctx->device));
  Scratch scratch(st);
  const int n = n_local;
  const int nchunk = (n + 255) / 256;
  SA_ALLOC(hist, int32_t, (size_t)std::max(nchunk, 1) * p);
  SA_ALLOC(base, int64_t, (size_t)std::max(nchunk, 1) * p);
  SA_ALLOC(perm, int32_t, std::max(n, 1));
  SA_ALLOC(lens, int64_t, std::max(n, 1));
  SA_ALLOC(part, int64_t, (n + 1023) / 1024 + 2);
  SA_TRY(bucket_perm_launch(bucket_of, n, p, hist, base, perm, st));
  if (!ctx->has_comm && !ctx->nccl) {   // single rank, no communicator: the send layout is the receive layout
    SA_TRY(perm_meta_launch(perm, n, offsets, bucket_of, first_global, lens, recv_global_idx, recv_bucket, st));
    SA_TRY(scan_launch(lens, n, recv_offsets, part, st));
    SA_TRY(copy_seqs_launch(perm, n, residues, offsets, recv_residues, recv_offsets, st));
    return SA_OK;
  }
  // ---- send side: bucket-major pack (buckets of rank d are contiguous)
  std::vector<int64_t> sseq(G, 0), sbytes(G, 0), rseq(G, 0), rbytes(G, 0);
  for (int b = 0; b < p; ++b) {
    sseq[b / pb] += counts_h[(size_t)r * p + b];
    sbytes[b / pb] += bytes_h[(size_t)r * p + b];
  }
  for (int g = 0; g < G; ++g)
    for (int b = r * pb; b < (r + 1) * pb; ++b) {
      rseq[g] += counts_h[(size_t)g * p + b];
      rbytes[g] += bytes_h[(size_t)g * p + b];
    }
  std::vector<int64_t> sseq_d(G), sbytes_d(G), rseq_d(G), rbytes_d(G);
  std::vector<int64_t> sm_b(G), sm_d(G), rm_b(G), rm_d(G);   // meta bytes / displs
  int64_t t_ss = 0, t_sb = 0, t_rs = 0, t_rb = 0;
  for (int g = 0; g < G; ++g) {
    sseq_d[g] = t_ss; t_ss += sseq[g];
    sbytes_d[g] = t_sb; t_sb += sbytes[g];
    rseq_d[g] = t_rs; t_rs += rseq[g];
    rbytes_d[g] = t_rb; t_rb += rbytes[g];
    sm_b[g] = sseq[g] * 16; sm_d[g] = sseq_d[g] * 16;
    rm_b[g] = rseq[g] * 16; rm_d[g] = rseq_d[g] * 16;
  }
  SA_ALLOC(soffs, int64_t, n + 1);
  SA_ALLOC(smeta, int64_t, (size_t)std::max(n, 1) * 2);
  SA_ALLOC(sres, uint8_t, std::max<int64_t>(t_sb, 1));
  SA_ALLOC(rmeta, int64_t, (size_t)std::max<int64_t>(t_rs, 1) * 2);
  SA_ALLOC(rres, uint8_t, std::max<int64_t>(t_rb, 1));
  SA_ALLOC(fmeta, int64_t, (size_t)std::max<int64_t>(t_rs, 1) * 2);
  SA_TRY(perm_meta_launch(perm, n, offsets, bucket_of, first_global, lens, nullptr, nullptr, st));
  SA_TRY(scan_launch(lens, n, soffs, part, st));
  SA_TRY(copy_seqs_launch(perm, n, residues, offsets, sres, soffs, st));
  SA_TRY(pack_meta_launch(perm, n, offsets, bucket_of, first_global, smeta, st));
  if (ctx->nccl) {
    SA_TRY(nccl_alltoallv(ctx->nccl, G, r, smeta, sm_b.data(), sm_d.data(), rmeta, rm_b.data(), rm_d.data(), st));
    SA_TRY(nccl_alltoallv(ctx->nccl, G, r, sres, sbytes.data(), sbytes_d.data(), rres, rbytes.data(), rbytes_d.data(),
                          st));
  } else {
    if (ctx->comm.alltoallv(ctx->comm.user, smeta, sm_b.data(), sm_d.data(), rmeta, rm_b.data(), rm_d.data(),
                            (void*)st))
      return fail(SA_E_COMM, "alltoallv (meta) callback failed");
    if (ctx->comm.alltoallv(ctx->comm.user, sres, sbytes.data(), sbytes_d.data(), rres, rbytes.data(), rbytes_d.data(),
                            (void*)st))
      return fail(SA_E_COMM, "alltoallv (residues) callback failed");
  }
  // ---- receive side: [src][bucket] -> [bucket][src] (ascending global id, Z17)
  const int nseg = G * pb;
  std::vector<char> segs_h(segcopy_size() * nseg);
  int t = 0;
  int64_t dst_m = 0, dst_r = 0;
  for (int b = r * pb; b < (r + 1) * pb; ++b) {
    for (int g = 0; g < G; ++g) {
      int64_t src_m = rseq_d[g], src_r = rbytes_d[g];
      for (int b2 = r * pb; b2 < b; ++b2) {
        src_m += counts_h[(size_t)g * p + b2];
        src_r += bytes_h[(size_t)g * p + b2];
      }
      const int64_t cnt = counts_h[(size_t)g * p + b], nb = bytes_h[(size_t)g * p + b];
      segcopy_fill(segs_h.data(), t++, src_m, dst_m, cnt, src_r, dst_r, nb);
      dst_m += cnt;
      dst_r += nb;
    }
  }
  SA_ALLOC(segs_d, char, segs_h.size());
  SA_CUDA(cudaMemcpyAsync(segs_d, segs_h.data(), segs_h.size(), cudaMemcpyHostToDevice, st));
  SA_TRY(seg_copy_launch(segs_d, nseg, rmeta, fmeta, rres, recv_residues, st));
  SA_ALLOC(rlens, int64_t, std::max<int64_t>(t_rs, 1));
  SA_ALLOC(rpart, int64_t, (t_rs + 1023) / 1024 + 2);
  SA_TRY(unpack_meta_launch(fmeta, (int)t_rs, recv_global_idx, rlens, recv_bucket, st));
  SA_TRY(scan_launch(rlens, t_rs, recv_offsets, rpart, st));
  // segs_h must outlive the async H2D copy from pageable memory: pageable
  // cudaMemcpyAsync returns after staging, so it is safe to release here.
  return SA_OK;
}

sa_status sa_bucket_similarity(sa_ctx* ctx, const uint16_t* profiles, const int32_t* nkmers, int32_t n, int32_t bins,
                               uint16_t* numerators, double* similarity, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (n < 0 || bins < 1 || bins > 65536) return fail(SA_E_INVAL, "bad n / bins");
  if (n == 0) return SA_OK;
  if (!profiles || !nkmers) return fail(SA_E_INVAL, "NULL required pointer");
  cudaStream_t st = (cudaStream_t)stream;
  SA_CUDA(cudaSetDevice(ctx->device));
  Scratch scratch(st);
  EngineOps E;
  SA_TRY(prepare_ops(ctx, scratch, profiles, n, profiles, n, bins, true, &E, st));
  MsProblem pr{};
  pr.A = pr.B = E.a16.rows;
  pr.nkA = pr.nkB = nkmers;
  pr.na = pr.nb = n;
  pr.sym = 1;
  pr.num = numerators;
  pr.sim = similarity;
  pr.ld = n;
  cudaEvent_t s0 = ev_begin(ctx, SA_PHASE_S5);
  SA_TRY(launch_ops(ctx, E, {pr}, st, s0, ev_end(ctx, SA_PHASE_S5), SA_PHASE_GEMM_S5));
  return SA_OK;
}

sa_status sa_guide_tree(sa_ctx* ctx, const double* similarity, int32_t n, int64_t ld, int32_t* merges,
                        double* heights, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (n < 1 || ld < n) return fail(SA_E_INVAL, "bad n / ld");
  if (n > 1 && (!similarity || !merges || !heights)) return fail(SA_E_INVAL, "NULL required pointer");
  SA_CUDA(cudaSetDevice(ctx->device));
  return upgma_launch(similarity, n, ld, merges, heights, tree_form_of(ctx), (cudaStream_t)stream);
}

sa_status sa_guide_tree_batch(sa_ctx* ctx, int32_t count, const double* const* similarity_h, const int32_t* n_h,
                              const int64_t* ld_h, int32_t* const* merges_h, double* const* heights_h, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (count < 0) return fail(SA_E_INVAL, "count < 0");
  if (count == 0) return SA_OK;
  if (!similarity_h || !n_h || !ld_h || !merges_h || !heights_h) return fail(SA_E_INVAL, "NULL required pointer");
  for (int i = 0; i < count; ++i) {
    if (n_h[i] < 1 || ld_h[i] < n_h[i]) return fail(SA_E_INVAL, "tree %d: bad n / ld", i);
    if (n_h[i] > 1 && (!similarity_h[i] || !merges_h[i] || !heights_h[i]))
      return fail(SA_E_INVAL, "tree %d: NULL required pointer", i);
  }
  SA_CUDA(cudaSetDevice(ctx->device));
  return upgma_launch_batch(count, similarity_h, n_h, ld_h, merges_h, heights_h, tree_form_of(ctx),
                            (cudaStream_t)stream);
}

}  // extern "C"
namespace sa {
template <class T>
static sa_status pack_upper(sa_ctx* ctx, const T* matrix, int32_t n, int64_t ld, T* packed, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (n < 0 || ld < n) return fail(SA_E_INVAL, "bad n / ld");
  if (n == 0) return SA_OK;
  if (!matrix || !packed) return fail(SA_E_INVAL, "NULL required pointer");
  SA_CUDA(cudaSetDevice(ctx->device));
  pack_upper_kernel<T><<<(unsigned)std::min<int64_t>(n, 148 * 16), 256, 0, (cudaStream_t)stream>>>(matrix, n, ld, packed);
  SA_LAUNCHED();
  return SA_OK;
}
}  // namespace sa
extern "C" {

sa_status sa_pack_upper_u16(sa_ctx* ctx, const uint16_t* matrix, int32_t n, int64_t ld, uint16_t* packed,
                            void* stream) {
  return pack_upper(ctx, matrix, n, ld, packed, stream);
}

sa_status sa_pack_upper_f64(sa_ctx* ctx, const double* matrix, int32_t n, int64_t ld, double* packed, void* stream) {
  return pack_upper(ctx, matrix, n, ld, packed, stream);
}

sa_status sa_bucket_similarity_batch(sa_ctx* ctx, int32_t nbuckets, const uint16_t* profiles, const int32_t* nkmers,
                                     const int64_t* row_begin_h, int32_t bins, uint16_t* const* numerators_h,
                                     double* const* similarity_h, const int64_t* ld_h, void* stream) {
  g_err.clear();
  if (!ctx) return fail(SA_E_INVAL, "ctx is NULL");
  if (nbuckets < 0 || bins < 1 || bins > 65536) return fail(SA_E_INVAL, "bad nbuckets / bins");
  if (nbuckets == 0) return SA_OK;
  if (!row_begin_h) return fail(SA_E_INVAL, "NULL row_begin_h");
  if (row_begin_h[0] != 0) return fail(SA_E_INVAL, "row_begin_h[0] must be 0");
  for (int b = 0; b < nbuckets; ++b) {
    if (row_begin_h[b + 1] < row_begin_h[b]) return fail(SA_E_INVAL, "row_begin_h must be non-decreasing");
    if (row_begin_h[b + 1] - row_begin_h[b] > INT32_MAX) return fail(SA_E_INVAL, "bucket too large");
    if (ld_h && ld_h[b] < row_begin_h[b + 1] - row_begin_h[b]) return fail(SA_E_INVAL, "ld_h[b] < bucket size");
  }
  const int64_t n = row_begin_h[nbuckets];
  if (n == 0) return SA_OK;
  if (!profiles || !nkmers) return fail(SA_E_INVAL, "NULL required pointer");
  cudaStream_t st = (cudaStream_t)stream;
  SA_CUDA(cudaSetDevice(ctx->device));
  Scratch scratch(st);
  EngineOps E;
  SA_TRY(prepare_ops(ctx, scratch, profiles, n, profiles, n, bins, true, &E, st));
  std::vector<MsProblem> probs;
  for (int b = 0; b < nbuckets; ++b) {
    const int64_t r0 = row_begin_h[b], nb = row_begin_h[b + 1] - r0;
    if (nb == 0) continue;
    MsProblem pr{};
    pr.A = pr.B = E.a16.rows + r0 * E.a16.ldw;
    pr.nkA = pr.nkB = nkmers + r0;
    pr.na = pr.nb = (int32_t)nb;
    pr.sym = 1;
    pr.num = numerators_h ? numerators_h[b] : nullptr;
    pr.sim = similarity_h ? similarity_h[b] : nullptr;
    pr.ld = ld_h ? ld_h[b] : nb;
    probs.push_back(pr);
  }
  cudaEvent_t s0 = ev_begin(ctx, SA_PHASE_S5);
  SA_TRY(launch_ops(ctx, E, probs, st, s0, ev_end(ctx, SA_PHASE_S5), SA_PHASE_GEMM_S5));
  return SA_OK;
}

}  // extern "C"
