/*
 * libsa -- the Sample-Align-D data-parallel hot path on B200 (sm_100a).
 *
 * Saeed & Khokhar, "A Domain Decomposition Strategy for Alignment of Multiple
 * Biological Sequences on Multiprocessor Platforms", arXiv 0905.1744.
 * Citations: P:a-b = /root/reference/PAPER.md lines (section / equation /
 * algorithm given alongside); Z-ids = the readings listed in DESIGN.md §2.
 *
 * The five steps (BASELINE.json north_star):
 *   S1  k-mer count profiles                      sa_kmer_profiles
 *   S2  k-mer rank vs a pool (Eq. 1 averaged)     sa_kmer_rank (S2a/S2d inside sa_partition)
 *   S3  rank-based sample-sort partition          sa_partition
 *   S4  all-to-all redistribution                 sa_redistribute
 *   S5  all-pairs similarity inside a bucket      sa_bucket_similarity (_batch)
 * and, past the hot path:
 *   N4  the bucket's guide tree (UPGMA)           sa_guide_tree
 *   result transfer: packed symmetric matrices    sa_pack_upper_u16 / _f64
 *
 * Conventions for every call:
 *   - pointers are DEVICE pointers unless the name ends in _h (host);
 *   - the caller allocates and frees every input and output; libsa owns only
 *     its context scratch;
 *   - work is enqueued on `stream` (a cudaStream_t passed as void*); calls
 *     are asynchronous except where a host block is documented;
 *   - errors are returned as sa_status, never thrown or aborted; the message
 *     is in sa_last_error() (thread-local, valid until the next sa_* call on
 *     that thread).  On error outputs are unspecified; the context stays
 *     usable unless SA_E_STATE is returned.
 *   - there is no CPU fallback: without a usable CUDA device every call that
 *     computes returns SA_E_CUDA.
 */
#ifndef SA_H_
#define SA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SA_OK = 0,
  SA_E_INVAL = 1,   /* host-checked argument error (before any launch) */
  SA_E_RANGE = 2,   /* device-detected: residue >= alphabet, or nk > 65535 */
  SA_E_CUDA = 3,    /* CUDA runtime error / no device */
  SA_E_COMM = 4,    /* a communicator callback returned non-zero */
  SA_E_NOMEM = 5,   /* scratch allocation failed */
  SA_E_STATE = 6    /* context unusable (sticky CUDA error) */
} sa_status;

typedef struct sa_ctx sa_ctx;

/* Exact-rank key ("exact ranks"): for a query i ranked against a
 * pool, key_i = sum_j floor(C_ij * 2^64 / D_ij) as an unsigned 128-bit
 * integer (lo = low 64 bits).  With V_i = sum_j C_ij / D_ij (Eq. 1 summed,
 * P:267-269, Eq. 3 in F form P:280-282), 2^64 V_i - npool < key_i <= 2^64 V_i,
 * so key_b - key_a >= npool certifies V_b > V_a.  Integer sums: the key is
 * independent of reduction order. */
typedef struct { uint64_t lo, hi; } sa_key128;

/* A pivot / regular-sample record: global rank key + tie-break. */
typedef struct {
  sa_key128 key;        /* global-rank key (pool = global sample S) */
  int64_t global_idx;   /* index tie-break (reading Z12) */
  int32_t nk;           /* k-mer count of the sequence */
  int32_t block;        /* logical block it was sampled from */
} sa_pivot;

/* Collective operations for sa_partition / sa_redistribute when the
 * context spans several processes (one per GPU).  Implemented by the caller
 * (the Python binding uses torch.distributed over NCCL).  Buffers are device
 * pointers; work must be ordered after prior work on `stream` and later work
 * on `stream` must observe it.  Return 0 on success. */
typedef struct {
  void* user;
  /* recv[r*bytes .. (r+1)*bytes) <- send of rank r, for r = 0..nranks-1 */
  int (*allgather)(void* user, const void* send, void* recv, int64_t bytes, void* stream);
  /* personalised all-to-all of variable byte counts (host arrays of nranks) */
  int (*alltoallv)(void* user, const void* send, const int64_t* send_bytes_h, const int64_t* send_displs_h,
                   void* recv, const int64_t* recv_bytes_h, const int64_t* recv_displs_h, void* stream);
} sa_comm_ops;

/* ------------------------------------------------------------ context ---- */
sa_status sa_ctx_create(int cuda_device, sa_ctx** out);
/* Attach a communicator (collective semantics: every rank attaches with the
 * same nranks).  Once callbacks are attached every exchange goes through them,
 * also for nranks == 1; a context that never attaches makes every exchange a
 * local copy.  `ops` is copied; its `user` pointer must stay valid. */
sa_status sa_ctx_attach_comm(sa_ctx* ctx, const sa_comm_ops* ops, int nranks, int rank);
/* libsa's own NCCL communicator: every exchange of
 * Algorithm 2 then runs as NCCL collectives on the call's stream, with no
 * host code in between -- C1 sample profiles, C2 regular-sample records and
 * C3 count rows by ncclAllGather, C4 the personalised all-to-all (P:625-641,
 * P:1265) by one group of ncclSend / ncclRecv.  sa_nccl_unique_id writes
 * ncclGetUniqueId's 128 bytes (call it on one rank, share them);
 * sa_ctx_attach_nccl is collective (ncclCommInitRank): every rank of the
 * group calls it with the same id and its own rank.  It takes precedence over
 * sa_ctx_attach_comm callbacks; the communicator is destroyed with the
 * context.  NCCL is resolved at run time (the process's libnccl.so.2, e.g.
 * PyTorch's): SA_E_COMM when it is missing or NCCL fails; SA_E_STATE when a
 * communicator is already attached. */
sa_status sa_nccl_unique_id(void* id_h);
sa_status sa_ctx_attach_nccl(sa_ctx* ctx, const void* id_h, int nranks, int rank);
/* Synchronises `stream`, then reports (and clears) the sticky device error
 * flags of the asynchronous calls (sa_kmer_profiles: SA_E_RANGE) and any
 * asynchronous NCCL error of the attached communicator (SA_E_COMM). */
sa_status sa_ctx_check(sa_ctx* ctx, void* stream);
sa_status sa_ctx_destroy(sa_ctx* ctx);
const char* sa_last_error(void);
/* Number of libsa kernels launched through this process since load. */
int64_t sa_launch_count(void);
/* When enabled, libsa records CUDA events around its phases on the call's
 * stream (cudaEventRecord only: recording never blocks the host).  The last
 * SA_PHASE_RING occurrences of every phase are kept, so a caller can run many
 * steps and read every step's phase times afterwards:
 *   sa_ctx_phase_ms       durations of the most recent occurrence of each phase;
 *   sa_ctx_phase_history  durations of the kept occurrences of one phase,
 *                         oldest first.
 * Both are host-blocking (they synchronise on the recorded events); call them
 * outside timed regions.  sa_ctx_set_timing clears the history. */
enum {
  SA_PHASE_S2A = 0,      /* local rank (min-sum engine, all local blocks)      */
  SA_PHASE_S2B = 1,      /* local block sort + sample pick                      */
  SA_PHASE_S2C = 2,      /* sample profile gather / allgather                   */
  SA_PHASE_S2D = 3,      /* global rank (min-sum engine)                        */
  SA_PHASE_S3 = 4,       /* block sort, regular samples, pivots, bucket assign  */
  SA_PHASE_S5 = 5,       /* last sa_bucket_similarity min-sum launch            */
  SA_PHASE_RANK = 6,     /* last sa_kmer_rank min-sum launch                    */
  SA_PHASE_GEMM = 7,     /* the tensor-core GEMM kernel alone of the last K2T launch (any call) */
  SA_PHASE_GEMM_S2A = 8, /* ... of sa_partition's S2a launch                    */
  SA_PHASE_GEMM_S2D = 9, /* ... of sa_partition's S2d launch                    */
  SA_PHASE_GEMM_S5 = 10, /* ... of an sa_bucket_similarity(_batch) launch       */
  SA_PHASE_COUNT = 11
};
enum { SA_PHASE_RING = 64 };
sa_status sa_ctx_set_timing(sa_ctx* ctx, int enable);
/* ms_h[i] for i < min(max, kept occurrences); returns how many were written
 * (0 when the phase never ran, -1 on a CUDA error or bad argument). */
int32_t sa_ctx_phase_history(sa_ctx* ctx, int32_t phase, float* ms_h, int32_t max);
/* Operand encoding of the last min-sum launch on this context:
 * 0 = uint16 counts (VIMNMX.U16x2 min + add; any count), 1 = uint8 counts
 * (C = (nk_a + nk_b - sum|a-b|)/2 with VABSDIFF4.U8.ACC; used when every
 * count is <= 255), 2 = uint16 with FMA-pipe adds (SA_ENGINE=u16imad),
 * 4 = tensor cores: 0/1 threshold layers min(a,b) = sum_r [a>=r][b>=r] as a
 * u8 tcgen05 GEMM (K2T; the default when every count is <= 32
 * and the kept layer columns fit, else the call falls back to 1 / 0 on the
 * device).  SA_ENGINE = auto|tc (default), sad|u8 (no K2T), u16, u16imad.
 * In the auto modes this call synchronises the device to read the choice. */
int sa_ctx_engine(const sa_ctx* ctx);
/* K2T only: the kept threshold-layer columns K' of each problem of the last
 * min-sum call on this context (the contraction length per pair; DESIGN.md
 * §4b), in call order, at most `max` of them.  Returns how many were written
 * (0 when the last call did not run K2T, -1 on a CUDA error).  Synchronises
 * the device.  Problems are: one per block (sa_partition S2a), one (S2d,
 * sa_kmer_rank), one per sa_bucket_similarity call. */
int32_t sa_ctx_tc_columns(const sa_ctx* ctx, int32_t* cols_h, int32_t max);
/* K2T only: how each problem of the last min-sum call on this context handled
 * threshold layers >= 2: mode_h[i] = 1 when problem i ran
 * SPARSE (tensor cores on layer 1 only, plus exact correction terms
 * min(c_i, c_j) - 1 for every bin both rows repeat, added in the GEMM
 * epilogue), 0 when it ran DENSE (layers >= 2 as MMA columns); terms_h[i]
 * (nullable) = its number of correction terms (pair, bin).  Problems in call
 * order as for sa_ctx_tc_columns; at most `max`.  Returns how many were
 * written (0 when the last call did not run K2T, -1 on a CUDA error).
 * Synchronises the device.  Environment: SA_K2T_SPARSE=0 disables the sparse
 * path; SA_K2T_SPARSE_BUDGET=b (default 8) makes a problem sparse when its
 * terms number at most pairs / b. */
int32_t sa_ctx_tc_sparse(const sa_ctx* ctx, int32_t* mode_h, int64_t* terms_h, int32_t max);
/* Self-test of the division-free F = C / D the K2T matrix epilogue uses
 * (Markstein correction on RN(1/D)): compares it bit for bit
 * with IEEE round-to-nearest division for every 0 <= C <= D <= 65535 on
 * `cuda_device` and returns the number of mismatches (expected 0). */
sa_status sa_selftest_f_division(int32_t cuda_device, int64_t* mismatches_h);
/* K2T operand format of this library: 1 = packed e2m1 0/1.0
 * columns on tcgen05 kind::mxf4 (default), 0 = u8 0/1 columns on kind::i8
 * (environment SA_K2T_FP4=0); -1 when the context has not launched K2T.
 * Both are exact. */
int sa_ctx_tc_operand(const sa_ctx* ctx);
sa_status sa_ctx_phase_ms(sa_ctx* ctx, float* ms_h /* [SA_PHASE_COUNT] */);

/* Rank form used by sa_kmer_rank and sa_partition on this context.
 *   SA_RANK_F  (default, BASELINE.json O1): R_i = mean_j F(i,j); keys are the
 *              exact-rank keys above; orders are exact.
 *   SA_RANK_DF (the paper's own Eq. 2-3): R_i =
 *              mean_j d^F(i,j), d^F = -ln(Delta + F) (Delta > 0; SPEC uses
 *              0.02, natural log).  key_i = sum_j round(2^52 (ln(1+Delta) -
 *              ln(Delta + F_ij))) (fixed point, so the sum is deterministic);
 *              rank_f64 = key 2^-52 / npool - ln(1+Delta).  Orders are by key,
 *              ties by index, ascending (most similar first); a comparison is
 *              certified when keys differ by >= 32 npool (log error bound,
 *              DESIGN.md §2 N1); there is no exact fallback -- uncertified
 *              comparisons are only counted (sa_partition_debug.uncertified_h).
 * SA_E_INVAL: unknown form, or Delta <= 0 / not finite for SA_RANK_DF. */
enum { SA_RANK_F = 0, SA_RANK_DF = 1 };
sa_status sa_ctx_set_rank_form(sa_ctx* ctx, int form, double delta);

/* Exact comparison of two ranks over the same pool (host memory, no GPU):
 * sign of V_a - V_b with V_x = sum_j C_xj / min(nk_x, nk_pool[j]) (terms with
 * a zero denominator are 0).  Ca_h / Cb_h: numerator rows [npool] (uint16).
 * Returns -1, 0 or +1; this is the big-integer routine sa_partition uses for
 * comparisons its keys do not certify. */
int sa_exact_rank_compare(const uint16_t* Ca_h, int32_t nka, const uint16_t* Cb_h, int32_t nkb,
                          const int32_t* nk_pool_h, int32_t npool);

/* Row stride (elements) of a profile matrix with `bins` = alphabet^k bins:
 * bins rounded up to a multiple of 64, the extra bins always zero. */
int32_t sa_profile_stride(int32_t bins);

/* ------------------------------------------------------ S1: profiles ---- */
/* c^X for every sequence: profiles[i][t] = number of positions u
 * with id(x_u .. x_{u+k-1}) = t, id = base-`alphabet` big-endian value of
 * the word (reading Z21); nkmers[i] = max(0, n_i - k + 1) (Eq. 1 denominator
 * term).  residues: uint8 codes 0..alphabet-1, CSR by offsets[0..n].
 * profiles: [n][sa_profile_stride(alphabet^k)] uint16 (padding zeroed).
 * SA_E_INVAL (returned): NULL pointer with n > 0, k < 1, alphabet < 2,
 * alphabet^k > 65536.  The call is asynchronous (no host synchronisation):
 * a residue >= alphabet or nk > 65535 (counts / numerators are uint16) sets
 * the context's sticky device flags, reported as SA_E_RANGE by sa_ctx_check
 * or by the next sa_partition on any rank (at its count exchange, C3); the
 * outputs are then unspecified.  n == 0 is a no-op. */
sa_status sa_kmer_profiles(sa_ctx* ctx, const uint8_t* residues, const int64_t* offsets, int32_t n,
                           int32_t k, int32_t alphabet, uint16_t* profiles, int32_t* nkmers, void* stream);

/* ---------------------------------------------------------- S2: rank ---- */
/* Rank of each query against a pool, Eq. 1 averaged (Eq. 3 in F form, reading
 * Z1/O1): R_q = (1/npool) sum_j F(q, j), F = C/D with
 * C = sum_t min(c^q_t, c^j_t) (reading Z3) and D = min(nk_q, nk_j)
 * (F = 0 if D = 0, reading Z4).  The self term is counted when the query is in
 * the pool (reading Z11).
 *   keys[nq]            exact-rank keys (sa_key128, see above)
 *   rank_f64[nq]        nullable: RN(key) * 2^-64 / npool  (|error| <= 2 ulp + npool*2^-64/npool)
 *   numerators[nq][npool] nullable: C as uint16, row-major
 * Profiles use the sa_profile_stride(bins) row stride.
 * SA_E_INVAL: npool == 0 ("empty pool"), NULL required pointer. */
sa_status sa_kmer_rank(sa_ctx* ctx, const uint16_t* q_prof, const int32_t* q_nk, int32_t nq,
                       const uint16_t* pool_prof, const int32_t* pool_nk, int32_t npool, int32_t bins,
                       sa_key128* keys, double* rank_f64, uint16_t* numerators, void* stream);

/* ----------------------------------------------------- S2-S3: partition -- */
/* Optional intermediate artifacts for parity checks (every field nullable). */
typedef struct {
  sa_key128* local_key;      /* [n_local] S2a keys (pool = own logical block)      */
  double* local_f64;         /* [n_local] S2a rank fp64                            */
  int64_t* local_order;      /* [n_local] S2b: global ids, each block sorted        */
  int64_t* sample_idx;       /* [p*samples_per_block] global sample S, (q, j) order */
  sa_key128* global_key;     /* [n_local] S2d keys (pool = S)                      */
  double* global_f64;        /* [n_local] S2d rank fp64                            */
  int64_t* global_order;     /* [n_local] S3a: global ids, each block sorted        */
  int64_t* candidates;       /* [p*(p-1)] S3b: sorted regular samples Y (global ids) */
  int32_t* exact_fallbacks_h;/* host int: ambiguous key comparisons resolved exactly */
  int32_t* uncertified_h;    /* host int: (d^F form) comparisons inside the error window */
  uint16_t* global_num;      /* [n_local][p*samples_per_block] S2d numerators C (row-major, columns in S's
                                (q, j) order), written by the S2d GEMM epilogue itself          */
} sa_partition_debug;

/* Algorithm 2 steps 1-11, the rank-based sample sort:
 *  - p logical blocks; block q = global ids [floor(qN/p), floor((q+1)N/p))
 *    (reading Z13).  The calling rank (of nranks) holds blocks
 *    [rank*p/nranks, (rank+1)*p/nranks) as a contiguous shard starting at
 *    global id first_global with n_local sequences: profiles/nkmers/offsets
 *    describe that shard (offsets: its residue CSR, used for byte counts).
 *  - S2a local rank vs own block, S2b sort + k_b samples
 *    at floor((j+1)w/(k_b+1)), S2c the s = p*k_b sample
 *    profiles replicated on every rank (profiles instead of residues,
 *    DESIGN.md §5), S2d rank vs S, S3a sort + p-1 regular samples at
 *    floor((j+1)w/p), S3b sort Y, pivots Y_{floor(p/2)+jp}
 *    (reading Z9; every rank derives the same pivots, O2),
 *    S3c bucket(i) = min{b : (R_i, i) <= pivot_b}, else p-1.
 *  - every order is by the exact rational rank, ties by global index (O4):
 *    keys decide when certified; otherwise the pair is resolved exactly on
 *    the host with big-integer arithmetic (rare).
 * Outputs: bucket_of[n_local] (device), pivots[p-1] (device),
 *   counts_h[nranks*p]: counts_h[r*p+b] = sequences of rank r in bucket b,
 *   bytes_h[nranks*p]: their residue bytes -- the receive sizes for
 *   sa_redistribute (host; filled on every rank).
 * Host-blocking: once, at the count exchange (C3); more in the exact path.
 * SA_E_INVAL: p < 1, n_total < p, nranks does not divide p, the shard does not
 * match blocks [rank*p/nranks, (rank+1)*p/nranks), samples_per_block < 1 or
 * larger than a block, NULL required pointers. */
sa_status sa_partition(sa_ctx* ctx, int32_t p, int32_t samples_per_block,
                       const uint16_t* profiles, const int32_t* nkmers, const int64_t* offsets, int32_t bins,
                       int64_t n_total, int64_t first_global, int32_t n_local,
                       int32_t* bucket_of, sa_pivot* pivots, int64_t* counts_h, int64_t* bytes_h,
                       sa_partition_debug* dbg, void* stream);

/* ------------------------------------------------- S4: redistribution ---- */
/* All-to-all personalised redistribution: every
 * sequence of the local shard goes to the rank owning its bucket (rank r owns
 * buckets [r*p/nranks, (r+1)*p/nranks)).  Received sequences are ordered by
 * (bucket, global id) (reading Z17).  Inputs: the shard's residue CSR, the
 * sa_partition outputs bucket_of / counts_h / bytes_h.  Outputs (device,
 * caller-sized from counts_h / bytes_h): recv_residues[sum bytes],
 * recv_offsets[recv_n+1], recv_global_idx[recv_n], recv_bucket[recv_n]. */
sa_status sa_redistribute(sa_ctx* ctx, int32_t p, const uint8_t* residues, const int64_t* offsets,
                          int32_t n_local, int64_t first_global, const int32_t* bucket_of,
                          const int64_t* counts_h, const int64_t* bytes_h,
                          uint8_t* recv_residues, int64_t* recv_offsets, int64_t* recv_global_idx,
                          int32_t* recv_bucket, void* stream);

/* -------------------------------------------- S5: bucket similarity ----- */
/* All-pairs k-mer similarity inside one bucket (the pairwise stage of
 * distance-based MSA; Eq. 1): for members in the given
 * order, numerators[i][j] = C_ij (uint16), similarity[i][j] = C_ij / D_ij in
 * fp64 with one IEEE round-to-nearest division (reading Z19), 0 if D_ij = 0
 * (so a member with nk = 0 has self-similarity 0, reading Z4).  Both outputs
 * are full symmetric n x n row-major matrices; each is nullable. */
sa_status sa_bucket_similarity(sa_ctx* ctx, const uint16_t* profiles, const int32_t* nkmers, int32_t n,
                               int32_t bins, uint16_t* numerators, double* similarity, void* stream);

/* The same for several buckets in one call (one engine launch over all of
 * them: the operand preparation and the tile schedule are shared, so many
 * small buckets cost no more launches than one large one).  Bucket b is rows
 * [row_begin_h[b], row_begin_h[b+1]) of `profiles` / `nkmers` (the layout
 * sa_redistribute produces: buckets contiguous, members ascending by global
 * id); its outputs are numerators_h[b] / similarity_h[b] (host arrays of
 * device pointers, each [n_b][n_b]; the arrays and any entry are nullable).
 * ld_h (host, nullable): row stride in elements of bucket b's matrices,
 * ld_h[b] >= n_b (NULL: n_b, dense); the columns [n_b, ld_h[b]) are not
 * written.  A multiple of 16 makes every row start on a 32-byte sector, so
 * the epilogue's stores are whole sectors (no partial-sector merges in L2).
 * Empty buckets are skipped.  SA_E_INVAL: nbuckets < 0, row_begin_h not
 * non-decreasing from 0, bad bins, NULL profiles / nkmers with rows,
 * ld_h[b] < n_b. */
sa_status sa_bucket_similarity_batch(sa_ctx* ctx, int32_t nbuckets, const uint16_t* profiles, const int32_t* nkmers,
                                     const int64_t* row_begin_h, int32_t bins, uint16_t* const* numerators_h,
                                     double* const* similarity_h, const int64_t* ld_h, void* stream);

/* --------------------------------------------- N4: bucket guide tree ----- */
/* The guide tree the underlying MSA builds from a bucket's similarity matrix
 * (SPEC build_guide_tree S:277-285): UPGMA on
 * d = 1 - F (readings T1-T3): n - 1 merges of the active pair
 * (a, b), a < b, of largest F, ties to the smallest (a, b); a cluster's id is
 * its smallest member; F(ab, c) = (n_a F_ac + n_b F_bc) / (n_a + n_b) with
 * IEEE round-to-nearest on every operation; merge height (1 - F_ab) / 2.
 * Inputs: similarity [n][ld] (device, row-major, symmetric; the diagonal is
 * ignored).  Outputs (device): merges [n-1][2] (a, b), heights [n-1], in
 * merge order (n = 1: nothing written).  The distance is the context's tree
 * form (sa_ctx_set_tree_form below; default d = 1 - F, heights (1 - F_ab) / 2
 * as above).  The merges are sequential; each
 * is O(n): n < 1024 runs them on one CTA, larger n on every SM of the device
 * (one cooperative launch, two device-wide barriers per merge; the same IEEE
 * operations and tie orders, so the same tree; SA_UPGMA_GRID=0/1 forces
 * either).  O(n^2) work, n^2 + O(n) doubles of scratch.  SA_E_INVAL: n < 1,
 * ld < n, NULL pointers. */
sa_status sa_guide_tree(sa_ctx* ctx, const double* similarity, int32_t n, int64_t ld, int32_t* merges,
                        double* heights, void* stream);

/* N4's distance (reading T4):
 *   SA_TREE_F  (default, reading T1): d = 1 - F -- UPGMA is then average
 *              linkage on F itself, every decision IEEE arithmetic on F;
 *   SA_TREE_DF (Eq. 2; "Eq. 2 distances"): d_ij =
 *              CR(-ln(RN(Delta + F_ij))), the double nearest the real -ln of
 *              the once-rounded Delta + F; UPGMA on d as above with "largest
 *              F" read as "smallest d", d(ab, c) = RN(RN(RN(n_a d_ac) +
 *              RN(n_b d_bc)) / (n_a + n_b)), height d_ab / 2.
 * The log is evaluated in double-double (~2^-100 relative error) and rounded
 * once; an element whose double-double value lies too close to a rounding
 * boundary to certify the rounding keeps the nearest double and is counted
 * (sa_ctx_tree_uncertified) -- the window treatment of N1.  Applies to
 * sa_guide_tree and sa_guide_tree_batch.  SA_E_INVAL: unknown form, Delta <=
 * 0 or not finite for SA_TREE_DF. */
enum { SA_TREE_F = 0, SA_TREE_DF = 1 };
sa_status sa_ctx_set_tree_form(sa_ctx* ctx, int form, double delta);
/* Uncertified correctly-rounded logs of the last tree call (0 for SA_TREE_F).
 * Blocks on `stream` (the stream of that call). */
sa_status sa_ctx_tree_uncertified(sa_ctx* ctx, int64_t* count_h, void* stream);

/* The guide trees of `count` buckets at once (same definition and outputs as
 * sa_guide_tree, tree i from similarity_h[i] [n_h[i]][ld_h[i]] into
 * merges_h[i] / heights_h[i]): one cooperative launch whose resident blocks
 * are shared out among the trees in proportion to n^2, each tree merging on
 * its own blocks with its own barriers -- the trees' sequential merge chains
 * run side by side.  Host arrays of device pointers; n = 1 trees are
 * skipped.  Synchronises `stream` before returning (the launch's task table
 * is host-built).  SA_E_INVAL: count < 0, bad n / ld, NULL pointers. */
sa_status sa_guide_tree_batch(sa_ctx* ctx, int32_t count, const double* const* similarity_h, const int32_t* n_h,
                              const int64_t* ld_h, int32_t* const* merges_h, double* const* heights_h, void* stream);

/* Packed upper triangle (diagonal included) of a symmetric n x n uint16
 * matrix with row stride ld >= n: row i's columns i..n-1 at packed offset
 * i*n - i*(i-1)/2, n(n+1)/2 elements in all -- the complete content of a
 * bucket's numerator matrix in half the bytes (the end-to-end bench moves
 * these to the host).  Device pointers; enqueued on `stream`.  SA_E_INVAL:
 * n < 0, ld < n, NULL pointers with n > 0. */
sa_status sa_pack_upper_u16(sa_ctx* ctx, const uint16_t* matrix, int32_t n, int64_t ld, uint16_t* packed,
                            void* stream);
/* The same for a symmetric fp64 similarity matrix (S5's F): n(n+1)/2 doubles. */
sa_status sa_pack_upper_f64(sa_ctx* ctx, const double* matrix, int32_t n, int64_t ld, double* packed, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SA_H_ */
