// K2T sparse layers >= 2 (tc_sparse.cu): launch description,
// device buffers and the entry format the GEMM epilogue consumes.
#pragma once
#include <cstdint>

#include "tc_gemm.cuh"

namespace sa {

constexpr int SP_BINS = 8192;                 // bins per side (TC_MAX_BINS)
constexpr int SP_BSTRIDE = SP_BINS + 1;       // binoff row: SP_BINS starts + the side's end
constexpr uint32_t SP_DEAD = 0xFFFF0000u;     // merged-away entry: column 0xFFFF is never in a tile
constexpr int SP_TN_MAX = 1024;               // column blocks per sparse problem (the row build's counters)

// A correction entry: (column within the tile's column block) << 16 | term,
// term = sum over the pair's shared repeated bins of min(c_i, c_j) - 1.
// Entries are grouped by key = (row of the problem's A side, column block):
// ents[koff[key] .. koff[key + 1]) sorted by column, and kpart[key] holds the
// entry count of each epilogue slice (8 bits per slice, slices in order).
// Record (appended by the histogram pass): x = row index in the launch's
// flattened rows, y = bin | count << 16.

struct SpLaunch {
  int64_t row_begin[2 * tc::MAXPROB + 1];   // sides, as in TcSides
  int nsides;
  int nprob;
  int side_a[tc::MAXPROB], side_b[tc::MAXPROB];   // side_b = -1: symmetric
  uint64_t key_base[tc::MAXPROB + 1];             // key index base of each problem
  int64_t abase[tc::MAXPROB + 1];                 // first A-side row of each problem (over all problems)
  int32_t tn[tc::MAXPROB];                        // column blocks of each problem
  uint64_t cap[tc::MAXPROB];                      // entry budget: sparse iff terms <= cap
  int64_t nkeys;                                  // keys = (row, column block) of every problem
  int bn, slice;                                  // column-block width, epilogue slice width
  uint32_t rec_cap;
  int enabled;                                    // 0: every problem dense (SA_K2T_SPARSE=0)
  unsigned long long* terms_out;                  // nullable: E of each problem (diagnostics)
};

struct SpBuffers {
  uint2* recs = nullptr;        // [rec_cap]
  uint32_t* nrec = nullptr;     // [0] record count, [1] carried count, [2] incomplete, [3] carried incomplete
  uint32_t* povf = nullptr;     // [MAXPROB] problem whose records overflowed (runs dense)
  uint32_t* bincnt = nullptr;   // [nsides][SP_BINS] (zeroed by the caller)
  uint32_t* binoff = nullptr;   // [nsides][SP_BSTRIDE]
  uint32_t* sidebase = nullptr; // [nsides] record totals per side (zeroed by the caller)
  uint2* blist = nullptr;       // [rec_cap] bin lists as scattered
  uint2* sorted = nullptr;      // [rec_cap] bin lists sorted by row
  uint32_t* bslot = nullptr;    // [rec_cap] row-list slot of each bin-list entry
  uint32_t* spos = nullptr;     // [rec_cap] per row-list slot: the record's position in its sorted bin list
  uint32_t* rcnt = nullptr;     // [R] records per launch row (zeroed by the caller)
  uint32_t* rstart = nullptr;   // [R + 1]
  uint32_t* rlist = nullptr;    // [rec_cap] row lists: bin | count << 16
  int32_t* mode = nullptr;      // [nprob] 1 = sparse
  uint32_t* flags = nullptr;    // [0] bit 0: some problem is sparse (zeroed by the caller)
  uint32_t* rowcnt = nullptr;   // [NA] terms per A-side row
  uint32_t* rowoff = nullptr;   // [NA + 1]
  uint32_t* koff = nullptr;     // [nkeys + 1]
  uint32_t* kpart = nullptr;    // [nkeys] entries per epilogue slice, 8 bits each
  uint32_t* scan_tmp = nullptr; // [max(R, NA) / 4096 + 2]
  uint32_t* ents = nullptr;     // [sum of caps]
};

// bin counts of the records and the per-problem plan (mode, flags)
sa_status sp_build(SpLaunch& L, SpBuffers& B, int sms, cudaStream_t st);
// bin lists, keys, entries (every kernel returns at once unless flags say some problem is sparse)
sa_status sp_entries(SpLaunch& L, SpBuffers& B, int sms, cudaStream_t st);
sa_status sp_copy_records(const uint2* src, const uint32_t* nsrc, uint32_t src_cap, uint2* dst, uint32_t* ndst,
                          int sms, cudaStream_t st);

}  // namespace sa
