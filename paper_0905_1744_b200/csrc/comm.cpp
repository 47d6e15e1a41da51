// libsa's own NCCL communicator (sa_ctx_attach_nccl, include/sa.h).
//
// Algorithm 2's exchanges (the two communication rounds
// of the cost model) are collectives on the context's stream:
//   C1 sample profiles / C2 regular-sample records / C3 count rows -> ncclAllGather
//   C4 the all-to-all personalised redistribution       -> grouped ncclSend / ncclRecv
// NCCL is resolved at run time (dlopen): the library the process already
// loaded (PyTorch's) when there is one, else libnccl.so.2 from the loader's
// path.  Without NCCL every NCCL entry point returns SA_E_COMM.
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "common.cuh"
#include "comm.h"

namespace sa {
namespace {

// The NCCL ABI subset libsa calls (types mirror nccl.h: an opaque comm
// pointer, a 128-byte unique id, int enums).
typedef int nccl_result;
typedef void* nccl_comm;
struct nccl_id {
  char internal[128];
};
enum { NCCL_CHAR = 0 };   // ncclInt8 / ncclChar

struct NcclApi {
  bool ok = false;
  nccl_result (*get_unique_id)(nccl_id*) = nullptr;
  nccl_result (*comm_init_rank)(nccl_comm*, int, nccl_id, int) = nullptr;
  nccl_result (*comm_destroy)(nccl_comm) = nullptr;
  nccl_result (*comm_get_async_error)(nccl_comm, nccl_result*) = nullptr;
  nccl_result (*all_gather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*group_start)() = nullptr;
  nccl_result (*group_end)() = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // already in the process (PyTorch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name)); };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.comm_get_async_error, "ncclCommGetAsyncError");
    sym(api.all_gather, "ncclAllGather");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.send && api.recv &&
             api.group_start && api.group_end;
  });
  return api;
}

sa_status nccl_fail(nccl_result r, const char* what) {
  const NcclApi& A = nccl();
  return fail(SA_E_COMM, "%s: NCCL error %d (%s)", what, r, A.error_string ? A.error_string(r) : "?");
}

}  // namespace

bool nccl_available() { return nccl().ok; }

sa_status nccl_unique_id(void* id_h) {
  const NcclApi& A = nccl();
  if (!A.ok) return fail(SA_E_COMM, "NCCL is not available (libnccl.so.2 not found)");
  nccl_id id;
  const nccl_result r = A.get_unique_id(&id);
  if (r != 0) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_h, &id, sizeof id);
  return SA_OK;
}

sa_status nccl_init(void** comm_out, const void* id_h, int nranks, int rank) {
  const NcclApi& A = nccl();
  if (!A.ok) return fail(SA_E_COMM, "NCCL is not available (libnccl.so.2 not found)");
  nccl_id id;
  std::memcpy(&id, id_h, sizeof id);
  nccl_comm c = nullptr;
  const nccl_result r = A.comm_init_rank(&c, nranks, id, rank);
  if (r != 0) return nccl_fail(r, "ncclCommInitRank");
  *comm_out = c;
  return SA_OK;
}

void nccl_destroy(void* comm) {
  const NcclApi& A = nccl();
  if (A.ok && comm) A.comm_destroy(static_cast<nccl_comm>(comm));
}

sa_status nccl_check(void* comm) {
  const NcclApi& A = nccl();
  if (!A.ok || !comm || !A.comm_get_async_error) return SA_OK;
  nccl_result async = 0;
  const nccl_result r = A.comm_get_async_error(static_cast<nccl_comm>(comm), &async);
  if (r != 0) return nccl_fail(r, "ncclCommGetAsyncError");
  if (async != 0) return nccl_fail(async, "NCCL communicator (asynchronous error)");
  return SA_OK;
}

sa_status nccl_allgather(void* comm, const void* send, void* recv, int64_t bytes, cudaStream_t st) {
  const NcclApi& A = nccl();
  if (bytes <= 0) return SA_OK;
  const nccl_result r = A.all_gather(send, recv, (size_t)bytes, NCCL_CHAR, static_cast<nccl_comm>(comm), st);
  if (r != 0) return nccl_fail(r, "ncclAllGather");
  return SA_OK;
}

// Personalised all-to-all: one NCCL group of point-to-point transfers (the
// rank's own block is a device copy).
sa_status nccl_alltoallv(void* comm, int nranks, int rank, const void* send, const int64_t* send_bytes,
                         const int64_t* send_displs, void* recv, const int64_t* recv_bytes,
                         const int64_t* recv_displs, cudaStream_t st) {
  const NcclApi& A = nccl();
  const uint8_t* s = static_cast<const uint8_t*>(send);
  uint8_t* d = static_cast<uint8_t*>(recv);
  if (send_bytes[rank] != recv_bytes[rank]) return fail(SA_E_COMM, "alltoallv: own block sizes differ");
  if (send_bytes[rank] > 0)
    SA_CUDA(cudaMemcpyAsync(d + recv_displs[rank], s + send_displs[rank], send_bytes[rank], cudaMemcpyDeviceToDevice,
                            st));
  nccl_result r = A.group_start();
  if (r != 0) return nccl_fail(r, "ncclGroupStart");
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) continue;
    if (send_bytes[p] > 0) {
      r = A.send(s + send_displs[p], (size_t)send_bytes[p], NCCL_CHAR, p, static_cast<nccl_comm>(comm), st);
      if (r != 0) {
        A.group_end();
        return nccl_fail(r, "ncclSend");
      }
    }
    if (recv_bytes[p] > 0) {
      r = A.recv(d + recv_displs[p], (size_t)recv_bytes[p], NCCL_CHAR, p, static_cast<nccl_comm>(comm), st);
      if (r != 0) {
        A.group_end();
        return nccl_fail(r, "ncclRecv");
      }
    }
  }
  r = A.group_end();
  if (r != 0) return nccl_fail(r, "ncclGroupEnd");
  return SA_OK;
}

}  // namespace sa
