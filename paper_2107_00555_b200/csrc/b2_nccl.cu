// b2_nccl.cu — NCCL collectives/P2P issued from libb2 on the executor's own
// stream, so halo exchanges and SUMMA broadcasts are captured in the same
// CUDA graph as the kernels (one graph launch per program run on every rank).
//
// libnccl is dlopen'ed ("libnccl.so.2": the one torch already loaded, else the
// system copy) so libb2 still loads on hosts without NCCL.
//
// Replaces the reference's simulated communication library nodes (ISEND /
// IRECV / WAITALL / BCAST / DIST_MATMUL events serviced by the missing rank
// simulator, interp.py:443-447, 483-489).

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>

#include "b2.h"
#include "b2_internal.h"

namespace {

typedef struct {
  char internal[128];
} NcclId;
typedef void *NcclComm;
typedef int (*PFN_GetUniqueId)(NcclId *);
typedef int (*PFN_CommInitRank)(NcclComm *, int, NcclId, int);
typedef int (*PFN_CommDestroy)(NcclComm);
typedef int (*PFN_Group)(void);
typedef int (*PFN_Send)(const void *, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*PFN_Recv)(void *, size_t, int, int, NcclComm, cudaStream_t);
// ncclBroadcast(sendbuff, recvbuff, count, datatype, root, comm, stream)
typedef int (*PFN_Bcast)(const void *, void *, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*PFN_AllReduce)(const void *, void *, size_t, int, int, NcclComm, cudaStream_t);
typedef const char *(*PFN_ErrStr)(int);

struct Nccl {
  std::once_flag once;
  void *h = nullptr;
  PFN_GetUniqueId getUniqueId = nullptr;
  PFN_CommInitRank commInitRank = nullptr;
  PFN_CommDestroy commDestroy = nullptr;
  PFN_Group groupStart = nullptr, groupEnd = nullptr;
  PFN_Send send = nullptr;
  PFN_Recv recv = nullptr;
  PFN_Bcast bcast = nullptr;
  PFN_AllReduce allReduce = nullptr;
  PFN_ErrStr errStr = nullptr;
} nc;

// ncclDataType_t / ncclRedOp_t values from nccl.h
constexpr int kNcclInt8 = 0, kNcclFloat64 = 8;
constexpr int kNcclSum = 0, kNcclProd = 1, kNcclMax = 2, kNcclMin = 3;

int load() {
  std::call_once(nc.once, [] {
    nc.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!nc.h) return;
#define B2_SYM(field, name, T) nc.field = (T)dlsym(nc.h, name);
    B2_SYM(getUniqueId, "ncclGetUniqueId", PFN_GetUniqueId)
    B2_SYM(commInitRank, "ncclCommInitRank", PFN_CommInitRank)
    B2_SYM(commDestroy, "ncclCommDestroy", PFN_CommDestroy)
    B2_SYM(groupStart, "ncclGroupStart", PFN_Group)
    B2_SYM(groupEnd, "ncclGroupEnd", PFN_Group)
    B2_SYM(send, "ncclSend", PFN_Send)
    B2_SYM(recv, "ncclRecv", PFN_Recv)
    B2_SYM(bcast, "ncclBroadcast", PFN_Bcast)
    B2_SYM(allReduce, "ncclAllReduce", PFN_AllReduce)
    B2_SYM(errStr, "ncclGetErrorString", PFN_ErrStr)
#undef B2_SYM
  });
  if (!nc.h || !nc.send || !nc.commInitRank)
    return b2_fail(B2_ERR_UNSUPPORTED, "libnccl.so.2 not available: %s", dlerror());
  return B2_OK;
}

int nccl_check(int r, const char *what) {
  if (r == 0) return B2_OK;
  return b2_fail(B2_ERR_CUDA, "%s: %s", what, nc.errStr ? nc.errStr(r) : "nccl error");
}

}  // namespace

extern "C" int b2_nccl_unique_id(void *out128) {
  int rc = load();
  if (rc) return rc;
  NcclId id;
  rc = nccl_check(nc.getUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(out128, &id, sizeof id);
  return B2_OK;
}

extern "C" int b2_nccl_init(int nranks, int rank, const void *id128, void **comm) {
  int rc = load();
  if (rc) return rc;
  NcclId id;
  memcpy(&id, id128, sizeof id);
  NcclComm c = nullptr;
  rc = nccl_check(nc.commInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm = c;
  return B2_OK;
}

extern "C" int b2_nccl_destroy(void *comm) {
  int rc = load();
  if (rc) return rc;
  return nccl_check(nc.commDestroy(comm), "ncclCommDestroy");
}

extern "C" int b2_nccl_group_p2p(void *comm, int n, const b2_p2p_t *ops, void *stream) {
  int rc = load();
  if (rc) return rc;
  if (n <= 0) return B2_OK;
  rc = nccl_check(nc.groupStart(), "ncclGroupStart");
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    const b2_p2p_t &o = ops[i];
    int r = o.send ? nc.send(o.ptr, o.bytes, kNcclInt8, o.peer, comm, (cudaStream_t)stream)
                   : nc.recv(o.ptr, o.bytes, kNcclInt8, o.peer, comm, (cudaStream_t)stream);
    if (r != 0) {
      nc.groupEnd();
      return nccl_check(r, o.send ? "ncclSend" : "ncclRecv");
    }
  }
  return nccl_check(nc.groupEnd(), "ncclGroupEnd");
}

extern "C" int b2_nccl_bcast(void *comm, void *buf, size_t bytes, int root, void *stream) {
  int rc = load();
  if (rc) return rc;
  return nccl_check(nc.bcast(buf, buf, bytes, kNcclInt8, root, comm, (cudaStream_t)stream),
                    "ncclBroadcast");
}

extern "C" int b2_nccl_allreduce_f64(void *comm, double *buf, size_t count, int wcr,
                                     void *stream) {
  int op;
  switch (wcr) {  // Wcr.ADD / MUL / MIN / MAX (ir.py:72-91); anything else is an error
    case B2_WCR_ADD: op = kNcclSum; break;
    case B2_WCR_MUL: op = kNcclProd; break;
    case B2_WCR_MIN: op = kNcclMin; break;
    case B2_WCR_MAX: op = kNcclMax; break;
    default:
      return b2_fail(B2_ERR_UNSUPPORTED, "b2_nccl_allreduce_f64: unsupported wcr code %d", wcr);
  }
  int rc = load();
  if (rc) return rc;
  return nccl_check(nc.allReduce(buf, buf, count, kNcclFloat64, op, comm, (cudaStream_t)stream),
                    "ncclAllReduce");
}
