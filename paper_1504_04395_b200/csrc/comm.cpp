// comm.cpp — NCCL plumbing for the multi-GPU path: one
// communicator per process (one process per GPU), created from a unique id that
// the caller broadcasts with torch.distributed. NCCL is resolved at run time with
// dlopen (the libnccl.so.2 torch already loaded, else the system one), so the
// library still loads on machines without NCCL; single-GPU use never touches it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "comm.h"

namespace srk {

using PFN_getUniqueId = ncclResult_t (*)(ncclUniqueId*);
using PFN_commInitRank = ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int);
using PFN_commDestroy = ncclResult_t (*)(ncclComm_t);
using PFN_allReduce = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                       cudaStream_t);
using PFN_send = ncclResult_t (*)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
using PFN_recv = ncclResult_t (*)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
using PFN_group = ncclResult_t (*)();
using PFN_errstr = const char* (*)(ncclResult_t);

struct Nccl {
  void* h = nullptr;
  PFN_getUniqueId getUniqueId = nullptr;
  PFN_commInitRank commInitRank = nullptr;
  PFN_commDestroy commDestroy = nullptr;
  PFN_allReduce allReduce = nullptr;
  PFN_send send = nullptr;
  PFN_recv recv = nullptr;
  PFN_group groupStart = nullptr;
  PFN_group groupEnd = nullptr;
  PFN_errstr errstr = nullptr;
};

static Nccl* nccl() {
  static Nccl N;
  static bool tried = false;
  if (tried) return N.h ? &N : nullptr;
  tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    N.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
    if (N.h) break;
  }
  if (!N.h)
    for (const char* nm : names) {
      N.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (N.h) break;
    }
  if (!N.h) return nullptr;
  N.getUniqueId = (PFN_getUniqueId)dlsym(N.h, "ncclGetUniqueId");
  N.commInitRank = (PFN_commInitRank)dlsym(N.h, "ncclCommInitRank");
  N.commDestroy = (PFN_commDestroy)dlsym(N.h, "ncclCommDestroy");
  N.allReduce = (PFN_allReduce)dlsym(N.h, "ncclAllReduce");
  N.send = (PFN_send)dlsym(N.h, "ncclSend");
  N.recv = (PFN_recv)dlsym(N.h, "ncclRecv");
  N.groupStart = (PFN_group)dlsym(N.h, "ncclGroupStart");
  N.groupEnd = (PFN_group)dlsym(N.h, "ncclGroupEnd");
  N.errstr = (PFN_errstr)dlsym(N.h, "ncclGetErrorString");
  if (!N.getUniqueId || !N.commInitRank || !N.allReduce || !N.send || !N.recv || !N.groupStart || !N.groupEnd) {
    N.h = nullptr;
    return nullptr;
  }
  return &N;
}

bool nccl_available() { return nccl() != nullptr; }

int nccl_unique_id(void* out128) {
  Nccl* N = nccl();
  if (!N) return -1;
  ncclUniqueId id;
  if (N->getUniqueId(&id) != ncclSuccess) return -2;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return 0;
}

Comm* comm_create(const void* id128, int nranks, int rank) {
  Nccl* N = nccl();
  if (!N) return nullptr;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  if (N->commInitRank(&c, nranks, id, rank) != ncclSuccess) return nullptr;
  auto* C = new Comm();
  C->nranks = nranks;
  C->rank = rank;
  C->nccl = c;
  return C;
}

void comm_destroy(Comm* C) {
  if (!C) return;
  if (C->vg) {  // the group is owned by its srk_vgroup handle
    delete C;
    return;
  }
  Nccl* N = nccl();
  if (N && N->commDestroy) N->commDestroy((ncclComm_t)C->nccl);
  delete C;
}

int comm_allreduce_sum(Comm* C, double* buf, size_t count, cudaStream_t st) {
  if (!C || C->nranks == 1 || count == 0) return 0;
  if (C->vg) return -5;  // the virtual group reduces out of place only (comm_allreduce_sum_many)
  Nccl* N = nccl();
  return N->allReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)C->nccl, st) == ncclSuccess ? 0 : -5;
}

int comm_allreduce_sum_many(Comm* C, const double* const* src, double* const* dst, const size_t* counts, int nbuf,
                            cudaStream_t st) {
  if (!C || C->nranks == 1 || nbuf == 0) return 0;
  if (C->vg) return vgroup_allreduce(C->vg, C->rank, src, dst, counts, nbuf, st);
  Nccl* N = nccl();
  if (N->groupStart() != ncclSuccess) return -5;
  int bad = 0;
  for (int i = 0; i < nbuf; ++i)
    if (counts[i] && N->allReduce(src[i], dst[i], counts[i], ncclFloat64, ncclSum, (ncclComm_t)C->nccl, st) != ncclSuccess)
      bad = 1;
  return (N->groupEnd() == ncclSuccess && !bad) ? 0 : -5;
}

int comm_halo(Comm* C, const double* sendbuf, const int64_t* send_off, double* recvbuf, const int64_t* recv_off,
              size_t doubles_per_row, cudaStream_t st) {
  if (!C || C->nranks == 1) return 0;
  if (C->vg) return vgroup_halo(C->vg, C->rank, sendbuf, send_off, recvbuf, recv_off, doubles_per_row, st);
  Nccl* N = nccl();
  if (N->groupStart() != ncclSuccess) return -5;
  for (int p = 0; p < C->nranks; ++p) {
    if (p == C->rank) continue;
    const int64_t ns = send_off[p + 1] - send_off[p];
    const int64_t nr = recv_off[p + 1] - recv_off[p];
    if (ns > 0) N->send(sendbuf + send_off[p] * doubles_per_row, ns * doubles_per_row, ncclFloat64, p,
                        (ncclComm_t)C->nccl, st);
    if (nr > 0) N->recv(recvbuf + recv_off[p] * doubles_per_row, nr * doubles_per_row, ncclFloat64, p,
                        (ncclComm_t)C->nccl, st);
  }
  return N->groupEnd() == ncclSuccess ? 0 : -5;
}

}  // namespace srk
