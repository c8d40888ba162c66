// comm.h — multi-GPU plumbing (NCCL over NVLink/NVSwitch), see comm.cpp.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace srk {

struct VGroup;  // single-GPU virtual partition (vcomm.cu)

struct Comm {
  int nranks = 1, rank = 0;
  void* nccl = nullptr;  // ncclComm_t
  VGroup* vg = nullptr;  // set: virtual rank `rank` of a VGroup on this GPU (no NCCL)
};

VGroup* vgroup_create(int k);
void vgroup_destroy(VGroup* g);
int vgroup_size(const VGroup* g);
int vgroup_allreduce(VGroup* g, int rank, const double* const* src, double* const* dst, const size_t* counts, int nbuf,
                     cudaStream_t st);
int vgroup_halo(VGroup* g, int rank, const double* sendbuf, const int64_t* send_off, double* recvbuf,
                const int64_t* recv_off, size_t doubles_per_row, cudaStream_t st);

bool nccl_available();
int nccl_unique_id(void* out128);
Comm* comm_create(const void* id128, int nranks, int rank);
void comm_destroy(Comm* c);
// in-place FP64 sum over ranks (ring/tree: the same bitwise result on every rank)
int comm_allreduce_sum(Comm* c, double* buf, size_t count, cudaStream_t st);
// several sums as one grouped call (one latency per reduction point): dst[i] = sum over
// ranks of src[i] (src[i] == dst[i] allowed); NCCL ranks or the virtual group
int comm_allreduce_sum_many(Comm* c, const double* const* src, double* const* dst, const size_t* counts, int nbuf,
                            cudaStream_t st);
// grouped point-to-point halo exchange: rows [send_off[p], send_off[p+1]) of sendbuf go
// to rank p, rows [recv_off[p], recv_off[p+1]) of recvbuf come from rank p
int comm_halo(Comm* c, const double* sendbuf, const int64_t* send_off, double* recvbuf, const int64_t* recv_off,
              size_t doubles_per_row, cudaStream_t st);

// halo plan of one distributed operator (A or A^H)
struct Halo {
  int nranks = 1;
  long long n_ghost = 0, n_send = 0;
  int* send_idx = nullptr;   // device, n_send local rows to pack, grouped by peer
  int64_t* send_off = nullptr;  // host, nranks + 1 (rows)
  int64_t* recv_off = nullptr;  // host, nranks + 1 (rows, relative to n_local)
};

}  // namespace srk
