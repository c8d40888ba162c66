// vcomm.cu — single-GPU "virtual partition" transport ("Multi-GPU without a
// cluster"): k row blocks of one operator on one GPU, one host thread and one stream per
// virtual rank, driving the SAME distributed solver code as the NCCL ranks (Eng::halo's
// pack kernel and ghost tail, finish_reds' per-reduction-point allreduce). Only the
// transport differs:
//   * halo: every rank packs its send rows (the same gather kernel), then each receiver
//     copies its ghost ranges device-to-device out of its peers' send buffers;
//   * allreduce: every rank sums the k ranks' partial vectors in RANK ORDER (one small
//     kernel per rank, identical bits on every rank).
// Cross-rank ordering uses CUDA events (cudaStreamWaitEvent) plus host barriers between
// the threads; no kernel ever waits on another kernel (B200_PROFILING.md: kernels that
// wait on one another must not share a GPU), so this is safe on one device.
#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "comm.h"

namespace srk {

constexpr int VMAX_RANKS = 16;
constexpr int VMAX_BUF = 8;

struct VGroup {
  int k = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<cudaEvent_t> ready, used;
  // per-rank registrations of the current collective (host data, valid between barriers)
  std::vector<std::vector<const double*>> src;
  std::vector<const double*> sendbuf;
  std::vector<const int64_t*> send_off;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == k) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

VGroup* vgroup_create(int k) {
  if (k < 1 || k > VMAX_RANKS) return nullptr;
  auto* G = new VGroup();
  G->k = k;
  G->ready.resize(k);
  G->used.resize(k);
  for (int r = 0; r < k; ++r) {
    if (cudaEventCreateWithFlags(&G->ready[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&G->used[r], cudaEventDisableTiming) != cudaSuccess) {
      vgroup_destroy(G);
      return nullptr;
    }
  }
  G->src.resize(k);
  G->sendbuf.assign(k, nullptr);
  G->send_off.assign(k, nullptr);
  return G;
}

void vgroup_destroy(VGroup* G) {
  if (!G) return;
  for (cudaEvent_t e : G->ready)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : G->used)
    if (e) cudaEventDestroy(e);
  delete G;
}

int vgroup_size(const VGroup* G) { return G ? G->k : 0; }

struct VSumArgs {
  int k, nbuf;
  const double* src[VMAX_RANKS][VMAX_BUF];
  double* dst[VMAX_BUF];
  long long count[VMAX_BUF];
};

// dst[b][j] = ((src[0][b][j] + src[1][b][j]) + ...) + src[k-1][b][j]: fixed rank order
__global__ void vsum_kernel(const __grid_constant__ VSumArgs a) {
  for (int b = 0; b < a.nbuf; ++b)
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < a.count[b];
         j += (long long)gridDim.x * blockDim.x) {
      double acc = a.src[0][b][j];
      for (int p = 1; p < a.k; ++p) acc += a.src[p][b][j];
      a.dst[b][j] = acc;
    }
}

int vgroup_allreduce(VGroup* G, int rank, const double* const* src, double* const* dst, const size_t* counts, int nbuf,
                     cudaStream_t st) {
  if (nbuf > VMAX_BUF) return -5;
  for (int b = 0; b < nbuf; ++b)
    if (src[b] == dst[b]) return -5;  // peers read src while this rank writes dst: out of place only
  G->src[rank].assign(src, src + nbuf);
  cudaEventRecord(G->ready[rank], st);
  G->barrier();  // every rank's partials are registered and recorded
  VSumArgs a{};
  a.k = G->k;
  a.nbuf = nbuf;
  long long mx = 1;
  bool bad = false;  // (no early return between the barriers: the peers would wait forever)
  for (int p = 0; p < G->k; ++p) {
    if (p != rank) cudaStreamWaitEvent(st, G->ready[p], 0);
    if ((int)G->src[p].size() != nbuf) bad = true;  // ranks disagree on the reduction point
    else
      for (int b = 0; b < nbuf; ++b) a.src[p][b] = G->src[p][b];
  }
  for (int b = 0; b < nbuf; ++b) {
    a.dst[b] = dst[b];
    a.count[b] = (long long)counts[b];
    mx = std::max(mx, a.count[b]);
  }
  if (!bad) vsum_kernel<<<(unsigned)std::min<long long>((mx + 255) / 256, 64), 256, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (bad) e = cudaErrorInvalidValue;
  cudaEventRecord(G->used[rank], st);
  G->barrier();  // every rank has enqueued its reads of the others' partials
  for (int p = 0; p < G->k; ++p)
    if (p != rank) cudaStreamWaitEvent(st, G->used[p], 0);  // before anyone rewrites them
  return e == cudaSuccess ? 0 : -5;
}

int vgroup_halo(VGroup* G, int rank, const double* sendbuf, const int64_t* send_off, double* recvbuf,
                const int64_t* recv_off, size_t dpr, cudaStream_t st) {
  G->sendbuf[rank] = sendbuf;
  G->send_off[rank] = send_off;
  cudaEventRecord(G->ready[rank], st);
  G->barrier();  // every rank's packed rows are registered and recorded
  cudaError_t e = cudaSuccess;
  for (int p = 0; p < G->k; ++p) {
    if (p == rank) continue;
    const int64_t nr = recv_off[p + 1] - recv_off[p];
    if (nr <= 0) continue;
    const int64_t ns = G->send_off[p][rank + 1] - G->send_off[p][rank];
    if (ns != nr) e = cudaErrorInvalidValue;  // inconsistent plans
    if (e != cudaSuccess) break;
    cudaStreamWaitEvent(st, G->ready[p], 0);
    e = cudaMemcpyAsync(recvbuf + recv_off[p] * dpr, G->sendbuf[p] + G->send_off[p][rank] * dpr,
                        (size_t)nr * dpr * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  cudaEventRecord(G->used[rank], st);
  G->barrier();
  for (int p = 0; p < G->k; ++p)
    if (p != rank) cudaStreamWaitEvent(st, G->used[p], 0);  // before a peer re-packs its send buffer
  return e == cudaSuccess ? 0 : -5;
}

}  // namespace srk
