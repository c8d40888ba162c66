// partition.cpp — host-side row partitioning and halo planning for the
// multi-GPU path: A and every n x s block are split
// into contiguous row ranges balanced by nnz; each rank keeps its rows of A with
// columns renumbered to [0, n_local) for owned rows and [n_local, n_local +
// n_ghost) for ghost rows (sorted by global index, hence grouped by owner rank),
// and a send list per peer (its owned rows that the peer references).
// Pure host code: no CUDA, callable (and tested with gloo) without a GPU.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/srk.h"

struct srk_plan {
  int nranks = 1, rank = 0;
  int64_t n = 0, off0 = 0, off1 = 0, nnz_local = 0;
  std::vector<int64_t> row_ptr;     // local, n_local + 1 (starts at 0)
  std::vector<int32_t> col;         // local numbering
  std::vector<int64_t> ghosts;      // global indices of ghost rows (sorted)
  std::vector<int32_t> recv_counts; // per peer
  std::vector<int32_t> send_counts; // per peer
  std::vector<int32_t> send_local;  // concatenated by peer: local row indices to send
};

static int owner_of(const std::vector<int64_t>& off, int64_t j) {
  // off has nranks+1 entries, contiguous ranges
  return (int)(std::upper_bound(off.begin(), off.end(), j) - off.begin()) - 1;
}

extern "C" {

int srk_partition_rows(int64_t n, const int64_t* row_ptr, int nranks, int64_t* offsets) {
  if (n <= 0 || !row_ptr || nranks < 1 || !offsets) return SRK_EINVAL;
  const int64_t nnz = row_ptr[n];
  offsets[0] = 0;
  int64_t r = 0;
  for (int p = 1; p < nranks; ++p) {
    // first row whose prefix nnz reaches p/nranks of the total (rows also balanced when nnz is uniform)
    const double target = (double)nnz * p / nranks;
    r = std::max(r, offsets[p - 1]);
    int64_t lo = r, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if ((double)row_ptr[mid] < target) lo = mid + 1; else hi = mid;
    }
    offsets[p] = lo;
  }
  offsets[nranks] = n;
  return SRK_OK;
}

int srk_plan_create(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int nranks, const int64_t* offsets,
                    int rank, srk_plan** out) {
  if (n <= 0 || !row_ptr || !col_idx || nranks < 1 || !offsets || rank < 0 || rank >= nranks || !out) return SRK_EINVAL;
  std::vector<int64_t> off(offsets, offsets + nranks + 1);
  for (int p = 0; p < nranks; ++p)
    if (off[p] > off[p + 1]) return SRK_EINVAL;
  if (off[0] != 0 || off[nranks] != n) return SRK_EINVAL;
  auto* P = new srk_plan();
  P->nranks = nranks;
  P->rank = rank;
  P->n = n;
  P->off0 = off[rank];
  P->off1 = off[rank + 1];
  const int64_t nl = P->off1 - P->off0;
  // ghosts of every rank q (needed for this rank's send lists): a boolean mark per
  // global row would cost n bytes per rank; instead collect per-rank sorted uniques.
  auto ghosts_of = [&](int q) {
    std::vector<int64_t> g;
    for (int64_t i = off[q]; i < off[q + 1]; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        const int64_t j = col_idx[k];
        if (j < off[q] || j >= off[q + 1]) g.push_back(j);
      }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    return g;
  };
  P->ghosts = ghosts_of(rank);
  // local CSR with renumbered columns
  P->row_ptr.resize(nl + 1);
  P->row_ptr[0] = 0;
  P->nnz_local = row_ptr[P->off1] - row_ptr[P->off0];
  P->col.resize(P->nnz_local);
  for (int64_t i = 0; i < nl; ++i) {
    const int64_t gi = P->off0 + i;
    for (int64_t k = row_ptr[gi]; k < row_ptr[gi + 1]; ++k) {
      const int64_t j = col_idx[k];
      int64_t lj;
      if (j >= P->off0 && j < P->off1) lj = j - P->off0;
      else lj = nl + (std::lower_bound(P->ghosts.begin(), P->ghosts.end(), j) - P->ghosts.begin());
      P->col[k - row_ptr[P->off0]] = (int32_t)lj;
    }
    P->row_ptr[i + 1] = row_ptr[gi + 1] - row_ptr[P->off0];
  }
  // entries keep the global order of the row (ascending global column), so the caller's
  // values slice values[row_ptr[off0] : row_ptr[off1]] applies unchanged; local column
  // indices are therefore not monotone within a row (owned and ghost ranges interleave)
  P->recv_counts.assign(nranks, 0);
  for (int64_t j : P->ghosts) P->recv_counts[owner_of(off, j)]++;
  P->send_counts.assign(nranks, 0);
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    // q's ghosts that this rank owns, in q's (sorted) order
    std::vector<int64_t> gq = ghosts_of(q);
    for (int64_t j : gq)
      if (j >= P->off0 && j < P->off1) {
        P->send_local.push_back((int32_t)(j - P->off0));
        P->send_counts[q]++;
      }
  }
  *out = P;
  return SRK_OK;
}

int srk_plan_sizes(const srk_plan* P, int64_t* n_local, int64_t* nnz_local, int64_t* n_ghost, int64_t* n_send) {
  if (!P) return SRK_EINVAL;
  if (n_local) *n_local = P->off1 - P->off0;
  if (nnz_local) *nnz_local = P->nnz_local;
  if (n_ghost) *n_ghost = (int64_t)P->ghosts.size();
  if (n_send) *n_send = (int64_t)P->send_local.size();
  return SRK_OK;
}

int srk_plan_arrays(const srk_plan* P, int64_t* row_ptr_local, int32_t* col_local, int64_t* ghost_global,
                    int32_t* recv_counts, int32_t* send_counts, int32_t* send_local) {
  if (!P) return SRK_EINVAL;
  if (row_ptr_local) std::copy(P->row_ptr.begin(), P->row_ptr.end(), row_ptr_local);
  if (col_local) std::copy(P->col.begin(), P->col.end(), col_local);
  if (ghost_global) std::copy(P->ghosts.begin(), P->ghosts.end(), ghost_global);
  if (recv_counts) std::copy(P->recv_counts.begin(), P->recv_counts.end(), recv_counts);
  if (send_counts) std::copy(P->send_counts.begin(), P->send_counts.end(), send_counts);
  if (send_local) std::copy(P->send_local.begin(), P->send_local.end(), send_local);
  return SRK_OK;
}

int srk_plan_destroy(srk_plan* P) {
  delete P;
  return SRK_OK;
}

// A^H = conj(A)^T by a counting sort over the columns (a0): stable, so the
// entries of each row of A^H come in ascending column order (the rows of A visited in
// order). Host code: every rank of a distributed operator builds it from the global CSR
// it already holds for srk_plan_create.
int srk_csr_adjoint_host(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, const void* values, int dtype,
                         int64_t* rpT, int32_t* ciT, void* valT) {
  if (n <= 0 || !row_ptr || !rpT || (dtype != SRK_F64 && dtype != SRK_C128)) return SRK_EINVAL;
  const int64_t nnz = row_ptr[n];
  if (nnz > 0 && (!col_idx || !values || !ciT || !valT)) return SRK_EINVAL;
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t k = 0; k < nnz; ++k) {
    if (col_idx[k] < 0 || col_idx[k] >= n) return SRK_EINVAL;
    cnt[col_idx[k] + 1]++;
  }
  for (int64_t j = 0; j < n; ++j) cnt[j + 1] += cnt[j];
  std::copy(cnt.begin(), cnt.end(), rpT);
  const int nd = dtype == SRK_C128 ? 2 : 1;
  const double* v = static_cast<const double*>(values);
  double* vT = static_cast<double*>(valT);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const int64_t d = cnt[col_idx[k]]++;
      ciT[d] = (int32_t)i;
      vT[d * nd] = v[k * nd];
      if (nd == 2) vT[d * nd + 1] = -v[k * nd + 1];  // conj
    }
  return SRK_OK;
}

}  // extern "C"
