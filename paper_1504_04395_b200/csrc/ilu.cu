// ilu.cu — right ILU(0) preconditioning (PAPER.md P:670-676,
// "a (right) no-fill ILU preconditioner obtained via the Matlab function
// ilu"). Host side: the no-fill factorisation of the operator's CSR in the IKJ order
// (Saad, Alg. 10.4) and the level schedules of the four triangular solves
// (M^-1 = U^-1 L^-1 forward/backward; M^-H = L^-H U^-H for the A^H products).
// Host code (compiled by nvcc for the shared headers). The factorisation is one-time
// operator preparation (a0); the solves run on the
// device (trsv.cu), one kernel per level, every row of a level in parallel.
#include <algorithm>
#include <climits>
#include <cmath>
#include <complex>
#include <queue>
#include <vector>

#include "engine.h"

namespace srk {

namespace {

enum { ILU_OK = 0, ILU_ZEROPIVOT = 1, ILU_NOMEM = 2, ILU_CUDA = 3 };

inline double cj(double x) { return x; }
inline std::complex<double> cj(std::complex<double> x) { return std::conj(x); }

template <typename V>
int factor(long long n, const std::vector<int>& rp, const std::vector<int>& ci, std::vector<V>& v) {
  std::vector<int> diag(n, -1), pos(n, -1);
  for (long long i = 0; i < n; ++i)
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) diag[i] = p;
  for (long long i = 0; i < n; ++i) {
    for (int p = rp[i]; p < rp[i + 1]; ++p) pos[ci[p]] = p;
    for (int p = rp[i]; p < rp[i + 1] && ci[p] < i; ++p) {
      const int k = ci[p];
      if (diag[k] < 0 || v[diag[k]] == V(0)) return ILU_ZEROPIVOT;
      v[p] /= v[diag[k]];
      const V lik = v[p];
      for (int q = diag[k] + 1; q < rp[k + 1]; ++q) {
        const int j = ci[q];
        if (pos[j] >= 0) v[pos[j]] -= lik * v[q];
      }
    }
    for (int p = rp[i]; p < rp[i + 1]; ++p) pos[ci[p]] = -1;
    if (diag[i] < 0 || v[diag[i]] == V(0)) return ILU_ZEROPIVOT;
  }
  return ILU_OK;
}

// one triangular factor as a CSR of its off-diagonal part (+ inverse diagonal)
template <typename V>
struct HostTri {
  std::vector<int> rp, ci;
  std::vector<V> val, dinv, diag;  // dinv / diag empty: unit diagonal
  std::vector<int> order, lvl;  // rows by level, level boundaries
};

template <typename V>
void schedule(HostTri<V>& t, long long n, bool forward) {
  std::vector<int> level(n, 0);
  int nlev = 0;
  if (forward) {
    for (long long i = 0; i < n; ++i) {
      int l = 0;
      for (int p = t.rp[i]; p < t.rp[i + 1]; ++p) l = std::max(l, level[t.ci[p]] + 1);
      level[i] = l;
      nlev = std::max(nlev, l + 1);
    }
  } else {
    for (long long i = n - 1; i >= 0; --i) {
      int l = 0;
      for (int p = t.rp[i]; p < t.rp[i + 1]; ++p) l = std::max(l, level[t.ci[p]] + 1);
      level[i] = l;
      nlev = std::max(nlev, l + 1);
    }
  }
  t.lvl.assign(nlev + 1, 0);
  for (long long i = 0; i < n; ++i) t.lvl[level[i] + 1]++;
  for (int l = 0; l < nlev; ++l) t.lvl[l + 1] += t.lvl[l];
  t.order.assign(n, 0);
  std::vector<int> fill(t.lvl.begin(), t.lvl.end() - 1);
  for (long long i = 0; i < n; ++i) t.order[fill[level[i]]++] = (int)i;  // ascending rows within a level
}

// off-diagonal part of rows with (lower ? j < i : j > i), optionally conjugate-transposed
template <typename V>
HostTri<V> extract(long long n, const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<V>& v,
                   bool lower, bool transpose_conj) {
  HostTri<V> t;
  t.rp.assign(n + 1, 0);
  if (!transpose_conj) {
    for (long long i = 0; i < n; ++i) {
      for (int p = rp[i]; p < rp[i + 1]; ++p)
        if (lower ? ci[p] < i : ci[p] > i) {
          t.ci.push_back(ci[p]);
          t.val.push_back(v[p]);
        }
      t.rp[i + 1] = (int)t.ci.size();
    }
    return t;
  }
  // (part)^H: entry (i, j) of the part becomes (j, i) with the conjugate value
  std::vector<int> cnt(n + 1, 0);
  for (long long i = 0; i < n; ++i)
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (lower ? ci[p] < i : ci[p] > i) cnt[ci[p] + 1]++;
  for (long long i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  t.rp = cnt;
  t.ci.assign(cnt[n], 0);
  t.val.assign(cnt[n], V(0));
  std::vector<int> fill(cnt.begin(), cnt.end() - 1);
  for (long long i = 0; i < n; ++i)  // ascending i keeps the new rows' columns sorted
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (lower ? ci[p] < i : ci[p] > i) {
        const int q = fill[ci[p]]++;
        t.ci[q] = (int)i;
        t.val[q] = cj(v[p]);
      }
  return t;
}

template <typename V>
int upload(const HostTri<V>& t, long long n, bool cplx, DevTri& d) {
  const size_t esz = cplx ? 16 : 8;
  const size_t nz = t.ci.size();
  if (cudaMalloc(&d.rp, sizeof(int) * (n + 1)) != cudaSuccess || cudaMalloc(&d.ci, sizeof(int) * (nz + 1)) != cudaSuccess ||
      cudaMalloc(&d.val, esz * (nz + 1)) != cudaSuccess || cudaMalloc(&d.order, sizeof(int) * (n + 1)) != cudaSuccess)
    return ILU_NOMEM;
  cudaMemcpy(d.rp, t.rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
  if (nz) {
    cudaMemcpy(d.ci, t.ci.data(), sizeof(int) * nz, cudaMemcpyHostToDevice);
    cudaMemcpy(d.val, t.val.data(), esz * nz, cudaMemcpyHostToDevice);
  }
  cudaMemcpy(d.order, t.order.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
  if (!t.dinv.empty()) {
    if (cudaMalloc(&d.dinv, esz * n) != cudaSuccess || cudaMalloc(&d.diag, esz * n) != cudaSuccess) return ILU_NOMEM;
    cudaMemcpy(d.dinv, t.dinv.data(), esz * n, cudaMemcpyHostToDevice);
    cudaMemcpy(d.diag, t.diag.data(), esz * n, cudaMemcpyHostToDevice);
  }
  d.lvl = t.lvl;
  return 0;
}

void free_tri(DevTri& d);

template <typename V>
int build(Mat& m, cudaStream_t st) {
  const long long n = m.n, nnz = m.nnz;
  std::vector<int> rp(n + 1), ci(nnz);
  std::vector<V> v(nnz);
  cudaMemcpyAsync(rp.data(), m.rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(ci.data(), m.ci, sizeof(int) * nnz, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(v.data(), m.val, sizeof(V) * nnz, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return ILU_CUDA;
  if (factor(n, rp, ci, v)) return ILU_ZEROPIVOT;
  Prec* P = new Prec();
  P->n = n;
  P->cplx = m.cplx;
  // M^-1 = U^-1 L^-1: L strictly lower (unit), U strictly upper + 1/u_ii
  HostTri<V> L = extract(n, rp, ci, v, true, false), U = extract(n, rp, ci, v, false, false);
  // M^-H = L^-H U^-H: U^H strictly lower + 1/conj(u_ii), L^H strictly upper (unit)
  HostTri<V> UH = extract(n, rp, ci, v, false, true), LH = extract(n, rp, ci, v, true, true);
  U.dinv.assign(n, V(0));
  UH.dinv.assign(n, V(0));
  U.diag.assign(n, V(0));
  UH.diag.assign(n, V(0));
  for (long long i = 0; i < n; ++i)
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) {
        U.diag[i] = v[p];
        UH.diag[i] = cj(v[p]);
        U.dinv[i] = V(1) / v[p];
        UH.dinv[i] = V(1) / cj(v[p]);
      }
  schedule(L, n, true);
  schedule(U, n, false);
  schedule(UH, n, true);
  schedule(LH, n, false);
  int r = upload(L, n, m.cplx, P->L);
  if (!r) r = upload(U, n, m.cplx, P->U);
  if (!r) r = upload(UH, n, m.cplx, P->UH);
  if (!r) r = upload(LH, n, m.cplx, P->LH);
  if (!r) {
    P->factor.resize((size_t)nnz * (m.cplx ? 2 : 1));
    std::copy(reinterpret_cast<const double*>(v.data()), reinterpret_cast<const double*>(v.data()) + P->factor.size(),
              P->factor.begin());
  }
  if (r) {
    free_prec(P);
    return r;
  }
  m.prec = P;
  return 0;
}

// ---------------------------------------------------------------------------
// ILUTP: the incomplete LU "with threshold and pivoting with a drop tolerance of 5e-2"
// of Ex. 4. Reading R14: left-looking (column) ILU with partial
// pivoting — column j: x = A(:, j); the pivoted rows are eliminated in step order k
// (x -= L(:, k) x_r, r = perm[k]), a multiplier with |x_r| < droptol ||A(:, j)||_2 dropped
// (not used, not stored); pivot = the largest |x_r| over the rows not yet pivoted (ties:
// smallest row; the original row j when |x_j| >= thresh max); the remaining entries below
// the tolerance are dropped, the others divided by the pivot form L(:, j). Pi A ~ L U with
// L unit lower / U upper in the pivot order. A min-heap of steps visits only the pivoted
// rows x reaches (the sparse left-looking elimination), a dense work vector holds x.
template <typename V>
int factor_ilutp(long long n, const std::vector<int>& rp, const std::vector<int>& ci, const std::vector<V>& v,
                 double droptol, double thresh, std::vector<int>& perm, std::vector<long long>& lp,
                 std::vector<int>& lr, std::vector<V>& lv, std::vector<long long>& up, std::vector<int>& uk,
                 std::vector<V>& uv) {
  // CSC of A (columns ascending rows)
  std::vector<long long> cp(n + 1, 0);
  for (long long i = 0; i < n; ++i)
    for (int p = rp[i]; p < rp[i + 1]; ++p) cp[ci[p] + 1]++;
  for (long long j = 0; j < n; ++j) cp[j + 1] += cp[j];
  std::vector<int> cr(cp[n]);
  std::vector<V> cv(cp[n]);
  {
    std::vector<long long> fill(cp.begin(), cp.end() - 1);
    for (long long i = 0; i < n; ++i)
      for (int p = rp[i]; p < rp[i + 1]; ++p) {
        const long long q = fill[ci[p]]++;
        cr[q] = (int)i;
        cv[q] = v[p];
      }
  }
  perm.assign(n, -1);
  std::vector<int> step(n, -1);        // original row -> pivot step
  std::vector<V> x(n, V(0));
  std::vector<int> mark(n, -1), nzr;   // rows present in x (stamp = column)
  std::vector<int> inheap(n, -1);      // steps pushed for this column
  lp.assign(1, 0);
  up.assign(1, 0);
  lr.clear(); lv.clear(); uk.clear(); uv.clear();
  std::priority_queue<int, std::vector<int>, std::greater<int>> heap;
  std::vector<std::pair<int, V>> ucol;
  for (long long j = 0; j < n; ++j) {
    nzr.clear();
    double nrm2 = 0.0;
    for (long long q = cp[j]; q < cp[j + 1]; ++q) {
      const int r = cr[q];
      x[r] = cv[q];
      mark[r] = (int)j;
      nzr.push_back(r);
      nrm2 += std::norm(std::complex<double>(cv[q]));
      if (step[r] >= 0 && inheap[step[r]] != (int)j) {
        inheap[step[r]] = (int)j;
        heap.push(step[r]);
      }
    }
    const double tol = droptol * std::sqrt(nrm2);
    ucol.clear();
    while (!heap.empty()) {
      const int k = heap.top();
      heap.pop();
      const int r = perm[k];
      const V ukj = x[r];
      x[r] = V(0);  // row r leaves x (its value is u_kj or dropped)
      if (ukj == V(0) || std::abs(ukj) < tol) continue;
      ucol.emplace_back(k, ukj);
      for (long long q = lp[k]; q < lp[k + 1]; ++q) {
        const int rr = lr[q];
        if (mark[rr] != (int)j) {
          mark[rr] = (int)j;
          x[rr] = V(0);
          nzr.push_back(rr);
        }
        x[rr] -= lv[q] * ukj;
        const int sr = step[rr];
        if (sr >= 0 && inheap[sr] != (int)j) {
          inheap[sr] = (int)j;
          heap.push(sr);
        }
      }
    }
    // pivot among the rows not yet pivoted
    double big = -1.0;
    int imax = -1;
    for (int r : nzr)
      if (step[r] < 0 && x[r] != V(0)) {
        const double a = std::abs(x[r]);
        if (a > big || (a == big && r < imax)) {
          big = a;
          imax = r;
        }
      }
    if (imax < 0) return ILU_ZEROPIVOT;
    int piv = imax;
    if (step[j] < 0 && mark[j] == (int)j && x[j] != V(0) && std::abs(x[j]) >= thresh * big) piv = (int)j;
    const V d = x[piv];
    perm[j] = piv;
    step[piv] = (int)j;
    std::sort(ucol.begin(), ucol.end(), [](const std::pair<int, V>& a, const std::pair<int, V>& b) { return a.first < b.first; });
    for (auto& e : ucol) {
      uk.push_back(e.first);
      uv.push_back(e.second);
    }
    uk.push_back((int)j);
    uv.push_back(d);
    up.push_back((long long)uk.size());
    std::vector<int> rows;
    for (int r : nzr)
      if (r != piv && step[r] < 0 && x[r] != V(0) && std::abs(x[r]) >= tol) rows.push_back(r);
    std::sort(rows.begin(), rows.end());
    for (int r : rows) {
      lr.push_back(r);
      lv.push_back(x[r] / d);
    }
    lp.push_back((long long)lr.size());
    for (int r : nzr) x[r] = V(0);
  }
  return ILU_OK;
}

template <typename V>
int build_tp(Mat& m, double droptol, double thresh, cudaStream_t st) {
  const long long n = m.n, nnz = m.nnz;
  std::vector<int> rp(n + 1), ci(nnz);
  std::vector<V> v(nnz);
  cudaMemcpyAsync(rp.data(), m.rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(ci.data(), m.ci, sizeof(int) * nnz, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(v.data(), m.val, sizeof(V) * nnz, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return ILU_CUDA;
  std::vector<int> perm, lr, uk;
  std::vector<long long> lp, up;
  std::vector<V> lv, uv;
  if (factor_ilutp(n, rp, ci, v, droptol, thresh, perm, lp, lr, lv, up, uk, uv)) return ILU_ZEROPIVOT;
  std::vector<int> step(n);
  for (long long k = 0; k < n; ++k) step[perm[k]] = (int)k;
  // the factor F = (L - I) + U as one CSR in the pivot order (L(i, k) at row step[r]),
  // columns ascending — then the same extraction / scheduling as ILU(0)
  std::vector<int> cnt(n + 1, 0);
  for (long long k = 0; k < n; ++k)
    for (long long q = lp[k]; q < lp[k + 1]; ++q) cnt[step[lr[q]] + 1]++;
  for (long long j = 0; j < n; ++j)
    for (long long q = up[j]; q < up[j + 1]; ++q) cnt[uk[q] + 1]++;
  for (long long i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  if ((long long)cnt[n] >= (long long)INT_MAX) return ILU_NOMEM;
  std::vector<int> frp(cnt), fci(cnt[n]);
  std::vector<V> fv(cnt[n]);
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    // columns visited in ascending order keep every row's columns sorted
    for (long long c = 0; c < n; ++c) {
      for (long long q = lp[c]; q < lp[c + 1]; ++q) {  // L(:, c): rows below c in the pivot order
        const int i = step[lr[q]];
        fci[fill[i]] = (int)c;
        fv[fill[i]++] = lv[q];
      }
      for (long long q = up[c]; q < up[c + 1]; ++q) {  // U(:, c): rows k <= c
        const int k = uk[q];
        fci[fill[k]] = (int)c;
        fv[fill[k]++] = uv[q];
      }
    }
  }
  Prec* P = new Prec();
  P->n = n;
  P->cplx = m.cplx;
  HostTri<V> L = extract(n, frp, fci, fv, true, false), U = extract(n, frp, fci, fv, false, false);
  HostTri<V> UH = extract(n, frp, fci, fv, false, true), LH = extract(n, frp, fci, fv, true, true);
  U.dinv.assign(n, V(0));
  UH.dinv.assign(n, V(0));
  U.diag.assign(n, V(0));
  UH.diag.assign(n, V(0));
  for (long long i = 0; i < n; ++i)
    for (int p = frp[i]; p < frp[i + 1]; ++p)
      if (fci[p] == i) {
        U.diag[i] = fv[p];
        UH.diag[i] = cj(fv[p]);
        U.dinv[i] = V(1) / fv[p];
        UH.dinv[i] = V(1) / cj(fv[p]);
      }
  schedule(L, n, true);
  schedule(U, n, false);
  schedule(UH, n, true);
  schedule(LH, n, false);
  int r = upload(L, n, m.cplx, P->L);
  if (!r) r = upload(U, n, m.cplx, P->U);
  if (!r) r = upload(UH, n, m.cplx, P->UH);
  if (!r) r = upload(LH, n, m.cplx, P->LH);
  bool ident = true;
  for (long long k = 0; k < n; ++k) ident &= (perm[k] == k);
  if (!r && !ident) {
    if (cudaMalloc(&P->perm, sizeof(int) * n) != cudaSuccess) r = ILU_NOMEM;
    else cudaMemcpy(P->perm, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
  }
  if (!r) {  // host copy of the factor (pivot-order CSR) and the permutation, for tests
    P->frp = frp;
    P->fci = fci;
    P->factor.resize(fv.size() * (m.cplx ? 2 : 1));
    std::copy(reinterpret_cast<const double*>(fv.data()), reinterpret_cast<const double*>(fv.data()) + P->factor.size(),
              P->factor.begin());
    P->hperm = perm;
    P->kind = 1;
  }
  if (r) {
    free_prec(P);
    return r;
  }
  m.prec = P;
  return 0;
}

void free_tri(DevTri& d) {
  if (d.rp) cudaFree(d.rp);
  if (d.ci) cudaFree(d.ci);
  if (d.val) cudaFree(d.val);
  if (d.dinv) cudaFree(d.dinv);
  if (d.diag) cudaFree(d.diag);
  if (d.order) cudaFree(d.order);
  if (d.flags) cudaFree(d.flags);
  d = DevTri{};
}

}  // namespace

void free_prec(Prec* P) {
  if (!P) return;
  free_tri(P->L);
  free_tri(P->U);
  free_tri(P->UH);
  free_tri(P->LH);
  if (P->perm) cudaFree(P->perm);
  for (void* b : P->scratch)
    if (b) cudaFree(b);
  delete P;
}

int build_ilutp(Mat& m, double droptol, double thresh, cudaStream_t st) {
  if (m.prec) {
    free_prec(m.prec);
    m.prec = nullptr;
  }
  return m.cplx ? build_tp<std::complex<double>>(m, droptol, thresh, st) : build_tp<double>(m, droptol, thresh, st);
}

int build_ilu0(Mat& m, cudaStream_t st) {
  if (m.prec) {
    free_prec(m.prec);
    m.prec = nullptr;
  }
  return m.cplx ? build<std::complex<double>>(m, st) : build<double>(m, st);
}

}  // namespace srk
