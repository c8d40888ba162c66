// engine.cu — host helpers that marshal the generic block kernels, plus the
// operator-preparation kernels (CSR validation and the
// explicit A^H = conj(A)^T copy used by the BiCG/QMR families).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "engine.h"

namespace srk {

int Ctx::ensure_partials(size_t n) {
  if (n <= pcap) return 0;
  if (partials) cudaFree(partials);
  partials = nullptr;
  pcap = 0;
  cudaError_t e = cudaMalloc(&partials, n * sizeof(double));
  if (e != cudaSuccess) return (int)e;
  pcap = n;
  return 0;
}

void Prof::begin(int t, cudaStream_t st, int signature, double nbytes) {
  if (!on) return;
  if (used * 2 + 2 > ev.size()) {
    for (int i = 0; i < 2; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    tag.push_back(0);
    sig.push_back(0);
    bytes.push_back(0.0);
  }
  tag[used] = t;
  sig[used] = signature;
  bytes[used] = nbytes;
  cudaEventRecord(ev[2 * used], st);
}
int Prof::read_launches(int* tag_out, int* sig_out, double* ms_out, double* bytes_out, int max) {
  const int k = (int)std::min(used, (size_t)max);
  for (int i = 0; i < k; ++i) {
    cudaEventSynchronize(ev[2 * i + 1]);
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]);
    tag_out[i] = tag[i];
    sig_out[i] = sig[i];
    ms_out[i] = t;
    bytes_out[i] = bytes[i];
  }
  used = 0;
  return k;
}
void Prof::end(cudaStream_t st) {
  if (!on) return;
  cudaEventRecord(ev[2 * used + 1], st);
  used++;
}
int Prof::read(double* ms, long long* cnt, int ntag) {
  for (int i = 0; i < ntag; ++i) { ms[i] = 0.0; cnt[i] = 0; }
  for (size_t i = 0; i < used; ++i) {
    cudaEventSynchronize(ev[2 * i + 1]);
    float t = 0.f;
    cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]);
    if (tag[i] < ntag) { ms[tag[i]] += t; cnt[tag[i]]++; }
  }
  used = 0;
  return 0;
}
Prof::~Prof() {
  for (auto e : ev) cudaEventDestroy(e);
}

// Persistent-style grid: exactly one wave, i.e. the SM count times the number of
// CTAs the occupancy calculator says are resident for this kernel instance (so
// no partial second wave), or fewer CTAs when n is small.
int Eng::grid_for(int cap, bool full, bool is_spmm, size_t smem, int nin) const {
  const long long rpc = rows_per_cta(cap, cplx);
  long long need = (n + rpc - 1) / rpc;
  static int occ_cache[2][2][2][65][MAX_IN + 1] = {};
  int& occ = occ_cache[is_spmm][cplx][full][cap][nin];
  if (occ == 0) {
    SpmmArgs sa{};
    UpdArgs ua{};
    ua.nin = nin;
    sa.team = is_spmm ? nin : 0;  // SpMM: nin carries the team flag
    occ = is_spmm ? launch_spmm(cplx, cap, full, sa, -1, 256, smem, nullptr)
                  : launch_upd(cplx, cap, full, ua, -1, 256, smem, nullptr);
    if (occ < 1) occ = 1;
  }
  const long long maxg = (long long)c->nsm * occ;
  if (need < 1) need = 1;
  return (int)std::min(need, maxg);
}

static void fill_red(Red& r, const RQ& q, int poff) {
  r.mode = q.mode;
  r.xsrc = q.x;
  r.ysrc = q.y;
  r.yext = q.yext;
  r.poff = poff;
}

static int finish_reds(Eng& e, const std::vector<RQ>& reds, const std::vector<int>& poffs, int s, int grid,
                       int pstride) {
  if (reds.empty()) return 0;
  FinArgs f{};
  f.partials = e.c->partials;
  f.nblk = grid;
  f.pstride = pstride;
  f.nseg = (int)reds.size();
  for (size_t i = 0; i < reds.size(); ++i) {
    f.seg[i].poff = poffs[i];
    f.seg[i].len = red_len(reds[i].mode, s, e.cplx);
    f.seg[i].woff = reds[i].woff;
  }
  // multi-GPU: fin writes this rank's sums to a staging mirror of the workspace and the
  // allreduce writes the global sums into ws (out of place). A fin skipped after the done
  // flag was raised leaves the staging slot with its last real local sums, so the
  // allreduce re-forms the same global value instead of scaling ws by the rank count.
  // (kernel-level calls run every fin and have no staging: NCCL reduces them in place)
  const bool multi = e.c->comm && e.c->comm->nranks > 1;
  if (multi && !e.wstage && e.c->comm->vg) return (int)cudaErrorInvalidValue;
  double* stage = (multi && e.wstage) ? e.wstage : e.ws;
  f.ws = stage;
  f.done = e.done;
  e.nlaunch++;
  if (e.prof) e.prof->begin(PT_FIN, e.c->st);
  int r = launch_fin(f, e.c->st);
  if (e.prof) e.prof->end(e.c->st);
  if (r) return r;
  if (multi) {
    if (e.prof) e.prof->begin(PT_OTHER, e.c->st);
    std::vector<const double*> src;
    std::vector<double*> dst;
    std::vector<size_t> counts;
    for (size_t i = 0; i < reds.size(); ++i) {
      src.push_back(stage + reds[i].woff);
      dst.push_back(e.ws + reds[i].woff);
      counts.push_back((size_t)red_len(reds[i].mode, s, e.cplx));
    }
    if (comm_allreduce_sum_many(e.c->comm, src.data(), dst.data(), counts.data(), (int)src.size(), e.c->st)) r = -5;
    if (e.prof) e.prof->end(e.c->st);
  }
  return r;
}

// Halo exchange of the ghost rows of P (multi-GPU operators): pack the rows the
// peers need, then grouped ncclSend/ncclRecv straight into P's ghost tail.
int Eng::halo(bool adj, const void* P, int s, cudaStream_t hs) {
  if (!hs) hs = c->st;
  Mat* M = const_cast<Mat*>(A);
  const Halo& H = adj ? M->haloH : M->halo;
  if (!M->dist || !c->comm || c->comm->nranks == 1) return 0;
  const int dpr = s * (cplx ? 2 : 1);
  const size_t need = (size_t)std::max<long long>(H.n_send, 1) * dpr;
  if (need > M->sendcap) {
    if (M->sendbuf) cudaFree(M->sendbuf);
    if (cudaMalloc(&M->sendbuf, need * sizeof(double)) != cudaSuccess) return (int)cudaErrorMemoryAllocation;
    M->sendcap = need;
  }
  if (prof && hs == c->st) prof->begin(PT_OTHER, c->st);
  int r = launch_gather_rows(reinterpret_cast<const double*>(P), M->sendbuf, H.send_idx, H.n_send, dpr, nullptr, hs);
  if (!r) r = comm_halo(c->comm, M->sendbuf, H.send_off, const_cast<double*>(reinterpret_cast<const double*>(P)) + (size_t)n * dpr,
                        H.recv_off, dpr, hs);
  if (prof && hs == c->st) prof->end(c->st);
  return r;
}

int Eng::spmm(bool adj, const void* P, void* Q, int s, std::vector<RQ> reds) {
  if (err) return err;
  if (A->prec && !raw) return spmm_prec(adj, P, Q, s, reds);
  if (A->bsr) return spmm_bsr(adj, P, Q, s, reds);
  // distributed operator with a halo: interior rows while the halo is in flight
  {
    const Mat::Sorted& in = adj ? A->innerH : A->inner;
    const Mat::Sorted& bd = adj ? A->bndH : A->bnd;
    const long long ni = adj ? A->n_innerH : A->n_inner, nbd = adj ? A->n_bndH : A->n_bnd;
    static const bool no_overlap = getenv("SRK_NO_HALO_OVERLAP") != nullptr;  // A/B switch
    bool full_any = false;
    for (auto& r : reds) full_any |= (r.mode == RED_FULL);
    if (!no_overlap && A->dist && c->comm && c->comm->nranks > 1 && in.perm && bd.perm && !full_any)
      return err = spmm_split(adj, P, Q, s, reds, in, ni, bd, nbd);
  }
  if ((err = halo(adj, P, s))) return err;
  const int cap = cap_for(s);
  // s x s Grams of 8 columns and more: Y^H Q on the tensor cores afterwards (the FMA
  // epilogue's s x s accumulators cost the SpMM more than the extra pass: config 2)
  std::vector<RQ> wide;
  if (!full_red_supported(cplx, cap) || s >= 8) {
    for (auto it = reds.begin(); it != reds.end();)
      if (it->mode == RED_FULL) {
        wide.push_back(*it);
        it = reds.erase(it);
      } else {
        ++it;
      }
  }
  if (!wide.empty()) {
    if ((err = spmm(adj, P, Q, s, reds))) return err;
    for (const RQ& q : wide)
      if ((err = gram_full(Q, q.yext, s, q.woff))) return err;
    return 0;
  }
  bool full = false;
  for (auto& r : reds) full |= (r.mode == RED_FULL);
  if (full && !full_supported(cplx, cap)) return err = (int)cudaErrorNotSupported;
  // banded operators: the bulk-copy kernel (band.cu) — non-FULL epilogues, local rows only
  // (measured on config 2 / 3 operators: 16-27% faster than the CSR kernel without a fused
  // Y-operand reduction, equal with one — so products with a SUMVEC / TRACE / DIAG operand
  // keep the CSR kernel unless SRK_BAND_ALL is set)
  const Mat::Band& bd = adj ? A->bandH : A->band;
  static const bool band_all = getenv("SRK_BAND_ALL") != nullptr;
  bool yred = false, yrow = false;
  for (auto& q : reds) {
    yred |= (q.mode != RED_NORM2 && q.mode != RED_COLNORM2);
    yrow |= (q.mode != RED_NORM2 && q.mode != RED_COLNORM2 && q.mode != RED_SUMVEC);
  }
  // the plane-marching kernel takes vector operands (staged per plane) and row operands (the input's
  // own rows from registers, one external block's rows by early loads)
  static const bool plane_rows = getenv("SRK_NO_PLANE_ROWS") == nullptr;  // A/B switch
  if (yred && (!yrow || plane_rows) && bd.K > 0 && band_plane_pattern(bd)) yred = false;
  if (bd.K > 0 && !full && (band_all || !yred) && A->ghost_rows() == 0 && band_supported(cplx, s) && reds.size() <= 2) {
    std::vector<Red> rr(reds.size());
    std::vector<int> poffs;
    int pstride = 0;
    for (size_t i = 0; i < reds.size(); ++i) {
      fill_red(rr[i], reds[i], pstride);
      poffs.push_back(pstride);
      pstride += red_len(reds[i].mode, s, cplx);
    }
    pstride = std::max(pstride, 1);
    int grid = 0;
    int r = launch_band(cplx, s, bd, P, Q, n, rr.data(), (int)rr.size(), nullptr, pstride, done, c->nsm, c->st, &grid);
    if (r == 0) {
      if ((err = c->ensure_partials((size_t)grid * pstride))) return err;
      nlaunch++;
      if (prof) {
        const double esz = cplx ? 16.0 : 8.0;
        // algorithmic bytes of the banded form: the K diagonals once, P read once, Q written once
        double nb = (double)bd.K * n * esz + 2.0 * (double)n * s * esz;
        for (auto& q : reds)
          if (q.yext && q.yext != P && q.mode != RED_NORM2 && q.mode != RED_COLNORM2)
            nb += (double)n * (q.mode == RED_SUMVEC ? 1 : s) * esz;
        prof->begin(adj ? PT_SPMM_ADJ : PT_SPMM, c->st, s, nb);
      }
      err = launch_band(cplx, s, bd, P, Q, n, rr.data(), (int)rr.size(), c->partials, pstride, done, c->nsm, c->st,
                        nullptr);
      if (prof) prof->end(c->st);
      if (err) return err;
      return err = finish_reds(*this, reds, poffs, s, grid, pstride);
    }
    if (r != (int)cudaErrorNotSupported) return err = r;
  }
  SpmmArgs a{};
  const Mat::Sorted& so = adj ? A->srtH : A->srt;
  if (so.perm) {  // irregular rows: the length-sorted copy
    a.row_ptr = so.rp;
    a.col_idx = so.ci;
    a.val = so.val;
    a.perm = so.perm;
  } else {
    a.row_ptr = adj ? A->rpH : A->rp;
    a.col_idx = adj ? A->ciH : A->ci;
    a.val = adj ? A->valH : A->val;
  }
  a.P = P;
  a.Q = Q;
  a.n = n;
  a.s = s;
  a.vec = cplx ? 1 : (s % 2 == 0);
  a.nred = (int)reds.size();
  std::vector<int> poffs;
  int pstride = 0, maxlen = 0;
  for (size_t i = 0; i < reds.size(); ++i) {
    fill_red(a.red[i], reds[i], pstride);
    poffs.push_back(pstride);
    const int len = red_len(reds[i].mode, s, cplx);
    pstride += len;
    maxlen = std::max(maxlen, len);
  }
  a.pstride = std::max(pstride, 1);
  const size_t smem = (size_t)8 * maxlen * sizeof(double);
  // narrow rows: a team of lanes per row when rows are long or irregular (config 5),
  // a lane per row for short regular rows (the stencil's A^H vector product)
  const long long nz = adj ? A->nnzH : A->nnz;
  a.team = (so.perm != nullptr || nz >= 12LL * std::max(1LL, n)) ? 1 : 0;
  int grid = grid_for(cap, full, true, 8 * 2 * 8 * 16 * 16, a.team);  // occupancy at the largest epilogue smem
  const Mat::Sell& se = adj ? A->sellH : A->sell;
  if (se.cs && (size_t)cap * (cplx ? 16 : 8) <= 32) {  // narrow block on an irregular operator: SELL-32-sigma
    a.sell_cs = se.cs;
    a.sell_ci = se.ci;
    a.sell_val = se.val;
    a.sell_row = se.row;
    a.sell_order = se.order;
    a.sell_nchunk = se.nchunk;
    grid = (int)std::max<long long>(1, std::min<long long>((se.nchunk + 7) / 8, (long long)c->nsm * 4));
  }
  if ((err = c->ensure_partials((size_t)grid * a.pstride))) return err;
  a.partials = c->partials;
  a.done = done;
  nlaunch++;
  if (prof) {
    const double esz = cplx ? 16.0 : 8.0;
    const double nz = (double)(adj ? A->nnzH : A->nnz);
    double nb = (double)(n + 1) * 4 + nz * (4 + esz) + 2.0 * (double)n * s * esz;
    for (auto& r : reds)
      if (r.yext && r.mode != RED_NORM2 && r.mode != RED_COLNORM2)
        nb += (double)n * (r.mode == RED_SUMVEC ? 1 : s) * esz;
    prof->begin(adj ? PT_SPMM_ADJ : PT_SPMM, c->st, s, nb);
  }
  err = launch_spmm(cplx, cap, full, a, grid, 256, smem, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  return err = finish_reds(*this, reds, poffs, s, grid, a.pstride);
}

int Eng::upd(int s, std::vector<const void*> in, std::vector<OutSpec> outs, std::vector<RQ> reds) {
  if (err) return err;
  // An n-vector update (s = 1) with one-or-scalar coefficients and only norm / trace
  // reductions does not depend on the row structure: run it as an (n/4) x 4 block
  // (two lanes per row with 16-byte loads instead of one 8-byte element per lane).
  // The same holds for any width whose rows map badly onto 16-byte lanes — fewer than 64 bytes, or
  // a lane count that is not a power of two (config 4's complex s = 12: 12 lanes per row, 8 of a
  // warp's 32 idle; its scalar updates ran at 65-69% of HBM) —: the n x s block is viewed as
  // (n s / w) x w with 128-byte rows (w = 16 real / 8 complex, else the widest divisor of n s).
  {
    const int esz = cplx ? 16 : 8;
    const int lanes = (s * esz + 15) / 16;
    const bool awkward = s * esz < 64 || (lanes & (lanes - 1)) != 0;
    const long long tot = n * (long long)s;
    int w = 0;
    for (int cand : {128 / esz, 64 / esz, 32 / esz})
      if (cand > 0 && tot % cand == 0 && tot >= cand) {
        w = cand;
        break;
      }
    bool flat = awkward && w > 0 && w != s && (w * esz > s * esz || (lanes & (lanes - 1)) != 0);
    if (flat) {
      for (const OutSpec& o : outs)
        for (const TermSpec& t : o.t) flat &= (t.c.kind == CK_ONE || t.c.kind == CK_SCALAR);
      for (const RQ& r : reds) flat &= (r.mode == RED_NORM2 || r.mode == RED_TRACE);
      // the flat view loads 16 bytes per lane: every operand must be 16-byte aligned
      // (a caller's view at an 8-byte offset, e.g. v[1:], keeps the element-wise path)
      auto a16 = [](const void* p) { return p == nullptr || ((uintptr_t)p & 15) == 0; };
      for (const void* p : in) flat &= a16(p);
      for (const OutSpec& o : outs) flat &= a16(o.ptr);
      for (const RQ& r : reds) flat &= a16(r.yext);
    }
    if (flat) {
      const long long n0 = n;
      n = tot / w;
      const int r = upd(w, std::move(in), std::move(outs), std::move(reds));
      n = n0;
      return r;
    }
  }
  // an external n x s reduction operand becomes one more input, so its rows are
  // requested together with the other inputs instead of after the outputs
  for (RQ& r : reds)
    if (r.y < 0 && r.yext && r.mode != RED_SUMVEC && r.mode != RED_NORM2 && r.mode != RED_COLNORM2 &&
        in.size() < (size_t)MAX_IN) {
      in.push_back(r.yext);
      r.y = (int)in.size() - 1;
      r.yext = nullptr;
    }
  const int cap = cap_for(s);
  // s x s Grams wider than the in-kernel epilogue run on the tensor cores: before the
  // update when they read only inputs, after it when they read an output
  struct Wide {
    const void *x, *y;
    int woff;
  };
  std::vector<Wide> pre, post;
  // updates with s x s coefficients run on the tensor cores (blk_mma.cu); their s x s
  // Grams then go to the tensor-core Gram kernel as well
  bool full_coef = false;
  for (auto& o : outs)
    for (auto& t : o.t) full_coef |= (t.c.kind == CK_FULL);
  static const bool no_mma = getenv("SRK_NO_DMMA_UPDATE") != nullptr;  // A/B switch for measurements
  const bool use_mma = full_coef && !no_mma && upd_mma_width(s * (cplx ? 2 : 1)) > 0;
  // (s >= 8: also a reductions-only pass such as Bl-QMR's delta = W^H V — the DMMA Gram
  // reads the two blocks at 4.8 TB/s against 1.5 for the FMA epilogue's s x s accumulators)
  if (!full_red_supported(cplx, cap) || use_mma || s >= 8) {
    auto ptr = [&](int src) -> const void* {
      if (src >= 0 && src < (int)in.size()) return in[src];
      if (src >= SRC_OUT && src - SRC_OUT < (int)outs.size()) {
        const OutSpec& o = outs[src - SRC_OUT];
        if (o.ptr) return o.ptr;
        // a register-only output that is a plain copy of an input is that input
        if (o.t.size() == 1 && o.t[0].c.kind == CK_ONE && !o.t[0].c.neg && o.t[0].src >= 0 && o.t[0].src < (int)in.size())
          return in[o.t[0].src];
      }
      return nullptr;
    };
    auto overwritten = [&](int src) {  // an input whose buffer an output rewrites
      if (src < 0 || src >= (int)in.size()) return false;
      for (auto& o : outs)
        if (o.ptr == in[src]) return true;
      return false;
    };
    for (auto it = reds.begin(); it != reds.end();) {
      if (it->mode != RED_FULL) {
        ++it;
        continue;
      }
      const void* x = ptr(it->x);
      const void* y = it->y >= 0 ? ptr(it->y) : it->yext;
      auto is_copy = [&](int src) {
        return src >= SRC_OUT && src - SRC_OUT < (int)outs.size() && !outs[src - SRC_OUT].ptr;
      };
      const bool after = (it->x >= SRC_OUT && !is_copy(it->x)) || (it->y >= SRC_OUT && !is_copy(it->y));
      if (!x || !y || (after && (overwritten(it->x) || overwritten(it->y)))) return err = (int)cudaErrorNotSupported;
      (after ? post : pre).push_back(Wide{x, y, it->woff});
      it = reds.erase(it);
    }
  }
  for (const Wide& w : pre)
    if ((err = gram_full(w.x, w.y, s, w.woff))) return err;
  if (!post.empty()) {
    if ((err = upd(s, in, outs, reds))) return err;
    for (const Wide& w : post)
      if ((err = gram_full(w.x, w.y, s, w.woff))) return err;
    return 0;
  }
  bool full = false;  // s x s Gram or s x s coefficient: the block-method kernel instance
  for (auto& r : reds) full |= (r.mode == RED_FULL);
  for (auto& o : outs)
    for (auto& t : o.t) full |= (t.c.kind == CK_FULL);
  if (full && !full_supported(cplx, cap)) return err = (int)cudaErrorNotSupported;
  if (in.size() > MAX_IN || outs.size() > MAX_OUT || reds.size() > MAX_RED) return err = (int)cudaErrorInvalidValue;
  UpdArgs a{};
  a.nin = (int)in.size();
  for (size_t i = 0; i < in.size(); ++i) a.in[i] = in[i];
  a.nout = (int)outs.size();
  for (int o = 0; o < MAX_OUT; ++o)
    for (int b = 0; b < MAX_SRC; ++b) a.cf[o][b].kind = CK_NONE;
  const int pw = padded_width(cap, cplx);
  int cslot = 0;
  for (size_t o = 0; o < outs.size(); ++o) {
    a.out[o] = outs[o].ptr;
    for (const TermSpec& t : outs[o].t) {
      const int src = t.src;
      // inputs 0..nin-1, or an earlier output (SRC_OUT + o' with o' < o); one term per source
      const bool ok = (src >= 0 && src < (int)in.size()) || (src >= SRC_OUT && src - SRC_OUT < (int)o);
      if (!ok || a.cf[o][src].kind != CK_NONE) return err = (int)cudaErrorInvalidValue;
      a.cf[o][src] = t.c;
      a.cslot[o][src] = cslot;
      const int k = t.c.kind;
      cslot += (k == CK_FULL) ? cap * pw : (k == CK_DIAG ? pw : 1);
      if (cslot & 1) cslot++;  // keep 16-byte alignment of the following slot
    }
  }
  a.cslot_total = cslot;
  a.nred = (int)reds.size();
  std::vector<int> poffs;
  int pstride = 0, maxlen = 0;
  for (size_t i = 0; i < reds.size(); ++i) {
    if (reds[i].mode == RED_FULL && i == 2) return err = (int)cudaErrorInvalidValue;  // slot 2 holds no s x s Gram
    fill_red(a.red[i], reds[i], pstride);
    poffs.push_back(pstride);
    const int len = red_len(reds[i].mode, s, cplx);
    pstride += len;
    maxlen = std::max(maxlen, len);
  }
  a.pstride = std::max(pstride, 1);
  a.ws = ws;
  a.n = n;
  a.s = s;
  a.vec = cplx ? 1 : (s % 2 == 0);
  a.done = done;
  const size_t esz = cplx ? 16 : 8;
  if (use_mma) {
    int nterm = 0;
    for (int o = 0; o < MAX_OUT; ++o)
      for (int q = 0; q < MAX_SRC; ++q) a.cslot[o][q] = a.cf[o][q].kind == CK_NONE ? -1 : nterm++;
    const int w = s * (cplx ? 2 : 1);
    static int occ_mma[3] = {0, 0, 0};
    int& occ = occ_mma[upd_mma_width(w) == 8 ? 0 : (upd_mma_width(w) == 16 ? 1 : 2)];
    if (occ == 0) occ = std::max(1, launch_upd_mma(a, cplx, MAX_OUT * 2, -1, nullptr));
    const long long need = (n + 63) / 64;  // 8 warps x 8 rows per CTA step
    const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)c->nsm * occ));
    if ((err = c->ensure_partials((size_t)grid * a.pstride))) return err;
    a.partials = c->partials;
    nlaunch++;
    if (prof) {
      int nw = 0;
      for (auto& o : outs) nw += o.ptr ? 1 : 0;
      prof->begin(PT_UPD, c->st, 16 * a.nin + a.nout, (double)n * s * esz * (a.nin + nw));
    }
    err = launch_upd_mma(a, cplx, nterm, grid, c->st);
    if (prof) prof->end(c->st);
    if (err) return err;
    return err = finish_reds(*this, reds, poffs, s, grid, a.pstride);
  }
  const size_t smem = (size_t)cslot * esz + (size_t)8 * maxlen * sizeof(double);
  const int grid = grid_for(cap, full, false, 48 * 1024, a.nin);  // occupancy at a fixed smem budget (deterministic grid)
  if ((err = c->ensure_partials((size_t)grid * a.pstride))) return err;
  a.partials = c->partials;
  nlaunch++;
  if (prof) {
    double nb = (double)n * s * esz * (double)a.nin;
    int nw = 0;
    for (auto& o : outs) nw += o.ptr ? 1 : 0;
    nb += (double)n * s * esz * nw;
    for (auto& r : reds)
      if (r.y < 0 && r.yext && r.mode != RED_NORM2 && r.mode != RED_COLNORM2)
        nb += (double)n * (r.mode == RED_SUMVEC ? 1 : s) * esz;
    prof->begin(PT_UPD, c->st, 16 * a.nin + a.nout, nb);
  }
  err = launch_upd(cplx, cap, full, a, grid, 256, smem, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  return err = finish_reds(*this, reds, poffs, s, grid, a.pstride);
}

static int log2_or_neg(int v) {
  for (int k = 0; k < 31; ++k)
    if ((1 << k) == v) return k;
  return -1;
}

int Eng::flat(int plan, int s, std::vector<const void*> in, std::vector<void*> out, std::vector<int> coff,
              std::vector<int> woff) {
  if (err) return err;
  const FlatPlanInfo pi = flat_plan_info(plan);
  if (!qmr_tail_ok(s) || pi.ni == 0 || (int)in.size() != pi.ni || (int)out.size() != pi.no || (int)coff.size() != pi.nc ||
      (int)woff.size() != pi.nr)
    return err = (int)cudaErrorInvalidValue;
  const size_t esz = cplx ? 16 : 8;
  FlatArgs a{};
  for (int i = 0; i < pi.ni; ++i) a.in[i] = in[i];
  for (int i = 0; i < pi.no; ++i) a.out[i] = out[i];
  for (int i = 0; i < pi.nc; ++i) a.coff[i] = coff[i];
  a.units = (long long)((size_t)n * s * esz / 16);
  a.ws = ws;
  a.done = done;
  std::vector<RQ> reds;
  std::vector<int> poffs;
  int pstride = 0;
  for (int r = 0; r < pi.nr; ++r) {
    reds.push_back(RQ{pi.rmode[r], 0, -1, nullptr, woff[r]});
    poffs.push_back(pstride);
    pstride += red_len(pi.rmode[r], s, cplx);  // NORM2: 1, TRACE: one value
  }
  a.pstride = std::max(pstride, 1);
  static std::atomic<int> occ_c[8][2] = {};
  int occ = occ_c[plan & 7][cplx].load();
  if (occ == 0) {
    occ = std::max(1, launch_flat(plan, cplx, a, -1, nullptr));
    occ_c[plan & 7][cplx].store(occ);
  }
  const long long need = std::max<long long>(1, (a.units + 255) / 256);
  const int grid = (int)std::min<long long>(need, (long long)c->nsm * occ);  // one wave
  if ((err = c->ensure_partials((size_t)grid * a.pstride))) return err;
  a.partials = c->partials;
  nlaunch++;
  if (prof) prof->begin(PT_UPD, c->st, 16 * pi.ni + pi.no, (double)(pi.ni + pi.no) * (double)n * s * esz);
  err = launch_flat(plan, cplx, a, grid, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  return err = finish_reds(*this, reds, poffs, s, grid, a.pstride);
}

int Eng::egl_bicg_flat(int which, int s, void* X, void* R, void* P, const void* Q, void* rh, void* ph, const void* qh,
                       int off_alpha, int off_beta, int woff_rhon, int woff_r2) {
  if (err) return err;
  if (!qmr_vec_ok(s)) return err = (int)cudaErrorInvalidValue;
  const size_t esz = cplx ? 16 : 8;
  EglFlatArgs a{};
  a.X = X; a.R = R; a.P = P; a.Q = Q; a.rh = rh; a.ph = ph; a.qh = qh;
  a.upr = (int)((size_t)s * esz / 16);
  a.sh = log2_or_neg(a.upr);
  a.units = n * (long long)a.upr;
  a.ws = ws;
  a.off_alpha = off_alpha; a.off_beta = off_beta;
  const int nd = cplx ? 2 : 1;
  a.pstride = nd + 1;
  a.done = done;
  static std::atomic<int> occ_c[2][2] = {};
  int occ = occ_c[which & 1][cplx].load();
  if (occ == 0) {
    occ = std::max(1, launch_egl_flat(which, cplx, a, -1, nullptr));
    occ_c[which & 1][cplx].store(occ);
  }
  const long long need = std::max<long long>(1, (a.units + 255) / 256);
  const int grid = (int)std::min<long long>(need, (long long)c->nsm * occ);  // one wave
  if (which == 0 && (err = c->ensure_partials((size_t)grid * a.pstride))) return err;
  a.partials = c->partials;
  nlaunch++;
  const double B = (double)n * s * esz, v = (double)n * esz;
  if (prof) prof->begin(PT_UPD, c->st, which == 0 ? 16 * 4 + 2 : 16 * 2 + 1, which == 0 ? 6.0 * B + 2.0 * v : 3.0 * B + 5.0 * v);
  err = launch_egl_flat(which, cplx, a, grid, c->st);
  if (prof) prof->end(c->st);
  if (err || which != 0) return err;
  return err = finish_reds(*this, {RQ{RED_SUMVEC, SRC_OUT + 1, -1, rh, woff_rhon}, RQ{RED_NORM2, SRC_OUT + 1, -1, nullptr, woff_r2}},
                           {0, nd}, s, grid, a.pstride);
}

int Eng::qmr_vt(int s, const void* Pt, void* Vt, const void* AHQ, const void* Wt, int off_br, int off_bx, int woff_rho2,
                int woff_k1, int woff_xi2) {
  if (err) return err;
  if (!qmr_vec_ok(s)) return err = (int)cudaErrorInvalidValue;
  const size_t esz = cplx ? 16 : 8;
  QmrVtArgs a{};
  a.Pt = Pt; a.Vt = Vt; a.AHQ = AHQ; a.Wt = Wt;
  a.upr = (int)((size_t)s * esz / 16);
  a.sh = log2_or_neg(a.upr);
  a.units = n * (long long)a.upr;
  a.ws = ws;
  a.off_br = off_br; a.off_bx = off_bx;
  a.pstride = 2 + (cplx ? 2 : 1);
  a.done = done;
  static std::atomic<int> occ_c[2] = {{0}, {0}};
  int occ = occ_c[cplx].load();
  if (occ == 0) {
    occ = std::max(1, launch_qmr_vt(cplx, a, -1, nullptr));
    occ_c[cplx].store(occ);
  }
  const long long need = std::max<long long>(1, (a.units + 255) / 256);
  const int grid = (int)std::min<long long>(need, (long long)c->nsm * occ);
  if ((err = c->ensure_partials((size_t)grid * a.pstride))) return err;
  a.partials = c->partials;
  nlaunch++;
  if (prof) prof->begin(PT_UPD, c->st, 16 * 2 + 1, 3.0 * (double)n * s * esz + 2.0 * (double)n * esz);
  err = launch_qmr_vt(cplx, a, grid, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  const int nd = cplx ? 2 : 1;
  return err = finish_reds(*this,
                           {RQ{RED_NORM2, SRC_OUT, -1, nullptr, woff_rho2}, RQ{RED_SUMVEC, SRC_OUT, -1, Wt, woff_k1},
                            RQ{RED_NORM2, SRC_OUT, -1, nullptr, woff_xi2}},
                           {0, 1, 1 + nd}, s, grid, a.pstride);
}

int Eng::qmr_tail(int s, void* P, void* D, const void* Pt, void* S, void* X, void* R, const void* Vt, int off_eta,
                  int off_f, int off_invrho, int off_c1, int woff_r2, const QmrVec* v) {
  if (err) return err;
  if (!qmr_tail_ok(s)) return err = (int)cudaErrorInvalidValue;
  const size_t esz = cplx ? 16 : 8;
  QmrTailArgs a{};
  a.P = P; a.D = D; a.S = S; a.X = X; a.R = R; a.Pt = Pt; a.Vt = Vt;
  a.units = (long long)((size_t)n * s * esz / 16);
  a.ws = ws;
  a.off_eta = off_eta; a.off_f = off_f; a.off_invrho = off_invrho; a.off_c1 = off_c1;
  a.pstride = 1;
  a.poff = 0;
  a.done = done;
  if (v) {
    if (!qmr_vec_ok(s)) return err = (int)cudaErrorInvalidValue;
    a.Wt = v->Wt; a.Qv = v->Qv; a.AHQ = v->AHQ;
    a.upr = (int)((size_t)s * esz / 16);
    a.sh = log2_or_neg(a.upr);
    a.off_bx = v->off_bx; a.off_invxi = v->off_invxi; a.off_c2 = v->off_c2;
  }
  static std::atomic<int> occ_c[2] = {{0}, {0}};
  int occ = occ_c[cplx].load();
  if (occ == 0) {
    occ = std::max(1, launch_qmr_tail(cplx, a, -1, nullptr));
    occ_c[cplx].store(occ);
  }
  const long long need = std::max<long long>(1, (a.units + 255) / 256);
  const int grid = (int)std::min<long long>(need, (long long)c->nsm * occ);  // one wave
  if ((err = c->ensure_partials((size_t)grid))) return err;
  a.partials = c->partials;
  nlaunch++;
  if (prof) prof->begin(PT_UPD, c->st, 16 * 7 + 5, 12.0 * (double)n * s * esz + (v ? 5.0 * (double)n * esz : 0.0));
  err = launch_qmr_tail(cplx, a, grid, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  return err = finish_reds(*this, {RQ{RED_NORM2, SRC_OUT + 3, -1, nullptr, woff_r2}}, {0}, s, grid, 1);
}

// Block-sparse operator: the BSR product, then the requested reductions over Q as
// one fused update pass (X = Q; Y the external operand, as in the CSR epilogue).
int Eng::spmm_bsr(bool adj, const void* P, void* Q, int s, const std::vector<RQ>& reds) {
  if (adj || !bsr_supported(A->bs, cplx, s)) return err = (int)cudaErrorNotSupported;
  // distributed lattice (t-slabs): the ghost block rows (12 P rows each) arrive first
  if ((err = halo(false, P, s))) return err;
  BsrArgs a{};
  a.brp = A->brp;
  a.bci = A->bci;
  a.val = A->bval;
  a.P = P;
  a.Q = Q;
  a.nb = A->nb;
  a.order = A->border;
  a.unit_diag = A->unit_diag;
  a.done = done;
  const int wpc = bsr_warps_per_cta();  // one warp per block row
  const int wsm = std::max(wpc, launch_bsr(a, s, -1, nullptr));  // resident warps per SM
  const long long need = (A->nb + wpc - 1) / wpc;
  const int grid = (int)std::max<long long>(1, std::min<long long>(need, (long long)c->nsm * (wsm / wpc)));
  // the epilogue fuses every reduction except the s x s Gram (a separate pass below)
  std::vector<RQ> fused, rest;
  for (const RQ& q : reds) (q.mode == RED_FULL ? rest : fused).push_back(q);
  if (fused.size() > 2) {
    rest.insert(rest.end(), fused.begin() + 2, fused.end());
    fused.resize(2);
  }
  std::vector<int> poffs;
  int pstride = 0;
  a.nred = (int)fused.size();
  for (size_t i = 0; i < fused.size(); ++i) {
    fill_red(a.red[i], fused[i], pstride);
    poffs.push_back(pstride);
    pstride += red_len(fused[i].mode, s, true);
  }
  a.pstride = std::max(pstride, 1);
  if (!fused.empty()) {
    if ((err = c->ensure_partials((size_t)grid * a.pstride))) return err;
    a.partials = c->partials;
  }
  nlaunch++;
  if (prof) {
    const double esz = 16.0;
    double nb = (double)(A->nb + 1) * 4 + (double)A->nnzb * (4 + A->bs * A->bs * esz) + 2.0 * (double)n * s * esz;
    for (const RQ& q : fused)
      if (q.yext && q.mode != RED_NORM2 && q.mode != RED_COLNORM2)
        nb += (double)n * (q.mode == RED_SUMVEC ? 1 : s) * esz;
    prof->begin(PT_SPMM, c->st, s, nb);
  }
  err = launch_bsr(a, s, grid, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  if (!fused.empty() && (err = finish_reds(*this, fused, poffs, s, grid, a.pstride))) return err;
  if (rest.empty()) return 0;
  std::vector<RQ> r2;
  for (const RQ& q : rest) r2.push_back(RQ{q.mode, 0, -1, q.yext, q.woff});
  return upd(s, {Q}, {}, r2);
}

// Right preconditioning: the solvers iterate on
// A M^-1 Y = B. A-products become Q = A (U^-1 L^-1 P) with the reductions fused as
// usual; A^H-products Q = L^-H U^-H (A^H P), reductions in one pass afterwards.
int Eng::spmm_prec(bool adj, const void* P, void* Q, int s, const std::vector<RQ>& reds) {
  Prec* M = A->prec;
  const size_t bytes = (size_t)n * s * (cplx ? 16 : 8);
  if (M->scratch_bytes < bytes) {  // (never inside a graph capture: the first iteration runs eagerly)
    for (void*& p : M->scratch) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    M->scratch_bytes = 0;
    if (cudaMalloc(&M->scratch[0], bytes) != cudaSuccess) return err = (int)cudaErrorMemoryAllocation;
    M->scratch_bytes = bytes;
  }
  void* T = M->scratch[0];
  auto tri = [&](const DevTri& t, const void* R, void* Z) {
    if (prof) prof->begin(PT_OTHER, c->st, s, 0.0);
    const int r = launch_trsv(t, cplx, n, s, R, Z, done, c->st);
    if (prof) prof->end(c->st);
    if (r < 0) return err = -r;
    nlaunch += r;
    return 0;
  };
  if (!adj) {
    if (M->perm) {  // ILUTP: U^-1 L^-1 (Pi P)
      nlaunch++;
      if ((err = launch_permute(M->perm, true, cplx, n, s, P, T, c->st))) return err;
      if (tri(M->L, T, T) || tri(M->U, T, T)) return err;
    } else if (tri(M->L, P, T) || tri(M->U, T, T)) {
      return err;
    }
    raw = true;
    const int r = spmm(false, T, Q, s, reds);
    raw = false;
    return r;
  }
  raw = true;
  int r = spmm(true, P, T, s, {});
  raw = false;
  if (r) return r;
  if (M->perm) {  // ILUTP: Pi^T L^-H U^-H (A^H P)
    if (tri(M->UH, T, T) || tri(M->LH, T, T)) return err;
    nlaunch++;
    if ((err = launch_permute(M->perm, false, cplx, n, s, T, Q, c->st))) return err;
  } else if (tri(M->UH, T, T) || tri(M->LH, T, Q)) {
    return err;
  }
  if (reds.empty()) return 0;
  std::vector<RQ> r2;
  for (const RQ& q : reds) r2.push_back(RQ{q.mode, 0, -1, q.yext, q.woff});
  return upd(s, {Q}, {}, r2);
}

int Eng::prec_solve(bool adj, const void* Y, void* X, int s) {
  Prec* M = A->prec;
  if (!M) return err = (int)cudaErrorInvalidValue;
  const DevTri& first = adj ? M->UH : M->L;
  const DevTri& second = adj ? M->LH : M->U;
  int r;
  if (M->perm && !adj) {  // U^-1 L^-1 (Pi Y)
    if (Y == X) {  // in place: the gather needs a copy of Y
      void* T = nullptr;
      const size_t bytes = (size_t)n * s * (cplx ? 16 : 8);
      if (cudaMalloc(&T, bytes) != cudaSuccess) return err = (int)cudaErrorMemoryAllocation;
      cudaMemcpyAsync(T, Y, bytes, cudaMemcpyDeviceToDevice, c->st);
      r = launch_permute(M->perm, true, cplx, n, s, T, X, c->st);
      cudaStreamSynchronize(c->st);
      cudaFree(T);
    } else {
      r = launch_permute(M->perm, true, cplx, n, s, Y, X, c->st);
    }
    if (r) return err = r;
    r = launch_trsv(first, cplx, n, s, X, X, nullptr, c->st);
  } else {
    r = launch_trsv(first, cplx, n, s, Y, X, nullptr, c->st);
  }
  if (r < 0) return err = -r;
  r = launch_trsv(second, cplx, n, s, X, X, nullptr, c->st);
  if (r < 0) return err = -r;
  if (M->perm && adj) {  // Pi^T (L^-H U^-H Y)
    void* T = nullptr;
    const size_t bytes = (size_t)n * s * (cplx ? 16 : 8);
    if (cudaMalloc(&T, bytes) != cudaSuccess) return err = (int)cudaErrorMemoryAllocation;
    cudaMemcpyAsync(T, X, bytes, cudaMemcpyDeviceToDevice, c->st);
    r = launch_permute(M->perm, false, cplx, n, s, T, X, c->st);
    cudaStreamSynchronize(c->st);
    cudaFree(T);
    if (r) return err = r;
  }
  return 0;
}

int Eng::prec_mul(const void* X, void* Y, int s) {  // Y = L (U X)
  Prec* M = A->prec;
  if (!M) return err = (int)cudaErrorInvalidValue;
  const size_t bytes = (size_t)n * s * (cplx ? 16 : 8);
  void* T = nullptr;
  if (cudaMalloc(&T, bytes) != cudaSuccess) return err = (int)cudaErrorMemoryAllocation;
  int r = launch_trimul(M->U, cplx, n, s, X, T, c->st);
  if (!r) r = launch_trimul(M->L, cplx, n, s, T, Y, c->st);
  if (!r && M->perm) {  // ILUTP: M X = Pi^T (L U X)
    cudaMemcpyAsync(T, Y, bytes, cudaMemcpyDeviceToDevice, c->st);
    r = launch_permute(M->perm, false, cplx, n, s, T, Y, c->st);
  }
  cudaStreamSynchronize(c->st);
  cudaFree(T);
  return err = r;
}

int Eng::gram_full(const void* X, const void* Y, int s, int woff) {
  if (err) return err;
  GramArgs g{};
  g.X = reinterpret_cast<const double*>(X);
  g.Y = reinterpret_cast<const double*>(Y);
  g.n = n;
  g.w = s * (cplx ? 2 : 1);
  g.s = s;
  g.cplx = cplx ? 1 : 0;
  const int len = red_len(RED_FULL, s, cplx);
  const int occ = std::max(1, launch_gram_mma(g, -1, c->st));
  const int grid = (int)std::max(1, std::min(c->nsm * occ, gram_mma_chunks(n)));
  if ((err = c->ensure_partials((size_t)grid * len))) return err;
  g.partials = c->partials;
  g.pstride = len;
  g.done = done;
  nlaunch++;
  if (prof) prof->begin(PT_UPD, c->st, 16 * (X == Y ? 1 : 2) + 0, (X == Y ? 1.0 : 2.0) * (double)n * s * (cplx ? 16 : 8));
  err = launch_gram_mma(g, grid, c->st);
  if (prof) prof->end(c->st);
  if (err) return err;
  return err = finish_reds(*this, {RQ{RED_FULL, 0, 1, nullptr, woff}}, {0}, s, grid, len);
}

// ---------------------------------------------------------------------------
// balanced row order (SELL-C-sigma's sorting step with sigma = n, C = one warp)
// ---------------------------------------------------------------------------
template <typename T>
__global__ static void gather_sorted_rows(const int* rp, const int* ci, const T* val, const int* perm, const int* rp2,
                                          int* ci2, T* val2, long long n) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long l = warp; l < n; l += nw) {
    const int src = perm[l];
    const int b = rp[src], len = rp[src + 1] - b, d = rp2[l];
    for (int j = lane; j < len; j += 32) {
      ci2[d + j] = ci[b + j];
      val2[d + j] = val[b + j];
    }
  }
}

int build_sell(Mat& m, bool adj, const std::vector<int>& h, cudaStream_t st);

int build_balanced_order(Mat& m, bool adj, cudaStream_t st) {
  const int* rp = adj ? m.rpH : m.rp;
  const int* ci = adj ? m.ciH : m.ci;
  const void* val = adj ? m.valH : m.val;
  const long long n = m.n, nnz = adj ? m.nnzH : m.nnz;
  if (n < 1 || nnz < 1 || !rp) return 0;
  std::vector<int> h(n + 1);
  if (cudaMemcpyAsync(h.data(), rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return (int)cudaErrorUnknown;
  long long maxlen = 0;
  for (long long i = 0; i < n; ++i) maxlen = std::max<long long>(maxlen, h[i + 1] - h[i]);
  const double mean = (double)nnz / (double)n;
  // regular lengths (stencils, lattices): a warp's rows already have equal work
  if ((double)maxlen < 4.0 * mean + 8.0) return 0;
  std::vector<int> perm(n);
  for (long long i = 0; i < n; ++i) perm[i] = (int)i;
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return h[x + 1] - h[x] > h[y + 1] - h[y]; });
  std::vector<int> rp2(n + 1);
  rp2[0] = 0;
  for (long long l = 0; l < n; ++l) rp2[l + 1] = rp2[l] + (h[perm[l] + 1] - h[perm[l]]);
  Mat::Sorted& so = adj ? m.srtH : m.srt;
  const size_t esz = m.cplx ? 16 : 8;
  if (cudaMalloc(&so.rp, sizeof(int) * (n + 1)) != cudaSuccess || cudaMalloc(&so.perm, sizeof(int) * n) != cudaSuccess ||
      cudaMalloc(&so.ci, sizeof(int) * (nnz + 1)) != cudaSuccess || cudaMalloc(&so.val, esz * (nnz + 1)) != cudaSuccess)
    return (int)cudaErrorMemoryAllocation;
  cudaMemcpyAsync(so.rp, rp2.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(so.perm, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st);
  const int grid = (int)std::min<long long>((n + 7) / 8, 148 * 16);
  if (m.cplx)
    gather_sorted_rows<double2><<<grid, 256, 0, st>>>(rp, ci, reinterpret_cast<const double2*>(val), so.perm, so.rp, so.ci,
                                                      reinterpret_cast<double2*>(so.val), n);
  else
    gather_sorted_rows<double><<<grid, 256, 0, st>>>(rp, ci, reinterpret_cast<const double*>(val), so.perm, so.rp, so.ci,
                                                     reinterpret_cast<double*>(so.val), n);
  if (cudaStreamSynchronize(st) != cudaSuccess) return (int)cudaErrorUnknown;  // rp2 / perm host buffers go out of scope
  return build_sell(m, adj, h, st);
}

// SELL-32-sigma (Kreutzer et al.'s format): sigma-window sort, 32-row chunks,
// column-major padded storage; filled on the device from the CSR arrays
template <typename T>
__global__ static void fill_sell(const int* rp, const int* ci, const T* val, const int* srow, const int* cs, int* ci2,
                                 T* val2, long long nchunk) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long c = warp; c < nchunk; c += nw) {
    const int base = cs[c], w = (cs[c + 1] - base) >> 5;
    const int src = srow[c * 32 + lane];
    const int b = src >= 0 ? rp[src] : 0, len = src >= 0 ? rp[src + 1] - b : 0;
    for (int j = 0; j < w; ++j) {
      const bool in = j < len;
      ci2[(size_t)base + (size_t)j * 32 + lane] = in ? ci[b + j] : -1;
      val2[(size_t)base + (size_t)j * 32 + lane] = in ? val[b + j] : T{};
    }
  }
}

int build_sell(Mat& m, bool adj, const std::vector<int>& h, cudaStream_t st) {
  static const bool off = getenv("SRK_NO_SELL") != nullptr;  // A/B switch: the team-per-row kernel instead
  if (off) return 0;
  static const int env_sigma = getenv("SRK_SELL_SIGMA") ? atoi(getenv("SRK_SELL_SIGMA")) : 0;
  const long long n = m.n;
  // sigma: the sorting window. Large windows pad least; the output rows of a chunk stay within one
  // window, so Q's scattered narrow writes merge in L2 (default 2^16 rows; <= 0: the whole matrix)
  const long long sigma = env_sigma > 0 ? std::max(32, env_sigma / 32 * 32) : (env_sigma < 0 ? n : 65536);
  const long long nchunk = (n + 31) / 32;
  std::vector<int> row(nchunk * 32, -1);
  for (long long i = 0; i < n; ++i) row[i] = (int)i;
  for (long long w0 = 0; w0 < n; w0 += sigma) {
    const long long w1 = std::min(n, w0 + sigma);
    std::stable_sort(row.begin() + w0, row.begin() + w1, [&](int x, int y) { return h[x + 1] - h[x] > h[y + 1] - h[y]; });
  }
  std::vector<int> cs(nchunk + 1), width(nchunk);
  long long tot = 0;
  for (long long c = 0; c < nchunk; ++c) {
    int w = 0;
    for (int l = 0; l < 32; ++l) {
      const int r = row[c * 32 + l];
      if (r >= 0) w = std::max(w, h[r + 1] - h[r]);
    }
    width[c] = w;
    cs[c] = (int)tot;
    tot += 32LL * w;
    if (tot > 0x7fffff00LL) return 0;  // int32 offsets: keep the sorted CSR
  }
  cs[nchunk] = (int)tot;
  const long long nnz = adj ? m.nnzH : m.nnz;
  if ((double)tot > 1.25 * (double)nnz) return 0;  // too much padding: keep the sorted CSR
  std::vector<int> order(nchunk);
  for (long long c = 0; c < nchunk; ++c) order[c] = (int)c;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return width[x] > width[y]; });
  Mat::Sell& se = adj ? m.sellH : m.sell;
  const size_t esz = m.cplx ? 16 : 8;
  if (cudaMalloc(&se.cs, sizeof(int) * (nchunk + 1)) != cudaSuccess ||
      cudaMalloc(&se.row, sizeof(int) * nchunk * 32) != cudaSuccess ||
      cudaMalloc(&se.order, sizeof(int) * nchunk) != cudaSuccess ||
      cudaMalloc(&se.ci, sizeof(int) * std::max<long long>(tot, 1)) != cudaSuccess ||
      cudaMalloc(&se.val, esz * std::max<long long>(tot, 1)) != cudaSuccess)
    return (int)cudaErrorMemoryAllocation;
  se.nchunk = nchunk;
  se.entries = tot;
  se.sigma = (int)std::min<long long>(sigma, n);
  cudaMemcpyAsync(se.cs, cs.data(), sizeof(int) * (nchunk + 1), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(se.row, row.data(), sizeof(int) * nchunk * 32, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(se.order, order.data(), sizeof(int) * nchunk, cudaMemcpyHostToDevice, st);
  const int* rp = adj ? m.rpH : m.rp;
  const int* ci = adj ? m.ciH : m.ci;
  const void* val = adj ? m.valH : m.val;
  const int grid = (int)std::min<long long>((nchunk + 7) / 8, 148 * 16);
  if (m.cplx)
    fill_sell<double2><<<grid, 256, 0, st>>>(rp, ci, reinterpret_cast<const double2*>(val), se.row, se.cs, se.ci,
                                             reinterpret_cast<double2*>(se.val), nchunk);
  else
    fill_sell<double><<<grid, 256, 0, st>>>(rp, ci, reinterpret_cast<const double*>(val), se.row, se.cs, se.ci,
                                            reinterpret_cast<double*>(se.val), nchunk);
  return (int)cudaStreamSynchronize(st);  // the host arrays go out of scope
}

void free_balanced_order(Mat& m) {
  for (Mat::Sell* se : {&m.sell, &m.sellH}) {
    if (se->cs) cudaFree(se->cs);
    if (se->ci) cudaFree(se->ci);
    if (se->val) cudaFree(se->val);
    if (se->row) cudaFree(se->row);
    if (se->order) cudaFree(se->order);
    *se = Mat::Sell{};
  }
  for (Mat::Sorted* so : {&m.inner, &m.bnd, &m.innerH, &m.bndH}) {
    if (so->rp) cudaFree(so->rp);
    if (so->ci) cudaFree(so->ci);
    if (so->val) cudaFree(so->val);
    if (so->perm) cudaFree(so->perm);
    *so = Mat::Sorted{};
  }
  for (Mat::Sorted* so : {&m.srt, &m.srtH}) {
    if (so->rp) cudaFree(so->rp);
    if (so->ci) cudaFree(so->ci);
    if (so->val) cudaFree(so->val);
    if (so->perm) cudaFree(so->perm);
    *so = Mat::Sorted{};
  }
}

// ---------------------------------------------------------------------------
// small helper kernels
// ---------------------------------------------------------------------------
template <typename T>
__global__ void row_mean_kernel(const T* X, T* out, long long n, int s, const int* done) {
  if (done && *done) return;
  const double inv = 1.0 / s;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    T acc = Ar<T>::zero();
    for (int c = 0; c < s; ++c) acc = Ar<T>::add(acc, X[i * s + c]);
    if constexpr (Ar<T>::cplx) out[i] = mk(acc.x * inv, acc.y * inv);
    else out[i] = acc * inv;
  }
}

int launch_row_mean(bool cplx, const void* X, void* out, long long n, int s, const int* done, cudaStream_t st) {
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  if (cplx)
    row_mean_kernel<double2><<<std::max(grid, 1), 256, 0, st>>>((const double2*)X, (double2*)out, n, s, done);
  else
    row_mean_kernel<double><<<std::max(grid, 1), 256, 0, st>>>((const double*)X, (double*)out, n, s, done);
  return (int)cudaGetLastError();
}

// CSR validation (SPEC SparseMatrix invariants S:36): row_ptr non-decreasing,
// row_ptr[0] = 0, row_ptr[n] = nnz, columns in [0, ncols), strictly increasing per
// row when `sorted` (local rows of a distributed operator keep the global order).
__global__ void csr_check_kernel(long long n, long long ncols, long long nnz, const int* rp, const int* ci, int sorted,
                                 int* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int b = rp[i], e = rp[i + 1];
    if (e < b || b < 0 || e > nnz) { atomicOr(bad, 1); continue; }
    if (i == 0 && b != 0) atomicOr(bad, 1);
    if (i == n - 1 && e != nnz) atomicOr(bad, 1);
    for (int j = b; j < e; ++j) {
      const int c = ci[j];
      if (c < 0 || c >= ncols) atomicOr(bad, 2);
      if (sorted && j > b && c <= ci[j - 1]) atomicOr(bad, 4);
    }
  }
}

int launch_csr_check(long long n, long long ncols, long long nnz, const int* rp, const int* ci, int sorted, int* bad,
                     cudaStream_t st) {
  const int grid = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
  csr_check_kernel<<<grid, 256, 0, st>>>(n, ncols, nnz, rp, ci, sorted, bad);
  return (int)cudaGetLastError();
}

// halo pack: dst row k = src row idx[k] (rows of doubles_per_row doubles)
__global__ void gather_rows_kernel(const double* src, double* dst, const int* idx, long long nrows, int dpr,
                                   const int* done) {
  if (done && *done) return;
  const long long total = nrows * dpr;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long k = t / dpr;
    const int c = (int)(t % dpr);
    dst[t] = src[(long long)idx[k] * dpr + c];
  }
}

int launch_gather_rows(const double* src, double* dst, const int* idx, long long nrows, int dpr, const int* done,
                       cudaStream_t st) {
  if (nrows <= 0) return 0;
  const int grid = (int)std::max<long long>(1, std::min<long long>((nrows * dpr + 255) / 256, 148 * 8));
  gather_rows_kernel<<<grid, 256, 0, st>>>(src, dst, idx, nrows, dpr, done);
  return (int)cudaGetLastError();
}

// A^H = conj(A)^T as CSR: (1) count entries per column, (2) exclusive scan,
// (3) scatter with per-column cursors, (4) sort each row of A^H by column so
// the result is deterministic (integer atomics only decide slot order, which the
// sort removes).
__global__ void colcount_kernel(long long nnz, const int* ci, int* cnt) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < nnz; j += (long long)gridDim.x * blockDim.x)
    atomicAdd(cnt + ci[j], 1);
}

// single-CTA exclusive scan of n+1 ints (cnt -> rpT), chunked
// Exclusive prefix sum of the column counts (row pointers of A^H), multi-CTA: 1) every
// CTA sums its segment, 2) one CTA scans the segment sums, 3) every CTA scans its segment
// from its offset (block scans by warp shuffles; integer, so any order gives the same bits).
__device__ long long block_excl_scan(long long v, long long* sh /* >= 33 */, long long* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    long long t = lane < nw ? sh[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) sh[lane] = t;  // inclusive warp-total prefix
  }
  __syncthreads();
  const long long before = (w > 0 ? sh[w - 1] : 0) + x - v;
  if (total) *total = sh[nw - 1];
  __syncthreads();
  return before;
}

__global__ void seg_sum_kernel(long long n, long long seg, const int* cnt, long long* bsum) {
  __shared__ long long sh[33];
  const long long b0 = blockIdx.x * seg, b1 = b0 + seg < n ? b0 + seg : n;
  long long loc = 0;
  for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) loc += cnt[i];
  long long tot = 0;
  block_excl_scan(loc, sh, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void seg_offsets_kernel(int nb, long long* bsum, long long n, int* rpT) {
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int b = 0; b < nb; ++b) {
      const long long v = bsum[b];
      bsum[b] = acc;
      acc += v;
    }
    rpT[n] = (int)acc;
  }
}

__global__ void seg_scan_kernel(long long n, long long seg, const int* cnt, const long long* boff, int* rpT) {
  __shared__ long long sh[33];
  __shared__ long long carry;
  const long long b0 = blockIdx.x * seg, b1 = b0 + seg < n ? b0 + seg : n;
  if (threadIdx.x == 0) carry = boff[blockIdx.x];
  __syncthreads();
  constexpr int PER = 8;
  for (long long base = b0; base < b1; base += (long long)blockDim.x * PER) {
    const long long t0 = base + (long long)threadIdx.x * PER;
    long long loc = 0;
    for (int k = 0; k < PER; ++k)
      if (t0 + k < b1) loc += cnt[t0 + k];
    long long tot = 0;
    long long acc = carry + block_excl_scan(loc, sh, &tot);
    for (int k = 0; k < PER; ++k)
      if (t0 + k < b1) {
        rpT[t0 + k] = (int)acc;
        acc += cnt[t0 + k];
      }
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

template <typename T>
__global__ void scatter_kernel(long long n, const int* rp, const int* ci, const T* val, int* cursor, int* ciT,
                               T* valT) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    for (int j = rp[i]; j < rp[i + 1]; ++j) {
      const int c = ci[j];
      const int pos = atomicAdd(cursor + c, 1);
      ciT[pos] = (int)i;
      valT[pos] = Ar<T>::conj(val[j]);
    }
  }
}

template <typename T>
__global__ void rowsort_kernel(long long n, const int* rpT, int* ciT, T* valT) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int b = rpT[i], e = rpT[i + 1];
    for (int j = b + 1; j < e; ++j) {  // insertion sort (rows are short)
      const int c = ciT[j];
      const T v = valT[j];
      int k = j - 1;
      while (k >= b && ciT[k] > c) {
        ciT[k + 1] = ciT[k];
        valT[k + 1] = valT[k];
        --k;
      }
      ciT[k + 1] = c;
      valT[k + 1] = v;
    }
  }
}

int launch_csr_transpose(bool cplx, long long n, long long nnz, const int* rp, const int* ci, const void* val,
                         int* rpT, int* ciT, void* valT, int* work, cudaStream_t st) {
  const int gridn = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
  const int gridz = (int)std::max<long long>(1, std::min<long long>((nnz + 255) / 256, 148 * 8));
  cudaMemsetAsync(work, 0, sizeof(int) * n, st);
  colcount_kernel<<<gridz, 256, 0, st>>>(nnz, ci, work);
  const int nseg = (int)std::max<long long>(1, std::min<long long>(148 * 8, (n + 4095) / 4096));
  const long long seg = (n + nseg - 1) / nseg;
  long long* bsum = nullptr;
  if (cudaMalloc(&bsum, sizeof(long long) * nseg) != cudaSuccess) return (int)cudaErrorMemoryAllocation;
  seg_sum_kernel<<<nseg, 256, 0, st>>>(n, seg, work, bsum);
  seg_offsets_kernel<<<1, 32, 0, st>>>(nseg, bsum, n, rpT);
  seg_scan_kernel<<<nseg, 256, 0, st>>>(n, seg, work, bsum, rpT);
  cudaStreamSynchronize(st);
  cudaFree(bsum);
  cudaMemcpyAsync(work, rpT, sizeof(int) * n, cudaMemcpyDeviceToDevice, st);
  if (cplx) {
    scatter_kernel<double2><<<gridn, 256, 0, st>>>(n, rp, ci, (const double2*)val, work, ciT, (double2*)valT);
    rowsort_kernel<double2><<<gridn, 256, 0, st>>>(n, rpT, ciT, (double2*)valT);
  } else {
    scatter_kernel<double><<<gridn, 256, 0, st>>>(n, rp, ci, (const double*)val, work, ciT, (double*)valT);
    rowsort_kernel<double><<<gridn, 256, 0, st>>>(n, rpT, ciT, (double*)valT);
  }
  return (int)cudaGetLastError();
}


// Interior / boundary SpMM of a distributed operator: the halo (pack + exchange) runs on the
// context's side stream while the interior rows (no ghost column) are multiplied on the main
// stream; the boundary rows follow once the ghost rows have arrived. The two launches write
// consecutive blocks of CTA partials, reduced together in fixed order by fin_kernel.
int Eng::spmm_split(bool adj, const void* P, void* Q, int s, const std::vector<RQ>& reds, const Mat::Sorted& in,
                    long long ni, const Mat::Sorted& bd, long long nbd) {
  if (!c->side) {
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_p, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_h, cudaEventDisableTiming) != cudaSuccess)
      return (int)cudaErrorUnknown;
  }
  const int cap = cap_for(s);
  SpmmArgs a{};
  a.P = P;
  a.Q = Q;
  a.s = s;
  a.vec = cplx ? 1 : (s % 2 == 0);
  a.nred = (int)reds.size();
  std::vector<int> poffs;
  int pstride = 0, maxlen = 0;
  for (size_t i = 0; i < reds.size(); ++i) {
    fill_red(a.red[i], reds[i], pstride);
    poffs.push_back(pstride);
    const int len = red_len(reds[i].mode, s, cplx);
    pstride += len;
    maxlen = std::max(maxlen, len);
  }
  a.pstride = std::max(pstride, 1);
  const size_t smem = (size_t)8 * maxlen * sizeof(double);
  a.done = done;
  a.team = 0;
  // grids sized to each part's rows (both in the persistent-grid budget of one launch)
  auto part_grid = [&](long long rows) {
    const int g = grid_for(cap, false, true, 8 * 2 * 8 * 16 * 16, 0);
    const long long need = std::max(1LL, (rows + 255) / 256);
    return (int)std::min<long long>(g, need);
  };
  const int g1 = ni > 0 ? part_grid(ni) : 0, g2 = nbd > 0 ? part_grid(nbd) : 0;
  if ((err = c->ensure_partials((size_t)(g1 + g2) * a.pstride))) return err;
  cudaEventRecord(c->ev_p, c->st);
  cudaStreamWaitEvent(c->side, c->ev_p, 0);
  if ((err = halo(adj, P, s, c->side))) return err;
  cudaEventRecord(c->ev_h, c->side);
  const double esz = cplx ? 16.0 : 8.0;
  const double nz = (double)(adj ? A->nnzH : A->nnz);
  if (g1 > 0) {
    a.row_ptr = in.rp;
    a.col_idx = in.ci;
    a.val = in.val;
    a.perm = in.perm;
    a.n = ni;
    a.partials = c->partials;
    nlaunch++;
    if (prof) prof->begin(adj ? PT_SPMM_ADJ : PT_SPMM, c->st, s, ((double)ni / n) * ((n + 1) * 4.0 + nz * (4 + esz) + 2.0 * n * s * esz));
    err = launch_spmm(cplx, cap, false, a, g1, 256, smem, c->st);
    if (prof) prof->end(c->st);
    if (err) return err;
  }
  cudaStreamWaitEvent(c->st, c->ev_h, 0);
  if (g2 > 0) {
    a.row_ptr = bd.rp;
    a.col_idx = bd.ci;
    a.val = bd.val;
    a.perm = bd.perm;
    a.n = nbd;
    a.partials = c->partials + (size_t)g1 * a.pstride;
    nlaunch++;
    if (prof) prof->begin(adj ? PT_SPMM_ADJ : PT_SPMM, c->st, s, ((double)nbd / n) * ((n + 1) * 4.0 + nz * (4 + esz) + 2.0 * n * s * esz));
    err = launch_spmm(cplx, cap, false, a, g2, 256, smem, c->st);
    if (prof) prof->end(c->st);
    if (err) return err;
  }
  if (g1 + g2 == 0) return 0;
  // both launches' partials: [g1 + g2][pstride], one fixed-order finalisation
  return finish_reds(*this, reds, poffs, s, g1 + g2, a.pstride);
}

int build_halo_split(Mat& m, bool adj, cudaStream_t st) {
  const int* rp = adj ? m.rpH : m.rp;
  const int* ci = adj ? m.ciH : m.ci;
  const void* val = adj ? m.valH : m.val;
  const long long n = m.n, nnz = adj ? m.nnzH : m.nnz;
  if (!m.dist || n < 1 || !rp || (adj ? m.srtH.perm : m.srt.perm)) return 0;  // (irregular: the sorted order)
  std::vector<int> h(n + 1), hc(std::max(1LL, nnz));
  if (cudaMemcpyAsync(h.data(), rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      (nnz > 0 && cudaMemcpyAsync(hc.data(), ci, sizeof(int) * nnz, cudaMemcpyDeviceToHost, st) != cudaSuccess) ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return (int)cudaErrorUnknown;
  std::vector<int> lst[2];  // 0 interior, 1 boundary
  for (long long i = 0; i < n; ++i) {
    bool ghost = false;
    for (int p = h[i]; p < h[i + 1]; ++p) ghost |= hc[p] >= n;
    lst[ghost ? 1 : 0].push_back((int)i);
  }
  if (lst[1].empty()) return 0;  // no halo: the plain product
  const size_t esz = m.cplx ? 16 : 8;
  for (int q = 0; q < 2; ++q) {
    Mat::Sorted& so = q ? (adj ? m.bndH : m.bnd) : (adj ? m.innerH : m.inner);
    long long& cnt = q ? (adj ? m.n_bndH : m.n_bnd) : (adj ? m.n_innerH : m.n_inner);
    const std::vector<int>& L = lst[q];
    cnt = (long long)L.size();
    std::vector<int> rp2(L.size() + 1);
    rp2[0] = 0;
    for (size_t l = 0; l < L.size(); ++l) rp2[l + 1] = rp2[l] + (h[L[l] + 1] - h[L[l]]);
    const long long nz = rp2.back();
    if (cudaMalloc(&so.rp, sizeof(int) * (L.size() + 1)) != cudaSuccess ||
        cudaMalloc(&so.perm, sizeof(int) * std::max<size_t>(1, L.size())) != cudaSuccess ||
        cudaMalloc(&so.ci, sizeof(int) * (nz + 1)) != cudaSuccess || cudaMalloc(&so.val, esz * (nz + 1)) != cudaSuccess)
      return (int)cudaErrorMemoryAllocation;
    cudaMemcpyAsync(so.rp, rp2.data(), sizeof(int) * (L.size() + 1), cudaMemcpyHostToDevice, st);
    if (!L.empty()) cudaMemcpyAsync(so.perm, L.data(), sizeof(int) * L.size(), cudaMemcpyHostToDevice, st);
    const int grid = (int)std::max<long long>(1, std::min<long long>(((long long)L.size() + 7) / 8, 148 * 16));
    if (!L.empty()) {
      if (m.cplx)
        gather_sorted_rows<double2><<<grid, 256, 0, st>>>(rp, ci, reinterpret_cast<const double2*>(val), so.perm, so.rp,
                                                          so.ci, reinterpret_cast<double2*>(so.val), (long long)L.size());
      else
        gather_sorted_rows<double><<<grid, 256, 0, st>>>(rp, ci, reinterpret_cast<const double*>(val), so.perm, so.rp,
                                                         so.ci, reinterpret_cast<double*>(so.val), (long long)L.size());
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return (int)cudaErrorUnknown;
  }
  return 0;
}

}  // namespace srk
