// coef.cu — single-CTA coefficient phases for the 13 methods.
// Each phase follows oracle/solvers.py's order of operations and breakdown
// rules line by line (readings G11, G12, G13, G26 in DESIGN.md).
#include <algorithm>

#include "coef.cuh"

namespace srk {

template <typename T>
__device__ __forceinline__ T* W(const CoefArgs& a, int slot) {
  return reinterpret_cast<T*>(a.ws + a.off[slot]);
}
__device__ __forceinline__ double* D(const CoefArgs& a, int slot) { return a.ws + a.off[slot]; }

#define T0 if (threadIdx.x == 0)
#define SYNC __syncthreads()

__device__ void set_brk(const CoefArgs& a, int kind) {
  if (a.ctl[CTL_FLAG] == FLAG_RUN) {
    a.ctl[CTL_FLAG] = FLAG_BRK;
    a.ctl[CTL_BKIND] = kind;
    // a breakdown in the start-up phases (||R0||, the initial thin QRs and coefficients:
    // phases 0, 9-13) happens before iteration 1: reported as iteration 0, as the oracle does
    const bool init = a.phase == 0 || (a.phase >= 9 && a.phase <= 13) || (a.phase >= 20 && (a.k1 & 4));
    a.ctl[CTL_BITER] = a.ctl[CTL_ITER] + (init ? 0 : 1);
  }
}

// Stopping rule: relative recursive residual of iteration ctl[ITER]+1.
__device__ void conv_check(const CoefArgs& a, double r2) {
  T0 {
    const double r0 = *D(a, SL_R0N);
    const double rel = r0 > 0 ? sqrt(r2) / r0 : 0.0;
    const int it = a.ctl[CTL_ITER];
    if (it < a.hist_cap) a.hist[it] = rel;
    if (!isfinite(rel)) set_brk(a, BK_NONFINITE);
    else if (rel <= a.tol) a.ctl[CTL_CONVPEND] = 1;
  }
  SYNC;
}

// scalar q = num / den with breakdown on a zero / non-finite operand
template <typename T>
__device__ bool sdiv(const CoefArgs& a, T num, T den, T* out, int kind) {
  if (is_zero(den) || !fin(num) || !fin(den)) { set_brk(a, kind); return false; }
  T q = cdiv(num, den);
  if (!fin(q)) { set_brk(a, kind); return false; }
  *out = q;
  return true;
}

// Li per-column division with the freeze policy (reading G13)
template <typename T>
__device__ T ldiv(const CoefArgs& a, int c, T num, T den) {
  int* fr = a.ctl + CTL_FROZEN;
  if (fr[c]) return Ar<T>::zero();
  if (is_zero(den)) { fr[c] = 1; return Ar<T>::zero(); }
  T q = cdiv(num, den);
  if (!fin(q)) { fr[c] = 1; return Ar<T>::zero(); }
  return q;
}

__device__ void li_all_frozen(const CoefArgs& a) {
  int n = 0;
  for (int c = 0; c < a.s; ++c) n += a.ctl[CTL_FROZEN + c] ? 1 : 0;
  a.ctl[CTL_NFROZEN] = n;
  if (n == a.s) set_brk(a, BK_LANCZOS);
}

__device__ void common_init(const CoefArgs& a) {
  T0 {
    const double r0 = sqrt(*D(a, SL_R0N2));
    *D(a, SL_R0N) = r0;
    for (int c = 0; c < 64; ++c) a.ctl[CTL_FROZEN + c] = 0;
    a.ctl[CTL_NFROZEN] = 0;
    if (r0 == 0.0) a.ctl[CTL_FLAG] = FLAG_CONV;  // B - A X0 = 0: nothing to do
  }
  SYNC;
}

// ---------------------------------------------------------------- BiCG family
// Gl-BiCG (Alg. 2) and eGl-BiCG (Alg. 4): scalar alpha, beta.
template <typename T>
__device__ void gl_bicg(const CoefArgs& a) {
  T0 {
    if (a.phase == 1) {  // alpha = rho / den
      T al;
      if (sdiv<T>(a, *W<T>(a, SL_RHO), *W<T>(a, SL_DEN), &al, BK_LANCZOS)) *W<T>(a, SL_ALPHA) = al;
    } else if (a.phase == 2) {  // beta = rho_new / rho ; rho = rho_new
      T be;
      if (sdiv<T>(a, *W<T>(a, SL_RHON), *W<T>(a, SL_RHO), &be, BK_LANCZOS)) {
        *W<T>(a, SL_BETA) = be;
        *W<T>(a, SL_RHO) = *W<T>(a, SL_RHON);
      }
    }
  }
  SYNC;
  if (a.phase == 2) conv_check(a, *D(a, SL_R2));
}

// Li-BiCG (Alg. 1): per-column alpha_i, beta_i
template <typename T>
__device__ void li_bicg(const CoefArgs& a) {
  T0 {
    T* rho = W<T>(a, SL_RHO);
    if (a.phase == 1) {
      for (int c = 0; c < a.s; ++c) W<T>(a, SL_ALPHA)[c] = ldiv<T>(a, c, rho[c], W<T>(a, SL_DEN)[c]);
    } else if (a.phase == 2) {
      for (int c = 0; c < a.s; ++c) {
        W<T>(a, SL_BETA)[c] = ldiv<T>(a, c, W<T>(a, SL_RHON)[c], rho[c]);
        rho[c] = W<T>(a, SL_RHON)[c];
      }
      li_all_frozen(a);
    }
  }
  SYNC;
  if (a.phase == 2) conv_check(a, *D(a, SL_R2));
}

// Bl-BiCG (Alg. 3) with the adjoint reuse of Prop. 1's proof
template <typename T>
__device__ void bl_bicg(const CoefArgs& a, T* sh) {
  const int s = a.s;
  if (a.phase == 1) {  // alpha = G^-1 M, alpha_hat = G^-H M^H
    if (sm_solve<T>(W<T>(a, SL_ALPHA), W<T>(a, SL_G), W<T>(a, SL_M), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_copy<T>(W<T>(a, SL_TMP0), W<T>(a, SL_M), s, s, 1);
    if (sm_solve<T>(W<T>(a, SL_AH), W<T>(a, SL_G), W<T>(a, SL_TMP0), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
  } else if (a.phase == 2) {  // beta = M^-1 M+, beta_hat = M^-H M+^H, M = M+
    if (sm_solve<T>(W<T>(a, SL_BETA), W<T>(a, SL_M), W<T>(a, SL_MN), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_copy<T>(W<T>(a, SL_TMP0), W<T>(a, SL_MN), s, s, 1);
    if (sm_solve<T>(W<T>(a, SL_BH), W<T>(a, SL_M), W<T>(a, SL_TMP0), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_copy<T>(W<T>(a, SL_M), W<T>(a, SL_MN), s, s, 0);
    conv_check(a, *D(a, SL_R2));
  }
}

// CholQR2 helper phases (reading G10): pass 1 R1 = chol(G) (rank test), pass 2 R2.
template <typename T>
__device__ bool cholqr_pass(const CoefArgs& a, int gslot, int rslot, int rislot, int rank_check) {
  if (sm_chol<T>(W<T>(a, rslot), W<T>(a, gslot), a.s, rank_check, a.eps_chol)) { T0 set_brk(a, BK_RANK); SYNC; return false; }
  sm_trinv<T>(W<T>(a, rislot), W<T>(a, rslot), a.s);
  return true;
}

// Sig = R2 R1 ; Cslot = Sig * Cslot (optional)
template <typename T>
__device__ void cholqr_sigma(const CoefArgs& a, int r2, int r1, int sig, int cslot) {
  const int s = a.s;
  sm_gemm<T>(W<T>(a, sig), W<T>(a, r2), W<T>(a, r1), s, s, s, 0, 0, one<T>());
  if (cslot >= 0) {
    sm_gemm<T>(W<T>(a, SL_TMP0), W<T>(a, sig), W<T>(a, cslot), s, s, s, 0, 0, one<T>());
    sm_copy<T>(W<T>(a, cslot), W<T>(a, SL_TMP0), s, s, 0);
  }
}

// Pass 1 of an rQ thin QR under rank_policy 1: the masked Cholesky finds every deficient
// column; if there is one, the mask goes to the control block and CTL_DIDLE drops to 0,
// which arms the repair kernels that follow (fill, Gram, phase 20, ..., phase 21).
template <typename T>
__device__ bool cholqr_pass1_cont(const CoefArgs& a, int gslot, int rslot, int rislot, int maskctl) {
  const unsigned long long m = sm_chol_mask<T>(W<T>(a, rslot), W<T>(a, gslot), a.s, a.eps_chol);
  if (m == ~0ull) { T0 set_brk(a, BK_RANK); SYNC; return false; }
  if (m) {
    T0 {
      a.ctl[maskctl] = (int)(unsigned)(m & 0xffffffffull);
      a.ctl[maskctl + 1] = (int)(unsigned)(m >> 32);
      a.ctl[CTL_DIDLE] = 0;
    }
    SYNC;
    return true;
  }
  sm_trinv<T>(W<T>(a, rislot), W<T>(a, rslot), a.s);
  return true;
}

// Bl-BiCG-rQ (Alg. 5, Eqs. (4)-(7))
template <typename T>
__device__ void bl_bicg_rq(const CoefArgs& a, T* sh) {
  const int s = a.s;
  if (a.phase == 0) {  // after the initial QRs: ||C0||
    double c2 = sm_fro2<T>(W<T>(a, SL_C), s * s, reinterpret_cast<double*>(sh));
    T0 *D(a, SL_C0N) = sqrt(c2);
    SYNC;
  } else if (a.phase == 1) {  // alpha = G1^-1 G2, alpha_hat = G1^-H G2^H, AC = alpha C
    if (sm_solve<T>(W<T>(a, SL_ALPHA), W<T>(a, SL_G1), W<T>(a, SL_G2), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_copy<T>(W<T>(a, SL_TMP0), W<T>(a, SL_G2), s, s, 1);
    if (sm_solve<T>(W<T>(a, SL_AH), W<T>(a, SL_G1), W<T>(a, SL_TMP0), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_gemm<T>(W<T>(a, SL_AC), W<T>(a, SL_ALPHA), W<T>(a, SL_C), s, s, s, 0, 0, one<T>());
  } else if (a.phase == 2) {  // CholQR pass 1 of Z and Z_hat
    if (a.defl) {
      if (!cholqr_pass1_cont<T>(a, SL_GZ, SL_R1, SL_R1I, CTL_DMASK)) return;
      cholqr_pass1_cont<T>(a, SL_GZH, SL_R1H, SL_R1HI, CTL_DMASKH);
      return;
    }
    if (!cholqr_pass<T>(a, SL_GZ, SL_R1, SL_R1I, 1)) return;
    if (!cholqr_pass<T>(a, SL_GZH, SL_R1H, SL_R1HI, 1)) return;
  } else if (a.phase == 3) {  // pass 2, Sig = R2 R1, C = Sig C
    if (!cholqr_pass<T>(a, SL_GZ, SL_R2F, SL_R2I, 0)) return;
    if (!cholqr_pass<T>(a, SL_GZH, SL_R2H, SL_R2HI, 0)) return;
    cholqr_sigma<T>(a, SL_R2F, SL_R1, SL_SIG, SL_C);
    cholqr_sigma<T>(a, SL_R2H, SL_R1H, SL_SIGH, SL_CH);
  } else if (a.phase == 4) {  // beta = G2^-1 Sig_h^H G2+, beta_hat = G2^-H Sig^H G2+^H (Eqs. 6-7)
    sm_gemm<T>(W<T>(a, SL_TMP1), W<T>(a, SL_SIGH), W<T>(a, SL_G2N), s, s, s, 1, 0, one<T>());
    if (sm_solve<T>(W<T>(a, SL_BETA), W<T>(a, SL_G2), W<T>(a, SL_TMP1), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_gemm<T>(W<T>(a, SL_TMP1), W<T>(a, SL_SIG), W<T>(a, SL_G2N), s, s, s, 1, 1, one<T>());
    if (sm_solve<T>(W<T>(a, SL_BH), W<T>(a, SL_G2), W<T>(a, SL_TMP1), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_copy<T>(W<T>(a, SL_G2), W<T>(a, SL_G2N), s, s, 0);
    double c2 = sm_fro2<T>(W<T>(a, SL_C), s * s, reinterpret_cast<double*>(sh));
    conv_check(a, c2);
  }
}

// ------------------------------------------------------------ BiCGStab family
__device__ void half_check(const CoefArgs& a, double s2, double ref) {
  T0 {
    const double r = sqrt(fmax(s2, 0.0));
    const double r0 = *D(a, SL_R0N);
    if (ref > 0 && r <= a.tol * ref) {
      const int it = a.ctl[CTL_ITER];
      if (it < a.hist_cap) a.hist[it] = r0 > 0 ? r / r0 : 0.0;
      a.ctl[CTL_FLAG] = FLAG_HALF;
    }
  }
  SYNC;
}

// Gl-BiCGStab [Jbilou05]
template <typename T>
__device__ void gl_bicgstab(const CoefArgs& a) {
  if (a.phase == 1) {
    T0 {
      T al;
      if (sdiv<T>(a, *W<T>(a, SL_RHO), *W<T>(a, SL_DEN), &al, BK_LANCZOS)) *W<T>(a, SL_ALPHA) = al;
    }
    SYNC;
  } else if (a.phase == 2) {
    half_check(a, *D(a, SL_S2), *D(a, SL_R0N));
  } else if (a.phase == 3) {  // omega = tr(T^H S) / tr(T^H T); SL_ST holds tr(S^H T)
    T0 {
      T om;
      const T num = Ar<T>::conj(*W<T>(a, SL_ST));
      const T den = mkT(*D(a, SL_TT), 0.0, T());
      if (sdiv<T>(a, num, den, &om, BK_OMEGA)) *W<T>(a, SL_OMEGA) = om;
    }
    SYNC;
  } else if (a.phase == 4) {  // beta = (rho+ alpha)/(rho omega); BW = beta omega
    T0 {
      T be;
      const T num = Ar<T>::mul(*W<T>(a, SL_RHON), *W<T>(a, SL_ALPHA));
      const T den = Ar<T>::mul(*W<T>(a, SL_RHO), *W<T>(a, SL_OMEGA));
      if (sdiv<T>(a, num, den, &be, BK_LANCZOS)) {
        *W<T>(a, SL_BETA) = be;
        *W<T>(a, SL_BW) = Ar<T>::mul(be, *W<T>(a, SL_OMEGA));
        *W<T>(a, SL_RHO) = *W<T>(a, SL_RHON);
      }
    }
    SYNC;
    conv_check(a, *D(a, SL_R2));
  }
}

// Li-BiCGStab: per column
template <typename T>
__device__ void li_bicgstab(const CoefArgs& a) {
  const int s = a.s;
  if (a.phase == 2) { half_check(a, *D(a, SL_S2), *D(a, SL_R0N)); return; }
  T0 {
    if (a.phase == 1) {
      for (int c = 0; c < s; ++c) W<T>(a, SL_ALPHA)[c] = ldiv<T>(a, c, W<T>(a, SL_RHO)[c], W<T>(a, SL_DEN)[c]);
    } else if (a.phase == 3) {  // omega_i = (t_i^H s_i) / (t_i^H t_i); SL_ST holds s_i^H t_i
      for (int c = 0; c < s; ++c)
        W<T>(a, SL_OMEGA)[c] = ldiv<T>(a, c, Ar<T>::conj(W<T>(a, SL_ST)[c]), mkT(D(a, SL_TT)[c], 0.0, T()));
    } else if (a.phase == 4) {
      for (int c = 0; c < s; ++c) {
        const T num = Ar<T>::mul(W<T>(a, SL_RHON)[c], W<T>(a, SL_ALPHA)[c]);
        const T den = Ar<T>::mul(W<T>(a, SL_RHO)[c], W<T>(a, SL_OMEGA)[c]);
        const T be = ldiv<T>(a, c, num, den);
        W<T>(a, SL_BETA)[c] = be;
        W<T>(a, SL_BW)[c] = Ar<T>::mul(be, W<T>(a, SL_OMEGA)[c]);
        W<T>(a, SL_RHO)[c] = W<T>(a, SL_RHON)[c];
      }
      li_all_frozen(a);
    }
  }
  SYNC;
  if (a.phase == 4) conv_check(a, *D(a, SL_R2));
}

// Bl-BiCGStab [ELg03] (reading G14)
template <typename T>
__device__ void bl_bicgstab(const CoefArgs& a, T* sh) {
  const int s = a.s;
  if (a.phase == 1) {  // alpha = G^-1 (Rt^H R)
    if (sm_solve<T>(W<T>(a, SL_ALPHA), W<T>(a, SL_G), W<T>(a, SL_M), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; }
  } else if (a.phase == 2) {
    half_check(a, *D(a, SL_S2), *D(a, SL_R0N));
  } else if (a.phase == 3) {
    T0 {
      T om;
      if (sdiv<T>(a, Ar<T>::conj(*W<T>(a, SL_ST)), mkT(*D(a, SL_TT), 0.0, T()), &om, BK_OMEGA)) *W<T>(a, SL_OMEGA) = om;
    }
    SYNC;
  } else if (a.phase == 4) {  // beta = -G^-1 (Rt^H T); BW = omega beta
    if (sm_solve<T>(W<T>(a, SL_TMP1), W<T>(a, SL_G), W<T>(a, SL_MN), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_scale<T>(W<T>(a, SL_BETA), W<T>(a, SL_TMP1), s * s, mkT(-1.0, 0.0, T()));
    sm_scale<T>(W<T>(a, SL_BW), W<T>(a, SL_BETA), s * s, *W<T>(a, SL_OMEGA));
    conv_check(a, *D(a, SL_R2));
  }
}

// Bl-BiCGStab-rQ (reading G16)
template <typename T>
__device__ void bl_bicgstab_rq(const CoefArgs& a, T* sh) {
  const int s = a.s;
  double* dsh = reinterpret_cast<double*>(sh);
  if (a.phase == 0) {
    double c2 = sm_fro2<T>(W<T>(a, SL_C), s * s, dsh);
    T0 *D(a, SL_C0N) = sqrt(c2);
    SYNC;
  } else if (a.phase == 1) {  // alpha = G^-1 GQ ; AC = alpha C
    if (sm_solve<T>(W<T>(a, SL_ALPHA), W<T>(a, SL_G), W<T>(a, SL_GQ), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_gemm<T>(W<T>(a, SL_AC), W<T>(a, SL_ALPHA), W<T>(a, SL_C), s, s, s, 0, 0, one<T>());
  } else if (a.phase == 2) {  // ||S||^2 = tr(C^H (Z^H Z) C)
    sm_gemm<T>(W<T>(a, SL_TMP0), W<T>(a, SL_ZZ), W<T>(a, SL_C), s, s, s, 0, 0, one<T>());
    sm_gemm<T>(W<T>(a, SL_TMP1), W<T>(a, SL_C), W<T>(a, SL_TMP0), s, s, s, 1, 0, one<T>());
    T0 {
      double tr = 0.0;
      for (int i = 0; i < s; ++i) tr += re(W<T>(a, SL_TMP1)[i * s + i]);
      dsh[0] = tr;
    }
    SYNC;
    half_check(a, dsh[0], *D(a, SL_C0N));
  } else if (a.phase == 3) {  // M = C C^H ; omega = tr((Y^H Z) M) / tr((Y^H Y) M); WC = omega C
    sm_gemm<T>(W<T>(a, SL_TMP0), W<T>(a, SL_C), W<T>(a, SL_C), s, s, s, 0, 1, one<T>());     // M
    sm_copy<T>(W<T>(a, SL_TMP3), W<T>(a, SL_YZ), s, s, 1);                                    // Y^H Z = (Z^H Y)^H
    sm_gemm<T>(W<T>(a, SL_TMP1), W<T>(a, SL_TMP3), W<T>(a, SL_TMP0), s, s, s, 0, 0, one<T>());
    sm_gemm<T>(W<T>(a, SL_TMP2), W<T>(a, SL_YY), W<T>(a, SL_TMP0), s, s, s, 0, 0, one<T>());
    T0 {
      T num = Ar<T>::zero(), den = Ar<T>::zero();
      for (int i = 0; i < s; ++i) {
        num = Ar<T>::add(num, W<T>(a, SL_TMP1)[i * s + i]);
        den = Ar<T>::add(den, W<T>(a, SL_TMP2)[i * s + i]);
      }
      T om;
      if (sdiv<T>(a, num, den, &om, BK_OMEGA)) *W<T>(a, SL_OMEGA) = om;
    }
    SYNC;
    if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
    sm_scale<T>(W<T>(a, SL_WC), W<T>(a, SL_C), s * s, *W<T>(a, SL_OMEGA));
  } else if (a.phase == 4) {
    if (a.defl) cholqr_pass1_cont<T>(a, SL_GZ, SL_R1, SL_R1I, CTL_DMASK);
    else cholqr_pass<T>(a, SL_GZ, SL_R1, SL_R1I, 1);
  } else if (a.phase == 5) {
    if (!cholqr_pass<T>(a, SL_GZ, SL_R2F, SL_R2I, 0)) return;
    cholqr_sigma<T>(a, SL_R2F, SL_R1, SL_SIG, SL_C);
  } else if (a.phase == 6) {  // beta = omega^-1 G^-1 GQ+ ; BW = omega beta ; GQ = GQ+
    if (sm_solve<T>(W<T>(a, SL_TMP1), W<T>(a, SL_G), W<T>(a, SL_GQN), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    const T om = *W<T>(a, SL_OMEGA);
    for (int i = threadIdx.x; i < s * s; i += blockDim.x) {
      const T b = cdiv(W<T>(a, SL_TMP1)[i], om);
      W<T>(a, SL_BETA)[i] = b;
      W<T>(a, SL_BW)[i] = Ar<T>::mul(om, b);
    }
    SYNC;
    sm_copy<T>(W<T>(a, SL_GQ), W<T>(a, SL_GQN), s, s, 0);
    double c2 = sm_fro2<T>(W<T>(a, SL_C), s * s, dsh);
    conv_check(a, c2);
  }
}

// ------------------------------------------------------------------ QMR family
// Li / Gl / eGl-QMR (readings G17, G18). mode 0 = Li (per
// column), 1 = Gl, 2 = eGl. rho, xi, gam, theta are real; eta complex.
template <typename T>
__device__ void qmr_scalar(const CoefArgs& a, int mode) {
  const int s = a.s;
  const int ncol = (mode == 0) ? s : 1;
  T0 {
    T* rho = W<T>(a, SL_QRHO);
    T* xi = W<T>(a, SL_QXI);
    if (a.phase == 0) {  // rho = ||Vt||, xi = ||Wt|| (eGl: sqrt(s) ||w||)
      for (int c = 0; c < ncol; ++c) {
        rho[c] = mkT(sqrt(D(a, SL_RHON2)[c]), 0.0, T());
        const double x = sqrt(D(a, SL_XI2)[c]);
        xi[c] = mkT(mode == 2 ? sqrt((double)s) * x : x, 0.0, T());
        W<T>(a, SL_GAMP)[c] = one<T>();
        W<T>(a, SL_ETA)[c] = mkT(-1.0, 0.0, T());
        W<T>(a, SL_THETAP)[c] = Ar<T>::zero();
      }
    } else if (a.phase == 1) {  // 1/rho, 1/xi
      for (int c = 0; c < ncol; ++c) {
        if (mode == 0) {
          W<T>(a, SL_INVRHO)[c] = ldiv<T>(a, c, one<T>(), rho[c]);
          W<T>(a, SL_INVXI)[c] = ldiv<T>(a, c, one<T>(), xi[c]);
        } else {
          T q;
          if (!sdiv<T>(a, one<T>(), rho[c], &q, BK_LANCZOS)) break;
          W<T>(a, SL_INVRHO)[c] = q;
          if (!sdiv<T>(a, one<T>(), xi[c], &q, BK_LANCZOS)) break;
          W<T>(a, SL_INVXI)[c] = q;
        }
      }
    } else if (a.phase == 2) {  // delta = <Ṽ, W̃>/(rho xi); P = V - (xi delta/eps) P ; Q = W - conj(rho delta/eps) Q
      for (int c = 0; c < ncol; ++c) {
        const T d = Ar<T>::mul(Ar<T>::mul(W<T>(a, SL_K1)[c], W<T>(a, SL_INVRHO)[c]), W<T>(a, SL_INVXI)[c]);
        W<T>(a, SL_DELTA)[c] = d;
        if (a.k1) {
          W<T>(a, SL_C1)[c] = Ar<T>::zero();
          W<T>(a, SL_C2)[c] = Ar<T>::zero();
          continue;
        }
        const T e = W<T>(a, SL_EPS)[c];
        const T n1 = Ar<T>::mul(xi[c], d), n2 = Ar<T>::mul(rho[c], d);
        if (mode == 0) {
          W<T>(a, SL_C1)[c] = ldiv<T>(a, c, n1, e);
          W<T>(a, SL_C2)[c] = Ar<T>::conj(ldiv<T>(a, c, n2, e));
        } else {
          T q1, q2;
          if (!sdiv<T>(a, n1, e, &q1, BK_LANCZOS)) break;
          if (!sdiv<T>(a, n2, e, &q2, BK_LANCZOS)) break;
          W<T>(a, SL_C1)[c] = q1;
          W<T>(a, SL_C2)[c] = Ar<T>::conj(q2);
        }
      }
    } else if (a.phase == 3) {  // beta = eps / delta ; BR = beta/rho ; BX = conj(beta)/xi
      for (int c = 0; c < ncol; ++c) {
        T be;
        if (mode == 0) {
          be = ldiv<T>(a, c, W<T>(a, SL_EPS)[c], W<T>(a, SL_DELTA)[c]);
        } else {
          if (!sdiv<T>(a, W<T>(a, SL_EPS)[c], W<T>(a, SL_DELTA)[c], &be, BK_LANCZOS)) break;
        }
        W<T>(a, SL_BETA)[c] = be;
        W<T>(a, SL_BR)[c] = Ar<T>::mul(be, W<T>(a, SL_INVRHO)[c]);
        W<T>(a, SL_BX)[c] = Ar<T>::mul(Ar<T>::conj(be), W<T>(a, SL_INVXI)[c]);
      }
    } else if (a.phase == 4) {  // theta, gamma, eta; f = (theta_prev gamma)^2
      for (int c = 0; c < ncol; ++c) {
        const double rn = sqrt(D(a, SL_RHON2)[c]);
        const double xin = sqrt(D(a, SL_XI2)[c]);
        const T be = W<T>(a, SL_BETA)[c];
        const double gp = re(W<T>(a, SL_GAMP)[c]);
        const double thp = re(W<T>(a, SL_THETAP)[c]);
        double th = rn / (gp * cabs(be));
        double ga = 1.0 / sqrt(1.0 + th * th);
        // eta = -eta * rho * gam^2 / (beta * gam_prev^2)
        T eta = W<T>(a, SL_ETA)[c];
        T num = scal(eta, -re(rho[c]) * ga * ga);
        T den = scal(be, gp * gp);
        eta = cdiv(num, den);
        if (mode == 0 && a.ctl[CTL_FROZEN + c]) { th = 0.0; ga = 1.0; eta = Ar<T>::zero(); }
        if (mode != 0 && (ga == 0.0 || !fin(eta))) { set_brk(a, BK_LANCZOS); break; }
        const double f = (thp * ga) * (thp * ga);
        W<T>(a, SL_ETA)[c] = eta;
        W<T>(a, SL_F)[c] = mkT(f, 0.0, T());
        rho[c] = mkT(rn, 0.0, T());
        xi[c] = mkT(mode == 2 ? sqrt((double)s) * xin : xin, 0.0, T());
        W<T>(a, SL_GAMP)[c] = mkT(ga, 0.0, T());
        W<T>(a, SL_THETAP)[c] = mkT(th, 0.0, T());
        if (mode != 0) {
          // next iteration's 1/rho and c1 = xi delta/eps for the fused tail (QMR::seg): the arithmetic
          // of phases 1-2 on the values they will see (rho, xi just set; K1 and eps of this iteration),
          // without their breakdown tests — those phases still run and raise the flag before anything
          // reads a P built from a non-finite coefficient
          const T ir = cdiv(one<T>(), rho[c]), ix = cdiv(one<T>(), xi[c]);
          const T dn = Ar<T>::mul(Ar<T>::mul(W<T>(a, SL_K1)[c], ir), ix);
          W<T>(a, SL_INVRHO_N)[c] = ir;
          W<T>(a, SL_C1_N)[c] = cdiv(Ar<T>::mul(xi[c], dn), W<T>(a, SL_EPS)[c]);
          W<T>(a, SL_INVXI_N)[c] = ix;
          W<T>(a, SL_C2_N)[c] = Ar<T>::conj(cdiv(Ar<T>::mul(rho[c], dn), W<T>(a, SL_EPS)[c]));
        }
      }
    } else if (a.phase == 5) {
      if (mode == 0) li_all_frozen(a);
    }
  }
  SYNC;
  if (a.phase == 5) conv_check(a, *D(a, SL_R2));
}

// Block QMR (reading G19)
template <typename T>
__device__ void bl_qmr(const CoefArgs& a, T* sh) {
  const int s = a.s, s2 = 2 * s;
  double* dsh = reinterpret_cast<double*>(sh);
  (void)dsh;
  if (a.phase == 0) {  // tau_t = rho ; Omega_prev = I (unused at k = 1)
    sm_copy<T>(W<T>(a, SL_TAUT), W<T>(a, SL_RHOB), s, s, 0);
  } else if (a.phase == 1) {  // c1 = eps^-1 xi^H delta ; c2 = eps^-H rho^H delta^H (k > 1)
    if (a.k1) {
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) {
        W<T>(a, SL_C1)[i] = Ar<T>::zero();
        W<T>(a, SL_C2)[i] = Ar<T>::zero();
      }
      SYNC;
      return;
    }
    sm_gemm<T>(W<T>(a, SL_TMP0), W<T>(a, SL_XIB), W<T>(a, SL_DELTA), s, s, s, 1, 0, one<T>());
    if (sm_solve<T>(W<T>(a, SL_C1), W<T>(a, SL_EPS), W<T>(a, SL_TMP0), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_gemm<T>(W<T>(a, SL_TMP0), W<T>(a, SL_RHOB), W<T>(a, SL_DELTA), s, s, s, 1, 1, one<T>());
    if (sm_solve<T>(W<T>(a, SL_C2), W<T>(a, SL_EPS), W<T>(a, SL_TMP0), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
  } else if (a.phase == 2) {  // beta = delta^-1 eps ; gamma_hat = delta^-H eps^H
    if (sm_solve<T>(W<T>(a, SL_BETA), W<T>(a, SL_DELTA), W<T>(a, SL_EPS), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_copy<T>(W<T>(a, SL_TMP0), W<T>(a, SL_EPS), s, s, 1);
    if (sm_solve<T>(W<T>(a, SL_GHAT), W<T>(a, SL_DELTA), W<T>(a, SL_TMP0), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
  } else if (a.phase == 3) {  // CholQR pass 1 of V~ and W~ (rank deficiency of V~ with V~ == 0 -> rho+ = 0, deferred)
    T0 *D(a, SL_PEND) = 0.0;
    SYNC;
    if (sm_chol<T>(W<T>(a, SL_R1), W<T>(a, SL_GZ), s, 1, a.eps_chol)) {
      double g2 = sm_fro2<T>(W<T>(a, SL_GZ), s * s, dsh);
      if (g2 != 0.0) { T0 set_brk(a, BK_RANK); SYNC; return; }
      T0 *D(a, SL_PEND) = 1.0;  // exactly zero block: rho+ = 0, breakdown deferred past the X update
      SYNC;
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) { W<T>(a, SL_R1)[i] = Ar<T>::zero(); W<T>(a, SL_R1I)[i] = Ar<T>::zero(); }
      SYNC;
    } else {
      sm_trinv<T>(W<T>(a, SL_R1I), W<T>(a, SL_R1), s);
    }
    if (sm_chol<T>(W<T>(a, SL_R1H), W<T>(a, SL_GZH), s, 1, a.eps_chol)) {
      double g2 = sm_fro2<T>(W<T>(a, SL_GZH), s * s, dsh);
      if (g2 != 0.0) { T0 set_brk(a, BK_RANK); SYNC; return; }
      T0 *D(a, SL_PEND) = 1.0;
      SYNC;
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) { W<T>(a, SL_R1H)[i] = Ar<T>::zero(); W<T>(a, SL_R1HI)[i] = Ar<T>::zero(); }
      SYNC;
    } else {
      sm_trinv<T>(W<T>(a, SL_R1HI), W<T>(a, SL_R1H), s);
    }
  } else if (a.phase == 4) {  // pass 2 -> rho+ = R2 R1, xi+ ; quasi-minimisation update
    const bool pend = *D(a, SL_PEND) != 0.0;
    if (!pend) {
      if (!cholqr_pass<T>(a, SL_GZ, SL_R2F, SL_R2I, 0)) return;
      cholqr_sigma<T>(a, SL_R2F, SL_R1, SL_RHOBN, -1);
      if (!cholqr_pass<T>(a, SL_GZH, SL_R2H, SL_R2HI, 0)) return;
      cholqr_sigma<T>(a, SL_R2H, SL_R1H, SL_XIBN, -1);
    } else {
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) {
        W<T>(a, SL_RHOBN)[i] = Ar<T>::zero();
        W<T>(a, SL_R2I)[i] = Ar<T>::zero();
        W<T>(a, SL_R2HI)[i] = Ar<T>::zero();
        W<T>(a, SL_XIBN)[i] = Ar<T>::zero();
      }
      SYNC;
    }
    // [top; c] = Omega_prev^H [0; beta]  (k = 1: top = 0, c = beta)
    T* top = W<T>(a, SL_TOP);
    T* stack = W<T>(a, SL_TMP1);  // 2s x s: [c; rho+]
    if (a.k1) {
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) { top[i] = Ar<T>::zero(); stack[i] = W<T>(a, SL_BETA)[i]; }
    } else {
      const T* Om = W<T>(a, SL_OMP);
      for (int idx = threadIdx.x; idx < s2 * s; idx += blockDim.x) {
        const int i = idx / s, j = idx % s;
        T acc = Ar<T>::zero();
        for (int l = 0; l < s; ++l) acc = Ar<T>::cfma(Om[(s + l) * s2 + i], W<T>(a, SL_BETA)[l * s + j], acc);
        if (i < s) top[i * s + j] = acc; else stack[(i - s) * s + j] = acc;
      }
    }
    SYNC;
    for (int i = threadIdx.x; i < s * s; i += blockDim.x) stack[s * s + i] = W<T>(a, SL_RHOBN)[i];
    SYNC;
    // [c; rho+] = Omega [Rii; 0]
    sm_qr_stack<T>(W<T>(a, SL_OMP), W<T>(a, SL_RII), stack, s, W<T>(a, SL_TMP2));
    // [tau; tau_t] = Omega^H [tau_t; 0]
    {
      const T* Om = W<T>(a, SL_OMP);
      T* tnew = W<T>(a, SL_TMP3);
      for (int idx = threadIdx.x; idx < s2 * s; idx += blockDim.x) {
        const int i = idx / s, j = idx % s;
        T acc = Ar<T>::zero();
        for (int l = 0; l < s; ++l) acc = Ar<T>::cfma(Om[l * s2 + i], W<T>(a, SL_TAUT)[l * s + j], acc);
        tnew[idx] = acc;
      }
      SYNC;
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) {
        W<T>(a, SL_TAU)[i] = tnew[i];
        W<T>(a, SL_TAUT)[i] = tnew[s * s + i];
      }
      SYNC;
    }
    // Rii^-1 (solve against I, as the oracle) and TR = top Rii^-1
    for (int i = threadIdx.x; i < s * s; i += blockDim.x) W<T>(a, SL_TMP0)[i] = (i / s == i % s) ? one<T>() : Ar<T>::zero();
    SYNC;
    if (sm_solve<T>(W<T>(a, SL_RIII), W<T>(a, SL_RII), W<T>(a, SL_TMP0), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_gemm<T>(W<T>(a, SL_TR), top, W<T>(a, SL_RIII), s, s, s, 0, 0, one<T>());
  } else if (a.phase == 5) {  // after X, R updates: rho, xi = rho+, xi+ ; convergence, deferred breakdown
    sm_copy<T>(W<T>(a, SL_RHOB), W<T>(a, SL_RHOBN), s, s, 0);
    sm_copy<T>(W<T>(a, SL_XIB), W<T>(a, SL_XIBN), s, s, 0);
    conv_check(a, *D(a, SL_R2));
    T0 {
      if (*D(a, SL_PEND) != 0.0 && a.ctl[CTL_CONVPEND] == 0) set_brk(a, BK_RANK);
    }
    SYNC;
  }
}

// ------------------------------------------------- QR of the search directions (f3)
// Bl-BiCG-sQ (oracle bl_bicg_sq, reading R9): P, P̂ orthonormal, so
// alpha = G^-1 (P̂^H R), alpha_hat = G^-H (P^H R̂), beta = -G^-1 (Q̂^H R+),
// beta_hat = -G^-H (Q^H R̂+), G = P̂^H A P; then CholQR2 of R + P beta and R̂ + P̂ beta_hat.
template <typename T>
__device__ void bl_bicg_sq(const CoefArgs& a, T* sh) {
  const int s = a.s;
  if (a.phase == 1) {
    if (sm_solve<T>(W<T>(a, SL_ALPHA), W<T>(a, SL_G), W<T>(a, SL_M), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    if (sm_solve<T>(W<T>(a, SL_AH), W<T>(a, SL_G), W<T>(a, SL_MH), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
  } else if (a.phase == 2) {
    if (sm_solve<T>(W<T>(a, SL_TMP1), W<T>(a, SL_G), W<T>(a, SL_MN), s, s, 0, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_scale<T>(W<T>(a, SL_BETA), W<T>(a, SL_TMP1), s * s, mkT(-1.0, 0.0, T()));
    if (sm_solve<T>(W<T>(a, SL_TMP1), W<T>(a, SL_G), W<T>(a, SL_MNH), s, s, 1, sh, a.eps_brk)) { T0 set_brk(a, BK_GRAM); SYNC; return; }
    sm_scale<T>(W<T>(a, SL_BH), W<T>(a, SL_TMP1), s * s, mkT(-1.0, 0.0, T()));
    conv_check(a, *D(a, SL_R2));
  } else if (a.phase == 3) {  // CholQR pass 1 of the new search directions (rank test)
    if (!cholqr_pass<T>(a, SL_GZ, SL_R1, SL_R1I, 1)) return;
    cholqr_pass<T>(a, SL_GZH, SL_R1H, SL_R1HI, 1);
  } else if (a.phase == 4) {  // pass 2
    if (!cholqr_pass<T>(a, SL_GZ, SL_R2F, SL_R2I, 0)) return;
    cholqr_pass<T>(a, SL_GZH, SL_R2H, SL_R2HI, 0);
  }
}

// Bl-BiCGStab-sQ: App. A.4's phases 1-4, then CholQR2 of the new search direction block
template <typename T>
__device__ void bl_bicgstab_sq(const CoefArgs& a, T* sh) {
  if (a.phase <= 4) bl_bicgstab<T>(a, sh);
  else if (a.phase == 5) cholqr_pass<T>(a, SL_GZ, SL_R1, SL_R1I, 1);
  else if (a.phase == 6) cholqr_pass<T>(a, SL_GZ, SL_R2F, SL_R2I, 0);
}

// --------------------------------------------- rank-deficiency continuation (f4)
// Phase 20 (repair, after the fill kernel replaced the deficient columns and the Gram of
// the modified block was formed): keep C_old, redo pass 1 strictly (a replacement vector
// in the span of the others would be a genuine rank breakdown). k1: bit 0 the residual
// side, bit 1 the shadow side, bit 2 the initial QR (C_old = I).
// Phase 21 (fix-up, after Q of the modified block exists and SIGT = Q^H Z_orig): the true
// factor Sig = triu(SIGT) with the replaced diagonal entries 0 and the others real, and
// C = Sig C_old; then the repair is disarmed.
template <typename T>
__device__ void defl_phase(const CoefArgs& a) {
  if (a.ctl[CTL_DIDLE]) return;
  const int s = a.s;
  const bool init = (a.k1 & 4) != 0;
  for (int side = 0; side < 2; ++side) {
    if (!(a.k1 & (1 << side))) continue;
    const int gz = side ? SL_GZH : SL_GZ, r1 = side ? SL_R1H : SL_R1, r1i = side ? SL_R1HI : SL_R1I;
    const int cs = side ? SL_CH : SL_C, co = side ? SL_COLDH : SL_COLD;
    const int sg = side ? SL_SIGH : SL_SIG, st = side ? SL_SIGTH : SL_SIGT;
    const int mk = side ? CTL_DMASKH : CTL_DMASK;
    if (a.phase == 20) {
      if (init) {
        for (int i = threadIdx.x; i < s * s; i += blockDim.x)
          W<T>(a, co)[i] = (i / s == i % s) ? one<T>() : Ar<T>::zero();
      } else {
        sm_copy<T>(W<T>(a, co), W<T>(a, cs), s, s, 0);
      }
      SYNC;
      if (!cholqr_pass<T>(a, gz, r1, r1i, 1)) return;
    } else {
      const unsigned long long m = (unsigned long long)(unsigned)a.ctl[mk] | ((unsigned long long)(unsigned)a.ctl[mk + 1] << 32);
      for (int i = threadIdx.x; i < s * s; i += blockDim.x) {
        const int r = i / s, c = i % s;
        T v = W<T>(a, st)[i];
        if (r > c || (r == c && ((m >> c) & 1ull))) v = Ar<T>::zero();
        else if (r == c) v = mkT(re(v), 0.0, T());
        W<T>(a, sg)[i] = v;
      }
      SYNC;
      sm_gemm<T>(W<T>(a, cs), W<T>(a, sg), W<T>(a, co), s, s, s, 0, 0, one<T>());
      SYNC;
    }
  }
  if (a.phase == 21) {
    T0 {
      int nrep = 0;
      for (int q = 0; q < 4; ++q) nrep += __popc((unsigned)a.ctl[CTL_DMASK + q]);
      a.ctl[CTL_DEFL] += nrep;
      for (int q = 0; q < 4; ++q) a.ctl[CTL_DMASK + q] = 0;
      a.ctl[CTL_DIDLE] = 1;
    }
    SYNC;
  }
}

// ------------------------------------------------------------------ dispatch
template <typename T>
__global__ void __launch_bounds__(256) coef_kernel(CoefArgs a) {
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  extern __shared__ double smraw[];
  T* sh = reinterpret_cast<T*>(smraw);
  if (a.phase == 9) {  // common start: ||R0||
    common_init(a);
    return;
  }
  if (a.phase >= 10 && a.phase <= 13) {  // device thin QR (CholQR2) of an initial block
    const bool hat = a.phase >= 12;
    const int gz = hat ? SL_GZH : SL_GZ;
    if ((a.phase & 1) == 0) {
      if (a.defl) cholqr_pass1_cont<T>(a, gz, hat ? SL_R1H : SL_R1, hat ? SL_R1HI : SL_R1I, hat ? CTL_DMASKH : CTL_DMASK);
      else cholqr_pass<T>(a, gz, hat ? SL_R1H : SL_R1, hat ? SL_R1HI : SL_R1I, 1);
    } else {
      if (!cholqr_pass<T>(a, gz, hat ? SL_R2H : SL_R2F, hat ? SL_R2HI : SL_R2I, 0)) return;
      cholqr_sigma<T>(a, hat ? SL_R2H : SL_R2F, hat ? SL_R1H : SL_R1, hat ? SL_CH : SL_C, -1);
    }
    return;
  }
  if (a.phase == 20 || a.phase == 21) {  // rank-deficiency continuation (f4)
    defl_phase<T>(a);
    return;
  }
  switch (a.method) {
    case M_BL_BICG_SQ: bl_bicg_sq<T>(a, sh); break;
    case M_BL_BICGSTAB_SQ: bl_bicgstab_sq<T>(a, sh); break;
    case M_GL_BICG:
    case M_EGL_BICG: gl_bicg<T>(a); break;
    case M_LI_BICG: li_bicg<T>(a); break;
    case M_BL_BICG: bl_bicg<T>(a, sh); break;
    case M_BL_BICG_RQ: bl_bicg_rq<T>(a, sh); break;
    case M_GL_BICGSTAB: gl_bicgstab<T>(a); break;
    case M_LI_BICGSTAB: li_bicgstab<T>(a); break;
    case M_BL_BICGSTAB: bl_bicgstab<T>(a, sh); break;
    case M_BL_BICGSTAB_RQ: bl_bicgstab_rq<T>(a, sh); break;
    case M_LI_QMR: qmr_scalar<T>(a, 0); break;
    case M_GL_QMR: qmr_scalar<T>(a, 1); break;
    case M_EGL_QMR: qmr_scalar<T>(a, 2); break;
    case M_BL_QMR: bl_qmr<T>(a, sh); break;
    default: break;
  }
}

// end of one iteration: count it and commit a pending convergence candidate
__global__ void end_iter_kernel(int* ctl) {
  if (ctl[CTL_FLAG] != FLAG_RUN) return;
  ctl[CTL_ITER] += 1;
  if (ctl[CTL_CONVPEND]) {
    ctl[CTL_CONVPEND] = 0;
    ctl[CTL_FLAG] = FLAG_CONV;
  }
}

int launch_coef(bool cplx, const CoefArgs& a, size_t smem, cudaStream_t st) {
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(coef_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(coef_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  if (cplx) coef_kernel<double2><<<1, 256, smem, st>>>(a);
  else coef_kernel<double><<<1, 256, smem, st>>>(a);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ small eGl-BiCG
// fixed-order CTA sum: warp butterflies, then warp 0 adds the warps in index order
template <typename T>
__device__ T cta_sum(T v, T* sh) {
  for (int m = 16; m > 0; m >>= 1) v = Ar<T>::add(v, Ar<T>::shfl_xor(v, m));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();  // sh may still be read by a previous sum
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  T r = Ar<T>::zero();
  for (int q = 0; q < nw; ++q) r = Ar<T>::add(r, sh[q]);
  return r;
}

template <typename T>
__global__ void __launch_bounds__(1024) egl_bicg_small_kernel(SmallBiCGArgs g) {
  CoefArgs a = g.ca;
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  __shared__ T red[32];
  __shared__ double redd[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long n = g.n;
  const int s = a.s;
  const T* val = reinterpret_cast<const T*>(g.val);
  const T* valH = reinterpret_cast<const T*>(g.valH);
  T* X = reinterpret_cast<T*>(g.X);
  T* R = reinterpret_cast<T*>(g.R);
  T* P = reinterpret_cast<T*>(g.P);
  T* Q = reinterpret_cast<T*>(g.Q);
  T* rh = reinterpret_cast<T*>(g.rh);
  T* ph = reinterpret_cast<T*>(g.ph);
  T* qh = reinterpret_cast<T*>(g.qh);
  // g.iters iterations in one launch: the operator and the blocks stay in L1 between them
  // (L1 is invalidated at kernel boundaries only)
  for (int it = 0; it < g.iters; ++it) {
  if (it > 0 && a.ctl[CTL_FLAG] != FLAG_RUN) return;
  // Q = A P ; den = sum(p̂^H Q)   and   q̂ = A^H p̂
  T part = Ar<T>::zero();
  for (long long i = tid; i < n; i += nt) {
    const int b = g.rp[i], e = g.rp[i + 1];
    T rs = Ar<T>::zero();
    if (s <= 8) {  // entries outer, the row's s accumulators in registers
      T acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = Ar<T>::zero();
      for (int p = b; p < e; ++p) {
        const T v = val[p];
        const T* Pr = P + (size_t)g.ci[p] * s;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < s) acc[c] = Ar<T>::fma(v, Pr[c], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < s) {
          Q[(size_t)i * s + c] = acc[c];
          rs = Ar<T>::add(rs, acc[c]);
        }
    } else {
      for (int c = 0; c < s; ++c) {
        T acc = Ar<T>::zero();
        for (int p = b; p < e; ++p) acc = Ar<T>::fma(val[p], P[(size_t)g.ci[p] * s + c], acc);
        Q[(size_t)i * s + c] = acc;
        rs = Ar<T>::add(rs, acc);
      }
    }
    part = Ar<T>::cfma(ph[i], rs, part);
    const int bh = g.rpH[i], eh = g.rpH[i + 1];
    T acc = Ar<T>::zero();
    for (int p = bh; p < eh; ++p) acc = Ar<T>::fma(valH[p], ph[g.ciH[p]], acc);
    qh[i] = acc;
  }
  const T den = cta_sum(part, red);
  if (tid == 0) *W<T>(a, SL_DEN) = den;
  __syncthreads();
  a.phase = 1;
  gl_bicg<T>(a);  // alpha = rho / den (ends with a CTA barrier)
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  const T alpha = *W<T>(a, SL_ALPHA);
  const T malc = Ar<T>::sub(Ar<T>::zero(), Ar<T>::conj(alpha));  // r̂ -= conj(alpha) q̂
  const T mal = Ar<T>::sub(Ar<T>::zero(), alpha);
  // r̂, X, R ; rho_new = sum(r̂^H R), ||R||^2 (each thread owns its rows: no barrier needed
  // between the r̂ update and its use in the same row)
  T rpart = Ar<T>::zero();
  double r2 = 0.0;
  for (long long i = tid; i < n; i += nt) {
    const T rhi = Ar<T>::fma(qh[i], malc, rh[i]);
    rh[i] = rhi;
    T rs = Ar<T>::zero();
    for (int c = 0; c < s; ++c) {
      const size_t k = (size_t)i * s + c;
      X[k] = Ar<T>::fma(P[k], alpha, X[k]);
      const T r = Ar<T>::fma(Q[k], mal, R[k]);
      R[k] = r;
      rs = Ar<T>::add(rs, r);
      r2 += Ar<T>::abs2(r);
    }
    rpart = Ar<T>::cfma(rhi, rs, rpart);
  }
  const T rhon = cta_sum(rpart, red);
  const double r2s = cta_sum(r2, redd);
  if (tid == 0) {
    *W<T>(a, SL_RHON) = rhon;
    *D(a, SL_R2) = r2s;
  }
  __syncthreads();
  a.phase = 2;
  gl_bicg<T>(a);  // beta = rho_new / rho, convergence test
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  const T beta = *W<T>(a, SL_BETA);
  const T bc = Ar<T>::conj(beta);
  for (long long i = tid; i < n; i += nt) {
    for (int c = 0; c < s; ++c) {
      const size_t k = (size_t)i * s + c;
      P[k] = Ar<T>::fma(P[k], beta, R[k]);
    }
    ph[i] = Ar<T>::fma(ph[i], bc, rh[i]);
  }
  // end of the iteration (end_iter_kernel's step): count it, commit a pending convergence
  if (tid == 0) {
    a.ctl[CTL_ITER] += 1;
    if (a.ctl[CTL_CONVPEND]) {
      a.ctl[CTL_CONVPEND] = 0;
      a.ctl[CTL_FLAG] = FLAG_CONV;
    }
  }
  __syncthreads();
  }  // iterations
}

template <typename T>
__global__ void __launch_bounds__(1024) egl_qmr_small_kernel(SmallQMRArgs g) {
  CoefArgs a = g.ca;
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  __shared__ T red[32];
  __shared__ double redd[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const long long n = g.n;
  const int s = a.s;
  const T* val = reinterpret_cast<const T*>(g.val);
  const T* valH = reinterpret_cast<const T*>(g.valH);
  T* X = reinterpret_cast<T*>(g.X);
  T* R = reinterpret_cast<T*>(g.R);
  T* Vt = reinterpret_cast<T*>(g.Vt);
  T* P = reinterpret_cast<T*>(g.P);
  T* Pt = reinterpret_cast<T*>(g.Pt);
  T* Dd = reinterpret_cast<T*>(g.D);
  T* S = reinterpret_cast<T*>(g.S);
  T* Wt = reinterpret_cast<T*>(g.Wt);
  T* Qv = reinterpret_cast<T*>(g.Qv);
  T* AHQ = reinterpret_cast<T*>(g.AHQ);
  const T zero = Ar<T>::zero();
  auto neg = [&](T v) { return Ar<T>::sub(zero, v); };
  for (int it = 0; it < g.iters; ++it) {
  if (it > 0 && a.ctl[CTL_FLAG] != FLAG_RUN) return;
  a.phase = 1;
  a.k1 = 0;
  qmr_scalar<T>(a, 2);  // 1/rho, 1/xi
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  a.phase = 2;
  a.k1 = a.ctl[CTL_ITER] == 0 ? 1 : 0;  // the first iteration (host_iter == 0 in QMR::seg)
  qmr_scalar<T>(a, 2);  // delta, c1, c2
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  {
    const T ir = *W<T>(a, SL_INVRHO), ix = *W<T>(a, SL_INVXI);
    const T mc1 = neg(*W<T>(a, SL_C1)), mc2 = neg(*W<T>(a, SL_C2));
    for (long long i = tid; i < n; i += nt) {  // P = Ṽ/rho - c1 P ; q = w̃/xi - c2 q
      for (int c = 0; c < s; ++c) {
        const size_t k = (size_t)i * s + c;
        P[k] = Ar<T>::fma(P[k], mc1, Ar<T>::mul(Vt[k], ir));
      }
      Qv[i] = Ar<T>::fma(Qv[i], mc2, Ar<T>::mul(Wt[i], ix));
    }
  }
  __syncthreads();
  // P~ = A P ; eps = sum(q^H P~) ; A^H q
  T part = zero;
  for (long long i = tid; i < n; i += nt) {
    const int b = g.rp[i], e = g.rp[i + 1];
    T rs = zero;
    for (int c = 0; c < s; ++c) {
      T acc = zero;
      for (int p = b; p < e; ++p) acc = Ar<T>::fma(val[p], P[(size_t)g.ci[p] * s + c], acc);
      Pt[(size_t)i * s + c] = acc;
      rs = Ar<T>::add(rs, acc);
    }
    part = Ar<T>::cfma(Qv[i], rs, part);
    const int bh = g.rpH[i], eh = g.rpH[i + 1];
    T acc = zero;
    for (int p = bh; p < eh; ++p) acc = Ar<T>::fma(valH[p], Qv[g.ciH[p]], acc);
    AHQ[i] = acc;
  }
  const T eps = cta_sum(part, red);
  if (tid == 0) *W<T>(a, SL_EPS) = eps;
  __syncthreads();
  a.phase = 3;
  qmr_scalar<T>(a, 2);  // beta, BR, BX
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  {
    const T mbx = neg(*W<T>(a, SL_BX)), mbr = neg(*W<T>(a, SL_BR));
    double xi2 = 0.0, rn2 = 0.0;
    T k1 = zero;
    for (long long i = tid; i < n; i += nt) {  // W̃ = A^H q - (conj(beta)/xi) W̃ ; Ṽ = P~ - (beta/rho) Ṽ
      const T w = Ar<T>::fma(Wt[i], mbx, AHQ[i]);
      Wt[i] = w;
      xi2 += Ar<T>::abs2(w);
      T rs = zero;
      for (int c = 0; c < s; ++c) {
        const size_t k = (size_t)i * s + c;
        const T v = Ar<T>::fma(Vt[k], mbr, Pt[k]);
        Vt[k] = v;
        rn2 += Ar<T>::abs2(v);
        rs = Ar<T>::add(rs, v);
      }
      k1 = Ar<T>::cfma(w, rs, k1);
    }
    const double xs = cta_sum(xi2, redd);
    const double rs2 = cta_sum(rn2, redd);
    const T k1s = cta_sum(k1, red);
    if (tid == 0) {
      *D(a, SL_XI2) = xs;
      *D(a, SL_RHON2) = rs2;
      *W<T>(a, SL_K1) = k1s;
    }
    __syncthreads();
  }
  a.phase = 4;
  qmr_scalar<T>(a, 2);  // theta, gamma, eta, f
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  {
    const T eta = *W<T>(a, SL_ETA), f = *W<T>(a, SL_F);
    double r2 = 0.0;
    for (long long i = tid; i < n; i += nt) {  // D = P eta + D f ; S = P~ eta + S f ; X += D ; R -= S
      for (int c = 0; c < s; ++c) {
        const size_t k = (size_t)i * s + c;
        const T d = Ar<T>::fma(Dd[k], f, Ar<T>::mul(P[k], eta));
        const T sv = Ar<T>::fma(S[k], f, Ar<T>::mul(Pt[k], eta));
        Dd[k] = d;
        S[k] = sv;
        X[k] = Ar<T>::add(X[k], d);
        const T r = Ar<T>::sub(R[k], sv);
        R[k] = r;
        r2 += Ar<T>::abs2(r);
      }
    }
    const double r2s = cta_sum(r2, redd);
    if (tid == 0) *D(a, SL_R2) = r2s;
    __syncthreads();
  }
  a.phase = 5;
  qmr_scalar<T>(a, 2);  // convergence test
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  if (tid == 0) {
    a.ctl[CTL_ITER] += 1;
    if (a.ctl[CTL_CONVPEND]) {
      a.ctl[CTL_CONVPEND] = 0;
      a.ctl[CTL_FLAG] = FLAG_CONV;
    }
  }
  __syncthreads();
  }  // iterations
}

int launch_egl_qmr_small(bool cplx, const SmallQMRArgs& g, cudaStream_t st) {
  const int threads = (int)std::min<long long>(1024, std::max<long long>(32, (g.n + 31) / 32 * 32));
  if (cplx) egl_qmr_small_kernel<double2><<<1, threads, 0, st>>>(g);
  else egl_qmr_small_kernel<double><<<1, threads, 0, st>>>(g);
  return (int)cudaGetLastError();
}

int launch_egl_bicg_small(bool cplx, const SmallBiCGArgs& g, cudaStream_t st) {
  const int threads = (int)std::min<long long>(1024, std::max<long long>(32, (g.n + 31) / 32 * 32));
  if (cplx) egl_bicg_small_kernel<double2><<<1, threads, 0, st>>>(g);
  else egl_bicg_small_kernel<double><<<1, threads, 0, st>>>(g);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------- small Bl-BiCGStab-rQ
// s x s Gram Y^H X over this thread's rows, then a fixed-order CTA sum into ws + slot
// (warp butterflies, then the warps in index order): G[a][c] = sum_i conj(Y[i][a]) X[i][c]
template <typename T, int SK>
__device__ void small_gram(const CoefArgs& a, int slot, const T* Xb, const T* Yb, long long n, int s, T* red) {
  T acc[SK * SK];
#pragma unroll
  for (int q = 0; q < SK * SK; ++q) acc[q] = Ar<T>::zero();
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
#pragma unroll
    for (int r = 0; r < SK; ++r)
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (r < s && c < s) acc[r * SK + c] = Ar<T>::cfma(Yb[(size_t)i * s + r], Xb[(size_t)i * s + c], acc[r * SK + c]);
  }
  // all s^2 entries at once: the same xor butterfly per entry, then the warps' values summed
  // in warp order (bitwise cta_sum's result), with two CTA barriers instead of 2 s^2
  // (red holds >= 32 values: the per-warp partials go to a private slice of shared memory)
#pragma unroll
  for (int q = 0; q < SK * SK; ++q)
    for (int m = 16; m > 0; m >>= 1) acc[q] = Ar<T>::add(acc[q], Ar<T>::shfl_xor(acc[q], m));
  __shared__ T wpart[(SK * SK) * 8];  // [warp][entry], up to 8 warps (the kernel runs 256 threads)
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int q = 0; q < SK * SK; ++q) wpart[w * SK * SK + q] = acc[q];
  __syncthreads();
  if (threadIdx.x < SK * SK) {
    const int r = threadIdx.x / SK, c = threadIdx.x % SK;
    if (r < s && c < s) {
      T v = Ar<T>::zero();
      for (int q = 0; q < nw; ++q) v = Ar<T>::add(v, wpart[q * SK * SK + threadIdx.x]);
      W<T>(a, slot)[r * s + c] = v;
    }
  }
  __syncthreads();
}

// out[i] = sum_t src_t[i] . C_t (row vector times s x s, C row-major), up to 3 terms
template <typename T, int SK>
__device__ __forceinline__ void row_times(T (&o)[SK], const T* x, const T* C, int s, bool neg) {
#pragma unroll
  for (int c = 0; c < SK; ++c) {
    if (c >= s) continue;
    T acc = Ar<T>::zero();
#pragma unroll
    for (int k = 0; k < SK; ++k)
      if (k < s) acc = Ar<T>::fma(x[k], C[k * s + c], acc);
    o[c] = neg ? Ar<T>::sub(o[c], acc) : Ar<T>::add(o[c], acc);
  }
}

template <typename T, int SK>
__device__ void small_spmm(const int* rp, const int* ci, const T* val, const T* P, T* Q, long long n, int s) {
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    T acc[SK];
#pragma unroll
    for (int c = 0; c < SK; ++c) acc[c] = Ar<T>::zero();
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
      const T v = val[p];
      const T* Pr = P + (size_t)ci[p] * s;
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (c < s) acc[c] = Ar<T>::fma(v, Pr[c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < SK; ++c)
      if (c < s) Q[(size_t)i * s + c] = acc[c];
  }
  __syncthreads();
}

template <typename T, int SK>
__global__ void __launch_bounds__(256) bl_bicgstab_rq_small_kernel(SmallBlStabArgs g) {
  CoefArgs a = g.ca;
  if (a.ctl[CTL_FLAG] != FLAG_RUN) return;
  // the s x s algebra is a chain of dependent accesses to the coefficient slots: with the
  // workspace in shared memory (copied in here, back at the end) each is ~30 cycles, not an
  // L2 round trip
  extern __shared__ double smraw[];
  double* const wsg = a.ws;
  for (long long q = threadIdx.x; q < g.ws_doubles; q += blockDim.x) smraw[q] = wsg[q];
  __syncthreads();
  a.ws = smraw;
  T* sh = reinterpret_cast<T*>(smraw + ((g.ws_doubles + 1) & ~1LL));
  __shared__ T red[32];
  const long long n = g.n;
  const int s = a.s;
  const T* val = reinterpret_cast<const T*>(g.val);
  T* X = reinterpret_cast<T*>(g.X);
  T* Qr = reinterpret_cast<T*>(g.Qr);
  const T* Q0 = reinterpret_cast<const T*>(g.Q0);
  T* V = reinterpret_cast<T*>(g.V);
  T* Wb = reinterpret_cast<T*>(g.W);
  T* Z = reinterpret_cast<T*>(g.Z);
  T* Y = reinterpret_cast<T*>(g.Y);
  for (int it = 0; it < g.iters; ++it) {
    if (it > 0 && a.ctl[CTL_FLAG] != FLAG_RUN) break;
    // W = A V ; G = Q̂0^H W
    small_spmm<T, SK>(g.rp, g.ci, val, V, Wb, n, s);
    small_gram<T, SK>(a, SL_G, Wb, Q0, n, s, red);
    a.phase = 1;
    bl_bicgstab_rq<T>(a, sh);  // alpha = G^-1 GQ, AC = alpha C
    if (a.ctl[CTL_FLAG] != FLAG_RUN) break;
    // Z = Qr - W alpha ; ZZ = Z^H Z
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      T o[SK];
#pragma unroll
      for (int c = 0; c < SK; ++c) o[c] = c < s ? Qr[(size_t)i * s + c] : Ar<T>::zero();
      row_times<T, SK>(o, Wb + (size_t)i * s, W<T>(a, SL_ALPHA), s, true);
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (c < s) Z[(size_t)i * s + c] = o[c];
    }
    __syncthreads();
    small_gram<T, SK>(a, SL_ZZ, Z, Z, n, s, red);
    a.phase = 2;
    bl_bicgstab_rq<T>(a, sh);  // half-step test (FLAG_HALF: the host finishes the iteration)
    if (a.ctl[CTL_FLAG] != FLAG_RUN) break;
    // Y = A Z ; YZ = Z^H Y, YY = Y^H Y
    small_spmm<T, SK>(g.rp, g.ci, val, Z, Y, n, s);
    small_gram<T, SK>(a, SL_YZ, Y, Z, n, s, red);
    small_gram<T, SK>(a, SL_YY, Y, Y, n, s, red);
    a.phase = 3;
    bl_bicgstab_rq<T>(a, sh);  // omega, WC = omega C
    if (a.ctl[CTL_FLAG] != FLAG_RUN) break;
    const T om = *W<T>(a, SL_OMEGA);
    // X += V AC + Z WC ; Z = Z - omega Y ; GZ = Z^H Z
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      T xo[SK], zo[SK];
#pragma unroll
      for (int c = 0; c < SK; ++c) {
        xo[c] = c < s ? X[(size_t)i * s + c] : Ar<T>::zero();
        zo[c] = c < s ? Z[(size_t)i * s + c] : Ar<T>::zero();
      }
      row_times<T, SK>(xo, V + (size_t)i * s, W<T>(a, SL_AC), s, false);
      row_times<T, SK>(xo, Z + (size_t)i * s, W<T>(a, SL_WC), s, false);
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (c < s) {
          X[(size_t)i * s + c] = xo[c];
          Z[(size_t)i * s + c] = Ar<T>::sub(zo[c], Ar<T>::mul(Y[(size_t)i * s + c], om));
        }
    }
    __syncthreads();
    small_gram<T, SK>(a, SL_GZ, Z, Z, n, s, red);
    a.phase = 4;
    bl_bicgstab_rq<T>(a, sh);  // CholQR pass 1
    if (a.ctl[CTL_FLAG] != FLAG_RUN) break;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      T o[SK];
#pragma unroll
      for (int c = 0; c < SK; ++c) o[c] = Ar<T>::zero();
      row_times<T, SK>(o, Z + (size_t)i * s, W<T>(a, SL_R1I), s, false);
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (c < s) Z[(size_t)i * s + c] = o[c];
    }
    __syncthreads();
    small_gram<T, SK>(a, SL_GZ, Z, Z, n, s, red);
    a.phase = 5;
    bl_bicgstab_rq<T>(a, sh);  // pass 2, Sig, C = Sig C
    if (a.ctl[CTL_FLAG] != FLAG_RUN) break;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      T o[SK];
#pragma unroll
      for (int c = 0; c < SK; ++c) o[c] = Ar<T>::zero();
      row_times<T, SK>(o, Z + (size_t)i * s, W<T>(a, SL_R2I), s, false);
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (c < s) Qr[(size_t)i * s + c] = o[c];
    }
    __syncthreads();
    small_gram<T, SK>(a, SL_GQN, Qr, Q0, n, s, red);
    a.phase = 6;
    bl_bicgstab_rq<T>(a, sh);  // beta, BW = omega beta, convergence test on ||C||
    if (a.ctl[CTL_FLAG] != FLAG_RUN) break;
    // V = Qr + V beta - W BW
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      T o[SK];
#pragma unroll
      for (int c = 0; c < SK; ++c) o[c] = c < s ? Qr[(size_t)i * s + c] : Ar<T>::zero();
      row_times<T, SK>(o, V + (size_t)i * s, W<T>(a, SL_BETA), s, false);
      row_times<T, SK>(o, Wb + (size_t)i * s, W<T>(a, SL_BW), s, true);
#pragma unroll
      for (int c = 0; c < SK; ++c)
        if (c < s) V[(size_t)i * s + c] = o[c];
    }
    if (threadIdx.x == 0) {  // end of the iteration (end_iter_kernel's step)
      a.ctl[CTL_ITER] += 1;
      if (a.ctl[CTL_CONVPEND]) {
        a.ctl[CTL_CONVPEND] = 0;
        a.ctl[CTL_FLAG] = FLAG_CONV;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  for (long long q = threadIdx.x; q < g.ws_doubles; q += blockDim.x) wsg[q] = smraw[q];
}

int launch_bl_bicgstab_rq_small(bool cplx, const SmallBlStabArgs& g, cudaStream_t st) {
  const int s = g.ca.s;
  const size_t sm = (size_t)((g.ws_doubles + 1) & ~1LL) * 8 + (size_t)(3 * s * s + 64) * (cplx ? 16 : 8) + 1024;
  if (sm > 220 * 1024) return (int)cudaErrorNotSupported;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(bl_bicgstab_rq_small_kernel<double, SMALL_BL_SMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(bl_bicgstab_rq_small_kernel<double2, SMALL_BL_SMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  if (cplx) bl_bicgstab_rq_small_kernel<double2, SMALL_BL_SMAX><<<1, 256, sm, st>>>(g);
  else bl_bicgstab_rq_small_kernel<double, SMALL_BL_SMAX><<<1, 256, sm, st>>>(g);
  return (int)cudaGetLastError();
}

int launch_end_iter(int* ctl, cudaStream_t st) {
  end_iter_kernel<<<1, 1, 0, st>>>(ctl);
  return (int)cudaGetLastError();
}

}  // namespace srk
