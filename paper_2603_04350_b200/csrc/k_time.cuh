// k_time.cuh -- K1, the time-local fused pass of one Exp-ParaDiag sweep (sm_100a, fp64).
//
// In the DST basis every spatial mode J is an independent length-Nt problem (V commutes
// with Q, Q_alpha and F (x) I).  One CTA owns a tile of S mode
// PAIRS x all Nt time slices; the two real modes of a pair travel as one complex
// sequence z_t = u_{2p}(t) + i u_{2p+1}(t) (Hermitian packing), which is also exactly
// how they sit in memory (one 16-byte double2 per pair and slice).  Per tile, in one HBM
// pass:
//   stage 1  r_t = E_J u_{t-1} + C1_J N_t - C2_J N_{t-1} - u_t        (R5/R6)
//            ||r||^2 partials                                         (stage 4 / conv. test)
//   stage 2  Step (a): y = Gamma_alpha r, Y = F y    (alpha^{t/Nt}, omega = e^{+2 pi i/Nt})
//            Step (b): X_k = Y_k / (1 - lambda_k E_J), lambda_k = alpha^{1/Nt} omega^k
//            Step (c): s = Gamma_alpha^{-1} F^* X
//   update   u_t <- u_t + s_t                                         ((3.2))
// The length-Nt DFT is a two-level four-step FFT Nt = P x Q: phase A (thread = pair, m2)
// does the DFT-P over t = Q m1 + m2 in registers and the inter-stage twiddle; phase B
// (thread = pair, {k1, P-k1}) does both DFT-Q's, so every thread holds each frequency k
// together with its Hermitian partner Nt-k and unpacks / divides / repacks the two modes
// in registers, then runs the inverse DFT-Q; phase C inverts the DFT-P and applies the
// update.  Shared memory carries the two transposes; the divisor's 1/Nt (both unitary
// 1/sqrt(Nt) factors) is folded into the reciprocal.
#pragma once
#include <cstdlib>

#include <cuda.h>

#include "expd_internal.h"
#include "fft_dev.cuh"
#include "tma_dev.cuh"

namespace expd {

template <int NT>
struct TimeCfg;
// Radix plan of the length-NT time FFT (Stockham stages R_0 .. R_{L-1}); the last stage
// has a small radix so that a thread can own a frequency set together with its Hermitian
// partner set; TPS = NT / R_0 threads per mode pair; S = 256 / TPS pairs per CTA.
#ifndef EXPD_K1_THREADS
#define EXPD_K1_THREADS 256
#endif
template <int NT> struct TimeCfg;
template <> struct TimeCfg<4>   { static constexpr int L = 1, R0 = 4, R1 = 1, R2 = 1; };
template <> struct TimeCfg<8>   { static constexpr int L = 1, R0 = 8, R1 = 1, R2 = 1; };
template <> struct TimeCfg<16>  { static constexpr int L = 2, R0 = 4, R1 = 4, R2 = 1; };
template <> struct TimeCfg<32>  { static constexpr int L = 2, R0 = 8, R1 = 4, R2 = 1; };
template <> struct TimeCfg<64>  { static constexpr int L = 2, R0 = 8, R1 = 8, R2 = 1; };
template <> struct TimeCfg<128> { static constexpr int L = 3, R0 = 8, R1 = 4, R2 = 4; };
template <> struct TimeCfg<256> { static constexpr int L = 3, R0 = 8, R1 = 8, R2 = 4; };
template <int NT>
struct TimeGeo {
  using C = TimeCfg<NT>;
  static constexpr int L = C::L, R0 = C::R0;
  static constexpr int RL = L == 1 ? C::R0 : (L == 2 ? C::R1 : C::R2);  // last forward radix
  static constexpr int TPS = NT / R0;                                    // threads per pair
  static constexpr int THREADS = EXPD_K1_THREADS;
  static constexpr int S = THREADS / TPS;                                // pairs per CTA
  static constexpr int NSL = NT / RL;                                    // Ns of the last stage
};

__device__ __forceinline__ double2 ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ld2cs(const double* p) {  // streaming: read once
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// 1/D for D in [(1-beta)^2, 4], beta in (0,1): MUFU reciprocal seed + two Newton steps
// (relative error < 2^-52; no branchy IEEE division sequence in the hot loop).
__device__ __forceinline__ double fast_rcp(double D) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(D));
  double e = fma(-D, r, 1.0);
  r = fma(r, e, r);
  e = fma(-D, r, 1.0);
  return fma(r, e, r);
}

// d/2 for one real mode: 1/(2 Nt (1 - beta e^{i theta})) = (1 - beta c + i beta s)/(2 Nt D)
__device__ __forceinline__ double2 half_divisor(double beta, double c, double s, double half_inv_nt) {
  double u = fma(-beta, c, 1.0);
  double v = beta * s;
  double D = fma(u, u, v * v);
  double r = half_inv_nt * fast_rcp(D);
  return make_double2(u * r, v * r);
}

// BDF2: 1 - 4/3 lambda_{0,k} E + 1/3 lambda_{1,k} E^2 with
// lambda_{1,k} = lambda_{0,k}^2 = (1 - x)(1 - x/3), x = beta e^{i theta}: the product of two
// first-order reciprocals.
__device__ __forceinline__ double2 half_divisor_bdf2(double beta, double c, double s, double half_inv_nt) {
  return cmul(half_divisor(beta, c, s, half_inv_nt), half_divisor(beta * (1.0 / 3.0), c, s, 1.0));
}

// 1/(Nt (1 - beta e^{i theta})) for a complex beta = a1 E_J (complex coefficients: every
// mode's time sequence is already complex, so each frequency divides on its own -- no
// Hermitian unpack; PAPER.md:113-124 with complex E_J, :983)
__device__ __forceinline__ double2 cx_divisor(double bx, double by, double c, double s, double inv_nt) {
  const double u = fma(-bx, c, fma(by, s, 1.0));  // Re(1 - beta e^{i theta})
  const double v = -fma(bx, s, by * c);           // Im(1 - beta e^{i theta})
  const double D = fma(u, u, v * v);
  const double r = inv_nt * fast_rcp(D);
  return make_double2(u * r, -v * r);
}

// NL == 3 marks the BDF2 system (linear): residual f2 - R v, Q-operator R v, BDF2 divisor.
// NL == 4 marks a complex-coefficient linear plan: a "pair" is one complex mode (re, im),
// E_J is complex, residual E z_{t-1} - z_t and Q v = v_t - E v_{t-1} in complex arithmetic.
// NL == 5: the BDF2 system with complex coefficients (both of the above).
template <int NL>
struct K1Form {
  static constexpr bool HASN = NL == 1 || NL == 2;  // an N-hat term in the residual
  static constexpr bool BDF = NL == 3 || NL == 5;
  static constexpr bool CX = NL == 4 || NL == 5;
};

// W_k = A Z_k + B conj(Z_kp),  W_kp = conj(A) Z_kp + conj(B) conj(Z_k)
// with A = (da + db)/2, B = (da - db)/2 for the two modes of the pair (Hermitian unpack,
// divide, repack in one step).  tw = e^{2 pi i k/Nt}.
template <bool BDF = false>
__device__ __forceinline__ void divide_pair(double2& Zk, double2& Zkp, double2 tw, double ba, double bb,
                                            double hin, bool self) {
  double2 da = BDF ? half_divisor_bdf2(ba, tw.x, tw.y, hin) : half_divisor(ba, tw.x, tw.y, hin);
  double2 db = BDF ? half_divisor_bdf2(bb, tw.x, tw.y, hin) : half_divisor(bb, tw.x, tw.y, hin);
  double2 A = cadd(da, db), B = csub(da, db);
  double2 zk = Zk, zkp = Zkp;
  // A*zk + B*conj(zkp)
  double2 wk = make_double2(fma(A.x, zk.x, fma(-A.y, zk.y, fma(B.x, zkp.x, B.y * zkp.y))),
                            fma(A.x, zk.y, fma(A.y, zk.x, fma(B.y, zkp.x, -B.x * zkp.y))));
  if (self) {
    Zk = wk;
    return;
  }
  // conj(A)*zkp + conj(B)*conj(zk)
  double2 wkp = make_double2(fma(A.x, zkp.x, fma(A.y, zkp.y, fma(B.x, zk.x, -B.y * zk.y))),
                             fma(A.x, zkp.y, fma(-A.y, zkp.x, fma(-B.y, zk.x, -B.x * zk.y))));
  Zk = wk;
  Zkp = wkp;
}

// One Stockham stage between shared buffers: job (s, j), inputs x[j + r NT/R], twiddle
// w^{r (j mod NS) NT/(NS R)} (w = e^{DIR 2 pi i/NT}), DFT-R, outputs y[(j/NS) NS R + j mod NS + r NS].
template <int NT, int S, int THREADS, int R, int NS, int DIR>
__device__ __forceinline__ void tstage(const double2* __restrict__ in, double2* __restrict__ out,
                                       const double2* __restrict__ stw) {
  constexpr int JOBS = S * (NT / R);
#pragma unroll
  for (int J = threadIdx.x; J < JOBS; J += THREADS) {
    const int s = J % S, j = J / S, k = j % NS;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[(j + r * (NT / R)) * S + s];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double2 w = stw[(r * k * (NT / (NS * R))) & (NT - 1)];
      v[r] = DIR > 0 ? cmul(v[r], w) : cmulc(v[r], w);
    }
    DFT<R, DIR>::run(v);
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) out[(base + r * NS) * S + s] = v[r];
  }
}

// v[r] *= w1^r (DIR > 0) or conj(w1)^r (DIR < 0), r = 1..R-1, powers by products from
// one base twiddle held in a register (binary splitting, <= 2 log2 R roundings deep): the
// twiddles cost fp64 products instead of shared-memory table loads.
template <int R, int DIR>
__device__ __forceinline__ void twpow_mul(double2* v, double2 w1) {
  if constexpr (R > 1) {
    double2 t[R];
    t[1] = w1;
#pragma unroll
    for (int r = 2; r < R; ++r) t[r] = (r % 2 == 0) ? cmul(t[r / 2], t[r / 2]) : cmul(t[r - 1], t[1]);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = DIR > 0 ? cmul(v[r], t[r]) : cmulc(v[r], t[r]);
  }
}

// tstage with the job's base twiddle w^{k NT/(NS R)} in a register: JPT jobs per thread
// (J, J + THREADS, ...), which share k = j mod NS when THREADS / S is a multiple of NS.
template <int NT, int S, int THREADS, int R, int NS, int DIR, int JPT = 1>
__device__ __forceinline__ void tstage_pw(const double2* __restrict__ in, double2* __restrict__ out, double2 w1,
                                          int J = threadIdx.x) {
  constexpr int JOBS = S * (NT / R);
  static_assert(JOBS == THREADS * JPT, "JPT jobs per thread");
  static_assert(JPT == 1 || (THREADS / S) % NS == 0, "the jobs of a thread share their twiddle");
#pragma unroll
  for (int jt = 0; jt < JPT; ++jt) {
    const int Jj = J + jt * THREADS;
    const int s = Jj % S, j = Jj / S, k = j % NS;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[(j + r * (NT / R)) * S + s];
    twpow_mul<R, DIR>(v, w1);
    DFT<R, DIR>::run(v);
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) out[(base + r * NS) * S + s] = v[r];
  }
}

// Last forward stage (radix RL, NS = NT/RL) of two partner jobs ja, jb (their frequency sets
// k = j + NS r are Hermitian partners), the pair divide, and the first inverse stage
// (radix RL, NS = 1: no twiddles) on the same sets.
template <int NT, int RL, bool BDF = false, bool CX = false>
__device__ __forceinline__ void pair_divide(double2 (&va)[RL], double2 (&vb)[RL], bool pj0, const double2* stw,
                                            int ja, int jb, double ba, double bb, double hin) {
  constexpr int NS = NT / RL;
  if constexpr (CX) {  // (ba, bb) = a1 E_J complex; frequency ja + NS r (and jb + NS r)
    const double inv_nt = 2.0 * hin;
    // BDF2: 1 - 4/3 lambda E + 1/3 lambda^2 E^2 = (1 - lambda E)(1 - lambda E / 3)
    auto div = [&](double2 w) {
      const double2 d = cx_divisor(ba, bb, w.x, w.y, inv_nt);
      return BDF ? cmul(d, cx_divisor(ba * (1.0 / 3.0), bb * (1.0 / 3.0), w.x, w.y, 1.0)) : d;
    };
#pragma unroll
    for (int r = 0; r < RL; ++r) va[r] = cmul(va[r], div(stw[ja + NS * r]));
    if (!pj0 || jb != ja) {
#pragma unroll
      for (int r = 0; r < RL; ++r) vb[r] = cmul(vb[r], div(stw[jb + NS * r]));
    }
    return;
  }
  if (!pj0) {
#pragma unroll
    for (int r = 0; r < RL; ++r) divide_pair<BDF>(va[r], vb[RL - 1 - r], stw[ja + NS * r], ba, bb, hin, false);
  } else {
    // ja = 0: frequencies NS r, partner NS (RL - r) mod RL; self at r = 0 and RL/2
    divide_pair<BDF>(va[0], va[0], stw[0], ba, bb, hin, true);
#pragma unroll
    for (int r = 1; r < (RL + 1) / 2; ++r) divide_pair<BDF>(va[r], va[RL - r], stw[NS * r], ba, bb, hin, false);
    if constexpr (RL % 2 == 0) divide_pair<BDF>(va[RL / 2], va[RL / 2], stw[NS * (RL / 2)], ba, bb, hin, true);
    if (jb != ja) {
      // jb = NS/2: frequencies NS/2 + NS r, partner index RL-1-r
#pragma unroll
      for (int r = 0; r < RL / 2; ++r)
        divide_pair<BDF>(vb[r], vb[RL - 1 - r], stw[jb + NS * r], ba, bb, hin, false);
      if constexpr (RL % 2 == 1)
        divide_pair<BDF>(vb[RL / 2], vb[RL / 2], stw[jb + NS * (RL / 2)], ba, bb, hin, true);
    }
  }
}

// BDF2 time-local residual / Q-operator of one mode pair at time t:
// RESID: r_t = 4/3 E p1 - 1/3 E^2 p2 - x_t, p1 = v_{t-1} (u_1 = E u_0 at t = 0), p2 = v_{t-2}
// (u_1 at t = 1, u_0 at t = 0);  QOP: (R v)_t = v_t - 4/3 E v_{t-1} + 1/3 E^2 v_{t-2}.
template <bool RESID, bool CX = false>
__device__ __forceinline__ double2 bdf2_form(double2 E, double2 xc, double2 xm1, double2 xm2, double2 u0, int t) {
  if constexpr (CX) {  // one complex mode: E, the states and u0 are complex numbers
    const double2 zero = make_double2(0.0, 0.0);
    const double2 u1 = cmul(E, u0);
    const double2 p1 = t >= 1 ? xm1 : (RESID ? u1 : zero);
    const double2 p2 = t >= 2 ? xm2 : (t == 1 ? (RESID ? u1 : zero) : (RESID ? u0 : zero));
    const double2 a = cmul(E, p1), b = cmul(E, cmul(E, p2));
    const double2 r = make_double2((4.0 / 3.0) * a.x - (1.0 / 3.0) * b.x, (4.0 / 3.0) * a.y - (1.0 / 3.0) * b.y);
    return RESID ? csub(r, xc) : csub(xc, r);
  }
  const double2 u1 = make_double2(E.x * u0.x, E.y * u0.y);
  const double2 zero = make_double2(0.0, 0.0);
  const double2 p1 = t >= 1 ? xm1 : (RESID ? u1 : zero);
  const double2 p2 = t >= 2 ? xm2 : (t == 1 ? (RESID ? u1 : zero) : (RESID ? u0 : zero));
  const double c43 = 4.0 / 3.0, c13 = 1.0 / 3.0;
  const double2 e2 = make_double2(E.x * E.x, E.y * E.y);
  double2 r;
  r.x = fma(c43 * E.x, p1.x, -c13 * e2.x * p2.x);
  r.y = fma(c43 * E.y, p1.y, -c13 * e2.y * p2.y);
  return RESID ? make_double2(r.x - xc.x, r.y - xc.y) : make_double2(xc.x - r.x, xc.y - r.y);
}

#ifndef EXPD_K1_MINB
#define EXPD_K1_MINB 2
#endif
#ifndef EXPD_K1_REREAD
#define EXPD_K1_REREAD 0
#endif
template <int NT, int RM, int OUTM, int NL>
__global__ void __launch_bounds__(EXPD_K1_THREADS, EXPD_K1_MINB) k_time_fused(const TimeArgs a) {
  using G = TimeGeo<NT>;
  using C = TimeCfg<NT>;
  constexpr int L = G::L, R0 = G::R0, RL = G::RL, TPS = G::TPS, S = G::S, THREADS = G::THREADS;
  constexpr int NSL = G::NSL;
  extern __shared__ double2 smem[];
  double2* buf0 = smem;                      // [NT][S]
  double2* buf1 = smem + (L > 1 ? NT * S : 0);
  double2* stw = smem + (L > 1 ? 2 * NT * S : 0);  // [NT] e^{+2 pi i q/NT}
  double* sg = reinterpret_cast<double*>(stw + NT);  // [NT] alpha^{t/NT}
  double* sgi = sg + NT;                              // [NT] alpha^{-t/NT}

  const int tid = threadIdx.x;
  for (int i = tid; i < NT; i += THREADS) {
    stw[i] = a.tw[i];
    sg[i] = a.g[i];
    sgi[i] = a.ginv[i];
  }
  __syncthreads();

  const long npad = a.npad;
  const long ntiles = (a.npairs + S - 1) / S;
  const double hin = a.half_inv_nt;
  double nrm = 0.0;
  const int s = tid % S;   // pair within the tile (fastest: conflict-free shared accesses)
  const int j = tid / S;   // stage-0 job: times j + r TPS

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long pair = tile * S + s;
    const bool valid = pair < a.npairs;
    const long base = 2 * pair;

    // ---- phase A: stage 1 residual (+ ||r||^2), Gamma_alpha, forward stage 0 ----------
    double2 y[R0];
    double2 xv[(OUTM == OUT_UPDATE && !EXPD_K1_REREAD) ? R0 : 1];
    double2 Ej = make_double2(0.0, 0.0), c1 = Ej, c2 = Ej;
    if (valid && RM != RM_INPUT) Ej = ld2(a.E + base);
    if (valid && K1Form<NL>::HASN) c1 = ld2(a.C1 + base);
    if (valid && NL == 2) c2 = ld2(a.C2 + base);
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      double2 cur = make_double2(0.0, 0.0), rr;
      if (valid) cur = (OUTM == OUT_UPDATE) ? ld2(a.X + (long)t * npad + base) : ld2cs(a.X + (long)t * npad + base);
      if constexpr (RM == RM_INPUT) {
        rr = cur;
      } else if constexpr (K1Form<NL>::BDF) {
        double2 xm1 = make_double2(0.0, 0.0), xm2 = xm1, u0 = xm1;
        if (valid) {
          if (t >= 1) xm1 = ld2(a.X + (long)(t - 1) * npad + base);
          if (t >= 2) xm2 = ld2(a.X + (long)(t - 2) * npad + base);
          if (RM == RM_RESID) u0 = ld2(a.u0h + base);
        }
        rr = bdf2_form<RM == RM_RESID, K1Form<NL>::CX>(Ej, cur, xm1, xm2, u0, t);
      } else {
        double2 prev = make_double2(0.0, 0.0);
        if (valid) {
          if (t > 0) prev = ld2(a.X + (long)(t - 1) * npad + base);
          else if (RM == RM_RESID) prev = ld2(a.u0h + base);
        }
        if constexpr (K1Form<NL>::CX) {
          const double2 ep = cmul(Ej, prev);
          rr = RM == RM_RESID ? csub(ep, cur) : csub(cur, ep);
        } else if constexpr (RM == RM_RESID) {
          rr = make_double2(fma(Ej.x, prev.x, -cur.x), fma(Ej.y, prev.y, -cur.y));
          if constexpr (K1Form<NL>::HASN) {
            double2 nm1 = valid ? ld2cs(a.Nh + (long)t * npad + base) : make_double2(0.0, 0.0);
            rr.x = fma(c1.x, nm1.x, rr.x);
            rr.y = fma(c1.y, nm1.y, rr.y);
            if constexpr (NL == 2) {
              double2 nm2 = valid ? ld2(a.Nh + (long)(t > 0 ? t - 1 : 0) * npad + base) : make_double2(0.0, 0.0);
              rr.x = fma(-c2.x, nm2.x, rr.x);
              rr.y = fma(-c2.y, nm2.y, rr.y);
            }
          }
        } else {  // RM_QOP: (Q v)_t = v_t - E v_{t-1}, v_{-1} = 0
          rr = make_double2(fma(-Ej.x, prev.x, cur.x), fma(-Ej.y, prev.y, cur.y));
        }
      }
      nrm = fma(rr.x, rr.x, fma(rr.y, rr.y, nrm));
      if constexpr (OUTM == OUT_UPDATE && !EXPD_K1_REREAD) xv[r] = cur;
      y[r] = cscale(rr, sg[t]);
    }
    DFT<R0, +1>::run(y);

    if constexpr (L == 1) {
      // single stage: job 0 owns every frequency; divide its Hermitian pairs in place
      const double2 Ep = valid ? ld2(a.E + base) : make_double2(0.0, 0.0);
      const double ba = a.a1 * Ep.x, bb = a.a1 * Ep.y;
      double2 dummy[R0];
      pair_divide<NT, R0, K1Form<NL>::BDF, K1Form<NL>::CX>(y, dummy, true, stw, 0, 0, ba, bb, hin);
      DFT<R0, -1>::run(y);
    } else {
#pragma unroll
      for (int r = 0; r < R0; ++r) buf0[(j * R0 + r) * S + s] = y[r];
      __syncthreads();
      const double2* pin = buf0;
      double2* pout = buf1;
      if constexpr (L == 3) {  // forward middle stage
        tstage<NT, S, THREADS, C::R1, R0, +1>(buf0, buf1, stw);
        __syncthreads();
        pin = buf1;
        pout = buf0;
      }
      // ---- pair stage: last forward stage, divide, first inverse stage ---------------
      for (int PJ = tid; PJ < S * (NSL / 2); PJ += THREADS) {
        const int ps = PJ % S, pj = PJ / S;
        const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
        const long jpair = tile * S + ps;
        double2 va[RL], vb[RL];
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          va[r] = pin[(ja + r * NSL) * S + ps];
          vb[r] = pin[(jb + r * NSL) * S + ps];
        }
#pragma unroll
        for (int r = 1; r < RL; ++r) {
          va[r] = cmul(va[r], stw[(r * ja) & (NT - 1)]);
          vb[r] = cmul(vb[r], stw[(r * jb) & (NT - 1)]);
        }
        DFT<RL, +1>::run(va);
        DFT<RL, +1>::run(vb);
        const double2 Ep = jpair < a.npairs ? ld2(a.E + 2 * jpair) : make_double2(0.0, 0.0);
        pair_divide<NT, RL, K1Form<NL>::BDF, K1Form<NL>::CX>(va, vb, pj == 0, stw, ja, jb, a.a1 * Ep.x,
                                                           a.a1 * Ep.y, hin);
        DFT<RL, -1>::run(va);
        DFT<RL, -1>::run(vb);
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          pout[(ja * RL + r) * S + ps] = va[r];
          pout[(jb * RL + r) * S + ps] = vb[r];
        }
      }
      __syncthreads();
      if constexpr (L == 3) {  // inverse middle stage (radix R1, NS = RL)
        tstage<NT, S, THREADS, C::R1, RL, -1>(buf0, buf1, stw);
        __syncthreads();
      }
      const double2* cin = (L == 3) ? buf1 : buf1;
      // ---- phase C input: inverse last stage (radix R0, NS = TPS) ----------------------
#pragma unroll
      for (int r = 0; r < R0; ++r) y[r] = cin[(j + r * TPS) * S + s];
#pragma unroll
      for (int r = 1; r < R0; ++r) y[r] = cmulc(y[r], stw[(r * j) & (NT - 1)]);
      DFT<R0, -1>::run(y);
    }
    // ---- phase C: Gamma_alpha^{-1}, update, store (times j + r TPS) -------------------
    if (valid) {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int t = j + r * TPS;
        double2 sv = cscale(y[r], sgi[t]);
        if constexpr (OUTM == OUT_UPDATE) {
          if constexpr (EXPD_K1_REREAD) sv = cadd(ld2(a.X + (long)t * npad + base), sv);  // L2 hit
          else sv = cadd(xv[r], sv);
        }
        EXPD_CHECK(base >= 0 && base + 1 < npad && t < NT, "K1: store index");
        EXPD_CHECK(base >= 0 && base + 1 < npad && t < NT, "K1 ring: store index");
      st2(a.Y + (long)t * npad + base, sv);
      }
    }
  }

  if (a.partial) {
    // fixed-order block reduction (deterministic for a fixed grid)
    __shared__ double red[THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if ((tid & 31) == 0) red[tid >> 5] = nrm;
    __syncthreads();
    if (tid < 32) {
      double v = tid < THREADS / 32 ? red[tid] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (tid == 0) a.partial[blockIdx.x] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K1, software-pipelined: one persistent CTA per SM; while tile i is transformed, the
// U-hat / N-hat time columns (and the per-mode tables) of tile i+1 stream into the other
// half of a double-buffered shared-memory stage with cp.async, so phase A never waits on
// HBM latency.  Phase C takes u_t for the update from the staged tile, not registers.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void cpa16(void* smem, const void* gmem, bool valid) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;  // zero-fill past the last mode pair
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// DB: double-buffered stage, one CTA per SM.  !DB: one stage per CTA, two CTAs per SM
// (the other CTA's math hides this one's cp.async latency); buf0 then aliases the N-hat
// part of the stage (N-hat is dead once phase A has run).
template <int NT, int RM, int NL, bool DB>
struct PipeLayout {
  using G = TimeGeo<NT>;
  static constexpr int S = G::S;
  static constexpr int TILE = NT * S;                   // double2 per staged array
  static constexpr int NARR = 1 + (NL ? 1 : 0);         // X (+ N-hat)
  static constexpr int AUX = 4 * S;                     // E, C1, C2, u0-hat per pair
  static constexpr int STAGE = NARR * TILE + AUX;       // double2 per pipeline stage
  static constexpr bool ALIAS = !DB && NL;              // buf0 inside the stage's N-hat block
  static constexpr int NSTAGE = DB ? 2 : 1;
  static constexpr int FFTBUF = ALIAS ? TILE : 2 * TILE;
  static constexpr size_t BYTES = sizeof(double2) * (NSTAGE * STAGE + FFTBUF + NT) + sizeof(double) * 2 * NT;
};

template <int NT, int RM, int NL, bool DB>
__device__ __forceinline__ void pipe_issue(const TimeArgs& a, long tile, double2* stage) {
  using PL = PipeLayout<NT, RM, NL, DB>;
  constexpr int S = PL::S, TILE = PL::TILE, THREADS = TimeGeo<NT>::THREADS;
  const long npad = a.npad;
  for (int c = threadIdx.x; c < TILE; c += THREADS) {
    const int t = c / S, s = c % S;
    const long pair = tile * S + s;
    const bool ok = pair < a.npairs;
    const long off = (long)t * npad + 2 * (ok ? pair : 0);
    cpa16(stage + c, a.X + off, ok);
    if constexpr (NL) cpa16(stage + TILE + c, a.Nh + off, ok);
  }
  if (threadIdx.x < S) {
    const int s = threadIdx.x;
    const long pair = tile * S + s;
    const bool ok = pair < a.npairs;
    const long off = 2 * (ok ? pair : 0);
    double2* aux = stage + PL::NARR * TILE;
    cpa16(aux + s, a.E + off, ok);
    if constexpr (NL >= 1) cpa16(aux + S + s, a.C1 + off, ok);
    if constexpr (NL == 2) cpa16(aux + 2 * S + s, a.C2 + off, ok);
    if constexpr (RM == RM_RESID) cpa16(aux + 3 * S + s, a.u0h + off, ok);
  }
  cpa_commit();
}

template <int NT, int RM, int OUTM, int NL, bool DB>
__global__ void __launch_bounds__(EXPD_K1_THREADS, DB ? 1 : 2) k_time_pipe(const TimeArgs a) {
  using G = TimeGeo<NT>;
  using C = TimeCfg<NT>;
  using PL = PipeLayout<NT, RM, NL, DB>;
  constexpr int L = G::L, R0 = G::R0, RL = G::RL, TPS = G::TPS, S = G::S, THREADS = G::THREADS;
  constexpr int NSL = G::NSL, TILE = PL::TILE;
  static_assert(L > 1, "pipelined kernel needs a multi-stage FFT");
  extern __shared__ double2 smem[];
  double2* buf0 = PL::ALIAS ? smem + TILE : smem + PL::NSTAGE * PL::STAGE;  // [NT][S]
  double2* buf1 = PL::ALIAS ? smem + PL::STAGE : buf0 + TILE;
  double2* stw = smem + PL::NSTAGE * PL::STAGE + PL::FFTBUF;  // [NT] e^{+2 pi i q/NT}
  double* sg = reinterpret_cast<double*>(stw + NT);
  double* sgi = sg + NT;

  const int tid = threadIdx.x;
  for (int i = tid; i < NT; i += THREADS) {
    stw[i] = a.tw[i];
    sg[i] = a.g[i];
    sgi[i] = a.ginv[i];
  }
  const long npad = a.npad;
  const long ntiles = (a.npairs + S - 1) / S;
  const double hin = a.half_inv_nt;
  double nrm = 0.0;
  const int s = tid % S;
  const int j = tid / S;

  long tile = blockIdx.x;
  int cur = 0;
  if (DB && tile < ntiles) pipe_issue<NT, RM, NL, DB>(a, tile, smem);
  for (; tile < ntiles; tile += gridDim.x, cur ^= (DB ? 1 : 0)) {
    if constexpr (DB) {
      const long next = tile + gridDim.x;
      if (next < ntiles) {
        pipe_issue<NT, RM, NL, DB>(a, next, smem + (cur ^ 1) * PL::STAGE);
        cpa_wait<1>();
      } else {
        cpa_wait<0>();
      }
    } else {
      pipe_issue<NT, RM, NL, DB>(a, tile, smem);
      cpa_wait<0>();
    }
    __syncthreads();
    const double2* X = smem + cur * PL::STAGE;
    const double2* NH = X + TILE;
    const double2* aux = X + PL::NARR * TILE;
    const long pair = tile * S + s;
    const bool valid = pair < a.npairs;
    const long base = 2 * pair;

    // ---- phase A: residual (+ ||r||^2), Gamma_alpha, forward stage 0 (times j + r TPS) ---
    double2 y[R0];
    const double2 Ej = aux[s];
    const double2 c1 = NL >= 1 ? aux[S + s] : make_double2(0.0, 0.0);
    const double2 c2 = NL == 2 ? aux[2 * S + s] : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      const double2 xc = X[t * S + s];
      double2 rr;
      if constexpr (RM == RM_INPUT) {
        rr = xc;
      } else {
        const double2 prev = t > 0 ? X[(t - 1) * S + s] : (RM == RM_RESID ? aux[3 * S + s] : make_double2(0.0, 0.0));
        if constexpr (K1Form<NL>::CX) {
          const double2 ep = cmul(Ej, prev);
          rr = RM == RM_RESID ? csub(ep, xc) : csub(xc, ep);
        } else if constexpr (RM == RM_RESID) {
          rr = make_double2(fma(Ej.x, prev.x, -xc.x), fma(Ej.y, prev.y, -xc.y));
          if constexpr (NL >= 1) {
            const double2 nm1 = NH[t * S + s];
            rr.x = fma(c1.x, nm1.x, rr.x);
            rr.y = fma(c1.y, nm1.y, rr.y);
            if constexpr (NL == 2) {
              const double2 nm2 = NH[(t > 0 ? t - 1 : 0) * S + s];
              rr.x = fma(-c2.x, nm2.x, rr.x);
              rr.y = fma(-c2.y, nm2.y, rr.y);
            }
          }
        } else {  // RM_QOP
          rr = make_double2(fma(-Ej.x, prev.x, xc.x), fma(-Ej.y, prev.y, xc.y));
        }
      }
      nrm = fma(rr.x, rr.x, fma(rr.y, rr.y, nrm));
      y[r] = cscale(rr, sg[t]);
    }
    DFT<R0, +1>::run(y);
    if constexpr (PL::ALIAS) __syncthreads();  // every thread is done reading N-hat
#pragma unroll
    for (int r = 0; r < R0; ++r) buf0[(j * R0 + r) * S + s] = y[r];
    __syncthreads();
    const double2* pin = buf0;
    double2* pout = buf1;
    if constexpr (L == 3) {
      tstage<NT, S, THREADS, C::R1, R0, +1>(buf0, buf1, stw);
      __syncthreads();
      pin = buf1;
      pout = buf0;
    }
    for (int PJ = tid; PJ < S * (NSL / 2); PJ += THREADS) {
      const int ps = PJ % S, pj = PJ / S;
      const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
      double2 va[RL], vb[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        va[r] = pin[(ja + r * NSL) * S + ps];
        vb[r] = pin[(jb + r * NSL) * S + ps];
      }
#pragma unroll
      for (int r = 1; r < RL; ++r) {
        va[r] = cmul(va[r], stw[(r * ja) & (NT - 1)]);
        vb[r] = cmul(vb[r], stw[(r * jb) & (NT - 1)]);
      }
      DFT<RL, +1>::run(va);
      DFT<RL, +1>::run(vb);
      const double2 Ep = aux[ps];
#ifdef EXPD_K1_NODIV_EXPERIMENT
      pair_divide<NT, RL>(va, vb, false, stw, ja, jb, a.a1 * Ep.x, a.a1 * Ep.y, hin);
#else
      pair_divide<NT, RL>(va, vb, pj == 0, stw, ja, jb, a.a1 * Ep.x, a.a1 * Ep.y, hin);
#endif
      DFT<RL, -1>::run(va);
      DFT<RL, -1>::run(vb);
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        pout[(ja * RL + r) * S + ps] = va[r];
        pout[(jb * RL + r) * S + ps] = vb[r];
      }
    }
    __syncthreads();
    if constexpr (L == 3) {
      tstage<NT, S, THREADS, C::R1, RL, -1>(buf0, buf1, stw);
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) y[r] = buf1[(j + r * TPS) * S + s];
#pragma unroll
    for (int r = 1; r < R0; ++r) y[r] = cmulc(y[r], stw[(r * j) & (NT - 1)]);
    DFT<R0, -1>::run(y);
    // ---- phase C: Gamma_alpha^{-1}, update (u_t from the staged tile), store ------------
    if (valid) {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int t = j + r * TPS;
        double2 sv = cscale(y[r], sgi[t]);
        if constexpr (OUTM == OUT_UPDATE) sv = cadd(X[t * S + s], sv);
        EXPD_CHECK(base >= 0 && base + 1 < npad && t < NT, "K1: store index");
        st2(a.Y + (long)t * npad + base, sv);
      }
    }
    __syncthreads();  // stage `cur` is refilled by the next iteration's prefetch
  }

  if (a.partial) {
    __shared__ double red[THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if ((tid & 31) == 0) red[tid >> 5] = nrm;
    __syncthreads();
    if (tid < 32) {
      double v = tid < THREADS / 32 ? red[tid] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (tid == 0) a.partial[blockIdx.x] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K1, TMA-fed: the U-hat / N-hat time columns of a tile (S mode pairs x all NT slices =
// one {2S doubles, NT rows} box per array) arrive by TMA tensor loads on an mbarrier (one
// instruction per array instead of 2 NT S / THREADS cp.async per thread); the per-mode
// tables by cp.async.  NST = 2: the next tile's loads overlap this tile's transform;
// NST = 1: the overlap comes from the other CTAs on the SM.  THR sets S = THR / TPS.
// ---------------------------------------------------------------------------------------
template <int NT, int THR>
struct TGeo {
  using C = TimeCfg<NT>;
  static constexpr int L = C::L, R0 = C::R0;
  static constexpr int RL = L == 1 ? C::R0 : (L == 2 ? C::R1 : C::R2);
  static constexpr int TPS = NT / R0;
  static constexpr int THREADS = THR;
  static constexpr int S = THR / TPS;
  static constexpr int NSL = NT / RL;
  static_assert(S >= 1 && S * TPS == THR, "THR must be a multiple of NT / R0");
};

template <int NT, int THR, int NL, int NST>
struct TmaLayout {
  using G = TGeo<NT, THR>;
  static constexpr int S = G::S;
  static constexpr int TILE = NT * S;                  // double2 per staged array
  static constexpr int NARR = 1 + (K1Form<NL>::HASN ? 1 : 0);
  static constexpr int AUX = 4 * S;                    // E, C1, C2, u0-hat per pair
  static constexpr int STAGE = ((NARR * TILE + AUX) + 7) / 8 * 8;  // 128-byte multiple
  static constexpr bool ALIAS = K1Form<NL>::HASN;      // buf0 in the stage's N-hat block
  static constexpr int FFTBUF = ALIAS ? TILE : 2 * TILE;
  static constexpr size_t BYTES =
      128 + sizeof(double2) * ((size_t)NST * STAGE + FFTBUF + NT) + sizeof(double) * 2 * NT + 16 * NST;
  static constexpr int MINB_SMEM = (int)((228 * 1024) / (BYTES + 1024));
  static constexpr int MINB = MINB_SMEM < 1 ? 1 : (MINB_SMEM > 8 ? 8 : MINB_SMEM);
};

template <int NT, int THR, int RM, int NL, int NST>
__device__ __forceinline__ void tma_tile_issue(const CUtensorMap* mx, const CUtensorMap* mn, const TimeArgs& a,
                                               long tile, double2* stage, uint64_t* bar) {
  using PL = TmaLayout<NT, THR, NL, NST>;
  constexpr int S = PL::S, TILE = PL::TILE;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, (uint32_t)(PL::NARR * TILE * 16));
    tma_load_2d(stage, mx, bar, (int)(2 * S * tile), 0);
    if constexpr (K1Form<NL>::HASN) tma_load_2d(stage + TILE, mn, bar, (int)(2 * S * tile), 0);
  }
  if (threadIdx.x < S) {
    const int s = threadIdx.x;
    const long pair = tile * S + s;
    const bool ok = pair < a.npairs;
    const long off = 2 * (ok ? pair : 0);
    double2* aux = stage + PL::NARR * TILE;
    cpa16(aux + s, a.E + off, ok);
    if constexpr (K1Form<NL>::HASN) cpa16(aux + S + s, a.C1 + off, ok);
    if constexpr (NL == 2) cpa16(aux + 2 * S + s, a.C2 + off, ok);
    if constexpr (RM == RM_RESID) cpa16(aux + 3 * S + s, a.u0h + off, ok);
  }
  cpa_commit();
}

template <int NT, int RM, int OUTM, int NL, int THR, int NST>
__global__ void __launch_bounds__(THR, (TmaLayout<NT, THR, NL, NST>::MINB))
    k_time_tma(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mn,
               const __grid_constant__ TimeArgs a) {
  using G = TGeo<NT, THR>;
  using C = TimeCfg<NT>;
  using PL = TmaLayout<NT, THR, NL, NST>;
  constexpr int L = G::L, R0 = G::R0, RL = G::RL, TPS = G::TPS, S = G::S, THREADS = THR;
  constexpr int NSL = G::NSL, TILE = PL::TILE;
  static_assert(L > 1, "TMA kernel needs a multi-stage FFT");
  extern __shared__ unsigned char tsm_raw[];
  // 128-byte aligned base as an offset from the __shared__ array (keeps LDS/STS)
  double2* smem = reinterpret_cast<double2*>(tsm_raw + ((128u - (smem_u32(tsm_raw) & 127u)) & 127u));
  double2* fft = smem + NST * PL::STAGE;
  double2* stw = fft + PL::FFTBUF;                     // [NT] e^{+2 pi i q/NT}
  double* sg = reinterpret_cast<double*>(stw + NT);    // [NT] alpha^{t/NT}
  double* sgi = sg + NT;                               // [NT] alpha^{-t/NT}
  uint64_t* bar = reinterpret_cast<uint64_t*>(sgi + NT);

  const int tid = threadIdx.x;
  __builtin_assume(tid < THREADS);
  for (int i = tid; i < NT; i += THREADS) {
    stw[i] = a.tw[i];
    sg[i] = a.g[i];
    sgi[i] = a.ginv[i];
  }
  if (tid == 0) {
    prefetch_tmap(&mx);
    if constexpr (K1Form<NL>::HASN) prefetch_tmap(&mn);
    for (int k = 0; k < NST; ++k) mbar_init(&bar[k], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const long ntiles = (a.npairs + S - 1) / S;
  const double hin = a.half_inv_nt;
  double nrm = 0.0;
  const int s = tid % S;
  const int j = tid / S;
  const long npad = a.npad;
  // loop-invariant base twiddles of this thread's jobs (each stage has one job per thread
  // in the L = 3 plans used at NT >= 64; other plans keep the table loads)
  constexpr bool PW = (L == 3) && (S * (NT / C::R1) == THREADS) && (S * (NSL / 2) == THREADS);
  double2 w_fm = make_double2(1.0, 0.0), w_im = w_fm, w_pa = w_fm, w_pb = w_fm, w_c = w_fm;
  if constexpr (PW) {
    w_fm = stw[((j % R0) * (NT / (R0 * C::R1))) & (NT - 1)];   // forward middle stage, NS = R0
    w_im = stw[((j % RL) * (NT / (RL * C::R1))) & (NT - 1)];   // inverse middle stage, NS = RL
    const int pj = tid / S;
    w_pa = stw[pj & (NT - 1)];
    w_pb = stw[(pj == 0 ? NSL / 2 : NSL - pj) & (NT - 1)];
    w_c = stw[j & (NT - 1)];                                     // phase C (inverse stage 0)
  }

  long tile = blockIdx.x;
  if (tile < ntiles) tma_tile_issue<NT, THR, RM, NL, NST>(&mx, &mn, a, tile, smem, &bar[0]);
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int cur = NST == 2 ? (it & 1) : 0;
    double2* stg = smem + cur * PL::STAGE;
    const long next = tile + gridDim.x;
    if constexpr (NST == 2) {
      if (next < ntiles) {
        tma_tile_issue<NT, THR, RM, NL, NST>(&mx, &mn, a, next, smem + (cur ^ 1) * PL::STAGE, &bar[cur ^ 1]);
        cpa_wait<1>();
      } else {
        cpa_wait<0>();
      }
    } else {
      cpa_wait<0>();
    }
    mbar_wait(&bar[cur], (uint32_t)((NST == 2 ? (it >> 1) : it) & 1));
    __syncthreads();  // the cp.async aux of every thread < S is visible
    const double2* X = stg;
    const double2* NH = stg + TILE;
    const double2* aux = stg + PL::NARR * TILE;
    double2* buf0 = PL::ALIAS ? stg + TILE : fft;
    double2* buf1 = PL::ALIAS ? fft : fft + TILE;
    const long pair = tile * S + s;
    const bool valid = pair < a.npairs;
    const long base = 2 * pair;

    // ---- phase A: residual (+ ||r||^2), Gamma_alpha, forward stage 0 (times j + r TPS) ---
    double2 y[R0];
    double2 xv[OUTM == OUT_UPDATE ? R0 : 1];  // u_t kept in registers for the update
    const double2 Ej = aux[s];
    const double2 c1 = K1Form<NL>::HASN ? aux[S + s] : make_double2(0.0, 0.0);
    const double2 c2 = NL == 2 ? aux[2 * S + s] : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      const double2 xc = X[t * S + s];
      if constexpr (OUTM == OUT_UPDATE) xv[r] = xc;
      double2 rr;
      if constexpr (RM == RM_INPUT) {
        rr = xc;
      } else if constexpr (K1Form<NL>::BDF) {
        const double2 zero = make_double2(0.0, 0.0);
        const double2 xm1 = t >= 1 ? X[(t - 1) * S + s] : zero;
        const double2 xm2 = t >= 2 ? X[(t - 2) * S + s] : zero;
        const double2 u0 = RM == RM_RESID ? aux[3 * S + s] : zero;
        rr = bdf2_form<RM == RM_RESID, K1Form<NL>::CX>(Ej, xc, xm1, xm2, u0, t);
      } else {
        const double2 prev = t > 0 ? X[(t - 1) * S + s] : (RM == RM_RESID ? aux[3 * S + s] : make_double2(0.0, 0.0));
        if constexpr (K1Form<NL>::CX) {
          const double2 ep = cmul(Ej, prev);
          rr = RM == RM_RESID ? csub(ep, xc) : csub(xc, ep);
        } else if constexpr (RM == RM_RESID) {
          rr = make_double2(fma(Ej.x, prev.x, -xc.x), fma(Ej.y, prev.y, -xc.y));
          if constexpr (K1Form<NL>::HASN) {
            const double2 nm1 = NH[t * S + s];
            rr.x = fma(c1.x, nm1.x, rr.x);
            rr.y = fma(c1.y, nm1.y, rr.y);
            if constexpr (NL == 2) {
              const double2 nm2 = NH[(t > 0 ? t - 1 : 0) * S + s];
              rr.x = fma(-c2.x, nm2.x, rr.x);
              rr.y = fma(-c2.y, nm2.y, rr.y);
            }
          }
        } else {  // RM_QOP
          rr = make_double2(fma(-Ej.x, prev.x, xc.x), fma(-Ej.y, prev.y, xc.y));
        }
      }
      nrm = fma(rr.x, rr.x, fma(rr.y, rr.y, nrm));
      y[r] = cscale(rr, sg[t]);
    }
    DFT<R0, +1>::run(y);
    if constexpr (PL::ALIAS) __syncthreads();  // every thread is done reading N-hat
#pragma unroll
    for (int r = 0; r < R0; ++r) buf0[(j * R0 + r) * S + s] = y[r];
    __syncthreads();
    const double2* pin = buf0;
    double2* pout = buf1;
    if constexpr (L == 3) {
      if constexpr (PW) tstage_pw<NT, S, THREADS, C::R1, R0, +1>(buf0, buf1, w_fm);
      else tstage<NT, S, THREADS, C::R1, R0, +1>(buf0, buf1, stw);
      __syncthreads();
      pin = buf1;
      pout = buf0;
    }
    for (int PJ = tid; PJ < S * (NSL / 2); PJ += THREADS) {
      const int ps = PJ % S, pj = PJ / S;
      const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
      double2 va[RL], vb[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        va[r] = pin[(ja + r * NSL) * S + ps];
        vb[r] = pin[(jb + r * NSL) * S + ps];
      }
      if constexpr (PW) {
        twpow_mul<RL, +1>(va, w_pa);
        twpow_mul<RL, +1>(vb, w_pb);
      } else {
#pragma unroll
        for (int r = 1; r < RL; ++r) {
          va[r] = cmul(va[r], stw[(r * ja) & (NT - 1)]);
          vb[r] = cmul(vb[r], stw[(r * jb) & (NT - 1)]);
        }
      }
      DFT<RL, +1>::run(va);
      DFT<RL, +1>::run(vb);
      const double2 Ep = aux[ps];
      pair_divide<NT, RL, K1Form<NL>::BDF, K1Form<NL>::CX>(va, vb, pj == 0, stw, ja, jb, a.a1 * Ep.x,
                                                           a.a1 * Ep.y, hin);
      DFT<RL, -1>::run(va);
      DFT<RL, -1>::run(vb);
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        pout[(ja * RL + r) * S + ps] = va[r];
        pout[(jb * RL + r) * S + ps] = vb[r];
      }
    }
    // last generic-proxy writes into the stage (buf0 aliases its N-hat block): order them
    // before the next TMA write into the stage (the later accesses are reads)
    if constexpr (PL::ALIAS) fence_proxy_async_smem();
    __syncthreads();
    if constexpr (L == 3) {
      if constexpr (PW) tstage_pw<NT, S, THREADS, C::R1, RL, -1>(buf0, buf1, w_im);
      else tstage<NT, S, THREADS, C::R1, RL, -1>(buf0, buf1, stw);
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) y[r] = buf1[(j + r * TPS) * S + s];
    if constexpr (PW) {
      twpow_mul<R0, -1>(y, w_c);
    } else {
#pragma unroll
      for (int r = 1; r < R0; ++r) y[r] = cmulc(y[r], stw[(r * j) & (NT - 1)]);
    }
    DFT<R0, -1>::run(y);
    // ---- phase C: Gamma_alpha^{-1}, update (u_t from the staged tile), store ------------
    if (valid) {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int t = j + r * TPS;
        double2 sv = cscale(y[r], sgi[t]);
        if constexpr (OUTM == OUT_UPDATE) sv = cadd(xv[r], sv);
        EXPD_CHECK(base >= 0 && base + 1 < npad && t < NT, "K1: store index");
        st2(a.Y + (long)t * npad + base, sv);
      }
    }
    __syncthreads();  // every read of the stage is done: it may be refilled by TMA
    if constexpr (NST == 1) {
      if (next < ntiles) tma_tile_issue<NT, THR, RM, NL, NST>(&mx, &mn, a, next, smem, &bar[0]);
    }
  }

  if (a.partial) {
    __shared__ double red[THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if ((tid & 31) == 0) red[tid >> 5] = nrm;
    __syncthreads();
    if (tid < 32) {
      double v = tid < THREADS / 32 ? red[tid] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (tid == 0) a.partial[blockIdx.x] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K1 "ring" variant (EXPD_K1V = 5123, the default for Nt = 128 / 256): one persistent CTA of
// TWO 256-thread warp groups per SM sharing a ring of THREE staged tiles.  Each group runs the
// same per-tile pipeline as k_time_tma (phase A, the Stockham stages, the Hermitian-pair
// divide, phase C) on every other tile of the CTA's sequence, synchronising on its own named
// barrier, so two tiles are transformed at once (16 warps per SM instead of 8: the latency
// that left k_time_tma issue-bound at 25 %) while the third buffer streams in.  A group that
// finishes tile i refills the tile's buffer with tile i + 3 (TMA tensor boxes for U-hat /
// N-hat, 1-D bulk copies for the per-mode tables, all on the buffer's mbarrier).  FFT scratch
// lives inside the tile's own buffer after phase A has read it (u_t stays in registers for the
// update): N-hat block and U-hat block (nonlinear forms), U-hat block and a per-group buffer
// (linear forms).  Requires npairs % S == 0 (full tiles).
// ---------------------------------------------------------------------------------------
// the plans with one job per thread in the first and partner stages of a 256-thread group
// and one or two in the middle stages (Nt = 256: 8 x 8 x 4, one; Nt = 128: 8 x 4 x 4, two,
// whose twiddles coincide)
template <int NT>
constexpr int ring_mid_jobs() {
  using G = TGeo<NT, 256>;
  return G::S * (NT / TimeCfg<NT>::R1) / 256;
}
template <int NT>
constexpr bool ring_capable() {
  using G = TGeo<NT, 256>;
  constexpr int jm = ring_mid_jobs<NT>();
  // two-stage plans (Nt = 16 / 32 / 64): one stage-0 job per thread, at most one partner job
  if (G::L == 2) return G::S * G::TPS == 256 && G::S * (G::NSL / 2) <= 256;
  return G::L == 3 && G::S * G::TPS == 256 && (jm == 1 || jm == 2) && G::S * (NT / TimeCfg<NT>::R1) == 256 * jm &&
         G::S * (G::NSL / 2) == 256 && (jm == 1 || ((256 / G::S) % G::R0 == 0 && (256 / G::S) % G::RL == 0));
}

template <int NT, int NL>
struct RingLayout {
  using G = TGeo<NT, 256>;
  static constexpr int S = G::S;
  static constexpr int TILE = NT * S;                      // double2 per staged array
  static constexpr int NARR = 1 + (K1Form<NL>::HASN ? 1 : 0);
  static constexpr int AUX = 4 * S;                        // E, C1, C2, u0-hat per pair
  static constexpr int STAGE = ((NARR * TILE + AUX) + 7) / 8 * 8;
  static constexpr int NBUF = 3;
  static constexpr int XBUF = K1Form<NL>::HASN ? 0 : TILE;  // per-group FFT buffer (linear forms)
  static constexpr size_t BYTES =
      128 + sizeof(double2) * ((size_t)NBUF * STAGE + 2 * XBUF + NT) + sizeof(double) * 2 * NT + 8 * NBUF + 16;
};

template <int NT, int RM, int NL>
__device__ __forceinline__ void ring_issue(const CUtensorMap* mx, const CUtensorMap* mn, const TimeArgs& a,
                                           long tile, double2* stage, uint64_t* bar) {
  using PL = RingLayout<NT, NL>;
  constexpr int S = PL::S, TILE = PL::TILE;
  constexpr uint32_t AUXB = 16 * S;
  constexpr int NAUX = 1 + (K1Form<NL>::HASN ? 1 : 0) + (NL == 2 ? 1 : 0) + (RM == RM_RESID ? 1 : 0);
  mbar_arrive_expect_tx(bar, (uint32_t)(PL::NARR * TILE * 16) + NAUX * AUXB);
  tma_load_2d(stage, mx, bar, (int)(2 * S * tile), 0);
  if constexpr (K1Form<NL>::HASN) tma_load_2d(stage + TILE, mn, bar, (int)(2 * S * tile), 0);
  double2* aux = stage + PL::NARR * TILE;
  const long off = 2 * S * tile;  // doubles
  bulk_load_1d(aux, a.E + off, AUXB, bar);
  if constexpr (K1Form<NL>::HASN) bulk_load_1d(aux + S, a.C1 + off, AUXB, bar);
  if constexpr (NL == 2) bulk_load_1d(aux + 2 * S, a.C2 + off, AUXB, bar);
  if constexpr (RM == RM_RESID) bulk_load_1d(aux + 3 * S, a.u0h + off, AUXB, bar);
}

template <int NT, int RM, int OUTM, int NL>
__global__ void __launch_bounds__(512, 1)
    k_time_ring(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mn,
                const __grid_constant__ TimeArgs a) {
  using G = TGeo<NT, 256>;
  using C = TimeCfg<NT>;
  using PL = RingLayout<NT, NL>;
  constexpr int L = G::L, R0 = G::R0, RL = G::RL, TPS = G::TPS, S = G::S, GT = 256;
  constexpr int NSL = G::NSL, TILE = PL::TILE, NBUF = PL::NBUF;
  static_assert(ring_capable<NT>(), "ring kernel: one job per thread outside the middle stages");
  constexpr int JM = ring_mid_jobs<NT>();
  extern __shared__ unsigned char rsm_raw[];
  double2* smem = reinterpret_cast<double2*>(rsm_raw + ((128u - (smem_u32(rsm_raw) & 127u)) & 127u));
  double2* xbuf = smem + NBUF * PL::STAGE;             // [2][XBUF] (linear forms)
  double2* stw = xbuf + 2 * PL::XBUF;                  // [NT] e^{+2 pi i q/NT}
  double* sg = reinterpret_cast<double*>(stw + NT);    // [NT] alpha^{t/NT}
  double* sgi = sg + NT;                               // [NT] alpha^{-t/NT}
  uint64_t* full = reinterpret_cast<uint64_t*>(sgi + NT);

  const int grp = threadIdx.x / GT;
  const int tid = threadIdx.x % GT;
  for (int i = threadIdx.x; i < NT; i += 2 * GT) {
    stw[i] = a.tw[i];
    sg[i] = a.g[i];
    sgi[i] = a.ginv[i];
  }
  const long ntiles = a.npairs / S;
  if (threadIdx.x == 0) {
    prefetch_tmap(&mx);
    if constexpr (K1Form<NL>::HASN) prefetch_tmap(&mn);
    for (int k = 0; k < NBUF; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
    for (int k = 0; k < NBUF; ++k) {
      const long t = blockIdx.x + (long)k * gridDim.x;
      if (t < ntiles) ring_issue<NT, RM, NL>(&mx, &mn, a, t, smem + k * PL::STAGE, &full[k]);
    }
  }
  __syncthreads();
  const double hin = a.half_inv_nt;
  double nrm = 0.0;
  const int s = tid % S;
  const int j = tid / S;
  const long npad = a.npad;
  const int pj = tid / S;
  // this thread's base twiddles, re-read from shared memory where used (an opaque copy of
  // the table pointer keeps the compiler from holding all five in registers for the loop)
  const int i_fm = ((j % R0) * (NT / (R0 * C::R1))) & (NT - 1);
  const int i_im = ((j % RL) * (NT / (RL * C::R1))) & (NT - 1);
  const int i_pa = pj & (NT - 1);
  const int i_pb = (pj == 0 ? NSL / 2 : NSL - pj) & (NT - 1);
  const int i_c = j & (NT - 1);
  const int barid = 1 + grp;

  for (long i = grp;; i += 2) {
    const long tile = blockIdx.x + i * gridDim.x;
    if (tile >= ntiles) break;
    const int b = (int)(i % NBUF);
    double2* stg = smem + b * PL::STAGE;
    mbar_wait(&full[b], (uint32_t)((i / NBUF) & 1));
    const double2* X = stg;
    const double2* NH = stg + TILE;
    const double2* aux = stg + PL::NARR * TILE;
    double2* buf0 = K1Form<NL>::HASN ? stg + TILE : stg;            // after phase A
    double2* buf1 = K1Form<NL>::HASN ? stg : xbuf + grp * PL::XBUF;
    const long pair = tile * S + s;
    const long base = 2 * pair;
    // an opaque zero OFFSET (not an opaque pointer, which would lose the shared address
    // space and turn the five twiddle reads into generic LD.E)
#ifdef EXPD_RING_GENERIC_TW  // A/B: the former opaque pointer
    const double2* tw = stw;
    asm volatile("" : "+l"(tw));
#else
    int two = 0;
    asm volatile("" : "+r"(two));
    const double2* tw = stw + two;
#endif

    // ---- phase A: residual (+ ||r||^2), Gamma_alpha, forward stage 0 -------------------
    double2 y[R0];
    double2 xv[OUTM == OUT_UPDATE ? R0 : 1];
    const double2 Ej = aux[s];
    const double2 c1 = K1Form<NL>::HASN ? aux[S + s] : make_double2(0.0, 0.0);
    const double2 c2 = NL == 2 ? aux[2 * S + s] : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      const double2 xc = X[t * S + s];
      if constexpr (OUTM == OUT_UPDATE) xv[r] = xc;
      double2 rr;
      if constexpr (RM == RM_INPUT) {
        rr = xc;
      } else if constexpr (K1Form<NL>::BDF) {
        const double2 zero = make_double2(0.0, 0.0);
        const double2 xm1 = t >= 1 ? X[(t - 1) * S + s] : zero;
        const double2 xm2 = t >= 2 ? X[(t - 2) * S + s] : zero;
        const double2 u0 = RM == RM_RESID ? aux[3 * S + s] : zero;
        rr = bdf2_form<RM == RM_RESID, K1Form<NL>::CX>(Ej, xc, xm1, xm2, u0, t);
      } else {
        const double2 prev = t > 0 ? X[(t - 1) * S + s] : (RM == RM_RESID ? aux[3 * S + s] : make_double2(0.0, 0.0));
        if constexpr (K1Form<NL>::CX) {
          const double2 ep = cmul(Ej, prev);
          rr = RM == RM_RESID ? csub(ep, xc) : csub(xc, ep);
        } else if constexpr (RM == RM_RESID) {
          rr = make_double2(fma(Ej.x, prev.x, -xc.x), fma(Ej.y, prev.y, -xc.y));
          if constexpr (K1Form<NL>::HASN) {
            const double2 nm1 = NH[t * S + s];
            rr.x = fma(c1.x, nm1.x, rr.x);
            rr.y = fma(c1.y, nm1.y, rr.y);
            if constexpr (NL == 2) {
              const double2 nm2 = NH[(t > 0 ? t - 1 : 0) * S + s];
              rr.x = fma(-c2.x, nm2.x, rr.x);
              rr.y = fma(-c2.y, nm2.y, rr.y);
            }
          }
        } else {  // RM_QOP
          rr = make_double2(fma(-Ej.x, prev.x, xc.x), fma(-Ej.y, prev.y, xc.y));
        }
      }
      nrm = fma(rr.x, rr.x, fma(rr.y, rr.y, nrm));
      y[r] = cscale(rr, sg[t]);
    }
    DFT<R0, +1>::run(y);
    named_bar(barid, GT);  // the group is done reading the tile (U-hat, N-hat)
#pragma unroll
    for (int r = 0; r < R0; ++r) buf0[(j * R0 + r) * S + s] = y[r];
    named_bar(barid, GT);
    // three-stage plans: the forward middle stage buf0 -> buf1, the partner stage reads buf1
    // and writes buf0; two-stage plans: the partner stage reads buf0 and writes buf1
    double2* pin = buf0;
    double2* pout = buf1;
    if constexpr (L == 3) {
      tstage_pw<NT, S, GT, C::R1, R0, +1, JM>(buf0, buf1, tw[i_fm], tid);
      named_bar(barid, GT);
      pin = buf1;
      pout = buf0;
    }
    if (S * (NSL / 2) == GT || pj < NSL / 2) {
      const int ps = s;
      const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
      double2 va[RL], vb[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        va[r] = pin[(ja + r * NSL) * S + ps];
        vb[r] = pin[(jb + r * NSL) * S + ps];
      }
      twpow_mul<RL, +1>(va, tw[i_pa]);
      twpow_mul<RL, +1>(vb, tw[i_pb]);
      DFT<RL, +1>::run(va);
      DFT<RL, +1>::run(vb);
      // one partner job per thread: its pair is this thread's pair s (Ej)
      pair_divide<NT, RL, K1Form<NL>::BDF, K1Form<NL>::CX>(va, vb, pj == 0, stw, ja, jb, a.a1 * Ej.x, a.a1 * Ej.y,
                                                           hin);
      DFT<RL, -1>::run(va);
      DFT<RL, -1>::run(vb);
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        pout[(ja * RL + r) * S + ps] = va[r];
        pout[(jb * RL + r) * S + ps] = vb[r];
      }
    }
    named_bar(barid, GT);
    if constexpr (L == 3) {
      tstage_pw<NT, S, GT, C::R1, RL, -1, JM>(buf0, buf1, tw[i_im], tid);
      named_bar(barid, GT);
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) y[r] = buf1[(j + r * TPS) * S + s];
    // every generic write into the buffer is ordered before the refill's async-proxy writes;
    // after the barrier no thread of the group reads it again.  (Releasing the buffer through
    // an `empty` mbarrier that only warp 0 waits on measured slower: K1 6.05 -> 6.26 ms.)
    fence_proxy_async_smem();
    named_bar(barid, GT);
    if (tid == 0) {
      const long nxt = blockIdx.x + (i + NBUF) * gridDim.x;
      if (nxt < ntiles) ring_issue<NT, RM, NL>(&mx, &mn, a, nxt, stg, &full[b]);
    }
    twpow_mul<R0, -1>(y, tw[i_c]);
    DFT<R0, -1>::run(y);
    // ---- phase C: Gamma_alpha^{-1}, update, store ----------------------------------------
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      double2 sv = cscale(y[r], sgi[t]);
      if constexpr (OUTM == OUT_UPDATE) sv = cadd(xv[r], sv);
      st2(a.Y + (long)t * npad + base, sv);
    }
  }

  if (a.partial) {
    __shared__ double red[2 * GT / 32];
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < 2 * GT / 32 ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) a.partial[blockIdx.x] = v;
    }
  }
}

template <int NT, int OUTM>
static size_t time_smem_bytes() {
  const size_t tile = TimeGeo<NT>::L > 1 ? (size_t)NT * TimeGeo<NT>::S : 0;
  return sizeof(double2) * (2 * tile + NT) + sizeof(double) * 2 * NT;
}

// EXPD_K1_PIPE: 0 = register-load kernel, 1 = double-buffered cp.async pipe (1 CTA/SM),
// 2 = single-stage cp.async pipe with two CTAs per SM, 3 (default) = TMA-fed kernel with
// the variant EXPD_K1V = <threads><stages> (e.g. 2561, 2562, 1281, 1282)
static int pipe_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EXPD_K1_PIPE");
    v = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 3;
    if (v == 3 && !tma_available()) v = 2;
  }
  return v;
}
// EXPD_K1V (read per launch, a tuning / A-B switch): 5123 the ring, 2562 / 2561 / 1282 the
// TMA kernel with <threads><stages>; 0 = automatic (use_ring, k1_variant).
static int k1_env() {
  const char* e = getenv("EXPD_K1V");
  int v = e ? atoi(e) : 0;
  return (v == 2562 || v == 1282 || v == 2561 || v == 5123 || v == 5124) ? v : 0;
}
// The TMA-kernel variant when the ring is not used: 2562 (256 threads, double-buffered tiles,
// 1 CTA/SM), 2561 (single stage, 2 CTAs/SM), 1282 (128 threads; round 1's Nt = 128 default).
// c5: 7.02 / 7.10 / 11.2 ms.
static int k1_variant(int nt) {
  const int v = k1_env();
  if (v && v != 5123) return v;
  return nt == 128 ? 1282 : 2562;
}
static bool use_pipe() { return pipe_mode() > 0; }

template <int NT, int RM, int OUTM, int NL, bool DB>
static cudaError_t launch_pipe(const TimeArgs& a, int grid, cudaStream_t st) {
  auto kp = k_time_pipe<NT, RM, OUTM, NL, DB>;
  const size_t smp = PipeLayout<NT, RM, NL, DB>::BYTES;
  static DevOnce attr_p;  // per instantiation and device
  if (cudaError_t e = smem_optin(attr_p, kp, smp); e != cudaSuccess) return e;
  kp<<<grid, TimeGeo<NT>::THREADS, smp, st>>>(a);
  return cudaGetLastError();
}

template <int NT, int RM, int OUTM, int NL, int THR, int NST>
static cudaError_t launch_tma(const TimeArgs& a, int grid, cudaStream_t st) {
  using PL = TmaLayout<NT, THR, NL, NST>;
  auto k = k_time_tma<NT, RM, OUTM, NL, THR, NST>;
  static DevOnce attr;  // per instantiation and device
  if (cudaError_t e = smem_optin(attr, k, PL::BYTES); e != cudaSuccess) return e;
  constexpr int S = PL::S;
  CUtensorMap mx, mn;
  cudaError_t e = make_tmap_2d(&mx, a.X, (unsigned long long)a.npad, (unsigned long long)a.nt,
                               (unsigned long long)a.npad * 8, 2 * S, NT);
  if (e != cudaSuccess) return e;
  mn = mx;
  if (K1Form<NL>::HASN && (e = make_tmap_2d(&mn, a.Nh, (unsigned long long)a.npad, (unsigned long long)a.nt,
                              (unsigned long long)a.npad * 8, 2 * S, NT)) != cudaSuccess)
    return e;
  // the caller's grid (time_fused_grid) is also the number of partial sums it reduces
  k<<<(unsigned)grid, THR, PL::BYTES, st>>>(mx, mn, a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// K1 warp-per-pair ring (the default for Nt = 256 Picard forms ETD1 / ETD2 / IF with residual +
// update and full tiles; EXPD_K1V = 5123 selects the ring instead): the ring above with the thread mapping turned around -- warp s of a
// 256-thread group owns mode pair s of the tile and lane j its stage-0 / middle / partner
// jobs, so every FFT exchange stays inside one warp (__syncwarp) and a tile needs two group
// barriers (tile read, result staged) instead of six.  Consequences of the mapping:
//  * the Û / N̂ tiles land with the 128-byte TMA swizzle (element (t, s) at chunk s ^ (t & 7)
//    of row t), so the lanes' reads of one pair down the time column are conflict free;
//  * warp s's FFT scratch is its own padded 4.5 KB slice of the N̂ tile plus a pad area after it
//    (free once the group has read the tile; the Û tile stays intact, so u_t is re-read for the
//    update instead of held in registers); each stage's layout (one pad slot per 8 or per 32
//    positions) and a lane -> partner-job table keep every access affine and conflict free;
//  * the result is staged into the tile's Û block (swizzled like the input: conflict free) and
//    leaves as ONE TMA store per tile (a lane-per-slice register store would touch 32 rows per
//    instruction), after which the issuing thread waits for the store to read the buffer and
//    refills it.
// Same arithmetic in the same order per mode as k_time_ring (identical results).
// ---------------------------------------------------------------------------------------
template <int NT, int NL>
struct WpLayout {
  static constexpr int S = 8;
  static constexpr int TILE = NT * S;                        // double2 per staged array
  static constexpr int AUX = 4 * S;
  static constexpr int WSLOTS = NT + NT / 8;                // a warp's scratch: 256 positions + pads
  // stage: [Û tile][N̂ tile][pad area][aux]: the warps' scratch runs from the N̂ tile into the pad
  // area (S WSLOTS = TILE + S NT/8 slots), so the Û tile stays intact until phase C
  static constexpr int AUXOFF = 2 * TILE + S * (NT / 8);
  static constexpr int STAGE = ((AUXOFF + AUX) + 63) / 64 * 64;  // 1 KB multiple (swizzle atoms)
  static constexpr int NBUF = 3;
  // twiddle power tables (EXPD_WP_TWTAB, default on): forward middle 7 x 8, inverse middle 7 x 4,
  // partner 3 x 72 (padded), final inverse 7 x 32
  static constexpr int TWTAB = 56 + 28 + 216 + 224;
  static constexpr size_t BYTES = 1024 + sizeof(double2) * ((size_t)NBUF * STAGE + NT + NT / 8 + TWTAB) +
                                  sizeof(double) * 2 * NT + 8 * NBUF + 16;
};

// EXPD_WP_LATE_REFILL (A/B): 0 = the refill right after the tile's store (the issuing thread
// waits for the store to read the buffer), 1 = deferred to after the group's next mbarrier
// wait, 2 = deferred to after the group's next phase-A barrier
#ifndef EXPD_WP_LATE_REFILL
#define EXPD_WP_LATE_REFILL 0
#endif
// (t, s) of a staged tile with the 128-byte swizzle: row t of 8 pairs (16-byte chunks)
__device__ __forceinline__ int wp_sw(int t, int s) { return t * 8 + (s ^ (t & 7)); }

// Lane -> partner job (ja; jb = 64 - ja, 32 for ja = 0) of the last stage: any bijection is
// valid; this one (a search over lane groupings, tools/wp_lanes.py) makes the partner reads of
// layout L2 and the partner writes of layout L3 bank-conflict free for both ja and jb.
__device__ const unsigned char kWpPj[32] = {8, 0, 25, 7, 13, 24, 16, 19, 22, 21, 2, 26, 1, 27, 10, 11,
                                            20, 30, 15, 17, 5, 4, 31, 14, 28, 3, 23, 12, 29, 9, 6, 18};

// ring_issue with the warp-per-pair stage layout (aux after the pad area)
template <int NT, int RM, int NL>
__device__ __forceinline__ void wp_issue(const CUtensorMap* mx, const CUtensorMap* mn, const TimeArgs& a, long tile,
                                         double2* stage, uint64_t* bar) {
  using PL = WpLayout<NT, NL>;
  constexpr int S = PL::S, TILE = PL::TILE;
  constexpr uint32_t AUXB = 16 * S;
  constexpr int NAUX = 2 + (NL == 2 ? 1 : 0) + 1;  // E, C1, (C2), u0-hat
  mbar_arrive_expect_tx(bar, (uint32_t)(2 * TILE * 16) + NAUX * AUXB);
  tma_load_2d(stage, mx, bar, (int)(2 * S * tile), 0);
  tma_load_2d(stage + TILE, mn, bar, (int)(2 * S * tile), 0);
  double2* aux = stage + PL::AUXOFF;
  const long off = 2 * S * tile;  // doubles
  bulk_load_1d(aux, a.E + off, AUXB, bar);
  bulk_load_1d(aux + S, a.C1 + off, AUXB, bar);
  if constexpr (NL == 2) bulk_load_1d(aux + 2 * S, a.C2 + off, AUXB, bar);
  bulk_load_1d(aux + 3 * S, a.u0h + off, AUXB, bar);
}

template <int NT, int RM, int OUTM, int NL>
__global__ void __launch_bounds__(512, 1)
    k_time_wp(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mn,
              const __grid_constant__ CUtensorMap my, const __grid_constant__ TimeArgs a) {
  static_assert(NT == 256 && (NL == 1 || NL == 2) && RM == RM_RESID && OUTM == OUT_UPDATE,
                "warp-per-pair K1: Nt = 256, Picard residual + update");
  using C = TimeCfg<NT>;
  using PL = WpLayout<NT, NL>;
  constexpr int R0 = C::R0, R1 = C::R1, RL = C::R2, TPS = NT / R0, S = PL::S, GT = 256;
  constexpr int NSL = NT / RL, TILE = PL::TILE, NBUF = PL::NBUF, WS = PL::WSLOTS;
  static_assert(R0 == 8 && R1 == 8 && RL == 4 && TPS == 32 && NSL / 2 == 32, "plan 8 x 8 x 4, one job per lane");
  static_assert(TILE + S * WS <= PL::AUXOFF, "the warps' scratch fits the N-hat tile and the pad area");
  static_assert(PL::BYTES + 2 * 256 / 32 * 8 <= 232448, "shared memory");
  extern __shared__ unsigned char wsm_raw[];
  double2* smem = reinterpret_cast<double2*>(wsm_raw + ((1024u - (smem_u32(wsm_raw) & 1023u)) & 1023u));
  double2* stwp = smem + NBUF * PL::STAGE;             // [NT + NT/8] e^{+2 pi i q/NT} padded (slot q + q/8)
  double2* ttab = stwp + NT + NT / 8;                  // [TWTAB] twiddle powers (see below)
  double* sg = reinterpret_cast<double*>(ttab + PL::TWTAB);  // [NT] alpha^{t/NT}
  double* sgi = sg + NT;                               // [NT] alpha^{-t/NT}
  uint64_t* full = reinterpret_cast<uint64_t*>(sgi + NT);

  const int grp = threadIdx.x / GT;
  const int tid = threadIdx.x % GT;
  for (int i = threadIdx.x; i < NT; i += 2 * GT) {
    stwp[i + (i >> 3)] = a.tw[i];
    sg[i] = a.g[i];
    sgi[i] = a.ginv[i];
  }
  // the stages' twiddle powers w^r = e^{2 pi i k r / NT} straight from the table (one rounding,
  // no products; K1-wp is fp64-issue bound and its shared memory has slack): FM[r-1][c]
  // (forward middle, k = 4c), IM[r-1][c] (inverse middle, k = 8c), PA[r-1][x + x/8] (partner
  // job x < 64, padded like stwp), FC[r-1][j] (final inverse stage, k = j)
  for (int q = threadIdx.x; q < PL::TWTAB; q += 2 * GT) {
    int e;
    if (q < 56) e = 4 * (q & 7) * (q / 8 + 1);
    else if (q < 84) e = 8 * ((q - 56) & 3) * ((q - 56) / 4 + 1);
    else if (q < 300) {
      const int r = (q - 84) / 72 + 1, y = (q - 84) % 72;  // y = x + x/8 for x < 64 (pads: y % 9 == 8)
      e = (y % 9 == 8) ? 0 : (y / 9 * 8 + y % 9) * r;
    } else e = ((q - 300) & 31) * ((q - 300) / 32 + 1);
    ttab[q] = a.tw[e & (NT - 1)];
  }
  const long ntiles = a.npairs / S;
  if (threadIdx.x == 0) {
    prefetch_tmap(&mx);
    prefetch_tmap(&mn);
    prefetch_tmap(&my);
    for (int k = 0; k < NBUF; ++k) mbar_init(&full[k], 1);
    mbar_fence_init();
    for (int k = 0; k < NBUF; ++k) {
      const long t = blockIdx.x + (long)k * gridDim.x;
      if (t < ntiles) wp_issue<NT, RM, NL>(&mx, &mn, a, t, smem + k * PL::STAGE, &full[k]);
    }
  }
  __syncthreads();
  const double hin = a.half_inv_nt;
  double nrm = 0.0;
  const int s = tid >> 5;   // this warp's mode pair
  const int j = tid & 31;   // lane: stage-0 / middle job
  const int ja = kWpPj[j];  // partner jobs
  const int jb = ja == 0 ? NSL / 2 : NSL - ja;
  const int barid = 1 + grp;
  long pend_nxt = -1;  // EXPD_WP_LATE_REFILL: the refill this group's thread 0 still owes
  int pend_b = 0;
  // scratch layouts (16-byte slots of the warp's region): L1 / L2 / L4 one pad slot per 8
  // positions (p + p/8), L3 one per 32 (p + p/32); every stage's reads and writes are
  // affine in r with a per-lane base and hit eight distinct bank groups per quarter warp
  const int l1w = 9 * j;                                   // stage-0 write  (p = 8j + r)
  const int lrd = j + (j >> 3);                            // reads p = j + 32r (L1, L4): + 36r
  const int l2w = (j >> 3) * 72 + (j & 7);                 // forward middle write: + 9r
  const int l2a = ja + (ja >> 3), l2b = jb + (jb >> 3);    // partner reads: + 72r
  const int l3a = 4 * ja + (ja >> 3), l3b = 4 * jb + (jb >> 3);  // partner writes: + r
  const int l4w = (j >> 2) * 36 + (j & 3);                 // inverse middle write: + 4r + r/2

  for (long i = grp;; i += 2) {
    const long tile = blockIdx.x + i * gridDim.x;
    if (tile >= ntiles) break;
    const int b = (int)(i % NBUF);
    double2* stg = smem + b * PL::STAGE;
    mbar_wait(&full[b], (uint32_t)((i / NBUF) & 1));
    if (EXPD_WP_LATE_REFILL == 1 && tid == 0 && pend_nxt >= 0) {
      bulk_wait_read0();
      wp_issue<NT, RM, NL>(&mx, &mn, a, pend_nxt, smem + pend_b * PL::STAGE, &full[pend_b]);
      pend_nxt = -1;
    }
    double2* X = stg;                              // Û tile (swizzled); later the staged result
    const double2* NH = stg + TILE;                // N̂ tile (swizzled)
    const double2* aux = stg + PL::AUXOFF;
    double2* W = stg + TILE + s * WS;              // this warp's FFT scratch (N̂ tile + pad area)
    int two = 0;
    asm volatile("" : "+r"(two));

    // ---- phase A: residual (+ ||r||^2), Gamma_alpha, forward stage 0 -------------------
    double2 y[R0];
    const double2 Ej = aux[s];
    const double2 c1 = aux[S + s];
    const double2 c2 = NL == 2 ? aux[2 * S + s] : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      const double2 xc = X[wp_sw(t, s)];
      const double2 prev = t > 0 ? X[wp_sw(t - 1, s)] : aux[3 * S + s];
      double2 rr = make_double2(fma(Ej.x, prev.x, -xc.x), fma(Ej.y, prev.y, -xc.y));
      const double2 nm1 = NH[wp_sw(t, s)];
      rr.x = fma(c1.x, nm1.x, rr.x);
      rr.y = fma(c1.y, nm1.y, rr.y);
      if constexpr (NL == 2) {
        const double2 nm2 = NH[wp_sw(t > 0 ? t - 1 : 0, s)];
        rr.x = fma(-c2.x, nm2.x, rr.x);
        rr.y = fma(-c2.y, nm2.y, rr.y);
      }
      nrm = fma(rr.x, rr.x, fma(rr.y, rr.y, nrm));
      y[r] = cscale(rr, sg[t]);
    }
    DFT<R0, +1>::run(y);
    named_bar(barid, GT);  // the group has read the N̂ tile: it becomes the warps' scratch
    if (EXPD_WP_LATE_REFILL == 2 && tid == 0 && pend_nxt >= 0) {
      bulk_wait_read0();
      wp_issue<NT, RM, NL>(&mx, &mn, a, pend_nxt, smem + pend_b * PL::STAGE, &full[pend_b]);
      pend_nxt = -1;
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) W[l1w + r] = y[r];
    __syncwarp();
    {  // forward middle stage (radix R1, NS = R0), in place
      double2 v[R1];
#pragma unroll
      for (int r = 0; r < R1; ++r) v[r] = W[lrd + 36 * r];
#pragma unroll
      for (int r = 1; r < R1; ++r) v[r] = cmul(v[r], ttab[(r - 1) * 8 + (j & 7)]);
      DFT<R1, +1>::run(v);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R1; ++r) W[l2w + 9 * r] = v[r];
      __syncwarp();
    }
    {  // last forward stage on Hermitian partner jobs, the divide, first inverse stage
      double2 va[RL], vb[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        va[r] = W[l2a + 72 * r];
        vb[r] = W[l2b + 72 * r];
      }
      // partner twiddles and the divide's e^{2 pi i k/NT} from the padded copy: the reads at
      // q = x + 64 r hit bank (x + x/8) mod 8, distinct over a quarter warp (kWpPj)
      const double2* twp = stwp + two;
#pragma unroll
      for (int r = 1; r < RL; ++r) {
        va[r] = cmul(va[r], ttab[84 + (r - 1) * 72 + l2a]);
        vb[r] = cmul(vb[r], ttab[84 + (r - 1) * 72 + l2b]);
      }
      DFT<RL, +1>::run(va);
      DFT<RL, +1>::run(vb);
      {  // pair_divide (k_time_ring) with the padded table
        const double ba = a.a1 * Ej.x, bb = a.a1 * Ej.y;
        if (ja != 0) {
#pragma unroll
          for (int r = 0; r < RL; ++r)
            divide_pair<false>(va[r], vb[RL - 1 - r], twp[l2a + 72 * r], ba, bb, hin, false);
        } else {
          // ja = 0: frequencies NSL r, partner NSL (RL - r) mod RL; self at r = 0 and RL/2;
          // jb = NSL/2: frequencies NSL/2 + NSL r, partner index RL-1-r
          divide_pair<false>(va[0], va[0], twp[0], ba, bb, hin, true);
#pragma unroll
          for (int r = 1; r < (RL + 1) / 2; ++r)
            divide_pair<false>(va[r], va[RL - r], twp[72 * r], ba, bb, hin, false);
          divide_pair<false>(va[RL / 2], va[RL / 2], twp[72 * (RL / 2)], ba, bb, hin, true);
#pragma unroll
          for (int r = 0; r < RL / 2; ++r)
            divide_pair<false>(vb[r], vb[RL - 1 - r], twp[l2b + 72 * r], ba, bb, hin, false);
        }
      }
      DFT<RL, -1>::run(va);
      DFT<RL, -1>::run(vb);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        W[l3a + r] = va[r];
        W[l3b + r] = vb[r];
      }
      __syncwarp();
    }
    {  // inverse middle stage (radix R1, NS = RL), in place
      double2 v[R1];
#pragma unroll
      for (int r = 0; r < R1; ++r) v[r] = W[j + 33 * r];
#pragma unroll
      for (int r = 1; r < R1; ++r) v[r] = cmulc(v[r], ttab[56 + (r - 1) * 4 + (j & 3)]);
      DFT<R1, -1>::run(v);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R1; ++r) W[l4w + 4 * r + (r >> 1)] = v[r];
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < R0; ++r) y[r] = W[lrd + 36 * r];
#pragma unroll
    for (int r = 1; r < R0; ++r) y[r] = cmulc(y[r], ttab[300 + (r - 1) * 32 + j]);
    DFT<R0, -1>::run(y);
    // ---- phase C: Gamma_alpha^{-1}, update, staged into the Û block, one TMA store ------
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int t = j + r * TPS;
      const int q = wp_sw(t, s);
      X[q] = cadd(X[q], cscale(y[r], sgi[t]));  // u_t re-read from the intact Û tile
    }
    fence_proxy_async_smem();
    named_bar(barid, GT);
    if (tid == 0) {
      tma_store_2d(&my, X, (int)(2 * S * tile), 0);
      bulk_commit();
      const long nxt = blockIdx.x + (i + NBUF) * gridDim.x;
      if (nxt < ntiles) {
        if (EXPD_WP_LATE_REFILL) {
          pend_nxt = nxt;
          pend_b = b;
        } else {
          bulk_wait_read0();  // the store has read the staged result: refill the buffer
          wp_issue<NT, RM, NL>(&mx, &mn, a, nxt, stg, &full[b]);
        }
      }
    }
  }
  if (tid == 0 && pend_nxt >= 0) {  // a refill another group's tile still needs
    bulk_wait_read0();
    wp_issue<NT, RM, NL>(&mx, &mn, a, pend_nxt, smem + pend_b * PL::STAGE, &full[pend_b]);
  }
  if (tid == 0) bulk_wait0();

  if (a.partial) {
    __shared__ double red[2 * GT / 32];
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x < 32) {
      double v = threadIdx.x < 2 * GT / 32 ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) a.partial[blockIdx.x] = v;
    }
  }
}

template <int NT, int RM, int OUTM, int NL>
static cudaError_t launch_wp(const TimeArgs& a, int grid, cudaStream_t st) {
  using PL = WpLayout<NT, NL>;
  auto k = k_time_wp<NT, RM, OUTM, NL>;
  static DevOnce attr;  // per instantiation and device
  if (cudaError_t e = smem_optin(attr, k, PL::BYTES); e != cudaSuccess) return e;
  constexpr int S = PL::S;
  CUtensorMap mx, mn, my;
  const unsigned long long np = (unsigned long long)a.npad, nt = (unsigned long long)a.nt, rb = np * 8;
  cudaError_t e = make_tmap_2d(&mx, a.X, np, nt, rb, 2 * S, NT, true);
  if (e == cudaSuccess) e = make_tmap_2d(&mn, a.Nh, np, nt, rb, 2 * S, NT, true);
  if (e == cudaSuccess) e = make_tmap_2d(&my, a.Y, np, nt, rb, 2 * S, NT, true);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)grid, 512, PL::BYTES, st>>>(mx, mn, my, a);
  return cudaGetLastError();
}

template <int NT, int RM, int OUTM, int NL>
static cudaError_t launch_ring(const TimeArgs& a, int grid, cudaStream_t st) {
  using PL = RingLayout<NT, NL>;
  auto k = k_time_ring<NT, RM, OUTM, NL>;
  static DevOnce attr;  // per instantiation and device
  if (cudaError_t e = smem_optin(attr, k, PL::BYTES); e != cudaSuccess) return e;
  constexpr int S = PL::S;
  CUtensorMap mx, mn;
  cudaError_t e = make_tmap_2d(&mx, a.X, (unsigned long long)a.npad, (unsigned long long)a.nt,
                               (unsigned long long)a.npad * 8, 2 * S, NT);
  if (e != cudaSuccess) return e;
  mn = mx;
  if (K1Form<NL>::HASN && (e = make_tmap_2d(&mn, a.Nh, (unsigned long long)a.npad, (unsigned long long)a.nt,
                              (unsigned long long)a.npad * 8, 2 * S, NT)) != cudaSuccess)
    return e;
  k<<<(unsigned)grid, 512, PL::BYTES, st>>>(mx, mn, a);
  return cudaGetLastError();
}
// the ring kernel takes full tiles only
template <int NT>
static bool ring_ok(long npairs) {
  if constexpr (ring_capable<NT>()) return npairs % RingLayout<NT, 1>::S == 0;
  return false;
}
static long k1_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
  return n[dev] > 0 ? n[dev] : 148;
}
// The ring (one CTA of two warp groups per SM) or the TMA kernel, measured per plan shape:
// Nt = 128 / 256 always (c5 K1 6.69 -> 6.02 ms, c3 0.184 -> 0.167, c7se 1.124 -> 1.115 against
// 1282, profiles/r02/k1_ring128_ab.txt); the two-stage plans (Nt = 16 / 32 / 64) only with at
// least 16 tiles per SM (c4 GMRES steps 18.66 -> 18.09 ms; c2's 1020 tiles: 0.030 -> 0.033 ms,
// too few to fill the persistent grid; profiles/r02/k1_ring64_ab.txt).  Partial tiles: TMA.
template <int NT>
static bool use_ring(long npairs) {
  if constexpr (!ring_capable<NT>()) {
    return false;
  } else {
    if (pipe_mode() != 3 || !ring_ok<NT>(npairs)) return false;
    const int v = k1_env();
    if (v) return v == 5123;
    if (NT >= 128) return true;
    return npairs / RingLayout<NT, 1>::S >= 16L * k1_sms();
  }
}

// the warp-per-pair K1 (the default for Nt = 256 Picard sweeps with full tiles; EXPD_K1V=5123
// forces the ring, profiles/r02/k1_wp_ab.txt)
template <int NT, int RM, int OUTM, int NL>
static bool use_wp(long npairs) {
  if constexpr (NT == 256 && (NL == 1 || NL == 2) && RM == RM_RESID && OUTM == OUT_UPDATE) {
    const int v = k1_env();
    return pipe_mode() == 3 && npairs % WpLayout<NT, NL>::S == 0 && (v == 0 || v == 5124);
  } else {
    return false;
  }
}

template <int NT, int RM, int OUTM, int NL>
static cudaError_t launch_t(const TimeArgs& a, int grid, cudaStream_t st) {
  if constexpr (NT == 256 && (NL == 1 || NL == 2) && RM == RM_RESID && OUTM == OUT_UPDATE) {
    if (use_wp<NT, RM, OUTM, NL>(a.npairs)) return launch_wp<NT, RM, OUTM, NL>(a, grid, st);
  }
  if constexpr (ring_capable<NT>()) {
    if (use_ring<NT>(a.npairs)) return launch_ring<NT, RM, OUTM, NL>(a, grid, st);
  }
  if constexpr (TimeGeo<NT>::L > 1 && NL >= 3) {  // BDF2 / complex: TMA or register kernel
    if (pipe_mode() == 3) {
      if (k1_variant(NT) == 1282) return launch_tma<NT, RM, OUTM, NL, 128, 2>(a, grid, st);
      if (k1_variant(NT) == 2561) return launch_tma<NT, RM, OUTM, NL, 256, 1>(a, grid, st);
      return launch_tma<NT, RM, OUTM, NL, 256, 2>(a, grid, st);
    }
  } else if constexpr (TimeGeo<NT>::L > 1) {
    if (pipe_mode() == 3) {
      if (k1_variant(NT) == 1282) return launch_tma<NT, RM, OUTM, NL, 128, 2>(a, grid, st);
      if (k1_variant(NT) == 2561) return launch_tma<NT, RM, OUTM, NL, 256, 1>(a, grid, st);
      return launch_tma<NT, RM, OUTM, NL, 256, 2>(a, grid, st);
    }
    if (pipe_mode() == 1) return launch_pipe<NT, RM, OUTM, NL, true>(a, grid, st);
    if (pipe_mode() == 2) return launch_pipe<NT, RM, OUTM, NL, false>(a, grid, st);
  }
  auto k = k_time_fused<NT, RM, OUTM, NL>;
  size_t sm = time_smem_bytes<NT, OUTM>();
  static DevOnce attr_done;  // per instantiation and device
  if (cudaError_t e = smem_optin(attr_done, k, sm); e != cudaSuccess) return e;
  k<<<grid, TimeGeo<NT>::THREADS, sm, st>>>(a);
  return cudaGetLastError();
}

template <int NT>
static cudaError_t dispatch_nt(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st) {
  if (nl == 3) {  // BDF2 system (linear)
    if (rm == RM_RESID && om == OUT_UPDATE) return launch_t<NT, RM_RESID, OUT_UPDATE, 3>(a, grid, st);
    if (rm == RM_RESID && om == OUT_S) return launch_t<NT, RM_RESID, OUT_S, 3>(a, grid, st);
    if (rm == RM_INPUT && om == OUT_S) return launch_t<NT, RM_INPUT, OUT_S, 3>(a, grid, st);
    if (rm == RM_QOP && om == OUT_S) return launch_t<NT, RM_QOP, OUT_S, 3>(a, grid, st);
    return cudaErrorInvalidValue;
  }
  if (nl == 4) {  // complex coefficients (linear)
    if (rm == RM_RESID && om == OUT_UPDATE) return launch_t<NT, RM_RESID, OUT_UPDATE, 4>(a, grid, st);
    if (rm == RM_RESID && om == OUT_S) return launch_t<NT, RM_RESID, OUT_S, 4>(a, grid, st);
    if (rm == RM_INPUT && om == OUT_S) return launch_t<NT, RM_INPUT, OUT_S, 4>(a, grid, st);
    if (rm == RM_QOP && om == OUT_S) return launch_t<NT, RM_QOP, OUT_S, 4>(a, grid, st);
    return cudaErrorInvalidValue;
  }
  if (nl == 5) {  // complex BDF2 system
    if (rm == RM_RESID && om == OUT_UPDATE) return launch_t<NT, RM_RESID, OUT_UPDATE, 5>(a, grid, st);
    if (rm == RM_RESID && om == OUT_S) return launch_t<NT, RM_RESID, OUT_S, 5>(a, grid, st);
    if (rm == RM_INPUT && om == OUT_S) return launch_t<NT, RM_INPUT, OUT_S, 5>(a, grid, st);
    if (rm == RM_QOP && om == OUT_S) return launch_t<NT, RM_QOP, OUT_S, 5>(a, grid, st);
    return cudaErrorInvalidValue;
  }
  if (rm == RM_RESID && om == OUT_UPDATE) {
    if (nl == 0) return launch_t<NT, RM_RESID, OUT_UPDATE, 0>(a, grid, st);
    if (nl == 1) return launch_t<NT, RM_RESID, OUT_UPDATE, 1>(a, grid, st);
    return launch_t<NT, RM_RESID, OUT_UPDATE, 2>(a, grid, st);
  }
  if (rm == RM_RESID && om == OUT_S) {
    if (nl == 0) return launch_t<NT, RM_RESID, OUT_S, 0>(a, grid, st);
    if (nl == 1) return launch_t<NT, RM_RESID, OUT_S, 1>(a, grid, st);
    return launch_t<NT, RM_RESID, OUT_S, 2>(a, grid, st);
  }
  if (rm == RM_INPUT && om == OUT_S) return launch_t<NT, RM_INPUT, OUT_S, 0>(a, grid, st);
  if (rm == RM_QOP && om == OUT_S) return launch_t<NT, RM_QOP, OUT_S, 0>(a, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace expd
