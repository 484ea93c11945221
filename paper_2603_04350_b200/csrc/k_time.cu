// k_time.cu -- K1, the time-local fused pass of one Exp-ParaDiag sweep (sm_100a, fp64).
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
#include "expd_internal.h"
#include "fft_dev.cuh"

namespace expd {

template <int NT>
struct TimeCfg;
// P x Q = NT; S mode pairs per CTA; MINB resident CTAs per SM (register budget)
template <> struct TimeCfg<4>   { static constexpr int P = 4,  Q = 1,  S = 128, MINB = 3; };
template <> struct TimeCfg<8>   { static constexpr int P = 8,  Q = 1,  S = 128, MINB = 3; };
template <> struct TimeCfg<16>  { static constexpr int P = 16, Q = 1,  S = 128, MINB = 3; };
template <> struct TimeCfg<32>  { static constexpr int P = 8,  Q = 4,  S = 32,  MINB = 3; };
template <> struct TimeCfg<64>  { static constexpr int P = 8,  Q = 8,  S = 16,  MINB = 3; };
template <> struct TimeCfg<128> { static constexpr int P = 16, Q = 8,  S = 16,  MINB = 3; };
template <> struct TimeCfg<256> { static constexpr int P = 16, Q = 16, S = 8,   MINB = 2; };

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

// W_k = A Z_k + B conj(Z_kp),  W_kp = conj(A) Z_kp + conj(B) conj(Z_k)
// with A = (da + db)/2, B = (da - db)/2 for the two modes of the pair (Hermitian unpack,
// divide, repack in one step).  tw = e^{2 pi i k/Nt}.
__device__ __forceinline__ void divide_pair(double2& Zk, double2& Zkp, double2 tw, double ba, double bb,
                                            double hin, bool self) {
  double2 da = half_divisor(ba, tw.x, tw.y, hin);
  double2 db = half_divisor(bb, tw.x, tw.y, hin);
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

template <int NT, int RM, int OUTM, int NL>
__global__ void __launch_bounds__(TimeCfg<NT>::S * TimeCfg<NT>::Q, TimeCfg<NT>::MINB)
    k_time_fused(const TimeArgs a) {
  constexpr int P = TimeCfg<NT>::P, Q = TimeCfg<NT>::Q, S = TimeCfg<NT>::S;
  constexpr int THREADS = S * Q;
  constexpr int NSTASH = (OUTM == OUT_UPDATE) ? NT * S : 0;
  static_assert(P * Q == NT, "cfg");
  extern __shared__ double2 smem[];
  double2* buf = smem;                    // [NT][S]   (index (k1*Q + m2)*S + s)
  double2* stash = smem + NT * S;         // [NT][S]   u_t of the tile (update mode)
  double2* stw = smem + NT * S + NSTASH;  // [NT]      twiddles
  double* sg = reinterpret_cast<double*>(stw + NT);  // [NT] gamma
  double* sgi = sg + NT;                  // [NT] gamma^{-1}

  const int tid = threadIdx.x;
  for (int i = tid; i < NT; i += THREADS) {
    stw[i] = a.tw[i];
    sg[i] = a.g[i];
    sgi[i] = a.ginv[i];
  }
  __syncthreads();

  const long npad = a.npad;
  const long ntiles = (a.npairs + S - 1) / S;
  double nrm = 0.0;
  const int s = tid % S;
  const int m2 = tid / S;

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long pair = tile * S + s;
    const bool valid = pair < a.npairs;
    const long base = 2 * pair;

    // ---------------- phase A: residual, Gamma, DFT-P over m1, twiddle -----------------
    double2 y[P];
    double2 Ej = make_double2(0.0, 0.0), c1 = Ej, c2 = Ej;
    if (valid && RM != RM_INPUT) Ej = ld2(a.E + base);
    if (valid && NL >= 1) c1 = ld2(a.C1 + base);
    if (valid && NL == 2) c2 = ld2(a.C2 + base);
#pragma unroll
    for (int m1 = 0; m1 < P; ++m1) {
      const int t = Q * m1 + m2;
      double2 cur = make_double2(0.0, 0.0), r;
      if (valid) cur = (OUTM == OUT_UPDATE) ? ld2(a.X + (long)t * npad + base) : ld2cs(a.X + (long)t * npad + base);
      if constexpr (RM == RM_INPUT) {
        r = cur;
      } else {
        double2 prev = make_double2(0.0, 0.0);
        if (valid) {
          if (t > 0) prev = ld2(a.X + (long)(t - 1) * npad + base);
          else if (RM == RM_RESID) prev = ld2(a.u0h + base);
        }
        if constexpr (RM == RM_RESID) {
          r = make_double2(fma(Ej.x, prev.x, -cur.x), fma(Ej.y, prev.y, -cur.y));
          if constexpr (NL >= 1) {
            double2 nm1 = valid ? ld2(a.Nh + (long)t * npad + base) : make_double2(0.0, 0.0);
            r.x = fma(c1.x, nm1.x, r.x);
            r.y = fma(c1.y, nm1.y, r.y);
            if constexpr (NL == 2) {
              double2 nm2 = valid ? ld2(a.Nh + (long)(t > 0 ? t - 1 : 0) * npad + base) : make_double2(0.0, 0.0);
              r.x = fma(-c2.x, nm2.x, r.x);
              r.y = fma(-c2.y, nm2.y, r.y);
            }
          }
        } else {  // RM_QOP: (Q v)_t = v_t - E v_{t-1}, v_{-1} = 0
          r = make_double2(fma(-Ej.x, prev.x, cur.x), fma(-Ej.y, prev.y, cur.y));
        }
      }
      nrm = fma(r.x, r.x, fma(r.y, r.y, nrm));
      if constexpr (OUTM == OUT_UPDATE) stash[t * S + s] = cur;
      y[m1] = cscale(r, sg[t]);
    }
    DFT<P, +1>::run(y);
#pragma unroll
    for (int k1 = 1; k1 < P; ++k1) y[k1] = cmul(y[k1], stw[(k1 * m2) % NT]);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) buf[(k1 * Q + m2) * S + s] = y[k1];
    __syncthreads();

    // ---------------- phase B: DFT-Q, Hermitian pair divide, inverse DFT-Q --------------
    for (int job = tid; job < S * (P / 2); job += THREADS) {
      const int js = job % S, kp = job / S;
      const long jpair = tile * S + js;
      const int k1a = kp == 0 ? 0 : kp;
      const int k1b = kp == 0 ? P / 2 : P - kp;
      double2 Za[Q], Zb[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        Za[q] = buf[(k1a * Q + q) * S + js];
        Zb[q] = buf[(k1b * Q + q) * S + js];
      }
      DFT<Q, +1>::run(Za);
      DFT<Q, +1>::run(Zb);
      double2 Ep = jpair < a.npairs ? ld2(a.E + 2 * jpair) : make_double2(0.0, 0.0);
      const double ba = a.a1 * Ep.x, bb = a.a1 * Ep.y, hin = a.half_inv_nt;
      if (kp != 0) {
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2)
          divide_pair(Za[k2], Zb[Q - 1 - k2], stw[k1a + P * k2], ba, bb, hin, false);
      } else {
        // k1 = 0: frequencies P k2, partner P (Q - k2) mod Q; self at k2 = 0 and Q/2
        divide_pair(Za[0], Za[0], stw[0], ba, bb, hin, true);
#pragma unroll
        for (int k2 = 1; k2 < (Q + 1) / 2; ++k2) divide_pair(Za[k2], Za[Q - k2], stw[P * k2], ba, bb, hin, false);
        if constexpr (Q % 2 == 0 && Q >= 2) divide_pair(Za[Q / 2], Za[Q / 2], stw[P * (Q / 2)], ba, bb, hin, true);
        // k1 = P/2: frequencies P/2 + P k2, partner index Q-1-k2
#pragma unroll
        for (int k2 = 0; k2 < Q / 2; ++k2)
          divide_pair(Zb[k2], Zb[Q - 1 - k2], stw[P / 2 + P * k2], ba, bb, hin, false);
        if constexpr (Q % 2 == 1) divide_pair(Zb[Q / 2], Zb[Q / 2], stw[P / 2 + P * (Q / 2)], ba, bb, hin, true);
      }
      DFT<Q, -1>::run(Za);
      DFT<Q, -1>::run(Zb);
#pragma unroll
      for (int q = 1; q < Q; ++q) {
        Za[q] = cmulc(Za[q], stw[(k1a * q) % NT]);
        Zb[q] = cmulc(Zb[q], stw[(k1b * q) % NT]);
      }
      // each job rewrites exactly the rows it read: no barrier needed inside phase B
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        buf[(k1a * Q + q) * S + js] = Za[q];
        buf[(k1b * Q + q) * S + js] = Zb[q];
      }
    }
    __syncthreads();

    // ---------------- phase C: inverse DFT-P over k1, Gamma^{-1}, update ----------------
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) y[k1] = buf[(k1 * Q + m2) * S + s];
    DFT<P, -1>::run(y);
    if (valid) {
#pragma unroll
      for (int m1 = 0; m1 < P; ++m1) {
        const int t = Q * m1 + m2;
        double2 sv = cscale(y[m1], sgi[t]);
        if constexpr (OUTM == OUT_UPDATE) sv = cadd(stash[t * S + s], sv);
        st2(a.Y + (long)t * npad + base, sv);
      }
    }
    __syncthreads();
  }

  if (a.partial) {
    // fixed-order block reduction (deterministic for a fixed grid)
    __shared__ double red[32];
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

template <int NT, int OUTM>
static size_t time_smem_bytes() {
  const size_t tile = (size_t)NT * TimeCfg<NT>::S;
  return sizeof(double2) * (tile * (OUTM == OUT_UPDATE ? 2 : 1) + NT) + sizeof(double) * 2 * NT;
}

template <int NT, int RM, int OUTM, int NL>
static cudaError_t launch_t(const TimeArgs& a, int grid, cudaStream_t st) {
  auto k = k_time_fused<NT, RM, OUTM, NL>;
  size_t sm = time_smem_bytes<NT, OUTM>();
  static bool attr_done = false;  // per-instantiation, host-side
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  k<<<grid, TimeCfg<NT>::S * TimeCfg<NT>::Q, sm, st>>>(a);
  return cudaGetLastError();
}

template <int NT>
static cudaError_t dispatch_nt(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st) {
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

cudaError_t launch_time_fused(const TimeArgs& a, int rmode, int outmode, int nl, int grid, cudaStream_t st) {
  switch (a.nt) {
    case 4: return dispatch_nt<4>(a, rmode, outmode, nl, grid, st);
    case 8: return dispatch_nt<8>(a, rmode, outmode, nl, grid, st);
    case 16: return dispatch_nt<16>(a, rmode, outmode, nl, grid, st);
    case 32: return dispatch_nt<32>(a, rmode, outmode, nl, grid, st);
    case 64: return dispatch_nt<64>(a, rmode, outmode, nl, grid, st);
    case 128: return dispatch_nt<128>(a, rmode, outmode, nl, grid, st);
    case 256: return dispatch_nt<256>(a, rmode, outmode, nl, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

// Persistent grid: a fixed multiple of the SM count (deterministic partial order), capped
// by the number of tiles.
int time_fused_grid(int nt, long npairs, int sms) {
  int S = 8;
  switch (nt) {
    case 4: case 8: case 16: S = 128; break;
    case 32: S = 32; break;
    case 64: case 128: S = 16; break;
    default: S = 8;
  }
  long ntiles = (npairs + S - 1) / S;
  long g = (long)sms * 3;
  return (int)(ntiles < g ? (ntiles > 0 ? ntiles : 1) : g);
}

// ---------------------------------------------------------------------------------------
// residual only (expd_residual): r_t = E u_{t-1} + C1 N_t - C2 N_{t-1} - u_t, spectral.
// ---------------------------------------------------------------------------------------
template <int NL>
__global__ void __launch_bounds__(256) k_resid_only(const TimeArgs a) {
  const long total = (long)a.nt * a.npairs;
  double nrm = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int t = (int)(i / a.npairs);
    const long base = 2 * (i % a.npairs);
    double2 E = ld2(a.E + base);
    double2 cur = ld2(a.X + (long)t * a.npad + base);
    double2 prev = t > 0 ? ld2(a.X + (long)(t - 1) * a.npad + base) : ld2(a.u0h + base);
    double2 r = make_double2(fma(E.x, prev.x, -cur.x), fma(E.y, prev.y, -cur.y));
    if constexpr (NL >= 1) {
      double2 c1 = ld2(a.C1 + base), nm1 = ld2(a.Nh + (long)t * a.npad + base);
      r.x = fma(c1.x, nm1.x, r.x);
      r.y = fma(c1.y, nm1.y, r.y);
      if constexpr (NL == 2) {
        double2 c2 = ld2(a.C2 + base), nm2 = ld2(a.Nh + (long)(t > 0 ? t - 1 : 0) * a.npad + base);
        r.x = fma(-c2.x, nm2.x, r.x);
        r.y = fma(-c2.y, nm2.y, r.y);
      }
    }
    nrm = fma(r.x, r.x, fma(r.y, r.y, nrm));
    st2(a.Y + (long)t * a.npad + base, r);
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0 && a.partial) a.partial[blockIdx.x] = v;
  }
}

cudaError_t launch_resid_only(const TimeArgs& a, int nl, int grid, cudaStream_t st) {
  if (nl == 0) k_resid_only<0><<<grid, 256, 0, st>>>(a);
  else if (nl == 1) k_resid_only<1><<<grid, 256, 0, st>>>(a);
  else k_resid_only<2><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace expd
