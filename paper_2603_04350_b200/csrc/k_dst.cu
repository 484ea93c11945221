// k_dst.cu -- K2/K3/K4: the orthonormal DST-I V ("L_h = V_h D_h V_h^{-1}"
// with V_h orthogonal; reading R1) along every axis of a slice, and the space-local
// nonlinear pass N-hat = V N(V u-hat) of the Picard sweep (stage 3; BASELINE.json:5).
//
// Algorithm: with M = n+1 = 2^m and F_j = sum_i x_i sin(pi i j / M),
//   y_0 = 0, y_i = sin(pi i/M)(x_i + x_{M-i}) + (x_i - x_{M-i})/2          (i = 1..M-1)
//   Y_k = sum_i y_i e^{-2 pi i ik/M}                                         (complex FFT)
//   F_{2k} = -Im Y_k,  F_1 = Re Y_0 / 2,  F_{2k+1} = F_{2k-1} + Re Y_k       (prefix sum)
// and V x = sqrt(2/M) F.  Two real lines travel as one complex sequence (rows 2q, 2q+1
// or columns 2c, 2c+1 -- for columns that is one aligned double2 per grid row), and
// their Y's are separated with the k <-> M-k Hermitian pairing.
//
// Per line pair, T = M/R0 threads run a register-resident Stockham FFT (radix R0 = 16 or
// 8 first, a middle radix, a small last radix): stage 0 is fed straight from global memory
// (preprocessing fused into the load), shared memory carries only the stage transposes,
// and the last stage is run on Hermitian partner jobs (j, NS - j) so the unpack happens
// in registers.  The prefix sum is a per-thread chunk scan + warp-shuffle scan +
// cross-warp offsets.  Shared layout [position][group] with a 1/16 padding swizzle keeps
// every 16-byte access conflict-free.  G line pairs share a CTA.
#include <cstdlib>

#include "expd_internal.h"
#include "fft_dev.cuh"

namespace expd {


// radix plan: R0 (first stage, fed from the load), up to two middle radices RM1, RM2
// (1 = absent) and the last radix RL (run on Hermitian partner jobs).
template <int M> struct DPlan;
template <> struct DPlan<4>    { static constexpr int NST = 1, R0 = 4,  RM1 = 1,  RM2 = 1, RL = 4; };
template <> struct DPlan<8>    { static constexpr int NST = 1, R0 = 8,  RM1 = 1,  RM2 = 1, RL = 8; };
template <> struct DPlan<16>   { static constexpr int NST = 1, R0 = 16, RM1 = 1,  RM2 = 1, RL = 16; };
template <> struct DPlan<32>   { static constexpr int NST = 2, R0 = 8,  RM1 = 1,  RM2 = 1, RL = 4; };
template <> struct DPlan<64>   { static constexpr int NST = 3, R0 = 8,  RM1 = 2,  RM2 = 1, RL = 4; };
template <> struct DPlan<128>  { static constexpr int NST = 2, R0 = 16, RM1 = 1,  RM2 = 1, RL = 8; };
template <> struct DPlan<256>  { static constexpr int NST = 3, R0 = 16, RM1 = 2,  RM2 = 1, RL = 8; };
template <> struct DPlan<512>  { static constexpr int NST = 3, R0 = 16, RM1 = 4,  RM2 = 1, RL = 8; };
template <> struct DPlan<1024> { static constexpr int NST = 3, R0 = 16, RM1 = 8,  RM2 = 1, RL = 8; };
template <> struct DPlan<2048> { static constexpr int NST = 3, R0 = 16, RM1 = 16, RM2 = 1, RL = 8; };
template <> struct DPlan<4096> { static constexpr int NST = 3, R0 = 16, RM1 = 16, RM2 = 1, RL = 16; };

template <int M, int G>
struct DGeo {
  using P = DPlan<M>;
  static constexpr int NST = P::NST, R0 = P::R0, RM1 = P::RM1, RM2 = P::RM2, RL = P::RL;
  static constexpr int T = M / R0;                 // threads per line pair
  static constexpr int THREADS = G * T;
  static constexpr int NSL = M / RL;               // Ns of the last stage
  static constexpr int L = (M / 2) / T;            // prefix-sum chunk per thread (= R0/2)
  static constexpr int PADP = R0 < 8 ? 8 : R0;     // swizzle period: one pad slot per PADP
  static constexpr int SW = M + M / PADP + 1;      // swizzled positions per group
  static constexpr int JW = G >= 32 ? 1 : 32 / G;  // threads of one group inside a warp
  static constexpr int NWB = (T + JW - 1) / JW;    // warp blocks per group
};

template <int PADP>
__device__ __forceinline__ int swz(int p) { return p + p / PADP; }

template <int G, int PADP>
__device__ __forceinline__ double2& at(double2* buf, int p, int g) {
  return buf[swz<PADP>(p) * G + g];
}

// y_i from z_i and its mirror z_{M-i} (sin(pi i/M) = sin(pi (M-i)/M))
__device__ __forceinline__ double2 preprocess(double2 z, double2 zm, double s) {
  double2 sum = cadd(z, zm), dif = csub(z, zm);
  return make_double2(fma(s, sum.x, 0.5 * dif.x), fma(s, sum.y, 0.5 * dif.y));
}

// e_k (even output F_{2k}) and w_k (prefix-sum increment) of both lines from Z_k, Z_{M-k}
__device__ __forceinline__ void unpack(double2 Zk, double2 Zm, bool k0, double2& e, double2& w) {
  e = make_double2(-0.5 * (Zk.y - Zm.y), 0.5 * (Zk.x - Zm.x));
  w = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y + Zm.y));
  if (k0) w = make_double2(0.5 * w.x, 0.5 * w.y);
}

// Shared-memory positions a + r*STRIDE of group g.  When STRIDE is a multiple of the
// swizzle period the swizzle is linear in r, so every access is base + immediate offset.
template <int G, int PADP, int STRIDE>
struct Walk {
  double2* p0;
  int a;
  __device__ __forceinline__ Walk(double2* buf, int a_, int g) : a(a_) {
    p0 = buf + ((STRIDE % PADP == 0) ? swz<PADP>(a_) * G + g : g);
  }
  __device__ __forceinline__ double2& operator[](int r) const {
    if constexpr (STRIDE % PADP == 0) return p0[r * (STRIDE + STRIDE / PADP) * G];
    else return p0[swz<PADP>(a + r * STRIDE) * G];
  }
};

// t[r] = w^{r b}, r = 0..R-1, from the single table entry w^b by products (binary
// splitting: at most 2 log2 R roundings deep), instead of R-1 table loads.
template <int R>
__device__ __forceinline__ void tw_powers(const double2* __restrict__ tw, int b, double2 (&t)[R]) {
  t[0] = make_double2(1.0, 0.0);
  if constexpr (R > 1) t[1] = __ldg(tw + b);
#pragma unroll
  for (int r = 2; r < R; ++r) t[r] = (r % 2 == 0) ? cmul(t[r / 2], t[r / 2]) : cmul(t[r - 1], t[1]);
}

// In-place middle Stockham stage (radix R, NS) on all groups.
template <int M, int G, int R, int NS>
__device__ __forceinline__ void mid_stage(double2* buf, const double2* __restrict__ tw) {
  using D = DGeo<M, G>;
  constexpr int JOBS = G * (M / R);
  constexpr int JT = (JOBS + D::THREADS - 1) / D::THREADS;
  constexpr int TWS = M / (NS * R);  // twiddle index step per k
  double2 v[JT][R];
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * D::THREADS;
    if (J < JOBS) {
      const int g = J % G, jm = J / G, k = jm % NS;
      Walk<G, D::PADP, M / R> in(buf, jm, g);
#pragma unroll
      for (int r = 0; r < R; ++r) v[jt][r] = in[r];
      double2 t[R];
      tw_powers<R>(tw, k * TWS, t);
#pragma unroll
      for (int r = 1; r < R; ++r) v[jt][r] = cmul(v[jt][r], t[r]);
      DFT<R, -1>::run(v[jt]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * D::THREADS;
    if (J < JOBS) {
      const int g = J % G, jm = J / G, k = jm % NS;
      Walk<G, D::PADP, NS> out(buf, (jm / NS) * NS * R + k, g);
#pragma unroll
      for (int r = 0; r < R; ++r) out[r] = v[jt][r];
    }
  }
  __syncthreads();
}

// The DST of G line pairs whose stage-0 inputs are already preprocessed in v[R0] (thread
// (g, j) holds y_i, i = j + T r).  Leaves F_{p+1} (unscaled) for the thread's positions
// p = 2 c L - 1 + q, q = 0..2L-1 (c = j) in out[].  Starts with a barrier (buf may be in
// use by the caller) and ends with buf holding this thread's positions' values.
template <int M, int G>
__device__ __forceinline__ void dst_core(double2 (&v)[DGeo<M, G>::R0], double2* buf, double2* wt,
                                         const double2* __restrict__ tw, double2 (&out)[2 * DGeo<M, G>::L]) {
  using D = DGeo<M, G>;
  constexpr int R0 = D::R0, RL = D::RL, NSL = D::NSL, T = D::T, L = D::L, PADP = D::PADP;
  const int g = threadIdx.x % G, j = threadIdx.x / G;
  DFT<R0, -1>::run(v);
  __syncthreads();
  if constexpr (D::NST == 1) {
    // one thread owns the whole sequence: unpack in registers
#pragma unroll
    for (int k = 0; k < M / 2; ++k) {
      double2 e, w;
      unpack(v[k], v[(M - k) % M], k == 0, e, w);
      if (k >= 1) at<G, PADP>(buf, 2 * k - 1, g) = e;
      at<G, PADP>(buf, 2 * k, g) = w;
    }
  } else {
    {
      // R0 (<= 16) consecutive positions from a multiple of R0: the swizzle is linear there
      double2* o0 = buf + swz<PADP>(j * R0) * G + g;
#pragma unroll
      for (int r = 0; r < R0; ++r) o0[r * G] = v[r];
    }
    __syncthreads();
    if constexpr (D::RM1 > 1) mid_stage<M, G, D::RM1, R0>(buf, tw);
    if constexpr (D::RM2 > 1) mid_stage<M, G, D::RM2, R0 * D::RM1>(buf, tw);
    // last stage on Hermitian partner jobs, then the unpack
    constexpr int PJOBS = G * (NSL / 2);
    constexpr int PJT = (PJOBS + D::THREADS - 1) / D::THREADS;
    double2 va[PJT][RL], vb[PJT][RL];
#pragma unroll
    for (int pt = 0; pt < PJT; ++pt) {
      const int PJ = threadIdx.x + pt * D::THREADS;
      if (PJ < PJOBS) {
        const int gg = PJ % G, pj = PJ / G;
        const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
        Walk<G, PADP, NSL> ia(buf, ja, gg), ib(buf, jb, gg);
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          va[pt][r] = ia[r];
          vb[pt][r] = ib[r];
        }
        {
          double2 t[RL];
          tw_powers<RL>(tw, ja, t);
#pragma unroll
          for (int r = 1; r < RL; ++r) va[pt][r] = cmul(va[pt][r], t[r]);
          tw_powers<RL>(tw, jb, t);
#pragma unroll
          for (int r = 1; r < RL; ++r) vb[pt][r] = cmul(vb[pt][r], t[r]);
        }
        DFT<RL, -1>::run(va[pt]);
        DFT<RL, -1>::run(vb[pt]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int pt = 0; pt < PJT; ++pt) {
      const int PJ = threadIdx.x + pt * D::THREADS;
      if (PJ < PJOBS) {
        const int gg = PJ % G, pj = PJ / G;
        const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
        // positions 2k-1 (e_k) and 2k (w_k) for k = ja + NSL r and k = jb + NSL r
        Walk<G, PADP, 2 * NSL> ea(buf, 2 * ja - 1 < 0 ? 0 : 2 * ja - 1, gg), wa(buf, 2 * ja, gg);
        Walk<G, PADP, 2 * NSL> eb(buf, 2 * jb - 1, gg), wb(buf, 2 * jb, gg);
#pragma unroll
        for (int r = 0; r < RL / 2; ++r) {
          double2 e, w;
          const int ka = ja + NSL * r;
          unpack(va[pt][r], pj == 0 ? va[pt][(RL - r) % RL] : vb[pt][RL - 1 - r], ka == 0, e, w);
          if (ka >= 1) {
            if (ja >= 1) ea[r] = e;
            else at<G, PADP>(buf, 2 * ka - 1, gg) = e;
          }
          wa[r] = w;
          unpack(vb[pt][r], pj == 0 ? vb[pt][RL - 1 - r] : va[pt][RL - 1 - r], false, e, w);
          eb[r] = e;
          wb[r] = w;
        }
      }
    }
  }
  __syncthreads();
  // prefix sum of w_k over k: chunk k in [c L, c L + L), c = j  (positions 2cL-1 .. 2cL+2L-2)
  double2 tot = make_double2(0.0, 0.0);
  {
    // positions 2jL .. 2jL+2L-1 (2L <= 16, 2jL a multiple of 2L): linear swizzle
    const double2* P = buf + swz<PADP>(2 * j * L) * G + g;
#pragma unroll
    for (int l = 0; l < L; ++l) {
      if (l >= 1) out[2 * l] = P[(2 * l - 1) * G];
      tot = cadd(tot, P[(2 * l) * G]);
      out[2 * l + 1] = tot;
    }
    out[0] = at<G, PADP>(buf, j > 0 ? 2 * j * L - 1 : 0, g);  // overwritten for j == 0 below
  }
  // inclusive scan of chunk totals across the group's threads (lanes g + G*j')
  double2 inc = tot;
  const int lane = threadIdx.x & 31;
  if constexpr (D::JW > 1) {
#pragma unroll
    for (int d = 1; d < D::JW; d <<= 1) {
      double ox = __shfl_up_sync(0xffffffffu, inc.x, d * G);
      double oy = __shfl_up_sync(0xffffffffu, inc.y, d * G);
      if (lane >= d * G) inc = cadd(inc, make_double2(ox, oy));
    }
  }
  const int jw = j / D::JW;
  if constexpr (D::NWB > 1) {
    if (j % D::JW == D::JW - 1 || j == T - 1) wt[jw * G + g] = inc;
    __syncthreads();
  }
  double2 off = csub(inc, tot);  // exclusive within the warp block
  if constexpr (D::NWB > 1) {
    for (int b = 0; b < jw; ++b) off = cadd(off, wt[b * G + g]);
  }
#pragma unroll
  for (int l = 0; l < L; ++l) out[2 * l + 1] = cadd(out[2 * l + 1], off);
  out[0] = j == 0 ? make_double2(0.0, 0.0) : out[0];  // position -1 does not exist
}

// ---------------------------------------------------------------------------------------
// x-axis transform of row pairs.  Row r of slice s at in + s*in_slice + r*in_rs (length
// n = M-1); output rows likewise (out_rs == M: padded spectral row, pad written as 0).
// MODE 0: V; 1: V N(in) (N applied on load, physical input); 2: V N(V in) (dim 1).
// Each thread loads only its own stage-0 elements (coalesced), parks them in shared
// memory for its mirror partner, and stores its outputs straight from registers.
// ---------------------------------------------------------------------------------------
template <int M, int G, int MODE>
__global__ void __launch_bounds__(DGeo<M, G>::THREADS, (DGeo<M, G>::THREADS <= 512 ? 512 / DGeo<M, G>::THREADS : 1))
    k_rows(const double* __restrict__ in, long in_slice, int in_rs, double* __restrict__ out, long out_slice,
           int out_rs, int rows_per_slice, const double2* __restrict__ tw, const double* __restrict__ sinp,
           Poly poly) {
  using D = DGeo<M, G>;
  constexpr int R0 = D::R0, T = D::T, L = D::L, PADP = D::PADP;
  extern __shared__ double2 dsm[];
  double2* buf = dsm;             // [SW][G] swizzled work buffer; also raw [M][G]
  double2* wt = dsm + D::SW * G;  // [NWB][G]
  const int g = threadIdx.x % G, j = threadIdx.x / G;
  const long slice = blockIdx.y;
  const int ra = 2 * (blockIdx.x * G + g), rb = ra + 1;
  const bool has_a = ra < rows_per_slice, has_b = rb < rows_per_slice;
  const double* ia = in + slice * in_slice + (long)ra * in_rs;
  const double* ib = in + slice * in_slice + (long)rb * in_rs;
  const double scale = sqrt(2.0 / (double)M);
  double2 o[2 * L];
#pragma unroll
  for (int pass = 0; pass < (MODE == 2 ? 2 : 1); ++pass) {
    double2 v[R0];
    if (pass == 0) {
      double2 z[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + T * r;
        double a = 0.0, b = 0.0;
        if (i >= 1) {
          if (has_a) a = __ldg(ia + i - 1);
          if (has_b) b = __ldg(ib + i - 1);
          if constexpr (MODE == 1) {
            a = has_a ? poly_eval(poly, a) : 0.0;
            b = has_b ? poly_eval(poly, b) : 0.0;
          }
        }
        z[r] = make_double2(a, b);
      }
#pragma unroll
      for (int r = 0; r < R0; ++r) dsm[(j + T * r) * G + g] = z[r];  // raw [M][G]
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + T * r;
        v[r] = i == 0 ? make_double2(0.0, 0.0) : preprocess(z[r], dsm[(M - i) * G + g], __ldg(sinp + i));
      }
    } else {
      // N(u) of the first transform sits in buf at position i-1 (grid index i)
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + T * r;
        v[r] = i == 0 ? make_double2(0.0, 0.0)
                      : preprocess(at<G, PADP>(buf, i - 1, g), at<G, PADP>(buf, M - i - 1, g), __ldg(sinp + i));
      }
    }
    dst_core<M, G>(v, buf, wt, tw, o);
    if (MODE == 2 && pass == 0) {
#pragma unroll
      for (int q = 0; q < 2 * L; ++q) {
        const int p = 2 * j * L - 1 + q;
        if (p >= 0) at<G, PADP>(buf, p, g) = make_double2(poly_eval(poly, scale * o[q].x), poly_eval(poly, scale * o[q].y));
      }
      __syncthreads();
    }
  }
  double* oa = out + slice * out_slice + (long)ra * out_rs;
  double* ob = out + slice * out_slice + (long)rb * out_rs;
#pragma unroll
  for (int q = 0; q < 2 * L; ++q) {
    const int p = 2 * j * L - 1 + q;
    if (p >= 0) {
      if (has_a) oa[p] = scale * o[q].x;
      if (has_b) ob[p] = scale * o[q].y;
    }
  }
  if (out_rs == M && j == T - 1) {  // pad position of a spectral row stays 0
    if (has_a) oa[M - 1] = 0.0;
    if (has_b) ob[M - 1] = 0.0;
  }
}

// ---------------------------------------------------------------------------------------
// strided-axis transform of column pairs in the padded spectral layout: line pair
// (o, cp): base = o*outer_stride + 2*cp, element i-1 at base + (i-1)*stride (one double2).
// NL: transform, N(u) pointwise, transform (the fused stage-3 visit).
// ---------------------------------------------------------------------------------------
template <int M, int G, bool NL>
__global__ void __launch_bounds__(DGeo<M, G>::THREADS, (DGeo<M, G>::THREADS <= 512 ? 512 / DGeo<M, G>::THREADS : 1))
    k_cols(const double* in, long in_slice, double* out, long out_slice, long stride, long outer_stride,
           const double2* __restrict__ tw, const double* __restrict__ sinp, Poly poly) {
  using D = DGeo<M, G>;
  constexpr int R0 = D::R0, T = D::T, L = D::L, PADP = D::PADP;
  constexpr int GROUPS = (M / 2) / G;  // column-pair groups per outer index
  extern __shared__ double2 dsm[];
  double2* buf = dsm;             // [SW][G] (also raw [M][G])
  double2* wt = dsm + D::SW * G;  // [NWB][G]
  const int g = threadIdx.x % G, j = threadIdx.x / G;
  const long slice = blockIdx.y;
  const long o = blockIdx.x / GROUPS;
  const int cp = (blockIdx.x % GROUPS) * G + g;
  const long st2 = stride / 2;  // in double2 units (stride is even: padded rows)
  const double2* ib = reinterpret_cast<const double2*>(in + slice * in_slice + o * outer_stride) + cp;
  double2* ob = reinterpret_cast<double2*>(out + slice * out_slice + o * outer_stride) + cp;
  const double scale = sqrt(2.0 / (double)M);
  double2 oo[2 * L];
#pragma unroll
  for (int pass = 0; pass < (NL ? 2 : 1); ++pass) {
    double2 v[R0];
    if (pass == 0) {
      double2 z[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + T * r;
        z[r] = i >= 1 ? ib[(long)(i - 1) * st2] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int r = 0; r < R0; ++r) dsm[(j + T * r) * G + g] = z[r];  // raw [M][G]
      __syncthreads();
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + T * r;
        v[r] = i == 0 ? make_double2(0.0, 0.0) : preprocess(z[r], dsm[(M - i) * G + g], __ldg(sinp + i));
      }
    } else {
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + T * r;
        v[r] = i == 0 ? make_double2(0.0, 0.0)
                      : preprocess(at<G, PADP>(buf, i - 1, g), at<G, PADP>(buf, M - i - 1, g), __ldg(sinp + i));
      }
    }
    dst_core<M, G>(v, buf, wt, tw, oo);
    if (NL && pass == 0) {
#pragma unroll
      for (int q = 0; q < 2 * L; ++q) {
        const int p = 2 * j * L - 1 + q;
        if (p >= 0) at<G, PADP>(buf, p, g) = make_double2(poly_eval(poly, scale * oo[q].x), poly_eval(poly, scale * oo[q].y));
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int q = 0; q < 2 * L; ++q) {
    const int p = 2 * j * L - 1 + q;
    if (p >= 0) ob[(long)p * st2] = make_double2(scale * oo[q].x, scale * oo[q].y);
  }
}

// ---------------------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------------------
template <int M> struct RowG { static constexpr int T = M / DPlan<M>::R0; static constexpr int G = T >= 128 ? 1 : 128 / T; };
template <int M> struct ColG { static constexpr int T = M / DPlan<M>::R0; static constexpr int G0 = T >= 128 ? 2 : 256 / T; static constexpr int G = G0 > M / 2 ? M / 2 : G0; };

struct RowsOp {
  const double* in; long in_slice; int in_rs; double* out; long out_slice; int out_rs; int rows; long nslices;
  bool nlload, nlmid;
};
struct ColsOp {
  const double* in; long in_slice; double* out; long out_slice; long stride, outer_stride, nouter, nslices;
  bool nl;
};

template <int M, int G>
static size_t dst_smem() {
  return sizeof(double2) * (size_t)(DGeo<M, G>::SW * G + DGeo<M, G>::NWB * G + 1);
}
template <typename K>
static cudaError_t smem_attr(K k, size_t bytes, DevOnce& done) {
  return smem_optin(done, k, bytes);
}

template <int M, int MODE>
static cudaError_t rows_launch(const RowsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  constexpr int G = RowG<M>::G;
  int pairs = (o.rows + 1) / 2;
  dim3 grid((pairs + G - 1) / G, (unsigned)o.nslices);
  const size_t sm = dst_smem<M, G>();
  static DevOnce done;  // per instantiation and device
  cudaError_t e = smem_attr(k_rows<M, G, MODE>, sm, done);
  if (e != cudaSuccess) return e;
  k_rows<M, G, MODE><<<grid, DGeo<M, G>::THREADS, sm, st>>>(o.in, o.in_slice, o.in_rs, o.out, o.out_slice, o.out_rs,
                                                            o.rows, t.tw, t.sinp, P);
  return cudaGetLastError();
}
template <int M>
static cudaError_t run_rows(const RowsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  if (o.nlload) return rows_launch<M, 1>(o, t, P, st);
  if (o.nlmid) return rows_launch<M, 2>(o, t, P, st);
  return rows_launch<M, 0>(o, t, P, st);
}
template <int M, int G>
static cudaError_t run_cols_g(const ColsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  dim3 grid((unsigned)(o.nouter * ((M / 2) / G)), (unsigned)o.nslices);
  const size_t sm = dst_smem<M, G>();
  cudaError_t e;
  static DevOnce done_nl, done_pl;  // per instantiation and device
  if (o.nl) {
    if ((e = smem_attr(k_cols<M, G, true>, sm, done_nl)) != cudaSuccess) return e;
    k_cols<M, G, true><<<grid, DGeo<M, G>::THREADS, sm, st>>>(o.in, o.in_slice, o.out, o.out_slice, o.stride,
                                                               o.outer_stride, t.tw, t.sinp, P);
  } else {
    if ((e = smem_attr(k_cols<M, G, false>, sm, done_pl)) != cudaSuccess) return e;
    k_cols<M, G, false><<<grid, DGeo<M, G>::THREADS, sm, st>>>(o.in, o.in_slice, o.out, o.out_slice, o.stride,
                                                                o.outer_stride, t.tw, t.sinp, P);
  }
  return cudaGetLastError();
}

template <int M>
static cudaError_t run_cols(const ColsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  if constexpr (M == 2048) {
    static int g1 = -1;  // tuning switch: EXPD_COLG=1 selects one column pair per CTA
    if (g1 < 0) {
      const char* e = getenv("EXPD_COLG");
      g1 = (e && e[0] == '1') ? 1 : 0;
    }
    if (g1) return run_cols_g<M, 1>(o, t, P, st);
  }
  return run_cols_g<M, ColG<M>::G>(o, t, P, st);
}

static cudaError_t rows(int M, const RowsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  switch (M) {
    case 4: return run_rows<4>(o, t, P, st);
    case 8: return run_rows<8>(o, t, P, st);
    case 16: return run_rows<16>(o, t, P, st);
    case 32: return run_rows<32>(o, t, P, st);
    case 64: return run_rows<64>(o, t, P, st);
    case 128: return run_rows<128>(o, t, P, st);
    case 256: return run_rows<256>(o, t, P, st);
    case 512: return run_rows<512>(o, t, P, st);
    case 1024: return run_rows<1024>(o, t, P, st);
    case 2048: return run_rows<2048>(o, t, P, st);
    case 4096: return run_rows<4096>(o, t, P, st);
    default: return cudaErrorInvalidValue;
  }
}
static cudaError_t cols(int M, const ColsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  switch (M) {
    case 4: return run_cols<4>(o, t, P, st);
    case 8: return run_cols<8>(o, t, P, st);
    case 16: return run_cols<16>(o, t, P, st);
    case 32: return run_cols<32>(o, t, P, st);
    case 64: return run_cols<64>(o, t, P, st);
    case 128: return run_cols<128>(o, t, P, st);
    case 256: return run_cols<256>(o, t, P, st);
    case 512: return run_cols<512>(o, t, P, st);
    case 1024: return run_cols<1024>(o, t, P, st);
    case 2048: return run_cols<2048>(o, t, P, st);
    case 4096: return run_cols<4096>(o, t, P, st);
    default: return cudaErrorInvalidValue;
  }
}

static Poly make_poly(int npoly, const double* q) {
  Poly P{};
  P.npoly = npoly;
  for (int i = 0; i < npoly && i < 8; ++i) P.q[i] = q[i];
  return P;
}

#define CK(x)                               \
  do {                                      \
    cudaError_t e_ = (x);                   \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)

// Strided-axis passes of a padded spectral slice.
static ColsOp col_op(const Geom& g, int axis, const double* in, double* out, long nslices, bool nl) {
  ColsOp o{};
  o.in = in; o.out = out; o.in_slice = g.npad; o.out_slice = g.npad; o.nslices = nslices; o.nl = nl;
  const long row = g.M, plane = (long)g.n * g.M;
  if (axis == 1) {            // y
    o.stride = row;
    o.outer_stride = plane;   // z planes (dim 3) ; dim 2: one outer
    o.nouter = g.dim == 3 ? g.n : 1;
  } else {                    // z
    o.stride = plane;
    o.outer_stride = row;     // y rows
    o.nouter = g.n;
  }
  return o;
}

static bool use_line(const Geom& g);
// one strided-axis pass of padded spectral slices (TMA line kernel when available)
static cudaError_t colpass(const Geom& g, const DstTables& t, const Poly& P, int ax, const double* in, double* out,
                           long nslices, cudaStream_t st) {
  if (use_line(g)) return line_pass(g, t, P, ax, false, in, out, nslices, st);
  return cols(g.M, col_op(g, ax, in, out, nslices, false), t, P, st);
}

// EXPD_PHYS_ROWS=1: the physical <-> spectral x pass through k_rows (the round-1 kernel that
// re-pitches inside the transform) instead of re-pitch copy + TMA row pass (A/B switch)
static bool phys_rows_kernel() {
  const char* e = getenv("EXPD_PHYS_ROWS");
  return e && e[0] == '1';
}

cudaError_t dst_slices(const Geom& g, const DstTables& t, const double* src, bool src_spectral, double* dst,
                       bool dst_spectral, long nslices, double* scratch, cudaStream_t st) {
  if (nslices <= 0) return cudaSuccess;
  Poly P = make_poly(0, nullptr);
  const int rows_ps = (int)(g.N / g.n);
  const long phys_slice = g.N;
  // dim >= 2 with the TMA line kernels: the x pass runs as the spectral TMA row pass in place
  // on padded rows and the physical <-> padded re-pitch is a plain copy pass (physical rows of
  // n doubles, n odd, are not 16-byte aligned, so TMA cannot read or write them).  Measured
  // (profiles/r02/phys_x_ab.txt): c5 precond_apply 31.6 -> 30.7 ms, c2 solve 0.197 -> 0.188 ms
  // against k_rows, which re-pitches inside its (non-TMA) transform.
  const bool tma_x = use_line(g) && g.dim >= 2 && !phys_rows_kernel();
  if (!src_spectral && dst_spectral) {
    // physical -> spectral: x first (into dst), then strided axes in place
    if (tma_x) {
      CK(repitch(src, g.n, dst, g.M, g.n, (long)rows_ps * nslices, st));
      CK(line_pass(g, t, P, 0, false, dst, dst, nslices, st));
    } else {
      RowsOp r{src, phys_slice, g.n, dst, g.npad, g.M, rows_ps, nslices, false, false};
      CK(rows(g.M, r, t, P, st));
    }
    for (int ax = 1; ax < g.dim; ++ax) CK(colpass(g, t, P, ax, dst, dst, nslices, st));
    return cudaSuccess;
  }
  if (src_spectral && !dst_spectral) {
    // spectral -> physical: strided axes into scratch (src untouched), then x into dst;
    // in chunks of nonlin_chunk_slices() slices (the scratch size)
    const long chunk = g.dim == 1 ? nslices : nonlin_chunk_slices(g);
    for (long s0 = 0; s0 < nslices; s0 += chunk) {
      const long ns = nslices - s0 < chunk ? nslices - s0 : chunk;
      const double* cur = src + s0 * g.npad;
      for (int ax = 1; ax < g.dim; ++ax) {
        CK(colpass(g, t, P, ax, cur, scratch, ns, st));
        cur = scratch;
      }
      if (tma_x) {
        CK(line_pass(g, t, P, 0, false, cur, scratch, ns, st));
        CK(repitch(scratch, g.M, dst + s0 * phys_slice, g.n, g.n, (long)rows_ps * ns, st));
        continue;
      }
      RowsOp r{cur, g.npad, g.M, dst + s0 * phys_slice, phys_slice, g.n, rows_ps, ns, false, false};
      CK(rows(g.M, r, t, P, st));
    }
    return cudaSuccess;
  }
  if (src_spectral && dst_spectral) {
    RowsOp r{src, g.npad, g.M, dst, g.npad, g.M, rows_ps, nslices, false, false};
    if (use_line(g)) CK(line_pass(g, t, P, 0, false, src, dst, nslices, st));
    else CK(rows(g.M, r, t, P, st));
    for (int ax = 1; ax < g.dim; ++ax) CK(colpass(g, t, P, ax, dst, dst, nslices, st));
    return cudaSuccess;
  }
  return cudaErrorInvalidValue;
}

int nonlin_chunk_slices(const Geom& g) {
  // slices per stage-3 chunk: the chunk's intermediate (npad doubles per slice) is about
  // EXPD_CHUNK_MB (default 512) MB.  Re-measured in round 2 (profiles/r02/chunk_sweep.txt):
  // 64 / 128 / 256 / 512 / 1024 / 2048 MB -> 23.5 / 22.3 / 21.9 / 21.7 / 21.7 / 21.9 ms per
  // sweep; at 4 GB and the whole 8.6 GB state the fused y-pass slows from 8.3 to 13-17 ms.  Measured on c5 (profiles/r01): 2-slice chunks that fit
  // the 126 MB L2 lose more to launch tails than the L2 residency saves -- the axis passes
  // are shared-memory / fp64 bound and the extra HBM round trip of the intermediate
  // overlaps them (64 MB: 21.7 ms stage 3, 512 MB: 18.9 ms)
  static long mb = -1;
  if (mb < 0) {
    const char* e = getenv("EXPD_CHUNK_MB");
    mb = e ? atol(e) : 512;
    if (mb < 1) mb = 512;
  }
  long per = g.npad * 8;
  long c = (mb << 20) / (per > 0 ? per : 1);
  return (int)(c < 1 ? 1 : (c > 64 ? 64 : c));
}

// EXPD_S3_FULLX=0 keeps the x passes chunked too when a whole-state intermediate is available
static bool s3_full_x() {
  const char* e = getenv("EXPD_S3_FULLX");
  return !(e && e[0] == '0');
}

int nonlin_kernel_launches(const Geom& g, long nslices, bool full_tmp) {
  if (full_tmp && use_line(g) && g.dim == 2 && s3_full_x())
    return 2 + (int)((nslices + nonlin_chunk_slices(g) - 1) / nonlin_chunk_slices(g));
  if (use_line(g) && nonlin_chunk_slices(g) >= 2 && stage3p_supported(g, nslices)) return 1;
  long chunk = nonlin_chunk_slices(g);
  long nch = (nslices + chunk - 1) / chunk;
  int per = g.dim == 1 ? 1 : (g.dim == 2 ? 3 : 5);
  return (int)(nch * per);
}

static bool use_line(const Geom& g) {
  static int v = -1;  // tuning switch: EXPD_LINE=0 keeps the k_rows / k_cols kernels
  if (v < 0) {
    const char* e = getenv("EXPD_LINE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v && g.dim >= 2 && line_supported(g);
}

static cudaError_t mark(PassTimer* tm, int kind, cudaStream_t st) {
  if (!tm || tm->used >= tm->cap) return cudaSuccess;
  cudaEvent_t e = tm->ev[tm->used];
  if (kind >= 0 && tm->used < 512) tm->kind[tm->used] = kind;
  ++tm->used;
  return tm->ext ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
}

// ring slots of the persistent stage 3's intermediate (EXPD_S3P_K, default 4: 134 MB at c5)
static int s3p_ring(long chunk) {
  const char* e = getenv("EXPD_S3P_K");
  long k = e ? atol(e) : 4;
  if (k < 2) k = 2;
  if (k > chunk) k = chunk;
  return (int)k;
}

cudaError_t nonlin_slices(const Geom& g, const DstTables& t, const double* uhat, double* nhat, long nslices,
                          int npoly, const double* q, double* scratch, cudaStream_t st, PassTimer* tm, void* s3ctl,
                          double* full_tmp, const PeerOut* peer) {
  Poly P = make_poly(npoly, q);
  const int rows_ps = (int)(g.N / g.n);
  const long chunk = nonlin_chunk_slices(g);
  const bool tl = use_line(g);
  if (tm) tm->used = 0;
  if (peer && (!tl || g.dim < 2)) return cudaErrorInvalidValue;  // peer stores: the line-kernel path
  if (tl && full_tmp && g.dim == 2 && s3_full_x() && !peer) {
    // the x passes over ALL slices in one launch each (an intermediate of the whole state):
    // no per-chunk launch tails (measured: x passes 7.7 -> 7.2 ms per c5 sweep); the fused
    // y pass stays in ~512 MB chunks (whole-state launches of it measured 1.6-2x slower)
    CK(mark(tm, 0, st));
    CK(line_pass(g, t, P, 0, false, uhat, full_tmp, nslices, st));
    for (long s0 = 0; s0 < nslices; s0 += chunk) {
      const long ns = nslices - s0 < chunk ? nslices - s0 : chunk;
      CK(mark(tm, 2, st));
      CK(line_pass(g, t, P, 1, true, full_tmp + s0 * g.npad, full_tmp + s0 * g.npad, ns, st));
    }
    CK(mark(tm, 0, st));
    CK(line_pass(g, t, P, 0, false, full_tmp, nhat, nslices, st));
    CK(mark(tm, -1, st));
    return cudaSuccess;
  }
  if (tl && s3ctl && chunk >= 2 && stage3p_supported(g, nslices) && !peer) {
    CK(mark(tm, 3, st));
    CK(stage3p(g, t, P, uhat, scratch, s3p_ring(chunk), nhat, nslices, s3ctl, st));
    CK(mark(tm, -1, st));
    return cudaSuccess;
  }
  for (long s0 = 0; s0 < nslices; s0 += chunk) {
    long ns = nslices - s0 < chunk ? nslices - s0 : chunk;
    const double* in = uhat + s0 * g.npad;
    double* out = nhat + s0 * g.npad;
    if (tl) {
      // x (inverse) -> scratch ; [dim 3: y] ; last axis fused [V, N, V] ; [dim 3: y] ; x -> out
      CK(mark(tm, 0, st));
      if (peer && peer->in_maps) {
        PeerOut pi{nullptr, 0, peer->in_maps, peer->in_slot0 + (int)s0};
        CK(line_pass(g, t, P, 0, false, nullptr, scratch, ns, st, &pi));
      } else {
        CK(line_pass(g, t, P, 0, false, in, scratch, ns, st));
      }
      if (g.dim == 3) {
        CK(mark(tm, 1, st));
        CK(line_pass(g, t, P, 1, false, scratch, scratch, ns, st));
      }
      CK(mark(tm, 2, st));
      CK(line_pass(g, t, P, g.dim - 1, true, scratch, scratch, ns, st));
      if (g.dim == 3) {
        CK(mark(tm, 1, st));
        CK(line_pass(g, t, P, 1, false, scratch, scratch, ns, st));
      }
      CK(mark(tm, 0, st));
      if (peer && peer->maps) {
        PeerOut po{peer->maps, peer->slot0 + (int)s0, nullptr, 0};
        CK(line_pass(g, t, P, 0, false, scratch, nullptr, ns, st, &po));
      } else {
        CK(line_pass(g, t, P, 0, false, scratch, out, ns, st));
      }
      continue;
    }
    if (g.dim == 1) {
      RowsOp r{in, g.npad, g.M, out, g.npad, g.M, rows_ps, ns, false, true};
      CK(rows(g.M, r, t, P, st));
      continue;
    }
    // x (inverse) -> scratch ; [dim 3: y in place] ; last axis fused with N ; back ; x -> out
    RowsOp r1{in, g.npad, g.M, scratch, g.npad, g.M, rows_ps, ns, false, false};
    CK(rows(g.M, r1, t, P, st));
    if (g.dim == 3) CK(cols(g.M, col_op(g, 1, scratch, scratch, ns, false), t, P, st));
    CK(cols(g.M, col_op(g, g.dim - 1, scratch, scratch, ns, true), t, P, st));
    if (g.dim == 3) CK(cols(g.M, col_op(g, 1, scratch, scratch, ns, false), t, P, st));
    RowsOp r2{scratch, g.npad, g.M, out, g.npad, g.M, rows_ps, ns, false, false};
    CK(rows(g.M, r2, t, P, st));
  }
  if (tl) CK(mark(tm, -1, st));  // end of the last pass
  return cudaSuccess;
}

cudaError_t nonlin_phys_slices(const Geom& g, const DstTables& t, const double* u, double* nhat, long nslices,
                               int npoly, const double* q, double* scratch, cudaStream_t st) {
  (void)scratch;
  Poly P = make_poly(npoly, q);
  const int rows_ps = (int)(g.N / g.n);
  RowsOp r{u, g.N, g.n, nhat, g.npad, g.M, rows_ps, nslices, true, false};
  CK(rows(g.M, r, t, P, st));
  Poly P0 = make_poly(0, nullptr);
  for (int ax = 1; ax < g.dim; ++ax) CK(colpass(g, t, P0, ax, nhat, nhat, nslices, st));
  return cudaSuccess;
}

// Diagnostics: time one kernel family on spectral slices of the workspace (which: 0 row
// pass, 1 strided pass, 2 fused strided N pass), reps launches, returns ms per launch.
cudaError_t dst_debug_time(const Geom& g, const DstTables& t, int which, double* a, double* b, long nslices,
                           int npoly, const double* q, int reps, float* ms, cudaStream_t st) {
  Poly P = make_poly(npoly, q);
  const int rows_ps = (int)(g.N / g.n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto one = [&]() -> cudaError_t {
    if (which >= 4) return line_pass(g, t, P, which == 4 ? 0 : g.dim - 1, which == 6, a, b, nslices, st);
    if (which == 0) {
      RowsOp r{a, g.npad, g.M, b, g.npad, g.M, rows_ps, nslices, false, false};
      return rows(g.M, r, t, P, st);
    }
    return cols(g.M, col_op(g, g.dim - 1, a, b, nslices, which == 2), t, P, st);
  };
  CK(one());
  cudaEventRecord(e0, st);
  for (int i = 0; i < reps; ++i) CK(one());
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  *ms /= reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError();
}

size_t dst_scratch_doubles(const Geom& g, long max_slices) { return (size_t)g.npad * (size_t)max_slices; }

}  // namespace expd
