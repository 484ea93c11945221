// fft_dev.cuh -- register-resident small DFTs (radix 2/4/8/16) in fp64 for sm_100a.
//
// Building block of the time DFT of the alpha-circulant preconditioner (Steps (a)/(c),
// PAPER.md:188-197, F = Nt^{-1/2}[omega^{(l1-1)(l2-1)}], omega = e^{+2 pi i/Nt},
// PAPER.md:114) and of the DST-I of the spatial solves ("executed
// efficiently using fast Fourier transforms").  DIR = +1 computes
// X_k = sum_m e^{+2 pi i k m / R} x_m, DIR = -1 the conjugate kernel; no normalisation.
// All twiddles inside a radix-R DFT are compile-time constants; multiplications by
// 1, -1, +-i are elided with if constexpr, so the SASS holds only the DFMA/DADD/DMUL the
// butterflies need.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace expd {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by s*i, s = +-1
template <int S>
__device__ __forceinline__ double2 mul_i(double2 a) {
  if constexpr (S > 0) return make_double2(-a.y, a.x);
  else return make_double2(a.y, -a.x);
}

// ---- compile-time loop ---------------------------------------------------------------
template <typename F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// cos / sin (2 pi e / 16) for e = 0..15 (exact decimal expansions to 20 digits)
__host__ __device__ constexpr double cos16(int e) {
  constexpr double c[16] = {1.0,
                            0.92387953251128675613,
                            0.70710678118654752440,
                            0.38268343236508977173,
                            0.0,
                            -0.38268343236508977173,
                            -0.70710678118654752440,
                            -0.92387953251128675613,
                            -1.0,
                            -0.92387953251128675613,
                            -0.70710678118654752440,
                            -0.38268343236508977173,
                            0.0,
                            0.38268343236508977173,
                            0.70710678118654752440,
                            0.92387953251128675613};
  return c[e & 15];
}
__host__ __device__ constexpr double sin16(int e) { return cos16(e - 4); }

// x *= e^{DIR 2 pi i E / R}, R | 16
template <int E, int R, int DIR>
__device__ __forceinline__ void twid(double2& x) {
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) {
    return;
  } else if constexpr (2 * e == R) {
    x = make_double2(-x.x, -x.y);
  } else if constexpr (4 * e == R) {
    x = mul_i<DIR>(x);
  } else if constexpr (4 * e == 3 * R) {
    x = mul_i<-DIR>(x);
  } else {
    constexpr int e16 = e * (16 / R);
    constexpr double c = cos16(e16);
    constexpr double s = DIR * sin16(e16);
    x = make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c));
  }
}

// ---- radix kernels, in place, natural order ---------------------------------------------
template <int DIR>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
template <int DIR>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  double2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_i<DIR>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <int R, int DIR>
struct DFT;
template <int DIR>
struct DFT<1, DIR> {
  __device__ __forceinline__ static void run(double2*) {}
};
template <int DIR>
struct DFT<2, DIR> {
  __device__ __forceinline__ static void run(double2* x) { dft2<DIR>(x[0], x[1]); }
};
template <int DIR>
struct DFT<4, DIR> {
  __device__ __forceinline__ static void run(double2* x) { dft4<DIR>(x[0], x[1], x[2], x[3]); }
};
// R = P1 * Q1 four-step: inner DFT-P1 over m1 (stride Q1), twiddle w_R^{k1 m2}, DFT-Q1 over m2.
template <int DIR>
struct DFT<8, DIR> {
  __device__ __forceinline__ static void run(double2* x) {
    // P1 = 4 (over x[2 m1 + m2]), Q1 = 2
    dft4<DIR>(x[0], x[2], x[4], x[6]);
    dft4<DIR>(x[1], x[3], x[5], x[7]);
    // now x[2 k1 + m2] holds T[k1][m2]; twiddle w8^{k1 * 1} on m2 = 1
    twid<1, 8, DIR>(x[3]);
    twid<2, 8, DIR>(x[5]);
    twid<3, 8, DIR>(x[7]);
    double2 y[8];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      y[k1] = cadd(x[2 * k1], x[2 * k1 + 1]);
      y[k1 + 4] = csub(x[2 * k1], x[2 * k1 + 1]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = y[i];
  }
};
template <int DIR>
struct DFT<16, DIR> {
  __device__ __forceinline__ static void run(double2* x) {
    // P1 = 4 over x[4 m1 + m2], Q1 = 4
#pragma unroll
    for (int m2 = 0; m2 < 4; ++m2) dft4<DIR>(x[m2], x[4 + m2], x[8 + m2], x[12 + m2]);
    // x[4 k1 + m2] = T[k1][m2]; twiddle w16^{k1 m2}
    sfor<4>([&](auto k1) {
      sfor<4>([&](auto m2) { twid<decltype(k1)::value * decltype(m2)::value, 16, DIR>(x[4 * k1 + m2]); });
    });
    double2 y[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 a = x[4 * k1], b = x[4 * k1 + 1], c = x[4 * k1 + 2], d = x[4 * k1 + 3];
      dft4<DIR>(a, b, c, d);
      y[k1] = a;
      y[k1 + 4] = b;
      y[k1 + 8] = c;
      y[k1 + 12] = d;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = y[i];
  }
};

}  // namespace expd
