// k_vec.cu -- per-mode multiplier tables, deterministic reductions, and the GMRES
// (classical Gram-Schmidt twice, R11) vector kernels K6/K7 (stage 4 of the hot path,
// BASELINE.json:5 "dot products and norms for the preconditioned-GMRES variant").
// Reductions are warp-shuffle + fixed-order block sums into per-CTA partials, then a
// fixed-order single-CTA sum: the result does not depend on scheduling.
#include "expd_internal.h"

namespace expd {

// ---------------------------------------------------------------------------------------
// E_J = exp(dt mu_J), mu_J = a sum_axes lambda_{j} - c (R1);
// ETD1: C1 = dt phi1(z); ETD2: C1 = dt (phi1 + phi2)(z), C2 = dt phi2(z), z = dt mu_J (R5,
// R6); Taylor series for |z| < 1/2 (R7).  Pad modes (jx = n) get 0.
// ---------------------------------------------------------------------------------------
__device__ void phi12(double z, double* p1, double* p2) {
  if (fabs(z) < 0.5) {
    // Horner on sum_k z^k/(k+1)! and sum_k z^k/(k+2)!, 22 terms (|z|^22/23! < 1e-29)
    double a = 0.0, b = 0.0;
    for (int k = 21; k >= 0; --k) {
      double f1 = 1.0, f2 = 1.0;
      // 1/(k+1)! and 1/(k+2)! computed exactly enough in double by a short product
      for (int i = 2; i <= k + 1; ++i) f1 /= (double)i;
      f2 = f1 / (double)(k + 2);
      a = fma(a, z, f1);
      b = fma(b, z, f2);
    }
    *p1 = a;
    *p2 = b;
  } else {
    double em1 = expm1(z);
    *p1 = em1 / z;
    *p2 = (em1 - z) / (z * z);
  }
}

__global__ void k_mode_tables(int dim, int n, int M, long npad, const double* lam, double a, double c, double dt,
                              int scheme, double* E, double* C1, double* C2) {
  for (long J = blockIdx.x * (long)blockDim.x + threadIdx.x; J < npad; J += (long)gridDim.x * blockDim.x) {
    const int jx = (int)(J % M);
    double e = 0.0, c1 = 0.0, c2 = 0.0;
    if (jx < n) {
      long r = J / M;
      double s = lam[jx];
      for (int ax = 1; ax < dim; ++ax) {
        s += lam[r % n];
        r /= n;
      }
      const double mu = a * s - c;
      const double z = dt * mu;
      e = exp(z);
      double p1, p2;
      phi12(z, &p1, &p2);
      if (scheme == 0) {
        c1 = dt * p1;
      } else if (scheme == 2) {  // IF / IMEX-type: dt N(u_n), no phi
        c1 = dt;
      } else {
        c1 = dt * (p1 + p2);
        c2 = dt * p2;
      }
    }
    E[J] = e;
    if (C1) C1[J] = c1;
    if (C2) C2[J] = c2;
  }
}

cudaError_t mode_tables(const Geom& g, const double* lam_axis, double a, double c, double dt, int scheme,
                        double* E, double* C1, double* C2, cudaStream_t st) {
  k_mode_tables<<<1024, 256, 0, st>>>(g.dim, g.n, g.M, g.npad, lam_axis, a, c, dt, scheme, E, C1, C2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// block reduction helper (256 threads)
// ---------------------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* out, int stride) {
  __shared__ double red[NV][8];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double x = v[i];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double x = 0.0;
    for (int w = 0; w < 8; ++w) x += red[threadIdx.x][w];
    out[threadIdx.x * stride + blockIdx.x] = x;
  }
}

__global__ void k_reduce_rows(const double* partial, int n, int rows, double* out) {
  // one warp per row, fixed lane order, then fixed shuffle tree
  const int row = blockIdx.x;
  if (row >= rows) return;
  double x = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) x += partial[(long)row * n + i];
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (threadIdx.x == 0) out[row] = x;
}

cudaError_t reduce_partials(const double* partial, int n, double* out, cudaStream_t st) {
  k_reduce_rows<<<1, 32, 0, st>>>(partial, n, 1, out);
  return cudaGetLastError();
}

int vec_grid(int sms) { return sms * 4; }

// The convergence test of the fixed-point / Picard iteration (R8) on the device: the body of
// the CUDA-graph WHILE loop of expd_fixed_point_solve (one sweep, the norm reduction, then
// this kernel).  rho_k = ||r^k|| / ||r^0||; stop on rho_k < tol (converged), on a non-finite
// norm (breakdown) or after sweep maxit; otherwise k += 1 and the loop runs another sweep.
__global__ void k_fp_conv(cudaGraphConditionalHandle h, FpLoopState* st, const double* norm2) {
  if (threadIdx.x != 0) return;
  const int k = st->k;
  const double n2 = norm2[0];
  unsigned int again = 0;
  if (!isfinite(n2)) {
    st->hist[k] = n2;
    st->status = 6;  // EXPD_ERR_BREAKDOWN
  } else {
    const double rn = sqrt(n2);
    if (k == 0) st->r0 = rn;
    const double rho = st->r0 > 0.0 ? rn / st->r0 : 0.0;
    st->hist[k] = rho;
    if (rho < st->tol) {
      st->status = 0;
    } else if (k >= st->maxit) {
      st->status = 7;  // EXPD_ERR_NOT_CONVERGED
    } else {
      st->k = k + 1;
      again = 1;
    }
  }
  st->s3skip = 0;  // only the first sweep of a zero-guess solve skips stage 3
  cudaGraphSetConditional(h, again);
}

cudaError_t launch_fp_conv(cudaGraphConditionalHandle h, FpLoopState* st, const double* norm2, cudaStream_t s) {
  k_fp_conv<<<1, 32, 0, s>>>(h, st, norm2);
  return cudaGetLastError();
}

struct VecPtrs {
  const double* v[32];
};

// h_i = <V_i, w>, i < nv   (K6 pass 1).  CX: the vectors are complex (interleaved), the
// inner product is the Hermitian one, h_i = sum conj(V_i) w -> (re, im) = rows 2i, 2i+1
// (complex GMRES, reading R18).
template <int NV, bool CX = false>
__global__ void __launch_bounds__(256) k_multi_dot(VecPtrs V, const double* __restrict__ w, long len2,
                                                   double* partial) {
  constexpr int NA = CX ? 2 * NV : NV;
  double acc[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < len2; e += (long)gridDim.x * blockDim.x) {
    double2 x = __ldcs(w2 + e);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double2 v = __ldcs(reinterpret_cast<const double2*>(V.v[i]) + e);
      if constexpr (CX) {
        acc[2 * i] = fma(v.x, x.x, fma(v.y, x.y, acc[2 * i]));
        acc[2 * i + 1] = fma(v.x, x.y, fma(-v.y, x.x, acc[2 * i + 1]));
      } else {
        acc[i] = fma(v.x, x.x, fma(v.y, x.y, acc[i]));
      }
    }
  }
  block_sum_store<NA>(acc, partial, gridDim.x);
}

// w <- w - sum_i coef_i V_i ; then (WANT == 1) h2_i = <V_i, w> or (WANT == 2) ||w||^2.
// CX: complex coefficients (coef[2i], coef[2i+1]) and the Hermitian h2_i (rows 2i, 2i+1).
template <int NV, int WANT, bool CX = false>
__global__ void __launch_bounds__(256) k_axpy_dot(VecPtrs V, const double* __restrict__ coef, double* w, long len2,
                                                  double* partial) {
  constexpr int NO = WANT == 1 ? (CX ? 2 * NV : NV) : 1;
  double acc[NO];
#pragma unroll
  for (int i = 0; i < NO; ++i) acc[i] = 0.0;
  double2 cf[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) cf[i] = CX ? make_double2(coef[2 * i], coef[2 * i + 1]) : make_double2(coef[i], 0.0);
  double2* w2 = reinterpret_cast<double2*>(w);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < len2; e += (long)gridDim.x * blockDim.x) {
    double2 x = w2[e];
    double2 vv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      vv[i] = __ldcs(reinterpret_cast<const double2*>(V.v[i]) + e);
      if constexpr (CX) {  // x -= cf * v (complex)
        x.x = fma(-cf[i].x, vv[i].x, fma(cf[i].y, vv[i].y, x.x));
        x.y = fma(-cf[i].x, vv[i].y, fma(-cf[i].y, vv[i].x, x.y));
      } else {
        x.x = fma(-cf[i].x, vv[i].x, x.x);
        x.y = fma(-cf[i].x, vv[i].y, x.y);
      }
    }
    w2[e] = x;
    if constexpr (WANT == 1) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        if constexpr (CX) {
          acc[2 * i] = fma(vv[i].x, x.x, fma(vv[i].y, x.y, acc[2 * i]));
          acc[2 * i + 1] = fma(vv[i].x, x.y, fma(-vv[i].y, x.x, acc[2 * i + 1]));
        } else {
          acc[i] = fma(vv[i].x, x.x, fma(vv[i].y, x.y, acc[i]));
        }
      }
    } else if constexpr (WANT == 2) {
      acc[0] = fma(x.x, x.x, fma(x.y, x.y, acc[0]));
    }
  }
  if constexpr (WANT > 0) block_sum_store<NO>(acc, partial, gridDim.x);
}

// x <- x + sum_i coef_i V_i   (K7); CX: complex coefficients (coef[2i], coef[2i+1])
template <int NV, bool CX = false>
__global__ void __launch_bounds__(256) k_lincomb(VecPtrs V, const double* __restrict__ coef, double* x, long len2) {
  double2 cf[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) cf[i] = CX ? make_double2(coef[2 * i], coef[2 * i + 1]) : make_double2(coef[i], 0.0);
  double2* x2 = reinterpret_cast<double2*>(x);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < len2; e += (long)gridDim.x * blockDim.x) {
    double2 a = x2[e];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double2 v = __ldcs(reinterpret_cast<const double2*>(V.v[i]) + e);
      if constexpr (CX) {
        a.x = fma(cf[i].x, v.x, fma(-cf[i].y, v.y, a.x));
        a.y = fma(cf[i].x, v.y, fma(cf[i].y, v.x, a.y));
      } else {
        a.x = fma(cf[i].x, v.x, a.x);
        a.y = fma(cf[i].x, v.y, a.y);
      }
    }
    x2[e] = a;
  }
}

__global__ void k_scale_copy(const double* __restrict__ x, double s, double* y, long len2) {
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double2* y2 = reinterpret_cast<double2*>(y);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < len2; e += (long)gridDim.x * blockDim.x) {
    double2 a = __ldcs(x2 + e);
    y2[e] = make_double2(s * a.x, s * a.y);
  }
}

#define NV_SWITCH(nv, EXPR)                                                           \
  switch (nv) {                                                                       \
    case 1: { constexpr int NVc = 1; EXPR; } break;                                   \
    case 2: { constexpr int NVc = 2; EXPR; } break;                                   \
    case 3: { constexpr int NVc = 3; EXPR; } break;                                   \
    case 4: { constexpr int NVc = 4; EXPR; } break;                                   \
    case 5: { constexpr int NVc = 5; EXPR; } break;                                   \
    case 6: { constexpr int NVc = 6; EXPR; } break;                                   \
    case 7: { constexpr int NVc = 7; EXPR; } break;                                   \
    case 8: { constexpr int NVc = 8; EXPR; } break;                                   \
    default: return cudaErrorInvalidValue;                                            \
  }

static VecPtrs pack(const double* const* V, int nv) {
  VecPtrs p{};
  for (int i = 0; i < nv && i < 32; ++i) p.v[i] = V[i];
  return p;
}

// For nv > 8 the vectors are processed in groups of up to 8 (one extra pass over w per
// group); restart <= 8 keeps every CGS2 sweep a single pass.
// cx: complex vectors / coefficients, every coefficient or inner product is 2 doubles
// (re, im) in the device arrays (out, coef_dev).
cudaError_t multi_dot(const double* const* V, int nv, const double* w, long len, double* partial, int grid,
                      double* out, cudaStream_t st, bool cx) {
  const long len2 = len / 2;
  const int K = cx ? 2 : 1;
  for (int g0 = 0; g0 < nv; g0 += 8) {
    int ng = nv - g0 < 8 ? nv - g0 : 8;
    VecPtrs p = pack(V + g0, ng);
    if (cx) NV_SWITCH(ng, (k_multi_dot<NVc, true><<<grid, 256, 0, st>>>(p, w, len2, partial)))
    else NV_SWITCH(ng, (k_multi_dot<NVc, false><<<grid, 256, 0, st>>>(p, w, len2, partial)))
    k_reduce_rows<<<K * ng, 32, 0, st>>>(partial, grid, K * ng, out + K * g0);
  }
  return cudaGetLastError();
}

cudaError_t multi_axpy_dot(const double* const* V, int nv, const double* coef_dev, double* w, long len,
                           double* partial, int grid, double* out, int want_dot, cudaStream_t st, bool cx) {
  const long len2 = len / 2;
  const int K = cx ? 2 : 1;
  for (int g0 = 0; g0 < nv; g0 += 8) {
    int ng = nv - g0 < 8 ? nv - g0 : 8;
    VecPtrs p = pack(V + g0, ng);
    const bool last = g0 + ng >= nv;
    const double* cf = coef_dev + K * g0;
    if (last && want_dot == 2) {
      if (cx) NV_SWITCH(ng, (k_axpy_dot<NVc, 2, true><<<grid, 256, 0, st>>>(p, cf, w, len2, partial)))
      else NV_SWITCH(ng, (k_axpy_dot<NVc, 2, false><<<grid, 256, 0, st>>>(p, cf, w, len2, partial)))
      k_reduce_rows<<<1, 32, 0, st>>>(partial, grid, 1, out);
    } else if (last && want_dot == 1 && nv <= 8) {
      if (cx) NV_SWITCH(ng, (k_axpy_dot<NVc, 1, true><<<grid, 256, 0, st>>>(p, cf, w, len2, partial)))
      else NV_SWITCH(ng, (k_axpy_dot<NVc, 1, false><<<grid, 256, 0, st>>>(p, cf, w, len2, partial)))
      k_reduce_rows<<<K * ng, 32, 0, st>>>(partial, grid, K * ng, out);
    } else {
      if (cx) NV_SWITCH(ng, (k_axpy_dot<NVc, 0, true><<<grid, 256, 0, st>>>(p, cf, w, len2, partial)))
      else NV_SWITCH(ng, (k_axpy_dot<NVc, 0, false><<<grid, 256, 0, st>>>(p, cf, w, len2, partial)))
    }
  }
  if (want_dot == 1 && nv > 8) return multi_dot(V, nv, w, len, partial, grid, out, st, cx);
  return cudaGetLastError();
}

cudaError_t lincomb_add(const double* const* V, int nv, const double* coef_dev, double* x, long len,
                        cudaStream_t st, bool cx) {
  const long len2 = len / 2;
  const int K = cx ? 2 : 1;
  for (int g0 = 0; g0 < nv; g0 += 8) {
    int ng = nv - g0 < 8 ? nv - g0 : 8;
    VecPtrs p = pack(V + g0, ng);
    if (cx) NV_SWITCH(ng, (k_lincomb<NVc, true><<<vec_grid(148), 256, 0, st>>>(p, coef_dev + K * g0, x, len2)))
    else NV_SWITCH(ng, (k_lincomb<NVc, false><<<vec_grid(148), 256, 0, st>>>(p, coef_dev + K * g0, x, len2)))
  }
  return cudaGetLastError();
}

// rows of `width` doubles at stride in_rs -> stride out_rs (physical <-> padded spectral
// rows); the pad columns [width, out_rs) of the output are zeroed when out_rs > width.  Each
// block walks whole rows: coalesced 8-byte accesses (n odd: rows are not 16-byte aligned).
__global__ void __launch_bounds__(256) k_repitch(const double* __restrict__ in, long in_rs, double* __restrict__ out,
                                                 long out_rs, int width, long rows) {
  const int ow = out_rs > width ? (int)out_rs : width;
  for (long r = blockIdx.x; r < rows; r += gridDim.x) {
    const double* a = in + r * in_rs;
    double* b = out + r * out_rs;
#pragma unroll 4
    for (int i = threadIdx.x; i < ow; i += blockDim.x) {
      EXPD_CHECK(i < out_rs && (i >= width || i < in_rs), "repitch: row index");
      b[i] = i < width ? __ldcs(a + i) : 0.0;
    }
  }
}
cudaError_t repitch(const double* in, long in_rs, double* out, long out_rs, int width, long rows, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const long grid = rows < 148L * 16 ? rows : 148L * 16;
  k_repitch<<<(unsigned)grid, 256, 0, st>>>(in, in_rs, out, out_rs, width, rows);
  return cudaGetLastError();
}

// complex interleaved slices <-> planar (re slice, im slice) pairs: slice t of `in` (len
// complex entries at stride in_stride doubles) -> slices 2t, 2t+1 of `out` (stride
// out_stride).  Complex plans run the real DST on the planar pairs (V is real).
__global__ void k_cx_split(const double* __restrict__ in, long in_stride, long len, double* __restrict__ out,
                           long out_stride, long nslices) {
  const long total = len * nslices;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long t = e / len, i = e - t * len;
    const double2 v = __ldcs(reinterpret_cast<const double2*>(in + t * in_stride) + i);
    out[2 * t * out_stride + i] = v.x;
    out[(2 * t + 1) * out_stride + i] = v.y;
  }
}
__global__ void k_cx_merge(const double* __restrict__ in, long in_stride, long len, double* __restrict__ out,
                           long out_stride, long nslices) {
  const long total = len * nslices;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long t = e / len, i = e - t * len;
    const double2 v = make_double2(__ldcs(in + 2 * t * in_stride + i), __ldcs(in + (2 * t + 1) * in_stride + i));
    reinterpret_cast<double2*>(out + t * out_stride)[i] = v;
  }
}
cudaError_t cx_split(const double* in, long in_stride, long len, double* out, long out_stride, long nslices,
                     cudaStream_t st) {
  k_cx_split<<<1184, 256, 0, st>>>(in, in_stride, len, out, out_stride, nslices);
  return cudaGetLastError();
}
cudaError_t cx_merge(const double* in, long in_stride, long len, double* out, long out_stride, long nslices,
                     cudaStream_t st) {
  k_cx_merge<<<1184, 256, 0, st>>>(in, in_stride, len, out, out_stride, nslices);
  return cudaGetLastError();
}

// y = (s_re + i s_im) x on interleaved complex vectors (complex BiCGStab)
__global__ void k_scale_copy_cx(const double* __restrict__ x, double sr, double si, double* y, long len2) {
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double2* y2 = reinterpret_cast<double2*>(y);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < len2; e += (long)gridDim.x * blockDim.x) {
    double2 a = x2[e];
    y2[e] = make_double2(fma(sr, a.x, -si * a.y), fma(sr, a.y, si * a.x));
  }
}

cudaError_t scale_copy_cx(const double* x, double sr, double si, double* y, long len, cudaStream_t st) {
  k_scale_copy_cx<<<1184, 256, 0, st>>>(x, sr, si, y, len / 2);
  return cudaGetLastError();
}

cudaError_t scale_copy(const double* x, double s, double* y, long len, cudaStream_t st) {
  k_scale_copy<<<1184, 256, 0, st>>>(x, s, y, len / 2);
  return cudaGetLastError();
}

}  // namespace expd
