// k_dst.cu -- K2/K3/K4: the orthonormal DST-I V ("L_h = V_h D_h V_h^{-1}"
// with V_h orthogonal; reading R1) along every axis of a slice, and the space-local
// nonlinear pass N-hat = V N(V u-hat) of the Picard sweep (stage 3; BASELINE.json:5).
//
// Algorithm: with M = n+1 = 2^m and F_j = sum_i x_i sin(pi i j / M),
//   y_0 = 0, y_i = sin(pi i/M)(x_i + x_{M-i}) + (x_i - x_{M-i})/2          (i = 1..M-1)
//   Y_k = sum_i y_i e^{-2 pi i ik/M}                                         (complex FFT)
//   F_{2k} = -Im Y_k,  F_1 = Re Y_0 / 2,  F_{2k+1} = F_{2k-1} + Re Y_k       (prefix sum)
// and V x = sqrt(2/M) F.  Two real lines travel as one complex sequence (their Y's are
// separated with the k <-> M-k Hermitian pairing), so one complex FFT of length M
// transforms two lines.  For strided axes the two lines are two adjacent columns, i.e.
// one 16-byte double2 per grid row in the padded spectral layout.
//
// One CTA owns PP line pairs in shared memory ([M][PP] complex, pair index fastest:
// conflict-free 16-byte accesses) and runs: load -> preprocess -> in-place Stockham
// radix-16 FFT -> Hermitian unpack -> chunked prefix sum -> scale -> store.  The fused
// nonlinear column kernel does transform -> N(u) pointwise -> transform in one visit.
#include "expd_internal.h"
#include "fft_dev.cuh"

namespace expd {

struct Poly {
  int npoly;
  double q[8];
};

__device__ __forceinline__ double poly_eval(const Poly& P, double u) {
  double acc = 0.0;
  for (int k = P.npoly - 1; k >= 0; --k) acc = fma(acc, u, P.q[k]);
  return acc;
}

template <int M>
struct DstCfg {
  static constexpr int PPmax = 4096 / M;
  static constexpr int PP = PPmax < M / 2 ? PPmax : (M / 2 > 0 ? M / 2 : 1);  // line pairs / CTA
  static constexpr int THREADS = (PP * M / 16) < 32 ? 32 : PP * M / 16;
  static constexpr int C = (M / 16 < 1) ? 1 : (M / 16 > 32 ? 32 : M / 16);  // scan chunks / pair
  static constexpr int L = (M / 2) / C;
};

// One in-place Stockham pass of radix R with NS = product of earlier radices.
template <int M, int PP, int THREADS, int R, int NS>
__device__ __forceinline__ void stockham_pass(double2* A, const double2* __restrict__ tw) {
  constexpr int JOBS = PP * M / R;
  constexpr int JT = (JOBS + THREADS - 1) / THREADS;
  double2 v[JT][R];
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * THREADS;
    if (J < JOBS) {
      const int p = J % PP, j = J / PP, k = j % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[jt][r] = A[(j + r * (M / R)) * PP + p];
      if constexpr (NS > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) v[jt][r] = cmul(v[jt][r], __ldg(tw + ((r * k * (M / (NS * R))) % M)));
      }
      DFT<R, -1>::run(v[jt]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * THREADS;
    if (J < JOBS) {
      const int p = J % PP, j = J / PP, k = j % NS;
      const int base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) A[(base + r * NS) * PP + p] = v[jt][r];
    }
  }
  __syncthreads();
}

template <int M, int PP, int THREADS>
__device__ __forceinline__ void fft_smem(double2* A, const double2* tw) {
  if constexpr (M == 4) {
    stockham_pass<M, PP, THREADS, 4, 1>(A, tw);
  } else if constexpr (M == 8) {
    stockham_pass<M, PP, THREADS, 8, 1>(A, tw);
  } else if constexpr (M == 16) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
  } else if constexpr (M == 32) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 2, 16>(A, tw);
  } else if constexpr (M == 64) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 4, 16>(A, tw);
  } else if constexpr (M == 128) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 8, 16>(A, tw);
  } else if constexpr (M == 256) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 16, 16>(A, tw);
  } else if constexpr (M == 512) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 16, 16>(A, tw);
    stockham_pass<M, PP, THREADS, 2, 256>(A, tw);
  } else if constexpr (M == 1024) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 16, 16>(A, tw);
    stockham_pass<M, PP, THREADS, 4, 256>(A, tw);
  } else if constexpr (M == 2048) {
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 16, 16>(A, tw);
    stockham_pass<M, PP, THREADS, 8, 256>(A, tw);
  } else {
    static_assert(M == 4096, "unsupported M");
    stockham_pass<M, PP, THREADS, 16, 1>(A, tw);
    stockham_pass<M, PP, THREADS, 16, 16>(A, tw);
    stockham_pass<M, PP, THREADS, 16, 256>(A, tw);
  }
}

// In: A[i][p] = z_i for i = 1..M-1 (A[0] ignored).  Out: A[pos][p] = F_{pos+1} (unscaled)
// for pos = 0..M-2.  tot: [C][PP] scratch.  Begins and ends with all threads synced.
template <int M>
__device__ __forceinline__ void dst_core(double2* A, double2* tot, const double2* tw, const double* sinp) {
  using Cf = DstCfg<M>;
  constexpr int PP = Cf::PP, THREADS = Cf::THREADS, C = Cf::C, L = Cf::L;
  const int tid = threadIdx.x;
  // preprocess: pairs (i, M-i), i = 1..M/2
  for (int J = tid; J < PP * (M / 2); J += THREADS) {
    const int p = J % PP, i = J / PP + 1;
    const double s = __ldg(sinp + i);
    double2 a = A[i * PP + p];
    if (i == M / 2) {
      A[i * PP + p] = make_double2(2.0 * s * a.x, 2.0 * s * a.y);
    } else {
      double2 b = A[(M - i) * PP + p];
      double2 sum = cadd(a, b), dif = csub(a, b);
      A[i * PP + p] = make_double2(fma(s, sum.x, 0.5 * dif.x), fma(s, sum.y, 0.5 * dif.y));
      A[(M - i) * PP + p] = make_double2(fma(s, sum.x, -0.5 * dif.x), fma(s, sum.y, -0.5 * dif.y));
    }
  }
  for (int p = tid; p < PP; p += THREADS) A[p] = make_double2(0.0, 0.0);
  __syncthreads();
  fft_smem<M, PP, THREADS>(A, tw);
  // Hermitian unpack of the two lines: even outputs and the prefix-sum increments w_k
  constexpr int KJ = (PP * (M / 2) + THREADS - 1) / THREADS;
  double2 ev[KJ], wv[KJ];
#pragma unroll
  for (int jt = 0; jt < KJ; ++jt) {
    const int J = tid + jt * THREADS;
    if (J < PP * (M / 2)) {
      const int p = J % PP, k = J / PP;
      double2 Zk = A[k * PP + p], Zm = A[((M - k) % M) * PP + p];
      ev[jt] = make_double2(-0.5 * (Zk.y - Zm.y), 0.5 * (Zk.x - Zm.x));
      wv[jt] = make_double2(0.5 * (Zk.x + Zm.x), 0.5 * (Zk.y + Zm.y));
      if (k == 0) wv[jt] = make_double2(0.5 * wv[jt].x, 0.5 * wv[jt].y);
    }
  }
  __syncthreads();
#pragma unroll
  for (int jt = 0; jt < KJ; ++jt) {
    const int J = tid + jt * THREADS;
    if (J < PP * (M / 2)) {
      const int p = J % PP, k = J / PP;
      if (k >= 1) A[(2 * k - 1) * PP + p] = ev[jt];
      A[(2 * k) * PP + p] = wv[jt];
    }
  }
  __syncthreads();
  // chunked inclusive scan of A[2k], k = 0..M/2-1, per pair
  const int p = tid % PP, c = tid / PP;
  double2 acc = make_double2(0.0, 0.0);
  if (c < C) {
#pragma unroll 4
    for (int l = 0; l < L; ++l) {
      const int k = c * L + l;
      acc = cadd(acc, A[(2 * k) * PP + p]);
      A[(2 * k) * PP + p] = acc;
    }
    tot[c * PP + p] = acc;
  }
  __syncthreads();
  if (c < C && c > 0) {
    double2 off = make_double2(0.0, 0.0);
    for (int cc = 0; cc < c; ++cc) off = cadd(off, tot[cc * PP + p]);
#pragma unroll 4
    for (int l = 0; l < L; ++l) {
      const int k = c * L + l;
      A[(2 * k) * PP + p] = cadd(A[(2 * k) * PP + p], off);
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------
// x-axis (contiguous) transform of row pairs.  rows_per_slice = n^{dim-1}.
// in: row r of slice s at in + s*in_slice + r*in_rs; out likewise.  NLOAD: apply N(u)
// to the loaded values (physical input); NLMID: transform, N, transform (dim == 1).
// ---------------------------------------------------------------------------------------
template <int M, bool NLOAD, bool NLMID>
__global__ void __launch_bounds__(DstCfg<M>::THREADS) k_dst_rows(const double* __restrict__ in, long in_slice,
                                                                 int in_rs, double* __restrict__ out,
                                                                 long out_slice, int out_rs, int rows_per_slice,
                                                                 const double2* tw, const double* sinp, Poly poly) {
  using Cf = DstCfg<M>;
  constexpr int PP = Cf::PP, THREADS = Cf::THREADS;
  constexpr int n = M - 1;
  extern __shared__ double2 sm[];
  double2* A = sm;
  double2* tot = sm + M * PP;
  const long slice = blockIdx.y;
  const int pair0 = blockIdx.x * PP;
  const double* inS = in + slice * in_slice;
  double* outS = out + slice * out_slice;
  // load: 2*PP rows, n values each, lanes along the row (coalesced)
  for (int J = threadIdx.x; J < 2 * PP * n; J += THREADS) {
    const int rr = J / n, i = J % n;  // local row, position
    const int p = rr >> 1, half = rr & 1;
    const int row = 2 * (pair0 + p) + half;
    double v = 0.0;
    if (row < rows_per_slice) v = __ldg(inS + (long)row * in_rs + i);
    if constexpr (NLOAD) v = poly_eval(poly, v);
    double* slot = reinterpret_cast<double*>(&A[(i + 1) * PP + p]) + half;
    *slot = v;
  }
  __syncthreads();
  dst_core<M>(A, tot, tw, sinp);
  const double scale = sqrt(2.0 / (double)M);
  if constexpr (NLMID) {
    // A[pos] = F_{pos+1}: physical values u = scale * F; N(u) moves to slot pos+1
    constexpr int JT = (PP * n + THREADS - 1) / THREADS;
    double2 tmp[JT];
#pragma unroll
    for (int jt = 0; jt < JT; ++jt) {
      const int J = threadIdx.x + jt * THREADS;
      if (J < PP * n) {
        double2 u = A[(J / PP) * PP + (J % PP)];
        tmp[jt] = make_double2(poly_eval(poly, scale * u.x), poly_eval(poly, scale * u.y));
      }
    }
    __syncthreads();
#pragma unroll
    for (int jt = 0; jt < JT; ++jt) {
      const int J = threadIdx.x + jt * THREADS;
      if (J < PP * n) A[(J / PP + 1) * PP + (J % PP)] = tmp[jt];
    }
    __syncthreads();
    dst_core<M>(A, tot, tw, sinp);
  }
  // store rows (out_rs == M: padded spectral row, write 0 at the pad position)
  for (int J = threadIdx.x; J < 2 * PP * out_rs; J += THREADS) {
    const int rr = J / out_rs, i = J % out_rs;
    const int p = rr >> 1, half = rr & 1;
    const int row = 2 * (pair0 + p) + half;
    if (row < rows_per_slice) {
      double v = 0.0;
      if (i < n) v = scale * reinterpret_cast<const double*>(&A[i * PP + p])[half];
      outS[(long)row * out_rs + i] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// strided-axis transform of column pairs in the padded spectral layout.
// line pair lp = (o, cp): base = o*outer_stride + 2*cp, element i at base + i*stride.
// NLMID: transform, N(u) pointwise, transform (the fused stage-3 visit).
// ---------------------------------------------------------------------------------------
template <int M, bool NLMID>
__global__ void __launch_bounds__(DstCfg<M>::THREADS) k_dst_cols(const double* in, long in_slice, double* out,
                                                                 long out_slice, long stride, long outer_stride,
                                                                 const double2* tw, const double* sinp,
                                                                 Poly poly) {
  using Cf = DstCfg<M>;
  constexpr int PP = Cf::PP, THREADS = Cf::THREADS;
  constexpr int n = M - 1;
  constexpr int GROUPS = (M / 2) / PP;  // column-pair groups per outer index
  extern __shared__ double2 sm[];
  double2* A = sm;
  double2* tot = sm + M * PP;
  const long slice = blockIdx.y;
  const long o = blockIdx.x / GROUPS;
  const int cp0 = (blockIdx.x % GROUPS) * PP;
  const double* inB = in + slice * in_slice + o * outer_stride + 2 * cp0;
  double* outB = out + slice * out_slice + o * outer_stride + 2 * cp0;
  for (int J = threadIdx.x; J < PP * n; J += THREADS) {
    const int p = J % PP, i = J / PP;
    A[(i + 1) * PP + p] = __ldg(reinterpret_cast<const double2*>(inB + (long)i * stride) + p);
  }
  __syncthreads();
  dst_core<M>(A, tot, tw, sinp);
  const double scale = sqrt(2.0 / (double)M);
  if constexpr (NLMID) {
    constexpr int JT = (PP * n + THREADS - 1) / THREADS;
    double2 tmp[JT];
#pragma unroll
    for (int jt = 0; jt < JT; ++jt) {
      const int J = threadIdx.x + jt * THREADS;
      if (J < PP * n) {
        double2 u = A[(J / PP) * PP + (J % PP)];
        tmp[jt] = make_double2(poly_eval(poly, scale * u.x), poly_eval(poly, scale * u.y));
      }
    }
    __syncthreads();
#pragma unroll
    for (int jt = 0; jt < JT; ++jt) {
      const int J = threadIdx.x + jt * THREADS;
      if (J < PP * n) A[(J / PP + 1) * PP + (J % PP)] = tmp[jt];
    }
    __syncthreads();
    dst_core<M>(A, tot, tw, sinp);
  }
  for (int J = threadIdx.x; J < PP * n; J += THREADS) {
    const int p = J % PP, i = J / PP;
    double2 v = A[i * PP + p];
    reinterpret_cast<double2*>(outB + (long)i * stride)[p] = make_double2(scale * v.x, scale * v.y);
  }
}

// ---------------------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------------------
template <int M>
static size_t dst_smem() {
  return sizeof(double2) * (size_t)(M * DstCfg<M>::PP + DstCfg<M>::C * DstCfg<M>::PP);
}

template <int M, bool A_, bool B_>
static cudaError_t rows_launch(const double* in, long in_slice, int in_rs, double* out, long out_slice, int out_rs,
                               int rows, long nslices, const DstTables& t, const Poly& P, cudaStream_t st) {
  auto k = k_dst_rows<M, A_, B_>;
  static bool attr = false;
  size_t sm = dst_smem<M>();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int pairs = (rows + 1) / 2;
  dim3 grid((pairs + DstCfg<M>::PP - 1) / DstCfg<M>::PP, (unsigned)nslices);
  k<<<grid, DstCfg<M>::THREADS, sm, st>>>(in, in_slice, in_rs, out, out_slice, out_rs, rows, t.tw, t.sinp, P);
  return cudaGetLastError();
}

template <int M, bool NL>
static cudaError_t cols_launch(const double* in, long in_slice, double* out, long out_slice, long stride,
                               long outer_stride, long nouter, long nslices, const DstTables& t, const Poly& P,
                               cudaStream_t st) {
  auto k = k_dst_cols<M, NL>;
  static bool attr = false;
  size_t sm = dst_smem<M>();
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((unsigned)(nouter * ((M / 2) / DstCfg<M>::PP)), (unsigned)nslices);
  k<<<grid, DstCfg<M>::THREADS, sm, st>>>(in, in_slice, out, out_slice, stride, outer_stride, t.tw, t.sinp, P);
  return cudaGetLastError();
}

struct RowsOp {
  const double* in; long in_slice; int in_rs; double* out; long out_slice; int out_rs; int rows; long nslices;
  bool nlload, nlmid;
};
struct ColsOp {
  const double* in; long in_slice; double* out; long out_slice; long stride, outer_stride, nouter, nslices;
  bool nl;
};

template <int M>
static cudaError_t run_rows(const RowsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  if (o.nlload) return rows_launch<M, true, false>(o.in, o.in_slice, o.in_rs, o.out, o.out_slice, o.out_rs, o.rows, o.nslices, t, P, st);
  if (o.nlmid) return rows_launch<M, false, true>(o.in, o.in_slice, o.in_rs, o.out, o.out_slice, o.out_rs, o.rows, o.nslices, t, P, st);
  return rows_launch<M, false, false>(o.in, o.in_slice, o.in_rs, o.out, o.out_slice, o.out_rs, o.rows, o.nslices, t, P, st);
}
template <int M>
static cudaError_t run_cols(const ColsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  if (o.nl) return cols_launch<M, true>(o.in, o.in_slice, o.out, o.out_slice, o.stride, o.outer_stride, o.nouter, o.nslices, t, P, st);
  return cols_launch<M, false>(o.in, o.in_slice, o.out, o.out_slice, o.stride, o.outer_stride, o.nouter, o.nslices, t, P, st);
}

template <int M> struct RowsCall { static cudaError_t go(const RowsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) { return run_rows<M>(o, t, P, st); } };
template <int M> struct ColsCall { static cudaError_t go(const ColsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) { return run_cols<M>(o, t, P, st); } };

static cudaError_t rows(int M, const RowsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  switch (M) {
    case 4: return RowsCall<4>::go(o, t, P, st);
    case 8: return RowsCall<8>::go(o, t, P, st);
    case 16: return RowsCall<16>::go(o, t, P, st);
    case 32: return RowsCall<32>::go(o, t, P, st);
    case 64: return RowsCall<64>::go(o, t, P, st);
    case 128: return RowsCall<128>::go(o, t, P, st);
    case 256: return RowsCall<256>::go(o, t, P, st);
    case 512: return RowsCall<512>::go(o, t, P, st);
    case 1024: return RowsCall<1024>::go(o, t, P, st);
    case 2048: return RowsCall<2048>::go(o, t, P, st);
    case 4096: return RowsCall<4096>::go(o, t, P, st);
    default: return cudaErrorInvalidValue;
  }
}
static cudaError_t cols(int M, const ColsOp& o, const DstTables& t, const Poly& P, cudaStream_t st) {
  switch (M) {
    case 4: return ColsCall<4>::go(o, t, P, st);
    case 8: return ColsCall<8>::go(o, t, P, st);
    case 16: return ColsCall<16>::go(o, t, P, st);
    case 32: return ColsCall<32>::go(o, t, P, st);
    case 64: return ColsCall<64>::go(o, t, P, st);
    case 128: return ColsCall<128>::go(o, t, P, st);
    case 256: return ColsCall<256>::go(o, t, P, st);
    case 512: return ColsCall<512>::go(o, t, P, st);
    case 1024: return ColsCall<1024>::go(o, t, P, st);
    case 2048: return ColsCall<2048>::go(o, t, P, st);
    case 4096: return ColsCall<4096>::go(o, t, P, st);
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

cudaError_t dst_slices(const Geom& g, const DstTables& t, const double* src, bool src_spectral, double* dst,
                       bool dst_spectral, long nslices, double* scratch, cudaStream_t st) {
  if (nslices <= 0) return cudaSuccess;
  Poly P = make_poly(0, nullptr);
  const int rows_ps = (int)(g.N / g.n);
  const long phys_slice = g.N;
  if (!src_spectral && dst_spectral) {
    // physical -> spectral: x first (into dst), then strided axes in place
    RowsOp r{src, phys_slice, g.n, dst, g.npad, g.M, rows_ps, nslices, false, false};
    CK(rows(g.M, r, t, P, st));
    for (int ax = 1; ax < g.dim; ++ax) CK(cols(g.M, col_op(g, ax, dst, dst, nslices, false), t, P, st));
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
        CK(cols(g.M, col_op(g, ax, cur, scratch, ns, false), t, P, st));
        cur = scratch;
      }
      RowsOp r{cur, g.npad, g.M, dst + s0 * phys_slice, phys_slice, g.n, rows_ps, ns, false, false};
      CK(rows(g.M, r, t, P, st));
    }
    return cudaSuccess;
  }
  if (src_spectral && dst_spectral) {
    RowsOp r{src, g.npad, g.M, dst, g.npad, g.M, rows_ps, nslices, false, false};
    CK(rows(g.M, r, t, P, st));
    for (int ax = 1; ax < g.dim; ++ax) CK(cols(g.M, col_op(g, ax, dst, dst, nslices, false), t, P, st));
    return cudaSuccess;
  }
  return cudaErrorInvalidValue;
}

int nonlin_chunk_slices(const Geom& g) {
  // keep one chunk's intermediate (npad doubles per slice) around 32 MB so it stays in L2
  long per = g.npad * 8;
  long c = (32l << 20) / (per > 0 ? per : 1);
  return (int)(c < 1 ? 1 : (c > 64 ? 64 : c));
}

int nonlin_kernel_launches(const Geom& g, long nslices) {
  long chunk = nonlin_chunk_slices(g);
  long nch = (nslices + chunk - 1) / chunk;
  int per = g.dim == 1 ? 1 : (g.dim == 2 ? 3 : 5);
  return (int)(nch * per);
}

cudaError_t nonlin_slices(const Geom& g, const DstTables& t, const double* uhat, double* nhat, long nslices,
                          int npoly, const double* q, double* scratch, cudaStream_t st) {
  Poly P = make_poly(npoly, q);
  const int rows_ps = (int)(g.N / g.n);
  const long chunk = nonlin_chunk_slices(g);
  for (long s0 = 0; s0 < nslices; s0 += chunk) {
    long ns = nslices - s0 < chunk ? nslices - s0 : chunk;
    const double* in = uhat + s0 * g.npad;
    double* out = nhat + s0 * g.npad;
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
  return cudaSuccess;
}

cudaError_t nonlin_phys_slices(const Geom& g, const DstTables& t, const double* u, double* nhat, long nslices,
                               int npoly, const double* q, double* scratch, cudaStream_t st) {
  (void)scratch;
  Poly P = make_poly(npoly, q);
  const int rows_ps = (int)(g.N / g.n);
  RowsOp r{u, g.N, g.n, nhat, g.npad, g.M, rows_ps, nslices, true, false};
  CK(rows(g.M, r, t, P, st));
  for (int ax = 1; ax < g.dim; ++ax) CK(cols(g.M, col_op(g, ax, nhat, nhat, nslices, false), t, P, st));
  return cudaSuccess;
}

size_t dst_scratch_doubles(const Geom& g, long max_slices) { return (size_t)g.npad * (size_t)max_slices; }

}  // namespace expd
