// k_line.cu -- K2/K3/K4 v2: the orthonormal DST-I V (L_h = V_h D_h V_h^{-1},
// V_h orthogonal; reading R1) along one axis of padded spectral slices, and the fused
// strided-axis pass [V, N(.), V] of stage 3 (N-hat = V N(V u-hat), BASELINE.json:5), for
// line lengths M = n+1 in {256, ..., 4096}.
//
// Same arithmetic as k_dst.cu (sinft pre-processing, complex FFT of two real lines packed
// as one complex sequence, Hermitian unpack, prefix sum for the odd outputs), re-organised
// around the Blackwell async-copy engine:
//   * persistent CTAs, one line pair per work item, two shared-memory buffers: the TMA
//     brings item i+1 while item i is transformed (no exposed HBM / L2 latency);
//   * x-axis (ROW) items: the two rows are loaded / stored as TMA tensor boxes
//     {16 doubles, M/16}: loaded linear (the stage-0 reads of x_i and of the mirror x_{M-i}
//     are runs of consecutive doubles per half-warp), stored with the 128-byte swizzle (the
//     per-thread chunk writes of the result, 128 bytes apart per lane, hit distinct banks);
//   * strided-axis (COL) items: one column pair (16 B per grid row) moved as TMA boxes
//     of {2 doubles, 256 rows} into / out of a linear layout (the result is compacted
//     from the padded work layout before the store);
//   * the last stage of the prefix sum leaves every thread 2L consecutive outputs
//     (F_{2k+1}, F_{2k+2}) pairs, written in the layout the TMA store reads.
// All loads and stores of the data go through the TMA: no thread issues a global access
// for the data, so the LSU carries only the twiddle / sine table reads.
//
// DST-I: with M = n+1 and F_j = sum_i x_i sin(pi i j / M),
//   y_0 = 0, y_i = sin(pi i/M)(x_i + x_{M-i}) + (x_i - x_{M-i})/2,   Y = FFT_M(y),
//   F_{2k} = -Im Y_k (k >= 1),  F_{2k+1} = sum_{k' <= k} Re Y_{k'} (Re Y_0 halved),
// V x = sqrt(2/M) F.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "expd_internal.h"
#include "fft_dev.cuh"
#include "tma_dev.cuh"

namespace expd {

// Radix plan: first radix R0 (fed by the pre-processing), middle radices RM1 (RM2 = 1
// here), last radix RL (run on Hermitian partner jobs).  T = M / R0 threads per line pair.
template <int M> struct LPlan;
template <> struct LPlan<256>  { static constexpr int R0 = 8,  RM1 = 4,  RL = 8; };
template <> struct LPlan<512>  { static constexpr int R0 = 16, RM1 = 4,  RL = 8; };
template <> struct LPlan<1024> { static constexpr int R0 = 16, RM1 = 8,  RL = 8; };
template <> struct LPlan<2048> { static constexpr int R0 = 16, RM1 = 16, RL = 8; };
template <> struct LPlan<4096> { static constexpr int R0 = 16, RM1 = 16, RL = 16; };

template <int M, int G, int NBUF>
struct LGeo {
  static constexpr int R0 = LPlan<M>::R0, RM1 = LPlan<M>::RM1, RL = LPlan<M>::RL;
  static_assert(R0 * RM1 * RL == M, "radix plan");
  static_assert(M % 256 == 0, "COL boxes of 256 rows");
  static constexpr int T = M / R0;            // threads per line pair
  static constexpr int THREADS = G * T;       // G line pairs per item (g = tid % G)
  static constexpr int NSL = M / RL;          // Ns of the last stage
  static constexpr int L = (M / 2) / T;       // k-values per thread in the prefix sum (= R0/2)
  static constexpr int PADP = R0;             // one pad slot per PADP positions
  static constexpr int SW = M + M / PADP;     // padded positions per line pair
  static constexpr int WS = (M / 2) / L * (L + 1);  // one unpacked array W or E (padded)
  static constexpr int SWB = SW > 2 * WS ? SW : 2 * WS;
  static constexpr int JW = 32 / G;           // threads of one line pair inside a warp
  static constexpr int NWB = T / JW;          // warp blocks per line pair
  static constexpr size_t BUFB = ((size_t)G * SWB * 16 + 1023) / 1024 * 1024;  // bytes per buffer
  // + the two TMA mbarriers and the kWarPoints write-after-read mbarriers
  static constexpr size_t SMEM = 1024 + NBUF * BUFB + 16 * (size_t)(NWB * G) + 48;
  // resident CTAs per SM: shared memory (228 KB, 1 KB reserved per CTA) and >= EXPD_LINE_REGS
  // registers per thread
#ifndef EXPD_LINE_REGS
#define EXPD_LINE_REGS 160
#endif
  static constexpr int MINB_SMEM = (int)((228 * 1024) / (SMEM + 1024));
  static constexpr int MINB_REG = 65536 / (THREADS * EXPD_LINE_REGS);
  static constexpr int MINB = MINB_SMEM < MINB_REG ? (MINB_SMEM > 0 ? MINB_SMEM : 1) : (MINB_REG > 0 ? MINB_REG : 1);
};

enum LineAxis { AX_ROW = 0, AX_COL_Y = 1, AX_COL_Z = 2 };
constexpr int CBR = 256;  // grid rows per TMA box of a strided-axis (COL) item

struct LineArgs {
  long nitems;
  int per_slice;   // items per slice
  int inner;       // ROW: row pairs per slice; COL: column-pair groups per outer index
  int rows;        // ROW: rows per slice (for the incomplete last pair)
  const double2* tw;   // [M] exp(-2 pi i q / M)
  const double* pa;    // [M] a_i = c (sin(pi i/M) + 1/2), c = sqrt(2/M)/2 (b_i = a_i - c)
  const double* sinp;  // [M] sin(pi i/M)
  double c;            // sqrt(2/M)/2
  Poly poly;
  const int* skip;     // device flag: non-zero -> the launch does nothing (nullable)
  const PeerMaps* peer;  // ROW only: store each row into its owner's N-hat slab (nullable)
  int peer_slot0;        // ... at slot peer_slot0 + slice
  const PeerMaps* peer_in;  // ROW only: load each row from its owner's U-hat slab (nullable)
  int peer_in_slot0;        // ... at slot peer_in_slot0 + slice
  double* outp;  // COL with the transposed store (TS): the output array (the tail rows' stores)
};

// The write-after-read points of the line transform (a stage reads the buffer, transforms in
// registers, writes the buffer).  WarSync (default): one __syncthreads before the writes.
// WarMbar (-DEXPD_WAR_MODE=1): a split barrier on an mbarrier per point -- each warp ARRIVES
// as soon as its reads are done (release) and WAITS (acquire) only before its writes, so the
// stage's DFT could overlap the slower warps' reads.  Measured (profiles/r02/war_barrier_ab.txt):
// dropping the three WAR barriers altogether (wrong results, timing only) would take stage 3
// from 15.8 to 14.8 ms on c5, but the split barrier is no faster than __syncthreads on c5 and
// 2 % slower on c3 (the mbarrier arrive / poll traffic goes through the same LSU pipe the
// transform is bound by).  Point k completes once per use; `ph` carries each point's phase
// parity (a point cannot complete twice before a warp waits on it: its next completion
// needs that warp's next arrival).
struct WarSync {
  __device__ __forceinline__ void arrive(int) {}
#ifdef EXPD_EXP_NOWAR  // timing experiment only (tools/gpu_r02s.sh): WRONG results
  __device__ __forceinline__ void wait(int) {}
#else
  __device__ __forceinline__ void wait(int) { __syncthreads(); }
#endif
};
struct WarMbar {
  uint64_t* b;  // kWarPoints mbarriers, count = warps of the CTA
  uint32_t ph;
  __device__ __forceinline__ void arrive(int k) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&b[k]);
  }
  __device__ __forceinline__ void wait(int k) {
    mbar_wait(&b[k], (ph >> k) & 1u);
    ph ^= 1u << k;
  }
};
// WarNone: the stages read and write different buffers (the ping-pong kernel k_line_pp): no
// write-after-read hazard, no barrier.
struct WarNone {
  __device__ __forceinline__ void arrive(int) {}
  __device__ __forceinline__ void wait(int) {}
};
// WarMask: the barrier of point k only where bit k is set (the hybrid buffer schedule of
// line_item HY, where a stage's output buffer is not the buffer its input is read from)
struct WarMask {
  unsigned m;
  __device__ __forceinline__ void arrive(int) {}
  __device__ __forceinline__ void wait(int k) {
    if ((m >> k) & 1u) __syncthreads();
  }
};
constexpr int kWarPoints = 3;  // 0: middle stage, 1: stage 0, 2: last stage -> unpack
#ifndef EXPD_LINE_DEFER
#define EXPD_LINE_DEFER 1  // defer the last prefix's cross-warp barrier (line_offw)
#endif
#ifndef EXPD_WAR_MODE
#define EXPD_WAR_MODE 0  // 0: WarSync in k_line, 1: WarMbar (A/B)
#endif

template <int PADP>
__device__ __forceinline__ int lswz(int p) { return p + p / PADP; }

// byte offset of double x of a row stored as TMA boxes {16, M/16} with the 128-byte swizzle
__device__ __forceinline__ uint32_t row_sw(int x) {
  const int o = x >> 4, c = x & 15;
  return (uint32_t)(o * 128 + ((((c >> 1) ^ (o & 7))) << 4) + ((c & 1) << 3));
}

// y_i = s_i (x_i + x_{M-i}) + (x_i - x_{M-i})/2 = a_i x_i + b_i x_{M-i} (times the folded scale
// c): a = c (s + 1/2), b = a - c
__device__ __forceinline__ double2 lpre(double2 z, double2 zm, double a, double c) {
  const double b = a - c;
  return make_double2(fma(a, z.x, b * zm.x), fma(a, z.y, b * zm.y));
}
// Hermitian unpack of the two real lines' transforms; the 1/2 of the textbook formulas and
// the orthonormal scale are folded into the pre-processing table (a_i, b_i)
__device__ __forceinline__ void lunpack(double2 Zk, double2 Zm, bool k0, double2& e, double2& w) {
  e = make_double2(Zm.y - Zk.y, Zk.x - Zm.x);
  w = make_double2(Zk.x + Zm.x, Zk.y + Zm.y);
  if (k0) w = make_double2(0.5 * w.x, 0.5 * w.y);
}
// v[r] *= w^{r b}, r = 1..R-1, from the single table entry w^b.  EXPD_LINE_TWSEQ: running
// product (two live twiddles, r roundings deep); default: binary splitting (all R powers
// live, <= 2 log2 R roundings deep).
template <int R>
__device__ __forceinline__ void ltwmul_w(double2 w1, double2* v) {
  if constexpr (R > 1) {
#ifdef EXPD_LINE_TWSEQ
    double2 cur = w1;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      v[r] = cmul(v[r], cur);
      if (r + 1 < R) cur = cmul(cur, w1);
    }
#else
    double2 t[R];
    t[1] = w1;
#pragma unroll
    for (int r = 2; r < R; ++r) t[r] = (r % 2 == 0) ? cmul(t[r / 2], t[r / 2]) : cmul(t[r - 1], t[1]);
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], t[r]);
#endif
  }
}
template <int R>
__device__ __forceinline__ void ltwmul(const double2* __restrict__ tw, int b, double2* v) {
  if constexpr (R > 1) ltwmul_w<R>(__ldg(tw + b), v);
}

// Per-thread table values of one item, loaded before the item's data lands (their L1 / L2
// latency then hides behind the TMA wait): sin(pi i/M) of the stage-0 positions and the
// base twiddles of the thread's middle-stage job and last-stage partner jobs (valid when
// each thread owns exactly one such job, the configurations used here).
template <int M, int G>
struct LPre {
  double sj, cj;       // sin / cos (pi j / M) of this thread's stage-0 job j (kept for the kernel)
  double2 tmid, ta, tb;  // base twiddles (re-loaded per item: held, they cost spills)
  int pj;  // this thread's partner job of the last stage (see partner_job)
};

// cos (2 pi e / 32) (exact decimal expansions to 20 digits)
__host__ __device__ constexpr double cos32(int e) {
  constexpr double c[9] = {1.0,
                           0.98078528040323044913,
                           0.92387953251128675613,
                           0.83146961230254523708,
                           0.70710678118654752440,
                           0.55557023301960222474,
                           0.38268343236508977173,
                           0.19509032201612826785,
                           0.0};
  e &= 31;
  return e <= 8 ? c[e] : (e <= 16 ? -c[16 - e] : (e <= 24 ? -c[e - 16] : c[32 - e]));
}
__host__ __device__ constexpr double sin32(int e) { return cos32(8 - e); }

// The per-thread constants of the line transform, computed ONCE per kernel (they depend only
// on the thread): the stage-0 angle pi j / M (the pre-processing weights sin(pi i / M), i = j +
// T r, follow by the addition theorem with the compile-time angles pi r / R0 -- no per-item
// table loads through the LSU, which is the line kernels' bottleneck) and the base twiddles
// of the middle stage and of the last stage's partner jobs.
template <int M, int G>
__device__ __forceinline__ LPre<M, G> line_pre(const LineArgs& a, int my_pj) {
  const int j = threadIdx.x / G;
  LPre<M, G> pre;
  pre.pj = my_pj;
  pre.sj = __ldg(a.sinp + j);
  pre.cj = __ldg(a.sinp + M / 2 - j);  // cos(pi j / M) = sin(pi (M/2 - j) / M), j <= M / 2
  return pre;
}
template <int M, int G>
__device__ __forceinline__ void line_pre_tw(LPre<M, G>& pre, const double2* __restrict__ tw) {
  using D = LGeo<M, G, 1>;
  constexpr int R0 = D::R0, NSL = D::NSL;
  const int j = threadIdx.x / G;
  constexpr int NS1 = R0, TWS1 = M / (NS1 * D::RM1);
  pre.tmid = __ldg(tw + (j % NS1) * TWS1);
  const int pj = pre.pj / G;  // the partner job's frequency set (G = 1: the table entry)
  pre.ta = __ldg(tw + (pj < NSL / 2 ? pj : 0));
  pre.tb = __ldg(tw + (pj == 0 ? NSL / 2 : (pj < NSL / 2 ? NSL - pj : 0)));
}

// a_i = c (sin(pi i/M) + 1/2) for i = j + T r: sin(pi j/M + pi r/R0) by the addition theorem
template <int R0, int r>
__device__ __forceinline__ double pre_a(double sj, double cj, double c) {
  constexpr int e = 16 * r / R0;  // pi r / R0 = 2 pi e / 32
  const double s = fma(sj, cos32(e), cj * sin32(e));
  return fma(c, s, 0.5 * c);
}

// Lane -> partner job of the last FFT stage.  With one pair job per thread (G = 1, NSL / 2 =
// T) any bijection works; the tables (tools/partner_lanes.py) group the jobs so that each
// 8-lane phase of the partner reads and unpack writes hits distinct bank groups (the
// identity walks the mirrored frequencies downwards and straddles a padding slot in half
// of the phases).  Other configurations: the identity.
#include "partner_lanes.inc"
template <int M, int G>
__device__ __forceinline__ int partner_job(int tid) {
  using D = LGeo<M, G, 1>;
  if constexpr (G == 1 && D::NSL / 2 == D::THREADS && (M == 512 || M == 1024 || M == 2048)) {
    if constexpr (M == 512) return __ldg(kPartnerJob512 + tid);
    else if constexpr (M == 1024) return __ldg(kPartnerJob1024 + tid);
    else return __ldg(kPartnerJob2048 + tid);
  }
  return tid;
}

// position p of line pair g in the padded work layout [SW][G]
template <int M, int G>
__device__ __forceinline__ double2& lat(double2* buf, int p, int g) {
  EXPD_CHECK(p >= 0 && p < M && g >= 0 && g < G, "line: padded position");
  return buf[lswz<LGeo<M, G, 1>::PADP>(p) * G + g];
}

// Middle Stockham stage (radix R, NS) of the G line pairs: reads in, writes buf (in place when
// they are the same buffer).
template <int M, int G, int R, int NS, class W>
__device__ __forceinline__ void lmid(double2* in, double2* buf, const double2* __restrict__ tw, double2 tpre,
                                     W& war) {
  using D = LGeo<M, G, 1>;
  constexpr int JOBS = G * (M / R);
  constexpr int JT = (JOBS + D::THREADS - 1) / D::THREADS;
  constexpr int TWS = M / (NS * R);
  double2 v[JT][R];
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * D::THREADS;
    if (JOBS % D::THREADS == 0 || J < JOBS) {
      const int g = J % G, jm = J / G;
#pragma unroll
      for (int r = 0; r < R; ++r) v[jt][r] = lat<M, G>(in, jm + r * (M / R), g);
    }
  }
  war.arrive(0);
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * D::THREADS;
    if (JOBS % D::THREADS == 0 || J < JOBS) {
      const int k = (J / G) % NS;
      if (JT == 1) ltwmul_w<R>(tpre, v[jt]);
      else ltwmul<R>(tw, k * TWS, v[jt]);
      DFT<R, -1>::run(v[jt]);
    }
  }
  war.wait(0);  // WAR: every warp's reads of buf are done before the writes
#pragma unroll
  for (int jt = 0; jt < JT; ++jt) {
    const int J = threadIdx.x + jt * D::THREADS;
    if (JOBS % D::THREADS == 0 || J < JOBS) {
      const int g = J % G, jm = J / G, k = jm % NS, base = (jm / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) lat<M, G>(buf, base + r * NS, g) = v[jt][r];
    }
  }
  __syncthreads();
}

// DST core of G line pairs: thread (g, j) holds the stage-0 inputs y_i (i = j + T r) of
// line pair g in v; leaves F (already scaled: V x) at natural positions [2jL, 2jL + 2L) in out
// (F_m sits at position m-1; position M-1 is the spectral pad and returns 0).  Starts with
// a barrier (buf may still be read by the caller's stage-0 loads).
// Buffers: X takes the stage-0 results (read by the middle stage), Y the middle stage's (read
// by the last stage), Z the unpacked arrays (read by the prefix scan); one buffer for all three
// with the WarSync / WarMbar policies, X = Z != Y with WarNone (k_line_pp).
template <int M, int G, class W>
__device__ __forceinline__ void lcore(double2 (&v)[LGeo<M, G, 1>::R0], double2* X, double2* Y, double2* Z,
                                      double2* wt, const double2* __restrict__ tw,
                                      double2 (&out)[2 * LGeo<M, G, 1>::L], const LPre<M, G>& pre, W& war,
                                      bool defer = false, double2* offw = nullptr) {
  using D = LGeo<M, G, 1>;
  constexpr int R0 = D::R0, RL = D::RL, NSL = D::NSL, T = D::T, L = D::L, PADP = D::PADP;
  const int g = threadIdx.x % G, j = threadIdx.x / G;
  war.arrive(1);  // this warp's stage-0 reads (the caller's) are done
  DFT<R0, -1>::run(v);
  war.wait(1);  // WAR: every warp's stage-0 reads are done before the writes
  {
    double2* o0 = X + lswz<PADP>(j * R0) * G + g;  // R0 = PADP consecutive positions: linear
#pragma unroll
    for (int r = 0; r < R0; ++r) o0[r * G] = v[r];
  }
  __syncthreads();
  lmid<M, G, D::RM1, R0>(X, Y, tw, pre.tmid, war);
  // last stage on Hermitian partner jobs (ja, jb): frequency sets k = ja + NSL r and
  // jb + NSL r pair up as k <-> M - k; then the unpack into e_k (position 2k-1), w_k (2k)
  constexpr int PJOBS = G * (NSL / 2);
  constexpr int PJT = (PJOBS + D::THREADS - 1) / D::THREADS;
  double2 va[PJT][RL], vb[PJT][RL];
#pragma unroll
  for (int pt = 0; pt < PJT; ++pt) {
    const int PJ = PJT == 1 ? pre.pj : threadIdx.x + pt * D::THREADS;
    if (PJOBS % D::THREADS == 0 || PJ < PJOBS) {
      const int gg = PJ % G, pj = PJ / G;
      const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
#pragma unroll
      for (int r = 0; r < RL; ++r) {
        va[pt][r] = lat<M, G>(Y, ja + r * NSL, gg);
        vb[pt][r] = lat<M, G>(Y, jb + r * NSL, gg);
      }
    }
  }
  war.arrive(2);
#pragma unroll
  for (int pt = 0; pt < PJT; ++pt) {
    const int PJ = PJT == 1 ? pre.pj : threadIdx.x + pt * D::THREADS;
    if (PJOBS % D::THREADS == 0 || PJ < PJOBS) {
      const int pj = PJ / G;
      const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
      if (PJT == 1) {
        ltwmul_w<RL>(pre.ta, va[pt]);
        ltwmul_w<RL>(pre.tb, vb[pt]);
      } else {
        ltwmul<RL>(tw, ja, va[pt]);
        ltwmul<RL>(tw, jb, vb[pt]);
      }
      DFT<RL, -1>::run(va[pt]);
      DFT<RL, -1>::run(vb[pt]);
    }
  }
  war.wait(2);  // WAR: every warp's partner reads are done before the unpack writes
  // unpack into two arrays W[k] = w_k (k = 0..M/2-1) and E[k] = e_k (k = 1..M/2), each
  // padded with one slot per L entries: consecutive threads write consecutive k and the
  // prefix below reads L consecutive entries per thread, both without bank conflicts
  double2* Wb = Z;
  double2* Eb = Z + D::WS * G;
#pragma unroll
  for (int pt = 0; pt < PJT; ++pt) {
    const int PJ = PJT == 1 ? pre.pj : threadIdx.x + pt * D::THREADS;
    if (PJOBS % D::THREADS == 0 || PJ < PJOBS) {
      const int gg = PJ % G, pj = PJ / G;
      const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
#pragma unroll
      for (int r = 0; r < RL / 2; ++r) {
        double2 e, w;
        const int ka = ja + NSL * r;
        lunpack(va[pt][r], pj == 0 ? va[pt][(RL - r) % RL] : vb[pt][RL - 1 - r], ka == 0, e, w);
        EXPD_CHECK(lswz<L>(ka) < D::WS && lswz<L>(jb + NSL * r) < D::WS, "line: unpack index");
        if (ka >= 1) Eb[lswz<L>(ka) * G + gg] = e;
        Wb[lswz<L>(ka) * G + gg] = w;
        const int kb = jb + NSL * r;
        lunpack(vb[pt][r], pj == 0 ? vb[pt][RL - 1 - r] : va[pt][RL - 1 - r], false, e, w);
        Eb[lswz<L>(kb) * G + gg] = e;
        Wb[lswz<L>(kb) * G + gg] = w;
      }
    }
  }
  __syncthreads();
  // prefix sum: thread (g, j) owns k in [jL, jL + L) -> positions [2jL, 2jL + 2L):
  // out[2l] = F_{2k+1} = sum_{k' <= k} w_k', out[2l+1] = F_{2k+2} = e_{k+1}
  double2 tot = make_double2(0.0, 0.0);
  {
    const double2* Pw = Wb + (j * (L + 1)) * G + g;  // W[jL .. jL + L): contiguous
    const double2* Pe = Eb + (j * (L + 1)) * G + g;  // E[jL + 1 .. jL + L]: skips the pad slot
#pragma unroll
    for (int l = 0; l < L; ++l) {
      tot = cadd(tot, Pw[l * G]);
      out[2 * l] = tot;
      const int el = l + 1 < L ? l + 1 : L + 1;
      out[2 * l + 1] = (j == T - 1 && l == L - 1) ? make_double2(0.0, 0.0) : Pe[el * G];
    }
  }
  double2 inc = tot;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < D::JW && d < T; d <<= 1) {
    double ox = __shfl_up_sync(0xffffffffu, inc.x, d * G);
    double oy = __shfl_up_sync(0xffffffffu, inc.y, d * G);
    if (lane >= d * G) inc = cadd(inc, make_double2(ox, oy));
  }
  double2 off = csub(inc, tot);
  if constexpr (D::NWB > 1) {
    const int jw = j / D::JW;
    if (j % D::JW == D::JW - 1) wt[jw * G + g] = inc;
    if (defer) {  // the caller adds the earlier warps' totals after its next barrier (line_offw)
      *offw = off;
      return;
    }
    __syncthreads();
    for (int b = 0; b < jw; ++b) off = cadd(off, wt[b * G + g]);
  }
#pragma unroll
  for (int l = 0; l < L; ++l) out[2 * l] = cadd(out[2 * l], off);
}

// The deferred end of lcore's prefix (defer = true): after a barrier that follows the wt
// writes, the same additions in the same order (bitwise equal to the immediate form).
template <int M, int G>
__device__ __forceinline__ void line_offw(const double2* wt, double2 off, double2 (&out)[2 * LGeo<M, G, 1>::L]) {
  using D = LGeo<M, G, 1>;
  const int g = threadIdx.x % G, j = threadIdx.x / G, jw = j / D::JW;
  for (int b = 0; b < jw; ++b) off = cadd(off, wt[b * G + g]);
#pragma unroll
  for (int l = 0; l < D::L; ++l) out[2 * l] = cadd(out[2 * l], off);
}

// ---------------------------------------------------------------------------------------
// the persistent line kernel
// ---------------------------------------------------------------------------------------
template <int AX, int G>
__device__ __forceinline__ void line_coords(const LineArgs& a, long item, int& c0, int& c1, int& c2, int& c3,
                                            int smod = 0) {
  // 32-bit unsigned arithmetic (item counts stay far below 2^32): a 64-bit division is a
  // long software sequence on the issuing thread's critical path to the TMA
  EXPD_CHECK(item >= 0 && item < a.nitems, "line: item index");
  const unsigned it = (unsigned)item, ps = (unsigned)a.per_slice;
  const unsigned s = it / ps;
  const int w = (int)(it - s * ps);
  if constexpr (AX == AX_ROW) {
    c0 = 0; c1 = 0; c2 = 2 * w; c3 = (int)s;  // rows 2w, 2w+1 of slice s
  } else {
    const int o = (int)((unsigned)w / (unsigned)a.inner), cg = w - o * a.inner;
    c0 = 2 * G * cg;
    if constexpr (AX == AX_COL_Y) { c1 = 0; c2 = o; }
    else { c1 = o; c2 = 0; }
    c3 = (int)s;
  }
  if (smod) c3 %= smod;  // a ring of smod slices (the persistent stage 3's intermediate)
}

template <int M, int AX, int G>
__device__ __forceinline__ void line_issue_load(const CUtensorMap* map, const LineArgs& a, long item, char* buf,
                                                uint64_t* bar, int smod = 0) {
  int c0, c1, c2, c3;
  line_coords<AX, G>(a, item, c0, c1, c2, c3, smod);
  mbar_arrive_expect_tx(bar, (uint32_t)(G * M * 16));
  if constexpr (AX == AX_ROW) {
    if (a.peer_in) {  // each row from the rank that owns its x-line (PeerMaps); a row past the
      // slice (odd row count) reads out of the last rank's box: zero-filled, bytes counted
      const PeerMaps* pm = a.peer_in;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = c2 + h;
        int q = 0;
        while (q + 1 < pm->nranks && row >= pm->unit_off[q + 1]) ++q;
        tma_load_4d(buf + h * M * 8, &pm->m[q], bar, 0, 0, row - pm->unit_off[q], a.peer_in_slot0 + c3);
      }
    } else {
      tma_load_4d(buf, map, bar, 0, 0, c2, c3);
      tma_load_4d(buf + M * 8, map, bar, 0, 0, c2 + 1, c3);
    }
  } else {
    // linear raw layout [row][G]: grid row p of pair g at double2 p*G + g (boxes of CBR rows)
#pragma unroll
    for (int b = 0; b < M / CBR; ++b) {
      char* dst = buf + (size_t)b * CBR * 16 * G;
      if constexpr (AX == AX_COL_Y) tma_load_4d(dst, map, bar, c0, b * CBR, c2, c3);
      else tma_load_4d(dst, map, bar, c0, c1, b * CBR, c3);
    }
  }
}

template <int M, int AX, int G, bool TS = false>
__device__ __forceinline__ void line_issue_store(const CUtensorMap* map, const LineArgs& a, long item,
                                                 const char* buf, int smod = 0) {
  int c0, c1, c2, c3;
  line_coords<AX, G>(a, item, c0, c1, c2, c3, smod);
  if constexpr (AX != AX_ROW && TS) {
    // ONE box of the transposed view (col_ts_map): rows 0 .. M - 2L - 1 of the G pairs
    if constexpr (AX == AX_COL_Y) tma_store_5d(map, buf, c0, 0, 0, c2, c3);
    else tma_store_5d(map, buf, c0, c1, 0, 0, c3);
  } else if constexpr (AX == AX_ROW) {
    if (a.peer) {  // each row to the rank that owns its x-line (PeerMaps)
      const PeerMaps* pm = a.peer;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = c2 + h;
        if (row >= a.rows) break;
        int q = 0;
        while (q + 1 < pm->nranks && row >= pm->unit_off[q + 1]) ++q;
        EXPD_CHECK(row - pm->unit_off[q] < pm->units[q], "line: peer row");
        tma_store_4d(&pm->m[q], buf + h * M * 8, 0, 0, row - pm->unit_off[q], a.peer_slot0 + c3);
      }
    } else {
      tma_store_4d(map, buf, 0, 0, c2, c3);
      if (c2 + 1 < a.rows) tma_store_4d(map, buf + M * 8, 0, 0, c2 + 1, c3);
    }
  } else {
#pragma unroll
    for (int b = 0; b < M / CBR; ++b) {
      const char* src = buf + (size_t)b * CBR * 16 * G;
      if constexpr (AX == AX_COL_Y) tma_store_4d(map, src, c0, b * CBR, c2, c3);
      else tma_store_4d(map, src, c0, c1, b * CBR, c3);
    }
  }
  bulk_commit();
}

// The transform of one item (G line pairs) whose input the TMA is bringing into cb (arrival
// on bar, phase parity): table values, the wait, [V] or [V, N, V], and the result written in
// the layout the item's TMA store reads.  Every thread of the CTA calls it.
// PP (ping-pong, k_line_pp): the result goes to a second buffer cbo and the transform's stages
// alternate between the two (lcore's X = Z = cbo, Y = cb), so no stage writes a buffer that
// another warp may still be reading: the write-after-read barriers disappear (WarNone).
// Otherwise cbo == cb and the policy W places them.
template <int M, int AX, bool NL, int G, class W, bool PP = false, bool TS = false, bool HY = false>
__device__ __forceinline__ void line_item(char* cb, char* cbo, double2* wt, const LineArgs& a,
                                          const LPre<M, G>& pre0, uint64_t* bar, uint32_t parity, W& war,
                                          long item = 0, char* coth = nullptr, const CUtensorMap* in_map = nullptr,
                                          uint64_t* bar_oth = nullptr, long next = -1) {
  using D = LGeo<M, G, 1>;
  constexpr int R0 = D::R0, T = D::T, L = D::L, PADP = D::PADP;
  const int tid = threadIdx.x;
  const int g = tid % G, j = tid / G;
  double2* buf = reinterpret_cast<double2*>(cb);
  double2* bufo = reinterpret_cast<double2*>(cbo);
    // the twiddle table is re-read every item: an opaque copy of the pointer keeps the
    // compiler from hoisting loop-invariant twiddles into registers for the whole loop
    const double2* tw = a.tw;
    asm volatile("" : "+l"(tw));
    LPre<M, G> pre = pre0;
    line_pre_tw<M, G>(pre, tw);
    mbar_wait(bar, parity);

    double2 out[2 * L];
    // NL: two passes [V, N, V] through ONE copy of the transform code (the trip count is
    // opaque to the compiler, which would otherwise unroll it into ~8000 instructions and
    // thrash the instruction cache)
    int npass = NL ? 2 : 1;
    asm volatile("" : "+r"(npass));
    // HY (hybrid buffer schedule, EXPD_LINE_HY): the middle stage writes the OTHER buffer (free:
    // the previous item's store has read it; the next item's load goes there only after this
    // item's last unpack), so its write-after-read barrier and the unpack's go; in the fused
    // pass the N step writes the other buffer too (no barrier before it) and pass 1 reads it,
    // which makes every barrier of pass 1's transform a read-after-write one
    double2* oth = reinterpret_cast<double2*>(coth);
    double2 offw = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int pass = 0; pass < npass; ++pass) {
      double2* src = (HY && pass) ? oth : buf;  // stage-0 input of this pass
      double2 v[R0];
      // opaque copies: the weights are recomputed in each pass instead of being hoisted out of
      // the pass loop (16 live doubles)
      double sj = pre.sj, cj = pre.cj;
      asm volatile("" : "+d"(sj), "+d"(cj));
      sfor<R0>([&](auto rr) {
        constexpr int r = decltype(rr)::value;
        const int i = j + T * r;
        const double av = pre_a<R0, r>(sj, cj, a.c);
        if (i == 0) {
          v[r] = make_double2(0.0, 0.0);
        } else if (AX == AX_ROW) {
          // the input rows land UNswizzled (linear): a half-warp's 16 reads of x_i at i - 1
          // and of the mirror at M - i - 1 each cover 16 consecutive doubles, i.e. 32
          // distinct banks (the 128-byte swizzle splits the i - 1 run over two lines)
          const uint32_t o1 = (uint32_t)(i - 1) * 8u, o2 = (uint32_t)(M - i - 1) * 8u;
          EXPD_CHECK(o1 < M * 8u && o2 < M * 8u, "line: row stage-0 read");
          const double2 z = make_double2(*reinterpret_cast<const double*>(cb + o1),
                                         *reinterpret_cast<const double*>(cb + M * 8 + o1));
          const double2 zm = make_double2(*reinterpret_cast<const double*>(cb + o2),
                                          *reinterpret_cast<const double*>(cb + M * 8 + o2));
          v[r] = lpre(z, zm, av, a.c);
        } else {
          // pass 0: raw [row][G] linear; pass 1: the padded layout written by the N step
          const int p1 = i - 1, p2 = M - i - 1;
          const int q1 = pass ? lswz<PADP>(p1) : p1, q2 = pass ? lswz<PADP>(p2) : p2;
          EXPD_CHECK(q1 >= 0 && q2 >= 0 && q1 < D::SWB && q2 < D::SWB, "line: column stage-0 read");
          v[r] = lpre(src[q1 * G + g], src[q2 * G + g], av, a.c);
        }
      });
      // the last pass defers the prefix's cross-warp barrier to the one before the result's
      // writes (the wt totals are read after it; EXPD_LINE_DEFER=0 at build time disables)
      const bool defer = EXPD_LINE_DEFER && !PP && D::NWB > 1 && pass + 1 == npass;
      if constexpr (HY) {
        // X = buf (in place over pass 0's input: its stage-0 reads are ordered by point 1; pass
        // 1's input is in oth), Y = oth, Z = buf
        WarMask wm{pass ? 0u : 2u};
        lcore<M, G>(v, buf, oth, buf, wt, tw, out, pre, wm, defer, &offw);
      } else {
        lcore<M, G>(v, PP ? bufo : buf, buf, PP ? bufo : buf, wt, tw, out, pre, war, defer, &offw);
      }
      if (NL && pass + 1 < npass) {
        if (!PP && !HY) __syncthreads();  // everyone has read (e, w) of pass 0
        double2* nb = HY ? oth : buf;
#pragma unroll
        for (int q = 0; q < 2 * L; ++q)
          lat<M, G>(nb, 2 * j * L + q, g) =
              make_double2(poly_eval(a.poly, out[q].x), poly_eval(a.poly, out[q].y));
        __syncthreads();
      }
    }
    if constexpr (HY) {
      // every thread has passed the last unpack barrier: nobody reads oth again -> prefetch
      if (threadIdx.x == 0 && next >= 0 && next < a.nitems) line_issue_load<M, AX, G>(in_map, a, next, coth, bar_oth);
    }
    // (e, w) reads done before the result overwrites their buffer (PP: only the row result
    // goes to it, and the prefix's cross-warp barrier already ordered them unless NWB == 1)
    if (!PP || TS || (AX == AX_ROW && D::NWB == 1)) __syncthreads();
    if (EXPD_LINE_DEFER && !PP && D::NWB > 1) line_offw<M, G>(wt, offw, out);
    if constexpr (AX != AX_ROW && TS) {
      // transposed store (TS): position p = 2L a + q of pair g goes to slot (q (T-1) + a) G + g,
      // the smem layout of the transposed TMA view (col_ts_map, box a < T-1): in each write
      // instruction consecutive threads hit consecutive 16-byte slots (conflict free), and the
      // result needs no compaction pass.  The last thread's rows M-2L .. M-2 (M-1 is the
      // spectral pad) lie outside that box: it stores them to global memory itself.
      if (j < T - 1) {
        double2* o = bufo + j * G + g;
#pragma unroll
        for (int q = 0; q < 2 * L; ++q) o[q * (T - 1) * G] = out[q];
      } else {
        int c0, c1, c2, c3;
        line_coords<AX, G>(a, item, c0, c1, c2, c3);
        const long npad = (long)a.rows * M;
        double* gp = a.outp + (long)c3 * npad + c0 + 2 * g;
#pragma unroll
        for (int q = 0; q < 2 * L - 1; ++q) {
          const int p = 2 * j * L + q;
          const long row = AX == AX_COL_Y ? (long)c2 * (M - 1) + p : (long)p * (M - 1) + c1;
          EXPD_CHECK(row * M + c0 + 2 * g + 1 < npad, "line: TS tail row");
          *reinterpret_cast<double2*>(gp + row * M) = out[q];
        }
      }
    } else if constexpr (AX == AX_ROW) {
      // rows a / b in the 128B-swizzled box layout: positions [2jL, 2jL+2L) as 16-byte pairs
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const int x = 2 * j * L + 2 * l;
        const uint32_t off = row_sw(x);
        EXPD_CHECK(off + 16u <= M * 8u, "line: row result slot");
        *reinterpret_cast<double2*>(cbo + off) = make_double2(out[2 * l].x, out[2 * l + 1].x);
        *reinterpret_cast<double2*>(cbo + M * 8 + off) = make_double2(out[2 * l].y, out[2 * l + 1].y);
      }
    } else {
      // chunk -> padded layout (conflict free), then compact in place to the linear [row][G]
      // layout the TMA store reads; thread (g, j) moves positions j + T r of pair g
#pragma unroll
      for (int q = 0; q < 2 * L; ++q) lat<M, G>(buf, 2 * j * L + q, g) = out[q];
      __syncthreads();
      double2 c[R0];
#pragma unroll
      for (int r = 0; r < R0; ++r) c[r] = lat<M, G>(buf, j + T * r, g);
      if (!PP) __syncthreads();
#pragma unroll
      for (int r = 0; r < R0; ++r) bufo[(j + T * r) * G + g] = c[r];
    }
}

// G line pairs per item, NBUF shared-memory buffers (2: the next item's TMA load overlaps
// this item's transform; 1: overlap comes from the other CTAs on the SM).
// PP: two buffers whose roles alternate per item (input of item i = output of item i - 1);
// the next item's load is issued once the store has read the output buffer (no prefetch
// during the transform -- the other CTAs of the SM cover the wait), and the transform runs
// without write-after-read barriers (line_item PP).
template <int M, int AX, bool NL, int G, int NBUF, bool PP = false, bool TS = false, bool HY = false>
__global__ void __launch_bounds__(LGeo<M, G, NBUF>::THREADS, LGeo<M, G, NBUF>::MINB)
    k_line(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
           const __grid_constant__ LineArgs a) {
  using D = LGeo<M, G, NBUF>;
  static_assert(AX != AX_ROW || G == 1, "row items are one row pair");
  static_assert(!PP || NBUF == 2, "ping-pong needs two buffers");
  static_assert(!HY || (NBUF == 2 && !PP), "the hybrid schedule needs two buffers");
  constexpr int R0 = D::R0, T = D::T, L = D::L, PADP = D::PADP;
  if (a.skip && *a.skip) return;  // stage 3 of a sweep whose result is known (line_skip_scope)
  extern __shared__ unsigned char lsm_raw[];
  // 1 KB-aligned base as an offset from the __shared__ array (pointer arithmetic on the
  // array keeps the shared address space: LDS/STS, not generic LD/ST)
  char* base = reinterpret_cast<char*>(lsm_raw + ((1024u - (smem_u32(lsm_raw) & 1023u)) & 1023u));
  double2* wt = reinterpret_cast<double2*>(base + NBUF * D::BUFB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wt + D::NWB * G);
  const int tid = threadIdx.x;
  __builtin_assume(tid < D::THREADS);
  const int g = tid % G, j = tid / G;
  const int my_pj = partner_job<M, G>(tid);
  const LPre<M, G> pre = line_pre<M, G>(a, my_pj);

  if (tid == 0) {
    prefetch_tmap(&in_map);
    prefetch_tmap(&out_map);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    if (EXPD_WAR_MODE)
      for (int k = 0; k < kWarPoints; ++k) mbar_init(&bar[2 + k], D::THREADS / 32);
    mbar_fence_init();
  }
  __syncthreads();
#if EXPD_WAR_MODE
  using WarP = WarMbar;
#else
  using WarP = WarSync;
#endif
  using WarT = std::conditional_t<PP, WarNone, WarP>;
  WarT war{};
  if constexpr (std::is_same_v<WarT, WarMbar>) war = WarMbar{bar + 2, 0u};
  long item = blockIdx.x;
  if (tid == 0 && item < a.nitems) line_issue_load<M, AX, G>(&in_map, a, item, base, &bar[0]);

  for (int it = 0; item < a.nitems; ++it, item += gridDim.x) {
    const int cur = NBUF == 2 ? (it & 1) : 0;
    char* cb = base + cur * D::BUFB;
    char* cbo = PP ? base + (cur ^ 1) * D::BUFB : cb;
    double2* buf = reinterpret_cast<double2*>(cb);
    const long next = item + gridDim.x;
    if (!PP && NBUF == 2 && tid == 0 && (HY || next < a.nitems)) {
      bulk_wait_read0();  // the previous item's stores have left the other buffer
      if (!HY) line_issue_load<M, AX, G>(&in_map, a, next, base + (cur ^ 1) * D::BUFB, &bar[cur ^ 1]);
    }
    line_item<M, AX, NL, G, WarT, PP, TS, HY>(cb, cbo, wt, a, pre, &bar[cur],
                                              (uint32_t)((NBUF == 2 ? (it >> 1) : it) & 1), war, item,
                                              base + (cur ^ 1) * D::BUFB, &in_map, &bar[cur ^ 1], next);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      line_issue_store<M, AX, G, TS>(&out_map, a, item, cbo);
      if (PP && next < a.nitems) {
        bulk_wait_read0();  // the store has read the output buffer: it is the next input
        line_issue_load<M, AX, G>(&in_map, a, next, cbo, &bar[cur ^ 1]);
      }
      if (NBUF == 1 && next < a.nitems) {
        bulk_wait_read0();  // the store has read the buffer: refill it
        line_issue_load<M, AX, G>(&in_map, a, next, base, &bar[0]);
      }
    }
  }
  if (tid == 0) {
    bulk_wait0();
    if (a.peer) __threadfence_system();  // the peer stores are complete before the kernel ends
  }
}

// ---------------------------------------------------------------------------------------
// Persistent stage 3 (2-D; SURVEY §7 "Hard parts"): ONE launch carries
// every slice through x-IDST -> fused y [V, N(u), V] -> x-DST with no kernel boundary.  The
// CTAs take one of three roles by (blockIdx mod #SMs) -- the three CTAs of an SM share a role,
// so an SM runs one code path -- and each role takes its items in slice order from its own
// ticket counter.  Dependencies are per slice and counted in global memory: y(s) waits until
// all x-IDST(s) items are stored, x-DST(s) until all y(s) items are, and x-IDST(s) until
// ring slot s mod K of the intermediate is free (x-DST(s - K) stored).  The intermediate is
// a ring of K slices (K x 33.5 MB at c5) that stays in the 126 MB L2, so HBM sees U-hat read
// once and N-hat written once (16 B per dof) instead of three round trips per slice, and the
// per-chunk launch tails disappear.  Progress: the pending item of the smallest slice always
// has its dependencies met (every earlier item of the producer role has been taken by a
// resident CTA, which finishes it without waiting), so the spin waits cannot deadlock for
// K >= 2; a CTA that must wait first completes and signals its own pending store.
// ---------------------------------------------------------------------------------------
constexpr int kS3MaxSlices = 272;
struct S3Ctl {
  unsigned int ticket[4];
  unsigned int done[3][kS3MaxSlices];
};
struct S3Args {
  LineArgs row, col;  // item geometry of the x passes / the fused y pass (tables, poly shared)
  S3Ctl* ctl;
  int nslices, K, sms, split0, split1;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait1() { asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); }

// sh: shared scratch of the issuing thread's state (keeps it out of the transform's registers):
// sh[0], sh[1] next items (double-buffered broadcast), sh[2] current item, sh[3] pending
// (stored, not yet signalled) item, sh[4] "current item's load issued", sh[5] "next issued"
template <int M, int AX, bool NL>
__device__ __forceinline__ void s3_role(const CUtensorMap* in_map, const CUtensorMap* out_map, const LineArgs& a,
                                     const S3Args& s3, int pass, char* base, double2* wt, uint64_t* bar,
                                     volatile long* sh, int my_pj) {
  using D = LGeo<M, 1, 2>;
  const int tid = threadIdx.x;
  WarSync war;  // (the persistent kernel's shared memory carries no WAR mbarriers)
  S3Ctl* ctl = s3.ctl;
  const unsigned per = (unsigned)a.per_slice;
  const unsigned total = per * (unsigned)s3.nslices;
  const int K = s3.K;
  const int smod_in = pass == 0 ? 0 : K, smod_out = pass == 2 ? 0 : K;
  const LPre<M, 1> pre = line_pre<M, 1>(a, my_pj);
  auto grab = [&]() -> long {
    const unsigned t = atomicAdd(&ctl->ticket[pass], 1u);
    return t < total ? (long)t : -1;
  };
  auto ready = [&](long item) -> bool {
    const int s = (int)((unsigned)item / per);
    if (pass == 0) return s < K || ld_acquire_u32(&ctl->done[2][s - K]) == per;
    return ld_acquire_u32(&ctl->done[pass - 1][s]) == per;
  };
  auto signal = [&](long item) {
    fence_proxy_async_global();
    __threadfence();
    atomicAdd(&ctl->done[pass][(unsigned)item / per], 1u);
  };
  if (tid == 0) {
    const long item = grab();
    sh[4] = 0;
    if (item >= 0 && ready(item)) {
      fence_proxy_async_global();
      line_issue_load<M, AX, 1>(in_map, a, item, base, &bar[0], smod_in);
      sh[4] = 1;
    }
    sh[2] = item;
    sh[3] = -1;
  }
  __syncthreads();
  for (int it = 0; sh[2] >= 0; ++it) {
    const int cur = it & 1;
    char* cb = base + cur * D::BUFB;
    if (tid == 0) {
      const long item = sh[2];
      if (!sh[4]) {  // deferred: complete and signal our own pending store, then wait
        if (sh[3] >= 0) {
          bulk_wait0();
          signal(sh[3]);
          sh[3] = -1;
        }
        const uint64_t t0 = global_ns();  // bounded: a dependency that never completes traps
        while (!ready(item)) {
          __nanosleep(128);
          if (global_ns() - t0 > 4000000000ull) {
            printf("expd: stage-3 dependency wait timed out (pass %d item %ld)\n", pass, item);
            __trap();
          }
        }
        fence_proxy_async_global();
        line_issue_load<M, AX, 1>(in_map, a, item, cb, &bar[cur], smod_in);
      }
      const long nxt = grab();
      bulk_wait_read0();  // the previous item's store has left the other buffer
      sh[5] = 0;
      if (nxt >= 0 && ready(nxt)) {
        fence_proxy_async_global();
        line_issue_load<M, AX, 1>(in_map, a, nxt, base + (cur ^ 1) * D::BUFB, &bar[cur ^ 1], smod_in);
        sh[5] = 1;
      }
      sh[it & 1] = nxt;
    }
    line_item<M, AX, NL, 1>(cb, cb, wt, a, pre, &bar[cur], (uint32_t)((it >> 1) & 1), war);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const long item = sh[2];
      line_issue_store<M, AX, 1>(out_map, a, item, cb, smod_out);
      if (sh[3] >= 0) {
        bulk_wait1();  // the previous item's store is complete
        signal(sh[3]);
      }
      sh[3] = item;
      sh[4] = sh[5];
      sh[2] = sh[it & 1];
    }
    __syncthreads();  // sh[2] (the next item) is visible
  }
  if (tid == 0) {
    bulk_wait0();
    if (sh[3] >= 0) signal(sh[3]);
  }
}

template <int M>
__global__ void __launch_bounds__(LGeo<M, 1, 2>::THREADS, LGeo<M, 1, 2>::MINB)
    k_stage3p(const __grid_constant__ CUtensorMap m_u, const __grid_constant__ CUtensorMap m_trow_out,
              const __grid_constant__ CUtensorMap m_tcol, const __grid_constant__ CUtensorMap m_trow_in,
              const __grid_constant__ CUtensorMap m_n, const __grid_constant__ S3Args s3) {
  using D = LGeo<M, 1, 2>;
  extern __shared__ unsigned char s3sm_raw[];
  char* base = reinterpret_cast<char*>(s3sm_raw + ((1024u - (smem_u32(s3sm_raw) & 1023u)) & 1023u));
  double2* wt = reinterpret_cast<double2*>(base + 2 * D::BUFB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wt + D::NWB);
  __shared__ long sh[6];
  const int tid = threadIdx.x;
  const int my_pj = partner_job<M, 1>(tid);
  const int b = (int)(blockIdx.x % (unsigned)s3.sms);
  const int role = b < s3.split0 ? 0 : (b < s3.split0 + s3.split1 ? 1 : 2);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (role == 0) {
    if (tid == 0) {
      prefetch_tmap(&m_u);
      prefetch_tmap(&m_trow_out);
    }
    s3_role<M, AX_ROW, false>(&m_u, &m_trow_out, s3.row, s3, 0, base, wt, bar, sh, my_pj);
  } else if (role == 1) {
    if (tid == 0) prefetch_tmap(&m_tcol);
    s3_role<M, AX_COL_Y, true>(&m_tcol, &m_tcol, s3.col, s3, 1, base, wt, bar, sh, my_pj);
  } else {
    if (tid == 0) {
      prefetch_tmap(&m_trow_in);
      prefetch_tmap(&m_n);
    }
    s3_role<M, AX_ROW, false>(&m_trow_in, &m_n, s3.row, s3, 2, base, wt, bar, sh, my_pj);
  }
}

// ---------------------------------------------------------------------------------------
// k_line2: the M = 2048 line transform with TWO threads per radix-16 job (256 threads per
// line pair).  Same arithmetic and data layout as k_line (sinft pre-processing, complex FFT
// 16 x 16 x 8 of the two packed lines, Hermitian unpack on partner jobs, prefix sum), but a
// thread holds 8 complex values instead of 16: each radix-16 DFT is split by decimation in
// time into the DFT-8 of the even inputs (lane half h = 0) and of the odd inputs (h = 1),
// joined by one register exchange with the partner lane (lane ^ 16, four complex values) and
// the last radix-2 butterfly; the Hermitian partner jobs (ja, jb) of the last stage sit in
// the same two lanes.  Half the registers per thread -> more resident warps per SM (16
// instead of 12).  MEASURED SLOWER on c5 (profiles/r02/bench_line2_ab_*.json): x-passes
// 7.53 -> 9.89 ms, fused y-pass 8.17 -> 10.74 ms per sweep (3 CTAs/SM at 80 registers with
// spills: 10.8 / 10.9): the line kernels are bound by the LSU data pipe (75 % busy with the
// shared-memory wavefronts of the exchanges), not by latency, and the partner-lane shuffles
// and selects add to it.  Kept as an opt-in record of the experiment (EXPD_LINE2=1).
// Lane mapping inside a warp w: h = lane >> 4, job j = 16 w + (lane & 15): each half warp
// reads one contiguous run of a stage's inputs.
// ---------------------------------------------------------------------------------------
struct L2Geo {
  static constexpr int M = 2048, T = 256, RL = 8, NSL = M / RL;  // last stage: 256 jobs of 8
  static constexpr int L = (M / 2) / T;                           // k-values per thread (4)
  static constexpr int PADP = 16;
  static constexpr int SW = M + M / PADP;                         // padded positions
  static constexpr size_t BUFB = ((size_t)SW * 16 + 1023) / 1024 * 1024;
  static constexpr int NW = T / 32;
};
template <int NBUF>
constexpr size_t line2_smem() {
  return 1024 + NBUF * L2Geo::BUFB + 16 * L2Geo::NW + 16;
}
#ifndef EXPD_LINE2_MINB
#define EXPD_LINE2_MINB 2
#endif

// W / E arrays of the unpack without padding: a 2-bit XOR inside each 8-entry block makes
// the prefix reads (thread t: entries 4t .. 4t+3) conflict free
__device__ __forceinline__ int l2we(int k) { return k ^ ((k >> 3) & 3); }

// the partner lane's value (lane ^ 16)
__device__ __forceinline__ double2 xch16(double2 v) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
}

// Two-lane radix-16 DFT (DIR = -1, X_k = sum_r x_r W16^{rk}), in place: this lane holds
// x_{2m+h} (m = 0..7) in v; on return v[q] = X_{4h+q}, v[4+q] = X_{4h+q+8} (q = 0..3).
__device__ __forceinline__ void dft16_2lane(double2 (&v)[8], int h) {
  DFT<8, -1>::run(v);  // h = 0: E_k = DFT8(x_even), h = 1: O_k = DFT8(x_odd)
  // h = 1: O'_k = W16^k O_k (compile-time twiddles; the select keeps the warp converged)
  sfor<8>([&](auto kk) {
    constexpr int k = decltype(kk)::value;
    double2 t = v[k];
    twid<k, 16, -1>(t);
    v[k] = h ? t : v[k];
  });
  // h = 0 keeps E_0..3 and needs O'_0..3; h = 1 keeps O'_4..7 and needs E_4..7
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 give = h ? v[q] : v[4 + q];
    const double2 got = xch16(give);
    const double2 E = h ? got : v[q];
    const double2 Op = h ? v[4 + q] : got;
    v[q] = cadd(E, Op);
    v[4 + q] = csub(E, Op);
  }
}

template <int AX, bool NL, int NBUF>
__global__ void __launch_bounds__(L2Geo::T, EXPD_LINE2_MINB)
    k_line2(const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map,
            const __grid_constant__ LineArgs a) {
  using D = L2Geo;
  constexpr int M = D::M, T = D::T, L = D::L, NSL = D::NSL, PADP = D::PADP;
  extern __shared__ unsigned char lsm2_raw[];
  char* base = reinterpret_cast<char*>(lsm2_raw + ((1024u - (smem_u32(lsm2_raw) & 1023u)) & 1023u));
  double2* wt = reinterpret_cast<double2*>(base + NBUF * D::BUFB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wt + D::NW);
  const int tid = threadIdx.x;
  __builtin_assume(tid < T);
  const int lane = tid & 31, w = tid >> 5;
  const int h = lane >> 4;                   // half of the radix-16 job / partner job
  const int j = (w << 4) | (lane & 15);      // stage-0 / middle job, partner-pair index
  const int pj = j;
  const int ja = pj, jb = pj == 0 ? NSL / 2 : NSL - pj;
  const int J = h ? jb : ja;                 // this lane's last-stage job

  if (tid == 0) {
    prefetch_tmap(&in_map);
    prefetch_tmap(&out_map);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  long item = blockIdx.x;
  if (tid == 0 && item < a.nitems) line_issue_load<M, AX, 1>(&in_map, a, item, base, &bar[0]);

  for (int it = 0; item < a.nitems; ++it, item += gridDim.x) {
    const int cur = NBUF == 2 ? (it & 1) : 0;
    char* cb = base + cur * D::BUFB;
    double2* buf = reinterpret_cast<double2*>(cb);
    const long next = item + gridDim.x;
    if (NBUF == 2 && tid == 0 && next < a.nitems) {
      bulk_wait_read0();
      line_issue_load<M, AX, 1>(&in_map, a, next, base + (cur ^ 1) * D::BUFB, &bar[cur ^ 1]);
    }
    const double2* tw = a.tw;
    const double* pa = a.pa;
    asm volatile("" : "+l"(tw), "+l"(pa));
#ifndef EXPD_LINE2_LAZY_A
    double pre_a[8];  // loaded before the TMA wait (their latency hides behind it)
#pragma unroll
    for (int m = 0; m < 8; ++m) pre_a[m] = __ldg(pa + j + 128 * (2 * m + h));
#define L2_PRE_A(m) pre_a[m]
#else
#define L2_PRE_A(m) __ldg(pa + j + 128 * (2 * (m) + h))
#endif
    const double2 tmid = __ldg(tw + (j & 15) * 8);  // middle stage (NS = 16): w^{(j mod 16) M/256}
    const double2 tlast = __ldg(tw + J);
    mbar_wait(&bar[cur], (uint32_t)((NBUF == 2 ? (it >> 1) : it) & 1));

    double2 out[2 * L];
    int npass = NL ? 2 : 1;
    asm volatile("" : "+r"(npass));
#pragma unroll 1
    for (int pass = 0; pass < npass; ++pass) {
      // ---- stage 0: pre-processing + two-lane radix 16 over i = j + 128 r ------------
      double2 v[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int i = j + 128 * (2 * m + h);
        if (i == 0) {
          v[m] = make_double2(0.0, 0.0);
        } else if (AX == AX_ROW) {
          const uint32_t o1 = (uint32_t)(i - 1) * 8u, o2 = (uint32_t)(M - i - 1) * 8u;
          const double2 z = make_double2(*reinterpret_cast<const double*>(cb + o1),
                                         *reinterpret_cast<const double*>(cb + M * 8 + o1));
          const double2 zm = make_double2(*reinterpret_cast<const double*>(cb + o2),
                                          *reinterpret_cast<const double*>(cb + M * 8 + o2));
          v[m] = lpre(z, zm, L2_PRE_A(m), a.c);
        } else {
          const int p1 = i - 1, p2 = M - i - 1;
          const int q1 = pass ? lswz<PADP>(p1) : p1, q2 = pass ? lswz<PADP>(p2) : p2;
          v[m] = lpre(buf[q1], buf[q2], L2_PRE_A(m), a.c);
        }
      }
      dft16_2lane(v, h);
      __syncthreads();  // stage-0 reads of buf done
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        buf[lswz<PADP>(j * 16 + 4 * h + q)] = v[q];
        buf[lswz<PADP>(j * 16 + 4 * h + 8 + q)] = v[4 + q];
      }
      __syncthreads();
      // ---- middle stage (radix 16, NS = 16): inputs jm + 128 r, twiddle w^{r (jm mod 16) 8}
#pragma unroll
      for (int m = 0; m < 8; ++m) v[m] = buf[lswz<PADP>(j + 128 * (2 * m + h))];
      {
        const double2 w2 = cmul(tmid, tmid);
        double2 tp = h ? tmid : make_double2(1.0, 0.0);  // w^{(2m + h) b}
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          if (m > 0 || h) v[m] = cmul(v[m], tp);
          if (m + 1 < 8) tp = cmul(tp, w2);
        }
      }
      dft16_2lane(v, h);
      __syncthreads();
      {
        const int mbase = (j >> 4) * 256 + (j & 15);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          buf[lswz<PADP>(mbase + 16 * (4 * h + q))] = v[q];
          buf[lswz<PADP>(mbase + 16 * (4 * h + 8 + q))] = v[4 + q];
        }
      }
      __syncthreads();
      // ---- last stage (radix 8, NS = 256) on this lane's job J ------------------------
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = buf[lswz<PADP>(J + NSL * r)];
#ifdef EXPD_LINE2_TWSEQ
      {  // running product: two live twiddles (register-light, 7 roundings deep)
        double2 tp = tlast;
#pragma unroll
        for (int r = 1; r < 8; ++r) {
          v[r] = cmul(v[r], tp);
          if (r + 1 < 8) tp = cmul(tp, tlast);
        }
      }
#else
      ltwmul_w<8>(tlast, v);
#endif
      DFT<8, -1>::run(v);
      __syncthreads();  // every read of buf done: the unpack arrays overwrite it
      // ---- Hermitian unpack: k = J + 256 r pairs with M - k = partner's J' + 256 (7 - r)
      {
        double2 rcv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) rcv[q] = xch16(v[4 + q]);
        double2* Wb = buf;
        double2* Eb = buf + M / 2;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int k = J + NSL * r;
          const double2 own = pj == 0 ? (h == 0 ? v[(8 - r) & 7] : v[7 - r]) : rcv[3 - r];
          double2 e, wv;
          lunpack(v[r], own, h == 0 && pj == 0 && r == 0, e, wv);
          if (k >= 1) Eb[l2we(k - 1)] = e;  // E[k - 1] = e_k, k = 1 .. M/2 - 1
          Wb[l2we(k)] = wv;
        }
      }
      __syncthreads();
      // ---- prefix sum: thread t owns k in [4t, 4t + 4) -> positions [8t, 8t + 8) --------
      double2 tot = make_double2(0.0, 0.0);
      {
        const double2* Wb = buf;
        const double2* Eb = buf + M / 2;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          const int k = 4 * tid + l;
          tot = cadd(tot, Wb[l2we(k)]);
          out[2 * l] = tot;
          out[2 * l + 1] = (k == M / 2 - 1) ? make_double2(0.0, 0.0) : Eb[l2we(k)];  // e_{k+1}
        }
      }
      double2 inc = tot;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double ox = __shfl_up_sync(0xffffffffu, inc.x, d);
        const double oy = __shfl_up_sync(0xffffffffu, inc.y, d);
        if (lane >= d) inc = cadd(inc, make_double2(ox, oy));
      }
      double2 off = csub(inc, tot);
      if (lane == 31) wt[w] = inc;
      __syncthreads();
      for (int b = 0; b < w; ++b) off = cadd(off, wt[b]);
#pragma unroll
      for (int l = 0; l < L; ++l) out[2 * l] = cadd(out[2 * l], off);
      if (NL && pass + 1 < npass) {
        __syncthreads();  // the (e, w) reads are done
#pragma unroll
        for (int q = 0; q < 2 * L; ++q)
          buf[lswz<PADP>(8 * tid + q)] = make_double2(poly_eval(a.poly, out[q].x), poly_eval(a.poly, out[q].y));
        __syncthreads();
      }
    }
    __syncthreads();  // (e, w) reads and the cross-warp offsets done before the output
    if constexpr (AX == AX_ROW) {
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const int x = 8 * tid + 2 * l;
        const uint32_t off = row_sw(x);
        *reinterpret_cast<double2*>(cb + off) = make_double2(out[2 * l].x, out[2 * l + 1].x);
        *reinterpret_cast<double2*>(cb + M * 8 + off) = make_double2(out[2 * l].y, out[2 * l + 1].y);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 2 * L; ++q) buf[lswz<PADP>(8 * tid + q)] = out[q];
      __syncthreads();
      double2 c[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) c[r] = buf[lswz<PADP>(tid + T * r)];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; ++r) buf[tid + T * r] = c[r];
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      line_issue_store<M, AX, 1>(&out_map, a, item, cb);
      if (NBUF == 1 && next < a.nitems) {
        bulk_wait_read0();
        line_issue_load<M, AX, 1>(&in_map, a, next, base, &bar[0]);
      }
    }
  }
  if (tid == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------------------
// host side: tensor maps and launches
// ---------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool line_supported(const Geom& g) {
  return g.M >= 256 && g.M <= 4096 && encode_fn() != nullptr;
}

// 4-D fp64 tensor map: dims d[0..3] (d[0] contiguous), byte strides s[1..3], box b[0..3]
static cudaError_t make_map(CUtensorMap* m, const double* ptr, const cuuint64_t d[4], const cuuint64_t s[3],
                            const cuuint32_t b[4], bool sw128) {
  EncodeTiledFn f = encode_fn();
  if (!f) return cudaErrorNotSupported;
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(ptr), d, s, b, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("EXPD_DEBUG"))
    fprintf(stderr, "expd: cuTensorMapEncodeTiled failed (%d): dims %llu %llu %llu %llu box %u %u %u %u\n", (int)r,
            (unsigned long long)d[0], (unsigned long long)d[1], (unsigned long long)d[2], (unsigned long long)d[3],
            b[0], b[1], b[2], b[3]);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// L2 promotion of the K1 tile loads (EXPD_K1_PROMO: 0 none = default, 1 64B, 2 128B, 3 256B).
// Measured on c5 (profiles/r02/ncu_k1_promo_*.csv): 256B promotion over-fetches 0.7-1.5 GB of
// DRAM reads per K1 launch (each 128-byte box row is a different time slice) at the same
// duration; without promotion the reads equal the algorithmic 17.3 GB.
static CUtensorMapL2promotion k1_promotion() {
  const char* e = getenv("EXPD_K1_PROMO");
  switch (e ? atoi(e) : 0) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// 2-D fp64 tensor map (no swizzle): rows of `cols` doubles at byte stride row_bytes.
cudaError_t make_tmap_2d(CUtensorMap* m, const double* ptr, unsigned long long cols, unsigned long long rows,
                         unsigned long long row_bytes, unsigned box_cols, unsigned box_rows, bool sw128) {
  EncodeTiledFn f = encode_fn();
  if (!f) return cudaErrorNotSupported;
  const cuuint64_t d[2] = {cols, rows};
  const cuuint64_t s[1] = {row_bytes};
  const cuuint32_t b[2] = {box_cols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), d, s, b, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                 k1_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
bool tma_available() { return encode_fn() != nullptr; }

// Tensor map of nslices padded spectral slices for one axis pass (COL: G column pairs).
// ROW: sw = true for the output map (the per-thread chunk writes need the 128-byte swizzle
// to be conflict free), false for the input map (linear, see k_line's stage-0 reads)
static cudaError_t axis_map(CUtensorMap* m, const Geom& g, int ax, const double* ptr, long nslices, int G,
                            bool sw = true) {
  const cuuint64_t M = (cuuint64_t)g.M, n = (cuuint64_t)g.n;
  const cuuint64_t rows = (cuuint64_t)(g.npad / g.M);  // spectral rows per slice
  const cuuint64_t sl = (cuuint64_t)g.npad * 8;
  if (ax == AX_ROW) {
    const cuuint64_t d[4] = {16, M / 16, rows, (cuuint64_t)nslices};
    const cuuint64_t s[3] = {128, M * 8, sl};
    const cuuint32_t b[4] = {16, (cuuint32_t)(M / 16), 1, 1};
    return make_map(m, ptr, d, s, b, sw);
  }
  const cuuint64_t nz = g.dim == 3 ? n : 1;
  const cuuint64_t d[4] = {M, n, nz, (cuuint64_t)nslices};
  const cuuint64_t s[3] = {M * 8, n * M * 8, sl};
  if (ax == AX_COL_Y) {
    const cuuint32_t b[4] = {(cuuint32_t)(2 * G), (cuuint32_t)CBR, 1, 1};
    return make_map(m, ptr, d, s, b, false);
  }
  const cuuint32_t b[4] = {(cuuint32_t)(2 * G), 1, (cuuint32_t)CBR, 1};
  return make_map(m, ptr, d, s, b, false);
}

// 5-D fp64 tensor map (no swizzle), the COL result's transposed view: dims d[0..4] (d[0]
// contiguous), byte strides s[1..4] in any order, box b[0..4]
static cudaError_t make_map5(CUtensorMap* m, const double* ptr, const cuuint64_t d[5], const cuuint64_t s[4],
                             const cuuint32_t b[5]) {
  EncodeTiledFn f = encode_fn();
  if (!f) return cudaErrorNotSupported;
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(ptr), d, s, b, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && getenv("EXPD_DEBUG"))
    fprintf(stderr, "expd: cuTensorMapEncodeTiled (5-D) failed (%d)\n", (int)r);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// The transposed store view of a COL pass (k_line TS): grid row p = 2L a + q along the
// transformed axis becomes the pair of dims (a, q) with a INNER in shared memory, so the box
// {2G doubles, a < T-1, q < 2L} lands at slot (q (T-1) + a) G + g -- the layout the threads
// write without bank conflicts.  Rows 2L (T-1) .. M-2 are the last thread's (stored directly).
template <int M, int G>
static cudaError_t col_ts_map(CUtensorMap* m, const Geom& g, int ax, const double* ptr, long nslices) {
  using D = LGeo<M, G, 1>;
  const cuuint64_t n = (cuuint64_t)g.n, L2 = 2 * D::L, T = D::T;
  const cuuint64_t sl = (cuuint64_t)g.npad * 8, row = (cuuint64_t)M * 8;
  const cuuint64_t nz = g.dim == 3 ? n : 1;
  if (ax == AX_COL_Y) {  // dims {x, a, q, z, slice}
    const cuuint64_t d[5] = {(cuuint64_t)M, T, L2, nz, (cuuint64_t)nslices};
    const cuuint64_t s[4] = {L2 * row, row, n * row, sl};
    const cuuint32_t b[5] = {(cuuint32_t)(2 * G), (cuuint32_t)(T - 1), (cuuint32_t)L2, 1, 1};
    return make_map5(m, ptr, d, s, b);
  }
  // AX_COL_Z: dims {x, y, a, q, slice}
  const cuuint64_t d[5] = {(cuuint64_t)M, n, T, L2, (cuuint64_t)nslices};
  const cuuint64_t s[4] = {row, L2 * n * row, n * row, sl};
  const cuuint32_t b[5] = {(cuuint32_t)(2 * G), 1, (cuuint32_t)(T - 1), (cuuint32_t)L2, 1};
  return make_map5(m, ptr, d, s, b);
}

cudaError_t peer_slab_map(CUtensorMap* m, const Geom& g, double* base, long units, long slots, long slot_doubles,
                          bool swizzled) {
  const cuuint64_t M = (cuuint64_t)g.M;
  const cuuint64_t d[4] = {16, M / 16, (cuuint64_t)units, (cuuint64_t)slots};
  const cuuint64_t s[3] = {128, M * 8, (cuuint64_t)slot_doubles * 8};
  const cuuint32_t b[4] = {16, (cuuint32_t)(M / 16), 1, 1};
  return make_map(m, base, d, s, b, swizzled);
}

static int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// The skip flag the k_line launches of this host thread carry (line_skip_scope).
static thread_local const int* t_line_skip = nullptr;
LineSkipScope::LineSkipScope(const int* flag) : prev(t_line_skip) { t_line_skip = flag; }
LineSkipScope::~LineSkipScope() { t_line_skip = prev; }

template <int M, int AX, bool NL, int G, int NBUF, bool PP = false, bool TS = false, bool HY = false>
static cudaError_t launch_line(const Geom& g, const DstTables& t, const Poly& P, const double* in, double* out,
                               long nslices, cudaStream_t st, const PeerOut* peer = nullptr) {
  using D = LGeo<M, G, NBUF>;
  static_assert(!TS || AX != AX_ROW, "the transposed store is a COL layout");
  auto k = k_line<M, AX, NL, G, NBUF, PP, TS, HY>;
  static DevOnce once;  // per instantiation and device
  int per_sm = 1;
  if (cudaError_t e = smem_optin(once, k, D::SMEM, D::THREADS, &per_sm); e != cudaSuccess) return e;
  CUtensorMap mi, mo;
  // (a peer side's own map is unused: any valid pointer of the launch describes it)
  const double* in_m = (peer && peer->in_maps) ? out : in;
  double* out_m = (peer && peer->maps) ? const_cast<double*>(in) : out;
  cudaError_t e = axis_map(&mi, g, AX, in_m, nslices, G, /*sw=*/false);
  if (e != cudaSuccess) return e;
  if constexpr (TS) e = col_ts_map<M, G>(&mo, g, AX, out_m, nslices);
  else e = axis_map(&mo, g, AX, out_m, nslices, G, /*sw=*/AX == AX_ROW);
  if (e != cudaSuccess) return e;
  LineArgs a{};
  a.outp = out;
  const int rows = (int)(g.npad / g.M);
  if (AX == AX_ROW) {
    a.inner = (rows + 1) / 2;
    a.per_slice = a.inner;
  } else {
    a.inner = g.M / (2 * G);
    a.per_slice = a.inner * (g.dim == 3 ? g.n : 1);
  }
  a.rows = rows;
  a.nitems = (long)a.per_slice * nslices;
  a.tw = t.tw;
  a.pa = t.pa;
  a.sinp = t.sinp;
  a.c = 0.5 * sqrt(2.0 / (double)g.M);
  a.poly = P;
  a.skip = t_line_skip;
  if (peer) {
    if (AX != AX_ROW) return cudaErrorInvalidValue;
    a.peer = peer->maps;
    a.peer_slot0 = peer->slot0;
    a.peer_in = peer->in_maps;
    a.peer_in_slot0 = peer->in_slot0;
  }
  long grid = (long)sm_count() * per_sm;
  if (grid > a.nitems) grid = a.nitems;
  if (grid < 1) return cudaSuccess;
  k<<<(unsigned)grid, D::THREADS, D::SMEM, st>>>(mi, mo, a);
  return cudaGetLastError();
}

// strided-axis variant (G column pairs per item, NBUF buffers); EXPD_COLV=<G><NBUF>
// (e.g. 12, 22, 21, 41) overrides the default for tuning
static int colv() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EXPD_COLV");
    v = e ? atoi(e) : 0;
  }
  return v;
}
// The hybrid buffer schedule of the default line kernels (line_item HY; EXPD_LINE_HY=0 keeps
// the in-place schedule with the next item's load issued at the item's start).  Measured on c5
// (profiles/r02/line_hy_ab.txt): stage 3 15.88 -> 15.55 ms, sweep 21.92 -> 21.67 ms.
static bool line_hy() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EXPD_LINE_HY");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}
// EXPD_COLTS=0: the strided-axis result compacted in shared memory and stored as boxes of
// CBR rows (the round-1/2 layout) instead of the transposed store (A/B at M = 2048)
static bool colts() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EXPD_COLTS");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

template <int M, int AX, bool NL>
static cudaError_t launch_col(const Geom& g, const DstTables& t, const Poly& P, const double* in, double* out,
                              long nslices, cudaStream_t st) {
  if constexpr (M == 2048) {
    // measured on c5 inside the sweep (profiles/r01): plain strided pass fastest with 2
    // column pairs per item (32-byte TMA rows), the fused [V, N, V] pass with 1 pair and 2
    // buffers (22.93 vs 23.02 ms per sweep with 1 buffer once the partner-lane tables made
    // its transforms faster and the exposed TMA wait grew to 21 % of its samples)
    switch (colv()) {
      case 11: return launch_line<M, AX, NL, 1, 1, false, true>(g, t, P, in, out, nslices, st);
      case 12: return launch_line<M, AX, NL, 1, 2>(g, t, P, in, out, nslices, st);
      case 21: return launch_line<M, AX, NL, 2, 1>(g, t, P, in, out, nslices, st);
      case 22: return launch_line<M, AX, NL, 2, 2>(g, t, P, in, out, nslices, st);
      case 41: return launch_line<M, AX, NL, 4, 1>(g, t, P, in, out, nslices, st);
      case 13: return launch_line<M, AX, NL, 1, 2, true>(g, t, P, in, out, nslices, st);  // ping-pong
      case 23: return launch_line<M, AX, NL, 2, 2, true>(g, t, P, in, out, nslices, st);
      default:
        if (!colts()) {
          if constexpr (NL) return launch_line<M, AX, NL, 1, 2>(g, t, P, in, out, nslices, st);
          else return launch_line<M, AX, NL, 2, 2>(g, t, P, in, out, nslices, st);
        }
        if (line_hy()) {
          if constexpr (NL) return launch_line<M, AX, NL, 1, 2, false, true, true>(g, t, P, in, out, nslices, st);
          else return launch_line<M, AX, NL, 2, 2, false, true, true>(g, t, P, in, out, nslices, st);
        }
        if constexpr (NL) return launch_line<M, AX, NL, 1, 2, false, true>(g, t, P, in, out, nslices, st);
        else return launch_line<M, AX, NL, 2, 2, false, true>(g, t, P, in, out, nslices, st);
    }
  } else if constexpr (M == 4096) {
    if (line_hy()) return launch_line<M, AX, NL, 1, 2, false, true, true>(g, t, P, in, out, nslices, st);
    return launch_line<M, AX, NL, 1, 2, false, true>(g, t, P, in, out, nslices, st);
  } else {
    if (line_hy()) return launch_line<M, AX, NL, 2, 2, false, true, true>(g, t, P, in, out, nslices, st);
    return launch_line<M, AX, NL, 2, 2, false, true>(g, t, P, in, out, nslices, st);
  }
}

template <int AX, bool NL, int NBUF>
static cudaError_t launch_line2(const Geom& g, const DstTables& t, const Poly& P, const double* in, double* out,
                                long nslices, cudaStream_t st) {
  auto k = k_line2<AX, NL, NBUF>;
  constexpr size_t SMEM = line2_smem<NBUF>();
  static DevOnce once;  // per instantiation and device
  int per_sm = 1;
  if (cudaError_t e = smem_optin(once, k, SMEM, L2Geo::T, &per_sm); e != cudaSuccess) return e;
  CUtensorMap mi, mo;
  cudaError_t e = axis_map(&mi, g, AX, in, nslices, 1, /*sw=*/false);
  if (e != cudaSuccess) return e;
  if ((e = axis_map(&mo, g, AX, out, nslices, 1, /*sw=*/AX == AX_ROW)) != cudaSuccess) return e;
  LineArgs a{};
  const int rows = (int)(g.npad / g.M);
  if (AX == AX_ROW) {
    a.inner = (rows + 1) / 2;
    a.per_slice = a.inner;
  } else {
    a.inner = g.M / 2;
    a.per_slice = a.inner * (g.dim == 3 ? g.n : 1);
  }
  a.rows = rows;
  a.nitems = (long)a.per_slice * nslices;
  a.tw = t.tw;
  a.pa = t.pa;
  a.sinp = t.sinp;
  a.c = 0.5 * sqrt(2.0 / (double)g.M);
  a.poly = P;
  long grid = (long)sm_count() * per_sm;
  if (grid > a.nitems) grid = a.nitems;
  if (grid < 1) return cudaSuccess;
  k<<<(unsigned)grid, L2Geo::T, SMEM, st>>>(mi, mo, a);
  return cudaGetLastError();
}
// EXPD_LINE2=1 selects k_line2 at M = 2048 (measured slower than k_line, see above)
static bool use_line2() {
  const char* e = getenv("EXPD_LINE2");
  return e && e[0] == '1';
}

template <int M>
static cudaError_t line_pass_m(const Geom& g, const DstTables& t, const Poly& P, int ax, bool nl, const double* in,
                               double* out, long nslices, cudaStream_t st, const PeerOut* peer = nullptr) {
  if (peer) {  // the peer-store x pass: the default row kernel only
    if (ax != AX_ROW || nl) return cudaErrorInvalidValue;
    return launch_line<M, AX_ROW, false, 1, 2>(g, t, P, in, out, nslices, st, peer);
  }
  if constexpr (M == 2048) {
    if (use_line2()) {
      if (ax == AX_ROW) return launch_line2<AX_ROW, false, 2>(g, t, P, in, out, nslices, st);
      if (ax == AX_COL_Y)
        return nl ? launch_line2<AX_COL_Y, true, 2>(g, t, P, in, out, nslices, st)
                  : launch_line2<AX_COL_Y, false, 2>(g, t, P, in, out, nslices, st);
      return nl ? launch_line2<AX_COL_Z, true, 2>(g, t, P, in, out, nslices, st)
                : launch_line2<AX_COL_Z, false, 2>(g, t, P, in, out, nslices, st);
    }
  }
  if (ax == AX_ROW) {
    static int rv = -1;  // EXPD_ROWV=1: one buffer per CTA (more CTAs per SM)
    if (rv < 0) {
      const char* e = getenv("EXPD_ROWV");
      rv = e ? atoi(e) : 2;
    }
    if (rv == 1) return launch_line<M, AX_ROW, false, 1, 1>(g, t, P, in, out, nslices, st);
    if (rv == 3) return launch_line<M, AX_ROW, false, 1, 2, true>(g, t, P, in, out, nslices, st);  // ping-pong
    if (line_hy()) return launch_line<M, AX_ROW, false, 1, 2, false, false, true>(g, t, P, in, out, nslices, st);
    return launch_line<M, AX_ROW, false, 1, 2>(g, t, P, in, out, nslices, st);
  }
  if (ax == AX_COL_Y)
    return nl ? launch_col<M, AX_COL_Y, true>(g, t, P, in, out, nslices, st)
              : launch_col<M, AX_COL_Y, false>(g, t, P, in, out, nslices, st);
  return nl ? launch_col<M, AX_COL_Z, true>(g, t, P, in, out, nslices, st)
            : launch_col<M, AX_COL_Z, false>(g, t, P, in, out, nslices, st);
}

// ---- persistent stage 3 (host) ----------------------------------------------------------
size_t stage3p_ctl_bytes() { return sizeof(S3Ctl); }

// roles (x-IDST : fused y : x-DST) of the SMs: EXPD_S3P_SPLIT="n0,n1" overrides; default by
// the measured per-slice costs of the passes (fused y ~ 2.2 x one x pass at M = 2048)
static void s3p_split(int sms, int& n0, int& n1) {
  const char* e = getenv("EXPD_S3P_SPLIT");
  if (e && sscanf(e, "%d,%d", &n0, &n1) == 2 && n0 > 0 && n1 > 0 && n0 + n1 < sms) return;
  const double ry = 2.2;
  n0 = (int)(sms / (2.0 + ry) + 0.5);
  if (n0 < 1) n0 = 1;
  n1 = sms - 2 * n0;
}

template <int M>
static cudaError_t launch_s3p(const Geom& g, const DstTables& t, const Poly& P, const double* uhat, double* ring,
                              int K, double* nhat, long nslices, void* ctl, cudaStream_t st) {
  using D = LGeo<M, 1, 2>;
  auto k = k_stage3p<M>;
  static DevOnce once;
  int per_sm = 1;
  if (cudaError_t e = smem_optin(once, k, D::SMEM, D::THREADS, &per_sm); e != cudaSuccess) return e;
  CUtensorMap mu, mto, mtc, mti, mn;
  cudaError_t e;
  if ((e = axis_map(&mu, g, AX_ROW, uhat, nslices, 1, false)) != cudaSuccess) return e;
  if ((e = axis_map(&mto, g, AX_ROW, ring, K, 1, true)) != cudaSuccess) return e;
  if ((e = axis_map(&mtc, g, AX_COL_Y, ring, K, 1, false)) != cudaSuccess) return e;
  if ((e = axis_map(&mti, g, AX_ROW, ring, K, 1, false)) != cudaSuccess) return e;
  if ((e = axis_map(&mn, g, AX_ROW, nhat, nslices, 1, true)) != cudaSuccess) return e;
  S3Args s{};
  const int rows = (int)(g.npad / g.M);
  s.row.inner = (rows + 1) / 2;
  s.row.per_slice = s.row.inner;
  s.row.rows = rows;
  s.col.inner = g.M / 2;
  s.col.per_slice = s.col.inner;
  s.col.rows = rows;
  for (LineArgs* la : {&s.row, &s.col}) {
    la->nitems = (long)la->per_slice * nslices;
    la->tw = t.tw;
    la->pa = t.pa;
    la->sinp = t.sinp;
    la->c = 0.5 * sqrt(2.0 / (double)g.M);
    la->poly = P;
  }
  s.ctl = reinterpret_cast<S3Ctl*>(ctl);
  s.nslices = (int)nslices;
  s.K = K;
  s.sms = sm_count();
  s3p_split(s.sms, s.split0, s.split1);
  if ((e = cudaMemsetAsync(ctl, 0, sizeof(S3Ctl), st)) != cudaSuccess) return e;
  k<<<(unsigned)(s.sms * per_sm), D::THREADS, D::SMEM, st>>>(mu, mto, mtc, mti, mn, s);
  return cudaGetLastError();
}

// Is the persistent stage 3 selected for this geometry (2-D, TMA line kernels, slices <=
// kS3MaxSlices)?  Opt-in (EXPD_S3P=1): measured on c5 (profiles/r02/) it takes 17.6 ms against
// the chunked passes' 15.9 ms per sweep, and ncu counts 49.7 GB of DRAM traffic per launch --
// as much as the chunked passes.  A slice is 33.5 MB and every slice moves ~200 MB through the
// L2 (U-hat, the intermediate's write / in-place pass / read, N-hat) between the x-IDST that
// writes its intermediate and the x-DST that reads it, so the ring cannot stay in the 126 MB
// L2 at this size, and the per-role SM split idles SMs whenever a role waits.
bool stage3p_supported(const Geom& g, long nslices) {
  const char* e = getenv("EXPD_S3P");
  if (!(e && e[0] == '1')) return false;
  return g.dim == 2 && line_supported(g) && g.M >= 512 && nslices <= kS3MaxSlices;
}

cudaError_t stage3p(const Geom& g, const DstTables& t, const Poly& P, const double* uhat, double* ring, int K,
                    double* nhat, long nslices, void* ctl, cudaStream_t st) {
  if (nslices <= 0) return cudaSuccess;
  switch (g.M) {
    case 512: return launch_s3p<512>(g, t, P, uhat, ring, K, nhat, nslices, ctl, st);
    case 1024: return launch_s3p<1024>(g, t, P, uhat, ring, K, nhat, nslices, ctl, st);
    case 2048: return launch_s3p<2048>(g, t, P, uhat, ring, K, nhat, nslices, ctl, st);
    case 4096: return launch_s3p<4096>(g, t, P, uhat, ring, K, nhat, nslices, ctl, st);
    default: return cudaErrorInvalidValue;
  }
}

// One axis pass (ax: 0 = x rows, 1 = y, 2 = z) of nslices padded spectral slices; nl
// (strided axes only) fuses [V, N, V].  in and out may alias (each item reads and writes
// only its own lines).
cudaError_t line_pass(const Geom& g, const DstTables& t, const Poly& P, int ax, bool nl, const double* in,
                      double* out, long nslices, cudaStream_t st, const PeerOut* peer) {
  if (nslices <= 0) return cudaSuccess;
  if (ax == AX_ROW && nl) return cudaErrorInvalidValue;
  switch (g.M) {
    case 256: return line_pass_m<256>(g, t, P, ax, nl, in, out, nslices, st, peer);
    case 512: return line_pass_m<512>(g, t, P, ax, nl, in, out, nslices, st, peer);
    case 1024: return line_pass_m<1024>(g, t, P, ax, nl, in, out, nslices, st, peer);
    case 2048: return line_pass_m<2048>(g, t, P, ax, nl, in, out, nslices, st, peer);
    case 4096: return line_pass_m<4096>(g, t, P, ax, nl, in, out, nslices, st, peer);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace expd
