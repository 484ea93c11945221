// expd_internal.h -- internal types shared by the host driver and the kernels of libexpd.so.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdio>
#include <cstdint>
#include <string>
#include <vector>

// Device-side bounds checks of the checked build (python -m paper_2603_04350_b200.build
// --checked -> libexpd_checked.so, compiled with -DEXPD_CHECKS; the default build compiles
// them out).  A failed check prints what and where, then traps -- the stand-in for
// compute-sanitizer, which this GPU pool does not allow.
#ifdef EXPD_CHECKS
#define EXPD_CHECK(cond, what)                                                                              \
  do {                                                                                                      \
    if (!(cond)) {                                                                                          \
      printf("expd check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                             \
      __trap();                                                                                             \
    }                                                                                                       \
  } while (0)
#else
#define EXPD_CHECK(cond, what) ((void)0)
#endif

namespace expd {

// One-time setup of a kernel per DEVICE (the dynamic shared-memory opt-in is a property of
// the device context, so a plan on a second GPU of the same process needs its own): a bitmask
// of the devices already done plus the occupancy found there, one object per call site.
// Concurrent first calls may both run the (idempotent) setup; the atomics keep it race free.
struct DevOnce {
  std::atomic<unsigned long long> done{0};
  std::atomic<int> per_sm[64];
};
template <typename K>
inline cudaError_t smem_optin(DevOnce& o, K k, size_t smem_bytes, int threads = 0, int* per_sm = nullptr) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  dev &= 63;
  const unsigned long long bit = 1ull << dev;
  if (!(o.done.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    int v = 1;
    if (threads > 0) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, threads, smem_bytes);
      if (e != cudaSuccess) return e;
      if (v < 1) v = 1;
    }
    o.per_sm[dev].store(v, std::memory_order_relaxed);
    o.done.fetch_or(bit, std::memory_order_release);
  }
  if (per_sm) *per_sm = o.per_sm[dev].load(std::memory_order_relaxed);
  return cudaSuccess;
}

// Spectral layout: every x-line of a spectral slice is padded
// from n to n+1 doubles (n+1 = 2^m), so a spectral slice holds n^{dim-1} (n+1) doubles,
// every line and every pair of modes (2p, 2p+1) is 16-byte aligned, and the pad entry
// (jx = n) is an inert dummy mode that stays exactly 0 (its tables are 0).
struct Geom {
  int dim, n;
  long N;     // n^dim physical points per slice
  long npad;  // spectral slice length n^{dim-1} (n+1)
  int M;      // n + 1
};

// Pointwise nonlinearity N(u) = sum_{p < npoly} q[p] u^p (stage 3; BASELINE.json:9, :11).
struct Poly {
  int npoly;
  double q[8];
};
#ifdef __CUDACC__
__device__ __forceinline__ double poly_eval(const Poly& P, double u) {
  // straight-line Horner (unused coefficients are 0): no loop, no dynamic indexing
  double acc = P.q[3];
  acc = fma(acc, u, P.q[2]);
  acc = fma(acc, u, P.q[1]);
  acc = fma(acc, u, P.q[0]);
  if (P.npoly > 4) {
    double hi = P.q[7];
    hi = fma(hi, u, P.q[6]);
    hi = fma(hi, u, P.q[5]);
    hi = fma(hi, u, P.q[4]);
    const double u2 = u * u;
    acc = fma(hi, u2 * u2, acc);
  }
  return acc;
}
#endif

// Per-launch parameters of the time-local fused kernel (K1).
struct TimeArgs {
  int nt;
  long npad;
  long npairs;        // npad / 2
  const double* X;    // input space-time vector [nt][npad]
  double* Y;          // output [nt][npad] (may alias X)
  const double* u0h;  // spectral u_0 [npad]
  const double* Nh;   // nonlinear history [nt][npad], Nh[m] = V N(u_m), m = 0..nt-1
  const double* E;    // [npad] E_J = exp(dt mu_J), 0 on pads
  const double* C1;   // [npad] ETD1: dt phi1 ; ETD2: dt (phi1 + phi2)
  const double* C2;   // [npad] ETD2: dt phi2
  const double* g;    // [nt] alpha^{t/nt}
  const double* ginv; // [nt] alpha^{-t/nt}
  const double2* tw;  // [nt] exp(+2 pi i q / nt)
  double a1;          // alpha^{1/nt}
  double half_inv_nt; // 1 / (2 nt)
  double* partial;    // [gridDim.x] per-CTA sum of r^2 (nullable)
};

enum ResidMode { RM_INPUT = 0, RM_RESID = 1, RM_QOP = 2 };
enum OutMode { OUT_S = 0, OUT_UPDATE = 1 };

// kernel launchers (k_time.cu)
cudaError_t launch_time_fused(const TimeArgs& a, int rmode, int outmode, int nl, int grid, cudaStream_t st);
int time_fused_grid(int nt, long npairs, int sms, int nl);
cudaError_t launch_resid_only(const TimeArgs& a, int nl, int grid, cudaStream_t st);

// DST-I / nonlinear (k_dst.cu)
struct DstTables {
  const double2* tw;   // [M] exp(-2 pi i q / M)
  const double* sinp;  // [M] sin(pi i / M)
  const double* pa;    // [M] a_i = c (sin(pi i/M) + 1/2), c = sqrt(2/M)/2 (the line kernels' folded pre-processing)
};
// Orthonormal DST-I of every slice along every axis: physical (row stride n) <-> spectral
// (row stride n+1).  src/dst may alias only when both are spectral.
cudaError_t dst_slices(const Geom& g, const DstTables& t, const double* src, bool src_spectral, double* dst,
                       bool dst_spectral, long nslices, double* scratch, cudaStream_t st);
// N-hat = V N(V u-hat) for nslices spectral slices (stage 3 of the sweep, K4).
// Optional in-stream timing of stage 3's passes (profiling runs): an event is recorded
// before every axis pass and after the last one; kind[k] says which pass interval k is
// (0 x-pass, 1 plain strided pass, 2 fused strided [V, N, V] pass).  ext: recording inside
// a CUDA-graph capture.
struct PassTimer {
  cudaEvent_t* ev;
  int cap;
  bool ext;
  int used;
  int kind[512];
};
// Peer access of the distributed stage 3 (the fused "NVLink-store transposes"):
// the first x pass (x-IDST) loads each spectral row straight from the U-hat mode slab of the
// rank that owns it and the final x pass (x-DST) stores each row straight into the owner's
// N-hat slab (device memory of another process / GPU, opened through CUDA IPC), instead of
// two all-to-alls through time-slab staging.  One tensor map per rank and slab (in device
// memory, 64-byte aligned), rows [unit_off[q], unit_off[q] + units[q]).
constexpr int kMaxPeers = 16;
struct PeerMaps {
  CUtensorMap m[kMaxPeers];
  int nranks;
  int unit_off[kMaxPeers];
  int units[kMaxPeers];
};
struct PeerOut {
  const PeerMaps* maps;     // device, nullable: the x-DST rows -> the owners' N-hat slabs
  int slot0;                // N-hat slot of the launch's first slice
  const PeerMaps* in_maps;  // device, nullable: the x-IDST rows <- the owners' U-hat slabs
  int in_slot0;             // U-hat slot of the launch's first slice
};
cudaError_t nonlin_slices(const Geom& g, const DstTables& t, const double* uhat, double* nhat, long nslices,
                          int npoly, const double* q, double* scratch, cudaStream_t st, struct PassTimer* timer = nullptr,
                          void* s3ctl = nullptr, double* full_tmp = nullptr, const PeerOut* peer = nullptr);
// persistent stage 3 (k_line.cu): one launch for all slices, intermediate in a ring of K
// slices (ring: K npad doubles), dependency counters in ctl (stage3p_ctl_bytes(), zeroed by the
// launch).  PassTimer kind 3 marks it.
size_t stage3p_ctl_bytes();
bool stage3p_supported(const Geom& g, long nslices);
cudaError_t stage3p(const Geom& g, const DstTables& t, const Poly& P, const double* uhat, double* ring, int K,
                    double* nhat, long nslices, void* ctl, cudaStream_t st);
// N-hat = V N(u) for physical slices u (row stride n).
cudaError_t nonlin_phys_slices(const Geom& g, const DstTables& t, const double* u, double* nhat, long nslices,
                               int npoly, const double* q, double* scratch, cudaStream_t st);
size_t dst_scratch_doubles(const Geom& g, long max_slices);
cudaError_t dst_debug_time(const Geom& g, const DstTables& t, int which, double* a, double* b, long nslices,
                           int npoly, const double* q, int reps, float* ms, cudaStream_t st);
int nonlin_chunk_slices(const Geom& g);
// TMA line kernels (k_line.cu): one axis pass (0 = x rows, 1 = y, 2 = z) over padded
// spectral slices, nl fusing [V, N, V] on a strided axis.  in / out may alias.
bool line_supported(const Geom& g);
bool tma_available();
cudaError_t make_tmap_2d(CUtensorMap* m, const double* ptr, unsigned long long cols, unsigned long long rows,
                         unsigned long long row_bytes, unsigned box_cols, unsigned box_rows, bool sw128 = false);
cudaError_t line_pass(const Geom& g, const DstTables& t, const Poly& P, int ax, bool nl, const double* in,
                      double* out, long nslices, cudaStream_t st, const PeerOut* peer = nullptr);
// the tensor map of one rank's slab for PeerMaps: units x-lines of M doubles per slot, slots
// slots, slot stride slot_doubles (the mode-slab length); swizzled = the row kernel's result
// layout (N-hat stores), else its linear input layout (U-hat loads)
cudaError_t peer_slab_map(CUtensorMap* m, const Geom& g, double* base, long units, long slots, long slot_doubles,
                          bool swizzled);
int nonlin_kernel_launches(const Geom& g, long nslices, bool full_tmp = false);
// While in scope, every k_line launch of this host thread (stage 3 included) reads the device
// int `flag` first and does nothing if it is non-zero: the device loop skips stage 3 of its
// first sweep when N-hat is known to be zero (zero guess, N(0) = 0), without a second graph.
struct LineSkipScope {
  explicit LineSkipScope(const int* flag);
  ~LineSkipScope();
  const int* prev;
};

// vector kernels (k_vec.cu)
cudaError_t mode_tables(const Geom& g, const double* lam_axis, double a, double c, double dt, int scheme,
                        double* E, double* C1, double* C2, cudaStream_t st);
cudaError_t reduce_partials(const double* partial, int n, double* out, cudaStream_t st);
// GMRES / CGS2 helpers over vectors of length len (all 16-byte aligned, len even)
// (cx: complex vectors, Hermitian inner products, complex coefficients as (re, im) pairs)
cudaError_t multi_dot(const double* const* V, int nv, const double* w, long len, double* partial, int grid,
                      double* out, cudaStream_t st, bool cx = false);
cudaError_t multi_axpy_dot(const double* const* V, int nv, const double* coef_dev, double* w, long len,
                           double* partial, int grid, double* out, int want_dot, cudaStream_t st, bool cx = false);
cudaError_t scale_copy(const double* x, double s, double* y, long len, cudaStream_t st);
cudaError_t scale_copy_cx(const double* x, double sr, double si, double* y, long len, cudaStream_t st);
cudaError_t lincomb_add(const double* const* V, int nv, const double* coef_dev, double* x, long len,
                        cudaStream_t st, bool cx = false);
// complex interleaved slices <-> planar (re, im) slice pairs (complex plans)
// physical rows (stride n) <-> padded spectral rows (stride M), zeroing the pad (k_vec.cu)
cudaError_t repitch(const double* in, long in_rs, double* out, long out_rs, int width, long rows, cudaStream_t st);
cudaError_t cx_split(const double* in, long in_stride, long len, double* out, long out_stride, long nslices,
                     cudaStream_t st);
cudaError_t cx_merge(const double* in, long in_stride, long len, double* out, long out_stride, long nslices,
                     cudaStream_t st);
int vec_grid(int sms);
// device-side fixed-point loop state (expd_fixed_point_solve's CUDA-graph WHILE loop)
constexpr int kFpLoopHist = 1024;  // history entries: the device loop takes maxit < kFpLoopHist
struct FpLoopState {
  int k, status, maxit;
  int s3skip;  // stage 3 of the next sweep is skipped (N-hat known to be 0); k_fp_conv clears it
  double r0, tol;
  double hist[kFpLoopHist];
};
cudaError_t launch_fp_conv(cudaGraphConditionalHandle h, FpLoopState* st, const double* norm2, cudaStream_t s);

// ---- multi-GPU (dist.cu) ----------------------------------------------------------------
constexpr int EXPD_MAX_RANKS = 64;
struct DistLayout {
  int rank, nranks, nt;
  long npad;                       // entries per full padded spectral slice
  long unit;                       // partition unit of the mode slabs
  long mode_off[EXPD_MAX_RANKS];   // mode slab of rank q: entries [off, off + len) of every slice
  long mode_len[EXPD_MAX_RANKS];
  int t0[EXPD_MAX_RANKS];          // time slab of rank q: slices [t0, t0 + ntl)
  int ntl[EXPD_MAX_RANKS];
};
struct A2AMsg {
  int peer;
  long src_off, dst_off, count;  // doubles
  int slice;                     // index of the slice within its time slab (pipelining key)
};
enum A2ADir { A2A_MODE_TO_TIME = 0, A2A_TIME_TO_MODE = 1 };
bool dist_layout(const Geom& g, int nt, int rank, int nranks, DistLayout* L);
// the geometry the partition of a complex plan is computed on: a spectral slice of 2 npad
// doubles with x-lines of 2 M doubles (interleaved (re, im) per mode)
inline Geom complex_layout_geom(const Geom& g) {
  Geom c = g;
  c.npad = 2 * g.npad;
  c.M = 2 * g.M;
  return c;
}
void a2a_schedule(const DistLayout& L, int dir, int shift, std::vector<A2AMsg>& sends, std::vector<A2AMsg>& recvs);
// executes the messages whose slice key lies in [s_lo, s_hi) (one chunk of a pipelined
// all-to-all; every rank must pass the same range)
int a2a_execute(void* comm, const DistLayout& L, const std::vector<A2AMsg>& sends, const std::vector<A2AMsg>& recvs,
                const double* src, double* dst, cudaStream_t st, std::string& err, int s_lo = 0,
                int s_hi = 1 << 30);
int allreduce_sum(void* comm, int nranks, double* buf, long count, cudaStream_t st, std::string& err);

}  // namespace expd
