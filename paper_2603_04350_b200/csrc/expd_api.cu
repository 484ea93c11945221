// expd_api.cu -- host side of libexpd.so: plan (tables), workspace carving, the C-ABI
// entry points of include/expd.h, and the solver drivers (Richardson / Picard (3.2) and
// left-preconditioned restarted GMRES with CGS2).  Every arithmetic step on the space-time
// data runs in the kernels of k_time.cu / k_dst.cu / k_vec.cu; the host does only the
// O(restart^2) Givens / least-squares scalars of GMRES and the convergence tests.
#include <cuda_runtime.h>

#include <chrono>
#include <cstddef>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <string>
#include <vector>

#include "../../include/expd.h"
#include "expd_internal.h"

using namespace expd;

struct expd_plan {
  expd_problem prob{};
  expd_dist dinfo{};
  int device = 0;
  cudaStream_t stream = nullptr;
  Geom g{};
  int sms = 148;
  int nl = 0;      // 0 linear, 1 ETD1 / IF-IMEX, 2 ETD2
  int nshift = 0;  // IF / IMEX-type: K1 reads N-hat of the same slice (one slice later)
  int k1 = 0;      // K1 form: nl, 3 for the BDF2 system, 4 for complex coefficients
  bool cx = false; // complex coefficients: spectral entries are (re, im) pairs, mlen = 2 npad
  std::vector<double> h_Ecx;  // complex E_J table (re, im) [2 npad], long double on the host
  double *X2 = nullptr, *X3 = nullptr;  // complex plans: planar (re / im) transform staging
  double a1 = 0.0;
  // small device tables owned by the plan
  double* d_lam = nullptr;   // [n]
  double2* d_twt = nullptr;  // [nt]  e^{+2 pi i q/nt}
  double* d_g = nullptr;     // [nt]  alpha^{t/nt}
  double* d_ginv = nullptr;  // [nt]
  double2* d_twM = nullptr;  // [M]   e^{-2 pi i q/M}
  double* d_sinp = nullptr;  // [M]   sin(pi i/M)
  double* d_pa = nullptr;    // [M]   c (sin(pi i/M) + 1/2), c = sqrt(2/M)/2
  double* h_pin = nullptr;   // pinned host scalars [256]
  // workspace (caller-owned)
  char* ws = nullptr;
  size_t ws_bytes = 0;
  // distribution: dist = the mode-slab / time-slab schedule with all-to-alls
  bool dist = false;
  DistLayout L{};
  long mlen = 0, moff = 0;  // this rank's mode slab (= the whole slice when !dist)
  int ntl = 0, t0 = 0;      // this rank's time slab (= all slices when !dist)
  std::vector<A2AMsg> m2t_s, m2t_r, t2m_s, t2m_r, t2m1_s, t2m1_r;  // all-to-all schedules
  double *UT = nullptr, *NT = nullptr;  // time-slab spectral staging [ntl][npad] (dist only)
  double *Uh = nullptr, *Nh = nullptr, *T1 = nullptr, *u0h = nullptr, *E = nullptr, *C1 = nullptr, *C2 = nullptr;
  double *scratch = nullptr, *partial = nullptr, *dscal = nullptr;
  double* krylov = nullptr;
  int krylov_cap = 0;
  int time_grid = 0, vgrid = 0;
  bool tables_ready = false;
  // CUDA graph of one sweep (captured on a private stream, launched on `stream`)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t sweep_exec = nullptr;
  // the fixed-point solve's device-side loop: WHILE (not converged) { sweep; reduce; test }
  cudaGraphExec_t loop_exec = nullptr;
  FpLoopState* loopst = nullptr;  // device state in the workspace
  void* s3ctl = nullptr;            // persistent stage 3's dependency counters (workspace)
  FpLoopState* h_loopst = nullptr;  // pinned host copy
  bool loop_failed = false;         // the graph could not be built: host-driven loop
  // solver I/O: zero initial guess (expd_set_zero_guess) and host u0 / U (staged, the final
  // inverse DST streamed out chunk by chunk with the device-to-host copy)
  bool zero_guess = false;
  double* hstage = nullptr;          // [N] (x2 complex) device staging of a host u0
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> cev;
  bool capturing = false;
  bool eager_done = false;  // one eager sweep (kernel attributes) before the first capture
  // optional stage timing: ev[0] before stage 3, ev[1] before K1, ev[2] after K1
  bool prof = false;
  int prof_level = 0;  // 1: stage events; 2: + an event between every stage-3 pass
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> tev;  // per-pass events of stage 3 (profiling, single GPU)
  PassTimer timer{};
  // distributed sweep pipelining: the all-to-alls run on comm_stream in chunks of the time
  // slab, overlapped with stage 3 of the neighbouring chunks (events in pev)
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> pev;
  // Krylov step timing (profiling on): device ms of every Arnoldi / BiCGStab step of the last
  // solve, from two events on the plan's stream around the step's kernels
  cudaEvent_t kev[2] = {nullptr, nullptr};
  std::vector<double> kstep_ms;
  // peer stores of the distributed stage 3 (expd_plan_enable_peer_stores): every rank's N-hat
  // mode slab (its own, or another process's opened through CUDA IPC) and their tensor maps
  std::vector<double*> peer_nh, peer_uh;
  std::vector<void*> peer_ipc;  // IPC-opened allocation bases (closed at destroy)
  PeerMaps* d_peer = nullptr;   // [0]: the N-hat slabs (stores), [1]: the U-hat slabs (loads)
  bool peer_on = false;
  std::string err;
};

static const size_t kAlign = 256;
static size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

static expd_status fail(expd_plan* p, expd_status s, const std::string& m) {
  if (p) p->err = m;
  return s;
}
#define CUDA_TRY(p, x)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      return fail(p, EXPD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

static bool is_pow2(long v) { return v > 0 && (v & (v - 1)) == 0; }

// ---------------------------------------------------------------------------------------
// tables (long double, rounded to double): PAPER.md:113-114 (omega, Gamma_alpha, lambda_k),
// reading R1 (lambda_j), DST-I twiddles.
// ---------------------------------------------------------------------------------------
static const long double PI_L = 3.141592653589793238462643383279502884197L;

static expd_status build_tables(expd_plan* p) {
  const expd_problem& P = p->prob;
  const int n = P.n, M = n + 1, nt = P.nt;
  std::vector<double> lam(n), g(nt), gi(nt), sinp(M);
  std::vector<double2> twt(nt), twM(M);
  std::vector<double> pa(M);
  const long double h = 1.0L / (long double)M;
  for (int j = 1; j <= n; ++j) {
    long double s = sinl(PI_L * (long double)j / (2.0L * (long double)M));
    lam[j - 1] = (double)(-4.0L / (h * h) * s * s);
  }
  for (int q = 0; q < nt; ++q) {
    long double ang = 2.0L * PI_L * (long double)q / (long double)nt;
    twt[q] = make_double2((double)cosl(ang), (double)sinl(ang));
    long double gq = powl((long double)P.alpha, (long double)q / (long double)nt);
    g[q] = (double)gq;
    gi[q] = (double)(1.0L / gq);
  }
  for (int q = 0; q < M; ++q) {
    long double ang = 2.0L * PI_L * (long double)q / (long double)M;
    twM[q] = make_double2((double)cosl(ang), (double)(-sinl(ang)));
    sinp[q] = (double)sinl(PI_L * (long double)q / (long double)M);
    // the line kernels' pre-processing y_i = s_i (x_i + x_{M-i}) + (x_i - x_{M-i})/2 written as
    // y_i = a_i x_i + b_i x_{M-i}, a = c (s + 1/2), b = a - c, with the orthonormal scale
    // sqrt(2/M) and the 1/2 of the Hermitian unpack folded in as c (the transform is linear)
    const long double cq = 0.5L * sqrtl(2.0L / (long double)M), sq = sinl(PI_L * (long double)q / (long double)M);
    pa[q] = (double)(cq * (sq + 0.5L));
  }
  p->a1 = (double)powl((long double)P.alpha, 1.0L / (long double)nt);
  CUDA_TRY(p, cudaSetDevice(p->device));
  CUDA_TRY(p, cudaMalloc(&p->d_lam, sizeof(double) * n));
  CUDA_TRY(p, cudaMalloc(&p->d_twt, sizeof(double2) * nt));
  CUDA_TRY(p, cudaMalloc(&p->d_g, sizeof(double) * nt));
  CUDA_TRY(p, cudaMalloc(&p->d_ginv, sizeof(double) * nt));
  CUDA_TRY(p, cudaMalloc(&p->d_twM, sizeof(double2) * M));
  CUDA_TRY(p, cudaMalloc(&p->d_sinp, sizeof(double) * M));
  CUDA_TRY(p, cudaMalloc(&p->d_pa, sizeof(double) * M));
  CUDA_TRY(p, cudaMallocHost(&p->h_pin, sizeof(double) * 512));
  CUDA_TRY(p, cudaMemcpy(p->d_lam, lam.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(p, cudaMemcpy(p->d_twt, twt.data(), sizeof(double2) * nt, cudaMemcpyHostToDevice));
  CUDA_TRY(p, cudaMemcpy(p->d_g, g.data(), sizeof(double) * nt, cudaMemcpyHostToDevice));
  CUDA_TRY(p, cudaMemcpy(p->d_ginv, gi.data(), sizeof(double) * nt, cudaMemcpyHostToDevice));
  CUDA_TRY(p, cudaMemcpy(p->d_twM, twM.data(), sizeof(double2) * M, cudaMemcpyHostToDevice));
  CUDA_TRY(p, cudaMemcpy(p->d_sinp, sinp.data(), sizeof(double) * M, cudaMemcpyHostToDevice));
  CUDA_TRY(p, cudaMemcpy(p->d_pa, pa.data(), sizeof(double) * M, cudaMemcpyHostToDevice));
  return EXPD_OK;
}

extern "C" expd_status expd_plan_create(const expd_problem* prob, const expd_dist* dist, int device,
                                        void* cuda_stream, expd_plan** out) {
  if (!prob || !out) return EXPD_ERR_INVALID_ARG;
  *out = nullptr;
  const expd_problem& P = *prob;
  const bool cx = P.a_im != 0.0 || P.c_im != 0.0;
  // real plans: a > 0, c >= 0; complex plans: Re a >= 0, Re c >= 0, a != 0 (|E_J| <= 1)
  const bool coef_ok = cx ? (P.a >= 0.0 && P.c >= 0.0 && (P.a > 0.0 || P.a_im != 0.0) && std::isfinite(P.a_im) &&
                             std::isfinite(P.c_im))
                          : (P.a > 0.0 && P.c >= 0.0);
  if (P.dim < 1 || P.dim > 3 || P.n < 3 || !is_pow2((long)P.n + 1) || P.n + 1 > 4096 || !coef_ok ||
      !(P.dt > 0.0) || P.nt < 4 || !is_pow2(P.nt) || !(P.alpha > 0.0) || !(P.alpha <= 1.0) ||
      P.npoly < 0 || P.npoly > 8 ||
      (P.scheme != EXPD_EXP_EULER && P.scheme != EXPD_ETD2 && P.scheme != EXPD_IF_IMEX &&
       P.scheme != EXPD_BDF2) ||
      (P.scheme == EXPD_BDF2 && P.npoly > 0) ||
      !std::isfinite(P.a) || !std::isfinite(P.c) || !std::isfinite(P.dt))
    return EXPD_ERR_INVALID_ARG;
  if (P.nt > 256) return EXPD_ERR_UNSUPPORTED;
  if (cx && (P.npoly > 0 || (P.scheme != EXPD_EXP_EULER && P.scheme != EXPD_BDF2)))
    return EXPD_ERR_UNSUPPORTED;  // complex plans: linear exponential Euler or BDF2
  int nranks = dist ? dist->nranks : 1;
  if (nranks < 1 || nranks > EXPD_MAX_RANKS || (dist && (dist->rank < 0 || dist->rank >= nranks)))
    return EXPD_ERR_INVALID_ARG;
  if (nranks > 1 && (!dist->nccl_comm || P.nt % nranks != 0)) return EXPD_ERR_INVALID_ARG;
  // breakdown guard: min_{k,J} |1 - lambda_k E_J| >= 1 - alpha^{1/nt} max_J E_J (R10)
  {
    long double h = 1.0L / (long double)(P.n + 1);
    long double s = sinl(PI_L / (2.0L * (long double)(P.n + 1)));
    long double mu_max = (long double)P.a * (long double)P.dim * (-4.0L / (h * h) * s * s) - (long double)P.c;
    long double Emax = expl((long double)P.dt * mu_max);
    long double a1 = powl((long double)P.alpha, 1.0L / (long double)P.nt);
    if (1.0L - a1 * Emax < 1e-14L) return EXPD_ERR_BREAKDOWN;
  }
  expd_plan* p = new expd_plan();
  p->prob = P;
  if (dist) p->dinfo = *dist;
  else p->dinfo.nranks = 1;
  p->device = device;
  p->stream = (cudaStream_t)cuda_stream;
  p->g.dim = P.dim;
  p->g.n = P.n;
  p->g.M = P.n + 1;
  long N = 1, npad = P.n + 1;
  for (int i = 0; i < P.dim; ++i) N *= P.n;
  for (int i = 1; i < P.dim; ++i) npad *= P.n;
  p->g.N = N;
  p->g.npad = npad;
  // K1 form: 0 linear, 1 one N-hat term (ETD1; IF/IMEX with N of the same slice), 2 ETD2
  p->nl = P.npoly > 0 ? (P.scheme == EXPD_ETD2 ? 2 : 1) : 0;
  p->nshift = (P.npoly > 0 && P.scheme == EXPD_IF_IMEX) ? 1 : 0;
  // K1 form: 3 BDF2 system, 4 complex coefficients, 5 complex BDF2
  p->k1 = P.scheme == EXPD_BDF2 ? (cx ? 5 : 3) : (cx ? 4 : p->nl);
  p->cx = cx;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete p;
    return EXPD_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
  expd_status st = build_tables(p);
  if (st != EXPD_OK) {
    expd_plan_destroy(p);
    return st;
  }
  p->dist = nranks > 1 || (dist && dist->nccl_comm);
  // the partition is computed in doubles of a spectral slice: a complex slice has 2 npad
  // (interleaved (re, im) per mode, whole padded x-lines of 2 M doubles per slab unit)
  if (!dist_layout(cx ? complex_layout_geom(p->g) : p->g, P.nt, p->dist ? dist->rank : 0, p->dist ? nranks : 1,
                   &p->L)) {
    expd_plan_destroy(p);
    return EXPD_ERR_INVALID_ARG;
  }
  p->mlen = p->L.mode_len[p->L.rank];  // doubles per slice of the mode slab
  p->moff = p->L.mode_off[p->L.rank];
  p->ntl = p->L.ntl[p->L.rank];
  p->t0 = p->L.t0[p->L.rank];
  if (p->dist) {
    a2a_schedule(p->L, A2A_MODE_TO_TIME, 0, p->m2t_s, p->m2t_r);
    a2a_schedule(p->L, A2A_TIME_TO_MODE, 0, p->t2m_s, p->t2m_r);
    a2a_schedule(p->L, A2A_TIME_TO_MODE, 1, p->t2m1_s, p->t2m1_r);
  }
  p->time_grid = time_fused_grid(P.nt, p->mlen / 2, p->sms, p->nl);
  if (cx) {
    // E_J = exp(dt (a mu_J^0 - c)), complex, in long double (the phase dt (Im a mu - Im c) reaches
    // ~1e5 rad at n = 1023: a double evaluation would lose ~1e-11 of it).  Pads get 0.
    const int n = P.n, M = n + 1;
    const long double h = 1.0L / (long double)M;
    std::vector<long double> lam(n);
    for (int j = 1; j <= n; ++j) {
      long double sn = sinl(PI_L * (long double)j / (2.0L * (long double)M));
      lam[j - 1] = -4.0L / (h * h) * sn * sn;
    }
    p->h_Ecx.assign(2 * (size_t)npad, 0.0);
    for (long J = 0; J < npad; ++J) {
      const int jx = (int)(J % M);
      if (jx >= n) continue;
      long r = J / M;
      long double mu = lam[jx];
      for (int ax = 1; ax < P.dim; ++ax) {
        mu += lam[r % n];
        r /= n;
      }
      const long double re = (long double)P.dt * ((long double)P.a * mu - (long double)P.c);
      const long double im = (long double)P.dt * ((long double)P.a_im * mu - (long double)P.c_im);
      const long double mag = expl(re);
      p->h_Ecx[2 * J] = (double)(mag * cosl(im));
      p->h_Ecx[2 * J + 1] = (double)(mag * sinl(im));
    }
  }
  p->vgrid = vec_grid(p->sms);
  *out = p;
  return EXPD_OK;
}

// workspace layout (every block 256-byte aligned)
struct Layout {
  size_t Uh, Nh, T1, UT, NT, X2, X3, u0h, E, C1, C2, scratch, partial, dscal, loopst, s3ctl, hstage, krylov, total,
      vec;
};
static Layout layout(const expd_plan* p, int kv) {
  Layout L{};
  // space-time vectors in the mode slab: [nt][mlen]; N-hat gets one extra slice when
  // distributed (stage 3 of the last time slab lands there, unused)
  const size_t vec = align_up(sizeof(double) * (size_t)p->prob.nt * (size_t)p->mlen);
  const size_t nhv = align_up(sizeof(double) * (size_t)(p->prob.nt + ((p->dist || p->nshift) ? 1 : 0)) *
                              (size_t)p->mlen);
  const size_t tsl =
      p->dist ? align_up(sizeof(double) * (size_t)p->ntl * (size_t)p->g.npad * (p->cx ? 2 : 1)) : 0;
  const size_t sl = align_up(sizeof(double) * (size_t)p->g.npad * (p->cx ? 2 : 1));
  size_t off = 0;
  L.vec = vec;
  L.Uh = off; off += vec;
  L.Nh = off; off += (p->nl ? nhv : 0);
  L.T1 = off; off += vec;
  L.UT = off; off += tsl;
  L.NT = off; off += (p->nl ? tsl : 0);
  // complex planar staging (cx_phys_to_mode / cx_mode_to_phys): up to ns = nt (one GPU) or
  // ntl (the time slab) slices, i.e. 2 ns npad doubles in X2 and 2 ns N <= 2 ns npad in X3 --
  // NOT the mode-slab vector size, which is smaller on ranks with a short mode slab
  const size_t cxs =
      p->cx ? align_up(sizeof(double) * 2 * (size_t)(p->dist ? p->ntl : p->prob.nt) * (size_t)p->g.npad) : 0;
  L.X2 = off; off += cxs;
  L.X3 = off; off += cxs;
  L.u0h = off; off += sl;
  L.E = off; off += sl;
  L.C1 = off; off += sl;
  L.C2 = off; off += sl;
  L.scratch = off; off += align_up(sizeof(double) * dst_scratch_doubles(p->g, nonlin_chunk_slices(p->g)));
  L.partial = off; off += align_up(sizeof(double) * 32 * (size_t)(p->sms * 8 + 64));
  L.dscal = off; off += align_up(sizeof(double) * 512);
  L.loopst = off; off += align_up(sizeof(FpLoopState));
  L.s3ctl = off; off += align_up(stage3p_ctl_bytes());
  L.hstage = off; off += align_up(sizeof(double) * (size_t)p->g.N * (p->cx ? 2 : 1));
  L.krylov = off; off += (size_t)kv * vec;
  L.total = off;
  return L;
}

extern "C" expd_status expd_plan_workspace_bytes(const expd_plan* p, int krylov_vectors, size_t* bytes) {
  if (!p || !bytes || krylov_vectors < 0 || krylov_vectors > 32) return EXPD_ERR_INVALID_ARG;
  *bytes = layout(p, krylov_vectors).total;
  return EXPD_OK;
}

extern "C" expd_status expd_plan_set_workspace(expd_plan* p, void* d_ptr, size_t bytes) {
  if (!p || !d_ptr) return EXPD_ERR_INVALID_ARG;
  p->peer_on = false;  // the N-hat slab moves: peers register again
  if (((uintptr_t)d_ptr) % kAlign) return fail(p, EXPD_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  Layout L0 = layout(p, 0);
  if (bytes < L0.total) return fail(p, EXPD_ERR_OOM, "workspace smaller than expd_plan_workspace_bytes(plan, 0)");
  int kv = (int)((bytes - L0.total) / L0.vec);
  if (kv > 32) kv = 32;
  Layout L = layout(p, kv);
  p->ws = (char*)d_ptr;
  p->ws_bytes = bytes;
  auto at = [&](size_t off) { return (double*)(p->ws + off); };
  p->Uh = at(L.Uh);
  p->Nh = p->nl ? at(L.Nh) : nullptr;
  p->T1 = at(L.T1);
  p->UT = p->dist ? at(L.UT) : nullptr;
  p->NT = (p->dist && p->nl) ? at(L.NT) : nullptr;
  p->X2 = p->cx ? at(L.X2) : nullptr;
  p->X3 = p->cx ? at(L.X3) : nullptr;
  p->u0h = at(L.u0h);
  p->E = at(L.E);
  p->C1 = at(L.C1);
  p->C2 = at(L.C2);
  p->scratch = at(L.scratch);
  p->partial = at(L.partial);
  p->dscal = at(L.dscal);
  p->loopst = reinterpret_cast<FpLoopState*>(p->ws + L.loopst);
  p->s3ctl = p->ws + L.s3ctl;
  p->hstage = at(L.hstage);
  p->krylov = kv ? at(L.krylov) : nullptr;
  p->krylov_cap = kv;
  if (p->sweep_exec) {
    cudaGraphExecDestroy(p->sweep_exec);
    p->sweep_exec = nullptr;
  }
  if (p->loop_exec) {  // both graphs hold workspace pointers
    cudaGraphExecDestroy(p->loop_exec);
    p->loop_exec = nullptr;
  }
  CUDA_TRY(p, cudaSetDevice(p->device));
  if (p->cx)
    CUDA_TRY(p, cudaMemcpyAsync(p->E, p->h_Ecx.data(), sizeof(double) * p->h_Ecx.size(), cudaMemcpyHostToDevice,
                                p->stream));
  else
    CUDA_TRY(p, mode_tables(p->g, p->d_lam, p->prob.a, p->prob.c, p->prob.dt, p->prob.scheme, p->E, p->C1, p->C2,
                            p->stream));
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));  // the host table outlives the copy
  p->tables_ready = true;
  return EXPD_OK;
}

extern "C" void expd_plan_destroy(expd_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->sweep_exec) cudaGraphExecDestroy(p->sweep_exec);
  if (p->loop_exec) cudaGraphExecDestroy(p->loop_exec);
  if (p->h_loopst) cudaFreeHost(p->h_loopst);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  for (cudaEvent_t e : p->cev) cudaEventDestroy(e);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->comm_stream) cudaStreamDestroy(p->comm_stream);
  for (cudaEvent_t e : p->pev) cudaEventDestroy(e);
  for (int i = 0; i < 3; ++i)
    if (p->ev[i]) cudaEventDestroy(p->ev[i]);
  for (cudaEvent_t e : p->tev) cudaEventDestroy(e);
  for (cudaEvent_t e : p->kev)
    if (e) cudaEventDestroy(e);
  for (void* b : p->peer_ipc) cudaIpcCloseMemHandle(b);
  cudaFree(p->d_peer);
  cudaFree(p->d_lam);
  cudaFree(p->d_twt);
  cudaFree(p->d_g);
  cudaFree(p->d_ginv);
  cudaFree(p->d_twM);
  cudaFree(p->d_sinp);
  cudaFree(p->d_pa);
  if (p->h_pin) cudaFreeHost(p->h_pin);
  delete p;
}

extern "C" const char* expd_plan_last_error(const expd_plan* p) { return p ? p->err.c_str() : "null plan"; }

// ---------------------------------------------------------------------------------------
// internal helpers
// ---------------------------------------------------------------------------------------
static DstTables dst_tables(const expd_plan* p) { return DstTables{p->d_twM, p->d_sinp, p->d_pa}; }

static TimeArgs time_args(const expd_plan* p, const double* X, double* Y, bool with_partial) {
  TimeArgs a{};
  a.nt = p->prob.nt;
  a.npad = p->mlen;  // mode slab: slice stride and mode count (= npad on one GPU)
  a.npairs = p->mlen / 2;
  a.X = X;
  a.Y = Y;
  a.u0h = p->u0h + p->moff;
  a.Nh = p->Nh ? p->Nh + p->nshift * p->mlen : nullptr;  // IF / IMEX: N-hat of u_{t+1} for slice t
  a.E = p->E + p->moff;
  a.C1 = p->C1 + p->moff;
  a.C2 = p->C2 + p->moff;
  a.g = p->d_g;
  a.ginv = p->d_ginv;
  a.tw = p->d_twt;
  a.a1 = p->a1;
  a.half_inv_nt = 0.5 / (double)p->prob.nt;
  a.partial = with_partial ? p->partial : nullptr;
  return a;
}

static expd_status ready(expd_plan* p) {
  if (!p) return EXPD_ERR_INVALID_ARG;
  if (!p->ws || !p->tables_ready) return fail(p, EXPD_ERR_INVALID_ARG, "workspace not set");
  if (cudaSetDevice(p->device) != cudaSuccess) return fail(p, EXPD_ERR_CUDA, "cudaSetDevice");
  return EXPD_OK;
}

// spectral u0 and (nonlinear) N-hat_0 = V N(u_0)
// ---- distribution helpers (no-ops / local copies on one GPU) ---------------------------
enum { A2A_M2T = 0, A2A_T2M = 1, A2A_T2M_SHIFT = 2 };
// one all-to-all (or the chunk of it whose messages carry slice keys in [lo, hi))
static expd_status a2a(expd_plan* p, int which, const double* src, double* dst, cudaStream_t st = nullptr,
                       int lo = 0, int hi = 1 << 30) {
  const std::vector<A2AMsg>* s = &p->m2t_s;
  const std::vector<A2AMsg>* r = &p->m2t_r;
  if (which == A2A_T2M) { s = &p->t2m_s; r = &p->t2m_r; }
  if (which == A2A_T2M_SHIFT) { s = &p->t2m1_s; r = &p->t2m1_r; }
  int e = a2a_execute(p->dinfo.nccl_comm, p->L, *s, *r, src, dst, st ? st : p->stream, p->err, lo, hi);
  return (expd_status)e;
}
static expd_status allreduce(expd_plan* p, double* buf, long count) {
  if (!p->dist) return EXPD_OK;
  return (expd_status)allreduce_sum(p->dinfo.nccl_comm, p->L.nranks, buf, count, p->stream, p->err);
}

// spectral u0 (full slice, every rank) and (nonlinear) N-hat_0 = V N(u_0) (this rank's
// mode slab of it in Nh slice 0)
// complex plans: ns interleaved complex physical slices <-> interleaved complex spectral
// slices, through the planar staging X3 (physical) / X2 (spectral) and the real DST
static expd_status cx_phys_to_mode(expd_plan* p, const double* U, double* mode, long ns) {
  const long N = p->g.N, np = p->g.npad;
  CUDA_TRY(p, cx_split(U, 2 * N, N, p->X3, N, ns, p->stream));
  CUDA_TRY(p, dst_slices(p->g, dst_tables(p), p->X3, false, p->X2, true, 2 * ns, p->scratch, p->stream));
  CUDA_TRY(p, cx_merge(p->X2, np, np, mode, 2 * np, ns, p->stream));
  return EXPD_OK;
}
static expd_status cx_mode_to_phys(expd_plan* p, const double* mode, double* U, long ns) {
  const long N = p->g.N, np = p->g.npad;
  CUDA_TRY(p, cx_split(mode, 2 * np, np, p->X2, np, ns, p->stream));
  CUDA_TRY(p, dst_slices(p->g, dst_tables(p), p->X2, true, p->X3, false, 2 * ns, p->scratch, p->stream));
  CUDA_TRY(p, cx_merge(p->X3, N, N, U, 2 * N, ns, p->stream));
  return EXPD_OK;
}

static expd_status load_u0(expd_plan* p, const double* u0) {
  if (p->cx) return cx_phys_to_mode(p, u0, p->u0h, 1);
  CUDA_TRY(p, dst_slices(p->g, dst_tables(p), u0, false, p->u0h, true, 1, p->scratch, p->stream));
  if (p->nl) {
    double* full = p->dist ? p->UT : p->Nh;
    CUDA_TRY(p, nonlin_phys_slices(p->g, dst_tables(p), u0, full, 1, p->prob.npoly, p->prob.q, p->scratch,
                                   p->stream));
    if (p->dist)
      CUDA_TRY(p, cudaMemcpyAsync(p->Nh, p->UT + p->moff, sizeof(double) * p->mlen, cudaMemcpyDeviceToDevice,
                                  p->stream));
  }
  return EXPD_OK;
}

// physical time-slab slices (the API layout) <-> the spectral mode slab
static expd_status phys_to_mode(expd_plan* p, const double* U, double* mode) {
  if (p->cx && !p->dist) return cx_phys_to_mode(p, U, mode, p->prob.nt);
  if (p->cx) {  // the local time slab -> interleaved complex spectral slices -> mode slab
    expd_status s = cx_phys_to_mode(p, U, p->UT, p->ntl);
    if (s) return s;
    return a2a(p, A2A_T2M, p->UT, mode);
  }
  if (!p->dist) {
    CUDA_TRY(p, dst_slices(p->g, dst_tables(p), U, false, mode, true, p->prob.nt, p->scratch, p->stream));
    return EXPD_OK;
  }
  CUDA_TRY(p, dst_slices(p->g, dst_tables(p), U, false, p->UT, true, p->ntl, p->scratch, p->stream));
  return a2a(p, A2A_T2M, p->UT, mode);
}
static expd_status mode_to_phys(expd_plan* p, const double* mode, double* U) {
  if (p->cx && !p->dist) return cx_mode_to_phys(p, mode, U, p->prob.nt);
  if (p->cx) {
    expd_status s = a2a(p, A2A_M2T, mode, p->UT);
    if (s) return s;
    return cx_mode_to_phys(p, p->UT, U, p->ntl);
  }
  if (!p->dist) {
    CUDA_TRY(p, dst_slices(p->g, dst_tables(p), mode, true, U, false, p->prob.nt, p->scratch, p->stream));
    return EXPD_OK;
  }
  expd_status s = a2a(p, A2A_M2T, mode, p->UT);
  if (s) return s;
  CUDA_TRY(p, dst_slices(p->g, dst_tables(p), p->UT, true, U, false, p->ntl, p->scratch, p->stream));
  return EXPD_OK;
}

// One sweep on the spectral state: stage 3 (nonlinear history of u_1..u_{nt-1}), then the
// fused residual / norm / preconditioner / update (stages 1, 2), then the norm reduction.
static cudaError_t record(expd_plan* p, int i, cudaStream_t st) {
  if (!p->prof) return cudaSuccess;
  return p->capturing ? cudaEventRecordWithFlags(p->ev[i], st, cudaEventRecordExternal) : cudaEventRecord(p->ev[i], st);
}

// K1 (residual, ||r||^2, preconditioner, update) and the norm reduction of one sweep
static cudaError_t enqueue_k1(expd_plan* p, cudaStream_t st) {
  TimeArgs a = time_args(p, p->Uh, p->Uh, true);
  cudaError_t e = launch_time_fused(a, RM_RESID, OUT_UPDATE, p->k1, p->time_grid, st);
  if (e != cudaSuccess) return e;
  if ((e = record(p, 2, st)) != cudaSuccess) return e;
  return reduce_partials(p->partial, p->time_grid, p->dscal, st);
}

static bool s3_skip0_enabled() {
  const char* e = getenv("EXPD_S3_SKIP0");
  return !(e && e[0] == '0');
}

static cudaError_t enqueue_sweep(expd_plan* p, cudaStream_t st) {
  cudaError_t e = record(p, 0, st);
  if (e != cudaSuccess) return e;
  if (p->nl) {
    PassTimer* tm = nullptr;
    if (p->prof_level >= 2 && !p->tev.empty()) {
      p->timer.ev = p->tev.data();
      p->timer.cap = (int)p->tev.size();
      p->timer.ext = p->capturing;
      tm = &p->timer;
    }
    e = nonlin_slices(p->g, dst_tables(p), p->Uh, p->Nh + p->g.npad, p->prob.nt - 1 + p->nshift, p->prob.npoly,
                      p->prob.q, p->scratch, st, tm, p->s3ctl, p->T1);  // T1 is free during a sweep
    if (e != cudaSuccess) return e;
  }
  if ((e = record(p, 1, st)) != cudaSuccess) return e;
  return enqueue_k1(p, st);
}

// The distributed sweep: all-to-all U-hat (mode -> time slab), stage 3 on the
// local time slices, all-to-all N-hat back (time slab -> mode slab, shifted one slice:
// N-hat_m = V N(u_m) sits in slice m while U-hat slice t holds u_{t+1}), K1 on the mode
// slab, allreduce of ||r||^2.
// Chunks of the time slab in the pipelined distributed sweep (EXPD_DIST_CHUNKS, default 8;
// 1 = the unpipelined schedule).
static int dist_chunks(const expd_plan* p) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EXPD_DIST_CHUNKS");
    v = e ? atoi(e) : 8;
    if (v < 1) v = 1;
  }
  return v < p->ntl ? v : p->ntl;
}

// Stage 3 of the distributed sweep, pipelined over chunks of the time slab: the mode ->
// time all-to-all of every chunk is posted on comm_stream up front; chunk c's stage 3 runs
// on the plan stream once its slices have landed, and its time -> mode all-to-all follows
// on comm_stream while stage 3 moves on to chunk c + 1.  Every rank posts the same chunk
// sequence (slice keys), so the NCCL groups match across ranks.
static expd_status allreduce(expd_plan* p, double* buf, long count);

// Stage 3 with peer access: the x-IDST pass loads every row of the time slab straight from its
// owner's U-hat slab (slot t) and the x-DST pass stores every row straight into its owner's
// N-hat slab (slot t + 1) -- no all-to-all, no time-slab staging.  Two allreduces are the
// barriers: every rank's U-hat is final before any rank loads it (after K1 of the last sweep
// or expd_load_state's all-to-all), and every rank's stores are done before any rank's K1.
static expd_status peer_barrier(expd_plan* p) {
  CUDA_TRY(p, cudaMemsetAsync(p->dscal + 500, 0, sizeof(double), p->stream));
  return allreduce(p, p->dscal + 500, 1);
}

static expd_status stage3_peer(expd_plan* p) {
  expd_status s;
  if ((s = peer_barrier(p))) return s;
  PeerOut po{p->d_peer, p->t0 + 1, p->d_peer + 1, p->t0};
  CUDA_TRY(p, nonlin_slices(p->g, dst_tables(p), nullptr, nullptr, p->ntl, p->prob.npoly, p->prob.q, p->scratch,
                            p->stream, nullptr, nullptr, nullptr, &po));
  return peer_barrier(p);
}

static expd_status stage3_dist(expd_plan* p) {
  expd_status s;
  if (p->peer_on) return stage3_peer(p);
  const int nch = dist_chunks(p);
  if (nch <= 1) {
    if ((s = a2a(p, A2A_M2T, p->Uh, p->UT))) return s;
    CUDA_TRY(p, nonlin_slices(p->g, dst_tables(p), p->UT, p->NT, p->ntl, p->prob.npoly, p->prob.q, p->scratch,
                              p->stream));
    return a2a(p, A2A_T2M_SHIFT, p->NT, p->Nh);
  }
  if (!p->comm_stream) {
    // highest priority: the exchange's kernels take SM slots as soon as a stage-3 kernel
    // releases them, instead of queueing behind the next persistent stage-3 grid
    int lo = 0, hi = 0;
    CUDA_TRY(p, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(p, cudaStreamCreateWithPriority(&p->comm_stream, cudaStreamNonBlocking, hi));
  }
  while ((int)p->pev.size() < 2 * nch + 2) {
    cudaEvent_t e;
    CUDA_TRY(p, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->pev.push_back(e);
  }
  const int k = (p->ntl + nch - 1) / nch;
  cudaStream_t cs = p->comm_stream;
  CUDA_TRY(p, cudaEventRecord(p->pev[0], p->stream));  // U-hat is final (K1 of the last sweep)
  CUDA_TRY(p, cudaStreamWaitEvent(cs, p->pev[0], 0));
  for (int c = 0; c < nch && c * k < p->ntl; ++c) {
    const int lo = c * k, hi = lo + k < p->ntl ? lo + k : p->ntl;
    if ((s = a2a(p, A2A_M2T, p->Uh, p->UT, cs, lo, hi))) return s;
    CUDA_TRY(p, cudaEventRecord(p->pev[2 + c], cs));
  }
  for (int c = 0; c < nch && c * k < p->ntl; ++c) {
    const int lo = c * k, hi = lo + k < p->ntl ? lo + k : p->ntl;
    CUDA_TRY(p, cudaStreamWaitEvent(p->stream, p->pev[2 + c], 0));
    CUDA_TRY(p, nonlin_slices(p->g, dst_tables(p), p->UT + (size_t)lo * p->g.npad, p->NT + (size_t)lo * p->g.npad,
                              hi - lo, p->prob.npoly, p->prob.q, p->scratch, p->stream));
    CUDA_TRY(p, cudaEventRecord(p->pev[2 + nch + c], p->stream));
    CUDA_TRY(p, cudaStreamWaitEvent(cs, p->pev[2 + nch + c], 0));
    if ((s = a2a(p, A2A_T2M_SHIFT, p->NT, p->Nh, cs, lo, hi))) return s;
  }
  CUDA_TRY(p, cudaEventRecord(p->pev[1], cs));
  CUDA_TRY(p, cudaStreamWaitEvent(p->stream, p->pev[1], 0));
  return EXPD_OK;
}

static expd_status sweep_dist(expd_plan* p) {
  expd_status s;
  CUDA_TRY(p, record(p, 0, p->stream));
  if (p->nl && (s = stage3_dist(p))) return s;
  CUDA_TRY(p, record(p, 1, p->stream));
  TimeArgs a = time_args(p, p->Uh, p->Uh, true);
  CUDA_TRY(p, launch_time_fused(a, RM_RESID, OUT_UPDATE, p->k1, p->time_grid, p->stream));
  CUDA_TRY(p, record(p, 2, p->stream));
  CUDA_TRY(p, reduce_partials(p->partial, p->time_grid, p->dscal, p->stream));
  return allreduce(p, p->dscal, 1);
}

static expd_status sweep(expd_plan* p, bool use_graph) {
  if (p->dist) return sweep_dist(p);
  if (!use_graph || !p->eager_done) {
    p->eager_done = true;
    CUDA_TRY(p, enqueue_sweep(p, p->stream));
    return EXPD_OK;
  }
  if (!p->sweep_exec) {
    cudaGraph_t graph;
    if (!p->cap_stream) CUDA_TRY(p, cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
    CUDA_TRY(p, cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
    p->capturing = true;
    cudaError_t e = enqueue_sweep(p, p->cap_stream);
    p->capturing = false;
    cudaError_t e2 = cudaStreamEndCapture(p->cap_stream, &graph);
    if (e != cudaSuccess) return fail(p, EXPD_ERR_CUDA, std::string("sweep capture: ") + cudaGetErrorString(e));
    if (e2 != cudaSuccess) return fail(p, EXPD_ERR_CUDA, std::string("end capture: ") + cudaGetErrorString(e2));
    e = cudaGraphInstantiate(&p->sweep_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(p, EXPD_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  }
  CUDA_TRY(p, cudaGraphLaunch(p->sweep_exec, p->stream));
  return EXPD_OK;
}

static bool graphs_enabled() {
  const char* s = getenv("EXPD_NO_GRAPH");
  return !(s && s[0] == '1');
}

static expd_status read_scalars(expd_plan* p, int count, double* out) {
  CUDA_TRY(p, cudaMemcpyAsync(p->h_pin, p->dscal, sizeof(double) * count, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));
  for (int i = 0; i < count; ++i) out[i] = p->h_pin[i];
  return EXPD_OK;
}

// ---------------------------------------------------------------------------------------
// C-ABI: primitives
// ---------------------------------------------------------------------------------------
extern "C" expd_status expd_residual(expd_plan* p, const double* u0, const double* U, double* R,
                                     double* rnorm2_host) {
  expd_status s = ready(p);
  if (s) return s;
  if (!u0 || !U || !R || U == R) return fail(p, EXPD_ERR_INVALID_ARG, "expd_residual: bad pointers");
  const long nt = p->prob.nt;
  s = load_u0(p, u0);
  if (s) return s;
  if ((s = phys_to_mode(p, U, p->Uh))) return s;
  if (p->nl && !p->dist && nt > 1)  // N-hat_m = V N(u_m), m = 1..nt-1, from the physical slices
    CUDA_TRY(p, nonlin_phys_slices(p->g, dst_tables(p), U, p->Nh + p->g.npad, nt - 1 + p->nshift, p->prob.npoly,
                                   p->prob.q, p->scratch, p->stream));
  if (p->nl && p->dist) {  // local physical slices -> N-hat time slab -> mode slab (shifted)
    CUDA_TRY(p, nonlin_phys_slices(p->g, dst_tables(p), U, p->NT, p->ntl, p->prob.npoly, p->prob.q, p->scratch,
                                   p->stream));
    if ((s = a2a(p, A2A_T2M_SHIFT, p->NT, p->Nh))) return s;
  }
  TimeArgs a = time_args(p, p->Uh, p->T1, true);
  CUDA_TRY(p, launch_resid_only(a, p->k1, p->time_grid, p->stream));
  CUDA_TRY(p, reduce_partials(p->partial, p->time_grid, p->dscal, p->stream));
  if ((s = allreduce(p, p->dscal, 1))) return s;
  if ((s = mode_to_phys(p, p->T1, R))) return s;
  if (rnorm2_host) return read_scalars(p, 1, rnorm2_host);
  return EXPD_OK;
}

extern "C" expd_status expd_precond_apply(expd_plan* p, const double* R, double* S) {
  expd_status s = ready(p);
  if (s) return s;
  if (!R || !S) return fail(p, EXPD_ERR_INVALID_ARG, "expd_precond_apply: bad pointers");
  if ((s = phys_to_mode(p, R, p->T1))) return s;
  TimeArgs a = time_args(p, p->T1, p->T1, false);
  CUDA_TRY(p, launch_time_fused(a, RM_INPUT, OUT_S, p->k1 >= 3 ? p->k1 : 0, p->time_grid, p->stream));
  return mode_to_phys(p, p->T1, S);
}

extern "C" expd_status expd_load_state(expd_plan* p, const double* u0, const double* U) {
  expd_status s = ready(p);
  if (s) return s;
  if (!u0) return fail(p, EXPD_ERR_INVALID_ARG, "expd_load_state: u0 is null");
  s = load_u0(p, u0);
  if (s) return s;
  if (U && !p->zero_guess) return phys_to_mode(p, U, p->Uh);
  CUDA_TRY(p, cudaMemsetAsync(p->Uh, 0, sizeof(double) * p->prob.nt * p->mlen, p->stream));
  return EXPD_OK;
}

extern "C" expd_status expd_sweep(expd_plan* p) {
  expd_status s = ready(p);
  if (s) return s;
  return sweep(p, graphs_enabled());
}

extern "C" expd_status expd_sweep_norm2(expd_plan* p, double* rnorm2_host) {
  expd_status s = ready(p);
  if (s) return s;
  if (!rnorm2_host) return EXPD_ERR_INVALID_ARG;
  return read_scalars(p, 1, rnorm2_host);
}

extern "C" expd_status expd_store_state(expd_plan* p, double* U) {
  expd_status s = ready(p);
  if (s) return s;
  if (!U) return EXPD_ERR_INVALID_ARG;
  return mode_to_phys(p, p->Uh, U);
}

extern "C" expd_status expd_dst(expd_plan* p, const double* in, double* out, long nslices) {
  expd_status s = ready(p);
  if (s) return s;
  if (!in || !out || nslices < 0) return fail(p, EXPD_ERR_INVALID_ARG, "expd_dst: bad args");
  // spectral temporary: T1 (nt padded slices) on one GPU, the time-slab staging otherwise
  const long chunk = p->dist ? p->ntl : p->prob.nt;
  double* tmp = p->dist ? p->UT : p->T1;
  for (long s0 = 0; s0 < nslices; s0 += chunk) {
    long ns = nslices - s0 < chunk ? nslices - s0 : chunk;
    CUDA_TRY(p, dst_slices(p->g, dst_tables(p), in + s0 * p->g.N, false, tmp, true, ns, p->scratch, p->stream));
    // drop the pad column: spectral rows of n+1 doubles -> rows of n doubles
    CUDA_TRY(p, repitch(tmp, p->g.M, out + s0 * p->g.N, p->g.n, p->g.n, ns * (p->g.N / p->g.n), p->stream));
  }
  return EXPD_OK;
}

extern "C" expd_status expd_nonlin_hat(expd_plan* p, const double* uhat, double* nhat, long nslices) {
  expd_status s = ready(p);
  if (s) return s;
  if (!uhat || !nhat || nslices < 0) return fail(p, EXPD_ERR_INVALID_ARG, "expd_nonlin_hat: bad args");
  // T1 (nt padded slices: input half, output half) on one GPU; UT / NT when distributed
  const long chunk = p->dist ? p->ntl : p->prob.nt / 2;
  const size_t rows = (size_t)(p->g.N / p->g.n);
  if (p->dist && !p->nl) return fail(p, EXPD_ERR_UNSUPPORTED, "expd_nonlin_hat: linear distributed plan");
  if (p->cx) return fail(p, EXPD_ERR_UNSUPPORTED, "expd_nonlin_hat: real plans only");
  double* tin = p->dist ? p->UT : p->T1;
  double* tout = p->dist ? p->NT : p->T1 + chunk * p->g.npad;
  for (long s0 = 0; s0 < nslices; s0 += chunk) {
    const long ns = nslices - s0 < chunk ? nslices - s0 : chunk;
    CUDA_TRY(p, repitch(uhat + s0 * p->g.N, p->g.n, tin, p->g.M, p->g.n, (long)(ns * rows), p->stream));
    CUDA_TRY(p, nonlin_slices(p->g, dst_tables(p), tin, tout, ns, p->prob.npoly, p->prob.q, p->scratch, p->stream));
    CUDA_TRY(p, repitch(tout, p->g.M, nhat + s0 * p->g.N, p->g.n, p->g.n, (long)(ns * rows), p->stream));
  }
  return EXPD_OK;
}

extern "C" expd_status expd_set_profiling(expd_plan* p, int enable) {
  expd_status s = ready(p);
  if (s) return s;
  for (int i = 0; i < 3; ++i)
    if (!p->ev[i]) CUDA_TRY(p, cudaEventCreate(&p->ev[i]));
  for (int i = 0; i < 2; ++i)
    if (!p->kev[i]) CUDA_TRY(p, cudaEventCreate(&p->kev[i]));
  if (p->tev.empty() && p->nl && !p->dist) {  // one event per stage-3 pass + the end
    const long ns = p->prob.nt - 1 + p->nshift, ch = nonlin_chunk_slices(p->g);
    const long cap = ((ns + ch - 1) / ch) * 5 + 2;
    p->tev.resize(cap < 512 ? cap : 512);
    for (auto& e : p->tev) CUDA_TRY(p, cudaEventCreate(&e));
  }
  const int level = enable <= 0 ? 0 : (enable >= 2 ? 2 : 1);
  if (p->prof_level != level && p->sweep_exec) {
    cudaGraphExecDestroy(p->sweep_exec);  // recapture with / without the event nodes
    p->sweep_exec = nullptr;
  }
  if (p->prof_level != level && p->loop_exec) {
    cudaGraphExecDestroy(p->loop_exec);
    p->loop_exec = nullptr;
  }
  p->prof = level != 0;
  p->prof_level = level;
  return EXPD_OK;
}

extern "C" expd_status expd_sweep_stage_ms(expd_plan* p, double* ms_nonlin, double* ms_time) {
  if (!p || !p->prof) return fail(p, EXPD_ERR_INVALID_ARG, "profiling not enabled");
  float a = 0.f, b = 0.f;
  CUDA_TRY(p, cudaEventSynchronize(p->ev[2]));
  CUDA_TRY(p, cudaEventElapsedTime(&a, p->ev[0], p->ev[1]));
  CUDA_TRY(p, cudaEventElapsedTime(&b, p->ev[1], p->ev[2]));
  if (ms_nonlin) *ms_nonlin = a;
  if (ms_time) *ms_time = b;
  return EXPD_OK;
}

extern "C" expd_status expd_sweep_pass_ms(expd_plan* p, double* ms_x, double* ms_strided, double* ms_fused,
                                          int* n_x, int* n_strided, int* n_fused) {
  if (!p || p->prof_level < 2) return fail(p, EXPD_ERR_INVALID_ARG, "pass profiling (level 2) not enabled");
  if (p->tev.empty() || p->timer.used < 2)
    return fail(p, EXPD_ERR_UNSUPPORTED, "no stage-3 pass timing (linear, distributed or non-TMA plan)");
  double t[3] = {0.0, 0.0, 0.0};
  int n[3] = {0, 0, 0};
  CUDA_TRY(p, cudaEventSynchronize(p->tev[p->timer.used - 1]));
  for (int k = 0; k + 1 < p->timer.used; ++k) {
    float m = 0.f;
    CUDA_TRY(p, cudaEventElapsedTime(&m, p->tev[k], p->tev[k + 1]));
    int kind = p->timer.kind[k];
    if (kind == 3) kind = 2;  // the persistent stage 3 (one launch, all passes) -> the fused slot
    if (kind >= 0 && kind < 3) {
      t[kind] += m;
      ++n[kind];
    }
  }
  if (ms_x) *ms_x = t[0];
  if (ms_strided) *ms_strided = t[1];
  if (ms_fused) *ms_fused = t[2];
  if (n_x) *n_x = n[0];
  if (n_strided) *n_strided = n[1];
  if (n_fused) *n_fused = n[2];
  return EXPD_OK;
}

extern "C" expd_status expd_solver_step_ms(const expd_plan* p, double* ms, int cap, int* count) {
  if (!p || !count || cap < 0 || (cap > 0 && !ms)) return EXPD_ERR_INVALID_ARG;
  const int n = (int)p->kstep_ms.size();
  for (int i = 0; i < n && i < cap; ++i) ms[i] = p->kstep_ms[i];
  *count = n;
  return EXPD_OK;
}

extern "C" expd_status expd_debug_kernel_ms(expd_plan* p, int which, long nslices, int reps, double* ms) {
  expd_status s = ready(p);
  if (s) return s;
  if (!ms || reps < 1 || nslices < 1 || nslices > p->prob.nt) return fail(p, EXPD_ERR_INVALID_ARG, "debug: bad args");
  if (p->dist) return fail(p, EXPD_ERR_UNSUPPORTED, "debug timing: single-GPU plans only");
  float m = 0.f;
  if (which >= 4 && (which > 6 || !line_supported(p->g) || p->g.dim < 2))
    return fail(p, EXPD_ERR_UNSUPPORTED, "debug: no line kernel for this geometry");
  if (which != 3) {
    CUDA_TRY(p, dst_debug_time(p->g, dst_tables(p), which, p->Uh, p->T1, nslices, p->prob.npoly, p->prob.q, reps, &m,
                               p->stream));
  } else {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    TimeArgs a = time_args(p, p->Uh, p->Uh, true);
    CUDA_TRY(p, launch_time_fused(a, RM_RESID, OUT_UPDATE, p->k1, p->time_grid, p->stream));
    cudaEventRecord(e0, p->stream);
    for (int i = 0; i < reps; ++i) CUDA_TRY(p, launch_time_fused(a, RM_RESID, OUT_UPDATE, p->k1, p->time_grid, p->stream));
    cudaEventRecord(e1, p->stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&m, e0, e1);
    m /= reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  *ms = m;
  return EXPD_OK;
}

extern "C" int expd_sweep_kernel_launches(const expd_plan* p) {
  if (!p) return 0;
  int k = 2;  // fused time pass + norm reduction
  if (p->nl) k += nonlin_kernel_launches(p->g, p->prob.nt - 1 + p->nshift, !p->dist);
  return k;
}

// ---------------------------------------------------------------------------------------
// solvers
// ---------------------------------------------------------------------------------------
static void fill_report(expd_report* r, int its, int sweeps, int conv, const std::vector<double>& hist,
                        double secs) {
  if (!r) return;
  r->iterations = its;
  r->sweeps = sweeps;
  r->converged = conv;
  r->rel_residual = hist.empty() ? 0.0 : hist.back();
  r->seconds = secs;
  r->hist_len = (int)hist.size();
  if (r->hist)
    for (size_t i = 0; i < hist.size(); ++i) r->hist[i] = hist[i];
}

// ---------------------------------------------------------------------------------------
// solver I/O with host buffers: u0 / U may be host pointers (pinned or pageable) on a
// single-GPU plan.  u0 is staged to the device; the initial guess (unless zero_guess) is
// copied into T1 and transformed from there; the solution's inverse DST runs chunk by chunk
// into T1 while the previous chunk streams to the host on a copy stream.
// ---------------------------------------------------------------------------------------
static bool is_host_ptr(const void* ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return true;  // unknown to CUDA: pageable host memory
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

struct SolveIO {
  bool host_u0 = false, host_U = false;
  const double* u0 = nullptr;  // device u0 (staged if host)
  const double* Uin = nullptr; // device initial guess (T1 if host), nullptr if zero_guess
};

static expd_status solve_in(expd_plan* p, const double* u0, const double* U, SolveIO& io) {
  io.host_u0 = is_host_ptr(u0);
  io.host_U = is_host_ptr(U);
  io.u0 = u0;
  io.Uin = U;
  if ((io.host_u0 || io.host_U) && p->dist)
    return fail(p, EXPD_ERR_INVALID_ARG, "host u0 / U: single-GPU plans only (distributed: device buffers)");
  const size_t slice = sizeof(double) * (size_t)p->g.N * (p->cx ? 2 : 1);
  if (io.host_u0) {
    CUDA_TRY(p, cudaMemcpyAsync(p->hstage, u0, slice, cudaMemcpyHostToDevice, p->stream));
    io.u0 = p->hstage;
  }
  if (p->zero_guess) {
    io.Uin = nullptr;
  } else if (io.host_U) {
    CUDA_TRY(p, cudaMemcpyAsync(p->T1, U, slice * p->prob.nt, cudaMemcpyHostToDevice, p->stream));
    io.Uin = p->T1;
  }
  return EXPD_OK;
}

// U = V U-hat into the caller's U: device pointer -> expd_store_state; host pointer -> the
// inverse DST of slice chunks into T1, each chunk copied out on copy_stream as soon as it is
// done (the copy of chunk c overlaps the transform of chunk c + 1).  Synchronises.
static expd_status solve_out(expd_plan* p, double* U, const SolveIO& io) {
  if (!io.host_U) {
    expd_status s = expd_store_state(p, U);
    if (s) return s;
    CUDA_TRY(p, cudaStreamSynchronize(p->stream));
    return EXPD_OK;
  }
  const long nt = p->prob.nt;
  const long per = (long)p->g.N * (p->cx ? 2 : 1);  // doubles per physical slice
  const int nch = nt >= 8 ? 8 : (int)nt;
  const long ck = (nt + nch - 1) / nch;
  if (!p->copy_stream) CUDA_TRY(p, cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  while ((int)p->cev.size() < nch + 1) {
    cudaEvent_t e;
    CUDA_TRY(p, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->cev.push_back(e);
  }
  int c = 0;
  for (long t0 = 0; t0 < nt; t0 += ck, ++c) {
    const long ns = nt - t0 < ck ? nt - t0 : ck;
    double* dst = p->T1 + t0 * per;
    if (p->cx) {
      expd_status s = cx_mode_to_phys(p, p->Uh + t0 * p->mlen, dst, ns);
      if (s) return s;
    } else {
      CUDA_TRY(p, dst_slices(p->g, dst_tables(p), p->Uh + t0 * p->mlen, true, dst, false, ns, p->scratch, p->stream));
    }
    CUDA_TRY(p, cudaEventRecord(p->cev[c], p->stream));
    CUDA_TRY(p, cudaStreamWaitEvent(p->copy_stream, p->cev[c], 0));
    CUDA_TRY(p, cudaMemcpyAsync(U + t0 * per, dst, sizeof(double) * ns * per, cudaMemcpyDeviceToHost, p->copy_stream));
  }
  CUDA_TRY(p, cudaEventRecord(p->cev[nch], p->copy_stream));
  CUDA_TRY(p, cudaStreamWaitEvent(p->stream, p->cev[nch], 0));  // later work on the plan stream follows
  CUDA_TRY(p, cudaStreamSynchronize(p->copy_stream));
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));
  return EXPD_OK;
}

extern "C" expd_status expd_set_zero_guess(expd_plan* p, int on) {
  if (!p) return EXPD_ERR_INVALID_ARG;
  p->zero_guess = on != 0;
  return EXPD_OK;
}

// The device-side fixed-point loop (single-GPU plans): one CUDA graph holding a WHILE
// conditional node whose body is the captured sweep (stage 3, K1, the norm reduction) and
// k_fp_conv, which records rho_k and sets the loop condition -- the iteration runs without a
// host round trip per sweep; the host reads the loop state once at the end.
static bool device_loop_enabled() {
  const char* s = getenv("EXPD_DEVICE_LOOP");
  return !(s && s[0] == '0');
}

static expd_status build_loop_graph(expd_plan* p) {
  if (!p->cap_stream) CUDA_TRY(p, cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  CUDA_TRY(p, cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp{};
  cudaGraphNode_t node;
  if (e == cudaSuccess) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  }
  if (e == cudaSuccess) {
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(p->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      const bool prof = p->prof;
      p->prof = false;  // no event records inside the conditional body
      p->capturing = true;
      cudaError_t e1;
      {
        LineSkipScope skip(&p->loopst->s3skip);  // stage 3 of the first sweep of a zero-guess solve
        e1 = enqueue_sweep(p, p->cap_stream);
      }
      if (e1 == cudaSuccess) e1 = launch_fp_conv(h, p->loopst, p->dscal, p->cap_stream);
      p->capturing = false;
      p->prof = prof;
      cudaError_t e2 = cudaStreamEndCapture(p->cap_stream, &body);
      e = e1 != cudaSuccess ? e1 : e2;
    }
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&p->loop_exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    p->loop_exec = nullptr;
    return fail(p, EXPD_ERR_CUDA, std::string("device loop graph: ") + cudaGetErrorString(e));
  }
  return EXPD_OK;
}

// N-hat of every slice stage 3 writes, zeroed: the first sweep from U-hat = 0 with N(0) = 0
static cudaError_t zero_stage3_nhat(expd_plan* p) {
  return cudaMemsetAsync(p->Nh + p->g.npad, 0, sizeof(double) * (size_t)(p->prob.nt - 1 + p->nshift) * p->g.npad,
                         p->stream);
}

static expd_status fixed_point_device_loop(expd_plan* p, double tol, int maxit, expd_report* report, bool skip0) {
  if (!p->h_loopst) CUDA_TRY(p, cudaMallocHost(&p->h_loopst, sizeof(FpLoopState)));
  if (!p->loop_exec) {
    expd_status s = build_loop_graph(p);
    if (s) return s;
  }
  FpLoopState* hs = p->h_loopst;
  hs->k = 0;
  hs->status = -1;
  hs->maxit = maxit;
  hs->r0 = 0.0;
  hs->tol = tol;
  hs->s3skip = skip0 ? 1 : 0;
  if (skip0) CUDA_TRY(p, zero_stage3_nhat(p));
  CUDA_TRY(p, cudaMemcpyAsync(p->loopst, hs, offsetof(FpLoopState, hist), cudaMemcpyHostToDevice, p->stream));
  auto t0 = std::chrono::steady_clock::now();
  CUDA_TRY(p, cudaGraphLaunch(p->loop_exec, p->stream));
  CUDA_TRY(p, cudaMemcpyAsync(hs, p->loopst, sizeof(FpLoopState), cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const int k = hs->k;
  std::vector<double> hist(hs->hist, hs->hist + k + 1);
  if (hs->status == 6) {
    fill_report(report, k, k + 1, 0, hist, 0.0);
    return fail(p, EXPD_ERR_BREAKDOWN, "non-finite residual norm");
  }
  if (hs->status != 0 && hs->status != 7)
    return fail(p, EXPD_ERR_CUDA, "device loop ended without a verdict");
  const int conv = hs->status == 0;
  fill_report(report, conv ? k : maxit, conv ? k + 1 : maxit + 1, conv, hist, secs);
  return conv ? EXPD_OK : EXPD_ERR_NOT_CONVERGED;
}

extern "C" expd_status expd_fixed_point_solve(expd_plan* p, const double* u0, double* U, double tol, int maxit,
                                              expd_report* report) {
  expd_status s = ready(p);
  if (s) return s;
  if (!u0 || !U || maxit < 0 || !(tol >= 0.0)) return fail(p, EXPD_ERR_INVALID_ARG, "fixed_point: bad args");
  SolveIO io;
  if ((s = solve_in(p, u0, U, io))) return s;
  s = expd_load_state(p, io.u0, io.Uin);
  if (s) return s;
  // From U-hat = 0 (the zero guess: expd_load_state zeroed it) and N(0) = 0, stage 3 of the
  // first sweep would compute N-hat = V N(V 0) = 0 exactly: it is skipped and N-hat zeroed
  // (bitwise the same iterates; EXPD_S3_SKIP0=0 disables, read per solve)
  const bool skip0 = p->nl && !p->dist && !io.Uin && !(p->prob.npoly > 0 && p->prob.q[0] != 0.0) && s3_skip0_enabled();
  if (!p->dist && graphs_enabled() && device_loop_enabled() && !p->loop_failed && maxit < kFpLoopHist) {
    if (!p->loop_exec && build_loop_graph(p) != EXPD_OK) {
      p->loop_failed = true;  // no conditional-node support: the host-driven loop below
      if (getenv("EXPD_DEBUG")) fprintf(stderr, "expd: %s; host loop\n", p->err.c_str());
      cudaGetLastError();
    }
  }
  if (!p->dist && graphs_enabled() && device_loop_enabled() && !p->loop_failed && maxit < kFpLoopHist) {
    s = fixed_point_device_loop(p, tol, maxit, report, skip0);
    if (s && s != EXPD_ERR_NOT_CONVERGED) return s;
    expd_status s2 = solve_out(p, U, io);
    return s2 ? s2 : s;
  }
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));
  const bool graphs = graphs_enabled();
  std::vector<double> hist;
  double r0 = 0.0;
  int k = 0, conv = 0;
  auto t0 = std::chrono::steady_clock::now();
  for (k = 0; k <= maxit; ++k) {
    if (k == 0 && skip0) {  // the first sweep without stage 3 (see skip0)
      CUDA_TRY(p, zero_stage3_nhat(p));
      CUDA_TRY(p, enqueue_k1(p, p->stream));
    } else {
      s = sweep(p, graphs);  // the first sweep of a plan runs eagerly, then the captured graph
      if (s) return s;
    }
    double rn2;
    s = read_scalars(p, 1, &rn2);
    if (s) return s;
    if (!std::isfinite(rn2)) {
      fill_report(report, k, k + 1, 0, hist, 0.0);
      return fail(p, EXPD_ERR_BREAKDOWN, "non-finite residual norm");
    }
    double rn = std::sqrt(rn2);
    if (k == 0) r0 = rn;
    double rho = r0 > 0.0 ? rn / r0 : 0.0;
    hist.push_back(rho);
    if (rho < tol) {
      conv = 1;
      break;
    }
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  int its = conv ? k : maxit;
  fill_report(report, its, conv ? k + 1 : maxit + 1, conv, hist, secs);
  s = solve_out(p, U, io);
  if (s) return s;
  return conv ? EXPD_OK : EXPD_ERR_NOT_CONVERGED;
}

// Scalar traits of the GMRES driver: real plans (double) and complex plans (GMRES over C with
// the Hermitian inner product, reading R18); K = doubles per coefficient on the device.
template <class T>
struct Scal;
template <>
struct Scal<double> {
  static constexpr int K = 1;
  static double conj(double x) { return x; }
  static double abs(double x) { return std::fabs(x); }
  static double get(const double* p) { return p[0]; }
  static void put(double* p, double v) { p[0] = v; }
  // Givens rotation zeroing b (real, >= 0) under a: returns the new diagonal entry
  static double givens(double a, double b, double& cs, double& sn) {
    const double den = std::sqrt(a * a + b * b);
    cs = den > 0.0 ? a / den : 1.0;
    sn = den > 0.0 ? b / den : 0.0;
    return den;
  }
};
template <>
struct Scal<std::complex<double>> {
  using C = std::complex<double>;
  static constexpr int K = 2;
  static C conj(C x) { return std::conj(x); }
  static double abs(C x) { return std::abs(x); }
  static C get(const double* p) { return C(p[0], p[1]); }
  static void put(double* p, C v) {
    p[0] = v.real();
    p[1] = v.imag();
  }
  // complex Givens [c s; -conj(s) c], c real: (a, b) -> (c a + s b, 0)
  static C givens(C a, double b, double& cs, C& sn) {
    const double aa = std::abs(a), den = std::sqrt(aa * aa + b * b);
    if (den == 0.0) {
      cs = 1.0;
      sn = 0.0;
    } else if (aa == 0.0) {
      cs = 0.0;
      sn = 1.0;
    } else {
      cs = aa / den;
      sn = (a / aa) * (b / den);
    }
    return cs * a + sn * b;
  }
};

template <class T>
static expd_status gmres_impl(expd_plan* p, const double* u0, double* U, double tol, int restart, int maxit,
                              expd_report* report) {
  using SC = Scal<T>;
  constexpr int K = SC::K;
  constexpr bool CX = K == 2;
  expd_status s;
  if (restart > p->krylov_cap)
    return fail(p, EXPD_ERR_OOM, "GMRES restart exceeds the Krylov vectors in the workspace");
  const int m = restart;
  const long len = (long)p->prob.nt * p->mlen;  // this rank's mode slab of a space-time vector
  const size_t vstride = align_up(sizeof(double) * (size_t)len) / sizeof(double);
  auto Vk = [&](int i) { return p->krylov + (size_t)i * vstride; };
  SolveIO io;
  if ((s = solve_in(p, u0, U, io))) return s;
  s = expd_load_state(p, io.u0, io.Uin);
  if (s) return s;
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));
  std::vector<double> hist{1.0};
  p->kstep_ms.clear();
  std::vector<T> H((size_t)(m + 1) * m), sn(m), gv(m + 1), y(m);
  std::vector<double> cs(m);
  std::vector<const double*> Vp(m + 1);
  double beta0 = -1.0;
  int its = 0, conv = 0;
  double* dcoef = p->dscal + 128;  // device coefficient scratch: h [0, 40K), h2 [40K, 80K), ||w||^2 at 80K
  const int O2 = 40 * K, O3 = 80 * K;
  auto t0 = std::chrono::steady_clock::now();
  while (its < maxit) {
    // z = Q_alpha^{-1}(f - Q x)  [K1: residual -> precondition], beta = ||z||
    TimeArgs a = time_args(p, p->Uh, p->T1, false);
    CUDA_TRY(p, launch_time_fused(a, RM_RESID, OUT_S, p->k1, p->time_grid, p->stream));
    const double* t1c = p->T1;
    CUDA_TRY(p, multi_dot(&t1c, 1, p->T1, len, p->partial, p->vgrid, p->dscal, p->stream));
    if ((s = allreduce(p, p->dscal, 1))) return s;
    double b2;
    s = read_scalars(p, 1, &b2);
    if (s) return s;
    double beta = std::sqrt(b2);
    if (beta0 < 0.0) beta0 = beta;
    if (beta0 == 0.0 || beta / beta0 < tol) {
      conv = 1;
      break;
    }
    CUDA_TRY(p, scale_copy(p->T1, 1.0 / beta, Vk(0), len, p->stream));
    std::fill(gv.begin(), gv.end(), T(0.0));
    gv[0] = beta;
    int j = 0, done = 0;
    for (j = 0; j < m && its < maxit; ++j) {
      for (int i = 0; i <= j; ++i) Vp[i] = Vk(i);
      if (p->prof) CUDA_TRY(p, cudaEventRecord(p->kev[0], p->stream));
      TimeArgs q = time_args(p, Vk(j), p->T1, false);
      CUDA_TRY(p, launch_time_fused(q, RM_QOP, OUT_S, p->k1, p->time_grid, p->stream));  // w = P Q v_j
      // CGS2: h = V^H w ; w -= V h ; h2 = V^H w ; w -= V h2 ; ||w||^2
      // (distributed: every partial inner product is completed by an allreduce before use)
      CUDA_TRY(p, multi_dot(Vp.data(), j + 1, p->T1, len, p->partial, p->vgrid, dcoef, p->stream, CX));
      if ((s = allreduce(p, dcoef, K * (j + 1)))) return s;
      CUDA_TRY(p, multi_axpy_dot(Vp.data(), j + 1, dcoef, p->T1, len, p->partial, p->vgrid, dcoef + O2, 1,
                                 p->stream, CX));
      if ((s = allreduce(p, dcoef + O2, K * (j + 1)))) return s;
      CUDA_TRY(p, multi_axpy_dot(Vp.data(), j + 1, dcoef + O2, p->T1, len, p->partial, p->vgrid, dcoef + O3, 2,
                                 p->stream, CX));
      if ((s = allreduce(p, dcoef + O3, 1))) return s;
      if (p->prof) CUDA_TRY(p, cudaEventRecord(p->kev[1], p->stream));
      CUDA_TRY(p, cudaMemcpyAsync(p->h_pin, dcoef, sizeof(double) * (O3 + 1), cudaMemcpyDeviceToHost, p->stream));
      CUDA_TRY(p, cudaStreamSynchronize(p->stream));
      if (p->prof) {
        float km = 0.f;
        CUDA_TRY(p, cudaEventElapsedTime(&km, p->kev[0], p->kev[1]));
        p->kstep_ms.push_back(km);
      }
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = SC::get(p->h_pin + K * i) + SC::get(p->h_pin + O2 + K * i);
      double hn = std::sqrt(p->h_pin[O3]);
      for (int i = 0; i < j; ++i) {
        T a0 = H[(size_t)i * m + j], b0 = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a0 + sn[i] * b0;
        H[(size_t)(i + 1) * m + j] = -SC::conj(sn[i]) * a0 + cs[i] * b0;
      }
      H[(size_t)j * m + j] = SC::givens(H[(size_t)j * m + j], hn, cs[j], sn[j]);
      gv[j + 1] = -SC::conj(sn[j]) * gv[j];
      gv[j] = cs[j] * gv[j];
      ++its;
      double rel = SC::abs(gv[j + 1]) / beta0;
      hist.push_back(rel);
      if (rel < tol || hn == 0.0) {
        done = 1;
        ++j;
        break;
      }
      if (j + 1 < m) CUDA_TRY(p, scale_copy(p->T1, 1.0 / hn, Vk(j + 1), len, p->stream));
    }
    for (int i = j - 1; i >= 0; --i) {
      T sacc = gv[i];
      for (int l = i + 1; l < j; ++l) sacc -= H[(size_t)i * m + l] * y[l];
      y[i] = sacc / H[(size_t)i * m + i];
    }
    for (int i = 0; i < j; ++i) {
      Vp[i] = Vk(i);
      SC::put(p->h_pin + K * i, y[i]);
    }
    CUDA_TRY(p, cudaMemcpyAsync(dcoef, p->h_pin, sizeof(double) * K * j, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(p, lincomb_add(Vp.data(), j, dcoef, p->Uh, len, p->stream, CX));
    CUDA_TRY(p, cudaStreamSynchronize(p->stream));
    if (done) {
      conv = 1;
      break;
    }
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  fill_report(report, its, its, conv, hist, secs);
  s = solve_out(p, U, io);
  if (s) return s;
  return conv ? EXPD_OK : EXPD_ERR_NOT_CONVERGED;
}

extern "C" expd_status expd_gmres_solve(expd_plan* p, const double* u0, double* U, double tol, int restart,
                                        int maxit, expd_report* report) {
  expd_status s = ready(p);
  if (s) return s;
  if (!u0 || !U || maxit < 0 || restart < 1 || !(tol >= 0.0)) return fail(p, EXPD_ERR_INVALID_ARG, "gmres: bad args");
  if (p->nl) return fail(p, EXPD_ERR_UNSUPPORTED, "GMRES is for linear problems (npoly == 0)");
  if (p->krylov_cap < 1) return fail(p, EXPD_ERR_OOM, "workspace holds no Krylov vectors");
  if (p->cx) return gmres_impl<std::complex<double>>(p, u0, U, tol, restart, maxit, report);
  return gmres_impl<double>(p, u0, U, tol, restart, maxit, report);
}

// ---------------------------------------------------------------------------------------
// left-preconditioned BiCGStab (reading R17, van der Vorst's steps
// with the half-step test): the operator B v = Q_alpha^{-1} Q v is one K1 pass (RM_QOP); the
// inner products are multi-dot partials (allreduced when distributed) read to the host.
// ---------------------------------------------------------------------------------------
template <class T>
static expd_status bicgstab_impl(expd_plan* p, const double* u0, double* U, double tol, int maxit,
                                 expd_report* report) {
  using SC = Scal<T>;
  constexpr int K = SC::K;
  constexpr bool CX = K == 2;
  expd_status s;
  const long len = (long)p->prob.nt * p->mlen;
  const size_t vstride = align_up(sizeof(double) * (size_t)len) / sizeof(double);
  double* r = p->krylov;
  double* rh = r + vstride;
  double* pv = rh + vstride;
  double* v = pv + vstride;
  double* sv = v + vstride;
  double* t = sv + vstride;
  double* x = p->Uh;
  double* dcoef = p->dscal + 128;
  SolveIO io;
  if ((s = solve_in(p, u0, U, io))) return s;
  s = expd_load_state(p, io.u0, io.Uin);
  if (s) return s;
  // <a, b> (Hermitian for complex plans) and ||a||^2, completed by allreduce, read to the host
  auto dot = [&](const double* a, const double* b, T* out) -> expd_status {
    CUDA_TRY(p, multi_dot(&a, 1, b, len, p->partial, p->vgrid, p->dscal, p->stream, CX));
    expd_status e = allreduce(p, p->dscal, K);
    if (e) return e;
    double h[2];
    if ((e = read_scalars(p, K, h))) return e;
    *out = SC::get(h);
    return EXPD_OK;
  };
  auto nrm2 = [&](const double* a, double* out) -> expd_status {
    CUDA_TRY(p, multi_dot(&a, 1, a, len, p->partial, p->vgrid, p->dscal, p->stream));
    expd_status e = allreduce(p, p->dscal, 1);
    if (e) return e;
    return read_scalars(p, 1, out);
  };
  auto bop = [&](const double* in, double* out) -> expd_status {  // out = Q_alpha^{-1} Q in
    TimeArgs q = time_args(p, in, out, false);
    CUDA_TRY(p, launch_time_fused(q, RM_QOP, OUT_S, p->k1, p->time_grid, p->stream));
    return EXPD_OK;
  };
  // out += sum_i c_i V_i (coefficients staged through pinned host memory)
  auto axpy = [&](double* out, std::initializer_list<const double*> V, std::initializer_list<T> c) -> expd_status {
    std::vector<const double*> vp(V);
    std::vector<T> cv(c);
    CUDA_TRY(p, cudaStreamSynchronize(p->stream));  // h_pin may still feed an earlier copy
    for (size_t i = 0; i < cv.size(); ++i) SC::put(p->h_pin + K * i, cv[i]);
    CUDA_TRY(p, cudaMemcpyAsync(dcoef, p->h_pin, sizeof(double) * K * cv.size(), cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(p, lincomb_add(vp.data(), (int)vp.size(), dcoef, out, len, p->stream, CX));
    return EXPD_OK;
  };
  // y = c y (a complex c scales the interleaved (re, im) pairs)
  auto scale = [&](double* y, T c) -> expd_status {
    if constexpr (CX) {
      CUDA_TRY(p, scale_copy_cx(y, c.real(), c.imag(), y, len, p->stream));
    } else {
      CUDA_TRY(p, scale_copy(y, c, y, len, p->stream));
    }
    return EXPD_OK;
  };
  CUDA_TRY(p, cudaMemsetAsync(pv, 0, sizeof(double) * len, p->stream));
  CUDA_TRY(p, cudaMemsetAsync(v, 0, sizeof(double) * len, p->stream));
  {  // r_0 = Q_alpha^{-1}(f - Q x_0), r-hat = r_0
    TimeArgs a0 = time_args(p, x, r, false);
    CUDA_TRY(p, launch_time_fused(a0, RM_RESID, OUT_S, p->k1, p->time_grid, p->stream));
    CUDA_TRY(p, scale_copy(r, 1.0, rh, len, p->stream));
  }
  double b2;
  if ((s = nrm2(r, &b2))) return s;
  const double beta0 = std::sqrt(b2);
  std::vector<double> hist{1.0};
  int its = 0, conv = beta0 == 0.0 ? 1 : 0;
  T rho_prev = 1.0, al = 1.0, om = 1.0;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; !conv && i < maxit; ++i) {
    T rho, rv, ts;
    double tt, sn2, rn2;
    if ((s = dot(rh, r, &rho))) return s;
    const T beta = (rho / rho_prev) * (al / om);
    // p = r + beta (p - om v) = beta p + r - beta om v
    if ((s = scale(pv, beta))) return s;
    if ((s = axpy(pv, {r, v}, {T(1.0), -beta * om}))) return s;
    if ((s = bop(pv, v))) return s;
    if ((s = dot(rh, v, &rv))) return s;
    al = rho / rv;
    CUDA_TRY(p, scale_copy(r, 1.0, sv, len, p->stream));  // s = r - al v
    if ((s = axpy(sv, {v}, {-al}))) return s;
    if ((s = nrm2(sv, &sn2))) return s;
    if (std::sqrt(sn2) / beta0 < tol) {  // half step
      if ((s = axpy(x, {pv}, {al}))) return s;
      its = i + 1;
      hist.push_back(std::sqrt(sn2) / beta0);
      conv = 1;
      break;
    }
    if ((s = bop(sv, t))) return s;
    if ((s = dot(t, sv, &ts))) return s;
    if ((s = nrm2(t, &tt))) return s;
    om = ts / tt;
    if ((s = axpy(x, {pv, sv}, {al, om}))) return s;
    CUDA_TRY(p, scale_copy(sv, 1.0, r, len, p->stream));  // r = s - om t
    if ((s = axpy(r, {t}, {-om}))) return s;
    rho_prev = rho;
    its = i + 1;
    if ((s = nrm2(r, &rn2))) return s;
    hist.push_back(std::sqrt(rn2) / beta0);
    if (hist.back() < tol) conv = 1;
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  fill_report(report, its, 2 * its + 1, conv, hist, secs);
  s = solve_out(p, U, io);
  if (s) return s;
  return conv ? EXPD_OK : EXPD_ERR_NOT_CONVERGED;
}

extern "C" expd_status expd_bicgstab_solve(expd_plan* p, const double* u0, double* U, double tol, int maxit,
                                           expd_report* report) {
  expd_status s = ready(p);
  if (s) return s;
  if (!u0 || !U || maxit < 0 || !(tol >= 0.0)) return fail(p, EXPD_ERR_INVALID_ARG, "bicgstab: bad args");
  if (p->nl) return fail(p, EXPD_ERR_UNSUPPORTED, "BiCGStab is for linear problems (npoly == 0)");
  if (p->krylov_cap < 6) return fail(p, EXPD_ERR_OOM, "BiCGStab needs 6 work vectors in the workspace");
  if (p->cx) return bicgstab_impl<std::complex<double>>(p, u0, U, tol, maxit, report);
  return bicgstab_impl<double>(p, u0, U, tol, maxit, report);
}

// ---------------------------------------------------------------------------------------
// Peer stores of the distributed stage 3 (include/expd.h "Multi-GPU")
// ---------------------------------------------------------------------------------------
typedef CUresult (*PFN_addr_range)(CUdeviceptr*, size_t*, CUdeviceptr);

extern "C" expd_status expd_plan_slab_ipc_handle(expd_plan* p, unsigned char handle[64], long* nhat_offset,
                                                 long* uhat_offset) {
  expd_status s = ready(p);
  if (s) return s;
  if (!handle || !nhat_offset || !uhat_offset) return fail(p, EXPD_ERR_INVALID_ARG, "slab_ipc_handle: bad args");
  if (!p->dist || !p->Nh) return fail(p, EXPD_ERR_UNSUPPORTED, "slab_ipc_handle: distributed nonlinear plans only");
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    return fail(p, EXPD_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (((PFN_addr_range)fn)(&base, &size, (CUdeviceptr)p->Nh) != CUDA_SUCCESS)
    return fail(p, EXPD_ERR_CUDA, "cuMemGetAddressRange failed");
  if ((CUdeviceptr)p->Uh < base || (CUdeviceptr)p->Uh >= base + size)
    return fail(p, EXPD_ERR_UNSUPPORTED, "slab_ipc_handle: U-hat and N-hat in different allocations");
  cudaIpcMemHandle_t h;
  CUDA_TRY(p, cudaIpcGetMemHandle(&h, (void*)base));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  memcpy(handle, &h, 64);
  *nhat_offset = (long)((CUdeviceptr)p->Nh - base);
  *uhat_offset = (long)((CUdeviceptr)p->Uh - base);
  return EXPD_OK;
}

extern "C" expd_status expd_plan_set_peer_slabs(expd_plan* p, int rank, const unsigned char handle[64],
                                                long nhat_offset, long uhat_offset) {
  expd_status s = ready(p);
  if (s) return s;
  if (!p->dist || !p->Nh || rank < 0 || rank >= p->L.nranks || p->L.nranks > kMaxPeers || !handle ||
      nhat_offset < 0 || uhat_offset < 0)
    return fail(p, EXPD_ERR_INVALID_ARG, "set_peer_slabs: bad args");
  if ((int)p->peer_nh.size() != p->L.nranks) {
    p->peer_nh.assign(p->L.nranks, nullptr);
    p->peer_uh.assign(p->L.nranks, nullptr);
  }
  if (rank == p->L.rank) {
    p->peer_nh[rank] = p->Nh;
    p->peer_uh[rank] = p->Uh;
    return EXPD_OK;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  void* base = nullptr;
  CUDA_TRY(p, cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  p->peer_ipc.push_back(base);
  p->peer_nh[rank] = reinterpret_cast<double*>(static_cast<char*>(base) + nhat_offset);
  p->peer_uh[rank] = reinterpret_cast<double*>(static_cast<char*>(base) + uhat_offset);
  return EXPD_OK;
}

extern "C" expd_status expd_plan_enable_peer_stores(expd_plan* p, int on) {
  expd_status s = ready(p);
  if (s) return s;
  if (!on) {
    p->peer_on = false;
    return EXPD_OK;
  }
  if (!p->dist || !p->nl || p->cx || p->g.dim < 2 || !line_supported(p->g))
    return fail(p, EXPD_ERR_UNSUPPORTED, "peer stores: distributed nonlinear real plans, dim >= 2, n + 1 >= 256");
  if ((int)p->peer_nh.size() != p->L.nranks) return fail(p, EXPD_ERR_INVALID_ARG, "peer stores: peers not set");
  PeerMaps h[2]{};  // [0] N-hat slabs (stores, the swizzled result layout), [1] U-hat slabs (loads)
  for (int k = 0; k < 2; ++k) h[k].nranks = p->L.nranks;
  for (int q = 0; q < p->L.nranks; ++q) {
    if (!p->peer_nh[q] || !p->peer_uh[q])
      return fail(p, EXPD_ERR_INVALID_ARG, "peer stores: peer " + std::to_string(q) + " not set");
    const long M = p->g.M;
    if (p->L.mode_off[q] % M || p->L.mode_len[q] % M)
      return fail(p, EXPD_ERR_UNSUPPORTED, "peer stores: mode slabs are not whole x-lines");
    for (int k = 0; k < 2; ++k) {
      h[k].unit_off[q] = (int)(p->L.mode_off[q] / M);
      h[k].units[q] = (int)(p->L.mode_len[q] / M);
    }
    CUDA_TRY(p, peer_slab_map(&h[0].m[q], p->g, p->peer_nh[q], h[0].units[q], p->prob.nt + 1, p->L.mode_len[q],
                              true));
    CUDA_TRY(p, peer_slab_map(&h[1].m[q], p->g, p->peer_uh[q], h[1].units[q], p->prob.nt, p->L.mode_len[q], false));
  }
  if (!p->d_peer) CUDA_TRY(p, cudaMalloc(&p->d_peer, 2 * sizeof(PeerMaps)));
  CUDA_TRY(p, cudaMemcpyAsync(p->d_peer, h, 2 * sizeof(PeerMaps), cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY(p, cudaStreamSynchronize(p->stream));
  p->peer_on = true;
  return EXPD_OK;
}
