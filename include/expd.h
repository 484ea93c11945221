/*
 * expd.h -- C-ABI of the B200-native Exp-ParaDiag hot path (libexpd.so).
 *
 * Method: Garai & Chamakuri, "Exp-ParaDiag: Time-Parallel Exponential Integrators for
 * Parabolic PDEs", arXiv 2603.04350.  Citations are PAPER.md line numbers (the paper's
 * LaTeX source) with the equation / step; "R<k>" are the readings listed in DESIGN.md.
 *
 * Problem: u_t = (a Delta - c) u + N(u) on (0,1)^dim,
 * homogeneous Dirichlet, n interior points per axis (h = 1/(n+1)), second-order finite
 * differences, N_t steps of size dt, alpha-circulant parameter alpha.
 *
 * Conventions for every entry point:
 *   - every call returns expd_status; nothing else crosses the ABI (no exceptions);
 *   - on any error the output buffers are left untouched when the error is detected
 *     before launch (INVALID_ARG / UNSUPPORTED); later CUDA errors may leave them
 *     partially written;
 *   - expd_plan_last_error() returns a human-readable message for the last failure;
 *   - device pointers must live on the plan's device; all work is enqueued on the
 *     plan's CUDA stream; "blocking" calls synchronise that stream;
 *   - layouts: a physical slice is n^dim doubles, x fastest ([z][y][x]); a space-time
 *     vector is nt_local consecutive slices, slice m-1 holding u_m (PAPER.md:98,
 *     U = (u_1, ..., u_Nt)); u0 is one slice;
 *   - with nranks > 1 every function is collective over the plan's communicator and
 *     must be called by all ranks in the same order with identical problems.
 *
 * Ownership: the caller owns u0, U, R, S and the workspace (e.g. torch tensors passed
 * as data_ptr()).  The plan owns only its small tables (KBs .. tens of MB of per-mode
 * multipliers live in the caller's workspace) and never allocates in a solve loop.
 */
#ifndef EXPD_H
#define EXPD_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EXPD_OK = 0,
  EXPD_ERR_INVALID_ARG = 1,   /* bad sizes, null pointers, alpha <= 0, ...        */
  EXPD_ERR_UNSUPPORTED = 2,   /* valid math, not built (e.g. nt not a power of 2) */
  EXPD_ERR_CUDA = 3,
  EXPD_ERR_NCCL = 4,
  EXPD_ERR_OOM = 5,           /* workspace too small                              */
  EXPD_ERR_BREAKDOWN = 6,     /* |1 - lambda_k E_J| < 1e-14, NaN/Inf residual     */
  EXPD_ERR_NOT_CONVERGED = 7  /* maxit reached; the report is still filled        */
} expd_status;

typedef enum {
  EXPD_EXP_EULER = 0, /* linear (npoly = 0) or ETD1: u_n = E u_{n-1} + dt phi1 N(u_{n-1}) (R5) */
  EXPD_ETD2 = 1,      /* u_n = E u_{n-1} + dt[(phi1+phi2) N_{n-1} - phi2 N_{n-2}] (R6)        */
  EXPD_IF_IMEX = 2,   /* the paper's own: IF scheme (6.1) u_n = E u_{n-1} + dt N(u_n)
                         (PAPER.md:815), solved by the IMEX-type iteration (7.2)/(7.3)
                         (PAPER.md:1209-1220): N of the same slice, lagged one sweep    */
  EXPD_BDF2 = 3       /* exponential BDF2 all-at-once system (4.1)-(4.5),
                         linear problems only (npoly = 0): the nt unknowns of U are
                         u_2 .. u_{nt+1} (u_1 = A u_0, reading R16; T = (nt+1) dt); the
                         preconditioner divides by 1 - 4/3 lambda_k E + 1/3 lambda_k^2 E^2 */
} expd_scheme;

typedef struct {
  int dim;            /* 1, 2 or 3 (Remark 2.2)                       */
  int n;              /* interior points per axis; requires n+1 = 2^m, 4 <= n+1 <= 4096 */
  double a, c;        /* L_h = a Delta_h - c I, a > 0, c >= 0      */
  double dt;          /* Delta t > 0                                                      */
  int nt;             /* N_t: a power of two, 4 <= nt <= 256                              */
  double alpha;       /* 0 < alpha <= 1 (Gamma_alpha singular at 0 -> INVALID_ARG, R10) */
  expd_scheme scheme;
  int npoly;          /* N(u) = sum_{p < npoly} q[p] u^p; 0 = linear; 0 <= npoly <= 8     */
  double q[8];
  double a_im, c_im;  /* imaginary parts of a and c (0 for the real problems above).  Either
                         non-zero makes a COMPLEX plan (the paper's Schroedinger tests, a = i,
                         c = 2i): u_t = (a Delta - c) u with a = a + i a_im,
                         c = c + i c_im, Re a >= 0 (a != 0), Re c >= 0; linear only
                         (npoly = 0), scheme EXPD_EXP_EULER or EXPD_BDF2, one or more
                         GPUs.  Every space-time / slice argument of a complex plan (u0,
                         U, R, S) is complex128: interleaved (re, im) doubles, 2 N doubles
                         per slice.
                         GMRES and BiCGStab run over C with the Hermitian inner product
                         (reading R18); expd_dst / expd_nonlin_hat stay real-only.       */
} expd_problem;

typedef struct {
  int rank, nranks;   /* 1 <= nranks <= 64, nt % nranks == 0                  */
  void* nccl_comm;    /* ncclComm_t (expd_nccl_comm_init), a host communicator
                         (expd_host_comm_create), or NULL when nranks == 1; with
                         nranks == 1 and a communicator the distributed schedule runs on one
                         GPU (all-to-alls become local copies) -- used by the GPU tests     */
} expd_dist;

/* Partition of a space-time vector over the ranks:
   time slab = slices [t0, t0 + nt_local) (physical API vectors U, R, S and stage 3);
   mode slab = padded spectral entries [mode_off, mode_off + mode_len) of every slice
   (the time-local fused kernel K1).  npad = entries of a padded spectral slice
   (n^{dim-1} (n+1)); complex problems count doubles of the interleaved (re, im) slice, so
   npad, mode_off and mode_len are twice the real ones. */
typedef struct {
  int rank, nranks;
  long npad, mode_off, mode_len;
  int t0, nt_local;
} expd_layout;

typedef struct expd_plan expd_plan;

typedef struct {
  int iterations;     /* fixed point: preconditioner updates applied before rho_k < tol
                         (R8); GMRES: Arnoldi matvecs                                   */
  int sweeps;         /* HBM passes of the fused sweep (fixed point: iterations + 1)    */
  int converged;      /* 1 if the tolerance was met                                     */
  int hist_len;       /* entries written to hist                                        */
  double rel_residual;/* last relative residual                                         */
  double seconds;     /* wall time of the iteration loop (excludes setup / final IDST)  */
  double* hist;       /* caller buffer of maxit + 2 doubles, or NULL                    */
} expd_report;

/* Validate the problem and build the plan's tables (per-axis eigenvalues lambda_j,
   twiddles omega^q, Gamma_alpha powers, lambda_k) in long double rounded to double.
   cuda_stream: a cudaStream_t (NULL = legacy default stream).  *out receives the plan. */
expd_status expd_plan_create(const expd_problem* prob, const expd_dist* dist, int device, void* cuda_stream,
                             expd_plan** out);
/* Workspace the caller must provide: the spectral state, nonlinear history, per-mode
   multiplier tables, transform scratch and krylov_vectors GMRES basis vectors
   (0 = fixed point / primitives only).  */
expd_status expd_plan_workspace_bytes(const expd_plan* plan, int krylov_vectors, size_t* bytes);
/* Hand the plan a device buffer of at least the queried size (256-byte aligned).  The
   number of GMRES basis vectors the buffer holds is derived from its size. */
expd_status expd_plan_set_workspace(expd_plan* plan, void* d_ptr, size_t bytes);
void expd_plan_destroy(expd_plan* plan);
const char* expd_plan_last_error(const expd_plan* plan);

/* All-at-once residual R = F(U) - Q U, slice by slice
   R_n = A u_{n-1} + Phi[N] - u_n,  A = exp(dt L_h) (R5, R6).
   u0: [n^dim], U, R: [nt][n^dim] physical, device.  rnorm2_host (nullable): receives
   ||R||_2^2 (the call then synchronises).  Async otherwise.  R must not alias U. */
expd_status expd_residual(expd_plan* plan, const double* u0, const double* U, double* R, double* rnorm2_host);

/* S = Q_alpha^{-1} R by Steps (a)-(c): alpha-scaled time DFT,
   per-frequency spatial solve (I - lambda_k A)^{-1} as DST / divide by (1 - lambda_k E_J)
   / IDST, inverse DFT and unscaling.  R, S: [nt][n^dim] physical, device; S may alias R.
   Async. */
expd_status expd_precond_apply(expd_plan* plan, const double* R, double* S);

/* Solver buffers (expd_fixed_point_solve, expd_gmres_solve, expd_bicgstab_solve): u0 and U
   are device pointers on the plan's device, or -- single-GPU plans -- HOST pointers (pinned
   for asynchronous copies, pageable accepted): u0 and the initial guess are then copied in
   inside the call, and the solution's inverse DST runs chunk by chunk while the finished
   chunks stream to the host, so the copy-out overlaps the transform.  Host buffers on a
   distributed plan: INVALID_ARG. */
/* With on != 0 the solvers (and expd_load_state) ignore the contents of U on entry and start
   from U = 0 (the paper's zero initial guess), skipping the transform (and, for
   host U, the copy) of the guess; U is still written with the solution.  Sticky per plan. */
expd_status expd_set_zero_guess(expd_plan* plan, int on);

/* Preconditioned Richardson / Picard (3.2) from the initial guess in
   U (zeros per PAPER.md:895): sweep k computes r^k = F(U^k) - Q U^k, rho_k =
   ||r^k|| / ||r^0||, U^{k+1} = U^k + Q_alpha^{-1} r^k; stops after the first sweep with
   rho_k < tol (R8), returning U^{k+1} in U.  Blocking.  report (nullable).  On one GPU
   the iteration runs as a CUDA graph with a device-side WHILE loop (the convergence test on
   the device, one synchronisation per solve).  With the zero guess
   (expd_set_zero_guess) and N(0) = 0 (q[0] = 0) the first sweep's stage 3 is skipped: from
   U = 0 it would compute N-hat = V N(0) = 0 exactly, so N-hat is zeroed instead (one-GPU
   plans; bitwise the same iterates; EXPD_S3_SKIP0=0 disables). */
expd_status expd_fixed_point_solve(expd_plan* plan, const double* u0, double* U, double tol, int maxit,
                                   expd_report* report);

/* Left-preconditioned restarted GMRES(restart) on Q_alpha^{-1} Q u = Q_alpha^{-1} f
   (PAPER.md:284-289), classical Gram-Schmidt applied twice (R11), Givens rotations;
   stops when ||Q_alpha^{-1}(f - Q x)|| / ||Q_alpha^{-1}(f - Q x_0)|| < tol.
   Linear problems only (npoly == 0, else UNSUPPORTED).  The workspace must hold >= restart
   Krylov vectors (expd_plan_workspace_bytes(plan, restart)), else EXPD_ERR_OOM.  U: initial
   guess in, solution out.  Blocking. */
expd_status expd_gmres_solve(expd_plan* plan, const double* u0, double* U, double tol, int restart, int maxit,
                             expd_report* report);

/* Left-preconditioned BiCGStab on Q_alpha^{-1} Q u = Q_alpha^{-1} f (PAPER.md:1088-1114,
   the paper's other Krylov method; reading R17): the preconditioned residual is iterated,
   stop when its norm relative to the initial one is < tol (also after the half step).
   Linear problems only; the workspace must hold >= 6 Krylov vectors.  iterations = BiCGStab
   steps (2 fused K1 passes each).  Blocking. */
expd_status expd_bicgstab_solve(expd_plan* plan, const double* u0, double* U, double tol, int maxit,
                                expd_report* report);

/* ---- multi-GPU ---------------------------------------------------------------------- */
/* The rank's slabs; INVALID_ARG when nt % nranks != 0 or there are fewer x-lines than ranks.
   Pure host computation (no device needed). */
expd_status expd_layout_query(const expd_problem* prob, int rank, int nranks, expd_layout* out);
/* The all-to-all schedule between the layouts, as the messages this rank posts, in order:
   direction 0 = mode slab [nt][mode_len] -> time slab [nt_local][npad]; 1 = time slab ->
   mode slab [nt + shift][mode_len] (global slice t lands in slice t + shift).  Each message
   is 4 longs {peer, src_off, dst_off, count} (doubles; src_off of recvs and dst_off of
   sends are 0).  Writes sends / recvs when cap >= the count; returns the number of messages
   per list (sends and recvs have equal length), or -1 on invalid arguments.  Host only. */
long expd_a2a_schedule(const expd_problem* prob, int rank, int nranks, int direction, int shift, long* sends,
                       long* recvs, long cap);
/* The same schedule with stride 4 or 5 longs per message; stride 5 appends the message's
   slice key (the index of its slice within the time slab it belongs to).  The distributed
   sweep pipelines its all-to-alls in chunks of slice keys: every
   rank's slab holds nt / nranks slices, so a key range is one symmetric chunk. */
long expd_a2a_schedule_keyed(const expd_problem* prob, int rank, int nranks, int direction, int shift,
                             long* sends, long* recvs, long cap, int stride);
/* A point-to-point transport for expd_a2a_execute_host: send / recv post one message of
   `count` doubles to / from `peer` (host memory, valid until group_end returns); group_start /
   group_end (nullable) bracket the messages of one all-to-all chunk, and group_end returns
   when all of them are complete.  Each returns 0 on success.  ctx is passed through. */
typedef struct {
  void* ctx;
  int (*group_start)(void* ctx);
  int (*send)(void* ctx, const double* buf, long count, int peer);
  int (*recv)(void* ctx, double* buf, long count, int peer);
  int (*group_end)(void* ctx);
} expd_transport;
/* Executes this rank's all-to-all schedule (direction, shift as expd_a2a_schedule) for the
   slice keys [s_lo, s_hi) on HOST buffers through `transport`: self messages are host
   copies, the others one group of sends then receives in the schedule's order.  It is the
   very routine the distributed sweep runs on the device, where the transport is
   cudaMemcpyAsync + ncclSend / ncclRecv inside ncclGroupStart / ncclGroupEnd -- exposed so
   the message selection, self pairing, ordering and chunking run under a CPU transport
   (tests/test_dist_cpu.py: torch.distributed gloo) without GPUs.  src / dst: the layouts of
   expd_a2a_schedule (doubles).  INVALID_ARG on bad arguments or a schedule mismatch,
   EXPD_ERR_NCCL if the transport fails. */
expd_status expd_a2a_execute_host(const expd_problem* prob, int rank, int nranks, int direction, int shift, int s_lo,
                                  int s_hi, const double* src, double* dst, const expd_transport* transport);
/* NCCL communicator for a plan (NCCL is loaded at run time: the process's libnccl.so.2).
   Rank 0 creates the 128-byte id, the caller broadcasts it (e.g. torch.distributed), every
   rank calls expd_nccl_comm_init (collective).  The caller owns the communicator. */
expd_status expd_nccl_unique_id(unsigned char id[128]);
expd_status expd_nccl_comm_init(const unsigned char id[128], int nranks, int rank, int device, void** comm);
void expd_nccl_comm_destroy(void* comm);
/* A HOST communicator for expd_dist.nccl_comm: the distributed plan's all-to-alls and
   allreduces run through host staging buffers and `transport` (the expd_transport of
   expd_a2a_execute_host, copied; ctx and the callbacks must outlive the communicator)
   instead of NCCL.  Every exchange blocks the calling thread: group_start synchronizes the
   stream, sends are staged device -> host and posted, receives land host -> device after
   group_end.  Allreduces send every rank's partial sums to every other rank and add them
   in rank order (all ranks hold the same bits).  It exists so the multi-rank plan runs
   with several processes on ONE GPU (NCCL refuses two ranks per device) and their kernels
   never wait on one another (tests/test_gpu_multirank.py); NVLink runs use NCCL.
   INVALID_ARG on a null transport / send / recv / comm or a bad rank. */
expd_status expd_host_comm_create(const expd_transport* transport, int rank, int nranks, void** comm);
/* Frees a host communicator (no-op for anything else).  expd_nccl_comm_destroy ignores host
   communicators. */
void expd_host_comm_destroy(void* comm);

/* Peer access (the fused "NVLink-store transposes" of SURVEY §8(f)): a
   distributed nonlinear plan's stage 3 can load every row of its time slab straight from the
   U-hat mode slab of the rank that owns the row and store every row of its result straight
   into the owner's N-hat slab -- another GPU's memory over NVLink, or another process's on the
   same GPU -- instead of two all-to-alls through time-slab staging.  Setup, collective over
   the ranks: every rank exports its slabs (expd_plan_slab_ipc_handle: a CUDA IPC handle of
   the workspace allocation and the two slabs' byte offsets), the caller exchanges them
   (e.g. torch.distributed all_gather), every rank registers every rank's
   (expd_plan_set_peer_slabs; its own rank maps its own slabs), then
   expd_plan_enable_peer_stores(plan, 1) (0 switches back to the all-to-alls).  Requirements:
   real coefficients, npoly > 0, dim >= 2, n + 1 >= 256 (the TMA line kernels), <= 16 ranks,
   mode slabs of whole x-lines.  A new workspace disables it (register again).  UNSUPPORTED /
   INVALID_ARG / EXPD_ERR_CUDA (e.g. a caching allocator without IPC-able segments). */
expd_status expd_plan_slab_ipc_handle(expd_plan* plan, unsigned char handle[64], long* nhat_offset,
                                      long* uhat_offset);
expd_status expd_plan_set_peer_slabs(expd_plan* plan, int rank, const unsigned char handle[64], long nhat_offset,
                                     long uhat_offset);
expd_status expd_plan_enable_peer_stores(expd_plan* plan, int on);

/* ---- lower-level entry points used by the solver loop and the benchmark -------------- */
/* Spectral-state sweep, the hot path of one Exp-ParaDiag iteration on data already in
   the workspace (after expd_load_state): [nonlinear: N-hat of every slice (stage 3)] ->
   fused residual + ||r||^2 + preconditioner + update (stages 1, 2).  Async; the residual
   norm squared of this sweep is left on the device (read by expd_sweep_norm2). */
expd_status expd_load_state(expd_plan* plan, const double* u0, const double* U);
expd_status expd_sweep(expd_plan* plan);
expd_status expd_sweep_norm2(expd_plan* plan, double* rnorm2_host); /* synchronises */
expd_status expd_store_state(expd_plan* plan, double* U);           /* U = V U-hat, async */
/* out = V in for nslices physical slices (the orthonormal DST-I along every axis,
   PAPER.md:141; V = V^T = V^{-1}).  in, out: [nslices][n^dim] device; out may alias in.
   Uses the workspace's transform scratch.  Async. */
expd_status expd_dst(expd_plan* plan, const double* in, double* out, long nslices);
/* nhat = V N(V uhat) for nslices slices of DST coefficients (stage 3 of a Picard sweep,
   BASELINE.json:5; N(u) = sum_p q[p] u^p from the plan's problem).  uhat, nhat:
   [nslices][n^dim] device, mode j_i - 1 along each axis, x fastest; nhat may alias uhat.
   Uses the workspace's spectral temporary and transform scratch.  Async. */
expd_status expd_nonlin_hat(expd_plan* plan, const double* uhat, double* nhat, long nslices);
/* Stage timing of expd_sweep with CUDA events recorded on the plan's stream (inside the
   sweep's CUDA graph): enable = 1 turns it on, 2 also records an event between every
   stage-3 pass (for expd_sweep_pass_ms; ~50 more graph nodes per sweep), 0 off.
   expd_sweep_stage_ms waits for the last sweep and returns the device time of stage 3
   (N-hat of all slices; 0 when linear) and of the fused time-local kernel K1, in ms. */
expd_status expd_set_profiling(expd_plan* plan, int enable);
expd_status expd_sweep_stage_ms(expd_plan* plan, double* ms_nonlin, double* ms_time);
/* Stage-3 pass times of the last sweep (set_profiling level 2, single-GPU nonlinear plans with
   the TMA line kernels): device ms summed over the sweep's x-passes, plain strided passes
   (3-D) and fused strided [V, N(u), V] passes, measured by CUDA events recorded on the
   plan's stream between consecutive passes inside the sweep, and the launch counts.  With
   the persistent stage 3 (one launch carrying all passes, 2-D) the whole stage is reported
   in ms_fused with n_fused = 1 and n_x = 0.
   UNSUPPORTED when no such timing exists.  Diagnostics for bench.py's per-kernel
   rooflines. */
expd_status expd_sweep_pass_ms(expd_plan* plan, double* ms_x, double* ms_strided, double* ms_fused, int* n_x,
                               int* n_strided, int* n_fused);
/* Diagnostics for tuning: average device time (ms, CUDA events) of `reps` back-to-back
   launches of one kernel family on the workspace's spectral state: which = 0 x-axis DST
   pass, 1 strided-axis DST pass, 2 fused strided IDST -> N -> DST pass (each over nslices
   slices, 1 <= nslices <= nt), 3 the fused time-local kernel K1 (whole state), 4 / 5 / 6
   the TMA line kernels (x-axis, strided axis, fused strided [V, N, V]).  The
   workspace contents are overwritten with transformed data. */
expd_status expd_debug_kernel_ms(expd_plan* plan, int which, long nslices, int reps, double* ms);
/* Device time (ms) of every Arnoldi step of the last expd_gmres_solve run with profiling on
   (expd_set_profiling >= 1): CUDA events on the plan's stream before the step's K1 operator
   pass and after its CGS2 / norm kernels (and allreduces), i.e. w = Q_alpha^{-1} Q v_j and the
   orthogonalisation of PAPER.md:284-289, without the host's Givens update.  Writes up to cap
   values to ms (caller-owned host buffer) and the number of steps to *count. */
expd_status expd_solver_step_ms(const expd_plan* plan, double* ms, int cap, int* count);
/* Number of kernels one expd_sweep launches (for the benchmark's launch count). */
int expd_sweep_kernel_launches(const expd_plan* plan);

#ifdef __cplusplus
}
#endif
#endif
