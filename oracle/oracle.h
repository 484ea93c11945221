/*
 * oracle.h -- the plain, slow CPU oracle for the Exp-ParaDiag hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2603_04350_b200/, libexpd.so) never links, loads or calls it, and the
 * two share no code, headers, tables or helpers.
 *
 * Everything is computed from the paper's definitions, written out literally:
 * naive O(n) sine sums per output (no FFT), naive O(Nt^2) DFTs, long-double
 * accumulation, long-double pi and exact integer twiddle indices.  Citations are
 * PAPER.md line numbers (the LaTeX source of arXiv 2603.04350) plus the
 * equation / step they fall in; readings of points the paper leaves open are the
 * DESIGN.md "Readings" table (R1..R14).
 *
 * Layouts: a physical or spectral slice is n^dim doubles, x fastest
 * ([z][y][x]); a space-time vector is nt slices, slice m-1 holding u_m
 * (U = (u_1, ..., u_Nt)).
 */
#ifndef EXPD_ORACLE_H
#define EXPD_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int dim;         /* 1, 2 or 3 (Remark 2.2)                     */
  int n;           /* interior points per axis, h = 1/(n+1), domain (0,1)^dim      */
  double a, c;     /* L_h = a Delta_h - c I                 */
  double dt;       /* Delta t                                       */
  int nt;          /* N_t                                                          */
  double alpha;    /* alpha-circulant parameter                  */
  int scheme;      /* 0: exponential Euler / ETD1, 1: ETD2 (readings R5, R6),      *
                    * 2: IF scheme (6.1) / IMEX-type iteration (7.2), *
                    * 3: exponential BDF2 (4.1)-(4.5), linear only:  *
                    *    nt unknowns u_2..u_{nt+1}, u_1 = A u_0 (reading R16)           */
  int npoly;       /* N(u) = sum_{p<npoly} q[p] u^p ; 0 = linear                   */
  double q[8];
  double a_im, c_im; /* imaginary parts of a and c (oracle_cplx.c only; 0 elsewhere)   */
} orc_problem;

long orc_nmodes(const orc_problem* p);

/* Delta_h eigenvalues of one axis, lam[j-1] = -(4/h^2) sin^2(j pi h / 2), j=1..n (R1). */
void orc_axis_eigs(int n, double* lam);
/* Per spectral mode J (same layout as a slice): mu_J = a sum_i lam_{j_i} - c,
   E_J = exp(dt mu_J), dt*phi1(dt mu_J), dt*phi2(dt mu_J).  Any pointer may be NULL. */
void orc_mode_tables(const orc_problem* p, double* mu, double* E, double* dtphi1, double* dtphi2);

/* Orthonormal DST-I along every axis: out = V in, V = V^T = V^{-1}. */
void orc_dst(const orc_problem* p, const double* in, double* out);
/* Selected entries of V in: out[s] = (V in)[idx[s]]. */
void orc_dst_sample_batch(const orc_problem* p, const double* in, long nslices, const long* idx, int ns,
                          double* out);
void orc_dst_x_rows(const orc_problem* p, const double* in, long nrows, double* out);
void orc_dst_sample(const orc_problem* p, const double* in, const long* idx, int ns, double* out);
/* A v = V diag(E) V v with A = exp(dt L_h). */
void orc_apply_A(const orc_problem* p, const double* v, double* out);
/* Pointwise N(u) = sum_p q_p u^p. */
void orc_nonlin(const orc_problem* p, const double* u, double* out);

/* Sequential time stepping (the fixed point of the all-at-once system):
   linear u_n = A u_{n-1}; ETD1 / ETD2 per readings R5, R6. */
void orc_sequential(const orc_problem* p, const double* u0, double* U);

/* All-at-once residual r = F(U) - Q U (PAPER.md:181-183 for the linear part),
   slice by slice r_n = A u_{n-1} + Phi[N] - u_n.  rnorm2 (nullable) = ||r||_2^2. */
void orc_residual(const orc_problem* p, const double* u0, const double* U, double* R, double* rnorm2);
/* The Q operator alone: (Q v)_n = v_n - A v_{n-1}, v_0 = 0. */
void orc_apply_Q(const orc_problem* p, const double* V, double* out);
/* The alpha-circulant Q_alpha applied: (Q_a v)_1 = v_1 - alpha A v_Nt, (Q_a v)_n = v_n - A v_{n-1}
   (PAPER.md:99-108, :186).  Used by tests as an inverse check. */
void orc_apply_Qalpha(const orc_problem* p, const double* V, double* out);
/* Preconditioner S = Q_alpha^{-1} R by the literal Steps (a)-(c).
   Returns the imaginary leakage max|Im s| / max|Re s|. */
double orc_precond(const orc_problem* p, const double* R, double* S);

/* Fixed-point (Richardson (3.2)) / Picard solve from the given U
   (zeros per PAPER.md:895).  Sweep k: r^k = F(U^k) - Q U^k, rho_k = ||r^k||/||r^0||,
   U^{k+1} = U^k + Q_alpha^{-1} r^k; stop after the first sweep with rho_k < tol.
   iterations = k (updates applied before convergence was detected); U returns U^{k+1}
   (reading R8).  hist[0..k] = rho.  Returns 0 converged, 7 not converged. */
int orc_fixed_point(const orc_problem* p, const double* u0, double* U, double tol, int maxit,
                    double* hist, int* iterations);
/* Left-preconditioned restarted GMRES(m) on Q_alpha^{-1} Q u = Q_alpha^{-1} f
   (PAPER.md:284-289), classical Gram-Schmidt applied twice, Givens rotations.
   Linear problems only.  hist[i] = ||g_{i}|| / ||Q_alpha^{-1}(f - Q U_init)|| after i matvecs.
   iterations = number of Arnoldi matvecs.  Returns 0 converged, 7 not converged,
   2 unsupported (nonlinear problem). */
int orc_gmres(const orc_problem* p, const double* u0, double* U, double tol, int restart, int maxit,
              double* hist, int* iterations);

/* Left-preconditioned BiCGStab on Q_alpha^{-1} Q (reading R17): same
   contract as orc_gmres (hist[k] = relative preconditioned residual after step k). */
int orc_bicgstab(const orc_problem* p, const double* u0, double* U, double tol, int maxit, double* hist,
                 int* iterations);

/* Per-spectral-mode versions (sampled full-size parity; reading R4: in the DST basis
   Step (b) is the divide by 1 - lambda_k E_J).
   uhat: [nt] (u_1..u_Nt of mode J), uhat0 = u_0 of mode J,
   nhat: [nt] (N_0..N_{Nt-1} of mode J, may be NULL when linear; scheme 2: N of u_1..u_Nt). */
void orc_mode_residual(const orc_problem* p, long J, const double* uhat, double uhat0, const double* nhat,
                       double* rhat);
void orc_mode_precond(const orc_problem* p, long J, const double* rhat, double* shat);

/* ---- complex coefficients (oracle_cplx.c), linear only (npoly = 0, scheme 0) ----------
 * Complex vectors are interleaved (re, im) doubles, same slice/time layout as above.     */
void orc_cplx_sequential(const orc_problem* p, const double* u0, double* U);
void orc_cplx_residual(const orc_problem* p, const double* u0, const double* U, double* R, double* rnorm2);
void orc_cplx_precond(const orc_problem* p, const double* R, double* S);
void orc_cplx_apply_Q(const orc_problem* p, const double* V, double* out);
int orc_cplx_fixed_point(const orc_problem* p, const double* u0, double* U, double tol, int maxit, double* hist,
                         int* iterations);
int orc_cplx_gmres(const orc_problem* p, const double* u0, double* U, double tol, int restart, int maxit,
                   double* hist, int* iterations);
int orc_cplx_bicgstab(const orc_problem* p, const double* u0, double* U, double tol, int maxit, double* hist,
                      int* iterations);

#ifdef __cplusplus
}
#endif
#endif
