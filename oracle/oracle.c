/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the Exp-ParaDiag hot path
 * (arXiv 2603.04350, "Exp-ParaDiag: Time-Parallel Exponential Integrators for Parabolic
 * PDEs").  TEST INFRASTRUCTURE: see oracle.h for who may call it.  It shares no code
 * with the CUDA path.
 *
 * Rules followed here (DESIGN.md section "Oracle"):
 *   - every operator is the paper's definition written out: sine sums O(n) per output,
 *     DFT sums O(Nt) per output, no FFT, no blocking or algebraic fusion;
 *   - long double (x87, 64-bit mantissa) accumulation everywhere, long-double pi,
 *     twiddle indices reduced exactly mod Nt / mod 2(n+1) in integers (R13);
 *   - OpenMP only over independent slices / lines / spatial points (each output is
 *     computed by one thread in a fixed order, so results do not depend on thread count).
 *
 * Parity pins for every function live in tests/test_oracle_pins.py (numpy/scipy dense
 * brute force, closed forms, the paper's theorems); none of them calls back into this file
 * to produce an expected value.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#define IN_PAR() omp_in_parallel()
#else
#define IN_PAR() 1
#endif

typedef long double ld;
static const ld PI_LD = 3.141592653589793238462643383279502884197L;

/* ------------------------------------------------------------------------------------ */
/* sizes                                                                                 */
/* ------------------------------------------------------------------------------------ */
static long ipow(long b, int e) {
  long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
long orc_nmodes(const orc_problem* p) { return ipow(p->n, p->dim); }

/* ------------------------------------------------------------------------------------ */
/* spectra  ("L_h = V_h D_h V_h^{-1}"; eigenvalues: reading R1)             */
/* ------------------------------------------------------------------------------------ */
/* lambda_j of the 1-D Dirichlet Delta_h on h = 1/(n+1): -(4/h^2) sin^2(j pi h / 2). */
static ld axis_eig_ld(int n, int j) {
  ld h = 1.0L / (ld)(n + 1);
  ld s = sinl(PI_LD * (ld)j / (2.0L * (ld)(n + 1)));
  return -4.0L / (h * h) * s * s;
}

void orc_axis_eigs(int n, double* lam) {
  for (int j = 1; j <= n; ++j) lam[j - 1] = (double)axis_eig_ld(n, j);
}

/* mu_J = a * sum_i lambda_{j_i} - c  (L_h = a Delta_h - c I; Kronecker sum
   over axes, Remark 2.2 PAPER.md:159-161). J is the slice index, x fastest. */
static ld mode_mu_ld(const orc_problem* p, long J) {
  ld s = 0.0L;
  long r = J;
  for (int ax = 0; ax < p->dim; ++ax) {
    int j = (int)(r % p->n) + 1;
    r /= p->n;
    s += axis_eig_ld(p->n, j);
  }
  return (ld)p->a * s - (ld)p->c;
}

/* phi1(z) = (e^z - 1)/z, phi2(z) = (e^z - 1 - z)/z^2 (reading R6); Taylor series for
   |z| < 1/2 where the closed forms cancel (reading R7). */
static void phi12_ld(ld z, ld* phi1, ld* phi2) {
  if (fabsl(z) < 0.5L) {
    ld t1 = 0.0L, t2 = 0.0L, zk = 1.0L, fact = 1.0L; /* fact = (k+1)! */
    for (int k = 0; k < 40; ++k) {
      fact *= (ld)(k + 1);
      t1 += zk / fact;              /* z^k/(k+1)! */
      t2 += zk / (fact * (ld)(k + 2)); /* z^k/(k+2)! */
      zk *= z;
    }
    *phi1 = t1;
    *phi2 = t2;
  } else {
    ld em1 = expm1l(z);
    *phi1 = em1 / z;
    *phi2 = (em1 - z) / (z * z);
  }
}

/* E_J = exp(dt mu_J) (A = exp(dt L_h)), dt phi1(dt mu_J), dt phi2(dt mu_J). */
static void mode_coefs_ld(const orc_problem* p, long J, ld* E, ld* dtphi1, ld* dtphi2) {
  ld z = (ld)p->dt * mode_mu_ld(p, J);
  ld f1, f2;
  phi12_ld(z, &f1, &f2);
  if (E) *E = expl(z);
  if (dtphi1) *dtphi1 = (ld)p->dt * f1;
  if (dtphi2) *dtphi2 = (ld)p->dt * f2;
}

void orc_mode_tables(const orc_problem* p, double* mu, double* E, double* dtphi1, double* dtphi2) {
  long N = orc_nmodes(p);
#pragma omp parallel for schedule(static)
  for (long J = 0; J < N; ++J) {
    ld e, f1, f2;
    mode_coefs_ld(p, J, &e, &f1, &f2);
    if (mu) mu[J] = (double)mode_mu_ld(p, J);
    if (E) E[J] = (double)e;
    if (dtphi1) dtphi1[J] = (double)f1;
    if (dtphi2) dtphi2[J] = (double)f2;
  }
}

/* ------------------------------------------------------------------------------------ */
/* the orthonormal DST-I V (V_h orthogonal; reading R1)                    */
/*   (V v)_j = sqrt(2/(n+1)) sum_{i=1}^{n} sin(pi i j/(n+1)) v_i, per axis               */
/* ------------------------------------------------------------------------------------ */
static ld* sine_table(int n) {
  ld* S = (ld*)malloc(sizeof(ld) * (size_t)n * n);
  ld scale = sqrtl(2.0L / (ld)(n + 1));
  for (int j = 1; j <= n; ++j)
    for (int i = 1; i <= n; ++i) {
      long q = ((long)j * i) % (2L * (n + 1)); /* exact reduction of the angle index */
      S[(size_t)(j - 1) * n + (i - 1)] = scale * sinl(PI_LD * (ld)q / (ld)(n + 1));
    }
  return S;
}

/* out = V_axis in along one axis of an n^dim array (long double, out != in). */
static void dst_axis_ld(const orc_problem* p, const ld* S, int ax, const ld* in, ld* out) {
  long n = p->n;
  long stride = ipow(n, ax);
  long outer = ipow(n, p->dim - 1 - ax);
  long nlines = outer * stride;
#pragma omp parallel for schedule(static) if (!IN_PAR())
  for (long l = 0; l < nlines; ++l) {
    long o = l / stride, in_ = l % stride;
    long base = o * stride * n + in_;
    for (long j = 0; j < n; ++j) {
      ld acc = 0.0L;
      const ld* Sj = S + j * n;
      for (long i = 0; i < n; ++i) acc += Sj[i] * in[base + i * stride];
      out[base + j * stride] = acc;
    }
  }
}

/* out = V in over all axes (in != out when dim == 1). */
static void dst_ld(const orc_problem* p, const ld* S, const ld* in, ld* out) {
  long N = orc_nmodes(p);
  ld* a = (ld*)malloc(sizeof(ld) * (size_t)N);
  ld* b = (ld*)malloc(sizeof(ld) * (size_t)N);
  const ld* src = in;
  for (int ax = 0; ax < p->dim; ++ax) {
    ld* dst = (ax == p->dim - 1) ? out : (ax % 2 == 0 ? a : b);
    dst_axis_ld(p, S, ax, src, dst);
    src = dst;
  }
  free(a);
  free(b);
}

void orc_dst(const orc_problem* p, const double* in, double* out) {
  long N = orc_nmodes(p);
  ld* S = sine_table(p->n);
  ld* a = (ld*)malloc(sizeof(ld) * (size_t)N);
  ld* b = (ld*)malloc(sizeof(ld) * (size_t)N);
  for (long i = 0; i < N; ++i) a[i] = in[i];
  dst_ld(p, S, a, b);
  for (long i = 0; i < N; ++i) out[i] = (double)b[i];
  free(S); free(a); free(b);
}

/* The x-axis factor of V on nrows rows of n points (plain O(n) sums per output, the first
   axis pass of orc_dst): the bounded CPU-baseline sample of bench.py.  The sine table is
   built once per n and kept (a whole sweep builds it once too; rebuilding its n^2 sinl
   values on every call made the sample mostly table construction).  Not thread safe:
   callers are sequential. */
void orc_dst_x_rows(const orc_problem* p, const double* in, long nrows, double* out) {
  static ld* S = NULL;
  static int Sn = -1;
  if (Sn != p->n) {
    free(S);
    S = sine_table(p->n);
    Sn = p->n;
  }
  long n = p->n;
#pragma omp parallel for schedule(static)
  for (long r = 0; r < nrows; ++r) {
    for (long j = 0; j < n; ++j) {
      ld acc = 0.0L;
      const ld* Sj = S + j * n;
      for (long i = 0; i < n; ++i) acc += Sj[i] * (ld)in[r * n + i];
      out[r * n + j] = (double)acc;
    }
  }
}

/* One entry of V in: sum over all grid points of prod_axes S[j_ax][i_ax] in[i]. */
void orc_dst_sample(const orc_problem* p, const double* in, const long* idx, int ns, double* out) {
  ld* S = sine_table(p->n);
  long N = orc_nmodes(p);
  long n = p->n;
  for (int s = 0; s < ns; ++s) {
    int j[3] = {0, 0, 0};
    long r = idx[s];
    for (int ax = 0; ax < p->dim; ++ax) { j[ax] = (int)(r % n); r /= n; }
    /* reduce axis by axis: first x for every (z,y), then y, then z */
    long rest = N / n;
    ld* red = (ld*)malloc(sizeof(ld) * (size_t)rest);
#pragma omp parallel for schedule(static)
    for (long l = 0; l < rest; ++l) {
      ld acc = 0.0L;
      const ld* Sj = S + (long)j[0] * n;
      for (long i = 0; i < n; ++i) acc += Sj[i] * in[l * n + i];
      red[l] = acc;
    }
    long len = rest;
    for (int ax = 1; ax < p->dim; ++ax) {
      long nl = len / n;
      const ld* Sj = S + (long)j[ax] * n;
      for (long l = 0; l < nl; ++l) {
        ld acc = 0.0L;
        for (long i = 0; i < n; ++i) acc += Sj[i] * red[l * n + i];
        red[l] = acc; /* l*n+i >= l for all i, and entries < l are already final: safe in order */
      }
      len = nl;
    }
    out[s] = (double)red[0];
    free(red);
  }
  free(S);
}

/* The same sampled outputs for nslices consecutive slices (one sine table for all; the
   sums per output are those of orc_dst_sample). */
void orc_dst_sample_batch(const orc_problem* p, const double* in, long nslices, const long* idx, int ns,
                          double* out) {
  ld* S = sine_table(p->n);
  long N = orc_nmodes(p);
  long n = p->n;
  long rest = N / n;
  ld* red = (ld*)malloc(sizeof(ld) * (size_t)rest);
  for (long t = 0; t < nslices; ++t) {
    const double* v = in + t * N;
    for (int s = 0; s < ns; ++s) {
      int j[3] = {0, 0, 0};
      long r = idx[s];
      for (int ax = 0; ax < p->dim; ++ax) { j[ax] = (int)(r % n); r /= n; }
#pragma omp parallel for schedule(static)
      for (long l = 0; l < rest; ++l) {
        ld acc = 0.0L;
        const ld* Sj = S + (long)j[0] * n;
        for (long i = 0; i < n; ++i) acc += Sj[i] * v[l * n + i];
        red[l] = acc;
      }
      long len = rest;
      for (int ax = 1; ax < p->dim; ++ax) {
        long nl = len / n;
        const ld* Sj = S + (long)j[ax] * n;
        for (long l = 0; l < nl; ++l) {
          ld acc = 0.0L;
          for (long i = 0; i < n; ++i) acc += Sj[i] * red[l * n + i];
          red[l] = acc;
        }
        len = nl;
      }
      out[t * ns + s] = (double)red[0];
    }
  }
  free(red);
  free(S);
}

/* ------------------------------------------------------------------------------------ */
/* operators on one slice                                                                */
/* ------------------------------------------------------------------------------------ */
typedef struct {
  const orc_problem* p;
  long N;
  ld* S;      /* sine table */
  ld* E;      /* per-mode E_J            */
  ld* dphi1;  /* per-mode dt phi1(z_J)   */
  ld* dphi2;  /* per-mode dt phi2(z_J)   */
} ctx_t;

static void ctx_init(ctx_t* c, const orc_problem* p) {
  c->p = p;
  c->N = orc_nmodes(p);
  c->S = sine_table(p->n);
  c->E = (ld*)malloc(sizeof(ld) * (size_t)c->N);
  c->dphi1 = (ld*)malloc(sizeof(ld) * (size_t)c->N);
  c->dphi2 = (ld*)malloc(sizeof(ld) * (size_t)c->N);
#pragma omp parallel for schedule(static)
  for (long J = 0; J < c->N; ++J) mode_coefs_ld(p, J, &c->E[J], &c->dphi1[J], &c->dphi2[J]);
}
static void ctx_free(ctx_t* c) {
  free(c->S); free(c->E); free(c->dphi1); free(c->dphi2);
}

/* out = V diag(m) V v : a spectral multiplier applied in physical space. */
static void apply_mult_ld(const ctx_t* c, const ld* m, const ld* v, ld* out) {
  long N = c->N;
  ld* t1 = (ld*)malloc(sizeof(ld) * (size_t)N);
  dst_ld(c->p, c->S, v, t1);
  for (long J = 0; J < N; ++J) t1[J] *= m[J];
  dst_ld(c->p, c->S, t1, out);
  free(t1);
}

/* N(u) = sum_p q_p u^p pointwise (BASELINE.json:5 "pointwise nonlinear evaluation"). */
static ld nonlin_ld(const orc_problem* p, ld u) {
  ld acc = 0.0L;
  for (int k = p->npoly - 1; k >= 0; --k) acc = acc * u + (ld)p->q[k];
  return acc;
}

/* N'(u) = sum_p p q_p u^{p-1} (the Newton step of the IF scheme's implicit solve). */
static ld dnonlin_ld(const orc_problem* p, ld u) {
  ld acc = 0.0L;
  for (int k = p->npoly - 1; k >= 1; --k) acc = acc * u + (ld)k * (ld)p->q[k];
  return acc;
}

/* IF scheme (6.1): the implicit part of one step, pointwise: the v with
   v - dt N(v) = w, by Newton's method from v = w (scalar, long double; for N = -u^3 the map
   v - dt N(v) is strictly increasing, so the root is unique). */
static ld if_solve_ld(const orc_problem* p, ld w) {
  ld v = w;
  for (int it = 0; it < 100; ++it) {
    ld f = v - (ld)p->dt * nonlin_ld(p, v) - w;
    ld df = 1.0L - (ld)p->dt * dnonlin_ld(p, v);
    ld dv = f / df;
    v -= dv;
    if (fabsl(dv) <= 1e-19L * (1.0L + fabsl(v))) break;
  }
  return v;
}

void orc_apply_A(const orc_problem* p, const double* v, double* out) {
  ctx_t c;
  ctx_init(&c, p);
  ld* a = (ld*)malloc(sizeof(ld) * (size_t)c.N);
  ld* b = (ld*)malloc(sizeof(ld) * (size_t)c.N);
  for (long i = 0; i < c.N; ++i) a[i] = v[i];
  apply_mult_ld(&c, c.E, a, b);
  for (long i = 0; i < c.N; ++i) out[i] = (double)b[i];
  free(a); free(b);
  ctx_free(&c);
}

void orc_nonlin(const orc_problem* p, const double* u, double* out) {
  long N = orc_nmodes(p);
  for (long i = 0; i < N; ++i) out[i] = (double)nonlin_ld(p, (ld)u[i]);
}

/* ------------------------------------------------------------------------------------ */
/* time stepping pieces                                                                  */
/* ------------------------------------------------------------------------------------ */
/* Phi-term of step n given the physical N(u_{n-1}) (nm1) and N(u_{n-2}) (nm2):
     ETD1 (R5):  V diag(dt phi1) V N(u_{n-1})
     ETD2 (R6):  V diag(dt phi1 + dt phi2) V N(u_{n-1}) - V diag(dt phi2) V N(u_{n-2})
   added into acc.  Each product is applied separately, as written. */
static void add_phi_terms_ld(const ctx_t* c, const ld* nm1, const ld* nm2, ld* acc) {
  const orc_problem* p = c->p;
  long N = c->N;
  ld* t = (ld*)malloc(sizeof(ld) * (size_t)N);
  if (p->scheme == 0) {
    apply_mult_ld(c, c->dphi1, nm1, t);
    for (long i = 0; i < N; ++i) acc[i] += t[i];
  } else {
    ld* m12 = (ld*)malloc(sizeof(ld) * (size_t)N);
    for (long J = 0; J < N; ++J) m12[J] = c->dphi1[J] + c->dphi2[J];
    apply_mult_ld(c, m12, nm1, t);
    for (long i = 0; i < N; ++i) acc[i] += t[i];
    apply_mult_ld(c, c->dphi2, nm2, t);
    for (long i = 0; i < N; ++i) acc[i] -= t[i];
    free(m12);
  }
  free(t);
}

/* Sequential stepping u_n = A u_{n-1} [+ Phi terms], n = 1..Nt (R5, R6). */
void orc_sequential(const orc_problem* p, const double* u0, double* U) {
  ctx_t c;
  ctx_init(&c, p);
  long N = c.N;
  int nonlin = p->npoly > 0;
  ld* prev = (ld*)malloc(sizeof(ld) * (size_t)N);
  ld* cur = (ld*)malloc(sizeof(ld) * (size_t)N);
  ld* nm1 = (ld*)malloc(sizeof(ld) * (size_t)N);
  ld* nm2 = (ld*)malloc(sizeof(ld) * (size_t)N);
  for (long i = 0; i < N; ++i) prev[i] = u0[i];
  if (p->scheme == 3) {
    /* exponential BDF2 (4.1): u_n = 4/3 A u_{n-1} - 1/3 B u_{n-2}, B = A^2,
       started by u_1 = A u_0 (reading R16); U holds the unknowns v = (u_2, .., u_{Nt+1})
       of the all-at-once system (4.2), Nt = p->nt of them. */
    ld* um2 = (ld*)malloc(sizeof(ld) * (size_t)N);
    ld* t1 = (ld*)malloc(sizeof(ld) * (size_t)N);
    memcpy(um2, prev, sizeof(ld) * (size_t)N);       /* u_0 */
    apply_mult_ld(&c, c.E, um2, prev);                /* u_1 = A u_0 */
    for (int n = 2; n <= p->nt + 1; ++n) {
      apply_mult_ld(&c, c.E, prev, cur);              /* A u_{n-1} */
      apply_mult_ld(&c, c.E, um2, t1);
      apply_mult_ld(&c, c.E, t1, nm1);                /* B u_{n-2} = A (A u_{n-2}) */
      for (long i = 0; i < N; ++i) cur[i] = (4.0L / 3.0L) * cur[i] - (1.0L / 3.0L) * nm1[i];
      for (long i = 0; i < N; ++i) U[(size_t)(n - 2) * N + i] = (double)cur[i];
      memcpy(um2, prev, sizeof(ld) * (size_t)N);
      memcpy(prev, cur, sizeof(ld) * (size_t)N);
    }
    free(um2); free(t1);
    free(prev); free(cur); free(nm1); free(nm2);
    ctx_free(&c);
    return;
  }
  /* N(u_{-1}) := N(u_0) (R6) */
  for (long i = 0; i < N; ++i) nm2[i] = nonlin_ld(p, prev[i]);
  for (int n = 1; n <= p->nt; ++n) {
    apply_mult_ld(&c, c.E, prev, cur);
    if (nonlin && p->scheme == 2) {
      /* IF (6.1): u_n = A u_{n-1} + dt N(u_n), implicit pointwise */
      for (long i = 0; i < N; ++i) cur[i] = if_solve_ld(p, cur[i]);
    } else if (nonlin) {
      for (long i = 0; i < N; ++i) nm1[i] = nonlin_ld(p, prev[i]);
      add_phi_terms_ld(&c, nm1, nm2, cur);
      memcpy(nm2, nm1, sizeof(ld) * (size_t)N);
    }
    for (long i = 0; i < N; ++i) U[(size_t)(n - 1) * N + i] = (double)cur[i];
    ld* t = prev; prev = cur; cur = t;
  }
  free(prev); free(cur); free(nm1); free(nm2);
  ctx_free(&c);
}

/* r_n = A u_{n-1} + Phi[N] - u_n, n = 1..Nt, U in long double (PAPER.md:181-183 gives
   f - Q u for the linear part: f = (A u_0, 0, ..., 0), (Q u)_n = u_n - A u_{n-1}). */
/* BDF2 (scheme 3): r = f_2 - R v, v = (u_2, .., u_{Nt+1}), u_1 = A u_0:
   r_1 = 4/3 A u_1 - 1/3 B u_0 - v_1, r_2 = 4/3 A v_1 - 1/3 B u_1 - v_2,
   r_n = 4/3 A v_{n-1} - 1/3 B v_{n-2} - v_n. */
static void residual_bdf2_ld(const ctx_t* c, const ld* u0, const ld* U, ld* R) {
  const orc_problem* p = c->p;
  long N = c->N;
  ld* u1 = (ld*)malloc(sizeof(ld) * (size_t)N);
  apply_mult_ld(c, c->E, u0, u1);
#pragma omp parallel for schedule(dynamic, 1)
  for (int n = 1; n <= p->nt; ++n) {
    const ld* p1 = (n == 1) ? u1 : U + (size_t)(n - 2) * N;                       /* v_{n-1} */
    const ld* p2 = (n == 1) ? u0 : (n == 2) ? u1 : U + (size_t)(n - 3) * N;       /* v_{n-2} */
    ld* r = R + (size_t)(n - 1) * N;
    ld* t1 = (ld*)malloc(sizeof(ld) * (size_t)N);
    ld* t2 = (ld*)malloc(sizeof(ld) * (size_t)N);
    apply_mult_ld(c, c->E, p1, r);
    apply_mult_ld(c, c->E, p2, t1);
    apply_mult_ld(c, c->E, t1, t2);
    const ld* vn = U + (size_t)(n - 1) * N;
    for (long i = 0; i < N; ++i) r[i] = (4.0L / 3.0L) * r[i] - (1.0L / 3.0L) * t2[i] - vn[i];
    free(t1); free(t2);
  }
  free(u1);
}

static void residual_ld(const ctx_t* c, const ld* u0, const ld* U, ld* R) {
  const orc_problem* p = c->p;
  long N = c->N;
  int nonlin = p->npoly > 0;
  if (p->scheme == 3) {
    residual_bdf2_ld(c, u0, U, R);
    return;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int n = 1; n <= p->nt; ++n) {
    const ld* prev = (n == 1) ? u0 : U + (size_t)(n - 2) * N;
    ld* r = R + (size_t)(n - 1) * N;
    apply_mult_ld(c, c->E, prev, r);
    if (nonlin && p->scheme == 2) {
      /* IF / IMEX-type: + dt N(u_n) of the same slice */
      const ld* un = U + (size_t)(n - 1) * N;
      for (long i = 0; i < N; ++i) r[i] += (ld)p->dt * nonlin_ld(p, un[i]);
    } else if (nonlin) {
      const ld* prev2 = (n <= 2) ? u0 : U + (size_t)(n - 3) * N; /* u_{n-2}; u_{-1} -> u_0 (R6) */
      ld* nm1 = (ld*)malloc(sizeof(ld) * (size_t)N);
      ld* nm2 = (ld*)malloc(sizeof(ld) * (size_t)N);
      for (long i = 0; i < N; ++i) nm1[i] = nonlin_ld(p, prev[i]);
      for (long i = 0; i < N; ++i) nm2[i] = nonlin_ld(p, prev2[i]);
      add_phi_terms_ld(c, nm1, nm2, r);
      free(nm1); free(nm2);
    }
    const ld* un = U + (size_t)(n - 1) * N;
    for (long i = 0; i < N; ++i) r[i] -= un[i];
  }
}

static ld norm2_ld(const ld* v, size_t len) {
  ld s = 0.0L;
  for (size_t i = 0; i < len; ++i) s += v[i] * v[i];
  return s;
}

void orc_residual(const orc_problem* p, const double* u0, const double* U, double* R, double* rnorm2) {
  ctx_t c;
  ctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  ld* u0l = (ld*)malloc(sizeof(ld) * N);
  ld* Ul = (ld*)malloc(sizeof(ld) * tot);
  ld* Rl = (ld*)malloc(sizeof(ld) * tot);
  for (size_t i = 0; i < N; ++i) u0l[i] = u0[i];
  for (size_t i = 0; i < tot; ++i) Ul[i] = U[i];
  residual_ld(&c, u0l, Ul, Rl);
  for (size_t i = 0; i < tot; ++i) R[i] = (double)Rl[i];
  if (rnorm2) *rnorm2 = (double)norm2_ld(Rl, tot);
  free(u0l); free(Ul); free(Rl);
  ctx_free(&c);
}

/* (Q v)_n = v_n - A v_{n-1}, v_0 = 0 (C_0 = C_0^alpha at alpha = 0);
   with corner = alpha this is Q_alpha: (Q_a v)_1 = v_1 - alpha A v_Nt. */
static void apply_Qcorner_ld(const ctx_t* c, ld corner, const ld* V, ld* out) {
  const orc_problem* p = c->p;
  long N = c->N;
  if (p->scheme == 3) {
    /* BDF2: R v = v - 4/3 (C_0 (x) A) v + 1/3 (C_1 (x) B) v; with
       corner alpha: R_alpha, C_0^alpha(1, L) = alpha, C_1^alpha(1, L-1) = C_1^alpha(2, L) =
       alpha */
    const int L = p->nt;
#pragma omp parallel for schedule(dynamic, 1)
    for (int n = 1; n <= L; ++n) {
      ld* o = out + (size_t)(n - 1) * N;
      const ld* vn = V + (size_t)(n - 1) * N;
      ld* t1 = (ld*)malloc(sizeof(ld) * (size_t)N);
      ld* t2 = (ld*)malloc(sizeof(ld) * (size_t)N);
      for (long i = 0; i < N; ++i) o[i] = vn[i];
      /* C_0 part: v_{n-1} (n >= 2), alpha v_L (n = 1) */
      const ld* a0 = (n >= 2) ? V + (size_t)(n - 2) * N : V + (size_t)(L - 1) * N;
      ld w0 = (n >= 2) ? 1.0L : corner;
      if (w0 != 0.0L) {
        apply_mult_ld(c, c->E, a0, t1);
        for (long i = 0; i < N; ++i) o[i] -= (4.0L / 3.0L) * w0 * t1[i];
      }
      /* C_1 part: v_{n-2} (n >= 3), alpha v_{L-1} (n = 1), alpha v_L (n = 2) */
      const ld* a1 = (n >= 3) ? V + (size_t)(n - 3) * N : V + (size_t)(L - 3 + n) * N;
      ld w1 = (n >= 3) ? 1.0L : corner;
      if (w1 != 0.0L) {
        apply_mult_ld(c, c->E, a1, t1);
        apply_mult_ld(c, c->E, t1, t2);
        for (long i = 0; i < N; ++i) o[i] += (1.0L / 3.0L) * w1 * t2[i];
      }
      free(t1); free(t2);
    }
    return;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int n = 1; n <= p->nt; ++n) {
    ld* o = out + (size_t)(n - 1) * N;
    const ld* vn = V + (size_t)(n - 1) * N;
    if (n == 1) {
      if (corner != 0.0L) {
        apply_mult_ld(c, c->E, V + (size_t)(p->nt - 1) * N, o);
        for (long i = 0; i < N; ++i) o[i] = vn[i] - corner * o[i];
      } else {
        for (long i = 0; i < N; ++i) o[i] = vn[i];
      }
    } else {
      apply_mult_ld(c, c->E, V + (size_t)(n - 2) * N, o);
      for (long i = 0; i < N; ++i) o[i] = vn[i] - o[i];
    }
  }
}

static void apply_Q_wrap(const orc_problem* p, ld corner, const double* V, double* out) {
  ctx_t c;
  ctx_init(&c, p);
  size_t tot = (size_t)c.N * (size_t)p->nt;
  ld* a = (ld*)malloc(sizeof(ld) * tot);
  ld* b = (ld*)malloc(sizeof(ld) * tot);
  for (size_t i = 0; i < tot; ++i) a[i] = V[i];
  apply_Qcorner_ld(&c, corner, a, b);
  for (size_t i = 0; i < tot; ++i) out[i] = (double)b[i];
  free(a); free(b);
  ctx_free(&c);
}
void orc_apply_Q(const orc_problem* p, const double* V, double* out) { apply_Q_wrap(p, 0.0L, V, out); }
void orc_apply_Qalpha(const orc_problem* p, const double* V, double* out) {
  apply_Q_wrap(p, (ld)p->alpha, V, out);
}

/* ------------------------------------------------------------------------------------ */
/* the alpha-circulant preconditioner, literal Steps (a)-(c)          */
/* ------------------------------------------------------------------------------------ */
/* Gamma_alpha = diag(alpha^{(m-1)/Nt}) ; F = Nt^{-1/2} [omega^{(l1-1)(l2-1)}], omega =
   e^{2 pi i/Nt} ; lambda_k = alpha^{1/Nt} omega^{k-1}.  Indices below
   are 0-based: m, k = 0..Nt-1 stand for the paper's m, k = 1..Nt. */
static ld precond_ld(const ctx_t* c, const ld* R, ld* Sout) {
  const orc_problem* p = c->p;
  int nt = p->nt;
  long N = c->N;
  size_t tot = (size_t)N * nt;
  ld* cs = (ld*)malloc(sizeof(ld) * nt);
  ld* sn = (ld*)malloc(sizeof(ld) * nt);
  ld* g = (ld*)malloc(sizeof(ld) * nt);
  for (int q = 0; q < nt; ++q) {
    cs[q] = cosl(2.0L * PI_LD * (ld)q / (ld)nt);
    sn[q] = sinl(2.0L * PI_LD * (ld)q / (ld)nt);
    g[q] = powl((ld)p->alpha, (ld)q / (ld)nt); /* alpha^{(m-1)/Nt} */
  }
  ld inv_sqrt_nt = 1.0L / sqrtl((ld)nt);
  ld* Yre = (ld*)malloc(sizeof(ld) * tot);
  ld* Yim = (ld*)malloc(sizeof(ld) * tot);

  /* Step (a): S_a = (F (x) I)(Gamma_alpha (x) I) r. */
#pragma omp parallel for schedule(static)
  for (long x = 0; x < N; ++x) {
    for (int k = 0; k < nt; ++k) {
      ld are = 0.0L, aim = 0.0L;
      for (int m = 0; m < nt; ++m) {
        int q = (int)(((long)k * m) % nt);
        ld y = g[m] * R[(size_t)m * N + x];
        are += cs[q] * y;
        aim += sn[q] * y;
      }
      Yre[(size_t)k * N + x] = inv_sqrt_nt * are;
      Yim[(size_t)k * N + x] = inv_sqrt_nt * aim;
    }
  }

  /* Step (b): S_{b,k} = (I - lambda_k A)^{-1} S_{a,k}; A = V diag(E) V, so
     (I - lambda_k A)^{-1} = V diag(1/(1 - lambda_k E_J)) V (reading R4). */
  ld a1 = powl((ld)p->alpha, 1.0L / (ld)nt);
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < nt; ++k) {
    ld* tr = (ld*)malloc(sizeof(ld) * (size_t)N);
    ld* ti = (ld*)malloc(sizeof(ld) * (size_t)N);
    ld* yr = Yre + (size_t)k * N;
    ld* yi = Yim + (size_t)k * N;
    dst_ld(p, c->S, yr, tr);
    dst_ld(p, c->S, yi, ti);
    ld lre = a1 * cs[k], lim = a1 * sn[k];
    /* BDF2: lambda_{1,k} = alpha^{2/L} e^{4 pi i (k-1)/L} */
    int q2 = (int)((2L * k) % nt);
    ld l1re = powl((ld)p->alpha, 2.0L / (ld)nt) * cs[q2], l1im = powl((ld)p->alpha, 2.0L / (ld)nt) * sn[q2];
    for (long J = 0; J < N; ++J) {
      ld dre = 1.0L - lre * c->E[J], dim = -lim * c->E[J]; /* 1 - lambda_k E_J */
      if (p->scheme == 3) {
        /* 1 - 4/3 lambda_{0,k} E_J + 1/3 lambda_{1,k} E_J^2 (Step (b), (4.5)) */
        ld e2 = c->E[J] * c->E[J];
        dre = 1.0L - (4.0L / 3.0L) * lre * c->E[J] + (1.0L / 3.0L) * l1re * e2;
        dim = -(4.0L / 3.0L) * lim * c->E[J] + (1.0L / 3.0L) * l1im * e2;
      }
      ld den = dre * dre + dim * dim;
      ld xr = (tr[J] * dre + ti[J] * dim) / den;
      ld xi = (ti[J] * dre - tr[J] * dim) / den;
      tr[J] = xr;
      ti[J] = xi;
    }
    dst_ld(p, c->S, tr, yr);
    dst_ld(p, c->S, ti, yi);
    free(tr); free(ti);
  }

  /* Step (c): s = (Gamma_alpha^{-1} (x) I)(F^* (x) I) S_b ; keep Re, measure Im. */
  ld maxre = 0.0L, maxim = 0.0L;
#pragma omp parallel for schedule(static) reduction(max : maxre, maxim)
  for (long x = 0; x < N; ++x) {
    for (int m = 0; m < nt; ++m) {
      ld are = 0.0L, aim = 0.0L;
      for (int k = 0; k < nt; ++k) {
        int q = (int)(((long)k * m) % nt);
        ld yr = Yre[(size_t)k * N + x], yi = Yim[(size_t)k * N + x];
        /* omega^{-q} = cs[q] - i sn[q] */
        are += cs[q] * yr + sn[q] * yi;
        aim += cs[q] * yi - sn[q] * yr;
      }
      ld sre = inv_sqrt_nt * are / g[m];
      ld sim = inv_sqrt_nt * aim / g[m];
      Sout[(size_t)m * N + x] = sre;
      if (fabsl(sre) > maxre) maxre = fabsl(sre);
      if (fabsl(sim) > maxim) maxim = fabsl(sim);
    }
  }
  free(cs); free(sn); free(g); free(Yre); free(Yim);
  return maxre > 0.0L ? maxim / maxre : 0.0L;
}

double orc_precond(const orc_problem* p, const double* R, double* S) {
  ctx_t c;
  ctx_init(&c, p);
  size_t tot = (size_t)c.N * (size_t)p->nt;
  ld* Rl = (ld*)malloc(sizeof(ld) * tot);
  ld* Sl = (ld*)malloc(sizeof(ld) * tot);
  for (size_t i = 0; i < tot; ++i) Rl[i] = R[i];
  ld leak = precond_ld(&c, Rl, Sl);
  for (size_t i = 0; i < tot; ++i) S[i] = (double)Sl[i];
  free(Rl); free(Sl);
  ctx_free(&c);
  return (double)leak;
}

/* ------------------------------------------------------------------------------------ */
/* solvers                                                                               */
/* ------------------------------------------------------------------------------------ */
int orc_fixed_point(const orc_problem* p, const double* u0, double* U, double tol, int maxit,
                    double* hist, int* iterations) {
  ctx_t c;
  ctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  ld* u0l = (ld*)malloc(sizeof(ld) * N);
  ld* Ul = (ld*)malloc(sizeof(ld) * tot);
  ld* Rl = (ld*)malloc(sizeof(ld) * tot);
  ld* Sl = (ld*)malloc(sizeof(ld) * tot);
  for (size_t i = 0; i < N; ++i) u0l[i] = u0[i];
  for (size_t i = 0; i < tot; ++i) Ul[i] = U[i];
  ld r0 = 0.0L;
  int status = 7;
  int k;
  for (k = 0; k <= maxit; ++k) {
    residual_ld(&c, u0l, Ul, Rl);                 /* r^k = F(U^k) - Q U^k            */
    ld rn = sqrtl(norm2_ld(Rl, tot));
    if (k == 0) r0 = rn;
    ld rho = (r0 > 0.0L) ? rn / r0 : 0.0L;
    if (hist) hist[k] = (double)rho;
    precond_ld(&c, Rl, Sl);                       /* s^k = Q_alpha^{-1} r^k (3.2)    */
    for (size_t i = 0; i < tot; ++i) Ul[i] += Sl[i]; /* U^{k+1} = U^k + s^k          */
    if (rho < (ld)tol) { status = 0; break; }
  }
  if (iterations) *iterations = (status == 0) ? k : maxit;
  for (size_t i = 0; i < tot; ++i) U[i] = (double)Ul[i];
  free(u0l); free(Ul); free(Rl); free(Sl);
  ctx_free(&c);
  return status;
}

int orc_gmres(const orc_problem* p, const double* u0, double* U, double tol, int restart, int maxit,
              double* hist, int* iterations) {
  if (p->npoly > 0) return 2;
  if (restart < 1) restart = 1;
  ctx_t c;
  ctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  int m = restart;
  ld* u0l = (ld*)malloc(sizeof(ld) * N);
  ld* x = (ld*)malloc(sizeof(ld) * tot);
  ld* r = (ld*)malloc(sizeof(ld) * tot);
  ld* w = (ld*)malloc(sizeof(ld) * tot);
  ld* t = (ld*)malloc(sizeof(ld) * tot);
  ld** V = (ld**)calloc((size_t)m + 1, sizeof(ld*));
  ld* H = (ld*)calloc((size_t)(m + 1) * m, sizeof(ld)); /* H[i*m + j] */
  ld* cs = (ld*)calloc((size_t)m, sizeof(ld));
  ld* sn = (ld*)calloc((size_t)m, sizeof(ld));
  ld* g = (ld*)calloc((size_t)m + 1, sizeof(ld));
  ld* y = (ld*)calloc((size_t)m, sizeof(ld));
  ld* h = (ld*)calloc((size_t)m + 1, sizeof(ld));
  ld* h2 = (ld*)calloc((size_t)m + 1, sizeof(ld));
  for (size_t i = 0; i < N; ++i) u0l[i] = u0[i];
  for (size_t i = 0; i < tot; ++i) x[i] = U[i];
  int its = 0, status = 7;
  ld beta0 = -1.0L;
  if (hist) hist[0] = 1.0;
  while (its < maxit) {
    /* r = Q_alpha^{-1} (f - Q x); for a linear problem f - Q x is the all-at-once residual. */
    residual_ld(&c, u0l, x, t);
    precond_ld(&c, t, r);
    ld beta = sqrtl(norm2_ld(r, tot));
    if (beta0 < 0.0L) beta0 = beta;
    if (beta0 == 0.0L || beta / beta0 < (ld)tol) { status = 0; break; }
    if (!V[0]) V[0] = (ld*)malloc(sizeof(ld) * tot);
    for (size_t i = 0; i < tot; ++i) V[0][i] = r[i] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0.0L;
    g[0] = beta;
    int j, done = 0;
    for (j = 0; j < m && its < maxit; ++j) {
      apply_Qcorner_ld(&c, 0.0L, V[j], t); /* Q v_j       */
      precond_ld(&c, t, w);                /* Q_a^{-1} Q v_j */
      /* classical Gram-Schmidt, applied twice (reading R11) */
      for (int pass = 0; pass < 2; ++pass) {
        ld* hh = pass == 0 ? h : h2;
        for (int i = 0; i <= j; ++i) {
          ld s = 0.0L;
          for (size_t q = 0; q < tot; ++q) s += V[i][q] * w[q];
          hh[i] = s;
        }
        for (int i = 0; i <= j; ++i)
          for (size_t q = 0; q < tot; ++q) w[q] -= hh[i] * V[i][q];
      }
      for (int i = 0; i <= j; ++i) H[i * m + j] = h[i] + h2[i];
      ld hn = sqrtl(norm2_ld(w, tot));
      H[(j + 1) * m + j] = hn;
      /* previous rotations, then a new one zeroing H[j+1][j] */
      for (int i = 0; i < j; ++i) {
        ld a = H[i * m + j], b = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * b;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
      }
      ld a = H[j * m + j], b = H[(j + 1) * m + j];
      ld den = sqrtl(a * a + b * b);
      cs[j] = den > 0.0L ? a / den : 1.0L;
      sn[j] = den > 0.0L ? b / den : 0.0L;
      H[j * m + j] = den;
      H[(j + 1) * m + j] = 0.0L;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++its;
      ld rel = fabsl(g[j + 1]) / beta0;
      if (hist) hist[its] = (double)rel;
      if (rel < (ld)tol || hn == 0.0L) { done = 1; ++j; break; }
      if (!V[j + 1]) V[j + 1] = (ld*)malloc(sizeof(ld) * tot);
      for (size_t q = 0; q < tot; ++q) V[j + 1][q] = w[q] / hn;
    }
    /* y = H^{-1} g (upper triangular, j x j), x += V y */
    for (int i = j - 1; i >= 0; --i) {
      ld s = g[i];
      for (int l = i + 1; l < j; ++l) s -= H[i * m + l] * y[l];
      y[i] = s / H[i * m + i];
    }
    for (int i = 0; i < j; ++i)
      for (size_t q = 0; q < tot; ++q) x[q] += y[i] * V[i][q];
    if (done) { status = 0; break; }
  }
  if (iterations) *iterations = its;
  for (size_t i = 0; i < tot; ++i) U[i] = (double)x[i];
  for (int i = 0; i <= m; ++i) free(V[i]);
  free(V); free(H); free(cs); free(sn); free(g); free(y); free(h); free(h2);
  free(u0l); free(x); free(r); free(w); free(t);
  ctx_free(&c);
  return status;
}

/* ------------------------------------------------------------------------------------ */
/* per-spectral-mode versions (sampled checks at full size)                              */
/* ------------------------------------------------------------------------------------ */
/* Left-preconditioned BiCGStab (van der Vorst) on Q_alpha^{-1} Q x = Q_alpha^{-1} f from
   x_0 = U (zeros), PAPER.md:1088-1114 ("preconditioned BiCGStab" with the same
   preconditioner), reading R17: the preconditioned residual r = Q_alpha^{-1}(f - Q x) is
   iterated and the stop is ||r|| / ||r_0|| < tol, also tested after the half step (s);
   iterations = BiCGStab steps (two operator applications each).  Linear problems. */
static ld dot_ld(const ld* a, const ld* b, size_t len) {
  ld s = 0.0L;
  for (size_t i = 0; i < len; ++i) s += a[i] * b[i];
  return s;
}
int orc_bicgstab(const orc_problem* p, const double* u0, double* U, double tol, int maxit, double* hist,
                 int* iterations) {
  if (p->npoly > 0) return 2;
  ctx_t c;
  ctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  ld* u0l = (ld*)malloc(sizeof(ld) * N);
  ld* x = (ld*)malloc(sizeof(ld) * tot);
  ld* r = (ld*)malloc(sizeof(ld) * tot);
  ld* rh = (ld*)malloc(sizeof(ld) * tot);
  ld* pv = (ld*)calloc(tot, sizeof(ld));
  ld* v = (ld*)calloc(tot, sizeof(ld));
  ld* s = (ld*)malloc(sizeof(ld) * tot);
  ld* t = (ld*)malloc(sizeof(ld) * tot);
  ld* w = (ld*)malloc(sizeof(ld) * tot);
  for (size_t i = 0; i < N; ++i) u0l[i] = u0[i];
  for (size_t i = 0; i < tot; ++i) x[i] = U[i];
  residual_ld(&c, u0l, x, w); /* f - Q x */
  precond_ld(&c, w, r);       /* r_0 */
  memcpy(rh, r, sizeof(ld) * tot);
  ld beta0 = sqrtl(norm2_ld(r, tot));
  if (hist) hist[0] = 1.0;
  int status = 7, its = 0;
  ld rho_prev = 1.0L, al = 1.0L, om = 1.0L;
  if (beta0 == 0.0L) status = 0;
  for (int i = 0; status != 0 && i < maxit; ++i) {
    ld rho = dot_ld(rh, r, tot);
    ld beta = (rho / rho_prev) * (al / om);
    for (size_t q = 0; q < tot; ++q) pv[q] = r[q] + beta * (pv[q] - om * v[q]);
    apply_Qcorner_ld(&c, 0.0L, pv, w);
    precond_ld(&c, w, v); /* v = Q_a^{-1} Q p */
    al = rho / dot_ld(rh, v, tot);
    for (size_t q = 0; q < tot; ++q) s[q] = r[q] - al * v[q];
    ld sn = sqrtl(norm2_ld(s, tot));
    if (sn / beta0 < (ld)tol) { /* half step */
      for (size_t q = 0; q < tot; ++q) x[q] += al * pv[q];
      its = i + 1;
      if (hist) hist[its] = (double)(sn / beta0);
      status = 0;
      break;
    }
    apply_Qcorner_ld(&c, 0.0L, s, w);
    precond_ld(&c, w, t); /* t = Q_a^{-1} Q s */
    om = dot_ld(t, s, tot) / dot_ld(t, t, tot);
    for (size_t q = 0; q < tot; ++q) {
      x[q] += al * pv[q] + om * s[q];
      r[q] = s[q] - om * t[q];
    }
    rho_prev = rho;
    its = i + 1;
    ld rn = sqrtl(norm2_ld(r, tot));
    if (hist) hist[its] = (double)(rn / beta0);
    if (rn / beta0 < (ld)tol) { status = 0; break; }
  }
  if (iterations) *iterations = its;
  for (size_t i = 0; i < tot; ++i) U[i] = (double)x[i];
  free(u0l); free(x); free(r); free(rh); free(pv); free(v); free(s); free(t); free(w);
  ctx_free(&c);
  return status;
}

void orc_mode_residual(const orc_problem* p, long J, const double* uhat, double uhat0, const double* nhat,
                       double* rhat) {
  ld E, f1, f2;
  mode_coefs_ld(p, J, &E, &f1, &f2);
  int nonlin = p->npoly > 0 && nhat;
  if (p->scheme == 3) {  /* BDF2 (see residual_bdf2_ld), u_1 = E u_0 */
    ld u1 = E * (ld)uhat0;
    for (int n = 1; n <= p->nt; ++n) {
      ld p1 = (n == 1) ? u1 : (ld)uhat[n - 2];
      ld p2 = (n == 1) ? (ld)uhat0 : (n == 2) ? u1 : (ld)uhat[n - 3];
      rhat[n - 1] = (double)((4.0L / 3.0L) * E * p1 - (1.0L / 3.0L) * E * E * p2 - (ld)uhat[n - 1]);
    }
    return;
  }
  for (int n = 1; n <= p->nt; ++n) {
    ld prev = (n == 1) ? (ld)uhat0 : (ld)uhat[n - 2];
    ld r = E * prev - (ld)uhat[n - 1];
    if (nonlin && p->scheme == 2) {
      r += (ld)p->dt * (ld)nhat[n - 1];  /* nhat[n-1] = N-hat of u_n (same slice) */
    } else if (nonlin) {
      ld nm1 = nhat[n - 1];                    /* N_{n-1}                       */
      ld nm2 = (n >= 2) ? nhat[n - 2] : nhat[0]; /* N_{n-2}, N_{-1} := N_0 (R6)   */
      if (p->scheme == 0) r += f1 * nm1;
      else r += (f1 + f2) * nm1 - f2 * nm2;
    }
    rhat[n - 1] = (double)r;
  }
}

void orc_mode_precond(const orc_problem* p, long J, const double* rhat, double* shat) {
  int nt = p->nt;
  ld E;
  mode_coefs_ld(p, J, &E, NULL, NULL);
  ld* cs = (ld*)malloc(sizeof(ld) * nt);
  ld* sn = (ld*)malloc(sizeof(ld) * nt);
  ld* g = (ld*)malloc(sizeof(ld) * nt);
  ld* Yr = (ld*)malloc(sizeof(ld) * nt);
  ld* Yi = (ld*)malloc(sizeof(ld) * nt);
  for (int q = 0; q < nt; ++q) {
    cs[q] = cosl(2.0L * PI_LD * (ld)q / (ld)nt);
    sn[q] = sinl(2.0L * PI_LD * (ld)q / (ld)nt);
    g[q] = powl((ld)p->alpha, (ld)q / (ld)nt);
  }
  ld is = 1.0L / sqrtl((ld)nt);
  ld a1 = powl((ld)p->alpha, 1.0L / (ld)nt);
  for (int k = 0; k < nt; ++k) { /* Step (a) */
    ld are = 0.0L, aim = 0.0L;
    for (int m = 0; m < nt; ++m) {
      int q = (int)(((long)k * m) % nt);
      ld y = g[m] * (ld)rhat[m];
      are += cs[q] * y;
      aim += sn[q] * y;
    }
    /* Step (b): divide by 1 - lambda_k E_J (BDF2: 1 - 4/3 lambda_{0,k} E + 1/3 lambda_{1,k} E^2) */
    ld dre = 1.0L - a1 * cs[k] * E, dim = -a1 * sn[k] * E;
    if (p->scheme == 3) {
      int q2 = (int)((2L * k) % nt);
      ld a2 = powl((ld)p->alpha, 2.0L / (ld)nt);
      dre = 1.0L - (4.0L / 3.0L) * a1 * cs[k] * E + (1.0L / 3.0L) * a2 * cs[q2] * E * E;
      dim = -(4.0L / 3.0L) * a1 * sn[k] * E + (1.0L / 3.0L) * a2 * sn[q2] * E * E;
    }
    ld den = dre * dre + dim * dim;
    ld yr = is * are, yi = is * aim;
    Yr[k] = (yr * dre + yi * dim) / den;
    Yi[k] = (yi * dre - yr * dim) / den;
  }
  for (int m = 0; m < nt; ++m) { /* Step (c) */
    ld are = 0.0L;
    for (int k = 0; k < nt; ++k) {
      int q = (int)(((long)k * m) % nt);
      are += cs[q] * Yr[k] + sn[q] * Yi[k];
    }
    shat[m] = (double)(is * are / g[m]);
  }
  free(cs); free(sn); free(g); free(Yr); free(Yi);
}
