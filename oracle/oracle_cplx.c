/*
 * oracle_cplx.c -- the CPU oracle for LINEAR problems with COMPLEX coefficients
 * (u_t = (a Delta - c) u, a, c complex: the paper's Schroedinger tests, a = i, c = 2i and
 * c = 200i).  TEST INFRASTRUCTURE, like oracle.c (see
 * oracle.h for who may call it); it shares no code with the CUDA path.
 *
 * Same rules as oracle.c: every operator is its definition written out (sine sums O(n)
 * per output, DFT sums O(Nt) per output), long double (complex) accumulation, long-double
 * pi, angle indices reduced exactly in integers.  Complex vectors are interleaved doubles
 * (re, im).  V (the orthonormal DST-I) is real, so V acts on the real and imaginary parts
 * separately; E_J = exp(dt (a mu_J^0 - c)) with mu_J^0 the eigenvalue of the discrete
 * Laplacian (reading R1) is complex; Step (a)-(c) and the solvers are those of oracle.c
 * with complex arithmetic.  GMRES is GMRES over C with the Hermitian inner product
 * <v, w> = sum conj(v) w (the paper runs MATLAB's gmres on complex vectors; reading R18).
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef long double ld;
typedef long double complex lc;
static const ld PI_C = 3.141592653589793238462643383279502884197L;

static long cx_nmodes(const orc_problem* p) {
  long r = 1;
  for (int i = 0; i < p->dim; ++i) r *= p->n;
  return r;
}

/* sum over axes of the 1-D Dirichlet eigenvalues -(4/h^2) sin^2(j pi h/2) (reading R1) */
static ld lap_eig_ld(const orc_problem* p, long J) {
  long n = p->n;
  ld h = 1.0L / (ld)(n + 1), s = 0.0L;
  long r = J;
  for (int ax = 0; ax < p->dim; ++ax) {
    int j = (int)(r % n) + 1;
    r /= n;
    ld sn = sinl(PI_C * (ld)j / (2.0L * (ld)(n + 1)));
    s += -4.0L / (h * h) * sn * sn;
  }
  return s;
}

/* E_J = exp(dt (a Delta_J - c)), complex a = a + i a_im, c = c + i c_im */
static lc mode_E(const orc_problem* p, long J) {
  lc a = (ld)p->a + I * (ld)p->a_im, c = (ld)p->c + I * (ld)p->c_im;
  return cexpl((ld)p->dt * (a * lap_eig_ld(p, J) - c));
}

static ld* sine_tab(int n) {
  ld* S = (ld*)malloc(sizeof(ld) * (size_t)n * n);
  ld scale = sqrtl(2.0L / (ld)(n + 1));
  for (int j = 1; j <= n; ++j)
    for (int i = 1; i <= n; ++i) {
      long q = ((long)j * i) % (2L * (n + 1));
      S[(size_t)(j - 1) * n + (i - 1)] = scale * sinl(PI_C * (ld)q / (ld)(n + 1));
    }
  return S;
}

/* out = V in for one complex slice: the real V along every axis, O(n) sums per output */
static void cdst(const orc_problem* p, const ld* S, const lc* in, lc* out) {
  long n = p->n, N = cx_nmodes(p);
  lc* a = (lc*)malloc(sizeof(lc) * (size_t)N);
  lc* b = (lc*)malloc(sizeof(lc) * (size_t)N);
  memcpy(a, in, sizeof(lc) * (size_t)N);
  long stride = 1;
  for (int ax = 0; ax < p->dim; ++ax) {
    for (long base = 0; base < N; ++base) {
      long i_ax = (base / stride) % n;
      if (i_ax != 0) continue;  /* one line per (base with axis index 0) */
      for (long j = 0; j < n; ++j) {
        lc acc = 0.0L;
        for (long i = 0; i < n; ++i) acc += S[j * n + i] * a[base + i * stride];
        b[base + j * stride] = acc;
      }
    }
    memcpy(a, b, sizeof(lc) * (size_t)N);
    stride *= n;
  }
  memcpy(out, a, sizeof(lc) * (size_t)N);
  free(a);
  free(b);
}

/* out = A in, A = V diag(E) V = exp(dt L_h) */
static void capply_A(const orc_problem* p, const ld* S, const lc* E, const lc* in, lc* out) {
  long N = cx_nmodes(p);
  lc* t = (lc*)malloc(sizeof(lc) * (size_t)N);
  cdst(p, S, in, t);
  for (long J = 0; J < N; ++J) t[J] *= E[J];
  cdst(p, S, t, out);
  free(t);
}

static lc* load_c(const double* x, size_t len) {
  lc* z = (lc*)malloc(sizeof(lc) * len);
  for (size_t i = 0; i < len; ++i) z[i] = (ld)x[2 * i] + I * (ld)x[2 * i + 1];
  return z;
}
static void store_c(const lc* z, double* x, size_t len) {
  for (size_t i = 0; i < len; ++i) {
    x[2 * i] = (double)creall(z[i]);
    x[2 * i + 1] = (double)cimagl(z[i]);
  }
}

typedef struct {
  const orc_problem* p;
  long N;
  ld* S;
  lc* E;
} cctx;
static void cctx_init(cctx* c, const orc_problem* p) {
  c->p = p;
  c->N = cx_nmodes(p);
  c->S = sine_tab(p->n);
  c->E = (lc*)malloc(sizeof(lc) * (size_t)c->N);
  for (long J = 0; J < c->N; ++J) c->E[J] = mode_E(p, J);
}
static void cctx_free(cctx* c) {
  free(c->S);
  free(c->E);
}

/* u_n = A u_{n-1}, n = 1..Nt; scheme 3: exponential BDF2 (4.1)
   u_n = 4/3 A u_{n-1} - 1/3 A^2 u_{n-2} from u_1 = A u_0 (reading R16), U holding
   u_2 .. u_{Nt+1} */
void orc_cplx_sequential(const orc_problem* p, const double* u0, double* U) {
  cctx c;
  cctx_init(&c, p);
  size_t N = (size_t)c.N;
  lc* prev = load_c(u0, N);
  lc* cur = (lc*)malloc(sizeof(lc) * N);
  if (p->scheme == 3) {
    lc* um2 = (lc*)malloc(sizeof(lc) * N);
    lc* t1 = (lc*)malloc(sizeof(lc) * N);
    lc* t2 = (lc*)malloc(sizeof(lc) * N);
    memcpy(um2, prev, sizeof(lc) * N);
    capply_A(p, c.S, c.E, um2, prev); /* u_1 */
    for (int n = 2; n <= p->nt + 1; ++n) {
      capply_A(p, c.S, c.E, prev, cur);
      capply_A(p, c.S, c.E, um2, t1);
      capply_A(p, c.S, c.E, t1, t2);
      for (size_t i = 0; i < N; ++i) cur[i] = (4.0L / 3.0L) * cur[i] - (1.0L / 3.0L) * t2[i];
      store_c(cur, U + 2 * (size_t)(n - 2) * N, N);
      memcpy(um2, prev, sizeof(lc) * N);
      memcpy(prev, cur, sizeof(lc) * N);
    }
    free(um2); free(t1); free(t2); free(prev); free(cur);
    cctx_free(&c);
    return;
  }
  for (int n = 1; n <= p->nt; ++n) {
    capply_A(p, c.S, c.E, prev, cur);
    store_c(cur, U + 2 * (size_t)(n - 1) * N, N);
    memcpy(prev, cur, sizeof(lc) * N);
  }
  free(prev);
  free(cur);
  cctx_free(&c);
}

/* r_n = A u_{n-1} - u_n (f - Q U); scheme 3: r = f_2 - R v
   (PAPER.md:440-442): r_n = 4/3 A v_{n-1} - 1/3 A^2 v_{n-2} - v_n with v_0 = u_1 = A u_0,
   v_{-1} = u_0 */
static void cresidual(const cctx* c, const lc* u0, const lc* U, lc* R) {
  size_t N = (size_t)c->N;
  if (c->p->scheme == 3) {
    lc* u1 = (lc*)malloc(sizeof(lc) * N);
    capply_A(c->p, c->S, c->E, u0, u1);
#pragma omp parallel for schedule(dynamic, 1)
    for (int n = 1; n <= c->p->nt; ++n) {
      const lc* p1 = n == 1 ? u1 : U + (size_t)(n - 2) * N;
      const lc* p2 = n == 1 ? u0 : n == 2 ? u1 : U + (size_t)(n - 3) * N;
      lc* r = R + (size_t)(n - 1) * N;
      lc* t1 = (lc*)malloc(sizeof(lc) * N);
      lc* t2 = (lc*)malloc(sizeof(lc) * N);
      capply_A(c->p, c->S, c->E, p1, r);
      capply_A(c->p, c->S, c->E, p2, t1);
      capply_A(c->p, c->S, c->E, t1, t2);
      for (size_t i = 0; i < N; ++i)
        r[i] = (4.0L / 3.0L) * r[i] - (1.0L / 3.0L) * t2[i] - U[(size_t)(n - 1) * N + i];
      free(t1); free(t2);
    }
    free(u1);
    return;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int n = 1; n <= c->p->nt; ++n) {
    const lc* prev = n == 1 ? u0 : U + (size_t)(n - 2) * N;
    lc* r = R + (size_t)(n - 1) * N;
    capply_A(c->p, c->S, c->E, prev, r);
    for (size_t i = 0; i < N; ++i) r[i] -= U[(size_t)(n - 1) * N + i];
  }
}

/* (Q v)_n = v_n - A v_{n-1}, v_0 = 0; scheme 3: R v = v - 4/3 (C_0 (x) A) v + 1/3 (C_1 (x) A^2) v
    */
static void capply_Q(const cctx* c, const lc* V, lc* out) {
  size_t N = (size_t)c->N;
  if (c->p->scheme == 3) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int n = 1; n <= c->p->nt; ++n) {
      lc* o = out + (size_t)(n - 1) * N;
      lc* t1 = (lc*)malloc(sizeof(lc) * N);
      lc* t2 = (lc*)malloc(sizeof(lc) * N);
      memcpy(o, V + (size_t)(n - 1) * N, sizeof(lc) * N);
      if (n >= 2) {
        capply_A(c->p, c->S, c->E, V + (size_t)(n - 2) * N, t1);
        for (size_t i = 0; i < N; ++i) o[i] -= (4.0L / 3.0L) * t1[i];
      }
      if (n >= 3) {
        capply_A(c->p, c->S, c->E, V + (size_t)(n - 3) * N, t1);
        capply_A(c->p, c->S, c->E, t1, t2);
        for (size_t i = 0; i < N; ++i) o[i] += (1.0L / 3.0L) * t2[i];
      }
      free(t1); free(t2);
    }
    return;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int n = 1; n <= c->p->nt; ++n) {
    lc* o = out + (size_t)(n - 1) * N;
    if (n == 1) {
      memcpy(o, V, sizeof(lc) * N);
    } else {
      capply_A(c->p, c->S, c->E, V + (size_t)(n - 2) * N, o);
      for (size_t i = 0; i < N; ++i) o[i] = V[(size_t)(n - 1) * N + i] - o[i];
    }
  }
}

/* Steps (a)-(c) on a complex space-time vector */
static void cprecond(const cctx* c, const lc* R, lc* Sout) {
  const orc_problem* p = c->p;
  int nt = p->nt;
  size_t N = (size_t)c->N;
  lc* w = (lc*)malloc(sizeof(lc) * nt);
  ld* g = (ld*)malloc(sizeof(ld) * nt);
  for (int q = 0; q < nt; ++q) {
    w[q] = cexpl(I * 2.0L * PI_C * (ld)q / (ld)nt); /* omega^q, omega = e^{2 pi i/Nt} */
    g[q] = powl((ld)p->alpha, (ld)q / (ld)nt);
  }
  ld is = 1.0L / sqrtl((ld)nt);
  lc* Y = (lc*)malloc(sizeof(lc) * N * nt);
#pragma omp parallel for schedule(static)
  for (long x = 0; x < (long)N; ++x)
    for (int k = 0; k < nt; ++k) {
      lc acc = 0.0L;
      for (int m = 0; m < nt; ++m) acc += w[((long)k * m) % nt] * g[m] * R[(size_t)m * N + x];
      Y[(size_t)k * N + x] = is * acc;
    }
  ld a1 = powl((ld)p->alpha, 1.0L / (ld)nt);
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < nt; ++k) {
    lc* t = (lc*)malloc(sizeof(lc) * N);
    cdst(p, c->S, Y + (size_t)k * N, t);
    lc lam = a1 * w[k];
    if (p->scheme == 3) { /* BDF2 Step (b) of (4.5): 1 - 4/3 lambda_{0,k} E + 1/3 lambda_{1,k} E^2,
                             lambda_{1,k} = alpha^{2/Nt} omega^{2k} */
      lc lam1 = powl((ld)p->alpha, 2.0L / (ld)nt) * w[(2L * k) % nt];
      for (size_t J = 0; J < N; ++J)
        t[J] /= (1.0L - (4.0L / 3.0L) * lam * c->E[J] + (1.0L / 3.0L) * lam1 * c->E[J] * c->E[J]);
    } else {
      for (size_t J = 0; J < N; ++J) t[J] /= (1.0L - lam * c->E[J]); /* Step (b) */
    }
    cdst(p, c->S, t, Y + (size_t)k * N);
    free(t);
  }
#pragma omp parallel for schedule(static)
  for (long x = 0; x < (long)N; ++x)
    for (int m = 0; m < nt; ++m) {
      lc acc = 0.0L;
      for (int k = 0; k < nt; ++k) acc += conjl(w[((long)k * m) % nt]) * Y[(size_t)k * N + x];
      Sout[(size_t)m * N + x] = is * acc / g[m];
    }
  free(w);
  free(g);
  free(Y);
}

static ld rdot(const lc* a, const lc* b, size_t len) { /* Re <a, b>; rdot(a, a) = ||a||^2 */
  ld s = 0.0L;
  for (size_t i = 0; i < len; ++i) s += creall(a[i]) * creall(b[i]) + cimagl(a[i]) * cimagl(b[i]);
  return s;
}

void orc_cplx_residual(const orc_problem* p, const double* u0, const double* U, double* R, double* rnorm2) {
  cctx c;
  cctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  lc *u = load_c(u0, N), *Ul = load_c(U, tot), *Rl = (lc*)malloc(sizeof(lc) * tot);
  cresidual(&c, u, Ul, Rl);
  store_c(Rl, R, tot);
  if (rnorm2) *rnorm2 = (double)rdot(Rl, Rl, tot);
  free(u); free(Ul); free(Rl);
  cctx_free(&c);
}

void orc_cplx_precond(const orc_problem* p, const double* R, double* S) {
  cctx c;
  cctx_init(&c, p);
  size_t tot = (size_t)c.N * (size_t)p->nt;
  lc *Rl = load_c(R, tot), *Sl = (lc*)malloc(sizeof(lc) * tot);
  cprecond(&c, Rl, Sl);
  store_c(Sl, S, tot);
  free(Rl); free(Sl);
  cctx_free(&c);
}

void orc_cplx_apply_Q(const orc_problem* p, const double* V, double* out) {
  cctx c;
  cctx_init(&c, p);
  size_t tot = (size_t)c.N * (size_t)p->nt;
  lc *Vl = load_c(V, tot), *O = (lc*)malloc(sizeof(lc) * tot);
  capply_Q(&c, Vl, O);
  store_c(O, out, tot);
  free(Vl); free(O);
  cctx_free(&c);
}

/* Richardson (3.2), zero initial guess, the stop of reading R8 */
int orc_cplx_fixed_point(const orc_problem* p, const double* u0, double* U, double tol, int maxit, double* hist,
                         int* iterations) {
  cctx c;
  cctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  lc *u = load_c(u0, N), *Ul = load_c(U, tot);
  lc *R = (lc*)malloc(sizeof(lc) * tot), *S = (lc*)malloc(sizeof(lc) * tot);
  ld r0 = 0.0L;
  int status = 7, k;
  for (k = 0; k <= maxit; ++k) {
    cresidual(&c, u, Ul, R);
    ld rn = sqrtl(rdot(R, R, tot));
    if (k == 0) r0 = rn;
    ld rho = r0 > 0.0L ? rn / r0 : 0.0L;
    if (hist) hist[k] = (double)rho;
    cprecond(&c, R, S);
    for (size_t i = 0; i < tot; ++i) Ul[i] += S[i];
    if (rho < (ld)tol) { status = 0; break; }
  }
  if (iterations) *iterations = status == 0 ? k : maxit;
  store_c(Ul, U, tot);
  free(u); free(Ul); free(R); free(S);
  cctx_free(&c);
  return status;
}

/* Hermitian inner product <a, b> = sum conj(a_i) b_i (complex GMRES, reading R18) */
static lc cdot(const lc* a, const lc* b, size_t len) {
  lc s = 0.0L;
  for (size_t i = 0; i < len; ++i) s += conjl(a[i]) * b[i];
  return s;
}

/* left-preconditioned GMRES(m) over C (the paper's MATLAB gmres on complex vectors,
   PAPER.md:983), CGS2 with the Hermitian inner product, complex Givens rotations,
   x0 = U (reading R11) */
int orc_cplx_gmres(const orc_problem* p, const double* u0, double* U, double tol, int restart, int maxit,
                   double* hist, int* iterations) {
  if (restart < 1) restart = 1;
  cctx c;
  cctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  int m = restart;
  lc *u = load_c(u0, N), *x = load_c(U, tot);
  lc *r = (lc*)malloc(sizeof(lc) * tot), *w = (lc*)malloc(sizeof(lc) * tot), *t = (lc*)malloc(sizeof(lc) * tot);
  lc** V = (lc**)calloc((size_t)m + 1, sizeof(lc*));
  lc* H = (lc*)calloc((size_t)(m + 1) * m, sizeof(lc));
  ld* cs = (ld*)calloc((size_t)m, sizeof(ld));
  lc* sn = (lc*)calloc((size_t)m, sizeof(lc));
  lc *g = (lc*)calloc((size_t)m + 1, sizeof(lc)), *y = (lc*)calloc((size_t)m, sizeof(lc));
  lc *h = (lc*)calloc((size_t)m + 1, sizeof(lc)), *h2 = (lc*)calloc((size_t)m + 1, sizeof(lc));
  int its = 0, status = 7;
  ld beta0 = -1.0L;
  if (hist) hist[0] = 1.0;
  while (its < maxit) {
    cresidual(&c, u, x, t);
    cprecond(&c, t, r);
    ld beta = sqrtl(rdot(r, r, tot));
    if (beta0 < 0.0L) beta0 = beta;
    if (beta0 == 0.0L || beta / beta0 < (ld)tol) { status = 0; break; }
    if (!V[0]) V[0] = (lc*)malloc(sizeof(lc) * tot);
    for (size_t i = 0; i < tot; ++i) V[0][i] = r[i] / beta;
    for (int i = 0; i <= m; ++i) g[i] = 0.0L;
    g[0] = beta;
    int j, done = 0;
    for (j = 0; j < m && its < maxit; ++j) {
      capply_Q(&c, V[j], t);
      cprecond(&c, t, w);
      for (int pass = 0; pass < 2; ++pass) {
        lc* hh = pass == 0 ? h : h2;
        for (int i = 0; i <= j; ++i) hh[i] = cdot(V[i], w, tot);
        for (int i = 0; i <= j; ++i)
          for (size_t q = 0; q < tot; ++q) w[q] -= hh[i] * V[i][q];
      }
      for (int i = 0; i <= j; ++i) H[i * m + j] = h[i] + h2[i];
      ld hn = sqrtl(rdot(w, w, tot));
      H[(j + 1) * m + j] = hn;
      for (int i = 0; i < j; ++i) { /* [c s; -conj(s) c] */
        lc a = H[i * m + j], b = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * b;
        H[(i + 1) * m + j] = -conjl(sn[i]) * a + cs[i] * b;
      }
      lc a = H[j * m + j];
      ld b = hn, aa = cabsl(a), den = sqrtl(aa * aa + b * b);
      if (den == 0.0L) { cs[j] = 1.0L; sn[j] = 0.0L; }
      else if (aa == 0.0L) { cs[j] = 0.0L; sn[j] = 1.0L; }
      else { cs[j] = aa / den; sn[j] = (a / aa) * b / den; }
      H[j * m + j] = cs[j] * a + sn[j] * b;
      H[(j + 1) * m + j] = 0.0L;
      g[j + 1] = -conjl(sn[j]) * g[j];
      g[j] = cs[j] * g[j];
      ++its;
      ld rel = cabsl(g[j + 1]) / beta0;
      if (hist) hist[its] = (double)rel;
      if (rel < (ld)tol || hn == 0.0L) { done = 1; ++j; break; }
      if (!V[j + 1]) V[j + 1] = (lc*)malloc(sizeof(lc) * tot);
      if (j + 1 < m)
        for (size_t q = 0; q < tot; ++q) V[j + 1][q] = w[q] / hn;
    }
    for (int i = j - 1; i >= 0; --i) {
      lc acc = g[i];
      for (int l = i + 1; l < j; ++l) acc -= H[i * m + l] * y[l];
      y[i] = acc / H[i * m + i];
    }
    for (int i = 0; i < j; ++i)
      for (size_t q = 0; q < tot; ++q) x[q] += y[i] * V[i][q];
    if (done) { status = 0; break; }
  }
  if (iterations) *iterations = its;
  store_c(x, U, tot);
  for (int i = 0; i <= m; ++i) free(V[i]);
  free(V); free(H); free(cs); free(sn); free(g); free(y); free(h); free(h2);
  free(u); free(x); free(r); free(w); free(t);
  cctx_free(&c);
  return status;
}

/* left-preconditioned BiCGStab over C (reading R17 with the Hermitian inner product of
   R18): the same steps as orc_bicgstab with rho = <r-hat, r>, alpha = rho / <r-hat, v>,
   omega = <t, s> / <t, t>, <v, w> = sum conj(v) w */
int orc_cplx_bicgstab(const orc_problem* p, const double* u0, double* U, double tol, int maxit, double* hist,
                      int* iterations) {
  cctx c;
  cctx_init(&c, p);
  size_t N = (size_t)c.N, tot = N * (size_t)p->nt;
  lc *u = load_c(u0, N), *x = load_c(U, tot);
  lc *r = (lc*)malloc(sizeof(lc) * tot), *rh = (lc*)malloc(sizeof(lc) * tot);
  lc *pv = (lc*)calloc(tot, sizeof(lc)), *v = (lc*)calloc(tot, sizeof(lc));
  lc *s = (lc*)malloc(sizeof(lc) * tot), *t = (lc*)malloc(sizeof(lc) * tot), *w = (lc*)malloc(sizeof(lc) * tot);
  cresidual(&c, u, x, w); /* f - Q x */
  cprecond(&c, w, r);     /* r_0 */
  memcpy(rh, r, sizeof(lc) * tot);
  ld beta0 = sqrtl(rdot(r, r, tot));
  if (hist) hist[0] = 1.0;
  int status = 7, its = 0;
  lc rho_prev = 1.0L, al = 1.0L, om = 1.0L;
  if (beta0 == 0.0L) status = 0;
  for (int i = 0; status != 0 && i < maxit; ++i) {
    lc rho = cdot(rh, r, tot);
    lc beta = (rho / rho_prev) * (al / om);
    for (size_t q = 0; q < tot; ++q) pv[q] = r[q] + beta * (pv[q] - om * v[q]);
    capply_Q(&c, pv, w);
    cprecond(&c, w, v); /* v = Q_a^{-1} Q p */
    al = rho / cdot(rh, v, tot);
    for (size_t q = 0; q < tot; ++q) s[q] = r[q] - al * v[q];
    ld sn = sqrtl(rdot(s, s, tot));
    if (sn / beta0 < (ld)tol) { /* half step */
      for (size_t q = 0; q < tot; ++q) x[q] += al * pv[q];
      its = i + 1;
      if (hist) hist[its] = (double)(sn / beta0);
      status = 0;
      break;
    }
    capply_Q(&c, s, w);
    cprecond(&c, w, t); /* t = Q_a^{-1} Q s */
    om = cdot(t, s, tot) / rdot(t, t, tot);
    for (size_t q = 0; q < tot; ++q) {
      x[q] += al * pv[q] + om * s[q];
      r[q] = s[q] - om * t[q];
    }
    rho_prev = rho;
    its = i + 1;
    ld rn = sqrtl(rdot(r, r, tot));
    if (hist) hist[its] = (double)(rn / beta0);
    if (rn / beta0 < (ld)tol) { status = 0; break; }
  }
  if (iterations) *iterations = its;
  store_c(x, U, tot);
  free(u); free(x); free(r); free(rh); free(pv); free(v); free(s); free(t); free(w);
  cctx_free(&c);
  return status;
}
