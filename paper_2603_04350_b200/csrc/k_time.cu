// k_time.cu -- K1 dispatch over Nt (the kernels are in k_time.cuh, instantiated per Nt in
// k_time_n<Nt>.cu), the persistent-grid sizing and the residual-only kernel.
#include "k_time.cuh"

namespace expd {

cudaError_t dispatch_time_n4(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);
cudaError_t dispatch_time_n8(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);
cudaError_t dispatch_time_n16(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);
cudaError_t dispatch_time_n32(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);
cudaError_t dispatch_time_n64(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);
cudaError_t dispatch_time_n128(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);
cudaError_t dispatch_time_n256(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st);

cudaError_t launch_time_fused(const TimeArgs& a, int rmode, int outmode, int nl, int grid, cudaStream_t st) {
  switch (a.nt) {
    case 4: return dispatch_time_n4(a, rmode, outmode, nl, grid, st);
    case 8: return dispatch_time_n8(a, rmode, outmode, nl, grid, st);
    case 16: return dispatch_time_n16(a, rmode, outmode, nl, grid, st);
    case 32: return dispatch_time_n32(a, rmode, outmode, nl, grid, st);
    case 64: return dispatch_time_n64(a, rmode, outmode, nl, grid, st);
    case 128: return dispatch_time_n128(a, rmode, outmode, nl, grid, st);
    case 256: return dispatch_time_n256(a, rmode, outmode, nl, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

// Persistent grid: a fixed multiple of the SM count (deterministic partial order), capped
// by the number of tiles.
// tiles per CTA-slot of the TMA variant: (pairs per tile, resident CTAs per SM)
template <int NT>
static void tma_shape(int nl, int& S, int& per_sm, long npairs) {
  if constexpr (ring_capable<NT>()) {
    if (use_ring<NT>(npairs)) {  // one 512-thread CTA per SM
      S = RingLayout<NT, 1>::S;
      per_sm = 1;
      return;
    }
  }
  if (k1_variant(NT) == 1282) {
    S = TmaLayout<NT, 128, 1, 2>::S;
    per_sm = nl ? TmaLayout<NT, 128, 1, 2>::MINB : TmaLayout<NT, 128, 0, 2>::MINB;
  } else if (k1_variant(NT) == 2561) {
    S = TmaLayout<NT, 256, 1, 1>::S;
    per_sm = nl ? TmaLayout<NT, 256, 1, 1>::MINB : TmaLayout<NT, 256, 0, 1>::MINB;
  } else {
    S = TmaLayout<NT, 256, 1, 2>::S;
    per_sm = nl ? TmaLayout<NT, 256, 1, 2>::MINB : TmaLayout<NT, 256, 0, 2>::MINB;
  }
}

// Persistent grid: a fixed multiple of the SM count (deterministic partial order), capped
// by the number of tiles.  nl: the plan's heaviest K1 variant (N-hat staged too).
int time_fused_grid(int nt, long npairs, int sms, int nl) {
  int S = 32, per_sm = EXPD_K1_MINB;
  switch (nt) {
    case 4: S = TimeGeo<4>::S; break;
    case 8: S = TimeGeo<8>::S; break;
    case 16: S = TimeGeo<16>::S; break;
    case 32: S = TimeGeo<32>::S; break;
    case 64: S = TimeGeo<64>::S; break;
    case 128: S = TimeGeo<128>::S; break;
    default: S = TimeGeo<256>::S;
  }
  if (nt >= 16 && use_pipe()) per_sm = pipe_mode() == 1 ? 1 : 2;
  if (nt >= 16 && pipe_mode() == 3) {
    switch (nt) {
      case 16: tma_shape<16>(nl, S, per_sm, npairs); break;
      case 32: tma_shape<32>(nl, S, per_sm, npairs); break;
      case 64: tma_shape<64>(nl, S, per_sm, npairs); break;
      case 128: tma_shape<128>(nl, S, per_sm, npairs); break;
      default: tma_shape<256>(nl, S, per_sm, npairs);
    }
  }
  long ntiles = (npairs + S - 1) / S;
  long g = (long)sms * per_sm;
  return (int)(ntiles < g ? (ntiles > 0 ? ntiles : 1) : g);
}

// ---------------------------------------------------------------------------------------
// residual only (expd_residual): r_t = E u_{t-1} + C1 N_t - C2 N_{t-1} - u_t, spectral.
// ---------------------------------------------------------------------------------------
template <int NL>
__global__ void __launch_bounds__(256) k_resid_only(const TimeArgs a) {
  const long total = (long)a.nt * a.npairs;
  double nrm = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int t = (int)(i / a.npairs);
    const long base = 2 * (i % a.npairs);
    double2 E = ld2(a.E + base);
    double2 cur = ld2(a.X + (long)t * a.npad + base);
    double2 prev = t > 0 ? ld2(a.X + (long)(t - 1) * a.npad + base) : ld2(a.u0h + base);
    double2 r = make_double2(fma(E.x, prev.x, -cur.x), fma(E.y, prev.y, -cur.y));
    if constexpr (NL == 4) r = csub(cmul(E, prev), cur);  // complex mode: E z_{t-1} - z_t
    if constexpr (K1Form<NL>::BDF) {  // BDF2: f2 - R v (NL 5: complex)
      const double2 zero = make_double2(0.0, 0.0);
      const double2 xm2 = t >= 2 ? ld2(a.X + (long)(t - 2) * a.npad + base) : zero;
      r = bdf2_form<true, K1Form<NL>::CX>(E, cur, t >= 1 ? prev : zero, xm2, ld2(a.u0h + base), t);
    }
    if constexpr (K1Form<NL>::HASN) {
      double2 c1 = ld2(a.C1 + base), nm1 = ld2(a.Nh + (long)t * a.npad + base);
      r.x = fma(c1.x, nm1.x, r.x);
      r.y = fma(c1.y, nm1.y, r.y);
      if constexpr (NL == 2) {
        double2 c2 = ld2(a.C2 + base), nm2 = ld2(a.Nh + (long)(t > 0 ? t - 1 : 0) * a.npad + base);
        r.x = fma(-c2.x, nm2.x, r.x);
        r.y = fma(-c2.y, nm2.y, r.y);
      }
    }
    nrm = fma(r.x, r.x, fma(r.y, r.y, nrm));
    st2(a.Y + (long)t * a.npad + base, r);
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0 && a.partial) a.partial[blockIdx.x] = v;
  }
}

cudaError_t launch_resid_only(const TimeArgs& a, int nl, int grid, cudaStream_t st) {
  if (nl == 0) k_resid_only<0><<<grid, 256, 0, st>>>(a);
  else if (nl == 1) k_resid_only<1><<<grid, 256, 0, st>>>(a);
  else if (nl == 3) k_resid_only<3><<<grid, 256, 0, st>>>(a);
  else if (nl == 4) k_resid_only<4><<<grid, 256, 0, st>>>(a);
  else if (nl == 5) k_resid_only<5><<<grid, 256, 0, st>>>(a);
  else k_resid_only<2><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace expd
