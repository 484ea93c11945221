// k_time_n16.cu -- the K1 instantiations for Nt = 16 (one translation unit per Nt so that
// nvcc builds the time-FFT variants in parallel; the kernels are in k_time.cuh).
#include "k_time.cuh"

namespace expd {
cudaError_t dispatch_time_n16(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st) {
  return dispatch_nt<16>(a, rm, om, nl, grid, st);
}
}  // namespace expd
