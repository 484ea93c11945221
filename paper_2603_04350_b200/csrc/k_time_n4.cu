// k_time_n4.cu -- the K1 instantiations for Nt = 4 (one translation unit per Nt so that
// nvcc builds the time-FFT variants in parallel; the kernels are in k_time.cuh).
#include "k_time.cuh"

namespace expd {
cudaError_t dispatch_time_n4(const TimeArgs& a, int rm, int om, int nl, int grid, cudaStream_t st) {
  return dispatch_nt<4>(a, rm, om, nl, grid, st);
}
}  // namespace expd
