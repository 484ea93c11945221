// Probe of TMA tensor-load configurations on B200 (debugging aid): each case loads one box
// into shared memory, waits on its mbarrier with a time bound and reports ok / timeout
// and the first loaded values.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2603_04350_b200/csrc/tma_dev.cuh"
using namespace expd;

__device__ bool wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint64_t t0 = global_ns();
  while (!mbar_try_wait(bar, parity))
    if (global_ns() - t0 > 500000000ull) return false;
  return true;
}

__global__ void probe(const __grid_constant__ CUtensorMap map, int rank, int c0, int c1, int c2, int c3,
                      unsigned bytes, double* out, int* status) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, bytes);
    if (rank == 2) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(smem_u32(sm)), "l"(&map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
    } else if (rank == 3) {
      tma_load_3d(sm, &map, bar, c0, c1, c2);
    } else {
      tma_load_4d(sm, &map, bar, c0, c1, c2, c3);
    }
    bool ok = wait_bounded(bar, 0);
    *status = ok ? 1 : 0;
    const double* d = reinterpret_cast<const double*>(sm);
    for (int i = 0; i < 8; ++i) out[i] = d[i];
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  printf("encode fn %p q=%d\n", p, (int)q);
  const int M = 256, n = 255, ns = 2;
  std::vector<double> h((size_t)M * n * ns);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double* d;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  double* dout;
  int* dst;
  cudaMalloc(&dout, 64);
  cudaMalloc(&dst, 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  struct Case { const char* name; int rank; cuuint64_t dim[4]; cuuint64_t str[3]; cuuint32_t box[4]; int sw; int c[4]; };
  Case cases[] = {
    {"2d box{2,128}", 2, {M, (cuuint64_t)n}, {M * 8}, {2, 128}, 0, {0, 0}},
    {"2d box{2,256} (> rows)", 2, {M, (cuuint64_t)n}, {M * 8}, {2, 256}, 0, {0, 0}},
    {"2d box{16,16}", 2, {M, (cuuint64_t)n}, {M * 8}, {16, 16}, 0, {0, 0}},
    {"3d box{2,128,1}", 3, {M, (cuuint64_t)n, ns}, {M * 8, (cuuint64_t)M * n * 8}, {2, 128, 1}, 0, {0, 0, 1}},
    {"4d box{2,128,1,1} nz=1", 4, {M, (cuuint64_t)n, 1, ns}, {M * 8, (cuuint64_t)M * n * 8, (cuuint64_t)M * n * 8}, {2, 128, 1, 1}, 0, {0, 0, 0, 1}},
    {"4d box{2,256,1,1} nz=1", 4, {M, (cuuint64_t)n, 1, ns}, {M * 8, (cuuint64_t)M * n * 8, (cuuint64_t)M * n * 8}, {2, 256, 1, 1}, 0, {0, 0, 0, 1}},
    {"4d row sw128 {16,16,1,1}", 4, {16, M / 16, (cuuint64_t)n, ns}, {128, M * 8, (cuuint64_t)M * n * 8}, {16, M / 16, 1, 1}, 1, {0, 0, 3, 1}},
  };
  for (auto& c : cases) {
    CUtensorMap map;
    const cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, c.rank, d, c.dim, c.str, c.box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned bytes = 8;
    for (int i = 0; i < c.rank; ++i) bytes *= c.box[i];
    int st = -1;
    double o[8] = {0};
    cudaMemset(dst, 0xff, 4);
    if (r == CUDA_SUCCESS) {
      probe<<<1, 32, 65536 + 64>>>(map, c.rank, c.c[0], c.c[1], c.c[2], c.c[3], bytes, dout, dst);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(o, dout, 64, cudaMemcpyDeviceToHost);
      printf("%-28s encode=%d bytes=%u status=%d err=%s vals %.0f %.0f %.0f %.0f %.0f\n", c.name, (int)r, bytes, st,
             cudaGetErrorString(e), o[0], o[1], o[2], o[3], o[4]);
    } else {
      printf("%-28s encode FAILED %d\n", c.name, (int)r);
    }
  }
  return 0;
}
