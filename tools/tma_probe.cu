// Standalone probe of TMA / mbarrier usage; argv[1] selects one variant per process.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1908_01961_b200/csrc/ls_common.cuh"
using namespace ls;

__global__ void k_mbar_only(float* out) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) mbar_expect_tx(&bar, 0);
  mbar_wait(&bar, 0);
  out[threadIdx.x] = 1.f;
}

__global__ void k_tma(const __grid_constant__ CUtensorMap m, float* out, int n, int c0, int c1, int dim3d) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, n * 4);
    if (dim3d) tma_load_3d(sm, &m, &bar, c0, c1, 0);
    else asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                      ::"r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(smem_u32(&bar)), "r"(c0), "r"(c1) : "memory");
  }
  mbar_wait(&bar, 0);
  for (int e = threadIdx.x; e < n; e += blockDim.x) out[e] = sm[e];
}

int main(int argc, char** argv) {
  int v = atoi(argv[1]);
  float* o; cudaMalloc(&o, 1 << 20);
  if (v == 0) {
    k_mbar_only<<<1, 128>>>(o);
    printf("mbar only: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
  }
  const int W = 24, H = 20, P = argc > 6 ? atoi(argv[6]) : 7;
  std::vector<float> h(W * H * P);
  for (int i = 0; i < (int)h.size(); ++i) h[i] = (float)i;
  float* d; cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  int bw = 8, bh = 8, bp = P, c0 = 0, c1 = 0, rank = 3;
  if (v == 1) { rank = 2; bp = 1; }                 // 2-D, in-bounds box
  if (v == 2) { }                                   // 3-D in-bounds box 8x8x7
  if (v == 3) { c0 = -1; c1 = -1; }                 // 3-D negative start
  if (v == 4) { bw = 36; bh = 10; c0 = -1; c1 = -1; }  // the solver's box
  if (v == 9) { bw = atoi(argv[2]); bh = atoi(argv[3]); c0 = atoi(argv[4]); c1 = atoi(argv[5]); }
  cuuint64_t dims[3] = {W, H, P}; cuuint64_t str[2] = {W * 4, W * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bp}, es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int n = bw * bh * bp;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int nthr = argc > 7 ? atoi(argv[7]) : 128;
  k_tma<<<1, nthr, n * 4 + (argc > 8 ? atoi(argv[8]) : 0)>>>(m, o, n, c0, c1, rank == 3);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> ho(n);
  int bad = -1;
  if (e == cudaSuccess) {
    cudaMemcpy(ho.data(), o, n * 4, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int pp = 0; pp < bp; ++pp) for (int y = 0; y < bh; ++y) for (int x = 0; x < bw; ++x) {
      int gx = x + c0, gy = y + c1;
      float want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[pp * W * H + gy * W + gx] : 0.f;
      if (ho[pp * bw * bh + y * bw + x] != want) ++bad;
    }
  }
  printf("variant %d encode %d: %s mismatches %d\n", v, (int)r, cudaGetErrorString(e), bad);
  return 0;
}
