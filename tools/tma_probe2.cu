// Probe: struct-of-maps __grid_constant__ param + prefetch + 3 boxes on one mbarrier.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1908_01961_b200/csrc/ls_common.cuh"
using namespace ls;
struct M3 { CUtensorMap a, b, c; };

template <int PREF>
__global__ void k3(const __grid_constant__ M3 m, float* out, int n1, int n2, int n3) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); fence_barrier_init();
    if (PREF) { tma_prefetch_desc(&m.a); tma_prefetch_desc(&m.b); tma_prefetch_desc(&m.c); }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, (n1 + n2 + n3) * 4);
    tma_load_3d(sm, &m.a, &bar, 1, 1, 0);
    tma_load_3d(sm + n1, &m.b, &bar, 1, 1, 0);
    tma_load_3d(sm + n1 + n2, &m.c, &bar, 1, 1, 0);
  }
  mbar_wait(&bar, 0);
  for (int e = threadIdx.x; e < n1 + n2 + n3; e += blockDim.x) out[e] = sm[e];
}

template <int MODE>
__global__ void kx(const __grid_constant__ CUtensorMap a, const __grid_constant__ CUtensorMap b,
                   const __grid_constant__ CUtensorMap c, const __grid_constant__ M3 m, float* out, int n1, int n2, int n3) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (MODE == 0) {  // struct, only first map
      mbar_expect_tx(&bar, n1 * 4);
      tma_load_3d(sm, &m.a, &bar, 1, 1, 0);
    } else if (MODE == 1) {  // separate params, three loads
      mbar_expect_tx(&bar, (n1 + n2 + n3) * 4);
      tma_load_3d(sm, &a, &bar, 1, 1, 0);
      tma_load_3d(sm + n1, &b, &bar, 1, 1, 0);
      tma_load_3d(sm + n1 + n2, &c, &bar, 1, 1, 0);
    } else if (MODE == 2) {  // separate params, only a
      mbar_expect_tx(&bar, n1 * 4);
      tma_load_3d(sm, &a, &bar, 1, 1, 0);
    } else if (MODE == 3) {  // only c (48x22x3)
      mbar_expect_tx(&bar, n3 * 4);
      tma_load_3d(sm, &c, &bar, 1, 1, 0);
    } else if (MODE == 4) {  // only b
      mbar_expect_tx(&bar, n2 * 4);
      tma_load_3d(sm, &b, &bar, 1, 1, 0);
    }
  }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) out[0] = sm[0];
}

__global__ void kg(const M3* __restrict__ gm, float* out, int n1, int n2, int n3, int nl) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, (n1 + (nl > 1 ? n2 : 0) + (nl > 2 ? n3 : 0)) * 4);
    tma_load_3d(sm, &gm->a, &bar, 1, 1, 0);
    if (nl > 1) tma_load_3d(sm + n1, &gm->b, &bar, 1, 1, 0);
    if (nl > 2) tma_load_3d(sm + n1 + n2, &gm->c, &bar, 1, 1, 0);
  }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) out[0] = sm[0];
}

__global__ void k1p(const __grid_constant__ CUtensorMap a, float* out, int n1) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, n1 * 4); tma_load_3d(sm, &a, &bar, 1, 1, 0); }
  mbar_wait(&bar, 0);
  if (threadIdx.x == 0) out[0] = sm[0];
}

int main(int argc, char** argv) {
  int v = atoi(argv[1]);
  const int W = argc > 2 ? atoi(argv[2]) : 40, H = argc > 3 ? atoi(argv[3]) : 33, P = 9;
  float *d, *o; cudaMalloc(&d, W * H * P * 4); cudaMalloc(&o, 1 << 20); cudaMemset(d, 0, W * H * P * 4);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  M3 m;
  auto enc = [&](CUtensorMap* t, float* base, int planes, int bw, int bh) {
    cuuint64_t dims[3] = {W, H, (cuuint64_t)planes}; cuuint64_t str[2] = {W * 4, W * H * 4};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)planes}, es[3] = {1, 1, 1};
    return (int)fn(t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  int r1 = enc(&m.a, d, 9, 36, 10), r2 = enc(&m.b, d + 3 * W * H, 6, 36, 10), r3 = enc(&m.c, d, 3, 48, 22);
  int n1 = 9 * 360, n2 = 6 * 360, n3 = 3 * 1056;
  if (v == 1) { n1 = (n1 + 31) & ~31; n2 = (n2 + 31) & ~31; }   // 128B-aligned destinations
  size_t smem = (n1 + n2 + n3) * 4 + 1024;
  cudaFuncSetAttribute(k3<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k3<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  n1 = (n1 + 31) & ~31; n2 = (n2 + 31) & ~31;
  cudaFuncSetAttribute(kx<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kx<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kx<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kx<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kx<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  M3* gm; cudaMalloc(&gm, sizeof(M3)); cudaMemcpy(gm, &m, sizeof(M3), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k1p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (v >= 20 && v <= 22) kg<<<1, 256, smem>>>(gm, o, n1, n2, n3, v - 19);
  if (v == 23) k1p<<<1, 256, smem>>>(m.a, o, n1);
  if (v == 10) kx<0><<<1, 256, smem>>>(m.a, m.b, m.c, m, o, n1, n2, n3);
  if (v == 11) kx<1><<<1, 256, smem>>>(m.a, m.b, m.c, m, o, n1, n2, n3);
  if (v == 12) kx<2><<<1, 256, smem>>>(m.a, m.b, m.c, m, o, n1, n2, n3);
  if (v == 13) kx<3><<<1, 256, smem>>>(m.a, m.b, m.c, m, o, n1, n2, n3);
  if (v == 14) kx<4><<<1, 256, smem>>>(m.a, m.b, m.c, m, o, n1, n2, n3);
  printf("v%d enc %d %d %d: %s\n", v, r1, r2, r3, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
