// Misclustering correction and layer edits:
//
//   k_flood_*     4-connected flood fill over pixels of one cluster id from a
//                 seed mask (correction.py:54-68), as repeated dilation of the
//                 frontier on the device; the host checks a mapped "changed"
//                 flag every kFloodBatch steps
//   k_recompose   R' * (T . B') recomposition of the edits (editing.py:24-74):
//                 per-channel reflectance ratio on one cluster, a modified
//                 palette matrix, clip to [0, 1], optional matte / background
//
// fp64 per pixel (the reference computes the edits in float64 numpy).
#include "ls_kernels.h"

namespace ls {

static inline int grid_of(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 8 * 148 * 4) b = 8 * 148 * 4;
  return (int)b;
}

__global__ void k_flood_init(const int32_t* __restrict__ ids, int target, const uint8_t* __restrict__ seeds,
                             int64_t N, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = (seeds[i] && ids[i] == target) ? 1 : 0;
}

// one dilation step restricted to the target id; *changed |= any growth
__global__ void k_flood_step(const int32_t* __restrict__ ids, int target, int H, int W,
                             const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int* changed) {
  const int64_t N = (int64_t)H * W;
  bool grew = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % W), y = (int)(i / W);
    uint8_t m = in[i];
    if (!m && ids[i] == target) {
      const bool nb = (x > 0 && in[i - 1]) || (x < W - 1 && in[i + 1]) || (y > 0 && in[i - W]) ||
                      (y < H - 1 && in[i + W]);
      if (nb) {
        m = 1;
        grew = true;
      }
    }
    out[i] = m;
  }
  if (__syncthreads_or(grew) && threadIdx.x == 0) *changed = 1;
}

__global__ void k_flag(int* f, int v) { *f = v; }

void launch_flood_init(cudaStream_t s, const int32_t* ids, int target, const uint8_t* seeds, int64_t N,
                       uint8_t* mask) {
  k_flood_init<<<grid_of(N), 256, 0, s>>>(ids, target, seeds, N, mask);
}
void launch_flood_step(cudaStream_t s, const int32_t* ids, int target, int H, int W, const uint8_t* in,
                       uint8_t* out, int* changed) {
  k_flood_step<<<grid_of((int64_t)H * W), 256, 0, s>>>(ids, target, H, W, in, out, changed);
}
void launch_set_flag(cudaStream_t s, int* f, int v) { k_flag<<<1, 1, 0, s>>>(f, v); }

__global__ void k_recompose(const float* __restrict__ X, int NT, int64_t N, const EditParams P,
                            const int32_t* __restrict__ ids, const uint8_t* __restrict__ matte,
                            const float* __restrict__ bg, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (matte && matte[i]) {
      for (int c = 0; c < 3; ++c) out[3 * i + c] = bg[3 * i + c];
      continue;
    }
    const bool sel = ids && P.k >= 1 && ids[i] == P.k;
    double S[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < NT; ++k) {
      const double t = (double)X[(3 + k) * N + i];
      for (int c = 0; c < 3; ++c) S[c] += t * P.B[3 * k + c];
    }
    for (int c = 0; c < 3; ++c) {
      double R = exp((double)X[c * N + i]);
      if (sel) R *= P.ratio[c];
      const double v = R * S[c];
      out[3 * i + c] = (float)(v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v));
    }
  }
}

void launch_recompose(cudaStream_t s, const float* X, int NT, int64_t N, const EditParams& P, const int32_t* ids,
                      const uint8_t* matte, const float* bg, float* out) {
  k_recompose<<<grid_of(N), 256, 0, s>>>(X, NT, N, P, ids, matte, bg, out);
}

}  // namespace ls
