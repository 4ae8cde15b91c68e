// Per-block residual protocol (reference energy.py:194-452): residual,
// apply_j, apply_jt (accumulating) and add_diag (accumulating) of each of the
// eight residual blocks, with IRLS weights / linearisation frozen at X0.
//
// This is the reference's block-level API (assemble_blocks returns the eight
// blocks, energy.py:478-496; stack_residuals concatenates their residuals,
// :499-500) for callers and tests that work block by block -- J against
// finite differences, J/J^T adjointness, diag against the explicit normal
// matrix (test_energy.py:285-321).  The solver itself never materialises a
// residual: it runs the fused kernels of ls_solver.cu.  These kernels are
// plain grid-stride loops in fp64 arithmetic over fp32 planar inputs.
//
// Row orders are the reference's (H, W, C) ravel of each block's residual:
//   data / clustering / monochrome  3N     row 3i + c
//   r_sparsity                      6N     x rows 3i + c, then y rows 3N + 3i + c
//   r_consistency                   3P     row 3j + c of pair j
//   i_sparsity                      K N    row K i + (k - 1), k = 1..K
//   smoothness                      2 NT N x rows NT i + k, then y rows NT N + NT i + k
//   non_neg                         NT N   row NT i + k
#include "ls_common.cuh"
#include "ls_kernels.h"

namespace ls {

namespace {

struct BlkCtx {
  Frame f;
  Coef<double> c;
  const float* X0;   // linearisation point, U planes
  BlockPairs pairs;
};

__device__ __forceinline__ double x0(const BlkCtx& b, int plane, int64_t i) {
  return (double)b.X0[(int64_t)plane * b.f.N + i];
}

__device__ __forceinline__ double S_of(const BlkCtx& b, const float* Y, int64_t i, int ch) {
  double s = 0.0;
  for (int k = 0; k < b.f.NT; ++k) s += (double)Y[(int64_t)(3 + k) * b.f.N + i] * b.c.B[k][ch];
  return s;
}

__device__ __forceinline__ double anchor_of(const BlkCtx& b, int64_t i, int ch) {
  if (b.f.ids) return b.c.anchor[b.f.ids[i]][ch];
  return (double)b.f.anchor[(int64_t)ch * b.f.N + i];
}

// sqrt of the r-sparsity weight at pixel (x, y) (energy.py:301-305)
__device__ __forceinline__ double a_rs(const BlkCtx& b, int x, int y) {
  const int W = b.f.W, H = b.f.H;
  const int64_t i = (int64_t)y * W + x;
  double s = 0.0;
  for (int ch = 0; ch < 3; ++ch) {
    const double v = x0(b, ch, i);
    const double gx = x < W - 1 ? x0(b, ch, i + 1) - v : 0.0;
    const double gy = y < H - 1 ? x0(b, ch, i + W) - v : 0.0;
    s += gx * gx + gy * gy;
  }
  return sqrt(b.c.lam_rs * irlsp(sqrt(s), b.c));
}

// sqrt of the smoothness weights of layer k at (x, y) (energy.py:314-318)
__device__ __forceinline__ double a_smx(const BlkCtx& b, int k, int x, int y) {
  const int64_t i = (int64_t)y * b.f.W + x;
  const double g = x < b.f.W - 1 ? x0(b, 3 + k, i + 1) - x0(b, 3 + k, i) : 0.0;
  return sqrt(b.c.lam_sm * irls1(g, b.c.eps_irls, b.c.inv_eps));
}
__device__ __forceinline__ double a_smy(const BlkCtx& b, int k, int x, int y) {
  const int64_t i = (int64_t)y * b.f.W + x;
  const double g = y < b.f.H - 1 ? x0(b, 3 + k, i + b.f.W) - x0(b, 3 + k, i) : 0.0;
  return sqrt(b.c.lam_sm * irls1(g, b.c.eps_irls, b.c.inv_eps));
}

__device__ __forceinline__ double a_is(const BlkCtx& b, int k, int64_t i) {
  return sqrt(b.c.lam_is * irls1(x0(b, 3 + k, i), b.c.eps_irls, b.c.inv_eps));
}
__device__ __forceinline__ double a_nn(const BlkCtx& b, int k, int64_t i) {
  return sqrt(b.c.lam_nn * nonneg_w(x0(b, 3 + k, i), b.c.eps_nn));
}

#define GRID_LOOP(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// residual (op 0) or J dX (op 1): Y is the evaluation point / direction
__global__ void k_block_rows(BlkCtx b, int block, int op, const float* __restrict__ Y, float* __restrict__ out) {
  const int W = b.f.W, H = b.f.H, NT = b.f.NT, K = NT - 1;
  const int64_t N = b.f.N;
  const bool jac = op == 1;
  if (block == BLK_CONSISTENCY) {
    const double lam = b.c.lam_rc;
    GRID_LOOP(j, b.pairs.n) {
      const int64_t s = b.pairs.src[j], d = b.pairs.dst[j];
      const bool tmp = b.pairs.temporal && b.pairs.temporal[j];
      const double a = sqrt(lam * (b.pairs.weight ? b.pairs.weight[j] : 1.0));
      for (int ch = 0; ch < 3; ++ch) {
        const double u = Y[(int64_t)ch * N + s];
        double p;
        if (tmp) p = jac ? 0.0 : (double)b.f.prev_r[(int64_t)ch * N + d];   // energy.py:352-357
        else p = Y[(int64_t)ch * N + d];
        out[3 * j + ch] = (float)(a * (u - p));
      }
    }
    return;
  }
  GRID_LOOP(i, N) {
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    switch (block) {
      case BLK_DATA: {
        const double a = sqrt(b.c.lam_d);
        for (int ch = 0; ch < 3; ++ch) {
          double v;
          if (!jac) {
            v = a * ((double)b.f.img[(int64_t)ch * N + i] - exp((double)Y[(int64_t)ch * N + i]) * S_of(b, Y, i, ch));
          } else {
            const double R0 = exp(x0(b, ch, i)), S0 = S_of(b, b.X0, i, ch);
            v = -a * (R0 * S0 * Y[(int64_t)ch * N + i] + R0 * S_of(b, Y, i, ch));
          }
          out[3 * i + ch] = (float)v;
        }
      } break;
      case BLK_CLUSTERING: {
        const double a = sqrt(b.c.lam_cl);
        for (int ch = 0; ch < 3; ++ch) {
          const double u = Y[(int64_t)ch * N + i];
          out[3 * i + ch] = (float)(a * (jac ? u : u - anchor_of(b, i, ch)));
        }
      } break;
      case BLK_RSPARSITY: {
        const double a = a_rs(b, x, y);
        for (int ch = 0; ch < 3; ++ch) {
          const double u = Y[(int64_t)ch * N + i];
          const double gx = x < W - 1 ? Y[(int64_t)ch * N + i + 1] - u : 0.0;
          const double gy = y < H - 1 ? Y[(int64_t)ch * N + i + W] - u : 0.0;
          out[3 * i + ch] = (float)(a * gx);
          out[3 * N + 3 * i + ch] = (float)(a * gy);
        }
      } break;
      case BLK_MONOCHROME: {
        const double a = sqrt(b.c.lam_m * (double)b.f.edge[i]);
        double s[3];
        for (int ch = 0; ch < 3; ++ch) {
          double v = 0.0;
          for (int k = 0; k < NT; ++k) v += (double)Y[(int64_t)(3 + k) * N + i] * (jac ? b.c.G[k][ch] : b.c.B[k][ch]);
          s[ch] = v;
        }
        const double mean = jac ? 0.0 : (s[0] + s[1] + s[2]) / 3.0;
        for (int ch = 0; ch < 3; ++ch) out[3 * i + ch] = (float)(a * (s[ch] - mean));
      } break;
      case BLK_ISPARSITY:
        for (int k = 1; k < NT; ++k)
          out[(int64_t)K * i + (k - 1)] = (float)(a_is(b, k, i) * Y[(int64_t)(3 + k) * N + i]);
        break;
      case BLK_SMOOTHNESS:
        for (int k = 0; k < NT; ++k) {
          const double u = Y[(int64_t)(3 + k) * N + i];
          const double gx = x < W - 1 ? Y[(int64_t)(3 + k) * N + i + 1] - u : 0.0;
          const double gy = y < H - 1 ? Y[(int64_t)(3 + k) * N + i + W] - u : 0.0;
          out[(int64_t)NT * i + k] = (float)(a_smx(b, k, x, y) * gx);
          out[(int64_t)NT * N + (int64_t)NT * i + k] = (float)(a_smy(b, k, x, y) * gy);
        }
        break;
      case BLK_NONNEG:
        for (int k = 0; k < NT; ++k)
          out[(int64_t)NT * i + k] = (float)(a_nn(b, k, i) * Y[(int64_t)(3 + k) * N + i]);
        break;
      default: break;
    }
  }
}

// out += J^T w (op 0) or out += diag(J^T J) (op 1), planar out; everything
// but the consistency block pulls its contributions per pixel
__global__ void k_block_cols(BlkCtx b, int block, int op, const float* __restrict__ w, float* __restrict__ out) {
  const int W = b.f.W, H = b.f.H, NT = b.f.NT, K = NT - 1;
  const int64_t N = b.f.N;
  const bool dg = op == 1;
  GRID_LOOP(i, N) {
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    switch (block) {
      case BLK_DATA: {   // energy.py:214-222
        const double a = sqrt(b.c.lam_d);
        double R0[3], S0[3];
        for (int ch = 0; ch < 3; ++ch) {
          R0[ch] = exp(x0(b, ch, i));
          S0[ch] = S_of(b, b.X0, i, ch);
          const double v = dg ? (a * R0[ch] * S0[ch]) * (a * R0[ch] * S0[ch]) : -a * R0[ch] * S0[ch] * w[3 * i + ch];
          out[(int64_t)ch * N + i] += (float)v;
        }
        for (int k = 0; k < NT; ++k) {
          double v = 0.0;
          for (int ch = 0; ch < 3; ++ch)
            v += dg ? a * a * R0[ch] * R0[ch] * b.c.B[k][ch] * b.c.B[k][ch] : -a * R0[ch] * w[3 * i + ch] * b.c.B[k][ch];
          out[(int64_t)(3 + k) * N + i] += (float)v;
        }
      } break;
      case BLK_CLUSTERING: {
        const double a = sqrt(b.c.lam_cl);
        for (int ch = 0; ch < 3; ++ch) out[(int64_t)ch * N + i] += (float)(dg ? a * a : a * w[3 * i + ch]);
      } break;
      case BLK_RSPARSITY: {   // energy.py:272-291 (rows on the far edge are zero)
        const double ac = a_rs(b, x, y);
        const double al = x > 0 ? a_rs(b, x - 1, y) : 0.0, au = y > 0 ? a_rs(b, x, y - 1) : 0.0;
        for (int ch = 0; ch < 3; ++ch) {
          double v = 0.0;
          if (dg) {
            v = (x < W - 1 ? ac * ac : 0.0) + al * al + (y < H - 1 ? ac * ac : 0.0) + au * au;
          } else {
            if (x > 0) v += al * w[3 * (i - 1) + ch];
            if (x < W - 1) v -= ac * w[3 * i + ch];
            if (y > 0) v += au * w[3 * N + 3 * (i - W) + ch];
            if (y < H - 1) v -= ac * w[3 * N + 3 * i + ch];
          }
          out[(int64_t)ch * N + i] += (float)v;
        }
      } break;
      case BLK_MONOCHROME: {   // energy.py:403-411
        const double a = sqrt(b.c.lam_m * (double)b.f.edge[i]);
        for (int k = 0; k < NT; ++k) {
          double v = 0.0;
          for (int ch = 0; ch < 3; ++ch) v += dg ? a * a * b.c.G[k][ch] * b.c.G[k][ch] : a * w[3 * i + ch] * b.c.G[k][ch];
          out[(int64_t)(3 + k) * N + i] += (float)v;
        }
      } break;
      case BLK_ISPARSITY:
        for (int k = 1; k < NT; ++k) {
          const double a = a_is(b, k, i);
          out[(int64_t)(3 + k) * N + i] += (float)(dg ? a * a : a * w[(int64_t)K * i + (k - 1)]);
        }
        break;
      case BLK_SMOOTHNESS:
        for (int k = 0; k < NT; ++k) {
          const double ax = a_smx(b, k, x, y), ay = a_smy(b, k, x, y);
          const double al = x > 0 ? a_smx(b, k, x - 1, y) : 0.0, au = y > 0 ? a_smy(b, k, x, y - 1) : 0.0;
          double v = 0.0;
          if (dg) {
            v = (x < W - 1 ? ax * ax : 0.0) + al * al + (y < H - 1 ? ay * ay : 0.0) + au * au;
          } else {
            const int64_t bx = (int64_t)NT * i + k, by = (int64_t)NT * N + bx;
            if (x > 0) v += al * w[bx - NT];
            if (x < W - 1) v -= ax * w[bx];
            if (y > 0) v += au * w[by - (int64_t)NT * W];
            if (y < H - 1) v -= ay * w[by];
          }
          out[(int64_t)(3 + k) * N + i] += (float)v;
        }
        break;
      case BLK_NONNEG:
        for (int k = 0; k < NT; ++k) {
          const double a = a_nn(b, k, i);
          out[(int64_t)(3 + k) * N + i] += (float)(dg ? a * a : a * w[(int64_t)NT * i + k]);
        }
        break;
      default: break;
    }
  }
}

// consistency J^T w / diag: a scatter over the pair rows (energy.py:359-381)
// into an fp64 scratch of 3N, then added to the fp32 planes
__global__ void k_block_pairs(BlkCtx b, int op, const float* __restrict__ w, double* __restrict__ acc) {
  const int64_t N = b.f.N;
  const double lam = b.c.lam_rc;
  GRID_LOOP(j, b.pairs.n) {
    const int64_t s = b.pairs.src[j], d = b.pairs.dst[j];
    const bool tmp = b.pairs.temporal && b.pairs.temporal[j];
    const double a2 = lam * (b.pairs.weight ? b.pairs.weight[j] : 1.0);
    const double a = sqrt(a2);
    for (int ch = 0; ch < 3; ++ch) {
      const double v = op == 1 ? a2 : a * w[3 * j + ch];
      atomicAdd(acc + (int64_t)ch * N + s, v);
      if (!tmp) atomicAdd(acc + (int64_t)ch * N + d, op == 1 ? v : -v);
    }
  }
}

__global__ void k_block_add(int64_t n, const double* __restrict__ acc, float* __restrict__ out) {
  GRID_LOOP(i, n) out[i] += (float)acc[i];
}

}  // namespace

int64_t block_rows(int block, int H, int W, int NT, int64_t n_pairs) {
  const int64_t N = (int64_t)H * W;
  switch (block) {
    case BLK_DATA: case BLK_CLUSTERING: case BLK_MONOCHROME: return 3 * N;
    case BLK_RSPARSITY: return 6 * N;
    case BLK_CONSISTENCY: return 3 * n_pairs;
    case BLK_ISPARSITY: return (int64_t)(NT - 1) * N;
    case BLK_SMOOTHNESS: return 2 * (int64_t)NT * N;
    case BLK_NONNEG: return (int64_t)NT * N;
    default: return -1;
  }
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

cudaError_t launch_block_rows(cudaStream_t s, const Frame& f, const Coef<double>& c, const float* X0,
                              const BlockPairs& pairs, int block, int op, const float* Y, float* out) {
  BlkCtx b{f, c, X0, pairs};
  const int64_t n = block == BLK_CONSISTENCY ? pairs.n : (int64_t)f.N;
  if (n > 0) k_block_rows<<<grid_for(n), 256, 0, s>>>(b, block, op, Y, out);
  return cudaGetLastError();
}

cudaError_t launch_block_cols(cudaStream_t s, const Frame& f, const Coef<double>& c, const float* X0,
                              const BlockPairs& pairs, int block, int op, const float* w, float* out) {
  BlkCtx b{f, c, X0, pairs};
  if (block != BLK_CONSISTENCY) {
    k_block_cols<<<grid_for(f.N), 256, 0, s>>>(b, block, op, w, out);
    return cudaGetLastError();
  }
  if (pairs.n == 0) return cudaSuccess;
  const int64_t n3 = 3 * (int64_t)f.N;
  double* acc = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&acc, sizeof(double) * n3, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(acc, 0, sizeof(double) * n3, s);
  k_block_pairs<<<grid_for(pairs.n), 256, 0, s>>>(b, op, w, acc);
  k_block_add<<<grid_for(n3), 256, 0, s>>>(n3, acc, out);
  cudaFreeAsync(acc, s);
  return cudaGetLastError();
}

}  // namespace ls
