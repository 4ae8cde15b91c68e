// Dense base-color phase:
//   k_dense_accum    per-pixel outer products of the refinement normal
//                    equations (energy.py:563-610), reduced over all pixels
//                    warp-cooperatively in fp64, fixed order, last block
//                    finalises
//   k_dense_solve    single-CTA assembly of the 3K x 3K system (+ clustering
//                    anchor rows, lambda_IR, lambda_CR projections) and a
//                    one-sided Jacobi SVD truncated solve (solver.py:195-204)
#include "ls_kernels.h"

namespace ls {

constexpr int kMaxN = 3 * (kMaxNT - 1);   // 36
constexpr int kSvdWarps = kMaxN / 2;      // 18

// sums layout: [M_c(k<=j) for c][rhs_c(k) for c][n_k][sum r_c over cluster k]
__host__ __device__ inline int dense_nm(int K) { return 3 * (K * (K + 1) / 2); }
__host__ __device__ inline int dense_ns(int K) { return dense_nm(K) + 3 * K + K + 3 * K; }
int dense_nsums(int K) { return dense_ns(K); }

constexpr int kDensePixVals = 3 + 3 + 3 + 1 + (kMaxNT - 1);   // R, res, r, id, T_ind
constexpr int kDenseMaxSums = 3 * ((kMaxNT - 1) * kMaxNT / 2) + 7 * (kMaxNT - 1);
constexpr int kDensePerLane = (kDenseMaxSums + 31) / 32;

__global__ void __launch_bounds__(128) k_dense_accum(Frame f, const double* __restrict__ colors, int K,
                                                     const float* __restrict__ X, int use_ids, double* part,
                                                     unsigned* ticket, double* sums) {
  __shared__ double pix[4][32][kDensePixVals];
  __shared__ double red[4][kDenseMaxSums];
  __shared__ short ent_c[kDenseMaxSums], ent_k[kDenseMaxSums], ent_j[kDenseMaxSums], ent_t[kDenseMaxSums];
  const int N = f.N, NT = K + 1;
  const int NS = dense_ns(K), NM = dense_nm(K);
  // entry decode table
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    short t, c = 0, k = 0, j = 0;
    if (e < NM) {
      t = 0;
      c = (short)(e / (K * (K + 1) / 2));
      int r = e % (K * (K + 1) / 2), kk = 0;
      while (r >= K - kk) { r -= K - kk; ++kk; }
      k = (short)kk;
      j = (short)(kk + r);
    } else if (e < NM + 3 * K) {
      t = 1; c = (short)((e - NM) / K); k = (short)((e - NM) % K);
    } else if (e < NM + 4 * K) {
      t = 2; k = (short)(e - NM - 3 * K);
    } else {
      t = 3; k = (short)((e - NM - 4 * K) / 3); c = (short)((e - NM - 4 * K) % 3);
    }
    ent_t[e] = t; ent_c[e] = c; ent_k[e] = k; ent_j[e] = j;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[kDensePerLane];
#pragma unroll
  for (int m = 0; m < kDensePerLane; ++m) acc[m] = 0.0;
  // row bands: only the band's own rows [y_lo, y_hi)
  const int i0 = f.y_lo * f.W, npx = (f.y_hi - f.y_lo) * f.W;
  const int nchunks = (npx + 31) / 32;
  for (int chunk = blockIdx.x * 4 + wid; chunk < nchunks; chunk += gridDim.x * 4) {
    const int i = i0 + chunk * 32 + lane;
    double* pv = pix[wid][lane];
    if (chunk * 32 + lane < npx) {
      double S[3] = {0.0, 0.0, 0.0};
      for (int k = 0; k < NT; ++k) {
        const double t = (double)X[(size_t)(3 + k) * N + i];
        const double b0 = k == 0 ? 1.0 : colors[3 * (k - 1)];
        const double b1 = k == 0 ? 1.0 : colors[3 * (k - 1) + 1];
        const double b2 = k == 0 ? 1.0 : colors[3 * (k - 1) + 2];
        S[0] += t * b0; S[1] += t * b1; S[2] += t * b2;
        if (k > 0) pv[10 + k - 1] = t;
      }
      for (int c = 0; c < 3; ++c) {
        const double r = (double)X[(size_t)c * N + i];
        const double R = exp(r);
        pv[c] = R;
        pv[3 + c] = (double)f.img[(size_t)c * N + i] - R * S[c];
        pv[6 + c] = r;
      }
      pv[9] = (use_ids && f.ids) ? (double)f.ids[i] : 0.0;
    } else {
      for (int v = 0; v < 10 + K; ++v) pv[v] = 0.0;
    }
    __syncwarp();
    const int np = min(32, npx - chunk * 32);
#pragma unroll
    for (int m = 0; m < kDensePerLane; ++m) {
      const int e = lane + 32 * m;
      if (e >= NS) break;
      const int t = ent_t[e], c = ent_c[e], k = ent_k[e], j = ent_j[e];
      double s = 0.0;
      for (int q = 0; q < np; ++q) {
        const double* pq = pix[wid][q];
        if (t == 0) s += pq[c] * pq[c] * pq[10 + k] * pq[10 + j];
        else if (t == 1) s += pq[10 + k] * (pq[c] * pq[3 + c]);
        else if (t == 2) s += (pq[9] == (double)(k + 1)) ? 1.0 : 0.0;
        else s += (pq[9] == (double)(k + 1)) ? pq[6 + c] : 0.0;
      }
      acc[m] += s;
    }
    __syncwarp();
  }
#pragma unroll
  for (int m = 0; m < kDensePerLane; ++m) {
    const int e = lane + 32 * m;
    if (e < NS) red[wid][e] = acc[m];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < 4; ++w) s += red[w][e];
    part[(size_t)blockIdx.x * NS + e] = s;
  }
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += ((volatile double*)part)[(size_t)b * NS + e];
    sums[e] = s;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// ---- k_dense_accum2: the same sums with per-thread register accumulation --
// Every warp works alone (no CTA barrier inside the loop): it takes 32
// pixels at a time; lane l computes pixel l's values -- v_c[k] = R_c T_{k+1}
// (3K), the data residual res_c (3), r_c (3) and the cluster id -- into the
// warp's shared-memory rows; then lane l runs job(s) l (+32) over the 32
// pixels: jobs 0..3K-1 are one row (c, k) of the data block, accumulating
// v_c[k] v_c[j] for every j (the lower part is dropped at the end) and
// v_c[k] res_c; jobs 3K..4K-1 are cluster k's count and r sums.  All
// accumulation is in registers (fp64); one fixed-order reduction per CTA,
// then the last CTA sums the CTA partials in CTA order.
constexpr int kDa2Threads = 128, kDa2Warps = kDa2Threads / 32;

template <int K>
__global__ void __launch_bounds__(kDa2Threads, 4) k_dense_accum2(Frame f, const double* __restrict__ colors,
                                                              const float* __restrict__ X, int use_ids,
                                                              double* part, unsigned* ticket, double* sums) {
  constexpr int NT = K + 1, NV = 3 * K + 7;   // per pixel: v (3K), res (3), r (3), id
  constexpr int NS = 3 * (K * (K + 1) / 2) + 7 * K, NM = 3 * (K * (K + 1) / 2);
  constexpr int NA = K + 1 > 4 ? K + 1 : 4;   // accumulators: a data row + rhs, or 4 cluster sums
  constexpr int NJ = 4 * K, JPL = (NJ + 31) / 32;   // jobs, jobs per lane
  constexpr int PS = NV | 1;   // odd row stride (doubles): the row writes are 2-way, not 32-way, banked
  // the pixel rows and, after the loop, the per-warp job sums share storage
  constexpr int kPixD = kDa2Warps * 32 * PS, kRedD = kDa2Warps * NJ * NA;
  __shared__ double shm[kPixD > kRedD ? kPixD : kRedD];
  double (*pix)[32][PS] = reinterpret_cast<double (*)[32][PS]>(shm);
  __shared__ double B[NT][3];
  if (threadIdx.x < NT * 3) {
    const int k = threadIdx.x / 3, c = threadIdx.x % 3;
    B[k][c] = k == 0 ? 1.0 : colors[3 * (k - 1) + c];
  }
  __syncthreads();
  const int N = f.N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i0 = f.y_lo * f.W, npx = (f.y_hi - f.y_lo) * f.W;
  double acc[JPL][NA];
#pragma unroll
  for (int q = 0; q < JPL; ++q)
#pragma unroll
    for (int j = 0; j < NA; ++j) acc[q][j] = 0.0;
  double (*wp)[PS] = pix[wid];
  const int gw = blockIdx.x * kDa2Warps + wid, nw = gridDim.x * kDa2Warps;
  for (int c0 = gw * 32; c0 < npx; c0 += nw * 32) {
    {   // lane = pixel
      double* pv = wp[lane];
      const int q = c0 + lane;
      if (q < npx) {
        const int i = i0 + q;
        double t[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) t[k] = (double)X[(size_t)(3 + k) * N + i];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double S = 0.0;
#pragma unroll
          for (int k = 0; k < NT; ++k) S += t[k] * B[k][c];
          const double r = (double)X[(size_t)c * N + i];
          const double R = exp(r);
#pragma unroll
          for (int k = 0; k < K; ++k) pv[c * K + k] = R * t[k + 1];
          pv[3 * K + c] = (double)f.img[(size_t)c * N + i] - R * S;
          pv[3 * K + 3 + c] = r;
        }
        pv[3 * K + 6] = (use_ids && f.ids) ? (double)f.ids[i] : 0.0;
      } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) pv[v] = 0.0;
      }
    }
    __syncwarp();
    const int qn = min(32, npx - c0);
#pragma unroll
    for (int qj = 0; qj < JPL; ++qj) {   // lane = job
      const int job = lane + 32 * qj;
      if (job < 3 * K) {
        const int jc = job / K, jk = job % K;
        for (int q = 0; q < qn; ++q) {
          const double* pv = wp[q];
          const double a = pv[jc * K + jk];
#pragma unroll
          for (int j = 0; j < K; ++j) acc[qj][j] = fma(a, pv[jc * K + j], acc[qj][j]);
          acc[qj][K] = fma(a, pv[3 * K + jc], acc[qj][K]);
        }
      } else if (job < NJ) {
        const double id = (double)(job - 3 * K + 1);
        for (int q = 0; q < qn; ++q) {
          const double* pv = wp[q];
          if (pv[3 * K + 6] == id) {
            acc[qj][0] += 1.0;
            acc[qj][1] += pv[3 * K + 3];
            acc[qj][2] += pv[3 * K + 4];
            acc[qj][3] += pv[3 * K + 5];
          }
        }
      }
    }
    __syncwarp();
  }
  // CTA reduction (warps in order) into the sums layout of dense_ns
  // (M_c upper triangle, rhs_c, n_k, sum r_c over cluster k)
  double (*red)[NJ][NA] = reinterpret_cast<double (*)[NJ][NA]>(shm);
  __syncthreads();   // every warp is done with its pixel rows
#pragma unroll
  for (int qj = 0; qj < JPL; ++qj) {
    const int job = lane + 32 * qj;
    if (job < NJ)
#pragma unroll
      for (int j = 0; j < NA; ++j) red[wid][job][j] = acc[qj][j];
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * NS;
  for (int job = threadIdx.x; job < NJ; job += kDa2Threads) {
    double v[NA];
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      double sacc = 0.0;
      for (int w = 0; w < kDa2Warps; ++w) sacc += red[w][job][j];
      v[j] = sacc;
    }
    if (job < 3 * K) {
      const int jc = job / K, jk = job % K;
      int off = 0;
      for (int kk = 0; kk < jk; ++kk) off += K - kk;
      for (int j = jk; j < K; ++j) out[jc * (K * (K + 1) / 2) + off + (j - jk)] = v[j];
      out[NM + jc * K + jk] = v[K];
    } else {
      const int jk = job - 3 * K;
      out[NM + 3 * K + jk] = v[0];
      for (int c = 0; c < 3; ++c) out[NM + 4 * K + 3 * jk + c] = v[1 + c];
    }
  }
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < NS; e += blockDim.x) {
    double s2 = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) s2 += ((volatile double*)part)[(size_t)b * NS + e];
    sums[e] = s2;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// band-ordered sum of gathered per-band partial sums [nbands][nv]
__global__ void k_band_sum(const double* __restrict__ g, int nbands, int nv, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nv; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nbands; ++b) s += g[(size_t)b * nv + j];
    out[j] = s;
  }
}
void launch_band_sum(cudaStream_t s, const double* gathered, int nbands, int nv, double* out) {
  k_band_sum<<<1, 256, 0, s>>>(gathered, nbands, nv, out);
}

// ---- one-sided Jacobi SVD truncated solve, single CTA ---------------------
// U holds the working columns of A (column-major), V accumulates rotations.
__device__ void jacobi_svd_solve(double (*U)[kMaxN + 1], double (*V)[kMaxN + 1], double* rhs, int n, double trunc,
                                 double* x_out) {
  __shared__ int order[kMaxN + 2];
  __shared__ int rotated;
  __shared__ double sig[kMaxN + 2];
  __shared__ int allzero;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int m = n + (n & 1);   // even number of columns (pad column is zero)
  if (threadIdx.x == 0) {
    allzero = 1;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        if (U[j][i] != 0.0) allzero = 0;
    for (int i = 0; i < m; ++i) order[i] = i;
  }
  __syncthreads();
  if (allzero) {   // solver.py:198-199
    for (int i = threadIdx.x; i < n; i += blockDim.x) x_out[i] = 0.0;
    return;
  }
  for (int sweep = 0; sweep < 80; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int step = 0; step < m - 1; ++step) {
      if (wid < m / 2) {
        const int p = order[wid], q = order[m - 1 - wid];
        if (p < n && q < n) {
          double a = 0.0, b = 0.0, g = 0.0;
          for (int i = lane; i < n; i += 32) {
            a += U[p][i] * U[p][i];
            b += U[q][i] * U[q][i];
            g += U[p][i] * U[q][i];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            g += __shfl_xor_sync(0xffffffffu, g, o);
          }
          if (fabs(g) > 1e-15 * sqrt(a * b) && g != 0.0) {
            const double zeta = (b - a) / (2.0 * g);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
            for (int i = lane; i < n; i += 32) {
              const double up = U[p][i], uq = U[q][i];
              U[p][i] = c * up - s * uq;
              U[q][i] = s * up + c * uq;
              const double vp = V[p][i], vq = V[q][i];
              V[p][i] = c * vp - s * vq;
              V[q][i] = s * vp + c * vq;
            }
            if (lane == 0) rotated = 1;
          }
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {   // round-robin: keep order[0], rotate the rest
        const int last = order[m - 1];
        for (int i = m - 1; i > 1; --i) order[i] = order[i - 1];
        order[1] = last;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += U[j][i] * U[j][i];
    sig[j] = sqrt(s);
  }
  __syncthreads();
  double smax = 0.0;
  for (int j = 0; j < n; ++j) smax = fmax(smax, sig[j]);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double xi = 0.0;
    if (smax > 0.0) {
      for (int j = 0; j < n; ++j) {
        if (!(sig[j] > trunc * smax)) continue;
        double ub = 0.0;
        for (int r = 0; r < n; ++r) ub += U[j][r] * rhs[r];
        xi += V[j][i] * (ub / (sig[j] * sig[j]));
      }
    }
    x_out[i] = xi;
  }
}

__global__ void __launch_bounds__(32 * kSvdWarps) k_svd_solve(int n, const double* A, const double* rhs_in,
                                                              double trunc, double* x) {
  __shared__ double U[kMaxN][kMaxN + 1], V[kMaxN][kMaxN + 1];
  __shared__ double rhs[kMaxN];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    U[c][r] = A[e];                 // A row-major -> columns
    V[c][r] = (r == c) ? 1.0 : 0.0;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) rhs[i] = rhs_in[i];
  __syncthreads();
  jacobi_svd_solve(U, V, rhs, n, trunc, x);
}

__global__ void __launch_bounds__(32 * kSvdWarps) k_dense_solve(const double* __restrict__ sums, int K,
                                                                const double* __restrict__ colors, int use_ids,
                                                                double lam_d, double lam_cl, double lam_ir,
                                                                double lam_cr, int chroma_identity, double trunc,
                                                                double* A_out, double* rhs_out, double* x) {
  __shared__ double U[kMaxN][kMaxN + 1], V[kMaxN][kMaxN + 1];
  __shared__ double A[kMaxN][kMaxN + 1];
  __shared__ double rhs[kMaxN];
  const int n = 3 * K, NM = dense_nm(K), half = K * (K + 1) / 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      rhs[i] = 0.0;
      for (int j = 0; j < n; ++j) A[i][j] = 0.0;
    }
    // data rows (energy.py:584-589)
    for (int c = 0; c < 3; ++c) {
      int e = c * half;
      for (int k = 0; k < K; ++k)
        for (int j = k; j < K; ++j, ++e) {
          const double v = lam_d * sums[e];
          A[3 * k + c][3 * j + c] += v;
          if (j != k) A[3 * j + c][3 * k + c] += v;
        }
      for (int k = 0; k < K; ++k) rhs[3 * k + c] += lam_d * sums[NM + c * K + k];
    }
    // clustering anchor rows (energy.py:590-604)
    if (use_ids) {
      for (int k = 0; k < K; ++k) {
        const double nk = sums[NM + 3 * K + k];
        if (nk == 0.0) continue;
        for (int c = 0; c < 3; ++c) {
          const double b = fmax(colors[3 * k + c], 1e-4);
          const double sr = sums[NM + 4 * K + 3 * k + c];
          A[3 * k + c][3 * k + c] += lam_cl * nk / (b * b);
          rhs[3 * k + c] += lam_cl * (sr - nk * log(b)) / b;
        }
      }
    }
    for (int i = 0; i < n; ++i) A[i][i] += lam_ir;   // energy.py:605
    for (int k = 0; k < K; ++k) {                     // energy.py:518-539, 606-609
      const double b0 = colors[3 * k], b1 = colors[3 * k + 1], b2 = colors[3 * k + 2];
      const double nrm = sqrt(b0 * b0 + b1 * b1 + b2 * b2);
      double P[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
      if (!chroma_identity && !(nrm < 1e-9)) {
        const double u[3] = {b0 / nrm, b1 / nrm, b2 / nrm};
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) P[a][b] -= u[a] * u[b];
      }
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) A[3 * k + a][3 * k + b] += lam_cr * P[a][b];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    U[c][r] = A[r][c];
    V[c][r] = (r == c) ? 1.0 : 0.0;
    if (A_out) A_out[e] = A[r][c];
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (rhs_out) rhs_out[i] = rhs[i];
  __syncthreads();
  jacobi_svd_solve(U, V, rhs, n, trunc, x);
}

void launch_dense_accum(cudaStream_t s, int grid, const Frame& f, const double* colors_dev, int K, const float* X,
                        int use_ids, double* part, unsigned* ticket, double* sums) {
  switch (K) {   // register-accumulating kernel for K = 1..12 (4K jobs <= 64 threads)
#define LS_DA2(KV) \
    case KV: k_dense_accum2<KV><<<grid, kDa2Threads, 0, s>>>(f, colors_dev, X, use_ids, part, ticket, sums); break;
    LS_DA2(1) LS_DA2(2) LS_DA2(3) LS_DA2(4) LS_DA2(5) LS_DA2(6) LS_DA2(7) LS_DA2(8) LS_DA2(9) LS_DA2(10)
    LS_DA2(11) LS_DA2(12)
#undef LS_DA2
    default: k_dense_accum<<<grid, 128, 0, s>>>(f, colors_dev, K, X, use_ids, part, ticket, sums); break;
  }
}
void launch_dense_assemble_solve(cudaStream_t s, const double* sums, int K, const double* colors_dev, int use_ids,
                                 double lam_d, double lam_cl, double lam_ir, double lam_cr, int chroma_identity,
                                 double trunc, double* A_out, double* rhs_out, double* x_out) {
  k_dense_solve<<<1, 32 * kSvdWarps, 0, s>>>(sums, K, colors_dev, use_ids, lam_d, lam_cl, lam_ir, lam_cr,
                                             chroma_identity, trunc, A_out, rhs_out, x_out);
}
void launch_svd_solve(cudaStream_t s, int n, const double* A, const double* rhs, double trunc, double* x) {
  k_svd_solve<<<1, 32 * kSvdWarps, 0, s>>>(n, A, rhs, trunc, x);
}

}  // namespace ls
