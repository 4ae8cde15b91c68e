// First-frame base-color estimation on the device (reference palette.py:81-238,
// estimate_palette): the 10x10 chroma histogram of the non-dark pixels, a
// population-weighted k-means over its populated bins, nearest-center
// assignment of every pixel, and the greedy merge of centers closer than 0.2
// whose survivors become the palette (mean RGB of their non-dark pixels).
//
//   k_pal_hist    per pixel: histogram bin of each non-dark pixel, integer
//                 counts (shared-memory bins, then global integer atomics)
//   k_pal_kmeans  one warp: the seeded first pick of numpy's
//                 Generator.choice(n, p) (PCG64 double, cdf search),
//                 farthest-point seeding and Lloyd rounds over <= 100 bins;
//                 the weighted center means add in bin order, as numpy's
//                 axis-0 reduction does, so the centers are bit-exact
//   k_pal_assign  per pixel: nearest center (first minimum); per-cluster
//                 non-dark counts and RGB sums reduced in a fixed order; the
//                 last CTA runs the merge and writes K and the colors
//
// Only the final color means differ from the reference's (sequential
// pixel-order) sums, by fp64 rounding of the summation order.
#include <cfloat>

#include "ls_kernels.h"

namespace ls {

namespace {

constexpr int kBins = 10;            // HIST_BINS (palette.py:19)
constexpr int kCells = kBins * kBins;
constexpr int kKmeansIters = 100;    // KMEANS_MAX_ITERS
constexpr double kMergeDist = 0.2;   // MERGE_DISTANCE
constexpr int kPalMaxK = 12;
constexpr int kPalNV = 4 * kPalMaxK; // per cluster: count, R, G, B sums

__device__ __forceinline__ double norm2(double a, double b) {
  return __dsqrt_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
}

// imaging.py:160-171: dark = channel sum < 0.02 (fp64, left to right)
__device__ __forceinline__ bool is_dark(const float* img, int N, int i) {
  const double s = __dadd_rn(__dadd_rn((double)img[i], (double)img[N + i]), (double)img[2 * N + i]);
  return s < 0.02;
}

// palette.py:81-89: bin = clip(int(c * 10), 0, 9), flat = g_bin * 10 + r_bin
__device__ __forceinline__ int hist_cell(double c0, double c1) {
  long long rb = (long long)__dmul_rn(c0, (double)kBins), gb = (long long)__dmul_rn(c1, (double)kBins);
  rb = rb < 0 ? 0 : (rb > kBins - 1 ? kBins - 1 : rb);
  gb = gb < 0 ? 0 : (gb > kBins - 1 ? kBins - 1 : gb);
  return (int)(gb * kBins + rb);
}

__global__ void k_pal_hist(const float* __restrict__ img, const double* __restrict__ chroma, int N,
                           int* __restrict__ pop) {
  __shared__ int h[kCells];
  for (int j = threadIdx.x; j < kCells; j += blockDim.x) h[j] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    if (!is_dark(img, N, i)) atomicAdd(&h[hist_cell(chroma[i], chroma[N + i])], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < kCells; j += blockDim.x)
    if (h[j]) atomicAdd(&pop[j], h[j]);
}

__device__ __forceinline__ uint64_t pcg64_out(unsigned __int128& s, unsigned __int128 inc) {
  const unsigned __int128 mult = ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  s = s * mult + inc;
  const unsigned rot = (unsigned)(s >> 122);
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

struct KmOut {
  double centers[kPalMaxK][2];
  int k;
};

// palette.py:106-138 (weighted_kmeans), one warp
__global__ void k_pal_kmeans(const int* __restrict__ pop, PalRng rng, int k_max, KmOut* out) {
  __shared__ double mx[kCells], my[kCells], w[kCells];
  __shared__ int n_s, assign[kCells], prev[kCells], chosen[kPalMaxK];
  __shared__ double cx[kPalMaxK], cy[kPalMaxK], dmin[kCells];
  const int lane = threadIdx.x;
  if (lane == 0) {   // populated bins in row-major (g, r) order (palette.py:40-44)
    int n = 0;
    for (int j = 0; j < kCells; ++j)
      if (pop[j] > 0) {
        const int gb = j / kBins, rb = j % kBins;
        mx[n] = __ddiv_rn((double)rb + 0.5, (double)kBins);
        my[n] = __ddiv_rn((double)gb + 0.5, (double)kBins);
        w[n] = (double)pop[j];
        ++n;
      }
    n_s = n;
  }
  __syncwarp();
  const int n = n_s;
  if (n == 0) {   // all pixels dark: EmptyHistogramError on the host
    if (lane == 0) out->k = 0;
    return;
  }
  const int k = k_max < n ? k_max : n;
  if (lane == 0) {
    // Generator.choice(n, p=pops/pops.sum()): cdf = cumsum(p) / cdf[-1],
    // u = next_double(), first index with cdf > u
    double tot = 0.0;
    for (int j = 0; j < n; ++j) tot = __dadd_rn(tot, w[j]);
    double cdf[kCells];
    double c = 0.0;
    for (int j = 0; j < n; ++j) {
      c = __dadd_rn(c, __ddiv_rn(w[j], tot));
      cdf[j] = c;
    }
    const double last = cdf[n - 1];
    unsigned __int128 s = ((unsigned __int128)rng.st_hi << 64) | rng.st_lo;
    const unsigned __int128 inc = ((unsigned __int128)rng.inc_hi << 64) | rng.inc_lo;
    const double u = (double)(pcg64_out(s, inc) >> 11) * (1.0 / 9007199254740992.0);
    int first = n;
    for (int j = 0; j < n; ++j)
      if (__ddiv_rn(cdf[j], last) > u) {
        first = j;
        break;
      }
    if (first >= n) first = n - 1;
    chosen[0] = first;
  }
  __syncwarp();
  // farthest-point seeding: argmax over bins of the distance to the nearest chosen
  for (int m = 1; m < k; ++m) {
    for (int j = lane; j < n; j += 32) {
      double d = DBL_MAX;
      for (int q = 0; q < m; ++q) {
        const double e = norm2(mx[j] - mx[chosen[q]], my[j] - my[chosen[q]]);
        d = e < d ? e : d;
      }
      dmin[j] = d;
    }
    __syncwarp();
    if (lane == 0) {
      int best = 0;
      for (int j = 1; j < n; ++j)
        if (dmin[j] > dmin[best]) best = j;
      chosen[m] = best;
    }
    __syncwarp();
  }
  if (lane < k) {
    cx[lane] = mx[chosen[lane]];
    cy[lane] = my[chosen[lane]];
  }
  __syncwarp();
  for (int it = 0; it < kKmeansIters; ++it) {
    for (int j = lane; j < n; j += 32) {
      int a = 0;
      double da = norm2(mx[j] - cx[0], my[j] - cy[0]);
      for (int q = 1; q < k; ++q) {
        const double e = norm2(mx[j] - cx[q], my[j] - cy[q]);
        if (e < da) {
          da = e;
          a = q;
        }
      }
      assign[j] = a;
    }
    __syncwarp();
    int same = 1;
    if (it > 0)
      for (int j = lane; j < n; j += 32) same &= assign[j] == prev[j];
    same = __all_sync(0xffffffffu, same);
    if (it > 0 && same) break;
    for (int j = lane; j < n; j += 32) prev[j] = assign[j];
    // np.average(mids[sel], axis=0, weights=pops[sel]): bin-order sums
    if (lane < k) {
      double sx = 0.0, sy = 0.0, sw = 0.0;
      bool any = false;
      for (int j = 0; j < n; ++j)
        if (assign[j] == lane) {
          sx = __dadd_rn(sx, __dmul_rn(mx[j], w[j]));
          sy = __dadd_rn(sy, __dmul_rn(my[j], w[j]));
          sw = __dadd_rn(sw, w[j]);
          any = true;
        }
      if (any) {
        cx[lane] = __ddiv_rn(sx, sw);
        cy[lane] = __ddiv_rn(sy, sw);
      }
    }
    __syncwarp();
  }
  if (lane < k) {
    out->centers[lane][0] = cx[lane];
    out->centers[lane][1] = cy[lane];
  }
  if (lane == 0) out->k = k;
}

// palette.py:141-192 (assign_pixels + merge_clusters)
__global__ void __launch_bounds__(kThreads) k_pal_assign(const float* __restrict__ img,
                                                          const double* __restrict__ chroma, int N,
                                                          const KmOut* __restrict__ km, double* part,
                                                          unsigned* ticket, double* __restrict__ out_colors,
                                                          int* __restrict__ out_k) {
  const int k = km->k;
  double acc[kPalNV];
#pragma unroll
  for (int j = 0; j < kPalNV; ++j) acc[j] = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (is_dark(img, N, i)) continue;   // merge counts / means use non-dark pixels only
    const double c0 = chroma[i], c1 = chroma[N + i];
    int a = 0;
    double da = norm2(c0 - km->centers[0][0], c1 - km->centers[0][1]);
    for (int q = 1; q < k; ++q) {
      const double e = norm2(c0 - km->centers[q][0], c1 - km->centers[q][1]);
      if (e < da) {
        da = e;
        a = q;
      }
    }
#pragma unroll
    for (int q = 0; q < kPalMaxK; ++q)
      if (q == a) {
        acc[4 * q] += 1.0;
        acc[4 * q + 1] += (double)img[i];
        acc[4 * q + 2] += (double)img[N + i];
        acc[4 * q + 3] += (double)img[2 * N + i];
      }
  }
  block_reduce_store<kPalNV>(acc, part);
  if (!last_block(ticket)) return;
  __shared__ double tot[kPalNV];
  for (int j = 0; j < kPalNV; ++j) {
    const double t = sum_partials<kPalNV>(part, gridDim.x, j);
    if (threadIdx.x == 0) tot[j] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  *ticket = 0u;
  // greedy merge: the closest pair under 0.2, smaller population into larger
  long long pops[kPalMaxK];
  double sums[kPalMaxK][3];
  int alive[kPalMaxK], na = k;
  for (int j = 0; j < k; ++j) {
    pops[j] = (long long)tot[4 * j];
    for (int ch = 0; ch < 3; ++ch) sums[j][ch] = tot[4 * j + 1 + ch];
    alive[j] = j;
  }
  while (na > 1) {
    int ba = -1, bb = -1;
    double bd = 0.0;
    for (int x = 0; x < na; ++x)
      for (int y = x + 1; y < na; ++y) {
        const int a = alive[x], b = alive[y];
        const double d = norm2(km->centers[a][0] - km->centers[b][0], km->centers[a][1] - km->centers[b][1]);
        if (d < kMergeDist && (ba < 0 || d < bd)) {
          bd = d;
          ba = a;
          bb = b;
        }
      }
    if (ba < 0) break;
    const int small = pops[ba] <= pops[bb] ? ba : bb, large = small == ba ? bb : ba;
    pops[large] += pops[small];
    pops[small] = 0;
    for (int ch = 0; ch < 3; ++ch) sums[large][ch] += sums[small][ch];
    int w = 0;
    for (int x = 0; x < na; ++x)
      if (alive[x] != small) alive[w++] = alive[x];
    na = w;
  }
  for (int x = 0; x < na; ++x) {
    const int j = alive[x];
    if (pops[j] > 0) {
      for (int ch = 0; ch < 3; ++ch) out_colors[3 * x + ch] = sums[j][ch] / (double)pops[j];
    } else {   // empty survivor: its chroma center lifted to RGB
      const double r = km->centers[j][0], g = km->centers[j][1];
      out_colors[3 * x] = r;
      out_colors[3 * x + 1] = g;
      out_colors[3 * x + 2] = fmax(0.0, 1.0 - r - g);
    }
  }
  *out_k = na;
}

}  // namespace

// palette.py:227-238 without the final segment: (K, colors) into caller
// device memory (out_colors: kPalMaxK x 3 doubles, out_k: 1 int).  The
// image is the planar float32 copy and chroma the fp64 planes of k_image.
cudaError_t launch_estimate_palette(cudaStream_t s, const float* img, const double* chroma, int N, int k_max,
                                    const PalRng& rng, void* scratch, double* out_colors, int* out_k) {
  if (k_max > kPalMaxK) return cudaErrorInvalidValue;
  char* p = static_cast<char*>(scratch);
  int* pop = reinterpret_cast<int*>(p);
  KmOut* km = reinterpret_cast<KmOut*>(p + 512);
  unsigned* ticket = reinterpret_cast<unsigned*>(p + 1024);
  double* part = reinterpret_cast<double*>(p + 2048);
  const int grid = std::max(1, std::min(4 * 148, (N + kThreads - 1) / kThreads));
  cudaError_t e = cudaMemsetAsync(scratch, 0, 2048, s);
  if (e != cudaSuccess) return e;
  k_pal_hist<<<std::max(1, std::min(2 * 148, (N + 255) / 256)), 256, 0, s>>>(img, chroma, N, pop);
  k_pal_kmeans<<<1, 32, 0, s>>>(pop, rng, k_max, km);
  k_pal_assign<<<grid, kThreads, 0, s>>>(img, chroma, N, km, part, ticket, out_colors, out_k);
  return cudaGetLastError();
}

size_t palette_scratch_bytes() { return 2048 + sizeof(double) * kPalNV * 4 * 148; }

}  // namespace ls
