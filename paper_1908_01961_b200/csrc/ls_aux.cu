// Per-frame auxiliary kernels:
//   image unpack + chromaticity (imaging.py:160-171), chroma-edge gate
//   (energy.py:121-136), the consistency-partner sampler bit-exact with
//   numpy's PCG64 + buffered Lemire draws (energy.py:154-187), the per-pixel
//   adjacency (CSR) the solver kernels pull from, segmentation
//   (palette.py:195-224) and first-frame initialisation (solver.py:295-308).
//
// Everything the reference computes in fp64 is computed here in fp64 with
// explicitly rounded operations (no FMA contraction) where the result feeds
// a comparison (chroma gate, nearest-palette argmin), so the integer outputs
// (partners, cluster ids) are bit-identical to the reference.
#include <climits>
#include <cstdlib>
#include <algorithm>

#include "ls_kernels.h"

namespace ls {

typedef unsigned __int128 u128;

constexpr unsigned long long kPcgMultHi = 0x2360ED051FC65DA4ULL;
constexpr unsigned long long kPcgMultLo = 0x4385DF649FCCF645ULL;

__device__ __forceinline__ u128 mk128(unsigned long long hi, unsigned long long lo) {
  return ((u128)hi << 64) | (u128)lo;
}

// XSL-RR 128/64 output function of numpy's PCG64
__device__ __forceinline__ unsigned long long pcg_out(u128 s) {
  const unsigned rot = (unsigned)(s >> 122);
  const unsigned long long x = (unsigned long long)(s >> 64) ^ (unsigned long long)s;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// host: the jump table of SampleParams.  M_0 = A, S_0 = 1;
// M_{k+1} = M_k^2, S_{k+1} = S_k (1 + M_k); C_k = inc * S_k (mod 2^128), so
// 2^k LCG steps map s to M_k s + C_k (the same residue Brown's squaring loop
// reaches, with one 128-bit multiply-add per set bit of the distance instead
// of four multiplies per bit)
static void fill_jump_table(SampleParams& P) {
  const u128 inc = ((u128)P.inc_hi << 64) | (u128)P.inc_lo;
  u128 M = ((u128)kPcgMultHi << 64) | (u128)kPcgMultLo, S = 1;
  for (int k = 0; k < kJumpBits; ++k) {
    const u128 C = inc * S;
    P.jump[k][0] = (unsigned long long)(M >> 64);
    P.jump[k][1] = (unsigned long long)M;
    P.jump[k][2] = (unsigned long long)(C >> 64);
    P.jump[k][3] = (unsigned long long)C;
    S = S * (M + 1);
    M = M * M;
  }
}

// state after `delta` LCG steps from the jump table
__device__ __forceinline__ u128 pcg_jump(const SampleParams& P, u128 state, unsigned long long delta) {
  for (int k = 0; delta && k < kJumpBits; ++k, delta >>= 1)
    if (delta & 1ULL) state = mk128(P.jump[k][0], P.jump[k][1]) * state + mk128(P.jump[k][2], P.jump[k][3]);
  return state;
}

// sequential reader of the u32 stream (low half of each 64-bit output first)
struct U32Stream {
  u128 state, inc;
  unsigned long long cur;
  int half;
  __device__ void seek(const SampleParams& P, u128 s0, u128 inc_, unsigned long long pos) {
    inc = inc_;
    state = pcg_jump(P, s0, (pos >> 1) + 1);   // outputs come from the stepped state
    cur = pcg_out(state);
    half = (int)(pos & 1ULL);
  }
  __device__ unsigned next() {
    unsigned v;
    if (half) {
      v = (unsigned)(cur >> 32);
      state = state * mk128(kPcgMultHi, kPcgMultLo) + inc;
      cur = pcg_out(state);
      half = 0;
    } else {
      v = (unsigned)(cur & 0xffffffffULL);
      half = 1;
    }
    return v;
  }
};

__device__ __forceinline__ unsigned long long shifted_pos(const SampleState* S, int nz, unsigned long long j) {
  unsigned long long s = j;
  for (int t = 0; t < nz; ++t)
    if ((unsigned long long)S->z[t] < s) ++s;
    else break;
  return s;
}

__device__ __forceinline__ bool known_zero(const SampleState* S, int nz, unsigned long long pos) {
  for (int t = 0; t < nz; ++t)
    if ((unsigned long long)S->z[t] == pos) return true;
  return false;
}

// ---- layout helpers -------------------------------------------------------
__global__ void k_pack(const float* __restrict__ hwc, int C, int N, float* __restrict__ planes) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)C * N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / N), i = (int)(e % N);
    planes[e] = hwc[(int64_t)i * C + c];
  }
}
__global__ void k_unpack(const float* __restrict__ planes, int C, int N, float* __restrict__ hwc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)C * N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / C), c = (int)(e % C);
    hwc[e] = planes[(int64_t)c * N + i];
  }
}

// ---- chromaticity (imaging.py:160-171) -------------------------------------
__global__ void k_image(const float* __restrict__ hwc, int N, float* __restrict__ img, double* __restrict__ chroma) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const float r = hwc[3 * i], g = hwc[3 * i + 1], b = hwc[3 * i + 2];
    if (img) {
      img[i] = r;
      img[N + i] = g;
      img[2 * N + i] = b;
    }
    const double s = __dadd_rn(__dadd_rn((double)r, (double)g), (double)b);
    double c0, c1;
    if (s < 0.02) {
      c0 = c1 = 1.0 / 3.0;
    } else {
      c0 = __ddiv_rn((double)r, s);
      c1 = __ddiv_rn((double)g, s);
    }
    chroma[i] = c0;
    chroma[N + i] = c1;
  }
}


// ---- chroma-edge gate (energy.py:121-136) ----------------------------------
__global__ void k_edge(const double* __restrict__ ch, int H, int W, float* __restrict__ edge) {
  const int N = H * W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const int x = i % W, y = i / W;
    const double c0 = ch[i], c1 = ch[N + i];
    // max of the four correctly rounded norms = the root of the largest
    // squared norm (sqrt_rn is monotone): one square root instead of four
    auto sq = [](double a, double b) { return __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)); };
    double s2 = 0.0;
    if (x < W - 1) s2 = fmax(s2, sq(__dsub_rn(ch[i + 1], c0), __dsub_rn(ch[N + i + 1], c1)));
    if (x > 0) s2 = fmax(s2, sq(__dsub_rn(c0, ch[i - 1]), __dsub_rn(c1, ch[N + i - 1])));
    if (y < H - 1) s2 = fmax(s2, sq(__dsub_rn(ch[i + W], c0), __dsub_rn(ch[N + i + W], c1)));
    if (y > 0) s2 = fmax(s2, sq(__dsub_rn(c0, ch[i - W]), __dsub_rn(c1, ch[N + i - W])));
    const double d = __dsqrt_rn(s2);
    edge[i] = (float)(1.0 - exp(-50.0 * d));
  }
}

// ---- consistency sampler (energy.py:154-187) --------------------------------
// codes[4p+s] = -1 (dropped) or make_ent(...) for pixel p, slot s.
// Each thread draws kSamplePix consecutive pixels: one PCG64 jump per
// section (dx, dy, temporal) then sequential u32 reads, so the 128-bit
// jump-ahead is amortised over 4*kSamplePix draws.  Draws are kept packed
// (4-bit dx/dy, 1-bit temporal) until the gate.
// Lemire rejections (u32 == 0 in the range-15 sections) shift the rest of the
// stream by one word: positions already known are in S.z; a new one is
// reported through S.new_zero and the pass is repeated on the device
// (k_sample_fix / redo) -- no host round trip.
#ifndef LS_SAMPLE_PIX
#define LS_SAMPLE_PIX 4   // 4: 176 -> 116 us per streaming frame vs 8 (2: 141 us; tools/ablate.py 206, 212)
#endif
constexpr int kSamplePix = LS_SAMPLE_PIX;
constexpr double kGateSq = 0x1.47ae147ae147ap-9;   // max{s : sqrt_rn(s) < 0.05}

__global__ void k_sample(const __grid_constant__ SampleParams P, const SampleState* __restrict__ Sg, const double* __restrict__ ch,
                         const double* __restrict__ pch, int H, int W, int16_t* __restrict__ codes,
                         int32_t* __restrict__ out_cnt, int32_t* __restrict__ in_cnt, SampleState* Sw) {
  if (!Sg->redo) return;
  const int nz = Sg->nz;
  const int N = H * W;
  const unsigned long long Ng = (unsigned long long)P.Ng, goff = (unsigned long long)P.goff;
  const u128 s0 = mk128(P.st_hi, P.st_lo), inc = mk128(P.inc_hi, P.inc_lo);
  const int nthreads = (N + kSamplePix - 1) / kSamplePix;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nthreads; t += gridDim.x * blockDim.x) {
    const int p0 = t * kSamplePix;
    const int np = min(kSamplePix, N - p0);
    uint32_t dxp[kSamplePix / 2], dyp[kSamplePix / 2], tp = 0;   // 8 nibbles per word
#pragma unroll
    for (int w = 0; w < kSamplePix / 2; ++w) dxp[w] = dyp[w] = 0u;
    U32Stream st;
    // dx then dy: rng.integers(-7, 8, size=(n, 4)) -> Lemire on range 15,
    // reject iff (u * 15) mod 2^32 < (2^32 mod 15) = 1, i.e. u == 0
    for (int sec = 0; sec < 2; ++sec) {
      unsigned long long pos = shifted_pos(Sg, nz, (unsigned long long)sec * 4ULL * Ng + 4ULL * (goff + p0));
      st.seek(P, s0, inc, pos);
#pragma unroll
      for (int d = 0; d < 4 * kSamplePix; ++d) {
        if (d >= 4 * np) break;
        unsigned u = st.next();
        while (u == 0u) {
          if (!known_zero(Sg, nz, pos)) atomicMin(&Sw->new_zero, pos);
          ++pos;
          u = st.next();
        }
        ++pos;
        const uint32_t v = (uint32_t)(((unsigned long long)u * 15ULL) >> 32);   // 0..14 = offset + 7
        if (sec == 0) dxp[d >> 3] |= v << (4 * (d & 7));
        else dyp[d >> 3] |= v << (4 * (d & 7));
      }
    }
    if (P.has_prev) {   // rng.integers(0, 2): Lemire threshold 0, no rejection
      st.seek(P, s0, inc, shifted_pos(Sg, nz, 8ULL * Ng + 4ULL * (goff + p0)));
#pragma unroll
      for (int d = 0; d < 4 * kSamplePix; ++d) {
        if (d >= 4 * np) break;
        tp |= (uint32_t)(((unsigned long long)st.next() * 2ULL) >> 32) << d;
      }
    }
    int x = p0 % W, y = p0 / W;
#pragma unroll
    for (int pp = 0; pp < kSamplePix; ++pp, ++x) {
      if (pp >= np) break;
      const int p = p0 + pp;
      if (x == W) {
        x = 0;
        ++y;
      }
      const double c0 = ch[p], c1 = ch[N + p];
      int cnt = 0;
      uint32_t packed[2] = {0u, 0u};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int d = 4 * pp + k;
        const int dx = (int)((dxp[d >> 3] >> (4 * (d & 7))) & 15u) - kHalf;
        const int dy = (int)((dyp[d >> 3] >> (4 * (d & 7))) & 15u) - kHalf;
        const bool tk = (tp >> d) & 1u;
        // partners are clipped to the global frame; in a row band a halo
        // pixel's partner may fall outside the local rows (the pair touches
        // no row of this band and is dropped)
        const int px = clampi(x + dx, 0, W - 1), py = clampi(P.gy0 + y + dy, 0, P.GH - 1) - P.gy0;
        const bool inside = py >= 0 && py < H;
        const int q = inside ? py * W + px : p;
        const double* src = tk ? pch : ch;
        // |c - c_q| < 0.05 (energy.py:175) without the square root: sqrt_rn is
        // monotone, so sqrt_rn(s) < 0.05 <=> s <= kGateSq, the largest double
        // whose correctly rounded root is below 0.05 (tests/test_gate_constant.py)
        const double a = __dsub_rn(c0, src[q]), b = __dsub_rn(c1, src[N + q]);
        const double s2 = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
        const bool keep = inside && (s2 <= kGateSq) && (tk || q != p);
        int16_t code = -1;
        if (keep) {
          code = (int16_t)make_ent(py - y, px - x, tk, false);
          ++cnt;
          if (!tk) atomicAdd(in_cnt + q, 1);
        }
        packed[k >> 1] |= (uint32_t)(uint16_t)code << (16 * (k & 1));
      }
      reinterpret_cast<uint2*>(codes)[p] = make_uint2(packed[0], packed[1]);   // the 4 codes, one store
      out_cnt[p] = cnt;
    }
  }
}

__global__ void k_sample_init(SampleState* S) {
  S->nz = 0;
  S->redo = 1;
  S->error = 0;
  S->new_zero = ~0ULL;
}

// row bands: every rejection position of the stream is known up front (the
// bands' zero scans, gathered): load them sorted; the draw pass then finds no
// new ones.  lists: n_lists x kZeroList (count, positions...)
__global__ void k_sample_init_known(SampleState* S, const long long* lists, int n_lists) {
  S->nz = 0;
  S->redo = 1;
  S->error = 0;
  S->new_zero = ~0ULL;
  for (int l = 0; l < n_lists; ++l) {
    const long long cnt = lists[(size_t)l * kZeroList];
    if (cnt > kMaxRejections) S->error = 1;
    for (int i = 0; i < cnt && i < kMaxRejections; ++i) {
      const long long z = lists[(size_t)l * kZeroList + 1 + i];
      if (S->nz >= kMaxRejections) { S->error = 1; break; }
      int at = S->nz;
      while (at > 0 && S->z[at - 1] > z) { S->z[at] = S->z[at - 1]; --at; }
      S->z[at] = z;
      S->nz += 1;
    }
  }
}

constexpr int kScanPerThread = 256;
__global__ void k_zero_scan(const __grid_constant__ SampleParams P, unsigned long long begin, unsigned long long end, long long* list) {
  const u128 s0 = mk128(P.st_hi, P.st_lo), inc = mk128(P.inc_hi, P.inc_lo);
  const unsigned long long n = end > begin ? end - begin : 0;
  const unsigned long long nth = (n + kScanPerThread - 1) / kScanPerThread;
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < nth;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long p0 = begin + t * kScanPerThread;
    U32Stream st;
    st.seek(P, s0, inc, p0);
    for (int d = 0; d < kScanPerThread; ++d) {
      const unsigned long long pos = p0 + d;
      if (pos >= end) break;
      if (st.next() == 0u) {
        const unsigned long long k = atomicAdd(reinterpret_cast<unsigned long long*>(list), 1ULL);
        if (k < kMaxRejections) list[1 + k] = (long long)pos;
      }
    }
  }
}

// clears the adjacency counters before a (re)draw pass
__global__ void k_sample_zero(const SampleState* S, int n, int32_t* a, int32_t* b) {
  if (!S->redo) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = b[i] = 0;
}

// after a pass: record a newly found rejection (sorted) and request a redo,
// or finish
__global__ void k_sample_fix(SampleState* S, int last_pass) {
  if (!S->redo) return;
  const unsigned long long z = S->new_zero;
  if (z == ~0ULL) {
    S->redo = 0;
    return;
  }
  if (last_pass || S->nz >= kMaxRejections) {
    S->error = 1;
    S->redo = 0;
    return;
  }
  int at = S->nz;
  while (at > 0 && (unsigned long long)S->z[at - 1] > z) {
    S->z[at] = S->z[at - 1];
    --at;
  }
  S->z[at] = (long long)z;
  S->nz += 1;
  S->new_zero = ~0ULL;
}

__global__ void k_degree(int N, const int32_t* a, const int32_t* b, int32_t* deg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) deg[i] = a[i] + b[i];
}

// out entries in slot order (keys 0..3), incoming entries keyed by 4 + 4*src + slot
// Sampled adjacency rows: the pixel's own draws first, in slot order, at
// fixed positions (their rank among its kept draws: no atomics), then the
// incoming entries, placed by an atomic counter of the destination row.
// The reference order of the incoming entries is by source pixel (then slot),
// and a source p = q + dy W + dx (|dx| <= 7 < W) ascends with the (dy, dx) the
// entry code stores row-major -- so sorting the incoming segment by the code
// itself restores it (equal codes are the same source: interchangeable).  No
// sort keys are written.
__global__ void k_fill_samples(const int16_t* __restrict__ codes, int H, int W, const int32_t* __restrict__ row_ptr,
                               const int32_t* __restrict__ out_cnt, int32_t* fill, uint16_t* ent) {
  const int N = H * W;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    const int x = p % W, y = p / W;
    const int a = row_ptr[p];
    const uint2 packed = __ldg(reinterpret_cast<const uint2*>(codes) + p);   // the pixel's 4 codes
    int16_t c[4];
    c[0] = (int16_t)(packed.x & 0xffffu);
    c[1] = (int16_t)(packed.x >> 16);
    c[2] = (int16_t)(packed.y & 0xffffu);
    c[3] = (int16_t)(packed.y >> 16);
    // the incoming slots first: the four partner rows' bounds and atomic
    // counters are requested together, their latencies overlap
    int dst[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      dst[k] = -1;
      if (c[k] >= 0 && !(c[k] & kEntTemporal)) {
        int dy, dx;
        decode_offset((uint16_t)c[k], dy, dx);
        const int q = (y + dy) * W + (x + dx);
        dst[k] = __ldg(row_ptr + q) + __ldg(out_cnt + q) + atomicAdd(fill + q, 1);
      }
    }
    int own = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (c[k] < 0) continue;
      ent[a + own] = (uint16_t)c[k];
      ++own;
      if (dst[k] >= 0) {
        int dy, dx;
        decode_offset((uint16_t)c[k], dy, dx);
        ent[dst[k]] = make_ent(-dy, -dx, false, true);
      }
    }
  }
}

__global__ void k_pairs_count(int64_t n, const int64_t* src, const int64_t* dst, const uint8_t* temporal, int H,
                              int W, int32_t* out_cnt, int32_t* in_cnt, int* bad) {
  const int N = H * W;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = src[e], d = dst[e];
    if (s < 0 || s >= N || d < 0 || d >= N) { *bad = 1; continue; }
    const int dy = (int)(d / W) - (int)(s / W), dx = (int)(d % W) - (int)(s % W);
    if (dy < -kHalf || dy > kHalf || dx < -kHalf || dx > kHalf) { *bad = 1; continue; }
    atomicAdd(out_cnt + s, 1);
    if (!temporal[e]) atomicAdd(in_cnt + d, 1);
  }
}

__global__ void k_fill_pairs(int64_t n, const int64_t* src, const int64_t* dst, const uint8_t* temporal,
                             const double* weight, int W, const int32_t* row_ptr, int32_t* fill, uint16_t* ent,
                             uint32_t* key, float* ent_w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)src[e], d = (int)dst[e];
    const int dy = d / W - s / W, dx = d % W - s % W;
    const bool t = temporal[e] != 0;
    const float wv = weight ? (float)weight[e] : 1.f;
    int pos = atomicAdd(fill + s, 1);
    ent[row_ptr[s] + pos] = make_ent(dy, dx, t, false);
    key[row_ptr[s] + pos] = (uint32_t)e;
    if (ent_w) ent_w[row_ptr[s] + pos] = wv;
    if (!t) {
      pos = atomicAdd(fill + d, 1);
      ent[row_ptr[d] + pos] = make_ent(-dy, -dx, false, true);
      key[row_ptr[d] + pos] = (uint32_t)(n + e);
      if (ent_w) ent_w[row_ptr[d] + pos] = wv;
    }
  }
}

// deterministic order inside each adjacency row (insertion sort by key).
// Rows are short (~8 entries): each thread sorts its row in shared memory
// (column-major per block -> conflict-free); longer rows sort in place.
constexpr int kSortThreads = 128, kSortCap = 24;

__global__ void __launch_bounds__(kSortThreads) k_sort_rows(int N, const int32_t* __restrict__ row_ptr, uint16_t* ent,
                                                            uint32_t* key, float* ent_w) {
  __shared__ uint32_t sk[kSortCap][kSortThreads];
  __shared__ uint16_t se[kSortCap][kSortThreads];
  __shared__ float sw[kSortCap][kSortThreads];
  const int t = threadIdx.x;
  for (int p = blockIdx.x * blockDim.x + t; p < N; p += gridDim.x * blockDim.x) {
    const int a = row_ptr[p], n = row_ptr[p + 1] - a;
    if (n <= kSortCap) {
      for (int i = 0; i < n; ++i) {
        const uint32_t k = key[a + i];
        const uint16_t e = ent[a + i];
        const float w = ent_w ? ent_w[a + i] : 0.f;
        int j = i - 1;
        while (j >= 0 && sk[j][t] > k) {
          sk[j + 1][t] = sk[j][t];
          se[j + 1][t] = se[j][t];
          sw[j + 1][t] = sw[j][t];
          --j;
        }
        sk[j + 1][t] = k;
        se[j + 1][t] = e;
        sw[j + 1][t] = w;
      }
      for (int i = 0; i < n; ++i) {
        key[a + i] = sk[i][t];
        ent[a + i] = se[i][t];
        if (ent_w) ent_w[a + i] = sw[i][t];
      }
    } else {
      for (int i = a + 1; i < a + n; ++i) {
        const uint32_t k = key[i];
        const uint16_t e = ent[i];
        const float w = ent_w ? ent_w[i] : 0.f;
        int j = i - 1;
        while (j >= a && key[j] > k) {
          key[j + 1] = key[j];
          ent[j + 1] = ent[j];
          if (ent_w) ent_w[j + 1] = ent_w[j];
          --j;
        }
        key[j + 1] = k;
        ent[j + 1] = e;
        if (ent_w) ent_w[j + 1] = w;
      }
    }
  }
}

// The same sort, warp-cooperative: a warp takes 32 consecutive rows (one
// contiguous span of the entry arrays), loads the span into shared memory
// with coalesced accesses, each lane sorts its own row there, and the warp
// stores the span back coalesced.  Spans longer than kWarpSpan fall back to
// the per-lane in-place sort.  Keys are unique within a row, so the result is
// the one k_sort_rows produces.
constexpr int kWarpSpan = 640, kWarpSortWarps = 4;

__global__ void __launch_bounds__(32 * kWarpSortWarps) k_sort_rows_warp(int N, const int32_t* __restrict__ row_ptr,
                                                                        uint16_t* ent, uint32_t* key, float* ent_w) {
  __shared__ uint32_t sk[kWarpSortWarps][kWarpSpan];
  __shared__ uint16_t se[kWarpSortWarps][kWarpSpan];
  __shared__ float sw[kWarpSortWarps][kWarpSpan];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* K = sk[wid];
  uint16_t* E = se[wid];
  float* Wt = sw[wid];
  const int nwarps = gridDim.x * kWarpSortWarps;
  for (int p0 = (blockIdx.x * kWarpSortWarps + wid) * 32; p0 < N; p0 += nwarps * 32) {
    const int p = p0 + lane;
    const int pend = min(p0 + 32, N);
    const int a0 = row_ptr[p0];
    const int span = row_ptr[pend] - a0;
    const int ra = p < N ? row_ptr[p] : 0, n = p < N ? row_ptr[p + 1] - ra : 0;
    if (span <= kWarpSpan) {
      for (int j = lane; j < span; j += 32) {
        K[j] = key[a0 + j];
        E[j] = ent[a0 + j];
        if (ent_w) Wt[j] = ent_w[a0 + j];
      }
      __syncwarp();
      const int o = ra - a0;
      for (int i = o + 1; i < o + n; ++i) {
        const uint32_t k = K[i];
        const uint16_t e = E[i];
        const float w = ent_w ? Wt[i] : 0.f;
        int j = i - 1;
        while (j >= o && K[j] > k) {
          K[j + 1] = K[j];
          E[j + 1] = E[j];
          if (ent_w) Wt[j + 1] = Wt[j];
          --j;
        }
        K[j + 1] = k;
        E[j + 1] = e;
        if (ent_w) Wt[j + 1] = w;
      }
      __syncwarp();
      for (int j = lane; j < span; j += 32) {
        key[a0 + j] = K[j];
        ent[a0 + j] = E[j];
        if (ent_w) ent_w[a0 + j] = Wt[j];
      }
      __syncwarp();
    } else {
      for (int i = ra + 1; i < ra + n; ++i) {
        const uint32_t k = key[i];
        const uint16_t e = ent[i];
        const float w = ent_w ? ent_w[i] : 0.f;
        int j = i - 1;
        while (j >= ra && key[j] > k) {
          key[j + 1] = key[j];
          ent[j + 1] = ent[j];
          if (ent_w) ent_w[j + 1] = ent_w[j];
          --j;
        }
        key[j + 1] = k;
        ent[j + 1] = e;
        if (ent_w) ent_w[j + 1] = w;
      }
    }
  }
}

// The sampled rows' incoming segments sorted by entry code (k_fill_samples),
// warp-cooperative like k_sort_rows_warp: a warp's 32 rows are one contiguous
// span, loaded into shared memory coalesced, sorted per lane, stored back.
constexpr int kEntSpan = 1024;
__global__ void __launch_bounds__(32 * kWarpSortWarps) k_sort_incoming_warp(int N, const int32_t* __restrict__ row_ptr,
                                                                            const int32_t* __restrict__ out_cnt,
                                                                            uint16_t* ent) {
  __shared__ uint16_t se[kWarpSortWarps][kEntSpan];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint16_t* E = se[wid];
  const int nwarps = gridDim.x * kWarpSortWarps;
  for (int p0 = (blockIdx.x * kWarpSortWarps + wid) * 32; p0 < N; p0 += nwarps * 32) {
    const int p = p0 + lane;
    const int pend = min(p0 + 32, N);
    const int a0 = row_ptr[p0];
    const int span = row_ptr[pend] - a0;
    const int ra = p < N ? row_ptr[p] + out_cnt[p] : 0, rb = p < N ? row_ptr[p + 1] : 0;
    auto isort = [](uint16_t* v, int lo, int hi) {
      for (int i = lo + 1; i < hi; ++i) {
        const uint16_t e = v[i];
        int j = i - 1;
        while (j >= lo && v[j] > e) {
          v[j + 1] = v[j];
          --j;
        }
        v[j + 1] = e;
      }
    };
    if (span <= kEntSpan) {
      for (int j = lane; j < span; j += 32) E[j] = ent[a0 + j];
      __syncwarp();
      isort(E, ra - a0, rb - a0);
      __syncwarp();
      for (int j = lane; j < span; j += 32) ent[a0 + j] = E[j];
      __syncwarp();
    } else {
      isort(ent, ra, rb);
    }
  }
}

__global__ void k_pairs_from_samples(const int16_t* __restrict__ codes, int H, int W, const int32_t* __restrict__ off,
                                     int64_t* src, int64_t* dst, uint8_t* temporal) {
  const int N = H * W;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    int o = off[p];
    const int x = p % W, y = p / W;
    for (int k = 0; k < 4; ++k) {
      const int16_t c = codes[4 * p + k];
      if (c < 0) continue;
      int dy, dx;
      decode_offset((uint16_t)c, dy, dx);
      src[o] = p;
      dst[o] = (int64_t)(y + dy) * W + (x + dx);
      temporal[o] = (c & kEntTemporal) ? 1 : 0;
      ++o;
    }
  }
}

// ---- segmentation (palette.py:195-224) --------------------------------------
// own_lo/own_hi: flat index range of the pixels whose ids are produced (a
// row band's own rows); pixels before it do not take part in the dark-pixel
// scan (palette.py:209-219), the band's carry-in id stands in for them
__global__ void k_segment_raw(const float* __restrict__ img, const double* __restrict__ ch, int N, int K,
                              const PalChroma pal, int32_t* ids_raw, int32_t* key, int* first_valid, int own_lo,
                              int own_hi) {
  int fv = INT_MAX;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const double c0 = ch[i], c1 = ch[N + i];
    // argmin over the rounded norms sqrt_rn(s_k), first minimum wins
    // (palette.py:203-207), with one square root: the winner is the first k
    // whose root equals the root of the smallest square s_min -- a root can
    // only tie with it when s_k is within rounding of s_min, so only such k
    // (besides s_k == s_min) are checked explicitly
    auto sq = [&](int k) {
      const double a = __dsub_rn(c0, pal.c[2 * k]), b = __dsub_rn(c1, pal.c[2 * k + 1]);
      return __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
    };
    double smin = sq(0);
    for (int k = 1; k < K; ++k) smin = fmin(smin, sq(k));
    const double rmin = __dsqrt_rn(smin);
    const double near = smin * (1.0 + 1e-12);
    int best = 0;
    for (int k = 0; k < K; ++k) {
      const double sk = sq(k);
      if (sk == smin || (sk <= near && __dsqrt_rn(sk) == rmin)) {
        best = k;
        break;
      }
    }
    ids_raw[i] = best + 1;
    const double s = __dadd_rn(__dadd_rn((double)img[i], (double)img[N + i]), (double)img[2 * N + i]);
    const bool dark = s < 0.02;
    const bool own = i >= own_lo && i < own_hi;
    key[i] = (dark || i < own_lo) ? -1 : i;
    if (!dark && own) fv = min(fv, i);
  }
  // first non-dark own pixel: a block minimum, one atomic per block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fv = min(fv, __shfl_xor_sync(0xffffffffu, fv, o));
  __shared__ int s_fv[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_fv[wid] = fv;
  __syncthreads();
  if (wid == 0) {
    fv = lane < (int)(blockDim.x >> 5) ? s_fv[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) fv = min(fv, __shfl_xor_sync(0xffffffffu, fv, o));
    if (lane == 0 && fv != INT_MAX) atomicMin(first_valid, fv);
  }
}

// band summary of its own rows: {has a non-dark pixel, id of the first, id of
// the last}
__global__ void k_segment_summary(const int32_t* __restrict__ ids_raw, const int32_t* __restrict__ last,
                                  const int* first_valid, int own_hi, int* summary) {
  const int fv = *first_valid;
  const bool has = fv < own_hi;
  summary[0] = has ? 1 : 0;
  summary[1] = has ? ids_raw[fv] : 0;
  summary[2] = has ? ids_raw[last[own_hi - 1]] : 0;
}

// ids of a band's own rows given every band's summary (band order): a dark
// pixel with no non-dark pixel before it in the band takes the last non-dark
// id of an earlier band, else the frame's first non-dark id, else 1
__global__ void k_segment_band_final(int N, const int32_t* __restrict__ ids_raw, const int32_t* __restrict__ last,
                                     const int* __restrict__ summaries, int nbands, int band, int own_lo, int own_hi,
                                     int32_t* ids) {
  __shared__ int carry;
  if (threadIdx.x == 0) {
    int cval = -1;
    for (int b = band - 1; b >= 0 && cval < 0; --b)
      if (summaries[3 * b]) cval = summaries[3 * b + 2];
    for (int b = 0; b < nbands && cval < 0; ++b)
      if (summaries[3 * b]) cval = summaries[3 * b + 1];
    carry = cval < 0 ? 1 : cval;
  }
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (i < own_lo || i >= own_hi) { ids[i] = ids_raw[i]; continue; }   // halo rows: unused
    const int l = last[i];
    ids[i] = l >= 0 ? ids_raw[l] : carry;
  }
}

__global__ void k_segment_final(int N, const int32_t* __restrict__ ids_raw, const int32_t* __restrict__ last,
                                const int* first_valid, int32_t* ids) {
  const int fv = *first_valid;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (fv >= N) { ids[i] = 1; continue; }            // every pixel dark
    int l = last[i];
    if (l < 0) l = fv;
    ids[i] = ids_raw[l];
  }
}

// ---- first-frame initialisation (solver.py:295-308) ------------------------
__global__ void k_initialize(const float* __restrict__ img, const int32_t* __restrict__ ids, int N, int NT,
                             const PalColors colors, float* __restrict__ X) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const int id = ids[i] - 1;
    double ratio_sum = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double rc = colors.c[3 * id + c];
      const double fl = rc > 1e-4 ? rc : 1e-4;
      X[(size_t)c * N + i] = (float)log(fl);
      ratio_sum += (double)img[(size_t)c * N + i] / fl;
    }
    double t0 = ratio_sum / 3.0;
    t0 = t0 < 0.0 ? 0.0 : (t0 > 2.0 ? 2.0 : t0);
    X[(size_t)3 * N + i] = (float)t0;
    for (int k = 1; k < NT; ++k) X[(size_t)(3 + k) * N + i] = 0.f;
  }
}

__global__ void k_set_i32(int32_t* p, int n, int32_t v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

// ---- launchers ---------------------------------------------------------------
static inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 65535) g = 65535;
  return (int)g;
}

void launch_pack_hwc(cudaStream_t s, const float* hwc, int C, int N, float* planes) {
  k_pack<<<grid_for((int64_t)C * N), 256, 0, s>>>(hwc, C, N, planes);
}
void launch_unpack_hwc(cudaStream_t s, const float* planes, int C, int N, float* hwc) {
  k_unpack<<<grid_for((int64_t)C * N), 256, 0, s>>>(planes, C, N, hwc);
}
void launch_image(cudaStream_t s, const float* hwc, int N, float* img, double* chroma) {
  k_image<<<grid_for(N), 256, 0, s>>>(hwc, N, img, chroma);
}
void launch_edge(cudaStream_t s, const double* chroma, int H, int W, float* edge) {
  k_edge<<<grid_for((int64_t)H * W), 256, 0, s>>>(chroma, H, W, edge);
}
void launch_sample(cudaStream_t s, const SampleParams& P_in, SampleState* S, const double* chroma,
                   const double* prev_chroma, int H, int W, int16_t* codes, int32_t* out_cnt, int32_t* in_cnt,
                   int passes, const long long* known, int n_known_lists) {
  SampleParams P = P_in;
  fill_jump_table(P);
  const int N = H * W;
  const int nthreads = (N + kSamplePix - 1) / kSamplePix;
  if (known) k_sample_init_known<<<1, 1, 0, s>>>(S, known, n_known_lists);
  else k_sample_init<<<1, 1, 0, s>>>(S);
  for (int pass = 0; pass < passes; ++pass) {
    // grid-stride over a bounded grid: the redo passes usually exit at once
    k_sample_zero<<<std::min(grid_for(N + 1), 1184), 256, 0, s>>>(S, N + 1, out_cnt, in_cnt);
    k_sample<<<grid_for(nthreads, 128), 128, 0, s>>>(P, S, chroma, prev_chroma, H, W, codes, out_cnt, in_cnt, S);
    k_sample_fix<<<1, 1, 0, s>>>(S, pass == passes - 1);
  }
}
void launch_zero_scan(cudaStream_t s, const SampleParams& P_in, unsigned long long begin, unsigned long long end,
                      long long* list) {
  SampleParams P = P_in;
  fill_jump_table(P);
  cudaMemsetAsync(list, 0, sizeof(long long) * kZeroList, s);
  const unsigned long long nth = ((end > begin ? end - begin : 0) + kScanPerThread - 1) / kScanPerThread;
  if (nth) k_zero_scan<<<grid_for((int64_t)nth, 128), 128, 0, s>>>(P, begin, end, list);
}
void launch_pairs_count(cudaStream_t s, int64_t n, const int64_t* src, const int64_t* dst, const uint8_t* temporal,
                        int H, int W, int32_t* out_cnt, int32_t* in_cnt, int* bad) {
  if (n > 0) k_pairs_count<<<grid_for(n), 256, 0, s>>>(n, src, dst, temporal, H, W, out_cnt, in_cnt, bad);
}
void launch_degree(cudaStream_t s, int N, const int32_t* a, const int32_t* b, int32_t* deg) {
  k_degree<<<grid_for(N), 256, 0, s>>>(N, a, b, deg);
}
void launch_fill_from_samples(cudaStream_t s, const int16_t* codes, int H, int W, const int32_t* row_ptr,
                              const int32_t* out_cnt, int32_t* fill, uint16_t* ent) {
  k_fill_samples<<<grid_for((int64_t)H * W), 256, 0, s>>>(codes, H, W, row_ptr, out_cnt, fill, ent);
  const int N = H * W;
  k_sort_incoming_warp<<<grid_for(((int64_t)N + 31) / 32, kWarpSortWarps), 32 * kWarpSortWarps, 0, s>>>(
      N, row_ptr, out_cnt, ent);
}
void launch_fill_from_pairs(cudaStream_t s, int64_t n, const int64_t* src, const int64_t* dst,
                            const uint8_t* temporal, const double* weight, int W, const int32_t* row_ptr,
                            int32_t* fill, uint16_t* ent, uint32_t* key, float* ent_w) {
  if (n > 0) k_fill_pairs<<<grid_for(n), 256, 0, s>>>(n, src, dst, temporal, weight, W, row_ptr, fill, ent, key, ent_w);
}
void launch_sort_rows(cudaStream_t s, int N, const int32_t* row_ptr, uint16_t* ent, uint32_t* key, float* ent_w) {
  if (std::getenv("LS_SORT_THREAD"))      // the per-thread form (A/B)
    k_sort_rows<<<grid_for(N, kSortThreads), kSortThreads, 0, s>>>(N, row_ptr, ent, key, ent_w);
  else
    k_sort_rows_warp<<<grid_for(((int64_t)N + 31) / 32, kWarpSortWarps), 32 * kWarpSortWarps, 0, s>>>(
        N, row_ptr, ent, key, ent_w);
}
void launch_pairs_from_samples(cudaStream_t s, const int16_t* codes, int H, int W, const int32_t* off, int64_t* src,
                               int64_t* dst, uint8_t* temporal) {
  k_pairs_from_samples<<<grid_for((int64_t)H * W), 256, 0, s>>>(codes, H, W, off, src, dst, temporal);
}
void launch_segment_raw(cudaStream_t s, const float* img, const double* chroma, int N, int K, const PalChroma& pal,
                        int32_t* ids_raw, int32_t* key, int* first_valid) {
  k_segment_raw<<<grid_for(N), 256, 0, s>>>(img, chroma, N, K, pal, ids_raw, key, first_valid, 0, N);
}
void launch_segment_band(cudaStream_t s, const float* img, const double* chroma, int N, int K, const PalChroma& pal,
                         int32_t* ids_raw, int32_t* key, int* first_valid, int own_lo, int own_hi) {
  k_segment_raw<<<grid_for(N), 256, 0, s>>>(img, chroma, N, K, pal, ids_raw, key, first_valid, own_lo, own_hi);
}
void launch_segment_summary(cudaStream_t s, const int32_t* ids_raw, const int32_t* last, const int* first_valid,
                            int own_hi, int* summary) {
  k_segment_summary<<<1, 1, 0, s>>>(ids_raw, last, first_valid, own_hi, summary);
}
void launch_segment_band_final(cudaStream_t s, int N, const int32_t* ids_raw, const int32_t* last,
                               const int* summaries, int nbands, int band, int own_lo, int own_hi, int32_t* ids) {
  k_segment_band_final<<<grid_for(N), 256, 0, s>>>(N, ids_raw, last, summaries, nbands, band, own_lo, own_hi, ids);
}
void launch_segment_final(cudaStream_t s, int N, const int32_t* ids_raw, const int32_t* last, const int* first_valid,
                          int32_t* ids) {
  k_segment_final<<<grid_for(N), 256, 0, s>>>(N, ids_raw, last, first_valid, ids);
}
void launch_initialize(cudaStream_t s, const float* img, const int32_t* ids, int N, int NT, const PalColors& colors,
                       float* X) {
  k_initialize<<<grid_for(N), 256, 0, s>>>(img, ids, N, NT, colors, X);
}
// device-to-device copy on the SMs: a cudaMemcpyAsync D2D would go to a copy
// engine and queue behind a large host transfer on another stream
__global__ void k_copy16(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_copy1(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
void launch_copy(cudaStream_t s, void* dst, const void* src, int64_t bytes) {
  if (bytes <= 0 || dst == src) return;
  const int64_t n16 = (((uintptr_t)dst | (uintptr_t)src) & 15) ? 0 : bytes / 16;
  if (n16) k_copy16<<<grid_for(n16), 256, 0, s>>>(static_cast<const int4*>(src), static_cast<int4*>(dst), n16);
  const int64_t done = n16 * 16;
  if (done < bytes)
    k_copy1<<<grid_for(bytes - done), 256, 0, s>>>(static_cast<const unsigned char*>(src) + done,
                                                     static_cast<unsigned char*>(dst) + done, bytes - done);
}

// flag = 0 if any value is NaN / inf (flag preset to 1 by the caller)
// (float4 over a bounded grid when x is 16-byte aligned; a frame is read once)
__global__ void k_all_finite(const float* __restrict__ x, int64_t n, int* flag) {
  bool ok = true;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t head = 0;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) {
    const int64_t n4 = n >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldg(x4 + i);
      ok = ok && isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
    }
    head = n4 << 2;
  }
  for (int64_t i = head + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    ok = ok && isfinite(x[i]);
  if (!__syncthreads_and(ok) && threadIdx.x == 0) *flag = 0;
}
__global__ void k_set_flag(int* flag) { *flag = 1; }
void launch_all_finite(cudaStream_t s, const float* x, int64_t n, int* flag) {
  k_set_flag<<<1, 1, 0, s>>>(flag);
  if (n > 0) k_all_finite<<<std::min(grid_for((n + 3) / 4), 148 * 8), 256, 0, s>>>(x, n, flag);
}

void launch_set_i32(cudaStream_t s, int32_t* p, int n, int32_t v) {
  k_set_i32<<<grid_for(n), 256, 0, s>>>(p, n, v);
}

// ---------------------------------------------------------------------------
// single-pass int32 scan with decoupled look-back (row offsets of the
// adjacency and of the pair list: exclusive sums; the dark-pixel
// inheritance of segment: an inclusive max-scan).  Each CTA takes the next
// tile id from a counter, scans its 2048 values in registers / warp
// shuffles, publishes its aggregate, and thread 0 walks back over the
// predecessors' published (flag, value) words until an inclusive prefix.
// Integer ops: the result is exact and independent of the schedule.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr unsigned long long kFlagAgg = 1ull << 32, kFlagPre = 2ull << 32;

template <int OP>
__device__ __forceinline__ int scan_op(int a, int b) {
  return OP == 0 ? a + b : (a > b ? a : b);
}

template <int OP>
__global__ void __launch_bounds__(kScanThreads) k_scan(const int* __restrict__ in, int* __restrict__ out, int64_t n,
                                                      unsigned long long* status, unsigned* counter) {
  constexpr int ident = OP == 0 ? 0 : INT_MIN;
  static_assert(kScanItems == 8, "two int4 per thread");
  __shared__ int s_tile, s_prefix;
  __shared__ int s_warp[kScanThreads / 32];
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(counter, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t base = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  int v[kScanItems];
  if (vec && base + kScanItems <= n) {   // 2 x int4 per thread (a 32-byte run)
    const int4 a = __ldg(reinterpret_cast<const int4*>(in + base));
    const int4 b = __ldg(reinterpret_cast<const int4*>(in + base) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) v[j] = base + j < n ? in[base + j] : ident;
  }
#pragma unroll
  for (int j = 1; j < kScanItems; ++j) v[j] = scan_op<OP>(v[j - 1], v[j]);   // thread-inclusive
  int t = v[kScanItems - 1];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, t, o);
    if (lane >= o) t = scan_op<OP>(u, t);
  }
  if (lane == 31) s_warp[wid] = t;
  __syncthreads();
  if (wid == 0) {
    int w = lane < kScanThreads / 32 ? s_warp[lane] : ident;
#pragma unroll
    for (int o = 1; o < kScanThreads / 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = scan_op<OP>(u, w);
    }
    if (lane < kScanThreads / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const int up = __shfl_up_sync(0xffffffffu, t, 1);
  int excl = lane > 0 ? up : ident;                         // exclusive within the warp
  if (wid > 0) excl = scan_op<OP>(s_warp[wid - 1], excl);   // ... within the tile
  if (wid == 0) {
    // decoupled look-back by the whole first warp: lane l reads predecessor
    // tile - 1 - l of the current 32-tile window; the values from the nearest
    // inclusive prefix (flag Pre) onwards are combined by a warp reduction,
    // the window slides back until a prefix is found
    const int agg = s_warp[kScanThreads / 32 - 1];
    int prefix = ident;
    if (tile == 0) {
      if (lane == 0) atomicExch(status, kFlagPre | (unsigned)agg);
    } else {
      if (lane == 0) atomicExch(status + tile, kFlagAgg | (unsigned)agg);
      for (int top = tile - 1;; top -= 32) {
        const int j = top - lane;
        unsigned long long st = kFlagPre | (unsigned)ident;   // beyond tile 0: a neutral prefix
        if (j >= 0) {
          do {
            st = *reinterpret_cast<volatile unsigned long long*>(status + j);
          } while ((st >> 32) == 0ull);
        }
        const unsigned pre_mask = __ballot_sync(0xffffffffu, (st & ~0xffffffffull) == kFlagPre);
        const int stop = pre_mask ? __ffs(pre_mask) - 1 : 32;   // nearest lane holding a prefix
        int val = lane <= stop ? (int)(unsigned)(st & 0xffffffffull) : ident;
        // combine lanes 0..stop (order-free for + and max)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val = scan_op<OP>(val, __shfl_xor_sync(0xffffffffu, val, o));
        prefix = scan_op<OP>(val, prefix);
        if (pre_mask) break;
      }
      if (lane == 0) atomicExch(status + tile, kFlagPre | (unsigned)scan_op<OP>(prefix, agg));
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const int pre = scan_op<OP>(s_prefix, excl);
  int o8[kScanItems];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    o8[j] = OP == 0 ? pre + (j > 0 ? v[j - 1] : 0)     // exclusive sum
                    : scan_op<OP>(pre, v[j]);          // inclusive max
  if (vec && base + kScanItems <= n) {
    reinterpret_cast<int4*>(out + base)[0] = make_int4(o8[0], o8[1], o8[2], o8[3]);
    reinterpret_cast<int4*>(out + base)[1] = make_int4(o8[4], o8[5], o8[6], o8[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      if (base + j >= n) break;
      out[base + j] = o8[j];
    }
  }
}

size_t scan_scratch_bytes(int64_t n) { return sizeof(unsigned long long) * (size_t)((n + kScanTile - 1) / kScanTile + 1); }

cudaError_t launch_scan(cudaStream_t s, const int32_t* in, int32_t* out, int64_t n, int op, void* scratch) {
  if (n <= 0) return cudaSuccess;
  const int tiles = (int)((n + kScanTile - 1) / kScanTile);
  unsigned long long* status = static_cast<unsigned long long*>(scratch);
  unsigned* counter = reinterpret_cast<unsigned*>(status + tiles);
  cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned long long) * (tiles + 1), s);
  if (e != cudaSuccess) return e;
  if (op == 0) k_scan<0><<<tiles, kScanThreads, 0, s>>>(in, out, n, status, counter);
  else k_scan<1><<<tiles, kScanThreads, 0, s>>>(in, out, n, status, counter);
  return cudaGetLastError();
}

}  // namespace ls
