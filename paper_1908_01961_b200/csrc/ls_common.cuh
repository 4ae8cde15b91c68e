// Shared device-side definitions for the lumisplit B200 kernels.
//
// Data layout in HBM: every per-pixel field is a
// set of planes of N = H*W float32 values, row-major.  The layer state X has
// U = NT + 3 planes: r (3) then T_0..T_{NT-1} (NT = K+1).  PCG vectors use
// the same plane order, i.e. the reference vector [r.ravel(), T.ravel()]
// (solver.py:110-122) up to the (H,W,C) -> (C,H,W) permutation.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ls {

constexpr int kMaxNT = 13;        // K <= 12
constexpr int kTerms = 8;
constexpr int kHalf = 7;          // CONSISTENCY_WINDOW // 2 (energy.py:23)
constexpr int kWin = 15;
constexpr int kTileW = 32;        // one warp per tile row
#ifndef LS_TILE_H
#define LS_TILE_H 8
#endif
constexpr int kTileH = LS_TILE_H;   // warps per block (one per tile row)
constexpr int kThreads = kTileW * kTileH;
// resident CTAs per SM the stencil kernels are compiled for (80 registers)
constexpr int kStencilMinBlocks = kTileH <= 8 ? 3 : 2;
constexpr int kHaloW = kTileW + 2 * kHalf;
constexpr int kHaloH = kTileH + 2 * kHalf;
constexpr int kMaxBlocks = 4096;  // partial-sum slots per reduction

// adjacency entry (uint16): bits 0-9 the partner offset pre-encoded for the
// 48-wide shared-memory window of the operand's r planes,
// (dy+7)*48 + (dx+7); bit 10 temporal; bit 11 incoming (pixel is the dst).
constexpr int kEntRW = 48;
constexpr int kEntBias = kHalf * kEntRW + kHalf;
constexpr uint16_t kEntOffMask = 0x3ff;
constexpr uint16_t kEntTemporal = 1u << 10;
constexpr uint16_t kEntIncoming = 1u << 11;

__host__ __device__ __forceinline__ uint16_t make_ent(int dy, int dx, bool temporal, bool incoming) {
  return (uint16_t)(((dy + kHalf) * kEntRW + (dx + kHalf)) | (temporal ? kEntTemporal : 0) |
                    (incoming ? kEntIncoming : 0));
}
// partner offset inside the 48-wide smem window
__host__ __device__ __forceinline__ int ent_soff(uint16_t e) { return (int)(e & kEntOffMask) - kEntBias; }

enum Term { T_DATA = 0, T_CLUSTER, T_RSPARSE, T_CONSIST, T_MONO, T_ISPARSE, T_SMOOTH, T_NONNEG };

// Frozen coefficients of the energy (EnergyWeights + palette), both in fp32
// (the PCG operator) and fp64 (energies, gradient, diagonal).
template <typename R>
struct Coef {
  R B[kMaxNT][3];      // palette matrix, row 0 white (palette.py:64-66)
  R G[kMaxNT][3];      // B - rowmean(B) (energy.py:396)
  R anchor[kMaxNT][3]; // log(max(color[id-1], 1e-4)) indexed by id (energy.py:470-472)
  R g2[kMaxNT];        // sum_c G[k][c]^2 (monochrome diagonal, energy.py:410-411), fma order of the kernels
  R lam_d, lam_cl, lam_rs, p, lam_rc, lam_m, lam_is, lam_sm, lam_nn;
  R eps_nn, eps_irls, inv_eps, floor_rs;
};

struct Frame {
  int H, W, N, NT;
  const float* img;       // 3 planes
  const float* edge;      // N
  const int32_t* ids;     // N or nullptr
  const float* anchor;    // 3 planes or nullptr (fixed log anchor)
  const float* prev_r;    // 3 planes or nullptr
  const int32_t* row_ptr; // N + 1
  const uint16_t* ent;    // adjacency entries
  const float* ent_w;     // per-entry pair weight or nullptr (all 1)
  // row band: the kernels produce rows [y_lo, y_hi)
  // of this H x W local frame; rows outside are halo copies of the
  // neighbouring bands.  A whole frame is y_lo = 0, y_hi = H.
  int y_lo, y_hi;
  // band partial mode: the last CTA writes its reduced sums here instead of
  // finalising the scalars (ls_band_finalize sums the bands in band order)
  double* bsum;
};

// device-resident PCG / step scalars (textbook Jacobi PCG of solver.py:79-107
// with the p-update fused into the operator kernel and a deferred x-update)
struct Scalars {
  double gamma, gamma_prev;   // rz_i = <r_i, z_i>, rz_{i-1}
  double delta;               // pAp_i
  double alpha, alpha_prev, beta;
  double bnorm2, rnorm2;
  double terms0[kTerms];      // energies at the linearisation point
  double terms1[kTerms];      // energies at the last trial point
  int iterations;
  int stop;
  int pending;                // (unused; kept for layout stability)
  int xinit;                  // x has been written (else it is zero)
  int plast;
  int ls_done;                // device line search: decided
  int accepted;
  int fault;                  // non-finite energy at the linearisation point
  double alpha_ls;            // accepted step length
  double e0, e1;              // Python-sum order of terms0 / terms1 (solver.py:139-140)
  double alpha_hist[64];      // alpha_i of every iteration (x = sum alpha_i p_i, k_pcg_combine)
};
constexpr int kMaxStoredDirs = 64;

// device-resident flip-flop of a streaming frame (solver.py:311-338 with
// refine = False): convergence test and step bookkeeping on the GPU
struct FrameCtl {
  int done;                   // converged or faulted: later kernels are no-ops
  int converged;
  int stalled;
  int has_hist;               // energy_history non-empty
  int e_prev_valid;
  int n_exec;                 // GN steps executed (records written)
  int cur;                    // which of the two state buffers holds the state
  int fault_step;             // index of a faulting step, -1 if none
  double e_last, e_prev;
};

struct StepRecord {
  double e0, e1, alpha, bnorm2, rnorm2;
  double terms0[kTerms], terms1[kTerms];
  int accepted, iterations, fault, pad;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may be scheduled before its
// predecessor finishes; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible (a no-op without the attribute), and
// pdl_trigger() lets this grid's successor be scheduled onto SMs as this
// grid's CTAs retire -- hiding the launch latency and the tail of every
// kernel boundary of the solver's graph.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename R>
__device__ __forceinline__ R irls1(R mag, R eps, R inv_eps) {
  // energy.py:102-112 with p = 1: 1/|m| above the floor eps, else 1/eps
  mag = mag < R(0) ? -mag : mag;
  return mag >= eps ? R(1) / mag : inv_eps;
}

template <typename R>
__device__ __forceinline__ R irlsp(R mag, const Coef<R>& c) {
  // general p (r-sparsity only): min(|m|^(p-2), 1/eps), floor eps^(1/(2-p))
  if (c.p >= R(2)) return R(1);
  mag = mag < R(0) ? -mag : mag;
  if (!(mag >= c.floor_rs)) return c.inv_eps;
  if (c.p == R(1)) return R(1) / mag;
  return pow(mag, c.p - R(2));
}

template <typename R>
__device__ __forceinline__ R nonneg_w(R t, R eps) {
  // energy.py:115-118
  return t > R(0) ? R(0) : R(1) / ((t < R(0) ? -t : t) + eps);
}

__host__ __device__ __forceinline__ void decode_offset(uint16_t e, int& dy, int& dx) {
  const int code = e & kEntOffMask;
  dy = code / kEntRW - kHalf;
  dx = code % kEntRW - kHalf;
}

// ---- deterministic block reduction + last-block finalisation -------------
// Each block reduces NV doubles (fixed shuffle tree), writes them to
// part[blockIdx.x * NV + j]; the last block to arrive (ticket) sums the
// partials over blocks in a fixed order and calls fin(j, total).
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* part) {
  __shared__ double red[kThreads / 32][NV];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double a = v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0) red[wid][j] = a;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    part[(size_t)blockIdx.x * NV + threadIdx.x] = s;
  }
}

// returns true in the (whole) last block after all partials are visible
__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(ticket, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// sum partial j over all blocks with a fixed assignment + fixed tree;
// result valid in thread 0.
template <int NV>
__device__ __forceinline__ double sum_partials(const double* part, int nblocks, int j) {
  __shared__ double red2[kThreads / 32];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += ((volatile const double*)part)[(size_t)b * NV + j];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  __syncthreads();
  if (lane == 0) red2[wid] = s;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red2[w];
  __syncthreads();
  return t;
}

}  // namespace ls

// ---- TMA / mbarrier helpers (sm_90+ PTX, used on sm_100a) -----------------
#include <cuda.h>

namespace ls {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 3-D tiled TMA load of box (c0, c1, c2) into shared memory; out-of-bounds
// elements (including negative coordinates) are zero-filled by the hardware
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace ls
