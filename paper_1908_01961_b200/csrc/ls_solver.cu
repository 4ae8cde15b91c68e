// Sparse-phase kernels of the alternating solver.
//
//   k_energy<NT, MODE_EG>    fused: 8 term energies at the linearisation point,
//                            b = -J^T F, diag(J^T J), Jacobi PCG init
//                            (energy.py:194-511, solver.py:125-140, 79-91)
//   k_energy<NT, MODE_TRIAL> line-search trial: candidate Y = X + a*dx (or an
//                            external Y) written, 8 energies with the IRLS
//                            weights frozen at X (solver.py:166-178)
//   k_apply<NT>              w = J^T J u (matrix-free, solver.py:110-122), the
//                            API operator (ls_apply_normal)
//   k_pcg_apply<NT>          PCG iteration: p = z + beta p formed over the
//                            tile + halo, q = J^T J p, <p,q>, deferred x-update
//   k_pcg_update             r -= alpha q, z = r / diag, <r,z>, |r|^2
//   k_pcg_xfinal             the last deferred x-update
//
// Tile scheme: persistent blocks of 256 threads walk 32x8 pixel tiles (one
// warp per tile row).  Each tile stages in shared memory
//   sX  all U state planes, tile + 1-pixel halo   (frozen weights, data term)
//   sT  the T planes of the operand, + 1 halo     (smoothness stencil)
//   sR  the 3 r planes of the operand, + 7 halo   (r-sparsity stencil and the
//                                                   15x15 consistency window,
//                                                   energy.py:23, 161-173)
// by TMA (cp.async.bulk.tensor.3d boxes, mbarrier completion), so every HBM
// word is read once per tile and all neighbour / partner reads hit shared
// memory.  IRLS weights are recomputed
// from sX (cheaper than storing 2K+3 weight planes).  Per-pixel arithmetic is
// fp32 (the data residual exactly rounded via fp64 FMA); reductions are fp64,
// fixed order, finished by the last block (no float atomics).
#include <cstdlib>
#include <string>
#include <utility>

#include "ls_common.cuh"
#include "ls_kernels.h"

// timing ablations of k_pcg_apply (tools/ablate.py only; 0 in every product build)
#ifndef LS_ABLATE
#define LS_ABLATE 0
#endif
#ifndef LS_XEARLY
#define LS_XEARLY 0
#endif
#ifndef LS_XDEFER
#define LS_XDEFER 0
#endif
// LS_PEARLY (default 1): the operator kernel prefetches the next tile's
// p_{i-1} window into the p region as soon as the current tile's operand is
// formed, on its own mbarrier (142.4 -> 140.7 us at 1080p K=8)
#ifndef LS_PEARLY
#define LS_PEARLY 1
#endif
// LS_PFORM_GLOBAL=1: the operator forms p = z + beta p_{i-1} with p_{i-1}
// read from global memory (L2) instead of a staged window: half the operand
// shared memory (46 KB per CTA)
#ifndef LS_PFORM_GLOBAL
#define LS_PFORM_GLOBAL 0
#endif
// LS_KEEP_R=1: round 1's PCG update (r and z stored, 5U per iteration)
#ifndef LS_KEEP_R
#define LS_KEEP_R 0
#endif

namespace ls {

// LS_PDL=1: launches of the solver's kernel sequence carry the programmatic-
// serialization attribute (PDL, see pdl_wait in ls_common.cuh).  Off by
// default: measured in the captured frame graph at 1080p K=8, 52.0 vs 54.6
// frames/s with it -- the kernels' own times are
// unchanged, the graph's kernel boundaries got slower.
static bool pdl_on() {
  static const bool on = std::getenv("LS_PDL") != nullptr && std::string(std::getenv("LS_PDL")) == "1";
  return on;
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

enum { MODE_EG = 0, MODE_TRIAL = 1 };

// shared-memory tile geometry (row widths padded to 16-byte TMA boxes)
// TMA requires the innermost box start to be 16-byte aligned, so the 1-halo
// window starts 4 columns left of the tile and the 7-halo window 8 columns.
constexpr int kSX = 4;                // column of tile x = 0 in a 1-halo row
constexpr int kSW = 40;               // 1-halo rows: cols tx0-4 .. tx0+35
constexpr int kSH = kTileH + 2;       // rows ty0-1 .. ty0+8
constexpr int kSP = kSW * kSH;        // floats per 1-halo plane
constexpr int kRX = 8;                // column of tile x = 0 in a 7-halo row
constexpr int kRW = 48;               // 7-halo rows: cols tx0-8 .. tx0+39
constexpr int kRP = kRW * kHaloH;     // rows ty0-7 .. ty0+14 (48 x 22)

__host__ __device__ constexpr int pad32(int v) { return (v + 31) & ~31; }   // 128-byte regions
__host__ __device__ constexpr int off_T(int NT) { return pad32((NT + 3) * kSP); }
__host__ __device__ constexpr int off_R(int NT, bool has_T) { return off_T(NT) + (has_T ? pad32(NT * kSP) : 0); }
__host__ __device__ constexpr int tile_floats(int NT, bool has_T) { return off_R(NT, has_T) + pad32(3 * kRP); }

// MUFU reciprocal / rsqrt (one instruction).  The IRLS weights only have to
// be the same deterministic function in every kernel; 1-ulp differences to
// the fp64 reference are far below the solver's tolerance.
__device__ __forceinline__ float rcpf(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float rsqrtf_fast(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// Tile coordinates of a persistent CTA's walk (tile = blockIdx.x + j gridDim.x)
// kept incrementally: the div / mod by the tile-row count cost ~35
// instructions per thread and tile (~3% of the operator's) when recomputed.
#ifndef LS_UPD_F32P
#define LS_UPD_F32P 0
#endif
#ifndef LS_TILEWALK
#define LS_TILEWALK 1   // 0: recompute tile / ntx, tile % ntx every tile (A/B)
#endif
struct TileWalk {
  int tx, ty, sx, sy, ntx;
  __device__ __forceinline__ TileWalk(int t0, int stride, int n) : ntx(n) {
    tx = t0 % n;
    ty = t0 / n;
    sx = stride % n;
    sy = stride / n;
  }
  __device__ __forceinline__ void next(int& nx, int& ny) const {
    nx = tx + sx;
    ny = ty + sy;
    if (nx >= ntx) {
      nx -= ntx;
      ++ny;
    }
  }
  __device__ __forceinline__ void advance() { next(tx, ty); }
};

// non-negativity weight (energy.py:115-118) with the MUFU reciprocal
__device__ __forceinline__ float nonneg_wf(float t, float eps) { return t > 0.f ? 0.f : rcpf(fabsf(t) + eps); }

// smoothness / i-sparsity IRLS factor (p = 1): 1/|g| above eps, else 1/eps
// (min(1/|g|, 1/eps) as one MUFU reciprocal of max(|g|, eps))
__device__ __forceinline__ float irls1f(float g, const Coef<float>& c) {
  return rcpf(fmaxf(fabsf(g), c.eps_irls));
}

// r-sparsity IRLS factor from the squared gradient magnitude s = |grad r|^2
__device__ __forceinline__ float irls_sq(float s, const Coef<float>& c) {
  if (c.p == 1.f) return rsqrtf_fast(fmaxf(s, c.eps_irls * c.eps_irls));
  if (c.p >= 2.f) return 1.f;
  const float mag = sqrtf(s);
  if (!(mag >= c.floor_rs)) return c.inv_eps;
  return powf(mag, c.p - 2.f);
}

// r-sparsity weight at smem coords (ix, iy) of the 1-halo state tile; hx / hy
// say whether the pixel has a right / lower neighbour in the image
__device__ __forceinline__ float wrs_s(const float* sX, int ix, int iy, bool hx, bool hy, const Coef<float>& c,
                                       int RW = kSW, int RP = kSP) {
  float sx = 0.f, syy = 0.f;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float* P = sX + ch * RP;
    const float v = P[iy * RW + ix];
    const float gx = hx ? P[iy * RW + ix + 1] - v : 0.f;
    const float gy = hy ? P[(iy + 1) * RW + ix] - v : 0.f;
    sx = fmaf(gx, gx, sx);
    syy = fmaf(gy, gy, syy);
  }
  return c.lam_rs * irls_sq(sx + syy, c);
}

// cooperative row loads of one tile: each warp takes whole (plane, row)
// segments, lanes walk the columns -- coalesced, no per-element div/mod.
// WIDTH x ROWS window starting HALO pixels up/left of the tile corner;
// optional Y = X + alpha*dx on the fly.
template <int NPL, int WIDTH, int ROWS, int XOFF, int HALO>
__device__ __forceinline__ void load_rows(float* dst, const float* __restrict__ src, const float* __restrict__ dx,
                                          float alpha, int N, int W, int H, int tx0, int ty0) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = kThreads / 32;
#pragma unroll 2
  for (int pr = wid; pr < NPL * ROWS; pr += NW) {
    const int p = pr / ROWS, r = pr - p * ROWS;
    const int gy = ty0 - HALO + r;
    const bool rowok = gy >= 0 && gy < H;
    const size_t rowoff = (size_t)p * N + (size_t)(rowok ? gy : 0) * W;
    float* d = dst + p * (ROWS * WIDTH) + r * WIDTH;
#pragma unroll
    for (int cc = lane; cc < WIDTH; cc += 32) {
      const int gx = tx0 - XOFF + cc;
      float v = 0.f;
      if (rowok && gx >= 0 && gx < W) {
        v = __ldg(src + rowoff + gx);
        if (dx) v = __fmaf_rn(alpha, __ldg(dx + rowoff + gx), v);
      }
      d[cc] = v;
    }
  }
}

template <int NPL>
__device__ __forceinline__ void load_halo1(float* dst, const float* __restrict__ src, int N, int W, int H, int tx0,
                                           int ty0) {
  load_rows<NPL, kSW, kSH, kSX, 1>(dst, src, nullptr, 0.f, N, W, H, tx0, ty0);
}

template <int NPL>
__device__ __forceinline__ void load_halo1_axpy(float* dst, const float* __restrict__ X, const float* __restrict__ dx,
                                                float alpha, int N, int W, int H, int tx0, int ty0) {
  load_rows<NPL, kSW, kSH, kSX, 1>(dst, X, dx, alpha, N, W, H, tx0, ty0);
}

__device__ __forceinline__ void load_halo7(float* dst, const float* __restrict__ src, const float* __restrict__ dx,
                                           float alpha, int N, int W, int H, int tx0, int ty0) {
  load_rows<3, kRW, kHaloH, kRX, kHalf>(dst, src, dx, alpha, N, W, H, tx0, ty0);
}

// TMA boxes of one tile: all state planes / operand T planes (1 halo) and the
// operand r planes (7 halo); see TileMaps in ls_kernels.h
template <int NT>
__device__ __forceinline__ void tma_issue_tile(float* stage, const TileMaps& m, uint64_t* bar, int tx0, int ty0) {
  constexpr uint32_t bytes = sizeof(float) * ((NT + 3) * kSP + NT * kSP + 3 * kRP);
  mbar_expect_tx(bar, bytes);
  tma_load_3d(stage, &m.X, bar, tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(stage + off_T(NT), &m.T, bar, tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(stage + off_R(NT, true), &m.R, bar, tx0 - kRX, ty0 - kHalf, 0);
}

// ---------------------------------------------------------------------------
// energy (+ gradient / diagonal / PCG init) kernel
// ---------------------------------------------------------------------------
// Shared-memory stage (TMA boxes, zero-filled outside the image):
//   sX  U state planes, 1 halo       sXR the 3 state r planes, 7 halo
//   sD  U planes of dx / Y, 1 halo   sDR their r planes, 7 halo   (trial only)
// In trial mode the evaluation point Y = X + alpha*dx is formed in place in
// sD / sDR right after the tile lands (the owner writes exactly these values
// to X_out, so the accepted state is the state that was evaluated).
__host__ __device__ constexpr int e_off_XR(int NT) { return pad32((NT + 3) * kSP); }
__host__ __device__ constexpr int e_off_D(int NT) { return e_off_XR(NT) + pad32(3 * kRP); }
__host__ __device__ constexpr int e_off_DR(int NT) { return e_off_D(NT) + pad32((NT + 3) * kSP); }
__host__ __device__ constexpr int e_stage(int NT, bool trial) {
  return trial ? e_off_DR(NT) + pad32(3 * kRP) : e_off_D(NT);
}

template <int NT>
__device__ __forceinline__ void tma_issue_energy(float* stage, const EnergyMaps& m, uint64_t* bar, int tx0, int ty0,
                                                 bool with_d) {
  constexpr uint32_t half = sizeof(float) * ((NT + 3) * kSP + 3 * kRP);
  mbar_expect_tx(bar, with_d ? 2 * half : half);
  tma_load_3d(stage, &m.X, bar, tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(stage + e_off_XR(NT), &m.XR, bar, tx0 - kRX, ty0 - kHalf, 0);
  if (with_d) {
    tma_load_3d(stage + e_off_D(NT), &m.D, bar, tx0 - kSX, ty0 - 1, 0);
    tma_load_3d(stage + e_off_DR(NT), &m.DR, bar, tx0 - kRX, ty0 - kHalf, 0);
  }
}

// per-pixel energy terms (+ gradient / diagonal / PCG init in MODE_EG);
// acc[] receives the 8 term energies (fp32 per pixel) and rz, |b|^2
// per-pixel global inputs of the energy kernel, read before the tile's TMA
// wait so their latency overlaps it
struct EPre {
  float img[3];
  float edge;
  int id, e0, e1;
};
__device__ __forceinline__ EPre energy_prefetch(const Frame& f, int x, int y, bool own) {
  // branch-free (pixel 0 stands in for a pixel outside the image; its values
  // are never used): inside an `if`, the compiler converted the image values
  // to fp64 right after their loads, stalling on them before the TMA wait
  EPre p;
  const int i = own ? y * f.W + x : 0;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) p.img[ch] = __ldg(f.img + ch * f.N + i);
  p.edge = __ldg(f.edge + i);
  p.id = f.ids ? __ldg(f.ids + i) : 0;
  p.e0 = __ldg(f.row_ptr + i);
  p.e1 = __ldg(f.row_ptr + i + 1);
  return p;
}

template <int NT, int MODE, bool IN>
__device__ __forceinline__ void energy_pixel(const Frame& f, const Coef<float>& c, const float* sX, const float* sXR,
                                             const float* sYT, const float* sYR, int x, int y, int cx, int cy,
                                             int rx, int ry, float* __restrict__ Xout, float* __restrict__ r_out,
                                             float* __restrict__ d_out, float* __restrict__ u_out,
                                             float* __restrict__ b_raw, float* __restrict__ diag_raw,
                                             double* acc, const EPre& pre) {
  const int W = f.W, H = f.H, N = f.N;
  const int i = y * W + x;
  const bool hx = IN || x < W - 1, hy = IN || y < H - 1, hl = IN || x > 0, hu = IN || y > 0;
  const int sc0 = cy * kSW + cx, rc0 = ry * kRW + rx;
  float r0[3], T0[NT], yr[3], yT[NT];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    r0[ch] = sXR[ch * kRP + rc0];
    yr[ch] = sYR[ch * kRP + rc0];
  }
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    T0[k] = sX[(3 + k) * kSP + sc0];
    yT[k] = sYT[k * kSP + sc0];
  }
  float img[3], anc[3];
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) img[ch] = pre.img[ch];
  if (f.ids) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) anc[ch] = c.anchor[pre.id][ch];
  } else {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) anc[ch] = __ldg(f.anchor + ch * N + i);
  }
  const float lm = c.lam_m * pre.edge;

  // data (energy.py:207-209), clustering (234-235), monochrome (399-401)
  float S[3], R[3], res[3], m[3];
  double e_data = 0.0;
  float e_cl = 0.f, e_mono = 0.f;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NT; ++k) s = fmaf(yT[k], c.B[k][ch], s);
    S[ch] = s;
    R[ch] = expf(yr[ch]);
    const double rd = fma(-(double)R[ch], (double)S[ch], (double)img[ch]);   // exactly rounded residual
    e_data = fma(rd, rd, e_data);
    res[ch] = (float)rd;
    const float dc = yr[ch] - anc[ch];
    e_cl = fmaf(dc, dc, e_cl);
  }
  const float mean = (S[0] + S[1] + S[2]) * (1.f / 3.f);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    m[ch] = S[ch] - mean;
    e_mono = fmaf(m[ch], m[ch], e_mono);
  }
  acc[T_DATA] += (double)c.lam_d * e_data;
  acc[T_CLUSTER] += (double)(c.lam_cl * e_cl);
  acc[T_MONO] += (double)(lm * e_mono);

  // r-sparsity: weight from X, gradient of Y (energy.py:264-267, 301-305)
  const float wrs = wrs_s(sXR, rx, ry, hx, hy, c, kRW, kRP);
  {
    float e = 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float* P = sYR + ch * kRP + rc0;
      const float gx = hx ? P[1] - yr[ch] : 0.f;
      const float gy = hy ? P[kRW] - yr[ch] : 0.f;
      e = fmaf(gx, gx, fmaf(gy, gy, e));
    }
    acc[T_RSPARSE] += (double)(wrs * e);
  }

  // per-layer diagonal terms and smoothness (energy.py:414-452, 308-318); in
  // MODE_EG the T_k rows of g = J^T F and diag(J^T J) are produced in the
  // same pass, reusing the two smoothness weights the energy needs
  float rz = 0.f, bb = 0.f;
  {
    float eis = 0.f, enn = 0.f, esm = 0.f;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const float* P = sX + (3 + k) * kSP + sc0;
      const float* Q = sYT + k * kSP + sc0;
      const float wis = (k >= 1) ? c.lam_is * irls1f(T0[k], c) : 0.f;
      const float wnn = c.lam_nn * nonneg_wf(T0[k], c.eps_nn);
      eis = fmaf(wis * yT[k], yT[k], eis);
      enn = fmaf(wnn * yT[k], yT[k], enn);
      float wx = 0.f, wy = 0.f;
      if (hx) {
        wx = irls1f(P[1] - T0[k], c);
        const float g = Q[1] - yT[k];
        esm = fmaf(wx * g, g, esm);
      }
      if (hy) {
        wy = irls1f(P[kSW] - T0[k], c);
        const float g = Q[kSW] - yT[k];
        esm = fmaf(wy * g, g, esm);
      }
      if (MODE == MODE_EG) {
        float g = 0.f, d = 0.f, gm = 0.f;
        const float g2 = c.g2[k];   // sum_c G_kc^2, precomputed (make_coef)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float rb = R[ch] * c.B[k][ch];
          g = fmaf(rb, res[ch], g);
          d = fmaf(rb, rb, d);
          gm = fmaf(c.G[k][ch], m[ch], gm);
        }
        const float wdk = wis + wnn;
        g = fmaf(-c.lam_d, g, fmaf(lm, gm, wdk * T0[k]));
        d = fmaf(c.lam_d, d, fmaf(lm, g2, wdk));
        const float v = T0[k];
        float gs = 0.f, ds = 0.f;
        if (hx) { gs = fmaf(wx, v - P[1], gs); ds += wx; }
        if (hl) { const float a = irls1f(v - P[-1], c); gs = fmaf(a, v - P[-1], gs); ds += a; }
        if (hy) { gs = fmaf(wy, v - P[kSW], gs); ds += wy; }
        if (hu) { const float a = irls1f(v - P[-kSW], c); gs = fmaf(a, v - P[-kSW], gs); ds += a; }
        g = fmaf(c.lam_sm, gs, g);
        d = fmaf(c.lam_sm, ds, d);
        const float bf = -g;
        const float di = rcpf(d > 0.f ? d : 1.f);   // Jacobi preconditioner 1/diag (solver.py:87), MUFU
        const float zf = bf * di;
        const size_t o = (size_t)(3 + k) * N + i;
        if (d_out) {
          if (LS_KEEP_R) r_out[o] = bf;   // r = b is never read again (z-only recurrence)
          d_out[o] = di;
          u_out[o] = zf;
        }
        if (b_raw) { b_raw[o] = bf; diag_raw[o] = d; }
        rz = fmaf(bf, zf, rz);
        bb = fmaf(bf, bf, bb);
      }
    }
    acc[T_ISPARSE] += (double)eis;
    acc[T_NONNEG] += (double)enn;
    acc[T_SMOOTH] += (double)(c.lam_sm * esm);
  }

  // consistency pairs (energy.py:348-350): energy counted at each pair's
  // src; gradient / diagonal from every incident pair (energy.py:359-381)
  float gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, dcons = 0.f;
  {
    const int e0 = pre.e0, e1 = pre.e1;
    float ec = 0.f;
    const float* YR = sYR + rc0;
    // partner values of one entry: the previous frame's r (temporal, global)
    // or the staged window (spatial)
    auto partner = [&](uint16_t ent, float& p0, float& p1, float& p2) {
      if (ent & kEntTemporal) {
        int ddy, ddx;
        decode_offset(ent, ddy, ddx);
        const int q = i + ddy * W + ddx;
        p0 = __ldg(f.prev_r + q);
        p1 = __ldg(f.prev_r + N + q);
        p2 = __ldg(f.prev_r + 2 * N + q);
      } else {
        const int o = ent_soff(ent);
        p0 = YR[o];
        p1 = YR[kRP + o];
        p2 = YR[2 * kRP + o];
      }
    };
    auto accum = [&](uint16_t ent, float wgt, float p0, float p1, float p2) {
      const float we = c.lam_rc * wgt;
      const float d0 = yr[0] - p0, d1 = yr[1] - p1, d2 = yr[2] - p2;
      if (!(ent & kEntIncoming)) ec = fmaf(we, fmaf(d0, d0, fmaf(d1, d1, d2 * d2)), ec);
      gc0 = fmaf(we, d0, gc0);
      gc1 = fmaf(we, d1, gc1);
      gc2 = fmaf(we, d2, gc2);
      dcons += we;
    };
    // four entries per round: their loads are issued together, the
    // accumulation stays in CSR order
    int e = e0;
    for (; e + 4 <= e1; e += 4) {
      uint16_t q[4];
      float wv[4], pv[4][3];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        q[j] = __ldg(f.ent + e + j);
        wv[j] = f.ent_w ? __ldg(f.ent_w + e + j) : 1.f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) partner(q[j], pv[j][0], pv[j][1], pv[j][2]);
#pragma unroll
      for (int j = 0; j < 4; ++j) accum(q[j], wv[j], pv[j][0], pv[j][1], pv[j][2]);
    }
    for (; e < e1; ++e) {
      const uint16_t ent = __ldg(f.ent + e);
      float p0, p1, p2;
      partner(ent, p0, p1, p2);
      accum(ent, f.ent_w ? __ldg(f.ent_w + e) : 1.f, p0, p1, p2);
    }
    acc[T_CONSIST] += (double)ec;
  }

  if (MODE == MODE_TRIAL) {
    if (Xout) {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) Xout[ch * N + i] = yr[ch];
#pragma unroll
      for (int k = 0; k < NT; ++k) Xout[(size_t)(3 + k) * N + i] = yT[k];
    }
    return;
  }

  // ======== MODE_EG: g = J^T F, diag(J^T J), PCG init (Y == X) ========
  const float wl = hl ? wrs_s(sXR, rx - 1, ry, true, hy, c, kRW, kRP) : 0.f;
  const float wu = hu ? wrs_s(sXR, rx, ry - 1, hx, true, c, kRW, kRP) : 0.f;
  const float gcons[3] = {gc0, gc1, gc2};
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float* P = sXR + ch * kRP + rc0;
    const float rs = R[ch] * S[ch];
    float g = fmaf(-c.lam_d * rs, res[ch], c.lam_cl * (r0[ch] - anc[ch]));
    float d = fmaf(c.lam_d * rs, rs, c.lam_cl);
    const float v = r0[ch];
    if (hx) { g = fmaf(wrs, v - P[1], g); d += wrs; }
    if (hl) { g = fmaf(wl, v - P[-1], g); d += wl; }
    if (hy) { g = fmaf(wrs, v - P[kRW], g); d += wrs; }
    if (hu) { g = fmaf(wu, v - P[-kRW], g); d += wu; }
    g += gcons[ch];
    d += dcons;
    const float bf = -g;
    const float di = rcpf(d > 0.f ? d : 1.f);   // Jacobi preconditioner 1/diag (solver.py:87), MUFU
    const float zf = bf * di;
    if (d_out) {
      if (LS_KEEP_R) r_out[ch * N + i] = bf;
      d_out[ch * N + i] = di;
      u_out[ch * N + i] = zf;
    }
    if (b_raw) { b_raw[ch * N + i] = bf; diag_raw[ch * N + i] = d; }
    rz = fmaf(bf, zf, rz);
    bb = fmaf(bf, bf, bb);
  }
  acc[kTerms] += (double)rz;
  acc[kTerms + 1] += (double)bb;
}


// ---------------------------------------------------------------------------
// finalisation of reduced sums: run by the last CTA of a kernel, or, for row
// bands, by k_band_finalize on the band-ordered sum of every band's partials
// ---------------------------------------------------------------------------
__device__ void fin_energy_eg(const double* tot, Scalars* sc, bool pcg_init) {
  bool finite = true;
  for (int j = 0; j < kTerms; ++j) finite = finite && isfinite(tot[j]);
  double e0 = 0.0;   // Python sum() order over the blocks (solver.py:139-140)
  for (int j = 0; j < kTerms; ++j) e0 += tot[j];
  sc->e0 = e0;
  sc->ls_done = 0;
  sc->accepted = 0;
  sc->fault = 0;
  sc->alpha_ls = 0.0;
  sc->e1 = e0;
  for (int j = 0; j < kTerms; ++j) sc->terms0[j] = tot[j];
  sc->gamma = tot[kTerms];
  sc->gamma_prev = 0.0;
  sc->bnorm2 = tot[kTerms + 1];
  sc->rnorm2 = tot[kTerms + 1];
  sc->alpha = sc->alpha_prev = sc->beta = sc->delta = 0.0;
  sc->iterations = 0;
  sc->pending = 0;
  sc->xinit = 0;
  sc->plast = 0;
  // zero rhs -> x = 0 (solver.py:85-86); non-finite -> host raises
  sc->stop = (!finite || tot[kTerms + 1] == 0.0 || !pcg_init) ? 1 : 0;
}

__device__ void fin_energy_trial(const double* tot, Scalars* sc, float alpha, int dev_ls, int last_trial) {
  for (int j = 0; j < kTerms; ++j) sc->terms1[j] = tot[j];
  if (dev_ls) {   // accept / halve decision of solver.py:169-178 on the device
    double e1 = 0.0;
    for (int j = 0; j < kTerms; ++j) e1 += tot[j];
    if (!isfinite(sc->e0)) {
      sc->fault = 1;
      sc->ls_done = 1;
    } else if (isfinite(e1) && e1 <= sc->e0) {
      sc->ls_done = 1;
      sc->accepted = 1;
      sc->alpha_ls = (double)alpha;
      sc->e1 = e1;
    } else if (last_trial) {
      sc->ls_done = 1;
    }
  }
}

__device__ void fin_pcg_apply(double pap, Scalars* sc, int iter) {
  if (sc->pending) {      // this apply folded alpha_{i-1} p_{i-1} into x
    sc->pending = 0;
    sc->xinit = 1;
  }
  sc->delta = pap;
  if (!(pap > 0.0) || !isfinite(pap)) {
    sc->stop = 1;                       // solver.py:95-96: break before the update
  } else {
    sc->alpha_prev = sc->alpha;
    sc->alpha = sc->gamma / pap;
    if (iter >= 0 && iter < kMaxStoredDirs) sc->alpha_hist[iter] = sc->alpha;
  }
}

__device__ void fin_pcg_update(double rz, double rn, Scalars* sc, int iter) {
  sc->iterations = iter + 1;
  sc->pending = 1;        // x += alpha_i p_i is deferred to the next apply (or k_pcg_xfinal)
  sc->gamma_prev = sc->gamma;
  sc->gamma = rz;
  sc->rnorm2 = rn;
  sc->beta = rz / sc->gamma_prev;
  if (rz <= 0.0) sc->stop = 1;          // solver.py:101-103
}

template <int NT, int MODE, bool TMA, bool COND = false>
#ifndef LS_EG_MINB
#define LS_EG_MINB kStencilMinBlocks
#endif
__global__ void __launch_bounds__(kThreads, LS_EG_MINB) k_energy(Frame f, Coef<float> c, const float* __restrict__ X,
                                                     const float* __restrict__ dx, float alpha,
                                                     const float* __restrict__ Yext, float* __restrict__ Xout,
                                                     float* __restrict__ r_out, float* __restrict__ d_out,
                                                     float* __restrict__ u_out, float* __restrict__ b_raw,
                                                     float* __restrict__ diag_raw, double* part,
                                                     unsigned* ticket, Scalars* sc, int ntiles,
                                                     const FrameCtl* ctl, int dev_ls, int last_trial,
                                                     const __grid_constant__ EnergyMaps maps,
                                                     unsigned long long next_cond) {
  constexpr int U = NT + 3;
  constexpr bool TRIAL = MODE == MODE_TRIAL;
  pdl_wait();
  pdl_trigger();
  // device-resident flip-flop: skip finished frames / decided line searches
  if (ctl && ctl->done) {
    if (!TRIAL && blockIdx.x == 0 && threadIdx.x == 0) sc->stop = 1;
    return;
  }
  if (TRIAL && dev_ls && sc->ls_done) return;
  constexpr int NST = (TMA && !TRIAL) ? 2 : 1;
  constexpr int STAGE = e_stage(NT, TRIAL);
  constexpr int NV = TRIAL ? kTerms : kTerms + 2;
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[2];
  const int W = f.W, H = f.H, N = f.N;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int cx = lx + kSX, cy = ly + 1, rx = lx + kRX, ry = ly + kHalf;
  const int ntx = (W + kTileW - 1) / kTileW;
  // the evaluation point: X itself, X + alpha*dx, or an external Y
  const bool ext = TRIAL && Yext != nullptr;
  const bool step = TRIAL && !ext && dx != nullptr && sc->xinit;
  const bool with_d = ext || step;
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_barrier_init();
      for (int j = 0; j < NST; ++j) {
        const int t = blockIdx.x + j * gridDim.x;
        if (t < ntiles) tma_issue_energy<NT>(smem + j * STAGE, maps, &bars[j], (t % ntx) * kTileW,
                                             f.y_lo + (t / ntx) * kTileH, with_d);
      }
    }
    __syncthreads();
  }
  uint32_t phase = 0;
  TileWalk walk(blockIdx.x, gridDim.x, ntx);
  for (int j = 0;; ++j, walk.advance()) {
    const int tile = blockIdx.x + j * gridDim.x;
    if (tile >= ntiles) break;
    const int tx0 = (LS_TILEWALK ? walk.tx : tile % ntx) * kTileW,
              ty0 = f.y_lo + (LS_TILEWALK ? walk.ty : tile / ntx) * kTileH;
    const int st = (NST == 2) ? (j & 1) : 0;
    float* sX = smem + st * STAGE;
    float* sXR = sX + e_off_XR(NT);
    float* sD = sX + e_off_D(NT);
    float* sDR = sX + e_off_DR(NT);
    const EPre pre = energy_prefetch(f, tx0 + lx, ty0 + ly, tx0 + lx < W && ty0 + ly < f.y_hi);
    if (TMA) {
      mbar_wait(&bars[st], (phase >> st) & 1u);
      phase ^= 1u << st;
    } else {
      __syncthreads();
      load_halo1<U>(sX, X, N, W, H, tx0, ty0);
      load_halo7(sXR, X, nullptr, 0.f, N, W, H, tx0, ty0);
      if (with_d) {
        load_halo1<U>(sD, ext ? Yext : dx, N, W, H, tx0, ty0);
        load_halo7(sDR, ext ? Yext : dx, nullptr, 0.f, N, W, H, tx0, ty0);
      }
      __syncthreads();
    }
    if (step) {   // Y = fma(alpha, dx, X) in place (T planes 1 halo, r planes 7 halo)
      __syncthreads();
      for (int e = threadIdx.x; e < NT * kSP; e += kThreads)
        sD[3 * kSP + e] = __fmaf_rn(alpha, sD[3 * kSP + e], sX[3 * kSP + e]);
      for (int e = threadIdx.x; e < 3 * kRP; e += kThreads) sDR[e] = __fmaf_rn(alpha, sDR[e], sXR[e]);
      __syncthreads();
    }
    const float* sYT = with_d ? sD + 3 * kSP : sX + 3 * kSP;
    const float* sYR = with_d ? sDR : sXR;
    const bool interior = tx0 > 0 && ty0 > 0 && tx0 + kTileW < W && ty0 + kTileH < H && ty0 + kTileH <= f.y_hi;
    if (interior)
      energy_pixel<NT, MODE, true>(f, c, sX, sXR, sYT, sYR, tx0 + lx, ty0 + ly, cx, cy, rx, ry, Xout, r_out, d_out,
                                   u_out, b_raw, diag_raw, acc, pre);
    else if (tx0 + lx < W && ty0 + ly < f.y_hi)
      energy_pixel<NT, MODE, false>(f, c, sX, sXR, sYT, sYR, tx0 + lx, ty0 + ly, cx, cy, rx, ry, Xout, r_out, d_out,
                                    u_out, b_raw, diag_raw, acc, pre);
    if (TMA) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const int t = blockIdx.x + (j + NST) * gridDim.x;
        if (t < ntiles) {   // NST tiles ahead
          TileWalk w2 = walk;
#pragma unroll
          for (int a = 0; a < NST; ++a) w2.advance();
          tma_issue_energy<NT>(sX, maps, &bars[st], w2.tx * kTileW, f.y_lo + w2.ty * kTileH, with_d);
        }
      }
    }
  }

  block_reduce_store<NV>(acc, part);
  if (!last_block(ticket)) return;
  double tot[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) tot[j] = sum_partials<NV>(part, gridDim.x, j);
  if (threadIdx.x == 0) {
    if (f.bsum) {
      for (int j = 0; j < NV; ++j) f.bsum[j] = tot[j];
    } else if (!TRIAL) {
      fin_energy_eg(tot, sc, r_out != nullptr);
    } else {
      fin_energy_trial(tot, sc, alpha, dev_ls, last_trial);
      // CUDA-graph flip-flop: the next halving's trial is the body of a
      // conditional node; it runs only while the line search is undecided
      // (a separate instantiation: a kernel calling the device graph API is
      // not listed by ncu inside graphs, and the default path never needs it)
      if (COND && next_cond) cudaGraphSetConditional(next_cond, sc->ls_done ? 0u : 1u);
    }
    *ticket = 0u;
  }
}

// One pixel of w = J^T J u.  IN: interior tile (every stencil neighbour is
// inside the image) -> no border masks.  Returns the pixel's <w, u>.
// Per-pixel global reads of the operator (CSR row bounds, edge gate), issued
// before the tile's TMA wait so their latency overlaps it.
struct PixPre {
  int e0, e1;
  float edge;
};
__device__ __forceinline__ PixPre pix_prefetch(const Frame& f, int x, int y, bool own) {
  PixPre p{0, 0, 0.f};
  if (own) {
    const int i = y * f.W + x;
    p.e0 = __ldg(f.row_ptr + i);
    p.e1 = __ldg(f.row_ptr + i + 1);
    p.edge = __ldg(f.edge + i);
  }
  return p;
}

// SCALE (the single-reduction PCG, k_cg_iter): the stored value is w * dinv
// (the preconditioned product M w); the returned <w, u> is of the unscaled w
template <int NT, bool IN, bool SCALE = false>
__device__ __forceinline__ float apply_pixel(const Frame& f, const Coef<float>& c, const float* sX, const float* sT,
                                             const float* sR, float* __restrict__ w, int x, int y, int cx, int cy,
                                             int rx, int ry, const PixPre& pre,
                                             const float* __restrict__ dinv = nullptr) {
  const int W = f.W, H = f.H, N = f.N;
  const int i = y * W + x;
  const bool hx = IN || x < W - 1, hy = IN || y < H - 1, hl = IN || x > 0, hu = IN || y > 0;
  const int sc0 = cy * kSW + cx, rc0 = ry * kRW + rx;

  float ur[3], R0[3], S0[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    ur[ch] = sR[ch * kRP + rc0];
    R0[ch] = __expf(sX[ch * kSP + sc0]);
  }
  float uT[NT], T0[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    uT[k] = sT[k * kSP + sc0];
    T0[k] = sX[(3 + k) * kSP + sc0];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) S0[ch] = fmaf(T0[k], c.B[k][ch], S0[ch]);
  }
  // data rows rho_c = R0 (S0 u_r + sum_k b_kc u_Tk) (energy.py:211-218) and
  // monochrome q_c = w_edge sum_k G_kc u_Tk (energy.py:403-408).  With
  // G = B - rowmean(B): sum_k G_kc u_k = s_c - mean_c(s) and sum_c q_c = 0,
  // so the T rows are sum_c B_kc (rho_c + q_c).
  float rq[3], outr[3], s[3] = {0.f, 0.f, 0.f};
  const float lm = c.lam_m * pre.edge;
#pragma unroll
  for (int k = 0; k < NT; ++k)
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) s[ch] = fmaf(uT[k], c.B[k][ch], s[ch]);
  const float smean = (s[0] + s[1] + s[2]) * (1.f / 3.f);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float r0s0 = R0[ch] * S0[ch];
    const float rr = fmaf(r0s0, ur[ch], R0[ch] * s[ch]);
    outr[ch] = fmaf(c.lam_d * r0s0, rr, c.lam_cl * ur[ch]);
    rq[ch] = fmaf(c.lam_d * R0[ch], rr, lm * (s[ch] - smean));
  }
  float dot = 0.f;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const float* P = sX + (3 + k) * kSP + sc0;
    const float* Q = sT + k * kSP + sc0;
    float a = c.B[k][0] * rq[0];
    a = fmaf(c.B[k][1], rq[1], a);
    a = fmaf(c.B[k][2], rq[2], a);
    const float v = T0[k], uv = uT[k];
    const float wis = (k >= 1) ? c.lam_is * irls1f(v, c) : 0.f;
    const float wnn = c.lam_nn * nonneg_wf(v, c.eps_nn);
    a = fmaf(wis + wnn, uv, a);
    // smoothness D^T W_k D u_Tk (energy.py:272-282), weights from X
    float sm = 0.f;
    if (LS_ABLATE != 3) {
    if (hx) sm = fmaf(irls1f(P[1] - v, c), uv - Q[1], sm);
    if (hl) sm = fmaf(irls1f(v - P[-1], c), uv - Q[-1], sm);
    if (hy) sm = fmaf(irls1f(P[kSW] - v, c), uv - Q[kSW], sm);
    if (hu) sm = fmaf(irls1f(v - P[-kSW], c), uv - Q[-kSW], sm);
    }
    a = fmaf(c.lam_sm, sm, a);
    w[(size_t)(3 + k) * N + i] = SCALE ? a * __ldg(dinv + (size_t)(3 + k) * N + i) : a;
    dot = fmaf(a, uv, dot);
  }
  // r-sparsity D^T W D u_r, one weight per pixel shared by the channels
  if (LS_ABLATE != 4) {
    const float wc = wrs_s(sX, cx, cy, hx, hy, c);
    const float wl = hl ? wrs_s(sX, cx - 1, cy, true, hy, c) : 0.f;
    const float wu = hu ? wrs_s(sX, cx, cy - 1, hx, true, c) : 0.f;
    const float wcx = hx ? wc : 0.f, wcy = hy ? wc : 0.f;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float* P = sR + ch * kRP + rc0;
      const float v = ur[ch];
      float a = wcx * (v - P[1]);
      a = fmaf(wl, v - P[-1], a);
      a = fmaf(wcy, v - P[kRW], a);
      a = fmaf(wu, v - P[-kRW], a);
      outr[ch] += a;
    }
  }
  // consistency graph Laplacian (energy.py:352-370): spatial pairs couple
  // u(x) - u(q); temporal partners are constant (energy.py:356).  Entries
  // carry the partner's offset in this smem window.
  {
    const int e0 = pre.e0, e1 = pre.e1;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    const float* R0p = sR + rc0;
    // entries are fetched four at a time so their load latencies overlap;
    // the accumulation order is the CSR order either way
    if (LS_ABLATE == 1) {
    } else if (f.ent_w == nullptr) {
      // unit weights: sum_e (u - u_partner) = deg * u - sum of the spatial
      // partners (a temporal partner is the constant previous frame)
      float s0 = 0.f, s1 = 0.f, s2 = 0.f;
      auto one = [&](uint16_t ent) {
        if (!(ent & kEntTemporal)) {
          const int o = ent_soff(ent);
          s0 += R0p[o];
          s1 += R0p[kRP + o];
          s2 += R0p[2 * kRP + o];
        }
      };
      int e = e0;
      for (; e + 4 <= e1; e += 4) {
        const uint16_t q0 = __ldg(f.ent + e), q1 = __ldg(f.ent + e + 1);
        const uint16_t q2 = __ldg(f.ent + e + 2), q3 = __ldg(f.ent + e + 3);
        one(q0); one(q1); one(q2); one(q3);
      }
      for (; e < e1; ++e) one(__ldg(f.ent + e));
      const float deg = (float)(e1 - e0);
      a0 = c.lam_rc * fmaf(deg, ur[0], -s0);
      a1 = c.lam_rc * fmaf(deg, ur[1], -s1);
      a2 = c.lam_rc * fmaf(deg, ur[2], -s2);
    } else {
      auto one = [&](uint16_t ent, float wgt) {
        const float we = c.lam_rc * wgt;
        const int o = ent_soff(ent);
        const bool tmp = ent & kEntTemporal;
        a0 = fmaf(we, ur[0] - (tmp ? 0.f : R0p[o]), a0);
        a1 = fmaf(we, ur[1] - (tmp ? 0.f : R0p[kRP + o]), a1);
        a2 = fmaf(we, ur[2] - (tmp ? 0.f : R0p[2 * kRP + o]), a2);
      };
      int e = e0;
      for (; e + 2 <= e1; e += 2) {
        const uint16_t q0 = __ldg(f.ent + e), q1 = __ldg(f.ent + e + 1);
        const float w0 = __ldg(f.ent_w + e), w1 = __ldg(f.ent_w + e + 1);
        one(q0, w0); one(q1, w1);
      }
      for (; e < e1; ++e) one(__ldg(f.ent + e), __ldg(f.ent_w + e));
    }
    outr[0] += a0; outr[1] += a1; outr[2] += a2;
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    w[(size_t)ch * N + i] = SCALE ? outr[ch] * __ldg(dinv + (size_t)ch * N + i) : outr[ch];
    dot = fmaf(outr[ch], ur[ch], dot);
  }
  return dot;
}

template <int NT, bool TMA>
__global__ void __launch_bounds__(kThreads, 2) k_apply(Frame f, Coef<float> c, const float* __restrict__ X,
                                                       const float* __restrict__ u, float* __restrict__ w,
                                                       double* part, unsigned* ticket, Scalars* sc, int iter,
                                                       int ntiles, const __grid_constant__ TileMaps maps) {
  constexpr int U = NT + 3;
  constexpr int STAGE = tile_floats(NT, true);
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[2];
  if (sc && sc->stop) return;
  const int W = f.W, H = f.H, N = f.N;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int cx = lx + kSX, cy = ly + 1, rx = lx + kRX, ry = ly + kHalf;
  const int ntx = (W + kTileW - 1) / kTileW;
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_barrier_init();
      tma_prefetch_desc(&maps.X);
      tma_prefetch_desc(&maps.T);
      tma_prefetch_desc(&maps.R);
      for (int j = 0; j < 2; ++j) {
        const int t = blockIdx.x + j * gridDim.x;
        if (t < ntiles)
          tma_issue_tile<NT>(smem + j * STAGE, maps, &bars[j], (t % ntx) * kTileW, f.y_lo + (t / ntx) * kTileH);
      }
    }
    __syncthreads();
  }
  uint32_t phase = 0;   // bit s: parity of the next wait on stage s
  float acc = 0.f;
  double accd = 0.0;
  for (int j = 0;; ++j) {
    const int tile = blockIdx.x + j * gridDim.x;
    if (tile >= ntiles) break;
    const int tx0 = (tile % ntx) * kTileW, ty0 = f.y_lo + (tile / ntx) * kTileH;
    const int st = TMA ? (j & 1) : 0;
    float* sX = smem + st * STAGE;
    float* sT = sX + off_T(NT);
    float* sR = sX + off_R(NT, true);
    const PixPre pre = pix_prefetch(f, tx0 + lx, ty0 + ly, tx0 + lx < W && ty0 + ly < f.y_hi);
    if (TMA) {
      mbar_wait(&bars[st], (phase >> st) & 1u);
      phase ^= 1u << st;
    } else {
      __syncthreads();
      load_halo1<U>(sX, X, N, W, H, tx0, ty0);
      load_halo1<NT>(sT, u + 3 * (size_t)N, N, W, H, tx0, ty0);
      load_halo7(sR, u, nullptr, 0.f, N, W, H, tx0, ty0);
      __syncthreads();
    }
    const bool interior = tx0 > 0 && ty0 > 0 && tx0 + kTileW < W && ty0 + kTileH < H && ty0 + kTileH <= f.y_hi;
    if (interior)
      acc += apply_pixel<NT, true>(f, c, sX, sT, sR, w, tx0 + lx, ty0 + ly, cx, cy, rx, ry, pre);
    else if (tx0 + lx < W && ty0 + ly < f.y_hi)
      acc += apply_pixel<NT, false>(f, c, sX, sT, sR, w, tx0 + lx, ty0 + ly, cx, cy, rx, ry, pre);
    if (TMA) {
      __syncthreads();   // every thread is done with this stage
      if (threadIdx.x == 0) {
        const int t = blockIdx.x + (j + 2) * gridDim.x;
        if (t < ntiles) tma_issue_tile<NT>(sX, maps, &bars[st], (t % ntx) * kTileW, f.y_lo + (t / ntx) * kTileH);
      }
    }
    accd += (double)acc;   // fp64 across tiles
    acc = 0.f;
  }
  (void)accd;   // the API operator (ls_apply_normal) needs no reduction
}

// ---------------------------------------------------------------------------
// textbook Jacobi PCG (solver.py:79-107), two kernels per iteration:
//   k_pcg_apply  i: p_i = z_i + beta_i p_{i-1} (formed in shared memory on the
//                   tile + halo), q_i = J^T J p_i, <p_i, q_i>;
//                   last CTA: alpha_i = rz_i / pAp_i or break (solver.py:95)
//   k_pcg_update i: x += alpha_i p_i, r_{i+1} = r_i - alpha_i q_i,
//                   z = r * dinv, <r, z>, |r|^2;
//                   last CTA: beta, break on rz <= 0 (solver.py:101-103)
// HBM words / pixel / iteration: (X + z + p_prev) + (p + q) +
// (r + q + dinv + p + x) + (r + z + x) = 13U (vs 15U for the CG form with a
// separate vector update; forming p costs no pass of its own).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int op_floats(int NT) { return pad32(NT * kSP) + pad32(3 * kRP); }
// X, z and p_{i-1} windows (p_i = z_i + beta p_{i-1} is formed in place over z)
__host__ __device__ constexpr int pcg_stage(int NT, bool) {
  return pad32((NT + 3) * kSP) + (LS_PFORM_GLOBAL ? 1 : 2) * op_floats(NT);
}

template <int NT>
// two barriers: bar[0] the operand windows (z, p_{i-1}) the formation pass
// needs first, bar[1] the state window, which lands during the formation
__device__ __forceinline__ void tma_issue_pcg(float* stage, const PcgMaps& m, uint64_t* bar, int tx0, int ty0,
                                              bool with_p) {
  constexpr uint32_t xb = sizeof(float) * (NT + 3) * kSP;
  constexpr uint32_t ob = sizeof(float) * (NT * kSP + 3 * kRP);
  const bool p_here = with_p && !LS_PEARLY && !LS_PFORM_GLOBAL;   // LS_PEARLY: the p window has its own barrier
  mbar_expect_tx(&bar[0], (p_here ? 2 : 1) * ob);
  mbar_expect_tx(&bar[1], xb);
  float* z = stage + pad32((NT + 3) * kSP);
  float* pp = z + op_floats(NT);
  tma_load_3d(z, &m.ZT, &bar[0], tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(z + pad32(NT * kSP), &m.ZR, &bar[0], tx0 - kRX, ty0 - kHalf, 0);
  if (p_here) {
    tma_load_3d(pp, &m.PT, &bar[0], tx0 - kSX, ty0 - 1, 0);
    tma_load_3d(pp + pad32(NT * kSP), &m.PR, &bar[0], tx0 - kRX, ty0 - kHalf, 0);
  }
  tma_load_3d(stage, &m.X, &bar[1], tx0 - kSX, ty0 - 1, 0);
}

// the p_{i-1} window alone (LS_PEARLY), on its own barrier
template <int NT>
__device__ __forceinline__ void tma_issue_pprev(float* stage, const PcgMaps& m, uint64_t* bar, int tx0, int ty0) {
  constexpr uint32_t ob = sizeof(float) * (NT * kSP + 3 * kRP);
  mbar_expect_tx(bar, ob);
  float* pp = stage + pad32((NT + 3) * kSP) + op_floats(NT);
  tma_load_3d(pp, &m.PT, bar, tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(pp + pad32(NT * kSP), &m.PR, bar, tx0 - kRX, ty0 - kHalf, 0);
}


template <int NT, bool TMA>
#ifndef LS_PCG_MINB
#define LS_PCG_MINB kStencilMinBlocks
#endif
__global__ void __launch_bounds__(kThreads, LS_PCG_MINB) k_pcg_apply(Frame f, Coef<float> c, const float* __restrict__ X,
                                                           const float* __restrict__ z,
                                                           const float* __restrict__ pprev,
                                                           float* __restrict__ pnew, float* __restrict__ q, double* part, unsigned* ticket,
                                                           Scalars* sc, int iter, int ntiles,
                                                           const __grid_constant__ PcgMaps maps,
                                                           float* __restrict__ xv) {
  constexpr int U = NT + 3;
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[3];
  pdl_wait();
  pdl_trigger();
  if (sc->stop) return;
  const int W = f.W, H = f.H, N = f.N;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int cx = lx + kSX, cy = ly + 1, rx = lx + kRX, ry = ly + kHalf;
  const int ntx = (W + kTileW - 1) / kTileW;
  const bool with_p = LS_ABLATE != 2 && iter > 0;
  const float beta = (float)sc->beta;
  // deferred PCG x-update (solver.py:98): x += alpha_{i-1} p_{i-1} for the own
  // pixels, p_{i-1} taken from the staged window -- k_pcg_update then streams
  // only r, q, dinv -> r, z
  const bool xupd = with_p && sc->pending && xv != nullptr;
  const bool xread = sc->xinit;
  const float ax = (float)sc->alpha;
  float* sX = smem;
  float* sZT = smem + pad32(U * kSP);
  float* sZR = sZT + pad32(NT * kSP);
  float* sPT = sZT + op_floats(NT);
  float* sPR = sPT + pad32(NT * kSP);
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_init(&bars[2], 1);
      fence_barrier_init();
      if ((int)blockIdx.x < ntiles) {
        const int t = blockIdx.x;
        tma_issue_pcg<NT>(smem, maps, &bars[0], (t % ntx) * kTileW, f.y_lo + (t / ntx) * kTileH, with_p);
        if (LS_PEARLY && with_p)
          tma_issue_pprev<NT>(smem, maps, &bars[2], (t % ntx) * kTileW, f.y_lo + (t / ntx) * kTileH);
      }
    }
    __syncthreads();
  }
  uint32_t phase = 0;
  float acc = 0.f;
  double accd = 0.0;
#if LS_XDEFER
  // the previous tile's x-update: loads issued after the TMA issue, the
  // fma + stores after the next tile's operand wait (latency hidden by it)
  float xo_d[U], pold_d[U];
  bool pend = false;
  size_t pend_i = 0;
#endif
  TileWalk walk(blockIdx.x, gridDim.x, ntx);
  for (int j = 0;; ++j, walk.advance()) {
    const int tile = blockIdx.x + j * gridDim.x;
    if (tile >= ntiles) break;
    const int tx0 = (LS_TILEWALK ? walk.tx : tile % ntx) * kTileW,
              ty0 = f.y_lo + (LS_TILEWALK ? walk.ty : tile / ntx) * kTileH;
    const int x = tx0 + lx, y = ty0 + ly;
    const bool own = x < W && y < f.y_hi;
    const PixPre pre = pix_prefetch(f, x, y, own);
    if (TMA) {
      mbar_wait(&bars[0], phase);   // operand windows
      if (LS_PEARLY && with_p) mbar_wait(&bars[2], phase);
    }
#if LS_XDEFER
    if (pend) {
#pragma unroll
      for (int u = 0; u < U; ++u) xv[(size_t)u * N + pend_i] = fmaf(ax, pold_d[u], xo_d[u]);
      pend = false;
    }
#endif
    if (!TMA) {
      __syncthreads();
      load_halo1<U>(sX, X, N, W, H, tx0, ty0);
      load_halo1<NT>(sZT, z + 3 * (size_t)N, N, W, H, tx0, ty0);
      load_halo7(sZR, z, nullptr, 0.f, N, W, H, tx0, ty0);
      if (with_p) {
        load_halo1<NT>(sPT, pprev + 3 * (size_t)N, N, W, H, tx0, ty0);
        load_halo7(sPR, pprev, nullptr, 0.f, N, W, H, tx0, ty0);
      }
      __syncthreads();
    }
    if (with_p) {   // operand p_i = z_i + beta_i p_{i-1} on the whole window
      // float4 over both regions (sizes and offsets are multiples of 4 words)
      static_assert((NT * kSP) % 4 == 0 && (3 * kRP) % 4 == 0, "float4 operand formation");
      auto form = [beta](float* zz, const float* pp, int n4) {
        float4* z4 = reinterpret_cast<float4*>(zz);
        const float4* p4 = reinterpret_cast<const float4*>(pp);
        for (int e = threadIdx.x; e < n4; e += kThreads) {
          float4 a = z4[e];
          const float4 b = p4[e];
          a.x = fmaf(beta, b.x, a.x); a.y = fmaf(beta, b.y, a.y);
          a.z = fmaf(beta, b.z, a.z); a.w = fmaf(beta, b.w, a.w);
          z4[e] = a;
        }
      };
#if LS_PFORM_GLOBAL
      {   // p_{i-1} from global (zero outside the image, like the TMA boxes)
        const float4* pg = reinterpret_cast<const float4*>(pprev);
        constexpr int c4t = kSW / 4, c4r = kRW / 4;
        for (int e = threadIdx.x; e < NT * kSH * c4t; e += kThreads) {
          const int k = e / (kSH * c4t), rem = e - k * (kSH * c4t), rr = rem / c4t, c4 = rem - rr * c4t;
          const int gy = ty0 - 1 + rr, gx = tx0 - kSX + 4 * c4;
          float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gy >= 0 && gy < H && gx >= 0 && gx < W) b = __ldg(pg + (((size_t)(3 + k) * N + (size_t)gy * W + gx) >> 2));
          float4* zp = reinterpret_cast<float4*>(sZT + k * kSP + rr * kSW + 4 * c4);
          float4 a = *zp;
          a.x = fmaf(beta, b.x, a.x); a.y = fmaf(beta, b.y, a.y);
          a.z = fmaf(beta, b.z, a.z); a.w = fmaf(beta, b.w, a.w);
          *zp = a;
        }
        for (int e = threadIdx.x; e < 3 * kHaloH * c4r; e += kThreads) {
          const int ch = e / (kHaloH * c4r), rem = e - ch * (kHaloH * c4r), rr = rem / c4r, c4 = rem - rr * c4r;
          const int gy = ty0 - kHalf + rr, gx = tx0 - kRX + 4 * c4;
          float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
          if (gy >= 0 && gy < H && gx >= 0 && gx < W) b = __ldg(pg + (((size_t)ch * N + (size_t)gy * W + gx) >> 2));
          float4* zp = reinterpret_cast<float4*>(sZR + ch * kRP + rr * kRW + 4 * c4);
          float4 a = *zp;
          a.x = fmaf(beta, b.x, a.x); a.y = fmaf(beta, b.y, a.y);
          a.z = fmaf(beta, b.z, a.z); a.w = fmaf(beta, b.w, a.w);
          *zp = a;
        }
      }
#else
      form(sZT, sPT, NT * kSP / 4);
      form(sZR, sPR, 3 * kRP / 4);
#endif
      if (!TMA) __syncthreads();
      if (TMA && LS_PEARLY && !xupd) {   // the p region is free: the next tile's p_{i-1} now
        __syncthreads();
        if (threadIdx.x == 0) {
          const int t = blockIdx.x + (j + 1) * gridDim.x;
          int nx, ny;
          walk.next(nx, ny);
          if (t < ntiles) tma_issue_pprev<NT>(smem, maps, &bars[2], nx * kTileW, f.y_lo + ny * kTileH);
        }
      }
    }
    if (TMA) {   // state window (arrived during the formation); the wait's
      mbar_wait(&bars[1], phase);   // acquire + the barrier below order the formed operand
      phase ^= 1u;
      if (with_p) __syncthreads();
    }
    const bool interior = tx0 > 0 && ty0 > 0 && tx0 + kTileW < W && ty0 + kTileH < H && ty0 + kTileH <= f.y_hi;
    if (interior)
      acc += apply_pixel<NT, true>(f, c, sX, sZT, sZR, q, x, y, cx, cy, rx, ry, pre);
    else if (own)
      acc += apply_pixel<NT, false>(f, c, sX, sZT, sZR, q, x, y, cx, cy, rx, ry, pre);
    float pold[U];
#if LS_XEARLY
    float xo[U];
    if (xupd && own) {   // x loads issued before the stage barrier (timing experiment)
      const size_t i = (size_t)y * W + x;
#pragma unroll
      for (int u = 0; u < U; ++u) xo[u] = xread ? xv[(size_t)u * N + i] : 0.f;
    }
#endif
    if (own) {
      const int i = y * W + x;
      const int sc0 = cy * kSW + cx, rc0 = ry * kRW + rx;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const size_t o = (size_t)ch * N + i;
        pnew[o] = sZR[ch * kRP + rc0];
      }
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const size_t o = (size_t)(3 + k) * N + i;
        pnew[o] = sZT[k * kSP + sc0];
      }
      if (xupd) {   // p_{i-1} of the own pixel into registers before the stage is released
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) pold[ch] = LS_PFORM_GLOBAL ? __ldg(pprev + (size_t)ch * N + i) : sPR[ch * kRP + rc0];
#pragma unroll
        for (int k = 0; k < NT; ++k)
          pold[3 + k] = LS_PFORM_GLOBAL ? __ldg(pprev + (size_t)(3 + k) * N + i) : sPT[k * kSP + sc0];
      }
    }
    if (TMA) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const int t = blockIdx.x + (j + 1) * gridDim.x;
        if (t < ntiles) {
          int nx, ny;
          walk.next(nx, ny);
          tma_issue_pcg<NT>(smem, maps, &bars[0], nx * kTileW, f.y_lo + ny * kTileH, with_p);
          if (LS_PEARLY && with_p && xupd)   // the deferred x-update still needed p_{i-1} here
            tma_issue_pprev<NT>(smem, maps, &bars[2], nx * kTileW, f.y_lo + ny * kTileH);
        }
      }
    }
    if (xupd && own) {   // x += alpha_{i-1} p_{i-1}, overlapping the next tile's loads
      const size_t i = (size_t)y * W + x;
#if LS_XDEFER
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xo_d[u] = xread ? xv[(size_t)u * N + i] : 0.f;
        pold_d[u] = pold[u];
      }
      pend = true;
      pend_i = i;
#else
#if !LS_XEARLY
      float xo[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xo[u] = xread ? xv[(size_t)u * N + i] : 0.f;
#endif
#pragma unroll
      for (int u = 0; u < U; ++u) xv[(size_t)u * N + i] = fmaf(ax, pold[u], xo[u]);
#endif
    }
    accd += (double)acc;
    acc = 0.f;
  }
#if LS_XDEFER
  if (pend) {
#pragma unroll
    for (int u = 0; u < U; ++u) xv[(size_t)u * N + pend_i] = fmaf(ax, pold_d[u], xo_d[u]);
  }
#endif
  double accv[1] = {accd};
  block_reduce_store<1>(accv, part);
  if (!last_block(ticket)) return;
  const double pap = sum_partials<1>(part, gridDim.x, 0);
  if (threadIdx.x == 0) {
    if (f.bsum) f.bsum[0] = pap;
    else fin_pcg_apply(pap, sc, iter);
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------
// Single-reduction PCG (Chronopoulos-Gear form of solver.py:79-107, the
// north star's "one grid-level reduction per PCG step"), ONE kernel per
// iteration, in preconditioned variables (M = diag^-1 = dinv):
//   u = M r,  m = M w (w = A u),  t = M s (s = w + beta s)
//   iteration i:  t_i = m_i + beta_i t_{i-1};  u_{i+1} = u_i - alpha_i t_i
//                 p_i = u_i + beta_i p_{i-1};   x += alpha_i p_i
//                 w_{i+1} = A u_{i+1},  m_{i+1} = M w_{i+1}
//                 gamma = (r, u) = sum u^2 / dinv,  delta = (w, u),  |r|^2
//   last CTA:     beta = gamma_{i+1} / gamma_i,
//                 pAp = delta - beta gamma_{i+1} / alpha_i,  alpha = gamma_{i+1} / pAp
// The three operands u_i, m_i, t_{i-1} are staged over tile + halo (t and
// u_{i+1} are formed over the whole window), so the stencil of u_{i+1} needs
// no second pass: 12U HBM words per pixel per iteration -- the same as the
// two-kernel textbook loop -- and one fp64 reduction of (delta, gamma, |r|^2).
// The textbook loop's breaks map one to one: gamma_{i+1} <= 0 is its
// rz_new <= 0 after update i, pAp_{i+1} <= 0 its pAp <= 0 before update i+1.
// Three operand windows are 100 KB of shared memory per CTA (2 CTAs / SM).
// CG_INIT: w_0 = A u_0, m_0 = M w_0, delta_0 (gamma_0 comes from EG).
// ---------------------------------------------------------------------------
enum { CG_INIT = 0, CG_ITER = 1, CG_LAST = 2 };
__host__ __device__ constexpr int cg_stage(int NT) { return pad32((NT + 3) * kSP) + 3 * op_floats(NT); }

template <int NT>
__device__ __forceinline__ void tma_issue_cg(float* stage, const CgMaps& m, uint64_t* bar, int tx0, int ty0,
                                             int mode, bool with_t) {
  constexpr uint32_t xb = sizeof(float) * (NT + 3) * kSP;
  constexpr uint32_t ob = sizeof(float) * (NT * kSP + 3 * kRP);
  const int nop = mode == CG_INIT ? 1 : (with_t ? 3 : 2);
  mbar_expect_tx(bar, xb + nop * ob);
  float* o = stage + pad32((NT + 3) * kSP);
  tma_load_3d(stage, &m.X, bar, tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(o, &m.UT, bar, tx0 - kSX, ty0 - 1, 0);
  tma_load_3d(o + pad32(NT * kSP), &m.UR, bar, tx0 - kRX, ty0 - kHalf, 0);
  if (mode != CG_INIT) {
    o += op_floats(NT);
    tma_load_3d(o, &m.MT, bar, tx0 - kSX, ty0 - 1, 0);
    tma_load_3d(o + pad32(NT * kSP), &m.MR, bar, tx0 - kRX, ty0 - kHalf, 0);
    if (with_t) {
      o += op_floats(NT);
      tma_load_3d(o, &m.TT, bar, tx0 - kSX, ty0 - 1, 0);
      tma_load_3d(o + pad32(NT * kSP), &m.TR, bar, tx0 - kRX, ty0 - kHalf, 0);
    }
  }
}

template <int NT, int MODE>
__global__ void __launch_bounds__(kThreads, 2) k_cg_iter(Frame f, Coef<float> c, const float* __restrict__ X,
                                                         const float* __restrict__ dinv, float* __restrict__ u_out,
                                                         float* __restrict__ m_out, float* __restrict__ t_out,
                                                         float* __restrict__ p, float* __restrict__ xv, double* part,
                                                         unsigned* ticket, Scalars* sc, int iter, int ntiles,
                                                         const __grid_constant__ CgMaps maps) {
  constexpr int U = NT + 3;
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bar;
  if (sc->stop) return;
  const int W = f.W, N = f.N;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int cx = lx + kSX, cy = ly + 1, rx = lx + kRX, ry = ly + kHalf;
  const int ntx = (W + kTileW - 1) / kTileW;
  const bool with_t = MODE != CG_INIT && iter > 0;
  const float alpha = (float)sc->alpha, beta = (float)sc->beta;
  const bool xread = sc->xinit;
  float* sX = smem;
  float* sUT = smem + pad32(U * kSP);
  float* sUR = sUT + pad32(NT * kSP);
  float* sMT = sUT + op_floats(NT);
  float* sTT = sMT + op_floats(NT);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    if ((int)blockIdx.x < ntiles) {
      const int t = blockIdx.x;
      tma_issue_cg<NT>(smem, maps, &bar, (t % ntx) * kTileW, f.y_lo + (t / ntx) * kTileH, MODE, with_t);
    }
  }
  __syncthreads();
  uint32_t phase = 0;
  double acc[3] = {0.0, 0.0, 0.0};   // delta = <w, u>, gamma = <r, u>, |r|^2
  for (int j = 0;; ++j) {
    const int tile = blockIdx.x + j * gridDim.x;
    if (tile >= ntiles) break;
    const int tx0 = (tile % ntx) * kTileW, ty0 = f.y_lo + (tile / ntx) * kTileH;
    const int x = tx0 + lx, y = ty0 + ly;
    const bool own = x < W && y < f.y_hi;
    const size_t i = (size_t)y * W + x;
    const PixPre pre = pix_prefetch(f, x, y, own);
    mbar_wait(&bar, phase);
    phase ^= 1u;
    const int sc0 = cy * kSW + cx, rc0 = ry * kRW + rx;
    if (MODE != CG_INIT) {
      float ui[U];     // u_i of the own pixel, before the window is advanced
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) ui[ch] = sUR[ch * kRP + rc0];
#pragma unroll
      for (int k = 0; k < NT; ++k) ui[3 + k] = sUT[k * kSP + sc0];
      __syncthreads();
      // t_i = m_i + beta t_{i-1};  u_{i+1} = u_i - alpha t_i  over tile + halo
      static_assert((NT * kSP) % 4 == 0 && (3 * kRP) % 4 == 0, "float4 formation");
      constexpr int n4 = op_floats(NT) / 4;
      float4* u4 = reinterpret_cast<float4*>(sUT);
      float4* m4 = reinterpret_cast<float4*>(sMT);
      const float4* t4 = reinterpret_cast<const float4*>(sTT);
      for (int e = threadIdx.x; e < n4; e += kThreads) {
        float4 tt = m4[e];
        if (with_t) {
          const float4 tp = t4[e];
          tt.x = fmaf(beta, tp.x, tt.x); tt.y = fmaf(beta, tp.y, tt.y);
          tt.z = fmaf(beta, tp.z, tt.z); tt.w = fmaf(beta, tp.w, tt.w);
        }
        float4 uu = u4[e];
        uu.x = fmaf(-alpha, tt.x, uu.x); uu.y = fmaf(-alpha, tt.y, uu.y);
        uu.z = fmaf(-alpha, tt.z, uu.z); uu.w = fmaf(-alpha, tt.w, uu.w);
        m4[e] = tt;     // t_i now lives in the m region
        u4[e] = uu;
      }
      __syncthreads();
      if (own) {   // p_i = u_i + beta p_{i-1};  x += alpha p_i;  t_i, u_{i+1} out
        float pv[U], xo[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          pv[u] = iter > 0 ? __ldg(p + (size_t)u * N + i) : 0.f;
          xo[u] = xread ? xv[(size_t)u * N + i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float pn = iter > 0 ? fmaf(beta, pv[u], ui[u]) : ui[u];
          p[(size_t)u * N + i] = pn;
          xv[(size_t)u * N + i] = fmaf(alpha, pn, xo[u]);
        }
        double gm = 0.0, rn = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool isr = u < 3;
          const float tv = isr ? sMT[pad32(NT * kSP) + u * kRP + rc0] : sMT[(u - 3) * kSP + sc0];
          const float uv = isr ? sUR[u * kRP + rc0] : sUT[(u - 3) * kSP + sc0];
          if (MODE == CG_ITER) {
            t_out[(size_t)u * N + i] = tv;
            u_out[(size_t)u * N + i] = uv;
          }
          const float rv = __fdividef(uv, __ldg(dinv + (size_t)u * N + i));   // r = u / dinv
          gm += (double)(rv * uv);
          rn += (double)(rv * rv);
        }
        acc[1] += gm;
        acc[2] += rn;
      }
    }
    if (MODE != CG_LAST) {   // w = A u (u_{i+1}, or u_0 in CG_INIT); m = dinv w written
      const bool interior = tx0 > 0 && ty0 > 0 && tx0 + kTileW < W && ty0 + kTileH < f.H && ty0 + kTileH <= f.y_hi;
      float d = 0.f;
      if (interior)
        d = apply_pixel<NT, true, true>(f, c, sX, sUT, sUR, m_out, x, y, cx, cy, rx, ry, pre, dinv);
      else if (own)
        d = apply_pixel<NT, false, true>(f, c, sX, sUT, sUR, m_out, x, y, cx, cy, rx, ry, pre, dinv);
      acc[0] += (double)d;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t = blockIdx.x + (j + 1) * gridDim.x;
      if (t < ntiles) tma_issue_cg<NT>(smem, maps, &bar, (t % ntx) * kTileW, f.y_lo + (t / ntx) * kTileH, MODE, with_t);
    }
  }
  block_reduce_store<3>(acc, part);
  if (!last_block(ticket)) return;
  const double delta = sum_partials<3>(part, gridDim.x, 0);
  const double gamma = sum_partials<3>(part, gridDim.x, 1);
  const double rn = sum_partials<3>(part, gridDim.x, 2);
  if (threadIdx.x == 0) {
    if (MODE == CG_INIT) {   // p_0 = u_0: pAp_0 = delta_0 (solver.py:94-96)
      sc->delta = delta;
      if (!(delta > 0.0) || !isfinite(delta)) sc->stop = 1;
      else { sc->alpha = sc->gamma / delta; sc->beta = 0.0; }
    } else {
      sc->iterations = iter + 1;   // x now holds iteration i's update
      sc->xinit = 1;
      sc->pending = 0;
      sc->rnorm2 = rn;
      if (MODE == CG_ITER) {
        if (gamma <= 0.0) {
          sc->stop = 1;              // rz_new <= 0 (solver.py:101-103)
        } else {
          const double b = gamma / sc->gamma;
          const double pap = delta - b * gamma / sc->alpha;
          sc->delta = pap;
          if (!(pap > 0.0) || !isfinite(pap)) {
            sc->stop = 1;            // the next iteration's pAp <= 0 (solver.py:95-96)
          } else {
            sc->beta = b;
            sc->alpha_prev = sc->alpha;
            sc->alpha = gamma / pap;
            sc->gamma_prev = sc->gamma;
            sc->gamma = gamma;
          }
        }
      }
    }
    *ticket = 0u;
  }
}

// Row bands (band.planes > 0): only rows [y_lo, y_hi) of every plane, as
// band.planes x band.len4 float4s starting at band.off4 of each plane.
struct BandSpan {
  int planes;
  int len4;
  int64_t off4, plane4;
};

__device__ __forceinline__ int64_t span_index(const BandSpan& b, int64_t j) {
  const int pl = (int)((uint32_t)j / (uint32_t)b.len4);
  return (int64_t)pl * b.plane4 + b.off4 + (j - (int64_t)pl * b.len4);
}

// LAST (the final iteration of a whole-frame PCG): r_{n} is needed only for
// the reported |r| (solver.py:106) and z / beta not at all, so the kernel
// reads r, q and -- instead of dinv -- p and x, folds the last deferred
// x-update x += alpha p in (what k_pcg_xfinal would do) and writes only x.
// LAST_NORM (the last iteration when the directions are stored and combined
// by k_pcg_combine): only |r|^2 is needed -- reads r and q, writes nothing.
template <bool LAST, bool NORM = false>
__global__ void __launch_bounds__(kThreads) k_pcg_update(int64_t M, float* __restrict__ r, const float* __restrict__ q,
                                                         const float* __restrict__ dinv, float* __restrict__ z,
                                                         double* part, unsigned* ticket, Scalars* sc, int iter,
                                                         BandSpan band, double* bsum, const float* __restrict__ p,
                                                         float* __restrict__ xv) {
  pdl_wait();
  pdl_trigger();
  if (sc->stop) return;
  const float a = (float)sc->alpha;
  const bool xread = LAST && sc->xinit;
  double acc[2] = {0.0, 0.0};
  const bool banded = band.planes > 0;
  const int64_t M4 = banded ? (int64_t)band.planes * band.len4 : (M >> 2);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#if LS_KEEP_R
  for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < M4; jj += stride) {
    const int64_t j = banded ? span_index(band, jj) : jj;
    float4 rr = reinterpret_cast<const float4*>(r)[j];
    const float4 qq = __ldg(reinterpret_cast<const float4*>(q) + j);
    rr = make_float4(fmaf(-a, qq.x, rr.x), fmaf(-a, qq.y, rr.y), fmaf(-a, qq.z, rr.z), fmaf(-a, qq.w, rr.w));
    if (NORM) {
    } else if (LAST) {
      const float4 pp = __ldg(reinterpret_cast<const float4*>(p) + j);
      float4 xx = xread ? reinterpret_cast<const float4*>(xv)[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      xx = make_float4(fmaf(a, pp.x, xx.x), fmaf(a, pp.y, xx.y), fmaf(a, pp.z, xx.z), fmaf(a, pp.w, xx.w));
      reinterpret_cast<float4*>(xv)[j] = xx;
    } else {
      const float4 di = __ldg(reinterpret_cast<const float4*>(dinv) + j);
      const float4 zz = make_float4(rr.x * di.x, rr.y * di.y, rr.z * di.z, rr.w * di.w);
      reinterpret_cast<float4*>(r)[j] = rr;
      reinterpret_cast<float4*>(z)[j] = zz;
      acc[0] += (double)fmaf(rr.x, zz.x, fmaf(rr.y, zz.y, fmaf(rr.z, zz.z, rr.w * zz.w)));
    }
    acc[1] += (double)fmaf(rr.x, rr.x, fmaf(rr.y, rr.y, fmaf(rr.z, rr.z, rr.w * rr.w)));
  }
  for (int64_t j = banded ? M : (M4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride) {
    const float rr = fmaf(-a, q[j], r[j]);
    if (NORM) {
    } else if (LAST) {
      xv[j] = fmaf(a, p[j], xread ? xv[j] : 0.f);
    } else {
      const float zz = rr * dinv[j];
      r[j] = rr;
      z[j] = zz;
      acc[0] += (double)rr * zz;
    }
    acc[1] += (double)rr * rr;
  }
#else
  // the preconditioned residual alone: z_{i+1} = z_i - alpha dinv q_i
  // (r_{i+1} = z_{i+1} / dinv is never stored; rz and |r|^2 use 1/dinv on the
  // fly) -- 4U words per iteration instead of 5U
  auto one = [&](float zv, float qv, float dv, float& zn, double& rz, double& rn) {
    zn = fmaf(-a, qv * dv, zv);
    const float rr = zn * rcpf(dv);
    rz += (double)(rr * zn);
    rn += (double)(rr * rr);
  };
  for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < M4; jj += stride) {
    const int64_t j = banded ? span_index(band, jj) : jj;
    const float4 zz = reinterpret_cast<const float4*>(z)[j];
    const float4 qq = __ldg(reinterpret_cast<const float4*>(q) + j);
    const float4 di = __ldg(reinterpret_cast<const float4*>(dinv) + j);
    float4 zn;
    double rz = 0.0, rn = 0.0;
#if LS_UPD_F32P
    {   // the float4's four products summed in fp32, one fp64 add each (A/B)
      float rz4 = 0.f, rn4 = 0.f;
      auto one4 = [&](float zv, float qv, float dv, float& znv) {
        znv = fmaf(-a, qv * dv, zv);
        const float rr = znv * rcpf(dv);
        rz4 = fmaf(rr, znv, rz4);
        rn4 = fmaf(rr, rr, rn4);
      };
      one4(zz.x, qq.x, di.x, zn.x);
      one4(zz.y, qq.y, di.y, zn.y);
      one4(zz.z, qq.z, di.z, zn.z);
      one4(zz.w, qq.w, di.w, zn.w);
      rz = (double)rz4;
      rn = (double)rn4;
    }
#else
    one(zz.x, qq.x, di.x, zn.x, rz, rn);
    one(zz.y, qq.y, di.y, zn.y, rz, rn);
    one(zz.z, qq.z, di.z, zn.z, rz, rn);
    one(zz.w, qq.w, di.w, zn.w, rz, rn);
#endif
    if (NORM) {
    } else if (LAST) {
      const float4 pp = __ldg(reinterpret_cast<const float4*>(p) + j);
      float4 xx = xread ? reinterpret_cast<const float4*>(xv)[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      xx = make_float4(fmaf(a, pp.x, xx.x), fmaf(a, pp.y, xx.y), fmaf(a, pp.z, xx.z), fmaf(a, pp.w, xx.w));
      reinterpret_cast<float4*>(xv)[j] = xx;
    } else {
      reinterpret_cast<float4*>(z)[j] = zn;
    }
    acc[0] += rz;
    acc[1] += rn;
  }
  for (int64_t j = banded ? M : (M4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride) {
    float zn;
    one(z[j], q[j], dinv[j], zn, acc[0], acc[1]);
    if (NORM) {
    } else if (LAST) {
      xv[j] = fmaf(a, p[j], xread ? xv[j] : 0.f);
    } else {
      z[j] = zn;
    }
  }
#endif
  block_reduce_store<2>(acc, part);
  if (!last_block(ticket)) return;
  const double rz = sum_partials<2>(part, gridDim.x, 0);
  const double rn = sum_partials<2>(part, gridDim.x, 1);
  if (threadIdx.x == 0) {
    if (bsum) {
      bsum[0] = rz;
      bsum[1] = rn;
    } else if (NORM) {   // the loop ends here: the count and |r| (x comes from k_pcg_combine)
      sc->iterations = iter + 1;
      sc->rnorm2 = rn;
    } else if (LAST) {   // the loop ends here: record the count and |r|, x is complete
      sc->iterations = iter + 1;
      sc->rnorm2 = rn;
      sc->pending = 0;
      sc->xinit = 1;
    } else {
      fin_pcg_update(rz, rn, sc, iter);
    }
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------
// host-side launchers (dispatch on NT)
// ---------------------------------------------------------------------------
#define LS_DISPATCH_NT(NTV, CALL)                       \
  switch (NTV) {                                        \
    case 1: { constexpr int NT_ = 1; CALL; } break;     \
    case 2: { constexpr int NT_ = 2; CALL; } break;     \
    case 3: { constexpr int NT_ = 3; CALL; } break;     \
    case 4: { constexpr int NT_ = 4; CALL; } break;     \
    case 5: { constexpr int NT_ = 5; CALL; } break;     \
    case 6: { constexpr int NT_ = 6; CALL; } break;     \
    case 7: { constexpr int NT_ = 7; CALL; } break;     \
    case 8: { constexpr int NT_ = 8; CALL; } break;     \
    case 9: { constexpr int NT_ = 9; CALL; } break;     \
    case 10: { constexpr int NT_ = 10; CALL; } break;   \
    case 11: { constexpr int NT_ = 11; CALL; } break;   \
    case 12: { constexpr int NT_ = 12; CALL; } break;   \
    case 13: { constexpr int NT_ = 13; CALL; } break;   \
    default: break;                                     \
  }

template <int NT>
static size_t energy_smem(int mode, bool tma) {
  const bool trial = mode == MODE_TRIAL;
  return sizeof(float) * e_stage(NT, trial) * ((tma && !trial) ? 2 : 1);
}
template <int NT>
static size_t apply_smem(bool tma) { return sizeof(float) * tile_floats(NT, true) * (tma ? 2 : 1); }

// LS_PCG_PAD (timing experiments only, tools/ablate.py): extra shared memory
// per CTA to pin the operator kernel's occupancy (e.g. 2 CTAs / SM)
#ifndef LS_PCG_PAD
#define LS_PCG_PAD 0
#endif
template <int NT>
static size_t pcg_smem(bool tma) { return sizeof(float) * pcg_stage(NT, tma) + LS_PCG_PAD; }

template <int NT>
static void prepare_nt() {
  cudaFuncSetAttribute(k_pcg_apply<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcg_smem<NT>(true));
  cudaFuncSetAttribute(k_pcg_apply<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcg_smem<NT>(false));
  cudaFuncSetAttribute(k_energy<NT, MODE_EG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)energy_smem<NT>(MODE_EG, true));
  cudaFuncSetAttribute(k_energy<NT, MODE_EG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)energy_smem<NT>(MODE_EG, false));
  cudaFuncSetAttribute(k_energy<NT, MODE_TRIAL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)energy_smem<NT>(MODE_TRIAL, true));
  cudaFuncSetAttribute(k_energy<NT, MODE_TRIAL, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)energy_smem<NT>(MODE_TRIAL, true));
  cudaFuncSetAttribute(k_energy<NT, MODE_TRIAL, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)energy_smem<NT>(MODE_TRIAL, false));
  cudaFuncSetAttribute(k_apply<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)apply_smem<NT>(true));
  cudaFuncSetAttribute(k_apply<NT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)apply_smem<NT>(false));
}

void prepare_kernels(int NT) { LS_DISPATCH_NT(NT, (prepare_nt<NT_>())); }

template <int NT, int MODE>
static void launch_energy_mt(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* dx,
                             float alpha, const float* Y, float* Xout, float* r_out, float* d_out, float* u_out,
                             float* b_raw, float* diag_raw, double* part, unsigned* ticket, Scalars* sc,
                             const EnergyMaps* maps, const FrameCtl* ctl, int dev_ls, int last_trial,
                             unsigned long long next_cond) {
  if constexpr (MODE == MODE_TRIAL) {
    if (maps && next_cond) {
      launch_pdl(k_energy<NT, MODE, true, true>, L.grid, kThreads, energy_smem<NT>(MODE, true), L.stream,
                 f, c, X, dx, alpha, Y, Xout, r_out, d_out, u_out, b_raw, diag_raw, part, ticket, sc, L.ntiles, ctl,
                 dev_ls, last_trial, *maps, next_cond);
      return;
    }
  }
  if (maps)
    launch_pdl(k_energy<NT, MODE, true>, L.grid, kThreads, energy_smem<NT>(MODE, true), L.stream,
               f, c, X, dx, alpha, Y, Xout, r_out, d_out, u_out, b_raw, diag_raw, part, ticket, sc, L.ntiles, ctl,
               dev_ls, last_trial, *maps, 0ULL);
  else
    k_energy<NT, MODE, false><<<L.grid, kThreads, energy_smem<NT>(MODE, false), L.stream>>>(
        f, c, X, dx, alpha, Y, Xout, r_out, d_out, u_out, b_raw, diag_raw, part, ticket, sc, L.ntiles, ctl, dev_ls,
        last_trial, EnergyMaps{}, next_cond);
}

template <int NT>
static void launch_energy_nt(int mode, const Launch& L, const Frame& f, const Coef<float>& c, const float* X,
                             const float* dx, float alpha, const float* Y, float* Xout, float* r_out, float* d_out,
                             float* u_out, float* b_raw, float* diag_raw, double* part, unsigned* ticket,
                             Scalars* sc, const EnergyMaps* maps, const FrameCtl* ctl, int dev_ls, int last_trial,
                             unsigned long long next_cond) {
  if (mode == MODE_EG)
    launch_energy_mt<NT, MODE_EG>(L, f, c, X, dx, alpha, Y, Xout, r_out, d_out, u_out, b_raw, diag_raw, part, ticket,
                                  sc, maps, ctl, dev_ls, last_trial, 0ULL);
  else
    launch_energy_mt<NT, MODE_TRIAL>(L, f, c, X, dx, alpha, Y, Xout, r_out, d_out, u_out, b_raw, diag_raw, part,
                                     ticket, sc, maps, ctl, dev_ls, last_trial, next_cond);
}

template <int NT>
static void launch_apply_nt(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* u,
                            float* w, double* part, unsigned* ticket, Scalars* sc, int iter, const TileMaps* maps) {
  if (maps)
    k_apply<NT, true><<<L.grid, kThreads, apply_smem<NT>(true), L.stream>>>(f, c, X, u, w, part, ticket, sc, iter,
                                                                          L.ntiles, *maps);
  else
    k_apply<NT, false><<<L.grid, kThreads, apply_smem<NT>(false), L.stream>>>(f, c, X, u, w, part, ticket, sc, iter,
                                                                            L.ntiles, TileMaps{});
}

void launch_energy(int mode, const Launch& L, const Frame& f, const Coef<float>& c, const float* X,
                   const float* dx, float alpha, const float* Y, float* Xout, float* r_out, float* d_out,
                   float* u_out, float* b_raw, float* diag_raw, double* part, unsigned* ticket, Scalars* sc,
                   const EnergyMaps* maps, const FrameCtl* ctl, int dev_ls, int last_trial,
                   unsigned long long next_cond) {
  LS_DISPATCH_NT(f.NT, (launch_energy_nt<NT_>(mode, L, f, c, X, dx, alpha, Y, Xout, r_out, d_out, u_out, b_raw,
                                              diag_raw, part, ticket, sc, maps, ctl, dev_ls, last_trial,
                                              next_cond)));
}

// ---------------------------------------------------------------------------
// device-resident flip-flop bookkeeping (solver.py:311-338, refine = False)
// ---------------------------------------------------------------------------
__global__ void k_frame_init(FrameCtl* ctl) {
  pdl_wait();
  pdl_trigger();
  ctl->done = ctl->converged = ctl->stalled = ctl->has_hist = ctl->e_prev_valid = 0;
  ctl->n_exec = 0;
  ctl->cur = 0;
  ctl->fault_step = -1;
  ctl->e_last = ctl->e_prev = 0.0;
}

// end of one GN step: the state moves to buffer `out_id` (copied through on a
// rejected step, solver.py:169-178 leaves it unchanged); record + bookkeeping
__global__ void k_step_end(FrameCtl* ctl, const Scalars* sc, const float* __restrict__ Xin, float* __restrict__ Xout,
                           int64_t M, int out_id, StepRecord* recs) {
  pdl_wait();
  pdl_trigger();
  if (ctl->done) return;
  const bool fault = sc->fault;
  const bool acc = sc->accepted && !fault;
  if (!acc && !fault)
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x)
      Xout[j] = Xin[j];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    StepRecord& R = recs[ctl->n_exec];
    R.e0 = sc->e0;
    R.e1 = acc ? sc->e1 : sc->e0;
    R.alpha = acc ? sc->alpha_ls : 0.0;
    R.bnorm2 = sc->bnorm2;
    R.rnorm2 = sc->rnorm2;
    for (int j = 0; j < kTerms; ++j) {
      R.terms0[j] = sc->terms0[j];
      R.terms1[j] = acc ? sc->terms1[j] : sc->terms0[j];
    }
    R.accepted = acc;
    R.iterations = sc->iterations;
    R.fault = fault;
    if (fault) {
      ctl->done = 1;
      ctl->fault_step = ctl->n_exec;
    } else {
      ctl->cur = out_id;
      if (acc) {
        ctl->e_last = sc->e1;
        ctl->has_hist = 1;
      } else {
        ctl->stalled = 1;
      }
    }
    ctl->n_exec += 1;
  }
}

// end of one outer iteration: relative-decrease convergence (solver.py:328-336)
__global__ void k_outer_end(FrameCtl* ctl, double tol_rel) {
  pdl_wait();
  pdl_trigger();
  if (ctl->done || !ctl->has_hist) return;
  const double e_now = ctl->e_last;
  if (ctl->e_prev_valid && ctl->e_prev > 0.0) {
    const double rel = (ctl->e_prev - e_now) / ctl->e_prev;
    if (0.0 <= rel && rel < tol_rel) {
      ctl->converged = 1;
      ctl->done = 1;
      return;
    }
  }
  ctl->e_prev = e_now;
  ctl->e_prev_valid = 1;
}

void launch_frame_init(cudaStream_t s, FrameCtl* ctl) { launch_pdl(k_frame_init, 1, 1, 0, s, ctl); }
void launch_step_end(cudaStream_t s, int grid, FrameCtl* ctl, const Scalars* sc, const float* Xin, float* Xout,
                     int64_t M, int out_id, StepRecord* recs) {
  launch_pdl(k_step_end, grid, kThreads, 0, s, ctl, sc, Xin, Xout, M, out_id, recs);
}
void launch_outer_end(cudaStream_t s, FrameCtl* ctl, double tol_rel) { launch_pdl(k_outer_end, 1, 1, 0, s, ctl, tol_rel); }

void launch_apply(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* u,
                  float* w, double* part, unsigned* ticket, Scalars* sc, int iter, const TileMaps* maps) {
  LS_DISPATCH_NT(f.NT, (launch_apply_nt<NT_>(L, f, c, X, u, w, part, ticket, sc, iter, maps)));
}

template <int NT>
static void launch_pcg_apply_nt(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* z,
                                const float* pprev, float* pnew, float* q, double* part, unsigned* ticket,
                                Scalars* sc, int iter, const PcgMaps* maps, float* x) {
  if (maps)
    launch_pdl(k_pcg_apply<NT, true>, L.grid, kThreads, pcg_smem<NT>(true), L.stream, f, c, X, z, pprev, pnew, q,
               part, ticket, sc, iter, L.ntiles, *maps, x);
  else
    k_pcg_apply<NT, false><<<L.grid, kThreads, pcg_smem<NT>(false), L.stream>>>(f, c, X, z, pprev, pnew, q, part, ticket,
                                                                          sc, iter, L.ntiles, PcgMaps{}, x);
}

void launch_pcg_apply(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* z,
                      const float* pprev, float* pnew, float* q, double* part, unsigned* ticket, Scalars* sc,
                      int iter, const PcgMaps* maps, float* x) {
  LS_DISPATCH_NT(f.NT, (launch_pcg_apply_nt<NT_>(L, f, c, X, z, pprev, pnew, q, part, ticket, sc, iter, maps, x)));
}

template <int NT>
static size_t cg_smem() { return sizeof(float) * cg_stage(NT); }

template <int NT>
static void launch_cg_nt(const Launch& L, int mode, const Frame& f, const Coef<float>& c, const float* X,
                         const float* dinv, float* u_out, float* m_out, float* t_out, float* p, float* xv,
                         double* part, unsigned* ticket, Scalars* sc, int iter, const CgMaps& maps) {
  const size_t sm = cg_smem<NT>();
  switch (mode) {
    case CG_INIT:
      cudaFuncSetAttribute(k_cg_iter<NT, CG_INIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_cg_iter<NT, CG_INIT><<<L.grid, kThreads, sm, L.stream>>>(f, c, X, dinv, u_out, m_out, t_out, p, xv, part,
                                                                 ticket, sc, iter, L.ntiles, maps);
      break;
    case CG_ITER:
      cudaFuncSetAttribute(k_cg_iter<NT, CG_ITER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_cg_iter<NT, CG_ITER><<<L.grid, kThreads, sm, L.stream>>>(f, c, X, dinv, u_out, m_out, t_out, p, xv, part,
                                                                 ticket, sc, iter, L.ntiles, maps);
      break;
    default:
      cudaFuncSetAttribute(k_cg_iter<NT, CG_LAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_cg_iter<NT, CG_LAST><<<L.grid, kThreads, sm, L.stream>>>(f, c, X, dinv, u_out, m_out, t_out, p, xv, part,
                                                                 ticket, sc, iter, L.ntiles, maps);
      break;
  }
}

void launch_cg(const Launch& L, int mode, const Frame& f, const Coef<float>& c, const float* X, const float* dinv,
               float* u_out, float* m_out, float* t_out, float* p, float* xv, double* part, unsigned* ticket,
               Scalars* sc, int iter, const CgMaps& maps) {
  LS_DISPATCH_NT(f.NT, (launch_cg_nt<NT_>(L, mode, f, c, X, dinv, u_out, m_out, t_out, p, xv, part, ticket, sc, iter,
                                          maps)));
}

int cg_grid_limit(int NT) {
  int nb = 0;
  LS_DISPATCH_NT(NT, (cudaFuncSetAttribute(k_cg_iter<NT_, CG_ITER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)cg_smem<NT_>()),
                      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cg_iter<NT_, CG_ITER>, kThreads,
                                                                    cg_smem<NT_>())));
  return nb;
}

// the last deferred x-update after the PCG loop: x += alpha_j p_j for the
// last completed iteration j (k_pcg_update's finalisation left it pending)
__global__ void __launch_bounds__(kThreads) k_pcg_xfinal(int64_t M, float* __restrict__ xv,
                                                         const float* __restrict__ p0,
                                                         const float* __restrict__ p1, Scalars* sc,
                                                         unsigned* ticket, BandSpan band) {
  pdl_wait();
  pdl_trigger();
  if (!sc->pending) return;
  const float a = (float)sc->alpha;
  const float* __restrict__ p = ((sc->iterations - 1) & 1) ? p1 : p0;
  const bool xread = sc->xinit;
  const bool banded = band.planes > 0;
  const int64_t M4 = banded ? (int64_t)band.planes * band.len4 : (M >> 2);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < M4; jj += stride) {
    const int64_t j = banded ? span_index(band, jj) : jj;
    const float4 pp = __ldg(reinterpret_cast<const float4*>(p) + j);
    float4 xx = xread ? reinterpret_cast<const float4*>(xv)[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    xx = make_float4(fmaf(a, pp.x, xx.x), fmaf(a, pp.y, xx.y), fmaf(a, pp.z, xx.z), fmaf(a, pp.w, xx.w));
    reinterpret_cast<float4*>(xv)[j] = xx;
  }
  for (int64_t j = banded ? M : (M4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride)
    xv[j] = fmaf(a, p[j], xread ? xv[j] : 0.f);
  if (!last_block(ticket)) return;
  if (threadIdx.x == 0) {
    sc->pending = 0;
    sc->xinit = 1;
    *ticket = 0u;
  }
}

static BandSpan band_span(const Frame* band) {
  BandSpan bs{0, 0, 0, 0};
  if (band && (band->y_lo != 0 || band->y_hi != band->H)) {   // W % 4 == 0 checked by ls_band_set
    bs.planes = band->NT + 3;
    bs.len4 = (band->y_hi - band->y_lo) * band->W / 4;
    bs.off4 = (int64_t)band->y_lo * band->W / 4;
    bs.plane4 = (int64_t)band->N / 4;
  }
  return bs;
}

// x = sum_i alpha_i p_i over the stored search directions of the finished
// loop (n = the iterations it ran), in iteration order with fmaf -- the
// same operations as the textbook loop's x += alpha_i p_i, so the same bits.
// Replaces the per-iteration x read / write of the deferred x-update.
__global__ void __launch_bounds__(kThreads) k_pcg_combine(int64_t M, DirList dl, float* __restrict__ xv, Scalars* sc) {
  const int n = min(sc->iterations, dl.n);
  if (n <= 0) return;
  __shared__ float a[kMaxStoredDirs];
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = (float)sc->alpha_hist[i];
  __syncthreads();
  const int64_t M4 = M >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M4; j += stride) {
    float4 xx = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
      const float4 pp = __ldg(reinterpret_cast<const float4*>(dl.p[i]) + j);
      xx = make_float4(fmaf(a[i], pp.x, xx.x), fmaf(a[i], pp.y, xx.y), fmaf(a[i], pp.z, xx.z), fmaf(a[i], pp.w, xx.w));
    }
    reinterpret_cast<float4*>(xv)[j] = xx;
  }
  for (int64_t j = (M4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride) {
    float xx = 0.f;
    for (int i = 0; i < n; ++i) xx = fmaf(a[i], dl.p[i][j], xx);
    xv[j] = xx;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->xinit = 1;
    sc->pending = 0;
  }
}

void launch_pcg_combine(const Launch& L, int64_t M, const DirList& dl, float* xv, Scalars* sc) {
  k_pcg_combine<<<L.grid, kThreads, 0, L.stream>>>(M, dl, xv, sc);
}

void launch_pcg_xfinal(const Launch& L, int64_t M, float* xv, const float* p0, const float* p1, Scalars* sc,
                       unsigned* ticket, const Frame* band) {
  launch_pdl(k_pcg_xfinal, L.grid, kThreads, 0, L.stream, M, xv, p0, p1, sc, ticket, band_span(band));
}

void launch_pcg_update(const Launch& L, int64_t M, float* r, const float* q, const float* dinv, float* z,
                       const float* p, float* xv, double* part, unsigned* ticket, Scalars* sc, int iter,
                       const Frame* band, int last) {
  const BandSpan bs = band_span(band);
  double* bsum = band ? band->bsum : nullptr;
  if (last == 2 && !band)
    launch_pdl(k_pcg_update<true, true>, L.grid, kThreads, 0, L.stream, M, r, q, dinv, z, part, ticket, sc, iter, bs,
               bsum, p, xv);
  else if (last && !band)
    launch_pdl(k_pcg_update<true>, L.grid, kThreads, 0, L.stream, M, r, q, dinv, z, part, ticket, sc, iter, bs, bsum,
               p, xv);
  else
    launch_pdl(k_pcg_update<false>, L.grid, kThreads, 0, L.stream, M, r, q, dinv, z, part, ticket, sc, iter, bs, bsum,
               p, xv);
}

// band-ordered sum of the gathered partials [nbands][nv], then the same
// finalisation the single-frame kernels run in their last CTA
__global__ void k_band_finalize(int phase, const double* __restrict__ g, int nbands, int nv, Scalars* sc, int iter,
                                float alpha, int dev_ls, int last_trial, const FrameCtl* ctl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // device-resident flip-flop: the kernels of a finished frame / decided
  // line search exited without writing partials
  if (ctl && ctl->done) return;
  if (phase == BAND_TRIAL && dev_ls && sc->ls_done) return;
  double tot[kTerms + 2];
  for (int j = 0; j < nv && j < kTerms + 2; ++j) {
    double s = 0.0;
    for (int b = 0; b < nbands; ++b) s += g[(size_t)b * nv + j];
    tot[j] = s;
  }
  switch (phase) {
    case BAND_EG: fin_energy_eg(tot, sc, true); break;
    case BAND_TRIAL: fin_energy_trial(tot, sc, alpha, dev_ls, last_trial); break;
    case BAND_APPLY: if (!sc->stop) fin_pcg_apply(tot[0], sc, iter); break;
    case BAND_UPDATE: if (!sc->stop) fin_pcg_update(tot[0], tot[1], sc, iter); break;
    default: break;
  }
}

void launch_band_finalize(cudaStream_t s, int phase, const double* gathered, int nbands, int nv, Scalars* sc,
                          int iter, float alpha, int dev_ls, int last_trial, const FrameCtl* ctl) {
  k_band_finalize<<<1, 32, 0, s>>>(phase, gathered, nbands, nv, sc, iter, alpha, dev_ls, last_trial, ctl);
}

// every band of one process at once: block b sums all bands' partials in band
// order (the same sums as k_band_finalize over the gathered copy) and
// finalises band b's scalars -- one launch instead of copies + a gather + one
// finalisation per band
__global__ void k_band_finalize_group(int phase, BandGroup g, int nv, int iter, float alpha, int last_trial) {
  if (threadIdx.x != 0 || blockIdx.x >= (unsigned)g.n) return;
  const int b = blockIdx.x;
  Scalars* sc = g.sc[b];
  const FrameCtl* ctl = g.ctl[b];
  if (ctl && ctl->done) return;
  if (phase == BAND_TRIAL && sc->ls_done) return;
  double tot[kTerms + 2];
  for (int j = 0; j < nv && j < kTerms + 2; ++j) {
    double s = 0.0;
    for (int bb = 0; bb < g.n; ++bb) s += ((volatile const double*)g.bsum[bb])[j];
    tot[j] = s;
  }
  switch (phase) {
    case BAND_EG: fin_energy_eg(tot, sc, true); break;
    case BAND_TRIAL: fin_energy_trial(tot, sc, alpha, 1, last_trial); break;
    case BAND_APPLY: if (!sc->stop) fin_pcg_apply(tot[0], sc, iter); break;
    case BAND_UPDATE: if (!sc->stop) fin_pcg_update(tot[0], tot[1], sc, iter); break;
    default: break;
  }
}

void launch_band_finalize_group(cudaStream_t s, int phase, const BandGroup& g, int nv, int iter, float alpha,
                                int last_trial) {
  k_band_finalize_group<<<g.n, 32, 0, s>>>(phase, g, nv, iter, alpha, last_trial);
}

// strided slab copies in one launch (the halo moves between the bands of one
// process): slab i copies planes x count floats, plane strides given
__global__ void k_copy_slabs(SlabList L) {
  for (int i = 0; i < L.n; ++i) {
    const Slab& sl = L.s[i];
    const int64_t total = (int64_t)sl.planes * sl.count;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t pl = e / sl.count, k = e - pl * sl.count;
      sl.dst[pl * sl.dst_stride + k] = sl.src[pl * sl.src_stride + k];
    }
  }
}

void launch_copy_slabs(cudaStream_t s, const SlabList& L, int grid) {
  if (L.n > 0) k_copy_slabs<<<grid, 256, 0, s>>>(L);
}

int pcg_apply_grid_limit(int NT) {
  int nb = 0;
  LS_DISPATCH_NT(NT, (prepare_nt<NT_>(), cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                             &nb, k_pcg_apply<NT_, true>, kThreads, pcg_smem<NT_>(true))));
  return nb;
}


int energy_grid_limit(int NT) {
  int nb = 0;
  LS_DISPATCH_NT(NT, (prepare_nt<NT_>(), cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                             &nb, k_energy<NT_, MODE_TRIAL, true>, kThreads,
                                             energy_smem<NT_>(MODE_TRIAL, true))));
  return nb;
}
int apply_grid_limit(int NT) {
  int nb = 0;
  LS_DISPATCH_NT(NT, (prepare_nt<NT_>(), cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                             &nb, k_apply<NT_, true>, kThreads, apply_smem<NT_>(true))));
  return nb;
}

int tile_box_w() { return kSW; }
int tile_box_rw() { return kRW; }
int update_grid_limit() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pcg_update<false>, kThreads, 0);
  return nb;
}

}  // namespace ls
