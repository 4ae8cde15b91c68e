// Sparse-phase kernels of the alternating solver.
//
//   k_energy<NT, MODE_EG>    fused: 8 term energies at the linearisation point,
//                            b = -J^T F, diag(J^T J), Jacobi PCG init
//                            (energy.py:194-511, solver.py:125-140, 79-91)
//   k_energy<NT, MODE_TRIAL> line-search trial: candidate X + a*dx written,
//                            8 energies with weights frozen at X
//                            (solver.py:166-178)
//   k_apply<NT>              w = J^T J u (matrix-free, solver.py:110-122)
//                            + <w,u>; last block advances the PCG scalars
//   k_update                 Chronopoulos-Gear vector update + <r,u>, |r|^2
//
// All heavy kernels are persistent over 32x8 pixel tiles (one warp per tile
// row, one pixel per thread, coalesced plane rows); the 3 log-reflectance
// planes of the operand are staged in shared memory with the 7-pixel halo
// the consistency window needs (energy.py:23, 161-173).  Reductions are
// fp64, fixed-order, finished by the last block (no float atomics).
#include "ls_common.cuh"
#include "ls_kernels.h"

namespace ls {

enum { MODE_EG = 0, MODE_TRIAL = 1 };

template <typename R>
struct PixCtx {
  int x, y, i, W, H, N;
};

// r-sparsity weight at pixel (x, y) from the state planes (energy.py:301-305)
template <typename R>
__device__ __forceinline__ R w_rs_at(const float* __restrict__ X, int N, int W, int H, int x, int y,
                                     const Coef<R>& c) {
  const int i = y * W + x;
  R sx = 0, sy = 0;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const R v = (R)__ldg(X + ch * N + i);
    const R gx = (x < W - 1) ? (R)__ldg(X + ch * N + i + 1) - v : R(0);
    const R gy = (y < H - 1) ? (R)__ldg(X + ch * N + i + W) - v : R(0);
    sx += gx * gx;
    sy += gy * gy;
  }
  return c.lam_rs * irlsp<R>(sqrt(sx + sy), c);
}

// smoothness weights of layer k at (x,y) in x and y (energy.py:314-318)
template <typename R>
__device__ __forceinline__ R w_smx_at(const float* __restrict__ Tk, int W, int i, const Coef<R>& c) {
  return c.lam_sm * irls1<R>((R)__ldg(Tk + i + 1) - (R)__ldg(Tk + i), c.eps_irls, c.inv_eps);
}
template <typename R>
__device__ __forceinline__ R w_smy_at(const float* __restrict__ Tk, int W, int i, const Coef<R>& c) {
  return c.lam_sm * irls1<R>((R)__ldg(Tk + i + W) - (R)__ldg(Tk + i), c.eps_irls, c.inv_eps);
}

__device__ __forceinline__ void tile_coords(int tile, int W, int& tx0, int& ty0) {
  const int ntx = (W + kTileW - 1) / kTileW;
  tx0 = (tile % ntx) * kTileW;
  ty0 = (tile / ntx) * kTileH;
}

// ---------------------------------------------------------------------------
// energy (+ gradient / diagonal / PCG init) kernel, fp64 per-pixel arithmetic
// ---------------------------------------------------------------------------
template <int NT, int MODE>
__global__ void __launch_bounds__(kThreads) k_energy(Frame f, Coef<double> c, const float* __restrict__ X,
                                                     const float* __restrict__ dx, float alpha,
                                                     const float* __restrict__ Yext, float* __restrict__ Xout,
                                                     float* __restrict__ r_out, float* __restrict__ d_out,
                                                     float* __restrict__ u_out, float* __restrict__ b_raw,
                                                     float* __restrict__ diag_raw, double* part,
                                                     unsigned* ticket, Scalars* sc, int ntiles) {
  constexpr int NV = (MODE == MODE_EG) ? kTerms + 2 : kTerms;
  __shared__ float sy[3][kHaloH][kHaloW];
  const int W = f.W, H = f.H, N = f.N;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  // trial: with an empty PCG step the update is zero (solver.py:85-86)
  bool use_dx = (MODE == MODE_TRIAL) && dx != nullptr && sc->iterations > 0;
  const float a = alpha;
  auto Yat = [&](int plane, int idx) -> float {
    if (MODE == MODE_TRIAL && Yext) return __ldg(Yext + (size_t)plane * N + idx);
    float v = __ldg(X + (size_t)plane * N + idx);
    if (MODE == MODE_TRIAL && use_dx) v = __fmaf_rn(a, __ldg(dx + (size_t)plane * N + idx), v);
    return v;
  };

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int tx0, ty0;
    tile_coords(tile, W, tx0, ty0);
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * kHaloH * kHaloW; e += kThreads) {
      const int ch = e / (kHaloH * kHaloW), rem = e % (kHaloH * kHaloW);
      const int yy = rem / kHaloW, xx = rem % kHaloW;
      const int gy = ty0 + yy - kHalf, gx = tx0 + xx - kHalf;
      sy[ch][yy][xx] = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? Yat(ch, gy * W + gx) : 0.f;
    }
    __syncthreads();
    const int x = tx0 + lx, y = ty0 + ly;
    if (x >= W || y >= H) continue;
    const int i = y * W + x;

    // --- state at x (linearisation point) and evaluation point Y ---
    double r0[3], T0[NT], yr[3], yT[NT];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      r0[ch] = (double)__ldg(X + ch * N + i);
      yr[ch] = (double)sy[ch][ly + kHalf][lx + kHalf];
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      T0[k] = (double)__ldg(X + (size_t)(3 + k) * N + i);
      yT[k] = (MODE == MODE_EG) ? T0[k] : (double)Yat(3 + k, i);
    }
    double img[3], anc[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) img[ch] = (double)__ldg(f.img + ch * N + i);
    if (f.ids) {
      const int id = __ldg(f.ids + i);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) anc[ch] = c.anchor[id][ch];
    } else {
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) anc[ch] = (double)__ldg(f.anchor + ch * N + i);
    }
    const double edge = (double)__ldg(f.edge + i);

    // --- data (energy.py:207-209) and monochrome (energy.py:399-401) ---
    double S[3], R[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NT; ++k) s += yT[k] * c.B[k][ch];
      S[ch] = s;
      R[ch] = exp(yr[ch]);
    }
    double res[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      res[ch] = img[ch] - R[ch] * S[ch];
      acc[T_DATA] += c.lam_d * res[ch] * res[ch];
      const double dc = yr[ch] - anc[ch];
      acc[T_CLUSTER] += c.lam_cl * dc * dc;
    }
    const double mean = (S[0] + S[1] + S[2]) / 3.0;
    double m[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      m[ch] = S[ch] - mean;
      acc[T_MONO] += c.lam_m * edge * m[ch] * m[ch];
    }

    // --- r-sparsity at x (weights from X, gradient of Y) ---
    const double wrs = w_rs_at<double>(X, N, W, H, x, y, c);
    {
      double e = 0.0;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const double gx = (x < W - 1) ? (double)sy[ch][ly + kHalf][lx + kHalf + 1] - yr[ch] : 0.0;
        const double gy = (y < H - 1) ? (double)sy[ch][ly + kHalf + 1][lx + kHalf] - yr[ch] : 0.0;
        e += gx * gx + gy * gy;
      }
      acc[T_RSPARSE] += wrs * e;
    }

    // --- per-layer diagonal terms and smoothness ---
    double wis[NT], wnn[NT], axx[NT], ayy[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      wis[k] = (k >= 1) ? c.lam_is * irls1<double>(T0[k], c.eps_irls, c.inv_eps) : 0.0;
      wnn[k] = c.lam_nn * nonneg_w<double>(T0[k], c.eps_nn);
      acc[T_ISPARSE] += wis[k] * yT[k] * yT[k];
      acc[T_NONNEG] += wnn[k] * yT[k] * yT[k];
      const float* Tk = X + (size_t)(3 + k) * N;
      axx[k] = (x < W - 1) ? w_smx_at<double>(Tk, W, i, c) : 0.0;
      ayy[k] = (y < H - 1) ? w_smy_at<double>(Tk, W, i, c) : 0.0;
      const double gx = (x < W - 1) ? (double)Yat(3 + k, i + 1) - yT[k] : 0.0;
      const double gy = (y < H - 1) ? (double)Yat(3 + k, i + W) - yT[k] : 0.0;
      acc[T_SMOOTH] += axx[k] * gx * gx + ayy[k] * gy * gy;
    }

    // --- consistency pairs (energy.py:348-350); each pair counted at its src ---
    double gcons[3] = {0.0, 0.0, 0.0}, dcons = 0.0;
    const int e0 = __ldg(f.row_ptr + i), e1 = __ldg(f.row_ptr + i + 1);
    for (int e = e0; e < e1; ++e) {
      const uint16_t ent = __ldg(f.ent + e);
      const double we = c.lam_rc * (f.ent_w ? (double)__ldg(f.ent_w + e) : 1.0);
      int ddy, ddx;
      decode_offset(ent, ddy, ddx);
      double part_v[3];
      if (ent & kEntTemporal) {
        const int q = i + ddy * W + ddx;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) part_v[ch] = (double)__ldg(f.prev_r + ch * N + q);
      } else {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) part_v[ch] = (double)sy[ch][ly + kHalf + ddy][lx + kHalf + ddx];
      }
      if (!(ent & kEntIncoming)) {
        double e2 = 0.0;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const double dd = yr[ch] - part_v[ch];
          e2 += dd * dd;
        }
        acc[T_CONSIST] += we * e2;
      }
      if (MODE == MODE_EG) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gcons[ch] += we * (yr[ch] - part_v[ch]);
        dcons += we;
      }
    }

    if (MODE == MODE_TRIAL) {
      if (Xout) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) Xout[ch * N + i] = (float)yr[ch];
#pragma unroll
        for (int k = 0; k < NT; ++k) Xout[(size_t)(3 + k) * N + i] = (float)yT[k];
      }
      continue;
    }

    // ======== MODE_EG: gradient g = J^T F, diag, PCG init ========
    const double wrs_l = (x > 0) ? w_rs_at<double>(X, N, W, H, x - 1, y, c) : 0.0;
    const double wrs_u = (y > 0) ? w_rs_at<double>(X, N, W, H, x, y - 1, c) : 0.0;
    double gr[3], dr[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const double rs = R[ch] * S[ch];
      double g = -c.lam_d * rs * res[ch] + c.lam_cl * (r0[ch] - anc[ch]);
      double d = c.lam_d * rs * rs + c.lam_cl;
      // D^T W D r0 at x (energy.py:272-282), weights shared by channels
      if (x < W - 1) { g += wrs * (r0[ch] - (double)sy[ch][ly + kHalf][lx + kHalf + 1]); d += wrs; }
      if (x > 0)     { g += wrs_l * (r0[ch] - (double)sy[ch][ly + kHalf][lx + kHalf - 1]); d += wrs_l; }
      if (y < H - 1) { g += wrs * (r0[ch] - (double)sy[ch][ly + kHalf + 1][lx + kHalf]); d += wrs; }
      if (y > 0)     { g += wrs_u * (r0[ch] - (double)sy[ch][ly + kHalf - 1][lx + kHalf]); d += wrs_u; }
      gr[ch] = g + gcons[ch];
      dr[ch] = d + dcons;
    }
    double rz = 0.0, bb = 0.0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float bf = (float)(-gr[ch]);
      const float df = (float)dr[ch];
      const float dd = df > 0.f ? df : 1.f;
      const float uf = bf / dd;
      if (r_out) { r_out[ch * N + i] = bf; d_out[ch * N + i] = dd; u_out[ch * N + i] = uf; }
      if (b_raw) { b_raw[ch * N + i] = bf; diag_raw[ch * N + i] = df; }
      rz += (double)bf * (double)uf;
      bb += (double)bf * (double)bf;
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      double g = 0.0, d = 0.0, gm = 0.0, g2 = 0.0;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        g += R[ch] * c.B[k][ch] * res[ch];
        d += R[ch] * R[ch] * c.B[k][ch] * c.B[k][ch];
        gm += c.G[k][ch] * m[ch];
        g2 += c.G[k][ch] * c.G[k][ch];
      }
      g = -c.lam_d * g + c.lam_m * edge * gm + (wis[k] + wnn[k]) * T0[k];
      d = c.lam_d * d + c.lam_m * edge * g2 + wis[k] + wnn[k];
      const float* Tk = X + (size_t)(3 + k) * N;
      if (x < W - 1) { g += axx[k] * (T0[k] - (double)__ldg(Tk + i + 1)); d += axx[k]; }
      if (x > 0) {
        const double wl = w_smx_at<double>(Tk, W, i - 1, c);
        g += wl * (T0[k] - (double)__ldg(Tk + i - 1));
        d += wl;
      }
      if (y < H - 1) { g += ayy[k] * (T0[k] - (double)__ldg(Tk + i + W)); d += ayy[k]; }
      if (y > 0) {
        const double wu = w_smy_at<double>(Tk, W, i - W, c);
        g += wu * (T0[k] - (double)__ldg(Tk + i - W));
        d += wu;
      }
      const float bf = (float)(-g);
      const float df = (float)d;
      const float dd = df > 0.f ? df : 1.f;
      const float uf = bf / dd;
      const size_t o = (size_t)(3 + k) * N + i;
      if (r_out) { r_out[o] = bf; d_out[o] = dd; u_out[o] = uf; }
      if (b_raw) { b_raw[o] = bf; diag_raw[o] = df; }
      rz += (double)bf * (double)uf;
      bb += (double)bf * (double)bf;
    }
    if (MODE == MODE_EG) {
      acc[kTerms] += rz;
      acc[kTerms + 1] += bb;
    }
  }

  block_reduce_store<NV>(acc, part);
  if (!last_block(ticket)) return;
  double tot[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) tot[j] = sum_partials<NV>(part, gridDim.x, j);
  if (threadIdx.x == 0) {
    bool finite = true;
    for (int j = 0; j < kTerms; ++j) finite = finite && isfinite(tot[j]);
    if (MODE == MODE_EG) {
      for (int j = 0; j < kTerms; ++j) sc->terms0[j] = tot[j];
      sc->gamma = tot[kTerms];
      sc->gamma_prev = 0.0;
      sc->bnorm2 = tot[kTerms + 1];
      sc->rnorm2 = tot[kTerms + 1];
      sc->alpha = sc->alpha_prev = sc->beta = sc->delta = 0.0;
      sc->iterations = 0;
      // zero rhs -> x = 0 (solver.py:85-86); non-finite -> host raises
      sc->stop = (!finite || tot[kTerms + 1] == 0.0 || r_out == nullptr) ? 1 : 0;
    } else {
      for (int j = 0; j < kTerms; ++j) sc->terms1[j] = tot[j];
    }
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------
// matrix-free normal operator w = J^T J u (fp32), frozen at X
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(kThreads) k_apply(Frame f, Coef<float> c, const float* __restrict__ X,
                                                    const float* __restrict__ u, float* __restrict__ w,
                                                    double* part, unsigned* ticket, Scalars* sc,
                                                    int iter, int ntiles) {
  __shared__ float su[3][kHaloH][kHaloW];
  if (sc && sc->stop) return;
  const int W = f.W, H = f.H, N = f.N;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  double acc[1] = {0.0};
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int tx0, ty0;
    tile_coords(tile, W, tx0, ty0);
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * kHaloH * kHaloW; e += kThreads) {
      const int ch = e / (kHaloH * kHaloW), rem = e % (kHaloH * kHaloW);
      const int yy = rem / kHaloW, xx = rem % kHaloW;
      const int gy = ty0 + yy - kHalf, gx = tx0 + xx - kHalf;
      su[ch][yy][xx] = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? __ldg(u + ch * N + gy * W + gx) : 0.f;
    }
    __syncthreads();
    const int x = tx0 + lx, y = ty0 + ly;
    if (x >= W || y >= H) continue;
    const int i = y * W + x;

    float ur[3], uT[NT], R0[3], S0[3], T0[NT];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      ur[ch] = su[ch][ly + kHalf][lx + kHalf];
      R0[ch] = expf(__ldg(X + ch * N + i));
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      uT[k] = __ldg(u + (size_t)(3 + k) * N + i);
      T0[k] = __ldg(X + (size_t)(3 + k) * N + i);
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < NT; ++k) s = fmaf(T0[k], c.B[k][ch], s);
      S0[ch] = s;
    }
    // data rows: rho_c = R0 (S0 u_r + sum_k b_kc u_Tk)   (energy.py:211-218)
    float rho[3], outr[3], outT[NT];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < NT; ++k) s = fmaf(uT[k], c.B[k][ch], s);
      rho[ch] = R0[ch] * fmaf(S0[ch], ur[ch], s);
      outr[ch] = c.lam_d * R0[ch] * S0[ch] * rho[ch] + c.lam_cl * ur[ch];
    }
    // monochrome: q_c = sum_k G_kc u_Tk  (energy.py:403-408)
    float q[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < NT; ++k) s = fmaf(uT[k], c.G[k][ch], s);
      q[ch] = s * c.lam_m * __ldg(f.edge + i);
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      float s = 0.f, m = 0.f;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        s = fmaf(R0[ch] * c.B[k][ch], rho[ch], s);
        m = fmaf(c.G[k][ch], q[ch], m);
      }
      const float wis = (k >= 1) ? c.lam_is * irls1<float>(T0[k], c.eps_irls, c.inv_eps) : 0.f;
      const float wnn = c.lam_nn * nonneg_w<float>(T0[k], c.eps_nn);
      outT[k] = c.lam_d * s + m + (wis + wnn) * uT[k];
    }
    // r-sparsity: D^T W D u_r
    {
      const float wrs = w_rs_at<float>(X, N, W, H, x, y, c);
      const float wl = (x > 0) ? w_rs_at<float>(X, N, W, H, x - 1, y, c) : 0.f;
      const float wu = (y > 0) ? w_rs_at<float>(X, N, W, H, x, y - 1, c) : 0.f;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float v = ur[ch];
        float a = 0.f;
        if (x < W - 1) a += wrs * (v - su[ch][ly + kHalf][lx + kHalf + 1]);
        if (x > 0)     a += wl * (v - su[ch][ly + kHalf][lx + kHalf - 1]);
        if (y < H - 1) a += wrs * (v - su[ch][ly + kHalf + 1][lx + kHalf]);
        if (y > 0)     a += wu * (v - su[ch][ly + kHalf - 1][lx + kHalf]);
        outr[ch] += a;
      }
    }
    // smoothness: per layer D^T W_k D u_Tk
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const float* Tk = X + (size_t)(3 + k) * N;
      const float* uk = u + (size_t)(3 + k) * N;
      float a = 0.f;
      if (x < W - 1) a += w_smx_at<float>(Tk, W, i, c) * (uT[k] - __ldg(uk + i + 1));
      if (x > 0)     a += w_smx_at<float>(Tk, W, i - 1, c) * (uT[k] - __ldg(uk + i - 1));
      if (y < H - 1) a += w_smy_at<float>(Tk, W, i, c) * (uT[k] - __ldg(uk + i + W));
      if (y > 0)     a += w_smy_at<float>(Tk, W, i - W, c) * (uT[k] - __ldg(uk + i - W));
      outT[k] += a;
    }
    // consistency graph Laplacian (energy.py:352-370): spatial pairs couple
    // u(x) - u(q); temporal partners are constant (energy.py:356)
    {
      const int e0 = __ldg(f.row_ptr + i), e1 = __ldg(f.row_ptr + i + 1);
      float a0 = 0.f, a1 = 0.f, a2 = 0.f;
      for (int e = e0; e < e1; ++e) {
        const uint16_t ent = __ldg(f.ent + e);
        const float we = c.lam_rc * (f.ent_w ? __ldg(f.ent_w + e) : 1.f);
        if (ent & kEntTemporal) {
          a0 += we * ur[0]; a1 += we * ur[1]; a2 += we * ur[2];
        } else {
          int ddy, ddx;
          decode_offset(ent, ddy, ddx);
          a0 += we * (ur[0] - su[0][ly + kHalf + ddy][lx + kHalf + ddx]);
          a1 += we * (ur[1] - su[1][ly + kHalf + ddy][lx + kHalf + ddx]);
          a2 += we * (ur[2] - su[2][ly + kHalf + ddy][lx + kHalf + ddx]);
        }
      }
      outr[0] += a0; outr[1] += a1; outr[2] += a2;
    }
    double dot = 0.0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      w[ch * N + i] = outr[ch];
      dot += (double)outr[ch] * (double)ur[ch];
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      w[(size_t)(3 + k) * N + i] = outT[k];
      dot += (double)outT[k] * (double)uT[k];
    }
    acc[0] += dot;
  }
  if (!sc) return;
  block_reduce_store<1>(acc, part);
  if (!last_block(ticket)) return;
  const double delta = sum_partials<1>(part, gridDim.x, 0);
  if (threadIdx.x == 0) {
    // Chronopoulos-Gear: denominator == p.Ap of the textbook loop (solver.py:93-97)
    double beta = 0.0, denom = delta;
    if (iter > 0) {
      beta = sc->gamma / sc->gamma_prev;
      denom = delta - beta * sc->gamma / sc->alpha_prev;
    }
    sc->delta = delta;
    sc->beta = beta;
    if (!(denom > 0.0) || !isfinite(denom)) sc->stop = 1;
    else sc->alpha = sc->gamma / denom;
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------
// PCG vector update (pointwise, float4):  p = u + b p ; s = w + b s ;
// x += a p ; r -= a s ; u = r / d   and partials <r,u>, <r,r>
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_update(int64_t M, float* __restrict__ x, float* __restrict__ r,
                                                     float* __restrict__ p, float* __restrict__ s,
                                                     const float* __restrict__ w, const float* __restrict__ d,
                                                     float* __restrict__ u, double* part, unsigned* ticket,
                                                     Scalars* sc, int iter) {
  if (sc->stop) return;
  const float a = (float)sc->alpha, b = (float)sc->beta;
  const bool first = (iter == 0);
  double acc[2] = {0.0, 0.0};
  const int64_t M4 = M >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M4; j += stride) {
    float4 uu = reinterpret_cast<const float4*>(u)[j];
    float4 ww = __ldg(reinterpret_cast<const float4*>(w) + j);
    float4 rr = reinterpret_cast<const float4*>(r)[j];
    float4 dd = __ldg(reinterpret_cast<const float4*>(d) + j);
    float4 pp, ss, xx;
    if (first) {
      pp = uu; ss = ww;
      xx = make_float4(a * pp.x, a * pp.y, a * pp.z, a * pp.w);
    } else {
      pp = reinterpret_cast<const float4*>(p)[j];
      ss = reinterpret_cast<const float4*>(s)[j];
      xx = reinterpret_cast<const float4*>(x)[j];
      pp = make_float4(fmaf(b, pp.x, uu.x), fmaf(b, pp.y, uu.y), fmaf(b, pp.z, uu.z), fmaf(b, pp.w, uu.w));
      ss = make_float4(fmaf(b, ss.x, ww.x), fmaf(b, ss.y, ww.y), fmaf(b, ss.z, ww.z), fmaf(b, ss.w, ww.w));
      xx = make_float4(fmaf(a, pp.x, xx.x), fmaf(a, pp.y, xx.y), fmaf(a, pp.z, xx.z), fmaf(a, pp.w, xx.w));
    }
    rr = make_float4(fmaf(-a, ss.x, rr.x), fmaf(-a, ss.y, rr.y), fmaf(-a, ss.z, rr.z), fmaf(-a, ss.w, rr.w));
    uu = make_float4(rr.x / dd.x, rr.y / dd.y, rr.z / dd.z, rr.w / dd.w);
    reinterpret_cast<float4*>(p)[j] = pp;
    reinterpret_cast<float4*>(s)[j] = ss;
    reinterpret_cast<float4*>(x)[j] = xx;
    reinterpret_cast<float4*>(r)[j] = rr;
    reinterpret_cast<float4*>(u)[j] = uu;
    acc[0] += (double)rr.x * uu.x + (double)rr.y * uu.y + (double)rr.z * uu.z + (double)rr.w * uu.w;
    acc[1] += (double)rr.x * rr.x + (double)rr.y * rr.y + (double)rr.z * rr.z + (double)rr.w * rr.w;
  }
  // scalar tail (M not a multiple of 4)
  for (int64_t j = (M4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride) {
    float uu = u[j], ww = w[j], rr = r[j], dd = d[j], pp, ss, xx;
    if (first) { pp = uu; ss = ww; xx = a * pp; }
    else { pp = fmaf(b, p[j], uu); ss = fmaf(b, s[j], ww); xx = fmaf(a, pp, x[j]); }
    rr = fmaf(-a, ss, rr);
    uu = rr / dd;
    p[j] = pp; s[j] = ss; x[j] = xx; r[j] = rr; u[j] = uu;
    acc[0] += (double)rr * uu;
    acc[1] += (double)rr * rr;
  }
  block_reduce_store<2>(acc, part);
  if (!last_block(ticket)) return;
  const double g = sum_partials<2>(part, gridDim.x, 0);
  const double rn = sum_partials<2>(part, gridDim.x, 1);
  if (threadIdx.x == 0) {
    sc->iterations = iter + 1;
    sc->gamma_prev = sc->gamma;
    sc->gamma = g;
    sc->alpha_prev = sc->alpha;
    sc->rnorm2 = rn;
    if (g <= 0.0) sc->stop = 1;   // solver.py:101-103
    *ticket = 0u;
  }
}

// ---------------------------------------------------------------------------
// host-side launchers (dispatch on NT)
// ---------------------------------------------------------------------------
template <int NT>
static void launch_energy_nt(int mode, const Launch& L, const Frame& f, const Coef<double>& c,
                             const float* X, const float* dx, float alpha, float* Xout, float* r_out,
                             float* d_out, float* u_out, float* b_raw, float* diag_raw, double* part,
                             unsigned* ticket, Scalars* sc) {
  if (mode == MODE_EG)
    k_energy<NT, MODE_EG><<<L.grid, kThreads, 0, L.stream>>>(f, c, X, dx, alpha, nullptr, Xout, r_out, d_out,
                                                             u_out, b_raw, diag_raw, part, ticket, sc, L.ntiles);
  else
    k_energy<NT, MODE_TRIAL><<<L.grid, kThreads, 0, L.stream>>>(f, c, X, dx, alpha, nullptr, Xout, r_out, d_out,
                                                                u_out, b_raw, diag_raw, part, ticket, sc,
                                                                L.ntiles);
}

template <int NT>
static void launch_energy_ext_nt(const Launch& L, const Frame& f, const Coef<double>& c, const float* X,
                                 const float* Y, double* part, unsigned* ticket, Scalars* sc) {
  k_energy<NT, MODE_TRIAL><<<L.grid, kThreads, 0, L.stream>>>(f, c, X, nullptr, 0.f, Y, nullptr, nullptr, nullptr,
                                                              nullptr, nullptr, nullptr, part, ticket, sc, L.ntiles);
}

template <int NT>
static void launch_apply_nt(const Launch& L, const Frame& f, const Coef<float>& c, const float* X,
                            const float* u, float* w, double* part, unsigned* ticket, Scalars* sc, int iter) {
  k_apply<NT><<<L.grid, kThreads, 0, L.stream>>>(f, c, X, u, w, part, ticket, sc, iter, L.ntiles);
}

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

void launch_energy(int mode, const Launch& L, const Frame& f, const Coef<double>& c, const float* X,
                   const float* dx, float alpha, float* Xout, float* r_out, float* d_out, float* u_out,
                   float* b_raw, float* diag_raw, double* part, unsigned* ticket, Scalars* sc) {
  LS_DISPATCH_NT(f.NT, (launch_energy_nt<NT_>(mode, L, f, c, X, dx, alpha, Xout, r_out, d_out, u_out, b_raw,
                                              diag_raw, part, ticket, sc)));
}

void launch_energy_ext(const Launch& L, const Frame& f, const Coef<double>& c, const float* X, const float* Y,
                       double* part, unsigned* ticket, Scalars* sc) {
  LS_DISPATCH_NT(f.NT, (launch_energy_ext_nt<NT_>(L, f, c, X, Y, part, ticket, sc)));
}

void launch_apply(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* u,
                  float* w, double* part, unsigned* ticket, Scalars* sc, int iter) {
  LS_DISPATCH_NT(f.NT, (launch_apply_nt<NT_>(L, f, c, X, u, w, part, ticket, sc, iter)));
}

void launch_update(const Launch& L, int64_t M, float* x, float* r, float* p, float* s, const float* w,
                   const float* d, float* u, double* part, unsigned* ticket, Scalars* sc, int iter) {
  k_update<<<L.grid, kThreads, 0, L.stream>>>(M, x, r, p, s, w, d, u, part, ticket, sc, iter);
}

int energy_grid_limit(int NT) {
  int nb = 0;
  LS_DISPATCH_NT(NT, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_energy<NT_, MODE_EG>, kThreads, 0)));
  return nb;
}
int apply_grid_limit(int NT) {
  int nb = 0;
  LS_DISPATCH_NT(NT, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_apply<NT_>, kThreads, 0)));
  return nb;
}
int update_grid_limit() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_update, kThreads, 0);
  return nb;
}

}  // namespace ls
