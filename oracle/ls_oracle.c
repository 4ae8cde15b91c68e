/*
 * ls_oracle.c -- compiled CPU restatement of the reference solver.
 *
 * TEST / MEASUREMENT INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_1908_01961_b200/) links or loads this file's library; it is used by
 * tests/ (as the checker at sizes the NumPy oracle is too slow for, e.g. the
 * 1920x1080 K=8 headline configuration) and by bench.py's cpu_baseline leg
 * and `--impl reference` arm (as the CPU implementation of the path, timed
 * on the host cores).
 *
 * It restates, in fp64 C with OpenMP over image rows, the same per-pixel
 * normal-equation form as oracle/lumisplit_oracle.py, which follows the
 * reference package lumisplit (/root/reference/pkg/src/lumisplit) and is
 * pinned to the reference's own outputs by tests/golden (tools/make_golden.py).
 * This file is pinned the same way: tests/test_oracle_c.py checks it against
 * every golden fixture and against the NumPy oracle.
 *
 * Layouts follow the reference: image / r are (H, W, 3), T is (H, W, K+1)
 * interleaved fp64, the PCG vector is [r.ravel(), T.ravel()]
 * (solver.py:110-122).  Reductions are accumulated per image row and the row
 * sums added in row order, so results do not depend on the thread count.
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NTERMS 8
#define MAXNT 13
enum { T_DATA, T_CLUSTER, T_RSPARSE, T_CONSIST, T_MONO, T_ISPARSE, T_SMOOTH, T_NONNEG };

/* energy.py:28-56 (EnergyWeights), chroma_reg 0 = projection, 1 = identity */
typedef struct {
  double lam_d, lam_cl, lam_rs, p, lam_rc, lam_m, lam_is, lam_sm, lam_nn, lam_ir, lam_cr, eps_nn, eps_irls;
  int chroma_reg;
} or_weights;

/* solver.py:32-49 (SolveConfig) */
typedef struct {
  int outer_iterations, gn_steps, pcg_iterations, max_halvings, refine, refine_warmup;
  double tol_rel, svd_truncation, max_delta_b, refine_gate_rel;
} or_config;

/* one record of solver.py:180-188 (sparse) / 245-252 (dense) */
typedef struct {
  int phase; /* 0 sparse, 1 dense */
  int accepted, pcg_iterations, pad;
  double energy_before, energy_after, alpha, initial_residual, final_residual, delta_b_norm;
  double terms[NTERMS];
} or_record;

typedef struct {
  int H, W, K, NT, N;
  or_weights w;
  const double* img; /* N*3 */
  double colors[3 * (MAXNT - 1)];
  double B[MAXNT][3], G[MAXNT][3];
  const double* edge; /* N */
  const int32_t* ids; /* N or NULL */
  double* anchor;     /* N*3 */
  const double* anchor_fixed;
  /* partner rows (energy.py:139-151) and their incidence lists */
  int64_t P;
  int32_t *src, *dst;
  uint8_t* tmp;
  double* pw; /* lambda_rc * weight */
  int64_t *out_ptr, *in_ptr;
  int32_t *out_idx, *in_idx;
  const double* prev_r; /* N*3 or NULL */
  int temporal_without_prev;
  /* linearisation point and frozen weights (energy.py:478-496) */
  double *r0, *T0, *R0, *S0, *w_rs, *w_smx, *w_smy, *w_is, *w_nn;
  double* rowbuf; /* H * 16 */
} or_sys;

/* ------------------------------------------------------------------------ */
/* helpers                                                                   */
/* ------------------------------------------------------------------------ */

/* energy.py:102-112 */
static inline double irls(double m, double p, double eps) {
  m = fabs(m);
  if (p >= 2.0) return 1.0;
  if (p == 1.0) return m >= eps ? 1.0 / m : 1.0 / eps;
  const double floor_ = pow(eps, 1.0 / (2.0 - p));
  return m >= floor_ ? pow(m, p - 2.0) : 1.0 / eps;
}

/* energy.py:115-118 */
static inline double nonneg_w(double t, double eps) { return t > 0.0 ? 0.0 : 1.0 / (fabs(t) + eps); }

static double sum_rows(const double* rows, int H, int stride, int j) {
  double s = 0.0;
  for (int y = 0; y < H; ++y) s += rows[(size_t)y * stride + j];
  return s;
}

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* per-frame auxiliary context                                              */
/* ------------------------------------------------------------------------ */

/* imaging.py:160-171: chroma (N*2), dark (N) */
void or_chromaticity(int H, int W, const double* img, double* chroma, uint8_t* dark) {
  const int64_t N = (int64_t)H * W;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    const double s = (img[3 * i] + img[3 * i + 1]) + img[3 * i + 2];
    const int d = s < 0.02;
    const double den = d ? 1.0 : s;
    chroma[2 * i] = d ? 1.0 / 3.0 : img[3 * i] / den;
    chroma[2 * i + 1] = d ? 1.0 / 3.0 : img[3 * i + 1] / den;
    if (dark) dark[i] = (uint8_t)d;
  }
}

/* energy.py:121-136 */
void or_edge_gate(int H, int W, const double* chroma, double* edge) {
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const int64_t i = (int64_t)y * W + x;
      double m = 0.0;
      const int nb[4][2] = {{0, 1}, {0, -1}, {1, 0}, {-1, 0}};
      for (int k = 0; k < 4; ++k) {
        const int yy = y + nb[k][0], xx = x + nb[k][1];
        if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
        const int64_t j = (int64_t)yy * W + xx;
        const double a = chroma[2 * j] - chroma[2 * i], b = chroma[2 * j + 1] - chroma[2 * i + 1];
        const double d = sqrt(a * a + b * b);
        if (d > m) m = d;
      }
      edge[i] = 1.0 - exp(-50.0 * m);
    }
}

/* numpy PCG64 (XSL-RR 128/64; the state steps before each output) */
typedef unsigned __int128 u128;
static inline uint64_t pcg64_next(u128* s, u128 inc) {
  const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  *s = *s * mult + inc;
  const unsigned rot = (unsigned)(*s >> 122);
  const uint64_t x = (uint64_t)(*s >> 64) ^ (uint64_t)*s;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

typedef struct {
  u128 s, inc;
  int bcnt;
  uint64_t buf;
} rng32;

/* numpy buffered_uint32: low half of a 64-bit output first */
static inline uint32_t next32(rng32* g) {
  if (!g->bcnt) {
    g->buf = pcg64_next(&g->s, g->inc);
    g->bcnt = 1;
  } else {
    g->buf >>= 32;
    g->bcnt = 0;
  }
  return (uint32_t)g->buf;
}

/* numpy buffered_bounded_lemire_uint32 for [0, rng] */
static inline uint32_t lemire(rng32* g, uint32_t rng) {
  const uint32_t excl = rng + 1;
  uint64_t m = (uint64_t)next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      m = (uint64_t)next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

/* energy.py:154-187 with Generator.integers as numpy runs it (each
 * `integers` call starts a fresh 32-bit buffer).  The draws are sequential;
 * the chroma gate runs in parallel.  Returns the number of kept rows; src,
 * dst (int64) and temporal need room for 4N rows. */
int64_t or_sample_consistency(int H, int W, const double* chroma, const double* prev_chroma, uint64_t st_hi,
                              uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t* src, int64_t* dst,
                              uint8_t* temporal) {
  const int64_t N = (int64_t)H * W, M = 4 * N;
  if (N <= 0) return 0;
  int8_t* d = (int8_t*)malloc((size_t)(3 * M));
  rng32 g = {((u128)st_hi << 64) | st_lo, ((u128)inc_hi << 64) | inc_lo, 0, 0};
  for (int64_t j = 0; j < M; ++j) d[j] = (int8_t)((int)lemire(&g, 14) - 7);
  g.bcnt = 0;
  for (int64_t j = 0; j < M; ++j) d[M + j] = (int8_t)((int)lemire(&g, 14) - 7);
  g.bcnt = 0;
  if (prev_chroma)
    for (int64_t j = 0; j < M; ++j) d[2 * M + j] = (int8_t)lemire(&g, 1);
  else
    memset(d + 2 * M, 0, (size_t)M);
  uint8_t* keep = (uint8_t*)malloc((size_t)M);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < M; ++j) {
    const int64_t s = j >> 2;
    const int y = (int)(s / W), x = (int)(s % W);
    int px = x + d[j], py = y + d[M + j];
    px = px < 0 ? 0 : (px > W - 1 ? W - 1 : px);
    py = py < 0 ? 0 : (py > H - 1 ? H - 1 : py);
    const int64_t t = (int64_t)py * W + px;
    const int tm = d[2 * M + j] != 0;
    const double* pc = tm ? prev_chroma : chroma;
    const double a = chroma[2 * s] - pc[2 * t], b = chroma[2 * s + 1] - pc[2 * t + 1];
    keep[j] = (uint8_t)(sqrt(a * a + b * b) < 0.05 && (tm || s != t));
    if (keep[j]) {
      dst[j] = t;
      temporal[j] = (uint8_t)tm;
    }
  }
  int64_t n = 0;
  for (int64_t j = 0; j < M; ++j)
    if (keep[j]) {
      src[n] = j >> 2;
      dst[n] = dst[j];
      temporal[n] = temporal[j];
      ++n;
    }
  free(keep);
  free(d);
  return n;
}

/* imaging.py:174-180 */
static void chroma_of_color(const double* c, double* out) {
  const double t = (c[0] + c[1]) + c[2];
  if (t > 1e-12) {
    out[0] = c[0] / t;
    out[1] = c[1] / t;
  } else {
    out[0] = out[1] = 1.0 / 3.0;
  }
}

/* palette.py:195-224 -> ids in 1..K */
void or_segment(int H, int W, const double* img, int K, const double* colors, int32_t* ids) {
  const int64_t N = (int64_t)H * W;
  double cc[MAXNT][2];
  for (int k = 0; k < K; ++k) chroma_of_color(colors + 3 * k, cc[k]);
  uint8_t* dark = (uint8_t*)malloc((size_t)N);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    const double s = (img[3 * i] + img[3 * i + 1]) + img[3 * i + 2];
    const int dk = s < 0.02;
    const double den = dk ? 1.0 : s;
    const double c0 = dk ? 1.0 / 3.0 : img[3 * i] / den, c1 = dk ? 1.0 / 3.0 : img[3 * i + 1] / den;
    int best = 0;
    double bd = 0.0;
    for (int k = 0; k < K; ++k) {
      const double a = c0 - cc[k][0], b = c1 - cc[k][1];
      const double d = sqrt(a * a + b * b);
      if (k == 0 || d < bd) {
        bd = d;
        best = k;
      }
    }
    ids[i] = best + 1;
    dark[i] = (uint8_t)dk;
  }
  int64_t first = -1;
  for (int64_t i = 0; i < N; ++i)
    if (!dark[i]) {
      first = i;
      break;
    }
  if (first < 0) {
    for (int64_t i = 0; i < N; ++i) ids[i] = 1;
  } else {
    int32_t last = ids[first];
    for (int64_t i = 0; i < N; ++i) {
      if (dark[i]) ids[i] = last;
      else last = ids[i];
    }
  }
  free(dark);
}

/* solver.py:295-308, first frame: r = ln max(R_cluster, 1e-4),
 * T0 = clip(mean_c I / max(R_cluster, 1e-4), 0, 2), T_k>=1 = 0 */
void or_initialize(int H, int W, int K, const double* img, const int32_t* ids, const double* colors, double* r,
                   double* T) {
  const int64_t N = (int64_t)H * W;
  const int NT = K + 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    const double* rc = colors + 3 * (ids[i] - 1);
    double m = 0.0;
    for (int c = 0; c < 3; ++c) {
      r[3 * i + c] = log(rc[c] > 1e-4 ? rc[c] : 1e-4);
      m += img[3 * i + c] / (rc[c] > 1e-4 ? rc[c] : 1e-4);
    }
    m /= 3.0;
    T[NT * i] = m < 0.0 ? 0.0 : (m > 2.0 ? 2.0 : m);
    for (int k = 1; k < NT; ++k) T[NT * i + k] = 0.0;
  }
}

/* ------------------------------------------------------------------------ */
/* the frozen system (energy.py:194-511, solver.py:110-140)                  */
/* ------------------------------------------------------------------------ */

void or_sys_set_colors(or_sys* s, const double* colors) {
  const int K = s->K;
  for (int i = 0; i < 3 * K; ++i) s->colors[i] = colors[i];
  for (int k = 0; k <= K; ++k) {
    for (int c = 0; c < 3; ++c) s->B[k][c] = k == 0 ? 1.0 : colors[3 * (k - 1) + c];
    const double mean = (s->B[k][0] + s->B[k][1] + s->B[k][2]) / 3.0;
    for (int c = 0; c < 3; ++c) s->G[k][c] = s->B[k][c] - mean;   /* energy.py:396 */
  }
  if (s->ids) { /* anchor follows the palette (energy.py:470-472) */
    const int64_t N = s->N;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i)
      for (int c = 0; c < 3; ++c) {
        const double b = colors[3 * (s->ids[i] - 1) + c];
        s->anchor[3 * i + c] = log(b > 1e-4 ? b : 1e-4);
      }
  }
}

or_sys* or_sys_create(int H, int W, int K, const or_weights* w, const double* img, const double* colors,
                      const double* edge, int64_t P, const int64_t* src, const int64_t* dst,
                      const uint8_t* temporal, const double* weight, const double* prev_r, const int32_t* ids,
                      const double* anchor) {
  if (K + 1 > MAXNT || (!ids && !anchor)) return NULL;
  or_sys* s = (or_sys*)calloc(1, sizeof(or_sys));
  const int64_t N = (int64_t)H * W;
  const int NT = K + 1;
  s->H = H;
  s->W = W;
  s->K = K;
  s->NT = NT;
  s->N = (int)N;
  s->w = *w;
  s->img = img;
  s->edge = edge;
  s->ids = ids;
  s->prev_r = prev_r;
  s->anchor = (double*)malloc(sizeof(double) * 3 * N);
  if (!ids) memcpy(s->anchor, anchor, sizeof(double) * 3 * N);
  or_sys_set_colors(s, colors);
  s->P = P;
  s->src = (int32_t*)malloc(sizeof(int32_t) * (P + 1));
  s->dst = (int32_t*)malloc(sizeof(int32_t) * (P + 1));
  s->tmp = (uint8_t*)malloc((size_t)P + 1);
  s->pw = (double*)malloc(sizeof(double) * (P + 1));
  for (int64_t j = 0; j < P; ++j) {
    s->src[j] = (int32_t)src[j];
    s->dst[j] = (int32_t)dst[j];
    s->tmp[j] = temporal ? temporal[j] : 0;
    s->pw[j] = w->lam_rc * (weight ? weight[j] : 1.0);
    if (s->tmp[j] && !prev_r) s->temporal_without_prev = 1;
  }
  /* incidence lists in pair order: out = pairs with src == x; in = spatial
   * pairs with dst == x (np.bincount's accumulation order, energy.py:359-381) */
  s->out_ptr = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
  s->in_ptr = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
  for (int64_t j = 0; j < P; ++j) {
    s->out_ptr[s->src[j] + 1]++;
    if (!s->tmp[j]) s->in_ptr[s->dst[j] + 1]++;
  }
  for (int64_t i = 0; i < N; ++i) {
    s->out_ptr[i + 1] += s->out_ptr[i];
    s->in_ptr[i + 1] += s->in_ptr[i];
  }
  s->out_idx = (int32_t*)malloc(sizeof(int32_t) * (s->out_ptr[N] + 1));
  s->in_idx = (int32_t*)malloc(sizeof(int32_t) * (s->in_ptr[N] + 1));
  int64_t* fo = (int64_t*)malloc(sizeof(int64_t) * N);
  int64_t* fi = (int64_t*)malloc(sizeof(int64_t) * N);
  memcpy(fo, s->out_ptr, sizeof(int64_t) * N);
  memcpy(fi, s->in_ptr, sizeof(int64_t) * N);
  for (int64_t j = 0; j < P; ++j) {
    s->out_idx[fo[s->src[j]]++] = (int32_t)j;
    if (!s->tmp[j]) s->in_idx[fi[s->dst[j]]++] = (int32_t)j;
  }
  free(fo);
  free(fi);
  s->r0 = (double*)malloc(sizeof(double) * 3 * N);
  s->T0 = (double*)malloc(sizeof(double) * NT * N);
  s->R0 = (double*)malloc(sizeof(double) * 3 * N);
  s->S0 = (double*)malloc(sizeof(double) * 3 * N);
  s->w_rs = (double*)malloc(sizeof(double) * N);
  s->w_smx = (double*)malloc(sizeof(double) * NT * N);
  s->w_smy = (double*)malloc(sizeof(double) * NT * N);
  s->w_is = (double*)malloc(sizeof(double) * NT * N);
  s->w_nn = (double*)malloc(sizeof(double) * NT * N);
  s->rowbuf = (double*)malloc(sizeof(double) * 16 * H);
  return s;
}

void or_sys_free(or_sys* s) {
  if (!s) return;
  void* ps[] = {s->anchor, s->src, s->dst, s->tmp, s->pw, s->out_ptr, s->in_ptr, s->out_idx, s->in_idx,
                s->r0, s->T0, s->R0, s->S0, s->w_rs, s->w_smx, s->w_smy, s->w_is, s->w_nn, s->rowbuf};
  for (size_t i = 0; i < sizeof(ps) / sizeof(ps[0]); ++i) free(ps[i]);
  free(s);
}

/* assemble_blocks at (r0, T0): linearisation and IRLS weights frozen
 * (energy.py:478-496, 207-218, 301-305, 314-318, 438-452) */
void or_linearize(or_sys* s, const double* r, const double* T) {
  const int H = s->H, W = s->W, NT = s->NT;
  const int64_t N = s->N;
  const or_weights* w = &s->w;
  memcpy(s->r0, r, sizeof(double) * 3 * N);
  memcpy(s->T0, T, sizeof(double) * NT * N);
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const int64_t i = (int64_t)y * W + x;
      double sq = 0.0;
      for (int c = 0; c < 3; ++c) {
        s->R0[3 * i + c] = exp(r[3 * i + c]);
        double S = 0.0;
        for (int k = 0; k < NT; ++k) S += T[NT * i + k] * s->B[k][c];
        s->S0[3 * i + c] = S;
      }
      double gx2 = 0.0, gy2 = 0.0;
      for (int c = 0; c < 3; ++c) {
        const double gx = x < W - 1 ? r[3 * (i + 1) + c] - r[3 * i + c] : 0.0;
        const double gy = y < H - 1 ? r[3 * (i + W) + c] - r[3 * i + c] : 0.0;
        gx2 += gx * gx;
        gy2 += gy * gy;
      }
      sq = gx2 + gy2;
      s->w_rs[i] = w->lam_rs * irls(sqrt(sq), w->p, w->eps_irls);
      for (int k = 0; k < NT; ++k) {
        const double t = T[NT * i + k];
        const double tx = x < W - 1 ? T[NT * (i + 1) + k] - t : 0.0;
        const double ty = y < H - 1 ? T[NT * (i + W) + k] - t : 0.0;
        s->w_smx[NT * i + k] = w->lam_sm * irls(tx, 1.0, w->eps_irls);
        s->w_smy[NT * i + k] = w->lam_sm * irls(ty, 1.0, w->eps_irls);
        s->w_is[NT * i + k] = k >= 1 ? w->lam_is * irls(t, 1.0, w->eps_irls) : 0.0;
        s->w_nn[NT * i + k] = w->lam_nn * nonneg_w(t, w->eps_nn);
      }
    }
}

/* consistency partner value of pair j for state r (energy.py:348-357) */
static inline const double* partner(const or_sys* s, const double* r, int64_t j) {
  return s->tmp[j] ? s->prev_r + 3 * (int64_t)s->dst[j] : r + 3 * (int64_t)s->dst[j];
}

/* block_energies at (r, T) with the frozen weights (energy.py:503-504) */
int or_terms(or_sys* s, const double* r, const double* T, double* out) {
  double Bl[MAXNT][3], Gl[MAXNT][3];
  memcpy(Bl, s->B, sizeof(Bl));
  memcpy(Gl, s->G, sizeof(Gl));
  const double* restrict img = s->img;
  const double* restrict edge = s->edge;
  const double* restrict anchor = s->anchor;
  const double* restrict R0a = s->R0;
  const double* restrict S0a = s->S0;
  const double* restrict w_rs = s->w_rs;
  const double* restrict w_smx = s->w_smx;
  const double* restrict w_smy = s->w_smy;
  const double* restrict w_is = s->w_is;
  const double* restrict w_nn = s->w_nn;
  const double* restrict pw = s->pw;
  const int64_t* restrict out_ptr = s->out_ptr;
  const int64_t* restrict in_ptr = s->in_ptr;
  const int32_t* restrict out_idx = s->out_idx;
  const int32_t* restrict in_idx = s->in_idx;
  const int32_t* restrict srcv = s->src;
  const int32_t* restrict dstv = s->dst;
  const uint8_t* restrict tmpv = s->tmp;
  (void)img; (void)edge; (void)anchor; (void)R0a; (void)S0a; (void)w_rs; (void)w_smx; (void)w_smy;
  (void)w_is; (void)w_nn; (void)pw; (void)out_ptr; (void)in_ptr; (void)out_idx; (void)in_idx;
  (void)srcv; (void)dstv; (void)tmpv; (void)Gl;
  const int H = s->H, W = s->W, NT = s->NT;
  const or_weights* w = &s->w;
  if (s->temporal_without_prev) return 2; /* energy.py:335-336 */
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y) {
    double e[NTERMS] = {0};
    for (int x = 0; x < W; ++x) {
      const int64_t i = (int64_t)y * W + x;
      double S[3];
      for (int c = 0; c < 3; ++c) {
        double v = 0.0;
        for (int k = 0; k < NT; ++k) v += T[NT * i + k] * Bl[k][c];
        S[c] = v;
        const double res = img[3 * i + c] - exp(r[3 * i + c]) * v;
        e[T_DATA] += res * res;
        const double dc = r[3 * i + c] - anchor[3 * i + c];
        e[T_CLUSTER] += dc * dc;
        const double gx = x < W - 1 ? r[3 * (i + 1) + c] - r[3 * i + c] : 0.0;
        const double gy = y < H - 1 ? r[3 * (i + W) + c] - r[3 * i + c] : 0.0;
        e[T_RSPARSE] += w_rs[i] * (gx * gx + gy * gy);
      }
      const double mean = (S[0] + S[1] + S[2]) / 3.0;
      double m2 = 0.0;
      for (int c = 0; c < 3; ++c) m2 += (S[c] - mean) * (S[c] - mean);
      e[T_MONO] += w->lam_m * edge[i] * m2;
      for (int k = 0; k < NT; ++k) {
        const double t = T[NT * i + k];
        if (k >= 1) e[T_ISPARSE] += w_is[NT * i + k] * t * t;
        const double tx = x < W - 1 ? T[NT * (i + 1) + k] - t : 0.0;
        const double ty = y < H - 1 ? T[NT * (i + W) + k] - t : 0.0;
        e[T_SMOOTH] += w_smx[NT * i + k] * tx * tx + w_smy[NT * i + k] * ty * ty;
        e[T_NONNEG] += w_nn[NT * i + k] * t * t;
      }
      for (int64_t q = out_ptr[i]; q < out_ptr[i + 1]; ++q) {
        const int64_t j = out_idx[q];
        const double* pp = partner(s, r, j);
        double d2 = 0.0;
        for (int c = 0; c < 3; ++c) d2 += (r[3 * i + c] - pp[c]) * (r[3 * i + c] - pp[c]);
        e[T_CONSIST] += pw[j] * d2;
      }
    }
    e[T_DATA] *= w->lam_d;
    e[T_CLUSTER] *= w->lam_cl;
    for (int t = 0; t < NTERMS; ++t) s->rowbuf[16 * y + t] = e[t];
  }
  for (int t = 0; t < NTERMS; ++t) out[t] = sum_rows(s->rowbuf, H, 16, t);
  return 0;
}

static double energy_sum(const double* t) {
  double e = 0.0; /* Python sum() over the block order (solver.py:139-140) */
  for (int j = 0; j < NTERMS; ++j) e += t[j];
  return e;
}

/* b = -J^T F and diag(J^T J) at the linearisation point (solver.py:125-136) */
void or_grad_diag(or_sys* s, double* restrict b, double* restrict diag) {
  double Bl[MAXNT][3], Gl[MAXNT][3];
  memcpy(Bl, s->B, sizeof(Bl));
  memcpy(Gl, s->G, sizeof(Gl));
  const double* restrict img = s->img;
  const double* restrict edge = s->edge;
  const double* restrict anchor = s->anchor;
  const double* restrict R0a = s->R0;
  const double* restrict S0a = s->S0;
  const double* restrict w_rs = s->w_rs;
  const double* restrict w_smx = s->w_smx;
  const double* restrict w_smy = s->w_smy;
  const double* restrict w_is = s->w_is;
  const double* restrict w_nn = s->w_nn;
  const double* restrict pw = s->pw;
  const int64_t* restrict out_ptr = s->out_ptr;
  const int64_t* restrict in_ptr = s->in_ptr;
  const int32_t* restrict out_idx = s->out_idx;
  const int32_t* restrict in_idx = s->in_idx;
  const int32_t* restrict srcv = s->src;
  const int32_t* restrict dstv = s->dst;
  const uint8_t* restrict tmpv = s->tmp;
  (void)img; (void)edge; (void)anchor; (void)R0a; (void)S0a; (void)w_rs; (void)w_smx; (void)w_smy;
  (void)w_is; (void)w_nn; (void)pw; (void)out_ptr; (void)in_ptr; (void)out_idx; (void)in_idx;
  (void)srcv; (void)dstv; (void)tmpv; (void)Gl;
  const int H = s->H, W = s->W, NT = s->NT;
  const int64_t N = s->N;
  const or_weights* w = &s->w;
  const double *r0 = s->r0, *T0 = s->T0;
  double* bT = b + 3 * N;
  double* dT = diag + 3 * N;
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const int64_t i = (int64_t)y * W + x;
      const double *R0 = R0a + 3 * i, *S0 = S0a + 3 * i;
      double res[3], m[3];
      for (int c = 0; c < 3; ++c) res[c] = img[3 * i + c] - R0[c] * S0[c];
      const double mean = (S0[0] + S0[1] + S0[2]) / 3.0;
      for (int c = 0; c < 3; ++c) m[c] = S0[c] - mean;
      const double wm = w->lam_m * edge[i];
      /* r rows: data, clustering, r-sparsity (D^T W D r), consistency */
      double cons_o[3] = {0, 0, 0}, cons_i[3] = {0, 0, 0}, cnt_o = 0.0, cnt_i = 0.0;
      for (int64_t q = out_ptr[i]; q < out_ptr[i + 1]; ++q) {
        const int64_t j = out_idx[q];
        const double* pp = partner(s, r0, j);
        for (int c = 0; c < 3; ++c) cons_o[c] += pw[j] * (r0[3 * i + c] - pp[c]);
        cnt_o += pw[j];
      }
      for (int64_t q = in_ptr[i]; q < in_ptr[i + 1]; ++q) {
        const int64_t j = in_idx[q];
        const int64_t a = srcv[j];
        for (int c = 0; c < 3; ++c) cons_i[c] += pw[j] * (r0[3 * a + c] - r0[3 * i + c]);
        cnt_i += pw[j];
      }
      const double wc = w_rs[i];
      const double wl = x > 0 ? w_rs[i - 1] : 0.0, wu = y > 0 ? w_rs[i - W] : 0.0;
      for (int c = 0; c < 3; ++c) {
        const double v = r0[3 * i + c];
        double g = -w->lam_d * R0[c] * S0[c] * res[c];
        g += w->lam_cl * (v - anchor[3 * i + c]);
        double dv = 0.0; /* div_adjoint(w gx, w gy) */
        if (x > 0) dv += wl * (v - r0[3 * (i - 1) + c]);
        if (x < W - 1) dv -= wc * (r0[3 * (i + 1) + c] - v);
        if (y > 0) dv += wu * (v - r0[3 * (i - W) + c]);
        if (y < H - 1) dv -= wc * (r0[3 * (i + W) + c] - v);
        g += dv;
        g += cons_o[c] - cons_i[c];
        b[3 * i + c] = -g;
        double d = w->lam_d * (R0[c] * S0[c]) * (R0[c] * S0[c]) + w->lam_cl;
        d += (x < W - 1 ? wc : 0.0) + wl + (y < H - 1 ? wc : 0.0) + wu;
        d += cnt_o + cnt_i;
        diag[3 * i + c] = d;
      }
      /* T rows: data, monochrome, i-sparsity, smoothness, non-negativity */
      for (int k = 0; k < NT; ++k) {
        const int64_t o = NT * i + k;
        const double v = T0[o];
        double g = 0.0, d = 0.0, g2 = 0.0;
        for (int c = 0; c < 3; ++c) {
          g += -w->lam_d * R0[c] * res[c] * Bl[k][c];
          d += w->lam_d * R0[c] * R0[c] * Bl[k][c] * Bl[k][c];
          g2 += Gl[k][c] * Gl[k][c];
        }
        double gm = 0.0;
        for (int c = 0; c < 3; ++c) gm += wm * m[c] * Gl[k][c];
        g += gm;
        d += wm * g2;
        if (k >= 1) {
          g += w_is[o] * v;
          d += w_is[o];
        }
        const double ax = w_smx[o], ay = w_smy[o];
        const double al = x > 0 ? w_smx[o - NT] : 0.0, au = y > 0 ? w_smy[o - (int64_t)NT * W] : 0.0;
        double dv = 0.0;
        if (x > 0) dv += al * (v - T0[o - NT]);
        if (x < W - 1) dv -= ax * (T0[o + NT] - v);
        if (y > 0) dv += au * (v - T0[o - (int64_t)NT * W]);
        if (y < H - 1) dv -= ay * (T0[o + (int64_t)NT * W] - v);
        g += dv;
        d += (x < W - 1 ? ax : 0.0) + al + (y < H - 1 ? ay : 0.0) + au;
        g += w_nn[o] * v;
        d += w_nn[o];
        bT[o] = -g;
        dT[o] = d;
      }
    }
}

/* J^T J p (solver.py:110-122), matrix-free */
void or_apply(or_sys* s, const double* restrict p, double* restrict Ap) {
  double Bl[MAXNT][3], Gl[MAXNT][3];
  memcpy(Bl, s->B, sizeof(Bl));
  memcpy(Gl, s->G, sizeof(Gl));
  const double* restrict img = s->img;
  const double* restrict edge = s->edge;
  const double* restrict anchor = s->anchor;
  const double* restrict R0a = s->R0;
  const double* restrict S0a = s->S0;
  const double* restrict w_rs = s->w_rs;
  const double* restrict w_smx = s->w_smx;
  const double* restrict w_smy = s->w_smy;
  const double* restrict w_is = s->w_is;
  const double* restrict w_nn = s->w_nn;
  const double* restrict pw = s->pw;
  const int64_t* restrict out_ptr = s->out_ptr;
  const int64_t* restrict in_ptr = s->in_ptr;
  const int32_t* restrict out_idx = s->out_idx;
  const int32_t* restrict in_idx = s->in_idx;
  const int32_t* restrict srcv = s->src;
  const int32_t* restrict dstv = s->dst;
  const uint8_t* restrict tmpv = s->tmp;
  (void)img; (void)edge; (void)anchor; (void)R0a; (void)S0a; (void)w_rs; (void)w_smx; (void)w_smy;
  (void)w_is; (void)w_nn; (void)pw; (void)out_ptr; (void)in_ptr; (void)out_idx; (void)in_idx;
  (void)srcv; (void)dstv; (void)tmpv; (void)Gl;
  const int H = s->H, W = s->W, NT = s->NT;
  const int64_t N = s->N;
  const or_weights* w = &s->w;
  const double* pr = p;
  const double* pT = p + 3 * N;
  double* ar = Ap;
  double* aT = Ap + 3 * N;
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const int64_t i = (int64_t)y * W + x;
      const double *R0 = R0a + 3 * i, *S0 = S0a + 3 * i;
      double rho[3], q[3];
      for (int c = 0; c < 3; ++c) {
        double sb = 0.0, sg = 0.0;
        for (int k = 0; k < NT; ++k) {
          sb += pT[NT * i + k] * Bl[k][c];
          sg += pT[NT * i + k] * Gl[k][c];
        }
        rho[c] = R0[c] * (S0[c] * pr[3 * i + c] + sb); /* data rows (energy.py:211-218) */
        q[c] = w->lam_m * edge[i] * sg;             /* monochrome (energy.py:403-408) */
      }
      double cons_o[3] = {0, 0, 0}, cons_i[3] = {0, 0, 0};
      for (int64_t qq = out_ptr[i]; qq < out_ptr[i + 1]; ++qq) {
        const int64_t j = out_idx[qq];
        for (int c = 0; c < 3; ++c)
          cons_o[c] += pw[j] * (pr[3 * i + c] - (tmpv[j] ? 0.0 : pr[3 * (int64_t)dstv[j] + c]));
      }
      for (int64_t qq = in_ptr[i]; qq < in_ptr[i + 1]; ++qq) {
        const int64_t j = in_idx[qq];
        const int64_t a = srcv[j];
        for (int c = 0; c < 3; ++c) cons_i[c] += pw[j] * (pr[3 * a + c] - pr[3 * i + c]);
      }
      const double wc = w_rs[i];
      const double wl = x > 0 ? w_rs[i - 1] : 0.0, wu = y > 0 ? w_rs[i - W] : 0.0;
      for (int c = 0; c < 3; ++c) {
        const double v = pr[3 * i + c];
        double a = w->lam_d * R0[c] * S0[c] * rho[c];
        a += w->lam_cl * v;
        double dv = 0.0;
        if (x > 0) dv += wl * (v - pr[3 * (i - 1) + c]);
        if (x < W - 1) dv -= wc * (pr[3 * (i + 1) + c] - v);
        if (y > 0) dv += wu * (v - pr[3 * (i - W) + c]);
        if (y < H - 1) dv -= wc * (pr[3 * (i + W) + c] - v);
        a += dv;
        a += cons_o[c] - cons_i[c];
        ar[3 * i + c] = a;
      }
      for (int k = 0; k < NT; ++k) {
        const int64_t o = NT * i + k;
        const double v = pT[o];
        double a = 0.0, am = 0.0;
        for (int c = 0; c < 3; ++c) {
          a += w->lam_d * R0[c] * rho[c] * Bl[k][c];
          am += q[c] * Gl[k][c];
        }
        a += am;
        if (k >= 1) a += w_is[o] * v;
        const double ax = w_smx[o], ay = w_smy[o];
        const double al = x > 0 ? w_smx[o - NT] : 0.0, au = y > 0 ? w_smy[o - (int64_t)NT * W] : 0.0;
        double dv = 0.0;
        if (x > 0) dv += al * (v - pT[o - NT]);
        if (x < W - 1) dv -= ax * (pT[o + NT] - v);
        if (y > 0) dv += au * (v - pT[o - (int64_t)NT * W]);
        if (y < H - 1) dv -= ay * (pT[o + (int64_t)NT * W] - v);
        a += dv;
        a += w_nn[o] * v;
        aT[o] = a;
      }
    }
}

/* ------------------------------------------------------------------------ */
/* PCG and the GN step (solver.py:79-192)                                    */
/* ------------------------------------------------------------------------ */

/* row-ordered dot product of two length-M vectors laid out as [r | T] */
static double vdot(const or_sys* s, const double* a, const double* b, double* rows) {
  const int H = s->H, W = s->W, NT = s->NT;
  const int64_t N = s->N;
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y) {
    double acc = 0.0;
    const int64_t r0 = (int64_t)y * W * 3, r1 = r0 + (int64_t)W * 3;
    for (int64_t j = r0; j < r1; ++j) acc += a[j] * b[j];
    const int64_t t0 = 3 * N + (int64_t)y * W * NT, t1 = t0 + (int64_t)W * NT;
    for (int64_t j = t0; j < t1; ++j) acc += a[j] * b[j];
    rows[y] = acc;
  }
  return sum_rows(rows, H, 1, 0);
}

/* solver.py:79-107: Jacobi PCG from x = 0; info = {iterations,
 * initial_residual, final_residual} */
void or_pcg(or_sys* s, const double* b, const double* diag, int iterations, double* x, double* info) {
  const int64_t M = (int64_t)s->N * (3 + s->NT);
  double* rows = (double*)malloc(sizeof(double) * s->H);
  double* r = (double*)malloc(sizeof(double) * M);
  double* d = (double*)malloc(sizeof(double) * M);
  double* p = (double*)malloc(sizeof(double) * M);
  double* Ap = (double*)malloc(sizeof(double) * M);
  memset(x, 0, sizeof(double) * M);
  const double bn = sqrt(vdot(s, b, b, rows));
  info[0] = 0;
  info[1] = bn;
  info[2] = bn;
  if (bn != 0.0) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < M; ++j) {
      d[j] = diag[j] > 0.0 ? diag[j] : 1.0;
      r[j] = b[j];
      p[j] = r[j] / d[j];
    }
    double rz = vdot(s, r, p, rows);
    for (int it = 0; it < iterations; ++it) {
      or_apply(s, p, Ap);
      const double pAp = vdot(s, p, Ap, rows);
      if (pAp <= 0.0 || !isfinite(pAp)) break;
      const double a = rz / pAp;
#pragma omp parallel for schedule(static)
      for (int64_t j = 0; j < M; ++j) {
        x[j] += a * p[j];
        r[j] -= a * Ap[j];
        Ap[j] = r[j] / d[j]; /* z */
      }
      info[0] = it + 1;
      const double rz_new = vdot(s, r, Ap, rows);
      if (rz_new <= 0.0) break;
      const double beta = rz_new / rz;
#pragma omp parallel for schedule(static)
      for (int64_t j = 0; j < M; ++j) p[j] = Ap[j] + beta * p[j];
      rz = rz_new;
    }
    info[2] = sqrt(vdot(s, r, r, rows));
  }
  free(rows);
  free(r);
  free(d);
  free(p);
  free(Ap);
}

/* solver.py:143-192 on the state (r, T) in place.  Returns 0, or 1 when the
 * energy at the linearisation point is not finite (NumericalFaultError). */
int or_gn_step(or_sys* s, double* r, double* T, int pcg_iterations, int max_halvings, or_record* rec) {
  const int64_t N = s->N, NT = s->NT, M = N * (3 + NT);
  memset(rec, 0, sizeof(*rec));
  or_linearize(s, r, T);
  double t0[NTERMS];
  int rc = or_terms(s, r, T, t0);
  if (rc) return rc;
  const double e0 = energy_sum(t0);
  for (int j = 0; j < NTERMS; ++j) rec->terms[j] = t0[j];
  rec->energy_before = rec->energy_after = e0;
  if (!isfinite(e0)) return 1;
  double* b = (double*)malloc(sizeof(double) * M);
  double* dg = (double*)malloc(sizeof(double) * M);
  double* dx = (double*)malloc(sizeof(double) * M);
  double* rn = (double*)malloc(sizeof(double) * 3 * N);
  double* Tn = (double*)malloc(sizeof(double) * NT * N);
  or_grad_diag(s, b, dg);
  double info[3];
  or_pcg(s, b, dg, pcg_iterations, dx, info);
  rec->pcg_iterations = (int)info[0];
  rec->initial_residual = info[1];
  rec->final_residual = info[2];
  double alpha = 1.0;
  for (int h = 0; h <= max_halvings; ++h) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < 3 * N; ++j) rn[j] = r[j] + alpha * dx[j];
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < NT * N; ++j) Tn[j] = T[j] + alpha * dx[3 * N + j];
    double tt[NTERMS];
    or_terms(s, rn, Tn, tt);
    const double et = energy_sum(tt);
    if (isfinite(et) && et <= e0) {
      memcpy(r, rn, sizeof(double) * 3 * N);
      memcpy(T, Tn, sizeof(double) * NT * N);
      rec->accepted = 1;
      rec->energy_after = et;
      rec->alpha = alpha;
      for (int j = 0; j < NTERMS; ++j) rec->terms[j] = tt[j];
      break;
    }
    alpha *= 0.5;
  }
  free(b);
  free(dg);
  free(dx);
  free(rn);
  free(Tn);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* dense base-color phase (energy.py:518-610, solver.py:195-255)             */
/* ------------------------------------------------------------------------ */

/* energy.py:563-610: A (3K x 3K), rhs (3K) at delta_b = 0 */
void or_dense_normal(or_sys* s, const double* r, const double* T, int use_ids, double* A, double* rhs) {
  const int H = s->H, W = s->W, K = s->K, NT = s->NT, n = 3 * K;
  const or_weights* w = &s->w;
  /* per-row partials: K*K*3 products + 3K rhs + K counts + 3K anchor sums */
  const int nv = 3 * K * K + 3 * K + K + 3 * K;
  double* rows = (double*)calloc((size_t)H * nv, sizeof(double));
#pragma omp parallel for schedule(static)
  for (int y = 0; y < H; ++y) {
    double* acc = rows + (size_t)y * nv;
    for (int x = 0; x < W; ++x) {
      const int64_t i = (int64_t)y * W + x;
      const double* t = T + NT * i;
      for (int c = 0; c < 3; ++c) {
        const double R = exp(r[3 * i + c]);
        double S = 0.0;
        for (int k = 0; k < NT; ++k) S += t[k] * s->B[k][c];
        const double res = s->img[3 * i + c] - R * S;
        for (int k = 0; k < K; ++k) {
          for (int j = 0; j < K; ++j) acc[(c * K + k) * K + j] += R * R * t[1 + k] * t[1 + j];
          acc[3 * K * K + 3 * k + c] += t[1 + k] * (R * res);
        }
      }
      if (use_ids && s->ids) {
        const int k = s->ids[i] - 1;
        acc[3 * K * K + 3 * K + k] += 1.0;
        for (int c = 0; c < 3; ++c) {
          const double bk = s->colors[3 * k + c] > 1e-4 ? s->colors[3 * k + c] : 1e-4;
          acc[3 * K * K + 4 * K + 3 * k + c] += r[3 * i + c] - log(bk);
        }
      }
    }
  }
  double* tot = (double*)calloc((size_t)nv, sizeof(double));
  for (int v = 0; v < nv; ++v) tot[v] = sum_rows(rows, H, nv, v);
  memset(A, 0, sizeof(double) * n * n);
  memset(rhs, 0, sizeof(double) * n);
  for (int c = 0; c < 3; ++c)
    for (int k = 0; k < K; ++k) {
      for (int j = 0; j < K; ++j) A[(3 * k + c) * n + 3 * j + c] = w->lam_d * tot[(c * K + k) * K + j];
      rhs[3 * k + c] = w->lam_d * tot[3 * K * K + 3 * k + c];
    }
  if (use_ids && s->ids)
    for (int k = 0; k < K; ++k) {
      const double nk = tot[3 * K * K + 3 * K + k];
      if (nk == 0.0) continue;
      for (int c = 0; c < 3; ++c) {
        const double bk = s->colors[3 * k + c] > 1e-4 ? s->colors[3 * k + c] : 1e-4;
        A[(3 * k + c) * n + 3 * k + c] += w->lam_cl * nk / (bk * bk);
        rhs[3 * k + c] += w->lam_cl * tot[3 * K * K + 4 * K + 3 * k + c] / bk;
      }
    }
  for (int j = 0; j < n; ++j) A[j * n + j] += w->lam_ir;
  for (int k = 0; k < K; ++k) { /* chroma_projections (energy.py:518-539) */
    const double* b = s->colors + 3 * k;
    const double nrm = sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) {
        double P = a == c ? 1.0 : 0.0;
        if (!(w->chroma_reg == 1 || nrm < 1e-9)) P -= (b[a] / nrm) * (b[c] / nrm);
        A[(3 * k + a) * n + 3 * k + c] += w->lam_cr * P;
      }
  }
  free(rows);
  free(tot);
}

/* solver.py:195-204: truncated-SVD minimum-norm solve (one-sided Jacobi SVD
 * in place of LAPACK gesdd; same singular triplets to rounding) */
void or_svd_solve(int n, const double* A_in, const double* rhs, double trunc, double* x) {
  memset(x, 0, sizeof(double) * n);
  int any = 0;
  for (int j = 0; j < n * n; ++j) any |= A_in[j] != 0.0;
  if (!any) return;
  double* U = (double*)malloc(sizeof(double) * n * n); /* columns of A V */
  double* V = (double*)calloc((size_t)n * n, sizeof(double));
  double* sv = (double*)malloc(sizeof(double) * n);
  int* ord = (int*)malloc(sizeof(int) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) U[i * n + j] = A_in[i * n + j];
  for (int j = 0; j < n; ++j) V[j * n + j] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int i = 0; i < n; ++i) {
          a += U[i * n + p] * U[i * n + p];
          b += U[i * n + q] * U[i * n + q];
          g += U[i * n + p] * U[i * n + q];
        }
        if (g == 0.0 || fabs(g) <= 1e-15 * sqrt(a * b)) continue;
        off = fmax(off, fabs(g) / sqrt(a * b));
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = 0; i < n; ++i) {
          const double up = U[i * n + p], uq = U[i * n + q];
          U[i * n + p] = cs * up - sn * uq;
          U[i * n + q] = sn * up + cs * uq;
          const double vp = V[i * n + p], vq = V[i * n + q];
          V[i * n + p] = cs * vp - sn * vq;
          V[i * n + q] = sn * vp + cs * vq;
        }
      }
    if (off < 1e-15) break;
  }
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int i = 0; i < n; ++i) s2 += U[i * n + j] * U[i * n + j];
    sv[j] = sqrt(s2);
    ord[j] = j;
  }
  for (int a = 0; a < n; ++a) /* descending singular values */
    for (int b2 = a + 1; b2 < n; ++b2)
      if (sv[ord[b2]] > sv[ord[a]]) {
        const int t = ord[a];
        ord[a] = ord[b2];
        ord[b2] = t;
      }
  const double s0 = sv[ord[0]];
  if (s0 > 0.0)
    for (int m = 0; m < n; ++m) {
      const int j = ord[m];
      if (!(sv[j] > trunc * s0)) continue;
      double c = 0.0;
      for (int i = 0; i < n; ++i) c += U[i * n + j] / sv[j] * rhs[i];
      c /= sv[j];
      for (int i = 0; i < n; ++i) x[i] += V[i * n + j] * c;
    }
  free(U);
  free(V);
  free(sv);
  free(ord);
}

static double frozen_energy_at(or_sys* s, const double* r, const double* T) {
  double t[NTERMS];
  or_linearize(s, r, T);
  or_terms(s, r, T, t);
  return energy_sum(t);
}

/* solver.py:207-255: one dense step on s->colors (updated in place) */
int or_dense_step(or_sys* s, const double* r, const double* T, const or_config* cfg, or_record* rec,
                  double* applied) {
  const int K = s->K, n = 3 * K;
  double A[36 * 36], rhs[36], db[36], cols[36], cand[36];
  memset(rec, 0, sizeof(*rec));
  rec->phase = 1;
  memset(applied, 0, sizeof(double) * n);
  or_dense_normal(s, r, T, s->ids != NULL, A, rhs);
  or_svd_solve(n, A, rhs, cfg->svd_truncation, db);
  int any = 0;
  for (int j = 0; j < n; ++j) any |= db[j] != 0.0;
  if (!any) return 0; /* solver.py:218-219: no record */
  double big = 0.0;
  for (int j = 0; j < n; ++j) big = fmax(big, fabs(db[j]));
  if (big > cfg->max_delta_b)
    for (int j = 0; j < n; ++j) db[j] *= cfg->max_delta_b / big;
  memcpy(cols, s->colors, sizeof(double) * n);
  const double e0 = frozen_energy_at(s, r, T);
  double alpha = 1.0, e1 = e0;
  int accepted = 0;
  for (int h = 0; h <= cfg->max_halvings; ++h) {
    for (int j = 0; j < n; ++j) {
      const double v = cols[j] + alpha * db[j];
      cand[j] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
    or_sys_set_colors(s, cand);
    const double et = frozen_energy_at(s, r, T);
    if (isfinite(et) && et <= e0) {
      double nrm = 0.0;
      for (int j = 0; j < n; ++j) {
        applied[j] = cand[j] - cols[j];
        nrm += applied[j] * applied[j];
      }
      rec->delta_b_norm = sqrt(nrm);
      e1 = et;
      accepted = 1;
      break;
    }
    alpha *= 0.5;
  }
  if (!accepted) or_sys_set_colors(s, cols);
  rec->energy_before = e0;
  rec->energy_after = e1;
  rec->accepted = accepted;
  rec->alpha = accepted ? alpha : 0.0;
  return 1;
}

/* solver state of the flip-flop (solver.py:66-76) */
typedef struct {
  double *r, *T;
  double colors[36];
  double* hist;
  int nhist;
  or_record* recs;
  int nrec, cap;
} fstate;

static void push_rec(fstate* f, const or_record* r) {
  if (f->nrec < f->cap) f->recs[f->nrec] = *r;
  f->nrec++;
  if (r->accepted) f->hist[f->nhist++] = r->energy_after;
}

static int sparse_step(or_sys* s, fstate* f, const or_config* cfg) {
  or_sys_set_colors(s, f->colors);
  or_record rec;
  const int rc = or_gn_step(s, f->r, f->T, cfg->pcg_iterations, cfg->max_halvings, &rec);
  if (rc) return rc;
  push_rec(f, &rec);
  return 0;
}

/* solver.py:274-292: plain sparse step vs dense + sparse; lower energy wins */
static int refine_round(or_sys* s, fstate* f, const or_config* cfg, int cap_hist) {
  const int64_t N = s->N, NT = s->NT;
  fstate ref = *f;
  ref.r = (double*)malloc(sizeof(double) * 3 * N);
  ref.T = (double*)malloc(sizeof(double) * NT * N);
  ref.hist = (double*)malloc(sizeof(double) * cap_hist);
  ref.recs = (or_record*)malloc(sizeof(or_record) * f->cap);
  memcpy(ref.r, f->r, sizeof(double) * 3 * N);
  memcpy(ref.T, f->T, sizeof(double) * NT * N);
  memcpy(ref.hist, f->hist, sizeof(double) * f->nhist);
  memcpy(ref.recs, f->recs, sizeof(or_record) * (f->nrec < f->cap ? f->nrec : f->cap));
  int rc = sparse_step(s, f, cfg); /* the plain branch runs on f itself */
  if (!rc) {
    or_sys_set_colors(s, ref.colors);
    or_record drec;
    double applied[36];
    if (or_dense_step(s, ref.r, ref.T, cfg, &drec, applied)) push_rec(&ref, &drec);
    memcpy(ref.colors, s->colors, sizeof(double) * 3 * s->K);
    rc = sparse_step(s, &ref, cfg);
  }
  if (!rc) {
    const double e_p = f->nhist ? f->hist[f->nhist - 1] : INFINITY;
    const double e_r = ref.nhist ? ref.hist[ref.nhist - 1] : INFINITY;
    if (e_r < e_p) {
      memcpy(f->r, ref.r, sizeof(double) * 3 * N);
      memcpy(f->T, ref.T, sizeof(double) * NT * N);
      memcpy(f->colors, ref.colors, sizeof(double) * 3 * s->K);
      memcpy(f->hist, ref.hist, sizeof(double) * ref.nhist);
      f->nhist = ref.nhist;
      memcpy(f->recs, ref.recs, sizeof(or_record) * (ref.nrec < f->cap ? ref.nrec : f->cap));
      f->nrec = ref.nrec;
    }
  }
  free(ref.r);
  free(ref.T);
  free(ref.hist);
  free(ref.recs);
  return rc;
}

/* solver.py:311-338 (flip_flop) on (r, T, colors) in place.  status:
 * 0 max_outer, 1 stalled, 2 converged.  Returns 0, 1 (non-finite), 2 (args). */
int or_flip_flop(or_sys* s, double* r, double* T, double* colors, const or_config* cfg, or_record* recs,
                 int cap, int* n_records, int* status) {
  const int cap_hist = 4 * (cfg->outer_iterations * (cfg->gn_steps + 3) + 8);
  fstate f;
  f.r = r;
  f.T = T;
  memcpy(f.colors, colors, sizeof(double) * 3 * s->K);
  f.hist = (double*)malloc(sizeof(double) * cap_hist);
  f.nhist = 0;
  f.recs = recs;
  f.nrec = 0;
  f.cap = cap;
  double e_prev = 0.0;
  int have_prev = 0, stalled = 0, rc = 0;
  *status = 0;
  for (int outer = 0; outer < cfg->outer_iterations && !rc; ++outer) {
    int have_rel = 0;
    double rel_s = 0.0;
    for (int g = 0; g < cfg->gn_steps && !rc; ++g) {
      rc = sparse_step(s, &f, cfg);
      if (rc) break;
      const or_record* last = &f.recs[(f.nrec - 1) < cap ? f.nrec - 1 : cap - 1];
      if (!last->accepted) stalled = 1;
      else if (last->energy_before > 0.0) {
        rel_s = (last->energy_before - last->energy_after) / last->energy_before;
        have_rel = 1;
      }
    }
    if (rc) break;
    const int settled = have_rel && rel_s < cfg->refine_gate_rel;
    if (cfg->refine && outer >= cfg->refine_warmup && (settled || stalled)) {
      rc = refine_round(s, &f, cfg, cap_hist);
      if (rc) break;
    }
    if (!f.nhist) continue;
    const double e_now = f.hist[f.nhist - 1];
    if (have_prev && e_prev > 0.0) {
      const double rel = (e_prev - e_now) / e_prev;
      if (0.0 <= rel && rel < cfg->tol_rel) {
        *status = 2;
        break;
      }
    }
    e_prev = e_now;
    have_prev = 1;
  }
  if (!rc && *status != 2) *status = stalled ? 1 : 0;
  memcpy(colors, f.colors, sizeof(double) * 3 * s->K);
  *n_records = f.nrec;
  free(f.hist);
  or_sys_set_colors(s, colors);
  return rc;
}
