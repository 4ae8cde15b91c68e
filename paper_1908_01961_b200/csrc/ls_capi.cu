// Context, workspace and the C ABI (include/lumisplit_b200.h).
//
// The context owns every device buffer the hot path touches, allocated once
// in ls_ctx_create: no cudaMalloc in the per-frame or per-step calls (the
// adjacency is regrown only if a hand-made pair list outgrows it).  The
// Gauss-Newton step is orchestrated here, natively: 1 fused energy/gradient
// kernel, PCG iterations of (apply, update) with device-resident scalars,
// and line-search trials.  ls_gn_step decides accept / halve on the host (one
// synchronisation per trial, solver.py:169-178); ls_flip_flop_stream /
// ls_flip_flop_graph decide everything on the device and synchronise once per
// frame, the latter as one CUDA-graph launch; the ls_band_* entry points are
// the same phases for one band of rows (bands.py).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lumisplit_b200.h"
#include "ls_kernels.h"

using namespace ls;

static thread_local std::string g_err;

#define LS_CK(call)                                                         \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) {                                                \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);           \
      return LS_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)

#define LS_ARG(cond, msg)        \
  do {                           \
    if (!(cond)) {               \
      g_err = (msg);             \
      return LS_ERR_ARG;         \
    }                            \
  } while (0)

// ---- TMA descriptors (driver entry point fetched through the runtime) ------
static PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// planes x H x W float32 tensor, box (boxw, boxh, planes)
static bool make_map(CUtensorMap* m, const float* base, int W, int H, int planes, int boxw, int boxh) {
  auto fn = tma_encode_fn();
  if (!fn || ((uintptr_t)base & 15) || (W % 4) != 0) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)boxh, (cuuint32_t)planes};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// CUDA-event timing of the solver kernels by class (bench.py roofline)
enum { PC_EG = 0, PC_APPLY, PC_UPDATE, PC_TRIAL, PC_DENSE, PC_N };
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  std::vector<std::pair<int, size_t>> pend;   // (class, index of start event)
  double ms[PC_N] = {0};
  long long cnt[PC_N] = {0};
};

struct ls_ctx {
  long long launches = 0;                      // every kernel this context launched
  Prof prof;
  bool use_tma = false;
  int dev = 0, H = 0, W = 0, N = 0, K = 0, NT = 0, U = 0;
  ls_weights w{};
  ls_solve_cfg cfg{};
  cudaStream_t stream = nullptr;
  int nsm = 0, ntiles = 0, grid_energy = 0, grid_apply = 0, grid_update = 0, grid_dense = 0, grid_pcg = 0;
  // per-frame aux
  float* img = nullptr;
  double* chroma = nullptr;
  double* prev_chroma = nullptr;
  float* scratch_img = nullptr;
  float* edge = nullptr;
  int32_t* ids = nullptr;
  float* anchor = nullptr;
  float* prev_r = nullptr;
  bool has_image = false, has_ids = false, has_anchor = false, has_prev_r = false;
  // adjacency
  int32_t* row_ptr = nullptr;
  uint16_t* ent = nullptr;
  float* ent_w = nullptr;
  uint32_t* key = nullptr;
  int64_t ent_cap = 0;
  bool has_ent_w = false, has_pairs = false, pairs_from_sampler = false;
  int64_t n_pairs = 0;
  int64_t n_entries = 0;
  int n_temporal = 0;
  int16_t* codes = nullptr;
  int32_t *out_cnt = nullptr, *in_cnt = nullptr, *deg = nullptr, *fill = nullptr, *pair_off = nullptr;
  int* small_i = nullptr;                     // [0] bad flag, [1] temporal count, [2] first_valid
  SampleState* sstate = nullptr;          // device-side sampler rejection bookkeeping
  bool sampled_counts_known = true;
  bool pair_off_ready = false;             // pair_off scanned from out_cnt (lazily, on demand)
  void* cub_tmp = nullptr;      // scan scratch (launch_scan)
  size_t cub_bytes = 0;
  int32_t *seg_raw = nullptr, *seg_key = nullptr, *seg_last = nullptr;
  double* pal_chroma = nullptr;
  // PCG workspace
  float *r = nullptr, *d = nullptr, *u = nullptr, *wv = nullptr, *p = nullptr, *s = nullptr, *x = nullptr;
  // stored search directions p_0 .. p_{n-1} of the whole-frame PCG (x is
  // combined from them once after the loop); LS_X_DEFERRED=1 keeps round 1's
  // per-iteration deferred x-update instead
  std::vector<float*> pdirs;
  bool x_deferred = false;
  // single-reduction PCG (LS_PCG=cg1 at context creation): two more vectors
  bool pcg_cg1 = false;
  int grid_cg = 0;
  float *cg_m1 = nullptr, *cg_t1 = nullptr;
  double* part = nullptr;
  size_t part_len = 0;
  unsigned* tickets = nullptr;
  Scalars* sc = nullptr;
  Scalars* sc_host = nullptr;
  // dense
  double *dense_sums = nullptr, *colors_dev = nullptr, *dense_A = nullptr, *dense_rhs = nullptr,
         *dense_x = nullptr;
  double* host_buf = nullptr;   // pinned, 2 * 36 * 36 + 64 doubles
  FrameCtl* ctl = nullptr;       // device-resident flip-flop control
  StepRecord* recs = nullptr;    // device step records
  StepRecord* recs_host = nullptr;
  FrameCtl* ctl_host = nullptr;
  // row band: this context holds local rows
  // [0, H) = global rows [gy0, gy0 + H) of a GH-row frame and produces rows
  // [y_lo, y_hi); kernels then write partial sums to bsum (band_partial)
  int gy0 = 0, GH = 0, y_lo = 0, y_hi = 0;
  bool band_partial = false;
  double* bsum = nullptr;        // 512 doubles
  long long* zlist = nullptr;    // kZeroList
  int* seg_sum = nullptr;        // 4 ints
  bool band_dev = false;         // inside ls_band_frame_begin / _end: device-side decisions
  float* ring[3] = {nullptr, nullptr, nullptr};   // state buffers of the graph flip-flop
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cond_stream = nullptr;      // captures the bodies of graph conditional nodes
  bool use_cond = false;                   // LS_GRAPH_COND=1: halvings as graph conditional nodes
  bool band_stored = false;                // row band: PCG directions kept (ls_band_dirs)
  cudaGraphExec_t graph_exec = nullptr;
  unsigned char graph_key[1024] = {0};
  long long graph_launches = 0;
  int graph_steps = 0;
  const long long* band_zeros = nullptr;   // gathered zero lists (caller memory) for the next draw
  int band_zero_lists = 0;
  std::vector<void*> allocs;
};

extern "C" {
static void prof_harvest(ls_ctx* c);
}

template <typename T>
static cudaError_t dalloc(ls_ctx* c, T** p, size_t n) {
  cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
  if (e == cudaSuccess) c->allocs.push_back((void*)*p);
  return e;
}

template <typename R>
static Coef<R> make_coef(const ls_weights& w, const double* colors, int K) {
  Coef<R> c;
  std::memset(&c, 0, sizeof(c));
  for (int k = 0; k <= K; ++k) {
    double b[3];
    for (int ch = 0; ch < 3; ++ch) b[ch] = (k == 0) ? 1.0 : colors[3 * (k - 1) + ch];
    const double mean = ((b[0] + b[1]) + b[2]) / 3.0;
    for (int ch = 0; ch < 3; ++ch) {
      c.B[k][ch] = (R)b[ch];
      c.G[k][ch] = (R)(b[ch] - mean);
      c.anchor[k][ch] = (k == 0) ? R(0) : (R)std::log(std::max(b[ch], 1e-4));
    }
    R g2 = R(0);
    for (int ch = 0; ch < 3; ++ch) g2 = std::fma(c.G[k][ch], c.G[k][ch], g2);
    c.g2[k] = g2;
  }
  c.lam_d = (R)w.lambda_data;
  c.lam_cl = (R)w.lambda_clustering;
  c.lam_rs = (R)w.lambda_r_sparsity;
  c.p = (R)w.p;
  c.lam_rc = (R)w.lambda_r_consistency;
  c.lam_m = (R)w.lambda_monochrome;
  c.lam_is = (R)w.lambda_i_sparsity;
  c.lam_sm = (R)w.lambda_smoothness;
  c.lam_nn = (R)w.lambda_non_neg;
  c.eps_nn = (R)w.eps_nonneg;
  c.eps_irls = (R)w.eps_irls;
  c.inv_eps = (R)(1.0 / w.eps_irls);
  c.floor_rs = (R)(w.p < 2.0 ? std::pow(w.eps_irls, 1.0 / (2.0 - w.p)) : 0.0);
  return c;
}

static Frame frame_of(const ls_ctx* c) {
  Frame f;
  std::memset(&f, 0, sizeof(f));   // padding bytes take part in graph keys
  f.H = c->H;
  f.W = c->W;
  f.N = c->N;
  f.NT = c->NT;
  f.img = c->img;
  f.edge = c->edge;
  f.ids = c->has_ids ? c->ids : nullptr;
  f.anchor = c->has_anchor ? c->anchor : nullptr;
  f.prev_r = c->has_prev_r ? c->prev_r : nullptr;
  f.row_ptr = c->row_ptr;
  f.ent = c->ent;
  f.ent_w = c->has_ent_w ? c->ent_w : nullptr;
  f.y_lo = c->y_lo;
  f.y_hi = c->y_hi;
  f.bsum = c->band_partial ? c->bsum : nullptr;
  return f;
}

// tile / grid geometry of the produced rows [y_lo, y_hi)
static void set_geometry(ls_ctx* c) {
  const int rows = c->y_hi - c->y_lo;
  c->ntiles = ((c->W + kTileW - 1) / kTileW) * ((rows + kTileH - 1) / kTileH);
  c->grid_energy = std::max(1, std::min({c->ntiles, c->nsm * std::max(1, energy_grid_limit(c->NT)), kMaxBlocks}));
  c->grid_apply = std::max(1, std::min({c->ntiles, c->nsm * std::max(1, apply_grid_limit(c->NT)), kMaxBlocks}));
  c->grid_pcg = std::max(1, std::min({c->ntiles, c->nsm * std::max(1, pcg_apply_grid_limit(c->NT)), kMaxBlocks}));
  const int64_t M = (int64_t)c->U * rows * c->W;
  const int64_t upd_blocks = (M / 4 + kThreads - 1) / kThreads;
  // LS_UPD_GRID: resident CTAs per SM of the streaming PCG update (A/B; default: its occupancy)
  const char* ug = std::getenv("LS_UPD_GRID");
  const int upd_per_sm = ug ? std::max(1, std::atoi(ug)) : std::max(1, update_grid_limit());
  c->grid_update = (int)std::max<int64_t>(1, std::min<int64_t>({upd_blocks, (int64_t)c->nsm * upd_per_sm, (int64_t)kMaxBlocks}));
  c->grid_dense = std::max(1, std::min(c->nsm * 8, (rows * c->W + 63) / 64));
}

// the whole-frame entry points finalise inside their kernels
static int whole_frame_only(ls_ctx* c) {
  LS_ARG(c && !c->band_partial, "context is a row band: use the ls_band_* entry points");
  return LS_OK;
}

extern "C" int ls_pair_count(ls_ctx* c, int64_t* n_pairs, int64_t* n_temporal, int64_t* n_entries);

static int check_ready(ls_ctx* c) {
  LS_ARG(c != nullptr, "null context");
  LS_ARG(c->has_image, "no frame image set (ls_set_image)");
  LS_ARG(c->has_pairs, "no consistency partners (ls_sample_consistency / ls_set_pairs)");
  LS_ARG(c->has_ids || c->has_anchor, "EnergyAux needs cluster_ids or r_cluster_log");
  if (c->n_temporal != 0 && !c->has_prev_r) {
    if (c->n_temporal < 0) {
      int rc = ls_pair_count(c, nullptr, nullptr, nullptr);
      if (rc) return rc;
    }
    LS_ARG(c->n_temporal == 0, "temporal partners need the previous frame's reflectance");
  }
  return LS_OK;
}

extern "C" {

const char* ls_version(void) { return "lumisplit_b200 0.1 (sm_100a)"; }
const char* ls_last_error(void) { return g_err.c_str(); }

int ls_set_weights(ls_ctx* c, const ls_weights* w, const ls_solve_cfg* cfg) {
  LS_ARG(c && w && cfg, "null argument");
  LS_ARG(w->eps_irls > 0.0, "eps_irls must be positive");
  LS_ARG(cfg->pcg_iterations >= 0 && cfg->max_halvings >= 0, "bad solve config");
  c->w = *w;
  c->cfg = *cfg;
  return LS_OK;
}

int ls_set_stream(ls_ctx* c, void* stream) {
  LS_ARG(c, "null context");
  c->stream = (cudaStream_t)stream;
  return LS_OK;
}

int ls_ctx_create(int device, int H, int W, int K, const ls_weights* w, const ls_solve_cfg* cfg, ls_ctx** out) {
  LS_ARG(out && w && cfg, "null argument");
  LS_ARG(H >= 1 && W >= 1 && (int64_t)H * W < (1LL << 28), "bad frame size");
  LS_ARG(K >= 0 && K <= LS_MAX_K, "K must be in [0, 12]");
  LS_CK(cudaSetDevice(device));
  ls_ctx* c = new ls_ctx();
  c->dev = device;
  c->H = H;
  c->W = W;
  c->N = H * W;
  c->K = K;
  c->NT = K + 1;
  c->U = K + 4;
  int rc = ls_set_weights(c, w, cfg);
  if (rc != LS_OK) { delete c; return rc; }
  cudaDeviceProp prop;
  LS_CK(cudaGetDeviceProperties(&prop, device));
  c->nsm = prop.multiProcessorCount;
  const int N = c->N, U = c->U;
  const int64_t M = (int64_t)U * N;
  c->GH = H;
  c->y_hi = H;
  set_geometry(c);
  c->use_tma = (W % 4 == 0) && tma_encode_fn() != nullptr && std::getenv("LS_NO_TMA") == nullptr;
  c->x_deferred = std::getenv("LS_X_DEFERRED") != nullptr && std::string(std::getenv("LS_X_DEFERRED")) == "1";
  c->use_cond = std::getenv("LS_GRAPH_COND") != nullptr && std::string(std::getenv("LS_GRAPH_COND")) == "1";
  {   // opt-in single-reduction PCG (whole frames with TMA only)
    const char* pv = std::getenv("LS_PCG");
    c->pcg_cg1 = pv && std::string(pv) == "cg1" && c->use_tma;
    if (c->pcg_cg1)
      c->grid_cg = std::max(1, std::min({c->ntiles, c->nsm * std::max(1, cg_grid_limit(c->NT)), kMaxBlocks}));
  }
  cudaError_t e = cudaSuccess;
#define A_(expr) \
  if (e == cudaSuccess) e = (expr)
  A_(dalloc(c, &c->img, 3 * (size_t)N));
  A_(dalloc(c, &c->chroma, 2 * (size_t)N));
  A_(dalloc(c, &c->prev_chroma, 2 * (size_t)N));
  A_(dalloc(c, &c->scratch_img, 3 * (size_t)N));
  A_(dalloc(c, &c->edge, (size_t)N));
  A_(dalloc(c, &c->ids, (size_t)N));
  A_(dalloc(c, &c->anchor, 3 * (size_t)N));
  A_(dalloc(c, &c->prev_r, 3 * (size_t)N));
  A_(dalloc(c, &c->row_ptr, (size_t)N + 1));
  c->ent_cap = 8 * (int64_t)N + 16;
  A_(cudaMalloc((void**)&c->ent, sizeof(uint16_t) * c->ent_cap));
  A_(cudaMalloc((void**)&c->ent_w, sizeof(float) * c->ent_cap));
  A_(cudaMalloc((void**)&c->key, sizeof(uint32_t) * c->ent_cap));
  A_(dalloc(c, &c->codes, 4 * (size_t)N));
  A_(dalloc(c, &c->out_cnt, (size_t)N + 1));
  A_(dalloc(c, &c->in_cnt, (size_t)N + 1));
  A_(dalloc(c, &c->deg, (size_t)N + 1));
  A_(dalloc(c, &c->fill, (size_t)N + 1));
  A_(dalloc(c, &c->pair_off, (size_t)N + 1));
  A_(dalloc(c, &c->small_i, 8));
  A_(dalloc(c, &c->sstate, 1));
  A_(dalloc(c, &c->seg_raw, (size_t)N));
  A_(dalloc(c, &c->seg_key, (size_t)N));
  A_(dalloc(c, &c->seg_last, (size_t)N));
  A_(dalloc(c, &c->pal_chroma, 2 * LS_MAX_K));
  for (float** v : {&c->r, &c->d, &c->u, &c->wv, &c->p, &c->s, &c->x}) A_(dalloc(c, v, (size_t)M));
  c->part_len = std::max<size_t>((size_t)kMaxBlocks * 12, (size_t)c->grid_dense * 320);
  A_(dalloc(c, &c->part, c->part_len));
  if (c->pcg_cg1) {
    A_(dalloc(c, &c->cg_m1, (size_t)M));
    A_(dalloc(c, &c->cg_t1, (size_t)M));
  }
  A_(dalloc(c, &c->tickets, 8));
  A_(dalloc(c, &c->sc, 1));
  A_(dalloc(c, &c->dense_sums, 512));
  A_(dalloc(c, &c->colors_dev, 3 * LS_MAX_K));
  A_(dalloc(c, &c->dense_A, 36 * 36));
  A_(dalloc(c, &c->dense_rhs, 36));
  A_(dalloc(c, &c->dense_x, 36));
  A_(dalloc(c, &c->bsum, 512));
  A_(dalloc(c, &c->zlist, kZeroList));
  A_(dalloc(c, &c->seg_sum, 4));
  A_(cudaMallocHost((void**)&c->sc_host, sizeof(Scalars)));
  A_(dalloc(c, &c->ctl, 1));
  A_(dalloc(c, &c->recs, kMaxStepRecords));
  A_(cudaHostAlloc((void**)&c->recs_host, sizeof(StepRecord) * kMaxStepRecords, cudaHostAllocMapped));   // kernel-written (UVA)
  A_(cudaHostAlloc((void**)&c->ctl_host, sizeof(FrameCtl), cudaHostAllocMapped));   // kernel-written (UVA)
  A_(cudaHostAlloc((void**)&c->host_buf, sizeof(double) * (2 * 36 * 36 + 64), cudaHostAllocMapped));   // kernel-written (UVA)
  A_(cudaMemset(c->tickets, 0, 8 * sizeof(unsigned)));
  A_(cudaMemset(c->sc, 0, sizeof(Scalars)));
  // scan scratch (tile status words + tile counter) for N+1 values
  c->cub_bytes = scan_scratch_bytes((int64_t)N + 1);
  A_(dalloc(c, (char**)&c->cub_tmp, c->cub_bytes));
#undef A_
  if (e != cudaSuccess) {
    g_err = std::string("ls_ctx_create: ") + cudaGetErrorString(e);
    ls_ctx_destroy(c);
    return LS_ERR_CUDA;
  }
  *out = c;
  return LS_OK;
}

int ls_profile(ls_ctx* c, int enable) {
  LS_ARG(c, "null context");
  if (enable && c->prof.pool.empty()) {
    c->prof.pool.resize(4096);
    for (auto& e : c->prof.pool) LS_CK(cudaEventCreate(&e));
  }
  LS_CK(cudaStreamSynchronize(c->stream));
  prof_harvest(c);
  for (int i = 0; i < PC_N; ++i) { c->prof.ms[i] = 0.0; c->prof.cnt[i] = 0; }
  c->prof.on = enable != 0;
  c->launches = 0;
  return LS_OK;
}

// launch bookkeeping for work replayed outside the context (a caller-side
// CUDA graph of ls_band_* calls): read the counter / add replayed launches
int ls_launch_count(ls_ctx* c, int64_t* n) {
  LS_ARG(c && n, "bad arguments");
  *n = c->launches;
  return LS_OK;
}

int ls_add_launches(ls_ctx* c, int64_t n) {
  LS_ARG(c && c->launches + n >= 0, "bad arguments");
  c->launches += n;
  return LS_OK;
}

int ls_state_key(ls_ctx* c, void* out, int64_t cap, int64_t* len) {
  LS_ARG(c && len && (out || cap == 0), "bad arguments");
  struct {
    ls_weights w;
    ls_solve_cfg cfg;
    Frame f;
    int use_tma;
  } key;
  std::memset(&key, 0, sizeof(key));
  key.w = c->w;
  key.cfg = c->cfg;
  key.f = frame_of(c);
  key.use_tma = c->use_tma;
  *len = (int64_t)sizeof(key);
  if (cap > 0) std::memcpy(out, &key, (size_t)std::min<int64_t>(cap, sizeof(key)));
  return LS_OK;
}

int ls_profile_read(ls_ctx* c, double* out) {
  LS_ARG(c && out, "bad arguments");
  LS_CK(cudaStreamSynchronize(c->stream));
  prof_harvest(c);
  for (int i = 0; i < PC_N; ++i) {
    out[2 * i] = (double)c->prof.cnt[i];
    out[2 * i + 1] = c->prof.ms[i];
  }
  out[2 * PC_N] = (double)c->launches;
  if (c->has_pairs && !c->sampled_counts_known) {
    const int rc = ls_pair_count(c, nullptr, nullptr, nullptr);
    if (rc) return rc;
  }
  out[2 * PC_N + 1] = (double)c->n_entries;
  out[2 * PC_N + 2] = (double)c->n_pairs;
  return LS_OK;
}

int ls_ctx_destroy(ls_ctx* c) {
  if (!c) return LS_OK;
  cudaSetDevice(c->dev);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->cond_stream) cudaStreamDestroy(c->cond_stream);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& e : c->prof.pool) cudaEventDestroy(e);
  cudaFree(c->ent);
  cudaFree(c->ent_w);
  cudaFree(c->key);
  if (c->sc_host) cudaFreeHost(c->sc_host);
  if (c->recs_host) cudaFreeHost(c->recs_host);
  if (c->ctl_host) cudaFreeHost(c->ctl_host);
  if (c->host_buf) cudaFreeHost(c->host_buf);
  delete c;
  return LS_OK;
}

int ls_pack_hwc(ls_ctx* c, const float* hwc, int C, float* planes) {
  LS_ARG(c && hwc && planes && C > 0, "bad arguments");
  launch_pack_hwc(c->stream, hwc, C, c->N, planes);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_unpack_hwc(ls_ctx* c, const float* planes, int C, float* hwc) {
  LS_ARG(c && hwc && planes && C > 0, "bad arguments");
  launch_unpack_hwc(c->stream, planes, C, c->N, hwc);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_set_image(ls_ctx* c, const float* image_hwc) {
  LS_ARG(c && image_hwc, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  launch_image(c->stream, image_hwc, c->N, c->img, c->chroma);
  launch_edge(c->stream, c->chroma, c->H, c->W, c->edge);
  c->launches += 2;
  LS_CK(cudaGetLastError());
  c->has_image = true;
  return LS_OK;
}

int ls_set_edge(ls_ctx* c, const float* edge) {
  LS_ARG(c && edge, "bad arguments");
  launch_copy(c->stream, c->edge, edge, sizeof(float) * c->N); LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_get_edge(ls_ctx* c, float* out) {
  LS_ARG(c && out, "bad arguments");
  launch_copy(c->stream, out, c->edge, sizeof(float) * c->N); LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_get_chroma(ls_ctx* c, double* out) {
  LS_ARG(c && out, "bad arguments");
  launch_copy(c->stream, out, c->chroma, sizeof(double) * 2 * c->N); LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_set_prev_r(ls_ctx* c, const float* prev) {
  LS_ARG(c, "null context");
  if (!prev) {
    c->has_prev_r = false;
    return LS_OK;
  }
  launch_copy(c->stream, c->prev_r, prev, sizeof(float) * 3 * c->N); LS_CK(cudaGetLastError());
  c->has_prev_r = true;
  return LS_OK;
}

int ls_set_anchor(ls_ctx* c, const int32_t* ids, const float* anchor) {
  LS_ARG(c, "null context");
  LS_ARG((ids != nullptr) != (anchor != nullptr), "exactly one of cluster_ids / r_cluster_log");
  if (ids) {
    launch_copy(c->stream, c->ids, ids, sizeof(int32_t) * c->N); LS_CK(cudaGetLastError());
    c->has_ids = true;
    c->has_anchor = false;
  } else {
    launch_copy(c->stream, c->anchor, anchor, sizeof(float) * 3 * c->N); LS_CK(cudaGetLastError());
    c->has_anchor = true;
    c->has_ids = false;
  }
  return LS_OK;
}

// build row_ptr from out/in counts; returns total entries (host sync)
static int build_rows(ls_ctx* c, int64_t* total) {
  const int N = c->N;
  launch_degree(c->stream, N, c->out_cnt, c->in_cnt, c->deg);
  LS_CK(cudaMemsetAsync(c->deg + N, 0, sizeof(int32_t), c->stream));
  LS_CK(launch_scan(c->stream, c->deg, c->row_ptr, (int64_t)N + 1, 0, c->cub_tmp));
  int32_t tot = 0;
  LS_CK(cudaMemcpyAsync(&tot, c->row_ptr + N, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  *total = tot;
  return LS_OK;
}

// the device scan the adjacency and segmentation use (decoupled look-back),
// exposed for its own tests: op 0 exclusive sum, 1 inclusive max; scratch of
// ls_scan_scratch_bytes(n) bytes (zeroed by the call)
int64_t ls_scan_scratch_bytes(int64_t n) { return (int64_t)scan_scratch_bytes(n); }

int ls_scan_i32(const int32_t* in, int32_t* out, int64_t n, int op, void* scratch, void* stream) {
  LS_ARG(n >= 0 && (op == 0 || op == 1), "bad arguments");
  LS_ARG(n == 0 || (in && out && scratch), "null arrays");
  LS_CK(launch_scan((cudaStream_t)stream, in, out, n, op, scratch));
  return LS_OK;
}

int ls_device_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  LS_ARG((dst && src) || bytes == 0, "bad arguments");
  LS_ARG(bytes >= 0, "bad size");
  launch_copy((cudaStream_t)stream, dst, src, bytes);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// imaging.py:36-57 frame check without a copy-engine read-back: the flag is
// written by the kernel into mapped host memory (one per host thread)
int ls_all_finite(const float* x, int64_t n, void* stream, int* all_finite) {
  LS_ARG((x || n == 0) && all_finite && n >= 0, "bad arguments");
  static thread_local int* flag = nullptr;
  if (!flag) LS_CK(cudaHostAlloc((void**)&flag, sizeof(int), cudaHostAllocMapped));
  launch_all_finite((cudaStream_t)stream, x, n, flag);
  LS_CK(cudaGetLastError());
  LS_CK(cudaStreamSynchronize((cudaStream_t)stream));
  *all_finite = *(volatile int*)flag;
  return LS_OK;
}

// correction.py:54-68: flood fill of `target` pixels from the seeds, on the
// device; convergence read back through a mapped flag every 16 steps
int ls_flood_fill(const int32_t* ids, int target, const uint8_t* seeds, int H, int W, uint8_t* mask,
                  uint8_t* scratch, void* stream) {
  LS_ARG(ids && seeds && mask && scratch && H >= 1 && W >= 1, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  static thread_local int* changed = nullptr;
  if (!changed) LS_CK(cudaHostAlloc((void**)&changed, sizeof(int), cudaHostAllocMapped));
  const int64_t N = (int64_t)H * W;
  launch_flood_init(st, ids, target, seeds, N, mask);
  uint8_t* buf[2] = {mask, scratch};
  int cur = 0;
  for (int64_t done = 0; done <= N; done += 16) {
    launch_set_flag(st, changed, 0);
    for (int j = 0; j < 16; ++j) {
      launch_flood_step(st, ids, target, H, W, buf[cur], buf[cur ^ 1], changed);
      cur ^= 1;
    }
    LS_CK(cudaGetLastError());
    LS_CK(cudaStreamSynchronize(st));
    if (!*(volatile int*)changed) break;
  }
  if (cur != 0) launch_copy(st, mask, buf[cur], N);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// editing.py:24-74: clip(R' * (T . B')), optional matte -> background
int ls_recompose(const float* X, int K, int H, int W, const double* B, int k, const double* ratio,
                 const int32_t* ids, const uint8_t* matte, const float* bg, float* out, void* stream) {
  LS_ARG(X && B && out && H >= 1 && W >= 1 && K >= 0 && K <= LS_MAX_K, "bad arguments");
  LS_ARG(!matte || bg, "a matte needs a background");
  LS_ARG(k == 0 || (k >= 1 && k <= K && ids), "cluster id outside 1..K or no ids");
  EditParams P;
  std::memset(&P, 0, sizeof(P));
  for (int i = 0; i < 3 * (K + 1); ++i) P.B[i] = B[i];
  for (int c = 0; c < 3; ++c) P.ratio[c] = ratio ? ratio[c] : 1.0;
  P.k = k;
  launch_recompose((cudaStream_t)stream, X, K + 1, (int64_t)H * W, P, ids, matte, bg, out);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_chromaticity(const float* image_hwc, int H, int W, double* out, void* stream) {
  LS_ARG(image_hwc && out && H >= 1 && W >= 1, "bad arguments");
  // planar image copy is not needed: write it into the second half of a scratch-free path
  launch_image((cudaStream_t)stream, image_hwc, H * W, nullptr, out);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_edge_from_chroma(const double* chroma, int H, int W, float* edge, void* stream) {
  LS_ARG(chroma && edge && H >= 1 && W >= 1, "bad arguments");
  launch_edge((cudaStream_t)stream, chroma, H, W, edge);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_sample_consistency(ls_ctx* c, const double* chroma, const double* prev_chroma, uint64_t st_hi, uint64_t st_lo,
                          uint64_t inc_hi, uint64_t inc_lo, int64_t* n_pairs_out) {
  LS_ARG(c && (chroma || c->has_image), "ls_set_image first");
  LS_CK(cudaSetDevice(c->dev));
  const int N = c->N;
  const double* cur = chroma ? chroma : c->chroma;
  SampleParams P;
  std::memset(&P, 0, sizeof(P));
  P.st_hi = st_hi;
  P.st_lo = st_lo;
  P.inc_hi = inc_hi;
  P.inc_lo = inc_lo;
  P.has_prev = prev_chroma ? 1 : 0;
  P.gy0 = c->gy0;
  P.GH = c->GH;
  P.goff = (long long)c->gy0 * c->W;
  P.Ng = (long long)c->GH * c->W;
  // draws + device-side rejection re-passes: no host synchronisation.  A row
  // band gets every rejection of the stream up front (ls_band_set_zeros).
  launch_sample(c->stream, P, c->sstate, cur, prev_chroma, c->H, c->W, c->codes, c->out_cnt, c->in_cnt,
                kSamplePasses, c->band_zeros, c->band_zero_lists);
  c->band_zeros = nullptr;
  c->band_zero_lists = 0;
  launch_degree(c->stream, N, c->out_cnt, c->in_cnt, c->deg);
  LS_CK(cudaMemsetAsync(c->deg + N, 0, sizeof(int32_t), c->stream));
  LS_CK(launch_scan(c->stream, c->deg, c->row_ptr, (int64_t)N + 1, 0, c->cub_tmp));
  LS_CK(cudaMemsetAsync(c->fill, 0, sizeof(int32_t) * N, c->stream));
  launch_fill_from_samples(c->stream, c->codes, c->H, c->W, c->row_ptr, c->out_cnt, c->fill, c->ent);
  // (pair offsets for ls_get_pairs / ls_pair_count: scanned when asked for,
  // ensure_pair_off -- the streaming solve never reads them)
  c->pair_off_ready = false;
  LS_CK(cudaGetLastError());
  c->launches += 1 + 3 * kSamplePasses + 5;
  c->n_pairs = -1;                       // resolved lazily by ls_pair_count
  c->n_entries = -1;
  c->n_temporal = P.has_prev ? -1 : 0;
  c->sampled_counts_known = false;
  c->has_ent_w = false;
  c->has_pairs = true;
  c->pairs_from_sampler = true;
  if (n_pairs_out) *n_pairs_out = -1;
  return LS_OK;
}

// pair offsets (src-major, slot order) of the sampled pairs
static int ensure_pair_off(ls_ctx* c) {
  if (c->pair_off_ready) return LS_OK;
  LS_CK(launch_scan(c->stream, c->out_cnt, c->pair_off, (int64_t)c->N + 1, 0, c->cub_tmp));
  LS_CK(cudaGetLastError());
  c->launches += 1;
  c->pair_off_ready = true;
  return LS_OK;
}

// pair / entry / temporal counts of the sampled adjacency (synchronises)
int ls_pair_count(ls_ctx* c, int64_t* n_pairs, int64_t* n_temporal, int64_t* n_entries) {
  LS_ARG(c && c->has_pairs, "no consistency partners");
  if (!c->sampled_counts_known) {
    const int rc = ensure_pair_off(c);
    if (rc) return rc;
    int32_t v[2] = {0, 0};
    int err = 0;
    LS_CK(cudaMemcpyAsync(&v[0], c->pair_off + c->N, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    LS_CK(cudaMemcpyAsync(&v[1], c->row_ptr + c->N, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    LS_CK(cudaMemcpyAsync(&err, &c->sstate->error, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    LS_CK(cudaStreamSynchronize(c->stream));
    if (err) {
      g_err = "consistency sampler: too many PCG64 rejections in one frame";
      return LS_ERR_CUDA;
    }
    c->n_pairs = v[0];
    c->n_entries = v[1];
    c->n_temporal = (c->n_temporal != 0) ? (int)(v[0] - (v[1] - v[0])) : 0;
    c->sampled_counts_known = true;
  }
  if (n_pairs) *n_pairs = c->n_pairs;
  if (n_temporal) *n_temporal = c->n_temporal;
  if (n_entries) *n_entries = c->n_entries;
  return LS_OK;
}

int ls_get_pairs(ls_ctx* c, int64_t* src, int64_t* dst, uint8_t* temporal) {
  LS_ARG(c && c->has_pairs && c->pairs_from_sampler, "no sampled pairs");
  const int rc = ensure_pair_off(c);
  if (rc) return rc;
  launch_pairs_from_samples(c->stream, c->codes, c->H, c->W, c->pair_off, src, dst, temporal);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_set_pairs(ls_ctx* c, int64_t n, const int64_t* src, const int64_t* dst, const uint8_t* temporal,
                 const double* weight) {
  LS_ARG(c && n >= 0, "bad arguments");
  LS_ARG(n == 0 || (src && dst && temporal), "null pair arrays");
  LS_CK(cudaSetDevice(c->dev));
  const int N = c->N;
  LS_CK(cudaMemsetAsync(c->out_cnt, 0, sizeof(int32_t) * (N + 1), c->stream));
  LS_CK(cudaMemsetAsync(c->in_cnt, 0, sizeof(int32_t) * (N + 1), c->stream));
  LS_CK(cudaMemsetAsync(c->small_i, 0, sizeof(int) * 8, c->stream));
  launch_pairs_count(c->stream, n, src, dst, temporal, c->H, c->W, c->out_cnt, c->in_cnt, c->small_i);
  int bad = 0;
  LS_CK(cudaMemcpyAsync(&bad, c->small_i, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  LS_ARG(!bad, "consistency partners must be valid pixels within the 15x15 window");
  int64_t total = 0;
  int rc = build_rows(c, &total);
  if (rc != LS_OK) return rc;
  if (total + 16 > c->ent_cap) {   // only hand-made pair lists can outgrow 8N
    cudaFree(c->ent);
    cudaFree(c->ent_w);
    cudaFree(c->key);
    c->ent = nullptr; c->ent_w = nullptr; c->key = nullptr;
    c->ent_cap = total + 16;
    LS_CK(cudaMalloc((void**)&c->ent, sizeof(uint16_t) * c->ent_cap));
    LS_CK(cudaMalloc((void**)&c->ent_w, sizeof(float) * c->ent_cap));
    LS_CK(cudaMalloc((void**)&c->key, sizeof(uint32_t) * c->ent_cap));
  }
  LS_CK(cudaMemsetAsync(c->fill, 0, sizeof(int32_t) * N, c->stream));
  launch_fill_from_pairs(c->stream, n, src, dst, temporal, weight, c->W, c->row_ptr, c->fill, c->ent, c->key,
                         weight ? c->ent_w : nullptr);
  launch_sort_rows(c->stream, N, c->row_ptr, c->ent, c->key, weight ? c->ent_w : nullptr);
  LS_CK(cudaGetLastError());
  c->n_pairs = n;
  c->sampled_counts_known = true;
  c->n_entries = total;
  c->n_temporal = (int)(n - (total - n));
  c->has_ent_w = weight != nullptr;
  c->has_pairs = true;
  c->pairs_from_sampler = false;
  return LS_OK;
}

int ls_segment(ls_ctx* c, const double* colors, int32_t* ids_out) {
  LS_ARG(c && c->has_image && colors && ids_out, "bad arguments");
  LS_ARG(c->K >= 1, "segment needs K >= 1");
  const int N = c->N, K = c->K;
  PalChroma pc;
  std::memset(&pc, 0, sizeof(pc));
  for (int k = 0; k < K; ++k) {   // chroma_of_color (imaging.py:174-180)
    const double s = (colors[3 * k] + colors[3 * k + 1]) + colors[3 * k + 2];
    pc.c[2 * k] = s > 1e-12 ? colors[3 * k] / s : 1.0 / 3.0;
    pc.c[2 * k + 1] = s > 1e-12 ? colors[3 * k + 1] / s : 1.0 / 3.0;
  }
  launch_set_i32(c->stream, c->small_i + 2, 1, N);
  launch_segment_raw(c->stream, c->img, c->chroma, N, K, pc, c->seg_raw, c->seg_key, c->small_i + 2);
  LS_CK(launch_scan(c->stream, c->seg_key, c->seg_last, (int64_t)N, 1, c->cub_tmp));
  launch_segment_final(c->stream, N, c->seg_raw, c->seg_last, c->small_i + 2, ids_out);
  c->launches += 4;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_initialize(ls_ctx* c, const double* colors, const int32_t* ids, float* X) {
  LS_ARG(c && c->has_image && colors && ids && X, "bad arguments");
  PalColors pc;
  std::memset(&pc, 0, sizeof(pc));
  for (int i = 0; i < 3 * c->K; ++i) pc.c[i] = colors[i];
  launch_initialize(c->stream, c->img, ids, c->N, c->NT, pc, X);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

static size_t prof_begin(ls_ctx* c) {
  if (!c->prof.on) return 0;
  if (c->prof.next + 2 > c->prof.pool.size()) return (size_t)-1;   // pool full: skip sample
  const size_t i = c->prof.next;
  c->prof.next += 2;
  cudaEventRecord(c->prof.pool[i], c->stream);
  return i;
}
static void prof_end(ls_ctx* c, int cls, size_t i) {
  if (!c->prof.on || i == (size_t)-1) return;
  cudaEventRecord(c->prof.pool[i + 1], c->stream);
  c->prof.pend.emplace_back(cls, i);
}
// call only after a stream synchronisation
static void prof_harvest(ls_ctx* c) {
  for (auto& pe : c->prof.pend) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, c->prof.pool[pe.second], c->prof.pool[pe.second + 1]) == cudaSuccess) {
      c->prof.ms[pe.first] += t;
      c->prof.cnt[pe.first] += 1;
    }
  }
  c->prof.pend.clear();
  c->prof.next = 0;
}

// tile descriptors for state X and operand v (both U planes); false -> no TMA
static bool tile_maps(ls_ctx* c, const float* X, const float* v, TileMaps* m) {
  if (!c->use_tma) return false;
  const int U = c->U, NT = c->NT, W = c->W, H = c->H;
  const size_t N = (size_t)c->N;
  return make_map(&m->X, X, W, H, U, tile_box_w(), kTileH + 2) &&
         make_map(&m->T, v + 3 * N, W, H, NT, tile_box_w(), kTileH + 2) &&
         make_map(&m->R, v, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf);
}

static bool energy_maps(ls_ctx* c, const float* X, const float* D, EnergyMaps* m) {
  if (!c->use_tma) return false;
  const int U = c->U, W = c->W, H = c->H;
  bool ok = make_map(&m->X, X, W, H, U, tile_box_w(), kTileH + 2) &&
            make_map(&m->XR, X, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf);
  if (ok && D)
    ok = make_map(&m->D, D, W, H, U, tile_box_w(), kTileH + 2) &&
         make_map(&m->DR, D, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf);
  return ok;
}

static Launch L_energy(ls_ctx* c) { return Launch{c->grid_energy, c->ntiles, c->stream}; }
static Launch L_apply(ls_ctx* c) { return Launch{c->grid_apply, c->ntiles, c->stream}; }
static Launch L_update(ls_ctx* c) { return Launch{c->grid_update, 0, c->stream}; }

int ls_energy_terms(ls_ctx* c, const double* colors, const float* X, const float* Y, double* terms) {
  int rc = whole_frame_only(c);
  if (!rc) rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(colors || c->K == 0, "null palette");
  LS_ARG(X && Y && terms, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  EnergyMaps em;
  const bool tma = energy_maps(c, X, Y, &em);
  launch_energy(1, L_energy(c), frame_of(c), cd, X, nullptr, 0.f, Y, nullptr, nullptr, nullptr, nullptr, nullptr,
                nullptr, c->part, c->tickets + 0, c->sc, tma ? &em : nullptr);
  LS_CK(cudaGetLastError());
  LS_CK(cudaMemcpyAsync(c->sc_host, c->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  for (int j = 0; j < kTerms; ++j) terms[j] = c->sc_host->terms1[j];
  return LS_OK;
}

int ls_grad_diag(ls_ctx* c, const double* colors, const float* X, float* b, float* diag) {
  int rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(X && b && diag, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  EnergyMaps em;
  const bool tma = energy_maps(c, X, nullptr, &em);
  launch_energy(0, L_energy(c), frame_of(c), cd, X, nullptr, 0.f, nullptr, nullptr, nullptr, nullptr, nullptr, b,
                diag, c->part, c->tickets + 0, c->sc, tma ? &em : nullptr);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_apply_normal(ls_ctx* c, const double* colors, const float* X, const float* p, float* Ap) {
  int rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(X && p && Ap, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  const Coef<float> cf = make_coef<float>(c->w, colors, c->K);
  TileMaps maps;
  const bool tma = tile_maps(c, X, p, &maps);
  launch_apply(L_apply(c), frame_of(c), cf, X, p, Ap, c->part, c->tickets + 1, nullptr, 0, tma ? &maps : nullptr);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// ---- first-frame palette estimation (ls_palette.cu) ------------------------
int ls_estimate_palette(const float* image_hwc, int H, int W, int k_max, uint64_t st_hi, uint64_t st_lo,
                        uint64_t inc_hi, uint64_t inc_lo, double* colors_out, int* K_out, void* stream) {
  LS_ARG(image_hwc && colors_out && K_out && H > 0 && W > 0, "bad arguments");
  LS_ARG(k_max >= 1, "k_max must be >= 1");
  LS_ARG(k_max <= LS_MAX_K, "k_max above the supported palette size (12)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int N = H * W;
  float* img = nullptr;
  double* chroma = nullptr;
  char* scratch = nullptr;
  double* cols = nullptr;
  const size_t sb = palette_scratch_bytes();
  LS_CK(cudaMallocAsync((void**)&img, sizeof(float) * 3 * (size_t)N, s));
  LS_CK(cudaMallocAsync((void**)&chroma, sizeof(double) * 2 * (size_t)N, s));
  LS_CK(cudaMallocAsync((void**)&scratch, sb + sizeof(double) * 3 * LS_MAX_K + 64, s));
  cols = reinterpret_cast<double*>(scratch + sb);
  int* kdev = reinterpret_cast<int*>(scratch + sb + sizeof(double) * 3 * LS_MAX_K);
  launch_image(s, image_hwc, N, img, chroma);
  LS_CK(cudaGetLastError());
  LS_CK(launch_estimate_palette(s, img, chroma, N, k_max, PalRng{st_hi, st_lo, inc_hi, inc_lo}, scratch, cols,
                                kdev));
  int K = 0;
  LS_CK(cudaMemcpyAsync(&K, kdev, sizeof(int), cudaMemcpyDeviceToHost, s));
  LS_CK(cudaMemcpyAsync(colors_out, cols, sizeof(double) * 3 * k_max, cudaMemcpyDeviceToHost, s));
  LS_CK(cudaFreeAsync(img, s));
  LS_CK(cudaFreeAsync(chroma, s));
  LS_CK(cudaFreeAsync(scratch, s));
  LS_CK(cudaStreamSynchronize(s));
  *K_out = K;
  return LS_OK;
}

// ---- per-block residual protocol (ls_blocks.cu) ---------------------------
int ls_block_rows(ls_ctx* c, int block, int64_t n_pairs, int64_t* rows) {
  LS_ARG(c && rows && block >= 0 && block < BLK_COUNT && n_pairs >= 0, "bad arguments");
  *rows = block_rows(block, c->H, c->W, c->NT, n_pairs);
  return LS_OK;
}

static int block_common(ls_ctx* c, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                        BlockPairs* bp) {
  int rc = whole_frame_only(c);
  if (rc) return rc;
  LS_ARG(c->has_image, "no frame installed");
  LS_ARG(colors || c->K == 0, "null palette");
  LS_ARG(X0 && block >= 0 && block < BLK_COUNT, "bad arguments");
  *bp = BlockPairs{0, nullptr, nullptr, nullptr, nullptr};
  if (block == BLK_CONSISTENCY) {
    LS_ARG(pairs && pairs->n >= 0 && (pairs->n == 0 || (pairs->src && pairs->dst)), "consistency block needs pairs");
    *bp = BlockPairs{pairs->n, pairs->src, pairs->dst, pairs->temporal, pairs->weight};
  }
  LS_CK(cudaSetDevice(c->dev));
  return LS_OK;
}

int ls_block_residual(ls_ctx* c, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                      const float* Y, float* out) {
  BlockPairs bp;
  int rc = block_common(c, colors, X0, block, pairs, &bp);
  if (rc) return rc;
  LS_ARG(Y && out, "bad arguments");
  LS_ARG(block != BLK_CLUSTERING || c->has_ids || c->has_anchor, "EnergyAux needs cluster_ids or r_cluster_log");
  LS_ARG(block != BLK_CONSISTENCY || !bp.temporal || c->has_prev_r,
         "temporal partners need the previous frame's reflectance");
  LS_CK(launch_block_rows(c->stream, frame_of(c), make_coef<double>(c->w, colors, c->K), X0, bp, block, 0, Y, out));
  c->launches += 1;
  return LS_OK;
}

int ls_block_apply_j(ls_ctx* c, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                     const float* dX, float* out) {
  BlockPairs bp;
  int rc = block_common(c, colors, X0, block, pairs, &bp);
  if (rc) return rc;
  LS_ARG(dX && out, "bad arguments");
  LS_CK(launch_block_rows(c->stream, frame_of(c), make_coef<double>(c->w, colors, c->K), X0, bp, block, 1, dX, out));
  c->launches += 1;
  return LS_OK;
}

int ls_block_apply_jt(ls_ctx* c, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                      const float* w, float* out) {
  BlockPairs bp;
  int rc = block_common(c, colors, X0, block, pairs, &bp);
  if (rc) return rc;
  LS_ARG(w && out, "bad arguments");
  LS_CK(launch_block_cols(c->stream, frame_of(c), make_coef<double>(c->w, colors, c->K), X0, bp, block, 0, w, out));
  c->launches += block == BLK_CONSISTENCY ? 2 : 1;
  return LS_OK;
}

int ls_block_add_diag(ls_ctx* c, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                      float* out) {
  BlockPairs bp;
  int rc = block_common(c, colors, X0, block, pairs, &bp);
  if (rc) return rc;
  LS_ARG(out, "bad arguments");
  LS_CK(launch_block_cols(c->stream, frame_of(c), make_coef<double>(c->w, colors, c->K), X0, bp, block, 1, nullptr,
                          out));
  c->launches += block == BLK_CONSISTENCY ? 2 : 1;
  return LS_OK;
}

static bool pcg_maps(ls_ctx* c, const float* X, const float* pprev, PcgMaps* m) {
  if (!c->use_tma) return false;
  const int U = c->U, NT = c->NT, W = c->W, H = c->H;
  const size_t N = (size_t)c->N;
  return make_map(&m->X, X, W, H, U, tile_box_w(), kTileH + 2) &&
         make_map(&m->ZT, c->u + 3 * N, W, H, NT, tile_box_w(), kTileH + 2) &&
         make_map(&m->ZR, c->u, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf) &&
         make_map(&m->PT, pprev + 3 * N, W, H, NT, tile_box_w(), kTileH + 2) &&
         make_map(&m->PR, pprev, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf);
}

// single-reduction PCG (k_cg_iter): EG (r, dinv, u_0, gamma_0), then
// w_0 = A u_0, then one kernel per iteration.  Ping-pong buffers: u {u, r},
// m {wv, cg_m1}, t {s, cg_t1}; p in place.
static int run_pcg_cg1(ls_ctx* c, const double* colors, const float* X, int iters, float* x,
                       const FrameCtl* ctl) {
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  size_t pi = prof_begin(c);
  EnergyMaps em;
  const bool etma = energy_maps(c, X, nullptr, &em);
  launch_energy(0, L_energy(c), f, cd, X, nullptr, 0.f, nullptr, nullptr, c->r, c->d, c->u, nullptr, nullptr,
                c->part, c->tickets + 0, c->sc, etma ? &em : nullptr, ctl);
  prof_end(c, PC_EG, pi);
  const int W = c->W, H = c->H, U = c->U, NT = c->NT;
  const size_t N = (size_t)c->N;
  float* ub[2] = {c->u, c->r};
  float* mb[2] = {c->wv, c->cg_m1};
  float* tb[2] = {c->s, c->cg_t1};
  auto maps_for = [&](const float* uin, const float* min, const float* tin, CgMaps* m) {
    return make_map(&m->X, X, W, H, U, tile_box_w(), kTileH + 2) &&
           make_map(&m->UT, uin + 3 * N, W, H, NT, tile_box_w(), kTileH + 2) &&
           make_map(&m->UR, uin, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf) &&
           make_map(&m->MT, min + 3 * N, W, H, NT, tile_box_w(), kTileH + 2) &&
           make_map(&m->MR, min, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf) &&
           make_map(&m->TT, tin + 3 * N, W, H, NT, tile_box_w(), kTileH + 2) &&
           make_map(&m->TR, tin, W, H, 3, tile_box_rw(), kTileH + 2 * kHalf);
  };
  CgMaps maps[2];   // by iteration parity: u_i = ub[i&1], m_i = mb[i&1], t_{i-1} = tb[(i+1)&1]
  LS_ARG(maps_for(ub[0], mb[0], tb[1], &maps[0]) && maps_for(ub[1], mb[1], tb[0], &maps[1]),
         "TMA descriptors for the single-reduction PCG");
  const Launch Lc{c->grid_cg, c->ntiles, c->stream};
  pi = prof_begin(c);
  launch_cg(Lc, 0, f, cd, X, c->d, nullptr, mb[0], nullptr, c->p, x, c->part, c->tickets + 1, c->sc, 0, maps[0]);
  prof_end(c, PC_APPLY, pi);
  for (int it = 0; it < iters; ++it) {
    pi = prof_begin(c);
    launch_cg(Lc, it == iters - 1 ? 2 : 1, f, cd, X, c->d, ub[(it + 1) & 1], mb[(it + 1) & 1], tb[it & 1], c->p, x,
              c->part, c->tickets + 1, c->sc, it, maps[it & 1]);
    prof_end(c, PC_APPLY, pi);
  }
  launch_pcg_xfinal(L_update(c), (int64_t)U * c->N, x, c->p, c->s, c->sc, c->tickets + 4);   // no-op (pending = 0)
  c->launches += 3 + iters;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// fused energy/gradient + textbook PCG loop (solver.py:79-107); x receives the step.
// Buffers: r, d = 1/diag, u = z = r/diag, wv = q = A p, p / s = ping-pong p.
// the stored-direction buffers for a loop of `iters` iterations (outside captures)
static int ensure_pdirs(ls_ctx* c, int iters) {
  if (c->x_deferred || c->pcg_cg1 || iters < 1 || iters > kMaxStoredDirs) return LS_OK;
  const size_t M = (size_t)c->U * c->N;
  while ((int)c->pdirs.size() < iters) {
    float* b = nullptr;
    LS_CK(dalloc(c, &b, M));
    c->pdirs.push_back(b);
  }
  return LS_OK;
}

// the textbook loop with every search direction kept (p_i in its own
// buffer, 1.6 GB at 1080p K=8 for 16 iterations -- HBM is 180 GB): the
// operator kernel no longer carries the deferred x-update (the x read and
// write of every iteration and their exposed load latency), the last
// update computes only |r|, and one streaming pass k_pcg_combine forms
// x = sum alpha_i p_i in iteration order (the same fmaf chain, the same bits)
static int run_pcg_stored(ls_ctx* c, const double* colors, const float* X, int iters, float* x,
                          const FrameCtl* ctl) {
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  const int64_t M = (int64_t)c->U * c->N;
  if ((int)c->pdirs.size() < iters) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LS_CK(cudaStreamIsCapturing(c->stream, &cs));
    LS_ARG(cs == cudaStreamCaptureStatusNone, "PCG direction buffers must exist before a graph capture");
    while ((int)c->pdirs.size() < iters) {
      float* b = nullptr;
      LS_CK(dalloc(c, &b, (size_t)M));
      c->pdirs.push_back(b);
    }
  }
  size_t pi = prof_begin(c);
  EnergyMaps em;
  const bool etma = energy_maps(c, X, nullptr, &em);
  launch_energy(0, L_energy(c), f, cd, X, nullptr, 0.f, nullptr, nullptr, c->r, c->d, c->u, nullptr, nullptr,
                c->part, c->tickets + 0, c->sc, etma ? &em : nullptr, ctl);
  prof_end(c, PC_EG, pi);
  const Launch La{c->grid_pcg, c->ntiles, c->stream};
  DirList dl;
  std::memset(&dl, 0, sizeof(dl));
  dl.n = iters;
  for (int it = 0; it < iters; ++it) {
    float* pprev = c->pdirs[it > 0 ? it - 1 : 0];
    float* pnew = c->pdirs[it];
    dl.p[it] = pnew;
    PcgMaps maps;
    const bool tma = pcg_maps(c, X, pprev, &maps);
    pi = prof_begin(c);
    launch_pcg_apply(La, f, cd, X, c->u, pprev, pnew, c->wv, c->part, c->tickets + 1, c->sc, it,
                     tma ? &maps : nullptr, nullptr);
    prof_end(c, PC_APPLY, pi);
    pi = prof_begin(c);
    launch_pcg_update(L_update(c), M, c->r, c->wv, c->d, c->u, pnew, nullptr, c->part, c->tickets + 2, c->sc, it,
                      nullptr, it == iters - 1 ? 2 : 0);
    prof_end(c, PC_UPDATE, pi);
  }
  launch_pcg_combine(L_update(c), M, dl, x, c->sc);
  c->launches += 2 + 2LL * iters;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

static int run_pcg(ls_ctx* c, const double* colors, const float* X, int iters, float* x,
                   const FrameCtl* ctl = nullptr) {
  if (c->pcg_cg1 && !c->band_partial) return run_pcg_cg1(c, colors, X, iters, x, ctl);
  if (!c->x_deferred && !c->band_partial && iters >= 1 && iters <= kMaxStoredDirs)
    return run_pcg_stored(c, colors, X, iters, x, ctl);
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  size_t pi = prof_begin(c);
  EnergyMaps em;
  const bool etma = energy_maps(c, X, nullptr, &em);
  launch_energy(0, L_energy(c), f, cd, X, nullptr, 0.f, nullptr, nullptr, c->r, c->d, c->u, nullptr, nullptr,
                c->part, c->tickets + 0, c->sc, etma ? &em : nullptr, ctl);
  prof_end(c, PC_EG, pi);
  const int64_t M = (int64_t)c->U * c->N;
  float* pbuf[2] = {c->p, c->s};
  PcgMaps maps[2];
  const bool tma = pcg_maps(c, X, pbuf[1], &maps[0]) && pcg_maps(c, X, pbuf[0], &maps[1]);
  const Launch La{c->grid_pcg, c->ntiles, c->stream};
  for (int it = 0; it < iters; ++it) {
    pi = prof_begin(c);
    launch_pcg_apply(La, f, cd, X, c->u, pbuf[(it + 1) & 1], pbuf[it & 1], c->wv, c->part, c->tickets + 1, c->sc,
                     it, tma ? &maps[it & 1] : nullptr, x);
    prof_end(c, PC_APPLY, pi);
    pi = prof_begin(c);
    launch_pcg_update(L_update(c), M, c->r, c->wv, c->d, c->u, pbuf[it & 1], x, c->part, c->tickets + 2, c->sc, it,
                      nullptr, it == iters - 1 ? 1 : 0);
    prof_end(c, PC_UPDATE, pi);
  }
  // the last x += alpha p when the loop broke early (the applies fold in the
  // earlier ones, the final update the last one; otherwise a no-op)
  launch_pcg_xfinal(L_update(c), M, x, pbuf[0], pbuf[1], c->sc, c->tickets + 4);
  c->launches += 2 + 2LL * iters;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_pcg(ls_ctx* c, const double* colors, const float* X, int iterations, float* x, double* info) {
  int rc = whole_frame_only(c);
  if (!rc) rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(X && x && info && iterations >= 0, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  LS_CK(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)c->U * c->N, c->stream));
  rc = run_pcg(c, colors, X, iterations, x);
  if (rc) return rc;
  LS_CK(cudaMemcpyAsync(c->sc_host, c->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  info[0] = c->sc_host->iterations;
  info[1] = std::sqrt(c->sc_host->bnorm2);
  info[2] = std::sqrt(c->sc_host->rnorm2);
  return LS_OK;
}

static double sum_terms(const double* t) {
  double s = 0.0;   // Python sum() order over the blocks (solver.py:139-140)
  for (int j = 0; j < kTerms; ++j) s += t[j];
  return s;
}

int ls_gn_step(ls_ctx* c, const double* colors, const float* X, float* X_out, ls_gn_record* rec) {
  int rc = whole_frame_only(c);
  if (!rc) rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(X && X_out && rec && X != X_out, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  std::memset(rec, 0, sizeof(*rec));
  rc = run_pcg(c, colors, X, c->cfg.pcg_iterations, c->x);
  if (rc) return rc;
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  double alpha = 1.0;
  double e0 = 0.0, e1 = 0.0;
  bool accepted = false;
  EnergyMaps em;
  const bool etma = energy_maps(c, X, c->x, &em);
  for (int h = 0; h <= c->cfg.max_halvings; ++h) {
    const size_t pi = prof_begin(c);
    launch_energy(1, L_energy(c), f, cd, X, c->x, (float)alpha, nullptr, X_out, nullptr, nullptr, nullptr, nullptr,
                  nullptr, c->part, c->tickets + 0, c->sc, etma ? &em : nullptr);
    prof_end(c, PC_TRIAL, pi);
    c->launches += 1;
    LS_CK(cudaGetLastError());
    LS_CK(cudaMemcpyAsync(c->sc_host, c->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
    if (h == 0 && !c->sampled_counts_known)
      LS_CK(cudaMemcpyAsync(c->host_buf, &c->sstate->error, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    LS_CK(cudaStreamSynchronize(c->stream));
    prof_harvest(c);
    if (h == 0 && !c->sampled_counts_known && *reinterpret_cast<int*>(c->host_buf)) {
      g_err = "consistency sampler: too many PCG64 rejections in one frame";
      return LS_ERR_CUDA;
    }
    const Scalars& s = *c->sc_host;
    if (h == 0) {
      std::memcpy(rec->terms_before, s.terms0, sizeof(rec->terms_before));
      e0 = sum_terms(s.terms0);
      rec->energy_before = e0;
      rec->pcg_iterations = s.iterations;
      rec->initial_residual = std::sqrt(s.bnorm2);
      rec->final_residual = std::sqrt(s.rnorm2);
      if (!std::isfinite(e0)) {
        std::memcpy(rec->terms, s.terms0, sizeof(rec->terms));
        g_err = "non-finite residuals in sparse phase";
        return LS_ERR_NONFINITE;
      }
    }
    e1 = sum_terms(s.terms1);
    if (std::isfinite(e1) && e1 <= e0) {
      accepted = true;
      std::memcpy(rec->terms, s.terms1, sizeof(rec->terms));
      break;
    }
    alpha *= 0.5;
  }
  rec->accepted = accepted ? 1 : 0;
  rec->alpha = accepted ? alpha : 0.0;
  rec->energy_after = accepted ? e1 : e0;
  if (!accepted) std::memcpy(rec->terms, rec->terms_before, sizeof(rec->terms));
  return LS_OK;
}

// Graph conditional nodes for the line-search halvings (opt-in,
// LS_GRAPH_COND=1 at context creation: measured slower -- 61.6 / 62.0 vs
// 62.3 / 62.4 frames/s at 1080p K=8 in two A/B pairs; the conditional nodes
// cost the graph more than the 16 early-exit launches per frame they
// remove).  Under stream capture,
// trial h >= 1 is the body of an IF node whose handle trial h-1's last CTA
// sets (1 while the search is undecided); the handle defaults to 0 at every
// graph launch, so a decided search -- or a skipped predecessor -- skips the
// rest without launching them (the eager path launches them and they exit
// at once).  cond_open adds the node after the capture's current
// dependencies and redirects the context's launches into the body.
static int cond_open(ls_ctx* c, cudaGraphConditionalHandle h, cudaStream_t* saved) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  LS_CK(cudaStreamGetCaptureInfo(c->stream, &st, &id, &g, &deps, &nd));
  LS_ARG(st == cudaStreamCaptureStatusActive, "conditional node outside a capture");
  alignas(cudaGraphNodeParams) unsigned char pbuf[sizeof(cudaGraphNodeParams)];
  std::memset(pbuf, 0, sizeof(pbuf));      // (no default constructor: unions)
  cudaGraphNodeParams& p = *reinterpret_cast<cudaGraphNodeParams*>(pbuf);
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node = nullptr;
  LS_CK(cudaGraphAddNode(&node, g, deps, nd, &p));
  LS_CK(cudaStreamUpdateCaptureDependencies(c->stream, &node, 1, cudaStreamSetCaptureDependencies));
  if (!c->cond_stream) LS_CK(cudaStreamCreateWithFlags(&c->cond_stream, cudaStreamNonBlocking));
  LS_CK(cudaStreamBeginCaptureToGraph(c->cond_stream, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal));
  *saved = c->stream;
  c->stream = c->cond_stream;
  return LS_OK;
}

static int cond_close(ls_ctx* c, cudaStream_t saved) {
  cudaGraph_t body = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c->stream, &body);
  c->stream = saved;
  LS_CK(e);
  return LS_OK;
}

// Whole streaming flip-flop (solver.py:311-338 with refine = False) enqueued
// without host round trips: per GN step the EG kernel, the PCG, up to
// max_halvings+1 trial kernels deciding accept / halve on the device, and a
// step-end kernel; per outer iteration the convergence test; finally the
// device -> pinned-host copies of the control block and the step records.
// `bufs` are the three state buffers (bufs[0] holds the input).  Enqueue only
// (also used under stream capture for the CUDA-graph variant).
static int enqueue_flip_flop(ls_ctx* c, const double* colors, float* const bufs[3], int outer, int gn_steps,
                             double tol_rel, int* nsteps) {
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  const int64_t M = (int64_t)c->U * c->N;
  launch_frame_init(c->stream, c->ctl);
  c->launches += 1;
  int k = 0;
  for (int o = 0; o < outer; ++o) {
    for (int g = 0; g < gn_steps; ++g, ++k) {
      const int in_id = (k == 0) ? 0 : 1 + ((k - 1) & 1), out_id = 1 + (k & 1);
      const int rc = run_pcg(c, colors, bufs[in_id], c->cfg.pcg_iterations, c->x, c->ctl);
      if (rc) return rc;
      EnergyMaps em;
      const bool etma = energy_maps(c, bufs[in_id], c->x, &em);
      // under capture: trials 1.. as conditional nodes (handles made first:
      // each trial's kernel carries its successor's)
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      LS_CK(cudaStreamIsCapturing(c->stream, &cs));
      const bool cond = cs == cudaStreamCaptureStatusActive && c->use_cond && c->cfg.max_halvings > 0;
      std::vector<cudaGraphConditionalHandle> hs(c->cfg.max_halvings + 2, 0);
      if (cond) {
        cudaStreamCaptureStatus st;
        unsigned long long id = 0;
        cudaGraph_t g = nullptr;
        LS_CK(cudaStreamGetCaptureInfo(c->stream, &st, &id, &g, nullptr, nullptr));
        for (int h = 1; h <= c->cfg.max_halvings; ++h)
          LS_CK(cudaGraphConditionalHandleCreate(&hs[h], g, 0, cudaGraphCondAssignDefault));
      }
      double alpha = 1.0;
      for (int h = 0; h <= c->cfg.max_halvings; ++h, alpha *= 0.5) {
        cudaStream_t saved = nullptr;
        if (cond && h >= 1) {
          const int rc = cond_open(c, hs[h], &saved);
          if (rc) return rc;
        }
        const size_t pi = prof_begin(c);
        launch_energy(1, L_energy(c), f, cd, bufs[in_id], c->x, (float)alpha, nullptr, bufs[out_id], nullptr, nullptr,
                      nullptr, nullptr, nullptr, c->part, c->tickets + 0, c->sc, etma ? &em : nullptr, c->ctl, 1,
                      h == c->cfg.max_halvings, hs[h + 1]);
        prof_end(c, PC_TRIAL, pi);
        if (cond && h >= 1) {
          const int rc = cond_close(c, saved);
          if (rc) return rc;
        }
      }
      launch_step_end(c->stream, c->grid_update, c->ctl, c->sc, bufs[in_id], bufs[out_id], M, out_id, c->recs);
      c->launches += 2 + c->cfg.max_halvings;
    }
    launch_outer_end(c->stream, c->ctl, tol_rel);
    c->launches += 1;
  }
  LS_CK(cudaGetLastError());
  // records to mapped host memory by a kernel, not a copy engine (which may
  // be busy with the caller's large host transfers on another stream)
  launch_copy(c->stream, c->ctl_host, c->ctl, sizeof(FrameCtl));
  if (k > 0) launch_copy(c->stream, c->recs_host, c->recs, sizeof(StepRecord) * k);
  launch_copy(c->stream, c->host_buf, &c->sstate->error, sizeof(int));
  LS_CK(cudaGetLastError());
  *nsteps = k;
  return LS_OK;
}

// after the stream synchronisation: records, status, state buffer
static int finish_flip_flop(ls_ctx* c, ls_gn_record* out, int* n_records, int* status, int* final_buffer,
                            int* fault_step) {
  if (!c->sampled_counts_known && *reinterpret_cast<int*>(c->host_buf)) {
    g_err = "consistency sampler: too many PCG64 rejections in one frame";
    return LS_ERR_CUDA;
  }
  const FrameCtl& ctl = *c->ctl_host;
  for (int i = 0; i < ctl.n_exec; ++i) {
    const StepRecord& R = c->recs_host[i];
    ls_gn_record& o = out[i];
    o.energy_before = R.e0;
    o.energy_after = R.e1;
    o.alpha = R.alpha;
    o.accepted = R.accepted;
    o.pcg_iterations = R.iterations;
    o.initial_residual = std::sqrt(R.bnorm2);
    o.final_residual = std::sqrt(R.rnorm2);
    std::memcpy(o.terms_before, R.terms0, sizeof(o.terms_before));
    std::memcpy(o.terms, R.terms1, sizeof(o.terms));
  }
  *n_records = ctl.n_exec;
  *status = ctl.converged ? 2 : (ctl.stalled ? 1 : 0);
  *final_buffer = ctl.cur;
  *fault_step = ctl.fault_step;
  return ctl.fault_step >= 0 ? LS_ERR_NONFINITE : LS_OK;
}

extern "C" int ls_flip_flop_stream(ls_ctx* c, const double* colors, float* X0, float* X1, float* X2, int outer,
                                   int gn_steps, double tol_rel, ls_gn_record* out, int* n_records, int* status,
                                   int* final_buffer, int* fault_step) {
  int rc = whole_frame_only(c);
  if (!rc) rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(X0 && X1 && X2 && out && n_records && status && final_buffer && fault_step, "bad arguments");
  LS_ARG(outer >= 0 && gn_steps >= 0 && (int64_t)outer * gn_steps <= kMaxStepRecords, "too many GN steps");
  LS_CK(cudaSetDevice(c->dev));
  float* const bufs[3] = {X0, X1, X2};
  int k = 0;
  rc = enqueue_flip_flop(c, colors, bufs, outer, gn_steps, tol_rel, &k);
  if (rc) return rc;
  LS_CK(cudaStreamSynchronize(c->stream));
  prof_harvest(c);
  return finish_flip_flop(c, out, n_records, status, final_buffer, fault_step);
}

// Independent flip-flops over n contexts as one launch sequence
// (correction.py:168-201's K candidate solves): every context's whole
// flip-flop is enqueued on that context's own stream before any is waited
// for, so small solves (the candidates' bounding boxes) run side by side on
// the GPU; then one synchronisation per context.  Per-context results as
// ls_flip_flop_stream's, records at out + i * outer * gn_steps; rcs[i] is the
// context's own code (a failed candidate does not stop the others).
extern "C" int ls_flip_flop_batch(ls_ctx* const* ctxs, int n, const double* colors, float* const* X0,
                                  float* const* X1, float* const* X2, int outer, int gn_steps, double tol_rel,
                                  ls_gn_record* out, int* n_records, int* status, int* final_buffer,
                                  int* fault_step, int* rcs) {
  LS_ARG(ctxs && n >= 0 && X0 && X1 && X2 && out && n_records && status && final_buffer && fault_step && rcs,
         "bad arguments");
  LS_ARG(outer >= 0 && gn_steps >= 0 && (int64_t)outer * gn_steps <= kMaxStepRecords, "too many GN steps");
  const int per = outer * gn_steps;
  std::vector<char> live(n, 0);
  for (int i = 0; i < n; ++i) {
    ls_ctx* c = ctxs[i];
    n_records[i] = 0;
    status[i] = 0;
    final_buffer[i] = 0;
    fault_step[i] = -1;
    LS_ARG(c && X0[i] && X1[i] && X2[i], "bad arguments");
    LS_ARG(c->dev == ctxs[0]->dev, "contexts on different devices");
    for (int j = 0; j < i; ++j) LS_ARG(ctxs[j] != c, "a context appears twice in the batch");
  }
  LS_CK(cudaSetDevice(ctxs[0]->dev));
  // allocations first (cudaMalloc may synchronise the device)
  for (int i = 0; i < n; ++i) {
    int rc = whole_frame_only(ctxs[i]);
    if (!rc) rc = check_ready(ctxs[i]);
    if (!rc) rc = ensure_pdirs(ctxs[i], ctxs[i]->cfg.pcg_iterations);
    rcs[i] = rc;
  }
  for (int i = 0; i < n; ++i) {
    if (rcs[i]) continue;
    float* const bufs[3] = {X0[i], X1[i], X2[i]};
    int k = 0;
    rcs[i] = enqueue_flip_flop(ctxs[i], colors, bufs, outer, gn_steps, tol_rel, &k);
    live[i] = rcs[i] == LS_OK;
  }
  for (int i = 0; i < n; ++i) {
    if (!live[i]) continue;
    ls_ctx* c = ctxs[i];
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      g_err = std::string("CUDA: ") + cudaGetErrorString(e);
      rcs[i] = LS_ERR_CUDA;
      continue;
    }
    prof_harvest(c);
    rcs[i] = finish_flip_flop(c, out + (size_t)i * per, n_records + i, status + i, final_buffer + i,
                              fault_step + i);
  }
  return LS_OK;
}

// The same flip-flop as ONE CUDA graph launch.  The graph is captured once
// over context-owned state buffers (so every pointer it bakes in -- kernel
// arguments and TMA descriptors -- stays valid) and replayed while the
// palette, weights, configuration and per-frame buffers are unchanged (the
// streaming case: the palette is frozen after frame 1).  Per frame: copy
// X_in into the ring, launch, synchronise, copy the final state to X_out.
struct GraphKey {
  double colors[3 * LS_MAX_K];
  ls_weights w;
  ls_solve_cfg cfg;
  Frame f;
  int outer, gn_steps, use_tma, pad;
  double tol_rel;
  cudaStream_t stream;
};

static_assert(sizeof(GraphKey) <= 1024, "graph key buffer");

extern "C" int ls_flip_flop_graph(ls_ctx* c, const double* colors, const float* X_in, float* X_out, int outer,
                                  int gn_steps, double tol_rel, ls_gn_record* out, int* n_records, int* status,
                                  int* fault_step) {
  int rc = whole_frame_only(c);
  if (!rc) rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(X_in && X_out && out && n_records && status && fault_step, "bad arguments");
  LS_ARG(outer >= 0 && gn_steps >= 0 && (int64_t)outer * gn_steps <= kMaxStepRecords, "too many GN steps");
  LS_CK(cudaSetDevice(c->dev));
  const size_t bytes = sizeof(float) * (size_t)c->U * c->N;
  if (!c->ring[0])
    for (float*& r : c->ring) LS_CK(dalloc(c, &r, (size_t)c->U * c->N));
  rc = ensure_pdirs(c, c->cfg.pcg_iterations);
  if (rc) return rc;
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  for (int i = 0; i < 3 * c->K; ++i) key.colors[i] = colors[i];
  key.w = c->w;
  key.cfg = c->cfg;
  key.f = frame_of(c);
  key.outer = outer;
  key.gn_steps = gn_steps;
  key.use_tma = c->use_tma;
  key.tol_rel = tol_rel;
  key.stream = c->stream;
  const bool reuse = c->graph_exec && !c->prof.on && std::memcmp(&key, c->graph_key, sizeof(key)) == 0;
  launch_copy(c->stream, c->ring[0], X_in, bytes); LS_CK(cudaGetLastError());
  int k = 0;
  if (c->prof.on) {   // profiling records events around kernels: run eagerly
    rc = enqueue_flip_flop(c, colors, c->ring, outer, gn_steps, tol_rel, &k);
    if (rc) return rc;
  } else {
    if (!reuse) {
      if (c->graph_exec) {
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
      }
      const long long before = c->launches;
      cudaGraph_t g = nullptr;
      // capture on a private stream (the caller's may be the legacy default
      // stream, which cannot capture); the graph is launched on the caller's
      if (!c->cap_stream) LS_CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
      cudaStream_t user = c->stream;
      c->stream = c->cap_stream;
      cudaError_t be = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
      if (be != cudaSuccess) {
        c->stream = user;
        g_err = std::string("graph capture: ") + cudaGetErrorString(be);
        return LS_ERR_CUDA;
      }
      rc = enqueue_flip_flop(c, colors, c->ring, outer, gn_steps, tol_rel, &k);
      const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
      c->stream = user;
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ce != cudaSuccess) {
        g_err = std::string("graph capture: ") + cudaGetErrorString(ce);
        return LS_ERR_CUDA;
      }
      const cudaError_t ie = cudaGraphInstantiate(&c->graph_exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) {
        c->graph_exec = nullptr;
        g_err = std::string("graph instantiate: ") + cudaGetErrorString(ie);
        return LS_ERR_CUDA;
      }
      c->graph_launches = c->launches - before;
      c->graph_steps = k;
      c->launches = before;
      std::memcpy(c->graph_key, &key, sizeof(key));
    }
    k = c->graph_steps;
    LS_CK(cudaGraphLaunch(c->graph_exec, c->stream));
    c->launches += c->graph_launches;
  }
  LS_CK(cudaStreamSynchronize(c->stream));
  prof_harvest(c);
  int final_buffer = 0;
  rc = finish_flip_flop(c, out, n_records, status, &final_buffer, fault_step);
  launch_copy(c->stream, X_out, c->ring[final_buffer], bytes); LS_CK(cudaGetLastError());
  return rc;
}

static int dense_system(ls_ctx* c, const double* colors, const float* X, int use_ids) {
  LS_CK(cudaMemcpyAsync(c->colors_dev, colors, sizeof(double) * 3 * c->K, cudaMemcpyHostToDevice, c->stream));
  const size_t pi = prof_begin(c);
  launch_dense_accum(c->stream, c->grid_dense, frame_of(c), c->colors_dev, c->K, X, use_ids, c->part,
                     c->tickets + 3, c->dense_sums);
  prof_end(c, PC_DENSE, pi);
  c->launches += 2;
  launch_dense_assemble_solve(c->stream, c->dense_sums, c->K, c->colors_dev, use_ids, c->w.lambda_data,
                              c->w.lambda_clustering, c->w.lambda_ir, c->w.lambda_cr, c->w.chroma_reg,
                              c->cfg.svd_truncation, c->dense_A, c->dense_rhs, c->dense_x);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_dense_normal(ls_ctx* c, const double* colors, const float* X, int use_ids, double* A, double* rhs) {
  LS_ARG(c && c->has_image && colors && X && A && rhs, "bad arguments");
  LS_ARG(c->K >= 1, "dense system needs K >= 1");
  LS_ARG(!use_ids || c->has_ids, "no cluster ids set");
  LS_CK(cudaSetDevice(c->dev));
  int rc = dense_system(c, colors, X, use_ids);
  if (rc) return rc;
  const int n = 3 * c->K;
  LS_CK(cudaMemcpyAsync(c->host_buf, c->dense_A, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaMemcpyAsync(c->host_buf + n * n, c->dense_rhs, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  std::memcpy(A, c->host_buf, sizeof(double) * n * n);
  std::memcpy(rhs, c->host_buf + n * n, sizeof(double) * n);
  return LS_OK;
}

int ls_svd_solve(ls_ctx* c, int n, const double* A, const double* rhs, double trunc, double* x) {
  LS_ARG(c && A && rhs && x && n >= 1 && n <= 3 * LS_MAX_K, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  std::memcpy(c->host_buf, A, sizeof(double) * n * n);
  std::memcpy(c->host_buf + n * n, rhs, sizeof(double) * n);
  LS_CK(cudaMemcpyAsync(c->dense_A, c->host_buf, sizeof(double) * n * n, cudaMemcpyHostToDevice, c->stream));
  LS_CK(cudaMemcpyAsync(c->dense_rhs, c->host_buf + n * n, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  launch_svd_solve(c->stream, n, c->dense_A, c->dense_rhs, trunc, c->dense_x);
  LS_CK(cudaGetLastError());
  LS_CK(cudaMemcpyAsync(c->host_buf, c->dense_x, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  std::memcpy(x, c->host_buf, sizeof(double) * n);
  return LS_OK;
}

int ls_dense_step(ls_ctx* c, double* colors, const float* X, double* applied, ls_dense_record* rec) {
  int rc = whole_frame_only(c);
  if (!rc) rc = check_ready(c);
  if (rc) return rc;
  LS_ARG(colors && X && applied && rec, "bad arguments");
  LS_ARG(c->K >= 1, "dense step needs K >= 1");
  LS_CK(cudaSetDevice(c->dev));
  std::memset(rec, 0, sizeof(*rec));
  const int K = c->K, n = 3 * K;
  rc = dense_system(c, colors, X, c->has_ids ? 1 : 0);
  if (rc) return rc;
  LS_CK(cudaMemcpyAsync(c->host_buf, c->dense_x, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  std::vector<double> db(c->host_buf, c->host_buf + n);
  for (int i = 0; i < n; ++i) applied[i] = 0.0;
  bool any = false;
  double big = 0.0;
  for (double v : db) {
    any = any || v != 0.0;
    big = std::max(big, std::fabs(v));
  }
  if (!any) return LS_OK;   // solver.py:218-219: no record
  rec->solved_nonzero = 1;
  if (big > c->cfg.max_delta_b)
    for (double& v : db) v = v * (c->cfg.max_delta_b / big);
  const Frame f = frame_of(c);
  auto energy_with = [&](const double* cols, double* out) -> int {
    const Coef<float> cd = make_coef<float>(c->w, cols, K);
    EnergyMaps em;
    const bool etma = energy_maps(c, X, nullptr, &em);
    launch_energy(1, L_energy(c), f, cd, X, nullptr, 0.f, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                  nullptr, c->part, c->tickets + 0, c->sc, etma ? &em : nullptr);
    c->launches += 1;
    LS_CK(cudaGetLastError());
    LS_CK(cudaMemcpyAsync(c->sc_host, c->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
    LS_CK(cudaStreamSynchronize(c->stream));
    prof_harvest(c);
    *out = sum_terms(c->sc_host->terms1);
    return LS_OK;
  };
  double e0 = 0.0;
  if ((rc = energy_with(colors, &e0))) return rc;
  double alpha = 1.0, e1 = e0;
  bool accepted = false;
  std::vector<double> cand(n);
  for (int h = 0; h <= c->cfg.max_halvings; ++h) {
    for (int i = 0; i < n; ++i) cand[i] = std::min(1.0, std::max(0.0, colors[i] + alpha * db[i]));
    double et = 0.0;
    if ((rc = energy_with(cand.data(), &et))) return rc;
    if (std::isfinite(et) && et <= e0) {
      double nrm = 0.0;
      for (int i = 0; i < n; ++i) {
        applied[i] = cand[i] - colors[i];
        nrm += applied[i] * applied[i];
        colors[i] = cand[i];
      }
      rec->delta_b_norm = std::sqrt(nrm);
      e1 = et;
      accepted = true;
      break;
    }
    alpha *= 0.5;
  }
  rec->energy_before = e0;
  rec->energy_after = accepted ? e1 : e0;
  rec->accepted = accepted ? 1 : 0;
  rec->alpha = accepted ? alpha : 0.0;
  return LS_OK;
}


// ---------------------------------------------------------------------------
// Row bands: one context per band of
// rows, every reduction written as a band partial and finalised from the
// band-ordered sum of all bands' partials (gathered by the host: a local
// copy on one GPU, an NCCL all-gather across GPUs).  Halo rows are refreshed
// by the host between the calls (ls_band_buffers).
// ---------------------------------------------------------------------------
static int band_ready(ls_ctx* c) {
  LS_ARG(c && c->band_partial, "not a row band (ls_band_set first)");
  return check_ready(c);
}

int ls_band_set(ls_ctx* c, int gy0, int GH, int y_lo, int y_hi) {
  LS_ARG(c, "null context");
  LS_ARG(0 <= y_lo && y_lo < y_hi && y_hi <= c->H, "band rows must satisfy 0 <= y_lo < y_hi <= H");
  LS_ARG(gy0 >= 0 && (int64_t)gy0 + c->H <= GH, "band outside the frame");
  LS_ARG(c->W % 4 == 0, "row bands need W % 4 == 0");
  c->gy0 = gy0;
  c->GH = GH;
  c->y_lo = y_lo;
  c->y_hi = y_hi;
  c->band_partial = true;
  set_geometry(c);
  return LS_OK;
}

int ls_band_clear(ls_ctx* c) {
  LS_ARG(c, "null context");
  c->gy0 = 0;
  c->GH = c->H;
  c->y_lo = 0;
  c->y_hi = c->H;
  c->band_partial = false;
  set_geometry(c);
  return LS_OK;
}

int ls_band_buffers(ls_ctx* c, void** out) {
  LS_ARG(c && out, "bad arguments");
  out[0] = c->bsum;
  out[1] = c->u;
  out[2] = c->p;
  out[3] = c->s;
  out[4] = c->x;
  out[5] = c->r;
  return LS_OK;
}

int ls_band_dirs(ls_ctx* c, int n, void** out) {
  LS_ARG(c && c->band_partial && out && n >= 1 && n <= kMaxStoredDirs, "bad arguments");
  LS_ARG(!c->x_deferred && !c->pcg_cg1, "stored PCG directions are off in this context");
  LS_CK(cudaSetDevice(c->dev));
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  LS_CK(cudaStreamIsCapturing(c->stream, &cs));
  LS_ARG(cs == cudaStreamCaptureStatusNone || (int)c->pdirs.size() >= n,
         "PCG direction buffers must exist before a graph capture");
  const int rc = ensure_pdirs(c, n);
  if (rc) return rc;
  for (int i = 0; i < n; ++i) out[i] = c->pdirs[i];
  c->band_stored = true;
  return LS_OK;
}

int ls_band_zero_scan(ls_ctx* c, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, uint64_t begin,
                      uint64_t end, int64_t* list) {
  LS_ARG(c && list && end >= begin, "bad arguments");
  LS_CK(cudaSetDevice(c->dev));
  SampleParams P;
  std::memset(&P, 0, sizeof(P));
  P.st_hi = st_hi;
  P.st_lo = st_lo;
  P.inc_hi = inc_hi;
  P.inc_lo = inc_lo;
  launch_zero_scan(c->stream, P, begin, end, reinterpret_cast<long long*>(list));
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_set_zeros(ls_ctx* c, const int64_t* lists, int n_lists) {
  LS_ARG(c && lists && n_lists >= 1, "bad arguments");
  c->band_zeros = reinterpret_cast<const long long*>(lists);
  c->band_zero_lists = n_lists;
  return LS_OK;
}

int ls_band_eg(ls_ctx* c, const double* colors, const float* X) {
  int rc = band_ready(c);
  if (rc) return rc;
  LS_ARG(X, "bad arguments");
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  EnergyMaps em;
  const bool etma = energy_maps(c, X, nullptr, &em);
  const size_t pi = prof_begin(c);
  launch_energy(0, L_energy(c), f, cd, X, nullptr, 0.f, nullptr, nullptr, c->r, c->d, c->u, nullptr, nullptr,
                c->part, c->tickets + 0, c->sc, etma ? &em : nullptr, c->band_dev ? c->ctl : nullptr);
  prof_end(c, PC_EG, pi);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_pcg_apply(ls_ctx* c, const double* colors, const float* X, int iter) {
  int rc = band_ready(c);
  if (rc) return rc;
  LS_ARG(X && iter >= 0, "bad arguments");
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  float* pbuf[2] = {c->p, c->s};
  // stored directions (ls_band_dirs): p_iter into its own buffer, no
  // deferred x-update in the operator -- x = sum alpha_i p_i in ls_band_pcg_finish
  const bool stored = c->band_stored && iter < (int)c->pdirs.size();
  float* pprev = stored ? c->pdirs[iter > 0 ? iter - 1 : 0] : pbuf[(iter + 1) & 1];
  float* pnew = stored ? c->pdirs[iter] : pbuf[iter & 1];
  PcgMaps maps;
  const bool tma = pcg_maps(c, X, pprev, &maps);
  const Launch La{c->grid_pcg, c->ntiles, c->stream};
  const size_t pi = prof_begin(c);
  launch_pcg_apply(La, f, cd, X, c->u, pprev, pnew, c->wv, c->part, c->tickets + 1, c->sc, iter,
                   tma ? &maps : nullptr, stored ? nullptr : c->x);
  prof_end(c, PC_APPLY, pi);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_pcg_update(ls_ctx* c, int iter) {
  int rc = band_ready(c);
  if (rc) return rc;
  LS_ARG(iter >= 0, "bad arguments");
  const Frame f = frame_of(c);
  float* pbuf[2] = {c->p, c->s};
  const int64_t M = (int64_t)c->U * c->N;
  const size_t pi = prof_begin(c);
  const bool stored = c->band_stored && iter < (int)c->pdirs.size();
  launch_pcg_update(L_update(c), M, c->r, c->wv, c->d, c->u, stored ? c->pdirs[iter] : pbuf[iter & 1],
                    stored ? nullptr : c->x, c->part, c->tickets + 2, c->sc, iter, &f);
  prof_end(c, PC_UPDATE, pi);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_pcg_finish(ls_ctx* c) {
  int rc = band_ready(c);
  if (rc) return rc;
  const Frame f = frame_of(c);
  if (c->band_stored && !c->pdirs.empty()) {   // x = sum alpha_i p_i over the whole local rows
    DirList dl;
    std::memset(&dl, 0, sizeof(dl));
    dl.n = std::min<int>((int)c->pdirs.size(), kMaxStoredDirs);
    for (int i = 0; i < dl.n; ++i) dl.p[i] = c->pdirs[i];
    launch_pcg_combine(L_update(c), (int64_t)c->U * c->N, dl, c->x, c->sc);
  } else {
    launch_pcg_xfinal(L_update(c), (int64_t)c->U * c->N, c->x, c->p, c->s, c->sc, c->tickets + 4, &f);
  }
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_trial(ls_ctx* c, const double* colors, const float* X, double alpha, float* X_out) {
  int rc = band_ready(c);
  if (rc) return rc;
  LS_ARG(X, "bad arguments");
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  EnergyMaps em;
  const float* dx = X_out ? c->x : nullptr;   // X_out == NULL: energies at X itself
  const bool etma = energy_maps(c, X, dx, &em);
  const size_t pi = prof_begin(c);
  launch_energy(1, L_energy(c), f, cd, X, dx, (float)alpha, nullptr, X_out, nullptr, nullptr, nullptr, nullptr,
                nullptr, c->part, c->tickets + 0, c->sc, etma ? &em : nullptr);
  prof_end(c, PC_TRIAL, pi);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_finalize(ls_ctx* c, int phase, const double* gathered, int nbands, int iter, double alpha) {
  LS_ARG(c && c->band_partial && gathered && nbands >= 1, "bad arguments");
  LS_ARG(phase >= BAND_EG && phase <= BAND_TRIAL, "bad band phase");
  const int nv = phase == BAND_EG ? kTerms + 2 : phase == BAND_APPLY ? 1 : phase == BAND_UPDATE ? 2 : kTerms;
  launch_band_finalize(c->stream, phase, gathered, nbands, nv, c->sc, iter, (float)alpha, 0, 0);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// ---- device-resident band flip-flop (the band form of ls_flip_flop_stream):
// every decision (line search, step bookkeeping, convergence) on the device,
// identical on every band, so the whole frame can be one CUDA graph (NCCL
// collectives and P2P copies included).
int ls_band_frame_begin(ls_ctx* c) {
  int rc = band_ready(c);
  if (rc) return rc;
  launch_frame_init(c->stream, c->ctl);
  c->band_dev = true;
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_trial_dev(ls_ctx* c, const double* colors, const float* X, double alpha, float* X_out, int last) {
  int rc = band_ready(c);
  if (rc) return rc;
  LS_ARG(X && X_out && c->band_dev, "bad arguments (ls_band_frame_begin first)");
  const Frame f = frame_of(c);
  const Coef<float> cd = make_coef<float>(c->w, colors, c->K);
  EnergyMaps em;
  const bool etma = energy_maps(c, X, c->x, &em);
  const size_t pi = prof_begin(c);
  launch_energy(1, L_energy(c), f, cd, X, c->x, (float)alpha, nullptr, X_out, nullptr, nullptr, nullptr, nullptr,
                nullptr, c->part, c->tickets + 0, c->sc, etma ? &em : nullptr, c->ctl, 1, last);
  prof_end(c, PC_TRIAL, pi);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_finalize_dev(ls_ctx* c, int phase, const double* gathered, int nbands, int iter, double alpha,
                         int last) {
  LS_ARG(c && c->band_partial && c->band_dev && gathered && nbands >= 1, "bad arguments");
  LS_ARG(phase >= BAND_EG && phase <= BAND_TRIAL, "bad band phase");
  const int nv = phase == BAND_EG ? kTerms + 2 : phase == BAND_APPLY ? 1 : phase == BAND_UPDATE ? 2 : kTerms;
  launch_band_finalize(c->stream, phase, gathered, nbands, nv, c->sc, iter, (float)alpha, 1, last, c->ctl);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// all bands of this process at once (in-process row bands: the gather is a
// read of the other bands' partial sums, no copies)
extern "C" int ls_band_finalize_group(ls_ctx* const* ctxs, int n, int phase, int iter, double alpha, int last) {
  LS_ARG(ctxs && n >= 1 && n <= kMaxGroupBands, "bad arguments");
  LS_ARG(phase >= BAND_EG && phase <= BAND_TRIAL, "bad band phase");
  BandGroup g;
  std::memset(&g, 0, sizeof(g));
  g.n = n;
  for (int i = 0; i < n; ++i) {
    ls_ctx* c = ctxs[i];
    LS_ARG(c && c->band_partial && c->band_dev && c->dev == ctxs[0]->dev, "bad band context");
    g.bsum[i] = c->bsum;
    g.sc[i] = c->sc;
    g.ctl[i] = c->ctl;
  }
  const int nv = phase == BAND_EG ? kTerms + 2 : phase == BAND_APPLY ? 1 : phase == BAND_UPDATE ? 2 : kTerms;
  launch_band_finalize_group(ctxs[0]->stream, phase, g, nv, iter, (float)alpha, last);
  ctxs[0]->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

// strided slab copies in one launch (halo moves between in-process bands)
extern "C" int ls_copy_slabs(int n, const float* const* src, float* const* dst, const int64_t* src_stride,
                             const int64_t* dst_stride, const int64_t* count, const int* planes, void* stream) {
  LS_ARG(n >= 0 && n <= kMaxSlabs, "too many slabs");
  LS_ARG(n == 0 || (src && dst && src_stride && dst_stride && count && planes), "bad arguments");
  SlabList L;
  std::memset(&L, 0, sizeof(L));
  L.n = n;
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    LS_ARG(src[i] && dst[i] && count[i] >= 0 && planes[i] >= 0, "bad slab");
    L.s[i] = Slab{src[i], dst[i], src_stride[i], dst_stride[i], count[i], planes[i]};
    total = std::max<int64_t>(total, count[i] * planes[i]);
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
  launch_copy_slabs((cudaStream_t)stream, L, grid);
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_step_end(ls_ctx* c, const float* X_in, float* X_out, int out_id) {
  LS_ARG(c && c->band_dev && X_in && X_out, "bad arguments");
  launch_step_end(c->stream, c->grid_update, c->ctl, c->sc, X_in, X_out, (int64_t)c->U * c->N, out_id, c->recs);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_outer_end(ls_ctx* c, double tol_rel) {
  LS_ARG(c && c->band_dev, "bad arguments");
  launch_outer_end(c->stream, c->ctl, tol_rel);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_frame_end(ls_ctx* c, int nsteps, ls_gn_record* out, int* n_records, int* status, int* final_buffer,
                      int* fault_step) {
  LS_ARG(c && c->band_partial && out && n_records && status && final_buffer && fault_step, "bad arguments");
  LS_ARG(nsteps >= 0 && nsteps <= kMaxStepRecords, "bad step count");   // (band_dev is host state of
  // the enqueue; a CUDA-graph replay runs without it)
  c->band_dev = false;
  launch_copy(c->stream, c->ctl_host, c->ctl, sizeof(FrameCtl));
  if (nsteps > 0) launch_copy(c->stream, c->recs_host, c->recs, sizeof(StepRecord) * nsteps);
  launch_copy(c->stream, c->host_buf, &c->sstate->error, sizeof(int));
  LS_CK(cudaGetLastError());
  LS_CK(cudaStreamSynchronize(c->stream));
  prof_harvest(c);
  return finish_flip_flop(c, out, n_records, status, final_buffer, fault_step);
}

int ls_band_read(ls_ctx* c, double* out) {
  LS_ARG(c && out, "bad arguments");
  LS_CK(cudaMemcpyAsync(c->sc_host, c->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  prof_harvest(c);
  const Scalars& s = *c->sc_host;
  for (int j = 0; j < kTerms; ++j) {
    out[j] = s.terms0[j];
    out[kTerms + j] = s.terms1[j];
  }
  out[16] = s.bnorm2;
  out[17] = s.rnorm2;
  out[18] = s.iterations;
  out[19] = s.stop;
  out[20] = s.xinit;
  return LS_OK;
}

int ls_band_dense_accum(ls_ctx* c, const double* colors, const float* X, int use_ids) {
  LS_ARG(c && c->band_partial && c->has_image && colors && X, "bad arguments");
  LS_ARG(c->K >= 1, "dense system needs K >= 1");
  LS_ARG(!use_ids || c->has_ids, "no cluster ids set");
  LS_CK(cudaMemcpyAsync(c->colors_dev, colors, sizeof(double) * 3 * c->K, cudaMemcpyHostToDevice, c->stream));
  const size_t pi = prof_begin(c);
  launch_dense_accum(c->stream, c->grid_dense, frame_of(c), c->colors_dev, c->K, X, use_ids, c->part,
                     c->tickets + 3, c->bsum);
  prof_end(c, PC_DENSE, pi);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_dense_nsums(ls_ctx* c) { return c ? dense_nsums(c->K) : 0; }

int ls_band_dense_solve(ls_ctx* c, const double* colors, const double* gathered, int nbands, int use_ids,
                        double* dx) {
  LS_ARG(c && colors && gathered && dx && nbands >= 1, "bad arguments");
  LS_ARG(c->K >= 1, "dense system needs K >= 1");
  const int n = 3 * c->K;
  LS_CK(cudaMemcpyAsync(c->colors_dev, colors, sizeof(double) * 3 * c->K, cudaMemcpyHostToDevice, c->stream));
  launch_band_sum(c->stream, gathered, nbands, dense_nsums(c->K), c->dense_sums);
  launch_dense_assemble_solve(c->stream, c->dense_sums, c->K, c->colors_dev, use_ids, c->w.lambda_data,
                              c->w.lambda_clustering, c->w.lambda_ir, c->w.lambda_cr, c->w.chroma_reg,
                              c->cfg.svd_truncation, c->dense_A, c->dense_rhs, c->dense_x);
  c->launches += 2;
  LS_CK(cudaGetLastError());
  LS_CK(cudaMemcpyAsync(c->host_buf, c->dense_x, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  LS_CK(cudaStreamSynchronize(c->stream));
  std::memcpy(dx, c->host_buf, sizeof(double) * n);
  return LS_OK;
}

int ls_band_segment(ls_ctx* c, const double* colors, int32_t* summary) {
  LS_ARG(c && c->has_image && colors && summary, "bad arguments");
  LS_ARG(c->K >= 1, "segment needs K >= 1");
  const int N = c->N, K = c->K;
  PalChroma pc;
  std::memset(&pc, 0, sizeof(pc));
  for (int k = 0; k < K; ++k) {   // chroma_of_color (imaging.py:174-180)
    const double s = (colors[3 * k] + colors[3 * k + 1]) + colors[3 * k + 2];
    pc.c[2 * k] = s > 1e-12 ? colors[3 * k] / s : 1.0 / 3.0;
    pc.c[2 * k + 1] = s > 1e-12 ? colors[3 * k + 1] / s : 1.0 / 3.0;
  }
  const int own_lo = c->y_lo * c->W, own_hi = c->y_hi * c->W;
  launch_set_i32(c->stream, c->small_i + 2, 1, N);
  launch_segment_band(c->stream, c->img, c->chroma, N, K, pc, c->seg_raw, c->seg_key, c->small_i + 2, own_lo, own_hi);
  LS_CK(launch_scan(c->stream, c->seg_key, c->seg_last, (int64_t)N, 1, c->cub_tmp));
  launch_segment_summary(c->stream, c->seg_raw, c->seg_last, c->small_i + 2, own_hi, summary);
  c->launches += 4;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

int ls_band_segment_final(ls_ctx* c, const int32_t* summaries, int nbands, int band, int32_t* ids_out) {
  LS_ARG(c && summaries && ids_out && nbands >= 1 && band >= 0 && band < nbands, "bad arguments");
  launch_segment_band_final(c->stream, c->N, c->seg_raw, c->seg_last, summaries, nbands, band, c->y_lo * c->W,
                            c->y_hi * c->W, ids_out);
  c->launches += 1;
  LS_CK(cudaGetLastError());
  return LS_OK;
}

}  // extern "C"
