// Internal launcher declarations shared by the .cu translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ls_common.cuh"

namespace ls {

// TMA descriptors of one tile (built on the host per operand buffer):
//   X  state planes,   box {kSW, kTileH+2, U}   at (tx0-1, ty0-1, 0)
//   T  operand T part,  box {kSW, kTileH+2, NT}  at (tx0-1, ty0-1, 0)
//   R  operand r part,  box {kRW, kTileH+14, 3}  at (tx0-7, ty0-7, 0)
struct TileMaps {
  CUtensorMap X, T, R;
};

// energy kernels: state X (1 halo, U planes; r planes 7 halo) and the second
// operand D = dx or an external Y (same two boxes)
struct EnergyMaps {
  CUtensorMap X, XR, D, DR;
};

// textbook-PCG operator kernel: state X, operand z (T 1 halo, r 7 halo) and
// the previous search direction p (same two boxes)
struct PcgMaps {
  CUtensorMap X, ZT, ZR, PT, PR;
};

// single-reduction PCG (k_cg_iter): state X, operands u (T 1 halo, r 7 halo),
// m and t (same boxes)
struct CgMaps {
  CUtensorMap X, UT, UR, MT, MR, TT, TR;
};

struct Launch {
  int grid;
  int ntiles;
  cudaStream_t stream;
};

// ls_solver.cu
void launch_energy(int mode, const Launch& L, const Frame& f, const Coef<float>& c, const float* X,
                   const float* dx, float alpha, const float* Y, float* Xout, float* r_out, float* d_out,
                   float* u_out, float* b_raw, float* diag_raw, double* part, unsigned* ticket, Scalars* sc,
                   const EnergyMaps* maps, const FrameCtl* ctl = nullptr, int dev_ls = 0, int last_trial = 0,
                   unsigned long long next_cond = 0);   // a trial's successor's graph conditional handle
void launch_frame_init(cudaStream_t s, FrameCtl* ctl);
void launch_step_end(cudaStream_t s, int grid, FrameCtl* ctl, const Scalars* sc, const float* Xin, float* Xout,
                     int64_t M, int out_id, StepRecord* recs);
void launch_outer_end(cudaStream_t s, FrameCtl* ctl, double tol_rel);
void launch_apply(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* u,
                  float* w, double* part, unsigned* ticket, Scalars* sc, int iter, const TileMaps* maps);
int tile_box_w();
int tile_box_rw();
void launch_pcg_apply(const Launch& L, const Frame& f, const Coef<float>& c, const float* X, const float* z,
                      const float* pprev, float* pnew, float* q, double* part, unsigned* ticket, Scalars* sc,
                      int iter, const PcgMaps* maps, float* x);
// last (whole frames only): 1 = the final iteration also folds in the last
// deferred x += alpha p (p = this iteration's direction) and skips z;
// 2 = the final iteration computes only |r| (the stored directions are
// combined into x by launch_pcg_combine)
void launch_pcg_update(const Launch& L, int64_t M, float* r, const float* q, const float* dinv, float* z,
                       const float* p, float* xv, double* part, unsigned* ticket, Scalars* sc, int iter,
                       const Frame* band = nullptr, int last = 0);
// the stored search directions p_0 .. p_{n-1} of one PCG loop
struct DirList {
  const float* p[kMaxStoredDirs];
  int n;
};
void launch_pcg_combine(const Launch& L, int64_t M, const DirList& dl, float* xv, Scalars* sc);
void launch_pcg_xfinal(const Launch& L, int64_t M, float* xv, const float* p0, const float* p1, Scalars* sc,
                       unsigned* ticket, const Frame* band = nullptr);
// single-reduction PCG: mode 0 init (w_0 = A u_0), 1 iteration, 2 last iteration
void launch_cg(const Launch& L, int mode, const Frame& f, const Coef<float>& c, const float* X, const float* dinv,
               float* u_out, float* m_out, float* t_out, float* p, float* xv, double* part, unsigned* ticket,
               Scalars* sc, int iter, const CgMaps& maps);
int cg_grid_limit(int NT);
// row bands: phases whose partial sums are gathered across bands
enum BandPhase { BAND_EG = 0, BAND_APPLY = 1, BAND_UPDATE = 2, BAND_TRIAL = 3, BAND_DENSE = 4 };
void launch_band_sum(cudaStream_t s, const double* gathered, int nbands, int nv, double* out);
void launch_band_finalize(cudaStream_t s, int phase, const double* gathered, int nbands, int nv, Scalars* sc,
                          int iter, float alpha, int dev_ls, int last_trial, const FrameCtl* ctl = nullptr);
// the bands of one process finalised together (k_band_finalize_group)
constexpr int kMaxGroupBands = 16;
struct BandGroup {
  const double* bsum[kMaxGroupBands];
  Scalars* sc[kMaxGroupBands];
  const FrameCtl* ctl[kMaxGroupBands];
  int n;
};
void launch_band_finalize_group(cudaStream_t s, int phase, const BandGroup& g, int nv, int iter, float alpha,
                                int last_trial);
// strided slab copies (halo moves) in one launch
constexpr int kMaxSlabs = 32;
struct Slab {
  const float* src;
  float* dst;
  int64_t src_stride, dst_stride, count;
  int planes;
};
struct SlabList {
  Slab s[kMaxSlabs];
  int n;
};
void launch_copy_slabs(cudaStream_t s, const SlabList& L, int grid);
int pcg_apply_grid_limit(int NT);
int energy_grid_limit(int NT);
void prepare_kernels(int NT);
int apply_grid_limit(int NT);
int update_grid_limit();

// ls_blocks.cu: the reference's per-block residual protocol (energy.py:194-452)
enum BlockId { BLK_DATA = 0, BLK_CLUSTERING, BLK_RSPARSITY, BLK_CONSISTENCY, BLK_MONOCHROME, BLK_ISPARSITY,
               BLK_SMOOTHNESS, BLK_NONNEG, BLK_COUNT };
struct BlockPairs {
  int64_t n;
  const int64_t* src;
  const int64_t* dst;
  const uint8_t* temporal;   // may be null (all spatial)
  const double* weight;      // may be null (all 1)
};
int64_t block_rows(int block, int H, int W, int NT, int64_t n_pairs);
// op 0: residual at Y, op 1: J Y (Y a direction); out has block_rows rows
cudaError_t launch_block_rows(cudaStream_t s, const Frame& f, const Coef<double>& c, const float* X0,
                              const BlockPairs& pairs, int block, int op, const float* Y, float* out);
// op 0: out += J^T w, op 1: out += diag(J^T J); out is U planes
cudaError_t launch_block_cols(cudaStream_t s, const Frame& f, const Coef<double>& c, const float* X0,
                              const BlockPairs& pairs, int block, int op, const float* w, float* out);

// ls_palette.cu: first-frame palette estimation (palette.py:81-238)
struct PalRng {   // numpy PCG64 state of default_rng(seed) (Generator.choice draw)
  unsigned long long st_hi, st_lo, inc_hi, inc_lo;
};
size_t palette_scratch_bytes();
cudaError_t launch_estimate_palette(cudaStream_t s, const float* img, const double* chroma, int N, int k_max,
                                    const PalRng& rng, void* scratch, double* out_colors, int* out_k);

// ls_aux.cu
// int32 scan (op 0: exclusive sum, op 1: inclusive max) of n values; scratch
// of scan_scratch_bytes(n) bytes (zeroed by the launcher on the stream)
size_t scan_scratch_bytes(int64_t n);
cudaError_t launch_scan(cudaStream_t s, const int32_t* in, int32_t* out, int64_t n, int op, void* scratch);
constexpr int kJumpBits = 40;   // stream positions < 2^41 u32 words
struct SampleParams {
  unsigned long long st_hi, st_lo, inc_hi, inc_lo;
  int has_prev;
  // row bands: local pixel 0 is global flat pixel goff of a GH x W frame
  // with Ng pixels (the PCG64 stream is indexed by global pixel)
  int gy0, GH;
  long long goff, Ng;
  // jump table of the LCG (filled by the launchers): 2^k steps are
  // s -> M_k s + C_k, as {M_k hi, M_k lo, C_k hi, C_k lo}
  unsigned long long jump[kJumpBits][4];
};
constexpr int kMaxRejections = 16;
// device-resident rejection bookkeeping of the partner sampler
struct SampleState {
  int nz, redo, error, pad;
  unsigned long long new_zero;
  long long z[kMaxRejections];   // rejected u32 stream positions, ascending
};
constexpr int kSamplePasses = 4;
constexpr int kMaxStepRecords = 256;
void launch_copy(cudaStream_t s, void* dst, const void* src, int64_t bytes);
// correction / edits (ls_edit.cu)
struct EditParams {
  double B[3 * kMaxNT];   // palette matrix rows (white, b_1..b_K), possibly modified
  double ratio[3];        // reflectance ratio applied to cluster k
  int k;                  // cluster whose reflectance is rescaled (0: none)
};
void launch_flood_init(cudaStream_t s, const int32_t* ids, int target, const uint8_t* seeds, int64_t N,
                       uint8_t* mask);
void launch_flood_step(cudaStream_t s, const int32_t* ids, int target, int H, int W, const uint8_t* in,
                       uint8_t* out, int* changed);
void launch_set_flag(cudaStream_t s, int* f, int v);
void launch_recompose(cudaStream_t s, const float* X, int NT, int64_t N, const EditParams& P, const int32_t* ids,
                      const uint8_t* matte, const float* bg, float* out);
void launch_all_finite(cudaStream_t s, const float* x, int64_t n, int* flag);
void launch_pack_hwc(cudaStream_t s, const float* hwc, int C, int N, float* planes);
void launch_unpack_hwc(cudaStream_t s, const float* planes, int C, int N, float* hwc);
void launch_image(cudaStream_t s, const float* hwc, int N, float* img_planes, double* chroma);
void launch_edge(cudaStream_t s, const double* chroma, int H, int W, float* edge);
void launch_sample(cudaStream_t s, const SampleParams& P, SampleState* S, const double* chroma,
                   const double* prev_chroma, int H, int W, int16_t* codes, int32_t* out_cnt, int32_t* in_cnt,
                   int passes, const long long* known = nullptr, int n_known_lists = 0);
// row bands: raw PCG64 u32 zeros (Lemire rejections) at stream positions
// [begin, end) -> list[0] = count, list[1..] = positions (unsorted)
constexpr int kZeroList = 1 + kMaxRejections;
void launch_zero_scan(cudaStream_t s, const SampleParams& P, unsigned long long begin, unsigned long long end,
                      long long* list);
void launch_pairs_count(cudaStream_t s, int64_t n, const int64_t* src, const int64_t* dst,
                        const uint8_t* temporal, int H, int W, int32_t* out_cnt, int32_t* in_cnt, int* bad);
void launch_degree(cudaStream_t s, int N, const int32_t* out_cnt, const int32_t* in_cnt, int32_t* deg);
// the sampled adjacency's rows in reference order (fill + incoming-segment sort)
void launch_fill_from_samples(cudaStream_t s, const int16_t* codes, int H, int W, const int32_t* row_ptr,
                              const int32_t* out_cnt, int32_t* fill, uint16_t* ent);
void launch_fill_from_pairs(cudaStream_t s, int64_t n, const int64_t* src, const int64_t* dst,
                            const uint8_t* temporal, const double* weight, int W, const int32_t* row_ptr,
                            int32_t* fill, uint16_t* ent, uint32_t* key, float* ent_w);
void launch_sort_rows(cudaStream_t s, int N, const int32_t* row_ptr, uint16_t* ent, uint32_t* key,
                      float* ent_w);
void launch_pairs_from_samples(cudaStream_t s, const int16_t* codes, int H, int W, const int32_t* pair_off,
                               int64_t* src, int64_t* dst, uint8_t* temporal);
struct PalChroma { double c[2 * (kMaxNT - 1)]; };   // palette chromas, by value
struct PalColors { double c[3 * (kMaxNT - 1)]; };   // palette colors, by value
void launch_segment_raw(cudaStream_t s, const float* img, const double* chroma, int N, int K,
                        const PalChroma& pal, int32_t* ids_raw, int32_t* key, int* first_valid);
void launch_segment_band(cudaStream_t s, const float* img, const double* chroma, int N, int K, const PalChroma& pal,
                         int32_t* ids_raw, int32_t* key, int* first_valid, int own_lo, int own_hi);
void launch_segment_summary(cudaStream_t s, const int32_t* ids_raw, const int32_t* last, const int* first_valid,
                            int own_hi, int* summary);
void launch_segment_band_final(cudaStream_t s, int N, const int32_t* ids_raw, const int32_t* last,
                               const int* summaries, int nbands, int band, int own_lo, int own_hi, int32_t* ids);
void launch_segment_final(cudaStream_t s, int N, const int32_t* ids_raw, const int32_t* last,
                          const int* first_valid, int32_t* ids);
void launch_initialize(cudaStream_t s, const float* img, const int32_t* ids, int N, int NT,
                       const PalColors& colors, float* X);
void launch_set_i32(cudaStream_t s, int32_t* p, int n, int32_t v);

// ls_dense.cu
int dense_nsums(int K);
void launch_dense_accum(cudaStream_t s, int grid, const Frame& f, const double* colors_dev, int K,
                        const float* X, int use_ids, double* part, unsigned* ticket, double* sums);
void launch_dense_assemble_solve(cudaStream_t s, const double* sums, int K, const double* colors_dev,
                                 int use_ids, double lam_d, double lam_cl, double lam_ir, double lam_cr,
                                 int chroma_identity, double trunc, double* A_out, double* rhs_out,
                                 double* x_out);
void launch_svd_solve(cudaStream_t s, int n, const double* A, const double* rhs, double trunc, double* x);

}  // namespace ls
