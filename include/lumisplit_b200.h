/*
 * lumisplit_b200 -- C ABI of the B200-native alternating sparse-dense solver.
 *
 * Drop-in boundary for the hot path of the reference package `lumisplit`
 * (/root/reference/pkg/src/lumisplit).  The reference is pure Python/NumPy
 * and has no FFI of its own; each entry point below replaces one reference
 * function (cited per declaration), and the Python host package
 * `paper_1908_01961_b200` binds them with ctypes (INTEGRATION.md shows the
 * binding a maintainer would add to the reference).
 *
 * Conventions
 *   - Every array argument is caller-owned DEVICE memory unless the comment
 *     says "host".  No allocation happens inside the per-iteration calls;
 *     the context preallocates all workspace in ls_ctx_create.
 *   - Layer state is ONE planar float32 buffer `X` of U = K+4 planes of H*W:
 *     planes 0..2 are log-reflectance r (R, G, B), planes 3..K+3 are the
 *     transport layers T_0 (direct) .. T_K.  The reference's (H, W, C)
 *     arrays are the (C, H, W) planes viewed with a permutation; the PCG
 *     vector [r.ravel(), T.ravel()] of solver.py:110-122 corresponds to the
 *     same planes.  ls_pack_hwc / ls_unpack_hwc convert.
 *   - Palettes are passed as host arrays of K*3 doubles (reference
 *     BaseColorPalette.colors, palette.py:56-66); row 0 (white) is implicit.
 *   - Status codes: LS_OK, LS_ERR_NONFINITE (-> NumericalFaultError),
 *     LS_ERR_ARG (-> ValueError), LS_ERR_CUDA.  Nothing throws across the ABI.
 *   - One context per stream; contexts share no mutable state, so separate
 *     host threads may drive separate contexts (correction.py:185-196).
 *   - Reductions run in a fixed order without float atomics: results are
 *     bitwise repeatable for a given device.
 */
#ifndef LUMISPLIT_B200_H
#define LUMISPLIT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define LS_API __attribute__((visibility("default")))
#else
#define LS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum { LS_OK = 0, LS_ERR_NONFINITE = 1, LS_ERR_ARG = 2, LS_ERR_CUDA = 3 };
enum { LS_NUM_TERMS = 8, LS_MAX_K = 12 };

/* energy.py:28-56 (EnergyWeights); chroma_reg: 0 = "projection", 1 = "identity". */
typedef struct {
  double lambda_data, lambda_clustering, lambda_r_sparsity, p;
  double lambda_r_consistency, lambda_monochrome, lambda_i_sparsity;
  double lambda_smoothness, lambda_non_neg, lambda_ir, lambda_cr;
  double eps_nonneg, eps_irls;
  int chroma_reg;
} ls_weights;

/* solver.py:32-49 (the SolveConfig fields the device path consumes). */
typedef struct {
  int pcg_iterations;
  int max_halvings;
  double svd_truncation;
  double max_delta_b;
} ls_solve_cfg;

/* One Gauss-Newton step record (solver.py:180-188).  Term order:
 * data, clustering, r_sparsity, r_consistency, monochrome, i_sparsity,
 * smoothness, non_neg (energy.py:197-448). */
typedef struct {
  double energy_before, energy_after, alpha;
  int accepted;
  int pcg_iterations;
  double initial_residual, final_residual;
  double terms_before[LS_NUM_TERMS];
  double terms[LS_NUM_TERMS];
} ls_gn_record;

/* Dense base-color step record (solver.py:245-252). */
typedef struct {
  double energy_before, energy_after, alpha, delta_b_norm;
  int accepted;
  int solved_nonzero;
} ls_dense_record;

typedef struct ls_ctx ls_ctx;

/* ---- context ----------------------------------------------------------- */
LS_API const char* ls_version(void);
LS_API const char* ls_last_error(void);
LS_API int ls_ctx_create(int device, int H, int W, int K, const ls_weights* w,
                  const ls_solve_cfg* cfg, ls_ctx** out);
LS_API int ls_ctx_destroy(ls_ctx* ctx);
LS_API int ls_set_weights(ls_ctx* ctx, const ls_weights* w, const ls_solve_cfg* cfg);
LS_API int ls_set_stream(ls_ctx* ctx, void* cuda_stream);
/* Instrumentation: enable=1 starts CUDA-event timing of the solver kernels
 * (resets counters); ls_profile_read fills 11 doubles: (count, total ms) for
 * {energy+gradient, J^T J apply, PCG update, line-search trial, dense
 * reduction}, then the number of kernels this context launched, the number
 * of adjacency entries and of partner pairs of the installed frame (13). */
LS_API int ls_profile(ls_ctx* ctx, int enable);
LS_API int ls_profile_read(ls_ctx* ctx, double* out13);

/* ---- layout helpers ---------------------------------------------------- */
/* (H, W, C) interleaved <-> C planes of H*W. */
LS_API int ls_pack_hwc(ls_ctx* ctx, const float* hwc, int C, float* planes);
LS_API int ls_unpack_hwc(ls_ctx* ctx, const float* planes, int C, float* hwc);

/* ---- per-frame auxiliary context (solver.py:341-351, energy.py:455-475) -- */
/* Frame image, (H, W, 3) float32 interleaved.  Computes the planar copy,
 * chromaticity (imaging.py:160-171, fp64) and the chroma-edge gate
 * (energy.py:121-136). */
LS_API int ls_set_image(ls_ctx* ctx, const float* image_hwc);
/* Draws the consistency partners on the device, bit-exact with
 * sample_consistency (energy.py:154-187): numpy PCG64 stream given by its
 * 128-bit (state, inc) -- the host passes np.random.PCG64(seed).state -- and
 * 32-bit buffered Lemire bounded integers.  prev_chroma_planes (2 planes of
 * fp64, as returned by ls_get_chroma for the previous frame) may be NULL
 * (first frame: spatial pairs only); chroma_planes NULL means the installed
 * image's chroma.  Builds the per-pixel adjacency. */
LS_API int ls_sample_consistency(ls_ctx* ctx, const double* chroma_planes, const double* prev_chroma_planes,
                          uint64_t state_hi, uint64_t state_lo,
                          uint64_t inc_hi, uint64_t inc_lo, int64_t* n_pairs_out);
/* Device-to-device copy on the SMs (stream-ordered; unlike a D2D
 * cudaMemcpyAsync it never waits for a copy engine busy with host I/O). */
LS_API int ls_device_copy(void* dst, const void* src, int64_t bytes, void* stream);
/* The device int32 scan behind the adjacency rows and the segmentation
 * (single pass, decoupled look-back): op 0 = exclusive sum, 1 = inclusive
 * max, over n values; scratch = ls_scan_scratch_bytes(n) bytes of device
 * memory, reset by the call.  Stream-ordered. */
LS_API int64_t ls_scan_scratch_bytes(int64_t n);
LS_API int ls_scan_i32(const int32_t* in, int32_t* out, int64_t n, int op, void* scratch, void* stream);
/* Frame validity (imaging.py:36-57): *all_finite = no NaN / inf in x[0..n).
 * Synchronises `stream`; the flag comes back through mapped host memory. */
LS_API int ls_all_finite(const float* x, int64_t n, void* stream, int* all_finite);
/* Misclustering correction (correction.py:54-68): mask (H*W uint8) = the
 * 4-connected pixels with ids == target reachable from seeds (uint8), by
 * device dilation; scratch is H*W bytes.  Synchronises `stream`. */
LS_API int ls_flood_fill(const int32_t* ids, int target, const uint8_t* seeds, int H, int W, uint8_t* mask,
                         uint8_t* scratch, void* stream);
/* Layer edits (editing.py:24-74): out (H, W, 3) = clip(R' * sum_k T_k B'_k, 0, 1)
 * from the planar state X, the (K+1) x 3 host matrix B' (row 0 white), the
 * reflectance of cluster k (ids == k, 0 = none) scaled by ratio[3] (host);
 * pixels with matte != 0 copy bg (H, W, 3).  fp64 per pixel. */
LS_API int ls_recompose(const float* X, int K, int H, int W, const double* B_host, int k,
                        const double* ratio_host, const int32_t* ids, const uint8_t* matte, const float* bg,
                        float* out_hwc, void* stream);
/* Counts of the installed partner rows (synchronises the stream): pairs,
 * temporal pairs, adjacency entries.  ls_sample_consistency itself does not
 * synchronise and reports n_pairs_out = -1. */
LS_API int ls_pair_count(ls_ctx* ctx, int64_t* n_pairs, int64_t* n_temporal, int64_t* n_entries);
/* Explicit partner rows (ConsistencySamples, energy.py:139-151); src/dst
 * flat pixel indices (int64), temporal as uint8, weight may be NULL (all 1).
 * Partners must lie in the 15x15 window (|dx|,|dy| <= 7) -> else LS_ERR_ARG. */
LS_API int ls_set_pairs(ls_ctx* ctx, int64_t n, const int64_t* src, const int64_t* dst,
                 const uint8_t* temporal, const double* weight);
/* Copies the current partner rows out (host-visible sizes via n_pairs_out of
 * ls_sample_consistency); arrays are device memory of length n. */
LS_API int ls_get_pairs(ls_ctx* ctx, int64_t* src, int64_t* dst, uint8_t* temporal);
/* Edge gate override (float32 H*W) -- for EnergyAux built by hand. */
LS_API int ls_set_edge(ls_ctx* ctx, const float* edge);
/* Previous frame log-reflectance (3 planes) or NULL. */
LS_API int ls_set_prev_r(ls_ctx* ctx, const float* prev_r_planes);
/* Clustered-reflectance anchor: cluster ids (int32 H*W, values 1..K) or a
 * fixed log anchor (3 planes); exactly one non-NULL (energy.py:470-475). */
LS_API int ls_set_anchor(ls_ctx* ctx, const int32_t* cluster_ids, const float* r_cluster_log_planes);
LS_API int ls_get_edge(ls_ctx* ctx, float* edge_out);
LS_API int ls_get_chroma(ls_ctx* ctx, double* chroma_planes_out);
/* Context-free: chromaticity planes (fp64) of an (H, W, 3) image
 * (imaging.py:160-171) and the chroma-edge gate of chroma planes
 * (energy.py:121-136), on the given stream. */
LS_API int ls_chromaticity(const float* image_hwc, int H, int W, double* chroma_planes_out,
                           void* cuda_stream);
LS_API int ls_edge_from_chroma(const double* chroma_planes, int H, int W, float* edge_out,
                               void* cuda_stream);

/* palette.py:195-224: nearest-chroma ids (int32 H*W, 1..K) of the current
 * image with dark-pixel scanline inheritance. */
LS_API int ls_segment(ls_ctx* ctx, const double* colors_host, int32_t* ids_out);
/* solver.py:295-308 first-frame initialisation into X (U planes). */
LS_API int ls_initialize(ls_ctx* ctx, const double* colors_host, const int32_t* ids, float* X);

/* ---- energy operators (energy.py:194-511, solver.py:110-140) ------------ */
/* Per-term energies at Y with IRLS weights and linearisation frozen at X
 * (assemble_blocks at X, block_energies at Y).  Y may equal X. */
LS_API int ls_energy_terms(ls_ctx* ctx, const double* colors_host, const float* X, const float* Y,
                    double terms_out_host[LS_NUM_TERMS]);
/* b = -J^T F and diag(J^T J) at X (solver.py:125-136); planar U*N float. */
LS_API int ls_grad_diag(ls_ctx* ctx, const double* colors_host, const float* X, float* b, float* diag);
/* Ap = J^T J p, operator frozen at X (solver.py:110-122). */
LS_API int ls_apply_normal(ls_ctx* ctx, const double* colors_host, const float* X, const float* p,
                    float* Ap);
/* Jacobi PCG on the frozen normal equations (solver.py:79-107), x planar.
 * info_host = {iterations, initial_residual, final_residual}. */
LS_API int ls_pcg(ls_ctx* ctx, const double* colors_host, const float* X, int iterations, float* x,
           double info_host[3]);

/* ---- solver steps (solver.py:143-255) ---------------------------------- */
/* One sparse Gauss-Newton step from X; the candidate state is written to
 * X_out (accepted iff rec->accepted; otherwise X_out is unspecified).
 * Returns LS_ERR_NONFINITE (rec->terms_before filled) for a non-finite
 * starting energy (solver.py:153-157). */
LS_API int ls_gn_step(ls_ctx* ctx, const double* colors_host, const float* X, float* X_out,
               ls_gn_record* rec);
/* Streaming flip-flop (solver.py:311-338 with refine = False), enqueued
 * without host round trips: line search, acceptance, state selection and the
 * relative-decrease convergence test run on the device; one synchronisation
 * at the end.  The state starts in X0; X1 / X2 are ping-pong buffers;
 * *final_buffer (0/1/2) says which holds the result.  out (host, outer *
 * gn_steps records) receives *n_records executed steps; *status: 0
 * max_outer, 1 stalled, 2 converged.  A non-finite starting energy returns
 * LS_ERR_NONFINITE with *fault_step the faulting record (solver.py:153-157). */
LS_API int ls_flip_flop_stream(ls_ctx* ctx, const double* colors_host, float* X0, float* X1, float* X2, int outer,
                               int gn_steps, double tol_rel, ls_gn_record* out, int* n_records, int* status,
                               int* final_buffer, int* fault_step);
/* ls_flip_flop_stream as ONE CUDA graph launch (captured on first use over
 * context-owned state buffers, replayed while palette, weights, config and
 * the frame's buffers are unchanged -- the streaming case).  X_in is copied
 * in, the final state is written to X_out (stream-ordered after return). */
LS_API int ls_flip_flop_graph(ls_ctx* ctx, const double* colors_host, const float* X_in, float* X_out, int outer,
                              int gn_steps, double tol_rel, ls_gn_record* out, int* n_records, int* status,
                              int* fault_step);
/* n independent flip-flops (one per context, same palette and schedule) as
 * one launch sequence: all are enqueued, each on its context's stream, before
 * any is waited for -- the K candidate solves of correct_reflectance
 * (correction.py:168-201, whose thread pool this replaces).  Per context i:
 * state buffers X0[i] (input) / X1[i] / X2[i], records at out + i*outer*gn_steps,
 * n_records[i], status[i], final_buffer[i], fault_step[i] as
 * ls_flip_flop_stream's, and its own return code in rcs[i].  Returns LS_OK
 * unless the arguments are invalid. */
LS_API int ls_flip_flop_batch(ls_ctx* const* ctxs, int n, const double* colors_host, float* const* X0,
                              float* const* X1, float* const* X2, int outer, int gn_steps, double tol_rel,
                              ls_gn_record* out, int* n_records, int* status, int* final_buffer,
                              int* fault_step, int* rcs);
/* Dense 3K x 3K refinement normal system at delta_b = 0 (energy.py:563-610);
 * uses the cluster ids set by ls_set_anchor when use_ids != 0.  Host outputs. */
LS_API int ls_dense_normal(ls_ctx* ctx, const double* colors_host, const float* X, int use_ids,
                    double* A_host, double* rhs_host);
/* Truncated-SVD minimum-norm solve (solver.py:195-204), one-sided Jacobi SVD
 * in fp64 on the device.  n <= 3*LS_MAX_K, host arrays. */
LS_API int ls_svd_solve(ls_ctx* ctx, int n, const double* A_host, const double* rhs_host,
                 double truncation, double* x_host);
/* solve_dense_block (solver.py:207-255): solve, trust cap, clipped line
 * search on the frozen energy.  colors_inout_host (K*3) is updated iff
 * accepted; applied_host (K*3) receives the applied update. */
LS_API int ls_dense_step(ls_ctx* ctx, double* colors_inout_host, const float* X, double* applied_host,
                  ls_dense_record* rec);

/* First-frame palette estimation (palette.py:227-238 without the final
 * segment, which is ls_segment): the 10x10 chroma histogram of the non-dark
 * pixels (:81-103), population-weighted k-means with the seeded first pick of
 * numpy's Generator.choice -- (state, inc) of np.random.PCG64(seed) as for
 * ls_sample_consistency -- and farthest-point seeding (:106-138), nearest-
 * center assignment and the greedy merge of centers closer than 0.2
 * (:141-192).  image_hwc: (H, W, 3) float32 device memory; colors_out: host,
 * room for 3 * k_max doubles; *K_out = 0 when every pixel is dark
 * (EmptyHistogramError).  k_max in 1..12.  Synchronises `stream`. */
LS_API int ls_estimate_palette(const float* image_hwc, int H, int W, int k_max, uint64_t state_hi,
                               uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double* colors_out,
                               int* K_out, void* stream);

/* ---- per-block residual protocol (energy.py:194-452) --------------------
 * The reference's assemble_blocks returns eight residual blocks
 * (energy.py:478-496), each with residual(r, T), apply_j(dr, dT),
 * apply_jt(w, out_dr, out_dT) (accumulating) and add_diag(out_dr, out_dT)
 * (accumulating); stack_residuals concatenates the residuals (:499-500).
 * These entry points are that protocol on the device, block by block, with
 * the IRLS weights and the linearisation frozen at the planar state X0 and
 * the frame installed in the context (ls_set_image / ls_set_edge /
 * ls_set_anchor / ls_set_prev_r).  Row vectors (residual, J dX, the w of
 * J^T w) are float32 in the reference's row order (the (H, W, C) ravel of
 * each block; r_consistency: pair-major, 3 rows per pair); X0, Y, dX and the
 * accumulated outputs are U planes.  The consistency block reads the partner
 * rows from `pairs` (device arrays, pair order = row order).  Block ids:
 * data, clustering, r_sparsity, r_consistency, monochrome, i_sparsity,
 * smoothness, non_neg (the LS term order). */
enum { LS_BLOCK_DATA = 0, LS_BLOCK_CLUSTERING, LS_BLOCK_R_SPARSITY, LS_BLOCK_R_CONSISTENCY,
       LS_BLOCK_MONOCHROME, LS_BLOCK_I_SPARSITY, LS_BLOCK_SMOOTHNESS, LS_BLOCK_NON_NEG };
typedef struct {
  int64_t n;
  const int64_t* src;
  const int64_t* dst;
  const uint8_t* temporal; /* NULL: all spatial */
  const double* weight;    /* NULL: all 1 */
} ls_pairs;
/* number of residual rows of a block (host-side, no device work) */
LS_API int ls_block_rows(ls_ctx* ctx, int block, int64_t n_pairs, int64_t* rows);
/* DataBlock.residual ... NonNegBlock.residual (energy.py:205-209, 234-235,
 * 264-267, 348-350, 399-401, 424-425) at the state Y */
LS_API int ls_block_residual(ls_ctx* ctx, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                             const float* Y, float* out_rows);
/* apply_j (energy.py:211-212, 237-238, 269-270, 352-357, 403-404, 427-428) */
LS_API int ls_block_apply_j(ls_ctx* ctx, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                            const float* dX, float* out_rows);
/* apply_jt, accumulating into out_dX (energy.py:214-218, 240-241, 272-282,
 * 359-370, 406-408, 430-431) */
LS_API int ls_block_apply_jt(ls_ctx* ctx, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                             const float* w_rows, float* out_dX);
/* add_diag, accumulating into out_dX (energy.py:220-222, 243-244, 284-291,
 * 372-381, 410-411, 433-434) */
LS_API int ls_block_add_diag(ls_ctx* ctx, const double* colors, const float* X0, int block, const ls_pairs* pairs,
                             float* out_dX);

/* ---- Row bands (SURVEY.md 8(e), configs[3]: >= 4K frames split spatially) --
 * One context per band of rows.  The context is created with the band's
 * LOCAL frame: global rows [gy0, gy0 + H) of a GH-row frame, i.e. the band's
 * own rows [y_lo, y_hi) plus up to 8 halo rows on each side that the caller
 * keeps equal to the neighbouring bands' rows.  In band mode every reduction
 * is written as this band's partial sum (ls_band_buffers()[0]); the caller
 * gathers all bands' partials in band order ([nbands][nv] doubles, device)
 * and ls_band_finalize runs the same finalisation the whole-frame kernels
 * run, so every band takes identical scalar decisions.  The whole-frame entry
 * points refuse a band context.  The orchestration (one GN step = EG, 16 x
 * (apply, update), trials; halo refresh between phases) is
 * paper_1908_01961_b200/bands.py.  Replaces no single reference function:
 * the reference solves the frame as one problem (solver.py:143-192); the
 * bands reproduce that problem's arithmetic up to the summation grouping. */
enum { LS_BAND_EG = 0, LS_BAND_APPLY = 1, LS_BAND_UPDATE = 2, LS_BAND_TRIAL = 3 };
/* kernels this context launched (ls_profile resets it); a caller replaying
 * captured ls_band_* work as its own CUDA graph adds the replayed launches */
LS_API int ls_launch_count(ls_ctx* ctx, int64_t* n);
LS_API int ls_add_launches(ls_ctx* ctx, int64_t n);
/* Bytes of everything the kernels of this context bake into their launch
 * arguments (weights, solve config, per-frame pointers and flags such as
 * prev_r / ids / anchor / pair weights, band rows, TMA use): a caller that
 * captures ls_band_* work as its own CUDA graph keys the graph on them.
 * Writes at most cap bytes to out and the full length to *len. */
LS_API int ls_state_key(ls_ctx* ctx, void* out, int64_t cap, int64_t* len);
LS_API int ls_band_set(ls_ctx* ctx, int gy0, int GH, int y_lo, int y_hi);
LS_API int ls_band_clear(ls_ctx* ctx);
/* out[6] = {partials (512 doubles), z, p_even, p_odd, x, r}: the PCG vectors
 * (U planes of H*W floats each) whose halo rows the caller refreshes. */
LS_API int ls_band_buffers(ls_ctx* ctx, void** out);
/* Keep the band's PCG search directions: allocates n (<= 64) buffers of U x H_local
 * x W floats (once; not during a graph capture) and returns them in out[0..n-1].
 * From then on ls_band_pcg_apply(iter) writes p_iter to out[iter] (the caller
 * exchanges its halo rows there) and leaves x alone, and ls_band_pcg_finish forms
 * x = sum alpha_i p_i in one pass -- the whole-frame loop's layout. */
LS_API int ls_band_dirs(ls_ctx* ctx, int n, void** out);
/* In-process row bands (one device, one stream): ls_band_finalize_dev of all
 * n bands at once, reading every band's partial sums directly (no gather
 * copies); the same band-ordered sums and decisions.  Launched on ctxs[0]'s
 * stream. */
LS_API int ls_band_finalize_group(ls_ctx* const* ctxs, int n, int phase, int iter, double alpha, int last);
/* n <= 32 strided slab copies in one launch: slab i copies planes[i] x count[i]
 * floats from src[i] + p * src_stride[i] to dst[i] + p * dst_stride[i]
 * (host arrays of device pointers; the halo moves between in-process bands). */
LS_API int ls_copy_slabs(int n, const float* const* src, float* const* dst, const int64_t* src_stride,
                         const int64_t* dst_stride, const int64_t* count, const int* planes, void* stream);
/* Raw PCG64 u32 zeros (the Lemire rejections of energy.py:162-171) at stream
 * positions [begin, end): list (device, 17 int64) = {count, positions...}.
 * The bands split [0, 12*GH*W + 64) and gather their lists; the gathered
 * lists (device, n_lists x 17) are handed to ls_band_set_zeros before the
 * band's ls_sample_consistency, which then draws with global pixel indices. */
LS_API int ls_band_zero_scan(ls_ctx* ctx, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, uint64_t begin, uint64_t end, int64_t* list);
LS_API int ls_band_set_zeros(ls_ctx* ctx, const int64_t* lists, int n_lists);
/* Phases of one GN step (solver.py:143-192), each writing its band partial:
 * EG (energies at X, b, diag, PCG init; nv = 10), apply (iteration iter,
 * p-update + J^T J p; nv = 1), update (nv = 2), trial (energies at
 * X + alpha*x into X_out, or at X itself when X_out is NULL; nv = 8). */
LS_API int ls_band_eg(ls_ctx* ctx, const double* colors_host, const float* X);
LS_API int ls_band_pcg_apply(ls_ctx* ctx, const double* colors_host, const float* X, int iter);
LS_API int ls_band_pcg_update(ls_ctx* ctx, int iter);
/* after the last update: the deferred x += alpha p of the final iteration */
LS_API int ls_band_pcg_finish(ls_ctx* ctx);
LS_API int ls_band_trial(ls_ctx* ctx, const double* colors_host, const float* X, double alpha, float* X_out);
LS_API int ls_band_finalize(ls_ctx* ctx, int phase, const double* gathered, int nbands, int iter, double alpha);
/* Device-resident band flip-flop (the band form of ls_flip_flop_stream):
 * frame_begin; per GN step eg / apply / update / finish as above, then up to
 * max_halvings+1 trial_dev + finalize_dev(TRIAL, last) -- the accept / halve
 * decision of solver.py:169-178 on the device, identical on every band --
 * and step_end (state moves to X_out, copied through on a reject, record);
 * per outer iteration outer_end (solver.py:328-336); frame_end reads the
 * records (one synchronisation).  No host decision inside a frame, so the
 * sequence with its gathers and halo copies can be one CUDA graph. */
LS_API int ls_band_frame_begin(ls_ctx* ctx);
LS_API int ls_band_trial_dev(ls_ctx* ctx, const double* colors_host, const float* X, double alpha, float* X_out,
                             int last);
LS_API int ls_band_finalize_dev(ls_ctx* ctx, int phase, const double* gathered, int nbands, int iter,
                                double alpha, int last);
LS_API int ls_band_step_end(ls_ctx* ctx, const float* X_in, float* X_out, int out_id);
LS_API int ls_band_outer_end(ls_ctx* ctx, double tol_rel);
LS_API int ls_band_frame_end(ls_ctx* ctx, int nsteps, ls_gn_record* out, int* n_records, int* status,
                             int* final_buffer, int* fault_step);
/* host out[21]: terms0[8], terms1[8], |b|^2, |r|^2, iterations, stop, xinit */
LS_API int ls_band_read(ls_ctx* ctx, double* out_host);
/* Dense system (energy.py:563-610) of the band's own pixels as partial sums
 * (ls_band_dense_nsums() doubles); ls_band_dense_solve sums the gathered
 * partials in band order, assembles and solves (solver.py:195-204). */
LS_API int ls_band_dense_accum(ls_ctx* ctx, const double* colors_host, const float* X, int use_ids);
LS_API int ls_band_dense_nsums(ls_ctx* ctx);
LS_API int ls_band_dense_solve(ls_ctx* ctx, const double* colors_host, const double* gathered, int nbands,
                               int use_ids, double* dx_host);
/* segment (palette.py:195-224) per band: summary (device, 3 int32) = {has a
 * non-dark own pixel, first id, last id}; with every band's summary gathered
 * (device, nbands x 3) the final ids of the own rows follow the reference's
 * raster-order dark-pixel inheritance across band boundaries. */
LS_API int ls_band_segment(ls_ctx* ctx, const double* colors_host, int32_t* summary);
LS_API int ls_band_segment_final(ls_ctx* ctx, const int32_t* summaries, int nbands, int band, int32_t* ids_out);

#ifdef __cplusplus
}
#endif
#endif /* LUMISPLIT_B200_H */
