/*
 * gsvr_b200.h -- C ABI of the B200-native GSVR hot path.
 *
 * Every entry point takes DEVICE pointers (caller-owned, contiguous, row-major
 * exactly as the reference's numpy arrays), plain sizes and a cudaStream_t
 * passed as void*.  Nothing here knows about torch.  Each call returns a status:
 *
 *   GSVR_OK            0
 *   GSVR_ERR_INVALID   1  -> errors.InvalidParameterError   (bad shape / id range)
 *   GSVR_ERR_NONFINITE 2  -> errors.TrainingDivergedError   (non-finite render)
 *   GSVR_ERR_DEGENERATE 3 -> errors.NumericalDegeneracyError (scale below floor)
 *   GSVR_ERR_CUDA      4  -> RuntimeError (CUDA failure; message via gsvr_last_error)
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/gsvr/):
 *   gsvr_render_forward        kernels.py:41-75   render_forward
 *   gsvr_train_step_backward   kernels.py:78-198  train_step_backward (+ the ordered
 *                              block sum of train.py:263-269: ONE reduced buffer set)
 *   gsvr_field_covariances     field.py:67-69 / geometry.py:143-165 covariances6
 *   gsvr_field_chain           train.py:271-282   covariance chain + regulariser grad
 *   gsvr_slice_chain           train.py:284-296   slice chain (dq_i, dlog_sigma, deta)
 *   gsvr_knn_*                 knn.py:33-75       build_index / query (exact, same ties)
 *   gsvr_eval_field            field.py:93-135    evaluate_field (PSF-free, clamp)
 *   gsvr_batch_* / gsvr_train_tiles / gsvr_*_adamw_step
 *                              train.py:373-497   the device-resident fit loop pieces
 *                              (optim.py:69-88 AdamW fused with the chains)
 */
#ifndef GSVR_B200_H
#define GSVR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSVR_OK 0
#define GSVR_ERR_INVALID 1
#define GSVR_ERR_NONFINITE 2
#define GSVR_ERR_DEGENERATE 3
#define GSVR_ERR_CUDA 4

#define GSVR_F32 0
#define GSVR_F64 1

/* ABI version (bumped on any signature change). */
int gsvr_abi_version(void);
/* Message of the last non-OK status on this thread ("" if none). */
const char *gsvr_last_error(void);
/* Index of the offending element of the last NONFINITE / DEGENERATE / INVALID
 * status on this thread (slice id, primitive id, ...), or -1. */
int64_t gsvr_last_error_index(void);
/* Extra scalar attached to the last status (e.g. the collapsed scale), or 0. */
double gsvr_last_error_value(void);

/* ---- field / geometry -------------------------------------------------- */

/* field.py:67-69: cov6 (N,6) = pack(R(q) diag(exp(2 ls)) R(q)^T).
 * If check_floor, returns GSVR_ERR_DEGENERATE naming the first primitive whose
 * smallest scale^2 < 1e-6 (train.py:162-169). */
int gsvr_field_covariances(int64_t N, const double *log_scales, const double *quats,
                           double *cov6, int check_floor, void *stream);

/* train.py:271-282.  dcov6 (N,6) -> dls (N,3), dq (N,4); adds the scale
 * regulariser lambda*2*(s - s_target)*s when lambda_reg > 0. */
int gsvr_field_chain(int64_t N, const double *log_scales, const double *quats,
                     const double *dcov6, double lambda_reg, double s_target,
                     double *dls, double *dq, void *stream);

/* train.py:145-152 + 284-290.  Per-slice inputs from slice states and the
 * chain of the slice gradients back to the state parameters.  Any output
 * pointer may be NULL to skip it. */
int gsvr_slice_inputs(int64_t S, const double *slice_quats, const double *stack_rots,
                      const int32_t *slice_to_stack, const double *log_sigma,
                      const double *psf_diags, double *Rc, double *R_eff, double *psf6s,
                      double *sigma_s, void *stream);
int gsvr_slice_chain(int64_t S, const double *slice_quats, const double *stack_rots,
                     const int32_t *slice_to_stack, const double *log_sigma,
                     const double *psf_diags, const double *dRc, const double *dpsf6,
                     const double *dsigraw, double *dq_slice, double *dlog_sigma,
                     void *stream);

/* ---- forward / fused train -------------------------------------------- */

/* kernels.py:41-75 (clamp at -80).  dtype GSVR_F32 or GSVR_F64 applies to
 * points/psf6/sigma/mu/cov6/cvals/out; nbr is int64 (nbr_i64=1) or int32.
 * Ids are validated (GSVR_ERR_INVALID on any id outside [0,N)). */
int gsvr_render_forward(int dtype, int64_t M, int64_t K, const void *points,
                        const void *psf6, const void *sigma, const void *nbr, int nbr_i64,
                        int64_t N, const void *mu, const void *cov6, const void *cvals,
                        double delta, void *out, void *stream);

/* kernels.py:78-198 (drop-below -80 semantics), float64 I/O like the reference,
 * fp32 per-pair arithmetic with tile-relative coordinates.  Gradient outputs
 * are ONE reduced set (no block axis), accumulated into (+=) caller-zeroed
 * buffers: dmu (N,3) dcov6 (N,6) dc (N) dt (S,3) dRc (S,3,3) dpsf6 (S,6)
 * dsigraw (S).  Internally: (slice, tile) binning of the points and their
 * neighbour lists, then the tiled fused kernel. */
int gsvr_train_step_backward(int64_t P, int64_t K, int64_t S, int64_t N,
                             const double *x0pts, const int32_t *sid, const double *Rc,
                             const double *tvec, const double *psf6s, const double *sigma_s,
                             const double *wdata_s, const double *I_obs, const void *nbr,
                             int nbr_i64, const double *mu, const double *cov6,
                             const double *cvals, double delta, double *I_hat,
                             double *absres, double *dmu, double *dcov6, double *dc,
                             double *dt, double *dRc, double *dpsf6, double *dsigraw,
                             void *stream);

/* Same call with every array in HOST memory (numpy / ctypes / cgo callers).
 * The neighbour upload (the bulk of the bytes) is chunked on a copy stream and
 * overlapped with batch planning and per-tile binning; pinned (page-locked)
 * buffers give full overlap.  dmu..dsigraw accumulate (caller-zeroed block of
 * kernels.py:79-82), I_hat / absres are overwritten.  Replaces the same
 * kernels.py:78-198 entry point for host-resident callers. */
int gsvr_train_step_backward_host(int64_t P, int64_t K, int64_t S, int64_t N, const double *x0pts,
                                  const int32_t *sid, const double *Rc, const double *tvec,
                                  const double *psf6s, const double *sigma_s, const double *wdata_s,
                                  const double *I_obs, const void *nbr, int nbr_i64, const double *mu,
                                  const double *cov6, const double *cvals, double delta, double *I_hat,
                                  double *absres, double *dmu, double *dcov6, double *dc, double *dt,
                                  double *dRc, double *dpsf6, double *dsigraw, void *stream);

/* train.py:189-206 render_batch: x = Rc[sid] x0 + t[sid], per-slice PSF and
 * sigma, clamp semantics, float64. */
int gsvr_render_batch(int64_t P, int64_t K, const double *x0, const int32_t *sid,
                      const double *Rc, const double *tvec, const double *psf6s,
                      const double *sigma_s, const void *nbr, int nbr_i64, int64_t N,
                      const double *mu, const double *cov6, const double *cvals, double delta,
                      double *out, void *stream);

/* train.py:305-309 corrected_points: out (P,3) = Rc[sid] x0 + t[sid]. */
int gsvr_corrected_points(int64_t P, const double *x0, const int32_t *sid, const double *Rc,
                          const double *tvec, double *out, void *stream);

/* field.py:93-135 evaluate_field: PSF-free, clamp at -80, float64. */
int gsvr_eval_field(int64_t M, int64_t K, const double *points, const void *nbr, int nbr_i64,
                    int64_t N, const double *mu, const double *log_scales,
                    const double *quats, const double *cvals, double delta, double *out,
                    void *stream);

/* ---- exact K-NN (knn.py:33-75) ----------------------------------------- */

typedef struct gsvr_knn_index gsvr_knn_index;

/* Snapshot the means (N,3) float64 into a uniform grid (cells sorted by a
 * device radix sort).  Returns GSVR_ERR_INVALID for N<1 or non-finite means. */
int gsvr_knn_build(int64_t N, const double *means, gsvr_knn_index **out, void *stream);
void gsvr_knn_free(gsvr_knn_index *index);
int64_t gsvr_knn_count(const gsvr_knn_index *index);
/* Top-K ids per point, rows ordered by (distance, index), boundary ties
 * re-resolved by (d2, index) exactly as knn.py:58-74.  points (M,3) float64;
 * out (M,K) int64 (out_i64=1) or int32. */
int gsvr_knn_query(const gsvr_knn_index *index, int64_t M, const double *points, int64_t K,
                   void *out, int out_i64, void *stream);

/* ---- device-resident fit loop pieces (train.py:373-497) ----------------- */

typedef struct gsvr_batch gsvr_batch;

/* Point batch (P points, S slices): sorts points by (slice, Morton code),
 * cuts single-slice tiles of <= tile_points points, stores tile-relative
 * fp32 offsets.  x0pts (P,3) f64, sid (P,) int32 in [0,S), I_obs (P,) f64. */
int gsvr_batch_create(int64_t P, int64_t S, const double *x0pts, const int32_t *sid,
                      const double *I_obs, int tile_points, gsvr_batch **out, void *stream);
void gsvr_batch_free(gsvr_batch *batch);
int64_t gsvr_batch_tiles(const gsvr_batch *batch);
/* Permutation internal -> caller order (P int32, device). */
const int32_t *gsvr_batch_perm(const gsvr_batch *batch);
/* Replace observed intensities (caller order, f64). */
int gsvr_batch_set_observed(gsvr_batch *batch, const double *I_obs, void *stream);

/* Neighbour refresh: exact K-NN of the points x = Rc x0 + t (per-slice Rc (S,3,3),
 * t (S,3)) against the index, then (slice, tile) binning. */
int gsvr_batch_refresh(gsvr_batch *batch, const gsvr_knn_index *index, int64_t K,
                       const double *Rc, const double *tvec, void *stream);

/* Rows of the last seeded refresh that the heap-free selection kernel handed
 * to the heap kernel (boundary bin over capacity), or -1 when the last refresh
 * ran the heap kernel for every row (unseeded / GSVR_KNN_SELECT=0). */
int64_t gsvr_batch_knn_fallback_rows(const gsvr_batch *batch);

/* Forget the previous lists as refresh seeds (e.g. after a reseed replaced the
 * field: its lists bound nothing useful); the next refresh runs unseeded. */
void gsvr_batch_invalidate_seeds(gsvr_batch *batch);
/* Binning from caller-supplied neighbour ids (P,K) in caller order. */
int gsvr_batch_bin(gsvr_batch *batch, int64_t K, int64_t N, const void *nbr, int nbr_i64,
                   void *stream);
/* Tile plane geometry (device buffers, any may be NULL): origin (T,3) f64,
 * basis (T,6) f64 = in-plane axes b1, b2 (nominal frame), ab (P,2) f32 =
 * in-plane coordinates of each point (internal order). */
int gsvr_batch_tile_geometry(const gsvr_batch *batch, double *origin, double *basis, float *ab,
                             void *stream);
/* Neighbour ids currently binned, written in caller order as int64 (P,K). */
int gsvr_batch_neighbors(const gsvr_batch *batch, int64_t *out, void *stream);
/* Unique (tile, Gaussian) records of the current binning (for reporting). */
int64_t gsvr_batch_tile_gaussians(const gsvr_batch *batch);
/* Copy the tile table and binning into caller device buffers (any may be NULL):
 * tile_start (T) int64 [internal index of the tile's first point], tile_n (T),
 * tile_slice (T), uoff (T+1) [offsets into gid], gid (U) [ascending unique ids
 * per tile], perm (P) [internal -> caller index].  The (slice, tile)
 * unique-Gaussian counts are uoff[t+1]-uoff[t]. */
int gsvr_batch_tile_info(const gsvr_batch *batch, int64_t *tile_start, int32_t *tile_n,
                         int32_t *tile_slice, int32_t *uoff, int32_t *gid, int32_t *perm,
                         void *stream);

/* One fused forward + L1 + backward pass over all tiles.
 * Field grads accumulate (+=) into fp32 dfield (N,10) = [dmu(3) dcov6(6) dc(1)];
 * slice grads into f64 dslice (S,20) = [dt(3) dRc(9) dpsf6(6) dsigraw(1) l1(1)].
 * I_hat / absres (caller order, f64) may be NULL.  nonfinite_first (device,
 * may be NULL, caller-initialised to ~0) receives the smallest caller index of
 * a non-finite rendered value.  Asynchronous. */
int gsvr_train_tiles(const gsvr_batch *batch, int64_t S, int64_t N, const double *Rc,
                     const double *tvec, const double *psf6s, const double *sigma_s,
                     const double *wdata_s, const double *mu, const double *cov6,
                     const double *cvals, double delta, float *dfield, double *dslice,
                     double *I_hat, double *absres, unsigned long long *nonfinite_first,
                     void *stream);

/* Max over points of |(Rc_a - Rc_b) x0 + (t_a - t_b)|^2, i.e. the staleness
 * test of train.py:458-461, written to *out (device f64). */
int gsvr_batch_displacement(const gsvr_batch *batch, const double *Rc_a, const double *t_a,
                            const double *Rc_b, const double *t_b, double *out, void *stream);

/* Fused field chain + AdamW (+ zero the grad buffer, + covariances, scale
 * regulariser and floor check of the UPDATED field for the next epoch).
 * params: means (N,3) ls (N,3) q (N,4) c (N) f64, in place.  m/v: (N,11) f64
 * [means ls q c].  lrs[4] (host) base rates for means, log_scales, quaternions,
 * intensities; lr_scale; bc1/bc2 = 1 - beta^t bias corrections.  do_step=0
 * only recomputes cov6/regulariser/floor.  stats_out is the caller's
 * workspace of gsvr_field_workspace_bytes() bytes, zero-filled once before
 * its first use (one per engine: steps sharing a workspace must not overlap;
 * steps with different workspaces may).  Writes cov6_out (N,6),
 * stats_out[0] = sum_j ||exp(ls_j) - s_target||^2 (device f64; its previous
 * value is copied to stats_prev_out[0] first when that is not NULL) and
 * floor_out (device) = first primitive whose smallest scale^2 < 1e-6, or ~0.
 * Launches one kernel (no memsets). */
int gsvr_field_adamw_step(int64_t N, double *means, double *log_scales, double *quats,
                          double *cvals, double *m, double *v, float *dfield,
                          double lambda_reg, double s_target, const double *lrs,
                          double lr_scale, double beta1, double beta2, double eps,
                          double weight_decay, double bc1, double bc2, int do_step,
                          double *cov6_out, double *stats_out,
                          unsigned long long *floor_out, double *stats_prev_out,
                          void *stream);

/* Bytes of the gsvr_field_adamw_step workspace (stats_out). */
int64_t gsvr_field_workspace_bytes(void);

/* Fused slice chain + AdamW + next-epoch slice inputs.
 * state (S,9) f64 = [q(4) t(3) log_sigma eta], m/v (S,9); dslice (S,20) as
 * above (zeroed after use).  step_mask bits: 1 = step at all, 2 = rotations
 * frozen (quaternion grads zeroed), anchor = slice kept fixed (-1 none).
 * Writes loss_out[0:3] = {data, outlier, l1_total} and the per-slice
 * inputs for the next epoch (Rc, tvec, psf6s, sigma_s, wdata_s). */
int gsvr_slice_adamw_step(int64_t S, double *state, double *m, double *v, double *dslice,
                          const double *stack_rots, const int32_t *slice_to_stack,
                          const double *psf_diags, const double *slice_counts,
                          int outlier_weighting, const double *lrs, double lr_scale,
                          double beta1, double beta2, double eps, double weight_decay,
                          double bc1, double bc2, int step_mask, int64_t anchor,
                          double *loss_out, double *Rc, double *tvec, double *psf6s,
                          double *sigma_s, double *wdata_s, void *stream);

/* ---- acquisition simulator (data generation) -------- */

/* simulate.py:142-205 (_psf_quadrature + _trilinear): out[p] = sum over the
 * tensor grid of slice-frame offsets (a_i, b_j, c_k) with weights
 * wx_i * wy_j * wz_k of the trilinear interpolation of the raster vol
 * (nx, ny, nz) f64, x-major, zero outside) at centre_p + A_s (a, b, c)^T,
 * where A_s = axes[sid[p]] (S, 3, 3) row-major (columns = world slice axes;
 * sid NULL -> axes[0] for every centre) and inv_affine (3, 4) host f64 maps
 * world mm to raster indices.  nodes (device) = [offx(n0) wx(n0) offy(n1)
 * wy(n1) offz(n2) wz(n2)], n* <= 128.  float64, every product and sum
 * rounded in the reference's order (no FMA): agrees with the numba kernel to
 * the last bits. */
int gsvr_psf_quadrature(int64_t nx, int64_t ny, int64_t nz, const double *vol,
                        const double *inv_affine, int64_t M, const double *centers,
                        const int32_t *sid, const double *axes, int64_t n0, int64_t n1,
                        int64_t n2, const double *nodes, double *out, void *stream);

/* ---- fit setup on the device ---------------------- */

/* One acquisition stack resident on the device (motion.py:21-57 SliceStack):
 * data (nx, ny, ns) f64 and mask (nx, ny, ns) u8 0/1, both C order on the
 * device; affine = the 4x4 index -> mm affine, row-major, by value. */
typedef struct gsvr_stack_view {
  int64_t nx, ny, ns;
  const double *data;
  const uint8_t *mask;
  double affine[16];
} gsvr_stack_view;

/* Masked pixels per slice (stack order, then slice) -> counts (HOST, S int64).
 * Synchronises the stream. */
int gsvr_stack_slice_counts(int n_stacks, const gsvr_stack_view *stacks, int64_t *counts, void *stream);

/* motion.py:183-237 build_point_batch: every masked pixel in stack -> slice ->
 * raster (u, v) order: x0 (P, 3) f64 lifted to mm (x @ A[:3,:3].T + A[:3,3] in
 * OpenBLAS's per-element order), slice_ids (P,) int32 (global slice), values
 * (P,) f64.  slice_counts (HOST, S) from gsvr_stack_slice_counts.  Bit-identical
 * to the reference's numpy on the same host. */
int gsvr_build_points(int n_stacks, const gsvr_stack_view *stacks, const int64_t *slice_counts,
                      double *x0, int32_t *slice_ids, double *intensities, void *stream);

/* initialization.py:44-106 sample_init_positions: weights (1 - lambda_init)
 * |grad| + lambda_init over the pooled masked pixels (stack order, C order
 * inside a stack), numpy's Generator.choice(P, n_draws, p=weights/sum) with the
 * caller's uniforms (device, n_draws f64 = the PCG64 stream's random(n_draws)),
 * drawn pixels lifted -> positions (device, n_draws x 3 f64).  *uniform_fallback
 * (HOST) = 1 when the weights summed to <= 0 and uniform weights were used
 * (the reference warns).  masked_sum (HOST, optional): numpy's sum of the
 * pooled masked values (the 'mean' intensity policy), accumulated in float32
 * when masked_sum_f32 (float32 stack data) else float64.  n_draws may be 0. */
int gsvr_init_sample(int n_stacks, const gsvr_stack_view *stacks, const int64_t *slice_counts,
                     double lambda_init, int64_t n_draws, const double *uniforms, double *positions,
                     int *uniform_fallback, double *masked_sum, int masked_sum_f32, void *stream);

/* initialization.py:109-130 _source_intensity: for every position (device,
 * N x 3) the value of the first stack pixel (stack order) it sits on (|index -
 * rint| < 1e-6 on every axis, in bounds) -> intensities (device, N).
 * inv_affines (HOST, n_stacks x 16): the inverse affines as np.linalg.inv
 * returns them.  *unmatched (HOST) = positions on no pixel (the reference
 * raises). */
int gsvr_init_source_intensity(int n_stacks, const gsvr_stack_view *stacks, const double *inv_affines,
                               int64_t N, const double *positions, double *intensities,
                               int64_t *unmatched, void *stream);

/* The pooled sampling weights alone (initialization.py:44-57, :95-96):
 * weights (device, P f64, P = total masked pixels) in the pooled order. */
int gsvr_init_weights(int n_stacks, const gsvr_stack_view *stacks, const int64_t *slice_counts,
                      double lambda_init, double *weights, void *stream);

/* numpy's np.cumsum of a (n,) f64 device array, in place (the sequential
 * add.accumulate chain, bit-identical; one thread, ~n dependent adds). */
int gsvr_cumsum(int64_t n, double *x, void *stream);

/* numpy's np.add.reduce of a (n,) f64 device array (pairwise summation,
 * bit-identical) -> *out (HOST). */
int gsvr_pairwise_sum(int64_t n, const double *x, double *out, void *stream);

/* ---- diagnostics ------------------------------------------------------- */

/* 1 if every tile of the batch is planar (real slices): gsvr_train_tiles then
 * runs the slice-plane kernel (2D conditional + through-plane form). */
int gsvr_batch_is_planar(const gsvr_batch *batch);
/* general != 0 forces the general 3D tile kernel even on planar batches
 * (process-wide; used to cross-check the two kernels). */
/* Measurement: with timing on, CUDA events are recorded on the launching stream
 * around every tile-kernel launch (k_train_planar / k_train_tiles, not their
 * gradient gathers); gsvr_kernel_time_ms sums their durations (waits for
 * them) and reports the launch count.  Turning timing on resets the record. */
int gsvr_set_kernel_timing(int on);
double gsvr_kernel_time_ms(int64_t *launches);

/* Diagnostics: bit 0 runs the general 3D tile kernel on planar batches, bit 1
 * makes the planar kernel keep its backward record halves in global memory
 * (the large-tile configuration) regardless of size. */
int gsvr_set_kernel_variant(int general);

/* Device -> host copy of `bytes` into any host buffer (pageable numpy arrays go
 * through a ring of pinned staging pieces moved out by host threads).
 * Synchronises the stream. */
int gsvr_copy_d2h(void *dst, const void *src, int64_t bytes, void *stream);

/* Measured FP32 FMA-pipe throughput of this device (TFLOP/s, best of 5). */
int gsvr_probe_fp32_peak(double *tflops_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GSVR_B200_H */
