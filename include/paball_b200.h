/*
 * paball_b200.h — C ABI of the B200-native SlingBAG Pro hot path.
 *
 * The reference (`paball`, pure Python/numpy) has no FFI: its single internal
 * seam is radiator._run_model(cloud, ctx, f, real, stage)
 * (/root/reference/pkg/src/paball/radiator.py:290), reached from
 * simulate_signals (:362), simulate_at_rate (:368) and backward (:419), plus
 * the driver's Adam update (optimizer.py:203-209) and cloud compaction
 * (model.py:239-244 via optimizer.py:255-256).  The entry points below are
 * what a binding of that seam needs (INTEGRATION.md shows the ctypes stub).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless stated; sizes are element
 *    counts; `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - Every function returns 0 on success, 1 on a bad argument, 4 when a CUDA
 *    launch failed.  Nothing throws across the boundary.
 *  - Device status words (int) collect per-pass error bits:
 *      2  ball coincident with a detector   -> SimulationError (radiator.py:190-193)
 *      8  non-finite gradient               -> OptimizationError (optimizer.py:284-294)
 *  - Ball clouds are packed once per change by pab_pack into processing order
 *    (lane groups of 32 balls ordered by a0 bucket, then 3-D Hilbert index).
 *    Record sizes: pab_record_sizes.
 *  - Detector auxiliary data `det_aux` is [n_det][9] doubles: receive
 *    direction (unit, = -outward normal), element axes e1, e2.
 *  - Directivity: dir_kind 0 none (reference semantics), 1 cos^p (dir_param =
 *    p), 2 square element of width dir_param metres.
 *  - Acquisition: v sound speed, t0/dt the FULL-rate grid, f the decimation
 *    factor, n_out = ceil(n_samples / f) the decimated sample count;
 *    n_out * f <= 2^21 (sample indices are rounded with FP32 magic constants
 *    off the conversion pipe; pab_forward / pab_adjoint return 1 beyond).
 */
#ifndef PABALL_B200_H
#define PABALL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int pab_version(void);
int pab_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, int* max_smem_optin);
const char* pab_last_cuda_error(void);
int pab_record_sizes(int* ball_a, int* ball_b, int* group_meta);

/* ---- Host staging of the API edge (no GPU work) ----
 * Copy `bytes` (resp. narrow n float64 to float32) from a pageable caller
 * array into a 16-byte aligned page-locked staging buffer with non-temporal
 * stores on `threads` threads, so the following upload DMA reads DRAM
 * instead of snooping dirty cache lines.  Return 0, or 1 on a bad argument.
 * Replaces: the implicit float64 reads of caller arrays (radiator.py:316-332). */
int pab_host_stage_copy(void* dst, const void* src, size_t bytes, int threads);
int pab_host_stage_narrow(float* dst, const double* src, size_t n, int threads);

/* Bounds of a cloud on the device: bounds[0..2] = min x, y, z, bounds[3] =
 * extent (largest side of the bounding box; 1 if degenerate), bounds[4..5] =
 * min / max a0 (exact min/max: deterministic).  workspace:
 * pab_cloud_bounds_workspace_bytes().  No host round trip. */
size_t pab_cloud_bounds_workspace_bytes(void);
int pab_cloud_bounds(const double* pos, const double* a0, int64_t n, double* bounds, void* workspace, void* stream);

/* pab_morton_keys with the cube and a0 range read from device `bounds`
 * (pab_cloud_bounds): the same keys, no host round trip. */
int pab_sort_keys(const double* pos, const double* a0, int64_t n, const double* bounds, int a0_buckets,
                  int64_t* keys, void* stream);

/* Stable LSD radix sort (five 7-bit passes over key bits [28, 63); the low
 * 28 bits are the input index, already ascending) of pab_sort_keys /
 * pab_morton_keys keys; writes perm[k] = index of the k-th smallest key.
 * `keys` is overwritten (ping-pong buffer).  workspace:
 * pab_sort_perm_workspace_bytes(n).  n < 2^28.
 * Replaces: nothing in the reference (it visits balls in input order); the
 * order only fixes the deterministic FP32 summation order. */
size_t pab_sort_perm_workspace_bytes(int64_t n);
int pab_sort_perm(int64_t* keys, int64_t n, int32_t* perm, void* workspace, void* stream);

/* Processing-order sort keys: key[i] = a0_bucket << 58 | hilbert30(pos[i]) << 28 | i
 * (hilbert30: 10-bit-per-axis 3-D Hilbert index of the position in the cube
 * [lo, lo + extent)^3; a0 buckets: a0_buckets equal bins of [a0lo, a0hi]; n < 2^28).
 * (The entry point keeps its first-version name; the key is a Hilbert key.)
 * Replaces: nothing (the reference visits balls in input order, radiator.py:185). */
int pab_morton_keys(const double* pos /*[n][3]*/, const double* a0, int64_t n, double lox, double loy,
                    double loz, double extent, double a0lo, double a0hi, int a0_buckets, int64_t* keys,
                    void* stream);

/* Pack a cloud (caller order, FP64 SoA) into processing-order records.
 * perm[i] = caller index of the i-th processed ball, or -1 for an inert
 * padding slot.  rec_a/rec_b hold
 * ceil(n/32)*32 records of 16 bytes, group_meta ceil(n/32) records of 48 bytes.
 * Replaces: PointCloud field coercion (model.py:186-205) at the radiator boundary. */
int pab_pack(const double* pos, const double* p0, const double* a0, const int32_t* perm /*-1: padding*/, int64_t n,
             void* rec_a, void* rec_b, void* group_meta, void* stream);

/* Exact FP64 ball-on-sensor test of a packed cloud: sets kStatusCoincident
 * (2) in *status when any ball of `pos` (caller order, [n][3]) lies within
 * 1e-12 of a detector (bounding-box prefilter per lane group).
 * Replaces: the distance check of radiator.py:189-193. */
int pab_coincident(const void* rec_b, const void* group_meta, int64_t n_groups, const double* pos,
                   const double* det_pos, int n_det, int* status, void* stream);

/* Dual-walk pairing table of a packed cloud (performance only): for each pair
 * of consecutive lane groups and each of 64 fixed directions, the 64 balls in
 * projection order, laid out [cell][unit][64] (pab_pair_table_bytes(n_groups)
 * bytes).  Rebuild after
 * every pab_pack.
 * Replaces: nothing (the reference evaluates balls one by one). */
size_t pab_pair_table_bytes(int64_t n_groups);
int pab_pair_table(const void* rec_a, const void* group_meta, int64_t n_groups, unsigned char* table,
                   void* stream);

/* Forward model: partial_rows[partitions][n_det][n_out] (FP32) for the given
 * detector set.  ops_total += in-window samples (the reference op counter).
 * `wide_list` (device, partitions * n_det * (wide_cap + 1) ints) is scratch
 * through which the sweep hands the groups wider than its tile to a second
 * kernel (per detector x partition: a count, then up to wide_cap group
 * indices; a larger count makes that kernel find them again itself).
 * `warps` = walker warps per CTA (the CTA also runs as many setup-producer
 * warps); `groups_per_cell` and `tile_rows` are reserved (ignored: the tile
 * height is a build constant).  `pair_table` (nullable) enables the dual
 * walk (two balls per lane) for cutoffs >= 5.8 sigma.
 * Replaces: radiator._block_pass forward (radiator.py:157-261). */
size_t pab_forward_smem_bytes(int n_out, int warps, int tile_rows);
int pab_forward(const void* rec_a, const void* rec_b, const void* group_meta, const unsigned char* pair_table,
                int64_t n_groups,
                const double* det_pos /*[n_det][3]*/, const double* det_aux /*[n_det][9]*/, int n_det,
                double v, double t0, double dt, int f, int n_out, double cutoff, int dir_kind,
                double dir_param, int groups_per_cell, int partitions, int warps, int tile_rows,
                float* partial_rows, int* wide_list, int wide_cap, unsigned long long* ops_total, int* status,
                void* stream);

/* Sum forward partitions; with `real` (nullable) write res = sim - real and
 * per-detector FP64 sum of squares to loss_rows, else write sim.
 * Replaces: radiator.py:263-264 (residual, loss part) and the block merge :339-344. */
int pab_residual(const float* partial_rows, int partitions, int n_det, int n_out, const float* real,
                 float* out, double* loss_rows, void* stream);

/* Adjoint: per-ball partial gradient sums grad_partial[chunks][5][n_groups*32]
 * from res[n_det][n_out] * res_sign (res_sign = -1 with `real` gives the
 * zero-pressure filter probe, optimizer.py:251-253).  stage 0 filter (p0),
 * 1 coarse (p0, a0), 2 fine (p0, a0, position).
 * Replaces: radiator.py:266-287 (gather + reductions). */
int pab_adjoint(const void* rec_a, const void* rec_b, const void* group_meta, int64_t n_groups,
                const double* det_pos, const double* det_aux, int n_det, double v, double t0, double dt,
                int f, int n_out, double cutoff, int dir_kind, double dir_param, const float* res,
                float res_sign, int stage, int chunks, int warps, double* grad_partial,
                unsigned long long* ops_total, int* status, void* stream);

/* Sum chunk partials in order, multiply by `scale` (2 / (n_det_total * n_out)),
 * scatter to caller order: d_p0[n], d_a0[n] (nullable), d_pos[n][3] (nullable).
 * Replaces: radiator.py:345-348, 356-358. */
int pab_grad_finalize(const double* grad_partial, int chunks, int64_t n_groups, const void* rec_b, double scale,
                      int stage, double* d_p0, double* d_a0, double* d_pos, int* status, void* stream);

/* Pass tail (4 doubles) appended to the per-ball gradient buffer, so that
 * one all-reduce per iteration carries gradients, loss, error flags and op
 * count across detector shards: tail[0] = sum of loss_rows[0..n_rows) in row
 * order (loss_rows nullable: 0), tail[1] = 1 if *status has the coincident
 * bit (SimulationError), tail[2] = 1 if it has the non-finite bit
 * (OptimizationError), tail[3] = *ops (nullable: 0).  After the sum over
 * ranks every rank raises the same error at the same step.
 * Replaces: the merge of block losses and op counts, radiator.py:336-344,
 * and the finite check of optimizer.py:284-294. */
int pab_pass_tail(const double* loss_rows, int n_rows, const unsigned long long* ops, const int* status,
                  double* tail, void* stream);

/* Pure decimation of FP32 rows: dst[r][k] = src[r][k*f], k < ceil(n_in/f).
 * Replaces: radiator.downsample (radiator.py:382-390). */
int pab_decimate(const float* src, int n_rows, int n_in, int f, float* dst, void* stream);

/* One Adam update of `count` FP64 values with bias corrections bc1 = 1-0.9^t,
 * bc2 = 1-0.999^t; use_floor applies max(value, floor_value).
 * Replaces: optimizer._adam_update (optimizer.py:203-209) and :298-304. */
int pab_adam(double* param, const double* grad, double* m, double* v, int64_t count, double lr, double bc1,
             double bc2, double floor_value, int use_floor, void* stream);

/* Stable compaction: idx_out <- ascending indices i with key[i] < 0 (mode 0),
 * <= 0 (mode 1), != 0 (mode 2), > 0 (mode 3) or == 0 (mode 4); *count_dev <-
 * their number.
 * Replaces: the boolean subset in optimizer.py:255-256 / model.py:239-244. */
size_t pab_compact_workspace_bytes(int64_t n);
int pab_compact(const double* key, int64_t n, int mode, int32_t* idx_out, int* count_dev, void* workspace,
                void* stream);

/* *out = sum_i (a[i] - b[i])^2 in FP64 (b nullable), fixed summation order.
 * Replaces: radiator.loss (radiator.py:393-402). */
size_t pab_sumsq_workspace_bytes(int64_t n);
int pab_sumsq_diff_f64(const double* a, const double* b, int64_t n, double* out, void* workspace, void* stream);

/* dst[r][c] = src[idx[r]][c] for r < m, c < width (FP64). */
int pab_gather_f64(const double* src, int width, const int32_t* idx, int64_t m, double* dst, void* stream);

/* ---- Adaptive density control (optimizer.py:314-406) ----
 * Exact k-th smallest (0-based) of x by 8-pass radix selection (workspace:
 * pab_select_workspace_bytes); the median is the mean of the two middle order
 * statistics for even n, as numpy's. */
size_t pab_select_workspace_bytes(void);
int pab_select_kth_f64(const double* x, int64_t n, int64_t k, double* out, void* workspace, void* stream);
/* key[i] = -1 keep / +1 destroy: p0 < frac * median or a0 outside [a0_min, a0_max]
 * (median_hi nullable: odd n).  Replaces optimizer.py:330-334. */
int pab_density_keep_key(const double* p0, const double* a0, int64_t n, const double* median_lo,
                         const double* median_hi, double frac, double a0_min, double a0_max, double* key,
                         void* stream);
/* key[i] = -1 split (a0 > split_a0) / +1 parent.  Replaces optimizer.py:349-350. */
int pab_density_split_key(const double* a0, int64_t n, double split_a0, double* key, void* stream);
/* out[r] = |v[idx[r]]| (idx nullable), numpy's sqrt((x*x + y*y) + z*z).  Replaces optimizer.py:345. */
int pab_row_norms(const double* v, const int32_t* idx, int64_t m, double* out, void* stream);
/* Duplicate selection (optimizer.py:378-384): key = -1 for gn > t, 0 for gn == t,
 * +1 below; then the first k_dup - n_above ties (ascending) are set to -1. */
int pab_density_dup_key(const double* gn, int64_t m, const double* t, double* key, void* stream);
int pab_density_take_ties(const int32_t* ties, const int* n_ties, const int* n_above, int k_dup, int64_t m,
                          double* key, void* stream);
/* Split children (optimizer.py:352-357): +child rows [0, m), -child rows [m, 2m). */
int pab_split_children(const double* pos, const double* p0, const double* a0, const double* unit, int64_t m,
                       double* out_pos, double* out_p0, double* out_a0, void* stream);
/* Duplicates (optimizer.py:385-389): pos + (a0 / 4) unit, p0 and a0 copied. */
int pab_duplicate(const double* pos, const double* p0, const double* a0, const double* unit, int64_t m,
                  double* out_pos, double* out_p0, double* out_a0, void* stream);

/* ---- positivity refinement ----------------------------
 * Replaces: optimizer.softplus (optimizer.py:507-510) and the chain-rule
 * factor d_a0 * sigmoid(a0_free) of positivity_refine (optimizer.py:526-533,
 * :563); FP64, the reference's expression trees. */
int pab_softplus_f64(const double* x, int64_t n, double* y, void* stream);
int pab_mul_sigmoid_f64(const double* g, const double* x, int64_t n, double* out, void* stream);

/* ---- voxelisation ------------------------------------
 * Replaces: render.voxelize (render.py:55-93).  order[r] = index of the r-th
 * ball in the canonical lexicographic (x, y, z, p0, a0) order (render.py:67-70).
 * Three passes: per-ball clipped voxel box and 8^3-brick count; (brick << 32 |
 * rank) keys at exclusive-scan offsets (caller sorts them ascending); per-brick
 * gather writing vol[nx][ny][nz] (FP64, every voxel written). */
int64_t pab_vox_brick_count(int nx, int ny, int nz);
int pab_vox_count(const double* pos, const double* p0, const double* a0, const int64_t* order, int64_t n, int nx,
                  int ny, int nz, double spacing, double ox, double oy, double oz, double support,
                  int* box /*[n][6]*/, int64_t* count /*[n]*/, void* stream);
int pab_vox_emit(const int* box, const int64_t* offset, int64_t n, int nx, int ny, int nz, int64_t* keys,
                 void* stream);
int pab_vox_gather(const double* pos, const double* p0, const double* a0, const int64_t* order, const int* box,
                   const int64_t* sorted_keys, int64_t total, int nx, int ny, int nz, double spacing, double ox,
                   double oy, double oz, double support, int64_t* start /*[bricks]*/, int64_t* end /*[bricks]*/,
                   double* vol, void* stream);

/* ---- universal back-projection baseline --------------
 * Replaces: baseline.ubp_reconstruct (baseline.py:52-89).  signals[n_det][n]
 * FP64 rows; det_pos[n_det][3]; vol[nx][ny][nz] receives
 * (1/J) sum_j [2 p_j(t) - 2 t dp_j/dt], t = |x - r_j| / v, detectors summed in
 * index order; *skipped (zeroed by the caller) += voxel-sensor pairs with t
 * outside [t0, t0 + (n-1) dt].  deriv_scratch: n_det * n doubles (np.gradient
 * of the rows).  Returns 1 for n < 2 with detectors, empty dims or null
 * buffers. */
int pab_ubp(const double* signals, int n_det, int n_samples, double t0, double dt, const double* det_pos,
            double sound_speed, int nx, int ny, int nz, double spacing, double ox, double oy, double oz,
            double* deriv_scratch, double* vol, unsigned long long* skipped, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PABALL_B200_H */
