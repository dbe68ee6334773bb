/* cvx.h — C-ABI of the B200-native coVoxSLAM submap builder (libcvx.so, sm_100a).
 *
 * The four calls of the problem statement (BASELINE.json north_star; §III.C-E):
 *   cvx_create_submap        — a submap = pose + block-hashed voxel volume
 *   cvx_integrate_pointcloud — raycast every point into the TSDF
 *   cvx_finalize_esdf        — exact Euclidean signed distance field
 *   cvx_query_distance       — trilinear distance look-ups
 * plus a batched integrate (same semantics as calling integrate once per frame: fusion is a sum with
 * no weight cap, "commutative and distributive"; reading R6), reset/stats, and the
 * inspection hooks the parity tests and the multi-GPU gather use (export/import/pack).
 *
 * Citations: P:Lnn = PAPER.md line nn, S:Lnn = SPEC.md line nn, O1..O13 / Q1..Q24 = the readings in
 * SURVEY.md §8c, restated in DESIGN.md.
 *
 * Conventions (all calls)
 *  - Every call returns cvx_status; 0 = CVX_OK.  On error cvx_last_error() returns a thread-local
 *    message.  Host-detectable errors (bad arguments, wrong state) return synchronously and leave the
 *    submap unchanged.
 *  - Buffers: pointers documented "device" must be CUDA device pointers on the submap's device (e.g.
 *    torch CUDA tensors' data_ptr()); "host" pointers are ordinary host memory.  The CALLER owns every
 *    buffer it passes; the library owns all submap state (hash table, block pool, ESDF, scratch) and
 *    frees it in cvx_destroy_submap.
 *  - Streams: `stream` is a cudaStream_t (NULL = legacy default stream).  Calls enqueue work on it and
 *    return without a host synchronisation unless documented "synchronising".
 *  - Device-side failures (block pool or hash table full, ray outside the 21-bit key domain) set a
 *    sticky flag; the next synchronising call returns CVX_E_CAPACITY / CVX_E_RANGE.  Dropped work is
 *    counted in the stats.
 *  - A submap is not thread-safe; distinct submaps may be used concurrently from different threads.
 */
#ifndef CVX_H_
#define CVX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t cvx_status;
#define CVX_OK 0
#define CVX_E_INVALID (-1)  /* bad argument (null pointer, bad size, non-orthonormal rotation, ...)  */
#define CVX_E_OOM (-2)      /* device allocation failed                                            */
#define CVX_E_CAPACITY (-3) /* block pool (max_blocks) or hash table overflowed           */
#define CVX_E_STATE (-4)    /* integrate after finalize, query before finalize            */
#define CVX_E_CUDA (-5)     /* CUDA runtime error (no device, launch failure, ...)                 */
#define CVX_E_RANGE (-6)    /* a ray left the 21-bit block-key domain or spans >= 2^15 voxels (O3)  */

/* Voxel grid of one submap.  Blocks of 8^3 voxels (Q17), hashed by 3-D block index
 * (P:L78-85).  voxel_size, truncation, site_threshold, weight_range_floor are metres. */
typedef struct {
  double voxel_size;         /* s > 0                                                              */
  int32_t block_side;        /* must be 8                                                          */
  double truncation;         /* tau >= 2*s: sdf clamp and extent behind the point */
  int32_t weighting;         /* 0 constant w = 1, 1 inverse square w = 1/max(L, floor)^2 (Q5) */
  double weight_range_floor; /* floor of L in the inverse-square weight (default 0.1 m)     */
  int32_t carve;             /* 1: update o -> p + tau*u (default); 0: band p +- tau*u (Q2) */
  double site_threshold;     /* ESDF site: observed and |D| <= site_threshold (O10, Q14; default s) */
  int64_t max_blocks;        /* block pool capacity; the hash table holds >= 2*max_blocks entries   */
  int32_t color;             /* 1: also fuse per-point colour (cvx_integrate_color; TSDF + Color) */
  double esdf_max_distance;  /* d_max > 0 of the incremental ESDF (cvx_update_esdf): distances are clamped
                                there (SPEC S:L373 default 2 m; R11).  cvx_finalize_esdf is exact
                                and unclamped (Q16) and ignores it.                                      */
} cvx_grid_config;

/* Sensor model of the incoming frames. */
typedef struct {
  int32_t kind;             /* 0 unorganised points [n][3]; 1 pinhole depth [height][width];
                               2 organised LiDAR points [height=rings][width=cols][3]               */
  int32_t width, height;    /* organisation; for kind 1 n must equal width*height                   */
  float fx, fy, cx, cy;     /* pinhole intrinsics (kind 1): p_c = (z(u-cx)/fx, z(v-cy)/fy, z) (O2)   */
  float min_range, max_range; /* inclusive range filter on the ray length L (Q10)                   */
} cvx_sensor_model;

typedef struct cvx_submap cvx_submap; /* opaque; owns all device state of one submap */

/* Cumulative counters of a submap since create/reset. */
typedef struct {
  int64_t rays_in;          /* points / pixels received                                            */
  int64_t rays_used;        /* rays traversed                                                      */
  int64_t skipped_invalid;  /* non-finite point, or depth <= 0 / non-finite                */
  int64_t skipped_range;    /* outside [min_range, max_range] (Q10)                                */
  int64_t skipped_domain;   /* outside the fixed-point / 21-bit key domain (O3) -> CVX_E_RANGE      */
  int64_t voxel_updates;    /* sum over used rays of the traversed voxel count (COUNT)  */
  int64_t new_blocks;       /* blocks allocated (ALLOCATE)                                  */
  int64_t total_blocks;     /* blocks in the submap                                                */
} cvx_integrate_stats;

/* Create an empty submap on CUDA device `device` with pose T_world_submap (host, fp64 4x4 row-major,
 * rotation orthonormal within 1e-6, last row 0 0 0 1).  Allocates and zeroes the block pool
 * (16 B TSDF sums + 4 B ESDF per voxel) and the hash table.  Synchronising.
 * Errors: CVX_E_INVALID (config/pose), CVX_E_OOM, CVX_E_CUDA. */
cvx_status cvx_create_submap(const cvx_grid_config* config, const double* T_world_submap, int device,
                             cvx_submap** out);

/* Free all device state of the submap (synchronises the device first).  NULL is a no-op. */
cvx_status cvx_destroy_submap(cvx_submap* submap);

/* Return the submap to the freshly-created state without reallocating: zeroes the used blocks, clears
 * the hash table, AABB, counters and the finalized flag.  Stream-ordered. */
cvx_status cvx_reset_submap(cvx_submap* submap, void* stream);

/* Replace the submap pose T_world_submap (host fp64 4x4, same checks as create).  Intended right after
 * cvx_reset_submap, to reuse one submap's device state for the next submap of a trajectory:
 * work already enqueued keeps the pose it was launched with; later integrate / query calls use the new
 * one.  Not synchronising. */
cvx_status cvx_set_submap_pose(cvx_submap* submap, const double* T_world_submap);

/* Integrate one frame.  `data` (device, fp32): kind 0/2 points [n][3] in the
 * sensor frame, kind 1 depth [height][width] metres (n = width*height).  T_world_sensor: host fp64 4x4
 * row-major.  Every used ray updates every voxel it traverses from the sensor origin to tau behind the
 * point (carve) with the projective sdf d = clamp((p - c_v).u, -tau, tau) and weight w (O4-O6); the TSDF
 * is the weighted average D = sum(w d)/sum(w), W = sum(w) (O8).  n = 0 is a no-op.
 * `stats` (nullable, host): if given the call synchronises `stream` and returns the cumulative counters.
 * Scratch (library-owned, grow-only, allocated stream-ordered on `stream` / the submap's side stream):
 * ray records (48 B per ray) and, with constant weights and no colour, the dense-window accumulators of
 * DESIGN.md R19 — block-major u64 over the block box of each launch's rays, sized on the first call to a
 * conservative box of the call's frames (balls of radius max_range + truncation around the sensor
 * origins) capped at 2^19 blocks = 2 GiB (environment CVX_DENSE_BLOCKS at submap creation; CVX_DENSE=0
 * disables the path); a launch whose box exceeds the buffer takes the slot-list path on the device, and a
 * call whose buffer cannot be allocated takes it on the host — same results either way.  ALLOCATE then
 * runs after the update walk (same block set).  The buffer lives until cvx_destroy_submap.
 * Errors: CVX_E_INVALID, CVX_E_STATE (after finalize), CVX_E_CUDA (also CVX_E_OOM-class CUDA errors when
 * the scratch cannot be allocated); with stats also CVX_E_CAPACITY / CVX_E_RANGE from the sticky flags. */
cvx_status cvx_integrate_pointcloud(cvx_submap* submap, const float* data, int64_t n,
                                    const double* T_world_sensor, const cvx_sensor_model* sensor,
                                    void* stream, cvx_integrate_stats* stats);

/* Integrate n_frames frames of n_per_frame points each in one pass: `data` (device) holds the frames
 * back to back, T_world_sensor (host) holds n_frames row-major 4x4 poses.  The result is identical,
 * bit for bit, to n_frames calls of cvx_integrate_pointcloud (the fused sums are exact fixed-point
 * integers, R6).  Same errors. */
cvx_status cvx_integrate_batch(cvx_submap* submap, const float* data, int64_t n_per_frame,
                               int32_t n_frames, const double* T_world_sensor,
                               const cvx_sensor_model* sensor, void* stream, cvx_integrate_stats* stats);

/* cvx_integrate_batch with the frames in HOST memory (page-locked recommended; pageable memory works
 * but its copies are synchronous): the library copies each launch's frames to the device on its own copy
 * stream into one of two staging buffers, each copy waiting only for the ingest that last read that
 * buffer, so the transfer of launch k+1 overlaps the ingest and update walk of launch k.  The copies are
 * NOT ordered after earlier work on `stream` (they may run under it, e.g. the previous submap's update
 * walk): `host_data` must hold its final contents when the call is made (not be the target of a pending
 * device-to-host copy) and stay valid and unmodified until `stream` has passed this call's work.  Same
 * results and errors. */
cvx_status cvx_integrate_batch_host(cvx_submap* submap, const float* host_data, int64_t n_per_frame,
                                    int32_t n_frames, const double* T_world_sensor,
                                    const cvx_sensor_model* sensor, void* stream, cvx_integrate_stats* stats);

/* Block-count submap trigger ("the area covered by sensor trajectory is approximated by
 * considering the number of blocks used by the current submap"): integrate the frames in
 * order, one launch per frame, and stop after the first frame at which the submap holds
 * >= block_threshold blocks; *frames_integrated (host) = the frames taken (the caller starts the next
 * submap with the rest).  The check runs on the device after each frame's ALLOCATE phase, so the frames
 * are still pipelined; one synchronisation at the end.  Same results as calling
 * cvx_integrate_pointcloud frame by frame and testing the block count after each.  Errors as
 * cvx_integrate_batch; CVX_E_INVALID if block_threshold is not in [1, max_blocks]. */
cvx_status cvx_integrate_until(cvx_submap* submap, const float* data, int64_t n_per_frame, int32_t n_frames,
                               const double* T_world_sensor, const cvx_sensor_model* sensor,
                               int64_t block_threshold, void* stream, int32_t* frames_integrated);

/* TSDF + Color (Fig. 4 "TSDF + Color"; R13): cvx_integrate_batch
 * plus per-point colour `rgb` (device uint8 [n_frames][n_per_frame][3], same order as `data`).  Every
 * update inside the truncation band (|sdf| < tau, before clamping) also adds w*(r,g,b) and w to the
 * voxel's colour sums, so colour = sum(w c) / sum(w) over the band updates.  Requires config.color = 1.
 * Errors as cvx_integrate_batch; CVX_E_INVALID without colour storage or with rgb NULL. */
cvx_status cvx_integrate_color(cvx_submap* submap, const float* data, const uint8_t* rgb, int64_t n_per_frame,
                               int32_t n_frames, const double* T_world_sensor, const cvx_sensor_model* sensor,
                               void* stream, cvx_integrate_stats* stats);

/* Projection-mapping integration (R14) — the KinectFusion / nvBlox voxel-centric
 * update the paper contrasts with its raycasting ("projects voxels in the visual field of
 * view into the depth image and computes their distance from the difference between the voxel centre
 * and the depth value in the image", "associating it with the nearest pixel"), for the in-house
 * raycast-vs-projection comparison.  `depth` (device fp32 [n_frames][height][width] metres) and the
 * poses as cvx_integrate_batch; sensor kind must be 1 (pinhole).  Per frame, in order: ALLOCATE exactly
 * as cvx_integrate_pointcloud (same block set, no update from the rays); then every voxel v of the
 * submap with camera-frame centre x (z = x_2 > 0) whose nearest pixel (floor(fx x_0 / z + cx + 1/2),
 * floor(fy x_1 / z + cy + 1/2)) lies in the image, has a valid depth m and a pixel ray length inside
 * [min_range, max_range] gets sdf = m - z; voxels with sdf < -tau (occluded), and in band mode
 * (carve = 0) sdf > tau, are skipped; d = min(sdf, tau) is fused with the weight of the pixel (O6).
 * Batches equal frame-by-frame calls bit for bit.  stats.voxel_updates counts the projective updates.
 * Errors as cvx_integrate_batch; CVX_E_INVALID for sensor kinds other than 1. */
cvx_status cvx_integrate_projective(cvx_submap* submap, const float* depth, int64_t n_per_frame, int32_t n_frames,
                                    const double* T_world_sensor, const cvx_sensor_model* sensor, void* stream,
                                    cvx_integrate_stats* stats);

/* Export the fused colour in slot order (synchronising): rgb (device fp32 [nb][512][3], 0..255; 0 where no
 * band update) and color_weight (device fp32 [nb][512], nullable).  Errors: CVX_E_INVALID without colour
 * storage, CVX_E_CAPACITY if nb > capacity_blocks. */
cvx_status cvx_export_color(const cvx_submap* submap, float* rgb, float* color_weight, int64_t capacity_blocks,
                            int64_t* n_out, void* stream);

/* Cumulative counters (synchronising). Returns the sticky device errors. */
cvx_status cvx_get_stats(const cvx_submap* submap, cvx_integrate_stats* out);

/* Number of allocated blocks (synchronising).  Returns the sticky device errors. */
cvx_status cvx_get_block_count(const cvx_submap* submap, int64_t* out);

/* Allocated-block AABB in block coordinates, lo/hi inclusive (host int32[3] each; synchronising).
 * Empty submap: lo > hi. */
cvx_status cvx_get_aabb(const cvx_submap* submap, int32_t* lo, int32_t* hi);

/* Exact ESDF over the allocated blocks (O10-O12): sites S = {v : W(v) > 0 and
 * |D(v)| <= site_threshold}; E(v) = sign(D(v)) * s * sqrt(min_{u in S} |v - u|^2) for observed v,
 * NaN for unobserved v, +inf for every observed v if S is empty.  Marks the submap finalized (no more
 * integration); calling it again recomputes the same ESDF (the TSDF is immutable).
 * Synchronising (reads the block count / AABB to size the dense EDT domain).  The dense AABB may span at
 * most 46336 voxels per axis (2-D squared distances fit 32 bits), else CVX_E_RANGE.  Scratch (6 bytes per
 * AABB voxel) is allocated stream-ordered (cudaMallocAsync) and kept for the next call.
 * Errors: CVX_E_CAPACITY / CVX_E_RANGE (sticky), CVX_E_OOM. */
cvx_status cvx_finalize_esdf(cvx_submap* submap, void* stream);

/* Incremental ESDF (R11): keep the ESDF of a submap that is still
 * being integrated current, recomputing only the blocks a change can reach.  The value maintained is the
 * exact EDT of cvx_finalize_esdf clamped at d_max = config.esdf_max_distance:
 *   E(v) = sign(D(v)) * min(s * sqrt(min_{u in S} |v - u|^2), d_max) for observed v (d_max if S is empty),
 *   NaN for unobserved v,
 * identical for every update schedule (after any sequence of integrate / update calls it equals the
 * clamped exact EDT of the current TSDF).  A site within d_max of a voxel lies within r = ceil(d_max / s)
 * voxels per axis, so each call classifies every allocated block (observed / sign / site bit-planes from
 * the fused sums), queues every block within ceil(r / 8) blocks of a block whose sites changed (raise and
 * lower alike) plus the blocks whose own planes changed or that are new (one region queue per 8^3 block,
 * P:L147), and recomputes each queued block exactly from the sites around it.  Windows of more than 7^3
 * blocks (d_max > 24 s) use the dense exact EDT of finalize with the clamp.  Enables cvx_query_distance.
 * Synchronising.  *blocks_updated (nullable, host) = the number of blocks recomputed.  Errors:
 * CVX_E_CAPACITY / CVX_E_RANGE (sticky), CVX_E_OOM. */
cvx_status cvx_update_esdf(cvx_submap* submap, void* stream, int32_t* blocks_updated);

/* Distance queries (O13).  points_world (device fp32 [m][3], world frame) ->
 * out_distance (device fp32 [m]) and out_status (device uint8 [m]: 0 OK trilinear over the 8 voxel
 * centres around x, 1 NEAREST = value of the voxel containing x, 2 UNKNOWN = NaN).
 * Errors: CVX_E_STATE before finalize / update_esdf, CVX_E_INVALID. */
cvx_status cvx_query_distance(const cvx_submap* submap, const float* points_world, int64_t m,
                              float* out_distance, uint8_t* out_status, void* stream);

/* Registration look-ups: cvx_query_distance plus the world-frame gradient of
 * the trilinear interpolant, grad (device fp32 [m][3]) = R_WS dE/dx_s; NaN unless status is OK.
 * Same errors as cvx_query_distance. */
cvx_status cvx_query_distance_gradient(const cvx_submap* submap, const float* points_world, int64_t m,
                                       float* out_distance, float* out_gradient, uint8_t* out_status,
                                       void* stream);

/* Weight-proportional surface-point sampling for registration (R12):
 * candidates = sites (observed, |D| <= site_threshold) in lexicographic (bx,by,bz) block order then
 * local index order, with integer weights W in units of 2^-20; each uniform u (device uint32 [m]) picks
 * the first candidate whose prefix sum exceeds floor(T u / 2^32) (T = total weight).  out_xyz (device
 * fp32 [m][3]) = the voxel centre in the world frame (NaN if there is no site), out_weight (device fp32
 * [m], nullable) = its W; *total_weight (host, nullable) = T.  Synchronising.  Works before and after
 * finalize.  Errors: CVX_E_INVALID, CVX_E_OOM, CVX_E_CUDA. */
cvx_status cvx_sample_surface(cvx_submap* submap, const uint32_t* uniforms, int64_t m, float* out_xyz,
                              float* out_weight, int64_t* total_weight, void* stream);

/* Export every allocated block in slot order (synchronising): bxyz (device int32 [nb][3] block coords),
 * D, W (device fp32 [nb][512], local index lx + 8 ly + 64 lz; D = sum(w d)/sum(w), 0 if W = 0), E
 * (device fp32 [nb][512] or NULL; valid after finalize).  capacity_blocks bounds nb; *n_out = nb.
 * Any of bxyz/D/W/E may be NULL to skip it.  Errors: CVX_E_CAPACITY if nb > capacity_blocks. */
cvx_status cvx_export_blocks(const cvx_submap* submap, int32_t* bxyz, float* D, float* W, float* E,
                             int64_t capacity_blocks, int64_t* n_out, void* stream);

/* Import TSDF blocks (device bxyz int32 [n][3], D, W fp32 [n][512]) into a non-finalized submap,
 * replacing the content of those blocks (used for stage-isolated ESDF parity and the ESDF stress
 * config).  Stream-ordered. */
cvx_status cvx_import_tsdf_blocks(cvx_submap* submap, const int32_t* bxyz, const float* D,
                                  const float* W, int64_t n_blocks, void* stream);

/* Pack the finalized ESDF for the multi-GPU gather (synchronises `stream`): dst (device) receives a
 * 256-byte header {u32 magic 'CVXE', i32 version 1, i64 n_blocks, f64 voxel_size, f64 T_world_submap[16],
 * zero padding} followed by n_blocks records {i32 bx, by, bz, slot; f32 E[512]} (2064 B each).
 * *used = bytes written.  dst = NULL: only *used = the bytes needed (ordered after `stream`'s work, unlike
 * cvx_packed_size, which synchronises the whole device).  Errors: CVX_E_STATE before finalize,
 * CVX_E_CAPACITY if dst_bytes too small. */
cvx_status cvx_pack_esdf(const cvx_submap* submap, void* dst, int64_t dst_bytes, int64_t* used,
                         void* stream);

/* Bytes cvx_pack_esdf needs (synchronises the whole device; see cvx_pack_esdf with dst = NULL). */
cvx_status cvx_packed_size(const cvx_submap* submap, int64_t* bytes);

/* Gathered submap ESDFs (SURVEY §8 e / f4; registration queries "between every overlapped
 * submap" — the consumer of the multi-GPU gather).  `payloads` (device) holds n_submaps cvx_pack_esdf
 * payloads (e.g. the output of an all-gather), payload k starting at byte offsets[k] (host int64 [n],
 * 16-byte aligned) inside a buffer of payload_bytes.  The set indexes the records in place: the CALLER keeps
 * `payloads` alive and unmodified until cvx_esdf_set_destroy.  Each submap keeps its own pose and voxel
 * size from its header.  Synchronising (reads the headers, builds the index on `stream`).
 * Errors: CVX_E_INVALID (bad header / offsets, a block listed twice, a payload not from a finalized
 * submap), CVX_E_OOM, CVX_E_CUDA. */
typedef struct cvx_esdf_set cvx_esdf_set;
cvx_status cvx_esdf_set_create(const void* payloads, int64_t payload_bytes, const int64_t* offsets, int32_t n_submaps,
                               int device, void* stream, cvx_esdf_set** out);
cvx_status cvx_esdf_set_destroy(cvx_esdf_set* set);

/* Batched look-ups across the set: point i (device fp32 [m][3], world frame) is queried in submap
 * submap_index[i] (device int32 [m]) exactly as cvx_query_distance_gradient queries that submap (O13 in
 * the submap's own frame: trilinear / NEAREST / UNKNOWN, world-frame gradient).  out_gradient (device fp32
 * [m][3]) may be NULL.  An index outside [0, n_submaps) gives UNKNOWN.  Stream-ordered.
 * Errors: CVX_E_INVALID, CVX_E_CUDA. */
cvx_status cvx_esdf_set_query(const cvx_esdf_set* set, const int32_t* submap_index, const float* points_world,
                              int64_t m, float* out_distance, float* out_gradient, uint8_t* out_status, void* stream);

/* Per-kernel timing of this submap's launches with CUDA events recorded on the launching stream
 * (off by default; enabling synchronises the device and clears earlier records).  enable: bit 0 =
 * record, bit 1 = serialise (the integration pipeline's side-stream work runs on the caller's stream,
 * so every kernel runs alone and its event time is its solo time).  Used by bench.py for the roofline
 * of the dominant kernel and the per-kernel shares. */
cvx_status cvx_profile_enable(cvx_submap* submap, int32_t enable);

/* Synchronising: writes a JSON object {"kernel": {"ms": total_ms, "n": launches}, ...} of the records
 * since the last report into buf (host, buflen bytes) and clears them.  CVX_E_CAPACITY if too small. */
cvx_status cvx_profile_report(cvx_submap* submap, char* buf, int64_t buflen);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* cvx_last_error(void);

/* Library build string (arch, version). */
const char* cvx_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CVX_H_ */
