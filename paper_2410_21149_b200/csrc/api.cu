// api.cu — the C-ABI entry points of libcvx (include/cvx.h): argument checks, error codes, the
// thread-local last error, device selection, stream-ordered launches.  No compute happens here;
// every step of the path runs in the kernels of integrate.cu / esdf.cu / query.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "esdf_set.h"
#include "submap.h"

namespace {

thread_local std::string g_last_error;

cvx_status fail(cvx_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

cvx_status cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear the non-sticky error
  return fail(e == cudaErrorMemoryAllocation ? CVX_E_OOM : CVX_E_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

bool valid_pose(const double* T) {
  if (!T) return false;
  for (int i = 0; i < 16; ++i) if (!std::isfinite(T[i])) return false;
  if (T[12] != 0.0 || T[13] != 0.0 || T[14] != 0.0 || T[15] != 1.0) return false;
  for (int i = 0; i < 3; ++i)         // R^T R = I within 1e-6
    for (int j = 0; j < 3; ++j) {
      double d = 0;
      for (int k = 0; k < 3; ++k) d += T[4 * k + i] * T[4 * k + j];
      if (std::fabs(d - (i == j ? 1.0 : 0.0)) > 1e-6) return false;
    }
  return true;
}

cvx_status check_sensor(const cvx_sensor_model* s, int64_t n_per_frame) {
  if (!s) return fail(CVX_E_INVALID, "sensor model is NULL");
  if (s->kind < 0 || s->kind > 2) return fail(CVX_E_INVALID, "sensor kind must be 0, 1 or 2");
  if (!(s->min_range >= 0.0f) || !(s->max_range >= s->min_range))
    return fail(CVX_E_INVALID, "need 0 <= min_range <= max_range");
  if (s->kind == 1) {
    if (s->width <= 0 || s->height <= 0 || (int64_t)s->width * s->height != n_per_frame)
      return fail(CVX_E_INVALID, "pinhole depth: n must equal width*height");
    if (!(s->fx != 0.0f) || !(s->fy != 0.0f) || !std::isfinite(s->fx) || !std::isfinite(s->fy) ||
        !std::isfinite(s->cx) || !std::isfinite(s->cy))
      return fail(CVX_E_INVALID, "pinhole intrinsics must be finite with fx, fy != 0");
  }
  if (s->kind == 2 && s->width > 0 && s->height > 0 && (int64_t)s->width * s->height != n_per_frame)
    return fail(CVX_E_INVALID, "organised LiDAR: n must equal width*height");
  return CVX_OK;
}

// Counter read-back.  Calls that take a stream read after that stream's work; the stream-less
// synchronising calls (get_stats / get_block_count / get_aabb / packed_size) pass whole_device and wait for
// the whole device first, so work on non-blocking streams (e.g. torch's pool streams) is included.
cvx_status read_counters(const cvx_submap* sm, cudaStream_t st, cvx::Counters* out, bool whole_device = false) {
  // a fold deferred by the last integrate call changes the block count / AABB: apply it first (R19)
  if (cudaError_t fe = cvx::flush_fold(const_cast<cvx_submap*>(sm), st)) return cuda_fail(fe, "deferred fold");
  if (whole_device) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "synchronising before the counter read");
  }
  cudaError_t e = cudaMemcpyAsync(sm->ctr_host, sm->ctr, sizeof(cvx::Counters), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "reading submap counters");
  *out = *sm->ctr_host;
  return CVX_OK;
}

cvx_status sticky(const cvx::Counters& c) {
  if (c.err & (cvx::kErrCapacity | cvx::kErrHashFull))
    return fail(CVX_E_CAPACITY, (c.err & cvx::kErrCapacity) ? "block pool overflow (max_blocks too small)"
                                                            : "hash table full");
  if (c.err & cvx::kErrRange) return fail(CVX_E_RANGE, "a ray or block left the 21-bit key / fixed-point domain");
  return CVX_OK;
}

void fill_stats(const cvx::Counters& c, int max_blocks, cvx_integrate_stats* s) {
  s->rays_in = (int64_t)c.rays_in;
  s->rays_used = (int64_t)c.rays_used;
  s->skipped_invalid = (int64_t)c.skipped_invalid;
  s->skipped_range = (int64_t)c.skipped_range;
  s->skipped_domain = (int64_t)c.skipped_domain;
  s->voxel_updates = (int64_t)c.voxel_updates;
  s->new_blocks = (int64_t)c.new_blocks;
  s->total_blocks = c.n_blocks < max_blocks ? c.n_blocks : max_blocks;
}

void free_all(cvx_submap* sm) {
  if (sm->hash.e) cudaFree(sm->hash.e);
  if (sm->pool.sums) cudaFree(sm->pool.sums);
  if (sm->pool.acc) cudaFree(sm->pool.acc);
  if (sm->pool.csum) cudaFree(sm->pool.csum);
  if (sm->pool.cacc) cudaFree(sm->pool.cacc);
  if (sm->pool.esdf) cudaFree(sm->pool.esdf);
  if (sm->pool.coords) cudaFree(sm->pool.coords);
  if (sm->pool.grid) cudaFree(sm->pool.grid);
  if (sm->ctr) cudaFree(sm->ctr);
  if (sm->acc_dirty) cudaFree(sm->acc_dirty);
  if (sm->dacc) cudaFree(sm->dacc);
  if (sm->dcacc) cudaFree(sm->dcacc);
  if (sm->ctr_host) cudaFreeHost(sm->ctr_host);
  for (auto& B : sm->buf) {
    if (B.frame_T) cudaFree(B.frame_T);
    if (B.rays) cudaFree(B.rays);
    if (B.rgbs) cudaFree(B.rgbs);
    if (B.ws) cudaFree(B.ws);
    if (B.slot_lists) cudaFree(B.slot_lists);
    if (B.lcnt) cudaFree(B.lcnt);
    if (B.cta_box) cudaFree(B.cta_box);
    if (B.cstat) cudaFree(B.cstat);
    if (B.staging) cudaFree(B.staging);
  }
  if (sm->side) cudaStreamDestroy(sm->side);
  if (sm->wstream) cudaStreamDestroy(sm->wstream);
  for (auto& e : sm->ev_w) if (e) cudaEventDestroy(e);
  if (sm->copy) cudaStreamDestroy(sm->copy);
  for (int b = 0; b < 2; ++b) {
    if (sm->ev_staged[b]) cudaEventDestroy(sm->ev_staged[b]);
    if (sm->ev_stage_free[b]) cudaEventDestroy(sm->ev_stage_free[b]);
  }
  if (sm->ev_entry) cudaEventDestroy(sm->ev_entry);
  if (sm->ev_walked) cudaEventDestroy(sm->ev_walked);
  for (int b = 0; b < 2; ++b) {
    if (sm->ev_prepared[b]) cudaEventDestroy(sm->ev_prepared[b]);
    if (sm->ev_free[b]) cudaEventDestroy(sm->ev_free[b]);
  }
  cvx::release_esdf(sm);
  if (sm->proj_birth) cudaFree(sm->proj_birth);
  if (sm->trig) cudaFree(sm->trig);
  if (sm->trig_host) cudaFreeHost(sm->trig_host);
  delete sm->prof;
  sm->prof = nullptr;
}

}  // namespace

extern "C" {

const char* cvx_last_error(void) { return g_last_error.c_str(); }

const char* cvx_version(void) { return "libcvx 0.1 (sm_100a; coVoxSLAM submap TSDF+ESDF, arXiv 2410.21149)"; }

cvx_status cvx_create_submap(const cvx_grid_config* cfg, const double* T_world_submap, int device,
                             cvx_submap** out) {
  g_last_error.clear();
  if (!cfg || !out) return fail(CVX_E_INVALID, "config and out must be non-NULL");
  *out = nullptr;
  if (!(cfg->voxel_size > 0) || !std::isfinite(cfg->voxel_size)) return fail(CVX_E_INVALID, "voxel_size must be > 0");
  if (cfg->block_side != 8) return fail(CVX_E_INVALID, "block_side must be 8");
  if (!(cfg->truncation > 0) || !std::isfinite(cfg->truncation)) return fail(CVX_E_INVALID, "truncation must be > 0");
  if (cfg->weighting != 0 && cfg->weighting != 1) return fail(CVX_E_INVALID, "weighting must be 0 or 1");
  if (cfg->weighting == 1 && !(cfg->weight_range_floor > 0)) return fail(CVX_E_INVALID, "weight_range_floor must be > 0");
  if (cfg->carve != 0 && cfg->carve != 1) return fail(CVX_E_INVALID, "carve must be 0 or 1");
  if (!(cfg->site_threshold >= 0) || !std::isfinite(cfg->site_threshold)) return fail(CVX_E_INVALID, "site_threshold must be >= 0");
  if (cfg->max_blocks < 1 || cfg->max_blocks >= (1ll << 23)) return fail(CVX_E_INVALID, "max_blocks must be in [1, 2^23)");
  if (cfg->color != 0 && cfg->color != 1) return fail(CVX_E_INVALID, "color must be 0 or 1");
  if (!(cfg->esdf_max_distance > 0) || !std::isfinite(cfg->esdf_max_distance))
    return fail(CVX_E_INVALID, "esdf_max_distance must be > 0 and finite");
  if (!valid_pose(T_world_submap)) return fail(CVX_E_INVALID, "T_world_submap must be a finite rigid 4x4 (orthonormal within 1e-6)");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(CVX_E_INVALID, "device index out of range");
  DeviceGuard g(device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");

  cvx_submap* sm = new cvx_submap();
  sm->prof = new cvx::Prof();
  if (const char* ag = std::getenv("CVX_AGGREGATE")) sm->aggregate = ag[0] != '0';  // tuning knob
  if (const char* b2 = std::getenv("CVX_BW2")) sm->bw2 = b2[0] != '0';              // tuning knob
  if (const char* b3 = std::getenv("CVX_BW3")) sm->bw3 = b3[0] != '0';              // tuning knob
  if (const char* wc = std::getenv("CVX_WALK_CW")) sm->walk_cw = wc[0] != '0';     // tuning knob
  if (const char* fa = std::getenv("CVX_FUSE_ALLOC")) sm->fuse_alloc = fa[0] != '0'; // tuning knob
  if (const char* lc = std::getenv("CVX_LIST_CAP")) sm->list_cap_limit = std::atoll(lc);  // test knob
  if (const char* dn = std::getenv("CVX_DENSE")) sm->dense_on = dn[0] != '0';         // R19 knob
  if (const char* wp = std::getenv("CVX_WALK_PRIO")) sm->walk_prio = wp[0] != '0';      // scheduling knob
  if (const char* dc = std::getenv("CVX_DENSE_COLOR")) sm->dense_color = dc[0] != '0';  // R19 knob (colour)
  if (const char* df = std::getenv("CVX_DEFER_FOLD")) sm->defer_fold = df[0] != '0';   // R19 knob (deferred fold)
  if (const char* db = std::getenv("CVX_DENSE_BLOCKS"))                                 // R19 capacity knob
    sm->dense_cap = std::max(1ll, std::min(std::atoll(db), 1ll << 22));
  sm->cfg = *cfg;
  std::memcpy(sm->T_ws, T_world_submap, sizeof(sm->T_ws));
  sm->device = device;
  int log2cap = 10;
  while ((1ll << log2cap) < 2 * cfg->max_blocks) ++log2cap;
  const size_t cap = (size_t)1 << log2cap;
  const size_t nb = (size_t)cfg->max_blocks;
  sm->hash.mask = (unsigned)(cap - 1);
  sm->hash.log2cap = log2cap;
  sm->pool.max_blocks = (int)nb;
  if ((e = cudaMalloc(&sm->hash.e, cap * sizeof(cvx::HashEntry))) != cudaSuccess ||
      (e = cudaMalloc(&sm->pool.sums, nb * cvx::kBlockVox * 16)) != cudaSuccess ||
      (e = cudaMalloc(&sm->pool.acc, (nb + cvx::kTrashBlocks) * cvx::kBlockVox * 8)) != cudaSuccess ||
      (e = cudaMalloc(&sm->pool.esdf, nb * cvx::kBlockVox * 4)) != cudaSuccess ||
      (e = cudaMalloc(&sm->pool.coords, nb * 16)) != cudaSuccess ||
      (e = cudaMalloc(&sm->pool.grid, sizeof(int) * cvx::kGridX * cvx::kGridY * cvx::kGridZ)) != cudaSuccess ||
      (e = cudaMalloc(&sm->ctr, sizeof(cvx::Counters))) != cudaSuccess ||
      (e = cudaMallocHost(&sm->ctr_host, sizeof(cvx::Counters))) != cudaSuccess ||
      (e = cudaMalloc(&sm->buf[0].frame_T, sizeof(double) * 16 * cvx::kMaxBatch)) != cudaSuccess ||
      (e = cudaMalloc(&sm->buf[1].frame_T, sizeof(double) * 16 * cvx::kMaxBatch)) != cudaSuccess ||
      (e = cudaMalloc(&sm->buf[0].lcnt, 64)) != cudaSuccess || (e = cudaMalloc(&sm->buf[1].lcnt, 64)) != cudaSuccess ||
      (e = cudaMalloc(&sm->acc_dirty, sizeof(int))) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&sm->ev_walked, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&sm->side, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&sm->ev_entry, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&sm->ev_prepared[0], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&sm->ev_prepared[1], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&sm->ev_free[0], cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&sm->ev_free[1], cudaEventDisableTiming)) != cudaSuccess ||
      (cfg->color && ((e = cudaMalloc(&sm->pool.csum, nb * cvx::kBlockVox * 32)) != cudaSuccess ||
                      (e = cudaMalloc(&sm->pool.cacc, (nb + cvx::kTrashBlocks) * cvx::kBlockVox * 16)) != cudaSuccess))) {
    free_all(sm);
    delete sm;
    return cuda_fail(e, "allocating submap");
  }
  // zero-initialised pool (a3 zero-init happens once here; reset re-zeroes only the used blocks)
  cudaMemset(sm->ctr, 0, sizeof(cvx::Counters));
  cudaMemset(sm->acc_dirty, 0, sizeof(int));
  cudaMemset(sm->pool.sums, 0, nb * cvx::kBlockVox * 16);
  cudaMemset(sm->pool.acc, 0, (nb + cvx::kTrashBlocks) * cvx::kBlockVox * 8);   // + the trash region (cvx_internal.cuh)
  cudaMemset(sm->pool.esdf, 0, nb * cvx::kBlockVox * 4);
  cudaMemset(sm->pool.grid, 0xff, sizeof(int) * cvx::kGridX * cvx::kGridY * cvx::kGridZ);   // all unknown
  if (cfg->color) {
    cudaMemset(sm->pool.csum, 0, nb * cvx::kBlockVox * 32);
    cudaMemset(sm->pool.cacc, 0, (nb + cvx::kTrashBlocks) * cvx::kBlockVox * 16);
  }
  e = cvx::launch_reset(sm, 0);
  if (e == cudaSuccess) e = cudaEventRecord(sm->ev_free[0], 0);
  if (e == cudaSuccess) e = cudaEventRecord(sm->ev_free[1], 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    free_all(sm);
    delete sm;
    return cuda_fail(e, "initialising submap");
  }
  *out = sm;
  return CVX_OK;
}

cvx_status cvx_destroy_submap(cvx_submap* sm) {
  g_last_error.clear();
  if (!sm) return CVX_OK;
  DeviceGuard g(sm->device);
  cudaDeviceSynchronize();
  free_all(sm);
  delete sm;
  return CVX_OK;
}

cvx_status cvx_reset_submap(cvx_submap* sm, void* stream) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  DeviceGuard g(sm->device);
  cudaError_t e = cvx::launch_reset(sm, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "reset");
  sm->finalized = false;
  sm->esdf_valid = false;
  sm->inc.nb_prev = 0;
  return CVX_OK;
}

static cvx_status integrate_impl(cvx_submap* sm, const float* data, int64_t n_per_frame, int32_t n_frames,
                                 const double* T_world_sensor, const cvx_sensor_model* sensor, void* stream,
                                 cvx_integrate_stats* stats, bool host_data, const uint8_t* rgb = nullptr,
                                 bool projective = false) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (sm->finalized) return fail(CVX_E_STATE, "submap is finalized (S:L443): integrate rejected");
  if (n_per_frame < 0 || n_frames < 0) return fail(CVX_E_INVALID, "negative sizes");
  cvx_status rc = check_sensor(sensor, n_per_frame);
  if (rc != CVX_OK) return rc;
  if (n_per_frame > 0 && n_frames > 0) {
    if (!data) return fail(CVX_E_INVALID, "data is NULL");
    if (!T_world_sensor) return fail(CVX_E_INVALID, "T_world_sensor is NULL");
    for (int f = 0; f < n_frames; ++f)
      if (!valid_pose(T_world_sensor + 16 * f)) return fail(CVX_E_INVALID, "T_world_sensor must be a finite rigid 4x4");
    if (n_per_frame >= (1ll << 31)) return fail(CVX_E_INVALID, "n_per_frame must be < 2^31");
  }
  DeviceGuard g(sm->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_per_frame > 0 && n_frames > 0) {
    cudaError_t e = projective
                        ? cvx::launch_integrate_projective(sm, data, n_per_frame, n_frames, T_world_sensor, *sensor, st)
                        : cvx::launch_integrate(sm, data, n_per_frame, n_frames, T_world_sensor, *sensor, st, host_data,
                                                nullptr, rgb);
    if (e != cudaSuccess) return cuda_fail(e, "integrate");
  }
  if (stats) {
    cvx::Counters c;
    if ((rc = read_counters(sm, st, &c)) != CVX_OK) return rc;
    fill_stats(c, sm->pool.max_blocks, stats);
    return sticky(c);
  }
  return CVX_OK;
}

cvx_status cvx_set_submap_pose(cvx_submap* sm, const double* T_world_submap) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (!valid_pose(T_world_submap)) return fail(CVX_E_INVALID, "T_world_submap must be a finite rigid 4x4");
  std::memcpy(sm->T_ws, T_world_submap, sizeof(sm->T_ws));
  return CVX_OK;
}

cvx_status cvx_integrate_batch(cvx_submap* sm, const float* data, int64_t n_per_frame, int32_t n_frames,
                               const double* T_world_sensor, const cvx_sensor_model* sensor, void* stream,
                               cvx_integrate_stats* stats) {
  return integrate_impl(sm, data, n_per_frame, n_frames, T_world_sensor, sensor, stream, stats, false);
}

cvx_status cvx_integrate_batch_host(cvx_submap* sm, const float* host_data, int64_t n_per_frame, int32_t n_frames,
                                    const double* T_world_sensor, const cvx_sensor_model* sensor, void* stream,
                                    cvx_integrate_stats* stats) {
  return integrate_impl(sm, host_data, n_per_frame, n_frames, T_world_sensor, sensor, stream, stats, true);
}

cvx_status cvx_integrate_color(cvx_submap* sm, const float* data, const uint8_t* rgb, int64_t n_per_frame,
                               int32_t n_frames, const double* T_world_sensor, const cvx_sensor_model* sensor,
                               void* stream, cvx_integrate_stats* stats) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (!sm->pool.csum) return fail(CVX_E_INVALID, "submap has no colour storage (config.color = 0)");
  if (!rgb && n_per_frame > 0 && n_frames > 0) return fail(CVX_E_INVALID, "rgb is NULL");
  return integrate_impl(sm, data, n_per_frame, n_frames, T_world_sensor, sensor, stream, stats, false, rgb);
}

cvx_status cvx_integrate_projective(cvx_submap* sm, const float* depth, int64_t n_per_frame, int32_t n_frames,
                                    const double* T_world_sensor, const cvx_sensor_model* sensor, void* stream,
                                    cvx_integrate_stats* stats) {
  g_last_error.clear();
  if (!sm || !sensor) return fail(CVX_E_INVALID, "NULL argument");
  if (sensor->kind != 1) return fail(CVX_E_INVALID, "projection mapping needs a pinhole depth sensor (kind 1)");
  return integrate_impl(sm, depth, n_per_frame, n_frames, T_world_sensor, sensor, stream, stats, false, nullptr, true);
}

cvx_status cvx_export_color(const cvx_submap* sm, float* rgb, float* color_weight, int64_t capacity_blocks,
                            int64_t* n_out, void* stream) {
  g_last_error.clear();
  if (!sm || !n_out || !rgb) return fail(CVX_E_INVALID, "NULL argument");
  if (!sm->pool.csum) return fail(CVX_E_INVALID, "submap has no colour storage (config.color = 0)");
  DeviceGuard g(sm->device);
  cudaStream_t st = (cudaStream_t)stream;
  cvx::Counters c;
  cvx_status rc = read_counters(sm, st, &c);
  if (rc != CVX_OK) return rc;
  const int nb = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  *n_out = nb;
  if (nb > capacity_blocks) return fail(CVX_E_CAPACITY, "export buffer smaller than the block count");
  cudaError_t e = cvx::launch_export_color(sm, nb, rgb, color_weight, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "export_color");
  return sticky(c);
}

cvx_status cvx_integrate_pointcloud(cvx_submap* sm, const float* data, int64_t n, const double* T_world_sensor,
                                    const cvx_sensor_model* sensor, void* stream, cvx_integrate_stats* stats) {
  return cvx_integrate_batch(sm, data, n, 1, T_world_sensor, sensor, stream, stats);
}

cvx_status cvx_integrate_until(cvx_submap* sm, const float* data, int64_t n_per_frame, int32_t n_frames,
                               const double* T_world_sensor, const cvx_sensor_model* sensor, int64_t block_threshold,
                               void* stream, int32_t* frames_integrated) {
  g_last_error.clear();
  if (!sm || !frames_integrated) return fail(CVX_E_INVALID, "NULL argument");
  if (block_threshold < 1 || block_threshold > sm->pool.max_blocks)
    return fail(CVX_E_INVALID, "block_threshold must be in [1, max_blocks]");
  *frames_integrated = 0;
  if (sm->finalized) return fail(CVX_E_STATE, "submap is finalized (S:L443): integrate rejected");
  if (n_per_frame < 0 || n_frames < 0) return fail(CVX_E_INVALID, "negative sizes");
  cvx_status rc = check_sensor(sensor, n_per_frame);
  if (rc != CVX_OK) return rc;
  if (n_frames == 0 || n_per_frame == 0) return CVX_OK;
  if (!data || !T_world_sensor) return fail(CVX_E_INVALID, "NULL buffer");
  for (int f = 0; f < n_frames; ++f)
    if (!valid_pose(T_world_sensor + 16 * f)) return fail(CVX_E_INVALID, "T_world_sensor must be a finite rigid 4x4");
  DeviceGuard g(sm->device);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (!sm->trig && ((e = cudaMalloc(&sm->trig, 16)) != cudaSuccess || (e = cudaMallocHost(&sm->trig_host, 16)) != cudaSuccess))
    return cuda_fail(e, "allocating trigger state");
  sm->trig_host[0] = (int)block_threshold; sm->trig_host[1] = 0; sm->trig_host[2] = 0; sm->trig_host[3] = 0;
  if ((e = cudaMemcpyAsync(sm->trig, sm->trig_host, 16, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "integrate_until");
  e = cvx::launch_integrate(sm, data, n_per_frame, n_frames, T_world_sensor, *sensor, st, false, sm->trig);
  if (e == cudaSuccess) e = cudaMemcpyAsync(sm->trig_host, sm->trig, 16, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "integrate_until");
  *frames_integrated = sm->trig_host[1] ? sm->trig_host[2] : n_frames;
  return CVX_OK;
}

cvx_status cvx_get_stats(const cvx_submap* sm, cvx_integrate_stats* out) {
  g_last_error.clear();
  if (!sm || !out) return fail(CVX_E_INVALID, "NULL argument");
  DeviceGuard g(sm->device);
  cvx::Counters c;
  cvx_status rc = read_counters(sm, 0, &c, true);
  if (rc != CVX_OK) return rc;
  fill_stats(c, sm->pool.max_blocks, out);
  return sticky(c);
}

cvx_status cvx_get_block_count(const cvx_submap* sm, int64_t* out) {
  g_last_error.clear();
  if (!sm || !out) return fail(CVX_E_INVALID, "NULL argument");
  DeviceGuard g(sm->device);
  cvx::Counters c;
  cvx_status rc = read_counters(sm, 0, &c, true);
  if (rc != CVX_OK) return rc;
  *out = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  return sticky(c);
}

cvx_status cvx_get_aabb(const cvx_submap* sm, int32_t* lo, int32_t* hi) {
  g_last_error.clear();
  if (!sm || !lo || !hi) return fail(CVX_E_INVALID, "NULL argument");
  DeviceGuard g(sm->device);
  cvx::Counters c;
  cvx_status rc = read_counters(sm, 0, &c, true);
  if (rc != CVX_OK) return rc;
  for (int a = 0; a < 3; ++a) { lo[a] = c.aabb_lo[a]; hi[a] = c.aabb_hi[a]; }
  return CVX_OK;
}

cvx_status cvx_finalize_esdf(cvx_submap* sm, void* stream) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  DeviceGuard g(sm->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  cvx::Counters c;
  cvx_status rc = read_counters(sm, st, &c);
  if (rc != CVX_OK) return rc;
  if ((rc = sticky(c)) != CVX_OK) return rc;
  const int nb = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  if (nb > 0) {
    for (int a = 0; a < 3; ++a)
      if ((int64_t)8 * ((int64_t)c.aabb_hi[a] - c.aabb_lo[a] + 1) > cvx::kMaxEdtAxis)
        return fail(CVX_E_RANGE, "submap AABB exceeds 46336 voxels along an axis (dense EDT domain: 2-D squared "
                                 "distances must fit 32 bits)");
    cudaError_t e = cvx::launch_finalize(sm, nb, c.aabb_lo, c.aabb_hi, st);
    if (e != cudaSuccess) return cuda_fail(e, "finalize_esdf");
  }
  sm->finalized = true;
  return CVX_OK;
}

cvx_status cvx_update_esdf(cvx_submap* sm, void* stream, int32_t* blocks_updated) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  DeviceGuard g(sm->device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaStream_t st = (cudaStream_t)stream;
  cvx::Counters c;
  cvx_status rc = read_counters(sm, st, &c);
  if (rc != CVX_OK) return rc;
  if ((rc = sticky(c)) != CVX_OK) return rc;
  const int nb = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  if (nb > 0)
    for (int a = 0; a < 3; ++a)
      if ((int64_t)8 * ((int64_t)c.aabb_hi[a] - c.aabb_lo[a] + 1) > cvx::kMaxEdtAxis)
        return fail(CVX_E_RANGE, "submap AABB exceeds 46336 voxels along an axis");
  int nq = 0;
  cudaError_t e = cvx::launch_update_esdf(sm, nb, c.aabb_lo, c.aabb_hi, st, &nq);
  if (e != cudaSuccess) return cuda_fail(e, "update_esdf");
  if (blocks_updated) *blocks_updated = nq;
  sm->esdf_valid = true;
  return CVX_OK;
}

cvx_status cvx_query_distance(const cvx_submap* sm, const float* pts, int64_t m, float* out, uint8_t* status,
                              void* stream) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (!sm->finalized && !sm->esdf_valid) return fail(CVX_E_STATE, "query before finalize_esdf / update_esdf");
  if (m < 0) return fail(CVX_E_INVALID, "m < 0");
  if (m > 0 && (!pts || !out || !status)) return fail(CVX_E_INVALID, "NULL buffer");
  DeviceGuard g(sm->device);
  cudaError_t e = cvx::flush_fold(const_cast<cvx_submap*>(sm), (cudaStream_t)stream);
  if (e == cudaSuccess) e = cvx::launch_query(sm, pts, m, out, status, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "query_distance");
  return CVX_OK;
}

cvx_status cvx_query_distance_gradient(const cvx_submap* sm, const float* pts, int64_t m, float* out, float* grad,
                                       uint8_t* status, void* stream) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (!sm->finalized && !sm->esdf_valid) return fail(CVX_E_STATE, "query before finalize_esdf / update_esdf");
  if (m < 0) return fail(CVX_E_INVALID, "m < 0");
  if (m > 0 && (!pts || !out || !grad || !status)) return fail(CVX_E_INVALID, "NULL buffer");
  DeviceGuard g(sm->device);
  cudaError_t e = cvx::flush_fold(const_cast<cvx_submap*>(sm), (cudaStream_t)stream);
  if (e == cudaSuccess) e = cvx::launch_query(sm, pts, m, out, status, (cudaStream_t)stream, grad);
  if (e != cudaSuccess) return cuda_fail(e, "query_distance_gradient");
  return CVX_OK;
}

cvx_status cvx_sample_surface(cvx_submap* sm, const uint32_t* uniforms, int64_t m, float* out_xyz, float* out_weight,
                              int64_t* total_weight, void* stream) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (m < 0) return fail(CVX_E_INVALID, "m < 0");
  if (m > 0 && (!uniforms || !out_xyz)) return fail(CVX_E_INVALID, "NULL buffer");
  DeviceGuard g(sm->device);
  cudaStream_t st = (cudaStream_t)stream;
  cvx::Counters c;
  cvx_status rc = read_counters(sm, st, &c);
  if (rc != CVX_OK) return rc;
  const int nb = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  long long tot = 0;
  cudaError_t e = cvx::launch_sample_surface(sm, nb, c.aabb_lo, c.aabb_hi, uniforms, m, out_xyz, out_weight, st, &tot);
  if (e != cudaSuccess) return cuda_fail(e, "sample_surface");
  if (total_weight) *total_weight = tot;
  return CVX_OK;
}

cvx_status cvx_export_blocks(const cvx_submap* sm, int32_t* bxyz, float* D, float* W, float* E,
                             int64_t capacity_blocks, int64_t* n_out, void* stream) {
  g_last_error.clear();
  if (!sm || !n_out) return fail(CVX_E_INVALID, "NULL argument");
  DeviceGuard g(sm->device);
  cudaStream_t st = (cudaStream_t)stream;
  cvx::Counters c;
  cvx_status rc = read_counters(sm, st, &c);
  if (rc != CVX_OK) return rc;
  const int nb = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  *n_out = nb;
  if (nb > capacity_blocks) return fail(CVX_E_CAPACITY, "export buffer smaller than the block count");
  cudaError_t e = cvx::launch_export(sm, nb, bxyz, D, W, E, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "export_blocks");
  return sticky(c);
}

cvx_status cvx_import_tsdf_blocks(cvx_submap* sm, const int32_t* bxyz, const float* D, const float* W,
                                  int64_t n, void* stream) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  if (sm->finalized) return fail(CVX_E_STATE, "submap is finalized");
  if (n < 0) return fail(CVX_E_INVALID, "n < 0");
  if (n > 0 && (!bxyz || !D || !W)) return fail(CVX_E_INVALID, "NULL buffer");
  DeviceGuard g(sm->device);
  cudaError_t e = cvx::flush_fold(sm, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cvx::launch_import(sm, bxyz, D, W, n, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "import_tsdf_blocks");
  return CVX_OK;
}

cvx_status cvx_packed_size(const cvx_submap* sm, int64_t* bytes) {
  int64_t nb = 0;
  cvx_status rc = cvx_get_block_count(sm, &nb);
  if (rc != CVX_OK && rc != CVX_E_CAPACITY && rc != CVX_E_RANGE) return rc;
  if (!bytes) return fail(CVX_E_INVALID, "NULL argument");
  *bytes = 256 + nb * (16 + 4 * cvx::kBlockVox);
  return CVX_OK;
}

cvx_status cvx_pack_esdf(const cvx_submap* sm, void* dst, int64_t dst_bytes, int64_t* used, void* stream) {
  g_last_error.clear();
  if (!sm || !used) return fail(CVX_E_INVALID, "NULL argument");
  if (!sm->finalized) return fail(CVX_E_STATE, "pack before finalize_esdf");
  DeviceGuard g(sm->device);
  cudaStream_t st = (cudaStream_t)stream;
  cvx::Counters c;
  cvx_status rc = read_counters(sm, st, &c);
  if (rc != CVX_OK) return rc;
  const int nb = c.n_blocks < sm->pool.max_blocks ? c.n_blocks : sm->pool.max_blocks;
  const int64_t need = 256 + (int64_t)nb * (16 + 4 * cvx::kBlockVox);
  *used = need;
  if (!dst) return CVX_OK;   // size query, ordered on `stream` only
  if (dst_bytes < need) return fail(CVX_E_CAPACITY, "pack buffer too small");
  unsigned char hdr[256];
  std::memset(hdr, 0, sizeof(hdr));
  const uint32_t magic = 0x45585643u;  // "CVXE"
  const int32_t version = 1;
  const int64_t n64 = nb;
  std::memcpy(hdr, &magic, 4);
  std::memcpy(hdr + 4, &version, 4);
  std::memcpy(hdr + 8, &n64, 8);
  std::memcpy(hdr + 16, &sm->cfg.voxel_size, 8);
  std::memcpy(hdr + 24, sm->T_ws, 128);
  cudaError_t e = cudaMemcpyAsync(dst, hdr, sizeof(hdr), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cvx::launch_pack(sm, nb, (unsigned char*)dst + 256, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "pack_esdf");
  return CVX_OK;
}

cvx_status cvx_esdf_set_create(const void* payloads, int64_t payload_bytes, const int64_t* offsets, int32_t n_submaps,
                               int device, void* stream, cvx_esdf_set** out) {
  g_last_error.clear();
  if (!out) return fail(CVX_E_INVALID, "out is NULL");
  *out = nullptr;
  if (n_submaps < 1 || n_submaps >= (1 << 24)) return fail(CVX_E_INVALID, "n_submaps must be in [1, 2^24)");
  if (!payloads || !offsets || payload_bytes <= 0) return fail(CVX_E_INVALID, "NULL / empty payload buffer");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(CVX_E_INVALID, "device index out of range");
  DeviceGuard g(device);
  cudaStream_t st = (cudaStream_t)stream;
  cvx_esdf_set* set = new cvx_esdf_set();
  set->device = device;
  set->n = n_submaps;
  set->payload = static_cast<const unsigned char*>(payloads);
  std::vector<unsigned char> hdr((size_t)n_submaps * 256);
  std::vector<long long> rec(n_submaps);
  auto bad = [&](cvx_status code, const std::string& msg) {
    cvx_esdf_set_destroy(set);
    return fail(code, msg);
  };
  for (int k = 0; k < n_submaps; ++k) {
    if (offsets[k] < 0 || offsets[k] % 16 != 0 || offsets[k] + 256 > payload_bytes)
      return bad(CVX_E_INVALID, "payload offset out of range or not 16-byte aligned");
    if ((e = cudaMemcpyAsync(hdr.data() + 256 * (size_t)k, set->payload + offsets[k], 256, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
      return bad(CVX_E_CUDA, std::string("reading payload headers: ") + cudaGetErrorString(e));
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return bad(CVX_E_CUDA, cudaGetErrorString(e));
  set->T.resize(16 * (size_t)n_submaps);
  set->s.resize(n_submaps);
  set->n_blocks.resize(n_submaps);
  for (int k = 0; k < n_submaps; ++k) {
    const unsigned char* h = hdr.data() + 256 * (size_t)k;
    uint32_t magic; int32_t version; int64_t nb; double vs;
    std::memcpy(&magic, h, 4); std::memcpy(&version, h + 4, 4); std::memcpy(&nb, h + 8, 8); std::memcpy(&vs, h + 16, 8);
    if (magic != 0x45585643u || version != 1) return bad(CVX_E_INVALID, "not a cvx_pack_esdf payload (magic / version)");
    if (nb < 0 || offsets[k] + 256 + nb * (16 + 4 * cvx::kBlockVox) > payload_bytes)
      return bad(CVX_E_INVALID, "payload block count exceeds the buffer");
    if (!(vs > 0)) return bad(CVX_E_INVALID, "payload voxel size must be > 0");
    std::memcpy(&set->T[16 * (size_t)k], h + 24, 128);
    if (!valid_pose(&set->T[16 * (size_t)k])) return bad(CVX_E_INVALID, "payload pose is not a rigid 4x4");
    set->s[k] = vs;
    set->n_blocks[k] = nb;
    rec[k] = offsets[k] + 256;
  }
  std::vector<double> Ts(set->T);
  Ts.insert(Ts.end(), set->s.begin(), set->s.end());
  if ((e = cudaMalloc(&set->T_dev, sizeof(double) * Ts.size())) != cudaSuccess ||
      (e = cudaMalloc(&set->rec_off, sizeof(long long) * n_submaps)) != cudaSuccess ||
      (e = cudaMalloc(&set->err, 4)) != cudaSuccess)
    return bad(e == cudaErrorMemoryAllocation ? CVX_E_OOM : CVX_E_CUDA, "allocating the set");
  cudaMemcpyAsync(set->T_dev, Ts.data(), sizeof(double) * Ts.size(), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(set->rec_off, rec.data(), sizeof(long long) * n_submaps, cudaMemcpyHostToDevice, st);
  unsigned err = 0;
  if ((e = cvx::launch_set_build(set, st, &err)) != cudaSuccess)
    return bad(e == cudaErrorMemoryAllocation ? CVX_E_OOM : CVX_E_CUDA, std::string("building the set: ") + cudaGetErrorString(e));
  if (err & 2u) return bad(CVX_E_INVALID, "a payload spans >= 8192 blocks along an axis (not a finalized submap)");
  if (err & 1u) return bad(CVX_E_INVALID, "a payload holds the same block twice");
  *out = set;
  return CVX_OK;
}

cvx_status cvx_esdf_set_destroy(cvx_esdf_set* set) {
  if (!set) return CVX_OK;
  DeviceGuard g(set->device);
  cudaDeviceSynchronize();
  if (set->T_dev) cudaFree(set->T_dev);
  if (set->rec_off) cudaFree(set->rec_off);
  if (set->table) cudaFree(set->table);
  if (set->err) cudaFree(set->err);
  delete set;
  return CVX_OK;
}

cvx_status cvx_esdf_set_query(const cvx_esdf_set* set, const int32_t* submap_index, const float* points_world,
                              int64_t m, float* out_distance, float* out_gradient, uint8_t* out_status, void* stream) {
  g_last_error.clear();
  if (!set) return fail(CVX_E_INVALID, "set is NULL");
  if (m < 0) return fail(CVX_E_INVALID, "m < 0");
  if (m > 0 && (!submap_index || !points_world || !out_distance || !out_status)) return fail(CVX_E_INVALID, "NULL buffer");
  DeviceGuard g(set->device);
  cudaError_t e = cvx::launch_set_query(set, submap_index, points_world, m, out_distance, out_gradient, out_status,
                                        (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "esdf_set_query");
  return CVX_OK;
}

cvx_status cvx_profile_enable(cvx_submap* sm, int32_t enable) {
  g_last_error.clear();
  if (!sm) return fail(CVX_E_INVALID, "submap is NULL");
  DeviceGuard g(sm->device);
  cudaDeviceSynchronize();
  sm->prof->recycle();
  sm->prof->on = (enable & 1) != 0;
  sm->serialize = (enable & 2) != 0;
  return CVX_OK;
}

cvx_status cvx_profile_report(cvx_submap* sm, char* buf, int64_t buflen) {
  g_last_error.clear();
  if (!sm || !buf || buflen <= 0) return fail(CVX_E_INVALID, "NULL argument");
  DeviceGuard g(sm->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "profile_report");
  std::vector<std::pair<std::string, std::pair<double, long long>>> acc;
  for (auto& r : sm->prof->recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) { cudaGetLastError(); continue; }
    size_t k = 0;
    while (k < acc.size() && acc[k].first != r.name) ++k;
    if (k == acc.size()) acc.push_back({r.name, {0.0, 0}});
    acc[k].second.first += ms;
    acc[k].second.second += 1;
  }
  sm->prof->recycle();
  std::string js = "{";
  for (size_t k = 0; k < acc.size(); ++k) {
    char item[256];
    std::snprintf(item, sizeof(item), "%s\"%s\": {\"ms\": %.6f, \"n\": %lld}", k ? ", " : "", acc[k].first.c_str(),
                  acc[k].second.first, acc[k].second.second);
    js += item;
  }
  js += "}";
  if ((int64_t)js.size() + 1 > buflen) return fail(CVX_E_CAPACITY, "report buffer too small");
  std::memcpy(buf, js.c_str(), js.size() + 1);
  return CVX_OK;
}

}  // extern "C"
