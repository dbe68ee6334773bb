// submap.h — host-side definition of the opaque cvx_submap and the internal launch entry points.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/cvx.h"
#include "cvx_internal.cuh"

namespace cvx {
// Optional per-kernel CUDA-event timing (cvx_profile_enable / cvx_profile_report): events are
// recorded on the launching stream around every kernel of the submap.
struct ProfRec { const char* name; cudaEvent_t a, b; };
struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t ev() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  int begin(const char* name, cudaStream_t st) {
    if (!on) return -1;
    ProfRec r{name, ev(), ev()};
    cudaEventRecord(r.a, st);
    recs.push_back(r);
    return (int)recs.size() - 1;
  }
  void end(int i, cudaStream_t st) { if (i >= 0) cudaEventRecord(recs[i].b, st); }
  void recycle() { for (auto& r : recs) { pool.push_back(r.a); pool.push_back(r.b); } recs.clear(); }
  ~Prof() { recycle(); for (auto e : pool) cudaEventDestroy(e); }
};
}  // namespace cvx

struct cvx_submap {
  cvx_grid_config cfg{};
  double T_ws[16] = {};    // world <- submap
  int device = 0;
  bool finalized = false;
  bool esdf_valid = false;    // an (incremental) ESDF was computed since the last reset

  // hash table + pool (HBM, see cvx_internal.cuh)
  cvx::HashView hash{};
  cvx::PoolView pool{};
  cvx::Counters* ctr = nullptr;       // device
  cvx::Counters* ctr_host = nullptr;  // pinned mirror for synchronising reads

  // integrate scratch, double-buffered (grow-only): the ingest + ALLOCATE phases of launch k+1 run on
  // `side` while the update walk of launch k runs on the caller's stream
  struct Buf {
    double* frame_T = nullptr;  // device [kMaxBatch][16]: R_SC, t_SC, q(t_SC), flag per frame
    void* rays = nullptr;       // device RayRec [ray_cap]
    int64_t ray_cap = 0;
    unsigned* rgbs = nullptr;   // device per-ray colour (TSDF + Color only)
    int64_t rgbs_cap = 0;
    float* ws = nullptr;        // device per-ray weight (weighting != 0 only)
    int64_t ws_cap = 0;
    int* slot_lists = nullptr;  // device block-slot lists of the rays of one launch
    int64_t slot_cap = 0;
    int* lcnt = nullptr;        // device {n_rays, n_slots, -, -, 4 spare, box lo[3], hi[3]} of the launch
    int* cta_box = nullptr;     // device per-CTA block boxes of prepare_kernel (dense-window path, R19)
    int64_t cta_box_cap = 0;
    unsigned long long* cstat = nullptr;   // device per-CTA look-back status of prepare_kernel
    int64_t cstat_cap = 0;
    float* staging = nullptr;   // device copy of host frames (cvx_integrate_batch_host)
    int64_t staging_cap = 0;
  } buf[2];
  cudaStream_t side = nullptr;
  cudaEvent_t ev_entry = nullptr, ev_prepared[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  // host frames (cvx_integrate_batch_host): H2D copies on their own stream, created on first use; the copy
  // into staging[b] waits only for the prepare that last read staging[b] (ev_stage_free), so it runs up
  // to one launch ahead of the side stream's ingest
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_staged[2] = {nullptr, nullptr}, ev_stage_free[2] = {nullptr, nullptr};
  int next_buf = 0;
  bool aggregate = true;      // warp-aggregate equal-voxel updates before the L2 atomics
  bool serialize = false;     // profiling: run the pipeline's side work on the caller's stream
  bool bw2 = true;            // software-pipelined ALLOCATE (block_walk2_kernel)
  bool bw3 = false;           // ALLOCATE through the dense slot cache (block_walk3_kernel): configs[1] step
                              // 8.33 -> 8.25 ms, but MAV submaps (50 scans, more new blocks) 133 -> 143 ms
  bool walk_cw = true;        // constant weights: incremental-address walk (walk_cw_kernel)
  long long list_cap_limit = 1ll << 62;   // test knob: cap on the per-ray slot-list buffer (full: walk hashes)
  bool fuse_alloc = false;    // constant weights: ALLOCATE inside walk_cw_kernel (measured 1.4x slower: off)
  // dense-window path (R19): block-major accumulators over the launch's block box, ALLOCATE after the walk
  bool walk_prio = false;    // CVX_WALK_PRIO: update walks on a high-priority library stream
  cudaStream_t wstream = nullptr;
  cudaEvent_t ev_w[2] = {nullptr, nullptr};
  bool dense_on = true;
  long long dense_cap = 1ll << 19;          // blocks (2 GiB of u64 accumulators; configs[1] / MAV boxes: <= 0.23 M)
  unsigned long long* dacc = nullptr;       // device [(dacc_blocks + kTrashBlocks) * 512], zero between folds
  long long dacc_blocks = 0;
  bool dense_color = true;                  // CVX_DENSE_COLOR: TSDF + Color through the dense window too
  bool defer_fold = false;                  // CVX_DEFER_FOLD=1: the call's last dense fold runs at the next access (measured slower)
  bool fold_pending = false;                // a deferred fold waits (flush_fold)
  int fold_buf = 0;                         //   its launch buffer (box in buf[fold_buf].lcnt + 8)
  long long fold_dcap = 0;
  bool fold_color = false;
  cudaEvent_t ev_walked = nullptr;          //   after that launch's walk
  unsigned long long* dcacc = nullptr;      // device [(dcacc_blocks + kTrashBlocks) * 512][2] colour accumulators
  long long dcacc_blocks = 0;
  int* acc_dirty = nullptr;                 // device: a dense-eligible launch fell back to the pool accumulators

  // ESDF scratch (grow-only, stream-ordered cudaMallocAsync on the calling stream)
  void* edt = nullptr;        // device: g2 u32 | g1 u16 over the dense AABB, then the column / row masks
  int64_t edt_bytes = 0;
  int* block_grid = nullptr;  // device int32 [nbz][nby][nbx]
  int64_t block_grid_cap = 0;
  // per-slot bit-planes of the last ESDF pass (pass x of finalize, or the incremental classify): 48 u32
  // words per slot = observed | D < 0 | site (O10), bit l = voxel local index l.  Two buffers: the
  // incremental update compares the new planes with the previous ones.
  unsigned* planes[2] = {nullptr, nullptr};
  int cur_planes = 0;

  // incremental ESDF state (R11: exact EDT clamped at esdf_max_distance)
  struct Inc {
    unsigned char* flags = nullptr;     // per slot: bit 0 site plane changed, bit 1 block must be recomputed
    int* list = nullptr;                // compacted queue of the blocks to recompute (one region per block)
    int* cnt = nullptr;
    int* cnt_host = nullptr;            // pinned
    int nb_prev = 0;                    // blocks covered by the last update (0: recompute everything)
  } inc;

  int* proj_birth = nullptr;  // device [max_blocks + 1]: birth frame per slot, then the block count at the
  int* proj_start = nullptr;  //   start of the call (projection mapping; proj_start points into proj_birth)
  int* trig = nullptr;        // device {threshold, hit, consumed, -} of cvx_integrate_until
  int* trig_host = nullptr;   // pinned mirror

  cvx::Prof* prof = nullptr;  // owned
};

// RAII timing scope around one kernel launch
struct ProfScope {
  cvx::Prof* p; int i; cudaStream_t st;
  ProfScope(const cvx_submap* sm, const char* name, cudaStream_t s) : p(sm->prof), i(-1), st(s) {
    if (p) i = p->begin(name, s);
  }
  ~ProfScope() { if (p) p->end(i, st); }
};

namespace cvx {

#ifndef CVX_MAX_BATCH
#define CVX_MAX_BATCH 200
#endif
constexpr int kMaxBatch = CVX_MAX_BATCH;   // frames per integrate launch (poses travel as kernel parameters)
constexpr int kSlotsPerRay = 40; // average block-slot list capacity per ray (overflow -> hashed walk)

// integrate.cu
cudaError_t launch_reset(cvx_submap* sm, cudaStream_t st);
cudaError_t flush_fold(cvx_submap* sm, cudaStream_t st);   // deferred dense fold (R19), if any
cudaError_t launch_integrate(cvx_submap* sm, const float* data, int64_t n_per_frame, int n_frames,
                             const double* T_world_sensor, const cvx_sensor_model& sensor, cudaStream_t st,
                             bool host_data, int* trig = nullptr, const unsigned char* rgb = nullptr);
cudaError_t launch_integrate_projective(cvx_submap* sm, const float* depth, int64_t n_per_frame, int n_frames,
                                        const double* T_world_sensor, const cvx_sensor_model& sensor,
                                        cudaStream_t st);
cudaError_t launch_export_color(const cvx_submap* sm, int n_blocks, float* rgb, float* cw, cudaStream_t st);
// esdf.cu
cudaError_t launch_finalize(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], cudaStream_t st);
cudaError_t launch_update_esdf(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], cudaStream_t st,
                               int* blocks_updated);
void release_esdf(cvx_submap* sm);   // frees the ESDF scratch, planes and incremental state
// query.cu
cudaError_t launch_query(const cvx_submap* sm, const float* pts, int64_t m, float* out, uint8_t* status,
                         cudaStream_t st, float* grad = nullptr);
// registration.cu
cudaError_t launch_sample_surface(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], const unsigned* uniforms,
                                  int64_t m, float* out_xyz, float* out_w, cudaStream_t st, long long* total_weight);
cudaError_t launch_export(const cvx_submap* sm, int n_blocks, int32_t* bxyz, float* D, float* W, float* E,
                          cudaStream_t st);
cudaError_t launch_import(cvx_submap* sm, const int32_t* bxyz, const float* D, const float* W, int64_t n,
                          cudaStream_t st);
cudaError_t launch_pack(const cvx_submap* sm, int n_blocks, void* dst_records, cudaStream_t st);

}  // namespace cvx
