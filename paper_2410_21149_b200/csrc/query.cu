// query.cu — distance queries (O13) and the block export / import /
// pack kernels of the inspection and multi-GPU gather hooks, for sm_100a.
#include "query_point.cuh"
#include "submap.h"

namespace cvx {
namespace {

struct QueryParams {
  const float* pts;
  long long m;
  float* out;
  float* grad;          // nullable: [m][3] world-frame gradient of the trilinear interpolant (status OK)
  unsigned char* status;
  HashView hash;
  const float* esdf;
  double T[16];     // T_world_submap
  double s;
};

__global__ void __launch_bounds__(256) query_kernel(const __grid_constant__ QueryParams p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.m) return;
  unsigned long long ckey = ~0ull;   // block of the last look-up (the 8 corners mostly share one)
  int cslot = -1;
  auto lookup = [&](int x, int y, int z, float* e) -> bool {
    if (!in_key_domain(x, y, z)) return false;
    const unsigned long long key = pack_key(x >> 3, y >> 3, z >> 3);
    if (key != ckey) { ckey = key; cslot = hash_find(p.hash, key); }
    if (cslot < 0) return false;
    const float v = p.esdf[(long long)cslot * kBlockVox + (x & 7) + 8 * (y & 7) + 64 * (z & 7)];
    if (isnan(v)) return false;
    *e = v;
    return true;
  };
  query_point(p.T, p.s, p.pts + 3 * i, lookup, p.out + i, p.grad ? p.grad + 3 * i : nullptr, p.status + i);
}

__global__ void export_kernel(const long long* sums, const float* esdf, const int4* coords, int nb,
                              int* bxyz, float* D, float* W, float* E) {
  const long long n = (long long)nb * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const longlong2 sw = reinterpret_cast<const longlong2*>(sums)[i];
    if (D) D[i] = sw.y > 0 ? (float)((double)sw.x / (double)sw.y) : 0.0f;   // O8: sum(w d) / sum(w)
    if (W) W[i] = (float)((double)sw.y * (1.0 / kFxScale));
    if (E) E[i] = esdf[i];
    if (bxyz && (i & 511) == 0) {
      const int4 c = coords[i >> 9];
      bxyz[3 * (i >> 9)] = c.x; bxyz[3 * (i >> 9) + 1] = c.y; bxyz[3 * (i >> 9) + 2] = c.z;
    }
  }
}

__global__ void import_slots_kernel(HashView h, PoolView pool, Counters* ctr, const int* bxyz, long long n, int* slots) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int bx = bxyz[3 * i], by = bxyz[3 * i + 1], bz = bxyz[3 * i + 2];
  const bool okr = bx >= -(1 << 20) && bx < (1 << 20) && by >= -(1 << 20) && by < (1 << 20) && bz >= -(1 << 20) && bz < (1 << 20);
  if (!okr) { atomicOr(&ctr->err, (unsigned)kErrRange); slots[i] = -1; return; }
  slots[i] = hash_activate(h, pool, ctr, pack_key(bx, by, bz), bx, by, bz);
}

__global__ void import_values_kernel(long long* sums, const int* slots, const float* D, const float* W, long long n) {
  const long long nv = n * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const int slot = slots[i >> 9];
    if (slot < 0) continue;
    const double w = (double)W[i];
    longlong2 v;
    v.y = w > 0 ? __double2ll_rn(w * kFxScale) : 0;
    v.x = w > 0 ? __double2ll_rn((double)D[i] * w * kFxScale) : 0;
    reinterpret_cast<longlong2*>(sums)[(long long)slot * kBlockVox + (i & 511)] = v;
  }
}

__global__ void pack_kernel(const float* esdf, const int4* coords, int nb, unsigned char* dst) {
  const long long n = (long long)nb * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i >> 9;
    unsigned char* rec = dst + b * (16 + 4 * kBlockVox);
    if ((i & 511) == 0) {
      const int4 c = coords[b];
      *reinterpret_cast<int4*>(rec) = make_int4(c.x, c.y, c.z, (int)b);
    }
    reinterpret_cast<float*>(rec + 16)[i & 511] = esdf[i];
  }
}

}  // namespace

cudaError_t launch_query(const cvx_submap* sm, const float* pts, int64_t m, float* out, uint8_t* status,
                         cudaStream_t st, float* grad) {
  if (m <= 0) return cudaSuccess;
  QueryParams q;
  q.pts = pts; q.m = m; q.out = out; q.status = status; q.grad = grad; q.hash = sm->hash; q.esdf = sm->pool.esdf;
  for (int i = 0; i < 16; ++i) q.T[i] = sm->T_ws[i];
  q.s = sm->cfg.voxel_size;
  {
    ProfScope ps_(sm, "query", st);
    query_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(q);
  }
  return cudaGetLastError();
}

cudaError_t launch_export(const cvx_submap* sm, int n_blocks, int32_t* bxyz, float* D, float* W, float* E,
                          cudaStream_t st) {
  if (n_blocks <= 0) return cudaSuccess;
  {
    ProfScope ps_(sm, "export", st);
    export_kernel<<<148 * 8, 256, 0, st>>>(sm->pool.sums, sm->pool.esdf, sm->pool.coords, n_blocks, bxyz, D, W, E);
  }
  return cudaGetLastError();
}

cudaError_t launch_import(cvx_submap* sm, const int32_t* bxyz, const float* D, const float* W, int64_t n,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  // slots scratch: the slot-list buffer of integrate buffer 0 (grown if needed); import runs on the
  // caller's stream after any integrate work on it, so the buffer is free
  cvx_submap::Buf& B = sm->buf[0];
  cudaStreamWaitEvent(st, sm->ev_free[0], 0);
  if (B.slot_cap < n) {   // stream-ordered growth (st already waits for buffer 0's last walk)
    if (B.slot_lists) cudaFreeAsync(B.slot_lists, st);
    B.slot_lists = nullptr; B.slot_cap = 0;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&B.slot_lists), sizeof(int) * (size_t)n, st);
    if (e != cudaSuccess) return e;
    B.slot_cap = n;
  }
  int* slots = B.slot_lists;
  {
    ProfScope ps_(sm, "import_slots", st);
    import_slots_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sm->hash, sm->pool, sm->ctr, bxyz, n, slots);
  }
  {
    ProfScope ps_(sm, "import_values", st);
    import_values_kernel<<<148 * 8, 256, 0, st>>>(sm->pool.sums, slots, D, W, n);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack(const cvx_submap* sm, int n_blocks, void* dst_records, cudaStream_t st) {
  if (n_blocks <= 0) return cudaSuccess;
  {
    ProfScope ps_(sm, "pack", st);
    pack_kernel<<<148 * 8, 256, 0, st>>>(sm->pool.esdf, sm->pool.coords, n_blocks, (unsigned char*)dst_records);
  }
  return cudaGetLastError();
}

}  // namespace cvx

namespace cvx {
// TSDF + Color (R13): colour = sum(w c) / sum(w) per voxel, slot order.
__global__ void export_color_kernel(const long long* csum, int n_blocks, float* rgb, float* cw) {
  const long long nv = (long long)n_blocks * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const longlong2 a = reinterpret_cast<const longlong2*>(csum)[2 * i];
    const longlong2 b = reinterpret_cast<const longlong2*>(csum)[2 * i + 1];
    const double w = (double)a.x;
    rgb[3 * i + 0] = a.x > 0 ? (float)((double)a.y / w) : 0.0f;
    rgb[3 * i + 1] = a.x > 0 ? (float)((double)b.x / w) : 0.0f;
    rgb[3 * i + 2] = a.x > 0 ? (float)((double)b.y / w) : 0.0f;
    if (cw) cw[i] = (float)((double)a.x * (1.0 / kFxScale));
  }
}

cudaError_t launch_export_color(const cvx_submap* sm, int n_blocks, float* rgb, float* cw, cudaStream_t st) {
  if (n_blocks <= 0) return cudaSuccess;
  export_color_kernel<<<148 * 8, 256, 0, st>>>(sm->pool.csum, n_blocks, rgb, cw);
  return cudaGetLastError();
}
}  // namespace cvx
