// query.cu — distance queries (O13) and the block export / import /
// pack kernels of the inspection and multi-GPU gather hooks, for sm_100a.
#include "submap.h"

namespace cvx {
namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

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

// Voxel coordinates of the 21-bit block-key domain (O3: |voxel| < 2^23, blocks in [-2^20, 2^20)); a
// coordinate outside it cannot be allocated, and pack_key would alias it onto an in-range block.
__device__ __forceinline__ bool in_key_domain(int x, int y, int z) {
  constexpr int lo = -(1 << 23), hi = (1 << 23) - 1;
  return x >= lo && x <= hi && y >= lo && y <= hi && z >= lo && z <= hi;
}

// E of voxel (x,y,z) through the hash (block cached); false if unallocated, outside the key domain or
// unobserved (NaN).
__device__ __forceinline__ bool voxel_e(const QueryParams& p, int x, int y, int z, unsigned long long& ckey,
                                        int& cslot, float* e) {
  if (!in_key_domain(x, y, z)) return false;
  const unsigned long long key = pack_key(x >> 3, y >> 3, z >> 3);
  if (key != ckey) { ckey = key; cslot = hash_find(p.hash, key); }
  if (cslot < 0) return false;
  const float v = p.esdf[(long long)cslot * kBlockVox + (x & 7) + 8 * (y & 7) + 64 * (z & 7)];
  if (isnan(v)) return false;
  *e = v;
  return true;
}

__global__ void __launch_bounds__(256) query_kernel(const __grid_constant__ QueryParams p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.m) return;
  const double x[3] = {p.pts[3 * i], p.pts[3 * i + 1], p.pts[3 * i + 2]};
  double xs[3], f[3];
  int i0[3];
  bool ok = true;
  for (int a = 0; a < 3; ++a) {   // x_s = T_WS^-1 x  (O13), same operation order as the oracle
    xs[a] = da(da(dm(p.T[0 * 4 + a], ds(x[0], p.T[3])), dm(p.T[1 * 4 + a], ds(x[1], p.T[7]))),
               dm(p.T[2 * 4 + a], ds(x[2], p.T[11])));
    const double g = ds(__ddiv_rn(xs[a], p.s), 0.5);
    const double fl = floor(g);
    if (!(fabs(fl) < 1073741824.0)) ok = false;
    i0[a] = ok ? (int)fl : 0;
    f[a] = ds(g, fl);
  }
  unsigned long long ckey = ~0ull;
  int cslot = -1;
  const float qnan = __int_as_float(0x7fc00000);
  if (ok) {
    double acc = 0.0, gs[3] = {0.0, 0.0, 0.0};
    bool all = true;
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
      float e;
      if (!voxel_e(p, i0[0] + dx, i0[1] + dy, i0[2] + dz, ckey, cslot, &e)) { all = false; break; }
      const double wx = dx ? f[0] : ds(1.0, f[0]), wy = dy ? f[1] : ds(1.0, f[1]), wz = dz ? f[2] : ds(1.0, f[2]);
      const double wgt = dm(dm(wx, wy), wz);
      if (wgt > 0) acc = da(acc, dm(wgt, (double)e));
      if (p.grad) {   // d/df of the trilinear weights (f4: value + gradient look-ups for registration)
        gs[0] += (dx ? 1.0 : -1.0) * wy * wz * (double)e;
        gs[1] += (dy ? 1.0 : -1.0) * wx * wz * (double)e;
        gs[2] += (dz ? 1.0 : -1.0) * wx * wy * (double)e;
      }
    }
    if (all) {
      p.out[i] = (float)acc;
      p.status[i] = 0;
      if (p.grad)   // dE/dx_world = R_WS dE/dx_s, dE/dx_s = (dE/df) / s
        for (int a = 0; a < 3; ++a)
          p.grad[3 * i + a] = (float)((p.T[4 * a] * gs[0] + p.T[4 * a + 1] * gs[1] + p.T[4 * a + 2] * gs[2]) / p.s);
      return;
    }
    if (p.grad) { p.grad[3 * i] = qnan; p.grad[3 * i + 1] = qnan; p.grad[3 * i + 2] = qnan; }
    int v[3];
    for (int a = 0; a < 3; ++a) {
      const double fv = floor(__ddiv_rn(xs[a], p.s));
      v[a] = fabs(fv) < 1073741824.0 ? (int)fv : (1 << 30);   // |v| >= 2^30: outside the key domain
    }
    float e;
    if (voxel_e(p, v[0], v[1], v[2], ckey, cslot, &e)) { p.out[i] = e; p.status[i] = 1; return; }
  }
  if (p.grad && !ok) { p.grad[3 * i] = qnan; p.grad[3 * i + 1] = qnan; p.grad[3 * i + 2] = qnan; }
  p.out[i] = qnan;
  p.status[i] = 2;
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
  if (B.slot_cap < n) {
    if (B.slot_lists) cudaFree(B.slot_lists);
    B.slot_lists = nullptr; B.slot_cap = 0;
    cudaError_t e = cudaMalloc(&B.slot_lists, sizeof(int) * (size_t)n);
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
