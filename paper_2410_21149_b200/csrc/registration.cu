// registration.cu — ESDF consumers for registration:
// weight-proportional surface-point sampling.  (Value + gradient look-ups are in query.cu.)
//
// Sampling definition (R12): the candidates are the sites (observed, |D| <= tau_site, R4) of
// all allocated blocks in lexicographic (bx, by, bz) block order and local index order inside a block;
// each carries the integer weight w_k = W_k in units of 2^-20 (W_k = the fused weight sum).  With
// T = sum w_k, a uniform u in [0, 2^32) selects target = floor(T u / 2^32) and the first candidate whose
// inclusive prefix sum exceeds it; the sample is that voxel's centre in the world frame.
#include <cub/cub.cuh>

#include "submap.h"

namespace cvx {
namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }

__global__ void sample_keys_kernel(const int4* coords, int nb, unsigned long long* keys, int* vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const int4 c = coords[i];
    keys[i] = ((unsigned long long)(c.x + (1 << 20)) << 42) | ((unsigned long long)(c.y + (1 << 20)) << 21) |
              (unsigned long long)(c.z + (1 << 20));
    vals[i] = i;
  }
}

__global__ void sample_weights_kernel(const long long* sums, const int* order, long long nvox, double thr,
                                      unsigned long long* w) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nvox; k += (long long)gridDim.x * blockDim.x) {
    const long long vi = (long long)order[k >> 9] * kBlockVox + (k & 511);
    const longlong2 sw = reinterpret_cast<const longlong2*>(sums)[vi];
    bool site = false;
    if (sw.y > 0) {
      const float D = (float)((double)sw.x / (double)sw.y);
      site = fabs((double)D) <= thr;
    }
    w[k] = site ? (unsigned long long)(sw.y >> 10) : 0ull;
  }
}

struct PickParams {
  const unsigned long long* cum;
  long long nvox;
  const unsigned* u;
  long long m;
  const int* order;
  const int4* coords;
  const long long* sums;
  double T[16];
  double s;
  float* xyz;
  float* w;
};

__global__ void sample_pick_kernel(const __grid_constant__ PickParams p) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.m) return;
  const unsigned long long total = p.cum[p.nvox - 1];
  if (total == 0ull) {
    const float qn = __int_as_float(0x7fc00000);
    p.xyz[3 * i] = qn; p.xyz[3 * i + 1] = qn; p.xyz[3 * i + 2] = qn;
    if (p.w) p.w[i] = 0.0f;
    return;
  }
  const unsigned long long target = __umul64hi(total, (unsigned long long)p.u[i] << 32);   // floor(T u / 2^32)
  long long lo = 0, hi = p.nvox - 1;                                                      // first cum > target
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (p.cum[mid] > target) hi = mid; else lo = mid + 1;
  }
  const int slot = p.order[lo >> 9], l = (int)(lo & 511);
  const int4 c = p.coords[slot];
  const double v[3] = {(double)(8 * c.x + (l & 7)), (double)(8 * c.y + ((l >> 3) & 7)), (double)(8 * c.z + (l >> 6))};
  double cs[3];
  for (int a = 0; a < 3; ++a) cs[a] = dm(da(v[a], 0.5), p.s);
  for (int a = 0; a < 3; ++a)   // world = R_WS c + t_WS, same order as the oracle
    p.xyz[3 * i + a] = (float)da(da(da(dm(p.T[4 * a], cs[0]), dm(p.T[4 * a + 1], cs[1])), dm(p.T[4 * a + 2], cs[2])), p.T[4 * a + 3]);
  if (p.w) p.w[i] = (float)((double)reinterpret_cast<const longlong2*>(p.sums)[(long long)slot * kBlockVox + l].y * (1.0 / kFxScale));
}

}  // namespace

cudaError_t launch_sample_surface(cvx_submap* sm, int n_blocks, const unsigned* uniforms, int64_t m, float* out_xyz,
                                  float* out_w, cudaStream_t st, long long* total_weight) {
  *total_weight = 0;
  if (m <= 0 || n_blocks <= 0) return cudaSuccess;
  const long long nvox = (long long)n_blocks * kBlockVox;
  unsigned long long *keys = nullptr, *keys2 = nullptr, *w = nullptr, *cum = nullptr;
  int *vals = nullptr, *order = nullptr;
  void* tmp = nullptr;
  size_t tmp1 = 0, tmp2 = 0;
  cudaError_t e = cudaSuccess;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp1, keys, keys2, vals, order, n_blocks, 0, 63, st);
  cub::DeviceScan::InclusiveSum(nullptr, tmp2, w, cum, nvox, st);
  if ((e = cudaMallocAsync(&keys, 8 * (size_t)n_blocks, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&keys2, 8 * (size_t)n_blocks, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&vals, 4 * (size_t)n_blocks, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&order, 4 * (size_t)n_blocks, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&w, 8 * (size_t)nvox, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&cum, 8 * (size_t)nvox, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&tmp, std::max(tmp1, tmp2), st)) != cudaSuccess)
    return e;
  {
    ProfScope ps_(sm, "sample_sort", st);
    sample_keys_kernel<<<(n_blocks + 255) / 256, 256, 0, st>>>(sm->pool.coords, n_blocks, keys, vals);
    cub::DeviceRadixSort::SortPairs(tmp, tmp1, keys, keys2, vals, order, n_blocks, 0, 63, st);
  }
  {
    ProfScope ps_(sm, "sample_scan", st);
    sample_weights_kernel<<<148 * 8, 256, 0, st>>>(sm->pool.sums, order, nvox, sm->cfg.site_threshold, w);
    cub::DeviceScan::InclusiveSum(tmp, tmp2, w, cum, nvox, st);
  }
  PickParams pp;
  pp.cum = cum; pp.nvox = nvox; pp.u = uniforms; pp.m = m; pp.order = order; pp.coords = sm->pool.coords;
  pp.sums = sm->pool.sums;
  for (int i = 0; i < 16; ++i) pp.T[i] = sm->T_ws[i];
  pp.s = sm->cfg.voxel_size; pp.xyz = out_xyz; pp.w = out_w;
  {
    ProfScope ps_(sm, "sample_pick", st);
    sample_pick_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(pp);
  }
  unsigned long long tot = 0;
  cudaMemcpyAsync(&tot, cum + nvox - 1, 8, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  *total_weight = (long long)tot;
  cudaFreeAsync(keys, st); cudaFreeAsync(keys2, st); cudaFreeAsync(vals, st); cudaFreeAsync(order, st);
  cudaFreeAsync(w, st); cudaFreeAsync(cum, st); cudaFreeAsync(tmp, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace cvx
