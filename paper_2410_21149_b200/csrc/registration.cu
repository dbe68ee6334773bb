// registration.cu — ESDF consumers for registration:
// weight-proportional surface-point sampling.  (Value + gradient look-ups are in query.cu.)
//
// Sampling definition (R12): the candidates are the sites (observed, |D| <= tau_site, R4) of
// all allocated blocks in lexicographic (bx, by, bz) block order and local index order inside a block;
// each carries the integer weight w_k = W_k in units of 2^-20 (W_k = the fused weight sum).  With
// T = sum w_k, a uniform u in [0, 2^32) selects target = floor(T u / 2^32) and the first candidate whose
// inclusive prefix sum exceeds it; the sample is that voxel's centre in the world frame.
//
// Implementation (no library primitives): the blocks are laid out in a lexicographic-major grid over their
// AABB (cell ((bx - lx) nby + (by - ly)) nbz + (bz - lz) holds the block's slot), each cell's total candidate
// weight is reduced by one warp, the cells' inclusive prefix sums are formed by a three-kernel exact integer
// scan (tile sums, one CTA over the tile sums, tiles), and each sample is picked by one warp: a binary search
// over the cells, then a warp prefix scan over the 512 voxel weights of the chosen block (16 per lane, local
// index order).  Integer arithmetic throughout: the picks equal the oracle's (R12).
#include "submap.h"

namespace cvx {
namespace {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }

// candidate weight of voxel vi (R12: sites of the R4 test, weight W in units of 2^-20)
__device__ __forceinline__ unsigned long long site_weight(const long long* sums, long long vi, double thr) {
  const longlong2 sw = reinterpret_cast<const longlong2*>(sums)[vi];
  if (sw.y <= 0) return 0ull;
  const float D = (float)((double)sw.x / (double)sw.y);
  return fabs((double)D) <= thr ? (unsigned long long)(sw.y >> 10) : 0ull;
}

__global__ void sample_grid_kernel(const int4* coords, int nb, int* grid, int lx, int ly, int lz, int nby, int nbz) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const int4 c = coords[i];
    grid[((long long)(c.x - lx) * nby + (c.y - ly)) * nbz + (c.z - lz)] = i;
  }
}

// one warp per cell: the block's total candidate weight (0 for an empty cell)
__global__ void sample_cell_weight_kernel(const long long* sums, const int* grid, long long ncell, double thr,
                                          unsigned long long* cw) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long c = w0; c < ncell; c += nw) {
    const int slot = grid[c];
    unsigned long long t = 0;
    if (slot >= 0)
      for (int j = 0; j < 16; ++j) t += site_weight(sums, (long long)slot * kBlockVox + 16 * lane + j, thr);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) cw[c] = t;
  }
}

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

// inclusive scan of the CTA's kScanTile values held kScanItems per thread (thread-contiguous); returns the
// thread's exclusive prefix within the tile and writes the tile total to *tile_total (thread 0)
__device__ __forceinline__ unsigned long long tile_prefix(unsigned long long mine, unsigned long long* tile_total) {
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  unsigned long long before = 0, total = 0;
  for (int w = 0; w < kScanThreads / 32; ++w) {
    if (w < warp) before += s_warp[w];
    total += s_warp[w];
  }
  __syncthreads();
  if (threadIdx.x == 0) *tile_total = total;
  return before + incl - mine;
}

__global__ void __launch_bounds__(kScanThreads) scan_tiles_kernel(const unsigned long long* in, long long n, unsigned long long* tsum) {
  const long long b = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  unsigned long long s = 0;
  for (int j = 0; j < kScanItems; ++j) if (b + j < n) s += in[b + j];
  __shared__ unsigned long long tot;
  tile_prefix(s, &tot);
  __syncthreads();
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
}

// one CTA: exclusive prefix of the tile sums, in place
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_kernel(unsigned long long* tsum, long long nt) {
  __shared__ unsigned long long tot;
  unsigned long long carry = 0;
  for (long long b0 = 0; b0 < nt; b0 += kScanTile) {
    const long long b = b0 + (long long)threadIdx.x * kScanItems;
    unsigned long long v[kScanItems], s = 0;
    for (int j = 0; j < kScanItems; ++j) { v[j] = b + j < nt ? tsum[b + j] : 0ull; s += v[j]; }
    unsigned long long ex = carry + tile_prefix(s, &tot);
    __syncthreads();
    for (int j = 0; j < kScanItems; ++j) { if (b + j < nt) tsum[b + j] = ex; ex += v[j]; }
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const unsigned long long* in, long long n,
                                                                  const unsigned long long* tex, unsigned long long* out) {
  const long long b = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  unsigned long long v[kScanItems], s = 0;
  for (int j = 0; j < kScanItems; ++j) { v[j] = b + j < n ? in[b + j] : 0ull; s += v[j]; }
  __shared__ unsigned long long tot;
  unsigned long long acc = tex[blockIdx.x] + tile_prefix(s, &tot);
  for (int j = 0; j < kScanItems; ++j) { acc += v[j]; if (b + j < n) out[b + j] = acc; }
}

struct PickParams {
  const unsigned long long* cum;   // inclusive prefix of the cell weights
  long long ncell;
  const int* grid;
  const unsigned* u;
  long long m;
  const int4* coords;
  const long long* sums;
  double thr;
  double T[16];
  double s;
  float* xyz;
  float* w;
};

// one warp per sample
__global__ void sample_pick_kernel(const __grid_constant__ PickParams p) {
  const int lane = threadIdx.x & 31;
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= p.m) return;
  const unsigned long long total = p.cum[p.ncell - 1];
  if (total == 0ull) {
    if (lane == 0) {
      const float qn = __int_as_float(0x7fc00000);
      p.xyz[3 * i] = qn; p.xyz[3 * i + 1] = qn; p.xyz[3 * i + 2] = qn;
      if (p.w) p.w[i] = 0.0f;
    }
    return;
  }
  const unsigned long long target = __umul64hi(total, (unsigned long long)p.u[i] << 32);   // floor(T u / 2^32)
  long long lo = 0, hi = p.ncell - 1;                                                     // first cum > target
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (p.cum[mid] > target) hi = mid; else lo = mid + 1;
  }
  const unsigned long long r = target - (lo > 0 ? p.cum[lo - 1] : 0ull);   // < the block's weight
  const int slot = p.grid[lo];
  unsigned long long wv[16], s = 0;
  for (int j = 0; j < 16; ++j) { wv[j] = site_weight(p.sums, (long long)slot * kBlockVox + 16 * lane + j, p.thr); s += wv[j]; }
  unsigned long long incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned long long excl = incl - s;
  const unsigned hit = __ballot_sync(0xffffffffu, r >= excl && r < incl);   // exactly one lane
  const int src = __ffs(hit) - 1;
  if (lane != src) return;
  unsigned long long acc = excl;
  int j = 0;
  while (acc + wv[j] <= r) acc += wv[j++];   // first voxel whose inclusive prefix exceeds r
  const int l = 16 * lane + j;
  const int4 c = p.coords[slot];
  const double v[3] = {(double)(8 * c.x + (l & 7)), (double)(8 * c.y + ((l >> 3) & 7)), (double)(8 * c.z + (l >> 6))};
  double cs[3];
  for (int a = 0; a < 3; ++a) cs[a] = dm(da(v[a], 0.5), p.s);
  for (int a = 0; a < 3; ++a)   // world = R_WS c + t_WS, same order as the oracle
    p.xyz[3 * i + a] = (float)da(da(da(dm(p.T[4 * a], cs[0]), dm(p.T[4 * a + 1], cs[1])), dm(p.T[4 * a + 2], cs[2])), p.T[4 * a + 3]);
  if (p.w) p.w[i] = (float)((double)reinterpret_cast<const longlong2*>(p.sums)[(long long)slot * kBlockVox + l].y * (1.0 / kFxScale));
}

}  // namespace

cudaError_t launch_sample_surface(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], const unsigned* uniforms,
                                  int64_t m, float* out_xyz, float* out_w, cudaStream_t st, long long* total_weight) {
  *total_weight = 0;
  if (m <= 0 || n_blocks <= 0) return cudaSuccess;
  const int nbx = hi[0] - lo[0] + 1, nby = hi[1] - lo[1] + 1, nbz = hi[2] - lo[2] + 1;
  const long long ncell = (long long)nbx * nby * nbz;
  const long long ntile = (ncell + kScanTile - 1) / kScanTile;
  int* grid = nullptr;
  unsigned long long *cw = nullptr, *cum = nullptr, *tsum = nullptr;
  cudaError_t e = cudaSuccess;
  if ((e = cudaMallocAsync(&grid, 4 * (size_t)ncell, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&cw, 8 * (size_t)ncell, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&cum, 8 * (size_t)ncell, st)) != cudaSuccess ||
      (e = cudaMallocAsync(&tsum, 8 * (size_t)ntile, st)) != cudaSuccess)
    return e;
  cudaMemsetAsync(grid, 0xff, 4 * (size_t)ncell, st);
  {
    ProfScope ps_(sm, "sample_sort", st);   // lexicographic block order = the grid's cell order
    sample_grid_kernel<<<148 * 4, 256, 0, st>>>(sm->pool.coords, n_blocks, grid, lo[0], lo[1], lo[2], nby, nbz);
  }
  {
    ProfScope ps_(sm, "sample_scan", st);
    sample_cell_weight_kernel<<<148 * 8, 256, 0, st>>>(sm->pool.sums, grid, ncell, sm->cfg.site_threshold, cw);
    scan_tiles_kernel<<<(unsigned)ntile, kScanThreads, 0, st>>>(cw, ncell, tsum);
    scan_tile_sums_kernel<<<1, kScanThreads, 0, st>>>(tsum, ntile);
    scan_apply_kernel<<<(unsigned)ntile, kScanThreads, 0, st>>>(cw, ncell, tsum, cum);
  }
  PickParams pp;
  pp.cum = cum; pp.ncell = ncell; pp.grid = grid; pp.u = uniforms; pp.m = m; pp.coords = sm->pool.coords;
  pp.sums = sm->pool.sums; pp.thr = sm->cfg.site_threshold;
  for (int i = 0; i < 16; ++i) pp.T[i] = sm->T_ws[i];
  pp.s = sm->cfg.voxel_size; pp.xyz = out_xyz; pp.w = out_w;
  {
    ProfScope ps_(sm, "sample_pick", st);
    sample_pick_kernel<<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(pp);
  }
  unsigned long long tot = 0;
  cudaMemcpyAsync(&tot, cum + ncell - 1, 8, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  *total_weight = (long long)tot;
  cudaFreeAsync(grid, st); cudaFreeAsync(cw, st); cudaFreeAsync(cum, st); cudaFreeAsync(tsum, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace cvx
