// esdf.cu — exact ESDF finalize for sm_100a.
//
// PBA-class separable exact EDT over the dense AABB of the allocated blocks (O10-O12):
//   block_grid_kernel  slot index per block of the AABB (direct index, no hashing in the passes)
//   pass_x_kernel      one warp per x-row: reads the TSDF sums of the row's allocated voxels (coalesced,
//                      8 voxels x 16 B per block row), decides sites S = {W > 0, |D| <= tau_site} with
//                      warp ballots, writes the sign/observed placeholder of E, and the exact 1-D
//                      distance to the nearest site along x (uint16) from per-chunk bit masks kept in
//                      shared memory (prefix max / suffix min scans across chunks).
//   pass_yz_kernel     one thread per line (consecutive x in a warp -> coalesced): lower envelope of
//                      parabolas f(q) + (p - q)^2 (Meijster / Felzenszwalb-Huttenlocher) with the
//                      stack stored in place as per-voxel {prev, start} links (PBA phase 2 idea: the
//                      proximate sites live at their own positions), integer arithmetic throughout.
//                      Pass y writes the 2-D squared distance (uint32); pass z writes E = sign * s *
//                      sqrt(d^2) straight into the 8^3 ESDF blocks (NaN unobserved, +inf no sites).
#include <algorithm>

#include "submap.h"

namespace cvx {
namespace {

constexpr unsigned kNone16 = 0xffffu;
constexpr unsigned kInf32 = 0xffffffffu;
constexpr long long kInfF = 1ll << 62;

// slot of every block of the AABB (-1 = not allocated) and, per (bx, by) column, whether any block of
// the column is allocated (pass z skips empty columns: they hold no voxel to write)
__global__ void block_grid_kernel(const Counters* ctr, const int4* coords, int max_blocks, int* grid,
                                  unsigned char* colmask, unsigned char* rowmask, int lx, int ly, int lz, int nbx,
                                  int nby) {
  const int nb = min(ctr->n_blocks, max_blocks);
  for (int sIdx = blockIdx.x * blockDim.x + threadIdx.x; sIdx < nb; sIdx += gridDim.x * blockDim.x) {
    int4 c = coords[sIdx];
    grid[((long long)(c.z - lz) * nby + (c.y - ly)) * nbx + (c.x - lx)] = sIdx;
    colmask[(long long)(c.y - ly) * nbx + (c.x - lx)] = 1;
    rowmask[(long long)(c.z - lz) * nby + (c.y - ly)] = 1;
  }
}

struct XParams {
  const long long* sums;
  float* esdf;
  const int* grid;
  const unsigned char* rowmask;   // (by, bz) block rows with allocated blocks
  unsigned short* g1;
  int nx, ny, nz, nbx, nby;
  double site_thr;
};

__global__ void __launch_bounds__(128) pass_x_kernel(const __grid_constant__ XParams p) {
  extern __shared__ unsigned smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (p.nx + 31) >> 5;
  unsigned* msk = smem + warp * 3 * nch;
  int* prv = reinterpret_cast<int*>(msk + nch);
  int* nxt = prv + nch;
  const long long rows = (long long)p.ny * p.nz;
  const int kNeg = -(1 << 30), kPos = 1 << 30;
  for (long long row = (long long)blockIdx.x * 4 + warp; row < rows; row += (long long)gridDim.x * 4) {
    const int y = (int)(row % p.ny), z = (int)(row / p.ny);
    if (!p.rowmask[(long long)(z >> 3) * p.nby + (y >> 3)]) {   // no block in this row: no site, no voxel
      unsigned short* out = p.g1 + row * p.nx;
      for (int x = lane; x < p.nx; x += 32) out[x] = (unsigned short)kNone16;
      continue;
    }
    const int* grow = p.grid + ((long long)(z >> 3) * p.nby + (y >> 3)) * p.nbx;
    const int lyz = 8 * (y & 7) + 64 * (z & 7);
    // 1) sites of the row -> one 32-bit mask per chunk; E placeholder (sign of D, NaN if unobserved)
    for (int c = 0; c < nch; ++c) {
      const int x = (c << 5) + lane;
      bool site = false;
      if (x < p.nx) {
        const int slot = grow[x >> 3];
        if (slot >= 0) {
          const long long vi = (long long)slot * kBlockVox + (x & 7) + lyz;
          const longlong2 sw = reinterpret_cast<const longlong2*>(p.sums)[vi];
          float ph;
          if (sw.y > 0) {
            const float D = (float)((double)sw.x / (double)sw.y);   // exported D (stage-isolated parity)
            site = fabs((double)D) <= p.site_thr;                    // O10
            ph = D < 0.0f ? -0.0f : 0.0f;
          } else {
            ph = __int_as_float(0x7fc00000);                        // unobserved -> NaN (O11)
          }
          p.esdf[vi] = ph;
        }
      }
      const unsigned b = __ballot_sync(0xffffffffu, site);
      if (lane == 0) msk[c] = b;
    }
    __syncwarp();
    // 2) nearest site strictly before / after each chunk (warp scans over groups of 32 chunks)
    int carry = kNeg;
    for (int g = 0; g < nch; g += 32) {
      const int c = g + lane;
      const unsigned m = c < nch ? msk[c] : 0u;
      int last = m ? (c << 5) + 31 - __clz(m) : kNeg;
      int incl = last;
      for (int o = 1; o < 32; o <<= 1) { int t = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl = max(incl, t); }
      int excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = kNeg;
      if (c < nch) prv[c] = max(excl, carry);
      carry = max(carry, __shfl_sync(0xffffffffu, incl, 31));
    }
    carry = kPos;
    for (int g = ((nch - 1) >> 5) << 5; g >= 0; g -= 32) {
      const int c = g + lane;
      const unsigned m = c < nch ? msk[c] : 0u;
      int first = m ? (c << 5) + __ffs(m) - 1 : kPos;
      int incl = first;
      for (int o = 1; o < 32; o <<= 1) { int t = __shfl_down_sync(0xffffffffu, incl, o); if (lane + o < 32) incl = min(incl, t); }
      int excl = __shfl_down_sync(0xffffffffu, incl, 1);
      if (lane == 31) excl = kPos;
      if (c < nch) nxt[c] = min(excl, carry);
      carry = min(carry, __shfl_sync(0xffffffffu, incl, 0));
    }
    __syncwarp();
    // 3) exact 1-D distance along x
    unsigned short* out = p.g1 + row * p.nx;
    for (int c = 0; c < nch; ++c) {
      const int x = (c << 5) + lane;
      if (x >= p.nx) break;
      const unsigned m = msk[c];
      const unsigned lm = m & (0xffffffffu >> (31 - lane));     // bits <= lane
      const unsigned rm = m & (0xffffffffu << lane);            // bits >= lane
      const int L = lm ? (c << 5) + 31 - __clz(lm) : prv[c];
      const int R = rm ? (c << 5) + __ffs(rm) - 1 : nxt[c];
      const long long dl = (long long)x - L, dr = (long long)R - x;
      const long long d = dl < dr ? dl : dr;
      out[x] = (unsigned short)(d >= (long long)kNone16 ? kNone16 : d);
    }
    __syncwarp();
  }
}

struct LineParams {
  const void* fin;          // pass y: uint16 1-D distances; pass z: uint32 squared distances
  unsigned* gout;           // pass y output (uint32 squared distances)
  unsigned* meta;           // per-voxel stack links {start t: hi 16, prev: lo 16}
  float* esdf;              // pass z output (ESDF blocks)
  const int* grid;
  const unsigned char* colmask;   // (bx, by) columns with allocated blocks
  int nx, ny, nz, nbx, nby;
  float s;
};

__device__ __forceinline__ long long floordiv(long long a, long long b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

// Lower envelope along one line of length m; element q lives at base + q*stride.
template <bool kZ>
__global__ void __launch_bounds__(256) pass_line_kernel(const __grid_constant__ LineParams p) {
  const long long nlines = kZ ? (long long)p.nx * p.ny : (long long)p.nx * p.nz;
  const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= nlines) return;
  const int x = (int)(line % p.nx);
  const int o2 = (int)(line / p.nx);                  // pass y: z ; pass z: y
  const int m = kZ ? p.nz : p.ny;
  const long long stride = kZ ? (long long)p.nx * p.ny : (long long)p.nx;
  const long long base = kZ ? (long long)o2 * p.nx + x : (long long)o2 * p.nx * p.ny + x;
  if (kZ && !p.colmask[(long long)(o2 >> 3) * p.nbx + (x >> 3)]) return;   // no allocated voxel in this line
  auto f_at = [&](int q) -> long long {
    if (kZ) {
      unsigned v = static_cast<const unsigned*>(p.fin)[base + q * stride];
      return v == kInf32 ? kInfF : (long long)v;
    } else {
      unsigned v = static_cast<const unsigned short*>(p.fin)[base + q * stride];
      return v == kNone16 ? kInfF : (long long)v * v;
    }
  };
  // forward: build the envelope (Meijster phase 2 with a linked stack).  The line is read in chunks
  // of 8 independent loads so each thread keeps 8 requests in flight (the pass is latency-bound).
  int top = -1, t_top = 0;
  long long f_top = 0;
  for (int q0 = 0; q0 < m; q0 += 8) {
    long long fv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) fv[u] = q0 + u < m ? f_at(q0 + u) : kInfF;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u;
      const long long fq = fv[u];
      if (fq >= kInfF) continue;
      while (top >= 0) {
        const long long a = (long long)(t_top - top), b = (long long)(t_top - q);
        if (a * a + f_top > b * b + fq) {                 // q beats top already at top's start: pop
          const unsigned mt = p.meta[base + (long long)top * stride];
          const int pr = (int)(mt & 0xffffu);
          if (pr == 0xffff) { top = -1; break; }
          top = pr;
          t_top = (int)(p.meta[base + (long long)top * stride] >> 16);
          f_top = f_at(top);
        } else {
          break;
        }
      }
      int tq;
      if (top < 0) {
        tq = 0;
      } else {
        const long long num = (long long)q * q - (long long)top * top + fq - f_top;
        const long long sep = floordiv(num, 2ll * (q - top));   // last position where top is <= q
        if (sep + 1 >= m) continue;                             // q never wins inside the line
        tq = (int)(sep + 1);
      }
      p.meta[base + (long long)q * stride] = ((unsigned)tq << 16) | (unsigned)(top < 0 ? 0xffff : top);
      top = q; t_top = tq; f_top = fq;
    }
  }
  // backward: read the envelope from the right, one 8-voxel chunk (= one block along the line) at a
  // time; pass z prefetches the chunk's sign/observed placeholders before evaluating it.
  const int bx = x >> 3;
  for (int q0 = m - 8; q0 >= 0; q0 -= 8) {
    int slot = -1;
    float ph[8];
    if (kZ) {
      slot = p.grid[((long long)(q0 >> 3) * p.nby + (o2 >> 3)) * p.nbx + bx];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        ph[u] = slot >= 0 ? p.esdf[(long long)slot * kBlockVox + (x & 7) + 8 * (o2 & 7) + 64 * u]
                          : __int_as_float(0x7fc00000);
    }
#pragma unroll
    for (int u = 7; u >= 0; --u) {
      const int q = q0 + u;
      long long d2 = kInfF;
      if (top >= 0) {
        const long long dq = (long long)(q - top);
        d2 = dq * dq + f_top;
      }
      if (!kZ) {
        p.gout[base + (long long)q * stride] = d2 >= kInfF ? kInf32 : (unsigned)d2;
      } else if (!isnan(ph[u])) {
        float e;
        if (d2 >= kInfF) e = __int_as_float(0x7f800000);             // S empty -> +inf (O11)
        else e = copysignf((float)((double)p.s * sqrt((double)d2)), ph[u]);
        p.esdf[(long long)slot * kBlockVox + (x & 7) + 8 * (o2 & 7) + 64 * u] = e;
      }
      if (top >= 0 && q == t_top) {
        const int pr = (int)(p.meta[base + (long long)top * stride] & 0xffffu);
        if (pr == 0xffff) { top = -1; }
        else { top = pr; t_top = (int)(p.meta[base + (long long)top * stride] >> 16); f_top = f_at(top); }
      }
    }
  }
}

}  // namespace

cudaError_t launch_finalize(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], cudaStream_t st) {
  if (n_blocks <= 0) return cudaSuccess;
  const int nbx = hi[0] - lo[0] + 1, nby = hi[1] - lo[1] + 1, nbz = hi[2] - lo[2] + 1;
  const int nx = 8 * nbx, ny = 8 * nby, nz = 8 * nbz;
  const long long nblk = (long long)nbx * nby * nbz;
  const long long nvox = (long long)nx * ny * nz;
  cudaError_t e;
  if (sm->block_grid_cap < nblk) {
    if (sm->block_grid) cudaFree(sm->block_grid);
    sm->block_grid = nullptr; sm->block_grid_cap = 0;
    if ((e = cudaMalloc(&sm->block_grid, sizeof(int) * (size_t)nblk)) != cudaSuccess) return e;
    sm->block_grid_cap = nblk;
  }
  const long long need = nvox * (2 + 4 + 4) + (long long)nbx * nby + (long long)nby * nbz + 256;
  if (sm->edt_bytes < need) {
    if (sm->edt) cudaFree(sm->edt);
    sm->edt = nullptr; sm->edt_bytes = 0;
    if ((e = cudaMalloc(&sm->edt, (size_t)need)) != cudaSuccess) return e;
    sm->edt_bytes = need;
  }
  unsigned* g2 = reinterpret_cast<unsigned*>(sm->edt);
  unsigned* meta = g2 + nvox;
  unsigned short* g1 = reinterpret_cast<unsigned short*>(meta + nvox);

  unsigned char* colmask = reinterpret_cast<unsigned char*>(g1 + nvox);
  cudaMemsetAsync(sm->block_grid, 0xff, sizeof(int) * (size_t)nblk, st);
  unsigned char* rowmask = colmask + (size_t)nbx * nby;
  cudaMemsetAsync(colmask, 0, (size_t)nbx * nby + (size_t)nby * nbz, st);
  {
    ProfScope ps_(sm, "esdf_block_grid", st);
    block_grid_kernel<<<148 * 4, 256, 0, st>>>(sm->ctr, sm->pool.coords, sm->pool.max_blocks, sm->block_grid,
                                               colmask, rowmask, lo[0], lo[1], lo[2], nbx, nby);
  }
  XParams xp;
  xp.sums = sm->pool.sums; xp.esdf = sm->pool.esdf; xp.grid = sm->block_grid; xp.g1 = g1; xp.rowmask = rowmask;
  xp.nx = nx; xp.ny = ny; xp.nz = nz; xp.nbx = nbx; xp.nby = nby; xp.site_thr = sm->cfg.site_threshold;
  const int nch = (nx + 31) / 32;
  const size_t smem = (size_t)4 * 3 * nch * sizeof(unsigned);
  if (smem > 48 * 1024) cudaFuncSetAttribute(pass_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long rows = (long long)ny * nz;
  const unsigned xblocks = (unsigned)std::min<long long>((rows + 3) / 4, 148ll * 16);
  {
    ProfScope ps_(sm, "esdf_pass_x", st);
    pass_x_kernel<<<xblocks, 128, smem, st>>>(xp);
  }

  LineParams lp;
  lp.fin = g1; lp.gout = g2; lp.meta = meta; lp.esdf = sm->pool.esdf; lp.grid = sm->block_grid; lp.colmask = colmask;
  lp.nx = nx; lp.ny = ny; lp.nz = nz; lp.nbx = nbx; lp.nby = nby; lp.s = (float)sm->cfg.voxel_size;
  long long nl = (long long)nx * nz;
  {
    ProfScope ps_(sm, "esdf_pass_y", st);
    pass_line_kernel<false><<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(lp);
  }
  lp.fin = g2;
  nl = (long long)nx * ny;
  {
    ProfScope ps_(sm, "esdf_pass_z", st);
    pass_line_kernel<true><<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(lp);
  }
  return cudaGetLastError();
}

}  // namespace cvx
