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

#ifndef CVX_XCH
#define CVX_XCH 4
#endif
constexpr int kXCh = CVX_XCH;   // chunks (32 voxels each) whose loads a warp issues together in pass x

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
    // 1) sites of the row -> one 32-bit mask per chunk; E placeholder (sign of D, NaN if unobserved).
    //    kXCh chunks per round: their slot look-ups, then their TSDF loads, are issued back to back so
    //    every warp keeps kXCh 512-byte requests in flight (the row loop is otherwise latency-bound).
    for (int c0 = 0; c0 < nch; c0 += kXCh) {
      int slot[kXCh];
#pragma unroll
      for (int u = 0; u < kXCh; ++u) {
        const int x = ((c0 + u) << 5) + lane;
        slot[u] = (c0 + u < nch && x < p.nx) ? grow[x >> 3] : -1;
      }
      longlong2 sw[kXCh];
#pragma unroll
      for (int u = 0; u < kXCh; ++u) {
        const long long vi = (long long)slot[u] * kBlockVox + (lane & 7) + lyz;   // x & 7 == lane & 7
        sw[u] = slot[u] >= 0 ? reinterpret_cast<const longlong2*>(p.sums)[vi] : make_longlong2(0, 0);
      }
#pragma unroll
      for (int u = 0; u < kXCh; ++u) {
        bool site = false;
        if (slot[u] >= 0) {
          const long long vi = (long long)slot[u] * kBlockVox + (lane & 7) + lyz;
          float ph;
          if (sw[u].y > 0) {
            const float D = (float)((double)sw[u].x / (double)sw[u].y);   // exported D (stage-isolated parity)
            site = fabs((double)D) <= p.site_thr;                          // O10
            ph = D < 0.0f ? -0.0f : 0.0f;
          } else {
            ph = __int_as_float(0x7fc00000);                              // unobserved -> NaN (O11)
          }
          p.esdf[vi] = ph;
        }
        const unsigned b = __ballot_sync(0xffffffffu, site);
        if (lane == 0 && c0 + u < nch) msk[c0 + u] = b;
      }
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
  void* meta;               // per pushed voxel q — pass z: u64 envelope state below q {f: hi 32, t: 16,
                            // prev: lo 16}; pass y: u32 {t_q: hi 16, prev: lo 16}
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
// kSplit = 2 (pass y, whose line count nx*nz is small): the two halves of a line go to lanes l and l+16
// of one warp; each builds the envelope of the sites in its half and evaluates it over the whole line,
// and the two results are combined with one shuffle per position (2x the evaluation work, 2x the
// threads in flight for a latency-bound pass).
#ifndef CVX_META64Y
#define CVX_META64Y 0
#endif
constexpr bool kMeta64Y = CVX_META64Y;
#ifndef CVX_EDT_LAYOUT
#define CVX_EDT_LAYOUT 0
#endif

template <bool kZ, int kSplit>
__global__ void __launch_bounds__(256) pass_line_kernel(const __grid_constant__ LineParams p) {
  const long long nlines = kZ ? (long long)p.nx * p.ny : (long long)p.nx * p.nz;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int half = kSplit == 2 ? (lane >> 4) : 0;
  const long long line = kSplit == 2 ? (tid >> 5) * 16 + (lane & 15) : tid;
  const bool valid = line < nlines;
  if (kSplit == 1 && !valid) return;
  if (kSplit == 2 && ((tid >> 5) * 16) >= nlines) return;   // whole warp beyond the lines
  const int x = valid ? (int)(line % p.nx) : 0;
  const int o2 = valid ? (int)(line / p.nx) : 0;      // pass y: z ; pass z: y
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
  const int qa = kSplit == 2 ? half * (m >> 1) : 0, qb = kSplit == 2 ? qa + (m >> 1) : m;
  int top = -1, t_top = 0;
  long long f_top = 0;
  // Stack links.  Pass z stores with every pushed q the full state of the element below it, so a pop
  // is ONE load; pass y (u16 input, re-read cheaply) keeps 4-byte links {t_q, prev} and re-reads f —
  // measured: the 8-byte form costs pass y more in bytes than it saves in latency, pass z the opposite.
  // forward: build the envelope (Meijster phase 2 with a linked stack) of the sites in [qa, qb).  The
  // line is read in chunks of 8 independent loads so each thread keeps 8 requests in flight.
  for (int q0 = qa; q0 < qb; q0 += 8) {
    long long fv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) fv[u] = (valid && q0 + u < qb) ? f_at(q0 + u) : kInfF;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u;
      const long long fq = fv[u];
      if (fq >= kInfF) continue;
      while (top >= 0) {
        const long long a = (long long)(t_top - top), b = (long long)(t_top - q);
        if (a * a + f_top > b * b + fq) {                 // q beats top already at top's start: pop
          if constexpr (kZ || kMeta64Y) {   // one load restores the whole state below top
            const unsigned long long mt = static_cast<const unsigned long long*>(p.meta)[base + (long long)top * stride];
            const int pr = (int)(mt & 0xffffu);
            if (pr == 0xffff) { top = -1; break; }
            top = pr; t_top = (int)((mt >> 16) & 0xffffu); f_top = (long long)(mt >> 32);
          } else {
            const unsigned mt = static_cast<const unsigned*>(p.meta)[base + (long long)top * stride];
            const int pr = (int)(mt & 0xffffu);
            if (pr == 0xffff) { top = -1; break; }
            top = pr;
            t_top = (int)(static_cast<const unsigned*>(p.meta)[base + (long long)top * stride] >> 16);
            f_top = f_at(top);
          }
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
      if constexpr (kZ || kMeta64Y)
        static_cast<unsigned long long*>(p.meta)[base + (long long)q * stride] = top < 0 ? 0xffffull
            : ((unsigned long long)f_top << 32) | ((unsigned long long)t_top << 16) | (unsigned long long)top;
      else
        static_cast<unsigned*>(p.meta)[base + (long long)q * stride] =
            ((unsigned)tq << 16) | (unsigned)(top < 0 ? 0xffff : top);
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
      if (kSplit == 2) d2 = min(d2, __shfl_xor_sync(0xffffffffu, d2, 16));
      if (!kZ) {
        if (valid && half == 0) p.gout[base + (long long)q * stride] = d2 >= kInfF ? kInf32 : (unsigned)d2;
      } else if (!isnan(ph[u])) {
        float e;
        if (d2 >= kInfF) e = __int_as_float(0x7f800000);             // S empty -> +inf (O11)
        else e = copysignf((float)((double)p.s * sqrt((double)d2)), ph[u]);
        p.esdf[(long long)slot * kBlockVox + (x & 7) + 8 * (o2 & 7) + 64 * u] = e;
      }
      if (top >= 0 && q == t_top) {
        if constexpr (kZ || kMeta64Y) {
          const unsigned long long mt = static_cast<const unsigned long long*>(p.meta)[base + (long long)top * stride];
          const int pr = (int)(mt & 0xffffu);
          if (pr == 0xffff) { top = -1; }
          else { top = pr; t_top = (int)((mt >> 16) & 0xffffu); f_top = (long long)(mt >> 32); }
        } else {
          const unsigned* mm = static_cast<const unsigned*>(p.meta);
          const int pr = (int)(mm[base + (long long)top * stride] & 0xffffu);
          if (pr == 0xffff) { top = -1; }
          else { top = pr; t_top = (int)(mm[base + (long long)top * stride] >> 16); f_top = f_at(top); }
        }
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
  const long long need = nvox * (2 + 4 + 8) + (long long)nbx * nby + (long long)nby * nbz + 256;
  if (sm->edt_bytes < need) {
    if (sm->edt) cudaFree(sm->edt);
    sm->edt = nullptr; sm->edt_bytes = 0;
    if ((e = cudaMalloc(&sm->edt, (size_t)need)) != cudaSuccess) return e;
    sm->edt_bytes = need;
  }
#if CVX_EDT_LAYOUT == 0
  unsigned* g2 = reinterpret_cast<unsigned*>(sm->edt);
  unsigned long long* meta = reinterpret_cast<unsigned long long*>(g2 + nvox);   // nvox % 512 == 0: aligned
  unsigned short* g1 = reinterpret_cast<unsigned short*>(meta + nvox);
  unsigned char* colmask = reinterpret_cast<unsigned char*>(g1 + nvox);
#else
  unsigned short* g1 = reinterpret_cast<unsigned short*>(sm->edt);
  unsigned* g2 = reinterpret_cast<unsigned*>(g1 + nvox);
  unsigned long long* meta = reinterpret_cast<unsigned long long*>(g2 + nvox);
  unsigned char* colmask = reinterpret_cast<unsigned char*>(meta + nvox);
#endif
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
    // (the 2-way split of pass_line_kernel measured no faster on configs[1] and 1.6x slower on configs[4])
    pass_line_kernel<false, 1><<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(lp);
  }
  lp.fin = g2;
  nl = (long long)nx * ny;
  {
    ProfScope ps_(sm, "esdf_pass_z", st);
    pass_line_kernel<true, 1><<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(lp);
  }
  return cudaGetLastError();
}

}  // namespace cvx

// ================================================================================================
// Incremental ESDF: keep, per voxel, a pointer to its nearest site
// (packed offset) and, after new integration, update only what changed:
//   inc_classify   new / removed sites (site = observed and |D| <= tau_site, R4) per voxel; new blocks
//                  start without a parent; blocks with changes are queued (one region queue = one block)
//   inc_invalidate "raise": every voxel whose parent is no longer a site loses it (one direct check per
//                  voxel instead of a wavefront)
//   inc_propagate  "lower": per queued block, one CTA relaxes the 8^3 voxels plus the neighbour faces in
//                  shared memory (sweeps along all axis directions until the block is stable, P:L149
//                  "process every axis direction within each queued block"), writes back, and queues the
//                  neighbour blocks whose shared face changed; repeated until no block is queued
//   inc_write      E = sign(D) s |v - parent| (NaN unobserved, +inf without a site)
// The fixpoint is the 6-neighbour parent-propagation distance of the paper's scheme, not always the
// exact EDT; tests/test_gpu_esdf_incremental.py bounds the difference to finalize_esdf.
namespace cvx {
namespace {

constexpr unsigned long long kNoPar = 1ull << 63;
constexpr unsigned long long kFld = (1ull << 21) - 1;

__device__ __forceinline__ unsigned long long pack3(int x, int y, int z) {
  return ((unsigned long long)(x & (int)kFld) << 42) | ((unsigned long long)(y & (int)kFld) << 21) |
         (unsigned long long)(z & (int)kFld);
}
__device__ __forceinline__ int fld(unsigned long long p, int sh) {
  return (int)((long long)(p << (43 - sh)) >> 43);   // sign-extend the 21-bit field at bit sh
}

struct IncParams {
  const long long* sums;
  float* esdf;
  const int4* coords;
  unsigned long long* par;   // per voxel: packed offset (parent - v), kNoPar = none
  unsigned* sitebits;        // per block: 16 x 32 bits
  int* active;               // per block: queued flag
  int* list;                 // compacted queue
  int* cnt;                  // queue length
  const int* grid;           // dense slot grid over the AABB
  int lo0, lo1, lo2, nbx, nby, nbz;
  int nb, nb_prev;
  double site_thr;
  float s;
};

__device__ __forceinline__ int grid_slot(const IncParams& p, int bx, int by, int bz) {
  bx -= p.lo0; by -= p.lo1; bz -= p.lo2;
  if (bx < 0 || by < 0 || bz < 0 || bx >= p.nbx || by >= p.nby || bz >= p.nbz) return -1;
  return p.grid[((long long)bz * p.nby + by) * p.nbx + bx];
}

__device__ __forceinline__ bool is_site(const IncParams& p, long long vi, bool& observed, bool& neg) {
  const longlong2 sw = reinterpret_cast<const longlong2*>(p.sums)[vi];
  observed = sw.y > 0;
  if (!observed) { neg = false; return false; }
  const float D = (float)((double)sw.x / (double)sw.y);
  neg = D < 0.0f;
  return fabs((double)D) <= p.site_thr;
}

__global__ void inc_classify(const __grid_constant__ IncParams p) {
  const long long n = (long long)p.nb * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int slot = (int)(i >> 9), l = (int)(i & 511);
    bool obs, neg;
    const bool site = is_site(p, i, obs, neg);
    const bool fresh = slot >= p.nb_prev;
    const bool old = !fresh && ((p.sitebits[(long long)slot * 16 + (l >> 5)] >> (l & 31)) & 1u);
    if (fresh) p.par[i] = site ? 0ull : kNoPar;
    else if (site && !old) p.par[i] = 0ull;
    else if (!site && old) p.par[i] = kNoPar;
    const unsigned bits = __ballot_sync(0xffffffffu, site);   // 32 consecutive voxels of one block
    if ((l & 31) == 0) p.sitebits[(long long)slot * 16 + (l >> 5)] = bits;
    if (fresh || site != old) p.active[slot] = 1;
  }
}

__global__ void inc_invalidate(const __grid_constant__ IncParams p) {
  const long long n = (long long)p.nb_prev * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long q = p.par[i];
    if (q == kNoPar || q == 0ull) continue;
    const int slot = (int)(i >> 9), l = (int)(i & 511);
    const int4 c = p.coords[slot];
    const int px = 8 * c.x + (l & 7) + fld(q, 42), py = 8 * c.y + ((l >> 3) & 7) + fld(q, 21),
              pz = 8 * c.z + (l >> 6) + fld(q, 0);
    const int ps = grid_slot(p, px >> 3, py >> 3, pz >> 3);
    const int pl = (px & 7) | ((py & 7) << 3) | ((pz & 7) << 6);
    const bool alive = ps >= 0 && ((p.sitebits[(long long)ps * 16 + (pl >> 5)] >> (pl & 31)) & 1u);
    if (!alive) { p.par[i] = kNoPar; p.active[slot] = 1; }
  }
}

__global__ void inc_compact(const __grid_constant__ IncParams p) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < p.nb; b += gridDim.x * blockDim.x)
    if (p.active[b]) { p.active[b] = 0; p.list[atomicAdd(p.cnt, 1)] = b; }
}

// squared distance from local voxel (x,y,z) to a parent given relative to the block origin
__device__ __forceinline__ long long pd2(unsigned long long a, int x, int y, int z) {
  const long long dx = fld(a, 42) - x, dy = fld(a, 21) - y, dz = fld(a, 0) - z;
  return dx * dx + dy * dy + dz * dz;
}

// one 64-thread CTA per queued block (grid-stride over the queue); shared memory holds the block + its 6
// face neighbours (10^3 halo cube) as parents relative to the block origin.  The block is relaxed by
// directional sweeps ("process every axis direction within each queued block"): thread t owns
// line t along the swept axis and carries the best parent forward (then backward) over the 8 voxels;
// rounds of the six sweeps repeat until no voxel changes, which is the 6-neighbour local fixpoint.
__global__ void __launch_bounds__(64) inc_propagate(const __grid_constant__ IncParams p) {
  __shared__ unsigned long long cur[1000];
  __shared__ int nb_slot[6];
  __shared__ int face_changed[6];
  const int qlen = *(volatile const int*)p.cnt;
  const int t = threadIdx.x;
  for (int qi = blockIdx.x; qi < qlen; qi += gridDim.x) {
    __syncthreads();
    const int slot = p.list[qi];
    const int4 c = p.coords[slot];
    if (t < 6) {
      const int d = (t >> 1), sg = (t & 1) ? 1 : -1;
      nb_slot[t] = grid_slot(p, c.x + (d == 0) * sg, c.y + (d == 1) * sg, c.z + (d == 2) * sg);
      face_changed[t] = 0;
    }
    __syncthreads();
    for (int l = t; l < 512; l += 64) {
      const int x = l & 7, y = (l >> 3) & 7, z = l >> 6;
      const unsigned long long q = p.par[(long long)slot * kBlockVox + l];
      cur[(x + 1) + 10 * (y + 1) + 100 * (z + 1)] = q == kNoPar ? kNoPar : pack3(x + fld(q, 42), y + fld(q, 21), z + fld(q, 0));
    }
    for (int k = t; k < 384; k += 64) {   // face halo: 6 faces x 64 voxels
      const int f = k >> 6, a = k & 7, b = (k >> 3) & 7, d = f >> 1, hi = f & 1;
      const int ns = nb_slot[f];
      int x, y, z, nl;
      if (d == 0) { x = hi ? 8 : -1; y = a; z = b; nl = (hi ? 0 : 7) | (a << 3) | (b << 6); }
      else if (d == 1) { x = a; y = hi ? 8 : -1; z = b; nl = a | ((hi ? 0 : 7) << 3) | (b << 6); }
      else { x = a; y = b; z = hi ? 8 : -1; nl = a | (b << 3) | ((hi ? 0 : 7) << 6); }
      unsigned long long v = kNoPar;
      if (ns >= 0) {
        const unsigned long long q = *(volatile const unsigned long long*)&p.par[(long long)ns * kBlockVox + nl];
        if (q != kNoPar) v = pack3(x + fld(q, 42), y + fld(q, 21), z + fld(q, 0));
      }
      cur[(x + 1) + 10 * (y + 1) + 100 * (z + 1)] = v;
    }
    __syncthreads();
    const int la = t & 7, lb = t >> 3;   // this thread's line: the two coordinates other than the swept one
    for (int round = 0; round < 16; ++round) {
      int changed = 0;
#pragma unroll 1
      for (int sw = 0; sw < 6; ++sw) {
        const int ax = sw >> 1, dir = (sw & 1) ? -1 : 1;
        const int stride = ax == 0 ? 1 : (ax == 1 ? 10 : 100);
        int x0, y0, z0;   // first voxel of the line in sweep order (local coords)
        if (ax == 0) { x0 = dir > 0 ? 0 : 7; y0 = la; z0 = lb; }
        else if (ax == 1) { x0 = la; y0 = dir > 0 ? 0 : 7; z0 = lb; }
        else { x0 = la; y0 = lb; z0 = dir > 0 ? 0 : 7; }
        int ci = (x0 + 1) + 10 * (y0 + 1) + 100 * (z0 + 1);
        unsigned long long carry = cur[ci - dir * stride];   // halo / previous voxel
        int x = x0, y = y0, z = z0;
        for (int st = 0; st < 8; ++st) {
          unsigned long long best = cur[ci];
          long long bd = best == kNoPar ? 0x7fffffffffffffffll : pd2(best, x, y, z);
          if (carry != kNoPar) {
            const long long d = pd2(carry, x, y, z);
            if (d < bd || (d == bd && carry < best)) { bd = d; best = carry; cur[ci] = best; changed = 1; }
          }
          carry = best;
          ci += dir * stride;
          if (ax == 0) x += dir; else if (ax == 1) y += dir; else z += dir;
        }
        __syncthreads();
      }
      if (!__syncthreads_or(changed)) break;
    }
    // write back; a changed face voxel queues the neighbour block across that face
    for (int l = t; l < 512; l += 64) {
      const int x = l & 7, y = (l >> 3) & 7, z = l >> 6;
      const unsigned long long b = cur[(x + 1) + 10 * (y + 1) + 100 * (z + 1)];
      const unsigned long long nq = b == kNoPar ? kNoPar : pack3(fld(b, 42) - x, fld(b, 21) - y, fld(b, 0) - z);
      unsigned long long* dst = &p.par[(long long)slot * kBlockVox + l];
      if (*dst != nq) {
        *dst = nq;
        if (x == 0) face_changed[0] = 1;
        if (x == 7) face_changed[1] = 1;
        if (y == 0) face_changed[2] = 1;
        if (y == 7) face_changed[3] = 1;
        if (z == 0) face_changed[4] = 1;
        if (z == 7) face_changed[5] = 1;
      }
    }
    __syncthreads();
    if (t < 6 && face_changed[t] && nb_slot[t] >= 0) p.active[nb_slot[t]] = 1;
  }
}

__global__ void inc_write(const __grid_constant__ IncParams p) {
  const long long n = (long long)p.nb * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    bool obs, neg;
    (void)is_site(p, i, obs, neg);
    float e;
    const unsigned long long q = p.par[i];
    if (!obs) e = __int_as_float(0x7fc00000);
    else if (q == kNoPar) e = __int_as_float(0x7f800000);
    else {
      const long long dx = fld(q, 42), dy = fld(q, 21), dz = fld(q, 0);
      const float m = (float)((double)p.s * sqrt((double)(dx * dx + dy * dy + dz * dz)));
      e = neg ? -m : m;
    }
    p.esdf[i] = e;
  }
}

}  // namespace

cudaError_t launch_update_esdf(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], cudaStream_t st,
                               int* iterations) {
  *iterations = 0;
  if (n_blocks <= 0) return cudaSuccess;
  cudaError_t e;
  const size_t mb = (size_t)sm->pool.max_blocks;
  if (!sm->inc.par) {
    if ((e = cudaMalloc(&sm->inc.par, mb * kBlockVox * 8)) != cudaSuccess ||
        (e = cudaMalloc(&sm->inc.sitebits, mb * 64)) != cudaSuccess ||
        (e = cudaMalloc(&sm->inc.active, mb * 4)) != cudaSuccess ||
        (e = cudaMalloc(&sm->inc.list, mb * 4)) != cudaSuccess ||
        (e = cudaMallocHost(&sm->inc.cnt_host, 4)) != cudaSuccess ||
        (e = cudaMalloc(&sm->inc.cnt, 4)) != cudaSuccess)
      return e;
    cudaMemsetAsync(sm->inc.active, 0, mb * 4, st);
    sm->inc.nb_prev = 0;
  }
  const int nbx = hi[0] - lo[0] + 1, nby = hi[1] - lo[1] + 1, nbz = hi[2] - lo[2] + 1;
  const long long nblk = (long long)nbx * nby * nbz;
  if (sm->block_grid_cap < nblk) {
    if (sm->block_grid) cudaFree(sm->block_grid);
    sm->block_grid = nullptr; sm->block_grid_cap = 0;
    if ((e = cudaMalloc(&sm->block_grid, sizeof(int) * (size_t)nblk)) != cudaSuccess) return e;
    sm->block_grid_cap = nblk;
  }
  // dense slot grid (the colmask / rowmask side outputs go to a scratch tail of the EDT buffer)
  const long long mask_bytes = (long long)nbx * nby + (long long)nby * nbz + 256;
  if (sm->edt_bytes < mask_bytes) {
    if (sm->edt) cudaFree(sm->edt);
    sm->edt = nullptr; sm->edt_bytes = 0;
    if ((e = cudaMalloc(&sm->edt, (size_t)mask_bytes)) != cudaSuccess) return e;
    sm->edt_bytes = mask_bytes;
  }
  unsigned char* colmask = reinterpret_cast<unsigned char*>(sm->edt);
  cudaMemsetAsync(sm->block_grid, 0xff, sizeof(int) * (size_t)nblk, st);
  {
    ProfScope ps_(sm, "inc_block_grid", st);
    block_grid_kernel<<<148 * 4, 256, 0, st>>>(sm->ctr, sm->pool.coords, sm->pool.max_blocks, sm->block_grid,
                                               colmask, colmask + (size_t)nbx * nby, lo[0], lo[1], lo[2], nbx, nby);
  }
  IncParams ip;
  ip.sums = sm->pool.sums; ip.esdf = sm->pool.esdf; ip.coords = sm->pool.coords; ip.par = sm->inc.par;
  ip.sitebits = sm->inc.sitebits; ip.active = sm->inc.active; ip.list = sm->inc.list; ip.cnt = sm->inc.cnt;
  ip.grid = sm->block_grid; ip.lo0 = lo[0]; ip.lo1 = lo[1]; ip.lo2 = lo[2]; ip.nbx = nbx; ip.nby = nby; ip.nbz = nbz;
  ip.nb = n_blocks; ip.nb_prev = std::min(sm->inc.nb_prev, n_blocks);
  ip.site_thr = sm->cfg.site_threshold; ip.s = (float)sm->cfg.voxel_size;
  {
    ProfScope ps_(sm, "inc_classify", st);
    inc_classify<<<148 * 8, 256, 0, st>>>(ip);
  }
  if (ip.nb_prev > 0) {
    ProfScope ps_(sm, "inc_invalidate", st);
    inc_invalidate<<<148 * 8, 256, 0, st>>>(ip);
  }
  // waves are launched in groups of kWaves between host checks of the queue: a wave whose queue is empty
  // costs two tiny launches (the propagate grid exits at once), a host round trip costs far more.
  // Each wave: propagate the queued blocks, then compact the blocks they queued into the next list.
  constexpr int kWaves = 8;
  const unsigned pgrid = (unsigned)std::min<long long>(n_blocks, 148ll * 32);
  auto compact = [&]() {
    cudaMemsetAsync(sm->inc.cnt, 0, 4, st);
    ProfScope ps_(sm, "inc_compact", st);
    inc_compact<<<(n_blocks + 255) / 256, 256, 0, st>>>(ip);
  };
  compact();
  cudaMemcpyAsync(sm->inc.cnt_host, sm->inc.cnt, 4, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  for (int group = 0; *sm->inc.cnt_host != 0 && group < 100000; ++group) {
    for (int w = 0; w < kWaves; ++w) {
      {
        ProfScope ps_(sm, "inc_propagate", st);
        inc_propagate<<<pgrid, 64, 0, st>>>(ip);
      }
      compact();
    }
    *iterations += kWaves;
    cudaMemcpyAsync(sm->inc.cnt_host, sm->inc.cnt, 4, cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  }
  {
    ProfScope ps_(sm, "inc_write", st);
    inc_write<<<148 * 8, 256, 0, st>>>(ip);
  }
  sm->inc.nb_prev = n_blocks;
  return cudaGetLastError();
}

}  // namespace cvx
