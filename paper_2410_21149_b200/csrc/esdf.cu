// esdf.cu — exact ESDF finalize and the incremental ESDF
// (row f1) for sm_100a.
//
// Finalize: PBA-class separable exact EDT over the dense AABB of the allocated blocks (O10-O12):
//   block_grid_kernel  slot index per block of the AABB (direct index, no hashing in the passes)
//   pass_x_kernel      one warp per x-row: reads the TSDF sums of the row's allocated voxels (coalesced),
//                      decides observed / sign / site S = {W > 0, |D| <= tau_site} with warp ballots and
//                      stores them as per-slot bit-planes (3 bits per voxel instead of a 4-byte E
//                      placeholder), and writes the exact 1-D distance to the nearest site along x (u16)
//                      from per-chunk bit masks (prefix max / suffix min scans across chunks).
//   pba_line_kernel    passes y and z: one CTA per tile of `tx` parallel lines (consecutive x, so every
//                      line position is one contiguous row segment) staged whole into shared memory by
//                      TMA (cp.async.bulk.tensor, one box per <= 256 positions, mbarrier completion).  Each
//                      line is cut into `nbands` bands (PBA's banding): every band builds the
//                      lower envelope of the parabolas f(q) + (p - q)^2 of its own sites over the whole
//                      line (Meijster / Felzenszwalb-Huttenlocher stack, kept in shared memory as an
//                      array in the band's own rows), the band envelopes are merged pairwise in log2(B)
//                      levels (the merge only touches the junction: it pops the left envelope's top and
//                      drops the right envelope's bottom while they are dominated — exactly the pushes
//                      the sequential algorithm would do), and every band then writes its own output
//                      range by walking the merged envelope.  Integer arithmetic throughout.
//                      Pass y writes the 2-D squared distance (u32, dense); pass z writes E = sign * s *
//                      sqrt(d^2) straight into the 8^3 ESDF blocks (NaN unobserved, +inf no sites).
//
// Incremental (f1, R11): the ESDF kept current while the submap is integrated is the exact EDT
// clamped at d_max = esdf_max_distance.  A site within d_max of a voxel is within r = ceil(d_max / s)
// voxels along every axis, so a site change can only move the (clamped) distance of blocks within
// Rb = ceil(r / 8) blocks of it.  Per update:
//   inc_classify   new bit-planes of every allocated block from the sums; a block whose site plane
//                  changed is a raise / lower source, a block whose planes changed at all (or is new)
//                  must be rewritten
//   inc_dilate     every block within Rb blocks of a source is queued ("Each region uses its own queue",
//                  one region = one block)
//   inc_window     one CTA per queued block: the exact clamped EDT of its 512 voxels from the site planes
//                  of the (2 Rb + 1)^3 blocks around it, by three separable passes in shared memory (bit
//                  scans along x, brute-force minima along y and z over the window) — the "axis
//                  direction" passes of P:L149, done once instead of iterated to a fixpoint.
//   Windows wider than 7^3 blocks fall back to the dense passes above with the clamp applied in pass z.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <type_traits>

#include "submap.h"

namespace cvx {
namespace {

constexpr unsigned kNone16 = 0xffffu;
constexpr unsigned kInf32 = 0xffffffffu;
constexpr long long kInfF = 1ll << 62;
constexpr int kPlaneWords = 48;   // per slot: observed[16] | negative[16] | site[16] (bit l = local index l)

// slot of every block of the AABB (-1 = not allocated) and, per (bx, by) column / (by, bz) row, whether
// any block of it is allocated (pass z skips empty columns: they hold no voxel to write)
__global__ void block_grid_kernel(const Counters* ctr, const int4* coords, int max_blocks, int* grid,
                                  unsigned char* colmask, unsigned char* rowmask, int lx, int ly, int lz, int nbx,
                                  int nby) {
  const int nb = min(ctr->n_blocks, max_blocks);
  for (int sIdx = blockIdx.x * blockDim.x + threadIdx.x; sIdx < nb; sIdx += gridDim.x * blockDim.x) {
    int4 c = coords[sIdx];
    grid[((long long)(c.z - lz) * nby + (c.y - ly)) * nbx + (c.x - lx)] = sIdx;
    if (colmask) colmask[(long long)(c.y - ly) * nbx + (c.x - lx)] = 1;
    if (rowmask) rowmask[(long long)(c.z - lz) * nby + (c.y - ly)] = 1;
  }
}

// O10 / R4: the site test on D rounded to fp32 (the value cvx_export_blocks returns), compared in fp64.
// Without the division where it cannot matter: with W > 0, sign(D) = sign(sum w d) (a non-zero quotient
// never rounds to zero in fp32 at these magnitudes), and |D| <= thr is decided by |sum w d| vs thr W
// unless they are within 2^-20 of each other (fp32 rounding of D and the fp64 products move them by less
// than 2^-23), where the exact rounded quotient decides.
__device__ __forceinline__ void classify_voxel(longlong2 sw, double thr, bool& obs, bool& neg, bool& site) {
  obs = sw.y > 0;
  neg = obs && sw.x < 0;
  site = false;
  if (obs) {
    const double a = fabs((double)sw.x), b = thr * (double)sw.y;
    if (a < b * (1.0 - 0x1p-20)) site = true;
    else if (a <= b * (1.0 + 0x1p-20)) {
      const float D = (float)((double)sw.x / (double)sw.y);
      site = fabs((double)D) <= thr;
    }
  }
}

struct XParams {
  const long long* sums;
  unsigned* planes;
  const int* grid;
  const unsigned char* rowmask;   // (by, bz) block rows with allocated blocks
  unsigned short* g1;
  int nx, ny, nz, nbx, nby;
  double site_thr;
  int max_blocks;
};

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

#ifndef CVX_XCH
#define CVX_XCH 4
#endif
constexpr int kXCh = CVX_XCH;   // chunks (32 voxels each) whose loads a warp issues together in pass x
#ifndef CVX_XPIPE
#define CVX_XPIPE 0             // pass x: 1 = cp.async ring of kXDepth chunks per warp instead of kXCh batches (measured: no gain)
#endif
#ifndef CVX_XDEPTH
#define CVX_XDEPTH 8
#endif
constexpr int kXDepth = CVX_XDEPTH;
// dynamic shared memory of pass_x_kernel: per warp msk / prv / nxt [nch], the CTA's plane bytes [3][nbx][4],
// then (CVX_XPIPE) per warp a ring of kXDepth chunks x 32 lanes x 16 bytes
__host__ __device__ inline size_t xring_off(int nch, int nbx) {
  return (((size_t)4 * 3 * nch * 4 + (size_t)3 * nbx * 4) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t xsmem_bytes(int nch, int nbx) {
  return xring_off(nch, nbx) + (CVX_XPIPE ? (size_t)4 * kXDepth * 32 * 16 : 0);
}

#ifdef CVX_PX_MINB
__global__ void __launch_bounds__(128, CVX_PX_MINB) pass_x_kernel(const __grid_constant__ XParams p) {
#else
__global__ void __launch_bounds__(128) pass_x_kernel(const __grid_constant__ XParams p) {
#endif
  extern __shared__ __align__(1024) unsigned char dsmem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (p.nx + 31) >> 5;
  unsigned* msk = reinterpret_cast<unsigned*>(dsmem) + warp * 3 * nch;
  int* prv = reinterpret_cast<int*>(msk + nch);
  int* nxt = prv + nch;
  // the CTA's 4 rows are 4 consecutive y of one z: byte (y & 3) of one plane word per block and plane, so
  // the planes are written as whole words (3 per block) once the 4 warps are done
  unsigned char* pb = reinterpret_cast<unsigned char*>(reinterpret_cast<unsigned*>(dsmem) + 4 * 3 * nch);
  const long long rows = (long long)p.ny * p.nz;   // a multiple of 8
  const int kNeg = -(1 << 30), kPos = 1 << 30;
  for (long long g = blockIdx.x; g * 4 < rows; g += gridDim.x) {
    const long long row = g * 4 + warp;
    const int y = (int)(row % p.ny), z = (int)(row / p.ny);
    if (!p.rowmask[(long long)(z >> 3) * p.nby + (y >> 3)]) {   // no block in these rows: no site, no voxel
      unsigned short* out = p.g1 + row * p.nx;
      for (int x = lane; x < p.nx; x += 32) out[x] = (unsigned short)kNone16;
      continue;
    }
    const int* grow = p.grid + ((long long)(z >> 3) * p.nby + (y >> 3)) * p.nbx;
    const int lyz = 8 * (y & 7) + 64 * (z & 7);
    // 1) sites of the row -> one 32-bit mask per chunk; the block's observed / sign / site plane bytes.
    //    kXCh chunks per round: their slot look-ups, then their TSDF loads, are issued back to back so
    //    every warp keeps kXCh 512-byte requests in flight (the row loop is otherwise latency-bound).
#if CVX_XPIPE
    // cp.async pipeline: the TSDF sums of chunk c + kXDepth are copied into this warp's shared ring while
    // chunk c is classified (the slot of the chunk after that is loaded one chunk ahead, in a register)
    {
      longlong2* ring = reinterpret_cast<longlong2*>(dsmem + xring_off(nch, p.nbx)) + warp * kXDepth * 32;
      auto slot_of = [&](int c) -> int {
        const int x = (c << 5) + lane;
        return (c < nch && x < p.nx) ? grow[x >> 3] : -1;
      };
      auto issue = [&](int c, int sl) {
        longlong2* dst = ring + (c % kXDepth) * 32 + lane;
        if (sl >= 0) {
          const longlong2* src = reinterpret_cast<const longlong2*>(p.sums) + (long long)sl * kBlockVox + (lane & 7) + lyz;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_addr(dst)), "l"(src) : "memory");
        } else {
          *dst = make_longlong2(0, 0);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      for (int c = 0; c < kXDepth; ++c) issue(c, slot_of(c));
      int nsl = slot_of(kXDepth);
      for (int c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;" :: "n"(kXDepth - 1) : "memory");
        const volatile long long* rv = reinterpret_cast<volatile long long*>(ring + (c % kXDepth) * 32 + lane);
        const longlong2 sw = make_longlong2(rv[0], rv[1]);
        const int sl = nsl;
        nsl = slot_of(c + kXDepth + 1);
        issue(c + kXDepth, sl);
        bool obs, neg, site;
        classify_voxel(sw, p.site_thr, obs, neg, site);
        const unsigned bs = __ballot_sync(0xffffffffu, site);
        const unsigned bo = __ballot_sync(0xffffffffu, obs);
        const unsigned bn = __ballot_sync(0xffffffffu, neg);
        if (lane == 0) msk[c] = bs;
        if ((lane & 7) == 0 && ((c << 5) + lane) < p.nx) {   // one lane per block: its row bytes
          const int blk = ((c << 5) + lane) >> 3;
          pb[(0 * p.nbx + blk) * 4 + (y & 3)] = (unsigned char)(bo >> lane);
          pb[(1 * p.nbx + blk) * 4 + (y & 3)] = (unsigned char)(bn >> lane);
          pb[(2 * p.nbx + blk) * 4 + (y & 3)] = (unsigned char)(bs >> lane);
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
#else
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
        bool obs, neg, site;
        classify_voxel(sw[u], p.site_thr, obs, neg, site);
        const unsigned bs = __ballot_sync(0xffffffffu, site);
        const unsigned bo = __ballot_sync(0xffffffffu, obs);
        const unsigned bn = __ballot_sync(0xffffffffu, neg);
        if (lane == 0 && c0 + u < nch) msk[c0 + u] = bs;
        if ((lane & 7) == 0 && (((c0 + u) << 5) + lane) < p.nx) {   // one lane per block: its row bytes
          const int blk = (((c0 + u) << 5) + lane) >> 3;
          pb[(0 * p.nbx + blk) * 4 + (y & 3)] = (unsigned char)(bo >> lane);
          pb[(1 * p.nbx + blk) * 4 + (y & 3)] = (unsigned char)(bn >> lane);
          pb[(2 * p.nbx + blk) * 4 + (y & 3)] = (unsigned char)(bs >> lane);
        }
      }
    }
#endif
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
    CVX_CHECK(row < (long long)p.ny * p.nz, "pass x row");
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
    __syncthreads();
    const int w = ((y & 7) >> 2) + 2 * (z & 7);   // plane word of rows (y & ~3 .. + 3, z)
    for (int i = threadIdx.x; i < 3 * p.nbx; i += blockDim.x) {
      const int pl = i / p.nbx, blk = i % p.nbx;
      const int slot = grow[blk];
      CVX_CHECK(slot < p.max_blocks, "pass x plane slot");
      if (slot >= 0) p.planes[(long long)slot * kPlaneWords + 16 * pl + w] = reinterpret_cast<const unsigned*>(pb)[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ TMA / mbarrier helpers
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile("{\n\t.reg .pred p;\n"
               "WAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra WAIT_%=;\n\t}" :: "r"(smem_addr(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(smem_addr(dst)), "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2),
                  "r"(smem_addr(bar)) : "memory");
}

// floor(num / den) for den > 0, |num| <= 2^35, den <= 2^17: the correctly rounded fp64 quotient is
// within half an ulp (<= 2^-18) of num/den, whose fractional part is 0 or >= 1/den >= 2^-17 away from
// the next integer, so its floor is the exact integer floor.
__device__ __forceinline__ long long floordiv_exact(long long num, long long den) {
  return (long long)floor((double)num / (double)den);
}

struct PbaParams {
  unsigned* g2;                   // pass y output: 2-D squared distances (u32, x-fastest dense AABB)
  float* esdf;                    // pass z output: ESDF blocks
  const int* grid;                // dense slot grid over the AABB
  const unsigned char* colmask;   // (bx, by) columns with allocated blocks
  const unsigned* planes;         // per-slot observed / negative / site bit-planes (pass x)
  int nx, ny, nz, nbx, nby;
  int m;                          // line length (ny for pass y, nz for pass z)
  int tx;                         // lines per tile (consecutive x)
  int nbands, lb;                 // bands per line (power of two <= 32) and band length
  int rows;                       // staged positions per line (nbox * box_h >= m)
  int box_h, nbox;                // TMA box height and boxes per tile
  int tiles_x;
  double s;
  int capped;                     // f1 fallback: E clamped at dmax
  double dmax;
};

// Shared memory of one tile ([row][line] arrays, line fastest):
//   fb   [rows][tx]  f per position (TMA destination; pass z reuses it for the output d^2 after the hulls)
//   hq   [rows][tx]  u16 hull sites of band b in rows [b lb, b lb + nh)
//   hf   [rows][tx]  u32 their f (pass z only; pass y re-reads the u16 input)
//   nh, hmin [nbands][tx]  hull size and min f of every band; then the mbarrier.
template <bool kZ>
__host__ __device__ inline size_t pba_smem_bytes(int rows, int tx, int nbands) {
  const size_t esize = kZ ? 4 : 2;
  size_t b = (size_t)rows * tx * (esize + 2 + (kZ ? 4 : 0)) + (size_t)nbands * tx * 8;
  return ((b + 15) & ~(size_t)15) + 16;
}

// One band hull = the lower envelope over the whole real line of the parabolas (p - q)^2 + f(q) of the
// band's sites q (equivalently the lower convex hull of the points (q, q^2 + f(q))), built by Andrew's
// monotone chain; a pointer walks it as p increases (the optimal hull element is non-decreasing in p).
struct HullPtr {
  int k, end;                // current element row, one past the last row
  long long q, f;            // current site and its f
};

template <bool kZ>
__global__ void __launch_bounds__(256) pba_line_kernel(const __grid_constant__ CUtensorMap tmap,
                                                       const __grid_constant__ PbaParams p) {
  using Elem = typename std::conditional<kZ, unsigned, unsigned short>::type;
  extern __shared__ __align__(1024) unsigned char dsmem[];
  const int tx = p.tx, B = p.nbands, m = p.m, rows = p.rows, lb = p.lb;
  Elem* fb = reinterpret_cast<Elem*>(dsmem);
  unsigned short* hq = reinterpret_cast<unsigned short*>(dsmem + (size_t)rows * tx * sizeof(Elem));
  unsigned* hf = reinterpret_cast<unsigned*>(hq + (size_t)rows * tx);                  // pass z only
  unsigned short* nhv = reinterpret_cast<unsigned short*>(kZ ? (unsigned char*)(hf + (size_t)rows * tx)
                                                             : (unsigned char*)(hq + (size_t)rows * tx));
  unsigned* hminv = reinterpret_cast<unsigned*>(nhv + B * tx + (B * tx & 1));
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(dsmem + pba_smem_bytes<kZ>(rows, tx, B) - 16);

  const int xt = blockIdx.x % p.tiles_x, o2 = blockIdx.x / p.tiles_x;   // o2: z (pass y) or y (pass z)
  const int x0 = xt * tx;
  const int xend = min(p.nx, x0 + tx);
  if (kZ) {   // a tile whose columns hold no allocated block has no voxel to write
    bool any = false;
    for (int bx = x0 >> 3; bx < (xend + 7) >> 3; ++bx) any |= p.colmask[(long long)(o2 >> 3) * p.nbx + bx] != 0;
    if (!any) return;
  }
  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(mbar, (unsigned)((size_t)rows * tx * sizeof(Elem)));
    for (int k = 0; k < p.nbox; ++k) {
      Elem* dst = fb + (size_t)k * p.box_h * tx;
      if (kZ) tma_load_3d(dst, &tmap, x0, o2, k * p.box_h, mbar);
      else tma_load_3d(dst, &tmap, x0, k * p.box_h, o2, mbar);
    }
  }
  const int xl = threadIdx.x % tx, b = threadIdx.x / tx;
  const bool valid = x0 + xl < p.nx;
  const int q0 = b * lb, q1 = min(m, q0 + lb);
  auto Fin = [&](int q) -> long long {         // f of position q from the staged input
    const Elem v = fb[(size_t)q * tx + xl];
    if (kZ) return v == kInf32 ? kInfF : (long long)v;
    return v == kNone16 ? kInfF : (long long)v * v;
  };
  auto HQ = [&](int r) -> unsigned short& { return hq[(size_t)r * tx + xl]; };
  auto HF = [&](int r) -> long long {          // f of the hull element in row r
    if (kZ) return (long long)hf[(size_t)r * tx + xl];
    return Fin(hq[(size_t)r * tx + xl]);
  };
  mbar_wait(mbar, 0);

  // ---- 1) band hulls (Andrew's monotone chain on (q, q^2 + f)); a middle point on or above the chord
  //         of its neighbours never gives a strictly smaller value and is dropped
  if (valid) {
    int n = 0;
    long long qa = 0, ga = 0, qb = 0, gb = 0;   // the last two hull points
    unsigned minf = kInf32;
    for (int q = q0; q < q1; ++q) {
      const long long fq = Fin(q);
      if (fq >= kInfF) continue;
      const long long gq = (long long)q * q + fq;
      while (n >= 2 && (gb - ga) * (q - qa) >= (gq - ga) * (qb - qa)) {
        --n;
        qb = qa; gb = ga;
        if (n >= 2) { qa = HQ(q0 + n - 2); ga = qa * qa + HF(q0 + n - 2); }
      }
      HQ(q0 + n) = (unsigned short)q;
      if (kZ) hf[(size_t)(q0 + n) * tx + xl] = (unsigned)fq;
      ++n;
      qa = qb; ga = gb; qb = q; gb = gq;
      if (fq < minf) minf = (unsigned)fq;
    }
    nhv[b * tx + xl] = (unsigned short)n;
    hminv[b * tx + xl] = minf;
  }
  __syncthreads();
  if (!valid || q0 >= m) return;

  // ---- 2) outputs of [q0, q1): min over the hulls of bands b-1, b, b+1 (pointer walks), then every
  //         other band whose lower bound gap^2 + min f is below the current maximum over the range
  auto start = [&](HullPtr& h, int c, int p0) {   // element of band c's hull optimal at p0
    const int r0 = c * lb, n = nhv[c * tx + xl];
    h.end = r0 + n;
    if (n == 0) { h.k = h.end; return; }
    if (c < b) {   // positions right of the band: walk back from the last element (optimum near the end)
      h.k = h.end - 1; h.q = HQ(h.k); h.f = HF(h.k);
      while (h.k > r0) {
        const long long q2 = HQ(h.k - 1), f2 = HF(h.k - 1);
        if ((p0 - q2) * (p0 - q2) + f2 > (p0 - h.q) * (p0 - h.q) + h.f) break;
        --h.k; h.q = q2; h.f = f2;
      }
    } else {
      h.k = r0; h.q = HQ(r0); h.f = HF(r0);
    }
  };
  auto value = [&](HullPtr& h, int pp) -> long long {   // advance to pp, return the hull's value there
    if (h.k >= h.end) return kInfF;
    long long d = pp - h.q, v = d * d + h.f;
    while (h.k + 1 < h.end) {
      const long long q2 = HQ(h.k + 1), f2 = HF(h.k + 1), d2 = pp - q2, v2 = d2 * d2 + f2;
      if (v2 >= v) break;
      ++h.k; h.q = q2; h.f = f2; v = v2;
    }
    return v;
  };
  const int x = x0 + xl;
  HullPtr w0, w1, w2;
  start(w0, max(b - 1, 0), q0);
  if (b == 0) w0.k = w0.end;
  start(w1, b, q0);
  start(w2, min(b + 1, B - 1), q0);
  if (b == B - 1) w2.k = w2.end;
  long long U = 0;
  unsigned* d2buf = reinterpret_cast<unsigned*>(fb);   // pass z: the input is no longer read
  for (int pp = q0; pp < q1; ++pp) {
    const long long v = min(value(w1, pp), min(value(w0, pp), value(w2, pp)));
    U = max(U, v);
    const unsigned o = v >= kInfF ? kInf32 : (unsigned)v;
    if (!kZ) {
      if (p.colmask[(long long)(pp >> 3) * p.nbx + (x >> 3)])   // only columns pass z will read
        p.g2[((long long)o2 * p.ny + pp) * p.nx + x] = o;
    } else {
      d2buf[(size_t)pp * tx + xl] = o;
    }
  }
  // far bands, nearest first; each one that can still win somewhere is swept into the outputs
  for (int dist = 2; dist < B && U > 0; ++dist) {
    for (int side = 0; side < 2; ++side) {
      const int c = side ? b + dist : b - dist;
      if (c < 0 || c >= B || nhv[c * tx + xl] == 0) continue;
      const long long gap = side ? (long long)c * lb - (q1 - 1) : (long long)q0 - (c * lb + lb - 1);
      if (gap * gap + (long long)hminv[c * tx + xl] >= U) continue;
      HullPtr h;
      start(h, c, q0);
      long long U2 = 0;
      for (int pp = q0; pp < q1; ++pp) {
        const long long v = value(h, pp);
        if (!kZ) {
          if (!p.colmask[(long long)(pp >> 3) * p.nbx + (x >> 3)]) continue;
          unsigned* o = p.g2 + ((long long)o2 * p.ny + pp) * p.nx + x;
          const long long cur = *o == kInf32 ? kInfF : (long long)*o;
          if (v < cur) *o = (unsigned)v;
          U2 = max(U2, min(v, cur));
        } else {
          unsigned& o = d2buf[(size_t)pp * tx + xl];
          const long long cur = o == kInf32 ? kInfF : (long long)o;
          if (v < cur) o = (unsigned)v;
          U2 = max(U2, min(v, cur));
        }
      }
      U = U2;
    }
  }
  if (!kZ) return;
  // ---- 3) pass z: E = sign(D) s sqrt(d^2) into the allocated blocks of this line
  int slot = -1, slot_bz = -1;
  for (int pp = q0; pp < q1; ++pp) {
    if ((pp >> 3) != slot_bz) {
      slot_bz = pp >> 3;
      slot = p.grid[((long long)slot_bz * p.nby + (o2 >> 3)) * p.nbx + (x >> 3)];
    }
    if (slot < 0) continue;
    const unsigned dd = d2buf[(size_t)pp * tx + xl];
    const int l = (x & 7) + 8 * (o2 & 7) + 64 * (pp & 7);
    const unsigned* pl = p.planes + (long long)slot * kPlaneWords;
    const bool obs = (pl[l >> 5] >> (l & 31)) & 1u, neg = (pl[16 + (l >> 5)] >> (l & 31)) & 1u;
    float e;
    if (!obs) e = __int_as_float(0x7fc00000);                           // unobserved -> NaN (O11)
    else if (p.capped) {
      const double md = dd == kInf32 ? p.dmax : fmin(p.s * sqrt((double)dd), p.dmax);
      e = (float)(neg ? -md : md);
    } else if (dd == kInf32) e = __int_as_float(0x7f800000);            // S empty -> +inf (O11)
    else {
      const double md = p.s * sqrt((double)dd);
      e = (float)(neg ? -md : md);
    }
    p.esdf[(long long)slot * kBlockVox + l] = e;
  }
}

// Passes y / z, streaming variant (CVX_EDT_KERNEL=0): one thread per line (consecutive x in a warp ->
// coalesced row reads), Meijster's lower envelope with the stack kept in place in global memory as
// per-position links (PBA's proximate sites at their own positions): pass y stores u32 {t: 16, prev: 16}
// per pushed position and re-reads f, pass z stores the full state below (u64 {f: 32, t: 16, prev: 16})
// so a pop is one load.  Same outputs as pba_line_kernel.
struct LinkParams {
  const unsigned char* rowmask;   // ring kernel, pass y: (by, bz) block rows with allocated blocks
  const void* fin;                // pass y: u16 1-D distances; pass z: u32 squared distances
  unsigned* g2;                   // pass y output
  void* meta;                     // stack links (8 bytes per AABB voxel)
  float* esdf;
  const int* grid;
  const unsigned char* colmask;
  const unsigned* planes;
  int nx, ny, nz, nbx, nby;
  double s;
  int capped;
  double dmax;
};

template <bool kZ>
__global__ void __launch_bounds__(256) link_line_kernel(const __grid_constant__ LinkParams p) {
  const long long nlines = kZ ? (long long)p.nx * p.ny : (long long)p.nx * p.nz;
  const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= nlines) return;
  const int x = (int)(line % p.nx);
  const int o2 = (int)(line / p.nx);      // pass y: z ; pass z: y
  const int m = kZ ? p.nz : p.ny;
  const long long stride = kZ ? (long long)p.nx * p.ny : (long long)p.nx;
  const long long base = kZ ? (long long)o2 * p.nx + x : (long long)o2 * p.nx * p.ny + x;
  if (kZ && !p.colmask[(long long)(o2 >> 3) * p.nbx + (x >> 3)]) return;   // no allocated voxel in this line
  auto f_at = [&](int q) -> long long {
    if (kZ) {
      const unsigned v = static_cast<const unsigned*>(p.fin)[base + q * stride];
      return v == kInf32 ? kInfF : (long long)v;
    }
    const unsigned v = static_cast<const unsigned short*>(p.fin)[base + q * stride];
    return v == kNone16 ? kInfF : (long long)v * v;
  };
  unsigned* m32 = static_cast<unsigned*>(p.meta);
  unsigned long long* m64 = static_cast<unsigned long long*>(p.meta);
  int top = -1, t_top = 0;
  long long f_top = 0;
  for (int q0 = 0; q0 < m; q0 += 8) {     // 8 independent loads in flight per thread
    long long fv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) fv[u] = q0 + u < m ? f_at(q0 + u) : kInfF;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u;
      const long long fq = fv[u];
      if (fq >= kInfF) continue;
      while (top >= 0) {
        const long long a = t_top - top, c = t_top - q;
        if (a * a + f_top > c * c + fq) {                 // q beats top already at top's start: pop
          if (kZ) {
            const unsigned long long mt = m64[base + (long long)top * stride];
            const int pr = (int)(mt & 0xffffu);
            if (pr == 0xffff) { top = -1; break; }
            top = pr; t_top = (int)((mt >> 16) & 0xffffu); f_top = (long long)(mt >> 32);
          } else {
            const int pr = (int)(m32[base + (long long)top * stride] & 0xffffu);
            if (pr == 0xffff) { top = -1; break; }
            top = pr;
            t_top = (int)(m32[base + (long long)top * stride] >> 16);
            f_top = f_at(top);
          }
        } else {
          break;
        }
      }
      int tq = 0;
      if (top >= 0) {
        const long long sep = floordiv_exact((long long)q * q - (long long)top * top + fq - f_top, 2ll * (q - top));
        if (sep + 1 >= m) continue;                        // q never wins inside the line
        tq = (int)(sep + 1);
      }
      if (kZ)
        m64[base + (long long)q * stride] = top < 0 ? 0xffffull
            : ((unsigned long long)f_top << 32) | ((unsigned long long)t_top << 16) | (unsigned long long)top;
      else
        m32[base + (long long)q * stride] = ((unsigned)tq << 16) | (unsigned)(top < 0 ? 0xffff : top);
      top = q; t_top = tq; f_top = fq;
    }
  }
  // backward: read the envelope from the right, one 8-position chunk (one block along the line) at a time
  for (int q0 = ((m - 1) >> 3) << 3; q0 >= 0; q0 -= 8) {
    int slot = -1;
    unsigned obsw = 0, negw = 0;   // pass z: bit u = observed / negative of position q0 + u (prefetched)
    const int lb = (x & 7) + 8 * (o2 & 7);
    if (kZ) {
      slot = p.grid[((long long)(q0 >> 3) * p.nby + (o2 >> 3)) * p.nbx + (x >> 3)];
      if (slot >= 0) {
        const unsigned* pl = p.planes + (long long)slot * kPlaneWords + (lb >> 5);
        unsigned ow[8], nw[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { ow[u] = pl[2 * u]; nw[u] = pl[16 + 2 * u]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { obsw |= ((ow[u] >> (lb & 31)) & 1u) << u; negw |= ((nw[u] >> (lb & 31)) & 1u) << u; }
      }
    }
    const bool wy = !kZ && p.colmask[(long long)(q0 >> 3) * p.nbx + (x >> 3)];
#pragma unroll
    for (int u = 7; u >= 0; --u) {
      const int q = q0 + u;
      if (q >= m) continue;
      long long d2 = kInfF;
      if (top >= 0) { const long long dq = q - top; d2 = dq * dq + f_top; }
      if (!kZ) {
        if (wy) p.g2[base + (long long)q * stride] = d2 >= kInfF ? kInf32 : (unsigned)d2;
      } else if (slot >= 0) {
        const int l = lb + 64 * u;
        const bool obs = (obsw >> u) & 1u, neg = (negw >> u) & 1u;
        float e;
        if (!obs) e = __int_as_float(0x7fc00000);
        else if (p.capped) {
          const double md = d2 >= kInfF ? p.dmax : fmin(p.s * sqrt((double)d2), p.dmax);
          e = (float)(neg ? -md : md);
        } else if (d2 >= kInfF) e = __int_as_float(0x7f800000);
        else {
          const double md = p.s * sqrt((double)d2);
          e = (float)(neg ? -md : md);
        }
        p.esdf[(long long)slot * kBlockVox + l] = e;
      }
      if (top >= 0 && q == t_top) {
        if (kZ) {
          const unsigned long long mt = m64[base + (long long)top * stride];
          const int pr = (int)(mt & 0xffffu);
          if (pr == 0xffff) top = -1;
          else { top = pr; t_top = (int)((mt >> 16) & 0xffffu); f_top = (long long)(mt >> 32); }
        } else {
          const int pr = (int)(m32[base + (long long)top * stride] & 0xffffu);
          if (pr == 0xffff) top = -1;
          else { top = pr; t_top = (int)(m32[base + (long long)top * stride] >> 16); f_top = f_at(top); }
        }
      }
    }
  }
}

// Passes y / z, ring variant (default when every quantity fits 24 bits, see ring_fits): one thread per
// line as above, but Meijster's stack is an explicit array per line in HBM ([line][k], contiguous per
// thread) whose top kRing entries live in a shared-memory ring:
//   * entries {f: 32, t: 16, s: 16} (site s, start t of its interval, f(s)); pops read the ring only
//     (a pop below the ring's window refills it from the array: rare);
//   * an entry is written to HBM only when a push displaces it from the ring (it has survived kRing
//     later pushes), so entries popped while young never leave the SM;
//   * the backward sweep takes the entries still in the ring, then the older ones from the array with
//     cp.async kAhead entries ahead into their ring slots (no dependent load chain);
//   * 32-bit arithmetic: with m^2 + max f < 2^24 every separator numerator is exact in fp32, and
//     floor(num / den) = the fp32 reciprocal estimate corrected by the exact integer remainder.
// Same outputs as link_line_kernel / pba_line_kernel (bit for bit: the envelope is unique and the
// output is its value).
#ifndef CVX_RING_MINB
#define CVX_RING_MINB 7
#endif
#ifndef CVX_RING_BPF
#define CVX_RING_BPF 1      // backward: masks / planes of the next chunk loaded one chunk ahead
#endif
#ifndef CVX_RING_EFAST
#define CVX_RING_EFAST 0    // 1: E = (float)(s sqrt(d2)) by an fp32 root refined in fp64 (esdf_value; measured slower)
#endif
#ifndef CVX_RING_BUNROLL
#define CVX_RING_BUNROLL 1  // unroll of the backward sweep over the 8 positions of a chunk (1 measured best: code size)
#endif
constexpr int kRingBUnroll = CVX_RING_BUNROLL;
#ifndef CVX_RING_BSKIP
#define CVX_RING_BSKIP 0    // 1: backward of pass z skips chunks no lane of the warp writes (measured: no gain; pass y slower)
#endif
#ifndef CVX_RING_INFSKIP
#define CVX_RING_INFSKIP 0  // 1: a batch of 8 positions without any site is skipped as a whole (per lane)
#endif
#ifndef CVX_RING_ROWSKIP
#define CVX_RING_ROWSKIP 1  // pass y: skip the y batches of block rows without allocated blocks
#endif
#ifndef CVX_RING_FSMEM
#define CVX_RING_FSMEM 0    // 1: the forward batch goes through shared memory (rolled loop, smaller code)
#endif
constexpr int kRing = 16, kAhead = 12, kRingThreads = 128;

__device__ __forceinline__ float rcp_approx32(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__device__ __forceinline__ int floordiv24(int num, int den) {   // den in [2, 2^17], |num| < 2^24
  int q = __float2int_rd((float)num * rcp_approx32((float)den));
  int r = num - q * den;
  while (r < 0) { --q; r += den; }
  while (r >= den) { ++q; r -= den; }
  return q;
}

// (float)(s * sqrt(d2)) correctly rounded as in fp64 (O11, the value the oracle computes), d2 < 2^24: an
// fp32 square root refined once in fp64 (relative error < 2^-44), rounded to fp32; only when the fp64
// value lies within 2^-40 (relative) of an fp32 rounding boundary is the IEEE fp64 sqrt taken.
[[maybe_unused]] __device__ __forceinline__ float esdf_value(double s, unsigned d2) {
  const float df = (float)d2;                               // exact (< 2^24)
  const float r = sqrtf(df);                                // |r - sqrt(d2)| <= ~1 ulp (fp32)
  if (r == 0.f) return 0.f;
  const double rd = (double)r;
  const double y = rd + ((double)d2 - rd * rd) * (0.5 / rd);   // one Newton step: error ~ 2^-46 relative
  const double v = s * y;
  const float lo = (float)(v * (1.0 - 0x1p-40)), hi = (float)(v * (1.0 + 0x1p-40));
  if (lo == hi) return lo;
  return (float)(s * sqrt((double)d2));
}

template <bool kZ>
__global__ void __launch_bounds__(kRingThreads, CVX_RING_MINB) ring_line_kernel(const __grid_constant__ LinkParams p) {
  __shared__ unsigned long long ring[kRing][kRingThreads];
  const long long nlines = kZ ? (long long)p.nx * p.ny : (long long)p.nx * p.nz;
  const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= nlines) return;
  const int x = (int)(line % p.nx);
  const int o2 = (int)(line / p.nx);      // pass y: z ; pass z: y
  const int m = kZ ? p.nz : p.ny;
  const long long stride = kZ ? (long long)p.nx * p.ny : (long long)p.nx;
  const long long base = kZ ? (long long)o2 * p.nx + x : (long long)o2 * p.nx * p.ny + x;
  if (kZ && !p.colmask[(long long)(o2 >> 3) * p.nbx + (x >> 3)]) return;   // no allocated voxel in this line
  unsigned long long* const gst = static_cast<unsigned long long*>(p.meta) + line * m;
  unsigned long long* const rg = &ring[0][threadIdx.x];   // ring slot j of this thread: rg[j * kRingThreads]
  // raw input (pass y: u16 1-D distance, pass z: u32 squared distance) and its f (kInf32 = no site)
  auto raw_at = [&](int q) -> unsigned {
    if (kZ) return static_cast<const unsigned*>(p.fin)[base + q * stride];
    return static_cast<const unsigned short*>(p.fin)[base + q * stride];
  };
  auto f_of = [](unsigned v) -> unsigned { return kZ ? v : (v == kNone16 ? kInf32 : v * v); };
  int k = -1, lo = 0;                      // stack [0, k]; indices < lo valid in gst, [lo, k] in the ring
  int s_top = 0, t_top = 0;
  unsigned f_top = 0;
  // forward (m is a multiple of 8): the loads of batch q0 + 8 are issued before batch q0 is consumed
  // pass y: an x-row block row (by, bz) without allocated blocks has no site, so f = inf on its 8 y
  // positions: such batches are neither loaded nor scanned (sparse AABBs: LiDAR / MAV submaps)
  auto row_has = [&](int q) -> bool {
    return kZ || !CVX_RING_ROWSKIP || p.rowmask[(long long)(o2 >> 3) * p.nby + (q >> 3)] != 0;
  };
  unsigned fa[8];
  bool ha = row_has(0);
#pragma unroll
  for (int u = 0; u < 8; ++u) fa[u] = ha ? raw_at(u) : kNone16;
#if CVX_RING_FSMEM
  __shared__ unsigned fsm[8][kRingThreads];
#endif
  for (int q0 = 0; q0 < m; q0 += 8) {
    unsigned fb[8];
    const int qn = q0 + 8 < m ? q0 + 8 : q0;
    const bool hb = row_has(qn);
#pragma unroll
    for (int u = 0; u < 8; ++u) fb[u] = hb ? raw_at(qn + u) : kNone16;
    bool skip = !ha;
#if CVX_RING_INFSKIP
    {   // the 8 positions of the batch hold no site of this line (raw all-ones = none / inf)
      unsigned a = fa[0];
#pragma unroll
      for (int u = 1; u < 8; ++u) a &= fa[u];
      skip |= a == (kZ ? kInf32 : kNone16);
    }
#endif
    if (skip) {
#pragma unroll
      for (int u = 0; u < 8; ++u) fa[u] = fb[u];
      ha = hb;
      continue;
    }
#if CVX_RING_FSMEM
#pragma unroll
    for (int u = 0; u < 8; ++u) fsm[u][threadIdx.x] = fa[u];
#pragma unroll 1
#else
#pragma unroll
#endif
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u;
#if CVX_RING_FSMEM
      const unsigned fq = f_of(fsm[u][threadIdx.x]);
#else
      const unsigned fq = f_of(fa[u]);
#endif
      if (fq == kInf32) continue;
      while (k >= 0) {
        const int a = t_top - s_top, c = t_top - q;
        if ((unsigned)(a * a) + f_top <= (unsigned)(c * c) + fq) break;   // q does not beat top at top's start
        if (--k < 0) break;
        if (k < lo) {                      // below the ring's window: refill kRing entries from the array
          const int j0 = max(0, k - (kRing - 1));
          CVX_CHECK(j0 >= 0 && k < lo && k < m, "ring refill range");
          for (int j = j0; j <= k; ++j) rg[(j & (kRing - 1)) * kRingThreads] = gst[j];
          lo = j0;
        }
        const unsigned long long e = rg[(k & (kRing - 1)) * kRingThreads];
        s_top = (int)(e & 0xffffu); t_top = (int)((e >> 16) & 0xffffu); f_top = (unsigned)(e >> 32);
      }
      int tq = 0;
      if (k >= 0) {
        const int sep = floordiv24(q * q - s_top * s_top + (int)fq - (int)f_top, 2 * (q - s_top));
        if (sep + 1 >= m) continue;        // q never wins inside the line
        tq = sep + 1;
      }
      ++k;
      unsigned long long* slot = rg + (k & (kRing - 1)) * kRingThreads;
      CVX_CHECK(k < m, "ring stack depth <= line length");
      if (k - kRing >= lo) { gst[k - kRing] = *slot; lo = k - kRing + 1; }   // displaced: write back
      *slot = ((unsigned long long)fq << 32) | ((unsigned)tq << 16) | (unsigned)q;
      s_top = q; t_top = tq; f_top = fq;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) fa[u] = fb[u];
    ha = hb;
  }
  // backward: the entries below the top in decreasing index order; entry j < lo is copied into its ring
  // slot by cp.async kAhead pops before it is needed (one commit group per pop, empty when j >= lo)
  auto issue = [&](int j) {
    if (j >= 0 && j < lo) {
      const unsigned sa = smem_addr(rg + (j & (kRing - 1)) * kRingThreads);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa), "l"(gst + j) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (k >= 0) {
#pragma unroll 1
    for (int i = 1; i <= kAhead; ++i) issue(k - i);
  }
  const int lb = (x & 7) + 8 * (o2 & 7);
  // per 8-position chunk: pass y whether its block column holds an allocated block; pass z the block's
  // slot and this column's observed / negative plane words (8 each).  Loaded one chunk ahead.
  auto chunk_slot = [&](int c0) -> int {
    if (c0 < 0) return -1;
    if (kZ) return p.grid[((long long)(c0 >> 3) * p.nby + (o2 >> 3)) * p.nbx + (x >> 3)];
    return p.colmask[(long long)(c0 >> 3) * p.nbx + (x >> 3)] ? 0 : -1;
  };
  unsigned ow[8], nw[8];
  auto load_planes = [&](int sl) {
    if (kZ && sl >= 0) {
      const unsigned* pl = p.planes + (long long)sl * kPlaneWords + (lb >> 5);
#pragma unroll
      for (int u = 0; u < 8; ++u) { ow[u] = pl[2 * u]; nw[u] = pl[16 + 2 * u]; }
    }
  };
  const int qlast = ((m - 1) >> 3) << 3;
#if CVX_RING_BPF
  int slot = chunk_slot(qlast);
  load_planes(slot);
  int nslot = chunk_slot(qlast - 8);
#endif
  for (int q0 = qlast; q0 >= 0; q0 -= 8) {
    unsigned obsw = 0, negw = 0;   // pass z: bit u = observed / negative of position q0 + u
#if !CVX_RING_BPF
    const int slot = chunk_slot(q0);
    load_planes(slot);
#endif
    if (kZ && slot >= 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) { obsw |= ((ow[u] >> (lb & 31)) & 1u) << u; negw |= ((nw[u] >> (lb & 31)) & 1u) << u; }
    }
    const int cur = slot;
#if CVX_RING_BPF
    slot = nslot;
    load_planes(slot);                     // chunk q0 - 8
    nslot = chunk_slot(q0 - 16);
#endif
#if CVX_RING_BSKIP
    if (kZ && __all_sync(__activemask(), cur < 0)) {   // no lane writes this chunk: only its pops (t strictly
      while (k >= 0 && t_top >= q0) {            // decreases down the stack)
        if (--k >= 0) {
          if (k < lo) asm volatile("cp.async.wait_group %0;" :: "n"(kAhead - 1) : "memory");
          const unsigned long long e = *(volatile unsigned long long*)(rg + (k & (kRing - 1)) * kRingThreads);
          s_top = (int)(e & 0xffffu); t_top = (int)((e >> 16) & 0xffffu); f_top = (unsigned)(e >> 32);
          issue(k - kAhead);
        }
      }
      continue;
    }
#endif
#pragma unroll kRingBUnroll
    for (int u = 7; u >= 0; --u) {
      const int q = q0 + u;
      unsigned d2 = kInf32;
      if (k >= 0) { const int dq = q - s_top; d2 = (unsigned)(dq * dq) + f_top; }
      CVX_CHECK(base + (long long)q * stride < (long long)p.nx * p.ny * p.nz, "line pass output index");
      if (!kZ) {
        if (cur >= 0) p.g2[base + (long long)q * stride] = d2;
      } else if (cur >= 0) {
        const bool obs = (obsw >> u) & 1u, neg = (negw >> u) & 1u;
        float e;
        if (!obs) e = __int_as_float(0x7fc00000);
        else if (d2 == kInf32) e = p.capped ? (float)(neg ? -p.dmax : p.dmax) : __int_as_float(0x7f800000);
        else {
#if CVX_RING_EFAST
          e = esdf_value(p.s, d2);
#else
          e = (float)(p.s * sqrt((double)d2));
#endif
          if (p.capped && (double)e > p.dmax) e = (float)p.dmax;
          if (neg) e = -e;
        }
        p.esdf[(long long)cur * kBlockVox + lb + 64 * u] = e;
      }
      if (k >= 0 && q == t_top) {          // pop: the entry below takes over left of t_top
        if (--k >= 0) {
          if (k < lo) asm volatile("cp.async.wait_group %0;" :: "n"(kAhead - 1) : "memory");
          const unsigned long long e = *(volatile unsigned long long*)(rg + (k & (kRing - 1)) * kRingThreads);
          s_top = (int)(e & 0xffffu); t_top = (int)((e >> 16) & 0xffffu); f_top = (unsigned)(e >> 32);
          issue(k - kAhead);
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Pass y with two threads per line, for AABBs with few long y lines (LiDAR / MAV submaps: ~1e5 lines of
// ~1000 positions, fewer than the GPU's resident threads): thread A runs the ring kernel's forward sweep on
// positions [0, h), thread B on [h, m), each from an empty stack.  A site B popped is dominated by B's own
// sites wherever it was minimal, so only B's final stack can enter the line's envelope: thread B then
// continues Meijster's sweep over those entries on top of A's final stack (pops and separators exactly as
// the sequential sweep would do them), writing the merged B part back into its own array; once an entry
// lands on its own B predecessor at an unchanged position the rest of B's stack is already right.  The two
// threads then write their halves of the output walking the merged stack (A part, then B part) from the
// entry covering their last position.  Same output as ring_line_kernel (the envelope's value is unique).
constexpr int kSplitLines = kRingThreads / 2;
__global__ void __launch_bounds__(kRingThreads, CVX_RING_MINB) ring2_line_kernel(const __grid_constant__ LinkParams p) {
  __shared__ unsigned long long ring[kRing][kRingThreads];
  __shared__ int s_k[kRingThreads];          // final stack top of every thread after its forward sweep
  __shared__ int s_ka[kSplitLines], s_rb[kSplitLines];   // merged stack: A part [0, ka], B part [0, rb]
  const int tid = threadIdx.x;
  const bool isB = tid >= kSplitLines;
  const int li = isB ? tid - kSplitLines : tid;
  const long long nlines = (long long)p.nx * p.nz;
  const long long line = (long long)blockIdx.x * kSplitLines + li;
  const bool valid = line < nlines;
  const int x = valid ? (int)(line % p.nx) : 0;
  const int o2 = valid ? (int)(line / p.nx) : 0;   // z
  const int m = p.ny;
  const int h = (m >> 4) << 3;                      // split position (multiple of 8; m >= 16)
  const long long stride = p.nx;
  const long long base = (long long)o2 * p.nx * p.ny + x;
  unsigned long long* const gA = static_cast<unsigned long long*>(p.meta) + (valid ? line : 0) * m;
  unsigned long long* const gB = gA + h;
  unsigned long long* const gst = isB ? gB : gA;    // this thread's own stack array
  unsigned long long* const rg = &ring[0][tid];
  auto raw_at = [&](int q) -> unsigned { return static_cast<const unsigned short*>(p.fin)[base + q * stride]; };
  auto f_of = [](unsigned v) -> unsigned { return v == kNone16 ? kInf32 : v * v; };
  auto row_has = [&](int q) -> bool {
    return !CVX_RING_ROWSKIP || p.rowmask[(long long)(o2 >> 3) * p.nby + (q >> 3)] != 0;
  };
  const int q_lo = isB ? h : 0, q_hi = isB ? m : h;
  int k = -1, lo = 0;
  int s_top = 0, t_top = 0;
  unsigned f_top = 0;
  if (valid) {   // ---- forward sweep of the own segment (as ring_line_kernel)
    unsigned fa[8];
    bool ha = row_has(q_lo);
#pragma unroll
    for (int u = 0; u < 8; ++u) fa[u] = ha ? raw_at(q_lo + u) : kNone16;
    for (int q0 = q_lo; q0 < q_hi; q0 += 8) {
      unsigned fb[8];
      const int qn = q0 + 8 < q_hi ? q0 + 8 : q0;
      const bool hb = row_has(qn);
#pragma unroll
      for (int u = 0; u < 8; ++u) fb[u] = hb ? raw_at(qn + u) : kNone16;
      if (ha) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u;
          const unsigned fq = f_of(fa[u]);
          if (fq == kInf32) continue;
          while (k >= 0) {
            const int a = t_top - s_top, c = t_top - q;
            if ((unsigned)(a * a) + f_top <= (unsigned)(c * c) + fq) break;
            if (--k < 0) break;
            if (k < lo) {
              const int j0 = max(0, k - (kRing - 1));
              for (int j = j0; j <= k; ++j) rg[(j & (kRing - 1)) * kRingThreads] = gst[j];
              lo = j0;
            }
            const unsigned long long e = rg[(k & (kRing - 1)) * kRingThreads];
            s_top = (int)(e & 0xffffu); t_top = (int)((e >> 16) & 0xffffu); f_top = (unsigned)(e >> 32);
          }
          int tq = 0;
          if (k >= 0) {
            const int sep = floordiv24(q * q - s_top * s_top + (int)fq - (int)f_top, 2 * (q - s_top));
            if (sep + 1 >= m) continue;
            tq = sep + 1;
          }
          ++k;
          unsigned long long* slot = rg + (k & (kRing - 1)) * kRingThreads;
          CVX_CHECK(k < q_hi - q_lo, "split stack depth <= segment length");
          if (k - kRing >= lo) { gst[k - kRing] = *slot; lo = k - kRing + 1; }
          *slot = ((unsigned long long)fq << 32) | ((unsigned)tq << 16) | (unsigned)q;
          s_top = q; t_top = tq; f_top = fq;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) fa[u] = fb[u];
      ha = hb;
    }
    for (int j = max(lo, 0); j <= k; ++j) gst[j] = rg[(j & (kRing - 1)) * kRingThreads];   // whole stack in HBM
  }
  s_k[tid] = k;
  __syncthreads();
  if (isB && valid) {   // ---- merge: B's stack entries continue the sweep on top of A's stack
    int ka = s_k[li];
    const int kb = k;
    int r = 0;          // B entries in the merged stack: gB[0, r)
    for (int j = 0; j <= kb; ++j) {
      const unsigned long long e = gB[j];
      const int es = (int)(e & 0xffffu);
      const unsigned ef = (unsigned)(e >> 32);
      while (r > 0 || ka >= 0) {
        const unsigned long long tp = r > 0 ? gB[r - 1] : gA[ka];
        const int ts = (int)(tp & 0xffffu), tt = (int)((tp >> 16) & 0xffffu);
        const unsigned tf = (unsigned)(tp >> 32);
        const int a = tt - ts, c = tt - es;
        if ((unsigned)(a * a) + tf <= (unsigned)(c * c) + ef) break;
        if (r > 0) --r; else --ka;
      }
      int tq = 0;
      bool on_pred = false;
      if (r > 0 || ka >= 0) {
        const unsigned long long tp = r > 0 ? gB[r - 1] : gA[ka];
        const int ts = (int)(tp & 0xffffu);
        const unsigned tf = (unsigned)(tp >> 32);
        const int sep = floordiv24(es * es - ts * ts + (int)ef - (int)tf, 2 * (es - ts));
        if (sep + 1 >= m) continue;                   // never wins inside the line: dropped
        tq = sep + 1;
        on_pred = r == j && r > 0;                     // on its own B predecessor, at its own position
      }
      gB[r] = ((unsigned long long)ef << 32) | ((unsigned)tq << 16) | (unsigned)es;   // r <= j
      ++r;
      if (on_pred) { r = kb + 1; break; }             // the rest of B's stack is unchanged
    }
    s_ka[li] = ka;
    s_rb[li] = r - 1;
  }
  __syncthreads();
  if (!valid) return;
  // ---- backward over the own half; unified index u: [0, ka] -> gA[u], then gB[u - ka - 1]
  const int ka = s_ka[li], rb = s_rb[li];
  auto at = [&](int u) -> const unsigned long long* { return u <= ka ? gA + u : gB + (u - ka - 1); };
  int u0;
  if (isB) u0 = ka + 1 + rb;                           // the top
  else {                                               // the entry covering h - 1
    int i = -1;
    while (i + 1 <= rb && (int)((gB[i + 1] >> 16) & 0xffffu) <= h - 1) ++i;
    if (i >= 0) u0 = ka + 1 + i;
    else {
      u0 = ka;
      while (u0 >= 0 && (int)((gA[u0] >> 16) & 0xffffu) > h - 1) --u0;
    }
  }
  k = u0;
  lo = u0 + 1;                                         // every entry comes from HBM (cp.async kAhead ahead)
  if (k >= 0) {
    const unsigned long long e = *at(k);
    s_top = (int)(e & 0xffffu); t_top = (int)((e >> 16) & 0xffffu); f_top = (unsigned)(e >> 32);
  }
  auto issue = [&](int j) {
    if (j >= 0 && j < lo) {
      const unsigned sa = smem_addr(rg + (j & (kRing - 1)) * kRingThreads);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(sa), "l"(at(j)) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (k >= 0) {
#pragma unroll 1
    for (int i = 1; i <= kAhead; ++i) issue(k - i);
  }
  const int qtop = isB ? (((m - 1) >> 3) << 3) : h - 8, qbot = isB ? h : 0;
  for (int q0 = qtop; q0 >= qbot; q0 -= 8) {
    const bool wy = p.colmask[(long long)(q0 >> 3) * p.nbx + (x >> 3)] != 0;
#pragma unroll kRingBUnroll
    for (int u = 7; u >= 0; --u) {
      const int q = q0 + u;
      unsigned d2 = kInf32;
      if (k >= 0) { const int dq = q - s_top; d2 = (unsigned)(dq * dq) + f_top; }
      CVX_CHECK(base + (long long)q * stride < (long long)p.nx * p.ny * p.nz, "split line output index");
      if (wy) p.g2[base + (long long)q * stride] = d2;
      if (k >= 0 && q == t_top) {
        if (--k >= 0) {
          if (k < lo) asm volatile("cp.async.wait_group %0;" :: "n"(kAhead - 1) : "memory");
          const unsigned long long e = *(volatile unsigned long long*)(rg + (k & (kRing - 1)) * kRingThreads);
          s_top = (int)(e & 0xffffu); t_top = (int)((e >> 16) & 0xffffu); f_top = (unsigned)(e >> 32);
          issue(k - kAhead);
        }
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ------------------------------------------------------------------------------- incremental (f1)
struct IncParams {
  const long long* sums;
  const unsigned* prev;       // bit-planes of the previous update (slots < nb_prev)
  unsigned* cur;              // bit-planes of this update
  unsigned char* flags;       // per slot: bit 0 site plane changed (source), bit 1 recompute
  int* list;
  int* cnt;
  const int* grid;            // dense slot grid over the AABB
  const int4* coords;
  float* esdf;
  int lo0, lo1, lo2, nbx, nby, nbz;
  int nb, nb_prev;
  double site_thr;
  double s, dmax;
  int r, rb, win;             // window radius (voxels), block radius, window side 8 + 2 r
};

__device__ __forceinline__ int grid_slot(const IncParams& p, int bx, int by, int bz) {
  bx -= p.lo0; by -= p.lo1; bz -= p.lo2;
  if (bx < 0 || by < 0 || bz < 0 || bx >= p.nbx || by >= p.nby || bz >= p.nbz) return -1;
  return p.grid[((long long)bz * p.nby + by) * p.nbx + bx];
}

// one warp per 32 voxels (= one plane word of one block)
// one warp per 4 plane words (128 consecutive voxels of one block) per step: the 4 loads of a lane are
// issued before any is classified
__global__ void inc_classify(const __grid_constant__ IncParams p) {
  const long long nw = (long long)p.nb * 16;                     // plane words
  const int lane = threadIdx.x & 31;
  const long long warp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w0 = warp0 * 4; w0 < nw; w0 += nwarps * 4) {   // nb * 16 is a multiple of 4
    longlong2 sw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sw[u] = reinterpret_cast<const longlong2*>(p.sums)[(w0 + u) * 32 + lane];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bool obs, neg, site;
      classify_voxel(sw[u], p.site_thr, obs, neg, site);
      const unsigned bo = __ballot_sync(0xffffffffu, obs), bn = __ballot_sync(0xffffffffu, neg),
                     bs = __ballot_sync(0xffffffffu, site);
      if (lane == u) {
        const int slot = (int)((w0 + u) >> 4), w = (int)((w0 + u) & 15);
        unsigned* c = p.cur + (long long)slot * kPlaneWords;
        c[w] = bo; c[16 + w] = bn; c[32 + w] = bs;
        unsigned char fl = 0;
        if (slot >= p.nb_prev) fl = (bs ? 1 : 0) | 2;    // new block: its sites are sources, it is written
        else {
          const unsigned* q = p.prev + (long long)slot * kPlaneWords;
          if (q[32 + w] != bs) fl = 3;
          else if (q[w] != bo || q[16 + w] != bn) fl = 2;
        }
        if (fl) atomicOr(reinterpret_cast<unsigned*>(p.flags + (slot & ~3)), (unsigned)fl << (8 * (slot & 3)));
      }
    }
  }
}

// queue every block within rb blocks (per axis) of a source block
__global__ void inc_dilate(const __grid_constant__ IncParams p) {
  const int k = 2 * p.rb + 1, k3 = k * k * k;
  const long long n = (long long)p.nb * k3;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int slot = (int)(i / k3), o = (int)(i % k3);
    if (!(p.flags[slot] & 1)) continue;
    const int4 c = p.coords[slot];
    const int ns = grid_slot(p, c.x + o % k - p.rb, c.y + (o / k) % k - p.rb, c.z + o / (k * k) - p.rb);
    if (ns >= 0 && !(p.flags[ns] & 2))
      atomicOr(reinterpret_cast<unsigned*>(p.flags + (ns & ~3)), 2u << (8 * (ns & 3)));
  }
}

__global__ void inc_compact(const __grid_constant__ IncParams p) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < p.nb; b += gridDim.x * blockDim.x) {
    const bool q = (p.flags[b] & 2) != 0;
    const unsigned m = __ballot_sync(__activemask(), q);
    if (!q) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(p.cnt, __popc(m));
    base = __shfl_sync(m, base, leader);
    p.list[base + __popc(m & ((1u << lane) - 1u))] = b;
  }
}

// exact clamped EDT of one queued block from the site planes of the (2 rb + 1)^3 blocks around it.
// Window: voxels [8 b - r, 8 b + 8 + r) per axis (W = 8 + 2 r <= 56 so an x-row is one u64).  Distances
// are exact below C = (r + 1)^2 and >= C otherwise (a saturated row distance r + 1 is <= the true one,
// and r >= d_max / s makes every value >= C clamp to d_max).
#ifndef CVX_INC_CTAS
#define CVX_INC_CTAS 16
#endif
__global__ void __launch_bounds__(256) inc_window(const __grid_constant__ IncParams p) {
  extern __shared__ __align__(1024) unsigned char dsmem[];
  unsigned char* smem = dsmem;
  const int k = 2 * p.rb + 1, k3 = k * k * k, W = p.win, r = p.r;
  unsigned* nbp = reinterpret_cast<unsigned*>(smem);                                 // [k3][16] site planes
  unsigned long long* rowm = reinterpret_cast<unsigned long long*>(smem + (size_t)k3 * 64);   // [W][W] (z, y)
  unsigned char* g1 = reinterpret_cast<unsigned char*>(rowm + (size_t)W * W);        // [W z][W y][8 x]
  unsigned short* g2 = reinterpret_cast<unsigned short*>(g1 + (size_t)W * W * 8);    // [W z][8 y][8 x]
  __shared__ int s_slot;
  __shared__ int s_nbs[343];      // slot of every block of the (2 Rb + 1)^3 neighbourhood (Rb <= 3)
  const int nq = *(volatile const int*)p.cnt;
  const int off = 8 * p.rb - r;   // window origin inside the neighbourhood (voxels)
  const unsigned C = (unsigned)((r + 1) * (r + 1));
  for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) s_slot = p.list[qi];
    __syncthreads();
    const int slot = s_slot;
    const int4 c = p.coords[slot];
    for (int o = threadIdx.x; o < k3; o += blockDim.x)
      s_nbs[o] = grid_slot(p, c.x + o % k - p.rb, c.y + (o / k) % k - p.rb, c.z + o / (k * k) - p.rb);
    __syncthreads();
    for (int i = threadIdx.x; i < k3 * 16; i += blockDim.x) {
      const int ns = s_nbs[i >> 4];
      nbp[i] = ns >= 0 ? p.cur[(long long)ns * kPlaneWords + 32 + (i & 15)] : 0u;
    }
    __syncthreads();
    // x-row bit masks of the window (row index i = zw W + yw kept incrementally: no divisions)
    const int dz_step = (int)blockDim.x / W, dy_step = (int)blockDim.x % W;
    int yw = (int)threadIdx.x % W, zw = (int)threadIdx.x / W;
    for (int i = threadIdx.x; i < W * W; i += blockDim.x, yw += dy_step, zw += dz_step) {
      if (yw >= W) { yw -= W; ++zw; }
      const int yn = yw + off, zn = zw + off;
      const int by = yn >> 3, bz = zn >> 3, row = (yn & 7) + 8 * (zn & 7);
      unsigned long long bits = 0;
      for (int bx = 0; bx < k; ++bx) {
        const unsigned wd = nbp[((bz * k + by) * k + bx) * 16 + (row >> 2)];
        bits |= (unsigned long long)((wd >> (8 * (row & 3))) & 0xffu) << (8 * bx);
      }
      bits >>= off;
      if (W < 64) bits &= (1ull << W) - 1ull;
      rowm[i] = bits;
    }
    __syncthreads();
    // pass x: distance along x to the nearest window site (saturated at r + 1), for the block's 8 columns
    for (int i = threadIdx.x; i < W * W * 8; i += blockDim.x) {
      const int x = i & 7, yz = i >> 3;
      const unsigned long long mk = rowm[yz];
      const int xw = r + x;
      int d = r + 1;
      const unsigned long long lm = mk & ((2ull << xw) - 1ull);
      if (lm) d = min(d, xw - (63 - __clzll(lm)));
      const unsigned long long rm = mk >> xw;
      if (rm) d = min(d, __ffsll(rm) - 1);
      g1[i] = (unsigned char)d;
    }
    __syncthreads();
    // pass y: min over the window's y of g1^2 + dy^2, for y in the block (saturated at C)
    for (int i = threadIdx.x; i < W * 64; i += blockDim.x) {
      const int x = i & 7, y = (i >> 3) & 7, zw = i >> 6;
      const int yc = r + y;
      unsigned best = C;
      const unsigned char* col = g1 + (size_t)zw * W * 8 + x;
      for (int yw = 0; yw < W; ++yw) {
        const unsigned g = col[yw * 8];
        const int dy = yc - yw;
        best = min(best, g * g + (unsigned)(dy * dy));
      }
      g2[i] = (unsigned short)best;
    }
    __syncthreads();
    // pass z + write-back: E = sign(D) min(s sqrt(d^2), d_max), NaN unobserved
    for (int l = threadIdx.x; l < kBlockVox; l += blockDim.x) {
      const int xy = l & 63, z = l >> 6;
      const int zc = r + z;
      unsigned best = C;
      for (int zw = 0; zw < W; ++zw) {
        const int dz = zc - zw;
        best = min(best, (unsigned)g2[zw * 64 + xy] + (unsigned)(dz * dz));
      }
      const unsigned* pl = p.cur + (long long)slot * kPlaneWords;
      const bool obs = (pl[l >> 5] >> (l & 31)) & 1u, neg = (pl[16 + (l >> 5)] >> (l & 31)) & 1u;
      float e;
      if (!obs) e = __int_as_float(0x7fc00000);
      else {
        const double md = best >= C ? p.dmax : fmin(p.s * sqrt((double)best), p.dmax);
        e = (float)(neg ? -md : md);
      }
      p.esdf[(long long)slot * kBlockVox + l] = e;
    }
  }
}

// ------------------------------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

cudaError_t grow_async(void** ptr, int64_t* cap, int64_t need, cudaStream_t st) {
  if (*cap >= need) return cudaSuccess;
  if (*ptr) cudaFreeAsync(*ptr, st);
  *ptr = nullptr;
  *cap = 0;
  cudaError_t e = cudaMallocAsync(ptr, (size_t)need, st);
  if (e == cudaSuccess) *cap = need;
  return e;
}

cudaError_t ensure_planes(cvx_submap* sm, cudaStream_t st) {
  if (sm->planes[0]) return cudaSuccess;
  const size_t bytes = (size_t)sm->pool.max_blocks * kPlaneWords * 4;
  cudaError_t e = cudaMallocAsync(&sm->planes[0], bytes, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&sm->planes[1], bytes, st);
  return e;
}

// dense slot grid over the AABB (+ optional column / row masks)
cudaError_t build_grid(cvx_submap* sm, const int lo[3], int nbx, int nby, int nbz, unsigned char* colmask,
                       unsigned char* rowmask, cudaStream_t st, const char* name) {
  const long long nblk = (long long)nbx * nby * nbz;
  void* g = sm->block_grid;
  cudaError_t e = grow_async(&g, &sm->block_grid_cap, nblk * (long long)sizeof(int), st);
  sm->block_grid = static_cast<int*>(g);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(sm->block_grid, 0xff, sizeof(int) * (size_t)nblk, st);
  ProfScope ps_(sm, name, st);
  block_grid_kernel<<<148 * 4, 256, 0, st>>>(sm->ctr, sm->pool.coords, sm->pool.max_blocks, sm->block_grid, colmask,
                                             rowmask, lo[0], lo[1], lo[2], nbx, nby);
  return cudaSuccess;
}

template <bool kZ>
cudaError_t launch_pba(cvx_submap* sm, const void* fin, const PbaParams& base, cudaStream_t st) {
  auto enc = tmap_encoder();
  if (!enc) return cudaErrorNotSupported;
  PbaParams p = base;
  const size_t esize = kZ ? 4 : 2;
  p.m = kZ ? p.nz : p.ny;
  p.nbox = (p.m + 255) / 256;
  p.box_h = ((p.m + p.nbox - 1) / p.nbox + 7) & ~7;   // box bytes a multiple of 128 (TMA smem alignment)
  p.rows = p.nbox * p.box_h;
  p.tx = 8;
  for (int t : {32, 16}) {
    if (pba_smem_bytes<kZ>(p.rows, t, 1) <= 80 * 1024 && t <= p.nx) { p.tx = t; break; }
  }
  int B = 1;
  while (B * 2 * p.tx <= 256 && B * 2 <= 32 && (p.m + B * 2 - 1) / (B * 2) >= 12) B *= 2;
  p.nbands = B;
  p.lb = (p.m + B - 1) / B;
  p.tiles_x = (p.nx + p.tx - 1) / p.tx;
  const size_t smem = pba_smem_bytes<kZ>(p.rows, p.tx, B);
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)p.nx, (cuuint64_t)p.ny, (cuuint64_t)p.nz};
  const cuuint64_t strides[2] = {(cuuint64_t)p.nx * esize, (cuuint64_t)p.nx * p.ny * esize};
  const cuuint32_t box[3] = {(cuuint32_t)p.tx, kZ ? 1u : (cuuint32_t)p.box_h, kZ ? (cuuint32_t)p.box_h : 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&tm, kZ ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                    const_cast<void*>(fin), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  cudaFuncSetAttribute(pba_line_kernel<kZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long tiles = (long long)p.tiles_x * (kZ ? p.ny : p.nz);
  ProfScope ps_(sm, kZ ? "esdf_pass_z" : "esdf_pass_y", st);
  pba_line_kernel<kZ><<<(unsigned)tiles, p.tx * B, smem, st>>>(tm, p);
  return cudaGetLastError();
}

// the dense exact EDT (finalize; capped = f1 fallback): planes go to sm->planes[sm->cur_planes]
cudaError_t dense_edt(cvx_submap* sm, const int lo[3], const int hi[3], cudaStream_t st, bool capped, double dmax) {
  const int nbx = hi[0] - lo[0] + 1, nby = hi[1] - lo[1] + 1, nbz = hi[2] - lo[2] + 1;
  const int nx = 8 * nbx, ny = 8 * nby, nz = 8 * nbz;
  const long long nvox = (long long)nx * ny * nz;
  cudaError_t e = ensure_planes(sm, st);
  if (e != cudaSuccess) return e;
  // passes y / z: 0 = ring kernel where it fits 24 bits, else the link kernel (default); 2 = the streaming
  // Meijster link kernel; 1 = TMA-staged band hulls
  static const int kernel = [] { const char* v = std::getenv("CVX_EDT_KERNEL"); return v ? std::atoi(v) : 0; }();
  const long long need = nvox * (4 + 2 + (kernel != 1 ? 8 : 0)) + (long long)nbx * nby + (long long)nby * nbz + 256;
  if ((e = grow_async(&sm->edt, &sm->edt_bytes, need, st)) != cudaSuccess) return e;
  unsigned* g2 = reinterpret_cast<unsigned*>(sm->edt);
  unsigned short* g1 = reinterpret_cast<unsigned short*>(g2 + nvox);   // nvox % 512 == 0: aligned
  void* meta = g1 + nvox;                                                  // link variant only
  unsigned char* colmask = reinterpret_cast<unsigned char*>(g1 + nvox) + (kernel != 1 ? 8 * nvox : 0);
  unsigned char* rowmask = colmask + (size_t)nbx * nby;
  cudaMemsetAsync(colmask, 0, (size_t)nbx * nby + (size_t)nby * nbz, st);
  if ((e = build_grid(sm, lo, nbx, nby, nbz, colmask, rowmask, st, "esdf_block_grid")) != cudaSuccess) return e;
  unsigned* planes = sm->planes[sm->cur_planes];
  XParams xp;
  xp.sums = sm->pool.sums; xp.planes = planes; xp.grid = sm->block_grid; xp.g1 = g1; xp.rowmask = rowmask;
  xp.nx = nx; xp.ny = ny; xp.nz = nz; xp.nbx = nbx; xp.nby = nby; xp.site_thr = sm->cfg.site_threshold;
  xp.max_blocks = sm->pool.max_blocks;
  const int nch = (nx + 31) / 32;
  const size_t smem = xsmem_bytes(nch, nbx);
  if (smem > 48 * 1024) cudaFuncSetAttribute(pass_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long rows = (long long)ny * nz;
  const unsigned xblocks = (unsigned)std::min<long long>(rows / 4, 148ll * 16);
  {
    ProfScope ps_(sm, "esdf_pass_x", st);
    pass_x_kernel<<<xblocks, 128, smem, st>>>(xp);
  }
  // ring kernel: every separator numerator and squared distance below 2^24 (exact in fp32 / int32)
  const long long mx2 = (long long)(nx - 1) * (nx - 1), my2 = (long long)(ny - 1) * (ny - 1);
  const bool ring_y = (long long)ny * ny + mx2 < (1ll << 24), ring_z = (long long)nz * nz + mx2 + my2 < (1ll << 24);
  if (kernel == 0 || kernel == 2) {
    LinkParams lp{};
    lp.fin = g1; lp.g2 = g2; lp.meta = meta; lp.esdf = sm->pool.esdf; lp.grid = sm->block_grid; lp.colmask = colmask;
    lp.rowmask = rowmask;
    lp.planes = planes; lp.nx = nx; lp.ny = ny; lp.nz = nz; lp.nbx = nbx; lp.nby = nby; lp.s = sm->cfg.voxel_size;
    lp.capped = capped ? 1 : 0; lp.dmax = dmax;
    {
      ProfScope ps_(sm, "esdf_pass_y", st);
      const long long nl = (long long)nx * nz;
      // few long lines (fewer than ~1.5 per resident thread slot): two threads per line
      // (serial ESDF: pass y 0.54 -> 0.40 ms on configs[1], 20.7 -> 15.5 ms over the MAV submaps; but beside a
      // concurrent update walk the wider kernel costs the walk more than it saves: configs[1] step 6.21 ->
      // 6.28 ms, MAV 80.8 -> 83.5-89.3 ms — so off by default, CVX_EDT_SPLIT=1 enables it per call)
      const char* sv = std::getenv("CVX_EDT_SPLIT");
      const int split = sv ? std::atoi(sv) : 0;
      if (kernel == 0 && ring_y && split && ny >= 64 && nl < 148ll * 7 * kRingThreads * 3 / 2)
        ring2_line_kernel<<<(unsigned)((nl + kSplitLines - 1) / kSplitLines), kRingThreads, 0, st>>>(lp);
      else if (kernel == 0 && ring_y) ring_line_kernel<false><<<(unsigned)((nl + kRingThreads - 1) / kRingThreads), kRingThreads, 0, st>>>(lp);
      else link_line_kernel<false><<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(lp);
    }
    lp.fin = g2;
    ProfScope ps_(sm, "esdf_pass_z", st);
    const long long nl = (long long)nx * ny;
    if (kernel == 0 && ring_z) ring_line_kernel<true><<<(unsigned)((nl + kRingThreads - 1) / kRingThreads), kRingThreads, 0, st>>>(lp);
    else link_line_kernel<true><<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(lp);
    return cudaGetLastError();
  }
  PbaParams pp{};
  pp.g2 = g2; pp.esdf = sm->pool.esdf; pp.grid = sm->block_grid; pp.colmask = colmask; pp.planes = planes;
  pp.nx = nx; pp.ny = ny; pp.nz = nz; pp.nbx = nbx; pp.nby = nby; pp.s = sm->cfg.voxel_size;
  pp.capped = capped ? 1 : 0; pp.dmax = dmax;
  if ((e = launch_pba<false>(sm, g1, pp, st)) != cudaSuccess) return e;
  return launch_pba<true>(sm, g2, pp, st);
}

}  // namespace

cudaError_t launch_finalize(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], cudaStream_t st) {
  sm->inc.nb_prev = 0;   // the uncapped ESDF is not the incremental one: the next update recomputes all
  if (n_blocks <= 0) return cudaSuccess;
  return dense_edt(sm, lo, hi, st, false, 0.0);
}

cudaError_t launch_update_esdf(cvx_submap* sm, int n_blocks, const int lo[3], const int hi[3], cudaStream_t st,
                               int* blocks_updated) {
  *blocks_updated = 0;
  if (n_blocks <= 0) { sm->inc.nb_prev = 0; return cudaSuccess; }
  cudaError_t e = ensure_planes(sm, st);
  if (e != cudaSuccess) return e;
  const double s = sm->cfg.voxel_size, dmax = sm->cfg.esdf_max_distance;
  const int r = std::max(1, (int)std::ceil(dmax / s));
  const int rb = (r + 7) / 8;
  if (rb > 3) {   // window of more than 7^3 blocks: the dense exact EDT, clamped (same values)
    sm->cur_planes ^= 1;
    if ((e = dense_edt(sm, lo, hi, st, true, dmax)) != cudaSuccess) return e;
    sm->inc.nb_prev = n_blocks;
    *blocks_updated = n_blocks;
    return cudaSuccess;
  }
  if (!sm->inc.flags) {
    const size_t mb = (size_t)sm->pool.max_blocks;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&sm->inc.flags), (mb + 3) & ~(size_t)3, st)) != cudaSuccess ||
        (e = cudaMallocAsync(reinterpret_cast<void**>(&sm->inc.list), mb * 4, st)) != cudaSuccess ||
        (e = cudaMallocAsync(reinterpret_cast<void**>(&sm->inc.cnt), 4, st)) != cudaSuccess ||
        (e = cudaMallocHost(&sm->inc.cnt_host, 4)) != cudaSuccess)
      return e;
  }
  const int nbx = hi[0] - lo[0] + 1, nby = hi[1] - lo[1] + 1, nbz = hi[2] - lo[2] + 1;
  if ((e = build_grid(sm, lo, nbx, nby, nbz, nullptr, nullptr, st, "inc_block_grid")) != cudaSuccess) return e;
  const int prev = sm->cur_planes, cur = prev ^ 1;
  IncParams ip;
  ip.sums = sm->pool.sums; ip.prev = sm->planes[prev]; ip.cur = sm->planes[cur];
  ip.flags = sm->inc.flags; ip.list = sm->inc.list; ip.cnt = sm->inc.cnt; ip.grid = sm->block_grid;
  ip.coords = sm->pool.coords; ip.esdf = sm->pool.esdf;
  ip.lo0 = lo[0]; ip.lo1 = lo[1]; ip.lo2 = lo[2]; ip.nbx = nbx; ip.nby = nby; ip.nbz = nbz;
  ip.nb = n_blocks; ip.nb_prev = std::min(sm->inc.nb_prev, n_blocks);
  ip.site_thr = sm->cfg.site_threshold; ip.s = s; ip.dmax = dmax;
  ip.r = r; ip.rb = rb; ip.win = 8 + 2 * r;
  cudaMemsetAsync(sm->inc.flags, 0, ((size_t)n_blocks + 3) & ~(size_t)3, st);
  cudaMemsetAsync(sm->inc.cnt, 0, 4, st);
  {
    ProfScope ps_(sm, "inc_classify", st);
    inc_classify<<<148 * 8, 256, 0, st>>>(ip);
  }
  {
    ProfScope ps_(sm, "inc_dilate", st);
    const long long n = (long long)n_blocks * (2 * rb + 1) * (2 * rb + 1) * (2 * rb + 1);
    inc_dilate<<<(unsigned)std::min<long long>((n + 255) / 256, 148ll * 16), 256, 0, st>>>(ip);
  }
  {
    ProfScope ps_(sm, "inc_compact", st);
    inc_compact<<<(n_blocks + 255) / 256, 256, 0, st>>>(ip);
  }
  const int k = 2 * rb + 1, W = ip.win;
  const size_t smem = (size_t)k * k * k * 64 + (size_t)W * W * 8 + (size_t)W * W * 8 + (size_t)W * 64 * 2;
  cudaFuncSetAttribute(inc_window, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  {
    ProfScope ps_(sm, "inc_window", st);
    inc_window<<<148 * CVX_INC_CTAS, 256, smem, st>>>(ip);
  }
  cudaMemcpyAsync(sm->inc.cnt_host, sm->inc.cnt, 4, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *blocks_updated = *sm->inc.cnt_host;
  sm->cur_planes = cur;
  sm->inc.nb_prev = n_blocks;
  return cudaGetLastError();
}

void release_esdf(cvx_submap* sm) {
  if (sm->edt) cudaFree(sm->edt);
  if (sm->block_grid) cudaFree(sm->block_grid);
  for (auto& pl : sm->planes) if (pl) cudaFree(pl);
  if (sm->inc.flags) cudaFree(sm->inc.flags);
  if (sm->inc.list) cudaFree(sm->inc.list);
  if (sm->inc.cnt) cudaFree(sm->inc.cnt);
  if (sm->inc.cnt_host) cudaFreeHost(sm->inc.cnt_host);
  sm->edt = nullptr; sm->block_grid = nullptr; sm->planes[0] = sm->planes[1] = nullptr;
  sm->inc = cvx_submap::Inc{};
}

}  // namespace cvx
