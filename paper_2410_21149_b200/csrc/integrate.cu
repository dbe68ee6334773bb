// integrate.cu — TSDF integration kernels for sm_100a.
//
//   compose_kernel  O1   T_SC = T_WS^-1 T_WC per frame (fp64, fixed order, no FMA)
//   prepare_kernel  a1+a2  point -> ray (O2-O3, O6), range filter, fixed-point endpoints, closed-form
//                        voxel count n_r = 1 + sum|dv| (COUNT) with warp-local counters
//                        reduced once per warp, warp-ballot compaction of the used rays
//                        Organised sensors are read in 4x8 pixel patches per warp so the 32 rays of a
//                        warp are spatial neighbours; each ray claims space for its block-slot list by a
//                        warp-aggregated atomicAdd on a pre-allocated buffer.
//   block_walk_kernel a3  ALLOCATE: the same exact integer traversal at block granularity (block
//                        boundaries are a subset of voxel boundaries, so the block sequence is exactly
//                        the one the voxel walk visits); every block is activated in the hash table
//                        (insert-if-absent + slot bump) and its slot recorded in the
//                        ray's list.
//   walk_kernel     a4+a5  exact integer 6-connected voxel traversal (O4) reading the block slots from
//                        the ray's list (prefetched one block ahead, no hashing in the hot loop); every
//                        voxel gets the projective sdf (O5) and (w d, w) is merged per voxel —
//                        lanes of a warp hitting the same voxel are reduced with match.any + a shuffle
//                        tree, then one 64-bit red.global.add pair per distinct voxel per warp step.  The
//                        TSDF state IS the pair of exact fixed-point sums, so the "fold"
//                        D = sum(wd)/sum(w) (a5) is evaluated on read (export / finalize) and
//                        fusion is order-independent and deterministic (R6).
//   reset kernels   zero the used blocks, counters and AABB.
#include <algorithm>
#include <vector>
#include <cmath>
#include <cstdio>
#include <type_traits>

#include "submap.h"

namespace cvx {
namespace {

// Fixed-point sdf along a ray: units of 2^-(q+kSdfF) metres, q = packed_q(tau).
constexpr int kSdfF = 20;

// Per used ray, written by prepare_kernel, read by the block walk and the update walk (48 B, SURVEY
// §8(a1) "<= 48 B/ray"): the fixed-point start A relative to the frame's fixed-point origin O (0 in
// carve mode), the end B relative to A, the first voxel's sdf with the frame index in its low 13 bits,
// the per-step sdf decrements (in units of 4) and the ray's block-slot list offset.  Colour and general
// weights live in per-ray side arrays, allocated only for those modes.
struct __align__(16) RayRec {
  int dA[3];          // A - O, fixed point 2^-16 voxel (O = q(t_SC) of the frame, compose_kernel)
  int dB[3];          // B - A (a span < 2^15 voxels per axis, O3)
  long long S0f;      // S0 << kFrameBits | frame, S0 = projective sdf of the first voxel (fixed point kSdfF)
  unsigned U[3];      // sdf decrement per voxel step along axis a, >> kUShift (>= 0)
  int list_off;       // offset of the ray's block-slot list, -1 if the list buffer was full
};
static_assert(sizeof(RayRec) == 48, "RayRec layout");
constexpr int kFrameBits = 13;      // frame index within a launch (< kMaxBatch)
constexpr int kUShift = 2;          // U <= s 2^(q + kSdfF) <= 2^34 (tau >= 2 s): U >> 2 fits 32 bits

// The ray as the kernels use it (expanded from RayRec + the frame records + the side arrays).
struct RayView {
  long long A[3], B[3];
  long long S0, U[3];
  float w;
  int n_vox, list_off, frame;
  unsigned rgb;
};

struct ComposeParams {
  double Tws[16];
  double Twc[kMaxBatch][16];
  double s;
  int n;
};

// per-frame record written by compose_kernel: R_SC (9), t_SC (3), fixed-point origin q(t_SC) (3 int64
// bit patterns), origin-in-domain flag
constexpr int kFrameRec = 16;

// Organised-sensor patch one warp's rays come from: CVX_PATCH_ROWS rows x 32 / CVX_PATCH_ROWS columns.
#ifndef CVX_BAND2
#define CVX_BAND2 1
#endif
// Slimmer block entry in walk_cw_kernel: the next slot is prefetched without a bound check (the slot-list
// buffer keeps one spare entry past list_cap) and mapped to the trash block with one unsigned min.
#ifndef CVX_ENTRY2
#define CVX_ENTRY2 1
#endif
#ifndef CVX_WG0
#define CVX_WG0 1
#endif
#ifndef CVX_COPY_EARLY
#define CVX_COPY_EARLY 1
#endif
#ifndef CVX_PATCH_ROWS
#define CVX_PATCH_ROWS 4
#endif
static_assert(CVX_PATCH_ROWS == 1 || CVX_PATCH_ROWS == 2 || CVX_PATCH_ROWS == 4 || CVX_PATCH_ROWS == 8, "patch rows");

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// x / s correctly rounded (IEEE, identical to __ddiv_rn and to the oracle's x / s) for s > 0, given any
// approximation rs of 1/s: Markstein's final step q = q0 + (x - q0 s) rs, then an exact check — the
// remainder r = x - q s is computed exactly by the FMA when q is within a few ulps, and |r| < s ulp(q) / 2
// proves q = RN(x / s) (RN is monotone, so a rounded remainder below the bound is a true one below it).
// Anything unproven (a power-of-two q, whose lower half-ulp is smaller; tiny / huge exponents; or a
// failed check) takes the IEEE division.  Replaces the Newton iteration of a reciprocal per division.
#ifndef CVX_FAST_DIV
#define CVX_FAST_DIV 1
#endif
__device__ __forceinline__ double div_rn(double x, double s, double rs) {
#if CVX_FAST_DIV
  const double q0 = __dmul_rn(x, rs);
  const double q = __fma_rn(__fma_rn(-q0, s, x), rs, q0);
  const double r = __fma_rn(-q, s, x);
  const int hi = __double2hiint(q), lo = __double2loint(q);
  const int e = (hi >> 20) & 0x7ff;
  if (e > 54 && e < 2046 && ((hi & 0xfffff) | lo) != 0) {
    const double h = __hiloint2double((e - 53) << 20, 0);   // ulp(q) / 2
    if (fabs(r) < __dmul_rn(h, s)) return q;
  }
#endif
  return __ddiv_rn(x, s);
}

// O3: q(x) = floor((x / s) * 2^16), rejected outside |voxel| < 2^23.  rs ~ 1/s (see div_rn).
__device__ __forceinline__ bool quantise(double x, double s, long long* q, double rs) {
  double a = dm(div_rn(x, s, rs), 65536.0);
  if (!(fabs(a) < 549755813888.0)) return false;
  *q = (long long)floor(a);
  return true;
}
__device__ __forceinline__ bool quantise(double x, double s, long long* q) {
  return quantise(x, s, q, __drcp_rn(s));
}

// n / d for n < 2^32, 0 < d < 2^32 given rd = RN(1/d): the truncated fp64 product is the quotient or one
// less (its absolute error (n/d) 2^-52 is below the 1/d gap to the next integer), fixed by one compare.
__device__ __forceinline__ unsigned udiv_fast(unsigned n, unsigned d, double rd) {
  unsigned q = __double2uint_rz(__dmul_rn((double)n, rd));
  if (n - q * d >= d) ++q;
  return q;
}

// O1: R_SC[i][j] = ((Rws[0][i] Rwc[0][j] + Rws[1][i] Rwc[1][j]) + Rws[2][i] Rwc[2][j]),
// t_SC[i] = ((Rws[0][i](twc0-tws0) + Rws[1][i](twc1-tws1)) + Rws[2][i](twc2-tws2)).
__global__ void compose_kernel(const __grid_constant__ ComposeParams p, double* out) {
  int f = threadIdx.x;
  if (f >= p.n) return;
  const double* W = p.Tws;
  const double* C = p.Twc[f];
  double* o = out + kFrameRec * f;
  bool ok = true;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j)
      o[3 * i + j] = da(da(dm(W[0 * 4 + i], C[0 * 4 + j]), dm(W[1 * 4 + i], C[1 * 4 + j])), dm(W[2 * 4 + i], C[2 * 4 + j]));
    o[9 + i] = da(da(dm(W[0 * 4 + i], ds(C[3], W[3])), dm(W[1 * 4 + i], ds(C[7], W[7]))),
                  dm(W[2 * 4 + i], ds(C[11], W[11])));
    long long q = 0;
    ok = quantise(o[9 + i], p.s, &q) && ok;     // O3: the carve start A = q(o) is shared by the frame
    o[12 + i] = __longlong_as_double(q);
  }
  o[15] = ok ? 1.0 : 0.0;
}

struct PrepParams {
  const float* data;
  long long n_per_frame;
  long long total;
  int kind, width;
  float fx, fy, cx, cy;
  double rmin, rmax, s, tau, rfloor;
  double sdf_scale;   // 2^(q + kSdfF)
  double rs;          // RN(1 / s) (fast correctly rounded divisions by s, div_rn)
  double r_npf, r_width, r_pcols;   // RN(1 / n_per_frame), RN(1 / width), RN(1 / (width / patch cols))
  int sec_cols, nframes;            // sector-major ray order (organised sensors): patch columns per sector, 0 = off
  double r_secpat, r_frmpat, r_seccols;   // RN(1 / patches per sector), RN(1 / patches per (sector, frame)), RN(1 / sec_cols)
  int weighting, carve;
  int height;
  const double* frame_T;
  RayRec* rays;
  unsigned* rgbs;   // nullable: per used ray colour r | g << 8 | b << 16 (TSDF + Color)
  float* ws;        // nullable: per used ray weight (weighting != 0)
  Counters* ctr;
  int* lcnt;        // {n_rays, n_slots} of this launch (8-byte aligned)
  int list_cap;
  const int* trig;  // nullable: {threshold, hit, consumed}; a hit submap takes no further frames
  const unsigned char* rgb;   // nullable: per-point colour [total][3]
  int count_vox;    // add the raycast voxel counts to ctr->voxel_updates (0: projection mapping)
  int* box;         // nullable: per CTA {lo[3], hi[3]} block box of its rays (dense-window path, R19)
  unsigned long long* cstat;   // nullable: per CTA look-back status (zeroed): rays claimed in CTA order
};

#ifndef CVX_PREP_MINB
#define CVX_PREP_MINB 5   // 48 registers, 5 CTAs per SM: prepare 0.505 -> 0.467 ms against __launch_bounds__(256) (56 registers)
#endif
#ifndef CVX_SECTOR_COLS
#define CVX_SECTOR_COLS 0    // > 0: sector-major ray order, patch columns per sector (measured slower: concurrent warps collide on the same voxels)
#endif
#ifndef CVX_PREP_ORDERED
#define CVX_PREP_ORDERED 0   // 1: rays claimed in CTA order (decoupled look-back) instead of atomic arrival order (walk -1.6 %, prepare +80 %: off)
#endif
#ifndef CVX_PREP_THREADS
#define CVX_PREP_THREADS 256
#endif
constexpr int kPrepThreads = CVX_PREP_THREADS;
__global__ void __launch_bounds__(kPrepThreads, CVX_PREP_MINB) prepare_kernel(const __grid_constant__ PrepParams p) {
  if (p.trig && *(volatile const int*)&p.trig[1]) return;   // block-count trigger fired: frame not taken
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int status = -1;  // -1 no thread, 0 used, 1 invalid, 2 range, 3 domain
  RayView rec;
  unsigned f_used = 0;
  if (idx < p.total) {
    // (index arithmetic in 32 bits: a launch holds < 2^31 rays; divisions by multiplication, udiv_fast)
    unsigned f = udiv_fast((unsigned)idx, (unsigned)p.n_per_frame, p.r_npf);
    unsigned i = (unsigned)idx - f * (unsigned)p.n_per_frame;
    constexpr int PR = CVX_PATCH_ROWS, PC = 32 / CVX_PATCH_ROWS;
    if (p.sec_cols > 0) {
      // sector-major order: azimuth sector s of every frame of the launch, then the next sector — the walk's
      // warps in flight then touch one sector's voxels (nearly the same for consecutive scans), a smaller L2
      // working set for their reductions.  Inside a (sector, frame): patch rows x sector patch columns.
      const unsigned P = (unsigned)idx >> 5, l = (unsigned)idx & 31u;
      const unsigned S = (unsigned)p.sec_cols, prows = (unsigned)p.height / PR;
      const unsigned PF = prows * S, PS = PF * (unsigned)p.nframes;
      const unsigned sec = udiv_fast(P, PS, p.r_secpat);
      const unsigned rem = P - sec * PS;
      f = udiv_fast(rem, PF, p.r_frmpat);
      const unsigned rem2 = rem - f * PF;
      const unsigned prow = udiv_fast(rem2, S, p.r_seccols);
      const unsigned pcol = sec * S + (rem2 - prow * S);
      const unsigned rr = l / PC, cc = (rr & 1) ? PC - 1 - (l % PC) : (l % PC);
      i = (prow * PR + rr) * (unsigned)p.width + pcol * PC + cc;
    } else if (p.kind != 0 && p.width > 0 && p.height > 0 && p.width % PC == 0 && p.height % PR == 0) {
      // organised sensor: warp = PR rows x PC columns patch (spatially coherent rays per warp)
      const unsigned pt = i >> 5, l = i & 31, pcols = (unsigned)p.width / PC;
      const unsigned rr = l / PC, cc = (rr & 1) ? PC - 1 - (l % PC) : (l % PC);   // serpentine: lane l+1 neighbours lane l
      const unsigned prow = udiv_fast(pt, pcols, p.r_pcols);
      const unsigned row = prow * PR + rr, col = (pt - prow * pcols) * PC + cc;
      i = row * (unsigned)p.width + col;
    }
    f_used = f;
    const long long src = f * p.n_per_frame + i;
    const double* T = p.frame_T + kFrameRec * f;
    double pc[3];
    status = 0;
    if (p.kind == 1) {  // O2: pinhole depth -> point in fp32 exactly as written, integer pixel (Q24)
      float z = p.data[src];
      if (!(z > 0.0f) || !isfinite(z)) status = 1;
      const unsigned vi = udiv_fast(i, (unsigned)p.width, p.r_width);
      float u = (float)(int)(i - vi * (unsigned)p.width), v = (float)(int)vi;
      pc[0] = (double)__fdiv_rn(__fmul_rn(z, __fsub_rn(u, p.cx)), p.fx);
      pc[1] = (double)__fdiv_rn(__fmul_rn(z, __fsub_rn(v, p.cy)), p.fy);
      pc[2] = (double)z;
    } else {
      const float* q = p.data + 3 * src;
      pc[0] = q[0]; pc[1] = q[1]; pc[2] = q[2];
      if (!isfinite(pc[0]) || !isfinite(pc[1]) || !isfinite(pc[2])) status = 1;
    }
    if (status == 0) {
      double pw[3], d[3];
      for (int a = 0; a < 3; ++a) {
        pw[a] = da(da(da(dm(T[3 * a + 0], pc[0]), dm(T[3 * a + 1], pc[1])), dm(T[3 * a + 2], pc[2])), T[9 + a]);
        d[a] = ds(pw[a], T[9 + a]);
      }
      double L = __dsqrt_rn(da(da(dm(d[0], d[0]), dm(d[1], d[1])), dm(d[2], d[2])));
      if (!(L >= p.rmin && L <= p.rmax) || !(L > 0.0)) status = 2;  // Q10
      if (status == 0) {
        if (p.carve && T[15] == 0.0) status = 3;
        const double rL = __drcp_rn(L);
        for (int a = 0; a < 3 && status == 0; ++a) {
          double ext = div_rn(dm(p.tau, d[a]), L, rL);
          double e = da(pw[a], ext);                         // tau behind the point
          bool okA = true;
          if (p.carve) rec.A[a] = __double_as_longlong(T[12 + a]);   // from the optical centre (Q2)
          else okA = quantise(ds(pw[a], ext), p.s, &rec.A[a], p.rs);
          if (!okA || !quantise(e, p.s, &rec.B[a], p.rs)) status = 3;
          else {
            long long span = (rec.B[a] >> 16) - (rec.A[a] >> 16);
            if (span >= 32768 || span <= -32768) status = 3;
          const long long dA = rec.A[a] - __double_as_longlong(T[12 + a]);   // band mode: A - O in int32
          if (dA >= (1ll << 31) || dA < -(1ll << 31)) status = 3;
          }
        }
        if (status == 0) {
          // O5 in fixed point: sdf of the first voxel v_A, then an exact per-axis decrement s |u_a| per
          // step (stepping axis a moves the voxel centre by s sign(u_a) e_a)
          double u[3], sdf0 = 0.0;
          const double inv_l = rL;
          for (int a = 0; a < 3; ++a) {
            u[a] = d[a] * inv_l;
            const double c = ((double)(rec.A[a] >> 16) + 0.5) * p.s;
            sdf0 += (pw[a] - c) * u[a];
            rec.U[a] = __double2ll_rn(fabs(u[a]) * p.s * p.sdf_scale);
          }
          rec.S0 = __double2ll_rn(sdf0 * p.sdf_scale);
          if (rec.S0 >= (1ll << 49) || rec.S0 < -(1ll << 49)) status = 3;   // (|sdf| / tau < 2^14: never)
        }
        if (p.weighting == 0) rec.w = 1.0f;                  // O6
        else { const float r = (float)fmax(L, p.rfloor); rec.w = __frcp_rn(r * r); }
        rec.n_vox = 1;
        for (int a = 0; a < 3; ++a) {
          long long dv = (rec.B[a] >> 16) - (rec.A[a] >> 16);
          rec.n_vox += (int)(dv < 0 ? -dv : dv);             // a2: n_r = 1 + sum |dv| (O4)
        }
        rec.list_off = -1;
        rec.rgb = 0u;
        if (p.rgb) {
          const unsigned char* c = p.rgb + 3 * src;
          rec.rgb = (unsigned)c[0] | ((unsigned)c[1] << 8) | ((unsigned)c[2] << 16);
        }
      }
    }
  }
  // Local counters combined hierarchically ("each thread or block maintains its local
  // counter, and the results are combined at the end"): warp ballots/reductions, a shared-memory scan
  // over the CTA's warps, then ONE 64-bit atomicAdd per CTA claims both the compacted ray positions
  // and the block-slot list space — no hot global counter per warp.
  __shared__ unsigned long long s_base;
  __shared__ unsigned s_w[8][7];   // per warp: used, slots, in, invalid, range, domain, voxels
  __shared__ int s_box[8][6];      // per warp: block box of its used rays (dense-window path)
  const int warp = threadIdx.x >> 5;
  if (p.box) {   // R19: the block box of every voxel the launch's rays traverse = that of the blocks of A and B
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int lo = 0x7fffffff, hi = (int)0x80000000;
      if (status == 0) {
        const int ba = (int)(rec.A[a] >> 19), bb = (int)(rec.B[a] >> 19);
        lo = min(ba, bb); hi = max(ba, bb);
      }
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      if (lane == 0) { s_box[warp][a] = lo; s_box[warp][3 + a] = hi; }
    }
  }
  const unsigned used = __ballot_sync(0xffffffffu, status == 0);
  int nb = 0;                      // block-slot list length: closed form 1 + sum |db| (a2)
  if (status == 0) {
    nb = 1;
    for (int a = 0; a < 3; ++a) {
      long long db = (rec.B[a] >> 19) - (rec.A[a] >> 19);
      nb += (int)(db < 0 ? -db : db);
    }
  }
  int incl = nb;
  for (int o = 1; o < 32; o <<= 1) { int t = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += t; }
  const unsigned nv = __reduce_add_sync(0xffffffffu, status == 0 ? (unsigned)rec.n_vox : 0u);
  const unsigned n_in = __popc(__ballot_sync(0xffffffffu, status >= 0));
  const unsigned n_inv = __popc(__ballot_sync(0xffffffffu, status == 1));
  const unsigned n_rng = __popc(__ballot_sync(0xffffffffu, status == 2));
  const unsigned n_dom = __popc(__ballot_sync(0xffffffffu, status == 3));
  if (lane == 31) {
    s_w[warp][0] = __popc(used); s_w[warp][1] = (unsigned)incl; s_w[warp][2] = n_in; s_w[warp][3] = n_inv;
    s_w[warp][4] = n_rng; s_w[warp][5] = n_dom; s_w[warp][6] = nv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c[7] = {0, 0, 0, 0, 0, 0, 0};
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w)
      for (int t = 0; t < 7; ++t) {
        const unsigned x = s_w[w][t];
        if (t < 2) s_w[w][t] = (unsigned)c[t];   // exclusive prefix of rays / slots
        c[t] += x;
      }
    unsigned long long base = 0;
    if (p.cstat) {
      // single-pass decoupled look-back: the CTA's rays / slots are placed after those of every lower CTA,
      // so the records keep the input order (consecutive patches stay adjacent for the walk's warps)
      constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1, kRayM = (1ull << 25) - 1;
      const unsigned long long agg = (c[1] << 25) | c[0];        // slots : 37 | rays : 25
      unsigned long long excl = 0;
      if (blockIdx.x > 0) {
        atomicExch(&p.cstat[blockIdx.x], kAgg | agg);
        for (long long j = (long long)blockIdx.x - 1;;) {
          const unsigned long long v = *(volatile unsigned long long*)&p.cstat[j];
          if (v == 0ull) continue;                                // not yet published
          excl += v & kVal;
          if (v & kInc) break;
          --j;
        }
      }
      const unsigned long long inc = excl + agg;
      atomicExch(&p.cstat[blockIdx.x], kInc | inc);
      atomicMax(&p.lcnt[0], (int)(inc & kRayM));
      atomicMax(&p.lcnt[1], (int)(inc >> 25));
      base = ((excl >> 25) << 32) | (excl & kRayM);
    } else if (c[0] | c[1]) {
      base = atomicAdd(reinterpret_cast<unsigned long long*>(p.lcnt), (c[1] << 32) | c[0]);
    }
    s_base = base;
    if (c[2]) atomicAdd(&p.ctr->rays_in, c[2]);
    if (c[0]) atomicAdd(&p.ctr->rays_used, c[0]);
    if (c[3]) atomicAdd(&p.ctr->skipped_invalid, c[3]);
    if (c[4]) atomicAdd(&p.ctr->skipped_range, c[4]);
    if (c[5]) { atomicAdd(&p.ctr->skipped_domain, c[5]); atomicOr(&p.ctr->err, (unsigned)kErrRange); }
    if (c[6] && p.count_vox) atomicAdd(&p.ctr->voxel_updates, c[6]);
  }
  if (p.box && threadIdx.x < 6) {   // the CTA's box component -> its slot (box_reduce_kernel combines them)
    const int a = threadIdx.x;
    int v = a < 3 ? 0x7fffffff : (int)0x80000000;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = a < 3 ? min(v, s_box[w][a]) : max(v, s_box[w][a]);
    p.box[6ll * blockIdx.x + a] = v;
  }
  __syncthreads();
  if (status == 0) {
    const long long off = (long long)(unsigned)(s_base >> 32) + s_w[warp][1] + incl - nb;
    rec.list_off = (off + nb <= p.list_cap) ? (int)off : -1;   // full buffer: the walk hashes instead
    const int pos = (int)(unsigned)(s_base & 0xffffffffu) + (int)s_w[warp][0] + __popc(used & ((1u << lane) - 1u));
    RayRec out;
    const double* T = p.frame_T + kFrameRec * f_used;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      out.dA[a] = (int)(rec.A[a] - __double_as_longlong(T[12 + a]));
      out.dB[a] = (int)(rec.B[a] - rec.A[a]);
      out.U[a] = (unsigned)min((rec.U[a] + (1ll << (kUShift - 1))) >> kUShift, 0xffffffffll);
    }
    out.S0f = (long long)((unsigned long long)rec.S0 << kFrameBits) | (long long)f_used;
    out.list_off = rec.list_off;
    p.rays[pos] = out;
    if (p.rgbs) p.rgbs[pos] = rec.rgb;
    if (p.ws) p.ws[pos] = rec.w;
  }
}

#ifndef CVX_RAY_LDCS
#define CVX_RAY_LDCS 0   // 1: evict-first loads of the ray records in the walk (measured neutral)
#endif
struct WalkParams {
  const RayRec* rays;
  const double* frame_T;   // compose_kernel records of the launch's frames (ray origins)
  const unsigned* rgbs;    // nullable: per ray colour (TSDF + Color)
  const float* ws;         // nullable: per ray weight (weighting != 0)
  int frame_base;          // projection mapping: call-relative index of the launch's first frame
  Counters* ctr;
  HashView hash;
  PoolView pool;
  int* slots;       // block-slot lists
  const int* lcnt;  // {n_rays, n_slots} of this launch
  float s, tau;
  int tq;           // round(tau 2^q): the clamp bound (and packed offset) of the quantised sdf
  int q;            // sdf quantum 2^-q m
  long long band;   // colour band |S| < band, S in the fixed-point sdf units 2^-(q+kSdfF) m (= tau)
  int* birth;       // projection mapping: per slot, first frame (RayRec::rgb) whose rays touch the block
  // dense-window path (R19): accumulators over the launch's block box, block-major; nullable dbox = off
  unsigned long long* dacc;
  const int* dbox;  // {lo[3], hi[3]} written by prepare_kernel
  long long dcap;   // capacity of dacc in blocks (excluding the trash region)
  unsigned char* dflag;   // per dense block: touched by the walk (cleared by dense_fold_kernel)
  unsigned long long* dcacc;   // TSDF + Color: dense packed colour accumulators (2 per voxel), nullable
  int* acc_dirty;   // set when a dense-eligible launch falls back to the pool accumulators
};

// R19: dims of the dense window of the launch; false if it does not fit the buffer (the launch then takes
// the slot-list path: block walk + walk_cw_kernel + fold_kernel).
__device__ __forceinline__ bool dense_dims(const int* box, long long cap, int& nbx, int& nby, int& nbz) {
  nbx = box[3] - box[0] + 1; nby = box[4] - box[1] + 1; nbz = box[5] - box[2] + 1;
  if (nbx <= 0 || nby <= 0 || nbz <= 0) { nbx = nby = nbz = 0; return true; }   // no used ray
  return (long long)nbx * nby * nbz <= cap;
}

__device__ __forceinline__ RayView load_ray(const WalkParams& p, int idx) {
#if CVX_RAY_LDCS
  // ray records are read once: streaming (evict-first) loads keep them from evicting the walk's hot
  // accumulator lines in L2
  RayRec r;
  {
    const int4* src = reinterpret_cast<const int4*>(p.rays + idx);
    int4* dst = reinterpret_cast<int4*>(&r);
    dst[0] = __ldcs(src); dst[1] = __ldcs(src + 1); dst[2] = __ldcs(src + 2);
  }
#else
  const RayRec r = p.rays[idx];
#endif
  RayView v;
  v.frame = (int)(r.S0f & ((1ll << kFrameBits) - 1));
  const double* T = p.frame_T + kFrameRec * v.frame;
  v.n_vox = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    v.A[a] = __double_as_longlong(T[12 + a]) + r.dA[a];
    v.B[a] = v.A[a] + r.dB[a];
    v.U[a] = (long long)r.U[a] << kUShift;
    const long long dv = (v.B[a] >> 16) - (v.A[a] >> 16);
    v.n_vox += (int)(dv < 0 ? -dv : dv);                 // a2: n_r = 1 + sum |dv| (O4)
  }
  v.S0 = r.S0f >> kFrameBits;
  v.list_off = r.list_off;
  v.w = p.ws ? p.ws[idx] : 1.0f;
  v.rgb = p.rgbs ? p.rgbs[idx] : 0u;
  return v;
}

// Segmented sum over lanes with equal `peers` groups (log-depth shuffle tree); result valid at the
// lowest lane of each group.  All lanes of `m` must call it.
__device__ __forceinline__ void reduce_peers(unsigned m, unsigned peers, int lane, long long& a, long long& b) {
  int rel = __popc(peers & ((1u << lane) - 1u));
  unsigned above = peers & (0xfffffffeu << lane);
  while (__any_sync(m, above != 0u)) {
    int next = __ffs(above);
    long long ta = __shfl_sync(m, a, next ? next - 1 : lane);
    long long tb = __shfl_sync(m, b, next ? next - 1 : lane);
    if (next) { a += ta; b += tb; }
    unsigned done = __ballot_sync(m, rel & 1);
    above &= ~done;
    rel >>= 1;
  }
}

// ALLOCATE (a3): block-granular exact traversal (boundaries every 2^19 fixed-point units = 8 voxels),
// activating every block a ray visits and recording its slot in the ray's list.  Same predicated
// difference-form DDA as the voxel walk.  The loop is warp-uniform; in each step only the first lane
// of every run of equal keys among adjacent lanes (adjacent rays) probes the hash table and the slot
// is shuffled to the rest of the run.
template <bool k32>   // 32-bit crossing-order differences, as in walk_kernel (unit 2^19 instead of 2^16)
__global__ void __launch_bounds__(256) block_walk_kernel(const __grid_constant__ WalkParams p) {
  using DT = typename std::conditional<k32, unsigned, unsigned long long>::type;
  using ST = typename std::conditional<k32, int, long long>::type;
  const int n_rays = p.lcnt[0];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((idx & ~31) >= n_rays) return;
  const bool have = idx < n_rays;
  int b0 = 0, b1 = 0, b2 = 0, s0 = 1, s1 = 1, s2 = 1, k0 = 0, k1 = 0, k2 = 0, nb = 0;
  DT D01 = 0, D02 = 0, D12 = 0, I0 = 0, I1 = 0, I2 = 0;
  int* list = nullptr;
  if (have) {
    const RayView r = load_ray(p, idx);
    long long R[3], AD[3];
    int bb[3], st[3], kk[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      bb[a] = (int)(r.A[a] >> 19);
      const int be = (int)(r.B[a] >> 19);
      const long long D = r.B[a] - r.A[a];
      kk[a] = be > bb[a] ? be - bb[a] : bb[a] - be;
      if (D > 0) { st[a] = 1; R[a] = (((long long)bb[a] + 1) << 19) - r.A[a]; }
      else { st[a] = -1; R[a] = r.A[a] - ((long long)bb[a] << 19); }
      AD[a] = D < 0 ? -D : D;
    }
    b0 = bb[0]; b1 = bb[1]; b2 = bb[2]; s0 = st[0]; s1 = st[1]; s2 = st[2]; k0 = kk[0]; k1 = kk[1]; k2 = kk[2];
    nb = 1 + k0 + k1 + k2;
    const long long C01 = R[0] * AD[1] - R[1] * AD[0];
    const long long C02 = R[0] * AD[2] - R[2] * AD[0];
    const long long C12 = R[1] * AD[2] - R[2] * AD[1];
    if (k32) {
      D01 = (DT)(-((-C01) >> 19)); D02 = (DT)(-((-C02) >> 19)); D12 = (DT)(-((-C12) >> 19));
      I0 = (DT)AD[0]; I1 = (DT)AD[1]; I2 = (DT)AD[2];
    } else {
      D01 = (DT)C01; D02 = (DT)C02; D12 = (DT)C12;
      I0 = (DT)(AD[0] << 19); I1 = (DT)(AD[1] << 19); I2 = (DT)(AD[2] << 19);
    }
    list = r.list_off >= 0 ? p.slots + r.list_off : nullptr;
  }
  const int maxnb = (int)__reduce_max_sync(0xffffffffu, (unsigned)nb);
  for (int j = 0; j < maxnb; ++j) {
    const bool act = j < nb;
    const unsigned long long key = act ? pack_key(b0, b1, b2) : ((1ull << 63) | (unsigned)lane);
    const unsigned long long prev = __shfl_up_sync(0xffffffffu, key, 1);
    const unsigned actm = __ballot_sync(0xffffffffu, act);
    const unsigned same = __ballot_sync(0xffffffffu, act && prev == key) & (actm << 1);
    const unsigned heads = actm & ~same;
    int slot = kFailed;
    if ((heads >> lane) & 1u) slot = hash_activate(p.hash, p.pool, p.ctr, key, b0, b1, b2);
    const unsigned hb = heads & (0xffffffffu >> (31 - lane));
    slot = __shfl_sync(0xffffffffu, slot, hb ? 31 - __clz(hb) : lane);
    if (act && list) list[j] = slot;
    // O4 at block granularity: earliest crossing among axes with crossings left, ties x < y < z
    const bool stp = j + 1 < nb;
    const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
    const bool yf = g1 & (!g0 | ((ST)D01 > 0));
    const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
    const bool bz = stp & zf, by = stp & yf & !zf, bx = stp & !yf & !zf;
    if (bx) { b0 += s0; --k0; D01 += I1; D02 += I2; }
    if (by) { b1 += s1; --k1; D01 -= I0; D12 += I2; }
    if (bz) { b2 += s2; --k2; D02 -= I0; D12 -= I1; }
  }
}

// Software-pipelined ALLOCATE: the hash entry of step j+1 is loaded (by the run heads of step j+1)
// before step j's probe is consumed, so the L2 latency of one probe overlaps the DDA and list write of
// the previous one.  Same decisions and results as block_walk_kernel.
__device__ __forceinline__ int key_field(unsigned long long key, int sh) {
  return ((int)((key >> sh) & 0x1fffffu) << 11) >> 11;          // 21-bit two's complement (pack_key)
}

// kGrid: the run heads read the dense slot cache (R15) instead of the hash entry for blocks inside its
// window; a cache miss activates through the hash (deduplicated across the run, as every probe here)
// and caches the slot.
template <bool k32, bool kBirth = false, bool kGrid = false>
__device__ __forceinline__ void block_walk2_body(const WalkParams& p, const int idx) {
  using DT = typename std::conditional<k32, unsigned, unsigned long long>::type;
  using ST = typename std::conditional<k32, int, long long>::type;
  const int n_rays = p.lcnt[0];
  const int lane = threadIdx.x & 31;
  if ((idx & ~31) >= n_rays) return;
  const bool have = idx < n_rays;
  int b0 = 0, b1 = 0, b2 = 0, s0 = 1, s1 = 1, s2 = 1, k0 = 0, k1 = 0, k2 = 0, nb = 0;
  DT D01 = 0, D02 = 0, D12 = 0, I0 = 0, I1 = 0, I2 = 0;
  int* list = nullptr;
  int frame = 0x7fffffff;
  if (have) {
    const RayView r = load_ray(p, idx);
    if (kBirth) frame = p.frame_base + r.frame;
    long long R[3], AD[3];
    int bb[3], st[3], kk[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      bb[a] = (int)(r.A[a] >> 19);
      const int be = (int)(r.B[a] >> 19);
      const long long D = r.B[a] - r.A[a];
      kk[a] = be > bb[a] ? be - bb[a] : bb[a] - be;
      if (D > 0) { st[a] = 1; R[a] = (((long long)bb[a] + 1) << 19) - r.A[a]; }
      else { st[a] = -1; R[a] = r.A[a] - ((long long)bb[a] << 19); }
      AD[a] = D < 0 ? -D : D;
    }
    b0 = bb[0]; b1 = bb[1]; b2 = bb[2]; s0 = st[0]; s1 = st[1]; s2 = st[2]; k0 = kk[0]; k1 = kk[1]; k2 = kk[2];
    nb = 1 + k0 + k1 + k2;
    const long long C01 = R[0] * AD[1] - R[1] * AD[0];
    const long long C02 = R[0] * AD[2] - R[2] * AD[0];
    const long long C12 = R[1] * AD[2] - R[2] * AD[1];
    if (k32) {
      D01 = (DT)(-((-C01) >> 19)); D02 = (DT)(-((-C02) >> 19)); D12 = (DT)(-((-C12) >> 19));
      I0 = (DT)AD[0]; I1 = (DT)AD[1]; I2 = (DT)AD[2];
    } else {
      D01 = (DT)C01; D02 = (DT)C02; D12 = (DT)C12;
      I0 = (DT)(AD[0] << 19); I1 = (DT)(AD[1] << 19); I2 = (DT)(AD[2] << 19);
    }
    list = r.list_off >= 0 ? p.slots + r.list_off : nullptr;
  }
  const int maxnb = (int)__reduce_max_sync(0xffffffffu, (unsigned)nb);
  // run heads of step j: first lane of every run of equal keys among adjacent active lanes
  auto heads_of = [&](bool act, unsigned long long key) -> unsigned {
    const unsigned long long prev = __shfl_up_sync(0xffffffffu, key, 1);
    const unsigned actm = __ballot_sync(0xffffffffu, act);
    const unsigned same = __ballot_sync(0xffffffffu, act && prev == key) & (actm << 1);
    return actm & ~same;
  };
  bool act = 0 < nb;
  unsigned long long key = act ? pack_key(b0, b1, b2) : ((1ull << 63) | (unsigned)lane);
  unsigned heads = heads_of(act, key);
  longlong2 ent = make_longlong2(0, 0);
  int gi = -1;   // kGrid: cache index of the head's block (-1: outside the window -> hash entry)
  auto probe = [&](unsigned long long k, int bx, int by, int bz, int& g) -> longlong2 {
    if (kGrid) {
      g = grid_cache_index(bx, by, bz);
      if (g >= 0) return make_longlong2((long long)k, (long long)(unsigned)p.pool.grid[g]);
    }
    return ld_entry(p.hash.e + hash_slot(k, p.hash));
  };
  if ((heads >> lane) & 1u) ent = probe(key, b0, b1, b2, gi);
  for (int j = 0; j < maxnb; ++j) {
    // advance the DDA to step j+1 (independent of the probe of step j)
    const bool stp = j + 1 < nb;
    const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
    const bool yf = g1 & (!g0 | ((ST)D01 > 0));
    const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
    const bool bz = stp & zf, by = stp & yf & !zf, bx = stp & !yf & !zf;
    if (bx) { b0 += s0; --k0; D01 += I1; D02 += I2; }
    if (by) { b1 += s1; --k1; D01 -= I0; D12 += I2; }
    if (bz) { b2 += s2; --k2; D02 -= I0; D12 -= I1; }
    const bool actn = stp;
    const unsigned long long keyn = actn ? pack_key(b0, b1, b2) : ((1ull << 63) | (unsigned)lane);
    const unsigned headsn = (j + 1 < maxnb) ? heads_of(actn, keyn) : 0u;
    longlong2 entn = make_longlong2(0, 0);
    int gin = -1;
    if ((headsn >> lane) & 1u) entn = probe(keyn, b0, b1, b2, gin);   // prefetch j+1
    // consume step j
    int slot = kFailed;
    if ((heads >> lane) & 1u) {   // hit on the prefetched entry: done; else the full activate (insert / probe / wait)
      slot = (int)(ent.y & 0xffffffffll);
      if ((unsigned long long)ent.x != key || slot < 0) {
        if (kGrid && gi >= 0) {
          slot = hash_activate(p.hash, p.pool, p.ctr, key, key_field(key, 42), key_field(key, 21), key_field(key, 0));
          if (slot >= 0) p.pool.grid[gi] = slot;
        } else {
          slot = hash_activate_pf(p.hash, p.pool, p.ctr, key, key_field(key, 42), key_field(key, 21), key_field(key, 0), ent);
        }
      }
    }
    const unsigned hb = heads & (0xffffffffu >> (31 - lane));
    slot = __shfl_sync(0xffffffffu, slot, hb ? 31 - __clz(hb) : lane);
    if (act && list) list[j] = slot;
    if (kBirth) {   // birth frame = min frame over the rays touching the block (one RED per run if uniform)
      const int fmin = __reduce_min_sync(0xffffffffu, act ? frame : 0x7fffffff);
      const int fmax = __reduce_max_sync(0xffffffffu, act ? frame : -1);
      const bool mine = fmin == fmax ? ((heads >> lane) & 1u) != 0u : act;
      // birth only decreases during a call, so a stale (L1) read is >= the true value: skipping when it is
      // already <= frame is exact, and it keeps hot blocks (near the sensor) free of same-address REDs
      if (mine && slot >= 0 && p.birth[slot] > frame) atomicMin(p.birth + slot, frame);
    }
    act = actn; key = keyn; heads = headsn; ent = entn; gi = gin;
  }
}

// Grid-stride over the rays (the dense-window path launches it with a small grid: usually a no-op)
template <bool k32, bool kBirth = false, bool kGrid = false>
__global__ void __launch_bounds__(256) block_walk2_kernel(const __grid_constant__ WalkParams p) {
  if (p.dbox) { int a, b, c; if (dense_dims(p.dbox, p.dcap, a, b, c)) return; }   // R19: the dense window runs
  const long long n = p.lcnt[0];
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += (long long)gridDim.x * blockDim.x)
    block_walk2_body<k32, kBirth, kGrid>(p, (int)(base + threadIdx.x));
}

// ALLOCATE through the dense slot cache (default): every lane walks its own ray at block granularity (no
// lockstep, no shuffles) and reads the slot of each block from the cache, the entry of step j+1 loaded
// before step j's is consumed; only an unknown block (-1) or one outside the cache window goes through
// hash_activate (insert-if-absent + slot bump), and its slot is then cached.  Same block
// sets and slot lists as block_walk2_kernel (the slots are the hash's).
#ifndef CVX_GRID_LD
#define CVX_GRID_LD(ptr) (*(ptr))   // L1-cacheable: a stale -1 only takes the hash path
#endif
#ifndef CVX_BW3_MINB
#define CVX_BW3_MINB 1
#endif
// the rare miss path out of line: the walk loop keeps few registers (more resident warps hide the cache
// entry's L2 latency)
__device__ __noinline__ int activate_cached(const WalkParams& p, int c0, int c1, int c2, int cgi) {
  const int slot = hash_activate(p.hash, p.pool, p.ctr, pack_key(c0, c1, c2), c0, c1, c2);
  if (slot >= 0 && cgi >= 0) p.pool.grid[cgi] = slot;
  return slot;
}
template <bool k32>
__global__ void __launch_bounds__(256, CVX_BW3_MINB) block_walk3_kernel(const __grid_constant__ WalkParams p) {
  using DT = typename std::conditional<k32, unsigned, unsigned long long>::type;
  using ST = typename std::conditional<k32, int, long long>::type;
  const int n_rays = p.lcnt[0];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rays) return;
  const RayView r = load_ray(p, idx);
  long long R[3], AD[3];
  int bb[3], st[3], kk[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bb[a] = (int)(r.A[a] >> 19);
    const int be = (int)(r.B[a] >> 19);
    const long long D = r.B[a] - r.A[a];
    kk[a] = be > bb[a] ? be - bb[a] : bb[a] - be;
    if (D > 0) { st[a] = 1; R[a] = (((long long)bb[a] + 1) << 19) - r.A[a]; }
    else { st[a] = -1; R[a] = r.A[a] - ((long long)bb[a] << 19); }
    AD[a] = D < 0 ? -D : D;
  }
  int b0 = bb[0], b1 = bb[1], b2 = bb[2], k0 = kk[0], k1 = kk[1], k2 = kk[2];
  const int s0 = st[0], s1 = st[1], s2 = st[2];
  const int nb = 1 + k0 + k1 + k2;
  DT D01, D02, D12, I0, I1, I2;
  {
    const long long C01 = R[0] * AD[1] - R[1] * AD[0];
    const long long C02 = R[0] * AD[2] - R[2] * AD[0];
    const long long C12 = R[1] * AD[2] - R[2] * AD[1];
    if (k32) {
      D01 = (DT)(-((-C01) >> 19)); D02 = (DT)(-((-C02) >> 19)); D12 = (DT)(-((-C12) >> 19));
      I0 = (DT)AD[0]; I1 = (DT)AD[1]; I2 = (DT)AD[2];
    } else {
      D01 = (DT)C01; D02 = (DT)C02; D12 = (DT)C12;
      I0 = (DT)(AD[0] << 19); I1 = (DT)(AD[1] << 19); I2 = (DT)(AD[2] << 19);
    }
  }
  int* const list = r.list_off >= 0 ? p.slots + r.list_off : nullptr;
  const int* const grid = p.pool.grid;
#if CVX_BW3_AHEAD2
  // entries of steps j+1 and j+2 in flight while step j is consumed
  auto adv = [&]() {
    const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
    const bool yf = g1 & (!g0 | ((ST)D01 > 0));
    const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
    if (zf) { b2 += s2; --k2; D02 -= I0; D12 -= I1; }
    else if (yf) { b1 += s1; --k1; D01 -= I0; D12 += I2; }
    else { b0 += s0; --k0; D01 += I1; D02 += I2; }
  };
  int c0 = b0, c1 = b1, c2 = b2, cgi = grid_cache_index(b0, b1, b2);
  int ent = cgi >= 0 ? CVX_GRID_LD(grid + cgi) : -1;
  int n0 = 0, n1 = 0, n2 = 0, ngi = -1, entn = -1;
  if (nb > 1) {
    adv();
    n0 = b0; n1 = b1; n2 = b2; ngi = grid_cache_index(b0, b1, b2);
    entn = ngi >= 0 ? CVX_GRID_LD(grid + ngi) : -1;
  }
  for (int j = 0; j < nb; ++j) {
    int ent2 = -1, gi2 = -1;
    if (j + 2 < nb) {
      adv();
      gi2 = grid_cache_index(b0, b1, b2);
      if (gi2 >= 0) ent2 = CVX_GRID_LD(grid + gi2);
    }
    int slot = ent;
    if (slot < 0) {
      slot = hash_activate(p.hash, p.pool, p.ctr, pack_key(c0, c1, c2), c0, c1, c2);
      if (slot >= 0 && cgi >= 0) p.pool.grid[cgi] = slot;
    }
    if (list) list[j] = slot;
    c0 = n0; c1 = n1; c2 = n2; cgi = ngi; ent = entn;
    n0 = b0; n1 = b1; n2 = b2; ngi = gi2; entn = ent2;
  }
#else
  int gi = grid_cache_index(b0, b1, b2);
  int ent = gi >= 0 ? CVX_GRID_LD(grid + gi) : -1;
  for (int j = 0; j < nb; ++j) {
    const int c0 = b0, c1 = b1, c2 = b2, cgi = gi;
    // advance the DDA to step j + 1 (O4 at block granularity: earliest crossing, ties x < y < z) and
    // load its cache entry before consuming step j's
    int entn = -1;
    if (j + 1 < nb) {
      const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
      const bool yf = g1 & (!g0 | ((ST)D01 > 0));
      const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
      if (zf) { b2 += s2; --k2; D02 -= I0; D12 -= I1; }
      else if (yf) { b1 += s1; --k1; D01 -= I0; D12 += I2; }
      else { b0 += s0; --k0; D01 += I1; D02 += I2; }
      gi = grid_cache_index(b0, b1, b2);
      if (gi >= 0) entn = CVX_GRID_LD(grid + gi);
    }
    const int slot = ent >= 0 ? ent : activate_cached(p, c0, c1, c2, cgi);
    if (list) list[j] = slot;
    ent = entn;
  }
#endif
}

// k32: the crossing-order differences fit 32 bits.  With r_i = rho_i + m_i 2^16 (m_i crossings done),
// E_ij = X_ij - X_ji = C_ij + 2^16 F_ij with C_ij = rho_i a_j - rho_j a_i and F_ij = m_i a_j - m_j a_i, so
// E_ij > 0  <=>  H_ij = F_ij - floor(-C_ij / 2^16) > 0; H_ij moves by a_j / -a_i per step like E_ij by
// 2^16 a_j / -2^16 a_i, and |H_ij| <= 3 max(a) while both axes have crossings left.  Exact whenever
// every |D_a| < 2^28 (spans < 2^12 voxels), which the launch checks from the sensor's max range.
#ifndef CVX_V_MINB
#define CVX_V_MINB 8
#endif
template <bool kAggregate, bool kConstW, bool k32, bool kColor = false>
__global__ void __launch_bounds__(128, CVX_V_MINB) walk_kernel(const __grid_constant__ WalkParams p) {
  using DT = typename std::conditional<k32, unsigned, unsigned long long>::type;
  using ST = typename std::conditional<k32, int, long long>::type;
  const int n_rays = p.lcnt[0];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((idx & ~31) >= n_rays) return;                       // whole warp beyond the rays
  const bool have = idx < n_rays;

  // DDA state (O4).  With X_ij = r_i |D_j|, axis i crosses before axis j <=> X_ij < X_ji; only the
  // three differences D01 = X01 - X10, D02 = X02 - X20, D12 = X12 - X21 are kept (exact int64).
  int v0 = 0, v1 = 0, v2 = 0, s0 = 1, s1 = 1, s2 = 1, k0 = 0, k1 = 0, k2 = 0, c0 = 0, c1 = 0, c2 = 0;
  DT D01 = 0, D02 = 0, D12 = 0, I0 = 0, I1 = 0, I2 = 0;   // wrap-around arithmetic, compared signed
  long long S = 0, U0 = 0, U1 = 0, U2 = 0;   // fixed-point sdf of the current voxel and its decrements
  int n = 0, nblk = 0, off = -1;
  unsigned rgb = 0;
  long long w_fx = 0;
  float w = 0.0f;
  if (have) {
    const RayView r = load_ray(p, idx);
    long long R[3], AD[3];
    int va[3], st[3], kk[3];
    nblk = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      va[a] = (int)(r.A[a] >> 16);
      const int vb = (int)(r.B[a] >> 16);
      const long long D = r.B[a] - r.A[a];
      kk[a] = vb > va[a] ? vb - va[a] : va[a] - vb;
      if (D > 0) { st[a] = 1; R[a] = (((long long)va[a] + 1) << 16) - r.A[a]; }
      else { st[a] = -1; R[a] = r.A[a] - ((long long)va[a] << 16); }
      AD[a] = D < 0 ? -D : D;
      const long long db = (r.B[a] >> 19) - (r.A[a] >> 19);
      nblk += (int)(db < 0 ? -db : db);
    }
    v0 = va[0]; v1 = va[1]; v2 = va[2]; s0 = st[0]; s1 = st[1]; s2 = st[2]; k0 = kk[0]; k1 = kk[1]; k2 = kk[2];
    c0 = s0 > 0 ? 0 : 7; c1 = s1 > 0 ? 0 : 7; c2 = s2 > 0 ? 0 : 7;   // local coordinate on block entry
    const long long C01 = R[0] * AD[1] - R[1] * AD[0];
    const long long C02 = R[0] * AD[2] - R[2] * AD[0];
    const long long C12 = R[1] * AD[2] - R[2] * AD[1];
    if (k32) {
      D01 = (DT)(-((-C01) >> 16)); D02 = (DT)(-((-C02) >> 16)); D12 = (DT)(-((-C12) >> 16));
      I0 = (DT)AD[0]; I1 = (DT)AD[1]; I2 = (DT)AD[2];
    } else {
      D01 = (DT)C01; D02 = (DT)C02; D12 = (DT)C12;
      I0 = (DT)(AD[0] << 16); I1 = (DT)(AD[1] << 16); I2 = (DT)(AD[2] << 16);
    }
    // S carries the rounding half and the clamp offset tq: dq + tq = clamp(S >> kSdfF, 0, 2 tq)
    S = r.S0 + (1ll << (kSdfF - 1)) + ((long long)p.tq << kSdfF);
    U0 = r.U[0]; U1 = r.U[1]; U2 = r.U[2];
    w = r.w;
    w_fx = __double2ll_rn((double)w * kFxScale);
    n = r.n_vox;
    off = r.list_off;
    rgb = r.rgb;
  }
  const int maxn = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
  const int* list = off >= 0 ? p.slots + off : nullptr;
  int slot = kFailed, nslot = kFailed, j = 0;
  if (have) {
    slot = list ? __ldg(list) : hash_find(p.hash, pack_key(v0 >> 3, v1 >> 3, v2 >> 3));
    if (list && nblk > 1) nslot = __ldg(list + 1);
  }
  const int tq = p.tq;
  const long long s_off = (1ll << (kSdfF - 1)) + ((long long)tq << kSdfF);
  const long long band_lo = s_off - p.band, band_hi = s_off + p.band;   // |sdf| < tau (colour, R13)
  unsigned long long* const sums = reinterpret_cast<unsigned long long*>(p.pool.sums);
  unsigned long long* const acc = p.pool.acc;
  for (int it = 0; it < maxn; ++it) {
    const bool upd = it < n && slot >= 0;
    // O5 + Q4: clamped projective sdf, quantised to 2^-q m: dq = clamp(round(sdf 2^q), -tq, tq)
    const int dpi = min(max((int)(S >> kSdfF), 0), 2 * tq);   // round(sdf 2^q) + tq, clamped
    const int dq = dpi - tq;
    const unsigned addr = (unsigned)slot * 512u + (unsigned)((v0 & 7) | ((v1 & 7) << 3) | ((v2 & 7) << 6));
    if (kAggregate && kConstW) {
      // constant weights: one packed 64-bit reduction per run of consecutive lanes with the same
      // (voxel, contribution) into the per-launch accumulator acc = count << 40 | sum(d'), d' = dq + tq
      // in [0, 2 tq] (fold_kernel moves it into the exact sums).  Lanes of a run add the same d', so
      // the run total is len * (1 << 40 | d').  Lanes hold spatially adjacent rays in a serpentine
      // order, so runs capture the rays that share a voxel; no match.any (its cost grows with the
      // number of distinct keys) and no shuffle tree.
      const unsigned dp = (unsigned)dpi;
      const unsigned long long key = ((unsigned long long)addr << 32) | dp;
      const unsigned long long prev = __shfl_up_sync(0xffffffffu, key, 1);
      const unsigned act = __ballot_sync(0xffffffffu, upd);
      // branch-free: lane 0 has no predecessor ((act << 1) >> 0 has bit 0 clear)
      const bool head = upd & (!(((act << 1) >> lane) & 1u) | (prev != key));
      const unsigned stops = __ballot_sync(0xffffffffu, head) | ~act;
      const unsigned above = stops & (0xfffffffeu << lane);
      const unsigned len = (unsigned)__clz(__brev(above)) - (unsigned)lane;
      const unsigned long long val = (unsigned long long)len * ((1ull << kCntShift) | (unsigned long long)dp);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.relaxed.gpu.global.add.u64 [%0], %1;\n\t}"
                   :: "l"(acc + addr), "l"(val), "r"((unsigned)head) : "memory");
    } else {
      long long a = __float2ll_rn(w * (float)dq * __int_as_float((127 + 30 - p.q) << 23));  // w d 2^30
      if (kAggregate) {
        const unsigned long long key = upd ? (unsigned long long)addr : (0x100000000ull | (unsigned)lane);
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        long long b = upd ? w_fx : 0;
        if (!upd) a = 0;
        reduce_peers(0xffffffffu, peers, lane, a, b);
        if (upd && lane == __ffs(peers) - 1) {
          atomicAdd(sums + 2ull * addr, (unsigned long long)a);
          atomicAdd(sums + 2ull * addr + 1, (unsigned long long)b);
        }
      } else if (upd) {
        atomicAdd(sums + 2ull * addr, (unsigned long long)a);
        atomicAdd(sums + 2ull * addr + 1, (unsigned long long)w_fx);
      }
    }
    if (kColor && upd && S > band_lo && S < band_hi) {
      // TSDF + Color (R13): band updates also fuse w (r, g, b); no run merging (neighbouring rays
      // differ in colour near the surface)
      const unsigned long long cr = rgb & 0xffu, cg = (rgb >> 8) & 0xffu, cb = (rgb >> 16) & 0xffu;
      if (kConstW) {
        atomicAdd(p.pool.cacc + 2ull * addr, (1ull << kCntShift) | cr);
        atomicAdd(p.pool.cacc + 2ull * addr + 1, (cg << 32) | cb);
      } else {
        unsigned long long* cs = reinterpret_cast<unsigned long long*>(p.pool.csum) + 4ull * addr;
        atomicAdd(cs, (unsigned long long)w_fx);
        atomicAdd(cs + 1, (unsigned long long)(w_fx * (long long)cr));
        atomicAdd(cs + 2, (unsigned long long)(w_fx * (long long)cg));
        atomicAdd(cs + 3, (unsigned long long)(w_fx * (long long)cb));
      }
    }
    // O4: step the axis with the earliest next crossing among those with crossings left (ties
    // x < y < z), predicated on the lane still having a voxel to go.
    const bool stp = it + 1 < n;
    const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
    const bool yf = g1 & (!g0 | ((ST)D01 > 0));
    const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
    const bool bz = stp & zf, by = stp & yf & !zf, bx = stp & !yf & !zf;
    if (bx) { v0 += s0; --k0; D01 += I1; D02 += I2; S -= U0; }
    if (by) { v1 += s1; --k1; D01 -= I0; D12 += I2; S -= U1; }
    if (bz) { v2 += s2; --k2; D02 -= I0; D12 -= I1; S -= U2; }
    const bool enter = (bx & ((v0 & 7) == c0)) | (by & ((v1 & 7) == c1)) | (bz & ((v2 & 7) == c2));
    if (enter) {                                // entered the next block of the ray
      ++j;
      if (list) {
        slot = nslot;
        if (j + 1 < nblk) nslot = __ldg(list + j + 1);   // prefetch one block ahead
      } else {
        slot = hash_find(p.hash, pack_key(v0 >> 3, v1 >> 3, v2 >> 3));
      }
    }
  }
}

// Predicated read-only load INTO the live register of `dst` (no copy: a plain conditional __ldg makes
// the compiler load into a temporary and move it, which waits for the load right where it is issued —
// ncu showed that move as the walk's top stall).  The value is consumed one block later.
#ifndef CVX_PF_ASM
#define CVX_PF_ASM 2
#endif
__device__ __forceinline__ void prefetch_slot(int& dst, const int* ptr, bool pred) {
#if CVX_PF_ASM
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.u32 %0, [%1];\n\t}"
               : "+r"(dst) : "l"(ptr), "r"((unsigned)pred));
#else
  if (pred) dst = __ldg(ptr);
#endif
}

// CVX_PF_ASM == 2: the next block's slot is prefetched with cp.async into a per-thread shared-memory
// word and read back (after cp.async.wait_all, long complete by then) at the next block entry.
__device__ __forceinline__ void pf_issue(int* sdst, const int* src, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p cp.async.ca.shared.global [%0], [%1], 4;\n\tcp.async.commit_group;\n\t}"
               :: "r"(sa), "l"(src), "r"((unsigned)pred) : "memory");
}
__device__ __forceinline__ void pf_issue_u(int* sdst, const int* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n\tcp.async.commit_group;" :: "r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ int pf_take(const int* sdst) {
#if CVX_WG0
  asm volatile("cp.async.wait_group 0;" ::: "memory");   // every cp.async here is committed at issue
#else
  asm volatile("cp.async.wait_all;" ::: "memory");
#endif
  return *(volatile const int*)sdst;
}

// Length of the run headed by `lane`: distance to the next run head above it (`above` = the heads above
// `lane`), 32 - lane for the last run.  brev + bfind.shiftamt is count-trailing-zeros, 0xffffffff for 0.
#ifndef CVX_RUNLEN_PTX
#define CVX_RUNLEN_PTX 1
#endif
__device__ __forceinline__ unsigned run_len(unsigned above, int lane) {
#if CVX_RUNLEN_PTX
  unsigned r;
  asm("{\n\t.reg .b32 t;\n\tbrev.b32 t, %1;\n\tbfind.shiftamt.u32 %0, t;\n\t}" : "=r"(r) : "r"(above));
  return min(r, 32u) - (unsigned)lane;
#else
  return (unsigned)__clz(__brev(above)) - (unsigned)lane;
#endif
}

// Approximate fp32 reciprocal / reciprocal square root (MUFU only; used for guesses that are checked
// exactly afterwards, so no IEEE slow path is needed).
__device__ __forceinline__ float rcp_approx(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }



// Constant-weight walk with the voxel address carried incrementally (same decisions as walk_kernel
// <true, true, k32, kColor>; see there for O4/O5).  Per step only the stepped axis' crossing count,
// DDA differences, sdf and address move; the voxel coordinates are implied by the remaining crossing
// counts (v = v_B - s k) and rebuilt only on block entry (one step in 8 or fewer per axis).  Block
// entry: the stepped axis' local field of the address reached its entry value.  Only clamped
// free-space updates (d' = 2 tq) are run-merged: in-band sdfs differ between rays at the 2^-q quantum,
// so merging them buys nothing; they go out as single-lane reductions.
// kFuse: ALLOCATE (a3) is done here instead of by block_walk2_kernel — the first block of a ray is
// activated at the start, and on entering each block its hash entry has already been fetched: at every
// block entry the entries of the three axis neighbours of the new block (the next block is one of them:
// the traversal crosses one block face at a time) are copied into shared memory with cp.async, and the
// next entry takes the one on the stepped axis; a hit is the slot, anything else (absent: insert, other
// key: probe on, pending) goes through hash_activate_pf with that entry as its first probe.
template <bool k32, bool kColor, bool kFuse = false>
__device__ __forceinline__ void walk_cw_body(const WalkParams& p, const int idx) {
  using DT = typename std::conditional<k32, unsigned, unsigned long long>::type;
  using ST = typename std::conditional<k32, int, long long>::type;
  const int n_rays = p.lcnt[0];
  const int lane = threadIdx.x & 31;
  if ((idx & ~31) >= n_rays) return;
  const bool have = idx < n_rays;
  int vb0 = 0, vb1 = 0, vb2 = 0, s0 = 1, s1 = 1, s2 = 1, k0 = 0, k1 = 0, k2 = 0;
  DT D01 = 0, D02 = 0, D12 = 0, I0 = 0, I1 = 0, I2 = 0;
  long long S = 0, U0 = 0, U1 = 0, U2 = 0;
  int n = 0, nblk = 0, off = -1;
  unsigned rgb = 0, cexp = 0, addr = 0;
  int v0 = 0, v1 = 0, v2 = 0;
  if (have) {
    const RayView r = load_ray(p, idx);
    long long R[3], AD[3];
    int va[3], vb[3], st[3], kk[3];
    nblk = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      va[a] = (int)(r.A[a] >> 16);
      vb[a] = (int)(r.B[a] >> 16);
      const long long D = r.B[a] - r.A[a];
      kk[a] = vb[a] > va[a] ? vb[a] - va[a] : va[a] - vb[a];
      if (D > 0) { st[a] = 1; R[a] = (((long long)va[a] + 1) << 16) - r.A[a]; }
      else { st[a] = -1; R[a] = r.A[a] - ((long long)va[a] << 16); }
      AD[a] = D < 0 ? -D : D;
      const long long db = (r.B[a] >> 19) - (r.A[a] >> 19);
      nblk += (int)(db < 0 ? -db : db);
    }
    v0 = va[0]; v1 = va[1]; v2 = va[2];
    vb0 = vb[0]; vb1 = vb[1]; vb2 = vb[2];
    s0 = st[0]; s1 = st[1]; s2 = st[2]; k0 = kk[0]; k1 = kk[1]; k2 = kk[2];
    cexp = (s0 > 0 ? 0u : 7u) | ((s1 > 0 ? 0u : 7u) << 3) | ((s2 > 0 ? 0u : 7u) << 6);
    const long long C01 = R[0] * AD[1] - R[1] * AD[0];
    const long long C02 = R[0] * AD[2] - R[2] * AD[0];
    const long long C12 = R[1] * AD[2] - R[2] * AD[1];
    if (k32) {
      D01 = (DT)(-((-C01) >> 16)); D02 = (DT)(-((-C02) >> 16)); D12 = (DT)(-((-C12) >> 16));
      I0 = (DT)AD[0]; I1 = (DT)AD[1]; I2 = (DT)AD[2];
    } else {
      D01 = (DT)C01; D02 = (DT)C02; D12 = (DT)C12;
      I0 = (DT)(AD[0] << 16); I1 = (DT)(AD[1] << 16); I2 = (DT)(AD[2] << 16);
    }
    S = r.S0 + (1ll << (kSdfF - 1)) + ((long long)p.tq << kSdfF);
    U0 = r.U[0]; U1 = r.U[1]; U2 = r.U[2];
    n = r.n_vox;
    off = r.list_off;
    rgb = r.rgb;
  }
  const int maxn = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
  const int* list = off >= 0 ? p.slots + off : nullptr;
  int slot = kFailed, nslot = kFailed, j = 0;
#if CVX_PF_ASM == 2
  __shared__ int s_pf[128];
#endif
  // Blocks without a slot (pool overflow: dropped updates, CVX_E_CAPACITY) and idle lanes address the
  // trash block `max_blocks` of the accumulator (never folded), so no update needs a slot predicate.
  const int trash = p.pool.max_blocks;
  addr = (unsigned)trash * 512u;
  // kFuse: current block coordinates and the prefetched neighbour entries, per thread
  __shared__ int4 s_cb[kFuse ? 128 : 1];
  __shared__ longlong2 s_cand[kFuse ? 3 * 128 : 1];
  auto issue_candidates = [&](const int4 cb) {
    const int sa[3] = {s0, s1, s2};
    const int kk[3] = {k0, k1, k2};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const unsigned long long key = pack_key(cb.x + (a == 0 ? sa[0] : 0), cb.y + (a == 1 ? sa[1] : 0),
                                              cb.z + (a == 2 ? sa[2] : 0));
      const HashEntry* src = p.hash.e + hash_slot(key, p.hash);
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_cand[3 * threadIdx.x + a]);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}"
                   :: "r"(dst), "l"(src), "r"((unsigned)(kk[a] > 0)) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // slot of the block entered by a step along axis ax (kFuse), or from the list / the hash
  auto next_slot = [&](const int ax) -> int {
    if constexpr (kFuse) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      int4 cb = s_cb[threadIdx.x];
      if (ax == 0) cb.x += s0; else if (ax == 1) cb.y += s1; else cb.z += s2;
      const unsigned long long key = pack_key(cb.x, cb.y, cb.z);
      const longlong2 e = s_cand[3 * threadIdx.x + ax];   // complete: cp.async.wait_all above
      int sl = (int)(e.y & 0xffffffffll);
      if ((unsigned long long)e.x != key || sl < 0) sl = hash_activate_pf(p.hash, p.pool, p.ctr, key, cb.x, cb.y, cb.z, e);
      s_cb[threadIdx.x] = cb;
      issue_candidates(cb);
      return CVX_ENTRY2 ? (int)min((unsigned)sl, (unsigned)trash) : sl;
    } else {
      if (off >= 0) {   // == list != nullptr, one 32-bit compare
#if CVX_PF_ASM == 2
        const int sl = pf_take(s_pf + threadIdx.x);
#if CVX_ENTRY2
        pf_issue_u(s_pf + threadIdx.x, list + j + 1);   // one block ahead; past the last block: the spare entry
        return (int)min((unsigned)sl, (unsigned)trash);   // kFailed (< 0) -> trash
#else
        pf_issue(s_pf + threadIdx.x, list + j + 1, j + 1 < nblk);   // prefetch one block ahead
        return sl;
#endif
#else
        const int sl = nslot;
        prefetch_slot(nslot, list + j + 1, CVX_ENTRY2 ? true : j + 1 < nblk);
        return CVX_ENTRY2 ? (int)min((unsigned)sl, (unsigned)trash) : sl;
#endif
      }
      const int sl = hash_find(p.hash, pack_key((vb0 - s0 * k0) >> 3, (vb1 - s1 * k1) >> 3, (vb2 - s2 * k2) >> 3));
      return CVX_ENTRY2 ? (int)min((unsigned)sl, (unsigned)trash) : sl;
    }
  };
  if (have) {
    if constexpr (kFuse) {
      const int4 cb = make_int4(v0 >> 3, v1 >> 3, v2 >> 3, 0);
      slot = hash_activate(p.hash, p.pool, p.ctr, pack_key(cb.x, cb.y, cb.z), cb.x, cb.y, cb.z);
      s_cb[threadIdx.x] = cb;
      issue_candidates(cb);
    } else {
      slot = list ? __ldg(list) : hash_find(p.hash, pack_key(v0 >> 3, v1 >> 3, v2 >> 3));
#if CVX_PF_ASM == 2
      pf_issue(s_pf + threadIdx.x, list + 1, CVX_ENTRY2 ? list != nullptr : (list && nblk > 1));
#else
      if (list && nblk > 1) nslot = __ldg(list + 1);
#endif
    }
    if (slot < 0) slot = trash;
    addr = (unsigned)slot * 512u + (unsigned)((v0 & 7) | ((v1 & 7) << 3) | ((v2 & 7) << 6));
  }
  if (!have) { k0 = 0x3fffffff; s0 = 0; cexp = 1u; }   // parked idle lane (see the free prefix below)
  const int da0 = s0, da1 = 8 * s1, da2 = 64 * s2;
  const int tq2 = 2 * p.tq;
  const long long s_off = (1ll << (kSdfF - 1)) + ((long long)p.tq << kSdfF);
  const long long band_lo = s_off - p.band, band_hi = s_off + p.band;
  unsigned long long* const acc = p.pool.acc;
  // Two phases.  While every lane of the warp is surely in clamped free space (S >= 2 tq 2^kSdfF, so
  // d' = 2 tq), the sdf is not tracked: S_i >= S_0 - i max_a U_a bounds it from the voxel index alone,
  // which gives each ray a free prefix of m voxels (< n).  After the prefix S is rebuilt exactly from
  // the steps taken per axis (S_0 - sum_a U_a (K_a - k_a)) and the full update continues.
  int mfree = 0x7fffffff;
  const int K0 = k0, K1 = k1, K2 = k2;
  if (have) {
    long long thr = (long long)tq2 << kSdfF;
    if (kColor) thr = max(thr, band_hi);
    const long long umax = max(U0, max(U1, U2));
    mfree = 0;
    if (S > thr && umax > 0) {
      // floor((S - thr) / umax), capped at n - 1: fp32 guess, then made exact (no fp64 / int64 division)
      const long long num = S - thr;
      long long m = (long long)fminf((float)num * rcp_approx((float)umax), (float)(n - 1));
      while (m > 0 && m * umax > num) --m;
      while (m < n - 1 && (m + 1) * umax <= num) ++m;
      mfree = (int)m;
    }
  }
  const int mw = (int)__reduce_min_sync(0xffffffffu, (unsigned)mfree);
  // General band step (TSDF + Color: colour sums need the per-lane band test; and CVX_BAND2 = 0): finished
  // lanes (it >= n) are masked instead of parked.
  auto band_body = [&](const int it) {
    const bool upd = it < n;
    const int dpi = min(max((int)(S >> kSdfF), 0), tq2);   // round(sdf 2^q) + tq, clamped (O5, Q4)
    {
      // key 0xffffffff (never an address: < 2^23 slots) = no merging (in-band or finished lane)
      const unsigned key = (upd & (dpi == tq2)) ? addr : 0xffffffffu;
      const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
      const bool head = upd & ((lane == 0) | (prev != key) | (key == 0xffffffffu));
      const unsigned stops = __ballot_sync(0xffffffffu, head | !upd);
      const unsigned len = run_len(stops & (0xfffffffeu << lane), lane);
      // len * (2^40 | dpi) as two 32-bit halves: hi = len << 8, lo = len * dpi (< 2^22, no carry)
      const unsigned long long val = ((unsigned long long)(len << (kCntShift - 32)) << 32) | (len * (unsigned)dpi);
      CVX_CHECK(!head || (long long)addr < ((long long)p.pool.max_blocks + kTrashBlocks) * kBlockVox, "pool accumulator address");
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.relaxed.gpu.global.add.u64 [%0], %1;\n\t}"
                   :: "l"(acc + addr), "l"(val), "r"((unsigned)head) : "memory");
    }
    if (kColor && upd && S > band_lo && S < band_hi) {
      const unsigned long long cr = rgb & 0xffu, cg = (rgb >> 8) & 0xffu, cb = (rgb >> 16) & 0xffu;
      atomicAdd(p.pool.cacc + 2ull * addr, (1ull << kCntShift) | cr);
      atomicAdd(p.pool.cacc + 2ull * addr + 1, (cg << 32) | cb);
    }
    const bool stp = it + 1 < n;
    const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
    const bool yf = g1 & (!g0 | ((ST)D01 > 0));
    const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
    const bool bz = stp & zf, by = stp & yf & !zf, bx = stp & !yf & !zf;
    if (bx) { addr += da0; --k0; D01 += I1; D02 += I2; S -= U0; }
    if (by) { addr += da1; --k1; D01 -= I0; D12 += I2; S -= U1; }
    if (bz) { addr += da2; --k2; D02 -= I0; D12 -= I1; S -= U2; }
    const unsigned m = zf ? 0x1c0u : (yf ? 0x38u : 7u);
    if (stp & (((addr ^ cexp) & m) == 0u)) {      // entered the next block of the ray
      ++j;
      if (list) {
        slot = nslot;
        prefetch_slot(nslot, list + j + 1, j + 1 < nblk);   // prefetch one block ahead
      } else {
        slot = hash_find(p.hash, pack_key((vb0 - s0 * k0) >> 3, (vb1 - s1 * k1) >> 3, (vb2 - s2 * k2) >> 3));
      }
      if (slot < 0) slot = trash;
      const int da = zf ? da2 : (yf ? da1 : da0);
      addr = (unsigned)slot * 512u + ((((addr - (unsigned)da) & 511u) & ~m) | (cexp & m));
    }
  };
  int it = 0;
  // Free prefix, hand-scheduled: every lane (idle lanes parked on the trash block, stepping x by 0 and
  // never meeting a block boundary) updates its voxel with the clamped d' = 2 tq; runs of equal
  // addresses in adjacent lanes issue one reduction of len * (2^40 | 2 tq).
  {
    const unsigned above_mask = 0xfffffffeu << lane;
    const bool lane0 = lane == 0;
    const unsigned utq2 = (unsigned)tq2;
    for (; it < mw; ++it) {
      const unsigned prev = __shfl_up_sync(0xffffffffu, addr, 1);
      const bool head = lane0 | (prev != addr);
      const unsigned stops = __ballot_sync(0xffffffffu, head);
      const unsigned len = run_len(stops & above_mask, lane);
      const unsigned long long val = ((unsigned long long)(len << (kCntShift - 32)) << 32) | (len * utq2);
      CVX_CHECK(!head || (long long)addr < ((long long)p.pool.max_blocks + kTrashBlocks) * kBlockVox, "pool accumulator address");
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.relaxed.gpu.global.add.u64 [%0], %1;\n\t}"
                   :: "l"(acc + addr), "l"(val), "r"((unsigned)head) : "memory");
      const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
      const bool yf = g1 & (!g0 | ((ST)D01 > 0));
      const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
      const bool by = yf & !zf, bx = !yf & !zf;
      if (bx) { addr += da0; --k0; D01 += I1; D02 += I2; }
      if (by) { addr += da1; --k1; D01 -= I0; D12 += I2; }
      if (zf) { addr += da2; --k2; D02 -= I0; D12 -= I1; }
      const unsigned m = zf ? 0x1c0u : (yf ? 0x38u : 7u);
      if (((addr ^ cexp) & m) == 0u) {      // entered the next block of the ray
        ++j;
        slot = next_slot(zf ? 2 : (yf ? 1 : 0));
        if (!CVX_ENTRY2 && slot < 0) slot = trash;
        const int da = zf ? da2 : (yf ? da1 : da0);
#if CVX_ENTRY2
        // the step wrapped the stepped axis' local field (carry / borrow into the next field): -8 da undoes
        // the carry and leaves the field at its entry value; keep the local bits, switch the slot
        addr = ((unsigned)slot << 9) | ((addr - 8u * (unsigned)da) & 511u);
#else
        addr = (unsigned)slot * 512u + ((((addr - (unsigned)da) & 511u) & ~m) | (cexp & m));
#endif
      }
    }
  }
  S -= U0 * (K0 - k0) + U1 * (K1 - k1) + U2 * (K2 - k2);
#if CVX_BAND2
  {
    // Rest of the rays, hand-scheduled like the free prefix: a lane that has written its last voxel
    // parks on its warp's trash spot (x step of 0, never a block boundary, d' = 2 tq forever, outside
    // the colour band) so no update or step needs a per-lane predicate; parked lanes' reductions land
    // in the trash region.
    const unsigned above_mask = 0xfffffffeu << lane;
    const bool lane0 = lane == 0;
    const unsigned spot = (unsigned)trash * 512u + ((((unsigned)idx >> 5) & 4095u) << 3);
    int dx0 = da0;
    if (it >= n) { addr = spot; k0 = 0x3fffffff; k1 = 0; k2 = 0; dx0 = 0; cexp = 1u; S = (long long)tq2 << (kSdfF + 1); U0 = 0; n = 0x7fffffff; }
    for (; it < maxn; ++it) {
      const int dpi = min(max((int)(S >> kSdfF), 0), tq2);   // round(sdf 2^q) + tq, clamped (O5, Q4)
      const unsigned key = dpi == tq2 ? addr : 0xffffffffu;     // only clamped updates merge
      const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
      const bool head = lane0 | (prev != key) | (key == 0xffffffffu);
      const unsigned stops = __ballot_sync(0xffffffffu, head);
      const unsigned len = run_len(stops & above_mask, lane);
      const unsigned long long val = ((unsigned long long)(len << (kCntShift - 32)) << 32) | (len * (unsigned)dpi);
      CVX_CHECK(!head || (long long)addr < ((long long)p.pool.max_blocks + kTrashBlocks) * kBlockVox, "pool accumulator address");
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.relaxed.gpu.global.add.u64 [%0], %1;\n\t}"
                   :: "l"(acc + addr), "l"(val), "r"((unsigned)head) : "memory");
      if (kColor && S > band_lo && S < band_hi) {   // TSDF + Color: band updates carry the point's colour (R13)
        const unsigned long long cr = rgb & 0xffu, cg = (rgb >> 8) & 0xffu, cb = (rgb >> 16) & 0xffu;
        atomicAdd(p.pool.cacc + 2ull * addr, (1ull << kCntShift) | cr);
        atomicAdd(p.pool.cacc + 2ull * addr + 1, (cg << 32) | cb);
      }
      if (it + 1 >= n) {   // that was the ray's last voxel: park
        addr = spot; k0 = 0x3fffffff; k1 = 0; k2 = 0; dx0 = 0; cexp = 1u; S = (long long)tq2 << (kSdfF + 1); U0 = 0;
        n = 0x7fffffff;
      }
      const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
      const bool yf = g1 & (!g0 | ((ST)D01 > 0));
      const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
      const bool by = yf & !zf, bx = !yf & !zf;
      if (bx) { addr += dx0; --k0; D01 += I1; D02 += I2; S -= U0; }
      if (by) { addr += da1; --k1; D01 -= I0; D12 += I2; S -= U1; }
      if (zf) { addr += da2; --k2; D02 -= I0; D12 -= I1; S -= U2; }
      const unsigned m = zf ? 0x1c0u : (yf ? 0x38u : 7u);
      if (((addr ^ cexp) & m) == 0u) {      // entered the next block of the ray
        ++j;
        slot = next_slot(zf ? 2 : (yf ? 1 : 0));
        if (!CVX_ENTRY2 && slot < 0) slot = trash;
        const int da = zf ? da2 : (yf ? da1 : dx0);
#if CVX_ENTRY2
        // the step wrapped the stepped axis' local field (carry / borrow into the next field): -8 da undoes
        // the carry and leaves the field at its entry value; keep the local bits, switch the slot
        addr = ((unsigned)slot << 9) | ((addr - 8u * (unsigned)da) & 511u);
#else
        addr = (unsigned)slot * 512u + ((((addr - (unsigned)da) & 511u) & ~m) | (cexp & m));
#endif
      }
    }
    return;
  }
#endif
#if CVX_PF_ASM == 2
  if (list) nslot = pf_take(s_pf + threadIdx.x);   // the general band body keeps the prefetch in a register
#endif
  for (; it < maxn; ++it) band_body(it);
}

// Grid-stride over the rays (the dense-window path launches it with a small grid: usually a no-op)
template <bool k32, bool kColor, bool kFuse = false>
__global__ void __launch_bounds__(128, CVX_V_MINB) walk_cw_kernel(const __grid_constant__ WalkParams p) {
  if (p.dbox) {   // R19: the dense window runs this launch unless its box exceeds the buffer
    int a, b, c;
    if (dense_dims(p.dbox, p.dcap, a, b, c)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) *p.acc_dirty = 1;   // fold_kernel has work
  }
  const long long n = p.lcnt[0];
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += (long long)gridDim.x * blockDim.x)
    walk_cw_body<k32, kColor, kFuse>(p, (int)(base + threadIdx.x));
}

// R19: the launch's block box = the union of prepare_kernel's per-CTA boxes
__global__ void __launch_bounds__(256) box_reduce_kernel(const int* cta_box, int n, int* box) {
  int v[6] = {0x7fffffff, 0x7fffffff, 0x7fffffff, (int)0x80000000, (int)0x80000000, (int)0x80000000};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 6; ++a) v[a] = a < 3 ? min(v[a], cta_box[6ll * i + a]) : max(v[a], cta_box[6ll * i + a]);
  }
#pragma unroll
  for (int a = 0; a < 6; ++a) v[a] = a < 3 ? __reduce_min_sync(0xffffffffu, v[a]) : __reduce_max_sync(0xffffffffu, v[a]);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) { atomicMin(box + a, v[a]); atomicMax(box + 3 + a, v[3 + a]); }
  }
}

// Dense-window walk (R19; constant weights, no colour): walk_cw_kernel's exact DDA, sdf and run merging,
// with the accumulators of the launch's block box laid out block-major (dense block index
// (bz - lz) nby nbx + (by - ly) nbx + (bx - lx), 512 voxels each).  Entering the next block along axis a is
// then pure arithmetic — the step wrapped the local field of a, -8 da undoes the carry and the block
// stride moves to the neighbour block: addr += s_a (block stride_a - 8 |da_a|) — so the walk has no slot
// lists, no prefetch and no divergent block-entry branch.  ALLOCATE runs afterwards (dense_fold_kernel)
// for the blocks the walk touched.
#ifndef CVX_DW_MINB
#define CVX_DW_MINB CVX_V_MINB
#endif
// timing experiments only (wrong results): CVX_DW_EXP=1 drops the reductions, =2 sends them to 32
// consecutive words per warp (lane-coherent)
#ifndef CVX_DW_EXP
#define CVX_DW_EXP 0
#endif
#if CVX_DW_EXP == 1
#define DW_RED(acc, addr, val, head) do { if ((head) && (addr) == 0xfffffff0u) (acc)[0] = (val); } while (0)
#elif CVX_DW_EXP == 2
#define DW_RED(acc, addr, val, head) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.relaxed.gpu.global.add.u64 [%0], %1;\n\t}" \
                   :: "l"((acc) + (((addr) & ~31u) | (threadIdx.x & 31))), "l"(val), "r"((unsigned)(head)) : "memory")
#else
#define DW_RED(acc, addr, val, head) do { \
    CVX_CHECK(!(head) || (long long)(addr) < (p.dcap + kTrashBlocks) * kBlockVox, "dense accumulator address"); \
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.relaxed.gpu.global.add.u64 [%0], %1;\n\t}" \
                   :: "l"((acc) + (addr)), "l"(val), "r"((unsigned)(head)) : "memory"); } while (0)
#endif
#ifndef CVX_DW_UNIFORM
#define CVX_DW_UNIFORM 0   // 1: free prefix takes a warp-uniform path when no two adjacent lanes share a voxel (measured slower)
#endif
#ifndef CVX_DW_FLAGS
#define CVX_DW_FLAGS 0
#endif
// mark dense block bi as touched: a plain (L1-cached) read first, so blocks already marked (the common case:
// neighbouring rays enter the same blocks) cost no L2 write; a stale 0 only repeats the store
__device__ __forceinline__ void mark_block(unsigned char* flags, unsigned bi, bool pred) {
#if CVX_DW_FLAGS
  if (pred && flags[bi] == 0) flags[bi] = 1;
#endif
}

template <bool k32, bool kColor = false>
__global__ void __launch_bounds__(128, CVX_DW_MINB) walk_dw_kernel(const __grid_constant__ WalkParams p) {
  using DT = typename std::conditional<k32, unsigned, unsigned long long>::type;
  using ST = typename std::conditional<k32, int, long long>::type;
  int nbx, nby, nbz;
  if (!dense_dims(p.dbox, p.dcap, nbx, nby, nbz)) return;   // the slot-list path runs this launch
  const int n_rays = p.lcnt[0];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((idx & ~31) >= n_rays) return;
  const bool have = idx < n_rays;
  // per-warp trash spots after the buffer's capacity (never inside any launch's box, never folded)
  const unsigned trash = (unsigned)(p.dcap * kBlockVox);
  int s0 = 1, s1 = 1, s2 = 1, k0 = 0, k1 = 0, k2 = 0;
  DT D01 = 0, D02 = 0, D12 = 0, I0 = 0, I1 = 0, I2 = 0;
  long long S = 0, U0 = 0, U1 = 0, U2 = 0;
  int n = 0;
  unsigned cexp = 0, addr = trash, rgb = 0;
  if (have) {
    const RayView r = load_ray(p, idx);
    long long R[3], AD[3];
    int va[3], st[3], kk[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      va[a] = (int)(r.A[a] >> 16);
      const int vb = (int)(r.B[a] >> 16);
      const long long D = r.B[a] - r.A[a];
      kk[a] = vb > va[a] ? vb - va[a] : va[a] - vb;
      if (D > 0) { st[a] = 1; R[a] = (((long long)va[a] + 1) << 16) - r.A[a]; }
      else { st[a] = -1; R[a] = r.A[a] - ((long long)va[a] << 16); }
      AD[a] = D < 0 ? -D : D;
    }
    s0 = st[0]; s1 = st[1]; s2 = st[2]; k0 = kk[0]; k1 = kk[1]; k2 = kk[2];
    cexp = (s0 > 0 ? 0u : 7u) | ((s1 > 0 ? 0u : 7u) << 3) | ((s2 > 0 ? 0u : 7u) << 6);
    const long long C01 = R[0] * AD[1] - R[1] * AD[0];
    const long long C02 = R[0] * AD[2] - R[2] * AD[0];
    const long long C12 = R[1] * AD[2] - R[2] * AD[1];
    if (k32) {
      D01 = (DT)(-((-C01) >> 16)); D02 = (DT)(-((-C02) >> 16)); D12 = (DT)(-((-C12) >> 16));
      I0 = (DT)AD[0]; I1 = (DT)AD[1]; I2 = (DT)AD[2];
    } else {
      D01 = (DT)C01; D02 = (DT)C02; D12 = (DT)C12;
      I0 = (DT)(AD[0] << 16); I1 = (DT)(AD[1] << 16); I2 = (DT)(AD[2] << 16);
    }
    S = r.S0 + (1ll << (kSdfF - 1)) + ((long long)p.tq << kSdfF);
    U0 = r.U[0]; U1 = r.U[1]; U2 = r.U[2];
    n = r.n_vox;
    rgb = r.rgb;
    CVX_CHECK((va[0] >> 3) >= p.dbox[0] && (va[0] >> 3) <= p.dbox[3] && (va[1] >> 3) >= p.dbox[1] && (va[1] >> 3) <= p.dbox[4] &&
              (va[2] >> 3) >= p.dbox[2] && (va[2] >> 3) <= p.dbox[5], "ray start inside the launch's block box");
    const unsigned blk = (unsigned)((((va[2] >> 3) - p.dbox[2]) * nby + ((va[1] >> 3) - p.dbox[1])) * nbx + ((va[0] >> 3) - p.dbox[0]));
    addr = blk * 512u + (unsigned)((va[0] & 7) | ((va[1] & 7) << 3) | ((va[2] & 7) << 6));
    mark_block(p.dflag, blk, true);
  }
  const int maxn = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
  if (!have) { k0 = 0x3fffffff; s0 = 0; cexp = 1u; }   // parked idle lane (x step of 0, never a block entry)
  const int da0 = s0, da1 = 8 * s1, da2 = 64 * s2;
  // block entry along axis a: addr += e_a (the neighbour block's base minus the local field's carry)
  const unsigned e0 = (unsigned)(s0 * (512 - 8)), e1 = (unsigned)((long long)s1 * (512ll * nbx - 64)),
                 e2 = (unsigned)((long long)s2 * (512ll * nbx * nby - 512));
  const int tq2 = 2 * p.tq;
  unsigned long long* const acc = p.dacc;
  int mfree = 0x7fffffff;
  const int K0 = k0, K1 = k1, K2 = k2;
  const long long s_off = (1ll << (kSdfF - 1)) + ((long long)p.tq << kSdfF);
  const long long band_lo = s_off - p.band, band_hi = s_off + p.band;   // colour band |S| < tau (R13)
  if (have) {
    long long thr = (long long)tq2 << kSdfF;
    if (kColor) thr = max(thr, band_hi);   // the free prefix never reaches the colour band
    const long long umax = max(U0, max(U1, U2));
    mfree = 0;
    if (S > thr && umax > 0) {
      const long long num = S - thr;
      long long m = (long long)fminf((float)num * rcp_approx((float)umax), (float)(n - 1));
      while (m > 0 && m * umax > num) --m;
      while (m < n - 1 && (m + 1) * umax <= num) ++m;
      mfree = (int)m;
    }
  }
  const int mw = (int)__reduce_min_sync(0xffffffffu, (unsigned)mfree);
  const unsigned above_mask = 0xfffffffeu << lane;
  const bool lane0 = lane == 0;
  int it = 0;
  {
    // free prefix (see walk_cw_kernel): every lane's update is the clamped one, merged over runs
    const unsigned utq2 = (unsigned)tq2;
    for (; it < mw; ++it) {
      const unsigned prev = __shfl_up_sync(0xffffffffu, addr, 1);
      const bool head = lane0 | (prev != addr) | !have;   // an idle lane is its own run ...
      const unsigned stops = __ballot_sync(0xffffffffu, head);
#if CVX_DW_UNIFORM
      if (stops == 0xffffffffu) {                          // every lane its own run (far field): len = 1
        DW_RED(acc, addr, (1ull << kCntShift) | utq2, have);
      } else {
        const unsigned len = run_len(stops & above_mask, lane);
        const unsigned long long val = ((unsigned long long)(len << (kCntShift - 32)) << 32) | (len * utq2);
        DW_RED(acc, addr, val, head & have);               // ... and issues no reduction
      }
#else
      const unsigned len = run_len(stops & above_mask, lane);
      const unsigned long long val = ((unsigned long long)(len << (kCntShift - 32)) << 32) | (len * utq2);
      DW_RED(acc, addr, val, head & have);                 // ... and issues no reduction
#endif
      const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
      const bool yf = g1 & (!g0 | ((ST)D01 > 0));
      const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
      const bool by = yf & !zf, bx = !yf & !zf;
      if (bx) { addr += da0; --k0; D01 += I1; D02 += I2; }
      if (by) { addr += da1; --k1; D01 -= I0; D12 += I2; }
      if (zf) { addr += da2; --k2; D02 -= I0; D12 -= I1; }
      const unsigned m = zf ? 0x1c0u : (yf ? 0x38u : 7u);
      const unsigned e = zf ? e2 : (yf ? e1 : e0);
      const bool ent = ((addr ^ cexp) & m) == 0u;     // entered the next block of the ray
      addr += ent ? e : 0u;
      mark_block(p.dflag, addr >> 9, ent);
    }
  }
  S -= U0 * (K0 - k0) + U1 * (K1 - k1) + U2 * (K2 - k2);
  {
    // rest of the rays (see walk_cw_kernel): a finished lane parks on its warp's trash spot
    const unsigned spot = trash + ((((unsigned)idx >> 5) & 4095u) << 3);
    int dx0 = da0;
    unsigned ex0 = e0;
    bool parked = it >= n;
    if (parked) { addr = spot; k0 = 0x3fffffff; k1 = 0; k2 = 0; dx0 = 0; cexp = 1u; S = (long long)tq2 << (kSdfF + 1); U0 = 0; n = 0x7fffffff; }
    for (; it < maxn; ++it) {
      const int dpi = min(max((int)(S >> kSdfF), 0), tq2);   // round(sdf 2^q) + tq, clamped (O5, Q4)
      const unsigned key = dpi == tq2 ? addr : 0xffffffffu;     // only clamped updates merge
      const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
      const bool head = lane0 | (prev != key) | (key == 0xffffffffu) | parked;   // a parked lane is its own run ...
      const unsigned stops = __ballot_sync(0xffffffffu, head);
      const unsigned len = run_len(stops & above_mask, lane);
      const unsigned long long val = ((unsigned long long)(len << (kCntShift - 32)) << 32) | (len * (unsigned)dpi);
      DW_RED(acc, addr, val, head & !parked);                  // ... and issues no reduction
      if (kColor && S > band_lo && S < band_hi) {   // TSDF + Color: band updates carry the point's colour (R13)
        const unsigned long long cr = rgb & 0xffu, cg = (rgb >> 8) & 0xffu, cb = (rgb >> 16) & 0xffu;
        CVX_CHECK((long long)addr < (p.dcap + kTrashBlocks) * kBlockVox, "dense colour accumulator address");
        atomicAdd(p.dcacc + 2ull * addr, (1ull << kCntShift) | cr);
        atomicAdd(p.dcacc + 2ull * addr + 1, (cg << 32) | cb);
      }
      if (it + 1 >= n) {   // that was the ray's last voxel: park
        addr = spot; k0 = 0x3fffffff; k1 = 0; k2 = 0; dx0 = 0; cexp = 1u; S = (long long)tq2 << (kSdfF + 1); U0 = 0;
        n = 0x7fffffff; ex0 = 0u; parked = true;
      }
      const bool g0 = k0 > 0, g1 = k1 > 0, g2 = k2 > 0;
      const bool yf = g1 & (!g0 | ((ST)D01 > 0));
      const bool zf = g2 & (yf ? ((ST)D12 > 0) : (!g0 | ((ST)D02 > 0)));
      const bool by = yf & !zf, bx = !yf & !zf;
      if (bx) { addr += dx0; --k0; D01 += I1; D02 += I2; S -= U0; }
      if (by) { addr += da1; --k1; D01 -= I0; D12 += I2; S -= U1; }
      if (zf) { addr += da2; --k2; D02 -= I0; D12 -= I1; S -= U2; }
      const unsigned m = zf ? 0x1c0u : (yf ? 0x38u : 7u);
      const unsigned e = zf ? e2 : (yf ? e1 : ex0);
      const bool ent = ((addr ^ cexp) & m) == 0u;     // entered the next block of the ray
      addr += ent ? e : 0u;
      mark_block(p.dflag, addr >> 9, ent);
    }
  }
}

// R19 ALLOCATE for the dense fold: insert-if-absent of one key.  Returns the slot of an existing key
// (waiting out a concurrent inserter's PENDING), or kPending with *ent = the entry this lane won (the
// caller assigns the slot for the whole warp and publishes it), or kFailed if the table is full.
__device__ __forceinline__ int dense_insert(const HashView& h, Counters* ctr, unsigned long long key, unsigned* ent) {
  unsigned i = hash_slot(key, h);
  for (unsigned n = 0; n <= h.mask; ++n) {
    const longlong2 en = ld_entry(h.e + i);
    unsigned long long k = (unsigned long long)en.x;
    int v = (int)(en.y & 0xffffffffll);
    if (k == kEmptyKey) {
      const unsigned long long old = atomicCAS(&h.e[i].key, kEmptyKey, key);
      if (old == kEmptyKey) { *ent = i; return kPending; }   // won the CAS: this lane inserts
      k = old;
      v = kPending;                                          // its slot is read below
    }
    if (k == key) {
      while (v == kPending) { v = ld_volatile(&h.e[i].val); if (v == kPending) __nanosleep(32); }
      return v;
    }
    i = (i + 1) & h.mask;
  }
  atomicOr(&ctr->err, (unsigned)kErrHashFull);
  return kFailed;
}

// blocks of the box per warp pass of dense_fold_kernel (<= 32): small groups spread the touched blocks of
// dense regions over more warps (each touched block is folded by its warp one after the other)
#ifndef CVX_FOLD_GROUP
#define CVX_FOLD_GROUP 4
#endif
constexpr int kFoldGroup = CVX_FOLD_GROUP;

// R19 ALLOCATE + FOLD of a dense-window launch.  A warp takes kFoldGroup consecutive blocks of the box: (1) it
// reads their accumulators (two blocks in flight) — a block whose accumulators are not all zero was
// traversed by a ray (every traversed voxel receives a count >= 1); (2) lane j activates block j if it
// was touched (insert-if-absent; the pool slots of the new blocks are bumped once per warp, P:L124,
// and the AABB / new-block counters updated once per warp) — the same block set as the block walk;
// (3) the touched blocks are folded into the exact sums one by one (fold_kernel's arithmetic) and their
// accumulators zeroed.
__global__ void __launch_bounds__(256) dense_fold_kernel(const __grid_constant__ WalkParams p) {
  int nbx, nby, nbz;
  if (!dense_dims(p.dbox, p.dcap, nbx, nby, nbz)) return;
  const long long nblk = (long long)nbx * nby * nbz;
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int shift = 30 - p.q;
  for (long long b0 = w0 * kFoldGroup; b0 < nblk; b0 += nw * kFoldGroup) {
    const int nb = (int)min((long long)kFoldGroup, nblk - b0);
    unsigned touched = 0;
    for (int j = 0; j < nb; j += 2) {
      const ulonglong2* s0 = reinterpret_cast<const ulonglong2*>(p.dacc + (b0 + j) * kBlockVox);
      const ulonglong2* s1 = reinterpret_cast<const ulonglong2*>(p.dacc + (b0 + min(j + 1, nb - 1)) * kBlockVox);
      ulonglong2 v[8], w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) { v[i] = s0[lane + 32 * i]; w[i] = s1[lane + 32 * i]; }
      unsigned long long av = 0, aw = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { av |= v[i].x | v[i].y; aw |= w[i].x | w[i].y; }
      touched |= (__any_sync(0xffffffffu, av != 0ull) ? 1u : 0u) << j;
      if (j + 1 < nb) touched |= (__any_sync(0xffffffffu, aw != 0ull) ? 1u : 0u) << (j + 1);
    }
    if (!touched) continue;
    // (2) activation, lane j <-> block b0 + j
    const bool mine = lane < kFoldGroup && ((touched >> lane) & 1u);
    const long long b = b0 + lane;
    const int bx = p.dbox[0] + (int)(b % nbx), by = p.dbox[1] + (int)((b / nbx) % nby),
              bz = p.dbox[2] + (int)(b / ((long long)nbx * nby));
    int slot = kFailed;
    unsigned ent = 0;
    if (mine) slot = dense_insert(p.hash, p.ctr, pack_key(bx, by, bz), &ent);
    const unsigned nm = __ballot_sync(0xffffffffu, mine && slot == kPending);
    if (nm) {
      const int lead = __ffs(nm) - 1;
      int base = 0;
      if (lane == lead) base = atomicAdd(&p.ctr->n_blocks, __popc(nm));
      base = __shfl_sync(0xffffffffu, base, lead);
      const bool isnew = (nm >> lane) & 1u;
      bool ok = false;
      if (isnew) {
        slot = base + __popc(nm & ((1u << lane) - 1u));
        if (slot >= p.pool.max_blocks) { atomicOr(&p.ctr->err, (unsigned)kErrCapacity); slot = kFailed; }
        else { p.pool.coords[slot] = make_int4(bx, by, bz, 0); ok = true; }
      }
      const int big = 0x7fffffff, small = (int)0x80000000;
      const int lo0 = __reduce_min_sync(0xffffffffu, ok ? bx : big), hi0 = __reduce_max_sync(0xffffffffu, ok ? bx : small);
      const int lo1 = __reduce_min_sync(0xffffffffu, ok ? by : big), hi1 = __reduce_max_sync(0xffffffffu, ok ? by : small);
      const int lo2 = __reduce_min_sync(0xffffffffu, ok ? bz : big), hi2 = __reduce_max_sync(0xffffffffu, ok ? bz : small);
      const unsigned nok = __popc(__ballot_sync(0xffffffffu, ok));
      if (lane == lead && nok) {
        atomicMin(&p.ctr->aabb_lo[0], lo0); atomicMin(&p.ctr->aabb_lo[1], lo1); atomicMin(&p.ctr->aabb_lo[2], lo2);
        atomicMax(&p.ctr->aabb_hi[0], hi0); atomicMax(&p.ctr->aabb_hi[1], hi1); atomicMax(&p.ctr->aabb_hi[2], hi2);
        atomicAdd(&p.ctr->new_blocks, (unsigned long long)nok);
      }
      __threadfence();   // coordinates before the published slots (one fence per warp, not per block)
      if (isnew) *(volatile int*)&p.hash.e[ent].val = slot;
    }
    // (3) fold the touched blocks
    for (unsigned t = touched; t; t &= t - 1) {
      const int j = __ffs(t) - 1;
      const int sl = __shfl_sync(0xffffffffu, slot, j);
      ulonglong2* src = reinterpret_cast<ulonglong2*>(p.dacc + (b0 + j) * kBlockVox);
      CVX_CHECK(sl < p.pool.max_blocks && b0 + j < p.dcap, "dense fold slot / block");
      longlong2* s2 = reinterpret_cast<longlong2*>(p.pool.sums) + (long long)(sl < 0 ? 0 : sl) * kBlockVox;
      ulonglong2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = src[lane + 32 * i];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if ((v[i].x | v[i].y) == 0ull) continue;
        const int e = lane + 32 * i;   // voxels 2e, 2e + 1
        if (sl >= 0) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const unsigned long long a = h ? v[i].y : v[i].x;
            if (!a) continue;
            const long long cnt = (long long)(a >> kCntShift), sd = (long long)(a & ((1ull << kCntShift) - 1));
            longlong2 x = s2[2 * e + h];
            x.x += (sd - cnt * p.tq) << shift;
            x.y += cnt << 30;
            s2[2 * e + h] = x;
          }
        }
        src[e] = make_ulonglong2(0ull, 0ull);
      }
      if (p.dcacc) {   // TSDF + Color: the block's packed colour accumulators (fold_color_kernel's arithmetic)
        ulonglong2* csrc = reinterpret_cast<ulonglong2*>(p.dcacc) + (b0 + j) * kBlockVox;
        longlong2* cs = reinterpret_cast<longlong2*>(p.pool.csum) + 2ll * (long long)(sl < 0 ? 0 : sl) * kBlockVox;
        for (int vx = lane; vx < kBlockVox; vx += 32) {
          const ulonglong2 cv = csrc[vx];
          if ((cv.x | cv.y) == 0ull) continue;
          if (sl >= 0) {
            longlong2 a = cs[2 * vx], c2 = cs[2 * vx + 1];
            a.x += (long long)(cv.x >> kCntShift) << 30;
            a.y += (long long)(cv.x & ((1ull << kCntShift) - 1)) << 30;
            c2.x += (long long)(cv.y >> 32) << 30;
            c2.y += (long long)(cv.y & 0xffffffffull) << 30;
            cs[2 * vx] = a; cs[2 * vx + 1] = c2;
          }
          csrc[vx] = make_ulonglong2(0ull, 0ull);
        }
      }
    }
  }
}

// Block-count submap trigger: after the ALLOCATE phase of frame k, fire once the
// submap holds >= threshold blocks; frame k is the last one it takes.
__global__ void trigger_check_kernel(const Counters* ctr, int* trig, int frame) {
  if (!trig[1] && ctr->n_blocks >= trig[0]) { trig[1] = 1; trig[2] = frame + 1; }
}

// TSDF + Color (R13): fold the packed colour accumulators {n << 40 | sum r, sum g << 32 | sum b} (w = 1)
// into the exact colour sums {sum w, sum w r, sum w g, sum w b} at 2^-30.
__global__ void fold_color_kernel(const Counters* ctr, unsigned long long* cacc, long long* csum, int max_blocks,
                                  const int* dirty) {
  if (dirty && !*dirty) return;   // R19: every launch since the last fold ran in its dense window
  const int nb = min(ctr->n_blocks, max_blocks);
  const long long nv = (long long)nb * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const ulonglong2 v = reinterpret_cast<ulonglong2*>(cacc)[i];
    if ((v.x | v.y) == 0ull) continue;
    longlong2* cs = reinterpret_cast<longlong2*>(csum) + 2 * i;
    longlong2 a = cs[0], b = cs[1];
    a.x += (long long)(v.x >> kCntShift) << 30;                  // sum w (w = 1 -> 2^30)
    a.y += (long long)(v.x & ((1ull << kCntShift) - 1)) << 30;   // sum w r
    b.x += (long long)(v.y >> 32) << 30;                  // sum w g
    b.y += (long long)(v.y & 0xffffffffull) << 30;        // sum w b
    cs[0] = a; cs[1] = b;
    reinterpret_cast<ulonglong2*>(cacc)[i] = make_ulonglong2(0ull, 0ull);
  }
}

// a5 FOLD of the packed per-launch accumulators into the exact sums: sum(w d) += (sum d' - n tq) 2^(30-q),
// sum(w) += n 2^30 (w = 1).  Every update contributes exactly round(d 2^q) 2^(30-q), so the result does
// not depend on how frames are grouped into launches.
__global__ void fold_kernel(const Counters* ctr, unsigned long long* acc, long long* sums, int max_blocks, int tq, int shift,
                            const int* dirty) {
  if (dirty && !*dirty) return;   // R19: every launch since the last fold ran in its dense window
  const int nb = min(ctr->n_blocks, max_blocks);
  const long long nv2 = (long long)nb * (kBlockVox / 2);
  ulonglong2* a2 = reinterpret_cast<ulonglong2*>(acc);
  longlong2* s2 = reinterpret_cast<longlong2*>(sums);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv2; i += (long long)gridDim.x * blockDim.x) {
    const ulonglong2 v = a2[i];
    if ((v.x | v.y) == 0ull) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned long long a = h ? v.y : v.x;
      if (!a) continue;
      const long long n = (long long)(a >> kCntShift), sd = (long long)(a & ((1ull << kCntShift) - 1));
      longlong2 x = s2[2 * i + h];
      x.x += (sd - n * tq) << shift;
      x.y += n << 30;
      s2[2 * i + h] = x;
    }
    a2[i] = make_ulonglong2(0ull, 0ull);
  }
}

__global__ void zero_blocks_kernel(Counters* ctr, long long* sums, unsigned long long* acc, int max_blocks) {
  const int nb = min(*(volatile int*)&ctr->n_blocks, max_blocks);
  const long long n16 = (long long)nb * kBlockVox;   // one longlong2 per voxel
  longlong2* s2 = reinterpret_cast<longlong2*>(sums);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) {
    s2[i] = make_longlong2(0, 0);
    if ((i & 1) == 0) reinterpret_cast<ulonglong2*>(acc)[i >> 1] = make_ulonglong2(0ull, 0ull);
  }
}

// reset: the dense slot cache entries of the used blocks go back to unknown
__global__ void clear_grid_kernel(Counters* ctr, const int4* coords, int* grid, int max_blocks) {
  const int nb = min(*(volatile int*)&ctr->n_blocks, max_blocks);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nb; s += gridDim.x * blockDim.x) {
    const int4 c = coords[s];
    const int gi = grid_cache_index(c.x, c.y, c.z);
    if (gi >= 0) grid[gi] = -1;
  }
}

__global__ void zero_color_kernel(Counters* ctr, long long* csum, unsigned long long* cacc, int max_blocks) {
  const int nb = min(*(volatile int*)&ctr->n_blocks, max_blocks);
  const long long nv = (long long)nb * kBlockVox;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    reinterpret_cast<longlong2*>(csum)[2 * i] = make_longlong2(0, 0);
    reinterpret_cast<longlong2*>(csum)[2 * i + 1] = make_longlong2(0, 0);
    reinterpret_cast<ulonglong2*>(cacc)[i] = make_ulonglong2(0ull, 0ull);
  }
}

// ---------------------------------------------------------------------------------- projection mapping
// SURVEY §8 f2 / DESIGN.md R14: the KinectFusion / nvBlox voxel-centric update the paper
// contrasts with raycasting.  ALLOCATE is the raycast one (prepare + block walk per frame); then every
// voxel of the submap is projected into the frame's depth image, associated with the nearest pixel and
// fused with sdf = depth - z.  One CTA owns one 8^3 block at a time (persistent grid-stride over the
// blocks), each thread 4 voxels, and loops over the frames of the launch with the sums in registers:
// the TSDF state is read and written once per launch, the depth images are gathered through L1/L2, and
// no atomics touch the voxels (a voxel has one owner thread).  A block created during this call
// (slot >= the block count at the call's start) carries its birth frame — the first frame whose rays
// reached it, recorded by the block walk — and skips the frames before it, so the result equals
// frame-by-frame integration exactly.  Every decision (z > 0, pixel, range, occlusion)
// is taken in the oracle's fp64 / fp32 operation order without FMA contraction.
struct ProjParams {
  const float* depth;      // [nf][height][width]
  const double* frame_T;   // compose_kernel records of the launch's frames
  const int* start;        // block count at the start of the call (older blocks see every frame)
  const int* birth;        // per slot: birth frame (call-relative) of blocks created in this call
  int frame_base;          // call-relative index of the launch's first frame
  PoolView pool;
  Counters* ctr;
  int nf, width, height;
  float fx, fy, cx, cy;
  double rmin, rmax, s, tau, rfloor;
  int weighting, carve, q;
};

constexpr int kProjThreads = 128;

__global__ void __launch_bounds__(kProjThreads) project_kernel(const __grid_constant__ ProjParams p) {
  __shared__ double sT[kMaxBatch][12];   // R_SC (row-major) and t_SC per frame
  for (int i = threadIdx.x; i < p.nf * 12; i += blockDim.x) sT[i / 12][i % 12] = p.frame_T[kFrameRec * (i / 12) + i % 12];
  __syncthreads();
  const int nb = min(p.ctr->n_blocks, p.pool.max_blocks);
  const int start = *p.start;
  const int t = threadIdx.x;
  const int lx = t & 7, ly = (t >> 3) & 7, lz0 = t >> 6;   // voxel k of the thread: lz = lz0 + 2k
  const double dq_scale = (double)(1ll << p.q);
  const int shift = 30 - p.q;
  unsigned long long n_upd = 0;
  for (int blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const int4 bc = p.pool.coords[blk];
    double cx0 = dm(da((double)(bc.x * 8 + lx), 0.5), p.s);
    double cy0 = dm(da((double)(bc.y * 8 + ly), 0.5), p.s);
    double cz[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cz[k] = dm(da((double)(bc.z * 8 + lz0 + 2 * k), 0.5), p.s);
    long long swd[4] = {0, 0, 0, 0}, sw[4] = {0, 0, 0, 0};
    const int j0 = blk < start ? 0 : max(0, p.birth[blk] - p.frame_base);   // CTA-uniform
    for (int j = j0; j < p.nf; ++j) {
      const double* T = sT[j];
      const float* img = p.depth + (long long)j * p.width * p.height;
      const double e0 = ds(cx0, T[9]), e1 = ds(cy0, T[10]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double e2 = ds(cz[k], T[11]);
        // x = R_SC^T (c - t_SC): x_i = (R[0][i] e0 + R[1][i] e1) + R[2][i] e2
        const double z = da(da(dm(T[2], e0), dm(T[5], e1)), dm(T[8], e2));
        if (!(z > 0.0)) continue;
        const double x0 = da(da(dm(T[0], e0), dm(T[3], e1)), dm(T[6], e2));
        const double x1 = da(da(dm(T[1], e0), dm(T[4], e1)), dm(T[7], e2));
        const double inv = __drcp_rn(z);
        const double uh = da(da(dm(dm((double)p.fx, x0), inv), (double)p.cx), 0.5);
        const double wh = da(da(dm(dm((double)p.fy, x1), inv), (double)p.cy), 0.5);
        if (!(uh >= 0.0 && uh < (double)p.width && wh >= 0.0 && wh < (double)p.height)) continue;
        const int px = (int)uh, py = (int)wh;   // non-negative: truncation == floor
        const float m = __ldg(img + py * p.width + px);
        if (!(m > 0.0f) || !isfinite(m)) continue;
        const float pc0 = __fdiv_rn(__fmul_rn(m, __fsub_rn((float)px, p.cx)), p.fx);
        const float pc1 = __fdiv_rn(__fmul_rn(m, __fsub_rn((float)py, p.cy)), p.fy);
        const double L = __dsqrt_rn(da(da(dm((double)pc0, (double)pc0), dm((double)pc1, (double)pc1)),
                                       dm((double)m, (double)m)));
        if (!(L >= p.rmin && L <= p.rmax)) continue;
        const double sdf = ds((double)m, z);
        if (sdf < -p.tau || (!p.carve && sdf > p.tau)) continue;
        const long long dq = __double2ll_rn(dm(fmin(sdf, p.tau), dq_scale));   // R2 quantum 2^-q
        if (p.weighting == 0) {
          swd[k] += dq << shift;
          sw[k] += 1ll << 30;
        } else {
          const double r = fmax(L, p.rfloor);
          const double w = __drcp_rn(dm(r, r));
          swd[k] += __double2ll_rn(dm(dm(w, (double)dq), (double)(1ll << shift)));
          sw[k] += __double2ll_rn(dm(w, kFxScale));
        }
        ++n_upd;
      }
    }
    longlong2* s2 = reinterpret_cast<longlong2*>(p.pool.sums) + (long long)blk * kBlockVox;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (sw[k] == 0) continue;
      const int l = t + kProjThreads * k;   // = lx + 8 ly + 64 (lz0 + 2k)
      longlong2 v = s2[l];
      v.x += swd[k];
      v.y += sw[k];
      s2[l] = v;
    }
  }
  n_upd = __reduce_add_sync(0xffffffffu, (unsigned)n_upd);
  if ((t & 31) == 0 && n_upd) atomicAdd(&p.ctr->voxel_updates, n_upd);
}

__global__ void record_count_kernel(const Counters* ctr, int* cnt, int j, int max_blocks) {
  cnt[j] = min(ctr->n_blocks, max_blocks);
}

__global__ void reset_counters_kernel(Counters* ctr) {
  Counters c = {};
  c.aabb_lo[0] = c.aabb_lo[1] = c.aabb_lo[2] = 0x7fffffff;
  c.aabb_hi[0] = c.aabb_hi[1] = c.aabb_hi[2] = (int)0x80000000;
  *ctr = c;
}

}  // namespace

// R19: apply a dense fold deferred by the last integrate call (ALLOCATE + FOLD of its last launch) on `st`,
// after that call's walk.  Every call that reads or changes the submap's state runs it first.
cudaError_t flush_fold(cvx_submap* sm, cudaStream_t st) {
  if (!sm->fold_pending) return cudaSuccess;
  sm->fold_pending = false;
  cudaStreamWaitEvent(st, sm->ev_walked, 0);
  const int q = packed_q(sm->cfg.truncation);
  WalkParams wp{};
  wp.hash = sm->hash; wp.pool = sm->pool; wp.ctr = sm->ctr;
  wp.q = q; wp.tq = (int)std::llround(std::ldexp(sm->cfg.truncation, q));
  wp.dacc = sm->dacc; wp.dbox = sm->buf[sm->fold_buf].lcnt + 8; wp.dcap = sm->fold_dcap;
  wp.dflag = reinterpret_cast<unsigned char*>(sm->dacc + (sm->fold_dcap + kTrashBlocks) * kBlockVox);
  wp.dcacc = sm->fold_color ? sm->dcacc : nullptr;
  {
    ProfScope ps_(sm, "dense_fold_allocate", st);
    dense_fold_kernel<<<148 * 8, 256, 0, st>>>(wp);
  }
  cudaEventRecord(sm->ev_free[sm->fold_buf], st);   // the buffer's box may be reused after the fold
  return cudaGetLastError();
}

cudaError_t launch_reset(cvx_submap* sm, cudaStream_t st) {
  if (cudaError_t fe = flush_fold(sm, st)) return fe;   // leaves the dense window zero
  {
    ProfScope ps_(sm, "reset_zero_blocks", st);
    zero_blocks_kernel<<<148 * 8, 256, 0, st>>>(sm->ctr, sm->pool.sums, sm->pool.acc, sm->pool.max_blocks);
  }
  if (sm->pool.csum) {
    ProfScope ps_(sm, "reset_zero_color", st);
    zero_color_kernel<<<148 * 8, 256, 0, st>>>(sm->ctr, sm->pool.csum, sm->pool.cacc, sm->pool.max_blocks);
  }
  {
    ProfScope ps_(sm, "reset_grid", st);
    clear_grid_kernel<<<148 * 2, 256, 0, st>>>(sm->ctr, sm->pool.coords, sm->pool.grid, sm->pool.max_blocks);
  }
  {
    ProfScope ps_(sm, "reset_counters", st);
    reset_counters_kernel<<<1, 1, 0, st>>>(sm->ctr);
  }
  cudaMemsetAsync(sm->hash.e, 0xff, sizeof(HashEntry) * ((size_t)sm->hash.mask + 1), st);   // EMPTY / PENDING
  return cudaGetLastError();
}

static void set_divisors(PrepParams& pp, const cvx_sensor_model& sensor) {
  constexpr int PC = 32 / CVX_PATCH_ROWS;
  pp.rs = 1.0 / pp.s;
  pp.r_npf = 1.0 / (double)pp.n_per_frame;
  pp.r_width = sensor.width > 0 ? 1.0 / (double)sensor.width : 0.0;
  pp.r_pcols = sensor.width >= PC ? 1.0 / (double)(sensor.width / PC) : 0.0;
}

// Grow-only scratch, stream-ordered (cudaMallocAsync / cudaFreeAsync on `st`): the caller
// orders `st` after every earlier user of the buffer before growing it.
static cudaError_t grow(void** ptr, int64_t* cap, int64_t need, size_t elem, cudaStream_t st) {
  if (*cap >= need) return cudaSuccess;
  if (*ptr) cudaFreeAsync(*ptr, st);
  *ptr = nullptr;
  *cap = 0;
  cudaError_t e = cudaMallocAsync(ptr, elem * (size_t)need, st);
  if (e == cudaSuccess) *cap = need;
  return e;
}

cudaError_t launch_integrate(cvx_submap* sm, const float* data, int64_t n_per_frame, int n_frames,
                             const double* T_world_sensor, const cvx_sensor_model& sensor, cudaStream_t st,
                             bool host_data, int* trig, const unsigned char* rgb) {
  if (cudaError_t fe = flush_fold(sm, st)) return fe;   // the previous call's deferred fold first
  if (n_per_frame <= 0 || n_frames <= 0) return cudaSuccess;
  // pipeline side stream (a1-a3 of launch k+1 under the walk of launch k); the caller's stream itself
  // when the submap is in serialised profiling mode
  const cudaStream_t side = sm->serialize ? st : sm->side;
  const long long elems_per_frame = n_per_frame * (sensor.kind == 1 ? 1 : 3);
  // launches of equal size; at most kMaxBatch frames and kLaunchRays rays (pipelining granularity).
  // Constant weights: the packed accumulators are folded whenever the next launch would take them past
  // kMaxPackedRays rays since the last fold, and at the end of the call (R6/R7)
  // Host frames use smaller launches (kLaunchRaysHost) so the H2D copies pipeline with the ingest of the
  // call's earlier launches (configs[1] e2e step, copies started early: 2^22 8.80 ms, 2^23 8.70, 2^24 8.8-9.0)
  const long long launch_rays = host_data ? kLaunchRaysHost : kLaunchRays;
  const bool cw_ok = sm->aggregate && sm->cfg.weighting == 0 && n_per_frame <= launch_rays;
  const long long ray_limit = cw_ok ? launch_rays : (1ll << 31) - 1;
  const int lim = trig ? 1 : (int)std::max<long long>(1, std::min<long long>(kMaxBatch, ray_limit / n_per_frame));
  std::vector<int> plan;                             // equal chunks
  {
    const int chunks = (n_frames + lim - 1) / lim;
    const int eq = (n_frames + chunks - 1) / chunks;
    for (int left = n_frames; left > 0; left -= eq) plan.push_back(std::min(eq, left));
  }
  const int per = *std::max_element(plan.begin(), plan.end());
  const long long cap_rays = (long long)per * n_per_frame;
  // scratch growth is stream-ordered on the side stream, after the walk that last read the buffer
  const cudaStream_t gs = sm->serialize ? st : sm->side;
  for (int b = 0; b < 2; ++b) {
    const bool need_grow = sm->buf[b].ray_cap < cap_rays || (sm->dense_on && sm->buf[b].cta_box_cap < 6 * ((cap_rays + kPrepThreads - 1) / kPrepThreads)) ||
                           (CVX_PREP_ORDERED && sm->buf[b].cstat_cap < (cap_rays + kPrepThreads - 1) / kPrepThreads) || sm->buf[b].slot_cap < cap_rays * kSlotsPerRay + 1024 ||
                           (rgb && sm->buf[b].rgbs_cap < cap_rays) || (sm->cfg.weighting != 0 && sm->buf[b].ws_cap < cap_rays) ||
                           (host_data && sm->buf[b].staging_cap < (long long)per * elems_per_frame);
    if (need_grow) {
      cudaEventRecord(sm->ev_entry, st);     // the caller's earlier work on the buffers, then their last walk
      cudaStreamWaitEvent(gs, sm->ev_entry, 0);
      cudaStreamWaitEvent(gs, sm->ev_free[b], 0);
      if (sm->copy) cudaStreamWaitEvent(gs, sm->ev_stage_free[b], 0);
    }
    cudaError_t e = grow(&sm->buf[b].rays, &sm->buf[b].ray_cap, cap_rays, sizeof(RayRec), gs);
    if (e == cudaSuccess && rgb)
      e = grow(reinterpret_cast<void**>(&sm->buf[b].rgbs), &sm->buf[b].rgbs_cap, cap_rays, sizeof(unsigned), gs);
    if (e == cudaSuccess && sm->cfg.weighting != 0)
      e = grow(reinterpret_cast<void**>(&sm->buf[b].ws), &sm->buf[b].ws_cap, cap_rays, sizeof(float), gs);
    if (e == cudaSuccess) e = grow(reinterpret_cast<void**>(&sm->buf[b].slot_lists), &sm->buf[b].slot_cap,
                                   cap_rays * kSlotsPerRay + 1024, sizeof(int), gs);
    if (e == cudaSuccess && sm->dense_on)
      e = grow(reinterpret_cast<void**>(&sm->buf[b].cta_box), &sm->buf[b].cta_box_cap, 6 * ((cap_rays + kPrepThreads - 1) / kPrepThreads), sizeof(int), gs);
    if (e == cudaSuccess && CVX_PREP_ORDERED)
      e = grow(reinterpret_cast<void**>(&sm->buf[b].cstat), &sm->buf[b].cstat_cap, (cap_rays + kPrepThreads - 1) / kPrepThreads,
               sizeof(unsigned long long), gs);
    if (e == cudaSuccess && host_data)
      e = grow(reinterpret_cast<void**>(&sm->buf[b].staging), &sm->buf[b].staging_cap, (long long)per * elems_per_frame,
               sizeof(float), gs);
    if (e != cudaSuccess) return e;
  }
  const int q = packed_q(sm->cfg.truncation);
  const int tq = (int)std::llround(std::ldexp(sm->cfg.truncation, q));
  // every ray spans < 2^12 voxels per axis if (max_range + tau) / s + 2 < 4096 (domain check O3 bounds
  // the rest): then the crossing-order differences fit 32 bits (see walk_kernel)
  const bool k32 = ((double)sensor.max_range + sm->cfg.truncation) / sm->cfg.voxel_size + 2.0 < 4096.0;
  // R19: the dense-window path (constant weights, no colour, no trigger, default ALLOCATE kernels): the
  // accumulator buffer covers a conservative box of the call (balls of radius max_range + tau around the
  // frames' sensor origins), capped at dense_cap blocks; each launch uses the exact box of its rays
  // (prepare_kernel) and falls back to the slot-list path on the device if that box exceeds the buffer.
  bool dense = cw_ok && sm->dense_on && sm->walk_cw && sm->bw2 && !sm->bw3 && !sm->fuse_alloc && !trig &&
               (!rgb || (sm->pool.csum && sm->dense_color));
  long long dcap = 0;
  if (dense) {
    const double* W = sm->T_ws;
    const double R = (double)sensor.max_range + sm->cfg.truncation, sv = sm->cfg.voxel_size;
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int f = 0; f < n_frames; ++f) {
      const double* C = T_world_sensor + 16 * f;
      for (int i = 0; i < 3; ++i) {
        const double o = W[0 * 4 + i] * (C[3] - W[3]) + W[1 * 4 + i] * (C[7] - W[7]) + W[2 * 4 + i] * (C[11] - W[11]);
        lo[i] = std::min(lo[i], o); hi[i] = std::max(hi[i], o);
      }
    }
    long long nblk = 1;
    for (int i = 0; i < 3; ++i) {
      const double b0 = std::floor((lo[i] - R) / sv / 8.0) - 1.0, b1 = std::floor((hi[i] + R) / sv / 8.0) + 1.0;
      nblk = (long long)std::min(1e15, (double)nblk * (b1 - b0 + 1.0));
    }
    dcap = std::min(nblk, sm->dense_cap);
    if (sm->dacc_blocks < dcap) {   // grow-only, zeroed once; the dense folds keep it zero
      if (sm->dacc) cudaFreeAsync(sm->dacc, st);
      sm->dacc = nullptr;
      sm->dacc_blocks = 0;
      // accumulators, the trash region, then one touched flag per block
      const size_t bytes = (size_t)(dcap + kTrashBlocks) * kBlockVox * sizeof(unsigned long long) + (size_t)dcap;
      if (cudaMallocAsync(reinterpret_cast<void**>(&sm->dacc), bytes, st) == cudaSuccess) {
        cudaMemsetAsync(sm->dacc, 0, bytes, st);
        sm->dacc_blocks = dcap;
      } else {                        // device memory short: this call takes the slot-list path instead
        cudaGetLastError();
        sm->dacc = nullptr;
        dense = false;
      }
    }
    dcap = sm->dacc_blocks;
    if (dense && rgb && sm->dcacc_blocks < dcap) {   // TSDF + Color: dense colour accumulators, same index space
      if (sm->dcacc) cudaFreeAsync(sm->dcacc, st);
      sm->dcacc = nullptr;
      sm->dcacc_blocks = 0;
      const size_t cbytes = (size_t)(dcap + kTrashBlocks) * kBlockVox * 2 * sizeof(unsigned long long);
      if (cudaMallocAsync(reinterpret_cast<void**>(&sm->dcacc), cbytes, st) == cudaSuccess) {
        cudaMemsetAsync(sm->dcacc, 0, cbytes, st);
        sm->dcacc_blocks = dcap;
      } else {
        cudaGetLastError();
        sm->dcacc = nullptr;
        dense = false;
      }
    }
  }
  long long pending = 0;                             // rays in the packed accumulators since the last fold
  auto fold = [&]() {
    if (pending == 0) return;
    {
      ProfScope ps_(sm, "fold", st);
      fold_kernel<<<148 * 8, 256, 0, st>>>(sm->ctr, sm->pool.acc, sm->pool.sums, sm->pool.max_blocks, tq, 30 - q,
                                           dense ? sm->acc_dirty : nullptr);
    }
    if (rgb) {
      ProfScope ps_(sm, "fold_color", st);
      fold_color_kernel<<<148 * 8, 256, 0, st>>>(sm->ctr, sm->pool.cacc, sm->pool.csum, sm->pool.max_blocks,
                                                 dense ? sm->acc_dirty : nullptr);
    }
    if (dense) cudaMemsetAsync(sm->acc_dirty, 0, sizeof(int), st);   // after both folds read it
    pending = 0;
  };
  cudaEventRecord(sm->ev_entry, st);                 // the side stream starts after the caller's prior work
  cudaStreamWaitEvent(side, sm->ev_entry, 0);
  cudaStream_t cstream = side;                       // host frames: H2D copies (own stream unless serialised)
  if (host_data && !sm->serialize) {
    if (!sm->copy) {
      cudaError_t e = cudaStreamCreateWithFlags(&sm->copy, cudaStreamNonBlocking);
      for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&sm->ev_staged[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sm->ev_stage_free[b], cudaEventDisableTiming);
      }
      if (e != cudaSuccess) return e;
    }
    cstream = sm->copy;
#if !CVX_COPY_EARLY
    cudaStreamWaitEvent(cstream, sm->ev_entry, 0);
#endif
    // CVX_COPY_EARLY: the copy into staging[b] waits only for the prepare that last read staging[b]
    // (ev_stage_free) — nothing else on the device touches the staging buffers — so a call's copies can
    // run under whatever the caller's stream is still doing (e.g. the previous submap's walk)
  }
  int f0 = 0;
  for (size_t li = 0; li < plan.size(); ++li) {
    const int nf = plan[li];
    const bool last_launch = li + 1 == plan.size();
    const long long total = (long long)nf * n_per_frame;
    const int b = sm->next_buf;
    sm->next_buf ^= 1;
    cvx_submap::Buf& B = sm->buf[b];
    const unsigned blocks = (unsigned)((total + 255) / 256);
    const float* chunk = data + (long long)f0 * elems_per_frame;
    if (host_data) {   // host frames: the H2D copy of launch k+1 overlaps the walk of launch k
      if (cstream != side) cudaStreamWaitEvent(cstream, sm->ev_stage_free[b], 0);   // prepare done with staging[b]
      cudaMemcpyAsync(B.staging, chunk, sizeof(float) * (size_t)(nf * elems_per_frame), cudaMemcpyHostToDevice,
                      cstream);
      if (cstream != side) cudaEventRecord(sm->ev_staged[b], cstream);
      chunk = B.staging;
    }
    // ---- side stream: a1-a3 (compose, prepare/COUNT, ALLOCATE) into buffer b
    cudaStreamWaitEvent(side, sm->ev_free[b], 0);   // the walk that last read buffer b is done
    ComposeParams cp;
    for (int i = 0; i < 16; ++i) cp.Tws[i] = sm->T_ws[i];
    for (int f = 0; f < nf; ++f)
      for (int i = 0; i < 16; ++i) cp.Twc[f][i] = T_world_sensor[16 * (f0 + f) + i];
    cp.n = nf;
    cp.s = sm->cfg.voxel_size;
    {
      ProfScope ps_(sm, "compose_poses", side);
      compose_kernel<<<1, kMaxBatch, 0, side>>>(cp, B.frame_T);
    }
    cudaMemsetAsync(B.lcnt, 0, 4 * sizeof(int), side);
    if (CVX_PREP_ORDERED) cudaMemsetAsync(B.cstat, 0, sizeof(unsigned long long) * (size_t)((total + kPrepThreads - 1) / kPrepThreads), side);
    if (dense) {   // box {lo[3], hi[3]} = {0x7f7f7f7f x3, 0x80808080 x3}: beyond any block coordinate (< 2^20)
      cudaMemsetAsync(B.lcnt + 8, 0x7f, 3 * sizeof(int), side);
      cudaMemsetAsync(B.lcnt + 11, 0x80, 3 * sizeof(int), side);
    }
    if (host_data && cstream != side) cudaStreamWaitEvent(side, sm->ev_staged[b], 0);
    PrepParams pp{};
    pp.data = chunk;
    pp.n_per_frame = n_per_frame; pp.total = total;
    pp.kind = sensor.kind; pp.width = sensor.width;
    pp.fx = sensor.fx; pp.fy = sensor.fy; pp.cx = sensor.cx; pp.cy = sensor.cy;
    pp.rmin = (double)sensor.min_range; pp.rmax = (double)sensor.max_range;
    pp.s = sm->cfg.voxel_size; pp.tau = sm->cfg.truncation; pp.rfloor = sm->cfg.weight_range_floor;
    pp.weighting = sm->cfg.weighting; pp.carve = sm->cfg.carve;
    pp.sdf_scale = std::ldexp(1.0, q + kSdfF);
    set_divisors(pp, sensor);
    pp.height = sensor.height;
    {
      constexpr int PR = CVX_PATCH_ROWS, PC = 32 / CVX_PATCH_ROWS;
      const int S = CVX_SECTOR_COLS;
      const bool org = sensor.kind != 0 && sensor.width > 0 && sensor.height > 0 && sensor.width % PC == 0 &&
                       sensor.height % PR == 0 && n_per_frame == (long long)sensor.width * sensor.height;
      if (S > 0 && org && (sensor.width / PC) % (S > 0 ? S : 1) == 0 && dense) {
        const double PF = (double)(sensor.height / PR) * S;
        pp.sec_cols = S; pp.nframes = nf;
        pp.r_frmpat = 1.0 / PF; pp.r_secpat = 1.0 / (PF * nf); pp.r_seccols = 1.0 / (double)(S > 0 ? S : 1);
      }
    }
    pp.frame_T = B.frame_T; pp.rays = (RayRec*)B.rays; pp.ctr = sm->ctr; pp.lcnt = B.lcnt;
    // one spare entry: walk_cw_kernel prefetches the entry after a ray's last block unconditionally
    pp.list_cap = (int)std::min<long long>(std::min<long long>(B.slot_cap - 1, sm->list_cap_limit), 0x7fffffffll);
    pp.trig = trig;
    pp.rgb = rgb ? rgb + (long long)f0 * n_per_frame * 3 : nullptr;
    pp.rgbs = rgb ? B.rgbs : nullptr;
    pp.ws = sm->cfg.weighting != 0 ? B.ws : nullptr;
    pp.count_vox = 1;
    pp.box = dense ? B.cta_box : nullptr;
    pp.cstat = CVX_PREP_ORDERED ? B.cstat : nullptr;
    {
      ProfScope ps_(sm, "ray_prepare", side);
      prepare_kernel<<<(unsigned)((total + kPrepThreads - 1) / kPrepThreads), kPrepThreads, 0, side>>>(pp);
    }
    if (dense) box_reduce_kernel<<<32, 256, 0, side>>>(B.cta_box, (int)((total + kPrepThreads - 1) / kPrepThreads), B.lcnt + 8);
    if (host_data && cstream != side) cudaEventRecord(sm->ev_stage_free[b], side);   // staging[b] consumed
    WalkParams wp{};
    wp.rays = (const RayRec*)B.rays; wp.ctr = sm->ctr; wp.hash = sm->hash; wp.pool = sm->pool;
    wp.slots = B.slot_lists; wp.lcnt = B.lcnt;
    wp.s = (float)sm->cfg.voxel_size; wp.tau = (float)sm->cfg.truncation;
    wp.tq = tq;
    wp.q = q;
    wp.band = std::llround(std::ldexp(sm->cfg.truncation, q + kSdfF));
    wp.birth = nullptr;
    wp.frame_T = B.frame_T; wp.rgbs = pp.rgbs; wp.ws = pp.ws; wp.frame_base = 0;
    wp.dacc = sm->dacc; wp.dbox = dense ? B.lcnt + 8 : nullptr; wp.dcap = dcap; wp.acc_dirty = sm->acc_dirty;
    wp.dflag = dense ? reinterpret_cast<unsigned char*>(sm->dacc + (dcap + kTrashBlocks) * kBlockVox) : nullptr;
    wp.dcacc = dense && rgb ? sm->dcacc : nullptr;
    const bool cw = cw_ok && total <= launch_rays;
    // constant weights, no colour, no block-count trigger: ALLOCATE runs inside the update walk
    const bool fuse = sm->fuse_alloc && cw && sm->aggregate && sm->walk_cw && !rgb && !trig;
    if (!fuse) {
      ProfScope ps_(sm, "block_walk_allocate", side);
      if (sm->bw3) {
        if (k32) block_walk3_kernel<true><<<blocks, 256, 0, side>>>(wp);
        else block_walk3_kernel<false><<<blocks, 256, 0, side>>>(wp);
      } else if (sm->bw2) {
        const unsigned bwb = dense ? std::min(blocks, 148u * 8u) : blocks;   // dense: grid-stride fallback only
        if (k32) block_walk2_kernel<true><<<bwb, 256, 0, side>>>(wp);
        else block_walk2_kernel<false><<<bwb, 256, 0, side>>>(wp);
      } else {
        if (k32) block_walk_kernel<true><<<blocks, 256, 0, side>>>(wp);
        else block_walk_kernel<false><<<blocks, 256, 0, side>>>(wp);
      }
    }
    if (trig) trigger_check_kernel<<<1, 1, 0, side>>>(sm->ctr, trig, f0);
    cudaEventRecord(sm->ev_prepared[b], side);
    // ---- caller's stream: a4 UPDATE + a5 FOLD of launch k
    if (cw && pending + total > kMaxPackedRays) fold();
    cudaStreamWaitEvent(st, sm->ev_prepared[b], 0);
    // CVX_WALK_PRIO: the update walk runs on a high-priority library stream (ordered after / before the
    // caller's stream by events), so a concurrent ESDF of another submap does not take its SMs
    cudaStream_t ws = st;
    if (sm->walk_prio && !sm->serialize) {
      if (!sm->wstream) {
        int lo_p = 0, hi_p = 0;
        cudaDeviceGetStreamPriorityRange(&lo_p, &hi_p);
        cudaStreamCreateWithPriority(&sm->wstream, cudaStreamNonBlocking, hi_p);
        cudaEventCreateWithFlags(&sm->ev_w[0], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&sm->ev_w[1], cudaEventDisableTiming);
      }
      ws = sm->wstream;
      cudaEventRecord(sm->ev_w[0], st);
      cudaStreamWaitEvent(ws, sm->ev_w[0], 0);
    }
    {
      ProfScope ps_(sm, "ray_walk_update", ws);
      const unsigned wblocks = (unsigned)((total + 127) / 128);   // 128-thread CTAs (measured best)
      if (cw && sm->aggregate && sm->walk_cw) {
        if (rgb) {
          if (dense) { if (k32) walk_dw_kernel<true, true><<<wblocks, 128, 0, ws>>>(wp); else walk_dw_kernel<false, true><<<wblocks, 128, 0, ws>>>(wp); }
          const unsigned fwb = dense ? std::min(wblocks, 148u * 16u) : wblocks;   // dense: fallback only
          if (k32) walk_cw_kernel<true, true><<<fwb, 128, 0, ws>>>(wp); else walk_cw_kernel<false, true><<<fwb, 128, 0, ws>>>(wp);
        }
        else if (fuse) { if (k32) walk_cw_kernel<true, false, true><<<wblocks, 128, 0, ws>>>(wp); else walk_cw_kernel<false, false, true><<<wblocks, 128, 0, ws>>>(wp); }
        else {
          if (dense) { if (k32) walk_dw_kernel<true><<<wblocks, 128, 0, ws>>>(wp); else walk_dw_kernel<false><<<wblocks, 128, 0, ws>>>(wp); }
          // (dense: runs only if this launch's box exceeds the dense buffer)
          const unsigned fwb = dense ? std::min(wblocks, 148u * 16u) : wblocks;
          if (k32) walk_cw_kernel<true, false><<<fwb, 128, 0, ws>>>(wp); else walk_cw_kernel<false, false><<<fwb, 128, 0, ws>>>(wp);
        }
      } else if (rgb) {
        if (cw) { if (k32) walk_kernel<true, true, true, true><<<wblocks, 128, 0, ws>>>(wp); else walk_kernel<true, true, false, true><<<wblocks, 128, 0, ws>>>(wp); }
        else { if (k32) walk_kernel<true, false, true, true><<<wblocks, 128, 0, ws>>>(wp); else walk_kernel<true, false, false, true><<<wblocks, 128, 0, ws>>>(wp); }
      } else if (sm->aggregate) {
        if (cw) { if (k32) walk_kernel<true, true, true><<<wblocks, 128, 0, ws>>>(wp); else walk_kernel<true, true, false><<<wblocks, 128, 0, ws>>>(wp); }
        else { if (k32) walk_kernel<true, false, true><<<wblocks, 128, 0, ws>>>(wp); else walk_kernel<true, false, false><<<wblocks, 128, 0, ws>>>(wp); }
      } else {
        walk_kernel<false, false, false><<<wblocks, 128, 0, ws>>>(wp);
      }
    }
    if (ws != st) { cudaEventRecord(sm->ev_w[1], ws); cudaStreamWaitEvent(st, sm->ev_w[1], 0); }
    if (dense && last_launch && sm->defer_fold) {
      // the call's last dense fold is deferred to the next call that reads or changes the submap (flush_fold):
      // a caller that integrates the next submap meanwhile overlaps this fold with that submap's walk
      cudaEventRecord(sm->ev_walked, st);
      sm->fold_pending = true; sm->fold_buf = b; sm->fold_dcap = dcap; sm->fold_color = rgb != nullptr;
    } else if (dense) {
      ProfScope ps_(sm, "dense_fold_allocate", st);
      dense_fold_kernel<<<148 * 8, 256, 0, st>>>(wp);
    }
    if (cw) pending += total;
    cudaEventRecord(sm->ev_free[b], st);
    f0 += nf;
  }
  fold();
  return cudaGetLastError();
}


// Projection-mapping integration (R14), all on the caller's stream:
//   record the block count at entry and clear the birth frames;
//   per group of <= kMaxBatch frames: ALLOCATE in launches of <= kLaunchRays rays (compose, prepare with
//   frame tags, block walk recording each new block's birth frame with one RED.MIN per run), then ONE
//   project_kernel over every block for all frames of the group.
cudaError_t launch_integrate_projective(cvx_submap* sm, const float* depth, int64_t n_per_frame, int n_frames,
                                        const double* T_world_sensor, const cvx_sensor_model& sensor,
                                        cudaStream_t st) {
  if (cudaError_t fe = flush_fold(sm, st)) return fe;
  if (n_per_frame <= 0 || n_frames <= 0) return cudaSuccess;
  const int lim = (int)std::max<long long>(1, std::min<long long>(kMaxBatch, kLaunchRays / n_per_frame));
  cvx_submap::Buf& B = sm->buf[0];
  cudaStreamWaitEvent(st, sm->ev_free[0], 0);   // the walk that last read buffer 0 (stream-ordered growth)
  cudaError_t e = grow(&B.rays, &B.ray_cap, (long long)lim * n_per_frame, sizeof(RayRec), st);
  if (e == cudaSuccess)
    e = grow(reinterpret_cast<void**>(&B.slot_lists), &B.slot_cap, (long long)lim * n_per_frame * kSlotsPerRay + 1024,
             sizeof(int), st);
  if (e == cudaSuccess && !sm->proj_birth) {
    e = cudaMallocAsync(reinterpret_cast<void**>(&sm->proj_birth), sizeof(int) * ((size_t)sm->pool.max_blocks + 1), st);
    if (e == cudaSuccess) sm->proj_start = sm->proj_birth + sm->pool.max_blocks;
  }
  if (e != cudaSuccess) return e;
  const int q = packed_q(sm->cfg.truncation);
  const bool k32 = ((double)sensor.max_range + sm->cfg.truncation) / sm->cfg.voxel_size + 2.0 < 4096.0;
  cudaMemsetAsync(sm->proj_birth, 0x7f, sizeof(int) * (size_t)sm->pool.max_blocks, st);   // "never"
  record_count_kernel<<<1, 1, 0, st>>>(sm->ctr, sm->proj_start, 0, sm->pool.max_blocks);
  auto compose = [&](int f0, int nf, double* out) {
    ComposeParams cp;
    for (int i = 0; i < 16; ++i) cp.Tws[i] = sm->T_ws[i];
    for (int f = 0; f < nf; ++f)
      for (int i = 0; i < 16; ++i) cp.Twc[f][i] = T_world_sensor[16 * (f0 + f) + i];
    cp.n = nf;
    cp.s = sm->cfg.voxel_size;
    ProfScope ps_(sm, "compose_poses", st);
    compose_kernel<<<1, kMaxBatch, 0, st>>>(cp, out);
  };
  for (int g0 = 0; g0 < n_frames; g0 += kMaxBatch) {
    const int gn = std::min(kMaxBatch, n_frames - g0);
    for (int f0 = g0; f0 < g0 + gn; f0 += lim) {   // ALLOCATE launches
      const int nf = std::min(lim, g0 + gn - f0);
      const long long total = (long long)nf * n_per_frame;
      const unsigned blocks = (unsigned)((total + 255) / 256);
      compose(f0, nf, B.frame_T);
      cudaMemsetAsync(B.lcnt, 0, 4 * sizeof(int), st);
      PrepParams pp{};
      pp.data = depth + (long long)f0 * n_per_frame;
      pp.n_per_frame = n_per_frame; pp.total = total;
      pp.kind = sensor.kind; pp.width = sensor.width;
      pp.fx = sensor.fx; pp.fy = sensor.fy; pp.cx = sensor.cx; pp.cy = sensor.cy;
      pp.rmin = (double)sensor.min_range; pp.rmax = (double)sensor.max_range;
      pp.s = sm->cfg.voxel_size; pp.tau = sm->cfg.truncation; pp.rfloor = sm->cfg.weight_range_floor;
      pp.weighting = sm->cfg.weighting; pp.carve = sm->cfg.carve;
      pp.sdf_scale = std::ldexp(1.0, q + kSdfF);
      set_divisors(pp, sensor);
      pp.height = sensor.height;
      pp.frame_T = B.frame_T; pp.rays = (RayRec*)B.rays; pp.ctr = sm->ctr; pp.lcnt = B.lcnt;
      pp.list_cap = (int)std::min<long long>(B.slot_cap - 1, 0x7fffffffll);
      pp.trig = nullptr;
      pp.rgb = nullptr;
      pp.rgbs = nullptr;
      pp.ws = nullptr;
      pp.count_vox = 0;   // voxel_updates counts the projective updates instead
      {
        ProfScope ps_(sm, "ray_prepare", st);
        prepare_kernel<<<(unsigned)((total + kPrepThreads - 1) / kPrepThreads), kPrepThreads, 0, st>>>(pp);
      }
      WalkParams wp{};
      wp.rays = (const RayRec*)B.rays; wp.ctr = sm->ctr; wp.hash = sm->hash; wp.pool = sm->pool;
      wp.slots = B.slot_lists; wp.lcnt = B.lcnt;
      wp.s = (float)sm->cfg.voxel_size; wp.tau = (float)sm->cfg.truncation;
      wp.tq = (int)std::llround(std::ldexp(sm->cfg.truncation, q));
      wp.q = q;
      wp.band = 0;
      wp.birth = sm->proj_birth;
      wp.frame_T = B.frame_T; wp.rgbs = nullptr; wp.ws = nullptr; wp.frame_base = f0;   // birth = f0 + frame
      {
        ProfScope ps_(sm, "block_walk_allocate", st);
        if (k32) block_walk2_kernel<true, true><<<blocks, 256, 0, st>>>(wp);
        else block_walk2_kernel<false, true><<<blocks, 256, 0, st>>>(wp);
      }
    }
    compose(g0, gn, sm->buf[1].frame_T);
    ProjParams pj;
    pj.depth = depth + (long long)g0 * n_per_frame;
    pj.frame_T = sm->buf[1].frame_T; pj.start = sm->proj_start; pj.birth = sm->proj_birth; pj.frame_base = g0;
    pj.pool = sm->pool; pj.ctr = sm->ctr;
    pj.nf = gn; pj.width = sensor.width; pj.height = sensor.height;
    pj.fx = sensor.fx; pj.fy = sensor.fy; pj.cx = sensor.cx; pj.cy = sensor.cy;
    pj.rmin = (double)sensor.min_range; pj.rmax = (double)sensor.max_range;
    pj.s = sm->cfg.voxel_size; pj.tau = sm->cfg.truncation; pj.rfloor = sm->cfg.weight_range_floor;
    pj.weighting = sm->cfg.weighting; pj.carve = sm->cfg.carve; pj.q = q;
    {
      ProfScope ps_(sm, "project_update", st);
      project_kernel<<<148 * 8, kProjThreads, 0, st>>>(pj);
    }
  }
  return cudaGetLastError();
}

}  // namespace cvx
