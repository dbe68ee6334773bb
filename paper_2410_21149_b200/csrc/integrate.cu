// integrate.cu — TSDF integration kernels for sm_100a.
//
//   compose_kernel  O1   T_SC = T_WS^-1 T_WC per frame (fp64, fixed order, no FMA)
//   prepare_kernel  a1+a2  point -> ray (O2-O3, O6), range filter, fixed-point endpoints, closed-form
//                        voxel count n_r = 1 + sum|dv| (COUNT) with warp-local counters
//                        reduced once per warp, warp-ballot compaction of the used rays
//   walk_kernel     a3+a4+a5  exact integer 6-connected traversal (O4); on entering a block the ray
//                        activates it in the hash table (ALLOCATE); every voxel gets the
//                        projective sdf (O5) and (w d, w) is merged per voxel — lanes of a warp
//                        hitting the same voxel are reduced with match.any + a shuffle tree, then one
//                        64-bit red.global.add per distinct voxel per warp step.  The TSDF state IS the
//                        pair of exact fixed-point sums, so the "fold" D = sum(wd)/sum(w) (a5)
//                        is evaluated on read (export / finalize) and fusion is order-independent and
//                        deterministic (R6).
//   reset kernels   zero the used blocks, counters and AABB.
#include <cstdio>

#include "submap.h"

namespace cvx {
namespace {

struct __align__(16) RayRec {
  long long A[3];   // fixed-point (2^-16 voxel) start of the updated segment (O3)
  long long B[3];   // fixed-point end: p + tau*u
  int vp[3];        // voxel containing p (precision anchor for the sdf)
  float w;          // weight (O6)
  float pm[3];      // p/s - vp - 1/2 (voxel units, in [-1/2, 1/2))
  int n_vox;        // closed-form voxel count (COUNT)
  float u[3];       // unit ray direction
  int pad;
};
static_assert(sizeof(RayRec) == 96, "RayRec layout");

struct ComposeParams {
  double Tws[16];
  double Twc[kMaxBatch][16];
  int n;
};

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// O1: R_SC[i][j] = ((Rws[0][i] Rwc[0][j] + Rws[1][i] Rwc[1][j]) + Rws[2][i] Rwc[2][j]),
// t_SC[i] = ((Rws[0][i](twc0-tws0) + Rws[1][i](twc1-tws1)) + Rws[2][i](twc2-tws2)).
__global__ void compose_kernel(const __grid_constant__ ComposeParams p, double* out) {
  int f = threadIdx.x;
  if (f >= p.n) return;
  const double* W = p.Tws;
  const double* C = p.Twc[f];
  double* o = out + 12 * f;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j)
      o[3 * i + j] = da(da(dm(W[0 * 4 + i], C[0 * 4 + j]), dm(W[1 * 4 + i], C[1 * 4 + j])), dm(W[2 * 4 + i], C[2 * 4 + j]));
    o[9 + i] = da(da(dm(W[0 * 4 + i], ds(C[3], W[3])), dm(W[1 * 4 + i], ds(C[7], W[7]))),
                  dm(W[2 * 4 + i], ds(C[11], W[11])));
  }
}

struct PrepParams {
  const float* data;
  long long n_per_frame;
  long long total;
  int kind, width;
  float fx, fy, cx, cy;
  double rmin, rmax, s, tau, rfloor;
  int weighting, carve;
  const double* frame_T;
  RayRec* rays;
  Counters* ctr;
};

// O3: q(x) = floor((x / s) * 2^16), rejected outside |voxel| < 2^23.
__device__ __forceinline__ bool quantise(double x, double s, long long* q) {
  double a = dm(__ddiv_rn(x, s), 65536.0);
  if (!(fabs(a) < 549755813888.0)) return false;
  *q = (long long)floor(a);
  return true;
}

__global__ void __launch_bounds__(256) prepare_kernel(const __grid_constant__ PrepParams p) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int status = -1;  // -1 no thread, 0 used, 1 invalid, 2 range, 3 domain
  RayRec rec;
  if (idx < p.total) {
    const long long f = idx / p.n_per_frame, i = idx - f * p.n_per_frame;
    const double* T = p.frame_T + 12 * f;
    double pc[3];
    status = 0;
    if (p.kind == 1) {  // O2: pinhole depth -> point in fp32 exactly as written, integer pixel (Q24)
      float z = p.data[idx];
      if (!(z > 0.0f) || !isfinite(z)) status = 1;
      float u = (float)(int)(i % p.width), v = (float)(int)(i / p.width);
      pc[0] = (double)__fdiv_rn(__fmul_rn(z, __fsub_rn(u, p.cx)), p.fx);
      pc[1] = (double)__fdiv_rn(__fmul_rn(z, __fsub_rn(v, p.cy)), p.fy);
      pc[2] = (double)z;
    } else {
      const float* q = p.data + 3 * idx;
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
        for (int a = 0; a < 3 && status == 0; ++a) {
          double ext = __ddiv_rn(dm(p.tau, d[a]), L);
          double e = da(pw[a], ext);                         // tau behind the point
          double st = p.carve ? T[9 + a] : ds(pw[a], ext);   // from the optical centre (Q2)
          if (!quantise(st, p.s, &rec.A[a]) || !quantise(e, p.s, &rec.B[a])) status = 3;
          else {
            long long span = (rec.B[a] >> 16) - (rec.A[a] >> 16);
            if (span >= 32768 || span <= -32768) status = 3;
          }
          double ps = __ddiv_rn(pw[a], p.s);
          double fl = floor(ps);
          rec.vp[a] = (int)fl;
          rec.pm[a] = (float)(ps - fl) - 0.5f;
          rec.u[a] = (float)__ddiv_rn(d[a], L);
        }
        if (p.weighting == 0) rec.w = 1.0f;                  // O6
        else { double r = fmax(L, p.rfloor); rec.w = (float)__ddiv_rn(1.0, dm(r, r)); }
        rec.n_vox = 1;
        for (int a = 0; a < 3; ++a) {
          long long dv = (rec.B[a] >> 16) - (rec.A[a] >> 16);
          rec.n_vox += (int)(dv < 0 ? -dv : dv);             // a2: n_r = 1 + sum |dv| (O4)
        }
        rec.pad = 0;
      }
    }
  }
  // warp-local counters, one atomic per warp ("each thread or block maintains its local
  // counter, and the results are combined at the end")
  const unsigned used = __ballot_sync(0xffffffffu, status == 0);
  const unsigned n_in = __popc(__ballot_sync(0xffffffffu, status >= 0));
  const unsigned n_inv = __popc(__ballot_sync(0xffffffffu, status == 1));
  const unsigned n_rng = __popc(__ballot_sync(0xffffffffu, status == 2));
  const unsigned n_dom = __popc(__ballot_sync(0xffffffffu, status == 3));
  const unsigned nv = __reduce_add_sync(0xffffffffu, status == 0 ? (unsigned)rec.n_vox : 0u);
  int base = 0;
  if (lane == 0) {
    if (used) base = atomicAdd(&p.ctr->n_rays, __popc(used));
    if (n_in) atomicAdd(&p.ctr->rays_in, (unsigned long long)n_in);
    if (used) atomicAdd(&p.ctr->rays_used, (unsigned long long)__popc(used));
    if (n_inv) atomicAdd(&p.ctr->skipped_invalid, (unsigned long long)n_inv);
    if (n_rng) atomicAdd(&p.ctr->skipped_range, (unsigned long long)n_rng);
    if (n_dom) { atomicAdd(&p.ctr->skipped_domain, (unsigned long long)n_dom); atomicOr(&p.ctr->err, (unsigned)kErrRange); }
    if (nv) atomicAdd(&p.ctr->voxel_updates, (unsigned long long)nv);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (status == 0) {
    const int pos = base + __popc(used & ((1u << lane) - 1u));   // order-preserving within the warp
    p.rays[pos] = rec;
  }
}

struct WalkParams {
  const RayRec* rays;
  Counters* ctr;
  HashView hash;
  PoolView pool;
  float s, tau;
};

constexpr long long kMax = 0x7fffffffffffffffll;

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

__global__ void __launch_bounds__(256) walk_kernel(const __grid_constant__ WalkParams p) {
  const int n_rays = *(volatile int*)&p.ctr->n_rays;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((idx & ~31) >= n_rays) return;                       // whole warp beyond the rays
  const bool have = idx < n_rays;

  int v0 = 0, v1 = 0, v2 = 0, s0 = 1, s1 = 1, s2 = 1, k0 = 0, k1 = 0, k2 = 0;
  long long X01 = kMax, X10 = 0, X02 = kMax, X20 = 0, X12 = kMax, X21 = 0;
  long long I01 = 0, I10 = 0, I02 = 0, I20 = 0, I12 = 0, I21 = 0;
  float d0 = 0, d1 = 0, d2 = 0, u0 = 0, u1 = 0, u2 = 0, pm0 = 0, pm1 = 0, pm2 = 0;
  int vp0 = 0, vp1 = 0, vp2 = 0, n = 0;
  long long w_fx = 0;
  float w = 0.0f;
  if (have) {
    const RayRec r = p.rays[idx];
    long long A[3] = {r.A[0], r.A[1], r.A[2]}, B[3] = {r.B[0], r.B[1], r.B[2]};
    long long R[3], AD[3];
    int va[3], st[3], kk[3];
    for (int a = 0; a < 3; ++a) {
      va[a] = (int)(A[a] >> 16);
      int vb = (int)(B[a] >> 16);
      long long D = B[a] - A[a];
      kk[a] = vb > va[a] ? vb - va[a] : va[a] - vb;
      if (D > 0) { st[a] = 1; R[a] = (((long long)va[a] + 1) << 16) - A[a]; }
      else { st[a] = -1; R[a] = A[a] - ((long long)va[a] << 16); }
      AD[a] = D < 0 ? -D : D;
    }
    v0 = va[0]; v1 = va[1]; v2 = va[2]; s0 = st[0]; s1 = st[1]; s2 = st[2]; k0 = kk[0]; k1 = kk[1]; k2 = kk[2];
    // X_ij = r_i |D_j|: axis i crosses before axis j  <=>  X_ij < X_ji  (O4, exact in int64)
    X01 = R[0] * AD[1]; X10 = R[1] * AD[0]; X02 = R[0] * AD[2]; X20 = R[2] * AD[0];
    X12 = R[1] * AD[2]; X21 = R[2] * AD[1];
    I01 = AD[1] << 16; I10 = AD[0] << 16; I02 = AD[2] << 16; I20 = AD[0] << 16; I12 = AD[2] << 16; I21 = AD[1] << 16;
    if (k0 == 0) { X01 = kMax; X02 = kMax; X10 = 0; X20 = 0; }
    if (k1 == 0) { X10 = kMax; X12 = kMax; X01 = 0; X21 = 0; }
    if (k2 == 0) { X20 = kMax; X21 = kMax; X02 = 0; X12 = 0; }
    if (k0 == 0 && k1 == 0) { X01 = kMax; X10 = kMax; }
    if (k0 == 0 && k2 == 0) { X02 = kMax; X20 = kMax; }
    if (k1 == 0 && k2 == 0) { X12 = kMax; X21 = kMax; }
    u0 = r.u[0]; u1 = r.u[1]; u2 = r.u[2];
    pm0 = r.pm[0]; pm1 = r.pm[1]; pm2 = r.pm[2];
    vp0 = r.vp[0]; vp1 = r.vp[1]; vp2 = r.vp[2];
    d0 = pm0 - (float)(v0 - vp0); d1 = pm1 - (float)(v1 - vp1); d2 = pm2 - (float)(v2 - vp2);
    w = r.w;
    w_fx = __double2ll_rn((double)w * kFxScale);
    n = r.n_vox;
  }
  const int maxn = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
  int slot = kFailed;
  bool need_block = true;
  const float s = p.s, tau = p.tau;
  for (int it = 0; it < maxn; ++it) {
    const bool act = it < n;
    if (act && need_block) {
      const int bx = v0 >> 3, by = v1 >> 3, bz = v2 >> 3;
      slot = hash_activate(p.hash, p.pool, p.ctr, pack_key(bx, by, bz), bx, by, bz);
      need_block = false;
    }
    const bool upd = act && slot >= 0;
    const unsigned m = __ballot_sync(0xffffffffu, upd);
    if (upd) {
      // O5: sdf = (p - c_v).u, in voxel units relative to the voxel of p, clamped before fusion (Q4)
      const float sdf = s * (d0 * u0 + d1 * u1 + d2 * u2);
      const float dcl = fminf(fmaxf(sdf, -tau), tau);
      long long a = __float2ll_rn((w * dcl) * 4294967296.0f);
      long long b = w_fx;
      const unsigned addr = (unsigned)slot * 512u + (unsigned)((v0 & 7) | ((v1 & 7) << 3) | ((v2 & 7) << 6));
      const unsigned peers = __match_any_sync(m, addr);
      reduce_peers(m, peers, lane, a, b);
      if (lane == __ffs(peers) - 1) {
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(p.pool.sums) + 2ull * addr;
        atomicAdd(dst, (unsigned long long)a);
        atomicAdd(dst + 1, (unsigned long long)b);
      }
    }
    if (act && it + 1 < n) {
      // O4: next axis = earliest crossing, ties x < y < z
      int ax = (X10 < X01) ? 1 : 0;
      if (ax == 0) { if (X20 < X02) ax = 2; }
      else { if (X21 < X12) ax = 2; }
      if (ax == 0) {
        v0 += s0; X01 += I01; X02 += I02; --k0;
        d0 = pm0 - (float)(v0 - vp0);
        need_block = (v0 & 7) == (s0 > 0 ? 0 : 7);
        if (k0 == 0) { X01 = kMax; X02 = kMax; X10 = 0; X20 = 0; }
      } else if (ax == 1) {
        v1 += s1; X10 += I10; X12 += I12; --k1;
        d1 = pm1 - (float)(v1 - vp1);
        need_block = (v1 & 7) == (s1 > 0 ? 0 : 7);
        if (k1 == 0) { X10 = kMax; X12 = kMax; X01 = 0; X21 = 0; }
      } else {
        v2 += s2; X20 += I20; X21 += I21; --k2;
        d2 = pm2 - (float)(v2 - vp2);
        need_block = (v2 & 7) == (s2 > 0 ? 0 : 7);
        if (k2 == 0) { X20 = kMax; X21 = kMax; X02 = 0; X12 = 0; }
      }
    }
  }
}

__global__ void zero_blocks_kernel(Counters* ctr, long long* sums, int max_blocks) {
  const int nb = min(*(volatile int*)&ctr->n_blocks, max_blocks);
  const long long n16 = (long long)nb * kBlockVox;   // one longlong2 per voxel
  longlong2* s2 = reinterpret_cast<longlong2*>(sums);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    s2[i] = make_longlong2(0, 0);
}

__global__ void reset_counters_kernel(Counters* ctr) {
  Counters c = {};
  c.aabb_lo[0] = c.aabb_lo[1] = c.aabb_lo[2] = 0x7fffffff;
  c.aabb_hi[0] = c.aabb_hi[1] = c.aabb_hi[2] = (int)0x80000000;
  *ctr = c;
}

}  // namespace

cudaError_t launch_reset(cvx_submap* sm, cudaStream_t st) {
  {
    ProfScope ps_(sm, "reset_zero_blocks", st);
    zero_blocks_kernel<<<148 * 8, 256, 0, st>>>(sm->ctr, sm->pool.sums, sm->pool.max_blocks);
  }
  {
    ProfScope ps_(sm, "reset_counters", st);
    reset_counters_kernel<<<1, 1, 0, st>>>(sm->ctr);
  }
  cudaMemsetAsync(sm->hash.keys, 0xff, sizeof(unsigned long long) * ((size_t)sm->hash.mask + 1), st);
  cudaMemsetAsync(sm->hash.vals, 0xff, sizeof(int) * ((size_t)sm->hash.mask + 1), st);
  return cudaGetLastError();
}

cudaError_t launch_integrate(cvx_submap* sm, const float* data, int64_t n_per_frame, int n_frames,
                             const double* T_world_sensor, const cvx_sensor_model& sensor, cudaStream_t st) {
  const long long total = (long long)n_per_frame * n_frames;
  if (total <= 0) return cudaSuccess;
  if (sm->ray_cap < total) {
    if (sm->rays) cudaFree(sm->rays);
    sm->rays = nullptr;
    sm->ray_cap = 0;
    cudaError_t e = cudaMalloc(&sm->rays, sizeof(RayRec) * (size_t)total);
    if (e != cudaSuccess) return e;
    sm->ray_cap = total;
  }
  ComposeParams cp;
  for (int i = 0; i < 16; ++i) cp.Tws[i] = sm->T_ws[i];
  for (int f = 0; f < n_frames; ++f)
    for (int i = 0; i < 16; ++i) cp.Twc[f][i] = T_world_sensor[16 * f + i];
  cp.n = n_frames;
  {
    ProfScope ps_(sm, "compose_poses", st);
    compose_kernel<<<1, kMaxBatch, 0, st>>>(cp, sm->frame_T);
  }
  cudaMemsetAsync(&sm->ctr->n_rays, 0, sizeof(int), st);

  PrepParams pp;
  pp.data = data; pp.n_per_frame = n_per_frame; pp.total = total;
  pp.kind = sensor.kind; pp.width = sensor.width;
  pp.fx = sensor.fx; pp.fy = sensor.fy; pp.cx = sensor.cx; pp.cy = sensor.cy;
  pp.rmin = (double)sensor.min_range; pp.rmax = (double)sensor.max_range;
  pp.s = sm->cfg.voxel_size; pp.tau = sm->cfg.truncation; pp.rfloor = sm->cfg.weight_range_floor;
  pp.weighting = sm->cfg.weighting; pp.carve = sm->cfg.carve;
  pp.frame_T = sm->frame_T; pp.rays = (RayRec*)sm->rays; pp.ctr = sm->ctr;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  {
    ProfScope ps_(sm, "ray_prepare", st);
    prepare_kernel<<<blocks, 256, 0, st>>>(pp);
  }

  WalkParams wp;
  wp.rays = (const RayRec*)sm->rays; wp.ctr = sm->ctr; wp.hash = sm->hash; wp.pool = sm->pool;
  wp.s = (float)sm->cfg.voxel_size; wp.tau = (float)sm->cfg.truncation;
  {
    ProfScope ps_(sm, "ray_walk_update", st);
    walk_kernel<<<blocks, 256, 0, st>>>(wp);
  }
  return cudaGetLastError();
}

}  // namespace cvx
