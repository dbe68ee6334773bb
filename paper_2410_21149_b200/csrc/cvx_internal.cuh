// cvx_internal.cuh — device-side state and helpers of libcvx (sm_100a).  Not part of the C-ABI.
//
// HBM layout of one submap:
//   table {u64 key, i32 slot, pad} [cap]  open-addressing hash table of packed 21-bit block keys
//                            (P:L78-85); slot is PENDING while the inserter publishes it
//   sums  i64x2 [max_blocks*512]  per voxel (sum w*d, sum w) in fixed point 2^-30 (O8 as exact sums)
//   acc   u64 [max_blocks*512]    packed per-launch accumulator {count:22 | sum d':42} (constant w)
//   esdf  f32 [max_blocks*512]    E per voxel (after finalize)
//   coords i32x4 [max_blocks]     slot -> block coordinates
//   ctr   Counters                pool bump index, AABB, sticky errors, stats
// Voxel local index inside a block: lx + 8 ly + 64 lz (O9); slot s owns voxels [s*512, s*512+512).
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

// Bounds-checked build (CVX_BOUNDS=1, tests/test_gpu_bounds.py): the hot kernels check the indices of
// their global writes / reductions and trap with a message on a violation (compute-sanitizer's memcheck
// is not available on every GPU pool).  Compiled out otherwise.
#ifndef CVX_BOUNDS
#define CVX_BOUNDS 0
#endif
#if CVX_BOUNDS
#include <cstdio>
#define CVX_CHECK(cond, what)                                                                       \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("cvx bounds check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,   \
             (int)blockIdx.x, (int)threadIdx.x);                                                    \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define CVX_CHECK(cond, what) do { } while (0)
#endif

namespace cvx {

constexpr int kBlockSide = 8;
constexpr int kBlockVox = 512;
constexpr unsigned long long kEmptyKey = ~0ull;
constexpr int kPending = -1;   // vals[] while the inserting thread publishes the slot
constexpr int kFailed = -2;    // pool overflow: updates to this block are dropped (CVX_E_CAPACITY)
constexpr double kFxScale = 1073741824.0;  // 2^30: fixed-point scale of the TSDF sums

enum ErrBits : unsigned { kErrCapacity = 1u, kErrHashFull = 2u, kErrRange = 4u };

struct Counters {
  int n_blocks;            // bump index of the block pool (may overshoot max_blocks on overflow)
  unsigned err;            // sticky ErrBits
  int aabb_lo[3];          // block coordinates
  int aabb_hi[3];
  unsigned long long rays_in, rays_used, skipped_invalid, skipped_range, skipped_domain, voxel_updates,
      new_blocks;
};

// One 16-byte entry per table slot so a probe is a single 128-bit load: {key, slot, pad}.
struct __align__(16) HashEntry {
  unsigned long long key;
  int val;
  int pad;
};

struct HashView {
  HashEntry* e;
  unsigned mask;           // cap - 1
  int log2cap;
};

struct PoolView {
  long long* sums;         // [max_blocks*512][2]
  unsigned long long* acc; // [max_blocks*512] packed per-launch accumulators (constant weights)
  long long* csum;         // colour: [max_blocks*512][4] exact sums {sum w, sum w r, sum w g, sum w b} (2^-30)
  unsigned long long* cacc;// colour: [max_blocks*512][2] packed per-launch {n<<42 | sum r, sum g<<32 | sum b}
  float* esdf;             // [max_blocks*512]
  int4* coords;            // [max_blocks]
  int max_blocks;
  int* grid;               // [kGridZ][kGridY][kGridX] dense slot cache of ALLOCATE
};

// 21-bit two's-complement fields per axis; never equals kEmptyKey.
__host__ __device__ inline unsigned long long pack_key(int bx, int by, int bz) {
  const unsigned long long m = (1ull << 21) - 1;
  return ((unsigned long long)(bx & (int)m) << 42) | ((unsigned long long)(by & (int)m) << 21) |
         (unsigned long long)(bz & (int)m);
}

__device__ inline unsigned hash_slot(unsigned long long key, const HashView& h) {
  return (unsigned)((key * 0x9E3779B97F4A7C15ull) >> (64 - h.log2cap));
}

__device__ inline int ld_volatile(const int* p) { return *(const volatile int*)p; }

__device__ __forceinline__ longlong2 ld_entry(const HashEntry* p) { return *reinterpret_cast<const longlong2*>(p); }

// Find-only probe: slot, or -1 if absent.  Table must be quiescent (no concurrent inserts).
__device__ inline int hash_find(const HashView& h, unsigned long long key) {
  unsigned i = hash_slot(key, h);
  for (unsigned p = 0; p <= h.mask; ++p) {
    const longlong2 en = ld_entry(h.e + i);
    if ((unsigned long long)en.x == key) return (int)(en.y & 0xffffffffll);
    if ((unsigned long long)en.x == kEmptyKey) return -1;
    i = (i + 1) & h.mask;
  }
  return -1;
}

// ASH-style activate: insert-if-absent and return the block's pool slot.  The winner of the
// key CAS claims a slot by bumping the pool index, records the block coordinates and AABB,
// then publishes the slot; concurrent finders of the same key wait for the publication.
// Keys only ever change EMPTY -> key, so the probe is a plain (L1-cacheable) 128-bit load of the
// {key, slot} entry: a stale EMPTY is corrected by the CAS, a stale PENDING by the volatile re-reads.
// `first` = the entry at hash_slot(key), already loaded by the caller (prefetched ahead of use).
__device__ inline int hash_activate_pf(const HashView& h, const PoolView& pool, Counters* ctr,
                                       unsigned long long key, int bx, int by, int bz, longlong2 first) {
  unsigned i = hash_slot(key, h);
  for (unsigned p = 0; p <= h.mask; ++p) {
    const longlong2 en = p == 0 ? first : ld_entry(h.e + i);
    unsigned long long k = (unsigned long long)en.x;
    if (k == key) {
      int v = (int)(en.y & 0xffffffffll);
      while (v == kPending) { __nanosleep(32); v = ld_volatile(&h.e[i].val); }
      return v;
    }
    if (k == kEmptyKey) {
      unsigned long long old = atomicCAS(&h.e[i].key, kEmptyKey, key);
      if (old == kEmptyKey) {
        int slot = atomicAdd(&ctr->n_blocks, 1);
        if (slot >= pool.max_blocks) {
          atomicOr(&ctr->err, (unsigned)kErrCapacity);
          slot = kFailed;
        } else {
          pool.coords[slot] = make_int4(bx, by, bz, 0);
          atomicMin(&ctr->aabb_lo[0], bx); atomicMin(&ctr->aabb_lo[1], by); atomicMin(&ctr->aabb_lo[2], bz);
          atomicMax(&ctr->aabb_hi[0], bx); atomicMax(&ctr->aabb_hi[1], by); atomicMax(&ctr->aabb_hi[2], bz);
          atomicAdd(&ctr->new_blocks, 1ull);
        }
        __threadfence();
        *(volatile int*)&h.e[i].val = slot;
        return slot;
      }
      if (old == key) {
        int v;
        while ((v = ld_volatile(&h.e[i].val)) == kPending) { __nanosleep(32); }
        return v;
      }
    }
    i = (i + 1) & h.mask;
  }
  atomicOr(&ctr->err, (unsigned)kErrHashFull);
  return kFailed;
}

__device__ inline int hash_activate(const HashView& h, const PoolView& pool, Counters* ctr,
                                    unsigned long long key, int bx, int by, int bz) {
  return hash_activate_pf(h, pool, ctr, key, bx, by, bz, ld_entry(h.e + hash_slot(key, h)));
}

// Packed accumulator u64 = count << kCntShift | sum(d'): between two folds at most kMaxPackedRays
// updates of one voxel (24-bit count), and the 40-bit field holds their sum of d' <= 2 round(tau 2^q)
// <= 2^16 with q = floor(log2(2^15 / tau)) (quantum tau 2^-15: rounding <= 1e-5 m at tau = 0.6 m).
constexpr int kCntShift = 40;
// Trash region of the accumulators after the pool (slots max_blocks ..): updates of blocks without a
// slot and of parked lanes land there; never folded or read.
constexpr int kTrashBlocks = 64;
constexpr long long kMaxPackedRays = (1ll << 24) - 1;
#ifndef CVX_LAUNCH_LOG2
#define CVX_LAUNCH_LOG2 24
#endif
constexpr long long kLaunchRays = (1ll << CVX_LAUNCH_LOG2) - 1;   // rays per walk launch (pipelining granularity)
static_assert(CVX_LAUNCH_LOG2 <= 24, "the fold runs once per 2^24 rays; a launch must not exceed it");
#ifndef CVX_HOST_LAUNCH_LOG2
#define CVX_HOST_LAUNCH_LOG2 24   // dense window (R19): one launch per configs[1] submap, e2e 6.59 -> 6.51 ms (2^23: two launches, two box folds)
#endif
constexpr long long kLaunchRaysHost = (1ll << CVX_HOST_LAUNCH_LOG2) - 1;   // host frames (copy pipelining)
inline int packed_q(double tau) {
  int q = (int)std::floor(std::log2(32768.0 / tau));
  return q < 0 ? 0 : (q > 30 ? 30 : q);
}

// Longest dense EDT axis (voxels, multiple of 8): 2 (n - 1)^2 < 2^32 - 1, so the 2-D squared distances
// of the ESDF's second pass fit uint32 with 0xffffffff left as the "no site" marker.
constexpr long long kMaxEdtAxis = 46336;

// Dense slot cache of ALLOCATE (a3): a fixed window of 256 x 256 x 64 blocks around the submap origin
// (block (0, 0, 0)), entry = the block's pool slot or -1 (not known yet).  The hash table stays the
// authority: a -1 (or a block outside the window) goes through hash_activate, whose slot is then cached.
// Entries only ever go -1 -> slot between resets, so a stale -1 is merely a slower path.
constexpr int kGridX = 256, kGridY = 256, kGridZ = 64;
__host__ __device__ inline int grid_cache_index(int bx, int by, int bz) {
  const unsigned ux = (unsigned)(bx + kGridX / 2), uy = (unsigned)(by + kGridY / 2), uz = (unsigned)(bz + kGridZ / 2);
  if (ux >= (unsigned)kGridX || uy >= (unsigned)kGridY || uz >= (unsigned)kGridZ) return -1;
  return (int)((uz * kGridY + uy) * kGridX + ux);
}

// Floor division / modulo by 8 on int32 voxel coordinates (S:L200-207 floor semantics).
__host__ __device__ inline int bdiv(int v) { return v >> 3; }
__host__ __device__ inline int bmod(int v) { return v & 7; }

}  // namespace cvx
