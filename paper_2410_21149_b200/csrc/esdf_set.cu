// esdf_set.cu — gathered submap ESDFs (SURVEY §8 row e, row f4; "ICP ... between every
// overlapped submap", the registration consumer of the multi-GPU gather).  A set indexes the records of
// several cvx_pack_esdf payloads in place (no copy of the E values): one open-addressing table maps
// (submap k, block) to the block's record, keyed by k << 39 | (bx, by, bz) mod 2^13 — injective because a
// finalized submap spans at most 46336 / 8 = 5792 < 2^13 blocks per axis (the dense EDT limit, checked).
// Queries take a submap index per point and run the O13 query of that submap in its own frame
// (T_world_submap from the payload header), value and gradient as cvx_query_distance_gradient.
#include "esdf_set.h"
#include "query_point.cuh"

namespace cvx {
namespace {

constexpr int kRecBytes = 16 + 4 * kBlockVox;

__device__ __forceinline__ unsigned long long set_key(int k, int bx, int by, int bz) {
  return ((unsigned long long)k << 39) | ((unsigned long long)(bx & 8191) << 26) |
         ((unsigned long long)(by & 8191) << 13) | (unsigned long long)(bz & 8191);
}
__device__ __forceinline__ unsigned set_slot(unsigned long long key, int log2cap) {
  return (unsigned)((key * 0x9E3779B97F4A7C15ull) >> (64 - log2cap));
}

struct SetBuild {
  const unsigned char* payload;
  const long long* rec_off;
  const long long* first;     // n + 1 prefix sums of the block counts
  int n;
  HashEntry* table;
  unsigned mask;
  int log2cap;
  int* lo;                    // n x 3 min block coordinate, then n x 3 max
  unsigned* err;
};

__global__ void set_span_kernel(const SetBuild b) {
  const long long total = b.first[b.n];
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < total; r += (long long)gridDim.x * blockDim.x) {
    int k = 0;
    while (b.first[k + 1] <= r) ++k;   // n is small (submaps of a trajectory)
    const int4 h = *reinterpret_cast<const int4*>(b.payload + b.rec_off[k] + (r - b.first[k]) * kRecBytes);
    atomicMin(&b.lo[6 * k + 0], h.x); atomicMin(&b.lo[6 * k + 1], h.y); atomicMin(&b.lo[6 * k + 2], h.z);
    atomicMax(&b.lo[6 * k + 3], h.x); atomicMax(&b.lo[6 * k + 4], h.y); atomicMax(&b.lo[6 * k + 5], h.z);
  }
}

__global__ void set_insert_kernel(const SetBuild b) {
  const long long total = b.first[b.n];
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < total; r += (long long)gridDim.x * blockDim.x) {
    int k = 0;
    while (b.first[k + 1] <= r) ++k;
    const int4 h = *reinterpret_cast<const int4*>(b.payload + b.rec_off[k] + (r - b.first[k]) * kRecBytes);
    for (int a = 0; a < 3; ++a) {
      const int span = b.lo[6 * k + 3 + a] - b.lo[6 * k + a];
      if (span >= 8192) atomicOr(b.err, 2u);
    }
    const unsigned long long key = set_key(k, h.x, h.y, h.z);
    unsigned i = set_slot(key, b.log2cap);
    for (unsigned p = 0; p <= b.mask; ++p) {
      const unsigned long long old = atomicCAS(&b.table[i].key, kEmptyKey, key);
      if (old == kEmptyKey) { b.table[i].val = (int)(r - b.first[k]); break; }
      if (old == key) { atomicOr(b.err, 1u); break; }   // the same block twice in one payload
      i = (i + 1) & b.mask;
    }
  }
}

struct SetQuery {
  const unsigned char* payload;
  const long long* rec_off;
  const double* T;            // n x 16, then n voxel sizes
  const HashEntry* table;
  unsigned mask;
  int log2cap;
  int n;
  const int* idx;
  const float* pts;
  long long m;
  float* out;
  float* grad;
  unsigned char* status;
};

__global__ void __launch_bounds__(256) set_query_kernel(const __grid_constant__ SetQuery q) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q.m) return;
  const int k = q.idx[i];
  if (k < 0 || k >= q.n) {   // no such submap: UNKNOWN
    const float qnan = __int_as_float(0x7fc00000);
    q.out[i] = qnan;
    q.status[i] = 2;
    if (q.grad) { q.grad[3 * i] = qnan; q.grad[3 * i + 1] = qnan; q.grad[3 * i + 2] = qnan; }
    return;
  }
  unsigned long long ckey = ~0ull;
  int crec = -1;
  const unsigned char* base = q.payload + q.rec_off[k];
  auto lookup = [&](int x, int y, int z, float* e) -> bool {
    if (!in_key_domain(x, y, z)) return false;
    const int bx = x >> 3, by = y >> 3, bz = z >> 3;
    const unsigned long long key = set_key(k, bx, by, bz);
    if (key != ckey) {
      ckey = key;
      crec = -1;
      unsigned s = set_slot(key, q.log2cap);
      for (unsigned p = 0; p <= q.mask; ++p) {
        const longlong2 en = *reinterpret_cast<const longlong2*>(q.table + s);
        if ((unsigned long long)en.x == key) { crec = (int)(en.y & 0xffffffffll); break; }
        if ((unsigned long long)en.x == kEmptyKey) break;
        s = (s + 1) & q.mask;
      }
      // the key keeps coordinates mod 2^13: confirm the record is this block
      if (crec >= 0) {
        const int4 h = *reinterpret_cast<const int4*>(base + (long long)crec * kRecBytes);
        if (h.x != bx || h.y != by || h.z != bz) crec = -1;
      }
    }
    if (crec < 0) return false;
    const float v = reinterpret_cast<const float*>(base + (long long)crec * kRecBytes + 16)[(x & 7) + 8 * (y & 7) + 64 * (z & 7)];
    if (isnan(v)) return false;
    *e = v;
    return true;
  };
  query_point(q.T + 16 * k, q.T[16 * q.n + k], q.pts + 3 * i, lookup, q.out + i, q.grad ? q.grad + 3 * i : nullptr,
              q.status + i);
}

}  // namespace

cudaError_t launch_set_build(cvx_esdf_set* set, cudaStream_t st, unsigned* err_host) {
  const int n = set->n;
  std::vector<long long> first(n + 1, 0), off(n);
  for (int k = 0; k < n; ++k) first[k + 1] = first[k] + set->n_blocks[k];
  const long long total = first[n];
  int log2cap = 10;
  while ((1ll << log2cap) < 2 * std::max<long long>(total, 1)) ++log2cap;
  set->log2cap = log2cap;
  set->mask = (unsigned)((1ll << log2cap) - 1);
  cudaError_t e;
  long long* first_dev = nullptr;
  int* lo = nullptr;
  if ((e = cudaMalloc(&set->table, sizeof(HashEntry) << log2cap)) != cudaSuccess ||
      (e = cudaMalloc(&first_dev, sizeof(long long) * (n + 1))) != cudaSuccess ||
      (e = cudaMalloc(&lo, sizeof(int) * 6 * n)) != cudaSuccess)
    return e;
  cudaMemsetAsync(set->table, 0xff, sizeof(HashEntry) << log2cap, st);
  cudaMemcpyAsync(first_dev, first.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, st);
  std::vector<int> lo_h(6 * n);
  for (int k = 0; k < n; ++k)
    for (int a = 0; a < 3; ++a) { lo_h[6 * k + a] = 0x7fffffff; lo_h[6 * k + 3 + a] = (int)0x80000000; }
  cudaMemcpyAsync(lo, lo_h.data(), sizeof(int) * 6 * n, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(set->err, 0, 4, st);
  SetBuild b{set->payload, set->rec_off, first_dev, n, set->table, set->mask, log2cap, lo, set->err};
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256 + 1, 148ll * 8);
  set_span_kernel<<<grid, 256, 0, st>>>(b);
  set_insert_kernel<<<grid, 256, 0, st>>>(b);
  cudaMemcpyAsync(err_host, set->err, 4, cudaMemcpyDeviceToHost, st);
  e = cudaStreamSynchronize(st);
  cudaFree(first_dev);
  cudaFree(lo);
  return e;
}

cudaError_t launch_set_query(const cvx_esdf_set* set, const int32_t* idx, const float* pts, int64_t m, float* out,
                             float* grad, uint8_t* status, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  SetQuery q{set->payload, set->rec_off, set->T_dev, set->table, set->mask, set->log2cap, set->n, idx, pts, m, out,
             grad, status};
  set_query_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(q);
  return cudaGetLastError();
}

}  // namespace cvx
