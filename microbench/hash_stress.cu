// hash_stress.cu — hash-table stress test of libcvx's voxel-block hash (P:L239-244:
// "50 million insertions in the hash table ... under different loading factors", Fig. 7).  Not part of
// libcvx: it drives the library's own device functions (`hash_activate`, `hash_find` from
// paper_2410_21149_b200/csrc/cvx_internal.cuh) on random distinct block keys.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o hash_stress hash_stress.cu
//   ./hash_stress <log2_capacity> <load_factor> [<log2_capacity> <load_factor> ...]
//
// Per (capacity, load factor): n = load * capacity random distinct keys (a bijection of the key index
// onto the 63-bit key space, split into three 21-bit block coordinates) are activated once (insert path),
// then activated again (find-existing path), then looked up with hash_find.  Prints one JSON line each:
// ns per key per phase, mean / max probe distance, and self-checks (every key got a distinct slot in
// [0, n), the second activation and the lookup return the same slot).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "../paper_2410_21149_b200/csrc/cvx_internal.cuh"

using namespace cvx;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1); } } while (0)

// bijection on [0, 2^63): odd multiply and xor-shifts mod 2^63
__host__ __device__ inline unsigned long long mix63(unsigned long long x) {
  const unsigned long long M = (1ull << 63) - 1;
  x = (x * 0x9E3779B97F4A7C15ull) & M;
  x ^= x >> 29;
  x = (x * 0xBF58476D1CE4E5B9ull) & M;
  x ^= x >> 31;
  return x;
}

__device__ inline void key_coords(unsigned long long i, int* bx, int* by, int* bz) {
  const unsigned long long h = mix63(i);
  auto f = [](unsigned long long v) { return ((int)(v & 0x1fffff) << 11) >> 11; };   // 21-bit signed
  *bx = f(h >> 42); *by = f(h >> 21); *bz = f(h);
}

__global__ void activate_kernel(HashView h, PoolView pool, Counters* ctr, long long n, int* slots) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int bx, by, bz;
    key_coords((unsigned long long)i, &bx, &by, &bz);
    slots[i] = hash_activate(h, pool, ctr, pack_key(bx, by, bz), bx, by, bz);
  }
}

__global__ void find_kernel(HashView h, long long n, int* slots) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int bx, by, bz;
    key_coords((unsigned long long)i, &bx, &by, &bz);
    slots[i] = hash_find(h, pack_key(bx, by, bz));
  }
}

// probe distance of every occupied entry from its home slot; checks slot uniqueness via a bitmap
__global__ void probe_kernel(HashView h, long long n, unsigned long long* sum, unsigned* maxp, unsigned* seen,
                             unsigned long long* bad) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e <= (long long)h.mask;
       e += (long long)gridDim.x * blockDim.x) {
    const unsigned long long key = h.e[e].key;
    if (key == kEmptyKey) continue;
    const unsigned home = hash_slot(key, h);
    const unsigned d = ((unsigned)e - home) & h.mask;
    atomicAdd(sum, (unsigned long long)d);
    atomicMax(maxp, d);
    const int s = h.e[e].val;
    if (s < 0 || s >= n) { atomicAdd(bad, 1ull); continue; }
    const unsigned old = atomicOr(seen + (s >> 5), 1u << (s & 31));
    if (old & (1u << (s & 31))) atomicAdd(bad, 1ull);
  }
}

__global__ void compare_kernel(const int* a, const int* b, long long n, unsigned long long* bad) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (a[i] != b[i] || a[i] < 0) atomicAdd(bad, 1ull);
}

__global__ void reset_counters(Counters* c) {
  Counters z = {};
  z.aabb_lo[0] = z.aabb_lo[1] = z.aabb_lo[2] = 0x7fffffff;
  z.aabb_hi[0] = z.aabb_hi[1] = z.aabb_hi[2] = (int)0x80000000;
  *c = z;
}

int main(int argc, char** argv) {
  if (argc < 3 || (argc - 1) % 2) {
    std::fprintf(stderr, "usage: %s <log2_capacity> <load_factor> [...]\n", argv[0]);
    return 2;
  }
  for (int a = 1; a + 1 < argc; a += 2) {
    const int lg = std::atoi(argv[a]);
    const double lf = std::atof(argv[a + 1]);
    const long long cap = 1ll << lg;
    const long long n = (long long)(lf * (double)cap);
    HashView h;
    h.mask = (unsigned)(cap - 1);
    h.log2cap = lg;
    PoolView pool = {};
    pool.max_blocks = (int)n;
    Counters* ctr;
    int *s1, *s2, *s3;
    unsigned long long* stats;   // probe sum, bad
    unsigned *maxp, *seen;
    CK(cudaMalloc(&h.e, sizeof(HashEntry) * cap));
    CK(cudaMalloc(&pool.coords, sizeof(int4) * n));
    CK(cudaMalloc(&ctr, sizeof(Counters)));
    CK(cudaMalloc(&s1, sizeof(int) * n)); CK(cudaMalloc(&s2, sizeof(int) * n)); CK(cudaMalloc(&s3, sizeof(int) * n));
    CK(cudaMalloc(&stats, 16)); CK(cudaMalloc(&maxp, 4)); CK(cudaMalloc(&seen, 4 * ((n + 31) / 32)));
    cudaEvent_t e[4];
    for (auto& x : e) CK(cudaEventCreate(&x));
    const int grid = 148 * 16, tpb = 256;
    float best[3] = {1e30f, 1e30f, 1e30f};
    for (int rep = 0; rep < 3; ++rep) {   // insert is destructive: reset the table every repetition
      CK(cudaMemset(h.e, 0xff, sizeof(HashEntry) * cap));
      reset_counters<<<1, 1>>>(ctr);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e[0]));
      activate_kernel<<<grid, tpb>>>(h, pool, ctr, n, s1);
      CK(cudaEventRecord(e[1]));
      activate_kernel<<<grid, tpb>>>(h, pool, ctr, n, s2);
      CK(cudaEventRecord(e[2]));
      find_kernel<<<grid, tpb>>>(h, n, s3);
      CK(cudaEventRecord(e[3]));
      CK(cudaEventSynchronize(e[3]));
      for (int k = 0; k < 3; ++k) {
        float ms;
        CK(cudaEventElapsedTime(&ms, e[k], e[k + 1]));
        if (ms < best[k]) best[k] = ms;
      }
    }
    CK(cudaMemset(stats, 0, 16)); CK(cudaMemset(maxp, 0, 4)); CK(cudaMemset(seen, 0, 4 * ((n + 31) / 32)));
    probe_kernel<<<grid, tpb>>>(h, n, stats, maxp, seen, stats + 1);
    compare_kernel<<<grid, tpb>>>(s1, s2, n, stats + 1);
    compare_kernel<<<grid, tpb>>>(s1, s3, n, stats + 1);
    unsigned long long hs[2];
    unsigned hmax;
    Counters c;
    CK(cudaMemcpy(hs, stats, 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&hmax, maxp, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&c, ctr, sizeof(c), cudaMemcpyDeviceToHost));
    const bool ok = hs[1] == 0 && c.n_blocks == n && c.err == 0;
    std::printf("{\"capacity\": %lld, \"load_factor\": %.4f, \"keys\": %lld, \"insert_ms\": %.4f, \"insert_ns_per_key\": %.5f, "
                "\"reactivate_ns_per_key\": %.5f, \"find_ns_per_key\": %.5f, \"insert_gkeys_per_s\": %.3f, "
                "\"mean_probe\": %.4f, \"max_probe\": %u, \"blocks\": %d, \"errors\": %llu, \"ok\": %s}\n",
                cap, (double)n / (double)cap, n, best[0], 1e6 * best[0] / (double)n, 1e6 * best[1] / (double)n,
                1e6 * best[2] / (double)n, (double)n / (best[0] * 1e6), (double)hs[0] / (double)n, hmax, c.n_blocks,
                hs[1], ok ? "true" : "false");
    std::fflush(stdout);
    cudaFree(h.e); cudaFree(pool.coords); cudaFree(ctr); cudaFree(s1); cudaFree(s2); cudaFree(s3);
    cudaFree(stats); cudaFree(maxp); cudaFree(seen);
    for (auto& x : e) cudaEventDestroy(x);
    if (!ok) return 1;
  }
  return 0;
}
