// l2_atomics.cu — microbenchmark of scattered global reductions on B200 (sm_100a): the ceiling the
// TSDF update kernel (ray_walk_update) is measured against.  Not part of libcvx.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_atomics l2_atomics.cu && ./l2_atomics
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0: one RED.64 per op; 1: two RED.64 to adjacent 8-byte words (the TSDF sums layout);
// 2: RED.32; 3: float2 vector atomicAdd (RED.v2.f32); 4: one RED.64 with spatially coherent lanes
// (lane l of a warp hits word base+l -> 32 distinct words in 2 lines)
template <int kMode>
__global__ void red_kernel(unsigned long long* buf64, unsigned* buf32, float2* bufv, uint32_t mask, int iters) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    uint32_t h = hash32(tid * 2654435761u + i * 40503u);
    if (kMode == 4) h = (hash32((tid >> 5) * 977u + i) & ~31u) | (tid & 31);
    const uint32_t a = h & mask;
    if (kMode == 0) atomicAdd(buf64 + a, 1ull);
    if (kMode == 1) { atomicAdd(buf64 + 2 * (a >> 1), 3ull); atomicAdd(buf64 + 2 * (a >> 1) + 1, 1ull); }
    if (kMode == 2) atomicAdd(buf32 + a, 1u);
    if (kMode == 3) atomicAdd(bufv + (a >> 1), make_float2(1.f, 2.f));
    if (kMode == 4) atomicAdd(buf64 + a, 1ull);
  }
}

template <int kMode>
double run(unsigned long long* b64, unsigned* b32, float2* bv, uint32_t mask, int blocks, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  red_kernel<kMode><<<blocks, 256>>>(b64, b32, bv, mask, iters);
  cudaEventRecord(e0);
  red_kernel<kMode><<<blocks, 256>>>(b64, b32, bv, mask, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * 256 * iters * (kMode == 1 ? 2 : 1);
  return ops / (ms * 1e-3) / 1e9;
}

int main() {
  const size_t words = 1ull << 26;  // 512 MB of u64
  unsigned long long* b64; unsigned* b32; float2* bv;
  cudaMalloc(&b64, words * 8); cudaMalloc(&b32, words * 4); cudaMalloc(&bv, words * 8);
  cudaMemset(b64, 0, words * 8); cudaMemset(b32, 0, words * 4); cudaMemset(bv, 0, words * 8);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, iters = 256;
  printf("{\"sms\": %d", sms);
  const uint32_t masks[] = {(1u << 22) - 1, (1u << 24) - 1, (1u << 26) - 1};   // 32 MB, 128 MB, 512 MB (u64)
  const char* names[] = {"32MB", "128MB", "512MB"};
  for (int m = 0; m < 3; ++m) {
    printf(", \"%s\": {\"red64_Gops\": %.1f, \"red64_pair_Gops\": %.1f, \"red32_Gops\": %.1f, \"redv2f32_Gops\": %.1f, "
           "\"red64_coherent_Gops\": %.1f}", names[m],
           run<0>(b64, b32, bv, masks[m], blocks, iters), run<1>(b64, b32, bv, masks[m], blocks, iters),
           run<2>(b64, b32, bv, masks[m], blocks, iters), run<3>(b64, b32, bv, masks[m], blocks, iters),
           run<4>(b64, b32, bv, masks[m], blocks, iters));
  }
  printf("}\n");
  return 0;
}
