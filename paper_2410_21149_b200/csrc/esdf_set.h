// esdf_set.h — host-side definition of the opaque cvx_esdf_set (gathered submap ESDFs, SURVEY §8 e / f4).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/cvx.h"
#include "cvx_internal.cuh"

struct cvx_esdf_set {
  int device = 0;
  int n = 0;                          // submaps
  const unsigned char* payload = nullptr;   // caller-owned device buffer (concatenated cvx_pack_esdf payloads)
  std::vector<double> T;              // host n x 16 T_world_submap (from the headers)
  std::vector<double> s;              // host voxel sizes
  std::vector<int64_t> n_blocks;      // host blocks per submap
  double* T_dev = nullptr;            // device n x 16, then voxel sizes
  long long* rec_off = nullptr;       // device n: byte offset of submap k's first record in the payload
  cvx::HashEntry* table = nullptr;    // (submap, block) -> record index inside its submap
  unsigned mask = 0;
  int log2cap = 0;
  unsigned* err = nullptr;            // device: bit 0 duplicate block, bit 1 span >= 8192 blocks
};

namespace cvx {
cudaError_t launch_set_build(cvx_esdf_set* set, cudaStream_t st, unsigned* err_host);
cudaError_t launch_set_query(const cvx_esdf_set* set, const int32_t* idx, const float* pts, int64_t m, float* out,
                             float* grad, uint8_t* status, cudaStream_t st);
}  // namespace cvx
