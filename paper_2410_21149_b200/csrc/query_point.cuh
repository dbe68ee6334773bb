// query_point.cuh — the per-point distance query of O13 (S:L486 trilinear over the 8 ESDF voxels around
// x; S:L491 the identity at a voxel centre) and its gradient (f4), shared by the single-submap
// query (query.cu) and the gathered-submap set query (esdf_set.cu).  `lookup(x, y, z, &e)` returns the
// E of integer voxel (x, y, z) of the submap, false if unallocated / unobserved / outside the key domain.
#pragma once
#include "cvx_internal.cuh"

namespace cvx {

template <class Lookup>
__device__ __forceinline__ void query_point(const double* T, double s, const float* pt, Lookup& lookup, float* out,
                                            float* grad, unsigned char* status) {
  auto dm = [](double a, double b) { return __dmul_rn(a, b); };
  auto da = [](double a, double b) { return __dadd_rn(a, b); };
  auto ds = [](double a, double b) { return __dsub_rn(a, b); };
  const double x[3] = {pt[0], pt[1], pt[2]};
  double xs[3], f[3];
  int i0[3];
  bool ok = true;
  for (int a = 0; a < 3; ++a) {   // x_s = T_WS^-1 x  (O13), same operation order as the oracle
    xs[a] = da(da(dm(T[0 * 4 + a], ds(x[0], T[3])), dm(T[1 * 4 + a], ds(x[1], T[7]))), dm(T[2 * 4 + a], ds(x[2], T[11])));
    const double g = ds(__ddiv_rn(xs[a], s), 0.5);
    const double fl = floor(g);
    if (!(fabs(fl) < 1073741824.0)) ok = false;
    i0[a] = ok ? (int)fl : 0;
    f[a] = ds(g, fl);
  }
  const float qnan = __int_as_float(0x7fc00000);
  if (ok) {
    double acc = 0.0, gs[3] = {0.0, 0.0, 0.0};
    bool all = true;
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
      float e;
      if (!lookup(i0[0] + dx, i0[1] + dy, i0[2] + dz, &e)) { all = false; break; }
      const double wx = dx ? f[0] : ds(1.0, f[0]), wy = dy ? f[1] : ds(1.0, f[1]), wz = dz ? f[2] : ds(1.0, f[2]);
      const double wgt = dm(dm(wx, wy), wz);
      if (wgt > 0) acc = da(acc, dm(wgt, (double)e));
      if (grad) {   // d/df of the trilinear weights (f4: value + gradient look-ups for registration)
        gs[0] += (dx ? 1.0 : -1.0) * wy * wz * (double)e;
        gs[1] += (dy ? 1.0 : -1.0) * wx * wz * (double)e;
        gs[2] += (dz ? 1.0 : -1.0) * wx * wy * (double)e;
      }
    }
    if (all) {
      *out = (float)acc;
      *status = 0;
      if (grad)   // dE/dx_world = R_WS dE/dx_s, dE/dx_s = (dE/df) / s
        for (int a = 0; a < 3; ++a) grad[a] = (float)((T[4 * a] * gs[0] + T[4 * a + 1] * gs[1] + T[4 * a + 2] * gs[2]) / s);
      return;
    }
    if (grad) { grad[0] = qnan; grad[1] = qnan; grad[2] = qnan; }
    int v[3];
    for (int a = 0; a < 3; ++a) {
      const double fv = floor(__ddiv_rn(xs[a], s));
      v[a] = fabs(fv) < 1073741824.0 ? (int)fv : (1 << 30);   // |v| >= 2^30: outside the key domain
    }
    float e;
    if (lookup(v[0], v[1], v[2], &e)) { *out = e; *status = 1; return; }
  }
  if (grad && !ok) { grad[0] = qnan; grad[1] = qnan; grad[2] = qnan; }
  *out = qnan;
  *status = 2;
}

// Voxel coordinates of the 21-bit block-key domain (O3: |voxel| < 2^23, blocks in [-2^20, 2^20)); a
// coordinate outside it cannot be allocated, and pack_key would alias it onto an in-range block.
__device__ __forceinline__ bool in_key_domain(int x, int y, int z) {
  constexpr int lo = -(1 << 23), hi = (1 << 23) - 1;
  return x >= lo && x <= hi && y >= lo && y <= hi && z >= lo && z <= hi;
}

}  // namespace cvx
