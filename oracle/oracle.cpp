// oracle.cpp — plain, slow, obviously-correct CPU oracle of the coVoxSLAM submap build path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this library.  The product path (paper_2410_21149_b200/) never
// links, imports or calls it, and shares no code, header, table or constant generator with it.
//
// Single-threaded, fp64, std::map / std::unordered_map based.  Every function cites the passage it
// follows: P:Lnn = /root/reference/PAPER.md line nn, S:Lnn = SPEC.md line nn, and O1..O13 / Q1..Q24
// are the readings written down in SURVEY.md §8c and DESIGN.md ("Readings of the paper").
// Built with -O2 -ffp-contract=off so every fp64 expression is evaluated exactly as written (no FMA).
//
// Pins (tests/test_oracle_*.py): closed-form voxel counts, S:L263/S:L265 examples, a Python
// dense-sampling brute force of the traversal, the S:L272-274 sdf/weight example, the analytic
// parallel-ray plane TSDF, the hollow-sphere bound, same-frame-twice, permutation
// invariance, brute-force EDT and scipy.ndimage.distance_transform_edt for the ESDF, and the
// voxel-centre identity of the query.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <unordered_map>
#include <vector>

extern "C" {

typedef struct {
  double voxel_size;          // s (voxels in blocks of n^3, n = 8)
  double truncation;          // tau ("truncation distance behind the point")
  int32_t weighting;          // 0 constant, 1 inverse square (Q5)
  double weight_range_floor;  // r_floor for 1/max(L, r_floor)^2
  int32_t carve;              // 1: o -> p + tau*u, 0: band p +- tau*u (Q2)
  double site_threshold;      // tau_site (O10, Q14)
} orc_grid;

typedef struct {
  int32_t kind;               // 0 unorganised points, 1 pinhole depth image, 2 organised LiDAR
  int32_t width, height;
  float fx, fy, cx, cy;       // pinhole only (fp32, O2)
  float min_range, max_range; // inclusive range filter on L (Q10)
} orc_sensor;

typedef struct {
  int64_t rays_in, rays_used, skipped_invalid, skipped_range, skipped_domain, voxel_updates,
      new_blocks, total_blocks;
} orc_stats;

}  // extern "C"

namespace {

constexpr int kB = 8;                       // block side n (Q17)
constexpr int kBV = kB * kB * kB;           // voxels per block
constexpr int64_t kOne = int64_t(1) << 16;  // fixed point F = 16 (O3)

struct V3 { int64_t x, y, z; };

struct Key {
  int64_t x, y, z;
  bool operator<(const Key& o) const {
    if (x != o.x) return x < o.x;
    if (y != o.y) return y < o.y;
    return z < o.z;
  }
};

// floor division by 8 for block coordinates (floor semantics across zero)
inline int64_t fdiv8(int64_t v) { return (v >= 0) ? v / 8 : -((-v + 7) / 8); }
inline int64_t fmod8(int64_t v) { return v - 8 * fdiv8(v); }

// swd, sw: O8 TSDF sums; cw, cc: TSDF + Color sums (R13) sum(w) and sum(w c) over band updates
struct Block { double swd[kBV]; double sw[kBV]; double cw[kBV]; double cc[kBV][3]; };

struct Oracle {
  orc_grid g;
  double Tws[16];
  std::map<Key, Block*> blocks;  // O7: block set; O8: sums of w*d and w per voxel
  ~Oracle() { for (auto& kv : blocks) delete kv.second; }
};

// O1: T_SC = T_WS^-1 * T_WC, fp64, fixed summation order, no FMA.
void compose_sc(const double* Tws, const double* Twc, double R[3][3], double t[3]) {
  double Rws[3][3], tws[3], Rwc[3][3], twc[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) { Rws[i][j] = Tws[4 * i + j]; Rwc[i][j] = Twc[4 * i + j]; }
    tws[i] = Tws[4 * i + 3]; twc[i] = Twc[4 * i + 3];
  }
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j)
      R[i][j] = ((Rws[0][i] * Rwc[0][j] + Rws[1][i] * Rwc[1][j]) + Rws[2][i] * Rwc[2][j]);
    t[i] = ((Rws[0][i] * (twc[0] - tws[0]) + Rws[1][i] * (twc[1] - tws[1])) +
            Rws[2][i] * (twc[2] - tws[2]));
  }
}

// O3: fixed-point quantisation q(x) = floor((x / s) * 2^16); false if outside the key domain.
bool quantise(double x, double s, int64_t* q) {
  double a = (x / s) * 65536.0;
  if (!(std::fabs(a) < 549755813888.0)) return false;  // |voxel| < 2^23  <=>  |a| < 2^39
  *q = (int64_t)std::floor(a);
  return true;
}

inline int64_t vox(int64_t q) { return q >> 16; }  // arithmetic shift == floor (O3)

// O4 ("voxels intersected by a ray"): 6-connected Amanatides-Woo walk in
// exact integer arithmetic from voxel(A) to voxel(B); ties between axes go to x < y < z.
void traverse(const int64_t A[3], const int64_t B[3], std::vector<V3>& out) {
  int64_t v[3], D[3], k[3], r[3], st[3];
  for (int i = 0; i < 3; ++i) {
    v[i] = vox(A[i]);
    int64_t vb = vox(B[i]);
    D[i] = B[i] - A[i];
    k[i] = vb > v[i] ? vb - v[i] : v[i] - vb;
    if (D[i] > 0) { st[i] = 1; r[i] = ((v[i] + 1) << 16) - A[i]; }
    else { st[i] = -1; r[i] = A[i] - (v[i] << 16); }
  }
  out.push_back({v[0], v[1], v[2]});
  while (k[0] + k[1] + k[2] > 0) {
    int best = -1;
    for (int i = 0; i < 3; ++i) {
      if (k[i] == 0) continue;
      if (best < 0) { best = i; continue; }
      // axis i crosses strictly earlier: r_i/|D_i| < r_best/|D_best|
      int64_t ai = D[i] < 0 ? -D[i] : D[i], ab = D[best] < 0 ? -D[best] : D[best];
      if (r[i] * ab < r[best] * ai) best = i;
    }
    v[best] += st[best];
    r[best] += kOne;
    k[best] -= 1;
    out.push_back({v[0], v[1], v[2]});
  }
}

struct Ray {
  double p[3], o[3], u[3], L, w;
  int64_t A[3], B[3];
};

// O2-O3, O6: one measured point -> ray in the submap frame.  Returns 0 ok, 1 invalid, 2 range, 3 domain.
int make_ray(const orc_grid& g, const orc_sensor& sm, const double R[3][3], const double t[3],
             const float pc[3], Ray* ray) {
  double pcd[3] = {pc[0], pc[1], pc[2]};
  for (int i = 0; i < 3; ++i) if (!std::isfinite(pcd[i])) return 1;
  for (int i = 0; i < 3; ++i) {
    ray->o[i] = t[i];
    ray->p[i] = ((R[i][0] * pcd[0] + R[i][1] * pcd[1]) + R[i][2] * pcd[2]) + t[i];
  }
  double d[3] = {ray->p[0] - ray->o[0], ray->p[1] - ray->o[1], ray->p[2] - ray->o[2]};
  double L = std::sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
  if (!(L >= (double)sm.min_range && L <= (double)sm.max_range) || !(L > 0.0)) return 2;  // Q10
  ray->L = L;
  double tau = g.truncation, s = g.voxel_size;
  double e[3], a[3];
  for (int i = 0; i < 3; ++i) {
    ray->u[i] = d[i] / L;
    double ext = (tau * d[i]) / L;
    e[i] = ray->p[i] + ext;                                   // tau behind the point
    a[i] = g.carve ? ray->o[i] : ray->p[i] - ext;             // carve from the optical centre (Q2)
  }
  for (int i = 0; i < 3; ++i) {
    if (!quantise(a[i], s, &ray->A[i]) || !quantise(e[i], s, &ray->B[i])) return 3;
    int64_t span = vox(ray->B[i]) - vox(ray->A[i]);
    if (span >= 32768 || span <= -32768) return 3;
  }
  if (g.weighting == 0) ray->w = 1.0;                         // O6 constant
  else { double r = std::max(L, g.weight_range_floor); ray->w = 1.0 / (r * r); }  // O6 1/r^2
  return 0;
}

}  // namespace

extern "C" {

void* orc_new(const orc_grid* g, const double* T_world_submap) {
  Oracle* o = new Oracle();
  o->g = *g;
  std::memcpy(o->Tws, T_world_submap, sizeof(o->Tws));
  return o;
}

void orc_free(void* h) { delete static_cast<Oracle*>(h); }

// Voxel list of one ray (test hook for the O3-O4 pins).  o, p: submap-frame fp64 points.
// Returns the number of voxels (written up to cap), or -1 if the ray is outside the domain.
int64_t orc_ray_voxels(const double* o, const double* p, double voxel_size, double truncation,
                       int32_t carve, int32_t* out_xyz, int64_t cap) {
  // build the ray directly in fp64 (no fp32 point rounding)
  Ray ray;
  double d[3];
  for (int i = 0; i < 3; ++i) { ray.o[i] = o[i]; ray.p[i] = p[i]; d[i] = p[i] - o[i]; }
  double L = std::sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
  if (!(L > 0)) return -1;
  double e[3], a[3];
  for (int i = 0; i < 3; ++i) {
    double ext = (truncation * d[i]) / L;
    e[i] = p[i] + ext;
    a[i] = carve ? o[i] : p[i] - ext;
    if (!quantise(a[i], voxel_size, &ray.A[i]) || !quantise(e[i], voxel_size, &ray.B[i])) return -1;
    int64_t span = vox(ray.B[i]) - vox(ray.A[i]);
    if (span >= 32768 || span <= -32768) return -1;
  }
  std::vector<V3> vs;
  traverse(ray.A, ray.B, vs);
  for (int64_t i = 0; i < (int64_t)vs.size() && i < cap; ++i) {
    out_xyz[3 * i] = (int32_t)vs[i].x; out_xyz[3 * i + 1] = (int32_t)vs[i].y; out_xyz[3 * i + 2] = (int32_t)vs[i].z;
  }
  return (int64_t)vs.size();
}

// integrate one frame: every used ray updates every traversed voxel with
// (w*d, w), d = clamp((p - c_v).u, -tau, tau) (O5, Q4); fusion = plain sums (O8: no weight cap, so
// D = sum(w d)/sum(w) equals the sequential fold of S:L281 in real arithmetic).
// TSDF + Color ("TSDF + Color"; R13): with rgb (uint8 [n][3]) every update
// whose unclamped sdf lies inside the truncation band, |sdf| < tau, also adds w and w * (r, g, b) to the
// voxel's colour sums; colour = sum(w c) / sum(w).
static int32_t integrate_frame(void* h, const float* data, const uint8_t* rgb, int64_t n,
                               const double* T_world_sensor, const orc_sensor* sm, orc_stats* st) {
  Oracle* O = static_cast<Oracle*>(h);
  const orc_grid& g = O->g;
  double R[3][3], t[3];
  compose_sc(O->Tws, T_world_sensor, R, t);
  orc_stats s = {};
  s.rays_in = n;
  size_t before = O->blocks.size();
  std::vector<V3> vs;
  const double sv = g.voxel_size, tau = g.truncation;
  for (int64_t i = 0; i < n; ++i) {
    float pc[3];
    if (sm->kind == 1) {  // O2: pinhole depth -> point, fp32 exactly as written, integer (u, v) (Q24)
      float z = data[i];
      if (!(z > 0.0f) || !std::isfinite(z)) { s.skipped_invalid++; continue; }
      float u = (float)(i % sm->width), v = (float)(i / sm->width);
      pc[0] = (z * (u - sm->cx)) / sm->fx;
      pc[1] = (z * (v - sm->cy)) / sm->fy;
      pc[2] = z;
    } else {
      pc[0] = data[3 * i]; pc[1] = data[3 * i + 1]; pc[2] = data[3 * i + 2];
    }
    Ray ray;
    int rc = make_ray(g, *sm, R, t, pc, &ray);
    if (rc == 1) { s.skipped_invalid++; continue; }
    if (rc == 2) { s.skipped_range++; continue; }
    if (rc == 3) { s.skipped_domain++; continue; }
    s.rays_used++;
    vs.clear();
    traverse(ray.A, ray.B, vs);
    for (const V3& v : vs) {
      // O5: c_v = (v + 1/2) s ; sdf = (p - c_v) . u, clamped before fusion (Q3, Q4)
      double c[3] = {((double)v.x + 0.5) * sv, ((double)v.y + 0.5) * sv, ((double)v.z + 0.5) * sv};
      double sdf = ((ray.p[0] - c[0]) * ray.u[0] + (ray.p[1] - c[1]) * ray.u[1]) + (ray.p[2] - c[2]) * ray.u[2];
      double d = std::min(std::max(sdf, -tau), tau);
      Key k = {fdiv8(v.x), fdiv8(v.y), fdiv8(v.z)};
      auto it = O->blocks.find(k);
      Block* b;
      if (it == O->blocks.end()) {  // O7: allocate every block containing a traversed voxel
        b = new Block();
        std::memset(b, 0, sizeof(Block));
        O->blocks.emplace(k, b);
      } else {
        b = it->second;
      }
      int local = (int)(fmod8(v.x) + 8 * fmod8(v.y) + 64 * fmod8(v.z));  // O9
      b->swd[local] += ray.w * d;
      b->sw[local] += ray.w;
      if (rgb && std::fabs(sdf) < tau) {
        b->cw[local] += ray.w;
        for (int c3 = 0; c3 < 3; ++c3) b->cc[local][c3] += ray.w * (double)rgb[3 * i + c3];
      }
      s.voxel_updates++;
    }
  }
  s.new_blocks = (int64_t)(O->blocks.size() - before);
  s.total_blocks = (int64_t)O->blocks.size();
  if (st) *st = s;
  return 0;
}

int32_t orc_integrate(void* h, const float* data, int64_t n, const double* T_world_sensor,
                      const orc_sensor* sm, orc_stats* st) {
  return integrate_frame(h, data, nullptr, n, T_world_sensor, sm, st);
}

int32_t orc_integrate_color(void* h, const float* data, const uint8_t* rgb, int64_t n, const double* T_world_sensor,
                            const orc_sensor* sm, orc_stats* st) {
  return integrate_frame(h, data, rgb, n, T_world_sensor, sm, st);
}

// Colour export in the order of orc_export: rgb = sum(w c) / sum(w) (0 where no band update), cw = sum(w).
void orc_export_color(void* h, double* rgb, double* cw) {
  Oracle* O = static_cast<Oracle*>(h);
  int64_t i = 0;
  for (auto& kv : O->blocks) {
    for (int l = 0; l < kBV; ++l) {
      double w = kv.second->cw[l];
      cw[i * kBV + l] = w;
      for (int c3 = 0; c3 < 3; ++c3) rgb[(i * kBV + l) * 3 + c3] = w > 0 ? kv.second->cc[l][c3] / w : 0.0;
    }
    ++i;
  }
}

// Projection-mapping integrator (R14) — the KinectFusion / nvBlox scheme the
// paper contrasts with raycasting ("projects voxels in the visual field of view into the
// depth image and computes their distance from the difference between the voxel centre and the depth
// value in the image", "associating it with the nearest pixel").  Pinhole depth frames only.
// Per frame, in this order:
//   1. ALLOCATE exactly as orc_integrate (every block holding a voxel traversed by a used ray, O2-O7),
//      with no TSDF update from the rays;
//   2. every voxel v of every block of the submap: c = (v + 1/2) s, x = R_SC^T (c - t_SC) (camera frame);
//      z = x_2 > 0; nearest pixel (px, py) = (floor(u + 1/2), floor(w + 1/2)) with
//      u = (fx x_0)(1/z) + cx, w = (fy x_1)(1/z) + cy (pixel centres at integers, Q24) inside the image;
//      the pixel's depth m valid (> 0, finite) and its O2 point's length L inside [r_min, r_max] (Q10);
//      sdf = m - z (projective distance along the optical axis); skipped if sdf < -tau (occluded) and,
//      in band mode (carve = 0), if sdf > tau; d = min(sdf, tau); w = O6 with the pixel's L;
//      swd += w d, sw += w.
// Step 2 for one voxel v (integer voxel coordinates): adds its projective update, if any, to (swd, sw).
static bool project_voxel(const orc_grid& g, const float* depth, const orc_sensor* sm, const double R[3][3],
                          const double t[3], const int64_t v[3], double* swd, double* sw) {
  const double sv = g.voxel_size, tau = g.truncation;
  double e[3], x[3];
  for (int k = 0; k < 3; ++k) e[k] = ((double)v[k] + 0.5) * sv - t[k];
  for (int i = 0; i < 3; ++i) x[i] = (R[0][i] * e[0] + R[1][i] * e[1]) + R[2][i] * e[2];
  const double z = x[2];
  if (!(z > 0.0)) return false;
  const double inv = 1.0 / z;
  const double uh = ((double)sm->fx * x[0]) * inv + (double)sm->cx + 0.5;
  const double wh = ((double)sm->fy * x[1]) * inv + (double)sm->cy + 0.5;
  if (!(uh >= 0.0 && uh < (double)sm->width && wh >= 0.0 && wh < (double)sm->height)) return false;
  const int64_t px = (int64_t)std::floor(uh), py = (int64_t)std::floor(wh);
  const float m = depth[py * sm->width + px];
  if (!(m > 0.0f) || !std::isfinite(m)) return false;
  const float pu = (float)px, pv = (float)py;   // O2 point of that pixel, fp32 as written
  const double pc[3] = {(double)((m * (pu - sm->cx)) / sm->fx), (double)((m * (pv - sm->cy)) / sm->fy), (double)m};
  const double L = std::sqrt((pc[0] * pc[0] + pc[1] * pc[1]) + pc[2] * pc[2]);
  if (!(L >= (double)sm->min_range && L <= (double)sm->max_range)) return false;
  const double sdf = (double)m - z;
  if (sdf < -tau) return false;
  if (!g.carve && sdf > tau) return false;
  const double d = std::min(sdf, tau);
  double w = 1.0;
  if (g.weighting != 0) { const double r = std::max(L, g.weight_range_floor); w = 1.0 / (r * r); }
  *swd += w * d;
  *sw += w;
  return true;
}

static void project_frame(Oracle* O, const float* depth, const orc_sensor* sm, const double R[3][3],
                          const double t[3], int64_t* n_updates) {
  for (auto& kv : O->blocks) {
    Block* b = kv.second;
    for (int l = 0; l < kBV; ++l) {
      const int64_t v[3] = {kv.first.x * kB + l % 8, kv.first.y * kB + (l / 8) % 8, kv.first.z * kB + l / 64};
      if (project_voxel(O->g, depth, sm, R, t, v, &b->swd[l], &b->sw[l])) ++*n_updates;
    }
  }
}

// Sampled check hook: the projective sums of m listed voxels (int32 [m][3]) over n_frames depth frames
// ([n_frames][h][w], poses [n_frames][16]) of a submap with pose T_world_submap, every voxel taking every
// frame (valid for voxels whose block exists from the first frame on).  swd, sw: fp64 [m].
void orc_project_voxels(const orc_grid* g, const double* T_world_submap, const float* depth, int32_t n_frames,
                        const double* T_world_sensor, const orc_sensor* sm, const int32_t* vox, int64_t m,
                        double* swd, double* sw) {
  for (int64_t i = 0; i < m; ++i) swd[i] = sw[i] = 0.0;
  const int64_t npix = (int64_t)sm->width * sm->height;
  for (int32_t f = 0; f < n_frames; ++f) {
    double R[3][3], t[3];
    compose_sc(T_world_submap, T_world_sensor + 16 * f, R, t);
    for (int64_t i = 0; i < m; ++i) {
      const int64_t v[3] = {vox[3 * i], vox[3 * i + 1], vox[3 * i + 2]};
      project_voxel(*g, depth + f * npix, sm, R, t, v, &swd[i], &sw[i]);
    }
  }
}

int32_t orc_integrate_projective(void* h, const float* depth, int64_t n, const double* T_world_sensor,
                                 const orc_sensor* sm, orc_stats* st) {
  Oracle* O = static_cast<Oracle*>(h);
  if (sm->kind != 1 || n != (int64_t)sm->width * sm->height) return -1;
  const orc_grid& g = O->g;
  double R[3][3], t[3];
  compose_sc(O->Tws, T_world_sensor, R, t);
  orc_stats s = {};
  s.rays_in = n;
  const size_t before = O->blocks.size();
  std::vector<V3> vs;
  for (int64_t i = 0; i < n; ++i) {   // 1. ALLOCATE (O2-O7), no update
    const float z = depth[i];
    if (!(z > 0.0f) || !std::isfinite(z)) { s.skipped_invalid++; continue; }
    const float u = (float)(i % sm->width), v = (float)(i / sm->width);
    const float pc[3] = {(z * (u - sm->cx)) / sm->fx, (z * (v - sm->cy)) / sm->fy, z};
    Ray ray;
    const int rc = make_ray(g, *sm, R, t, pc, &ray);
    if (rc == 1) { s.skipped_invalid++; continue; }
    if (rc == 2) { s.skipped_range++; continue; }
    if (rc == 3) { s.skipped_domain++; continue; }
    s.rays_used++;
    vs.clear();
    traverse(ray.A, ray.B, vs);
    for (const V3& vv : vs) {
      const Key k = {fdiv8(vv.x), fdiv8(vv.y), fdiv8(vv.z)};
      if (O->blocks.find(k) == O->blocks.end()) {
        Block* b = new Block();
        std::memset(b, 0, sizeof(Block));
        O->blocks.emplace(k, b);
      }
    }
  }
  project_frame(O, depth, sm, R, t, &s.voxel_updates);   // 2. projective update of every voxel
  s.new_blocks = (int64_t)(O->blocks.size() - before);
  s.total_blocks = (int64_t)O->blocks.size();
  if (st) *st = s;
  return 0;
}

int64_t orc_num_blocks(void* h) { return (int64_t)static_cast<Oracle*>(h)->blocks.size(); }

// Export in (bx, by, bz) lexicographic order: D = sum(w d)/sum(w) (O8), W = sum(w); D = W = 0 where
// unobserved.
void orc_export(void* h, int32_t* bxyz, double* D, double* W) {
  Oracle* O = static_cast<Oracle*>(h);
  int64_t i = 0;
  for (auto& kv : O->blocks) {
    bxyz[3 * i] = (int32_t)kv.first.x; bxyz[3 * i + 1] = (int32_t)kv.first.y; bxyz[3 * i + 2] = (int32_t)kv.first.z;
    for (int l = 0; l < kBV; ++l) {
      double w = kv.second->sw[l];
      W[i * kBV + l] = w;
      D[i * kBV + l] = w > 0 ? kv.second->swd[l] / w : 0.0;
    }
    ++i;
  }
}

// ---------------------------------------------------------------------------------------- ESDF
// O10-O12 ("distance to the nearest obstacle"; P:L139 PBA = exact EDT; BJ "exact"):
//   sites S = { v observed : |D(v)| <= tau_site };  d2(v) = min_{u in S} |v - u|^2 (voxel units);
//   E(v) = sign(D(v)) * s * sqrt(d2(v)); NaN if v unobserved; +inf if S is empty.
// `brute` = 1 evaluates the minimum literally over all sites; 0 uses the separable exact EDT
// (Felzenszwalb-Huttenlocher lower envelope of parabolas, one axis at a time) over the dense
// AABB of the allocated blocks.  Both give the same integers; the tests pin that.
namespace {

const int64_t kInf = int64_t(1) << 60;

// 1-D squared-distance transform of sampled function f (Felzenszwalb & Huttenlocher 2012):
// d(q) = min_p (q - p)^2 + f(p), entries with f = kInf are absent.
void dt1d(const std::vector<int64_t>& f, std::vector<int64_t>& d) {
  const int64_t n = (int64_t)f.size();
  std::vector<int64_t> v(n);
  std::vector<double> z(n + 1);
  int64_t k = -1;
  auto sep = [&](int64_t p, int64_t q) {  // abscissa where the parabolas rooted at p < q intersect
    return (double)((f[q] + q * q) - (f[p] + p * p)) / (double)(2 * q - 2 * p);
  };
  for (int64_t q = 0; q < n; ++q) {
    if (f[q] >= kInf) continue;
    if (k < 0) { k = 0; v[0] = q; z[0] = -HUGE_VAL; z[1] = HUGE_VAL; continue; }
    double s = sep(v[k], q);
    while (s <= z[k]) { --k; s = sep(v[k], q); }  // terminates: z[0] = -inf
    ++k; v[k] = q; z[k] = s; z[k + 1] = HUGE_VAL;
  }
  if (k < 0) { for (int64_t q = 0; q < n; ++q) d[q] = kInf; return; }
  int64_t j = 0;
  for (int64_t q = 0; q < n; ++q) {
    while (z[j + 1] < (double)q) ++j;
    int64_t p = v[j];
    d[q] = (q - p) * (q - p) + f[p];
  }
}

}  // namespace

// bxyz [nb][3], D/W [nb][512] (local = lx + 8 ly + 64 lz); E_out [nb][512]; d2_out (nullable) [nb][512].
int32_t orc_esdf(const int32_t* bxyz, const double* D, const double* W, int64_t nb, double voxel_size,
                 double site_threshold, int32_t brute, double* E_out, int64_t* d2_out) {
  if (nb <= 0) return 0;
  std::vector<V3> sites;
  int64_t lo[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, hi[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
  for (int64_t b = 0; b < nb; ++b) {
    for (int a = 0; a < 3; ++a) { lo[a] = std::min<int64_t>(lo[a], bxyz[3 * b + a]); hi[a] = std::max<int64_t>(hi[a], bxyz[3 * b + a]); }
    for (int l = 0; l < kBV; ++l) {
      double w = W[b * kBV + l], d = D[b * kBV + l];
      if (w > 0 && std::fabs(d) <= site_threshold)
        sites.push_back({8 * (int64_t)bxyz[3 * b] + l % 8, 8 * (int64_t)bxyz[3 * b + 1] + (l / 8) % 8,
                         8 * (int64_t)bxyz[3 * b + 2] + l / 64});
    }
  }
  std::vector<int64_t> d2(nb * kBV, kInf);
  if (brute) {
    for (int64_t b = 0; b < nb; ++b)
      for (int l = 0; l < kBV; ++l) {
        int64_t x = 8 * (int64_t)bxyz[3 * b] + l % 8, y = 8 * (int64_t)bxyz[3 * b + 1] + (l / 8) % 8,
                z = 8 * (int64_t)bxyz[3 * b + 2] + l / 64;
        int64_t best = kInf;
        for (const V3& s : sites) {
          int64_t dd = (x - s.x) * (x - s.x) + (y - s.y) * (y - s.y) + (z - s.z) * (z - s.z);
          best = std::min(best, dd);
        }
        d2[b * kBV + l] = best;
      }
  } else if (!sites.empty()) {
    const int64_t nx = 8 * (hi[0] - lo[0] + 1), ny = 8 * (hi[1] - lo[1] + 1), nz = 8 * (hi[2] - lo[2] + 1);
    const int64_t ox = 8 * lo[0], oy = 8 * lo[1], oz = 8 * lo[2];
    std::vector<int64_t> G((size_t)(nx * ny * nz), kInf);
    auto at = [&](int64_t x, int64_t y, int64_t z) -> int64_t& { return G[(size_t)((z * ny + y) * nx + x)]; };
    for (const V3& s : sites) at(s.x - ox, s.y - oy, s.z - oz) = 0;
    std::vector<int64_t> f, d;
    f.resize(nx); d.resize(nx);
    for (int64_t z = 0; z < nz; ++z) for (int64_t y = 0; y < ny; ++y) {
      for (int64_t x = 0; x < nx; ++x) f[x] = at(x, y, z);
      dt1d(f, d);
      for (int64_t x = 0; x < nx; ++x) at(x, y, z) = d[x];
    }
    f.resize(ny); d.resize(ny);
    for (int64_t z = 0; z < nz; ++z) for (int64_t x = 0; x < nx; ++x) {
      for (int64_t y = 0; y < ny; ++y) f[y] = at(x, y, z);
      dt1d(f, d);
      for (int64_t y = 0; y < ny; ++y) at(x, y, z) = d[y];
    }
    f.resize(nz); d.resize(nz);
    for (int64_t y = 0; y < ny; ++y) for (int64_t x = 0; x < nx; ++x) {
      for (int64_t z = 0; z < nz; ++z) f[z] = at(x, y, z);
      dt1d(f, d);
      for (int64_t z = 0; z < nz; ++z) at(x, y, z) = d[z];
    }
    for (int64_t b = 0; b < nb; ++b)
      for (int l = 0; l < kBV; ++l)
        d2[b * kBV + l] = at(8 * (int64_t)bxyz[3 * b] + l % 8 - ox, 8 * (int64_t)bxyz[3 * b + 1] + (l / 8) % 8 - oy,
                             8 * (int64_t)bxyz[3 * b + 2] + l / 64 - oz);
  }
  for (int64_t i = 0; i < nb * kBV; ++i) {
    if (d2_out) d2_out[i] = d2[i] >= kInf ? -1 : d2[i];
    if (!(W[i] > 0)) { E_out[i] = std::numeric_limits<double>::quiet_NaN(); continue; }  // unobserved
    if (d2[i] >= kInf) { E_out[i] = HUGE_VAL; continue; }                              // S empty
    double sg = D[i] < 0 ? -1.0 : 1.0;
    E_out[i] = sg * voxel_size * std::sqrt((double)d2[i]);
  }
  return 0;
}

// f1 incremental ESDF (R11): the value the incremental update keeps
// is the exact EDT of O11 clamped at max_distance d_max ("max_esdf_distance default 2.0 m";
// the paper gives no cap, and without one a single site change can move distances anywhere):
//   E(v) = NaN if v unobserved; sign(D(v)) * min(s * sqrt(d2(v)), d_max) otherwise (d_max when S is empty).
// Written out on top of orc_esdf's d2 (same sites, same integers).
int32_t orc_esdf_capped(const int32_t* bxyz, const double* D, const double* W, int64_t nb, double voxel_size,
                        double site_threshold, double max_distance, int32_t brute, double* E_out) {
  if (nb <= 0) return 0;
  std::vector<double> E(nb * kBV);
  std::vector<int64_t> d2(nb * kBV);
  int32_t rc = orc_esdf(bxyz, D, W, nb, voxel_size, site_threshold, brute, E.data(), d2.data());
  if (rc != 0) return rc;
  for (int64_t i = 0; i < nb * kBV; ++i) {
    if (!(W[i] > 0)) { E_out[i] = std::numeric_limits<double>::quiet_NaN(); continue; }
    const double sg = D[i] < 0 ? -1.0 : 1.0;
    const double m = d2[i] < 0 ? HUGE_VAL : voxel_size * std::sqrt((double)d2[i]);
    E_out[i] = sg * std::min(m, max_distance);
  }
  return 0;
}

// Brute force O11 at sample voxels (full-size parity): d2 of each sample voxel (int64 [m][3] voxel
// coordinates) to the nearest site of the given TSDF, literally min over all sites; -1 if no site.
int32_t orc_esdf_sample(const int32_t* bxyz, const double* D, const double* W, int64_t nb, double site_threshold,
                        const int64_t* vox, int64_t m, int64_t* d2_out) {
  std::vector<V3> sites;
  for (int64_t b = 0; b < nb; ++b)
    for (int l = 0; l < kBV; ++l) {
      double w = W[b * kBV + l], d = D[b * kBV + l];
      if (w > 0 && std::fabs(d) <= site_threshold)
        sites.push_back({8 * (int64_t)bxyz[3 * b] + l % 8, 8 * (int64_t)bxyz[3 * b + 1] + (l / 8) % 8,
                         8 * (int64_t)bxyz[3 * b + 2] + l / 64});
    }
  for (int64_t i = 0; i < m; ++i) {
    int64_t best = -1;
    for (const V3& s : sites) {
      int64_t dx = vox[3 * i] - s.x, dy = vox[3 * i + 1] - s.y, dz = vox[3 * i + 2] - s.z;
      int64_t dd = dx * dx + dy * dy + dz * dz;
      if (best < 0 || dd < best) best = dd;
    }
    d2_out[i] = best;
  }
  return 0;
}

// ---------------------------------------------------------------------------------------- query
// O13 (S:L486 trilinear over 8 ESDF voxels; S:L491 identity at a voxel centre):
//   x_s = T_WS^-1 x ; g = x_s/s - 1/2 ; i0 = floor(g) ; f = g - i0.
//   all 8 corners observed -> sum over corners with non-zero weight of weight*E (status 0 OK);
//   else voxel floor(x_s/s) observed -> its E (status 1 NEAREST); else NaN (status 2 UNKNOWN).
// grad (nullable) [m][3]: world-frame gradient of the trilinear interpolant for status OK (f4),
// NaN otherwise: dE/dx_world = R_WS (dE/df) / s with dE/df_x = sum_c (dx ? 1 : -1) w_y w_z E_c (all 8 corners).
int32_t orc_query(const int32_t* bxyz, const double* E, int64_t nb, double voxel_size,
                  const double* T_world_submap, const float* pts, int64_t m, double* out, uint8_t* status,
                  double* grad) {
  std::unordered_map<int64_t, int64_t> idx;
  auto pack = [](int64_t x, int64_t y, int64_t z) {
    return ((x + (1 << 20)) << 42) | ((y + (1 << 20)) << 21) | (z + (1 << 20));
  };
  for (int64_t b = 0; b < nb; ++b) idx[pack(bxyz[3 * b], bxyz[3 * b + 1], bxyz[3 * b + 2])] = b;
  auto lookup = [&](int64_t x, int64_t y, int64_t z, double* e) -> bool {
    auto it = idx.find(pack(fdiv8(x), fdiv8(y), fdiv8(z)));
    if (it == idx.end()) return false;
    double v = E[it->second * kBV + fmod8(x) + 8 * fmod8(y) + 64 * fmod8(z)];
    if (std::isnan(v)) return false;
    *e = v;
    return true;
  };
  const double* T = T_world_submap;
  for (int64_t i = 0; i < m; ++i) {
    double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]}, xs[3];
    for (int a = 0; a < 3; ++a)
      xs[a] = ((T[0 * 4 + a] * (x[0] - T[3]) + T[1 * 4 + a] * (x[1] - T[7])) + T[2 * 4 + a] * (x[2] - T[11]));
    double gg[3], f[3];
    int64_t i0[3];
    for (int a = 0; a < 3; ++a) {
      gg[a] = xs[a] / voxel_size - 0.5;
      double fl = std::floor(gg[a]);
      i0[a] = (int64_t)fl;
      f[a] = gg[a] - fl;
    }
    double acc = 0.0, gs[3] = {0.0, 0.0, 0.0};
    bool all = true;
    for (int c = 0; c < 8 && all; ++c) {
      int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
      double e;
      if (!lookup(i0[0] + dx, i0[1] + dy, i0[2] + dz, &e)) { all = false; break; }
      double wx = dx ? f[0] : 1.0 - f[0], wy = dy ? f[1] : 1.0 - f[1], wz = dz ? f[2] : 1.0 - f[2];
      double wgt = (wx * wy) * wz;
      if (wgt > 0) acc += wgt * e;
      gs[0] += (dx ? 1.0 : -1.0) * wy * wz * e;
      gs[1] += (dy ? 1.0 : -1.0) * wx * wz * e;
      gs[2] += (dz ? 1.0 : -1.0) * wx * wy * e;
    }
    if (grad)
      for (int a = 0; a < 3; ++a)
        grad[3 * i + a] = all ? (T[4 * a] * gs[0] + T[4 * a + 1] * gs[1] + T[4 * a + 2] * gs[2]) / voxel_size
                              : std::numeric_limits<double>::quiet_NaN();
    if (all) { out[i] = acc; status[i] = 0; continue; }
    double e;
    int64_t v[3] = {(int64_t)std::floor(xs[0] / voxel_size), (int64_t)std::floor(xs[1] / voxel_size),
                    (int64_t)std::floor(xs[2] / voxel_size)};
    if (grad) for (int a = 0; a < 3; ++a) grad[3 * i + a] = std::numeric_limits<double>::quiet_NaN();
    if (lookup(v[0], v[1], v[2], &e)) { out[i] = e; status[i] = 1; continue; }
    out[i] = std::numeric_limits<double>::quiet_NaN();
    status[i] = 2;
  }
  return 0;
}

// Weight-proportional surface sampling (f4; R12), written out: sites in
// lexicographic block order then local order, integer weights floor(round(W 2^30) / 2^10), prefix sums,
// target = floor(T u / 2^32), first candidate with prefix sum > target, world voxel centre.
int32_t orc_sample_surface(const int32_t* bxyz, const double* D, const double* W, int64_t nb, double site_threshold,
                           double voxel_size, const double* T, const uint32_t* u, int64_t m, float* xyz, double* wout,
                           uint64_t* total) {
  std::vector<int64_t> order(nb);
  for (int64_t b = 0; b < nb; ++b) order[b] = b;
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    Key ka = {bxyz[3 * a], bxyz[3 * a + 1], bxyz[3 * a + 2]}, kb = {bxyz[3 * b], bxyz[3 * b + 1], bxyz[3 * b + 2]};
    return ka < kb;
  });
  std::vector<uint64_t> cum;
  std::vector<int64_t> idx;   // flat voxel index b * 512 + l of each candidate
  uint64_t acc = 0;
  for (int64_t ob : order)
    for (int l = 0; l < kBV; ++l) {
      const double w = W[ob * kBV + l], d = D[ob * kBV + l];
      if (!(w > 0 && std::fabs(d) <= site_threshold)) continue;
      const uint64_t wi = (uint64_t)std::llround(w * 1073741824.0) >> 10;
      acc += wi;
      cum.push_back(acc);
      idx.push_back(ob * kBV + l);
    }
  if (total) *total = acc;
  for (int64_t i = 0; i < m; ++i) {
    if (acc == 0) {
      for (int a = 0; a < 3; ++a) xyz[3 * i + a] = std::numeric_limits<float>::quiet_NaN();
      if (wout) wout[i] = 0.0;
      continue;
    }
    const uint64_t target = (uint64_t)(((unsigned __int128)acc * u[i]) >> 32);
    const int64_t k = std::upper_bound(cum.begin(), cum.end(), target) - cum.begin();
    const int64_t b = idx[k] / kBV;
    const int l = (int)(idx[k] % kBV);
    const double v[3] = {(double)(8 * (int64_t)bxyz[3 * b] + l % 8), (double)(8 * (int64_t)bxyz[3 * b + 1] + (l / 8) % 8),
                         (double)(8 * (int64_t)bxyz[3 * b + 2] + l / 64)};
    double c[3];
    for (int a = 0; a < 3; ++a) c[a] = (v[a] + 0.5) * voxel_size;
    for (int a = 0; a < 3; ++a)
      xyz[3 * i + a] = (float)(((T[4 * a] * c[0] + T[4 * a + 1] * c[1]) + T[4 * a + 2] * c[2]) + T[4 * a + 3]);
    if (wout) wout[i] = W[idx[k]];
  }
  return 0;
}

}  // extern "C"
