// Pocket-side kernels: exact voxel candidate-list build, overlap_score of
// arbitrary poses (drop-in API), and the fp64 pipe probe used as the
// roofline denominator.
#include "device_common.cuh"

namespace gdb200 {
namespace {

// --------------------------------------------------------------------------
// overlap_score for arbitrary poses: one thread per pose.
// --------------------------------------------------------------------------
template <bool CP>
__global__ void score_poses_kernel(PocketView pk, const double* xyz, int n_atoms, int n_poses,
                                   double* out) {
  stage_tab<CP>(pk);
  const int pose = blockIdx.x * blockDim.x + threadIdx.x;
  if (pose >= n_poses) return;
  const double* q = xyz + static_cast<size_t>(3) * n_atoms * pose;
  Work<false> wk;
  double sum = 0.0;
  for (int i = 0; i < n_atoms; ++i)
    sum = dadd(sum, fmax(kMinDistanceSq, min_dist_sq<false, CP>(pk, q[3 * i], q[3 * i + 1], q[3 * i + 2], wk)));
  out[pose] = __ddiv_rn(static_cast<double>(n_atoms), sum);
}

// --------------------------------------------------------------------------
// Voxel candidate lists.  For voxel box B (expanded by kVoxEps):
//   U    = min_j maxdist^2(B, P_j)          (an upper bound on the NN d^2)
//   C    = { j : mindist^2(B, P_j) <= U + margin }
//   keep = { a in C : no b in C with d^2(q,b) < d^2(q,a) - margin at all 8
//            corners q of B }  (d^2(q,b) - d^2(q,a) is affine in q, so the
//            corners bound it over B)
// margin (1e-9 A^2) is orders above fp64 rounding of d^2 (~1e-13), so no
// dropped point can attain the fp64 minimum anywhere in B.
// --------------------------------------------------------------------------
constexpr double kVoxEps = 1e-6;
constexpr double kVoxMargin = 1e-9;
constexpr int kVoxMaxCand = 1024;

// Does point b beat point a by more than the margin everywhere in box
// [bl, bh]?  d^2(q,b) - d^2(q,a) is affine in q, so the 8 corners decide.
__device__ bool dominates(const P3& b, const P3& a, const double* bl, const double* bh) {
  for (int corner = 0; corner < 8; ++corner) {
    const double qx = (corner & 1) ? bh[0] : bl[0];
    const double qy = (corner & 2) ? bh[1] : bl[1];
    const double qz = (corner & 4) ? bh[2] : bl[2];
    const double da = (qx - a.x) * (qx - a.x) + (qy - a.y) * (qy - a.y) + (qz - a.z) * (qz - a.z);
    const double db = (qx - b.x) * (qx - b.x) + (qy - b.y) * (qy - b.y) + (qz - b.z) * (qz - b.z);
    if (!(db < da - kVoxMargin)) return false;
  }
  return true;
}

// The two coarse passes (the upper bound U and the distance pre-filter)
// stream every pocket point, so they run over shared-memory tiles of fp32
// copies with margins far above fp32 rounding (coordinates < ~1e2 A, so
// |error of a d^2| < ~1e-2 A^2): the pre-filter can only admit more points,
// never drop one the exact rule keeps.  Every decision that shapes the list
// -- dominance by the centre-nearest point and the pairwise dominance pass
// -- stays exact fp64 on the exact coordinates.  (Any superset of the
// candidates that can attain the minimum gives the same, exact, query
// result; the margins only cost list length.)
constexpr int kBuildThreads = 128;
constexpr int kTile = 1024;
constexpr float kPassRel = 1e-4f;   // relative margin on U
constexpr float kPassAbs = 5e-2f;   // absolute margin, A^2

// Candidate list of voxel v; every thread of the CTA must call it (tiles),
// `active` false for threads past the grid.  Returns the count, or -1 when
// more than kVoxMaxCand points survive (the caller then keeps every point).
__device__ int voxel_list(const double* pts, int P, const VoxelGrid& g, int v, bool active,
                          int* cand, float4* tile) {
  const int iz = v % g.dim_z;
  const int iy = (v / g.dim_z) % g.dim_y;
  const int ix = v / (g.dim_z * g.dim_y);
  const double bl[3] = {g.lo_x + ix * g.h - kVoxEps, g.lo_y + iy * g.h - kVoxEps,
                        g.lo_z + iz * g.h - kVoxEps};
  const double bh[3] = {bl[0] + g.h + 2 * kVoxEps, bl[1] + g.h + 2 * kVoxEps,
                        bl[2] + g.h + 2 * kVoxEps};
  const float lx = static_cast<float>(bl[0]), ly = static_cast<float>(bl[1]),
              lz = static_cast<float>(bl[2]);
  const float hx = static_cast<float>(bh[0]), hy = static_cast<float>(bh[1]),
              hz = static_cast<float>(bh[2]);
  const float cx = 0.5f * (lx + hx), cy = 0.5f * (ly + hy), cz = 0.5f * (lz + hz);
  auto load_tile = [&](int t0, int cnt) {
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const double* q = pts + 4 * static_cast<size_t>(t0 + i);
      tile[i] = make_float4(static_cast<float>(q[0]), static_cast<float>(q[1]),
                            static_cast<float>(q[2]), 0.0f);
    }
    __syncthreads();
  };
  // Pass 1 (fp32): U = min_j maxdist^2(B, P_j), and the point nearest the
  // box centre (a strong dominator for pass 2; any choice is correct).
  float U = 3.0e38f, dc = 3.0e38f;
  int jc = 0;
  for (int t0 = 0; t0 < P; t0 += kTile) {
    const int cnt = min(kTile, P - t0);
    load_tile(t0, cnt);
    if (!active) continue;
    for (int i = 0; i < cnt; ++i) {
      const float4 q = tile[i];
      const float fx = fmaxf(fabsf(q.x - lx), fabsf(q.x - hx));
      const float fy = fmaxf(fabsf(q.y - ly), fabsf(q.y - hy));
      const float fz = fmaxf(fabsf(q.z - lz), fabsf(q.z - hz));
      U = fminf(U, fx * fx + fy * fy + fz * fz);
      const float d = (q.x - cx) * (q.x - cx) + (q.y - cy) * (q.y - cy) + (q.z - cz) * (q.z - cz);
      if (d < dc) {
        dc = d;
        jc = t0 + i;
      }
    }
  }
  const float lim = U * (1.0f + kPassRel) + kPassAbs;
  const P3 C = ldp(pts, active ? jc : 0);
  // Pass 2: points that may be nearest somewhere in B (fp32 with margins)
  // and that the centre-nearest point does not dominate (exact).
  int k = 0;
  bool over = false;
  for (int t0 = 0; t0 < P; t0 += kTile) {
    const int cnt = min(kTile, P - t0);
    load_tile(t0, cnt);
    if (!active || over) continue;
    for (int i = 0; i < cnt; ++i) {
      const float4 q = tile[i];
      const float nx = fmaxf(0.0f, fmaxf(lx - q.x, q.x - hx));
      const float ny = fmaxf(0.0f, fmaxf(ly - q.y, q.y - hy));
      const float nz = fmaxf(0.0f, fmaxf(lz - q.z, q.z - hz));
      if (nx * nx + ny * ny + nz * nz > lim) continue;
      const P3 Q = ldp(pts, t0 + i);
      if (dominates(C, Q, bl, bh)) continue;
      if (k >= min(g.overflow, kVoxMaxCand)) {
        over = true;
        break;
      }
      cand[k++] = t0 + i;
    }
  }
  if (!active) return 0;
  if (over) return -1;
  // Pass 3 (exact): full dominance pruning among the survivors.
  int kept = 0;
  for (int a = 0; a < k; ++a) {
    const P3 A = ldp(pts, cand[a]);
    bool dominated = false;
    for (int b = 0; b < k && !dominated; ++b)
      if (b != a) dominated = dominates(ldp(pts, cand[b]), A, bl, bh);
    if (!dominated) cand[kept++] = cand[a];
  }
  return kept;
}

// Culled build (pockets up to kMaxTiles x 32 points).  The host stores the
// points in Morton order, so 32-point tiles are spatially compact, with
// outward-rounded fp32 bounding boxes.  A CTA owns a 4 x 4 x 8 brick of
// voxels, ranks the tiles by their distance to the brick and walks them
// nearest first:
//   pass 1 stops once the next tile is farther than every voxel's current
//   U (no point beyond can lower a U: maxdist >= mindist; and any U is a
//   valid bound, so culling here can only lengthen lists);
//   pass 2 stops once the next tile is beyond every voxel's limit plus a
//   pad far above fp32 rounding, so no point the exact rule keeps is
//   skipped.
// Lists are the same as the full scan's up to the centre-nearest choice and
// an upper bound U that may only be larger, i.e. exact.
constexpr int kTilePts = 32;
constexpr int kMaxTiles = 512;
constexpr int kGroupTiles = 8;  // tiles staged per round (256 points)
constexpr int kBrickX = 4, kBrickY = 4, kBrickZ = 8;
static_assert(kBrickX * kBrickY * kBrickZ == kBuildThreads, "one voxel per thread");

struct BrickScratch {
  float dB[kMaxTiles];    // squared distance brick -> tile box (shrunk: a lower bound)
  short ord[kMaxTiles];   // tiles by ascending dB
  int bound;              // CTA max of a per-voxel bound (float bits, >= 0)
};

__device__ __forceinline__ float box_gap(float alo, float ahi, float blo, float bhi) {
  return fmaxf(0.0f, fmaxf(alo - bhi, blo - ahi));
}

// The voxel of this thread in brick `b` (x-major voxel numbering).
__device__ __forceinline__ bool brick_voxel(const VoxelGrid& g, int b, int& ix, int& iy, int& iz) {
  const int nby = (g.dim_y + kBrickY - 1) / kBrickY, nbz = (g.dim_z + kBrickZ - 1) / kBrickZ;
  const int bx = b / (nby * nbz), by = (b / nbz) % nby, bz = b % nbz;
  const int t = threadIdx.x;
  ix = bx * kBrickX + t / (kBrickY * kBrickZ);
  iy = by * kBrickY + (t / kBrickZ) % kBrickY;
  iz = bz * kBrickZ + t % kBrickZ;
  return ix < g.dim_x && iy < g.dim_y && iz < g.dim_z;
}

__device__ int voxel_list_culled(const double* pts, int P, const VoxelGrid& g, int b, int ix,
                                 int iy, int iz, bool active, int* cand, float4* tile,
                                 const float* tbox, int nt, BrickScratch& sc) {
  const double bl[3] = {g.lo_x + ix * g.h - kVoxEps, g.lo_y + iy * g.h - kVoxEps,
                        g.lo_z + iz * g.h - kVoxEps};
  const double bh[3] = {bl[0] + g.h + 2 * kVoxEps, bl[1] + g.h + 2 * kVoxEps,
                        bl[2] + g.h + 2 * kVoxEps};
  const float lx = static_cast<float>(bl[0]), ly = static_cast<float>(bl[1]),
              lz = static_cast<float>(bl[2]);
  const float hx = static_cast<float>(bh[0]), hy = static_cast<float>(bh[1]),
              hz = static_cast<float>(bh[2]);
  const float cx = 0.5f * (lx + hx), cy = 0.5f * (ly + hy), cz = 0.5f * (lz + hz);
  // The brick's box (all its voxel boxes, grid-clipped or not: a superset
  // only lowers dB), shrunk by a hair so dB stays a lower bound.
  const int nby = (g.dim_y + kBrickY - 1) / kBrickY, nbz = (g.dim_z + kBrickZ - 1) / kBrickZ;
  const int bx = b / (nby * nbz), by = (b / nbz) % nby, bz = b % nbz;
  const float pad = 1e-3f;
  const float Bl[3] = {static_cast<float>(g.lo_x + bx * kBrickX * g.h) - pad,
                       static_cast<float>(g.lo_y + by * kBrickY * g.h) - pad,
                       static_cast<float>(g.lo_z + bz * kBrickZ * g.h) - pad};
  const float Bh[3] = {static_cast<float>(g.lo_x + (bx + 1) * kBrickX * g.h) + pad,
                       static_cast<float>(g.lo_y + (by + 1) * kBrickY * g.h) + pad,
                       static_cast<float>(g.lo_z + (bz + 1) * kBrickZ * g.h) + pad};
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    const float* q = tbox + 6 * t;
    const float gx = box_gap(Bl[0], Bh[0], q[0], q[3]);
    const float gy = box_gap(Bl[1], Bh[1], q[1], q[4]);
    const float gz = box_gap(Bl[2], Bh[2], q[2], q[5]);
    sc.dB[t] = gx * gx + gy * gy + gz * gz;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {  // rank sort (distinct by index)
    const float d = sc.dB[t];
    int r = 0;
    for (int u = 0; u < nt; ++u) {
      const float e = sc.dB[u];
      r += (e < d) || (e == d && u < t);
    }
    sc.ord[r] = static_cast<short>(t);
  }
  __syncthreads();
  // Stages sorted tiles [k0, k0 + kGroupTiles) into `tile` (w = the point's
  // index bits); returns the number of points staged.
  // Staged tile g occupies tile[g * kTilePts, + size); the stage holds
  // min(kGroupTiles, nt - k0) tiles.
  auto stage = [&](int k0) {
    __syncthreads();
    for (int k = k0; k < min(nt, k0 + kGroupTiles); ++k) {
      const int t = sc.ord[k];
      const int cnt = min(kTilePts, P - t * kTilePts);
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const double* q = pts + 4 * static_cast<size_t>(t * kTilePts + i);
        tile[(k - k0) * kTilePts + i] =
            make_float4(static_cast<float>(q[0]), static_cast<float>(q[1]), static_cast<float>(q[2]),
                        __int_as_float(t * kTilePts + i));
      }
    }
    __syncthreads();
    return min(kGroupTiles, nt - k0);
  };
  // Squared gap between this voxel's box and a tile's box (a lower bound on
  // the squared distance from the voxel to any of the tile's points).
  auto vgap2 = [&](int t) {
    const float* q = tbox + 6 * t;
    const float gx = box_gap(lx, hx, q[0], q[3]);
    const float gy = box_gap(ly, hy, q[1], q[4]);
    const float gz = box_gap(lz, hz, q[2], q[5]);
    return gx * gx + gy * gy + gz * gz;
  };
  auto cta_max = [&](float x) {  // max over active threads (x >= 0)
    __syncthreads();
    if (threadIdx.x == 0) sc.bound = 0;
    __syncthreads();
    if (active) atomicMax(&sc.bound, __float_as_int(x));
    __syncthreads();
    return __int_as_float(sc.bound);
  };
  // Pass 1 (fp32): U and the point nearest the box centre, nearest tiles first.
  float U = 3.0e38f, dc = 3.0e38f;
  int jc = 0;
  float Umax = 3.0e38f;
  for (int k0 = 0; k0 < nt; k0 += kGroupTiles) {
    if (sc.dB[sc.ord[k0]] > Umax) break;  // uniform: every later tile is farther
    const int ng = stage(k0);
    for (int gt = 0; gt < ng && active; ++gt) {
      const int t = sc.ord[k0 + gt];
      if (vgap2(t) > U) continue;  // none of its points can lower this U
      const int cnt = min(kTilePts, P - t * kTilePts);
      for (int i = gt * kTilePts; i < gt * kTilePts + cnt; ++i) {
        const float4 q = tile[i];
        const float fx = fmaxf(fabsf(q.x - lx), fabsf(q.x - hx));
        const float fy = fmaxf(fabsf(q.y - ly), fabsf(q.y - hy));
        const float fz = fmaxf(fabsf(q.z - lz), fabsf(q.z - hz));
        U = fminf(U, fx * fx + fy * fy + fz * fz);
        const float d = (q.x - cx) * (q.x - cx) + (q.y - cy) * (q.y - cy) + (q.z - cz) * (q.z - cz);
        if (d < dc) {
          dc = d;
          jc = __float_as_int(q.w);
        }
      }
    }
    Umax = cta_max(U);
  }
  const float lim = U * (1.0f + kPassRel) + kPassAbs;
  const float cut = cta_max(lim) * (1.0f + kPassRel) + 1e-2f;
  const P3 C = ldp(pts, active ? jc : 0);
  // Pass 2: every tile that can hold a point within some voxel's limit.
  int k = 0;
  bool over = false;
  for (int k0 = 0; k0 < nt; k0 += kGroupTiles) {
    if (sc.dB[sc.ord[k0]] > cut) break;  // uniform
    const int ng = stage(k0);
    if (!active || over) continue;
    const float vcut = lim * (1.0f + kPassRel) + 1e-2f;
    for (int gt = 0; gt < ng && !over; ++gt) {
      const int t = sc.ord[k0 + gt];
      if (vgap2(t) > vcut) continue;  // every point of it fails the test below
      const int cnt = min(kTilePts, P - t * kTilePts);
      for (int i = gt * kTilePts; i < gt * kTilePts + cnt; ++i) {
        const float4 q = tile[i];
        const float nx = fmaxf(0.0f, fmaxf(lx - q.x, q.x - hx));
        const float ny = fmaxf(0.0f, fmaxf(ly - q.y, q.y - hy));
        const float nz = fmaxf(0.0f, fmaxf(lz - q.z, q.z - hz));
        if (nx * nx + ny * ny + nz * nz > lim) continue;
        const int j = __float_as_int(q.w);
        const P3 Q = ldp(pts, j);
        if (dominates(C, Q, bl, bh)) continue;
        if (k >= min(g.overflow, kVoxMaxCand)) {
          over = true;
          break;
        }
        cand[k++] = j;
      }
    }
  }
  if (!active) return 0;
  if (over) return -1;
  int kept = 0;  // pass 3 (exact): full dominance pruning among the survivors
  for (int a = 0; a < k; ++a) {
    const P3 A = ldp(pts, cand[a]);
    bool dominated = false;
    for (int c = 0; c < k && !dominated; ++c)
      if (c != a) dominated = dominates(ldp(pts, cand[c]), A, bl, bh);
    if (!dominated) cand[kept++] = cand[a];
  }
  return kept;
}

// Culled builds keep each voxel's first kKeep candidates (point indices)
// in `keep` [nv][kKeep], so the fill pass copies instead of recomputing
// (a CTA recomputes only if one of its voxels has more).
constexpr int kKeep = 8;

__global__ void __launch_bounds__(kBuildThreads) voxel_count_kernel(const double* pts, int P,
                                                                    VoxelGrid g, int32_t* counts,
                                                                    const float* tbox, int nt,
                                                                    int32_t* keep) {
  __shared__ float4 tile[kTile];
  __shared__ BrickScratch sc;
  int cand[kVoxMaxCand];
  if (nt > 0) {
    int ix, iy, iz;
    const bool in = brick_voxel(g, blockIdx.x, ix, iy, iz);
    const int k = voxel_list_culled(pts, P, g, blockIdx.x, ix, iy, iz, in, cand, tile, tbox, nt, sc);
    if (in) {
      const int v = (ix * g.dim_y + iy) * g.dim_z + iz;
      counts[v] = k;  // -1: overflow (the voxel scans the whole pocket, see fill)
      if (keep != nullptr)
        for (int a = 0; a < min(max(k, 0), kKeep); ++a) keep[kKeep * static_cast<size_t>(v) + a] = cand[a];
    }
    return;
  }
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const int nv = g.dim_x * g.dim_y * g.dim_z;
  const int k = voxel_list(pts, P, g, min(v, nv - 1), v < nv, cand, tile);
  if (v < nv) counts[v] = k;  // -1: overflow (the voxel scans the whole pocket, see fill)
}

__global__ void __launch_bounds__(kBuildThreads) voxel_fill_kernel(const double* pts, int P,
                                                                   VoxelGrid g,
                                                                   const int32_t* offsets,
                                                                   double* rec, double* lst,
                                                                   const float* tbox, int nt,
                                                                   const int32_t* counts,
                                                                   const int32_t* keep,
                                                                   const uint16_t* codes) {
  __shared__ float4 tile[kTile];
  __shared__ BrickScratch sc;
  int cand[kVoxMaxCand];
  int v, k;
  if (nt > 0) {
    int ix, iy, iz;
    const bool in = brick_voxel(g, blockIdx.x, ix, iy, iz);
    v = in ? (ix * g.dim_y + iy) * g.dim_z + iz : 0;
    const int c = in ? counts[v] : 0;
    if (keep != nullptr && !__syncthreads_or(c > kKeep || c < 0)) {  // uniform: copy the kept lists
      if (!in) return;
      k = c;
      for (int a = 0; a < k; ++a) cand[a] = keep[kKeep * static_cast<size_t>(v) + a];
    } else {
      k = voxel_list_culled(pts, P, g, blockIdx.x, ix, iy, iz, in, cand, tile, tbox, nt, sc);
      if (!in) return;
    }
  } else {
    v = blockIdx.x * blockDim.x + threadIdx.x;
    const int nv = g.dim_x * g.dim_y * g.dim_z;
    k = voxel_list(pts, P, g, min(v, nv - 1), v < nv, cand, tile);
    if (v >= nv) return;
  }
  // Overflow (more than kVoxMaxCand survivors, e.g. inside a hollow shell
  // pocket where no surface point dominates another): the voxel's list is
  // the whole pocket, which the list array holds once at its head (records
  // [0, P), copied by the host), so the record is {start 1, count P, point
  // 0 inline} and costs no list memory.
  const int len = k < 0 ? P : k;  // >= 1: the nearest point always survives
  const int start = k < 0 ? 1 : offsets[v];
  if (codes != nullptr) {
    // Coded: {start, count, 4 candidates} and list blocks of 5 past the
    // inline ones.  Overflow voxels: the head holds points 4.. of the whole
    // pocket in blocks of 5 from unit 0, the inline ones are points 0..3.
    auto pt = [&](int a) { return k < 0 ? a : cand[a]; };
    uint32_t* r = reinterpret_cast<uint32_t*>(rec + 4 * static_cast<size_t>(v));
    r[0] = static_cast<uint32_t>(k < 0 ? 0 : start);
    r[1] = static_cast<uint32_t>(len);
    uint16_t* e = reinterpret_cast<uint16_t*>(r + 2);
    for (int q = 0; q < kCodedInline; ++q) {
      const int j = pt(min(q, len - 1));
      for (int c = 0; c < 3; ++c) e[3 * q + c] = codes[3 * j + c];
    }
    if (k < 0) return;
    uint16_t* out = reinterpret_cast<uint16_t*>(lst + 4 * static_cast<size_t>(start));
    for (int a = kCodedInline; a < len; ++a) {
      const int b = a - kCodedInline;
      uint16_t* blk = out + 16 * (b / kCodedBlock) + 3 * (b % kCodedBlock);
      for (int c = 0; c < 3; ++c) blk[c] = codes[3 * pt(a) + c];
    }
    return;
  }
  double* r = rec + kRecDoubles * static_cast<size_t>(v);
  reinterpret_cast<int2*>(r)[0] = make_int2(start, len);
  for (int q = 0; q < kVoxInline; ++q) {
    const int a = min(q, len - 1);  // one candidate: repeat it
    const int j = k < 0 ? a : cand[a];
    for (int c = 0; c < 3; ++c) r[1 + 3 * q + c] = pts[4 * j + c];
  }
  if (kRecDoubles == 8) r[7] = 0.0;
  if (k < 0) return;
  double* out = lst + 4 * static_cast<size_t>(start);
  for (int a = kVoxInline; a < len; ++a) {
    const int j = cand[a];
    for (int c = 0; c < 4; ++c) out[4 * (a - kVoxInline) + c] = pts[4 * j + c];
  }
}

// List offsets on the device: offsets[v] = sum over earlier voxels of
// max(count - kVoxInline, 0); totals = {listed entries, candidates, max
// count}.  Three passes over 1024-voxel blocks (block sums, one-block scan
// of the sums, block-local scans), so the build needs no host round trip of
// the counts.
constexpr int kScanBlock = 1024;

__device__ __forceinline__ long long block_sum_ll(long long x, long long* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  long long t = 0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
  __syncthreads();
  return t;
}

// 32-byte list units of a voxel with `raw` candidates (overflow voxels,
// raw < 0, share the head: none of their own).
__device__ __forceinline__ int list_units(int raw, int compact) {
  return compact ? (max(raw - kCodedInline, 0) + kCodedBlock - 1) / kCodedBlock : max(raw - kVoxInline, 0);
}

__global__ void __launch_bounds__(kScanBlock) list_block_sums(const int32_t* counts, int nv, int P,
                                                              int compact, long long* bsum,
                                                              long long* bcand, int* bmax) {
  __shared__ long long red[kScanBlock / 32];
  __shared__ int mx;
  const int v = blockIdx.x * kScanBlock + threadIdx.x;
  const int raw = v < nv ? counts[v] : 0;
  const int c = raw < 0 ? P : raw;  // overflow voxels list the shared whole-pocket head
  if (threadIdx.x == 0) mx = 0;
  __syncthreads();
  atomicMax(&mx, c);
  const long long l = block_sum_ll(list_units(raw, compact), red);
  const long long t = block_sum_ll(c, red);
  if (threadIdx.x == 0) {
    bsum[blockIdx.x] = l;
    bcand[blockIdx.x] = t;
    bmax[blockIdx.x] = mx;
  }
}

// One block: exclusive scan of the block sums in place, and the totals.
__global__ void __launch_bounds__(kScanBlock) list_scan_sums(long long* bsum, const long long* bcand,
                                                             const int* bmax, int nb, long long base,
                                                             long long* totals) {
  __shared__ long long part[kScanBlock];
  __shared__ long long red[kScanBlock / 32];
  __shared__ int mx;
  const int per = (nb + kScanBlock - 1) / kScanBlock;  // consecutive sums per thread
  const int b0 = threadIdx.x * per;
  long long s = 0, cand = 0;
  int m = 0;
  for (int b = b0; b < min(nb, b0 + per); ++b) {
    s += bsum[b];
    cand += bcand[b];
    m = max(m, bmax[b]);
  }
  if (threadIdx.x == 0) mx = 0;
  part[threadIdx.x] = s;
  __syncthreads();
  atomicMax(&mx, m);
  for (int o = 1; o < kScanBlock; o <<= 1) {  // inclusive Hillis-Steele scan
    const long long y = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += y;
    __syncthreads();
  }
  long long run = base + part[threadIdx.x] - s;  // exclusive base of this thread's run
  for (int b = b0; b < min(nb, b0 + per); ++b) {
    const long long x = bsum[b];
    bsum[b] = run;
    run += x;
  }
  const long long tc = block_sum_ll(cand, red);
  if (threadIdx.x == kScanBlock - 1) totals[0] = base + part[kScanBlock - 1];
  if (threadIdx.x == 0) {
    totals[1] = tc;
    totals[2] = mx;
  }
}

__global__ void __launch_bounds__(kScanBlock) list_apply(const int32_t* counts, int nv, int compact,
                                                         const long long* bsum, int32_t* offsets) {
  __shared__ long long part[kScanBlock];
  const int v = blockIdx.x * kScanBlock + threadIdx.x;
  const long long x = v < nv ? list_units(counts[v], compact) : 0;
  part[threadIdx.x] = x;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {
    const long long y = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += y;
    __syncthreads();
  }
  if (v < nv) offsets[v] = static_cast<int32_t>(bsum[blockIdx.x] + part[threadIdx.x] - x);
}

// FP64 peak probe: 8 independent chains per thread of a DMUL and a DADD
// (no FMA: the hot path's recipe forbids it), 2 ops per step per chain.
__global__ void fp64_probe_kernel(double* sink, int iters) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = 1.0 + 1e-9 * (threadIdx.x + c);
  const double m = 0.9999999, d = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = dadd(dmul(a[c], m), d);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  if (s == 12345.0) sink[0] = s;  // keeps the chains live
}

// L2 gather probe: random 32-byte read-only loads (L1::no_allocate, as the
// index gathers) over a buffer that stays L2-resident, four independent
// loads in flight per thread.  The achieved rate is the denominator of the
// L2-gather roofline.
__global__ void l2_gather_probe_kernel(const double* buf, unsigned long long n_rec, int iters,
                                       double* sink) {
  unsigned long long h = (blockIdx.x * 0x9E3779B97F4A7C15ull) ^ (threadIdx.x * 0xBF58476D1CE4E5B9ull);
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      h ^= h >> 31;
      h *= 0x94D049BB133111EBull;
      h ^= h >> 29;
      double x, y, z, w;
      ld256<true>(buf + 4 * (h % n_rec), x, y, z, w);
      a[k] = x + w;
    }
    acc += (a[0] + a[1]) + (a[2] + a[3]);
  }
  if (acc == 12345.678) sink[0] = acc;  // keeps the loads live
}

// The same random 32-byte L1-bypassing gathers with one load in flight per
// thread: each address depends on the previous load's value (the buffer is
// zero, so the chain is real but the addresses stay random) -- the rate a
// kernel with `threads` resident lanes each waiting on its own gather gets.
__global__ void l2_chase_probe_kernel(const double* buf, unsigned long long n_rec, int iters, double* sink) {
  unsigned long long h = (blockIdx.x * 0x9E3779B97F4A7C15ull) ^ (threadIdx.x * 0xBF58476D1CE4E5B9ull);
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    h ^= h >> 31;
    h *= 0x94D049BB133111EBull;
    h ^= h >> 29;
    double x, y, z, w;
    ld256<true>(buf + 4 * (h % n_rec), x, y, z, w);
    h ^= static_cast<unsigned long long>(__double_as_longlong(x + w));
    acc += y;
  }
  if (acc == 12345.678) sink[0] = acc;
}

}  // namespace

int launch_l2_chase_probe(const double* buf, unsigned long long n_rec, int blocks, int threads, int iters,
                          double* sink, void* stream) {
  l2_chase_probe_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(buf, n_rec, iters, sink);
  return cudaGetLastError();
}

int launch_l2_gather_probe(const double* buf, unsigned long long n_rec, int blocks, int threads,
                           int iters, double* sink, void* stream) {
  l2_gather_probe_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(buf, n_rec,
                                                                                   iters, sink);
  return cudaGetLastError();
}

int launch_fp64_probe(double* sink, int blocks, int threads, int iters, void* stream) {
  fp64_probe_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(sink, iters);
  return cudaGetLastError();
}

int launch_score_poses(const PocketView& pk, const double* xyz, int n_atoms, int n_poses,
                       double* out, void* stream) {
  if (n_poses <= 0) return cudaSuccess;
  const int bt = 128;
  const unsigned blocks = (n_poses + bt - 1) / bt;
  if (pk.compact)
    score_poses_kernel<true><<<blocks, bt, 0, static_cast<cudaStream_t>(stream)>>>(pk, xyz, n_atoms,
                                                                                 n_poses, out);
  else
    score_poses_kernel<false><<<blocks, bt, 0, static_cast<cudaStream_t>(stream)>>>(pk, xyz, n_atoms,
                                                                                  n_poses, out);
  return cudaGetLastError();
}

static unsigned build_blocks(const VoxelGrid& g, int nt) {
  if (nt > 0)
    return static_cast<unsigned>(((g.dim_x + kBrickX - 1) / kBrickX) *
                                 ((g.dim_y + kBrickY - 1) / kBrickY) *
                                 ((g.dim_z + kBrickZ - 1) / kBrickZ));
  const int nv = g.dim_x * g.dim_y * g.dim_z;
  return static_cast<unsigned>((nv + kBuildThreads - 1) / kBuildThreads);
}

int launch_voxel_count(const double* pts, int P, VoxelGrid g, int32_t* counts, const float* tbox,
                       int nt, int32_t* keep, void* stream) {
  if (nt > kMaxTiles) nt = 0;  // too many tiles for the brick scratch: full scan
  voxel_count_kernel<<<build_blocks(g, nt), kBuildThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      pts, P, g, counts, tbox, nt, keep);
  return cudaGetLastError();
}

int launch_voxel_fill(const double* pts, int P, VoxelGrid g, const int32_t* offsets, double* rec,
                      double* lst, const float* tbox, int nt, const int32_t* counts,
                      const int32_t* keep, const uint16_t* codes, void* stream) {
  if (nt > kMaxTiles) nt = 0;
  voxel_fill_kernel<<<build_blocks(g, nt), kBuildThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      pts, P, g, offsets, rec, lst, tbox, nt, counts, keep, codes);
  return cudaGetLastError();
}

int list_offsets_scratch_bytes(int nv) {
  const int nb = (nv + kScanBlock - 1) / kScanBlock;
  return 3 * 8 * nb + 64;
}

int launch_list_offsets(const int32_t* counts, int nv, int P, long long base, int compact,
                        int32_t* offsets, void* scratch, long long* totals, void* stream) {
  const int nb = (nv + kScanBlock - 1) / kScanBlock;
  auto* bsum = static_cast<long long*>(scratch);
  long long* bcand = bsum + nb;
  int* bmax = reinterpret_cast<int*>(bcand + nb);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  list_block_sums<<<nb, kScanBlock, 0, st>>>(counts, nv, P, compact, bsum, bcand, bmax);
  list_scan_sums<<<1, kScanBlock, 0, st>>>(bsum, bcand, bmax, nb, base, totals);
  list_apply<<<nb, kScanBlock, 0, st>>>(counts, nv, compact, bsum, offsets);
  return cudaGetLastError();
}

}  // namespace gdb200
