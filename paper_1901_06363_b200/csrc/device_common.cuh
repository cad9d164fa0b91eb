// Device helpers shared by the sm_100a kernels (rigid.cu, flex.cu,
// pocket_index.cu).
//
// Numerics: every decision-critical value is computed in fp64 with
// __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn in the reference's
// expression order (vec3.hpp:19-44, geometry.hpp:140-213), so no FMA
// contraction can change a bit; the TUs are also built with -fmad=false.
// Scores, committed poses and all argmax/top-K decisions are therefore
// bit-identical to the reference CPU path.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "kernels.h"

namespace gdb200 {
namespace {

constexpr double kMinDistanceSq = 1e-12;  // geometry.hpp:33
constexpr double kBumpScale = 0.8;        // geometry.hpp:37
constexpr double kMinAxisLength = 1e-9;   // geometry.hpp:43
constexpr double kInfinity = __builtin_huge_val();
constexpr double kInfeasible = -1.0;      // scores are > 0

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// distance_sq (vec3.hpp:44): d = a - b; (d.x*d.x + d.y*d.y) + d.z*d.z.
__device__ __forceinline__ double dist_sq(double ax, double ay, double az, double bx, double by,
                                          double bz) {
  const double dx = dsub(ax, bx), dy = dsub(ay, by), dz = dsub(az, bz);
  return dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
}

// One 256-bit read-only load (LDG.256 on sm_100a) of a 32-byte record.
// Cache policy: voxel records and candidate lists are loaded with
// L1::no_allocate (scattered, rarely re-hit) so L1 keeps what does get
// re-read (spill slots, trig and orientation tables): c1 449k -> 471k
// ligands/s.  GD_REC_NA / GD_LST_NA = 0 restore allocation (A/B).
#ifndef GD_REC_NA
#define GD_REC_NA 1
#endif
#ifndef GD_LST_NA
#define GD_LST_NA 1
#endif
#ifndef GD_WHATIF_NOLIST
#define GD_WHATIF_NOLIST 0
#endif
template <bool NoAlloc = false>
__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  if constexpr (NoAlloc)
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
        : "l"(p));
  else
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
        : "l"(p));
}

// 32-byte point record (x, y, z, pad).
struct P3 {
  double x, y, z;
};
template <bool NoAlloc = false>
__device__ __forceinline__ P3 ldp(const double* base, int j) {
  double x, y, z, w;
  ld256<NoAlloc>(base + 4 * static_cast<size_t>(j), x, y, z, w);
  return P3{x, y, z};
}

// Executed-work counters (exact; DESIGN.md §4 turns them into FLOPs): fp64
// work {point pairs, rotated atoms, bump pairs, queries, score terms,
// candidate evaluations, rigid-transformed atoms}, then the fp32 screen's
// {point pairs, rotated atoms (rigid-transformed in the sweep), bump pairs,
// queries} and the candidates the screen had to resolve exactly.
// Kernels are instantiated twice: Work<true> counts (GD_FLAG_COUNT_WORK),
// Work<false> compiles every increment away so the timed kernels carry no
// counter registers.
enum WorkKind { kPairs, kRot, kBump, kQuery, kTerms, kEvals, kXform, kPairs32, kRot32, kBump32,
                kQuery32, kExactEvals, kWorkKinds };
template <bool On>
struct Work {
  unsigned c[kWorkKinds];
  __device__ Work() {
    if constexpr (On)
      for (int k = 0; k < kWorkKinds; ++k) c[k] = 0;
  }
  __device__ __forceinline__ void add(int k, unsigned v) {
    if constexpr (On) c[k] += v;
  }
};

// Per-thread publish (rigid kernel: all threads reach it).
template <bool On>
__device__ void publish(const Work<On>& w, unsigned long long* out, int base) {
  if constexpr (On) {
    if (out == nullptr) return;
    for (int k = 0; k < kWorkKinds; ++k) atomicAdd(out + base + k, static_cast<unsigned long long>(w.c[k]));
  }
}

// min_j distance_sq(q, P_j) over every pocket point (geometry.hpp:149-150).
// Out of line with plain arguments, so the rare call does not force the
// kernel parameters into local memory.
__device__ __noinline__ double min_dist_sq_brute(const double* pts, int P, double x, double y,
                                                 double z) {
  double m = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (int j = 0; j < P; ++j) {
    const P3 p = ldp(pts, j);
    m = fmin(m, dist_sq(x, y, z, p.x, p.y, p.z));
  }
  return m;
}

// 128-bit read-only loads of fp32 index records (L1::no_allocate: they are
// scattered and rarely re-hit; L1 keeps spill slots and the small tables).
struct F4 {
  float x, y, z;
  uint32_t w;
};
__device__ __forceinline__ F4 ld128(const float* p) {
  F4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldw(const float* p) {  // the w word of a record
  uint32_t w;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(w) : "l"(p + 3));
  return w;
}

// fp32 squared distance (explicit FMAs: the TU is built with -fmad=false).
__device__ __forceinline__ float d2f(float x, float y, float z, const F4& r) {
  const float dx = x - r.x, dy = y - r.y, dz = z - r.z;
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
}

// The voxel of (x, y, z) in the first grid level containing it, -1 if none.
template <class T>
__device__ __forceinline__ int voxel_of(const GridLevel& g, T fx, T fy, T fz) {
  if (fx >= T(0) && fy >= T(0) && fz >= T(0) && fx < T(g.dim_x) && fy < T(g.dim_y) && fz < T(g.dim_z))
    return (static_cast<int>(fx) * g.dim_y + static_cast<int>(fy)) * g.dim_z + static_cast<int>(fz);
  return -1;
}

__device__ __forceinline__ int count_of(const GridLevel& g, int v, uint32_t w) {
  const int cf = static_cast<int>(w >> kCountShift);
  return cf ? cf : __ldg(g.big + v);
}

// Exact nearest-point query (fp64, bit-identical to the brute-force scan):
// the voxel's candidate list holds every point that can attain the fp64
// minimum anywhere in the (slightly expanded) voxel -- the reference's
// PocketIndex makes the same exactness argument (geometry.hpp:45-46).  The
// voxel is located in fp64; candidates' fp64 coordinates come from the
// point table by index.  Fine level first, then the coarse far field;
// beyond both, the full scan.
template <bool On>
__device__ __forceinline__ double min_dist_sq(const PocketView& pk, double x, double y, double z,
                                              Work<On>& w) {
  w.add(kQuery, 1);
  if (pk.use_index) {
#pragma unroll
    for (int L = 0; L < kGridLevels; ++L) {
      const GridLevel& g = pk.lv[L];
      const int v = voxel_of(g, (x - g.lo_x) * g.inv_h, (y - g.lo_y) * g.inv_h, (z - g.lo_z) * g.inv_h);
      if (v < 0) continue;
      const uint32_t hw = ldw(g.rec + 4 * static_cast<size_t>(v));
      const int cnt = count_of(g, v, hw);
      w.add(kPairs, cnt);
      if (cnt == 1) {
        const P3 p = ldp<GD_LST_NA>(pk.pts, static_cast<int>(hw & kPayloadMask));
        return dist_sq(x, y, z, p.x, p.y, p.z);
      }
      const float* l = g.lst + 4 * static_cast<size_t>(hw & kPayloadMask);
      double m = __longlong_as_double(0x7ff0000000000000ll);
      for (int k = 0; k < cnt; k += 2) {  // two candidates per round in flight
        const bool two = k + 1 < cnt;
        const uint32_t i0 = ldw(l + 4 * k), i1 = two ? ldw(l + 4 * (k + 1)) : i0;
        const P3 p0 = ldp<GD_LST_NA>(pk.pts, static_cast<int>(i0));
        const P3 p1 = ldp<GD_LST_NA>(pk.pts, static_cast<int>(i1));
        m = fmin(m, dist_sq(x, y, z, p0.x, p0.y, p0.z));
        m = fmin(m, dist_sq(x, y, z, p1.x, p1.y, p1.z));
      }
      return m;
    }
  }
  w.add(kPairs, pk.P);
  return min_dist_sq_brute(pk.pts, pk.P, x, y, z);
}

__device__ __noinline__ float min_d2_brute_f32(const float* pts32, int P, float x, float y, float z) {
  float m = __int_as_float(0x7f800000);
  for (int j = 0; j < P; ++j) m = fminf(m, d2f(x, y, z, ld128(pts32 + 4 * j)));
  return m;
}

// fp32 screen queries, M at a time: min over the candidate list of the
// voxel containing each fp32 point (located in fp32) of fp32 squared
// distances to the fp32 coordinates; within the error bound the screens
// derive (flex.cu: screen_scores) of the exact minimum at the exact (fp64)
// position.  Latency-bound gathers, so everything is issued as early as
// possible: the M record loads together, then the lists walked two
// entries per query per round (2M loads in flight).
template <int M, bool On>
__device__ __forceinline__ void min_d2_f32(const PocketView& pk, const float* x, const float* y,
                                           const float* z, float* m, Work<On>& w) {
  w.add(kQuery32, M);
  int lv[M], vox[M];
#pragma unroll
  for (int r = 0; r < M; ++r) {
    lv[r] = -1;
    vox[r] = 0;
    if (pk.use_index) {
#pragma unroll
      for (int L = kGridLevels - 1; L >= 0; --L) {  // the finest level containing the point wins
        const GridLevel& g = pk.lv[L];
        const int v = voxel_of(g, (x[r] - g.flo_x) * g.finv_h, (y[r] - g.flo_y) * g.finv_h,
                               (z[r] - g.flo_z) * g.finv_h);
        if (v >= 0) {
          lv[r] = L;
          vox[r] = v;
        }
      }
    }
  }
  F4 rec[M];
  const float* lst[M];
  int cnt[M];
#pragma unroll
  for (int r = 0; r < M; ++r) {
    const GridLevel& g = pk.lv[lv[r] > 0 ? 1 : 0];
    rec[r] = lv[r] >= 0 ? ld128(g.rec + 4 * static_cast<size_t>(vox[r])) : F4{0.f, 0.f, 0.f, 1u << kCountShift};
    lst[r] = g.lst;
  }
  int most = 1;
#pragma unroll
  for (int r = 0; r < M; ++r) {
    const GridLevel& g = pk.lv[lv[r] > 0 ? 1 : 0];
    const int cf = static_cast<int>(rec[r].w >> kCountShift);
    cnt[r] = cf ? cf : __ldg(g.big + vox[r]);
    lst[r] += 4 * static_cast<size_t>(rec[r].w & kPayloadMask);
    m[r] = d2f(x[r], y[r], z[r], rec[r]);
    w.add(kPairs32, lv[r] >= 0 ? cnt[r] : 0);
    most = max(most, cnt[r]);
  }
#if GD_WHATIF_NOLIST
  most = 1;  // timing experiment only: wrong minima
#endif
  for (int k = 1; k < most; k += 2) {
    F4 e0[M], e1[M];
#pragma unroll
    for (int r = 0; r < M; ++r) {
      if (k < cnt[r]) e0[r] = ld128(lst[r] + 4 * k);
      if (k + 1 < cnt[r]) e1[r] = ld128(lst[r] + 4 * (k + 1));
    }
#pragma unroll
    for (int r = 0; r < M; ++r) {
      if (k < cnt[r]) m[r] = fminf(m[r], d2f(x[r], y[r], z[r], e0[r]));
      if (k + 1 < cnt[r]) m[r] = fminf(m[r], d2f(x[r], y[r], z[r], e1[r]));
    }
  }
#pragma unroll
  for (int r = 0; r < M; ++r)
    if (lv[r] < 0) {  // beyond both grids: the whole pocket
      w.add(kPairs32, pk.P);
      m[r] = min_d2_brute_f32(pk.pts32, pk.P, x[r], y[r], z[r]);
    }
}

// Rodrigues rotation of one atom (geometry.hpp:182-184):
// ((o + v*c) + cross(k,v)*s) + k*(dot(k,v)*(1-c)), v = p - o.
struct Axis {
  double ox, oy, oz, kx, ky, kz;
};
// The angle-independent part of a Rodrigues rotation of point p about the
// axis: v = p - o, k x v and k . v (geometry.hpp:180-184) ...
struct Arm {
  double vx, vy, vz, crx, cry, crz, d;
};
__device__ __forceinline__ Arm arm_of(const Axis& a, double px, double py, double pz) {
  Arm r;
  r.vx = dsub(px, a.ox);
  r.vy = dsub(py, a.oy);
  r.vz = dsub(pz, a.oz);
  r.crx = dsub(dmul(a.ky, r.vz), dmul(a.kz, r.vy));
  r.cry = dsub(dmul(a.kz, r.vx), dmul(a.kx, r.vz));
  r.crz = dsub(dmul(a.kx, r.vy), dmul(a.ky, r.vx));
  r.d = dadd(dadd(dmul(a.kx, r.vx), dmul(a.ky, r.vy)), dmul(a.kz, r.vz));
  return r;
}
// ... and the per-angle part: ((o + v c) + (k x v) s) + k ((k . v)(1 - c)).
__device__ __forceinline__ void turn(const Axis& a, const Arm& r, double c, double s, double omc,
                                     double& qx, double& qy, double& qz) {
  const double w = dmul(r.d, omc);
  qx = dadd(dadd(dadd(a.ox, dmul(r.vx, c)), dmul(r.crx, s)), dmul(a.kx, w));
  qy = dadd(dadd(dadd(a.oy, dmul(r.vy, c)), dmul(r.cry, s)), dmul(a.ky, w));
  qz = dadd(dadd(dadd(a.oz, dmul(r.vz, c)), dmul(r.crz, s)), dmul(a.kz, w));
}
__device__ __forceinline__ void rodrigues(const Axis& a, double c, double s, double omc, double px,
                                          double py, double pz, double& qx, double& qy,
                                          double& qz) {
  turn(a, arm_of(a, px, py, pz), c, s, omc, qx, qy, qz);
}

// Rigid pose (E3): p' = c + R (p - c), rows summed left to right.
__device__ __forceinline__ void rigid_apply(const double* R, double cx, double cy, double cz,
                                            double vx, double vy, double vz, double& x, double& y,
                                            double& z) {
  x = dadd(cx, dadd(dadd(dmul(R[0], vx), dmul(R[1], vy)), dmul(R[2], vz)));
  y = dadd(cy, dadd(dadd(dmul(R[3], vx), dmul(R[4], vy)), dmul(R[5], vz)));
  z = dadd(cz, dadd(dadd(dmul(R[6], vx), dmul(R[7], vy)), dmul(R[8], vz)));
}

// (score desc, slot asc): does (ka, ia) precede (kb, ib)?
__device__ __forceinline__ bool precede(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

}  // namespace
}  // namespace gdb200
