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
#include <type_traits>

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

// Executed-work counters (exact; DESIGN.md §4 turns them into fp64 FLOPs).
// Kernels are instantiated twice: Work<true> counts (GD_FLAG_COUNT_WORK),
// Work<false> compiles every increment away so the timed kernels carry no
// counter registers.
enum WorkKind { kPairs, kRot, kBump, kQuery, kTerms, kEvals, kXform, kWorkKinds };
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

// Exact nearest-point query: the voxel's candidate list holds every point
// that can attain the fp64 minimum anywhere in the (slightly expanded)
// voxel, so the minimum is bit-identical to the brute-force scan (the
// reference's PocketIndex makes the same exactness argument,
// geometry.hpp:45-46).  Fine level first, then the coarse far-field level;
// queries beyond both fall back to the full scan.
//
// Two record formats (kernels.h), both in 32-byte units:
//   fp64  {int32 start, int32 count, x0, y0, z0}, list entries (x, y, z, pad);
//   coded {u32 start, u32 count, 4 inline candidates}, list blocks of 5
//         candidates; a candidate is three 16-bit indices into the pocket's
//         table of distinct coordinate values (PocketView::tab), chosen when
//         that table is small (lattice pockets).  The query reads the very
//         same doubles from the table, so the minimum has the same bits;
//         with four candidates inline almost no query needs a dependent
//         list load.
// Translation units compiled with GD_TU_COMPACT=1 (flex_cp, rigid_cp) read
// the coded format; the launchers dispatch on PocketView::compact.
#ifndef GD_TU_COMPACT
#define GD_TU_COMPACT 0
#endif
constexpr bool kCompactTU = GD_TU_COMPACT != 0;
#if GD_TU_COMPACT
#define GD_API(name) name##_cp
#else
#define GD_API(name) name
#endif

template <bool NoAlloc = false>
__device__ __forceinline__ void ld256w(const void* p, uint32_t (&w)[8]) {
  if constexpr (NoAlloc)
    asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
        : "l"(p));
  else
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
        : "l"(p));
}
// 16-bit field K (compile-time) of a word array.
template <int K, int N>
__device__ __forceinline__ unsigned u16at(const uint32_t (&w)[N]) {
  return (K & 1) ? (w[K >> 1] >> 16) : (w[K >> 1] & 0xffffu);
}
// The coded format's coordinate table, staged per CTA into shared memory
// (stage_tab) by every kernel that queries a coded pocket: a candidate
// coordinate is one shared load at [byte offset + table base].
__shared__ __align__(16) double s_tab[kCodedTab];
// A no-op in kernels compiled for the fp64 format (CP false: no table).
// The copy is one TMA bulk transfer (cp.async.bulk, SASS UBLKCP) of the whole
// zero-padded table, issued by thread 0 and awaited by every thread on an
// mbarrier, so no thread spends load/store instructions on it.
// GD_TAB_TMA=0 restores the cooperative copy (A/B).
#ifndef GD_TAB_TMA
#define GD_TAB_TMA 1
#endif
template <bool CP>
__device__ __forceinline__ void stage_tab(const PocketView& pk) {
  if constexpr (CP) {
#if GD_TAB_TMA
    __shared__ __align__(8) unsigned long long s_tab_bar;
    const unsigned bar = static_cast<unsigned>(__cvta_generic_to_shared(&s_tab_bar));
    constexpr unsigned kBytes = sizeof(double) * kCodedTab;
    static_assert(kBytes % 16 == 0, "bulk copies move multiples of 16 bytes");
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kBytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<unsigned>(__cvta_generic_to_shared(s_tab))),
          "l"(__cvta_generic_to_global(pk.tab)), "r"(kBytes), "r"(bar)
          : "memory");
    }
    __syncthreads();  // the initialised barrier is visible to every waiter
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar)
          : "memory");
#else
    for (int i = threadIdx.x; i < pk.ntab; i += blockDim.x) s_tab[i] = pk.tab[i];
    __syncthreads();
#endif
  }
}
__device__ __forceinline__ double tab_at(unsigned off) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const unsigned char*>(s_tab) + off);
}
// distance_sq to coded candidate C of a word array (fields 3C..3C+2).
template <int C, int N>
__device__ __forceinline__ double coded_d2(const double*, const uint32_t (&w)[N], double x, double y,
                                           double z) {
  return dist_sq(x, y, z, tab_at(u16at<3 * C>(w)), tab_at(u16at<3 * C + 1>(w)), tab_at(u16at<3 * C + 2>(w)));
}

// Voxel lookup: the record of the first grid level containing q (one or
// two independent 256-bit loads); lst == nullptr means the full-scan
// fallback.
struct Loc {
  const double* lst;  // further candidates (start already applied)
  int count;          // candidates in the voxel (>= 1)
  double x0, y0, z0;  // the inline candidates (the second only with
  double x1, y1, z1;  // kVoxInline == 2; it repeats the first when count == 1)
};
struct LocC {
  const double* lst;  // list blocks (start already applied)
  int count;          // candidates in the voxel (>= 1)
  uint32_t w[6];      // the inline candidates' table indices
};
template <bool CP>
using LocT = typename std::conditional<CP, LocC, Loc>::type;

// GD_LOCATE_FLAT=1 (coded format, two levels): both levels' voxels are
// computed up front and the record comes from ONE load -- the fine level's if
// the query is inside it, else the coarse level's -- instead of a second,
// divergent lookup (with its own L2 round trip) for the lanes outside the
// fine grid.  r3j, same box: c1 flex 10.57 -> 10.25 ms, c2 37.7 -> 36.4;
// rigid.cu opts out (it loses 5%).
#ifndef GD_LOCATE_FLAT
#define GD_LOCATE_FLAT 1
#endif
template <bool CP = kCompactTU>
__device__ __forceinline__ LocT<CP> locate(const PocketView& pk, double x, double y, double z) {
#if GD_LOCATE_FLAT
  if constexpr (CP && kGridLevels == 2) {
    if (pk.use_index) {
      const GridLevel& g0 = pk.lv[0];
      const GridLevel& g1 = pk.lv[1];
      const double fx = (x - g0.lo_x) * g0.inv_h, fy = (y - g0.lo_y) * g0.inv_h, fz = (z - g0.lo_z) * g0.inv_h;
      const double cx = (x - g1.lo_x) * g1.inv_h, cy = (y - g1.lo_y) * g1.inv_h, cz = (z - g1.lo_z) * g1.inv_h;
      const bool in0 = fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < g0.fdim_x && fy < g0.fdim_y && fz < g0.fdim_z;
      const bool in1 = cx >= 0.0 && cy >= 0.0 && cz >= 0.0 && cx < g1.fdim_x && cy < g1.fdim_y && cz < g1.fdim_z;
      if (in0 || in1) {
        const int v0 = (static_cast<int>(fx) * g0.dim_y + static_cast<int>(fy)) * g0.dim_z + static_cast<int>(fz);
        const int v1 = (static_cast<int>(cx) * g1.dim_y + static_cast<int>(cy)) * g1.dim_z + static_cast<int>(cz);
        const double* rec = in0 ? g0.rec + 4 * static_cast<size_t>(v0) : g1.rec + 4 * static_cast<size_t>(v1);
        uint32_t w[8];
        ld256w<GD_REC_NA>(rec, w);
        LocC l;
        l.count = static_cast<int>(w[1]);
        l.lst = (in0 ? g0.lst : g1.lst) + 4 * static_cast<size_t>(w[0]);
#pragma unroll
        for (int k = 0; k < 6; ++k) l.w[k] = w[2 + k];
        return l;
      }
    }
    LocC l{};
    l.lst = nullptr;
    return l;
  }
#endif
  if (pk.use_index) {
#pragma unroll
    for (int L = 0; L < kGridLevels; ++L) {
      const GridLevel& g = pk.lv[L];
      const double fx = (x - g.lo_x) * g.inv_h;
      const double fy = (y - g.lo_y) * g.inv_h;
      const double fz = (z - g.lo_z) * g.inv_h;
      if (fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < g.fdim_x && fy < g.fdim_y && fz < g.fdim_z) {
        const int v = (static_cast<int>(fx) * g.dim_y + static_cast<int>(fy)) * g.dim_z +
                      static_cast<int>(fz);
        if constexpr (CP) {
          uint32_t w[8];
          ld256w<GD_REC_NA>(g.rec + 4 * static_cast<size_t>(v), w);
          LocC l;
          l.count = static_cast<int>(w[1]);
          l.lst = g.lst + 4 * static_cast<size_t>(w[0]);
#pragma unroll
          for (int k = 0; k < 6; ++k) l.w[k] = w[2 + k];
          return l;
        } else {
          const double* r = g.rec + kRecDoubles * static_cast<size_t>(v);
          double hdr, pad;
          Loc l;
          ld256<GD_REC_NA>(r, hdr, l.x0, l.y0, l.z0);
          if constexpr (kVoxInline == 2) ld256<GD_REC_NA>(r + 4, l.x1, l.y1, l.z1, pad);
          const long long h = __double_as_longlong(hdr);
          l.count = static_cast<int>(h >> 32);
          l.lst = g.lst + 4 * static_cast<size_t>(static_cast<unsigned>(h & 0xffffffffll));
          return l;
        }
      }
    }
  }
  LocT<CP> l{};
  l.lst = nullptr;
  return l;
}

// min over the inline candidates; the list scan covers the rest.
__device__ __forceinline__ double inline_min(const PocketView&, const Loc& a, double x, double y, double z) {
  double m = dist_sq(x, y, z, a.x0, a.y0, a.z0);
  if constexpr (kVoxInline == 2) m = fmin(m, dist_sq(x, y, z, a.x1, a.y1, a.z1));
  return m;
}
// Unused inline slots of a coded record repeat its last candidate
// (voxel_fill_kernel), so slots can be evaluated two at a time without a
// count test in between: a warp runs the second pair whenever any lane's
// voxel holds more than two candidates (almost always), and two independent
// distance chains overlap where four predicated ones ran back to back.
// GD_CODED_PAIRED=0 restores one test per slot (r3j, same box: c1 flex
// 11.09 -> 10.82 ms, rigid 2.585 -> 2.550); 2 evaluates all four slots with
// no test (flex 10.52 vs 10.57, but rigid 2.68 vs 2.55: not adopted).
#ifndef GD_CODED_PAIRED
#define GD_CODED_PAIRED 1
#endif
__device__ __forceinline__ double inline_min(const PocketView& pk, const LocC& a, double x, double y,
                                             double z) {
#if GD_CODED_PAIRED == 2
  // All four slots, no count test at all.
  return fmin(fmin(coded_d2<0>(pk.tab, a.w, x, y, z), coded_d2<1>(pk.tab, a.w, x, y, z)),
              fmin(coded_d2<2>(pk.tab, a.w, x, y, z), coded_d2<3>(pk.tab, a.w, x, y, z)));
#elif GD_CODED_PAIRED
  double m = fmin(coded_d2<0>(pk.tab, a.w, x, y, z), coded_d2<1>(pk.tab, a.w, x, y, z));
  if (a.count > 2)
    m = fmin(m, fmin(coded_d2<2>(pk.tab, a.w, x, y, z), coded_d2<3>(pk.tab, a.w, x, y, z)));
  return m;
#else
  double m = coded_d2<0>(pk.tab, a.w, x, y, z);
  if (a.count > 1) m = fmin(m, coded_d2<1>(pk.tab, a.w, x, y, z));
  if (a.count > 2) m = fmin(m, coded_d2<2>(pk.tab, a.w, x, y, z));
  if (a.count > 3) m = fmin(m, coded_d2<3>(pk.tab, a.w, x, y, z));
  return m;
#endif
}
// List loads of a located voxel (0 on the full-scan fallback).
__device__ __forceinline__ int listed(const Loc& a) { return a.lst ? a.count - kVoxInline : 0; }
__device__ __forceinline__ int listed(const LocC& a) {
  return a.lst ? (max(a.count - kCodedInline, 0) + kCodedBlock - 1) / kCodedBlock : 0;
}
// Folds list load k of a located voxel into m.
__device__ __forceinline__ void list_min(const PocketView&, const Loc& a, int k, double x, double y,
                                         double z, double& m) {
  const P3 p = ldp<GD_LST_NA>(a.lst, k);
  m = fmin(m, dist_sq(x, y, z, p.x, p.y, p.z));
}
__device__ __forceinline__ void list_min(const PocketView& pk, const LocC& a, int k, double x, double y,
                                         double z, double& m) {
  uint32_t w[8];
  ld256w<GD_LST_NA>(a.lst + 4 * static_cast<size_t>(k), w);
  const int left = a.count - kCodedInline - kCodedBlock * k;  // >= 1
  m = fmin(m, coded_d2<0>(pk.tab, w, x, y, z));
  if (left > 1) m = fmin(m, coded_d2<1>(pk.tab, w, x, y, z));
  if (left > 2) m = fmin(m, coded_d2<2>(pk.tab, w, x, y, z));
  if (left > 3) m = fmin(m, coded_d2<3>(pk.tab, w, x, y, z));
  if (left > 4) m = fmin(m, coded_d2<4>(pk.tab, w, x, y, z));
}

template <bool On, bool CP = kCompactTU>
__device__ __forceinline__ double min_dist_sq(const PocketView& pk, double x, double y, double z,
                                              Work<On>& w) {
  w.add(kQuery, 1);
  const auto a = locate<CP>(pk, x, y, z);
  if (a.lst == nullptr) {
    w.add(kPairs, pk.P);
    return min_dist_sq_brute(pk.pts, pk.P, x, y, z);
  }
  w.add(kPairs, a.count);
  double m = inline_min(pk, a, x, y, z);
  const int nl = listed(a);
  for (int k = 0; k < nl; ++k) list_min(pk, a, k, x, y, z, m);
  return m;
}

// Two independent queries with both record loads issued before either scan
// and the two candidate scans interleaved (memory-level parallelism 2).
template <bool On>
__device__ __forceinline__ void min_dist_sq2(const PocketView& pk, double x0, double y0, double z0,
                                             double x1, double y1, double z1, double& m0,
                                             double& m1, Work<On>& w) {
  w.add(kQuery, 2);
  const auto a = locate(pk, x0, y0, z0);
  const auto b = locate(pk, x1, y1, z1);
  const int na = listed(a), nb = listed(b);
  w.add(kPairs, (a.lst ? a.count : 0) + (b.lst ? b.count : 0));
  m0 = inline_min(pk, a, x0, y0, z0);
  m1 = inline_min(pk, b, x1, y1, z1);
#if GD_WHATIF_NOLIST
  const int nmax = 0;  // timing experiment only: wrong minima
#else
  const int nmax = max(na, nb);
#endif
  for (int k = 0; k < nmax; ++k) {
    if (k < na) list_min(pk, a, k, x0, y0, z0, m0);
    if (k < nb) list_min(pk, b, k, x1, y1, z1, m1);
  }
  if (a.lst == nullptr) {
    w.add(kPairs, pk.P);
    m0 = min_dist_sq_brute(pk.pts, pk.P, x0, y0, z0);
  }
  if (b.lst == nullptr) {
    w.add(kPairs, pk.P);
    m1 = min_dist_sq_brute(pk.pts, pk.P, x1, y1, z1);
  }
}

// M independent queries: all M record loads in flight before any scan, the
// M candidate scans interleaved (memory-level parallelism M).
template <int M, bool On>
__device__ __forceinline__ void min_dist_sqM(const PocketView& pk, const double* x, const double* y,
                                             const double* z, double* m, Work<On>& w) {
  w.add(kQuery, M);
  LocT<kCompactTU> a[M];
#pragma unroll
  for (int r = 0; r < M; ++r) a[r] = locate(pk, x[r], y[r], z[r]);
  int nmax = 0;
#pragma unroll
  for (int r = 0; r < M; ++r) {
    m[r] = inline_min(pk, a[r], x[r], y[r], z[r]);
    nmax = max(nmax, listed(a[r]));
    if (a[r].lst) w.add(kPairs, a[r].count);
  }
  for (int k = 0; k < nmax; ++k) {
#pragma unroll
    for (int r = 0; r < M; ++r)
      if (k < listed(a[r])) list_min(pk, a[r], k, x[r], y[r], z[r], m[r]);
  }
#pragma unroll
  for (int r = 0; r < M; ++r) {
    if (a[r].lst == nullptr) {
      w.add(kPairs, pk.P);
      m[r] = min_dist_sq_brute(pk.pts, pk.P, x[r], y[r], z[r]);
    }
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
