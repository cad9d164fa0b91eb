// B200 (sm_100a) kernels of the GeoDock-MA pose-search hot path.
//
//   rigid_topk_kernel  (1)+(4)+(5b): one CTA per ligand; one thread per
//                      orientation of the rigid Euler grid scores the rotated
//                      ligand, then a shared-memory bitonic merge keeps the
//                      top-K seeds (score desc, orientation asc).
//   flex_kernel        (2)+(3)+(4)+(5a): one CTA per ligand, G seed chains
//                      resident in shared memory; each greedy sub-step
//                      evaluates every (chain, angle) candidate in parallel
//                      (Rodrigues rotation, bump check, overlap score), then
//                      reduces per chain with the reference's tie rules and
//                      commits.  Restarts = KnobConfig::repetitions.
//   score_poses_kernel overlap_score for arbitrary poses (drop-in API).
//   voxel_*_kernel     exact voxel candidate lists for nearest-point queries.
//
// Numerics: every decision-critical value is computed in fp64 with
// __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn in the reference's
// expression order (vec3.hpp:19-44, geometry.hpp:140-213), so no FMA
// contraction can change a bit; the TU is also built with -fmad=false.
// Scores, committed poses and all argmax/top-K decisions are therefore
// bit-identical to the reference CPU path.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "kernels.h"

namespace gdb200 {
namespace {

constexpr double kMinDistanceSq = 1e-12;  // geometry.hpp:33
constexpr double kBumpScale = 0.8;        // geometry.hpp:37
constexpr double kMinAxisLength = 1e-9;   // geometry.hpp:43
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

// 32-byte point record (x, y, z, pad) through the read-only path.
struct P3 {
  double x, y, z;
};
__device__ __forceinline__ P3 ldp(const double* base, int j) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(base) + 2 * j);
  const double b = __ldg(base + 4 * j + 2);
  return P3{a.x, a.y, b};
}

// min_j distance_sq(q, P_j) over every pocket point (geometry.hpp:149-150).
__device__ __noinline__ double min_dist_sq_brute(const PocketView& pk, double x, double y,
                                                 double z) {
  double m = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  for (int j = 0; j < pk.P; ++j) {
    const P3 p = ldp(pk.pts, j);
    m = fmin(m, dist_sq(x, y, z, p.x, p.y, p.z));
  }
  return m;
}

// Exact nearest-point query: the voxel's candidate list holds every point
// that can attain the fp64 minimum anywhere in the (slightly expanded)
// voxel, so the minimum is bit-identical to the brute-force scan; queries
// outside the grid fall back to the scan (the reference's PocketIndex makes
// the same exactness argument, geometry.hpp:45-46).
// Work counted per thread (exact, for the roofline's algorithmic FLOPs;
// published to DockParams::counters only when that pointer is set).
struct Work {
  unsigned long long pairs = 0;  // atom x pocket-point distance evaluations
  unsigned long long rot = 0;    // atoms rotated (Rodrigues)
  unsigned long long bump = 0;   // bump pairs tested
  unsigned long long query = 0;  // nearest-point queries
  unsigned long long terms = 0;  // score-sum terms
  unsigned long long evals = 0;  // nonzero-angle candidates evaluated
  unsigned long long xform = 0;  // rigid-transformed atoms
};

__device__ __forceinline__ double min_dist_sq(const PocketView& pk, double x, double y, double z,
                                              Work& w) {
  ++w.query;
  if (pk.use_index) {
#pragma unroll
    for (int L = 0; L < kGridLevels; ++L) {
      const GridLevel& g = pk.lv[L];
      const double fx = (x - g.lo_x) * g.inv_h;
      const double fy = (y - g.lo_y) * g.inv_h;
      const double fz = (z - g.lo_z) * g.inv_h;
      if (fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < g.dim_x && fy < g.dim_y && fz < g.dim_z) {
        const int v = (static_cast<int>(fx) * g.dim_y + static_cast<int>(fy)) * g.dim_z +
                      static_cast<int>(fz);
        const int s = __ldg(g.off + v), e = __ldg(g.off + v + 1);
        w.pairs += e - s;
        double m = __longlong_as_double(0x7ff0000000000000ll);
        for (int k = s; k < e; ++k) {
          const P3 p = ldp(g.pts, k);
          m = fmin(m, dist_sq(x, y, z, p.x, p.y, p.z));
        }
        return m;
      }
    }
  }
  w.pairs += pk.P;
  return min_dist_sq_brute(pk, x, y, z);
}

__device__ void publish(const Work& w, unsigned long long* c, int base) {
  if (c == nullptr) return;
  atomicAdd(c + base + 0, w.pairs);
  atomicAdd(c + base + 1, w.rot);
  atomicAdd(c + base + 2, w.bump);
  atomicAdd(c + base + 3, w.query);
  atomicAdd(c + base + 4, w.terms);
  atomicAdd(c + base + 5, w.evals);
  atomicAdd(c + base + 6, w.xform);
}

// Rodrigues rotation of one atom (geometry.hpp:182-184):
// ((o + v*c) + cross(k,v)*s) + k*(dot(k,v)*(1-c)), v = p - o.
struct Axis {
  double ox, oy, oz, kx, ky, kz;
};
__device__ __forceinline__ void rodrigues(const Axis& a, double c, double s, double omc, double px,
                                          double py, double pz, double& qx, double& qy,
                                          double& qz) {
  const double vx = dsub(px, a.ox), vy = dsub(py, a.oy), vz = dsub(pz, a.oz);
  const double crx = dsub(dmul(a.ky, vz), dmul(a.kz, vy));
  const double cry = dsub(dmul(a.kz, vx), dmul(a.kx, vz));
  const double crz = dsub(dmul(a.kx, vy), dmul(a.ky, vx));
  const double d = dadd(dadd(dmul(a.kx, vx), dmul(a.ky, vy)), dmul(a.kz, vz));
  const double w = dmul(d, omc);
  qx = dadd(dadd(dadd(a.ox, dmul(vx, c)), dmul(crx, s)), dmul(a.kx, w));
  qy = dadd(dadd(dadd(a.oy, dmul(vy, c)), dmul(cry, s)), dmul(a.ky, w));
  qz = dadd(dadd(dadd(a.oz, dmul(vz, c)), dmul(crz, s)), dmul(a.kz, w));
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

template <int BT>
__device__ void bitonic_sort(double* key, int* idx, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += BT) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const double ki = key[i], kj = key[ixj];
          const int ii = idx[i], ij = idx[ixj];
          const bool sw = up ? precede(kj, ij, ki, ii) : precede(ki, ii, kj, ij);
          if (sw) {
            key[i] = kj;
            key[ixj] = ki;
            idx[i] = ij;
            idx[ixj] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// (1) rigid sweep + (5b) top-K seed selection.
// --------------------------------------------------------------------------
template <int BT>
__global__ void __launch_bounds__(BT) rigid_topk_kernel(DockParams p, int sort_slots) {
  const int l = p.order[blockIdx.x];
  const LigMeta m = p.meta[l];
  if (m.status != 0) {
    if (threadIdx.x == 0) p.k_eff[l] = 0;
    return;
  }
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = m.n;
  double* vx = reinterpret_cast<double*>(smem);
  double* vy = vx + n;
  double* vz = vy + n;
  double* key = vz + n;
  int* slot = reinterpret_cast<int*>(key + sort_slots);

  // v = p - c once per atom (the first operation of E3).
  for (int i = threadIdx.x; i < n; i += BT) {
    const double* q = p.xyz + 3 * (m.atom_off + i);
    vx[i] = dsub(q[0], p.cx);
    vy[i] = dsub(q[1], p.cy);
    vz[i] = dsub(q[2], p.cz);
  }
  __syncthreads();

  const int No = p.n_orient;
  const int K = min(p.top_k, No);
  const double dn = static_cast<double>(n);
  Work wk;
  int carry = 0;
  for (int base = 0; base < No;) {
    const int take = min(sort_slots - carry, No - base);
    for (int t = threadIdx.x; t < sort_slots - carry; t += BT) {
      double score = kInfeasible;
      int s = INT_MAX;
      if (t < take) {
        s = base + t;
        double R[9];
#pragma unroll
        for (int r = 0; r < 9; ++r) R[r] = __ldg(p.orient_R + 9 * s + r);
        // overlap_score (geometry.hpp:143-154): atom-order sum.
        double sum = 0.0;
        for (int i = 0; i < n; ++i) {
          double x, y, z;
          rigid_apply(R, p.cx, p.cy, p.cz, vx[i], vy[i], vz[i], x, y, z);
          ++wk.xform;
          sum = dadd(sum, fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk)));
        }
        score = __ddiv_rn(dn, sum);
      }
      key[carry + t] = score;
      slot[carry + t] = s;
    }
    base += take;
    __syncthreads();
    bitonic_sort<BT>(key, slot, sort_slots);
    carry = min(K, carry + take);
  }
  for (int r = threadIdx.x; r < K; r += BT) {
    p.seed_slot[l * p.top_k + r] = slot[r];
    p.seed_score[l * p.top_k + r] = key[r];
  }
  if (threadIdx.x == 0) p.k_eff[l] = K;
  publish(wk, p.counters, 0);
}

// --------------------------------------------------------------------------
// (2)(3)(4)(5a) fragment optimisation with restarts, K chains per ligand.
// --------------------------------------------------------------------------
struct FlexSmem {
  double* radius;   // [n]
  uint64_t* far;    // [n*W]
  double *px, *py, *pz, *minc;  // [G*n] chain poses and per-atom minima
  double* score;    // [G*amax] candidate scores of the current sub-step
  double* cur;      // [G] committed score
  double *ox, *oy, *oz, *kx, *ky, *kz;  // [G] rotation axis of the step
  double *best_s, *win_s;               // [G]
  long long *evals, *checks;            // [G]
  int *best_a, *win_t, *have;           // [G]
  double* fin;      // [K] final scores in rank order (for E7)
  uint64_t* fmask;  // [W] current fragment
  int* flag;        // [1] degenerate axis seen
};

__device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__device__ FlexSmem carve(unsigned char* base, int n, int W, int G, int amax, int K) {
  FlexSmem s;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    unsigned char* ptr = base + o;
    o = align16(o + bytes);
    return ptr;
  };
  s.radius = reinterpret_cast<double*>(take(sizeof(double) * n));
  s.far = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n * W));
  s.px = reinterpret_cast<double*>(take(sizeof(double) * G * n));
  s.py = reinterpret_cast<double*>(take(sizeof(double) * G * n));
  s.pz = reinterpret_cast<double*>(take(sizeof(double) * G * n));
  s.minc = reinterpret_cast<double*>(take(sizeof(double) * G * n));
  s.score = reinterpret_cast<double*>(take(sizeof(double) * G * amax));
  s.cur = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.ox = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.oy = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.oz = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.kx = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.ky = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.kz = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.best_s = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.win_s = reinterpret_cast<double*>(take(sizeof(double) * G));
  s.evals = reinterpret_cast<long long*>(take(sizeof(long long) * G));
  s.checks = reinterpret_cast<long long*>(take(sizeof(long long) * G));
  s.best_a = reinterpret_cast<int*>(take(sizeof(int) * G));
  s.win_t = reinterpret_cast<int*>(take(sizeof(int) * G));
  s.have = reinterpret_cast<int*>(take(sizeof(int) * G));
  s.fin = reinterpret_cast<double*>(take(sizeof(double) * K));
  s.fmask = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 4));
  s.flag = reinterpret_cast<int*>(take(sizeof(int) * 4));
  return s;
}

size_t flex_smem_bytes_impl(int n, int W, int G, int amax, int K) {
  auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t o = 0;
  o += a16(sizeof(double) * n);
  o += a16(sizeof(uint64_t) * n * W);
  o += 4 * a16(sizeof(double) * G * n);
  o += a16(sizeof(double) * G * amax);
  o += 9 * a16(sizeof(double) * G);
  o += 2 * a16(sizeof(long long) * G);
  o += 3 * a16(sizeof(int) * G);
  o += a16(sizeof(double) * K);
  o += a16(sizeof(uint64_t) * 4);
  o += a16(sizeof(int) * 4);
  return o;
}

// CandidateEvaluator::evaluate (kernel.hpp:100-112) for chain g at a
// nonzero angle: rotate the fragment, check_bumps (geometry.hpp:199-213),
// then overlap_score with the unchanged atoms' minima reused from the
// committed pose (identical values, identical atom-order sum).
__device__ double evaluate(const FlexSmem& s, const DockParams& p, int n, int W, int g, int angle,
                           Work& wk) {
  ++wk.evals;
  const double c = __ldg(p.cos_deg + angle), sn = __ldg(p.sin_deg + angle);
  const double omc = dsub(1.0, c);
  const Axis ax{s.ox[g], s.oy[g], s.oz[g], s.kx[g], s.ky[g], s.kz[g]};
  const double* px = s.px + g * n;
  const double* py = s.py + g * n;
  const double* pz = s.pz + g * n;
  // Bump pass: any fragment atom vs any non-fragment atom >= 4 bonds away.
  for (int w = 0; w < W; ++w) {
    uint64_t bits = s.fmask[w];
    while (bits) {
      const int i = w * 64 + __ffsll(static_cast<long long>(bits)) - 1;
      bits &= bits - 1;
      double qx, qy, qz;
      rodrigues(ax, c, sn, omc, px[i], py[i], pz[i], qx, qy, qz);
      ++wk.rot;
      const double ri = s.radius[i];
      for (int w2 = 0; w2 < W; ++w2) {
        uint64_t partners = s.far[i * W + w2] & ~s.fmask[w2];
        while (partners) {
          const int j = w2 * 64 + __ffsll(static_cast<long long>(partners)) - 1;
          partners &= partners - 1;
          ++wk.bump;
          const double cutoff = dmul(kBumpScale, dadd(ri, s.radius[j]));
          if (dist_sq(qx, qy, qz, px[j], py[j], pz[j]) < dmul(cutoff, cutoff)) return kInfeasible;
        }
      }
    }
  }
  // Score pass.
  const double* mc = s.minc + g * n;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    double mi;
    if ((s.fmask[i >> 6] >> (i & 63)) & 1ull) {
      double qx, qy, qz;
      rodrigues(ax, c, sn, omc, px[i], py[i], pz[i], qx, qy, qz);
      ++wk.rot;
      mi = min_dist_sq(p.pocket, qx, qy, qz, wk);
    } else {
      mi = mc[i];
    }
    sum = dadd(sum, fmax(kMinDistanceSq, mi));
  }
  wk.terms += n;
  return __ddiv_rn(static_cast<double>(n), sum);
}

// Angle of candidate k of chain g in the current sub-step.
struct SubStep {
  int kind;    // 0 = flat, 1 = refined phase 1, 2 = refined phase 2
  int step;    // flat step / hp
  int tile;
  int count;   // candidates per chain
};
__device__ __forceinline__ int angle_of(const SubStep& ss, const FlexSmem& s, int g, int k) {
  if (ss.kind == 0) return (k + 1) * ss.step;
  if (ss.kind == 1) return k * ss.tile + ss.tile / 2;
  return s.win_t[g] * ss.tile + k * ss.step;
}

template <int BT>
__device__ void eval_substep(const FlexSmem& s, const DockParams& p, int n, int W, int G,
                             const SubStep& ss, Work& wk) {
  const int total = G * ss.count;
  for (int t = threadIdx.x; t < total; t += BT) {
    const int g = t / ss.count, k = t - g * ss.count;
    if (ss.kind == 2 && s.win_t[g] < 0) continue;
    const int angle = angle_of(ss, s, g, k);
    // Angle 0 is the committed pose: always feasible, score == cur (the
    // committed pose is bit-identical to the candidate it was scored as).
    s.score[g * p.amax + k] = angle == 0 ? s.cur[g] : evaluate(s, p, n, W, g, angle, wk);
  }
  __syncthreads();
}

template <int BT>
__global__ void __launch_bounds__(BT) flex_kernel(DockParams p) {
  const int l = p.order[blockIdx.x];
  const LigMeta m = p.meta[l];
  if (m.status != 0) return;
  const int n = m.n, W = m.words;
  const int K = p.rigid ? p.k_eff[l] : 1;
  const int G = min(p.chains_per_cta, K);
  extern __shared__ __align__(16) unsigned char smem[];
  const FlexSmem s = carve(smem, n, W, G, p.amax, p.rigid ? p.top_k : 1);

  for (int i = threadIdx.x; i < n; i += BT) s.radius[i] = p.radii[m.atom_off + i];
  for (int i = threadIdx.x; i < n * W; i += BT) s.far[i] = p.far_mask[m.far_off + i];
  if (threadIdx.x == 0) s.flag[0] = 0;

  const int slots = p.top_k;
  Work wk;
  for (int g0 = 0; g0 < K; g0 += G) {
    const int Gc = min(G, K - g0);
    // Chain start poses: the rigid seed pose (E3) or the given pose.
    for (int t = threadIdx.x; t < Gc * n; t += BT) {
      const int g = t / n, i = t - g * n;
      const double* q = p.xyz + 3 * (m.atom_off + i);
      double x = q[0], y = q[1], z = q[2];
      if (p.rigid) {
        const int o = p.seed_slot[l * slots + g0 + g];
        double R[9];
#pragma unroll
        for (int r = 0; r < 9; ++r) R[r] = __ldg(p.orient_R + 9 * o + r);
        rigid_apply(R, p.cx, p.cy, p.cz, dsub(x, p.cx), dsub(y, p.cy), dsub(z, p.cz), x, y, z);
      }
      s.px[g * n + i] = x;
      s.py[g * n + i] = y;
      s.pz[g * n + i] = z;
      if (p.rigid) ++wk.xform;
      s.minc[g * n + i] = min_dist_sq(p.pocket, x, y, z, wk);
    }
    __syncthreads();
    // match_probes_shape prologue (kernel.hpp:215-218).
    for (int g = threadIdx.x; g < Gc; g += BT) {
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum = dadd(sum, fmax(kMinDistanceSq, s.minc[g * n + i]));
      s.cur[g] = __ddiv_rn(static_cast<double>(n), sum);
      if (!p.rigid) p.seed_score[l * slots + g0 + g] = s.cur[g];  // input pose score
      s.evals[g] = 1;
      s.checks[g] = 1;
    }
    __syncthreads();

    for (int rep = 0; rep < p.reps; ++rep) {
      for (int f = 0; f < m.nfrag; ++f) {
        const int fo = m.frag_off + f;
        const int axis = p.frag_axis[fo], anchor = p.frag_anchor[fo];
        const double rel = p.frag_rel[fo];
        // Dispatch (kernel.hpp:229-239).
        const bool low = rel <= p.threshold;
        const bool refined = !low && p.refine;
        const int step = low ? p.lp : p.hp;
        const int A = 360 / step;
        const bool rotates = refined || A > 1;
        for (int w = threadIdx.x; w < W; w += BT) s.fmask[w] = p.frag_mask[m.fmask_off + f * W + w];
        // rotate_fragment_into axis (geometry.hpp:165-169).
        for (int g = threadIdx.x; g < Gc; g += BT) {
          const double ox = s.px[g * n + axis], oy = s.py[g * n + axis], oz = s.pz[g * n + axis];
          const double ax = dsub(s.px[g * n + anchor], ox);
          const double ay = dsub(s.py[g * n + anchor], oy);
          const double az = dsub(s.pz[g * n + anchor], oz);
          const double len = __dsqrt_rn(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az)));
          if (rotates && len < kMinAxisLength) atomicExch(s.flag, 1);
          s.ox[g] = ox;
          s.oy[g] = oy;
          s.oz[g] = oz;
          s.kx[g] = __ddiv_rn(ax, len);
          s.ky[g] = __ddiv_rn(ay, len);
          s.kz[g] = __ddiv_rn(az, len);
        }
        __syncthreads();
        if (s.flag[0]) {  // "rotate_fragment: degenerate rotation axis"
          if (threadIdx.x == 0) p.status[l] = 3;
          return;
        }
        if (!refined) {
          // optimize_fragment_flat (kernel.hpp:125-143).
          if (A > 1) eval_substep<BT>(s, p, n, W, Gc, SubStep{0, step, 0, A - 1}, wk);
          for (int g = threadIdx.x; g < Gc; g += BT) {
            int best_a = 0;
            double best = s.cur[g];
            long long nf = 0;
            for (int k = 0; k < A - 1; ++k) {
              const double sc = s.score[g * p.amax + k];
              if (sc == kInfeasible) continue;
              ++nf;
              if (sc > best) {
                best = sc;
                best_a = (k + 1) * step;
              }
            }
            s.checks[g] += A;
            s.evals[g] += 1 + nf;
            s.best_a[g] = best_a;
            s.best_s[g] = best;
          }
        } else {
          // optimize_fragment_refined (kernel.hpp:150-198).
          const int T = p.tile, tc = 360 / T;
          eval_substep<BT>(s, p, n, W, Gc, SubStep{1, p.hp, T, tc}, wk);
          for (int g = threadIdx.x; g < Gc; g += BT) {
            int have = 0, best_a = 0, wt = -1;
            double best = 0.0, ws = 0.0;
            long long nf = 0;
            for (int t = 0; t < tc; ++t) {
              const double sc = s.score[g * p.amax + t];
              if (sc == kInfeasible) continue;
              ++nf;
              if (!have || sc > best) {
                best = sc;
                best_a = t * T + T / 2;
                have = 1;
              }
              if (wt < 0 || sc > ws) {
                wt = t;
                ws = sc;
              }
            }
            s.checks[g] += tc;
            s.evals[g] += nf;
            s.have[g] = have;
            s.best_a[g] = best_a;
            s.best_s[g] = best;
            s.win_t[g] = wt;
          }
          __syncthreads();
          int cnt2 = 0;
          while ((cnt2 + 1) * p.hp <= T) ++cnt2;
          eval_substep<BT>(s, p, n, W, Gc, SubStep{2, p.hp, T, cnt2}, wk);
          for (int g = threadIdx.x; g < Gc; g += BT) {
            int have = s.have[g], best_a = s.best_a[g];
            double best = s.best_s[g];
            if (s.win_t[g] >= 0) {
              long long nf = 0;
              for (int k = 0; k < cnt2; ++k) {
                const double sc = s.score[g * p.amax + k];
                if (sc == kInfeasible) continue;
                ++nf;
                if (!have || sc > best) {
                  best = sc;
                  best_a = s.win_t[g] * T + k * p.hp;
                  have = 1;
                }
              }
              s.checks[g] += cnt2;
              s.evals[g] += nf;
            }
            // Entry pose comparison (kernel.hpp:192-194), one more check.
            s.checks[g] += 1;
            if (!have || s.cur[g] > best) {
              best = s.cur[g];
              best_a = 0;
            }
            s.best_a[g] = best_a;
            s.best_s[g] = best;
          }
        }
        __syncthreads();
        // commit_angle (kernel.hpp:115-117): fresh rotation of the entry
        // pose, bit-identical to the scored candidate; refresh its minima.
        for (int w = 0; w < W; ++w) {
          for (int t = threadIdx.x; t < Gc * 64; t += BT) {
            const int g = t >> 6, b = t & 63;
            const int i = w * 64 + b;
            const int a = s.best_a[g];
            if (a == 0 || !((s.fmask[w] >> b) & 1ull)) continue;
            const Axis axs{s.ox[g], s.oy[g], s.oz[g], s.kx[g], s.ky[g], s.kz[g]};
            const double c = __ldg(p.cos_deg + a), sn = __ldg(p.sin_deg + a);
            double qx, qy, qz;
            rodrigues(axs, c, sn, dsub(1.0, c), s.px[g * n + i], s.py[g * n + i],
                      s.pz[g * n + i], qx, qy, qz);
            s.px[g * n + i] = qx;
            s.py[g * n + i] = qy;
            s.pz[g * n + i] = qz;
            ++wk.rot;
            s.minc[g * n + i] = min_dist_sq(p.pocket, qx, qy, qz, wk);
          }
        }
        for (int g = threadIdx.x; g < Gc; g += BT) s.cur[g] = s.best_s[g];
        __syncthreads();
      }
    }
    // Per-chain results in rank order.
    for (int g = threadIdx.x; g < Gc; g += BT) {
      const int e = l * slots + g0 + g;
      s.fin[g0 + g] = s.cur[g];
      p.out_final[e] = s.cur[g];  // rank-order staging, permuted below
      p.out_evals[e] = s.evals[g];
      p.out_checks[e] = s.checks[g];
    }
    if (p.stage_pose != nullptr) {
      for (int t = threadIdx.x; t < Gc * n; t += BT) {
        const int g = t / n, i = t - g * n;
        double* dst = p.stage_pose + 3 * (static_cast<size_t>(slots) * m.atom_off +
                                          static_cast<size_t>(g0 + g) * n + i);
        dst[0] = s.px[g * n + i];
        dst[1] = s.py[g * n + i];
        dst[2] = s.pz[g * n + i];
      }
    }
    __syncthreads();
  }

  // (E7) final order: (final score desc, seed rank asc).  Each rank's
  // destination is the number of ranks that precede it (K <= BT: one rank
  // per thread).
  const int e = threadIdx.x;
  long long ev = 0, ck = 0;
  int pos = 0;
  if (e < K) {
    const double fe = s.fin[e];
    for (int e2 = 0; e2 < K; ++e2) pos += precede(s.fin[e2], e2, fe, e) ? 1 : 0;
    ev = p.out_evals[l * slots + e];
    ck = p.out_checks[l * slots + e];
  }
  __syncthreads();
  long long scored = 0;
  if (e < K) {
    const int d = l * slots + pos;
    p.out_final[d] = s.fin[e];
    p.out_evals[d] = ev;
    p.out_checks[d] = ck;
    p.out_rank[d] = e;
    p.out_orient[d] = p.rigid ? p.orient_idx[p.seed_slot[l * slots + e]] : -1;
    p.out_rigid[d] = p.seed_score[l * slots + e];
    if (p.out_pose != nullptr) {
      const size_t src = 3 * (static_cast<size_t>(slots) * m.atom_off + static_cast<size_t>(e) * n);
      const size_t dd = 3 * (static_cast<size_t>(slots) * m.atom_off + static_cast<size_t>(pos) * n);
      for (int i = 0; i < 3 * n; ++i) p.out_pose[dd + i] = p.stage_pose[src + i];
    }
    scored = ev;
  }
  // poses scored (E8) = rigid orientations + sum of evaluations.
  typedef unsigned long long ull;
  __shared__ ull total;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  atomicAdd(&total, static_cast<ull>(scored));
  __syncthreads();
  if (threadIdx.x == 0) {
    p.poses_scored[l] = static_cast<long long>(total) + (p.rigid ? p.n_orient : 0);
    if (!p.rigid) p.k_eff[l] = 1;
  }
  publish(wk, p.counters, 8);
}

// --------------------------------------------------------------------------
// overlap_score for arbitrary poses: one thread per pose.
// --------------------------------------------------------------------------
__global__ void score_poses_kernel(PocketView pk, const double* xyz, int n_atoms, int n_poses,
                                   double* out) {
  const int pose = blockIdx.x * blockDim.x + threadIdx.x;
  if (pose >= n_poses) return;
  const double* q = xyz + static_cast<size_t>(3) * n_atoms * pose;
  Work wk;
  double sum = 0.0;
  for (int i = 0; i < n_atoms; ++i)
    sum = dadd(sum, fmax(kMinDistanceSq, min_dist_sq(pk, q[3 * i], q[3 * i + 1], q[3 * i + 2], wk)));
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

__device__ int voxel_list(const double* pts, int P, const VoxelGrid& g, int v, int* cand) {
  const int iz = v % g.dim_z;
  const int iy = (v / g.dim_z) % g.dim_y;
  const int ix = v / (g.dim_z * g.dim_y);
  const double bl[3] = {g.lo_x + ix * g.h - kVoxEps, g.lo_y + iy * g.h - kVoxEps,
                        g.lo_z + iz * g.h - kVoxEps};
  const double bh[3] = {bl[0] + g.h + 2 * kVoxEps, bl[1] + g.h + 2 * kVoxEps,
                        bl[2] + g.h + 2 * kVoxEps};
  const double cx = 0.5 * (bl[0] + bh[0]), cy = 0.5 * (bl[1] + bh[1]), cz = 0.5 * (bl[2] + bh[2]);
  // Pass 1: U (upper bound on the NN distance^2 anywhere in B) and the point
  // nearest the box centre, a strong dominator for pass 2's pre-filter.
  double U = 1e300, dc = 1e300;
  int jc = 0;
  for (int j = 0; j < P; ++j) {
    const P3 q = ldp(pts, j);
    const double fx = fmax(fabs(q.x - bl[0]), fabs(q.x - bh[0]));
    const double fy = fmax(fabs(q.y - bl[1]), fabs(q.y - bh[1]));
    const double fz = fmax(fabs(q.z - bl[2]), fabs(q.z - bh[2]));
    U = fmin(U, fx * fx + fy * fy + fz * fz);
    const double d = (q.x - cx) * (q.x - cx) + (q.y - cy) * (q.y - cy) + (q.z - cz) * (q.z - cz);
    if (d < dc) {
      dc = d;
      jc = j;
    }
  }
  const double lim = U * (1.0 + 1e-12) + kVoxMargin;
  const P3 C = ldp(pts, jc);
  // Pass 2: points that can be nearest somewhere in B and that jc does not
  // dominate (a point dominated by anything is dominated by a kept point,
  // by transitivity, so the final set does not depend on this filter).
  int k = 0;
  for (int j = 0; j < P; ++j) {
    const P3 q = ldp(pts, j);
    const double nx = fmax(0.0, fmax(bl[0] - q.x, q.x - bh[0]));
    const double ny = fmax(0.0, fmax(bl[1] - q.y, q.y - bh[1]));
    const double nz = fmax(0.0, fmax(bl[2] - q.z, q.z - bh[2]));
    if (nx * nx + ny * ny + nz * nz <= lim && !dominates(C, q, bl, bh)) {
      if (k >= kVoxMaxCand) return -1;
      cand[k++] = j;
    }
  }
  // Pass 3: full dominance pruning among the survivors.
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

__global__ void voxel_count_kernel(const double* pts, int P, VoxelGrid g, int32_t* counts) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const int nv = g.dim_x * g.dim_y * g.dim_z;
  if (v >= nv) return;
  int cand[kVoxMaxCand];
  const int k = voxel_list(pts, P, g, v, cand);
  counts[v] = k < 0 ? P : k;  // overflow: keep every point (exact, rare)
}

__global__ void voxel_fill_kernel(const double* pts, int P, VoxelGrid g, const int32_t* offsets,
                                  double* vox_pts) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const int nv = g.dim_x * g.dim_y * g.dim_z;
  if (v >= nv) return;
  int cand[kVoxMaxCand];
  const int k = voxel_list(pts, P, g, v, cand);
  double* out = vox_pts + 4 * static_cast<size_t>(offsets[v]);
  for (int a = 0; a < (k < 0 ? P : k); ++a) {
    const int j = k < 0 ? a : cand[a];
    for (int c = 0; c < 4; ++c) out[4 * a + c] = pts[4 * j + c];
  }
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

constexpr int kRigidThreads = 256;
constexpr int kFlexThreads = 256;

}  // namespace

size_t rigid_smem_bytes(const DockParams& p, int sort_slots) {
  return sizeof(double) * 3 * p.max_n + (sizeof(double) + sizeof(int)) * sort_slots;
}

size_t flex_smem_bytes(const DockParams& p) {
  const int W = (p.max_n + 63) / 64;
  return flex_smem_bytes_impl(p.max_n, W, p.chains_per_cta, p.amax, p.rigid ? p.top_k : 1);
}

int launch_rigid_topk(const DockParams& p, int sort_slots, void* stream) {
  const size_t smem = rigid_smem_bytes(p, sort_slots);
  cudaError_t e = cudaFuncSetAttribute(rigid_topk_kernel<kRigidThreads>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  rigid_topk_kernel<kRigidThreads><<<p.n_lig, kRigidThreads, smem,
                                     static_cast<cudaStream_t>(stream)>>>(p, sort_slots);
  return cudaGetLastError();
}

int launch_flex(const DockParams& p, void* stream) {
  const size_t smem = flex_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(flex_kernel<kFlexThreads>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  flex_kernel<kFlexThreads><<<p.n_lig, kFlexThreads, smem, static_cast<cudaStream_t>(stream)>>>(p);
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
  score_poses_kernel<<<(n_poses + bt - 1) / bt, bt, 0, static_cast<cudaStream_t>(stream)>>>(
      pk, xyz, n_atoms, n_poses, out);
  return cudaGetLastError();
}

int launch_voxel_count(const double* pts, int P, VoxelGrid g, int32_t* counts, void* stream) {
  const int nv = g.dim_x * g.dim_y * g.dim_z;
  const int bt = 128;
  voxel_count_kernel<<<(nv + bt - 1) / bt, bt, 0, static_cast<cudaStream_t>(stream)>>>(pts, P, g,
                                                                                      counts);
  return cudaGetLastError();
}

int launch_voxel_fill(const double* pts, int P, VoxelGrid g, const int32_t* offsets,
                      double* vox_pts, void* stream) {
  const int nv = g.dim_x * g.dim_y * g.dim_z;
  const int bt = 128;
  voxel_fill_kernel<<<(nv + bt - 1) / bt, bt, 0, static_cast<cudaStream_t>(stream)>>>(
      pts, P, g, offsets, vox_pts);
  return cudaGetLastError();
}

}  // namespace gdb200
