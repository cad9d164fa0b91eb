// (2) fragment optimisation + (3) bump check + (4) scoring + (5a) restarts,
// and (E7) the final ordering.
//
// flex_chain_kernel: one WARP per (ligand, seed rank) chain, i.e. one
// match_probes_shape call (reference kernel.hpp:205-248).  Chains are
// independent, so warps never wait for each other: a CTA is just 4 to 12
// chains (usually of the same ligand, in longest-ligand-first order) with
// private shared-memory state.  Within a chain the greedy dependency
// (rep -> rotamer -> left/right fragment, kernel.hpp:225-242) is sequential;
// each fragment search evaluates its candidate angles in batches of B:
//
//   * bump phase  -- lanes over (candidate, surviving bump pair): Rodrigues
//                    rotation (geometry.hpp:182-184) + the clash rule
//                    (geometry.hpp:199-213); warp OR-reduce per candidate;
//   * query phase -- lanes over (feasible candidate, fragment atom): rotation
//                    + exact nearest-pocket-point query (voxel index);
//   * fold phase  -- lane c folds candidate c's overlap score in atom order
//                    (geometry.hpp:143-154), reusing the committed pose's
//                    terms for atoms outside the fragment and a per-step
//                    prefix for the atoms before the first fragment atom.
//
// The bump-pair list is rebuilt once per fragment step and pruned exactly:
// a pair (i in F, j not in F) whose distance from j to the whole circle
// that atom i sweeps stays above the cutoff (1e-6 relative margin) cannot
// bump at any angle, so dropping it changes no decision.
//
// All decisions reproduce the reference: strict '>' with first-encountered
// ties (kernel.hpp:136, :169, :173, :185, :194), angle 0 = committed pose,
// feasibility_checks / evaluations counted as CandidateEvaluator does.
#include <algorithm>
#include <cassert>
#include <cstdlib>

// Inline-slot evaluation in this translation unit (device_common.cuh,
// GD_CODED_PAIRED): 1 = two slots at a time; 2 = all four with no count test.
#ifndef GD_FLEX_SLOTS
#define GD_FLEX_SLOTS 1
#endif
#ifndef GD_CODED_PAIRED
#define GD_CODED_PAIRED GD_FLEX_SLOTS
#endif
#include "device_common.cuh"

namespace gdb200 {
namespace {

// CTA shape: W chains (warps) per CTA, 24 / W CTAs per SM (the register
// budget: 65536 / (24 * 32) = 85 registers).  12-chain CTAs for batches of
// up to 6 candidates (r3e, after the live-only query batches: c1 11.55 vs
// 11.65 ms with 8; r2k had 8 ahead of 12), 4-chain CTAs for 8-candidate
// batches, whose larger v rows fit better (c2 52.4 vs 52.8 ms with 8).
#ifndef GD_FLEX_RESIDENT
#define GD_FLEX_RESIDENT 24  // warps per SM the register budget targets
#endif
// Candidates evaluated together by one warp: a template parameter (4 or 8,
// chosen per launch from the knobs, launch_flex); GD_FLEX_BATCH forces one.
#ifndef GD_FLEX_BATCH
#define GD_FLEX_BATCH 0
#endif
static_assert(GD_FLEX_BATCH == 0 || GD_FLEX_BATCH == 4 || GD_FLEX_BATCH == 6 || GD_FLEX_BATCH == 8,
              "instantiated batch sizes: 4, 6, 8");
#ifndef GD_BUMP_PAIRMAJOR
#define GD_BUMP_PAIRMAJOR 1  // bump checks pair-major (0: (candidate, pair) items)
#endif
// Debug builds (-DGD_DEBUG_BOUNDS=1, tools/sanitize_small.py) assert the
// shared-memory capacity invariants the kernels rely on.
#ifndef GD_DEBUG_BOUNDS
#define GD_DEBUG_BOUNDS 0
#endif
#if GD_DEBUG_BOUNDS
#define GD_BOUND(cond) assert(cond)
#else
#define GD_BOUND(cond) ((void)0)
#endif
#ifndef GD_PAIRMAJOR_MIN
#define GD_PAIRMAJOR_MIN 16  // surviving pairs from which bump checks go pair-major (r2l: 16
                             // beats 32 by 0.3-0.5% on c1/c2; 8 and 1 lose)
#endif
#ifndef GD_FOLD_UNROLL
#define GD_FOLD_UNROLL 4
#endif
constexpr int kFoldUnroll = GD_FOLD_UNROLL;
#ifndef GD_BUMP_SHARE
#define GD_BUMP_SHARE 1      // pair-major: share found bumps across the warp per pair chunk
#endif
#ifndef GD_AXIS_SMEM
#define GD_AXIS_SMEM 1       // the step's rotation axis read from the warp's shared slot
#endif
#ifndef GD_META_RELOAD
#define GD_META_RELOAD 0     // 1: ligand descriptor fields re-read from global when used (r2b's
                             // win; after r2h's query change 0 is 0.4% faster)
#endif
#ifndef GD_PHASE_CLOCKS
#define GD_PHASE_CLOCKS 0    // 1: per-phase clock64 attribution (gd_phase_clocks)
#endif
#ifndef GD_FIXED_POINT
#define GD_FIXED_POINT 1     // chains with several restarts replay the counts of steps past
                             // their fixed point instead of searching again
#endif
#ifndef GD_PREF_PACK
#define GD_PREF_PACK 0       // 1: prefilter's per-atom (axial, radial^2, radius) as one float4 record
                             // (two 128-bit loads per pair test instead of six 32-bit): slower,
                             // c1 flex 10.82 vs 10.57 ms, c2 38.7 vs 37.7 (r3j)
#endif
#ifndef GD_COMMIT_REUSE
#define GD_COMMIT_REUSE 1    // commits take the winner's terms from v when its batch was the search's last
#endif
#ifndef GD_FLEX_WARPS6
#define GD_FLEX_WARPS6 12    // chains per CTA for batches of up to 6 candidates (r3e: c1 flex
                             // 11.55 ms vs 11.65 at 8, 12.44 at 4)
#endif
#ifndef GD_FLEX_WARPS8
#define GD_FLEX_WARPS8 4     // chains per CTA for 8-candidate batches
#endif
template <int B>
constexpr int warps_for() {
  return B == 8 ? GD_FLEX_WARPS8 : GD_FLEX_WARPS6;
}
constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ __forceinline__ size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
// Row stride (doubles) of the candidate-term table v.  GD_V_PAD=1 makes it
// odd, so the fold's lanes -- one per candidate, all at the same atom -- hit
// distinct banks (stride n puts candidates 0, 2, 4 of an n = 40 ligand on
// the same ones); measured neutral (c1 flex 11.03 vs 11.06 ms, and 11.06 vs
// 10.95 on top of the SoA pose table), so rows stay unpadded.
#ifndef GD_V_PAD
#define GD_V_PAD 0
#endif
__host__ __device__ __forceinline__ int vrow(int n) { return GD_V_PAD ? (n | 1) : n; }

template <int B>
__host__ __device__ __forceinline__ size_t warp_bytes(int n, int W, int max_pairs) {
  return a16(8ull * n) + a16(8ull * n * W) + 4 * a16(8ull * n) + a16(8ull * B * vrow(n)) +
         a16(2ull * max_pairs) + a16(n) + a16(32) + a16(16) + a16(sizeof(Axis)) + a16(8);
}

// One atom of a chain's committed pose and its overlap term max(1e-12,
// min_j d^2): 32 bytes, two 128-bit shared loads from one address.
struct __align__(16) PT {
  double x, y, z, t;
};

// The chain's pose table in shared memory.  Lanes mostly read consecutive
// atoms, and 32-byte records read with 128-bit loads put atoms i and i + 4
// on the same banks (a quarter warp's eight 16-byte chunks must fall in the
// eight distinct 16-byte bank groups): ncu counted 45-65% excess wavefronts
// on these loads with the shared-memory pipe at 50% of its peak (r3f).
// GD_PT_LAYOUT 2 keeps x, y, z and t in four arrays (64-bit loads,
// conflict-free for consecutive atoms, an unused t is never loaded): c1 flex
// 11.06 -> 10.95 ms, c2 39.3 -> 38.6 (r3h).  1 swaps the (x, y) and (z, t)
// halves of every second group of four atoms so eight consecutive atoms
// cover all eight bank groups (11.15 ms: the address arithmetic costs more
// than the conflicts); 0 is the plain record array.
#ifndef GD_PT_LAYOUT
#define GD_PT_LAYOUT 2
#endif
struct Pose {
  double* b;
  int n;
  __device__ __forceinline__ PT get(int i) const {
#if GD_PT_LAYOUT == 2
    return PT{b[i], b[n + i], b[2 * n + i], b[3 * n + i]};
#elif GD_PT_LAYOUT == 1
    const double2* c = reinterpret_cast<const double2*>(b);
    const int h = (i >> 2) & 1;
    const double2 xy = c[2 * i + h], zt = c[2 * i + 1 - h];
    return PT{xy.x, xy.y, zt.x, zt.y};
#else
    return reinterpret_cast<const PT*>(b)[i];
#endif
  }
  __device__ __forceinline__ double t(int i) const {
#if GD_PT_LAYOUT == 2
    return b[3 * n + i];
#elif GD_PT_LAYOUT == 1
    return b[4 * i + 3 - 2 * ((i >> 2) & 1)];
#else
    return b[4 * i + 3];
#endif
  }
  __device__ __forceinline__ void set(int i, const PT& v) const {
#if GD_PT_LAYOUT == 2
    b[i] = v.x;
    b[n + i] = v.y;
    b[2 * n + i] = v.z;
    b[3 * n + i] = v.t;
#elif GD_PT_LAYOUT == 1
    double2* c = reinterpret_cast<double2*>(b);
    const int h = (i >> 2) & 1;
    c[2 * i + h] = make_double2(v.x, v.y);
    c[2 * i + 1 - h] = make_double2(v.z, v.t);
#else
    reinterpret_cast<PT*>(b)[i] = v;
#endif
  }
};

struct WarpMem {
  double* radius;        // [n]
  uint64_t* far;         // [n*W]  bit j of row i: capped graph distance >= 4
  Pose pt;               // [n]    committed pose + terms of the chain
  double* v;             // [B*n] candidate terms of fragment atoms
  uint16_t* pairs;       // [max_pairs] surviving bump pairs: F-slot | j << 8
  uint8_t* fidx;         // [n] fragment atoms, ascending
  uint64_t* fm;          // [4] fragment membership bits
  long long* tally;      // [2] the chain's evaluations, feasibility checks (lane 0)
  Axis* ax;              // [1] the step's rotation axis (GD_AXIS_SMEM)
  uint8_t* lidx;         // [8] the batch's live candidates, ascending (GD_QUERY_LIVE)
};

template <int B>
__device__ WarpMem carve(unsigned char* base, int n, int W, int max_pairs) {
  WarpMem s;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    unsigned char* q = base + o;
    o += a16(bytes);
    return q;
  };
  s.radius = reinterpret_cast<double*>(take(8ull * n));
  s.far = reinterpret_cast<uint64_t*>(take(8ull * n * W));
  s.pt = Pose{reinterpret_cast<double*>(take(32ull * n)), n};
  s.v = reinterpret_cast<double*>(take(8ull * B * vrow(n)));
  s.pairs = reinterpret_cast<uint16_t*>(take(2ull * max_pairs));
  s.fidx = reinterpret_cast<uint8_t*>(take(n));
  s.fm = reinterpret_cast<uint64_t*>(take(32));
  s.tally = reinterpret_cast<long long*>(take(16));
  s.ax = reinterpret_cast<Axis*>(take(sizeof(Axis)));
  s.lidx = reinterpret_cast<uint8_t*>(take(8));
  GD_BOUND(o <= warp_bytes<B>(n, W, max_pairs));
  return s;
}

__device__ __forceinline__ bool in_frag(const uint64_t* fm, int i) {
  return (fm[i >> 6] >> (i & 63)) & 1ull;
}

// floor(t / d) for 0 <= t < 2^16, 1 <= d <= 256 via an fp32 reciprocal:
// (2t+1)/(2d) is never within 1/(2d) >= 2e-3 of an integer, far beyond the
// ~1e-4 fp32 error at these magnitudes, so truncation is exact.
__device__ __forceinline__ int qdiv(int t, float rcp) {
  return static_cast<int>((static_cast<float>(t) + 0.5f) * rcp);
}

// Per-phase SM-clock attribution of a chain (diagnostic builds only; the
// disabled form compiles to nothing).
enum Phase { kPhInit, kPhSetup, kPhPrefilter, kPhPrefill, kPhBump, kPhQuery, kPhFold, kPhDecide,
             kPhCommit, kPhases };
template <bool On>
struct Clocks {
  long long last;
  unsigned long long acc[kPhases];
  __device__ Clocks() {
    if constexpr (On) {
      last = clock64();
      for (int k = 0; k < kPhases; ++k) acc[k] = 0;
    }
  }
  __device__ __forceinline__ void mark(int k) {
    if constexpr (On) {
      const long long t = clock64();
      acc[k] += static_cast<unsigned long long>(t - last);
      last = t;
    }
  }
  __device__ void publish(unsigned long long* c, int lane) const {
    if constexpr (On) {
      if (c != nullptr && lane == 0)
        for (int k = 0; k < kPhases; ++k) atomicAdd(c + kPhaseBase + k, acc[k]);
    }
  }
};

// One bump-check item t of a batch: candidate c = t / np against surviving
// pair t % np (Rodrigues rotation of the moving atom, geometry.hpp:182-184,
// then the clash rule, geometry.hpp:199-213).  Candidates already known to
// bump (or the angle-0 candidate, always feasible) are skipped.
template <bool On>
__device__ __forceinline__ void bump_item(const WarpMem& s, const DockParams& p, const Axis& X, int t,
                                          float rnp, int np, int a0, int da, unsigned skip,
                                          unsigned& bl, Work<On>& wk) {
  const int c = qdiv(t, rnp);
  if (((bl | skip) >> c) & 1u) return;
  const int pr = s.pairs[t - c * np];
  const int i = pr & 0xff, j = pr >> 8;
  const int a = a0 + c * da;
  const double cs = __ldg(p.cos_deg + a), sn = __ldg(p.sin_deg + a);
  double qx, qy, qz;
  const PT ai = s.pt.get(i), aj = s.pt.get(j);
  rodrigues(X, cs, sn, dsub(1.0, cs), ai.x, ai.y, ai.z, qx, qy, qz);
  wk.add(kRot, 1);
  wk.add(kBump, 1);
  const double cut = dmul(kBumpScale, dadd(s.radius[i], s.radius[j]));
  if (dist_sq(qx, qy, qz, aj.x, aj.y, aj.z) < dmul(cut, cut)) bl |= 1u << c;
}

// Query phase: lanes over (live candidate, fragment atom), two items per
// lane per iteration (t, t + 32) so both nearest-point lookups are in flight;
// candidate c's term of atom i lands in v[c * n + i].
#ifndef GD_QUERY_LIVE
#define GD_QUERY_LIVE 1      // query items over live candidates only, via a byte table (r3e: c1 flex
                             // 12.22 -> 11.85 ms, c2 58.2 -> 56.6; the n-th-set-bit form lost at r2)
#endif
#ifndef GD_QUERY_MLP
#define GD_QUERY_MLP 1       // lookups in flight per lane in the query phase (1 or 2; r2h: 1 wins, c1 flex 13.63 -> 12.36 ms)
#endif
template <bool On>
__device__ __forceinline__ void query_phase(const WarpMem& s, const DockParams& p, const Axis& X,
                                            int n, int nf, unsigned live, int a0, int da, int nb,
                                            int lane, Work<On>& wk) {
  const int tq = nb * nf;
  const float rnf = 1.0f / static_cast<float>(nf);
#if GD_QUERY_LIVE
  // Items over the live candidates only (a bumped candidate's items would
  // idle their lanes): the batch's live candidates in a byte table.
  const int nl = __popc(live);
  if (lane < nb && ((live >> lane) & 1u)) s.lidx[__popc(live & ((1u << lane) - 1u))] = static_cast<uint8_t>(lane);
  __syncwarp();
  for (int t = lane; t < nl * nf; t += 32) {
    const int cl = qdiv(t, rnf);
    const int c = s.lidx[cl];
    const int i = s.fidx[t - cl * nf];
    const int ac = a0 + c * da;
    const double cs = __ldg(p.cos_deg + ac), sn = __ldg(p.sin_deg + ac);
    double x, y, z;
    const PT q = s.pt.get(i);
    rodrigues(X, cs, sn, dsub(1.0, cs), q.x, q.y, q.z, x, y, z);
    wk.add(kRot, 1);
    s.v[c * vrow(n) + i] = fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk));
  }
  return;
#endif
#if GD_QUERY_MLP == 1
  for (int t = lane; t < tq; t += 32) {
    const int c = qdiv(t, rnf);
    if (!((live >> c) & 1u)) continue;
    const int i = s.fidx[t - c * nf];
    const int ac = a0 + c * da;
    const double cs = __ldg(p.cos_deg + ac), sn = __ldg(p.sin_deg + ac);
    double x, y, z;
    const PT q = s.pt.get(i);
    rodrigues(X, cs, sn, dsub(1.0, cs), q.x, q.y, q.z, x, y, z);
    wk.add(kRot, 1);
    s.v[c * vrow(n) + i] = fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk));
  }
  return;
#endif
  for (int t = lane; t < tq; t += 64) {
    const int c0 = qdiv(t, rnf);
    const int t1 = t + 32 < tq ? t + 32 : t;
    const int c1 = qdiv(t1, rnf);
    const bool l0 = (live >> c0) & 1u, l1 = t1 != t && ((live >> c1) & 1u);
    if (!l0 && !l1) continue;
    const int i0 = s.fidx[t - c0 * nf], i1 = s.fidx[t1 - c1 * nf];
    const int a0c = a0 + c0 * da, a1c = a0 + c1 * da;
    const double cs0 = __ldg(p.cos_deg + a0c), sn0 = __ldg(p.sin_deg + a0c);
    const double cs1 = __ldg(p.cos_deg + a1c), sn1 = __ldg(p.sin_deg + a1c);
    double x0, y0, z0, x1, y1, z1, m0, m1;
    const PT q0 = s.pt.get(i0), q1 = s.pt.get(i1);
    rodrigues(X, cs0, sn0, dsub(1.0, cs0), q0.x, q0.y, q0.z, x0, y0, z0);
    rodrigues(X, cs1, sn1, dsub(1.0, cs1), q1.x, q1.y, q1.z, x1, y1, z1);
    wk.add(kRot, 2);
    min_dist_sq2(p.pocket, x0, y0, z0, x1, y1, z1, m0, m1, wk);
    if (l0) s.v[c0 * vrow(n) + i0] = fmax(kMinDistanceSq, m0);
    if (l1) s.v[c1 * vrow(n) + i1] = fmax(kMinDistanceSq, m1);
  }
}

// Evaluates candidates angle(c) = a0 + c*da, c < nb, of the current fragment
// (CandidateEvaluator::evaluate, kernel.hpp:100-112).  Returns, in lane c,
// candidate c's overlap score (cur for angle 0), and warp-uniformly the
// mask of candidates that bumped.
template <bool On, class CK>
__device__ void eval_batch(const WarpMem& s, const DockParams& p, const Axis& X, int n, int nf,
                           int np, int first, double pre, double cur, int a0, int da, int nb,
                           int lane, double& score_out, unsigned& bumped_out, Work<On>& wk,
                           CK& ck) {
  ck.mark(kPhDecide);
  const unsigned zero = (a0 == 0) ? 1u : 0u;  // only c = 0 can be angle 0
  unsigned bl = 0;
  // Pair-major when there are at least GD_PAIRMAJOR_MIN pairs and the batch
  // is at most 6 candidates (measured: c1 16.57 vs 16.84 ms; at 8 candidates the serial
  // per-lane candidate loop loses, c2 76.3 vs 74.1): lane per surviving pair, the
  // angle-independent part of the moving atom's rotation once, then every
  // candidate angle (cos/sin from the candidate's lane); same expressions as
  // rodrigues, so the same bits.  Fewer pairs: lanes over (candidate, pair)
  // items, so candidates share the warp instead of leaving lanes idle.
  if (GD_BUMP_PAIRMAJOR && np >= GD_PAIRMAJOR_MIN && nb <= 6) {
    const int ac = a0 + min(lane, nb - 1) * da;
    const double cs_l = __ldg(p.cos_deg + ac), sn_l = __ldg(p.sin_deg + ac);
    for (int t0 = 0; t0 < np; t0 += 32) {
      const int t = t0 + lane;
      const bool act = t < np;
      Arm r{};
      PT aj{};
      double cut2 = 0.0;
      if (act) {
        const int pr = s.pairs[t];
        const int i = pr & 0xff, j = pr >> 8;
        const PT ai = s.pt.get(i);
        aj = s.pt.get(j);
        r = arm_of(X, ai.x, ai.y, ai.z);
        const double cut = dmul(kBumpScale, dadd(s.radius[i], s.radius[j]));
        cut2 = dmul(cut, cut);
      }
      for (int c = 0; c < nb; ++c) {
        const double cs = __shfl_sync(kFull, cs_l, c), sn = __shfl_sync(kFull, sn_l, c);
        if (!act || (((bl | zero) >> c) & 1u)) continue;
        double qx, qy, qz;
        turn(X, r, cs, sn, dsub(1.0, cs), qx, qy, qz);
        wk.add(kRot, 1);
        wk.add(kBump, 1);
        if (dist_sq(qx, qy, qz, aj.x, aj.y, aj.z) < cut2) bl |= 1u << c;
      }
      if (GD_BUMP_SHARE) {
        bl = __reduce_or_sync(kFull, bl);  // later pairs skip known bumps
        if ((bl | zero) == (1u << nb) - 1u) break;  // every candidate has bumped
      }
    }
  } else {
    const int total = nb * np;
    const float rnp = 1.0f / static_cast<float>(max(np, 1));
    for (int t = lane; t < total; t += 32) bump_item(s, p, X, t, rnp, np, a0, da, zero, bl, wk);
  }
  const unsigned bumped = __reduce_or_sync(kFull, bl);
  const unsigned live = ((1u << nb) - 1u) & ~bumped & ~zero;
  ck.mark(kPhBump);
  query_phase(s, p, X, n, nf, live, a0, da, nb, lane, wk);
  __syncwarp();
  ck.mark(kPhQuery);
  // Fold phase: lane c, atom order.
  double score = cur;
  if (lane < nb && ((live >> lane) & 1u)) {
    double sum = pre;
    const double* vc = s.v + lane * vrow(n);
#pragma unroll kFoldUnroll
    for (int i = first; i < n; ++i) sum = dadd(sum, vc[i]);
    score = __ddiv_rn(static_cast<double>(n), sum);
    wk.add(kTerms, n);
    wk.add(kEvals, 1);
  }
  __syncwarp();
  ck.mark(kPhFold);
  score_out = score;
  bumped_out = bumped;
}

// A batch's contribution to the running argmax under the reference's
// sequential rule (strict '>' against the running best, first-encountered
// ties; kernel.hpp:136, :169, :185): the scan ends on the batch maximum M
// over the feasible candidates, first reached at the lowest candidate
// holding M, and it replaces the best iff M > best.  Lane c < nb holds
// candidate c's score; returns M warp-uniformly and that candidate in
// `first_c` (-1 when nothing is feasible).  B <= 8: one 8-lane butterfly.
__device__ __forceinline__ double batch_max(double sc, unsigned bumped, int nb, int lane,
                                            int& first_c) {
  const bool feas = lane < nb && !((bumped >> lane) & 1u);
  const double v = feas ? sc : -kInfinity;
  double m = v;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  m = __shfl_sync(kFull, m, 0);
  first_c = __ffs(__ballot_sync(kFull, feas && v == m)) - 1;
  return m;
}

template <bool On>
__device__ void publish_warp(const Work<On>& w, unsigned long long* c, int base, int lane) {
  if constexpr (On) {
    if (c == nullptr) return;
#pragma unroll
    for (int k = 0; k < kWorkKinds; ++k) {
      const unsigned s = __reduce_add_sync(kFull, w.c[k]);
      if (lane == 0) atomicAdd(c + base + k, static_cast<unsigned long long>(s));
    }
  }
}

// Fragment step setup, shared by the search and the profile kernels: the
// fragment mask, the rotation axis (rotate_fragment_into, geometry.hpp:
// 165-169, identical in every lane), the ascending fragment atoms, the fold
// prefix of the atoms before the first fragment atom, the surviving bump
// pairs and the per-candidate pre-fill of the non-fragment terms.  `left_np`
// carries a left step's pair count to its right step (-1: rebuild).
// Returns false on a degenerate axis.
struct StepInfo {
  Axis X;
  int nf, first, np;
  double pre;
};

template <int B, class CK>
__device__ __forceinline__ bool setup_step(const WarpMem& s, const DockParams& p, const LigMeta& m,
                                           int f, int axis, int anchor, uint64_t fm_word, int lane,
                                           int& left_np, StepInfo& st, CK& ck) {
  const int n = m.n, W = m.words;
  if (lane < W) s.fm[lane] = fm_word;  // loaded by the caller with the descriptors
  // rotate_fragment_into axis (geometry.hpp:165-169), identical in every lane.
  const PT pa = s.pt.get(axis), pb = s.pt.get(anchor);
  const double ox = pa.x, oy = pa.y, oz = pa.z;
  const double ax = dsub(pb.x, ox), ay = dsub(pb.y, oy), az = dsub(pb.z, oz);
  const double len = __dsqrt_rn(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az)));
  if (len < kMinAxisLength) return false;  // "rotate_fragment: degenerate rotation axis"
  st.X = Axis{ox, oy, oz, __ddiv_rn(ax, len), __ddiv_rn(ay, len), __ddiv_rn(az, len)};
  const Axis& X = st.X;
  __syncwarp();
  // Fragment atoms, ascending.
  int nf = 0;
  for (int b = 0; b < n; b += 32) {
    const int i = b + lane;
    const bool in = i < n && in_frag(s.fm, i);
    const unsigned mask = __ballot_sync(kFull, in);
    if (in) s.fidx[nf + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint8_t>(i);
    nf += __popc(mask);
  }
  __syncwarp();
  GD_BOUND(nf >= 1 && nf < n);
  const int first = s.fidx[0];
  double pre = 0.0;
  if (lane == 0) {
#pragma unroll 4
    for (int i = 0; i < first; ++i) pre = dadd(pre, s.pt.t(i));
  }
  pre = __shfl_sync(kFull, pre, 0);
  ck.mark(kPhSetup);
  // Surviving bump pairs: drop (i, j) when the circle atom i sweeps never
  // comes within the cutoff of j: dmin^2 = h^2 + (sigma - rho)^2 > cut^2,
  // tested without square roots as L = s2 + r2 + h2 - C > 0 && L^2 > 4 s2 r2.
  // Per-atom axial coordinate a = k.(p - o) and squared axis distance
  // r2 = |p - o|^2 - a^2 first, lane-parallel, in the (free) v scratch.
  // The pair list holds (moving atom | fixed atom << 8).  A rotamer's
  // right step reuses its left step's list with the roles swapped: both
  // rotate about the same bond line, the left commit rotated the left
  // atoms about that very line, and the circle test depends only on the
  // atoms' axial and radial coordinates relative to it (rotation
  // invariants).  The test itself is a conservative filter, so it runs
  // in fp32 with a wide margin; the kept pairs are decided exactly.
  int np = 0;
  if ((f & 1) && left_np >= 0) {
    np = left_np;
    for (int t = lane; t < np; t += 32) {
      const unsigned pr = s.pairs[t];
      s.pairs[t] = static_cast<uint16_t>((pr >> 8) | ((pr & 0xffu) << 8));
    }
  } else {
#if GD_PREF_PACK
    // One 16-byte record per atom (axial coordinate, squared axis distance,
    // radius): a pair test is two 128-bit shared loads instead of six 32-bit.
    float4* pa = reinterpret_cast<float4*>(s.v);
    float* rf = reinterpret_cast<float*>(pa + n) - n;  // pref follows the records (rf + n below)
    for (int i = lane; i < n; i += 32) {
      const PT q = s.pt.get(i);
      const double vx = q.x - ox, vy = q.y - oy, vz = q.z - oz;
      const double a = X.kx * vx + X.ky * vy + X.kz * vz;
      pa[i] = make_float4(static_cast<float>(a),
                          static_cast<float>(fmax(0.0, vx * vx + vy * vy + vz * vz - a * a)),
                          static_cast<float>(s.radius[i]), 0.0f);
    }
    __syncwarp();
    auto test = [&](int i, int j) {
      const float4 ai = pa[i], aj = pa[j];
      const float h = aj.x - ai.x;
      const float s2 = aj.y, r2 = ai.y;
      const float cut = 0.8f * (ai.z + aj.z);
      const float C = __fmaf_rn(cut * cut, 1.0001f, 1e-2f);
      const float Lq = (s2 + r2) + __fmaf_rn(h, h, -C);
      return !(Lq > 0.0f && Lq * Lq > 4.00004f * s2 * r2);
    };
#else
    float* axc = reinterpret_cast<float*>(s.v);
    float* rad2 = axc + n;
    float* rf = rad2 + n;
    for (int i = lane; i < n; i += 32) {
      const PT q = s.pt.get(i);
      const double vx = q.x - ox, vy = q.y - oy, vz = q.z - oz;
      const double a = X.kx * vx + X.ky * vy + X.kz * vz;
      axc[i] = static_cast<float>(a);
      rad2[i] = static_cast<float>(fmax(0.0, vx * vx + vy * vy + vz * vz - a * a));
      rf[i] = static_cast<float>(s.radius[i]);
    }
    __syncwarp();
    auto test = [&](int i, int j) {
      const float h = axc[j] - axc[i];
      const float s2 = rad2[j], r2 = rad2[i];
      const float cut = 0.8f * (rf[i] + rf[j]);
      const float C = __fmaf_rn(cut * cut, 1.0001f, 1e-2f);
      const float Lq = (s2 + r2) + __fmaf_rn(h, h, -C);
      return !(Lq > 0.0f && Lq * Lq > 4.00004f * s2 * r2);
    };
#endif
    {
      // Flattened over the actual partner pairs: per-slot partner counts and
      // a warp prefix sum give each slot its range of pair indices; slot
      // lanes then write every candidate pair in place (walking their
      // partner bits; total <= nf (n - nf) <= the pair buffer's n^2/4), and
      // the warp tests and compacts them in place (writes never pass the
      // chunk being read).
      int* pref = reinterpret_cast<int*>(rf + n);
      GD_BOUND((GD_PREF_PACK ? 16 : 12) * n + 4 * nf <= 8 * B * n);  // per-atom floats + pref fit the v scratch
      int total = 0;
      for (int b = 0; b < nf; b += 32) {
        const int sl = b + lane;
        int cnt = 0;
        if (sl < nf) {
          const int i = s.fidx[sl];
          if (W == 1) {
            cnt = __popcll(s.far[i] & ~s.fm[0]);
          } else {
            for (int w = 0; w < W; ++w) cnt += __popcll(s.far[i * W + w] & ~s.fm[w]);
          }
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, inc, o);
          if (lane >= o) inc += y;
        }
        if (sl < nf) pref[sl] = total + inc - cnt;
        total += __shfl_sync(kFull, inc, 31);
      }
      __syncwarp();
      GD_BOUND(total <= p.max_pairs);  // nf (n - nf) <= n^2 / 4
      for (int sl = lane; sl < nf; sl += 32) {
        const int i = s.fidx[sl];
        int pos = pref[sl];
        if (W == 1) {
          uint64_t m = s.far[i] & ~s.fm[0];
          while (m) {
            const int j = __ffsll(static_cast<long long>(m)) - 1;
            m &= m - 1;
            s.pairs[pos++] = static_cast<uint16_t>(i | (j << 8));
          }
        } else {
          for (int w = 0; w < W; ++w) {
            uint64_t m = s.far[i * W + w] & ~s.fm[w];
            while (m) {
              const int j = 64 * w + __ffsll(static_cast<long long>(m)) - 1;
              m &= m - 1;
              s.pairs[pos++] = static_cast<uint16_t>(i | (j << 8));
            }
          }
        }
      }
      __syncwarp();
      for (int t0 = 0; t0 < total; t0 += 32) {
        const int t = t0 + lane;
        bool keep = false;
        unsigned pr = 0;
        if (t < total) {
          pr = s.pairs[t];
          keep = test(static_cast<int>(pr & 0xffu), static_cast<int>(pr >> 8));
        }
        const unsigned mask = __ballot_sync(kFull, keep);
        __syncwarp();
        if (keep) s.pairs[np + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint16_t>(pr);
        np += __popc(mask);
      }
    }
  }
  __syncwarp();
  left_np = (f & 1) ? -1 : np;  // a left step's list serves its right step
  ck.mark(kPhPrefilter);
  // Non-fragment terms are the same for every candidate of this step:
  // pre-fill them into each candidate slot so the fold is a plain sum.
  for (int i = lane; i < n; i += 32)
    if (!in_frag(s.fm, i)) {
      const double t = s.pt.t(i);
#pragma unroll
      for (int c = 0; c < B; ++c) s.v[c * vrow(n) + i] = t;
    }
  __syncwarp();
  ck.mark(kPhPrefill);
  st.nf = nf;
  st.first = first;
  st.pre = pre;
  st.np = np;
  return true;
}

#ifndef GD_FLAT_LIVE
#define GD_FLAT_LIVE 1       // flat searches: bump-check up to 32 candidates at once, then query
                             // and fold only the live ones in batches of B
#endif
#ifndef GD_FLAT_LIVE_MINC
#define GD_FLAT_LIVE_MINC 1  // ... for searches of at least this many candidates
#endif
#ifndef GD_GROUP_PAIRMAJOR_MIN
#define GD_GROUP_PAIRMAJOR_MIN 32  // bump_group goes pair-major from this many surviving pairs (r3g, coded
                                   // records: c1 flex 10.90 ms at 32, 11.07 at 64, 11.43 at 128) ...
#endif
#ifndef GD_GROUP_PAIRMAJOR_MIN_WIDE
#define GD_GROUP_PAIRMAJOR_MIN_WIDE 24  // ... or this many for groups of more than 16 candidates
                                        // (r3e: c1 flex 11.65 ms at 64 / 12.22 at 16, c2 54.2 at 24 / 55.7 at 64)
#endif

// Bump checks of candidates angle(c) = a0 + c*da, c < nb <= 32 (check_bumps,
// geometry.hpp:199-213): the mask of those that clash.  Pair-major over the
// surviving pairs (each lane's pair rotated to every candidate angle,
// found bumps shared across the warp) or, for few pairs, lanes over
// (candidate, pair) items.
template <bool On>
__device__ __forceinline__ unsigned bump_group(const WarpMem& s, const DockParams& p, const Axis& X, int np,
                                               int a0, int da, int nb, int lane, Work<On>& wk) {
  const unsigned all = nb == 32 ? kFull : (1u << nb) - 1u;
  unsigned bl = 0;
  if (np >= (nb > 16 ? GD_GROUP_PAIRMAJOR_MIN_WIDE : GD_GROUP_PAIRMAJOR_MIN)) {
    const int ac = a0 + min(lane, nb - 1) * da;
    const double cs_l = __ldg(p.cos_deg + ac), sn_l = __ldg(p.sin_deg + ac);
    for (int t0 = 0; t0 < np; t0 += 32) {
      const int t = t0 + lane;
      const bool act = t < np;
      Arm r{};
      PT aj{};
      double cut2 = 0.0;
      if (act) {
        const int pr = s.pairs[t];
        const int i = pr & 0xff, j = pr >> 8;
        const PT ai = s.pt.get(i);
        aj = s.pt.get(j);
        r = arm_of(X, ai.x, ai.y, ai.z);
        const double cut = dmul(kBumpScale, dadd(s.radius[i], s.radius[j]));
        cut2 = dmul(cut, cut);
      }
      for (int c = 0; c < nb; ++c) {
        const double cs = __shfl_sync(kFull, cs_l, c), sn = __shfl_sync(kFull, sn_l, c);
        if (!act || ((bl >> c) & 1u)) continue;
        double qx, qy, qz;
        turn(X, r, cs, sn, dsub(1.0, cs), qx, qy, qz);
        wk.add(kRot, 1);
        wk.add(kBump, 1);
        if (dist_sq(qx, qy, qz, aj.x, aj.y, aj.z) < cut2) bl |= 1u << c;
      }
      bl = __reduce_or_sync(kFull, bl);  // later pairs skip known bumps
      if (bl == all) break;              // every candidate has bumped
    }
  } else {
    const int total = nb * np;
    const float rnp = 1.0f / static_cast<float>(max(np, 1));
    for (int t = lane; t < total; t += 32) bump_item(s, p, X, t, rnp, np, a0, da, 0u, bl, wk);
  }
  return __reduce_or_sync(kFull, bl) & all;
}

// Query phase over a batch of live candidates: slot k < nb is candidate
// s.lidx[k] (angle a0 + lidx[k]*da); its terms land in row k of v.
#ifndef GD_QUERY_PAIRS
#define GD_QUERY_PAIRS 0     // 1: a lane serves one atom for two live slots (shared rotation arm,
                             // two lookups in flight): exact, but c1 flex 13.05 vs 10.79 ms and c2
                             // 52.4 vs 38.6 (r3i) -- two queries' state per lane and a scan as long
                             // as the longer of the two candidate lists
#endif
template <bool On>
__device__ __forceinline__ void query_slots(const WarpMem& s, const DockParams& p, const Axis& X, int n,
                                            int nf, int nb, int a0, int da, int lane, Work<On>& wk) {
  const float rnf = 1.0f / static_cast<float>(nf);
#if GD_QUERY_PAIRS
  if (nb >= 2) {
    const int npair = (nb + 1) >> 1;
    for (int t = lane; t < npair * nf; t += 32) {
      const int j = qdiv(t, rnf);
      const int i = s.fidx[t - j * nf];
      const int k0 = 2 * j, k1 = min(2 * j + 1, nb - 1);
      const int ac0 = a0 + s.lidx[k0] * da, ac1 = a0 + s.lidx[k1] * da;
      const double cs0 = __ldg(p.cos_deg + ac0), sn0 = __ldg(p.sin_deg + ac0);
      const double cs1 = __ldg(p.cos_deg + ac1), sn1 = __ldg(p.sin_deg + ac1);
      const PT q = s.pt.get(i);
      const Arm r = arm_of(X, q.x, q.y, q.z);
      double x0, y0, z0, x1, y1, z1, m0, m1;
      turn(X, r, cs0, sn0, dsub(1.0, cs0), x0, y0, z0);
      turn(X, r, cs1, sn1, dsub(1.0, cs1), x1, y1, z1);
      wk.add(kRot, k1 != k0 ? 2 : 1);
      min_dist_sq2(p.pocket, x0, y0, z0, x1, y1, z1, m0, m1, wk);
      s.v[k0 * vrow(n) + i] = fmax(kMinDistanceSq, m0);
      if (k1 != k0) s.v[k1 * vrow(n) + i] = fmax(kMinDistanceSq, m1);
    }
    return;
  }
#endif
  for (int t = lane; t < nb * nf; t += 32) {
    const int k = qdiv(t, rnf);
    const int i = s.fidx[t - k * nf];
    const int ac = a0 + s.lidx[k] * da;
    const double cs = __ldg(p.cos_deg + ac), sn = __ldg(p.sin_deg + ac);
    double x, y, z;
    const PT q = s.pt.get(i);
    rodrigues(X, cs, sn, dsub(1.0, cs), q.x, q.y, q.z, x, y, z);
    wk.add(kRot, 1);
    s.v[k * vrow(n) + i] = fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk));
  }
}

// One fragment search from the committed pose, whose score is `cur`:
// optimize_fragment_flat (kernel.hpp:125-143) with `step`, or
// optimize_fragment_refined (:150-198) with high-precision step `step`, tile
// p.tile and the entry score `entry` (the reference's optional entry_score;
// the chains pass cur).  Returns the winning angle and score warp-uniformly
// and the CandidateEvaluator tallies (evaluations, feasibility checks).
template <bool On, int B, class CK>
__device__ __forceinline__ void search_fragment(const WarpMem& s, const DockParams& p, const Axis& X,
                                                int n, int nf, int np, int first, double pre,
                                                double cur, double entry, int step, bool refined,
                                                int lane, int& best_a, double& best, int& evals,
                                                int& checks, int& win_row, Work<On>& wk, CK& ck) {
  best_a = 0;
  best = cur;
  win_row = -1;  // row of v still holding the winner's terms (flat searches, GD_COMMIT_REUSE)
  if (!refined && GD_FLAT_LIVE && 360 / step - 1 >= GD_FLAT_LIVE_MINC) {
    // optimize_fragment_flat (kernel.hpp:125-143): candidates c*step,
    // c = 1..A-1, bump-checked 32 at a time, then the live ones queried and
    // folded in batches of B in angle order -- the first-encountered
    // maximum under strict '>' is the reference's choice whatever the
    // batching.  Bumped candidates cost no query lanes and no fold.
    const int A = 360 / step;
    int nfeas = 0;
    for (int g0 = 1; g0 < A; g0 += 32) {
      const int ng = min(32, A - g0);
      const int a0 = g0 * step;
      ck.mark(kPhDecide);
      unsigned live = (ng == 32 ? kFull : (1u << ng) - 1u) & ~bump_group(s, p, X, np, a0, step, ng, lane, wk);
      ck.mark(kPhBump);
      nfeas += __popc(live);
      while (live) {
        const bool mine = (live >> lane) & 1u;
        const int rank = __popc(live & ((1u << lane) - 1u));
        const unsigned take = __ballot_sync(kFull, mine && rank < B);
        if (mine && rank < B) s.lidx[rank] = static_cast<uint8_t>(lane);
        const int nb = __popc(take);
        live &= ~take;
        __syncwarp();
        query_slots(s, p, X, n, nf, nb, a0, step, lane, wk);
        __syncwarp();
        ck.mark(kPhQuery);
        double score = -kInfinity;
        if (lane < nb) {
          double sum = pre;
          const double* vc = s.v + lane * vrow(n);
#pragma unroll kFoldUnroll
          for (int i = first; i < n; ++i) sum = dadd(sum, vc[i]);
          score = __ddiv_rn(static_cast<double>(n), sum);
          wk.add(kTerms, n);
          wk.add(kEvals, 1);
        }
        __syncwarp();
        ck.mark(kPhFold);
        int c;
        const double v = batch_max(score, 0u, nb, lane, c);
        win_row = -1;  // this batch overwrote the rows of every earlier one
        if (c >= 0 && v > best) {
          best = v;
          best_a = a0 + s.lidx[c] * step;
          win_row = c;
        }
        __syncwarp();
      }
    }
    evals = 1 + nfeas;
    checks = A;
    return;
  }
  if (!refined) {
    // optimize_fragment_flat (kernel.hpp:125-143).
    const int A = 360 / step;
    int nfeas = 0;
    for (int kb = 0; kb < A - 1; kb += B) {
      const int nb = min(B, A - 1 - kb);
      const int a0 = (kb + 1) * step;
      double sc;
      unsigned bumped;
      eval_batch(s, p, X, n, nf, np, first, pre, cur, a0, step, nb, lane, sc, bumped, wk, ck);
      int c;
      const double v = batch_max(sc, bumped, nb, lane, c);
      nfeas += __popc(~bumped & ((1u << nb) - 1u));
      if (c >= 0 && v > best) {
        best = v;
        best_a = a0 + c * step;
      }
    }
    evals = 1 + nfeas;
    checks = A;
    return;
  }
  // optimize_fragment_refined (kernel.hpp:150-198).
  const int T = p.tile, tc = 360 / T;
  bool have = false;
  int wt = -1;
  double ws = 0.0;
  int nfeas = 0;
  best = 0.0;
  for (int kb = 0; kb < tc; kb += B) {
    const int nb = min(B, tc - kb);
    const int a0 = kb * T + T / 2;
    double sc;
    unsigned bumped;
    eval_batch(s, p, X, n, nf, np, first, pre, cur, a0, T, nb, lane, sc, bumped, wk, ck);
    int c;
    const double v = batch_max(sc, bumped, nb, lane, c);
    nfeas += __popc(~bumped & ((1u << nb) - 1u));
    if (c >= 0 && (!have || v > best)) {
      best = v;
      best_a = a0 + c * T;
      have = true;
    }
    if (c >= 0 && (wt < 0 || v > ws)) {
      wt = kb + c;
      ws = v;
    }
  }
  checks = tc;
  if (wt >= 0) {
    int cnt2 = 0;
    while ((cnt2 + 1) * step <= T) ++cnt2;
    for (int kb = 0; kb < cnt2; kb += B) {
      const int nb = min(B, cnt2 - kb);
      const int a0 = wt * T + kb * step;
      double sc;
      unsigned bumped;
      eval_batch(s, p, X, n, nf, np, first, pre, cur, a0, step, nb, lane, sc, bumped, wk, ck);
      int c;
      const double v = batch_max(sc, bumped, nb, lane, c);
      nfeas += __popc(~bumped & ((1u << nb) - 1u));
      if (c >= 0 && (!have || v > best)) {
        best = v;
        best_a = a0 + c * step;
        have = true;
      }
    }
    checks += cnt2;
  }
  checks += 1;  // entry-pose comparison (kernel.hpp:192-194)
  if (!have || entry > best) {
    best = entry;
    best_a = 0;
  }
  evals = nfeas;
}

template <bool On, int B, int kWarps = warps_for<B>(), bool kReplay = false>
__global__ void __launch_bounds__(kWarps * 32, GD_FLEX_RESIDENT / kWarps)
    flex_chain_kernel(DockParams p) {
  static_assert(B >= 1 && B <= 8, "batch_max reduces over an 8-lane butterfly");
  extern __shared__ __align__(16) unsigned char smem[];
  stage_tab<kCompactTU>(p.pocket);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.k_slots;
  const long long item = static_cast<long long>(blockIdx.x) * kWarps + warp;
  if (item >= static_cast<long long>(p.n_lig) * K) return;
  const int l = p.order[item / K];
  const int r = static_cast<int>(item % K);
#if GD_META_RELOAD
  const LigMeta& m = p.meta[l];
#else
  const LigMeta m = p.meta[l];
#endif
  if (m.status != 0 || m.n > kNarrowAtoms) return;  // wide ligands: flex_wide_kernel
  const int n = m.n, W = m.words;
  const WarpMem s =
      carve<B>(smem + warp * warp_bytes<B>(p.max_n, (p.max_n + 63) / 64, p.max_pairs), n, W,
               p.max_pairs);
  const size_t e = static_cast<size_t>(l) * p.top_k + r;
  Work<On> wk;
  Clocks<On && GD_PHASE_CLOCKS> ck;

  for (int i = lane; i < n; i += 32) s.radius[i] = __ldg(p.radii + m.atom_off + i);
  for (int i = lane; i < n * W; i += 32) s.far[i] = __ldg(p.far_mask + m.far_off + i);
  // Chain start: the rigid seed pose (E3) or the given pose.
  double R[9];
  if (p.rigid) {
    const int o = p.seed_slot[e];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(p.orient_R + 9 * o + k);
  }
  for (int i = lane; i < n; i += 32) {
    const double* q = p.xyz + 3 * (m.atom_off + i);
    double x = q[0], y = q[1], z = q[2];
    if (p.rigid) {
      rigid_apply(R, p.cx, p.cy, p.cz, dsub(x, p.cx), dsub(y, p.cy), dsub(z, p.cz), x, y, z);
      wk.add(kXform, 1);
    }
    s.pt.set(i, PT{x, y, z, fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk))});
  }
  __syncwarp();
  // match_probes_shape prologue (kernel.hpp:215-218).
  double cur = 0.0;
  if (lane == 0) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum = dadd(sum, s.pt.t(i));
    cur = __ddiv_rn(static_cast<double>(n), sum);
  }
  cur = __shfl_sync(kFull, cur, 0);
  if (!p.rigid && lane == 0) p.seed_score[e] = cur;
  // The chain's evaluation / feasibility-check counts live in the warp's
  // shared slot (lane 0), not in registers the batch loop needs.
  if (lane == 0) s.tally[0] = s.tally[1] = 1;
  auto tally = [&](int ev, int ck) {
    if (lane == 0) {
      s.tally[0] += ev;
      s.tally[1] += ck;
    }
  };
  int left_np = -1;  // bump-pair count of the preceding left step, -1 if none
  ck.mark(kPhInit);

  // Fixed point (reps > 1): a step is a pure function of the committed pose,
  // so once nfrag consecutive steps -- every fragment once -- have kept
  // angle 0, each later step repeats its last outcome: angle 0 again and the
  // same CandidateEvaluator counts.  Those steps only replay their counts
  // (lane f keeps step f's last evaluations << 16 | checks; chains of more
  // than 32 fragments run every step).  On config 2 (3 restarts) a quarter
  // of the steps are replays.  kReplay instantiations serve launches with
  // several restarts; single-restart launches carry none of it.
  const bool ff = kReplay && m.nfrag <= 32;
  int streak = 0;
  unsigned hist = 0;
  for (int rep = 0; rep < p.reps; ++rep) {
    for (int f = 0; f < m.nfrag; ++f) {
      if (kReplay && ff && streak >= m.nfrag) {
        const unsigned h = __shfl_sync(kFull, hist, f);
        tally(static_cast<int>(h >> 16), static_cast<int>(h & 0xffffu));
        continue;
      }
      const int fo = m.frag_off + f;
      // The step's descriptors and fragment-mask words, all in flight at once.
      const int axis = __ldg(p.frag_axis + fo), anchor = __ldg(p.frag_anchor + fo);
      const double rel = __ldg(p.frag_rel + fo);
      const uint64_t fm_word = lane < W ? __ldg(p.frag_mask + m.fmask_off + f * W + lane) : 0ull;
      // Dispatch (kernel.hpp:229-239).
      const bool low = rel <= p.threshold;
      const bool refined = !low && p.refine;
      const int step = low ? p.lp : p.hp;
      const int A = 360 / step;
      if (!refined && A == 1) {  // step 360: only the committed pose
        tally(1, 1);
        left_np = -1;
        if (kReplay) {
          if (lane == f) hist = (1u << 16) | 1u;
          ++streak;
        }
        continue;
      }
      StepInfo st;
      if (!setup_step<B>(s, p, m, f, axis, anchor, fm_word, lane, left_np, st, ck)) {
        if (lane == 0) p.status[l] = 3;  // "rotate_fragment: degenerate rotation axis"
        return;
      }
#if GD_AXIS_SMEM
      if (lane == 0) *s.ax = st.X;
      __syncwarp();
      const Axis& X = *s.ax;
#else
      const Axis& X = st.X;
#endif
      const int nf = st.nf, first = st.first, np = st.np;
      const double pre = st.pre;

      int best_a = 0;
      double best = cur;
      int evals = 0, checks = 0, win_row = -1;
      search_fragment<On, B>(s, p, X, n, nf, np, first, pre, cur, cur, step, refined, lane, best_a,
                             best, evals, checks, win_row, wk, ck);
      tally(evals, checks);
      if (kReplay) {
        if (lane == f) hist = (static_cast<unsigned>(evals) << 16) | static_cast<unsigned>(checks);
        streak = best_a != 0 ? 0 : streak + 1;
      }
      ck.mark(kPhDecide);
      // commit_angle (kernel.hpp:115-117): a fresh rotation of the entry pose,
      // bit-identical to the scored candidate; refresh the fragment's terms.
      if (best_a != 0) {
        const double cs = __ldg(p.cos_deg + best_a), sn = __ldg(p.sin_deg + best_a);
        const double omc = dsub(1.0, cs);
        for (int sl = lane; sl < nf; sl += 32) {
          const int i = s.fidx[sl];
          double qx, qy, qz;
          const PT q = s.pt.get(i);
          rodrigues(X, cs, sn, omc, q.x, q.y, q.z, qx, qy, qz);
          wk.add(kRot, 1);
          // The winner's terms are still in its row of v when it was scored
          // in the search's last batch: the same rotation, the same query,
          // so the same bits -- no second lookup.
          const double t = (GD_COMMIT_REUSE && win_row >= 0)
                               ? s.v[win_row * vrow(n) + i]
                               : fmax(kMinDistanceSq, min_dist_sq(p.pocket, qx, qy, qz, wk));
          s.pt.set(i, PT{qx, qy, qz, t});
        }
      }
      __syncwarp();
      ck.mark(kPhCommit);
      cur = best;
    }
  }
  if (lane == 0) {
    p.st_final[e] = cur;
    p.st_evals[e] = s.tally[0];
    p.st_checks[e] = s.tally[1];
  }
  // Final pose staging.  Top-1-only callers (top_best set) stage a chain's
  // pose only if its score is >= every score the ligand's finished chains
  // have published (scores are positive doubles, so their bit patterns
  // order as integers): the E7 winner always stages (ties included), most
  // chains skip the write.
  bool stage = p.stage_pose != nullptr;
  if (stage && p.top_best != nullptr) {
    unsigned long long old = 0;
    if (lane == 0) old = atomicMax(p.top_best + l, static_cast<unsigned long long>(__double_as_longlong(cur)));
    stage = __longlong_as_double(static_cast<long long>(__shfl_sync(kFull, old, 0))) <= cur;
  }
  if (stage) {
    double* dst = p.stage_pose + 3 * (static_cast<size_t>(p.top_k) * m.atom_off + static_cast<size_t>(r) * n);
    for (int i = lane; i < n; i += 32) {
      const PT q = s.pt.get(i);
      dst[3 * i] = q.x;
      dst[3 * i + 1] = q.y;
      dst[3 * i + 2] = q.z;
    }
  }
  publish_warp(wk, p.counters, 8, lane);
  ck.publish(p.counters, lane);
}

// Wide ligands (more than kNarrowAtoms atoms): one CTA per (ligand, seed
// rank) chain, the chain's state -- committed pose and terms, the candidate
// pose, the candidate terms: 8 doubles per atom -- in HBM, far masks and
// fragment masks read from HBM, candidates evaluated one after another
// exactly as CandidateEvaluator does (kernel.hpp:100-112): rotate the
// fragment, check_bumps over every (fragment atom, far partner) pair, then
// the overlap terms of the rotated atoms and an atom-order fold by thread 0.
// Same expressions and decisions as flex_chain_kernel, so the same bits; no
// pair prefilter and no batching, because such ligands are rare and their
// chains are long enough to fill the GPU with a CTA each.
constexpr int kWideThreads = 256;
template <bool On>
__global__ void __launch_bounds__(kWideThreads) flex_wide_kernel(DockParams p) {
  stage_tab<kCompactTU>(p.pocket);
  __shared__ double s_val;
  __shared__ int s_stage;
  const int K = p.k_slots;
  const int b = blockIdx.x / K, r = blockIdx.x % K;
  const int l = p.wide_list[b];
  const LigMeta m = p.meta[l];
  if (m.status != 0) return;
  const int n = m.n, W = m.words, tid = threadIdx.x;
  const size_t e = static_cast<size_t>(l) * p.top_k + r;
  double* px = p.wide_scratch + 8 * (static_cast<size_t>(p.wide_off[b]) * K + static_cast<size_t>(r) * n);
  double *py = px + n, *pz = py + n, *pt = pz + n;  // committed pose and terms
  double *qx = pt + n, *qy = qx + n, *qz = qy + n;  // candidate pose (fragment atoms)
  double* v = qz + n;                               // candidate terms
  const double* rad = p.radii + m.atom_off;
  const uint64_t* far = p.far_mask + m.far_off;
  Work<On> wk;

  // Chain start: the rigid seed pose (E3) or the given pose.
  double R[9];
  if (p.rigid) {
    const int o = p.seed_slot[e];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(p.orient_R + 9 * o + k);
  }
  for (int i = tid; i < n; i += kWideThreads) {
    const double* q = p.xyz + 3 * (static_cast<size_t>(m.atom_off) + i);
    double x = q[0], y = q[1], z = q[2];
    if (p.rigid) {
      rigid_apply(R, p.cx, p.cy, p.cz, dsub(x, p.cx), dsub(y, p.cy), dsub(z, p.cz), x, y, z);
      wk.add(kXform, 1);
    }
    px[i] = x;
    py[i] = y;
    pz[i] = z;
    pt[i] = fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk));
  }
  __syncthreads();
  // overlap_score fold (geometry.hpp:143-154) of `terms`, broadcast.
  auto fold = [&](const double* terms) {
    if (tid == 0) {
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum = dadd(sum, terms[i]);
      s_val = __ddiv_rn(static_cast<double>(n), sum);
    }
    __syncthreads();
    const double sc = s_val;
    __syncthreads();
    return sc;
  };
  double cur = fold(pt);
  if (!p.rigid && tid == 0) p.seed_score[e] = cur;
  long long evals = 1, checks = 1;  // uniform across the CTA

  for (int rep = 0; rep < p.reps; ++rep) {
    for (int f = 0; f < m.nfrag; ++f) {
      const int fo = m.frag_off + f;
      const int axis = __ldg(p.frag_axis + fo), anchor = __ldg(p.frag_anchor + fo);
      const double rel = __ldg(p.frag_rel + fo);
      const uint64_t* fm = p.frag_mask + m.fmask_off + static_cast<size_t>(f) * W;
      const bool low = rel <= p.threshold;
      const bool refined = !low && p.refine;
      const int step = low ? p.lp : p.hp;
      const int A = 360 / step;
      if (!refined && A == 1) {  // step 360: only the committed pose
        evals += 1;
        checks += 1;
        continue;
      }
      // rotate_fragment_into axis (geometry.hpp:165-169).
      const double ox = px[axis], oy = py[axis], oz = pz[axis];
      const double ax = dsub(px[anchor], ox), ay = dsub(py[anchor], oy), az = dsub(pz[anchor], oz);
      const double len = __dsqrt_rn(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az)));
      if (len < kMinAxisLength) {
        if (tid == 0) p.status[l] = 3;  // "rotate_fragment: degenerate rotation axis"
        return;
      }
      const Axis X{ox, oy, oz, __ddiv_rn(ax, len), __ddiv_rn(ay, len), __ddiv_rn(az, len)};
      // CandidateEvaluator::evaluate of one angle != 0 (uniform result).
      auto evaluate = [&](int a, double& score) -> bool {
        const double cs = __ldg(p.cos_deg + a), sn = __ldg(p.sin_deg + a), omc = dsub(1.0, cs);
        for (int i = tid; i < n; i += kWideThreads)
          if (in_frag(fm, i)) {
            rodrigues(X, cs, sn, omc, px[i], py[i], pz[i], qx[i], qy[i], qz[i]);
            wk.add(kRot, 1);
          }
        __syncthreads();
        bool bump = false;
        for (int i = tid; i < n && !bump; i += kWideThreads) {
          if (!in_frag(fm, i)) continue;
          for (int w = 0; w < W && !bump; ++w)
            for (uint64_t bits = far[static_cast<size_t>(i) * W + w] & ~fm[w]; bits; bits &= bits - 1) {
              const int j = 64 * w + __ffsll(static_cast<long long>(bits)) - 1;
              const double cut = dmul(kBumpScale, dadd(rad[i], rad[j]));
              wk.add(kBump, 1);
              if (dist_sq(qx[i], qy[i], qz[i], px[j], py[j], pz[j]) < dmul(cut, cut)) {
                bump = true;
                break;
              }
            }
        }
        if (__syncthreads_or(bump)) return false;
        for (int i = tid; i < n; i += kWideThreads)
          v[i] = in_frag(fm, i) ? fmax(kMinDistanceSq, min_dist_sq(p.pocket, qx[i], qy[i], qz[i], wk)) : pt[i];
        __syncthreads();
        wk.add(kTerms, tid == 0 ? n : 0);
        wk.add(kEvals, tid == 0 ? 1 : 0);
        score = fold(v);
        return true;
      };
      int best_a = 0;
      double best = cur;
      if (!refined) {
        // optimize_fragment_flat (kernel.hpp:125-143); angle 0 is the pose.
        int nfeas = 0;
        for (int c = 1; c < A; ++c) {
          double sc;
          if (!evaluate(c * step, sc)) continue;
          ++nfeas;
          if (sc > best) {
            best = sc;
            best_a = c * step;
          }
        }
        evals += 1 + nfeas;
        checks += A;
      } else {
        // optimize_fragment_refined (kernel.hpp:150-198).
        const int T = p.tile, tc = 360 / T;
        bool have = false;
        int wt = -1, nfeas = 0;
        double ws = 0.0;
        best = 0.0;
        auto visit = [&](int a, int tile) {
          double sc = cur;
          if (a != 0 && !evaluate(a, sc)) return;
          ++nfeas;
          if (!have || sc > best) {
            best = sc;
            best_a = a;
            have = true;
          }
          if (tile >= 0 && (wt < 0 || sc > ws)) {
            wt = tile;
            ws = sc;
          }
        };
        for (int t = 0; t < tc; ++t) visit(t * T + T / 2, t);
        checks += tc;
        if (wt >= 0) {
          int cnt2 = 0;
          while ((cnt2 + 1) * step <= T) ++cnt2;
          for (int k = 0; k < cnt2; ++k) visit(wt * T + k * step, -1);
          checks += cnt2;
        }
        checks += 1;  // entry-pose comparison (kernel.hpp:192-194)
        if (!have || cur > best) {
          best = cur;
          best_a = 0;
        }
        evals += nfeas;
      }
      // commit_angle (kernel.hpp:115-117).
      if (best_a != 0) {
        const double cs = __ldg(p.cos_deg + best_a), sn = __ldg(p.sin_deg + best_a);
        const double omc = dsub(1.0, cs);
        for (int i = tid; i < n; i += kWideThreads)
          if (in_frag(fm, i)) {
            double x, y, z;
            rodrigues(X, cs, sn, omc, px[i], py[i], pz[i], x, y, z);
            wk.add(kRot, 1);
            qx[i] = x;
            qy[i] = y;
            qz[i] = z;
            v[i] = fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk));
          }
        __syncthreads();  // every thread read the axis atoms' old coordinates above
        for (int i = tid; i < n; i += kWideThreads)
          if (in_frag(fm, i)) {
            px[i] = qx[i];
            py[i] = qy[i];
            pz[i] = qz[i];
            pt[i] = v[i];
          }
        __syncthreads();
      }
      cur = best;
    }
  }
  if (tid == 0) {
    p.st_final[e] = cur;
    p.st_evals[e] = evals;
    p.st_checks[e] = checks;
  }
  // Final pose staging, as flex_chain_kernel.
  if (p.stage_pose != nullptr) {
    if (tid == 0) {
      int stage = 1;
      if (p.top_best != nullptr) {
        const unsigned long long old =
            atomicMax(p.top_best + l, static_cast<unsigned long long>(__double_as_longlong(cur)));
        stage = __longlong_as_double(static_cast<long long>(old)) <= cur;
      }
      s_stage = stage;
    }
    __syncthreads();
    if (s_stage) {
      double* dst = p.stage_pose + 3 * (static_cast<size_t>(p.top_k) * m.atom_off + static_cast<size_t>(r) * n);
      for (int i = tid; i < n; i += kWideThreads) {
        dst[3 * i] = px[i];
        dst[3 * i + 1] = py[i];
        dst[3 * i + 2] = pz[i];
      }
    }
  }
  publish(wk, p.counters, 8);
}

// Rotation profiles (reference rotation_profile, analysis.hpp:37-56): one
// warp per (ligand, fragment) item scores the fragment at every integer
// angle about its bond, from the ligand's staged pose.  Angle 0 is the pose
// itself with its own bump check (check_bumps over the surviving pairs:
// a dropped pair cannot bump at any angle); angles 1..359 go through
// eval_batch exactly like search candidates.  Invalid angles report score 0,
// the reference's value-initialised array entry.
template <bool On, int B, int kWarps = warps_for<B>()>
__global__ void __launch_bounds__(kWarps * 32, GD_FLEX_RESIDENT / kWarps)
    profile_kernel(DockParams p, const int32_t* items, int n_items, double* scores, uint8_t* valid) {
  static_assert(B >= 1 && B <= 8, "batch_max reduces over an 8-lane butterfly");
  extern __shared__ __align__(16) unsigned char smem[];
  stage_tab<kCompactTU>(p.pocket);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kWarps + warp;
  if (item >= n_items) return;
  const int l = items[2 * item], f = items[2 * item + 1];
  const LigMeta m = p.meta[l];
  const int n = m.n, W = m.words;
  const WarpMem s =
      carve<B>(smem + warp * warp_bytes<B>(p.max_n, (p.max_n + 63) / 64, p.max_pairs), n, W,
               p.max_pairs);
  Work<On> wk;
  Clocks<false> ck;
  double* out = scores + 360ll * item;
  uint8_t* vout = valid + 360ll * item;

  for (int i = lane; i < n; i += 32) s.radius[i] = __ldg(p.radii + m.atom_off + i);
  for (int i = lane; i < n * W; i += 32) s.far[i] = __ldg(p.far_mask + m.far_off + i);
  for (int i = lane; i < n; i += 32) {
    const double* q = p.xyz + 3 * (m.atom_off + i);
    s.pt.set(i, PT{q[0], q[1], q[2], fmax(kMinDistanceSq, min_dist_sq(p.pocket, q[0], q[1], q[2], wk))});
  }
  __syncwarp();
  double cur = 0.0;
  if (lane == 0) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum = dadd(sum, s.pt.t(i));
    cur = __ddiv_rn(static_cast<double>(n), sum);
  }
  cur = __shfl_sync(kFull, cur, 0);

  const int fo = m.frag_off + f;
  int left_np = -1;
  StepInfo st;
  const uint64_t fm_word = lane < W ? __ldg(p.frag_mask + m.fmask_off + f * W + lane) : 0ull;
  if (!setup_step<B>(s, p, m, f, __ldg(p.frag_axis + fo), __ldg(p.frag_anchor + fo), fm_word, lane,
                     left_np, st, ck)) {
    if (lane == 0) p.status[l] = 3;  // "rotate_fragment: degenerate rotation axis"
    for (int a = lane; a < 360; a += 32) {
      out[a] = 0.0;
      vout[a] = 0;
    }
    publish_warp(wk, p.counters, 8, lane);
    return;
  }
  bool b0 = false;
  for (int t = lane; t < st.np; t += 32) {
    const int pr = s.pairs[t];
    const int i = pr & 0xff, j = pr >> 8;
    const PT ai = s.pt.get(i), aj = s.pt.get(j);
    const double cut = dmul(kBumpScale, dadd(s.radius[i], s.radius[j]));
    wk.add(kBump, 1);
    if (dist_sq(ai.x, ai.y, ai.z, aj.x, aj.y, aj.z) < dmul(cut, cut)) b0 = true;
  }
  b0 = __any_sync(kFull, b0);
  if (lane == 0) {
    vout[0] = b0 ? 0 : 1;
    out[0] = b0 ? 0.0 : cur;
  }
#if GD_FLAT_LIVE
  // As the flat searches: bump checks 32 angles at a time, then only the
  // live angles queried and folded, B at a time.
  for (int g0 = 1; g0 < 360; g0 += 32) {
    const int ng = min(32, 360 - g0);
    const unsigned bumped = bump_group(s, p, st.X, st.np, g0, 1, ng, lane, wk);
    if (lane < ng && ((bumped >> lane) & 1u)) {
      vout[g0 + lane] = 0;
      out[g0 + lane] = 0.0;
    }
    unsigned live = (ng == 32 ? kFull : (1u << ng) - 1u) & ~bumped;
    while (live) {
      const bool mine = (live >> lane) & 1u;
      const int rank = __popc(live & ((1u << lane) - 1u));
      const unsigned take = __ballot_sync(kFull, mine && rank < B);
      if (mine && rank < B) s.lidx[rank] = static_cast<uint8_t>(lane);
      const int nb = __popc(take);
      live &= ~take;
      __syncwarp();
      query_slots(s, p, st.X, n, st.nf, nb, g0, 1, lane, wk);
      __syncwarp();
      if (lane < nb) {
        double sum = st.pre;
        const double* vc = s.v + lane * vrow(n);
#pragma unroll kFoldUnroll
        for (int i = st.first; i < n; ++i) sum = dadd(sum, vc[i]);
        const int a = g0 + s.lidx[lane];
        out[a] = __ddiv_rn(static_cast<double>(n), sum);
        vout[a] = 1;
        wk.add(kTerms, n);
        wk.add(kEvals, 1);
      }
      __syncwarp();
    }
  }
#else
  for (int kb = 0; kb < 359; kb += B) {
    const int nb = min(B, 359 - kb);
    const int a0 = 1 + kb;
    double sc;
    unsigned bumped;
    eval_batch(s, p, st.X, n, st.nf, st.np, st.first, st.pre, cur, a0, 1, nb, lane, sc, bumped, wk,
               ck);
    if (lane < nb) {
      const bool ok = !((bumped >> lane) & 1u);
      vout[a0 + lane] = ok ? 1 : 0;
      out[a0 + lane] = ok ? sc : 0.0;
    }
  }
#endif
  publish_warp(wk, p.counters, 8, lane);
}

// ---------------------------------------------------------------------------
// Fine-grained drop-in entry points (gd_optimize_fragment_batch,
// gd_rotate_fragment_batch, gd_check_bumps_batch): one warp per ligand of
// the staged batch, each ligand carrying exactly one caller-given fragment
// (meta.nfrag == 1 at frag_off == l).
// ---------------------------------------------------------------------------

// optimize_fragment_flat / optimize_fragment_refined (kernel.hpp:125-198)
// from the ligand's staged pose: the same setup, candidate evaluator and
// decisions as a chain's fragment step, then commit_angle (:115-117).
template <bool On, int B, int kWarps = warps_for<B>()>
__global__ void __launch_bounds__(kWarps * 32, GD_FLEX_RESIDENT / kWarps)
    fragment_search_kernel(DockParams p, FragmentIO io) {
  static_assert(B >= 1 && B <= 8, "batch_max reduces over an 8-lane butterfly");
  extern __shared__ __align__(16) unsigned char smem[];
  stage_tab<kCompactTU>(p.pocket);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.x * kWarps + warp;
  if (l >= p.n_lig) return;
  const LigMeta m = p.meta[l];
  if (m.status != 0) return;
  const int n = m.n, W = m.words;
  const WarpMem s =
      carve<B>(smem + warp * warp_bytes<B>(p.max_n, (p.max_n + 63) / 64, p.max_pairs), n, W,
               p.max_pairs);
  Work<On> wk;
  Clocks<false> ck;
  for (int i = lane; i < n; i += 32) s.radius[i] = __ldg(p.radii + m.atom_off + i);
  for (int i = lane; i < n * W; i += 32) s.far[i] = __ldg(p.far_mask + m.far_off + i);
  for (int i = lane; i < n; i += 32) {
    const double* q = p.xyz + 3 * (m.atom_off + i);
    s.pt.set(i, PT{q[0], q[1], q[2], fmax(kMinDistanceSq, min_dist_sq(p.pocket, q[0], q[1], q[2], wk))});
  }
  __syncwarp();
  double cur = 0.0;
  if (lane == 0) {
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum = dadd(sum, s.pt.t(i));
    cur = __ddiv_rn(static_cast<double>(n), sum);
  }
  cur = __shfl_sync(kFull, cur, 0);
  const double given = io.entry_score ? io.entry_score[l] : cur;
  const double entry = given == given ? given : cur;  // NaN: not given
  const bool refined = io.refined != 0;
  const int step = p.hp;
  int best_a = 0, evals = 1, checks = 1;
  double best = cur;
  if (refined || step != 360) {  // flat at 360: angle 0 alone, no rotation
    StepInfo st;
    int left_np = -1;
    const uint64_t fm_word = lane < W ? __ldg(p.frag_mask + m.fmask_off + lane) : 0ull;
    if (!setup_step<B>(s, p, m, 0, __ldg(p.frag_axis + l), __ldg(p.frag_anchor + l), fm_word, lane,
                       left_np, st, ck)) {
      if (lane == 0) p.status[l] = 3;  // "rotate_fragment: degenerate rotation axis"
      return;
    }
    int win_row = -1;
    search_fragment<On, B>(s, p, st.X, n, st.nf, st.np, st.first, st.pre, cur, entry, step, refined,
                           lane, best_a, best, evals, checks, win_row, wk, ck);
    if (best_a != 0) {  // commit_angle: rotate the fragment by the winning angle
      const double cs = __ldg(p.cos_deg + best_a), sn = __ldg(p.sin_deg + best_a);
      const double omc = dsub(1.0, cs);
      for (int sl = lane; sl < st.nf; sl += 32) {
        const int i = s.fidx[sl];
        const PT q = s.pt.get(i);
        double qx, qy, qz;
        rodrigues(st.X, cs, sn, omc, q.x, q.y, q.z, qx, qy, qz);
        s.pt.set(i, PT{qx, qy, qz, 0.0});
      }
    }
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) {
    const PT q = s.pt.get(i);
    double* d = io.pose + 3 * (static_cast<size_t>(m.atom_off) + i);
    d[0] = q.x;
    d[1] = q.y;
    d[2] = q.z;
  }
  if (lane == 0) {
    io.best_angle[l] = best_a;
    io.best_score[l] = best;
    io.evaluations[l] = evals;
    io.checks[l] = checks;
  }
  publish_warp(wk, p.counters, 8, lane);
}

// rotate_fragment_into (geometry.hpp:161-186): the axis from the staged
// pose (degenerate below 1e-9 A, checked before the angle-0 shortcut), then
// every fragment atom rotated by the ligand's angle (host cos/sin of
// angle * (pi/180), as the reference computes them) and the rest copied.
__global__ void __launch_bounds__(256) fragment_rotate_kernel(DockParams p, const double* cs_in,
                                                               const double* sn_in,
                                                               const uint8_t* is_zero,
                                                               double* out) {
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (l >= p.n_lig) return;
  const LigMeta m = p.meta[l];
  if (m.status != 0) return;
  const double* xyz = p.xyz + 3 * static_cast<size_t>(m.atom_off);
  const int ia = __ldg(p.frag_axis + l), ib = __ldg(p.frag_anchor + l);
  const double ox = xyz[3 * ia], oy = xyz[3 * ia + 1], oz = xyz[3 * ia + 2];
  const double ax = dsub(xyz[3 * ib], ox), ay = dsub(xyz[3 * ib + 1], oy), az = dsub(xyz[3 * ib + 2], oz);
  const double len = __dsqrt_rn(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az)));
  if (len < kMinAxisLength) {
    if (lane == 0) p.status[l] = 3;
    return;
  }
  const Axis X{ox, oy, oz, __ddiv_rn(ax, len), __ddiv_rn(ay, len), __ddiv_rn(az, len)};
  const bool zero = is_zero[l] != 0;
  const double cs = cs_in[l], sn = sn_in[l], omc = dsub(1.0, cs);
  const uint64_t* fm = p.frag_mask + m.fmask_off;
  double* o = out + 3 * static_cast<size_t>(m.atom_off);
  for (int i = lane; i < m.n; i += 32) {
    double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    if (!zero && ((fm[i >> 6] >> (i & 63)) & 1ull)) rodrigues(X, cs, sn, omc, x, y, z, x, y, z);
    o[3 * i] = x;
    o[3 * i + 1] = y;
    o[3 * i + 2] = z;
  }
}

// check_bumps (geometry.hpp:199-213) of the staged pose against the
// ligand's fragment: lanes over fragment atoms i, each scanning its
// partners j outside the fragment at capped graph distance >= 4.
__global__ void __launch_bounds__(256) fragment_bumps_kernel(DockParams p, uint8_t* feasible) {
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (l >= p.n_lig) return;
  const LigMeta m = p.meta[l];
  if (m.status != 0) return;
  const double* xyz = p.xyz + 3 * static_cast<size_t>(m.atom_off);
  const double* rad = p.radii + m.atom_off;
  const uint64_t* fm = p.frag_mask + m.fmask_off;
  const uint64_t* far = p.far_mask + m.far_off;
  bool bump = false;
  for (int i = lane; i < m.n && !bump; i += 32) {
    if (!((fm[i >> 6] >> (i & 63)) & 1ull)) continue;
    for (int w = 0; w < m.words && !bump; ++w) {
      uint64_t bits = far[static_cast<size_t>(i) * m.words + w] & ~fm[w];
      while (bits) {
        const int j = 64 * w + __ffsll(static_cast<long long>(bits)) - 1;
        bits &= bits - 1;
        const double cut = dmul(kBumpScale, dadd(rad[i], rad[j]));
        if (dist_sq(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], xyz[3 * j], xyz[3 * j + 1],
                    xyz[3 * j + 2]) < dmul(cut, cut)) {
          bump = true;
          break;
        }
      }
    }
  }
  bump = __any_sync(kFull, bump);
  if (lane == 0) feasible[l] = bump ? 0 : 1;
}

// (E7) final order: (final score desc, seed rank asc), one rank per thread;
// each rank's destination is the number of ranks that precede it.
__global__ void __launch_bounds__(256) finalize_kernel(DockParams p) {
  const int l = p.order[blockIdx.x];
  const LigMeta m = p.meta[l];
  const int K = p.k_slots, slots = p.top_k;
  // Empty slots read as orientation -2 and zeros on the device too (the
  // gd_device_results table equals the downloaded gd_result).
  const bool failed = m.status != 0 || p.status[l] != 0;
  for (int e = (failed ? 0 : K) + threadIdx.x; e < slots; e += blockDim.x) {
    const size_t d = static_cast<size_t>(l) * slots + e;
    p.out_final[d] = 0.0;
    p.out_evals[d] = 0;
    p.out_checks[d] = 0;
    p.out_rank[d] = 0;
    p.out_orient[d] = -2;
    p.out_rigid[d] = 0.0;
  }
  if (failed) {
    if (threadIdx.x == 0) {
      p.poses_scored[l] = 0;
      p.k_eff[l] = 0;
    }
    if (p.out_top != nullptr)
      for (int i = threadIdx.x; i < 3 * m.n; i += blockDim.x) p.out_top[3 * static_cast<size_t>(m.atom_off) + i] = 0.0;
    return;
  }
  __shared__ double fin[256];
  __shared__ unsigned long long total;
  const int e = threadIdx.x;
  if (e < K) fin[e] = p.st_final[static_cast<size_t>(l) * slots + e];
  if (e == 0) total = 0;
  __syncthreads();
  if (e < K) {
    const double fe = fin[e];
    int pos = 0;
    for (int e2 = 0; e2 < K; ++e2) pos += precede(fin[e2], e2, fe, e) ? 1 : 0;
    const size_t src = static_cast<size_t>(l) * slots + e;
    const size_t d = static_cast<size_t>(l) * slots + pos;
    const long long ev = p.st_evals[src];
    p.out_final[d] = fe;
    p.out_evals[d] = ev;
    p.out_checks[d] = p.st_checks[src];
    p.out_rank[d] = e;
    p.out_orient[d] = p.rigid ? p.orient_idx[p.seed_slot[src]] : -1;
    p.out_rigid[d] = p.seed_score[src];
    if (p.out_pose != nullptr) {
      const int n = m.n;
      const double* from = p.stage_pose + 3 * (static_cast<size_t>(slots) * m.atom_off + static_cast<size_t>(e) * n);
      double* to = p.out_pose + 3 * (static_cast<size_t>(slots) * m.atom_off + static_cast<size_t>(pos) * n);
      for (int i = 0; i < 3 * n; ++i) to[i] = from[i];
    }
    if (p.out_top != nullptr && pos == 0) {
      const int n = m.n;
      const double* from = p.stage_pose + 3 * (static_cast<size_t>(slots) * m.atom_off + static_cast<size_t>(e) * n);
      double* to = p.out_top + 3 * static_cast<size_t>(m.atom_off);
      for (int i = 0; i < 3 * n; ++i) to[i] = from[i];
    }
    atomicAdd(&total, static_cast<unsigned long long>(ev));
  }
  __syncthreads();
  if (e == 0) {
    p.poses_scored[l] = static_cast<long long>(total) + (p.rigid ? p.n_orient : 0);
    p.k_eff[l] = K;
  }
}

template <int B, int W>
size_t flex_smem_bytes(const DockParams& p) {
  return W * warp_bytes<B>(p.max_n, (p.max_n + 63) / 64, p.max_pairs);
}

// Batch size from the high-precision step's c = 360/hp - 1 candidates: the
// fewest batches of at most 8, evenly filled, rounded up to an
// instantiated size (4, 6, 8).  Measured (c1: c = 11 -> 6; c2: c = 35 -> 8):
// c1 flex 17.29 / 16.84 / 17.07 / 17.78 ms at B = 4 / 6 / 8 / 12; c2 74.1 ms
// at 8 vs 75.5 at 6 and 78.1 at 12.
int flex_batch(const DockParams& p) {
  if (GD_FLEX_BATCH) return GD_FLEX_BATCH;
  const int c = std::max(1, 360 / p.hp - 1);
  if (c <= 8) return c <= 4 ? 4 : c <= 6 ? 6 : 8;  // one batch
  // Many candidates (flat searches batch only the live ones since r3e): 8
  // (c2's 35: flex 52.4 ms vs 54.2 at 6).  A few more than 8: at most 6
  // each (c1's 11: 11.65 ms vs 12.41 at 8).
  if (c > 16) return 8;
  const int batches = (c + 5) / 6;
  return (c + batches - 1) / batches <= 4 ? 4 : 6;
}

// Dynamic shared memory a CTA may opt into (the coded format's kernels also
// hold the static coordinate table).
int max_smem_optin() {
  static int v = [] {
    int dev = 0, bytes = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return bytes - (kCompactTU ? static_cast<int>(sizeof(double)) * kCodedTab : 0);
  }();
  return v;
}

template <int B, int W>
int launch_flex_bw(const DockParams& p, long long chains, cudaStream_t stream) {
  const size_t smem = flex_smem_bytes<B, W>(p);
  const bool replay = GD_FIXED_POINT && p.reps > 1;
  auto kernel = p.counters ? (replay ? flex_chain_kernel<true, B, W, true> : flex_chain_kernel<true, B, W>)
                           : (replay ? flex_chain_kernel<false, B, W, true> : flex_chain_kernel<false, B, W>);
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  // Shared memory and L1 share the SM's 256 KB; the voxel-record gathers
  // live in L1, so the carveout is an explicit tuning knob.
  if (const char* cv = std::getenv("GD_FLEX_CARVEOUT")) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(cv));
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (chains + W - 1) / W;
  kernel<<<static_cast<unsigned>(blocks), W * 32, smem, stream>>>(p);
  return cudaGetLastError();
}

// The preferred CTA shape when its shared memory fits the opt-in limit,
// else narrower CTAs (large ligands: ~30 KB per chain at 150 atoms).
template <int B>
int launch_flex_b(const DockParams& p, long long chains, cudaStream_t stream) {
  const size_t lim = static_cast<size_t>(max_smem_optin());
  constexpr int W0 = warps_for<B>();
  if (flex_smem_bytes<B, W0>(p) <= lim) return launch_flex_bw<B, W0>(p, chains, stream);
  if (flex_smem_bytes<B, 4>(p) <= lim) return launch_flex_bw<B, 4>(p, chains, stream);
  if (flex_smem_bytes<B, 2>(p) <= lim) return launch_flex_bw<B, 2>(p, chains, stream);
  return launch_flex_bw<B, 1>(p, chains, stream);
}

template <int B, int W>
int launch_profiles_bw(const DockParams& p, const int32_t* items, int n_items, double* scores,
                       uint8_t* valid, cudaStream_t stream) {
  const size_t smem = flex_smem_bytes<B, W>(p);
  auto kernel = p.counters ? profile_kernel<true, B, W> : profile_kernel<false, B, W>;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int blocks = (n_items + W - 1) / W;
  kernel<<<blocks, W * 32, smem, stream>>>(p, items, n_items, scores, valid);
  return cudaGetLastError();
}

template <int B>
int launch_profiles_b(const DockParams& p, const int32_t* items, int n_items, double* scores,
                      uint8_t* valid, cudaStream_t stream) {
  const size_t lim = static_cast<size_t>(max_smem_optin());
  constexpr int W0 = warps_for<B>();
  if (flex_smem_bytes<B, W0>(p) <= lim)
    return launch_profiles_bw<B, W0>(p, items, n_items, scores, valid, stream);
  if (flex_smem_bytes<B, 2>(p) <= lim)
    return launch_profiles_bw<B, 2>(p, items, n_items, scores, valid, stream);
  return launch_profiles_bw<B, 1>(p, items, n_items, scores, valid, stream);
}

}  // namespace

int GD_API(launch_flex)(const DockParams& p, void* stream) {
  const long long chains = static_cast<long long>(p.n_lig) * p.k_slots;
  if (chains == 0) return cudaSuccess;
  const auto s = static_cast<cudaStream_t>(stream);
  switch (flex_batch(p)) {
    case 8: return launch_flex_b<8>(p, chains, s);
    case 6: return launch_flex_b<6>(p, chains, s);
    default: return launch_flex_b<4>(p, chains, s);
  }
}

int GD_API(launch_flex_wide)(const DockParams& p, void* stream) {
  const long long chains = static_cast<long long>(p.n_wide) * p.k_slots;
  if (chains == 0) return cudaSuccess;
  auto kernel = p.counters ? flex_wide_kernel<true> : flex_wide_kernel<false>;
  kernel<<<static_cast<unsigned>(chains), kWideThreads, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError();
}

int GD_API(launch_profiles)(const DockParams& p, const int32_t* items, int n_items, double* scores,
                            uint8_t* valid, void* stream) {
  if (n_items == 0) return cudaSuccess;
#ifndef GD_PROFILE_BATCH
#define GD_PROFILE_BATCH 8
#endif
  // 359 candidates per fragment: the wide batch.
  return launch_profiles_b<GD_PROFILE_BATCH>(p, items, n_items, scores, valid,
                                             static_cast<cudaStream_t>(stream));
}

template <int B, int W>
int launch_fragment_search_bw(const DockParams& p, const FragmentIO& io, cudaStream_t stream) {
  const size_t smem = flex_smem_bytes<B, W>(p);
  auto kernel = p.counters ? fragment_search_kernel<true, B, W> : fragment_search_kernel<false, B, W>;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kernel<<<(p.n_lig + W - 1) / W, W * 32, smem, stream>>>(p, io);
  return cudaGetLastError();
}

int GD_API(launch_fragment_search)(const DockParams& p, const FragmentIO& io, void* stream) {
  if (p.n_lig == 0) return cudaSuccess;
  const auto s = static_cast<cudaStream_t>(stream);
  if (flex_smem_bytes<8, 4>(p) <= static_cast<size_t>(max_smem_optin()))
    return launch_fragment_search_bw<8, 4>(p, io, s);
  return launch_fragment_search_bw<8, 1>(p, io, s);
}

#if !GD_TU_COMPACT  // format-independent launchers: defined once
int launch_fragment_rotate(const DockParams& p, const double* cs, const double* sn,
                           const uint8_t* is_zero, double* out, void* stream) {
  if (p.n_lig == 0) return cudaSuccess;
  fragment_rotate_kernel<<<(p.n_lig + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p, cs, sn, is_zero, out);
  return cudaGetLastError();
}

int launch_fragment_bumps(const DockParams& p, uint8_t* feasible, void* stream) {
  if (p.n_lig == 0) return cudaSuccess;
  fragment_bumps_kernel<<<(p.n_lig + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(p,
                                                                                         feasible);
  return cudaGetLastError();
}

int launch_finalize(const DockParams& p, void* stream) {
  if (p.n_lig == 0) return cudaSuccess;
  finalize_kernel<<<p.n_lig, 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError();
}
#endif

}  // namespace gdb200
