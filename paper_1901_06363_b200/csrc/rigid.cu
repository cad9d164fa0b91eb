// (1) rigid initial-pose sweep + (4) overlap scoring + (5b) top-K seeds.
//
// One CTA per ligand, one thread per orientation of the (de-duplicated)
// Euler grid: the thread rotates the ligand about the pocket centre
// (E3) atom by atom and folds the overlap score in atom order
// (reference overlap_score, geometry.hpp:143-154).  Top K by (score desc,
// orientation index asc) (E5): for K <= 32 each warp keeps a sorted top-32
// in registers (shuffle networks) and a 3-level tree merges the 8 warp
// lists; larger K keeps a sorted shared-memory list into which each round's
// winners (scores beating the current K-th) are merged by rank.
#include <algorithm>

// The rigid sweep keeps the two-step voxel lookup: its atoms sit around the
// pocket centre, mostly inside the fine level, and at 40 registers the
// branch-free form's extra arithmetic costs more than the rare second lookup
// (r3j: c1 rigid 2.68 vs 2.55 ms, c2 18.1 vs 17.0; the fragment search gains
// 3% from it, see device_common.cuh).
#ifndef GD_LOCATE_FLAT
#define GD_LOCATE_FLAT 0
#endif
#include "device_common.cuh"

namespace gdb200 {
namespace {

// With the orientation matrix in shared memory (GD_RIGID_RSMEM), one lookup
// in flight at 6 CTAs per SM (40 registers) beats two at 5 (r2g: c1 rigid
// 2.91 -> 2.78 ms, c2 19.8 -> 18.1 ms; 7 CTAs spill).
#ifndef GD_RIGID_MINB
#define GD_RIGID_MINB 6  // resident CTAs per SM the register budget targets
#endif
#ifndef GD_RIGID_MLP
#define GD_RIGID_MLP 1   // atoms whose nearest-point lookups are in flight together
#endif
#ifndef GD_RIGID_RSMEM
#define GD_RIGID_RSMEM 1 // the orientation matrix re-read from shared memory per atom group (c1 rigid 2.96 -> 2.91 ms, c2 20.9 -> 19.9)
#endif
constexpr int kRigidThreads = 256;

// Score of orientation s: rotate every atom (E3) and fold the overlap terms
// strictly in atom order (geometry.hpp:143-154); atoms go in groups of
// GD_RIGID_MLP so their nearest-point lookups are in flight together.
template <bool On>
__device__ __forceinline__ double score_orientation(const DockParams& p, int s, int n,
                                                   const double* vx, const double* vy,
                                                   const double* vz, Work<On>& wk) {
#if GD_RIGID_RSMEM
  // The thread's column of a [9][256] shared table: 18 registers free for
  // the lookups, at 9 shared loads per atom group.
  __shared__ double Rs[9 * kRigidThreads];
  volatile double* Rv = Rs + threadIdx.x;
#pragma unroll
  for (int r = 0; r < 9; ++r) Rv[r * kRigidThreads] = __ldg(p.orient_R + 9 * s + r);
#else
  double R[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) R[r] = __ldg(p.orient_R + 9 * s + r);
#endif
  double sum = 0.0;
  int i = 0;
  for (; i + GD_RIGID_MLP - 1 < n; i += GD_RIGID_MLP) {
#if GD_RIGID_RSMEM
    double R[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) R[r] = Rv[r * kRigidThreads];
#endif
    double x[GD_RIGID_MLP], y[GD_RIGID_MLP], z[GD_RIGID_MLP], mm[GD_RIGID_MLP];
#pragma unroll
    for (int r = 0; r < GD_RIGID_MLP; ++r)
      rigid_apply(R, p.cx, p.cy, p.cz, vx[i + r], vy[i + r], vz[i + r], x[r], y[r], z[r]);
    wk.add(kXform, GD_RIGID_MLP);
    min_dist_sqM<GD_RIGID_MLP>(p.pocket, x, y, z, mm, wk);
#pragma unroll
    for (int r = 0; r < GD_RIGID_MLP; ++r) sum = dadd(sum, fmax(kMinDistanceSq, mm[r]));
  }
  for (; i < n; ++i) {
#if GD_RIGID_RSMEM
    double R[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) R[r] = Rv[r * kRigidThreads];
#endif
    double x, y, z;
    rigid_apply(R, p.cx, p.cy, p.cz, vx[i], vy[i], vz[i], x, y, z);
    wk.add(kXform, 1);
    sum = dadd(sum, fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk)));
  }
  wk.add(kTerms, n);
  return __ddiv_rn(static_cast<double>(n), sum);
}

// --- warp-register top-32 (K <= 32) -----------------------------------------
// A warp holds a list of 32 (score, slot) entries, one per lane, lane 0 the
// best under E5's order.  All steps are compare-exchange networks over
// shuffles; entries are distinct (slots are unique), so the result equals a
// full sort's first K entries.
struct Entry {
  double k;
  int i;
};

__device__ __forceinline__ Entry shfl_xor(Entry e, int m) {
  return Entry{__shfl_xor_sync(0xffffffffu, e.k, m), __shfl_xor_sync(0xffffffffu, e.i, m)};
}

// One compare-exchange stage at distance j: the lower lane of each pair
// keeps the preceding entry when `first` holds, the other one otherwise.
__device__ __forceinline__ Entry cx_stage(Entry e, int j, bool first) {
  const Entry o = shfl_xor(e, j);
  const bool lower = (threadIdx.x & j) == 0;
  const bool o_first = precede(o.k, o.i, e.k, e.i);
  return (lower == first) == o_first ? o : e;
}

__device__ __forceinline__ Entry warp_sort32(Entry e) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) e = cx_stage(e, j, (lane & k) == 0);
  return e;
}

// a, b sorted: the sorted best 32 of their union.
__device__ __forceinline__ Entry warp_merge32(Entry a, Entry b) {
  const Entry br{__shfl_sync(0xffffffffu, b.k, 31 - (threadIdx.x & 31)),
                 __shfl_sync(0xffffffffu, b.i, 31 - (threadIdx.x & 31))};
  Entry e = precede(br.k, br.i, a.k, a.i) ? br : a;  // bitonic
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) e = cx_stage(e, j, true);
  return e;
}

template <int BT, bool On>
__global__ void __launch_bounds__(BT, GD_RIGID_MINB) rigid_top32_kernel(DockParams p) {
  static_assert(BT == 256, "tree merge below assumes 8 warps");
  const int l = p.order[blockIdx.x];
  const LigMeta m = p.meta[l];
  if (m.status != 0) {
    if (threadIdx.x == 0) p.k_eff[l] = 0;
    return;
  }
  if (!p.wide_pass && m.n > kNarrowAtoms) return;  // swept by the wide ligands' own launch
  stage_tab<kCompactTU>(p.pocket);
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = m.n;
  double* vx = reinterpret_cast<double*>(smem);
  double* vy = vx + n;
  double* vz = vy + n;
  __shared__ double mkey[BT];
  __shared__ int mslot[BT];
  for (int i = threadIdx.x; i < n; i += BT) {
    const double* q = p.xyz + 3 * (m.atom_off + i);
    vx[i] = dsub(q[0], p.cx);
    vy[i] = dsub(q[1], p.cy);
    vz[i] = dsub(q[2], p.cz);
  }
  __syncthreads();

  const int No = p.n_orient;
  const int K = min(p.top_k, No);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Work<On> wk;
  Entry list{kInfeasible, INT_MAX};
  for (int base = warp * 32; base < No; base += BT) {
    Entry e{kInfeasible, INT_MAX};
    if (base + lane < No) {
      e.i = base + lane;
      e.k = score_orientation(p, e.i, n, vx, vy, vz, wk);
    }
    const double wk_k = __shfl_sync(0xffffffffu, list.k, 31);
    const int wk_i = __shfl_sync(0xffffffffu, list.i, 31);
    if (__any_sync(0xffffffffu, precede(e.k, e.i, wk_k, wk_i)))
      list = warp_merge32(list, warp_sort32(e));
  }
  // Tree merge of the 8 warp lists: 8 -> 4 -> 2 -> 1.
#pragma unroll
  for (int half = 4; half >= 1; half >>= 1) {
    if (warp >= half && warp < 2 * half) {
      mkey[threadIdx.x] = list.k;
      mslot[threadIdx.x] = list.i;
    }
    __syncthreads();
    if (warp < half) {
      const Entry o{mkey[threadIdx.x + 32 * half], mslot[threadIdx.x + 32 * half]};
      list = warp_merge32(list, o);
    }
    if (half > 1) __syncthreads();
  }
  if (warp == 0 && lane < K) {
    p.seed_slot[static_cast<size_t>(l) * p.top_k + lane] = list.i;
    p.seed_score[static_cast<size_t>(l) * p.top_k + lane] = list.k;
  }
  if (threadIdx.x == 0) p.k_eff[l] = K;
  publish(wk, p.counters, 0);
}

// --- general K: threshold + compaction + rank merge --------------------------
// Orientations are scored in rounds of BT (one per thread).  Only scores
// that precede the current K-th entry are compacted into a pending buffer;
// the pending entries are ranked among themselves (O(pending) each) and
// merged into the sorted list by rank: an entry's new position is its rank
// in its own list plus the number of entries of the other list preceding it
// (a binary search).  A round whose scores all lose costs one ballot.
template <int BT, bool On>
__global__ void __launch_bounds__(BT, GD_RIGID_MINB) rigid_topk_kernel(DockParams p) {
  const int l = p.order[blockIdx.x];
  const LigMeta m = p.meta[l];
  if (m.status != 0) {
    if (threadIdx.x == 0) p.k_eff[l] = 0;
    return;
  }
  if (!p.wide_pass && m.n > kNarrowAtoms) return;  // swept by the wide ligands' own launch
  stage_tab<kCompactTU>(p.pocket);
  const int n = m.n;
  const int No = p.n_orient;
  const int K = min(p.top_k, No);
  extern __shared__ __align__(16) unsigned char smem[];
  double* vx = reinterpret_cast<double*>(smem);
  double* vy = vx + n;
  double* vz = vy + n;
  double* lk = vz + n;   // [K] sorted list (keys) ...
  double* nk = lk + K;   // [K] ... and its merge target
  double* pk = nk + K;   // [BT] pending, arrival order
  double* qk = pk + BT;  // [BT] pending, sorted
  int* ls = reinterpret_cast<int*>(qk + BT);
  int* ns = ls + K;
  int* ps = ns + K;
  int* qs = ps + BT;
  __shared__ int wcnt[BT / 32];

  for (int i = threadIdx.x; i < n; i += BT) {
    const double* q = p.xyz + 3 * (m.atom_off + i);
    vx[i] = dsub(q[0], p.cx);
    vy[i] = dsub(q[1], p.cy);
    vz[i] = dsub(q[2], p.cz);
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Work<On> wk;
  int kept = 0;
  for (int base = 0; base < No; base += BT) {
    const int s = base + threadIdx.x;
    double score = kInfeasible;
    bool q = false;
    if (s < No) {
      score = score_orientation(p, s, n, vx, vy, vz, wk);
      q = kept < K || precede(score, s, lk[K - 1], ls[K - 1]);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, q);
    if (lane == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < BT / 32; ++w) {
      const int c = wcnt[w];
      off += w < warp ? c : 0;
      total += c;
    }
    if (q) {
      const int at = off + __popc(bal & ((1u << lane) - 1u));
      pk[at] = score;
      ps[at] = s;
    }
    __syncthreads();
    if (total == 0) continue;
    if (threadIdx.x < total) {
      const double k0 = pk[threadIdx.x];
      const int s0 = ps[threadIdx.x];
      int r = 0;
      for (int j = 0; j < total; ++j) r += precede(pk[j], ps[j], k0, s0) ? 1 : 0;
      qk[r] = k0;
      qs[r] = s0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < kept + total; j += BT) {
      const bool old = j < kept;
      const int t = old ? j : j - kept;
      const double k0 = old ? lk[t] : qk[t];
      const int s0 = old ? ls[t] : qs[t];
      const double* ok = old ? qk : lk;
      const int* os = old ? qs : ls;
      int lo = 0, hi = old ? total : kept;  // entries of the other list preceding (k0, s0)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (precede(ok[mid], os[mid], k0, s0)) lo = mid + 1;
        else hi = mid;
      }
      const int pos = t + lo;
      if (pos < K) {
        nk[pos] = k0;
        ns[pos] = s0;
      }
    }
    __syncthreads();
    kept = min(K, kept + total);
    double* tk = lk;
    lk = nk;
    nk = tk;
    int* ts = ls;
    ls = ns;
    ns = ts;
  }
  for (int r = threadIdx.x; r < K; r += BT) {
    p.seed_slot[static_cast<size_t>(l) * p.top_k + r] = ls[r];
    p.seed_score[static_cast<size_t>(l) * p.top_k + r] = lk[r];
  }
  if (threadIdx.x == 0) p.k_eff[l] = K;
  publish(wk, p.counters, 0);
}

template <bool On>
int launch(const DockParams& p, cudaStream_t stream) {
  if (p.top_k <= 32) {
    const size_t smem = sizeof(double) * 3 * p.max_n;
    cudaError_t e = cudaFuncSetAttribute(rigid_top32_kernel<kRigidThreads, On>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    rigid_top32_kernel<kRigidThreads, On><<<p.n_lig, kRigidThreads, smem, stream>>>(p);
    return cudaGetLastError();
  }
  const int K = std::min(p.top_k, p.n_orient);
  const size_t smem = sizeof(double) * 3 * p.max_n +
                      (sizeof(double) + sizeof(int)) * (2 * static_cast<size_t>(K) + 2 * kRigidThreads);
  cudaError_t e = cudaFuncSetAttribute(rigid_topk_kernel<kRigidThreads, On>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  rigid_topk_kernel<kRigidThreads, On><<<p.n_lig, kRigidThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

int GD_API(launch_rigid_topk)(const DockParams& p, void* stream) {
  const auto s = static_cast<cudaStream_t>(stream);
  return p.counters ? launch<true>(p, s) : launch<false>(p, s);
}

}  // namespace gdb200
