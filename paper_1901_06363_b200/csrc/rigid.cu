// (1) rigid initial-pose sweep + (4) overlap scoring + (5b) top-K seeds.
//
// One CTA per ligand, one thread per orientation of the (de-duplicated)
// Euler grid: the thread rotates the ligand about the pocket centre
// (E3) atom by atom and folds the overlap score in atom order
// (reference overlap_score, geometry.hpp:143-154).  Top K by (score desc,
// orientation index asc) (E5): for K <= 32 each warp keeps a sorted top-32
// in registers (shuffle networks) and a 3-level tree merges the 8 warp
// lists; larger K goes through a shared-memory bitonic sort chunk by chunk.
#include "device_common.cuh"

namespace gdb200 {
namespace {

#ifndef GD_RIGID_MINB
#define GD_RIGID_MINB 4  // resident CTAs per SM the register budget targets
#endif
#ifndef GD_RIGID_MLP
#define GD_RIGID_MLP 2   // atoms whose nearest-point lookups are in flight together
#endif
constexpr int kRigidThreads = 256;

// Score of orientation s: rotate every atom (E3) and fold the overlap terms
// strictly in atom order (geometry.hpp:143-154); atoms go in groups of
// GD_RIGID_MLP so their nearest-point lookups are in flight together.
template <bool On>
__device__ __forceinline__ double score_orientation(const DockParams& p, int s, int n,
                                                   const double* vx, const double* vy,
                                                   const double* vz, Work<On>& wk) {
  double R[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) R[r] = __ldg(p.orient_R + 9 * s + r);
  double sum = 0.0;
  int i = 0;
  for (; i + GD_RIGID_MLP - 1 < n; i += GD_RIGID_MLP) {
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
    p.seed_slot[l * p.top_k + lane] = list.i;
    p.seed_score[l * p.top_k + lane] = list.k;
  }
  if (threadIdx.x == 0) p.k_eff[l] = K;
  publish(wk, p.counters, 0);
}

// --- general K: shared-memory bitonic sort over chunks -----------------------
template <int BT, bool On>
__global__ void __launch_bounds__(BT, GD_RIGID_MINB) rigid_topk_kernel(DockParams p, int sort_slots) {
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
  Work<On> wk;
  int carry = 0;
  for (int base = 0; base < No;) {
    const int take = min(sort_slots - carry, No - base);
    for (int t = threadIdx.x; t < sort_slots - carry; t += BT) {
      double score = kInfeasible;
      int s = INT_MAX;
      if (t < take) {
        s = base + t;
        score = score_orientation(p, s, n, vx, vy, vz, wk);
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

template <bool On>
int launch(const DockParams& p, int sort_slots, cudaStream_t stream) {
  if (p.top_k <= 32) {
    const size_t smem = sizeof(double) * 3 * p.max_n;
    cudaError_t e = cudaFuncSetAttribute(rigid_top32_kernel<kRigidThreads, On>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    rigid_top32_kernel<kRigidThreads, On><<<p.n_lig, kRigidThreads, smem, stream>>>(p);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(double) * 3 * p.max_n + (sizeof(double) + sizeof(int)) * sort_slots;
  cudaError_t e = cudaFuncSetAttribute(rigid_topk_kernel<kRigidThreads, On>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  rigid_topk_kernel<kRigidThreads, On><<<p.n_lig, kRigidThreads, smem, stream>>>(p, sort_slots);
  return cudaGetLastError();
}

}  // namespace

int launch_rigid_topk(const DockParams& p, int sort_slots, void* stream) {
  const auto s = static_cast<cudaStream_t>(stream);
  return p.counters ? launch<true>(p, sort_slots, s) : launch<false>(p, sort_slots, s);
}

}  // namespace gdb200
