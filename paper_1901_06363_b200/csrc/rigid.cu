// (1) rigid initial-pose sweep + (4) overlap scoring + (5b) top-K seeds.
//
// One CTA per ligand, one thread per orientation of the (de-duplicated)
// Euler grid: the thread rotates the ligand about the pocket centre
// (E3) atom by atom and folds the overlap score in atom order
// (reference overlap_score, geometry.hpp:143-154).  Scores land in a
// shared-memory buffer that a bitonic sort merges chunk by chunk, keeping
// the top K by (score desc, orientation index asc) (E5).
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
  const double dn = static_cast<double>(n);
  Work<On> wk;
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
        // Atoms in pairs: both nearest-point lookups in flight at once, the
        // fold still strictly in atom order.
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
        if (i < n) {
          double x, y, z;
          rigid_apply(R, p.cx, p.cy, p.cz, vx[i], vy[i], vz[i], x, y, z);
          wk.add(kXform, 1);
          sum = dadd(sum, fmax(kMinDistanceSq, min_dist_sq(p.pocket, x, y, z, wk)));
        }
        wk.add(kTerms, n);
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

template <bool On>
int launch(const DockParams& p, int sort_slots, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(rigid_topk_kernel<kRigidThreads, On>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  rigid_topk_kernel<kRigidThreads, On><<<p.n_lig, kRigidThreads, smem, stream>>>(p, sort_slots);
  return cudaGetLastError();
}

}  // namespace

size_t rigid_smem_bytes(const DockParams& p, int sort_slots) {
  return sizeof(double) * 3 * p.max_n + (sizeof(double) + sizeof(int)) * sort_slots;
}

int launch_rigid_topk(const DockParams& p, int sort_slots, void* stream) {
  const size_t smem = rigid_smem_bytes(p, sort_slots);
  const auto s = static_cast<cudaStream_t>(stream);
  return p.counters ? launch<true>(p, sort_slots, smem, s) : launch<false>(p, sort_slots, smem, s);
}

}  // namespace gdb200
