// Ligand preprocessing on the GPU: the per-ligand work the reference does in
// the Ligand constructor and find_rotamers / grow_fragments
// (molecule.hpp:66-140, :190-301), restated as bit-parallel graph
// operations, one WARP per ligand.  The host only copies raw atoms and bonds
// (xyz, radii, bond pairs, rotatable flags) and fills offsets; everything
// the search kernels read is produced here, in HBM:
//
//   * validation (radii > 0, finite positions, no self/out-of-range/duplicate
//     bonds, connected) -> meta.status; the reference's message for a
//     rejected ligand is re-derived on the host (prep.cpp), only for those;
//   * the adjacency as n x W bit rows in shared memory (atomicOr; a bit
//     already set is a duplicate bond);
//   * far masks: bit j of row i iff bond-graph distance(i, j) >= 4, from
//     the 3-hop closure S3 = S2 | adj(S2 \ S1) (S1 = {i} | adj(i));
//   * rotamers: a rotatable bond (lo, hi) is a bridge iff the BFS from lo
//     that ignores it never reaches hi -- that BFS's visited set is the left
//     fragment (grow_fragments, :255-301); rotamers are ordered by (lo, hi)
//     (find_rotamers, :237-250) by ranking the unique keys lo << 8 | hi;
//   * fragments 2r (left: axis lo, anchor hi) and 2r+1 (right: axis hi,
//     anchor lo), relative_size = |F| / n in fp64 (the host's division).
//
// Ligands of fewer than 2 atoms are rejected by the host before the launch
// (status already set); ligands of more than 256 atoms (kNarrowAtoms) are
// preprocessed on the host (prep.cpp) and skipped here.  A second kernel orders
// the chunk's ligands longest-first for the search kernels' CTA order.
#include <cstdint>

#include "device_common.cuh"

namespace gdb200 {
namespace {

constexpr int kPrepWarps = 4;  // ligands per CTA

// Per warp: adjacency rows [max_n * Wm], left-fragment masks and keys of at
// most max_n rotamers.
__host__ __device__ __forceinline__ size_t smem_per_warp(int max_n) {
  const size_t Wm = (max_n + 63) / 64;
  return ((16 * Wm * max_n + 4 * static_cast<size_t>(max_n)) + 15) & ~size_t(15);
}
constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ uint64_t warp_or64(uint64_t x) {
  const unsigned lo = __reduce_or_sync(kAll, static_cast<unsigned>(x));
  const unsigned hi = __reduce_or_sync(kAll, static_cast<unsigned>(x >> 32));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ bool has(const uint64_t* s, int i) { return (s[i >> 6] >> (i & 63)) & 1ull; }

// OR of the adjacency rows of every atom in set `s` (W words) into `out`.
__device__ __forceinline__ void expand(const uint64_t* adj, int W, const uint64_t* s, uint64_t* out) {
  for (int w = 0; w < W; ++w)
    for (uint64_t b = s[w]; b; b &= b - 1) {
      const int a = 64 * w + __ffsll(static_cast<long long>(b)) - 1;
      for (int v = 0; v < W; ++v) out[v] |= adj[a * W + v];
    }
}

__global__ void __launch_bounds__(32 * kPrepWarps) prep_kernel(PrepParams q) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = q.l0 + blockIdx.x * kPrepWarps + warp;
  if (l >= q.l1) return;
  LigMeta& m = q.meta[l];
  if (m.status != 0 || m.n > kNarrowAtoms) {  // rejected on the host, or a wide ligand the host
    if (lane == 0) q.status[l] = m.status;  // preprocessed (descriptors uploaded separately)
    return;
  }
  const int n = m.n, W = m.words;
  const int b0 = q.boff[l], nb = q.boff[l + 1] - b0;
  const int Wm = (q.max_n + 63) / 64;
  unsigned char* base = smem + warp * smem_per_warp(q.max_n);
  uint64_t* adj = reinterpret_cast<uint64_t*>(base);                         // [max_n * Wm]
  uint64_t* left = adj + static_cast<size_t>(q.max_n) * Wm;                 // [max_n * Wm]
  int32_t* key = reinterpret_cast<int32_t*>(left + static_cast<size_t>(q.max_n) * Wm);  // [max_n]

  // Ligand::validate (molecule.hpp:66-89): atoms.
  bool bad = false;
  for (int i = lane; i < n; i += 32) {
    const double* p = q.xyz + 3 * static_cast<size_t>(m.atom_off + i);
    const double r = q.radii[m.atom_off + i];
    bad |= !(r > 0.0) || !isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2]);
  }
  for (int i = lane; i < n * W; i += 32) adj[i] = 0;
  __syncwarp();
  // Bonds: range and self-bonds, then the adjacency; a bit already set is a
  // duplicate bond (either orientation).
  for (int b = lane; b < nb; b += 32) {
    const int a0 = q.bonds[2 * (b0 + b)], a1 = q.bonds[2 * (b0 + b) + 1];
    if (a0 == a1 || a0 < 0 || a0 >= n || a1 < 0 || a1 >= n) {
      bad = true;
      continue;
    }
    const unsigned long long bit1 = 1ull << (a1 & 63), bit0 = 1ull << (a0 & 63);
    // Both orientations of a duplicate pair OR the same two words, so the
    // later of the two ORs on either word sees the bit.
    const unsigned long long o1 =
        atomicOr(reinterpret_cast<unsigned long long*>(adj + a0 * W + (a1 >> 6)), bit1);
    const unsigned long long o0 =
        atomicOr(reinterpret_cast<unsigned long long*>(adj + a1 * W + (a0 >> 6)), bit0);
    if ((o1 & bit1) || (o0 & bit0)) bad = true;
  }
  __syncwarp();
  if (__any_sync(kAll, bad)) {
    if (lane == 0) {
      m.status = 1;  // GD_LIG_INVALID
      m.nfrag = 0;
      q.status[l] = 1;
    }
    return;
  }

  // Connectivity (molecule.hpp:97-114): frontier BFS from atom 0, the
  // frontier's rows OR-ed across the warp.
  {
    uint64_t vis[4] = {1ull, 0, 0, 0}, fr[4] = {1ull, 0, 0, 0};
    for (;;) {
      uint64_t nx[4] = {0, 0, 0, 0};
      for (int w = 0; w < W; ++w) {
        // Lanes take the frontier's set bits round-robin.
        uint64_t bits = fr[w];
        int k = 0;
        for (; bits; bits &= bits - 1, ++k)
          if ((k & 31) == lane) {
            const int a = 64 * w + __ffsll(static_cast<long long>(bits)) - 1;
            for (int v = 0; v < W; ++v) nx[v] |= adj[a * W + v];
          }
      }
      bool any = false;
      for (int v = 0; v < W; ++v) {
        nx[v] = warp_or64(nx[v]) & ~vis[v];
        vis[v] |= nx[v];
        fr[v] = nx[v];
        any |= nx[v] != 0;
      }
      if (!any) break;
    }
    int cnt = 0;
    for (int v = 0; v < W; ++v) cnt += __popcll(vis[v]);
    if (cnt != n) {
      if (lane == 0) {
        m.status = 1;
        m.nfrag = 0;
        q.status[l] = 1;
      }
      return;
    }
  }

  // Far masks (molecule.hpp:117-140, kept as the kernels use them).
  for (int i = lane; i < n; i += 32) {
    uint64_t s1[4] = {0, 0, 0, 0}, s2[4], s3[4];
    for (int v = 0; v < W; ++v) s1[v] = adj[i * W + v];
    s1[i >> 6] |= 1ull << (i & 63);
    for (int v = 0; v < W; ++v) s2[v] = s1[v];
    uint64_t d1[4] = {0, 0, 0, 0};
    for (int v = 0; v < W; ++v) d1[v] = adj[i * W + v];
    expand(adj, W, d1, s2);  // distance <= 2
    uint64_t d2[4];
    for (int v = 0; v < W; ++v) {
      d2[v] = s2[v] & ~s1[v];
      s3[v] = s2[v];
    }
    expand(adj, W, d2, s3);  // distance <= 3
    uint64_t* row = q.far + m.far_off + static_cast<size_t>(i) * W;
    for (int v = 0; v < W; ++v) {
      const int bits = min(64, n - 64 * v);
      const uint64_t valid = bits == 64 ? ~0ull : ((1ull << bits) - 1ull);
      row[v] = ~s3[v] & valid;
    }
  }

  // Rotamers and their left fragments: a lane per rotatable bond, in rounds
  // of 32; bridges (at most n - 1 in any graph) are appended to a compact
  // list, so shared memory is sized by the atom count, not the bond count.
  int nrot = 0;
  for (int b0r = 0; b0r < nb; b0r += 32) {
    const int b = b0r + lane;
    bool bridge = false;
    int kb = 0;
    uint64_t vis[4] = {0, 0, 0, 0};
    if (b < nb && q.rot[b0 + b]) {
      const int a0 = q.bonds[2 * (b0 + b)], a1 = q.bonds[2 * (b0 + b) + 1];
      const int lo = min(a0, a1), hi = max(a0, a1);
      uint64_t fr[4] = {0, 0, 0, 0};
      vis[lo >> 6] = fr[lo >> 6] = 1ull << (lo & 63);
      for (;;) {
        uint64_t nx[4] = {0, 0, 0, 0};
        for (int w = 0; w < W; ++w)
          for (uint64_t bits = fr[w]; bits; bits &= bits - 1) {
            const int a = 64 * w + __ffsll(static_cast<long long>(bits)) - 1;
            for (int v = 0; v < W; ++v) {
              uint64_t row = adj[a * W + v];
              if (a == lo && v == (hi >> 6)) row &= ~(1ull << (hi & 63));  // the bond itself is cut
              nx[v] |= row;
            }
          }
        bool any = false;
        for (int v = 0; v < W; ++v) {
          nx[v] &= ~vis[v];
          vis[v] |= nx[v];
          fr[v] = nx[v];
          any |= nx[v] != 0;
        }
        if (!any) break;
      }
      bridge = !has(vis, hi);  // in a ring: not a bridge, not a rotamer
      kb = (lo << 8) | hi;
    }
    const unsigned bal = __ballot_sync(kAll, bridge);
    if (bridge) {
      const int at = nrot + __popc(bal & ((1u << lane) - 1u));
      key[at] = kb;
      for (int v = 0; v < W; ++v) left[at * Wm + v] = vis[v];
    }
    nrot += __popc(bal);
  }
  __syncwarp();
  for (int e = lane; e < nrot; e += 32) {
    const int kb = key[e];
    int r = 0;  // find_rotamers order: rank of the unique key (lo, hi)
    for (int c = 0; c < nrot; ++c) r += key[c] < kb;
    const int lo = kb >> 8, hi = kb & 0xff;
    int size = 0;
    for (int v = 0; v < W; ++v) size += __popcll(left[e * Wm + v]);
    for (int side = 0; side < 2; ++side) {
      const int f = m.frag_off + 2 * r + side;
      uint64_t* fm = q.fmask + m.fmask_off + static_cast<size_t>(2 * r + side) * W;
      for (int v = 0; v < W; ++v) {
        const int bits = min(64, n - 64 * v);
        const uint64_t valid = bits == 64 ? ~0ull : ((1ull << bits) - 1ull);
        fm[v] = side == 0 ? left[e * Wm + v] : (~left[e * Wm + v] & valid);
      }
      const int sz = side == 0 ? size : n - size;
      q.frel[f] = __ddiv_rn(static_cast<double>(sz), static_cast<double>(n));
      q.fax[f] = side == 0 ? lo : hi;
      q.fan[f] = side == 0 ? hi : lo;
    }
  }
  if (lane == 0) {
    m.nfrag = 2 * nrot;
    q.status[l] = 0;
  }
}

// Longest-first CTA order of ligands [l0, l1) by the cost n (4 + nfrag):
// a counting sort over 1,024 cost buckets in one CTA (the order only
// schedules; results do not depend on it).
constexpr int kOrderThreads = 1024;
constexpr int kBuckets = 1024;
__global__ void __launch_bounds__(kOrderThreads) order_kernel(const LigMeta* meta, int l0, int l1,
                                                             int32_t* order) {
  __shared__ int hist[kBuckets];
  __shared__ int scan_tmp[kOrderThreads];
  for (int k = threadIdx.x; k < kBuckets; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  auto bucket = [&](int l) {
    const LigMeta& m = meta[l];
    const int cost = m.status != 0 ? 0 : m.n * (4 + m.nfrag);
    return kBuckets - 1 - min(kBuckets - 1, cost >> 2);  // descending cost
  };
  for (int l = l0 + threadIdx.x; l < l1; l += blockDim.x) atomicAdd(&hist[bucket(l)], 1);
  __syncthreads();
  // Exclusive scan of the histogram (one bucket per thread).
  const int t = threadIdx.x;
  int v = hist[t];
  scan_tmp[t] = v;
  __syncthreads();
  for (int o = 1; o < kOrderThreads; o <<= 1) {
    const int add = t >= o ? scan_tmp[t - o] : 0;
    __syncthreads();
    scan_tmp[t] += add;
    __syncthreads();
  }
  hist[t] = scan_tmp[t] - v;
  __syncthreads();
  for (int l = l0 + threadIdx.x; l < l1; l += blockDim.x) order[l0 + atomicAdd(&hist[bucket(l)], 1)] = l;
}

}  // namespace

size_t prep_smem_per_warp(int max_n) { return smem_per_warp(max_n); }

int launch_prep(const PrepParams& q, void* stream) {
  const int cnt = q.l1 - q.l0;
  if (cnt <= 0) return 0;
  const size_t smem = kPrepWarps * prep_smem_per_warp(q.max_n);
  if (smem > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  auto s = static_cast<cudaStream_t>(stream);
  prep_kernel<<<(cnt + kPrepWarps - 1) / kPrepWarps, 32 * kPrepWarps, smem, s>>>(q);
  order_kernel<<<1, kOrderThreads, 0, s>>>(q.meta, q.l0, q.l1, q.order);
  return cudaGetLastError();
}

}  // namespace gdb200
