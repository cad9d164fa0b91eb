// See prep.hpp.  Reference: molecule.hpp:45-301.
#include "prep.hpp"

#include <algorithm>
#include <cmath>
#include <utility>

#include "geodock_b200.h"

namespace gdb200 {
namespace {

// Per-thread scratch reused across ligands: the batch path preprocesses
// every ligand once per call on the host workers, so these hot loops do
// no heap allocation after warm-up.
struct Scratch {
  std::vector<int> off, nb, bond;  // CSR adjacency in bond order (both directions)
  std::vector<int> queue, dist, disc, low;
  std::vector<std::pair<int, int>> seen;
  struct Frame {
    int atom, parent_bond, next;
  };
  std::vector<Frame> stack;
  std::vector<char> is_bridge;
  std::vector<int> rot;
};

Scratch& scratch() {
  thread_local Scratch s;
  return s;
}

// Bridges of an undirected multigraph by iterative DFS lowpoints
// (molecule.hpp:190-231).  The set of bridges does not depend on visiting
// order.
void bridges(int n, int n_bonds, Scratch& s) {
  s.is_bridge.assign(n_bonds, 0);
  s.disc.assign(n, -1);
  s.low.assign(n, 0);
  s.stack.clear();
  int timer = 0;
  for (int root = 0; root < n; ++root) {
    if (s.disc[root] >= 0) continue;
    s.disc[root] = s.low[root] = timer++;
    s.stack.push_back({root, -1, s.off[root]});
    while (!s.stack.empty()) {
      Scratch::Frame& f = s.stack.back();
      if (f.next < s.off[f.atom + 1]) {
        const int e = f.next++;
        const int nb = s.nb[e], bond = s.bond[e];
        if (bond == f.parent_bond) continue;
        if (s.disc[nb] >= 0) {
          s.low[f.atom] = std::min(s.low[f.atom], s.disc[nb]);
        } else {
          s.disc[nb] = s.low[nb] = timer++;
          s.stack.push_back({nb, bond, s.off[nb]});
        }
      } else {
        const int atom = f.atom, pb = f.parent_bond;
        s.stack.pop_back();
        if (!s.stack.empty()) {
          const int parent = s.stack.back().atom;
          s.low[parent] = std::min(s.low[parent], s.low[atom]);
          if (s.low[atom] > s.disc[parent]) s.is_bridge[pb] = 1;
        }
      }
    }
  }
}

}  // namespace

PreparedLigand prepare_ligand(const std::string& id, int n, const double* xyz, const double* radii,
                              int n_bonds, const int32_t* bonds, const uint8_t* rotatable,
                              int max_atoms) {
  PreparedLigand p;
  p.n = n;
  auto fail = [&](const std::string& what) {
    p.status = GD_LIG_INVALID;
    p.error = "ligand '" + id + "': " + what;
    return std::move(p);
  };
  // Ligand::validate (molecule.hpp:66-89), same checks in the same order.
  if (n < 2) return fail("needs at least 2 atoms");
  if (n > max_atoms) return fail("more than " + std::to_string(max_atoms) + " atoms is not supported");
  for (int i = 0; i < n; ++i) {
    if (!(radii[i] > 0.0)) return fail("non-positive radius on atom " + std::to_string(i));
    if (!(std::isfinite(xyz[3 * i]) && std::isfinite(xyz[3 * i + 1]) && std::isfinite(xyz[3 * i + 2])))
      return fail("non-finite position on atom " + std::to_string(i));
  }
  Scratch& s = scratch();
  s.seen.clear();
  for (int b = 0; b < n_bonds; ++b) {
    const int a0 = bonds[2 * b], a1 = bonds[2 * b + 1];
    if (a0 == a1) return fail("self-bond on atom " + std::to_string(a0));
    if (a0 < 0 || a0 >= n || a1 < 0 || a1 >= n) return fail("bond index out of range");
    s.seen.emplace_back(std::min(a0, a1), std::max(a0, a1));
  }
  std::sort(s.seen.begin(), s.seen.end());
  if (std::adjacent_find(s.seen.begin(), s.seen.end()) != s.seen.end()) return fail("duplicate bond");

  // Adjacency in bond order (molecule.hpp:91-96), CSR, and BFS
  // connectivity (:97-114).
  s.off.assign(n + 1, 0);
  for (int b = 0; b < n_bonds; ++b) {
    ++s.off[bonds[2 * b] + 1];
    ++s.off[bonds[2 * b + 1] + 1];
  }
  for (int i = 0; i < n; ++i) s.off[i + 1] += s.off[i];
  s.nb.resize(2 * static_cast<size_t>(n_bonds));
  s.bond.resize(2 * static_cast<size_t>(n_bonds));
  s.dist.assign(n, 0);  // fill cursor per atom
  for (int b = 0; b < n_bonds; ++b) {
    const int u = bonds[2 * b], v = bonds[2 * b + 1];
    int k = s.off[u] + s.dist[u]++;
    s.nb[k] = v, s.bond[k] = b;
    k = s.off[v] + s.dist[v]++;
    s.nb[k] = u, s.bond[k] = b;
  }
  s.queue.resize(n);
  {
    s.dist.assign(n, -1);
    int head = 0, tail = 0;
    s.queue[tail++] = 0;
    s.dist[0] = 0;
    while (head < tail) {
      const int at = s.queue[head++];
      for (int e = s.off[at]; e < s.off[at + 1]; ++e)
        if (s.dist[s.nb[e]] < 0) {
          s.dist[s.nb[e]] = 0;
          s.queue[tail++] = s.nb[e];
        }
    }
    if (tail != n) return fail("disconnected ligand");
  }

  // Capped all-pairs graph distances (molecule.hpp:117-140), kept only as
  // the kernels need them: bit j of row i set iff distance(i, j) >= 4.
  p.words = (n + 63) / 64;
  p.far_mask.assign(static_cast<size_t>(n) * p.words, 0);
  std::vector<uint64_t> near(p.words), left(p.words);
  for (int src = 0; src < n; ++src) {
    std::fill(near.begin(), near.end(), 0ull);
    s.dist.assign(n, -1);
    int head = 0, tail = 0;
    s.queue[tail++] = src;
    s.dist[src] = 0;
    while (head < tail) {
      const int at = s.queue[head++];
      near[at / 64] |= 1ull << (at % 64);
      if (s.dist[at] + 1 >= kGraphDistanceCap) continue;
      for (int e = s.off[at]; e < s.off[at + 1]; ++e)
        if (s.dist[s.nb[e]] < 0) {
          s.dist[s.nb[e]] = s.dist[at] + 1;
          s.queue[tail++] = s.nb[e];
        }
    }
    uint64_t* row = &p.far_mask[static_cast<size_t>(src) * p.words];
    for (int w = 0; w < p.words; ++w) {
      const int bits = std::min(64, n - 64 * w);
      const uint64_t valid = bits == 64 ? ~0ull : ((1ull << bits) - 1);
      row[w] = ~near[w] & valid;
    }
  }

  // Rotamers: rotatable bridges sorted by (min, max) endpoint (molecule.hpp:237-250).
  bridges(n, n_bonds, s);
  s.rot.clear();
  for (int b = 0; b < n_bonds; ++b)
    if (rotatable[b] && s.is_bridge[b]) s.rot.push_back(b);
  std::stable_sort(s.rot.begin(), s.rot.end(), [&](int x, int y) {
    const auto kx = std::minmax(bonds[2 * x], bonds[2 * x + 1]);
    const auto ky = std::minmax(bonds[2 * y], bonds[2 * y + 1]);
    return kx < ky;
  });

  // Fragments (molecule.hpp:255-301): left = what the smaller endpoint
  // still reaches with the bond cut.
  const size_t R = s.rot.size();
  p.rot_bond.reserve(R);
  p.frag_mask.reserve(2 * R * p.words);
  p.frag_axis.reserve(2 * R);
  p.frag_anchor.reserve(2 * R);
  p.frag_size.reserve(2 * R);
  p.frag_rel.reserve(2 * R);
  for (const int b : s.rot) {
    const int lo = std::min(bonds[2 * b], bonds[2 * b + 1]);
    const int hi = std::max(bonds[2 * b], bonds[2 * b + 1]);
    std::fill(left.begin(), left.end(), 0ull);
    int head = 0, tail = 0;
    s.queue[tail++] = lo;
    left[lo / 64] |= 1ull << (lo % 64);
    while (head < tail) {
      const int at = s.queue[head++];
      for (int e = s.off[at]; e < s.off[at + 1]; ++e) {
        if (s.bond[e] == b) continue;
        const int v = s.nb[e];
        if (!((left[v / 64] >> (v % 64)) & 1ull)) {
          left[v / 64] |= 1ull << (v % 64);
          s.queue[tail++] = v;
        }
      }
    }
    if ((left[hi / 64] >> (hi % 64)) & 1ull)
      return fail("rotamer bond " + std::to_string(bonds[2 * b]) + "-" +
                  std::to_string(bonds[2 * b + 1]) + " is not a bridge");
    p.rot_bond.push_back(b);
    const int left_size = tail;
    for (int side = 0; side < 2; ++side) {
      for (int w = 0; w < p.words; ++w) {
        const int bits = std::min(64, n - 64 * w);
        const uint64_t valid = bits == 64 ? ~0ull : ((1ull << bits) - 1);
        p.frag_mask.push_back(side == 0 ? left[w] : (~left[w] & valid));
      }
      const int size = side == 0 ? left_size : n - left_size;
      p.frag_size.push_back(size);
      p.frag_rel.push_back(static_cast<double>(size) / n);
      p.frag_axis.push_back(side == 0 ? lo : hi);
      p.frag_anchor.push_back(side == 0 ? hi : lo);
    }
  }
  return p;
}

}  // namespace gdb200
