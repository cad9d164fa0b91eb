// See prep.hpp.  Reference: molecule.hpp:45-301.
#include "prep.hpp"

#include <algorithm>
#include <cmath>
#include <utility>

#include "geodock_b200.h"

namespace gdb200 {
namespace {

struct Edge {
  int nb;
  int bond;
};

// Bridges of an undirected multigraph by iterative DFS lowpoints.  The set
// of bridges does not depend on visiting order.
std::vector<char> bridges(int n, const std::vector<std::vector<Edge>>& adj, int n_bonds) {
  std::vector<char> is_bridge(n_bonds, 0);
  std::vector<int> disc(n, -1), low(n, 0);
  struct Frame {
    int atom, parent_bond;
    size_t next;
  };
  std::vector<Frame> stack;
  int timer = 0;
  for (int root = 0; root < n; ++root) {
    if (disc[root] >= 0) continue;
    disc[root] = low[root] = timer++;
    stack.push_back({root, -1, 0});
    while (!stack.empty()) {
      Frame& f = stack.back();
      if (f.next < adj[f.atom].size()) {
        const Edge e = adj[f.atom][f.next++];
        if (e.bond == f.parent_bond) continue;
        if (disc[e.nb] >= 0) {
          low[f.atom] = std::min(low[f.atom], disc[e.nb]);
        } else {
          disc[e.nb] = low[e.nb] = timer++;
          stack.push_back({e.nb, e.bond, 0});
        }
      } else {
        const int atom = f.atom, pb = f.parent_bond;
        stack.pop_back();
        if (!stack.empty()) {
          const int parent = stack.back().atom;
          low[parent] = std::min(low[parent], low[atom]);
          if (low[atom] > disc[parent]) is_bridge[pb] = 1;
        }
      }
    }
  }
  return is_bridge;
}

PreparedLigand fail(PreparedLigand p, std::string msg) {
  p.status = GD_LIG_INVALID;
  p.error = std::move(msg);
  return p;
}

}  // namespace

PreparedLigand prepare_ligand(const std::string& id, int n, const double* xyz, const double* radii,
                              int n_bonds, const int32_t* bonds, const uint8_t* rotatable) {
  PreparedLigand p;
  p.n = n;
  const std::string tag = "ligand '" + id + "': ";
  // Ligand::validate (molecule.hpp:66-89), same checks in the same order.
  if (n < 2) return fail(std::move(p), tag + "needs at least 2 atoms");
  if (n > kMaxAtoms) return fail(std::move(p), tag + "more than 256 atoms is not supported");
  for (int i = 0; i < n; ++i) {
    if (!(radii[i] > 0.0)) return fail(std::move(p), tag + "non-positive radius on atom " + std::to_string(i));
    if (!(std::isfinite(xyz[3 * i]) && std::isfinite(xyz[3 * i + 1]) && std::isfinite(xyz[3 * i + 2])))
      return fail(std::move(p), tag + "non-finite position on atom " + std::to_string(i));
  }
  std::vector<std::pair<int, int>> seen;
  seen.reserve(n_bonds);
  for (int b = 0; b < n_bonds; ++b) {
    const int a0 = bonds[2 * b], a1 = bonds[2 * b + 1];
    if (a0 == a1) return fail(std::move(p), tag + "self-bond on atom " + std::to_string(a0));
    if (a0 < 0 || a0 >= n || a1 < 0 || a1 >= n) return fail(std::move(p), tag + "bond index out of range");
    seen.emplace_back(std::min(a0, a1), std::max(a0, a1));
  }
  std::sort(seen.begin(), seen.end());
  if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
    return fail(std::move(p), tag + "duplicate bond");

  // Adjacency in bond order (molecule.hpp:91-96) and BFS connectivity (:97-114).
  std::vector<std::vector<Edge>> adj(n);
  for (int b = 0; b < n_bonds; ++b) {
    adj[bonds[2 * b]].push_back({bonds[2 * b + 1], b});
    adj[bonds[2 * b + 1]].push_back({bonds[2 * b], b});
  }
  std::vector<int> queue(n);
  {
    std::vector<char> seen_atom(n, 0);
    int head = 0, tail = 0;
    queue[tail++] = 0;
    seen_atom[0] = 1;
    while (head < tail) {
      const int at = queue[head++];
      for (const Edge& e : adj[at])
        if (!seen_atom[e.nb]) {
          seen_atom[e.nb] = 1;
          queue[tail++] = e.nb;
        }
    }
    if (tail != n) return fail(std::move(p), tag + "disconnected ligand");
  }

  // Capped all-pairs graph distances (molecule.hpp:117-140).
  p.words = (n + 63) / 64;
  p.capped.assign(static_cast<size_t>(n) * n, kGraphDistanceCap);
  std::vector<int> dist(n);
  for (int src = 0; src < n; ++src) {
    std::fill(dist.begin(), dist.end(), -1);
    int head = 0, tail = 0;
    queue[tail++] = src;
    dist[src] = 0;
    p.capped[static_cast<size_t>(src) * n + src] = 0;
    while (head < tail) {
      const int at = queue[head++];
      if (dist[at] >= kGraphDistanceCap) continue;
      for (const Edge& e : adj[at])
        if (dist[e.nb] < 0) {
          dist[e.nb] = dist[at] + 1;
          p.capped[static_cast<size_t>(src) * n + e.nb] = static_cast<uint8_t>(dist[e.nb]);
          queue[tail++] = e.nb;
        }
    }
  }
  p.far_mask.assign(static_cast<size_t>(n) * p.words, 0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (p.capped[static_cast<size_t>(i) * n + j] >= kGraphDistanceCap)
        p.far_mask[static_cast<size_t>(i) * p.words + j / 64] |= 1ull << (j % 64);

  // Rotamers: rotatable bridges sorted by (min, max) endpoint (molecule.hpp:237-250).
  const std::vector<char> is_bridge = bridges(n, adj, n_bonds);
  std::vector<int> rot;
  for (int b = 0; b < n_bonds; ++b)
    if (rotatable[b] && is_bridge[b]) rot.push_back(b);
  std::stable_sort(rot.begin(), rot.end(), [&](int x, int y) {
    const auto kx = std::minmax(bonds[2 * x], bonds[2 * x + 1]);
    const auto ky = std::minmax(bonds[2 * y], bonds[2 * y + 1]);
    return kx < ky;
  });

  // Fragments (molecule.hpp:255-301).
  std::vector<char> in_left(n);
  for (int b : rot) {
    const int lo = std::min(bonds[2 * b], bonds[2 * b + 1]);
    const int hi = std::max(bonds[2 * b], bonds[2 * b + 1]);
    std::fill(in_left.begin(), in_left.end(), 0);
    int head = 0, tail = 0;
    queue[tail++] = lo;
    in_left[lo] = 1;
    while (head < tail) {
      const int at = queue[head++];
      for (const Edge& e : adj[at]) {
        if (e.bond == b) continue;
        if (!in_left[e.nb]) {
          in_left[e.nb] = 1;
          queue[tail++] = e.nb;
        }
      }
    }
    if (in_left[hi])
      return fail(std::move(p), tag + "rotamer bond " + std::to_string(bonds[2 * b]) + "-" +
                                    std::to_string(bonds[2 * b + 1]) + " is not a bridge");
    p.rot_bond.push_back(b);
    int left_size = 0;
    for (int i = 0; i < n; ++i) left_size += in_left[i];
    for (int side = 0; side < 2; ++side) {
      const size_t base = p.frag_mask.size();
      p.frag_mask.resize(base + p.words, 0);
      for (int i = 0; i < n; ++i)
        if ((in_left[i] != 0) == (side == 0)) p.frag_mask[base + i / 64] |= 1ull << (i % 64);
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
