// Synthetic BASELINE data: lattice-ellipsoid pockets and seeded random-walk
// tree ligands (BASELINE.json configs; SURVEY.md §8(d) "Generator rules").
//
// This is input production for tests and the benchmark, not the hot path.
// The reference's own generator (synthetic.hpp:71-188) builds rigid 3-6 atom
// groups in a sphere pocket; BASELINE asks for a different family, so this is
// new code.  Everything is deterministic from (base_seed, ligand id): ligand i
// is seeded with splitmix64(base ^ i), so any GPU shard regenerates its own
// ligands without communication.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "geodock_b200.h"

namespace {

uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// xoshiro256** seeded through splitmix64.
class Rng {
 public:
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (uint64_t& w : s_) w = splitmix64(x);
  }
  uint64_t next() {
    const uint64_t result = rotl(s_[1] * 5, 7) * 9;
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return result;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  // Integer in [0, n).
  int32_t below(uint32_t n) { return static_cast<int32_t>(((next() >> 32) * n) >> 32); }

 private:
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t s_[4];
};

struct V {
  double x, y, z;
};
V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V operator-(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V operator*(V a, double s) { return {a.x * s, a.y * s, a.z * s}; }
double dotv(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
V crossv(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
V unit(V a) { return a * (1.0 / std::sqrt(dotv(a, a))); }

constexpr double kPi = 3.14159265358979323846;
constexpr double kBond = 1.5;              // Angstrom, exact bond length
constexpr double kAngle = 109.5;           // degrees, +- 5
constexpr double kClearanceMargin = 1.05;  // self-avoidance margin on the bump rule

V random_unit(Rng& rng) {
  const double z = rng.uniform(-1.0, 1.0);
  const double phi = rng.uniform(0.0, 2.0 * kPi);
  const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
  return {r * std::cos(phi), r * std::sin(phi), z};
}

uint64_t ligand_seed(uint64_t base, int64_t id) {
  uint64_t x = base ^ static_cast<uint64_t>(id);
  return splitmix64(x);
}

int32_t draw_n(Rng& rng, int32_t n_lo, int32_t n_hi, int32_t fixed_n) {
  const int32_t drawn = n_lo + rng.below(static_cast<uint32_t>(std::max(0, n_hi - n_lo) + 1));
  return fixed_n > 0 ? fixed_n : drawn;
}

}  // namespace

extern "C" int gd_synth_ligand_size(uint64_t base_seed, int64_t id, int32_t n_lo, int32_t n_hi,
                                    int32_t fixed_n, int32_t* n_atoms) {
  if (n_atoms == nullptr || (fixed_n <= 0 && (n_lo < 2 || n_hi < n_lo))) return GD_ERR_INVALID;
  Rng rng(ligand_seed(base_seed, id));
  *n_atoms = draw_n(rng, n_lo, n_hi, fixed_n);
  return GD_OK;
}

extern "C" int gd_synth_ligand(uint64_t base_seed, int64_t id, int32_t n_lo, int32_t n_hi,
                               int32_t fixed_n, int32_t r_cap, int32_t fixed_r,
                               const double centre[3], double* xyz, double* radii, int32_t* bonds,
                               uint8_t* rotatable) {
  if (fixed_n <= 0 && (n_lo < 2 || n_hi < n_lo)) return -1;
  Rng rng(ligand_seed(base_seed, id));
  const int n = draw_n(rng, n_lo, n_hi, fixed_n);
  if (n < 2) return -1;
  const int r_max = std::min(r_cap, n / 4);
  const int r_drawn = rng.below(static_cast<uint32_t>(std::max(0, r_max) + 1));
  int n_rot = fixed_r >= 0 ? fixed_r : r_drawn;

  std::vector<V> pos(n);
  std::vector<double> rad(n);
  std::vector<int> parent(n, -1), degree(n, 0);
  std::vector<std::vector<int>> nbrs(n);
  std::vector<int> dist(static_cast<size_t>(n) * n, 0);  // tree graph distance

  rad[0] = rng.uniform(1.2, 1.9);
  pos[0] = {0.0, 0.0, 0.0};

  for (int a = 1; a < n; ++a) {
    rad[a] = rng.uniform(1.2, 1.9);
    V best_pos{0, 0, 0};
    int best_parent = -1;
    double best_clear = -1e300;
    for (int ptry = 0; ptry < 8 && best_clear < 0.0; ++ptry) {
      // Random walk: usually extend from the newest atom, otherwise branch
      // from a random atom with free valence (<= 4 bonds).
      int p = -1;
      if (ptry == 0 && rng.uniform() < 0.7 && degree[a - 1] < 4) {
        p = a - 1;
      } else {
        std::vector<int> open;
        for (int j = 0; j < a; ++j)
          if (degree[j] < 4) open.push_back(j);
        p = open[rng.below(static_cast<uint32_t>(open.size()))];
      }
      for (int attempt = 0; attempt < 24; ++attempt) {
        V cand;
        if (nbrs[p].empty()) {
          cand = pos[p] + random_unit(rng) * kBond;
        } else {
          const int g = nbrs[p][0];
          const V u = unit(pos[p] - pos[g]);
          V ref{1.0, 0.0, 0.0};
          for (int h : nbrs[g])
            if (h != p) {
              ref = pos[h] - pos[g];
              break;
            }
          V n1 = ref - u * dotv(ref, u);
          if (dotv(n1, n1) < 1e-12) {
            ref = std::fabs(u.x) < 0.9 ? V{1.0, 0.0, 0.0} : V{0.0, 1.0, 0.0};
            n1 = ref - u * dotv(ref, u);
          }
          n1 = unit(n1);
          const V n2 = crossv(u, n1);
          const double theta = (kAngle + rng.uniform(-5.0, 5.0)) * (kPi / 180.0);
          const double phi = rng.uniform(0.0, 2.0 * kPi);
          const V b = u * (-std::cos(theta)) +
                      (n1 * std::cos(phi) + n2 * std::sin(phi)) * std::sin(theta);
          cand = pos[p] + b * kBond;
        }
        // Self-avoidance under the reference bump rule (geometry.hpp:199-213):
        // pairs at graph distance >= 4 keep 0.8*(ri+rj) (plus a margin).
        double clear = 1e300;
        for (int j = 0; j < a; ++j) {
          const int gd = dist[static_cast<size_t>(p) * n + j] + 1;
          if (gd < 4) continue;
          const V d = cand - pos[j];
          clear = std::min(clear, std::sqrt(dotv(d, d)) -
                                      0.8 * kClearanceMargin * (rad[a] + rad[j]));
        }
        if (clear > best_clear) {
          best_clear = clear;
          best_pos = cand;
          best_parent = p;
        }
        if (clear >= 0.0) break;
      }
    }
    const int p = best_parent;
    parent[a] = p;
    pos[a] = best_pos;
    ++degree[p];
    ++degree[a];
    nbrs[p].push_back(a);
    nbrs[a].push_back(p);
    for (int j = 0; j < a; ++j) {
      const int d = dist[static_cast<size_t>(p) * n + j] + 1;
      dist[static_cast<size_t>(a) * n + j] = d;
      dist[static_cast<size_t>(j) * n + a] = d;
    }
  }

  // Rotatable bonds: uniform among non-terminal bonds (both ends degree >= 2).
  // Trees have no rings, so every chosen bond is a rotamer (molecule.hpp:237-250).
  std::vector<int> eligible;
  for (int a = 1; a < n; ++a)
    if (degree[a] >= 2 && degree[parent[a]] >= 2) eligible.push_back(a);
  n_rot = std::min<int>(n_rot, static_cast<int>(eligible.size()));
  for (int i = 0; i < n_rot; ++i) {
    const int j = i + rng.below(static_cast<uint32_t>(eligible.size() - i));
    std::swap(eligible[i], eligible[j]);
  }
  std::vector<uint8_t> rot(n, 0);
  for (int i = 0; i < n_rot; ++i) rot[eligible[i]] = 1;

  // Move the centroid (atom-order mean) onto the requested centre.
  V mean{0.0, 0.0, 0.0};
  for (int a = 0; a < n; ++a) mean = mean + pos[a];
  mean = {mean.x / n, mean.y / n, mean.z / n};
  const V c = centre ? V{centre[0], centre[1], centre[2]} : V{0.0, 0.0, 0.0};
  for (int a = 0; a < n; ++a) {
    const V q = (pos[a] - mean) + c;
    xyz[3 * a + 0] = q.x;
    xyz[3 * a + 1] = q.y;
    xyz[3 * a + 2] = q.z;
    radii[a] = rad[a];
  }
  for (int a = 1; a < n; ++a) {
    bonds[2 * (a - 1) + 0] = parent[a];
    bonds[2 * (a - 1) + 1] = a;
    rotatable[a - 1] = rot[a];
  }
  return n_rot;
}

extern "C" int32_t gd_synth_pocket(double a, double b, double c, double spacing, double rough_max,
                                   uint64_t seed, double* xyz, int32_t cap) {
  if (!(a > 0 && b > 0 && c > 0 && spacing > 0)) return -1;
  const int ia = static_cast<int>(std::floor(a / spacing));
  const int ib = static_cast<int>(std::floor(b / spacing));
  const int ic = static_cast<int>(std::floor(c / spacing));
  std::vector<V> pts;
  std::vector<double> rho;
  for (int i = -ia; i <= ia; ++i)
    for (int j = -ib; j <= ib; ++j)
      for (int k = -ic; k <= ic; ++k) {
        const double x = i * spacing, y = j * spacing, z = k * spacing;
        const double q = (x * x) / (a * a) + (y * y) / (b * b) + (z * z) / (c * c);
        if (q <= 1.0) {
          pts.push_back({x, y, z});
          rho.push_back(std::sqrt(q));
        }
      }
  if (rough_max > 0.0 && !pts.empty()) {
    // Surface roughness: drop the outermost U(0, rough_max) fraction of
    // points, outermost judged by ellipsoidal radius plus seeded noise.
    uint64_t s = seed;
    Rng rng(splitmix64(s));
    const double frac = rng.uniform(0.0, rough_max);
    const size_t drop = static_cast<size_t>(std::llround(frac * static_cast<double>(pts.size())));
    std::vector<double> key(pts.size());
    for (size_t p = 0; p < pts.size(); ++p) key[p] = rho[p] + 0.35 * rng.uniform();
    std::vector<size_t> order(pts.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t x, size_t y) { return key[x] > key[y]; });
    std::vector<char> keep(pts.size(), 1);
    for (size_t r = 0; r < drop && r + 1 < pts.size(); ++r) keep[order[r]] = 0;
    std::vector<V> kept;
    for (size_t p = 0; p < pts.size(); ++p)
      if (keep[p]) kept.push_back(pts[p]);
    pts.swap(kept);
  }
  const int32_t count = static_cast<int32_t>(pts.size());
  if (xyz != nullptr)
    for (int32_t p = 0; p < std::min(count, cap); ++p) {
      xyz[3 * p + 0] = pts[p].x;
      xyz[3 * p + 1] = pts[p].y;
      xyz[3 * p + 2] = pts[p].z;
    }
  return count;
}
