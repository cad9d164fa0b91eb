// geodock_b200/geodock.hpp -- C++ drop-in for the reference GeoDock-MA API.
//
// Mirrors the public surface a caller of /root/reference/proj/include/geodock
// uses on the pose-search path, with the same names, argument meaning and
// error behaviour, executed on a B200 through the C-ABI in geodock_b200.h:
//
//   reference (header)                         here
//   -----------------------------------------  ---------------------------------
//   Vec3 / Atom / Bond (vec3.hpp, molecule.hpp) same value types
//   Ligand(id, atoms, bonds)  molecule.hpp:45  same validation + messages
//   find_rotamers / grow_fragments             gd_ligand_graph / host BFS
//     (molecule.hpp:237-301)
//   Pocket(id, points)        molecule.hpp:152 same; stages itself on the GPU lazily
//   PocketIndex(pocket)       geometry.hpp:47  accepted, no-op (the GPU always
//                                              uses its exact voxel index)
//   overlap_score             geometry.hpp:140 gd_overlap_score_batch
//   rotate_fragment(_into)    geometry.hpp:161 gd_rotate_fragment_batch
//   check_bumps               geometry.hpp:199 gd_check_bumps_batch
//   KnobConfig::validate      kernel.hpp:28    same messages
//   optimal_tile_size         kernel.hpp:62    gd_optimal_tile_size
//   SearchCounters, FragmentSearchResult (kernel.hpp:77-85)   same types
//   optimize_fragment_flat    kernel.hpp:125   gd_optimize_fragment_batch
//   optimize_fragment_refined kernel.hpp:150   gd_optimize_fragment_batch
//   match_probes_shape        kernel.hpp:205   gd_dock_batch (rigid_step 0, K 1)
//   screen                    screening.hpp:96 streamed: bounded chunks through
//                                              gd_multi_dock_batch on every GPU
//   top1pct_mean_score        screening.hpp:78 same
//   overlap_degradation       screening.hpp:190 same
//   (new) dock_batch                           the north-star batch path:
//                                              rigid sweep + top-K + restarts
//   analysis.hpp (rotation profiles, peaks)    geodock_b200/analysis.hpp
//   perf_model.hpp + autotuner.hpp (planner)   geodock_b200/planner.hpp
//   formats.hpp (files, reports, CSVs)         geodock_b200/formats.hpp
//
// Results are bit-identical to the reference.  Link with
// paper_1901_06363_b200/libgeodock_b200.so.  The batch calls (screen,
// dock_batch, match_probes_shape) run on every visible GPU through
// gd_multi; the environment variable GEODOCK_B200_DEVICES ("0,2,3") or the
// macro GEODOCK_B200_DEVICE (one GPU) restricts them.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <queue>
#include <thread>
#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <variant>
#include <vector>

#include "geodock_b200.h"

namespace geodock {

// ---- error.hpp -----------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

/// Parse failures carry the 1-based line (error.hpp:19-27).
class ParseError : public Error {
 public:
  ParseError(const std::string& what, int line)
      : Error(what + " at line " + std::to_string(line)), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};

// ---- vec3.hpp (value type and host helpers; the hot path runs on the GPU) -----
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  constexpr Vec3() = default;
  constexpr Vec3(double px, double py, double pz) : x(px), y(py), z(pz) {}
  constexpr Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  constexpr Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  constexpr Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  constexpr Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
  constexpr Vec3& operator+=(const Vec3& o) {
    x += o.x;
    y += o.y;
    z += o.z;
    return *this;
  }
  constexpr bool operator==(const Vec3& o) const { return x == o.x && y == o.y && z == o.z; }
};
// Same expression trees as vec3.hpp:28-46 (left-associative sums).
constexpr double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
constexpr Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
constexpr double norm_sq(const Vec3& a) { return dot(a, a); }
inline double norm(const Vec3& a) { return std::sqrt(norm_sq(a)); }
constexpr double distance_sq(const Vec3& a, const Vec3& b) { return norm_sq(a - b); }
inline double distance(const Vec3& a, const Vec3& b) { return std::sqrt(distance_sq(a, b)); }
inline bool is_finite(const Vec3& a) { return std::isfinite(a.x) && std::isfinite(a.y) && std::isfinite(a.z); }

// ---- molecule.hpp --------------------------------------------------------
struct Atom {
  int index = 0;
  Vec3 position;
  double radius = 0.0;
};

struct Bond {
  int a = 0;
  int b = 0;
  bool rotatable = false;
};

struct SkippedRecord {
  std::string id;
  std::string reason;
  friend bool operator==(const SkippedRecord&, const SkippedRecord&) = default;
};

namespace detail {
inline bool finite(const Vec3& v) { return std::isfinite(v.x) && std::isfinite(v.y) && std::isfinite(v.z); }
}  // namespace detail

/// Flexible molecule, validated like the reference (molecule.hpp:66-115).
/// Graph preprocessing (capped distances, rotamers, fragments) happens in the
/// native library when the ligand is docked.
class Ligand {
 public:
  Ligand(std::string id, std::vector<Atom> atoms, std::vector<Bond> bonds)
      : id_(std::move(id)), atoms_(std::move(atoms)), bonds_(std::move(bonds)) {
    const int n = static_cast<int>(atoms_.size());
    const std::string tag = "ligand '" + id_ + "': ";
    if (n < 2) throw Error(tag + "needs at least 2 atoms");
    for (int i = 0; i < n; ++i) {
      if (atoms_[i].index != i) throw Error(tag + "atom index mismatch at position " + std::to_string(i));
      if (!(atoms_[i].radius > 0.0)) throw Error(tag + "non-positive radius on atom " + std::to_string(i));
      if (!detail::finite(atoms_[i].position))
        throw Error(tag + "non-finite position on atom " + std::to_string(i));
    }
    std::vector<std::pair<int, int>> seen;
    for (const Bond& b : bonds_) {
      if (b.a == b.b) throw Error(tag + "self-bond on atom " + std::to_string(b.a));
      if (b.a < 0 || b.a >= n || b.b < 0 || b.b >= n) throw Error(tag + "bond index out of range");
      seen.emplace_back(std::min(b.a, b.b), std::max(b.a, b.b));
    }
    std::sort(seen.begin(), seen.end());
    if (std::adjacent_find(seen.begin(), seen.end()) != seen.end()) throw Error(tag + "duplicate bond");
    // Connectivity (molecule.hpp:97-114).
    std::vector<std::vector<int>> adj(n);
    for (const Bond& b : bonds_) {
      adj[b.a].push_back(b.b);
      adj[b.b].push_back(b.a);
    }
    std::vector<char> vis(n, 0);
    std::vector<int> q{0};
    vis[0] = 1;
    for (size_t h = 0; h < q.size(); ++h)
      for (int nb : adj[q[h]])
        if (!vis[nb]) vis[nb] = 1, q.push_back(nb);
    if (static_cast<int>(q.size()) != n) throw Error(tag + "disconnected ligand");
  }
  static constexpr int kGraphDistanceCap = 4;  // molecule.hpp:43

  const std::string& id() const { return id_; }
  const std::vector<Atom>& atoms() const { return atoms_; }
  const std::vector<Bond>& bonds() const { return bonds_; }
  int atom_count() const { return static_cast<int>(atoms_.size()); }
  /// (neighbour, bond index) pairs in bond order (molecule.hpp:58, :91-96).
  const std::vector<std::pair<int, int>>& neighbors(int atom) const { return graph().adj[atom]; }
  /// Bond-graph distance capped at kGraphDistanceCap (molecule.hpp:61-63).
  int graph_distance_capped(int i, int j) const {
    return graph().capped[static_cast<size_t>(i) * atoms_.size() + j];
  }

 private:
  // The host graph (adjacency, capped BFS distances; molecule.hpp:91-140)
  // is built on first use: the GPU batch path preprocesses ligands in the
  // native library and never needs it.  Copies share it (a Ligand is
  // immutable).
  struct Graph {
    std::once_flag once;
    std::vector<std::vector<std::pair<int, int>>> adj;
    std::vector<uint8_t> capped;
  };
  const Graph& graph() const {
    std::call_once(graph_->once, [this] {
      const size_t n = atoms_.size();
      Graph& g = *graph_;
      g.adj.assign(n, {});
      for (int bi = 0; bi < static_cast<int>(bonds_.size()); ++bi) {
        g.adj[bonds_[bi].a].emplace_back(bonds_[bi].b, bi);
        g.adj[bonds_[bi].b].emplace_back(bonds_[bi].a, bi);
      }
      g.capped.assign(n * n, static_cast<uint8_t>(kGraphDistanceCap));
      std::vector<int> dist(n);
      for (size_t src = 0; src < n; ++src) {
        std::fill(dist.begin(), dist.end(), -1);
        std::queue<int> q;
        q.push(static_cast<int>(src));
        dist[src] = 0;
        g.capped[src * n + src] = 0;
        while (!q.empty()) {
          const int at = q.front();
          q.pop();
          if (dist[at] >= kGraphDistanceCap) continue;
          for (const auto& [nb, bond] : g.adj[at])
            if (dist[nb] < 0) {
              dist[nb] = dist[at] + 1;
              g.capped[src * n + nb] = static_cast<uint8_t>(dist[nb]);
              q.push(nb);
            }
        }
      }
    });
    return *graph_;
  }
  std::string id_;
  std::vector<Atom> atoms_;
  std::vector<Bond> bonds_;
  std::shared_ptr<Graph> graph_ = std::make_shared<Graph>();
};

/// A rotatable bridge bond (molecule.hpp:167-171).
struct Rotamer {
  Bond bond;
  int bond_index = 0;  // position in Ligand::bonds()
};

enum class Side { left, right };

/// One side of a cut rotamer bond (molecule.hpp:175-185); the left fragment
/// holds the bond endpoint with the smaller index.
struct Fragment {
  Rotamer rotamer;
  Side side = Side::left;
  std::vector<int> atom_indices;  // ascending
  std::vector<char> membership;   // per-atom flag, size == atom count
  double relative_size = 0.0;     // |atom_indices| / atom count
  int axis_atom = 0;              // bond endpoint inside this fragment
  int anchor_atom = 0;            // bond endpoint on the other side
};

/// Rotatable bridge bonds ordered by (min endpoint, max endpoint)
/// (molecule.hpp:237-250), from the native preprocessing the batch path
/// uses (gd_ligand_graph).
inline std::vector<Rotamer> find_rotamers(const Ligand& ligand) {
  const int n = ligand.atom_count();
  const int nb = static_cast<int>(ligand.bonds().size());
  std::vector<double> xyz, radii;
  std::vector<int32_t> bonds, rb(std::max(nb, 1));
  std::vector<uint8_t> rot;
  for (const Atom& a : ligand.atoms()) {
    xyz.insert(xyz.end(), {a.position.x, a.position.y, a.position.z});
    radii.push_back(a.radius);
  }
  for (const Bond& b : ligand.bonds()) {
    bonds.insert(bonds.end(), {b.a, b.b});
    rot.push_back(b.rotatable ? 1 : 0);
  }
  int32_t count = 0;
  char msg[256] = {0};
  if (gd_ligand_graph(n, xyz.data(), radii.data(), nb, bonds.data(), rot.data(), &count, rb.data(),
                      nullptr, msg, sizeof msg) != GD_LIG_OK)
    throw Error(msg);
  std::vector<Rotamer> out;
  for (int r = 0; r < count; ++r) out.push_back({ligand.bonds()[rb[r]], rb[r]});
  return out;
}

/// The two fragments a rotamer bond splits off (molecule.hpp:255-301): the
/// left one is what the smaller endpoint still reaches once the bond is cut.
inline std::pair<Fragment, Fragment> grow_fragments(const Ligand& ligand, const Rotamer& rotamer) {
  const int n = ligand.atom_count();
  const int lo = std::min(rotamer.bond.a, rotamer.bond.b);
  const int hi = std::max(rotamer.bond.a, rotamer.bond.b);
  std::vector<std::vector<std::pair<int, int>>> adj(n);  // (neighbour, bond index)
  for (int bi = 0; bi < static_cast<int>(ligand.bonds().size()); ++bi) {
    const Bond& b = ligand.bonds()[bi];
    adj[b.a].push_back({b.b, bi});
    adj[b.b].push_back({b.a, bi});
  }
  std::vector<char> reach(n, 0);
  std::vector<int> frontier{lo};
  reach[lo] = 1;
  for (size_t h = 0; h < frontier.size(); ++h)
    for (const auto& [nb, bi] : adj[frontier[h]])
      if (bi != rotamer.bond_index && !reach[nb]) reach[nb] = 1, frontier.push_back(nb);
  if (reach[hi])
    throw Error("ligand '" + ligand.id() + "': rotamer bond " + std::to_string(rotamer.bond.a) + "-" +
                std::to_string(rotamer.bond.b) + " is not a bridge");
  std::pair<Fragment, Fragment> out;
  Fragment* sides[2] = {&out.first, &out.second};
  for (int s = 0; s < 2; ++s) {
    Fragment& f = *sides[s];
    f.rotamer = rotamer;
    f.side = s == 0 ? Side::left : Side::right;
    f.membership.assign(n, 0);
    for (int i = 0; i < n; ++i)
      if ((reach[i] != 0) == (s == 0)) {
        f.atom_indices.push_back(i);
        f.membership[i] = 1;
      }
    f.relative_size = static_cast<double>(f.atom_indices.size()) / n;
    f.axis_atom = s == 0 ? lo : hi;
    f.anchor_atom = s == 0 ? hi : lo;
  }
  return out;
}

namespace detail {

/// The process's GPUs (gd_multi over every visible device, or the
/// GEODOCK_B200_DEVICES list / GEODOCK_B200_DEVICE macro), shared by all
/// calls.  Batch calls use every device; fine-grained calls use the first.
class Device {
 public:
  static Device& get() {
    static Device d;
    return d;
  }
  gd_multi* multi() { return multi_; }
  gd_ctx* ctx() { return gd_multi_context(multi_, 0); }
  int size() const { return gd_multi_size(multi_); }
  std::mutex& mu() { return mu_; }
  uint64_t staged_serial = 0;

  ~Device() {
    if (multi_) gd_multi_destroy(multi_);
  }

 private:
  Device() {
    std::vector<int32_t> devs;
#ifdef GEODOCK_B200_DEVICE
    devs.push_back(GEODOCK_B200_DEVICE);
#endif
    if (const char* e = std::getenv("GEODOCK_B200_DEVICES")) {
      devs.clear();
      std::string list(e);
      for (size_t at = 0; at < list.size();) {
        const size_t comma = std::min(list.find(',', at), list.size());
        if (comma > at) devs.push_back(std::stoi(list.substr(at, comma - at)));
        at = comma + 1;
      }
    }
    const int rc = devs.empty() ? gd_multi_create(nullptr, 0, &multi_)
                                : gd_multi_create(devs.data(), static_cast<int32_t>(devs.size()), &multi_);
    if (rc != GD_OK) throw Error(std::string("geodock_b200: ") + gd_multi_last_error(nullptr));
  }
  gd_multi* multi_ = nullptr;
  std::mutex mu_;
};

/// Error of the last failed call on the first device's context.
inline void check(int rc) {
  if (rc != GD_OK) throw Error(gd_last_error(Device::get().ctx()));
}
/// Error of the last failed multi-device call.
inline void check_multi(int rc) {
  if (rc != GD_OK) throw Error(gd_multi_last_error(Device::get().multi()));
}

inline uint64_t next_serial() {
  static std::atomic<uint64_t> s{1};
  return s++;
}

}  // namespace detail

/// Rigid binding site (molecule.hpp:150-165).  Staged on the GPU on first
/// use; every copy keeps its own identity for staging.
class Pocket {
 public:
  Pocket(std::string id, std::vector<Vec3> points)
      : id_(std::move(id)), points_(std::move(points)), serial_(detail::next_serial()) {
    if (points_.empty()) throw Error("pocket '" + id_ + "': needs at least 1 point");
    for (const Vec3& p : points_)
      if (!detail::finite(p)) throw Error("pocket '" + id_ + "': non-finite point");
  }
  const std::string& id() const { return id_; }
  const std::vector<Vec3>& points() const { return points_; }

  /// Makes this pocket the staged pocket of every device (caller holds the
  /// lock).  The devices cache recent pockets by their coordinates, so
  /// alternating pockets re-stages without rebuilding indexes.
  void stage(detail::Device& d) const {
    if (d.staged_serial == serial_) return;
    std::vector<double> xyz;
    xyz.reserve(points_.size() * 3);
    for (const Vec3& p : points_) xyz.insert(xyz.end(), {p.x, p.y, p.z});
    detail::check_multi(gd_multi_set_pocket(d.multi(), xyz.data(), static_cast<int32_t>(points_.size())));
    d.staged_serial = serial_;
  }

 private:
  std::string id_;
  std::vector<Vec3> points_;
  uint64_t serial_;
};

/// Accepted for signature compatibility (geometry.hpp:47); the GPU path
/// always uses its own exact voxel index, which gives the same minima.
class PocketIndex {
 public:
  explicit PocketIndex(const Pocket&) {}
};

// ---- geometry.hpp --------------------------------------------------------
struct Pose {
  std::vector<Vec3> positions;
};

inline Pose make_initial_pose(const Ligand& ligand) {
  Pose pose;
  pose.positions.reserve(ligand.atoms().size());
  for (const Atom& a : ligand.atoms()) pose.positions.push_back(a.position);
  return pose;
}

inline double overlap_score(const Pose& pose, const Pocket& pocket, const PocketIndex* = nullptr) {
  if (pose.positions.empty()) throw Error("overlap_score: empty pose");
  auto& d = detail::Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  pocket.stage(d);
  std::vector<double> xyz;
  for (const Vec3& p : pose.positions) xyz.insert(xyz.end(), {p.x, p.y, p.z});
  double out = 0.0;
  detail::check(gd_overlap_score_batch(d.ctx(), xyz.data(), static_cast<int32_t>(pose.positions.size()),
                                       1, 0u, &out));
  return out;
}

namespace detail {

struct Packed {
  std::vector<int32_t> atom_off{0}, bond_off{0}, bonds;
  std::vector<double> xyz, radii;
  std::vector<uint8_t> rot;
  void add(const Ligand& l, const Pose* pose) {
    for (int i = 0; i < l.atom_count(); ++i) {
      const Vec3& p = pose ? pose->positions[i] : l.atoms()[i].position;
      xyz.insert(xyz.end(), {p.x, p.y, p.z});
      radii.push_back(l.atoms()[i].radius);
    }
    for (const Bond& b : l.bonds()) {
      bonds.insert(bonds.end(), {b.a, b.b});
      rot.push_back(b.rotatable ? 1 : 0);
    }
    atom_off.push_back(static_cast<int32_t>(radii.size()));
    bond_off.push_back(static_cast<int32_t>(rot.size()));
  }
  gd_ligand_batch view() const {
    return gd_ligand_batch{static_cast<int32_t>(atom_off.size() - 1), atom_off.data(), xyz.data(),
                           radii.data(), bond_off.data(), bonds.data(), rot.data()};
  }
};

struct Results {
  std::vector<int32_t> orientation, rank, k_eff, status;
  std::vector<double> rigid, final_score, pose;
  std::vector<int64_t> evals, checks, scored;
  gd_result view() {
    return gd_result{orientation.data(), rank.data(),   rigid.data(),  final_score.data(),
                     evals.data(),       checks.data(), pose.empty() ? nullptr : pose.data(),
                     k_eff.data(),       scored.data(), status.data()};
  }
  Results(size_t L, size_t K, size_t atoms, bool poses)
      : orientation(L * K), rank(L * K), k_eff(L), status(L), rigid(L * K), final_score(L * K),
        pose(poses ? atoms * K * 3 : 0), evals(L * K), checks(L * K), scored(L) {}
};


// One ligand with one fragment, staged for the fine-grained entry points.
struct OneFragment {
  Packed pk;
  std::vector<uint8_t> mem;
  int32_t axis = 0, anchor = 0;
  OneFragment(const Ligand& l, const Pose& pose, const Fragment& f) : axis(f.axis_atom), anchor(f.anchor_atom) {
    pk.add(l, &pose);
    mem.assign(f.membership.begin(), f.membership.end());
    mem.resize(l.atom_count(), 0);
  }
  gd_fragment_set set() const { return gd_fragment_set{mem.data(), &axis, &anchor}; }
};

// The validation text of a skipped ligand under its own id (the library
// names ligands by batch position).
inline std::string ligand_error_text(const char* raw, int32_t pos, const std::string& id) {
  std::string m(raw);
  const std::string pre = "ligand '" + std::to_string(pos) + "': ";
  if (m.rfind(pre, 0) == 0) m = "ligand '" + id + "': " + m.substr(pre.size());
  return m.empty() ? "ligand '" + id + "': invalid" : m;
}

// Rethrows a per-ligand status of a fine-grained call as geodock::Error.
inline void raise_status(int32_t st, const Ligand& l) {
  if (st == GD_LIG_OK) return;
  if (st == GD_LIG_DEGENERATE) throw Error("rotate_fragment: degenerate rotation axis");
  char buf[512] = {0};
  gd_ligand_error(Device::get().ctx(), 0, buf, sizeof buf);
  throw Error(ligand_error_text(buf, 0, l.id()));
}

}  // namespace detail

/// rotate_fragment_into (geometry.hpp:161-186), on the GPU: the fragment's
/// atoms rotated by `angle_deg` (any angle; cos/sin from the host libm as
/// the reference evaluates them) about axis_atom -> anchor_atom, the rest
/// copied; angle 0 is the exact identity.
inline void rotate_fragment_into(const Pose& pose, const Ligand& ligand, const Fragment& fragment,
                                 double angle_deg, Pose& out) {
  if (pose.positions.size() != static_cast<size_t>(ligand.atom_count()))
    throw Error("rotate_fragment: pose/ligand size mismatch");
  const detail::OneFragment one(ligand, pose, fragment);
  const gd_ligand_batch b = one.pk.view();
  const gd_fragment_set fs = one.set();
  std::vector<double> xyz(3 * pose.positions.size());
  int32_t status = 0;
  auto& d = detail::Device::get();
  {
    std::lock_guard<std::mutex> lock(d.mu());
    detail::check(gd_rotate_fragment_batch(d.ctx(), &b, &fs, &angle_deg, xyz.data(), &status));
    detail::raise_status(status, ligand);
  }
  out.positions.resize(pose.positions.size());
  for (size_t i = 0; i < pose.positions.size(); ++i) out.positions[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
}

inline Pose rotate_fragment(const Pose& pose, const Ligand& ligand, const Fragment& fragment,
                            double angle_deg) {
  Pose out;
  rotate_fragment_into(pose, ligand, fragment, angle_deg, out);
  return out;
}

/// check_bumps (geometry.hpp:199-213), on the GPU: false iff a fragment
/// atom and a non-fragment atom at capped graph distance >= 4 sit closer
/// than 0.8 times the sum of their radii.
inline bool check_bumps(const Pose& pose, const Ligand& ligand, const Fragment& fragment) {
  if (pose.positions.size() != static_cast<size_t>(ligand.atom_count()))
    throw Error("check_bumps: pose/ligand size mismatch");
  const detail::OneFragment one(ligand, pose, fragment);
  const gd_ligand_batch b = one.pk.view();
  const gd_fragment_set fs = one.set();
  uint8_t feasible = 0;
  int32_t status = 0;
  auto& d = detail::Device::get();
  std::lock_guard<std::mutex> lock(d.mu());
  detail::check(gd_check_bumps_batch(d.ctx(), &b, &fs, &feasible, &status));
  detail::raise_status(status, ligand);
  return feasible != 0;
}

// ---- kernel.hpp ----------------------------------------------------------
struct KnobConfig {
  int high_precision_step = 1;
  int low_precision_step = 45;
  double threshold = 0.0;
  int repetitions = 3;
  bool enable_refinement = false;

  void validate() const {
    gd_knobs k = to_c(0, 1);
    char msg[256];
    if (gd_validate_knobs(&k, msg, sizeof msg) != GD_OK) throw Error(msg);
  }
  gd_knobs to_c(int rigid_step, int top_k) const {
    return gd_knobs{high_precision_step, low_precision_step, threshold, repetitions,
                    enable_refinement ? 1 : 0, rigid_step, top_k, 0u};
  }
  friend bool operator==(const KnobConfig&, const KnobConfig&) = default;
};

/// Canonical knob order (kernel.hpp:44-48): the planner's final tie-break.
inline bool knob_order_less(const KnobConfig& a, const KnobConfig& b) {
  return std::tie(a.high_precision_step, a.low_precision_step, a.threshold, a.repetitions,
                  a.enable_refinement) < std::tie(b.high_precision_step, b.low_precision_step,
                                                  b.threshold, b.repetitions, b.enable_refinement);
}

struct PoseResult {
  std::string ligand_id;
  double score = 0.0;
  Pose final_pose;
  long evaluations = 0;
  long feasibility_checks = 0;
  double wall_time_seconds = 0.0;
};

inline int optimal_tile_size(int high_precision_step) {
  if (high_precision_step < 1) throw Error("optimal_tile_size: step must be >= 1");
  return gd_optimal_tile_size(high_precision_step);
}

struct SearchCounters {
  long evaluations = 0;
  long feasibility_checks = 0;
};

struct FragmentSearchResult {
  int best_angle = 0;
  double best_score = 0.0;
};

namespace detail {
inline FragmentSearchResult optimize_fragment(Pose& pose, const Ligand& ligand, const Fragment& fragment,
                                              const Pocket& pocket, int step, bool refined,
                                              SearchCounters* counters, const double* entry) {
  const detail::OneFragment one(ligand, pose, fragment);
  const gd_ligand_batch b = one.pk.view();
  const gd_fragment_set fs = one.set();
  int32_t angle = 0, status = 0;
  double score = 0.0;
  int64_t evals = 0, checks = 0;
  std::vector<double> xyz(3 * pose.positions.size());
  auto& d = detail::Device::get();
  {
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    detail::check(gd_optimize_fragment_batch(d.ctx(), &b, &fs, step, refined ? 1 : 0, entry, &angle,
                                             &score, &evals, &checks, xyz.data(), &status));
    detail::raise_status(status, ligand);
  }
  for (size_t i = 0; i < pose.positions.size(); ++i) pose.positions[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  if (counters != nullptr) {
    counters->evaluations += evals;
    counters->feasibility_checks += checks;
  }
  return FragmentSearchResult{angle, score};
}
}  // namespace detail

/// optimize_fragment_flat (kernel.hpp:125-143), on the GPU: angles 0, step,
/// ..., 360-step from `pose`; the first feasible best wins; `pose` is
/// committed to it.
inline FragmentSearchResult optimize_fragment_flat(Pose& pose, const Ligand& ligand, const Fragment& fragment,
                                                   const Pocket& pocket, int step,
                                                   SearchCounters* counters = nullptr,
                                                   const PocketIndex* = nullptr) {
  if (step < 1 || 360 % step != 0) throw Error("optimize_fragment_flat: step must divide 360");
  if (pose.positions.size() != static_cast<size_t>(ligand.atom_count()))
    throw Error("rotate_fragment: pose/ligand size mismatch");
  return detail::optimize_fragment(pose, ligand, fragment, pocket, step, false, counters, nullptr);
}

/// optimize_fragment_refined (kernel.hpp:150-198), on the GPU: tile centres,
/// then the winning tile at `high_precision_step`; the entry pose (score
/// `entry_score`, else its overlap score) is kept only if strictly better.
inline FragmentSearchResult optimize_fragment_refined(Pose& pose, const Ligand& ligand,
                                                      const Fragment& fragment, const Pocket& pocket,
                                                      int high_precision_step,
                                                      SearchCounters* counters = nullptr,
                                                      std::optional<double> entry_score = std::nullopt,
                                                      const PocketIndex* = nullptr) {
  if (high_precision_step < 1 || 360 % high_precision_step != 0)
    throw Error("optimize_fragment_refined: step must divide 360");
  if (pose.positions.size() != static_cast<size_t>(ligand.atom_count()))
    throw Error("rotate_fragment: pose/ligand size mismatch");
  const double e = entry_score ? *entry_score : 0.0;
  return detail::optimize_fragment(pose, ligand, fragment, pocket, high_precision_step, true, counters,
                                   entry_score ? &e : nullptr);
}


/// Pose-optimization kernel (kernel.hpp:205-248), on the GPU.
inline PoseResult match_probes_shape(const Ligand& ligand, const Pocket& pocket,
                                     const Pose& initial_pose, const KnobConfig& config,
                                     const PocketIndex* = nullptr) {
  config.validate();
  if (initial_pose.positions.size() != static_cast<size_t>(ligand.atom_count()))
    throw Error("match_probes_shape: pose/ligand size mismatch");
  const auto t0 = std::chrono::steady_clock::now();
  detail::Packed pk;
  pk.add(ligand, &initial_pose);
  detail::Results res(1, 1, ligand.atom_count(), true);
  const gd_ligand_batch b = pk.view();
  const gd_knobs k = config.to_c(0, 1);
  gd_result r = res.view();
  auto& d = detail::Device::get();
  {
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    detail::check(gd_dock_batch(d.ctx(), &b, &k, &r));
    detail::raise_status(res.status[0], ligand);
  }
  PoseResult out;
  out.ligand_id = ligand.id();
  out.score = res.final_score[0];
  out.evaluations = static_cast<long>(res.evals[0]);
  out.feasibility_checks = static_cast<long>(res.checks[0]);
  for (int i = 0; i < ligand.atom_count(); ++i)
    out.final_pose.positions.push_back({res.pose[3 * i], res.pose[3 * i + 1], res.pose[3 * i + 2]});
  out.wall_time_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

// ---- screening.hpp -------------------------------------------------------
struct LigandResult {
  std::string ligand_id;
  double score = 0.0;
  long evaluations = 0;
  double time_seconds = 0.0;
  friend bool operator==(const LigandResult&, const LigandResult&) = default;
};

struct ScreeningReport {
  std::string pocket_id;
  KnobConfig config;
  std::vector<LigandResult> per_ligand;  // sorted by ligand_id
  std::vector<SkippedRecord> skipped;
  double throughput = 0.0;  // ligand atoms per second
  long total_atoms = 0;
  double wall_time_seconds = 0.0;
  double top1pct_mean = 0.0;
  friend bool operator==(const ScreeningReport&, const ScreeningReport&) = default;
};

class LigandSource {
 public:
  virtual ~LigandSource() = default;
  virtual std::optional<std::variant<Ligand, SkippedRecord>> next() = 0;
};

class VectorLigandSource : public LigandSource {
 public:
  explicit VectorLigandSource(const std::vector<Ligand>& ligands) : ligands_(ligands) {}
  std::optional<std::variant<Ligand, SkippedRecord>> next() override {
    if (cursor_ >= ligands_.size()) return std::nullopt;
    return ligands_[cursor_++];
  }

 private:
  const std::vector<Ligand>& ligands_;
  size_t cursor_ = 0;
};

inline double top1pct_mean_score(const std::vector<LigandResult>& results) {
  if (results.empty()) return 0.0;
  const size_t k = std::max<size_t>(1, static_cast<size_t>(std::ceil(0.01 * results.size())));
  std::vector<double> s;
  for (const LigandResult& r : results) s.push_back(r.score);
  std::partial_sort(s.begin(), s.begin() + k, s.end(), std::greater<double>());
  double sum = 0.0;
  for (size_t i = 0; i < k; ++i) sum += s[i];
  return sum / k;
}

namespace detail {

// Ligands of one screen chunk docked through every GPU; appends results
// and skips.  A ligand's time_seconds is the chunk's wall time split by its
// share of the chunk's estimated cost (the work its dock executes:
// n (1 + 2R 360/hp) reps), the batched analogue of the reference's
// per-call wall time (kernel.hpp:245-247).
inline void screen_chunk(const Pocket& pocket, const std::vector<Ligand>& ligands, const KnobConfig& config,
                         std::vector<LigandResult>& results, std::vector<SkippedRecord>& skipped,
                         long& total_atoms) {
  if (ligands.empty()) return;
  const auto t0 = std::chrono::steady_clock::now();
  Packed pk;
  for (const Ligand& l : ligands) pk.add(l, nullptr);
  Results res(ligands.size(), 1, pk.radii.size(), false);
  const gd_ligand_batch b = pk.view();
  const gd_knobs k = config.to_c(0, 1);
  gd_result r = res.view();
  auto& d = Device::get();
  std::vector<std::string> why(ligands.size());
  {
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    check_multi(gd_multi_dock_batch(d.multi(), &b, &k, &r));
    for (size_t l = 0; l < ligands.size(); ++l)
      if (res.status[l] == GD_LIG_INVALID) {
        char buf[512] = {0};
        gd_multi_ligand_error(d.multi(), static_cast<int32_t>(l), buf, sizeof buf);
        why[l] = ligand_error_text(buf, static_cast<int32_t>(l), ligands[l].id());
      }
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<double> cost(ligands.size());
  double sum = 0.0;
  for (size_t l = 0; l < ligands.size(); ++l) {
    int R = 0;
    for (const Bond& bd : ligands[l].bonds()) R += bd.rotatable ? 1 : 0;
    cost[l] = ligands[l].atom_count() * (1.0 + 2.0 * R * (360.0 / config.high_precision_step)) * config.repetitions;
    sum += cost[l];
  }
  for (size_t l = 0; l < ligands.size(); ++l) {
    if (res.status[l] == GD_LIG_OK) {
      results.push_back({ligands[l].id(), res.final_score[l], static_cast<long>(res.evals[l]),
                         sum > 0 ? wall * cost[l] / sum : 0.0});
      total_atoms += ligands[l].atom_count();
    } else {
      skipped.push_back({ligands[l].id(), res.status[l] == GD_LIG_DEGENERATE
                                              ? "rotate_fragment: degenerate rotation axis"
                                              : why[l]});
    }
  }
}

}  // namespace detail

/// Screens a ligand stream against one pocket (screening.hpp:96-178) on
/// every GPU.  The stream is consumed in bounded chunks: while the GPUs dock
/// chunk k, this thread reads chunk k+1 from the source, so host memory is
/// two chunks of ligands (plus the per-ligand results) whatever the stream
/// length -- the reference's bounded queue of 4 x workers ligands, sized
/// for GPUs (`workers` x 1024 ligands per chunk, at least 4096, at most
/// 65536).  Per-ligand failures are recorded as skipped with the reference
/// message; results are in ligand-id order.
inline ScreeningReport screen(const Pocket& pocket, LigandSource& source, const KnobConfig& config,
                              int workers, const PocketIndex* = nullptr) {
  config.validate();
  if (workers < 1) throw Error("screen: workers must be >= 1");
  const auto t0 = std::chrono::steady_clock::now();
  const size_t chunk = std::clamp<size_t>(static_cast<size_t>(workers) * 1024, 4096, 65536);
  ScreeningReport report;
  std::vector<LigandResult> results;
  std::vector<SkippedRecord> skipped;
  long total_atoms = 0;
  // One docking thread consumes full chunks; the caller's thread fills the
  // next one meanwhile (a two-slot hand-off).
  std::mutex mu;
  std::condition_variable cv;
  std::optional<std::vector<Ligand>> pending;
  bool finished = false;
  std::exception_ptr failure;
  std::thread docker([&] {
    for (;;) {
      std::vector<Ligand> batch;
      {
        std::unique_lock<std::mutex> lock(mu);
        cv.wait(lock, [&] { return pending.has_value() || finished; });
        if (!pending) return;
        batch = std::move(*pending);
        pending.reset();
      }
      cv.notify_all();
      try {
        detail::screen_chunk(pocket, batch, config, results, report.skipped, total_atoms);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        failure = std::current_exception();
        finished = true;
        cv.notify_all();
        return;
      }
    }
  });
  auto hand_off = [&](std::vector<Ligand>&& b) {
    std::unique_lock<std::mutex> lock(mu);
    cv.wait(lock, [&] { return !pending.has_value() || failure; });
    if (!failure) pending = std::move(b);
    cv.notify_all();
  };
  std::vector<Ligand> fill;
  try {
    while (auto rec = source.next()) {
      if (std::holds_alternative<SkippedRecord>(*rec)) {
        skipped.push_back(std::get<SkippedRecord>(std::move(*rec)));
        continue;
      }
      fill.push_back(std::get<Ligand>(std::move(*rec)));
      if (fill.size() == chunk) {
        hand_off(std::move(fill));
        fill = std::vector<Ligand>();
        fill.reserve(chunk);
        std::lock_guard<std::mutex> lock(mu);
        if (failure) break;
      }
    }
    if (!fill.empty()) hand_off(std::move(fill));
  } catch (...) {
    {
      std::lock_guard<std::mutex> lock(mu);
      finished = true;
    }
    cv.notify_all();
    docker.join();
    throw;
  }
  {
    std::unique_lock<std::mutex> lock(mu);
    cv.wait(lock, [&] { return !pending.has_value() || failure; });
    finished = true;
  }
  cv.notify_all();
  docker.join();
  if (failure) std::rethrow_exception(failure);
  report.skipped.insert(report.skipped.end(), skipped.begin(), skipped.end());
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::sort(results.begin(), results.end(),
            [](const LigandResult& a, const LigandResult& b) { return a.ligand_id < b.ligand_id; });
  std::sort(report.skipped.begin(), report.skipped.end(),
            [](const SkippedRecord& a, const SkippedRecord& b) { return a.id < b.id; });
  report.per_ligand = std::move(results);
  report.pocket_id = pocket.id();
  report.config = config;
  report.total_atoms = total_atoms;
  report.wall_time_seconds = wall;
  report.throughput = report.per_ligand.empty() ? 0.0 : static_cast<double>(total_atoms) / wall;
  report.top1pct_mean = top1pct_mean_score(report.per_ligand);
  return report;
}

inline ScreeningReport screen(const Pocket& pocket, const std::vector<Ligand>& ligands,
                              const KnobConfig& config, int workers,
                              const PocketIndex* index = nullptr) {
  VectorLigandSource source(ligands);
  return screen(pocket, source, config, workers, index);
}

inline double overlap_degradation(const ScreeningReport& approx, const ScreeningReport& baseline) {
  if (baseline.top1pct_mean == 0.0) throw Error("overlap_degradation: degenerate baseline");
  return (1.0 - approx.top1pct_mean / baseline.top1pct_mean) * 100.0;
}

// ---- north-star batch path -------------------------------------------------
/// One kept pose of a docked ligand (E7).
struct DockedPose {
  int orientation = -1;  // Euler-grid linear index of the rigid seed
  int seed_rank = 0;     // rank of the seed in the rigid top-K
  double rigid_score = 0.0;
  double score = 0.0;    // final PoseResult::score
  long evaluations = 0;
  long feasibility_checks = 0;
  Pose final_pose;
};

struct DockedLigand {
  std::string ligand_id;
  bool ok = false;
  std::vector<DockedPose> poses;  // (score desc, seed rank asc)
  long poses_scored = 0;
};

/// Rigid sweep (step `rigid_step`) + top-K + K restart chains of
/// match_probes_shape(config) per ligand, on every GPU (gd_multi).
inline std::vector<DockedLigand> dock_batch(const Pocket& pocket, const std::vector<Ligand>& ligands,
                                            const KnobConfig& config, int rigid_step, int top_k,
                                            bool keep_poses = false) {
  config.validate();
  detail::Packed pk;
  for (const Ligand& l : ligands) pk.add(l, nullptr);
  const size_t K = rigid_step > 0 ? top_k : 1;
  detail::Results res(ligands.size(), K, pk.radii.size(), keep_poses);
  const gd_knobs k = config.to_c(rigid_step, top_k);
  {
    char msg[256];
    if (gd_validate_knobs(&k, msg, sizeof msg) != GD_OK) throw Error(msg);
  }
  if (!ligands.empty()) {
    const gd_ligand_batch b = pk.view();
    gd_result r = res.view();
    auto& d = detail::Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    detail::check_multi(gd_multi_dock_batch(d.multi(), &b, &k, &r));
  }
  std::vector<DockedLigand> out(ligands.size());
  for (size_t l = 0; l < ligands.size(); ++l) {
    DockedLigand& dl = out[l];
    dl.ligand_id = ligands[l].id();
    dl.ok = res.status[l] == GD_LIG_OK;
    dl.poses_scored = static_cast<long>(res.scored[l]);
    const int n = ligands[l].atom_count();
    for (int e = 0; e < res.k_eff[l]; ++e) {
      const size_t s = l * K + e;
      DockedPose p{res.orientation[s], res.rank[s], res.rigid[s], res.final_score[s],
                   static_cast<long>(res.evals[s]), static_cast<long>(res.checks[s]), {}};
      if (keep_poses) {
        const double* q = res.pose.data() + 3 * (K * pk.atom_off[l] + static_cast<size_t>(e) * n);
        for (int i = 0; i < n; ++i) p.final_pose.positions.push_back({q[3 * i], q[3 * i + 1], q[3 * i + 2]});
      }
      dl.poses.push_back(std::move(p));
    }
  }
  return out;
}

}  // namespace geodock
