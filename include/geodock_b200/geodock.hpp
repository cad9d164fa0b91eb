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
//   KnobConfig::validate      kernel.hpp:28    same messages
//   optimal_tile_size         kernel.hpp:62    gd_optimal_tile_size
//   match_probes_shape        kernel.hpp:205   gd_dock_batch (rigid_step 0, K 1)
//   screen                    screening.hpp:96 one gd_dock_batch over the batch
//   top1pct_mean_score        screening.hpp:78 same
//   overlap_degradation       screening.hpp:190 same
//   (new) dock_batch                           the north-star batch path:
//                                              rigid sweep + top-K + restarts
//   analysis.hpp (rotation profiles, peaks)    geodock_b200/analysis.hpp
//   perf_model.hpp + autotuner.hpp (planner)   geodock_b200/planner.hpp
//   formats.hpp (files, reports, CSVs)         geodock_b200/formats.hpp
//
// Results are bit-identical to the reference.  Link with
// paper_1901_06363_b200/libgeodock_b200.so.  Define GEODOCK_B200_DEVICE to
// pick the GPU (default 0).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
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

#ifndef GEODOCK_B200_DEVICE
#define GEODOCK_B200_DEVICE 0
#endif

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

// ---- vec3.hpp (value type only; the math runs on the GPU) ---------------------
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  constexpr Vec3() = default;
  constexpr Vec3(double px, double py, double pz) : x(px), y(py), z(pz) {}
  constexpr bool operator==(const Vec3& o) const { return x == o.x && y == o.y && z == o.z; }
};

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
  const std::string& id() const { return id_; }
  const std::vector<Atom>& atoms() const { return atoms_; }
  const std::vector<Bond>& bonds() const { return bonds_; }
  int atom_count() const { return static_cast<int>(atoms_.size()); }

 private:
  std::string id_;
  std::vector<Atom> atoms_;
  std::vector<Bond> bonds_;
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

/// One device context per process (per device), shared by all calls.
class Device {
 public:
  static Device& get() {
    static Device d;
    return d;
  }
  gd_ctx* ctx() { return ctx_; }
  std::mutex& mu() { return mu_; }
  const void* staged = nullptr;  // Pocket currently staged (identity)
  uint64_t staged_serial = 0;

  ~Device() {
    if (ctx_) gd_destroy(ctx_);
  }

 private:
  Device() {
    if (gd_create(GEODOCK_B200_DEVICE, &ctx_) != GD_OK)
      throw Error(std::string("geodock_b200: ") + gd_last_error(nullptr));
  }
  gd_ctx* ctx_ = nullptr;
  std::mutex mu_;
};

inline void check(int rc) {
  if (rc != GD_OK) throw Error(gd_last_error(Device::get().ctx()));
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

  /// Makes this pocket the device's staged pocket (caller holds the lock).
  void stage(detail::Device& d) const {
    if (d.staged_serial == serial_) return;
    std::vector<double> xyz;
    xyz.reserve(points_.size() * 3);
    for (const Vec3& p : points_) xyz.insert(xyz.end(), {p.x, p.y, p.z});
    detail::check(gd_set_pocket(d.ctx(), xyz.data(), static_cast<int32_t>(points_.size())));
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

}  // namespace detail

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
  }
  if (res.status[0] == GD_LIG_DEGENERATE) throw Error("rotate_fragment: degenerate rotation axis");
  if (res.status[0] != GD_LIG_OK) throw Error("ligand '" + ligand.id() + "': invalid");
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

/// Screens a ligand stream against one pocket (screening.hpp:96-178): the
/// whole stream goes through one batched GPU call; per-ligand failures are
/// recorded as skipped, results are in ligand-id order.  `workers` is
/// validated and otherwise ignored (the GPU is the worker pool).
inline ScreeningReport screen(const Pocket& pocket, LigandSource& source, const KnobConfig& config,
                              int workers, const PocketIndex* = nullptr) {
  config.validate();
  if (workers < 1) throw Error("screen: workers must be >= 1");
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<Ligand> ligands;
  ScreeningReport report;
  while (auto rec = source.next()) {
    if (std::holds_alternative<SkippedRecord>(*rec)) report.skipped.push_back(std::get<SkippedRecord>(*rec));
    else ligands.push_back(std::get<Ligand>(std::move(*rec)));
  }
  detail::Packed pk;
  for (const Ligand& l : ligands) pk.add(l, nullptr);
  detail::Results res(ligands.size(), 1, pk.radii.size(), false);
  if (!ligands.empty()) {
    const gd_ligand_batch b = pk.view();
    const gd_knobs k = config.to_c(0, 1);
    gd_result r = res.view();
    auto& d = detail::Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    detail::check(gd_dock_batch(d.ctx(), &b, &k, &r));
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (size_t l = 0; l < ligands.size(); ++l) {
    if (res.status[l] == GD_LIG_OK) {
      report.per_ligand.push_back({ligands[l].id(), res.final_score[l], static_cast<long>(res.evals[l]),
                                   wall / ligands.size()});
      report.total_atoms += ligands[l].atom_count();
    } else {
      report.skipped.push_back({ligands[l].id(), res.status[l] == GD_LIG_DEGENERATE
                                                     ? "rotate_fragment: degenerate rotation axis"
                                                     : "invalid ligand"});
    }
  }
  std::sort(report.per_ligand.begin(), report.per_ligand.end(),
            [](const LigandResult& a, const LigandResult& b) { return a.ligand_id < b.ligand_id; });
  std::sort(report.skipped.begin(), report.skipped.end(),
            [](const SkippedRecord& a, const SkippedRecord& b) { return a.id < b.id; });
  report.pocket_id = pocket.id();
  report.config = config;
  report.wall_time_seconds = wall;
  report.throughput = report.per_ligand.empty() ? 0.0 : static_cast<double>(report.total_atoms) / wall;
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
/// match_probes_shape(config) per ligand, all on the GPU.
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
    detail::check(gd_dock_batch(d.ctx(), &b, &k, &r));
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
