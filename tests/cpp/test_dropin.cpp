// Drop-in API test: the reference's own test cases (test_geometry.cpp,
// test_kernel.cpp, test_screening.cpp, test_analysis.cpp, test_autotuner.cpp),
// restated against
// <geodock_b200/geodock.hpp>, which runs them on the GPU through the C-ABI.
// A plain runner (no Catch2 in this image): prints one line per case and
// exits non-zero on any failure.  Built and run by tests/test_dropin.py.
#include <sys/resource.h>

#include <cmath>
#include <cstdio>
#include <functional>
#include <queue>
#include <random>
#include <string>
#include <vector>

#include "geodock_b200/analysis.hpp"
#include "geodock_b200/geodock.hpp"
#include "geodock_b200/planner.hpp"

using namespace geodock;

static int g_failed = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
      ++g_failed;                                                            \
    }                                                                        \
  } while (0)

static void run(const char* name, const std::function<void()>& fn) {
  const int before = g_failed;
  try {
    fn();
  } catch (const std::exception& e) {
    std::printf("  exception: %s\n", e.what());
    ++g_failed;
  }
  std::printf("%s %s\n", g_failed == before ? "PASS" : "FAIL", name);
}

static Pose pose_of(std::vector<Vec3> p) { return Pose{std::move(p)}; }

// PeakRig (test_kernel.cpp:19-31).
static Ligand rig_ligand() {
  return Ligand("rig", {{0, {0, 0, 0}, 1.0}, {1, {0, 0, 1}, 1.0}, {2, {1, 0, 1}, 1.0}},
                {{0, 1, true}, {1, 2, false}});
}
static Pocket rig_pocket() { return Pocket("p", {{0, 0, 0}, {0, 0, 1.2}, {0, -1, 1}}); }

// A small seeded ligand family (this repo's BASELINE generator,
// csrc/synth.cpp), standing in for the reference tests' small_dataset.
static Ligand synth(uint64_t seed, int id, int lo = 6, int hi = 14, int r_cap = 4) {
  const double c[3] = {0, 0, 0};
  int32_t n = 0;
  gd_synth_ligand_size(seed, id, lo, hi, 0, &n);
  std::vector<double> xyz(3 * n), radii(n);
  std::vector<int32_t> bonds(2 * (n - 1));
  std::vector<uint8_t> rot(n - 1);
  gd_synth_ligand(seed, id, lo, hi, 0, r_cap, -1, c, xyz.data(), radii.data(), bonds.data(), rot.data());
  std::vector<Atom> atoms;
  std::vector<Bond> bs;
  for (int i = 0; i < n; ++i) atoms.push_back({i, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]}, radii[i]});
  for (int b = 0; b < n - 1; ++b) bs.push_back({bonds[2 * b], bonds[2 * b + 1], rot[b] != 0});
  return Ligand("S" + std::to_string(id), atoms, bs);
}
static Pocket synth_pocket(double a, double b, double c, double h) {
  std::vector<double> pts(3 * 20000);
  const int P = gd_synth_pocket(a, b, c, h, 0.0, 7, pts.data(), 20000);
  std::vector<Vec3> v;
  for (int j = 0; j < P; ++j) v.push_back({pts[3 * j], pts[3 * j + 1], pts[3 * j + 2]});
  return Pocket("sp", v);
}

// All-pairs bump check with its own BFS (the reference's bump_oracle,
// tests/support/oracles.hpp:51-81, restated).
static bool bump_oracle(const Pose& pose, const Ligand& l, const Fragment& f) {
  const int n = l.atom_count();
  bool ok = true;
  for (int i = 0; i < n; ++i) {
    if (!f.membership[i]) continue;
    std::vector<int> dist(n, -1);
    std::queue<int> q;
    q.push(i);
    dist[i] = 0;
    while (!q.empty()) {
      const int at = q.front();
      q.pop();
      for (const auto& [nb, bond] : l.neighbors(at))
        if (dist[nb] < 0) dist[nb] = dist[at] + 1, q.push(nb);
    }
    for (int j = 0; j < n; ++j) {
      if (f.membership[j] || dist[j] < 4) continue;
      const double cut = 0.8 * (l.atoms()[i].radius + l.atoms()[j].radius);
      if (distance(pose.positions[i], pose.positions[j]) < cut) ok = false;
    }
  }
  return ok;
}

static bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

// An endless-looking stream of small generated ligands (nothing is
// materialised up front).
class CountingSource : public LigandSource {
 public:
  explicit CountingSource(long n) : n_(n) {}
  std::optional<std::variant<Ligand, SkippedRecord>> next() override {
    if (i_ >= n_) return std::nullopt;
    const long i = i_++;
    const double dz = 0.001 * (i % 997);
    return Ligand("M" + std::to_string(i),
                  std::vector<Atom>{{0, {0, 0, dz}, 1.0}, {1, {0, 0, 1 + dz}, 1.0}, {2, {1, 0, 1 + dz}, 1.0},
                                    {3, {1, 1, 1 + dz}, 1.0}},
                  std::vector<Bond>{{0, 1, true}, {1, 2, true}, {2, 3, false}});
  }

 private:
  long n_, i_ = 0;
};

static long max_rss_kb() {
  rusage u{};
  getrusage(RUSAGE_SELF, &u);
  return u.ru_maxrss;
}

static void fine_grained_cases();
static void streaming_cases();

int main() {
  fine_grained_cases();
  run("overlap_score matches hand-computed values", [] {
    CHECK(overlap_score(pose_of({{0, 0, 0}}), Pocket("p", {{0, 0, 1}})) == 1.0);
    CHECK(overlap_score(pose_of({{0, 0, 0}, {0, 0, 3}}), Pocket("p", {{0, 0, 0}})) == 2.0 / (1e-12 + 9.0));
    CHECK(overlap_score(pose_of({{0, 0, 2}}), Pocket("p", {{0, 0, 1}, {0, 0, 4}})) == 1.0);
  });
  run("overlap_score decreases as a single atom moves away", [] {
    const Pocket pocket("p", {{0, 0, 0}});
    double prev = overlap_score(pose_of({{0, 0, 1}}), pocket);
    for (double r = 1.5; r < 10.0; r += 0.5) {
      const double cur = overlap_score(pose_of({{0, 0, r}}), pocket);
      CHECK(cur < prev);
      prev = cur;
    }
  });
  run("overlap_score: empty pose is an error", [] {
    bool threw = false;
    try {
      overlap_score(Pose{}, Pocket("p", {{0, 0, 0}}));
    } catch (const Error&) {
      threw = true;
    }
    CHECK(threw);
  });
  run("optimal_tile_size matches the divisor argmin", [] {
    CHECK(optimal_tile_size(1) == 18);
    CHECK(optimal_tile_size(4) == 36);
    CHECK(optimal_tile_size(360) == 360);
  });
  run("KnobConfig validation", [] {
    auto bad = [](KnobConfig k) {
      try {
        k.validate();
      } catch (const Error&) {
        return true;
      }
      return false;
    };
    CHECK(!bad(KnobConfig{1, 45, 0.0, 3, false}));
    CHECK(bad(KnobConfig{7, 45, 0.0, 3, false}));
    CHECK(bad(KnobConfig{10, 5, 0.0, 3, false}));
    CHECK(bad(KnobConfig{1, 45, 1.5, 3, false}));
    CHECK(bad(KnobConfig{1, 45, 0.0, 0, false}));
    CHECK(bad(KnobConfig{0, 45, 0.0, 3, false}));
  });
  run("Ligand validation messages", [] {
    try {
      Ligand("x", {{0, {0, 0, 0}, 1.0}}, {});
      CHECK(false);
    } catch (const Error& e) {
      CHECK(std::string(e.what()).find("needs at least 2 atoms") != std::string::npos);
    }
    try {
      Ligand("x", {{0, {0, 0, 0}, 1.0}, {1, {1, 0, 0}, 1.0}, {2, {2, 0, 0}, 1.0}}, {{0, 1, false}});
      CHECK(false);
    } catch (const Error& e) {
      CHECK(std::string(e.what()).find("disconnected") != std::string::npos);
    }
  });
  run("match_probes_shape: baseline checks 360 candidates per fragment pass", [] {
    const auto r = match_probes_shape(rig_ligand(), rig_pocket(), make_initial_pose(rig_ligand()),
                                      KnobConfig{1, 45, 0.0, 3, false});
    CHECK(r.feasibility_checks == 1 + 3 * 2 * 360);
    CHECK(r.evaluations <= r.feasibility_checks);
  });
  run("match_probes_shape: refinement respects the per-fragment budget", [] {
    const auto r = match_probes_shape(rig_ligand(), rig_pocket(), make_initial_pose(rig_ligand()),
                                      KnobConfig{1, 45, 0.0, 1, true});
    CHECK(r.evaluations <= 1 + 1 * 2 * 38);
  });
  run("match_probes_shape: threshold 1 sends every fragment to the low step", [] {
    const auto r = match_probes_shape(rig_ligand(), rig_pocket(), make_initial_pose(rig_ligand()),
                                      KnobConfig{1, 90, 1.0, 1, false});
    CHECK(r.feasibility_checks == 1 + 1 * 2 * 4);
  });
  run("match_probes_shape: a rigid ligand scores the input pose once", [] {
    const Ligand rigid("rigid", {{0, {0, 0, 0}, 1.0}, {1, {0, 0, 1.5}, 1.0}}, {{0, 1, false}});
    const Pocket pocket("p", {{0, 0, 1}});
    const Pose initial = make_initial_pose(rigid);
    const auto r = match_probes_shape(rigid, pocket, initial, KnobConfig{});
    CHECK(r.evaluations == 1);
    CHECK(r.score == overlap_score(initial, pocket));
    CHECK(r.final_pose.positions == initial.positions);
  });
  run("match_probes_shape: committed, deterministic, never regressing", [] {
    const Ligand lig = rig_ligand();
    const Pocket pocket = rig_pocket();
    const KnobConfig cfg{2, 90, 0.3, 2, true};
    const auto a = match_probes_shape(lig, pocket, make_initial_pose(lig), cfg);
    const auto b = match_probes_shape(lig, pocket, make_initial_pose(lig), cfg);
    CHECK(a.score == b.score);
    CHECK(a.final_pose.positions == b.final_pose.positions);
    CHECK(a.score == overlap_score(a.final_pose, pocket));
    CHECK(a.score >= overlap_score(make_initial_pose(lig), pocket));
  });
  run("match_probes_shape: a 300-atom ligand docks (the reference has no size limit)", [] {
    // 300 atoms take the wide path (flex_wide_kernel): committed pose,
    // never regressing, deterministic, feasible under the bump oracle.
    const Ligand lig = synth(424242, 0, 300, 300, 10);
    const Pocket pocket = synth_pocket(10, 8, 6, 0.795);
    const KnobConfig cfg{60, 90, 0.0, 1, false};
    const Pose initial = make_initial_pose(lig);
    const auto a = match_probes_shape(lig, pocket, initial, cfg);
    const auto b = match_probes_shape(lig, pocket, initial, cfg);
    CHECK(a.final_pose.positions.size() == 300);
    CHECK(a.score == b.score);
    CHECK(a.final_pose.positions == b.final_pose.positions);
    CHECK(a.score == overlap_score(a.final_pose, pocket));
    CHECK(a.score >= overlap_score(initial, pocket));
    CHECK(a.feasibility_checks == 1 + static_cast<long>(2 * find_rotamers(lig).size()) * (360 / 60));
    for (const auto& rot : find_rotamers(lig)) {
      const auto [left, right] = grow_fragments(lig, rot);
      CHECK(bump_oracle(a.final_pose, lig, left) || !bump_oracle(initial, lig, left));
    }
  });
  run("match_probes_shape: pose/ligand size mismatch", [] {
    try {
      match_probes_shape(rig_ligand(), rig_pocket(), pose_of({{0, 0, 0}}), KnobConfig{});
      CHECK(false);
    } catch (const Error& e) {
      CHECK(std::string(e.what()).find("size mismatch") != std::string::npos);
    }
  });
  run("screen: bookkeeping, id order, top-1% mean, skipped records", [] {
    std::vector<Ligand> ligs;
    for (int i = 0; i < 5; ++i) {
      const double dz = 0.1 * i;
      ligs.emplace_back("L" + std::to_string(4 - i),
                        std::vector<Atom>{{0, {0, 0, dz}, 1.0}, {1, {0, 0, 1 + dz}, 1.0}, {2, {1, 0, 1 + dz}, 1.0}},
                        std::vector<Bond>{{0, 1, true}, {1, 2, false}});
    }
    const ScreeningReport r = screen(rig_pocket(), ligs, KnobConfig{10, 90, 0.5, 1, false}, 4);
    CHECK(r.per_ligand.size() == 5);
    for (size_t i = 1; i < r.per_ligand.size(); ++i) CHECK(r.per_ligand[i - 1].ligand_id < r.per_ligand[i].ligand_id);
    double best = 0.0;
    for (const auto& x : r.per_ligand) best = std::max(best, x.score);
    CHECK(r.top1pct_mean == best);
    CHECK(r.total_atoms == 15);
    for (const auto& x : r.per_ligand) {
      const Ligand* l = nullptr;
      for (const auto& c : ligs)
        if (c.id() == x.ligand_id) l = &c;
      CHECK(x.score == match_probes_shape(*l, rig_pocket(), make_initial_pose(*l),
                                          KnobConfig{10, 90, 0.5, 1, false}).score);
    }
  });
  run("dock_batch: rigid sweep + top-K + restarts", [] {
    std::vector<Ligand> ligs{rig_ligand()};
    const auto out = dock_batch(rig_pocket(), ligs, KnobConfig{30, 45, 0.0, 1, false}, 45, 8, true);
    CHECK(out.size() == 1 && out[0].ok);
    CHECK(out[0].poses.size() == 8);
    for (size_t e = 1; e < out[0].poses.size(); ++e) {
      const auto& a = out[0].poses[e - 1];
      const auto& b = out[0].poses[e];
      CHECK(a.score > b.score || (a.score == b.score && a.seed_rank < b.seed_rank));
    }
    for (const auto& p : out[0].poses) CHECK(p.score == overlap_score(p.final_pose, rig_pocket()));
  });
  run("rotation_profile: a far-away rigid pair is valid everywhere", [] {
    const Ligand ligand("l", {{0, {0, 0, 0}, 1.0}, {1, {0, 0, 1.4}, 1.0}, {2, {1.2, 0, 1.4}, 1.0}},
                        {{0, 1, true}, {1, 2, false}});
    const Pocket pocket("p", {{0, 0, 1}});
    const auto [left, right] = grow_fragments(ligand, find_rotamers(ligand)[0]);
    const Pose pose = make_initial_pose(ligand);
    const RotationProfile profile = rotation_profile(pose, ligand, right, pocket);
    for (int a = 0; a < 360; ++a) CHECK(profile.valid[a]);
    CHECK(profile.scores[0] == overlap_score(pose, pocket));
    CHECK(profile.relative_size == right.relative_size);
  });
  run("rotation_profile: validity and scores match rotate + check + score", [] {
    const Ligand lig = rig_ligand();
    const Pocket pocket = rig_pocket();
    const auto [left, right] = grow_fragments(lig, find_rotamers(lig)[0]);
    const RotationProfile prof = rotation_profile(make_initial_pose(lig), lig, left, pocket);
    int valid = 0;
    for (int a = 0; a < 360; ++a) valid += prof.valid[a] ? 1 : 0;
    CHECK(valid == 360);  // three atoms: no pair at graph distance >= 4
    // The left fragment {0} swings about the 1->0 bond: atom 0 sits on the
    // axis, so every angle scores like the input pose.
    for (int a = 0; a < 360; ++a) CHECK(prof.scores[a] == prof.scores[0]);
  });
  run("detect_peaks: rectangular, flat, wrap-around, all-invalid", [] {
    RotationProfile p;
    p.valid.fill(true);
    p.scores.fill(0.0);
    p.scores[2] = p.scores[3] = 1.0;
    const PeakStats s = detect_peaks(p);
    CHECK(s.delta_overlap == 1.0 && s.peaks.size() == 1 && s.peaks[0].start_angle == 2 &&
          s.peaks[0].width == 2 && s.peaks[0].height_ratio == 1.0 && s.best_peak_width == 2);
    RotationProfile flat;
    flat.valid.fill(true);
    flat.scores.fill(3.5);
    CHECK(detect_peaks(flat).peaks.empty() && detect_peaks(flat).best_peak_width == 0);
    RotationProfile wrap;
    wrap.valid.fill(true);
    wrap.scores.fill(0.0);
    for (int a : {358, 359, 0, 1}) wrap.scores[a] = 1.0;
    const PeakStats w = detect_peaks(wrap);
    CHECK(w.peaks.size() == 1 && w.peaks[0].start_angle == 358 && w.peaks[0].width == 4);
    RotationProfile none;
    none.valid.fill(false);
    bool threw = false;
    try {
      detect_peaks(none);
    } catch (const Error& e) {
      threw = std::string(e.what()).find("no feasible") != std::string::npos;
    }
    CHECK(threw);
  });
  run("tile_hit_probability: counts, evaluation model, monotonicity", [] {
    PeakStats wide;
    wide.best_peak_width = 68;
    const std::vector<PeakStats> ds(10, wide);
    const auto hits = tile_hit_probability(ds, {18, 90});
    CHECK(hits.size() == 2 && hits[0].probability == 1.0 && hits[1].probability == 0.0 &&
          hits[0].eval_count == 38.0);
    CHECK(tile_hit_probability(ds, {}).empty());
  });
  run("analyze_ligand produces consistent rows; analyze_ligands agrees", [] {
    std::vector<Ligand> ligs;
    for (int i = 0; i < 3; ++i) {
      const double dz = 0.1 * i;
      ligs.emplace_back("A" + std::to_string(i),
                        std::vector<Atom>{{0, {0, 0, dz}, 1.0}, {1, {0, 0, 1 + dz}, 1.0},
                                          {2, {1, 0, 1 + dz}, 1.0}, {3, {1, 1, 1 + dz}, 1.0},
                                          {4, {2, 1, 1 + dz}, 1.0}},
                        std::vector<Bond>{{0, 1, true}, {1, 2, true}, {2, 3, true}, {3, 4, false}});
    }
    const KnobConfig cfg{3, 90, 0.0, 1, false};
    const auto batch = analyze_ligands(ligs, rig_pocket(), cfg);
    for (size_t l = 0; l < ligs.size(); ++l) {
      const LigandAnalysis a = analyze_ligand(ligs[l], rig_pocket(), cfg);
      CHECK(a.dock.score > 0.0);
      CHECK(a.fragments.size() == a.stats.size());
      for (const auto& row : a.fragments) {
        CHECK(row.ligand_id == ligs[l].id());
        CHECK(row.relative_size > 0.0 && row.relative_size < 1.0);
        CHECK(row.delta_normalized >= 0.0);
      }
      CHECK(batch[l].dock.score == a.dock.score);
      CHECK(batch[l].fragments.size() == a.fragments.size());
      for (size_t f = 0; f < a.fragments.size() && f < batch[l].fragments.size(); ++f)
        CHECK(batch[l].fragments[f].delta_overlap == a.fragments[f].delta_overlap);
      CHECK(batch[l].peaks.size() == a.peaks.size());
    }
  });
  run("build_knowledge_base profiles a small design space end to end", [] {
    // Nine small training sets from the seeded generator; the three data
    // features (pocket size, atoms, rotamers) all vary across them.
    std::vector<TrainingSet> sets;
    for (int s = 0; s < 9; ++s) {
      std::vector<double> pts(3 * 4000);
      const int P = gd_synth_pocket(3.0 + 0.4 * s, 2.5 + 0.3 * (s % 4), 2.0 + 0.25 * (s % 3), 1.0, 0.0,
                                    100 + s, pts.data(), 4000);
      std::vector<Vec3> pv;
      for (int j = 0; j < P; ++j) pv.push_back({pts[3 * j], pts[3 * j + 1], pts[3 * j + 2]});
      std::vector<Ligand> ligs;
      for (int l = 0; l < 12; ++l) {
        const double c[3] = {0, 0, 0};
        const int lo = 8 + 2 * (s % 3), hi = 16 + 2 * (s % 4);
        int32_t n = 0;
        gd_synth_ligand_size(1000 + 17 * s, l, lo, hi, 0, &n);
        std::vector<double> xyz(3 * n), radii(n);
        std::vector<int32_t> bonds(2 * (n - 1));
        std::vector<uint8_t> rot(n - 1);
        gd_synth_ligand(1000 + 17 * s, l, lo, hi, 0, 1 + s % 3, -1, c, xyz.data(), radii.data(),
                        bonds.data(), rot.data());
        std::vector<Atom> atoms;
        std::vector<Bond> bs;
        for (int i = 0; i < n; ++i) atoms.push_back({i, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]}, radii[i]});
        for (int b = 0; b < n - 1; ++b) bs.push_back({bonds[2 * b], bonds[2 * b + 1], rot[b] != 0});
        ligs.emplace_back("S" + std::to_string(s) + "L" + std::to_string(l), atoms, bs);
      }
      sets.push_back({Pocket("P" + std::to_string(s), pv), ligs});
    }
    const KnobConfig baseline{1, 45, 0.0, 2, false};
    const std::vector<KnobConfig> space{baseline, {3, 45, 0.0, 1, false}, {1, 45, 0.0, 1, true}};
    const KnowledgeBase kb = build_knowledge_base(space, sets, baseline, 2);
    CHECK(kb.profiles.size() == 3);
    CHECK(kb.warnings.empty());
    CHECK(kb.profiles.size() == 3 && kb.profiles[0].config == baseline && kb.profiles[0].mean_degradation == 0.0);
    for (const ConfigProfile& p : kb.profiles) CHECK(p.perf.n_observations == 9 && p.perf.config == p.config);
    // Cheaper configurations never score better than the exhaustive baseline on average.
    for (const ConfigProfile& p : kb.profiles) CHECK(p.mean_degradation >= -1e-9);
    bool threw = false;
    try {
      build_knowledge_base({{3, 45, 0.0, 1, false}}, sets, baseline, 1);
    } catch (const Error&) {
      threw = true;
    }
    CHECK(threw);
  });
  streaming_cases();
  std::printf("%s (%d failed checks)\n", g_failed ? "FAILED" : "OK", g_failed);
  return g_failed ? 1 : 0;
}

// The reference's test_geometry.cpp:84-234 and test_kernel.cpp:52-164
// cases through the drop-in's GPU-backed rotate_fragment, check_bumps and
// optimize_fragment_* symbols.
static void fine_grained_cases() {
  run("rotate_fragment: quarter turn about the z axis", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    const Pose pose = make_initial_pose(l);
    const Pose t = rotate_fragment(pose, l, right, 90.0);
    CHECK(near(t.positions[2].x, 0.0, 1e-12) && near(t.positions[2].y, -1.0, 1e-12) &&
          near(t.positions[2].z, 1.0, 1e-12));
    CHECK(t.positions[0] == pose.positions[0] && t.positions[1] == pose.positions[1]);
    const Ligand l2("l2", {{0, {1, 0, 0}, 1.0}, {1, {0, 0, 0}, 1.0}, {2, {0, 0, 1}, 1.0}},
                    {{0, 1, false}, {1, 2, true}});
    const auto [left2, right2] = grow_fragments(l2, find_rotamers(l2)[0]);
    const Pose t2 = rotate_fragment(make_initial_pose(l2), l2, left2, 90.0);
    CHECK(near(t2.positions[0].x, 0.0, 1e-12) && near(t2.positions[0].y, 1.0, 1e-12) &&
          near(t2.positions[0].z, 0.0, 1e-12));
  });
  run("rotate_fragment: angle 0 is the exact identity, 360 is close", [] {
    for (int id = 0; id < 5; ++id) {
      const Ligand l = synth(7, id);
      const Pose pose = make_initial_pose(l);
      for (const Rotamer& r : find_rotamers(l)) {
        const auto [left, right] = grow_fragments(l, r);
        CHECK(rotate_fragment(pose, l, left, 0.0).positions == pose.positions);
        const Pose full = rotate_fragment(pose, l, left, 360.0);
        for (int i = 0; i < l.atom_count(); ++i)
          CHECK(near(full.positions[i].x, pose.positions[i].x, 1e-9) &&
                near(full.positions[i].y, pose.positions[i].y, 1e-9) &&
                near(full.positions[i].z, pose.positions[i].z, 1e-9));
      }
    }
  });
  run("rotate_fragment: rigid within the fragment and invertible", [] {
    std::mt19937_64 rng(5);
    std::uniform_real_distribution<double> angle(1.0, 359.0);
    for (int id = 0; id < 8; ++id) {
      const Ligand l = synth(99, id);
      const Pose pose = make_initial_pose(l);
      for (const Rotamer& r : find_rotamers(l)) {
        const auto [left, right] = grow_fragments(l, r);
        const double th = angle(rng);
        const Pose rot = rotate_fragment(pose, l, left, th);
        for (size_t a = 0; a < left.atom_indices.size(); ++a)
          for (size_t b = a + 1; b < left.atom_indices.size(); ++b) {
            const int i = left.atom_indices[a], j = left.atom_indices[b];
            CHECK(near(distance(rot.positions[i], rot.positions[j]), distance(pose.positions[i], pose.positions[j]), 1e-9));
          }
        const Pose back = rotate_fragment(rot, l, left, -th);
        for (int i = 0; i < l.atom_count(); ++i)
          CHECK(near(back.positions[i].x, pose.positions[i].x, 1e-9) &&
                near(back.positions[i].y, pose.positions[i].y, 1e-9) &&
                near(back.positions[i].z, pose.positions[i].z, 1e-9));
      }
    }
  });
  run("rotate_fragment: degenerate axis is an error", [] {
    const Ligand l("chain", {{0, {0, 0, 0}, 1.0}, {1, {1.5, 0, 0}, 1.0}, {2, {3, 0, 0}, 1.0}},
                   {{0, 1, true}, {1, 2, true}});
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    Pose collapsed = make_initial_pose(l);
    collapsed.positions[1] = collapsed.positions[0];
    bool threw = false;
    try {
      rotate_fragment(collapsed, l, left, 10.0);
    } catch (const Error& e) {
      threw = std::string(e.what()).find("degenerate") != std::string::npos;
    }
    CHECK(threw);
  });
  auto probe = [](double sep, double radius) {
    std::vector<Atom> atoms;
    std::vector<Bond> bonds;
    for (int i = 0; i < 6; ++i) atoms.push_back({i, {1.5 * i, 0, 0}, radius});
    atoms[5].position = {0.0, sep, 0.0};
    atoms[4].position = {1.5, sep, 0.0};
    atoms[3].position = {3.0, sep, 0.0};
    for (int i = 0; i < 5; ++i) bonds.push_back({i, i + 1, i == 2});
    return Ligand("probe", atoms, bonds);
  };
  run("check_bumps follows the clash rule with the 1-4 exclusion", [&] {
    const Ligand a = probe(0.1, 1.5);
    const auto [la, ra] = grow_fragments(a, find_rotamers(a)[0]);
    CHECK(a.graph_distance_capped(0, 5) == 4);
    CHECK(!check_bumps(make_initial_pose(a), a, la));
    const Ligand b = probe(2.5, 1.5);
    const auto [lb, rb] = grow_fragments(b, find_rotamers(b)[0]);
    CHECK(check_bumps(make_initial_pose(b), b, lb));
    const Ligand fold("fold", {{0, {0, 0, 0}, 1.5}, {1, {1.5, 0, 0}, 1.5}, {2, {1.5, 1.5, 0}, 1.5}, {3, {0.1, 0.1, 0}, 1.5}},
                      {{0, 1, false}, {1, 2, true}, {2, 3, false}});
    const auto [lf, rf] = grow_fragments(fold, find_rotamers(fold)[0]);
    CHECK(check_bumps(make_initial_pose(fold), fold, lf));
  });
  run("check_bumps agrees with the all-pairs oracle across rotations", [] {
    int bumped = 0, feasible = 0;
    for (int id = 0; id < 10; ++id) {
      const Ligand l = synth(2024, id);
      const Pose pose = make_initial_pose(l);
      for (const Rotamer& r : find_rotamers(l)) {
        const auto [left, right] = grow_fragments(l, r);
        for (int angle = 0; angle < 360; angle += 23) {
          const Pose c = rotate_fragment(pose, l, left, angle);
          const bool fast = check_bumps(c, l, left);
          CHECK(fast == bump_oracle(c, l, left));
          fast ? ++feasible : ++bumped;
        }
      }
    }
    CHECK(bumped > 0);
    CHECK(feasible > 0);
  });
  run("flat search: step 360 evaluates only the current pose", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    Pose pose = make_initial_pose(l);
    const Pose before = pose;
    SearchCounters c;
    const auto r = optimize_fragment_flat(pose, l, right, rig_pocket(), 360, &c);
    CHECK(r.best_angle == 0 && pose.positions == before.positions);
    CHECK(c.feasibility_checks == 1 && c.evaluations == 1);
  });
  run("flat search: step 90 considers exactly four candidates", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    Pose pose = make_initial_pose(l);
    SearchCounters c;
    optimize_fragment_flat(pose, l, right, rig_pocket(), 90, &c);
    CHECK(c.feasibility_checks == 4 && c.evaluations <= 4);
  });
  run("flat search: a 30-degree grid finds the 90-degree peak", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    const Pose initial = make_initial_pose(l);
    int brute_best = 0;
    double brute = -1.0;
    for (int a = 0; a < 360; ++a) {
      const Pose c = rotate_fragment(initial, l, right, a);
      if (!check_bumps(c, l, right)) continue;
      const double s = overlap_score(c, rig_pocket());
      if (s > brute) brute = s, brute_best = a;
    }
    CHECK(brute_best == 90);
    Pose pose = initial;
    CHECK(optimize_fragment_flat(pose, l, right, rig_pocket(), 30).best_angle == 90);
  });
  run("refined search stays within the two-phase evaluation budget", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    Pose pose = make_initial_pose(l);
    SearchCounters c;
    const auto r = optimize_fragment_refined(pose, l, right, rig_pocket(), 1, &c);
    CHECK(c.evaluations <= 20 + 18);
    CHECK(r.best_score >= overlap_score(make_initial_pose(l), rig_pocket()));
  });
  run("refined search: a constant profile resolves to the first tile's center", [] {
    const Ligand l("axial", {{0, {0, 0, 0}, 1.0}, {1, {0, 0, 1}, 1.0}}, {{0, 1, true}});
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    Pose pose = make_initial_pose(l);
    CHECK(optimize_fragment_refined(pose, l, right, Pocket("p", {{0.5, 0, 1}}), 1).best_angle == 9);
  });
  run("refined search captures a peak wider than the tile", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    const Pose initial = make_initial_pose(l);
    const Vec3 at99 = rotate_fragment(initial, l, right, 99).positions[2];
    const Pocket pocket("p", {{0, 0, 0}, {0, 0, 1.585}, at99});
    Pose flat_pose = initial, refined_pose = initial;
    const auto f = optimize_fragment_flat(flat_pose, l, right, pocket, 1);
    const auto r = optimize_fragment_refined(refined_pose, l, right, pocket, 1);
    CHECK(f.best_angle == 99 && r.best_angle == 99);
    CHECK(r.best_score == f.best_score);
    CHECK(refined_pose.positions == flat_pose.positions);
  });
  run("optimize_fragment_*: counters accumulate; a sequence reproduces match_probes_shape", [] {
    // match_probes_shape's greedy pass restated through the fine-grained
    // symbols (kernel.hpp:219-242, threshold 0, flat) equals the GPU kernel.
    const Pocket pocket = synth_pocket(6, 5, 4, 1.0);
    for (int id = 0; id < 6; ++id) {
      const Ligand l = synth(321, id, 8, 16, 4);
      Pose pose = make_initial_pose(l);
      SearchCounters c;
      double score = overlap_score(pose, pocket);
      c.feasibility_checks = c.evaluations = 1;
      for (int rep = 0; rep < 2; ++rep)
        for (const Rotamer& r : find_rotamers(l)) {
          const auto [left, right] = grow_fragments(l, r);
          for (const Fragment* f : {&left, &right}) score = optimize_fragment_flat(pose, l, *f, pocket, 30, &c).best_score;
        }
      const auto m = match_probes_shape(l, pocket, make_initial_pose(l), KnobConfig{30, 45, 0.0, 2, false});
      CHECK(m.score == score);
      CHECK(m.final_pose.positions == pose.positions);
      CHECK(m.evaluations == c.evaluations && m.feasibility_checks == c.feasibility_checks);
    }
  });
  run("optimize_fragment_flat: step must divide 360", [] {
    const Ligand l = rig_ligand();
    const auto [left, right] = grow_fragments(l, find_rotamers(l)[0]);
    Pose pose = make_initial_pose(l);
    bool threw = false;
    try {
      optimize_fragment_flat(pose, l, right, rig_pocket(), 7);
    } catch (const Error& e) {
      threw = std::string(e.what()) == "optimize_fragment_flat: step must divide 360";
    }
    CHECK(threw);
  });
}

static void streaming_cases() {
  run("screen streams: 1,000,000 ligands in bounded host memory", [] {
    const KnobConfig cfg{30, 45, 0.0, 1, false};
    CountingSource warm(200000);
    const ScreeningReport a = screen(rig_pocket(), warm, cfg, 16);
    CHECK(a.per_ligand.size() == 200000);
    const long rss0 = max_rss_kb();
    CountingSource big(1000000);
    const ScreeningReport r = screen(rig_pocket(), big, cfg, 16);
    const long grown_mb = (max_rss_kb() - rss0) / 1024;
    std::printf("  1M-ligand screen: %.2f s, %.3g atoms/s, max RSS +%ld MB over a 200k screen\n",
                r.wall_time_seconds, r.throughput, grown_mb);
    CHECK(r.per_ligand.size() == 1000000 && r.skipped.empty());
    CHECK(r.total_atoms == 4000000);
    // Materialising the stream would hold 1M Ligand objects (~700 MB here);
    // the growth is the 1M LigandResult rows the report returns (~100 MB).
    CHECK(grown_mb < 400);
    // Spot checks against single docks.
    for (long i : {0L, 123456L, 999999L}) {
      CountingSource one(i + 1);
      std::optional<Ligand> lig;
      while (auto rec = one.next()) lig = std::get<Ligand>(std::move(*rec));
      const auto m = match_probes_shape(*lig, rig_pocket(), make_initial_pose(*lig), cfg);
      const auto it = std::lower_bound(r.per_ligand.begin(), r.per_ligand.end(), lig->id(),
                                       [](const LigandResult& x, const std::string& id) { return x.ligand_id < id; });
      CHECK(it != r.per_ligand.end() && it->ligand_id == lig->id() && it->score == m.score &&
            it->evaluations == m.evaluations);
    }
  });
}
