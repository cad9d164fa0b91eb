// geodock_b200/analysis.hpp -- drop-in for geodock/analysis.hpp.
//
//   reference (analysis.hpp)          here
//   --------------------------------  ------------------------------------------
//   rotation_profile        :37-56    gd_rotation_profiles (GPU, one warp per
//                                     fragment, 360 angles)
//   detect_peaks            :61-126   gd_detect_peaks (native host)
//   tile_hit_probability    :133-147  gd_tile_hit_probability (native host)
//   analyze_ligand          :177-215  gd_dock_batch (given pose) + one
//                                     gd_rotation_profiles call
//   (new) rotation_profiles           every fragment of a pose in one call
//   (new) analyze_ligands             a whole batch in two GPU calls
//
// Profiles, peaks and rows are bit-identical to the reference
// (tests/test_gpu_analysis.py, tests/test_analysis_cpu.py).
#pragma once

#include <array>
#include <string>
#include <vector>

#include "geodock_b200/geodock.hpp"

namespace geodock {

struct RotationProfile {
  double relative_size = 0.0;
  std::array<double, 360> scores{};  // meaningful only where valid
  std::array<bool, 360> valid{};
};

struct Peak {
  int start_angle = 0;
  int width = 0;
  double height_ratio = 0.0;
};

struct PeakStats {
  double delta_overlap = 0.0;
  std::vector<Peak> peaks;  // ordered by start angle (a wrapped peak last)
  int best_peak_width = 0;
};

struct TileHit {
  int tile_size = 0;
  double probability = 0.0;
  double eval_count = 0.0;
};

struct FragmentProfileRow {
  std::string ligand_id;
  int rotamer_index = 0;
  Side side = Side::left;
  double relative_size = 0.0;
  double delta_overlap = 0.0;
  double delta_normalized = 0.0;
  int peak_count = 0;
  int best_peak_width = 0;
};

struct PeakRow {
  std::string ligand_id;
  int rotamer_index = 0;
  Side side = Side::left;
  int start_angle = 0;
  int width = 0;
  double height_ratio = 0.0;
};

struct LigandAnalysis {
  PoseResult dock;
  std::vector<FragmentProfileRow> fragments;
  std::vector<PeakRow> peaks;
  std::vector<PeakStats> stats;
};

namespace detail {

/// Profiles of every fragment of every (ligand, pose) in reference order
/// (ligand by ligand; rotamer r -> left 2r, right 2r+1).  offsets[l] is
/// ligand l's first profile; status[l] its GD_LIG_* code.
inline std::vector<RotationProfile> profile_batch(const std::vector<const Ligand*>& ligands,
                                                  const std::vector<const Pose*>& poses,
                                                  const Pocket& pocket,
                                                  std::vector<int32_t>& offsets,
                                                  std::vector<int32_t>& status) {
  Packed pk;
  size_t rot_bonds = 0;
  for (size_t l = 0; l < ligands.size(); ++l) {
    pk.add(*ligands[l], poses[l]);
    for (const Bond& b : ligands[l]->bonds()) rot_bonds += b.rotatable ? 1 : 0;
  }
  const size_t cap = std::max<size_t>(1, 2 * rot_bonds);
  std::vector<double> scores(cap * 360), rel(cap);
  std::vector<uint8_t> valid(cap * 360);
  offsets.assign(ligands.size() + 1, 0);
  status.assign(std::max<size_t>(1, ligands.size()), 0);
  if (!ligands.empty()) {
    const gd_ligand_batch b = pk.view();
    auto& d = Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    check(gd_upload(d.ctx(), &b));
    check(gd_rotation_profiles(d.ctx(), 0u, scores.data(), valid.data(), rel.data(), offsets.data(),
                               status.data(), static_cast<int64_t>(cap)));
  }
  std::vector<RotationProfile> out(offsets.back());
  for (size_t f = 0; f < out.size(); ++f) {
    out[f].relative_size = rel[f];
    for (int a = 0; a < 360; ++a) {
      out[f].scores[a] = scores[360 * f + a];
      out[f].valid[a] = valid[360 * f + a] != 0;
    }
  }
  return out;
}

inline void check_pose(const Pose& pose, const Ligand& ligand, const char* who) {
  if (pose.positions.size() != static_cast<size_t>(ligand.atom_count()))
    throw Error(std::string(who) + ": pose/ligand size mismatch");
}

}  // namespace detail

/// Every fragment's profile from `pose`, in reference fragment order.
inline std::vector<RotationProfile> rotation_profiles(const Pose& pose, const Ligand& ligand,
                                                      const Pocket& pocket,
                                                      const PocketIndex* = nullptr) {
  detail::check_pose(pose, ligand, "rotation_profile");
  std::vector<int32_t> offsets, status;
  auto out = detail::profile_batch({&ligand}, {&pose}, pocket, offsets, status);
  if (status[0] == GD_LIG_DEGENERATE) throw Error("rotate_fragment: degenerate rotation axis");
  if (status[0] != GD_LIG_OK) throw Error("ligand '" + ligand.id() + "': invalid");
  return out;
}

/// rotation_profile (analysis.hpp:37-56) of one fragment, which must be one
/// of grow_fragments(ligand, r) for r in find_rotamers(ligand).
inline RotationProfile rotation_profile(const Pose& pose, const Ligand& ligand,
                                        const Fragment& fragment, const Pocket& pocket,
                                        const PocketIndex* index = nullptr) {
  const std::vector<Rotamer> rots = find_rotamers(ligand);
  int r = 0;
  while (r < static_cast<int>(rots.size()) && rots[r].bond_index != fragment.rotamer.bond_index) ++r;
  if (r == static_cast<int>(rots.size()))
    throw Error("rotation_profile: fragment is not a rotamer fragment of ligand '" + ligand.id() + "'");
  const auto all = rotation_profiles(pose, ligand, pocket, index);
  return all[2 * r + (fragment.side == Side::left ? 0 : 1)];
}

/// detect_peaks (analysis.hpp:61-126).
inline PeakStats detect_peaks(const RotationProfile& profile) {
  std::array<uint8_t, 360> valid;
  for (int a = 0; a < 360; ++a) valid[a] = profile.valid[a] ? 1 : 0;
  std::array<gd_peak, 360> buf;
  PeakStats st;
  int32_t best = 0, np = 0;
  if (gd_detect_peaks(profile.scores.data(), valid.data(), &st.delta_overlap, &best, buf.data(),
                      &np) != GD_OK)
    throw Error("detect_peaks: no feasible rotation");
  st.best_peak_width = best;
  for (int k = 0; k < np; ++k) st.peaks.push_back({buf[k].start_angle, buf[k].width, buf[k].height_ratio});
  return st;
}

/// tile_hit_probability (analysis.hpp:133-147).
inline std::vector<TileHit> tile_hit_probability(const std::vector<PeakStats>& dataset,
                                                 const std::vector<int>& tile_sizes) {
  if (dataset.empty()) throw Error("tile_hit_probability: empty dataset");
  std::vector<int32_t> widths, tiles(tile_sizes.begin(), tile_sizes.end());
  for (const PeakStats& s : dataset) widths.push_back(s.best_peak_width);
  std::vector<double> prob(tiles.size()), ev(tiles.size());
  if (gd_tile_hit_probability(widths.data(), static_cast<int64_t>(widths.size()), tiles.data(),
                              static_cast<int32_t>(tiles.size()), prob.data(), ev.data()) != GD_OK)
    throw Error("tile_hit_probability: empty dataset");
  std::vector<TileHit> out;
  for (size_t t = 0; t < tiles.size(); ++t) out.push_back({tiles[t], prob[t], ev[t]});
  return out;
}

namespace detail {

inline void fill_analysis(LigandAnalysis& a, const Ligand& ligand,
                          const std::vector<RotationProfile>& profiles, size_t first, size_t last) {
  for (size_t f = first; f < last; ++f) {
    PeakStats st;
    try {
      st = detect_peaks(profiles[f]);
    } catch (const Error&) {
      continue;  // no feasible rotation for this fragment
    }
    const int fl = static_cast<int>(f - first);
    const Side side = fl % 2 == 0 ? Side::left : Side::right;
    FragmentProfileRow row;
    row.ligand_id = ligand.id();
    row.rotamer_index = fl / 2;
    row.side = side;
    row.relative_size = profiles[f].relative_size;
    row.delta_overlap = st.delta_overlap;
    row.delta_normalized = a.dock.score > 0.0 ? st.delta_overlap / a.dock.score : 0.0;
    row.peak_count = static_cast<int>(st.peaks.size());
    row.best_peak_width = st.best_peak_width;
    a.fragments.push_back(row);
    for (const Peak& p : st.peaks)
      a.peaks.push_back({ligand.id(), fl / 2, side, p.start_angle, p.width, p.height_ratio});
    a.stats.push_back(std::move(st));
  }
}

}  // namespace detail

/// analyze_ligand (analysis.hpp:177-215): dock from the input pose, then
/// profile every fragment from the final committed pose.
inline LigandAnalysis analyze_ligand(const Ligand& ligand, const Pocket& pocket,
                                     const KnobConfig& config, const PocketIndex* index = nullptr) {
  LigandAnalysis a;
  a.dock = match_probes_shape(ligand, pocket, make_initial_pose(ligand), config, index);
  const auto profiles = rotation_profiles(a.dock.final_pose, ligand, pocket, index);
  detail::fill_analysis(a, ligand, profiles, 0, profiles.size());
  return a;
}

/// analyze_ligand over a batch: one docking call and one profile call for
/// all ligands.  A ligand that fails validation or hits a degenerate axis
/// throws, as analyze_ligand would for it.
inline std::vector<LigandAnalysis> analyze_ligands(const std::vector<Ligand>& ligands,
                                                   const Pocket& pocket, const KnobConfig& config) {
  config.validate();
  detail::Packed pk;
  for (const Ligand& l : ligands) pk.add(l, nullptr);
  detail::Results res(ligands.size(), 1, pk.radii.size(), true);
  if (!ligands.empty()) {
    const gd_ligand_batch b = pk.view();
    const gd_knobs k = config.to_c(0, 1);
    gd_result r = res.view();
    auto& d = detail::Device::get();
    std::lock_guard<std::mutex> lock(d.mu());
    pocket.stage(d);
    detail::check(gd_dock_batch(d.ctx(), &b, &k, &r));
  }
  std::vector<LigandAnalysis> out(ligands.size());
  std::vector<const Ligand*> lp;
  std::vector<const Pose*> pp;
  for (size_t l = 0; l < ligands.size(); ++l) {
    if (res.status[l] == GD_LIG_DEGENERATE) throw Error("rotate_fragment: degenerate rotation axis");
    if (res.status[l] != GD_LIG_OK) throw Error("ligand '" + ligands[l].id() + "': invalid");
    PoseResult& pr = out[l].dock;
    pr.ligand_id = ligands[l].id();
    pr.score = res.final_score[l];
    pr.evaluations = static_cast<long>(res.evals[l]);
    pr.feasibility_checks = static_cast<long>(res.checks[l]);
    const double* q = res.pose.data() + 3 * pk.atom_off[l];
    for (int i = 0; i < ligands[l].atom_count(); ++i)
      pr.final_pose.positions.push_back({q[3 * i], q[3 * i + 1], q[3 * i + 2]});
    lp.push_back(&ligands[l]);
    pp.push_back(&pr.final_pose);
  }
  std::vector<int32_t> offsets, status;
  const auto profiles = detail::profile_batch(lp, pp, pocket, offsets, status);
  for (size_t l = 0; l < ligands.size(); ++l) {
    if (status[l] == GD_LIG_DEGENERATE) throw Error("rotate_fragment: degenerate rotation axis");
    detail::fill_analysis(out[l], ligands[l], profiles, offsets[l], offsets[l + 1]);
  }
  return out;
}

}  // namespace geodock
