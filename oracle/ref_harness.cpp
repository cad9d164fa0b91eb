// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the reference GeoDock-MA headers straight from
// /root/reference/proj/include (never copied into this repo; see
// oracle/Makefile) and exposes them through extern "C" entry points with the
// same array layout as the product C-ABI (include/geodock_b200.h):
//   * gdref_dock_batch: E1-E8 built only on reference calls --
//     geodock::overlap_score (geometry.hpp:140) for the rigid sweep and
//     geodock::match_probes_shape (kernel.hpp:205) per seed -- with an
//     optional geodock::PocketIndex and a std::thread pool like
//     geodock::screen (screening.hpp:96-178).  This is bench.py's reference
//     arm and the generator of tests/golden fixtures.
//   * gdref_rotation_profiles / gdref_detect_peaks / gdref_tile_hits: the
//     reference analysis (analysis.hpp:37-147) over a batch, in the layout
//     of gd_rotation_profiles -- the parity anchor of that C-ABI entry.
//   * fine-grained wrappers for known-answer tests.
// Only the Eigen-free headers are included.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "geodock/analysis.hpp"
#include "geodock/geometry.hpp"
#include "geodock/kernel.hpp"
#include "geodock/molecule.hpp"
#include "geodock/screening.hpp"
#include "geodock/synthetic.hpp"
#include "geodock_b200.h"

extern "C" int gdo_orientations(int step, int** idx_out, double** R_out);
extern "C" void gdo_free(void* p);

namespace {

thread_local std::string g_err;

geodock::Ligand make_ligand(const std::string& id, int n, const double* xyz, const double* radii,
                            int nb, const int32_t* bonds, const uint8_t* rot) {
  std::vector<geodock::Atom> atoms;
  atoms.reserve(n);
  for (int i = 0; i < n; ++i)
    atoms.push_back({i, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]}, radii[i]});
  std::vector<geodock::Bond> bs;
  bs.reserve(nb);
  for (int b = 0; b < nb; ++b) bs.push_back({bonds[2 * b], bonds[2 * b + 1], rot[b] != 0});
  return geodock::Ligand(id, std::move(atoms), std::move(bs));
}

geodock::Pocket make_pocket(const double* pts, int P) {
  std::vector<geodock::Vec3> v;
  v.reserve(P);
  for (int j = 0; j < P; ++j) v.push_back({pts[3 * j], pts[3 * j + 1], pts[3 * j + 2]});
  return geodock::Pocket("pocket", std::move(v));
}

geodock::KnobConfig knobs_of(const gd_knobs* k) {
  return geodock::KnobConfig{k->high_precision_step, k->low_precision_step, k->threshold,
                             k->repetitions, k->enable_refinement != 0};
}

struct Entry {
  double s;
  int i;
};
bool entry_less(const Entry& a, const Entry& b) { return a.s > b.s || (a.s == b.s && a.i < b.i); }

}  // namespace

extern "C" const char* gdref_last_error() { return g_err.c_str(); }

extern "C" double gdref_overlap_score(const double* xyz, int n, const double* pocket, int P,
                                      int use_index) {
  geodock::Pose pose;
  for (int i = 0; i < n; ++i) pose.positions.push_back({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
  const geodock::Pocket pk = make_pocket(pocket, P);
  if (use_index) {
    const geodock::PocketIndex index(pk);
    return geodock::overlap_score(pose, pk, &index);
  }
  return geodock::overlap_score(pose, pk);
}

extern "C" int gdref_optimal_tile_size(int step) { return geodock::optimal_tile_size(step); }

// match_probes_shape on the given pose.  Returns 0, or 1 on geodock::Error
// (message in gdref_last_error()).
extern "C" int gdref_match_probes_shape(int n, const double* xyz, const double* radii, int nb,
                                        const int32_t* bonds, const uint8_t* rot,
                                        const double* pocket, int P, const gd_knobs* k,
                                        int use_index, double* pose_out, double* score,
                                        long long* evals, long long* checks) {
  try {
    const geodock::Ligand lig = make_ligand("L", n, xyz, radii, nb, bonds, rot);
    const geodock::Pocket pk = make_pocket(pocket, P);
    std::unique_ptr<geodock::PocketIndex> index;
    if (use_index) index = std::make_unique<geodock::PocketIndex>(pk);
    const geodock::PoseResult r =
        geodock::match_probes_shape(lig, pk, geodock::make_initial_pose(lig), knobs_of(k), index.get());
    for (int i = 0; i < n; ++i) {
      pose_out[3 * i] = r.final_pose.positions[i].x;
      pose_out[3 * i + 1] = r.final_pose.positions[i].y;
      pose_out[3 * i + 2] = r.final_pose.positions[i].z;
    }
    *score = r.score;
    *evals = r.evaluations;
    *checks = r.feasibility_checks;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// rotate_fragment + check_bumps on fragment f (rotamer f/2, left if even).
extern "C" int gdref_rotate_fragment(int n, const double* xyz, const double* radii, int nb,
                                     const int32_t* bonds, const uint8_t* rot, const double* pose,
                                     int f, double angle_deg, double* out, int* feasible) {
  try {
    const geodock::Ligand lig = make_ligand("L", n, xyz, radii, nb, bonds, rot);
    const auto rots = geodock::find_rotamers(lig);
    if (f < 0 || f >= 2 * static_cast<int>(rots.size())) throw geodock::Error("no such fragment");
    const auto frags = geodock::grow_fragments(lig, rots[f / 2]);
    const geodock::Fragment& fr = (f % 2 == 0) ? frags.first : frags.second;
    geodock::Pose p;
    for (int i = 0; i < n; ++i) p.positions.push_back({pose[3 * i], pose[3 * i + 1], pose[3 * i + 2]});
    const geodock::Pose r = geodock::rotate_fragment(p, lig, fr, angle_deg);
    for (int i = 0; i < n; ++i) {
      out[3 * i] = r.positions[i].x;
      out[3 * i + 1] = r.positions[i].y;
      out[3 * i + 2] = r.positions[i].z;
    }
    if (feasible) *feasible = geodock::check_bumps(r, lig, fr) ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// optimize_fragment_flat / optimize_fragment_refined (kernel.hpp:125-198)
// on fragment f (rotamer f/2, left if even) from `pose`, with the
// reference's SearchCounters and optional entry score (has_entry).
extern "C" int gdref_optimize_fragment(int n, const double* xyz, const double* radii, int nb,
                                       const int32_t* bonds, const uint8_t* rot,
                                       const double* pocket, int P, const double* pose, int f,
                                       int refined, int step, int has_entry, double entry_score,
                                       double* pose_out, int* best_angle, double* best_score,
                                       long long* evals, long long* checks) {
  try {
    const geodock::Ligand lig = make_ligand("L", n, xyz, radii, nb, bonds, rot);
    const geodock::Pocket pk = make_pocket(pocket, P);
    const auto rots = geodock::find_rotamers(lig);
    if (f < 0 || f >= 2 * static_cast<int>(rots.size())) throw geodock::Error("no such fragment");
    const auto frags = geodock::grow_fragments(lig, rots[f / 2]);
    const geodock::Fragment& fr = (f % 2 == 0) ? frags.first : frags.second;
    geodock::Pose p;
    for (int i = 0; i < n; ++i) p.positions.push_back({pose[3 * i], pose[3 * i + 1], pose[3 * i + 2]});
    geodock::SearchCounters c;
    const geodock::FragmentSearchResult r =
        refined ? geodock::optimize_fragment_refined(
                      p, lig, fr, pk, step, &c,
                      has_entry ? std::optional<double>(entry_score) : std::nullopt)
                : geodock::optimize_fragment_flat(p, lig, fr, pk, step, &c);
    for (int i = 0; i < n; ++i) {
      pose_out[3 * i] = p.positions[i].x;
      pose_out[3 * i + 1] = p.positions[i].y;
      pose_out[3 * i + 2] = p.positions[i].z;
    }
    *best_angle = r.best_angle;
    *best_score = r.best_score;
    *evals = c.evaluations;
    *checks = c.feasibility_checks;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reference generator (synthetic.hpp:71-188) for fixture datasets, sizes
// first: call with null outputs to get counts.
extern "C" int gdref_generate_synthetic(int count, uint64_t seed, int atom_lo, int atom_hi,
                                        int rot_lo, int rot_hi, int pocket_points,
                                        double pocket_radius, int* total_atoms, int* total_bonds,
                                        double* pocket, int32_t* atom_off, double* xyz,
                                        double* radii, int32_t* bond_off, int32_t* bonds,
                                        uint8_t* rot) {
  geodock::DatasetSpec spec;
  spec.ligand_count = count;
  spec.atom_min = atom_lo;
  spec.atom_max = atom_hi;
  spec.rotamer_min = rot_lo;
  spec.rotamer_max = rot_hi;
  spec.pocket_points = pocket_points;
  spec.pocket_radius = pocket_radius;
  spec.seed = seed;
  std::optional<geodock::SyntheticDataset> maybe;
  try {
    maybe.emplace(geodock::generate_synthetic(spec));
  } catch (const std::exception& e) {  // infeasible spec: report, do not abort
    g_err = e.what();
    return -1;
  }
  const auto& ds = *maybe;
  int ta = 0, tb = 0;
  for (const auto& l : ds.ligands) {
    ta += l.atom_count();
    tb += static_cast<int>(l.bonds().size());
  }
  *total_atoms = ta;
  *total_bonds = tb;
  if (xyz == nullptr) return 0;
  for (int j = 0; j < pocket_points; ++j) {
    pocket[3 * j] = ds.pocket.points()[j].x;
    pocket[3 * j + 1] = ds.pocket.points()[j].y;
    pocket[3 * j + 2] = ds.pocket.points()[j].z;
  }
  int a = 0, b = 0;
  for (int l = 0; l < count; ++l) {
    const auto& lig = ds.ligands[l];
    atom_off[l] = a;
    bond_off[l] = b;
    for (const auto& at : lig.atoms()) {
      xyz[3 * a] = at.position.x;
      xyz[3 * a + 1] = at.position.y;
      xyz[3 * a + 2] = at.position.z;
      radii[a++] = at.radius;
    }
    for (const auto& bd : lig.bonds()) {
      bonds[2 * b] = bd.a;
      bonds[2 * b + 1] = bd.b;
      rot[b++] = bd.rotatable ? 1 : 0;
    }
  }
  atom_off[count] = a;
  bond_off[count] = b;
  return 0;
}

// E1-E8 over a batch with reference calls; same layout as gd_dock_batch.
extern "C" int gdref_dock_batch(const gd_ligand_batch* b, const double* pocket, int P,
                                const gd_knobs* k, int threads, int use_index, gd_result* r) {
  const geodock::Pocket pk = make_pocket(pocket, P);
  std::unique_ptr<geodock::PocketIndex> index;
  if (use_index) index = std::make_unique<geodock::PocketIndex>(pk);
  // E1: centre, index-order sum.
  double c[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < P; ++j)
    for (int d = 0; d < 3; ++d) c[d] += pocket[3 * j + d];
  for (double& v : c) v /= P;
  const bool rigid = k->rigid_step > 0;
  int* oidx = nullptr;
  double* oR = nullptr;
  const int n_orient = rigid ? gdo_orientations(k->rigid_step, &oidx, &oR) : 0;
  const int K = rigid ? k->top_k : 1;
  const geodock::KnobConfig cfg = knobs_of(k);
  std::atomic<int> next{0};

  auto dock_one = [&](int l) {
    const int a0 = b->atom_offsets[l], n = b->atom_offsets[l + 1] - a0;
    const int b0 = b->bond_offsets[l], nb = b->bond_offsets[l + 1] - b0;
    for (int e = 0; e < K; ++e) {
      const size_t d = static_cast<size_t>(l) * K + e;
      if (r->orientation) r->orientation[d] = -2;
      if (r->seed_rank) r->seed_rank[d] = 0;
      if (r->rigid_score) r->rigid_score[d] = 0.0;
      if (r->final_score) r->final_score[d] = 0.0;
      if (r->evaluations) r->evaluations[d] = 0;
      if (r->feasibility_checks) r->feasibility_checks[d] = 0;
      if (r->final_pose && n > 0)
        std::memset(r->final_pose + 3 * (static_cast<size_t>(K) * a0 + static_cast<size_t>(e) * n), 0,
                    sizeof(double) * 3 * n);
    }
    if (r->k_eff) r->k_eff[l] = 0;
    if (r->poses_scored) r->poses_scored[l] = 0;
    std::optional<geodock::Ligand> lig;
    try {
      lig.emplace(make_ligand("L" + std::to_string(l), n, b->xyz + 3 * a0, b->radii + a0, nb,
                              b->bonds + 2 * b0, b->bond_rotatable + b0));
    } catch (const std::exception&) {
      if (r->status) r->status[l] = GD_LIG_INVALID;
      return;
    }
    geodock::Pose given = geodock::make_initial_pose(*lig);
    std::vector<Entry> seeds;
    std::vector<geodock::Pose> seed_pose;
    auto rigid_pose = [&](int o) {
      geodock::Pose p;
      p.positions.reserve(n);
      const double* R = oR + 9 * o;
      for (const geodock::Vec3& q : given.positions) {
        const double vx = q.x - c[0], vy = q.y - c[1], vz = q.z - c[2];
        p.positions.push_back({c[0] + (R[0] * vx + R[1] * vy + R[2] * vz),
                               c[1] + (R[3] * vx + R[4] * vy + R[5] * vz),
                               c[2] + (R[6] * vx + R[7] * vy + R[8] * vz)});
      }
      return p;
    };
    if (rigid) {
      seeds.resize(n_orient);
      for (int o = 0; o < n_orient; ++o) seeds[o] = {geodock::overlap_score(rigid_pose(o), pk, index.get()), o};
      const int keff = std::min(K, n_orient);
      std::partial_sort(seeds.begin(), seeds.begin() + keff, seeds.end(), entry_less);  // E5
      seeds.resize(keff);
    } else {
      seeds.push_back({geodock::overlap_score(given, pk, index.get()), -1});
    }
    std::vector<geodock::PoseResult> res;
    long long scored = rigid ? n_orient : 0;
    try {
      for (const Entry& s : seeds) {  // E6
        res.push_back(geodock::match_probes_shape(*lig, pk, rigid ? rigid_pose(s.i) : given, cfg,
                                                  index.get()));
        scored += res.back().evaluations;
      }
    } catch (const std::exception&) {
      if (r->status) r->status[l] = GD_LIG_DEGENERATE;
      return;
    }
    std::vector<Entry> fin(res.size());
    for (size_t s = 0; s < res.size(); ++s) fin[s] = {res[s].score, static_cast<int>(s)};
    std::sort(fin.begin(), fin.end(), entry_less);  // E7
    for (size_t e = 0; e < fin.size(); ++e) {
      const int s = fin[e].i;
      const size_t d = static_cast<size_t>(l) * K + e;
      if (r->orientation) r->orientation[d] = rigid ? oidx[seeds[s].i] : -1;
      if (r->seed_rank) r->seed_rank[d] = s;
      if (r->rigid_score) r->rigid_score[d] = seeds[s].s;
      if (r->final_score) r->final_score[d] = res[s].score;
      if (r->evaluations) r->evaluations[d] = res[s].evaluations;
      if (r->feasibility_checks) r->feasibility_checks[d] = res[s].feasibility_checks;
      if (r->final_pose) {
        double* dst = r->final_pose + 3 * (static_cast<size_t>(K) * a0 + e * n);
        for (int i = 0; i < n; ++i) {
          dst[3 * i] = res[s].final_pose.positions[i].x;
          dst[3 * i + 1] = res[s].final_pose.positions[i].y;
          dst[3 * i + 2] = res[s].final_pose.positions[i].z;
        }
      }
    }
    if (r->k_eff) r->k_eff[l] = static_cast<int>(fin.size());
    if (r->poses_scored) r->poses_scored[l] = scored;
    if (r->status) r->status[l] = 0;
  };

  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t)
    pool.emplace_back([&] {
      for (int l; (l = next.fetch_add(1)) < b->n_ligands;) dock_one(l);
    });
  for (auto& t : pool) t.join();
  gdo_free(oidx);
  gdo_free(oR);
  return 0;
}

// geodock::rotation_profile of every fragment of every ligand, from each
// ligand's batch pose, numbered like gd_rotation_profiles (ligand order,
// rotamer r -> left 2r, right 2r+1).  A ligand that fails the Ligand ctor
// gets status 1 and no fragments; a fragment whose rotation throws
// (degenerate axis) sets status 3 and is reported all-invalid.  Returns the
// number of fragments, or -1 when `capacity` is too small.
extern "C" long long gdref_rotation_profiles(const gd_ligand_batch* b, const double* pocket, int P,
                                             int use_index, int threads, double* scores,
                                             uint8_t* valid, double* rel, int32_t* frag_offsets,
                                             int32_t* status, long long capacity) {
  const geodock::Pocket pk = make_pocket(pocket, P);
  std::unique_ptr<geodock::PocketIndex> index;
  if (use_index) index = std::make_unique<geodock::PocketIndex>(pk);
  const int L = b->n_ligands;
  std::vector<std::optional<geodock::Ligand>> ligs(L);
  std::vector<std::vector<geodock::Rotamer>> rots(L);
  frag_offsets[0] = 0;
  for (int l = 0; l < L; ++l) {
    const int a0 = b->atom_offsets[l], n = b->atom_offsets[l + 1] - a0;
    const int b0 = b->bond_offsets[l], nb = b->bond_offsets[l + 1] - b0;
    status[l] = GD_LIG_OK;
    try {
      ligs[l].emplace(make_ligand("L" + std::to_string(l), n, b->xyz + 3 * a0, b->radii + a0, nb,
                                  b->bonds + 2 * b0, b->bond_rotatable + b0));
      rots[l] = geodock::find_rotamers(*ligs[l]);
    } catch (const std::exception&) {
      ligs[l].reset();
      status[l] = GD_LIG_INVALID;
    }
    frag_offsets[l + 1] = frag_offsets[l] + (ligs[l] ? 2 * static_cast<int>(rots[l].size()) : 0);
  }
  if (frag_offsets[L] > capacity) return -1;
  std::atomic<int> next{0};
  auto work = [&] {
    for (int l; (l = next.fetch_add(1)) < L;) {
      if (!ligs[l]) continue;
      const geodock::Ligand& lig = *ligs[l];
      const geodock::Pose pose = geodock::make_initial_pose(lig);
      for (size_t ri = 0; ri < rots[l].size(); ++ri) {
        const auto frags = geodock::grow_fragments(lig, rots[l][ri]);
        const geodock::Fragment* fs[2] = {&frags.first, &frags.second};
        for (int side = 0; side < 2; ++side) {
          const long long f = frag_offsets[l] + 2 * static_cast<long long>(ri) + side;
          rel[f] = fs[side]->relative_size;
          try {
            const geodock::RotationProfile pr =
                geodock::rotation_profile(pose, lig, *fs[side], pk, index.get());
            for (int a = 0; a < 360; ++a) {
              scores[360 * f + a] = pr.scores[a];
              valid[360 * f + a] = pr.valid[a] ? 1 : 0;
            }
          } catch (const std::exception&) {
            status[l] = GD_LIG_DEGENERATE;
            for (int a = 0; a < 360; ++a) {
              scores[360 * f + a] = 0.0;
              valid[360 * f + a] = 0;
            }
          }
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < std::max(1, threads); ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return frag_offsets[L];
}

// geodock::detect_peaks on one profile.  Returns 0, or 1 when it throws (no
// feasible rotation; message in gdref_last_error()).  Peaks go to
// starts/widths/heights (capacity 360, ordered as the reference orders them).
extern "C" int gdref_detect_peaks(const double* scores, const uint8_t* valid, double* delta,
                                  int* best_width, int* n_peaks, int32_t* starts, int32_t* widths,
                                  double* heights) {
  geodock::RotationProfile pr;
  for (int a = 0; a < 360; ++a) {
    pr.scores[a] = scores[a];
    pr.valid[a] = valid[a] != 0;
  }
  try {
    const geodock::PeakStats st = geodock::detect_peaks(pr);
    *delta = st.delta_overlap;
    *best_width = st.best_peak_width;
    *n_peaks = static_cast<int>(st.peaks.size());
    for (size_t k = 0; k < st.peaks.size(); ++k) {
      starts[k] = st.peaks[k].start_angle;
      widths[k] = st.peaks[k].width;
      heights[k] = st.peaks[k].height_ratio;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// geodock::tile_hit_probability over datasets given by their best peak widths.
extern "C" int gdref_tile_hits(const int32_t* best_widths, int n, const int32_t* tiles, int nt,
                               double* probability, double* eval_count) {
  std::vector<geodock::PeakStats> ds(n);
  for (int i = 0; i < n; ++i) ds[i].best_peak_width = best_widths[i];
  try {
    const auto hits = geodock::tile_hit_probability(ds, std::vector<int>(tiles, tiles + nt));
    for (int k = 0; k < nt; ++k) {
      probability[k] = hits[k].probability;
      eval_count[k] = hits[k].eval_count;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// geodock::find_rotamers + grow_fragments: rotamer bond indices and the
// fragments' membership (row 2r = left, 2r+1 = right).  Returns the rotamer
// count, or -1 when the Ligand ctor throws (message in gdref_last_error()).
extern "C" int gdref_ligand_graph(int n, const double* xyz, const double* radii, int nb,
                                  const int32_t* bonds, const uint8_t* rot, int32_t* rot_bonds,
                                  uint8_t* membership) {
  try {
    const geodock::Ligand lig = make_ligand("L", n, xyz, radii, nb, bonds, rot);
    const auto rots = geodock::find_rotamers(lig);
    for (size_t r = 0; r < rots.size(); ++r) {
      rot_bonds[r] = rots[r].bond_index;
      const auto fr = geodock::grow_fragments(lig, rots[r]);
      for (int i = 0; i < n; ++i) {
        membership[(2 * r) * n + i] = fr.first.membership[i] ? 1 : 0;
        membership[(2 * r + 1) * n + i] = fr.second.membership[i] ? 1 : 0;
      }
    }
    return static_cast<int>(rots.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
