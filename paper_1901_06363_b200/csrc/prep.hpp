// Host-side ligand preprocessing for the device descriptors.
//
// Restates, in native C++, what the reference does once per ligand before
// the search starts:
//   * Ligand::validate / build_adjacency / build_capped_distances
//     (reference molecule.hpp:66-140): validation messages, BFS
//     connectivity, all-pairs bond-graph distances capped at 4;
//   * find_rotamers (molecule.hpp:237-250): rotatable bridge bonds ordered
//     by (min endpoint, max endpoint), bridges by DFS lowpoints (:190-231);
//   * grow_fragments (molecule.hpp:255-301): left = component of the
//     smaller endpoint, relative_size = |F|/n, axis/anchor atoms.
// The result is packed as bitmasks (ceil(n / 64) words per row) for the kernels.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gdb200 {

constexpr int kMaxAtoms = 256;  // 4 x 64-bit mask words: the GPU preprocessing and the warp-per-chain kernels
constexpr int kMaxWords = kMaxAtoms / 64;
constexpr int kGraphDistanceCap = 4;  // molecule.hpp:43, geometry.hpp:40

struct PreparedLigand {
  int n = 0;
  int words = 0;  // ceil(n / 64)
  int status = 0; // GD_LIG_*
  std::string error;
  std::vector<uint64_t> far_mask;     // n*words: bit j of row i set iff capped(i,j) >= 4
  // Fragments in reference order: for each rotamer (sorted), left then right.
  std::vector<int32_t> rot_bond;      // bond index of each rotamer, find_rotamers order
  std::vector<int32_t> frag_axis, frag_anchor, frag_size;
  std::vector<double> frag_rel;       // relative_size = double(|F|) / n
  std::vector<uint64_t> frag_mask;    // nfrag*words membership bits
  int nfrag() const { return static_cast<int>(frag_axis.size()); }
};

// Validates and preprocesses one ligand given SoA atoms and bonds.
// `id` only feeds error messages ("ligand '<id>': ...", as the reference).
// Ligands of more than `max_atoms` atoms are rejected ("more than <max_atoms>
// atoms is not supported"): kMaxAtoms for the warp-per-chain kernels'
// callers, kernels.h's kWideAtoms for the batch docking path.
PreparedLigand prepare_ligand(const std::string& id, int n, const double* xyz, const double* radii,
                              int n_bonds, const int32_t* bonds, const uint8_t* rotatable,
                              int max_atoms = kMaxAtoms);

}  // namespace gdb200
