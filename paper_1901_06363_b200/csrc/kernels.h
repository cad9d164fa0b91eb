// Device data layout and kernel launchers shared by capi.cpp (host, g++)
// and kernels.cu (device, nvcc -fmad=false).  No CUDA headers needed here.
#pragma once

#include <cstddef>
#include <cstdint>

namespace gdb200 {

// One record per ligand; offsets index the flat SoA arrays below.
struct LigMeta {
  int32_t atom_off;   // into xyz (x3) and radii
  int32_t n;          // atoms
  int32_t frag_off;   // into frag_* arrays
  int32_t nfrag;      // 2 x rotamers, reference order (kernel.hpp:221-227)
  int32_t far_off;    // into far_mask (words)
  int32_t fmask_off;  // into frag_mask (words)
  int32_t words;      // ceil(n/64)
  int32_t status;     // GD_LIG_*
};

// One level of the exact voxel candidate-list index.  Voxel v's record is
// {int32 start, int32 count, x0, y0, z0[, x1, y1, z1, pad]}: the first
// kVoxInline candidates inline (a voxel with one candidate repeats it), the
// rest at lst[start..) as 32-byte (x, y, z, pad) records.  Two inline
// candidates (a 64-byte record, two independent 256-bit loads) spare most
// queries their dependent list load but double the record traffic; on
// config 1 that is 7% slower, so one is the default.
#ifndef GD_VOX_INLINE
#define GD_VOX_INLINE 1
#endif
constexpr int kVoxInline = GD_VOX_INLINE;
static_assert(kVoxInline == 1 || kVoxInline == 2, "1 or 2 inline candidates");
constexpr int kRecDoubles = kVoxInline == 1 ? 4 : 8;
// Coded format, chosen per pocket when its distinct coordinate values are
// few (lattice pockets: a table of at most kCodedTab doubles): a candidate
// is three 16-bit indices into that table (PocketView::tab); record {u32
// start, u32 count, 4 candidates} (32 B; entries past count are unused),
// list blocks of 5 candidates (32 B).  Each index is stored pre-scaled to
// a byte offset (8 x index).  `start` counts 32-byte units in both formats.
// Exact: the query reads the pocket's own doubles from the table.
constexpr int kCodedTab = 128;    // table capacity (1 KB, staged in shared memory: larger tables
                                  // would cost the 4-chain CTAs their sixth slot per SM)
constexpr int kCodedInline = 4;  // candidates in a coded record
constexpr int kCodedBlock = 5;   // candidates per coded list block
struct GridLevel {
  const double* rec;       // [nvox*kRecDoubles] voxel records
  const double* lst;       // [sum max(count-kVoxInline,0) * 4] further candidates, voxel-major
  double lo_x, lo_y, lo_z; // grid origin
  double inv_h;            // 1 / voxel edge
  int32_t dim_x, dim_y, dim_z;
  int32_t pad;
  double fdim_x, fdim_y, fdim_z;  // the dims as doubles (no conversion per query)
};

// Ligands of up to kNarrowAtoms atoms take the warp-per-chain kernels (8-bit
// atom indices, four mask words, chain state in shared memory); larger ones
// (up to kWideAtoms) are preprocessed on the host and searched by
// flex_wide_kernel.
constexpr int kNarrowAtoms = 256;
constexpr int kWideAtoms = 4096;  // the rigid sweep holds a ligand's atoms in shared memory

constexpr int kGridLevels = 2;  // fine (near field) + coarse (far field)
constexpr int kPhaseBase = 16;     // counters[16..32): flex phase clocks
constexpr int kCounterSlots = 32;

// Exact nearest-pocket-point structure staged in HBM.
struct PocketView {
  const double* pts;       // [P*4] x,y,z,pad (32-B records)
  int32_t P;
  int32_t use_index;       // 0 = brute force only
  int32_t compact;         // 1: coded voxel records (see below), tab set
  const double* tab;       // coded: the distinct coordinate values (x's, y's, z's)
  int32_t ntab;            // coded: table entries (<= kCodedTab)
  GridLevel lv[kGridLevels];
};

struct DockParams {
  int32_t n_lig;
  const int32_t* order;  // CTA b docks ligand order[b] (cost-descending)
  const LigMeta* meta;
  const double* xyz;       // [3*atoms] initial pose
  const double* radii;     // [atoms]
  const uint64_t* far_mask;
  const uint64_t* frag_mask;
  const int32_t* frag_axis;
  const int32_t* frag_anchor;
  const double* frag_rel;

  PocketView pocket;
  double cx, cy, cz;       // rigid-sweep centre (E1)

  // Rigid Euler grid (E2): distinct orientations, ascending linear index.
  int32_t n_orient;
  const int32_t* orient_idx;
  const double* orient_R;  // [n_orient*9] row-major
  const double* cos_deg;   // [360] std::cos(a * (pi/180)) from the host libm
  const double* sin_deg;   // [360]

  // Knobs (kernel.hpp:21-26) + batch knobs.
  int32_t hp, lp, reps, refine, tile;
  double threshold;
  int32_t top_k;           // slots per ligand in the outputs
  int32_t rigid;           // 1 = rigid sweep + top-K seeds, 0 = dock given pose
  int32_t k_slots;         // chains per ligand: min(top_k, n_orient) (1 if no sweep)
  int32_t max_n;           // largest warp-path ligand (<= kNarrowAtoms atoms) of the launch (smem sizing)
  int32_t max_pairs;       // bump-pair list capacity per warp (floor(max_n^2/4))

  // Wide ligands (more than kNarrowAtoms atoms): their chains run in
  // flex_wide_kernel, one CTA per chain, with the chain state in HBM.
  int32_t wide_pass;         // rigid sweep: 1 = this launch's ligands are the wide ones
                             // (order = wide_list); 0 = skip wide ligands
  int32_t n_wide;            // wide ligands of this launch
  const int32_t* wide_list;  // [n_wide] their ligand indices
  const int64_t* wide_off;   // [n_wide] atoms of the batch's wide ligands before ligand b: its
                             // scratch is k_slots x 8n doubles at 8 * k_slots * wide_off[b]
  double* wide_scratch;

  // Rigid -> flex hand-off (rank order).
  int32_t* seed_slot;      // [L*K] position in the orientation list
  double* seed_score;      // [L*K]
  int32_t* k_eff;          // [L]

  // Chain results in rank order (flex -> finalize).
  double* st_final;
  int64_t* st_evals;
  int64_t* st_checks;

  // Outputs, final order (E7).
  int32_t* out_orient;
  int32_t* out_rank;
  double* out_rigid;
  double* out_final;
  int64_t* out_evals;
  int64_t* out_checks;
  double* out_pose;        // nullable; [K*atoms*3]
  double* stage_pose;      // nullable; rank-order staging, same shape
  double* out_top;         // nullable; [3*atoms] each ligand's slot-0 pose (needs stage_pose)
  unsigned long long* top_best;  // nullable; [L] running max of finished chains' scores
                                 // (bits), zeroed per launch: only improving chains stage
  int64_t* poses_scored;   // [L]
  int32_t* status;         // [L]
  // Optional exact work counters: [0..6] rigid kernel, [8..14] flex kernel,
  // each {pairs, rotated atoms, bump pairs, queries, sum terms, candidate
  // evaluations, rigid-transformed atoms}; [kPhaseBase..+16) flex phase
  // clocks (GD_PHASE_CLOCKS builds).
  unsigned long long* counters;
};

// FP64 pipe probe: independent DADD/DMUL chains, returns fp64 ops executed.
int launch_fp64_probe(double* sink, int blocks, int threads, int iters, void* stream);
// L2 gather probe: random 32-byte loads over an L2-resident buffer of n_rec
// records; blocks * threads * iters * 4 loads.
int launch_l2_chase_probe(const double* buf, unsigned long long n_rec, int blocks, int threads, int iters,
                          double* sink, void* stream);
int launch_l2_gather_probe(const double* buf, unsigned long long n_rec, int blocks, int threads,
                           int iters, double* sink, void* stream);

// Launchers; return cudaError_t as int.  `stream` is a cudaStream_t.
int launch_rigid_topk(const DockParams& p, void* stream);
// One warp per (ligand, seed-rank) chain: n_lig * k_slots chains.
int launch_flex(const DockParams& p, void* stream);
// One CTA per (wide ligand, seed-rank) chain: n_wide * k_slots chains.
int launch_flex_wide(const DockParams& p, void* stream);
// Rotation profiles: one warp per (ligand, fragment) item of `items`
// ([2*n_items] ligand, fragment), 360 scores + validity flags per item.
int launch_profiles(const DockParams& p, const int32_t* items, int n_items, double* scores,
                    uint8_t* valid, void* stream);
// Fine-grained drop-in kernels over a staged batch whose ligand l carries
// one caller-given fragment (meta.nfrag == 1, frag_off == l).  Search:
// p.hp = step, p.tile = optimal_tile_size(step).
struct FragmentIO {
  int32_t refined;             // 0: optimize_fragment_flat, 1: _refined
  const double* entry_score;   // nullable [L]; NaN = not given
  int32_t* best_angle;         // [L]
  double* best_score;          // [L]
  int64_t* evaluations;        // [L]
  int64_t* checks;             // [L]
  double* pose;                // [3*atoms] committed poses
};
int launch_fragment_search(const DockParams& p, const FragmentIO& io, void* stream);
int launch_fragment_rotate(const DockParams& p, const double* cs, const double* sn,
                           const uint8_t* is_zero, double* out, void* stream);
int launch_fragment_bumps(const DockParams& p, uint8_t* feasible, void* stream);
// E7 final ordering + poses scored, one CTA per ligand.
int launch_finalize(const DockParams& p, void* stream);
// The same launchers compiled for the compact index format (GD_TU_COMPACT=1:
// flex_cp.cu, rigid_cp.cu); callers dispatch on PocketView::compact.
int launch_rigid_topk_cp(const DockParams& p, void* stream);
int launch_flex_cp(const DockParams& p, void* stream);
int launch_flex_wide_cp(const DockParams& p, void* stream);
int launch_profiles_cp(const DockParams& p, const int32_t* items, int n_items, double* scores,
                       uint8_t* valid, void* stream);
int launch_fragment_search_cp(const DockParams& p, const FragmentIO& io, void* stream);
int launch_score_poses(const PocketView& pk, const double* xyz, int n_atoms, int n_poses,
                       double* out, void* stream);

// Ligand preprocessing on the GPU (prep.cu), ligands [l0, l1) of a batch.
// The host fills meta[] except nfrag/status (status pre-set to 1 for atom
// counts outside [2, kMaxAtoms]) with far_off = prefix of n*words,
// frag_off = 2 * first bond, fmask_off = prefix of 2 * bonds * words; the
// kernel writes status[] (and meta.status / nfrag), the far masks and the
// fragments, and order[l0..l1) = the ligands longest-first.
struct PrepParams {
  int32_t l0, l1;
  int32_t max_n;           // largest atom count (<= kMaxAtoms) in [l0, l1)
  LigMeta* meta;
  const int32_t* boff;     // [L+1] bond offsets
  const int32_t* bonds;    // [2*bonds] ligand-local atom pairs
  const uint8_t* rot;      // [bonds] Bond::rotatable
  const double* xyz;       // [3*atoms]
  const double* radii;     // [atoms]
  uint64_t* far;
  uint64_t* fmask;
  int32_t* fax;
  int32_t* fan;
  double* frel;
  int32_t* status;         // [L] per-ligand status (GD_LIG_*)
  int32_t* order;          // [L] CTA order
};
size_t prep_smem_per_warp(int max_n);
int launch_prep(const PrepParams& q, void* stream);

// Voxel index build (two passes: count, then fill after a host scan).
struct VoxelGrid {
  double lo_x, lo_y, lo_z, h;
  int32_t dim_x, dim_y, dim_z;
  int32_t overflow = 1024;  // more survivors than this: the voxel lists the whole pocket
                            // (<= 1024; lowered only by tests, GD_VOXEL_OVERFLOW)
};
// counts[v] = candidates of voxel v (>= 1), or -1 when more than 1,024
// survive (the voxel then scans the whole pocket, held once at the head of
// the list array); the fill pass writes each voxel's record and its
// candidates past the inline ones at the device-scanned list offsets.
// tbox [nt][6] (lo xyz, hi xyz; fp32, outward-rounded) are the bounding
// boxes of the Morton-ordered points' 32-point tiles: with nt > 0 the build
// culls tiles per 4x4x8 voxel brick (pocket_index.cu); nt = 0 scans all.
// keep [nv][8] (nullable): the count pass stores each voxel's first 8
// candidates there and the fill pass copies them instead of recomputing.
int launch_voxel_count(const double* pts, int P, VoxelGrid g, int32_t* counts, const float* tbox,
                       int nt, int32_t* keep, void* stream);
int launch_voxel_fill(const double* pts, int P, VoxelGrid g, const int32_t* offsets, double* rec,
                      double* lst, const float* tbox, int nt, const int32_t* counts,
                      const int32_t* keep, const uint16_t* codes, void* stream);
// codes (nullable) [P][3]: the coded format's table indices of each point.
// offsets[v] = base + exclusive prefix of the voxels' list units (32 B:
// max(counts - kVoxInline, 0) fp64 entries, or ceil(max(counts - 4, 0) / 5)
// coded blocks) over voxels (the first `base` units hold the whole pocket
// for overflow voxels); totals[3] (device) = {list units incl. base,
// candidates, max count}; `scratch` holds list_offsets_scratch_bytes(nv).
int list_offsets_scratch_bytes(int nv);
int launch_list_offsets(const int32_t* counts, int nv, int P, long long base, int compact,
                        int32_t* offsets, void* scratch, long long* totals, void* stream);

}  // namespace gdb200
