/*
 * geodock_b200.h -- C-ABI of the B200-native GeoDock-MA pose-search hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, integer return
 * codes, no exceptions and no torch types.  Every entry point names the
 * reference interface (under /root/reference/proj/include/geodock/) it
 * replaces.  The C++ drop-in header <geodock_b200/geodock.hpp> maps these
 * calls back onto the reference's own C++ API (geodock::match_probes_shape,
 * geodock::screen, geodock::overlap_score, ...), including its exception
 * messages; bindings for other hosts (ctypes, cgo, JNI) bind this file.
 *
 * Numerics: every score, coordinate and decision is computed in fp64 with
 * the reference's exact expression trees (no FMA contraction, atom-order
 * sums, host-built trig tables), so results are bit-identical to the
 * reference CPU path.  See DESIGN.md.
 *
 * Threading: one gd_ctx per device, not thread-safe per context.
 */
#ifndef GEODOCK_B200_H
#define GEODOCK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  GD_ERR_INVALID/GD_ERR_DEGENERATE map onto geodock::Error
 * (reference error.hpp:14-17); the message is in gd_last_error(). */
#define GD_OK 0
#define GD_ERR_INVALID 1    /* argument / validation failure            */
#define GD_ERR_CUDA 2       /* CUDA runtime failure (device, OOM, ...)  */
#define GD_ERR_DEGENERATE 3 /* degenerate rotation axis (geometry.hpp:168) */
#define GD_ERR_NO_POCKET 4  /* gd_set_pocket not called                 */

/* Per-ligand status codes written to gd_result.status. */
#define GD_LIG_OK 0
#define GD_LIG_INVALID 1    /* Ligand ctor validation failed (molecule.hpp:66-115) */
#define GD_LIG_DEGENERATE 3 /* rotate_fragment threw "degenerate rotation axis"   */

/* gd_knobs.flags */
#define GD_FLAG_BRUTE_FORCE 1u /* scan every pocket point instead of the voxel index */
#define GD_FLAG_KEEP_POSES 2u  /* gd_dock_resident: keep final poses for gd_download */
#define GD_FLAG_COUNT_WORK 4u  /* count executed work (gd_work_counters) */
#define GD_FLAG_TOP_POSE 16u   /* gd_dock_resident: keep each ligand's top-1 pose
                                  for gd_download's top_pose */

typedef struct gd_ctx gd_ctx;

/* A batch of ligands, SoA, caller-owned; copied in by the call.
 * Mirrors geodock::Ligand(id, atoms, bonds) (molecule.hpp:45-50) and the
 * initial pose make_initial_pose (geometry.hpp:23-28). */
typedef struct {
  int32_t n_ligands;
  const int32_t* atom_offsets;   /* [n_ligands+1] prefix sums of atom counts      */
  const double* xyz;             /* [total_atoms*3] initial pose, Angstrom         */
  const double* radii;           /* [total_atoms] Angstrom, > 0                    */
  const int32_t* bond_offsets;   /* [n_ligands+1] prefix sums of bond counts       */
  const int32_t* bonds;          /* [total_bonds*2] ligand-local atom indices a,b  */
  const uint8_t* bond_rotatable; /* [total_bonds] Bond::rotatable                  */
} gd_ligand_batch;

/* The five reference knobs (KnobConfig, kernel.hpp:21-26) plus the three
 * north-star knobs of the batch path. */
typedef struct {
  int32_t high_precision_step; /* KnobConfig::high_precision_step */
  int32_t low_precision_step;  /* KnobConfig::low_precision_step  */
  double threshold;            /* KnobConfig::threshold           */
  int32_t repetitions;         /* KnobConfig::repetitions (restarts) */
  int32_t enable_refinement;   /* KnobConfig::enable_refinement   */
  int32_t rigid_step;          /* degrees of the rigid Euler grid; 0 = no sweep:
                                  dock the given pose (reference screen semantics) */
  int32_t top_k;               /* poses kept per ligand (>= 1)    */
  uint32_t flags;              /* GD_FLAG_*                       */
} gd_knobs;

/* Caller-allocated results, ligand-major, top_k slots per ligand.  Slot
 * (l, e) lives at index l*top_k + e, sorted by (final score desc, seed rank
 * asc); slots e >= k_eff[l] are zero with orientation = -2. */
typedef struct {
  int32_t* orientation;          /* [L*K] Euler-grid linear index, -1 = given pose  */
  int32_t* seed_rank;            /* [L*K] rank of the seed in the rigid top-K        */
  double* rigid_score;           /* [L*K] overlap score of the rigid seed pose       */
  double* final_score;           /* [L*K] PoseResult::score                          */
  int64_t* evaluations;          /* [L*K] PoseResult::evaluations                    */
  int64_t* feasibility_checks;   /* [L*K] PoseResult::feasibility_checks             */
  double* final_pose;            /* optional (NULL): [K*total_atoms*3]; ligand l,
                                    slot e at (K*atom_offsets[l] + e*n_l)*3         */
  int32_t* k_eff;                /* [L] min(top_k, distinct orientations) (1 if no sweep) */
  int64_t* poses_scored;         /* [L] rigid orientations scored + sum evaluations  */
  int32_t* status;               /* [L] GD_LIG_*                                     */
  double* top_pose;              /* optional (NULL): [total_atoms*3], ligand l's
                                    top-1 final pose (PoseResult::final_pose of slot
                                    0) at atom_offsets[l]*3; zeros if skipped        */
} gd_result;

/* Device-side timing of the last gd_dock_* call (CUDA events on the
 * context stream). */
typedef struct {
  float upload_ms;     /* H2D of descriptors (0 for gd_dock_resident)  */
  float rigid_ms;      /* rigid sweep + top-K kernel                   */
  float flex_ms;       /* fragment-optimisation/restart kernel         */
  float download_ms;   /* D2H of results                               */
  float total_ms;      /* first to last event                          */
  int64_t rigid_atom_queries; /* atoms x orientations scored in the sweep */
  int64_t flex_atom_queries;  /* fragment-atom nearest-point queries      */
  int64_t launches;    /* kernels launched by the call                 */
  int64_t h2d_bytes;   /* bytes copied host->device by the last upload */
  int64_t d2h_bytes;   /* bytes copied device->host by the last download */
  float host_prep_ms;  /* host wall time: messages of rejected ligands (the
                          validation and graph preprocessing run on the GPU) */
  float host_pack_ms;  /* host wall time: offsets + raw atoms/bonds into pinned staging */
  float host_post_ms;  /* host wall time: result download + bookkeeping */
} gd_timing;

/* ---- context ------------------------------------------------------------ */
int gd_create(int device, gd_ctx** out);
int gd_destroy(gd_ctx* ctx);
/* Message of the last failed call on ctx (or of gd_create when ctx is NULL). */
const char* gd_last_error(const gd_ctx* ctx);
/* Run kernels on this cudaStream_t (NULL = the context's own stream). */
int gd_set_stream(gd_ctx* ctx, void* cuda_stream);
const char* gd_version(void);

/* ---- pocket ------------------------------------------------------------- */
/* Stages the pocket in HBM and builds the exact voxel nearest-point index.
 * Replaces geodock::Pocket(id, points) validation (molecule.hpp:152-157)
 * and PocketIndex(pocket) (geometry.hpp:49-65).  Also fixes the rigid-sweep
 * centre c = (sum_j P_j)/P, summed in index order (E1).  The
 * context caches the last GD_POCKET_CACHE (env, default 16) pockets by
 * their coordinates: re-staging one of them is a lookup, not a rebuild. */
int gd_set_pocket(gd_ctx* ctx, const double* xyz, int32_t n_points);
/* Centre and index statistics of the staged pocket. */
int gd_pocket_info(const gd_ctx* ctx, double centre[3], int32_t dims[3], double* voxel,
                   int64_t* n_candidates, int32_t* max_candidates);
/* Per level of the staged pocket's exact voxel index (0 = fine near field,
 * 1 = coarse far field): grid dims, voxel edge (A), candidates, and the
 * HBM bytes of its voxel records and candidate lists. */
typedef struct {
  int32_t dims[3];
  double voxel;
  int64_t candidates;
  int64_t record_bytes;
  int64_t list_bytes;
} gd_index_level;
int gd_pocket_index_stats(const gd_ctx* ctx, gd_index_level out[2]);
/* Record format of the staged pocket's index: 1 = coded (the pocket's
 * distinct coordinate values fit a 128-entry table, e.g. lattice pockets:
 * 32-byte records with four candidates inline as table indices), 0 = fp64
 * records; GD_ERR_NO_POCKET without a pocket.  Both are exact; the choice
 * is made per pocket by gd_set_pocket (GD_INDEX_COMPACT=0 forces fp64). */
int gd_pocket_index_format(const gd_ctx* ctx);
/* Record format of the staged pocket's index: 1 = coded (the pocket's
 * distinct coordinate values fit a 128-entry table, e.g. lattice pockets:
 * 32-byte records with four candidates inline as table indices), 0 = fp64
 * records; GD_ERR_NO_POCKET without a pocket.  Both are exact; the choice
 * is made per pocket by gd_set_pocket (GD_INDEX_COMPACT=0 forces fp64). */
int gd_pocket_index_format(const gd_ctx* ctx);

/* ---- batch docking (the hot path) --------------------------------------- */
/* Host buffers in, host buffers out: validate + preprocess (Ligand ctor,
 * find_rotamers, grow_fragments; molecule.hpp:45-301), H2D, rigid sweep,
 * top-K, K x match_probes_shape (kernel.hpp:205-248), final ordering, D2H.
 * With rigid_step == 0 and top_k == 1 this is geodock::screen
 * (screening.hpp:96-178) without the thread pool. */
int gd_dock_batch(gd_ctx* ctx, const gd_ligand_batch* batch, const gd_knobs* knobs,
                  gd_result* result);

/* Split form used to time the device-resident path: gd_upload preprocesses
 * and copies a batch into HBM (kept in the context, replacing any previous
 * one); gd_dock_resident runs the kernels on it; gd_download copies the
 * results of the last gd_dock_resident into `result`. */
int gd_upload(gd_ctx* ctx, const gd_ligand_batch* batch);
int gd_dock_resident(gd_ctx* ctx, const gd_knobs* knobs);
int gd_download(gd_ctx* ctx, gd_result* result);
int gd_last_timing(const gd_ctx* ctx, gd_timing* out);

/* ---- multi-device dispatch ------------------------------------------------- */
/* One process driving several GPUs: a gd_ctx, a host thread and its streams
 * per device.  gd_multi_dock_batch cuts the batch into chunks of equal
 * estimated cost (n (N_orient + K reps (1 + 2R 360/hp)) per ligand, about
 * four per device) that the device threads pull from a shared cursor --
 * the reference screen's work queue (screening.hpp:96-178) with GPUs as the
 * workers -- and writes every chunk's results into the caller's arrays at
 * the chunk's global offsets.  Results are bit-identical to gd_dock_batch
 * on one context, for any device count.  The same device may be listed
 * twice (two contexts on one GPU).  Host preprocessing threads are shared
 * out: each context gets host CPUs / devices. */
typedef struct gd_multi gd_multi;
typedef struct {
  int64_t ligands;  /* ligands docked by this device in the last call */
  int64_t chunks;   /* chunks it pulled */
  float busy_ms;    /* host wall time inside its gd_dock_batch calls */
} gd_multi_stats;
/* devices[n_devices] (CUDA ordinals), or devices == NULL: the first
 * n_devices visible GPUs (n_devices <= 0: all of them). */
int gd_multi_create(const int32_t* devices, int32_t n_devices, gd_multi** out);
int gd_multi_destroy(gd_multi* m);
const char* gd_multi_last_error(const gd_multi* m);  /* NULL m: gd_multi_create's */
int32_t gd_multi_size(const gd_multi* m);
/* Context i (for the fine-grained and diagnostic entry points); owned by m. */
gd_ctx* gd_multi_context(gd_multi* m, int32_t i);
/* gd_set_pocket on every device, in parallel. */
int gd_multi_set_pocket(gd_multi* m, const double* xyz, int32_t n_points);
/* gd_dock_batch over every device (same arguments and result layout). */
int gd_multi_dock_batch(gd_multi* m, const gd_ligand_batch* batch, const gd_knobs* knobs,
                        gd_result* result);
/* gd_ligand_error for the last gd_multi_dock_batch, by batch position. */
int gd_multi_ligand_error(const gd_multi* m, int32_t ligand, char* msg, size_t msg_len);
/* Per-device statistics of the last gd_multi_dock_batch: out[min(cap, size)]. */
int gd_multi_last_stats(const gd_multi* m, gd_multi_stats* out, int32_t cap);

/* ---- planner (host) ------------------------------------------------------ */
/* The seven interaction features (perf_model.hpp:36-47) of one dataset
 * summary {pocket points, avg atoms, avg rotamers}: x[7]. */
void gd_cost_features(const double* features, double* x);
/* fit (perf_model.hpp:57-105): OLS of seconds per ligand on the seven
 * features plus an intercept, column-pivoting Householder QR.  features:
 * n x 3 summaries; times: n seconds per ligand; out: coef[7], intercept,
 * adjusted R^2.  GD_ERR_INVALID with the reference's message in msg for
 * n < 9, a non-positive time or a rank-deficient design ("collinear
 * columns: ..."). */
int gd_fit_cost_model(const double* features, const double* times, int32_t n, double* coef,
                      double* intercept, double* adjusted_r2, char* msg, size_t msg_len);

/* ---- ligand graph (host) ------------------------------------------------ */
/* The batch path's host preprocessing of one ligand, exposed for the C++
 * drop-in: Ligand validation (molecule.hpp:66-115; the reference's message
 * goes to msg), find_rotamers (molecule.hpp:237-250: rotamer_bonds[r] =
 * Ligand::bonds() index of rotamer r) and grow_fragments membership
 * (molecule.hpp:255-301: membership[(2r + side) * n + i], side 0 = left).
 * Capacities: rotamer_bonds >= n_bonds, membership >= 2 * n_bonds * n.
 * Returns GD_LIG_OK or GD_LIG_INVALID. */
int gd_ligand_graph(int32_t n_atoms, const double* xyz, const double* radii, int32_t n_bonds,
                    const int32_t* bonds, const uint8_t* rotatable, int32_t* n_rotamers,
                    int32_t* rotamer_bonds, uint8_t* membership, char* msg, size_t msg_len);

/* ---- rotation profiles (analysis) --------------------------------------- */
/* rotation_profile (analysis.hpp:37-56) of every fragment of the batch staged
 * by the last gd_upload (or gd_dock_batch), from each ligand's pose in that
 * batch's xyz.
 * Fragments are numbered ligand by ligand in the reference order (rotamer r
 * -> left 2r, right 2r+1; kernel.hpp:221-227).  For fragment f and integer
 * angle a: valid[360 f + a] = check_bumps of the pose with the fragment
 * rotated by a degrees (angle 0 = the pose itself), scores[360 f + a] its
 * overlap_score where valid and 0 elsewhere.  frag_offsets[L+1] receives
 * the per-ligand fragment prefix (skipped ligands have none);
 * relative_size[f] (nullable) Fragment::relative_size; status[L] (nullable)
 * GD_LIG_* per ligand (GD_LIG_DEGENERATE: a fragment's axis is degenerate,
 * its profile is all-invalid; a ligand of more than 256 atoms is reported
 * GD_LIG_INVALID with no fragments -- the docking entry points take such
 * ligands, this warp-per-fragment kernel does not).  `capacity` is in fragments; twice the
 * number of rotatable bonds always suffices.  flags: GD_FLAG_BRUTE_FORCE,
 * GD_FLAG_COUNT_WORK (work lands in gd_work_counters' flex slots); the
 * kernel time goes to gd_last_timing's flex_ms. */
int gd_rotation_profiles(gd_ctx* ctx, uint32_t flags, double* scores, uint8_t* valid,
                         double* relative_size, int32_t* frag_offsets, int32_t* status,
                         int64_t capacity);

/* One peak of a rotation profile (analysis.hpp:25-29). */
typedef struct {
  int32_t start_angle;  /* first angle of the run (circular) */
  int32_t width;        /* degrees */
  double height_ratio;  /* (peak max - min) / delta, in [0, 1] */
} gd_peak;
/* detect_peaks (analysis.hpp:61-126) on one 360-angle profile: a peak is a
 * maximal circularly-contiguous run of valid angles scoring strictly above
 * min + delta/2; runs through 359 -> 0 merge.  peaks needs room for 180.
 * Returns GD_ERR_INVALID when no angle is valid (the reference throws
 * "detect_peaks: no feasible rotation"). */
int gd_detect_peaks(const double* scores, const uint8_t* valid, double* delta_overlap,
                    int32_t* best_peak_width, gd_peak* peaks, int32_t* n_peaks);
/* tile_hit_probability (analysis.hpp:133-147): per tile size, the fraction
 * of profiles whose best peak is wider than the tile and the two-phase
 * evaluation count 360/tile + tile.  GD_ERR_INVALID on an empty dataset. */
int gd_tile_hit_probability(const int32_t* best_peak_widths, int64_t n, const int32_t* tiles,
                            int32_t n_tiles, double* probability, double* eval_count);

/* Why ligand `ligand` (batch position) of the last gd_upload / gd_dock_batch
 * was skipped with GD_LIG_INVALID: the reference's Ligand validation text
 * (molecule.hpp:66-115) with the batch position as the ligand id, e.g.
 * "ligand '17': duplicate bond", or this path's size limit "ligand '17':
 * more than 4096 atoms is not supported" (docking entry points; 256 for the
 * fine-grained fragment and profile entry points).  Empty for accepted ligands;
 * GD_LIG_DEGENERATE means the reference's "rotate_fragment: degenerate
 * rotation axis" (geometry.hpp:168). */
int gd_ligand_error(const gd_ctx* ctx, int32_t ligand, char* msg, size_t msg_len);

/* Device-resident results of the last gd_dock_resident (valid until the
 * next dock call): every gd_result field except the poses, in the same
 * layout and with the same empty-slot values (orientation -2, zeros).  Lets
 * a multi-GPU host gather per-ligand top-K tables over NCCL without a host
 * round trip. */
typedef struct {
  const int32_t* orientation;        /* [n_ligands*top_k] as gd_result  */
  const int32_t* seed_rank;          /* [n_ligands*top_k]               */
  const double* final_score;         /* [n_ligands*top_k]               */
  const int64_t* evaluations;        /* [n_ligands*top_k]               */
  int32_t n_ligands;
  int32_t top_k;
  const double* rigid_score;         /* [n_ligands*top_k]               */
  const int64_t* feasibility_checks; /* [n_ligands*top_k]               */
  const int32_t* k_eff;              /* [n_ligands]                     */
  const int64_t* poses_scored;       /* [n_ligands]                     */
  const int32_t* status;             /* [n_ligands] GD_LIG_*            */
} gd_device_result;
int gd_device_results(const gd_ctx* ctx, gd_device_result* out);
/* Exact work executed by the last call made with GD_FLAG_COUNT_WORK:
 * out[0..6] rigid kernel, out[8..14] flex kernel, each {point pairs, rotated
 * atoms, bump pairs, nearest-point queries, score-sum terms, candidate
 * evaluations, rigid-transformed atoms}.  DESIGN.md §4 turns them into FLOPs. */
int gd_work_counters(const gd_ctx* ctx, uint64_t out[16]);
/* Diagnostic: SM clock cycles the flex kernel's warps spent per phase in
 * the last GD_FLAG_COUNT_WORK call, summed over warps: out[0] chain start,
 * [1] step setup (axis, fragment list, prefix), [2] bump-pair prefilter,
 * [3] term pre-fill, [4] bump checks, [5] nearest-point queries, [6] score
 * folds, [7] search decisions, [8] commit.  All zero unless the library was
 * built with -DGD_PHASE_CLOCKS=1 (GD_DEFS); the clocks cost registers, so
 * such builds are for attribution, not timing. */
int gd_phase_clocks(const gd_ctx* ctx, uint64_t out[16]);
/* Measures this device's fp64 DADD/DMUL issue rate (TFLOP/s, no FMA) with
 * a probe kernel; the denominator of the fp64 roofline. */
int gd_fp64_peak(gd_ctx* ctx, double* tflops);
/* Measures this device's L2 random-gather rate (GB/s): 32-byte read-only
 * loads, not allocated in L1, at random over an L2-resident 48 MB buffer --
 * the access pattern of the voxel-index gathers; the denominator of the
 * L2-gather roofline. */
int gd_l2_gather_peak(gd_ctx* ctx, double* gbs);
/* Latency-bound counterpart (diagnostic): the same random 32-byte gathers
 * with ONE dependent load in flight per thread and warps_per_sm resident
 * warps per SM (e.g. the flex kernel's 24): what a kernel whose lanes each
 * wait on their own gather can reach at that residency (GB/s). */
int gd_l2_gather_rate(gd_ctx* ctx, int32_t warps_per_sm, double* gbs);

/* ---- fine-grained kernels ------------------------------------------------ */
/* overlap_score (geometry.hpp:140-155) of n_poses poses of n_atoms atoms
 * each, xyz pose-major [n_poses*n_atoms*3]. */
int gd_overlap_score_batch(gd_ctx* ctx, const double* xyz, int32_t n_atoms, int32_t n_poses,
                           uint32_t flags, double* out_scores);

/* One caller-given fragment per ligand of a batch (reference Fragment,
 * molecule.hpp:177-185): membership[atom_offsets[l] + i] = 1 when atom i of
 * ligand l is in its fragment (Fragment::membership; the fragment's atoms
 * are the set members in ascending order, Fragment::atom_indices), and the
 * rotation axis runs from axis_atom[l] (the bond endpoint inside the
 * fragment) to anchor_atom[l] (the endpoint on the other side). */
typedef struct {
  const uint8_t* membership; /* [total_atoms] */
  const int32_t* axis_atom;  /* [n_ligands] ligand-local atom index */
  const int32_t* anchor_atom;/* [n_ligands] ligand-local atom index */
} gd_fragment_set;

/* The fine-grained entry points below stage `batch` (replacing any staged
 * batch: gd_rotation_profiles needs a fresh gd_upload afterwards), validate
 * and preprocess every ligand as the batch path does, and run one warp per
 * ligand on that ligand's pose (batch xyz) and fragment.  Per-ligand
 * outcomes land in status[L] (GD_LIG_OK, GD_LIG_INVALID with the text in
 * gd_ligand_error, GD_LIG_DEGENERATE for "rotate_fragment: degenerate
 * rotation axis", geometry.hpp:168).  A fragment with an axis/anchor atom
 * out of range, axis == anchor, or holding no atom or every atom fails the
 * call with GD_ERR_INVALID. */

/* optimize_fragment_flat (kernel.hpp:125-143; refined == 0, `step` must
 * divide 360: "optimize_fragment_flat: step must divide 360") or
 * optimize_fragment_refined (kernel.hpp:150-198; refined != 0, step = the
 * high-precision step, "optimize_fragment_refined: step must divide 360")
 * of each ligand's fragment against the staged pocket.  entry_score
 * (nullable [L]; NaN = not given) is the refined search's optional entry
 * score.  Out [L]: FragmentSearchResult {best_angle, best_score} and the
 * SearchCounters {evaluations, feasibility_checks} (kernel.hpp:77-85);
 * out_pose [total_atoms*3]: the pose committed to the best angle
 * (commit_angle, kernel.hpp:115-117).  Bit-identical to the reference. */
int gd_optimize_fragment_batch(gd_ctx* ctx, const gd_ligand_batch* batch,
                               const gd_fragment_set* fragments, int32_t step, int32_t refined,
                               const double* entry_score, int32_t* best_angle, double* best_score,
                               int64_t* evaluations, int64_t* feasibility_checks,
                               double* out_pose, int32_t* status);

/* rotate_fragment_into / rotate_fragment (geometry.hpp:161-193): each
 * ligand's pose with its fragment rotated by angles_deg[l] degrees (any
 * double; cos/sin from the host libm exactly as the reference evaluates
 * them; angle 0 is an exact copy) into out_pose [total_atoms*3].  Needs no
 * pocket. */
int gd_rotate_fragment_batch(gd_ctx* ctx, const gd_ligand_batch* batch,
                             const gd_fragment_set* fragments, const double* angles_deg,
                             double* out_pose, int32_t* status);

/* check_bumps (geometry.hpp:199-213) of each ligand's pose against its
 * fragment: feasible[l] = 0 iff a fragment atom i and a non-fragment atom j
 * at capped graph distance >= 4 sit closer than 0.8 (r_i + r_j).  Needs no
 * pocket. */
int gd_check_bumps_batch(gd_ctx* ctx, const gd_ligand_batch* batch,
                         const gd_fragment_set* fragments, uint8_t* feasible, int32_t* status);

/* ---- host helpers (no device work) --------------------------------------- */
/* optimal_tile_size (kernel.hpp:62-75); returns -1 when step < 1. */
int32_t gd_optimal_tile_size(int32_t high_precision_step);
/* KnobConfig::validate (kernel.hpp:28-38) + batch-knob checks.  Returns
 * GD_OK or GD_ERR_INVALID with the reference message copied to msg. */
int gd_validate_knobs(const gd_knobs* knobs, char* msg, size_t msg_len);
/* Distinct orientations of the rigid Euler grid (E2): writes up
 * to cap linear indices (ascending) and, if R != NULL, their row-major 3x3
 * matrices; returns the count or -1 when step does not divide 360. */
int32_t gd_orientations(int32_t rigid_step, int32_t* indices, double* R, int32_t cap);

/* ---- synthetic BASELINE data (tools; not the hot path) ------------------ */
/* Lattice ellipsoid pocket, points in (i,j,k) lexicographic order, centred
 * at the origin; rough_max > 0 removes a seeded U(0, rough_max) fraction of
 * the outermost points.  Returns the point count (writes at most cap). */
int32_t gd_synth_pocket(double a, double b, double c, double spacing, double rough_max,
                        uint64_t seed, double* xyz, int32_t cap);
/* Sizes of ligand `id` of the seeded random-walk-tree family: n ~ U{n_lo..n_hi}
 * (or fixed_n > 0), rotatable bonds R ~ U{0..min(r_cap, n/4)} (or fixed_r >= 0). */
int gd_synth_ligand_size(uint64_t base_seed, int64_t id, int32_t n_lo, int32_t n_hi,
                         int32_t fixed_n, int32_t* n_atoms);
/* Ligand `id`: writes n atoms (xyz, radii) and n-1 bonds; centroid moved to
 * `centre`.  Returns the number of rotatable bonds. */
int gd_synth_ligand(uint64_t base_seed, int64_t id, int32_t n_lo, int32_t n_hi, int32_t fixed_n,
                    int32_t r_cap, int32_t fixed_r, const double centre[3], double* xyz,
                    double* radii, int32_t* bonds, uint8_t* rotatable);

#ifdef __cplusplus
}
#endif
#endif /* GEODOCK_B200_H */
