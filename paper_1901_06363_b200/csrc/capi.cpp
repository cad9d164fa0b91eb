// C-ABI of the B200 pose-search path (include/geodock_b200.h).
//
// Host runtime: validation and preprocessing (prep.cpp), pinned staging,
// one CUDA stream per context, the voxel index build, and the two hot-path
// launches (rigid_topk_kernel, flex_kernel).  No CPU fallback exists: every
// score comes from the kernels in kernels.cu.
#include <cuda_runtime.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "geodock_b200.h"
#include "kernels.h"
#include "orient.hpp"
#include "prep.hpp"

using namespace gdb200;

namespace {

thread_local std::string g_create_error;

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (ptr) cudaFree(ptr);
  }
  // Grows geometrically (x1.5): pockets and batches of slowly rising size
  // must not pay a cudaFree + cudaMalloc each (those stall for hundreds of
  // ms when large allocations are live).
  cudaError_t ensure(size_t n) {
    if (n <= bytes && ptr) return cudaSuccess;
    const size_t want = std::max<size_t>({n, 256, bytes + bytes / 2});
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e != cudaSuccess && want > n) {  // tight on memory: exactly n
      cudaGetLastError();
      e = cudaMalloc(&ptr, std::max<size_t>(n, 256));
      if (e == cudaSuccess) bytes = std::max<size_t>(n, 256);
      return e;
    }
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

struct PinnedBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes && ptr) return cudaSuccess;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    const cudaError_t e = cudaHostAlloc(&ptr, std::max<size_t>(n, 256), cudaHostAllocDefault);
    if (e == cudaSuccess) bytes = std::max<size_t>(n, 256);
    return e;
  }
};

double env_double(const char* name, double dflt) {
  const char* v = std::getenv(name);
  return v ? std::atof(v) : dflt;
}

}  // namespace

namespace {

// Host threads for one context: GD_HOST_THREADS, else the CPUs this process
// may run on divided among the node's ranks (LOCAL_WORLD_SIZE, set by
// torchrun), so one-process-per-GPU runs do not oversubscribe the host.
static int host_threads() {
  if (const char* e = std::getenv("GD_HOST_THREADS")) {
    const int v = std::atoi(e);
    if (v > 0) return v;
  }
  int cpus = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  cpu_set_t set;
  if (sched_getaffinity(0, sizeof set, &set) == 0) cpus = std::max(1, CPU_COUNT(&set));
  int ranks = 1;
  if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) ranks = std::max(1, std::atoi(e));
  return std::max(1, cpus / ranks);
}

// Persistent host workers for ligand preprocessing: run(fn) executes fn on
// every worker and on the caller and returns when all have finished (fn
// pulls its items from a shared atomic cursor).  Created once per context,
// so a pipelined batch does not pay thread creation per chunk.
class WorkerPool {
 public:
  explicit WorkerPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void run(const std::function<void()>& fn) {
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &fn;
      busy_ = static_cast<int>(th_.size());
      ++gen_;
    }
    cv_.notify_all();
    fn();
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return busy_ == 0; });
  }

 private:
  void loop() {
    int seen = 0;
    for (;;) {
      const std::function<void()>* job;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      (*job)();
      std::lock_guard<std::mutex> g(mu_);
      if (--busy_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void()>* job_ = nullptr;
  int gen_ = 0, busy_ = 0;
  bool stop_ = false;
};

}  // namespace

// One staged pocket: its points (Morton order) and exact voxel index in
// HBM, plus the host copy that identifies it.  A context keeps up to
// GD_POCKET_CACHE (default 16) of them, so screens that alternate pockets
// (config 3's 16 pockets, the drop-in's Pocket objects) re-stage a pocket
// by lookup instead of rebuilding its index.
struct PocketSlot {
  std::vector<double> host;  // caller's xyz, the identity key
  uint64_t hash = 0;
  uint64_t last_use = 0;
  int32_t P = 0;
  double centre[3] = {0, 0, 0};
  DevBuf pts, vox_off[kGridLevels], vox_pts[kGridLevels], tab;
  VoxelGrid grid[kGridLevels] = {};
  int64_t n_cand = 0;
  int32_t max_cand = 0;
  gd_index_level stats[kGridLevels] = {};
  PocketView view{};
};

struct gd_ctx {
  int device = 0;
  int pool_threads = 0;  // host preprocessing threads (0: host_threads())
  cudaStream_t own_stream = nullptr;
  std::vector<cudaStream_t> aux_streams;  // further streams of the pipelined gd_dock_batch
  cudaStream_t stream = nullptr;
  std::string err;
  cudaEvent_t ev[5] = {};
  std::vector<cudaEvent_t> chunk_ev;       // one per pipelined chunk (no timing)
  std::unique_ptr<WorkerPool> pool;        // host preprocessing workers

  // Pocket: the active slot and its mirrors (P == 0: none staged), the
  // slot cache, and the index build's scratch.
  std::vector<std::unique_ptr<PocketSlot>> slots;
  uint64_t use_clock = 0;
  int32_t P = 0;
  double centre[3] = {0, 0, 0};
  VoxelGrid grid[kGridLevels] = {};
  int64_t n_cand = 0;
  int32_t max_cand = 0;
  PocketView view{};
  DevBuf tiles, vox_counts, vox_doff, vox_keep, vox_scan, vox_codes;

  DevBuf cos_t, sin_t;
  int orient_step = -1;
  int32_t n_orient = 0;
  std::vector<int32_t> orient_idx_host;
  DevBuf orient_idx, orient_R;

  // Resident batch.
  int32_t n_lig = 0;
  int32_t total_atoms = 0;
  int32_t max_n = 0;
  int max_nfrag = 0;
  std::vector<int32_t> atom_off;
  std::vector<int32_t> status_host;
  std::vector<std::string> errors;
  DevBuf meta, xyz, radii, bonds, rot, boff;  // staged raw ligands (+ host-filled offsets)
  DevBuf far, fmask, fax, fan, frel, order;   // written by the GPU preprocessing
  size_t frag_total = 0;                      // fragment slots allocated (2 x bonds)
  // Wide ligands (more than kNarrowAtoms atoms) of the staged batch, ascending:
  // preprocessed on the host (prepare_ligand) while their chunk is packed,
  // searched by flex_wide_kernel with per-chain scratch in HBM.
  std::vector<int32_t> wide_idx;               // ligand indices
  std::vector<int64_t> wide_pref;              // atoms of the wide ligands before each
  std::vector<PreparedLigand> wide_prep;       // host descriptors (uploaded per chunk)
  DevBuf wide_list_d, wide_off_d, wide_scratch;
  PinnedBuf staging;
  PinnedBuf res_staging;         // pinned D2H targets of gd_dock_batch
  unsigned char* pin[10] = {};   // per-segment pointers into staging

  // Outputs of the last gd_dock_resident.
  int32_t last_topk = 0;
  bool last_rigid = false;
  bool last_pose = false;
  bool last_top = false;
  bool have_result = false;
  DevBuf counters;
  bool counted = false;
  DevBuf prof_items, prof_scores, prof_valid;
  bool staged = false;  // a batch is staged (gd_upload / gd_dock_batch)
  DevBuf st_final, st_evals, st_checks;
  DevBuf seed_slot, seed_score, k_eff, o_orient, o_rank, o_rigid, o_final, o_evals, o_checks,
      o_pose, stage_pose, o_top, top_best, o_scored, o_status;
  std::vector<double> initial_score;  // given-pose mode: rigid_score column

  gd_timing timing{};

  int fail(int code, std::string msg) {
    err = std::move(msg);
    return code;
  }
  int cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return GD_OK;
    return fail(GD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
};

#define GD_CUDA(ctx, expr)                          \
  do {                                              \
    const int _rc = (ctx)->cuda((expr), #expr);     \
    if (_rc != GD_OK) return _rc;                   \
  } while (0)

extern "C" const char* gd_version(void) { return "geodock_b200 0.1 (sm_100a, fp64 exact)"; }

extern "C" int gd_create(int device, gd_ctx** out) {
  if (out == nullptr) {
    g_create_error = "gd_create: null output pointer";
    return GD_ERR_INVALID;
  }
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    g_create_error = std::string("gd_create: no CUDA device: ") + cudaGetErrorString(e);
    return GD_ERR_CUDA;
  }
  if (device < 0 || device >= count) {
    g_create_error = "gd_create: device index out of range";
    return GD_ERR_INVALID;
  }
  auto* ctx = new gd_ctx();
  ctx->device = device;
  e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  for (int i = 0; i < 5 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev[i]);
  if (e != cudaSuccess) {
    g_create_error = std::string("gd_create: ") + cudaGetErrorString(e);
    delete ctx;
    return GD_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  std::vector<double> c, s;
  trig_tables(c, s);
  if (ctx->cos_t.ensure(360 * sizeof(double)) != cudaSuccess ||
      ctx->sin_t.ensure(360 * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(ctx->cos_t.ptr, c.data(), 360 * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(ctx->sin_t.ptr, s.data(), 360 * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    g_create_error = "gd_create: trig table upload failed";
    delete ctx;
    return GD_ERR_CUDA;
  }
  *out = ctx;
  return GD_OK;
}

extern "C" int gd_destroy(gd_ctx* ctx) {
  if (ctx == nullptr) return GD_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (cudaEvent_t ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : ctx->chunk_ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  for (cudaStream_t st : ctx->aux_streams) cudaStreamDestroy(st);
  delete ctx;
  return GD_OK;
}

extern "C" const char* gd_last_error(const gd_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

extern "C" int gd_set_stream(gd_ctx* ctx, void* cuda_stream) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
  return GD_OK;
}

extern "C" int32_t gd_optimal_tile_size(int32_t step) {
  // kernel.hpp:62-75: argmin over divisors x of step*(360/x) + x, smaller x on ties.
  if (step < 1) return -1;
  long best = -1;
  int32_t tile = 360;
  for (int x = 1; x <= 360; ++x) {
    if (360 % x) continue;
    const long v = static_cast<long>(step) * (360 / x) + x;
    if (best < 0 || v < best) {
      best = v;
      tile = x;
    }
  }
  return tile;
}

extern "C" int gd_validate_knobs(const gd_knobs* k, char* msg, size_t msg_len) {
  const char* m = nullptr;
  if (k == nullptr) m = "knob config: null";
  // KnobConfig::validate (kernel.hpp:28-38), same order and messages.
  else if (k->high_precision_step < 1 || 360 % k->high_precision_step != 0)
    m = "knob config: high-precision step must be a divisor of 360";
  else if (k->low_precision_step < 1 || 360 % k->low_precision_step != 0)
    m = "knob config: low-precision step must be a divisor of 360";
  else if (k->low_precision_step < k->high_precision_step)
    m = "knob config: low-precision step must be >= high-precision step";
  else if (!(k->threshold >= 0.0 && k->threshold <= 1.0))
    m = "knob config: threshold must be in [0,1]";
  else if (k->repetitions < 1)
    m = "knob config: repetitions must be >= 1";
  else if (k->rigid_step < 0 || (k->rigid_step > 0 && 360 % k->rigid_step != 0))
    m = "knob config: rigid step must be 0 or a divisor of 360";
  else if (k->top_k < 1 || k->top_k > 256)
    m = "knob config: top_k must be in [1,256]";
  if (m == nullptr) return GD_OK;
  if (msg && msg_len) {
    std::strncpy(msg, m, msg_len - 1);
    msg[msg_len - 1] = 0;
  }
  return GD_ERR_INVALID;
}

extern "C" int32_t gd_orientations(int32_t step, int32_t* indices, double* R, int32_t cap) {
  if (step < 1 || 360 % step != 0) return -1;
  std::vector<int32_t> idx;
  std::vector<double> mats;
  rigid_orientations(step, idx, mats);
  const int32_t n = static_cast<int32_t>(idx.size());
  for (int32_t i = 0; i < std::min(n, cap); ++i) {
    if (indices) indices[i] = idx[i];
    if (R) std::memcpy(R + 9 * i, mats.data() + 9 * i, 9 * sizeof(double));
  }
  return n;
}

// ---------------------------------------------------------------------------
// Pocket staging and the voxel index.
// ---------------------------------------------------------------------------
extern "C" int gd_set_pocket(gd_ctx* ctx, const double* xyz, int32_t n) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  // Pocket ctor validation (molecule.hpp:152-157).
  if (n < 1 || xyz == nullptr) return ctx->fail(GD_ERR_INVALID, "pocket: needs at least 1 point");
  for (int32_t j = 0; j < 3 * n; ++j)
    if (!std::isfinite(xyz[j])) return ctx->fail(GD_ERR_INVALID, "pocket: non-finite point");
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  // Cache lookup: FNV-1a of the coordinate bytes, confirmed by comparison.
  uint64_t hash = 1469598103934665603ull;
  {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(xyz);
    for (size_t i = 0; i < sizeof(double) * 3 * static_cast<size_t>(n); ++i)
      hash = (hash ^ b[i]) * 1099511628211ull;
  }
  auto activate = [ctx](PocketSlot& sl) {
    sl.last_use = ++ctx->use_clock;
    ctx->P = sl.P;
    for (int k = 0; k < 3; ++k) ctx->centre[k] = sl.centre[k];
    for (int L = 0; L < kGridLevels; ++L) ctx->grid[L] = sl.grid[L];
    ctx->n_cand = sl.n_cand;
    ctx->max_cand = sl.max_cand;
    ctx->view = sl.view;
  };
  for (auto& sl : ctx->slots)
    if (sl->P == n && sl->hash == hash &&
        std::memcmp(sl->host.data(), xyz, sizeof(double) * 3 * static_cast<size_t>(n)) == 0) {
      activate(*sl);
      return GD_OK;
    }
  static const size_t kCache = static_cast<size_t>(std::max(1.0, env_double("GD_POCKET_CACHE", 16)));
  PocketSlot* slot = nullptr;
  if (ctx->slots.size() < kCache) {
    ctx->slots.push_back(std::make_unique<PocketSlot>());
    slot = ctx->slots.back().get();
  } else {  // least recently used
    slot = std::min_element(ctx->slots.begin(), ctx->slots.end(), [](const auto& a, const auto& b) {
             return a->last_use < b->last_use;
           })->get();
  }
  slot->P = 0;  // invalid until the build completes
  slot->hash = hash;
  slot->host.assign(xyz, xyz + 3 * static_cast<size_t>(n));
  ctx->P = 0;
  // E1: centre = (sum_j P_j) / P, summed in index order.
  double sx = 0.0, sy = 0.0, sz = 0.0, lo[3], hi[3];
  for (int k = 0; k < 3; ++k) lo[k] = hi[k] = xyz[k];
  for (int32_t j = 0; j < n; ++j) {
    sx += xyz[3 * j];
    sy += xyz[3 * j + 1];
    sz += xyz[3 * j + 2];
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], xyz[3 * j + k]);
      hi[k] = std::max(hi[k], xyz[3 * j + k]);
    }
  }
  slot->centre[0] = sx / n;
  slot->centre[1] = sy / n;
  slot->centre[2] = sz / n;

  // Device copy of the points in Morton order (10 bits per axis over the
  // bounding box): every use is a minimum over points, so the order is
  // free, and 32-point tiles become spatially compact for the culled index
  // build (pocket_index.cu), which gets their outward-rounded fp32 boxes.
  std::vector<std::pair<uint32_t, int32_t>> key(n);
  auto spread = [](uint32_t x) {  // 10 bits -> every third bit
    x &= 0x3ff;
    x = (x | (x << 16)) & 0x030000ff;
    x = (x | (x << 8)) & 0x0300f00f;
    x = (x | (x << 4)) & 0x030c30c3;
    x = (x | (x << 2)) & 0x09249249;
    return x;
  };
  for (int32_t j = 0; j < n; ++j) {
    uint32_t c[3];
    for (int k = 0; k < 3; ++k) {
      const double ext = hi[k] - lo[k];
      c[k] = ext > 0 ? static_cast<uint32_t>(std::min(1023.0, (xyz[3 * j + k] - lo[k]) / ext * 1023.0)) : 0;
    }
    key[j] = {spread(c[0]) | (spread(c[1]) << 1) | (spread(c[2]) << 2), j};
  }
  std::sort(key.begin(), key.end());
  std::vector<double> padded(4 * static_cast<size_t>(n), 0.0);
  for (int32_t q = 0; q < n; ++q)
    for (int k = 0; k < 3; ++k) padded[4 * q + k] = xyz[3 * key[q].second + k];
  GD_CUDA(ctx, slot->pts.ensure(padded.size() * sizeof(double)));
  GD_CUDA(ctx, cudaMemcpy(slot->pts.ptr, padded.data(), padded.size() * sizeof(double),
                          cudaMemcpyHostToDevice));
  static const bool kCull = env_double("GD_VOXEL_CULL", 1) != 0;
  const int n_tiles = kCull ? (n + 31) / 32 : 0;
  std::vector<float> tbox(6 * static_cast<size_t>(std::max(n_tiles, 1)), 0.0f);
  for (int t = 0; t < n_tiles; ++t) {
    double blo[3], bhi[3];
    for (int k = 0; k < 3; ++k) blo[k] = bhi[k] = padded[4 * (32 * t) + k];
    for (int q = 32 * t; q < std::min(n, 32 * t + 32); ++q)
      for (int k = 0; k < 3; ++k) {
        blo[k] = std::min(blo[k], padded[4 * q + k]);
        bhi[k] = std::max(bhi[k], padded[4 * q + k]);
      }
    for (int k = 0; k < 3; ++k) {
      float fl = static_cast<float>(blo[k]), fh = static_cast<float>(bhi[k]);
      if (static_cast<double>(fl) > blo[k]) fl = std::nextafter(fl, -INFINITY);
      if (static_cast<double>(fh) < bhi[k]) fh = std::nextafter(fh, INFINITY);
      tbox[6 * t + k] = fl;
      tbox[6 * t + 3 + k] = fh;
    }
  }
  // Coded index records when the pocket's distinct coordinate values fit a
  // small table (lattice pockets; kernels.h): the table (x values, then y,
  // then z, each ascending) and each point's three indices into it.
  // GD_INDEX_COMPACT=0 forces the fp64 records (read per call).
  bool compact = env_double("GD_INDEX_COMPACT", 1) != 0;
  std::vector<double> tab;
  std::vector<uint16_t> codes;
  if (compact) {
    int base[3];
    std::vector<double> axis[3];
    for (int k = 0; k < 3 && compact; ++k) {
      axis[k].resize(n);
      for (int32_t j = 0; j < n; ++j) axis[k][j] = padded[4 * j + k];
      std::sort(axis[k].begin(), axis[k].end());
      axis[k].erase(std::unique(axis[k].begin(), axis[k].end(),
                                [](double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }),
                    axis[k].end());
      base[k] = static_cast<int>(tab.size());
      tab.insert(tab.end(), axis[k].begin(), axis[k].end());
      compact = tab.size() <= static_cast<size_t>(kCodedTab);
    }
    if (compact) {
      codes.resize(3 * static_cast<size_t>(n));
      for (int32_t j = 0; j < n; ++j)
        for (int k = 0; k < 3; ++k) {
          const double x = padded[4 * j + k];
          const size_t at = std::lower_bound(axis[k].begin(), axis[k].end(), x) - axis[k].begin();
          codes[3 * j + k] = static_cast<uint16_t>(8 * (base[k] + at));  // byte offset
        }
    }
  }
  std::vector<uint16_t> head;  // coded list head: points 4.. of the pocket in blocks of 5
  if (compact) {
    const int32_t rest = std::max(n - kCodedInline, 0);
    head.assign(16 * static_cast<size_t>((rest + kCodedBlock - 1) / kCodedBlock), 0);
    for (int32_t b = 0; b < rest; ++b)
      for (int k = 0; k < 3; ++k)
        head[16 * (b / kCodedBlock) + 3 * (b % kCodedBlock) + k] = codes[3 * (kCodedInline + b) + k];
    // The kernels stage the table with one fixed-size bulk copy (stage_tab):
    // the device copy is always kCodedTab doubles, zero-padded.
    std::vector<double> full(tab);
    full.resize(kCodedTab, 0.0);
    GD_CUDA(ctx, slot->tab.ensure(sizeof(double) * full.size()));
    GD_CUDA(ctx, cudaMemcpy(slot->tab.ptr, full.data(), sizeof(double) * full.size(), cudaMemcpyHostToDevice));
    GD_CUDA(ctx, ctx->vox_codes.ensure(sizeof(uint16_t) * codes.size()));
    GD_CUDA(ctx, cudaMemcpy(ctx->vox_codes.ptr, codes.data(), sizeof(uint16_t) * codes.size(),
                            cudaMemcpyHostToDevice));
  }
  GD_CUDA(ctx, ctx->tiles.ensure(tbox.size() * sizeof(float)));
  GD_CUDA(ctx, cudaMemcpy(ctx->tiles.ptr, tbox.data(), tbox.size() * sizeof(float),
                          cudaMemcpyHostToDevice));

  // Two grid levels over the pocket bounding box: a fine near field (voxel
  // 0.2 A, margin 3 A) and a coarse far field (0.75 A, margin 32 A); queries
  // beyond both fall back to the exact full scan.
  PocketView& v = slot->view;
  v.pts = slot->pts.as<double>();
  v.P = n;
  v.use_index = 1;
  v.compact = compact ? 1 : 0;
  v.tab = compact ? slot->tab.as<double>() : nullptr;
  v.ntab = compact ? static_cast<int32_t>(tab.size()) : 0;
  slot->n_cand = 0;
  slot->max_cand = 0;
  // Edges/margins from A/B on config 1 (profiles/r1_voxel_ab.md, DESIGN
  // §10): 0.2 A fine / 0.75 A far-field voxels.  A level whose grid would
  // exceed kMaxVoxels grows its edge (x1.25 steps) until it fits, so both
  // levels' records (32 B each) stay well inside the 126 MB L2 even for the
  // largest config-3 pockets.
  const double hs[kGridLevels] = {env_double("GD_VOXEL_H", 0.2), env_double("GD_VOXEL_H2", 0.75)};
  const double ms[kGridLevels] = {env_double("GD_VOXEL_MARGIN", 3.0),
                                  env_double("GD_VOXEL_MARGIN2", 32.0)};
  const long kMaxVoxels = static_cast<long>(env_double("GD_VOXEL_MAX", 1.5e6));
  for (int L = 0; L < kGridLevels; ++L) {
    double h = hs[L];
    const double margin = ms[L];
    VoxelGrid g{};
    for (;;) {
      int dims[3];
      long total = 1;
      for (int k = 0; k < 3; ++k) {
        dims[k] = static_cast<int>(std::floor((hi[k] - lo[k] + 2 * margin) / h)) + 1;
        total *= dims[k];
      }
      if (total <= kMaxVoxels) {
        g = VoxelGrid{lo[0] - margin, lo[1] - margin, lo[2] - margin, h, dims[0], dims[1], dims[2],
                      static_cast<int32_t>(env_double("GD_VOXEL_OVERFLOW", 1024))};
        break;
      }
      h *= 1.25;
    }
    const int nv = g.dim_x * g.dim_y * g.dim_z;
    DevBuf& counts = ctx->vox_counts;
    GD_CUDA(ctx, counts.ensure(sizeof(int32_t) * nv));
    int32_t* keep = nullptr;  // the count pass's first 8 candidates per voxel
    if (n_tiles > 0) {
      GD_CUDA(ctx, ctx->vox_keep.ensure(sizeof(int32_t) * 8 * static_cast<size_t>(nv)));
      keep = ctx->vox_keep.as<int32_t>();
    }
    GD_CUDA(ctx, static_cast<cudaError_t>(launch_voxel_count(slot->pts.as<double>(), n, g,
                                                             counts.as<int32_t>(),
                                                             ctx->tiles.as<float>(), n_tiles, keep,
                                                             ctx->stream)));
    // List offsets (exclusive scan of each voxel's 32-byte list units) and
    // the totals on the device; only the three totals come back.
    DevBuf& doff = ctx->vox_doff;
    GD_CUDA(ctx, doff.ensure(sizeof(int32_t) * nv));
    GD_CUDA(ctx, ctx->vox_scan.ensure(static_cast<size_t>(list_offsets_scratch_bytes(nv)) + 64));
    long long* dtot = reinterpret_cast<long long*>(static_cast<unsigned char*>(ctx->vox_scan.ptr) +
                                                   list_offsets_scratch_bytes(nv));
    GD_CUDA(ctx, static_cast<cudaError_t>(launch_list_offsets(counts.as<int32_t>(), nv, n,
                                                              compact ? static_cast<long long>(head.size() / 16) : n,
                                                              compact ? 1 : 0, doff.as<int32_t>(), ctx->vox_scan.ptr,
                                                              dtot, ctx->stream)));
    long long tot[3];
    GD_CUDA(ctx, cudaMemcpyAsync(tot, dtot, sizeof tot, cudaMemcpyDeviceToHost, ctx->stream));
    GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const int64_t listed = tot[0], total = tot[1];
    const int32_t mx = static_cast<int32_t>(tot[2]);
    if (listed > (1ll << 30)) return ctx->fail(GD_ERR_INVALID, "pocket: voxel index too large");
    const size_t rec_bytes = (compact ? 32 : sizeof(double) * kRecDoubles) * static_cast<size_t>(nv);
    GD_CUDA(ctx, slot->vox_off[L].ensure(rec_bytes));
    GD_CUDA(ctx, slot->vox_pts[L].ensure(sizeof(double) * 4 * std::max<int64_t>(listed, 1)));
    // List head: the whole pocket, the list of every overflow voxel.
    if (compact)
      GD_CUDA(ctx, cudaMemcpyAsync(slot->vox_pts[L].ptr, head.data(), sizeof(uint16_t) * head.size(),
                                   cudaMemcpyHostToDevice, ctx->stream));
    else
      GD_CUDA(ctx, cudaMemcpyAsync(slot->vox_pts[L].ptr, slot->pts.ptr, sizeof(double) * 4 * n,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
    GD_CUDA(ctx, static_cast<cudaError_t>(
                     launch_voxel_fill(slot->pts.as<double>(), n, g, doff.as<int32_t>(),
                                       slot->vox_off[L].as<double>(), slot->vox_pts[L].as<double>(),
                                       ctx->tiles.as<float>(), n_tiles, counts.as<int32_t>(),
                                       keep, compact ? ctx->vox_codes.as<uint16_t>() : nullptr,
                                       ctx->stream)));
    GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    slot->grid[L] = g;
    slot->stats[L] = gd_index_level{{g.dim_x, g.dim_y, g.dim_z}, g.h, total,
                                    static_cast<int64_t>(rec_bytes),
                                    static_cast<int64_t>(sizeof(double) * 4) * std::max<int64_t>(listed, 1)};
    slot->n_cand += total;
    slot->max_cand = std::max(slot->max_cand, mx);
    GridLevel& gl = v.lv[L];
    gl.rec = slot->vox_off[L].as<double>();
    gl.lst = slot->vox_pts[L].as<double>();
    gl.lo_x = g.lo_x;
    gl.lo_y = g.lo_y;
    gl.lo_z = g.lo_z;
    gl.inv_h = 1.0 / g.h;
    gl.dim_x = g.dim_x;
    gl.dim_y = g.dim_y;
    gl.dim_z = g.dim_z;
    gl.fdim_x = g.dim_x;
    gl.fdim_y = g.dim_y;
    gl.fdim_z = g.dim_z;
  }
  slot->P = n;
  activate(*slot);
  return GD_OK;
}

extern "C" int gd_pocket_index_format(const gd_ctx* ctx) {
  if (ctx == nullptr || ctx->P == 0) return GD_ERR_NO_POCKET;
  return ctx->view.compact ? 1 : 0;
}

extern "C" int gd_pocket_index_stats(const gd_ctx* ctx, gd_index_level out[2]) {
  if (ctx == nullptr || ctx->P == 0 || out == nullptr) return GD_ERR_NO_POCKET;
  for (const auto& sl : ctx->slots)
    if (sl->last_use == ctx->use_clock) {  // the active slot
      for (int L = 0; L < kGridLevels; ++L) out[L] = sl->stats[L];
      return GD_OK;
    }
  return GD_ERR_NO_POCKET;
}

extern "C" int gd_pocket_info(const gd_ctx* ctx, double centre[3], int32_t dims[3], double* voxel,
                              int64_t* n_candidates, int32_t* max_candidates) {
  if (ctx == nullptr || ctx->P == 0) return GD_ERR_NO_POCKET;
  if (centre)
    for (int k = 0; k < 3; ++k) centre[k] = ctx->centre[k];
  if (dims) {
    dims[0] = ctx->grid[0].dim_x;
    dims[1] = ctx->grid[0].dim_y;
    dims[2] = ctx->grid[0].dim_z;
  }
  if (voxel) *voxel = ctx->grid[0].h;
  if (n_candidates) *n_candidates = ctx->n_cand;
  if (max_candidates) *max_candidates = ctx->max_cand;
  return GD_OK;
}

// ---------------------------------------------------------------------------
// Batch staging.  The host copies each ligand range ("chunk") of raw atoms
// and bonds into a pinned arena and fills the per-ligand offsets (O(L));
// the chunk is copied to HBM and preprocessed there (prep.cu: validation,
// far masks, rotamers, fragments, CTA order), so chunk k+1 is packed on the
// host while chunk k is copied, preprocessed and docked on the GPU.
// ---------------------------------------------------------------------------
namespace {

enum Seg { kMeta, kXyz, kRad, kBonds, kRot, kBoff, kSegs };

struct Running {
  size_t fo = 0, wo = 0, mo = 0;  // frag, far-word, fmask-word cursors
};

// Atom counts the batch path docks (the rest is rejected up front): up to
// kNarrowAtoms on the warp-per-chain kernels with GPU preprocessing, up to
// kWideAtoms on the wide path.
bool size_ok(int n) { return n >= 2 && n <= kWideAtoms; }
bool is_wide(int n) { return n > kNarrowAtoms; }
static_assert(kNarrowAtoms == kMaxAtoms, "the GPU preprocessing's limit is the warp path's");

}  // namespace

// Validates the batch, sizes the pinned arena and the device buffers with
// upper bounds, and resets the host bookkeeping.
static int begin_batch(gd_ctx* ctx, const gd_ligand_batch* b, Running& run) {
  if (b == nullptr || b->n_ligands < 0 || (b->n_ligands > 0 &&
      (!b->atom_offsets || !b->xyz || !b->radii || !b->bond_offsets ||
       (b->bond_offsets[b->n_ligands] > 0 && (!b->bonds || !b->bond_rotatable)))))
    return ctx->fail(GD_ERR_INVALID, "gd_upload: invalid ligand batch");
  const int L = b->n_ligands;
  size_t far_ub = 0, fmask_ub = 0;
  int64_t wide_atoms = 0;
  ctx->wide_idx.clear();
  ctx->wide_pref.clear();
  for (int l = 0; l < L; ++l) {
    const int n = b->atom_offsets[l + 1] - b->atom_offsets[l];
    const int nb = b->bond_offsets[l + 1] - b->bond_offsets[l];
    if (n < 0 || nb < 0) return ctx->fail(GD_ERR_INVALID, "gd_upload: offsets not ascending");
    if (!size_ok(n)) continue;
    const size_t W = static_cast<size_t>((n + 63) / 64);
    far_ub += static_cast<size_t>(n) * W;
    fmask_ub += 2 * static_cast<size_t>(nb) * W;
    if (is_wide(n)) {
      ctx->wide_idx.push_back(l);
      ctx->wide_pref.push_back(wide_atoms);
      wide_atoms += n;
    }
  }
  ctx->wide_pref.push_back(wide_atoms);
  ctx->wide_prep.assign(ctx->wide_idx.size(), PreparedLigand{});
  if (!ctx->wide_idx.empty()) {
    GD_CUDA(ctx, ctx->wide_list_d.ensure(sizeof(int32_t) * ctx->wide_idx.size()));
    GD_CUDA(ctx, ctx->wide_off_d.ensure(sizeof(int64_t) * ctx->wide_pref.size()));
    GD_CUDA(ctx, cudaMemcpy(ctx->wide_list_d.ptr, ctx->wide_idx.data(),
                            sizeof(int32_t) * ctx->wide_idx.size(), cudaMemcpyHostToDevice));
    GD_CUDA(ctx, cudaMemcpy(ctx->wide_off_d.ptr, ctx->wide_pref.data(),
                            sizeof(int64_t) * ctx->wide_pref.size(), cudaMemcpyHostToDevice));
  }
  const int32_t A = L > 0 ? b->atom_offsets[L] : 0;
  const int64_t B = L > 0 ? b->bond_offsets[L] : 0;
  const size_t frag_ub = 2 * static_cast<size_t>(B);
  const size_t sizes[kSegs] = {sizeof(LigMeta) * std::max(L, 1), sizeof(double) * 3 * std::max(A, 1),
                               sizeof(double) * std::max(A, 1),
                               sizeof(int32_t) * 2 * std::max<size_t>(B, 1),
                               std::max<size_t>(B, 1), sizeof(int32_t) * (std::max(L, 1) + 1)};
  size_t arena = 0;
  for (size_t sz : sizes) arena += (sz + 255) & ~size_t(255);
  GD_CUDA(ctx, ctx->staging.ensure(arena));
  unsigned char* base = static_cast<unsigned char*>(ctx->staging.ptr);
  size_t o = 0;
  DevBuf* dev[kSegs] = {&ctx->meta, &ctx->xyz, &ctx->radii, &ctx->bonds, &ctx->rot, &ctx->boff};
  for (int i = 0; i < kSegs; ++i) {
    ctx->pin[i] = base + o;
    o += (sizes[i] + 255) & ~size_t(255);
    GD_CUDA(ctx, dev[i]->ensure(sizes[i]));
  }
  GD_CUDA(ctx, ctx->far.ensure(sizeof(uint64_t) * std::max<size_t>(far_ub, 1)));
  GD_CUDA(ctx, ctx->fmask.ensure(sizeof(uint64_t) * std::max<size_t>(fmask_ub, 1)));
  GD_CUDA(ctx, ctx->fax.ensure(sizeof(int32_t) * std::max<size_t>(frag_ub, 1)));
  GD_CUDA(ctx, ctx->fan.ensure(sizeof(int32_t) * std::max<size_t>(frag_ub, 1)));
  GD_CUDA(ctx, ctx->frel.ensure(sizeof(double) * std::max<size_t>(frag_ub, 1)));
  GD_CUDA(ctx, ctx->order.ensure(sizeof(int32_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_status.ensure(sizeof(int32_t) * std::max(L, 1)));
  ctx->frag_total = frag_ub;
  ctx->errors.assign(L, std::string());
  ctx->status_host.assign(L, 0);
  // An empty batch may pass null offset arrays (nothing is read from them).
  if (L > 0) ctx->atom_off.assign(b->atom_offsets, b->atom_offsets + L + 1);
  else ctx->atom_off.assign(1, 0);
  ctx->n_lig = L;
  ctx->total_atoms = A;
  ctx->max_n = 1;
  ctx->have_result = false;
  ctx->staged = false;
  ctx->timing = gd_timing{};
  run = Running{};
  return GD_OK;
}

// Host half of a chunk: offsets of ligands [c0, c1) into the descriptor
// arrays, and their raw atoms and bonds into the pinned arena (the bulk
// copy on the worker pool for large chunks).  Returns the chunk's largest
// atom count (of ligands the GPU preprocesses).
static void pack_range(gd_ctx* ctx, const gd_ligand_batch* b, int c0, int c1, Running& run,
                       int& chunk_max_n) {
  chunk_max_n = 1;
  if (c1 <= c0) return;
  auto* meta = reinterpret_cast<LigMeta*>(ctx->pin[kMeta]);
  for (int l = c0; l < c1; ++l) {
    LigMeta& m = meta[l];
    m.atom_off = b->atom_offsets[l];
    m.n = b->atom_offsets[l + 1] - b->atom_offsets[l];
    const int nb = b->bond_offsets[l + 1] - b->bond_offsets[l];
    m.words = (m.n + 63) / 64;
    m.nfrag = 0;
    m.frag_off = 2 * b->bond_offsets[l];
    m.far_off = static_cast<int32_t>(run.wo);
    m.fmask_off = static_cast<int32_t>(run.mo);
    m.status = size_ok(m.n) ? GD_LIG_OK : GD_LIG_INVALID;
    if (m.status != GD_LIG_OK) continue;
    run.wo += static_cast<size_t>(m.n) * m.words;
    run.mo += 2 * static_cast<size_t>(nb) * m.words;
    if (is_wide(m.n)) {
      // Wide ligand: the graph preprocessing on the host, now; its
      // descriptors follow the chunk's raw copy (h2d_prep_range).
      const size_t w = std::lower_bound(ctx->wide_idx.begin(), ctx->wide_idx.end(), l) - ctx->wide_idx.begin();
      PreparedLigand& q = ctx->wide_prep[w];
      q = prepare_ligand(std::to_string(l), m.n, b->xyz + 3 * static_cast<size_t>(m.atom_off),
                         b->radii + m.atom_off, nb, b->bonds + 2 * static_cast<size_t>(b->bond_offsets[l]),
                         b->bond_rotatable + b->bond_offsets[l], kWideAtoms);
      m.status = q.status;
      m.nfrag = q.status == GD_LIG_OK ? q.nfrag() : 0;
      continue;
    }
    chunk_max_n = std::max(chunk_max_n, m.n);
  }
  auto* bo = reinterpret_cast<int32_t*>(ctx->pin[kBoff]);
  for (int l = c0; l <= c1; ++l) bo[l] = b->bond_offsets[l];
  const size_t a0 = b->atom_offsets[c0], a1 = b->atom_offsets[c1];
  const size_t q0 = b->bond_offsets[c0], q1 = b->bond_offsets[c1];
  struct Part {
    unsigned char* dst;
    const unsigned char* src;
    size_t bytes;
  } parts[4] = {
      {ctx->pin[kXyz] + 24 * a0, reinterpret_cast<const unsigned char*>(b->xyz + 3 * a0), 24 * (a1 - a0)},
      {ctx->pin[kRad] + 8 * a0, reinterpret_cast<const unsigned char*>(b->radii + a0), 8 * (a1 - a0)},
      {ctx->pin[kBonds] + 8 * q0, reinterpret_cast<const unsigned char*>(b->bonds + 2 * q0), 8 * (q1 - q0)},
      {ctx->pin[kRot] + q0, b->bond_rotatable + q0, q1 - q0}};
  size_t total = 0;
  for (const Part& pt : parts) total += pt.bytes;
  constexpr size_t kBlock = 256 << 10;
  if (total < 4 * kBlock) {
    for (const Part& pt : parts)
      if (pt.bytes) std::memcpy(pt.dst, pt.src, pt.bytes);
  } else {
    if (!ctx->pool)
      ctx->pool = std::make_unique<WorkerPool>((ctx->pool_threads > 0 ? ctx->pool_threads : host_threads()) - 1);
    size_t starts[5] = {0};
    for (int k = 0; k < 4; ++k) starts[k + 1] = starts[k] + (parts[k].bytes + kBlock - 1) / kBlock;
    std::atomic<size_t> next{0};
    ctx->pool->run([&] {
      for (size_t bi; (bi = next.fetch_add(1)) < starts[4];) {
        int k = 0;
        while (starts[k + 1] <= bi) ++k;
        const size_t off = (bi - starts[k]) * kBlock;
        std::memcpy(parts[k].dst + off, parts[k].src + off, std::min(kBlock, parts[k].bytes - off));
      }
    });
  }
  ctx->max_n = std::max(ctx->max_n, chunk_max_n);
}

// Copy half of a chunk (pinned -> HBM) and its GPU preprocessing, on stream s.
static int h2d_prep_range(gd_ctx* ctx, const gd_ligand_batch* b, int c0, int c1, int max_n,
                          cudaStream_t s) {
  if (c1 <= c0) return GD_OK;
  auto cp = [&](DevBuf& d, int seg, size_t off, size_t bytes) -> int {
    if (bytes == 0) return GD_OK;
    ctx->timing.h2d_bytes += static_cast<int64_t>(bytes);
    return ctx->cuda(cudaMemcpyAsync(static_cast<unsigned char*>(d.ptr) + off, ctx->pin[seg] + off,
                                     bytes, cudaMemcpyHostToDevice, s), "h2d");
  };
  const size_t a0 = ctx->atom_off[c0], a1 = ctx->atom_off[c1];
  const size_t q0 = b->bond_offsets[c0], q1 = b->bond_offsets[c1];
  int rc = GD_OK;
  if ((rc = cp(ctx->meta, kMeta, sizeof(LigMeta) * c0, sizeof(LigMeta) * (c1 - c0)))) return rc;
  if ((rc = cp(ctx->xyz, kXyz, 24 * a0, 24 * (a1 - a0)))) return rc;
  if ((rc = cp(ctx->radii, kRad, 8 * a0, 8 * (a1 - a0)))) return rc;
  if ((rc = cp(ctx->bonds, kBonds, 8 * q0, 8 * (q1 - q0)))) return rc;
  if ((rc = cp(ctx->rot, kRot, q0, q1 - q0))) return rc;
  if ((rc = cp(ctx->boff, kBoff, 4 * static_cast<size_t>(c0), 4 * static_cast<size_t>(c1 - c0 + 1)))) return rc;
  PrepParams q{};
  q.l0 = c0;
  q.l1 = c1;
  q.max_n = max_n;
  q.meta = ctx->meta.as<LigMeta>();
  q.boff = ctx->boff.as<int32_t>();
  q.bonds = ctx->bonds.as<int32_t>();
  q.rot = ctx->rot.as<uint8_t>();
  q.xyz = ctx->xyz.as<double>();
  q.radii = ctx->radii.as<double>();
  q.far = ctx->far.as<uint64_t>();
  q.fmask = ctx->fmask.as<uint64_t>();
  q.fax = ctx->fax.as<int32_t>();
  q.fan = ctx->fan.as<int32_t>();
  q.frel = ctx->frel.as<double>();
  q.status = ctx->o_status.as<int32_t>();
  q.order = ctx->order.as<int32_t>();
  GD_CUDA(ctx, static_cast<cudaError_t>(launch_prep(q, s)));
  ctx->timing.launches += 2;
  // Wide ligands of the chunk: their host-made descriptors (prep_kernel
  // leaves them alone).
  const auto* meta = reinterpret_cast<const LigMeta*>(ctx->pin[kMeta]);
  for (size_t w = std::lower_bound(ctx->wide_idx.begin(), ctx->wide_idx.end(), c0) - ctx->wide_idx.begin();
       w < ctx->wide_idx.size() && ctx->wide_idx[w] < c1; ++w) {
    const PreparedLigand& g = ctx->wide_prep[w];
    const LigMeta& m = meta[ctx->wide_idx[w]];
    if (g.status != GD_LIG_OK) continue;
    auto up = [&](DevBuf& d, size_t elem, size_t off, const void* src, size_t cnt) -> int {
      if (cnt == 0) return GD_OK;
      ctx->timing.h2d_bytes += static_cast<int64_t>(elem * cnt);
      return ctx->cuda(cudaMemcpyAsync(static_cast<unsigned char*>(d.ptr) + elem * off, src, elem * cnt,
                                       cudaMemcpyHostToDevice, s), "h2d wide");
    };
    const size_t nf = static_cast<size_t>(g.nfrag());
    if ((rc = up(ctx->far, 8, m.far_off, g.far_mask.data(), g.far_mask.size()))) return rc;
    if ((rc = up(ctx->fmask, 8, m.fmask_off, g.frag_mask.data(), g.frag_mask.size()))) return rc;
    if ((rc = up(ctx->fax, 4, m.frag_off, g.frag_axis.data(), nf))) return rc;
    if ((rc = up(ctx->fan, 4, m.frag_off, g.frag_anchor.data(), nf))) return rc;
    if ((rc = up(ctx->frel, 8, m.frag_off, g.frag_rel.data(), nf))) return rc;
  }
  return GD_OK;
}

// Host bookkeeping once a batch's statuses are known: the per-ligand
// status mirror, and the reference's message for every rejected ligand
// (re-derived on the host, prep.cpp; the batch is still the caller's).
static void note_status(gd_ctx* ctx, const gd_ligand_batch* b, const int32_t* status) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int l = 0; l < ctx->n_lig; ++l) {
    ctx->status_host[l] = status[l];
    if (status[l] != GD_LIG_INVALID) continue;
    const int a0 = b->atom_offsets[l], b0 = b->bond_offsets[l];
    const PreparedLigand p = prepare_ligand(std::to_string(l), b->atom_offsets[l + 1] - a0, b->xyz + 3 * a0,
                                            b->radii + a0, b->bond_offsets[l + 1] - b0, b->bonds + 2 * b0,
                                            b->bond_rotatable + b0, kWideAtoms);
    ctx->errors[l] = p.error.empty() ? "ligand '" + std::to_string(l) + "': invalid" : p.error;
  }
  ctx->timing.host_prep_ms =
      std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" int gd_upload(gd_ctx* ctx, const gd_ligand_batch* b) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  Running run;
  int rc = begin_batch(ctx, b, run);
  if (rc != GD_OK) return rc;
  const auto t0 = std::chrono::steady_clock::now();
  int mx = 1;
  pack_range(ctx, b, 0, ctx->n_lig, run, mx);
  ctx->timing.host_pack_ms =
      std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  cudaEventRecord(ctx->ev[0], ctx->stream);
  rc = h2d_prep_range(ctx, b, 0, ctx->n_lig, mx, ctx->stream);
  if (rc != GD_OK) return rc;
  cudaEventRecord(ctx->ev[1], ctx->stream);
  // The statuses (and rejected ligands' messages) while the batch is at hand.
  std::vector<int32_t> st(std::max(ctx->n_lig, 1));
  if (ctx->n_lig > 0)
    GD_CUDA(ctx, cudaMemcpyAsync(st.data(), ctx->o_status.ptr, sizeof(int32_t) * ctx->n_lig,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cudaEventElapsedTime(&ctx->timing.upload_ms, ctx->ev[0], ctx->ev[1]);
  note_status(ctx, b, st.data());
  ctx->staged = true;
  return GD_OK;
}

// ---------------------------------------------------------------------------
// The hot path.
// ---------------------------------------------------------------------------
static int ensure_orientations(gd_ctx* ctx, int step) {
  if (ctx->orient_step == step) return GD_OK;
  std::vector<int32_t> idx;
  std::vector<double> R;
  rigid_orientations(step, idx, R);
  GD_CUDA(ctx, ctx->orient_idx.ensure(sizeof(int32_t) * idx.size()));
  GD_CUDA(ctx, ctx->orient_R.ensure(sizeof(double) * R.size()));
  GD_CUDA(ctx, cudaMemcpy(ctx->orient_idx.ptr, idx.data(), sizeof(int32_t) * idx.size(),
                          cudaMemcpyHostToDevice));
  GD_CUDA(ctx, cudaMemcpy(ctx->orient_R.ptr, R.data(), sizeof(double) * R.size(),
                          cudaMemcpyHostToDevice));
  ctx->orient_step = step;
  ctx->n_orient = static_cast<int32_t>(idx.size());
  ctx->orient_idx_host = idx;
  return GD_OK;
}

// Validates knobs, allocates every output buffer for the whole batch (before
// any asynchronous work: a reallocation would free memory in flight) and
// returns the launch parameters common to all chunks.
static int prepare_dock(gd_ctx* ctx, const gd_knobs* k, bool keep_pose, bool keep_top, DockParams& p) {
  char msg[128];
  if (gd_validate_knobs(k, msg, sizeof msg) != GD_OK) return ctx->fail(GD_ERR_INVALID, msg);
  if (ctx->P == 0) return ctx->fail(GD_ERR_NO_POCKET, "gd_dock: no pocket staged (gd_set_pocket)");
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  const bool rigid = k->rigid_step > 0;
  if (rigid) {
    const int rc = ensure_orientations(ctx, k->rigid_step);
    if (rc != GD_OK) return rc;
  }
  const int L = ctx->n_lig;
  const int K = rigid ? k->top_k : 1;
  const size_t slots = static_cast<size_t>(std::max(L, 1)) * K;
  GD_CUDA(ctx, ctx->seed_slot.ensure(sizeof(int32_t) * slots));
  GD_CUDA(ctx, ctx->seed_score.ensure(sizeof(double) * slots));
  GD_CUDA(ctx, ctx->k_eff.ensure(sizeof(int32_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_orient.ensure(sizeof(int32_t) * slots));
  GD_CUDA(ctx, ctx->o_rank.ensure(sizeof(int32_t) * slots));
  GD_CUDA(ctx, ctx->o_rigid.ensure(sizeof(double) * slots));
  GD_CUDA(ctx, ctx->o_final.ensure(sizeof(double) * slots));
  GD_CUDA(ctx, ctx->o_evals.ensure(sizeof(int64_t) * slots));
  GD_CUDA(ctx, ctx->o_checks.ensure(sizeof(int64_t) * slots));
  GD_CUDA(ctx, ctx->st_final.ensure(sizeof(double) * slots));
  GD_CUDA(ctx, ctx->st_evals.ensure(sizeof(int64_t) * slots));
  GD_CUDA(ctx, ctx->st_checks.ensure(sizeof(int64_t) * slots));
  GD_CUDA(ctx, ctx->o_scored.ensure(sizeof(int64_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_status.ensure(sizeof(int32_t) * std::max(L, 1)));
  if (keep_pose || keep_top) {
    const size_t pose_bytes = sizeof(double) * 3 * static_cast<size_t>(std::max(ctx->total_atoms, 1)) * K;
    if (keep_pose) GD_CUDA(ctx, ctx->o_pose.ensure(pose_bytes));
    GD_CUDA(ctx, ctx->stage_pose.ensure(pose_bytes));
  }
  if (keep_top) {
    GD_CUDA(ctx, ctx->o_top.ensure(sizeof(double) * 3 * static_cast<size_t>(std::max(ctx->total_atoms, 1))));
    GD_CUDA(ctx, ctx->top_best.ensure(sizeof(unsigned long long) * std::max(L, 1)));
  }
  if (!ctx->wide_idx.empty())
    GD_CUDA(ctx, ctx->wide_scratch.ensure(sizeof(double) * 8 * static_cast<size_t>(K) *
                                          static_cast<size_t>(ctx->wide_pref.back())));
  p = DockParams{};
  p.wide_scratch = ctx->wide_scratch.as<double>();
  p.order = ctx->order.as<int32_t>();
  p.meta = ctx->meta.as<LigMeta>();
  p.xyz = ctx->xyz.as<double>();
  p.radii = ctx->radii.as<double>();
  p.far_mask = ctx->far.as<uint64_t>();
  p.frag_mask = ctx->fmask.as<uint64_t>();
  p.frag_axis = ctx->fax.as<int32_t>();
  p.frag_anchor = ctx->fan.as<int32_t>();
  p.frag_rel = ctx->frel.as<double>();
  p.pocket = ctx->view;
  p.pocket.use_index = (k->flags & GD_FLAG_BRUTE_FORCE) ? 0 : ctx->view.use_index;
  p.cx = ctx->centre[0];
  p.cy = ctx->centre[1];
  p.cz = ctx->centre[2];
  p.n_orient = rigid ? ctx->n_orient : 0;
  p.orient_idx = ctx->orient_idx.as<int32_t>();
  p.orient_R = ctx->orient_R.as<double>();
  p.cos_deg = ctx->cos_t.as<double>();
  p.sin_deg = ctx->sin_t.as<double>();
  p.hp = k->high_precision_step;
  p.lp = k->low_precision_step;
  p.reps = k->repetitions;
  p.refine = k->enable_refinement ? 1 : 0;
  p.tile = gd_optimal_tile_size(k->high_precision_step);
  p.threshold = k->threshold;
  p.top_k = K;
  p.rigid = rigid ? 1 : 0;
  p.k_slots = rigid ? std::min(K, ctx->n_orient) : 1;
  p.st_final = ctx->st_final.as<double>();
  p.st_evals = ctx->st_evals.as<int64_t>();
  p.st_checks = ctx->st_checks.as<int64_t>();
  p.seed_slot = ctx->seed_slot.as<int32_t>();
  p.seed_score = ctx->seed_score.as<double>();
  p.k_eff = ctx->k_eff.as<int32_t>();
  p.out_orient = ctx->o_orient.as<int32_t>();
  p.out_rank = ctx->o_rank.as<int32_t>();
  p.out_rigid = ctx->o_rigid.as<double>();
  p.out_final = ctx->o_final.as<double>();
  p.out_evals = ctx->o_evals.as<int64_t>();
  p.out_checks = ctx->o_checks.as<int64_t>();
  p.out_pose = keep_pose ? ctx->o_pose.as<double>() : nullptr;
  p.stage_pose = (keep_pose || keep_top) ? ctx->stage_pose.as<double>() : nullptr;
  p.out_top = keep_top ? ctx->o_top.as<double>() : nullptr;
  // Top-1 only: chains stage their pose only while improving their ligand's best.
  p.top_best = (keep_top && !keep_pose) ? ctx->top_best.as<unsigned long long>() : nullptr;
  p.poses_scored = ctx->o_scored.as<int64_t>();
  p.status = ctx->o_status.as<int32_t>();
  p.counters = nullptr;
  if (k->flags & GD_FLAG_COUNT_WORK) {
    GD_CUDA(ctx, ctx->counters.ensure(sizeof(unsigned long long) * kCounterSlots));
    GD_CUDA(ctx, cudaMemsetAsync(ctx->counters.ptr, 0, sizeof(unsigned long long) * kCounterSlots,
                                 ctx->stream));
    p.counters = ctx->counters.as<unsigned long long>();
  }
  ctx->counted = p.counters != nullptr;
  ctx->last_topk = K;
  ctx->last_rigid = rigid;
  ctx->last_pose = keep_pose;
  ctx->last_top = keep_top;
  return GD_OK;
}

// The three hot-path launches over CTA-order positions [c0, c1).
static int launch_range(gd_ctx* ctx, DockParams p, int c0, int c1, int max_n, cudaStream_t s,
                        cudaEvent_t e_mid) {
  p.n_lig = c1 - c0;
  p.order = ctx->order.as<int32_t>() + c0;
  p.max_n = max_n;
  p.max_pairs = std::max(1, max_n * max_n / 4);
  if (p.n_lig == 0) return GD_OK;
  if (p.top_best != nullptr)
    GD_CUDA(ctx, cudaMemsetAsync(p.top_best + c0, 0, sizeof(unsigned long long) * (c1 - c0), s));
  // Wide ligands among ligands [c0, c1) (chunks are ligand ranges; `order`
  // permutes within them): their own rigid launch (shared memory sized by
  // their atoms) and the wide search kernel; the regular launches skip them.
  const size_t w0 = std::lower_bound(ctx->wide_idx.begin(), ctx->wide_idx.end(), c0) - ctx->wide_idx.begin();
  const size_t w1 = std::lower_bound(ctx->wide_idx.begin(), ctx->wide_idx.end(), c1) - ctx->wide_idx.begin();
  DockParams pw = p;
  pw.n_wide = static_cast<int32_t>(w1 - w0);
  pw.wide_list = ctx->wide_list_d.as<int32_t>() + w0;
  pw.wide_off = ctx->wide_off_d.as<int64_t>() + w0;
  if (p.rigid) {
    GD_CUDA(ctx, static_cast<cudaError_t>(p.pocket.compact ? launch_rigid_topk_cp(p, s)
                                                           : launch_rigid_topk(p, s)));
    ctx->timing.launches += 1;
    if (pw.n_wide > 0) {
      DockParams pr = pw;
      pr.order = pw.wide_list;
      pr.n_lig = pw.n_wide;
      pr.wide_pass = 1;
      pr.max_n = 1;
      for (size_t w = w0; w < w1; ++w)
        pr.max_n = std::max(pr.max_n, static_cast<int32_t>(ctx->wide_pref[w + 1] - ctx->wide_pref[w]));
      GD_CUDA(ctx, static_cast<cudaError_t>(p.pocket.compact ? launch_rigid_topk_cp(pr, s)
                                                             : launch_rigid_topk(pr, s)));
      ctx->timing.launches += 1;
    }
  }
  if (e_mid) cudaEventRecord(e_mid, s);
  GD_CUDA(ctx, static_cast<cudaError_t>(p.pocket.compact ? launch_flex_cp(p, s) : launch_flex(p, s)));
  if (pw.n_wide > 0) {
    GD_CUDA(ctx, static_cast<cudaError_t>(p.pocket.compact ? launch_flex_wide_cp(pw, s)
                                                           : launch_flex_wide(pw, s)));
    ctx->timing.launches += 1;
  }
  GD_CUDA(ctx, static_cast<cudaError_t>(launch_finalize(p, s)));
  ctx->timing.launches += 2;
  return GD_OK;
}

extern "C" int gd_dock_resident(gd_ctx* ctx, const gd_knobs* knobs) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  if (knobs == nullptr) return ctx->fail(GD_ERR_INVALID, "knob config: null");
  DockParams p;
  int rc = prepare_dock(ctx, knobs, (knobs->flags & GD_FLAG_KEEP_POSES) != 0,
                        (knobs->flags & GD_FLAG_TOP_POSE) != 0, p);
  if (rc != GD_OK) return rc;
  ctx->timing.launches = 0;
  cudaEventRecord(ctx->ev[2], ctx->stream);
  rc = launch_range(ctx, p, 0, ctx->n_lig, ctx->max_n, ctx->stream, ctx->ev[3]);
  if (rc != GD_OK) return rc;
  cudaEventRecord(ctx->ev[4], ctx->stream);
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->have_result = true;
  cudaEventElapsedTime(&ctx->timing.rigid_ms, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&ctx->timing.flex_ms, ctx->ev[3], ctx->ev[4]);
  ctx->timing.total_ms = ctx->timing.rigid_ms + ctx->timing.flex_ms;
  return GD_OK;
}

// Result copy of ligands [l0, l1) from HBM into the destination arrays
// (user or pinned), asynchronously on stream s.
static int d2h_range(gd_ctx* ctx, const gd_result* r, int l0, int l1, cudaStream_t s) {
  const int K = ctx->last_topk;
  const size_t s0 = static_cast<size_t>(l0) * K, ns = static_cast<size_t>(l1 - l0) * K;
  auto cp = [&](void* dst, const DevBuf& src, size_t elem, size_t off, size_t cnt) -> int {
    if (dst == nullptr || cnt == 0) return GD_OK;
    ctx->timing.d2h_bytes += static_cast<int64_t>(elem * cnt);
    return ctx->cuda(cudaMemcpyAsync(static_cast<unsigned char*>(dst) + elem * off,
                                     static_cast<const unsigned char*>(src.ptr) + elem * off,
                                     elem * cnt, cudaMemcpyDeviceToHost, s), "d2h");
  };
  int rc = GD_OK;
  if ((rc = cp(r->orientation, ctx->o_orient, 4, s0, ns))) return rc;
  if ((rc = cp(r->seed_rank, ctx->o_rank, 4, s0, ns))) return rc;
  if ((rc = cp(r->rigid_score, ctx->o_rigid, 8, s0, ns))) return rc;
  if ((rc = cp(r->final_score, ctx->o_final, 8, s0, ns))) return rc;
  if ((rc = cp(r->evaluations, ctx->o_evals, 8, s0, ns))) return rc;
  if ((rc = cp(r->feasibility_checks, ctx->o_checks, 8, s0, ns))) return rc;
  if ((rc = cp(r->k_eff, ctx->k_eff, 4, l0, l1 - l0))) return rc;
  if ((rc = cp(r->poses_scored, ctx->o_scored, 8, l0, l1 - l0))) return rc;
  if ((rc = cp(r->status, ctx->o_status, 4, l0, l1 - l0))) return rc;
  if (r->final_pose != nullptr) {
    const size_t a0 = ctx->atom_off[l0], a1 = ctx->atom_off[l1];
    if ((rc = cp(r->final_pose, ctx->o_pose, 24, K * a0, K * (a1 - a0)))) return rc;
  }
  if (r->top_pose != nullptr) {
    const size_t a0 = ctx->atom_off[l0], a1 = ctx->atom_off[l1];
    if ((rc = cp(r->top_pose, ctx->o_top, 24, a0, a1 - a0))) return rc;
  }
  return GD_OK;
}

// Empty slots (ligands that failed, or slots past k_eff) read as
// orientation -2 and zeros; needs k_eff and status already on the host.
static void fill_empty(gd_ctx* ctx, gd_result* r, const int32_t* keff, const int32_t* stat,
                       int l0 = 0, int l1 = -1) {
  const int K = ctx->last_topk;
  if (l1 < 0) l1 = ctx->n_lig;
  for (int l = l0; l < l1; ++l) {
    const int kk = stat[l] != 0 ? 0 : (ctx->last_rigid ? keff[l] : 1);
    if (r->k_eff) r->k_eff[l] = kk;
    if (stat[l] != 0 && r->poses_scored) r->poses_scored[l] = 0;
    const int n = ctx->atom_off[l + 1] - ctx->atom_off[l];
    for (int e = kk; e < K; ++e) {
      const size_t d = static_cast<size_t>(l) * K + e;
      if (r->orientation) r->orientation[d] = -2;
      if (r->seed_rank) r->seed_rank[d] = 0;
      if (r->rigid_score) r->rigid_score[d] = 0.0;
      if (r->final_score) r->final_score[d] = 0.0;
      if (r->evaluations) r->evaluations[d] = 0;
      if (r->feasibility_checks) r->feasibility_checks[d] = 0;
      if (r->final_pose)
        std::memset(r->final_pose + 3 * (static_cast<size_t>(K) * ctx->atom_off[l] + size_t(e) * n), 0,
                    sizeof(double) * 3 * n);
    }
  }
}

static int download(gd_ctx* ctx, gd_result* r) {
  if (!ctx->have_result) return ctx->fail(GD_ERR_INVALID, "gd_download: nothing docked yet");
  if (r->final_pose != nullptr && !ctx->last_pose)
    return ctx->fail(GD_ERR_INVALID, "gd_download: poses were not kept");
  if (r->top_pose != nullptr && !ctx->last_top)
    return ctx->fail(GD_ERR_INVALID, "gd_download: top poses were not kept (GD_FLAG_TOP_POSE)");
  const int L = ctx->n_lig;
  ctx->timing.d2h_bytes = 0;
  int rc = d2h_range(ctx, r, 0, L, ctx->stream);
  if (rc != GD_OK) return rc;
  std::vector<int32_t> keff(std::max(L, 1)), stat(std::max(L, 1));
  GD_CUDA(ctx, cudaMemcpyAsync(keff.data(), ctx->k_eff.ptr, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, ctx->stream));
  GD_CUDA(ctx, cudaMemcpyAsync(stat.data(), ctx->o_status.ptr, sizeof(int32_t) * L, cudaMemcpyDeviceToHost, ctx->stream));
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  fill_empty(ctx, r, keff.data(), stat.data());
  return GD_OK;
}

extern "C" int gd_download(gd_ctx* ctx, gd_result* r) {
  if (ctx == nullptr || r == nullptr) return GD_ERR_INVALID;
  return download(ctx, r);
}

// Host buffers in, host buffers out, pipelined: the batch is split into
// chunks; while the GPU copies and docks chunk k (alternating two streams so
// one chunk's kernel tail overlaps the next chunk's start), the host threads
// preprocess chunk k+1.  Results land in a pinned arena and are copied into
// the caller's arrays at the end.
extern "C" int gd_dock_batch(gd_ctx* ctx, const gd_ligand_batch* batch, const gd_knobs* knobs,
                             gd_result* result) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  if (result == nullptr) return ctx->fail(GD_ERR_INVALID, "gd_dock_batch: null result");
  if (knobs == nullptr) return ctx->fail(GD_ERR_INVALID, "knob config: null");
  char msg[128];
  if (gd_validate_knobs(knobs, msg, sizeof msg) != GD_OK) return ctx->fail(GD_ERR_INVALID, msg);
  const auto t_start = std::chrono::steady_clock::now();
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  Running run;
  int rc = begin_batch(ctx, batch, run);
  if (rc != GD_OK) return rc;
  const bool keep_pose = result->final_pose != nullptr;
  const bool keep_top = result->top_pose != nullptr;
  DockParams p;
  rc = prepare_dock(ctx, knobs, keep_pose, keep_top, p);
  if (rc != GD_OK) return rc;
  const int L = ctx->n_lig, K = ctx->last_topk;
  static const int kStreams = std::max(1, static_cast<int>(env_double("GD_E2E_STREAMS", 6)));
  while (static_cast<int>(ctx->aux_streams.size()) < kStreams - 1) {
    cudaStream_t st;
    GD_CUDA(ctx, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    ctx->aux_streams.push_back(st);
  }
  // Pinned result arena: the async D2H targets.
  const size_t slots = static_cast<size_t>(std::max(L, 1)) * K;
  const size_t pose_elems = keep_pose ? 3 * static_cast<size_t>(std::max(ctx->total_atoms, 1)) * K : 0;
  const size_t top_elems = keep_top ? 3 * static_cast<size_t>(std::max(ctx->total_atoms, 1)) : 0;
  const size_t rbytes = slots * (4 + 4 + 8 + 8 + 8 + 8) + static_cast<size_t>(std::max(L, 1)) * (4 + 8 + 4) +
                        8 * (pose_elems + top_elems) + 1024;
  GD_CUDA(ctx, ctx->res_staging.ensure(rbytes));
  unsigned char* rb = static_cast<unsigned char*>(ctx->res_staging.ptr);
  size_t ro = 0;
  auto take = [&](size_t bytes) {
    void* q = rb + ro;
    ro += (bytes + 15) & ~size_t(15);
    return q;
  };
  gd_result pr{};
  pr.orientation = result->orientation ? static_cast<int32_t*>(take(4 * slots)) : nullptr;
  pr.seed_rank = result->seed_rank ? static_cast<int32_t*>(take(4 * slots)) : nullptr;
  pr.rigid_score = result->rigid_score ? static_cast<double*>(take(8 * slots)) : nullptr;
  pr.final_score = result->final_score ? static_cast<double*>(take(8 * slots)) : nullptr;
  pr.evaluations = result->evaluations ? static_cast<int64_t*>(take(8 * slots)) : nullptr;
  pr.feasibility_checks = result->feasibility_checks ? static_cast<int64_t*>(take(8 * slots)) : nullptr;
  pr.k_eff = static_cast<int32_t*>(take(4 * std::max(L, 1)));
  pr.poses_scored = result->poses_scored ? static_cast<int64_t*>(take(8 * std::max(L, 1))) : nullptr;
  pr.status = static_cast<int32_t*>(take(4 * std::max(L, 1)));
  pr.final_pose = keep_pose ? static_cast<double*>(take(8 * pose_elems)) : nullptr;
  pr.top_pose = keep_top ? static_cast<double*>(take(8 * top_elems)) : nullptr;

  // Chunk plan: a small head chunk (the only host packing nothing
  // overlaps), then chunks growing geometrically by 1.3x, spread over six
  // streams so each chunk's kernels start while earlier chunks' tails and
  // copies drain.  Re-tuned once preprocessing moved to the GPU (r3b,
  // tools/e2e_ab.py, c1 with top-1 poses: 2 streams / 1.6x 17.1-17.3 ms,
  // 3 streams 16.3-16.4, 4 streams 16.2-16.3, 6 streams / 1.3x 16.15-16.18;
  // mirrored "tapered" plans 16.5-17.7).  GD_E2E_GROWTH<=1 selects the equal
  // split into GD_E2E_CHUNKS parts.
  std::vector<int> bounds{0};
  static const int kHead = static_cast<int>(env_double("GD_E2E_HEAD", 256));
  static const int kParts = static_cast<int>(env_double("GD_E2E_CHUNKS", 15));
  static const double kGrowth = env_double("GD_E2E_GROWTH", 1.3);
  if (L > 2048 && kGrowth > 1.0) {
    bounds.push_back(kHead);
    double sz = kHead;
    while (bounds.back() < L) {
      sz *= kGrowth;
      const int nxt = static_cast<int>(std::min<double>(L, bounds.back() + sz));
      bounds.push_back(L - nxt < sz / 2 ? L : nxt);
    }
  } else if (L > 2048) {
    const int head = kHead, rest = L - head, parts = std::min(kParts, std::max(1, rest / 512));
    bounds.push_back(head);
    for (int c = 1; c <= parts; ++c)
      bounds.push_back(head + static_cast<int>(static_cast<long long>(rest) * c / parts));
  } else {
    bounds.push_back(L);
  }
  const int chunks = static_cast<int>(bounds.size()) - 1;
  while (static_cast<int>(ctx->chunk_ev.size()) < chunks) {
    cudaEvent_t e;
    GD_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->chunk_ev.push_back(e);
  }
  float prep_ms = 0.0f;
  ctx->timing.launches = 0;
  // Diagnostic timeline (GD_E2E_TRACE=1): per chunk, host prep interval and
  // GPU start/end relative to the call, printed to stderr at the end.
  static const bool kTrace = env_double("GD_E2E_TRACE", 0) != 0;
  std::vector<cudaEvent_t> tev;
  std::vector<double> tprep;
  cudaEvent_t tev0 = nullptr;
  if (kTrace) {
    tev.resize(2 * chunks);
    for (auto& e : tev) GD_CUDA(ctx, cudaEventCreate(&e));
    GD_CUDA(ctx, cudaEventCreate(&tev0));
    GD_CUDA(ctx, cudaEventRecord(tev0, ctx->stream));
  }
  for (int c = 0; c < chunks; ++c) {
    const int c0 = bounds[c], c1 = bounds[c + 1];
    cudaStream_t s = (c % kStreams) ? ctx->aux_streams[c % kStreams - 1] : ctx->stream;
    const auto t0 = std::chrono::steady_clock::now();
    int mx = 1;
    pack_range(ctx, batch, c0, c1, run, mx);
    const auto t1 = std::chrono::steady_clock::now();
    prep_ms += std::chrono::duration<float, std::milli>(t1 - t0).count();
    if (kTrace) {
      tprep.push_back(std::chrono::duration<double, std::milli>(t0 - t_start).count());
      tprep.push_back(std::chrono::duration<double, std::milli>(t1 - t_start).count());
      GD_CUDA(ctx, cudaEventRecord(tev[2 * c], s));
    }
    if ((rc = h2d_prep_range(ctx, batch, c0, c1, mx, s)) != GD_OK) return rc;
    if ((rc = launch_range(ctx, p, c0, c1, mx, s, nullptr)) != GD_OK) return rc;
    if ((rc = d2h_range(ctx, &pr, c0, c1, s)) != GD_OK) return rc;
    if (kTrace) GD_CUDA(ctx, cudaEventRecord(tev[2 * c + 1], s));
    GD_CUDA(ctx, cudaEventRecord(ctx->chunk_ev[c], s));
  }
  // Results chunk by chunk, in order: pinned arena -> caller arrays while the
  // later chunks are still on the GPU.
  float post_ms = 0.0f;
  for (int c = 0; c < chunks; ++c) {
    GD_CUDA(ctx, cudaEventSynchronize(ctx->chunk_ev[c]));
    const auto t_post = std::chrono::steady_clock::now();
    const int l0 = bounds[c], l1 = bounds[c + 1];
    const size_t s0 = static_cast<size_t>(l0) * K, sn = static_cast<size_t>(l1 - l0) * K;
    struct Seg {
      unsigned char* dst;
      const unsigned char* src;
      size_t bytes;
    };
    Seg segs[10];
    int nseg = 0;
    size_t total = 0;
    auto copy = [&](void* dst, const void* src, size_t elem, size_t off, size_t cnt) {
      if (dst && src && cnt) {
        segs[nseg++] = Seg{static_cast<unsigned char*>(dst) + elem * off,
                           static_cast<const unsigned char*>(src) + elem * off, elem * cnt};
        total += elem * cnt;
      }
    };
    copy(result->orientation, pr.orientation, 4, s0, sn);
    copy(result->seed_rank, pr.seed_rank, 4, s0, sn);
    copy(result->rigid_score, pr.rigid_score, 8, s0, sn);
    copy(result->final_score, pr.final_score, 8, s0, sn);
    copy(result->evaluations, pr.evaluations, 8, s0, sn);
    copy(result->feasibility_checks, pr.feasibility_checks, 8, s0, sn);
    copy(result->poses_scored, pr.poses_scored, 8, l0, l1 - l0);
    copy(result->status, pr.status, 4, l0, l1 - l0);
    if (keep_pose) {
      const size_t p0 = 3 * static_cast<size_t>(K) * ctx->atom_off[l0];
      const size_t p1 = 3 * static_cast<size_t>(K) * ctx->atom_off[l1];
      copy(result->final_pose, pr.final_pose, 8, p0, p1 - p0);
    }
    if (keep_top) {
      const size_t p0 = 3 * static_cast<size_t>(ctx->atom_off[l0]), p1 = 3 * static_cast<size_t>(ctx->atom_off[l1]);
      copy(result->top_pose, pr.top_pose, 8, p0, p1 - p0);
    }
    // Pinned arena -> caller arrays: large chunks in 64 KiB blocks over the
    // worker pool (the last chunk's copy is on the critical path).
    constexpr size_t kBlock = 64 << 10;
    if (total >= 4 * kBlock && ctx->pool) {
      size_t starts[11];
      starts[0] = 0;
      for (int k = 0; k < nseg; ++k) starts[k + 1] = starts[k] + (segs[k].bytes + kBlock - 1) / kBlock;
      std::atomic<size_t> next{0};
      const size_t blocks = starts[nseg];
      ctx->pool->run([&] {
        for (size_t bi; (bi = next.fetch_add(1)) < blocks;) {
          int k = 0;
          while (starts[k + 1] <= bi) ++k;
          const size_t off = (bi - starts[k]) * kBlock;
          std::memcpy(segs[k].dst + off, segs[k].src + off, std::min(kBlock, segs[k].bytes - off));
        }
      });
    } else {
      for (int k = 0; k < nseg; ++k) std::memcpy(segs[k].dst, segs[k].src, segs[k].bytes);
    }
    fill_empty(ctx, result, pr.k_eff, pr.status, l0, l1);
    post_ms += std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_post).count();
  }
  if (L == 0) fill_empty(ctx, result, pr.k_eff, pr.status);
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (cudaStream_t st : ctx->aux_streams) GD_CUDA(ctx, cudaStreamSynchronize(st));
  note_status(ctx, batch, pr.status);
  ctx->have_result = true;
  ctx->staged = true;
  const auto t_end = std::chrono::steady_clock::now();
  if (kTrace) {
    // GPU times are relative to tev0, recorded right after the call began.
    for (int c = 0; c < chunks; ++c) {
      float g0 = 0.0f, g1 = 0.0f;
      cudaEventElapsedTime(&g0, tev0, tev[2 * c]);
      cudaEventElapsedTime(&g1, tev0, tev[2 * c + 1]);
      std::fprintf(stderr, "chunk %2d ligands %5d-%5d host prep %7.3f-%7.3f ms  gpu %7.3f-%7.3f ms\n", c,
                   bounds[c], bounds[c + 1], tprep[2 * c], tprep[2 * c + 1], g0, g1);
    }
    std::fprintf(stderr, "call total %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t_end - t_start).count());
    for (auto e : tev) cudaEventDestroy(e);
    cudaEventDestroy(tev0);
  }
  ctx->timing.host_pack_ms = prep_ms;
  ctx->timing.host_post_ms = post_ms;
  ctx->timing.total_ms = std::chrono::duration<float, std::milli>(t_end - t_start).count();
  return GD_OK;
}

// ---------------------------------------------------------------------------
// Fine-grained drop-in entry points: every ligand of `b` with one
// caller-given fragment (the device descriptors carry it as the ligand's
// only fragment: nfrag 1 at frag_off l).
// ---------------------------------------------------------------------------
static int stage_fragments(gd_ctx* ctx, const gd_ligand_batch* b, const gd_fragment_set* fs,
                           const char* who, DockParams& p) {
  if (b == nullptr || fs == nullptr || b->n_ligands < 0 ||
      (b->n_ligands > 0 && (!b->atom_offsets || !b->xyz || !b->radii || !b->bond_offsets ||
                            !fs->membership || !fs->axis_atom || !fs->anchor_atom ||
                            (b->bond_offsets[b->n_ligands] > 0 && (!b->bonds || !b->bond_rotatable)))))
    return ctx->fail(GD_ERR_INVALID, std::string(who) + ": invalid ligand batch or fragments");
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  const int L = b->n_ligands;
  for (int l = 0; l < L; ++l) {
    const int a0 = b->atom_offsets[l], n = b->atom_offsets[l + 1] - a0;
    if (n < 0 || b->bond_offsets[l + 1] < b->bond_offsets[l])
      return ctx->fail(GD_ERR_INVALID, std::string(who) + ": offsets not ascending");
    const int ax = fs->axis_atom[l], an = fs->anchor_atom[l];
    if (ax < 0 || ax >= n || an < 0 || an >= n || ax == an)
      return ctx->fail(GD_ERR_INVALID, std::string(who) + ": fragment axis/anchor atom out of range");
    int nf = 0;
    for (int i = 0; i < n; ++i) nf += fs->membership[a0 + i] != 0;
    if (nf < 1 || nf >= n)
      return ctx->fail(GD_ERR_INVALID, std::string(who) + ": fragment must hold 1..n-1 atoms");
  }
  std::vector<PreparedLigand> prep(L);
  std::atomic<int> next{0};
  auto work = [&] {
    for (int l; (l = next.fetch_add(1)) < L;) {
      const int a0 = b->atom_offsets[l], b0 = b->bond_offsets[l];
      prep[l] = prepare_ligand(std::to_string(l), b->atom_offsets[l + 1] - a0, b->xyz + 3 * a0,
                               b->radii + a0, b->bond_offsets[l + 1] - b0, b->bonds + 2 * b0,
                               b->bond_rotatable + b0);
    }
  };
  if (L < 64) {
    work();
  } else {
    if (!ctx->pool)
      ctx->pool = std::make_unique<WorkerPool>((ctx->pool_threads > 0 ? ctx->pool_threads : host_threads()) - 1);
    ctx->pool->run(work);
  }
  const int A = L > 0 ? b->atom_offsets[L] : 0;
  std::vector<LigMeta> meta(std::max(L, 1));
  std::vector<uint64_t> far, fmask;
  std::vector<int32_t> fax(std::max(L, 1)), fan(std::max(L, 1)), stat(std::max(L, 1), 0);
  std::vector<double> frel(std::max(L, 1));
  ctx->errors.assign(L, std::string());
  ctx->status_host.assign(L, 0);
  int max_n = 1;
  for (int l = 0; l < L; ++l) {
    const PreparedLigand& q = prep[l];
    const int a0 = b->atom_offsets[l], n = b->atom_offsets[l + 1] - a0;
    LigMeta& m = meta[l];
    m.atom_off = a0;
    m.n = n;
    m.status = q.status;
    m.frag_off = l;
    m.nfrag = q.status == 0 ? 1 : 0;
    m.far_off = static_cast<int32_t>(far.size());
    m.fmask_off = static_cast<int32_t>(fmask.size());
    m.words = q.words;
    stat[l] = q.status;
    ctx->status_host[l] = q.status;
    ctx->errors[l] = q.error;
    fax[l] = fs->axis_atom[l];
    fan[l] = fs->anchor_atom[l];
    frel[l] = 0.0;
    if (q.status != 0) continue;
    far.insert(far.end(), q.far_mask.begin(), q.far_mask.end());
    int nf = 0;
    for (int w = 0; w < q.words; ++w) {
      uint64_t word = 0;
      for (int i = 64 * w; i < std::min(n, 64 * w + 64); ++i)
        if (fs->membership[a0 + i]) word |= 1ull << (i - 64 * w);
      nf += __builtin_popcountll(word);
      fmask.push_back(word);
    }
    frel[l] = static_cast<double>(nf) / n;
    max_n = std::max(max_n, n);
  }
  auto up = [&](DevBuf& d, const void* src, size_t bytes) -> int {
    GD_CUDA(ctx, d.ensure(std::max<size_t>(bytes, 8)));
    if (bytes) GD_CUDA(ctx, cudaMemcpyAsync(d.ptr, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return GD_OK;
  };
  int rc;
  if ((rc = up(ctx->meta, meta.data(), sizeof(LigMeta) * L))) return rc;
  if ((rc = up(ctx->xyz, b->xyz, sizeof(double) * 3 * A))) return rc;
  if ((rc = up(ctx->radii, b->radii, sizeof(double) * A))) return rc;
  if ((rc = up(ctx->far, far.data(), sizeof(uint64_t) * far.size()))) return rc;
  if ((rc = up(ctx->fmask, fmask.data(), sizeof(uint64_t) * fmask.size()))) return rc;
  if ((rc = up(ctx->fax, fax.data(), sizeof(int32_t) * L))) return rc;
  if ((rc = up(ctx->fan, fan.data(), sizeof(int32_t) * L))) return rc;
  if ((rc = up(ctx->frel, frel.data(), sizeof(double) * L))) return rc;
  if ((rc = up(ctx->o_status, stat.data(), sizeof(int32_t) * L))) return rc;
  // The staged descriptors now hold one caller fragment per ligand, not a
  // dockable batch.
  ctx->staged = false;
  ctx->have_result = false;
  ctx->n_lig = L;
  ctx->total_atoms = A;
  ctx->max_n = max_n;
  if (L > 0) ctx->atom_off.assign(b->atom_offsets, b->atom_offsets + L + 1);
  else ctx->atom_off.assign(1, 0);
  p = DockParams{};
  p.n_lig = L;
  p.meta = ctx->meta.as<LigMeta>();
  p.xyz = ctx->xyz.as<double>();
  p.radii = ctx->radii.as<double>();
  p.far_mask = ctx->far.as<uint64_t>();
  p.frag_mask = ctx->fmask.as<uint64_t>();
  p.frag_axis = ctx->fax.as<int32_t>();
  p.frag_anchor = ctx->fan.as<int32_t>();
  p.frag_rel = ctx->frel.as<double>();
  p.pocket = ctx->view;
  p.cos_deg = ctx->cos_t.as<double>();
  p.sin_deg = ctx->sin_t.as<double>();
  p.max_n = max_n;
  p.max_pairs = std::max(1, max_n * max_n / 4);
  p.status = ctx->o_status.as<int32_t>();
  p.reps = 1;
  return GD_OK;
}

static int fetch(gd_ctx* ctx, void* dst, const DevBuf& src, size_t bytes) {
  if (dst == nullptr || bytes == 0) return GD_OK;
  return ctx->cuda(cudaMemcpyAsync(dst, src.ptr, bytes, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
}

extern "C" int gd_optimize_fragment_batch(gd_ctx* ctx, const gd_ligand_batch* batch,
                                          const gd_fragment_set* fragments, int32_t step,
                                          int32_t refined, const double* entry_score,
                                          int32_t* best_angle, double* best_score,
                                          int64_t* evaluations, int64_t* feasibility_checks,
                                          double* out_pose, int32_t* status) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  const char* who = refined ? "optimize_fragment_refined" : "optimize_fragment_flat";
  if (step < 1 || 360 % step != 0) return ctx->fail(GD_ERR_INVALID, std::string(who) + ": step must divide 360");
  if (ctx->P == 0) return ctx->fail(GD_ERR_NO_POCKET, std::string(who) + ": no pocket staged (gd_set_pocket)");
  DockParams p;
  int rc = stage_fragments(ctx, batch, fragments, who, p);
  if (rc != GD_OK) return rc;
  const int L = p.n_lig;
  const size_t A = static_cast<size_t>(ctx->total_atoms);
  p.hp = step;
  p.lp = step;
  p.refine = refined ? 1 : 0;
  p.tile = gd_optimal_tile_size(step);
  GD_CUDA(ctx, ctx->st_final.ensure(sizeof(double) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->st_evals.ensure(sizeof(int64_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->st_checks.ensure(sizeof(int64_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_orient.ensure(sizeof(int32_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->seed_score.ensure(sizeof(double) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_pose.ensure(sizeof(double) * 3 * std::max<size_t>(A, 1)));
  if (entry_score && L > 0)
    GD_CUDA(ctx, cudaMemcpyAsync(ctx->seed_score.ptr, entry_score, sizeof(double) * L,
                                 cudaMemcpyHostToDevice, ctx->stream));
  FragmentIO io{};
  io.refined = refined ? 1 : 0;
  io.entry_score = entry_score ? ctx->seed_score.as<double>() : nullptr;
  io.best_angle = ctx->o_orient.as<int32_t>();
  io.best_score = ctx->st_final.as<double>();
  io.evaluations = ctx->st_evals.as<int64_t>();
  io.checks = ctx->st_checks.as<int64_t>();
  io.pose = ctx->o_pose.as<double>();
  GD_CUDA(ctx, static_cast<cudaError_t>(p.pocket.compact ? launch_fragment_search_cp(p, io, ctx->stream)
                                                         : launch_fragment_search(p, io, ctx->stream)));
  if ((rc = fetch(ctx, best_angle, ctx->o_orient, sizeof(int32_t) * L))) return rc;
  if ((rc = fetch(ctx, best_score, ctx->st_final, sizeof(double) * L))) return rc;
  if ((rc = fetch(ctx, evaluations, ctx->st_evals, sizeof(int64_t) * L))) return rc;
  if ((rc = fetch(ctx, feasibility_checks, ctx->st_checks, sizeof(int64_t) * L))) return rc;
  if ((rc = fetch(ctx, out_pose, ctx->o_pose, sizeof(double) * 3 * A))) return rc;
  if ((rc = fetch(ctx, status, ctx->o_status, sizeof(int32_t) * L))) return rc;
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->timing = gd_timing{};
  ctx->timing.launches = L > 0 ? 1 : 0;
  return GD_OK;
}

extern "C" int gd_rotate_fragment_batch(gd_ctx* ctx, const gd_ligand_batch* batch,
                                        const gd_fragment_set* fragments, const double* angles_deg,
                                        double* out_pose, int32_t* status) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  if (batch && batch->n_ligands > 0 && (angles_deg == nullptr || out_pose == nullptr))
    return ctx->fail(GD_ERR_INVALID, "rotate_fragment: null angles or output");
  DockParams p;
  int rc = stage_fragments(ctx, batch, fragments, "rotate_fragment", p);
  if (rc != GD_OK) return rc;
  const int L = p.n_lig;
  const size_t A = static_cast<size_t>(ctx->total_atoms);
  // cos/sin of angle * (pi/180) from the host libm (geometry.hpp:176-178).
  std::vector<double> cs(std::max(L, 1)), sn(std::max(L, 1));
  std::vector<uint8_t> zero(std::max(L, 1));
  for (int l = 0; l < L; ++l) {
    zero[l] = angles_deg[l] == 0.0;
    trig_of(angles_deg[l], cs[l], sn[l]);
  }
  GD_CUDA(ctx, ctx->st_final.ensure(sizeof(double) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->seed_score.ensure(sizeof(double) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_orient.ensure(sizeof(int32_t) * std::max(L, 1)));
  GD_CUDA(ctx, ctx->o_pose.ensure(sizeof(double) * 3 * std::max<size_t>(A, 1)));
  if (L > 0) {
    GD_CUDA(ctx, cudaMemcpyAsync(ctx->st_final.ptr, cs.data(), sizeof(double) * L, cudaMemcpyHostToDevice, ctx->stream));
    GD_CUDA(ctx, cudaMemcpyAsync(ctx->seed_score.ptr, sn.data(), sizeof(double) * L, cudaMemcpyHostToDevice, ctx->stream));
    GD_CUDA(ctx, cudaMemcpyAsync(ctx->o_orient.ptr, zero.data(), L, cudaMemcpyHostToDevice, ctx->stream));
  }
  GD_CUDA(ctx, static_cast<cudaError_t>(launch_fragment_rotate(
                   p, ctx->st_final.as<double>(), ctx->seed_score.as<double>(),
                   static_cast<const uint8_t*>(ctx->o_orient.ptr), ctx->o_pose.as<double>(), ctx->stream)));
  if ((rc = fetch(ctx, out_pose, ctx->o_pose, sizeof(double) * 3 * A))) return rc;
  if ((rc = fetch(ctx, status, ctx->o_status, sizeof(int32_t) * L))) return rc;
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GD_OK;
}

extern "C" int gd_check_bumps_batch(gd_ctx* ctx, const gd_ligand_batch* batch,
                                    const gd_fragment_set* fragments, uint8_t* feasible,
                                    int32_t* status) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  if (batch && batch->n_ligands > 0 && feasible == nullptr)
    return ctx->fail(GD_ERR_INVALID, "check_bumps: null output");
  DockParams p;
  int rc = stage_fragments(ctx, batch, fragments, "check_bumps", p);
  if (rc != GD_OK) return rc;
  const int L = p.n_lig;
  GD_CUDA(ctx, ctx->o_orient.ensure(sizeof(int32_t) * std::max(L, 1)));
  GD_CUDA(ctx, static_cast<cudaError_t>(launch_fragment_bumps(
                   p, static_cast<uint8_t*>(ctx->o_orient.ptr), ctx->stream)));
  if (L > 0) GD_CUDA(ctx, cudaMemcpyAsync(feasible, ctx->o_orient.ptr, L, cudaMemcpyDeviceToHost, ctx->stream));
  if ((rc = fetch(ctx, status, ctx->o_status, sizeof(int32_t) * L))) return rc;
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GD_OK;
}

extern "C" int gd_ligand_graph(int32_t n_atoms, const double* xyz, const double* radii,
                               int32_t n_bonds, const int32_t* bonds, const uint8_t* rotatable,
                               int32_t* n_rotamers, int32_t* rotamer_bonds, uint8_t* membership,
                               char* msg, size_t msg_len) {
  if (n_atoms < 0 || n_bonds < 0 || (n_atoms > 0 && (!xyz || !radii)) ||
      (n_bonds > 0 && (!bonds || !rotatable)) || !n_rotamers)
    return GD_LIG_INVALID;
  // The graph itself has no size limit (host code); the docking path's is kWideAtoms.
  const PreparedLigand p = prepare_ligand("L", n_atoms, xyz, radii, n_bonds, bonds, rotatable, kWideAtoms);
  if (msg && msg_len) {
    std::strncpy(msg, p.error.c_str(), msg_len - 1);
    msg[msg_len - 1] = 0;
  }
  *n_rotamers = p.status == GD_LIG_OK ? static_cast<int32_t>(p.rot_bond.size()) : 0;
  if (p.status != GD_LIG_OK) return p.status;
  for (int r = 0; r < *n_rotamers; ++r) {
    if (rotamer_bonds) rotamer_bonds[r] = p.rot_bond[r];
    if (membership)
      for (int side = 0; side < 2; ++side)
        for (int i = 0; i < n_atoms; ++i)
          membership[static_cast<size_t>(2 * r + side) * n_atoms + i] =
              (p.frag_mask[static_cast<size_t>(2 * r + side) * p.words + i / 64] >> (i % 64)) & 1u;
  }
  return GD_LIG_OK;
}

extern "C" int gd_rotation_profiles(gd_ctx* ctx, uint32_t flags, double* scores, uint8_t* valid,
                                    double* relative_size, int32_t* frag_offsets, int32_t* status,
                                    int64_t capacity) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  if (!ctx->staged) return ctx->fail(GD_ERR_INVALID, "gd_rotation_profiles: no batch staged (gd_upload)");
  if (ctx->P == 0)
    return ctx->fail(GD_ERR_NO_POCKET, "gd_rotation_profiles: no pocket staged (gd_set_pocket)");
  if (frag_offsets == nullptr || (capacity > 0 && (scores == nullptr || valid == nullptr)))
    return ctx->fail(GD_ERR_INVALID, "gd_rotation_profiles: null output");
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  const int L = ctx->n_lig;
  // The fragment counts and relative sizes the GPU preprocessing wrote.
  std::vector<LigMeta> meta(std::max(L, 1));
  std::vector<double> hrel(std::max<size_t>(ctx->frag_total, 1));
  if (L > 0) {
    GD_CUDA(ctx, cudaMemcpyAsync(meta.data(), ctx->meta.ptr, sizeof(LigMeta) * L, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    GD_CUDA(ctx, cudaMemcpyAsync(hrel.data(), ctx->frel.ptr, sizeof(double) * hrel.size(),
                                 cudaMemcpyDeviceToHost, ctx->stream));
    GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  std::vector<int32_t> items;
  frag_offsets[0] = 0;
  std::vector<int> wide_skipped;
  for (int l = 0; l < L; ++l) {
    int nf = ctx->status_host[l] == 0 ? meta[l].nfrag : 0;
    if (nf > 0 && is_wide(meta[l].n)) {
      // The profile kernel is a warp-per-fragment kernel (8-bit atom
      // indices): wide ligands are reported as skipped, not profiled.
      nf = 0;
      wide_skipped.push_back(l);
      ctx->errors[l] = "ligand '" + std::to_string(l) + "': more than " + std::to_string(kNarrowAtoms) +
                       " atoms is not supported by gd_rotation_profiles";
    }
    for (int f = 0; f < nf; ++f) {
      items.push_back(l);
      items.push_back(f);
    }
    frag_offsets[l + 1] = frag_offsets[l] + nf;
  }
  const int64_t n_items = static_cast<int64_t>(items.size() / 2);
  if (n_items > capacity) {
    return ctx->fail(GD_ERR_INVALID, "gd_rotation_profiles: capacity " + std::to_string(capacity) +
                                         " < " + std::to_string(n_items) + " fragments");
  }
  if (relative_size)
    for (int64_t it = 0; it < n_items; ++it)
      relative_size[it] = hrel[meta[items[2 * it]].frag_off + items[2 * it + 1]];
  if (n_items > 0) {
    GD_CUDA(ctx, ctx->prof_items.ensure(sizeof(int32_t) * items.size()));
    GD_CUDA(ctx, ctx->prof_scores.ensure(sizeof(double) * 360 * n_items));
    GD_CUDA(ctx, ctx->prof_valid.ensure(360 * n_items));
    GD_CUDA(ctx, cudaMemcpyAsync(ctx->prof_items.ptr, items.data(), sizeof(int32_t) * items.size(),
                                 cudaMemcpyHostToDevice, ctx->stream));
    DockParams p{};
    p.meta = ctx->meta.as<LigMeta>();
    p.xyz = ctx->xyz.as<double>();
    p.radii = ctx->radii.as<double>();
    p.far_mask = ctx->far.as<uint64_t>();
    p.frag_mask = ctx->fmask.as<uint64_t>();
    p.frag_axis = ctx->fax.as<int32_t>();
    p.frag_anchor = ctx->fan.as<int32_t>();
    p.frag_rel = ctx->frel.as<double>();
    p.pocket = ctx->view;
    p.pocket.use_index = (flags & GD_FLAG_BRUTE_FORCE) ? 0 : ctx->view.use_index;
    p.cos_deg = ctx->cos_t.as<double>();
    p.sin_deg = ctx->sin_t.as<double>();
    p.max_n = ctx->max_n;
    p.max_pairs = std::max(1, ctx->max_n * ctx->max_n / 4);
    p.status = ctx->o_status.as<int32_t>();
    if (flags & GD_FLAG_COUNT_WORK) {
      GD_CUDA(ctx, ctx->counters.ensure(sizeof(unsigned long long) * kCounterSlots));
      GD_CUDA(ctx, cudaMemsetAsync(ctx->counters.ptr, 0, sizeof(unsigned long long) * kCounterSlots,
                                   ctx->stream));
      p.counters = ctx->counters.as<unsigned long long>();
    }
    ctx->counted = p.counters != nullptr;
    ctx->timing = gd_timing{};
    cudaEventRecord(ctx->ev[2], ctx->stream);
    GD_CUDA(ctx, static_cast<cudaError_t>((p.pocket.compact ? launch_profiles_cp : launch_profiles)(
                     p, ctx->prof_items.as<int32_t>(), static_cast<int>(n_items),
                     ctx->prof_scores.as<double>(), ctx->prof_valid.as<uint8_t>(), ctx->stream)));
    cudaEventRecord(ctx->ev[3], ctx->stream);
    GD_CUDA(ctx, cudaMemcpyAsync(scores, ctx->prof_scores.ptr, sizeof(double) * 360 * n_items,
                                 cudaMemcpyDeviceToHost, ctx->stream));
    GD_CUDA(ctx, cudaMemcpyAsync(valid, ctx->prof_valid.ptr, 360 * n_items, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    cudaEventRecord(ctx->ev[4], ctx->stream);
    ctx->timing.launches = 1;
    ctx->timing.h2d_bytes = static_cast<int64_t>(sizeof(int32_t) * items.size());
    ctx->timing.d2h_bytes = static_cast<int64_t>(9 * 360 * n_items);
  }
  if (status && L > 0)
    GD_CUDA(ctx, cudaMemcpyAsync(status, ctx->o_status.ptr, sizeof(int32_t) * L,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (status)
    for (const int l : wide_skipped) status[l] = GD_LIG_INVALID;
  if (n_items > 0) {
    cudaEventElapsedTime(&ctx->timing.flex_ms, ctx->ev[2], ctx->ev[3]);
    cudaEventElapsedTime(&ctx->timing.total_ms, ctx->ev[2], ctx->ev[4]);
  }
  return GD_OK;
}

extern "C" int gd_ligand_error(const gd_ctx* ctx, int32_t ligand, char* msg, size_t msg_len) {
  if (ctx == nullptr || ligand < 0 || ligand >= static_cast<int32_t>(ctx->errors.size()))
    return GD_ERR_INVALID;
  if (msg && msg_len) {
    std::strncpy(msg, ctx->errors[ligand].c_str(), msg_len - 1);
    msg[msg_len - 1] = 0;
  }
  return GD_OK;
}

extern "C" int gd_device_results(const gd_ctx* ctx, gd_device_result* out) {
  if (ctx == nullptr || out == nullptr || !ctx->have_result) return GD_ERR_INVALID;
  out->orientation = ctx->o_orient.as<int32_t>();
  out->seed_rank = ctx->o_rank.as<int32_t>();
  out->final_score = ctx->o_final.as<double>();
  out->evaluations = ctx->o_evals.as<int64_t>();
  out->n_ligands = ctx->n_lig;
  out->top_k = ctx->last_topk;
  out->rigid_score = ctx->o_rigid.as<double>();
  out->feasibility_checks = ctx->o_checks.as<int64_t>();
  out->k_eff = ctx->k_eff.as<int32_t>();
  out->poses_scored = ctx->o_scored.as<int64_t>();
  out->status = ctx->o_status.as<int32_t>();
  return GD_OK;
}

extern "C" int gd_work_counters(const gd_ctx* ctx, uint64_t out[16]) {
  if (ctx == nullptr || out == nullptr) return GD_ERR_INVALID;
  if (!ctx->counted) return GD_ERR_INVALID;
  if (cudaMemcpy(out, ctx->counters.ptr, sizeof(uint64_t) * 16, cudaMemcpyDeviceToHost) != cudaSuccess)
    return GD_ERR_CUDA;
  return GD_OK;
}

extern "C" int gd_phase_clocks(const gd_ctx* ctx, uint64_t out[16]) {
  if (ctx == nullptr || out == nullptr) return GD_ERR_INVALID;
  if (!ctx->counted) return GD_ERR_INVALID;
  if (cudaMemcpy(out, ctx->counters.as<unsigned long long>() + kPhaseBase, sizeof(uint64_t) * 16,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return GD_ERR_CUDA;
  return GD_OK;
}

extern "C" int gd_fp64_peak(gd_ctx* ctx, double* tflops) {
  if (ctx == nullptr || tflops == nullptr) return GD_ERR_INVALID;
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  int sms = 0;
  GD_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  DevBuf sink;
  GD_CUDA(ctx, sink.ensure(64));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    GD_CUDA(ctx, cudaEventRecord(ctx->ev[0], ctx->stream));
    GD_CUDA(ctx, static_cast<cudaError_t>(
                     launch_fp64_probe(sink.as<double>(), blocks, threads, iters, ctx->stream)));
    GD_CUDA(ctx, cudaEventRecord(ctx->ev[1], ctx->stream));
    GD_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    if (rep > 0) best = std::min(best, ms);
  }
  const double ops = 2.0 * 8.0 * static_cast<double>(blocks) * threads * iters;
  *tflops = ops / (best * 1e-3) / 1e12;
  return GD_OK;
}

extern "C" int gd_l2_gather_peak(gd_ctx* ctx, double* gbs) {
  if (ctx == nullptr || gbs == nullptr) return GD_ERR_INVALID;
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  int sms = 0;
  GD_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const unsigned long long n_rec = (48ull << 20) / 32;  // 48 MB of 32-byte records
  DevBuf buf, sink;
  GD_CUDA(ctx, buf.ensure(32 * n_rec));
  GD_CUDA(ctx, sink.ensure(64));
  GD_CUDA(ctx, cudaMemsetAsync(buf.ptr, 0, 32 * n_rec, ctx->stream));
  const int blocks = sms * 8, threads = 256, iters = 256;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {  // the first pass warms L2
    GD_CUDA(ctx, cudaEventRecord(ctx->ev[0], ctx->stream));
    GD_CUDA(ctx, static_cast<cudaError_t>(launch_l2_gather_probe(
                     buf.as<double>(), n_rec, blocks, threads, iters, sink.as<double>(), ctx->stream)));
    GD_CUDA(ctx, cudaEventRecord(ctx->ev[1], ctx->stream));
    GD_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    if (rep > 0) best = std::min(best, ms);
  }
  const double bytes = 32.0 * 4.0 * static_cast<double>(blocks) * threads * iters;
  *gbs = bytes / (best * 1e-3) / 1e9;
  return GD_OK;
}

extern "C" int gd_l2_gather_rate(gd_ctx* ctx, int32_t warps_per_sm, double* gbs) {
  if (ctx == nullptr || gbs == nullptr || warps_per_sm < 1) return GD_ERR_INVALID;
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  int sms = 0;
  GD_CUDA(ctx, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const unsigned long long n_rec = (48ull << 20) / 32;  // the same 48 MB L2-resident buffer
  DevBuf buf, sink;
  GD_CUDA(ctx, buf.ensure(32 * n_rec));
  GD_CUDA(ctx, sink.ensure(64));
  GD_CUDA(ctx, cudaMemsetAsync(buf.ptr, 0, 32 * n_rec, ctx->stream));
  const int threads = 32 * std::min(warps_per_sm, 32), blocks = sms * ((warps_per_sm + 31) / 32);
  const int iters = 1024;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    GD_CUDA(ctx, cudaEventRecord(ctx->ev[0], ctx->stream));
    GD_CUDA(ctx, static_cast<cudaError_t>(launch_l2_chase_probe(buf.as<double>(), n_rec, blocks, threads,
                                                                 iters, sink.as<double>(), ctx->stream)));
    GD_CUDA(ctx, cudaEventRecord(ctx->ev[1], ctx->stream));
    GD_CUDA(ctx, cudaEventSynchronize(ctx->ev[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    if (rep > 0) best = std::min(best, ms);
  }
  *gbs = 32.0 * static_cast<double>(blocks) * threads * iters / (best * 1e-3) / 1e9;
  return GD_OK;
}

extern "C" int gd_last_timing(const gd_ctx* ctx, gd_timing* out) {
  if (ctx == nullptr || out == nullptr) return GD_ERR_INVALID;
  *out = ctx->timing;
  return GD_OK;
}

extern "C" int gd_overlap_score_batch(gd_ctx* ctx, const double* xyz, int32_t n_atoms,
                                      int32_t n_poses, uint32_t flags, double* out) {
  if (ctx == nullptr) return GD_ERR_INVALID;
  if (ctx->P == 0) return ctx->fail(GD_ERR_NO_POCKET, "overlap_score: no pocket staged");
  if (n_atoms < 1) return ctx->fail(GD_ERR_INVALID, "overlap_score: empty pose");
  if (n_poses < 0 || (n_poses > 0 && (xyz == nullptr || out == nullptr)))
    return ctx->fail(GD_ERR_INVALID, "overlap_score: invalid arguments");
  if (n_poses == 0) return GD_OK;
  GD_CUDA(ctx, cudaSetDevice(ctx->device));
  DevBuf dx, dout;
  const size_t bytes = sizeof(double) * 3 * static_cast<size_t>(n_atoms) * n_poses;
  GD_CUDA(ctx, dx.ensure(bytes));
  GD_CUDA(ctx, dout.ensure(sizeof(double) * n_poses));
  GD_CUDA(ctx, cudaMemcpyAsync(dx.ptr, xyz, bytes, cudaMemcpyHostToDevice, ctx->stream));
  PocketView v = ctx->view;
  v.use_index = (flags & GD_FLAG_BRUTE_FORCE) ? 0 : 1;
  GD_CUDA(ctx, static_cast<cudaError_t>(launch_score_poses(v, dx.as<double>(), n_atoms, n_poses,
                                                           dout.as<double>(), ctx->stream)));
  GD_CUDA(ctx, cudaMemcpyAsync(out, dout.ptr, sizeof(double) * n_poses, cudaMemcpyDeviceToHost,
                               ctx->stream));
  GD_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GD_OK;
}

// ---------------------------------------------------------------------------
// Multi-device dispatch (gd_multi_*): one gd_ctx, host thread and set of
// streams per device; a batch is cut into cost-weighted chunks that the
// device threads pull from a shared atomic cursor (the GPU analogue of the
// reference screen's bounded work queue, screening.hpp:96-178), each chunk
// docked by the pipelined single-device path and its results written
// straight into the caller's arrays at the chunk's global offsets.
// ---------------------------------------------------------------------------
struct gd_multi {
  std::vector<gd_ctx*> ctx;
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable cv, done;
  const std::function<void(int)>* job = nullptr;
  int gen = 0, busy = 0;
  bool stop = false;
  std::string err;
  std::vector<gd_multi_stats> stats;
  std::vector<std::pair<int, std::string>> lig_errors;  // last call: (global position, text)

  void loop(int d) {
    int seen = 0;
    for (;;) {
      const std::function<void(int)>* j;
      {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        j = job;
      }
      (*j)(d);
      std::lock_guard<std::mutex> g(mu);
      if (--busy == 0) done.notify_one();
    }
  }
  // Runs fn(d) on every device thread; returns when all have finished.
  void run(const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> g(mu);
      job = &fn;
      busy = static_cast<int>(th.size());
      ++gen;
    }
    cv.notify_all();
    std::unique_lock<std::mutex> g(mu);
    done.wait(g, [&] { return busy == 0; });
  }
  ~gd_multi() {
    {
      std::lock_guard<std::mutex> g(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
    for (gd_ctx* c : ctx) gd_destroy(c);
  }
};

namespace {
thread_local std::string g_multi_create_error;
}

extern "C" int gd_multi_create(const int32_t* devices, int32_t n_devices, gd_multi** out) {
  if (out == nullptr) {
    g_multi_create_error = "gd_multi_create: null output pointer";
    return GD_ERR_INVALID;
  }
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    g_multi_create_error = "gd_multi_create: no CUDA device";
    return GD_ERR_CUDA;
  }
  std::vector<int> devs;
  if (devices != nullptr) {
    if (n_devices < 1) {
      g_multi_create_error = "gd_multi_create: empty device list";
      return GD_ERR_INVALID;
    }
    devs.assign(devices, devices + n_devices);
  } else {
    const int k = n_devices > 0 ? std::min<int>(n_devices, count) : count;
    for (int d = 0; d < k; ++d) devs.push_back(d);
  }
  auto m = std::make_unique<gd_multi>();
  // The host cores are shared by the device threads' preprocessing pools.
  const int per = std::max(1, host_threads() / static_cast<int>(devs.size()));
  for (int d : devs) {
    gd_ctx* c = nullptr;
    const int rc = gd_create(d, &c);
    if (rc != GD_OK) {
      g_multi_create_error = std::string("gd_multi_create: ") + gd_last_error(nullptr);
      return rc;
    }
    c->pool_threads = per;
    m->ctx.push_back(c);
  }
  m->stats.assign(devs.size(), gd_multi_stats{});
  for (size_t d = 0; d < devs.size(); ++d) m->th.emplace_back([p = m.get(), d] { p->loop(static_cast<int>(d)); });
  *out = m.release();
  return GD_OK;
}

extern "C" int gd_multi_destroy(gd_multi* m) {
  delete m;
  return GD_OK;
}

extern "C" const char* gd_multi_last_error(const gd_multi* m) {
  return m ? m->err.c_str() : g_multi_create_error.c_str();
}

extern "C" int32_t gd_multi_size(const gd_multi* m) { return m ? static_cast<int32_t>(m->ctx.size()) : 0; }

extern "C" gd_ctx* gd_multi_context(gd_multi* m, int32_t i) {
  return (m && i >= 0 && i < static_cast<int32_t>(m->ctx.size())) ? m->ctx[i] : nullptr;
}

extern "C" int gd_multi_set_pocket(gd_multi* m, const double* xyz, int32_t n_points) {
  if (m == nullptr) return GD_ERR_INVALID;
  std::vector<int> rc(m->ctx.size(), GD_OK);
  m->run([&](int d) { rc[d] = gd_set_pocket(m->ctx[d], xyz, n_points); });
  for (size_t d = 0; d < rc.size(); ++d)
    if (rc[d] != GD_OK) {
      m->err = m->ctx[d]->err;
      return rc[d];
    }
  return GD_OK;
}

extern "C" int gd_multi_dock_batch(gd_multi* m, const gd_ligand_batch* b, const gd_knobs* k,
                                   gd_result* r) {
  if (m == nullptr) return GD_ERR_INVALID;
  auto fail = [&](int code, const std::string& msg) {
    m->err = msg;
    return code;
  };
  if (r == nullptr) return fail(GD_ERR_INVALID, "gd_dock_batch: null result");
  if (k == nullptr) return fail(GD_ERR_INVALID, "knob config: null");
  char msg[128];
  if (gd_validate_knobs(k, msg, sizeof msg) != GD_OK) return fail(GD_ERR_INVALID, msg);
  if (b == nullptr || b->n_ligands < 0 ||
      (b->n_ligands > 0 && (!b->atom_offsets || !b->xyz || !b->radii || !b->bond_offsets ||
                            (b->bond_offsets[b->n_ligands] > 0 && (!b->bonds || !b->bond_rotatable)))))
    return fail(GD_ERR_INVALID, "gd_upload: invalid ligand batch");
  const int L = b->n_ligands;
  const int D = static_cast<int>(m->ctx.size());
  for (auto& st : m->stats) st = gd_multi_stats{};
  const bool rigid = k->rigid_step > 0;
  const int K = rigid ? k->top_k : 1;
  // Cost per ligand ~ rigid atom-orientations + restart chains' rotated
  // atoms: n (N_orient + K reps (1 + 2R (360/hp))).
  const int32_t n_orient = rigid ? gd_orientations(k->rigid_step, nullptr, nullptr, 0) : 0;
  std::vector<double> cost(L);
  double total = 0.0;
  for (int l = 0; l < L; ++l) {
    const int n = b->atom_offsets[l + 1] - b->atom_offsets[l];
    int R = 0;
    for (int e = b->bond_offsets[l]; e < b->bond_offsets[l + 1]; ++e) R += b->bond_rotatable[e] != 0;
    const double keff = rigid ? std::min(K, std::max<int32_t>(n_orient, 1)) : 1;
    cost[l] = std::max(n, 1) * (n_orient + keff * k->repetitions * (1.0 + 2.0 * R * (360.0 / k->high_precision_step)));
    total += cost[l];
  }
  // Chunks: ~4 per device of equal cost (at least 256 ligands), so the
  // cursor balances the ~10x cost spread of BASELINE ligands while each
  // chunk stays large enough for the single-device pipeline.
  std::vector<int> bounds{0};
  if (L > 0) {
    // One device has nothing to balance: one chunk, one pipeline ramp (c3
    // on one GPU: 0.80 s vs 0.86 s with 2 chunks per 4 x 100k docks).
    const int per_dev_chunks = D == 1 ? 1 : static_cast<int>(env_double("GD_MULTI_CHUNKS", 4));
    const double target = total / std::max(1, D * per_dev_chunks);
    double acc = 0.0;
    for (int l = 0; l < L; ++l) {
      acc += cost[l];
      if ((acc >= target && l + 1 - bounds.back() >= 256) || l + 1 == L) {
        bounds.push_back(l + 1);
        acc = 0.0;
      }
    }
  }
  const int chunks = static_cast<int>(bounds.size()) - 1;
  std::atomic<int> cursor{0};
  std::vector<int> rc(D, GD_OK);
  std::vector<std::string> errs(D);
  std::vector<std::vector<std::pair<int, std::string>>> lerr(D);
  m->lig_errors.clear();
  m->run([&](int d) {
    gd_ctx* c = m->ctx[d];
    std::vector<int32_t> ao, bo;
    for (int ci; (ci = cursor.fetch_add(1)) < chunks;) {
      const auto t0 = std::chrono::steady_clock::now();
      const int c0 = bounds[ci], c1 = bounds[ci + 1];
      const int a0 = b->atom_offsets[c0], e0 = b->bond_offsets[c0];
      ao.resize(c1 - c0 + 1);
      bo.resize(c1 - c0 + 1);
      for (int l = c0; l <= c1; ++l) {
        ao[l - c0] = b->atom_offsets[l] - a0;
        bo[l - c0] = b->bond_offsets[l] - e0;
      }
      const gd_ligand_batch sub{c1 - c0, ao.data(), b->xyz + 3 * static_cast<size_t>(a0),
                                b->radii + a0, bo.data(), b->bonds ? b->bonds + 2 * static_cast<size_t>(e0) : nullptr,
                                b->bond_rotatable ? b->bond_rotatable + e0 : nullptr};
      const size_t s0 = static_cast<size_t>(c0) * K;
      auto off = [](auto* p, size_t o) { return p ? p + o : nullptr; };
      gd_result sr{off(r->orientation, s0), off(r->seed_rank, s0), off(r->rigid_score, s0),
                   off(r->final_score, s0), off(r->evaluations, s0), off(r->feasibility_checks, s0),
                   off(r->final_pose, 3 * static_cast<size_t>(K) * a0), off(r->k_eff, c0),
                   off(r->poses_scored, c0), off(r->status, c0),
                   off(r->top_pose, 3 * static_cast<size_t>(a0))};
      const int e = gd_dock_batch(c, &sub, k, &sr);
      if (e != GD_OK) {
        rc[d] = e;
        errs[d] = c->err;
        cursor.store(chunks);  // stop handing out work
        return;
      }
      // Validation texts, re-keyed from chunk to batch positions.
      for (int l = 0; l < c1 - c0; ++l)
        if (!c->errors[l].empty()) {
          std::string t = c->errors[l];
          const std::string pre = "ligand '" + std::to_string(l) + "': ";
          if (t.rfind(pre, 0) == 0) t = "ligand '" + std::to_string(c0 + l) + "': " + t.substr(pre.size());
          lerr[d].emplace_back(c0 + l, std::move(t));
        }
      gd_multi_stats& st = m->stats[d];
      st.ligands += c1 - c0;
      st.chunks += 1;
      st.busy_ms += std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
  for (int d = 0; d < D; ++d)
    if (rc[d] != GD_OK) return fail(rc[d], errs[d]);
  for (auto& v : lerr) m->lig_errors.insert(m->lig_errors.end(), v.begin(), v.end());
  std::sort(m->lig_errors.begin(), m->lig_errors.end());
  return GD_OK;
}

extern "C" int gd_multi_ligand_error(const gd_multi* m, int32_t ligand, char* msg, size_t msg_len) {
  if (m == nullptr || ligand < 0) return GD_ERR_INVALID;
  const auto it = std::lower_bound(m->lig_errors.begin(), m->lig_errors.end(),
                                   std::make_pair(static_cast<int>(ligand), std::string()));
  const bool hit = it != m->lig_errors.end() && it->first == ligand;
  if (msg && msg_len) {
    std::strncpy(msg, hit ? it->second.c_str() : "", msg_len - 1);
    msg[msg_len - 1] = 0;
  }
  return GD_OK;
}

extern "C" int gd_multi_last_stats(const gd_multi* m, gd_multi_stats* out, int32_t cap) {
  if (m == nullptr || out == nullptr) return GD_ERR_INVALID;
  for (int32_t d = 0; d < std::min<int32_t>(cap, static_cast<int32_t>(m->stats.size())); ++d) out[d] = m->stats[d];
  return GD_OK;
}
