// Host half of the rotation-profile analysis (reference analysis.hpp:
// 61-147): peak extraction and the tile-hit model.  Both are O(360) per
// profile, so they stay on the host; the profiles themselves come from the
// GPU (gd_rotation_profiles, flex.cu profile_kernel).
#include <algorithm>
#include <cstdint>

#include "geodock_b200.h"

namespace {

// Closes the run [start, end) of qualifying angles into a peak.
gd_peak close_run(const double* scores, int start, int end, double vmin, double delta) {
  double top = scores[start];
  for (int a = start + 1; a < end; ++a) top = std::max(top, scores[a]);
  return gd_peak{start, end - start, (top - vmin) / delta};
}

}  // namespace

extern "C" int gd_detect_peaks(const double* scores, const uint8_t* valid, double* delta_overlap,
                               int32_t* best_peak_width, gd_peak* peaks, int32_t* n_peaks) {
  if (scores == nullptr || valid == nullptr || peaks == nullptr || n_peaks == nullptr)
    return GD_ERR_INVALID;
  // Range over valid angles; the first angle attaining the maximum wins.
  int arg_max = -1;
  double vmin = 0.0, vmax = 0.0;
  for (int a = 0; a < 360; ++a) {
    if (!valid[a]) continue;
    const double s = scores[a];
    if (arg_max < 0) {
      vmin = vmax = s;
      arg_max = a;
    } else {
      vmin = std::min(vmin, s);
      if (s > vmax) {
        vmax = s;
        arg_max = a;
      }
    }
  }
  *n_peaks = 0;
  if (best_peak_width) *best_peak_width = 0;
  if (arg_max < 0) return GD_ERR_INVALID;  // "detect_peaks: no feasible rotation"
  const double delta = vmax - vmin;
  if (delta_overlap) *delta_overlap = delta;
  if (delta == 0.0) return GD_OK;  // a flat profile has no peaks

  const double cut = vmin + 0.5 * delta;
  auto above = [&](int a) { return valid[a] && scores[a] > cut; };
  int np = 0, open = -1;
  for (int a = 0; a < 360; ++a) {
    if (above(a)) {
      if (open < 0) open = a;
    } else if (open >= 0) {
      peaks[np++] = close_run(scores, open, a, vmin, delta);
      open = -1;
    }
  }
  if (open >= 0) {
    gd_peak last = close_run(scores, open, 360, vmin, delta);
    if (np > 0 && peaks[0].start_angle == 0) {
      // The run through 359 continues at 0: fold the head run into it; the
      // merged peak keeps the tail's start and goes last.
      last.width += peaks[0].width;
      last.height_ratio = std::max(last.height_ratio, peaks[0].height_ratio);
      std::copy(peaks + 1, peaks + np, peaks);
      --np;
    }
    peaks[np++] = last;
  }
  *n_peaks = np;
  if (best_peak_width)
    for (int k = 0; k < np; ++k)
      if ((arg_max - peaks[k].start_angle + 360) % 360 < peaks[k].width) {
        *best_peak_width = peaks[k].width;
        break;
      }
  return GD_OK;
}

extern "C" int gd_tile_hit_probability(const int32_t* best_peak_widths, int64_t n,
                                       const int32_t* tiles, int32_t n_tiles, double* probability,
                                       double* eval_count) {
  if (n <= 0 || best_peak_widths == nullptr) return GD_ERR_INVALID;  // "empty dataset"
  if (n_tiles > 0 && (tiles == nullptr || probability == nullptr || eval_count == nullptr))
    return GD_ERR_INVALID;
  for (int32_t t = 0; t < n_tiles; ++t) {
    int64_t hits = 0;
    for (int64_t i = 0; i < n; ++i) hits += best_peak_widths[i] > tiles[t] ? 1 : 0;
    probability[t] = static_cast<double>(hits) / static_cast<double>(n);
    eval_count[t] = 360.0 / tiles[t] + static_cast<double>(tiles[t]);
  }
  return GD_OK;
}
