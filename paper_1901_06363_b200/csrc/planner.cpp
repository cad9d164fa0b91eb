// Host half of the planner (reference perf_model.hpp:57-105): the
// per-configuration cost model t = intercept + sum_j c_j x_j over the seven
// interaction features of (pocket points, avg atoms, avg rotamers), fitted
// by ordinary least squares.  The reference solves it with Eigen's
// ColPivHouseholderQR; Eigen is not part of this build, so this is a
// self-contained column-pivoting Householder QR (Businger-Golub) with the
// same rank rule (|R_kk| <= eps * min(n, p) * |R_00| ends the rank) and the
// same error messages.  Results agree with any exact least-squares solver to
// rounding (tests/test_planner_cpu.py checks numpy's lstsq and the
// reference's own test cases).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "geodock_b200.h"

namespace {

constexpr int kPredictors = 7;
constexpr int kCols = kPredictors + 1;  // + intercept
const char* const kNames[kCols] = {"pocket_points",
                                   "avg_atoms",
                                   "avg_rotamers",
                                   "pocket_points*avg_atoms",
                                   "pocket_points*avg_rotamers",
                                   "avg_atoms*avg_rotamers",
                                   "pocket_points*avg_atoms*avg_rotamers",
                                   "intercept"};

int fail(char* msg, size_t len, const std::string& text) {
  if (msg && len) {
    std::strncpy(msg, text.c_str(), len - 1);
    msg[len - 1] = 0;
  }
  return GD_ERR_INVALID;
}

}  // namespace

extern "C" void gd_cost_features(const double* features, double* x) {
  const double pp = features[0], la = features[1], lr = features[2];
  const double v[kPredictors] = {pp, la, lr, pp * la, pp * lr, la * lr, pp * la * lr};
  for (int j = 0; j < kPredictors; ++j) x[j] = v[j];
}

extern "C" int gd_fit_cost_model(const double* features, const double* times, int32_t n,
                                 double* coef, double* intercept, double* adjusted_r2, char* msg,
                                 size_t msg_len) {
  const int p = kCols;
  if (n < p + 1)
    return fail(msg, msg_len, "fit: needs at least " + std::to_string(p + 1) +
                                  " observations, got " + std::to_string(n));
  if (!features || !times || !coef || !intercept || !adjusted_r2)
    return fail(msg, msg_len, "fit: null argument");
  // Design matrix (row-major n x p) and target.
  std::vector<double> A(static_cast<size_t>(n) * p), b(n), A0, b0;
  for (int i = 0; i < n; ++i) {
    if (!(times[i] > 0.0)) return fail(msg, msg_len, "fit: non-positive observation time");
    gd_cost_features(features + 3 * i, &A[static_cast<size_t>(i) * p]);
    A[static_cast<size_t>(i) * p + kPredictors] = 1.0;
    b[i] = times[i];
  }
  A0 = A;
  b0 = b;
  auto at = [&](int i, int j) -> double& { return A[static_cast<size_t>(i) * p + j]; };

  int perm[kCols];
  for (int j = 0; j < p; ++j) perm[j] = j;
  const double tol = std::numeric_limits<double>::epsilon() * std::min(n, p);
  double r00 = 0.0;
  int rank = p;
  for (int k = 0; k < p; ++k) {
    // Pivot: the remaining column of largest norm below row k.
    int jmax = k;
    double best = -1.0;
    for (int j = k; j < p; ++j) {
      double s = 0.0;
      for (int i = k; i < n; ++i) s += at(i, j) * at(i, j);
      if (s > best) {
        best = s;
        jmax = j;
      }
    }
    if (jmax != k) {
      for (int i = 0; i < n; ++i) std::swap(at(i, k), at(i, jmax));
      std::swap(perm[k], perm[jmax]);
    }
    const double alpha = std::sqrt(best);
    if (k == 0) r00 = alpha;
    if (alpha <= tol * r00 || alpha == 0.0) {
      rank = k;
      break;
    }
    // Householder reflector zeroing column k below the diagonal.
    const double akk = at(k, k);
    const double beta = akk >= 0.0 ? -alpha : alpha;  // new R_kk
    std::vector<double> v(n - k);
    v[0] = akk - beta;
    for (int i = k + 1; i < n; ++i) v[i - k] = at(i, k);
    double vv = 0.0;
    for (double e : v) vv += e * e;
    if (vv > 0.0) {
      for (int j = k + 1; j < p; ++j) {
        double d = 0.0;
        for (int i = k; i < n; ++i) d += v[i - k] * at(i, j);
        const double f = 2.0 * d / vv;
        for (int i = k; i < n; ++i) at(i, j) -= f * v[i - k];
      }
      double d = 0.0;
      for (int i = k; i < n; ++i) d += v[i - k] * b[i];
      const double f = 2.0 * d / vv;
      for (int i = k; i < n; ++i) b[i] -= f * v[i - k];
    }
    at(k, k) = beta;
    for (int i = k + 1; i < n; ++i) at(i, k) = 0.0;
  }
  if (rank < p) {
    std::string names;
    for (int j = rank; j < p; ++j) {
      if (!names.empty()) names += ", ";
      names += kNames[perm[j]];
    }
    return fail(msg, msg_len, "fit: rank-deficient design matrix; collinear columns: " + names);
  }
  // R z = Q^T b, then undo the column permutation.
  double z[kCols];
  for (int k = p - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j < p; ++j) s -= at(k, j) * z[j];
    z[k] = s / at(k, k);
  }
  double sol[kCols];
  for (int j = 0; j < p; ++j) sol[perm[j]] = z[j];
  // Goodness of fit from the residual of the original system (perf_model.hpp:90-101).
  double sse = 0.0, mean = 0.0;
  for (int i = 0; i < n; ++i) mean += b0[i];
  mean /= n;
  double sst = 0.0;
  for (int i = 0; i < n; ++i) {
    double pred = 0.0;
    for (int j = 0; j < p; ++j) pred += A0[static_cast<size_t>(i) * p + j] * sol[j];
    const double r = b0[i] - pred;
    sse += r * r;
    sst += (b0[i] - mean) * (b0[i] - mean);
  }
  const double r2 = sst > 0.0 ? 1.0 - sse / sst : (sse <= 0.0 ? 1.0 : 0.0);
  for (int j = 0; j < kPredictors; ++j) coef[j] = sol[j];
  *intercept = sol[kPredictors];
  *adjusted_r2 = 1.0 - (1.0 - r2) * (n - 1) / static_cast<double>(n - p);
  return GD_OK;
}
