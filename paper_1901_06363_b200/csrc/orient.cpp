// See orient.hpp.
#include "orient.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <numeric>

namespace gdb200 {
namespace {

constexpr double kPi = 3.141592653589793;  // std::numbers::pi

// Out-of-line so the compiler cannot constant-fold the libm call.
__attribute__((noinline)) double libm_cos(double x) { return std::cos(x); }
__attribute__((noinline)) double libm_sin(double x) { return std::sin(x); }

}  // namespace

void trig_of(double angle_deg, double& c, double& s) {
  const double theta = angle_deg * (kPi / 180.0);
  c = libm_cos(theta);
  s = libm_sin(theta);
}

void trig_tables(std::vector<double>& cos_deg, std::vector<double>& sin_deg) {
  cos_deg.resize(360);
  sin_deg.resize(360);
  for (int a = 0; a < 360; ++a) {
    const double theta = static_cast<double>(a) * (kPi / 180.0);
    cos_deg[a] = libm_cos(theta);
    sin_deg[a] = libm_sin(theta);
  }
}

void rigid_orientations(int step, std::vector<int32_t>& index, std::vector<double>& R) {
  index.clear();
  R.clear();
  if (step < 1 || 360 % step != 0) return;
  std::vector<double> c, s;
  trig_tables(c, s);
  const int m = 360 / step;
  const int total = m * m * m;
  std::vector<std::array<double, 9>> mats(total);
  std::vector<std::array<long long, 9>> keys(total);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      for (int k = 0; k < m; ++k) {
        const int idx = (i * m + j) * m + k;
        const double ca = c[i * step], sa = s[i * step];
        const double cb = c[j * step], sb = s[j * step];
        const double cg = c[k * step], sg = s[k * step];
        std::array<double, 9>& r = mats[idx];
        r[0] = cg * cb;
        r[1] = cg * sb * sa - sg * ca;
        r[2] = cg * sb * ca + sg * sa;
        r[3] = sg * cb;
        r[4] = sg * sb * sa + cg * ca;
        r[5] = sg * sb * ca - cg * sa;
        r[6] = -sb;
        r[7] = cb * sa;
        r[8] = cb * ca;
        for (int e = 0; e < 9; ++e) keys[idx][e] = std::llround(r[e] * 1e6);
      }
  std::vector<int32_t> order(total);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return keys[a] != keys[b] ? keys[a] < keys[b] : a < b;
  });
  for (int t = 0; t < total; ++t)
    if (t == 0 || keys[order[t]] != keys[order[t - 1]]) index.push_back(order[t]);
  std::sort(index.begin(), index.end());
  R.reserve(index.size() * 9);
  for (int32_t idx : index) R.insert(R.end(), mats[idx].begin(), mats[idx].end());
}

}  // namespace gdb200
