// Drop-in planner test: the reference's test_autotuner.cpp and
// test_perf_model.cpp cases (select_config, scenario_sweep, pareto_front,
// predict, fit) and the planner file formats, restated against
// <geodock_b200/planner.hpp> and <geodock_b200/formats.hpp>.  No GPU
// needed; tests/test_dropin.py runs it in the CPU suite.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "geodock_b200/formats.hpp"
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

static ConfigProfile flat(const KnobConfig& c, double degradation, double per_ligand) {
  ConfigProfile p;
  p.config = c;
  p.mean_degradation = degradation;
  p.perf.config = c;
  p.perf.intercept = per_ligand;
  p.perf.adjusted_r2 = 1.0;
  p.perf.n_observations = 9;
  return p;
}

static const DataFeatures kFeatures{100, 10.0, 3.0, 1000};

int main() {
  run("feature_vector lists the base terms and every interaction", [] {
    CHECK((feature_vector({1, 1, 1, 1}) == std::array<double, 7>{1, 1, 1, 1, 1, 1, 1}));
    CHECK((feature_vector({2, 3, 0, 1}) == std::array<double, 7>{2, 3, 0, 6, 0, 0, 0}));
  });
  run("fit recovers exact coefficients; predict scales with size and workers", [] {
    std::mt19937_64 rng(9);
    std::uniform_real_distribution<double> pp(20, 200), la(5, 40), lr(2, 12);
    const std::array<double, 7> truth{2e-5, 1e-4, 3e-4, 4e-7, 5e-7, 6e-6, 1e-8};
    std::vector<Observation> obs;
    for (int i = 0; i < 40; ++i) {
      const DataFeatures f{static_cast<int>(pp(rng)), la(rng), lr(rng), 1};
      const auto x = feature_vector(f);
      double t = 0.01;
      for (int j = 0; j < 7; ++j) t += truth[j] * x[j];
      obs.push_back({f, t});
    }
    const PerfModel m = fit(KnobConfig{}, obs);
    for (int j = 0; j < 7; ++j) CHECK(std::abs(m.coefficients[j] - truth[j]) <= 1e-6 * std::abs(truth[j]));
    CHECK(std::abs(m.intercept - 0.01) <= 1e-8 && m.adjusted_r2 > 0.999999 && m.n_observations == 40);
    PerfModel flat_model;
    flat_model.intercept = 2.0;
    CHECK(predict(flat_model, {10, 10, 3, 10}, 1).seconds == 20.0);
    CHECK(predict(flat_model, {10, 10, 3, 10}, 10).seconds == 2.0);
    flat_model.intercept = -1.0;
    CHECK(predict(flat_model, {10, 10, 3, 10}, 1).clamped);
    bool threw = false;
    try {
      fit(KnobConfig{}, std::vector<Observation>(obs.begin(), obs.begin() + 8));
    } catch (const Error& e) {
      threw = std::string(e.what()).find("at least 9") != std::string::npos;
    }
    CHECK(threw);
  });
  run("select_config: budget, accuracy, completion, ties, workers", [] {
    std::vector<ConfigProfile> kb{flat({1, 45, 0.0, 3, false}, 0.0, 0.1), flat({5, 45, 0.0, 1, false}, 8.0, 0.01)};
    Plan p = select_config(kb, kFeatures, 50.0, 1);
    CHECK(p.chosen == kb[1].config && p.expected_completion_pct == 100.0 && p.expected_degradation_pct == 8.0);
    CHECK(select_config(kb, kFeatures, 1000.0, 1).chosen == kb[0].config);
    kb = {flat({1, 45, 0.0, 3, false}, 0.0, 0.1), flat({5, 45, 0.0, 1, false}, 8.0, 0.05)};
    p = select_config(kb, kFeatures, 25.0, 1);
    CHECK(p.chosen == kb[1].config && p.expected_completion_pct == 50.0);
    kb = {flat({1, 45, 0.0, 3, false}, 2.0, 0.02), flat({2, 45, 0.0, 3, false}, 2.0, 0.01)};
    CHECK(select_config(kb, kFeatures, 100.0, 1).chosen == kb[1].config);
    kb = {flat({2, 90, 0.0, 3, false}, 2.0, 0.01), flat({2, 45, 0.0, 3, false}, 2.0, 0.01)};
    CHECK(select_config(kb, kFeatures, 100.0, 1).chosen == kb[1].config);
    kb = {flat({1, 45, 0.0, 3, false}, 0.0, 0.1)};
    CHECK(select_config(kb, kFeatures, 30.0, 1).expected_completion_pct == 30.0);
    CHECK(select_config(kb, kFeatures, 30.0, 4).expected_completion_pct == 100.0);
    bool threw = false;
    try {
      select_config({}, kFeatures, 1.0, 1);
    } catch (const Error&) {
      threw = true;
    }
    CHECK(threw);
  });
  run("scenario_sweep over budgets and database sizes", [] {
    const std::vector<ConfigProfile> kb{flat({1, 45, 0.0, 3, false}, 0.0, 0.1),
                                        flat({2, 45, 0.0, 3, false}, 1.5, 0.05),
                                        flat({3, 45, 0.0, 2, false}, 3.0, 0.02),
                                        flat({5, 90, 0.6, 1, true}, 9.0, 0.004)};
    std::vector<double> budgets;
    for (double b = 1.0; b <= 150.0; b *= 1.5) budgets.push_back(b);
    const auto rows = scenario_sweep(kb, kFeatures, 1, SweepVariable::budget, budgets, 1000);
    CHECK(rows.size() == budgets.size());
    for (size_t i = 1; i < rows.size(); ++i)
      CHECK(rows[i].plan.expected_degradation_pct <= rows[i - 1].plan.expected_degradation_pct);
    CHECK(rows.back().plan.chosen == kb[0].config);
    const std::vector<ConfigProfile> two{kb[0], flat({5, 90, 0.6, 1, true}, 9.0, 0.001)};
    const auto by_size = scenario_sweep(two, kFeatures, 1, SweepVariable::database_size,
                                        {100, 1000, 10000, 100000}, 50.0);
    CHECK(by_size[0].plan.chosen == two[0].config && by_size[3].plan.chosen == two[1].config);
    const std::string csv = render_sweep_csv(by_size);
    CHECK(csv.rfind("swept_value,completion_pct,degradation_pct,hp_step,lp_step,threshold,repetitions,"
                    "refinement\n100,100,0,1,45,0,3,0\n", 0) == 0);
  });
  run("pareto_front keeps exactly the non-dominated points", [] {
    const auto f = pareto_front({{100, 0.0}, {200, 1.0}, {150, 2.0}, {300, 5.0}, {250, 8.0}, {300, 4.0}});
    CHECK((f == std::vector<std::size_t>{5, 1, 0}));
  });
  run("knowledge bases round-trip bit-exactly; design spaces expand full factorial", [] {
    std::vector<ConfigProfile> kb{flat({1, 45, 0.0, 3, false}, 0.0, 0.1), flat({5, 90, 0.6, 1, true}, 9.25, 1.0 / 3.0)};
    kb[1].perf.coefficients = {1e-7, -2.5e-3, 1.0 / 7.0, 0.0, 3e-12, -0.0, 12345.678901234567};
    kb[1].perf.adjusted_r2 = 0.98765432101234567;
    const std::string text = render_knowledge_base(kb);
    const auto back = parse_knowledge_base(text);
    CHECK(back == kb);
    CHECK(render_knowledge_base(back) == text);
    CHECK(text.rfind("# geodock knowledge base\n# hp_step,lp_step,", 0) == 0);
    const auto space = parse_design_space("# sweep\nhp_step = 1, 5\nrepetitions=1,3\nrefinement = 0,1\n");
    CHECK(space.size() == 8);
    CHECK(space[0] == (KnobConfig{1, 1, 0.0, 1, false}) && space[7] == (KnobConfig{5, 5, 0.0, 3, true}));
    const auto lp = parse_design_space("hp_step = 10\nlp_step = 45, 90\nthreshold = 0.2\n");
    CHECK(lp.size() == 2 && lp[1] == (KnobConfig{10, 90, 0.2, 3, false}));
    std::string err;
    try {
      parse_design_space("hp_step = 7\n");  // 7 does not divide 360
    } catch (const Error& e) {
      err = e.what();
    }
    CHECK(!err.empty());
    try {
      parse_design_space("speed = 3\n");
    } catch (const Error& e) {
      err = e.what();
    }
    CHECK(err.find("unknown knob 'speed' at line 1") != std::string::npos);
  });
  std::printf("%s (%d failed checks)\n", g_failed ? "FAILED" : "OK", g_failed);
  return g_failed ? 1 : 0;
}
