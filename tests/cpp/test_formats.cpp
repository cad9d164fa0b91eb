// Drop-in formats test: the reference's test_formats.cpp cases (and the
// host-only graph helpers) restated against <geodock_b200/formats.hpp>.
// Nothing here needs a GPU; tests/test_dropin.py builds and runs it in the
// CPU suite.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "geodock_b200/formats.hpp"

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

static bool contains(const std::string& s, const std::string& part) { return s.find(part) != std::string::npos; }

template <class F>
static std::string error_of(F&& fn) {
  try {
    fn();
  } catch (const std::exception& e) {
    return e.what();
  }
  return "";
}

// Random trees with awkward doubles (shortest-decimal stress).
static std::vector<Ligand> random_ligands(int count, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-20.0, 20.0), r(1.2, 1.9);
  std::vector<Ligand> out;
  for (int l = 0; l < count; ++l) {
    const int n = 2 + static_cast<int>(rng() % 30);
    std::vector<Atom> atoms;
    std::vector<Bond> bonds;
    for (int i = 0; i < n; ++i) {
      atoms.push_back({i, {u(rng), u(rng) / 3.0, u(rng) * 1e-7}, r(rng)});
      if (i > 0) bonds.push_back({static_cast<int>(rng() % i), i, (rng() & 1) != 0});
    }
    out.emplace_back("L" + std::to_string(l), std::move(atoms), std::move(bonds));
  }
  return out;
}

int main() {
  run("parse_pocket accepts the documented grammar", [] {
    const Pocket p = parse_pocket("POCKET p1 1\n0 0 1\n");
    CHECK(p.id() == "p1");
    CHECK(p.points().size() == 1 && p.points()[0] == Vec3(0, 0, 1));
    CHECK(parse_pocket("# comment\nPOCKET p2 2\n1 2 3\n# mid\n4 5 6\n").points().size() == 2);
    CHECK(parse_pocket("  POCKET p3 1\r\n\t-1.5  2e-3 7\r\n").points()[0] == Vec3(-1.5, 2e-3, 7));
  });
  run("parse_pocket reports failures with line numbers", [] {
    CHECK(contains(error_of([] { parse_pocket("POCKET p1 2\n0 0 0\n"); }),
                   "expected 2 points, found 1 at line 3"));
    CHECK(contains(error_of([] { parse_pocket("POCKET p1 1\n0 zero 0\n"); }), "at line 2"));
    bool parse_error = false;
    try {
      parse_pocket("");
    } catch (const ParseError& e) {
      parse_error = e.line() == 1;
    }
    CHECK(parse_error);
    CHECK(contains(error_of([] { parse_pocket("BUCKET p1 1\n0 0 0\n"); }), "expected 'POCKET <id> <n>'"));
    CHECK(contains(error_of([] { parse_pocket("POCKET p1 1\n0 0 0\n1 1 1\n"); }), "unexpected content"));
    CHECK(contains(error_of([] { parse_pocket("POCKET p1 0\n"); }), "at least 1 point"));
  });
  run("ligand records parse, skip, and resynchronize", [] {
    const std::string text =
        "LIGAND good 2 1\nATOM 0 0 0 0 1.5\nATOM 1 0 0 1.4 1.5\nBOND 0 1 R\n"
        "LIGAND self 2 1\nATOM 0 0 0 0 1.5\nATOM 1 0 0 1.4 1.5\nBOND 0 0 R\n"
        "LIGAND mangled 2 1\nATOM 0 0 0 0 1.5\nATOM oops\nBOND 0 1 R\n"
        "LIGAND split 3 1\nATOM 0 0 0 0 1.5\nATOM 1 0 0 1.4 1.5\nATOM 2 9 9 9 1.5\nBOND 0 1 F\n"
        "LIGAND tail 2 1\nATOM 0 0 0 0 1.2\nATOM 1 1.4 0 0 1.2\nBOND 1 0 F\n";
    std::istringstream in(text);
    LigandParser parser(in);
    std::vector<std::string> ok, skipped, reasons;
    while (auto rec = parser.next()) {
      if (auto* l = std::get_if<Ligand>(&*rec)) {
        ok.push_back(l->id());
      } else {
        skipped.push_back(std::get<SkippedRecord>(*rec).id);
        reasons.push_back(std::get<SkippedRecord>(*rec).reason);
      }
    }
    CHECK((ok == std::vector<std::string>{"good", "tail"}));
    CHECK((skipped == std::vector<std::string>{"self", "mangled", "split"}));
    CHECK(reasons.size() == 3 && contains(reasons[0], "self-bond") && contains(reasons[1], "ATOM") &&
          contains(reasons[2], "disconnected"));
    CHECK(contains(reasons[1], "at line 11"));
    const auto strict = parse_ligands("LIGAND l 2 1\nATOM 0 0 0 0 1.5\nATOM 1 0 0 1.4 1.5\nBOND 0 1 R\n");
    CHECK(find_rotamers(strict[0]).size() == 1);
    CHECK(contains(error_of([] {
                     parse_ligands("LIGAND bad 2 1\nATOM 0 0 0 0 1\nATOM 1 1 0 0 1\nBOND 0 0 R\n");
                   }),
                   "self-bond"));
  });
  run("ligand parser: bad header, truncated record, resync to the next header", [] {
    std::istringstream in(
        "ATOM 0 0 0 0 1\nLIGAND a 2 1\nATOM 0 0 0 0 1\nATOM 1 1.4 0 0 1\nBOND 0 1 X\nBOND 0 1 R\n"
        "LIGAND b 2 1\nATOM 0 0 0 0 1\nATOM 1 1.4 0 0 1\nBOND 0 1 F\nLIGAND c 3 0\nATOM 0 0 0 0 1\n");
    LigandParser parser(in);
    std::vector<std::string> seen;
    while (auto rec = parser.next()) {
      if (auto* l = std::get_if<Ligand>(&*rec)) seen.push_back("ok:" + l->id());
      else seen.push_back("skip:" + std::get<SkippedRecord>(*rec).id + ":" + std::get<SkippedRecord>(*rec).reason);
    }
    CHECK(seen.size() == 4);
    CHECK(seen[0] == "skip:record@line1:expected 'LIGAND <id> <natoms> <nbonds>' at line 1");
    CHECK(contains(seen[1], "skip:a:expected 'BOND <i> <j> <R|F>' at line 5"));
    CHECK(seen[2] == "ok:b");
    CHECK(contains(seen[3], "skip:c:unexpected end of record in ligand 'c' at line 13"));
  });
  run("pocket and ligand files round-trip bit-exactly", [] {
    std::mt19937_64 rng(20250803);
    std::uniform_real_distribution<double> u(-30.0, 30.0);
    std::vector<Vec3> pts;
    for (int j = 0; j < 500; ++j) pts.push_back({u(rng), u(rng) * 1e-9, u(rng) * 1e9});
    const Pocket pocket("pk", pts);
    const std::string ptext = render_pocket(pocket);
    const Pocket back = parse_pocket(ptext);
    CHECK(back.points() == pocket.points());
    CHECK(render_pocket(back) == ptext);
    const auto ligs = random_ligands(15, 7);
    const std::string ltext = render_ligands(ligs);
    const auto parsed = parse_ligands(ltext);
    CHECK(parsed.size() == ligs.size());
    CHECK(render_ligands(parsed) == ltext);
    for (size_t l = 0; l < ligs.size() && l < parsed.size(); ++l)
      for (int i = 0; i < ligs[l].atom_count(); ++i) {
        CHECK(parsed[l].atoms()[i].position == ligs[l].atoms()[i].position);
        CHECK(parsed[l].atoms()[i].radius == ligs[l].atoms()[i].radius);
      }
  });
  run("screening reports round-trip through CSV plus summary", [] {
    ScreeningReport report;
    report.pocket_id = "P7";
    report.config = {2, 90, 0.3, 2, true};
    report.per_ligand = {{"L000000", 1.25, 481, 0.00325}, {"L000001", 0.07775918000916349, 1081, 0.0123}};
    report.skipped = {{"L000002", "disconnected ligand"}};
    report.total_atoms = 23;
    report.wall_time_seconds = 0.0201;
    report.throughput = 23 / 0.0201;
    report.top1pct_mean = 1.25;
    const std::string csv = render_report_csv(report), summary = render_report_summary(report);
    const ScreeningReport parsed = parse_report(csv, summary);
    CHECK(parsed == report);
    CHECK(render_report_csv(parsed) == csv);
    CHECK(render_report_summary(parsed) == summary);
    CHECK(csv.rfind("ligand_id,score,evaluations,time_seconds\nL000000,1.25,481,0.00325\n", 0) == 0);
    CHECK(contains(summary, "refinement=1\n") && contains(summary, "skipped=L000002: disconnected ligand\n"));
    CHECK(contains(error_of([&] { parse_report("x\n", summary); }), "bad report CSV header"));
    CHECK(contains(error_of([&] { parse_report(csv, "bogus=1\n"); }), "unknown summary key 'bogus'"));
    CHECK(contains(error_of([&] { parse_report(csv, "n_ligands=3\n"); }), "row count"));
  });
  run("format_double renders shortest round-trip decimals", [] {
    for (const double v : {0.1, 1.0 / 3.0, 12345.678901234567, 1e-12, -0.0, 7.0, 5e-324, 1.7976931348623157e308}) {
      const std::string t = format_double(v);
      double back = 1.0;
      std::from_chars(t.data(), t.data() + t.size(), back);
      CHECK(back == v && std::signbit(back) == std::signbit(v));
    }
    CHECK(format_double(0.5) == "0.5");
    CHECK(format_double(2.0) == "2");
  });
  run("find_rotamers / grow_fragments (molecule.hpp:237-301)", [] {
    // 0-1-2-3 chain with a ring 3-4-5-3: bonds 1-2 rotatable bridge, 3-4
    // rotatable but inside the ring (not a rotamer), 0-1 non-rotatable.
    const Ligand l("g", {{0, {0, 0, 0}, 1}, {1, {1, 0, 0}, 1}, {2, {2, 0, 0}, 1}, {3, {3, 0, 0}, 1},
                         {4, {4, 1, 0}, 1}, {5, {4, -1, 0}, 1}},
                   {{2, 1, true}, {0, 1, false}, {2, 3, true}, {3, 4, true}, {4, 5, false}, {5, 3, false}});
    const auto rots = find_rotamers(l);
    CHECK(rots.size() == 2 && rots[0].bond_index == 0 && rots[1].bond_index == 2);
    const auto [left, right] = grow_fragments(l, rots[0]);
    CHECK((left.atom_indices == std::vector<int>{0, 1}));
    CHECK((right.atom_indices == std::vector<int>{2, 3, 4, 5}));
    CHECK(left.axis_atom == 1 && left.anchor_atom == 2 && right.axis_atom == 2 && right.anchor_atom == 1);
    CHECK(left.relative_size == 2.0 / 6.0 && right.side == Side::right);
    CHECK(contains(error_of([&] { grow_fragments(l, Rotamer{{3, 4, true}, 3}); }), "is not a bridge"));
  });
  run("parsers survive random corruption (parse or throw geodock::Error, never crash)", [] {
    const std::string pocket = render_pocket(Pocket("pk", {{0, 0, 0}, {1.5, -2, 3}, {4, 5, 6.25}}));
    const std::string ligs = render_ligands(random_ligands(3, 11));
    ScreeningReport rep;
    rep.pocket_id = "P";
    rep.per_ligand = {{"A", 1.5, 3, 0.25}};
    const std::string csv = render_report_csv(rep), summary = render_report_summary(rep);
    const std::string space = "hp_step = 1, 5\nrepetitions = 1,3\n";
    std::mt19937_64 rng(2024);
    const std::string alphabet = "0123456789 .-+eE\n\t#,=:RFABLIGNDPOCKETXYZ";
    auto mutate = [&](std::string t) {
      const int edits = 1 + static_cast<int>(rng() % 4);
      for (int e = 0; e < edits && !t.empty(); ++e) {
        const size_t at = rng() % t.size();
        switch (rng() % 3) {
          case 0: t[at] = alphabet[rng() % alphabet.size()]; break;
          case 1: t.erase(at, 1 + rng() % 3); break;
          default: t.insert(at, 1, alphabet[rng() % alphabet.size()]); break;
        }
      }
      return t;
    };
    int parsed = 0, rejected = 0;
    for (int k = 0; k < 3000; ++k) {
      try {
        switch (k % 5) {
          case 0: parse_pocket(mutate(pocket)); break;
          case 1: parse_ligands(mutate(ligs)); break;
          case 2: {
            std::istringstream in(mutate(ligs));
            LigandParser parser(in);
            while (parser.next()) {
            }
            break;
          }
          case 3: parse_report(mutate(csv), mutate(summary)); break;
          default: parse_design_space(mutate(space)); break;
        }
        ++parsed;
      } catch (const Error&) {
        ++rejected;
      }
    }
    CHECK(parsed > 0 && rejected > 0 && parsed + rejected == 3000);
  });
  std::printf("%s (%d failed checks)\n", g_failed ? "FAILED" : "OK", g_failed);
  return g_failed ? 1 : 0;
}
