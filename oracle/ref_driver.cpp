// Test-infrastructure driver over the REFERENCE stripefrac library (built from
// /root/reference/proj/src by oracle/Makefile). Two jobs:
//   golden <outdir>   write golden vectors (tests/golden/*.json) from the
//                     reference's own compute_unifrac / Embedder / condense;
//   bench ...         time the reference CPU hot path on a bounded sample
//                     (bench.py --impl reference, cpu_baseline kind "reference");
//   instance ...      digest of a random_instance (pins our generator);
//   dm ...            full-range reference run on a synthetic instance.
// Never linked into, or called by, the product path.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "stripefrac/kernels.hpp"
#include "stripefrac/synth.hpp"
#include "stripefrac/validate.hpp"

using namespace stripefrac;

namespace {

std::string num(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

template <class M>
std::string arr(const M& m) {
  std::string out = "[";
  for (Eigen::Index i = 0; i < m.size(); ++i) {
    if (i) out += ",";
    out += num(static_cast<double>(m.data()[i]));
  }
  return out + "]";
}

std::string quote(const std::string& s) {
  std::string out = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') out.push_back('\\');
    if (c == '\n') {
      out += "\\n";
      continue;
    }
    if (c == '\t') {
      out += "\\t";
      continue;
    }
    out.push_back(c);
  }
  return out + "\"";
}

// sparse triplet serialisation with a pinned sample order; %.17g round-trips
std::string table_text(const SampleTable& t) {
  std::string out = "#samples";
  for (const auto& s : t.sample_ids) out += "\t" + s;
  out += "\n";
  for (int f = 0; f < t.n_features(); ++f)
    for (const auto& [s, c] : t.entries[static_cast<std::size_t>(f)])
      out += t.feature_ids[static_cast<std::size_t>(f)] + "\t" +
             t.sample_ids[static_cast<std::size_t>(s)] + "\t" + num(c) + "\n";
  return out;
}

const Metric kMetrics[] = {Metric::Unweighted, Metric::WeightedUnnormalized,
                           Metric::WeightedNormalized};

KernelConfig cfg_of(Metric m, Precision p) {
  KernelConfig c;
  c.metric = m;
  c.precision = p;
  return c;
}

template <class Real>
std::string stripes_json(const PhyloTree& tree, const SampleTable& table, Metric m,
                         int start, int stop) {
  KernelCounters counters;
  const Precision p = std::is_same_v<Real, float> ? Precision::Fp32 : Precision::Fp64;
  auto set = compute_unifrac<Real>(tree, table, cfg_of(m, p), start, stop, 1, &counters);
  std::string out = "{\"metric\":" + quote(std::string(name(m))) + ",\"precision\":" +
                    quote(std::string(name(p))) + ",\"start\":" + std::to_string(set.start) +
                    ",\"stop\":" + std::to_string(set.stop) +
                    ",\"distances\":" + arr(set.distances);
  out += ",\"totals\":" + (set.has_totals() ? arr(set.totals) : std::string("[]"));
  out += ",\"counters\":[" + std::to_string(counters.accumulator_writes) + "," +
         std::to_string(counters.embedding_reads) + "," +
         std::to_string(counters.kernel_passes) + "]}";
  return out;
}

// Raw (pre-finalize) totals are not observable through compute_unifrac (it
// finalizes in place; totals stay raw). distances are finalized.
std::string case_json(const std::string& case_name, const PhyloTree& tree,
                      const SampleTable& table, const std::string& params,
                      bool with_embedding, bool with_fp32,
                      const std::vector<std::pair<int, int>>& ranges = {}) {
  std::string out = "{\"name\":" + quote(case_name) + ",\"params\":" + params;
  out += ",\"newick\":" + quote(to_newick(tree));
  out += ",\"table\":" + quote(table_text(table));
  out += ",\"sample_ids\":[";
  for (int i = 0; i < table.n_samples(); ++i)
    out += (i ? "," : "") + quote(table.sample_ids[static_cast<std::size_t>(i)]);
  out += "],\"feature_ids\":[";
  for (int f = 0; f < table.n_features(); ++f)
    out += (f ? "," : "") + quote(table.feature_ids[static_cast<std::size_t>(f)]);
  out += "]";
  const std::string nwk = to_newick(tree);
  const std::string tbl = table_text(table);
  out += ",\"newick_fnv\":" + quote(hex64(fnv1a64(nwk.data(), nwk.size())));
  out += ",\"table_fnv\":" + quote(hex64(fnv1a64(tbl.data(), tbl.size())));
  out += ",\"sample_totals\":[";
  for (int i = 0; i < table.n_samples(); ++i)
    out += (i ? "," : "") + num(table.sample_totals[static_cast<std::size_t>(i)]);
  out += "]";

  // sheared postorder rows: parent row, length, leaf feature
  const PhyloTree sh = sheared_to_table(tree, table);
  std::vector<int> row_of(static_cast<std::size_t>(sh.n_nodes()), -1);
  for (std::size_t r = 0; r < sh.postorder.size(); ++r) row_of[static_cast<std::size_t>(sh.postorder[r])] = static_cast<int>(r);
  std::string parents = "[", lens = "[", names = "[";
  for (std::size_t r = 0; r < sh.postorder.size(); ++r) {
    const int v = sh.postorder[r];
    const int par = sh.nodes[static_cast<std::size_t>(v)].parent;
    parents += (r ? "," : "") + std::to_string(par == sh.root ? -1 : row_of[static_cast<std::size_t>(par)]);
    lens += (r ? "," : "") + num(sh.nodes[static_cast<std::size_t>(v)].length);
    names += (r ? "," : "") + quote(sh.is_leaf(v) ? sh.nodes[static_cast<std::size_t>(v)].name : std::string());
  }
  out += ",\"rows\":{\"parent\":" + parents + "],\"length\":" + lens + "],\"leaf_name\":" + names + "]}";

  if (with_embedding) {
    for (EmbedMode mode : {EmbedMode::Unweighted, EmbedMode::Weighted}) {
      Embedder em(sh, table, mode, 1);
      std::string rows = "[";
      bool first = true;
      while (auto b = em.next_batch(1 << 20)) {
        for (int r = 0; r < b->filled; ++r) {
          if (!first) rows += ",";
          first = false;
          rows += arr(RowMatrix<double>(b->emb.row(r)));
        }
      }
      out += std::string(",\"embedding_") + (mode == EmbedMode::Weighted ? "weighted" : "unweighted") +
             "\":" + rows + "]";
    }
  }

  out += ",\"results\":[";
  bool first = true;
  const int S = total_stripes(table.n_samples());
  for (Metric m : kMetrics) {
    if (!first) out += ",";
    first = false;
    out += stripes_json<double>(tree, table, m, 0, S);
    if (with_fp32) out += "," + stripes_json<float>(tree, table, m, 0, S);
    for (auto [a, b] : ranges) out += "," + stripes_json<double>(tree, table, m, a, b);
  }
  out += "]";

  // the full condensed matrix (fp64) for the first metric set, plus
  // brute-force oracle values for cross-checking
  out += ",\"brute_force\":[";
  first = true;
  for (Metric m : kMetrics) {
    if (table.n_samples() > 64) break;  // keep the fixtures small
    if (!first) out += ",";
    first = false;
    out += arr(brute_force_unifrac(tree, table, m).values);
  }
  out += "]}";
  return out;
}

SampleTable dense_table(const std::vector<std::string>& samples,
                        const std::vector<std::string>& features,
                        const std::vector<double>& counts) {
  RowMatrix<double> m(static_cast<Eigen::Index>(features.size()),
                      static_cast<Eigen::Index>(samples.size()));
  for (std::size_t i = 0; i < counts.size(); ++i) m.data()[i] = counts[i];
  return make_table(samples, features, m);
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw Error("cannot open " + path);
  out << text;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error("cannot open " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

int cmd_golden(const std::string& dir, const std::string& demo_dir) {
  // C1: the bundled demo data (dense TSV), all metrics, both precisions,
  // and three partitions of its 4 stripes.
  {
    const PhyloTree tree = parse_newick_file(demo_dir + "/demo_tree.nwk");
    const SampleTable table = load_table_file(demo_dir + "/demo_table.tsv", TableFormat::TsvDense);
    std::string j = case_json("demo", tree, table, "{\"kind\":\"demo\"}", true, true,
                              {{0, 1}, {1, 3}, {3, 4}});
    // full condensed matrices through compute_distance_matrix + TSV bytes
    j.pop_back();
    j += ",\"dm\":[";
    bool first = true;
    for (Metric m : kMetrics)
      for (Precision p : {Precision::Fp64, Precision::Fp32}) {
        if (!first) j += ",";
        first = false;
        const auto dm = p == Precision::Fp64
                            ? compute_distance_matrix<double>(tree, table, cfg_of(m, p))
                            : compute_distance_matrix<float>(tree, table, cfg_of(m, p));
        j += "{\"metric\":" + quote(std::string(name(m))) + ",\"precision\":" +
             quote(std::string(name(p))) + ",\"values\":" + arr(dm.values) +
             ",\"tsv\":" + quote(to_tsv(dm)) + "}";
      }
    // demo WN fp64 vs fp32 Mantel, 999 permutations, seed 7 (README.md:119-126)
    {
      const auto d64 = compute_distance_matrix<double>(tree, table, cfg_of(Metric::WeightedNormalized, Precision::Fp64));
      const auto d32 = compute_distance_matrix<float>(tree, table, cfg_of(Metric::WeightedNormalized, Precision::Fp32));
      const auto r = mantel(d64, d32, 999, 7);
      j += "],\"mantel_wn_fp64_fp32\":{\"r\":" + num(r.r) + ",\"r_squared\":" + num(r.r_squared) +
           ",\"p_value\":" + num(r.p_value) + "}}";
    }
    write_file(dir + "/demo.json", j);
  }

  // hand-worked trees (test_kernels.cpp:49-78, test_embed.cpp:14-80)
  {
    std::string j = "[";
    j += case_json("two_leaf", parse_newick("(A:1,B:1);"),
                   dense_table({"s1", "s2"}, {"A", "B"}, {4, 0, 0, 4}), "{\"kind\":\"hand\"}",
                   true, true);
    j += "," + case_json("three_leaf", parse_newick("((A:1,B:1):1,C:1);"),
                         dense_table({"s1", "s2"}, {"A", "B", "C"}, {1, 0, 0, 1, 0, 0}),
                         "{\"kind\":\"hand\"}", true, true);
    j += "," + case_json("embed_demo", parse_newick("((A:1,B:2)ab:0.5,C:3);"),
                         dense_table({"s1", "s2", "s3"}, {"A", "B", "C"},
                                     {4, 0, 1, 0, 2, 1, 4, 2, 2}),
                         "{\"kind\":\"hand\"}", true, true);
    // a multifurcating tree with a leaf subset (exercise shear + child order)
    j += "," + case_json("multifurcating_subset",
                         parse_newick("((A:0.5,B:0.25,(C:1,D:0.125)cd:0.75)abcd:0.3,(E:2,(F:0.1,G:0.2):0.4)efg:0.6,H:1.5);"),
                         dense_table({"s1", "s2", "s3", "s4", "s5"}, {"A", "C", "D", "F", "H"},
                                     {1, 0, 3, 0, 2, 0, 5, 0, 1, 1, 2, 2, 0, 0, 7, 0, 0, 4, 4, 0, 9, 0, 0, 1, 1}),
                         "{\"kind\":\"hand\"}", true, true);
    write_file(dir + "/hand.json", j + "]");
  }

  // 30 seeded instances as in test_kernels.cpp:80-99 (n in [2,32], F in [2,64],
  // every 3rd on a leaf subset), density 0.35
  {
    std::string j = "[";
    for (int i = 0; i < 30; ++i) {
      std::mt19937_64 rng(500 + static_cast<std::uint64_t>(i));
      std::uniform_int_distribution<int> ns(2, 32), nf(2, 64);
      const int n = ns(rng), f = nf(rng);
      const int subset = (i % 3 == 0 && f > 3) ? (2 * f) / 3 : 0;
      const SynthInstance inst = random_instance(500 + static_cast<std::uint64_t>(i), n, f, 0.35, subset);
      char params[160];
      std::snprintf(params, sizeof(params),
                    "{\"kind\":\"instance\",\"seed\":%d,\"n\":%d,\"leaves\":%d,\"density\":0.35,\"subset\":%d}",
                    500 + i, n, f, subset);
      if (i) j += ",";
      j += case_json("seed" + std::to_string(500 + i), inst.tree, inst.table, params, i < 6, i % 2 == 0);
    }
    write_file(dir + "/instances_small.json", j + "]");
  }

  // partition independence (test_kernels.cpp:154-170) and medium instances
  {
    std::string j = "[";
    {
      const SynthInstance inst = random_instance(1234, 17, 40, 0.4);
      j += case_json("seed1234", inst.tree, inst.table,
                     "{\"kind\":\"instance\",\"seed\":1234,\"n\":17,\"leaves\":40,\"density\":0.4,\"subset\":0}",
                     false, false, {{0, 1}, {1, 2}, {2, 5}, {5, 8}, {0, 4}, {4, 8}});
    }
    {
      const SynthInstance inst = random_instance(4242, 64, 200, 0.35);
      j += "," + case_json("seed4242", inst.tree, inst.table,
                           "{\"kind\":\"instance\",\"seed\":4242,\"n\":64,\"leaves\":200,\"density\":0.35,\"subset\":0}",
                           false, true, {{0, 16}, {16, 32}, {3, 29}});
    }
    {
      const SynthInstance inst = random_instance(4243, 97, 300, 0.05, 250);
      j += "," + case_json("seed4243", inst.tree, inst.table,
                           "{\"kind\":\"instance\",\"seed\":4243,\"n\":97,\"leaves\":300,\"density\":0.05,\"subset\":250}",
                           false, true, {{5, 48}});
    }
    {
      const SynthInstance inst = random_instance(4244, 160, 400, 0.02);
      j += "," + case_json("seed4244", inst.tree, inst.table,
                           "{\"kind\":\"instance\",\"seed\":4244,\"n\":160,\"leaves\":400,\"density\":0.02,\"subset\":0}",
                           false, true, {{0, 33}, {33, 80}});
    }
    write_file(dir + "/instances_medium.json", j + "]");
  }
  return 0;
}

// Wide branch-length goldens (tests/golden/instances_wide.json): the
// reference's results on trees whose lengths span many binades, so the
// GPU path's exact fixed-point levels are exercised where one 63-bit grid
// would round short branches. Three families:
//  * random_instance trees with every length redrawn log-uniformly in
//    [10^lo, 2] (deterministic mt19937_64 stream per seed);
//  * "twin" samples: cherries with tiny twigs (1e-12 .. 1e-9) under normal
//    internal branches; sample pairs pick the same cherries and differ only
//    in which twig, so their distance is carried by branches <= 1e-9 alone;
//  * a tree whose lengths need several fixed-point levels (1e-300 .. 1e3).
std::string fmt_len(double v) { return num(v); }

int cmd_wide_golden(const std::string& dir) {
  std::string j = "[";
  bool first_case = true;
  auto add = [&](const std::string& name, const PhyloTree& tree, const SampleTable& table, const std::string& params,
                 std::vector<std::pair<int, int>> ranges) {
    if (!first_case) j += ",";
    first_case = false;
    j += case_json(name, tree, table, params, false, true, ranges);
  };
  // (1) log-uniform lengths on random_instance trees
  struct W { std::uint64_t seed; int n, leaves; double dens; double lo; };
  const W ws[] = {{7001, 40, 120, 0.2, -12.0}, {7002, 33, 200, 0.05, -15.0}, {7003, 64, 300, 0.1, -9.0}};
  for (const W& w : ws) {
    SynthInstance inst = random_instance(w.seed, w.n, w.leaves, w.dens);
    std::mt19937_64 rng(w.seed * 7919);
    std::uniform_real_distribution<double> u(w.lo, std::log10(2.0));
    for (auto& nd : inst.tree.nodes) nd.length = std::pow(10.0, u(rng));
    const PhyloTree tree = parse_newick(to_newick(inst.tree));
    char params[200];
    std::snprintf(params, sizeof(params),
                  "{\"kind\":\"wide\",\"seed\":%llu,\"n\":%d,\"leaves\":%d,\"density\":%g,\"log10_min\":%g}",
                  static_cast<unsigned long long>(w.seed), w.n, w.leaves, w.dens, w.lo);
    add("wide" + std::to_string(w.seed), tree, inst.table, params, {{0, 3}, {w.n / 4, w.n / 2}});
  }
  // (2) twins: distance carried only by twigs <= 1e-9
  for (std::uint64_t seed : {7101ull, 7102ull}) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> tw(-12.0, -9.0), nl(0.01, 2.0), coin(0.0, 1.0);
    const int m = seed == 7101 ? 24 : 41;  // cherries
    const int pairs = seed == 7101 ? 10 : 17;
    std::vector<std::string> sub;
    for (int i = 0; i < m; ++i) {
      char buf[160];
      std::snprintf(buf, sizeof(buf), "(T%da:%s,T%db:%s)c%d:%s", i, fmt_len(std::pow(10.0, tw(rng))).c_str(), i,
                    fmt_len(std::pow(10.0, tw(rng))).c_str(), i, fmt_len(nl(rng)).c_str());
      sub.push_back(buf);
    }
    int inner = 0;
    while (sub.size() > 1) {  // random joins
      std::uniform_int_distribution<std::size_t> pick(0, sub.size() - 1);
      const std::size_t a = pick(rng);
      std::string A = sub[a];
      sub.erase(sub.begin() + static_cast<std::ptrdiff_t>(a));
      std::uniform_int_distribution<std::size_t> pick2(0, sub.size() - 1);
      const std::size_t b = pick2(rng);
      std::string B = sub[b];
      sub.erase(sub.begin() + static_cast<std::ptrdiff_t>(b));
      sub.push_back("(" + A + "," + B + ")i" + std::to_string(inner++) + ":" + fmt_len(nl(rng)));
    }
    const PhyloTree tree = parse_newick(sub[0] + ";");
    std::vector<std::string> samples, features;
    for (int s = 0; s < 2 * pairs; ++s) samples.push_back("s" + std::to_string(s));
    for (int i = 0; i < m; ++i) {
      features.push_back("T" + std::to_string(i) + "a");
      features.push_back("T" + std::to_string(i) + "b");
    }
    std::vector<double> counts(static_cast<std::size_t>(2 * m) * static_cast<std::size_t>(2 * pairs), 0.0);
    auto at = [&](int f, int s) -> double& { return counts[static_cast<std::size_t>(f) * (2 * pairs) + s]; };
    for (int p = 0; p < pairs; ++p) {
      int flips = 0;
      for (int i = 0; i < m; ++i) {
        if (coin(rng) > 0.4) continue;
        const int side = coin(rng) < 0.5 ? 0 : 1;
        const bool flip = flips < 1 + p % 3 && coin(rng) < 0.3;
        flips += flip ? 1 : 0;
        at(2 * i + side, 2 * p) = 1.0 + std::floor(coin(rng) * 20.0);
        at(2 * i + (flip ? 1 - side : side), 2 * p + 1) = 1.0 + std::floor(coin(rng) * 20.0);
      }
      at(0, 2 * p) += 1.0;  // every sample nonempty
      at(0, 2 * p + 1) += 1.0;
    }
    char params[120];
    std::snprintf(params, sizeof(params), "{\"kind\":\"twins\",\"seed\":%llu,\"cherries\":%d,\"pairs\":%d}",
                  static_cast<unsigned long long>(seed), m, pairs);
    add("twins" + std::to_string(seed), tree, dense_table(samples, features, counts), params, {{1, pairs}});
  }
  // (3) lengths needing several fixed-point levels
  {
    SynthInstance inst = random_instance(7201, 21, 60, 0.3);
    std::mt19937_64 rng(7201);
    std::uniform_real_distribution<double> u(-300.0, 3.0);
    for (auto& nd : inst.tree.nodes) nd.length = std::pow(10.0, u(rng));
    const PhyloTree tree = parse_newick(to_newick(inst.tree));
    add("levels7201", tree, inst.table, "{\"kind\":\"wide\",\"seed\":7201,\"n\":21,\"leaves\":60,\"density\":0.3,\"log10_min\":-300}",
        {{2, 7}});
  }
  write_file(dir + "/instances_wide.json", j + "]");
  return 0;
}

// Mantel golden vectors (validate.cpp:111-159): reference DMs of seeded
// instances, r / r^2 / p for several seeds and permutation counts, and the
// first permutations of a seed (the stream the GPU path must reproduce).
std::uint64_t mix64(std::uint64_t x) {  // validate.cpp:101-106 (file-local there)
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

int cmd_mantel_golden(const std::string& dir) {
  std::string j = "{\"cases\":[";
  struct C { std::uint64_t seed; int n, leaves; double dens; };
  const C cases[] = {{71, 40, 120, 0.1}, {72, 97, 300, 0.05}, {73, 160, 500, 0.02}};
  bool first = true;
  for (const C& c : cases) {
    const SynthInstance inst = random_instance(c.seed, c.n, c.leaves, c.dens);
    const auto uw = compute_distance_matrix<double>(inst.tree, inst.table, cfg_of(Metric::Unweighted, Precision::Fp64));
    const auto wn = compute_distance_matrix<double>(inst.tree, inst.table, cfg_of(Metric::WeightedNormalized, Precision::Fp64));
    const auto wn32 = compute_distance_matrix<float>(inst.tree, inst.table, cfg_of(Metric::WeightedNormalized, Precision::Fp32));
    // an independent instance of the same size: r near 0, p-values in the bulk
    const SynthInstance other = random_instance(c.seed + 100, c.n, c.leaves, c.dens);
    auto wn_other = compute_distance_matrix<double>(other.tree, other.table, cfg_of(Metric::WeightedNormalized, Precision::Fp64));
    wn_other.sample_ids = wn.sample_ids;  // same labels: mantel compares by position
    char params[160];
    std::snprintf(params, sizeof(params), "\"seed\":%llu,\"n\":%d,\"leaves\":%d,\"density\":%g",
                  static_cast<unsigned long long>(c.seed), c.n, c.leaves, c.dens);
    struct R { const char* a; const char* b; const DistanceMatrix* x; const DistanceMatrix* y; int perms; std::uint64_t ms; };
    const R runs[] = {{"unweighted-fp64", "weighted-normalized-fp64", &uw, &wn, 199, 3},
                      {"unweighted-fp64", "weighted-normalized-fp64", &uw, &wn, 999, 17},
                      {"weighted-normalized-fp64", "weighted-normalized-fp32", &wn, &wn32, 99, 11},
                      {"unweighted-fp64", "weighted-normalized-fp64-other", &uw, &wn_other, 999, 5},
                      {"unweighted-fp64", "weighted-normalized-fp64-other", &uw, &wn_other, 499, 6}};
    for (const R& r : runs) {
      const auto res = mantel(*r.x, *r.y, r.perms, r.ms);
      if (!first) j += ",";
      first = false;
      j += std::string("{") + params + ",\"x\":" + quote(r.a) + ",\"y\":" + quote(r.b) +
           ",\"permutations\":" + std::to_string(r.perms) + ",\"mantel_seed\":" + std::to_string(r.ms) +
           ",\"r\":" + num(res.r) + ",\"r_squared\":" + num(res.r_squared) + ",\"p_value\":" +
           num(res.p_value) + "}";
    }
  }
  j += "],\"permutations\":[";
  first = true;
  for (int n : {2, 7, 50})
    for (std::uint64_t seed : {0ull, 7ull, 123456789ull})
      for (int p = 0; p < 3; ++p) {
        std::vector<int> perm(static_cast<std::size_t>(n));
        std::mt19937_64 rng(mix64(seed ^ mix64(static_cast<std::uint64_t>(p) + 1)));
        std::iota(perm.begin(), perm.end(), 0);
        std::shuffle(perm.begin(), perm.end(), rng);
        if (!first) j += ",";
        first = false;
        j += "{\"n\":" + std::to_string(n) + ",\"seed\":" + std::to_string(seed) + ",\"p\":" +
             std::to_string(p) + ",\"perm\":[";
        for (int i = 0; i < n; ++i) j += (i ? "," : "") + std::to_string(perm[static_cast<std::size_t>(i)]);
        j += "]}";
      }
  write_file(dir + "/mantel.json", j + "]}");
  return 0;
}

// .strf files written by the reference itself (stripes.cpp:179-201) for the
// demo data: byte-level fixtures for the device-streamed writer.
int cmd_strf_golden(const std::string& dir, const std::string& demo_dir) {
  const PhyloTree tree = parse_newick_file(demo_dir + "/demo_tree.nwk");
  const SampleTable table = load_table_file(demo_dir + "/demo_table.tsv", TableFormat::TsvDense);
  write_stripe_file(dir + "/demo_wn_fp64_0_4.strf",
                    compute_unifrac<double>(tree, table, cfg_of(Metric::WeightedNormalized, Precision::Fp64), 0, 4));
  write_stripe_file(dir + "/demo_uw_fp32_1_3.strf",
                    compute_unifrac<float>(tree, table, cfg_of(Metric::Unweighted, Precision::Fp32), 1, 3));
  write_stripe_file(dir + "/demo_wu_fp64_0_4.strf",
                    compute_unifrac<double>(tree, table, cfg_of(Metric::WeightedUnnormalized, Precision::Fp64), 0, 4));
  return 0;
}

// digest of a random_instance, to pin the port of the generator at scale
int cmd_instance(std::uint64_t seed, int n, int leaves, double density, int subset) {
  const auto t0 = std::chrono::steady_clock::now();
  const SynthInstance inst = random_instance(seed, n, leaves, density, subset);
  const double gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const std::string nwk = to_newick(inst.tree);
  std::uint64_t h = 0xcbf29ce484222325ull, nnz = 0;
  for (int f = 0; f < inst.table.n_features(); ++f)
    for (const auto& [s, c] : inst.table.entries[static_cast<std::size_t>(f)]) {
      h = fnv1a64(&f, sizeof(f), h);
      h = fnv1a64(&s, sizeof(s), h);
      h = fnv1a64(&c, sizeof(c), h);
      ++nnz;
    }
  std::printf("{\"newick_fnv\":\"%s\",\"table_fnv\":\"%s\",\"nnz\":%" PRIu64 ",\"gen_s\":%.3f}\n",
              hex64(fnv1a64(nwk.data(), nwk.size())).c_str(), hex64(h).c_str(), nnz, gen_s);
  return 0;
}

// Reference CPU hot path on a bounded sample of a synthetic workload: build
// the instance and the reference Embedder once, then each repetition takes
// the next embedding batch (B rows, postorder) and runs the reference's
// accumulate_stripes over stripes [0, n_stripes) fanned out over `threads`
// std::threads exactly as compute_unifrac does (kernels.hpp:289-310).
int cmd_bench(std::uint64_t seed, int n, int leaves, double density, int subset, Metric m,
              Precision p, int n_stripes, int reps, int threads, int batch) {
  const auto t0 = std::chrono::steady_clock::now();
  const SynthInstance inst = random_instance(seed, n, leaves, density, subset);
  const PhyloTree sh = sheared_to_table(inst.tree, inst.table);
  KernelConfig cfg = cfg_of(m, p);
  cfg.batch_capacity = batch;
  Embedder em(sh, inst.table, embed_mode(m), cfg.resolved_step_size());
  const double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const int S = total_stripes(n);
  if (n_stripes > S) n_stripes = S;

  auto run = [&](auto tag) {
    using Real = decltype(tag);
    auto set = allocate_stripes<Real>(n, 0, n_stripes, m);
    std::vector<double> secs;
    std::uint64_t updates = 0;
    for (int r = 0; r < reps; ++r) {
      // timed: the reference's per-batch work, Embedder::next_batch +
      // cast_batch + accumulate_stripes over the worker split
      const auto t1 = std::chrono::steady_clock::now();
      auto b64 = em.next_batch(cfg.batch_capacity);
      if (!b64) break;
      const EmbeddingBatch<Real> b = cast_batch<Real>(*b64);
      const int workers = std::min(threads, set.n_stripes());
      std::vector<KernelCounters> partial(static_cast<std::size_t>(workers));
      std::vector<std::thread> pool;
      for (int w = 0; w < workers; ++w) {
        const int a = static_cast<int>(static_cast<std::int64_t>(n_stripes) * w / workers);
        const int bb = static_cast<int>(static_cast<std::int64_t>(n_stripes) * (w + 1) / workers);
        pool.emplace_back([&, a, bb, w] {
          detail::accumulate_stripes(set, b, cfg, partial[static_cast<std::size_t>(w)], a, bb);
        });
      }
      for (auto& t : pool) t.join();
      secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count());
      updates = static_cast<std::uint64_t>(b.filled) * static_cast<std::uint64_t>(n_stripes) *
                static_cast<std::uint64_t>(n);
    }
    std::printf("{\"setup_s\":%.3f,\"updates_per_rep\":%" PRIu64 ",\"threads\":%d,\"seconds\":[",
                setup_s, updates, threads);
    for (std::size_t i = 0; i < secs.size(); ++i) std::printf("%s%.6f", i ? "," : "", secs[i]);
    std::printf("]}\n");
  };
  if (p == Precision::Fp64)
    run(double{});
  else
    run(float{});
  return 0;
}

// full reference run on a synthetic instance (timed), raw stripes to a file
int cmd_dm(std::uint64_t seed, int n, int leaves, double density, int subset, Metric m,
           Precision p, int start, int stop, int threads, const std::string& out_path) {
  const SynthInstance inst = random_instance(seed, n, leaves, density, subset);
  const auto t0 = std::chrono::steady_clock::now();
  KernelCounters c;
  std::string blob;
  int real_stop = stop;
  if (p == Precision::Fp64) {
    auto set = compute_unifrac<double>(inst.tree, inst.table, cfg_of(m, p), start, stop, threads, &c);
    real_stop = set.stop;
    blob.append(reinterpret_cast<const char*>(set.distances.data()), set.distances.size() * sizeof(double));
    blob.append(reinterpret_cast<const char*>(set.totals.data()), set.totals.size() * sizeof(double));
  } else {
    auto set = compute_unifrac<float>(inst.tree, inst.table, cfg_of(m, p), start, stop, threads, &c);
    real_stop = set.stop;
    blob.append(reinterpret_cast<const char*>(set.distances.data()), set.distances.size() * sizeof(float));
    blob.append(reinterpret_cast<const char*>(set.totals.data()), set.totals.size() * sizeof(float));
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (!out_path.empty()) write_file(out_path, blob);
  std::printf("{\"seconds\":%.6f,\"stop\":%d,\"counters\":[%" PRIu64 ",%" PRIu64 ",%" PRIu64 "]}\n",
              secs, real_stop, c.accumulator_writes, c.embedding_reads, c.kernel_passes);
  return 0;
}

// dm_multi: one reference instance, several (metric, precision, range)
// computations: compute_unifrac<Real> per spec "metric:precision:start:stop",
// stripes (finalized distances, raw totals) to <outdir>/<spec>.bin, one JSON
// line per spec (tools/reference_at_scale.sh).
int cmd_dm_multi(std::uint64_t seed, int n, int leaves, double density, int subset, int threads,
                 const std::string& outdir, int nspec, char** specs) {
  const auto tg = std::chrono::steady_clock::now();
  const SynthInstance inst = random_instance(seed, n, leaves, density, subset);
  const double gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - tg).count();
  for (int i = 0; i < nspec; ++i) {
    std::string spec = specs[i];
    std::vector<std::string> f;
    for (std::size_t a = 0, b; a <= spec.size(); a = b + 1) {
      b = spec.find(':', a);
      if (b == std::string::npos) b = spec.size();
      f.push_back(spec.substr(a, b - a));
    }
    if (f.size() != 4) throw Error("spec must be metric:precision:start:stop");
    const Metric m = metric_from_name(f[0]);
    const Precision p = precision_from_name(f[1]);
    const int start = std::atoi(f[2].c_str()), stop = std::atoi(f[3].c_str());
    const auto t0 = std::chrono::steady_clock::now();
    std::string blob;
    if (p == Precision::Fp64) {
      auto set = compute_unifrac<double>(inst.tree, inst.table, cfg_of(m, p), start, stop, threads, nullptr);
      blob.append(reinterpret_cast<const char*>(set.distances.data()), set.distances.size() * sizeof(double));
      blob.append(reinterpret_cast<const char*>(set.totals.data()), set.totals.size() * sizeof(double));
    } else {
      auto set = compute_unifrac<float>(inst.tree, inst.table, cfg_of(m, p), start, stop, threads, nullptr);
      blob.append(reinterpret_cast<const char*>(set.distances.data()), set.distances.size() * sizeof(float));
      blob.append(reinterpret_cast<const char*>(set.totals.data()), set.totals.size() * sizeof(float));
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::string name = f[0] + "_" + f[1] + "_" + f[2] + "_" + f[3];
    write_file(outdir + "/" + name + ".bin", blob);
    std::printf("{\"spec\":\"%s\",\"seconds\":%.3f,\"instance_seconds\":%.3f,\"threads\":%d}\n", name.c_str(),
                secs, gen_s, threads);
    std::fflush(stdout);
  }
  return 0;
}

// The reference's own load_table_file on a table file, dumped as one JSON
// object (ids, CSR with %.17g values, totals) or {"error": "..."} — the
// checker of the native sparse loader (tests/test_abi.py).
int cmd_table(const std::string& path, const std::string& fmt, bool timing_only) {
  auto jstr = [](const std::string& x) {
    std::string o = "\"";
    for (const unsigned char c : x) {
      if (c == '"' || c == '\\') {
        o += '\\';
        o += static_cast<char>(c);
      } else if (c < 0x20) {
        char b[8];
        std::snprintf(b, sizeof(b), "\\u%04x", c);
        o += b;
      } else {
        o += static_cast<char>(c);
      }
    }
    return o + "\"";
  };
  try {
    const auto t0 = std::chrono::steady_clock::now();
    const SampleTable t = load_table_file(path, table_format_from_name(fmt));
    if (timing_only) {
      std::printf("{\"seconds\":%.3f,\"features\":%zu,\"samples\":%zu}\n",
                  std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(), t.feature_ids.size(),
                  t.sample_ids.size());
      return 0;
    }
    std::string o = "{\"samples\":[";
    for (size_t i = 0; i < t.sample_ids.size(); ++i) o += (i ? "," : "") + jstr(t.sample_ids[i]);
    o += "],\"features\":[";
    for (size_t i = 0; i < t.feature_ids.size(); ++i) o += (i ? "," : "") + jstr(t.feature_ids[i]);
    o += "],\"feat_ptr\":[0";
    size_t nnz = 0;
    for (const auto& row : t.entries) o += "," + std::to_string(nnz += row.size());
    o += "],\"sample_idx\":[";
    bool first = true;
    for (const auto& row : t.entries)
      for (const auto& e : row) {
        o += (first ? "" : ",") + std::to_string(e.first);
        first = false;
      }
    char b[40];
    o += "],\"counts\":[";
    first = true;
    for (const auto& row : t.entries)
      for (const auto& e : row) {
        std::snprintf(b, sizeof(b), "%.17g", e.second);
        o += (first ? "" : ",") + std::string(b);
        first = false;
      }
    o += "],\"totals\":[";
    for (size_t i = 0; i < t.sample_totals.size(); ++i) {
      std::snprintf(b, sizeof(b), "%.17g", t.sample_totals[i]);
      o += (i ? "," : "") + std::string(b);
    }
    std::printf("%s]}\n", o.c_str());
  } catch (const std::exception& e) {
    std::printf("{\"error\":%s}\n", jstr(e.what()).c_str());
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw Error("usage: ref_driver golden|instance|bench|dm ...");
    const std::string cmd = argv[1];
    if (cmd == "golden" && argc >= 4) return cmd_golden(argv[2], argv[3]);
    if (cmd == "mantel_golden" && argc >= 3) return cmd_mantel_golden(argv[2]);
    if (cmd == "wide_golden" && argc >= 3) return cmd_wide_golden(argv[2]);
    if (cmd == "dm_multi" && argc >= 10)
      return cmd_dm_multi(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]), std::atoi(argv[4]),
                          std::atof(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]), argv[8], argc - 9, argv + 9);
    if (cmd == "strf_golden" && argc >= 4) return cmd_strf_golden(argv[2], argv[3]);
    if (cmd == "table" && argc >= 4) return cmd_table(argv[2], argv[3], argc >= 5 && std::string(argv[4]) == "time");
    if (cmd == "instance" && argc >= 7)
      return cmd_instance(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]), std::atoi(argv[4]),
                          std::atof(argv[5]), std::atoi(argv[6]));
    if (cmd == "bench" && argc >= 13)
      return cmd_bench(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]), std::atoi(argv[4]),
                       std::atof(argv[5]), std::atoi(argv[6]), metric_from_name(argv[7]),
                       precision_from_name(argv[8]), std::atoi(argv[9]), std::atoi(argv[10]),
                       std::atoi(argv[11]), std::atoi(argv[12]));
    if (cmd == "dm" && argc >= 12)
      return cmd_dm(std::strtoull(argv[2], nullptr, 10), std::atoi(argv[3]), std::atoi(argv[4]),
                    std::atof(argv[5]), std::atoi(argv[6]), metric_from_name(argv[7]),
                    precision_from_name(argv[8]), std::atoi(argv[9]), std::atoi(argv[10]),
                    std::atoi(argv[11]), argc >= 13 ? argv[12] : "");
    throw Error("bad arguments");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_driver: %s\n", e.what());
    return 1;
  }
}
