// wbc -- command-line drop-in for the reference's `wbc` tool
// (proj/tools/main.cpp), with betweenness computed on the B200 engine.
//
// Subcommands and their contracts follow the reference:
//   compute <edges> [-o F] [--strategy S] [--lane-width W] [--workers T]
//           [--edge-bc] [--normalize raw|half] [--unit-weights] [--strict]
//           [--sources-sample K] [--seed S] [--default-weight W]
//       node TSV (+ edge TSV) on stdout or -o (report.cpp:20-46); stderr line
//       "n=.. m=.. strategy=.. wall_time=..s" (main.cpp:154-155).  The CPU
//       schedule options are validated exactly as the reference does
//       (engine.cpp:21-40,110-114,373-374) but do not change the GPU run.
//   generate --model er|kronecker|ba|grid [...] [-o F]   (main.cpp:159-207;
//       ba/grid are the new generators of BASELINE configs 2 and 4)
//   stats <edges> [--depth] [--sources-sample K] [--seed S]   (main.cpp:226-246)
// Exit status 0 when the artifact was fully written, 2 on any bad input or
// argument (main.cpp:308-324).  The reference's `bench` (CPU strategy
// comparison) is not part of the GPU engine: bench.py measures the GPU path.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "wbc/engine.hpp"
#include "wbc/generate.hpp"
#include "wbc/graph.hpp"
#include "wbc/report.hpp"

namespace {

struct Args {
  std::string sub;
  std::vector<std::string> positional;
  std::map<std::string, std::string> opts;
  std::set<std::string> flags;
};

// Parses `--name value`, `--name=value`, `-o value` and bare flags against
// the subcommand's declared options; anything else is an error.
Args parse_args(int argc, char** argv, const std::set<std::string>& valued, const std::set<std::string>& bare,
                size_t max_positional) {
  Args a;
  if (argc < 2) throw std::invalid_argument("a subcommand is required (compute, generate, stats)");
  a.sub = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string t = argv[i];
    if (t == "-o") t = "--output";
    if (t.rfind("--", 0) == 0) {
      std::string name = t, value;
      bool has_value = false;
      const size_t eq = t.find('=');
      if (eq != std::string::npos) {
        name = t.substr(0, eq);
        value = t.substr(eq + 1);
        has_value = true;
      }
      if (bare.count(name)) {
        if (has_value) throw std::invalid_argument(name + " takes no value");
        a.flags.insert(name);
      } else if (valued.count(name)) {
        if (!has_value) {
          if (i + 1 >= argc) throw std::invalid_argument(name + " requires a value");
          value = argv[++i];
        }
        a.opts[name] = value;
      } else {
        throw std::invalid_argument("unknown option " + name);
      }
    } else {
      a.positional.push_back(t);
    }
  }
  if (a.positional.size() > max_positional) throw std::invalid_argument("unexpected argument " + a.positional.back());
  return a;
}

std::uint64_t to_u64(const std::string& name, const std::string& s) {
  size_t pos = 0;
  unsigned long long v = 0;
  try {
    v = std::stoull(s, &pos);
  } catch (...) {
    pos = 0;
  }
  if (pos != s.size() || s.empty() || s[0] == '-') throw std::invalid_argument(name + ": not a non-negative integer: " + s);
  return v;
}

int to_int(const std::string& name, const std::string& s) {
  size_t pos = 0;
  int v = 0;
  try {
    v = std::stoi(s, &pos);
  } catch (...) {
    pos = 0;
  }
  if (pos != s.size() || s.empty()) throw std::invalid_argument(name + ": not an integer: " + s);
  return v;
}

double to_double(const std::string& name, const std::string& s) {
  size_t pos = 0;
  double v = 0;
  try {
    v = std::stod(s, &pos);
  } catch (...) {
    pos = 0;
  }
  if (pos != s.size() || s.empty()) throw std::invalid_argument(name + ": not a number: " + s);
  return v;
}

std::uint64_t ensure_seed(std::optional<std::uint64_t>& seed) {
  if (!seed) {
    seed = std::random_device{}();
    std::cerr << "seed: " << *seed << " (drawn; pass --seed to reproduce)\n";
  }
  return *seed;
}

wbc::CsrGraph load_graph(const std::string& path, double default_weight, bool unit_weights) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("cannot open input file '" + path + "'");
  wbc::EdgeList edges = wbc::parse_edge_list(f, default_weight);
  if (unit_weights)
    for (wbc::WeightedEdge& e : edges.entries) e.w = 1.0;
  return wbc::build_csr(edges);
}

bool write_artifact(const std::string& path, const std::string& text) {
  if (path.empty() || path == "-") {
    std::cout << text;
    std::cout.flush();
    return static_cast<bool>(std::cout);
  }
  std::ofstream f(path);
  if (!f) return false;
  f << text;
  f.flush();
  return static_cast<bool>(f);
}

std::string fmt_avg(double x) {  // main.cpp:106-113
  char buf[48];
  if (x == static_cast<double>(static_cast<std::uint64_t>(x)))
    std::snprintf(buf, sizeof buf, "%.1f", x);
  else
    std::snprintf(buf, sizeof buf, "%g", x);
  return buf;
}

std::optional<std::vector<wbc::NodeId>> sample_or_all(const wbc::CsrGraph& g, std::uint64_t k,
                                                      std::optional<std::uint64_t>& seed) {
  if (k == 0 || k >= g.n) return std::nullopt;
  return wbc::sample_sources(g.n, static_cast<wbc::NodeId>(k), ensure_seed(seed));
}

std::optional<std::uint64_t> opt_seed(const Args& a) {
  auto it = a.opts.find("--seed");
  if (it == a.opts.end()) return std::nullopt;
  return to_u64("--seed", it->second);
}

std::string get(const Args& a, const std::string& k, const std::string& dflt) {
  auto it = a.opts.find(k);
  return it == a.opts.end() ? dflt : it->second;
}

int run_compute(int argc, char** argv) {
  const Args a = parse_args(argc, argv,
                            {"--output", "--strategy", "--lane-width", "--workers", "--normalize",
                             "--sources-sample", "--seed", "--default-weight"},
                            {"--edge-bc", "--unit-weights", "--strict"}, 1);
  if (a.positional.empty()) throw std::invalid_argument("compute: input file required");
  const std::string normalize = get(a, "--normalize", "raw");
  if (normalize != "raw" && normalize != "half") throw std::invalid_argument("--normalize must be raw or half");
  const std::string strategy = get(a, "--strategy", "we-warp32");
  const int lane_width = to_int("--lane-width", get(a, "--lane-width", "0"));
  const int workers = to_int("--workers", get(a, "--workers", std::to_string(std::thread::hardware_concurrency())));
  const std::uint64_t k = to_u64("--sources-sample", get(a, "--sources-sample", "0"));
  std::optional<std::uint64_t> seed = opt_seed(a);
  const wbc::CsrGraph g = load_graph(a.positional[0], to_double("--default-weight", get(a, "--default-weight", "1")),
                                     a.flags.count("--unit-weights") > 0);
  wbc::EngineOptions opt;
  std::string label;
  if (strategy == "seq" || strategy == "sequential") {
    label = "sequential";  // the oracle's schedule; the GPU computes the same BC
  } else {
    opt.strategy = wbc::parse_strategy(strategy);
    if (lane_width != 0) {
      opt.strategy.lane_width = lane_width;
      if (!wbc::valid_lane_width(lane_width))
        throw std::invalid_argument("invalid --lane-width (expected 1, 4, 8, 16 or 32)");
    }
    label = wbc::strategy_name(opt.strategy);
  }
  opt.workers = std::max(1, workers);
  opt.compute_edge_bc = a.flags.count("--edge-bc") > 0;
  opt.normalization = normalize == "half" ? wbc::Normalization::Halved : wbc::Normalization::Raw;
  opt.strict_merge = a.flags.count("--strict") > 0;
  if (auto sub = sample_or_all(g, k, seed)) opt.sources = *sub;
  const wbc::BcResult r = wbc::bc_parallel(g, opt);
  std::string text = wbc::format_node_bc_tsv(g, r);
  if (opt.compute_edge_bc) text += wbc::format_edge_bc_tsv(g, r);
  const std::string out = get(a, "--output", "");
  if (!write_artifact(out, text)) throw std::runtime_error("failed to write output '" + out + "'");
  std::cerr << "n=" << g.n << " m=" << g.m << " strategy=" << label << " wall_time=" << r.elapsed.count() << "s\n";
  return 0;
}

int run_generate(int argc, char** argv) {
  const Args a = parse_args(argc, argv,
                            {"--model", "--nodes", "--scale", "--avg-degree", "--seed", "--weight-lo",
                             "--weight-hi", "--initiator", "--output", "--m-per", "--rows", "--cols"},
                            {}, 0);
  const std::string model = get(a, "--model", "");
  if (model.empty()) throw std::invalid_argument("--model is required");
  std::optional<std::uint64_t> seed_opt = opt_seed(a);
  const int lo = to_int("--weight-lo", get(a, "--weight-lo", "1"));
  const int hi = to_int("--weight-hi", get(a, "--weight-hi", "10"));
  wbc::EdgeList edges;
  std::vector<std::string> header;
  std::uint64_t requested = 0;
  std::uint64_t seed = 0;
  std::ostringstream params;
  if (model == "er" || model == "kronecker") {
    if (!a.opts.count("--avg-degree")) throw std::invalid_argument("--avg-degree is required");
    const double avg = to_double("--avg-degree", get(a, "--avg-degree", "0"));
    if (model == "er") {
      const std::uint64_t nodes = to_u64("--nodes", get(a, "--nodes", "0"));
      if (nodes == 0) throw std::invalid_argument("--model er requires --nodes");
      seed = ensure_seed(seed_opt);
      requested = static_cast<std::uint64_t>(std::llround(nodes * avg / 2.0));
      edges = wbc::gen_er(nodes, avg, seed);
      params << "model=er nodes=" << nodes << " avg_degree=" << avg << " seed=" << seed << " weight_lo=" << lo
             << " weight_hi=" << hi;
    } else {
      const int scale = to_int("--scale", get(a, "--scale", "0"));
      if (scale == 0) throw std::invalid_argument("--model kronecker requires --scale");
      seed = ensure_seed(seed_opt);
      wbc::KroneckerInitiator init;
      if (a.opts.count("--initiator")) {
        std::vector<double> v;
        std::stringstream ss(a.opts.at("--initiator"));
        std::string tok;
        while (std::getline(ss, tok, ',')) v.push_back(to_double("--initiator", tok));
        if (v.size() != 4) throw std::invalid_argument("--initiator needs exactly 4 values a,b,c,d");
        init = {v[0], v[1], v[2], v[3]};
      }
      requested = static_cast<std::uint64_t>(std::llround(static_cast<double>(1ULL << scale) * avg / 2.0));
      edges = wbc::gen_kronecker(scale, avg, seed, init);
      params << "model=kronecker scale=" << scale << " avg_degree=" << avg << " seed=" << seed
             << " initiator=" << init.a << ',' << init.b << ',' << init.c << ',' << init.d << " weight_lo=" << lo
             << " weight_hi=" << hi;
    }
  } else if (model == "ba") {
    const std::uint64_t nodes = to_u64("--nodes", get(a, "--nodes", "0"));
    const std::uint64_t mper = to_u64("--m-per", get(a, "--m-per", "0"));
    if (nodes == 0 || mper == 0) throw std::invalid_argument("--model ba requires --nodes and --m-per");
    seed = ensure_seed(seed_opt);
    edges = wbc::gen_ba(nodes, static_cast<std::uint32_t>(mper), seed);
    requested = edges.entries.size();
    params << "model=ba nodes=" << nodes << " m_per=" << mper << " seed=" << seed << " weight_lo=" << lo
           << " weight_hi=" << hi;
  } else if (model == "grid") {
    const std::uint64_t rows = to_u64("--rows", get(a, "--rows", "0"));
    const std::uint64_t cols = to_u64("--cols", get(a, "--cols", "0"));
    if (rows == 0 || cols == 0) throw std::invalid_argument("--model grid requires --rows and --cols");
    seed = ensure_seed(seed_opt);
    edges = wbc::gen_grid(static_cast<std::uint32_t>(rows), static_cast<std::uint32_t>(cols));
    requested = edges.entries.size();
    params << "model=grid rows=" << rows << " cols=" << cols << " seed=" << seed << " weight_lo=" << lo
           << " weight_hi=" << hi;
  } else {
    throw std::invalid_argument("--model must be er, kronecker, ba or grid");
  }
  header.push_back(params.str());
  if (edges.entries.size() < requested)
    std::cerr << "warning: achieved " << edges.entries.size() << " of " << requested
              << " requested edges (resampling cap)\n";
  edges = wbc::assign_weights(std::move(edges), lo, hi, seed);
  std::ostringstream counts;
  counts << "edges_requested=" << requested << " edges_achieved=" << edges.entries.size();
  header.push_back(counts.str());
  std::ostringstream body;
  wbc::write_edge_list(body, edges, header);
  const std::string out = get(a, "--output", "");
  if (!write_artifact(out, body.str())) throw std::runtime_error("failed to write output '" + out + "'");
  return 0;
}

int run_stats(int argc, char** argv) {
  const Args a = parse_args(argc, argv, {"--sources-sample", "--seed", "--default-weight"}, {"--depth"}, 1);
  if (a.positional.empty()) throw std::invalid_argument("stats: input file required");
  const wbc::CsrGraph g =
      load_graph(a.positional[0], to_double("--default-weight", get(a, "--default-weight", "1")), false);
  const wbc::GraphStats s = wbc::graph_stats(g);
  std::ostringstream line;
  line << "n=" << s.n << " m=" << s.m << " max_degree=" << s.max_degree << " avg_degree=" << fmt_avg(s.avg_degree);
  if (a.flags.count("--depth") && g.n > 0) {
    std::optional<std::uint64_t> seed = opt_seed(a);
    const std::uint64_t k = to_u64("--sources-sample", get(a, "--sources-sample", "64"));
    std::vector<wbc::NodeId> sources;
    if (auto sub = sample_or_all(g, k, seed))
      sources = *sub;
    else
      for (wbc::NodeId v = 0; v < g.n; ++v) sources.push_back(v);
    // Eq. 4 settlement depth per source (solve_source in the reference,
    // main.cpp:234-240) from the GPU run's depth_per_source
    wbc::EngineOptions opt;
    opt.sources = sources;
    const wbc::BcResult r = wbc::bc_parallel(g, opt);
    double sum = 0.0;
    for (const wbc::NodeId src : sources) sum += r.depth_per_source[src];
    line << " avg_depth=" << fmt_avg(sum / static_cast<double>(sources.size()));
  }
  line << '\n';
  if (!write_artifact("", line.str())) throw std::runtime_error("failed to write stats");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string sub = argc >= 2 ? argv[1] : "";
    if (sub == "compute") return run_compute(argc, argv);
    if (sub == "generate") return run_generate(argc, argv);
    if (sub == "stats") return run_stats(argc, argv);
    if (sub == "bench")
      throw std::invalid_argument("bench compares the reference's CPU schedules; the GPU engine is measured by bench.py");
    throw std::invalid_argument(sub.empty() ? "a subcommand is required (compute, generate, stats)"
                                            : "unknown subcommand '" + sub + "'");
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
