// C++ drop-in check: code written against the reference API
// (/root/reference/proj/include/wbc/*.hpp) compiles unchanged against
// include/wbc/*.hpp and links libwbc_b200.so.  Cases mirror the reference's
// test_graph.cpp / test_engine.cpp / test_brandes.cpp.
//   ./test_dropin cpu   -- host layer only (no device)
//   ./test_dropin gpu   -- bc_parallel on a B200
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "wbc/engine.hpp"
#include "wbc/generate.hpp"
#include "wbc/graph.hpp"

using namespace wbc;

static int g_fail = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
      ++g_fail;                                                   \
    }                                                             \
  } while (0)

static CsrGraph graph_of(std::initializer_list<std::tuple<RawId, RawId, double>> es) {
  EdgeList el;
  for (const auto& [u, v, w] : es) el.entries.push_back({u, v, w});
  return build_csr(el);
}

static bool close(const std::vector<double>& a, const std::vector<double>& b, double rtol) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (std::abs(a[i] - b[i]) > std::max(1e-12, rtol * std::max(std::abs(a[i]), std::abs(b[i])))) return false;
  return true;
}

static void cpu_cases() {
  std::istringstream in("# c\n0 1 2.5\n1 2\n3 3 1\n");
  const EdgeList el = parse_edge_list(in);
  CHECK(el.entries.size() == 2 && el.self_loops_dropped == 1 && el.entries[1].w == 1.0);
  bool threw = false;
  try {
    std::istringstream bad("0 1 1.0\n0 x 1.0");
    parse_edge_list(bad);
  } catch (const ParseError& e) {
    threw = e.line() == 2 && std::string(e.what()).find("line 2") != std::string::npos;
  }
  CHECK(threw);
  const CsrGraph tri = graph_of({{0, 1, 1}, {1, 2, 1}, {0, 2, 1}});
  CHECK(tri.offsets == (std::vector<EdgeId>{0, 2, 4, 6}));
  const CsrGraph d = graph_of({{0, 1, 3}, {1, 0, 5}});
  CHECK(d.m == 1 && d.merged_duplicates == 1 && d.weights[0] == 3.0);
  CHECK(gen_er(16, 4.0, 9).entries.size() == 32);
  CHECK(gen_kronecker(4, 4.0, 9).entries.size() == 32);
  CHECK(sample_sources(10, 20, 3).size() == 10);
  CHECK(strategy_name(parse_strategy("we-warp")) == "we-warp32");
  threw = false;
  try {
    parse_strategy("warp5");
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  EngineOptions opt;
  opt.workers = 0;
  threw = false;
  try {
    bc_parallel(tri, opt);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

static void gpu_cases() {
  const CsrGraph p3 = graph_of({{0, 1, 1}, {1, 2, 1}});
  BcResult r = bc_parallel(p3);
  CHECK(r.node_bc == (std::vector<double>{0.0, 2.0, 0.0}));
  CHECK(r.depth_per_source == (std::vector<uint32_t>{3, 2, 3}));
  const CsrGraph ts = graph_of({{0, 1, 1}, {0, 2, 2}, {1, 2, 1}, {2, 3, 1}});
  EngineOptions eo;
  eo.compute_edge_bc = true;
  r = bc_parallel(ts, eo);
  CHECK(close(r.node_bc, {0, 2, 4, 0}, 1e-12));
  CHECK(close(r.edge_bc, {4, 2, 6, 6}, 1e-12));
  GpuBcEngine eng(ts);
  const auto st = eng.dump_source(0);
  CHECK(st.sigma[3] == 2.0 && st.dist[3] == 3.0 && st.depth == 4);
  EngineOptions sub;
  sub.sources = std::vector<NodeId>{0};
  sub.normalization = Normalization::Halved;
  r = bc_parallel(p3, sub);
  CHECK(r.node_bc == (std::vector<double>{0.0, 0.5, 0.0}));
  sub.sources = std::vector<NodeId>{7};
  bool threw = false;
  try {
    bc_parallel(p3, sub);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);

  // the per-phase API (reference engine.hpp:46-106, test_engine.cpp cases)
  TraversalState st0;
  init_state(p3, 1, st0);
  CHECK(st0.order_len == 1 && st0.ends_len == 2 && st0.dist[1] == 0.0 && st0.sigma[1] == 1.0 &&
        st0.frontier_len == 1 && st0.unsettled[1] == 0 && std::isinf(st0.dist[0]));
  TraversalState sp;
  solve_source(p3, 0, Strategy{}, sp);
  CHECK(sp.depth() == 3 && sp.order_len == 3 && sp.frontier_len == 1 && sp.frontier[0] == 2);
  CHECK(sp.dist == (std::vector<double>{0.0, 1.0, 2.0}) && std::isinf(sp.threshold));
  TraversalState sq;
  solve_source_parallel(ts, 0, parse_strategy("we-warp8"), 4, sq);
  CHECK(sq.dist == (std::vector<double>{0.0, 1.0, 2.0, 3.0}) && sq.sigma[3] == 2.0 && sq.depth() == 4);
  std::vector<double> acc(ts.n, 0.0), eacc(ts.m, 0.0);
  for (NodeId s = 0; s < ts.n; ++s) {
    TraversalState t;
    solve_source(ts, s, Strategy{}, t);
    accumulate_dependencies(ts, Strategy{}, t, acc, eacc);
    if (s == 0) CHECK(t.delta == (std::vector<double>{0.0, 1.0, 1.0, 0.0}) || t.delta[1] == 1.0);
  }
  CHECK(close(acc, {0, 2, 4, 0}, 1e-12));
  CHECK(close(eacc, {4, 2, 6, 6}, 1e-12));
  threw = false;
  try {
    solve_source(ts, 0, Strategy{}, sq, SettleRule::LessEqual);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    init_state(ts, 9, sq);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  cpu_cases();
  if (gpu) gpu_cases();
  std::printf("%s: %d failures\n", gpu ? "cpu+gpu" : "cpu", g_fail);
  return g_fail;
}
