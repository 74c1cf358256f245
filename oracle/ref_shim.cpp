// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library, compiled together
// with the reference's own sources straight from /root/reference/proj/src
// (see oracle/Makefile) into oracle/_ref/libwbc_ref.so.  Tests, the golden
// fixture generator and bench.py's reference/cpu_baseline arm load it through
// ctypes; nothing in paper_1701_05975_b200/ may.
//
// Every entry point forwards to the reference API it names:
//   ref_parse_edge_list   -> wbc::parse_edge_list   (proj/include/wbc/graph.hpp:47)
//   ref_csr_build         -> wbc::build_csr         (proj/include/wbc/graph.hpp:74)
//   ref_gen_er/_kronecker -> wbc::gen_er / gen_kronecker (proj/include/wbc/generate.hpp:20-27)
//   ref_assign_weights    -> wbc::assign_weights    (generate.hpp:31)
//   ref_sample_sources    -> wbc::sample_sources    (generate.hpp:35)
//   ref_brandes           -> wbc::brandes_sequential (proj/include/wbc/brandes.hpp:24)
//   ref_brute_force       -> wbc::brute_force_bc    (brandes.hpp:30)
//   ref_bc_parallel       -> wbc::bc_parallel       (proj/include/wbc/engine.hpp:130)
//   ref_solve_source      -> wbc::solve_source + accumulate_dependencies (engine.hpp:93-99)
//   ref_format_*_tsv      -> wbc::format_node_bc_tsv / format_edge_bc_tsv (report.hpp:11,14)
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "wbc/brandes.hpp"
#include "wbc/engine.hpp"
#include "wbc/generate.hpp"
#include "wbc/graph.hpp"
#include "wbc/report.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

// Error codes mirror the product's C ABI: -1 invalid_argument, -2 ParseError,
// -3 anything else.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const wbc::ParseError& e) {
    return fail(e, -2);
  } catch (const std::invalid_argument& e) {
    return fail(e, -1);
  } catch (const std::exception& e) {
    return fail(e, -3);
  }
}

std::optional<std::vector<wbc::NodeId>> sources_of(const uint32_t* src, int64_t k) {
  if (k < 0) return std::nullopt;  // all vertices
  return std::vector<wbc::NodeId>(src, src + k);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- edge lists -----------------------------------------------------------
void* ref_edges_new(void) { return new wbc::EdgeList(); }
void ref_edges_free(void* h) { delete static_cast<wbc::EdgeList*>(h); }
uint64_t ref_edges_len(void* h) { return static_cast<wbc::EdgeList*>(h)->entries.size(); }
uint64_t ref_edges_self_loops(void* h) {
  return static_cast<wbc::EdgeList*>(h)->self_loops_dropped;
}
void ref_edges_get(void* h, uint64_t* u, uint64_t* v, double* w) {
  const auto& es = static_cast<wbc::EdgeList*>(h)->entries;
  for (size_t i = 0; i < es.size(); ++i) {
    u[i] = es[i].u;
    v[i] = es[i].v;
    w[i] = es[i].w;
  }
}
void ref_edges_set(void* h, uint64_t len, const uint64_t* u, const uint64_t* v, const double* w) {
  auto& es = static_cast<wbc::EdgeList*>(h)->entries;
  es.resize(len);
  for (size_t i = 0; i < len; ++i) es[i] = {u[i], v[i], w[i]};
}

int ref_parse_edge_list(const char* text, double default_weight, void** out) {
  return guarded([&] {
    std::istringstream in(text);
    *out = new wbc::EdgeList(wbc::parse_edge_list(in, default_weight));
  });
}

int ref_gen_er(uint64_t n, double avg_degree, uint64_t seed, void** out) {
  return guarded([&] { *out = new wbc::EdgeList(wbc::gen_er(n, avg_degree, seed)); });
}

int ref_gen_kronecker(int scale, double avg_degree, uint64_t seed, void** out) {
  return guarded([&] { *out = new wbc::EdgeList(wbc::gen_kronecker(scale, avg_degree, seed)); });
}

int ref_assign_weights(void* h, int lo, int hi, uint64_t seed) {
  return guarded([&] {
    auto* el = static_cast<wbc::EdgeList*>(h);
    *el = wbc::assign_weights(std::move(*el), lo, hi, seed);
  });
}

int ref_sample_sources(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out, uint32_t* out_len) {
  return guarded([&] {
    const auto s = wbc::sample_sources(n, k, seed);
    std::memcpy(out, s.data(), s.size() * sizeof(uint32_t));
    *out_len = static_cast<uint32_t>(s.size());
  });
}

// ---- CSR ------------------------------------------------------------------
int ref_csr_build(void* edges, void** out) {
  return guarded(
      [&] { *out = new wbc::CsrGraph(wbc::build_csr(*static_cast<wbc::EdgeList*>(edges))); });
}
// A CsrGraph filled from caller arrays (the repo's build_csr output, which
// tests/test_host_graph.py proves array-identical to the reference's): lets
// the CPU baseline skip the reference's single-threaded build at R-MAT-24.
// original_id / edge_u / edge_v may be null (brandes_sequential never reads them).
int ref_csr_from_arrays(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
                        const double* weights, const uint32_t* edge_id, const double* min_incident_weight,
                        void** out) {
  return guarded([&] {
    auto* g = new wbc::CsrGraph();
    g->n = n;
    g->m = m;
    g->offsets.assign(offsets, offsets + uint64_t{n} + 1);
    g->adjacency.assign(adjacency, adjacency + 2 * uint64_t{m});
    g->weights.assign(weights, weights + 2 * uint64_t{m});
    g->edge_id.assign(edge_id, edge_id + 2 * uint64_t{m});
    g->min_incident_weight.assign(min_incident_weight, min_incident_weight + n);
    g->original_id.resize(n);
    for (uint32_t i = 0; i < n; ++i) g->original_id[i] = i;
    *out = g;
  });
}
void ref_csr_free(void* h) { delete static_cast<wbc::CsrGraph*>(h); }
uint32_t ref_csr_n(void* h) { return static_cast<wbc::CsrGraph*>(h)->n; }
uint32_t ref_csr_m(void* h) { return static_cast<wbc::CsrGraph*>(h)->m; }
uint64_t ref_csr_merged(void* h) { return static_cast<wbc::CsrGraph*>(h)->merged_duplicates; }
void ref_csr_get(void* h, uint32_t* offsets, uint32_t* adjacency, double* weights,
                 uint32_t* edge_id, double* min_incident_weight, uint64_t* original_id,
                 uint32_t* edge_u, uint32_t* edge_v) {
  const auto& g = *static_cast<wbc::CsrGraph*>(h);
  std::memcpy(offsets, g.offsets.data(), g.offsets.size() * 4);
  std::memcpy(adjacency, g.adjacency.data(), g.adjacency.size() * 4);
  std::memcpy(weights, g.weights.data(), g.weights.size() * 8);
  std::memcpy(edge_id, g.edge_id.data(), g.edge_id.size() * 4);
  std::memcpy(min_incident_weight, g.min_incident_weight.data(), g.min_incident_weight.size() * 8);
  std::memcpy(original_id, g.original_id.data(), g.original_id.size() * 8);
  std::memcpy(edge_u, g.edge_u.data(), g.edge_u.size() * 4);
  std::memcpy(edge_v, g.edge_v.data(), g.edge_v.size() * 4);
}

// ---- algorithms -----------------------------------------------------------
// k < 0 means "all vertices" (EngineOptions::sources left empty).
int ref_brandes(void* h, const uint32_t* sources, int64_t k, int edge_bc, int halved,
                double eps, double* node_bc, double* edge_bc_out, double* elapsed) {
  return guarded([&] {
    const auto& g = *static_cast<wbc::CsrGraph*>(h);
    wbc::BrandesOptions opt;
    opt.compute_edge_bc = edge_bc != 0;
    opt.normalization = halved ? wbc::Normalization::Halved : wbc::Normalization::Raw;
    opt.equality_epsilon = eps;
    opt.sources = sources_of(sources, k);
    const wbc::BcResult r = wbc::brandes_sequential(g, opt);
    std::memcpy(node_bc, r.node_bc.data(), r.node_bc.size() * 8);
    if (edge_bc) std::memcpy(edge_bc_out, r.edge_bc.data(), r.edge_bc.size() * 8);
    if (elapsed) *elapsed = r.elapsed.count();
  });
}

int ref_brute_force(void* h, double* node_bc) {
  return guarded([&] {
    const wbc::BcResult r = wbc::brute_force_bc(*static_cast<wbc::CsrGraph*>(h));
    std::memcpy(node_bc, r.node_bc.data(), r.node_bc.size() * 8);
  });
}

int ref_bc_parallel(void* h, const char* strategy, int workers, const uint32_t* sources,
                    int64_t k, int edge_bc, int halved, int strict_merge, int less_equal,
                    double* node_bc, double* edge_bc_out, uint32_t* depth, double* elapsed) {
  return guarded([&] {
    const auto& g = *static_cast<wbc::CsrGraph*>(h);
    wbc::EngineOptions opt;
    opt.strategy = wbc::parse_strategy(strategy);
    opt.workers = workers;
    opt.compute_edge_bc = edge_bc != 0;
    opt.normalization = halved ? wbc::Normalization::Halved : wbc::Normalization::Raw;
    opt.strict_merge = strict_merge != 0;
    opt.settle_rule = less_equal ? wbc::SettleRule::LessEqual : wbc::SettleRule::StrictLess;
    opt.sources = sources_of(sources, k);
    const wbc::BcResult r = wbc::bc_parallel(g, opt);
    std::memcpy(node_bc, r.node_bc.data(), r.node_bc.size() * 8);
    if (edge_bc) std::memcpy(edge_bc_out, r.edge_bc.data(), r.edge_bc.size() * 8);
    if (depth) std::memcpy(depth, r.depth_per_source.data(), r.depth_per_source.size() * 4);
    if (elapsed) *elapsed = r.elapsed.count();
  });
}

// One source through the public per-phase API (engine.hpp:93-99): solve_source
// then accumulate_dependencies.  order has n entries, ends n+2.
int ref_solve_source(void* h, uint32_t source, const char* strategy, int less_equal,
                     double* dist, double* sigma, double* delta, uint32_t* depth,
                     uint32_t* order, uint32_t* order_len, uint32_t* ends, uint32_t* ends_len,
                     double* node_acc) {
  return guarded([&] {
    const auto& g = *static_cast<wbc::CsrGraph*>(h);
    const wbc::Strategy strat = wbc::parse_strategy(strategy);
    wbc::TraversalState st;
    wbc::solve_source(g, source, strat, st,
                      less_equal ? wbc::SettleRule::LessEqual : wbc::SettleRule::StrictLess);
    std::vector<double> acc(g.n, 0.0);
    wbc::accumulate_dependencies(g, strat, st, acc);
    std::memcpy(dist, st.dist.data(), g.n * 8);
    std::memcpy(sigma, st.sigma.data(), g.n * 8);
    std::memcpy(delta, st.delta.data(), g.n * 8);
    if (node_acc) std::memcpy(node_acc, acc.data(), g.n * 8);
    *depth = st.depth();
    if (order) std::memcpy(order, st.order.data(), st.order_len * 4);
    if (order_len) *order_len = st.order_len;
    if (ends) std::memcpy(ends, st.ends.data(), st.ends_len * 4);
    if (ends_len) *ends_len = st.ends_len;
  });
}

// Reference TSV report bytes; returns required length (call with cap 0 first).
uint64_t ref_format_node_tsv(void* h, const double* node_bc, char* out, uint64_t cap) {
  const auto& g = *static_cast<wbc::CsrGraph*>(h);
  wbc::BcResult r;
  r.node_bc.assign(node_bc, node_bc + g.n);
  const std::string s = wbc::format_node_bc_tsv(g, r);
  if (cap >= s.size()) std::memcpy(out, s.data(), s.size());
  return s.size();
}

uint64_t ref_format_edge_tsv(void* h, const double* edge_bc, char* out, uint64_t cap) {
  const auto& g = *static_cast<wbc::CsrGraph*>(h);
  wbc::BcResult r;
  r.edge_bc.assign(edge_bc, edge_bc + g.m);
  const std::string s = wbc::format_edge_bc_tsv(g, r);
  if (cap >= s.size()) std::memcpy(out, s.data(), s.size());
  return s.size();
}

}  // extern "C"
