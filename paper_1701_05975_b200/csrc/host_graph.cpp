// Native CSR loader: parse_edge_list / build_csr with the reference's exact
// semantics (reference: proj/src/graph.cpp:40-133, contract graph.hpp:43-74).
//
// Behavioural contract reproduced (each pinned by tests/test_host_graph.py):
//  * parser: blank lines are those with only ' ', '\t', '\r'; '#' after
//    leading blanks starts a comment; 2 or 3 whitespace-separated fields;
//    ids are unsigned decimal without sign; weights parse with strtod, must be
//    finite and > 0; u == v is dropped and counted; errors carry the 1-based
//    line and the reference's message text.
//  * build_csr: dense ids by first appearance (u before v), duplicate
//    undirected edges merged to the minimum weight keeping the first
//    orientation, degree prefix sums, slots emitted u->v then v->u per
//    canonical edge in canonical order, min incident weight per vertex.
// The implementation differs: one pass with an open-addressing interner
// instead of std::unordered_map, and a pre-sized slot fill.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <istream>
#include <iterator>
#include <ostream>

#include "host_hash.hpp"
#include "wbc/graph.hpp"

namespace wbc {

ParseError::ParseError(std::size_t line, const std::string& what)
    : std::runtime_error("line " + std::to_string(line) + ": " + what), line_(line) {}

namespace {

inline bool is_blank_char(char c) { return c == ' ' || c == '\t' || c == '\r'; }
// std::istream >> std::string splits on isspace() in the "C" locale.
inline bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

bool to_raw_id(const std::string& tok, RawId& out) {
  if (tok.empty() || tok[0] == '-' || tok[0] == '+') return false;
  errno = 0;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(tok.c_str(), &end, 10);
  if (errno != 0 || end != tok.c_str() + tok.size()) return false;
  out = v;
  return true;
}

bool to_weight(const std::string& tok, double& out) {
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(tok.c_str(), &end);
  if (errno != 0 || end != tok.c_str() + tok.size() || !std::isfinite(v)) return false;
  out = v;
  return true;
}

void parse_line(const char* b, const char* e, std::size_t lineno, double default_weight,
                EdgeList& out, std::string (&tok)[4]) {
  const char* first = b;
  while (first < e && is_blank_char(*first)) ++first;
  if (first == e) return;     // blank
  if (*first == '#') return;  // comment
  int nt = 0;
  for (const char* p = b; p < e;) {
    while (p < e && is_space(*p)) ++p;
    if (p == e) break;
    const char* q = p;
    while (q < e && !is_space(*q)) ++q;
    if (nt < 4) tok[nt].assign(p, q);
    ++nt;
    p = q;
  }
  if (nt < 2 || nt > 3)
    throw ParseError(lineno, "expected 'u v' or 'u v w', got " + std::to_string(nt) + " fields");
  RawId u, v;
  if (!to_raw_id(tok[0], u)) throw ParseError(lineno, "bad node id '" + tok[0] + "'");
  if (!to_raw_id(tok[1], v)) throw ParseError(lineno, "bad node id '" + tok[1] + "'");
  double w = default_weight;
  if (nt == 3 && !to_weight(tok[2], w)) throw ParseError(lineno, "bad weight '" + tok[2] + "'");
  if (!(w > 0.0)) throw ParseError(lineno, "non-positive weight " + tok[nt - 1]);
  if (u == v) {
    ++out.self_loops_dropped;
    return;
  }
  out.entries.push_back({u, v, w});
}

}  // namespace

EdgeList parse_edge_list_text(const char* data, std::size_t len, double default_weight) {
  if (!(default_weight > 0.0))
    throw std::invalid_argument("parse_edge_list: default weight must be positive");
  EdgeList out;
  std::string tok[4];
  std::size_t lineno = 0;
  const char* p = data;
  const char* end = data + len;
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<std::size_t>(end - p)));
    const char* le = nl ? nl : end;
    ++lineno;
    parse_line(p, le, lineno, default_weight, out, tok);
    p = nl ? nl + 1 : end;
  }
  return out;
}

EdgeList parse_edge_list(std::istream& in, double default_weight) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return parse_edge_list_text(text.data(), text.size(), default_weight);
}

CsrGraph build_csr(const EdgeList& edges) {
  CsrGraph g;
  const std::size_t len = edges.entries.size();
  detail::U64Map dense(std::min<std::size_t>(2 * len, 1u << 20));
  detail::U64Map seen(std::min<std::size_t>(len, 1u << 20));
  std::vector<double> edge_w;
  edge_w.reserve(len);
  g.edge_u.reserve(len);
  g.edge_v.reserve(len);
  const auto intern = [&](RawId raw) -> NodeId {
    auto [slot, fresh] = dense.try_emplace(raw, static_cast<NodeId>(g.original_id.size()));
    if (fresh) g.original_id.push_back(raw);
    return *slot;
  };
  for (const WeightedEdge& e : edges.entries) {
    const NodeId a = intern(e.u);
    const NodeId b = intern(e.v);
    if (a == b) continue;
    const std::uint64_t key = a < b ? (std::uint64_t{a} << 32 | b) : (std::uint64_t{b} << 32 | a);
    auto [slot, fresh] = seen.try_emplace(key, static_cast<EdgeId>(g.edge_u.size()));
    if (fresh) {
      g.edge_u.push_back(a);
      g.edge_v.push_back(b);
      edge_w.push_back(e.w);
    } else {
      double& keep = edge_w[*slot];
      if (e.w < keep) keep = e.w;
      ++g.merged_duplicates;
    }
  }
  g.n = static_cast<NodeId>(g.original_id.size());
  g.m = static_cast<EdgeId>(g.edge_u.size());
  g.offsets.assign(std::size_t{g.n} + 1, 0);
  for (EdgeId e = 0; e < g.m; ++e) {
    ++g.offsets[g.edge_u[e] + 1];
    ++g.offsets[g.edge_v[e] + 1];
  }
  for (NodeId v = 0; v < g.n; ++v) g.offsets[v + 1] += g.offsets[v];
  const std::size_t slots = 2 * std::size_t{g.m};
  g.adjacency.resize(slots);
  g.weights.resize(slots);
  g.edge_id.resize(slots);
  g.min_incident_weight.assign(g.n, kInf);
  std::vector<EdgeId> fill(g.offsets.begin(), g.offsets.end() - 1);
  for (EdgeId e = 0; e < g.m; ++e) {
    const NodeId a = g.edge_u[e], b = g.edge_v[e];
    const double w = edge_w[e];
    const EdgeId sa = fill[a]++, sb = fill[b]++;
    g.adjacency[sa] = b;
    g.weights[sa] = w;
    g.edge_id[sa] = e;
    g.adjacency[sb] = a;
    g.weights[sb] = w;
    g.edge_id[sb] = e;
    if (w < g.min_incident_weight[a]) g.min_incident_weight[a] = w;
    if (w < g.min_incident_weight[b]) g.min_incident_weight[b] = w;
  }
  return g;
}

GraphStats graph_stats(const CsrGraph& g) {
  GraphStats s;
  s.n = g.n;
  s.m = g.m;
  for (NodeId v = 0; v < g.n; ++v) s.max_degree = std::max(s.max_degree, g.degree(v));
  s.avg_degree = g.n ? 2.0 * static_cast<double>(g.m) / static_cast<double>(g.n) : 0.0;
  return s;
}

EdgeList to_edge_list(const CsrGraph& g) {
  std::vector<double> w(g.m, 0.0);
  for (std::size_t s = 0; s < g.weights.size(); ++s) w[g.edge_id[s]] = g.weights[s];
  EdgeList out;
  out.entries.resize(g.m);
  for (EdgeId e = 0; e < g.m; ++e)
    out.entries[e] = {g.original_id[g.edge_u[e]], g.original_id[g.edge_v[e]], w[e]};
  return out;
}

void write_edge_list(std::ostream& out, const EdgeList& edges,
                     std::span<const std::string> header) {
  for (const std::string& h : header) out << "# " << h << '\n';
  char buf[96];
  for (const WeightedEdge& e : edges.entries) {
    const int k = std::snprintf(buf, sizeof buf, "%llu %llu %.17g\n",
                                static_cast<unsigned long long>(e.u),
                                static_cast<unsigned long long>(e.v), e.w);
    out.write(buf, k);
  }
}

}  // namespace wbc
