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
#include <atomic>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <istream>
#include <iterator>
#include <ostream>

#include "host_hash.hpp"
#include "host_parallel.hpp"
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

namespace {

// Parallel build_csr with output identical to the serial one (the
// reference's graph.cpp:75-133): dense ids by first appearance over the
// (u, v) sequence, canonical edges by first occurrence keeping that
// occurrence's orientation and the minimum weight, rows filled in edge-id
// order.  Only for raw ids below 2^32 and not far above the entry count
// (direct first-appearance table); returns false otherwise.
bool build_csr_parallel(const EdgeList& edges, CsrGraph& g) {
  const std::size_t len = edges.entries.size();
  const unsigned T = detail::host_threads();
  RawId max_raw = 0;
  for (const WeightedEdge& e : edges.entries) max_raw = std::max({max_raw, e.u, e.v});
  if (max_raw >= 0xFFFFFFFFULL || max_raw > 8 * len + (1u << 20) || 2 * len >= 0xFFFFFFFFULL) return false;
  const std::size_t R = static_cast<std::size_t>(max_raw) + 1;
  constexpr std::uint32_t kNone = 0xFFFFFFFFu;
  // 1. first appearance of every raw id (position 2i for u, 2i+1 for v)
  std::vector<std::atomic<std::uint32_t>> first(R);
  detail::parallel_chunks(R, T, [&](unsigned, std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t i = b; i < e; ++i) first[i].store(kNone, std::memory_order_relaxed);
  });
  auto amin = [](std::atomic<std::uint32_t>& a, std::uint32_t v) {
    std::uint32_t cur = a.load(std::memory_order_relaxed);
    while (v < cur && !a.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
    }
  };
  detail::parallel_chunks(len, T, [&](unsigned, std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t i = b; i < e; ++i) {
      amin(first[edges.entries[i].u], static_cast<std::uint32_t>(2 * i));
      amin(first[edges.entries[i].v], static_cast<std::uint32_t>(2 * i + 1));
    }
  });
  std::vector<std::pair<std::uint32_t, std::uint32_t>> order;  // (first position, raw)
  order.reserve(len < R ? 2 * len : R);
  for (std::size_t r = 0; r < R; ++r) {
    const std::uint32_t f = first[r].load(std::memory_order_relaxed);
    if (f != kNone) order.emplace_back(f, static_cast<std::uint32_t>(r));
  }
  std::sort(order.begin(), order.end());
  std::vector<NodeId> dense(R, kNone);
  g.original_id.resize(order.size());
  for (std::size_t k = 0; k < order.size(); ++k) {
    dense[order[k].second] = static_cast<NodeId>(k);
    g.original_id[k] = order[k].second;
  }
  std::vector<std::atomic<std::uint32_t>>().swap(first);
  g.n = static_cast<NodeId>(order.size());
  const std::size_t n = g.n;
  // 2. canonical edges: group occurrences by the smaller endpoint (stable
  //    counting sort), find each key's first occurrence and minimum weight
  std::vector<std::uint32_t> cnt(static_cast<std::size_t>(T) * n, 0);
  detail::parallel_chunks(len, T, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint32_t* c = cnt.data() + static_cast<std::size_t>(t) * n;
    for (std::uint64_t i = b; i < e; ++i) {
      const NodeId a = dense[edges.entries[i].u], bb = dense[edges.entries[i].v];
      if (a != bb) ++c[std::min(a, bb)];
    }
  });
  std::vector<std::uint64_t> gstart(n + 1, 0);
  for (std::size_t x = 0; x < n; ++x) {  // exclusive positions, thread-major within a group
    std::uint64_t acc = gstart[x];
    for (unsigned t = 0; t < T; ++t) {
      const std::uint32_t c = cnt[static_cast<std::size_t>(t) * n + x];
      cnt[static_cast<std::size_t>(t) * n + x] = static_cast<std::uint32_t>(acc - gstart[x]);
      acc += c;
    }
    gstart[x + 1] = acc;
  }
  const std::uint64_t valid = gstart[n];
  std::vector<std::uint32_t> gidx(valid);  // entry index, grouped by smaller endpoint, in entry order
  detail::parallel_chunks(len, T, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint32_t* c = cnt.data() + static_cast<std::size_t>(t) * n;
    for (std::uint64_t i = b; i < e; ++i) {
      const NodeId a = dense[edges.entries[i].u], bb = dense[edges.entries[i].v];
      if (a == bb) continue;
      const NodeId lo = std::min(a, bb);
      gidx[gstart[lo] + c[lo]++] = static_cast<std::uint32_t>(i);
    }
  });
  std::vector<std::uint8_t> keep(len, 0);
  std::vector<double> wmin(len, 0.0);
  std::atomic<std::uint64_t> merged{0};
  detail::parallel_chunks(n, T, [&](unsigned, std::uint64_t b, std::uint64_t e) {
    std::vector<std::pair<NodeId, std::uint32_t>> grp;
    std::uint64_t mloc = 0;
    for (std::uint64_t x = b; x < e; ++x) {
      grp.clear();
      for (std::uint64_t k = gstart[x]; k < gstart[x + 1]; ++k) {
        const std::uint32_t i = gidx[k];
        const NodeId a = dense[edges.entries[i].u], bb = dense[edges.entries[i].v];
        grp.emplace_back(std::max(a, bb), i);
      }
      std::sort(grp.begin(), grp.end());  // by other endpoint, then entry index
      for (std::size_t k = 0; k < grp.size();) {
        std::size_t j = k;
        double w = edges.entries[grp[k].second].w;
        while (++j < grp.size() && grp[j].first == grp[k].first) w = std::min(w, edges.entries[grp[j].second].w);
        keep[grp[k].second] = 1;
        wmin[grp[k].second] = w;
        mloc += j - k - 1;
        k = j;
      }
    }
    merged += mloc;
  });
  std::vector<std::uint32_t>().swap(gidx);
  g.merged_duplicates = merged.load();
  // edge id of a first occurrence = number of first occurrences before it
  std::vector<std::uint64_t> part(T + 1, 0);
  detail::parallel_chunks(len, T, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint64_t c = 0;
    for (std::uint64_t i = b; i < e; ++i) c += keep[i];
    part[t + 1] = c;
  });
  for (unsigned t = 0; t < T; ++t) part[t + 1] += part[t];
  g.m = static_cast<EdgeId>(part[T]);
  const std::size_t m = g.m;
  g.edge_u.resize(m);
  g.edge_v.resize(m);
  std::vector<double> edge_w(m);
  detail::parallel_chunks(len, T, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint64_t id = part[t];
    for (std::uint64_t i = b; i < e; ++i)
      if (keep[i]) {
        g.edge_u[id] = dense[edges.entries[i].u];
        g.edge_v[id] = dense[edges.entries[i].v];
        edge_w[id] = wmin[i];
        ++id;
      }
  });
  std::vector<std::uint8_t>().swap(keep);
  std::vector<double>().swap(wmin);
  std::vector<NodeId>().swap(dense);
  // 3. rows in edge-id order: stable counting sort of the 2m (vertex, edge)
  //    incidences, per-thread counts over contiguous edge ranges
  std::fill(cnt.begin(), cnt.end(), 0u);
  detail::parallel_chunks(m, T, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint32_t* c = cnt.data() + static_cast<std::size_t>(t) * n;
    for (std::uint64_t k = b; k < e; ++k) {
      ++c[g.edge_u[k]];
      ++c[g.edge_v[k]];
    }
  });
  g.offsets.assign(n + 1, 0);
  for (std::size_t x = 0; x < n; ++x) {
    std::uint64_t acc = g.offsets[x];
    for (unsigned t = 0; t < T; ++t) {
      const std::uint32_t c = cnt[static_cast<std::size_t>(t) * n + x];
      cnt[static_cast<std::size_t>(t) * n + x] = static_cast<std::uint32_t>(acc);
      acc += c;
    }
    g.offsets[x + 1] = static_cast<EdgeId>(acc);
  }
  const std::size_t slots = 2 * m;
  g.adjacency.resize(slots);
  g.weights.resize(slots);
  g.edge_id.resize(slots);
  detail::parallel_chunks(m, T, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint32_t* c = cnt.data() + static_cast<std::size_t>(t) * n;
    for (std::uint64_t k = b; k < e; ++k) {
      const NodeId a = g.edge_u[k], bb = g.edge_v[k];
      const std::uint32_t sa = c[a]++, sb = c[bb]++;
      g.adjacency[sa] = bb;
      g.weights[sa] = edge_w[k];
      g.edge_id[sa] = static_cast<EdgeId>(k);
      g.adjacency[sb] = a;
      g.weights[sb] = edge_w[k];
      g.edge_id[sb] = static_cast<EdgeId>(k);
    }
  });
  g.min_incident_weight.assign(n, kInf);
  detail::parallel_chunks(n, T, [&](unsigned, std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t x = b; x < e; ++x)
      for (EdgeId s = g.offsets[x]; s < g.offsets[x + 1]; ++s)
        g.min_incident_weight[x] = std::min(g.min_incident_weight[x], g.weights[s]);
  });
  return true;
}

}  // namespace

CsrGraph build_csr(const EdgeList& edges) {
  CsrGraph g;
  if (edges.entries.size() >= detail::parallel_min_entries() && detail::host_threads() > 1) {
    CsrGraph p;
    if (build_csr_parallel(edges, p)) return p;
  }
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
