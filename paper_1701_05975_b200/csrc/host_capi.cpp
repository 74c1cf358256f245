// extern "C" exports of the native host layer (CSR loader + generators),
// declared in include/wbc_gpu.h.  Thin: each call forwards to the C++ API in
// include/wbc/{graph,generate}.hpp and converts exceptions to status codes.
#include <cstring>
#include <stdexcept>
#include <string>

#include "wbc/generate.hpp"
#include "wbc/graph.hpp"
#include "wbc_gpu.h"

namespace wbc {
EdgeList parse_edge_list_text(const char* data, std::size_t len, double default_weight);
}

struct wbc_edge_list {
  wbc::EdgeList el;
};
struct wbc_csr {
  wbc::CsrGraph g;
};

// Shared with wbc_gpu.cu through this symbol (one error slot per thread).
extern "C" const char* wbc_gpu_last_error(void);
namespace wbc_host {
int set_error(int code, const std::string& msg);
}

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return WBC_OK;
  } catch (const wbc::ParseError& e) {
    return wbc_host::set_error(WBC_E_PARSE, e.what());
  } catch (const std::invalid_argument& e) {
    return wbc_host::set_error(WBC_E_INVALID, e.what());
  } catch (const std::bad_alloc&) {
    return wbc_host::set_error(WBC_E_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return wbc_host::set_error(WBC_E_CUDA, e.what());
  }
}

}  // namespace

extern "C" {

int wbc_host_parse_edge_list(const char* text, size_t len, double default_weight,
                             wbc_edge_list** out, uint64_t* err_line) {
  if (err_line) *err_line = 0;
  try {
    auto* h = new wbc_edge_list{wbc::parse_edge_list_text(text, len, default_weight)};
    *out = h;
    return WBC_OK;
  } catch (const wbc::ParseError& e) {
    if (err_line) *err_line = e.line();
    return wbc_host::set_error(WBC_E_PARSE, e.what());
  } catch (const std::invalid_argument& e) {
    return wbc_host::set_error(WBC_E_INVALID, e.what());
  } catch (const std::exception& e) {
    return wbc_host::set_error(WBC_E_NOMEM, e.what());
  }
}

wbc_edge_list* wbc_host_edges_new(uint64_t len, const uint64_t* u, const uint64_t* v,
                                  const double* w) {
  auto* h = new wbc_edge_list();
  h->el.entries.resize(len);
  for (uint64_t i = 0; i < len; ++i) h->el.entries[i] = {u[i], v[i], w[i]};
  return h;
}

uint64_t wbc_host_edges_len(const wbc_edge_list* e) { return e->el.entries.size(); }
uint64_t wbc_host_edges_self_loops(const wbc_edge_list* e) { return e->el.self_loops_dropped; }

void wbc_host_edges_get(const wbc_edge_list* e, uint64_t* u, uint64_t* v, double* w) {
  const auto& es = e->el.entries;
  for (size_t i = 0; i < es.size(); ++i) {
    u[i] = es[i].u;
    v[i] = es[i].v;
    w[i] = es[i].w;
  }
}

void wbc_host_edges_free(wbc_edge_list* e) { delete e; }

int wbc_host_gen_er(uint64_t n, double avg_degree, uint64_t seed, wbc_edge_list** out) {
  return guarded([&] { *out = new wbc_edge_list{wbc::gen_er(n, avg_degree, seed)}; });
}

int wbc_host_gen_kronecker(int scale, double avg_degree, uint64_t seed, wbc_edge_list** out) {
  return guarded([&] { *out = new wbc_edge_list{wbc::gen_kronecker(scale, avg_degree, seed)}; });
}

int wbc_host_gen_ba(uint64_t n, uint32_t m_per_node, uint64_t seed, wbc_edge_list** out) {
  return guarded([&] { *out = new wbc_edge_list{wbc::gen_ba(n, m_per_node, seed)}; });
}

int wbc_host_gen_grid(uint32_t rows, uint32_t cols, wbc_edge_list** out) {
  return guarded([&] { *out = new wbc_edge_list{wbc::gen_grid(rows, cols)}; });
}

int wbc_host_assign_weights(wbc_edge_list* e, int lo, int hi, uint64_t seed) {
  return guarded([&] { e->el = wbc::assign_weights(std::move(e->el), lo, hi, seed); });
}

int wbc_host_sample_sources(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out,
                            uint32_t* out_len) {
  return guarded([&] {
    const auto s = wbc::sample_sources(n, k, seed);
    if (!s.empty()) std::memcpy(out, s.data(), s.size() * 4);
    *out_len = static_cast<uint32_t>(s.size());
  });
}

int wbc_host_build_csr(const wbc_edge_list* e, wbc_csr** out) {
  return guarded([&] { *out = new wbc_csr{wbc::build_csr(e->el)}; });
}

void wbc_host_csr_dims(const wbc_csr* g, uint32_t* n, uint32_t* m, uint64_t* merged) {
  if (n) *n = g->g.n;
  if (m) *m = g->g.m;
  if (merged) *merged = g->g.merged_duplicates;
}

void wbc_host_csr_get(const wbc_csr* h, uint32_t* offsets, uint32_t* adjacency, double* weights,
                      uint32_t* edge_id, double* min_incident_weight, uint64_t* original_id,
                      uint32_t* edge_u, uint32_t* edge_v) {
  const wbc::CsrGraph& g = h->g;
  auto cp = [](void* dst, const auto& vec) {
    if (dst && !vec.empty()) std::memcpy(dst, vec.data(), vec.size() * sizeof(vec[0]));
  };
  cp(offsets, g.offsets);
  cp(adjacency, g.adjacency);
  cp(weights, g.weights);
  cp(edge_id, g.edge_id);
  cp(min_incident_weight, g.min_incident_weight);
  cp(original_id, g.original_id);
  cp(edge_u, g.edge_u);
  cp(edge_v, g.edge_v);
}

void wbc_host_csr_free(wbc_csr* g) { delete g; }

}  // extern "C"
