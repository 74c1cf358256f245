// wbc::bc_parallel drop-in (include/wbc/engine.hpp) over the C ABI.
//
// Option handling follows the reference exactly: strategy tokens and lane
// widths (engine.cpp:12-40), validate_strategy / workers >= 1
// (engine.cpp:110-114, 373-374), source range check (engine.cpp:349-361),
// empty source list / empty graph return zeros (engine.cpp:382-385),
// depth_per_source sized n (engine.cpp:379), Halved (engine.cpp:451-454).
// The GPU computes the same sums; the CPU schedule fields only validate.
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "wbc/engine.hpp"
#include "wbc_gpu.h"

namespace wbc {

bool valid_lane_width(int w) {
  switch (w) {
    case 1: case 4: case 8: case 16: case 32: return true;
    default: return false;
  }
}

std::string strategy_name(const Strategy& s) {
  const bool q = s.frontier_mode == FrontierMode::Queue;
  if (s.lane_width == 1) return q ? "we" : "np";
  return (q ? "we-warp" : "warp") + std::to_string(s.lane_width);
}

Strategy parse_strategy(const std::string& token) {
  if (token == "np") return {FrontierMode::ScanAll, 1};
  if (token == "we") return {FrontierMode::Queue, 1};
  Strategy s;
  std::string width;
  if (token.rfind("we-warp", 0) == 0) {
    s.frontier_mode = FrontierMode::Queue;
    width = token.substr(7);
  } else if (token.rfind("warp", 0) == 0) {
    s.frontier_mode = FrontierMode::ScanAll;
    width = token.substr(4);
  } else {
    throw std::invalid_argument("unknown strategy '" + token + "'");
  }
  s.lane_width = width.empty() ? 32 : std::atoi(width.c_str());
  if (!valid_lane_width(s.lane_width))
    throw std::invalid_argument("invalid lane width in strategy '" + token +
                                "' (expected 1, 4, 8, 16 or 32)");
  return s;
}

namespace {

[[noreturn]] void throw_status(int rc) {
  const std::string msg = wbc_gpu_last_error();
  if (rc == WBC_E_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void validate(const EngineOptions& opt) {
  if (!valid_lane_width(opt.strategy.lane_width))
    throw std::invalid_argument("invalid lane width " + std::to_string(opt.strategy.lane_width) +
                                " (expected 1, 4, 8, 16 or 32)");
  if (opt.workers < 1) throw std::invalid_argument("bc_parallel: workers must be >= 1");
  if (opt.settle_rule != SettleRule::StrictLess)
    throw std::invalid_argument(
        "bc_parallel: SettleRule::LessEqual is a CPU-only negative control (not run on GPU)");
}

}  // namespace

namespace {

// GpuOptions::device >= 0: that device.  -1: the devices listed in
// WBC_GPU_DEVICES ("0,1,2" -- repeats allowed, for tests -- or "all"), else
// every visible device.
std::vector<int> resolve_devices(int device) {
  if (device >= 0) return {device};
  int count = 0;
  if (wbc_gpu_device_count(&count) || count < 1) return {-1};  // fails loudly at create
  std::vector<int> out;
  const char* e = std::getenv("WBC_GPU_DEVICES");
  if (e && std::string(e) != "all") {
    std::stringstream ss(e);
    std::string tok;
    while (std::getline(ss, tok, ','))
      if (!tok.empty()) out.push_back(std::stoi(tok));
  }
  if (out.empty())
    for (int d = 0; d < count; ++d) out.push_back(d);
  return out;
}

}  // namespace

struct GpuBcEngine::Impl {
  wbc_gpu_graph* h = nullptr;   // one device
  wbc_gpu_multi* mh = nullptr;  // several devices: sources sharded, one all-reduce
  ~Impl() {
    if (mh)
      wbc_gpu_multi_destroy(mh);
    else
      wbc_gpu_graph_destroy(h);
  }
};

GpuBcEngine::GpuBcEngine(const CsrGraph& g, const GpuOptions& gpu)
    : impl_(std::make_unique<Impl>()), n_(g.n), m_(g.m) {
  const std::vector<int> devs = resolve_devices(gpu.device);
  const uint32_t* eid = g.edge_id.empty() ? nullptr : g.edge_id.data();
  int rc;
  if (devs.size() > 1) {
    rc = wbc_gpu_multi_create(g.n, g.m, g.offsets.data(), g.adjacency.data(), g.weights.data(),
                              g.min_incident_weight.data(), eid, devs.data(), static_cast<int>(devs.size()), 0,
                              &impl_->mh);
    if (rc) throw_status(rc);
    impl_->h = wbc_gpu_multi_device_graph(impl_->mh, 0);
  } else {
    rc = wbc_gpu_graph_create(g.n, g.m, g.offsets.data(), g.adjacency.data(), g.weights.data(),
                              g.min_incident_weight.data(), eid, devs[0], &impl_->h);
    if (rc) throw_status(rc);
  }
  if (gpu.threads_per_cta || gpu.max_slots)
    for (int i = 0; wbc_gpu_graph* dh = impl_->mh ? wbc_gpu_multi_device_graph(impl_->mh, i) : (i ? nullptr : impl_->h);
         ++i)
      wbc_gpu_set_tuning(dh, gpu.threads_per_cta, gpu.max_slots, 0, -1);
}

GpuBcEngine::~GpuBcEngine() = default;

BcResult GpuBcEngine::bc(const EngineOptions& opt) const {
  validate(opt);
  BcResult r;
  r.node_bc.assign(n_, 0.0);
  if (opt.compute_edge_bc) r.edge_bc.assign(m_, 0.0);
  r.depth_per_source.assign(n_, 0);
  uint32_t flags = 0;
  if (opt.normalization == Normalization::Halved) flags |= WBC_HALVED;
  if (opt.compute_edge_bc) flags |= WBC_EDGE_BC;
  if (opt.strict_merge) flags |= WBC_STRICT_MERGE | WBC_LANE_WIDTH(opt.strategy.lane_width);
  const NodeId* src = nullptr;
  std::uint64_t k = 0;
  if (opt.sources) {
    src = opt.sources->data();
    k = opt.sources->size();
    if (k == 0) return r;  // engine.cpp:382-385
  }
  double elapsed = 0.0;
  const int rc = impl_->mh ? wbc_gpu_multi_bc(impl_->mh, src, k, flags, r.node_bc.data(),
                                              opt.compute_edge_bc ? r.edge_bc.data() : nullptr,
                                              r.depth_per_source.data(), &elapsed)
                           : wbc_gpu_bc(impl_->h, src, k, flags, r.node_bc.data(),
                                        opt.compute_edge_bc ? r.edge_bc.data() : nullptr,
                                        r.depth_per_source.data(), &elapsed);
  if (rc) throw_status(rc);
  r.elapsed = std::chrono::duration<double>(elapsed);
  return r;
}

GpuBcEngine::SourceState GpuBcEngine::dump_source(NodeId s) const {
  SourceState st;
  st.dist.resize(n_);
  st.sigma.resize(n_);
  st.delta.resize(n_);
  const int rc =
      wbc_gpu_sssp_dump(impl_->h, s, st.dist.data(), st.sigma.data(), st.delta.data(), &st.depth);
  if (rc) throw_status(rc);
  return st;
}

BcResult bc_parallel(const CsrGraph& g, const EngineOptions& opt) {
  validate(opt);
  if (opt.sources)
    for (NodeId s : *opt.sources)
      if (s >= g.n) throw std::invalid_argument("bc_parallel: source id out of range");
  if (g.n == 0) return BcResult{};
  if (opt.sources) {
    if (opt.sources->empty()) {
      BcResult r;
      r.node_bc.assign(g.n, 0.0);
      if (opt.compute_edge_bc) r.edge_bc.assign(g.m, 0.0);
      r.depth_per_source.assign(g.n, 0);
      return r;
    }
  }
  GpuBcEngine engine(g);
  return engine.bc(opt);
}

}  // namespace wbc
