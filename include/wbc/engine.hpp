// wbc/engine.hpp -- the BC entry point, source-compatible with the reference.
//
// Mirrors the option/strategy surface of /root/reference/proj/include/wbc/
// engine.hpp (Strategy :14-29, parse_strategy :36-38, SettleRule :40-44,
// EngineOptions :108-120, bc_parallel :122-130).  bc_parallel here runs the
// per-source Brandes pipeline on a B200 through the C ABI in wbc_gpu.h; the
// CPU schedule knobs (strategy, workers) are validated exactly like the
// reference (engine.cpp:110-114,373-374) but do not change the GPU schedule --
// results are schedule-independent by the reference's own contract
// (engine.hpp:127-129).  strict_merge = true commits sources in list order and
// sums each delta in the reference's slot order with strategy.lane_width
// lanes: node/edge BC are then bitwise the reference's bc_parallel output
// (WBC_STRICT_MERGE).
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "wbc/graph.hpp"
#include "wbc/result.hpp"

namespace wbc {

enum class FrontierMode { ScanAll, Queue };

struct Strategy {
  FrontierMode frontier_mode = FrontierMode::Queue;
  int lane_width = 1;  // one of 1, 4, 8, 16, 32
};

bool valid_lane_width(int w);
std::string strategy_name(const Strategy& s);
Strategy parse_strategy(const std::string& token);

enum class SettleRule { StrictLess, LessEqual };

struct EngineOptions {
  Strategy strategy{};
  int workers = 1;
  bool compute_edge_bc = false;
  Normalization normalization = Normalization::Raw;
  bool strict_merge = false;
  SettleRule settle_rule = SettleRule::StrictLess;
  std::optional<std::vector<NodeId>> sources;
};

/// GPU knobs live outside the reference's option struct.
struct GpuOptions {
  int device = -1;          // >= 0: that device; -1: WBC_GPU_DEVICES ("0,1,..." or "all"),
                            //   else every visible device (sources sharded, one all-reduce)
  int threads_per_cta = 0;  // 0: automatic
  int max_slots = 0;        // 0: automatic (resident sources per GPU)
};

/// Drop-in for wbc::bc_parallel (reference engine.cpp:372-457).  Uploads g to
/// every visible GPU (or WBC_GPU_DEVICES) on each call, shards the sources
/// across them and combines the partial BC with one NCCL all-reduce; use
/// GpuBcEngine to keep the graph resident.
/// settle_rule = LessEqual (a CPU-only negative control) is rejected with
/// std::invalid_argument.
BcResult bc_parallel(const CsrGraph& g, const EngineOptions& opt = {});

/// Resident-graph engine: one upload, many bc() calls.
class GpuBcEngine {
 public:
  explicit GpuBcEngine(const CsrGraph& g, const GpuOptions& gpu = {});
  ~GpuBcEngine();
  GpuBcEngine(const GpuBcEngine&) = delete;
  GpuBcEngine& operator=(const GpuBcEngine&) = delete;

  BcResult bc(const EngineOptions& opt = {}) const;

  struct SourceState {
    std::vector<double> dist, sigma, delta;
    std::uint32_t depth = 0;
  };
  /// One source's final dist / sigma / delta (parity debugging).
  SourceState dump_source(NodeId s) const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  NodeId n_ = 0;
  EdgeId m_ = 0;
};

}  // namespace wbc
