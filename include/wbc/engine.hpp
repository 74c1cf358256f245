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
#include <span>
#include <string>
#include <vector>

#include "wbc/graph.hpp"
#include "wbc/result.hpp"

struct wbc_gpu_graph;  // wbc_gpu.h

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

/// Per-source working set, field for field the reference's
/// (engine.hpp:49-65).  Filled by solve_source below from one GPU run:
/// dist (+inf unreached), sigma, the Eq. 4 rounds as order / ends
/// (order[ends[k-1] .. ends[k]) is round k's settled set; the order *within*
/// a round is unspecified), unsettled = 1 exactly for unreached vertices,
/// the last round as the frontier, threshold = +inf.  delta is filled by
/// accumulate_dependencies.
struct TraversalState {
  std::vector<double> dist;
  std::vector<double> sigma;
  std::vector<double> delta;
  std::vector<std::uint8_t> unsettled;
  std::vector<std::uint8_t> in_frontier;
  std::vector<NodeId> frontier;
  std::uint32_t frontier_len = 0;
  std::vector<NodeId> order;
  std::uint32_t order_len = 0;
  std::vector<std::uint32_t> ends;
  std::uint32_t ends_len = 0;
  double threshold = 0.0;
  NodeId source = 0;

  std::uint32_t depth() const { return ends_len - 1; }
};

/// Resets st for a run from `source` exactly like the reference
/// (engine.cpp:118-142): d[s]=0, sigma[s]=1, s settled and the sole frontier
/// member, order=[s], ends=[0,1], threshold=0.  Host-side bookkeeping only.
void init_state(const CsrGraph& g, NodeId source, TraversalState& st);

/// The whole single-source phase (engine.cpp:214-222) on the GPU: one run of
/// the device pipeline for `source`, its distances, sigma and Eq. 4 rounds
/// copied into st.  strat is validated like the reference's; the GPU schedule
/// ignores it.  SettleRule::LessEqual (a CPU-only negative control) throws
/// std::invalid_argument.  The graph's device replica is shared with
/// bc_parallel's cache.
void solve_source(const CsrGraph& g, NodeId source, const Strategy& strat, TraversalState& st,
                  SettleRule rule = SettleRule::StrictLess);
/// Same as solve_source (the GPU team already cooperates on every round);
/// workers is validated (>= 1) and otherwise ignored.
void solve_source_parallel(const CsrGraph& g, NodeId source, const Strategy& strat, int workers,
                           TraversalState& st, SettleRule rule = SettleRule::StrictLess);

/// Brandes dependency accumulation for st.source (engine.cpp:183-212) on the
/// GPU: st.delta is filled, node_acc[w] += delta[w] for w != source and, when
/// edge_acc is non-empty, each DAG edge's term is added at its canonical id.
/// Empty spans skip the respective accumulation (the reference's contract).
/// The reference's round primitives relax_frontier / compute_threshold /
/// settle_and_advance are not provided: the GPU runs rounds on the device.
void accumulate_dependencies(const CsrGraph& g, const Strategy& strat, TraversalState& st,
                             std::span<double> node_acc, std::span<double> edge_acc = {});

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
/// every visible GPU (WBC_GPU_DEVICES overrides; under a one-process-per-GPU
/// launcher, WORLD_SIZE > 1 or LOCAL_RANK set, the current device only),
/// shards the sources across them and combines the partial BC with one NCCL
/// all-reduce.  The replica of the last graph is kept and reused while later
/// calls pass the same graph (content fingerprint); GpuBcEngine keeps a graph
/// resident explicitly.
/// settle_rule = LessEqual (a CPU-only negative control) is rejected with
/// std::invalid_argument.
BcResult bc_parallel(const CsrGraph& g, const EngineOptions& opt = {});

/// Frees the device replica bc_parallel keeps between calls.
void release_bc_parallel_cache();

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
  /// The C ABI handle of the first device's replica (wbc_gpu.h).
  wbc_gpu_graph* device_handle() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  NodeId n_ = 0;
  EdgeId m_ = 0;
};

}  // namespace wbc
