// wbc/generate.hpp -- synthetic inputs for the measurement configs.
//
// gen_er / gen_kronecker / assign_weights / sample_sources mirror
// /root/reference/proj/include/wbc/generate.hpp:10-35 and reproduce the
// reference's output streams exactly (same mt19937_64(splitmix64(seed ^
// splitmix64(stream))) derivation and the same libstdc++ distributions,
// generate.cpp:13-28).  gen_ba and gen_grid are new: the reference has no
// Barabasi-Albert or grid generator but BASELINE.json configs 2 and 4 need them.
#pragma once

#include <cstdint>

#include "wbc/graph.hpp"

namespace wbc {

struct KroneckerInitiator {
  double a = 0.57;
  double b = 0.19;
  double c = 0.19;
  double d = 0.05;
};

EdgeList gen_er(std::uint64_t n, double avg_degree, std::uint64_t seed);
EdgeList gen_kronecker(int scale, double avg_degree, std::uint64_t seed,
                       const KroneckerInitiator& init = {});
EdgeList assign_weights(EdgeList edges, int lo, int hi, std::uint64_t seed);
std::vector<NodeId> sample_sources(NodeId n, NodeId k, std::uint64_t seed);

/// Barabasi-Albert preferential attachment: an (m+1)-clique on ids 0..m, then
/// every new vertex t attaches to m distinct earlier vertices drawn from the
/// repeated-endpoint list (probability proportional to degree).  Edge count
/// is m(m+1)/2 + (n-m-1)*m.  Stream: topology stream of `seed`.
EdgeList gen_ba(std::uint64_t n, std::uint32_t m, std::uint64_t seed);

/// rows x cols 4-neighbour lattice, row-major ids; per cell the right edge is
/// emitted before the down edge.  Weights 1 (see assign_weights).
EdgeList gen_grid(std::uint32_t rows, std::uint32_t cols);

}  // namespace wbc
