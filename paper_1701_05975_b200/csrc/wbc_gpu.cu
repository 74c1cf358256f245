// wbc_gpu.cu -- the C ABI (include/wbc_gpu.h) over the sm_100a kernels.
//
// Owns the device CSR replica and the per-slot workspaces; validates the
// reference's argument contract (engine.cpp:349-361,372-385) at the boundary;
// launches the persistent per-source kernel (bc_kernels.cuh) on the caller's
// stream.  No CPU fallback exists: without a device every entry point fails
// with WBC_E_CUDA / WBC_E_NOT_BUILT.
//
// Device layout: vertices are relabelled by degree, highest
// first (ties by id), each row's slots sorted by relabelled neighbour, and a
// slot is one u32 (neighbour << wbits | weight) when it fits, else a uint2.
// Results are mapped back to the caller's dense ids on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "bc_flat.cuh"
#include "bc_kernels.cuh"
#include "bc_team.cuh"
#include "wbc_gpu.h"

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define WBC_CUDA_TRY(expr)                                                                  \
  do {                                                                                      \
    const cudaError_t err_ = (expr);                                                        \
    if (err_ != cudaSuccess)                                                                \
      return set_error(err_ == cudaErrorMemoryAllocation ? WBC_E_NOMEM : WBC_E_CUDA,        \
                       std::string(#expr) + ": " + cudaGetErrorString(err_));               \
  } while (0)

template <class T>
T* dev_alloc(size_t count, cudaError_t& err) {
  void* p = nullptr;
  err = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  return static_cast<T*>(p);
}

uint32_t bits_for(uint64_t x) {  // bits needed to store values 0..x
  uint32_t b = 1;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

template <class F>
void parallel_for(uint64_t n, F&& f) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536 || hw == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  const uint64_t chunk = (n + hw - 1) / hw;
  for (unsigned t = 0; t < hw; ++t) {
    const uint64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b < e) ts.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& t : ts) t.join();
}

}  // namespace

namespace wbc_host {
// The host layer (host_capi.cpp) reports through the same thread-local slot.
int set_error(int code, const std::string& msg) { return ::set_error(code, msg); }
}  // namespace wbc_host

struct LaunchShape {
  uint32_t near_width = 0; // 0: the graph's automatic width
  bool flat = false;       // bc_flat_kernel (CTA per source, distance-first; team fallback)
  int cluster = 0;         // 0: per-CTA kernel; else CTAs per team (team kernel, 1024 threads)
  int threads = 128;
  uint32_t hot = 0;        // vertices with shared-memory distances
  uint32_t l2hot = 0;      // vertices whose distance accesses carry an evict-last hint
  size_t dyn_smem = 0;     // bytes
  uint32_t flat_sq = 0;    // flat kernel: shared-memory near-queue entries per buffer
};

struct wbc_gpu_graph {
  int device = 0;
  uint32_t n = 0, m = 0;
  uint32_t max_weight = 0;
  bool packed = true;
  uint32_t wbits = 0;
  uint32_t near_width = 1;
  int sm_count = 0;
  int smem_per_sm = 0;
  int smem_optin = 0;
  double hot_coverage_25k = 0;  // share of neighbour accesses landing on the top 25K ids
  bool skewed = false;          // heavy-tailed degrees: max degree >= 16 x average
  // device CSR replica (relabelled ids)
  uint32_t* d_offsets = nullptr;
  uint32_t* d_slots32 = nullptr;
  uint2* d_slots64 = nullptr;
  uint32_t* d_minw = nullptr;
  uint32_t* d_edge_id = nullptr;
  // the same rows in the caller's slot order (strict merge: the reference's
  // summation order, engine.cpp:193-206)
  uint32_t* d_ref_slots32 = nullptr;
  uint2* d_ref_slots64 = nullptr;
  uint32_t* d_ref_edge_id = nullptr;
  double* d_stage = nullptr;  // strict batches: per-source delta rows, then edge rows
  uint64_t stage_bytes = 0;
  uint32_t* d_perm = nullptr;  // device id -> caller id
  uint32_t* d_inv = nullptr;   // caller id -> device id
  std::vector<uint32_t> perm;  // host copy
  uint64_t graph_bytes = 0;
  // workspace
  int ws_slots = 0;
  void* d_ws = nullptr;
  uint64_t ws_bytes = 0;
  wbc_dev::Workspace ws{};
  bool last_flat = false;     // the last run used bc_flat_kernel
  // ELL copy of the rows for bc_flat_kernel (flat graphs only): per vertex a
  // record of flat_ke slots and flat_ke sweep keys (weight + minw(neighbour)),
  // and the slots' canonical edge ids
  int flat_ke = 0;
  uint32_t* d_ell = nullptr;
  uint32_t* d_ell_eid = nullptr;
  int fill = 0;               // 2-CTA fill clusters beside a C >= 4 team launch
  // launch decisions are cached until a tuning knob changes
  uint64_t tune_gen = 1, shape_gen = 0, ws_gen = 0;
  LaunchShape shape_cache{};
  int ws_want = -1, ws_slots_cached = 0;
  int ws_shape_key = -1;      // launch shape the workspace was carved for
  int tune_fill = -1;         // -1 auto (the fill teams' distances fit the L2 budget), 0 off, 1 on
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  unsigned long long* d_counter = nullptr;
  unsigned int* d_overflow = nullptr;
  unsigned long long* d_prof = nullptr;
  double* d_node_dev = nullptr;  // device-id partial BC of the current run
  // scratch for host-buffer runs
  double* d_node = nullptr;
  double* d_edge = nullptr;
  uint32_t* d_depth = nullptr;
  uint32_t* d_sources = nullptr;
  uint64_t d_sources_cap = 0;
  // tuning
  int tune_threads = 0;
  int tune_slots = 0;
  int64_t tune_hot = -1;
  int64_t tune_l2hot = -1;
  bool tune_near = false;      // near_width set explicitly (else the launch shape may adjust it)
  int tune_flat = -1;          // -1 auto (flat, large graphs), 0 off, 1 wherever eligible
  uint32_t tune_flat_delta = 0;  // near-far window of bc_flat_kernel (0: max weight)
  int tune_flat_threads = 0;     // bc_flat_kernel CTA size (0: kFlatT)
  int tune_flat_sq = -1;         // bc_flat_kernel shared-memory near-queue entries per buffer (-1: auto)
  uint32_t max_degree = 0, max_minw = 0;
  bool symmetric = false;
  int scale_k = 0;             // weights scaled by 2^scale_k to integers (dumps scale distances back)
  wbc_dev::FlatWs fw{};
  int tune_cluster = -1;       // -1 auto, 0 per-CTA kernel, else team kernel with this cluster size
  bool ws_team = false;        // workspace carries the team-kernel arrays
  bool profiling = false;
  uint64_t stats[4] = {0, 0, 0, 0};
  std::string last_kernel;
  uint64_t prof_host[wbc_dev::kProfCounters] = {};

  ~wbc_gpu_graph() {
    cudaSetDevice(device);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    for (void* p : {(void*)d_offsets, (void*)d_slots32, (void*)d_slots64, (void*)d_minw,
                    (void*)d_edge_id, (void*)d_perm, (void*)d_inv, d_ws, (void*)d_counter,
                    (void*)d_ell, (void*)d_ell_eid,
                    (void*)d_overflow, (void*)d_prof, (void*)d_node_dev, (void*)d_node,
                    (void*)d_edge, (void*)d_depth, (void*)d_sources, (void*)d_ref_slots32,
                    (void*)d_ref_slots64, (void*)d_ref_edge_id, (void*)d_stage})
      cudaFree(p);
  }
};

namespace {

using KernelFn = void (*)(const wbc_dev::RunParams);

template <bool PACKED, bool PROF>
KernelFn pick_kernel_t(int threads) {
  using namespace wbc_dev;
  if (threads <= 128) return bc_sources_kernel<128, PACKED, PROF>;
  if (threads <= 256) return bc_sources_kernel<256, PACKED, PROF>;
  if (threads <= 512) return bc_sources_kernel<512, PACKED, PROF>;
  return bc_sources_kernel<1024, PACKED, PROF>;
}

KernelFn pick_kernel(int threads, bool packed, bool prof = false) {
  if (packed) return prof ? pick_kernel_t<true, true>(threads) : pick_kernel_t<true, false>(threads);
  return prof ? pick_kernel_t<false, true>(threads) : pick_kernel_t<false, false>(threads);
}

template <bool PACKED, bool PROF>
KernelFn pick_team_t(int c, int threads) {
  using namespace wbc_dev;
  if (threads <= 32) return bc_team_kernel<32, 1, PACKED, PROF>;
  switch (c) {
    case 1: return bc_team_kernel<1024, 1, PACKED, PROF>;
    case 2: return bc_team_kernel<1024, 2, PACKED, PROF>;
    case 4: return bc_team_kernel<1024, 4, PACKED, PROF>;
    case 8: return bc_team_kernel<1024, 8, PACKED, PROF>;
#ifdef WBC_TEAM_ODD_CLUSTERS
    case 6: return bc_team_kernel<1024, 6, PACKED, PROF>;
    case 9: return bc_team_kernel<1024, 9, PACKED, PROF>;
    case 12: return bc_team_kernel<1024, 12, PACKED, PROF>;
#endif
    default: return bc_team_kernel<1024, 16, PACKED, PROF>;
  }
}

KernelFn pick_team(int c, int threads, bool packed, bool prof = false) {
  if (packed) return prof ? pick_team_t<true, true>(c, threads) : pick_team_t<true, false>(c, threads);
  return prof ? pick_team_t<false, true>(c, threads) : pick_team_t<false, false>(c, threads);
}


// Launch shape policy:
//  * small graphs (n*4 <= 24 KB): every distance in shared memory, 128-thread
//    CTAs, many sources in flight;
//  * skewed graphs (the top 25K ids take >= 40% of neighbour accesses: R-MAT,
//    BA): 512-thread CTAs for the large frontiers;
//  * flat graphs (grid, sparse ER): 128-thread CTAs, many sources in flight;
//    the per-round latency dominates.
// Unless tuned, the shared-memory distance cache gets exactly the shared
// memory left over at the register-limited occupancy, so it never costs
// resident sources.
LaunchShape pick_shape_uncached(const wbc_gpu_graph* g);

LaunchShape pick_shape(wbc_gpu_graph* g);

// In-flight distance arrays of the team kernel's resident sources, summed:
// kept near the 126 MB L2 (launch-shape policy below).
constexpr uint64_t kTeamL2Budget = 128ULL << 20;

// Largest power-of-two denominator of a dyadic weight (prepare_host).
constexpr int kMaxWeightScaleBits = 20;

// bc_flat_kernel: CTA size (two CTAs per SM: its phases are latency-bound)
constexpr int kFlatT = 1024;  // default; set_param("flat_threads", 256 | 512 | 1024)

using FlatFn = void (*)(const wbc_dev::RunParams, const wbc_dev::FlatWs);
FlatFn pick_flat(int threads, int ke) {
  using namespace wbc_dev;
  if (threads <= 256) return ke == 4 ? bc_flat_kernel<256, 4> : bc_flat_kernel<256, 8>;
  if (threads <= 512) return ke == 4 ? bc_flat_kernel<512, 4> : bc_flat_kernel<512, 8>;
  return ke == 4 ? bc_flat_kernel<1024, 4> : bc_flat_kernel<1024, 8>;
}

// bc_flat_kernel's bucket array: a power of two > max weight + max minw + 1.
uint32_t flat_buckets(const wbc_gpu_graph* g) {
  uint32_t b = 32;
  while (b < static_cast<uint64_t>(g->max_weight) + g->max_minw + 2) b <<= 1;
  return b;
}

// window width of bc_flat_kernel's near-far SSSP
uint32_t flat_delta(const wbc_gpu_graph* g) {
  const uint32_t d = g->tune_flat_delta ? g->tune_flat_delta : std::max<uint32_t>(1, g->max_weight);
  return std::min<uint32_t>(d, wbc_dev::kFlatBuckets);
}
uint32_t flat_delta_words(const wbc_gpu_graph* g) { return (flat_delta(g) + 31) / 32 * 32; }

bool flat_eligible(const wbc_gpu_graph* g) {
  // the ELL copy exists (packed slots, degree <= 8, mirror-image rows: the
  // pull passes read a DAG edge from either end), the sweep keys fit the
  // shared-memory ring, and threshold keys stay below 2^32
  return g->n > 0 && g->d_ell && flat_buckets(g) <= static_cast<uint32_t>(wbc_dev::kFlatBuckets) &&
         (uint64_t{g->n} - 1) * g->max_weight + 2ULL * flat_buckets(g) < 0xFFFFFFFFULL;
}

LaunchShape pick_shape_uncached(const wbc_gpu_graph* g) {
  LaunchShape s;
  // Flat, large-diameter graphs (grid / road-like, degree <= 8, n >= 2^18)
  // take the distance-first kernel: grid-2048 x 1024 sources 2.98 s vs 5.4 s
  // for one-warp Eq. 4 teams, grid-512 2.93 vs 2.70 GTEPS; smaller graphs keep
  // the teams, which fit every source in flight (grid-128: 2.08 vs 0.52).
  const bool auto_flat = g->tune_flat < 0 && g->tune_cluster < 0 && g->tune_threads == 0 &&
                         !g->skewed && g->n >= (1u << 18);
  if ((g->tune_flat > 0 || auto_flat) && flat_eligible(g)) {
    s.flat = true;
    s.threads = g->tune_flat_threads ? (g->tune_flat_threads <= 256 ? 256 : g->tune_flat_threads <= 512 ? 512 : 1024)
                                     : kFlatT;
    s.dyn_smem = wbc_dev::flat_dyn_smem(flat_delta_words(g), flat_buckets(g), g->flat_ke);
    // the near queues' first entries live in shared memory (two buffers),
    // sized to the room left below the 64 KB carveout step: more shared
    // memory would shrink L1, which the kernel needs more
    const size_t used = s.dyn_smem + wbc_dev::flat_static_smem(s.threads) + 1024;
    const size_t room = used < wbc_dev::kFlatSmemStep ? (wbc_dev::kFlatSmemStep - used) / 8 : 0;
    const size_t want = g->tune_flat_sq >= 0 ? static_cast<size_t>(g->tune_flat_sq) : wbc_dev::kFlatSQ;
    s.flat_sq = static_cast<uint32_t>(std::min(want, g->tune_flat_sq >= 0 ? want : room) / 32 * 32);
    s.dyn_smem += size_t{2} * s.flat_sq * 4;
    return s;
  }
  const uint64_t n = g->n;
  const bool tiny = n * 4 <= 24 * 1024;
  if (g->tune_cluster > 0) {
    s.cluster = g->tune_cluster <= 1 ? 1 : g->tune_cluster <= 2 ? 2 : g->tune_cluster <= 4 ? 4
              : g->tune_cluster <= 8 ? 8 : 16;
#ifdef WBC_TEAM_ODD_CLUSTERS
    if (g->tune_cluster == 6 || g->tune_cluster == 9 || g->tune_cluster == 12) s.cluster = g->tune_cluster;
#endif
    s.threads = (s.cluster == 1 && g->tune_threads > 0 && g->tune_threads <= 32) ? 32 : 1024;
    s.dyn_smem = wbc_dev::team_dyn_smem(s.threads);
    return s;
  }
  // Skewed graphs run on the team kernel (bc_team.cuh), with the smallest
  // cluster whose in-flight distance arrays stay near L2 size: one CTA per
  // source while 148 of them fit in 64 MB (BA-65536: 27.5 vs 18.0 GTEPS for
  // the per-CTA kernel), else the smallest C in {2,4,8,16} with
  // (148/C) * 4n <= kTeamL2Budget (R-MAT-20: C=4 with 2-CTA fill teams on
  // the SMs 4-CTA clusters strand, 48.6 vs 46.3 GTEPS at C=2; R-MAT-24: C=16,
  // 34.0 vs 31.9 at C=8 and 21.8 at C=2).  Measured on B200, DESIGN.md §4.
  if (g->tune_cluster < 0 && !tiny && g->skewed) {
    const uint64_t per = n * 4;
    int c = 1;
    if (per * static_cast<uint64_t>(g->sm_count) > (64ULL << 20)) {
      c = 2;
      while (c < 16 && per * static_cast<uint64_t>(g->sm_count / c) > kTeamL2Budget) c *= 2;
    }
    s.cluster = c;
    s.threads = 1024;
    s.dyn_smem = wbc_dev::team_dyn_smem(s.threads);
    // near window (weights up to 255): 6 for single-CTA teams (BA 33.0 vs 32.8
    // at 8, 32.5 at 10, 32.2 at 12, 28.7 at 2), 12 for clusters (R-MAT-20 at
    // C = 4: 51.4 vs 51.1-51.3 at 10-16, 50.5 at 20; R-MAT-24: 35.3 vs 35.2 at
    // 8, 34.8 at 16)
    if (!g->tune_near) s.near_width = c >= 2 ? 12 : 6;
    return s;
  }
  // Flat, large graphs (grid / road-like: latency-bound rounds, small
  // frontiers): one warp per source (grid-2048: 1.56 vs 1.1 GTEPS for the
  // 128-thread per-CTA kernel).  Tiny graphs keep the per-CTA kernel with
  // every distance in shared memory (ER-4096: 14.3 vs 11.8).
  if (g->tune_cluster < 0 && !tiny && g->tune_threads == 0) {
    s.cluster = 1;
    s.threads = 32;
    s.dyn_smem = wbc_dev::team_dyn_smem(s.threads);
    return s;
  }
  const void* fn = reinterpret_cast<const void*>(pick_kernel(s.threads, g->packed));
  cudaFuncAttributes attr{};
  cudaFuncGetAttributes(&attr, fn);
  const uint64_t cap = (static_cast<uint64_t>(g->smem_optin) - attr.sharedSizeBytes) / 4;
  uint64_t hot;
  if (g->tune_hot >= 0) {
    hot = static_cast<uint64_t>(g->tune_hot);
  } else if (tiny) {
    hot = n;
  } else if (s.threads >= 1024) {
    hot = 0;  // measured: the L2-hinted global path beats a shared-memory cache here
  } else {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, s.threads, 0);
    per_sm = std::max(1, per_sm);
    const int64_t per_cta = static_cast<int64_t>(g->smem_per_sm) / per_sm - 1024 -
                            static_cast<int64_t>(attr.sharedSizeBytes);
    hot = per_cta > 0 ? static_cast<uint64_t>(per_cta) / 4 / 256 * 256 : 0;
  }
  hot = std::min<uint64_t>(std::min<uint64_t>(hot, n), cap);
  s.hot = static_cast<uint32_t>(hot);
  s.dyn_smem = hot * 4;
  return s;
}

LaunchShape pick_shape(wbc_gpu_graph* g) {
  if (g->shape_gen != g->tune_gen) {
    g->shape_cache = pick_shape_uncached(g);
    g->shape_gen = g->tune_gen;
  }
  return g->shape_cache;
}

// Per-slot workspace bytes of each kernel family.
uint64_t ws_ns(const wbc_gpu_graph* g) { return round_up(uint64_t{g->n} + 2, 64); }
uint64_t ws_dcap(const wbc_gpu_graph* g) {
  const uint64_t n = g->n;
  return round_up(n + n / 2 + 1024, 64);
}
// bc_flat_kernel's per-source arrays: n_stride rounded to the
// sweep ring's chunk, so a chunk copy never leaves the slot
uint64_t flat_ns(const wbc_gpu_graph* g) { return round_up(uint64_t{g->n} + 2, wbc_dev::kFlatChunk); }
uint64_t ws_flat_per_slot(const wbc_gpu_graph* g) {
  const uint64_t ke = static_cast<uint64_t>(std::max(4, g->flat_ke));
  const uint64_t bufs = 2 * wbc_dev::kSweepers;  // sweep inputs: two buffers per sweeper warp
  return flat_ns(g) * (8 + 4 + bufs * 4 + 4 + 16 + 8 + 8 + 4 + 4 * ke + bufs * 4 * ke);
}

void carve_flat(wbc_gpu_graph* g, char* p, uint64_t slots) {
  const uint64_t ns = flat_ns(g), ke = static_cast<uint64_t>(std::max(4, g->flat_ke));
  auto carve = [&](uint64_t bytes) {
    char* q = p;
    p += bytes * slots;
    return q;
  };
  wbc_dev::FlatWs& w = g->fw;
  w.n_stride = ns;
  w.dp = reinterpret_cast<uint2*>(carve(ns * 8));
  w.psig = reinterpret_cast<double*>(carve(ns * 8));
  w.pcoef = reinterpret_cast<double*>(carve(ns * 8));
  w.psucc = reinterpret_cast<uint32_t*>(carve(ns * 4 * ke));
  const uint64_t bufs = 2 * wbc_dev::kSweepers;
  w.ent = reinterpret_cast<uint32_t*>(carve(bufs * ns * 4 * ke));  // two buffers per sweeper
  w.order = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.ord_d = reinterpret_cast<uint32_t*>(carve(bufs * ns * 4));
  w.mem = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.q0 = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.q1 = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.q2 = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.q3 = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.pinfo = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.ell = g->d_ell;
  w.ell_eid = g->d_ell_eid;
  w.delta_w = flat_delta(g);
  w.buckets = flat_buckets(g);
  w.delta_words = flat_delta_words(g);
}

uint64_t ws_per_slot(const wbc_gpu_graph* g, bool team, bool one_warp = false) {
  const uint64_t ns = ws_ns(g);
  // one-warp teams compact their queues in place (a step reads its entries
  // before it writes, and writes never pass reads): no second buffers
  return ns * (4 + 8 + 8 + 4 + 4 + 4 + 4 + 4 + (team ? (one_warp ? 12 : 20) : 0)) + ws_dcap(g) * 8;
}

wbc_dev::Workspace carve_cta_team(const wbc_gpu_graph* g, char* p, uint64_t slots, bool team,
                                  bool one_warp = false) {
  const uint64_t ns = ws_ns(g), dag_cap = ws_dcap(g);
  auto carve = [&](uint64_t bytes) {
    char* q = p;
    p += bytes * slots;
    return q;
  };
  wbc_dev::Workspace w{};
  w.n_stride = ns;
  w.dag_cap = dag_cap;
  w.sigma = reinterpret_cast<double*>(carve(ns * 8));
  w.delta = reinterpret_cast<double*>(carve(ns * 8));
  w.dag = reinterpret_cast<uint2*>(carve(dag_cap * 8));
  w.dist = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.order = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.level_ends = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.near_q = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.far_q = reinterpret_cast<uint32_t*>(carve(ns * 4));
  w.dag_ends = reinterpret_cast<uint32_t*>(carve(ns * 4));
  if (team) {
    w.ord_d = reinterpret_cast<uint32_t*>(carve(ns * 4));
    w.ord_row = reinterpret_cast<uint32_t*>(carve(ns * 4));
    w.epref = reinterpret_cast<uint32_t*>(carve(ns * 4));
    w.near_q2 = one_warp ? w.near_q : reinterpret_cast<uint32_t*>(carve(ns * 4));
    w.far_q2 = one_warp ? w.far_q : reinterpret_cast<uint32_t*>(carve(ns * 4));
  }
  return w;
}

int ensure_bytes(wbc_gpu_graph* g, uint64_t bytes) {
  if (g->d_ws && g->ws_bytes >= bytes) return WBC_OK;
  cudaFree(g->d_ws);
  g->d_ws = nullptr;
  g->ws_bytes = 0;
  void* base = nullptr;
  const cudaError_t err = cudaMalloc(&base, bytes);
  if (err != cudaSuccess)
    return set_error(WBC_E_NOMEM, "workspace allocation of " + std::to_string(bytes) +
                                      " bytes failed: " + cudaGetErrorString(err));
  g->d_ws = base;
  g->ws_bytes = bytes;
  return WBC_OK;
}

// Ensure a workspace for `want` slots exists (shape-dependent occupancy).
int ensure_workspace(wbc_gpu_graph* g, int want, const LaunchShape& shape, int* slots_out) {
  // same knobs, same request, layout still carved: nothing to query or carve
  const int shape_key = shape.cluster * 8192 + shape.threads * 4 + (shape.flat ? 2 : 0) + static_cast<int>(shape.flat_sq) * 65536;
  if (g->d_ws && g->ws_gen == g->tune_gen && g->ws_want == want && g->ws_shape_key == shape_key) {
    *slots_out = g->ws_slots_cached;
    return WBC_OK;
  }
  g->ws_gen = 0;
  const bool team = shape.cluster > 0;
  const bool one_warp = team && shape.cluster == 1 && shape.threads <= 32;
  const uint64_t per_slot = shape.flat ? ws_flat_per_slot(g) : ws_per_slot(g, team, one_warp);
  int slots = 0;
  if (shape.flat) {
    const void* f = reinterpret_cast<const void*>(pick_flat(shape.threads, g->flat_ke));
    WBC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shape.dyn_smem)));
    int per_sm = 0;
    WBC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, shape.threads, shape.dyn_smem));
    if (per_sm < 1) return set_error(WBC_E_CUDA, "flat kernel does not fit on an SM");
    slots = per_sm * g->sm_count;
  }
  if (team) {
    for (const bool prof : {false, true}) {
      const void* f = reinterpret_cast<const void*>(pick_team(shape.cluster, shape.threads, g->packed, prof));
      if (shape.cluster > 8)
        WBC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      WBC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(shape.dyn_smem)));
    }
    {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = shape.cluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(shape.cluster * g->sm_count, 1, 1);
      cfg.blockDim = dim3(shape.threads, 1, 1);
      cfg.dynamicSmemBytes = shape.dyn_smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int clusters = 0;
      const void* fk = reinterpret_cast<const void*>(pick_team(shape.cluster, shape.threads, g->packed));
      if (shape.cluster == 1) {  // plain launch: resident CTAs per SM x SMs
        WBC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&clusters, fk, shape.threads, shape.dyn_smem));
        clusters *= g->sm_count;
      } else {
        WBC_CUDA_TRY(cudaOccupancyMaxActiveClusters(&clusters, fk, &cfg));
      }
      if (clusters < 1) return set_error(WBC_E_CUDA, "team kernel: no cluster of this size fits");
      slots = clusters;
    }
  } else if (!shape.flat) {
    const KernelFn fn = pick_kernel(shape.threads, g->packed);
    for (const bool prof : {false, true})
      WBC_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(pick_kernel(shape.threads, g->packed, prof)),
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(shape.dyn_smem)));
    int per_sm = 0;
    WBC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, reinterpret_cast<const void*>(fn), shape.threads, shape.dyn_smem));
    if (per_sm < 1) return set_error(WBC_E_CUDA, "kernel does not fit on an SM with this launch shape");
    slots = per_sm * g->sm_count;
  }
  if (g->tune_slots) slots = std::min(slots, g->tune_slots);
  slots = std::max(1, std::min(slots, want));
  // Clusters of 4..16 CTAs strand the SMs no such cluster fits on (7 x 16
  // CTAs leave 36 of 148 SMs idle): a concurrent launch of 2-CTA clusters
  // fills them, sharing the source counter.
  int fill = 0;
  if (team && shape.cluster >= 4 && g->tune_fill != 0 && want > slots) {
    fill = std::max(0, (g->sm_count - slots * shape.cluster) / 2);
    fill = std::min<int>(fill, want - slots);
    // auto: only while every in-flight distance array still fits the L2
    // budget (R-MAT-20 C=4: 33 + 8 teams x 2.6 MB, 48.6 vs 44.9 GTEPS without
    // the fill; R-MAT-24 C=8: 27.2 vs 31.9 -- the extra teams thrash L2)
    if (g->tune_fill < 0 && uint64_t(slots + fill) * g->n * 4 > kTeamL2Budget) fill = 0;
    if (g->tune_fill > 1) fill = std::min(fill, g->tune_fill - 1);  // tests / experiments: at most fill - 1 teams
    if (fill > 0)
      for (const bool prof : {false, true})
        WBC_CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(pick_team(2, shape.threads, g->packed, prof)),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(shape.dyn_smem)));
  }
  size_t free_b = 0, total_b = 0;
  WBC_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  uint64_t avail = free_b + (g->d_ws ? g->ws_bytes : 0);
  const uint64_t reserve = (4ULL << 30) + total_b / 10;  // 4 GiB + 10% headroom
  avail = avail > reserve ? avail - reserve : 0;
  slots = static_cast<int>(std::min<uint64_t>(slots, std::max<uint64_t>(1, avail / per_slot)));
  fill = static_cast<int>(std::min<uint64_t>(fill, avail / per_slot - std::min<uint64_t>(avail / per_slot, slots)));
  g->fill = fill;
  int rc = ensure_bytes(g, per_slot * (slots + fill));
  if (rc) return rc;
  *slots_out = slots;
  char* base = static_cast<char*>(g->d_ws);
  g->last_flat = shape.flat;
  if (shape.flat) {
    carve_flat(g, static_cast<char*>(g->d_ws), slots);
    g->ws_slots = slots;
    g->ws_team = false;
  } else {
    g->ws = carve_cta_team(g, base, slots + fill, team, one_warp);
    g->ws_slots = slots;
    g->ws_team = team;
  }
  g->ws_gen = g->tune_gen;
  g->ws_want = want;
  g->ws_slots_cached = slots;
  g->ws_shape_key = shape_key;
  return WBC_OK;
}

// Lane width of a strict-merge request (0: not strict); validates it like
// validate_strategy (engine.cpp:110-114).
int strict_lanes_of(uint32_t flags, uint32_t* lanes) {
  *lanes = 0;
  if (!(flags & WBC_STRICT_MERGE)) return WBC_OK;
  uint32_t w = (flags >> 8) & 0xFFu;
  if (w == 0) w = 1;
  if (w != 1 && w != 4 && w != 8 && w != 16 && w != 32)
    return set_error(WBC_E_INVALID, "invalid lane width " + std::to_string(w) + " (expected 1, 4, 8, 16 or 32)");
  *lanes = w;
  return WBC_OK;
}

int launch_grid(uint64_t len) { return static_cast<int>(std::min<uint64_t>((len + 255) / 256, 4096)); }

// Enqueue one run: d_sources may be null (all vertices).  Accumulates node BC
// (caller ids) into d_node, edge BC into d_edge; writes depth of run sources.
int launch_strict(wbc_gpu_graph* g, const LaunchShape& shape, int slots, wbc_dev::RunParams p, uint64_t k,
                  bool edge_bc, double* d_edge, uint32_t lanes, cudaStream_t stream);

int launch_run(wbc_gpu_graph* g, const uint32_t* d_sources, uint64_t k, bool edge_bc,
               double* d_node, double* d_edge, uint32_t* d_depth, cudaStream_t stream,
               bool single_slot, bool keep_state, uint32_t strict_lanes = 0) {
  g->stats[3] = 0;
  if (k == 0 || g->n == 0) return WBC_OK;
  LaunchShape shape = pick_shape(g);
  if (shape.flat && (single_slot || strict_lanes)) {
    // dumps and strict merges run on one-warp teams (their layouts / row-scan backward)
    shape = LaunchShape{};
    shape.cluster = 1;
    shape.threads = 32;
    shape.dyn_smem = wbc_dev::team_dyn_smem(32);
  }
  if (strict_lanes && shape.cluster == 0) {
    // strict merge runs on the team kernel (its row-scan backward)
    shape = LaunchShape{};
    shape.cluster = 1;
    shape.threads = g->skewed ? 1024 : 32;
    shape.dyn_smem = wbc_dev::team_dyn_smem(shape.threads);
  }
  const int want = single_slot ? 1 : static_cast<int>(std::min<uint64_t>(k, 1u << 30));
  int slots = 0;
  int rc = ensure_workspace(g, want, shape, &slots);
  if (rc) return rc;
  if (single_slot) slots = 1;
  wbc_dev::RunParams p{};
  p.g.n = g->n;
  p.g.m = g->m;
  p.g.offsets = g->d_offsets;
  p.g.slots32 = g->d_slots32;
  p.g.slots64 = g->d_slots64;
  p.g.minw = g->d_minw;
  p.g.edge_id = g->d_edge_id;
  p.g.wbits = g->wbits;
  p.g.wmask = g->wbits >= 32 ? 0xFFFFFFFFu : ((1u << g->wbits) - 1);
  p.g.long_rows = g->n && 2ULL * g->m >= 32ULL * g->n;
  p.ws = g->ws;
  p.sources = d_sources;
  p.k = k;
  p.counter = g->d_counter;
  p.node_bc = g->d_node_dev;
  p.edge_bc = edge_bc ? d_edge : nullptr;
  p.depth = d_depth;
  p.near_width = shape.near_width ? shape.near_width : g->near_width;
  p.overflow = g->d_overflow;
  p.keep_state = keep_state ? 1 : 0;
  p.inv = g->d_inv;
  p.hot = shape.hot;
  // evict-last budget: ~48 MB of the 126 MB L2 for the hottest distances of
  // all resident sources together.
  p.l2hot = g->tune_l2hot >= 0
                ? static_cast<uint32_t>(std::min<int64_t>(g->tune_l2hot, g->n))
                : static_cast<uint32_t>(std::min<uint64_t>(g->n, (48ULL << 20) / 4 / std::max(1, slots)));
  p.prof = g->profiling ? g->d_prof : nullptr;
  WBC_CUDA_TRY(cudaMemsetAsync(g->d_counter, 0, sizeof(unsigned long long), stream));
  WBC_CUDA_TRY(cudaMemsetAsync(g->d_overflow, 0, 4 * sizeof(unsigned int), stream));
  WBC_CUDA_TRY(cudaMemsetAsync(g->d_node_dev, 0, uint64_t{g->n} * 8, stream));
  if (g->profiling)
    WBC_CUDA_TRY(cudaMemsetAsync(g->d_prof, 0, sizeof(unsigned long long) * wbc_dev::kProfCounters, stream));
  if (strict_lanes) {
    rc = launch_strict(g, shape, slots, p, k, edge_bc, d_edge, strict_lanes, stream);
    if (rc) return rc;
  } else if (shape.flat) {
    wbc_dev::FlatWs fw = g->fw;
    fw.sq_cap = shape.flat_sq;
    pick_flat(shape.threads, g->flat_ke)<<<slots, shape.threads, shape.dyn_smem, stream>>>(p, fw);
    WBC_CUDA_TRY(cudaGetLastError());
  } else if (shape.cluster > 0) {
    // whole distance arrays of the few in-flight teams get evict-last
    if (g->tune_l2hot < 0) p.l2hot = g->n;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = shape.cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(slots * shape.cluster, 1, 1);
    cfg.blockDim = dim3(shape.threads, 1, 1);
    cfg.dynamicSmemBytes = shape.dyn_smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = shape.cluster > 1 ? 1 : 0;
    const int fill = single_slot ? 0 : g->fill;
    if (fill > 0) {  // fork: the fill launch runs beside the main one on a side stream
      if (!g->side) {
        WBC_CUDA_TRY(cudaStreamCreateWithFlags(&g->side, cudaStreamNonBlocking));
        WBC_CUDA_TRY(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
        WBC_CUDA_TRY(cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming));
      }
      WBC_CUDA_TRY(cudaEventRecord(g->ev_fork, stream));
      WBC_CUDA_TRY(cudaStreamWaitEvent(g->side, g->ev_fork, 0));
    }
    WBC_CUDA_TRY(cudaLaunchKernelEx(&cfg, pick_team(shape.cluster, shape.threads, g->packed, g->profiling), p));
    if (fill > 0) {
      wbc_dev::RunParams pf = p;
      pf.team_base = static_cast<uint32_t>(slots);
      attr[0].val.clusterDim.x = 2;
      cfg.gridDim = dim3(fill * 2, 1, 1);
      cfg.numAttrs = 1;
      cfg.stream = g->side;
      WBC_CUDA_TRY(cudaLaunchKernelEx(&cfg, pick_team(2, shape.threads, g->packed, g->profiling), pf));
      WBC_CUDA_TRY(cudaEventRecord(g->ev_join, g->side));
      WBC_CUDA_TRY(cudaStreamWaitEvent(stream, g->ev_join, 0));  // join
    }
  } else {
    pick_kernel(shape.threads, g->packed, g->profiling)<<<slots, shape.threads, shape.dyn_smem, stream>>>(p);
    WBC_CUDA_TRY(cudaGetLastError());
  }
  wbc_dev::scatter_add_kernel<<<launch_grid(g->n), 256, 0, stream>>>(d_node, g->d_node_dev, g->d_perm, g->n);
  WBC_CUDA_TRY(cudaGetLastError());
  g->stats[0] = slots;
  g->stats[1] = shape.threads * std::max(1, shape.cluster);
  g->last_kernel = shape.flat ? "bc_flat_kernel<" + std::to_string(shape.threads) + "," + std::to_string(g->flat_ke) + ">"
                  : shape.cluster > 0 ? "bc_team_kernel<" + std::to_string(shape.threads) + "," +
                                            std::to_string(shape.cluster) + ">"
                                      : "bc_sources_kernel<" + std::to_string(shape.threads) + ">";
  if (!strict_lanes) g->stats[3] = (shape.cluster > 0 && !single_slot && g->fill > 0) ? 3 : 2;
  return WBC_OK;
}

// Strict merge (EngineOptions::strict_merge, engine.cpp:389-413): sources run
// in batches of at most `slots`; each source's delta row (and edge terms) land
// in a stage row, and strict_merge_kernel commits the batch in source order.
// The result is bitwise the reference's for the same lane width.
int launch_strict(wbc_gpu_graph* g, const LaunchShape& shape, int slots, wbc_dev::RunParams p, uint64_t k,
                  bool edge_bc, double* d_edge, uint32_t lanes, cudaStream_t stream) {
  const uint64_t ns = g->ws.n_stride, m = g->m;
  const uint64_t per = ns * 8 + (edge_bc ? m * 8 : 0);
  // several sources per team and batch: a batch ends with its slowest source
  uint64_t B = std::min<uint64_t>(static_cast<uint64_t>(slots) * 8, k);
  size_t free_b = 0, total_b = 0;
  WBC_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t avail = free_b + g->stage_bytes;
  const uint64_t reserve = (2ULL << 30) + total_b / 20;
  B = std::max<uint64_t>(1, std::min<uint64_t>(B, avail > reserve ? (avail - reserve) / per : 1));
  if (g->stage_bytes < B * per) {
    cudaFree(g->d_stage);
    g->d_stage = nullptr;
    g->stage_bytes = 0;
    cudaError_t err = cudaSuccess;
    g->d_stage = dev_alloc<double>(B * per / 8, err);
    if (err != cudaSuccess) return set_error(WBC_E_NOMEM, std::string("strict stage: ") + cudaGetErrorString(err));
    g->stage_bytes = B * per;
  }
  // lanes per row: the next power of two of the mean degree, at least the lane width
  const double avg = g->n ? 2.0 * m / g->n : 1.0;
  uint32_t G = 1;
  while (G < 32 && G < avg) G <<= 1;
  p.strict_lanes = lanes;
  p.strict_group = std::max(G, lanes);
  p.ref_slots32 = g->d_ref_slots32;
  p.ref_slots64 = g->d_ref_slots64;
  p.ref_edge_id = g->d_ref_edge_id;
  p.stage_node = g->d_stage;
  p.stage_edge = edge_bc ? g->d_stage + B * ns : nullptr;
  const uint32_t* d_sources = p.sources;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = shape.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<uint64_t>(B, slots)) * shape.cluster, 1, 1);
  cfg.blockDim = dim3(shape.threads, 1, 1);
  cfg.dynamicSmemBytes = shape.dyn_smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = shape.cluster > 1 ? 1 : 0;
  uint64_t launches = 0;
  for (uint64_t b0 = 0; b0 < k; b0 += B) {
    const uint64_t kb = std::min<uint64_t>(B, k - b0);
    WBC_CUDA_TRY(cudaMemsetAsync(g->d_stage, 0, kb * ns * 8, stream));
    if (edge_bc) WBC_CUDA_TRY(cudaMemsetAsync(p.stage_edge, 0, kb * m * 8, stream));
    WBC_CUDA_TRY(cudaMemsetAsync(g->d_counter, 0, sizeof(unsigned long long), stream));
    p.sources = d_sources ? d_sources + b0 : nullptr;
    p.src_base = d_sources ? 0 : b0;
    p.k = kb;
    WBC_CUDA_TRY(cudaLaunchKernelEx(&cfg, pick_team(shape.cluster, shape.threads, g->packed, g->profiling), p));
    wbc_dev::strict_merge_kernel<<<launch_grid(g->n), 256, 0, stream>>>(
        g->d_node_dev, g->d_stage, ns, g->n, static_cast<int>(kb), p.sources, p.src_base, g->d_inv, 1);
    if (edge_bc && m)
      wbc_dev::strict_merge_kernel<<<launch_grid(m), 256, 0, stream>>>(d_edge, p.stage_edge, m, m, static_cast<int>(kb),
                                                                       nullptr, 0, nullptr, 0);
    WBC_CUDA_TRY(cudaGetLastError());
    launches += edge_bc && m ? 3 : 2;
  }
  g->stats[3] = launches + 1;  // + the scatter
  return WBC_OK;
}

// Slot-0 state of the last single-source run (dumps run on the team or
// per-CTA kernels, never on the flat kernel).
struct Slot0 {
  uint32_t* dist;
  double* sigma;
  double* delta;
  uint32_t* order;
  uint32_t* level_ends;
  uint32_t* dag_ends;
  uint2* dag;
  bool pred_dag;   // dag entries are (pred, succ) instead of (slot, succ)
};

int slot0_state(wbc_gpu_graph* g, Slot0* out) {
  const wbc_dev::Workspace& w = g->ws;
  // team-kernel DAG records hold the predecessor (single-source runs never
  // compute edge BC); the per-CTA kernel records the slot
  *out = Slot0{w.dist, w.sigma, w.delta, w.order, w.level_ends, w.dag_ends, w.dag, g->ws_team};
  return WBC_OK;
}

int scale_async(double* x, uint64_t len, double f, cudaStream_t stream) {
  if (!len) return WBC_OK;
  wbc_dev::scale_kernel<<<launch_grid(len), 256, 0, stream>>>(x, len, f);
  WBC_CUDA_TRY(cudaGetLastError());
  return WBC_OK;
}

}  // namespace

namespace {

// Host side of a graph upload, computed once and shared by every device of
// a multi-GPU handle: validation, degree-descending relabel, packed slots.
struct HostCsr {
  uint32_t n = 0, m = 0, max_weight = 0, wbits = 0, near_width = 1, max_degree = 0, max_minw = 0;
  bool symmetric = false;  // every slot u->v (w) has a twin v->u (w); checked for low-degree graphs
  int scale_k = 0;         // weights were scaled by 2^scale_k to integers
  bool packed = true, skewed = false, has_edge_id = false;
  double hot_coverage_25k = 0;
  std::vector<uint32_t> perm, inv, noff, slot32, eid, minw, ref_slot32, ref_eid;
  std::vector<uint2> slot64, ref_slot64;
  // ELL copy for bc_flat_kernel (flat graphs): per vertex 2 ke words, the
  // ke packed slots then ke u16 sweep keys (two per word), zero padded
  int ke = 0;
  std::vector<uint32_t> ell, ell_eid;
};

int prepare_host(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
                 const double* weights, const double* min_incident_weight, const uint32_t* edge_id,
                 HostCsr& h) {
  const uint64_t slots = 2ULL * m;
  if (slots >= (1ULL << 32)) return set_error(WBC_E_UNSUPPORTED, "2m must fit in u32 slots");
  if (n > 0 && (!offsets || !min_incident_weight))
    return set_error(WBC_E_INVALID, "offsets / min_incident_weight are required");
  if (slots > 0 && (!adjacency || !weights))
    return set_error(WBC_E_INVALID, "adjacency / weights are required");
  if (n > 0 && (offsets[0] != 0 || offsets[n] != slots))
    return set_error(WBC_E_INVALID, "offsets must start at 0 and end at 2m");
  if (n == 0 && slots != 0) return set_error(WBC_E_INVALID, "edges without vertices");
  // validation, thread-parallel: the first failing slot (lowest index) is reported
  std::atomic<uint64_t> bad_off{UINT64_MAX}, bad_adj{UINT64_MAX}, bad_w{UINT64_MAX};
  std::atomic<uint64_t> maxw_a{0};
  auto atomic_min = [](std::atomic<uint64_t>& a, uint64_t v) {
    uint64_t cur = a.load();
    while (v < cur && !a.compare_exchange_weak(cur, v)) {}
  };
  parallel_for(n, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v)
      if (offsets[v + 1] < offsets[v]) {
        atomic_min(bad_off, v);
        return;
      }
  });
  if (bad_off.load() != UINT64_MAX) return set_error(WBC_E_INVALID, "offsets not monotone");
  // Weights: positive dyadic rationals w = i / 2^k (integers k = 0, and e.g.
  // 0.5 or 2.5), scaled by the common 2^K to integers.  Scaling by a power of
  // two is exact in fp64, so every distance the reference computes is 2^-K
  // times an exact integer sum (while below 2^53, which the u32 bound below
  // implies): distances, ties, the Eq. 4 thresholds d + minw (hence
  // depth_per_source) and sigma / delta / BC are those of the integer graph.
  std::atomic<int> scale_k{0};
  parallel_for(slots, [&](uint64_t b, uint64_t e) {
    int kk = 0;
    for (uint64_t x = b; x < e; ++x) {
      const double w = weights[x];
      if (adjacency[x] >= n) {
        atomic_min(bad_adj, x);
        break;
      }
      if (!(w > 0.0) || !std::isfinite(w)) {
        atomic_min(bad_w, x);
        break;
      }
      int k = 0;
      while (k <= kMaxWeightScaleBits && std::ldexp(w, k) != std::floor(std::ldexp(w, k))) ++k;
      if (k > kMaxWeightScaleBits) {
        atomic_min(bad_w, x);
        break;
      }
      kk = std::max(kk, k);
    }
    int cur = scale_k.load();
    while (kk > cur && !scale_k.compare_exchange_weak(cur, kk)) {}
  });
  if (bad_adj.load() < bad_w.load()) return set_error(WBC_E_INVALID, "adjacency entry out of range");
  if (bad_w.load() != UINT64_MAX)
    return set_error(WBC_E_UNSUPPORTED,
                     "weights must be positive integers or dyadic fractions i / 2^k, k <= " +
                         std::to_string(kMaxWeightScaleBits) + " (exact integer distances on the GPU); got " +
                         std::to_string(weights[bad_w.load()]));
  const int K = scale_k.load();
  h.scale_k = K;
  parallel_for(slots, [&](uint64_t b, uint64_t e) {
    uint64_t mw = 0;
    for (uint64_t x = b; x < e; ++x) {
      const double w = std::ldexp(weights[x], K);
      mw = std::max<uint64_t>(mw, w > 4294967295.0 ? UINT64_MAX : static_cast<uint64_t>(w));
    }
    uint64_t cur = maxw_a.load();
    while (mw > cur && !maxw_a.compare_exchange_weak(cur, mw)) {}
  });
  const uint64_t maxw = maxw_a.load();
  if (maxw > 0xFFFFFFFFULL || (n > 0 && uint64_t{n} * std::max<uint64_t>(maxw, 1) >= 0xFFFFFFFFULL))
    return set_error(WBC_E_UNSUPPORTED, "n * max_weight (scaled to integers) must stay below 2^32-1");
  h.n = n;
  h.m = m;
  h.has_edge_id = edge_id != nullptr;
  h.max_weight = static_cast<uint32_t>(maxw);
  h.wbits = bits_for(std::max<uint64_t>(maxw, 1));
  const uint32_t nbits = bits_for(n ? n - 1 : 0);
  h.packed = (h.wbits + nbits) <= 32;

  // ---- degree-descending relabel (ties by id) ---------------------------
  std::vector<uint32_t>& perm = h.perm;
  perm.resize(n);
  std::iota(perm.begin(), perm.end(), 0u);
  std::stable_sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) {
    return offsets[a + 1] - offsets[a] > offsets[b + 1] - offsets[b];
  });
  std::vector<uint32_t>& inv = h.inv;
  inv.resize(n);
  for (uint32_t i = 0; i < n; ++i) inv[perm[i]] = i;
  std::vector<uint32_t>& noff = h.noff;
  noff.assign(uint64_t{n} + 1, 0);
  for (uint32_t i = 0; i < n; ++i) noff[i + 1] = noff[i] + (offsets[perm[i] + 1] - offsets[perm[i]]);
  if (slots) {
    uint64_t top = 0;
    for (uint32_t i = 0; i < std::min<uint32_t>(n, 25 * 1024); ++i) top += noff[i + 1] - noff[i];
    h.hot_coverage_25k = static_cast<double>(top) / static_cast<double>(slots);
    const double avg = static_cast<double>(slots) / n;
    h.skewed = static_cast<double>(noff[1] - noff[0]) >= 16.0 * avg;  // perm[0] has the max degree
  }
  h.slot32.assign(h.packed ? slots : 0, 0);
  h.slot64.assign(h.packed ? 0 : slots, make_uint2(0, 0));
  h.eid.assign(edge_id ? slots : 0, 0);
  h.ref_slot32.assign(h.packed ? slots : 0, 0);
  h.ref_slot64.assign(h.packed ? 0 : slots, make_uint2(0, 0));
  h.ref_eid.assign(edge_id ? slots : 0, 0);
  h.minw.assign(n, 0);
  double sum_minw = 0;
  uint64_t cnt_minw = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t v = perm[i];
    const double x = min_incident_weight[v];
    if (std::isinf(x) || offsets[v + 1] == offsets[v]) {
      h.minw[i] = wbc_dev::kInfDist;
    } else {
      h.minw[i] = static_cast<uint32_t>(std::ldexp(x, K));
      sum_minw += std::ldexp(x, K);
      ++cnt_minw;
    }
  }
  const uint32_t wbits = h.wbits;
  const bool packed = h.packed;
  parallel_for(n, [&](uint64_t b, uint64_t e) {
    std::vector<std::pair<uint32_t, uint32_t>> row;  // (new neighbour, old slot)
    for (uint64_t i = b; i < e; ++i) {
      const uint32_t v = perm[i];
      row.clear();
      for (uint32_t s = offsets[v]; s < offsets[v + 1]; ++s) row.emplace_back(inv[adjacency[s]], s);
      uint32_t o = noff[i];
      for (const auto& [u, s] : row) {  // caller's order (strict merge)
        const uint32_t w = static_cast<uint32_t>(std::ldexp(weights[s], K));
        if (packed)
          h.ref_slot32[o] = (u << wbits) | w;
        else
          h.ref_slot64[o] = make_uint2(u, w);
        if (edge_id) h.ref_eid[o] = edge_id[s];
        ++o;
      }
      std::sort(row.begin(), row.end());
      o = noff[i];
      for (const auto& [u, s] : row) {
        const uint32_t w = static_cast<uint32_t>(std::ldexp(weights[s], K));
        if (packed)
          h.slot32[o] = (u << wbits) | w;
        else
          h.slot64[o] = make_uint2(u, w);
        if (edge_id) h.eid[o] = edge_id[s];
        ++o;
      }
    }
  });
  // Near-window width: about a third of the mean minimum incident weight balances
  // near rescans against far refills.
  h.near_width = cnt_minw ? std::max<uint32_t>(1, static_cast<uint32_t>(sum_minw / cnt_minw / 3.0 + 0.5)) : 1;
  for (uint32_t i = 0; i < n; ++i) {
    h.max_degree = std::max(h.max_degree, h.noff[i + 1] - h.noff[i]);
    if (h.minw[i] != wbc_dev::kInfDist) h.max_minw = std::max(h.max_minw, h.minw[i]);
  }
  // The flat kernel's dataflows count DAG edges from both ends; a caller CSR
  // whose rows are not mirror images (not from build_csr) must not reach it.
  if (h.max_degree <= static_cast<uint32_t>(wbc_dev::kFlatMaxDeg)) {
    std::atomic<bool> sym{true};
    parallel_for(n, [&](uint64_t ub, uint64_t ue) {
    bool ok = true;
    for (uint32_t u = static_cast<uint32_t>(ub); u < ue && ok && sym.load(std::memory_order_relaxed); ++u)
      for (uint32_t e = h.noff[u]; e < h.noff[u + 1] && ok; ++e) {
        const uint32_t v = packed ? h.slot32[e] >> wbits : h.slot64[e].x;
        const uint32_t w = packed ? h.slot32[e] & ((wbits >= 32) ? 0xFFFFFFFFu : ((1u << wbits) - 1)) : h.slot64[e].y;
        uint32_t twins = 0, same = 0;
        for (uint32_t f = h.noff[v]; f < h.noff[v + 1]; ++f) {
          const uint32_t x = packed ? h.slot32[f] >> wbits : h.slot64[f].x;
          const uint32_t y = packed ? h.slot32[f] & ((wbits >= 32) ? 0xFFFFFFFFu : ((1u << wbits) - 1)) : h.slot64[f].y;
          twins += x == u && y == w;
        }
        for (uint32_t f = h.noff[u]; f < h.noff[u + 1]; ++f) {
          const uint32_t x = packed ? h.slot32[f] >> wbits : h.slot64[f].x;
          const uint32_t y = packed ? h.slot32[f] & ((wbits >= 32) ? 0xFFFFFFFFu : ((1u << wbits) - 1)) : h.slot64[f].y;
          same += x == v && y == w;
        }
        ok = twins == same && u != v;
      }
    if (!ok) sym.store(false);
    });
    h.symmetric = sym.load();
  }
  // ELL rows for the distance-first kernel: packed slots, weight 0 pads
  uint64_t max_key = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (h.minw[i] != wbc_dev::kInfDist) max_key = std::max<uint64_t>(max_key, uint64_t{h.minw[i]} + maxw);
  if (h.symmetric && packed && n > 0 && slots > 0 && max_key < 65536) {
    const int ke = h.max_degree <= 4 ? 4 : 8;
    h.ke = ke;
    h.ell.assign(uint64_t{n} * 2 * ke, 0);
    if (edge_id) h.ell_eid.assign(uint64_t{n} * ke, 0);
    const uint32_t wm = (wbits >= 32) ? 0xFFFFFFFFu : ((1u << wbits) - 1);
    parallel_for(n, [&](uint64_t b, uint64_t e) {
      for (uint64_t v = b; v < e; ++v)
        for (uint32_t j = 0; j < h.noff[v + 1] - h.noff[v]; ++j) {
          const uint32_t x = h.slot32[h.noff[v] + j];
          uint32_t* const rec = h.ell.data() + v * 2 * ke;
          rec[j] = x;
          rec[ke + j / 2] |= ((x & wm) + h.minw[x >> wbits]) << (16 * (j & 1));
          if (edge_id) h.ell_eid[v * ke + j] = h.eid[h.noff[v] + j];
        }
    });
  }
  return WBC_OK;
}

// Device side: one replica of a prepared graph on `device`.
int upload_graph(const HostCsr& h, int device, wbc_gpu_graph** out) {
  const uint32_t n = h.n;
  const uint64_t slots = 2ULL * h.m;
  auto g = new wbc_gpu_graph();
  int dev = device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
    delete g;
    return set_error(WBC_E_NOT_BUILT, "no CUDA device available");
  }
  g->device = dev;
  cudaError_t err = cudaSetDevice(dev);
  if (err != cudaSuccess) {
    delete g;
    return set_error(WBC_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(err));
  }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&g->smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&g->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (major < 10) {
    delete g;
    return set_error(WBC_E_NOT_BUILT, "device is not sm_100 class (built for sm_100a only)");
  }
  if (const char* e = std::getenv("WBC_GPU_CLUSTER")) g->tune_cluster = std::atoi(e);  // tuning default
  g->n = n;
  g->m = h.m;
  g->max_weight = h.max_weight;
  g->wbits = h.wbits;
  g->packed = h.packed;
  g->perm = h.perm;
  g->hot_coverage_25k = h.hot_coverage_25k;
  g->skewed = h.skewed;
  g->near_width = h.near_width;
  g->max_degree = h.max_degree;
  g->max_minw = h.max_minw;
  g->symmetric = h.symmetric;
  g->scale_k = h.scale_k;
  const bool packed = h.packed;
  g->d_offsets = dev_alloc<uint32_t>(uint64_t{n} + 1, err);
  if (err == cudaSuccess) g->d_minw = dev_alloc<uint32_t>(n, err);
  if (err == cudaSuccess) g->d_perm = dev_alloc<uint32_t>(n, err);
  if (err == cudaSuccess) g->d_inv = dev_alloc<uint32_t>(n, err);
  if (err == cudaSuccess) g->d_node_dev = dev_alloc<double>(n, err);
  if (err == cudaSuccess) g->d_counter = dev_alloc<unsigned long long>(1, err);
  if (err == cudaSuccess) g->d_overflow = dev_alloc<unsigned int>(4, err);
  if (err == cudaSuccess) g->d_prof = dev_alloc<unsigned long long>(wbc_dev::kProfCounters, err);
  if (err == cudaSuccess) {
    if (packed)
      g->d_slots32 = dev_alloc<uint32_t>(slots, err);
    else
      g->d_slots64 = dev_alloc<uint2>(slots, err);
  }
  if (err == cudaSuccess) {
    if (packed)
      g->d_ref_slots32 = dev_alloc<uint32_t>(slots, err);
    else
      g->d_ref_slots64 = dev_alloc<uint2>(slots, err);
  }
  if (err == cudaSuccess && h.has_edge_id) g->d_edge_id = dev_alloc<uint32_t>(slots, err);
  if (err == cudaSuccess && h.has_edge_id) g->d_ref_edge_id = dev_alloc<uint32_t>(slots, err);
  g->flat_ke = h.ke;
  if (err == cudaSuccess && h.ke) {
    g->d_ell = dev_alloc<uint32_t>(h.ell.size(), err);
    if (err == cudaSuccess && h.has_edge_id) g->d_ell_eid = dev_alloc<uint32_t>(h.ell_eid.size(), err);
  }
  if (err != cudaSuccess) {
    delete g;
    return set_error(WBC_E_NOMEM, std::string("graph upload: ") + cudaGetErrorString(err));
  }
  if (n) {
    err = cudaMemcpy(g->d_offsets, h.noff.data(), (uint64_t{n} + 1) * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(g->d_minw, h.minw.data(), uint64_t{n} * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(g->d_perm, h.perm.data(), uint64_t{n} * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(g->d_inv, h.inv.data(), uint64_t{n} * 4, cudaMemcpyHostToDevice);
  }
  if (err == cudaSuccess && slots) {
    if (packed)
      err = cudaMemcpy(g->d_slots32, h.slot32.data(), slots * 4, cudaMemcpyHostToDevice);
    else
      err = cudaMemcpy(g->d_slots64, h.slot64.data(), slots * 8, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) {
      if (packed)
        err = cudaMemcpy(g->d_ref_slots32, h.ref_slot32.data(), slots * 4, cudaMemcpyHostToDevice);
      else
        err = cudaMemcpy(g->d_ref_slots64, h.ref_slot64.data(), slots * 8, cudaMemcpyHostToDevice);
    }
    if (err == cudaSuccess && h.has_edge_id)
      err = cudaMemcpy(g->d_edge_id, h.eid.data(), slots * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess && h.has_edge_id)
      err = cudaMemcpy(g->d_ref_edge_id, h.ref_eid.data(), slots * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess && h.ke) {
      err = cudaMemcpy(g->d_ell, h.ell.data(), h.ell.size() * 4, cudaMemcpyHostToDevice);
      if (err == cudaSuccess && h.has_edge_id)
        err = cudaMemcpy(g->d_ell_eid, h.ell_eid.data(), h.ell_eid.size() * 4, cudaMemcpyHostToDevice);
    }
  }
  if (err != cudaSuccess) {
    delete g;
    return set_error(WBC_E_CUDA, std::string("graph upload: ") + cudaGetErrorString(err));
  }
  g->graph_bytes = (uint64_t{n} + 1) * 4 + uint64_t{n} * 12 + 2 * slots * (packed ? 4 : 8) +
                   (h.has_edge_id ? 2 * slots * 4 : 0);
  g->graph_bytes += h.ell.size() * 4 + h.ell_eid.size() * 4;
  *out = g;
  return WBC_OK;
}

}  // namespace

extern "C" {

const char* wbc_gpu_last_error(void) { return g_last_error.c_str(); }

int wbc_gpu_graph_create(uint32_t n, uint32_t m, const uint32_t* offsets,
                         const uint32_t* adjacency, const double* weights,
                         const double* min_incident_weight, const uint32_t* edge_id, int device,
                         wbc_gpu_graph** out) {
  if (!out) return set_error(WBC_E_INVALID, "out is null");
  *out = nullptr;
  HostCsr h;
  const int rc = prepare_host(n, m, offsets, adjacency, weights, min_incident_weight, edge_id, h);
  if (rc) return rc;
  return upload_graph(h, device, out);
}

void wbc_gpu_graph_destroy(wbc_gpu_graph* g) { delete g; }

int wbc_gpu_graph_info(wbc_gpu_graph* g, uint32_t* n, uint32_t* m, uint32_t* max_weight,
                       int* packed_slots, uint32_t* near_width, uint64_t* graph_bytes) {
  if (!g) return set_error(WBC_E_INVALID, "null graph");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (max_weight) *max_weight = g->max_weight;
  if (packed_slots) *packed_slots = g->packed ? 1 : 0;
  if (near_width) *near_width = g->near_width;
  if (graph_bytes) *graph_bytes = g->graph_bytes;
  return WBC_OK;
}

int wbc_gpu_set_tuning(wbc_gpu_graph* g, int threads_per_cta, int max_slots, uint32_t near_width,
                       int64_t hot_vertices) {
  if (!g) return set_error(WBC_E_INVALID, "null graph");
  if (threads_per_cta < 0 || max_slots < 0) return set_error(WBC_E_INVALID, "negative tuning value");
  ++g->tune_gen;
  g->tune_threads = threads_per_cta;
  g->tune_slots = max_slots;
  g->tune_hot = hot_vertices;
  if (near_width) {
    g->near_width = near_width;
    g->tune_near = true;
  }
  return WBC_OK;
}

int wbc_gpu_set_param(wbc_gpu_graph* g, const char* name, int64_t value) {
  if (!g || !name) return set_error(WBC_E_INVALID, "null argument");
  ++g->tune_gen;
  const std::string k = name;
  if (k == "threads") g->tune_threads = static_cast<int>(value);
  else if (k == "slots") g->tune_slots = static_cast<int>(value);
  else if (k == "near_width") {
    g->near_width = value > 0 ? static_cast<uint32_t>(value) : g->near_width;
    g->tune_near = value > 0;
  }
  else if (k == "hot") g->tune_hot = value;
  else if (k == "l2hot") g->tune_l2hot = value;
  else if (k == "cluster") g->tune_cluster = static_cast<int>(value);
  else if (k == "fill") g->tune_fill = static_cast<int>(value);
  else if (k == "flat") g->tune_flat = static_cast<int>(value);
  else if (k == "flat_delta") g->tune_flat_delta = static_cast<uint32_t>(std::max<int64_t>(0, value));
  else if (k == "flat_threads") g->tune_flat_threads = static_cast<int>(value);
  else if (k == "flat_sq") g->tune_flat_sq = static_cast<int>(std::max<int64_t>(-1, std::min<int64_t>(value, 1 << 14)));
  else return set_error(WBC_E_INVALID, "unknown tuning parameter '" + k + "'");
  return WBC_OK;
}

int wbc_gpu_set_profiling(wbc_gpu_graph* g, int on) {
  if (!g) return set_error(WBC_E_INVALID, "null graph");
  g->profiling = on != 0;
  return WBC_OK;
}

int wbc_gpu_profile_counters(wbc_gpu_graph* g, uint64_t* out16) {
  if (!g || !out16) return set_error(WBC_E_INVALID, "null argument");
  WBC_CUDA_TRY(cudaSetDevice(g->device));
  WBC_CUDA_TRY(cudaDeviceSynchronize());
  uint64_t tmp[16] = {};
  static_assert(wbc_dev::kProfCounters <= 16, "counter block");
  WBC_CUDA_TRY(cudaMemcpy(tmp, g->d_prof, sizeof(unsigned long long) * wbc_dev::kProfCounters,
                          cudaMemcpyDeviceToHost));
  std::memcpy(out16, tmp, sizeof tmp);
  return WBC_OK;
}

int wbc_gpu_last_run_stats(wbc_gpu_graph* g, uint64_t* stats4) {
  if (!g || !stats4) return set_error(WBC_E_INVALID, "null argument");
  std::memcpy(stats4, g->stats, sizeof g->stats);
  return WBC_OK;
}

int wbc_gpu_last_run_info(wbc_gpu_graph* g, uint64_t* out, uint32_t cap) {
  if (!g || (!out && cap)) return set_error(WBC_E_INVALID, "null argument");
  WBC_CUDA_TRY(cudaSetDevice(g->device));
  WBC_CUDA_TRY(cudaDeviceSynchronize());  // the run's device-side counters are final
  unsigned int ov[2] = {0, 0};
  const unsigned long long fb = 0;  // bc_flat_kernel completes every source (no hand-back since round 2)
  if (g->stats[3]) WBC_CUDA_TRY(cudaMemcpy(ov, g->d_overflow, sizeof ov, cudaMemcpyDeviceToHost));
  const uint64_t v[WBC_RUN_INFO_FIELDS] = {g->stats[0], g->stats[1], ov[0], g->stats[3], fb, ov[1] ? 1u : 0u};
  for (uint32_t i = 0; i < cap && i < WBC_RUN_INFO_FIELDS; ++i) out[i] = v[i];
  return WBC_OK;
}

int wbc_gpu_bc_device(wbc_gpu_graph* g, const uint32_t* d_sources, uint64_t k, uint32_t flags,
                      double* d_node_bc, double* d_edge_bc, uint32_t* d_depth_per_source,
                      void* stream) {
  if (!g) return set_error(WBC_E_INVALID, "null graph");
  if (!d_node_bc && g->n) return set_error(WBC_E_INVALID, "node_bc is required");
  const bool edge = flags & WBC_EDGE_BC;
  if (edge && !g->d_edge_id)
    return set_error(WBC_E_INVALID, "edge BC requested but the graph was created without edge_id");
  if (edge && !d_edge_bc && g->m) return set_error(WBC_E_INVALID, "edge_bc is required");
  uint32_t lanes = 0;
  int rc = strict_lanes_of(flags, &lanes);
  if (rc) return rc;
  WBC_CUDA_TRY(cudaSetDevice(g->device));
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t kk = d_sources ? k : g->n;
  rc = launch_run(g, d_sources, kk, edge, d_node_bc, d_edge_bc, d_depth_per_source, st, false, false, lanes);
  if (rc) return rc;
  if (flags & WBC_HALVED) {
    if ((rc = scale_async(d_node_bc, g->n, 0.5, st))) return rc;
    if (edge && (rc = scale_async(d_edge_bc, g->m, 0.5, st))) return rc;
  }
  return WBC_OK;
}

int wbc_gpu_bc(wbc_gpu_graph* g, const uint32_t* sources, uint64_t k, uint32_t flags,
               double* node_bc, double* edge_bc, uint32_t* depth_per_source, double* elapsed_s) {
  if (!g) return set_error(WBC_E_INVALID, "null graph");
  const bool edge = flags & WBC_EDGE_BC;
  if (!node_bc && g->n) return set_error(WBC_E_INVALID, "node_bc is required");
  if (edge && !edge_bc && g->m) return set_error(WBC_E_INVALID, "edge_bc is required");
  if (edge && !g->d_edge_id)
    return set_error(WBC_E_INVALID, "edge BC requested but the graph was created without edge_id");
  uint32_t lanes = 0;
  if (const int rl = strict_lanes_of(flags, &lanes)) return rl;
  if (sources)  // resolve_sources (engine.cpp:349-361)
    for (uint64_t i = 0; i < k; ++i)
      if (sources[i] >= g->n)
        return set_error(WBC_E_INVALID, "bc_parallel: source id out of range");
  const auto t0 = std::chrono::steady_clock::now();
  WBC_CUDA_TRY(cudaSetDevice(g->device));
  cudaError_t err = cudaSuccess;
  if (!g->d_node) g->d_node = dev_alloc<double>(g->n, err);
  if (err == cudaSuccess && !g->d_depth) g->d_depth = dev_alloc<uint32_t>(g->n, err);
  if (err == cudaSuccess && edge && !g->d_edge) g->d_edge = dev_alloc<double>(g->m, err);
  if (err != cudaSuccess) return set_error(WBC_E_NOMEM, cudaGetErrorString(err));
  const cudaStream_t st = 0;
  const uint64_t kk = sources ? k : g->n;
  if (sources && k > g->d_sources_cap) {
    cudaFree(g->d_sources);
    g->d_sources = dev_alloc<uint32_t>(k, err);
    if (err != cudaSuccess) {
      g->d_sources_cap = 0;
      return set_error(WBC_E_NOMEM, cudaGetErrorString(err));
    }
    g->d_sources_cap = k;
  }
  if (sources && k)
    WBC_CUDA_TRY(cudaMemcpyAsync(g->d_sources, sources, k * 4, cudaMemcpyHostToDevice, st));
  if (g->n) {
    WBC_CUDA_TRY(cudaMemsetAsync(g->d_node, 0, uint64_t{g->n} * 8, st));
    WBC_CUDA_TRY(cudaMemsetAsync(g->d_depth, 0, uint64_t{g->n} * 4, st));
  }
  if (edge && g->m) WBC_CUDA_TRY(cudaMemsetAsync(g->d_edge, 0, uint64_t{g->m} * 8, st));
  int rc = launch_run(g, sources ? g->d_sources : nullptr, kk, edge, g->d_node, g->d_edge,
                      g->d_depth, st, false, false, lanes);
  if (rc) return rc;
  if (flags & WBC_HALVED) {  // engine.cpp:451-454
    if ((rc = scale_async(g->d_node, g->n, 0.5, st))) return rc;
    if (edge && (rc = scale_async(g->d_edge, g->m, 0.5, st))) return rc;
  }
  if (g->n) {
    WBC_CUDA_TRY(cudaMemcpyAsync(node_bc, g->d_node, uint64_t{g->n} * 8, cudaMemcpyDeviceToHost, st));
    if (depth_per_source)
      WBC_CUDA_TRY(cudaMemcpyAsync(depth_per_source, g->d_depth, uint64_t{g->n} * 4,
                                   cudaMemcpyDeviceToHost, st));
  }
  if (edge && g->m)
    WBC_CUDA_TRY(cudaMemcpyAsync(edge_bc, g->d_edge, uint64_t{g->m} * 8, cudaMemcpyDeviceToHost, st));
  unsigned int overflow = 0;
  WBC_CUDA_TRY(cudaMemcpyAsync(&overflow, g->d_overflow, 4, cudaMemcpyDeviceToHost, st));
  WBC_CUDA_TRY(cudaStreamSynchronize(st));
  g->stats[2] = kk ? overflow : 0;
  if (elapsed_s)
    *elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return WBC_OK;
}

int wbc_gpu_sssp_dump(wbc_gpu_graph* g, uint32_t source, double* dist, double* sigma,
                      double* delta, uint32_t* depth) {
  if (!g) return set_error(WBC_E_INVALID, "null graph");
  if (source >= g->n) return set_error(WBC_E_INVALID, "init_state: source out of range");
  WBC_CUDA_TRY(cudaSetDevice(g->device));
  const uint64_t n = g->n;
  int slots = 0;
  int rc = ensure_workspace(g, 1, pick_shape(g), &slots);
  if (rc) return rc;
  cudaError_t err = cudaSuccess;
  double* d_scratch = dev_alloc<double>(n, err);
  uint32_t* d_src = err == cudaSuccess ? dev_alloc<uint32_t>(1, err) : nullptr;
  uint32_t* d_dep = err == cudaSuccess ? dev_alloc<uint32_t>(n, err) : nullptr;
  if (err != cudaSuccess) {
    cudaFree(d_scratch);
    cudaFree(d_src);
    return set_error(WBC_E_NOMEM, cudaGetErrorString(err));
  }
  std::vector<uint32_t> du(n);
  std::vector<double> tmp(n);
  auto body = [&]() -> int {
    WBC_CUDA_TRY(cudaMemcpy(d_src, &source, 4, cudaMemcpyHostToDevice));
    WBC_CUDA_TRY(cudaMemset(d_scratch, 0, n * 8));
    WBC_CUDA_TRY(cudaMemset(d_dep, 0, n * 4));
    // slot 0's sigma and delta (identical offsets in every layout at one
    // slot): unreached vertices stay 0
    WBC_CUDA_TRY(cudaMemset(g->d_ws, 0, std::min<uint64_t>(g->ws_bytes, ws_ns(g) * 16)));
    int r = launch_run(g, d_src, 1, false, d_scratch, nullptr, d_dep, 0, true, true);
    if (r) return r;
    WBC_CUDA_TRY(cudaDeviceSynchronize());
    Slot0 st{};
    if ((r = slot0_state(g, &st))) return r;
    WBC_CUDA_TRY(cudaMemcpy(du.data(), st.dist, n * 4, cudaMemcpyDeviceToHost));
    if (dist)
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t d = du[i];
        dist[g->perm[i]] = d == wbc_dev::kInfDist ? HUGE_VAL : std::ldexp(static_cast<double>(d), -g->scale_k);
      }
    if (sigma) {
      WBC_CUDA_TRY(cudaMemcpy(tmp.data(), st.sigma, n * 8, cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i < n; ++i) sigma[g->perm[i]] = tmp[i];
    }
    if (delta) {
      WBC_CUDA_TRY(cudaMemcpy(tmp.data(), st.delta, n * 8, cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i < n; ++i) delta[g->perm[i]] = tmp[i];
    }
    if (depth) WBC_CUDA_TRY(cudaMemcpy(depth, d_dep + source, 4, cudaMemcpyDeviceToHost));
    return WBC_OK;
  };
  rc = body();
  cudaFree(d_scratch);
  cudaFree(d_src);
  cudaFree(d_dep);
  return rc;
}

int wbc_gpu_last_kernel(wbc_gpu_graph* g, char* buf, size_t cap) {
  if (!g || !buf || !cap) return set_error(WBC_E_INVALID, "null argument");
  const size_t k = std::min(cap - 1, g->last_kernel.size());
  std::memcpy(buf, g->last_kernel.data(), k);
  buf[k] = 0;
  return WBC_OK;
}

int wbc_gpu_sssp_dag(wbc_gpu_graph* g, uint32_t source, uint32_t* pred, uint32_t* succ,
                     uint32_t* dag_ends, uint32_t* levels, uint32_t* overflow) {
  if (!g || !pred || !succ || !dag_ends || !levels || !overflow) return set_error(WBC_E_INVALID, "null argument");
  if (source >= g->n) return set_error(WBC_E_INVALID, "init_state: source out of range");
  uint32_t depth = 0;
  int rc = wbc_gpu_sssp_dump(g, source, nullptr, nullptr, nullptr, &depth);
  if (rc) return rc;
  unsigned int ov = 0;
  WBC_CUDA_TRY(cudaMemcpy(&ov, g->d_overflow, 4, cudaMemcpyDeviceToHost));
  Slot0 st{};
  if ((rc = slot0_state(g, &st))) return rc;
  std::vector<uint32_t> de(uint64_t{depth} + 1);
  WBC_CUDA_TRY(cudaMemcpy(de.data(), st.dag_ends, de.size() * 4, cudaMemcpyDeviceToHost));
  const uint32_t len = std::min<uint64_t>(de[depth], g->ws.dag_cap);
  std::vector<uint2> d(len);
  if (len) WBC_CUDA_TRY(cudaMemcpy(d.data(), st.dag, uint64_t{len} * 8, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> slots(g->packed ? 2ULL * g->m : 0);
  std::vector<uint2> slots64(g->packed ? 0 : 2ULL * g->m);
  if (g->m) {
    if (g->packed)
      WBC_CUDA_TRY(cudaMemcpy(slots.data(), g->d_slots32, 8ULL * g->m, cudaMemcpyDeviceToHost));
    else
      WBC_CUDA_TRY(cudaMemcpy(slots64.data(), g->d_slots64, 16ULL * g->m, cudaMemcpyDeviceToHost));
  }
  for (uint32_t i = 0; i < len; ++i) {
    const uint32_t u = st.pred_dag ? d[i].x : g->packed ? slots[d[i].x] >> g->wbits : slots64[d[i].x].x;
    pred[i] = g->perm[u];
    succ[i] = g->perm[d[i].y];
  }
  std::memcpy(dag_ends, de.data(), de.size() * 4);
  *levels = depth;
  *overflow = ov;
  return WBC_OK;
}

int wbc_gpu_sssp_levels(wbc_gpu_graph* g, uint32_t source, uint32_t* order, uint32_t* order_len,
                        uint32_t* level_ends, uint32_t* levels) {
  if (!g || !order || !order_len || !level_ends || !levels) return set_error(WBC_E_INVALID, "null argument");
  if (source >= g->n) return set_error(WBC_E_INVALID, "init_state: source out of range");
  uint32_t depth = 0;
  int rc = wbc_gpu_sssp_dump(g, source, nullptr, nullptr, nullptr, &depth);
  if (rc) return rc;
  // workspace slot 0 still holds the source's order / level ends
  Slot0 st{};
  if ((rc = slot0_state(g, &st))) return rc;
  std::vector<uint32_t> lev(uint64_t{depth} + 1);
  WBC_CUDA_TRY(cudaMemcpy(lev.data(), st.level_ends, lev.size() * 4, cudaMemcpyDeviceToHost));
  const uint32_t len = lev[depth];
  std::vector<uint32_t> ord(len);
  if (len) WBC_CUDA_TRY(cudaMemcpy(ord.data(), st.order, uint64_t{len} * 4, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < len; ++i) order[i] = g->perm[ord[i]];
  std::memcpy(level_ends, lev.data(), lev.size() * 4);
  *order_len = len;
  *levels = depth;
  return WBC_OK;
}

}  // extern "C"

// ===========================================================================
// One process, several GPUs (SURVEY.md §8(b) num_gpus, §8(e)): sources are
// sharded strided across the devices, each holding a full CSR replica; the
// partial node/edge BC and depth vectors are combined by ONE NCCL all-reduce
// (sum / sum / max).  NCCL is dlopen'ed on first use -- if the process already
// loaded a libnccl (e.g. torch's), that one is used -- so the library itself
// has no link-time NCCL dependency.  When NCCL is unavailable or a device
// repeats (the test mode of one-GPU machines), the partials are combined by
// device-to-device copies and an add kernel on the first device instead.
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return a;
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.CommInitAll && a.AllReduce && a.GroupStart && a.GroupEnd && a.CommDestroy && a.GetErrorString;
    return a;
  }();
  return api;
}

}  // namespace

struct wbc_gpu_multi {
  uint32_t n = 0, m = 0;
  std::vector<wbc_gpu_graph*> g;
  std::vector<cudaStream_t> st;
  std::vector<ncclComm_t> comm;
  bool use_nccl = false;
  std::vector<double*> d_node, d_edge;
  std::vector<uint32_t*> d_depth, d_src;
  std::vector<uint64_t> src_cap;
  double* d_tmp = nullptr;      // first device: staging for the copy reduction
  uint32_t* d_tmp32 = nullptr;
  ~wbc_gpu_multi() {
    if (use_nccl)
      for (ncclComm_t c : comm) nccl_api().CommDestroy(c);
    for (size_t i = 0; i < g.size(); ++i) {
      if (!g[i]) continue;
      cudaSetDevice(g[i]->device);
      cudaFree(d_node[i]);
      cudaFree(d_edge[i]);
      cudaFree(d_depth[i]);
      cudaFree(d_src[i]);
      if (st[i]) cudaStreamDestroy(st[i]);
      if (i == 0) {
        cudaFree(d_tmp);
        cudaFree(d_tmp32);
      }
      delete g[i];
    }
  }
};

extern "C" {

int wbc_gpu_device_count(int* count) {
  if (!count) return set_error(WBC_E_INVALID, "null argument");
  *count = 0;
  if (cudaGetDeviceCount(count) != cudaSuccess) {
    *count = 0;
    return set_error(WBC_E_NOT_BUILT, "no CUDA device available");
  }
  return WBC_OK;
}

int wbc_gpu_multi_create(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
                         const double* weights, const double* min_incident_weight, const uint32_t* edge_id,
                         const int* devices, int num_devices, int flags, wbc_gpu_multi** out) {
  if (!out || !devices || num_devices < 1) return set_error(WBC_E_INVALID, "devices / out required");
  *out = nullptr;
  HostCsr h;
  int rc = prepare_host(n, m, offsets, adjacency, weights, min_incident_weight, edge_id, h);
  if (rc) return rc;
  auto mh = new wbc_gpu_multi();
  mh->n = n;
  mh->m = m;
  const size_t D = static_cast<size_t>(num_devices);
  mh->g.assign(D, nullptr);
  mh->st.assign(D, nullptr);
  mh->d_node.assign(D, nullptr);
  mh->d_edge.assign(D, nullptr);
  mh->d_depth.assign(D, nullptr);
  mh->d_src.assign(D, nullptr);
  mh->src_cap.assign(D, 0);
  for (size_t i = 0; i < D; ++i) {
    if ((rc = upload_graph(h, devices[i], &mh->g[i]))) {
      delete mh;
      return rc;
    }
    cudaError_t err = cudaSetDevice(mh->g[i]->device);
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&mh->st[i], cudaStreamNonBlocking);
    if (err == cudaSuccess) mh->d_node[i] = dev_alloc<double>(n, err);
    if (err == cudaSuccess) mh->d_depth[i] = dev_alloc<uint32_t>(n, err);
    if (err == cudaSuccess && edge_id) mh->d_edge[i] = dev_alloc<double>(m, err);
    if (err == cudaSuccess && i == 0 && D > 1) mh->d_tmp = dev_alloc<double>(std::max(n, m), err);
    if (err == cudaSuccess && i == 0 && D > 1) mh->d_tmp32 = dev_alloc<uint32_t>(n, err);
    if (err != cudaSuccess) {
      delete mh;
      return set_error(WBC_E_NOMEM, std::string("multi-GPU setup: ") + cudaGetErrorString(err));
    }
  }
  // NCCL for distinct devices (or forced for a single device, to exercise it)
  std::vector<int> devs(D);
  for (size_t i = 0; i < D; ++i) devs[i] = mh->g[i]->device;
  std::vector<int> sorted = devs;
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  const bool want_nccl = (flags & WBC_MULTI_NO_NCCL) == 0 && distinct && (D > 1 || (flags & WBC_MULTI_FORCE_NCCL));
  if (want_nccl && nccl_api().ok) {
    mh->comm.assign(D, nullptr);
    if (nccl_api().CommInitAll(mh->comm.data(), static_cast<int>(D), devs.data()) == ncclSuccess)
      mh->use_nccl = true;
    else
      mh->comm.clear();
  }
  *out = mh;
  return WBC_OK;
}

void wbc_gpu_multi_destroy(wbc_gpu_multi* h) { delete h; }

int wbc_gpu_multi_info(wbc_gpu_multi* h, int* num_devices, int* uses_nccl) {
  if (!h) return set_error(WBC_E_INVALID, "null handle");
  if (num_devices) *num_devices = static_cast<int>(h->g.size());
  if (uses_nccl) *uses_nccl = h->use_nccl ? 1 : 0;
  return WBC_OK;
}

wbc_gpu_graph* wbc_gpu_multi_device_graph(wbc_gpu_multi* h, int i) {
  if (!h || i < 0 || static_cast<size_t>(i) >= h->g.size()) return nullptr;
  return h->g[i];
}

int wbc_gpu_multi_bc(wbc_gpu_multi* h, const uint32_t* sources, uint64_t k, uint32_t flags, double* node_bc,
                     double* edge_bc, uint32_t* depth_per_source, double* elapsed_s) {
  if (!h) return set_error(WBC_E_INVALID, "null handle");
  const bool edge = flags & WBC_EDGE_BC;
  const uint32_t n = h->n, m = h->m;
  if (!node_bc && n) return set_error(WBC_E_INVALID, "node_bc is required");
  if (edge && !edge_bc && m) return set_error(WBC_E_INVALID, "edge_bc is required");
  if (edge && !h->d_edge[0])
    return set_error(WBC_E_INVALID, "edge BC requested but the graph was created without edge_id");
  uint32_t lanes = 0;
  if (const int rl = strict_lanes_of(flags, &lanes)) return rl;
  if (sources)  // resolve_sources (engine.cpp:349-361)
    for (uint64_t i = 0; i < k; ++i)
      if (sources[i] >= n) return set_error(WBC_E_INVALID, "bc_parallel: source id out of range");
  const auto t0 = std::chrono::steady_clock::now();
  const size_t D = h->g.size();
  const uint64_t total = sources ? k : n;
  // strided shard of the source list per device (sources[i::D]); a strict
  // merge keeps every source on the first device (one ordered commit), the
  // others contribute exact zeros
  std::vector<std::vector<uint32_t>> shard(D);
  for (uint64_t i = 0; i < total; ++i)
    shard[lanes ? 0 : i % D].push_back(sources ? sources[i] : static_cast<uint32_t>(i));
  for (size_t d = 0; d < D; ++d) {
    wbc_gpu_graph* g = h->g[d];
    WBC_CUDA_TRY(cudaSetDevice(g->device));
    const cudaStream_t st = h->st[d];
    const uint64_t kd = shard[d].size();
    if (kd > h->src_cap[d]) {
      cudaFree(h->d_src[d]);
      cudaError_t err = cudaSuccess;
      h->d_src[d] = dev_alloc<uint32_t>(kd, err);
      if (err != cudaSuccess) return set_error(WBC_E_NOMEM, cudaGetErrorString(err));
      h->src_cap[d] = kd;
    }
    if (kd) WBC_CUDA_TRY(cudaMemcpyAsync(h->d_src[d], shard[d].data(), kd * 4, cudaMemcpyHostToDevice, st));
    if (n) {
      WBC_CUDA_TRY(cudaMemsetAsync(h->d_node[d], 0, uint64_t{n} * 8, st));
      WBC_CUDA_TRY(cudaMemsetAsync(h->d_depth[d], 0, uint64_t{n} * 4, st));
    }
    if (edge && m) WBC_CUDA_TRY(cudaMemsetAsync(h->d_edge[d], 0, uint64_t{m} * 8, st));
    // (a pageable H2D copy is staged before cudaMemcpyAsync returns: the
    // shard may go out of scope; the devices run concurrently)
    const int rc = launch_run(g, h->d_src[d], kd, edge, h->d_node[d], edge ? h->d_edge[d] : nullptr,
                              h->d_depth[d], st, false, false, lanes);
    if (rc) return rc;
  }
  // ---- the one collective: sum node / edge BC, max depth over devices
  if (h->use_nccl) {  // (a forced single-device comm runs it too)
    const NcclApi& nc = nccl_api();
    nc.GroupStart();
    ncclResult_t r = ncclSuccess;
    for (size_t d = 0; d < D && r == ncclSuccess; ++d) {
      r = nc.AllReduce(h->d_node[d], h->d_node[d], n, ncclFloat64, ncclSum, h->comm[d], h->st[d]);
      if (r == ncclSuccess && edge)
        r = nc.AllReduce(h->d_edge[d], h->d_edge[d], m, ncclFloat64, ncclSum, h->comm[d], h->st[d]);
      if (r == ncclSuccess)
        r = nc.AllReduce(h->d_depth[d], h->d_depth[d], n, ncclUint32, ncclMax, h->comm[d], h->st[d]);
    }
    const ncclResult_t r2 = nc.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
      return set_error(WBC_E_CUDA, std::string("ncclAllReduce: ") + nc.GetErrorString(r != ncclSuccess ? r : r2));
  } else if (D > 1) {
    for (size_t d = 1; d < D; ++d) {  // partials complete before the peer copies
      WBC_CUDA_TRY(cudaSetDevice(h->g[d]->device));
      WBC_CUDA_TRY(cudaStreamSynchronize(h->st[d]));
    }
    const int d0 = h->g[0]->device;
    WBC_CUDA_TRY(cudaSetDevice(d0));
    for (size_t d = 1; d < D; ++d) {
      const int dd = h->g[d]->device;
      WBC_CUDA_TRY(cudaMemcpyPeerAsync(h->d_tmp, d0, h->d_node[d], dd, uint64_t{n} * 8, h->st[0]));
      wbc_dev::add_f64_kernel<<<launch_grid(n), 256, 0, h->st[0]>>>(h->d_node[0], h->d_tmp, n);
      WBC_CUDA_TRY(cudaMemcpyPeerAsync(h->d_tmp32, d0, h->d_depth[d], dd, uint64_t{n} * 4, h->st[0]));
      wbc_dev::max_u32_kernel<<<launch_grid(n), 256, 0, h->st[0]>>>(h->d_depth[0], h->d_tmp32, n);
      if (edge) {
        WBC_CUDA_TRY(cudaMemcpyPeerAsync(h->d_tmp, d0, h->d_edge[d], dd, uint64_t{m} * 8, h->st[0]));
        wbc_dev::add_f64_kernel<<<launch_grid(m), 256, 0, h->st[0]>>>(h->d_edge[0], h->d_tmp, m);
      }
      WBC_CUDA_TRY(cudaGetLastError());
    }
  }
  WBC_CUDA_TRY(cudaSetDevice(h->g[0]->device));
  const cudaStream_t s0 = h->st[0];
  int rc = WBC_OK;
  if (flags & WBC_HALVED) {  // engine.cpp:451-454
    if ((rc = scale_async(h->d_node[0], n, 0.5, s0))) return rc;
    if (edge && (rc = scale_async(h->d_edge[0], m, 0.5, s0))) return rc;
  }
  if (n) {
    WBC_CUDA_TRY(cudaMemcpyAsync(node_bc, h->d_node[0], uint64_t{n} * 8, cudaMemcpyDeviceToHost, s0));
    if (depth_per_source)
      WBC_CUDA_TRY(cudaMemcpyAsync(depth_per_source, h->d_depth[0], uint64_t{n} * 4, cudaMemcpyDeviceToHost, s0));
  }
  if (edge && m) WBC_CUDA_TRY(cudaMemcpyAsync(edge_bc, h->d_edge[0], uint64_t{m} * 8, cudaMemcpyDeviceToHost, s0));
  WBC_CUDA_TRY(cudaStreamSynchronize(s0));
  if (elapsed_s) *elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return WBC_OK;
}

}  // extern "C"
