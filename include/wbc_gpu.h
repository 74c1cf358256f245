/* wbc_gpu.h -- C ABI of the B200-native weighted betweenness-centrality engine.
 *
 * This is the drop-in boundary for the reference's hot path
 *   wbc::BcResult wbc::bc_parallel(const CsrGraph&, const EngineOptions&)
 *   (/root/reference/proj/include/wbc/engine.hpp:130, src/engine.cpp:372-457).
 * The C++ wrapper in include/wbc/engine.hpp (same signature as the reference)
 * and the Python mirror (paper_1701_05975_b200/__init__.py) both call these
 * entry points; INTEGRATION.md shows the binding a reference maintainer adds.
 *
 * Conventions: 0 = OK, negative = error (WBC_E_*); no exceptions cross the
 * ABI; host buffers are caller-owned; the library owns device memory through
 * the opaque handle.  wbc_gpu_last_error() returns a thread-local message for
 * the last failing call on this thread.
 */
#ifndef WBC_GPU_H
#define WBC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes.  The C++ wrapper maps WBC_E_INVALID to std::invalid_argument
 * (the reference's exception type for bad sources / options,
 * engine.cpp:110-114,354,373-374) and everything else to std::runtime_error. */
#define WBC_OK 0
#define WBC_E_INVALID (-1)     /* bad argument: source out of range, bad graph arrays */
#define WBC_E_UNSUPPORTED (-2) /* weights not positive integers or dyadic fractions, distance bound >= 2^32 */
#define WBC_E_CUDA (-3)        /* CUDA runtime failure (message has cudaGetErrorString) */
#define WBC_E_NOMEM (-4)       /* device allocation failed */
#define WBC_E_NOT_BUILT (-5)   /* library built without a usable sm_100a device */

/* Flags for wbc_gpu_bc / wbc_gpu_bc_device. */
#define WBC_HALVED 1u   /* Normalization::Halved (result.hpp:9-12): scale by 0.5 */
#define WBC_EDGE_BC 2u  /* EngineOptions::compute_edge_bc (engine.hpp:111) */
/* EngineOptions::strict_merge (engine.hpp:112-115, engine.cpp:389-413): per-
 * source contributions are committed in source-list order and each source's
 * delta is summed in the reference's own slot order with the strategy's lane
 * width, so node / edge BC are bitwise the reference's bc_parallel output
 * for that lane width (any worker count).  Runs in batches on the team
 * kernel; slower than the default.  On a multi-GPU handle it runs on the
 * first device only. */
#define WBC_STRICT_MERGE 4u
#define WBC_LANE_WIDTH(w) (((uint32_t)(w) & 0xFFu) << 8) /* Strategy::lane_width; 0 means 1 */
#define WBC_DETERMINISTIC WBC_STRICT_MERGE /* SURVEY.md §8(b) name for the same flag */

typedef struct wbc_gpu_graph wbc_gpu_graph;

/* Upload an immutable CsrGraph (graph.hpp:56-69) to `device`.
 * Replaces: the reference has no upload; bc_parallel reads CsrGraph fields
 * directly (engine.cpp:59-212).
 *   offsets[n+1], adjacency[2m], weights[2m], min_incident_weight[n]
 *   (+inf for isolated vertices), edge_id[2m] (nullable: edge BC then
 *   unavailable).  Weights must be positive integers (all reference configs
 *   use assign_weights integers, generate.cpp:121-128) or dyadic fractions
 *   i / 2^k (k <= 20; e.g. 0.5, 2.5), which run scaled by the common 2^K:
 *   power-of-two scaling is exact in fp64, so the reference's distances are
 *   2^-K times exact integers.  (n-1)*max_weight (scaled) must stay below
 *   2^32-1 so that distances are exact u32; anything else returns
 *   WBC_E_UNSUPPORTED.  device < 0 selects the current CUDA device. */
int wbc_gpu_graph_create(uint32_t n, uint32_t m, const uint32_t* offsets,
                         const uint32_t* adjacency, const double* weights,
                         const double* min_incident_weight, const uint32_t* edge_id,
                         int device, wbc_gpu_graph** out);

/* Release the handle and all device memory it owns. */
void wbc_gpu_graph_destroy(wbc_gpu_graph* g);

/* Betweenness centrality over a source list, host buffers in and out.
 * Replaces: wbc::bc_parallel (engine.cpp:372-457) after option validation.
 *   sources == NULL: every vertex (EngineOptions::sources unset); otherwise
 *   the k listed sources in order, duplicates counted twice
 *   (engine.cpp:349-361); any source >= n -> WBC_E_INVALID with the
 *   reference's message.
 *   node_bc[n] (required), edge_bc[m] (required iff WBC_EDGE_BC),
 *   depth_per_source[n] (nullable; settlement rounds of each run source,
 *   0 otherwise -- result.hpp:19-22), elapsed_s (nullable; wall time from
 *   after validation to after normalization, like BcResult::elapsed,
 *   engine.cpp:375,455). */
int wbc_gpu_bc(wbc_gpu_graph* g, const uint32_t* sources, uint64_t k, uint32_t flags,
               double* node_bc, double* edge_bc, uint32_t* depth_per_source,
               double* elapsed_s);

/* Same computation with device-resident buffers on a caller stream
 * (cudaStream_t passed as void*; NULL = legacy default stream).  Outputs are
 * ACCUMULATED into d_node_bc / d_edge_bc (caller zeroes them), which is what
 * a multi-rank run needs before its one allreduce; depth entries of run
 * sources are overwritten.  Normalization is applied only if WBC_HALVED is
 * set.  Asynchronous: returns after enqueueing.  Sources are NOT range
 * checked on the device path (caller validated them). */
int wbc_gpu_bc_device(wbc_gpu_graph* g, const uint32_t* d_sources, uint64_t k,
                      uint32_t flags, double* d_node_bc, double* d_edge_bc,
                      uint32_t* d_depth_per_source, void* stream);

/* Parity/debug: one source's final traversal state, host buffers.
 * Replaces: solve_source + accumulate_dependencies (engine.hpp:93-99,
 * engine.cpp:183-222).  dist[n] (+inf unreachable), sigma[n], delta[n]
 * (nullable each), depth (nullable). */
int wbc_gpu_sssp_dump(wbc_gpu_graph* g, uint32_t source, double* dist, double* sigma,
                      double* delta, uint32_t* depth);

/* Level structure of one source, for the reference's level invariants
 * (test_engine.cpp:266-302: TraversalState::order / level_ends,
 * engine.hpp:49-65).  order[n] receives the settlement order in caller ids
 * (entries past *order_len are untouched), level_ends[n+1] the Eq. 4 level
 * boundaries (level L = order[level_ends[L], level_ends[L+1])),
 * *levels = depth.  Within a level the GPU's order is unspecified; compare
 * levels as sets. */
/* The kernel the last run launched, e.g. "bc_team_kernel<1024,2>"
 * (NUL-terminated, truncated to cap bytes). */
int wbc_gpu_last_kernel(wbc_gpu_graph* g, char* buf, size_t cap);

/* Test introspection: the shortest-path DAG edges one source recorded, per
 * level (pred[i] -> succ[i] in caller ids; level L's edges are
 * [dag_ends[L], dag_ends[L+1])).  pred/succ need room for 2m entries,
 * dag_ends for n+1.  *levels = depth; *overflow = 1 if the per-source DAG
 * buffer overflowed (the row-scan fallback then ran instead). */
int wbc_gpu_sssp_dag(wbc_gpu_graph* g, uint32_t source, uint32_t* pred, uint32_t* succ,
                     uint32_t* dag_ends, uint32_t* levels, uint32_t* overflow);

int wbc_gpu_sssp_levels(wbc_gpu_graph* g, uint32_t source, uint32_t* order, uint32_t* order_len,
                        uint32_t* level_ends, uint32_t* levels);

/* Introspection for benches/tests.  Any pointer may be NULL. */
int wbc_gpu_graph_info(wbc_gpu_graph* g, uint32_t* n, uint32_t* m, uint32_t* max_weight,
                       int* packed_slots, uint32_t* near_width, uint64_t* graph_bytes);

/* Tuning knobs (0 = automatic): threads per CTA (128/256/512/1024),
 * resident source slots (CTAs), near-window width of the pending split, and
 * the number of highest-degree vertices whose distances live in shared
 * memory (-1 = automatic). */
int wbc_gpu_set_tuning(wbc_gpu_graph* g, int threads_per_cta, int max_slots,
                       uint32_t near_width, int64_t hot_vertices);

/* Named tuning parameter (experiments/benches): "threads", "slots",
 * "near_width", "hot" (shared-memory distance entries; -1 auto), "l2hot"
 * (ids whose distance accesses carry an L2 evict-last hint; -1 auto),
 * "cluster" (team kernel CTAs per source; -1 auto, 0 per-CTA kernel),
 * "fill" (2-CTA fill clusters beside C >= 4 on the SMs they strand; -1 auto
 * = while the in-flight distances fit the L2 budget, 0 off, 1 on, k > 1: at
 * most k - 1 fill teams),
 * "flat" (distance-first kernel for flat graphs: -1 auto = degree <= 8 and
 * n >= 2^18, 0 off, 1 wherever eligible), "flat_delta" (its near-far window;
 * 0 = max weight), "flat_threads" (its CTA size: 256, 512 or 1024),
 * "flat_sq" (its shared-memory near-queue entries per buffer; -1 = auto:
 * what fits below the 64 KB carveout step, 0 = global-memory queues only).  Unknown
 * names return WBC_E_INVALID. */
int wbc_gpu_set_param(wbc_gpu_graph* g, const char* name, int64_t value);

/* Work counters of subsequent runs (off by default; a few atomics per
 * source): [0] settlement rounds, [1] relaxed slots, [2] near entries
 * scanned, [3] far entries scanned, [4] far refills, [5] distance
 * improvements, [6] DAG edges, [7..11] SM clock cycles spent by each CTA in
 * init / relax / threshold / settle / backward, [12..15] unused.  Summed over
 * the sources of the last run. */
int wbc_gpu_set_profiling(wbc_gpu_graph* g, int on);
int wbc_gpu_profile_counters(wbc_gpu_graph* g, uint64_t* out16);

/* Counters of the last run: [0]=slots used, [1]=threads per CTA,
 * [2]=sources that overflowed the DAG-edge buffer (row-scan fallback;
 * host-buffer runs only), [3]=kernel launches issued by the last call. */
int wbc_gpu_last_run_stats(wbc_gpu_graph* g, uint64_t* stats4);

/* The last run's outcome, read from the device after synchronising it:
 * [0]=slots used, [1]=threads per team, [2]=sources that overflowed the
 * DAG-edge buffer, [3]=kernel launches, [4]=sources handed to a fallback
 * kernel (0: since round 2 bc_flat_kernel completes every source),
 * [5]=1 when some shortest-path count sigma reached 2^53: sigma is an
 * integer-valued fp64 count (engine.cpp:73-77) that is exact only below it,
 * so BC from such a run may differ from the reference's.  Writes
 * min(cap, WBC_RUN_INFO_FIELDS) entries. */
#define WBC_RUN_INFO_FIELDS 6
int wbc_gpu_last_run_info(wbc_gpu_graph* g, uint64_t* out, uint32_t cap);

const char* wbc_gpu_last_error(void);

/* ---- host-side helpers (the CSR loader and generators of the reference,
 * re-implemented natively with identical output; exported for bindings) ---- */

typedef struct wbc_edge_list wbc_edge_list;
typedef struct wbc_csr wbc_csr;

/* parse_edge_list (graph.hpp:47): text in, edge list out.  On ParseError
 * returns WBC_E_PARSE and *err_line = the 1-based line. */
#define WBC_E_PARSE (-6)
int wbc_host_parse_edge_list(const char* text, size_t len, double default_weight,
                             wbc_edge_list** out, uint64_t* err_line);
wbc_edge_list* wbc_host_edges_new(uint64_t len, const uint64_t* u, const uint64_t* v,
                                  const double* w);
uint64_t wbc_host_edges_len(const wbc_edge_list* e);
uint64_t wbc_host_edges_self_loops(const wbc_edge_list* e);
void wbc_host_edges_get(const wbc_edge_list* e, uint64_t* u, uint64_t* v, double* w);
void wbc_host_edges_free(wbc_edge_list* e);

/* Generators (generate.hpp:20-35) with the reference's exact output streams,
 * plus two configs the reference lacks: Barabasi-Albert and a
 * row-major 4-neighbour grid.  Weights are 1 until wbc_host_assign_weights. */
int wbc_host_gen_er(uint64_t n, double avg_degree, uint64_t seed, wbc_edge_list** out);
int wbc_host_gen_kronecker(int scale, double avg_degree, uint64_t seed, wbc_edge_list** out);
int wbc_host_gen_ba(uint64_t n, uint32_t m_per_node, uint64_t seed, wbc_edge_list** out);
int wbc_host_gen_grid(uint32_t rows, uint32_t cols, wbc_edge_list** out);
int wbc_host_assign_weights(wbc_edge_list* e, int lo, int hi, uint64_t seed);
int wbc_host_sample_sources(uint32_t n, uint32_t k, uint64_t seed, uint32_t* out,
                            uint32_t* out_len);

/* build_csr (graph.hpp:74): identical CsrGraph arrays. */
int wbc_host_build_csr(const wbc_edge_list* e, wbc_csr** out);
void wbc_host_csr_dims(const wbc_csr* g, uint32_t* n, uint32_t* m, uint64_t* merged);
void wbc_host_csr_get(const wbc_csr* g, uint32_t* offsets, uint32_t* adjacency,
                      double* weights, uint32_t* edge_id, double* min_incident_weight,
                      uint64_t* original_id, uint32_t* edge_u, uint32_t* edge_v);
void wbc_host_csr_free(wbc_csr* g);

/* ---- One process, several GPUs (SURVEY.md §8(b) num_gpus, §8(e)). -------
 * Replaces: the reference's single-process bc_parallel over all workers
 * (engine.cpp:372-457), here over several devices: each holds a full CSR
 * replica, sources are sharded strided across them (sources[i::D]), and the
 * partial node/edge BC and depth vectors are combined by one NCCL all-reduce
 * (sum / sum / max) -- NCCL is loaded at run time (the process's own libnccl
 * if already loaded).  Without NCCL, or when a device repeats in `devices`
 * (test mode on one-GPU machines), device-to-device copies plus an add kernel
 * on the first device combine them instead.  Same argument contract and
 * error behaviour as wbc_gpu_graph_create / wbc_gpu_bc. */
typedef struct wbc_gpu_multi wbc_gpu_multi;
#define WBC_MULTI_NO_NCCL 1     /* combine with device copies even if NCCL is available */
#define WBC_MULTI_FORCE_NCCL 2  /* use NCCL even for a single device (tests) */
int wbc_gpu_device_count(int* count);
int wbc_gpu_multi_create(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
                         const double* weights, const double* min_incident_weight,
                         const uint32_t* edge_id, const int* devices, int num_devices, int flags,
                         wbc_gpu_multi** out);
int wbc_gpu_multi_bc(wbc_gpu_multi* h, const uint32_t* sources, uint64_t k, uint32_t flags,
                     double* node_bc, double* edge_bc, uint32_t* depth_per_source,
                     double* elapsed_s);
int wbc_gpu_multi_info(wbc_gpu_multi* h, int* num_devices, int* uses_nccl);
/* The per-device graph handle (tuning knobs, last_run_stats); owned by h. */
wbc_gpu_graph* wbc_gpu_multi_device_graph(wbc_gpu_multi* h, int i);
void wbc_gpu_multi_destroy(wbc_gpu_multi* h);

#ifdef __cplusplus
}
#endif

#endif /* WBC_GPU_H */
