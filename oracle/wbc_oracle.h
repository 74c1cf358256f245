/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the weighted-BC hot path.
 *
 * Plain-C restatement of the reference algorithms (citations are to
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker.
 * The product (paper_1701_05975_b200/) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * the reference's known-answer vectors (tests/golden/) and, when
 * oracle/_ref/libwbc_ref.so is present, bit-for-bit against the reference
 * library compiled from its own sources.
 */
#ifndef WBC_ORACLE_H
#define WBC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* build_csr (graph.cpp:75-133): first-appearance id compaction, min-weight
 * duplicate merge, two slots per canonical edge, emitted u->v then v->u in
 * canonical order.  Caller sizes: offsets >= 2*len+1, adjacency/weights/
 * edge_id >= 2*len, minw/original_id >= 2*len, edge_u/edge_v >= len.
 * Returns 0, or -1 on allocation failure. */
int orc_build_csr(uint64_t len, const uint64_t* u, const uint64_t* v, const double* w,
                  uint32_t* n_out, uint32_t* m_out, uint32_t* offsets, uint32_t* adjacency,
                  double* weights, uint32_t* edge_id, double* minw, uint64_t* original_id,
                  uint32_t* edge_u, uint32_t* edge_v, uint64_t* merged_out);

/* brandes_sequential (brandes.cpp:34-104), exact DAG equality (eps = 0).
 * k < 0 means every vertex as a source.  edge_bc may be NULL. */
int orc_brandes(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
                const double* weights, const uint32_t* edge_id, const uint32_t* sources,
                int64_t k, int halved, double* node_bc, double* edge_bc);

/* One source through the Eq. 4 round process with the work-efficient
 * strategy: init_state (engine.cpp:118-142), relax/threshold/settle loop
 * (engine.cpp:144-181, 214-222), then accumulate_dependencies
 * (engine.cpp:183-212).  order[n], ends[n+2].  node_acc may be NULL
 * (else node_acc[w] += delta[w] for w != s); edge_acc may be NULL.
 * less_equal selects the SettleRule::LessEqual negative control. */
int orc_eq4_source(uint32_t n, const uint32_t* offsets, const uint32_t* adjacency,
                   const double* weights, const uint32_t* edge_id, const double* minw,
                   uint32_t s, int less_equal, double* dist, double* sigma, double* delta,
                   uint32_t* order, uint32_t* order_len, uint32_t* ends, uint32_t* ends_len,
                   double* node_acc, double* edge_acc);

/* bc_parallel semantics (engine.cpp:372-457) restated sequentially: sources
 * in list order (duplicates counted twice), node/edge BC summed in source
 * order, depth_per_source[s] = rounds, Halved scales by 0.5.  k < 0 = all.
 * Returns -1 if a source is out of range (reference throws). */
int orc_bc_eq4(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
               const double* weights, const uint32_t* edge_id, const double* minw,
               const uint32_t* sources, int64_t k, int halved, double* node_bc,
               double* edge_bc, uint32_t* depth_per_source);

/* Diagnostic (design sizing only): per-source Eq. 4 process statistics.
 * stats[0]=rounds, [1]=sum over rounds of |pending| after relax,
 * [2]=relaxed slots, [3]=distance improvements, [4]=DAG edges,
 * [5]=max |pending|, [6]=max frontier, [7]=reached vertices,
 * [8]=max distance. */
int orc_eq4_profile(uint32_t n, const uint32_t* offsets, const uint32_t* adjacency,
                    const double* weights, const double* minw, uint32_t s, double* stats);

#ifdef __cplusplus
}
#endif

#endif
