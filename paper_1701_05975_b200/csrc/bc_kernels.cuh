// bc_kernels.cuh -- sm_100a kernels for the per-source Brandes hot path.
//
// One CTA owns one source at a time ("one block processes one root",
// PAPER.md:77) and runs the whole pipeline with CTA-local barriers only, so
// the 10^5-round grid config never pays a grid-wide sync.  A persistent grid
// of CTAs pulls sources from a global counter; every CTA has a private
// workspace slot in HBM (dist/sigma/delta/order/near/far/DAG-edge arrays).
//
// Per source (reference semantics in brackets):
//  (1) Eq. 4 round process [engine.cpp:118-222]: each round relaxes the
//      vertices settled in the previous round, then settles every pending
//      vertex with d < Delta, Delta = min over pending of d + min_w
//      [compute_threshold :149-156, settle_and_advance :158-181].
//      * relax is edge-balanced across the CTA (block scan of frontier
//        degrees + per-edge binary search), distances are u32 with
//        atomicMin (integer weights: exact [SURVEY §8 a'8]);
//      * the pending set is split near (d < F) / far (d >= F); Delta is
//        computed on near only while it is provably exact (Delta_near <= F,
//        every far key is >= F+1), and far is folded in otherwise.  Delta
//        for the next round is folded into the relax (min over improvements)
//        and the settle pass (min over kept entries): no extra pass.
//  (2) sigma [Alg. 2 L8-9; brute_force_bc's pull, brandes.cpp:139-159]: a
//      vertex settled in round r is relaxed in round r+1; the same row scan
//      pulls sigma from its DAG predecessors (d[u] + w == d[v]), which all
//      settled in earlier rounds, so sigma is exact integer fp64 and
//      order-independent -- no locks, no extra pass.  Each DAG edge found is
//      recorded (slot, v) per level.
//  (3) delta [accumulate_dependencies :183-212]: reverse level sweep over the
//      recorded DAG edges only (~1.05 per reached vertex on every config,
//      vs 2m row slots), delta[u] += sigma[u]/sigma[v]*(1+delta[v]) with the
//      reference's exact term, fused with node BC += delta (w != s) and the
//      optional edge BC.  If a source's DAG exceeds the buffer, a row-scan
//      pull fallback computes the same sums.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <cub/block/block_scan.cuh>

namespace wbc_dev {

namespace cg = cooperative_groups;

constexpr uint32_t kInfDist = 0xFFFFFFFFu;
#ifndef WBC_TEAM_UNROLL
#define WBC_TEAM_UNROLL 2
#endif
constexpr int kUnroll = WBC_TEAM_UNROLL;  // 32-edge groups per warp step in relax (R-MAT-20 at C=2: 1: 38.2, 2: 44.8, 3: 44.4, 4: 43.9, 6: 32.3, 8: 17.3 GTEPS)
#ifndef WBC_SRC_UNROLL
#define WBC_SRC_UNROLL 1
#endif
// the same, in bc_sources_kernel (ER-4096: 1: 16.9, 2: 16.65, 3: 16.3, 4: 15.25 GTEPS)
constexpr int kSrcUnroll = WBC_SRC_UNROLL;

// ---- L2 residency hints.  The CSR slot stream (read once per source, 4 B
// per slot, far larger than L2) is marked evict-first and skips L1; the
// distance entries of the highest-degree ids (the ones most neighbour
// accesses hit) are marked evict-last, so the stream cannot push them out.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* a, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ld_stream_u64(const uint2* a, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y) : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ld_cg_hint(const uint32_t* a, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t atom_min_hint(uint32_t* a, uint32_t v, uint64_t pol) {
  uint32_t r;
  asm volatile("atom.global.min.u32.L2::cache_hint %0, [%1], %2, %3;" : "=r"(r) : "l"(a), "r"(v), "l"(pol) : "memory");
  return r;
}


struct GraphView {
  uint32_t n, m;
  const uint32_t* __restrict__ offsets;  // n+1
  const uint32_t* __restrict__ slots32;  // 2m, (neighbour << wbits) | weight
  const uint2* __restrict__ slots64;     // 2m, (neighbour, weight) when not packable
  const uint32_t* __restrict__ minw;     // n, min incident weight (kInfDist isolated)
  const uint32_t* __restrict__ edge_id;  // 2m or null
  uint32_t wbits, wmask;
  int long_rows;  // average degree >= 32: group_row fast path
};

// Workspace of resident source slot `slot`: arrays of n_stride elements
// (dag: dag_cap entries) at base + slot * stride.
struct Workspace {
  uint32_t* dist;
  double* sigma;
  double* delta;
  uint32_t* order;       // settlement order; level L = order[lev[L], lev[L+1])
  uint32_t* level_ends;  // n_stride
  uint32_t* near_q;      // pending with d < F
  uint32_t* far_q;       // pending with d >= F at insertion (may hold stale ids)
  uint32_t* dag_ends;    // per level: DAG edges of level L = dag[de[L], de[L+1])
  uint2* dag;            // (slot of v's row pointing at predecessor u, v)
  // team kernel only (bc_team.cuh): per order position the distance, row
  // start and running edge prefix; second near/far buffers (ping-pong)
  uint32_t* ord_d;
  uint32_t* ord_row;
  uint32_t* epref;
  uint32_t* near_q2;
  uint32_t* far_q2;
  uint64_t n_stride;
  uint64_t dag_cap;
};

struct RunParams {
  GraphView g;
  Workspace ws;
  const uint32_t* sources;  // null: source index i is vertex i
  uint64_t k;
  unsigned long long* counter;
  double* node_bc;
  double* edge_bc;         // null unless edge BC requested
  uint32_t* depth;         // null or n entries
  uint32_t near_width;     // S: width of the near window
  unsigned int* overflow;  // [0] count of sources that used the row-scan fallback,
                           // [1] set when some sigma reached 2^53 (no longer exact)
  int keep_state;          // debug: write the shared-memory distances back (dump)
  const uint32_t* inv;     // original dense id -> device id (degree-descending relabel)
  uint32_t hot;            // device ids < hot keep their distance in shared memory
  uint32_t l2hot;          // device ids < l2hot get evict-last L2 hints
  unsigned long long* prof;  // null or kProfCounters per-run work counters
  const unsigned long long* k_dev;  // if set, the source count is read here (device-side)
  uint32_t team_base;               // first workspace slot of this launch (fill launches)
  // strict merge (bc_team.cuh): delta per source by the reference's row scan
  // (engine.cpp:183-212) into stage_node[i], edge terms into stage_edge[i];
  // strict_merge_kernel then adds them in source order
  uint32_t strict_lanes;            // 0: off; else the strategy's lane width
  uint32_t strict_group;            // threads per vertex row (power of two, >= lanes, <= 32)
  const uint32_t* ref_slots32;      // rows in the caller's slot order (relabelled ids)
  const uint2* ref_slots64;
  const uint32_t* ref_edge_id;
  double* stage_node;               // k x n_stride
  double* stage_edge;               // k x m, or null
  uint64_t src_base;                // sources == null: source index i is vertex src_base + i
};

// Work counters (accumulated per source when RunParams::prof is set).
enum ProfCounter {
  kProfRounds = 0,
  kProfRelaxSlots,
  kProfNearScanned,
  kProfFarScanned,
  kProfRefills,
  kProfImprovements,
  kProfDagEdges,
  kProfCyclesInit,
  kProfCyclesRelax,
  kProfCyclesThreshold,
  kProfCyclesSettle,
  kProfCyclesBackward,
  kProfAbortNear,   // reserved (kept for the counter block layout)
  kProfAbortFront,
  kProfAbortDag,
  kProfAbortDist,
  kProfCounters
};

// Distances: device ids below `hot` live in the CTA's shared memory (the
// degree-descending relabel puts the vertices that absorb most neighbour
// accesses there: on R-MAT-20 the top 5% of ids take 69% of them), the rest
// in the slot's global array.  Values only decrease within a source, so a
// stale read can only cost an extra atomic, never a wrong result.
struct DistView {
  uint32_t* sm;
  uint32_t* gl;
  uint32_t hot;     // ids below: shared memory
  uint32_t l2hot;   // ids below (and >= hot): global with an evict-last hint
  uint64_t keep;    // evict-last policy
  __device__ __forceinline__ uint32_t load(uint32_t u) const {
    if (u < hot) return *(volatile uint32_t*)(sm + u);
    return u < l2hot ? ld_cg_hint(gl + u, keep) : __ldcg(gl + u);
  }
  __device__ __forceinline__ uint32_t fetch_min(uint32_t u, uint32_t v) const {
    if (u < hot) return atomicMin(sm + u, v);
    return u < l2hot ? atom_min_hint(gl + u, v, keep) : atomicMin(gl + u, v);
  }
  __device__ __forceinline__ void store(uint32_t u, uint32_t v) const {
    if (u < hot)
      sm[u] = v;
    else
      gl[u] = v;
  }
};

// sigma is an integer-valued fp64 count (engine.cpp:73-77): exact in any
// summation order while every partial sum stays below 2^53, i.e. while the
// final value does.  A count at or above it is flagged (overflow[1]) so the
// caller knows sigma-derived results may differ from the reference's.
__device__ __forceinline__ void note_sigma(unsigned int* overflow, double s) {
  if (s >= 9007199254740992.0) atomicOr(overflow + 1, 1u);
}

template <bool PACKED>
__device__ __forceinline__ void load_slot(const GraphView& g, uint32_t e, uint32_t& u,
                                          uint32_t& w, uint64_t pol) {
  if constexpr (PACKED) {
    const uint32_t x = ld_stream_u32(g.slots32 + e, pol);
    u = x >> g.wbits;
    w = x & g.wmask;
  } else {
    const uint2 x = ld_stream_u64(g.slots64 + e, pol);
    u = x.x;
    w = x.y;
  }
}

template <bool PACKED>
__device__ __forceinline__ void load_slot(const GraphView& g, uint32_t e, uint32_t& u,
                                          uint32_t& w) {
  if constexpr (PACKED) {
    const uint32_t x = __ldg(g.slots32 + e);
    u = x >> g.wbits;
    w = x & g.wmask;
  } else {
    const uint2 x = __ldg(g.slots64 + e);
    u = x.x;
    w = x.y;
  }
}

// Largest j in [0, cnt) with pref[j] <= e (pref non-decreasing, pref[0] = 0).
__device__ __forceinline__ int find_row(const uint32_t* pref, int cnt, uint32_t e) {
  int lo = 0, hi = cnt - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= e)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Edge-balanced expansion of a staged chunk without a per-edge search.  The
// chunk's `total` edges (rows sh.row[j], prefix sh.pref[j], pref[cnt] =
// total) are cut into one contiguous range per warp; the warp walks its range
// 32 edges (a "group") at a time.  Every staged row has >= 1 edge (frontier
// vertices were reached through an edge; an isolated source has total == 0),
// so a group crosses at most 31 row ends: lane l loads the end of row j0+l,
// the ends inside the group are OR-reduced into a bit mask, and each lane's
// row is j0 + popc(mask below its position).  One LDS per lane per 32 edges
// instead of a log2(T)-step binary search per edge.
//
// group_row returns the lane's row for the group starting at e0 and advances
// j0 to the row holding e0 + 32.
__device__ __forceinline__ int group_row(const uint32_t* pref, int cnt, uint32_t e0, int& j0,
                                         bool long_rows = false) {
  // fast path (warp-uniform): the whole group lies in row j0 -- the common
  // case on graphs whose edges sit mostly in long rows (R-MAT-20: +2.6%;
  // enabled by GraphView::long_rows, it costs BA's shorter rows 1.7%)
  if (long_rows) {
    const uint32_t nx = j0 + 1 <= cnt ? pref[j0 + 1] : 0xFFFFFFFFu;
    if (nx >= e0 + 32) {
      const int j = j0;
      if (nx == e0 + 32) ++j0;
      return j;
    }
  }
  const int lane = threadIdx.x & 31;
  const int jl = j0 + 1 + lane;
  const uint32_t pe = jl <= cnt ? pref[jl] : 0xFFFFFFFFu;
  const uint32_t q = pe - e0;  // position of a row end inside the group
  const uint32_t bit = (pe > e0 && q < 32) ? (1u << q) : 0u;
  const uint32_t mask = __reduce_or_sync(0xffffffffu, bit);
  const int j = j0 + __popc(mask & ((2u << lane) - 1u));
  const int j31 = j0 + __popc(mask);
  j0 = j31 + ((j31 + 1 <= cnt && pref[j31 + 1] <= e0 + 32) ? 1 : 0);
  return j;
}

// The warp's contiguous edge range [b, e_end) of a chunk.
template <int T>
__device__ __forceinline__ bool warp_range(uint32_t total, uint32_t& b, uint32_t& e_end) {
  constexpr uint32_t kWarps = T / 32;
  const uint32_t warp = threadIdx.x >> 5;
  // round the per-warp share up to whole groups so groups stay aligned
  const uint32_t per = ((total + kWarps - 1) / kWarps + 31) & ~31u;
  b = min(total, per * warp);
  e_end = min(total, b + per);
  return b < e_end;
}

// Single-group-per-step expansion (cold paths: the row-scan delta fallback).
template <int T, class F>
__device__ __forceinline__ void expand_edges(const uint32_t* pref, int cnt, uint32_t total, F&& f) {
  uint32_t b, e_end;
  if (!warp_range<T>(total, b, e_end)) return;
  int j0 = find_row(pref, cnt, b);
  for (uint32_t e0 = b; e0 < e_end; e0 += 32) {
    const int j = group_row(pref, cnt, e0, j0);
    const uint32_t e = e0 + (threadIdx.x & 31);
    if (e < e_end) f(e, j);
  }
}

// Warp-aggregated append: one shared atomic per converged group.
__device__ __forceinline__ uint32_t group_append(uint32_t* counter) {
  cg::coalesced_group grp = cg::coalesced_threads();
  uint32_t base = 0;
  if (grp.thread_rank() == 0) base = atomicAdd(counter, grp.size());
  base = grp.shfl(base, 0);
  return base + grp.thread_rank();
}

__device__ __forceinline__ uint32_t block_min_to(uint32_t v, uint32_t* target) {
  v = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) atomicMin(target, v);
  return v;
}

template <int T>
struct Shared {
  typename cub::BlockScan<uint32_t, T, cub::BLOCK_SCAN_WARP_SCANS>::TempStorage scan;
  uint32_t v[T];
  uint32_t dv[T];
  uint32_t row[T];
  uint32_t pref[T + 1];
  double acc[T];
  unsigned long long src_idx;
  uint32_t near_len, far_len, order_len, dag_len, keep;
  uint32_t key_min, aux_min;
  int dag_over;
};

// Loads the frontier chunk order[c, c+cnt) into shared memory and returns
// the edge total.  Caller must __syncthreads() before reading sh.pref/row.
template <int T>
__device__ __forceinline__ uint32_t stage_chunk(const GraphView& g, const uint32_t* order,
                                                const DistView& dist, uint32_t c, int cnt,
                                                Shared<T>& sh) {
  using Scan = cub::BlockScan<uint32_t, T, cub::BLOCK_SCAN_WARP_SCANS>;
  const int tid = threadIdx.x;
  uint32_t deg = 0;
  if (tid < cnt) {
    const uint32_t v = __ldcg(order + c + tid);
    const uint32_t r0 = __ldg(g.offsets + v);
    deg = __ldg(g.offsets + v + 1) - r0;
    sh.v[tid] = v;
    sh.dv[tid] = dist.load(v);
    sh.row[tid] = r0;
    sh.acc[tid] = 0.0;
  }
  uint32_t pref, total;
  Scan(sh.scan).ExclusiveSum(deg, pref, total);
  if (tid < cnt) sh.pref[tid] = pref;
  return total;
}

template <int T, bool PACKED, bool PROF>
__global__ void __launch_bounds__(T, (T >= 1024 ? 1 : 1536 / T)) bc_sources_kernel(const RunParams p) {
  __shared__ Shared<T> sh;
  extern __shared__ uint32_t hot_dist[];
  const GraphView& g = p.g;
  const int tid = threadIdx.x;
  const uint64_t off = static_cast<uint64_t>(blockIdx.x) * p.ws.n_stride;
  const DistView dist{hot_dist, p.ws.dist + off, p.hot, p.l2hot, l2_policy_evict_last()};
  const uint64_t stream_pol = l2_policy_evict_first();
  double* const sigma = p.ws.sigma + off;
  double* const delta = p.ws.delta + off;
  uint32_t* const order = p.ws.order + off;
  uint32_t* const lev = p.ws.level_ends + off;
  uint32_t* const near_q = p.ws.near_q + off;
  uint32_t* const far_q = p.ws.far_q + off;
  uint32_t* const dag_ends = p.ws.dag_ends + off;
  uint2* const dag = p.ws.dag + static_cast<uint64_t>(blockIdx.x) * p.ws.dag_cap;
  const uint32_t dag_cap = static_cast<uint32_t>(p.ws.dag_cap);
  const uint32_t n = g.n;
  const uint32_t S = p.near_width;
  unsigned long long c_relax = 0, c_near = 0, c_far = 0, c_refill = 0, c_impr = 0;
  // phase clocks (thread 0, only when profiling)
  unsigned long long t_last = 0, t_phase[5] = {0, 0, 0, 0, 0};
  const bool timing = PROF && tid == 0;
  auto tick = [&](int k) {
    if (timing) {
      const unsigned long long t = clock64();
      t_phase[k] += t - t_last;
      t_last = t;
    }
  };

  for (;;) {
    if (tid == 0) sh.src_idx = atomicAdd(p.counter, 1ULL);
    __syncthreads();
    const unsigned long long idx = sh.src_idx;
    if (idx >= p.k) break;
    const uint32_t s_orig = p.sources ? __ldg(p.sources + idx) : static_cast<uint32_t>(idx);
    const uint32_t s = __ldg(p.inv + s_orig);
    if (timing) t_last = clock64();

    // ---- init_state (engine.cpp:118-142): d = inf, d[s] = 0, level 0 = {s}
    for (uint32_t i = tid; i < p.hot; i += T) hot_dist[i] = kInfDist;
    for (uint32_t i = p.hot + tid; i < n; i += T) dist.gl[i] = kInfDist;
    if (tid == 0) {
      sh.near_len = 0;
      sh.far_len = 0;
      sh.order_len = 1;
      sh.dag_len = 0;
      sh.dag_over = 0;
      sh.key_min = kInfDist;
      sh.aux_min = kInfDist;
    }
    __syncthreads();
    if (tid == 0) {
      dist.store(s, 0);
      order[0] = s;
      lev[0] = 0;
      lev[1] = 1;
      dag_ends[0] = 0;
    }
    __syncthreads();

    tick(0);
    uint32_t fb = 0, fe = 1, nlev = 1;  // frontier = order[fb, fe) = level nlev-1
    uint64_t F = S;                      // near window bound (d < F is near)
    uint32_t kept_min = kInfDist;        // min key of near entries kept by the last settle

    for (;;) {
      // ---------------- relax level nlev-1, pull its sigma, record DAG edges
      uint32_t kmin = kInfDist;
      const uint32_t Fu = F >= kInfDist ? kInfDist : static_cast<uint32_t>(F);
      for (uint32_t c = fb; c < fe; c += T) {
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(T), fe - c));
        const uint32_t total = stage_chunk<T>(g, order, dist, c, cnt, sh);
        if (tid == 0) sh.pref[cnt] = total;
        __syncthreads();
        c_relax += total;
        uint32_t wb, we;
        if (warp_range<T>(total, wb, we)) {
          int j0 = find_row(sh.pref, cnt, wb);
          // kSrcUnroll independent slot -> dist chains per lane: all slot loads,
          // then all distance loads, then the compare / atomic / append work.
          for (uint32_t e0 = wb; e0 < we; e0 += 32 * kSrcUnroll) {
            int jj[kSrcUnroll];
            uint32_t slot[kSrcUnroll], uu[kSrcUnroll], ww[kSrcUnroll], du[kSrcUnroll];
#pragma unroll
            for (int k = 0; k < kSrcUnroll; ++k) {
              const uint32_t eg = e0 + 32 * k;
              jj[k] = eg < we ? group_row(sh.pref, cnt, eg, j0) : 0;
              const uint32_t e = eg + (tid & 31);
              slot[k] = e < we ? sh.row[jj[k]] + (e - sh.pref[jj[k]]) : 0xFFFFFFFFu;
            }
#pragma unroll
            for (int k = 0; k < kSrcUnroll; ++k)
              if (slot[k] != 0xFFFFFFFFu) load_slot<PACKED>(g, slot[k], uu[k], ww[k], stream_pol);
#pragma unroll
            for (int k = 0; k < kSrcUnroll; ++k)
              if (slot[k] != 0xFFFFFFFFu) du[k] = dist.load(uu[k]);
#pragma unroll
            for (int k = 0; k < kSrcUnroll; ++k) {
              if (slot[k] == 0xFFFFFFFFu) continue;
              const int j = jj[k];
              const uint32_t u = uu[k], w = ww[k];
              const uint32_t dv = sh.dv[j];
              if (dv >= w && du[k] == dv - w) {
                // u precedes v on a shortest path: u settled in an earlier
                // round, so sigma[u] is final (see header).
                atomicAdd(&sh.acc[j], __ldcg(sigma + u));
                const uint32_t pos = group_append(&sh.dag_len);
                if (pos < dag_cap)
                  dag[pos] = make_uint2(slot[k], sh.v[j]);
                else
                  sh.dag_over = 1;
              }
              const uint32_t nd = dv + w;
              if (nd < du[k]) {
                const uint32_t old = dist.fetch_min(u, nd);
                if (nd < old) {
                  ++c_impr;
                  if (nd < Fu) {
                    kmin = min(kmin, nd + __ldg(g.minw + u));
                    if (old >= Fu) near_q[group_append(&sh.near_len)] = u;
                  } else if (old == kInfDist) {
                    far_q[group_append(&sh.far_len)] = u;
                  }
                }
              }
            }
          }
        }
        __syncthreads();
        if (tid < cnt) {
          const uint32_t v = sh.v[tid];
          sigma[v] = (v == s) ? 1.0 : sh.acc[tid];
          note_sigma(p.overflow, sh.acc[tid]);
          delta[v] = 0.0;
        }
        __syncthreads();
      }
      block_min_to(kmin, &sh.key_min);
      __syncthreads();
      if (tid == 0) dag_ends[nlev] = sh.dag_len;
      uint32_t thr = min(kept_min, sh.key_min);
      uint32_t near_len = sh.near_len, far_len = sh.far_len;
      __syncthreads();
      if (tid == 0) sh.key_min = kInfDist;
      tick(1);

      // ---------------- threshold: make the near-only Delta exact
      bool done = (near_len == 0 && far_len == 0);
      uint64_t far_min = kInfDist;
      while (!done && thr > F) {
        // fold far entries with d < F_new into near (in-place compaction)
        uint64_t F_new = F + S;
        if (far_min != kInfDist) {
          const uint64_t jump = far_min + S < thr ? far_min + S : static_cast<uint64_t>(thr);
          if (jump > F_new) F_new = jump;
        }
        const uint32_t Fo = F >= kInfDist ? kInfDist : static_cast<uint32_t>(F);
        const uint32_t Fn = F_new >= kInfDist ? kInfDist : static_cast<uint32_t>(F_new);
        if (tid == 0) {
          sh.keep = 0;
          sh.aux_min = kInfDist;
        }
        __syncthreads();
        uint32_t lkey = kInfDist, lfar = kInfDist;
        c_far += far_len;
        ++c_refill;
        for (uint32_t c = 0; c < far_len; c += T) {
          const uint32_t i = c + tid;
          uint32_t u = 0, du = 0;
          if (i < far_len) {
            u = __ldcg(far_q + i);
            du = dist.load(u);
          }
          __syncthreads();
          if (i < far_len && du >= Fo) {  // du < Fo: already near or settled
            if (du < Fn) {
              near_q[group_append(&sh.near_len)] = u;
              lkey = min(lkey, du + __ldg(g.minw + u));
            } else {
              far_q[group_append(&sh.keep)] = u;
              lfar = min(lfar, du);
            }
          }
        }
        block_min_to(lkey, &sh.key_min);
        block_min_to(lfar, &sh.aux_min);
        __syncthreads();
        thr = min(thr, sh.key_min);
        far_min = sh.aux_min;
        near_len = sh.near_len;
        far_len = sh.keep;
        F = F_new;
        __syncthreads();
        if (tid == 0) {
          sh.far_len = far_len;
          sh.key_min = kInfDist;
          sh.aux_min = kInfDist;
        }
        done = (near_len == 0 && far_len == 0);
      }
      tick(2);
      if (done) break;

      // ---------------- settle: d < Delta joins level nlev (in-place compaction)
      if (tid == 0) sh.keep = 0;
      __syncthreads();
      const uint32_t before = sh.order_len;
      uint32_t lkept = kInfDist;
      c_near += near_len;
      for (uint32_t c = 0; c < near_len; c += T) {
        const uint32_t i = c + tid;
        uint32_t u = 0, du = 0;
        if (i < near_len) {
          u = __ldcg(near_q + i);
          du = dist.load(u);
        }
        __syncthreads();
        if (i < near_len) {
          if (du < thr) {
            order[group_append(&sh.order_len)] = u;
          } else {
            near_q[group_append(&sh.keep)] = u;
            lkept = min(lkept, du + __ldg(g.minw + u));
          }
        }
      }
      block_min_to(lkept, &sh.aux_min);
      __syncthreads();
      kept_min = sh.aux_min;
      const uint32_t after = sh.order_len;
      __syncthreads();
      if (tid == 0) {
        sh.near_len = sh.keep;
        sh.aux_min = kInfDist;
        lev[nlev + 1] = after;
      }
      fb = before;
      fe = after;
      ++nlev;
      tick(3);
      // (the next relax's first __syncthreads orders these smem writes)
    }

    // ---------------- dependency accumulation, deepest level first
    __syncthreads();
    const bool use_dag = !sh.dag_over;
    if (use_dag) {
      for (uint32_t L = nlev - 1; L >= 1; --L) {
        const uint32_t b = __ldcg(dag_ends + L), e = __ldcg(dag_ends + L + 1);
        for (uint32_t i = b + tid; i < e; i += T) {
          const uint2 d = __ldcg(dag + i);
          uint32_t u, w;
          load_slot<PACKED>(g, d.x, u, w);
          const uint32_t v = d.y;
          // reference term: sw / sigma[v] * (1.0 + delta[v])  (engine.cpp:201)
          const double c = __ldcg(sigma + u) / __ldcg(sigma + v) * (1.0 + __ldcg(delta + v));
          atomicAdd(delta + u, c);
          if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + d.x), c);
        }
        __syncthreads();
        if (L >= 2) {  // level L-1 is final now; level 0 is the source itself
          const uint32_t pb = __ldcg(lev + L - 1), pe = __ldcg(lev + L);
          for (uint32_t q = pb + tid; q < pe; q += T) {
            const uint32_t w = __ldcg(order + q);
            atomicAdd(p.node_bc + w, __ldcg(delta + w));
          }
        }
      }
    } else {
      // Row-scan pull fallback (the reference's own loop shape): delta of
      // level L from all row slots, deepest level first.
      if (tid == 0) atomicAdd(p.overflow, 1u);
      for (int L = static_cast<int>(nlev) - 1; L >= 0; --L) {
        const uint32_t pb = __ldcg(lev + L), pe = __ldcg(lev + L + 1);
        for (uint32_t c = pb; c < pe; c += T) {
          const int cnt = static_cast<int>(min(static_cast<uint32_t>(T), pe - c));
          const uint32_t total = stage_chunk<T>(g, order, dist, c, cnt, sh);
          if (tid == 0) sh.pref[cnt] = total;
          __syncthreads();
          expand_edges<T>(sh.pref, cnt, total, [&](uint32_t e, int j) {
            const uint32_t slot = sh.row[j] + (e - sh.pref[j]);
            uint32_t x, w;
            load_slot<PACKED>(g, slot, x, w);
            const uint32_t dx = dist.load(x);
            if (dx != kInfDist && dx == sh.dv[j] + w) {
              const uint32_t wv = sh.v[j];
              const double c2 = __ldcg(sigma + wv) / __ldcg(sigma + x) * (1.0 + __ldcg(delta + x));
              atomicAdd(&sh.acc[j], c2);
              if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + slot), c2);
            }
          });
          __syncthreads();
          if (tid < cnt) {
            const uint32_t wv = sh.v[tid];
            delta[wv] = sh.acc[tid];
            if (L >= 1) atomicAdd(p.node_bc + wv, sh.acc[tid]);
          }
          __syncthreads();
        }
      }
    }
    __syncthreads();
    tick(4);
    if (tid == 0 && p.depth) p.depth[s_orig] = nlev;
    if (p.keep_state)
      for (uint32_t i = tid; i < p.hot; i += T) dist.gl[i] = hot_dist[i];
    if (PROF && tid == 0) {
      atomicAdd(p.prof + kProfRounds, nlev);
      atomicAdd(p.prof + kProfDagEdges, sh.dag_len);
      atomicAdd(p.prof + kProfRelaxSlots, c_relax);
      atomicAdd(p.prof + kProfNearScanned, c_near);
      atomicAdd(p.prof + kProfFarScanned, c_far);
      atomicAdd(p.prof + kProfRefills, c_refill);
      for (int k = 0; k < 5; ++k) {
        atomicAdd(p.prof + kProfCyclesInit + k, t_phase[k]);
        t_phase[k] = 0;
      }
      c_relax = c_near = c_far = c_refill = 0;
    }
    if (PROF) {
      c_impr = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c_impr));
      if ((tid & 31) == 0) atomicAdd(p.prof + kProfImprovements, c_impr);
      c_impr = 0;
    }
    __syncthreads();
  }
}

__global__ void scale_kernel(double* x, uint64_t len, double f) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x[i] *= f;
}

// out[perm[i]] += in[i]: device-id partial BC back to original dense ids.
__global__ void scatter_add_kernel(double* out, const double* in, const uint32_t* perm, uint64_t len) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[perm[i]] += in[i];
}

// Ordered commit of a strict batch (engine.cpp:389-413): acc[v] += stage[i][v]
// for i = 0..B-1 in source-list order, skipping v == source i when
// `sources_dev` is set.  One thread per entry: the sum order is fixed.
__global__ void strict_merge_kernel(double* acc, const double* stage, uint64_t stride, uint64_t len, int B,
                                    const uint32_t* sources, uint64_t src_base, const uint32_t* inv,
                                    int skip_source) {
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < len;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double a = acc[v];
    for (int i = 0; i < B; ++i) {
      if (skip_source) {
        const uint32_t so = sources ? __ldg(sources + i) : static_cast<uint32_t>(src_base + i);
        if (__ldg(inv + so) == v) continue;
      }
      a = __dadd_rn(a, __ldcg(stage + i * stride + v));
    }
    acc[v] = a;
  }
}

// dst += src (partial BC of another device, multi-GPU reduction without NCCL)
__global__ void add_f64_kernel(double* dst, const double* src, uint64_t len) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

// dst = max(dst, src) (depth_per_source of disjoint source shards)
__global__ void max_u32_kernel(uint32_t* dst, const uint32_t* src, uint64_t len) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = max(dst[i], src[i]);
}

__global__ void fill_u32_kernel(uint32_t* x, uint64_t len, uint32_t v) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x[i] = v;
}

}  // namespace wbc_dev
