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

struct GraphView {
  uint32_t n, m;
  const uint32_t* __restrict__ offsets;  // n+1
  const uint32_t* __restrict__ slots32;  // 2m, (neighbour << wbits) | weight
  const uint2* __restrict__ slots64;     // 2m, (neighbour, weight) when not packable
  const uint32_t* __restrict__ minw;     // n, min incident weight (kInfDist isolated)
  const uint32_t* __restrict__ edge_id;  // 2m or null
  uint32_t wbits, wmask;
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
  unsigned int* overflow;  // count of sources that used the row-scan fallback
  int keep_state;          // debug: zero-copy dump of slot 0 (sigma/delta kept)
};

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
                                                const uint32_t* dist, uint32_t c, int cnt,
                                                Shared<T>& sh) {
  using Scan = cub::BlockScan<uint32_t, T, cub::BLOCK_SCAN_WARP_SCANS>;
  const int tid = threadIdx.x;
  uint32_t deg = 0;
  if (tid < cnt) {
    const uint32_t v = __ldcg(order + c + tid);
    const uint32_t r0 = __ldg(g.offsets + v);
    deg = __ldg(g.offsets + v + 1) - r0;
    sh.v[tid] = v;
    sh.dv[tid] = __ldcg(dist + v);
    sh.row[tid] = r0;
    sh.acc[tid] = 0.0;
  }
  uint32_t pref, total;
  Scan(sh.scan).ExclusiveSum(deg, pref, total);
  if (tid < cnt) sh.pref[tid] = pref;
  return total;
}

template <int T, bool PACKED>
__global__ void __launch_bounds__(T) bc_sources_kernel(const RunParams p) {
  __shared__ Shared<T> sh;
  const GraphView& g = p.g;
  const int tid = threadIdx.x;
  const uint64_t off = static_cast<uint64_t>(blockIdx.x) * p.ws.n_stride;
  uint32_t* const dist = p.ws.dist + off;
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

  for (;;) {
    if (tid == 0) sh.src_idx = atomicAdd(p.counter, 1ULL);
    __syncthreads();
    const unsigned long long idx = sh.src_idx;
    if (idx >= p.k) break;
    const uint32_t s = p.sources ? __ldg(p.sources + idx) : static_cast<uint32_t>(idx);

    // ---- init_state (engine.cpp:118-142): d = inf, d[s] = 0, level 0 = {s}
    for (uint32_t i = tid; i < n; i += T) dist[i] = kInfDist;
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
      dist[s] = 0;
      order[0] = s;
      lev[0] = 0;
      lev[1] = 1;
      dag_ends[0] = 0;
    }
    __syncthreads();

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
        for (uint32_t e = tid; e < total; e += T) {
          const int j = find_row(sh.pref, cnt, e);
          const uint32_t slot = sh.row[j] + (e - sh.pref[j]);
          const uint32_t dv = sh.dv[j];
          uint32_t u, w;
          load_slot<PACKED>(g, slot, u, w);
          const uint32_t du = __ldcg(dist + u);
          if (dv >= w && du == dv - w) {
            // u precedes v on a shortest path: u settled in an earlier round,
            // so sigma[u] is final (see header).
            atomicAdd(&sh.acc[j], __ldcg(sigma + u));
            const uint32_t pos = group_append(&sh.dag_len);
            if (pos < dag_cap)
              dag[pos] = make_uint2(slot, sh.v[j]);
            else
              sh.dag_over = 1;
          }
          const uint32_t nd = dv + w;
          if (nd < du) {
            const uint32_t old = atomicMin(dist + u, nd);
            if (nd < old) {
              if (nd < Fu) {
                kmin = min(kmin, nd + __ldg(g.minw + u));
                if (old >= Fu) near_q[group_append(&sh.near_len)] = u;
              } else if (old == kInfDist) {
                far_q[group_append(&sh.far_len)] = u;
              }
            }
          }
        }
        __syncthreads();
        if (tid < cnt) {
          const uint32_t v = sh.v[tid];
          sigma[v] = (v == s) ? 1.0 : sh.acc[tid];
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
        for (uint32_t c = 0; c < far_len; c += T) {
          const uint32_t i = c + tid;
          uint32_t u = 0, du = 0;
          if (i < far_len) {
            u = __ldcg(far_q + i);
            du = __ldcg(dist + u);
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
      if (done) break;

      // ---------------- settle: d < Delta joins level nlev (in-place compaction)
      if (tid == 0) sh.keep = 0;
      __syncthreads();
      const uint32_t before = sh.order_len;
      uint32_t lkept = kInfDist;
      for (uint32_t c = 0; c < near_len; c += T) {
        const uint32_t i = c + tid;
        uint32_t u = 0, du = 0;
        if (i < near_len) {
          u = __ldcg(near_q + i);
          du = __ldcg(dist + u);
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
          for (uint32_t e = tid; e < total; e += T) {
            const int j = find_row(sh.pref, cnt, e);
            const uint32_t slot = sh.row[j] + (e - sh.pref[j]);
            uint32_t x, w;
            load_slot<PACKED>(g, slot, x, w);
            const uint32_t dx = __ldcg(dist + x);
            if (dx != kInfDist && dx == sh.dv[j] + w) {
              const uint32_t wv = sh.v[j];
              const double c2 = __ldcg(sigma + wv) / __ldcg(sigma + x) * (1.0 + __ldcg(delta + x));
              atomicAdd(&sh.acc[j], c2);
              if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + slot), c2);
            }
          }
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
    if (tid == 0 && p.depth) p.depth[s] = nlev;
    __syncthreads();
  }
}

__global__ void scale_kernel(double* x, uint64_t len, double f) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x[i] *= f;
}

__global__ void fill_u32_kernel(uint32_t* x, uint64_t len, uint32_t v) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x[i] = v;
}

}  // namespace wbc_dev
