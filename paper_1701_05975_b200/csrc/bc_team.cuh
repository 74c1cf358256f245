// bc_team.cuh -- the per-source Brandes pipeline run by a TEAM of C CTAs (one
// thread-block cluster) per source.
//
// Why teams: with one CTA per source, 148 sources are in flight and their
// distance arrays (4n bytes each: 2.6 MB at R-MAT-20, 388 MB together) cannot
// stay in the 126 MB L2, so every random dist[u] gather of the relax misses to
// HBM (ncu: 2.0 GB of DRAM traffic per source against 1.27 GB algorithmic,
// 32% L2 hit rate).  A cluster of C CTAs working on ONE source divides the
// number of in-flight sources by C (C = 8: 18 sources, 47 MB of distances),
// so the gathers hit L2 and HBM only streams the CSR slots.
//
// Same semantics and round structure as bc_sources_kernel (bc_kernels.cuh,
// reference engine.cpp:118-222 and :183-212); what changes is the
// decomposition:
//  * settle appends each settled vertex to the order together with its
//    distance, row start and the running edge prefix (a warp scan plus one
//    packed 64-bit atomicAdd per warp hands out (position, edge offset)
//    pairs), so the next relax splits the level's EDGES evenly across the C
//    CTAs without a scan, and stages its rows with coalesced loads;
//  * sigma is pulled with one fire-and-forget global fp64 RED per DAG edge
//    (a hub row may be split between CTAs; the sums are integer-valued, hence
//    exact in any order), and the relax issues the atomicMin, min-weight and
//    sigma accesses of all its unrolled groups before consuming any of them;
//    a DAG record holds the predecessor itself (the slot only when edge BC
//    needs edge_id), so the backward sweep gathers no CSR slot;
//    queue appends are ballot-aggregated, one atomic per queue per warp step;
//  * the near/far queues are ping-pong buffers (in-place compaction across
//    warps would race; one-warp teams get the same buffer twice, which is
//    safe because a warp step reads all its entries before it writes and a
//    write position never passes a read position);
//  * team scalars (queue append counters, Delta minima, the next source
//    index) live in a ring of 4 slots in rank 0's shared memory (DSMEM):
//    phase p appends/reduces into slot p%4, every thread reads slot p%4 right
//    after the barrier that ends phase p, and slot (p+2)%4 is cleared during
//    phase p -- its last readers finished before that phase began, and its
//    next writers start after the next barrier.  Queue lengths are therefore
//    team-uniform registers (base + appended count), never reset in place.
// C == 1 degenerates to one CTA with __syncthreads() as the team barrier.
#pragma once

#include <type_traits>

#include "bc_kernels.cuh"

#ifndef WBC_TEAM_REFILL_U
#define WBC_TEAM_REFILL_U 4
#endif
#ifndef WBC_TEAM_SETTLE_U
#define WBC_TEAM_SETTLE_U 2
#endif
#ifndef WBC_TEAM_BACK_U
#define WBC_TEAM_BACK_U 4
#endif

namespace wbc_dev {

struct TeamRed {
  unsigned long long ord;  // settle: (count << 32) | edges appended to the order
  unsigned long long src;  // next source index (fetched by the leader)
  uint32_t near_app, far_app, dag_app, keep_app;
  uint32_t min1, min2;
  uint32_t flags;
  uint32_t pad;
};

__device__ __forceinline__ void team_red_reset(TeamRed& r) {
  r.ord = 0;
  r.near_app = r.far_app = r.dag_app = r.keep_app = 0;
  r.min1 = r.min2 = kInfDist;
  r.flags = 0;
}

// Frontier vertices staged per chunk: T, and at least 128 so a one-warp team
// relaxes a typical large-diameter level (~50 vertices) in one chunk.
// (4096-vertex chunks for T = 1024 measured 2.4x SLOWER: the larger shared
// footprint shrinks L1 to ~30 KB and the kernel's register spills thrash.)
template <int T>
constexpr int team_chunk() { return T < 128 ? 128 : T; }

template <int T>
struct TeamShared {
  static constexpr int CH = team_chunk<T>();
  uint32_t v[CH];
  uint32_t dv[CH];
  uint32_t rowadj[CH];  // row start + chunk base - first edge (mod 2^32)
  uint32_t pref[CH + 1];
  TeamRed ring[4];     // used through rank 0's copy
  uint32_t bcast;
  unsigned long long src_idx;  // launch-relative index of the current source (strict merge)
};

// Warp-aggregated append to a (possibly remote) counter; returns the slot.
__device__ __forceinline__ uint32_t team_append(uint32_t* counter) {
  cg::coalesced_group grp = cg::coalesced_threads();
  uint32_t base = 0;
  if (grp.thread_rank() == 0) base = atomicAdd(counter, grp.size());
  base = grp.shfl(base, 0);
  return base + grp.thread_rank();
}

// Distances of a team's source: ids below `hot` (the degree-descending
// relabel puts the most-gathered vertices first) carry the L2 evict-last
// hint, the rest evict-normal; the policy is selected per access in a
// register (no branch).  hot = n marks every entry.
#ifndef WBC_TEAM_L1
#define WBC_TEAM_L1 1
#endif
// Single-CTA teams own every word of their workspace, so reads of it may go
// through L1 (ld.ca; coherent within the CTA after a barrier): bit 0 the
// distances, bit 1 sigma / delta.  Clusters read words other SMs wrote: L2.
template <int C, int BIT, class X>
__device__ __forceinline__ X ld_team(const X* p) {
  if constexpr (C == 1 && (WBC_TEAM_L1 >> BIT & 1))
    return __ldca(p);
  else
    return __ldcg(p);
}

struct TeamDist {
  uint32_t* gl;
  uint64_t keep, norm;
  uint32_t hot;
  __device__ __forceinline__ uint64_t pol(uint32_t u) const { return u < hot ? keep : norm; }
  __device__ __forceinline__ uint32_t load(uint32_t u) const { return ld_cg_hint(gl + u, pol(u)); }
  template <int C>
  __device__ __forceinline__ uint32_t get(uint32_t u) const {
    if constexpr (C == 1 && (WBC_TEAM_L1 & 1))
      return __ldca(gl + u);
    else
      return load(u);
  }
  __device__ __forceinline__ uint32_t fetch_min(uint32_t u, uint32_t v) const {
    return atom_min_hint(gl + u, v, pol(u));
  }
};

__device__ __forceinline__ void team_min(uint32_t v, uint32_t* target) {
  v = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v != kInfDist) atomicMin(target, v);
}

// Largest j in [lo, hi) with key[j] <= x (key non-decreasing, key[lo] <= x),
// found by the whole CTA with T-ary sampling: ceil(log_T(hi-lo)) rounds of
// one coalesced load + one __syncthreads_count.
template <int T>
__device__ __forceinline__ uint32_t block_find(const uint32_t* key, uint32_t lo, uint32_t hi, uint32_t x) {
  while (hi - lo > 1) {
    const uint32_t len = hi - lo;
    const uint32_t q = lo + static_cast<uint32_t>((static_cast<uint64_t>(len) * threadIdx.x) / T);
    const int ok = __ldcg(key + q) <= x;
    const int c = __syncthreads_count(ok);  // >= 1: sample 0 is lo
    const uint32_t t = static_cast<uint32_t>(c - 1);
    const uint32_t nlo = lo + static_cast<uint32_t>((static_cast<uint64_t>(len) * t) / T);
    const uint32_t nhi = (t + 1 < T) ? lo + static_cast<uint32_t>((static_cast<uint64_t>(len) * (t + 1)) / T) : hi;
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// Per-warp compaction queues of the two-pass relax (dynamic shared memory):
// 5 arrays of kTeamQ u32 per warp; a warp holds < 32 entries between drains
// and adds at most 32 * team_unroll per step.
// Relax groups per warp step: 3 for 1024-thread teams (R-MAT-20 at C = 4:
// 50.7 vs 48.6 GTEPS at 2, 48.7 at 4; R-MAT-24: 35.3 vs 35.0; BA-65536 at
// C = 1: 33.2 vs 32.7 at 2, 30.0 at 1), kUnroll for one-warp teams.
#ifndef WBC_TEAM_CUNROLL
#define WBC_TEAM_CUNROLL 3
#endif
template <int T, int C>
constexpr int team_unroll() { return T >= 1024 ? WBC_TEAM_CUNROLL : kUnroll; }
constexpr uint32_t kTeamQ = 32 * (WBC_TEAM_CUNROLL > kUnroll ? WBC_TEAM_CUNROLL : kUnroll) + 32;
__host__ __device__ constexpr size_t team_q_bytes(int threads) { return size_t(threads / 32) * 5 * kTeamQ * 4; }
template <int T>
constexpr size_t team_sh_bytes() { return (sizeof(TeamShared<T>) + 15) / 16 * 16; }
// Dynamic shared memory of a team CTA: the staged chunk + phase ring, then the
// per-warp queues.
#ifndef WBC_TEAM_SMEM_PAD
#define WBC_TEAM_SMEM_PAD 0
#endif
inline size_t team_dyn_smem(int threads) {
  return threads <= 32 ? team_sh_bytes<32>() + team_q_bytes(32) : team_sh_bytes<1024>() + team_q_bytes(1024) + WBC_TEAM_SMEM_PAD;
}

// 1024-thread CTAs: one per SM.  32-thread CTAs (one warp per source, for
// large-diameter graphs whose rounds are latency-bound): 16 per SM, 128 regs.
constexpr int team_min_blocks(int threads) { return threads >= 1024 ? 1 : (threads >= 128 ? 2048 / threads : 16); }

template <int T, int C, bool PACKED, bool PROF>
__global__ void __launch_bounds__(T, team_min_blocks(T)) bc_team_kernel(const RunParams p) {
  extern __shared__ __align__(16) unsigned char team_raw[];
  TeamShared<T>& sh = *reinterpret_cast<TeamShared<T>*>(team_raw);
  uint32_t* const team_q = reinterpret_cast<uint32_t*>(team_raw + team_sh_bytes<T>());
  const GraphView& g = p.g;
  const int tid = threadIdx.x;
  uint32_t rank = 0;
  TeamRed* ring = sh.ring;
  if constexpr (C > 1) {
    cg::cluster_group cl = cg::this_cluster();
    rank = cl.block_rank();
    ring = cl.map_shared_rank(sh.ring, 0);
  }
  const bool leader = rank == 0 && tid == 0;
  const uint32_t team = p.team_base + blockIdx.x / C;
  const uint64_t off = static_cast<uint64_t>(team) * p.ws.n_stride;
  const uint64_t keep_pol = l2_policy_evict_last();
  const uint64_t stream_pol = l2_policy_evict_first();
  const TeamDist dist{p.ws.dist + off, keep_pol, l2_policy_evict_normal(), p.l2hot};
  double* const sigma = p.ws.sigma + off;
  double* const delta = p.ws.delta + off;
  uint32_t* const order = p.ws.order + off;
  uint32_t* const ord_d = p.ws.ord_d + off;
  uint32_t* const ord_row = p.ws.ord_row + off;
  uint32_t* const epref = p.ws.epref + off;
  uint32_t* const lev = p.ws.level_ends + off;
  uint32_t* const nq0 = p.ws.near_q + off;
  uint32_t* const nq1 = p.ws.near_q2 + off;
  uint32_t* const fq0 = p.ws.far_q + off;
  uint32_t* const fq1 = p.ws.far_q2 + off;
  uint32_t* const dag_ends = p.ws.dag_ends + off;
  uint2* const dag = p.ws.dag + static_cast<uint64_t>(team) * p.ws.dag_cap;
  const uint32_t dag_cap = static_cast<uint32_t>(p.ws.dag_cap);
  const uint32_t n = g.n;
  const uint32_t S = p.near_width;
  constexpr uint32_t TT = static_cast<uint32_t>(T) * C;  // team threads
  const uint32_t gtid = rank * T + tid;                 // team thread id

  unsigned long long c_relax = 0, c_near = 0, c_far = 0, c_refill = 0, c_impr = 0;
  unsigned long long t_last = 0, t_phase[5] = {0, 0, 0, 0, 0};
  const bool timing = PROF && leader;
  auto tick = [&](int k) {
    if (timing) {
      const unsigned long long t = clock64();
      t_phase[k] += t - t_last;
      t_last = t;
    }
  };

  uint32_t ph = 0;
  auto tsync = [&]() {
    if constexpr (C == 1)
      __syncthreads();
    else
      cg::this_cluster().sync();
    ++ph;
    if (leader) team_red_reset(ring[(ph + 2) & 3]);
  };
  auto cur = [&]() -> TeamRed& { return ring[ph & 3]; };
  auto prev = [&]() -> TeamRed& { return ring[(ph - 1) & 3]; };

  if (tid == 0 && rank == 0) {
    for (int k = 0; k < 4; ++k) team_red_reset(sh.ring[k]);
    sh.ring[0].src = atomicAdd(p.counter, 1ULL);
  }

  // Stages the edges [cb, my_e) of the level's vertices starting at order
  // position j (edge prefix epref, vertices j.. have epref < my_e) into
  // shared memory; returns the chunk's vertex count and sets ce.
  constexpr int CH = TeamShared<T>::CH;
  auto stage = [&](uint32_t j, uint32_t fe, uint32_t cb, uint32_t my_e, uint32_t Ee, uint32_t& ce) -> int {
    constexpr int R = CH / T;
    uint32_t gs[R], ov[R], od[R], orow[R];
    bool use[R];
    // every load of the chunk in flight before the first barrier
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t jt = j + r * T + tid;
      gs[r] = jt < fe ? __ldcg(epref + jt) : Ee;
      ov[r] = jt < fe ? __ldcg(order + jt) : 0u;
      od[r] = jt < fe ? __ldcg(ord_d + jt) : 0u;
      orow[r] = jt < fe ? __ldcg(ord_row + jt) : 0u;
    }
    const uint32_t nxt = (tid == T - 1 && j + CH < fe) ? __ldcg(epref + j + CH) : Ee;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t t = r * T + tid;
      use[r] = j + t < fe && gs[r] < my_e;
      if (use[r]) {
        sh.v[t] = ov[r];
        sh.dv[t] = od[r];
        sh.rowadj[t] = orow[r] + cb - gs[r];
        sh.pref[t] = (gs[r] > cb ? gs[r] : cb) - cb;
      }
    }
    if (tid == T - 1) sh.bcast = nxt;
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) cnt += __syncthreads_count(use[r]);
    ce = (cnt < CH) ? my_e : min(sh.bcast, my_e);
    if (tid == 0) sh.pref[cnt] = ce - cb;
    __syncthreads();
    return cnt;
  };

  const unsigned long long k_total = p.k_dev ? __ldcg(p.k_dev) : p.k;
  for (;;) {
    tsync();
    const unsigned long long idx = prev().src;
    if (idx >= k_total) break;
    const uint32_t s_orig = p.sources ? __ldg(p.sources + idx) : static_cast<uint32_t>(p.src_base + idx);
    const uint32_t s = __ldg(p.inv + s_orig);
    if (tid == 0) sh.src_idx = idx;  // read back by the strict backward (keeps idx out of registers)
    if (timing) t_last = clock64();

    // ---- init_state (engine.cpp:118-142): d = inf except d[s] = 0, level 0 = {s}
    for (uint32_t i = gtid; i < n; i += TT) dist.gl[i] = (i == s) ? 0u : kInfDist;
    const uint32_t s_row = __ldg(g.offsets + s);
    const uint32_t s_deg = __ldg(g.offsets + s + 1) - s_row;
    if (leader) {
      order[0] = s;
      ord_d[0] = 0;
      ord_row[0] = s_row;
      epref[0] = 0;
      sigma[s] = 1.0;
      delta[s] = 0.0;
      lev[0] = 0;
      lev[1] = 1;
      dag_ends[0] = 0;
    }
    // team-uniform registers
    uint32_t fb = 0, fe = 1, nlev = 1, ord_len = 1, ord_edges = s_deg, Eb = 0, Ee = s_deg;
    uint32_t near_len = 0, far_len = 0, dag_len = 0;
    int nc = 0, fc = 0;
    uint64_t F = S;
    uint32_t kept_min = kInfDist;
    bool dag_over = false;
    tsync();
    tick(0);

    for (;;) {
      // ---------------- relax level nlev-1, pull its sigma, record DAG edges
      {
        TeamRed& R = cur();
        uint32_t kmin = kInfDist;
        bool over = false;
        uint32_t* const nqc = nc ? nq1 : nq0;
        uint32_t* const fqc = fc ? fq1 : fq0;
        const uint32_t Fu = F >= kInfDist ? kInfDist : static_cast<uint32_t>(F);
        const uint32_t E = Ee - Eb;
        const uint32_t my_b = Eb + static_cast<uint32_t>((static_cast<uint64_t>(E) * rank) / C);
        const uint32_t my_e = Eb + static_cast<uint32_t>((static_cast<uint64_t>(E) * (rank + 1)) / C);
        c_relax += (rank == 0) ? E : 0;
        if (my_b < my_e) {
          uint32_t j = C == 1 ? fb : block_find<T>(epref, fb, fe, my_b);
          uint32_t cb = my_b;
          while (cb < my_e) {
            uint32_t ce;
            const int cnt = stage(j, fe, cb, my_e, Ee, ce);
            const uint32_t total = ce - cb;
            // one contiguous edge range per warp (measured: handing out
            // 128-edge blocks dynamically was not faster)
            uint32_t wb, we;
            const uint32_t lane = tid & 31;
            if (warp_range<T>(total, wb, we)) {
              int j0 = find_row(sh.pref, cnt, wb);
              const uint32_t lt = (1u << lane) - 1u;
              uint32_t* const q = team_q + (tid >> 5) * (5 * kTeamQ);
              uint32_t* const qiu = q;               // improvement candidates: u
              uint32_t* const qid = q + kTeamQ;      //   tentative distance
              uint32_t* const qpu = q + 2 * kTeamQ;  // DAG predecessors: u
              uint32_t* const qpv = q + 3 * kTeamQ;  //   v (row owner)
              uint32_t* const qps = q + 4 * kTeamQ;  //   slot of v's row
              uint32_t iq_n = 0, pq_n = 0;           // warp-uniform queue lengths
              // Pass 2a: the last `m` improvement candidates, one per lane:
              // atomicMin and min-weight gather in flight together; Delta
              // candidates need no atomic result (a lane that lost the race
              // recorded a key >= the winner's); queue appends ballot-aggregated.
              auto drain_imp = [&](uint32_t m) {
                const uint32_t i = iq_n - m + lane;
                const bool act = lane < m;
                uint32_t u = 0, nd = 0, old = kInfDist, mw = 0;
                if (act) {
                  u = qiu[i];
                  nd = qid[i];
                  old = dist.fetch_min(u, nd);
                  if (nd < Fu) mw = __ldg(g.minw + u);
                }
                if (act && nd < Fu) kmin = min(kmin, nd + mw);
                const bool imp = act && nd < old;
                c_impr += imp;
                const uint32_t bn = __ballot_sync(0xffffffffu, imp && nd < Fu && old >= Fu);
                const uint32_t bf = __ballot_sync(0xffffffffu, imp && nd >= Fu && old == kInfDist);
                if (bn | bf) {
                  uint32_t b_n = 0, b_f = 0;
                  if (lane == 0) {
                    if (bn) b_n = atomicAdd(&R.near_app, __popc(bn));
                    if (bf) b_f = atomicAdd(&R.far_app, __popc(bf));
                  }
                  b_n = near_len + __shfl_sync(0xffffffffu, b_n, 0);
                  b_f = far_len + __shfl_sync(0xffffffffu, b_f, 0);
                  if (bn >> lane & 1u) nqc[b_n + __popc(bn & lt)] = u;
                  if (bf >> lane & 1u) fqc[b_f + __popc(bf & lt)] = u;
                }
                iq_n -= m;
              };
              // Pass 2b: the last `m` DAG predecessors: sigma pull (fp64 RED,
              // integer-valued so exact in any order) and the DAG record.
              auto drain_pred = [&](uint32_t m) {
                const uint32_t i = pq_n - m + lane;
                const bool act = lane < m;
                uint32_t u = 0, v = 0, sl = 0;
                double sg = 0.0;
                if (act) {
                  u = qpu[i];
                  v = qpv[i];
                  sl = qps[i];
                  sg = ld_team<C, 1>(sigma + u);
                }
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&R.dag_app, m);
                base = dag_len + __shfl_sync(0xffffffffu, base, 0);
                if (act) {
                  atomicAdd(sigma + v, sg);
                  // (predecessor, v); (slot of v's row, v) when edge BC needs edge_id
                  if (base + lane < dag_cap)
                    dag[base + lane] = make_uint2(p.edge_bc ? sl : u, v);
                  else
                    over = true;
                }
                pq_n -= m;
              };
              constexpr int kTU = team_unroll<T, C>();
              // Pass 1: stream kTU groups of 32 edges; software-pipelined:
              // the next step's slot words are in flight while this step's
              // distance gathers resolve.  Only lanes that need more work are
              // kept (compacted into the warp's queues).
              // Slot words stay packed until used (PACKED: one register).
              using Word = typename std::conditional<PACKED, uint32_t, uint2>::type;
              constexpr Word kNoWord = Word{};
              int jj[kTU];
              Word xw[kTU];
              auto fetch = [&](uint32_t e0) {
                uint32_t slot[kTU];
#pragma unroll
                for (int k = 0; k < kTU; ++k) {
                  const uint32_t eg = e0 + 32 * k;
                  jj[k] = eg < we ? group_row(sh.pref, cnt, eg, j0, g.long_rows) : 0;
                  const uint32_t e = eg + lane;
                  slot[k] = e < we ? sh.rowadj[jj[k]] + e : 0xFFFFFFFFu;
                }
#pragma unroll
                for (int k = 0; k < kTU; ++k) {
                  xw[k] = kNoWord;
                  if (slot[k] != 0xFFFFFFFFu) {
                    if constexpr (PACKED)
                      xw[k] = ld_stream_u32(g.slots32 + slot[k], stream_pol);
                    else
                      xw[k] = ld_stream_u64(g.slots64 + slot[k], stream_pol);
                  }
                }
              };
              auto nbr = [&](const Word& x) -> uint32_t {
                if constexpr (PACKED) return x >> g.wbits; else return x.x;
              };
              auto wgt = [&](const Word& x) -> uint32_t {
                if constexpr (PACKED) return x & g.wmask; else return x.y;
              };
              fetch(wb);
              for (uint32_t e0 = wb; e0 < we; e0 += 32 * kTU) {
                const uint32_t cwe = we;
                uint32_t du[kTU];
                Word cx[kTU];
                int cj[kTU];
#pragma unroll
                for (int k = 0; k < kTU; ++k) {
                  const bool valid = e0 + 32 * k + lane < cwe;
                  du[k] = valid ? dist.template get<C>(nbr(xw[k])) : 0u;
                  cx[k] = xw[k];
                  cj[k] = jj[k];
                }
                if (e0 + 32 * kTU < we) fetch(e0 + 32 * kTU);
#pragma unroll
                for (int k = 0; k < kTU; ++k) {
                  const uint32_t e = e0 + 32 * k + lane;
                  const bool valid = e < cwe;
                  const uint32_t dv = sh.dv[cj[k]];
                  const uint32_t u = nbr(cx[k]), w = wgt(cx[k]);
                  const uint32_t nd = dv + w;
                  // u precedes v on a shortest path (d[u] + w == d[v]); u then
                  // settled in an earlier round, so sigma[u] is final
                  const bool isp = valid && du[k] != kInfDist && du[k] + w == dv;
                  const bool isi = valid && nd < du[k];
                  const uint32_t bp = __ballot_sync(0xffffffffu, isp);
                  const uint32_t bi = __ballot_sync(0xffffffffu, isi);
                  if (isi) {
                    const uint32_t pos = iq_n + __popc(bi & lt);
                    qiu[pos] = u;
                    qid[pos] = nd;
                  }
                  if (isp) {
                    const uint32_t pos = pq_n + __popc(bp & lt);
                    qpu[pos] = u;
                    qpv[pos] = sh.v[cj[k]];
                    qps[pos] = sh.rowadj[cj[k]] + e;
                  }
                  iq_n += __popc(bi);
                  pq_n += __popc(bp);
                }
                if (iq_n >= 32 || pq_n >= 32) {
                  __syncwarp();
                  while (iq_n >= 32) drain_imp(32);
                  while (pq_n >= 32) drain_pred(32);
                  __syncwarp();
                }
              }
              __syncwarp();
              if (iq_n) drain_imp(iq_n);
              if (pq_n) drain_pred(pq_n);
            }
            __syncthreads();  // staged chunk fully consumed
            j += cnt;
            cb = ce;
          }
        }
        team_min(kmin, &R.min1);
        if (over) R.flags = 1;
      }
      tsync();
      uint32_t thr;
      {
        TeamRed& Q = prev();
        near_len += Q.near_app;
        far_len += Q.far_app;
        dag_len += Q.dag_app;
        thr = min(kept_min, Q.min1);
        dag_over = dag_over || Q.flags;
      }
      if (leader) dag_ends[nlev] = dag_len;
      tick(1);

      // ---------------- threshold: make the near-only Delta exact
      bool done = (near_len == 0 && far_len == 0);
      uint64_t far_min = kInfDist;
      while (!done && thr > F) {
        uint64_t F_new = F + S;
        if (far_min != kInfDist) {
          const uint64_t jump = far_min + S < thr ? far_min + S : static_cast<uint64_t>(thr);
          if (jump > F_new) F_new = jump;
        }
        const uint32_t Fo = F >= kInfDist ? kInfDist : static_cast<uint32_t>(F);
        const uint32_t Fn = F_new >= kInfDist ? kInfDist : static_cast<uint32_t>(F_new);
        TeamRed& R = cur();
        uint32_t lkey = kInfDist, lfar = kInfDist;
        c_far += (rank == 0) ? far_len : 0;
        c_refill += (rank == 0) ? 1 : 0;
        const uint32_t* src = fc ? fq1 : fq0;
        uint32_t* dst = fc ? fq0 : fq1;
        uint32_t* const nqc = nc ? nq1 : nq0;
        constexpr int kRefillU = T <= 32 ? 8 : WBC_TEAM_REFILL_U;  // far entries per lane per step
        for (uint32_t c = gtid; c < far_len; c += TT * kRefillU) {
          uint32_t u[kRefillU], du[kRefillU];
#pragma unroll
          for (int k = 0; k < kRefillU; ++k) {
            const uint32_t i = c + k * TT;
            u[k] = i < far_len ? __ldcg(src + i) : 0u;
          }
#pragma unroll
          for (int k = 0; k < kRefillU; ++k) du[k] = c + k * TT < far_len ? dist.template get<C>(u[k]) : 0u;
#pragma unroll
          for (int k = 0; k < kRefillU; ++k) {
            if (c + k * TT < far_len && du[k] >= Fo) {  // du < Fo: already near or settled
              if (du[k] < Fn) {
                nqc[near_len + team_append(&R.near_app)] = u[k];
                lkey = min(lkey, du[k] + __ldg(g.minw + u[k]));
              } else {
                dst[team_append(&R.far_app)] = u[k];
                lfar = min(lfar, du[k]);
              }
            }
          }
        }
        team_min(lkey, &R.min1);
        team_min(lfar, &R.min2);
        tsync();
        {
          TeamRed& Q = prev();
          near_len += Q.near_app;
          far_len = Q.far_app;
          fc ^= 1;
          thr = min(thr, Q.min1);
          far_min = Q.min2;
        }
        F = F_new;
        done = (near_len == 0 && far_len == 0);
      }
      tick(2);
      if (done) break;

      // ---------------- settle: d < Delta joins level nlev, with its row data
      {
        TeamRed& R = cur();
        uint32_t lkept = kInfDist;
        c_near += (rank == 0) ? near_len : 0;
        const uint32_t* src = nc ? nq1 : nq0;
        uint32_t* dst = nc ? nq0 : nq1;
        const uint32_t sb = static_cast<uint32_t>((static_cast<uint64_t>(near_len) * rank) / C);
        const uint32_t se = static_cast<uint32_t>((static_cast<uint64_t>(near_len) * (rank + 1)) / C);
        // warp-level, kSettleU entries per lane per step: the near-queue
        // loads, distance and row-offset gathers of the step are in flight
        // together; a warp scan plus one packed atomic hands out (order
        // position, edge offset) for the settled lanes; no CTA barrier.
        constexpr int kSettleU = T <= 32 ? 8 : WBC_TEAM_SETTLE_U;  // R-MAT-20 (C = 2): 2: 45.1, 4: 44.8, 8: 43.5 GTEPS
        const uint32_t lane = tid & 31;
        const uint32_t lt = (1u << lane) - 1u;
        for (uint32_t c = sb + (tid & ~31u) * kSettleU; c < se; c += T * kSettleU) {
          uint32_t u[kSettleU], du[kSettleU], row[kSettleU], deg[kSettleU];
          bool have[kSettleU], st[kSettleU];
#pragma unroll
          for (int k = 0; k < kSettleU; ++k) {
            const uint32_t i = c + 32 * k + lane;
            have[k] = i < se;
            u[k] = have[k] ? __ldcg(src + i) : 0u;
          }
#pragma unroll
          for (int k = 0; k < kSettleU; ++k) du[k] = have[k] ? dist.template get<C>(u[k]) : kInfDist;
#pragma unroll
          for (int k = 0; k < kSettleU; ++k) {
            st[k] = have[k] && du[k] < thr;
            row[k] = st[k] ? __ldg(g.offsets + u[k]) : 0u;
            deg[k] = st[k] ? __ldg(g.offsets + u[k] + 1) : 0u;
          }
          uint32_t bs[kSettleU], pe[kSettleU], nset = 0, eset = 0;
#pragma unroll
          for (int k = 0; k < kSettleU; ++k) {
            deg[k] -= row[k];
            bs[k] = __ballot_sync(0xffffffffu, st[k]);
            pe[k] = deg[k];  // inclusive warp scan of degrees
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, pe[k], o);
              if (lane >= static_cast<uint32_t>(o)) pe[k] += y;
            }
            // exclusive prefix of this lane within the whole step
            pe[k] = pe[k] - deg[k] + eset;
            eset += __shfl_sync(0xffffffffu, pe[k] + deg[k], 31) - eset;
            nset += __popc(bs[k]);
          }
          if (nset) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&R.ord, (static_cast<unsigned long long>(nset) << 32) | eset);
            base = __shfl_sync(0xffffffffu, base, 0);
            uint32_t pos = ord_len + static_cast<uint32_t>(base >> 32);
            const uint32_t ebase = ord_edges + static_cast<uint32_t>(base);
#pragma unroll
            for (int k = 0; k < kSettleU; ++k) {
              if (st[k]) {
                const uint32_t q = pos + __popc(bs[k] & lt);
                order[q] = u[k];
                ord_d[q] = du[k];
                ord_row[q] = row[k];
                epref[q] = ebase + pe[k];
                sigma[u[k]] = 0.0;
                delta[u[k]] = 0.0;
              }
              pos += __popc(bs[k]);
            }
          }
          uint32_t bk[kSettleU], nkeep = 0;
#pragma unroll
          for (int k = 0; k < kSettleU; ++k) {
            bk[k] = __ballot_sync(0xffffffffu, have[k] && !st[k]);
            nkeep += __popc(bk[k]);
          }
          if (nkeep) {
            uint32_t kb = 0;
            if (lane == 0) kb = atomicAdd(&R.keep_app, nkeep);
            kb = __shfl_sync(0xffffffffu, kb, 0);
            uint32_t mw[kSettleU];
#pragma unroll
            for (int k = 0; k < kSettleU; ++k) mw[k] = (bk[k] >> lane & 1u) ? __ldg(g.minw + u[k]) : 0u;
#pragma unroll
            for (int k = 0; k < kSettleU; ++k) {
              if (bk[k] >> lane & 1u) {
                dst[kb + __popc(bk[k] & lt)] = u[k];
                lkept = min(lkept, du[k] + mw[k]);
              }
              kb += __popc(bk[k]);
            }
          }
        }
        team_min(lkept, &R.min1);
      }
      tsync();
      {
        TeamRed& Q = prev();
        fb = ord_len;
        ord_len += static_cast<uint32_t>(Q.ord >> 32);
        fe = ord_len;
        Eb = ord_edges;
        ord_edges += static_cast<uint32_t>(Q.ord);
        Ee = ord_edges;
        near_len = Q.keep_app;
        nc ^= 1;
        kept_min = Q.min1;
        ++nlev;
      }
      if (leader) lev[nlev] = ord_len;
      tick(3);
    }

    // ---------------- dependency accumulation, deepest level first
    if (p.strict_lanes) {
      // The reference's own loop (engine.cpp:183-212), bit for bit: every
      // vertex w of level L sums c = sw / sigma[v] * (1 + delta[v]) over its
      // row in the caller's slot order, as `lanes` interleaved partial sums
      // (slot j of the row feeds part[j % lanes]) combined in lane order.  A
      // group of G threads takes one row, G consecutive slots per step; the
      // hits of a step are folded into their lane's partial in slot order by
      // a warp-uniform walk over the ballot mask.  Edge terms go to the
      // source's stage row (one writer per edge and source).
      GraphView gr = g;
      gr.slots32 = p.ref_slots32;
      gr.slots64 = p.ref_slots64;
      const uint32_t LW = p.strict_lanes, G = p.strict_group;
      const uint32_t lane = tid & 31, gl = lane & (G - 1), gb = lane & ~(G - 1);
      constexpr uint32_t kWarps = TT / 32;
      const uint32_t wid = gtid >> 5, per_warp = 32 / G;
      const unsigned long long si = sh.src_idx;
      double* const eacc = p.stage_edge ? p.stage_edge + si * static_cast<uint64_t>(g.m) : nullptr;
      double* const sdelta = p.stage_node + si * p.ws.n_stride;  // this source's delta row
      for (int L = static_cast<int>(nlev) - 1; L >= 0; --L) {
        const uint32_t vb = __ldcg(lev + L), ve = static_cast<uint32_t>(L) + 1 == nlev ? ord_len : __ldcg(lev + L + 1);
        for (uint32_t q0 = vb + wid * per_warp; q0 < ve; q0 += kWarps * per_warp) {
          const uint32_t q = q0 + lane / G;
          const bool has = q < ve;
          const uint32_t w = has ? __ldcg(order + q) : 0u;
          const uint32_t dw = has ? __ldcg(ord_d + q) : 0u;
          const uint32_t rb = has ? __ldg(g.offsets + w) : 0u, re = has ? __ldg(g.offsets + w + 1) : 0u;
          const double sw = has ? ld_team<C, 1>(sigma + w) : 0.0;
          double part = 0.0;
          for (uint32_t st = 0; __any_sync(0xffffffffu, rb + st < re); st += G) {
            const uint32_t e = rb + st + gl;
            double c = 0.0;
            bool hit = false;
            if (e < re) {
              uint32_t x, wt;
              load_slot<PACKED>(gr, e, x, wt);
              const uint32_t dx = dist.template get<C>(x);
              if (dx != kInfDist && dx == dw + wt) {
                hit = true;
                const double sx = ld_team<C, 1>(sigma + x);
                note_sigma(p.overflow, sx);
                c = __dmul_rn(__ddiv_rn(sw, sx), __dadd_rn(1.0, ld_team<C, 1>(sdelta + x)));
                if (eacc) eacc[__ldg(p.ref_edge_id + e)] = c;
              }
            }
            uint32_t mask = __ballot_sync(0xffffffffu, hit);
            while (mask) {
              const uint32_t t = __ffs(mask) - 1;
              mask &= mask - 1;
              const double ct = __shfl_sync(0xffffffffu, c, t);
              if (lane == (t & ~(G - 1)) + (t & (G - 1)) % LW) part = __dadd_rn(part, ct);
            }
          }
          double dsw = 0.0;
          for (uint32_t j = 0; j < LW; ++j) dsw = __dadd_rn(dsw, __shfl_sync(0xffffffffu, part, gb + j));
          if (has && gl == 0) sdelta[w] = dsw;
        }
        tsync();
      }
    } else if (!dag_over) {
      for (uint32_t L = nlev - 1; L >= 1; --L) {
        // dag_ends[nlev] is written by the leader in this very phase: use the register
        const uint32_t b = __ldcg(dag_ends + L), e = L + 1 == nlev ? dag_len : __ldcg(dag_ends + L + 1);
        constexpr int kBackU = WBC_TEAM_BACK_U;  // DAG edges per thread per step, loads in flight together
        for (uint32_t c = b + gtid; c < e; c += TT * kBackU) {
          uint2 d[kBackU];
          uint32_t u[kBackU];
#pragma unroll
          for (int k = 0; k < kBackU; ++k) d[k] = c + k * TT < e ? __ldcg(dag + c + k * TT) : make_uint2(0, 0);
#pragma unroll
          for (int k = 0; k < kBackU; ++k) {
            uint32_t w;
            u[k] = d[k].x;  // the predecessor itself unless edge BC stored the slot
            if (p.edge_bc && c + k * TT < e) load_slot<PACKED>(g, d[k].x, u[k], w);
          }
#pragma unroll
          for (int k = 0; k < kBackU; ++k) {
            if (c + k * TT >= e) continue;
            const uint32_t v = d[k].y;
            // reference term: sw / sigma[v] * (1.0 + delta[v])  (engine.cpp:201)
            const double sv = ld_team<C, 1>(sigma + v);
            note_sigma(p.overflow, sv);
            const double cc = ld_team<C, 1>(sigma + u[k]) / sv * (1.0 + ld_team<C, 1>(delta + v));
            atomicAdd(delta + u[k], cc);
            if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + d[k].x), cc);
          }
        }
        // level L's delta is final (levels > L were done in earlier phases)
        const uint32_t vb = __ldcg(lev + L), ve = L + 1 == nlev ? ord_len : __ldcg(lev + L + 1);
        for (uint32_t q = vb + gtid; q < ve; q += TT) {
          const uint32_t w = __ldcg(order + q);
          atomicAdd(p.node_bc + w, __ldcg(delta + w));
        }
        tsync();
      }
    } else {
      // Row-scan pull fallback (the reference's loop shape) when the DAG
      // buffer overflowed: phase L computes delta of level L from its rows
      // and adds the (final) delta of level L+1 to node BC.
      if (leader) atomicAdd(p.overflow, 1u);
      // per-chunk delta sums live in the (now idle) relax queues: keeping
      // them out of TeamShared keeps the CTA's shared memory within the
      // 100 KB carveout, which leaves L1 156 KB instead of 124 KB
      static_assert(team_q_bytes(T) >= CH * sizeof(double), "acc fits the queue region");
      double* const acc = reinterpret_cast<double*>(team_q);
      for (int t = tid; t < CH; t += T) acc[t] = 0.0;
      __syncthreads();
      for (int L = static_cast<int>(nlev) - 1; L >= 0; --L) {
        const uint32_t pb = __ldcg(lev + L), pe = static_cast<uint32_t>(L) + 1 == nlev ? ord_len : __ldcg(lev + L + 1);
        const uint32_t lEb = __ldcg(epref + pb);
        const uint32_t lEe = pe < ord_len ? __ldcg(epref + pe) : ord_edges;
        const uint32_t E = lEe - lEb;
        const uint32_t my_b = lEb + static_cast<uint32_t>((static_cast<uint64_t>(E) * rank) / C);
        const uint32_t my_e = lEb + static_cast<uint32_t>((static_cast<uint64_t>(E) * (rank + 1)) / C);
        if (my_b < my_e) {
          uint32_t j = C == 1 ? pb : block_find<T>(epref, pb, pe, my_b);
          uint32_t cb = my_b;
          while (cb < my_e) {
            uint32_t ce;
            const int cnt = stage(j, pe, cb, my_e, lEe, ce);
            expand_edges<T>(sh.pref, cnt, ce - cb, [&](uint32_t e, int jl) {
              const uint32_t slot = sh.rowadj[jl] + e;
              uint32_t x, w;
              load_slot<PACKED>(g, slot, x, w);
              const uint32_t dx = dist.template get<C>(x);
              if (dx != kInfDist && dx == sh.dv[jl] + w) {
                const uint32_t wv = sh.v[jl];
                const double sx = ld_team<C, 1>(sigma + x);
                note_sigma(p.overflow, sx);
                const double c2 = ld_team<C, 1>(sigma + wv) / sx * (1.0 + ld_team<C, 1>(delta + x));
                atomicAdd(&acc[jl], c2);
                if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + slot), c2);
              }
            });
            __syncthreads();
            for (int t = tid; t < cnt; t += T)
              if (acc[t] != 0.0) {
                atomicAdd(delta + sh.v[t], acc[t]);
                acc[t] = 0.0;
              }
            __syncthreads();
            j += cnt;
            cb = ce;
          }
        }
        if (static_cast<uint32_t>(L) + 1 < nlev) {
          const uint32_t vb = __ldcg(lev + L + 1), ve = static_cast<uint32_t>(L) + 2 == nlev ? ord_len : __ldcg(lev + L + 2);
          for (uint32_t q = vb + gtid; q < ve; q += TT) {
            const uint32_t w = __ldcg(order + q);
            atomicAdd(p.node_bc + w, __ldcg(delta + w));
          }
        }
        tsync();
      }
    }
    tick(4);
    if (leader) {
      if (p.depth) p.depth[s_orig] = nlev;
      cur().src = atomicAdd(p.counter, 1ULL);
    }
    if (PROF && leader) {
      atomicAdd(p.prof + kProfRounds, nlev);
      atomicAdd(p.prof + kProfDagEdges, dag_len);
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
  }
  // no CTA may leave while others can still touch its shared memory
  if constexpr (C > 1) cg::this_cluster().sync();
}

}  // namespace wbc_dev
