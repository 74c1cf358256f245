// bc_flat.cuh -- per-source pipeline for flat, large-diameter graphs (grid /
// road-like: small degrees, ~10^5 Eq. 4 rounds per source).
//
// The Eq. 4 round process (engine.cpp:144-222) is inherently sequential: one
// round settles ~45 vertices of a 2048^2 grid, and the team kernel spends
// ~50K cycles of dependent memory round trips on each (profiles/
// r01_ncu_team_grid2048.md).  This kernel takes the rounds off the critical
// path.  Everything the result needs is a function of the final distances
// (tests/test_depth_theory.py):
//   * sigma / delta need only the shortest-path DAG, in any topological order;
//   * the Eq. 4 levels are S_{r+1} = {v : d(v) < D_r} with
//     D_r = min over slots u->v, d(u) < D_{r-1} <= d(v), of d(u) + w + minw(v),
//     so depth_per_source is one monotone sweep over the distance-sorted
//     vertices.
// One CTA per source runs:
//   A. near-far SSSP (Bellman-Ford inside a window of width `delta`, a far
//      pile beyond it), distances only;
//   B. DAG in-/out-degrees, reached count, max distance;
//   C. sigma by a dependency-counted dataflow (a vertex is queued when its
//      last predecessor is done: integer-valued fp64 sums, exact in any order;
//      the hand-off is a CTA-scope acq_rel decrement, release store, acquire
//      load);
//   D. delta the same way in reverse, with the reference's term
//      sigma[u] / sigma[v] * (1 + delta[v]) (engine.cpp:201) and node / edge BC;
//   E. a counting sort of the distances, then one warp sweeps the thresholds
//      with a shared-memory bucket array (key -> largest successor distance),
//      concurrently with C and D on the other warps.
// Sources whose distances exceed the counting-sort range are handed to the
// team kernel (abort list), before anything is accumulated.
#pragma once

#include "bc_kernels.cuh"

namespace wbc_dev {

constexpr uint32_t kFlatEmpty = 0xFFFFFFFFu;
constexpr int kFlatMaxDeg = 8;        // interval slots per vertex in the sweep input
constexpr int kFlatBuckets = 16384;   // shared-memory keys: maxw + max minw + 2 must fit

struct FlatWs {
  uint64_t n_stride;
  uint32_t* dist;
  double* sigma;
  double* delta;
  uint32_t* npred;
  uint32_t* nsucc;
  uint32_t* flag;
  uint32_t* q0;
  uint32_t* q1;
  uint32_t* q2;
  uint32_t* q3;
  uint32_t* hist;      // n_stride entries: the counting-sort range of distances
  uint32_t* sorted_d;  // their distances
  uint2* ivl;          // per sorted position, ivl_stride (key, successor distance + 1) pairs
  uint32_t ivl_stride; // the graph's max degree (<= kFlatMaxDeg)
  uint32_t delta_w;    // near-far window width
  uint32_t buckets;    // power of two >= maxw + max minw + 2
  uint32_t* abort_list;
  unsigned long long* abort_count;
};

__device__ __forceinline__ uint32_t ld_vol(const uint32_t* a) { return *reinterpret_cast<const volatile uint32_t*>(a); }
__device__ __forceinline__ void st_vol(uint32_t* a, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(a) = v; }
// CTA-scope acquire load / release store / acq_rel decrement (the dataflow
// hand-off: a vertex's sums are visible to whoever dequeues it)
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.cta.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint32_t* a, uint32_t v) {
  asm volatile("st.release.cta.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t dec_acq_rel(uint32_t* a) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(0xFFFFFFFFu) : "memory");
  return old;
}

template <int T, bool PACKED>
__global__ void __launch_bounds__(T, 1024 / T) bc_flat_kernel(const RunParams p, const FlatWs w) {
  // p.prof: per-phase SM cycles of thread 0, reusing the team kernel's counter
  // slots: init -> kProfCyclesInit, A -> kProfCyclesRelax, B ->
  // kProfCyclesThreshold, E1 histogram -> kProfFarScanned, scan ->
  // kProfImprovements, scatter + sweep input -> kProfNearScanned, E2 || C/D ->
  // kProfRefills; A's phases -> kProfRounds
  unsigned long long t_last = 0;
  auto tick = [&](int slot) {
    if (p.prof && threadIdx.x == 0) {
      const unsigned long long t = clock64();
      if (slot >= 0) atomicAdd(p.prof + slot, t - t_last);
      t_last = t;
    }
  };
  __shared__ unsigned long long s_src;
  __shared__ uint32_t s_ring[3][4];  // per-phase counters: [append a, append b, min, spare]
  __shared__ uint32_t s_reached, s_maxd, s_head, s_tail, s_carry;
  __shared__ uint32_t s_warp[T / 32];
  extern __shared__ uint32_t bucket[];  // w.buckets entries (dynamic)
  const GraphView& g = p.g;
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31, wid = tid >> 5;
  const uint64_t off = static_cast<uint64_t>(blockIdx.x) * w.n_stride;
  uint32_t* const dist = w.dist + off;
  double* const sigma = w.sigma + off;
  double* const delta = w.delta + off;
  uint32_t* const npred = w.npred + off;
  uint32_t* const nsucc = w.nsucc + off;
  uint32_t* const flag = w.flag + off;
  uint32_t* const hist = w.hist + off;
  uint32_t* const sorted_d = w.sorted_d + off;
  const uint32_t kE = w.ivl_stride;
  uint2* const ivl = w.ivl + off * kE;
  const uint32_t n = g.n;
  const unsigned long long k_total = p.k_dev ? __ldcg(p.k_dev) : p.k;
  auto row_of = [&](uint32_t v, uint32_t& b, uint32_t& e) {
    b = __ldg(g.offsets + v);
    e = __ldg(g.offsets + v + 1);
  };

  for (;;) {
    if (tid == 0) s_src = atomicAdd(p.counter, 1ULL);
    __syncthreads();
    const unsigned long long idx = s_src;
    if (idx >= k_total) break;
    const uint32_t s_orig = p.sources ? __ldg(p.sources + idx) : static_cast<uint32_t>(p.src_base + idx);
    const uint32_t s = __ldg(p.inv + s_orig);
    tick(-1);

    // ---- init
    for (uint32_t i = tid; i < n; i += T) {
      dist[i] = i == s ? 0u : kInfDist;
      sigma[i] = 0.0;
      delta[i] = 0.0;
      npred[i] = 0;
      flag[i] = 0;
    }
    if (tid < 12) (&s_ring[0][0])[tid] = tid % 4 == 2 ? kInfDist : 0u;
    if (tid == 0) w.q0[off] = s;
    __syncthreads();
    tick(kProfCyclesInit);

    // ---- A. near-far SSSP
    uint32_t* nq = w.q0 + off;
    uint32_t* nn = w.q1 + off;
    uint32_t* fq = w.q2 + off;
    uint32_t* fq2 = w.q3 + off;
    uint32_t near_len = 1, far_len = 0, iter = 1, ph = 0;
    uint64_t thr = w.delta_w;
    for (;;) {
      uint32_t* R = s_ring[ph % 3];
      if (tid == 0) {
        uint32_t* Z = s_ring[(ph + 1) % 3];
        Z[0] = 0;
        Z[1] = 0;
        Z[2] = kInfDist;
      }
      const uint32_t thr32 = thr >= kInfDist ? kInfDist : static_cast<uint32_t>(thr);
      if (near_len) {
        // relax every near vertex (thread per vertex: flat rows are short)
        // (the row's slot words, then its distance gathers, then its atomics:
        // each stage's loads are in flight together)
        for (uint32_t i = tid; i < near_len; i += T) {
          const uint32_t v = nq[i];
          const uint32_t dv = __ldcg(dist + v);
          uint32_t b, e;
          row_of(v, b, e);
          uint32_t us[kFlatMaxDeg], nd[kFlatMaxDeg], old[kFlatMaxDeg];
#pragma unroll
          for (int x = 0; x < kFlatMaxDeg; ++x) {
            us[x] = kFlatEmpty;
            nd[x] = kInfDist;
            if (b + x < e) {
              uint32_t wt;
              load_slot<PACKED>(g, b + x, us[x], wt);
              nd[x] = dv + wt;
            }
          }
#pragma unroll
          for (int x = 0; x < kFlatMaxDeg; ++x)
            if (us[x] != kFlatEmpty && nd[x] >= __ldcg(dist + us[x])) us[x] = kFlatEmpty;
#pragma unroll
          for (int x = 0; x < kFlatMaxDeg; ++x) old[x] = us[x] != kFlatEmpty ? atomicMin(dist + us[x], nd[x]) : 0u;
#pragma unroll
          for (int x = 0; x < kFlatMaxDeg; ++x) {
            if (us[x] == kFlatEmpty || nd[x] >= old[x]) continue;
            const uint32_t u = us[x];
            if (nd[x] < thr32) {
              if (atomicExch(flag + u, iter + 1) != iter + 1) nn[atomicAdd(&R[0], 1u)] = u;
            } else if (old[x] == kInfDist) {
              fq[far_len + atomicAdd(&R[1], 1u)] = u;
            }
          }
        }
        __syncthreads();
        near_len = R[0];
        far_len += R[1];
        uint32_t* t = nq;
        nq = nn;
        nn = t;
        ++iter;
        ++ph;
        continue;
      }
      if (far_len == 0) break;
      // refill: far entries inside the next window become near; the rest are
      // compacted into the other far buffer
      const uint64_t thr_new = thr + w.delta_w;
      const uint32_t tn32 = thr_new >= kInfDist ? kInfDist : static_cast<uint32_t>(thr_new);
      for (uint32_t i = tid; i < far_len; i += T) {
        const uint32_t u = fq[i];
        const uint32_t du = __ldcg(dist + u);
        if (du < thr32) continue;  // reached the near window earlier: relaxed already
        if (du < tn32) {
          if (atomicExch(flag + u, iter + 1) != iter + 1) nq[atomicAdd(&R[0], 1u)] = u;
        } else {
          fq2[atomicAdd(&R[1], 1u)] = u;
          atomicMin(&R[2], du);
        }
      }
      __syncthreads();
      near_len = R[0];
      far_len = R[1];
      {
        uint32_t* t = fq;
        fq = fq2;
        fq2 = t;
      }
      thr = thr_new;
      if (near_len == 0 && far_len) thr = static_cast<uint64_t>(R[2]);  // jump: next refill opens [min, min + delta)
      ++iter;
      ++ph;
    }

    tick(kProfCyclesRelax);
    if (p.prof && tid == 0) atomicAdd(p.prof + kProfRounds, static_cast<unsigned long long>(iter));
    // ---- B. the DAG: per vertex a successor mask (slots u->v with
    // d(v) = d(u) + w) and a predecessor mask (d(u) = d(v) + w) in `flag`
    // (free after A), successor counts, predecessor counts, reached count,
    // max distance
    if (tid == 0) {
      s_reached = 0;
      s_maxd = 0;
    }
    __syncthreads();
    {
      uint32_t reached = 0, maxd = 0;
      for (uint32_t u = tid; u < n; u += T) {
        const uint32_t du = __ldcg(dist + u);
        if (du == kInfDist) continue;
        ++reached;
        maxd = max(maxd, du);
        uint32_t b, e, sm = 0, pm = 0;
        row_of(u, b, e);
        for (uint32_t x = b; x < e; ++x) {
          uint32_t v, wt;
          load_slot<PACKED>(g, x, v, wt);
          const uint32_t dv = __ldcg(dist + v);
          if (dv == du + wt) {
            sm |= 1u << (x - b);
            atomicAdd(npred + v, 1u);
          } else if (dv != kInfDist && dv + wt == du) {
            pm |= 1u << (x - b);
          }
        }
        nsucc[u] = __popc(sm);
        flag[u] = sm | pm << 16;
      }
      reached = __reduce_add_sync(0xffffffffu, reached);
      maxd = __reduce_max_sync(0xffffffffu, maxd);
      if (lane == 0) {
        atomicAdd(&s_reached, reached);
        atomicMax(&s_maxd, maxd);
      }
    }
    __syncthreads();
    const uint32_t reached = s_reached, maxd = s_maxd;
    tick(kProfCyclesThreshold);
    if (static_cast<uint64_t>(maxd) >= w.n_stride) {
      // distances beyond the counting-sort range: the team kernel runs this
      // source instead (nothing has been accumulated yet)
      if (tid == 0) w.abort_list[atomicAdd(w.abort_count, 1ULL)] = s_orig;
      continue;
    }

    // ---- E1. counting sort of the distances and the sweep input
    for (uint32_t i = tid; i <= maxd; i += T) hist[i] = 0;
    __syncthreads();
    constexpr int kH = 8;  // vertices per thread and step: their loads in flight together
    for (uint32_t u0 = tid; u0 < n; u0 += T * kH) {
      uint32_t du[kH];
#pragma unroll
      for (int j = 0; j < kH; ++j) du[j] = u0 + j * T < n ? __ldcg(dist + u0 + j * T) : kInfDist;
#pragma unroll
      for (int j = 0; j < kH; ++j)
        if (du[j] != kInfDist) atomicAdd(hist + du[j], 1u);
    }
    if (tid == 0) s_carry = 0;
    __syncthreads();
    tick(kProfFarScanned);  // --prof: histogram
    for (uint32_t base = 0; base <= maxd; base += T) {  // exclusive scan, T entries per step
      const uint32_t i = base + tid;
      const uint32_t x = i <= maxd ? hist[i] : 0u;
      uint32_t incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
      }
      if (lane == 31) s_warp[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        uint32_t ws = lane < T / 32 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
          if (lane >= static_cast<uint32_t>(o)) ws += y;
        }
        if (lane < T / 32) s_warp[lane] = ws;
      }
      __syncthreads();
      const uint32_t before = s_carry + (wid ? s_warp[wid - 1] : 0u);
      if (i <= maxd) hist[i] = before + incl - x;
      __syncthreads();
      if (tid == T - 1) s_carry = before + incl;
      __syncthreads();
    }
    tick(kProfImprovements);  // --prof: scan
    // scatter into distance order, writing each vertex's sweep input at its
    // position: its slots u->v with d(v) > d(u) as (key d(u) + w + minw(v),
    // d(v) + 1), zero pairs pad.  One vertex per thread and step, every
    // load of a step in flight together (host: max degree <= kFlatMaxDeg).
    uint32_t* const pos_of = w.q2 + off;  // sorted position per vertex (q2 is free after A)
    for (uint32_t u0 = tid; u0 < n; u0 += T * kH) {
      uint32_t du[kH], ps[kH];
#pragma unroll
      for (int j = 0; j < kH; ++j) du[j] = u0 + j * T < n ? __ldcg(dist + u0 + j * T) : kInfDist;
#pragma unroll
      for (int j = 0; j < kH; ++j) ps[j] = du[j] != kInfDist ? atomicAdd(hist + du[j], 1u) : 0u;
#pragma unroll
      for (int j = 0; j < kH; ++j)
        if (du[j] != kInfDist) {
          pos_of[u0 + j * T] = ps[j];
          sorted_d[ps[j]] = du[j];
        }
    }
    constexpr int kU = 1;
    for (uint32_t u0 = tid; u0 < n; u0 += T * kU) {
      uint32_t du[kU], pos[kU], rb[kU], re[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t u = u0 + j * T;
        du[j] = u < n ? __ldcg(dist + u) : kInfDist;
        rb[j] = re[j] = 0;
        pos[j] = 0;
        if (du[j] != kInfDist) {
          row_of(u, rb[j], re[j]);
          pos[j] = pos_of[u];
        }
      }
      uint32_t v[kU][kFlatMaxDeg], wt[kU][kFlatMaxDeg], dv[kU][kFlatMaxDeg], mw[kU][kFlatMaxDeg];
#pragma unroll
      for (int j = 0; j < kU; ++j)
#pragma unroll
        for (int x = 0; x < kFlatMaxDeg; ++x) {
          v[j][x] = 0;
          wt[j][x] = 0;
          if (rb[j] + x < re[j]) load_slot<PACKED>(g, rb[j] + x, v[j][x], wt[j][x]);
        }
#pragma unroll
      for (int j = 0; j < kU; ++j)
#pragma unroll
        for (int x = 0; x < kFlatMaxDeg; ++x) {
          const bool ok = rb[j] + x < re[j];
          dv[j][x] = ok ? __ldcg(dist + v[j][x]) : kInfDist;
          mw[j][x] = ok ? __ldg(g.minw + v[j][x]) : 0u;
        }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        if (du[j] == kInfDist) continue;
        uint2* const out = ivl + static_cast<uint64_t>(pos[j]) * kE;
        int t = 0;
#pragma unroll
        for (int x = 0; x < kFlatMaxDeg; ++x)
          if (dv[j][x] != kInfDist && dv[j][x] > du[j]) out[t++] = make_uint2(du[j] + wt[j][x] + mw[j][x], dv[j][x] + 1);
        for (; t < static_cast<int>(kE); ++t) out[t] = make_uint2(0, 0);
      }
    }
    __syncthreads();
    for (uint32_t i = tid; i < w.buckets; i += T) bucket[i] = 0;
    __syncthreads();
    tick(kProfNearScanned);
    // Warp 0 sweeps the Eq. 4 thresholds (E2) while the other warps run the
    // sigma (C) and delta (D) dataflows; they synchronise on named barrier 1.
    if (wid == 0) {
      // ---- E2. threshold sweep
      const uint32_t B = w.buckets, M = B - 1;
      // bucket[k & M] = 1 + largest d(v) over inserted slots with key k; the
      // key is live at threshold tau iff that d(v) >= tau
      auto insert_slow = [&](uint32_t eb, uint32_t ee) {  // entries [eb, ee), 8 loads per lane in flight
        for (uint32_t c0 = eb; c0 < ee; c0 += 256) {
          uint2 kv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t c = c0 + lane + 32 * j;
            kv[j] = c < ee ? __ldcg(ivl + c) : make_uint2(0, 0);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (kv[j].y) atomicMax(&bucket[kv[j].x & M], kv[j].y);
        }
      };
      // Lookahead registers, refilled at the end of each round for the next
      // one: distances of sorted positions [sd_base, sd_base + 128) and sweep
      // entries [iv_base, iv_base + 256) (positions iv_base / 8 ..).
      uint32_t sd[4];
      uint2 iv[8];
      uint32_t sd_base = 0, iv_base = 0;
      auto prefetch = [&](uint32_t q0) {
        sd_base = q0;
        iv_base = q0 * kE;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t q = q0 + lane + 32 * j;
          sd[j] = q < reached ? __ldcg(sorted_d + q) : kInfDist;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t c = iv_base + lane + 32 * j;
          iv[j] = c < reached * kE ? __ldcg(ivl + c) : make_uint2(0, 0);
        }
      };
      uint32_t tau = 1, pos = 1, levels = 1;
      insert_slow(0, kE);
      __syncwarp();
      prefetch(1);
      for (;;) {
        uint32_t nxt = kInfDist;
        for (uint32_t base = tau + 1; base < tau + B; base += 32) {
          const uint32_t k = base + lane;
          const bool live = k < tau + B && bucket[k & M] >= tau + 1;
          const uint32_t m = __ballot_sync(0xffffffffu, live);
          if (m) {
            nxt = base + __ffs(m) - 1;
            break;
          }
        }
        if (nxt == kInfDist) break;
        for (uint32_t k = tau + 1 + lane; k <= nxt; k += 32) bucket[k & M] = 0;
        __syncwarp();
        // the new level: sorted positions [pos, end) with d < nxt (pos == sd_base)
        uint32_t end = pos;
        bool open = true;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t m = __ballot_sync(0xffffffffu, sd[j] < nxt);
          if (open) end += __popc(m);
          open = open && m == 0xffffffffu;
        }
        while (open) {  // a level wider than the lookahead
          const uint32_t q = end + lane;
          const uint32_t m = __ballot_sync(0xffffffffu, q < reached && __ldcg(sorted_d + q) < nxt);
          end += __popc(m);
          open = m == 0xffffffffu;
        }
        // its sweep entries: from the lookahead, then the rest directly
        const uint32_t eb = pos * kE, ee = end * kE;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t c = iv_base + lane + 32 * j;
          if (c >= eb && c < ee && iv[j].y) atomicMax(&bucket[iv[j].x & M], iv[j].y);
        }
        if (ee > iv_base + 256) insert_slow(iv_base + 256, ee);
        __syncwarp();
        pos = end;
        tau = nxt;
        ++levels;
        prefetch(pos);
      }
      if (lane == 0 && p.depth) p.depth[s_orig] = levels;
    } else {
      constexpr uint32_t TG = T - 32;  // dataflow threads
      const uint32_t gt = tid - 32;
      auto gsync = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(TG) : "memory"); };
      // ---- C. sigma, forward dataflow over the DAG
      uint32_t* const qf = w.q0 + off;
      for (uint32_t i = gt; i < reached; i += TG) qf[i] = kFlatEmpty;
      gsync();
      if (gt == 0) {
        sigma[s] = 1.0;
        s_head = 0;
        s_tail = 1;
        st_vol(qf, s);
      }
      gsync();
      for (;;) {
        const uint32_t i = atomicAdd(&s_head, 1u);
        if (i >= reached) break;
        uint32_t u;
        while ((u = ld_acq(qf + i)) == kFlatEmpty) __nanosleep(32);
        const double su = __ldcg(sigma + u);
        const uint32_t b = __ldg(g.offsets + u);
        for (uint32_t sm = __ldcg(flag + u) & 0xFFFFu; sm; sm &= sm - 1) {
          uint32_t v, wt;
          load_slot<PACKED>(g, b + __ffs(sm) - 1, v, wt);
          atomicAdd(sigma + v, su);
          if (dec_acq_rel(npred + v) == 1u) st_rel(qf + atomicAdd(&s_tail, 1u), v);
        }
      }
      gsync();
      // ---- D. delta, reverse dataflow; node / edge BC
      uint32_t* const qb = w.q1 + off;
      for (uint32_t i = gt; i < reached; i += TG) qb[i] = kFlatEmpty;
      if (gt == 0) {
        s_head = 0;
        s_tail = 0;
      }
      gsync();
      for (uint32_t u = gt; u < n; u += TG)  // the DAG's sinks start the sweep
        if (__ldcg(dist + u) != kInfDist && nsucc[u] == 0) st_vol(qb + atomicAdd(&s_tail, 1u), u);
      gsync();
      for (;;) {
        const uint32_t i = atomicAdd(&s_head, 1u);
        if (i >= reached) break;
        uint32_t v;
        while ((v = ld_acq(qb + i)) == kFlatEmpty) __nanosleep(32);
        const double dvv = __ldcg(delta + v);
        const double sv = __ldcg(sigma + v);
        if (v != s) atomicAdd(p.node_bc + v, dvv);
        const uint32_t b = __ldg(g.offsets + v);
        for (uint32_t pm = __ldcg(flag + v) >> 16; pm; pm &= pm - 1) {
          const uint32_t x = b + __ffs(pm) - 1;
          uint32_t u, wt;
          load_slot<PACKED>(g, x, u, wt);
          // reference term: sw / sigma[v] * (1.0 + delta[v])  (engine.cpp:201)
          const double c = __ldcg(sigma + u) / sv * (1.0 + dvv);
          atomicAdd(delta + u, c);
          if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + x), c);
          if (dec_acq_rel(nsucc + u) == 1u) st_rel(qb + atomicAdd(&s_tail, 1u), u);
        }
      }
    }
    __syncthreads();
    tick(kProfRefills);
  }
}

}  // namespace wbc_dev
