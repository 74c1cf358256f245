// bc_flat.cuh -- per-source pipeline for flat, large-diameter graphs (grid /
// road-like: degree <= 8, ~10^5 Eq. 4 rounds per source).
//
// The Eq. 4 round process (engine.cpp:144-222) is inherently sequential: one
// round settles ~45 vertices of a 2048^2 grid, and a round-by-round kernel
// spends ~50K cycles of dependent memory round trips on each (profiles/
// r01_ncu_team_grid2048.md).  This kernel takes the rounds off the critical
// path.  Everything the result needs is a function of the final distances
// (tests/test_depth_theory.py):
//   * sigma / delta need only the shortest-path DAG, in any topological
//     order -- distance order is one;
//   * the Eq. 4 levels are S_{r+1} = {v : d(v) < D_r} with
//     D_r = min over slots u->v, d(u) < D_{r-1} <= d(v), of d(u) + w + minw(v),
//     so depth_per_source is one monotone sweep over the distance-sorted
//     vertices.
//
// One CTA per source.  The graph is read through an ELL copy of its rows:
// one record per vertex (KE packed slots and KE sweep keys, 32 B for KE = 4,
// so one sector), no offsets lookup.  The only vertex-indexed state is one
// 8-byte word per vertex, (distance, sorted position); everything else lives
// in distance order, where the pull passes below touch it coalesced or
// within a few thousand positions of the current one (L2-resident):
//   A. near-far SSSP, distances only: Bellman-Ford inside a window
//      [lo, lo + delta) of width `delta_w`, a far pile beyond it.  A vertex
//      joins the window's member list exactly once, when its distance first
//      drops below the window end (the atomicMin that sees the crossing, or
//      the far refill).  When a window closes its members are final; a
//      shared-memory counting sort on d - lo appends them to `order` /
//      `ord_d` and writes each one's position into its word, so the whole
//      source ends up sorted by distance with no pass over n.  The near
//      queues' first sq_cap entries live in shared memory.
//   B. sigma, pulled in distance order, a block of kBlk positions at a time
//      (kU per worker thread): predecessors (d(u) + w == d(v)) in earlier
//      blocks are final in `psig`; those inside the block resolve in barrier
//      rounds over the block's shared-memory copy (read, barrier, publish;
//      sigma >= 1, so 0 means not yet final).  Integer-valued fp64, exact in
//      any order below 2^53 (engine.cpp:73-77).  The same pass writes, per
//      position, the successor mask and positions and the threshold-sweep
//      entries of every slot to a farther neighbour (w + minw(v),
//      d(v) - d(u)), all coalesced.
//   C. delta, pulled in reverse distance order the same way:
//      c = sigma(u) * coef(v) over DAG successors v, where
//      coef(v) = (1 + delta(v)) / sigma(v) (positive: its own completion
//      flag); the reference's term is sigma[u] / sigma[v] * (1 + delta[v])
//      (engine.cpp:201), equal up to fp64 rounding.  Node BC += delta
//      (u != s), edge BC += c.
// A dedicated sweeper warp runs the Eq. 4 threshold sweep of the previous
// source while the workers run A/B/C of the next (its sorted distances and
// entries are double-buffered): a shared-memory bucket ring keyed by
// d(u) + w + minw(v) holds the largest successor distance + 1 (a key is live
// while that is above the threshold); positions stream through a cp.async
// ring, so a level costs shared-memory work only.
// Everything a CTA gathers in B and C (and its own distances in A) it wrote
// itself: those loads go through L1 (ld.ca, coherent within the CTA after a
// barrier), which on this kernel is worth more than any further shared memory.
// No source is ever handed back: the window sort's range is delta_w, not the
// distance range.
#pragma once

#include "bc_kernels.cuh"

namespace wbc_dev {

constexpr int kFlatMaxDeg = 8;        // ELL row width: 4 or 8 slots
constexpr int kFlatBuckets = 16384;   // shared-memory keys: maxw + max minw + 2 must fit
constexpr int kFlatChunk = 256;       // sweep ring: positions per chunk
constexpr int kFlatRing = 4;          // sweep ring: chunks (kFlatRing - 1 in flight)
#ifndef WBC_FLAT_RELAX_U
#define WBC_FLAT_RELAX_U 1
#endif
#ifndef WBC_FLAT_PRECHECK
#define WBC_FLAT_PRECHECK 0
#endif
#ifndef WBC_FLAT_PREFETCH
#define WBC_FLAT_PREFETCH 0
#endif
#ifndef WBC_FLAT_SORT_U
#define WBC_FLAT_SORT_U 4  // window-sort members / far entries per thread and step
#endif
#ifndef WBC_FLAT_KU
#define WBC_FLAT_KU 2
#endif
#ifndef WBC_FLAT_SQ
#define WBC_FLAT_SQ 4096
#endif
constexpr size_t kFlatSQ = WBC_FLAT_SQ;             // cap of the shared-memory near-queue entries per buffer
constexpr size_t kFlatSmemStep = 64 * 1024;         // the carveout step the kernel's other shared memory fits in
#ifndef WBC_FLAT_MEMD
#define WBC_FLAT_MEMD 1
#endif
#ifndef WBC_FLAT_L1
#define WBC_FLAT_L1 15
#endif
// loads of data this CTA wrote (distances, positions, sigma, coef) through
// L1 (ld.ca) instead of L2 only: bit 0 pass A distances, bit 1 pass B
// neighbour words, bit 2 pass B predecessor sigma, bit 3 pass C coef
constexpr int kFlatL1 = WBC_FLAT_L1;
template <int BIT, class X>
__device__ __forceinline__ X ld_own(const X* p) {
  if constexpr (kFlatL1 >> BIT & 1)
    return __ldca(p);
  else
    return __ldcg(p);
}
constexpr bool kSortKeepD = WBC_FLAT_MEMD;  // the window sort's counting pass parks each member's distance (coalesced) for the scatter pass
constexpr bool kRelaxPrefetch = WBC_FLAT_PREFETCH;  // prefetch a pushed vertex's ELL row into L2
#ifndef WBC_FLAT_SWEEPERS
#define WBC_FLAT_SWEEPERS 1
#endif
constexpr int kSweepers = WBC_FLAT_SWEEPERS;  // sweeper warps per CTA (<= 3)
constexpr int kRelaxU = WBC_FLAT_RELAX_U;  // near vertices per thread and step in A (grid-2048: 1 beats 2 by 3.6% since the L1 read paths)
constexpr bool kRelaxPrecheck = WBC_FLAT_PRECHECK;   // gather before the atomicMin

struct FlatWs {
  uint64_t n_stride;        // multiple of kFlatChunk
  uint2* dp;                // by vertex: (distance, sorted position)
  uint32_t* order;          // by position: vertex in distance order
  uint32_t* ord_d;          // by position: its distance (two buffers: the sweeper reads the last source's)
  uint32_t* mem;            // the open window's members (unsorted)
  uint32_t* q0;             // near / next near / far / next far queues
  uint32_t* q1;
  uint32_t* q2;
  uint32_t* q3;
  double* psig;             // by position: sigma, 0 until final
  double* pcoef;            // by position: (1 + delta) / sigma, 0 until final
  uint32_t* pinfo;          // by position: successor mask | predecessor mask << 8
  uint32_t* psucc;          // by position: KE neighbour positions (successor slots only)
  uint32_t* ent;            // by position: KE sweep entries (w + minw(v)) | (d(v) - d(u)) << 16, 0 = none
                            // (two buffers, like ord_d)
  const uint32_t* ell;      // n x 2KE words: KE slots (neighbour << wbits | weight, weight 0 = empty),
                            // KE u16 keys weight + minw(neighbour), padding to a 32-byte multiple
  const uint32_t* ell_eid;  // n x KE canonical edge ids (edge BC)
  uint32_t delta_w;         // window width (<= kFlatBuckets)
  uint32_t buckets;         // power of two >= maxw + max minw + 2
  uint32_t delta_words;     // shared-memory words of the window-sort histogram (>= delta_w)
  uint32_t sq_cap;          // near-queue entries per buffer kept in shared memory (the rest spill to q0 / q1)
};

__device__ __forceinline__ double ld_relaxed_f64(const double* a) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* a, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
// spin until a completion-flag value (nonzero) appears
__device__ __forceinline__ double wait_nonzero(const double* a) {
  double v = ld_relaxed_f64(a);
  while (v == 0.0) {
    __nanosleep(64);
    v = ld_relaxed_f64(a);
  }
  return v;
}
// barrier `id` over `count` threads that also ORs a predicate across them
__device__ __forceinline__ int bar_or(uint32_t pred, int id, int count) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(pred), "r"(id), "r"(count)
      : "memory");
  return r;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Dynamic shared memory of bc_flat_kernel<T, KE>: the workers' window-sort
// histogram, then per sweeper its bucket ring and cp.async ring.
// static shared memory of bc_flat_kernel<T, *> (s_blk dominates), rounded up
inline size_t flat_static_smem(int threads) {
  return static_cast<size_t>(threads - 32 * kSweepers) * WBC_FLAT_KU * 8 + threads / 8 + 1024;
}
// without the near queues (the host adds 2 * sq_cap words)
inline size_t flat_dyn_smem(uint32_t delta_words, uint32_t buckets, int ke) {
  return (static_cast<size_t>(delta_words) +
          kSweepers * (buckets + static_cast<size_t>(kFlatRing) * kFlatChunk * (1 + ke))) * 4;
}

// ELL record of v: 2 KE words (slots, then keys two per word)
template <int KE>
__device__ __forceinline__ const uint4* ell_rec(const FlatWs& w, uint32_t v) {
  return reinterpret_cast<const uint4*>(w.ell + static_cast<uint64_t>(v) * (2 * KE));
}
template <int KE>
__device__ __forceinline__ void ell_row(const FlatWs& w, uint32_t v, uint32_t (&r)[KE]) {
  const uint4* p = ell_rec<KE>(w, v);
#pragma unroll
  for (int q = 0; q < KE / 4; ++q) {
    const uint4 x = __ldg(p + q);
    r[4 * q] = x.x;
    r[4 * q + 1] = x.y;
    r[4 * q + 2] = x.z;
    r[4 * q + 3] = x.w;
  }
}
template <int KE>
__device__ __forceinline__ void ell_keys(const FlatWs& w, uint32_t v, uint32_t (&k)[KE]) {
  const uint4* p = ell_rec<KE>(w, v) + KE / 4;
  if constexpr (KE == 4) {
    const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
    k[0] = x.x & 0xFFFFu;
    k[1] = x.x >> 16;
    k[2] = x.y & 0xFFFFu;
    k[3] = x.y >> 16;
  } else {
    const uint4 x = __ldg(p);
    const uint32_t a[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      k[2 * i] = a[i] & 0xFFFFu;
      k[2 * i + 1] = a[i] >> 16;
    }
  }
}
__device__ __forceinline__ uint32_t* dist_of(uint2* dp, uint32_t v) { return reinterpret_cast<uint32_t*>(dp + v); }
// The whole KE = 4 record (slots and keys, 32 bytes) in one 256-bit load.
__device__ __forceinline__ void ell_rec4(const FlatWs& w, uint32_t v, uint32_t (&r)[4], uint32_t (&k)[4]) {
  const uint32_t* p = w.ell + static_cast<uint64_t>(v) * 8;
  uint32_t k01, k23;
  asm("{.reg .b32 z0, z1;\n\t"
      "ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,z0,z1}, [%6];}"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(k01), "=r"(k23)
      : "l"(p));
  k[0] = k01 & 0xFFFFu;
  k[1] = k01 >> 16;
  k[2] = k23 & 0xFFFFu;
  k[3] = k23 >> 16;
}

// The Eq. 4 threshold sweep of one source, run by one warp: ord_d / ent are
// the source's sorted distances and sweep entries (reached positions);
// bucket (B words) and the cp.async ring s_sd (kFlatRing * kFlatChunk) /
// s_en (x KE) are the warp's shared memory.  Returns depth_per_source.
// bucket[k & M] = 1 + the largest d(v) over inserted slots u->v with key k;
// k is live at threshold tau iff that d(v) >= tau.  A slot's stale value
// (key k - B) is always below tau + 1 (its d(v) < k - B < tau), so slots are
// cleared only per source.
template <int KE>
__device__ __forceinline__ uint32_t flat_sweep(const uint32_t* __restrict__ ord_d, const uint32_t* __restrict__ ent,
                                              uint32_t reached, uint32_t B, uint32_t* bucket, uint32_t* s_sd,
                                              uint32_t* s_en, uint32_t lane) {
  const uint32_t M = B - 1;
  constexpr uint32_t kRingPos = kFlatRing * kFlatChunk;
  static_assert(kFlatChunk >= 64, "a 64-position block spans at most two chunks");
  for (uint32_t i = lane; i < B; i += 32) bucket[i] = 0;
  auto stage = [&](uint32_t c) {  // chunk c -> ring slot c % kFlatRing
    if (c * kFlatChunk < reached) {
      const uint32_t sl = c % kFlatRing;
      for (uint32_t k = lane; k < kFlatChunk / 4; k += 32)
        cp_async16(s_sd + sl * kFlatChunk + 4 * k, ord_d + c * kFlatChunk + 4 * k);
      for (uint32_t k = lane; k < kFlatChunk * KE / 4; k += 32)
        cp_async16(s_en + sl * kFlatChunk * KE + 4 * k,
                   ent + static_cast<uint64_t>(c) * kFlatChunk * KE + 4 * k);
    }
    cp_async_commit();
  };
  // chunks [cur, cur + kFlatRing) are issued; cur and cur + 1 are complete
  uint32_t issued = 0, cur = 0;
  for (; issued < static_cast<uint32_t>(kFlatRing); ++issued) stage(issued);
  cp_async_wait<kFlatRing - 2>();
  __syncwarp();
  auto advance_to = [&](uint32_t q) {  // position q (only grows) moves the window
    while (cur < q / kFlatChunk) {
      __syncwarp();  // every lane is done with chunk cur's slot
      ++cur;
      stage(issued++);
      cp_async_wait<kFlatRing - 2>();
      __syncwarp();
    }
  };
  // level 0 = {s}: insert its entries (d(s) = 0)
  uint32_t newmin = kInfDist;  // smallest key inserted by the last level, live at its threshold
  if (lane < KE) {
    const uint32_t e = s_en[lane];
    if (e) {
      atomicMax(bucket + ((e & 0xFFFFu) & M), (e >> 16) + 1);
      newmin = e & 0xFFFFu;  // d(v) = e >> 16 >= 1 = tau: live
    }
  }
  newmin = __reduce_min_sync(0xffffffffu, newmin);
  __syncwarp();
  uint32_t tau = 1, pos = 1, levels = 1;
  // the first 32 positions of the next level, loaded ahead of its threshold
  auto load_step = [&](uint32_t q, uint32_t& d, uint32_t (&e)[KE]) {
    const uint32_t qq = q + lane;
    d = qq < reached ? s_sd[qq % kRingPos] : kInfDist;
    const uint4* e4 = reinterpret_cast<const uint4*>(s_en + (qq % kRingPos) * KE);
#pragma unroll
    for (int h = 0; h < KE / 4; ++h) {
      const uint4 t = e4[h];
      e[4 * h] = t.x;
      e[4 * h + 1] = t.y;
      e[4 * h + 2] = t.z;
      e[4 * h + 3] = t.w;
    }
  };
  uint32_t pd, pe[KE];
  advance_to(pos);
  load_step(pos, pd, pe);
  for (;;) {
    // the next threshold: the first live key > tau in the ring, or newmin
    uint32_t nxt = newmin;
    for (uint32_t base = tau + 1; base < tau + B && base <= nxt; base += 32) {
      const uint32_t k = base + lane;
      const bool live = k < tau + B && bucket[k & M] >= tau + 1;
      __syncwarp();  // orders the last level's inserts before the scans after this one
      const uint32_t m = __ballot_sync(0xffffffffu, live);
      if (m) {
        nxt = min(nxt, base + __ffs(m) - 1);
        break;
      }
    }
    if (nxt == kInfDist) break;
    // the new level: positions [pos, end) with d < nxt, 32 per step
    uint32_t q = pos, lmin = kInfDist;
    uint32_t d = pd, ex[KE];
#pragma unroll
    for (int x = 0; x < KE; ++x) ex[x] = pe[x];
    for (;;) {
      const bool in = d < nxt;  // d = kInfDist past the end
      const uint32_t got = __popc(__ballot_sync(0xffffffffu, in));
#pragma unroll
      for (int x = 0; x < KE; ++x) {
        const uint32_t dvp1 = d + (ex[x] >> 16) + 1;
        const uint32_t key = d + (ex[x] & 0xFFFFu);
        const bool v = in && ex[x] != 0u && dvp1 > nxt;
        atomicMax(bucket + (key & M), v ? dvp1 : 0u);  // unconditional: no branch per entry
        lmin = v ? min(lmin, key) : lmin;
      }
      q += got;
      if (got < 32 || q >= reached) break;
      advance_to(q);
      load_step(q, d, ex);
    }
    newmin = __reduce_min_sync(0xffffffffu, lmin);
    pos = q;
    tau = nxt;
    ++levels;
    if (pos < reached) {
      advance_to(pos);
      load_step(pos, pd, pe);
    } else {
      pd = kInfDist;
#pragma unroll
      for (int x = 0; x < KE; ++x) pe[x] = 0;
    }
  }
  cp_async_wait<0>();
  __syncwarp();
  return levels;
}

// Named barriers of bc_flat_kernel (0 is __syncthreads, unused in the loop):
// 1 = the worker group (warps 1..), 2 / 3 = buffer 0 / 1 ready for the
// sweeper, 4 / 5 = buffer 0 / 1 released by the sweeper.
template <int ID>
__device__ __forceinline__ void nbar_sync(int count) {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(count) : "memory");
}
template <int ID>
__device__ __forceinline__ void nbar_arrive(int count) {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(count) : "memory");
}
// Sweeper j's buffer parity p: ready barrier 2 + 4j + p (workers arrive,
// the sweeper waits), released barrier 4 + 4j + p (the sweeper arrives, the
// workers wait).  kSweepers <= 3 keeps every id below 16.
template <bool READY>
__device__ __forceinline__ void buf_bar(bool sync, uint32_t j, uint32_t par, int count) {
  const uint32_t c = j * 2 + par;
  constexpr int kB = READY ? 2 : 4;
#define WBC_BUF_CASE(C)                                                   \
  case C:                                                                 \
    if (sync) nbar_sync<kB + 4 * ((C) / 2) + (C) % 2>(count);             \
    else nbar_arrive<kB + 4 * ((C) / 2) + (C) % 2>(count);                \
    break;
  switch (c) {
    WBC_BUF_CASE(0)
    WBC_BUF_CASE(1)
    WBC_BUF_CASE(2)
    WBC_BUF_CASE(3)
    WBC_BUF_CASE(4)
    WBC_BUF_CASE(5)
  }
#undef WBC_BUF_CASE
}

template <int T, int KE>
__global__ void __launch_bounds__(T, 1024 / T) bc_flat_kernel(const RunParams p, const FlatWs w) {
  static_assert(KE == 4 || KE == 8, "ELL row width");
  constexpr uint32_t kSW = kSweepers;       // sweeper warps (0 .. kSW - 1)
  constexpr uint32_t TG = T - 32 * kSW;     // worker threads (the other warps)
  constexpr int kBarN = TG + 32;            // threads on a ready / released barrier
  constexpr int kU = WBC_FLAT_KU;           // positions per thread in a pull block
  constexpr uint32_t kBlk = TG * kU;        // pull block (passes B and C)
  __shared__ unsigned long long s_src;
  __shared__ uint32_t s_ring[3][4];          // per-phase counters: [near, far, members, far min]
  __shared__ uint32_t s_warp[T / 32];
  __shared__ double s_blk[kBlk];             // the block's sigma (B) / coef (C); 0 = not final
  __shared__ uint32_t s_sw[kSW][2][3];       // per sweeper and buffer: reached, source, exit
  extern __shared__ uint32_t smem[];         // hist | per sweeper: buckets, sweep ring | near queues
  const GraphView& g = p.g;
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31, wid = tid >> 5;
  const uint64_t off = static_cast<uint64_t>(blockIdx.x) * w.n_stride;
  uint2* const dp = w.dp + off;
  uint32_t* const order = w.order + off;
  uint32_t* const mem = w.mem + off;
  double* const psig = w.psig + off;
  double* const pcoef = w.pcoef + off;
  uint32_t* const pinfo = w.pinfo + off;
  uint32_t* const psucc = w.psucc + off * KE;
  uint32_t* const hist = smem;
  // near queues: entries [0, sq_cap) in shared memory, the rest in q0 / q1
  uint32_t* const sq0 = smem + w.delta_words + kSW * (w.buckets + kFlatRing * kFlatChunk * (1 + KE));
  uint32_t* const sq1 = sq0 + w.sq_cap;
  const uint32_t sqc = w.sq_cap;
  const uint32_t wbits = g.wbits, wmask = g.wmask;
  // the sweep inputs are double-buffered per sweeper: buffer (j, parity)
  auto ord_d_of = [&](uint32_t j, uint32_t par) { return w.ord_d + (2 * kSW * off + (2 * j + par) * w.n_stride); };
  auto ent_of = [&](uint32_t j, uint32_t par) {
    return w.ent + (2 * kSW * off + (2 * j + par) * w.n_stride) * KE;
  };

  if (wid < kSW) {
    // ===================== sweeper j (warp j): the Eq. 4 thresholds of the
    // sources j, j + kSW, j + 2 kSW, ... this CTA runs, each while the
    // workers run the following ones (one sweep takes about as long as a
    // source's SSSP + sigma + delta, so kSW sweepers keep up).
    const uint32_t j = wid, B = w.buckets;
    uint32_t* const bucket = smem + w.delta_words + j * (B + kFlatRing * kFlatChunk * (1 + KE));
    uint32_t* const s_sd = bucket + B;
    uint32_t* const s_en = s_sd + kFlatRing * kFlatChunk;
    for (uint32_t m = 0;; ++m) {
      const uint32_t par = m & 1;
      buf_bar<true>(true, j, par, kBarN);
      if (s_sw[j][par][2]) break;
      const unsigned long long t_sweep = clock64();
      const uint32_t reached = s_sw[j][par][0], s_orig = s_sw[j][par][1];
      const uint32_t levels = flat_sweep<KE>(ord_d_of(j, par), ent_of(j, par), reached, B, bucket, s_sd, s_en, lane);
      if (lane == 0 && p.depth) p.depth[s_orig] = levels;
      if (p.prof && lane == 0) atomicAdd(p.prof + kProfCyclesSettle, clock64() - t_sweep);
      buf_bar<false>(false, j, par, kBarN);  // buffer (j, par) is free again
    }
    return;
  }

  // ======================= the workers (warps kSW..): SSSP, sigma, delta
  const uint32_t gt = tid - 32 * kSW, gw = wid - kSW;  // worker thread / warp index
  auto gsync = [&]() { nbar_sync<1>(TG); };
  auto gsync_or = [&](uint32_t pred) { return bar_or(pred, 1, TG); };
  // p.prof: per-phase SM cycles of worker 0 (init -> kProfCyclesInit, A ->
  // kProfCyclesRelax, B -> kProfCyclesThreshold, C -> kProfCyclesBackward),
  // A's barrier phases -> kProfRounds, windows -> kProfRefills; the sweeper
  // adds its own cycles to kProfCyclesSettle
  unsigned long long t_last = 0;
  auto tick = [&](int slot) {
    if (p.prof && gt == 0) {
      const unsigned long long t = clock64();
      if (slot >= 0) atomicAdd(p.prof + slot, t - t_last);
      t_last = t;
    }
  };
  uint32_t nsrc = 0;  // sources this CTA has run
  for (;; ++nsrc) {
    if (gt == 0) s_src = atomicAdd(p.counter, 1ULL);
    gsync();
    const unsigned long long idx = s_src;
    // source nsrc goes to sweeper sj, its m-th, buffer parity sp
    const uint32_t sj = nsrc % kSW, sm_ = nsrc / kSW, sp = sm_ & 1;
    if (idx >= p.k) {
      // release every sweeper: consume its outstanding releases, signal the exit
      for (uint32_t jj = 0; jj < kSW; ++jj) {
        const uint32_t cnt = (nsrc + kSW - 1 - jj) / kSW;  // sources sweeper jj got
        if (cnt >= 2) buf_bar<false>(true, jj, cnt & 1, kBarN);  // sweep cnt - 2 released
        if (gt == 0) s_sw[jj][cnt & 1][2] = 1;
        buf_bar<true>(false, jj, cnt & 1, kBarN);
        if (cnt >= 1) buf_bar<false>(true, jj, (cnt - 1) & 1, kBarN);  // sweep cnt - 1 released
      }
      break;
    }
    const uint32_t s_orig = p.sources ? __ldg(p.sources + idx) : static_cast<uint32_t>(p.src_base + idx);
    const uint32_t s = __ldg(p.inv + s_orig);
    tick(-1);
    if (sm_ >= 2) buf_bar<false>(true, sj, sp, kBarN);  // sweeper sj is done with this buffer (its m - 2)
    uint32_t* const ord_d = ord_d_of(sj, sp);
    uint32_t* const ent = ent_of(sj, sp);

    // ---- init: every word (infinite distance, position 0)
    {
      uint4* const d4 = reinterpret_cast<uint4*>(dp);
      const uint32_t n2 = static_cast<uint32_t>(w.n_stride / 2);
      for (uint32_t i = gt; i < n2; i += TG) __stcg(d4 + i, make_uint4(kInfDist, 0u, kInfDist, 0u));
    }
    if (gt < 12) (&s_ring[0][0])[gt] = gt % 4 == 3 ? kInfDist : 0u;
    gsync();
    if (gt == 0) {
      *dist_of(dp, s) = 0;
      if (sqc)
        sq0[0] = s;
      else
        w.q0[off] = s;
      mem[0] = s;
    }
    gsync();
    tick(kProfCyclesInit);

    // ---- A. near-far SSSP; windows sorted into `order` as they close
    uint32_t* nq = w.q0 + off;
    uint32_t* nn = w.q1 + off;
    uint32_t* snq = sq0;
    uint32_t* snn = sq1;
    uint32_t* fq = w.q2 + off;
    uint32_t* fq2 = w.q3 + off;
    uint32_t near_len = 1, far_len = 0, mem_len = 1, olen = 0, ph = 0, windows = 0;
    uint64_t lo = 0, thr = w.delta_w;
    for (;;) {
      uint32_t* R = s_ring[ph % 3];
      if (gt == 0) {
        uint32_t* Z = s_ring[(ph + 1) % 3];
        Z[0] = 0;
        Z[1] = 0;
        Z[2] = 0;
        Z[3] = kInfDist;
      }
      const uint32_t thr32 = thr >= kInfDist ? kInfDist : static_cast<uint32_t>(thr);
      if (near_len) {
        // relax every near vertex: its ELL slots, then the neighbours'
        // distances, then the atomics (each stage's loads in flight together)
        for (uint32_t i0 = gt; i0 < near_len; i0 += TG * kRelaxU) {
          uint32_t dv[kRelaxU], r[kRelaxU][KE], nd[kRelaxU][KE], old[kRelaxU][KE];
#pragma unroll
          for (int j = 0; j < kRelaxU; ++j) {
            const uint32_t i = i0 + j * TG;
            const uint32_t v = i < near_len ? (i < sqc ? snq[i] : nq[i]) : kInfDist;
            dv[j] = v != kInfDist ? ld_own<0>(dist_of(dp, v)) : kInfDist;
            if (v != kInfDist)
              ell_row<KE>(w, v, r[j]);
            else
#pragma unroll
              for (int x = 0; x < KE; ++x) r[j][x] = 0;
          }
#pragma unroll
          for (int j = 0; j < kRelaxU; ++j)
#pragma unroll
            for (int x = 0; x < KE; ++x) {
              const uint32_t wt = r[j][x] & wmask;
              nd[j][x] = wt ? dv[j] + wt : kInfDist;
            }
          if constexpr (kRelaxPrecheck) {
#pragma unroll
            for (int j = 0; j < kRelaxU; ++j)
#pragma unroll
              for (int x = 0; x < KE; ++x)
                if (nd[j][x] != kInfDist && nd[j][x] >= __ldcg(dist_of(dp, r[j][x] >> wbits))) nd[j][x] = kInfDist;
          }
#pragma unroll
          for (int j = 0; j < kRelaxU; ++j)
#pragma unroll
            for (int x = 0; x < KE; ++x)
              old[j][x] = nd[j][x] != kInfDist ? atomicMin(dist_of(dp, r[j][x] >> wbits), nd[j][x]) : 0u;
#pragma unroll
          for (int j = 0; j < kRelaxU; ++j)
#pragma unroll
            for (int x = 0; x < KE; ++x) {
              if (nd[j][x] == kInfDist || nd[j][x] >= old[j][x]) continue;
              const uint32_t u = r[j][x] >> wbits;
              if (nd[j][x] < thr32) {
                // duplicates in the next near list are harmless (a re-relax
                // reads the current distance); members are appended once, at
                // the crossing below the window end
                const uint32_t k = atomicAdd(&R[0], 1u);
                if (k < sqc)
                  snn[k] = u;
                else
                  nn[k] = u;
                if constexpr (kRelaxPrefetch) asm volatile("prefetch.global.L2 [%0];" ::"l"(ell_rec<KE>(w, u)));
                if (old[j][x] >= thr32) mem[mem_len + atomicAdd(&R[2], 1u)] = u;
              } else if (old[j][x] == kInfDist) {
                fq[far_len + atomicAdd(&R[1], 1u)] = u;
              }
            }
        }
        gsync();
#ifdef WBC_FLAT_SSSP_PROF
        if (p.prof && gt == 0) atomicAdd(p.prof + kProfNearScanned, static_cast<unsigned long long>(near_len));
#endif
        near_len = R[0];
        far_len += R[1];
        mem_len += R[2];
        uint32_t* t = nq;
        nq = nn;
        nn = t;
        t = snq;
        snq = snn;
        snn = t;
        ++ph;
        continue;
      }
      // the window [lo, thr) is closed: its members are final.  Counting
      // sort on d - lo (< delta_w) appends them to order / ord_d and records
      // each one's position; its sigma flag is cleared for pass B.
      if (mem_len) {
        const uint32_t span = static_cast<uint32_t>(thr - lo < w.delta_w ? thr - lo : w.delta_w);
        for (uint32_t i = gt; i < span; i += TG) hist[i] = 0;
        gsync();
        constexpr int kM = WBC_FLAT_SORT_U;  // members per thread and step, gathers in flight together
        for (uint32_t i0 = gt; i0 < mem_len; i0 += TG * kM) {
          uint32_t u[kM], du[kM];
#pragma unroll
          for (int j = 0; j < kM; ++j) u[j] = i0 + j * TG < mem_len ? mem[i0 + j * TG] : kInfDist;
#pragma unroll
          for (int j = 0; j < kM; ++j) du[j] = u[j] != kInfDist ? ld_own<0>(dist_of(dp, u[j])) : 0u;
#pragma unroll
          for (int j = 0; j < kM; ++j)
            if (u[j] != kInfDist) {
              atomicAdd(hist + (du[j] - lo), 1u);
              if constexpr (kSortKeepD) fq2[i0 + j * TG] = du[j];  // the far spare is free until the refill
            }
        }
        gsync();
        // exclusive scan of hist[0, span): a contiguous chunk per thread
        const uint32_t per = (span + TG - 1) / TG, b0 = min(span, gt * per), b1 = min(span, b0 + per);
        uint32_t loc = 0;
        for (uint32_t i = b0; i < b1; ++i) loc += hist[i];
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        if (lane == 31) s_warp[gw] = incl;
        gsync();
        if (gw == 0) {
          uint32_t ws = lane < TG / 32 ? s_warp[lane] : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= static_cast<uint32_t>(o)) ws += y;
          }
          if (lane < TG / 32) s_warp[lane] = ws;
        }
        gsync();
        uint32_t run = olen + (gw ? s_warp[gw - 1] : 0u) + incl - loc;
        for (uint32_t i = b0; i < b1; ++i) {
          const uint32_t c = hist[i];
          hist[i] = run;
          run += c;
        }
        gsync();
        for (uint32_t i0 = gt; i0 < mem_len; i0 += TG * kM) {
          uint32_t u[kM], du[kM];
#pragma unroll
          for (int j = 0; j < kM; ++j) u[j] = i0 + j * TG < mem_len ? mem[i0 + j * TG] : kInfDist;
#pragma unroll
          for (int j = 0; j < kM; ++j)
            du[j] = u[j] == kInfDist ? 0u : kSortKeepD ? fq2[i0 + j * TG] : __ldcg(dist_of(dp, u[j]));
#pragma unroll
          for (int j = 0; j < kM; ++j) {
            if (u[j] == kInfDist) continue;
            const uint32_t q = atomicAdd(hist + (du[j] - lo), 1u);
            order[q] = u[j];
            ord_d[q] = du[j];
            dp[u[j]].y = q;
            __stcg(psig + q, 0.0);
          }
        }
        olen += mem_len;
        mem_len = 0;
        ++windows;
        gsync();
      }
      if (far_len == 0) break;
      // next window [thr, thr + delta): far entries inside it become near
      // (and members); the rest are compacted into the other far buffer
      const uint64_t thr_new = thr + w.delta_w;
      const uint32_t tn32 = thr_new >= kInfDist ? kInfDist : static_cast<uint32_t>(thr_new);
      constexpr int kF = WBC_FLAT_SORT_U;  // far entries per thread and step, gathers in flight together
      for (uint32_t i0 = gt; i0 < far_len; i0 += TG * kF) {
        uint32_t u[kF], du[kF];
#pragma unroll
        for (int j = 0; j < kF; ++j) u[j] = i0 + j * TG < far_len ? fq[i0 + j * TG] : kInfDist;
#pragma unroll
        for (int j = 0; j < kF; ++j) du[j] = u[j] != kInfDist ? ld_own<0>(dist_of(dp, u[j])) : 0u;
#pragma unroll
        for (int j = 0; j < kF; ++j) {
          if (u[j] == kInfDist || du[j] < thr32) continue;  // joined an earlier window: sorted already
          if (du[j] < tn32) {
            const uint32_t k = atomicAdd(&R[0], 1u);
            if (k < sqc)
              snq[k] = u[j];
            else
              nq[k] = u[j];
            if constexpr (kRelaxPrefetch) asm volatile("prefetch.global.L2 [%0];" ::"l"(ell_rec<KE>(w, u[j])));
            mem[atomicAdd(&R[2], 1u)] = u[j];
          } else {
            fq2[atomicAdd(&R[1], 1u)] = u[j];
            atomicMin(&R[3], du[j]);
          }
        }
      }
      gsync();
      near_len = R[0];
      far_len = R[1];
      mem_len = R[2];
      {
        uint32_t* t = fq;
        fq = fq2;
        fq2 = t;
      }
      lo = thr;
      thr = thr_new;
      if (near_len == 0 && far_len) thr = static_cast<uint64_t>(R[3]);  // jump: the next window opens at the far minimum
      ++ph;
    }
    const uint32_t reached = olen;
    tick(kProfCyclesRelax);
    if (p.prof && gt == 0) {
      atomicAdd(p.prof + kProfRounds, static_cast<unsigned long long>(ph));
      atomicAdd(p.prof + kProfRefills, static_cast<unsigned long long>(windows));
    }

    // ---- B. sigma in distance order, a block of kBlk positions at a time.
    // Predecessors in earlier blocks are final (global psig); those inside
    // the block are resolved by barrier rounds over the block's shared-memory
    // copy (0 = not yet final: sigma >= 1).  The same pass writes per
    // position the successor mask and positions, the sweep entries, and
    // clears pcoef for pass C -- all coalesced.
    for (uint32_t a = 0; a < reached; a += kBlk) {
      uint32_t v[kU], dv[kU], r[kU][KE], kk[kU][KE], sp[kU][KE], pend[kU];
      uint2 nb[kU][KE];
      double sg[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t q = a + gt + j * TG;
        v[j] = q < reached ? __ldcg(order + q) : 0u;
        dv[j] = q < reached ? __ldcg(ord_d + q) : kInfDist;
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        if (dv[j] != kInfDist) {
          if constexpr (KE == 4) {
            ell_rec4(w, v[j], r[j], kk[j]);
          } else {
            ell_row<KE>(w, v[j], r[j]);
            ell_keys<KE>(w, v[j], kk[j]);
          }
        } else {
#pragma unroll
          for (int x = 0; x < KE; ++x) r[j][x] = kk[j][x] = 0;
        }
      }
#pragma unroll
      for (int j = 0; j < kU; ++j)
#pragma unroll
        for (int x = 0; x < KE; ++x)
          nb[j][x] = (r[j][x] & wmask) ? ld_own<1>(dp + (r[j][x] >> wbits)) : make_uint2(kInfDist, 0u);
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t q = a + gt + j * TG;
        pend[j] = 0;
        sg[j] = 0.0;
        uint32_t pm = 0, sm = 0, e[KE];
#pragma unroll
        for (int x = 0; x < KE; ++x) {
          const uint32_t wt = r[j][x] & wmask, d = nb[j][x].x;
          e[x] = 0;
          sp[j][x] = nb[j][x].y;
          if (!wt || d == kInfDist) continue;  // padding (a reached vertex's neighbours are reached)
          if (d + wt == dv[j]) pm |= 1u << x;
          if (dv[j] + wt == d) sm |= 1u << x;
          if (d > dv[j]) e[x] = kk[j][x] | (d - dv[j]) << 16;
        }
        if (q >= reached) continue;
        __stcg(pcoef + q, 0.0);
        __stcg(pinfo + q, sm | pm << 8);
        uint4* const so = reinterpret_cast<uint4*>(psucc + static_cast<uint64_t>(q) * KE);
        uint4* const eo = reinterpret_cast<uint4*>(ent + static_cast<uint64_t>(q) * KE);
#pragma unroll
        for (int x = 0; x < KE / 4; ++x) {
          __stcg(so + x, make_uint4(sp[j][4 * x], sp[j][4 * x + 1], sp[j][4 * x + 2], sp[j][4 * x + 3]));
          __stcg(eo + x, make_uint4(e[4 * x], e[4 * x + 1], e[4 * x + 2], e[4 * x + 3]));
        }
        if (q == 0) {
          sg[j] = 1.0;  // the source (the only vertex at distance 0)
        } else {
#pragma unroll
          for (int x = 0; x < KE; ++x)
            if (pm >> x & 1u) {
              if (sp[j][x] < a)
                sg[j] += ld_own<2>(psig + sp[j][x]);
              else
                pend[j] |= 1u << x;
            }
        }
        s_blk[q - a] = pend[j] ? 0.0 : sg[j];
      }
      for (;;) {
        uint32_t any = 0;
#pragma unroll
        for (int j = 0; j < kU; ++j) any |= pend[j];
        if (!gsync_or(any)) break;
        // a round: read the values final so far, then (after a barrier) publish
        // the ones this round completed -- reads and writes never overlap
        uint32_t fin = 0;
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          if (!pend[j]) continue;
#pragma unroll
          for (int x = 0; x < KE; ++x)
            if (pend[j] >> x & 1u) {
              const double y = s_blk[sp[j][x] - a];
              if (y != 0.0) {
                sg[j] += y;
                pend[j] &= ~(1u << x);
              }
            }
          if (!pend[j]) fin |= 1u << j;
        }
        gsync();
#pragma unroll
        for (int j = 0; j < kU; ++j)
          if (fin >> j & 1u) s_blk[gt + j * TG] = sg[j];
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t q = a + gt + j * TG;
        if (q >= reached) continue;
        note_sigma(p.overflow, sg[j]);
        __stcg(psig + q, sg[j]);
      }
      gsync();  // the block's sigma is visible to the next block's loads
    }
    tick(kProfCyclesThreshold);
    // hand the distances and entries to the sweeper (buffer b)
    if (gt == 0) {
      s_sw[sj][sp][0] = reached;
      s_sw[sj][sp][1] = s_orig;
      s_sw[sj][sp][2] = 0;
    }
    buf_bar<true>(false, sj, sp, kBarN);

    // ---- C. delta in reverse distance order, a block of kBlk positions at a
    // time: successors in later blocks are final (global pcoef), those inside
    // the block resolve by barrier rounds over its shared-memory copy.  Node
    // BC += delta (u != s), edge BC += c.
    for (uint32_t bend = reached; bend > 0;) {
      const uint32_t a = bend > kBlk ? bend - kBlk : 0u;
      uint32_t u[kU], sm[kU], sp[kU][KE];
      double su[kU], dsum[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t i = gt + j * TG;  // q = bend - 1 - i, in [a, bend) when i < bend - a
        const bool ok = i < bend - a;
        const uint32_t q = ok ? bend - 1 - i : 0u;
        u[j] = ok ? __ldcg(order + q) : 0u;
        sm[j] = ok ? __ldcg(pinfo + q) & 0xFFu : 0u;
        su[j] = ok ? __ldcg(psig + q) : 1.0;
        const uint4* so = reinterpret_cast<const uint4*>(psucc + static_cast<uint64_t>(q) * KE);
#pragma unroll
        for (int x = 0; x < KE / 4; ++x) {
          const uint4 t4 = sm[j] ? __ldcg(so + x) : make_uint4(0, 0, 0, 0);
          sp[j][4 * x] = t4.x;
          sp[j][4 * x + 1] = t4.y;
          sp[j][4 * x + 2] = t4.z;
          sp[j][4 * x + 3] = t4.w;
        }
      }
      uint32_t pend[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t i = gt + j * TG;
        dsum[j] = 0.0;
        pend[j] = 0;
#pragma unroll
        for (int x = 0; x < KE; ++x) {
          if (!(sm[j] >> x & 1u)) continue;
          if (sp[j][x] >= bend) {
            const double c = su[j] * ld_own<3>(pcoef + sp[j][x]);
            dsum[j] += c;
            if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(w.ell_eid + static_cast<uint64_t>(u[j]) * KE + x), c);
          } else {
            pend[j] |= 1u << x;
          }
        }
        if (i < bend - a) s_blk[bend - 1 - i - a] = pend[j] ? 0.0 : (1.0 + dsum[j]) / su[j];
      }
      for (;;) {
        uint32_t any = 0;
#pragma unroll
        for (int j = 0; j < kU; ++j) any |= pend[j];
        if (!gsync_or(any)) break;
        uint32_t fin = 0;  // a round: reads, barrier, then this round's completions
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          if (!pend[j]) continue;
#pragma unroll
          for (int x = 0; x < KE; ++x)
            if (pend[j] >> x & 1u) {
              const double y = s_blk[sp[j][x] - a];
              if (y != 0.0) {
                const double c = su[j] * y;
                dsum[j] += c;
                if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(w.ell_eid + static_cast<uint64_t>(u[j]) * KE + x), c);
                pend[j] &= ~(1u << x);
              }
            }
          if (!pend[j]) fin |= 1u << j;
        }
        gsync();
#pragma unroll
        for (int j = 0; j < kU; ++j)
          if (fin >> j & 1u) s_blk[bend - 1 - (gt + j * TG) - a] = (1.0 + dsum[j]) / su[j];
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const uint32_t i = gt + j * TG;
        if (i >= bend - a) continue;
        const uint32_t q = bend - 1 - i;
        __stcg(pcoef + q, (1.0 + dsum[j]) / su[j]);
        if (q != 0 && dsum[j] != 0.0) atomicAdd(p.node_bc + u[j], dsum[j]);  // not the source
      }
      gsync();  // the block's coef is visible to the next block
      bend = a;
    }
    tick(kProfCyclesBackward);
  }
}

}  // namespace wbc_dev
