// bc_warp.cuh -- one WARP per source, for flat large-diameter graphs (grid /
// road-like: ~10^5 Eq. 4 rounds per source, ~50-vertex levels).
//
// Such sources are bound by the number of serialised global-memory round
// trips per round, so everything a round needs besides the graph and the
// per-vertex arrays stays on chip, in registers and the CTA's shared memory
// (the CTA is the one warp):
//  * the near set (pending vertices with d < F, or any pending vertex that
//    improved while in it) is a dense shared-memory list of (u, d, min_w,
//    row, deg) with an open-addressing hash index u -> list position: the
//    threshold min(d + min_w) and the settle are shared-memory scans, and the
//    row data of a settled vertex was gathered when it entered the set;
//  * the level being relaxed (the frontier) is a shared-memory list too;
//  * settled vertices carry kSettledBit in their distance word, so the relax
//    tells DAG predecessors (settled, d + w == d[v]) from improvable
//    neighbours (unsettled, d + w < d[u]) with the one gather it needs anyway.
// Per round that leaves three dependent trips (slot words, distance gathers,
// then atomicMin / min-weight / row offsets / sigma together) instead of
// the team kernel's ~20.  The far set stays a global list of ids, refilled
// by the near/far window rule of bc_team.cuh (exact Delta).
//
// Anything the fixed on-chip capacities cannot hold (a frontier above
// kWFront, a near set above kWNear, a DAG above its buffer, a distance
// that would reach the settled bit) ABORTS the
// source before anything was accumulated: its index goes to an abort list
// and the launcher re-runs those sources with the team kernel in the same
// stream.  Results never depend on the fast path succeeding.
//
// Semantics as bc_team.cuh / the reference: engine.cpp:118-222 (Eq. 4
// rounds), :183-212 (dependency accumulation), SURVEY.md §8(a').
#pragma once

#include <type_traits>

#include "bc_kernels.cuh"

namespace wbc_dev {

constexpr uint32_t kSettledBit = 0x80000000u;
constexpr uint32_t kDistMask = 0x7FFFFFFFu;
constexpr int kWNear = 1024;   // near-set capacity (entries)
constexpr int kWHash = 2048;   // hash slots (power of two, >= 2 * kWNear)
constexpr int kWFront = 256;   // frontier capacity (one level)
constexpr int kWQ = 32 * kUnroll + 32;  // pass-1 compaction queue capacity
constexpr uint32_t kHEmpty = 0xFFFFFFFFu;
constexpr uint32_t kHTomb = 0xFFFFFFFEu;

struct WarpSmem {
  uint32_t hkey[kWHash];  // vertex id, kHEmpty or kHTomb
  uint32_t hval[kWHash];  // position in the near list
  uint32_t nu[kWNear], nd[kWNear], nmw[kWNear], nrow[kWNear], ndeg[kWNear], nh[kWNear];
  uint32_t fv[kWFront], fd[kWFront], frow[kWFront], fpref[kWFront + 1];
  uint32_t qiu[kWQ], qid[kWQ], qpu[kWQ], qpv[kWQ], qps[kWQ];
};

struct WarpParams {
  GraphView g;
  // per-slot arrays, slot stride n_stride (dag: dag_cap)
  uint32_t* dist;
  double* sigma;
  double* delta;
  uint32_t* order;
  uint32_t* level_ends;
  uint32_t* dag_ends;
  uint32_t* far_q;
  uint2* dag;        // (predecessor u, successor v)
  uint32_t* dag_slot;  // slot of v's row (edge BC only)
  uint64_t n_stride, dag_cap;
  const uint32_t* sources;
  uint64_t k;
  unsigned long long* counter;
  double* node_bc;
  double* edge_bc;
  uint32_t* depth;
  uint32_t near_width;
  const uint32_t* inv;
  uint32_t* abort_list;               // original ids of aborted sources
  unsigned long long* abort_count;
  unsigned long long* prof;
};

__device__ __forceinline__ uint32_t whash(uint32_t u) { return (u * 0x9E3779B1u) >> (32 - 11); }
static_assert(kWHash == 2048, "whash yields 11 bits");

// Open addressing with linear probing; tombstones are never reused (the
// index is rebuilt between rounds once a quarter of it is occupied, and a
// round adds at most kWNear keys), so an empty slot always exists.
__device__ __forceinline__ uint32_t wfind(const uint32_t* hkey, uint32_t u) {
  uint32_t h = whash(u);
  for (int t = 0; t < kWHash; ++t) {
    const uint32_t key = hkey[h];
    if (key == u) return h;
    if (key == kHEmpty) return kHEmpty;
    h = (h + 1) & (kWHash - 1);
  }
  return kHEmpty;
}
// Returns the slot holding u (claimed if absent); sets created.  kHEmpty if full.
__device__ __forceinline__ uint32_t wclaim(uint32_t* hkey, uint32_t u, bool& created) {
  uint32_t h = whash(u);
  created = false;
  for (int t = 0; t < kWHash; ++t) {
    const uint32_t prevk = atomicCAS(&hkey[h], kHEmpty, u);
    if (prevk == kHEmpty) { created = true; return h; }
    if (prevk == u) return h;
    h = (h + 1) & (kWHash - 1);
  }
  return kHEmpty;
}

template <bool PACKED, bool PROF>
__global__ void __launch_bounds__(32, 4) bc_warp_kernel(const WarpParams p) {
  extern __shared__ __align__(16) unsigned char warp_smem_raw[];
  WarpSmem& sh = *reinterpret_cast<WarpSmem*>(warp_smem_raw);
  const GraphView& g = p.g;
  const uint32_t lane = threadIdx.x;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t off = static_cast<uint64_t>(blockIdx.x) * p.n_stride;
  const uint64_t keep_pol = l2_policy_evict_last();
  const uint64_t stream_pol = l2_policy_evict_first();
  uint32_t* const dist = p.dist + off;
  double* const sigma = p.sigma + off;
  double* const delta = p.delta + off;
  uint32_t* const order = p.order + off;
  uint32_t* const lev = p.level_ends + off;
  uint32_t* const dag_ends = p.dag_ends + off;
  uint32_t* const far_q = p.far_q + off;
  uint2* const dag = p.dag + static_cast<uint64_t>(blockIdx.x) * p.dag_cap;
  uint32_t* const dag_slot = p.dag_slot ? p.dag_slot + static_cast<uint64_t>(blockIdx.x) * p.dag_cap : nullptr;
  const uint32_t dag_cap = static_cast<uint32_t>(p.dag_cap);
  const uint32_t n = g.n;
  const uint32_t W = p.near_width;
  auto dload = [&](uint32_t u) { return ld_cg_hint(dist + u, keep_pol); };
  unsigned long long c_relax = 0, c_near = 0, c_far = 0, c_refill = 0, c_impr = 0, c_rounds = 0;
  unsigned long long t_last = 0, t_phase[5] = {0, 0, 0, 0, 0};
  auto tick = [&](int k) {
    if (PROF && lane == 0) {
      const unsigned long long t = clock64();
      t_phase[k] += t - t_last;
      t_last = t;
    }
  };

  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(p.counter, 1ULL);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= p.k) break;
    const uint32_t s_orig = p.sources ? __ldg(p.sources + idx) : static_cast<uint32_t>(idx);
    const uint32_t s = __ldg(p.inv + s_orig);
    if (PROF && lane == 0) t_last = clock64();

    // ---- init_state (engine.cpp:118-142)
    {
      uint4* d4 = reinterpret_cast<uint4*>(dist);
      const uint4 inf4 = make_uint4(kInfDist, kInfDist, kInfDist, kInfDist);
      for (uint32_t i = lane; i < n / 4; i += 32) d4[i] = inf4;
      for (uint32_t i = (n / 4) * 4 + lane; i < n; i += 32) dist[i] = kInfDist;
      for (uint32_t i = lane; i < kWHash; i += 32) sh.hkey[i] = kHEmpty;
    }
    __syncwarp();
    const uint32_t s_row = __ldg(g.offsets + s);
    const uint32_t s_deg = __ldg(g.offsets + s + 1) - s_row;
    if (lane == 0) {
      dist[s] = kSettledBit;  // d = 0, settled
      order[0] = s;
      lev[0] = 0;
      lev[1] = 1;
      dag_ends[0] = 0;
      sigma[s] = 1.0;
      delta[s] = 0.0;
      sh.fv[0] = s;
      sh.fd[0] = 0;
      sh.frow[0] = s_row;
      sh.fpref[0] = 0;
      sh.fpref[1] = s_deg;
    }
    __syncwarp();
    uint32_t fcnt = 1, fb = 0, nlev = 1, ord_len = 1, dag_len = 0, near_n = 0, far_len = 0, htomb = 0;
    uint64_t F = W;
    bool abort = false;
    int cause = -1;  // kProfAbort* (profiling only)
    tick(0);

    for (;;) {
      ++c_rounds;
      // ---------------- relax level nlev-1: from shared memory, or (levels
      // above kWFront) in chunks streamed from the global order
      const uint32_t Fu = F >= kInfDist ? kInfDist : static_cast<uint32_t>(F);
      uint32_t iq_n = 0, pq_n = 0;
      // improvements: atomicMin with the new vertex's min-weight and row
      // offsets in flight; near set updated in shared memory
      auto drain_imp = [&](uint32_t m) {
        const uint32_t i = iq_n - m + lane;
        const bool act = lane < m;
        uint32_t u = 0, nd = 0, old = kInfDist, mw = 0, r0 = 0, r1 = 0;
        if (act) {
          u = sh.qiu[i];
          nd = sh.qid[i];
          old = atom_min_hint(dist + u, nd, keep_pol);
          mw = __ldg(g.minw + u);
          r0 = __ldg(g.offsets + u);
          r1 = __ldg(g.offsets + u + 1);
        }
        const bool imp = act && nd < old;
        c_impr += imp;
        // find u in the near index
        uint32_t h = 0, pos = kHEmpty;
        if (imp) pos = wfind(sh.hkey, u);
        // not in the near set: insert (d < F) or append to far (first reach)
        const bool ins = imp && pos == kHEmpty && nd < Fu;
        const bool far = imp && pos == kHEmpty && nd >= Fu && old == kInfDist;
        if (ins) {
          // claim a hash slot (several lanes may carry the same u)
          bool created = false;
          h = wclaim(sh.hkey, u, created);
          if (h == kHEmpty) abort = true;
          pos = h == kHEmpty ? kHEmpty : (created ? 0xFFFFFFFDu : h);  // creators allocate below
        }
        // creators: allocate near-list positions (ballot-aggregated)
        const uint32_t bc = __ballot_sync(0xffffffffu, ins && pos == 0xFFFFFFFDu);
        if (bc) {
          if (bc >> lane & 1u) {
            const uint32_t np = near_n + __popc(bc & lt);
            if (np < kWNear) {
              sh.nu[np] = u;
              sh.nd[np] = nd;
              sh.nmw[np] = mw;
              sh.nrow[np] = r0;
              sh.ndeg[np] = r1 - r0;
              sh.nh[np] = h;
              sh.hval[h] = np;
            } else {
              abort = true;
            }
            pos = h;
          }
          near_n += __popc(bc);
        }
        __syncwarp();
        // everyone holding a hash slot lowers the entry's distance
        if (imp && pos != kHEmpty && !(ins && (bc >> lane & 1u))) {
          const uint32_t np = sh.hval[pos];
          if (np < kWNear) atomicMin(&sh.nd[np], nd);
        }
        const uint32_t bf = __ballot_sync(0xffffffffu, far);
        if (bf) {
          if (far) far_q[far_len + __popc(bf & lt)] = u;
          far_len += __popc(bf);
        }
        __syncwarp();
        iq_n -= m;
      };
      // DAG predecessors: sigma pull (integer-valued fp64, exact in any order)
      auto drain_pred = [&](uint32_t m) {
        const uint32_t i = pq_n - m + lane;
        const bool act = lane < m;
        uint32_t u = 0, v = 0, sl = 0;
        double sg = 0.0;
        if (act) {
          u = sh.qpu[i];
          v = sh.qpv[i];
          sl = sh.qps[i];
          sg = __ldcg(sigma + u);
        }
        if (act) {
          atomicAdd(sigma + v, sg);
          const uint32_t q = dag_len + lane;
          if (q < dag_cap) {
            dag[q] = make_uint2(u, v);
            if (dag_slot) dag_slot[q] = sl;
          }
        }
        dag_len += m;
        __syncwarp();
        pq_n -= m;
      };
      for (uint32_t cs = 0; cs < fcnt; cs += kWFront) {
        const uint32_t ccnt = min(static_cast<uint32_t>(kWFront), fcnt - cs);
        if (fcnt > kWFront) {  // stage the chunk: order -> distance and row offsets
          uint32_t carry = 0;
          for (uint32_t c = 0; c < ccnt; c += 32) {
            const uint32_t i = c + lane;
            uint32_t v = 0, d = 0, r0 = 0, r1 = 0;
            if (i < ccnt) {
              v = __ldcg(order + fb + cs + i);
              d = dload(v) & kDistMask;
              r0 = __ldg(g.offsets + v);
              r1 = __ldg(g.offsets + v + 1);
            }
            uint32_t x = r1 - r0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
              if (lane >= static_cast<uint32_t>(o)) x += y;
            }
            if (i < ccnt) {
              sh.fv[i] = v;
              sh.fd[i] = d;
              sh.frow[i] = r0;
              sh.fpref[i + 1] = carry + x;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
          }
          if (lane == 0) sh.fpref[0] = 0;
          __syncwarp();
        }
        const uint32_t total = sh.fpref[ccnt];
        c_relax += total;
        if (!total) continue;
        int j0 = 0;
        using Word = typename std::conditional<PACKED, uint32_t, uint2>::type;
        for (uint32_t e0 = 0; e0 < total; e0 += 32 * kUnroll) {
          int jj[kUnroll];
          Word xw[kUnroll];
          uint32_t du[kUnroll];
#pragma unroll
          for (int k = 0; k < kUnroll; ++k) {
            const uint32_t eg = e0 + 32 * k;
            jj[k] = eg < total ? group_row(sh.fpref, ccnt, eg, j0) : 0;
            const uint32_t e = eg + lane;
            xw[k] = Word{};
            if (e < total) {
              const uint32_t slot = sh.frow[jj[k]] + (e - sh.fpref[jj[k]]);
              if constexpr (PACKED)
                xw[k] = ld_stream_u32(g.slots32 + slot, stream_pol);
              else
                xw[k] = ld_stream_u64(g.slots64 + slot, stream_pol);
            }
          }
#pragma unroll
          for (int k = 0; k < kUnroll; ++k) {
            uint32_t u;
            if constexpr (PACKED) u = xw[k] >> g.wbits; else u = xw[k].x;
            du[k] = (e0 + 32 * k + lane < total) ? dload(u) : 0u;
          }
#pragma unroll
          for (int k = 0; k < kUnroll; ++k) {
            const uint32_t e = e0 + 32 * k + lane;
            const bool valid = e < total;
            uint32_t u, w;
            if constexpr (PACKED) { u = xw[k] >> g.wbits; w = xw[k] & g.wmask; } else { u = xw[k].x; w = xw[k].y; }
            const uint32_t dv = sh.fd[jj[k]];
            const uint32_t nd = dv + w;
            const bool settled = (du[k] & kSettledBit) && du[k] != kInfDist;
            // predecessor: settled with d[u] + w == d[v] (engine.cpp:70, exact ties)
            const bool isp = valid && settled && (du[k] & kDistMask) + w == dv;
            const bool isi = valid && !settled && nd < du[k];
            if (isi && nd >= kDistMask) {  // settled-bit distances need d < 2^31 - 1
              abort = true;
              cause = kProfAbortDist;
            }
            const uint32_t bp = __ballot_sync(0xffffffffu, isp);
            const uint32_t bi = __ballot_sync(0xffffffffu, isi);
            if (isi) {
              const uint32_t q = iq_n + __popc(bi & lt);
              sh.qiu[q] = u;
              sh.qid[q] = nd;
            }
            if (isp) {
              const uint32_t q = pq_n + __popc(bp & lt);
              sh.qpu[q] = u;
              sh.qpv[q] = sh.fv[jj[k]];
              sh.qps[q] = sh.frow[jj[k]] + (e - sh.fpref[jj[k]]);
            }
            iq_n += __popc(bi);
            pq_n += __popc(bp);
          }
          __syncwarp();
          while (iq_n >= 32) drain_imp(32);
          while (pq_n >= 32) drain_pred(32);
        }
        __syncwarp();
        if (iq_n) drain_imp(iq_n);
        if (pq_n) drain_pred(pq_n);
      }
      if (near_n > kWNear) cause = kProfAbortNear;
      if (dag_len > dag_cap) cause = kProfAbortDag;
      if (near_n > kWNear || dag_len > dag_cap) abort = true;
      abort = __any_sync(0xffffffffu, abort);
      if (abort) break;
      if (lane == 0) dag_ends[nlev] = dag_len;
      tick(1);

      // ---------------- threshold: exact Delta from the near set + window rule
      auto near_min = [&]() {
        uint32_t m = kInfDist;
        for (uint32_t i = lane; i < near_n; i += 32) m = min(m, sh.nd[i] + sh.nmw[i]);
        return __reduce_min_sync(0xffffffffu, m);
      };
      uint32_t thr = near_min();
      c_near += near_n;
      bool done = near_n == 0 && far_len == 0;
      uint64_t far_min = kInfDist;
      while (!done && thr > F) {
        uint64_t F_new = F + W;
        if (far_min != kInfDist) {
          const uint64_t jump = far_min + W < thr ? far_min + W : static_cast<uint64_t>(thr);
          if (jump > F_new) F_new = jump;
        }
        const uint32_t Fn = F_new >= kInfDist ? kInfDist : static_cast<uint32_t>(F_new);
        c_far += far_len;
        ++c_refill;
        uint32_t keep = 0, lfar = kInfDist;
        // in-place compaction (one warp: a step reads before it writes)
        for (uint32_t c = 0; c < far_len; c += 32 * 4) {
          uint32_t u[4], du[4], mw[4], r0[4], r1[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) u[k] = c + 32 * k + lane < far_len ? __ldcg(far_q + c + 32 * k + lane) : 0u;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool v = c + 32 * k + lane < far_len;
            du[k] = v ? dload(u[k]) : kInfDist;
            mw[k] = v ? __ldg(g.minw + u[k]) : 0u;
            r0[k] = v ? __ldg(g.offsets + u[k]) : 0u;
            r1[k] = v ? __ldg(g.offsets + u[k] + 1) : 0u;
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool v = c + 32 * k + lane < far_len;
            // stale entries: settled, or already in the near set (improved below F)
            bool live = v && !(du[k] & kSettledBit) && du[k] != kInfDist;
            if (live && wfind(sh.hkey, u[k]) != kHEmpty) live = false;
            const bool to_near = live && du[k] < Fn;
            const bool stay = live && !to_near;
            const uint32_t bn = __ballot_sync(0xffffffffu, to_near);
            const uint32_t bs = __ballot_sync(0xffffffffu, stay);
            if (to_near) {
              const uint32_t np = near_n + __popc(bn & lt);
              bool created;
              const uint32_t h = np < kWNear ? wclaim(sh.hkey, u[k], created) : kHEmpty;
              if (h != kHEmpty) {
                sh.nu[np] = u[k];
                sh.nd[np] = du[k];
                sh.nmw[np] = mw[k];
                sh.nrow[np] = r0[k];
                sh.ndeg[np] = r1[k] - r0[k];
                sh.nh[np] = h;
                sh.hval[h] = np;
                thr = min(thr, du[k] + mw[k]);
              } else {
                abort = true;
              }
            }
            if (stay) {
              far_q[keep + __popc(bs & lt)] = u[k];
              lfar = min(lfar, du[k]);
            }
            near_n += __popc(bn);
            keep += __popc(bs);
            __syncwarp();
          }
        }
        thr = __reduce_min_sync(0xffffffffu, thr);
        far_min = __reduce_min_sync(0xffffffffu, lfar);
        far_len = keep;
        F = F_new;
        if (__any_sync(0xffffffffu, abort) || near_n > kWNear) {
          abort = true;
          cause = kProfAbortNear;
          break;
        }
        done = near_n == 0 && far_len == 0;
      }
      tick(2);
      if (abort || done) break;

      // ---------------- settle: d < Delta becomes level nlev (the next frontier)
      uint32_t nf = 0, kept = 0;
      for (uint32_t c = 0; c < near_n; c += 32) {
        const uint32_t i = c + lane;
        const bool have = i < near_n;
        uint32_t u = 0, d = 0, mw = 0, r = 0, dg = 0, h = 0;
        if (have) {
          u = sh.nu[i];
          d = sh.nd[i];
          mw = sh.nmw[i];
          r = sh.nrow[i];
          dg = sh.ndeg[i];
          h = sh.nh[i];
        }
        const bool st = have && d < thr;
        const uint32_t bs = __ballot_sync(0xffffffffu, st);
        const uint32_t bk = __ballot_sync(0xffffffffu, have && !st);
        __syncwarp();  // all entries of this step read before any is overwritten
        if (st) {
          const uint32_t q = nf + __popc(bs & lt);
          if (q < kWFront) {
            sh.fv[q] = u;
            sh.fd[q] = d;
            sh.frow[q] = r;
            sh.fpref[q + 1] = dg;  // scanned below
          }
          order[ord_len + q] = u;
          dist[u] = d | kSettledBit;
          sigma[u] = 0.0;
          delta[u] = 0.0;
          sh.hkey[h] = kHTomb;
        } else if (have) {
          const uint32_t q = kept + __popc(bk & lt);
          sh.nu[q] = u;
          sh.nd[q] = d;
          sh.nmw[q] = mw;
          sh.nrow[q] = r;
          sh.ndeg[q] = dg;
          sh.nh[q] = h;
          sh.hval[h] = q;
        }
        nf += __popc(bs);
        kept += __popc(bk);
        __syncwarp();
      }
      htomb += nf;
      near_n = kept;
      // frontier prefix of degrees (fpref[1..nf] hold degrees); a level above
      // kWFront is restaged chunk by chunk from the global order instead
      if (nf <= kWFront) {
        uint32_t carry = 0;
        for (uint32_t c = 0; c < nf; c += 32) {
          const uint32_t i = c + lane;
          uint32_t x = i < nf ? sh.fpref[i + 1] : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
          }
          __syncwarp();
          if (i < nf) sh.fpref[i + 1] = carry + x;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) sh.fpref[0] = 0;
      }
      fcnt = nf;
      fb = ord_len;
      ord_len += nf;
      ++nlev;
      if (lane == 0) lev[nlev] = ord_len;
      // hash index: rebuild when tombstones pile up
      if (htomb + near_n > kWHash / 4) {
        __syncwarp();
        for (uint32_t i = lane; i < kWHash; i += 32) sh.hkey[i] = kHEmpty;
        __syncwarp();
        for (uint32_t i = lane; i < near_n; i += 32) {
          bool created;
          const uint32_t h = wclaim(sh.hkey, sh.nu[i], created);  // near_n <= kWNear: never full
          sh.hval[h] = i;
          sh.nh[i] = h;
        }
        htomb = 0;
      }
      __syncwarp();
      tick(3);
    }

    if (abort) {
      if (lane == 0) p.abort_list[atomicAdd(p.abort_count, 1ULL)] = s_orig;
      if (PROF) {
        cause = __reduce_max_sync(0xffffffffu, cause);
        if (lane == 0 && cause >= 0) atomicAdd(p.prof + cause, 1ULL);
      }
      continue;
    }

    // ---------------- dependency accumulation, deepest level first: the DAG
    // edges of level L and the node-BC update of level L are independent, so
    // their loads are in flight together
    __threadfence_block();
    __syncwarp();
    for (uint32_t L = nlev - 1; L >= 1; --L) {
      const uint32_t b = __ldcg(dag_ends + L), e = L + 1 == nlev ? dag_len : __ldcg(dag_ends + L + 1);
      const uint32_t vb = __ldcg(lev + L), ve = L + 1 == nlev ? ord_len : __ldcg(lev + L + 1);
      for (uint32_t c = b; c < e; c += 32 * 4) {
        uint2 d[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) d[k] = c + 32 * k + lane < e ? __ldcg(dag + c + 32 * k + lane) : make_uint2(0, 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (c + 32 * k + lane >= e) continue;
          const uint32_t u = d[k].x, v = d[k].y;
          // reference term: sw / sigma[v] * (1.0 + delta[v])  (engine.cpp:201)
          const double cc = __ldcg(sigma + u) / __ldcg(sigma + v) * (1.0 + __ldcg(delta + v));
          atomicAdd(delta + u, cc);
          if (p.edge_bc) atomicAdd(p.edge_bc + __ldg(g.edge_id + __ldcg(dag_slot + c + 32 * k + lane)), cc);
        }
      }
      for (uint32_t q = vb + lane; q < ve; q += 32) {
        const uint32_t w = __ldcg(order + q);
        atomicAdd(p.node_bc + w, __ldcg(delta + w));
      }
      __threadfence_block();
      __syncwarp();
    }
    tick(4);
    if (lane == 0 && p.depth) p.depth[s_orig] = nlev;
    if (PROF && lane == 0) {
      for (int k = 0; k < 5; ++k) {
        atomicAdd(p.prof + kProfCyclesInit + k, t_phase[k]);
        t_phase[k] = 0;
      }
      atomicAdd(p.prof + kProfRounds, nlev);
      atomicAdd(p.prof + kProfDagEdges, dag_len);
      atomicAdd(p.prof + kProfRelaxSlots, c_relax);
      atomicAdd(p.prof + kProfNearScanned, c_near);
      atomicAdd(p.prof + kProfFarScanned, c_far);
      atomicAdd(p.prof + kProfRefills, c_refill);
    }
    if (PROF) {
      const unsigned ci = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c_impr));
      if (lane == 0) atomicAdd(p.prof + kProfImprovements, ci);
    }
    c_relax = c_near = c_far = c_refill = c_impr = c_rounds = 0;
  }
}

}  // namespace wbc_dev
