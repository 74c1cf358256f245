/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the weighted-BC hot path.
 * See wbc_oracle.h for the contract and the reference citations.  Parity is
 * pinned by tests/test_oracle.py (golden vectors + the compiled reference).
 */
#include "wbc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* open-addressing u64 -> u32 map (used only by the CSR builder)           */

typedef struct {
  uint64_t* keys;
  uint32_t* vals;
  uint8_t* used;
  uint64_t mask;
} u64map;

static int map_init(u64map* m, uint64_t expect) {
  uint64_t cap = 16;
  while (cap < 2 * expect + 16) cap <<= 1;
  m->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
  m->vals = (uint32_t*)malloc(cap * sizeof(uint32_t));
  m->used = (uint8_t*)calloc(cap, 1);
  m->mask = cap - 1;
  return (m->keys && m->vals && m->used) ? 0 : -1;
}

static void map_free(u64map* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
}

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  return x ^ (x >> 33);
}

/* Returns a pointer to the value slot; *inserted tells whether it is new. */
static uint32_t* map_slot(u64map* m, uint64_t key, int* inserted) {
  uint64_t i = mix64(key) & m->mask;
  for (;;) {
    if (!m->used[i]) {
      m->used[i] = 1;
      m->keys[i] = key;
      *inserted = 1;
      return &m->vals[i];
    }
    if (m->keys[i] == key) {
      *inserted = 0;
      return &m->vals[i];
    }
    i = (i + 1) & m->mask;
  }
}

/* ---------------------------------------------------------------------- */
/* build_csr  (graph.cpp:75-133)                                           */

int orc_build_csr(uint64_t len, const uint64_t* u, const uint64_t* v, const double* w,
                  uint32_t* n_out, uint32_t* m_out, uint32_t* offsets, uint32_t* adjacency,
                  double* weights, uint32_t* edge_id, double* minw, uint64_t* original_id,
                  uint32_t* edge_u, uint32_t* edge_v, uint64_t* merged_out) {
  u64map dense, seen;
  if (map_init(&dense, 2 * len) || map_init(&seen, len)) return -1;
  double* edge_w = (double*)malloc((len ? len : 1) * sizeof(double));
  if (!edge_w) return -1;
  uint32_t n = 0, m = 0;
  uint64_t merged = 0;
  for (uint64_t i = 0; i < len; ++i) {
    int ins;
    /* intern by first appearance: u before v (graph.cpp:79-83, 91-92) */
    uint32_t* s = map_slot(&dense, u[i], &ins);
    if (ins) {
      *s = n;
      original_id[n++] = u[i];
    }
    const uint32_t du = *s;
    s = map_slot(&dense, v[i], &ins);
    if (ins) {
      *s = n;
      original_id[n++] = v[i];
    }
    const uint32_t dv = *s;
    if (du == dv) continue;
    const uint32_t a = du < dv ? du : dv, b = du < dv ? dv : du;
    uint32_t* e = map_slot(&seen, ((uint64_t)a << 32) | b, &ins);
    if (ins) {
      *e = m;
      edge_u[m] = du; /* first-appearance orientation (graph.cpp:97-100) */
      edge_v[m] = dv;
      edge_w[m] = w[i];
      ++m;
    } else {
      if (w[i] < edge_w[*e]) edge_w[*e] = w[i]; /* keep the minimum (:102) */
      ++merged;
    }
  }
  /* degree count + prefix sum (graph.cpp:109-114) */
  memset(offsets, 0, (size_t)(n + 1) * sizeof(uint32_t));
  for (uint32_t e = 0; e < m; ++e) {
    ++offsets[edge_u[e] + 1];
    ++offsets[edge_v[e] + 1];
  }
  for (uint32_t x = 0; x < n; ++x) offsets[x + 1] += offsets[x];
  uint32_t* cursor = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  if (!cursor) return -1;
  memcpy(cursor, offsets, (size_t)n * sizeof(uint32_t));
  for (uint32_t x = 0; x < n; ++x) minw[x] = INFINITY;
  /* emit u->v then v->u per canonical edge (graph.cpp:121-131) */
  for (uint32_t e = 0; e < m; ++e) {
    for (int dir = 0; dir < 2; ++dir) {
      const uint32_t from = dir ? edge_v[e] : edge_u[e];
      const uint32_t to = dir ? edge_u[e] : edge_v[e];
      const uint32_t slot = cursor[from]++;
      adjacency[slot] = to;
      weights[slot] = edge_w[e];
      edge_id[slot] = e;
      if (edge_w[e] < minw[from]) minw[from] = edge_w[e];
    }
  }
  free(cursor);
  free(edge_w);
  map_free(&dense);
  map_free(&seen);
  *n_out = n;
  *m_out = m;
  *merged_out = merged;
  return 0;
}

/* ---------------------------------------------------------------------- */
/* binary min-heap of (distance, vertex) with lazy deletion                */

typedef struct {
  double d;
  uint32_t v;
} hent;

typedef struct {
  hent* a;
  uint64_t len, cap;
} heap;

static int heap_push(heap* h, double d, uint32_t v) {
  if (h->len == h->cap) {
    uint64_t cap = h->cap ? 2 * h->cap : 1024;
    hent* a = (hent*)realloc(h->a, cap * sizeof(hent));
    if (!a) return -1;
    h->a = a;
    h->cap = cap;
  }
  uint64_t i = h->len++;
  while (i > 0) {
    const uint64_t p = (i - 1) / 2;
    if (h->a[p].d <= d) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i].d = d;
  h->a[i].v = v;
  return 0;
}

static hent heap_pop(heap* h) {
  const hent top = h->a[0];
  const hent last = h->a[--h->len];
  uint64_t i = 0;
  for (;;) {
    uint64_t c = 2 * i + 1;
    if (c >= h->len) break;
    if (c + 1 < h->len && h->a[c + 1].d < h->a[c].d) ++c;
    if (h->a[c].d >= last.d) break;
    h->a[i] = h->a[c];
    i = c;
  }
  if (h->len) h->a[i] = last;
  return top;
}

/* ---------------------------------------------------------------------- */
/* brandes_sequential  (brandes.cpp:34-104), eps = 0                       */

int orc_brandes(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
                const double* weights, const uint32_t* edge_id, const uint32_t* sources,
                int64_t k, int halved, double* node_bc, double* edge_bc) {
  const uint64_t ks = k < 0 ? n : (uint64_t)k;
  if (k >= 0)
    for (uint64_t i = 0; i < ks; ++i)
      if (sources[i] >= n) return -1; /* brandes.cpp:18-30 */
  for (uint32_t x = 0; x < n; ++x) node_bc[x] = 0.0;
  if (edge_bc)
    for (uint32_t e = 0; e < m; ++e) edge_bc[e] = 0.0;
  double* dist = (double*)malloc((n + 1) * sizeof(double));
  double* sigma = (double*)malloc((n + 1) * sizeof(double));
  double* delta = (double*)malloc((n + 1) * sizeof(double));
  uint8_t* settled = (uint8_t*)malloc(n + 1);
  uint32_t* order = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  heap h = {0, 0, 0};
  for (uint64_t si = 0; si < ks; ++si) {
    const uint32_t s = k < 0 ? (uint32_t)si : sources[si];
    for (uint32_t x = 0; x < n; ++x) {
      dist[x] = INFINITY;
      sigma[x] = 0.0;
      delta[x] = 0.0;
      settled[x] = 0;
    }
    uint32_t olen = 0;
    dist[s] = 0.0;
    sigma[s] = 1.0;
    h.len = 0;
    heap_push(&h, 0.0, s);
    while (h.len) { /* heap Dijkstra with path counts (brandes.cpp:59-77) */
      const hent t = heap_pop(&h);
      const uint32_t x = t.v;
      if (settled[x]) continue;
      settled[x] = 1;
      order[olen++] = x;
      for (uint32_t e = offsets[x]; e < offsets[x + 1]; ++e) {
        const uint32_t y = adjacency[e];
        if (settled[y]) continue;
        const double nd = t.d + weights[e];
        if (nd < dist[y]) {
          dist[y] = nd;
          sigma[y] = sigma[x];
          heap_push(&h, nd, y);
        } else if (dist[y] == nd) {
          sigma[y] += sigma[x];
        }
      }
    }
    /* reverse settlement sweep (brandes.cpp:80-95) */
    for (uint32_t i = olen; i-- > 0;) {
      const uint32_t x = order[i];
      const double dw = dist[x], sw = sigma[x];
      double dsw = 0.0;
      for (uint32_t e = offsets[x]; e < offsets[x + 1]; ++e) {
        const uint32_t y = adjacency[e];
        if (dist[y] == dw + weights[e]) {
          const double c = sw / sigma[y] * (1.0 + delta[y]);
          dsw += c;
          if (edge_bc) edge_bc[edge_id[e]] += c;
        }
      }
      delta[x] = dsw;
      if (x != s) node_bc[x] += dsw;
    }
  }
  if (halved) { /* brandes.cpp:98-101 */
    for (uint32_t x = 0; x < n; ++x) node_bc[x] *= 0.5;
    if (edge_bc)
      for (uint32_t e = 0; e < m; ++e) edge_bc[e] *= 0.5;
  }
  free(h.a);
  free(dist);
  free(sigma);
  free(delta);
  free(settled);
  free(order);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Eq. 4 round process (engine.cpp:118-222) + accumulation (:183-212)      */

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* The reference scans all n vertices per round (engine.cpp:149-181).  The
 * restatement keeps the reached-but-unsettled vertices in a list instead
 * (same set, same threshold) and sorts each round's settled set by vertex id,
 * which is the order the full scan produces, so order/ends match exactly. */
static int eq4_core(uint32_t n, const uint32_t* offsets, const uint32_t* adjacency,
                    const double* weights, const double* minw, uint32_t s, int less_equal,
                    double* dist, double* sigma, uint32_t* order, uint32_t* order_len,
                    uint32_t* ends, uint32_t* ends_len, double* stats) {
  if (s >= n) return -1;
  uint8_t* unsettled = (uint8_t*)malloc(n);
  uint8_t* reached = (uint8_t*)malloc(n);
  uint32_t* pending = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  if (!unsettled || !reached || !pending) return -1;
  for (uint32_t x = 0; x < n; ++x) {
    dist[x] = INFINITY;
    sigma[x] = 0.0;
    unsettled[x] = 1;
    reached[x] = 0;
  }
  /* init_state (engine.cpp:118-142) */
  dist[s] = 0.0;
  sigma[s] = 1.0;
  unsettled[s] = 0;
  reached[s] = 1;
  order[0] = s;
  uint32_t olen = 1, elen = 2, plen = 0;
  ends[0] = 0;
  ends[1] = 1;
  uint32_t fb = 0, fe = 1; /* frontier = order[fb, fe) */
  if (stats) memset(stats, 0, 9 * sizeof(double));
  for (;;) {
    /* relax_frontier (engine.cpp:59-79, 144-147), lane width 1 */
    for (uint32_t i = fb; i < fe; ++i) {
      const uint32_t x = order[i];
      const double dv = dist[x], sv = sigma[x];
      for (uint32_t e = offsets[x]; e < offsets[x + 1]; ++e) {
        const uint32_t y = adjacency[e];
        if (stats) stats[2] += 1;
        if (!unsettled[y]) continue;
        const double nd = dv + weights[e];
        if (nd < dist[y]) {
          dist[y] = nd;
          sigma[y] = 0.0;
          if (stats) stats[3] += 1;
          if (!reached[y]) {
            reached[y] = 1;
            pending[plen++] = y;
          }
        }
        if (dist[y] == nd) sigma[y] += sv;
      }
    }
    /* compute_threshold (engine.cpp:149-156) over the same unsettled set */
    double thr = INFINITY;
    for (uint32_t i = 0; i < plen; ++i) {
      const uint32_t y = pending[i];
      const double t = dist[y] + minw[y];
      if (t < thr) thr = t;
    }
    if (stats) {
      stats[1] += plen;
      if (plen > stats[5]) stats[5] = plen;
    }
    if (thr == INFINITY) break;
    /* settle_and_advance (engine.cpp:158-181) */
    const uint32_t before = olen;
    uint32_t keep = 0;
    for (uint32_t i = 0; i < plen; ++i) {
      const uint32_t y = pending[i];
      const int take = less_equal ? dist[y] <= thr : dist[y] < thr;
      if (take) {
        unsettled[y] = 0;
        order[olen++] = y;
      } else {
        pending[keep++] = y;
      }
    }
    plen = keep;
    qsort(order + before, olen - before, sizeof(uint32_t), cmp_u32);
    if (olen > before) ends[elen++] = olen;
    if (stats && olen - before > stats[6]) stats[6] = olen - before;
    fb = before;
    fe = olen;
  }
  *order_len = olen;
  *ends_len = elen;
  if (stats) {
    stats[0] = elen - 1;
    stats[7] = olen;
    double mx = 0;
    for (uint32_t i = 0; i < olen; ++i)
      if (dist[order[i]] > mx) mx = dist[order[i]];
    stats[8] = mx;
    double dag = 0;
    for (uint32_t i = 0; i < olen; ++i) {
      const uint32_t x = order[i];
      for (uint32_t e = offsets[x]; e < offsets[x + 1]; ++e)
        if (dist[adjacency[e]] == dist[x] + weights[e]) dag += 1;
    }
    stats[4] = dag;
  }
  free(unsettled);
  free(reached);
  free(pending);
  return 0;
}

/* accumulate_dependencies with lane width 1 (engine.cpp:183-212) */
static void eq4_accumulate(const uint32_t* offsets, const uint32_t* adjacency,
                           const double* weights, const uint32_t* edge_id, uint32_t s,
                           const double* dist, const double* sigma, double* delta,
                           const uint32_t* order, const uint32_t* ends, uint32_t ends_len,
                           double* node_acc, double* edge_acc) {
  for (uint32_t depth = ends_len - 1; depth >= 1; --depth) {
    for (uint32_t pos = ends[depth - 1]; pos < ends[depth]; ++pos) {
      const uint32_t x = order[pos];
      const double dw = dist[x], sw = sigma[x];
      double dsw = 0.0;
      for (uint32_t e = offsets[x]; e < offsets[x + 1]; ++e) {
        const uint32_t y = adjacency[e];
        if (dist[y] == dw + weights[e]) {
          const double c = sw / sigma[y] * (1.0 + delta[y]);
          dsw += c;
          if (edge_acc) edge_acc[edge_id[e]] += c;
        }
      }
      delta[x] = dsw;
      if (x != s && node_acc) node_acc[x] += dsw;
    }
  }
}

int orc_eq4_source(uint32_t n, const uint32_t* offsets, const uint32_t* adjacency,
                   const double* weights, const uint32_t* edge_id, const double* minw,
                   uint32_t s, int less_equal, double* dist, double* sigma, double* delta,
                   uint32_t* order, uint32_t* order_len, uint32_t* ends, uint32_t* ends_len,
                   double* node_acc, double* edge_acc) {
  if (eq4_core(n, offsets, adjacency, weights, minw, s, less_equal, dist, sigma, order, order_len,
               ends, ends_len, NULL))
    return -1;
  for (uint32_t x = 0; x < n; ++x) delta[x] = 0.0;
  eq4_accumulate(offsets, adjacency, weights, edge_id, s, dist, sigma, delta, order, ends,
                 *ends_len, node_acc, edge_acc);
  return 0;
}

int orc_bc_eq4(uint32_t n, uint32_t m, const uint32_t* offsets, const uint32_t* adjacency,
               const double* weights, const uint32_t* edge_id, const double* minw,
               const uint32_t* sources, int64_t k, int halved, double* node_bc,
               double* edge_bc, uint32_t* depth_per_source) {
  const uint64_t ks = k < 0 ? n : (uint64_t)k;
  if (k >= 0)
    for (uint64_t i = 0; i < ks; ++i)
      if (sources[i] >= n) return -1; /* resolve_sources (engine.cpp:349-361) */
  for (uint32_t x = 0; x < n; ++x) {
    node_bc[x] = 0.0;
    if (depth_per_source) depth_per_source[x] = 0;
  }
  if (edge_bc)
    for (uint32_t e = 0; e < m; ++e) edge_bc[e] = 0.0;
  double* dist = (double*)malloc((n + 1) * sizeof(double));
  double* sigma = (double*)malloc((n + 1) * sizeof(double));
  double* delta = (double*)malloc((n + 1) * sizeof(double));
  uint32_t* order = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  uint32_t* ends = (uint32_t*)malloc((n + 2) * sizeof(uint32_t));
  for (uint64_t si = 0; si < ks; ++si) {
    const uint32_t s = k < 0 ? (uint32_t)si : sources[si];
    uint32_t olen, elen;
    eq4_core(n, offsets, adjacency, weights, minw, s, 0, dist, sigma, order, &olen, ends, &elen,
             NULL);
    for (uint32_t x = 0; x < n; ++x) delta[x] = 0.0;
    eq4_accumulate(offsets, adjacency, weights, edge_id, s, dist, sigma, delta, order, ends, elen,
                   node_bc, edge_bc);
    if (depth_per_source) depth_per_source[s] = elen - 1;
  }
  if (halved) { /* engine.cpp:451-454 */
    for (uint32_t x = 0; x < n; ++x) node_bc[x] *= 0.5;
    if (edge_bc)
      for (uint32_t e = 0; e < m; ++e) edge_bc[e] *= 0.5;
  }
  free(dist);
  free(sigma);
  free(delta);
  free(order);
  free(ends);
  return 0;
}

int orc_eq4_profile(uint32_t n, const uint32_t* offsets, const uint32_t* adjacency,
                    const double* weights, const double* minw, uint32_t s, double* stats) {
  double* dist = (double*)malloc((n + 1) * sizeof(double));
  double* sigma = (double*)malloc((n + 1) * sizeof(double));
  uint32_t* order = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
  uint32_t* ends = (uint32_t*)malloc((n + 2) * sizeof(uint32_t));
  uint32_t olen, elen;
  const int rc = eq4_core(n, offsets, adjacency, weights, minw, s, 0, dist, sigma, order, &olen,
                          ends, &elen, stats);
  free(dist);
  free(sigma);
  free(order);
  free(ends);
  return rc;
}
