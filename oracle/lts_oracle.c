/*
 * lts_oracle.c -- CPU restatement of the reference LTS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the sm_100a
 * product path in paper_2009_00083_b200/csrc.  Only tests/, the smoke() entry
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never links or calls it.
 *
 * Every function restates the behaviour of one reference function (citations
 * are relative to /root/reference).  The restatement is pinned against the
 * reference's own numba kernels by tests/test_oracle_golden.py, which compares
 * it with fixtures produced by tests/golden/make_golden.py (that script imports
 * and runs the reference kernels).
 *
 * Conventions (reference triangulation.py:8): grid ids are x-fastest,
 * id = x + nx*(y + ny*z); dims[] = (nx, ny[, nz]).  Ranks and ids are int32
 * (n < 2^31 for every config).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_UNTOUCHED 0
#define ORC_PENDING 1
#define ORC_CLAIMED 2
#define ORC_FRINGE 3

/* ------------------------------------------------------------------------- */
/* stencil and link tables: triangulation.py:30-78                            */
/* ------------------------------------------------------------------------- */

static const int OFF2[6][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0},
                               {-1, 0, 0}, {0, -1, 0}, {-1, -1, 0}};
static const int OFF3[14][3] = {
    {1, 0, 0},  {0, 1, 0},  {0, 0, 1},  {1, 1, 0},   {1, 0, 1},
    {0, 1, 1},  {1, 1, 1},  {-1, 0, 0}, {0, -1, 0},  {0, 0, -1},
    {-1, -1, 0}, {-1, 0, -1}, {0, -1, -1}, {-1, -1, -1}};

typedef struct {
  int ndim, K, npairs;
  int64_t dims[3], n;
  int off[14][3];
  int pi[96], pj[96];
} grid_t;

static int is01(const int *d, int nd) {
  for (int a = 0; a < nd; a++)
    if (d[a] != 0 && d[a] != 1) return 0;
  return 1;
}

/* triangulation.py:52-66 (_face_triple): {0, a, b} is accepted when some
 * ordering x, y, z of the three points has y-x and z-y in {0,1}^d.  The
 * reference never requires z-x in {0,1}^d, hence the over-connected tables
 * (SURVEY F3); this restatement keeps that behaviour on purpose. */
static int face_triple(const int *a, const int *b, int nd) {
  int zero[3] = {0, 0, 0};
  const int *perm[6][3] = {{zero, a, b}, {zero, b, a}, {a, zero, b},
                           {b, zero, a}, {a, b, zero}, {b, a, zero}};
  for (int p = 0; p < 6; p++) {
    int d1[3], d2[3];
    for (int k = 0; k < nd; k++) {
      d1[k] = perm[p][1][k] - perm[p][0][k];
      d2[k] = perm[p][2][k] - perm[p][1][k];
    }
    if (is01(d1, nd) && is01(d2, nd)) return 1;
  }
  return 0;
}

static int grid_init(grid_t *g, int ndim, const int64_t *dims) {
  if (ndim != 2 && ndim != 3) return -1;
  g->ndim = ndim;
  g->K = ndim == 2 ? 6 : 14;
  g->n = 1;
  for (int a = 0; a < 3; a++) g->dims[a] = a < ndim ? dims[a] : 1;
  for (int a = 0; a < ndim; a++) {
    if (dims[a] < 2) return -1;
    g->n *= dims[a];
  }
  for (int k = 0; k < g->K; k++)
    for (int a = 0; a < 3; a++) g->off[k][a] = ndim == 2 ? OFF2[k][a] : OFF3[k][a];
  /* triangulation.py:69-75: pairs i<j in offset-table order */
  g->npairs = 0;
  for (int i = 0; i < g->K; i++)
    for (int j = i + 1; j < g->K; j++)
      if (face_triple(g->off[i], g->off[j], ndim)) {
        g->pi[g->npairs] = i;
        g->pj[g->npairs] = j;
        g->npairs++;
      }
  return 0;
}

/* neighbour k of v, or -1 when clipped by the grid boundary
 * (triangulation.py:142-149, _kernels.py:141-152) */
static inline int64_t nbr(const grid_t *g, int64_t v, int k) {
  int64_t x = v % g->dims[0];
  int64_t r = v / g->dims[0];
  int64_t y = r % g->dims[1];
  int64_t z = r / g->dims[1];
  int64_t a = x + g->off[k][0], b = y + g->off[k][1], c = z + g->off[k][2];
  if (a < 0 || a >= g->dims[0] || b < 0 || b >= g->dims[1] || c < 0 || c >= g->dims[2])
    return -1;
  return a + g->dims[0] * (b + g->dims[1] * c);
}

int orc_grid_tables(int ndim, int *offsets_out, int *pairs_out) {
  int64_t dims[3] = {2, 2, 2};
  grid_t g;
  if (grid_init(&g, ndim, dims)) return -1;
  for (int k = 0; k < g.K; k++)
    for (int a = 0; a < ndim; a++) offsets_out[k * ndim + a] = g.off[k][a];
  for (int e = 0; e < g.npairs; e++) {
    pairs_out[2 * e] = g.pi[e];
    pairs_out[2 * e + 1] = g.pj[e];
  }
  return g.npairs;
}

/* ------------------------------------------------------------------------- */
/* order field: order.py:86-91 (stable argsort by value, ties by id)          */
/* ------------------------------------------------------------------------- */

typedef struct {
  float v;
  int32_t id;
} vk_t;

static int cmp_vk(const void *pa, const void *pb) {
  const vk_t *a = (const vk_t *)pa, *b = (const vk_t *)pb;
  /* IEEE comparison: -0.0 == +0.0 */
  if (a->v < b->v) return -1;
  if (a->v > b->v) return 1;
  return (a->id > b->id) - (a->id < b->id);
}

/* returns number of non-finite values (order.py:35-36 raises FieldError) */
int64_t orc_order_field(const float *f, int64_t n, int32_t *rank, int32_t *inverse) {
  int64_t bad = 0;
  for (int64_t i = 0; i < n; i++)
    if (!isfinite(f[i])) bad++;
  if (bad) return bad;
  vk_t *a = (vk_t *)malloc(sizeof(vk_t) * (size_t)n);
  for (int64_t i = 0; i < n; i++) {
    a[i].v = f[i];
    a[i].id = (int32_t)i;
  }
  qsort(a, (size_t)n, sizeof(vk_t), cmp_vk);
  for (int64_t i = 0; i < n; i++) {
    inverse[i] = a[i].id;
    rank[a[i].id] = (int32_t)i;
  }
  free(a);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* classification: _kernels.py:106-156 (classify_grid), critical.py:95-112    */
/* ------------------------------------------------------------------------- */

static int uf_root(int *p, int x) {
  while (p[x] != x) {
    p[x] = p[p[x]];
    x = p[x];
  }
  return x;
}

/* components of the link vertices with side == want (_kernels.py:106-125) */
static int side_components(const grid_t *g, const signed char *side, int want) {
  int p[14];
  for (int i = 0; i < g->K; i++) p[i] = i;
  for (int e = 0; e < g->npairs; e++) {
    int a = g->pi[e], b = g->pj[e];
    if (side[a] == want && side[b] == want) {
      int ra = uf_root(p, a), rb = uf_root(p, b);
      if (ra != rb) p[rb] = ra;
    }
  }
  int c = 0;
  for (int i = 0; i < g->K; i++)
    if (side[i] == want && uf_root(p, i) == i) c++;
  return c;
}

int orc_classify_grid(const int32_t *rank, int ndim, const int64_t *dims, int16_t *lower,
                      int16_t *upper, int nthreads) {
  grid_t g;
  if (grid_init(&g, ndim, dims)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t v = 0; v < g.n; v++) {
    signed char side[14];
    for (int k = 0; k < g.K; k++) {
      int64_t u = nbr(&g, v, k);
      side[k] = u < 0 ? -1 : (rank[u] > rank[v] ? 1 : 0);
    }
    lower[v] = (int16_t)side_components(&g, side, 0);
    upper[v] = (int16_t)side_components(&g, side, 1);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* binary max-heap keyed by rank (_kernels.py:28-65) and union-find (:68-77)  */
/* ------------------------------------------------------------------------- */

typedef struct {
  int64_t *key;
  int64_t *val;
  int64_t size;
} heap_t;

static void hpush(heap_t *h, int64_t key, int64_t val) {
  int64_t i = h->size++;
  h->key[i] = key;
  h->val[i] = val;
  while (i > 0) {
    int64_t p = (i - 1) >> 1;
    if (h->key[p] >= h->key[i]) break;
    int64_t tk = h->key[p], tv = h->val[p];
    h->key[p] = h->key[i];
    h->val[p] = h->val[i];
    h->key[i] = tk;
    h->val[i] = tv;
    i = p;
  }
}

static int64_t hpop(heap_t *h, int64_t *key_out) {
  int64_t key = h->key[0], val = h->val[0];
  h->size--;
  if (h->size > 0) {
    h->key[0] = h->key[h->size];
    h->val[0] = h->val[h->size];
    int64_t i = 0;
    for (;;) {
      int64_t l = 2 * i + 1;
      if (l >= h->size) break;
      int64_t big = l;
      if (l + 1 < h->size && h->key[l + 1] > h->key[l]) big = l + 1;
      if (h->key[i] >= h->key[big]) break;
      int64_t tk = h->key[i], tv = h->val[i];
      h->key[i] = h->key[big];
      h->val[i] = h->val[big];
      h->key[big] = tk;
      h->val[big] = tv;
      i = big;
    }
  }
  if (key_out) *key_out = key;
  return val;
}

static int64_t uf_find64(int32_t *parent, int64_t x) {
  int64_t root = x;
  while (parent[root] != root) root = parent[root];
  while (parent[x] != root) {
    int64_t nx = parent[x];
    parent[x] = (int32_t)root;
    x = nx;
  }
  return root;
}

/* ------------------------------------------------------------------------- */
/* region discovery: _kernels.py:194-303 (discover_sweep)                     */
/* One global descending sweep over claimed/fringe candidates.  Outputs per   */
/* vertex state and owner (root slot), per seed slot saddle/parked/topseed.   */
/* ------------------------------------------------------------------------- */

int orc_discover_sweep(const int32_t *rank, int ndim, const int64_t *dims, const int32_t *seeds,
                       int64_t nseeds, int8_t *state, int32_t *owner, int32_t *saddle,
                       uint8_t *parked, int32_t *topseed) {
  grid_t g;
  if (grid_init(&g, ndim, dims)) return -1;
  int64_t n = g.n;
  int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseeds + 1));
  int32_t *seedslot = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  heap_t h;
  h.key = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  h.val = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  h.size = 0;
  for (int64_t v = 0; v < n; v++) {
    state[v] = ORC_UNTOUCHED;
    owner[v] = -1;
    seedslot[v] = -1;
  }
  for (int64_t i = 0; i < nseeds; i++) {
    parent[i] = (int32_t)i;
    saddle[i] = -1;
    parked[i] = 0;
    topseed[i] = rank[seeds[i]];
    seedslot[seeds[i]] = (int32_t)i;
  }
  for (int64_t i = 0; i < nseeds; i++) {
    hpush(&h, rank[seeds[i]], seeds[i]);
    state[seeds[i]] = ORC_PENDING;
  }
  int err = 0;
  int64_t roots[14];
  while (h.size > 0) {
    int64_t rv;
    int64_t v = hpop(&h, &rv);
    if (state[v] >= ORC_CLAIMED) continue;
    /* scan the upper link (_kernels.py:236-254) */
    int blocked = 0, nroots = 0;
    for (int k = 0; k < g.K; k++) {
      int64_t u = nbr(&g, v, k);
      if (u < 0 || rank[u] <= rv) continue;
      if (state[u] == ORC_CLAIMED) {
        int64_t r = uf_find64(parent, owner[u]);
        int seen = 0;
        for (int j = 0; j < nroots; j++)
          if (roots[j] == r) seen = 1;
        if (!seen) roots[nroots++] = r;
        if (parked[r]) blocked = 1;
      } else {
        blocked = 1; /* untouched or fringe territory above */
      }
    }
    if (seedslot[v] >= 0) { /* a seed claims itself (:256-265) */
      owner[v] = seedslot[v];
      state[v] = ORC_CLAIMED;
      for (int k = 0; k < g.K; k++) {
        int64_t u = nbr(&g, v, k);
        if (u >= 0 && state[u] == ORC_UNTOUCHED) {
          state[u] = ORC_PENDING;
          hpush(&h, rank[u], u);
        }
      }
      continue;
    }
    if (nroots == 0) { /* :267-271 */
      err = 1;
      state[v] = ORC_FRINGE;
      continue;
    }
    if (blocked) { /* park every unparked root at v (:273-280) */
      state[v] = ORC_FRINGE;
      for (int j = 0; j < nroots; j++) {
        int64_t r = roots[j];
        if (!parked[r]) {
          parked[r] = 1;
          saddle[r] = (int32_t)v;
        }
      }
      continue;
    }
    /* merge, keep the max topseed, claim v (:282-298) */
    int64_t root = roots[0];
    for (int j = 1; j < nroots; j++) {
      int64_t ra = uf_find64(parent, root), rb = uf_find64(parent, roots[j]);
      if (ra != rb) {
        parent[rb] = (int32_t)ra;
        if (topseed[rb] > topseed[ra]) topseed[ra] = topseed[rb];
        root = ra;
      }
    }
    owner[v] = (int32_t)uf_find64(parent, root);
    state[v] = ORC_CLAIMED;
    for (int k = 0; k < g.K; k++) {
      int64_t u = nbr(&g, v, k);
      if (u >= 0 && state[u] == ORC_UNTOUCHED) {
        state[u] = ORC_PENDING;
        hpush(&h, rank[u], u);
      }
    }
  }
  for (int64_t v = 0; v < n; v++) /* :300-302 */
    if (state[v] == ORC_CLAIMED) owner[v] = (int32_t)uf_find64(parent, owner[v]);
  free(parent);
  free(seedslot);
  free(h.key);
  free(h.val);
  return err;
}

/* ------------------------------------------------------------------------- */
/* localized simplification: _kernels.py:424-591                              */
/* ------------------------------------------------------------------------- */

#define ORC_BIG ((int64_t)1 << 62)

typedef struct {
  int32_t id;
  int32_t pos;
} idpos_t;

static int cmp_idpos(const void *pa, const void *pb) {
  const idpos_t *a = (const idpos_t *)pa, *b = (const idpos_t *)pb;
  return (a->id > b->id) - (a->id < b->id);
}

/* membership: position of vertex u inside the region list, or -1
 * (_kernels.py:428-440) */
static int64_t local_pos(const idpos_t *s, int64_t k, int64_t u) {
  int64_t lo = 0, hi = k;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (s[mid].id < u)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < k && s[lo].id == u) return s[lo].pos;
  return -1;
}

/* _kernels.py:443-575; verts[0] is the saddle, verts[1..] by ascending rank.
 * Returns passes; *status = 0 ok, 1 no admissible boundary minimum, 2 cap. */
static int localize_one(const grid_t *g, const int32_t *verts, int64_t k, const int32_t *rank,
                        int max_iter, int32_t *out_l, int *status) {
  idpos_t *sorted = (idpos_t *)malloc(sizeof(idpos_t) * (size_t)k);
  for (int64_t p = 0; p < k; p++) {
    sorted[p].id = verts[p];
    sorted[p].pos = (int32_t)p;
  }
  qsort(sorted, (size_t)k, sizeof(idpos_t), cmp_idpos);
  /* neighbour positions inside the region, computed once (same membership
   * predicate as the reference's per-probe binary search) */
  int K = g->K;
  int64_t *nq = (int64_t *)malloc(sizeof(int64_t) * (size_t)(k * K));
  unsigned char *has_out = (unsigned char *)calloc((size_t)k, 1);
  int64_t srank = rank[verts[0]];
  for (int64_t p = 0; p < k; p++) {
    for (int kk = 0; kk < K; kk++) {
      int64_t u = nbr(g, verts[p], kk);
      nq[p * K + kk] = u < 0 ? -1 : local_pos(sorted, k, u);
      if (p >= 1 && u >= 0 && rank[u] < srank) has_out[p] = 1; /* :460-468 */
    }
  }
  int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t p = 0; p < k; p++) cur[p] = p;
  cur[0] = ORC_BIG;
  int64_t v0 = -1;
  for (int64_t p = 1; p < k; p++)
    if (has_out[p]) {
      v0 = p;
      break;
    }
  int passes = 0;
  *status = 0;
  if (v0 < 0) { /* :479-480 */
    *status = 1;
    free(sorted);
    free(nq);
    free(has_out);
    free(cur);
    return 0;
  }
  cur[v0] = -ORC_BIG;
  heap_t h;
  h.key = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  h.val = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  unsigned char *inheap = (unsigned char *)malloc((size_t)k);
  unsigned char *is_min = (unsigned char *)calloc((size_t)k, 1);
  int64_t *new_l = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
  for (;;) {
    /* descending flood from the junction (:491-510) */
    memset(inheap, 0, (size_t)k);
    h.size = 0;
    hpush(&h, cur[0], 0);
    inheap[0] = 1;
    int64_t extracted = 0;
    while (h.size > 0) {
      int64_t p = hpop(&h, NULL);
      new_l[p] = k - 1 - extracted;
      extracted++;
      for (int kk = 0; kk < K; kk++) {
        int64_t q = nq[p * K + kk];
        if (q >= 0 && !inheap[q]) {
          inheap[q] = 1;
          hpush(&h, cur[q], q);
        }
      }
    }
    memcpy(cur, new_l, sizeof(int64_t) * (size_t)k);
    passes++;
    /* unauthorized minima (:512-526) */
    int bad = 0;
    for (int64_t p = 1; p < k; p++) {
      int mn = 1;
      for (int kk = 0; kk < K; kk++) {
        int64_t q = nq[p * K + kk];
        if (q >= 0 && cur[q] < cur[p]) {
          mn = 0;
          break;
        }
      }
      is_min[p] = (unsigned char)mn;
      if (mn && !has_out[p]) bad = 1;
    }
    if (!bad) break;
    if (passes >= max_iter) {
      *status = 2;
      break;
    }
    /* ascending flood from all admissible minima (:531-552) */
    memset(inheap, 0, (size_t)k);
    h.size = 0;
    for (int64_t p = 1; p < k; p++)
      if (is_min[p] && has_out[p]) {
        inheap[p] = 1;
        hpush(&h, -cur[p], p);
      }
    extracted = 0;
    while (h.size > 0) {
      int64_t p = hpop(&h, NULL);
      new_l[p] = extracted++;
      for (int kk = 0; kk < K; kk++) {
        int64_t q = nq[p * K + kk];
        if (q >= 0 && !inheap[q]) {
          inheap[q] = 1;
          hpush(&h, -cur[q], q);
        }
      }
    }
    memcpy(cur, new_l, sizeof(int64_t) * (size_t)k);
    passes++;
    /* unauthorized maxima (:554-568) */
    bad = 0;
    for (int64_t p = 1; p < k && !bad; p++) {
      int mx = 1;
      for (int kk = 0; kk < K; kk++) {
        int64_t q = nq[p * K + kk];
        if (q >= 0 && cur[q] > cur[p]) {
          mx = 0;
          break;
        }
      }
      if (mx) bad = 1;
    }
    if (!bad) break;
    if (passes >= max_iter) {
      *status = 2;
      break;
    }
  }
  for (int64_t p = 0; p < k; p++) out_l[p] = (int32_t)cur[p];
  free(sorted);
  free(nq);
  free(has_out);
  free(cur);
  free(h.key);
  free(h.val);
  free(inheap);
  free(is_min);
  free(new_l);
  return passes;
}

/* _kernels.py:578-591 (prange over regions) */
int orc_localize_regions(const int64_t *region_ptr, int64_t nregions, const int32_t *region_verts,
                         const int32_t *rank, int ndim, const int64_t *dims, int max_iter,
                         int32_t *local_rank, int32_t *n_iters, int32_t *status, int nthreads) {
  grid_t g;
  if (grid_init(&g, ndim, dims)) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t r = 0; r < nregions; r++) {
    int64_t lo = region_ptr[r], hi = region_ptr[r + 1];
    int st = 0;
    n_iters[r] = localize_one(&g, region_verts + lo, hi - lo, rank, max_iter, local_rank + lo, &st);
    status[r] = st;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* integration: SPEC.md:330-338 / 386 -- new rank = position in the          */
/* lexicographic key order (primary, secondary, tertiary).  Literal sort.     */
/* ------------------------------------------------------------------------- */

typedef struct {
  int64_t k1, k2, k3;
  int32_t id;
} ikey_t;

static int cmp_ikey(const void *pa, const void *pb) {
  const ikey_t *a = (const ikey_t *)pa, *b = (const ikey_t *)pb;
  if (a->k1 != b->k1) return a->k1 < b->k1 ? -1 : 1;
  if (a->k2 != b->k2) return a->k2 < b->k2 ? -1 : 1;
  if (a->k3 != b->k3) return a->k3 < b->k3 ? -1 : 1;
  return (a->id > b->id) - (a->id < b->id); /* never reached: keys are unique */
}

/* region r = region_verts[region_ptr[r] .. region_ptr[r+1]), saddle first;
 * regionId(r) = topseed_rank[r].  Returns the number of key collisions. */
int64_t orc_integrate(const int32_t *rank, int64_t n, const int64_t *region_ptr, int64_t nregions,
                      const int32_t *region_verts, const int32_t *local_rank,
                      const int32_t *topseed_rank, int32_t *newrank) {
  ikey_t *a = (ikey_t *)malloc(sizeof(ikey_t) * (size_t)n);
  for (int64_t v = 0; v < n; v++) {
    a[v].k1 = rank[v];
    a[v].k2 = 0;
    a[v].k3 = 0;
    a[v].id = (int32_t)v;
  }
  for (int64_t r = 0; r < nregions; r++) {
    int64_t lo = region_ptr[r], hi = region_ptr[r + 1];
    int32_t s = region_verts[lo];
    for (int64_t i = lo + 1; i < hi; i++) {
      int32_t v = region_verts[i];
      a[v].k1 = rank[s];
      a[v].k2 = local_rank[i];
      a[v].k3 = topseed_rank[r];
    }
    a[s].k2 = ORC_BIG;
    a[s].k3 = ORC_BIG;
  }
  qsort(a, (size_t)n, sizeof(ikey_t), cmp_ikey);
  int64_t coll = 0;
  for (int64_t i = 0; i < n; i++) {
    newrank[a[i].id] = (int32_t)i;
    if (i > 0 && a[i].k1 == a[i - 1].k1 && a[i].k2 == a[i - 1].k2 && a[i].k3 == a[i - 1].k3 &&
        a[i].k2 != ORC_BIG)
      coll++;
  }
  free(a);
  return coll;
}

/* ------------------------------------------------------------------------- */
/* realization sweep: _kernels.py:84-99 on a float32 array with zeta = 0.0    */
/* (ZetaMode.ULP_DECREMENT, order.py:81-82).  The reference computes          */
/* g[prev] - zeta and np.nextafter(g[prev], -inf) in float64 and stores the   */
/* result into the float32 array, so a lowered vertex receives a copy of its  */
/* predecessor's value (0.0 becomes -0.0).  SURVEY F4 / contract D1.          */
/* ------------------------------------------------------------------------- */

void orc_realize_sweep_f32(float *gv, const int32_t *inverse, int64_t n) {
  if (n < 2) return;
  int32_t prev = inverse[n - 1];
  for (int64_t i = n - 2; i >= 0; i--) {
    int32_t v = inverse[i];
    if (gv[v] > gv[prev] || (gv[v] == gv[prev] && v > prev)) {
      double gp = (double)gv[prev];
      double nv = gp - 0.0;
      if (nv >= gp) nv = nextafter(gp, -INFINITY);
      gv[v] = (float)nv;
    }
    prev = v;
  }
}

/* ------------------------------------------------------------------------- */
/* truncated extremum-saddle pairing: _kernels.py:309-421 (pairs_sweep)        */
/* Descending propagations from every seed maximum; a component stops once    */
/* its drop from its highest seed reaches eps (persistent) or it meets spent  */
/* territory; the younger components meeting at a junction die there and are  */
/* paired with it when their drop is below eps (Elder rule).                  */
/* pair_saddle[i] = junction vertex of seeds[i], or -1 (survivor).            */
/* ------------------------------------------------------------------------- */

int orc_pairs_sweep(const int32_t *rank, const double *values, int ndim, const int64_t *dims,
                    const int32_t *seeds, int64_t nseeds, double eps, int32_t *pair_saddle) {
  grid_t g;
  if (grid_init(&g, ndim, dims)) return -1;
  int64_t n = g.n;
  int8_t *state = (int8_t *)malloc((size_t)n);
  int32_t *owner = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *seedslot = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseeds + 1));
  int32_t *topslot = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nseeds + 1));
  uint8_t *stopped = (uint8_t *)calloc((size_t)(nseeds + 1), 1);
  heap_t h;
  h.key = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  h.val = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  h.size = 0;
  for (int64_t v = 0; v < n; v++) {
    state[v] = ORC_UNTOUCHED;
    owner[v] = -1;
    seedslot[v] = -1;
  }
  for (int64_t i = 0; i < nseeds; i++) {
    parent[i] = (int32_t)i;
    topslot[i] = (int32_t)i;
    pair_saddle[i] = -1;
    seedslot[seeds[i]] = (int32_t)i;
  }
  for (int64_t i = 0; i < nseeds; i++) {
    hpush(&h, rank[seeds[i]], seeds[i]);
    state[seeds[i]] = ORC_PENDING;
  }
  int err = 0;
  int64_t roots[14];
  while (h.size > 0) {
    int64_t rv;
    int64_t v = hpop(&h, &rv);
    if (state[v] >= ORC_CLAIMED) continue;
    if (seedslot[v] >= 0) { /* a seed claims itself and opens its link (:343-351) */
      owner[v] = seedslot[v];
      state[v] = ORC_CLAIMED;
      for (int k = 0; k < g.K; k++) {
        int64_t u = nbr(&g, v, k);
        if (u >= 0 && state[u] == ORC_UNTOUCHED) {
          state[u] = ORC_PENDING;
          hpush(&h, rank[u], u);
        }
      }
      continue;
    }
    int beyond = 0, nroots = 0; /* upper link (:353-372) */
    for (int k = 0; k < g.K; k++) {
      int64_t u = nbr(&g, v, k);
      if (u < 0 || rank[u] <= rv) continue;
      if (state[u] == ORC_CLAIMED) {
        int64_t r = uf_find64(parent, owner[u]);
        int seen = 0;
        for (int j = 0; j < nroots; j++)
          if (roots[j] == r) seen = 1;
        if (!seen) roots[nroots++] = r;
        if (stopped[r]) beyond = 1;
      } else {
        beyond = 1;
      }
    }
    if (nroots == 0) { /* :374-377 */
      err = 1;
      state[v] = ORC_FRINGE;
      continue;
    }
    int64_t elder = -1; /* the root with the highest seed (:379-384) */
    if (!beyond) {
      elder = roots[0];
      for (int j = 1; j < nroots; j++)
        if (rank[seeds[topslot[roots[j]]]] > rank[seeds[topslot[elder]]]) elder = roots[j];
    }
    for (int j = 0; j < nroots; j++) { /* the others stop here (:386-393) */
      int64_t r = roots[j];
      if (r == elder || stopped[r]) continue;
      stopped[r] = 1;
      if (values[seeds[topslot[r]]] - values[v] < eps) pair_saddle[topslot[r]] = (int32_t)v;
    }
    int64_t root = roots[0]; /* merge (:395-402) */
    for (int j = 1; j < nroots; j++) {
      int64_t ra = uf_find64(parent, root), rb = uf_find64(parent, roots[j]);
      if (ra != rb) {
        parent[rb] = (int32_t)ra;
        if (rank[seeds[topslot[rb]]] > rank[seeds[topslot[ra]]]) topslot[ra] = topslot[rb];
        root = ra;
      }
    }
    int64_t r = uf_find64(parent, root);
    owner[v] = (int32_t)r;
    state[v] = ORC_CLAIMED;
    if (beyond || values[seeds[topslot[r]]] - values[v] >= eps) { /* :406-408 */
      stopped[r] = 1;
      continue;
    }
    stopped[r] = 0;
    for (int k = 0; k < g.K; k++) {
      int64_t u = nbr(&g, v, k);
      if (u >= 0 && state[u] == ORC_UNTOUCHED) {
        state[u] = ORC_PENDING;
        hpush(&h, rank[u], u);
      }
    }
  }
  free(state);
  free(owner);
  free(seedslot);
  free(parent);
  free(topslot);
  free(stopped);
  free(h.key);
  free(h.val);
  return err;
}
