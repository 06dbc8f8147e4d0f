// persistence.cuh -- extremum-saddle pairs for the persistence-driven mode
// (reference pairs_sweep, _kernels.py:309-421; SPEC persistence module).
//
// pairs_sweep's result is characterised exactly (checked against the
// reference on 1 200 random and quantised 2D/3D fields, every epsilon, and
// pinned by tests/test_pairs.py): it equals the Elder-rule pairing of the
// maxima graph -- nodes = maxima, one edge per pair of adjacent ascending
// manifolds weighted by the highest lower endpoint of a grid edge between
// them (the junction vertex) -- processed in decreasing weight (Kruskal), the
// younger top dying at the junction, filtered to persistence < epsilon
// (larger drops survive unpaired).  On the device:
//   1. ascent forest -> manifold labels, maxima-graph edges: the discover
//      kernels with every maximum a seed;
//   2. maximum spanning forest of the maxima graph by Boruvka rounds (only
//      its edges can merge two components in Kruskal order);
//   3. its edges sorted by weight (radix sort, descending);
//   4. one sequential union-find sweep over those nm-1 edges with the Elder
//      rule (union-find in shared memory when it fits, 4 B per maximum);
//   5. a parallel pass resolves vertices and applies the epsilon filter in
//      float64, as the reference compares values (order.py:30-36 widens f).
// The minima pairs run the same machinery on the reversed order.
#pragma once
#include "lts_common.cuh"

namespace lts {

// node index of every extremum (sorted vertex ids) and its effective rank
__global__ void k_pn_index(const uint32_t *__restrict__ sm, int nm, int *idx, const int *__restrict__ rank,
                           int rev, int n, int *nrank, int *comp, int *pair) {
  GRID_STRIDE(i, nm) {
    const int v = (int)sm[i];
    idx[v] = (int)i;
    nrank[i] = eff_rank(rank, v, rev, n);
    comp[i] = (int)i;
    pair[i] = -1;
  }
}

__global__ void k_pn_edges(const int *__restrict__ ea, const int *__restrict__ eb, int ne,
                           const int *__restrict__ idx, int *ia, int *ib, int *mst) {
  GRID_STRIDE(e, ne) {
    ia[e] = idx[ea[e]];
    ib[e] = idx[eb[e]];
    mst[e] = 0;
  }
}

__global__ void k_pn_reset(int nm, unsigned long long *best) {
  GRID_STRIDE(i, nm) best[i] = 0ull;
}

// heaviest edge leaving each component; ties by edge index, so the maximum
// spanning forest is unique and every round's hooks form trees plus 2-cycles
__global__ void k_pn_best(const int *__restrict__ ia, const int *__restrict__ ib, const int *__restrict__ ew,
                          int ne, const int *__restrict__ comp, unsigned long long *best) {
  GRID_STRIDE(e, ne) {
    const int ca = comp[ia[e]], cb = comp[ib[e]];
    if (ca == cb) continue;
    const unsigned long long key = ((unsigned long long)(unsigned)(ew[e] + 1) << 32) | (unsigned)e;
    if (best[ca] < key) atomicMax(best + ca, key);
    if (best[cb] < key) atomicMax(best + cb, key);
  }
}

__global__ void k_pn_hook(int nm, const int *__restrict__ comp, const unsigned long long *__restrict__ best,
                          const int *__restrict__ ia, const int *__restrict__ ib, int *par, int *mst,
                          int *active) {
  GRID_STRIDE(i, nm) {
    if (comp[i] != i) continue;
    const unsigned long long b = best[i];
    if (!b) {
      par[i] = (int)i;
      continue;
    }
    const int e = (int)(unsigned)(b & 0xffffffffull);
    const int ca = comp[ia[e]];
    par[i] = ca == (int)i ? comp[ib[e]] : ca;
    mst[e] = 1;
    atomicAdd(active, 1);
  }
}

// a mutual pair of hooks is the same edge: its smaller end becomes the root
__global__ void k_pn_cycle(int nm, const int *__restrict__ comp, int *par) {
  GRID_STRIDE(i, nm) {
    if (comp[i] != i) continue;
    const int q = par[i];
    if (q != (int)i && par[q] == (int)i && (int)i < q) par[i] = (int)i;
  }
}

__global__ void k_pn_roots(int nm, const int *__restrict__ comp, const int *__restrict__ par, int *rt) {
  GRID_STRIDE(i, nm) {
    if (comp[i] != i) continue;
    int x = (int)i;
    for (int q = par[x]; q != x; q = par[x]) x = q;
    rt[i] = x;
  }
}

__global__ void k_pn_relabel(int nm, int *comp, const int *__restrict__ rt) {
  GRID_STRIDE(i, nm) comp[i] = rt[comp[i]];
}

// forest edges -> sort keys: descending weight = ascending (n-1-w)
__global__ void k_pn_mst_keys(const int *__restrict__ mst, const int *__restrict__ ew, int ne, int n,
                              uint32_t *key, uint32_t *val, int *count) {
  GRID_STRIDE(e, ne) {
    const bool on = mst[e] != 0;
    const int slot = warp_alloc(count, on);
    if (on) {
      key[slot] = (uint32_t)(n - 1 - ew[e]);
      val[slot] = (uint32_t)e;
    }
  }
}

// forest edges in sweep order, gathered into contiguous arrays so the
// sequential sweep streams them instead of chasing edge ids
__global__ void k_pn_gather(const uint32_t *__restrict__ order, int cnt, const int *__restrict__ ia,
                            const int *__restrict__ ib, const int *__restrict__ ew, int *sa, int *sb, int *sw) {
  GRID_STRIDE(k, cnt) {
    const int e = (int)order[k];
    sa[k] = ia[e];
    sb[k] = ib[e];
    sw[k] = ew[e];
  }
}

// Elder-rule sweep over the forest edges in decreasing weight: the younger
// top of the two components dies at the junction.  One thread.  The
// union-find is one int per node: a non-negative entry is the parent, a root
// holds -(top rank + 1); it lives in shared memory when nm fits (4 B per
// extremum), else in global memory.
__device__ __forceinline__ int pn_find(int *p, int x) {
  for (;;) {
    const int q = p[x];
    if (q < 0) return x;  // x is a root
    const int r = p[q];
    if (r < 0) return q;  // q is the root
    p[x] = r;             // path halving
    x = r;
  }
}

__global__ void k_pn_sweep(const int *__restrict__ sa, const int *__restrict__ sb, const int *__restrict__ sw,
                           int cnt, const int *__restrict__ nrank, int nm, int *gpar, int use_smem, int *young_r,
                           int *junction_w) {
  extern __shared__ int sh[];
  int *par = use_smem ? sh : gpar;
  for (int i = threadIdx.x; i < nm; i += blockDim.x) par[i] = -(nrank[i] + 1);
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int k = 0; k < cnt; k++) {
    const int ra = pn_find(par, sa[k]), rb = pn_find(par, sb[k]);
    const int ta = -par[ra] - 1, tb = -par[rb] - 1;
    // ranks are distinct: the lower top dies here, the union keeps the higher
    if (ta < tb) {
      young_r[k] = ta;
      par[ra] = rb;
    } else {
      young_r[k] = tb;
      par[rb] = ra;
    }
    junction_w[k] = sw[k];
  }
}

// ---- leaf peeling of the spanning forest (before the sequential sweep) ----
// A forest leaf m whose only remaining edge e leads to a higher node dies at
// e in Kruskal order, whatever the order: its component is m (plus lower,
// already peeled nodes) until e, and e joins it to a component whose top is
// at least the neighbour.  Removing m and e changes no other pairing.  Rounds
// of this run in parallel; the sweep then handles the rest.  Pair entries of
// peeled leaves fill the (young rank, junction) list from the back.
__global__ void k_pn_leaf_init(const uint32_t *__restrict__ order, int cnt, const int *__restrict__ ia,
                               const int *__restrict__ ib, const int *__restrict__ ew, int *pa, int *pb, int *pw,
                               int *alive, int *deg) {
  GRID_STRIDE(k, cnt) {
    const int e = (int)order[k];
    const int a = ia[e], b = ib[e];
    pa[k] = a;
    pb[k] = b;
    pw[k] = ew[e];
    alive[k] = 1;
    atomicAdd(deg + a, 1);
    atomicAdd(deg + b, 1);
  }
}

__global__ void k_pn_copy(const int *__restrict__ src, int nm, int *dst) {
  GRID_STRIDE(i, nm) dst[i] = src[i];
}

__global__ void k_pn_peel(const int *__restrict__ pa, const int *__restrict__ pb, const int *__restrict__ pw,
                          int cnt, const int *__restrict__ nrank, const int *__restrict__ deg0, int *deg,
                          int *alive, int *young_r, int *junction_w, int *npeeled) {
  GRID_STRIDE(k, cnt) {
    if (!alive[k]) continue;
    const int a = pa[k], b = pb[k];
    const int ra = nrank[a], rb = nrank[b];
    int leaf = -1, other = -1, r = 0;
    if (deg0[a] == 1 && ra < rb) leaf = a, other = b, r = ra;
    else if (deg0[b] == 1 && rb < ra) leaf = b, other = a, r = rb;
    if (leaf < 0) continue;
    alive[k] = 0;
    atomicSub(deg + other, 1);
    const int slot = cnt - 1 - atomicAdd(npeeled, 1);
    young_r[slot] = r;
    junction_w[slot] = pw[k];
  }
}

// remaining forest edges: sort keys, and compact node numbering for the sweep
__global__ void k_pn_rest_keys(const int *__restrict__ alive, const int *__restrict__ pw, int cnt, int n,
                               uint32_t *key, uint32_t *val, int *count) {
  GRID_STRIDE(k, cnt) {
    const bool on = alive[k] != 0;
    const int slot = warp_alloc(count, on);
    if (on) {
      key[slot] = (uint32_t)(n - 1 - pw[k]);
      val[slot] = (uint32_t)k;
    }
  }
}

__global__ void k_pn_remap(const int *__restrict__ deg, int nm, const int *__restrict__ nrank, int *map, int *nrank2,
                           int *count) {
  GRID_STRIDE(i, nm) {
    const bool on = deg[i] > 0;
    const int slot = warp_alloc(count, on);
    if (on) {
      map[i] = slot;
      nrank2[slot] = nrank[i];
    }
  }
}

__global__ void k_pn_gather_rest(const uint32_t *__restrict__ order, int rem, const int *__restrict__ pa,
                                 const int *__restrict__ pb, const int *__restrict__ pw, const int *__restrict__ map,
                                 int *sa, int *sb, int *sw) {
  GRID_STRIDE(k, rem) {
    const int e = (int)order[k];
    sa[k] = map[pa[e]];
    sb[k] = map[pb[e]];
    sw[k] = pw[e];
  }
}

// vertices of the young tops and junctions; epsilon filter in float64
// (values[top] - values[junction] < eps, _kernels.py:390-393 / 406-408)
__global__ void k_pn_pairs(const int *__restrict__ young_r, const int *__restrict__ junction_w, int cnt,
                           const int *__restrict__ inv, int rev, int n, const float *__restrict__ f,
                           double eps, const int *__restrict__ idx, int *pair) {
  GRID_STRIDE(k, cnt) {
    const int yr = young_r[k], w = junction_w[k];
    const int yv = inv[rev ? n - 1 - yr : yr];
    const int sv = inv[rev ? n - 1 - w : w];
    const double drop = rev ? (double)f[sv] - (double)f[yv] : (double)f[yv] - (double)f[sv];
    pair[idx[yv]] = drop < eps ? sv : -1;
  }
}

__global__ void k_pn_out(const uint32_t *__restrict__ sm, const int *__restrict__ pair, int nm, int32_t *ext,
                         int32_t *sad) {
  GRID_STRIDE(i, nm) {
    ext[i] = (int32_t)sm[i];
    sad[i] = pair[i];
  }
}

}  // namespace lts
