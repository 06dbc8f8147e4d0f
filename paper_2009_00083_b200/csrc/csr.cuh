// csr.cuh -- the explicit-triangle-mesh kernels of the LTS path.
//
// The reference runs the same propagations on explicit 2-manifold meshes:
// classify_explicit (_kernels.py:159-187) counts the lower / upper link
// components of every vertex from per-vertex link edges, and discover_sweep /
// localize_regions (_kernels.py:194-303, 578-591) only ever see the symmetric
// CSR adjacency (triangulation.py:81-125).  On the device an explicit mesh is
// a Grid with ndim 0 carrying that CSR; every other kernel of the pass reads
// its neighbours through Nb<0> (lts_common.cuh).  The two grid kernels that
// exploit the stencil -- classification and the maxima-graph edge emission --
// have the CSR counterparts below.
#pragma once
#include "lts_common.cuh"
#include "classify.cuh"   // PTR_* kinds
#include "discover.cuh"   // EdgeHash, edge_global

namespace lts {

// Per vertex: extremum flags (bit0 minimum: no lower neighbour, bit1 maximum:
// no upper one), optionally the lower / upper link component counts (union-find
// over the vertex's link edges, as _count_side_components, _kernels.py:104-125)
// and the steepest ascent (PTR_ASC) or descent (PTR_DESC) pointer (self at an
// extremum of that kind), one thread per vertex.
template <int PTR>
__global__ void k_classify_csr(Grid g, const int32_t *__restrict__ rank, uint8_t *flags, int16_t *lower,
                               int16_t *upper, const int *__restrict__ lptr, const int *__restrict__ la,
                               const int *__restrict__ lb, int32_t *ptr) {
  GRID_STRIDE(v, g.n) {
    const int lo = g.cptr[v], deg = g.cptr[v + 1] - lo;
    const int rv = rank[v];
    unsigned up = 0;
    int best = -1, bu = (int)v, worst = 0x7fffffff, wu = (int)v;
    for (int k = 0; k < deg; k++) {
      const int u = g.cidx[lo + k];
      const int ru = rank[u];
      if (ru > rv) {
        up |= 1u << k;
        if (ru > best) { best = ru; bu = u; }
      } else if (ru < worst) {
        worst = ru;
        wu = u;
      }
    }
    const unsigned all = deg >= 32 ? 0xffffffffu : ((1u << deg) - 1u);
    const bool ismax = up == 0, ismin = (up & all) == all;
    if (flags) flags[v] = (uint8_t)((ismax ? FL_MAX : 0) | (ismin ? FL_MIN : 0));
    if (PTR == PTR_ASC) ptr[v] = ismax ? (int)v : bu;
    if (PTR == PTR_DESC) ptr[v] = ismin ? (int)v : wu;
    if (lower) {
      int par[32];
      for (int k = 0; k < deg; k++) par[k] = k;
      for (int e = lptr[v]; e < lptr[v + 1]; e++) {
        int ia = -1, ib = -1;
        for (int k = 0; k < deg; k++) {
          const int u = g.cidx[lo + k];
          if (u == la[e]) ia = k;
          if (u == lb[e]) ib = k;
        }
        if (ia < 0 || ib < 0) continue;
        if (((up >> ia) & 1u) != ((up >> ib) & 1u)) continue;
        while (par[ia] != ia) ia = par[ia];
        while (par[ib] != ib) ib = par[ib];
        if (ia != ib) par[ib] = ia;
      }
      int cl = 0, cu = 0;
      for (int k = 0; k < deg; k++)
        if (par[k] == k) {
          if ((up >> k) & 1u) cu++;
          else cl++;
        }
      lower[v] = (int16_t)cl;
      upper[v] = (int16_t)cu;
    }
  }
}

// largest vertex degree (the device rows hold kCsrK neighbours)
__global__ void k_max_degree(const int *__restrict__ cptr, int64_t n, int *out) {
  int m = 0;
  GRID_STRIDE(v, n) m = max(m, cptr[v + 1] - cptr[v]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Cross-manifold edges of the maxima graph on an explicit mesh, with the grid
// kernel's ownership rule: every mesh edge is owned by its lower endpoint u
// (weight = effective rank of u), and u emits one edge per distinct
// neighbouring manifold.
__global__ void k_edges_csr(Grid g, const int *__restrict__ rank, int rev, const int *__restrict__ M,
                            const uint8_t *__restrict__ vcls, int *ea, int *eb, int *ew, int *ecount,
                            unsigned long long *bestP, EdgeHash H) {
  const int n = (int)g.n;
  GRID_STRIDE(v, g.n) {
    const int a = M[v];
    const int rv = eff_rank(rank, (int)v, rev, n);
    int seen[kCsrK];
    int ns = 0;
    for (int e = g.cptr[v]; e < g.cptr[v + 1]; e++) {
      const int u = g.cidx[e];
      const int b = M[u];
      if (b == a || eff_rank(rank, u, rev, n) < rv) continue;
      bool dup = false;
      for (int i = 0; i < ns; i++) dup |= seen[i] == b;
      if (dup) continue;
      if (ns < kCsrK) seen[ns++] = b;
      edge_global(H, vcls, bestP, ea, eb, ew, ecount, a, b, rv);
    }
  }
}

inline void launch_classify_csr(const Grid &g, const int32_t *rank, uint8_t *flags, int16_t *lower,
                                int16_t *upper, const int *lptr, const int *la, const int *lb, int32_t *ptr,
                                int ptr_kind, cudaStream_t s) {
  const int nb = grid_blocks(g.n, 256);
  if (ptr_kind == PTR_ASC) k_classify_csr<PTR_ASC><<<nb, 256, 0, s>>>(g, rank, flags, lower, upper, lptr, la, lb, ptr);
  else if (ptr_kind == PTR_DESC) k_classify_csr<PTR_DESC><<<nb, 256, 0, s>>>(g, rank, flags, lower, upper, lptr, la, lb, ptr);
  else k_classify_csr<PTR_NONE><<<nb, 256, 0, s>>>(g, rank, flags, lower, upper, lptr, la, lb, ptr);
  g_launches++;
}

}  // namespace lts
